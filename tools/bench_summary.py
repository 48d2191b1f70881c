import json,sys
r=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(r["value"], r["ms_per_step"], r.get("roofline",{}).get("frac"), r.get("e2e",{}).get("value"), r["roofline"]["kernel_ms"])
for k,v in r.get("configs",{}).items():
    imp=(v.get("implementations") or {}).get("ms_per_step") or {}
    print(k, round(v.get("value"),2), round(v.get("ms_per_step"),4), {a[:12]:round(b,4) for a,b in imp.items()}, v.get("unsettled_stacks"), (v.get("parity") or {}).get("image0_bit_exact_vs_oracle") if isinstance(v.get("parity"), dict) else "")
