"""Shared-memory bank conflicts per instruction from an ncu source-page CSV
(--page source --csv --print-source sass).  usage: python tools/conflicts_from_csv.py src.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
out = []
seq = []
for r in rows[2:]:
    try:
        seq.append((r[1].strip()[:56], int(r[ix["Instructions Executed"]] or 0),
                    int(r[ix["L1 Wavefronts Shared Excessive"]] or 0), int(r[ix["L1 Wavefronts Shared"]] or 0),
                    int(r[ix["L1 Wavefronts Shared Ideal"]] or 0)))
    except (ValueError, IndexError):
        pass
tot_ex = sum(s[2] for s in seq)
tot = sum(s[3] for s in seq)
ti = sum(s[1] for s in seq)
print(f"{sys.argv[1]}: warp inst {ti}, shared wavefronts {tot}, excessive {tot_ex}")
groups = {}
for i, (s, n, e, w, wi) in enumerate(seq):
    if e > 0:
        key = (s.split()[0], n, w // max(n, 1), wi // max(n, 1))
        groups.setdefault(key, [0, i])[0] += e
for (op, n, wpi, wipi), (e, i) in sorted(groups.items(), key=lambda x: -x[1][0])[:12]:
    ctx = " | ".join(x[0][:40] for x in seq[max(0, i - 2):i + 2])
    print(f"  {op:14s} exec {n:7d} wavefronts/inst {wpi} (ideal {wipi}) excess {e:8d}  e.g. {ctx}")
