import itertools
def dsw(C):
    x = C >> 3
    f = (x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7
    f ^= ((C >> 6) & 1) * 6
    return C ^ f
def rev(i, bits):
    r = 0
    for b in range(bits): r |= ((i >> b) & 1) << (bits - 1 - b)
    return r
def gather_cost(n, perm):
    T = n // 32; lt = T.bit_length() - 1
    W = max(T, 32); LPR = W >> lt
    def belem(j): return (j >> (0 if lt > 5 else 5 - lt)) * (W * 32) + (j & (LPR - 1)) * n
    tot = 0
    for warp in range(4):
        for m in range(32):
            # 64-bit loads: wavefronts = max over 32 banks of distinct 8B words (per warp)
            banks = {}
            for lane in range(32):
                tid = warp * 32 + lane
                j = perm(tid >> lt)
                tl = tid & (T - 1)
                e = belem(j) + m * T + (rev(tl, lt) if lt else 0)
                C = e >> 1
                addr = dsw(C) * 16 + (e & 1) * 8
                b = (addr // 4) % 32
                banks.setdefault(b, set()).add(addr // 8)
            tot += max(len(v) for v in banks.values())
    return tot / (4 * 32)
if __name__ == "__main__":
    for n in (64, 128, 256, 512):
        T = n // 32; lpw = 32 // T
        ident = lambda j: j
        best = None
        # permutations of the low log2(lpw) bits of the line index
        nb = lpw.bit_length() - 1
        for p in itertools.permutations(range(nb)):
            def perm(j, p=p):
                lo = j & (lpw - 1); r = 0
                for i, b in enumerate(p): r |= ((lo >> b) & 1) << i
                return (j & ~(lpw - 1)) | r
            c = gather_cost(n, perm)
            if best is None or c < best[0]: best = (c, p)
        print(n, "identity", gather_cost(n, ident), "best", best)
    print("half-warp model")
    def gather_cost_hw(n, perm):
        T = n // 32; lt = T.bit_length() - 1
        W = max(T, 32); LPR = W >> lt
        def belem(j): return (j >> (0 if lt > 5 else 5 - lt)) * (W * 32) + (j & (LPR - 1)) * n
        tot = 0
        for warp in range(4):
            for m in range(32):
                for hw in range(2):
                    banks = {}
                    for lane in range(16):
                        tid = warp * 32 + hw * 16 + lane
                        j = perm(tid >> lt); tl = tid & (T - 1)
                        e = belem(j) + m * T + (rev(tl, lt) if lt else 0)
                        addr = dsw(e >> 1) * 16 + (e & 1) * 8
                        banks.setdefault((addr // 4) % 32, set()).add(addr // 8)
                    tot += max(len(v) for v in banks.values())
        return tot / (4 * 32)
    for n in (64, 128, 256, 512):
        T = n // 32; lpw = 32 // T; nb = lpw.bit_length() - 1
        res = []
        for p in itertools.permutations(range(nb)):
            def perm(j, p=p):
                lo = j & (lpw - 1); r = 0
                for i, b in enumerate(p): r |= ((lo >> b) & 1) << i
                return (j & ~(lpw - 1)) | r
            res.append((gather_cost_hw(n, perm), p))
        print(n, sorted(res)[:3], "identity", gather_cost_hw(n, lambda j: j))
