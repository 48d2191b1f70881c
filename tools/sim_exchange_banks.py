# bank-conflict simulation of the shared-memory exchange patterns (16-byte chunks,
# 8 bank groups of 16 B; a warp's 128-bit access = 4 phases of 8 consecutive lanes)
def dsw(C):
    x = C >> 3
    f = (x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7
    f ^= ((C >> 6) & 1) * 6
    return C ^ f

def geometry(n):
    T = n // 32; lt = T.bit_length() - 1
    W = max(T, 32); LPR = W >> lt
    def belem(j, q):
        return (j >> (0 if lt > 5 else 5 - lt)) * (W * 32) + (j & (LPR - 1)) * n + q
    return T, lt, belem

def check(n, pattern, name):
    """pattern(tl) -> list of element offsets (run starts, multiples of 8/16) within the line,
    one per access instruction index; each access covers 1 chunk (c added by caller)"""
    T, lt, belem = geometry(n)
    worst = 1
    nacc = len(pattern(0))
    for warp in range(128 // 32):
        for a in range(nacc):
            for c in range(pattern.chunks):
                for ph in range(4):
                    banks = []
                    for lane in range(8):
                        tid = warp * 32 + ph * 8 + lane
                        tl = tid & (T - 1)
                        e = belem(tid >> lt, 0) + pattern(tl)[a]
                        C = e // 2 + c
                        banks.append(dsw(C) & 7)
                    m = max(banks.count(b) for b in set(banks))
                    worst = max(worst, m)
    return worst

def single_read(s):
    def p(tl):
        b0 = 16 * tl; h = 1 << s; j0 = b0 & (h - 1)
        U = ((b0 >> s) << (s + 1)) + j0
        return [U, U + h]
    p.chunks = 8
    return p

def pair_read(s):
    def p(tl):
        h = 1 << s; u = 8 * tl; g = u // h; j0 = u % h
        base = g * 4 * h
        return [base + k * h + j0 for k in range(4)]
    p.chunks = 4
    return p

for n in (64, 128, 256, 512, 1024, 2048, 4096):
    L = n.bit_length() - 1
    res = []
    for s in range(5, L):
        res.append(f"s{s}:single {check(n, single_read(s), 'single')}")
        if s + 1 < L:
            res.append(f"s{s}:pair {check(n, pair_read(s), 'pair')}")
    print(n, " ".join(res))
