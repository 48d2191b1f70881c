"""Bank-conflict simulation of the paired strided copy-out (LDS.64 of two
adjacent lines per thread, mxfft_lines.cuh) for n <= 256, with an optional
XOR remap of the pair index pa by the position index (half-warp model)."""
import itertools
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sim_gather_banks import dsw  # noqa: E402


def cost(n, remap):
    T = n // 32
    lt = T.bit_length() - 1
    W = max(T, 32)
    LPR = W >> lt
    LPC = 128 >> lt
    LLPC = 7 - lt

    def belem(j, q):
        return (j >> (0 if lt > 5 else 5 - lt)) * (W * 32) + (j & (LPR - 1)) * n + q

    tot = 0
    for warp in range(4):
        for k in range(16):
            for which in (0, 1):
                for hw in range(2):
                    banks = {}
                    for lane in range(16):
                        tid = warp * 32 + hw * 16 + lane
                        pa = tid & ((LPC >> 1) - 1)
                        pq0 = tid >> (LLPC - 1 if LLPC > 0 else 0)
                        pa = remap(pa, pq0)
                        e = belem(2 * pa + which, pq0) + 2 * T * k
                        addr = dsw(e >> 1) * 16 + (e & 1) * 8
                        banks.setdefault((addr // 4) % 32, set()).add(addr // 8)
                    tot += max(len(v) for v in banks.values())
    return tot / (4 * 16 * 2)


if __name__ == "__main__":
    for n in (32, 64, 128, 256):
        T = n // 32
        lt = T.bit_length() - 1
        LPC = 128 >> lt
        npa = LPC >> 1
        base = cost(n, lambda pa, q: pa)
        best = (base, "identity")
        for c in range(1, npa):
            for sh in range(0, 4):
                f = lambda pa, q, c=c, sh=sh: pa ^ ((c * ((q >> sh) & 1)) & (npa - 1))
                v = cost(n, f)
                if v < best[0]:
                    best = (v, f"pa ^ ({c} if bit {sh} of pq0)")
        print(n, "identity", base, "best", best)


def cost_map(n, mapping):
    """mapping(tid) -> (pa, pq0)"""
    T = n // 32
    lt = T.bit_length() - 1
    W = max(T, 32)
    LPR = W >> lt

    def belem(j, q):
        return (j >> (0 if lt > 5 else 5 - lt)) * (W * 32) + (j & (LPR - 1)) * n + q

    tot = 0
    for warp in range(4):
        for k in range(16):
            for which in (0, 1):
                for hw in range(2):
                    banks = {}
                    for lane in range(16):
                        pa, pq0 = mapping(warp * 32 + hw * 16 + lane)
                        e = belem(2 * pa + which, pq0) + 2 * T * k
                        addr = dsw(e >> 1) * 16 + (e & 1) * 8
                        banks.setdefault((addr // 4) % 32, set()).add(addr // 8)
                    tot += max(len(v) for v in banks.values())
    return tot / (4 * 16 * 2)


def split_map(n):
    """pa bits 0-2 from tid bits 0-2, pq0 bit 0 from tid bit 3, the rest of pa next, then pq0"""
    T = n // 32
    lt = T.bit_length() - 1
    npa = (128 >> lt) >> 1
    hb = max(npa.bit_length() - 1 - 3, 0)  # pa bits above bit 2

    def m(tid):
        if npa <= 8:
            return tid & (npa - 1), tid >> (npa.bit_length() - 1)
        pa = (tid & 7) | (((tid >> 4) & ((1 << hb) - 1)) << 3)
        pq0 = ((tid >> 3) & 1) | ((tid >> (4 + hb)) << 1)
        return pa, pq0
    return m


if __name__ == "__main__":
    for n in (32, 64, 128, 256):
        print(n, "split map", cost_map(n, split_map(n)))
