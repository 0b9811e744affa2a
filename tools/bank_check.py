"""Exhaustive shared-memory bank check of the fused7 layouts (tools only; mirrors fused7.cuh).

8-byte elements, 16 bank pairs per 128-byte wavefront; each half-warp access must hit
distinct bank pairs (identical addresses broadcast).  Thread-role maps (128 threads):
  S1 / M1 : slot s8 = tid & 7, t (or i) = tid >> 3
  M3      : warp w, lane L: slot 4 (w >> 1) + (L >> 3), i = (L & 7) + 8 (w & 1)
Exchange: slot(s, m1, t) = P(s) XS + 17 m1 + t, P(s) = 4 (s & 1) + (s >> 1), XS = 17*16 + 2
(one round of 16 m1 values).  Writers (S1) write every m1 < 16 at their t; readers (M1, M3)
read their sequence m1 = i at every t.  F buffer: column stride D + 2; the Zak tile writes
F[s8][16 r + i + R1 m2] (M1), product tile h gathers F[2h + (s8 >> 2)][(sigma - t - 16 k) mod D]
(S1) for sigma = 0.
"""


def wavefronts(addrs):
    banks = {}
    for a in set(addrs):
        banks.setdefault(a % 16, set()).add(a)
    return max(len(v) for v in banks.values())


S1 = lambda tid: (tid & 7, tid >> 3)
M1 = S1
M3 = lambda tid: (4 * ((tid >> 5) >> 1) + ((tid & 31) >> 3), ((tid & 31) & 7) + 8 * ((tid >> 5) & 1))
XS = 17 * 16 + 2
P = lambda s: 4 * (s & 1) + (s >> 1)
xslot = lambda s, m, t: P(s) * XS + 17 * m + t


def check(D):
    R1 = D // 16
    worst = {}
    hws = [list(range(hw * 16, hw * 16 + 16)) for hw in range(8)]
    w = 0
    for m in range(16):
        for hw in hws:
            w = max(w, wavefronts([xslot(S1(t)[0], m, S1(t)[1]) for t in hw]))
    worst["exchange write (S1)"] = w
    for name, role in (("exchange read (M1)", M1), ("exchange read (M3)", M3)):
        w = 0
        for tt in range(16):
            for hw in hws:
                w = max(w, wavefronts([xslot(role(t)[0], role(t)[1], tt) for t in hw]))
        worst[name] = w
    FS = D + 2
    w = 0
    for r in range(R1 // 16):
        for m2 in range(16):
            for hw in hws:
                w = max(w, wavefronts([(t & 7) * FS + 16 * r + (t >> 3) + R1 * m2 for t in hw]))
    worst["F write (M1)"] = w
    w = 0
    for h in range(4):
        for k in range(R1):
            for hw in hws:
                w = max(w, wavefronts([(2 * h + ((t & 7) >> 2)) * FS + ((-(t >> 3) - 16 * k) % D) for t in hw]))
    worst["F gather (S1)"] = w
    return worst


if __name__ == "__main__":
    for D in (256, 512):
        res = check(D)
        print(f"D={D}:", res)
        assert max(res.values()) == 1, "bank conflict"
    print("all half-warp accesses conflict-free")
