"""Exhaustive shared-memory bank check of the fused7 exchange-buffer swizzle (tools only).

Slot(col, m1, t) = col*D + m1*16 + (t ^ f(col, m1)), 8-byte slots, 16 bank pairs per
128-byte wavefront.  Writers: stage-1 roles (col, t) write m1 = 0..R1-1.  Readers: stage-2
roles (col, i) read sequences m1 = 16 r + i (r = 0, 1), every t.  Each half-warp access
must hit 16 distinct bank pairs (identical addresses broadcast)."""
import itertools

D, R1 = 512, 32
roles_w = {
    'S1_16': lambda tid: (tid & 15, tid >> 4),
    'S1_8': lambda tid: ((tid & 7, tid >> 3) if tid < 128 else None),
}
roles_r = {
    'M1_16': lambda tid: (tid & 15, tid >> 4),
    'M1_8': lambda tid: ((tid & 7, tid >> 3) if tid < 128 else None),
    # u-tile stage 2: warp w -> column w >> 1; lane L -> u = L >> 3, i = (L & 7) + 8 (w & 1)
    'M3': lambda tid: (4 * ((tid >> 5) >> 1) + ((tid & 31) >> 3), ((tid & 31) & 7) + 8 * ((tid >> 5) & 1)),
}


def wavefronts(addrs):
    banks = {}
    for a in set(addrs):
        banks.setdefault(a % 16, set()).add(a)
    return max(len(v) for v in banks.values())


def cost(f):
    slot = lambda col, m, t: col * D + m * 16 + (t ^ f(col, m))
    tot = worst = 0
    for rn, role in roles_w.items():
        for m in range(R1):
            for hw in range(16):
                a = [slot(*((role(hw * 16 + L)[0], m, role(hw * 16 + L)[1]))) for L in range(16) if role(hw * 16 + L)]
                if a:
                    w = wavefronts(a); tot += w; worst = max(worst, w)
    for rn, role in roles_r.items():
        for r in range(R1 // 16):
            for tt in range(16):
                for hw in range(16):
                    a = []
                    for L in range(16):
                        x = role(hw * 16 + L)
                        if x:
                            a.append(slot(x[0], 16 * r + x[1], tt))
                    if a:
                        w = wavefronts(a); tot += w; worst = max(worst, w)
    return tot, worst


if __name__ == '__main__':
    cur = lambda c, m: (2 * c + (c >> 3) + m) & 15
    print('current f = (2c + (c>>3) + m) & 15:', cost(cur))
    best = None
    for a, b, e, g in itertools.product(range(16), (1, 3, 5, 7), range(16), range(4)):
        f = lambda c, m, a=a, b=b, e=e, g=g: (a * c + b * m + e * (c >> 3) + g * (c >> 2)) & 15
        r = cost(f)
        if best is None or r < best[0]:
            best = (r, a, b, e, g)
            if r[1] == 1:
                break
    print('best (total, worst), f = (a c + b m + e (c>>3) + g (c>>2)) & 15:', best)
