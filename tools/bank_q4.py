"""Bank model of the k_sweepq shared-memory traffic per batch (16 Q4 elements of one colour)
and a local search over the layout knobs.  Offline design tool.

Model: 16-byte accesses are served per quarter-warp (8 lanes, 8 bank groups of 16 B): a
quarter costs max over groups of the distinct 16-B addresses in that group.  8-byte accesses
per half-warp (16 lanes, 16 bank pairs).  Idle lanes cost nothing."""
import random, sys

NODE = [(0, 0), (1, 0), (1, 1), (0, 1)]     # Q4 node -> (x, y) offset
B1 = [1, 2, 0]
NROW, TX, NSS = 81, 31, 7


def wf(addrs, width):
    """addrs: per-lane address (None = idle) in units of `width` bytes; returns wavefronts"""
    per = 8 if width == 16 else 16
    mod = 8 if width == 16 else 16
    tot = 0
    for q in range(0, len(addrs), per):
        grp = {}
        for a in addrs[q:q + per]:
            if a is not None:
                grp.setdefault(a % mod, set()).add(a)
        if grp:
            tot += max(len(v) for v in grp.values())
    return tot


def cost(L, detail=False):
    lanes, swp, EL2, GS2, RS2, bo = L['lanes'], L['swp'], L['EL2'], L['GS2'], L['RS2'], L['bo']
    NSUM2 = 2 * GS2
    HDR2 = NSUM2 + 12
    parts = {}
    # C record loads (16 B): A chunks 0..4, B chunks {0,2,3,4,5,6} of first / second pair
    c = 0
    for g in range(4):
        for ch in range(5):
            c += wf([None if t is None else t[0] * EL2 + g * GS2 + t[1] * RS2 + ch for t in lanes], 16)
        for first in (0, 1):
            for ch in (0, 2, 3, 4, 5, 6):
                ad = []
                for t, s in zip(lanes, swp):
                    if t is None:
                        ad.append(None); continue
                    second = first ^ s[0]
                    node = B1[t[1]] if second == 0 else 3
                    ad.append(t[0] * EL2 + g * GS2 + node * RS2 + ch)
                c += wf(ad, 16)
        c += wf([None if t is None else t[0] * EL2 + HDR2 + g for t in lanes], 16)
    parts['C loads'] = c
    # C node-sum reads (8 B)
    c = 0
    for q in range(6):
        c += wf([None if t is None else 2 * (t[0] * EL2 + NSUM2) + t[1] * 6 + q for t in lanes], 8)
        c += wf([None if t is None else 2 * (t[0] * EL2 + NSUM2) + 18 + q for t in lanes], 8)
    parts['C ns reads'] = c
    # PC record / node-sum / hdr stores (16 B): lane = (el, g)
    c = 0
    pcl = [(lid >> 2, lid & 3) for lid in range(64)]
    for a in range(4):
        for ch in range(7):
            c += wf([el * EL2 + g * GS2 + a * RS2 + ch for el, g in pcl], 16)
    for q in range(3):
        c += wf([el * EL2 + NSUM2 + g * 3 + q for el, g in pcl], 16)
    c += wf([el * EL2 + HDR2 + g for el, g in pcl], 16)
    parts['PC stores'] = c
    # adds (8 B RMW: count load + store): blocks in the row buffers, 3 parities of the row
    c = 0
    for sp in range(3):
        for step in range(4):
            for r in range(3):
                for j in range(3):
                    ad = []
                    for t, s in zip(lanes, swp):
                        if t is None:
                            ad.append(None); continue
                        cel, ck = t
                        pairsel = (step >> 1) ^ s[1]
                        blk = (step & 1) ^ s[2]
                        A, B = ck, (B1[ck] if pairsel == 0 else 3)
                        (ax, az), (bx, bz) = NODE[A], NODE[B]
                        X, Z, dx, dz = (ax, az, bx - ax, bz - az) if blk == 0 else (bx, bz, ax - bx, az - bz)
                        x = 2 * cel + X
                        zb = (sp + Z) % 3
                        ad.append(bo[zb] + zb * TX * NROW + x * NROW + r * 27 + (dz + 1) * 9 + (dx + 1) * 3 + j)
                    c += 2 * wf(ad, 8)
    parts['adds'] = c / 3
    tot = sum(parts.values())
    return (tot, parts) if detail else tot


def current():
    return dict(lanes=[(gt // 3, gt % 3) if gt < 48 else None for gt in range(64)],
                swp=[(0, 0, 0)] * 64, EL2=141, GS2=30, RS2=7, bo=[0, 0, 0])


if __name__ == '__main__':
    cur = current()
    print('current', cost(cur, True))
    random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
    import math
    best = None
    for trial in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
        L = current()
        c = cost(L)
        T0 = 8.0
        iters = int(sys.argv[3]) if len(sys.argv) > 3 else 6000
        for it in range(iters):
            T = T0 * (1 - it / iters) + 0.05
            N = dict(L)
            mv = random.randrange(7)
            if mv <= 2:
                i, j = random.sample(range(48), 2); N['lanes'] = L['lanes'][:]; N['lanes'][i], N['lanes'][j] = N['lanes'][j], N['lanes'][i]
            elif mv <= 4:
                i = random.randrange(48); N['swp'] = L['swp'][:]; f = list(N['swp'][i]); k = random.randrange(3); f[k] ^= 1; N['swp'][i] = tuple(f)
            elif mv == 5:
                N['GS2'] = random.randrange(28, 35); N['EL2'] = min(152, max(N['EL2'], 2 * N['GS2'] + 16))
                if rand_el := random.random() < 0.5: N['EL2'] = random.randrange(2 * N['GS2'] + 16, 153)
            else:
                N['bo'] = L['bo'][:]; N['bo'][random.randrange(1, 3)] = random.randrange(16)
            nc = cost(N)
            if nc <= c or random.random() < math.exp((c - nc) / T):
                L, c = N, nc
            if best is None or c < best[0]:
                best = (c, dict(L))
        print('trial', trial, 'end', c, 'best so far', best[0], cost(best[1], True)[1], flush=True)
    c, L = best
    print('best', cost(L, True))
    print('L =', L)
