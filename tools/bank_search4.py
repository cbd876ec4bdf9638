"""Quarter-warp bank model of the k_sweep4 block adds (16-byte RMW of pair blocks into the
shared-memory planes) and a local search over layout parameters.  Offline design tool."""
import itertools, random
random.seed(1)

def node_off(a):   # Hex8 node order (x, y, z) bits as node_off<3>
    tab = [(0,0,0),(1,0,0),(1,1,0),(0,1,0),(0,0,1),(1,0,1),(1,1,1),(0,1,1)]
    return tab[a]

PAIRS = [(a, b) for a in range(8) for b in range(a + 1, 8)]

def slot(dx, dy):
    return (dy + 1) * 3 + (dx + 1)

def accesses(pairs, parity):
    """per instruction group: list over lanes of (col, plane, slot)"""
    out = {}
    for kind in ("AB", "BA"):
        lst = []
        for (a, b) in pairs:
            A, B = (a, b) if kind == "AB" else (b, a)
            ax, ay, az = node_off(A); bx, by, bz = node_off(B)
            col = ax + 3 * ay
            dz = bz - az
            if dz == 0:
                plane = "Z%d" % ((parity + az) & 1)
            elif dz == 1:
                plane = "UP"
            else:
                plane = "DN"
            lst.append((col, plane, slot(bx - ax, by - ay)))
        out[kind] = lst
    return out

def cost(pairs, cs, poff, pos):
    tot = 0
    for parity in (0, 1):
        acc = accesses(pairs, parity)
        for kind, lst in acc.items():
            for h in (0, 1):
                for q in range(4):
                    lanes = lst[8 * q: 8 * q + 8]
                    groups = {}
                    for (col, plane, sl) in lanes:
                        addr = col * 1000 + {"Z0": 0, "Z1": 1, "UP": 2, "DN": 3}[plane] * 100 + sl * 2 + h
                        res = (cs * col + poff[plane] + pos[sl][h]) % 8
                        groups.setdefault(res, set()).add(addr)
                    if lanes:
                        tot += max(len(v) for v in groups.values())
    return tot

def ideal(pairs):
    n = 0
    for parity in (0, 1):
        for kind in ("AB", "BA"):
            for h in (0, 1):
                n += (len(pairs) + 7) // 8
    return n

cur_pos = [[(2 * sl + (h ^ ((sl >> 2) & 1))) for h in (0, 1)] for sl in range(9)]
cur_poff = {"Z0": 0, "Z1": 73, "UP": 146, "DN": 219}
print("ideal", ideal(PAIRS))
print("current", cost(PAIRS, 301, cur_poff, cur_pos))
ident_pos = [[2 * sl + h for h in (0, 1)] for sl in range(9)]
print("current, identity swz", cost(PAIRS, 301, cur_poff, ident_pos))

best = None
for trial in range(60):
    pairs = PAIRS[:]
    random.shuffle(pairs)
    cs = random.randrange(8)
    poff = {k: random.randrange(8) for k in ("Z0", "Z1", "UP", "DN")}
    perm = list(range(18)); random.shuffle(perm)
    pos = [[perm[2 * sl + h] for h in (0, 1)] for sl in range(9)]
    c = cost(pairs, cs, poff, pos)
    for it in range(4000):
        mv = random.randrange(4)
        np_, ncs, npo, npos = pairs, cs, poff, pos
        if mv == 0:
            i, j = random.sample(range(28), 2); np_ = pairs[:]; np_[i], np_[j] = np_[j], np_[i]
        elif mv == 1:
            ncs = random.randrange(8)
        elif mv == 2:
            npo = dict(poff); npo[random.choice(list(npo))] = random.randrange(8)
        else:
            flat = [p for r in pos for p in r]; i, j = random.sample(range(18), 2); flat[i], flat[j] = flat[j], flat[i]
            npos = [[flat[2 * sl + h] for h in (0, 1)] for sl in range(9)]
        nc = cost(np_, ncs, npo, npos)
        if nc <= c:
            pairs, cs, poff, pos, c = np_, ncs, npo, npos, nc
    if best is None or c < best[0]:
        best = (c, pairs, cs, poff, pos)
        print("trial", trial, "cost", c)
c, pairs, cs, poff, pos = best
print("best", c, "cs", cs, "poff", poff)
print("pairs", pairs)
print("pos", pos)
