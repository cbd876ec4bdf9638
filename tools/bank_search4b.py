"""Bank search for k_sweep4 with two pairs per pair lane (14 lanes x 2-stars sharing the row
node A): K8 decomposition into 2-stars, lane order, plane-row chunk positions, plane and
column offsets mod 8.  Quarter-warp model of the 16-byte block adds.  Offline design tool."""
import random, math, sys

def node_off(a):
    return [(0,0,0),(1,0,0),(1,1,0),(0,1,0),(0,0,1),(1,0,1),(1,1,1),(0,1,1)][a]

EDGES = [(a, b) for a in range(8) for b in range(a + 1, 8)]

def slot(dx, dy):
    return (dy + 1) * 3 + (dx + 1)

def random_decomp():
    while True:
        owner = {}
        cnt = [0] * 8
        for e in random.sample(EDGES, len(EDGES)):
            a, b = e
            # prefer the endpoint with an odd count (to complete a 2-star)
            if cnt[a] % 2 == 1 and cnt[b] % 2 == 0: o = a
            elif cnt[b] % 2 == 1 and cnt[a] % 2 == 0: o = b
            else: o = random.choice(e)
            owner[e] = o
            cnt[o] += 1
        if all(c % 2 == 0 for c in cnt):
            break
    lanes = []
    for n in range(8):
        leaves = [b if a == n else a for (a, b), o in owner.items() if o == n]
        random.shuffle(leaves)
        for k in range(0, len(leaves), 2):
            lanes.append((n, leaves[k], leaves[k + 1]))
    random.shuffle(lanes)
    return lanes

def cost(lanes, cs, poff, pos):
    tot = 0
    for parity in (0, 1):
        for k in (1, 2):
            for kind in ("AB", "BA"):
                for h in (0, 1):
                    for q in (0, 1):
                        grp = {}
                        for (A0, B1, B2) in lanes[8 * q: 8 * q + 8]:
                            B0 = B1 if k == 1 else B2
                            A, B = (A0, B0) if kind == "AB" else (B0, A0)
                            ax, ay, az = node_off(A); bx, by, bz = node_off(B)
                            col = ax + 3 * ay
                            dz = bz - az
                            plane = ("Z%d" % ((parity + az) & 1)) if dz == 0 else ("UP" if dz == 1 else "DN")
                            sl = slot(bx - ax, by - ay)
                            addr = (col, plane, sl, h)
                            res = (cs * col + poff[plane] + pos[sl][h]) % 8
                            grp.setdefault(res, set()).add(addr)
                        if grp:
                            tot += max(len(v) for v in grp.values())
    return tot

if __name__ == "__main__":
    random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    print("ideal", 2 * 2 * 2 * 2 * 2)
    best = None
    for trial in range(int(sys.argv[3]) if len(sys.argv) > 3 else 8):
        lanes = random_decomp()
        cs = random.randrange(8)
        poff = {p: random.randrange(8) for p in ("Z0", "Z1", "UP", "DN")}
        perm = list(range(18)); random.shuffle(perm)
        pos = [[perm[2 * s], perm[2 * s + 1]] for s in range(9)]
        c = cost(lanes, cs, poff, pos)
        for it in range(iters):
            T = 2.0 * (1 - it / iters) + 0.02
            mv = random.randrange(5)
            nl, ncs, npo, npos = lanes, cs, poff, pos
            if mv == 0:
                i, j = random.sample(range(14), 2); nl = lanes[:]; nl[i], nl[j] = nl[j], nl[i]
            elif mv == 1:
                i = random.randrange(14); nl = lanes[:]; a, b1, b2 = nl[i]; nl[i] = (a, b2, b1)
            elif mv == 2:
                ncs = random.randrange(8)
            elif mv == 3:
                npo = dict(poff); npo[random.choice(list(npo))] = random.randrange(8)
            else:
                flat = [p for r in pos for p in r]; i, j = random.sample(range(18), 2); flat[i], flat[j] = flat[j], flat[i]
                npos = [[flat[2 * s], flat[2 * s + 1]] for s in range(9)]
            nc = cost(nl, ncs, npo, npos)
            if nc <= c or random.random() < math.exp((c - nc) / T):
                lanes, cs, poff, pos, c = nl, ncs, npo, npos, nc
            if best is None or c < best[0]:
                best = (c, lanes, cs, dict(poff), [r[:] for r in pos])
        print("trial", trial, "end", c, "best", best[0], flush=True)
    c, lanes, cs, poff, pos = best
    print("best", c, "cs", cs, "poff", poff)
    print("lanes", lanes)
    print("pos", pos)
