"""YX field with a per-k offset table: addr = cell*CS + i + j*Pj + KT[k] (k is per-thread in
every YX access: y-write of line (i, k), x-read of line (j, k)), half-warp cost model of
smem_layout_search6.py, current k_kron4 thread mapping.  Random restarts + coordinate descent
over Pj, the residues of KT[k] mod 16 and of CS mod 16; offsets are then the smallest values
with those residues that keep the k-slabs and cells disjoint.
Usage: smem_ktable_search.py n R cpb [seed [threads per cell, padded]]"""
import random
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
from smem_layout_search6 import hw_cost  # noqa: E402


def layout(n, Pj, res, csr):
    span = (n - 1) * Pj + n
    kt, cur = [], 0
    for k in range(n):
        v = cur
        while v % 16 != res[k]:
            v += 1
        kt.append(v)
        cur = v + span
    cs = cur
    while cs % 16 != csr:
        cs += 1
    return kt, cs


TPCP = None   # padded threads per cell (None: n * NB, the current mapping)
XSW = 0       # 1: the x stage handles line (j, k) = (b + r NB, a)
PJR = 4       # Pj range searched: n .. n + PJR - 1


def cost(n, R, cpb, Pj, kt, CS, stage):
    NB = -(-n // R)
    tpc = n * NB
    tpcp = TPCP or tpc
    threads = cpb * tpcp
    tot = ideal = 0
    for w0 in range(0, threads, 32):
        for r in range(R):
            for s in range(n):
                addrs = []
                for t in range(w0, w0 + 32):
                    if t >= threads:
                        addrs.append(None)
                        continue
                    c, rem = divmod(t, tpcp)
                    if rem >= tpc:
                        addrs.append(None)
                        continue
                    a, bp = rem % n, rem // n
                    b = bp + r * NB
                    if b >= n:
                        addrs.append(None)
                        continue
                    if stage == "y":
                        i, j, k = a, s, b
                    else:
                        i, j, k = (s, b, a) if XSW else (s, a, b)
                    if k >= n or j >= n:
                        addrs.append(None)
                        continue
                    addrs.append(c * CS + i + j * Pj + kt[k])
                if any(x is not None for x in addrs):
                    tot += hw_cost(addrs)
                    ideal += sum(1 for h in (addrs[:16], addrs[16:]) if any(x is not None for x in h))
    return tot / ideal


def total(n, R, cpb, Pj, res, csr):
    kt, cs = layout(n, Pj, res, csr)
    c = max(cost(n, R, cpb, Pj, kt, cs, "y"), cost(n, R, cpb, Pj, kt, cs, "x"))
    return (round(c, 4), cs), kt, cs


def run(n, R, cpb, seed=0, restarts=30):
    rnd = random.Random(seed)
    best = None
    for _ in range(restarts):
        Pj = rnd.randrange(n, n + PJR)
        res = [rnd.randrange(16) for _ in range(n)]
        csr = rnd.randrange(16)
        cur = total(n, R, cpb, Pj, res, csr)
        improved = True
        while improved:
            improved = False
            for var in range(n + 2):
                for v in (range(n, n + PJR) if var == n else range(16)):
                    P2, r2, c2 = Pj, list(res), csr
                    if var < n:
                        r2[var] = v
                    elif var == n:
                        P2 = v
                    else:
                        c2 = v
                    t = total(n, R, cpb, P2, r2, c2)
                    if t[0] < cur[0]:
                        cur, Pj, res, csr, improved = t, P2, r2, c2, True
        if best is None or cur[0] < best[0][0]:
            best = (cur, Pj)
        if best[0][0][0] <= 1.0:
            break
    (key, kt, cs), Pj = best
    return key[0], Pj, kt, cs


if __name__ == "__main__":
    n, R, cpb = map(int, sys.argv[1:4])
    seed = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    TPCP = int(sys.argv[5]) if len(sys.argv) > 5 else None
    XSW = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    PJR = int(sys.argv[7]) if len(sys.argv) > 7 else 4
    print(n, R, cpb, run(n, R, cpb, seed), flush=True)
