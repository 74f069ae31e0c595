"""Extended bank-conflict search (see smem_layout_search.py) including the y-phase
thread ordering (i fastest vs k fastest) and wider pitch ranges."""
import sys
from smem_layout_search import wavefronts


def cost(n, cpb, Pj, Pk, CS, pattern, yorder):
    nn = n * n
    threads = cpb * nn
    tot = 0
    for w0 in range(0, threads, 32):
        tids = range(w0, min(w0 + 32, threads))
        for s in range(n):
            addrs = []
            for t in tids:
                c, l = divmod(t, nn)
                a, b = l % n, l // n
                if pattern == "x":
                    i, j, k = s, a, b
                elif pattern == "y":
                    i, j, k = (a, s, b) if yorder == 0 else (b, s, a)
                else:
                    i, j, k = a, b, s
                addrs.append(c * CS + i + j * Pj + k * Pk)
            tot += wavefronts(addrs)
    return tot / (2 * n * ((threads + 31) // 32))


def search(n, cpb, pats, yorder, span=20):
    best = None
    for Pj in range(n, n + span):
        for Pk in range(n * Pj, n * Pj + span):
            for CS in range(n * Pk, n * Pk + 17, 1):
                c = max(cost(n, cpb, Pj, Pk, CS, p, yorder) for p in pats)
                key = (round(c, 3), CS)
                if best is None or key < best[0]:
                    best = (key, Pj, Pk, CS)
                if c <= 1.0:
                    break
    return best


if __name__ == "__main__":
    cpbs = {2: 64, 3: 29, 4: 16, 5: 11, 6: 8, 7: 6, 8: 4, 9: 4}
    for n in map(int, sys.argv[1:]):
        for yo in (0, 1):
            xy = search(n, cpbs[n], "xy", yo)
            yz = search(n, cpbs[n], "yz", yo)
            print(f"n={n} yorder={yo} xy={xy} yz={yz}", flush=True)
