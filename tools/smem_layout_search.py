"""Bank-conflict model for the line-per-thread kernels (64-bit smem accesses).

A warp instruction touching double-addresses a_t costs max(2, max_b #distinct{a_t : a_t % 16 == b})
wavefronts (32 banks x 4 B; a double spans a bank pair).  Field layout: addr(i,j,k) = i + j*Pj + k*Pk,
cell c at c*CS.  Thread tid -> cell tid // n^2, line tid % n^2.  Patterns:
  x: line=(j,k), loop i;  y: line=(i,k), loop j;  z: line=(i,j), loop k.
"""
import itertools
import sys


def wavefronts(addrs):
    by = {}
    for a in set(addrs):
        by.setdefault(a % 16, 0)
        by[a % 16] += 1
    return max(2, max(by.values()))


def cost(n, cpb, Pj, Pk, CS, pattern):
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
                    i, j, k = a, s, b
                else:
                    i, j, k = a, b, s
                addrs.append(c * CS + i + j * Pj + k * Pk)
            tot += wavefronts(addrs)
    ideal = sum(2 * n for _ in range(0, threads, 32))
    return tot / ideal


def best(n, cpb, pats):
    res = []
    for Pj in range(n, n + 9):
        for Pk in range(n * Pj, n * Pj + 17):
            base = n * Pk
            for CS in range(base, base + 17):
                c = max(cost(n, cpb, Pj, Pk, CS, p) for p in pats)
                res.append((c, Pj * 0 + Pk * n + CS * 0, Pj, Pk, CS))
    res.sort(key=lambda r: (round(r[0], 3), r[4]))
    return res[0]


if __name__ == "__main__":
    cpbs = {2: 64, 3: 29, 4: 16, 5: 11, 6: 8, 7: 6, 8: 4, 9: 4}
    for n in map(int, sys.argv[1:] or range(2, 10)):
        cpb = cpbs[n]
        cur = {p: round(cost(n, cpb, n | 1, n * (n | 1), n * n * (n | 1), p), 2) for p in "xyz"}
        bx = best(n, cpb, "x")
        bxy = best(n, cpb, "xy")
        byz = best(n, cpb, "yz")
        print(f"n={n} cpb={cpb} current(P=n|1): {cur}  best x: {bx[0]:.2f} (Pj={bx[2]},Pk={bx[3]},CS={bx[4]})"
              f"  best xy: {bxy[0]:.2f} (Pj={bxy[2]},Pk={bxy[3]},CS={bxy[4]})  best yz: {byz[0]:.2f} (Pj={byz[2]},Pk={byz[3]},CS={byz[4]})",
              flush=True)
