"""Shared-memory layout search for the warp-private basis-change kernel k_bchgw:
addr(cell, k, j, i) = i + j*Pj + k*Pk + cell*CS; lane l of round r owns line l + 32 r of a sweep
(x-lines: (cell, k, j), j fastest; y-lines: (cell, k, i); z-lines: (cell, j, i), i fastest).
Cost = shared wavefronts of the 64-bit line accesses in the half-warp model (16 lanes, 16 banks
of 8 B), summed over the three sweeps, per tile of C cells.  Usage: bchgw_layout_search.py n C"""
import sys


def cost(n, C, Pj, Pk, CS):
    tot = 0
    for d in range(3):
        L = C * n * n
        for r0 in range(0, L, 32):
            for h in range(0, 32, 16):
                lanes = [q for q in range(r0 + h, min(r0 + h + 16, L))]
                if not lanes:
                    continue
                for s in range(n):
                    banks = {}
                    for q in lanes:
                        c, rem = divmod(q, n * n)
                        a, b = rem % n, rem // n
                        if d == 0:
                            i, j, k = s, a, b
                        elif d == 1:
                            i, j, k = a, s, b
                        else:
                            i, j, k = a, b, s
                        ad = i + j * Pj + k * Pk + c * CS
                        banks.setdefault(ad % 16, set()).add(ad)
                    tot += max(len(v) for v in banks.values())
    return tot


def main():
    n, C = int(sys.argv[1]), int(sys.argv[2])
    best = []
    for Pj in range(n, n + 3):
        for Pk in range(n * Pj, n * Pj + 10):
            for CS in range((n - 1) * Pk + (n - 1) * Pj + n, n * Pk + 18):
                best.append((cost(n, C, Pj, Pk, CS), C * CS, Pj, Pk, CS))
    best.sort()
    ideal = 3 * n * 2 * ((C * n * n + 31) // 32)
    print("n", n, "C", C, "ideal", ideal, "natural", cost(n, C, n, n * n, n ** 3))
    for b in best[:4]:
        print(b)


main()
