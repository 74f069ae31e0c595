"""Shared-memory layout search for k_kron6 (in-place fields, one layout per field).

k_kron6 keeps every cell field in ONE layout addr = i + j*Pj + k*Pk + cell*CS for all three
line directions (z-lines written in stage Z, y-lines read and rewritten in place in stage Y,
x-lines read in stage X), so that stage Y needs no barrier between its reads and writes.
Thread t of a block = ta + n*(tb + NB*cell); thread (ta, tb) owns lines (ta, tb + r*NB).
Cost model (tools/smem_layout_search6.py): 64-bit accesses are served per half-warp; the
cost of a warp instruction is the sum over both half-warps of the largest number of
distinct doubles mapping to one bank pair (addr % 16).  Prints the cheapest (max over the
three patterns, then smem size) layout per n.
"""
import sys


def hw_cost(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        half = [a for a in half if a is not None]
        if not half:
            continue
        by = {}
        for a in set(half):
            by[a % 16] = by.get(a % 16, 0) + 1
        tot += max(by.values())
    return tot


def cost(n, R, cpb, Pj, Pk, CS, pat):
    NB = -(-n // R)
    tpc = n * NB
    threads = cpb * tpc
    tot = ideal = 0
    for w0 in range(0, threads, 32):
        for r in range(R):
            for s in range(n):
                addrs = []
                for t in range(w0, w0 + 32):
                    if t >= threads:
                        addrs.append(None)
                        continue
                    c, rem = divmod(t, tpc)
                    a, bp = rem % n, rem // n
                    b = bp + r * NB
                    if b >= n:
                        addrs.append(None)
                        continue
                    if pat == "x":
                        i, j, k = s, a, b
                    elif pat == "y":
                        i, j, k = a, s, b
                    else:
                        i, j, k = a, b, s
                    addrs.append(c * CS + i + j * Pj + k * Pk)
                if any(x is not None for x in addrs):
                    tot += hw_cost(addrs)
                    ideal += sum(1 for h in (addrs[:16], addrs[16:]) if any(x is not None for x in h))
    return tot / ideal


def search(n, R, cpb, span=10):
    best = None
    for Pj in range(n, n + span + 1):
        for Pk in range(n * Pj, n * Pj + 2 * span):
            for CS in range(n * Pk, n * Pk + 17):
                c = max(cost(n, R, cpb, Pj, Pk, CS, p) for p in "xyz")
                key = (round(c, 3), CS)
                if best is None or key < best[0]:
                    best = (key, Pj, Pk, CS)
    return best


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        n, R, cpb = map(int, arg.split(","))
        b = search(n, R, cpb)
        print(f"n={n} R={R} CPB={cpb}: cost {b[0][0]} layout Pj={b[1]} Pk={b[2]} CS={b[3]} "
              f"({b[3] / n ** 3:.2f}x n^3)", flush=True)
