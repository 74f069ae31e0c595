"""Bank-conflict search for k_kron4 with R lines per thread (thread (a, b') of a cell
handles lines (a, b' + r*NB), NB = ceil(n/R)).  Cost model as smem_layout_search.py.
Fields addr = i + j*Pj + k*Pk + cell*CS:
  ZY: written by z-lines (line (i,j)), read by y-lines (line (i,k))
  YX: written by y-lines, read by x-lines (line (j,k))
  XZ: written by x-lines, read by z-lines
"""
import sys
from smem_layout_search import wavefronts


def cost(n, R, cpb, Pj, Pk, CS, pat):
    NB = -(-n // R)
    tpc = n * NB
    threads = cpb * tpc
    tot = ideal = 0
    for w0 in range(0, threads, 32):
        tids = range(w0, min(w0 + 32, threads))
        for r in range(R):
            for s in range(n):
                addrs = []
                for t in tids:
                    c, rem = divmod(t, tpc)
                    a, bp = rem % n, rem // n
                    b = bp + r * NB
                    if b >= n:
                        continue
                    if pat == "x":
                        i, j, k = s, a, b
                    elif pat == "y":
                        i, j, k = a, s, b
                    else:
                        i, j, k = a, b, s
                    addrs.append(c * CS + i + j * Pj + k * Pk)
                if addrs:
                    tot += wavefronts(addrs)
                    ideal += 2
    return tot / ideal


def search(n, R, cpb, pats, span=12):
    best = None
    for Pj in range(n, n + span):
        for Pk in range(n * Pj, n * Pj + span):
            for CS in range(n * Pk, n * Pk + 17):
                c = max(cost(n, R, cpb, Pj, Pk, CS, p) for p in pats)
                key = (round(c, 3), CS)
                if best is None or key < best[0]:
                    best = (key, Pj, Pk, CS)
                if c <= 1.0:
                    return best
    return best


if __name__ == "__main__":
    n, R, cpb = map(int, sys.argv[1:4])
    out = {f: search(n, R, cpb, f.lower()) for f in ("ZY", "YX", "XZ")}
    print(n, R, cpb, {f: (v[0][0], v[1], v[2], v[3]) for f, v in out.items()}, flush=True)
