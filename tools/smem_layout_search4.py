"""Bank-conflict search for the z-first Kronecker kernel (k_kron4.cu).

Same cost model as smem_layout_search.py (64-bit accesses, a double spans a bank
pair, cost = max(2, max bank-pair multiplicity) wavefronts per warp instruction).
Layouts addr(i,j,k) = i + j*Pj + k*Pk + cell*CS, searched per field:
  ZY: written by z-lines (thread (i,j), loop k), read by y-lines (thread (i,k), loop j)
  YX: written by y-lines, read by x-lines (thread (j,k), loop i)
  XZ: written by x-lines, read by z-lines
"""
import sys
from smem_layout_search import cost

CPB = {3: 32, 4: 16, 5: 12, 6: 8, 7: 5, 8: 4, 9: 3}


def search(n, cpb, pats, span=12):
    best = None
    for Pj in range(n, n + span):
        for Pk in range(n * Pj, n * Pj + span):
            for CS in range(n * Pk, n * Pk + 17):
                c = max(cost(n, cpb, Pj, Pk, CS, p) for p in pats)
                key = (round(c, 3), CS)
                if best is None or key < best[0]:
                    best = (key, Pj, Pk, CS)
                if c <= 1.0:
                    return best
    return best


if __name__ == "__main__":
    for n in map(int, sys.argv[1:] or CPB):
        out = {f: search(n, CPB[n], f.lower()) for f in ("ZY", "YX", "XZ")}
        print(n, CPB[n], {f: (v[0][0], v[1], v[2], v[3]) for f, v in out.items()}, flush=True)
