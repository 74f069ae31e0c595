"""Bank-conflict search for k_kron4 (R lines per thread), half-warp cost model.

64-bit shared accesses are served per half-warp (16 lanes x 8 B = one 128 B wavefront when
conflict-free): cost of one warp instruction = sum over the two half-warps of the largest
number of distinct double addresses mapping to the same bank pair (addr % 16).  This model
reproduces the measured excess wavefronts of the n=7 layouts in profiles (the whole-warp
model of smem_layout_search5.py under-counts).  Fields addr = i + j*Pj + k*Pk + cell*CS:
  ZY: z-write (line (i,j)) / y-read (line (i,k));  YX: y-write / x-read (line (j,k));
  XZ: x-write / z-read.
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


def search(n, R, cpb, pats, pjmax=None, csmax=None, span=12):
    best = None
    for Pj in range(n, (pjmax or n + span) + 1):
        for Pk in range(n * Pj, n * Pj + span):
            for CS in range(n * Pk, n * Pk + 17):
                if csmax and CS > csmax:
                    break
                c = max(cost(n, R, cpb, Pj, Pk, CS, p) for p in pats)
                key = (round(c, 3), CS)
                if best is None or key < best[0]:
                    best = (key, Pj, Pk, CS)
                if c <= 1.0:
                    return best
    return best


if __name__ == "__main__":
    n, R, cpb = map(int, sys.argv[1:4])
    csmax = int(sys.argv[4]) if len(sys.argv) > 4 else None
    cur = {"6": {"ZY": (6, 38, 228), "YX": (9, 54, 324)}, "7": {"ZY": (7, 55, 396), "YX": (7, 52, 364)}}
    for f, L in cur.get(str(n), {}).items():
        print("current", f, L, round(max(cost(n, R, cpb, *L, p) for p in f.lower()), 3))
    out = {f: search(n, R, cpb, f.lower(), csmax=csmax) for f in ("ZY", "YX", "XZ")}
    print(n, R, cpb, {f: (v[0][0], v[1], v[2], v[3]) for f, v in out.items()}, flush=True)
