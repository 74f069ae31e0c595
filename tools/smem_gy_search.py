"""Bank-conflict search for the y-ghost buffer GY of k_kron4 (half-warp model of
smem_layout_search6.py): addr(c,f,l,k,i) = c*GYC + (f*NL + l)*FS + k*PG + i.
  read  (stage Y): thread (cell c, i, k) reads every (f, l)
  write (stage Z jobs): job j = (cell, f, l, i) writes every k; lanes = consecutive jobs
"""
import sys
from smem_layout_search6 import hw_cost


def cost(n, nl, cpb, PG, FS, GYC):
    tpc = n * n
    T = cpb * tpc
    tot = ideal = 0
    for w0 in range(0, T, 32):                       # reads
        for f in range(2):
            for l in range(nl):
                addrs = []
                for t in range(w0, w0 + 32):
                    if t >= T:
                        addrs.append(None)
                        continue
                    c, line = divmod(t, tpc)
                    i, k = line % n, line // n
                    addrs.append(c * GYC + (f * nl + l) * FS + k * PG + i)
                tot += hw_cost(addrs)
                ideal += sum(1 for h in (addrs[:16], addrs[16:]) if any(a is not None for a in h))
    nyj = 2 * nl * n
    J = cpb * nyj
    for w0 in range(0, J, 32):                       # job writes
        for k in range(n):
            addrs = []
            for j in range(w0, w0 + 32):
                if j >= J:
                    addrs.append(None)
                    continue
                c, jj = divmod(j, nyj)
                f, l, i = jj // (nl * n), (jj // n) % nl, jj % n
                addrs.append(c * GYC + (f * nl + l) * FS + k * PG + i)
            tot += hw_cost(addrs)
            ideal += sum(1 for h in (addrs[:16], addrs[16:]) if any(a is not None for a in h))
    return tot / ideal


n, nl, cpb = map(int, sys.argv[1:4])
best = None
for PG in range(n, n + 9):
    for FS in range(n * PG, n * PG + 17):
        for GYC in range(2 * nl * FS, 2 * nl * FS + 17):
            c = cost(n, nl, cpb, PG, FS, GYC)
            key = (round(c, 3), GYC)
            if best is None or key < best[0]:
                best = (key, PG, FS, GYC)
print(n, nl, cpb, "current", round(cost(n, nl, cpb, n | 1, n * (n | 1), 2 * nl * n * (n | 1)), 3), "best", best)
