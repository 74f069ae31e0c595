"""Shared-memory layout search for the i-pair scheme of k_kron6 (even n).

A field is addr = i + j*Pj + k*Pk + cell*CS (doubles; Pj, Pk, CS even so that an i-pair
(2q, 2q+1) is one 16-byte word).  Thread t of a cell (TPC = n/2 * n threads, cells
consecutive in the block):
  Z stage (write):  pair q = t % NP, line j = t // NP, loop over k      -> word q + Pj/2 j + Pk/2 k
  Y stage (r/w):    pair q = t % NP, line k = t // NP, loop over j      -> word q + Pj/2 j + Pk/2 k
  X stage (read):   lines (j, k) = (t % n, t // n + r*NP), r = 0, 1, loop over pairs q
128-bit accesses are served per quarter-warp (8 lanes x 16 B); the cost of a warp
instruction is the sum over the four quarters of the largest number of distinct words in
one bank quad (word % 8).  Prints the cheapest layout (max cost over the patterns, then
size) for each n and cells per block.
"""
import sys


def q_cost(words):
    tot = 0
    for qq in range(4):
        part = [w for w in words[8 * qq:8 * qq + 8] if w is not None]
        if not part:
            continue
        by = {}
        for w in set(part):
            by[w % 8] = by.get(w % 8, 0) + 1
        tot += max(by.values())
    return tot


def cost(n, cpb, Pj, Pk, CS, pat):
    NP = n // 2
    tpc = NP * n
    threads = cpb * tpc
    tot = ideal = 0
    for w0 in range(0, threads, 32):
        loops = [(s, r) for s in range(n) for r in range(2)] if pat == "x" else [(s, 0) for s in range(n)]
        for s, r in loops:
            if pat == "x" and s >= NP:
                continue
            words = []
            for t in range(w0, w0 + 32):
                if t >= threads:
                    words.append(None)
                    continue
                c, tt = divmod(t, tpc)
                if pat == "z":
                    q, j, k = tt % NP, tt // NP, s
                elif pat == "y":
                    q, k, j = tt % NP, tt // NP, s
                else:
                    q, j, k = s, tt % n, tt // n + r * NP
                words.append((c * CS + 2 * q + j * Pj + k * Pk) // 2)
            tot += q_cost(words)
            ideal += sum(1 for qq in range(4) if any(w is not None for w in words[8 * qq:8 * qq + 8]))
    return tot / ideal


def search(n, cpb, span=12):
    best = None
    for Pj in range(n, n + span + 1, 2):
        for Pk in range(n * Pj, n * Pj + 2 * span, 2):
            for CS in range(n * Pk, n * Pk + 33, 2):
                c = max(cost(n, cpb, Pj, Pk, CS, p) for p in "zyx")
                key = (round(c, 3), CS)
                if best is None or key < best[0]:
                    best = (key, Pj, Pk, CS)
                if c <= 1.0 and CS <= n ** 3 + 16:
                    return best
    return best


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        n, cpb = map(int, arg.split(","))
        b = search(n, cpb)
        print(f"n={n} CPB={cpb}: cost {b[0][0]} Pj={b[1]} Pk={b[2]} CS={b[3]} ({b[3] / n ** 3:.3f} n^3)", flush=True)
