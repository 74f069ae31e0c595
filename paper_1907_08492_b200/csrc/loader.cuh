// Per-cell staging of the own coefficients and the NL neighbour layers of the six
// faces (Hermite-like reads (p+1)^3 + 4d(p+1)^{d-1} words per cell).
//
// One thread per line of the cell (n^2 threads per cell).  Cell coordinates and
// the six neighbour source pointers are computed once per thread; every thread
// then issues n own loads (coalesced across the cell's threads) and 6*NL face
// loads, all independent (memory-level parallelism), and writes them into the
// cell's shared-memory slots:
//   own   : U[(k*n + j)*P + i]
//   face f: F[f*FACE + (l*n + b)*P + a]   (l = neighbour layer in increasing order)
// Mirror faces read the own cell reflected and negated (ghost = -reflect(u):
// trace -u, normal derivative +du/dn).
#pragma once
#include <cstdint>

#include "dg_internal.h"

namespace dgb {

template <int N>
__device__ __forceinline__ int face_elem(int d, int m, int a, int b) {
  return d == 0 ? (b * N + a) * N + m : (d == 1 ? (b * N + m) * N + a : (m * N + b) * N + a);
}

struct FaceSrc {
  const double* base;   // element (m, a, b) at base + face_elem(d, m', a, b)
  double sign;          // -1 for mirror ghosts
  int reflect;          // m' = N-1-m (mirror) or m
  int mirror;           // 1 if the face is a mirror boundary
};

template <int N, int NL>
__device__ __forceinline__ FaceSrc face_source(const GridArgs& g, const double* __restrict__ u,
                                               int64_t cid, int cx, int cy, int cz, int f) {
  constexpr int NN = N * N;
  const int d = f >> 1, s = f & 1;
  const int cd = d == 0 ? cx : (d == 1 ? cy : cz);
  const int Nd = d == 0 ? g.Nx : (d == 1 ? g.Ny : g.nz);
  int nb = cd + (s ? 1 : -1);
  FaceSrc r;
  r.sign = 1.0;
  r.reflect = 0;
  r.mirror = 0;
  bool halo = false;
  if (nb < 0 || nb >= Nd) {
    int src;
    if (d < 2)
      src = g.bc[d] == DG_BC_PERIODIC ? ZSRC_LOCAL : ZSRC_MIRROR;
    else
      src = s == 0 ? g.zlo : g.zhi;
    if (src == ZSRC_LOCAL) {
      nb = nb < 0 ? nb + Nd : nb - Nd;
    } else if (src == ZSRC_MIRROR) {
      r.mirror = 1;
    } else {
      halo = true;
    }
  }
  if (r.mirror) {
    r.base = u + cid * (int64_t)(N * NN);
    r.sign = -1.0;
    r.reflect = 1;
  } else if (halo) {
    const int64_t cxy = cx + (int64_t)g.Nx * cy;
    const double* hb = s == 0 ? g.halo_lo : g.halo_hi;
    // halo layout [cxy][l][b][a] = layer L = (s==0 ? N-NL+l : l) of a z-neighbour
    r.base = hb + cxy * (NL * NN) - (s == 0 ? (N - NL) * NN : 0);
  } else {
    const int64_t ncid = cid + (int64_t)(nb - cd) *
                                   (d == 0 ? 1 : (d == 1 ? (int64_t)g.Nx : (int64_t)g.Nx * g.Ny));
    r.base = u + ncid * (int64_t)(N * NN);
  }
  return r;
}

// Stage own cell + 6 x NL neighbour layers of cell `cid` into smem (U: own field,
// F: face block).  `line` in [0, n^2).  Returns the per-face mirror flags (bit f).
template <int N, int NL, int P, int FACE>
__device__ __forceinline__ int stage_cell(const GridArgs& g, const double* __restrict__ u,
                                          int64_t cid, int line, double* U, double* F) {
  constexpr int NN = N * N;
  const int plane = g.Nx * g.Ny;
  const int cz = (int)(cid / plane);
  const int rem = (int)(cid - (int64_t)cz * plane);
  const int cy = rem / g.Nx, cx = rem - cy * g.Nx;
  const double* own = u + cid * (int64_t)(N * NN);
  double v[N];
#pragma unroll
  for (int r = 0; r < N; ++r) v[r] = __ldg(own + line + r * NN);
  const int a = line % N, b = line / N;
  double fv[6][NL];
  int mirror_bits = 0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const FaceSrc src = face_source<N, NL>(g, u, cid, cx, cy, cz, f);
    mirror_bits |= src.mirror << f;
    const int d = f >> 1, s = f & 1;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int L = s == 0 ? N - NL + l : l;
      const int m = src.reflect ? N - 1 - L : L;
      fv[f][l] = src.sign * __ldg(src.base + face_elem<N>(d, m, a, b));
    }
  }
#pragma unroll
  for (int r = 0; r < N; ++r) {
    const int e = line + r * NN;
    U[(e / N) * P + e % N] = v[r];
  }
#pragma unroll
  for (int f = 0; f < 6; ++f)
#pragma unroll
    for (int l = 0; l < NL; ++l) F[f * FACE + (l * N + b) * P + a] = fv[f][l];
  return mirror_bits;
}

}  // namespace dgb
