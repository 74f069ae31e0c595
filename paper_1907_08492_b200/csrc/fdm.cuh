// FDM transforms of the block-Jacobi preconditioner (Eqs. (13)-(15)),
// shared by the fused Chebyshev kernel (k_kron4.cu) and the standalone P^{-1} (k_solver.cu).
#pragma once
#include "dg_internal.h"

namespace dgb {

// FDM transforms (Eqs. (13)-(15)), even/odd by eigenvector parity (see KronParams):
// forward o = Z^T v (output in the packed eigen index), backward y = Z x.
template <int N, typename KP, typename T>
__device__ __forceinline__ void fdm_fwd(const KP& kp, const T (&v)[N], T (&o)[N]) {
  constexpr int H = N / 2, HS = (N + 1) / 2, HA = N / 2;
  T e[H > 0 ? H : 1], od[H > 0 ? H : 1];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    e[i] = v[i] + v[N - 1 - i];
    od[i] = v[i] - v[N - 1 - i];
  }
#pragma unroll
  for (int s = 0; s < HS; ++s) {
    T acc = (N & 1) ? kp.Zs[H * HS + s] * v[H] : T(0);
#pragma unroll
    for (int i = 0; i < H; ++i) acc = fma(kp.Zs[i * HS + s], e[i], acc);
    o[s] = acc;
  }
#pragma unroll
  for (int a = 0; a < HA; ++a) {
    T acc = T(0);
#pragma unroll
    for (int i = 0; i < H; ++i) acc = fma(kp.Za[i * HA + a], od[i], acc);
    o[HS + a] = acc;
  }
}

template <int N, typename KP, typename T>
__device__ __forceinline__ void fdm_bwd(const KP& kp, const T (&x)[N], T (&y)[N]) {
  constexpr int H = N / 2, HS = (N + 1) / 2, HA = N / 2;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T E = T(0), O = T(0);
#pragma unroll
    for (int s = 0; s < HS; ++s) E = fma(kp.Zs[i * HS + s], x[s], E);
#pragma unroll
    for (int a = 0; a < HA; ++a) O = fma(kp.Za[i * HA + a], x[HS + a], O);
    y[i] = E + O;
    y[N - 1 - i] = E - O;
  }
  if (N & 1) {
    T E = T(0);
#pragma unroll
    for (int s = 0; s < HS; ++s) E = fma(kp.Zs[H * HS + s], x[s], E);
    y[H] = E;
  }
}


}  // namespace dgb
