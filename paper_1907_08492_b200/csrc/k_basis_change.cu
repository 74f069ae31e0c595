// Sum-factorised basis change v_K = (B (x) B (x) B) u_K per cell, B in
// {T, T^{-1}, T^T, T^{-T}}, T[i][j] = phi_j^H(x_i^GL)  (Eq. (12), PAPER.md:1902-1918;
// SURVEY.md §8(a) a12).  HBM-bound: 16 B/DoF, 3 even-odd sweeps.
// One thread per line (n^2 per cell): coalesced load -> smem, x-sweep and
// y-sweep through smem, z-sweep in registers -> coalesced store.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dg_internal.h"

namespace dgb {
namespace {

template <int N, int CPB, typename Real, typename BP>
__global__ void __launch_bounds__(CPB * N * N)
k_bchg(const __grid_constant__ BP bp, const Real* __restrict__ in,
       Real* __restrict__ out, int64_t ncells) {
  constexpr int P = N | 1, NN = N * N, FIELD = N * N * P;
  __shared__ Real sm[CPB * FIELD];
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int ncell = (int)(ncells - cell0 < CPB ? ncells - cell0 : CPB);
  const int tid = threadIdx.x;
  const Real* src = in + cell0 * (N * NN);
  for (int e = tid; e < ncell * N * NN; e += CPB * NN) {
    const int c = e / (N * NN), r = e % (N * NN);
    sm[c * FIELD + (r / N) * P + r % N] = src[e];
  }
  __syncthreads();
  const int cs = tid / NN, line = tid % NN;
  const bool active = cs < ncell;
  Real* F = sm + cs * FIELD;
  if (active) {  // x-lines
    const int j = line % N, k = line / N;
    Real x[N], o[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = F[(k * N + j) * P + i];
    eo_apply<N, 1>(bp.B, x, o);
#pragma unroll
    for (int i = 0; i < N; ++i) F[(k * N + j) * P + i] = o[i];
  }
  __syncthreads();
  if (active) {  // y-lines
    const int i = line % N, k = line / N;
    Real x[N], o[N];
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = F[(k * N + j) * P + i];
    eo_apply<N, 1>(bp.B, x, o);
#pragma unroll
    for (int j = 0; j < N; ++j) F[(k * N + j) * P + i] = o[j];
  }
  __syncthreads();
  if (active) {  // z-lines, coalesced store
    const int i = line % N, j = line / N;
    Real x[N], o[N];
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = F[(k * N + j) * P + i];
    eo_apply<N, 1>(bp.B, x, o);
    Real* dst = out + (cell0 + cs) * (N * NN) + j * N + i;
#pragma unroll
    for (int k = 0; k < N; ++k) dst[k * NN] = o[k];
  }
}

template <int N, typename Real, typename BP>
cudaError_t launch_n(const BP& bp, const Real* in, Real* out, int64_t ncells, cudaStream_t s) {
  constexpr int CPB = (256 + N * N - 1) / (N * N);
  if (ncells <= 0) return cudaSuccess;
  const int64_t blocks = (ncells + CPB - 1) / CPB;
  k_bchg<N, CPB, Real, BP><<<(unsigned)blocks, CPB * N * N, 0, s>>>(bp, in, out, ncells);
  return cudaGetLastError();
}

template <typename Real, typename BP>
cudaError_t launch_any(int n, const BP& bp, const Real* in, Real* out, int64_t ncells, cudaStream_t s) {
  switch (n) {
    case 2: return launch_n<2>(bp, in, out, ncells, s);
    case 3: return launch_n<3>(bp, in, out, ncells, s);
    case 4: return launch_n<4>(bp, in, out, ncells, s);
    case 5: return launch_n<5>(bp, in, out, ncells, s);
    case 6: return launch_n<6>(bp, in, out, ncells, s);
    case 7: return launch_n<7>(bp, in, out, ncells, s);
    case 8: return launch_n<8>(bp, in, out, ncells, s);
    case 9: return launch_n<9>(bp, in, out, ncells, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_basis_change(int n, const BchgParams& bp, const double* in, double* out,
                                int64_t ncells, cudaStream_t s) {
  return launch_any<double>(n, bp, in, out, ncells, s);
}

// fp32 basis change: the same kernel on floats, B rounded once
cudaError_t launch_basis_change_f32(int n, const BchgParamsF& bp, const float* in, float* out,
                                    int64_t ncells, cudaStream_t s) {
  return launch_any<float>(n, bp, in, out, ncells, s);
}

}  // namespace dgb
