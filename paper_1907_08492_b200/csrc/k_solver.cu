// Kernels behind the GPU Lanczos estimate and the preconditioned CG (SURVEY.md §8(f)
// NEXT#4): the standalone inner preconditioner P^{-1} (GL-Jacobi of
// Eq. (12), point Jacobi, or FDM of Eqs. (13)-(15)), a deterministic two-level dot
// product, and the vector updates of the Lanczos and CG recurrences.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dg_internal.h"
#include "fdm.cuh"

namespace dgb {
namespace {

// P^{-1} per cell: x, y, z forward sweeps, diagonal, z, y, x backward sweeps
// (one thread per line, cell staged in smem with a padded row pitch).
template <int N, int CPB, int INNER>
__global__ void __launch_bounds__(CPB * N * N)
k_pinv(const __grid_constant__ KronParams kp, const double* __restrict__ r, const double* __restrict__ dinv,
       double* __restrict__ z, int64_t ncells) {
  constexpr int P = N | 1, NN = N * N, N3 = N * NN, FIELD = N * N * P;
  __shared__ double sm[CPB * FIELD];
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int ncell = (int)(ncells - cell0 < CPB ? ncells - cell0 : CPB);
  const int tid = threadIdx.x;
  for (int e = tid; e < ncell * N3; e += CPB * NN) {
    const int c = e / N3, q = e % N3;
    sm[c * FIELD + (q / N) * P + q % N] = r[cell0 * N3 + e];
  }
  __syncthreads();
  const int cs = tid / NN, line = tid % NN;
  const bool active = cs < ncell;
  double* F = sm + cs * FIELD;
  const int a = line % N, b = line / N;
  auto pre = [&](const double(&x)[N], double(&o)[N]) {
    if constexpr (INNER == DG_INNER_FDM) fdm_fwd<N>(kp, x, o);
    else eo_apply<N, 1>(kp.TiT, x, o);
  };
  auto post = [&](const double(&x)[N], double(&o)[N]) {
    if constexpr (INNER == DG_INNER_FDM) fdm_bwd<N>(kp, x, o);
    else eo_apply<N, 1>(kp.Ti, x, o);
  };
  double x[N], o[N];
  if (active) {   // x-lines (j = a, k = b)
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = F[(b * N + a) * P + i];
    pre(x, o);
#pragma unroll
    for (int i = 0; i < N; ++i) F[(b * N + a) * P + i] = o[i];
  }
  __syncthreads();
  if (active) {   // y-lines (i = a, k = b)
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = F[(b * N + j) * P + a];
    pre(x, o);
#pragma unroll
    for (int j = 0; j < N; ++j) F[(b * N + j) * P + a] = o[j];
  }
  __syncthreads();
  if (active) {   // z-lines (i = a, j = b): forward, diagonal, backward
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = F[(k * N + b) * P + a];
    pre(x, o);
    if constexpr (INNER == DG_INNER_FDM) {
      const double base = fma(kp.cdir[0], kp.lam[a], kp.cdir[1] * kp.lam[b]);
#pragma unroll
      for (int k = 0; k < N; ++k) o[k] /= fma(kp.cdir[2], kp.lam[k], base);
    } else {
      const double* dv = dinv + (cell0 + cs) * N3 + b * N + a;
#pragma unroll
      for (int k = 0; k < N; ++k) o[k] *= __ldg(dv + k * NN);
    }
    post(o, x);
#pragma unroll
    for (int k = 0; k < N; ++k) F[(k * N + b) * P + a] = x[k];
  }
  __syncthreads();
  if (active) {   // y-lines backward
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = F[(b * N + j) * P + a];
    post(x, o);
#pragma unroll
    for (int j = 0; j < N; ++j) F[(b * N + j) * P + a] = o[j];
  }
  __syncthreads();
  if (active) {   // x-lines backward
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = F[(b * N + a) * P + i];
    post(x, o);
#pragma unroll
    for (int i = 0; i < N; ++i) F[(b * N + a) * P + i] = o[i];
  }
  __syncthreads();
  for (int e = tid; e < ncell * N3; e += CPB * NN) {
    const int c = e / N3, q = e % N3;
    z[cell0 * N3 + e] = sm[c * FIELD + (q / N) * P + q % N];
  }
}

__global__ void k_scale(const double* __restrict__ r, const double* __restrict__ d, double* __restrict__ z,
                        int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = r[i] * d[i];
}

constexpr int kDotBlocks = 148 * 4, kDotThreads = 256;

// deterministic dot: fixed grid, per-block tree sums, then one block over the partials
__global__ void __launch_bounds__(kDotThreads) k_dot1(const double* __restrict__ a, const double* __restrict__ b,
                                                      int64_t n, double* __restrict__ part) {
  __shared__ double s[kDotThreads];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kDotThreads + threadIdx.x; i < n; i += (int64_t)kDotBlocks * kDotThreads)
    acc = fma(a[i], b[i], acc);
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void __launch_bounds__(kDotThreads) k_dot2(const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double s[kDotThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) acc += part[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// y = alpha x + beta y  (alpha, beta by value)
__global__ void k_axpby(double alpha, const double* __restrict__ x, double beta, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(alpha, x[i], beta * y[i]);
}

// Lanczos start vector: v_g = (g mod 12) - 5.5, g the global DoF index
__global__ void k_lanczos_start(double* __restrict__ v, int64_t n, int64_t g0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (double)((g0 + i) % 12) - 5.5;
}

__global__ void k_d2f(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}

__global__ void k_f2d(const float* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}

template <int N, int INNER>
cudaError_t launch_pinv_n(const KronParams& kp, const double* r, const double* dinv, double* z, int64_t ncells,
                          cudaStream_t s) {
  constexpr int CPB = (256 + N * N - 1) / (N * N);
  if (ncells <= 0) return cudaSuccess;
  k_pinv<N, CPB, INNER><<<(unsigned)((ncells + CPB - 1) / CPB), CPB * N * N, 0, s>>>(kp, r, dinv, z, ncells);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_pinv_inner(int inner, const KronParams& kp, const double* r, const double* dinv, double* z,
                              int64_t ncells, cudaStream_t s) {
  if (inner == DG_INNER_FDM) return launch_pinv_n<N, DG_INNER_FDM>(kp, r, dinv, z, ncells, s);
  return launch_pinv_n<N, DG_INNER_GL_JACOBI>(kp, r, dinv, z, ncells, s);
}

}  // namespace

cudaError_t launch_pinv(int n, int inner, const KronParams& kp, const double* r, const double* dinv, double* z,
                        int64_t ncells, cudaStream_t s) {
  if (inner == DG_INNER_POINT_JACOBI) {
    const int64_t nd = ncells * n * n * n;
    if (nd <= 0) return cudaSuccess;
    k_scale<<<148 * 8, 256, 0, s>>>(r, dinv, z, nd);
    return cudaGetLastError();
  }
  switch (n) {
    case 2: return launch_pinv_inner<2>(inner, kp, r, dinv, z, ncells, s);
    case 3: return launch_pinv_inner<3>(inner, kp, r, dinv, z, ncells, s);
    case 4: return launch_pinv_inner<4>(inner, kp, r, dinv, z, ncells, s);
    case 5: return launch_pinv_inner<5>(inner, kp, r, dinv, z, ncells, s);
    case 6: return launch_pinv_inner<6>(inner, kp, r, dinv, z, ncells, s);
    case 7: return launch_pinv_inner<7>(inner, kp, r, dinv, z, ncells, s);
    case 8: return launch_pinv_inner<8>(inner, kp, r, dinv, z, ncells, s);
    case 9: return launch_pinv_inner<9>(inner, kp, r, dinv, z, ncells, s);
  }
  return cudaErrorInvalidValue;
}

int dot_partials() { return kDotBlocks; }

cudaError_t launch_d2f(const double* in, float* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_d2f<<<148 * 8, 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t launch_f2d(const float* in, double* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_f2d<<<148 * 8, 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* a, const double* b, int64_t n, double* part, double* out, cudaStream_t s) {
  k_dot1<<<kDotBlocks, kDotThreads, 0, s>>>(a, b, n, part);
  k_dot2<<<1, kDotThreads, 0, s>>>(part, out);
  return cudaGetLastError();
}

cudaError_t launch_axpby(double alpha, const double* x, double beta, double* y, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_axpby<<<148 * 8, 256, 0, s>>>(alpha, x, beta, y, n);
  return cudaGetLastError();
}

cudaError_t launch_lanczos_start(double* v, int64_t n, int64_t g0, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_lanczos_start<<<148 * 8, 256, 0, s>>>(v, n, g0);
  return cudaGetLastError();
}

}  // namespace dgb
