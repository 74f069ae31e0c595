// Design probe (dg_measure_peak kinds 13..18 = 10 + n, not a product kernel): an upper bound
// for the matvec schedule DESIGN.md §11 proposes for n >= 4 -- k_kron6's i-plane arithmetic on
// k_bchgp's skeleton (warp-private cp.async tile slots two stages ahead, no block barrier).
// It performs the Cartesian matvec's seven 1D sweeps and its shared-memory crossings on
// synthetic (pseudo-random) data, WITHOUT the neighbour terms (no z/y/x ghost layers, no boundary logic):
//   plane phase (lane owns the n^2 plane of one cell index): per row  t = A1 u, a = A2 u  (the
//     z stage: M_z, L_z), per column  b = A1 a + A2 t, c = A1 t  (the y stage); b overwrites the
//     plane in the slot, c goes to a second warp-private buffer;
//   line phase (lane owns a line across the planes): y = A1 b + A2 c (the x stage), stored
//     straight to global.
// 16 B/DoF of HBM traffic like the matvec, 40 B/DoF of shared-memory traffic (k_kron4: 64+).
// The number it returns (GDoF/s) bounds what the full kernel could reach; the real kernel adds
// the 2 x NL neighbour layers per face (L2 reads, ~20 % more FMAs) and the boundary cases.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dg_internal.h"

namespace dgb {
namespace {

struct ProbeParams {
  double A1[kEO];
  double A2[kEO];
};

template <int N> struct PPC;   // cells per tile (C n planes <= 32 lanes)
template <> struct PPC<3> { static constexpr int C = 10; };
template <> struct PPC<4> { static constexpr int C = 8; };
template <> struct PPC<5> { static constexpr int C = 6; };
template <> struct PPC<6> { static constexpr int C = 5; };
template <> struct PPC<7> { static constexpr int C = 4; };
template <> struct PPC<8> { static constexpr int C = 4; };

__device__ __forceinline__ void cp8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

template <int N, int NSLOT>
__global__ void __launch_bounds__(128)
k_plane_probe(const __grid_constant__ ProbeParams pp, const double* __restrict__ in,
              double* __restrict__ out, int64_t ntiles) {
  constexpr int C = PPC<N>::C, NN = N * N, N3 = N * NN;
  constexpr int PK = NN | 1, CS = N * PK;
  constexpr int TE = C * N3, NCP = (TE + 31) / 32;
  constexpr int NP = C * N;                       // planes (one round)
  constexpr int L = C * NN, ZR = (L + 31) / 32;
  constexpr int SLOT = C * CS + ((C * CS) & 1);
  extern __shared__ __align__(16) unsigned char pp_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* const slots = reinterpret_cast<double*>(pp_raw) + warp * ((NSLOT + 1) * SLOT);
  double* const Cb = slots + NSLOT * SLOT;        // the c field of the current tile

  int off[NCP];
#pragma unroll
  for (int m = 0; m < NCP; ++m) {
    const int e = lane + 32 * m;
    off[m] = e + (e / NN) * (PK - NN);
  }
  int bz[ZR], gz[ZR];
#pragma unroll
  for (int r = 0; r < ZR; ++r) {
    const int q = lane + 32 * r, c = q / NN, rem = q % NN;
    bz[r] = c * CS + rem;
    gz[r] = c * N3 + rem;
  }
  const int64_t gw = (int64_t)blockIdx.x * 4 + warp, nw = (int64_t)gridDim.x * 4;
  auto issue = [&](int64_t t, int s) {
    const double* src = in + t * TE;
    double* dst = slots + s * SLOT;
#pragma unroll
    for (int m = 0; m < NCP; ++m)
      if (lane + 32 * m < TE) cp8(dst + off[m], src + lane + 32 * m);
  };
#pragma unroll
  for (int s = 0; s < NSLOT - 1; ++s) {
    const int64_t t = gw + s * nw;
    if (t < ntiles) issue(t, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int cur = 0;
  for (int64_t t = gw; t < ntiles; t += nw) {
    {
      const int64_t tn = t + (NSLOT - 1) * nw;
      int ls = cur + NSLOT - 1;
      if (ls >= NSLOT) ls -= NSLOT;
      if (tn < ntiles) issue(tn, ls);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group %0;" ::"n"(NSLOT - 1) : "memory");
    __syncwarp();
    double* F = slots + cur * SLOT;
    if (lane < NP) {
      double* P = F + lane * PK;
      double* Q = Cb + lane * PK;
      double tt[N][N], aa[N][N];
#pragma unroll
      for (int j = 0; j < N; ++j) {          // "z stage": two operators on every row
        double x[N];
#pragma unroll
        for (int i = 0; i < N; ++i) x[i] = P[j * N + i];
        const auto sx = eo_split<N>(x);
        eo_mul<N, 1, false>(pp.A1, sx, tt[j]);
        eo_mul<N, 1, false>(pp.A2, sx, aa[j]);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {          // "y stage": b = A1 a + A2 t, c = A1 t per column
        double xa[N], xt[N], b[N], c[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          xa[j] = aa[j][i];
          xt[j] = tt[j][i];
        }
        const auto st = eo_split<N>(xt);
        eo_mul<N, 1, false>(pp.A1, eo_split<N>(xa), b);
        eo_mul<N, 1, true>(pp.A2, st, b);
        eo_mul<N, 1, false>(pp.A1, st, c);
#pragma unroll
        for (int j = 0; j < N; ++j) {
          P[j * N + i] = b[j];
          Q[j * N + i] = c[j];
        }
      }
    }
    __syncwarp();
    double* dst = out + t * TE;
#pragma unroll
    for (int r = 0; r < ZR; ++r) {
      if (lane + 32 * r < L) {               // "x stage": y = A1 b + A2 c along the lines
        double xb[N], xc[N], y[N];
#pragma unroll
        for (int s = 0; s < N; ++s) {
          xb[s] = F[bz[r] + s * PK];
          xc[s] = Cb[bz[r] + s * PK];
        }
        eo_mul<N, 1, false>(pp.A1, eo_split<N>(xb), y);
        eo_mul<N, 1, true>(pp.A2, eo_split<N>(xc), y);
#pragma unroll
        for (int s = 0; s < N; ++s) dst[gz[r] + s * NN] = y[s];
      }
    }
    __syncwarp();
    if (++cur == NSLOT) cur = 0;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// pseudo-random doubles in [-1, 1) (zeros would toggle fewer bits and flatter the power-capped clocks)
__global__ void k_probe_fill(double* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    a[i] = (double)(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

template <int N>
cudaError_t probe_n(double* gdofs, cudaStream_t s) {
  constexpr int C = PPC<N>::C, N3 = N * N * N, NSLOT = 3;
  constexpr int CS = N * ((N * N) | 1), SLOT = C * CS + ((C * CS) & 1);
  constexpr int smem = 4 * (NSLOT + 1) * SLOT * 8;
  const int64_t ntiles = (int64_t)(110.6e6 / (C * N3));       // ~110 M DoF like the C4 meshes
  const int64_t nd = ntiles * C * N3;
  double *a, *b;
  cudaError_t e = cudaMalloc(&a, nd * 8);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&b, nd * 8);
  if (e != cudaSuccess) {
    cudaFree(a);
    return e;
  }
  k_probe_fill<<<148 * 8, 256, 0, s>>>(a, nd);
  ProbeParams pp{};
  for (int k = 0; k < kEO; ++k) {
    pp.A1[k] = 0.25 + 0.01 * k;
    pp.A2[k] = -0.125 + 0.02 * k;
  }
  auto kern = k_plane_probe<N, NSLOT>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 0, bps = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 128, smem);
  if (e == cudaSuccess && bps < 1) e = cudaErrorLaunchOutOfResources;
  float best = 1e30f;
  if (e == cudaSuccess) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int cap = 1; cap <= 2 && cap <= bps; ++cap) {        // one and two blocks per SM
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, s);
        kern<<<sms * cap, 128, smem, s>>>(pp, a, b, ntiles);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
    }
    e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  cudaFree(a);
  cudaFree(b);
  *gdofs = (double)nd / (best * 1e-3) / 1e9;
  return e;
}

}  // namespace

// kind = 10 + n, n = 3..8: GDoF/s of the pipelined-plane matvec proxy (see the header)
cudaError_t measure_plane_probe(int n, double* value, cudaStream_t s) {
  switch (n) {
    case 3: return probe_n<3>(value, s);
    case 4: return probe_n<4>(value, s);
    case 5: return probe_n<5>(value, s);
    case 6: return probe_n<6>(value, s);
    case 7: return probe_n<7>(value, s);
    case 8: return probe_n<8>(value, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dgb
