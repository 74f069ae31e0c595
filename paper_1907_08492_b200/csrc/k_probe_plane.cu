// Design probe (dg_measure_peak kinds 13..18 = 10 + n and, with neighbour traffic, 23..26 = 20 + n;
// not a product kernel): an upper bound
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

// NB = 1 adds the neighbour traffic and arithmetic of the real matvec: per cell 8 n^2 more values
// (2 layers x 4 face neighbours in the two in-plane directions, taken as contiguous 2 n^2 chunks
// of the tiles +-1 row and +-1 plane away, so they come from L2 like the real re-reads) copied
// into the slot with the own tile; per plane 4 ghost lines get a mass sweep and are coupled
// into b, and 4 x 2 neighbour values per row are coupled into a.
template <int N, int NSLOT, int NB>
__global__ void __launch_bounds__(128)
k_plane_probe(const __grid_constant__ ProbeParams pp, const double* __restrict__ in,
              double* __restrict__ out, int64_t ntiles, int64_t trow, int64_t tplane) {
  constexpr int C = PPC<N>::C, NN = N * N, N3 = N * NN;
  constexpr int PK = NN | 1, CS = N * PK;
  constexpr int TE = C * N3, NCP = (TE + 31) / 32;
  constexpr int NP = C * N;                       // planes (one round)
  constexpr int L = C * NN, ZR = (L + 31) / 32;
  constexpr int SLOT0 = C * CS + ((C * CS) & 1);
  constexpr int GH = NB ? 4 * C * 2 * NN : 0;      // ghost values per tile: 4 neighbours x 2 layers
  constexpr int SLOT = SLOT0 + GH + (GH & 1);
  extern __shared__ __align__(16) unsigned char pp_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* const slots = reinterpret_cast<double*>(pp_raw) + warp * (NSLOT * SLOT + SLOT0);
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
    if constexpr (NB) {
      // ghost g = (f, cell, 2 n^2 values): neighbour tile f of {-row, +row, -plane, +plane};
      // even n copies pairs (16-byte cp.async), odd n single values
      constexpr int GV = (N % 2 == 0) ? 2 : 1;
#pragma unroll
      for (int m = 0; m < (GH / GV + 31) / 32; ++m) {
        const int e = (lane + 32 * m) * GV;
        if (e < GH) {
          const int f = e / (C * 2 * NN), r = e % (C * 2 * NN), c = r / (2 * NN), v = r % (2 * NN);
          int64_t tn = t + (f == 0 ? -trow : (f == 1 ? trow : (f == 2 ? -tplane : tplane)));
          if (tn < 0) tn += ntiles;
          if (tn >= ntiles) tn -= ntiles;
          const double* sp = in + tn * TE + c * N3 + ((f & 1) ? v : N3 - 2 * NN + v);
          if constexpr (GV == 2) {
            const unsigned da = (unsigned)__cvta_generic_to_shared(dst + SLOT0 + e);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(da), "l"(sp) : "memory");
          } else {
            cp8(dst + SLOT0 + e, sp);
          }
        }
      }
    }
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
        if constexpr (NB) {   // 2 + 2 neighbour values of this row (the z+- layers)
          const double* G = F + SLOT0 + (2 * C + lane / N) * 2 * NN + (lane % N) * N + j;
          const double zm0 = G[0], zm1 = G[NN], zp0 = G[C * 2 * NN], zp1 = G[C * 2 * NN + NN];
          aa[j][0] = fma(pp.A2[0], zm0, fma(pp.A2[1], zm1, aa[j][0]));
          aa[j][1] = fma(pp.A2[2], zm0, fma(pp.A2[3], zm1, aa[j][1]));
          aa[j][N - 2] = fma(pp.A2[4], zp0, fma(pp.A2[5], zp1, aa[j][N - 2]));
          aa[j][N - 1] = fma(pp.A2[6], zp0, fma(pp.A2[7], zp1, aa[j][N - 1]));
        }
      }
      double gy[4][N];        // M applied to the 4 ghost lines of this plane (the y+- layers)
      if constexpr (NB) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          double x[N];
          const double* G = F + SLOT0 + ((g >> 1) * C + lane / N) * 2 * NN + (g & 1) * NN + (lane % N) * N;
#pragma unroll
          for (int i = 0; i < N; ++i) x[i] = G[i];
          eo_mul<N, 1, false>(pp.A1, eo_split<N>(x), gy[g]);
        }
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
        if constexpr (NB) {
          b[0] = fma(pp.A2[0], gy[0][i], fma(pp.A2[1], gy[1][i], b[0]));
          b[1] = fma(pp.A2[2], gy[0][i], fma(pp.A2[3], gy[1][i], b[1]));
          b[N - 2] = fma(pp.A2[4], gy[2][i], fma(pp.A2[5], gy[3][i], b[N - 2]));
          b[N - 1] = fma(pp.A2[6], gy[2][i], fma(pp.A2[7], gy[3][i], b[N - 1]));
        }
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

template <int N, int NB>
cudaError_t probe_n(double* gdofs, cudaStream_t s) {
  constexpr int C = PPC<N>::C, N3 = N * N * N, NSLOT = (NB && N >= 6) ? 2 : 3;
  constexpr int CS = N * ((N * N) | 1), SLOT0 = C * CS + ((C * CS) & 1);
  constexpr int GH = NB ? 4 * C * 2 * N * N : 0, SLOT = SLOT0 + GH + (GH & 1);
  constexpr int smem = 4 * (NSLOT * SLOT + SLOT0) * 8;
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
  auto kern = k_plane_probe<N, NSLOT, NB>;
  const int64_t trow = 480 / (N * C) + 1, tplane = trow * (480 / N);   // tiles per x-row / per plane of a C4-like mesh
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
        kern<<<sms * cap, 128, smem, s>>>(pp, a, b, ntiles, trow, tplane);
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

// kind = 10 + n, n = 3..8: GDoF/s of the pipelined-plane matvec proxy (see the header);
// kind = 20 + n, n = 3..6: the same with the neighbour traffic and couplings (NB = 1)
cudaError_t measure_plane_probe(int n, double* value, cudaStream_t s) {
  switch (n) {
    case 3: return probe_n<3, 0>(value, s);
    case 4: return probe_n<4, 0>(value, s);
    case 5: return probe_n<5, 0>(value, s);
    case 6: return probe_n<6, 0>(value, s);
    case 7: return probe_n<7, 0>(value, s);
    case 8: return probe_n<8, 0>(value, s);
    case 13: return probe_n<3, 1>(value, s);
    case 14: return probe_n<4, 1>(value, s);
    case 15: return probe_n<5, 1>(value, s);
    case 16: return probe_n<6, 1>(value, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dgb
