// Warp-private, software-pipelined basis change (k_bchgw): v_K = (B (x) B (x) B) u_K per cell,
// B in {T, T^{-1}, T^T, T^{-T}} (Eq. (12)).
// HBM-bound: 16 B/DoF, 3 even-odd sweeps.
//
// The block-staged k_bchg loads, sweeps and stores a tile between block barriers, so the bytes
// a SM keeps in flight are whatever its resident blocks happen to be loading (4.2-5.7 TB/s on
// the C4 meshes).  Here every warp streams its own tiles of C cells through NSLOT private
// shared-memory slots: the tiles NSLOT-1 ahead are in flight as 8-byte (4-byte for fp32)
// cp.async copies into a padded layout while the current one is swept in place (x, y, z; lane l
// of round r owns line l + 32 r; only __syncwarp between sweeps, no block barrier), and the
// result leaves with fully coalesced stores.  In place (in == out) is safe: a tile is complete
// in its slot before any of it is written, and tiles are disjoint.
// Layouts addr = i + j*Pj + k*Pk + cell*CS from tools/bchgw_layout_search.py (half-warp model).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "dg_internal.h"

namespace dgb {
namespace {

template <int N> struct BWC;
template <> struct BWC<2> { static constexpr int C = 32, Pj = 2, Pk = 5, CS = 12; };
template <> struct BWC<3> { static constexpr int C = 16, Pj = 3, Pk = 9, CS = 27; };
template <> struct BWC<4> { static constexpr int C = 8, Pj = 4, Pk = 19, CS = 73; };
template <> struct BWC<5> { static constexpr int C = 5, Pj = 5, Pk = 25, CS = 125; };
template <> struct BWC<6> { static constexpr int C = 4, Pj = 6, Pk = 39, CS = 244; };
template <> struct BWC<7> { static constexpr int C = 3, Pj = 7, Pk = 52, CS = 369; };
template <> struct BWC<8> { static constexpr int C = 2, Pj = 9, Pk = 72, CS = 575; };
template <> struct BWC<9> { static constexpr int C = 1, Pj = 9, Pk = 81, CS = 729; };

constexpr int kBwWarps = 4;     // warps per block (independent of each other)
#ifndef K_BPC4
#define K_BPC4 8                // plane mode: cells per tile at n = 4 / n = 6
#endif
#ifndef K_BPC6
#define K_BPC6 5
#endif

template <typename Real>
__device__ __forceinline__ void cp_async_elem(Real* dst, const Real* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if constexpr (sizeof(Real) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

// one sweep over the lines of a tile, two rounds at a time (loads of both lines first)
template <int N, int NR, int STRIDE, typename Real>
__device__ __forceinline__ void sweep_tile(Real* __restrict__ F, const int (&base)[NR], int lane, int nl,
                                           const Real* __restrict__ B) {
#pragma unroll
  for (int r = 0; r < NR; r += 2) {
    Real x0[N], x1[N], o[N];
    const bool a0 = lane + 32 * r < nl;
    const bool a1 = (r + 1 < NR) && (lane + 32 * (r + 1) < nl);
    if (a0) {
#pragma unroll
      for (int s = 0; s < N; ++s) x0[s] = F[base[r] + s * STRIDE];
    }
    if (a1) {
#pragma unroll
      for (int s = 0; s < N; ++s) x1[s] = F[base[r + 1 < NR ? r + 1 : r] + s * STRIDE];
    }
    if (a0) {
      eo_apply<N, 1>(B, x0, o);
#pragma unroll
      for (int s = 0; s < N; ++s) F[base[r] + s * STRIDE] = o[s];
    }
    if (a1) {
      eo_apply<N, 1>(B, x1, o);
#pragma unroll
      for (int s = 0; s < N; ++s) F[base[r + 1 < NR ? r + 1 : r] + s * STRIDE] = o[s];
    }
  }
}

template <int N, int NSLOT, bool ZDIRECT, typename Real, typename BP>
__global__ void __launch_bounds__(kBwWarps * 32)
k_bchgw(const __grid_constant__ BP bp, const Real* __restrict__ in, Real* __restrict__ out,
        int64_t ncells, int64_t ntiles) {
  using W = BWC<N>;
  constexpr int C = W::C, NN = N * N, N3 = N * NN;
  constexpr int TE = C * N3;                 // elements of a full tile
  constexpr int NCP = (TE + 31) / 32;        // copy rounds
  constexpr int L = C * NN;                  // lines per sweep
  constexpr int NR = (L + 31) / 32;          // line rounds
  constexpr int SLOT = C * W::CS + ((C * W::CS) & 1);
  extern __shared__ __align__(16) unsigned char bw_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Real* const slots = reinterpret_cast<Real*>(bw_raw) + warp * (NSLOT * SLOT);

  // tile-invariant offsets of this lane: copy elements and the line bases of the three sweeps
  int off[NCP];
#pragma unroll
  for (int m = 0; m < NCP; ++m) {
    const int e = lane + 32 * m, c = e / N3, r = e % N3;
    off[m] = (r % N) + ((r / N) % N) * W::Pj + (r / NN) * W::Pk + c * W::CS;
  }
  int bx[NR], by[NR], bz[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int q = lane + 32 * r, c = q / NN, rem = q % NN, a = rem % N, b = rem / N;
    bx[r] = c * W::CS + b * W::Pk + a * W::Pj;   // x-line (j, k) = (a, b)
    by[r] = c * W::CS + b * W::Pk + a;           // y-line (i, k) = (a, b)
    bz[r] = c * W::CS + b * W::Pj + a;           // z-line (i, j) = (a, b)
  }

  const int64_t gw = (int64_t)blockIdx.x * kBwWarps + warp, nw = (int64_t)gridDim.x * kBwWarps;
  auto tile_cells = [&](int64_t t) -> int {
    const int64_t left = ncells - t * C;
    return (int)(left < C ? left : C);
  };
  auto issue = [&](int64_t t, int s) {
    const int ne = tile_cells(t) * N3;
    const Real* src = in + t * TE;
    Real* dst = slots + s * SLOT;
#pragma unroll
    for (int m = 0; m < NCP; ++m)
      if (lane + 32 * m < ne) cp_async_elem(dst + off[m], src + lane + 32 * m);
  };

#pragma unroll
  for (int s = 0; s < NSLOT - 1; ++s) {
    const int64_t t = gw + s * nw;
    if (t < ntiles) issue(t, s);
    cp_async_commit();
  }
  int cur = 0;
  for (int64_t t = gw; t < ntiles; t += nw) {
    {
      const int64_t tn = t + (NSLOT - 1) * nw;
      int ls = cur + NSLOT - 1;
      if (ls >= NSLOT) ls -= NSLOT;
      if (tn < ntiles) issue(tn, ls);
      cp_async_commit();
    }
    cp_async_wait<NSLOT - 1>();
    __syncwarp();
    Real* F = slots + cur * SLOT;
    const int nc = tile_cells(t), nl = nc * NN, ne = nc * N3;
    sweep_tile<N, NR, 1>(F, bx, lane, nl, bp.B);
    __syncwarp();
    sweep_tile<N, NR, W::Pj>(F, by, lane, nl, bp.B);
    __syncwarp();
    Real* dst = out + t * TE;
    if constexpr (ZDIRECT) {
      // z-lines straight to global: n^2-contiguous segments per k
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (lane + 32 * r < nl) {
          Real x[N], o[N];
#pragma unroll
          for (int s = 0; s < N; ++s) x[s] = F[bz[r] + s * W::Pk];
          eo_apply<N, 1>(bp.B, x, o);
          const int q = lane + 32 * r, c = q / NN, rem = q % NN;
#pragma unroll
          for (int s = 0; s < N; ++s) dst[c * N3 + s * NN + rem] = o[s];
        }
      }
    } else {
      sweep_tile<N, NR, W::Pk>(F, bz, lane, nl, bp.B);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < NCP; ++m)
        if (lane + 32 * m < ne) dst[lane + 32 * m] = F[off[m]];
    }
    __syncwarp();   // the slot is refilled by the next iteration's copies
    if (++cur == NSLOT) cur = 0;
  }
  cp_async_wait<0>();
}


// ---- plane mode (k_bchgp) ---------------------------------------------------------------
// The line sweeps above move every value through shared memory six times (1.3-1.6x that in
// wavefronts with the bank conflicts the padded layouts cannot remove), and ncu shows the LSU
// pipe, not HBM, bounding k_bchgw.  Here a lane owns a whole (i, j) plane of one cell (n^2
// values in registers): the x- and y-sweeps run in registers, so a value crosses shared memory
// three times (cp.async in, plane write-back, z-line read), all conflict free with the plane
// pitch Pk = n^2 | 1 (lane stride odd; CS = n Pk makes plane q of a tile start at q Pk; see bp_pk).  The
// z-lines are stored straight to global (n^2-contiguous segments per k).
template <int N> struct BPC;   // cells per tile: C n planes fill one or more rounds of 32 lanes
template <> struct BPC<2> { static constexpr int C = 32; };
template <> struct BPC<3> { static constexpr int C = 32; };
template <> struct BPC<4> { static constexpr int C = K_BPC4; };
template <> struct BPC<5> { static constexpr int C = 12; };
template <> struct BPC<6> { static constexpr int C = K_BPC6; };
template <> struct BPC<7> { static constexpr int C = 4; };
template <> struct BPC<8> { static constexpr int C = 4; };
template <> struct BPC<9> { static constexpr int C = 3; };

// fp64 at even n moves pairs: 16-byte cp.async, LDS.128 / STS.128 on the planes (pitch n^2 + 2:
// the lane stride is an odd number of 16-byte units, conflict free per quarter-warp) and two
// adjacent z-lines per lane with 16-byte global stores; half the memory instructions (ncu: the
// 8-byte version at n = 4 stalls on mio_throttle, 3.2 cycles per issue with 16 warps per SM).
// Measured (C4, GB/s): n = 4 5592 -> 6321, n = 6 5040 -> 6326; n = 8 is slower with pairs (6206 -> 5640:
// 176 registers), so it keeps the 8-byte path.
template <int N, typename Real> constexpr int bp_vec() { return (sizeof(Real) == 8 && N % 2 == 0 && N < 8) ? 2 : 1; }
template <int N, typename Real> constexpr int bp_pk() { return bp_vec<N, Real>() == 2 ? N * N + 2 : ((N * N) | 1); }

template <int N, int NSLOT, typename Real, typename BP>
__global__ void __launch_bounds__(kBwWarps * 32)
k_bchgp(const __grid_constant__ BP bp, const Real* __restrict__ in, Real* __restrict__ out,
        int64_t ncells, int64_t ntiles) {
  constexpr int C = BPC<N>::C, NN = N * N, N3 = N * NN;
  constexpr int VEC = bp_vec<N, Real>();
  constexpr int PK = bp_pk<N, Real>(), CS = N * PK;
  constexpr int TE = C * N3, NCP = (TE / VEC + 31) / 32;   // copy rounds (chunks of VEC elements)
  constexpr int NP = C * N, PR = (NP + 31) / 32;           // planes, plane rounds
  constexpr int L = C * NN / VEC, ZR = (L + 31) / 32;      // z-line groups (VEC adjacent lines), rounds
  constexpr int SLOT = C * CS + ((C * CS) & 1);
  constexpr bool PAD = PK != NN;
  extern __shared__ __align__(16) unsigned char bw_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Real* const slots = reinterpret_cast<Real*>(bw_raw) + warp * (NSLOT * SLOT);

  int off[PAD ? NCP : 1];
  if constexpr (PAD) {
#pragma unroll
    for (int m = 0; m < NCP; ++m) {
      const int e = (lane + 32 * m) * VEC;
      off[m] = e + (e / NN) * (PK - NN);
    }
  }
  int bz[ZR], gz[ZR];
#pragma unroll
  for (int r = 0; r < ZR; ++r) {
    const int q = (lane + 32 * r) * VEC, c = q / NN, rem = q % NN;
    bz[r] = c * CS + rem;
    gz[r] = c * N3 + rem;
  }

  const int64_t gw = (int64_t)blockIdx.x * kBwWarps + warp, nw = (int64_t)gridDim.x * kBwWarps;
  auto tile_cells = [&](int64_t t) -> int {
    const int64_t left = ncells - t * C;
    return (int)(left < C ? left : C);
  };
  auto issue = [&](int64_t t, int s) {
    const int ne = tile_cells(t) * N3;
    const Real* src = in + t * TE;
    Real* dst = slots + s * SLOT;
#pragma unroll
    for (int m = 0; m < NCP; ++m) {
      const int e = (lane + 32 * m) * VEC;
      if (e < ne) {
        Real* d = dst + (PAD ? off[PAD ? m : 0] : e);
        if constexpr (VEC == 2) {
          const unsigned da = (unsigned)__cvta_generic_to_shared(d);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(da), "l"(src + e) : "memory");
        } else {
          cp_async_elem(d, src + e);
        }
      }
    }
  };

#pragma unroll
  for (int s = 0; s < NSLOT - 1; ++s) {
    const int64_t t = gw + s * nw;
    if (t < ntiles) issue(t, s);
    cp_async_commit();
  }
  int cur = 0;
  for (int64_t t = gw; t < ntiles; t += nw) {
    {
      const int64_t tn = t + (NSLOT - 1) * nw;
      int ls = cur + NSLOT - 1;
      if (ls >= NSLOT) ls -= NSLOT;
      if (tn < ntiles) issue(tn, ls);
      cp_async_commit();
    }
    cp_async_wait<NSLOT - 1>();
    __syncwarp();
    Real* F = slots + cur * SLOT;
    const int nc = tile_cells(t), np = nc * N, nl = nc * NN / VEC;
#pragma unroll
    for (int r = 0; r < PR; ++r) {
      if (lane + 32 * r < np) {
        Real* P = F + (lane + 32 * r) * PK;
        Real v[N][N], o[N];
        if constexpr (VEC == 2) {
#pragma unroll
          for (int j = 0; j < N; ++j)
#pragma unroll
            for (int i = 0; i < N; i += 2) {
              const double2 w = *reinterpret_cast<const double2*>(P + j * N + i);
              v[j][i] = w.x;
              v[j][i + 1] = w.y;
            }
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j)
#pragma unroll
            for (int i = 0; i < N; ++i) v[j][i] = P[j * N + i];
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {   // x-lines
          eo_apply<N, 1>(bp.B, v[j], o);
#pragma unroll
          for (int i = 0; i < N; ++i) v[j][i] = o[i];
        }
#pragma unroll
        for (int i = 0; i < N; i += VEC) {   // y-lines (VEC adjacent ones, written back together)
          Real x[N], o2[N];
#pragma unroll
          for (int j = 0; j < N; ++j) x[j] = v[j][i];
          eo_apply<N, 1>(bp.B, x, o);
          if constexpr (VEC == 2) {
#pragma unroll
            for (int j = 0; j < N; ++j) x[j] = v[j][i + 1];
            eo_apply<N, 1>(bp.B, x, o2);
#pragma unroll
            for (int j = 0; j < N; ++j)
              *reinterpret_cast<double2*>(P + j * N + i) = make_double2((double)o[j], (double)o2[j]);
          } else {
#pragma unroll
            for (int j = 0; j < N; ++j) P[j * N + i] = o[j];
          }
        }
      }
    }
    __syncwarp();
    Real* dst = out + t * TE;
#pragma unroll
    for (int r = 0; r < ZR; ++r) {
      if (lane + 32 * r < nl) {
        Real x[N], o[N];
        if constexpr (VEC == 2) {
          Real x2[N], o2[N];
#pragma unroll
          for (int s = 0; s < N; ++s) {
            const double2 w = *reinterpret_cast<const double2*>(F + bz[r] + s * PK);
            x[s] = w.x;
            x2[s] = w.y;
          }
          eo_apply<N, 1>(bp.B, x, o);
          eo_apply<N, 1>(bp.B, x2, o2);
#pragma unroll
          for (int s = 0; s < N; ++s)
            *reinterpret_cast<double2*>(dst + gz[r] + s * NN) = make_double2((double)o[s], (double)o2[s]);
        } else {
#pragma unroll
          for (int s = 0; s < N; ++s) x[s] = F[bz[r] + s * PK];
          eo_apply<N, 1>(bp.B, x, o);
#pragma unroll
          for (int s = 0; s < N; ++s) dst[gz[r] + s * NN] = o[s];
        }
      }
    }
    __syncwarp();   // the slot is refilled by the next iteration's copies
    if (++cur == NSLOT) cur = 0;
  }
  cp_async_wait<0>();
}

template <int N, int NSLOT, bool ZD, bool PLANE, typename Real, typename BP>
cudaError_t launch_cfg(const BP& bp, const Real* in, Real* out, int64_t ncells, cudaStream_t s) {
  using W = BWC<N>;
  constexpr int TC = PLANE ? BPC<N>::C : W::C;                       // cells per tile
  constexpr int TS = PLANE ? BPC<N>::C * N * bp_pk<N, Real>() : W::C * W::CS;
  constexpr int SLOT = TS + (TS & 1);
  constexpr int smem = kBwWarps * NSLOT * SLOT * (int)sizeof(Real);
  void (*kern)(BP, const Real*, Real*, int64_t, int64_t);
  if constexpr (PLANE) kern = k_bchgp<N, NSLOT, Real, BP>;
  else kern = k_bchgw<N, NSLOT, ZD, Real, BP>;
  // SMs x resident blocks (> 0) or minus the CUDA error, found once per instantiation
  // (thread-safe static: the slab-transport tests call this from several host threads)
  static const int grid_cap = [&]() -> int {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return -(int)e;
    int dev = 0, sms = 0, bps = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kBwWarps * 32, smem);
    if (e != cudaSuccess) return -(int)e;
    if (bps < 1 || sms < 1) return -(int)cudaErrorLaunchOutOfResources;
    // blocks per SM: DG_BCHGW_BPS, else one block (4 warps) in plane mode at n = 4 and 6, where more
    // resident warps measured slower (n = 4: 6321 vs 5836 GB/s, n = 6: 6326 vs 5802)
    const char* v = std::getenv("DG_BCHGW_BPS");
    const int cap = v ? std::atoi(v) : ((PLANE && (N == 4 || N == 6)) ? 1 : 0);
    if (cap > 0 && bps > cap) bps = cap;
    int grid = sms * bps;
    // DG_BCHGW_GRID: cap on the number of blocks (tests: many tiles per warp on small meshes)
    const char* g = std::getenv("DG_BCHGW_GRID");
    if (g && std::atoi(g) > 0 && std::atoi(g) < grid) grid = std::atoi(g);
    return grid;
  }();
  if (grid_cap <= 0) return (cudaError_t)(-grid_cap);
  const int64_t ntiles = (ncells + TC - 1) / TC;
  int64_t blocks = (ntiles + kBwWarps - 1) / kBwWarps;
  if (blocks > grid_cap) blocks = grid_cap;
  kern<<<(unsigned)blocks, kBwWarps * 32, smem, s>>>(bp, in, out, ncells, ntiles);
  return cudaGetLastError();
}

template <int N, typename Real, typename BP>
cudaError_t launch_n(const BP& bp, const Real* in, Real* out, int64_t ncells, cudaStream_t s) {
  if (ncells <= 0) return cudaSuccess;
  // mode bit 0 = z-sweep stores straight to global, bit 1 = two slots instead of three (more
  // warps per SM), bit 2 = plane mode (k_bchgp).  Per-n default by measurement (tools/gpu_bchgw.sh,
  // tools/gpu_bchgp*.sh; C4, GB/s at p = 2..8: line mode best 5537/5893/5843/5372/4633/5087/5923,
  // plane mode 6364/6321/6557/6326/6418/6206/3541 (n = 9 spills)); DG_BCHGW_MODE forces one.
  static const int mode = [] {
    const char* v = std::getenv("DG_BCHGW_MODE");
    if (v) return std::atoi(v);
    if (sizeof(Real) == 4) return 6;   // fp32 (8 B/DoF): plane mode, two slots (tools/gpu_bchg_misc.sh)
    return N == 9 ? 3 : (N == 6 ? 6 : 4);
  }();
  if constexpr (sizeof(Real) == 8) {
    switch (mode & 7) {
      case 1: return launch_cfg<N, 3, true, false>(bp, in, out, ncells, s);
      case 2: return launch_cfg<N, 2, false, false>(bp, in, out, ncells, s);
      case 3: return launch_cfg<N, 2, true, false>(bp, in, out, ncells, s);
      case 4: return launch_cfg<N, 3, true, true>(bp, in, out, ncells, s);    // plane mode, 3 slots
      case 6: return launch_cfg<N, 2, true, true>(bp, in, out, ncells, s);    // plane mode, 2 slots
      default: break;
    }
  } else {
    if ((mode & 7) == 4) return launch_cfg<N, 3, true, true>(bp, in, out, ncells, s);
    if ((mode & 7) == 6) return launch_cfg<N, 2, true, true>(bp, in, out, ncells, s);
  }
  return launch_cfg<N, 3, false, false>(bp, in, out, ncells, s);
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

cudaError_t launch_basis_change_w(int n, const BchgParams& bp, const double* in, double* out,
                                  int64_t ncells, cudaStream_t s) {
  return launch_any<double>(n, bp, in, out, ncells, s);
}

cudaError_t launch_basis_change_w_f32(int n, const BchgParamsF& bp, const float* in, float* out,
                                      int64_t ncells, cudaStream_t s) {
  return launch_any<float>(n, bp, in, out, ncells, s);
}

}  // namespace dgb
