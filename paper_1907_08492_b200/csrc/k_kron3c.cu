// Cartesian fast path at n = 3 (p = 2): one thread per cell (k_kron3c).
//
// Same operator as k_kron4 — the Kronecker form of Eq. (14) with the
// neighbour couplings N^{+-} on the NL layers next to each face — and the
// same fused Chebyshev step (Eqs. (11)-(12)).  At n = 3 a
// cell has 27 DoF, so a thread keeps the whole cell in registers: every 1D sweep of every
// direction runs in registers with the coefficients amortised over the cell's 9 lines, and no
// shared-memory transposes or block barriers are needed (k_kron4 at n = 3 spends ~120 of its
// 270 instructions per DoF on index/control work and runs its LSU pipe at 87 %).
//
// A warp owns a tile of up to 32 consecutive cells of one x-row (lane = cell).  Global data
// moves through per-warp shared-memory slots filled by cp.async with coalesced addresses
// (lane l copies elements l, l+32, ... of the contiguous tile) and read back per cell with
// stride 27 doubles (conflict free).  Neighbours:
//   z: the tile of the plane above / below (or the slab halo, or the mirror ghost);
//   y: the tile of the row above / below -> M_z on its NL layers (the y-ghost of k_kron4);
//   x: the c = M_y M_z u field of the adjacent lane by warp shuffle; at the tile edges the
//      x-neighbour's NL layers are swept by 2*NL*3 helper lanes (z then y), or mirrored.
// Slot schedule (3 slots S0..S2, cp.async groups; K3_NSLOT=4 is the measured-slower variant):
//   u -> S0, z- -> S1, z+ -> S2;  Z stage;  y- -> S0, y+ -> S1 (b -> S2);  Y, X stages;
//   (residual; dinv -> S0, u -> S1, u_prev -> S2;  P^-1 x, y;  z with dinv;  y, x;  update)
//   result staged in S2 (matvec) or S0 and stored with coalesced addresses.  Three full-cell
//   slots (20.7 KB per warp) and 168 registers give 10 warps per SM; copying only the NL layers a
//   neighbour reads (12 warps) measured slower (the per-element 8-byte copies cost more).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "dg_internal.h"
#include "fdm.cuh"

namespace dgb {
namespace {

#ifndef K3_NSLOT
#define K3_NSLOT 3      // tile slots per warp: 3 (10 warps per SM) or 4 (y- copied with the Z-stage
                        // tiles, 8 warps per SM; measured slower: p = 2 Chebyshev 103 vs 119 GDoF/s)
#endif
#ifndef K3_PF
#define K3_PF 0         // L2 prefetch at block start: bit 0 the next plane's u tile, bit 1 this tile's
                        // later Chebyshev streams (b, dinv, u_{j-1}); measured neutral / slower
#endif
#ifndef K3_FAST
#define K3_FAST 1       // full-tile specialisation where the launch allows it (0: always the general kernel)
#endif
#ifndef K3_MINB
#define K3_MINB 10      // __launch_bounds__ min blocks (= warps) per SM: the 3-slot shared-memory limit
#endif

constexpr int N = 3, NN = 9, N3 = 27, TW = 32, NSLOT = K3_NSLOT;
// slot roles (see the schedule in the header)
constexpr int SL_U = 0, SL_ZM = 1, SL_ZP = 2;
constexpr int SL_YM = NSLOT == 4 ? 3 : 0, SL_YP = NSLOT == 4 ? 0 : 1;
constexpr int SL_B = NSLOT == 4 ? 1 : 2, SL_D = NSLOT == 4 ? 2 : 0;
constexpr int SL_UJ = NSLOT == 4 ? 3 : 1, SL_UP = NSLOT == 4 ? 0 : 2;
constexpr int SL_OUT_APPLY = NSLOT == 4 ? 1 : 2, SL_OUT_CHEBY = NSLOT == 4 ? 1 : 0;

__device__ __forceinline__ void l2pf_range(const double* p, int cnt, int lane) {
  const char* c = reinterpret_cast<const char*>(p);
  for (int o = lane * 128; o < cnt * 8; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
}

__device__ __forceinline__ int ix(int i, int j, int k) { return k * NN + j * N + i; }

__device__ __forceinline__ void cpa8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa16(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

// warp-cooperative copy of cnt contiguous doubles into a slot (16-byte copies when both ends
// are 16-byte aligned; the slot bases are), then one commit (an empty group if src == nullptr)
template <bool FAST>
__device__ __forceinline__ void tile_load(double* dst, const double* src, int cnt, int lane) {
  if (src) {
    const bool al16 = FAST || (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    if (FAST || (cnt == TW * N3 && al16)) {   // full tile: 432 16-byte copies, unrolled
#pragma unroll
      for (int it = 0; it < (TW * N3 / 2) / 32; ++it) cpa16(dst + 2 * (lane + 32 * it), src + 2 * (lane + 32 * it));
      if constexpr ((TW * N3 / 2) % 32 != 0) {
        constexpr int e0 = ((TW * N3 / 2) / 32) * 32;
        if (lane < (TW * N3 / 2) % 32) cpa16(dst + 2 * (e0 + lane), src + 2 * (e0 + lane));
      }
    } else if constexpr (FAST) {
    } else if (al16) {
      const int c2 = cnt >> 1;
      for (int e = lane; e < c2; e += 32) cpa16(dst + 2 * e, src + 2 * e);
      if ((cnt & 1) && lane == 0) cpa8(dst + cnt - 1, src + cnt - 1);
    } else {
      for (int e = lane; e < cnt; e += 32) cpa8(dst + e, src + e);
    }
  }
  cpa_commit();
}

// coalesced store of a staged tile (full tiles: unrolled 16-byte stores when aligned)
template <bool FAST>
__device__ __forceinline__ void tile_store(double* dst, const double* src, int cnt, int lane) {
  if (FAST || (cnt == TW * N3 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
    for (int it = 0; it < (TW * N3 / 2) / 32; ++it) {
      const int e = 2 * (lane + 32 * it);
      *reinterpret_cast<double2*>(dst + e) = *reinterpret_cast<const double2*>(src + e);
    }
    if constexpr ((TW * N3 / 2) % 32 != 0) {
      const int e = 2 * (((TW * N3 / 2) / 32) * 32 + lane);
      if (lane < (TW * N3 / 2) % 32) *reinterpret_cast<double2*>(dst + e) = *reinterpret_cast<const double2*>(src + e);
    }
  } else if constexpr (!FAST) {
    for (int e = lane; e < cnt; e += 32) dst[e] = src[e];
  }
}

// FAST: every tile of the launch is a full 32-cell tile with 16-byte aligned sources and
// destinations and no slab halo (the launcher checks), so the copy/store fallbacks, the
// partial-tile guards and the halo path are compiled out (smaller code: fewer instruction
// fetch stalls)
template <int NL, int MODE, bool FAST>
__global__ void __launch_bounds__(TW, K3_MINB) k_kron3c(const __grid_constant__ KronParams kp, const __grid_constant__ GridArgs g,
                                               const double* __restrict__ u, double* __restrict__ y,
                                               const __grid_constant__ ChebyArgs ch) {
  __shared__ __align__(16) double S[NSLOT][TW * N3];
  __shared__ double EXT[2][NL][N][N];   // edge helpers: (M_z u_{x+-})[l][j'][k] at the NL i-layers
  __shared__ double EX[2][NL][N][N];    // edge helpers: c_{x+-} = (M_y M_z u_{x+-})[l][j][k]

  const int lane = threadIdx.x;
  const int cx0 = blockIdx.x * TW, cy = blockIdx.y, cz = g.zbeg + blockIdx.z;
  const int ncell = g.Nx - cx0 < TW ? g.Nx - cx0 : TW;
  const bool active = FAST || lane < ncell;
  const int64_t plane = (int64_t)g.Nx * g.Ny;
  const int64_t rowcell = ((int64_t)cz * g.Ny + cy) * g.Nx;
  const int64_t c0 = rowcell + cx0;   // first cell of the tile
  const int tcnt = ncell * N3;

  // x-neighbour sources of the tile edges (cell index in the row, or -1: mirror)
  const bool xper = g.bc[0] == DG_BC_PERIODIC;
  const int h0 = cx0 > 0 ? cx0 - 1 : (xper ? g.Nx - 1 : -1);
  const int h1 = cx0 + ncell < g.Nx ? cx0 + ncell : (xper ? 0 : -1);
  // y-neighbour rows (-1: mirror)
  const bool yper = g.bc[1] == DG_BC_PERIODIC;
  const int ym_row = cy > 0 ? cy - 1 : (yper ? g.Ny - 1 : -1);
  const int yp_row = cy + 1 < g.Ny ? cy + 1 : (yper ? 0 : -1);
  // z-neighbour tiles: source, cell stride (own layout 27, halo NL*9), layer offset
  const double* zsrc[2];
  int zcs[2], zoff[2];
  bool zmir[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int nz = cz + (s ? 1 : -1);
    zcs[s] = N3;
    zoff[s] = 0;
    zmir[s] = false;
    if (nz >= 0 && nz < g.nz) {
      zsrc[s] = u + (c0 + (s ? plane : -plane)) * N3;
    } else {
      const int src = s ? g.zhi : g.zlo;
      if (src == ZSRC_MIRROR) {
        zsrc[s] = nullptr;
        zmir[s] = true;
      } else if (src == ZSRC_LOCAL) {   // periodic wrap inside the slab
        zsrc[s] = u + (c0 + (s ? -(int64_t)(g.nz - 1) : (int64_t)(g.nz - 1)) * plane) * N3;
      } else if constexpr (!FAST) {     // slab halo: [cell][NL][n][n]
        zsrc[s] = (s ? g.halo_hi : g.halo_lo) + ((int64_t)cy * g.Nx + cx0) * (NL * NN);
        zcs[s] = NL * NN;
        zoff[s] = s ? 0 : (N - NL) * NN;
      }
    }
  }

  const double* ym_src = ym_row >= 0 ? u + (((int64_t)cz * g.Ny + ym_row) * g.Nx + cx0) * N3 : nullptr;
  const double* yp_src = yp_row >= 0 ? u + (((int64_t)cz * g.Ny + yp_row) * g.Nx + cx0) * N3 : nullptr;
  // ---- stage 0: issue the tile copies of the Z stage (and y- with 4 slots)
  tile_load<FAST>(S[SL_U], u + c0 * N3, tcnt, lane);
  tile_load<FAST>(S[SL_ZM], zsrc[0], ncell * zcs[0], lane);
  tile_load<FAST>(S[SL_ZP], zsrc[1], ncell * zcs[1], lane);
  if constexpr (NSLOT == 4) tile_load<FAST>(S[SL_YM], ym_src, tcnt, lane);
  if constexpr ((K3_PF & 2) != 0 && MODE != KMODE_APPLY) {
    l2pf_range(ch.b + c0 * N3, tcnt, lane);
    if (ch.dinv) l2pf_range(ch.dinv + c0 * N3, tcnt, lane);
    if (!ch.first) l2pf_range(ch.u_prev + c0 * N3, tcnt, lane);
  }
  if constexpr ((K3_PF & 1) != 0) {
    if (cz + 1 < g.zend) l2pf_range(u + (c0 + plane) * N3, tcnt, lane);
  }
  // edge helpers (lanes < 2*NL*N): z-line (l, j') of the NL i-layers of the x-neighbour
  constexpr int NEDGE = 2 * NL * N;
  const int es = lane / (NL * N), erem = lane - es * (NL * N), el = erem / N, ejk = erem - el * N;
  const int eh = es ? h1 : h0;
  const bool edge = lane < NEDGE && eh >= 0;
  double eu[N];
  if (edge) {
    const int ei = es ? el : N - NL + el;
    const double* src = u + (rowcell + eh) * N3 + ejk * N + ei;
#pragma unroll
    for (int k = 0; k < N; ++k) eu[k] = __ldg(src + k * NN);
  }

  if constexpr (NSLOT == 4) cpa_wait<1>();   // u, z-, z+ landed (y- may be in flight)
  else cpa_wait<0>();
  __syncwarp();

  // ---- Z: t = M_z u, a = L_z u + N_z^{+-} u_{z+-}
  double t[N3], a[N3];
  if (active) {
    const double* us = S[SL_U] + lane * N3;
    const double* zm_t = S[SL_ZM] + lane * zcs[0] - zoff[0];
    const double* zp_t = S[SL_ZP] + lane * zcs[1] - zoff[1];
#pragma unroll
    for (int j = 0; j < N; ++j) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double uz[N], zm[NL], zp[NL], tl[N], al[N];
#pragma unroll
        for (int k = 0; k < N; ++k) uz[k] = us[ix(i, j, k)];
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int Lm = N - NL + l, Lp = l;
          zm[l] = zmir[0] ? -uz[N - 1 - Lm] : zm_t[ix(i, j, Lm)];
          zp[l] = zmir[1] ? -uz[N - 1 - Lp] : zp_t[ix(i, j, Lp)];
        }
        const auto su = eo_split<N>(uz);
        eo_mul<N, 1, false>(kp.M, su, tl);
        eo_mul<N, 1, false>(kp.L[2], su, al);
        dense_add<NL, NL>(kp.Nm[2], zm, &al[0]);
        dense_add<NL, NL>(kp.Np[2], zp, &al[N - NL]);
#pragma unroll
        for (int k = 0; k < N; ++k) {
          t[ix(i, j, k)] = tl[k];
          a[ix(i, j, k)] = al[k];
        }
      }
    }
  }
  if (edge) {
    double o[N];
    eo_apply<N, 1>(kp.M, eu, o);
#pragma unroll
    for (int k = 0; k < N; ++k) EXT[es][el][ejk][k] = o[k];
  }
  __syncwarp();   // S0..S2 read, EXT written

  // ---- issue the next copies: y+ (y- with 3 slots; the Chebyshev b, and dinv with 4 slots)
  if constexpr (NSLOT == 3) tile_load<FAST>(S[SL_YM], ym_src, tcnt, lane);
  tile_load<FAST>(S[SL_YP], yp_src, tcnt, lane);
  if constexpr (MODE != KMODE_APPLY) {
    tile_load<FAST>(S[SL_B], ch.b + c0 * N3, tcnt, lane);
    if constexpr (NSLOT == 4) {
      tile_load<FAST>(S[SL_D], MODE == KMODE_CHEBY_FDM ? nullptr : ch.dinv + c0 * N3, tcnt, lane);
      cpa_wait<2>();   // y-, y+ landed
    } else {
      cpa_wait<1>();
    }
  } else {
    cpa_wait<0>();
  }
  __syncwarp();

  // ---- Y: b = M_y a + L_y t + N_y^{+-} (M_z u_{y+-}),  c = M_y t   (in place: a <- b, t <- c)
  if (edge) {   // edge helpers: y-sweep of EXT -> EX
    double v[N], o[N];
#pragma unroll
    for (int jp = 0; jp < N; ++jp) v[jp] = EXT[es][el][jp][ejk];   // ejk = k here
    eo_apply<N, 1>(kp.M, v, o);
#pragma unroll
    for (int j = 0; j < N; ++j) EX[es][el][j][ejk] = o[j];
  }
  if (active) {
    const double* ym_t = S[SL_YM] + lane * N3;
    const double* yp_t = S[SL_YP] + lane * N3;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      // y-ghosts of this i: (M_z u_{y+-}) at the neighbours' NL layers, [l][k]
      double gym[NL][N], gyp[NL][N];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        if (ym_row >= 0) {
          double v[N];
#pragma unroll
          for (int k = 0; k < N; ++k) v[k] = ym_t[ix(i, N - NL + l, k)];
          eo_apply<N, 1>(kp.M, v, gym[l]);
        }
        if (yp_row >= 0) {
          double v[N];
#pragma unroll
          for (int k = 0; k < N; ++k) v[k] = yp_t[ix(i, l, k)];
          eo_apply<N, 1>(kp.M, v, gyp[l]);
        }
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double al[N], tl[N], bl[N], cl[N], gm[NL], gp[NL];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          al[j] = a[ix(i, j, k)];
          tl[j] = t[ix(i, j, k)];
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          gm[l] = ym_row >= 0 ? gym[l][k] : -tl[NL - 1 - l];
          gp[l] = yp_row >= 0 ? gyp[l][k] : -tl[N - 1 - l];
        }
        const auto st = eo_split<N>(tl);
        eo_mul2<N, 1>(kp.M, eo_split<N>(al), kp.L[1], st, bl);
        eo_mul<N, 1, false>(kp.M, st, cl);
        dense_add<NL, NL>(kp.Nm[1], gm, &bl[0]);
        dense_add<NL, NL>(kp.Np[1], gp, &bl[N - NL]);
#pragma unroll
        for (int j = 0; j < N; ++j) {
          a[ix(i, j, k)] = bl[j];
          t[ix(i, j, k)] = cl[j];
        }
      }
    }
  }
  __syncwarp();   // EX written, S3 / S0 (y tiles) read

  // ---- X: y = M_x b + L_x c + N_x^{+-} c_{x+-}   (c of the adjacent lanes by shuffle)
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double bl[N], cl[N], res[N], cxm[NL], cxp[NL];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        bl[i] = a[ix(i, j, k)];
        cl[i] = t[ix(i, j, k)];
      }
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int Lm = N - NL + l, Lp = l;
        const double vm = __shfl_up_sync(full, cl[Lm], 1);
        const double vp = __shfl_down_sync(full, cl[Lp], 1);
        cxm[l] = lane > 0 ? vm : (h0 >= 0 ? EX[0][l][j][k] : -cl[N - 1 - Lm]);
        cxp[l] = lane + 1 < ncell ? vp : (h1 >= 0 ? EX[1][l][j][k] : -cl[N - 1 - Lp]);
      }
      eo_mul2<N, 1>(kp.M, eo_split<N>(bl), kp.L[0], eo_split<N>(cl), res);
      dense_add<NL, NL>(kp.Nm[0], cxm, &res[0]);
      dense_add<NL, NL>(kp.Np[0], cxp, &res[N - NL]);
#pragma unroll
      for (int i = 0; i < N; ++i) a[ix(i, j, k)] = res[i];
    }
  }

  if constexpr (MODE == KMODE_APPLY) {
    double* O = S[SL_OUT_APPLY];
    if (active) {
#pragma unroll
      for (int e = 0; e < N3; ++e) O[lane * N3 + e] = a[e];
    }
    __syncwarp();
    double* yt = y + c0 * N3;
    tile_store<FAST>(yt, O, tcnt, lane);
    return;
  } else {
    if constexpr (NSLOT == 4) cpa_wait<1>();   // b landed (dinv may be in flight)
    else cpa_wait<0>();
    __syncwarp();
    if (active) {   // r = b - A u
      const double* bs = S[SL_B] + lane * N3;
#pragma unroll
      for (int e = 0; e < N3; ++e) a[e] = bs[e] - a[e];
    }
    __syncwarp();   // the y tiles and b are free
    if constexpr (NSLOT == 3) tile_load<FAST>(S[SL_D], MODE == KMODE_CHEBY_FDM ? nullptr : ch.dinv + c0 * N3, tcnt, lane);
    tile_load<FAST>(S[SL_UJ], u + c0 * N3, tcnt, lane);
    tile_load<FAST>(S[SL_UP], ch.first ? nullptr : ch.u_prev + c0 * N3, tcnt, lane);
    double* z = a;   // P^{-1} r in place
    if constexpr (MODE == KMODE_CHEBY_PJ) {
      cpa_wait<2>();   // dinv
      __syncwarp();
      if (active) {
        const double* ds = S[SL_D] + lane * N3;
#pragma unroll
        for (int e = 0; e < N3; ++e) z[e] *= ds[e];
      }
    } else {
      // x, y: T^{-T} (FDM: Z^T)
#pragma unroll
      for (int k = 0; k < N; ++k) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double v[N], o[N];
#pragma unroll
          for (int i = 0; i < N; ++i) v[i] = z[ix(i, j, k)];
          if constexpr (MODE == KMODE_CHEBY_FDM) fdm_fwd<N>(kp, v, o);
          else eo_apply<N, 1>(kp.TiT, v, o);
#pragma unroll
          for (int i = 0; i < N; ++i) z[ix(i, j, k)] = o[i];
        }
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double v[N], o[N];
#pragma unroll
          for (int j = 0; j < N; ++j) v[j] = z[ix(i, j, k)];
          if constexpr (MODE == KMODE_CHEBY_FDM) fdm_fwd<N>(kp, v, o);
          else eo_apply<N, 1>(kp.TiT, v, o);
#pragma unroll
          for (int j = 0; j < N; ++j) z[ix(i, j, k)] = o[j];
        }
      }
      cpa_wait<2>();   // dinv
      __syncwarp();
      // z: T^{-T}, diag(A_GL)^{-1}, T^{-1}   (FDM: Z^T, 1/(sum_d c_d lam), Z)
      const double* ds = S[SL_D] + lane * N3;
#pragma unroll
      for (int j = 0; j < N; ++j) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double v[N], o[N];
#pragma unroll
          for (int k = 0; k < N; ++k) v[k] = z[ix(i, j, k)];
          if constexpr (MODE == KMODE_CHEBY_FDM) {
            fdm_fwd<N>(kp, v, o);
            const double base = fma(kp.cdir[0], kp.lam[i], kp.cdir[1] * kp.lam[j]);
#pragma unroll
            for (int k = 0; k < N; ++k) o[k] /= fma(kp.cdir[2], kp.lam[k], base);
            fdm_bwd<N>(kp, o, v);
          } else {
            eo_apply<N, 1>(kp.TiT, v, o);
            if (active) {
#pragma unroll
              for (int k = 0; k < N; ++k) o[k] *= ds[ix(i, j, k)];
            }
            eo_apply<N, 1>(kp.Ti, o, v);
          }
#pragma unroll
          for (int k = 0; k < N; ++k) z[ix(i, j, k)] = v[k];
        }
      }
      // y, x: T^{-1} (FDM: Z)
#pragma unroll
      for (int k = 0; k < N; ++k) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double v[N], o[N];
#pragma unroll
          for (int j = 0; j < N; ++j) v[j] = z[ix(i, j, k)];
          if constexpr (MODE == KMODE_CHEBY_FDM) fdm_bwd<N>(kp, v, o);
          else eo_apply<N, 1>(kp.Ti, v, o);
#pragma unroll
          for (int j = 0; j < N; ++j) z[ix(i, j, k)] = o[j];
        }
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double v[N], o[N];
#pragma unroll
          for (int i = 0; i < N; ++i) v[i] = z[ix(i, j, k)];
          if constexpr (MODE == KMODE_CHEBY_FDM) fdm_bwd<N>(kp, v, o);
          else eo_apply<N, 1>(kp.Ti, v, o);
#pragma unroll
          for (int i = 0; i < N; ++i) z[ix(i, j, k)] = o[i];
        }
      }
    }
    cpa_wait<0>();   // u, u_prev
    __syncwarp();
    // three-term update, Eq. (11): u_{j+1} = u_j + c_prev (u_j - u_{j-1}) + c_z z
    double* O = S[SL_OUT_CHEBY];
    if (active) {
      const double* uj = S[SL_UJ] + lane * N3;
      const double* up = S[SL_UP] + lane * N3;
#pragma unroll
      for (int e = 0; e < N3; ++e) {
        double v = fma(ch.c_z, z[e], uj[e]);
        if (!ch.first) v = fma(ch.c_prev, uj[e] - up[e], v);
        O[lane * N3 + e] = v;
      }
    }
    __syncwarp();
    double* ot = ch.u_next + c0 * N3;
    tile_store<FAST>(ot, O, tcnt, lane);
  }
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int NL, int MODE>
cudaError_t launch_t(const KronParams& kp, const GridArgs& g, const double* u, double* y, const ChebyArgs& ch,
                     cudaStream_t s) {
  const int planes = g.zend - g.zbeg;
  if (planes <= 0 || g.Nx <= 0 || g.Ny <= 0) return cudaSuccess;
  if (g.Ny > 65535 || planes > 65535) return cudaErrorInvalidValue;
  const dim3 grid((g.Nx + TW - 1) / TW, g.Ny, planes);
  const bool ptrs = MODE == KMODE_APPLY ? al16(u) && al16(y)
                                        : al16(u) && al16(ch.b) && al16(ch.u_next) && (ch.first || al16(ch.u_prev)) &&
                                              (MODE == KMODE_CHEBY_FDM || al16(ch.dinv));
  const bool fast = K3_FAST && g.Nx % TW == 0 && g.zlo != ZSRC_HALO && g.zhi != ZSRC_HALO && ptrs;
  if (fast)
    k_kron3c<NL, MODE, true><<<grid, TW, 0, s>>>(kp, g, u, y, ch);
  else
    k_kron3c<NL, MODE, false><<<grid, TW, 0, s>>>(kp, g, u, y, ch);
  return cudaGetLastError();
}

template <int NL>
cudaError_t launch_mode(int mode, const KronParams& kp, const GridArgs& g, const double* u, double* y,
                        const ChebyArgs& ch, cudaStream_t s) {
  switch (mode) {
    case KMODE_APPLY: return launch_t<NL, KMODE_APPLY>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_GL: return launch_t<NL, KMODE_CHEBY_GL>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_PJ: return launch_t<NL, KMODE_CHEBY_PJ>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_FDM: return launch_t<NL, KMODE_CHEBY_FDM>(kp, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool kron3c_supported(int n, int NL) { return n == 3 && (NL == 2 || NL == 3); }

cudaError_t launch_kron3c(int NL, int mode, const KronParams& kp, const GridArgs& g, const double* u, double* y,
                          const ChebyArgs& ch, cudaStream_t s) {
  if (NL == 2) return launch_mode<2>(mode, kp, g, u, y, ch, s);
  if (NL == 3) return launch_mode<3>(mode, kp, g, u, y, ch, s);
  return cudaErrorInvalidValue;
}

}  // namespace dgb
