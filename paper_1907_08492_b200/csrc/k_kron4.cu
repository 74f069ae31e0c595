// Cartesian fast path of the SIPG operator, z-first schedule (k_kron4).
//
// On a Cartesian cell the quadrature operator of Eq. (1)
// equals the Kronecker form of Eq. (14) (the paper names the
// reference-coordinate form at PAPER.md:336-344):
//   y_K = (M (x) M (x) L_z + M (x) L_y (x) M + L_x (x) M (x) M) u_K
//       + (M_x M_y N_z^{+-}) u_{z+-} + (M_x N_y^{+-} M_z) u_{y+-} + (N_x^{+-} M_y M_z) u_{x+-}
// (operators act on the index of their direction; N^{+-} touch only the NL = 2 layers
// of the neighbour next to the face for the Hermite-like basis).
//
// Thread mapping: a block is a run of CPB cells of one x-row (grid = x-runs x rows x
// planes); thread t = cell*TPCP + b'*n + a (TPCP = n*NB, or padded, K4C::TP) owns the R lines (a, b' + r*NB),
// NB = ceil(n/R), of every sweep direction, so per-thread setup and the coefficient
// loads are amortised over R lines.  Sweeping z first lets the own data and the raw
// z-neighbour layers stream from HBM along coalesced z-lines:
//   Z  (line (i,j)):  t = M_z u,  a = L_z u + N_z^{+-} u_{z+-}           -> smem (ZY)
//      jobs: M_z on the z-lines of the NL y-neighbour layers (-> GY) and of the NL
//            x-neighbour layers of cells outside the block (-> HT)
//   Y  (line (i,k)):  b = M_y a + L_y t + N_y^{+-} (M_z u_{y+-}),  c = M_y t  -> smem (YX)
//      jobs: M_y on HT -> HC
//   X  (line (j,k)):  y = M_x b + L_x c + N_x^{+-} c_{x+-}
// where c_{x+-} = (M_y M_z u)_{x+-} at the NL layers next to the face is the c field of
// the x-neighbour: read from its block slot, from HC (block edges) or, on mirror faces,
// from the own c reflected and negated.  Mirror faces use the ghost -(own reflected)
// (PAPER.md:172-174): z from the own line in registers, y from the own t, x from c.
// The result is staged in smem and written with coalesced stores.
//
// Fused Chebyshev step (merged; inner GL-Jacobi or FDM): after X, r = b - Au,
// then P^{-1} r = (T^{-1})^{(x)3} diag(A_GL)^{-1} (T^{-T})^{(x)3} r (Eq. (12), R13)
// as x: T^{-T}; z: T^{-T}; y: T^{-T}, diag, T^{-1}; x: T^{-1}; z: T^{-1} + the
// three-term update of Eq. (11) along the z-lines.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "dg_internal.h"
#include "fdm.cuh"

namespace dgb {
namespace {

struct Lay3 {
  int Pj, Pk, CS;
};

#ifndef K4_RLINE
#define K4_RLINE 1      // 1: the R lines of a thread are swept together (coefficients loaded once)
#endif

#ifndef K4_STAGE
#define K4_STAGE 0      // 1: the Chebyshev streams b, u_{j-1}, dinv of the block's cells are copied to
                        //    shared memory with cp.async at block start (CPBS cells per block)
#endif

// Chebyshev L1 prefetch of the block's later stream tiles, issued stages ahead (per n):
// bit 0 b (at the Y stage), bit 1 dinv (at the first P^-1 stage), bit 2 u and u_{j-1} (at the
// second P^-1 stage).  Measured (tools/gpu_r2_ab.sh, C4): dinv +1.5 % at n = 6, u/u_{j-1} +1-2 %
// at n = 8, every bit slower at n = 4, 5, 7, 9; K4_L1PF forces one mask for all n.
#ifdef K4_L1PF
template <int N> constexpr int k4_l1pf() { return K4_L1PF; }
#else
template <int N> constexpr int k4_l1pf() { return N == 6 ? 2 : (N == 8 ? 4 : 0); }
#endif

#ifndef K4_PREB_ODD
#define K4_PREB_ODD 1   // odd-n Chebyshev b preload: 0 none, 1 after the Y->X barrier, 2 before it
#endif

// Per n: lines per thread R, cells per block CPB, and the field layouts
// addr = i + j*Pj + k*Pk + cell*CS chosen by tools/smem_layout_search6.py (half-warp model)
// (ZY: z-write/y-read, YX: y-write/x-read, XZ: x-write/z-read).
template <int N, int ALT = 0> struct K4C;
template <> struct K4C<3> { static constexpr int R = 1, CPB = 32, CPBS = 20, TP = 0, XSW = 0; static constexpr Lay3 ZY{3, 19, 57}, YX{3, 9, 27}, XZ{3, 18, 57}; };
template <> struct K4C<4> { static constexpr int R = 2, CPB = 30, CPBS = 18, TP = 0, XSW = 0; static constexpr Lay3 ZY{4, 20, 88}, YX{5, 20, 88}, XZ{5, 20, 84}; };
template <> struct K4C<5> { static constexpr int R = 2, CPB = 16, CPBS = 11, TP = 0, XSW = 0; static constexpr Lay3 ZY{5, 26, 143}, YX{5, 25, 134}, XZ{5, 25, 139}; };
template <> struct K4C<6> { static constexpr int R = 1, CPB = 8, CPBS = 5, TP = 0, XSW = 0; static constexpr Lay3 ZY{6, 38, 228}, YX{9, 54, 324}, XZ{11, 66, 402}; };
// n = 7 default since round 2 (DG_K4_ALT7, default 2): 32 threads per cell (4 idle), ZY and XZ conflict free
template <> struct K4C<7, 2> { static constexpr int R = 2, CPB = 10, CPBS = 4, TP = 32, XSW = 0; static constexpr Lay3 ZY{7, 55, 385}, YX{7, 56, 392}, XZ{7, 49, 343}; };
template <> struct K4C<7> { static constexpr int R = 2, CPB = 10, CPBS = 4, TP = 0, XSW = 0; static constexpr Lay3 ZY{7, 55, 396}, YX{7, 56, 392}, XZ{7, 49, 344}; };
template <> struct K4C<8> { static constexpr int R = 1, CPB = 4, CPBS = 3, TP = 0, XSW = 0; static constexpr Lay3 ZY{8, 72, 576}, YX{9, 72, 576}, XZ{12, 97, 776}; };
// n = 9 alternate (DG_K4_ALT9=2): the y->x layout padded to a row pitch of 17 (conflict free;
// the default YX{9,85,765} costs 1.94x in the half-warp model).  Measured slower (C4 p=8:
// matvec 139.8 -> 131.6, Chebyshev 87.1 -> 78.0 GDoF/s: 1.7x the shared memory per cell)
template <> struct K4C<9, 2> { static constexpr int R = 1, CPB = 3, CPBS = 2, TP = 0, XSW = 0; static constexpr Lay3 ZY{9, 89, 801}, YX{17, 153, 1377}, XZ{9, 81, 729}; };
template <> struct K4C<9> { static constexpr int R = 1, CPB = 3, CPBS = 2, TP = 0, XSW = 0; static constexpr Lay3 ZY{9, 89, 801}, YX{9, 85, 765}, XZ{9, 81, 729}; };
// alternates (DG_K4_ALT=1): two lines per thread
template <> struct K4C<6, 1> { static constexpr int R = 2, CPB = 16, CPBS = 8, TP = 0, XSW = 0; static constexpr Lay3 ZY{6, 38, 242}, YX{9, 54, 338}, XZ{6, 36, 217}; };
template <> struct K4C<8, 1> { static constexpr int R = 2, CPB = 8, CPBS = 4, TP = 0, XSW = 0; static constexpr Lay3 ZY{8, 72, 576}, YX{9, 72, 576}, XZ{9, 72, 576}; };
// n = 5 alternate: 16 threads per cell (one idle) so that a half-warp never straddles two cells,
// and the x stage maps thread (a, b) to line (j, k) = (b + r NB, a); with these the Y/X
// transposes are bank-conflict free (tools/smem_layout_search7.py / smem_ktable_search.py)
template <> struct K4C<5, 1> { static constexpr int R = 2, CPB = 16, CPBS = 11, TP = 16, XSW = 1; static constexpr Lay3 ZY{5, 27, 135}, YX{7, 37, 185}, XZ{5, 31, 155}; };
// n = 5 default since round 2 (DG_K4_ALT5, default 2): 16 threads per cell without the x-stage swap
// (coalesced x-line accesses), ZY and XZ conflict free, YX 1.5x (tools/k4_tp_layout_search.py 5 2 16 16 0)
template <> struct K4C<5, 2> { static constexpr int R = 2, CPB = 16, CPBS = 11, TP = 16, XSW = 0; static constexpr Lay3 ZY{5, 27, 135}, YX{5, 25, 125}, XZ{5, 25, 125}; };
// n = 3 alternate: 12 threads per cell (3 idle: they take block jobs) so that all three
// transposes are bank-conflict free (the unpadded y->x layout costs 2x; ncu: 25 % of the
// Chebyshev step's shared wavefronts were conflicts, LSU pipe 87 %)
template <> struct K4C<3, 1> { static constexpr int R = 1, CPB = 24, CPBS = 16, TP = 12, XSW = 0; static constexpr Lay3 ZY{3, 19, 57}, YX{4, 19, 57}, XZ{3, 9, 27}; };
template <int N> struct K4HasAlt { static constexpr bool value = N == 3 || N == 5 || N == 6 || N == 8; };

constexpr int imax(int a, int b) { return a > b ? a : b; }

template <int N, int NL, int ALT = 0, int MODE = KMODE_APPLY>
struct K4Layout {
  // the x->z layout is only used by point Jacobi and by the odd-n Chebyshev order
  static constexpr bool USE_XZ = MODE == KMODE_CHEBY_PJ || (N % 2 == 1 && MODE != KMODE_APPLY && MODE != KMODE_CHEBY_GLT);
  // K4_STAGE: Chebyshev streams staged in smem (b, u_{j-1}, and dinv unless FDM)
  static constexpr int NSTG = (K4_STAGE && MODE != KMODE_APPLY) ? (MODE == KMODE_CHEBY_FDM ? 2 : 3) : 0;
  static constexpr int R = K4C<N, ALT>::R, CPB = NSTG ? K4C<N, ALT>::CPBS : K4C<N, ALT>::CPB;
  static constexpr int NB = (N + R - 1) / R;          // thread rows per cell
  static constexpr int TPC = N * NB;                   // working threads per cell
  static constexpr int TPCP = K4C<N, ALT>::TP ? K4C<N, ALT>::TP : TPC;   // incl. idle padding
  static constexpr bool XSW = K4C<N, ALT>::XSW;       // x stage: line (j,k) = (b', a) instead of (a, b')
  static constexpr Lay3 ZY = K4C<N, ALT>::ZY, YX = K4C<N, ALT>::YX, XZ = K4C<N, ALT>::XZ;
  static constexpr int P = N | 1;                      // output staging row pitch
  static constexpr Lay3 OUT{P, N * P, N * N * P};
  // R1: T -> B -> (P^-1: z->y, x->z) -> output;  R2: A -> C -> (P^-1: x->z, y->x)
  static constexpr int S1 = imax(imax(imax(ZY.CS, YX.CS), OUT.CS), USE_XZ ? XZ.CS : 0);
  static constexpr int S2 = imax(imax(ZY.CS, YX.CS), USE_XZ ? XZ.CS : 0);
  static constexpr int PG = N | 1;                     // x-halo row pitch
  // y-ghost rows per cell, addr (f*NL + l)*GFS + k*GPG + i (tools/smem_gy_search.py for NL = 2)
  static constexpr int GPG = N;
  static constexpr int GFS = NL == 2 ? (N == 3 ? 22 : (N == 4 ? 20 : (N == 5 ? 37 : (N == 6 ? 38 : (N == 7 ? 55 : (N == 8 ? 72 : 89))))))
                                     : N * N + 2;
  static constexpr int GYC = 2 * NL * GFS + (N == 3 && NL == 2 ? 1 : 0);
  static constexpr int HS = NL * N * PG;               // one x-halo field [l][k][j]
  static constexpr int STGOFF = CPB * (S1 + S2 + GYC) + 2 * 2 * HS;   // staging [stream][cell][n^3]
  static constexpr int doubles() { return STGOFF + (STGOFF & 1) + NSTG * CPB * N * N * N; }
  static constexpr int bytes() { return doubles() * 8; }
};

__device__ __forceinline__ int at(const Lay3& L, int i, int j, int k) { return i + j * L.Pj + k * L.Pk; }

template <int N, int NL, int ALT, typename Real, int MODE>
constexpr int k4_min_blocks() {
  using L = K4Layout<N, NL, ALT, MODE>;
  constexpr int b = (227 * 1024) / (L::doubles() * (int)sizeof(Real));
  constexpr int t = 2048 / (L::CPB * L::TPCP);
  constexpr int m = b < t ? b : t;
  constexpr int cap = sizeof(Real) == 4 ? (N == 7 ? 3 : 5) : (N == 3 ? 4 : 3);   // measured (r1)
  return m < 1 ? 1 : (m > cap ? cap : m);
}

// L2 prefetch of a contiguous range (all threads of the block cooperate, one
// prefetch per 128-byte line).  Used to pull in the tile one plane up, which a block
// scheduled about one wave later will read.
template <typename T>
__device__ __forceinline__ void l2_prefetch(const T* p, int64_t count, int btid, int bt) {
  const char* c = reinterpret_cast<const char*>(p);
  const int64_t bytes = count * (int64_t)sizeof(T);
  for (int64_t o = (int64_t)btid * 128; o < bytes; o += (int64_t)bt * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
}

// L1 prefetch of a contiguous range (one prefetch per 128-byte line, block-cooperative)
template <typename T>
__device__ __forceinline__ void l1_prefetch(const T* p, int64_t count, int btid, int bt) {
  const char* c = reinterpret_cast<const char*>(p);
  const int64_t bytes = count * (int64_t)sizeof(T);
  for (int64_t o = (int64_t)btid * 128; o < bytes; o += (int64_t)bt * 128)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(c + o));
}

// M (even-odd) applied to N values read with a stride, written with a stride
template <int N, typename T>
__device__ __forceinline__ void mass_line(const T* __restrict__ M, const T* src, int ss, T* dst, int ds) {
  T v[N], o[N];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = src[k * ss];
  eo_apply<N, 1>(M, v, o);
#pragma unroll
  for (int k = 0; k < N; ++k) dst[k * ds] = o[k];
}

// KMODE_CHEBY_GLT: y = A s (+ A2 s2) + T^{-T} (N^- gm + N^+ gp), the neighbour term added in the
// even-odd domain before the recombination (KronParams::Ft packing: Fe, Fo, Fm); both sides
// cost n NL FMAs per line
template <int N, int NL, typename T>
__device__ __forceinline__ void face_eo(const T* __restrict__ F, const T (&gm)[NL], const T (&gp)[NL], int i,
                                        T& ye, T& yo) {
  constexpr int H = N / 2;
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    ye = fma(F[i * NL + l], gm[l] + gp[NL - 1 - l], ye);
    yo = fma(F[H * NL + i * NL + l], gm[l] - gp[NL - 1 - l], yo);
  }
}
template <int N, int NL, typename T>
__device__ __forceinline__ void face_mid(const T* __restrict__ F, const T (&gm)[NL], const T (&gp)[NL], T& ym) {
  constexpr int H = N / 2;
#pragma unroll
  for (int l = 0; l < NL; ++l) ym = fma(F[2 * H * NL + l], gm[l] + gp[NL - 1 - l], ym);
}
template <int N, int NL, typename T>
__device__ __forceinline__ void eo_mul_f(const T* __restrict__ A, const EOSplit<N, T>& s, const T* __restrict__ F,
                                         const T (&gm)[NL], const T (&gp)[NL], T (&y)[N]) {
  constexpr int H = N / 2;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T ye = T(0), yo = T(0);
    if (N & 1) ye = A[2 * H * H + i] * s.m;
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ye = fma(A[i * H + j], s.e[j], ye);
      yo = fma(A[H * H + i * H + j], s.o[j], yo);
    }
    face_eo<N, NL>(F, gm, gp, i, ye, yo);
    y[i] = ye + yo;
    y[N - 1 - i] = ye - yo;
  }
  if (N & 1) {
    const T* Rw = A + 2 * H * H + H;
    T ym = Rw[H] * s.m;
#pragma unroll
    for (int j = 0; j < H; ++j) ym = fma(Rw[j], s.e[j], ym);
    face_mid<N, NL>(F, gm, gp, ym);
    y[H] = ym;
  }
}
template <int N, int NL, typename T>
__device__ __forceinline__ void eo_mul2_f(const T* __restrict__ A1, const EOSplit<N, T>& s1,
                                          const T* __restrict__ A2, const EOSplit<N, T>& s2,
                                          const T* __restrict__ F, const T (&gm)[NL], const T (&gp)[NL],
                                          T (&y)[N]) {
  constexpr int H = N / 2;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T ye = T(0), yo = T(0);
    if (N & 1) ye = fma(A2[2 * H * H + i], s2.m, A1[2 * H * H + i] * s1.m);
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ye = fma(A1[i * H + j], s1.e[j], ye);
      yo = fma(A1[H * H + i * H + j], s1.o[j], yo);
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ye = fma(A2[i * H + j], s2.e[j], ye);
      yo = fma(A2[H * H + i * H + j], s2.o[j], yo);
    }
    face_eo<N, NL>(F, gm, gp, i, ye, yo);
    y[i] = ye + yo;
    y[N - 1 - i] = ye - yo;
  }
  if (N & 1) {
    const T* R1 = A1 + 2 * H * H + H;
    const T* R2 = A2 + 2 * H * H + H;
    T ym = fma(R2[H], s2.m, R1[H] * s1.m);
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ym = fma(R1[j], s1.e[j], ym);
      ym = fma(R2[j], s2.e[j], ym);
    }
    face_mid<N, NL>(F, gm, gp, ym);
    y[H] = ym;
  }
}

// P^{-1} building blocks of the fused Chebyshev step: GL-Jacobi (Eq. (12)) or FDM
template <int N, int MODE, typename KP, typename T>
__device__ __forceinline__ void pinv_pre(const KP& kp, const T (&v)[N], T (&o)[N]) {
  if constexpr (MODE == KMODE_CHEBY_FDM) fdm_fwd<N>(kp, v, o);
  else eo_apply<N, 1>(kp.TiT, v, o);
}
template <int N, int MODE, typename KP, typename T>
__device__ __forceinline__ void pinv_post(const KP& kp, const T (&v)[N], T (&o)[N]) {
  if constexpr (MODE == KMODE_CHEBY_FDM) fdm_bwd<N>(kp, v, o);
  else eo_apply<N, 1>(kp.Ti, v, o);
}
// middle-stage diagonal of P^{-1} on a line with fixed packed indices (a1, a2) in the
// other two directions (weights c1, c2) and running index m along direction d (weight cd)
template <int N, int MODE, typename KP, typename T>
__device__ __forceinline__ void pinv_diag(const KP& kp, const T* __restrict__ dinv, int stride, T c1, int a1,
                                          T c2, int a2, T cd, T (&o)[N]) {
  if constexpr (MODE == KMODE_CHEBY_FDM) {
    const T base = fma(c1, kp.lam[a1], c2 * kp.lam[a2]);
#pragma unroll
    for (int m = 0; m < N; ++m) o[m] /= fma(cd, kp.lam[m], base);
  } else {
#pragma unroll
    for (int m = 0; m < N; ++m) o[m] *= __ldg(dinv + m * stride);
  }
}

// cp.async (LDGSTS) of W doubles (W = 1: 8 bytes, W = 2: 16 bytes), completion per thread by
// cp.async.wait_all; used by K4_STAGE to stage the Chebyshev streams at block start
template <int WB>
__device__ __forceinline__ void cp_async_w(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if constexpr (WB == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else if constexpr (WB == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
}

// read of a staged (shared) or global stream
template <bool SMEM, typename T>
__device__ __forceinline__ T ldsrc(const T* p) {
  if constexpr (SMEM) return *p;
  else return __ldg(p);
}

template <typename Real> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

template <int N, int NL, int MODE, int OUTD, int ALT, typename Real>
__global__ void __launch_bounds__(K4Layout<N, NL, ALT, MODE>::CPB * K4Layout<N, NL, ALT, MODE>::TPCP,
                                  (k4_min_blocks<N, NL, ALT, Real, MODE>()))
k_kron4(const __grid_constant__ KronParamsT<Real> kp, const __grid_constant__ GridArgs g,
        const Real* __restrict__ u, Real* __restrict__ y, const __grid_constant__ ChebyArgsT<Real> ch) {
  using V2 = typename Vec2<Real>::type;
  using Lay = K4Layout<N, NL, ALT, MODE>;
  constexpr int R = Lay::R, NB = Lay::NB, TPC = Lay::TPC, CPB = Lay::CPB;
  constexpr int NN = N * N, N3 = N * NN;
  constexpr Lay3 LZY = Lay::ZY, LYX = Lay::YX, LXZ = Lay::XZ, LOUT = Lay::OUT;
  // R lines swept together (K4_RLINE): measured +2.5-3 % for the n = 4 Chebyshev step, -3..-5 %
  // at n = 5 (more live registers), n = 7 spills at its register cap; so n = 4 only
  // KMODE_CHEBY_GLT: the matvec stages use T^{-T}-premultiplied factors (kp.Mt, kp.Lt, kp.Ft)
  constexpr bool kT = MODE == KMODE_CHEBY_GLT;
  constexpr bool kRL = K4_RLINE && R > 1 && N == 4 && !kT;
  const Real* cM = kT ? kp.Mt : kp.M;
  constexpr int PG = Lay::PG, GPG = Lay::GPG, GFS = Lay::GFS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real* smem = reinterpret_cast<Real*>(smem_raw);
  Real* R1 = smem;
  Real* R2 = R1 + CPB * Lay::S1;
  Real* GYb = R2 + CPB * Lay::S2;
  Real* HX = GYb + CPB * Lay::GYC;   // [h][field: 0 = t, 1 = c][l][k][j]

  constexpr int TPCP = Lay::TPCP;
  constexpr bool XSW = Lay::XSW;
  // block (n, NB*CPB) unpadded; 1D (CPB*TPCP) when padded: tb >= NB is an idle padding
  // thread (jobs only)
  const int cslot = TPCP == TPC ? threadIdx.y / NB : threadIdx.x / TPCP;
  const int tb = TPCP == TPC ? threadIdx.y - cslot * NB : (threadIdx.x - cslot * TPCP) / N;
  const int ta = TPCP == TPC ? threadIdx.x : threadIdx.x - cslot * TPCP - tb * N;
  const int cx0 = blockIdx.x * CPB;
  const int cy = blockIdx.y;
  const int cz = g.zbeg + blockIdx.z;
  const int ncell = g.Nx - cx0 < CPB ? g.Nx - cx0 : CPB;
  const bool active = cslot < ncell && (TPCP == TPC || tb < NB);
  const int cx = cx0 + cslot;
  const int64_t plane = (int64_t)g.Nx * g.Ny;
  const int64_t rowcell = ((int64_t)cz * g.Ny + cy) * g.Nx;
  const int64_t cid = rowcell + cx;
  const Real* ucell = u + cid * N3;

  Real* GY = GYb + cslot * Lay::GYC;

  // x-neighbour sources of the block edges (halo cell index or -1)
  const bool xper = g.bc[0] == DG_BC_PERIODIC;
  int h0 = cx0 > 0 ? cx0 - 1 : (xper ? g.Nx - 1 : -1);
  int h1 = cx0 + ncell < g.Nx ? cx0 + ncell : (xper ? 0 : -1);
  if (ncell == g.Nx) h0 = h1 = -1;   // whole row in this block: periodic wrap stays inside
  const bool need_h0 = cslot == 0 && h0 >= 0;
  const bool need_h1 = cslot == ncell - 1 && h1 >= 0;
  // y-neighbour rows (-1: mirror)
  const bool yper = g.bc[1] == DG_BC_PERIODIC;
  const int ym_row = cy > 0 ? cy - 1 : (yper ? g.Ny - 1 : -1);
  const int yp_row = cy + 1 < g.Ny ? cy + 1 : (yper ? 0 : -1);

  // z-neighbour sources for this plane
  int zsrc[2];
  const Real* zbase[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int nz = cz + (s ? 1 : -1);
    if (nz >= 0 && nz < g.nz) {
      zsrc[s] = ZSRC_LOCAL;
      zbase[s] = ucell + (s ? plane * N3 : -plane * N3);
    } else {
      zsrc[s] = s ? g.zhi : g.zlo;
      zbase[s] = ucell + (s ? -(int64_t)(g.nz - 1) : (int64_t)(g.nz - 1)) * plane * N3;   // periodic wrap
      if constexpr (std::is_same<Real, double>::value) {   // fp32 meshes are single-slab
        if (zsrc[s] == ZSRC_HALO)
          zbase[s] = (s ? g.halo_hi : g.halo_lo) + ((int64_t)cy * g.Nx + cx) * (NL * NN) -
                     (s ? 0 : (N - NL) * NN);
      }
    }
  }

  // ================================================================ Z
  // Block-level job list (balanced over all threads of the block):
  //   [0, ncell*NYJ):  y-neighbour z-lines (cell, f, l, i) -> GY = (M_z u_{y+-})[k][j_l][i]
  //   then NL*N x-halo z-lines (l, j) per needed block edge -> HT[h][l][k][j]
  // Every job is "load a z-line (stride n^2), apply M_z, store with stride PG".
  constexpr int NYJ = 2 * NL * N;
  constexpr int BT = CPB * TPCP;
  const int btid = TPCP == TPC ? threadIdx.x + N * threadIdx.y : threadIdx.x;
  const int nyj = ncell * NYJ;
  const int nh0 = h0 >= 0 ? NL * N : 0, nh1 = h1 >= 0 ? NL * N : 0;
  const int njobs = nyj + nh0 + nh1;
  auto job_target = [&](int job, const Real*& src, Real*& dst, int& ds) {
    if (job < nyj) {
      const int c = job / NYJ, jj = job - c * NYJ;
      const int f = jj / (NL * N), l = (jj / N) % NL, i = jj % N;
      const int nrow = f ? yp_row : ym_row;
      if (nrow < 0) {   // mirror: from the own t in stage Y
        src = nullptr;
        return;
      }
      const int jl = f ? l : N - NL + l;
      src = u + (((int64_t)cz * g.Ny + nrow) * g.Nx + cx0 + c) * N3 + jl * N + i;
      dst = GYb + c * Lay::GYC + (f * NL + l) * GFS + i;
      ds = GPG;
    } else {
      const int hj = job - nyj;
      const int h = hj < nh0 ? 0 : 1;
      const int q = hj - (h ? nh0 : 0);
      const int l = q / N, j = q - l * N;
      const int il = h == 0 ? N - NL + l : l;
      src = u + (rowcell + (h ? h1 : h0)) * N3 + j * N + il;
      dst = HX + ((h * 2 + 0) * NL + l) * N * PG + j;
      ds = PG;
    }
  };
  // next plane's tile (same x-run and row) into L2: its block runs about one wave later
  // DG_L2PF=3: also pull this block's own tiles of the later Chebyshev streams into L2 now,
  // so that their loads (b in X, dinv and u_{j-1} in the P^{-1} stages) hit L2
  if (MODE != KMODE_APPLY && g.l2pf == 3) {
    const int64_t off = (rowcell + cx0) * N3, cnt = (int64_t)ncell * N3;
    l2_prefetch(ch.b + off, cnt, btid, BT);
    if (ch.dinv) l2_prefetch(ch.dinv + off, cnt, btid, BT);
    if (!ch.first) l2_prefetch(ch.u_prev + off, cnt, btid, BT);
  }
  if (g.l2pf && cz + 1 < g.zend) {
    const int64_t off = (rowcell + plane + cx0) * N3, cnt = (int64_t)ncell * N3;
    l2_prefetch(u + off, cnt, btid, BT);
    if (MODE != KMODE_APPLY && g.l2pf == 2) {
      l2_prefetch(ch.b + off, cnt, btid, BT);
      if (ch.dinv) l2_prefetch(ch.dinv + off, cnt, btid, BT);
      if (!ch.first) l2_prefetch(ch.u_prev + off, cnt, btid, BT);
    }
  }
  // K4_STAGE: stage the block's tiles of b, u_{j-1} (if read) and dinv in shared memory now;
  // they are consumed from the X stage on, long after this latency has passed
  constexpr bool kStage = Lay::NSTG > 0;
  Real* STG = smem + Lay::STGOFF + (Lay::STGOFF & 1);
  if constexpr (kStage) {
    constexpr int W = (N % 2 == 0) ? 2 : 1;                  // doubles per copy (16 / 8 bytes)
    constexpr int WB = W * (int)sizeof(Real);
    const int nchunk = ncell * N3 / W;
    const int64_t off = (rowcell + cx0) * N3;
    const Real* srcs[3] = {ch.b, ch.u_prev, ch.dinv};
#pragma unroll
    for (int st = 0; st < Lay::NSTG; ++st) {
      if (st == 1 && ch.first) continue;
      const Real* src = srcs[st] + off;
      Real* dst = STG + st * CPB * N3;
      for (int e = btid; e < nchunk; e += BT) cp_async_w<WB>(dst + e * W, src + e * W);
    }
  }
  auto sb = [&]() -> const Real* { return kStage ? STG + cslot * N3 : ch.b + cid * N3; };
  auto sp = [&]() -> const Real* { return kStage ? STG + (CPB + cslot) * N3 : ch.u_prev + cid * N3; };
  auto sd = [&]() -> const Real* { return kStage ? STG + (2 * CPB + cslot) * N3 : ch.dinv + cid * N3; };
  // the first job's loads are issued together with the own z-lines
  const Real* jsrc = nullptr;
  Real* jdst = nullptr;
  int jds = PG;
  Real jv[N];
  if (btid < njobs) job_target(btid, jsrc, jdst, jds);
  if (jsrc) {
#pragma unroll
    for (int k = 0; k < N; ++k) jv[k] = __ldg(jsrc + k * NN);
  }
  if (kRL && active) {
    // all R z-lines of the thread together: each coefficient of M_z, L_z loaded once
    Real uz[R][N], zm[R][NL], zp[R][NL];
    EOSplit<N, Real> su[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int zj = tb + r * NB;
      const bool ok = N % R == 0 || zj < N;
#pragma unroll
      for (int k = 0; k < N; ++k) uz[r][k] = ok ? __ldg(ucell + k * NN + zj * N + ta) : Real(0);
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int Lm = N - NL + l, Lp = l;
        zm[r][l] = zsrc[0] == ZSRC_MIRROR ? -uz[r][N - 1 - Lm]
                                           : (ok ? __ldg(zbase[0] + Lm * NN + zj * N + ta) : Real(0));
        zp[r][l] = zsrc[1] == ZSRC_MIRROR ? -uz[r][N - 1 - Lp]
                                           : (ok ? __ldg(zbase[1] + Lp * NN + zj * N + ta) : Real(0));
      }
      su[r] = eo_split<N>(uz[r]);
    }
    Real t[R][N], a[R][N];
    eo_mul_R<N, 1, false, R>(kp.M, su, t);
    eo_mul_R<N, 1, false, R>(kp.L[2], su, a);
    Real* T = R1 + cslot * LZY.CS;
    Real* A = R2 + cslot * LZY.CS;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int zj = tb + r * NB;
      if (N % R != 0 && zj >= N) break;
      dense_add<NL, NL>(kp.Nm[2], zm[r], &a[r][0]);
      dense_add<NL, NL>(kp.Np[2], zp[r], &a[r][N - NL]);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        T[at(LZY, ta, zj, k)] = t[r][k];
        A[at(LZY, ta, zj, k)] = a[r][k];
      }
    }
  } else if (active) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int zj = tb + r * NB;
      if (N % R != 0 && zj >= N) break;
      const int zi = ta;
      Real uz[N];
#pragma unroll
      for (int k = 0; k < N; ++k) uz[k] = __ldg(ucell + k * NN + zj * N + zi);
      Real zm[NL], zp[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int Lm = N - NL + l, Lp = l;
        zm[l] = zsrc[0] == ZSRC_MIRROR ? -uz[N - 1 - Lm] : __ldg(zbase[0] + Lm * NN + zj * N + zi);
        zp[l] = zsrc[1] == ZSRC_MIRROR ? -uz[N - 1 - Lp] : __ldg(zbase[1] + Lp * NN + zj * N + zi);
      }
      Real t[N], a[N];
      const auto su = eo_split<N>(uz);
      eo_mul<N, 1, false>(cM, su, t);
      if constexpr (kT) {
        eo_mul_f<N, NL>(kp.Lt[2], su, kp.Ft[2], zm, zp, a);
      } else {
        eo_mul<N, 1, false>(kp.L[2], su, a);
        dense_add<NL, NL>(kp.Nm[2], zm, &a[0]);
        dense_add<NL, NL>(kp.Np[2], zp, &a[N - NL]);
      }
      Real* T = R1 + cslot * LZY.CS;
      Real* A = R2 + cslot * LZY.CS;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        T[at(LZY, zi, zj, k)] = t[k];
        A[at(LZY, zi, zj, k)] = a[k];
      }
    }
  }
  if (jsrc) {
    Real o[N];
    eo_apply<N, 1>(cM, jv, o);
#pragma unroll
    for (int k = 0; k < N; ++k) jdst[k * jds] = o[k];
  }
#pragma unroll 1
  for (int job = btid + BT; job < njobs; job += BT) {
    const Real* src;
    Real* dst;
    int ds = PG;
    job_target(job, src, dst, ds);
    if (src) mass_line<N>(cM, src, NN, dst, ds);
  }
  __syncthreads();

  // ================================================================ Y
  const int64_t tile0 = (rowcell + cx0) * N3, tilecnt = (int64_t)ncell * N3;
  if constexpr ((k4_l1pf<N>() & 1) && MODE != KMODE_APPLY && !kStage) l1_prefetch(ch.b + tile0, tilecnt, btid, BT);
  {
    Real bl[R][N], cl[R][N];
    if (kRL && active) {
      const Real* T = R1 + cslot * LZY.CS;
      const Real* A = R2 + cslot * LZY.CS;
      EOSplit<N, Real> sa[R], st[R];
      Real gym[R][NL], gyp[R][NL];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int yk = (N % R == 0 || tb + r * NB < N) ? tb + r * NB : 0;   // a spare line recomputes k = 0
        Real al[N], tl[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          al[j] = A[at(LZY, ta, j, yk)];
          tl[j] = T[at(LZY, ta, j, yk)];
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          gym[r][l] = ym_row >= 0 ? GY[(0 * NL + l) * GFS + yk * GPG + ta] : -tl[NL - 1 - l];
          gyp[r][l] = yp_row >= 0 ? GY[(1 * NL + l) * GFS + yk * GPG + ta] : -tl[N - 1 - l];
        }
        sa[r] = eo_split<N>(al);
        st[r] = eo_split<N>(tl);
      }
      eo_mul2_R<N, 1, R>(kp.M, sa, kp.L[1], st, bl);
      eo_mul_R<N, 1, false, R>(kp.M, st, cl);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        dense_add<NL, NL>(kp.Nm[1], gym[r], &bl[r][0]);
        dense_add<NL, NL>(kp.Np[1], gyp[r], &bl[r][N - NL]);
      }
    } else if (active) {
      const Real* T = R1 + cslot * LZY.CS;
      const Real* A = R2 + cslot * LZY.CS;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int yk = tb + r * NB, yi = ta;
        if (N % R != 0 && yk >= N) break;
        Real al[N], tl[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          al[j] = A[at(LZY, yi, j, yk)];
          tl[j] = T[at(LZY, yi, j, yk)];
        }
        Real gym[NL], gyp[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          gym[l] = ym_row >= 0 ? GY[(0 * NL + l) * GFS + yk * GPG + yi] : -tl[NL - 1 - l];
          gyp[l] = yp_row >= 0 ? GY[(1 * NL + l) * GFS + yk * GPG + yi] : -tl[N - 1 - l];
        }
        const auto st = eo_split<N>(tl);
        if constexpr (kT) {
          eo_mul2_f<N, NL>(kp.Mt, eo_split<N>(al), kp.Lt[1], st, kp.Ft[1], gym, gyp, bl[r]);
          eo_mul<N, 1, false>(kp.Mt, st, cl[r]);
        } else {
          eo_mul2<N, 1>(kp.M, eo_split<N>(al), kp.L[1], st, bl[r]);
          eo_mul<N, 1, false>(kp.M, st, cl[r]);
          dense_add<NL, NL>(kp.Nm[1], gym, &bl[r][0]);
          dense_add<NL, NL>(kp.Np[1], gyp, &bl[r][N - NL]);
        }
      }
    }
    {   // halo jobs: HC[h][l][k][j] = M_y HT[h][l][k][:], spread over the block
      const int nh0 = h0 >= 0 ? NL * N : 0, nh1 = h1 >= 0 ? NL * N : 0;
      for (int job = btid; job < nh0 + nh1; job += BT) {
        const int h = job < nh0 ? 0 : 1;
        const int q = job - (h ? nh0 : 0);
        const int l = q / N, k = q - l * N;
        mass_line<N>(cM, HX + (((h * 2 + 0) * NL + l) * N + k) * PG, 1,
                     HX + (((h * 2 + 1) * NL + l) * N + k) * PG, 1);
      }
    }
    __syncthreads();   // all of T, A read: their regions take B, C
    if (active) {
      Real* Bf = R1 + cslot * LYX.CS;
      Real* Cf = R2 + cslot * LYX.CS;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int yk = tb + r * NB, yi = ta;
        if (N % R != 0 && yk >= N) break;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          Bf[at(LYX, yi, j, yk)] = bl[r][j];
          Cf[at(LYX, yi, j, yk)] = cl[r][j];
        }
      }
    }
  }
  // Chebyshev, n = 3, 7: scalar x-line loads of b issued ahead of the residual (measured
  // +3% / +0.4% at p = 2 / 6; n = 5 has no registers to spare, n = 9 spills: -0.8%)
  constexpr bool kPreBs = K4_PREB_ODD != 0 && MODE != KMODE_APPLY && (N == 3 || N == 7);
  Real bso[kPreBs ? R : 1][kPreBs ? N : 1];
  auto load_bso = [&]() {
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int xb = tb + r * NB;
        if (N % R != 0 && xb >= N) break;
        const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
        const Real* bb = sb() + (xk * N + xj) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) bso[r][i] = ldsrc<kStage>(bb + i);
      }
    }
  };
  if constexpr (kPreBs && K4_PREB_ODD == 2) load_bso();
  if constexpr (kStage) cp_async_commit_wait_all();   // own staged chunks landed; the barrier publishes them
  __syncthreads();
  if constexpr (kPreBs && K4_PREB_ODD == 1) load_bso();

  // ================================================================ X
  Real res[R][N];
  // Chebyshev, even n: issue the x-line loads of b before the stage's arithmetic
  constexpr bool kPreB = MODE != KMODE_APPLY && N % 2 == 0;
  V2 bpre[kPreB ? R : 1][kPreB ? N / 2 : 1];
  if constexpr (kPreB) {
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int xb = tb + r * NB;
        if (N % R != 0 && xb >= N) break;
        const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
        const Real* bb = sb() + (xk * N + xj) * N;
#pragma unroll
        for (int i = 0; i < N; i += 2) bpre[r][i / 2] = ldsrc<kStage>(reinterpret_cast<const V2*>(bb + i));
      }
    }
  }
  if (active) {
    const Real* Bf = R1 + cslot * LYX.CS;
    const Real* Cf = R2 + cslot * LYX.CS;
    // x-neighbour c source per side: 1 in-block slot offset, 2 halo, 0 mirror
    const bool inb_m = cslot > 0, inb_p = cslot + 1 < ncell;
    const bool wrap = xper && ncell == g.Nx;   // periodic row inside the block
    const int offm = inb_m ? -LYX.CS : (ncell - 1) * LYX.CS;
    const int offp = inb_p ? LYX.CS : -(ncell - 1) * LYX.CS;
    const bool slot_m = inb_m || wrap, slot_p = inb_p || wrap;
    if constexpr (kRL) {
      EOSplit<N, Real> sbl[R], scl[R];
      Real cxm[R][NL], cxp[R][NL];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int xb = (N % R == 0 || tb + r * NB < N) ? tb + r * NB : 0;   // spare line: recompute 0
        const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
        Real bl[N], cl[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          bl[i] = Bf[at(LYX, i, xj, xk)];
          cl[i] = Cf[at(LYX, i, xj, xk)];
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int Lm = N - NL + l, Lp = l;
          cxm[r][l] = slot_m ? Cf[offm + at(LYX, Lm, xj, xk)]
                             : (need_h0 ? HX[(((0 * 2 + 1) * NL + l) * N + xk) * PG + xj] : -cl[N - 1 - Lm]);
          cxp[r][l] = slot_p ? Cf[offp + at(LYX, Lp, xj, xk)]
                             : (need_h1 ? HX[(((1 * 2 + 1) * NL + l) * N + xk) * PG + xj] : -cl[N - 1 - Lp]);
        }
        sbl[r] = eo_split<N>(bl);
        scl[r] = eo_split<N>(cl);
      }
      eo_mul2_R<N, 1, R>(kp.M, sbl, kp.L[0], scl, res);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        dense_add<NL, NL>(kp.Nm[0], cxm[r], &res[r][0]);
        dense_add<NL, NL>(kp.Np[0], cxp[r], &res[r][N - NL]);
      }
    } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int xb = tb + r * NB;
      if (N % R != 0 && xb >= N) break;
      const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
      Real bl[N], cl[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        bl[i] = Bf[at(LYX, i, xj, xk)];
        cl[i] = Cf[at(LYX, i, xj, xk)];
      }
      Real cxm[NL], cxp[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int Lm = N - NL + l, Lp = l;
        cxm[l] = slot_m ? Cf[offm + at(LYX, Lm, xj, xk)]
                        : (need_h0 ? HX[(((0 * 2 + 1) * NL + l) * N + xk) * PG + xj] : -cl[N - 1 - Lm]);
        cxp[l] = slot_p ? Cf[offp + at(LYX, Lp, xj, xk)]
                        : (need_h1 ? HX[(((1 * 2 + 1) * NL + l) * N + xk) * PG + xj] : -cl[N - 1 - Lp]);
      }
      if constexpr (kT) {
        eo_mul2_f<N, NL>(kp.Mt, eo_split<N>(bl), kp.Lt[0], eo_split<N>(cl), kp.Ft[0], cxm, cxp, res[r]);
      } else {
        eo_mul2<N, 1>(kp.M, eo_split<N>(bl), kp.L[0], eo_split<N>(cl), res[r]);
        dense_add<NL, NL>(kp.Nm[0], cxm, &res[r][0]);
        dense_add<NL, NL>(kp.Np[0], cxp, &res[r][N - NL]);
      }
    }
    }
  }

  if constexpr (MODE == KMODE_APPLY && OUTD) {
    // direct stores along the x-lines (no staging barriers)
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int xb = tb + r * NB;
        if (N % R != 0 && xb >= N) break;
        const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
        Real* out = y + cid * N3 + (xk * N + xj) * N;
        if constexpr (N % 2 == 0) {
#pragma unroll
          for (int i = 0; i < N; i += 2)
            *reinterpret_cast<V2*>(out + i) = V2{res[r][i], res[r][i + 1]};
        } else {
#pragma unroll
          for (int i = 0; i < N; ++i) out[i] = res[r][i];
        }
      }
    }
    return;
  } else if constexpr (MODE == KMODE_APPLY) {
    __syncthreads();   // B, C fully read: R1 takes the output
    Real* O = R1 + cslot * LOUT.CS;
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int xb = tb + r * NB;
        if (N % R != 0 && xb >= N) break;
        const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
#pragma unroll
        for (int i = 0; i < N; ++i) O[at(LOUT, i, xj, xk)] = res[r][i];
      }
    }
    __syncthreads();
    if (active) {
      // element e = lt + q*TPC of the cell: i = ta, row (j + N k) = tb + q*NB
      Real* out = y + cid * N3;
#pragma unroll
      for (int q = 0; q < (NN + NB - 1) / NB; ++q) {
        const int rowi = tb + q * NB;
        if (NN % NB == 0 || rowi < NN) out[rowi * N + ta] = O[rowi * LOUT.Pj + ta];
      }
    }
    return;
  } else {
    // residual r = b - A u along the x-lines
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int xb = tb + r * NB;
        if (N % R != 0 && xb >= N) break;
        const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
        const Real* bb = sb() + (xk * N + xj) * N;
        if constexpr (kPreB) {
#pragma unroll
          for (int i = 0; i < N; i += 2) {
            const V2 bv = bpre[r][i / 2];
            res[r][i] = bv.x - res[r][i];
            res[r][i + 1] = bv.y - res[r][i + 1];
          }
        } else if constexpr (kPreBs) {
#pragma unroll
          for (int i = 0; i < N; ++i) res[r][i] = bso[r][i] - res[r][i];
        } else {
#pragma unroll
          for (int i = 0; i < N; ++i) res[r][i] = ldsrc<kStage>(bb + i) - res[r][i];
        }
      }
    }
    if constexpr (kT) {
      // transformed residual r~ = b~ - (T^{-T})^{(x)3} A u on the x-lines: P^{-1} r = (T^{-1})^{(x)3}
      // diag(A_GL)^{-1} r~ as x: diag, T^{-1}; y: T^{-1}; z: T^{-1} + the update of Eq. (11)
      Real dl[R][N];
      if (active) {   // the x-line diagonal, issued before the barrier
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          const Real* dv = ch.dinv + cid * N3 + (xk * N + xj) * N;
          if constexpr (N % 2 == 0) {
#pragma unroll
            for (int i = 0; i < N; i += 2) {
              const V2 d2 = __ldg(reinterpret_cast<const V2*>(dv + i));
              dl[r][i] = d2.x;
              dl[r][i + 1] = d2.y;
            }
          } else {
#pragma unroll
            for (int i = 0; i < N; ++i) dl[r][i] = __ldg(dv + i);
          }
        }
      }
      __syncthreads();   // B, C fully read (C also by the neighbour slots)
      if (active) {   // x: diag, T^{-1} -> R2 (x-write / y-read)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          Real v[N], o[N];
#pragma unroll
          for (int i = 0; i < N; ++i) v[i] = res[r][i] * dl[r][i];
          eo_apply<N, 1>(kp.Ti, v, o);
          Real* W = R2 + cslot * LYX.CS;
#pragma unroll
          for (int i = 0; i < N; ++i) W[at(LYX, i, xj, xk)] = o[i];
        }
      }
      __syncthreads();
      Real ujz[R][N], upz[R][N];   // the update's inputs along the z-lines, loaded one stage early
      if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int zj = tb + r * NB, zi = ta;
          if (N % R != 0 && zj >= N) break;
          const int64_t gbase = cid * N3 + zj * N + zi;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            ujz[r][k] = __ldg(u + gbase + k * NN);
            if (!ch.first) upz[r][k] = __ldg(ch.u_prev + gbase + k * NN);
          }
        }
      }
      if (active) {   // y: T^{-1} -> R1 (y-write / z-read)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int yk = tb + r * NB, yi = ta;
          if (N % R != 0 && yk >= N) break;
          const Real* Rd = R2 + cslot * LYX.CS;
          Real* W = R1 + cslot * LZY.CS;
          Real v[N], o[N];
#pragma unroll
          for (int j = 0; j < N; ++j) v[j] = Rd[at(LYX, yi, j, yk)];
          eo_apply<N, 1>(kp.Ti, v, o);
#pragma unroll
          for (int j = 0; j < N; ++j) W[at(LZY, yi, j, yk)] = o[j];
        }
      }
      __syncthreads();
      if (active) {   // z: T^{-1}, three-term update (Eq. (11)) along the z-lines
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int zj = tb + r * NB, zi = ta;
          if (N % R != 0 && zj >= N) break;
          const Real* Rd = R1 + cslot * LZY.CS;
          Real v[N], z[N];
#pragma unroll
          for (int k = 0; k < N; ++k) v[k] = Rd[at(LZY, zi, zj, k)];
          eo_apply<N, 1>(kp.Ti, v, z);
          const int64_t gbase = cid * N3 + zj * N + zi;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            Real vv = fma((Real)ch.c_z, z[k], ujz[r][k]);
            if (!ch.first) vv = fma((Real)ch.c_prev, ujz[r][k] - upz[r][k], vv);
            ch.u_next[gbase + k * NN] = vv;
          }
        }
      }
      return;
    }
    __syncthreads();   // B, C fully read (C also by the neighbour slots)
    if constexpr ((MODE == KMODE_CHEBY_GL || MODE == KMODE_CHEBY_FDM) && N % 2 == 0) {
      // even n: x: T^{-T}; y: T^{-T}; z: T^{-T}, diag (coalesced z-lines), T^{-1}; y: T^{-1};
      // x: T^{-1} + update along the x-lines with 128-bit accesses
      if constexpr ((k4_l1pf<N>() & 2) && MODE == KMODE_CHEBY_GL && !kStage) l1_prefetch(ch.dinv + tile0, tilecnt, btid, BT);
      if (active) {   // x: T^{-T} -> R2 (x-write / y-read)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          Real o[N];
          pinv_pre<N, MODE>(kp, res[r], o);
          Real* W = R2 + cslot * LYX.CS;
#pragma unroll
          for (int i = 0; i < N; ++i) W[at(LYX, i, xj, xk)] = o[i];
        }
      }
      __syncthreads();
      Real dpre[MODE == KMODE_CHEBY_GL ? R : 1][MODE == KMODE_CHEBY_GL ? N : 1];
      if constexpr (MODE == KMODE_CHEBY_GL) {   // the next stage's diagonal, loaded one stage early
        if (active) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int zj = tb + r * NB, zi = ta;
            if (N % R != 0 && zj >= N) break;
            const Real* dv = sd() + zj * N + zi;
#pragma unroll
            for (int k = 0; k < N; ++k) dpre[r][k] = ldsrc<kStage>(dv + k * NN);
          }
        }
      }
      if constexpr ((k4_l1pf<N>() & 4) && !kStage) {
        l1_prefetch(u + tile0, tilecnt, btid, BT);
        if (!ch.first) l1_prefetch(ch.u_prev + tile0, tilecnt, btid, BT);
      }
      if (active) {   // y: T^{-T} -> R1 (y-write / z-read)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int yk = tb + r * NB, yi = ta;
          if (N % R != 0 && yk >= N) break;
          const Real* Rd = R2 + cslot * LYX.CS;
          Real* W = R1 + cslot * LZY.CS;
          Real v[N], o[N];
#pragma unroll
          for (int j = 0; j < N; ++j) v[j] = Rd[at(LYX, yi, j, yk)];
          pinv_pre<N, MODE>(kp, v, o);
#pragma unroll
          for (int j = 0; j < N; ++j) W[at(LZY, yi, j, yk)] = o[j];
        }
      }
      __syncthreads();
      if (active) {   // z: T^{-T}, diag(A_GL)^{-1}, T^{-1} -> R2 (z-write / y-read)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int zj = tb + r * NB, zi = ta;
          if (N % R != 0 && zj >= N) break;
          const Real* Rd = R1 + cslot * LZY.CS;
          Real* W = R2 + cslot * LZY.CS;
          Real v[N], o[N];
#pragma unroll
          for (int k = 0; k < N; ++k) v[k] = Rd[at(LZY, zi, zj, k)];
          pinv_pre<N, MODE>(kp, v, o);
          if constexpr (MODE == KMODE_CHEBY_GL) {
#pragma unroll
            for (int k = 0; k < N; ++k) o[k] *= dpre[r][k];
          } else {
            pinv_diag<N, MODE>(kp, ch.dinv + cid * N3 + zj * N + zi, NN, kp.cdir[0], zi, kp.cdir[1], zj,
                               kp.cdir[2], o);
          }
          pinv_post<N, MODE>(kp, o, v);
#pragma unroll
          for (int k = 0; k < N; ++k) W[at(LZY, zi, zj, k)] = v[k];
        }
      }
      __syncthreads();
      V2 ujpre[R][N / 2], uppre[R][N / 2];   // the update's inputs, loaded one stage early
      if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          const int64_t gb = cid * N3 + (xk * N + xj) * N;
#pragma unroll
          for (int i = 0; i < N; i += 2) {
            ujpre[r][i / 2] = __ldg(reinterpret_cast<const V2*>(u + gb + i));
            if (!ch.first) uppre[r][i / 2] = *reinterpret_cast<const V2*>(sp() + (gb - cid * N3) + i);
          }
        }
      }
      if (active) {   // y: T^{-1} -> R1 (y-write / x-read)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int yk = tb + r * NB, yi = ta;
          if (N % R != 0 && yk >= N) break;
          const Real* Rd = R2 + cslot * LZY.CS;
          Real* W = R1 + cslot * LYX.CS;
          Real v[N], o[N];
#pragma unroll
          for (int j = 0; j < N; ++j) v[j] = Rd[at(LZY, yi, j, yk)];
          pinv_post<N, MODE>(kp, v, o);
#pragma unroll
          for (int j = 0; j < N; ++j) W[at(LYX, yi, j, yk)] = o[j];
        }
      }
      __syncthreads();
      if (active) {   // x: T^{-1}, three-term update (Eq. (11)) along the x-lines
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          const Real* Rd = R1 + cslot * LYX.CS;
          Real v[N], z[N];
#pragma unroll
          for (int i = 0; i < N; ++i) v[i] = Rd[at(LYX, i, xj, xk)];
          pinv_post<N, MODE>(kp, v, z);
          const int64_t gb = cid * N3 + (xk * N + xj) * N;
#pragma unroll
          for (int i = 0; i < N; i += 2) {
            const V2 uj = ujpre[r][i / 2];
            V2 o;
            o.x = fma((Real)ch.c_z, z[i], uj.x);
            o.y = fma((Real)ch.c_z, z[i + 1], uj.y);
            if (!ch.first) {
              const V2 up = uppre[r][i / 2];
              o.x = fma((Real)ch.c_prev, uj.x - up.x, o.x);
              o.y = fma((Real)ch.c_prev, uj.y - up.y, o.y);
            }
            *reinterpret_cast<V2*>(ch.u_next + gb + i) = o;
          }
        }
      }
      return;
    } else if constexpr (MODE == KMODE_CHEBY_GL || MODE == KMODE_CHEBY_FDM) {
      Real* X2 = R2 + cslot * LXZ.CS;
      Real* Z1 = R1 + cslot * LZY.CS;
      Real* Y2 = R2 + cslot * LYX.CS;
      Real* X1 = R1 + cslot * LXZ.CS;
      if constexpr ((k4_l1pf<N>() & 2) && MODE == KMODE_CHEBY_GL && !kStage) l1_prefetch(ch.dinv + tile0, tilecnt, btid, BT);
      if (active) {   // x: T^{-T}
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          Real o[N];
          pinv_pre<N, MODE>(kp, res[r], o);
#pragma unroll
          for (int i = 0; i < N; ++i) X2[at(LXZ, i, xj, xk)] = o[i];
        }
      }
      __syncthreads();
      Real dpre[MODE == KMODE_CHEBY_GL ? R : 1][MODE == KMODE_CHEBY_GL ? N : 1];
      if constexpr (MODE == KMODE_CHEBY_GL) {   // the y stage's diagonal, loaded one stage early
        if (active) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int yk = tb + r * NB, yi = ta;
            if (N % R != 0 && yk >= N) break;
            const Real* dv = sd() + yk * NN + yi;
#pragma unroll
            for (int j = 0; j < N; ++j) dpre[r][j] = ldsrc<kStage>(dv + j * N);
          }
        }
      }
      if constexpr ((k4_l1pf<N>() & 4) && !kStage) {
        l1_prefetch(u + tile0, tilecnt, btid, BT);
        if (!ch.first) l1_prefetch(ch.u_prev + tile0, tilecnt, btid, BT);
      }
      if (active) {   // z: T^{-T}
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int zj = tb + r * NB, zi = ta;
          if (N % R != 0 && zj >= N) break;
          Real v[N], o[N];
#pragma unroll
          for (int k = 0; k < N; ++k) v[k] = X2[at(LXZ, zi, zj, k)];
          pinv_pre<N, MODE>(kp, v, o);
#pragma unroll
          for (int k = 0; k < N; ++k) Z1[at(LZY, zi, zj, k)] = o[k];
        }
      }
      __syncthreads();
      if (active) {   // y: T^{-T}, diag(A_GL)^{-1}, T^{-1}
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int yk = tb + r * NB, yi = ta;
          if (N % R != 0 && yk >= N) break;
          Real v[N], o[N];
#pragma unroll
          for (int j = 0; j < N; ++j) v[j] = Z1[at(LZY, yi, j, yk)];
          pinv_pre<N, MODE>(kp, v, o);
          if constexpr (MODE == KMODE_CHEBY_GL) {
#pragma unroll
            for (int j = 0; j < N; ++j) o[j] *= dpre[r][j];
          } else {
            pinv_diag<N, MODE>(kp, ch.dinv + cid * N3 + yk * NN + yi, N, kp.cdir[0], yi, kp.cdir[2], yk,
                               kp.cdir[1], o);
          }
          pinv_post<N, MODE>(kp, o, v);
#pragma unroll
          for (int j = 0; j < N; ++j) Y2[at(LYX, yi, j, yk)] = v[j];
        }
      }
      __syncthreads();
      Real ujz[R][N], upz[R][N];   // the update's inputs along the z-lines, loaded one stage early
      if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int zj = tb + r * NB, zi = ta;
          if (N % R != 0 && zj >= N) break;
          const int64_t gbase = cid * N3 + zj * N + zi;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            ujz[r][k] = __ldg(u + gbase + k * NN);
            if (!ch.first) upz[r][k] = sp()[gbase - cid * N3 + k * NN];
          }
        }
      }
      if (active) {   // x: T^{-1}
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          Real v[N], o[N];
#pragma unroll
          for (int i = 0; i < N; ++i) v[i] = Y2[at(LYX, i, xj, xk)];
          pinv_post<N, MODE>(kp, v, o);
#pragma unroll
          for (int i = 0; i < N; ++i) X1[at(LXZ, i, xj, xk)] = o[i];
        }
      }
      __syncthreads();
      if (active) {   // z: T^{-1} -> res along the z-lines
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int zj = tb + r * NB, zi = ta;
          if (N % R != 0 && zj >= N) break;
          Real v[N];
#pragma unroll
          for (int k = 0; k < N; ++k) v[k] = X1[at(LXZ, zi, zj, k)];
          pinv_post<N, MODE>(kp, v, res[r]);
          // three-term update, Eq. (11)
          const int64_t gbase = cid * N3 + zj * N + zi;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            Real vv = fma((Real)ch.c_z, res[r][k], ujz[r][k]);
            if (!ch.first) vv = fma((Real)ch.c_prev, ujz[r][k] - upz[r][k], vv);
            ch.u_next[gbase + k * NN] = vv;
          }
        }
      }
      return;
    } else {
      // point Jacobi: diagonal along the x-lines, then to z-lines through smem
      Real* X1 = R1 + cslot * LXZ.CS;
      if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int xb = tb + r * NB;
          if (N % R != 0 && xb >= N) break;
          const int xj = XSW ? xb : ta, xk = XSW ? ta : xb;
          const Real* dv = sd() + (xk * N + xj) * N;
#pragma unroll
          for (int i = 0; i < N; ++i) X1[at(LXZ, i, xj, xk)] = res[r][i] * ldsrc<kStage>(dv + i);
        }
      }
      __syncthreads();
      if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int zj = tb + r * NB, zi = ta;
          if (N % R != 0 && zj >= N) break;
#pragma unroll
          for (int k = 0; k < N; ++k) res[r][k] = X1[at(LXZ, zi, zj, k)];
        }
      }
    }
    // three-term update, Eq. (11), along the z-lines
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int zj = tb + r * NB, zi = ta;
        if (N % R != 0 && zj >= N) break;
        const int64_t gbase = cid * N3 + zj * N + zi;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int64_t gi = gbase + k * NN;
          const Real uj = __ldg(u + gi);   // re-read (L1/L2): saves R*N live registers
          Real v = fma((Real)ch.c_z, res[r][k], uj);
          if (!ch.first) v = fma((Real)ch.c_prev, uj - sp()[gi - cid * N3], v);
          ch.u_next[gi] = v;
        }
      }
    }
  }
}

template <int N, int NL, int MODE, int OUTD, int ALT, typename Real>
cudaError_t launch_t(const KronParamsT<Real>& kp, const GridArgs& g, const Real* u, Real* y,
                     const ChebyArgsT<Real>& ch, cudaStream_t s) {
  using Lay = K4Layout<N, NL, ALT, MODE>;
  const int planes = g.zend - g.zbeg;
  if (planes <= 0 || g.Nx <= 0 || g.Ny <= 0) return cudaSuccess;
  if (g.Ny > 65535 || planes > 65535) return cudaErrorInvalidValue;
  const dim3 grid((g.Nx + Lay::CPB - 1) / Lay::CPB, g.Ny, planes);
  const dim3 block = Lay::TPCP == Lay::TPC ? dim3(N, Lay::NB * Lay::CPB) : dim3(Lay::CPB * Lay::TPCP);
  const size_t smem = (size_t)Lay::doubles() * sizeof(Real);
  auto kern = k_kron4<N, NL, MODE, OUTD, ALT, Real>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, block, smem, s>>>(kp, g, u, y, ch);
  return cudaGetLastError();
}

// KMODE_CHEBY_GLT exists for fp64 and NL = 2 only (KronParams::Ft is packed for NL = 2)
template <int N, int NL, int OUTD, int ALT, typename Real>
cudaError_t launch_glt(const KronParamsT<Real>& kp, const GridArgs& g, const Real* u, Real* y,
                       const ChebyArgsT<Real>& ch, cudaStream_t s) {
  if constexpr (std::is_same<Real, double>::value && NL == 2)
    return launch_t<N, NL, KMODE_CHEBY_GLT, OUTD, ALT, Real>(kp, g, u, y, ch, s);
  return cudaErrorInvalidValue;
}

template <int N, int NL, typename Real>
cudaError_t launch_mode(int mode, const KronParamsT<Real>& kp, const GridArgs& g, const Real* u, Real* y,
                        const ChebyArgsT<Real>& ch, cudaStream_t s) {
  static const int outd = [] {   // DG_K4_OUT=0: smem-staged coalesced stores (comparison)
    const char* e = std::getenv("DG_K4_OUT");
    return e ? std::atoi(e) : (N % 2 == 0 ? 1 : 0);   // measured: direct wins for even n only
  }();
  static const int alt_mask = [] {   // DG_K4_ALT: bit n-3 selects the alternate configuration
    const char* e = std::getenv("DG_K4_ALT");
    return e ? std::atoi(e) : 0;
  }();
  if constexpr (N == 5) {   // default: the unswapped padded configuration K4C<5, 2> (DG_K4_ALT5=0: K4C<5>)
    static const int alt5 = [] {
      const char* e = std::getenv("DG_K4_ALT5");
      return e ? std::atoi(e) : 2;   // measured (C4 p=4): matvec 120 -> 132, Chebyshev step 75.6 -> 81.1 GDoF/s
    }();
    if (alt5 == 2) {
      switch (mode) {
        case KMODE_APPLY: return launch_t<N, NL, KMODE_APPLY, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GL: return launch_t<N, NL, KMODE_CHEBY_GL, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_PJ: return launch_t<N, NL, KMODE_CHEBY_PJ, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_FDM: return launch_t<N, NL, KMODE_CHEBY_FDM, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GLT: return launch_glt<N, NL, 0, 2, Real>(kp, g, u, y, ch, s);
      }
      return cudaErrorInvalidValue;
    }
  }
  if constexpr (N == 7) {   // default: the padded configuration K4C<7, 2> (DG_K4_ALT7=0: K4C<7>)
    static const int alt7 = [] {
      const char* e = std::getenv("DG_K4_ALT7");
      return e ? std::atoi(e) : 2;   // measured (C4 p=6): matvec 118.6 -> 125.9, Chebyshev 72.2 -> 74.6 GDoF/s
    }();
    if (alt7 == 2) {
      switch (mode) {
        case KMODE_APPLY: return launch_t<N, NL, KMODE_APPLY, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GL: return launch_t<N, NL, KMODE_CHEBY_GL, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_PJ: return launch_t<N, NL, KMODE_CHEBY_PJ, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_FDM: return launch_t<N, NL, KMODE_CHEBY_FDM, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GLT: return launch_glt<N, NL, 0, 2, Real>(kp, g, u, y, ch, s);
      }
      return cudaErrorInvalidValue;
    }
  }
  if constexpr (N == 9) {   // DG_K4_ALT9=2: the padded-YX alternate K4C<9, 2> (A/B)
    static const int alt9 = [] {
      const char* e = std::getenv("DG_K4_ALT9");
      return e ? std::atoi(e) : 0;
    }();
    if (alt9 == 2) {
      switch (mode) {
        case KMODE_APPLY: return launch_t<N, NL, KMODE_APPLY, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GL: return launch_t<N, NL, KMODE_CHEBY_GL, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_PJ: return launch_t<N, NL, KMODE_CHEBY_PJ, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_FDM: return launch_t<N, NL, KMODE_CHEBY_FDM, 0, 2, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GLT: return launch_glt<N, NL, 0, 2, Real>(kp, g, u, y, ch, s);
      }
      return cudaErrorInvalidValue;
    }
  }
  if constexpr (K4HasAlt<N>::value) {
    if ((alt_mask >> (N - 3)) & 1) {
      switch (mode) {
        case KMODE_APPLY:
          return outd ? launch_t<N, NL, KMODE_APPLY, 1, 1, Real>(kp, g, u, y, ch, s)
                      : launch_t<N, NL, KMODE_APPLY, 0, 1, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GL: return launch_t<N, NL, KMODE_CHEBY_GL, 0, 1, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_PJ: return launch_t<N, NL, KMODE_CHEBY_PJ, 0, 1, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_FDM: return launch_t<N, NL, KMODE_CHEBY_FDM, 0, 1, Real>(kp, g, u, y, ch, s);
        case KMODE_CHEBY_GLT: return launch_glt<N, NL, 0, 1, Real>(kp, g, u, y, ch, s);
      }
      return cudaErrorInvalidValue;
    }
  }
  switch (mode) {
    case KMODE_APPLY:
      return outd ? launch_t<N, NL, KMODE_APPLY, 1, 0, Real>(kp, g, u, y, ch, s)
                  : launch_t<N, NL, KMODE_APPLY, 0, 0, Real>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_GL: return launch_t<N, NL, KMODE_CHEBY_GL, 0, 0, Real>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_PJ: return launch_t<N, NL, KMODE_CHEBY_PJ, 0, 0, Real>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_FDM: return launch_t<N, NL, KMODE_CHEBY_FDM, 0, 0, Real>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_GLT: return launch_glt<N, NL, 0, 0, Real>(kp, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

template <int N, typename Real>
cudaError_t launch_nl(int NL, int mode, const KronParamsT<Real>& kp, const GridArgs& g, const Real* u, Real* y,
                      const ChebyArgsT<Real>& ch, cudaStream_t s) {
  if (NL == 2 && N > 2) return launch_mode<N, 2, Real>(mode, kp, g, u, y, ch, s);
  if (NL == N) return launch_mode<N, N, Real>(mode, kp, g, u, y, ch, s);
  return cudaErrorInvalidValue;
}

// Basis change v_K = (B (x) B (x) B) u_K per cell (Eq. (12)) in the same
// z-first thread mapping and transposition layouts as k_kron4: z-lines straight from HBM
// (coalesced), z -> y -> x transposes through two smem fields, output along the x-lines
// (128-bit stores for even n, smem-staged coalesced stores for odd n).  HBM-bound, 16 B/DoF.
template <int N>
__global__ void __launch_bounds__(K4Layout<N, 2>::CPB * K4Layout<N, 2>::TPC)
k_bchg4(const __grid_constant__ BchgParams bp, const double* __restrict__ in, double* __restrict__ out,
        int64_t ncells) {
  using Lay = K4Layout<N, 2>;
  constexpr int R = Lay::R, NB = Lay::NB, CPB = Lay::CPB;
  constexpr int NN = N * N, N3 = N * NN;
  constexpr Lay3 LZY = Lay::ZY, LYX = Lay::YX, LOUT = Lay::OUT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* R1 = reinterpret_cast<double*>(smem_raw);
  double* R2 = R1 + CPB * Lay::S1;
  const int ta = threadIdx.x, cslot = threadIdx.y / NB, tb = threadIdx.y - cslot * NB;
  const int64_t cell0 = (int64_t)blockIdx.x * CPB;
  const int ncell = (int)(ncells - cell0 < CPB ? ncells - cell0 : CPB);
  const bool active = cslot < ncell;
  const int64_t cid = cell0 + cslot;
  if (active) {   // z
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int zj = tb + r * NB, zi = ta;
      if (N % R != 0 && zj >= N) break;
      double v[N], o[N];
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = __ldg(in + cid * N3 + k * NN + zj * N + zi);
      eo_apply<N, 1>(bp.B, v, o);
      double* W = R1 + cslot * LZY.CS;
#pragma unroll
      for (int k = 0; k < N; ++k) W[at(LZY, zi, zj, k)] = o[k];
    }
  }
  __syncthreads();
  if (active) {   // y
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int yk = tb + r * NB, yi = ta;
      if (N % R != 0 && yk >= N) break;
      double v[N], o[N];
      const double* Rd = R1 + cslot * LZY.CS;
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = Rd[at(LZY, yi, j, yk)];
      eo_apply<N, 1>(bp.B, v, o);
      double* W = R2 + cslot * LYX.CS;
#pragma unroll
      for (int j = 0; j < N; ++j) W[at(LYX, yi, j, yk)] = o[j];
    }
  }
  __syncthreads();
  double res[R][N];
  if (active) {   // x
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int xk = tb + r * NB, xj = ta;
      if (N % R != 0 && xk >= N) break;
      double v[N];
      const double* Rd = R2 + cslot * LYX.CS;
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = Rd[at(LYX, i, xj, xk)];
      eo_apply<N, 1>(bp.B, v, res[r]);
      if constexpr (N % 2 == 0) {
        double* o = out + cid * N3 + (xk * N + xj) * N;
#pragma unroll
        for (int i = 0; i < N; i += 2) *reinterpret_cast<double2*>(o + i) = make_double2(res[r][i], res[r][i + 1]);
      }
    }
  }
  if constexpr (N % 2 == 1) {   // stage in R1 (free since the y stage) for coalesced stores
    double* O = R1 + cslot * LOUT.CS;
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int xk = tb + r * NB, xj = ta;
        if (N % R != 0 && xk >= N) break;
#pragma unroll
        for (int i = 0; i < N; ++i) O[at(LOUT, i, xj, xk)] = res[r][i];
      }
    }
    __syncthreads();
    if (active) {
      double* o = out + cid * N3;
#pragma unroll
      for (int q = 0; q < (NN + NB - 1) / NB; ++q) {
        const int rowi = tb + q * NB;
        if (NN % NB == 0 || rowi < NN) o[rowi * N + ta] = O[rowi * LOUT.Pj + ta];
      }
    }
  }
}

template <int N>
cudaError_t launch_bchg4_n(const BchgParams& bp, const double* in, double* out, int64_t ncells, cudaStream_t s) {
  using Lay = K4Layout<N, 2>;
  if (ncells <= 0) return cudaSuccess;
  const size_t smem = (size_t)Lay::CPB * (Lay::S1 + Lay::S2) * sizeof(double);
  auto kern = k_bchg4<N>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)((ncells + Lay::CPB - 1) / Lay::CPB), dim3(N, Lay::NB * Lay::CPB), smem, s>>>(bp, in, out, ncells);
  return cudaGetLastError();
}

}  // namespace

// n in 3..9 (p = 2..8); p = 1 uses the general quadrature kernel k_quad
bool kron4_supported(int n) { return n >= 3 && n <= 9; }

template <typename Real>
cudaError_t launch_kron4_t(int n, int NL, int mode, const KronParamsT<Real>& kp, const GridArgs& g, const Real* u,
                           Real* y, const ChebyArgsT<Real>& ch, cudaStream_t s) {
  switch (n) {
    case 3: return launch_nl<3, Real>(NL, mode, kp, g, u, y, ch, s);
    case 4: return launch_nl<4, Real>(NL, mode, kp, g, u, y, ch, s);
    case 5: return launch_nl<5, Real>(NL, mode, kp, g, u, y, ch, s);
    case 6: return launch_nl<6, Real>(NL, mode, kp, g, u, y, ch, s);
    case 7: return launch_nl<7, Real>(NL, mode, kp, g, u, y, ch, s);
    case 8: return launch_nl<8, Real>(NL, mode, kp, g, u, y, ch, s);
    case 9: return launch_nl<9, Real>(NL, mode, kp, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_kron4(int n, int NL, int mode, const KronParams& kp, const GridArgs& g,
                         const double* u, double* y, const ChebyArgs& ch, cudaStream_t s) {
  return launch_kron4_t<double>(n, NL, mode, kp, g, u, y, ch, s);
}

cudaError_t launch_kron4_f32(int n, int NL, int mode, const KronParamsF& kp, const GridArgs& g,
                             const float* u, float* y, const ChebyArgsF& ch, cudaStream_t s) {
  return launch_kron4_t<float>(n, NL, mode, kp, g, u, y, ch, s);
}

}  // namespace dgb

namespace dgb {
cudaError_t launch_basis_change4(int n, const BchgParams& bp, const double* in, double* out, int64_t ncells,
                                 cudaStream_t s) {
  switch (n) {
    case 3: return launch_bchg4_n<3>(bp, in, out, ncells, s);
    case 4: return launch_bchg4_n<4>(bp, in, out, ncells, s);
    case 5: return launch_bchg4_n<5>(bp, in, out, ncells, s);
    case 6: return launch_bchg4_n<6>(bp, in, out, ncells, s);
    case 7: return launch_bchg4_n<7>(bp, in, out, ncells, s);
    case 8: return launch_bchg4_n<8>(bp, in, out, ncells, s);
    case 9: return launch_bchg4_n<9>(bp, in, out, ncells, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace dgb
