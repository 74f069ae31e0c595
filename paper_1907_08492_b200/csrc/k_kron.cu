// Cartesian fast path of the SIPG operator: the element-centric kernel in the
// reference-coordinate Kronecker form (PAPER.md:336-344 mentions it; Eq. (14),
// PAPER.md:2137-2145 states it).
//
// On a Cartesian cell the quadrature operator of Eq. (1) equals exactly
//   y_K = sum_d (Mhat (x) Mhat (x) L_d) u_K + sum_{faces} (Mhat (x) Mhat) (x) N^{+-}_d u_{K+-}
// with Mhat the 1D mass, L_d = (V/h_d^2) Lhat the 1D interior-cell SIPG block and
// N^{+-} the 1D couplings to the neighbour.  For the Hermite-like basis N^{+-}
// touches only the NL = 2 neighbour layers nearest the face (value + derivative,
// PAPER.md:753-762); for the nodal GL basis it touches all NL = n layers.
// Mirror Dirichlet faces use a ghost neighbour = -(own cell reflected across the
// face): its trace is -u and its normal derivative +du/dn.
//
// Schedule per cell (7 even-odd line sweeps, register-resident lines, smem
// transposes between directions; one thread per line, n^2 threads per cell):
//   x-lines:  t = M u,           a = L_x u + N_x^{+-} u_{x+-}
//             (extra) M_x on the y- and z-neighbour layers
//   y-lines:  b = M a + L_y t + N_y^{+-} (M_x u_{y+-}),   c = M t
//             (extra) M_y on the z-neighbour layers
//   z-lines:  y = M b + L_z c + N_z^{+-} (M_y M_x u_{z+-})      -> one coalesced write
// The fused Chebyshev step ("merged") continues on the
// z-lines in registers: r = b - y, P^{-1} r by 6 more sweeps (T^{-T} in z,y,x;
// diagonal; T^{-1} in x,y,z; Eq. (12)), then the three-term update of Eq. (11).
#include <cuda_runtime.h>

#include "common.cuh"
#include "dg_internal.h"
#include "loader.cuh"

namespace dgb {
namespace {

template <int N, int NL>
struct KLayout {
  static constexpr int P = N | 1;                // odd pitch: conflict-free x-lines
  static constexpr int FIELD = N * N * P;        // one n^3 field
  static constexpr int FACE = NL * N * P;        // NL layers of one face, rows (l,b)
  static constexpr int PER_CELL = 3 * FIELD + 6 * FACE;
};

template <int N>
__device__ __forceinline__ int64_t cell_off(int64_t c) { return c * (int64_t)(N * N * N); }

template <int N, int NL, int CPB, int MODE>
__global__ void __launch_bounds__(CPB * N * N)
k_kron(const __grid_constant__ KronParams kp, const __grid_constant__ GridArgs g,
       const double* __restrict__ u, double* __restrict__ y, const __grid_constant__ ChebyArgs ch) {
  using Lay = KLayout<N, NL>;
  constexpr int P = Lay::P;
  constexpr int NN = N * N;
  extern __shared__ double smem[];

  const int plane = g.Nx * g.Ny;
  const int64_t cbeg = (int64_t)g.zbeg * plane;
  const int64_t cend = (int64_t)g.zend * plane;
  const int64_t cell0 = cbeg + (int64_t)blockIdx.x * CPB;
  const int ncell = (int)(cend - cell0 < CPB ? cend - cell0 : CPB);
  const int tid = threadIdx.x;

  // ---------------------------------------------------------------- P0: loads
  const int cslot = tid / NN;
  const int line = tid % NN;
  const bool active = cslot < ncell;
  double* F0 = smem + cslot * Lay::PER_CELL;        // u, later b / residual
  double* F1 = F0 + Lay::FIELD;                      // t, later c
  double* F2 = F1 + Lay::FIELD;                      // a
  double* FC = F2 + Lay::FIELD;                      // 6 faces
  if (active) stage_cell<N, NL, P, Lay::FACE>(g, u, cell0 + cslot, line, F0, FC);
  __syncthreads();

  // ---------------------------------------------------------------- P1: x-lines
  if (active) {
    const int j = line % N, k = line / N;
    double x[N], t[N], a[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = F0[(k * N + j) * P + i];
    const EOSplit<N> sp = eo_split<N>(x);
    eo_mul<N, 1, false>(kp.M, sp, t);
    eo_mul<N, 1, false>(kp.L[0], sp, a);
    double xm[NL], xp[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      xm[l] = FC[0 * Lay::FACE + (l * N + k) * P + j];
      xp[l] = FC[1 * Lay::FACE + (l * N + k) * P + j];
    }
    dense_add<NL, NL>(kp.Nm[0], xm, &a[0]);
    dense_add<NL, NL>(kp.Np[0], xp, &a[N - NL]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      F1[(k * N + j) * P + i] = t[i];
      F2[(k * N + j) * P + i] = a[i];
    }
    // extra: M along x on the rows of the y- and z-neighbour layers (faces 2..5)
    for (int job = line; job < 4 * NL * N; job += NN) {
      double* row = FC + (2 + job / (NL * N)) * Lay::FACE + (job % (NL * N)) * P;
      double r[N], o[N];
#pragma unroll
      for (int i = 0; i < N; ++i) r[i] = row[i];
      eo_apply<N, 1>(kp.M, r, o);
#pragma unroll
      for (int i = 0; i < N; ++i) row[i] = o[i];
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- P2: y-lines
  if (active) {
    const int i = line % N, k = line / N;
    double al[N], tl[N], bl[N], cl[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      al[j] = F2[(k * N + j) * P + i];
      tl[j] = F1[(k * N + j) * P + i];
    }
    const EOSplit<N> st = eo_split<N>(tl);
    eo_mul<N, 1, false>(kp.M, eo_split<N>(al), bl);
    eo_mul<N, 1, true>(kp.L[1], st, bl);
    eo_mul<N, 1, false>(kp.M, st, cl);
    double ym[NL], yp[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      ym[l] = FC[2 * Lay::FACE + (l * N + k) * P + i];
      yp[l] = FC[3 * Lay::FACE + (l * N + k) * P + i];
    }
    dense_add<NL, NL>(kp.Nm[1], ym, &bl[0]);
    dense_add<NL, NL>(kp.Np[1], yp, &bl[N - NL]);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      F0[(k * N + j) * P + i] = bl[j];
      F1[(k * N + j) * P + i] = cl[j];
    }
    // extra: M along y on the (x-swept) z-neighbour layers: lines (f, l, a=i) along b=j
    for (int job = line; job < 2 * NL * N; job += NN) {
      const int f = 4 + job / (NL * N), l = (job / N) % NL, ii = job % N;
      double* base = FC + f * Lay::FACE + (l * N) * P + ii;
      double r[N], o[N];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) r[jj] = base[jj * P];
      eo_apply<N, 1>(kp.M, r, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj) base[jj * P] = o[jj];
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- P3: z-lines
  double res[N];
  const int zi = line % N, zj = line / N;
  if (active) {
    double bl[N], cl[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      bl[k] = F0[(k * N + zj) * P + zi];
      cl[k] = F1[(k * N + zj) * P + zi];
    }
    eo_mul<N, 1, false>(kp.M, eo_split<N>(bl), res);
    eo_mul<N, 1, true>(kp.L[2], eo_split<N>(cl), res);
    double zm[NL], zp[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      zm[l] = FC[4 * Lay::FACE + (l * N + zj) * P + zi];
      zp[l] = FC[5 * Lay::FACE + (l * N + zj) * P + zi];
    }
    dense_add<NL, NL>(kp.Nm[2], zm, &res[0]);
    dense_add<NL, NL>(kp.Np[2], zp, &res[N - NL]);
  }
  const int64_t gbase = cell_off<N>(cell0 + cslot) + zj * N + zi;   // + k*N*N

  if constexpr (MODE == KMODE_APPLY) {
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) y[gbase + k * NN] = res[k];
    }
    return;
  } else {
    // residual r = b - A u (z-line layout, coalesced loads)
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) res[k] = __ldg(ch.b + gbase + k * NN) - res[k];
    }
    if constexpr (MODE == KMODE_CHEBY_GL) {
      // (T^{-T})_z in registers
      if (active) {
        double o[N];
        eo_apply<N, 1>(kp.TiT, res, o);
#pragma unroll
        for (int k = 0; k < N; ++k) F2[(k * N + zj) * P + zi] = o[k];
      }
      __syncthreads();
      // (T^{-T})_y
      if (active) {
        const int i = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = F2[(k * N + j) * P + i];
        eo_apply<N, 1>(kp.TiT, r, o);
#pragma unroll
        for (int j = 0; j < N; ++j) F2[(k * N + j) * P + i] = o[j];
      }
      __syncthreads();
      // (T^{-T})_x, diag(A_GL)^{-1}, (T^{-1})_x
      if (active) {
        const int j = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int i = 0; i < N; ++i) r[i] = F2[(k * N + j) * P + i];
        eo_apply<N, 1>(kp.TiT, r, o);
        const double* dv = ch.dinv + cell_off<N>(cell0 + cslot) + (k * N + j) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) o[i] *= __ldg(dv + i);
        eo_apply<N, 1>(kp.Ti, o, r);
#pragma unroll
        for (int i = 0; i < N; ++i) F2[(k * N + j) * P + i] = r[i];
      }
      __syncthreads();
      // (T^{-1})_y
      if (active) {
        const int i = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = F2[(k * N + j) * P + i];
        eo_apply<N, 1>(kp.Ti, r, o);
#pragma unroll
        for (int j = 0; j < N; ++j) F2[(k * N + j) * P + i] = o[j];
      }
      __syncthreads();
      // (T^{-1})_z back to registers
      if (active) {
        double r[N];
#pragma unroll
        for (int k = 0; k < N; ++k) r[k] = F2[(k * N + zj) * P + zi];
        eo_apply<N, 1>(kp.Ti, r, res);
      }
    } else {
      // point Jacobi in the working basis
      if (active) {
#pragma unroll
        for (int k = 0; k < N; ++k) res[k] *= __ldg(ch.dinv + gbase + k * NN);
      }
    }
    // three-term update, Eq. (11): u_{j+1} = u_j + c_prev (u_j - u_{j-1}) + c_z P^{-1} r
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int64_t gi = gbase + k * NN;
        const double uj = __ldg(u + gi);
        double v = fma(ch.c_z, res[k], uj);
        if (!ch.first) v = fma(ch.c_prev, uj - ch.u_prev[gi], v);
        ch.u_next[gi] = v;
      }
    }
  }
}

template <int N, int NL>
constexpr int cells_per_block() {
  // target ~256 threads per block and <= ~100 KB of shared memory
  constexpr int byT = (256 + N * N - 1) / (N * N);
  constexpr int byS = (100 * 1024) / (KLayout<N, NL>::PER_CELL * 8);
  constexpr int c = byT < byS ? byT : byS;
  return c < 1 ? 1 : c;
}

template <int N, int NL, int MODE>
cudaError_t launch_t(const KronParams& kp, const GridArgs& g, const double* u, double* y,
                     const ChebyArgs& ch, cudaStream_t s) {
  constexpr int CPB = cells_per_block<N, NL>();
  const int64_t ncells = (int64_t)(g.zend - g.zbeg) * g.Nx * g.Ny;
  if (ncells <= 0) return cudaSuccess;
  const int64_t blocks = (ncells + CPB - 1) / CPB;
  const size_t smem = (size_t)CPB * KLayout<N, NL>::PER_CELL * sizeof(double);
  auto kern = k_kron<N, NL, CPB, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)blocks, CPB * N * N, smem, s>>>(kp, g, u, y, ch);
  return cudaGetLastError();
}

template <int N, int NL>
cudaError_t launch_mode(int mode, const KronParams& kp, const GridArgs& g, const double* u,
                        double* y, const ChebyArgs& ch, cudaStream_t s) {
  switch (mode) {
    case KMODE_APPLY: return launch_t<N, NL, KMODE_APPLY>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_GL: return launch_t<N, NL, KMODE_CHEBY_GL>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_PJ: return launch_t<N, NL, KMODE_CHEBY_PJ>(kp, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

template <int N>
cudaError_t launch_nl(int NL, int mode, const KronParams& kp, const GridArgs& g, const double* u,
                      double* y, const ChebyArgs& ch, cudaStream_t s) {
  if (NL == 2 && N > 2) return launch_mode<N, 2>(mode, kp, g, u, y, ch, s);
  if (NL == N) return launch_mode<N, N>(mode, kp, g, u, y, ch, s);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_kron(int n, int NL, int mode, const KronParams& kp, const GridArgs& g,
                        const double* u, double* y, const ChebyArgs& ch, cudaStream_t s) {
  switch (n) {
    case 2: return launch_nl<2>(NL, mode, kp, g, u, y, ch, s);
    case 3: return launch_nl<3>(NL, mode, kp, g, u, y, ch, s);
    case 4: return launch_nl<4>(NL, mode, kp, g, u, y, ch, s);
    case 5: return launch_nl<5>(NL, mode, kp, g, u, y, ch, s);
    case 6: return launch_nl<6>(NL, mode, kp, g, u, y, ch, s);
    case 7: return launch_nl<7>(NL, mode, kp, g, u, y, ch, s);
    case 8: return launch_nl<8>(NL, mode, kp, g, u, y, ch, s);
    case 9: return launch_nl<9>(NL, mode, kp, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dgb
