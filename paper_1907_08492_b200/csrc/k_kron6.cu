// Cartesian SIPG matvec, "i-plane" schedule (k_kron6): fewer shared-memory transposes.
//
// Same operator as k_kron4 (the Kronecker form of Eq. (14), of the
// quadrature operator of Eq. (1) on Cartesian cells), different data flow.  k_kron4 sweeps
// z, y and x in three line stages with two shared-memory transposes of two fields each
// (t, a after z; b, c after y): 64 B/DoF of shared traffic, the limiter measured by ncu
// (LSU pipe 70-84 %, profiles/r1_*).  Here one thread owns the whole (j, k) plane of one x
// index i of a cell, so the z and the y sweeps run in registers:
//   stage A (thread (cell, i)):  t = M_z u, a = L_z u + N_z^{+-} u_{z+-}   (z-lines j of the plane)
//                                b = M_y a + L_y t [+ N_y^{+-} (M_z u_{y+-})],  c = M_y t   (y-lines k)
//                                b, c -> shared memory (one transpose, two fields)
//   stage X (thread (cell, j)):  y = M_x b + L_x c + N_x^{+-} c_{x+-}   along the x-lines (j, k)
// The y-neighbour term is added to b afterwards in place (the neighbour's two layers, M_z
// along their z-lines).  x-neighbours outside the block are computed as extra "virtual"
// cells (their c planes at the two layers next to the face); mirror faces copy -c
// reflected, a periodic row inside the block copies the other end.
// Shared traffic 16 B/DoF written + 16 B/DoF read.  fp64, Hermite-like basis (NL = 2),
// n = 3..6 (the plane, 2 n^2 doubles, lives in registers).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "dg_internal.h"

namespace dgb {
namespace {

// TP threads per cell (N working + padding for odd N so the shared accesses are
// conflict-free), CPB cells per block, shared layout addr = i + Sj j + Sk k + CS slot
// (tools/k6_iplane_layout.py: half-warp cost model, 1.0 = conflict-free for both the
// stage-A writes and the stage-X reads).
template <int N> struct K6;
template <> struct K6<3> { static constexpr int TP = 4, CPB = 40, Sj = 3, Sk = 9, CS = 28, MINB = 4; };
template <> struct K6<4> { static constexpr int TP = 4, CPB = 32, Sj = 5, Sk = 20, CS = 84, MINB = 3; };
template <> struct K6<5> { static constexpr int TP = 6, CPB = 24, Sj = 9, Sk = 45, CS = 230, MINB = 2; };
template <> struct K6<6> { static constexpr int TP = 6, CPB = 20, Sj = 9, Sk = 54, CS = 326, MINB = 2; };

template <int N>
__device__ __forceinline__ int k6a(int i, int j, int k) {
  return i + K6<N>::Sj * j + K6<N>::Sk * k;
}

// one 1D operator (even-odd packed, parity +1) on a line held in registers
template <int N>
__device__ __forceinline__ void line_apply(const double* __restrict__ A, const double (&x)[N], double (&y)[N]) {
  eo_mul<N, 1, false>(A, eo_split<N>(x), y);
}

template <int N, int MODE>
__global__ void __launch_bounds__((K6<N>::CPB + 2) * K6<N>::TP, K6<N>::MINB)
k_kron6(const __grid_constant__ KronParams kp, const __grid_constant__ GridArgs g,
        const double* __restrict__ u, double* __restrict__ y, const __grid_constant__ ChebyArgs ch) {
  using C = K6<N>;
  constexpr int NL = 2, NN = N * N, N3 = N * NN, TP = C::TP, CPB = C::CPB, CS = C::CS;
  extern __shared__ __align__(16) double sm6[];
  double* Bf = sm6;                      // b field, slots [-1, CPB] (virtual slots unused)
  double* Cf = sm6 + (CPB + 2) * CS;     // c field
  const int tid = threadIdx.x;
  const int slot = tid / TP - 1;         // -1 .. CPB
  const int x = tid - (slot + 1) * TP;   // i in stage A, j in stage X
  const int cx0 = blockIdx.x * CPB;
  const int cy = blockIdx.y;
  const int cz = g.zbeg + blockIdx.z;
  const int ncell = g.Nx - cx0 < CPB ? g.Nx - cx0 : CPB;
  const int64_t plane = (int64_t)g.Nx * g.Ny;
  const int64_t rowcell = ((int64_t)cz * g.Ny + cy) * g.Nx;

  // x-neighbours of the block edges
  const bool xper = g.bc[0] == DG_BC_PERIODIC;
  int h0 = cx0 > 0 ? cx0 - 1 : (xper ? g.Nx - 1 : -1);
  int h1 = cx0 + ncell < g.Nx ? cx0 + ncell : (xper ? 0 : -1);
  const bool wrap = xper && ncell == g.Nx;   // whole periodic row in the block
  if (wrap) h0 = h1 = -1;
  const bool real = slot >= 0 && slot < ncell && x < N;
  // virtual halo planes: left cell h0 planes i >= N-NL, right cell h1 planes i < NL
  const bool vleft = slot == -1 && h0 >= 0 && x < N && x >= N - NL;
  const bool vright = slot == ncell && h1 >= 0 && x < N && x < NL;
  const bool work = real || vleft || vright;
  const int cx = real ? cx0 + slot : (vleft ? h0 : (vright ? h1 : cx0));
  const int i = x;
  double* Bc = Bf + (slot + 1) * CS;
  double* Cc = Cf + (slot + 1) * CS;

  // ================================================================ stage A
  if (work) {
    const double* ucell = u + (rowcell + cx) * N3 + i;
    // z-neighbour sources (plane below / above): local, halo or mirror
    const double* zb[2];
    int zmode[2];   // 0 local/halo pointer, 1 mirror
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int nz = cz + (s ? 1 : -1);
      if (nz >= 0 && nz < g.nz) {
        zmode[s] = 0;
        zb[s] = ucell + (s ? plane * N3 : -plane * N3);
      } else {
        const int src = s ? g.zhi : g.zlo;
        zmode[s] = src == ZSRC_MIRROR;
        zb[s] = ucell + (s ? -(int64_t)(g.nz - 1) : (int64_t)(g.nz - 1)) * plane * N3;   // periodic wrap
        if (src == ZSRC_HALO)
          zb[s] = (s ? g.halo_hi : g.halo_lo) + ((int64_t)cy * g.Nx + cx) * (NL * NN) + i - (s ? 0 : (N - NL) * NN);
      }
    }
    double t[N][N], a[N][N];   // [j][k]
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double zl[N];
#pragma unroll
      for (int k = 0; k < N; ++k) zl[k] = __ldg(ucell + k * NN + j * N);
      double zm[NL], zp[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int Lm = N - NL + l, Lp = l;
        zm[l] = zmode[0] ? -zl[N - 1 - Lm] : __ldg(zb[0] + Lm * NN + j * N);
        zp[l] = zmode[1] ? -zl[N - 1 - Lp] : __ldg(zb[1] + Lp * NN + j * N);
      }
      const auto sz = eo_split<N>(zl);
      eo_mul<N, 1, false>(kp.M, sz, t[j]);
      eo_mul<N, 1, false>(kp.L[2], sz, a[j]);
      dense_add<NL, NL>(kp.Nm[2], zm, &a[j][0]);
      dense_add<NL, NL>(kp.Np[2], zp, &a[j][N - NL]);
    }
    // y-lines: b = M_y a + L_y t (+ mirror ghosts), c = M_y t
    const bool yper = g.bc[1] == DG_BC_PERIODIC;
    const int ym_row = cy > 0 ? cy - 1 : (yper ? g.Ny - 1 : -1);
    const int yp_row = cy + 1 < g.Ny ? cy + 1 : (yper ? 0 : -1);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double al[N], tl[N], bl[N], cl[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        al[j] = a[j][k];
        tl[j] = t[j][k];
      }
      const auto st = eo_split<N>(tl);
      eo_mul2<N, 1>(kp.M, eo_split<N>(al), kp.L[1], st, bl);
      eo_mul<N, 1, false>(kp.M, st, cl);
      if (ym_row < 0) {   // mirror: ghost layers -t reflected
        double gm[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) gm[l] = -tl[NL - 1 - l];
        dense_add<NL, NL>(kp.Nm[1], gm, &bl[0]);
      }
      if (yp_row < 0) {
        double gp[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) gp[l] = -tl[N - 1 - l];
        dense_add<NL, NL>(kp.Np[1], gp, &bl[N - NL]);
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        Bc[k6a<N>(i, j, k)] = bl[j];
        Cc[k6a<N>(i, j, k)] = cl[j];
      }
    }
    // y-neighbour layers (real cells only): b rows next to the face += N_y (M_z u_{y+-})
    if (real) {
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int nrow = f ? yp_row : ym_row;
        if (nrow < 0) continue;
        const double* src = u + (((int64_t)cz * g.Ny + nrow) * g.Nx + cx) * N3 + i;
        double gz[NL][N];
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int jl = f ? l : N - NL + l;
          double zl[N];
#pragma unroll
          for (int k = 0; k < N; ++k) zl[k] = __ldg(src + k * NN + jl * N);
          line_apply<N>(kp.M, zl, gz[l]);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double gk[NL];
#pragma unroll
          for (int l = 0; l < NL; ++l) gk[l] = gz[l][k];
#pragma unroll
          for (int r = 0; r < NL; ++r) {
            const int j = f ? N - NL + r : r;
            const double* Nmat = f ? kp.Np[1] : kp.Nm[1];
            double acc = Bc[k6a<N>(i, j, k)];
#pragma unroll
            for (int l = 0; l < NL; ++l) acc = fma(Nmat[r * NL + l], gk[l], acc);
            Bc[k6a<N>(i, j, k)] = acc;
          }
        }
      }
    }
  }
  // mirror / in-block wrap x-neighbours of the edge cells: fill the virtual slots' c planes
  // (left slot -1 holds planes N-NL.., right slot ncell planes ..NL-1 of the neighbour)
  if (real) {
    const bool lmir = cx0 == 0 && !xper, rmir = cx0 + ncell == g.Nx && !xper;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      int dst_i = -1;
      double sgn = 1.0;
      if (side == 0 && slot == 0 && i < NL && lmir) { dst_i = N - 1 - i; sgn = -1.0; }           // mirror
      if (side == 0 && slot == ncell - 1 && i >= N - NL && wrap) dst_i = i;                         // wrap
      if (side == 1 && slot == ncell - 1 && i >= N - NL && rmir) { dst_i = N - 1 - i; sgn = -1.0; }
      if (side == 1 && slot == 0 && i < NL && wrap) dst_i = i;
      if (dst_i < 0) continue;
      double* D = Cf + (side ? ncell + 1 : 0) * CS;
#pragma unroll
      for (int k = 0; k < N; ++k)
#pragma unroll
        for (int j = 0; j < N; ++j) D[k6a<N>(dst_i, j, k)] = sgn * Cc[k6a<N>(i, j, k)];
    }
  }
  __syncthreads();

  // ================================================================ stage X
  const int j = x;
  const int64_t cbase = (rowcell + cx0 + slot) * N3;   // own cell (real threads)
  double* Bs = Bf + (slot + 1) * CS;
  if (real) {
    const double* Cs = Cf + (slot + 1) * CS;
    const double* Cm = Cs - CS;
    const double* Cp = Cs + CS;
    double* out = y + cbase + j * N;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double bl[N], cl[N], res[N];
#pragma unroll
      for (int ii = 0; ii < N; ++ii) {
        bl[ii] = Bs[k6a<N>(ii, j, k)];
        cl[ii] = Cs[k6a<N>(ii, j, k)];
      }
      double cxm[NL], cxp[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        cxm[l] = Cm[k6a<N>(N - NL + l, j, k)];
        cxp[l] = Cp[k6a<N>(l, j, k)];
      }
      eo_mul2<N, 1>(kp.M, eo_split<N>(bl), kp.L[0], eo_split<N>(cl), res);
      dense_add<NL, NL>(kp.Nm[0], cxm, &res[0]);
      dense_add<NL, NL>(kp.Np[0], cxp, &res[N - NL]);
      if constexpr (MODE == KMODE_APPLY) {
        if constexpr (N % 2 == 0) {
#pragma unroll
          for (int ii = 0; ii < N; ii += 2)
            *reinterpret_cast<double2*>(out + k * NN + ii) = make_double2(res[ii], res[ii + 1]);
        } else {
#pragma unroll
          for (int ii = 0; ii < N; ++ii) out[k * NN + ii] = res[ii];
        }
      } else {
        // fused Chebyshev step (Eq. (11)): r = b - A u along the x-line
        const double* bb = ch.b + cbase + k * NN + j * N;
#pragma unroll
        for (int ii = 0; ii < N; ++ii) res[ii] = __ldg(bb + ii) - res[ii];
        if constexpr (MODE == KMODE_CHEBY_PJ) {   // P^{-1} = diag(A)^{-1}: update right here
          const double* dv = ch.dinv + cbase + k * NN + j * N;
          const double* uj = u + cbase + k * NN + j * N;
          const double* up = ch.u_prev + cbase + k * NN + j * N;
          double* un = ch.u_next + cbase + k * NN + j * N;
#pragma unroll
          for (int ii = 0; ii < N; ++ii) {
            const double ujv = __ldg(uj + ii);
            double v = fma(ch.c_z, res[ii] * __ldg(dv + ii), ujv);
            if (!ch.first) v = fma(ch.c_prev, ujv - up[ii], v);
            un[ii] = v;
          }
        } else {   // GL-Jacobi, Eq. (12): x-direction T^{-T} now, in place over b (own positions)
          double o[N];
          eo_apply<N, 1>(kp.TiT, res, o);
#pragma unroll
          for (int ii = 0; ii < N; ++ii) Bs[k6a<N>(ii, j, k)] = o[ii];
        }
      }
    }
  }
  if constexpr (MODE == KMODE_CHEBY_GL) {
    __syncthreads();
    // stage P (thread (cell, i), the plane again): y and z directions of
    // P^{-1} = (T^{-1})^{x3} diag(A_GL)^{-1} (T^{-T})^{x3} (Eq. (12), R13) in registers
    if (real) {
      double pl[N][N];   // [j][k]
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double v[N], o[N];
#pragma unroll
        for (int jj = 0; jj < N; ++jj) v[jj] = Bc[k6a<N>(i, jj, k)];
        eo_apply<N, 1>(kp.TiT, v, o);               // y: T^{-T}
#pragma unroll
        for (int jj = 0; jj < N; ++jj) pl[jj][k] = o[jj];
      }
      const double* dv = ch.dinv + cbase + i;
#pragma unroll
      for (int jj = 0; jj < N; ++jj) {
        double o[N], w[N];
        eo_apply<N, 1>(kp.TiT, pl[jj], o);          // z: T^{-T}
#pragma unroll
        for (int k = 0; k < N; ++k) o[k] *= __ldg(dv + k * NN + jj * N);   // diag(A_GL)^{-1}
        eo_apply<N, 1>(kp.Ti, o, w);                // z: T^{-1}
#pragma unroll
        for (int k = 0; k < N; ++k) pl[jj][k] = w[k];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double v[N], o[N];
#pragma unroll
        for (int jj = 0; jj < N; ++jj) v[jj] = pl[jj][k];
        eo_apply<N, 1>(kp.Ti, v, o);                // y: T^{-1}
#pragma unroll
        for (int jj = 0; jj < N; ++jj) Bc[k6a<N>(i, jj, k)] = o[jj];
      }
    }
    __syncthreads();
    // stage X2 (x-lines): T^{-1} and the three-term update of Eq. (11)
    if (real) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double v[N], z[N];
#pragma unroll
        for (int ii = 0; ii < N; ++ii) v[ii] = Bs[k6a<N>(ii, j, k)];
        eo_apply<N, 1>(kp.Ti, v, z);
        const int64_t o0 = cbase + k * NN + j * N;
        if constexpr (N % 2 == 0) {
#pragma unroll
          for (int ii = 0; ii < N; ii += 2) {
            const double2 uj = __ldg(reinterpret_cast<const double2*>(u + o0 + ii));
            double2 r;
            r.x = fma(ch.c_z, z[ii], uj.x);
            r.y = fma(ch.c_z, z[ii + 1], uj.y);
            if (!ch.first) {
              const double2 up = *reinterpret_cast<const double2*>(ch.u_prev + o0 + ii);
              r.x = fma(ch.c_prev, uj.x - up.x, r.x);
              r.y = fma(ch.c_prev, uj.y - up.y, r.y);
            }
            *reinterpret_cast<double2*>(ch.u_next + o0 + ii) = r;
          }
        } else {
#pragma unroll
          for (int ii = 0; ii < N; ++ii) {
            const double ujv = __ldg(u + o0 + ii);
            double r = fma(ch.c_z, z[ii], ujv);
            if (!ch.first) r = fma(ch.c_prev, ujv - ch.u_prev[o0 + ii], r);
            ch.u_next[o0 + ii] = r;
          }
        }
      }
    }
  }
}

template <int N, int MODE>
cudaError_t launch_mode(const KronParams& kp, const GridArgs& g, const double* u, double* y, const ChebyArgs& ch,
                        cudaStream_t s) {
  using C = K6<N>;
  const int planes = g.zend - g.zbeg;
  if (planes <= 0 || g.Nx <= 0 || g.Ny <= 0) return cudaSuccess;
  if (g.Ny > 65535 || planes > 65535) return cudaErrorInvalidValue;
  const dim3 grid((g.Nx + C::CPB - 1) / C::CPB, g.Ny, planes);
  const size_t smem = (size_t)2 * (C::CPB + 2) * C::CS * sizeof(double);
  auto kern = k_kron6<N, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, (C::CPB + 2) * C::TP, smem, s>>>(kp, g, u, y, ch);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_n(int mode, const KronParams& kp, const GridArgs& g, const double* u, double* y,
                     const ChebyArgs& ch, cudaStream_t s) {
  switch (mode) {
    case KMODE_APPLY: return launch_mode<N, KMODE_APPLY>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_GL: return launch_mode<N, KMODE_CHEBY_GL>(kp, g, u, y, ch, s);
    case KMODE_CHEBY_PJ: return launch_mode<N, KMODE_CHEBY_PJ>(kp, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool kron6_supported(int n, int NL, int mode) {
  return NL == 2 && n >= 3 && n <= 6 &&
         (mode == KMODE_APPLY || mode == KMODE_CHEBY_GL || mode == KMODE_CHEBY_PJ);
}

cudaError_t launch_kron6(int n, int mode, const KronParams& kp, const GridArgs& g, const double* u, double* y,
                         const ChebyArgs& ch, cudaStream_t s) {
  switch (n) {
    case 3: return launch_n<3>(mode, kp, g, u, y, ch, s);
    case 4: return launch_n<4>(mode, kp, g, u, y, ch, s);
    case 5: return launch_n<5>(mode, kp, g, u, y, ch, s);
    case 6: return launch_n<6>(mode, kp, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dgb
