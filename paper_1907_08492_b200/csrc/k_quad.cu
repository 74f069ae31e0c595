// General element-centric SIPG kernel: the paper's formulation by quadrature with
// sum factorisation (Eqs. (3)-(5)), element-wise face
// arrangement, Hermite-like face access.
// Handles any geometry the library stores: a constant merged tensor
// (PAPER.md:798-804), per-cell affine J^-1 or per-quadrature-point merged tensors
// with per-face-point normal data.
//
// One thread per line (n^2 threads per cell), lines register-resident, smem
// transposes between directions.  Per cell:
//   P0  stage own coefficients + NL neighbour layers per face (loader.cuh)
//   F1  lines along a of every face: V = S_f-trace, D = D_f-trace of own and
//       neighbour layers; S V, DS V, S D                       (Eq. (5))
//   F2  lines along b: u, grad_xi u at the n^2 face points of both sides,
//       SIPG flux of Eq. (1), transposed b-sweeps of the test terms
//   F3  transposed a-sweeps -> two layer contributions R0 (S_f^T), R1 (D_f^T)
//   X   a = S u, b = DS u                     (cell interpolation in the DS form:
//   Y   c1 = S b, c2 = DS a, c3 = S a          grad_xi u = (S S DS, S DS S, DS S S) u)
//   Z   g = (S c1, S c2, DS c3); t = G_q g; d = (S^T t_x, S^T t_y, DS^T t_z)
//   YT  e1 = S^T d1, e2 = DS^T d2 + S^T d3
//   XT  y = DS^T e1 + S^T e2 + face injections of R0, R1 (single write)
// The fused Chebyshev variants continue from XT in registers.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dg_internal.h"
#include "loader.cuh"

namespace dgb {
namespace {

template <int N, int NL>
struct QLayout {
  static constexpr int P = N | 1;
  static constexpr int FIELD = N * N * P;
  static constexpr int FACE = NL * N * P;
  static constexpr int FW = 6 * 6 * N * P;
  static constexpr int CELLW = 5 * FIELD;
  static constexpr int W = FW > CELLW ? FW : CELLW;
  static constexpr int R = 6 * 2 * N * P;
  static constexpr int PER_CELL = FIELD + 6 * FACE + W + R;
};

__device__ __forceinline__ double pick3(const double (&v)[3], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]);
}

// own coefficient (d-coordinate m, tangential a, b) in the padded smem field
template <int N, int P>
__device__ __forceinline__ int own_idx(int d, int m, int a, int b) {
  return d == 0 ? (b * N + a) * P + m : (d == 1 ? (b * N + m) * P + a : (m * N + b) * P + a);
}

// Face geometry of cell K at face f, point (qa, qb): ck_m = dA J_K^-1 n_K,
// ck_p = dA J_{K+}^-1 n_K (neighbour reference frame), sdA = sigma dA.
template <int N, int GEOM>
__device__ __forceinline__ void face_geom(const QuadParams& qp, const GeomArgs& ga, const GridArgs& g,
                                          int64_t cid, int cx, int cy, int czl, int f, int qa, int qb,
                                          double (&ckm)[3], double (&ckp)[3], double& sdA, bool mirror) {
  const int d = f >> 1, s = f & 1;
  const double nu = s ? 1.0 : -1.0;
  if constexpr (GEOM == GEOM_CONST) {
    const double ww = qp.w[qa] * qp.w[qb];
#pragma unroll
    for (int k = 0; k < 3; ++k) ckm[k] = ckp[k] = nu * ww * qp.cw0[d][k];
    sdA = ww * qp.sdA0[d];
  } else if constexpr (GEOM == GEOM_PER_QPOINT) {
    int64_t fid;
    if (d == 0) fid = ((int64_t)czl * g.Ny + cy) * (g.Nx + 1) + cx + s;
    else if (d == 1) fid = ((int64_t)czl * (g.Ny + 1) + cy + s) * g.Nx + cx;
    else fid = ((int64_t)(czl + s) * g.Ny + cy) * g.Nx + cx;
    const double* fd = ga.face[d] + fid * (4 * N * N) + qb * N + qa;
#pragma unroll
    for (int k = 0; k < 3; ++k) ckm[k] = ckp[k] = nu * __ldg(fd + k * N * N);
    sdA = __ldg(fd + 3 * N * N);
  } else {  // GEOM_PER_CELL: affine cells, J^-1 + det J per cell (plus ghost planes)
    const int plane = g.Nx * g.Ny;
    const double* jo = ga.jinv + ((int64_t)(czl + 1) * plane + (int64_t)cy * g.Nx + cx) * 10;
    double r[3], Ji[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Ji[k] = __ldg(jo + k);
    const double detJ = __ldg(jo + 9);
#pragma unroll
    for (int k = 0; k < 3; ++k) r[k] = d == 0 ? Ji[k] : (d == 1 ? Ji[3 + k] : Ji[6 + k]);
    const double nr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    const double ww = qp.w[qa] * qp.w[qb];
    const double fac = nu * ww * detJ;
#pragma unroll
    for (int k = 0; k < 3; ++k) ckm[k] = fac * (Ji[k * 3] * r[0] + Ji[k * 3 + 1] * r[1] + Ji[k * 3 + 2] * r[2]);
    double sig;
    int64_t fid;   // face index in the layout of the per-face arrays (user penalties)
    if (d == 0) fid = ((int64_t)czl * g.Ny + cy) * (g.Nx + 1) + cx + s;
    else if (d == 1) fid = ((int64_t)czl * (g.Ny + 1) + cy + s) * g.Nx + cx;
    else fid = ((int64_t)(czl + s) * g.Ny + cy) * g.Nx + cx;
    if (mirror) {
#pragma unroll
      for (int k = 0; k < 3; ++k) ckp[k] = ckm[k];
      sig = ga.pen * nr;
    } else {
      int nx = cx, ny = cy, nz = czl;
      if (d == 0) nx = (cx + (s ? 1 : -1) + g.Nx) % g.Nx;
      if (d == 1) ny = (cy + (s ? 1 : -1) + g.Ny) % g.Ny;
      if (d == 2) nz = czl + (s ? 1 : -1);
      const double* jn = ga.jinv + ((int64_t)(nz + 1) * plane + (int64_t)ny * g.Nx + nx) * 10;
      double Jn[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) Jn[k] = __ldg(jn + k);
#pragma unroll
      for (int k = 0; k < 3; ++k) ckp[k] = fac * (Jn[k * 3] * r[0] + Jn[k * 3 + 1] * r[1] + Jn[k * 3 + 2] * r[2]);
      double rp[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) rp[k] = d == 0 ? Jn[k] : (d == 1 ? Jn[3 + k] : Jn[6 + k]);
      const double nrp = sqrt(rp[0] * rp[0] + rp[1] * rp[1] + rp[2] * rp[2]);
      sig = ga.pen * 0.5 * (nr + nrp);
    }
    if (ga.sig[d]) sig = __ldg(ga.sig[d] + fid);   // dg.h user_penalty: sigma_F as given
    sdA = sig * detJ * nr * ww;
    (void)cid;
  }
}

__device__ __forceinline__ void l2_prefetch_range(const double* p, int64_t ndoubles, int tid, int bt) {
  const char* c = reinterpret_cast<const char*>(p);
  for (int64_t o = (int64_t)tid * 128; o < ndoubles * 8; o += (int64_t)bt * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
}

template <int N, int NL, int CPB, int GEOM, int MODE>
__global__ void __launch_bounds__(CPB * N * N)
k_quad(const __grid_constant__ QuadParams qp, const __grid_constant__ GeomArgs ga,
       const __grid_constant__ GridArgs g, const double* __restrict__ u, double* __restrict__ y,
       const __grid_constant__ ChebyArgs ch) {
  using Lay = QLayout<N, NL>;
  constexpr int P = Lay::P;
  constexpr int NN = N * N;
  extern __shared__ double smem[];

  const int plane = g.Nx * g.Ny;
  const int64_t cbeg = (int64_t)g.zbeg * plane;
  const int64_t cend = (int64_t)g.zend * plane;
  const int64_t cell0 = cbeg + (int64_t)blockIdx.x * CPB;
  const int ncell = (int)(cend - cell0 < CPB ? cend - cell0 : CPB);
  const int tid = threadIdx.x;
  const int cslot = tid / NN;
  const int line = tid % NN;
  const bool active = cslot < ncell;
  const int64_t cid = cell0 + cslot;
  double* U = smem + cslot * Lay::PER_CELL;
  double* FN = U + Lay::FIELD;
  double* W = FN + 6 * Lay::FACE;
  double* R = W + Lay::W;
  const int czl = (int)(cid / plane);
  const int crem = (int)(cid - (int64_t)czl * plane);
  const int cy = crem / g.Nx, cx = crem - cy * g.Nx;

  // L2 prefetch: this block's per-q-point tensors (read in stage Z, after the face
  // work) and the next plane's tile (u, tensors; its block runs about a wave later)
  if (GEOM == GEOM_PER_QPOINT && g.l2pf) {
    const int64_t cnt = (int64_t)ncell * 6 * N * NN;
    l2_prefetch_range(ga.G + cell0 * (6 * N * NN), cnt, tid, blockDim.x);
    if (cell0 + plane + ncell <= (int64_t)g.nz * plane) {
      l2_prefetch_range(ga.G + (cell0 + plane) * (6 * N * NN), cnt, tid, blockDim.x);
      l2_prefetch_range(u + (cell0 + plane) * (N * NN), (int64_t)ncell * N * NN, tid, blockDim.x);
    }
  }
  // ---------------------------------------------------------------- P0
  int mirror_bits = 0;
  if (active) mirror_bits = stage_cell<N, NL, P, Lay::FACE>(g, u, cid, line, U, FN);
  __syncthreads();

  // ---------------------------------------------------------------- F1: a-lines
  if (active) {
    for (int job = line; job < 6 * N; job += NN) {
      const int f = job / N, b = job % N, d = f >> 1, s = f & 1;
      double Vm[N], Dm[N], Vp[N], Dp[N];
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double v = 0.0, dd = 0.0, vp = 0.0, dp = 0.0;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int L = s ? N - NL + l : l;
          const double x = U[own_idx<N, P>(d, L, a, b)];
          v = fma(qp.sf[s][l], x, v);
          dd = fma(qp.df[s][l], x, dd);
          const double xn = FN[f * Lay::FACE + (l * N + b) * P + a];
          vp = fma(qp.sfn[s][l], xn, vp);
          dp = fma(qp.dfn[s][l], xn, dp);
        }
        Vm[a] = v;
        Dm[a] = dd;
        Vp[a] = vp;
        Dp[a] = dp;
      }
      double o[N];
      double* base = W + (f * 6 * N + b) * P;   // field q at base + q*N*P
      {
        const EOSplit<N> sv = eo_split<N>(Vm);
        eo_mul<N, 1, false>(qp.S, sv, o);
#pragma unroll
        for (int a = 0; a < N; ++a) base[0 * N * P + a] = o[a];
        eo_mul<N, -1, false>(qp.D, sv, o);
#pragma unroll
        for (int a = 0; a < N; ++a) base[1 * N * P + a] = o[a];
        eo_apply<N, 1>(qp.S, Dm, o);
#pragma unroll
        for (int a = 0; a < N; ++a) base[2 * N * P + a] = o[a];
      }
      if (!((mirror_bits >> f) & 1)) {
        const EOSplit<N> sv = eo_split<N>(Vp);
        eo_mul<N, 1, false>(qp.S, sv, o);
#pragma unroll
        for (int a = 0; a < N; ++a) base[3 * N * P + a] = o[a];
        eo_mul<N, -1, false>(qp.D, sv, o);
#pragma unroll
        for (int a = 0; a < N; ++a) base[4 * N * P + a] = o[a];
        eo_apply<N, 1>(qp.S, Dp, o);
#pragma unroll
        for (int a = 0; a < N; ++a) base[5 * N * P + a] = o[a];
      }
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- F2: b-lines + flux
  if (active) {
    for (int job = line; job < 6 * N; job += NN) {
      const int f = job / N, qa = job % N, d = f >> 1;
      const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
      const bool mir = (mirror_bits >> f) & 1;
      double* col = W + (f * 6 * N) * P + qa;     // field q, row b at col[(q*N + b)*P]
      double x0[N], x1[N], x2[N];
#pragma unroll
      for (int b = 0; b < N; ++b) {
        x0[b] = col[(0 * N + b) * P];
        x1[b] = col[(1 * N + b) * P];
        x2[b] = col[(2 * N + b) * P];
      }
      double um[N], gam[N], gbm[N], gnm[N];
      {
        const EOSplit<N> s0 = eo_split<N>(x0);
        eo_mul<N, 1, false>(qp.S, s0, um);
        eo_mul<N, -1, false>(qp.D, s0, gbm);
      }
      eo_apply<N, 1>(qp.S, x1, gam);
      eo_apply<N, 1>(qp.S, x2, gnm);
      double up[N], gap[N], gbp[N], gnp[N];
      if (!mir) {
#pragma unroll
        for (int b = 0; b < N; ++b) {
          x0[b] = col[(3 * N + b) * P];
          x1[b] = col[(4 * N + b) * P];
          x2[b] = col[(5 * N + b) * P];
        }
        const EOSplit<N> s0 = eo_split<N>(x0);
        eo_mul<N, 1, false>(qp.S, s0, up);
        eo_mul<N, -1, false>(qp.D, s0, gbp);
        eo_apply<N, 1>(qp.S, x1, gap);
        eo_apply<N, 1>(qp.S, x2, gnp);
      }
      double rv[N], ra[N], rb[N], rn[N];
#pragma unroll
      for (int qb = 0; qb < N; ++qb) {
        double ckm[3], ckp[3], sdA;
        face_geom<N, GEOM>(qp, ga, g, cid, cx, cy, czl, f, qa, qb, ckm, ckp, sdA, mir);
        const double cmn = pick3(ckm, d), cma = pick3(ckm, t1), cmb = pick3(ckm, t2);
        const double dotm = cmn * gnm[qb] + cma * gam[qb] + cmb * gbm[qb];
        double jump, avg;
        if (mir) {
          jump = 2.0 * um[qb];
          avg = dotm;
        } else {
          const double dotp = pick3(ckp, d) * gnp[qb] + pick3(ckp, t1) * gap[qb] + pick3(ckp, t2) * gbp[qb];
          jump = um[qb] - up[qb];
          avg = 0.5 * (dotm + dotp);
        }
        rv[qb] = sdA * jump - avg;
        const double hj = -0.5 * jump;
        rn[qb] = hj * cmn;
        ra[qb] = hj * cma;
        rb[qb] = hj * cmb;
      }
      double T1[N], T2[N], T3[N];
      eo_apply<N, 1>(qp.St, rv, T1);
      eo_apply_add<N, -1>(qp.Dt, rb, T1);
      eo_apply<N, 1>(qp.St, ra, T2);
      eo_apply<N, 1>(qp.St, rn, T3);
#pragma unroll
      for (int b = 0; b < N; ++b) {
        col[(0 * N + b) * P] = T1[b];
        col[(1 * N + b) * P] = T2[b];
        col[(2 * N + b) * P] = T3[b];
      }
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- F3: a-lines (transposed)
  if (active) {
    for (int job = line; job < 6 * N; job += NN) {
      const int f = job / N, b = job % N;
      const double* base = W + (f * 6 * N + b) * P;
      double t1[N], t2[N], t3[N], r0[N], r1[N];
#pragma unroll
      for (int a = 0; a < N; ++a) {
        t1[a] = base[0 * N * P + a];
        t2[a] = base[1 * N * P + a];
        t3[a] = base[2 * N * P + a];
      }
      eo_apply<N, 1>(qp.St, t1, r0);
      eo_apply_add<N, -1>(qp.Dt, t2, r0);
      eo_apply<N, 1>(qp.St, t3, r1);
      double* rb = R + (f * 2 * N + b) * P;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        rb[a] = r0[a];
        rb[N * P + a] = r1[a];
      }
    }
  }
  __syncthreads();

  double* A = W;
  double* B = W + Lay::FIELD;
  double* C1 = W + 2 * Lay::FIELD;
  double* C2 = W + 3 * Lay::FIELD;
  double* C3 = W + 4 * Lay::FIELD;
  // ---------------------------------------------------------------- X
  if (active) {
    const int j = line % N, k = line / N;
    double x[N], o[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = U[(k * N + j) * P + i];
    const EOSplit<N> sx = eo_split<N>(x);
    eo_mul<N, 1, false>(qp.S, sx, o);
#pragma unroll
    for (int i = 0; i < N; ++i) A[(k * N + j) * P + i] = o[i];
    eo_mul<N, -1, false>(qp.D, sx, o);
#pragma unroll
    for (int i = 0; i < N; ++i) B[(k * N + j) * P + i] = o[i];
  }
  __syncthreads();
  // ---------------------------------------------------------------- Y
  if (active) {
    const int i = line % N, k = line / N;
    double al[N], bl[N], o[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      al[j] = A[(k * N + j) * P + i];
      bl[j] = B[(k * N + j) * P + i];
    }
    eo_apply<N, 1>(qp.S, bl, o);
#pragma unroll
    for (int j = 0; j < N; ++j) C1[(k * N + j) * P + i] = o[j];
    const EOSplit<N> sa = eo_split<N>(al);
    eo_mul<N, -1, false>(qp.D, sa, o);
#pragma unroll
    for (int j = 0; j < N; ++j) C2[(k * N + j) * P + i] = o[j];
    eo_mul<N, 1, false>(qp.S, sa, o);
#pragma unroll
    for (int j = 0; j < N; ++j) C3[(k * N + j) * P + i] = o[j];
  }
  __syncthreads();
  // ---------------------------------------------------------------- Z (+ q-point work)
  if (active) {
    const int i = line % N, j = line / N;
    double c1[N], c2[N], c3[N], gx[N], gy[N], gz[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      c1[k] = C1[(k * N + j) * P + i];
      c2[k] = C2[(k * N + j) * P + i];
      c3[k] = C3[(k * N + j) * P + i];
    }
    eo_apply<N, 1>(qp.S, c1, gx);
    eo_apply<N, 1>(qp.S, c2, gy);
    eo_apply<N, -1>(qp.D, c3, gz);
    double Gc[6];
    if constexpr (GEOM == GEOM_PER_CELL) {
      const double* jo = ga.jinv + ((int64_t)(czl + 1) * plane + (int64_t)cy * g.Nx + cx) * 10;
      double Ji[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) Ji[q] = __ldg(jo + q);
      const double dj = __ldg(jo + 9);
      // det J J^-1 J^-T : (a,b) = sum_k Ji[a][k] Ji[b][k]
      Gc[0] = dj * (Ji[0] * Ji[0] + Ji[1] * Ji[1] + Ji[2] * Ji[2]);
      Gc[1] = dj * (Ji[3] * Ji[3] + Ji[4] * Ji[4] + Ji[5] * Ji[5]);
      Gc[2] = dj * (Ji[6] * Ji[6] + Ji[7] * Ji[7] + Ji[8] * Ji[8]);
      Gc[3] = dj * (Ji[0] * Ji[3] + Ji[1] * Ji[4] + Ji[2] * Ji[5]);
      Gc[4] = dj * (Ji[0] * Ji[6] + Ji[1] * Ji[7] + Ji[2] * Ji[8]);
      Gc[5] = dj * (Ji[3] * Ji[6] + Ji[4] * Ji[7] + Ji[5] * Ji[8]);
    } else if constexpr (GEOM == GEOM_CONST) {
#pragma unroll
      for (int q = 0; q < 6; ++q) Gc[q] = qp.G0[q];
    }
    const double wij = qp.w[i] * qp.w[j];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double G[6];
      if constexpr (GEOM == GEOM_PER_QPOINT) {
        const double* gp = ga.G + cid * (int64_t)(6 * N * NN) + gq<N>(i, j, k);
#pragma unroll
        for (int q = 0; q < 6; ++q) G[q] = __ldg(gp + q * N * NN);
      } else {
        const double wq = wij * qp.w[k];
#pragma unroll
        for (int q = 0; q < 6; ++q) G[q] = wq * Gc[q];
      }
      const double tx = G[0] * gx[k] + G[3] * gy[k] + G[4] * gz[k];
      const double ty = G[3] * gx[k] + G[1] * gy[k] + G[5] * gz[k];
      const double tz = G[4] * gx[k] + G[5] * gy[k] + G[2] * gz[k];
      gx[k] = tx;
      gy[k] = ty;
      gz[k] = tz;
    }
    eo_apply<N, 1>(qp.St, gx, c1);
    eo_apply<N, 1>(qp.St, gy, c2);
    eo_apply<N, -1>(qp.Dt, gz, c3);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      C1[(k * N + j) * P + i] = c1[k];
      C2[(k * N + j) * P + i] = c2[k];
      C3[(k * N + j) * P + i] = c3[k];
    }
  }
  __syncthreads();
  // ---------------------------------------------------------------- YT
  if (active) {
    const int i = line % N, k = line / N;
    double d1[N], d2[N], d3[N], e[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      d1[j] = C1[(k * N + j) * P + i];
      d2[j] = C2[(k * N + j) * P + i];
      d3[j] = C3[(k * N + j) * P + i];
    }
    eo_apply<N, 1>(qp.St, d1, e);
#pragma unroll
    for (int j = 0; j < N; ++j) A[(k * N + j) * P + i] = e[j];
    eo_apply<N, -1>(qp.Dt, d2, e);
    eo_apply_add<N, 1>(qp.St, d3, e);
#pragma unroll
    for (int j = 0; j < N; ++j) B[(k * N + j) * P + i] = e[j];
  }
  __syncthreads();
  // ---------------------------------------------------------------- XT + face injection
  double res[N];
  const int xj = line % N, xk = line / N;
  if (active) {
    double e1[N], e2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      e1[i] = A[(xk * N + xj) * P + i];
      e2[i] = B[(xk * N + xj) * P + i];
    }
    eo_apply<N, -1>(qp.Dt, e1, res);
    eo_apply_add<N, 1>(qp.St, e2, res);
    // x-faces: layers i near the face, point (a=j, b=k)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double* rf = R + ((0 + s) * 2 * N + xk) * P + xj;
      const double r0 = rf[0], r1 = rf[N * P];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int L = s ? N - NL + l : l;
        res[L] += qp.sf[s][l] * r0 + qp.df[s][l] * r1;
      }
    }
    // y-faces: rows j near the face, points (a=i, b=k)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int L = s ? N - NL + l : l;
        if (xj == L) {
          const double* rf = R + ((2 + s) * 2 * N + xk) * P;
          const double cs = qp.sf[s][l], cd = qp.df[s][l];
#pragma unroll
          for (int i = 0; i < N; ++i) res[i] += cs * rf[i] + cd * rf[N * P + i];
        }
      }
    }
    // z-faces: planes k near the face, points (a=i, b=j)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int L = s ? N - NL + l : l;
        if (xk == L) {
          const double* rf = R + ((4 + s) * 2 * N + xj) * P;
          const double cs = qp.sf[s][l], cd = qp.df[s][l];
#pragma unroll
          for (int i = 0; i < N; ++i) res[i] += cs * rf[i] + cd * rf[N * P + i];
        }
      }
    }
  }
  const int64_t xbase = cid * (int64_t)(N * NN) + (xk * N + xj) * N;   // + i

  if constexpr (MODE == KMODE_APPLY) {
    // stage the result for a coalesced store
    if (active) {
#pragma unroll
      for (int i = 0; i < N; ++i) C1[(xk * N + xj) * P + i] = res[i];
    }
    __syncthreads();
    if (active) {
      double* out = y + cid * (int64_t)(N * NN);
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const int e = line + r * NN;
        out[e] = C1[(e / N) * P + e % N];
      }
    }
    return;
  } else {
    if (active) {
#pragma unroll
      for (int i = 0; i < N; ++i) res[i] = __ldg(ch.b + xbase + i) - res[i];
    }
    if constexpr (MODE == KMODE_CHEBY_GL) {
      if (active) {  // T^{-T} along x
        double o[N];
        eo_apply<N, 1>(qp.TiT, res, o);
#pragma unroll
        for (int i = 0; i < N; ++i) C1[(xk * N + xj) * P + i] = o[i];
      }
      __syncthreads();
      if (active) {  // T^{-T} along y
        const int i = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = C1[(k * N + j) * P + i];
        eo_apply<N, 1>(qp.TiT, r, o);
#pragma unroll
        for (int j = 0; j < N; ++j) C1[(k * N + j) * P + i] = o[j];
      }
      __syncthreads();
      if (active) {  // T^{-T} along z, diagonal, T^{-1} along z
        const int i = line % N, j = line / N;
        double r[N], o[N];
#pragma unroll
        for (int k = 0; k < N; ++k) r[k] = C1[(k * N + j) * P + i];
        eo_apply<N, 1>(qp.TiT, r, o);
        const double* dv = ch.dinv + cid * (int64_t)(N * NN) + j * N + i;
#pragma unroll
        for (int k = 0; k < N; ++k) o[k] *= __ldg(dv + k * NN);
        eo_apply<N, 1>(qp.Ti, o, r);
#pragma unroll
        for (int k = 0; k < N; ++k) C1[(k * N + j) * P + i] = r[k];
      }
      __syncthreads();
      if (active) {  // T^{-1} along y
        const int i = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = C1[(k * N + j) * P + i];
        eo_apply<N, 1>(qp.Ti, r, o);
#pragma unroll
        for (int j = 0; j < N; ++j) C1[(k * N + j) * P + i] = o[j];
      }
      __syncthreads();
      if (active) {  // T^{-1} along x
        double r[N];
#pragma unroll
        for (int i = 0; i < N; ++i) r[i] = C1[(xk * N + xj) * P + i];
        eo_apply<N, 1>(qp.Ti, r, res);
      }
    } else {
      if (active) {
#pragma unroll
        for (int i = 0; i < N; ++i) res[i] *= __ldg(ch.dinv + xbase + i);
      }
    }
    if (active) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int64_t gi = xbase + i;
        const double uj = U[(xk * N + xj) * P + i];
        double v = fma(ch.c_z, res[i], uj);
        if (!ch.first) v = fma(ch.c_prev, uj - ch.u_prev[gi], v);
        ch.u_next[gi] = v;
      }
    }
  }
}


// Diagonal of the operator for the basis given by `t` (GL for the GL-Jacobi inner
// preconditioner of Eq. (12), or the working basis for point Jacobi), any geometry:
//   a(l_i, l_i) = sum_q grad l_i . G_q grad l_i
//               + sum_faces sum_pts m_F (sigma dA l_i^2 - l_i (dA J^-1 n_K) . grad_xi l_i),
// m_F = 1 on interior faces (neighbour trial function zero), 2 on mirror faces
// (u+ = -u-, grad u+ = grad u-), from Eq. (1) with u = l_i on K only.
template <int N, int GEOM>
__global__ void k_diag_general(const __grid_constant__ DiagTables t, const __grid_constant__ QuadParams qp,
                               const __grid_constant__ GeomArgs ga, const __grid_constant__ GridArgs g,
                               int invert, double* __restrict__ out) {
  constexpr int NN = N * N, N3 = N * NN;
  const int plane = g.Nx * g.Ny;
  const int64_t total = (int64_t)plane * g.nz * N3;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < total;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cid = gi / N3;
    const int r = (int)(gi % N3);
    const int ii[3] = {r % N, (r / N) % N, r / NN};
    const int czl = (int)(cid / plane);
    const int crem = (int)(cid - (int64_t)czl * plane);
    const int cy = crem / g.Nx, cx = crem - cy * g.Nx;
    double acc = 0.0;
    double Gc[6];
    if constexpr (GEOM == GEOM_PER_CELL) {
      const double* jo = ga.jinv + ((int64_t)(czl + 1) * plane + (int64_t)cy * g.Nx + cx) * 10;
      double Ji[9];
      for (int q = 0; q < 9; ++q) Ji[q] = jo[q];
      const double dj = jo[9];
      Gc[0] = dj * (Ji[0] * Ji[0] + Ji[1] * Ji[1] + Ji[2] * Ji[2]);
      Gc[1] = dj * (Ji[3] * Ji[3] + Ji[4] * Ji[4] + Ji[5] * Ji[5]);
      Gc[2] = dj * (Ji[6] * Ji[6] + Ji[7] * Ji[7] + Ji[8] * Ji[8]);
      Gc[3] = dj * (Ji[0] * Ji[3] + Ji[1] * Ji[4] + Ji[2] * Ji[5]);
      Gc[4] = dj * (Ji[0] * Ji[6] + Ji[1] * Ji[7] + Ji[2] * Ji[8]);
      Gc[5] = dj * (Ji[3] * Ji[6] + Ji[4] * Ji[7] + Ji[5] * Ji[8]);
    } else {
      for (int q = 0; q < 6; ++q) Gc[q] = qp.G0[q];
    }
    for (int q = 0; q < N3; ++q) {
      const int q0 = q % N, q1 = (q / N) % N, q2 = q / NN;
      const double s0 = t.S[q0 * N + ii[0]], s1 = t.S[q1 * N + ii[1]], s2 = t.S[q2 * N + ii[2]];
      const double g0 = t.DS[q0 * N + ii[0]] * s1 * s2;
      const double g1 = s0 * t.DS[q1 * N + ii[1]] * s2;
      const double g2 = s0 * s1 * t.DS[q2 * N + ii[2]];
      double G[6];
      if constexpr (GEOM == GEOM_PER_QPOINT) {
        for (int m = 0; m < 6; ++m) G[m] = ga.G[cid * (6 * N3) + m * N3 + gq<N>(q0, q1, q2)];
      } else {
        const double w = qp.w[q0] * qp.w[q1] * qp.w[q2];
        for (int m = 0; m < 6; ++m) G[m] = w * Gc[m];
      }
      acc += G[0] * g0 * g0 + G[1] * g1 * g1 + G[2] * g2 * g2 +
             2.0 * (G[3] * g0 * g1 + G[4] * g0 * g2 + G[5] * g1 * g2);
    }
    for (int f = 0; f < 6; ++f) {
      const int d = f >> 1, s = f & 1;
      const double v = t.v[s][ii[d]], dv = t.d[s][ii[d]];
      const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
      const int cd = d == 0 ? cx : (d == 1 ? cy : czl);
      const int Nd = d == 0 ? g.Nx : (d == 1 ? g.Ny : g.nz);
      const int nb = cd + (s ? 1 : -1);
      bool mirror = false, self = false;
      if (nb < 0 || nb >= Nd) {
        if (d < 2) mirror = g.bc[d] != DG_BC_PERIODIC;
        else mirror = (s == 0 ? g.zlo : g.zhi) == ZSRC_MIRROR;
        // periodic with one cell in this direction: the neighbour is the cell itself, so
        // the trial function l_i is also nonzero on the other side of the face
        self = !mirror && Nd == 1 && (d < 2 || (s == 0 ? g.zlo : g.zhi) == ZSRC_LOCAL);
      }
      const double vp = self ? t.v[1 - s][ii[d]] : 0.0, dvp = self ? t.d[1 - s][ii[d]] : 0.0;
      if (v == 0.0 && dv == 0.0 && vp == 0.0 && dvp == 0.0) continue;
      for (int qb = 0; qb < N; ++qb)
        for (int qa = 0; qa < N; ++qa) {
          double ckm[3], ckp[3], sdA;
          face_geom<N, GEOM>(qp, ga, g, cid, cx, cy, czl, f, qa, qb, ckm, ckp, sdA, mirror);
          const double sa = t.S[qa * N + ii[t1]], sb = t.S[qb * N + ii[t2]];
          const double da = t.DS[qa * N + ii[t1]], db = t.DS[qb * N + ii[t2]];
          // own side (test and trial): value and reference gradient of l_i at the face point
          const double l = v * sa * sb;
          double gr[3];
          gr[d] = dv * sa * sb;
          gr[t1] = v * da * sb;
          gr[t2] = v * sa * db;
          const double cg = ckm[0] * gr[0] + ckm[1] * gr[1] + ckm[2] * gr[2];
          // other side of the face (Eq. (1)): 0 (interior: l_i lives on K only), the mirror
          // ghost (-l, grad l), or l_i itself at the opposite face (self-periodic)
          double up, cgp;
          if (mirror) {
            up = -l;
            cgp = cg;
          } else if (self) {
            up = vp * sa * sb;
            double grp[3];
            grp[d] = dvp * sa * sb;
            grp[t1] = vp * da * sb;
            grp[t2] = vp * sa * db;
            cgp = ckp[0] * grp[0] + ckp[1] * grp[1] + ckp[2] * grp[2];
          } else {
            up = 0.0;
            cgp = 0.0;
          }
          const double jump = l - up;
          acc += sdA * jump * l - 0.5 * l * (cg + cgp) - 0.5 * cg * jump;
        }
    }
    out[gi] = invert ? 1.0 / acc : acc;
  }
}

template <int N>
cudaError_t launch_diag_n(int geom, const DiagTables& t, const QuadParams& qp, const GeomArgs& ga,
                          const GridArgs& g, int invert, double* out, cudaStream_t s) {
  const int grid = 148 * 8, bs = 128;
  switch (geom) {
    case GEOM_CONST: k_diag_general<N, GEOM_CONST><<<grid, bs, 0, s>>>(t, qp, ga, g, invert, out); break;
    case GEOM_PER_CELL: k_diag_general<N, GEOM_PER_CELL><<<grid, bs, 0, s>>>(t, qp, ga, g, invert, out); break;
    case GEOM_PER_QPOINT: k_diag_general<N, GEOM_PER_QPOINT><<<grid, bs, 0, s>>>(t, qp, ga, g, invert, out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int N, int NL>
constexpr int qcells_per_block() {
  constexpr int byT = (192 + N * N - 1) / (N * N);
  constexpr int byS = (110 * 1024) / (QLayout<N, NL>::PER_CELL * 8);
  constexpr int c = byT < byS ? byT : byS;
  return c < 1 ? 1 : c;
}

template <int N, int NL, int GEOM, int MODE>
cudaError_t launch_t(const QuadParams& qp, const GeomArgs& ga, const GridArgs& g, const double* u,
                     double* y, const ChebyArgs& ch, cudaStream_t s) {
  constexpr int CPB = qcells_per_block<N, NL>();
  const int64_t ncells = (int64_t)(g.zend - g.zbeg) * g.Nx * g.Ny;
  if (ncells <= 0) return cudaSuccess;
  const int64_t blocks = (ncells + CPB - 1) / CPB;
  const size_t smem = (size_t)CPB * QLayout<N, NL>::PER_CELL * sizeof(double);
  auto kern = k_quad<N, NL, CPB, GEOM, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)blocks, CPB * N * N, smem, s>>>(qp, ga, g, u, y, ch);
  return cudaGetLastError();
}

template <int N, int NL, int GEOM>
cudaError_t launch_mode(int mode, const QuadParams& qp, const GeomArgs& ga, const GridArgs& g,
                        const double* u, double* y, const ChebyArgs& ch, cudaStream_t s) {
  switch (mode) {
    case KMODE_APPLY: return launch_t<N, NL, GEOM, KMODE_APPLY>(qp, ga, g, u, y, ch, s);
    case KMODE_CHEBY_GL: return launch_t<N, NL, GEOM, KMODE_CHEBY_GL>(qp, ga, g, u, y, ch, s);
    case KMODE_CHEBY_PJ: return launch_t<N, NL, GEOM, KMODE_CHEBY_PJ>(qp, ga, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

template <int N, int NL>
cudaError_t launch_geom(int geom, int mode, const QuadParams& qp, const GeomArgs& ga, const GridArgs& g,
                        const double* u, double* y, const ChebyArgs& ch, cudaStream_t s) {
  switch (geom) {
    case GEOM_CONST: return launch_mode<N, NL, GEOM_CONST>(mode, qp, ga, g, u, y, ch, s);
    case GEOM_PER_CELL: return launch_mode<N, NL, GEOM_PER_CELL>(mode, qp, ga, g, u, y, ch, s);
    case GEOM_PER_QPOINT: return launch_mode<N, NL, GEOM_PER_QPOINT>(mode, qp, ga, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

template <int N>
cudaError_t launch_nl(int NL, int geom, int mode, const QuadParams& qp, const GeomArgs& ga,
                      const GridArgs& g, const double* u, double* y, const ChebyArgs& ch, cudaStream_t s) {
  if (NL == 2 && N > 2) return launch_geom<N, 2>(geom, mode, qp, ga, g, u, y, ch, s);
  if (NL == N) return launch_geom<N, N>(geom, mode, qp, ga, g, u, y, ch, s);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_diag_general(int n, int geom, const DiagTables& t, const QuadParams& qp,
                                const GeomArgs& ga, const GridArgs& g, int invert, double* out,
                                cudaStream_t s) {
  switch (n) {
    case 2: return launch_diag_n<2>(geom, t, qp, ga, g, invert, out, s);
    case 3: return launch_diag_n<3>(geom, t, qp, ga, g, invert, out, s);
    case 4: return launch_diag_n<4>(geom, t, qp, ga, g, invert, out, s);
    case 5: return launch_diag_n<5>(geom, t, qp, ga, g, invert, out, s);
    case 6: return launch_diag_n<6>(geom, t, qp, ga, g, invert, out, s);
    case 7: return launch_diag_n<7>(geom, t, qp, ga, g, invert, out, s);
    case 8: return launch_diag_n<8>(geom, t, qp, ga, g, invert, out, s);
    case 9: return launch_diag_n<9>(geom, t, qp, ga, g, invert, out, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_quad(int n, int NL, int geom, int mode, const QuadParams& qp, const GeomArgs& ga,
                        const GridArgs& g, const double* u, double* y, const ChebyArgs& ch,
                        cudaStream_t s) {
  switch (n) {
    case 2: return launch_nl<2>(NL, geom, mode, qp, ga, g, u, y, ch, s);
    case 3: return launch_nl<3>(NL, geom, mode, qp, ga, g, u, y, ch, s);
    case 4: return launch_nl<4>(NL, geom, mode, qp, ga, g, u, y, ch, s);
    case 5: return launch_nl<5>(NL, geom, mode, qp, ga, g, u, y, ch, s);
    case 6: return launch_nl<6>(NL, geom, mode, qp, ga, g, u, y, ch, s);
    case 7: return launch_nl<7>(NL, geom, mode, qp, ga, g, u, y, ch, s);
    case 8: return launch_nl<8>(NL, geom, mode, qp, ga, g, u, y, ch, s);
    case 9: return launch_nl<9>(NL, geom, mode, qp, ga, g, u, y, ch, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dgb
