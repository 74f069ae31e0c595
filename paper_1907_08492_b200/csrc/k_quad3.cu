// General quadrature SIPG kernel, z-first schedule with the faces folded into the line
// stages (k_quad3).  Same operator as k_quad.cu — the paper's formulation by quadrature
// with sum factorisation (Eqs. (3)-(5)), element-wise face arrangement
// (PAPER.md:323-330), Hermite-like face access (only NL layers of each neighbour,
// PAPER.md:753-762) — for geometry stored as a constant merged tensor or per quadrature
// point (DG_GEOM_CONSTANT / DG_GEOM_PER_QPOINT, where the face data dA J^-1 n is single
// valued); per-cell affine geometry stays on k_quad.cu.
//
// Cell term, one thread per 1D line, lines register-resident, smem transposes:
//   Z   a = S_z u, b = DS_z u                          (u read along coalesced z-lines)
//   Y   c1 = S_y a, c2 = DS_y a, c3 = S_y b
//   X   g = (DS_x c1, S_x c2, S_x c3) = grad_xi u at the q-points; t = G_q g;
//       q1 = DS_x^T t_x, q2 = S_x^T t_y, q3 = S_x^T t_z
//   YT  r1 = S_y^T q1 + DS_y^T q2, r2 = S_y^T q3
//   ZT  y = S_z^T r1 + DS_z^T r2                        (written along z-lines)
// Faces (Eq. (1), element-wise, both sides at every face point).  Because c = dA J^-1 n
// is the same from both sides on these meshes, only the jump and the sum of the two
// sides' traces need interpolating:  jump = u- - u+,  avg = c . (grad u- + grad u+)/2.
//   x-faces: the traces of c1, c2, c3 at the NL layers next to the face are already the
//     face-point values (u, d_y u, d_z u; d_x u via D_f) — flux in registers in stage X
//     and the tests injected into q1..q3 (zero extra sweeps; the cell/face sharing of
//     PAPER.md:318-321).  The neighbour's c fields come from its block slot, or from
//     halo jobs at the block edges.
//   y-faces: traces of a, b along j in stage Y (neighbour: jobs in stage Z apply S_z, DS_z
//     to the trace of its NL layers), x-sweeps + flux + transposed x-sweeps as jobs in
//     stage X, injected into r1, r2 in stage YT.
//   z-faces: traces of u along k in stage Z (neighbour layers read along z-lines), y- and
//     x-sweeps as jobs in stages Y and X, transposed x- and y-sweeps in X and YT, injected
//     in stage ZT.
// Mirror faces: u+ = -u-, grad u+ = grad u- (PAPER.md:172-174), i.e. jump = 2u-, sum = 2 grad u-.
// The fused Chebyshev step continues from ZT: r = b - Au, P^-1 = (T^-1)^{x3} diag^-1 (T^-T)^{x3}
// as z, y, x(diag), y, z and the three-term update of Eq. (11) along the z-lines.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dg_internal.h"

namespace dgb {
namespace {

struct Lay3 {
  int Pj, Pk, CS;
};

#ifndef Q3_GEARLY
#define Q3_GEARLY 0     // 1: the X stage's per-q-point tensors (and x-face geometry) are loaded before the
                        //    Y->X barrier, so their latency overlaps the barrier wait
#endif
#ifndef Q3_JOBPRE
#define Q3_JOBPRE 0     // 1: the y/z-face jobs of stage X load their face geometry before their sweeps
#endif

// per n: cells per block and the two transposition layouts (ZY: z-write / y-read,
// YX: y-write / x-read; the reverse transposes use the same two by symmetry)
template <int N> struct Q3C;
template <> struct Q3C<3> { static constexpr int CPB = 16; static constexpr Lay3 ZY{3, 19, 57}, YX{3, 9, 27}; };
template <> struct Q3C<4> { static constexpr int CPB = 12; static constexpr Lay3 ZY{4, 20, 88}, YX{5, 20, 88}; };
template <> struct Q3C<5> { static constexpr int CPB = 8; static constexpr Lay3 ZY{5, 26, 143}, YX{5, 25, 134}; };
template <> struct Q3C<6> { static constexpr int CPB = 6; static constexpr Lay3 ZY{6, 38, 228}, YX{6, 37, 222}; };
template <> struct Q3C<7> { static constexpr int CPB = 4; static constexpr Lay3 ZY{7, 55, 396}, YX{7, 56, 392}; };
template <> struct Q3C<8> { static constexpr int CPB = 4; static constexpr Lay3 ZY{8, 72, 576}, YX{9, 72, 576}; };
template <> struct Q3C<9> { static constexpr int CPB = 2; static constexpr Lay3 ZY{9, 89, 801}, YX{9, 85, 765}; };

constexpr int imax3(int a, int b) { return a > b ? a : b; }

template <int N, int NL>
struct Q3Layout {
  static constexpr int CPB = Q3C<N>::CPB;
  static constexpr Lay3 ZY = Q3C<N>::ZY, YX = Q3C<N>::YX;
  static constexpr int S = imax3(ZY.CS, YX.CS);
  static constexpr int PG = N | 1;             // face row pitch (odd: spreads banks)
  static constexpr int FP = N * PG;            // one face field (n x n)
  // per-cell strides padded off multiples of 16 doubles (jobs of several cells share a warp)
  static constexpr int pad16(int x) { return (x % 16 == 0) ? x + 4 : x; }
  // FA: (Z->Y) FZ[s][3] + GYn[f][3];  (X->YT) PY[f][3] + QZm[s][3]
  static constexpr int FAC = pad16(12 * FP);
  // FB: (Y->X) FY[f][4] + FZm[s][4];  (YT->ZT) QZo[s][2]
  static constexpr int FBC = pad16(16 * FP);
  // x-halo: per block edge h: HZ[3] (Z->Y) and HXo[4] (Y->X)
  static constexpr int HXC = 7 * FP;
  static constexpr int doubles() { return CPB * (3 * S + FAC + FBC) + 2 * HXC; }
  static constexpr int bytes() { return doubles() * 8; }
};

__device__ __forceinline__ int at(const Lay3& L, int i, int j, int k) { return i + j * L.Pj + k * L.Pk; }

// register cap so that the smem-limited number of resident blocks (at most 2) fits
#ifndef Q3_MAXREG
#define Q3_MAXREG 0     // > 0: register cap override (e.g. 255: one block per SM, room for early loads)
#endif
template <int N, int NL>
constexpr int q3_maxreg_auto();
template <int N, int NL>
constexpr int q3_maxreg() {
  return Q3_MAXREG > 0 ? Q3_MAXREG : q3_maxreg_auto<N, NL>();
}
template <int N, int NL>
constexpr int q3_maxreg_auto() {
  constexpr int b0 = (227 * 1024) / Q3Layout<N, NL>::bytes();
  constexpr int b = b0 < 1 ? 1 : (b0 > 2 ? 2 : b0);
  constexpr int warps = (Q3Layout<N, NL>::CPB * N * N + 31) / 32;
  // 16K registers per SM sub-partition; a block's warps are spread over the four
  constexpr int per_smsp = (b * warps + 3) / 4;
  constexpr int r = (16384 / (per_smsp * 32)) / 8 * 8;
  return r > 255 ? 255 : r;
}

__device__ __forceinline__ void l2_prefetch_q3(const double* p, int64_t ndoubles, int tid, int bt) {
  const char* c = reinterpret_cast<const char*>(p);
  for (int64_t o = (int64_t)tid * 128; o < ndoubles * 8; o += (int64_t)bt * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
}

// Face geometry at face point (qa, qb) of face (d, s) of cell (cx, cy, czl):
// c = dA J^-1 n_K (outward) and sigma dA.
template <int N, int GEOM>
__device__ __forceinline__ void fgeom(const QuadParams& qp, const GeomArgs& ga, const GridArgs& g, int cx,
                                      int cy, int czl, int d, int s, int qa, int qb, double (&c)[3],
                                      double& sdA) {
  const double nu = s ? 1.0 : -1.0;
  if constexpr (GEOM == GEOM_CONST) {
    const double ww = qp.w[qa] * qp.w[qb];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = nu * ww * qp.cw0[d][k];
    sdA = ww * qp.sdA0[d];
  } else {
    int64_t fid;
    if (d == 0) fid = ((int64_t)czl * g.Ny + cy) * (g.Nx + 1) + cx + s;
    else if (d == 1) fid = ((int64_t)czl * (g.Ny + 1) + cy + s) * g.Nx + cx;
    else fid = ((int64_t)(czl + s) * g.Ny + cy) * g.Nx + cx;
    const double* fd = ga.face[d] + fid * (4 * N * N) + qb * N + qa;
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = nu * __ldg(fd + k * N * N);
    sdA = __ldg(fd + 3 * N * N);
  }
}

// flux at one face point from the interpolated jump and gradient sum (reference
// components: normal n = axis d, tangential a, b) -> the four test values
//   rv = sigma dA jump - c.(sum)/2,  (rn, ra, rb) = -jump/2 (c_d, c_a, c_b)
__device__ __forceinline__ void flux(const double (&c)[3], double sdA, int d, double jump, double sn,
                                     double sa, double sb, double& rv, double& rn, double& ra, double& rb) {
  const int ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
  const double cn = d == 0 ? c[0] : (d == 1 ? c[1] : c[2]);
  const double ca = ta == 0 ? c[0] : c[1];
  const double cb = tb == 1 ? c[1] : c[2];
  rv = sdA * jump - 0.5 * (cn * sn + ca * sa + cb * sb);
  const double hj = -0.5 * jump;
  rn = hj * cn;
  ra = hj * ca;
  rb = hj * cb;
}

template <int N, int S>
__device__ __forceinline__ void ld_line(const double* p, int stride, double (&v)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = p[k * stride];
}
template <int N>
__device__ __forceinline__ void st_line(double* p, int stride, const double (&v)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) p[k * stride] = v[k];
}

template <int N, int NL, int GEOM, int MODE>
__global__ void __maxnreg__((q3_maxreg<N, NL>()))
k_quad3(const __grid_constant__ QuadParams qp, const __grid_constant__ GeomArgs ga,
        const __grid_constant__ GridArgs g, const double* __restrict__ u, double* __restrict__ y,
        const __grid_constant__ ChebyArgs ch) {
  using Lay = Q3Layout<N, NL>;
  constexpr int CPB = Lay::CPB, NN = N * N, N3 = N * NN, PG = Lay::PG, FP = Lay::FP;
  constexpr Lay3 LZY = Lay::ZY, LYX = Lay::YX;
  constexpr int BT = CPB * NN;
  extern __shared__ double smem[];
  double* R1 = smem;
  double* R2 = R1 + CPB * Lay::S;
  double* R3 = R2 + CPB * Lay::S;
  double* FAb = R3 + CPB * Lay::S;
  double* FBb = FAb + CPB * Lay::FAC;
  double* HXb = FBb + CPB * Lay::FBC;   // [h][HZ 3 | HXo 4][FP]

  const int ta = threadIdx.x, cslot = threadIdx.y / N, tb = threadIdx.y - cslot * N;
  const int btid = threadIdx.x + N * threadIdx.y;
  const int cx0 = blockIdx.x * CPB;
  const int cy = blockIdx.y;
  const int cz = g.zbeg + blockIdx.z;
  const int ncell = g.Nx - cx0 < CPB ? g.Nx - cx0 : CPB;
  const bool active = cslot < ncell;
  const int cx = cx0 + cslot;
  const int64_t plane = (int64_t)g.Nx * g.Ny;
  const int64_t rowcell = ((int64_t)cz * g.Ny + cy) * g.Nx;
  const int64_t cid = rowcell + cx;
  double* FA = FAb + cslot * Lay::FAC;
  double* FB = FBb + cslot * Lay::FBC;

  // neighbours
  const bool xper = g.bc[0] == DG_BC_PERIODIC;
  int h0 = cx0 > 0 ? cx0 - 1 : (xper ? g.Nx - 1 : -1);
  int h1 = cx0 + ncell < g.Nx ? cx0 + ncell : (xper ? 0 : -1);
  if (ncell == g.Nx) h0 = h1 = -1;   // whole row in the block: periodic wrap inside
  const bool yper = g.bc[1] == DG_BC_PERIODIC;
  const int ym_row = cy > 0 ? cy - 1 : (yper ? g.Ny - 1 : -1);
  const int yp_row = cy + 1 < g.Ny ? cy + 1 : (yper ? 0 : -1);
  int zsrc[2];
  const double* zbase[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int nz = cz + (s ? 1 : -1);
    if (nz >= 0 && nz < g.nz) {
      zsrc[s] = ZSRC_LOCAL;
      zbase[s] = u + (cid + (s ? plane : -plane)) * N3;
    } else {
      zsrc[s] = s ? g.zhi : g.zlo;
      zbase[s] = u + (cid + (s ? -(int64_t)(g.nz - 1) : (int64_t)(g.nz - 1)) * plane) * N3;
      if (zsrc[s] == ZSRC_HALO)
        zbase[s] = (s ? g.halo_hi : g.halo_lo) + ((int64_t)cy * g.Nx + cx) * (NL * NN) -
                   (s ? 0 : (N - NL) * NN);
    }
  }
  // L2 prefetch of this block's q-point tensors and of the next plane's tile
  if (GEOM == GEOM_PER_QPOINT && g.l2pf) {
    l2_prefetch_q3(ga.G + (rowcell + cx0) * (6 * N3), (int64_t)ncell * 6 * N3, btid, BT);
    if (cz + 1 < g.zend) {
      l2_prefetch_q3(ga.G + (rowcell + plane + cx0) * (6 * N3), (int64_t)ncell * 6 * N3, btid, BT);
      l2_prefetch_q3(u + (rowcell + plane + cx0) * N3, (int64_t)ncell * N3, btid, BT);
    }
  }

  // ================================================================ Z
  const int zi = ta, zj = tb;
  if (active) {
    double uz[N];
#pragma unroll
    for (int k = 0; k < N; ++k) uz[k] = __ldg(u + cid * N3 + k * NN + zj * N + zi);
    double a[N], b[N];
    const EOSplit<N> su = eo_split<N>(uz);
    eo_mul<N, 1, false>(qp.S, su, a);
    eo_mul<N, -1, false>(qp.D, su, b);
    st_line<N>(R1 + cslot * LZY.CS + at(LZY, zi, zj, 0), LZY.Pk, a);
    st_line<N>(R2 + cslot * LZY.CS + at(LZY, zi, zj, 0), LZY.Pk, b);
    // z-face traces: jump, value sum, normal-derivative sum -> FZ[s][3][j][i]
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      double V = 0.0, D = 0.0;
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int L = s ? N - NL + l : l;
        V = fma(qp.sf[s][l], uz[L], V);
        D = fma(qp.df[s][l], uz[L], D);
      }
      double J, Sv, Sd;
      if (zsrc[s] == ZSRC_MIRROR) {
        J = 2.0 * V;
        Sv = 2.0 * V;
        Sd = 2.0 * D;
      } else {
        double Vn = 0.0, Dn = 0.0;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int Ln = s ? l : N - NL + l;
          const double v = __ldg(zbase[s] + Ln * NN + zj * N + zi);
          Vn = fma(qp.sfn[s][l], v, Vn);
          Dn = fma(qp.dfn[s][l], v, Dn);
        }
        J = V - Vn;
        Sv = V + Vn;
        Sd = D + Dn;
      }
      double* fz = FA + (s * 3) * FP + zj * PG + zi;
      fz[0 * FP] = J;
      fz[1 * FP] = Sv;
      fz[2 * FP] = Sd;
    }
  }
  // jobs: (a) y-neighbour traces (cell, f, i): w = sum_l sfn v_l, dn = sum_l dfn v_l over the
  //           neighbour's NL layers along k -> GYn[f][3][qz][i] = (S_z w, DS_z w, S_z dn)
  //       (b) x-halo traces (h, j): same along k for the NL i-layers of the edge neighbour
  //           -> HZ[h][3][qz][j]
  {
    constexpr int NYJ = 2 * N;
    const int nyj = ncell * NYJ;
    const int nh0 = h0 >= 0 ? N : 0, nh1 = h1 >= 0 ? N : 0;
    for (int job = btid; job < nyj + nh0 + nh1; job += BT) {
      const double* src;
      int lstride, f;
      double* dst;
      if (job < nyj) {
        const int c = job / NYJ, jj = job - c * NYJ;
        f = jj / N;
        const int i = jj - f * N;
        const int nrow = f ? yp_row : ym_row;
        if (nrow < 0) continue;
        src = u + (((int64_t)cz * g.Ny + nrow) * g.Nx + cx0 + c) * N3 + i;   // + k*NN + j*N
        lstride = N;
        dst = FAb + c * Lay::FAC + (6 + f * 3) * FP + i;                    // + field*FP + qz*PG
      } else {
        const int hj = job - nyj;
        const int h = hj < nh0 ? 0 : 1;
        const int j = hj - (h ? nh0 : 0);
        f = h;   // face side of the edge cell: h = 0 -> s = 0 face, its neighbour's layers N-NL..
        src = u + (rowcell + (h ? h1 : h0)) * N3 + j * N;                     // + k*NN + i
        lstride = 1;
        dst = HXb + h * Lay::HXC + j;                                         // + field*FP + qz*PG
      }
      double w[N], dn[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double ws = 0.0, ds = 0.0;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int Ln = f ? l : N - NL + l;
          const double v = __ldg(src + k * NN + Ln * lstride);
          ws = fma(qp.sfn[f][l], v, ws);
          ds = fma(qp.dfn[f][l], v, ds);
        }
        w[k] = ws;
        dn[k] = ds;
      }
      double o[N];
      const EOSplit<N> sw = eo_split<N>(w);
      eo_mul<N, 1, false>(qp.S, sw, o);
      st_line<N>(dst + 0 * FP, PG, o);
      eo_mul<N, -1, false>(qp.D, sw, o);
      st_line<N>(dst + 1 * FP, PG, o);
      eo_apply<N, 1>(qp.S, dn, o);
      st_line<N>(dst + 2 * FP, PG, o);
    }
  }
  __syncthreads();

  // ================================================================ Y
  const int yi = ta, yq = tb;   // y-line (i, qz)
  {
    double c1[N], c2[N], c3[N];
    if (active) {
      double a[N], b[N];
      ld_line<N, 0>(R1 + cslot * LZY.CS + at(LZY, yi, 0, yq), LZY.Pj, a);
      ld_line<N, 0>(R2 + cslot * LZY.CS + at(LZY, yi, 0, yq), LZY.Pj, b);
      const EOSplit<N> sa = eo_split<N>(a);
      eo_mul<N, 1, false>(qp.S, sa, c1);
      eo_mul<N, -1, false>(qp.D, sa, c2);
      eo_apply<N, 1>(qp.S, b, c3);
      // y-face traces -> FY[f][4][qz][i]: jump, sum(a) (-> d_x), sum(b) (= d_z), sum(D_f a) (= d_y)
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        double Va = 0.0, Da = 0.0, Vb = 0.0;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int L = f ? N - NL + l : l;
          Va = fma(qp.sf[f][l], a[L], Va);
          Da = fma(qp.df[f][l], a[L], Da);
          Vb = fma(qp.sf[f][l], b[L], Vb);
        }
        double J, Sa, Sb, Sd;
        if ((f ? yp_row : ym_row) < 0) {
          J = 2.0 * Va;
          Sa = 2.0 * Va;
          Sb = 2.0 * Vb;
          Sd = 2.0 * Da;
        } else {
          const double* gy = FA + (6 + f * 3) * FP + yq * PG + yi;
          const double Vn = gy[0], Vnb = gy[FP], Dn = gy[2 * FP];
          J = Va - Vn;
          Sa = Va + Vn;
          Sb = Vb + Vnb;
          Sd = Da + Dn;
        }
        double* fy = FB + (f * 4) * FP + yq * PG + yi;
        fy[0 * FP] = J;
        fy[1 * FP] = Sa;
        fy[2 * FP] = Sb;
        fy[3 * FP] = Sd;
      }
    }
    // jobs: z-face y-sweeps (cell, s, i): FZ[s][J, Sv, Sd][j][i] ->
    //   FZm[s][4][qy][i] = (S_y J, DS_y Sv, S_y Sv, S_y Sd);  x-halo y-sweeps (h, qz):
    //   HZ[h][3][qz][j] -> HXo[h][4][qz][qy] = (S_y w (u+), S_y dn (d_x u+), DS_y w (d_y u+), S_y DS_z w (d_z u+))
    {
      constexpr int NZJ = 2 * N;
      const int nzj = ncell * NZJ;
      const int nh0 = h0 >= 0 ? N : 0, nh1 = h1 >= 0 ? N : 0;
      for (int job = btid; job < nzj + nh0 + nh1; job += BT) {
        if (job < nzj) {
          const int c = job / NZJ, jj = job - c * NZJ;
          const int s = jj / N, i = jj - s * N;
          const double* fz = FAb + c * Lay::FAC + (s * 3) * FP + i;
          double* fm = FBb + c * Lay::FBC + (8 + s * 4) * FP + i;
          double v[N], o[N];
          ld_line<N, 0>(fz + 0 * FP, PG, v);
          eo_apply<N, 1>(qp.S, v, o);
          st_line<N>(fm + 0 * FP, PG, o);
          ld_line<N, 0>(fz + 1 * FP, PG, v);
          const EOSplit<N> sv = eo_split<N>(v);
          eo_mul<N, -1, false>(qp.D, sv, o);
          st_line<N>(fm + 1 * FP, PG, o);
          eo_mul<N, 1, false>(qp.S, sv, o);
          st_line<N>(fm + 2 * FP, PG, o);
          ld_line<N, 0>(fz + 2 * FP, PG, v);
          eo_apply<N, 1>(qp.S, v, o);
          st_line<N>(fm + 3 * FP, PG, o);
        } else {
          const int hj = job - nzj;
          const int h = hj < nh0 ? 0 : 1;
          const int q = hj - (h ? nh0 : 0);   // qz
          const double* hz = HXb + h * Lay::HXC + q * PG;
          double* ho = HXb + h * Lay::HXC + 3 * FP + q * PG;
          double v[N], o[N];
          ld_line<N, 0>(hz + 0 * FP, 1, v);       // S_z w along j
          const EOSplit<N> sv = eo_split<N>(v);
          eo_mul<N, 1, false>(qp.S, sv, o);
          st_line<N>(ho + 0 * FP, 1, o);          // u+
          eo_mul<N, -1, false>(qp.D, sv, o);
          st_line<N>(ho + 2 * FP, 1, o);          // d_y u+
          ld_line<N, 0>(hz + 2 * FP, 1, v);       // S_z dn
          eo_apply<N, 1>(qp.S, v, o);
          st_line<N>(ho + 1 * FP, 1, o);          // d_x u+ (normal)
          ld_line<N, 0>(hz + 1 * FP, 1, v);       // DS_z w
          eo_apply<N, 1>(qp.S, v, o);
          st_line<N>(ho + 3 * FP, 1, o);          // d_z u+
        }
      }
    }
    __syncthreads();   // a, b fully read: R1..R3 take c1..c3
    if (active) {
      st_line<N>(R1 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, c1);
      st_line<N>(R2 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, c2);
      st_line<N>(R3 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, c3);
    }
  }
  const int xq1 = ta, xq2 = tb;   // x-line (qy, qz)
  constexpr bool kGE = Q3_GEARLY && GEOM == GEOM_PER_QPOINT;
  double Gl[GEOM == GEOM_PER_QPOINT ? 6 : 1][N];
  double xcv[kGE ? 2 : 1][3], xsd[kGE ? 2 : 1];
  auto load_G = [&]() {
    const double* Gp = ga.G + cid * (6 * N3) + gq<N>(0, xq1, xq2);
#pragma unroll
    for (int m = 0; m < 6; ++m) {
#pragma unroll
      for (int k = 0; k < N; ++k) Gl[m][k] = __ldg(Gp + m * N3 + k * N * N);
    }
  };
  if constexpr (kGE) {
    if (active) {
      load_G();
#pragma unroll
      for (int s = 0; s < 2; ++s) fgeom<N, GEOM>(qp, ga, g, cx, cy, cz, 0, s, xq1, xq2, xcv[s], xsd[s]);
    }
  }
  __syncthreads();

  // ================================================================ X (+ X^T)
  {
    double q1[N], q2[N], q3[N];
    if (active) {
      double c1[N], c2[N], c3[N];
      ld_line<N, 0>(R1 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, c1);
      ld_line<N, 0>(R2 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, c2);
      ld_line<N, 0>(R3 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, c3);
      // x-face traces first (the c fields die after the interpolation below):
      //   jump, and the sums of d_x (normal), d_y, d_z of both sides
      double xj[2], xsn[2], xsa[2], xsb[2];
      const bool wrap = xper && ncell == g.Nx;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double um = 0.0, gn = 0.0, gya = 0.0, gzb = 0.0;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int L = s ? N - NL + l : l;
          um = fma(qp.sf[s][l], c1[L], um);
          gn = fma(qp.df[s][l], c1[L], gn);
          gya = fma(qp.sf[s][l], c2[L], gya);
          gzb = fma(qp.sf[s][l], c3[L], gzb);
        }
        const bool inb = s ? (cslot + 1 < ncell) : (cslot > 0);
        const bool halo = s ? (cslot == ncell - 1 && h1 >= 0) : (cslot == 0 && h0 >= 0);
        double up, gnp, gyp, gzp;
        if (inb || (wrap && !halo)) {
          const int off = inb ? (s ? LYX.CS : -LYX.CS) : (s ? -(ncell - 1) : (ncell - 1)) * LYX.CS;
          up = gnp = gyp = gzp = 0.0;
#pragma unroll
          for (int l = 0; l < NL; ++l) {
            const int Ln = s ? l : N - NL + l;
            const int o = cslot * LYX.CS + off + at(LYX, Ln, xq1, xq2);
            const double n1 = R1[o], n2 = R2[o], n3 = R3[o];
            up = fma(qp.sfn[s][l], n1, up);
            gnp = fma(qp.dfn[s][l], n1, gnp);
            gyp = fma(qp.sfn[s][l], n2, gyp);
            gzp = fma(qp.sfn[s][l], n3, gzp);
          }
        } else if (halo) {
          const double* ho = HXb + s * Lay::HXC + 3 * FP + xq2 * PG + xq1;
          up = ho[0];
          gnp = ho[FP];
          gyp = ho[2 * FP];
          gzp = ho[3 * FP];
        } else {   // mirror
          up = -um;
          gnp = gn;
          gyp = gya;
          gzp = gzb;
        }
        xj[s] = um - up;
        xsn[s] = gn + gnp;
        xsa[s] = gya + gyp;
        xsb[s] = gzb + gzp;
      }
      // q-point: g = grad_xi u, t = G g
      double gx[N], gy[N], gz[N];
      eo_apply<N, -1>(qp.D, c1, gx);
      eo_apply<N, 1>(qp.S, c2, gy);
      eo_apply<N, 1>(qp.S, c3, gz);
      const double wyz = qp.w[xq1] * qp.w[xq2];
      // the x-line's tensors: consecutive lines are consecutive addresses at every position k (gq)
      if constexpr (GEOM == GEOM_PER_QPOINT && !kGE) load_G();
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double G[6];
        if constexpr (GEOM == GEOM_PER_QPOINT) {
#pragma unroll
          for (int m = 0; m < 6; ++m) G[m] = Gl[m][k];
        } else {
          const double wq = wyz * qp.w[k];
#pragma unroll
          for (int m = 0; m < 6; ++m) G[m] = wq * qp.G0[m];
        }
        const double tx = G[0] * gx[k] + G[3] * gy[k] + G[4] * gz[k];
        const double ty = G[3] * gx[k] + G[1] * gy[k] + G[5] * gz[k];
        const double tz = G[4] * gx[k] + G[5] * gy[k] + G[2] * gz[k];
        gx[k] = tx;
        gy[k] = ty;
        gz[k] = tz;
      }
      eo_apply<N, -1>(qp.Dt, gx, q1);
      eo_apply<N, 1>(qp.St, gy, q2);
      eo_apply<N, 1>(qp.St, gz, q3);
      // x-face fluxes, tests injected into q1..q3
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double cvec[3], sdA;
        if constexpr (kGE) {
          cvec[0] = xcv[s][0];
          cvec[1] = xcv[s][1];
          cvec[2] = xcv[s][2];
          sdA = xsd[s];
        } else {
          fgeom<N, GEOM>(qp, ga, g, cx, cy, cz, 0, s, xq1, xq2, cvec, sdA);
        }
        double rv, rn, ra, rb;
        flux(cvec, sdA, 0, xj[s], xsn[s], xsa[s], xsb[s], rv, rn, ra, rb);
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int L = s ? N - NL + l : l;
          q1[L] = fma(qp.sf[s][l], rv, fma(qp.df[s][l], rn, q1[L]));
          q2[L] = fma(qp.sf[s][l], ra, q2[L]);
          q3[L] = fma(qp.sf[s][l], rb, q3[L]);
        }
      }
    }
    // jobs: y-faces (cell, f, qz): FY -> PY[f][3][qz][i];  z-faces (cell, s, qy): FZm -> QZm[s][3][qy][i]
    {
      constexpr int NJ = 4 * N;
      for (int job = btid; job < ncell * NJ; job += BT) {
        const int c = job / NJ, jj = job - c * NJ;
        const int kind = jj / (2 * N);         // 0: y-face, 1: z-face
        const int s = (jj / N) & 1, q = jj % N;
        const int ccx = cx0 + c;
        const int d = kind ? 2 : 1;
        const double* fin = FBb + c * Lay::FBC + (kind * 8 + s * 4) * FP + q * PG;
        double jcv[Q3_JOBPRE ? N : 1][3], jsd[Q3_JOBPRE ? N : 1];
        if constexpr (Q3_JOBPRE) {
#pragma unroll
          for (int qx = 0; qx < N; ++qx) fgeom<N, GEOM>(qp, ga, g, ccx, cy, cz, d, s, qx, q, jcv[qx], jsd[qx]);
        }
        double J[N], Sa[N], Sb[N], Sd[N];
        {
          double v[N];
          ld_line<N, 0>(fin + 0 * FP, 1, v);
          eo_apply<N, 1>(qp.S, v, J);           // jump at (qx, q)
          if (kind == 0) {
            ld_line<N, 0>(fin + 1 * FP, 1, v);
            eo_apply<N, -1>(qp.D, v, Sa);       // sum d_x
            ld_line<N, 0>(fin + 2 * FP, 1, v);
            eo_apply<N, 1>(qp.S, v, Sb);        // sum d_z
            ld_line<N, 0>(fin + 3 * FP, 1, v);
            eo_apply<N, 1>(qp.S, v, Sd);        // sum d_y (normal)
          } else {
            ld_line<N, 0>(fin + 2 * FP, 1, v);  // S_y Sv
            eo_apply<N, -1>(qp.D, v, Sa);       // sum d_x
            ld_line<N, 0>(fin + 1 * FP, 1, v);  // DS_y Sv
            eo_apply<N, 1>(qp.S, v, Sb);        // sum d_y
            ld_line<N, 0>(fin + 3 * FP, 1, v);  // S_y Sd
            eo_apply<N, 1>(qp.S, v, Sd);        // sum d_z (normal)
          }
        }
        double rv[N], rn[N], ra[N], rb[N];
#pragma unroll
        for (int qx = 0; qx < N; ++qx) {
          if constexpr (Q3_JOBPRE) {
            flux(jcv[qx], jsd[qx], d, J[qx], Sd[qx], Sa[qx], Sb[qx], rv[qx], rn[qx], ra[qx], rb[qx]);
          } else {
            double cvec[3], sdA;
            fgeom<N, GEOM>(qp, ga, g, ccx, cy, cz, d, s, qx, q, cvec, sdA);
            flux(cvec, sdA, d, J[qx], Sd[qx], Sa[qx], Sb[qx], rv[qx], rn[qx], ra[qx], rb[qx]);
          }
        }
        // transposed x-sweeps: Pv = S^T rv + DS^T ra (tangential a = x), Pb = S^T rb, Pn = S^T rn
        double o[N];
        double* pout = FAb + c * Lay::FAC + (kind * 6 + s * 3) * FP + q * PG;
        eo_apply<N, 1>(qp.St, rv, o);
        eo_apply_add<N, -1>(qp.Dt, ra, o);
        st_line<N>(pout + 0 * FP, 1, o);
        eo_apply<N, 1>(qp.St, rb, o);
        st_line<N>(pout + 1 * FP, 1, o);
        eo_apply<N, 1>(qp.St, rn, o);
        st_line<N>(pout + 2 * FP, 1, o);
      }
    }
    __syncthreads();   // c fields (own and neighbour slots) read: R1..R3 take q1..q3
    if (active) {
      st_line<N>(R1 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, q1);
      st_line<N>(R2 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, q2);
      st_line<N>(R3 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, q3);
    }
  }
  __syncthreads();

  // ================================================================ Y^T
  {
    double r1[N], r2[N];
    if (active) {
      double v1[N], v2[N], v3[N];
      ld_line<N, 0>(R1 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, v1);
      ld_line<N, 0>(R2 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, v2);
      ld_line<N, 0>(R3 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, v3);
      eo_apply<N, 1>(qp.St, v1, r1);
      eo_apply_add<N, -1>(qp.Dt, v2, r1);
      eo_apply<N, 1>(qp.St, v3, r2);
      // y-face injections from PY[f][3][qz][i]
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double* py = FA + (0 * 6 + f * 3) * FP + yq * PG + yi;
        const double Pv = py[0], Pb = py[FP], Pn = py[2 * FP];
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int L = f ? N - NL + l : l;
          r1[L] = fma(qp.sf[f][l], Pv, fma(qp.df[f][l], Pn, r1[L]));
          r2[L] = fma(qp.sf[f][l], Pb, r2[L]);
        }
      }
    }
    // jobs: z-face transposed y-sweeps (cell, s, i): QZm[s][3][qy][i] -> QZo[s][2][j][i]
    {
      constexpr int NZJ = 2 * N;
      for (int job = btid; job < ncell * NZJ; job += BT) {
        const int c = job / NZJ, jj = job - c * NZJ;
        const int s = jj / N, i = jj - s * N;
        const double* qin = FAb + c * Lay::FAC + (6 + s * 3) * FP + i;
        double* qo = FBb + c * Lay::FBC + (s * 2) * FP + i;
        double v[N], o[N];
        ld_line<N, 0>(qin + 0 * FP, PG, v);
        eo_apply<N, 1>(qp.St, v, o);
        ld_line<N, 0>(qin + 1 * FP, PG, v);
        eo_apply_add<N, -1>(qp.Dt, v, o);
        st_line<N>(qo + 0 * FP, PG, o);
        ld_line<N, 0>(qin + 2 * FP, PG, v);
        eo_apply<N, 1>(qp.St, v, o);
        st_line<N>(qo + 1 * FP, PG, o);
      }
    }
    __syncthreads();   // q fields read: R1, R2 take r1, r2
    if (active) {
      st_line<N>(R1 + cslot * LZY.CS + at(LZY, yi, 0, yq), LZY.Pj, r1);
      st_line<N>(R2 + cslot * LZY.CS + at(LZY, yi, 0, yq), LZY.Pj, r2);
    }
  }
  __syncthreads();

  // ================================================================ Z^T
  double res[N];
  double bz[MODE == KMODE_APPLY ? 1 : N];   // Chebyshev: b along the z-line, issued before the sweeps
  if constexpr (MODE != KMODE_APPLY) {
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) bz[k] = __ldg(ch.b + cid * N3 + k * NN + zj * N + zi);
    }
  }
  if (active) {
    double v1[N], v2[N];
    ld_line<N, 0>(R1 + cslot * LZY.CS + at(LZY, zi, zj, 0), LZY.Pk, v1);
    ld_line<N, 0>(R2 + cslot * LZY.CS + at(LZY, zi, zj, 0), LZY.Pk, v2);
    eo_apply<N, 1>(qp.St, v1, res);
    eo_apply_add<N, -1>(qp.Dt, v2, res);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double* qo = FB + (s * 2) * FP + zj * PG + zi;
      const double Qv = qo[0], Qn = qo[FP];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int L = s ? N - NL + l : l;
        res[L] = fma(qp.sf[s][l], Qv, fma(qp.df[s][l], Qn, res[L]));
      }
    }
  }
  const int64_t gbase = cid * N3 + zj * N + zi;   // + k*NN
  if constexpr (MODE == KMODE_APPLY) {
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) y[gbase + k * NN] = res[k];
    }
    return;
  } else {
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) res[k] = bz[k] - res[k];
    }
    double ujz[N], upz[N];   // the update's inputs
    if constexpr (MODE == KMODE_CHEBY_GL) {
      // z: T^-T -> R1 (ZY);  y: T^-T -> R2 (YX);  x: T^-T, diag, T^-1 -> R1 (YX);
      // y: T^-1 -> R2 (ZY);  z: T^-1 + update
      __syncthreads();   // r1, r2 read
      if (active) {
        double o[N];
        eo_apply<N, 1>(qp.TiT, res, o);
        st_line<N>(R1 + cslot * LZY.CS + at(LZY, zi, zj, 0), LZY.Pk, o);
      }
      __syncthreads();
      double dx[N];   // the x stage's diagonal, loaded one stage early
      if (active) {
        const double* dv = ch.dinv + cid * N3 + (xq2 * N + xq1) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) dx[i] = __ldg(dv + i);
      }
      if (active) {
        double v[N], o[N];
        ld_line<N, 0>(R1 + cslot * LZY.CS + at(LZY, yi, 0, yq), LZY.Pj, v);
        eo_apply<N, 1>(qp.TiT, v, o);
        st_line<N>(R2 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, o);
      }
      __syncthreads();
      if (active) {
        double v[N], o[N];
        ld_line<N, 0>(R2 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, v);
        eo_apply<N, 1>(qp.TiT, v, o);
#pragma unroll
        for (int i = 0; i < N; ++i) o[i] *= dx[i];
        eo_apply<N, 1>(qp.Ti, o, v);
        st_line<N>(R1 + cslot * LYX.CS + at(LYX, 0, xq1, xq2), 1, v);
      }
      __syncthreads();
      if (active) {   // update inputs along the z-line, one stage early
#pragma unroll
        for (int k = 0; k < N; ++k) {
          ujz[k] = __ldg(u + gbase + k * NN);
          if (!ch.first) upz[k] = ch.u_prev[gbase + k * NN];
        }
      }
      if (active) {
        double v[N], o[N];
        ld_line<N, 0>(R1 + cslot * LYX.CS + at(LYX, yi, 0, yq), LYX.Pj, v);
        eo_apply<N, 1>(qp.Ti, v, o);
        st_line<N>(R2 + cslot * LZY.CS + at(LZY, yi, 0, yq), LZY.Pj, o);
      }
      __syncthreads();
      if (active) {
        double v[N];
        ld_line<N, 0>(R2 + cslot * LZY.CS + at(LZY, zi, zj, 0), LZY.Pk, v);
        eo_apply<N, 1>(qp.Ti, v, res);
      }
    } else {
      if (active) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          res[k] *= __ldg(ch.dinv + gbase + k * NN);
          ujz[k] = __ldg(u + gbase + k * NN);
          if (!ch.first) upz[k] = ch.u_prev[gbase + k * NN];
        }
      }
    }
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double v = fma(ch.c_z, res[k], ujz[k]);
        if (!ch.first) v = fma(ch.c_prev, ujz[k] - upz[k], v);
        ch.u_next[gbase + k * NN] = v;
      }
    }
  }
}

template <int N, int NL, int GEOM, int MODE>
cudaError_t launch_t(const QuadParams& qp, const GeomArgs& ga, const GridArgs& g, const double* u,
                     double* y, const ChebyArgs& ch, cudaStream_t s) {
  using Lay = Q3Layout<N, NL>;
  const int planes = g.zend - g.zbeg;
  if (planes <= 0 || g.Nx <= 0 || g.Ny <= 0) return cudaSuccess;
  if (g.Ny > 65535 || planes > 65535) return cudaErrorInvalidValue;
  const dim3 grid((g.Nx + Lay::CPB - 1) / Lay::CPB, g.Ny, planes);
  const dim3 block(N, N * Lay::CPB);
  const size_t smem = Lay::bytes();
  auto kern = k_quad3<N, NL, GEOM, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, block, smem, s>>>(qp, ga, g, u, y, ch);
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

bool quad3_supported(int n, int geom) {
  return n >= 3 && n <= 9 && (geom == GEOM_CONST || geom == GEOM_PER_QPOINT);
}

cudaError_t launch_quad3(int n, int NL, int geom, int mode, const QuadParams& qp, const GeomArgs& ga,
                         const GridArgs& g, const double* u, double* y, const ChebyArgs& ch,
                         cudaStream_t s) {
  switch (n) {
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
