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
// Schedule per cell (7 even-odd line sweeps, register-resident lines, one thread per
// line, n^2 threads per cell):
//   P0 loads: own cell -> smem; x-neighbour layers of the thread's own x-line -> registers;
//             rows of the y/z-neighbour layers loaded by row jobs and swept with M_x
//   x-lines:  t = M u,   a = L_x u + N_x^{+-} u_{x+-}
//   y-lines:  b = M a + L_y t + N_y^{+-} (M_x u_{y+-}),   c = M t;  M_y on the z-layer rows
//   z-lines:  y = M b + L_z c + N_z^{+-} (M_y M_x u_{z+-})      -> one coalesced write
// Shared-memory fields use per-access-pattern layouts addr = i + j*Pj + k*Pk (+ cell*CS)
// chosen by tools/smem_layout_search*.py so that the x-write/y-read and the
// y-write/z-read transposes are free of bank conflicts.
// The fused Chebyshev step ("merged") continues on the
// z-lines in registers: r = b - y, P^{-1} r by 6 more sweeps (T^{-T} in z,y,x;
// diagonal; T^{-1} in x,y,z; Eq. (12)), then the three-term update of Eq. (11).
#include <cuda_runtime.h>

#include "common.cuh"
#include "dg_internal.h"
#include "loader.cuh"

namespace dgb {
namespace {

struct Lay3 {
  int Pj, Pk, CS;
};

// (x-read), (x-write + y-read), (y-write + z-read) layouts per n
template <int N>
struct KL;
template <> struct KL<2> { static constexpr Lay3 X{3, 6, 12}, XY{2, 5, 10}, YZ{2, 4, 10}; };
template <> struct KL<3> { static constexpr Lay3 X{3, 9, 27}, XY{17, 51, 153}, YZ{3, 19, 57}; };
template <> struct KL<4> { static constexpr Lay3 X{5, 20, 80}, XY{5, 20, 80}, YZ{4, 18, 72}; };
template <> struct KL<5> { static constexpr Lay3 X{5, 25, 125}, XY{17, 85, 425}, YZ{5, 37, 185}; };
template <> struct KL<6> { static constexpr Lay3 X{7, 42, 252}, XY{9, 54, 324}, YZ{6, 38, 228}; };
template <> struct KL<7> { static constexpr Lay3 X{7, 49, 343}, XY{17, 119, 833}, YZ{7, 55, 385}; };
template <> struct KL<8> { static constexpr Lay3 X{9, 72, 576}, XY{9, 72, 576}, YZ{8, 68, 544}; };
template <> struct KL<9> { static constexpr Lay3 X{9, 81, 729}, XY{17, 153, 1377}, YZ{9, 89, 801}; };

constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <int N, int NL>
struct KLayout {
  static constexpr int P = N | 1;                       // rows of face layers / residual field
  static constexpr Lay3 X = KL<N>::X, XY = KL<N>::XY, YZ = KL<N>::YZ;
  static constexpr Lay3 R{P, N * P, N * N * P};          // Chebyshev residual field
  static constexpr int S0 = cmax(X.CS, YZ.CS);           // u, then b
  static constexpr int S1 = cmax(XY.CS, YZ.CS);          // t, then c
  static constexpr int S2 = cmax(XY.CS, R.CS);           // a, then the residual
  static constexpr int FACE = NL * N * P;                // one face's NL rows
  static constexpr int SF = 4 * FACE;                    // y-, y+, z-, z+ faces
  static constexpr int bytes(int cpb) { return cpb * (S0 + S1 + S2 + SF) * 8; }
};

__device__ __forceinline__ int at(const Lay3& L, int i, int j, int k) { return i + j * L.Pj + k * L.Pk; }

template <int N>
__device__ __forceinline__ int64_t cell_off(int64_t c) { return c * (int64_t)(N * N * N); }

template <int N, int NL>
constexpr int cells_per_block();

// resident blocks per SM allowed by shared memory (tells ptxas its register budget)
template <int N, int NL, int CPB>
constexpr int kron_min_blocks() {
  constexpr int b = (227 * 1024) / KLayout<N, NL>::bytes(CPB);
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

template <int N, int NL, int CPB, int MODE>
__global__ void __launch_bounds__(CPB * N * N, (kron_min_blocks<N, NL, CPB>()))
k_kron(const __grid_constant__ KronParams kp, const __grid_constant__ GridArgs g,
       const double* __restrict__ u, double* __restrict__ y, const __grid_constant__ ChebyArgs ch) {
  using Lay = KLayout<N, NL>;
  constexpr int P = Lay::P;
  constexpr int NN = N * N;
  constexpr Lay3 LX = Lay::X, LXY = Lay::XY, LYZ = Lay::YZ, LR = Lay::R;
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

  double* R0 = smem;                                   // u (X) -> b (YZ)
  double* R1 = R0 + CPB * Lay::S0;                     // t (XY) -> c (YZ)
  double* R2 = R1 + CPB * Lay::S1;                     // a (XY) -> residual (R)
  double* RF = R2 + CPB * Lay::S2;                     // face rows
  double* U = R0 + cslot * LX.CS;
  double* Bf = R0 + cslot * LYZ.CS;
  double* T = R1 + cslot * LXY.CS;
  double* Cf = R1 + cslot * LYZ.CS;
  double* A = R2 + cslot * LXY.CS;
  double* Rr = R2 + cslot * LR.CS;
  double* F = RF + cslot * Lay::SF;

  // ---------------------------------------------------------------- P0: loads
  // own cell: coalesced; y/z-neighbour layers: coalesced along their contiguous runs into
  // smem rows; x-neighbour layers: from the neighbouring slot's smem when that cell is in
  // this block (x-consecutive), else from global into registers here.
  double xm[NL], xp[NL];
  bool xm_smem = false, xp_smem = false;
  if (active) {
    const int cz = (int)(cid / plane);
    const int rem = (int)(cid - (int64_t)cz * plane);
    const int cy = rem / g.Nx, cx = rem - cy * g.Nx;
    const double* own = u + cell_off<N>(cid);
    double v[N];
#pragma unroll
    for (int r = 0; r < N; ++r) v[r] = __ldg(own + line + r * NN);
    xm_smem = cslot > 0 && cx > 0;
    xp_smem = cslot + 1 < ncell && cx + 1 < g.Nx;
    {
      const int a = line % N, b = line / N;   // this thread's x-line (j, k)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (s == 0 ? xm_smem : xp_smem) continue;
        const FaceSrc src = face_source<N, NL>(g, u, cid, cx, cy, cz, s);
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const int L = s == 0 ? N - NL + l : l;
          const int m = src.reflect ? N - 1 - L : L;
          const double val = src.sign * __ldg(src.base + face_elem<N>(0, m, a, b));
          if (s == 0) xm[l] = val; else xp[l] = val;
        }
      }
    }
    // y/z faces: element q of a face in contiguous-address order
    //   y: (a fastest, then l, then b) -> global (b*N + L)*N + a
    //   z: (a, b, l)                   -> global (L*N + b)*N + a
    double fvals[4][NL];
#pragma unroll
    for (int fr = 0; fr < 4; ++fr) {
      const int f = 2 + fr, d = f >> 1, s = f & 1;
      const FaceSrc src = face_source<N, NL>(g, u, cid, cx, cy, cz, f);
#pragma unroll
      for (int q = 0; q < NL; ++q) {
        const int e = line + q * NN;
        int a, l, b;
        if (d == 1) { a = e % N; l = (e / N) % NL; b = e / (N * NL); }
        else        { a = e % N; b = (e / N) % N; l = e / NN; }
        const int L = s == 0 ? N - NL + l : l;
        const int m = src.reflect ? N - 1 - L : L;
        fvals[fr][q] = src.sign * __ldg(src.base + face_elem<N>(d, m, a, b));
      }
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      const int e = line + r * NN;
      U[at(LX, e % N, (e / N) % N, e / NN)] = v[r];
    }
#pragma unroll
    for (int fr = 0; fr < 4; ++fr) {
      const int d = (2 + fr) >> 1;
#pragma unroll
      for (int q = 0; q < NL; ++q) {
        const int e = line + q * NN;
        int a, l, b;
        if (d == 1) { a = e % N; l = (e / N) % NL; b = e / (N * NL); }
        else        { a = e % N; b = (e / N) % N; l = e / NN; }
        F[fr * Lay::FACE + (l * N + b) * P + a] = fvals[fr][q];
      }
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- x-lines
  if (active) {
    const int j = line % N, k = line / N;
    if (xm_smem) {
      const double* Ul = U - LX.CS;
#pragma unroll
      for (int l = 0; l < NL; ++l) xm[l] = Ul[at(LX, N - NL + l, j, k)];
    }
    if (xp_smem) {
      const double* Ur = U + LX.CS;
#pragma unroll
      for (int l = 0; l < NL; ++l) xp[l] = Ur[at(LX, l, j, k)];
    }
    double x[N], t[N], a[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = U[at(LX, i, j, k)];
    const EOSplit<N> sp = eo_split<N>(x);
    eo_mul<N, 1, false>(kp.M, sp, t);
    eo_mul<N, 1, false>(kp.L[0], sp, a);
    dense_add<NL, NL>(kp.Nm[0], xm, &a[0]);
    dense_add<NL, NL>(kp.Np[0], xp, &a[N - NL]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      T[at(LXY, i, j, k)] = t[i];
      A[at(LXY, i, j, k)] = a[i];
    }
    // M along x on the rows of the y- and z-neighbour layers (in place)
    for (int job = line; job < 4 * NL * N; job += NN) {
      double* row = F + (job / (NL * N)) * Lay::FACE + (job % (NL * N)) * P;
      double r[N], o[N];
#pragma unroll
      for (int i = 0; i < N; ++i) r[i] = row[i];
      eo_apply<N, 1>(kp.M, r, o);
#pragma unroll
      for (int i = 0; i < N; ++i) row[i] = o[i];
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- y-lines
  double cl[N];
  if (active) {
    const int i = line % N, k = line / N;
    double al[N], tl[N], bl[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      al[j] = A[at(LXY, i, j, k)];
      tl[j] = T[at(LXY, i, j, k)];
    }
    const EOSplit<N> st = eo_split<N>(tl);
    eo_mul<N, 1, false>(kp.M, eo_split<N>(al), bl);
    eo_mul<N, 1, true>(kp.L[1], st, bl);
    eo_mul<N, 1, false>(kp.M, st, cl);
    double ym[NL], yp[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      ym[l] = F[0 * Lay::FACE + (l * N + k) * P + i];
      yp[l] = F[1 * Lay::FACE + (l * N + k) * P + i];
    }
    dense_add<NL, NL>(kp.Nm[1], ym, &bl[0]);
    dense_add<NL, NL>(kp.Np[1], yp, &bl[N - NL]);
#pragma unroll
    for (int j = 0; j < N; ++j) Bf[at(LYZ, i, j, k)] = bl[j];    // region of u: free
    // M along y on the (x-swept) z-layer rows: lines (fr, l, a=ii) along b=j
    for (int job = line; job < 2 * NL * N; job += NN) {
      const int fr = 2 + job / (NL * N), l = (job / N) % NL, ii = job % N;
      double* base = F + fr * Lay::FACE + (l * N) * P + ii;
      double r[N], o[N];
#pragma unroll
      for (int jj = 0; jj < N; ++jj) r[jj] = base[jj * P];
      eo_apply<N, 1>(kp.M, r, o);
#pragma unroll
      for (int jj = 0; jj < N; ++jj) base[jj * P] = o[jj];
    }
  }
  __syncthreads();                      // every thread has read t: its region takes c
  if (active) {
    const int i = line % N, k = line / N;
#pragma unroll
    for (int j = 0; j < N; ++j) Cf[at(LYZ, i, j, k)] = cl[j];
  }
  __syncthreads();

  // ---------------------------------------------------------------- z-lines
  double res[N];
  const int zi = line % N, zj = line / N;
  if (active) {
    double bl[N], cz[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      bl[k] = Bf[at(LYZ, zi, zj, k)];
      cz[k] = Cf[at(LYZ, zi, zj, k)];
    }
    eo_mul<N, 1, false>(kp.M, eo_split<N>(bl), res);
    eo_mul<N, 1, true>(kp.L[2], eo_split<N>(cz), res);
    double zm[NL], zp[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      zm[l] = F[2 * Lay::FACE + (l * N + zj) * P + zi];
      zp[l] = F[3 * Lay::FACE + (l * N + zj) * P + zi];
    }
    dense_add<NL, NL>(kp.Nm[2], zm, &res[0]);
    dense_add<NL, NL>(kp.Np[2], zp, &res[N - NL]);
  }
  const int64_t gbase = cell_off<N>(cid) + zj * N + zi;   // + k*N*N

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
      if (active) {  // (T^{-T})_z in registers
        double o[N];
        eo_apply<N, 1>(kp.TiT, res, o);
#pragma unroll
        for (int k = 0; k < N; ++k) Rr[at(LR, zi, zj, k)] = o[k];
      }
      __syncthreads();
      if (active) {  // (T^{-T})_y
        const int i = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = Rr[at(LR, i, j, k)];
        eo_apply<N, 1>(kp.TiT, r, o);
#pragma unroll
        for (int j = 0; j < N; ++j) Rr[at(LR, i, j, k)] = o[j];
      }
      __syncthreads();
      if (active) {  // (T^{-T})_x, diag(A_GL)^{-1}, (T^{-1})_x
        const int j = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int i = 0; i < N; ++i) r[i] = Rr[at(LR, i, j, k)];
        eo_apply<N, 1>(kp.TiT, r, o);
        const double* dv = ch.dinv + cell_off<N>(cid) + (k * N + j) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) o[i] *= __ldg(dv + i);
        eo_apply<N, 1>(kp.Ti, o, r);
#pragma unroll
        for (int i = 0; i < N; ++i) Rr[at(LR, i, j, k)] = r[i];
      }
      __syncthreads();
      if (active) {  // (T^{-1})_y
        const int i = line % N, k = line / N;
        double r[N], o[N];
#pragma unroll
        for (int j = 0; j < N; ++j) r[j] = Rr[at(LR, i, j, k)];
        eo_apply<N, 1>(kp.Ti, r, o);
#pragma unroll
        for (int j = 0; j < N; ++j) Rr[at(LR, i, j, k)] = o[j];
      }
      __syncthreads();
      if (active) {  // (T^{-1})_z back to registers
        double r[N];
#pragma unroll
        for (int k = 0; k < N; ++k) r[k] = Rr[at(LR, zi, zj, k)];
        eo_apply<N, 1>(kp.Ti, r, res);
      }
    } else {
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
  // ~256 threads per block, at most ~76 KB shared memory (3 blocks per SM)
  constexpr int byT = (256 + N * N - 1) / (N * N);
  constexpr int byS = (76 * 1024) / KLayout<N, NL>::bytes(1);
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
  const size_t smem = KLayout<N, NL>::bytes(CPB);
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
