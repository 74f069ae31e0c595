// C ABI of dg_b200 (include/dg.h): mesh setup, operator dispatch, basis change,
// fused Chebyshev driver, z-slab halo exchange over NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "dg_internal.h"
#include "halo_index.h"

using namespace dgb;

namespace {

thread_local std::string g_err = "no error";

dg_status fail(dg_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

// Vector arguments: the kernels use 128-bit accesses (double2 / float4 lines for even n),
// so every caller vector must be 16-byte aligned (dg.h "Conventions"); a misaligned
// pointer is rejected here instead of faulting (and poisoning the context) in a kernel.
bool misaligned(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 15u) != 0; }

#define CHECK_ALIGNED(ptr)                                                          \
  do {                                                                              \
    if (misaligned(ptr))                                                            \
      return fail(DG_ERR_PARAM, "%s = %p is not 16-byte aligned", #ptr, (const void*)(ptr)); \
  } while (0)

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DG_DEBUG_SYNC");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v == 1;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(DG_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                              \
  } while (0)

#define NCCL_TRY(expr)                                                              \
  do {                                                                              \
    ncclResult_t r_ = (expr);                                                       \
    if (r_ != ncclSuccess)                                                          \
      return fail(DG_ERR_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(r_),    \
                  __FILE__, __LINE__);                                              \
  } while (0)

// pack an n x n row-major matrix into the even-odd layout of common.cuh
// FDM setup (Eqs. (13)-(15)): generalized symmetric definite
// eigenproblem L z = lam M z of the 1D interior element in long double: Cholesky
// M = C C^T, cyclic Jacobi on K = C^-1 L C^-T, Z = C^-T V (so Z^T M Z = I).  The
// eigenvectors of this reflection-symmetric pencil are symmetric or antisymmetric;
// they are packed by parity for the even/odd application in k_kron4.  Returns false
// if M is not SPD or the parity split fails.
bool fdm_setup(const double* L, const double* M, int n, KronParams& kp) {
  typedef long double R;
  R C[kMaxN][kMaxN] = {}, Ci[kMaxN][kMaxN] = {}, K[kMaxN][kMaxN], V[kMaxN][kMaxN], Z[kMaxN][kMaxN];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      R acc = M[i * n + j];
      for (int k = 0; k < j; ++k) acc -= C[i][k] * C[j][k];
      if (i == j) {
        if (!(acc > 0)) return false;
        C[i][i] = std::sqrt(acc);
      } else {
        C[i][j] = acc / C[j][j];
      }
    }
  for (int j = 0; j < n; ++j) {   // Ci = C^-1 (lower triangular), column by column
    for (int i = 0; i < n; ++i) {
      R acc = (i == j) ? 1 : 0;
      for (int k = 0; k < i; ++k) acc -= C[i][k] * Ci[k][j];
      Ci[i][j] = acc / C[i][i];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      R acc = 0;
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) acc += Ci[i][a] * L[a * n + b] * Ci[j][b];
      K[i][j] = acc;
      V[i][j] = (i == j) ? 1 : 0;
    }
  for (int sweep = 0; sweep < 100; ++sweep) {
    R off = 0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += K[p][q] * K[p][q];
    if (off < 1e-60L) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (K[p][q] == 0) continue;
        const R th = (K[q][q] - K[p][p]) / (2 * K[p][q]);
        const R t = (th >= 0 ? 1 : -1) / (std::fabs(th) + std::sqrt(th * th + 1));
        const R c = 1 / std::sqrt(t * t + 1), sn = t * c;
        for (int k = 0; k < n; ++k) {
          const R kp_ = K[k][p], kq = K[k][q];
          K[k][p] = c * kp_ - sn * kq;
          K[k][q] = sn * kp_ + c * kq;
        }
        for (int k = 0; k < n; ++k) {
          const R kp_ = K[p][k], kq = K[q][k];
          K[p][k] = c * kp_ - sn * kq;
          K[q][k] = sn * kp_ + c * kq;
        }
        for (int k = 0; k < n; ++k) {
          const R vp = V[k][p], vq = V[k][q];
          V[k][p] = c * vp - sn * vq;
          V[k][q] = sn * vp + c * vq;
        }
      }
  }
  for (int i = 0; i < n; ++i)      // Z = C^-T V
    for (int m = 0; m < n; ++m) {
      R acc = 0;
      for (int k = 0; k < n; ++k) acc += Ci[k][i] * V[k][m];
      Z[i][m] = acc;
    }
  const int h = n / 2, hs = (n + 1) / 2, ha = n / 2;
  int ns = 0, na = 0;
  for (int m = 0; m < n; ++m) {
    R sym = 0, anti = 0, nrm = 0;
    for (int i = 0; i < n; ++i) {
      sym += std::fabs(Z[i][m] - Z[n - 1 - i][m]);
      anti += std::fabs(Z[i][m] + Z[n - 1 - i][m]);
      nrm += std::fabs(Z[i][m]);
    }
    const bool is_sym = sym < 1e-12L * nrm;
    const bool is_anti = anti < 1e-12L * nrm;
    if (is_sym == is_anti) return false;
    if (is_sym) {
      if (ns >= hs) return false;
      for (int i = 0; i < hs; ++i) kp.Zs[i * hs + ns] = (double)Z[i][m];
      kp.lam[ns++] = (double)K[m][m];
    } else {
      if (na >= ha) return false;
      for (int i = 0; i < h; ++i) kp.Za[i * ha + na] = (double)Z[i][m];
      kp.lam[hs + na++] = (double)K[m][m];
    }
  }
  return ns == hs && na == ha;
}

void pack_eo(const double* A, int n, double* out);

// Tables of the transformed-residual Chebyshev step (KronParams::Mt/Lt/Ft, KMODE_CHEBY_GLT):
// T^{-T} times Mhat, L_d and the neighbour block N^-_d, accumulated in long double.  Returns
// false (mode unavailable) unless the products keep the reflection symmetry the even-odd
// packing assumes: A[n-1-i][n-1-j] = A[i][j] and (T^{-T} N^+)[n-1-i][NL-1-l] = (T^{-T} N^-)[i][l].
bool glt_setup(const Tables1D& t, int n, int NL, const double* h, KronParams& kp) {
  using R = long double;
  const double V = h[0] * h[1] * h[2];
  auto mul = [&](const double* A, int cols, int lda, int c0, double sc, R* out) {   // T^{-T} (sc A[:, c0:c0+cols])
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < cols; ++c) {
        R acc = 0;
        for (int k = 0; k < n; ++k) acc += (R)t.Tinv[k * n + i] * ((R)sc * (R)A[k * lda + c0 + c]);
        out[i * cols + c] = acc;
      }
  };
  auto centro = [&](const R* A) {
    R mx = 0, err = 0;
    for (int q = 0; q < n * n; ++q) mx = std::max(mx, std::fabs(A[q]));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) err = std::max(err, std::fabs(A[i * n + j] - A[(n - 1 - i) * n + n - 1 - j]));
    return err <= 1e-13L * mx;
  };
  R A[kMaxN * kMaxN];
  double Ad[kMaxN * kMaxN];
  mul(t.Mhat, n, n, 0, 1.0, A);
  if (!centro(A)) return false;
  for (int q = 0; q < n * n; ++q) Ad[q] = (double)A[q];
  pack_eo(Ad, n, kp.Mt);
  const int H = n / 2;
  for (int dd = 0; dd < 3; ++dd) {
    const double sc = V / (h[dd] * h[dd]);
    mul(t.Lhat, n, n, 0, sc, A);
    if (!centro(A)) return false;
    for (int q = 0; q < n * n; ++q) Ad[q] = (double)A[q];
    pack_eo(Ad, n, kp.Lt[dd]);
    R Pm[kMaxN * 2], Pp[kMaxN * 2];
    mul(t.Nm, NL, n, n - NL, sc, Pm);   // own rows x neighbour layers [n-NL, n)
    mul(t.Np, NL, n, 0, sc, Pp);        // own rows x neighbour layers [0, NL)
    R mx = 0, err = 0;
    for (int i = 0; i < n; ++i)
      for (int l = 0; l < NL; ++l) {
        mx = std::max(mx, std::fabs(Pm[i * NL + l]));
        err = std::max(err, std::fabs(Pp[(n - 1 - i) * NL + (NL - 1 - l)] - Pm[i * NL + l]));
      }
    if (!(err <= 1e-13L * mx)) return false;
    int o = 0;
    for (int i = 0; i < H; ++i)
      for (int l = 0; l < NL; ++l) kp.Ft[dd][o++] = (double)(0.5L * (Pm[i * NL + l] + Pm[(n - 1 - i) * NL + l]));
    for (int i = 0; i < H; ++i)
      for (int l = 0; l < NL; ++l) kp.Ft[dd][o++] = (double)(0.5L * (Pm[i * NL + l] - Pm[(n - 1 - i) * NL + l]));
    if (n & 1)
      for (int l = 0; l < NL; ++l) kp.Ft[dd][o++] = (double)Pm[H * NL + l];
  }
  return true;
}

void pack_eo(const double* A, int n, double* out) {
  const int h = n / 2, mid = h;
  int o = 0;
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < h; ++j) out[o++] = 0.5 * (A[i * n + j] + A[i * n + n - 1 - j]);
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < h; ++j) out[o++] = 0.5 * (A[i * n + j] - A[i * n + n - 1 - j]);
  for (int i = 0; i < h; ++i) out[o++] = (n & 1) ? A[i * n + mid] : 0.0;
  for (int j = 0; j < h; ++j) out[o++] = (n & 1) ? A[mid * n + j] : 0.0;
  out[o++] = (n & 1) ? A[mid * n + mid] : 0.0;
}

double inv3_host(const double* J, double* Ji) {
  const double a = J[0], b = J[1], c = J[2], d = J[3], e = J[4], f = J[5], g = J[6], h = J[7], i = J[8];
  const double A = e * i - f * h, B = -(d * i - f * g), C = d * h - e * g;
  const double det = a * A + b * B + c * C;
  const double id = 1.0 / det;
  Ji[0] = A * id; Ji[3] = B * id; Ji[6] = C * id;
  Ji[1] = -(b * i - c * h) * id; Ji[4] = (a * i - c * g) * id; Ji[7] = -(a * h - b * g) * id;
  Ji[2] = (b * f - c * e) * id; Ji[5] = -(a * f - c * d) * id; Ji[8] = (a * e - b * d) * id;
  return det;
}

void transpose(const double* A, int n, double* At) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) At[j * n + i] = A[i * n + j];
}

}  // namespace

struct dg_mesh_s {
  dg_mesh_desc desc{};
  Tables1D tab;
  int n = 0, NL = 0;
  int N[3] = {0, 0, 0};
  int z_begin = 0, z_end = 0, nz = 0;
  int64_t ncells_local = 0, ndofs_local = 0, ndofs_global = 0;
  double h[3] = {0, 0, 0};
  bool cartesian = false;
  int geom = GEOM_CONST;          // general path geometry storage
  KronParams kp{};
  QuadParams qp{};
  GeomArgs ga{};
  double* d_G = nullptr;          // PER_QPOINT cell tensors
  double* d_face[3] = {nullptr, nullptr, nullptr};
  double* d_jinv = nullptr;       // PER_CELL J^-1 + det J (with ghost planes)
  double* d_usig[3] = {nullptr, nullptr, nullptr};   // user sigma_F per face (dg.h user_penalty)
  bool user_pen = false;
  int zlo = ZSRC_MIRROR, zhi = ZSRC_MIRROR;
  // lazily built inverse diagonals
  double* d_dinv_gl = nullptr;
  double* d_dinv_pj = nullptr;
  // halo (z-slabs)
  double* d_recv_lo = nullptr;
  double* d_recv_hi = nullptr;
  double* d_send_lo = nullptr;
  double* d_send_hi = nullptr;
  int64_t halo_count = 0;         // doubles per halo buffer
  ncclComm_t comm = nullptr;
  bool external = false;          // nranks > 1 without NCCL: dg_halo_pack / dg_halo_set
  dg_transport transport{};       // external mode: caller's halo / all-reduce callbacks
  std::string comm_key;           // NCCL unique id bytes of the shared communicator
  int lo_peer = -1, hi_peer = -1;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  int rank = 0, nranks = 1;
  int64_t launches = 0;
  bool fdm_ok = false;            // FDM tables built (Cartesian meshes)
  bool glt_ok = false;            // transformed-residual Chebyshev tables built (KronParams::Mt/Lt/Ft)
  double* d_bt = nullptr;         // (T^{-T})^{(x)3} b of the current GLT Chebyshev sweep
  double* d_dot = nullptr;        // dot-product scratch: partials + result
  // fp32 path: rounded Kronecker tables and inverse diagonals
  KronParamsF kpf{};
  bool kpf_ok = false;
  float* d_dinv_gl_f = nullptr;
  float* d_dinv_pj_f = nullptr;
  // host-buffer apply (dg_apply_laplace_host): device staging, copy streams, per-chunk events
  double* d_hu = nullptr;
  double* d_hy = nullptr;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  std::vector<cudaEvent_t> ev_h2d, ev_comp;
  cudaEvent_t ev_done = nullptr;
};

namespace {

dg_status post_launch(dg_mesh m, cudaError_t e, const char* what, cudaStream_t s) {
  if (e != cudaSuccess) return fail(DG_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  m->launches++;
  if (debug_sync()) {
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (e2 != cudaSuccess) return fail(DG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e2));
  }
  return DG_OK;
}

// Cartesian kernel selection: k_kron4 (z-first) for p = 2..8; p = 1 runs the general
// quadrature kernel k_quad on the constant geometry (the same operator)
bool kron_v4(int n) { return kron4_supported(n); }

// Cartesian matvec kernel: k_kron6 (i-plane schedule) where DG_K6 selects it for this n
// (bit n-3 of the mask; see DESIGN.md for the measured choice), else k_kron4
bool kron6_use(int n, int NL, int mode) {
  static const int mask = [] {
    const char* e = std::getenv("DG_K6");
    return e ? std::atoi(e) : 1;   // measured: k_kron6 wins only for the n = 3 matvec
  }();
  // bits 0-3: matvec at n = 3..6; bits 4-7: the fused Chebyshev step at n = 3..6
  const int bit = (mode == KMODE_APPLY ? 0 : 4) + (n - 3);
  return kron6_supported(n, NL, mode) && ((mask >> bit) & 1);
}

// n = 3 cell-per-thread kernel k_kron3c (DG_K3C=0 falls back to k_kron6 / k_kron4)
bool kron3c_use(int n, int NL) {
  static const int v = [] {
    const char* e = std::getenv("DG_K3C");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0 && kron3c_supported(n, NL);
}

// transformed-residual GL-Jacobi Chebyshev (KMODE_CHEBY_GLT) where the step runs on k_kron4 and
// bit n-3 of DG_CHEBY_GLT is set.  Default by measurement (same-box A/B, C4, GDoF/s per step,
// direct -> transformed): n = 4 91.5 -> 93.3, n = 5 77.3 -> 81.2, n = 6 98.3 -> 95.9 (off),
// n = 7 70.2 -> 71.4, n = 8 85.8 -> 102.9, n = 9 82.6 -> 87.1; n = 3 runs k_kron3c (direct step)
bool glt_use(dg_mesh m) {
  static const int mask = [] {
    const char* e = std::getenv("DG_CHEBY_GLT");
    return e ? std::atoi(e) : 0x77;   // all n but 6
  }();
  return ((mask >> (m->n - 3)) & 1) && m->glt_ok && m->cartesian && kron_v4(m->n) && !kron3c_use(m->n, m->NL);
}

// general kernel selection: k_quad3 (z-first) unless DG_QUAD=1 asks for k_quad.cu
bool quad_v3(int n, int geom) {
  static const int v = [] {
    const char* e = std::getenv("DG_QUAD");
    return e ? std::atoi(e) : 3;
  }();
  return v != 1 && quad3_supported(n, geom);
}

GridArgs grid_args(dg_mesh m, int zbeg, int zend) {
  GridArgs g{};
  g.Nx = m->N[0];
  g.Ny = m->N[1];
  g.nz = m->nz;
  g.bc[0] = m->desc.bc[0];
  g.bc[1] = m->desc.bc[1];
  g.bc[2] = m->desc.bc[2];
  g.zlo = m->zlo;
  g.zhi = m->zhi;
  g.zbeg = zbeg;
  g.zend = zend;
  g.halo_lo = m->d_recv_lo;
  g.halo_hi = m->d_recv_hi;
  static const int l2pf = [] {
    const char* e = std::getenv("DG_L2PF");
    return e ? std::atoi(e) : -1;
  }();
  // default: next plane's u tile; at n = 3 also the own Chebyshev tiles (measured +4-5% for
  // the p = 2 Chebyshev step, neutral elsewhere)
  g.l2pf = l2pf >= 0 ? l2pf : (m->n == 3 ? 3 : 1);
  return g;
}

// 1D diagonal variants [interior, left bdry, right bdry, both] of the 1D block L
void diag_variants(const double* L, const double* Nm, const double* Np, int n, int bc, int Nd,
                   double scale_unused, double out[4][kMaxN]) {
  (void)scale_unused;
  for (int i = 0; i < n; ++i) {
    const double li = L[i * n + i];
    const double cl = -Nm[i * n + (n - 1 - i)];   // mirror ghost of the face at xi=0
    const double cr = -Np[i * n + (n - 1 - i)];   // mirror ghost of the face at xi=1
    if (bc == DG_BC_PERIODIC) {
      for (int v = 0; v < 4; ++v) out[v][i] = li;
      if (Nd == 1) out[3][i] = li + Nm[i * n + i] + Np[i * n + i];
    } else {
      out[0][i] = li;
      out[1][i] = li + cl;
      out[2][i] = li + cr;
      out[3][i] = li + cl + cr;
    }
  }
}

dg_status build_diag(dg_mesh m, bool gl, double** dst, cudaStream_t s) {
  if (*dst) return DG_OK;
  const Tables1D& t = m->tab;
  if (!m->cartesian) {
    DiagTables dt{};
    const int n = m->n;
    std::memcpy(dt.S, gl ? t.gl_S : t.S, sizeof(double) * n * n);
    std::memcpy(dt.DS, gl ? t.gl_DS : t.DS, sizeof(double) * n * n);
    std::memcpy(dt.v[0], gl ? t.gl_v0 : t.v0, sizeof(double) * n);
    std::memcpy(dt.v[1], gl ? t.gl_v1 : t.v1, sizeof(double) * n);
    std::memcpy(dt.d[0], gl ? t.gl_d0 : t.d0, sizeof(double) * n);
    std::memcpy(dt.d[1], gl ? t.gl_d1 : t.d1, sizeof(double) * n);
    std::memcpy(dt.w, t.wq, sizeof(double) * n);
    CUDA_TRY(cudaMalloc(dst, sizeof(double) * (size_t)std::max<int64_t>(m->ndofs_local, 1)));
    return post_launch(m, launch_diag_general(n, m->geom, dt, m->qp, m->ga, grid_args(m, 0, m->nz), 1,
                                              *dst, s), "diag_general", s);
  }
  const int n = m->n;
  const double* M = gl ? t.gl_Mhat : t.Mhat;
  const double* L = gl ? t.gl_Lhat : t.Lhat;
  const double* Nm = gl ? t.gl_Nm : t.Nm;
  const double* Np = gl ? t.gl_Np : t.Np;
  CartDiagParams p{};
  for (int i = 0; i < n; ++i) p.mdiag[i] = M[i * n + i];
  const double V = m->h[0] * m->h[1] * m->h[2];
  for (int d = 0; d < 3; ++d) {
    diag_variants(L, Nm, Np, n, m->desc.bc[d], m->N[d], 0, p.ldiag[d]);
    p.scale[d] = V / (m->h[d] * m->h[d]);
  }
  p.invert = 1;
  CUDA_TRY(cudaMalloc(dst, sizeof(double) * (size_t)std::max<int64_t>(m->ndofs_local, 1)));
  dg_status st = post_launch(m, launch_cart_diag(n, p, m->N[0], m->N[1], m->nz, m->z_begin,
                                                 m->N[2], *dst, s),
                             "cart_diag", s);
  return st;
}

dg_status halo_exchange_impl(dg_mesh m, const double* u, cudaStream_t s);
dg_status run_pass(dg_mesh m, int mode, bool kron, const double* u, double* y, const ChebyArgs& ch,
                   bool halo_ready, cudaStream_t s);

// Per-face penalties from the caller's per-cell array (dg.h user_penalty):
// sig[d][fid] in the face layout of the geometry arrays (x: [z][y][Nx+1], y: [z][Ny+1][x],
// z: [nz+1][y][x]; local planes).  The face between lower cell (plane pl-1, face 2d+1) and
// upper cell (plane pl, face 2d) takes their common value; both present and different ->
// DG_ERR_PARAM.  z faces of a slab boundary with a remote peer take the owned side.
dg_status build_user_sigma(const double* up, const int N[3], int nz, int bc[3], bool zwrap,
                           std::vector<double> sig[3]) {
  const int Nx = N[0], Ny = N[1];
  const int64_t plane = (int64_t)Nx * Ny;
  const int64_t ncl = plane * nz;
  for (int64_t c = 0; c < ncl * 6; ++c)
    if (!(up[c] >= 0.0) || !std::isfinite(up[c]))
      return fail(DG_ERR_PARAM, "user_penalty[%lld] = %g is negative or not finite", (long long)c, up[c]);
  const int nloc[3] = {Nx, Ny, nz};
  for (int d = 0; d < 3; ++d) {
    const int nf[3] = {Nx + (d == 0), Ny + (d == 1), nz + (d == 2)};
    const bool per = d < 2 ? bc[d] == DG_BC_PERIODIC : zwrap;
    sig[d].assign((size_t)nf[0] * nf[1] * nf[2], 0.0);
    for (int fz = 0; fz < nf[2]; ++fz)
      for (int fy = 0; fy < nf[1]; ++fy)
        for (int fx = 0; fx < nf[0]; ++fx) {
          const int64_t fid = ((int64_t)fz * nf[1] + fy) * nf[0] + fx;
          int c[3] = {fx, fy, fz};
          const int pl = c[d], Nd = nloc[d];
          double vals[2];
          int nv = 0;
          int lo = pl - 1, hi = pl;
          if (lo < 0) lo = per ? Nd - 1 : -1;
          if (hi >= Nd) hi = per ? 0 : -1;
          if (lo >= 0) {
            int cc[3] = {c[0], c[1], c[2]};
            cc[d] = lo;
            vals[nv++] = up[(((int64_t)cc[2] * Ny + cc[1]) * Nx + cc[0]) * 6 + 2 * d + 1];
          }
          if (hi >= 0) {
            int cc[3] = {c[0], c[1], c[2]};
            cc[d] = hi;
            vals[nv++] = up[(((int64_t)cc[2] * Ny + cc[1]) * Nx + cc[0]) * 6 + 2 * d];
          }
          if (nv == 2 && vals[0] != vals[1])
            return fail(DG_ERR_PARAM, "user_penalty differs on the two sides of face (d=%d, %d,%d,%d): %g vs %g",
                        d, fx, fy, fz, vals[0], vals[1]);
          sig[d][fid] = nv ? vals[0] : 0.0;
        }
  }
  return DG_OK;
}

// NCCL communicators shared by every mesh built from the same unique id (one
// ncclCommInitRank per id and rank; e.g. the per-degree meshes of the bench), refcounted.
struct CommEntry {
  ncclComm_t comm;
  int refs;
};
std::mutex g_comm_mu;
std::map<std::string, CommEntry> g_comms;

ncclResult_t comm_acquire(const void* id128, int nranks, int rank, ncclComm_t* out, std::string* key) {
  std::lock_guard<std::mutex> lk(g_comm_mu);
  std::string k(reinterpret_cast<const char*>(id128), 128);
  k += std::to_string(nranks) + ":" + std::to_string(rank);
  auto it = g_comms.find(k);
  if (it != g_comms.end()) {
    it->second.refs++;
    *out = it->second.comm;
    *key = k;
    return ncclSuccess;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return r;
  g_comms[k] = CommEntry{c, 1};
  *out = c;
  *key = k;
  return ncclSuccess;
}

void comm_release(const std::string& key) {
  std::lock_guard<std::mutex> lk(g_comm_mu);
  auto it = g_comms.find(key);
  if (it == g_comms.end()) return;
  if (--it->second.refs == 0) {
    ncclCommDestroy(it->second.comm);
    g_comms.erase(it);
  }
}

// z-slab partition and peers (shared by dg_slab_plan and dg_mesh_setup)
void slab_plan(int Nz, int P, int r, int bcz, int out[4]) {
  out[0] = (int)((int64_t)r * Nz / P);
  out[1] = (int)((int64_t)(r + 1) * Nz / P);
  const bool per = bcz == DG_BC_PERIODIC;
  out[2] = P == 1 ? -1 : (r > 0 ? r - 1 : (per ? P - 1 : -1));
  out[3] = P == 1 ? -1 : (r < P - 1 ? r + 1 : (per ? 0 : -1));
}

}  // namespace

extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }

const char* dg_version(void) { return "dg_b200 0.1 sm_100a fp64"; }

dg_status dg_get_nccl_unique_id(void* out128) {
  if (!out128) return fail(DG_ERR_PARAM, "out128 is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
  return DG_OK;
}

dg_status dg_mesh_setup(const dg_mesh_desc* d, dg_mesh* out) {
  if (!d || !out) return fail(DG_ERR_PARAM, "NULL desc or out");
  *out = nullptr;
  if (d->degree < 1 || d->degree > 8) return fail(DG_ERR_PARAM, "degree %d not in 1..8", d->degree);
  if (d->basis != DG_BASIS_HERMITE_LIKE && d->basis != DG_BASIS_NODAL_GL)
    return fail(DG_ERR_PARAM, "bad basis %d", d->basis);
  for (int k = 0; k < 3; ++k) {
    if (d->n_cells[k] < 1) return fail(DG_ERR_PARAM, "n_cells[%d] = %d", k, d->n_cells[k]);
    if (!(d->box_hi[k] > d->box_lo[k])) return fail(DG_ERR_PARAM, "box_hi[%d] <= box_lo[%d]", k, k);
    if (d->bc[k] != DG_BC_DIRICHLET_MIRROR && d->bc[k] != DG_BC_PERIODIC)
      return fail(DG_ERR_PARAM, "bad bc[%d]", k);
  }
  if (d->geometry < DG_GEOM_CONSTANT || d->geometry > DG_GEOM_PER_QPOINT)
    return fail(DG_ERR_PARAM, "bad geometry %d", d->geometry);
  if (d->deform_amp != 0.0 && d->geometry != DG_GEOM_PER_QPOINT)
    return fail(DG_ERR_PARAM, "deform_amp != 0 requires DG_GEOM_PER_QPOINT");
  const int nranks = d->nranks < 1 ? 1 : d->nranks;
  if (d->rank < 0 || d->rank >= nranks) return fail(DG_ERR_PARAM, "rank %d of %d", d->rank, nranks);
  if (d->n_cells[2] < nranks) return fail(DG_ERR_PARAM, "Nz=%d < nranks=%d", d->n_cells[2], nranks);

  dg_mesh m = new dg_mesh_s();
  m->desc = *d;
  m->desc.user_inv_jac = nullptr;
  m->desc.user_penalty = nullptr;
  m->rank = d->rank;
  m->nranks = nranks;
  if (!build_tables(d->degree, d->basis, d->penalty_factor, &m->tab)) {
    delete m;
    return fail(DG_ERR_PARAM, "build_tables failed");
  }
  const int n = m->n = d->degree + 1;
  m->NL = (d->basis == DG_BASIS_HERMITE_LIKE && n > 2) ? 2 : n;
  for (int k = 0; k < 3; ++k) m->N[k] = d->n_cells[k];
  {
    int plan[4];
    slab_plan(m->N[2], nranks, d->rank, d->bc[2], plan);
    m->z_begin = plan[0];
    m->z_end = plan[1];
    m->lo_peer = plan[2];
    m->hi_peer = plan[3];
  }
  m->nz = m->z_end - m->z_begin;
  const int64_t n3 = (int64_t)n * n * n;
  m->ncells_local = (int64_t)m->N[0] * m->N[1] * m->nz;
  m->ndofs_local = m->ncells_local * n3;
  m->ndofs_global = (int64_t)m->N[0] * m->N[1] * m->N[2] * n3;

  // geometry: Cartesian = identity-or-diagonal linear map, no deformation
  double L[9];
  bool allzero = true;
  for (int k = 0; k < 9; ++k) {
    L[k] = d->linear_map[k];
    if (L[k] != 0.0) allzero = false;
  }
  if (allzero) {
    for (int k = 0; k < 9; ++k) L[k] = (k % 4 == 0) ? 1.0 : 0.0;
  }
  const bool diagonal = L[1] == 0 && L[2] == 0 && L[3] == 0 && L[5] == 0 && L[6] == 0 && L[7] == 0;
  m->cartesian = diagonal && d->deform_amp == 0.0 && d->geometry == DG_GEOM_CONSTANT;
  for (int k = 0; k < 3; ++k) m->h[k] = (d->box_hi[k] - d->box_lo[k]) / m->N[k];
  m->geom = d->geometry == DG_GEOM_PER_QPOINT ? GEOM_PER_QPOINT
            : (d->geometry == DG_GEOM_PER_CELL ? GEOM_PER_CELL : GEOM_CONST);
  if (d->user_penalty) {
    // per-face penalties: the general kernels with per-face data (constant geometry is
    // stored per quadrature point so the penalty can ride in the face arrays)
    m->user_pen = true;
    m->cartesian = false;
    if (m->geom == GEOM_CONST) m->geom = GEOM_PER_QPOINT;
  }
  if (d->geometry != DG_GEOM_PER_CELL && d->user_inv_jac) {
    delete m;
    return fail(DG_ERR_PARAM, "user_inv_jac requires DG_GEOM_PER_CELL");
  }
  // affine Jacobian of the undeformed map: J_im = L_im h_m
  double J0[9], Ji0[9];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) J0[i * 3 + k] = L[i * 3 + k] * m->h[k];
  const double det0 = inv3_host(J0, Ji0);
  if (!(det0 > 0) || !std::isfinite(det0)) {
    delete m;
    return fail(DG_ERR_NUMERIC, "det(L diag(h)) = %g <= 0", det0);
  }
  const double pen = (double)(n * n) * (d->penalty_factor > 0 ? d->penalty_factor : 1.0);
  {
    // general-path parameters (Eqs. (3)-(5))
    const Tables1D& t = m->tab;
    QuadParams& qp = m->qp;
    std::memset(&qp, 0, sizeof qp);
    double St[kMaxN * kMaxN], Dt[kMaxN * kMaxN];
    transpose(t.S, n, St);
    transpose(t.DS, n, Dt);
    pack_eo(t.S, n, qp.S);
    pack_eo(t.DS, n, qp.D);
    pack_eo(St, n, qp.St);
    pack_eo(Dt, n, qp.Dt);
    const int NLq = (d->basis == DG_BASIS_HERMITE_LIKE && n > 2) ? 2 : n;
    for (int sd = 0; sd < 2; ++sd)
      for (int l = 0; l < NLq; ++l) {
        const int Lo = sd ? n - NLq + l : l;
        const int Ln = sd ? l : n - NLq + l;
        qp.sf[sd][l] = sd ? t.v1[Lo] : t.v0[Lo];
        qp.df[sd][l] = sd ? t.d1[Lo] : t.d0[Lo];
        qp.sfn[sd][l] = sd ? t.v0[Ln] : t.v1[Ln];
        qp.dfn[sd][l] = sd ? t.d0[Ln] : t.d1[Ln];
      }
    for (int q = 0; q < n; ++q) qp.w[q] = t.wq[q];
    // constant geometry: G0 = det J J^-1 J^-T; per direction d, r = row d of J^-1:
    //   dA_ref J^-1 n_+ = det J J^-1 r,  sigma dA_ref = pen |r| det J |r|
    qp.G0[0] = det0 * (Ji0[0] * Ji0[0] + Ji0[1] * Ji0[1] + Ji0[2] * Ji0[2]);
    qp.G0[1] = det0 * (Ji0[3] * Ji0[3] + Ji0[4] * Ji0[4] + Ji0[5] * Ji0[5]);
    qp.G0[2] = det0 * (Ji0[6] * Ji0[6] + Ji0[7] * Ji0[7] + Ji0[8] * Ji0[8]);
    qp.G0[3] = det0 * (Ji0[0] * Ji0[3] + Ji0[1] * Ji0[4] + Ji0[2] * Ji0[5]);
    qp.G0[4] = det0 * (Ji0[0] * Ji0[6] + Ji0[1] * Ji0[7] + Ji0[2] * Ji0[8]);
    qp.G0[5] = det0 * (Ji0[3] * Ji0[6] + Ji0[4] * Ji0[7] + Ji0[5] * Ji0[8]);
    for (int dd = 0; dd < 3; ++dd) {
      const double* r = Ji0 + 3 * dd;
      const double nr = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
      for (int k = 0; k < 3; ++k)
        qp.cw0[dd][k] = det0 * (Ji0[k * 3] * r[0] + Ji0[k * 3 + 1] * r[1] + Ji0[k * 3 + 2] * r[2]);
      qp.sdA0[dd] = pen * nr * det0 * nr;
    }
    double TiT[kMaxN * kMaxN];
    transpose(t.Tinv, n, TiT);
    pack_eo(TiT, n, qp.TiT);
    pack_eo(t.Tinv, n, qp.Ti);
    m->ga.pen = pen;
  }
  if (m->cartesian) {
    for (int k = 0; k < 3; ++k) m->h[k] = L[4 * k] * (d->box_hi[k] - d->box_lo[k]) / m->N[k];
    for (int k = 0; k < 3; ++k)
      if (!(m->h[k] > 0) || !std::isfinite(m->h[k])) {
        delete m;
        return fail(DG_ERR_NUMERIC, "non-positive cell size in direction %d", k);
      }
  }
  // Kronecker parameters: L_d = (V/h_d^2) Lhat, Nm/Np blocks [NL][NL]
  {
    const Tables1D& t = m->tab;
    KronParams& kp = m->kp;
    std::memset(&kp, 0, sizeof kp);
    pack_eo(t.Mhat, n, kp.M);
    const double V = m->h[0] * m->h[1] * m->h[2];
    const int NL = m->NL;
    for (int dd = 0; dd < 3; ++dd) {
      const double sc = V / (m->h[dd] * m->h[dd]);
      double Ls[kMaxN * kMaxN];
      for (int q = 0; q < n * n; ++q) Ls[q] = sc * t.Lhat[q];
      pack_eo(Ls, n, kp.L[dd]);
      for (int i = 0; i < NL; ++i)
        for (int l = 0; l < NL; ++l) {
          kp.Nm[dd][i * NL + l] = sc * t.Nm[i * n + (n - NL + l)];
          kp.Np[dd][i * NL + l] = sc * t.Np[(n - NL + i) * n + l];
        }
    }
    double TiT[kMaxN * kMaxN];
    transpose(t.Tinv, n, TiT);
    pack_eo(TiT, n, kp.TiT);
    pack_eo(t.Tinv, n, kp.Ti);
    for (int dd = 0; dd < 3; ++dd) kp.cdir[dd] = V / (m->h[dd] * m->h[dd]);
    m->fdm_ok = m->cartesian && fdm_setup(t.Lhat, t.Mhat, n, kp);
    m->glt_ok = m->cartesian && NL == 2 && glt_setup(t, n, NL, m->h, kp);
  }

  // z sources and halo
  const bool zper = d->bc[2] == DG_BC_PERIODIC;
  if (nranks == 1) {
    m->zlo = m->zhi = zper ? ZSRC_LOCAL : ZSRC_MIRROR;
  } else {
    m->zlo = m->lo_peer >= 0 ? ZSRC_HALO : ZSRC_MIRROR;
    m->zhi = m->hi_peer >= 0 ? ZSRC_HALO : ZSRC_MIRROR;
  }
  cudaStream_t s = (cudaStream_t)d->stream;
  if (m->zlo == ZSRC_HALO || m->zhi == ZSRC_HALO) {
    m->halo_count = (int64_t)m->N[0] * m->N[1] * m->NL * n * n;
    const size_t bytes = sizeof(double) * (size_t)m->halo_count;
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&m->d_recv_lo, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&m->d_recv_hi, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&m->d_send_lo, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&m->d_send_hi, bytes);
    if (e != cudaSuccess) {
      dg_mesh_destroy(m);
      return fail(DG_ERR_CUDA, "halo alloc: %s", cudaGetErrorString(e));
    }
    cudaMemsetAsync(m->d_recv_lo, 0, bytes, s);
    cudaMemsetAsync(m->d_recv_hi, 0, bytes, s);
    if (d->nccl_unique_id) {
      ncclResult_t r = comm_acquire(d->nccl_unique_id, nranks, d->rank, &m->comm, &m->comm_key);
      if (r != ncclSuccess) {
        m->comm = nullptr;
        dg_mesh_destroy(m);
        return fail(DG_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
      }
      cudaError_t ce = cudaStreamCreateWithFlags(&m->comm_stream, cudaStreamNonBlocking);
      if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&m->ev_ready, cudaEventDisableTiming);
      if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&m->ev_halo, cudaEventDisableTiming);
      if (ce != cudaSuccess) {
        dg_mesh_destroy(m);
        return fail(DG_ERR_CUDA, "comm stream/events: %s", cudaGetErrorString(ce));
      }
    } else {
      m->external = true;
    }
  }
  if (m->geom == GEOM_PER_CELL) {
    const int64_t plane = (int64_t)m->N[0] * m->N[1];
    const int64_t cnt = plane * (m->nz + 2);
    std::vector<double> h(cnt * 10);
    if (d->user_inv_jac && nranks > 1) {
      dg_mesh_destroy(m);
      return fail(DG_ERR_UNSUPPORTED, "user_inv_jac with nranks > 1 (ghost-plane exchange) not in this build");
    }
    for (int64_t c = 0; c < cnt; ++c) {
      const int zl = (int)(c / plane) - 1;
      const int64_t rem = c % plane;
      double Ji[9];
      if (d->user_inv_jac) {
        int zs = zl;
        if (zs < 0) zs = (d->bc[2] == DG_BC_PERIODIC) ? m->nz - 1 : 0;
        if (zs >= m->nz) zs = (d->bc[2] == DG_BC_PERIODIC) ? 0 : m->nz - 1;
        std::memcpy(Ji, d->user_inv_jac + ((int64_t)zs * plane + rem) * 9, sizeof Ji);
      } else {
        std::memcpy(Ji, Ji0, sizeof Ji);
      }
      double Jm[9];
      const double dinv = inv3_host(Ji, Jm);      // det(J^-1)
      const double detJ = 1.0 / dinv;
      if (!(detJ > 0) || !std::isfinite(detJ)) {
        dg_mesh_destroy(m);
        return fail(DG_ERR_NUMERIC, "per-cell det J <= 0 or non-finite at cell %lld", (long long)c);
      }
      std::memcpy(&h[c * 10], Ji, sizeof Ji);
      h[c * 10 + 9] = detJ;
    }
    cudaError_t e1 = cudaMalloc(&m->d_jinv, sizeof(double) * h.size());
    if (e1 == cudaSuccess)
      e1 = cudaMemcpyAsync(m->d_jinv, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s);
    if (e1 == cudaSuccess) e1 = cudaStreamSynchronize(s);
    if (e1 != cudaSuccess) {
      dg_mesh_destroy(m);
      return fail(DG_ERR_CUDA, "per-cell geometry: %s", cudaGetErrorString(e1));
    }
    m->ga.jinv = m->d_jinv;
  }
  std::vector<double> usig[3];
  if (m->user_pen) {
    int bcv[3] = {d->bc[0], d->bc[1], d->bc[2]};
    dg_status st = build_user_sigma(d->user_penalty, m->N, m->nz, bcv, m->zlo == ZSRC_LOCAL, usig);
    if (st != DG_OK) {
      dg_mesh_destroy(m);
      return st;
    }
    for (int k = 0; k < 3; ++k) {
      cudaError_t e1 = cudaMalloc(&m->d_usig[k], sizeof(double) * std::max<size_t>(usig[k].size(), 1));
      if (e1 == cudaSuccess)
        e1 = cudaMemcpy(m->d_usig[k], usig[k].data(), sizeof(double) * usig[k].size(), cudaMemcpyHostToDevice);
      if (e1 != cudaSuccess) {
        dg_mesh_destroy(m);
        return fail(DG_ERR_CUDA, "user penalty upload: %s", cudaGetErrorString(e1));
      }
    }
    if (m->geom == GEOM_PER_CELL)
      for (int k = 0; k < 3; ++k) m->ga.sig[k] = m->d_usig[k];
  }
  if (m->geom == GEOM_PER_QPOINT) {
    const int64_t n3 = (int64_t)n * n * n;
    MapParams mp{};
    for (int k = 0; k < 9; ++k) mp.L[k] = L[k];
    for (int k = 0; k < 3; ++k) {
      mp.h[k] = m->h[k];
      mp.Nglob[k] = m->N[k];
      mp.bc[k] = d->bc[k];
    }
    mp.amp = d->deform_amp;
    mp.z0 = m->z_begin;
    mp.pen = pen;
    for (int q = 0; q < n; ++q) {
      mp.xq[q] = m->tab.xq[q];
      mp.wq[q] = m->tab.wq[q];
    }
    const int Nx = m->N[0], Ny = m->N[1], nz = m->nz;
    size_t fcount[3] = {(size_t)(Nx + 1) * Ny * nz, (size_t)Nx * (Ny + 1) * nz, (size_t)Nx * Ny * (nz + 1)};
    int* d_err = nullptr;
    cudaError_t e1 = cudaMalloc(&m->d_G, sizeof(double) * (size_t)(m->ncells_local * 6 * n3));
    for (int k = 0; k < 3 && e1 == cudaSuccess; ++k)
      e1 = cudaMalloc(&m->d_face[k], sizeof(double) * fcount[k] * 4 * n * n);
    if (e1 == cudaSuccess) e1 = cudaMalloc(&d_err, sizeof(int));
    if (e1 == cudaSuccess) e1 = cudaMemsetAsync(d_err, 0, sizeof(int), s);
    const double* const us[3] = {m->d_usig[0], m->d_usig[1], m->d_usig[2]};
    if (e1 == cudaSuccess) e1 = launch_geom_qpoint(n, mp, Nx, Ny, nz, m->d_G, m->d_face, us, d_err, s);
    int herr = 0;
    if (e1 == cudaSuccess) e1 = cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e1 == cudaSuccess) e1 = cudaStreamSynchronize(s);
    cudaFree(d_err);
    m->launches += 5;
    if (e1 != cudaSuccess) {
      dg_mesh_destroy(m);
      return fail(DG_ERR_CUDA, "per-q-point geometry: %s", cudaGetErrorString(e1));
    }
    if (herr) {
      dg_mesh_destroy(m);
      return fail(DG_ERR_NUMERIC, "det J <= 0 or non-finite at some quadrature point");
    }
    m->ga.G = m->d_G;
    for (int k = 0; k < 3; ++k) m->ga.face[k] = m->d_face[k];
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    dg_mesh_destroy(m);
    return fail(DG_ERR_CUDA, "setup sync: %s", cudaGetErrorString(e));
  }
  *out = m;
  return DG_OK;
}

dg_status dg_mesh_destroy(dg_mesh m) {
  if (!m) return DG_OK;
  cudaFree(m->d_G);
  for (int d = 0; d < 3; ++d) cudaFree(m->d_face[d]);
  cudaFree(m->d_jinv);
  for (int d = 0; d < 3; ++d) cudaFree(m->d_usig[d]);
  cudaFree(m->d_dinv_gl);
  cudaFree(m->d_bt);
  cudaFree(m->d_dinv_pj);
  cudaFree(m->d_dot);
  cudaFree(m->d_dinv_gl_f);
  cudaFree(m->d_dinv_pj_f);
  cudaFree(m->d_hu);
  cudaFree(m->d_hy);
  for (cudaEvent_t e : m->ev_h2d) cudaEventDestroy(e);
  for (cudaEvent_t e : m->ev_comp) cudaEventDestroy(e);
  if (m->ev_done) cudaEventDestroy(m->ev_done);
  if (m->h2d_stream) cudaStreamDestroy(m->h2d_stream);
  if (m->d2h_stream) cudaStreamDestroy(m->d2h_stream);
  cudaFree(m->d_recv_lo);
  cudaFree(m->d_recv_hi);
  cudaFree(m->d_send_lo);
  cudaFree(m->d_send_hi);
  if (m->comm) comm_release(m->comm_key);
  if (m->ev_ready) cudaEventDestroy(m->ev_ready);
  if (m->ev_halo) cudaEventDestroy(m->ev_halo);
  if (m->comm_stream) cudaStreamDestroy(m->comm_stream);
  delete m;
  return DG_OK;
}

dg_status dg_mesh_query(dg_mesh m, int64_t* nl, int64_t* ng, int32_t* zb, int32_t* ze) {
  if (!m) return fail(DG_ERR_PARAM, "NULL mesh");
  if (nl) *nl = m->ndofs_local;
  if (ng) *ng = m->ndofs_global;
  if (zb) *zb = m->z_begin;
  if (ze) *ze = m->z_end;
  return DG_OK;
}

int64_t dg_kernel_launch_count(dg_mesh m) { return m ? m->launches : -1; }

dg_status dg_slab_plan(int32_t Nz, int32_t nranks, int32_t rank, int32_t bc_z, int32_t degree,
                       int32_t basis, int32_t* out6) {
  if (!out6 || Nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || Nz < nranks || degree < 1 ||
      degree > 8)
    return fail(DG_ERR_PARAM, "bad slab plan arguments");
  int plan[4];
  slab_plan(Nz, nranks, rank, bc_z, plan);
  for (int k = 0; k < 4; ++k) out6[k] = plan[k];
  out6[4] = (basis == DG_BASIS_HERMITE_LIKE && degree >= 2) ? 2 : degree + 1;
  out6[5] = 0;
  return DG_OK;
}

dg_status dg_halo_pack_host(const double* u_slab, int32_t degree, int32_t basis, int32_t Nx, int32_t Ny,
                            int32_t nz, double* send_lo, double* send_hi) {
  if (!u_slab || degree < 1 || degree > 8 || Nx < 1 || Ny < 1 || nz < 1)
    return fail(DG_ERR_PARAM, "bad halo pack arguments");
  const int n = degree + 1;
  const int NL = (basis == DG_BASIS_HERMITE_LIKE && degree >= 2) ? 2 : n;
  const int64_t pc = (int64_t)Nx * Ny, total = pc * NL * n * n;
  for (int64_t e = 0; e < total; ++e) {
    if (send_lo) send_lo[e] = u_slab[halo_src(e, n, NL, pc, nz, false)];
    if (send_hi) send_hi[e] = u_slab[halo_src(e, n, NL, pc, nz, true)];
  }
  return DG_OK;
}

dg_status dg_mesh_query_halo(dg_mesh m, int64_t* count, int32_t* lo_peer, int32_t* hi_peer) {
  if (!m) return fail(DG_ERR_PARAM, "NULL mesh");
  if (count) *count = m->halo_count;
  if (lo_peer) *lo_peer = m->lo_peer;
  if (hi_peer) *hi_peer = m->hi_peer;
  return DG_OK;
}

dg_status dg_halo_pack(dg_mesh m, const double* u, double* send_lo, double* send_hi, void* stream) {
  if (!m || !u) return fail(DG_ERR_PARAM, "NULL argument");
  if (m->halo_count == 0) return DG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  return post_launch(m, launch_halo_pack(u, send_lo, send_hi, m->n, m->NL, (int64_t)m->N[0] * m->N[1],
                                         m->nz, s), "halo_pack", s);
}

dg_status dg_halo_set(dg_mesh m, const double* recv_lo, const double* recv_hi, void* stream) {
  if (!m) return fail(DG_ERR_PARAM, "NULL mesh");
  if (m->halo_count == 0) return DG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * (size_t)m->halo_count;
  if (recv_lo) CUDA_TRY(cudaMemcpyAsync(m->d_recv_lo, recv_lo, bytes, cudaMemcpyDeviceToDevice, s));
  if (recv_hi) CUDA_TRY(cudaMemcpyAsync(m->d_recv_hi, recv_hi, bytes, cudaMemcpyDeviceToDevice, s));
  return DG_OK;
}

dg_status dg_measure_peak(int32_t kind, double* value, void* stream) {
  if (!value || kind < 0 || (kind > 4 && (kind < 13 || kind > 18) && (kind < 23 || kind > 26))) return fail(DG_ERR_PARAM, "bad kind or NULL value");
  CUDA_TRY(measure_peak(kind, value, (cudaStream_t)stream));
  return DG_OK;
}

dg_status dg_tables_1d(int32_t degree, int32_t basis, double pf, double* out, int64_t out_len) {
  if (!out) return fail(DG_ERR_PARAM, "NULL out");
  Tables1D t;
  if (!build_tables(degree, basis, pf, &t)) return fail(DG_ERR_PARAM, "bad degree/basis");
  const int n = t.n;
  const int64_t need = 6 * n + 9 * n * n;
  if (out_len < need) return fail(DG_ERR_PARAM, "out_len %lld < %lld", (long long)out_len, (long long)need);
  double* o = out;
  auto put = [&](const double* a, int cnt) { std::memcpy(o, a, sizeof(double) * cnt); o += cnt; };
  put(t.xq, n); put(t.wq, n); put(t.S, n * n); put(t.DS, n * n);
  put(t.v0, n); put(t.v1, n); put(t.d0, n); put(t.d1, n);
  put(t.Mhat, n * n); put(t.Ahat, n * n); put(t.Lhat, n * n); put(t.Nm, n * n); put(t.Np, n * n);
  put(t.T, n * n); put(t.Tinv, n * n);
  return DG_OK;
}

dg_status dg_set_transport(dg_mesh m, const dg_transport* t) {
  if (!m) return fail(DG_ERR_PARAM, "NULL mesh");
  if (t && (!t->halo || !t->allreduce_sum)) return fail(DG_ERR_PARAM, "dg_transport needs both callbacks");
  if (t && !m->external) return fail(DG_ERR_PARAM, "dg_set_transport: mesh is not in external-transport mode");
  m->transport = t ? *t : dg_transport{};
  return DG_OK;
}

dg_status dg_halo_exchange(dg_mesh m, const double* u, void* stream) {
  if (!m || !u) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(u);
  return halo_exchange_impl(m, u, (cudaStream_t)stream);
}

dg_status dg_apply_laplace(dg_mesh m, const double* u, double* y, int32_t flags, void* stream) {
  if (!m || !u || !y) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(u);
  CHECK_ALIGNED(y);
  if (u == y) return fail(DG_ERR_PARAM, "u and y alias");
  if (flags & ~(DG_APPLY_HALO_READY | DG_APPLY_QUADRATURE)) return fail(DG_ERR_PARAM, "bad flags");
  cudaStream_t s = (cudaStream_t)stream;
  ChebyArgs ch{};
  const bool kron = m->cartesian && !(flags & DG_APPLY_QUADRATURE);
  return run_pass(m, KMODE_APPLY, kron, u, y, ch, (flags & DG_APPLY_HALO_READY) != 0, s);
}

dg_status dg_basis_change(dg_mesh m, int32_t op, const double* in, double* out, void* stream) {
  if (!m || !in || !out) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(in);
  CHECK_ALIGNED(out);
  const int n = m->n;
  const Tables1D& t = m->tab;
  double B[kMaxN * kMaxN];
  switch (op) {
    case DG_BCHG_H_TO_GL: std::memcpy(B, t.T, sizeof B); break;
    case DG_BCHG_GL_TO_H: std::memcpy(B, t.Tinv, sizeof B); break;
    case DG_BCHG_H_TO_GL_T: transpose(t.T, n, B); break;
    case DG_BCHG_GL_TO_H_T: transpose(t.Tinv, n, B); break;
    default: return fail(DG_ERR_PARAM, "bad basis-change op %d", op);
  }
  BchgParams bp{};
  pack_eo(B, n, bp.B);
  cudaStream_t s = (cudaStream_t)stream;
  // Three kernels: k_bchg (block-staged), the z-first k_bchg4 (out of place only) and the
  // warp-private pipelined k_bchgw / k_bchgp (k_bchgw.cu).  Default by measurement (C4, GB/s at
  // p = 2..8: k_bchg 4245/5869/4736/4925/4435/5855/4853, k_bchg4 4477/5188/4185/4856/4186/4471/5231,
  // k_bchgw.cu in its per-n default mode 6364/6321/6557/6326/6418/6206/5904 = 0.90-1.00 of the
  // measured copy bandwidth): k_bchgw.cu for n >= 3, k_bchg for n = 2; DG_BCHG=1 / 4 / 5 force one.
  static const int v = [] {
    const char* e = std::getenv("DG_BCHG");
    return e ? std::atoi(e) : 0;
  }();
  const bool usew = v == 5 || (v == 0 && n >= 3);
  if (usew)
    return post_launch(m, launch_basis_change_w(n, bp, in, out, m->ncells_local, s), "basis_change", s);
  if (v == 4 && in != out && kron4_supported(n))
    return post_launch(m, launch_basis_change4(n, bp, in, out, m->ncells_local, s), "basis_change", s);
  return post_launch(m, launch_basis_change(n, bp, in, out, m->ncells_local, s), "basis_change", s);
}

dg_status dg_basis_change_f32(dg_mesh m, int32_t op, const float* in, float* out, void* stream) {
  if (!m || !in || !out) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(in);
  CHECK_ALIGNED(out);
  const int n = m->n;
  const Tables1D& t = m->tab;
  double B[kMaxN * kMaxN];
  switch (op) {
    case DG_BCHG_H_TO_GL: std::memcpy(B, t.T, sizeof B); break;
    case DG_BCHG_GL_TO_H: std::memcpy(B, t.Tinv, sizeof B); break;
    case DG_BCHG_H_TO_GL_T: transpose(t.T, n, B); break;
    case DG_BCHG_GL_TO_H_T: transpose(t.Tinv, n, B); break;
    default: return fail(DG_ERR_PARAM, "bad basis-change op %d", op);
  }
  BchgParams bp{};
  pack_eo(B, n, bp.B);
  BchgParamsF bf{};
  for (int k = 0; k < kEO; ++k) bf.B[k] = (float)bp.B[k];
  cudaStream_t s = (cudaStream_t)stream;
  static const int v = [] {
    const char* e = std::getenv("DG_BCHG");
    return e ? std::atoi(e) : 0;
  }();
  // fp32 default by measurement (C4, GB/s at 8 B/DoF, p = 2..8: k_bchg 2993/4419/3908/3475/3489/4941/3844,
  // k_bchgw.cu plane mode with two slots 5150/3281/5014/3953/4994/5045/4560): k_bchg at n = 2 and 4
  if (v == 5 || (v == 0 && n >= 3 && n != 4))
    return post_launch(m, launch_basis_change_w_f32(n, bf, in, out, m->ncells_local, s), "basis_change_f32", s);
  return post_launch(m, launch_basis_change_f32(n, bf, in, out, m->ncells_local, s), "basis_change_f32", s);
}

dg_status dg_inverse_diagonal(dg_mesh m, int32_t inner, double* out, void* stream) {
  if (!m || !out) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(out);
  cudaStream_t s = (cudaStream_t)stream;
  const bool gl = inner == DG_INNER_GL_JACOBI;
  if (!gl && inner != DG_INNER_POINT_JACOBI) return fail(DG_ERR_PARAM, "bad inner %d", inner);
  double** dst = gl ? &m->d_dinv_gl : &m->d_dinv_pj;
  dg_status st = build_diag(m, gl, dst, s);
  if (st != DG_OK) return st;
  CUDA_TRY(cudaMemcpyAsync(out, *dst, sizeof(double) * (size_t)m->ndofs_local,
                           cudaMemcpyDeviceToDevice, s));
  return DG_OK;
}

dg_status dg_chebyshev_smooth(dg_mesh m, const double* b, double* x, double* work2, int32_t degree,
                              double lambda_max, double lo_frac, double hi_frac, int32_t inner,
                              void* stream) {
  if (!m || !b || !x || !work2) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(b);
  CHECK_ALIGNED(x);
  CHECK_ALIGNED(work2);
  if (degree < 0) return fail(DG_ERR_PARAM, "degree < 0");
  const double alpha = lo_frac * lambda_max, beta = hi_frac * lambda_max;
  if (!(alpha > 0 && beta > alpha) || !std::isfinite(beta))
    return fail(DG_ERR_PARAM, "need 0 < lo_frac*lambda_max < hi_frac*lambda_max");
  if (inner != DG_INNER_GL_JACOBI && inner != DG_INNER_POINT_JACOBI && inner != DG_INNER_FDM)
    return fail(DG_ERR_PARAM, "bad inner %d", inner);
  if (inner == DG_INNER_FDM && !(m->fdm_ok && kron_v4(m->n)))
    return fail(DG_ERR_UNSUPPORTED, "DG_INNER_FDM needs a Cartesian mesh, degree 2..8 and the k_kron4 path");
  const int64_t nd = m->ndofs_local;
  double* W0 = work2;
  double* W1 = work2 + nd;
  if ((b >= W0 && b < W1 + nd) || (x >= W0 && x < W1 + nd) || b == x)
    return fail(DG_ERR_PARAM, "b, x and work2 must not overlap");
  if (degree == 0) return DG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const bool fdm = inner == DG_INNER_FDM;
  const bool gl = inner == DG_INNER_GL_JACOBI && m->desc.basis == DG_BASIS_HERMITE_LIKE;
  double* dnone = nullptr;
  double** dsrc = fdm ? &dnone : (gl ? &m->d_dinv_gl : &m->d_dinv_pj);
  dg_status st = fdm ? DG_OK : build_diag(m, inner == DG_INNER_GL_JACOBI, dsrc, s);
  if (st != DG_OK) return st;
  int mode = fdm ? KMODE_CHEBY_FDM : (gl ? KMODE_CHEBY_GL : KMODE_CHEBY_PJ);
  // GL-Jacobi on the k_kron4 path: transform the rhs once, b~ = (T^{-T})^{(x)3} b, and run the
  // steps on the transformed residual (KMODE_CHEBY_GLT: three P^{-1} sweeps and two
  // transposes fewer per step).  DG_CHEBY_GLT=0 keeps the direct step.
  const double* bstep = b;
  if (mode == KMODE_CHEBY_GL && glt_use(m)) {
    if (!m->d_bt) CUDA_TRY(cudaMalloc(&m->d_bt, sizeof(double) * (size_t)std::max<int64_t>(nd, 1)));
    st = dg_basis_change(m, DG_BCHG_GL_TO_H_T, b, m->d_bt, stream);
    if (st != DG_OK) return st;
    bstep = m->d_bt;
    mode = KMODE_CHEBY_GLT;
  }

  // storage of u_j so that u_degree lands in x (in-place updates over u_{j-1})
  double* buf[3] = {x, W0, W1};
  std::vector<int> where(degree + 1);
  where[0] = 0;
  if (degree == 1) {
    where[1] = 1;
  } else if (degree % 2 == 0) {
    for (int j = 1; j <= degree; ++j) where[j] = (j % 2 == 1) ? 1 : 0;
  } else {
    where[1] = 1;
    where[2] = 2;
    for (int j = 3; j <= degree; ++j) where[j] = (j % 2 == 1) ? 0 : 2;
  }
  const double c = 0.5 * (beta + alpha), delta = 0.5 * (beta - alpha);
  const double sigma1 = c / delta;
  double rho = 1.0 / sigma1;
  for (int j = 0; j < degree; ++j) {
    ChebyArgs ch{};
    ch.b = bstep;
    ch.dinv = *dsrc;
    ch.u_next = buf[where[j + 1]];
    if (j == 0) {
      ch.first = 1;
      ch.c_z = 1.0 / c;
      ch.c_prev = 0.0;
      ch.u_prev = nullptr;
    } else {
      const double rho_n = 1.0 / (2.0 * sigma1 - rho);
      ch.first = 0;
      ch.c_prev = rho_n * rho;
      ch.c_z = 2.0 * rho_n / delta;
      ch.u_prev = buf[where[j - 1]];
      rho = rho_n;
    }
    const double* uj = buf[where[j]];
    st = run_pass(m, mode, m->cartesian, uj, nullptr, ch, false, s);
    if (st != DG_OK) return st;
  }
  if (where[degree] != 0)
    CUDA_TRY(cudaMemcpyAsync(x, buf[where[degree]], sizeof(double) * (size_t)nd,
                             cudaMemcpyDeviceToDevice, s));
  return DG_OK;
}

}  // extern "C"

namespace {

dg_status halo_exchange_impl(dg_mesh m, const double* u, cudaStream_t s) {
  if (m->zlo != ZSRC_HALO && m->zhi != ZSRC_HALO) return DG_OK;
  if (m->external && !m->transport.halo)
    return fail(DG_ERR_UNSUPPORTED, "external halo transport: call dg_halo_pack/dg_halo_set and "
                                    "DG_APPLY_HALO_READY, or install a dg_transport");
  const int64_t plane_cells = (int64_t)m->N[0] * m->N[1];
  if (m->external) {   // caller's transport: pack here, the callback fills recv_lo / recv_hi
    cudaError_t e = launch_halo_pack(u, m->lo_peer >= 0 ? m->d_send_lo : nullptr,
                                     m->hi_peer >= 0 ? m->d_send_hi : nullptr, m->n, m->NL, plane_cells,
                                     m->nz, s);
    if (e != cudaSuccess) return fail(DG_ERR_CUDA, "halo pack: %s", cudaGetErrorString(e));
    m->launches++;
    const bool lo = m->lo_peer >= 0, hi = m->hi_peer >= 0;
    if (m->transport.halo(m->transport.user, lo ? m->d_send_lo : nullptr, hi ? m->d_send_hi : nullptr,
                          lo ? m->d_recv_lo : nullptr, hi ? m->d_recv_hi : nullptr, m->halo_count, s) != 0)
      return fail(DG_ERR_NCCL, "transport failed (halo callback returned non-zero)");
    return DG_OK;
  }
  cudaError_t e = launch_halo_pack(u, m->lo_peer >= 0 ? m->d_send_lo : nullptr,
                                   m->hi_peer >= 0 ? m->d_send_hi : nullptr, m->n, m->NL, plane_cells,
                                   m->nz, s);
  if (e != cudaSuccess) return fail(DG_ERR_CUDA, "halo pack: %s", cudaGetErrorString(e));
  m->launches++;
  const size_t cnt = (size_t)m->halo_count;
  NCCL_TRY(ncclGroupStart());
  // "up": top layers to the upper peer, lower peer's top layers into recv_lo
  if (m->hi_peer >= 0) NCCL_TRY(ncclSend(m->d_send_hi, cnt, ncclDouble, m->hi_peer, m->comm, s));
  if (m->lo_peer >= 0) NCCL_TRY(ncclRecv(m->d_recv_lo, cnt, ncclDouble, m->lo_peer, m->comm, s));
  // "down": bottom layers to the lower peer, upper peer's bottom layers into recv_hi
  if (m->lo_peer >= 0) NCCL_TRY(ncclSend(m->d_send_lo, cnt, ncclDouble, m->lo_peer, m->comm, s));
  if (m->hi_peer >= 0) NCCL_TRY(ncclRecv(m->d_recv_hi, cnt, ncclDouble, m->hi_peer, m->comm, s));
  NCCL_TRY(ncclGroupEnd());
  if (debug_sync()) CUDA_TRY(cudaStreamSynchronize(s));
  return DG_OK;
}

// One operator pass (apply or fused Chebyshev step) over the owned planes.  With an
// NCCL halo the exchange runs on the comm stream while the interior planes compute;
// the two boundary planes follow once the halo has arrived.
dg_status run_pass(dg_mesh m, int mode, bool kron, const double* u, double* y, const ChebyArgs& ch,
                   bool halo_ready, cudaStream_t s) {
  auto launch = [&](int zb, int ze) -> dg_status {
    if (ze <= zb) return DG_OK;
    GridArgs g = grid_args(m, zb, ze);
    cudaError_t e;
    if (mode == KMODE_CHEBY_GLT)
      e = launch_kron4(m->n, m->NL, mode, m->kp, g, u, y, ch, s);
    else if (kron && kron3c_use(m->n, m->NL))
      e = launch_kron3c(m->NL, mode, m->kp, g, u, y, ch, s);
    else if (kron && kron6_use(m->n, m->NL, mode))
      e = launch_kron6(m->n, mode, m->kp, g, u, y, ch, s);
    else if (kron && kron_v4(m->n))
      e = launch_kron4(m->n, m->NL, mode, m->kp, g, u, y, ch, s);
    else if (quad_v3(m->n, m->geom))
      e = launch_quad3(m->n, m->NL, m->geom, mode, m->qp, m->ga, g, u, y, ch, s);
    else
      e = launch_quad(m->n, m->NL, m->geom, mode, m->qp, m->ga, g, u, y, ch, s);
    return post_launch(m, e, kron ? "kron" : "quad", s);
  };
  const bool need = (m->zlo == ZSRC_HALO || m->zhi == ZSRC_HALO) && !halo_ready;
  if (!need) return launch(0, m->nz);
  if (m->external) {   // caller's transport: exchange first, then every plane
    dg_status st = halo_exchange_impl(m, u, s);
    if (st != DG_OK) return st;
    return launch(0, m->nz);
  }
  CUDA_TRY(cudaEventRecord(m->ev_ready, s));
  CUDA_TRY(cudaStreamWaitEvent(m->comm_stream, m->ev_ready, 0));
  dg_status st = halo_exchange_impl(m, u, m->comm_stream);
  if (st != DG_OK) return st;
  CUDA_TRY(cudaEventRecord(m->ev_halo, m->comm_stream));
  const int zi0 = m->zlo == ZSRC_HALO ? 1 : 0;
  const int zi1 = m->zhi == ZSRC_HALO ? m->nz - 1 : m->nz;
  if (zi1 > zi0) {
    st = launch(zi0, zi1);
    if (st != DG_OK) return st;
  }
  CUDA_TRY(cudaStreamWaitEvent(s, m->ev_halo, 0));
  if (zi1 <= zi0) return launch(0, m->nz);
  st = launch(0, zi0);
  if (st != DG_OK) return st;
  return launch(zi1, m->nz);
}

}  // namespace

// ================================================================ solvers (NEXT#4)
// GPU Lanczos estimate of lambda_max(P^{-1}A) and preconditioned CG with the Chebyshev
// sweep as preconditioner.
namespace {

dg_status pinv_impl(dg_mesh m, int inner, const double* r, double* z, cudaStream_t s) {
  if (inner == DG_INNER_FDM) {
    if (!m->fdm_ok) return fail(DG_ERR_UNSUPPORTED, "DG_INNER_FDM needs a Cartesian mesh");
    return post_launch(m, launch_pinv(m->n, DG_INNER_FDM, m->kp, r, nullptr, z, m->ncells_local, s), "pinv", s);
  }
  const bool gl = inner == DG_INNER_GL_JACOBI && m->desc.basis == DG_BASIS_HERMITE_LIKE;
  double** dsrc = gl ? &m->d_dinv_gl : &m->d_dinv_pj;
  dg_status st = build_diag(m, inner == DG_INNER_GL_JACOBI, dsrc, s);
  if (st != DG_OK) return st;
  return post_launch(m, launch_pinv(m->n, gl ? DG_INNER_GL_JACOBI : DG_INNER_POINT_JACOBI, m->kp, r, *dsrc, z,
                                    m->ncells_local, s), "pinv", s);
}

dg_status dot_impl(dg_mesh m, const double* a, const double* b, double* out, cudaStream_t s) {
  if (!m->d_dot) CUDA_TRY(cudaMalloc(&m->d_dot, sizeof(double) * (dot_partials() + 1)));
  double* res = m->d_dot + dot_partials();
  dg_status st = post_launch(m, launch_dot(a, b, m->ndofs_local, m->d_dot, res, s), "dot", s);
  if (st != DG_OK) return st;
  m->launches++;   // two kernels
  if (m->nranks > 1) {
    if (m->comm) {
      NCCL_TRY(ncclAllReduce(res, res, 1, ncclDouble, ncclSum, m->comm, s));
    } else if (!m->transport.allreduce_sum) {
      return fail(DG_ERR_UNSUPPORTED, "global dot products need the NCCL communicator or a dg_transport");
    }
  }
  CUDA_TRY(cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (m->nranks > 1 && !m->comm && m->transport.allreduce_sum(m->transport.user, out) != 0)
    return fail(DG_ERR_NCCL, "transport failed (allreduce_sum callback returned non-zero)");
  return DG_OK;
}

dg_status axpby(dg_mesh m, double a, const double* x, double b, double* y, cudaStream_t s) {
  return post_launch(m, launch_axpby(a, x, b, y, m->ndofs_local, s), "axpby", s);
}

// largest eigenvalue of the symmetric tridiagonal (alpha, beta) by cyclic Jacobi
double tridiag_max_eig(const std::vector<double>& al, const std::vector<double>& be) {
  const int k = (int)al.size();
  std::vector<long double> A((size_t)k * k, 0.0L);
  for (int i = 0; i < k; ++i) {
    A[i * k + i] = al[i];
    if (i + 1 < k) A[i * k + i + 1] = A[(i + 1) * k + i] = be[i];
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    long double off = 0;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) off += A[p * k + q] * A[p * k + q];
    if (off < 1e-60L) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        if (A[p * k + q] == 0) continue;
        const long double th = (A[q * k + q] - A[p * k + p]) / (2 * A[p * k + q]);
        const long double t = (th >= 0 ? 1 : -1) / (std::fabs(th) + std::sqrt(th * th + 1));
        const long double c = 1 / std::sqrt(t * t + 1), sn = t * c;
        for (int r = 0; r < k; ++r) {
          const long double ap = A[r * k + p], aq = A[r * k + q];
          A[r * k + p] = c * ap - sn * aq;
          A[r * k + q] = sn * ap + c * aq;
        }
        for (int r = 0; r < k; ++r) {
          const long double ap = A[p * k + r], aq = A[q * k + r];
          A[p * k + r] = c * ap - sn * aq;
          A[q * k + r] = sn * ap + c * aq;
        }
      }
  }
  long double mx = A[0];
  for (int i = 1; i < k; ++i) mx = std::max(mx, A[i * k + i]);
  return (double)mx;
}

struct DevVecs {
  std::vector<double*> v;
  ~DevVecs() {
    for (double* p : v) cudaFree(p);
  }
};

}  // namespace

extern "C" {

dg_status dg_apply_preconditioner(dg_mesh m, int32_t inner, const double* r, double* z, void* stream) {
  if (!m || !r || !z) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(r);
  CHECK_ALIGNED(z);
  if (inner != DG_INNER_GL_JACOBI && inner != DG_INNER_POINT_JACOBI && inner != DG_INNER_FDM)
    return fail(DG_ERR_PARAM, "bad inner %d", inner);
  return pinv_impl(m, inner, r, z, (cudaStream_t)stream);
}

dg_status dg_dot(dg_mesh m, const double* a, const double* b, double* out, void* stream) {
  if (!m || !a || !b || !out) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(a);
  CHECK_ALIGNED(b);
  return dot_impl(m, a, b, out, (cudaStream_t)stream);
}

dg_status dg_lanczos_lambda_max(dg_mesh m, int32_t inner, int32_t iters, double* lambda_max, void* stream) {
  if (!m || !lambda_max) return fail(DG_ERR_PARAM, "NULL argument");
  if (iters < 1 || iters > 200) return fail(DG_ERR_PARAM, "iters %d not in 1..200", iters);
  if (inner != DG_INNER_GL_JACOBI && inner != DG_INNER_POINT_JACOBI && inner != DG_INNER_FDM)
    return fail(DG_ERR_PARAM, "bad inner %d", inner);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nd = m->ndofs_local;
  DevVecs w;
  for (int i = 0; i < 5; ++i) {
    double* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, sizeof(double) * (size_t)std::max<int64_t>(nd, 1)));
    w.v.push_back(p);
  }
  double *v = w.v[0], *vp = w.v[1], *z = w.v[2], *ww = w.v[3], *wz = w.v[4];
  const int64_t plane_dofs = (int64_t)m->N[0] * m->N[1] * m->n * m->n * m->n;
  dg_status st = post_launch(m, launch_lanczos_start(v, nd, (int64_t)m->z_begin * plane_dofs, s), "lanczos", s);
  if (st != DG_OK) return st;
  if ((st = pinv_impl(m, inner, v, z, s)) != DG_OK) return st;
  double vz;
  if ((st = dot_impl(m, v, z, &vz, s)) != DG_OK) return st;
  if (!(vz > 0)) return fail(DG_ERR_NUMERIC, "P^-1 not positive definite in Lanczos");
  double beta = std::sqrt(vz);
  if ((st = axpby(m, 0.0, v, 1.0 / beta, v, s)) != DG_OK) return st;
  if ((st = axpby(m, 0.0, z, 1.0 / beta, z, s)) != DG_OK) return st;
  CUDA_TRY(cudaMemsetAsync(vp, 0, sizeof(double) * (size_t)nd, s));
  std::vector<double> al, be;
  double b_prev = 0.0;
  ChebyArgs none{};
  for (int it = 0; it < iters; ++it) {
    if ((st = run_pass(m, KMODE_APPLY, m->cartesian, z, ww, none, false, s)) != DG_OK) return st;
    double a;
    if ((st = dot_impl(m, ww, z, &a, s)) != DG_OK) return st;
    if ((st = axpby(m, -a, v, 1.0, ww, s)) != DG_OK) return st;
    if ((st = axpby(m, -b_prev, vp, 1.0, ww, s)) != DG_OK) return st;
    if ((st = pinv_impl(m, inner, ww, wz, s)) != DG_OK) return st;
    double wwz;
    if ((st = dot_impl(m, ww, wz, &wwz, s)) != DG_OK) return st;
    const double b = std::sqrt(std::max(wwz, 0.0));
    al.push_back(a);
    if (b < 1e-300) break;
    be.push_back(b);
    std::swap(vp, v);                      // v_prev <- v
    if ((st = axpby(m, 1.0 / b, ww, 0.0, v, s)) != DG_OK) return st;   // v <- w / b
    if ((st = axpby(m, 1.0 / b, wz, 0.0, z, s)) != DG_OK) return st;   // z <- wz / b
    b_prev = b;
  }
  *lambda_max = tridiag_max_eig(al, be);
  return DG_OK;
}

}  // extern "C"

namespace {

dg_status f32_check(dg_mesh m);

// CG around the Chebyshev sweep (mixed: the sweep runs in fp32, CG in fp64)
dg_status pcg_impl(dg_mesh m, const double* b, double* x, double rel_tol, int32_t max_iter, int32_t cheby_degree,
                   double lambda_max, double lo_frac, double hi_frac, int32_t inner, int32_t* iters,
                   double* rel_res, cudaStream_t s, bool mixed) {
  if (!m || !b || !x) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(b);
  CHECK_ALIGNED(x);
  if (max_iter < 0 || cheby_degree < 1) return fail(DG_ERR_PARAM, "max_iter < 0 or cheby_degree < 1");
  if (b == x) return fail(DG_ERR_PARAM, "b and x must not alias");
  if (mixed) {
    dg_status st = f32_check(m);
    if (st != DG_OK) return st;
  }
  const int64_t nd = m->ndofs_local;
  DevVecs w;
  for (int i = 0; i < 4; ++i) {
    double* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, sizeof(double) * (size_t)std::max<int64_t>(nd, 1)));
    w.v.push_back(p);
  }
  double* work2 = nullptr;
  CUDA_TRY(cudaMalloc(&work2, sizeof(double) * (size_t)std::max<int64_t>(2 * nd, 1)));
  w.v.push_back(work2);
  double *r = w.v[0], *z = w.v[1], *p = w.v[2], *q = w.v[3];
  // fp32 buffers of the mixed variant (r32, z32 and the sweep's two work vectors) in work2's space
  float* r32 = reinterpret_cast<float*>(work2);
  float* z32 = r32 + ((nd + 3) & ~int64_t(3));
  float* w32 = nullptr;
  if (mixed) {
    double* tmp = nullptr;
    CUDA_TRY(cudaMalloc(&tmp, sizeof(double) * (size_t)std::max<int64_t>(nd + 4, 1)));
    w.v.push_back(tmp);
    w32 = reinterpret_cast<float*>(tmp);
  }
  ChebyArgs none{};
  auto precond = [&](const double* rin, double* zout) -> dg_status {   // z = Chebyshev sweep from 0
    if (!mixed) {
      CUDA_TRY(cudaMemsetAsync(zout, 0, sizeof(double) * (size_t)nd, s));
      return dg_chebyshev_smooth(m, rin, zout, work2, cheby_degree, lambda_max, lo_frac, hi_frac, inner, s);
    }
    dg_status st = post_launch(m, launch_d2f(rin, r32, nd, s), "d2f", s);
    if (st != DG_OK) return st;
    CUDA_TRY(cudaMemsetAsync(z32, 0, sizeof(float) * (size_t)nd, s));
    st = dg_chebyshev_smooth_f32(m, r32, z32, w32, cheby_degree, lambda_max, lo_frac, hi_frac, inner, s);
    if (st != DG_OK) return st;
    return post_launch(m, launch_f2d(z32, zout, nd, s), "f2d", s);
  };
  dg_status st;
  // r = b - A x
  if ((st = run_pass(m, KMODE_APPLY, m->cartesian, x, r, none, false, s)) != DG_OK) return st;
  if ((st = axpby(m, 1.0, b, -1.0, r, s)) != DG_OK) return st;
  double rr0;
  if ((st = dot_impl(m, r, r, &rr0, s)) != DG_OK) return st;
  const double r0 = std::sqrt(rr0);
  double res = r0 > 0 ? 1.0 : 0.0;
  int k = 0;
  if (r0 > 0 && max_iter > 0) {
    if ((st = precond(r, z)) != DG_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(p, z, sizeof(double) * (size_t)nd, cudaMemcpyDeviceToDevice, s));
    double rz;
    if ((st = dot_impl(m, r, z, &rz, s)) != DG_OK) return st;
    for (k = 1; k <= max_iter; ++k) {
      if ((st = run_pass(m, KMODE_APPLY, m->cartesian, p, q, none, false, s)) != DG_OK) return st;
      double pq;
      if ((st = dot_impl(m, p, q, &pq, s)) != DG_OK) return st;
      if (!(pq > 0)) return fail(DG_ERR_NUMERIC, "CG breakdown: p.Ap = %g", pq);
      const double alpha = rz / pq;
      if ((st = axpby(m, alpha, p, 1.0, x, s)) != DG_OK) return st;
      if ((st = axpby(m, -alpha, q, 1.0, r, s)) != DG_OK) return st;
      double rr;
      if ((st = dot_impl(m, r, r, &rr, s)) != DG_OK) return st;
      res = std::sqrt(rr) / r0;
      if (res <= rel_tol || k == max_iter) break;
      if ((st = precond(r, z)) != DG_OK) return st;
      double rz_new;
      if ((st = dot_impl(m, r, z, &rz_new, s)) != DG_OK) return st;
      const double beta = rz_new / rz;
      if ((st = axpby(m, 1.0, z, beta, p, s)) != DG_OK) return st;   // p = z + beta p
      rz = rz_new;
    }
    if (k > max_iter) k = max_iter;
  }
  if (iters) *iters = k;
  if (rel_res) *rel_res = res;
  return DG_OK;
}

}  // namespace

extern "C" {

dg_status dg_pcg(dg_mesh m, const double* b, double* x, double rel_tol, int32_t max_iter, int32_t cheby_degree,
                 double lambda_max, double lo_frac, double hi_frac, int32_t inner, int32_t* iters, double* rel_res,
                 void* stream) {
  return pcg_impl(m, b, x, rel_tol, max_iter, cheby_degree, lambda_max, lo_frac, hi_frac, inner, iters, rel_res,
                  (cudaStream_t)stream, false);
}

dg_status dg_pcg_mixed(dg_mesh m, const double* b, double* x, double rel_tol, int32_t max_iter,
                       int32_t cheby_degree, double lambda_max, double lo_frac, double hi_frac, int32_t inner,
                       int32_t* iters, double* rel_res, void* stream) {
  return pcg_impl(m, b, x, rel_tol, max_iter, cheby_degree, lambda_max, lo_frac, hi_frac, inner, iters, rel_res,
                  (cudaStream_t)stream, true);
}

}  // extern "C"

// ================================================================ fp32 path (NEXT#3)
// The Cartesian matvec and the fused Chebyshev smoother in single precision (the paper runs
// its smoothers and V-cycle in fp32): the same k_kron4
// kernels instantiated for float, with the 1D tables rounded once from the fp64 setup.
namespace {

dg_status f32_check(dg_mesh m) {
  if (!m->cartesian || !kron_v4(m->n))
    return fail(DG_ERR_UNSUPPORTED, "fp32 path: Cartesian meshes of degree 2..8 on the k_kron4 path only");
  if (m->zlo == ZSRC_HALO || m->zhi == ZSRC_HALO)
    return fail(DG_ERR_UNSUPPORTED, "fp32 path: single z-slab only (no fp32 halo buffers)");
  if (!m->kpf_ok) {
    const double* src = reinterpret_cast<const double*>(&m->kp);
    float* dst = reinterpret_cast<float*>(&m->kpf);
    static_assert(sizeof(KronParams) == 2 * sizeof(KronParamsF), "KronParams layout");
    for (size_t i = 0; i < sizeof(KronParams) / sizeof(double); ++i) dst[i] = (float)src[i];
    m->kpf_ok = true;
  }
  return DG_OK;
}

}  // namespace

extern "C" {

dg_status dg_apply_laplace_f32(dg_mesh m, const float* u, float* y, void* stream) {
  if (!m || !u || !y) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(u);
  CHECK_ALIGNED(y);
  if (u == y) return fail(DG_ERR_PARAM, "u and y must not alias");
  dg_status st = f32_check(m);
  if (st != DG_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  GridArgs g = grid_args(m, 0, m->nz);
  ChebyArgsF ch{};
  return post_launch(m, launch_kron4_f32(m->n, m->NL, KMODE_APPLY, m->kpf, g, u, y, ch, s), "kron4_f32", s);
}

dg_status dg_chebyshev_smooth_f32(dg_mesh m, const float* b, float* x, float* work2, int32_t degree,
                                  double lambda_max, double lo_frac, double hi_frac, int32_t inner,
                                  void* stream) {
  if (!m || !b || !x || !work2) return fail(DG_ERR_PARAM, "NULL argument");
  CHECK_ALIGNED(b);
  CHECK_ALIGNED(x);
  CHECK_ALIGNED(work2);
  if (degree < 0) return fail(DG_ERR_PARAM, "degree < 0");
  const double alpha = lo_frac * lambda_max, beta = hi_frac * lambda_max;
  if (!(alpha > 0 && beta > alpha) || !std::isfinite(beta))
    return fail(DG_ERR_PARAM, "need 0 < lo_frac*lambda_max < hi_frac*lambda_max");
  if (inner != DG_INNER_GL_JACOBI && inner != DG_INNER_POINT_JACOBI && inner != DG_INNER_FDM)
    return fail(DG_ERR_PARAM, "bad inner %d", inner);
  dg_status st = f32_check(m);
  if (st != DG_OK) return st;
  if (inner == DG_INNER_FDM && !m->fdm_ok) return fail(DG_ERR_UNSUPPORTED, "FDM tables missing");
  const int64_t nd = m->ndofs_local;
  float* W0 = work2;
  float* W1 = work2 + nd;
  if ((b >= W0 && b < W1 + nd) || (x >= W0 && x < W1 + nd) || b == x)
    return fail(DG_ERR_PARAM, "b, x and work2 must not overlap");
  if (degree == 0) return DG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const bool fdm = inner == DG_INNER_FDM;
  const bool gl = inner == DG_INNER_GL_JACOBI && m->desc.basis == DG_BASIS_HERMITE_LIKE;
  float* dinv = nullptr;
  if (!fdm) {   // fp32 copy of the fp64 inverse diagonal
    double** dsrc = gl ? &m->d_dinv_gl : &m->d_dinv_pj;
    float** fdst = gl ? &m->d_dinv_gl_f : &m->d_dinv_pj_f;
    if ((st = build_diag(m, inner == DG_INNER_GL_JACOBI, dsrc, s)) != DG_OK) return st;
    if (!*fdst) {
      CUDA_TRY(cudaMalloc(fdst, sizeof(float) * (size_t)std::max<int64_t>(nd, 1)));
      if ((st = post_launch(m, launch_d2f(*dsrc, *fdst, nd, s), "d2f", s)) != DG_OK) return st;
    }
    dinv = *fdst;
  }
  const int mode = fdm ? KMODE_CHEBY_FDM : (gl ? KMODE_CHEBY_GL : KMODE_CHEBY_PJ);
  float* buf[3] = {x, W0, W1};
  std::vector<int> where(degree + 1);
  where[0] = 0;
  if (degree == 1) {
    where[1] = 1;
  } else if (degree % 2 == 0) {
    for (int j = 1; j <= degree; ++j) where[j] = (j % 2 == 1) ? 1 : 0;
  } else {
    where[1] = 1;
    where[2] = 2;
    for (int j = 3; j <= degree; ++j) where[j] = (j % 2 == 1) ? 0 : 2;
  }
  const double c = 0.5 * (beta + alpha), delta = 0.5 * (beta - alpha);
  const double sigma1 = c / delta;
  double rho = 1.0 / sigma1;
  GridArgs g = grid_args(m, 0, m->nz);
  for (int j = 0; j < degree; ++j) {
    ChebyArgsF ch{};
    ch.b = b;
    ch.dinv = dinv;
    ch.u_next = buf[where[j + 1]];
    if (j == 0) {
      ch.first = 1;
      ch.c_z = 1.0 / c;
      ch.c_prev = 0.0;
      ch.u_prev = nullptr;
    } else {
      const double rho_n = 1.0 / (2.0 * sigma1 - rho);
      ch.first = 0;
      ch.c_prev = rho_n * rho;
      ch.c_z = 2.0 * rho_n / delta;
      ch.u_prev = buf[where[j - 1]];
      rho = rho_n;
    }
    st = post_launch(m, launch_kron4_f32(m->n, m->NL, mode, m->kpf, g, buf[where[j]], nullptr, ch, s),
                     "kron4_f32", s);
    if (st != DG_OK) return st;
  }
  if (where[degree] != 0)
    CUDA_TRY(cudaMemcpyAsync(x, buf[where[degree]], sizeof(float) * (size_t)nd, cudaMemcpyDeviceToDevice, s));
  return DG_OK;
}

}  // extern "C"

// ================================================================ host-buffer matvec
// y_host = A u_host with the host<->device copies inside the call, overlapped plane-chunk by
// plane-chunk with the kernels: H2D of chunk c+1 on one copy stream while chunk c computes
// (it needs the first plane of chunk c+1 as its z-neighbour) and the D2H of chunk c-1 drains
// on a second copy stream.  Pinned host memory makes the copies asynchronous (pageable memory
// is accepted and copied synchronously by the driver).
namespace {

dg_status launch_apply_range(dg_mesh m, bool kron, const double* u, double* y, int zb, int ze, cudaStream_t s) {
  if (ze <= zb) return DG_OK;
  GridArgs g = grid_args(m, zb, ze);
  ChebyArgs ch{};
  cudaError_t e;
  if (kron && kron3c_use(m->n, m->NL))
    e = launch_kron3c(m->NL, KMODE_APPLY, m->kp, g, u, y, ch, s);
  else if (kron && kron6_use(m->n, m->NL, KMODE_APPLY))
    e = launch_kron6(m->n, KMODE_APPLY, m->kp, g, u, y, ch, s);
  else if (kron && kron_v4(m->n))
    e = launch_kron4(m->n, m->NL, KMODE_APPLY, m->kp, g, u, y, ch, s);
  else if (quad_v3(m->n, m->geom))
    e = launch_quad3(m->n, m->NL, m->geom, KMODE_APPLY, m->qp, m->ga, g, u, y, ch, s);
  else
    e = launch_quad(m->n, m->NL, m->geom, KMODE_APPLY, m->qp, m->ga, g, u, y, ch, s);
  return post_launch(m, e, "apply", s);
}

}  // namespace

extern "C" {

dg_status dg_apply_laplace_host(dg_mesh m, const double* u_host, double* y_host, void* stream) {
  if (!m || !u_host || !y_host) return fail(DG_ERR_PARAM, "NULL argument");
  if (u_host == y_host) return fail(DG_ERR_PARAM, "u and y alias");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nd = m->ndofs_local;
  const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(nd, 1);
  if (!m->d_hu) {
    CUDA_TRY(cudaMalloc(&m->d_hu, bytes));
    CUDA_TRY(cudaMalloc(&m->d_hy, bytes));
    CUDA_TRY(cudaStreamCreateWithFlags(&m->h2d_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&m->d2h_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&m->ev_done, cudaEventDisableTiming));
  }
  const bool kron = m->cartesian;
  const bool zwrap = m->zlo == ZSRC_LOCAL || m->zhi == ZSRC_LOCAL;   // periodic single slab
  const bool halo = m->zlo == ZSRC_HALO || m->zhi == ZSRC_HALO;
  if (zwrap || halo || m->nz < 4) {   // whole-vector path (the exchange needs all planes first)
    CUDA_TRY(cudaMemcpyAsync(m->d_hu, u_host, sizeof(double) * nd, cudaMemcpyHostToDevice, s));
    ChebyArgs ch{};
    dg_status st = run_pass(m, KMODE_APPLY, kron, m->d_hu, m->d_hy, ch, false, s);
    if (st != DG_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(y_host, m->d_hy, sizeof(double) * nd, cudaMemcpyDeviceToHost, s));
    return DG_OK;
  }
  const int64_t plane = (int64_t)m->N[0] * m->N[1] * m->n * m->n * m->n;
  // z-plane chunks: the first chunk's copy-in and the last chunk's copy-out are not overlapped,
  // so more chunks hide more of the PCIe time (DG_HOST_CHUNKS overrides the cap)
  const char* hc = std::getenv("DG_HOST_CHUNKS");
  // default: up to 32 chunks of at least 4 MB (small meshes lose more to per-chunk overhead)
  const int cap = hc ? std::max(1, std::atoi(hc))
                     : (int)std::min<int64_t>(32, std::max<int64_t>(1, nd * 8 / (4 << 20)));
  const int nchunk = std::max(1, std::min(cap, m->nz / 2));
  while ((int)m->ev_h2d.size() < nchunk) {
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    m->ev_h2d.push_back(a);
    m->ev_comp.push_back(b);
  }
  auto zb = [&](int c) { return (int)((int64_t)m->nz * c / nchunk); };
  // everything before this call on `stream` happens first
  CUDA_TRY(cudaEventRecord(m->ev_done, s));
  CUDA_TRY(cudaStreamWaitEvent(m->h2d_stream, m->ev_done, 0));
  CUDA_TRY(cudaStreamWaitEvent(m->d2h_stream, m->ev_done, 0));
  for (int c = 0; c < nchunk; ++c) {
    const int64_t o = zb(c) * plane, cnt = (int64_t)(zb(c + 1) - zb(c)) * plane;
    CUDA_TRY(cudaMemcpyAsync(m->d_hu + o, u_host + o, sizeof(double) * cnt, cudaMemcpyHostToDevice,
                             m->h2d_stream));
    CUDA_TRY(cudaEventRecord(m->ev_h2d[c], m->h2d_stream));
  }
  for (int c = 0; c < nchunk; ++c) {
    // planes [zb(c), zb(c+1)) need the first plane of the next chunk
    CUDA_TRY(cudaStreamWaitEvent(s, m->ev_h2d[std::min(c + 1, nchunk - 1)], 0));
    dg_status st = launch_apply_range(m, kron, m->d_hu, m->d_hy, zb(c), zb(c + 1), s);
    if (st != DG_OK) return st;
    CUDA_TRY(cudaEventRecord(m->ev_comp[c], s));
    CUDA_TRY(cudaStreamWaitEvent(m->d2h_stream, m->ev_comp[c], 0));
    const int64_t o = zb(c) * plane, cnt = (int64_t)(zb(c + 1) - zb(c)) * plane;
    CUDA_TRY(cudaMemcpyAsync(y_host + o, m->d_hy + o, sizeof(double) * cnt, cudaMemcpyDeviceToHost,
                             m->d2h_stream));
  }
  CUDA_TRY(cudaEventRecord(m->ev_done, m->d2h_stream));
  CUDA_TRY(cudaStreamWaitEvent(s, m->ev_done, 0));
  return DG_OK;
}

}  // extern "C"
