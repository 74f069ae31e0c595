/*
 * dg.h — C ABI of the B200 (sm_100a) fp64 matrix-free SIPG library for the
 * Hermite-like basis of arXiv 1907.08492 (Kronbichler, Kormann, Wall 2019).
 *
 * Operation defined by the paper (citations are PAPER.md line numbers):
 *   y = A u, A the symmetric interior penalty (SIPG) discretisation of -Laplace
 *   on hexahedra, Eq. (1), in the tensor-product basis of
 *   Eq. (2) built from the Hermite-like 1D polynomials of
 *   Sec. 4.1, integrated with (p+1)^3 Gauss points in the
 *   cell and (p+1)^2 per face, mirror-principle Dirichlet
 *   boundaries u+ = -u- (PAPER.md:172-174), penalty (p+1)^2 * A_F / V_K
 *   (BASELINE.json configs), element-wise face arrangement
 *   (PAPER.md:323-330).  Readings of silent/ambiguous points: DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Vectors are caller-owned DEVICE pointers to fp64, n_local_dofs long, in
 *     cell-wise layout: DoF (i,j,k) of cell (cx,cy,cz) at
 *         ((cz_local*Ny + cy)*Nx + cx) * n^3 + (k*n + j)*n + i,   n = degree+1,
 *     x fastest inside a cell and across cells, z slowest (a z-slab of a rank
 *     is one contiguous range).
 *   - Every vector pointer passed to a call must be 16-byte aligned (the kernels
 *     move even-n lines with 128-bit accesses); a misaligned pointer returns
 *     DG_ERR_PARAM before any launch.  cudaMalloc / torch allocations are; a
 *     view at an odd element offset is not.
 *   - Calls are stream-ordered and asynchronous on the given cudaStream_t
 *     (passed as void*; NULL = legacy default stream).  Asynchronous CUDA/NCCL
 *     faults surface on a later call, or immediately with DG_DEBUG_SYNC=1.
 *   - A handle owns: the 1D tables, geometry, penalties, the GL inverse
 *     diagonal, the halo buffers, the NCCL communicator, internal events.  A
 *     handle must not be used from two streams concurrently (halo buffers are
 *     shared).
 *   - Every function returns a dg_status; on a non-OK status dg_last_error()
 *     returns a thread-local message.  No function aborts the process.
 */
#ifndef DG_B200_H
#define DG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DG_OK = 0,
  DG_ERR_PARAM = 1,        /* bad degree/size/flag, NULL or aliased pointer, lo>=hi, ... */
  DG_ERR_NUMERIC = 2,      /* det J <= 0, non-finite geometry, non-positive diagonal      */
  DG_ERR_CUDA = 3,         /* CUDA runtime error (message has the CUDA error string)     */
  DG_ERR_NCCL = 4,         /* NCCL error                                                  */
  DG_ERR_UNSUPPORTED = 5   /* combination not implemented (message says which)            */
} dg_status;

enum { DG_BASIS_HERMITE_LIKE = 0, DG_BASIS_NODAL_GL = 1 };
enum { DG_GEOM_CONSTANT = 0, DG_GEOM_PER_CELL = 1, DG_GEOM_PER_QPOINT = 2 };
enum { DG_BC_DIRICHLET_MIRROR = 0, DG_BC_PERIODIC = 1 };

/* dg_apply_laplace flags (bitwise or) */
enum {
  DG_APPLY_DEFAULT = 0,          /* exchange halo (if nranks>1) and overlap inside          */
  DG_APPLY_HALO_READY = 1,       /* caller already ran dg_halo_exchange(m, u, stream)       */
  DG_APPLY_QUADRATURE = 2        /* force the general quadrature kernel (paper formulation)
                                    even where the Cartesian Kronecker kernel applies      */
};

/* dg_basis_change ops: v = B (x) B (x) B u per cell */
enum {
  DG_BCHG_H_TO_GL = 0,     /* B = T,      T[i][j] = phi_j^H(x_i^GL)  (values at GL nodes) */
  DG_BCHG_GL_TO_H = 1,     /* B = T^{-1}                                                  */
  DG_BCHG_H_TO_GL_T = 2,   /* B = T^T                                                     */
  DG_BCHG_GL_TO_H_T = 3    /* B = T^{-T}                                                  */
};

/* dg_chebyshev_smooth inner preconditioners */
enum {
  DG_INNER_GL_JACOBI = 0,    /* P^{-1} = (T^{-1})^{x3} diag(A_GL)^{-1} (T^{-T})^{x3}, Eq. (12) */
  DG_INNER_POINT_JACOBI = 1, /* P^{-1} = diag(A)^{-1} in the working basis    */
  DG_INNER_FDM = 2           /* fast-diagonalisation block Jacobi, Eqs. (13)-(15)
                                (PAPER.md:2117-2165): P^{-1} = Z^{x3} (Lam (+) Lam (+) Lam)^{-1}
                                (Z^T)^{x3} with L_DG Z = M Z Lam, Z^T M Z = I of the interior
                                1D element, used on every cell.  Cartesian meshes only
                                (DG_ERR_UNSUPPORTED otherwise); no diagonal vector. */
};

typedef struct dg_mesh_s* dg_mesh;   /* opaque, library-owned, freed by dg_mesh_destroy */

typedef struct {
  int32_t degree;          /* p, 1..8                                                      */
  int32_t basis;           /* DG_BASIS_*                                                   */
  int32_t n_cells[3];      /* GLOBAL Nx, Ny, Nz (>= 1)                                     */
  double  box_lo[3];       /* undeformed box [lo, hi], hi > lo                             */
  double  box_hi[3];
  double  linear_map[9];   /* row-major L of x = L X; all-zero = identity */
  double  deform_amp;      /* x_i += amp sin(2 pi Xh_j) sin(2 pi Xh_k), (i,j,k) cyclic,
                              Xh the unit-box coordinate; 0 = affine                       */
  int32_t geometry;        /* DG_GEOM_*; CONSTANT/PER_CELL require deform_amp == 0          */
  int32_t bc[3];           /* DG_BC_* per direction                                         */
  double  penalty_factor;  /* multiplies (p+1)^2 A_F/V_K; <= 0 means 1.0 (paper value)       */
  const double* user_inv_jac; /* optional HOST array, PER_CELL only: exactly 9 doubles per OWNED
                              cell (9 * Nx * Ny * nz_local; the library reads that many and
                              cannot check the length), row-major J^{-1}, cell order as the
                              DoF layout; NULL = derive                                    */
  const double* user_penalty; /* optional HOST array of sigma_F, 6 doubles per OWNED cell in face
                              order 2d+s (face xi_d = s of the cell), cell order as the DoF
                              layout; the value is sigma_F itself (penalty_factor is not
                              applied).  The two cells of every face inside the slab (also
                              across a periodic wrap) must carry bit-equal values, else
                              DG_ERR_PARAM; non-finite or negative values -> DG_ERR_PARAM.
                              NULL = (p+1)^2 pf mean(A_F/V_K).  A mesh with
                              user penalties runs the general quadrature kernels (geometry
                              stored per quadrature point, or per cell for PER_CELL), never
                              the Cartesian Kronecker, FDM or fp32 paths, whose 1D blocks
                              assume one penalty per direction.                            */
  int32_t rank, nranks;    /* z-slab decomposition: rank r owns planes
                              [r*Nz/nranks, (r+1)*Nz/nranks)                                */
  const void* nccl_unique_id; /* 128 bytes from dg_get_nccl_unique_id on rank 0, broadcast
                                 by the caller; NULL when nranks == 1, or NULL with
                                 nranks > 1 for an external halo transport
                                 (dg_halo_pack / dg_halo_set)                               */
  void*   stream;          /* cudaStream_t for setup work (NULL = default)                 */
} dg_mesh_desc;

/* Message for the last non-OK status of the calling thread (never NULL). */
const char* dg_last_error(void);

/* Version / build string, e.g. "dg_b200 0.1 sm_100a". */
const char* dg_version(void);

/* NCCL unique id (128 bytes) into out128 (host memory).  Call on rank 0 only. */
dg_status dg_get_nccl_unique_id(void* out128);

/* Build the mesh handle: 1D tables (extended precision on the host), geometry and
 * penalties, the GL inverse diagonal (Eq. (12)),
 * halo buffers and (nranks > 1) the NCCL communicator.  Synchronises `stream`. */
dg_status dg_mesh_setup(const dg_mesh_desc* desc, dg_mesh* out);

dg_status dg_mesh_destroy(dg_mesh m);

/* Sizes of the local slab: owned DoFs, global DoFs, owned planes [z_begin, z_end). */
dg_status dg_mesh_query(dg_mesh m, int64_t* n_local_dofs, int64_t* n_global_dofs,
                        int32_t* z_begin, int32_t* z_end);

/* Host-only slab plan for z-slab decomposition (no GPU needed):
 * out[0] = z_begin, out[1] = z_end (owned planes [z_begin, z_end) = [r*Nz/P, (r+1)*Nz/P)),
 * out[2] = lower peer rank (-1: mirror boundary, rank itself never), out[3] = upper peer,
 * out[4] = NL (layers per halo plane: 2 Hermite-like (p>=2), n otherwise).
 * Message order of one exchange (both directions, grouped): first "up"  (send the top
 * NL layers of the top plane to the upper peer, receive the lower peer's into recv_lo),
 * then "down" (send the bottom NL layers of the bottom plane to the lower peer, receive
 * the upper peer's into recv_hi).  Halo layout: [cx + Nx*cy][l][j][i]. */
dg_status dg_slab_plan(int32_t Nz, int32_t nranks, int32_t rank, int32_t bc_z, int32_t degree,
                       int32_t basis, int32_t* out6);

/* Halo buffers with an external transport (NCCL-free; e.g. one-GPU loopback tests):
 * dg_halo_pack writes the two send planes of u (device, count doubles each, count from
 * dg_mesh_query_halo); dg_halo_set installs received planes (device) as the halo.
 * Meshes built with nranks > 1 and nccl_unique_id == NULL use this external mode. */
/* Host-only reference packer (no GPU): the two send planes of a host slab u_slab
 * (nz local planes of Nx*Ny cells), same index map as the device pack kernel. */
dg_status dg_halo_pack_host(const double* u_slab, int32_t degree, int32_t basis, int32_t Nx,
                            int32_t Ny, int32_t nz, double* send_lo, double* send_hi);
dg_status dg_mesh_query_halo(dg_mesh m, int64_t* count, int32_t* lo_peer, int32_t* hi_peer);
dg_status dg_halo_pack(dg_mesh m, const double* u, double* send_lo, double* send_hi, void* stream);
dg_status dg_halo_set(dg_mesh m, const double* recv_lo, const double* recv_hi, void* stream);

/* Caller-provided transport for a mesh built with nranks > 1 and nccl_unique_id == NULL
 * (external mode), so that the calls which need an exchange inside them -- the fused
 * Chebyshev sweep (one halo per step), dg_dot, dg_lanczos_lambda_max, dg_pcg and
 * dg_apply_laplace without DG_APPLY_HALO_READY -- run over any transport (MPI, a Python
 * process group, or the one-GPU loopback of the tests).
 *   halo:  called after the library packed the send planes of the current operand on
 *          `stream` (device buffers, `count` doubles each; send_lo / recv_lo are NULL when
 *          there is no lower peer, likewise for hi).  It must leave recv_lo / recv_hi (the
 *          library-owned halo) holding the peers' planes when work enqueued on `stream`
 *          after the return runs (synchronous copies, or copies ordered on `stream`).
 *          Message order as dg_slab_plan: the lower peer's top planes go to recv_lo, the
 *          upper peer's bottom planes to recv_hi.
 *   allreduce_sum: replace *value (host) by its sum over all ranks.
 * Both return 0 on success; non-zero becomes DG_ERR_NCCL ("transport failed").
 * Passing NULL removes the transport.  The callbacks run on the calling thread. */
typedef struct {
  int (*halo)(void* user, const double* send_lo, const double* send_hi, double* recv_lo,
              double* recv_hi, int64_t count, void* stream);
  int (*allreduce_sum)(void* user, double* value);
  void* user;
} dg_transport;
dg_status dg_set_transport(dg_mesh m, const dg_transport* t);

/* Fill the library-owned z-halo of u: the two Hermite face layers (all n layers for
 * the GL basis) of the neighbouring ranks' boundary planes, via grouped ncclSend/
 * ncclRecv.  No-op when nranks == 1 and no periodic wrap in z. */
dg_status dg_halo_exchange(dg_mesh m, const double* u, void* stream);

/* y = A u on the owned cells.  u and y must not alias (DG_ERR_PARAM). */
dg_status dg_apply_laplace(dg_mesh m, const double* u, double* y, int32_t flags, void* stream);

/* out = B^{x3} in per cell (see DG_BCHG_*); in == out is allowed. */
dg_status dg_basis_change(dg_mesh m, int32_t op, const double* in, double* out, void* stream);

/* y_host = A u_host with HOST vectors (n_local_dofs each): the host->device copy, the matvec
 * and the device->host copy run in z-plane chunks (up to 32 of >= 4 MB, at most nz/2; env
 * DG_HOST_CHUNKS sets the cap)
 * overlapped on internal copy streams (the chunk being computed needs the first plane of the
 * next one).  Stream-ordered on `stream`:
 * y_host is complete when `stream` reaches the end of the call.  Pinned host memory is needed
 * for the overlap (pageable memory works, copied synchronously by the driver).  Periodic z,
 * several slabs or fewer than 4 planes use one whole-vector copy each way.  The library keeps
 * two device vectors of staging per mesh after the first call. */
dg_status dg_apply_laplace_host(dg_mesh m, const double* u_host, double* y_host, void* stream);

/* Chebyshev iteration of Eq. (11), `degree` operator
 * applications, range [lo_frac, hi_frac] * lambda_max (paper: 0.06, 1.2).
 * b: right-hand side; x: in x_0, out x_degree; work2: 2 * n_local_dofs doubles
 * of caller scratch.  Each step is one fused kernel: matvec + residual + P^{-1}
 * + three-term update ("merged" variant). */
dg_status dg_chebyshev_smooth(dg_mesh m, const double* b, double* x, double* work2,
                              int32_t degree, double lambda_max, double lo_frac,
                              double hi_frac, int32_t inner, void* stream);

/* ---------------------------------------------------------------- solver layer
 * (PAPER.md:1811-1832).  All vectors are device, n_local_dofs
 * long; dot products are global over the z-slabs (ncclAllReduce when nranks > 1, the
 * dg_transport's allreduce_sum in external mode, DG_ERR_UNSUPPORTED in external mode
 * without a transport).  These calls synchronise `stream`. */

/* z = P^{-1} r, the inner preconditioner of dg_chebyshev_smooth (DG_INNER_*). */
dg_status dg_apply_preconditioner(dg_mesh m, int32_t inner, const double* r, double* z, void* stream);

/* *out (host) = a . b over all ranks (deterministic two-level reduction). */
dg_status dg_dot(dg_mesh m, const double* a, const double* b, double* out, void* stream);

/* lambda_max(P^{-1} A) from `iters` (1..200) Lanczos steps started from the vector
 * [-5.5, -4.5, ..., 5.5] repeated over the global DoF index (the
 * paper uses 15).  Largest eigenvalue of the Lanczos tridiagonal. */
dg_status dg_lanczos_lambda_max(dg_mesh m, int32_t inner, int32_t iters, double* lambda_max, void* stream);

/* Conjugate gradients preconditioned by one degree-`cheby_degree` Chebyshev sweep from a
 * zero initial guess (range [lo_frac, hi_frac] * lambda_max, inner preconditioner `inner`):
 * a fixed symmetric polynomial preconditioner.  x: in initial guess, out iterate.  Stops
 * when ||r_k|| <= rel_tol ||r_0|| or after max_iter iterations; *iters and *rel_res
 * (host, may be NULL) report the outcome.  DG_ERR_NUMERIC on breakdown (p.Ap <= 0). */
dg_status dg_pcg(dg_mesh m, const double* b, double* x, double rel_tol, int32_t max_iter,
                 int32_t cheby_degree, double lambda_max, double lo_frac, double hi_frac, int32_t inner,
                 int32_t* iters, double* rel_res, void* stream);

/* ---------------------------------------------------------------- fp32 path
 * (the paper's smoothers run in fp32).
 * Same operator and smoother as the fp64 calls with float vectors: the 1D tables are
 * rounded to float once, every contraction and the update run in fp32.  Cartesian meshes
 * (degree 2..8, k_kron4 path) on a single z-slab only; DG_ERR_UNSUPPORTED otherwise. */
dg_status dg_apply_laplace_f32(dg_mesh m, const float* u, float* y, void* stream);
dg_status dg_chebyshev_smooth_f32(dg_mesh m, const float* b, float* x, float* work2, int32_t degree,
                                  double lambda_max, double lo_frac, double hi_frac, int32_t inner,
                                  void* stream);

/* out = B^{x3} in per cell in single precision (B rounded to float once; in == out allowed);
 * any geometry (the basis change is cell-local and geometry-free). */
dg_status dg_basis_change_f32(dg_mesh m, int32_t op, const float* in, float* out, void* stream);

/* Mixed-precision variant of dg_pcg (fp64 CG around a single-precision
 * preconditioner): CG vectors, matvec and dot products in fp64; every preconditioner
 * application z = M r rounds r to float, runs the degree-`cheby_degree` Chebyshev sweep
 * of dg_chebyshev_smooth_f32 from zero and widens z back to double.  Cartesian single-slab
 * meshes (the fp32 kernels), else DG_ERR_UNSUPPORTED.  Arguments as dg_pcg. */
dg_status dg_pcg_mixed(dg_mesh m, const double* b, double* x, double rel_tol, int32_t max_iter,
                       int32_t cheby_degree, double lambda_max, double lo_frac, double hi_frac,
                       int32_t inner, int32_t* iters, double* rel_res, void* stream);

/* Inverse of the inner preconditioner's diagonal, copied to `out` (device,
 * n_local_dofs): diag(A_GL)^{-1} (GL_JACOBI) or diag(A)^{-1} (POINT_JACOBI). */
dg_status dg_inverse_diagonal(dg_mesh m, int32_t inner, double* out, void* stream);

/* Host-only diagnostic (no GPU needed): the 1D tables the kernels are built from,
 * for the working basis `basis` at degree p (n = p+1), packed as
 *   xq[n] wq[n] S[n*n] DS[n*n] v0[n] v1[n] d0[n] d1[n]
 *   Mhat[n*n] Ahat[n*n] Lhat[n*n] Nm[n*n] Np[n*n] T[n*n] Tinv[n*n]
 * (row-major; S[q][j] = phi_j(xq_q); T[i][j] = phi_j^H(x_i^GL)); 6n + 9n^2 doubles.
 * Lhat/Nm/Np are the 1D SIPG blocks on the unit interval with sigma = (p+1)^2 *
 * penalty_factor (Eq. (14)).  out_len < 6n + 9n^2 -> DG_ERR_PARAM. */
dg_status dg_tables_1d(int32_t degree, int32_t basis, double penalty_factor, double* out,
                       int64_t out_len);

/* Machine characterisation (roofline denominators measured on the running GPU):
 * kind 0: fp64 FMA throughput in TFLOP/s (DFMA chains, 148*8 blocks);
 * kind 1: streaming copy bandwidth in GB/s (read + write bytes, 2 GiB buffers);
 * kind 2: streaming read bandwidth in GB/s;
 * kind 3: fp64 tensor-core throughput in TFLOP/s (DMMA, mma.sync m8n8k4 f64 chains);
 * kind 4: DMMA chains and DFMA chains interleaved in one kernel, total TFLOP/s (if the two
 *         used separate pipes this would approach the sum of kinds 0 and 3);
 * kind 10 + n (n = 3..8): design probe, GDoF/s of a warp-private, cp.async-pipelined
 *         plane-per-lane proxy of the Cartesian matvec's seven sweeps without neighbour terms
 *         (csrc/k_probe_plane.cu; an upper bound for the schedule DESIGN.md §11 proposes);
 * kind 20 + n (n = 3..6): the same probe with the neighbour-layer traffic and couplings.
 * Best of 5 timed launches. */
dg_status dg_measure_peak(int32_t kind, double* value, void* stream);

/* Number of kernels this library launched since the handle was created. */
int64_t dg_kernel_launch_count(dg_mesh m);

#ifdef __cplusplus
}
#endif

#endif /* DG_B200_H */
