// Geometry setup for the per-quadrature-point path:
//   cells: G_q = w_q det J_q J_q^-1 J_q^-T (6 words per q-point) and V_K = sum_q w_q det J_q
//   faces: per face point dA J^-1 n_+ (3 words) and sigma_F dA, with
//          n_+ = J^-T e_d / |J^-T e_d|, dA = det J |J^-T e_d| w_a w_b,
//          sigma_F = (p+1)^2 pf (A_F/V_K- + A_F/V_K+)/2 (boundary: A_F/V_K of the cell)
// The map is analytic (SURVEY.md §8(c) item 3 / reading 6):
//   x_i = sum_m L_im X_m + amp sin(2 pi Xh_j) sin(2 pi Xh_k),  Xh_m = (c_m + xi_m)/N_m.
#include <cuda_runtime.h>

#include "dg_internal.h"

namespace dgb {
namespace {

__device__ void map_jacobian(const MapParams& mp, int cx, int cy, int cz, double x0, double x1,
                             double x2, double* J) {
  const int c[3] = {cx, cy, cz};
  const double xi[3] = {x0, x1, x2};
  double Xh[3], sn[3], cs[3];
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    Xh[m] = ((double)c[m] + xi[m]) / (double)mp.Nglob[m];
    sincospi(2.0 * Xh[m], &sn[m], &cs[m]);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int m = 0; m < 3; ++m) J[i * 3 + m] = mp.L[i * 3 + m] * mp.h[m];
  if (mp.amp != 0.0) {
    const double tp = 6.283185307179586476925286766559;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int j = (i + 1) % 3, k = (i + 2) % 3;
      J[i * 3 + j] += mp.amp * tp / mp.Nglob[j] * cs[j] * sn[k];
      J[i * 3 + k] += mp.amp * tp / mp.Nglob[k] * sn[j] * cs[k];
    }
  }
}

__device__ double inv3(const double* J, double* Ji) {
  const double a = J[0], b = J[1], c = J[2], d = J[3], e = J[4], f = J[5], g = J[6], h = J[7], i = J[8];
  const double A = e * i - f * h, B = -(d * i - f * g), C = d * h - e * g;
  const double det = a * A + b * B + c * C;
  const double id = 1.0 / det;
  Ji[0] = A * id;
  Ji[3] = B * id;
  Ji[6] = C * id;
  Ji[1] = -(b * i - c * h) * id;
  Ji[4] = (a * i - c * g) * id;
  Ji[7] = -(a * h - b * g) * id;
  Ji[2] = (b * f - c * e) * id;
  Ji[5] = -(a * f - c * d) * id;
  Ji[8] = (a * e - b * d) * id;
  return det;
}

// global cell coordinate along z of local plane zl, wrapped if periodic; -1 if outside
__device__ int wrap_z(const MapParams& mp, int zl) {
  int z = mp.z0 + zl;
  if (z < 0 || z >= mp.Nglob[2]) {
    if (mp.bc[2] != DG_BC_PERIODIC) return -1;
    z = (z + mp.Nglob[2]) % mp.Nglob[2];
  }
  return z;
}

template <int N>
__global__ void k_volumes(const MapParams mp, int Nx, int Ny, int nz, double* V) {
  // planes -1 .. nz (ghosts included)
  const int64_t total = (int64_t)Nx * Ny * (nz + 2);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int cx = (int)(t % Nx), cy = (int)((t / Nx) % Ny), zl = (int)(t / ((int64_t)Nx * Ny)) - 1;
    const int cz = wrap_z(mp, zl);
    double v = 1.0;
    if (cz >= 0) {
      v = 0.0;
      for (int q = 0; q < N * N * N; ++q) {
        double J[9], Ji[9];
        map_jacobian(mp, cx, cy, cz, mp.xq[q % N], mp.xq[(q / N) % N], mp.xq[q / (N * N)], J);
        v += mp.wq[q % N] * mp.wq[(q / N) % N] * mp.wq[q / (N * N)] * inv3(J, Ji);
      }
    }
    V[t] = v;
  }
}

template <int N>
__global__ void k_geom_cells(const MapParams mp, int Nx, int Ny, int nz, double* G, int* err) {
  constexpr int N3 = N * N * N;
  const int64_t total = (int64_t)Nx * Ny * nz * N3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = t / N3;
    const int q = (int)(t % N3);
    const int cx = (int)(cell % Nx), cy = (int)((cell / Nx) % Ny), zl = (int)(cell / ((int64_t)Nx * Ny));
    const int q0 = q % N, q1 = (q / N) % N, q2 = q / (N * N);
    double J[9], Ji[9];
    map_jacobian(mp, cx, cy, mp.z0 + zl, mp.xq[q0], mp.xq[q1], mp.xq[q2], J);
    const double det = inv3(J, Ji);
    if (!(det > 0.0) || !isfinite(det)) atomicOr(err, 1);
    const double w = mp.wq[q0] * mp.wq[q1] * mp.wq[q2] * det;
    double* g = G + cell * (6 * N3) + gq<N>(q0, q1, q2);
    // (a,b) = sum_k Ji[a][k] Ji[b][k]
    g[0 * N3] = w * (Ji[0] * Ji[0] + Ji[1] * Ji[1] + Ji[2] * Ji[2]);
    g[1 * N3] = w * (Ji[3] * Ji[3] + Ji[4] * Ji[4] + Ji[5] * Ji[5]);
    g[2 * N3] = w * (Ji[6] * Ji[6] + Ji[7] * Ji[7] + Ji[8] * Ji[8]);
    g[3 * N3] = w * (Ji[0] * Ji[3] + Ji[1] * Ji[4] + Ji[2] * Ji[5]);
    g[4 * N3] = w * (Ji[0] * Ji[6] + Ji[1] * Ji[7] + Ji[2] * Ji[8]);
    g[5 * N3] = w * (Ji[3] * Ji[6] + Ji[4] * Ji[7] + Ji[5] * Ji[8]);
  }
}

template <int N>
__global__ void k_geom_faces(const MapParams mp, int d, int Nx, int Ny, int nz, const double* V,
                             const double* __restrict__ usig, double* F, int* err) {
  constexpr int NN = N * N;
  const int nfx = d == 0 ? Nx + 1 : Nx, nfy = d == 1 ? Ny + 1 : Ny, nfz = d == 2 ? nz + 1 : nz;
  const int64_t total = (int64_t)nfx * nfy * nfz;
  const int Nd = mp.Nglob[d];
  const int64_t plane = (int64_t)Nx * Ny;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int fx = (int)(t % nfx), fy = (int)((t / nfx) % nfy), fz = (int)(t / ((int64_t)nfx * nfy));
    // lower cell coords (c - e_d) and upper cell coords
    const int pl = d == 0 ? fx : (d == 1 ? fy : fz);                  // face plane (local)
    const int gpl = d == 2 ? mp.z0 + pl : pl;                         // global plane
    const bool periodic = mp.bc[d] == DG_BC_PERIODIC;
    const bool has_lo = gpl >= 1 || periodic;
    const bool has_hi = gpl <= Nd - 1 || periodic;
    // volumes of the adjacent cells (V has ghost planes -1..nz for z; x/y wrap)
    auto vol = [&](int ox) -> double {   // ox = -1 (lower) or 0 (upper), offset along d
      int cx = fx, cy = fy, zl = fz;
      if (d == 0) cx = ((fx + ox) % Nx + Nx) % Nx;
      if (d == 1) cy = ((fy + ox) % Ny + Ny) % Ny;
      if (d == 2) zl = fz + ox;
      return V[(int64_t)(zl + 1) * plane + (int64_t)cy * Nx + cx];
    };
    // evaluation cell: upper if it exists (xi_d = 0), else lower (xi_d = 1), global coords
    int ec[3] = {fx, fy, mp.z0 + fz};
    double exi = 0.0;
    if (!has_hi || gpl == Nd) {
      ec[d] = (d == 2 ? gpl : pl) - 1;
      exi = 1.0;
    } else {
      ec[d] = d == 2 ? gpl : pl;
    }
    if (ec[d] >= Nd) ec[d] -= Nd;
    if (ec[d] < 0) ec[d] += Nd;
    const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
    double AF = 0.0;
    double* out = F + t * (4 * NN);
    for (int p = 0; p < NN; ++p) {
      const int qa = p % N, qb = p / N;
      double xi[3];
      xi[d] = exi;
      xi[t1] = mp.xq[qa];
      xi[t2] = mp.xq[qb];
      double J[9], Ji[9];
      map_jacobian(mp, ec[0], ec[1], ec[2], xi[0], xi[1], xi[2], J);
      const double det = inv3(J, Ji);
      if (!(det > 0.0) || !isfinite(det)) atomicOr(err, 1);
      const double r0 = Ji[d * 3], r1 = Ji[d * 3 + 1], r2 = Ji[d * 3 + 2];
      const double nr = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
      const double dA = det * nr * mp.wq[qa] * mp.wq[qb];
      // dA J^-1 n_+ = det * w * J^-1 r
      const double f = det * mp.wq[qa] * mp.wq[qb];
      out[0 * NN + p] = f * (Ji[0] * r0 + Ji[1] * r1 + Ji[2] * r2);
      out[1 * NN + p] = f * (Ji[3] * r0 + Ji[4] * r1 + Ji[5] * r2);
      out[2 * NN + p] = f * (Ji[6] * r0 + Ji[7] * r1 + Ji[8] * r2);
      out[3 * NN + p] = dA;
      AF += dA;
    }
    double sig;
    if (has_lo && has_hi)
      sig = mp.pen * 0.5 * (AF / vol(-1) + AF / vol(0));
    else if (has_hi)
      sig = mp.pen * AF / vol(0);
    else
      sig = mp.pen * AF / vol(-1);
    if (usig) sig = usig[t];   // the caller's sigma_F (dg.h user_penalty), same face layout
    for (int p = 0; p < NN; ++p) out[3 * NN + p] *= sig;
  }
}

template <int N>
cudaError_t run(const MapParams& mp, int Nx, int Ny, int nz, double* G, double* face[3],
                const double* const usig[3], int* err, cudaStream_t s) {
  double* V = nullptr;
  cudaError_t e = cudaMallocAsync(&V, sizeof(double) * (size_t)Nx * Ny * (nz + 2), s);
  if (e != cudaSuccess) return e;
  const int grid = 148 * 8, bs = 256;
  k_volumes<N><<<grid, bs, 0, s>>>(mp, Nx, Ny, nz, V);
  k_geom_cells<N><<<grid, bs, 0, s>>>(mp, Nx, Ny, nz, G, err);
  for (int d = 0; d < 3; ++d) k_geom_faces<N><<<grid, bs, 0, s>>>(mp, d, Nx, Ny, nz, V, usig[d], face[d], err);
  e = cudaGetLastError();
  cudaFreeAsync(V, s);
  return e;
}

}  // namespace

cudaError_t launch_geom_qpoint(int n, const MapParams& mp, int Nx, int Ny, int nz, double* G,
                               double* face[3], const double* const usig[3], int* err_flag, cudaStream_t s) {
  switch (n) {
    case 2: return run<2>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
    case 3: return run<3>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
    case 4: return run<4>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
    case 5: return run<5>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
    case 6: return run<6>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
    case 7: return run<7>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
    case 8: return run<8>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
    case 9: return run<9>(mp, Nx, Ny, nz, G, face, usig, err_flag, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dgb
