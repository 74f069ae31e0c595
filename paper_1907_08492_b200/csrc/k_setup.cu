// Setup kernels (run once per mesh).
//
// k_cart_diag: point-Jacobi diagonal of the Cartesian operator
// in either working basis.  With Eq. (14) the diagonal is
//   d[i,j,k] = s_x Lx_ii M_jj M_kk + s_y M_ii Ly_jj M_kk + s_z M_ii M_jj Lz_kk
// where L_d's 1D diagonal depends on whether the cell touches a mirror boundary in
// direction d (the ghost coupling adds -N(i, n-1-i)); the host precomputes the four
// 1D variants [interior, left boundary, right boundary, both].
#include <cuda_runtime.h>

#include "dg_internal.h"

namespace dgb {
namespace {

template <int N>
__global__ void k_cart_diag(const __grid_constant__ CartDiagParams p, int Nx, int Ny, int nz,
                            int z0, int Nz_global, double* __restrict__ out) {
  const int64_t total = (int64_t)Nx * Ny * nz * N * N * N;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / (N * N * N);
    const int r = (int)(g % (N * N * N));
    const int i = r % N, j = (r / N) % N, k = r / (N * N);
    const int cx = (int)(cell % Nx), cy = (int)((cell / Nx) % Ny), cz = (int)(cell / ((int64_t)Nx * Ny)) + z0;
    auto variant = [](int c, int n) { return (c == 0 ? 1 : 0) + (c == n - 1 ? 2 : 0); };
    const int vx = variant(cx, Nx), vy = variant(cy, Ny), vz = variant(cz, Nz_global);
    const double d = p.scale[0] * p.ldiag[0][vx][i] * p.mdiag[j] * p.mdiag[k] +
                     p.scale[1] * p.mdiag[i] * p.ldiag[1][vy][j] * p.mdiag[k] +
                     p.scale[2] * p.mdiag[i] * p.mdiag[j] * p.ldiag[2][vz][k];
    out[g] = p.invert ? 1.0 / d : d;
  }
}

}  // namespace

cudaError_t launch_cart_diag(int n, const CartDiagParams& p, int Nx, int Ny, int nz, int z0,
                             int Nz_global, double* out, cudaStream_t s) {
  const int bs = 256, grid = 148 * 8;
  switch (n) {
#define CASE(NN) \
  case NN: k_cart_diag<NN><<<grid, bs, 0, s>>>(p, Nx, Ny, nz, z0, Nz_global, out); break;
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace dgb
