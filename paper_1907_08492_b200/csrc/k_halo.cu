// z-slab halo packing (ghost exchange of 2(p+1)^{d-1} values per
// face for the Hermite-like basis).  The bottom plane's layers [0, NL) go to the lower
// peer, the top plane's layers [n-NL, n) to the upper peer; layout [cxy][l][j][i].
#include <cuda_runtime.h>

#include "dg_internal.h"
#include "halo_index.h"

namespace dgb {
namespace {

__global__ void k_halo_pack(const double* __restrict__ u, double* __restrict__ send_lo,
                            double* __restrict__ send_hi, int n, int NL, int64_t plane_cells,
                            int nz) {
  const int64_t total = plane_cells * NL * n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (send_lo) send_lo[e] = u[halo_src(e, n, NL, plane_cells, nz, false)];
    if (send_hi) send_hi[e] = u[halo_src(e, n, NL, plane_cells, nz, true)];
  }
}

}  // namespace

cudaError_t launch_halo_pack(const double* u, double* send_lo, double* send_hi, int n, int NL,
                             int64_t plane_cells, int nz, cudaStream_t s) {
  const int64_t total = plane_cells * NL * n * n;
  const int bs = 256;
  int64_t grid = (total + bs - 1) / bs;
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  k_halo_pack<<<(unsigned)grid, bs, 0, s>>>(u, send_lo, send_hi, n, NL, plane_cells, nz);
  return cudaGetLastError();
}

}  // namespace dgb
