// Halo packing index shared by the device pack kernel (k_halo.cu) and the host
// reference packer (dg_halo_pack_host): element e of a send plane
// [cxy][l][j][i] comes from u at the returned offset (bottom plane: layers [0,NL);
// top plane: layers [n-NL, n)).
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define DGB_HD __host__ __device__ __forceinline__
#else
#define DGB_HD inline
#endif

namespace dgb {

DGB_HD int64_t halo_src(int64_t e, int n, int NL, int64_t plane_cells, int nz, bool top) {
  const int n2 = n * n;
  const int64_t per = (int64_t)NL * n2;
  const int64_t cxy = e / per;
  const int r = (int)(e % per);
  const int l = r / n2, ji = r % n2;
  const int64_t cell = top ? (int64_t)(nz - 1) * plane_cells + cxy : cxy;
  const int layer = top ? n - NL + l : l;
  return cell * (int64_t)(n2 * n) + (int64_t)layer * n2 + ji;
}

}  // namespace dgb
