// k3_tables.cuh -- compile-time slice index maps for K = 3 (convention P1).
// Slice (b, r) reads base tap t at gather offset (di, dj): Y_{b,r}(p) += Z_t(p + (di, dj)).
// Built exactly like rco_slice_tap_map (oracle) / slice_tap_offsets (capi.cu):
// rot90^r of the tap-id plane (tensor.hpp:348-360), reversed for the scatter convention
// (scatter_conv.hpp:72-79, 189-193).
#pragma once

namespace rc {

struct K3Tables {
  int di[4][9];
  int dj[4][9];
};

__host__ __device__ constexpr K3Tables make_k3(int conv) {
  K3Tables T{};
  for (int r = 0; r < 4; ++r) {
    int cur[9] = {0, 1, 2, 3, 4, 5, 6, 7, 8};
    for (int q = 0; q < r; ++q) {
      int nxt[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) nxt[i * 3 + j] = cur[j * 3 + (2 - i)];
      for (int t = 0; t < 9; ++t) cur[t] = nxt[t];
    }
    for (int pos = 0; pos < 9; ++pos) {
      const int t = conv == 0 ? cur[8 - pos] : cur[pos];
      T.di[r][t] = pos / 3 - 1;
      T.dj[r][t] = pos % 3 - 1;
    }
  }
  return T;
}

}  // namespace rc
