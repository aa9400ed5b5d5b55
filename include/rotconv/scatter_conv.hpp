// rotconv/scatter_conv.hpp -- drop-in for the reference's single-orientation scatter
// convolution API (/root/reference/proj/include/rotconv/scatter_conv.hpp), served by the
// sm_100a kernels of librotconv_b200.so through the C-ABI.
//
//   reference                                   here
//   MultCounter / AuxMemCounter  (:28-57)        same fields and accumulate semantics
//   TileConfig / ScatterStrategy (:59-70)        same; validated, the result is tile-invariant
//   reverse_plane / reverse_bank (:72-90)        host index permutations (unchanged)
//   detail::clipped_writes       (:94-110)       rc_clipped_writes
//   scatter_conv_raw_single      (:114-141)      rc_ri_conv_forward_host, convention raw
//   scatter_conv_single          (:143-149)      raw on reverse_plane(w)
//   scatter_conv_raw_multi       (:151-187)      rc_ri_conv_forward_host, convention raw
//   scatter_conv_multi           (:189-193)      rc_ri_conv_forward_host, convention scatter
//   tiled_scatter_conv           (:330-368)      rc_tiled_scatter_conv_host
//
// Semantics are the reference's: raw scatter with kernel W equals gather-"same" with W;
// the convenience forms pre-reverse the kernel (header comment :10-23).  Counters receive
// the reference's analytic counts (:137-139, :183-185, :361-366).  Every call is one GPU
// round trip (H2D, kernels, D2H) on rotconv::b200::device(); batched callers should use
// the batch entry points in group_conv.hpp (or the C-ABI device entry points) instead of
// looping over images.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "rotconv/device.hpp"
#include "rotconv/tensor.hpp"

namespace rotconv {

struct MultCounter {
  unsigned long long scalar_multiplications = 0;
  unsigned long long scalar_additions = 0;
  void add(unsigned long long mults, unsigned long long adds) {
    scalar_multiplications += mults;
    scalar_additions += adds;
  }
  void reset() { scalar_multiplications = scalar_additions = 0; }
};

// high-water mark of auxiliary bytes, with the reference's accounting (:351-360): the
// private tile accumulators of tile_private (tile_h * tile_w * sizeof(T) * workers)
struct AuxMemCounter {
  std::size_t current_bytes = 0;
  std::size_t peak_bytes = 0;
  void acquire(std::size_t bytes) {
    current_bytes += bytes;
    peak_bytes = std::max(peak_bytes, current_bytes);
  }
  void release(std::size_t bytes) { current_bytes = bytes > current_bytes ? 0 : current_bytes - bytes; }
  void reset() { current_bytes = peak_bytes = 0; }
};

struct TileConfig {
  int tile_h = 32;
  int tile_w = 32;
  int halo = 1;
};

enum class ScatterStrategy { tile_private, phase_parallel };

template <typename T>
MatrixRM<T> reverse_plane(const MatrixRM<T>& w) {
  return rot90_plane(w, 2);  // reversing both axes is a half turn
}

template <typename T>
FilterBank<T> reverse_bank(const FilterBank<T>& w) {
  FilterBank<T> out(w.out_channels(), w.in_channels(), w.kernel_h(), w.kernel_w());
  const int taps = w.kernel_h() * w.kernel_w();
  for (int co = 0; co < w.out_channels(); ++co)
    for (int ci = 0; ci < w.in_channels(); ++ci) {
      const T* s = w.plane(co, ci);
      std::reverse_copy(s, s + taps, out.plane(co, ci));
    }
  return out;
}

namespace detail {

inline unsigned long long clipped_writes(int h, int w, int kh, int kw) { return rc_clipped_writes(h, w, kh, kw); }

inline rc_desc single_desc(int n, int cin, int h, int w, int cout, int k, int convention) {
  rc_desc d{};
  d.n = n;
  d.c_in = cin;
  d.h = h;
  d.w = w;
  d.c_out = cout;
  d.k = k;
  d.group = RC_GROUP_SINGLE;
  d.orientations = 1;
  d.pool = RC_POOL_NONE;
  d.pool_group = 1;
  d.convention = convention;
  d.precision = static_cast<int>(b200::precision());
  return d;
}

// one image, one orientation, square kernel: the fused layer with R = 1
inline void run_single(const float* x, int cin, int h, int w, const float* wt, int cout, int k, int convention,
                       float* y) {
  const rc_desc d = single_desc(1, cin, h, w, cout, k, convention);
  b200::throw_on(rc_ri_conv_forward_host(&d, x, wt, nullptr, nullptr, y, nullptr, b200::device()));
}

}  // namespace detail

// Single plane, raw indices.  Rectangular kernels are embedded in the smallest
// square that keeps their centre (K/2 - kh/2 zero rows above); zero taps add exact zeros.
template <typename T>
MatrixRM<T> scatter_conv_raw_single(const MatrixRM<T>& x, const MatrixRM<T>& w, MultCounter* counter = nullptr) {
  ROTCONV_REQUIRE_FLOAT(T);
  const int kh = w.rows(), kw = w.cols(), K = std::max(kh, kw);
  std::vector<float> sq(static_cast<std::size_t>(K) * K, 0.f);
  const int oi = K / 2 - kh / 2, oj = K / 2 - kw / 2;
  for (int i = 0; i < kh; ++i)
    for (int j = 0; j < kw; ++j) sq[(i + oi) * K + (j + oj)] = w(i, j);
  MatrixRM<T> y(x.rows(), x.cols());
  detail::run_single(x.data(), 1, x.rows(), x.cols(), sq.data(), 1, K, RC_CONV_RAW, y.data());
  if (counter)
    counter->add(static_cast<unsigned long long>(x.rows()) * x.cols() * kh * kw,
                 detail::clipped_writes(x.rows(), x.cols(), kh, kw));
  return y;
}

template <typename T>
MatrixRM<T> scatter_conv_single(const MatrixRM<T>& x, const MatrixRM<T>& w, MultCounter* counter = nullptr) {
  return scatter_conv_raw_single(x, reverse_plane(w), counter);
}

namespace detail {
template <typename T>
Tensor3<T> multi(const Tensor3<T>& x, const FilterBank<T>& w, MultCounter* counter, int convention) {
  ROTCONV_REQUIRE_FLOAT(T);
  detail::check(x.channels() == w.in_channels(), "scatter_conv_multi: channel mismatch");
  Tensor3<T> y(w.out_channels(), x.height(), x.width());
  if (w.square()) {
    run_single(x.data(), x.channels(), x.height(), x.width(), w.data(), w.out_channels(), w.kernel_h(), convention,
               y.data());
  } else {  // embed in a square kernel (see scatter_conv_raw_single); raw indices throughout
    const FilterBank<T> src = convention == RC_CONV_SCATTER ? reverse_bank(w) : w;
    const int kh = w.kernel_h(), kw = w.kernel_w(), K = std::max(kh, kw);
    const int oi = K / 2 - kh / 2, oj = K / 2 - kw / 2;
    FilterBank<float> sq(w.out_channels(), w.in_channels(), K, K);
    for (int co = 0; co < w.out_channels(); ++co)
      for (int ci = 0; ci < w.in_channels(); ++ci)
        for (int i = 0; i < kh; ++i)
          for (int j = 0; j < kw; ++j) sq(co, ci, i + oi, j + oj) = src(co, ci, i, j);
    run_single(x.data(), x.channels(), x.height(), x.width(), sq.data(), w.out_channels(), K, RC_CONV_RAW,
               y.data());
  }
  if (counter)
    counter->add(static_cast<unsigned long long>(x.height()) * x.width() * w.kernel_h() * w.kernel_w() *
                     x.channels() * w.out_channels(),
                 clipped_writes(x.height(), x.width(), w.kernel_h(), w.kernel_w()) * w.out_channels());
  return y;
}
}  // namespace detail

template <typename T>
Tensor3<T> scatter_conv_raw_multi(const Tensor3<T>& x, const FilterBank<T>& w, MultCounter* counter = nullptr) {
  return detail::multi(x, w, counter, RC_CONV_RAW);
}

template <typename T>
Tensor3<T> scatter_conv_multi(const Tensor3<T>& x, const FilterBank<T>& w, MultCounter* counter = nullptr) {
  return detail::multi(x, w, counter, RC_CONV_SCATTER);
}

// The shipped drop-in entry point.  Validation order and messages are the reference's
// (scatter_conv.hpp:339-346, inside rc_tiled_scatter_conv_host); the GPU result does not
// depend on tile, workers or strategy, exactly like the reference (:21-23).
template <typename T>
Tensor3<T> tiled_scatter_conv(const Tensor3<T>& x, const FilterBank<T>& w, const TileConfig& cfg, int workers,
                              MultCounter* counter = nullptr, AuxMemCounter* aux = nullptr,
                              ScatterStrategy strategy = ScatterStrategy::tile_private) {
  ROTCONV_REQUIRE_FLOAT(T);
  Tensor3<T> y;
  unsigned long long mults = 0, adds = 0, aux_bytes = 0;
  // the output is allocated only after validation, so probe with a null output first
  if (x.channels() == w.in_channels() && w.square() && cfg.tile_h >= 1 && cfg.tile_w >= 1 &&
      cfg.halo == w.kernel_h() / 2 && workers >= 1)
    y = Tensor3<T>(w.out_channels(), x.height(), x.width());
  b200::throw_on(rc_tiled_scatter_conv_host(x.data(), x.channels(), x.height(), x.width(), w.data(),
                                            w.out_channels(), w.in_channels(), w.kernel_h(), w.kernel_w(),
                                            cfg.tile_h, cfg.tile_w, cfg.halo, workers,
                                            static_cast<int>(strategy), y.data(), &mults, &adds, &aux_bytes,
                                            static_cast<int>(b200::precision()), b200::device()));
  if (aux && strategy == ScatterStrategy::tile_private) {
    aux->acquire(aux_bytes);
    aux->release(aux_bytes);
  }
  if (counter) counter->add(mults, adds);
  return y;
}

}  // namespace rotconv
