// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/rotconv/*.hpp), compiled in place by oracle/Makefile
// into oracle/_ref/librc_ref.so.  TEST INFRASTRUCTURE ONLY: used to pin the C
// oracle (rc_oracle.c) bit-for-bit and, when present, as bench.py's CPU baseline
// (cpu_baseline.kind = "reference").  No reference source is copied into this repo.
//
// The reference namespace is renamed so these symbols can never collide with the
// product's own rotconv:: C++ drop-in (include/rotconv/*.hpp).
#define rotconv rotconv_ref
#include "rotconv/reference_conv.hpp"
#include "rotconv/scatter_conv.hpp"
#include "rotconv/tensor.hpp"
#undef rotconv

#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace R = rotconv_ref;

namespace {

template <typename T>
R::Tensor3<T> t3(const T* p, int c, int h, int w) {
  return R::Tensor3<T>::from_data(c, h, w, std::vector<T>(p, p + (size_t)c * h * w));
}
template <typename T>
R::FilterBank<T> fb(const T* p, int co, int ci, int kh, int kw) {
  return R::FilterBank<T>::from_data(co, ci, kh, kw,
                                     std::vector<T>(p, p + (size_t)co * ci * kh * kw));
}
template <typename T>
void put(const R::Tensor3<T>& t, T* out) {
  std::memcpy(out, t.data(), sizeof(T) * t.size());
}
void set_err(char* buf, size_t n, const char* s) {
  if (buf && n) {
    std::strncpy(buf, s, n - 1);
    buf[n - 1] = 0;
  }
}

// transform_kernel built from the reference plane ops.
template <typename T>
R::FilterBank<T> transform(const R::FilterBank<T>& w, int r, bool mirror) {
  R::FilterBank<T> out(w.out_channels(), w.in_channels(), w.kernel_h(), w.kernel_w());
  for (int co = 0; co < w.out_channels(); ++co)
    for (int ci = 0; ci < w.in_channels(); ++ci) {
      auto plane = R::MatrixRM<T>::from_data(
          w.kernel_h(), w.kernel_w(),
          std::vector<T>(w.plane(co, ci), w.plane(co, ci) + w.kernel_h() * w.kernel_w()));
      if (mirror) plane = R::mirror_plane(plane);
      plane = R::rot90_plane(plane, r);
      std::memcpy(out.plane(co, ci), plane.data(), sizeof(T) * plane.size());
    }
  return out;
}

template <typename T>
int tiled(const T* x, int c, int h, int w, const T* wt, int cout, int cin_w, int kh, int kw, int tile_h,
          int tile_w, int halo, int workers, int strategy, T* y, unsigned long long* mults,
          unsigned long long* adds, unsigned long long* aux_peak, char* err, size_t errn) {
  try {
    R::MultCounter mc;
    R::AuxMemCounter aux;
    R::TileConfig cfg{tile_h, tile_w, halo};
    auto out = R::tiled_scatter_conv(t3(x, c, h, w), fb(wt, cout, cin_w, kh, kw), cfg, workers, &mc,
                                     &aux,
                                     strategy == 0 ? R::ScatterStrategy::tile_private
                                                   : R::ScatterStrategy::phase_parallel);
    put(out, y);
    if (mults) *mults = mc.scalar_multiplications;
    if (adds) *adds = mc.scalar_additions;
    if (aux_peak) *aux_peak = aux.peak_bytes;
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return -1;
  }
}

// Unpooled RI output built ONLY from reference primitives: slice o = (b, r) is
// tiled_scatter_conv(X, rot90^r(K_b)) -- i.e. the no-reuse "R x tiled_scatter_conv"
// path -- with K_b = W (p4/single), mirror(W) (p4m, b = 1) or the caller-supplied
// steered bases (steer: SPEC-only, no reference code exists).
// convention 1 (raw) uses scatter_conv_raw_multi instead.
template <typename T>
int ri_slices(int group, int orientations, int convention, const T* x, int cin, int h, int w,
              const T* bases_or_w, int cout, int k, T* f) {
  const int rpb = group == 0 ? 1 : 4;
  const int nb = group == 0 ? 1 : (group == 2 ? 2 : (group == 3 ? orientations / 4 : 1));
  const size_t per = (size_t)cout * cin * k * k, plane = (size_t)h * w;
  const int RR = nb * rpb;
  auto X = t3(x, cin, h, w);
  for (int b = 0; b < nb; ++b) {
    R::FilterBank<T> base = group == 3 ? fb(bases_or_w + b * per, cout, cin, k, k)
                                       : fb(bases_or_w, cout, cin, k, k);
    if (group == 2 && b == 1) base = transform(base, 0, true);
    for (int r = 0; r < rpb; ++r) {
      auto kr = transform(base, r, false);
      R::Tensor3<T> s = convention == 0
                            ? R::tiled_scatter_conv(X, kr, R::TileConfig{32, 32, k / 2}, 1)
                            : R::scatter_conv_raw_multi(X, kr);
      for (int co = 0; co < cout; ++co)
        std::memcpy(f + ((size_t)co * RR + b * rpb + r) * plane, s.plane(co), sizeof(T) * plane);
    }
  }
  return 0;
}

}  // namespace

extern "C" {

void ref_rot90_d(const double* in, int rows, int cols, int q, double* out, int* orows,
                 int* ocols) {
  auto m = R::rot90_plane(
      R::MatrixRM<double>::from_data(rows, cols, std::vector<double>(in, in + rows * cols)), q);
  std::memcpy(out, m.data(), sizeof(double) * m.size());
  *orows = m.rows();
  *ocols = m.cols();
}
void ref_mirror_d(const double* in, int rows, int cols, double* out) {
  auto m = R::mirror_plane(
      R::MatrixRM<double>::from_data(rows, cols, std::vector<double>(in, in + rows * cols)));
  std::memcpy(out, m.data(), sizeof(double) * m.size());
}
void ref_reverse_bank_d(const double* in, int co, int ci, int kh, int kw, double* out) {
  auto b = R::reverse_bank(fb(in, co, ci, kh, kw));
  std::memcpy(out, b.data(), sizeof(double) * b.size());
}
unsigned long long ref_clipped_writes(int h, int w, int kh, int kw) {
  return R::detail::clipped_writes(h, w, kh, kw);
}
void ref_scatter_conv_single_d(const double* x, int h, int w, const double* k, int kh, int kw,
                               double* y, unsigned long long* mults, unsigned long long* adds) {
  R::MultCounter mc;
  auto out = R::scatter_conv_single(
      R::MatrixRM<double>::from_data(h, w, std::vector<double>(x, x + h * w)),
      R::MatrixRM<double>::from_data(kh, kw, std::vector<double>(k, k + kh * kw)), &mc);
  std::memcpy(y, out.data(), sizeof(double) * out.size());
  *mults = mc.scalar_multiplications;
  *adds = mc.scalar_additions;
}

#define REF_T(T, S)                                                                           \
  void ref_scatter_conv_multi_##S(const T* x, int c, int h, int w, const T* wt, int cout,      \
                                  int kh, int kw, T* y, unsigned long long* mults) {           \
    R::MultCounter mc;                                                                        \
    put(R::scatter_conv_multi(t3(x, c, h, w), fb(wt, cout, c, kh, kw), &mc), y);              \
    if (mults) *mults = mc.scalar_multiplications;                                            \
  }                                                                                           \
  void ref_scatter_conv_raw_multi_##S(const T* x, int c, int h, int w, const T* wt, int cout,  \
                                      int kh, int kw, T* y) {                                 \
    put(R::scatter_conv_raw_multi(t3(x, c, h, w), fb(wt, cout, c, kh, kw)), y);               \
  }                                                                                           \
  void ref_conv_gather_same_##S(const T* x, int c, int h, int w, const T* wt, int cout, int kh, \
                                int kw, T* y) {                                               \
    put(R::conv_gather_same(t3(x, c, h, w), fb(wt, cout, c, kh, kw)), y);                     \
  }                                                                                           \
  int ref_tiled_scatter_conv_##S(const T* x, int c, int h, int w, const T* wt, int cout,       \
                                 int cin_w, int kh, int kw, int tile_h, int tile_w, int halo,             \
                                 int workers, int strategy, T* y, unsigned long long* mults,   \
                                 unsigned long long* adds, unsigned long long* aux_peak,       \
                                 char* err, size_t errn) {                                    \
    return tiled<T>(x, c, h, w, wt, cout, cin_w, kh, kw, tile_h, tile_w, halo, workers, strategy, y,  \
                    mults, adds, aux_peak, err, errn);                                        \
  }                                                                                           \
  int ref_ri_slices_##S(int group, int orientations, int convention, const T* x, int cin,      \
                        int h, int w, const T* bases_or_w, int cout, int k, T* f) {           \
    return ri_slices<T>(group, orientations, convention, x, cin, h, w, bases_or_w, cout, k,   \
                        f);                                                                   \
  }

REF_T(float, f)
REF_T(double, d)
#undef REF_T

// Batched single-orientation reference path for the CPU baseline: images
// [begin, end) of an NCHW batch through tiled_scatter_conv (default TileConfig,
// workers = 1 per call), one std::thread per host core, images round-robin.
int ref_tiled_batch_f(const float* x, int n, int c, int h, int w, const float* wt, int cout,
                      int k, float* y, int nthreads, int begin, int end) {
  if (end > n) end = n;
  const size_t xin = (size_t)c * h * w, yout = (size_t)cout * h * w;
  auto bank = fb(wt, cout, c, k, k);
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t)
    pool.emplace_back([&, t] {
      for (int i = begin + t; i < end; i += nthreads) {
        auto out = R::tiled_scatter_conv(t3(x + i * xin, c, h, w), bank,
                                         R::TileConfig{32, 32, k / 2}, 1);
        std::memcpy(y + i * yout, out.data(), sizeof(float) * yout);
      }
    });
  for (auto& th : pool) th.join();
  return 0;
}

// The whole RI layer on a batch from the reference's own code path (the CPU baseline and
// reference arm of bench.py for R > 1): for every image the R orientation slices as
// R x tiled_scatter_conv (ri_slices above: the reference has no reuse path), then the
// SPEC orientation reduction (the reference ships no pooling) and the bias
// (P5), with the conventions of DESIGN.md (P2 orbit-major order, P3 argmax: global for
// max, block-local for subgroup, ties -> smallest index).  pool: 0 none, 1 avg, 2 max,
// 3 subgroup.  Images [begin, end), one std::thread per host core, round-robin.
int ref_ri_batch_f(int group, int orientations, int convention, int pool, int pool_group,
                   const float* x, int n, int cin, int h, int w, const float* bases_or_w, int cout,
                   int k, const float* bias, float* y, uint8_t* am, int nthreads, int begin,
                   int end) {
  if (end > n) end = n;
  const int R = orientations;
  const int gf = pool == 0 ? 1 : (pool == 3 ? pool_group : R);
  const int RO = R / gf;
  const size_t plane = (size_t)h * w, xin = (size_t)cin * plane, yout = (size_t)cout * RO * plane;
  std::vector<std::thread> pool_threads;
  for (int t = 0; t < nthreads; ++t)
    pool_threads.emplace_back([&, t] {
      std::vector<float> f((size_t)cout * R * plane);
      for (int i = begin + t; i < end; i += nthreads) {
        ri_slices<float>(group, R, convention, x + i * xin, cin, h, w, bases_or_w, cout, k, f.data());
        float* yi = y + i * yout;
        uint8_t* ai = am ? am + i * yout : nullptr;
        for (int co = 0; co < cout; ++co) {
          const float bz = bias ? bias[co] : 0.f;
          for (int s = 0; s < RO; ++s)
            for (size_t p = 0; p < plane; ++p) {
              const float* fs = f.data() + ((size_t)co * R + (size_t)s * gf) * plane + p;
              float v = fs[0];
              int arg = 0;
              if (pool == 1) {
                for (int r = 1; r < R; ++r) v += fs[(size_t)r * plane];
                v = v / (float)R;
              } else {
                for (int r = 1; r < gf; ++r)
                  if (fs[(size_t)r * plane] > v) {
                    v = fs[(size_t)r * plane];
                    arg = r;
                  }
              }
              const size_t o = ((size_t)co * RO + s) * plane + p;
              yi[o] = v + bz;
              if (ai) ai[o] = (uint8_t)arg;
            }
        }
      }
    });
  for (auto& th : pool_threads) th.join();
  return 0;
}

void ref_pack_cnhw_f(const float* batch, int n, int c, int h, int w, float* out) {
  std::vector<R::Tensor3<float>> ts;
  for (int i = 0; i < n; ++i) ts.push_back(t3(batch + (size_t)i * c * h * w, c, h, w));
  auto m = R::pack_cnhw(std::span<const R::Tensor3<float>>(ts));
  std::memcpy(out, m.data(), sizeof(float) * m.size());
}
void ref_pack_nhwc_f(const float* bank, int co, int ci, int kh, int kw, float* out) {
  auto m = R::pack_nhwc(fb(bank, co, ci, kh, kw));
  std::memcpy(out, m.data(), sizeof(float) * m.size());
}

}  // extern "C"
