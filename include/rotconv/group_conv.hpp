// rotconv/group_conv.hpp -- the rotation-invariant (RI) layer of arXiv 2512.08888 on B200.
//
// The reference ships no code for this layer: SPEC.md defines it (group_conv module,
// SPEC:245-334; steerable module).  This header gives those SPEC operations
// C++ signatures in the style of the shipped headers (namespace rotconv, containers by
// const&, results by value, optional accumulating counters) and serves them with the
// sm_100a kernels behind the C-ABI:
//
//   GroupSpec, transform_kernel        SPEC:250-264   rc_orientation_bank_host (bank kernel)
//   group_conv_gather                  SPEC:265-273   fused kernel, convention raw
//   group_conv_scatter_reuse           SPEC:274-282   fused kernel, convention scatter
//   orientation_pool_avg / _max        SPEC:283-300   rc_orientation_pool_host
//   subgroup_pool_max                  SPEC:301-309   rc_orientation_pool_host
//   SteerableBasis, OrientationSet
//   steer                              SPEC:439-447   rc_steer_host
//   build_orientation_bank             SPEC:448-456   rc_orientation_bank_host
//   gaussian_derivative_basis          SPEC:484-492   host (test fixture, K*K values)
//   loss_mag / loss_orth / total_loss  SPEC:457-483   host (B scalars; training regularisers)
//   RILayer / ri_conv_forward          (north star)   rc_ri_conv_forward_host /
//                                                     rc_mgpu_forward_host: reuse scatter +
//                                                     orientation pooling + bias, one kernel
//
// Conventions pinned in DESIGN.md (the reference leaves them open):
//   P1 slice (b, r) of the scatter convention == scatter_conv_multi(X, rot90^r(K_b));
//      the raw convention (group_conv_gather) == conv_gather_same(X, rot90^r(K_b)).
//   P2 orientation order is orbit-major, o = b*4 + r (p4m: rotations, then the mirrored
//      block; steerable: base angle 2*pi*b/N, quarter turn r).
//   P3 argmax: global index for orientation_pool_max, block-local for subgroup_pool_max,
//      ties -> smallest index; stored in ArgmaxMap (uint8).
//   P5 bias is added after the orientation reduction.
#pragma once

#include <cmath>
#include <cstdint>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "rotconv/device.hpp"
#include "rotconv/scatter_conv.hpp"
#include "rotconv/tensor.hpp"

namespace rotconv {

// ------------------------------------------------------------------------ group specs
struct GroupSpec {
  enum class Kind { p4, p4m };
  Kind kind = Kind::p4;
  int size() const { return kind == Kind::p4 ? 4 : 8; }
  static GroupSpec p4() { return {Kind::p4}; }
  static GroupSpec p4m() { return {Kind::p4m}; }
};

// group element of p4m: `mirror` (horizontal flip) applied before `r` CCW quarter turns
struct GroupElement {
  int r = 0;
  bool mirror = false;
};

enum class Pooling { none = RC_POOL_NONE, avg = RC_POOL_AVG, max = RC_POOL_MAX, subgroup = RC_POOL_SUBGROUP };

namespace detail {

inline rc_desc group_desc(int n, int cin, int h, int w, int cout, int k, int group, int R, Pooling pool,
                          int pool_group, int convention, b200::Precision prec, int activation = RC_ACT_NONE) {
  rc_desc d{};
  d.n = n;
  d.c_in = cin;
  d.h = h;
  d.w = w;
  d.c_out = cout;
  d.k = k;
  d.group = group;
  d.orientations = R;
  d.pool = static_cast<int>(pool);
  d.pool_group = pool_group;
  d.convention = convention;
  d.precision = static_cast<int>(prec);
  d.activation = activation;
  return d;
}

inline int group_code(const GroupSpec& g) { return g.kind == GroupSpec::Kind::p4 ? RC_GROUP_P4 : RC_GROUP_P4M; }

// all orbit-major kernels of a bank descriptor, [R][Cout][Cin][K][K]
inline std::vector<float> orbit_kernels(const rc_desc& d, const float* w0, const float* w1) {
  std::vector<float> out(static_cast<std::size_t>(d.orientations) * d.c_out * d.c_in * d.k * d.k);
  b200::throw_on(rc_orientation_bank_host(&d, w0, w1, out.data(), b200::device()));
  return out;
}

template <typename T>
FilterBank<T> bank_slice(const std::vector<float>& all, int o, int cout, int cin, int k) {
  const std::size_t per = static_cast<std::size_t>(cout) * cin * k * k;
  return FilterBank<T>::from_data(cout, cin, k, k, std::vector<T>(all.begin() + o * per, all.begin() + (o + 1) * per));
}

}  // namespace detail

// SPEC:256-264.  Odd square kernels go through the GPU bank kernel (the same index maps the
// conv kernels use); other shapes are exact host permutations (r in {1,3} needs square).
template <typename T>
FilterBank<T> transform_kernel(const FilterBank<T>& w, GroupElement g) {
  ROTCONV_REQUIRE_FLOAT(T);
  const int r = ((g.r % 4) + 4) % 4;
  detail::check(w.square() || r % 2 == 0, "transform_kernel: rotation needs a square kernel");
  if (w.square() && w.kernel_h() % 2 == 1) {
    const rc_desc d = detail::group_desc(1, w.in_channels(), 1, 1, w.out_channels(), w.kernel_h(), RC_GROUP_P4M, 8,
                                         Pooling::none, 1, RC_CONV_SCATTER, b200::Precision::fp32);
    const std::vector<float> all = detail::orbit_kernels(d, w.data(), nullptr);
    return detail::bank_slice<T>(all, (g.mirror ? 4 : 0) + r, w.out_channels(), w.in_channels(), w.kernel_h());
  }
  FilterBank<T> out(w.out_channels(), w.in_channels(), r % 2 ? w.kernel_w() : w.kernel_h(),
                    r % 2 ? w.kernel_h() : w.kernel_w());
  for (int co = 0; co < w.out_channels(); ++co)
    for (int ci = 0; ci < w.in_channels(); ++ci) {
      MatrixRM<T> p = MatrixRM<T>::from_data(w.kernel_h(), w.kernel_w(),
                                             std::vector<T>(w.plane(co, ci), w.plane(co, ci) + w.kernel_h() * w.kernel_w()));
      if (g.mirror) p = mirror_plane(p);
      p = rot90_plane(p, r);
      std::copy(p.data(), p.data() + p.size(), out.plane(co, ci));
    }
  return out;
}

template <typename T>
FilterBank<T> transform_kernel(const FilterBank<T>& w, int r) {
  return transform_kernel(w, GroupElement{r, false});
}

namespace detail {
template <typename T>
OrientedFeature<T> group_conv(const Tensor3<T>& x, const FilterBank<T>& w, const GroupSpec& g, MultCounter* counter,
                              int convention) {
  ROTCONV_REQUIRE_FLOAT(T);
  detail::check(x.channels() == w.in_channels(), "group_conv: channel mismatch");
  detail::check(w.square() && w.kernel_h() % 2 == 1, "transform_kernel: rotation groups need odd square kernels");
  const rc_desc d = group_desc(1, x.channels(), x.height(), x.width(), w.out_channels(), w.kernel_h(), group_code(g),
                               g.size(), Pooling::none, 1, convention, b200::precision());
  OrientedFeature<T> f(w.out_channels(), g.size(), x.height(), x.width());
  b200::throw_on(rc_ri_conv_forward_host(&d, x.data(), w.data(), nullptr, nullptr, f.data(), nullptr, b200::device()));
  if (counter) {  // one channel dot per (h,w,co,m,n) per base, |G|-independent
    unsigned long long m = 0, a = 0;
    b200::throw_on(rc_analytic_counts(&d, &m, &a));
    counter->add(m, a);
  }
  return f;
}
}  // namespace detail

// slice r = conv_gather_same(X, transform_kernel(W, r)) (raw convention)
template <typename T>
OrientedFeature<T> group_conv_gather(const Tensor3<T>& x, const FilterBank<T>& w, const GroupSpec& g) {
  return detail::group_conv(x, w, g, nullptr, RC_CONV_RAW);
}

// one channel dot per (h,w,co,m,n), scattered to |G| orientation planes
// (scatter convention, P1: slice r == scatter_conv_multi(X, transform_kernel(W, r)))
template <typename T>
OrientedFeature<T> group_conv_scatter_reuse(const Tensor3<T>& x, const FilterBank<T>& w, const GroupSpec& g,
                                            MultCounter* counter = nullptr) {
  return detail::group_conv(x, w, g, counter, RC_CONV_SCATTER);
}

// ---------------------------------------------------------------- orientation pooling
namespace detail {
inline void pool_host(const float* f, int cout, int R, int h, int w, Pooling p, int g, float* y, std::uint8_t* am) {
  b200::throw_on(rc_orientation_pool_host(1, cout, R, h, w, static_cast<int>(p), g, f, nullptr, y, am, b200::device()));
}
}  // namespace detail

// Eq. (9): (1/R) sum_r F[co, r, h, w]
template <typename T>
Tensor3<T> orientation_pool_avg(const OrientedFeature<T>& f) {
  ROTCONV_REQUIRE_FLOAT(T);
  Tensor3<T> y(f.out_channels(), f.height(), f.width());
  detail::pool_host(f.data(), f.out_channels(), f.orientations(), f.height(), f.width(), Pooling::avg, 1, y.data(),
                    nullptr);
  return y;
}

// Eq. (10): per-pixel max over r and its argmax r* (ties -> smallest r)
template <typename T>
std::pair<Tensor3<T>, ArgmaxMap> orientation_pool_max(const OrientedFeature<T>& f) {
  ROTCONV_REQUIRE_FLOAT(T);
  Tensor3<T> y(f.out_channels(), f.height(), f.width());
  ArgmaxMap a(f.out_channels(), 1, f.height(), f.width());
  detail::pool_host(f.data(), f.out_channels(), f.orientations(), f.height(), f.width(), Pooling::max, 1, y.data(),
                    a.data());
  return {std::move(y), std::move(a)};
}

// max over contiguous blocks of group_size orientations, block-local argmax
template <typename T>
std::pair<OrientedFeature<T>, ArgmaxMap> subgroup_pool_max(const OrientedFeature<T>& f, int group_size = 4) {
  ROTCONV_REQUIRE_FLOAT(T);
  detail::check(group_size >= 1 && f.orientations() % group_size == 0,
                "subgroup_pool_max: R not divisible by group_size");
  const int ro = f.orientations() / group_size;
  OrientedFeature<T> y(f.out_channels(), ro, f.height(), f.width());
  ArgmaxMap a(f.out_channels(), ro, f.height(), f.width());
  detail::pool_host(f.data(), f.out_channels(), f.orientations(), f.height(), f.width(), Pooling::subgroup, group_size,
                    y.data(), a.data());
  return {std::move(y), std::move(a)};
}

// ------------------------------------------------------------------------- steerable
template <typename T>
struct SteerableBasis {
  FilterBank<T> f_x;
  FilterBank<T> f_y;
};

struct OrientationSet {
  int count = 4;
  explicit OrientationSet(int n) : count(n) {
    detail::check(n >= 4 && n % 4 == 0, "build_orientation_bank: N must be a multiple of 4");
  }
  double angle(int k) const { return 2.0 * M_PI * k / count; }
  int first_quadrant() const { return count / 4; }
};

// Eq. (17): sin(theta) f_x + cos(theta) f_y, coefficients rounded once from double
template <typename T>
FilterBank<T> steer(const SteerableBasis<T>& basis, double theta) {
  ROTCONV_REQUIRE_FLOAT(T);
  detail::check(basis.f_x.same_shape(basis.f_y), "SteerableBasis: f_x and f_y shapes must be equal");
  const FilterBank<T>& fx = basis.f_x;
  FilterBank<T> out(fx.out_channels(), fx.in_channels(), fx.kernel_h(), fx.kernel_w());
  b200::throw_on(rc_steer_host(fx.data(), basis.f_y.data(), fx.size(), theta, out.data(), b200::device()));
  return out;
}

struct OrientationTag {
  double base_angle;  // theta_b = 2*pi*b/N, first quadrant
  int quadrant;       // r: the kernel is rot90^r(steer(theta_b)), never re-steered
};

template <typename T>
struct OrientationBank {
  std::vector<FilterBank<T>> kernels;  // orbit-major, o = b*4 + r
  std::vector<OrientationTag> tags;
};

// SPEC:448-456
template <typename T>
OrientationBank<T> build_orientation_bank(const SteerableBasis<T>& basis, int n) {
  ROTCONV_REQUIRE_FLOAT(T);
  const OrientationSet set(n);
  detail::check(basis.f_x.same_shape(basis.f_y), "SteerableBasis: f_x and f_y shapes must be equal");
  const FilterBank<T>& fx = basis.f_x;
  detail::check(fx.square() && fx.kernel_h() % 2 == 1, "transform_kernel: rotation groups need odd square kernels");
  const rc_desc d = detail::group_desc(1, fx.in_channels(), 1, 1, fx.out_channels(), fx.kernel_h(), RC_GROUP_STEER, n,
                                       Pooling::none, 1, RC_CONV_SCATTER, b200::Precision::fp32);
  const std::vector<float> all = detail::orbit_kernels(d, fx.data(), basis.f_y.data());
  OrientationBank<T> bank;
  for (int b = 0; b < set.first_quadrant(); ++b)
    for (int r = 0; r < 4; ++r) {
      bank.kernels.push_back(detail::bank_slice<T>(all, b * 4 + r, fx.out_channels(), fx.in_channels(), fx.kernel_h()));
      bank.tags.push_back({set.angle(b), r});
    }
  return bank;
}

// SPEC:484-492 (test fixture): f_x ~ -x exp(-(x^2+y^2)/2s^2), f_y ~ -y exp(..), unit L2,
// grid centred at (K/2, K/2); x runs along columns, y along rows.
template <typename T>
SteerableBasis<T> gaussian_derivative_basis(int k, double sigma, int out_channels = 1, int in_channels = 1) {
  detail::check(k >= 1 && k % 2 == 1, "gaussian_derivative_basis: K must be odd");
  detail::check(sigma > 0, "gaussian_derivative_basis: sigma must be positive");
  std::vector<double> gx(k * k), gy(k * k);
  double nx = 0, ny = 0;
  const int c = k / 2;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      const double x = j - c, y = i - c, g = std::exp(-(x * x + y * y) / (2 * sigma * sigma));
      gx[i * k + j] = -x * g;
      gy[i * k + j] = -y * g;
      nx += gx[i * k + j] * gx[i * k + j];
      ny += gy[i * k + j] * gy[i * k + j];
    }
  SteerableBasis<T> b{FilterBank<T>(out_channels, in_channels, k, k), FilterBank<T>(out_channels, in_channels, k, k)};
  for (int co = 0; co < out_channels; ++co)
    for (int ci = 0; ci < in_channels; ++ci)
      for (int t = 0; t < k * k; ++t) {
        b.f_x.plane(co, ci)[t] = static_cast<T>(gx[t] / std::sqrt(nx));
        b.f_y.plane(co, ci)[t] = static_cast<T>(gy[t] / std::sqrt(ny));
      }
  return b;
}

// SPEC:457-483 regularisers (per filter b = output channel co): host arithmetic over B
// filter pairs, not part of the forward hot path.
template <typename T>
double loss_mag(const SteerableBasis<T>& basis) {
  const int B = basis.f_x.out_channels();
  const std::size_t per = basis.f_x.size() / B;
  double acc = 0;
  for (int b = 0; b < B; ++b) {
    double sx = 0, sy = 0;
    for (std::size_t i = 0; i < per; ++i) {
      sx += double(basis.f_x.data()[b * per + i]) * basis.f_x.data()[b * per + i];
      sy += double(basis.f_y.data()[b * per + i]) * basis.f_y.data()[b * per + i];
    }
    const double d = std::sqrt(sx) - std::sqrt(sy);
    acc += d * d;
  }
  return acc / B;
}

template <typename T>
double loss_orth(const SteerableBasis<T>& basis, double eps = 1e-8) {
  detail::check(eps > 0, "loss_orth: eps must be positive");
  const int B = basis.f_x.out_channels();
  const std::size_t per = basis.f_x.size() / B;
  double acc = 0;
  for (int b = 0; b < B; ++b) {
    double sx = 0, sy = 0, sxy = 0;
    for (std::size_t i = 0; i < per; ++i) {
      const double x = basis.f_x.data()[b * per + i], y = basis.f_y.data()[b * per + i];
      sx += x * x;
      sy += y * y;
      sxy += x * y;
    }
    const double c = sxy / (std::sqrt(sx) * std::sqrt(sy) + eps);
    acc += c * c;
  }
  return acc / B;
}

template <typename T>
double total_loss(double ce, const SteerableBasis<T>& basis, double lambda_mag, double lambda_orth, double eps = 1e-8) {
  detail::check(lambda_mag >= 0 && lambda_orth >= 0, "total_loss: lambdas must be >= 0");
  return ce + lambda_mag * loss_mag(basis) + lambda_orth * loss_orth(basis, eps);
}

// ------------------------------------------------------------- the fused RI layer
// One layer = bank precompute + reuse scatter + orientation reduction + bias, over a batch
// of images, in one fused kernel launch per device.  group: p4 / p4m (w0 = W) or steer
// (w0 = f_x, w1 = f_y, `orientations` = N).
struct RILayerSpec {
  int group = RC_GROUP_STEER;
  int orientations = 8;
  Pooling pool = Pooling::subgroup;
  int pool_group = 4;
  int convention = RC_CONV_SCATTER;
  b200::Precision precision = b200::Precision::automatic;
  int activation = RC_ACT_NONE;  // RC_ACT_RELU fuses a ReLU after the bias

  int out_orientations() const {
    if (pool == Pooling::none) return orientations;
    if (pool == Pooling::subgroup) return orientations / pool_group;
    return 1;
  }
  bool has_argmax() const { return pool == Pooling::max || pool == Pooling::subgroup; }
};

struct RIBatchOutput {
  std::vector<OrientedFeature<float>> y;  // per image: Cout x R' x H x W
  std::vector<ArgmaxMap> argmax;          // per image (max / subgroup pooling), else empty
};

// Flat form: x = N contiguous Tensor3 (NCHW); y / argmax = N contiguous (Cout, R', H, W).
// devices: empty -> rotconv::b200::device(); more than one -> batch-sharded across them.
inline void ri_conv_forward(const RILayerSpec& s, int n, int cin, int h, int w, int cout, int k, const float* x,
                            const float* w0, const float* w1, const float* bias, float* y, std::uint8_t* argmax,
                            std::span<const int> devices = {}) {
  const rc_desc d = detail::group_desc(n, cin, h, w, cout, k, s.group, s.orientations, s.pool, s.pool_group,
                                       s.convention, s.precision, s.activation);
  if (devices.size() > 1)
    b200::throw_on(rc_mgpu_forward_host(&d, x, w0, w1, bias, y, argmax, static_cast<int>(devices.size()),
                                        devices.data()));
  else
    b200::throw_on(rc_ri_conv_forward_host(&d, x, w0, w1, bias, y, argmax,
                                           devices.empty() ? b200::device() : devices[0]));
}

// Container form over a batch (the reference loops over images; here the whole
// batch is one launch).  w1 is required for steerable layers.
inline RIBatchOutput ri_conv_forward(const RILayerSpec& s, std::span<const Tensor3<float>> batch,
                                     const FilterBank<float>& w0, const FilterBank<float>* w1 = nullptr,
                                     const std::vector<float>* bias = nullptr, std::span<const int> devices = {},
                                     MultCounter* counter = nullptr) {
  detail::check(!batch.empty(), "ri_conv_forward: empty batch");
  const Tensor3<float>& f = batch.front();
  for (const Tensor3<float>& t : batch) detail::check(t.same_shape(f), "ri_conv_forward: shape mismatch across the batch");
  detail::check(f.channels() == w0.in_channels(), "ri_conv_forward: channel mismatch");
  detail::check(w0.square(), "ri_conv_forward: kernel must be square");
  if (s.group == RC_GROUP_STEER)
    detail::check(w1 != nullptr && w1->same_shape(w0), "SteerableBasis: f_x and f_y shapes must be equal");
  if (bias) detail::check(static_cast<int>(bias->size()) == w0.out_channels(), "ri_conv_forward: bias must have Cout elements");
  const int n = static_cast<int>(batch.size());
  const std::size_t xi = f.size();
  std::vector<float> x(xi * n);
  for (int i = 0; i < n; ++i) std::copy(batch[i].data(), batch[i].data() + xi, x.data() + i * xi);
  const int ro = s.out_orientations();
  const std::size_t yi = static_cast<std::size_t>(w0.out_channels()) * ro * f.height() * f.width();
  std::vector<float> y(yi * n);
  std::vector<std::uint8_t> am(s.has_argmax() ? yi * n : 0);
  ri_conv_forward(s, n, f.channels(), f.height(), f.width(), w0.out_channels(), w0.kernel_h(), x.data(), w0.data(),
                  w1 ? w1->data() : nullptr, bias ? bias->data() : nullptr, y.data(), am.empty() ? nullptr : am.data(),
                  devices);
  RIBatchOutput out;
  for (int i = 0; i < n; ++i) {
    OrientedFeature<float> o(w0.out_channels(), ro, f.height(), f.width());
    std::copy(y.data() + i * yi, y.data() + (i + 1) * yi, o.data());
    out.y.push_back(std::move(o));
    if (!am.empty()) {
      ArgmaxMap a(w0.out_channels(), ro, f.height(), f.width());
      std::copy(am.data() + i * yi, am.data() + (i + 1) * yi, a.data());
      out.argmax.push_back(std::move(a));
    }
  }
  if (counter) {
    const rc_desc d = detail::group_desc(n, f.channels(), f.height(), f.width(), w0.out_channels(), w0.kernel_h(),
                                         s.group, s.orientations, s.pool, s.pool_group, s.convention, s.precision);
    unsigned long long m = 0, a = 0;
    b200::throw_on(rc_analytic_counts(&d, &m, &a));
    counter->add(m, a);
  }
  return out;
}

}  // namespace rotconv
