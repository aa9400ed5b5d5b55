// test_cpp_api.cpp -- the C++ drop-in API (include/rotconv/*.hpp) exercised the way the
// reference's own users call it, checked against the CPU oracle (oracle/librc_oracle.so,
// the C restatement pinned to the reference) and the SPEC known-answer examples.
//
//   test_cpp_api --cpu   containers, plane transforms, packers, validation messages:
//                        nothing that needs a GPU (runs in the CPU suite)
//   test_cpp_api --gpu   every GPU-served op vs the oracle (pytest -m gpu)
//
// Exit status 0 = all checks passed; every failure prints one line.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "rc_oracle.h"
#include "rotconv/group_conv.hpp"
#include "rotconv/scatter_conv.hpp"
#include "rotconv/tensor.hpp"

using namespace rotconv;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, ...)                           \
  do {                                             \
    if (cond) {                                    \
      ++g_pass;                                    \
    } else {                                       \
      ++g_fail;                                    \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                    \
      std::printf("\n");                           \
    }                                              \
  } while (0)

template <typename E>
static std::string thrown(const std::function<void()>& f) {
  try {
    f();
  } catch (const E& e) {
    return e.what();
  } catch (...) {
    return "<other exception>";
  }
  return "<no exception>";
}

// dyadic values k/4, k in [-4, 4]: all products and partial sums exact in FP32
static std::vector<float> dyadic(std::mt19937_64& g, std::size_t n) {
  std::uniform_int_distribution<int> d(-4, 4);
  std::vector<float> v(n);
  for (float& x : v) x = d(g) / 4.0f;
  return v;
}

static rco_desc odesc(int n, int cin, int h, int w, int cout, int k, int group, int R, int pool, int g, int conv) {
  rco_desc d{n, cin, h, w, cout, k, group, R, pool, g, conv};
  return d;
}

// ---------------------------------------------------------------------------- CPU part
static void test_containers() {
  Tensor3<float> t(2, 3, 4, 1.5f);
  CHECK(t.size() == 24 && t(1, 2, 3) == 1.5f, "Tensor3 fill");
  t(1, 2, 3) = 7;
  CHECK(t.plane(1)[2 * 4 + 3] == 7, "Tensor3 plane layout");
  CHECK(thrown<std::invalid_argument>([] { Tensor3<float>(0, 1, 1); }) == "Tensor3: dimensions must be positive",
        "Tensor3 ctor message");
  CHECK(thrown<std::out_of_range>([&] { (void)t.at(2, 0, 0); }) == "Tensor3: index (2,0,0) out of range",
        "Tensor3 at message");
  CHECK(thrown<std::invalid_argument>([] { Tensor3<float>::from_data(1, 2, 2, {1, 2, 3}); }) ==
            "Tensor3: data length must equal C*H*W",
        "from_data message");
  FilterBank<double> b(2, 3, 3, 3);
  b(1, 2, 0, 1) = 4;
  CHECK(b.plane(1, 2)[1] == 4, "FilterBank layout");
  CHECK(thrown<std::invalid_argument>([] { FilterBank<float>(1, 0, 3, 3); }) ==
            "FilterBank: channel counts must be positive",
        "FilterBank message");
  CHECK(thrown<std::invalid_argument>([] { FilterBank<float>(1, 1, 0, 3); }) == "FilterBank: kernel dims must be >= 1",
        "FilterBank kernel message");
  CHECK(thrown<std::out_of_range>([&] { (void)b.at(0, 0, 3, 0); }) == "FilterBank: index out of range", "FilterBank at");
  OrientedFeature<float> f(2, 4, 3, 3);
  f(1, 3, 2, 1) = 5;
  CHECK(f.slice(1, 3)[2 * 3 + 1] == 5 && f.orientation(3)(1, 2, 1) == 5, "OrientedFeature layout");
  CHECK(thrown<std::invalid_argument>([] { OrientedFeature<float>(1, 0, 1, 1); }) ==
            "OrientedFeature: orientations must be >= 1",
        "OrientedFeature message");
  MatrixRM<float> I = MatrixRM<float>::identity(3);
  CHECK(I(1, 1) == 1 && I(0, 1) == 0, "identity");
  CHECK(thrown<std::invalid_argument>([] { MatrixRM<float>(0, 2); }) == "MatrixRM: dimensions must be positive",
        "MatrixRM message");
}

static void test_transforms() {
  // rot90([[1..9]], 1) = [[3,6,9],[2,5,8],[1,4,7]], 4 turns = identity
  auto m = MatrixRM<float>::from_data(3, 3, {1, 2, 3, 4, 5, 6, 7, 8, 9});
  auto r1 = rot90_plane(m, 1);
  const float want[9] = {3, 6, 9, 2, 5, 8, 1, 4, 7};
  CHECK(std::memcmp(r1.data(), want, sizeof want) == 0, "rot90 KAT");
  auto r4 = rot90_plane(rot90_plane(r1, 2), 1);
  CHECK(std::memcmp(r4.data(), m.data(), 9 * sizeof(float)) == 0, "rot90^4 identity");
  auto two = rot90_plane(MatrixRM<float>::from_data(2, 2, {1, 2, 3, 4}), 2);
  const float w2[4] = {4, 3, 2, 1};
  CHECK(std::memcmp(two.data(), w2, sizeof w2) == 0, "rot90^2 KAT");
  // rectangular plane vs the oracle (index permutation, exact)
  auto rect = MatrixRM<float>::from_data(2, 3, {1, 2, 3, 4, 5, 6});
  for (int q = -1; q < 6; ++q) {
    double in[6], out[6];
    for (int i = 0; i < 6; ++i) in[i] = rect.data()[i];
    int orows, ocols;
    rco_rot90_plane_d(in, 2, 3, q, out, &orows, &ocols);
    auto r = rot90_plane(rect, q);
    bool ok = r.rows() == orows && r.cols() == ocols;
    for (int i = 0; ok && i < 6; ++i) ok = r.data()[i] == out[i];
    CHECK(ok, "rot90 rect q=%d vs oracle", q);
  }
  auto mir = mirror_plane(MatrixRM<float>::from_data(1, 3, {1, 2, 3}));
  CHECK(mir(0, 0) == 3 && mir(0, 2) == 1, "mirror KAT (SPEC:60)");
  auto rp = reverse_plane(m);
  CHECK(rp(0, 0) == 9 && rp(2, 2) == 1 && rp(1, 0) == 6, "reverse_plane");
}

static void test_packers() {
  std::mt19937_64 g(5);
  std::vector<Tensor3<float>> batch;
  for (int n = 0; n < 3; ++n) batch.push_back(Tensor3<float>::from_data(2, 3, 4, dyadic(g, 24)));
  auto m = pack_cnhw<float>(batch);
  CHECK(m.rows() == 2 && m.cols() == 36 && m(1, 12 + 5) == batch[1].plane(1)[5], "pack_cnhw layout");
  auto back = unpack_cnhw(m, 2, 3, 4, 3);
  bool same = true;
  for (int n = 0; n < 3; ++n) same = same && std::memcmp(back[n].data(), batch[n].data(), 24 * 4) == 0;
  CHECK(same, "cnhw round trip");
  CHECK(thrown<std::invalid_argument>([] { pack_cnhw<float>(std::span<const Tensor3<float>>{}); }) ==
            "pack_cnhw: empty batch",
        "pack_cnhw empty");
  auto w = FilterBank<float>::from_data(2, 3, 3, 3, dyadic(g, 54));
  auto p = pack_nhwc(w);
  CHECK(p(1, (1 * 3 + 2) * 3 + 2) == w(1, 2, 1, 2), "pack_nhwc layout");
  auto wb = unpack_nhwc(p, 2, 3, 3, 3);
  CHECK(std::memcmp(wb.data(), w.data(), 54 * 4) == 0, "nhwc round trip");
}

static void test_validation_without_device() {
  // tiled_scatter_conv preconditions, reference order and messages (scatter_conv.hpp:339-346)
  Tensor3<float> x(3, 4, 4);
  FilterBank<float> w3(2, 3, 3, 3), w2(2, 2, 3, 3), wr(2, 3, 3, 5);
  auto msg = [&](const FilterBank<float>& w, TileConfig c, int workers) {
    return thrown<std::invalid_argument>([&] { tiled_scatter_conv(x, w, c, workers); });
  };
  CHECK(msg(w2, {}, 1) == "tiled_scatter_conv: channel mismatch", "channel mismatch: %s", msg(w2, {}, 1).c_str());
  CHECK(msg(wr, {}, 1) == "tiled_scatter_conv: kernel must be square", "square");
  CHECK(msg(w3, {0, 4, 1}, 1) == "tiled_scatter_conv: tile dims must be >= 1", "tile dims");
  CHECK(msg(w3, {8, 8, 2}, 1) == "tiled_scatter_conv: invalid halo", "halo");
  CHECK(msg(w3, {8, 8, 1}, 0) == "tiled_scatter_conv: workers must be >= 1", "workers");
  CHECK(thrown<std::invalid_argument>([] { OrientationSet(6); }) == "build_orientation_bank: N must be a multiple of 4",
        "OrientationSet");
  OrientedFeature<float> f(1, 6, 2, 2);
  CHECK(thrown<std::invalid_argument>([&] { subgroup_pool_max(f, 4); }) ==
            "subgroup_pool_max: R not divisible by group_size",
        "subgroup divisibility");
  // analytic counters (scatter_conv.hpp:94-110; SURVEY 0.1 probe values)
  CHECK(detail::clipped_writes(16, 16, 3, 3) == 2116 && detail::clipped_writes(32, 32, 3, 3) == 8836 &&
            detail::clipped_writes(8, 8, 3, 3) == 484,
        "clipped_writes");
  // loss KATs: norms 3 and 1 -> 4; w_y = w_x -> ~1
  SteerableBasis<float> b{FilterBank<float>::from_data(1, 1, 1, 1, {3}), FilterBank<float>::from_data(1, 1, 1, 1, {1})};
  CHECK(std::fabs(loss_mag(b) - 4.0) < 1e-12, "loss_mag KAT");
  CHECK(std::fabs(loss_orth(b) - 1.0) < 1e-6, "loss_orth correlated");
  auto gd = gaussian_derivative_basis<double>(5, 1.0);
  CHECK(loss_mag(gd) < 1e-20 && loss_orth(gd) < 1e-20, "gaussian basis orthogonal, equal norms");
  CHECK(std::fabs(gd.f_x(0, 0, 3, 2)) == 0.0, "f_x zero column at x=0");
}

// ---------------------------------------------------------------------------- GPU part
static void test_scatter_single_kats() {
  // 3x3 all-ones on [[1..9]] -> Y[1,1] = 45, Y[0,0] = 12, mults 81, adds 49
  auto x = MatrixRM<float>::from_data(3, 3, {1, 2, 3, 4, 5, 6, 7, 8, 9});
  MatrixRM<float> ones(3, 3, 1.f);
  MultCounter c;
  auto y = scatter_conv_single(x, ones, &c);
  CHECK(y(1, 1) == 45 && y(0, 0) == 12, "scatter_single KAT: %g %g", y(1, 1), y(0, 0));
  CHECK(c.scalar_multiplications == 81 && c.scalar_additions == 49, "counter KAT");
  // delta kernel -> identity; rectangular kernels vs the oracle
  MatrixRM<float> delta(3, 3);
  delta(1, 1) = 1;
  auto yd = scatter_conv_single(x, delta);
  CHECK(std::memcmp(yd.data(), x.data(), 36) == 0, "delta identity");
  std::mt19937_64 g(11);
  for (auto [kh, kw] : {std::pair{1, 3}, {3, 1}, {2, 3}, {4, 2}, {2, 2}, {5, 3}}) {
    auto xs = MatrixRM<float>::from_data(6, 7, dyadic(g, 42));
    auto ks = MatrixRM<float>::from_data(kh, kw, dyadic(g, kh * kw));
    for (int raw = 0; raw < 2; ++raw) {
      auto yy = raw ? scatter_conv_raw_single(xs, ks) : scatter_conv_single(xs, ks);
      std::vector<float> ref(42);
      unsigned long long m, a;
      if (raw)
        rco_scatter_conv_raw_single_f(xs.data(), 6, 7, ks.data(), kh, kw, ref.data(), &m, &a);
      else
        rco_scatter_conv_single_f(xs.data(), 6, 7, ks.data(), kh, kw, ref.data(), &m, &a);
      CHECK(std::memcmp(yy.data(), ref.data(), 42 * 4) == 0, "single %dx%d raw=%d bit-exact", kh, kw, raw);
    }
  }
}

static void test_multi_and_tiled() {
  std::mt19937_64 g(21);
  struct Case {
    int cin, h, w, cout, k;
  };
  for (Case c : {Case{3, 8, 8, 5, 3}, Case{64, 8, 8, 256, 3}, Case{4, 7, 9, 3, 5}, Case{2, 5, 6, 3, 1},
                 Case{3, 6, 5, 2, 2}}) {
    auto x = Tensor3<float>::from_data(c.cin, c.h, c.w, dyadic(g, (size_t)c.cin * c.h * c.w));
    auto w = FilterBank<float>::from_data(c.cout, c.cin, c.k, c.k, dyadic(g, (size_t)c.cout * c.cin * c.k * c.k));
    std::vector<float> ref((size_t)c.cout * c.h * c.w), rraw(ref.size());
    rco_scatter_conv_multi_f(x.data(), c.cin, c.h, c.w, w.data(), c.cout, c.k, c.k, ref.data());
    rco_scatter_conv_raw_multi_f(x.data(), c.cin, c.h, c.w, w.data(), c.cout, c.k, c.k, rraw.data());
    MultCounter mc;
    auto y = scatter_conv_multi(x, w, &mc);
    CHECK(std::memcmp(y.data(), ref.data(), ref.size() * 4) == 0, "scatter_conv_multi cin=%d k=%d", c.cin, c.k);
    {  // the FP32 CUDA-core path, selected per thread, agrees bit-for-bit on dyadic inputs
      b200::PrecisionScope fp32(b200::Precision::fp32);
      auto y32 = scatter_conv_multi(x, w);
      CHECK(std::memcmp(y32.data(), ref.data(), ref.size() * 4) == 0, "scatter_conv_multi fp32 cin=%d", c.cin);
    }
    CHECK(b200::precision() == b200::Precision::automatic, "default precision restored");
    auto yr = scatter_conv_raw_multi(x, w);
    CHECK(std::memcmp(yr.data(), rraw.data(), ref.size() * 4) == 0, "scatter_conv_raw_multi k=%d", c.k);
    CHECK(mc.scalar_multiplications == (unsigned long long)c.h * c.w * c.k * c.k * c.cin * c.cout, "multi mults");
    if (c.k % 2 == 1) {
      for (auto strat : {ScatterStrategy::tile_private, ScatterStrategy::phase_parallel}) {
        MultCounter tc;
        AuxMemCounter aux;
        auto yt = tiled_scatter_conv(x, w, TileConfig{5, 5, c.k / 2}, 4, &tc, &aux, strat);
        CHECK(std::memcmp(yt.data(), ref.data(), ref.size() * 4) == 0, "tiled_scatter_conv k=%d", c.k);
        CHECK(tc.scalar_multiplications == mc.scalar_multiplications &&
                  tc.scalar_additions == detail::clipped_writes(c.h, c.w, c.k, c.k) * c.cout,
              "tiled counters");
        CHECK(aux.current_bytes == 0, "aux released");
        // the reference's accounting (scatter_conv.hpp:351-360): 5x5 float tiles x 4 workers
        CHECK(aux.peak_bytes == (strat == ScatterStrategy::tile_private ? 5u * 5u * 4u * 4u : 0u),
              "aux peak %zu", aux.peak_bytes);
      }
    }
  }
  // rectangular multi-channel kernel (reference accepts it in scatter_conv_multi)
  auto x = Tensor3<float>::from_data(2, 5, 6, dyadic(g, 60));
  auto w = FilterBank<float>::from_data(3, 2, 1, 3, dyadic(g, 18));
  std::vector<float> ref(90);
  rco_scatter_conv_multi_f(x.data(), 2, 5, 6, w.data(), 3, 1, 3, ref.data());
  auto y = scatter_conv_multi(x, w);
  CHECK(std::memcmp(y.data(), ref.data(), 90 * 4) == 0, "scatter_conv_multi rectangular");
}

static void test_group_ops() {
  std::mt19937_64 g(31);
  // transform_kernel KATs
  auto k = FilterBank<float>::from_data(1, 1, 3, 3, {1, 2, 3, 4, 5, 6, 7, 8, 9});
  auto t1 = transform_kernel(k, 1);
  const float want[9] = {3, 6, 9, 2, 5, 8, 1, 4, 7};
  CHECK(std::memcmp(t1.data(), want, sizeof want) == 0, "transform_kernel r=1 KAT");
  auto t22 = transform_kernel(transform_kernel(k, 2), 2);
  CHECK(std::memcmp(t22.data(), k.data(), 36) == 0, "r=2 twice identity");
  auto km = transform_kernel(k, GroupElement{1, true});
  std::vector<float> okm(9);
  rco_transform_kernel_f(k.data(), 1, 1, 3, 1, 1, okm.data());
  CHECK(std::memcmp(km.data(), okm.data(), 36) == 0, "p4m element vs oracle");
  // group convs vs the oracle, dyadic (bit-exact)
  for (auto gs : {GroupSpec::p4(), GroupSpec::p4m()}) {
    const int cin = 5, h = 9, w = 7, cout = 6, R = gs.size();
    auto x = Tensor3<float>::from_data(cin, h, w, dyadic(g, cin * h * w));
    auto W = FilterBank<float>::from_data(cout, cin, 3, 3, dyadic(g, cout * cin * 9));
    for (int conv = 0; conv < 2; ++conv) {
      MultCounter mc;
      auto f = conv == 0 ? group_conv_scatter_reuse(x, W, gs, &mc) : group_conv_gather(x, W, gs);
      const rco_desc d = odesc(1, cin, h, w, cout, 3, gs.size() == 4 ? RCO_GROUP_P4 : RCO_GROUP_P4M, R, RCO_POOL_NONE,
                               1, conv == 0 ? RCO_CONV_SCATTER : RCO_CONV_RAW);
      std::vector<float> ref((size_t)cout * R * h * w);
      rco_ri_forward_f(&d, x.data(), W.data(), nullptr, nullptr, ref.data(), nullptr, 1, 0, 1);
      CHECK(std::memcmp(f.data(), ref.data(), ref.size() * 4) == 0, "group conv R=%d conv=%d", R, conv);
      if (conv == 0)
        CHECK(mc.scalar_multiplications == (unsigned long long)h * w * 9 * cin * cout * (R == 8 ? 2 : 1),
              "reuse mult count per base");
      if (conv == 0) {  // pools on the GPU-computed stack vs the oracle pools
        std::vector<float> pa((size_t)cout * h * w), pm(pa.size()), ps((size_t)cout * (R / 4) * h * w);
        std::vector<uint8_t> am(pm.size()), as(ps.size());
        rco_orientation_pool_avg_f(f.data(), cout, R, h, w, pa.data());
        rco_orientation_pool_max_f(f.data(), cout, R, h, w, pm.data(), am.data());
        rco_subgroup_pool_max_f(f.data(), cout, R, h, w, 4, ps.data(), as.data());
        auto ya = orientation_pool_avg(f);
        auto [ym, aa] = orientation_pool_max(f);
        auto [ys, sa] = subgroup_pool_max(f, 4);
        CHECK(std::memcmp(ya.data(), pa.data(), pa.size() * 4) == 0, "pool avg");
        CHECK(std::memcmp(ym.data(), pm.data(), pm.size() * 4) == 0 && std::memcmp(aa.data(), am.data(), am.size()) == 0,
              "pool max + argmax");
        CHECK(std::memcmp(ys.data(), ps.data(), ps.size() * 4) == 0 && std::memcmp(sa.data(), as.data(), as.size()) == 0,
              "subgroup pool + argmax");
      }
    }
  }
  // pool KATs
  OrientedFeature<float> f(1, 4, 1, 1);
  for (int r = 0; r < 4; ++r) f(0, r, 0, 0) = r + 1.f;
  CHECK(orientation_pool_avg(f)(0, 0, 0) == 2.5f, "avg KAT");
  auto [mv, ma] = orientation_pool_max(f);
  CHECK(mv(0, 0, 0) == 4 && ma(0, 0, 0, 0) == 3, "max KAT");
  OrientedFeature<float> e(1, 4, 1, 1, 2.f);
  CHECK(orientation_pool_max(e).second(0, 0, 0, 0) == 0, "tie -> smallest r");
}

static void test_steerable_and_layer() {
  // steer KATs
  auto gd = gaussian_derivative_basis<float>(3, 1.0, 2, 2);
  auto s0 = steer(gd, 0.0);
  bool eq0 = true;  // value equality: 0*f_x + (-0) is +0, so signed zeros may differ
  for (size_t i = 0; i < s0.size(); ++i) eq0 = eq0 && s0.data()[i] == gd.f_y.data()[i];
  CHECK(eq0, "steer(0) = f_y");
  auto s90 = steer(gd, M_PI / 2);
  double e90 = 0;
  for (size_t i = 0; i < s90.size(); ++i) e90 = std::max(e90, (double)std::fabs(s90.data()[i] - gd.f_x.data()[i]));
  CHECK(e90 < 1e-7, "steer(pi/2) = f_x (%g)", e90);
  // build_orientation_bank vs the oracle bank, bit-exact (same rounding of the coefficients)
  std::mt19937_64 g(41);
  const int cout = 3, cin = 2;
  SteerableBasis<float> basis{FilterBank<float>::from_data(cout, cin, 3, 3, dyadic(g, cout * cin * 9)),
                              FilterBank<float>::from_data(cout, cin, 3, 3, dyadic(g, cout * cin * 9))};
  for (int N : {4, 8, 16}) {
    auto bank = build_orientation_bank(basis, N);
    CHECK((int)bank.kernels.size() == N && bank.tags[4 % N].quadrant == (N == 4 ? 0 : 0), "bank size N=%d", N);
    const rco_desc d = odesc(1, cin, 1, 1, cout, 3, RCO_GROUP_STEER, N, RCO_POOL_NONE, 1, RCO_CONV_SCATTER);
    std::vector<float> ref((size_t)N * cout * cin * 9);
    rco_build_orientation_bank_f(&d, basis.f_x.data(), basis.f_y.data(), ref.data());
    bool ok = true;
    for (int o = 0; o < N; ++o) ok = ok && std::memcmp(bank.kernels[o].data(), ref.data() + o * cout * cin * 9, cout * cin * 9 * 4) == 0;
    CHECK(ok, "build_orientation_bank N=%d vs oracle", N);
  }
  // the fused layer: batch, steer R=8, subgroup-4 max + argmax + bias, on 1 and 2 "devices"
  const int n = 3, lc = 8, h = 16, w = 16, lo = 16;
  std::vector<Tensor3<float>> batch;
  for (int i = 0; i < n; ++i) batch.push_back(Tensor3<float>::from_data(lc, h, w, dyadic(g, lc * h * w)));
  auto fx = FilterBank<float>::from_data(lo, lc, 3, 3, dyadic(g, lo * lc * 9));
  auto fy = FilterBank<float>::from_data(lo, lc, 3, 3, dyadic(g, lo * lc * 9));
  std::vector<float> bias = dyadic(g, lo);
  for (int group : {RC_GROUP_P4M, RC_GROUP_STEER}) {
    RILayerSpec s;
    s.group = group;
    s.orientations = 8;
    MultCounter mc;
    auto out = ri_conv_forward(s, batch, fx, group == RC_GROUP_STEER ? &fy : nullptr, &bias, {}, &mc);
    const rco_desc d = odesc(n, lc, h, w, lo, 3, group == RC_GROUP_STEER ? RCO_GROUP_STEER : RCO_GROUP_P4M, 8,
                             RCO_POOL_SUBGROUP, 4, RCO_CONV_SCATTER);
    std::vector<float> x(n * lc * h * w), ref(n * lo * 2 * h * w);
    std::vector<uint8_t> am(ref.size());
    for (int i = 0; i < n; ++i) std::copy(batch[i].data(), batch[i].data() + lc * h * w, x.data() + i * lc * h * w);
    rco_ri_forward_f(&d, x.data(), fx.data(), group == RC_GROUP_STEER ? fy.data() : nullptr, bias.data(), ref.data(),
                     am.data(), 1, 0, n);
    double err = 0, mx = 0;
    int amis = 0;
    for (int i = 0; i < n; ++i)
      for (size_t j = 0; j < out.y[i].size(); ++j) {
        err = std::max(err, (double)std::fabs(out.y[i].data()[j] - ref[i * out.y[i].size() + j]));
        mx = std::max(mx, (double)std::fabs(ref[i * out.y[i].size() + j]));
        amis += out.argmax[i].data()[j] != am[i * out.y[i].size() + j];
      }
    // p4m dyadic: exact; steer: irrational coefficients -> FP32 tolerance
    if (group == RC_GROUP_P4M)
      CHECK(err == 0 && amis == 0, "fused p4m layer bit-exact (err %g, argmax mismatches %d)", err, amis);
    else
      CHECK(err <= 2e-6 * mx, "fused steer layer normwise %g", err / mx);
    CHECK(mc.scalar_multiplications == (unsigned long long)n * h * w * 9 * lc * lo * 2, "layer mults");
    // batch-sharded over the same device twice is rejected; over {0} is the plain path
    const int devs1[1] = {0};
    auto out1 = ri_conv_forward(s, batch, fx, group == RC_GROUP_STEER ? &fy : nullptr, &bias, devs1);
    bool same = true;
    for (int i = 0; i < n; ++i) same = same && std::memcmp(out1.y[i].data(), out.y[i].data(), out.y[i].size() * 4) == 0;
    CHECK(same, "explicit device list");
    const int dup[2] = {0, 0};
    CHECK(thrown<std::invalid_argument>([&] { ri_conv_forward(s, batch, fx, &fy, &bias, dup); }) ==
              "mgpu_forward: duplicate device",
          "duplicate device rejected");
  }
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  test_containers();
  test_transforms();
  test_packers();
  test_validation_without_device();
  if (gpu) {
    test_scatter_single_kats();
    test_multi_and_tiled();
    test_group_ops();
    test_steerable_and_layer();
  }
  std::printf("%s: %d passed, %d failed\n", gpu ? "gpu" : "cpu", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
