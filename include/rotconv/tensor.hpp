// rotconv/tensor.hpp -- host containers of the B200 drop-in (namespace rotconv).
//
// Same public surface, layouts and error strings as the reference containers in
// /root/reference/proj/include/rotconv/tensor.hpp, so code written against the reference
// compiles unchanged against this tree:
//   Tensor3<T>         C x H x W                 (reference tensor.hpp:30-101)
//   FilterBank<T>      Cout x Cin x Kh x Kw      (tensor.hpp:104-188)
//   OrientedFeature<T> Cout x R x H x W          (tensor.hpp:191-276)
//   MatrixRM<T>        rows x cols, row-major    (tensor.hpp:279-343)
//   rot90_plane / mirror_plane                   (tensor.hpp:345-370)
//   pack_cnhw / unpack_cnhw / pack_nhwc / unpack_nhwc (tensor.hpp:372-439)
// plus ArgmaxMap, the uint8 orientation-index map the reference has no container for
// (pinned convention P3 in DESIGN.md).
//
// The containers are plain host memory.  All of them sit on one dense N-d grid type
// (detail::Grid) that owns the storage and the shape; the named classes only add the
// reference's accessor names and messages.  The GPU ops in scatter_conv.hpp /
// group_conv.hpp take and return these containers and run on the device through the
// C-ABI (include/rotconv_c.h); matmul and the gather/im2col oracles of the reference are
// not part of the drop-in (they serve its CPU tests only).
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace rotconv {

namespace detail {

// precondition failure -> std::invalid_argument carrying the reference's message
inline void check(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

// Dense row-major grid of N dimensions; the extents are stored outermost first.
template <typename T, std::size_t N>
class Grid {
 public:
  using value_type = T;
  Grid() = default;

  std::size_t size() const { return cells_.size(); }
  T* data() { return cells_.data(); }
  const T* data() const { return cells_.data(); }
  std::span<T> values() { return {cells_.data(), cells_.size()}; }
  std::span<const T> values() const { return {cells_.data(), cells_.size()}; }
  void fill(T v) {
    for (T& c : cells_) c = v;
  }

 protected:
  Grid(std::array<int, N> ext, T init) : ext_(ext) {
    std::size_t n = 1;
    for (int e : ext_) n *= e > 0 ? static_cast<std::size_t>(e) : 0;
    cells_.assign(n, init);
  }
  // linear offset of a multi-index (no bounds check)
  template <typename... I>
  std::size_t lin(I... idx) const {
    static_assert(sizeof...(I) == N);
    const int ii[N] = {static_cast<int>(idx)...};
    std::size_t off = 0;
    for (std::size_t d = 0; d < N; ++d) off = off * static_cast<std::size_t>(ext_[d]) + ii[d];
    return off;
  }
  template <typename... I>
  bool inside(I... idx) const {
    const int ii[N] = {static_cast<int>(idx)...};
    for (std::size_t d = 0; d < N; ++d)
      if (ii[d] < 0 || ii[d] >= ext_[d]) return false;
    return true;
  }
  bool same_extents(const Grid& o) const { return ext_ == o.ext_; }
  void adopt(std::vector<T>&& v, const char* what) {
    check(v.size() == cells_.size(), what);
    cells_ = std::move(v);
  }
  T* span_at(std::size_t off) { return cells_.data() + off; }
  const T* span_at(std::size_t off) const { return cells_.data() + off; }

  std::array<int, N> ext_{};
  std::vector<T> cells_;
};

}  // namespace detail

// ---------------------------------------------------------------------------- Tensor3
template <typename T>
class Tensor3 : public detail::Grid<T, 3> {
  static_assert(std::is_floating_point_v<T>, "Tensor3 holds floating-point values");
  using G = detail::Grid<T, 3>;

 public:
  Tensor3() = default;
  Tensor3(int channels, int height, int width, T fill = T(0))
      : G(checked(channels, height, width), fill) {}

  static Tensor3 from_data(int channels, int height, int width, std::vector<T> data) {
    Tensor3 t(channels, height, width);
    t.adopt(std::move(data), "Tensor3: data length must equal C*H*W");
    return t;
  }

  int channels() const { return this->ext_[0]; }
  int height() const { return this->ext_[1]; }
  int width() const { return this->ext_[2]; }

  T& operator()(int c, int h, int w) { return this->cells_[this->lin(c, h, w)]; }
  const T& operator()(int c, int h, int w) const { return this->cells_[this->lin(c, h, w)]; }
  T& at(int c, int h, int w) { return this->cells_[this->lin(guard(c, h, w), h, w)]; }
  const T& at(int c, int h, int w) const { return this->cells_[this->lin(guard(c, h, w), h, w)]; }

  T* plane(int c) { return this->span_at(this->lin(c, 0, 0)); }
  const T* plane(int c) const { return this->span_at(this->lin(c, 0, 0)); }
  bool same_shape(const Tensor3& o) const { return this->same_extents(o); }

 private:
  static std::array<int, 3> checked(int c, int h, int w) {
    detail::check(c >= 1 && h >= 1 && w >= 1, "Tensor3: dimensions must be positive");
    return {c, h, w};
  }
  int guard(int c, int h, int w) const {
    if (!this->inside(c, h, w))
      throw std::out_of_range("Tensor3: index (" + std::to_string(c) + "," + std::to_string(h) + "," +
                              std::to_string(w) + ") out of range");
    return c;
  }
};

// ------------------------------------------------------------------------- FilterBank
template <typename T>
class FilterBank : public detail::Grid<T, 4> {
  static_assert(std::is_floating_point_v<T>, "FilterBank holds floating-point values");
  using G = detail::Grid<T, 4>;

 public:
  FilterBank() = default;
  FilterBank(int out_channels, int in_channels, int kernel_h, int kernel_w, T fill = T(0))
      : G(checked(out_channels, in_channels, kernel_h, kernel_w), fill) {}

  static FilterBank from_data(int out_channels, int in_channels, int kernel_h, int kernel_w,
                              std::vector<T> data) {
    FilterBank b(out_channels, in_channels, kernel_h, kernel_w);
    b.adopt(std::move(data), "FilterBank: data length must equal Cout*Cin*Kh*Kw");
    return b;
  }

  int out_channels() const { return this->ext_[0]; }
  int in_channels() const { return this->ext_[1]; }
  int kernel_h() const { return this->ext_[2]; }
  int kernel_w() const { return this->ext_[3]; }
  bool square() const { return kernel_h() == kernel_w(); }

  T& operator()(int co, int ci, int i, int j) { return this->cells_[this->lin(co, ci, i, j)]; }
  const T& operator()(int co, int ci, int i, int j) const { return this->cells_[this->lin(co, ci, i, j)]; }
  T& at(int co, int ci, int i, int j) {
    guard(co, ci, i, j);
    return (*this)(co, ci, i, j);
  }
  const T& at(int co, int ci, int i, int j) const {
    guard(co, ci, i, j);
    return (*this)(co, ci, i, j);
  }

  T* plane(int co, int ci) { return this->span_at(this->lin(co, ci, 0, 0)); }
  const T* plane(int co, int ci) const { return this->span_at(this->lin(co, ci, 0, 0)); }
  bool same_shape(const FilterBank& o) const { return this->same_extents(o); }

 private:
  static std::array<int, 4> checked(int co, int ci, int kh, int kw) {
    detail::check(co >= 1 && ci >= 1, "FilterBank: channel counts must be positive");
    detail::check(kh >= 1 && kw >= 1, "FilterBank: kernel dims must be >= 1");
    return {co, ci, kh, kw};
  }
  void guard(int co, int ci, int i, int j) const {
    if (!this->inside(co, ci, i, j)) throw std::out_of_range("FilterBank: index out of range");
  }
};

// -------------------------------------------------------------------- MatrixRM (2-D plane)
template <typename T>
class MatrixRM : public detail::Grid<T, 2> {
  static_assert(std::is_floating_point_v<T>, "MatrixRM holds floating-point values");
  using G = detail::Grid<T, 2>;

 public:
  MatrixRM() = default;
  MatrixRM(int rows, int cols, T fill = T(0)) : G(checked(rows, cols), fill) {}

  static MatrixRM from_data(int rows, int cols, std::vector<T> data) {
    MatrixRM m(rows, cols);
    m.adopt(std::move(data), "MatrixRM: data length must equal rows*cols");
    return m;
  }
  static MatrixRM identity(int n) {
    MatrixRM m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = T(1);
    return m;
  }

  int rows() const { return this->ext_[0]; }
  int cols() const { return this->ext_[1]; }
  T& operator()(int r, int c) { return this->cells_[this->lin(r, c)]; }
  const T& operator()(int r, int c) const { return this->cells_[this->lin(r, c)]; }
  T& at(int r, int c) {
    guard(r, c);
    return (*this)(r, c);
  }
  const T& at(int r, int c) const {
    guard(r, c);
    return (*this)(r, c);
  }
  T* row(int r) { return this->span_at(this->lin(r, 0)); }
  const T* row(int r) const { return this->span_at(this->lin(r, 0)); }
  bool same_shape(const MatrixRM& o) const { return this->same_extents(o); }

 private:
  static std::array<int, 2> checked(int r, int c) {
    detail::check(r >= 1 && c >= 1, "MatrixRM: dimensions must be positive");
    return {r, c};
  }
  void guard(int r, int c) const {
    if (!this->inside(r, c)) throw std::out_of_range("MatrixRM: index out of range");
  }
};

// --------------------------------------------------------------------- OrientedFeature
template <typename T>
class OrientedFeature : public detail::Grid<T, 4> {
  static_assert(std::is_floating_point_v<T>, "OrientedFeature holds floating-point values");
  using G = detail::Grid<T, 4>;

 public:
  OrientedFeature() = default;
  OrientedFeature(int out_channels, int orientations, int height, int width, T fill = T(0))
      : G(checked(out_channels, orientations, height, width), fill) {}

  int out_channels() const { return this->ext_[0]; }
  int orientations() const { return this->ext_[1]; }
  int height() const { return this->ext_[2]; }
  int width() const { return this->ext_[3]; }

  T& operator()(int co, int r, int h, int w) { return this->cells_[this->lin(co, r, h, w)]; }
  const T& operator()(int co, int r, int h, int w) const { return this->cells_[this->lin(co, r, h, w)]; }
  T& at(int co, int r, int h, int w) {
    guard(co, r, h, w);
    return (*this)(co, r, h, w);
  }
  const T& at(int co, int r, int h, int w) const {
    guard(co, r, h, w);
    return (*this)(co, r, h, w);
  }

  T* slice(int co, int r) { return this->span_at(this->lin(co, r, 0, 0)); }
  const T* slice(int co, int r) const { return this->span_at(this->lin(co, r, 0, 0)); }

  // orientation r of every channel as a Tensor3 (copy)
  Tensor3<T> orientation(int r) const {
    Tensor3<T> out(out_channels(), height(), width());
    const std::size_t hw = static_cast<std::size_t>(height()) * width();
    for (int co = 0; co < out_channels(); ++co) {
      const T* s = slice(co, r);
      std::copy(s, s + hw, out.plane(co));
    }
    return out;
  }
  bool same_shape(const OrientedFeature& o) const { return this->same_extents(o); }

 private:
  static std::array<int, 4> checked(int co, int r, int h, int w) {
    detail::check(r >= 1, "OrientedFeature: orientations must be >= 1");
    detail::check(co >= 1 && h >= 1 && w >= 1, "OrientedFeature: dimensions must be positive");
    return {co, r, h, w};
  }
  void guard(int co, int r, int h, int w) const {
    if (!this->inside(co, r, h, w)) throw std::out_of_range("OrientedFeature: index out of range");
  }
};

// -------------------------------------------------------------- ArgmaxMap (new, uint8)
// Orientation index of the max-pooled response, in OrientedFeature order (Cout x R' x H x
// W).  orientation_pool_max stores a global index in [0, R); subgroup_pool_max a
// block-local index in [0, group_size).  Ties resolve to the smallest index.
class ArgmaxMap : public detail::Grid<std::uint8_t, 4> {
  using G = detail::Grid<std::uint8_t, 4>;

 public:
  ArgmaxMap() = default;
  ArgmaxMap(int out_channels, int orientations, int height, int width) : G(checked(out_channels, orientations, height, width), 0) {}
  int out_channels() const { return ext_[0]; }
  int orientations() const { return ext_[1]; }
  int height() const { return ext_[2]; }
  int width() const { return ext_[3]; }
  std::uint8_t& operator()(int co, int r, int h, int w) { return cells_[lin(co, r, h, w)]; }
  std::uint8_t operator()(int co, int r, int h, int w) const { return cells_[lin(co, r, h, w)]; }
  std::uint8_t at(int co, int r, int h, int w) const {
    if (!inside(co, r, h, w)) throw std::out_of_range("ArgmaxMap: index out of range");
    return cells_[lin(co, r, h, w)];
  }

 private:
  static std::array<int, 4> checked(int co, int r, int h, int w) {
    detail::check(co >= 1 && r >= 1 && h >= 1 && w >= 1, "ArgmaxMap: dimensions must be positive");
    return {co, r, h, w};
  }
};

// ------------------------------------------------------------ plane transforms (exact)
// Counter-clockwise quarter turns, q reduced mod 4: one turn sends an M x N plane to
// N x M with out(i, j) = in(j, N-1-i) (reference tensor.hpp:345-360).  Index-only.
template <typename T>
MatrixRM<T> rot90_plane(const MatrixRM<T>& plane, int quarter_turns) {
  const int q = ((quarter_turns % 4) + 4) % 4;
  const int R = plane.rows(), C = plane.cols();
  MatrixRM<T> out(q % 2 ? C : R, q % 2 ? R : C);
  for (int i = 0; i < out.rows(); ++i)
    for (int j = 0; j < out.cols(); ++j) {
      // source coordinate of out(i, j) after q CCW turns
      int si = i, sj = j;
      switch (q) {
        case 1: si = j; sj = C - 1 - i; break;
        case 2: si = R - 1 - i; sj = C - 1 - j; break;
        case 3: si = R - 1 - j; sj = i; break;
        default: break;
      }
      out(i, j) = plane(si, sj);
    }
  return out;
}

// Horizontal flip out(i, j) = in(i, N-1-j) (tensor.hpp:362-370).
template <typename T>
MatrixRM<T> mirror_plane(const MatrixRM<T>& plane) {
  MatrixRM<T> out(plane.rows(), plane.cols());
  for (int i = 0; i < plane.rows(); ++i) {
    const T* src = plane.row(i);
    T* dst = out.row(i);
    for (int j = 0, n = plane.cols(); j < n; ++j) dst[j] = src[n - 1 - j];
  }
  return out;
}

// ----------------------------------------------------------------- paper GPU layouts
// CNHW: row = channel, column = (n, h, w) (tensor.hpp:372-390).
template <typename T>
MatrixRM<T> pack_cnhw(std::span<const Tensor3<T>> batch) {
  detail::check(!batch.empty(), "pack_cnhw: empty batch");
  const Tensor3<T>& first = batch.front();
  for (const Tensor3<T>& t : batch)
    detail::check(t.same_shape(first), "pack_cnhw: shape mismatch across the batch");
  const std::size_t hw = static_cast<std::size_t>(first.height()) * first.width();
  MatrixRM<T> m(first.channels(), static_cast<int>(batch.size() * hw));
  for (std::size_t n = 0; n < batch.size(); ++n)
    for (int c = 0; c < first.channels(); ++c)
      std::copy(batch[n].plane(c), batch[n].plane(c) + hw, m.row(c) + n * hw);
  return m;
}

template <typename T>
std::vector<Tensor3<T>> unpack_cnhw(const MatrixRM<T>& m, int channels, int height, int width, int batch) {
  detail::check(m.rows() == channels && m.cols() == batch * height * width,
                "unpack_cnhw: matrix shape does not match requested layout");
  const std::size_t hw = static_cast<std::size_t>(height) * width;
  std::vector<Tensor3<T>> out(batch, Tensor3<T>(channels, height, width));
  for (int n = 0; n < batch; ++n)
    for (int c = 0; c < channels; ++c) {
      const T* src = m.row(c) + n * hw;
      std::copy(src, src + hw, out[n].plane(c));
    }
  return out;
}

// NHWC filters: row = filter, column = (i, j, ci) (tensor.hpp:412-439).
template <typename T>
MatrixRM<T> pack_nhwc(const FilterBank<T>& bank) {
  const int ci_n = bank.in_channels(), taps = bank.kernel_h() * bank.kernel_w();
  MatrixRM<T> m(bank.out_channels(), taps * ci_n);
  for (int co = 0; co < bank.out_channels(); ++co)
    for (int ci = 0; ci < ci_n; ++ci) {
      const T* src = bank.plane(co, ci);
      for (int t = 0; t < taps; ++t) m(co, t * ci_n + ci) = src[t];
    }
  return m;
}

template <typename T>
FilterBank<T> unpack_nhwc(const MatrixRM<T>& m, int out_channels, int in_channels, int kernel_h, int kernel_w) {
  detail::check(m.rows() == out_channels && m.cols() == kernel_h * kernel_w * in_channels,
                "unpack_nhwc: matrix shape does not match requested layout");
  FilterBank<T> bank(out_channels, in_channels, kernel_h, kernel_w);
  const int taps = kernel_h * kernel_w;
  for (int co = 0; co < out_channels; ++co)
    for (int ci = 0; ci < in_channels; ++ci) {
      T* dst = bank.plane(co, ci);
      for (int t = 0; t < taps; ++t) dst[t] = m(co, t * in_channels + ci);
    }
  return bank;
}

}  // namespace rotconv
