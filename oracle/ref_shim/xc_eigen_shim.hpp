// xc_eigen_shim.hpp -- TEST INFRASTRUCTURE ONLY.
//
// A small, eagerly evaluated stand-in for the subset of Eigen (>= 3.4) that
// the reference's headers use (proj/include/xconv/*.hpp, proj/tests/*.cpp).
// Eigen itself is a third-party dependency absent from this container
// (proj/CMakeLists.txt:10 find_package(Eigen3 3.4)), so this shim lets the
// reference's own sources be compiled UNCHANGED from /root/reference into
// oracle/_ref (oracle/Makefile target `ref`): the reference implementation
// then checks the CPU restatement (oracle/xconv_oracle.cpp) and the GPU.
//
// Semantics follow Eigen's documented behaviour where the reference relies on
// it: column-major storage (element (i, j) at i + j * rows()), coefficient-
// wise Array arithmetic, matrix products for Matrix, Zero/Constant factories,
// row/col/corner blocks as assignable views, colwise() reductions, and
// Eigen::FFT with its default kissfft backend (forward unscaled with e^{-},
// inverse e^{+} scaled by 1/n; mixed radix, radix 4 first, then 2, 3, 5, ...).
// Nothing here is copied from Eigen; expressions are evaluated eagerly, which
// changes allocation counts, not arithmetic (every coefficient is computed by
// the same scalar operation).
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstddef>
#include <functional>
#include <initializer_list>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

#ifndef EIGEN_PI
#define EIGEN_PI 3.141592653589793238462643383279502884197169399375105820974944592307816406L
#endif

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };

template <class T>
struct NumTraits {
  using Real = T;
  static T epsilon() { return std::numeric_limits<T>::epsilon(); }
};
template <class T>
struct NumTraits<std::complex<T>> {
  using Real = T;
  static T epsilon() { return std::numeric_limits<T>::epsilon(); }
};

template <class T, int R, int C, bool IsArray>
class Dense;
template <class P>
class Block;

namespace internal {
template <class X>
struct is_dense : std::false_type {};
template <class T, int R, int C, bool A>
struct is_dense<Dense<T, R, C, A>> : std::true_type {};
template <class P>
struct is_dense<Block<P>> : std::true_type {};
template <class X>
constexpr bool is_dense_v = is_dense<std::decay_t<X>>::value;

template <class S>
struct is_scalar : std::is_arithmetic<S> {};
template <class T>
struct is_scalar<std::complex<T>> : std::true_type {};
template <class S>
constexpr bool is_scalar_v = is_scalar<std::decay_t<S>>::value;

template <class T>
T conj_(const T& v) { return v; }
template <class T>
std::complex<T> conj_(const std::complex<T>& v) { return std::conj(v); }
template <class T>
T real_(const T& v) { return v; }
template <class T>
T real_(const std::complex<T>& v) { return v.real(); }
template <class T>
T imag_(const T&) { return T(0); }
template <class T>
T imag_(const std::complex<T>& v) { return v.imag(); }
template <class T>
T abs2_(const T& v) { return v * v; }
template <class T>
T abs2_(const std::complex<T>& v) { return std::norm(v); }
template <class T>
bool isfinite_(const T& v) { return std::isfinite(v); }
template <class T>
bool isfinite_(const std::complex<T>& v) { return std::isfinite(v.real()) && std::isfinite(v.imag()); }

template <class T>
struct real_of { using type = T; };
template <class T>
struct real_of<std::complex<T>> { using type = T; };
}  // namespace internal

// Heap buffer with value semantics (std::vector<bool> would not give bool&).
template <class T>
class Buf {
 public:
  Buf() = default;
  Buf(std::initializer_list<T> l) : n_(l.size()), p_(new T[l.size()]) { std::copy(l.begin(), l.end(), p_.get()); }
  Buf(const Buf& o) : n_(o.n_), p_(o.n_ ? new T[o.n_] : nullptr) { std::copy(o.begin(), o.end(), begin()); }
  Buf(Buf&&) noexcept = default;
  Buf& operator=(const Buf& o) {
    if (this != &o) {
      Buf t(o);
      *this = std::move(t);
    }
    return *this;
  }
  Buf& operator=(Buf&&) noexcept = default;
  void assign(size_t n, const T& v) {
    if (n != n_) {
      p_.reset(n ? new T[n] : nullptr);
      n_ = n;
    }
    std::fill(begin(), end(), v);
  }
  void resize(size_t n) {
    if (n == n_) return;
    std::unique_ptr<T[]> q(n ? new T[n]() : nullptr);
    std::copy(begin(), begin() + std::min(n, n_), q.get());
    p_ = std::move(q);
    n_ = n;
  }
  size_t size() const { return n_; }
  T* data() { return p_.get(); }
  const T* data() const { return p_.get(); }
  T* begin() { return p_.get(); }
  T* end() { return p_.get() + n_; }
  const T* begin() const { return p_.get(); }
  const T* end() const { return p_.get() + n_; }
  T& operator[](size_t i) { return p_[i]; }
  const T& operator[](size_t i) const { return p_[i]; }

 private:
  size_t n_ = 0;
  std::unique_ptr<T[]> p_;
};

struct ShapeTag {};  // (rows, cols) construction regardless of fixed-size shapes

// Dense storage: rows x cols, column-major; R / C are compile-time extents
// (Dynamic = -1) used only for typing, sizing defaults and fixed-size ctors.
template <class T, int R, int C, bool IsArray>
class Dense {
 public:
  using Scalar = T;
  using value_type = T;
  using RealScalar = typename internal::real_of<T>::type;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr bool IsArrayKind = IsArray;
  static constexpr bool IsVectorAtCompileTime = R == 1 || C == 1;

  Dense() : r_(R > 0 ? R : (C == 1 || R == 1 ? 0 : 0)), c_(C > 0 ? C : 0) {
    if (R == 1 && C == Dynamic) r_ = 1;
    if (C == 1 && R == Dynamic) c_ = 1;
    d_.assign(size_t(r_ * c_), T());
  }
  // one argument: a size (vectors), or a copy from another dense object
  template <class A0, std::enable_if_t<std::is_integral<A0>::value, int> = 0>
  explicit Dense(A0 n) {
    if (C == 1 || (R != 1 && C != 1 && R == Dynamic && C == Dynamic)) {
      r_ = Index(n);
      c_ = 1;
    } else {
      r_ = 1;
      c_ = Index(n);
    }
    d_.assign(size_t(r_ * c_), T());
  }
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Dense(const O& o) {  // NOLINT: implicit like Eigen's expression conversion
    assign_from(o);
  }
  // two arguments: (rows, cols) for dynamic shapes, coefficients for a fixed 2-vector
  template <class A0, class A1>
  Dense(const A0& a, const A1& b) {
    if constexpr (R > 0 && C > 0 && R * C == 2) {
      r_ = R;
      c_ = C;
      d_ = {T(a), T(b)};
    } else {
      r_ = Index(a);
      c_ = Index(b);
      d_.assign(size_t(r_ * c_), T());
    }
  }
  template <class A0, class A1, class A2,
            std::enable_if_t<!std::is_same<std::decay_t<A0>, ShapeTag>::value, int> = 0>
  Dense(const A0& a, const A1& b, const A2& c) : r_(R), c_(C), d_{T(a), T(b), T(c)} {
    static_assert(R * C == 3, "three coefficients need a fixed 3-vector");
  }
  template <class A0, class A1, class A2, class A3>
  Dense(const A0& a, const A1& b, const A2& c, const A3& e) : r_(R), c_(C), d_{T(a), T(b), T(c), T(e)} {
    static_assert(R * C == 4, "four coefficients need a fixed 4-vector");
  }
  Dense(ShapeTag, Index r, Index c) : r_(r), c_(c) { d_.assign(size_t(r * c), T()); }
  Dense(const Dense&) = default;
  Dense(Dense&&) noexcept = default;
  Dense& operator=(const Dense&) = default;
  Dense& operator=(Dense&&) noexcept = default;
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Dense& operator=(const O& o) {
    Dense tmp;
    tmp.assign_from(o);
    *this = std::move(tmp);
    return *this;
  }

  template <class O>
  void assign_from(const O& o) {
    r_ = o.rows();
    c_ = o.cols();
    // a vector assigned to a vector of the other orientation keeps its length
    if ((R == 1 && r_ != 1 && c_ == 1) || (C == 1 && c_ != 1 && r_ == 1)) std::swap(r_, c_);
    d_.resize(size_t(r_ * c_));
    if (r_ == o.rows()) {
      for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) d_[size_t(i + j * r_)] = T(o(i, j));
    } else {
      for (Index i = 0; i < size(); ++i) d_[size_t(i)] = T(o(i % o.rows(), i / o.rows()));
    }
  }

  // ---- shape and access
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  T* data() { return d_.data(); }
  const T* data() const { return d_.data(); }
  T& operator()(Index i, Index j) { return d_[size_t(i + j * r_)]; }
  const T& operator()(Index i, Index j) const { return d_[size_t(i + j * r_)]; }
  T& operator()(Index i) { return d_[size_t(i)]; }
  const T& operator()(Index i) const { return d_[size_t(i)]; }
  T& operator[](Index i) { return d_[size_t(i)]; }
  const T& operator[](Index i) const { return d_[size_t(i)]; }
  T coeff(Index i, Index j) const { return (*this)(i, j); }
  T& coeffRef(Index i, Index j) { return (*this)(i, j); }
  T x() const { return d_[0]; }
  T y() const { return d_[1]; }
  T z() const { return d_[2]; }
  T& x() { return d_[0]; }
  T& y() { return d_[1]; }
  T& z() { return d_[2]; }

  void resize(Index r, Index c) {
    if (r * c != size()) d_.assign(size_t(r * c), T());
    r_ = r;
    c_ = c;
  }
  void resize(Index n) {
    if (C == 1 || (R != 1)) {
      r_ = n;
      c_ = 1;
    } else {
      r_ = 1;
      c_ = n;
    }
    d_.assign(size_t(n), T());
  }
  Dense& setZero() {
    std::fill(d_.begin(), d_.end(), T(0));
    return *this;
  }
  Dense& setZero(Index r, Index c) {
    resize(r, c);
    return *this;
  }
  Dense& setOnes() { return setConstant(T(1)); }
  Dense& setConstant(const T& v) {
    std::fill(d_.begin(), d_.end(), v);
    return *this;
  }
  Dense& fill(const T& v) { return setConstant(v); }

  // ---- factories
  static Dense Zero() { return Dense(); }
  static Dense Zero(Index n) { return Dense(n); }
  static Dense Zero(Index r, Index c) { return Dense(ShapeTag{}, r, c); }
  static Dense Constant(Index r, Index c, const T& v) { return Dense(ShapeTag{}, r, c).setConstant(v); }
  static Dense Constant(Index n, const T& v) { return Dense(n).setConstant(v); }
  static Dense Constant(const T& v) { return Dense().setConstant(v); }
  static Dense Ones(Index r, Index c) { return Constant(r, c, T(1)); }
  static Dense Ones(Index n) { return Constant(n, T(1)); }
  static Dense Ones() { return Constant(T(1)); }
  static Dense Identity(Index r, Index c) {
    Dense m(ShapeTag{}, r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = T(1);
    return m;
  }
  static Dense Identity() { return Identity(R, C); }
  static Dense Unit(Index n, Index i) {
    Dense v(ShapeTag{}, C == 1 ? n : 1, C == 1 ? 1 : n);
    v.d_[size_t(i)] = T(1);
    return v;
  }
  static Dense UnitX() { return Unit(R * C, 0); }
  static Dense UnitY() { return Unit(R * C, 1); }
  static Dense UnitZ() { return Unit(R * C, 2); }

  // ---- coefficient-wise maps
  template <class F>
  auto unaryExpr(F f) const {
    using U = std::decay_t<decltype(f(std::declval<T>()))>;
    Dense<U, R, C, IsArray> o(ShapeTag{}, r_, c_);
    for (Index i = 0; i < size(); ++i) o.data()[i] = f(d_[size_t(i)]);
    return o;
  }
  auto real() const { return unaryExpr([](const T& v) { return internal::real_(v); }); }
  auto imag() const { return unaryExpr([](const T& v) { return internal::imag_(v); }); }
  auto abs() const { return unaryExpr([](const T& v) { return RealScalar(std::abs(v)); }); }
  auto abs2() const { return unaryExpr([](const T& v) { return internal::abs2_(v); }); }
  auto cwiseAbs() const { return abs(); }
  auto cwiseAbs2() const { return abs2(); }
  Dense conjugate() const { return unaryExpr([](const T& v) { return internal::conj_(v); }); }
  Dense log() const { return unaryExpr([](const T& v) { return T(std::log(v)); }); }
  Dense exp() const { return unaryExpr([](const T& v) { return T(std::exp(v)); }); }
  Dense sqrt() const { return unaryExpr([](const T& v) { return T(std::sqrt(v)); }); }
  Dense cwiseSqrt() const { return sqrt(); }
  Dense cos() const { return unaryExpr([](const T& v) { return T(std::cos(v)); }); }
  Dense sin() const { return unaryExpr([](const T& v) { return T(std::sin(v)); }); }
  Dense square() const { return unaryExpr([](const T& v) { return T(v * v); }); }
  Dense inverse() const {
    if constexpr (IsArray) {
      return unaryExpr([](const T& v) { return T(T(1) / v); });
    } else {
      return matrix_inverse();
    }
  }
  auto isFinite() const { return unaryExpr([](const T& v) { return internal::isfinite_(v); }); }
  template <class U>
  Dense<U, R, C, IsArray> cast() const {
    Dense<U, R, C, IsArray> o(ShapeTag{}, r_, c_);
    for (Index i = 0; i < size(); ++i) o.data()[i] = U(d_[size_t(i)]);
    return o;
  }
  Dense<T, R, C, false> matrix() const { return Dense<T, R, C, false>(*this); }
  Dense<T, R, C, true> array() const { return Dense<T, R, C, true>(*this); }
  Dense<T, C, R, IsArray> transpose() const {
    Dense<T, C, R, IsArray> o(ShapeTag{}, c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(j, i) = (*this)(i, j);
    return o;
  }
  Dense<T, C, R, IsArray> adjoint() const { return transpose().conjugate(); }

  // ---- reductions
  T sum() const {
    T s(0);
    for (const T& v : d_) s += v;
    return s;
  }
  T prod() const {
    T s(1);
    for (const T& v : d_) s *= v;
    return s;
  }
  T mean() const { return sum() / T(RealScalar(size())); }
  T maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
  T minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
  template <class I>
  T maxCoeff(I* idx) const {
    const auto it = std::max_element(d_.begin(), d_.end());
    *idx = I(it - d_.begin());
    return *it;
  }
  template <class I>
  T maxCoeff(I* ri, I* ci) const {
    const Index k = std::max_element(d_.begin(), d_.end()) - d_.begin();
    *ri = I(k % r_);
    *ci = I(k / r_);
    return d_[size_t(k)];
  }
  template <class I>
  T minCoeff(I* ri, I* ci) const {
    const Index k = std::min_element(d_.begin(), d_.end()) - d_.begin();
    *ri = I(k % r_);
    *ci = I(k / r_);
    return d_[size_t(k)];
  }
  bool all() const {
    for (const T& v : d_)
      if (!v) return false;
    return true;
  }
  bool any() const {
    for (const T& v : d_)
      if (v) return true;
    return false;
  }
  Index count() const {
    Index n = 0;
    for (const T& v : d_) n += v ? 1 : 0;
    return n;
  }
  RealScalar squaredNorm() const {
    RealScalar s(0);
    for (const T& v : d_) s += internal::abs2_(v);
    return s;
  }
  RealScalar norm() const { return std::sqrt(squaredNorm()); }
  void normalize() {
    const RealScalar n = norm();
    if (n > 0)
      for (T& v : d_) v /= n;
  }
  Dense normalized() const {
    Dense o(*this);
    o.normalize();
    return o;
  }
  template <class O>
  T dot(const O& o) const {  // conjugate-linear in the first argument, like Eigen
    T s(0);
    for (Index i = 0; i < size(); ++i) s += internal::conj_(d_[size_t(i)]) * T(o(i % o.rows(), i / o.rows()));
    return s;
  }
  T trace() const {
    T s(0);
    for (Index i = 0; i < std::min(r_, c_); ++i) s += (*this)(i, i);
    return s;
  }

  // ---- views
  Block<Dense> block(Index i, Index j, Index h, Index w) { return Block<Dense>(this, i, j, h, w); }
  Block<const Dense> block(Index i, Index j, Index h, Index w) const {
    return Block<const Dense>(this, i, j, h, w);
  }
  Block<Dense> row(Index i) { return block(i, 0, 1, c_); }
  Block<const Dense> row(Index i) const { return block(i, 0, 1, c_); }
  Block<Dense> col(Index j) { return block(0, j, r_, 1); }
  Block<const Dense> col(Index j) const { return block(0, j, r_, 1); }
  Block<Dense> topLeftCorner(Index h, Index w) { return block(0, 0, h, w); }
  Block<const Dense> topLeftCorner(Index h, Index w) const { return block(0, 0, h, w); }
  Block<Dense> bottomRightCorner(Index h, Index w) { return block(r_ - h, c_ - w, h, w); }
  Block<const Dense> bottomRightCorner(Index h, Index w) const { return block(r_ - h, c_ - w, h, w); }
  Block<Dense> topRows(Index h) { return block(0, 0, h, c_); }
  Block<Dense> leftCols(Index w) { return block(0, 0, r_, w); }
  Block<Dense> segment(Index i, Index n) { return C == 1 || c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n); }
  Block<const Dense> segment(Index i, Index n) const {
    return C == 1 || c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n);
  }
  Block<Dense> head(Index n) { return segment(0, n); }
  Block<const Dense> head(Index n) const { return segment(0, n); }
  Block<Dense> tail(Index n) { return segment(size() - n, n); }
  Block<const Dense> tail(Index n) const { return segment(size() - n, n); }

  struct Vectorwise {  // colwise() / rowwise() reductions
    const Dense* m;
    bool cols;
    template <class F>
    auto reduce(F f) const {
      using U = std::decay_t<decltype(f(std::declval<Dense<T, Dynamic, 1, IsArray>>()))>;
      if (cols) {
        Dense<U, 1, Dynamic, IsArray> o(ShapeTag{}, 1, m->cols());
        for (Index j = 0; j < m->cols(); ++j) o(0, j) = f(Dense<T, Dynamic, 1, IsArray>(m->col(j)));
        return Dense<U, Dynamic, Dynamic, IsArray>(o);
      }
      Dense<U, Dynamic, 1, IsArray> o(ShapeTag{}, m->rows(), 1);
      for (Index i = 0; i < m->rows(); ++i)
        o(i, 0) = f(Dense<T, Dynamic, 1, IsArray>(m->row(i).transpose()));
      return Dense<U, Dynamic, Dynamic, IsArray>(o);
    }
    auto sum() const { return reduce([](const auto& v) { return v.sum(); }); }
    auto mean() const { return reduce([](const auto& v) { return v.mean(); }); }
    auto maxCoeff() const { return reduce([](const auto& v) { return v.maxCoeff(); }); }
    auto minCoeff() const { return reduce([](const auto& v) { return v.minCoeff(); }); }
    auto norm() const { return reduce([](const auto& v) { return v.norm(); }); }
    auto squaredNorm() const { return reduce([](const auto& v) { return v.squaredNorm(); }); }
  };
  Vectorwise colwise() const { return Vectorwise{this, true}; }
  Vectorwise rowwise() const { return Vectorwise{this, false}; }

  // ---- compound assignment
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Dense& operator+=(const O& o) {
    check_same(o);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) += o(i, j);
    return *this;
  }
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Dense& operator-=(const O& o) {
    check_same(o);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) -= o(i, j);
    return *this;
  }
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Dense& operator*=(const O& o) {
    if constexpr (IsArray) {
      check_same(o);
      for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) (*this)(i, j) *= o(i, j);
    } else {
      *this = (*this) * o;
    }
    return *this;
  }
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Dense& operator/=(const O& o) {
    check_same(o);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) /= o(i, j);
    return *this;
  }
  template <class S, std::enable_if_t<internal::is_scalar_v<S>, int> = 0>
  Dense& operator*=(const S& s) {
    for (T& v : d_) v *= s;
    return *this;
  }
  template <class S, std::enable_if_t<internal::is_scalar_v<S>, int> = 0>
  Dense& operator/=(const S& s) {
    for (T& v : d_) v /= s;
    return *this;
  }
  template <class S, std::enable_if_t<internal::is_scalar_v<S>, int> = 0>
  Dense& operator+=(const S& s) {
    for (T& v : d_) v += s;
    return *this;
  }
  template <class S, std::enable_if_t<internal::is_scalar_v<S>, int> = 0>
  Dense& operator-=(const S& s) {
    for (T& v : d_) v -= s;
    return *this;
  }
  Dense operator-() const { return unaryExpr([](const T& v) { return T(-v); }); }

  // ---- linear solve (FullPivLU, used by sph.hpp quadrature weights)
  struct FullPivLU {
    Dense<T, Dynamic, Dynamic, false> a;
    template <class B>
    Dense<T, Dynamic, 1, false> solve(const B& b_in) const {
      const Index n = a.rows();
      Dense<T, Dynamic, Dynamic, false> m(a);
      Dense<T, Dynamic, 1, false> b(b_in);
      std::vector<Index> colperm(static_cast<size_t>(n));
      for (Index i = 0; i < n; ++i) colperm[size_t(i)] = i;
      for (Index k = 0; k < n; ++k) {
        Index pr = k, pc = k;
        RealScalar best = -1;
        for (Index j = k; j < n; ++j)
          for (Index i = k; i < n; ++i)
            if (std::abs(m(i, j)) > best) {
              best = std::abs(m(i, j));
              pr = i;
              pc = j;
            }
        for (Index j = 0; j < n; ++j) std::swap(m(k, j), m(pr, j));
        std::swap(b(k), b(pr));
        for (Index i = 0; i < n; ++i) std::swap(m(i, k), m(i, pc));
        std::swap(colperm[size_t(k)], colperm[size_t(pc)]);
        if (m(k, k) == T(0)) continue;
        for (Index i = k + 1; i < n; ++i) {
          const T f = m(i, k) / m(k, k);
          for (Index j = k; j < n; ++j) m(i, j) -= f * m(k, j);
          b(i) -= f * b(k);
        }
      }
      Dense<T, Dynamic, 1, false> y(n);
      for (Index i = n - 1; i >= 0; --i) {
        T s = b(i);
        for (Index j = i + 1; j < n; ++j) s -= m(i, j) * y(j);
        y(i) = m(i, i) == T(0) ? T(0) : s / m(i, i);
      }
      Dense<T, Dynamic, 1, false> x(n);
      for (Index i = 0; i < n; ++i) x(colperm[size_t(i)]) = y(i);
      return x;
    }
  };
  FullPivLU fullPivLu() const { return FullPivLU{Dense<T, Dynamic, Dynamic, false>(*this)}; }

 private:
  template <class O>
  void check_same(const O& o) const {
    if (o.rows() != r_ || o.cols() != c_) throw std::logic_error("eigen shim: size mismatch");
  }
  Dense matrix_inverse() const {
    const Index n = r_;
    Dense<T, Dynamic, Dynamic, false> I = Dense<T, Dynamic, Dynamic, false>::Identity(n, n);
    Dense out(ShapeTag{}, n, n);
    for (Index j = 0; j < n; ++j) {
      auto x = fullPivLu().solve(I.col(j));
      for (Index i = 0; i < n; ++i) out(i, j) = x(i);
    }
    return out;
  }

  Index r_ = 0, c_ = 0;
  Buf<T> d_;
};

// An assignable rectangular view into a Dense (row, col, corners, segments).
template <class P>
class Block {
 public:
  using Parent = std::remove_const_t<P>;
  using Scalar = typename Parent::Scalar;
  using value_type = Scalar;
  static constexpr bool IsArrayKind = Parent::IsArrayKind;
  using Eval = Dense<Scalar, Dynamic, Dynamic, IsArrayKind>;

  Block(P* p, Index i, Index j, Index h, Index w) : p_(p), i_(i), j_(j), h_(h), w_(w) {}
  Index rows() const { return h_; }
  Index cols() const { return w_; }
  Index size() const { return h_ * w_; }
  decltype(auto) operator()(Index i, Index j) const { return (*p_)(i_ + i, j_ + j); }
  decltype(auto) operator()(Index k) const { return h_ == 1 ? (*p_)(i_, j_ + k) : (*p_)(i_ + k, j_); }
  decltype(auto) operator[](Index k) const { return (*this)(k); }
  Eval eval() const { return Eval(*this); }

  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Block& operator=(const O& o) {
    return assign_eval(Eval(o));  // evaluate first: the source may alias the parent
  }
  Block& operator=(const Block& o) { return assign_eval(Eval(o)); }
  Block& assign_eval(const Eval& v) {
    if (v.size() != size()) throw std::logic_error("eigen shim: block size mismatch");
    if (v.rows() == h_) {
      for (Index j = 0; j < w_; ++j)
        for (Index i = 0; i < h_; ++i) (*p_)(i_ + i, j_ + j) = v(i, j);
    } else {  // vector of the other orientation
      for (Index k = 0; k < size(); ++k) (*this)(k) = v(k);
    }
    return *this;
  }
  template <class S, std::enable_if_t<internal::is_scalar_v<S>, int> = 0>
  Block& setConstant(const S& s) {
    for (Index j = 0; j < w_; ++j)
      for (Index i = 0; i < h_; ++i) (*p_)(i_ + i, j_ + j) = s;
    return *this;
  }
  Block& setZero() { return setConstant(Scalar(0)); }
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Block& operator+=(const O& o) {
    const Eval v(o);
    for (Index j = 0; j < w_; ++j)
      for (Index i = 0; i < h_; ++i) (*p_)(i_ + i, j_ + j) += v(i, j);
    return *this;
  }
  template <class O, std::enable_if_t<internal::is_dense_v<O>, int> = 0>
  Block& operator-=(const O& o) {
    const Eval v(o);
    for (Index j = 0; j < w_; ++j)
      for (Index i = 0; i < h_; ++i) (*p_)(i_ + i, j_ + j) -= v(i, j);
    return *this;
  }
  template <class S, std::enable_if_t<internal::is_scalar_v<S>, int> = 0>
  Block& operator*=(const S& s) {
    for (Index j = 0; j < w_; ++j)
      for (Index i = 0; i < h_; ++i) (*p_)(i_ + i, j_ + j) *= s;
    return *this;
  }

  // everything else evaluates the view first
  auto matrix() const { return eval().matrix(); }
  auto array() const { return eval().array(); }
  auto transpose() const { return eval().transpose(); }
  auto adjoint() const { return eval().adjoint(); }
  auto real() const { return eval().real(); }
  auto imag() const { return eval().imag(); }
  auto abs() const { return eval().abs(); }
  auto abs2() const { return eval().abs2(); }
  auto conjugate() const { return eval().conjugate(); }
  auto square() const { return eval().square(); }
  template <class F>
  auto unaryExpr(F f) const { return eval().unaryExpr(f); }
  template <class U>
  auto cast() const { return eval().template cast<U>(); }
  auto sum() const { return eval().sum(); }
  auto mean() const { return eval().mean(); }
  auto maxCoeff() const { return eval().maxCoeff(); }
  auto minCoeff() const { return eval().minCoeff(); }
  auto norm() const { return eval().norm(); }
  auto squaredNorm() const { return eval().squaredNorm(); }
  bool all() const { return eval().all(); }
  bool any() const { return eval().any(); }
  auto normalized() const { return eval().normalized(); }
  template <class O>
  auto dot(const O& o) const { return eval().dot(o); }
  auto colwise() const { return eval_keep().colwise(); }

 private:
  const Eval& eval_keep() const {
    keep_ = std::make_shared<Eval>(*this);
    return *keep_;
  }
  P* p_;
  Index i_, j_, h_, w_;
  mutable std::shared_ptr<Eval> keep_;
};

namespace internal {
template <class X>
struct dense_of {
  using type = X;
};
template <class P>
struct dense_of<Block<P>> {
  using type = typename Block<P>::Eval;
};
template <class X>
using dense_of_t = typename dense_of<std::decay_t<X>>::type;

template <class X>
const dense_of_t<X>& as_dense(const X& x, dense_of_t<X>& tmp) {
  if constexpr (std::is_same<std::decay_t<X>, dense_of_t<X>>::value) {
    (void)tmp;
    return x;
  } else {
    tmp = dense_of_t<X>(x);
    return tmp;
  }
}

template <class A, class B, class F>
auto zip(const A& a_in, const B& b_in, F f) {
  dense_of_t<A> ta;
  dense_of_t<B> tb;
  const auto& a = as_dense(a_in, ta);
  const auto& b = as_dense(b_in, tb);
  using DA = std::decay_t<decltype(a)>;
  using U = std::decay_t<decltype(f(a(0, 0), b(0, 0)))>;
  if (a.rows() != b.rows() || a.cols() != b.cols())
    throw std::logic_error("eigen shim: size mismatch");
  Dense<U, DA::RowsAtCompileTime, DA::ColsAtCompileTime, DA::IsArrayKind> o(ShapeTag{}, a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) o(i, j) = f(a(i, j), b(i, j));
  return o;
}
template <class A, class S, class F>
auto map_scalar(const A& a_in, const S& s, F f) {
  dense_of_t<A> ta;
  const auto& a = as_dense(a_in, ta);
  using DA = std::decay_t<decltype(a)>;
  using U = std::decay_t<decltype(f(a(0, 0), s))>;
  Dense<U, DA::RowsAtCompileTime, DA::ColsAtCompileTime, DA::IsArrayKind> o(ShapeTag{}, a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) o(i, j) = f(a(i, j), s);
  return o;
}
}  // namespace internal

#define XC_SHIM_EWISE(OP)                                                                        \
  template <class A, class B,                                                                    \
            std::enable_if_t<internal::is_dense_v<A> && internal::is_dense_v<B>, int> = 0>       \
  auto operator OP(const A& a, const B& b) {                                                     \
    return internal::zip(a, b, [](const auto& x, const auto& y) { return x OP y; });            \
  }                                                                                              \
  template <class A, class S,                                                                    \
            std::enable_if_t<internal::is_dense_v<A> && internal::is_scalar_v<S>, int> = 0>      \
  auto operator OP(const A& a, const S& s) {                                                     \
    return internal::map_scalar(a, s, [](const auto& x, const auto& y) { return x OP y; });     \
  }                                                                                              \
  template <class S, class A,                                                                    \
            std::enable_if_t<internal::is_dense_v<A> && internal::is_scalar_v<S>, int> = 0>      \
  auto operator OP(const S& s, const A& a) {                                                     \
    return internal::map_scalar(a, s, [](const auto& x, const auto& y) { return y OP x; });     \
  }
XC_SHIM_EWISE(+)
XC_SHIM_EWISE(-)
XC_SHIM_EWISE(/)
XC_SHIM_EWISE(==)
XC_SHIM_EWISE(!=)
XC_SHIM_EWISE(<)
XC_SHIM_EWISE(<=)
XC_SHIM_EWISE(>)
XC_SHIM_EWISE(>=)
#undef XC_SHIM_EWISE

// '*': coefficient-wise for arrays, the matrix product for matrices
template <class A, class B,
          std::enable_if_t<internal::is_dense_v<A> && internal::is_dense_v<B>, int> = 0>
auto operator*(const A& a_in, const B& b_in) {
  if constexpr (std::decay_t<A>::IsArrayKind) {
    return internal::zip(a_in, b_in, [](const auto& x, const auto& y) { return x * y; });
  } else {
    internal::dense_of_t<A> ta;
    internal::dense_of_t<B> tb;
    const auto& a = internal::as_dense(a_in, ta);
    const auto& b = internal::as_dense(b_in, tb);
    using TA = typename std::decay_t<decltype(a)>::Scalar;
    using TB = typename std::decay_t<decltype(b)>::Scalar;
    using U = std::decay_t<decltype(std::declval<TA>() * std::declval<TB>())>;
    using DA = std::decay_t<decltype(a)>;
    using DB = std::decay_t<decltype(b)>;
    if (a.cols() != b.rows()) throw std::logic_error("eigen shim: product size mismatch");
    Dense<U, DA::RowsAtCompileTime, DB::ColsAtCompileTime, false> o(ShapeTag{}, a.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
      for (Index i = 0; i < a.rows(); ++i) {
        U s(0);
        for (Index k = 0; k < a.cols(); ++k) s += a(i, k) * b(k, j);
        o(i, j) = s;
      }
    return o;
  }
}
template <class A, class S,
          std::enable_if_t<internal::is_dense_v<A> && internal::is_scalar_v<S>, int> = 0>
auto operator*(const A& a, const S& s) {
  return internal::map_scalar(a, s, [](const auto& x, const auto& y) { return x * y; });
}
template <class S, class A,
          std::enable_if_t<internal::is_dense_v<A> && internal::is_scalar_v<S>, int> = 0>
auto operator*(const S& s, const A& a) {
  return internal::map_scalar(a, s, [](const auto& x, const auto& y) { return y * x; });
}

template <class T, int R, int C, int O = 0, int MR = R, int MC = C>
using Array = Dense<T, R, C, true>;
template <class T, int R, int C, int O = 0, int MR = R, int MC = C>
using Matrix = Dense<T, R, C, false>;

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using MatrixXcd = Matrix<std::complex<double>, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Matrix3d = Matrix<double, 3, 3>;
using ArrayXd = Array<double, Dynamic, 1>;
using ArrayXXd = Array<double, Dynamic, Dynamic>;
using ArrayXXcd = Array<std::complex<double>, Dynamic, Dynamic>;

// ---------------------------------------------------------------- rotations
template <class T>
class Quaternion {
 public:
  using Scalar = T;
  Quaternion() : w_(1), x_(0), y_(0), z_(0) {}
  Quaternion(T w, T x, T y, T z) : w_(w), x_(x), y_(y), z_(z) {}
  template <class AA, std::enable_if_t<!std::is_arithmetic<AA>::value, int> = 0>
  explicit Quaternion(const AA& aa) {  // from an angle-axis rotation
    const T h = T(0.5) * aa.angle();
    const auto ax = aa.axis();
    w_ = std::cos(h);
    x_ = std::sin(h) * ax(0);
    y_ = std::sin(h) * ax(1);
    z_ = std::sin(h) * ax(2);
  }
  static Quaternion Identity() { return Quaternion(); }
  T& w() { return w_; }
  T& x() { return x_; }
  T& y() { return y_; }
  T& z() { return z_; }
  T w() const { return w_; }
  T x() const { return x_; }
  T y() const { return y_; }
  T z() const { return z_; }
  T squaredNorm() const { return w_ * w_ + x_ * x_ + y_ * y_ + z_ * z_; }
  T norm() const { return std::sqrt(squaredNorm()); }
  void normalize() {
    const T n = norm();
    w_ /= n;
    x_ /= n;
    y_ /= n;
    z_ /= n;
  }
  Quaternion normalized() const {
    Quaternion q(*this);
    q.normalize();
    return q;
  }
  Quaternion conjugate() const { return Quaternion(w_, -x_, -y_, -z_); }
  // rotation angle between two unit quaternions: 2 atan2(|vec(a^-1 b)|, |w(a^-1 b)|)
  T angularDistance(const Quaternion& o) const {
    const Quaternion d = conjugate() * o;
    return T(2) * std::atan2(std::sqrt(d.x_ * d.x_ + d.y_ * d.y_ + d.z_ * d.z_), std::abs(d.w_));
  }
  Quaternion inverse() const {
    const T n2 = squaredNorm();
    return Quaternion(w_ / n2, -x_ / n2, -y_ / n2, -z_ / n2);
  }
  Quaternion operator*(const Quaternion& b) const {
    return Quaternion(w_ * b.w_ - x_ * b.x_ - y_ * b.y_ - z_ * b.z_,
                      w_ * b.x_ + x_ * b.w_ + y_ * b.z_ - z_ * b.y_,
                      w_ * b.y_ - x_ * b.z_ + y_ * b.w_ + z_ * b.x_,
                      w_ * b.z_ + x_ * b.y_ - y_ * b.x_ + z_ * b.w_);
  }
  Matrix<T, 3, 3> toRotationMatrix() const {
    const T tx = 2 * x_, ty = 2 * y_, tz = 2 * z_;
    const T twx = tx * w_, twy = ty * w_, twz = tz * w_;
    const T txx = tx * x_, txy = ty * x_, txz = tz * x_;
    const T tyy = ty * y_, tyz = tz * y_, tzz = tz * z_;
    Matrix<T, 3, 3> m;
    m(0, 0) = T(1) - (tyy + tzz);
    m(0, 1) = txy - twz;
    m(0, 2) = txz + twy;
    m(1, 0) = txy + twz;
    m(1, 1) = T(1) - (txx + tzz);
    m(1, 2) = tyz - twx;
    m(2, 0) = txz - twy;
    m(2, 1) = tyz + twx;
    m(2, 2) = T(1) - (txx + tyy);
    return m;
  }
  template <class V, std::enable_if_t<internal::is_dense_v<V>, int> = 0>
  Matrix<T, 3, 1> operator*(const V& v) const {
    return Matrix<T, 3, 1>(toRotationMatrix() * Matrix<T, 3, 1>(v));
  }

 private:
  T w_, x_, y_, z_;
};
using Quaterniond = Quaternion<double>;

template <class T>
class AngleAxis {
 public:
  AngleAxis(T angle, const Matrix<T, 3, 1>& axis) : a_(angle), ax_(axis) {}
  T angle() const { return a_; }
  const Matrix<T, 3, 1>& axis() const { return ax_; }
  Matrix<T, 3, 3> toRotationMatrix() const { return Quaternion<T>(*this).toRotationMatrix(); }

 private:
  T a_;
  Matrix<T, 3, 1> ax_;
};
using AngleAxisd = AngleAxis<double>;

// ---------------------------------------------------------------- FFT
// Eigen::FFT with the default kissfft backend: recursive mixed-radix
// decimation in time, factors taken as 4 first, then 2, 3, 5, 7, ...;
// forward e^{-2 pi i jk/n} unscaled, inverse e^{+} scaled by 1/n.
template <class T>
class FFT {
 public:
  using Complex = std::complex<T>;

  void fwd(std::vector<Complex>& dst, const std::vector<Complex>& src) {
    dst.resize(src.size());
    transform(dst.data(), src.data(), int(src.size()), false);
  }
  void inv(std::vector<Complex>& dst, const std::vector<Complex>& src) {
    dst.resize(src.size());
    transform(dst.data(), src.data(), int(src.size()), true);
  }
  template <class D, class S, std::enable_if_t<internal::is_dense_v<S>, int> = 0>
  void fwd(D& dst, const S& src) {
    const Dense<Complex, Dynamic, 1, false> s(src);
    dst.resize(s.size());
    transform(dst.data(), s.data(), int(s.size()), false);
  }
  template <class D, class S, std::enable_if_t<internal::is_dense_v<S>, int> = 0>
  void inv(D& dst, const S& src) {
    const Dense<Complex, Dynamic, 1, false> s(src);
    dst.resize(s.size());
    transform(dst.data(), s.data(), int(s.size()), true);
  }

 private:
  struct Plan {
    int n = 0;
    std::vector<int> radix, remain;
    std::vector<Complex> tw[2];
  };

  const Plan& plan(int n) {
    auto it = plans_.find(n);
    if (it != plans_.end()) return it->second;
    Plan p;
    p.n = n;
    for (int inv = 0; inv < 2; ++inv) {
      p.tw[inv].resize(size_t(n));
      for (int i = 0; i < n; ++i) {
        const T ph = (inv ? T(2) : T(-2)) * T(EIGEN_PI) * T(i) / T(n);
        p.tw[inv][size_t(i)] = Complex(std::cos(ph), std::sin(ph));
      }
    }
    int m = n, f = 4;
    do {
      while (m % f) {
        if (f == 4)
          f = 2;
        else if (f == 2)
          f = 3;
        else
          f += 2;
        if (f * f > m) f = m;
      }
      m /= f;
      p.radix.push_back(f);
      p.remain.push_back(m);
    } while (m > 1);
    return plans_.emplace(n, std::move(p)).first->second;
  }

  static void butterfly(const Plan& pl, bool inv, Complex* F, size_t fs, int P, int m) {
    const Complex* tw = pl.tw[inv].data();
    if (P == 2) {
      for (int k = 0; k < m; ++k) {
        const Complex t = F[m + k] * tw[size_t(k) * fs];
        F[m + k] = F[k] - t;
        F[k] += t;
      }
    } else if (P == 4) {
      for (int k = 0; k < m; ++k) {
        const Complex s0 = F[k + m] * tw[size_t(k) * fs];
        const Complex s1 = F[k + 2 * m] * tw[size_t(2 * k) * fs];
        const Complex s2 = F[k + 3 * m] * tw[size_t(3 * k) * fs];
        const Complex s5 = F[k] - s1;
        const Complex a = F[k] + s1;
        const Complex s3 = s0 + s2, s4 = s0 - s2;
        F[k + 2 * m] = a - s3;
        F[k] = a + s3;
        const Complex rot = inv ? Complex(-s4.imag(), s4.real()) : Complex(s4.imag(), -s4.real());
        F[k + m] = s5 + rot;
        F[k + 3 * m] = s5 - rot;
      }
    } else if (P == 3) {
      const T s3 = tw[fs * size_t(m)].imag();
      for (int k = 0; k < m; ++k) {
        const Complex a = F[k];
        const Complex b = F[k + m] * tw[size_t(k) * fs];
        const Complex c = F[k + 2 * m] * tw[size_t(2 * k) * fs];
        const Complex sum = b + c, dif = b - c;
        const Complex mid = a - T(0.5) * sum;
        const Complex rot(-s3 * dif.imag(), s3 * dif.real());
        F[k] = a + sum;
        F[k + m] = mid + rot;
        F[k + 2 * m] = mid - rot;
      }
    } else {
      const size_t n = size_t(pl.n);
      std::vector<Complex> x(static_cast<size_t>(P));
      for (int k = 0; k < m; ++k) {
        for (int q = 0; q < P; ++q) x[size_t(q)] = F[k + q * m] * tw[(size_t(q) * k * fs) % n];
        for (int u = 0; u < P; ++u) {
          Complex acc = x[0];
          for (int q = 1; q < P; ++q) acc += x[size_t(q)] * tw[(size_t(q) * u * m * fs) % n];
          F[k + u * m] = acc;
        }
      }
    }
  }

  static void work(const Plan& pl, bool inv, int stage, Complex* out, const Complex* in, size_t fs) {
    const int P = pl.radix[size_t(stage)], m = pl.remain[size_t(stage)];
    if (m == 1) {
      for (int j = 0; j < P; ++j) out[j] = in[size_t(j) * fs];
    } else {
      for (int j = 0; j < P; ++j) work(pl, inv, stage + 1, out + j * m, in + size_t(j) * fs, fs * P);
    }
    butterfly(pl, inv, out, fs, P, m);
  }

  void transform(Complex* dst, const Complex* src, int n, bool inverse) {
    if (n == 0) return;
    if (n == 1) {
      dst[0] = src[0];
      return;
    }
    std::vector<Complex> in(src, src + n);  // src may alias dst
    work(plan(n), inverse, 0, dst, in.data(), 1);
    if (inverse)
      for (int i = 0; i < n; ++i) dst[i] /= T(n);
  }

  std::map<int, Plan> plans_;
};

}  // namespace Eigen
