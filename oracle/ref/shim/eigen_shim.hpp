// ORACLE SHIM — TEST INFRASTRUCTURE ONLY (builds oracle/_ref, never product).
//
// A small, eager subset of the Eigen 3.4 dense API: exactly the surface that
// the reference hot-path sources (/root/reference/proj/core/src/*.cpp) and
// their doctest suites use, so those files compile VERBATIM against it
// (SURVEY.md §8c option A). Eigen itself is absent from this image.
//
// Semantics kept from Eigen, per coefficient:
//   * column-major storage (types.hpp:12-14);
//   * scalar*matrix, matrix/scalar, diag*matrix (row scaling) and
//     matrix*diag (column scaling) evaluate lhs-op-rhs per coefficient;
//   * complex products use the packet formula (ar*br - ai*bi, ar*bi + ai*br);
//   * norm() = sqrt(sum |a_ij|^2); allFinite() = every coefficient finite;
//   * PartialPivLU follows Eigen's PartialPivLU.h `unblocked_lu`: abs-scored
//     partial pivoting, first maximum wins, column scaled by the pivot, rank-1
//     update of the trailing block; solve() = P, unit-lower, upper solves.
// Not Eigen: no expression templates (every operation evaluates into a
// Matrix), GEMM blocking / summation order (complex GEMM and triangular
// solves go to OpenBLAS, single-threaded, as SURVEY.md §8c recommends), and
// the blocked LU Eigen switches to above 16 columns. Results therefore match a
// real Eigen build to rounding only.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

extern "C" {
// OpenBLAS as shipped with scipy (LP64, symbol prefix scipy_), linked by oracle/Makefile.
void scipy_cblas_zgemm(int order, int ta, int tb, int m, int n, int k, const void* alpha, const void* a,
                       int lda, const void* b, int ldb, const void* beta, void* c, int ldc);
void scipy_cblas_ztrsm(int order, int side, int uplo, int ta, int diag, int m, int n, const void* alpha,
                       const void* a, int lda, void* b, int ldb);
int scipy_LAPACKE_zgeev(int layout, char jobvl, char jobvr, int n, std::complex<double>* a, int lda,
                        std::complex<double>* w, std::complex<double>* vl, int ldvl, std::complex<double>* vr,
                        int ldvr);
void scipy_openblas_set_num_threads(int n);
}

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;

namespace shim {

template <class T> struct real_of { using type = T; };
template <class T> struct real_of<std::complex<T>> { using type = T; };
template <class T> using real_t = typename real_of<T>::type;
template <class T> inline constexpr bool is_complex_v = false;
template <class T> inline constexpr bool is_complex_v<std::complex<T>> = true;
template <class T>
inline constexpr bool is_scalar_v = std::is_arithmetic_v<T> || is_complex_v<T>;

// Eigen promotes an integer literal to the matrix's (real) scalar.
template <class M, class S>
inline auto lit(const S& s) {
  if constexpr (std::is_integral_v<S> && !std::is_integral_v<M>)
    return (real_t<M>)s;
  else
    return s;
}

// products in Eigen's packet form (no NaN-recovery branch of std::complex)
template <class A, class B>
inline auto mul(const A& a, const B& b) {
  if constexpr (is_complex_v<A> && is_complex_v<B>)
    return A(a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real());
  else
    return a * b;
}
// complex quotient a / b as Eigen's SSE pdiv: a * conj(b) / |b|^2
template <class A, class B>
inline auto quo(const A& a, const B& b) {
  if constexpr (is_complex_v<A> && is_complex_v<B>) {
    const double s = b.real() * b.real() + b.imag() * b.imag();
    const A n(a.real() * b.real() + a.imag() * b.imag(), a.imag() * b.real() - a.real() * b.imag());
    return A(n.real() / s, n.imag() / s);
  } else {
    return a / b;
  }
}
template <class A, class B>
using mul_t = decltype(mul(std::declval<A>(), std::declval<B>()));

template <class T>
inline double abs2(const T& x) {
  if constexpr (is_complex_v<T>)
    return x.real() * x.real() + x.imag() * x.imag();
  else
    return (double)x * (double)x;
}
template <class T>
inline bool finite(const T& x) {
  if constexpr (is_complex_v<T>)
    return std::isfinite(x.real()) && std::isfinite(x.imag());
  else
    return std::isfinite((double)x);
}

inline void blas_init() {
  static const bool once = (scipy_openblas_set_num_threads(1), true);
  (void)once;
}

}  // namespace shim

template <class S, int R = Dynamic, int C = Dynamic>
class Matrix;
template <class M>
class Block;
template <class S>
class DiagonalWrapper;
template <class MatrixType>
class PartialPivLU;

template <class X>
concept DenseExpr = requires { typename X::Scalar; } && X::is_dense_expr;

template <class S, int R, int C>
using Mat = Matrix<S, R, C>;

template <class D>
struct DenseBase {
  const D& derived() const { return static_cast<const D&>(*this); }
  Index size() const { return derived().rows() * derived().cols(); }
  auto lin(Index i) const {
    const D& d = derived();
    return d.rows() == 1 ? d.coeff(0, i) : d.coeff(i % d.rows(), i / d.rows());
  }

  auto eval() const {
    using S = typename D::Scalar;
    return Matrix<S, D::RowsAtCompileTime, D::ColsAtCompileTime>(derived());
  }
  auto transpose() const {
    using S = typename D::Scalar;
    const D& d = derived();
    Matrix<S, D::ColsAtCompileTime, D::RowsAtCompileTime> t;
    t.resize(d.cols(), d.rows());
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i) t.coeffRef(j, i) = d.coeff(i, j);
    return t;
  }
  auto conjugate() const {
    using S = typename D::Scalar;
    const D& d = derived();
    Matrix<S, D::RowsAtCompileTime, D::ColsAtCompileTime> t;
    t.resize(d.rows(), d.cols());
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i) {
        if constexpr (shim::is_complex_v<S>)
          t.coeffRef(i, j) = std::conj(d.coeff(i, j));
        else
          t.coeffRef(i, j) = d.coeff(i, j);
      }
    return t;
  }
  auto adjoint() const { return conjugate().transpose(); }
  template <class F>
  auto map(F f) const {
    using S = typename D::Scalar;
    using T = decltype(f(std::declval<S>()));
    const D& d = derived();
    Matrix<T, D::RowsAtCompileTime, D::ColsAtCompileTime> t;
    t.resize(d.rows(), d.cols());
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i) t.coeffRef(i, j) = f(d.coeff(i, j));
    return t;
  }
  auto cwiseAbs() const {
    return map([](const auto& x) { return (shim::real_t<typename D::Scalar>)std::abs(x); });
  }
  auto cwiseAbs2() const {
    return map([](const auto& x) { return (shim::real_t<typename D::Scalar>)shim::abs2(x); });
  }
  auto real() const {
    return map([](const auto& x) { return (shim::real_t<typename D::Scalar>)std::real(x); });
  }
  auto imag() const {
    return map([](const auto& x) { return (shim::real_t<typename D::Scalar>)std::imag(x); });
  }

  auto sum() const {
    const D& d = derived();
    typename D::Scalar s(0);
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i) s += d.coeff(i, j);
    return s;
  }
  auto prod() const {
    const D& d = derived();
    typename D::Scalar s(1);
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i) s = shim::mul(s, d.coeff(i, j));
    return s;
  }
  auto trace() const {
    const D& d = derived();
    typename D::Scalar s(0);
    for (Index i = 0; i < std::min(d.rows(), d.cols()); ++i) s += d.coeff(i, i);
    return s;
  }
  double squaredNorm() const {
    const D& d = derived();
    double s = 0.0;
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i) s += shim::abs2(d.coeff(i, j));
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  bool allFinite() const {
    const D& d = derived();
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i)
        if (!shim::finite(d.coeff(i, j))) return false;
    return true;
  }
  bool hasNaN() const {
    const D& d = derived();
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i)
        if (d.coeff(i, j) != d.coeff(i, j)) return true;
    return false;
  }
  // first extremum wins (Eigen's max_coeff_visitor: strict comparison)
  template <bool MAX>
  auto extremum(Index* ri, Index* ci) const {
    const D& d = derived();
    if (d.size() == 0) throw std::runtime_error("eigen shim: extremum of an empty matrix");
    typename D::Scalar best = d.coeff(0, 0);
    Index bi = 0, bj = 0;
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i) {
        const auto v = d.coeff(i, j);
        if (MAX ? (v > best) : (v < best)) {
          best = v;
          bi = i;
          bj = j;
        }
      }
    if (ri && ci) {
      *ri = bi;
      *ci = bj;
    } else if (ri) {
      *ri = d.rows() == 1 ? bj : bi;
    }
    return best;
  }
  auto maxCoeff() const { return extremum<true>(nullptr, nullptr); }
  auto minCoeff() const { return extremum<false>(nullptr, nullptr); }
  template <class I>
  auto maxCoeff(I* idx) const {
    Index k;
    auto v = extremum<true>(&k, nullptr);
    *idx = (I)k;
    return v;
  }
  template <class I>
  auto minCoeff(I* idx) const {
    Index k;
    auto v = extremum<false>(&k, nullptr);
    *idx = (I)k;
    return v;
  }
  // Eigen's dot is conjugate-linear in the first argument
  template <DenseExpr O>
  auto dot(const O& o) const {
    const D& d = derived();
    using S = shim::mul_t<typename D::Scalar, typename O::Scalar>;
    S s(0);
    for (Index i = 0; i < d.size(); ++i) {
      auto a = d.lin(i);
      if constexpr (shim::is_complex_v<decltype(a)>) a = std::conj(a);
      s += shim::mul(a, o.lin(i));
    }
    return s;
  }

  // column sums / row sums
  struct Colwise {
    const D& d;
    auto sum() const {
      Matrix<typename D::Scalar, 1, Dynamic> r;
      r.resize(1, d.cols());
      for (Index j = 0; j < d.cols(); ++j) {
        typename D::Scalar s(0);
        for (Index i = 0; i < d.rows(); ++i) s += d.coeff(i, j);
        r.coeffRef(0, j) = s;
      }
      return r;
    }
    auto maxCoeff() const {
      Matrix<typename D::Scalar, 1, Dynamic> r;
      r.resize(1, d.cols());
      for (Index j = 0; j < d.cols(); ++j) {
        auto s = d.coeff(0, j);
        for (Index i = 1; i < d.rows(); ++i) s = std::max(s, d.coeff(i, j));
        r.coeffRef(0, j) = s;
      }
      return r;
    }
  };
  struct Rowwise {
    const D& d;
    auto sum() const {
      Matrix<typename D::Scalar, Dynamic, 1> r;
      r.resize(d.rows(), 1);
      for (Index i = 0; i < d.rows(); ++i) {
        typename D::Scalar s(0);
        for (Index j = 0; j < d.cols(); ++j) s += d.coeff(i, j);
        r.coeffRef(i, 0) = s;
      }
      return r;
    }
  };
  Colwise colwise() const { return Colwise{derived()}; }
  Rowwise rowwise() const { return Rowwise{derived()}; }

  auto diagonal() const {
    const D& d = derived();
    Matrix<typename D::Scalar, Dynamic, 1> v;
    v.resize(std::min(d.rows(), d.cols()), 1);
    for (Index i = 0; i < v.rows(); ++i) v.coeffRef(i, 0) = d.coeff(i, i);
    return v;
  }
  auto asDiagonal() const {
    const D& d = derived();
    Matrix<typename D::Scalar, Dynamic, 1> v;
    v.resize(d.size(), 1);
    for (Index i = 0; i < d.size(); ++i) v.coeffRef(i, 0) = d.lin(i);
    return DiagonalWrapper<typename D::Scalar>(std::move(v));
  }
  auto determinant() const {
    return PartialPivLU<Matrix<typename D::Scalar, Dynamic, Dynamic>>(derived()).determinant();
  }
  auto inverse() const {
    return PartialPivLU<Matrix<typename D::Scalar, Dynamic, Dynamic>>(derived()).inverse();
  }

  // read-only views
  Block<const D> block(Index r, Index c, Index nr, Index nc) const { return {&derived(), r, c, nr, nc}; }
  Block<const D> col(Index j) const { return block(0, j, derived().rows(), 1); }
  Block<const D> row(Index i) const { return block(i, 0, 1, derived().cols()); }
  Block<const D> topLeftCorner(Index nr, Index nc) const { return block(0, 0, nr, nc); }
  Block<const D> topRightCorner(Index nr, Index nc) const { return block(0, derived().cols() - nc, nr, nc); }
  Block<const D> bottomLeftCorner(Index nr, Index nc) const { return block(derived().rows() - nr, 0, nr, nc); }
  Block<const D> bottomRightCorner(Index nr, Index nc) const {
    return block(derived().rows() - nr, derived().cols() - nc, nr, nc);
  }
  Block<const D> topRows(Index n) const { return block(0, 0, n, derived().cols()); }
  Block<const D> bottomRows(Index n) const { return block(derived().rows() - n, 0, n, derived().cols()); }
  Block<const D> leftCols(Index n) const { return block(0, 0, derived().rows(), n); }
  Block<const D> rightCols(Index n) const { return block(0, derived().cols() - n, derived().rows(), n); }
  Block<const D> segment(Index s, Index n) const {
    return derived().cols() == 1 ? block(s, 0, n, 1) : block(0, s, 1, n);
  }
  Block<const D> head(Index n) const { return segment(0, n); }
  Block<const D> tail(Index n) const { return segment(derived().size() - n, n); }

  auto x() const { return lin(0); }
  auto y() const { return lin(1); }
  auto z() const { return lin(2); }
};

// Writable views: Matrix and Block<non-const>.
template <class D>
struct MutableBase : DenseBase<D> {
  using DenseBase<D>::block;
  using DenseBase<D>::col;
  using DenseBase<D>::row;
  using DenseBase<D>::topLeftCorner;
  using DenseBase<D>::topRightCorner;
  using DenseBase<D>::bottomLeftCorner;
  using DenseBase<D>::bottomRightCorner;
  using DenseBase<D>::topRows;
  using DenseBase<D>::bottomRows;
  using DenseBase<D>::leftCols;
  using DenseBase<D>::rightCols;
  using DenseBase<D>::segment;
  using DenseBase<D>::head;
  using DenseBase<D>::tail;
  D& self() { return static_cast<D&>(*this); }

  Block<D> block(Index r, Index c, Index nr, Index nc) { return {&self(), r, c, nr, nc}; }
  Block<D> col(Index j) { return block(0, j, self().rows(), 1); }
  Block<D> row(Index i) { return block(i, 0, 1, self().cols()); }
  Block<D> topLeftCorner(Index nr, Index nc) { return block(0, 0, nr, nc); }
  Block<D> topRightCorner(Index nr, Index nc) { return block(0, self().cols() - nc, nr, nc); }
  Block<D> bottomLeftCorner(Index nr, Index nc) { return block(self().rows() - nr, 0, nr, nc); }
  Block<D> bottomRightCorner(Index nr, Index nc) {
    return block(self().rows() - nr, self().cols() - nc, nr, nc);
  }
  Block<D> topRows(Index n) { return block(0, 0, n, self().cols()); }
  Block<D> bottomRows(Index n) { return block(self().rows() - n, 0, n, self().cols()); }
  Block<D> leftCols(Index n) { return block(0, 0, self().rows(), n); }
  Block<D> rightCols(Index n) { return block(0, self().cols() - n, self().rows(), n); }
  Block<D> segment(Index s, Index n) { return self().cols() == 1 ? block(s, 0, n, 1) : block(0, s, 1, n); }
  Block<D> head(Index n) { return segment(0, n); }
  Block<D> tail(Index n) { return segment(self().size() - n, n); }

  D& setZero() {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = typename D::Scalar(0);
    return self();
  }
  template <class V>
  D& setConstant(const V& v) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = v;
    return self();
  }
  template <class V>
  D& fill(const V& v) { return setConstant(v); }
  D& setIdentity() {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = typename D::Scalar(i == j ? 1 : 0);
    return self();
  }
  template <DenseExpr O>
  D& operator+=(const O& o) {
    const auto t = o.eval();  // alias-safe
    check(t);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) += t.coeff(i, j);
    return self();
  }
  template <DenseExpr O>
  D& operator-=(const O& o) {
    const auto t = o.eval();
    check(t);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) -= t.coeff(i, j);
    return self();
  }
  template <class S>
    requires shim::is_scalar_v<S>
  D& operator*=(const S& s) {
    const auto v = shim::lit<typename D::Scalar>(s);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = shim::mul(self().coeff(i, j), v);
    return self();
  }
  template <class S>
    requires shim::is_scalar_v<S>
  D& operator/=(const S& s) {
    const auto v = shim::lit<typename D::Scalar>(s);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = shim::quo(self().coeff(i, j), v);
    return self();
  }
  // comma initializer (Eigen fills row by row): m << a, b, c, ...
  struct CommaInit {
    D& m;
    Index k;
    template <class V>
    CommaInit& operator,(const V& v) {
      put(v);
      return *this;
    }
    template <class V>
    void put(const V& v) {
      if (k >= m.size()) throw std::runtime_error("eigen shim: too many coefficients in comma initializer");
      m.coeffRef(k / m.cols(), k % m.cols()) = (typename D::Scalar)v;
      ++k;
    }
  };
  template <class V>
    requires shim::is_scalar_v<V>
  CommaInit operator<<(const V& v) {
    CommaInit c{self(), 0};
    c.put(v);
    return c;
  }
  template <class T>
  void check(const T& t) const {
    const D& d = static_cast<const D&>(*this);
    if (t.rows() != d.rows() || t.cols() != d.cols())
      throw std::runtime_error("eigen shim: dimension mismatch in compound assignment");
  }
  template <DenseExpr O>
  void assign_from(const O& o) {
    const auto t = o.eval();
    check(t);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = t.coeff(i, j);
  }
};

template <class S, int R, int C>
class Matrix : public MutableBase<Matrix<S, R, C>> {
 public:
  using Scalar = S;
  using RealScalar = shim::real_t<S>;
  static constexpr bool is_dense_expr = true;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr bool IsFixed = R > 0 && C > 0;

  Matrix() : r_(R > 0 ? R : 0), c_(C > 0 ? C : 0), v_((std::size_t)(r_ * c_)) {}
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) noexcept = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) noexcept = default;

  // size constructor for dynamic vectors
  template <class I>
    requires std::is_integral_v<I> && (R == 1 || C == 1) && (!IsFixed)
  explicit Matrix(I n) : Matrix() {
    resize((Index)n);
  }
  // (rows, cols) for dynamic matrices; coefficients for fixed 2-vectors
  template <class A, class B>
    requires shim::is_scalar_v<A> && shim::is_scalar_v<B>
  Matrix(const A& a, const B& b) : Matrix() {
    if constexpr (IsFixed && R * C == 2) {
      v_[0] = (S)a;
      v_[1] = (S)b;
    } else if constexpr (std::is_integral_v<A> && std::is_integral_v<B>) {
      resize((Index)a, (Index)b);
    } else {
      static_assert(IsFixed && R * C == 2, "eigen shim: 2 coefficients need a fixed 2-vector");
    }
  }
  template <class A, class B, class D3>
    requires(IsFixed && R * C == 3)
  Matrix(const A& a, const B& b, const D3& c) : Matrix() {
    v_[0] = (S)a;
    v_[1] = (S)b;
    v_[2] = (S)c;
  }
  template <DenseExpr O>
    requires(!std::is_same_v<O, Matrix>)
  Matrix(const O& o) : Matrix() {
    resize(o.rows(), o.cols());
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) coeffRef(i, j) = (S)o.coeff(i, j);
  }
  template <DenseExpr O>
    requires(!std::is_same_v<O, Matrix>)
  Matrix& operator=(const O& o) {
    Matrix t(o);
    *this = std::move(t);
    return *this;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  S* data() { return v_.data(); }
  const S* data() const { return v_.data(); }
  const S& coeff(Index i, Index j) const { return v_[(std::size_t)(j * r_ + i)]; }
  S& coeffRef(Index i, Index j) { return v_[(std::size_t)(j * r_ + i)]; }
  const S& operator()(Index i, Index j) const { return coeff(i, j); }
  S& operator()(Index i, Index j) { return coeffRef(i, j); }
  const S& operator()(Index i) const { return v_[(std::size_t)i]; }
  S& operator()(Index i) { return v_[(std::size_t)i]; }
  const S& operator[](Index i) const { return v_[(std::size_t)i]; }
  S& operator[](Index i) { return v_[(std::size_t)i]; }
  const S& x() const { return v_[0]; }
  const S& y() const { return v_[1]; }
  const S& z() const { return v_[2]; }
  S& x() { return v_[0]; }
  S& y() { return v_[1]; }
  S& z() { return v_[2]; }

  void resize(Index r, Index c) {
    if ((R > 0 && r != R) || (C > 0 && c != C))
      throw std::runtime_error("eigen shim: resize conflicts with a fixed dimension");
    r_ = r;
    c_ = c;
    v_.assign((std::size_t)(r * c), S(0));
  }
  void resize(Index n) {
    if constexpr (C == 1)
      resize(n, 1);
    else if constexpr (R == 1)
      resize(1, n);
    else
      throw std::runtime_error("eigen shim: resize(n) needs a vector type");
  }
  Matrix& noalias() { return *this; }
  void swap(Matrix& o) { std::swap(r_, o.r_), std::swap(c_, o.c_), v_.swap(o.v_); }

  static Matrix Zero(Index r, Index c) {
    Matrix m;
    m.resize(r, c);
    return m;
  }
  static Matrix Zero(Index n) {
    Matrix m;
    m.resize(n);
    return m;
  }
  static Matrix Zero() { return Matrix(); }
  static Matrix Constant(Index r, Index c, const S& v) {
    Matrix m = Zero(r, c);
    m.setConstant(v);
    return m;
  }
  static Matrix Constant(Index n, const S& v) {
    Matrix m = Zero(n);
    m.setConstant(v);
    return m;
  }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, S(1)); }
  static Matrix Ones(Index n) { return Constant(n, S(1)); }
  static Matrix Identity(Index r, Index c) {
    Matrix m = Zero(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m.coeffRef(i, i) = S(1);
    return m;
  }
  static Matrix Identity() { return Identity(R, C); }
  static Matrix Unit(Index k) {
    Matrix m;
    m.v_[(std::size_t)k] = S(1);
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }

 private:
  Index r_, c_;
  std::vector<S> v_;
};

template <class M>
class Block : public std::conditional_t<std::is_const_v<M>, DenseBase<Block<M>>, MutableBase<Block<M>>> {
 public:
  using Scalar = typename std::remove_const_t<M>::Scalar;
  static constexpr bool is_dense_expr = true;
  static constexpr int RowsAtCompileTime = Dynamic;
  static constexpr int ColsAtCompileTime = Dynamic;

  Block(M* m, Index r0, Index c0, Index nr, Index nc) : m_(m), r0_(r0), c0_(c0), nr_(nr), nc_(nc) {
    if (r0 < 0 || c0 < 0 || nr < 0 || nc < 0 || r0 + nr > m->rows() || c0 + nc > m->cols())
      throw std::runtime_error("eigen shim: block out of range");
  }
  Block(const Block&) = default;
  Block& operator=(const Block& o) {
    this->assign_from(o);
    return *this;
  }
  template <DenseExpr O>
  Block& operator=(const O& o) {
    this->assign_from(o);
    return *this;
  }

  Index rows() const { return nr_; }
  Index cols() const { return nc_; }
  Index size() const { return nr_ * nc_; }
  Scalar coeff(Index i, Index j) const { return m_->coeff(r0_ + i, c0_ + j); }
  auto& coeffRef(Index i, Index j)
    requires(!std::is_const_v<M>)
  {
    return m_->coeffRef(r0_ + i, c0_ + j);
  }
  Scalar operator()(Index i, Index j) const { return coeff(i, j); }
  auto& operator()(Index i, Index j)
    requires(!std::is_const_v<M>)
  {
    return coeffRef(i, j);
  }
  Scalar operator()(Index i) const { return nr_ == 1 ? coeff(0, i) : coeff(i, 0); }
  auto& operator()(Index i)
    requires(!std::is_const_v<M>)
  {
    return nr_ == 1 ? coeffRef(0, i) : coeffRef(i, 0);
  }
  Scalar operator[](Index i) const { return (*this)(i); }

 private:
  M* m_;
  Index r0_, c0_, nr_, nc_;
};

template <class S>
class DiagonalWrapper {
 public:
  explicit DiagonalWrapper(Matrix<S, Dynamic, 1> d) : d_(std::move(d)) {}
  const Matrix<S, Dynamic, 1>& diagonal() const { return d_; }
  Index rows() const { return d_.rows(); }
  Index cols() const { return d_.rows(); }
  Matrix<S, Dynamic, Dynamic> toDenseMatrix() const {
    auto m = Matrix<S, Dynamic, Dynamic>::Zero(rows(), rows());
    for (Index i = 0; i < rows(); ++i) m.coeffRef(i, i) = d_(i);
    return m;
  }

 private:
  Matrix<S, Dynamic, 1> d_;
};


namespace shim {

template <int A, int B>
inline constexpr int pick = A != Dynamic ? A : B;

template <class F, DenseExpr A, DenseExpr B>
inline auto zip(const A& a, const B& b, F f) {
  if (a.rows() != b.rows() || a.cols() != b.cols())
    throw std::runtime_error("eigen shim: dimension mismatch in a coefficient-wise operation");
  using T = decltype(f(a.coeff(0, 0), b.coeff(0, 0)));
  Matrix<T, pick<A::RowsAtCompileTime, B::RowsAtCompileTime>, pick<A::ColsAtCompileTime, B::ColsAtCompileTime>> r;
  r.resize(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) r.coeffRef(i, j) = f(a.coeff(i, j), b.coeff(i, j));
  return r;
}

// contiguous column-major view of any dense expression
template <class S, DenseExpr X>
inline Matrix<S, Dynamic, Dynamic> dense(const X& x) {
  return Matrix<S, Dynamic, Dynamic>(x);
}

using cd = std::complex<double>;

inline void zgemm(Index m, Index n, Index k, const cd* a, const cd* b, cd* c) {
  blas_init();
  const cd one(1.0, 0.0), zero(0.0, 0.0);
  scipy_cblas_zgemm(102, 111, 111, (int)m, (int)n, (int)k, &one, a, (int)std::max<Index>(1, m), b,
                    (int)std::max<Index>(1, k), &zero, c, (int)std::max<Index>(1, m));
}

}  // namespace shim

// ---------------------------------------------------------------- arithmetic
template <DenseExpr A, DenseExpr B>
auto operator+(const A& a, const B& b) {
  return shim::zip(a, b, [](const auto& x, const auto& y) { return x + y; });
}
template <DenseExpr A, DenseExpr B>
auto operator-(const A& a, const B& b) {
  return shim::zip(a, b, [](const auto& x, const auto& y) { return x - y; });
}
template <DenseExpr A>
auto operator-(const A& a) {
  return a.map([](const auto& x) { return -x; });
}
template <class S, DenseExpr A>
  requires shim::is_scalar_v<S>
auto operator*(const S& s, const A& a) {
  const auto v = shim::lit<typename A::Scalar>(s);
  return a.map([v](const auto& x) { return shim::mul(v, x); });
}
template <class S, DenseExpr A>
  requires shim::is_scalar_v<S>
auto operator*(const A& a, const S& s) {
  const auto v = shim::lit<typename A::Scalar>(s);
  return a.map([v](const auto& x) { return shim::mul(x, v); });
}
template <class S, DenseExpr A>
  requires shim::is_scalar_v<S>
auto operator/(const A& a, const S& s) {
  const auto v = shim::lit<typename A::Scalar>(s);
  return a.map([v](const auto& x) { return shim::quo(x, v); });
}
template <DenseExpr A, DenseExpr B>
bool operator==(const A& a, const B& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i)
      if (!(a.coeff(i, j) == b.coeff(i, j))) return false;
  return true;
}
template <DenseExpr A, DenseExpr B>
bool operator!=(const A& a, const B& b) {
  return !(a == b);
}

// matrix product
template <DenseExpr A, DenseExpr B>
auto operator*(const A& a, const B& b) {
  using T = shim::mul_t<typename A::Scalar, typename B::Scalar>;
  if (a.cols() != b.rows()) throw std::runtime_error("eigen shim: product dimension mismatch");
  Matrix<T, A::RowsAtCompileTime, B::ColsAtCompileTime> r;
  r.resize(a.rows(), b.cols());
  if constexpr (std::is_same_v<T, shim::cd> && std::is_same_v<typename A::Scalar, shim::cd> &&
                std::is_same_v<typename B::Scalar, shim::cd>) {
    if (r.size() == 0) return r;
    if (a.cols() == 0) return r;
    const auto ad = shim::dense<shim::cd>(a);
    const auto bd = shim::dense<shim::cd>(b);
    shim::zgemm(a.rows(), b.cols(), a.cols(), ad.data(), bd.data(), r.data());
  } else {
    for (Index j = 0; j < b.cols(); ++j)
      for (Index i = 0; i < a.rows(); ++i) {
        T s(0);
        for (Index k = 0; k < a.cols(); ++k) s += shim::mul(a.coeff(i, k), b.coeff(k, j));
        r.coeffRef(i, j) = s;
      }
  }
  return r;
}
// diagonal products: row scaling / column scaling, lhs-op-rhs per coefficient
template <class S, DenseExpr A>
auto operator*(const DiagonalWrapper<S>& d, const A& a) {
  if (d.cols() != a.rows()) throw std::runtime_error("eigen shim: diagonal product dimension mismatch");
  using T = shim::mul_t<S, typename A::Scalar>;
  Matrix<T, A::RowsAtCompileTime, A::ColsAtCompileTime> r;
  r.resize(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) r.coeffRef(i, j) = shim::mul(d.diagonal()(i), a.coeff(i, j));
  return r;
}
template <class S, DenseExpr A>
auto operator*(const A& a, const DiagonalWrapper<S>& d) {
  if (a.cols() != d.rows()) throw std::runtime_error("eigen shim: diagonal product dimension mismatch");
  using T = shim::mul_t<typename A::Scalar, S>;
  Matrix<T, A::RowsAtCompileTime, A::ColsAtCompileTime> r;
  r.resize(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) r.coeffRef(i, j) = shim::mul(a.coeff(i, j), d.diagonal()(j));
  return r;
}

// ---------------------------------------------------------------- LU
template <class MatrixType>
class PartialPivLU {
 public:
  using Scalar = typename MatrixType::Scalar;
  PartialPivLU() = default;
  template <DenseExpr O>
  explicit PartialPivLU(const O& a) {
    compute(a);
  }

  // PartialPivLU.h partial_lu_impl::unblocked_lu, column k at a time
  template <DenseExpr O>
  PartialPivLU& compute(const O& a) {
    lu_ = MatrixType(a);
    const Index n = lu_.rows();
    if (lu_.cols() != n) throw std::runtime_error("eigen shim: PartialPivLU needs a square matrix");
    transp_.assign((std::size_t)n, 0);
    ntransp_ = 0;
    Scalar* A = lu_.data();
    for (Index k = 0; k < n; ++k) {
      Scalar* ck = A + k * n;
      Index p = k;
      double best = std::abs(ck[k]);
      for (Index i = k + 1; i < n; ++i) {
        const double s = std::abs(ck[i]);
        if (s > best) {
          best = s;
          p = i;
        }
      }
      transp_[(std::size_t)k] = p;
      if (best != 0.0) {
        if (p != k) {
          for (Index j = 0; j < n; ++j) std::swap(A[j * n + k], A[j * n + p]);
          ++ntransp_;
        }
        const Scalar piv = ck[k];
        for (Index i = k + 1; i < n; ++i) ck[i] = shim::quo(ck[i], piv);
      }
      for (Index j = k + 1; j < n; ++j) {
        Scalar* cj = A + j * n;
        const Scalar u = cj[k];
        for (Index i = k + 1; i < n; ++i) cj[i] -= shim::mul(ck[i], u);
      }
    }
    return *this;
  }
  const MatrixType& matrixLU() const { return lu_; }

  template <DenseExpr O>
  Matrix<Scalar, Dynamic, Dynamic> solve(const O& b) const {
    const Index n = lu_.rows();
    Matrix<Scalar, Dynamic, Dynamic> x(b);
    if (x.rows() != n) throw std::runtime_error("eigen shim: LU solve dimension mismatch");
    const Index m = x.cols();
    for (Index k = 0; k < n; ++k) {
      const Index p = transp_[(std::size_t)k];
      if (p != k)
        for (Index j = 0; j < m; ++j) std::swap(x.coeffRef(k, j), x.coeffRef(p, j));
    }
    if (n == 0 || m == 0) return x;
    if constexpr (std::is_same_v<Scalar, shim::cd>) {
      shim::blas_init();
      const shim::cd one(1.0, 0.0);
      scipy_cblas_ztrsm(102, 141, 122, 111, 132, (int)n, (int)m, &one, lu_.data(), (int)n, x.data(), (int)n);
      scipy_cblas_ztrsm(102, 141, 121, 111, 131, (int)n, (int)m, &one, lu_.data(), (int)n, x.data(), (int)n);
    } else {
      for (Index j = 0; j < m; ++j) {
        for (Index i = 0; i < n; ++i)
          for (Index k = 0; k < i; ++k) x.coeffRef(i, j) -= shim::mul(lu_.coeff(i, k), x.coeff(k, j));
        for (Index i = n - 1; i >= 0; --i) {
          for (Index k = i + 1; k < n; ++k) x.coeffRef(i, j) -= shim::mul(lu_.coeff(i, k), x.coeff(k, j));
          x.coeffRef(i, j) = shim::quo(x.coeff(i, j), lu_.coeff(i, i));
        }
      }
    }
    return x;
  }
  Scalar determinant() const {
    Scalar d = (ntransp_ % 2) ? Scalar(-1) : Scalar(1);
    for (Index i = 0; i < lu_.rows(); ++i) d = shim::mul(d, lu_.coeff(i, i));
    return d;
  }
  MatrixType inverse() const { return MatrixType(solve(MatrixType::Identity(lu_.rows(), lu_.rows()))); }

 private:
  MatrixType lu_;
  std::vector<Index> transp_;
  int ntransp_ = 0;
};


// ---------------------------------------------------------------- eigenvalues
template <class MatrixType>
class ComplexEigenSolver {
 public:
  template <DenseExpr O>
  explicit ComplexEigenSolver(const O& a, bool /*computeEigenvectors*/ = true) {
    Matrix<shim::cd, Dynamic, Dynamic> m(a);
    const Index n = m.rows();
    w_.resize(n);
    if (n > 0) {
      const int info = scipy_LAPACKE_zgeev(102, 'N', 'N', (int)n, m.data(), (int)n, w_.data(), nullptr, 1,
                                           nullptr, 1);
      if (info != 0) throw std::runtime_error("eigen shim: zgeev failed");
    }
  }
  const Matrix<shim::cd, Dynamic, 1>& eigenvalues() const { return w_; }

 private:
  Matrix<shim::cd, Dynamic, 1> w_;
};

// ---------------------------------------------------------------- fixed-size aliases
using MatrixXcd = Matrix<std::complex<double>, Dynamic, Dynamic>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector2i = Matrix<int, 2, 1>;
using Matrix3d = Matrix<double, 3, 3>;

// Geometry: AngleAxis::toRotationMatrix (Eigen/src/Geometry/AngleAxis.h)
template <class S>
class AngleAxis {
 public:
  AngleAxis(S angle, const Matrix<S, 3, 1>& axis) : a_(angle), ax_(axis) {}
  Matrix<S, 3, 3> toRotationMatrix() const {
    Matrix<S, 3, 3> res;
    const Matrix<S, 3, 1> sin_axis = std::sin(a_) * ax_;
    const S c = std::cos(a_);
    const Matrix<S, 3, 1> cos1_axis = (S(1) - c) * ax_;
    S tmp = cos1_axis.x() * ax_.y();
    res(0, 1) = tmp - sin_axis.z();
    res(1, 0) = tmp + sin_axis.z();
    tmp = cos1_axis.x() * ax_.z();
    res(0, 2) = tmp + sin_axis.y();
    res(2, 0) = tmp - sin_axis.y();
    tmp = cos1_axis.y() * ax_.z();
    res(1, 2) = tmp - sin_axis.x();
    res(2, 1) = tmp + sin_axis.x();
    for (int i = 0; i < 3; ++i) res(i, i) = cos1_axis(i) * ax_(i) + c;
    return res;
  }
  template <DenseExpr V>
  Matrix<S, 3, 1> operator*(const V& v) const {
    return Matrix<S, 3, 1>(toRotationMatrix() * v);
  }

 private:
  S a_;
  Matrix<S, 3, 1> ax_;
};
using AngleAxisd = AngleAxis<double>;

}  // namespace Eigen
