// Minimal Eigen-3.4-API shim: just enough of the Eigen surface that the reference
// (pdeopt, /root/reference/proj) uses on the range-space Schur path, so its UNMODIFIED
// sources (src/{mesh,fem,feti,control,mmio}.cpp + include/pdeopt/*.hpp) and its own doctest
// unit tests compile and run in this image, which has no Eigen (proj/CMakeLists.txt:15).
//
// TEST INFRASTRUCTURE ONLY (oracle/_ref): nothing in the product links or includes it.
// Written from the public Eigen API documentation (class/method names and their
// documented semantics), not from Eigen's sources.  Everything is eager (no expression
// templates): every arithmetic expression evaluates into a Matrix.  Decompositions are
// exact direct methods, so results agree with Eigen's to rounding:
//   SparseLU       -> banded LU with partial pivoting in the natural order
//                     (Eigen: supernodal LU, COLAMD order, threshold pivoting)
//   PartialPivLU   -> dense LU with partial (row) pivoting, LAPACK getf2 order
//   SimplicialLLT  -> banded Cholesky of the lower triangle, natural order (Eigen: AMD)
//   LLT            -> dense Cholesky
//   SelfAdjointEigenSolver / GeneralizedSelfAdjointEigenSolver -> cyclic Jacobi
//                     (generalized: B = L L^T, eig(L^-1 A L^-T), x = L^-T y, x^T B x = 1)
// Semantics kept: dot() conjugates its FIRST argument, norm() is the 2-/Frobenius norm,
// setFromTriplets() sums duplicates, SparseMatrix is column-major, dense storage
// column-major, comma initialisers fill row by row.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;
inline constexpr int Infinity = -1;

enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions {
  EigenvaluesOnly = 0x40,
  ComputeEigenvectors = 0x80,
  Ax_lBx = 0x100,
  ABx_lx = 0x200,
  BAx_lx = 0x400
};
enum StorageOptions { ColMajor = 0, RowMajor = 1, AutoAlign = 0 };
enum UpLoType { Lower = 1, Upper = 2 };

namespace internal {
template <class T> struct real_of { using type = T; };
template <class T> struct real_of<std::complex<T>> { using type = T; };
template <class T> struct is_cplx : std::false_type {};
template <class T> struct is_cplx<std::complex<T>> : std::true_type {};
template <class T> inline T conj_(const T& x) {
  if constexpr (is_cplx<T>::value) return std::conj(x); else return x;
}
template <class T> inline typename real_of<T>::type abs2_(const T& x) {
  if constexpr (is_cplx<T>::value) return std::norm(x); else return x * x;
}
template <class A, class B> using prod_t = decltype(std::declval<A>() * std::declval<B>());
template <class X> inline constexpr bool is_scalar_v = std::is_arithmetic_v<X> || is_cplx<X>::value;
template <class S, class D> inline D cast_(const S& v) {
  if constexpr (is_cplx<S>::value && !is_cplx<D>::value) return static_cast<D>(v.real());
  else return static_cast<D>(v);
}
inline constexpr int pick(int a, int b) { return a != Dynamic ? a : b; }
}  // namespace internal

template <class T> struct NumTraits {
  using Real = typename internal::real_of<T>::type;
  static Real epsilon() { return std::numeric_limits<Real>::epsilon(); }
  static Real dummy_precision() { return Real(1e-12); }
  static Real highest() { return std::numeric_limits<Real>::max(); }
};

template <class Derived> class DenseBase;
template <class S, int R = Dynamic, int C = Dynamic, int Opt = 0, int MR = R, int MC = C> class Matrix;
template <class S, int R, int C> class View;
template <class S, int Opt = 0, class SI = int> class SparseMatrix;

template <class S, int R, int C> using Array = Matrix<S, R, C>;
template <class S, int N> using Vector = Matrix<S, N, 1>;
template <class S, int N> using RowVector = Matrix<S, 1, N>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using MatrixXcd = Matrix<std::complex<double>, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;
using VectorXi = Matrix<int, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;

template <class D> struct is_dense : std::is_base_of<DenseBase<D>, D> {};

// Comma initializer: fills row by row (Eigen's order).
template <class Target> class CommaInit {
 public:
  using S = typename std::remove_reference_t<Target>::Scalar;
  CommaInit(Target t, const S& first) : t_(std::forward<Target>(t)) { put(first); }
  template <class D, std::enable_if_t<is_dense<D>::value, int> = 0> CommaInit(Target t, const D& first)
      : t_(std::forward<Target>(t)) { put_block(first); }
  CommaInit& operator,(const S& v) { put(v); return *this; }
  template <class D, std::enable_if_t<is_dense<D>::value, int> = 0> CommaInit& operator,(const D& b) {
    put_block(b);
    return *this;
  }

 private:
  void put(const S& v) {
    const Index c = t_.cols();
    t_.coeffRef(k_ / c, k_ % c) = v;
    ++k_;
  }
  template <class D> void put_block(const D& b) {  // vector targets: blocks are stacked
    if (t_.cols() != 1 || b.cols() != 1) throw std::invalid_argument("Eigen shim: block comma init needs vectors");
    for (Index i = 0; i < b.rows(); ++i) put(static_cast<S>(b.coeff(i, 0)));
  }
  Target t_;
  Index k_ = 0;
};

// CRTP base: every dense object exposes a strided column-major window
// (ptr_, rows, cols, row stride rs_, column stride cs_).
template <class Derived> class DenseBase {
 public:
  Derived& derived() { return static_cast<Derived&>(*this); }
  const Derived& derived() const { return static_cast<const Derived&>(*this); }

  Index size() const { return derived().rows() * derived().cols(); }

  template <class S> using Rl = typename internal::real_of<S>::type;
};

#define EIGEN_SHIM_DENSE_COMMON(SCALAR, RC, CC)                                                   \
  using Scalar = SCALAR;                                                                          \
  using RealScalar = typename internal::real_of<SCALAR>::type;                                     \
  static constexpr int RowsAtCompileTime = RC;                                                    \
  static constexpr int ColsAtCompileTime = CC;                                                    \
  static constexpr bool IsVectorAtCompileTime = (RC == 1 || CC == 1);                             \
  Index size() const { return rows() * cols(); }                                                  \
  Scalar& coeffRef(Index i, Index j) { return ptr_()[i * rs_() + j * cs_()]; }                    \
  const Scalar& coeff(Index i, Index j) const { return ptr_()[i * rs_() + j * cs_()]; }           \
  Scalar& operator()(Index i, Index j) { return coeffRef(i, j); }                                 \
  const Scalar& operator()(Index i, Index j) const { return coeff(i, j); }                        \
  Scalar& coeffRef(Index k) { return ptr_()[lin_(k)]; }                                           \
  const Scalar& coeff(Index k) const { return ptr_()[lin_(k)]; }                                  \
  Scalar& operator()(Index k) { return coeffRef(k); }                                             \
  const Scalar& operator()(Index k) const { return coeff(k); }                                    \
  Scalar& operator[](Index k) { return coeffRef(k); }                                             \
  const Scalar& operator[](Index k) const { return coeff(k); }                                    \
  Index lin_(Index k) const {                                                                     \
    if (cols() == 1) return k * rs_();                                                            \
    if (rows() == 1) return k * cs_();                                                            \
    return (k % rows()) * rs_() + (k / rows()) * cs_();                                           \
  }                                                                                               \
  Index innerStride() const { return rs_(); }                                                     \
  Index outerStride() const { return cs_(); }

// ---------------------------------------------------------------------------------------
// Shared member functions (views and owning matrices), via a mixin over the concrete type.
template <class Self, class S, int RC, int CC> struct DenseOps {
  Self& self() { return static_cast<Self&>(*this); }
  const Self& self() const { return static_cast<const Self&>(*this); }
  using Real = typename internal::real_of<S>::type;

  // --- views ----------------------------------------------------------------------------
  View<S, Dynamic, Dynamic> block(Index i, Index j, Index r, Index c) const {
    return View<S, Dynamic, Dynamic>(const_cast<S*>(&self().coeff(i, j)), r, c, self().rs_(), self().cs_());
  }
  template <int R2, int C2> View<S, R2, C2> block(Index i, Index j) const {
    return View<S, R2, C2>(const_cast<S*>(&self().coeff(i, j)), R2, C2, self().rs_(), self().cs_());
  }
  View<S, Dynamic, 1> col(Index j) const {
    return View<S, Dynamic, 1>(const_cast<S*>(self().ptr_() + j * self().cs_()), self().rows(), 1, self().rs_(), self().cs_());
  }
  View<S, 1, Dynamic> row(Index i) const {
    return View<S, 1, Dynamic>(const_cast<S*>(self().ptr_() + i * self().rs_()), 1, self().cols(), self().rs_(), self().cs_());
  }
  View<S, RC, Dynamic> leftCols(Index n) const {
    return View<S, RC, Dynamic>(const_cast<S*>(self().ptr_()), self().rows(), n, self().rs_(), self().cs_());
  }
  View<S, RC, Dynamic> rightCols(Index n) const {
    return View<S, RC, Dynamic>(const_cast<S*>(self().ptr_() + (self().cols() - n) * self().cs_()), self().rows(), n,
                                self().rs_(), self().cs_());
  }
  View<S, RC, Dynamic> middleCols(Index j, Index n) const {
    return View<S, RC, Dynamic>(const_cast<S*>(self().ptr_() + j * self().cs_()), self().rows(), n, self().rs_(), self().cs_());
  }
  View<S, Dynamic, CC> topRows(Index n) const {
    return View<S, Dynamic, CC>(const_cast<S*>(self().ptr_()), n, self().cols(), self().rs_(), self().cs_());
  }
  View<S, Dynamic, CC> bottomRows(Index n) const {
    return View<S, Dynamic, CC>(const_cast<S*>(self().ptr_() + (self().rows() - n) * self().rs_()), n, self().cols(),
                                self().rs_(), self().cs_());
  }
  View<S, Dynamic, CC> middleRows(Index i, Index n) const {
    return View<S, Dynamic, CC>(const_cast<S*>(self().ptr_() + i * self().rs_()), n, self().cols(), self().rs_(), self().cs_());
  }
  View<S, Dynamic, Dynamic> topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }
  auto segment(Index i, Index n) const { return vec_view(i, n); }
  auto head(Index n) const { return vec_view(0, n); }
  auto tail(Index n) const { return vec_view(self().size() - n, n); }
  View<S, Dynamic, 1> diagonal() const {
    return View<S, Dynamic, 1>(const_cast<S*>(self().ptr_()), std::min(self().rows(), self().cols()), 1,
                               self().rs_() + self().cs_(), 0);
  }
  View<S, CC, RC> transpose() const {
    return View<S, CC, RC>(const_cast<S*>(self().ptr_()), self().cols(), self().rows(), self().cs_(), self().rs_());
  }
  auto real() const {
    if constexpr (internal::is_cplx<S>::value) {
      return View<Real, RC, CC>(reinterpret_cast<Real*>(const_cast<S*>(self().ptr_())), self().rows(), self().cols(),
                                2 * self().rs_(), 2 * self().cs_());
    } else {
      return View<S, RC, CC>(const_cast<S*>(self().ptr_()), self().rows(), self().cols(), self().rs_(), self().cs_());
    }
  }
  auto imag() const {
    if constexpr (internal::is_cplx<S>::value) {
      return View<Real, RC, CC>(reinterpret_cast<Real*>(const_cast<S*>(self().ptr_())) + 1, self().rows(), self().cols(),
                                2 * self().rs_(), 2 * self().cs_());
    } else {
      return Matrix<S, RC, CC>::Zero(self().rows(), self().cols());
    }
  }

  // --- evaluation -----------------------------------------------------------------------
  Matrix<S, RC, CC> eval() const { return Matrix<S, RC, CC>(self()); }
  template <class D> Matrix<D, RC, CC> cast() const {
    Matrix<D, RC, CC> out(self().rows(), self().cols());
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) out(i, j) = internal::cast_<S, D>(self().coeff(i, j));
    return out;
  }
  template <class F> auto unary_(F f) const {
    using R = decltype(f(std::declval<S>()));
    Matrix<R, RC, CC> out(self().rows(), self().cols());
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) out(i, j) = f(self().coeff(i, j));
    return out;
  }
  Matrix<Real, RC, CC> cwiseAbs() const { return unary_([](const S& v) -> Real { return std::abs(v); }); }
  Matrix<Real, RC, CC> cwiseAbs2() const { return unary_([](const S& v) -> Real { return internal::abs2_(v); }); }
  Matrix<S, RC, CC> cwiseSqrt() const { return unary_([](const S& v) -> S { return std::sqrt(v); }); }
  Matrix<S, RC, CC> cwiseInverse() const { return unary_([](const S& v) -> S { return S(1) / v; }); }
  Matrix<S, RC, CC> conjugate() const { return unary_([](const S& v) -> S { return internal::conj_(v); }); }
  Matrix<S, CC, RC> adjoint() const { return Matrix<S, CC, RC>(transpose()).conjugate(); }
  template <class O> auto cwiseProduct(const O& o) const {
    Matrix<internal::prod_t<S, typename O::Scalar>, RC, CC> out(self().rows(), self().cols());
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) out(i, j) = self().coeff(i, j) * o.coeff(i, j);
    return out;
  }
  template <class O> auto cwiseQuotient(const O& o) const {
    Matrix<internal::prod_t<S, typename O::Scalar>, RC, CC> out(self().rows(), self().cols());
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) out(i, j) = self().coeff(i, j) / o.coeff(i, j);
    return out;
  }
  template <class O> Matrix<S, RC, CC> cwiseMax(const O& o) const {
    Matrix<S, RC, CC> out(self().rows(), self().cols());
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) out(i, j) = std::max(self().coeff(i, j), o.coeff(i, j));
    return out;
  }
  template <class O> Matrix<S, RC, CC> cwiseMin(const O& o) const {
    Matrix<S, RC, CC> out(self().rows(), self().cols());
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) out(i, j) = std::min(self().coeff(i, j), o.coeff(i, j));
    return out;
  }

  // --- reductions -----------------------------------------------------------------------
  S sum() const {
    S acc = S(0);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) acc += self().coeff(i, j);
    return acc;
  }
  S prod() const {
    S acc = S(1);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) acc *= self().coeff(i, j);
    return acc;
  }
  S mean() const { return sum() / S(Real(self().size())); }
  S trace() const {
    S acc = S(0);
    for (Index i = 0; i < std::min(self().rows(), self().cols()); ++i) acc += self().coeff(i, i);
    return acc;
  }
  Real squaredNorm() const {
    Real acc = 0;
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) acc += internal::abs2_(self().coeff(i, j));
    return acc;
  }
  Real norm() const { return std::sqrt(squaredNorm()); }
  Matrix<S, RC, CC> normalized() const {
    Matrix<S, RC, CC> out(self());
    const Real n = norm();
    if (n > 0) out /= S(n);
    return out;
  }
  void normalize() {
    const Real n = norm();
    if (n > 0) self() /= S(n);
  }
  template <int P> Real lpNorm() const {
    Real acc = 0;
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) {
        const Real a = std::abs(self().coeff(i, j));
        if constexpr (P == Infinity) acc = std::max(acc, a);
        else if constexpr (P == 1) acc += a;
        else acc += std::pow(a, Real(P));
      }
    if constexpr (P == Infinity || P == 1) return acc;
    else return std::pow(acc, Real(1) / Real(P));
  }
  S maxCoeff() const {
    S m = self().coeff(0, 0);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) m = std::max(m, self().coeff(i, j));
    return m;
  }
  S minCoeff() const {
    S m = self().coeff(0, 0);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) m = std::min(m, self().coeff(i, j));
    return m;
  }
  template <class I> S maxCoeff(I* idx) const {
    Index best = 0;
    for (Index k = 1; k < self().size(); ++k)
      if (self().coeff(k) > self().coeff(best)) best = k;
    *idx = static_cast<I>(best);
    return self().coeff(best);
  }
  template <class I> S minCoeff(I* idx) const {
    Index best = 0;
    for (Index k = 1; k < self().size(); ++k)
      if (self().coeff(k) < self().coeff(best)) best = k;
    *idx = static_cast<I>(best);
    return self().coeff(best);
  }
  // Hermitian inner product: conj(this) . other (Eigen's dot()).
  template <class O> auto dot(const O& o) const {
    using R = internal::prod_t<S, typename O::Scalar>;
    if (self().size() != o.size()) throw std::invalid_argument("Eigen shim: dot size mismatch");
    R acc = R(0);
    for (Index k = 0; k < self().size(); ++k) acc += internal::conj_(self().coeff(k)) * o.coeff(k);
    return acc;
  }
  bool allFinite() const {
    for (Index k = 0; k < self().size(); ++k)
      if (!std::isfinite(std::abs(self().coeff(k)))) return false;
    return true;
  }
  bool hasNaN() const {
    for (Index k = 0; k < self().size(); ++k)
      if (std::isnan(std::abs(self().coeff(k)))) return true;
    return false;
  }
  template <class O> bool isApprox(const O& o, Real prec = Real(1e-12)) const {
    Real d = 0;
    for (Index k = 0; k < self().size(); ++k) d += internal::abs2_(self().coeff(k) - o.coeff(k));
    return std::sqrt(d) <= prec * std::min(norm(), Matrix<typename O::Scalar, Dynamic, Dynamic>(o).norm());
  }

  // --- in-place -------------------------------------------------------------------------
  Self& setZero() { return setConstant(S(0)); }
  Self& setOnes() { return setConstant(S(1)); }
  Self& setConstant(const S& v) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = v;
    return self();
  }
  void fill(const S& v) { setConstant(v); }
  Self& setIdentity() {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) = S(i == j ? 1 : 0);
    return self();
  }
  template <class O> Self& operator+=(const O& o) {
    const Matrix<typename O::Scalar, Dynamic, Dynamic> t(o);  // alias-safe
    check_same_(t);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) += t(i, j);
    return self();
  }
  template <class O> Self& operator-=(const O& o) {
    const Matrix<typename O::Scalar, Dynamic, Dynamic> t(o);
    check_same_(t);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) -= t(i, j);
    return self();
  }
  template <class X, std::enable_if_t<internal::is_scalar_v<X>, int> = 0> Self& operator*=(const X& a) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) *= a;
    return self();
  }
  template <class X, std::enable_if_t<internal::is_scalar_v<X>, int> = 0> Self& operator/=(const X& a) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) self().coeffRef(i, j) /= a;
    return self();
  }
  CommaInit<View<S, RC, CC>> operator<<(const S& v) {
    return CommaInit<View<S, RC, CC>>(
        View<S, RC, CC>(self().ptr_(), self().rows(), self().cols(), self().rs_(), self().cs_()), v);
  }
  template <class D, std::enable_if_t<is_dense<D>::value, int> = 0> CommaInit<View<S, RC, CC>> operator<<(const D& b) {
    return CommaInit<View<S, RC, CC>>(
        View<S, RC, CC>(self().ptr_(), self().rows(), self().cols(), self().rs_(), self().cs_()), b);
  }

  template <class T> void check_same_(const T& t) const {
    if (t.rows() != self().rows() || t.cols() != self().cols())
      throw std::invalid_argument("Eigen shim: shape mismatch in compound assignment");
  }

 private:
  auto vec_view(Index i, Index n) const {
    if (self().cols() == 1 || RC != 1)
      return View<S, RC == 1 ? 1 : Dynamic, RC == 1 ? Dynamic : 1>(const_cast<S*>(self().ptr_() + i * (RC == 1 ? self().cs_() : self().rs_())),
                                                                   RC == 1 ? 1 : n, RC == 1 ? n : 1, self().rs_(),
                                                                   self().cs_());
    return View<S, RC == 1 ? 1 : Dynamic, RC == 1 ? Dynamic : 1>(const_cast<S*>(self().ptr_() + i * self().cs_()), 1, n,
                                                                 self().rs_(), self().cs_());
  }
};

// ---------------------------------------------------------------------------------------
// Non-owning strided view (block, segment, column, transpose, real/imag part, diagonal).
template <class S, int RC, int CC> class View : public DenseBase<View<S, RC, CC>>, public DenseOps<View<S, RC, CC>, S, RC, CC> {
 public:
  EIGEN_SHIM_DENSE_COMMON(S, RC, CC)
  using DenseOps<View, S, RC, CC>::operator<<;
  View(S* p, Index r, Index c, Index rs, Index cs) : p_(p), r_(r), c_(c), rs__(rs), cs__(cs) {}
  View(const View&) = default;

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  S* ptr_() const { return p_; }
  Index rs_() const { return rs__; }
  Index cs_() const { return cs__; }
  S* data() const { return p_; }

  View& operator=(const View& o) { return assign_(o); }
  template <class O, std::enable_if_t<is_dense<O>::value, int> = 0> View& operator=(const O& o) { return assign_(o); }

 private:
  template <class O> View& assign_(const O& o) {
    const Matrix<typename O::Scalar, Dynamic, Dynamic> t(o);  // alias-safe
    if (t.rows() != r_ || t.cols() != c_) throw std::invalid_argument("Eigen shim: shape mismatch in block assignment");
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) coeffRef(i, j) = static_cast<S>(t(i, j));
    return *this;
  }
  S* p_;
  Index r_, c_, rs__, cs__;
};

// ---------------------------------------------------------------------------------------
// Owning column-major matrix / vector.
template <class S, int RC, int CC, int Opt, int MR, int MC>
class Matrix : public DenseBase<Matrix<S, RC, CC, Opt, MR, MC>>, public DenseOps<Matrix<S, RC, CC, Opt, MR, MC>, S, RC, CC> {
 public:
  EIGEN_SHIM_DENSE_COMMON(S, RC, CC)
  using DenseOps<Matrix, S, RC, CC>::operator<<;

  Matrix() : r_(RC == Dynamic ? 0 : RC), c_(CC == Dynamic ? 0 : CC), v_(static_cast<std::size_t>(r_ * c_)) {}
  // Matrix(n): vector of length n (Eigen semantics for vector types)
  explicit Matrix(Index n) {
    if constexpr (CC == 1) init_(n, 1);
    else if constexpr (RC == 1) init_(1, n);
    else init_(n, n);  // not valid Eigen; never used by the reference
  }
  Matrix(Index r, Index c) { init_(r, c); }
  Matrix(int r, int c) { init_(r, c); }
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) noexcept = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) noexcept = default;

  template <class O, std::enable_if_t<is_dense<O>::value, int> = 0> Matrix(const O& o) { assign_(o); }
  template <class O, std::enable_if_t<is_dense<O>::value, int> = 0> Matrix& operator=(const O& o) {
    if constexpr (std::is_same_v<O, Matrix>) {
      if (&o == this) return *this;
    }
    Matrix tmp;
    tmp.assign_(o);
    *this = std::move(tmp);
    return *this;
  }
  // dense from sparse (DenseMatrix<T>(sparse))
  template <class T2, int O2, class SI2> Matrix(const SparseMatrix<T2, O2, SI2>& sp);

  static Matrix Zero() { Matrix m; m.setZero(); return m; }
  static Matrix Zero(Index n) { Matrix m(n); m.setZero(); return m; }
  static Matrix Zero(Index r, Index c) { Matrix m(r, c); m.setZero(); return m; }
  static Matrix Ones() { Matrix m; m.setOnes(); return m; }
  static Matrix Ones(Index n) { Matrix m(n); m.setOnes(); return m; }
  static Matrix Ones(Index r, Index c) { Matrix m(r, c); m.setOnes(); return m; }
  static Matrix Constant(Index n, const S& v) { Matrix m(n); m.setConstant(v); return m; }
  static Matrix Constant(Index r, Index c, const S& v) { Matrix m(r, c); m.setConstant(v); return m; }
  static Matrix Identity() { Matrix m; m.setIdentity(); return m; }
  static Matrix Identity(Index r, Index c) { Matrix m(r, c); m.setIdentity(); return m; }
  static Matrix Unit(Index n, Index i) { Matrix m = Zero(n); m(i) = S(1); return m; }
  static Matrix LinSpaced(Index n, const S& lo, const S& hi) {
    Matrix m(n);
    for (Index k = 0; k < n; ++k) m(k) = n > 1 ? lo + (hi - lo) * S(double(k) / double(n - 1)) : hi;
    return m;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  S* ptr_() const { return const_cast<S*>(v_.data()); }
  Index rs_() const { return 1; }
  Index cs_() const { return r_; }
  S* data() { return v_.data(); }
  const S* data() const { return v_.data(); }

  void resize(Index n) {
    if constexpr (CC == 1) init_(n, 1);
    else if constexpr (RC == 1) init_(1, n);
    else init_(n, n);
  }
  void resize(Index r, Index c) { init_(r, c); }
  void conservativeResize(Index n) {
    Matrix m(n);
    m.setZero();
    for (Index k = 0; k < std::min(n, this->size()); ++k) m(k) = (*this)(k);
    *this = std::move(m);
  }
  void conservativeResize(Index r, Index c) {
    Matrix m(r, c);
    m.setZero();
    for (Index j = 0; j < std::min(c, c_); ++j)
      for (Index i = 0; i < std::min(r, r_); ++i) m(i, j) = (*this)(i, j);
    *this = std::move(m);
  }
  void swap(Matrix& o) { std::swap(r_, o.r_); std::swap(c_, o.c_); v_.swap(o.v_); }

 private:
  template <class, int, int, int, int, int> friend class Matrix;
  void init_(Index r, Index c) {
    if (r < 0 || c < 0) throw std::invalid_argument("Eigen shim: negative dimension");
    r_ = r;
    c_ = c;
    v_.assign(static_cast<std::size_t>(r * c), S());
  }
  template <class O> void assign_(const O& o) {
    init_(o.rows(), o.cols());
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) v_[static_cast<std::size_t>(i + j * r_)] = static_cast<S>(o.coeff(i, j));
  }
  Index r_ = 0, c_ = 0;
  std::vector<S> v_;
};

// ---------------------------------------------------------------------------------------
// Arithmetic (eager).
template <class A, class B, class F> auto binary_(const A& a, const B& b, F f) {
  using R = decltype(f(std::declval<typename A::Scalar>(), std::declval<typename B::Scalar>()));
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::invalid_argument("Eigen shim: shape mismatch");
  Matrix<R, internal::pick(A::RowsAtCompileTime, B::RowsAtCompileTime), internal::pick(A::ColsAtCompileTime, B::ColsAtCompileTime)>
      out(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out(i, j) = f(a.coeff(i, j), b.coeff(i, j));
  return out;
}
template <class A, class B, std::enable_if_t<is_dense<A>::value && is_dense<B>::value, int> = 0>
auto operator+(const A& a, const B& b) {
  return binary_(a, b, [](const auto& x, const auto& y) { return x + y; });
}
template <class A, class B, std::enable_if_t<is_dense<A>::value && is_dense<B>::value, int> = 0>
auto operator-(const A& a, const B& b) {
  return binary_(a, b, [](const auto& x, const auto& y) { return x - y; });
}
template <class A, std::enable_if_t<is_dense<A>::value, int> = 0> auto operator-(const A& a) {
  return a.unary_([](const auto& x) { return -x; });
}
template <class X, class A, std::enable_if_t<internal::is_scalar_v<X> && is_dense<A>::value, int> = 0>
auto operator*(const X& s, const A& a) {
  return a.unary_([s](const auto& x) { return s * x; });
}
template <class A, class X, std::enable_if_t<internal::is_scalar_v<X> && is_dense<A>::value, int> = 0>
auto operator*(const A& a, const X& s) {
  return a.unary_([s](const auto& x) { return x * s; });
}
template <class A, class X, std::enable_if_t<internal::is_scalar_v<X> && is_dense<A>::value, int> = 0>
auto operator/(const A& a, const X& s) {
  return a.unary_([s](const auto& x) { return x / s; });
}
template <class A, class B, std::enable_if_t<is_dense<A>::value && is_dense<B>::value, int> = 0>
auto operator*(const A& a, const B& b) {
  using R = internal::prod_t<typename A::Scalar, typename B::Scalar>;
  if (a.cols() != b.rows()) throw std::invalid_argument("Eigen shim: product dimension mismatch");
  Matrix<R, A::RowsAtCompileTime, B::ColsAtCompileTime> out(a.rows(), b.cols());
  out.setZero();
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k) {
      const auto bkj = b.coeff(k, j);
      if (bkj == typename B::Scalar(0)) continue;
      for (Index i = 0; i < a.rows(); ++i) out(i, j) += a.coeff(i, k) * bkj;
    }
  return out;
}
template <class A, class B, std::enable_if_t<is_dense<A>::value && is_dense<B>::value, int> = 0>
bool operator==(const A& a, const B& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i)
      if (!(a.coeff(i, j) == b.coeff(i, j))) return false;
  return true;
}
template <class A, class B, std::enable_if_t<is_dense<A>::value && is_dense<B>::value, int> = 0>
bool operator!=(const A& a, const B& b) {
  return !(a == b);
}

// ---------------------------------------------------------------------------------------
// Sparse (compressed column storage).
template <class S, class SI = int> class Triplet {
 public:
  Triplet() : r_(0), c_(0), v_(0) {}
  Triplet(const SI& r, const SI& c, const S& v = S(0)) : r_(r), c_(c), v_(v) {}
  const SI& row() const { return r_; }
  const SI& col() const { return c_; }
  const S& value() const { return v_; }

 private:
  SI r_, c_;
  S v_;
};

template <class S, int Opt, class SI> class SparseMatrix {
 public:
  using Scalar = S;
  using StorageIndex = SI;
  using RealScalar = typename internal::real_of<S>::type;

  SparseMatrix() : colptr_(1, 0) {}
  SparseMatrix(Index r, Index c) { resize(r, c); }
  template <class D, std::enable_if_t<is_dense<D>::value, int> = 0> explicit SparseMatrix(const D& d) {
    std::vector<Triplet<S, SI>> t;
    for (Index j = 0; j < d.cols(); ++j)
      for (Index i = 0; i < d.rows(); ++i)
        if (d.coeff(i, j) != S(0)) t.emplace_back(SI(i), SI(j), S(d.coeff(i, j)));
    resize(d.rows(), d.cols());
    setFromTriplets(t.begin(), t.end());
  }

  void resize(Index r, Index c) {
    rows_ = r;
    cols_ = c;
    colptr_.assign(static_cast<std::size_t>(c + 1), SI(0));
    rowidx_.clear();
    vals_.clear();
  }
  void setZero() { resize(rows_, cols_); }
  template <class It> void setFromTriplets(It first, It last) {
    std::vector<std::pair<std::pair<Index, Index>, S>> t;  // (col,row),value
    for (It it = first; it != last; ++it) {
      const Index r = it->row(), c = it->col();
      if (r < 0 || r >= rows_ || c < 0 || c >= cols_) throw std::invalid_argument("Eigen shim: triplet out of range");
      t.push_back({{c, r}, S(it->value())});
    }
    std::stable_sort(t.begin(), t.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    colptr_.assign(static_cast<std::size_t>(cols_ + 1), SI(0));
    rowidx_.clear();
    vals_.clear();
    for (std::size_t k = 0; k < t.size();) {
      const auto key = t[k].first;
      S v = t[k].second;
      std::size_t m = k + 1;
      for (; m < t.size() && t[m].first == key; ++m) v += t[m].second;  // duplicates are summed
      rowidx_.push_back(SI(key.second));
      vals_.push_back(v);
      colptr_[static_cast<std::size_t>(key.first + 1)]++;
      k = m;
    }
    for (Index c = 0; c < cols_; ++c) colptr_[c + 1] += colptr_[c];
  }
  void makeCompressed() {}
  bool isCompressed() const { return true; }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index nonZeros() const { return static_cast<Index>(vals_.size()); }
  Index outerSize() const { return cols_; }
  S coeff(Index i, Index j) const {
    for (SI k = colptr_[j]; k < colptr_[j + 1]; ++k)
      if (rowidx_[k] == i) return vals_[k];
    return S(0);
  }
  const SI* outerIndexPtr() const { return colptr_.data(); }
  const SI* innerIndexPtr() const { return rowidx_.data(); }
  const S* valuePtr() const { return vals_.data(); }

  // Lazy transpose (like Eigen's): products A^T x run straight off the CSC arrays; the view
  // converts to a materialised SparseMatrix where one is needed.
  class TransposeView {
   public:
    explicit TransposeView(const SparseMatrix& a) : a_(a) {}
    operator SparseMatrix() const { return a_.transposed(); }
    Index rows() const { return a_.cols(); }
    Index cols() const { return a_.rows(); }
    const SparseMatrix& nested() const { return a_; }
    // y = A^T x with A in CSC: y[c] = the dot of column c of A with x
    template <class D, std::enable_if_t<is_dense<D>::value, int> = 0>
    friend auto operator*(const TransposeView& at, const D& x) {
      const SparseMatrix& a = at.a_;
      using R = internal::prod_t<S, typename D::Scalar>;
      if (a.rows() != x.rows()) throw std::invalid_argument("Eigen shim: sparse product dimension mismatch");
      Matrix<R, Dynamic, D::ColsAtCompileTime> y(a.cols(), x.cols());
      for (Index j = 0; j < x.cols(); ++j)
        for (Index c = 0; c < a.cols(); ++c) {
          R acc = R(0);
          for (SI k = a.colptr_[c]; k < a.colptr_[c + 1]; ++k) acc += a.vals_[k] * x.coeff(a.rowidx_[k], j);
          y(c, j) = acc;
        }
      return y;
    }

   private:
    const SparseMatrix& a_;
  };
  TransposeView transpose() const { return TransposeView(*this); }
  SparseMatrix transposed() const {
    std::vector<Triplet<S, SI>> t;
    t.reserve(vals_.size());
    for (Index c = 0; c < cols_; ++c)
      for (SI k = colptr_[c]; k < colptr_[c + 1]; ++k) t.emplace_back(SI(c), rowidx_[k], vals_[k]);
    SparseMatrix out(cols_, rows_);
    out.setFromTriplets(t.begin(), t.end());
    return out;
  }
  SparseMatrix adjoint() const {
    SparseMatrix out = transposed();
    for (auto& v : out.vals_) v = internal::conj_(v);
    return out;
  }
  template <class D> SparseMatrix<D, Opt, SI> cast() const {
    SparseMatrix<D, Opt, SI> out;
    std::vector<Triplet<D, SI>> t;
    for (Index c = 0; c < cols_; ++c)
      for (SI k = colptr_[c]; k < colptr_[c + 1]; ++k) t.emplace_back(rowidx_[k], SI(c), internal::cast_<S, D>(vals_[k]));
    out.resize(rows_, cols_);
    out.setFromTriplets(t.begin(), t.end());
    return out;
  }
  Matrix<S, Dynamic, Dynamic> toDense() const { return Matrix<S, Dynamic, Dynamic>(*this); }
  RealScalar norm() const {
    RealScalar a = 0;
    for (const auto& v : vals_) a += internal::abs2_(v);
    return std::sqrt(a);
  }

 private:
  template <class, int, class> friend class SparseMatrix;
  Index rows_ = 0, cols_ = 0;
  std::vector<SI> colptr_, rowidx_;
  std::vector<S> vals_;
};

template <class S, int RC, int CC, int Opt, int MR, int MC>
template <class T2, int O2, class SI2>
Matrix<S, RC, CC, Opt, MR, MC>::Matrix(const SparseMatrix<T2, O2, SI2>& sp) {
  init_(sp.rows(), sp.cols());
  const SI2* cp = sp.outerIndexPtr();
  const SI2* ri = sp.innerIndexPtr();
  const T2* vv = sp.valuePtr();
  for (Index c = 0; c < sp.cols(); ++c)
    for (SI2 k = cp[c]; k < cp[c + 1]; ++k) (*this)(ri[k], c) = static_cast<S>(vv[k]);
}

template <class S, int O, class SI, class D, std::enable_if_t<is_dense<D>::value, int> = 0>
auto operator*(const SparseMatrix<S, O, SI>& a, const D& x) {
  using R = internal::prod_t<S, typename D::Scalar>;
  if (a.cols() != x.rows()) throw std::invalid_argument("Eigen shim: sparse product dimension mismatch");
  Matrix<R, Dynamic, D::ColsAtCompileTime> y(a.rows(), x.cols());
  y.setZero();
  const SI* cp = a.outerIndexPtr();
  const SI* ri = a.innerIndexPtr();
  const S* vv = a.valuePtr();
  for (Index j = 0; j < x.cols(); ++j)
    for (Index c = 0; c < a.cols(); ++c) {
      const auto xc = x.coeff(c, j);
      for (SI k = cp[c]; k < cp[c + 1]; ++k) y(ri[k], j) += vv[k] * xc;
    }
  return y;
}
template <class X, class S, int O, class SI, std::enable_if_t<internal::is_scalar_v<X>, int> = 0>
SparseMatrix<S, O, SI> operator*(const X& s, const SparseMatrix<S, O, SI>& a) {
  SparseMatrix<S, O, SI> out = a;
  auto* vv = const_cast<S*>(out.valuePtr());
  for (Index k = 0; k < out.nonZeros(); ++k) vv[k] = S(s) * vv[k];
  return out;
}

// ---------------------------------------------------------------------------------------
// Dense LU with partial pivoting (row interchanges): P A = L U, L unit lower.
template <class M> class PartialPivLU {
 public:
  using Scalar = typename M::Scalar;
  using Real = typename internal::real_of<Scalar>::type;
  PartialPivLU() = default;
  template <class D> explicit PartialPivLU(const D& a) { compute(a); }
  template <class D> PartialPivLU& compute(const D& a) {
    lu_ = Matrix<Scalar, Dynamic, Dynamic>(a);
    const Index n = lu_.rows();
    if (lu_.cols() != n) throw std::invalid_argument("Eigen shim: PartialPivLU needs a square matrix");
    perm_.resize(static_cast<std::size_t>(n));
    for (Index i = 0; i < n; ++i) perm_[i] = i;
    Scalar* A = lu_.data();
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      Real best = std::abs(A[k + k * n]);
      for (Index i = k + 1; i < n; ++i) {
        const Real v = std::abs(A[i + k * n]);
        if (v > best) { best = v; p = i; }
      }
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(A[k + j * n], A[p + j * n]);
        std::swap(perm_[k], perm_[p]);
      }
      const Scalar piv = A[k + k * n];
      if (piv == Scalar(0)) continue;  // singular column: leave it (caller checks the U diagonal)
      for (Index i = k + 1; i < n; ++i) A[i + k * n] /= piv;
      for (Index j = k + 1; j < n; ++j) {
        const Scalar ukj = A[k + j * n];
        if (ukj == Scalar(0)) continue;
        Scalar* cj = A + j * n;
        const Scalar* ck = A + k * n;
        for (Index i = k + 1; i < n; ++i) cj[i] -= ck[i] * ukj;
      }
    }
    return *this;
  }
  const Matrix<Scalar, Dynamic, Dynamic>& matrixLU() const { return lu_; }
  template <class D> Matrix<internal::prod_t<Scalar, typename D::Scalar>, Dynamic, D::ColsAtCompileTime> solve(const D& b) const {
    using R = internal::prod_t<Scalar, typename D::Scalar>;
    const Index n = lu_.rows();
    Matrix<R, Dynamic, D::ColsAtCompileTime> x(n, b.cols());
    const Scalar* A = lu_.data();
    for (Index c = 0; c < b.cols(); ++c) {
      for (Index i = 0; i < n; ++i) x(i, c) = b.coeff(perm_[i], c);
      R* xc = &x(0, c);
      for (Index k = 0; k < n; ++k) {
        const R v = xc[k];
        for (Index i = k + 1; i < n; ++i) xc[i] -= A[i + k * n] * v;
      }
      for (Index k = n - 1; k >= 0; --k) {
        xc[k] /= A[k + k * n];
        const R v = xc[k];
        for (Index i = 0; i < k; ++i) xc[i] -= A[i + k * n] * v;
      }
    }
    return x;
  }
  Scalar determinant() const {
    Scalar d = Scalar(1);
    for (Index i = 0; i < lu_.rows(); ++i) d *= lu_(i, i);
    Index swaps = 0;
    std::vector<Index> p = perm_;
    for (Index i = 0; i < Index(p.size()); ++i)
      while (p[i] != i) { std::swap(p[i], p[p[i]]); ++swaps; }
    return (swaps % 2) ? -d : d;
  }

 private:
  Matrix<Scalar, Dynamic, Dynamic> lu_;
  std::vector<Index> perm_;  // row i of P A is row perm_[i] of A
};
template <class M> using FullPivLU = PartialPivLU<M>;

// ---------------------------------------------------------------------------------------
// Sparse LU: banded LU with partial pivoting (LAPACK gbtf2 storage, natural order).
template <class M, class Ordering = void> class SparseLU {
 public:
  using Scalar = typename M::Scalar;
  using Real = typename internal::real_of<Scalar>::type;
  SparseLU() = default;
  explicit SparseLU(const M& a) { compute(a); }
  void analyzePattern(const M& a) {
    n_ = a.rows();
    kl_ = ku_ = 0;
    const auto* cp = a.outerIndexPtr();
    const auto* ri = a.innerIndexPtr();
    for (Index c = 0; c < a.cols(); ++c)
      for (auto k = cp[c]; k < cp[c + 1]; ++k) {
        kl_ = std::max<Index>(kl_, ri[k] - c);
        ku_ = std::max<Index>(ku_, c - ri[k]);
      }
    analyzed_ = true;
  }
  void factorize(const M& a) {
    if (!analyzed_) analyzePattern(a);
    if (a.rows() != a.cols()) { info_ = InvalidInput; return; }
    ld_ = 2 * kl_ + ku_ + 1;
    ab_.assign(static_cast<std::size_t>(ld_ * n_), Scalar(0));
    ipiv_.assign(static_cast<std::size_t>(n_), 0);
    const auto* cp = a.outerIndexPtr();
    const auto* ri = a.innerIndexPtr();
    const auto* vv = a.valuePtr();
    const Index kv = kl_ + ku_;
    for (Index c = 0; c < n_; ++c)
      for (auto k = cp[c]; k < cp[c + 1]; ++k) at(kv + ri[k] - c, c) += vv[k];
    info_ = Success;
    Index ju = 0;
    for (Index j = 0; j < n_; ++j) {
      const Index km = std::min(kl_, n_ - 1 - j);
      Index jp = 0;
      Real best = std::abs(at(kv, j));
      for (Index i = 1; i <= km; ++i) {
        const Real v = std::abs(at(kv + i, j));
        if (v > best) { best = v; jp = i; }
      }
      ipiv_[j] = j + jp;
      if (at(kv + jp, j) == Scalar(0)) { info_ = NumericalIssue; return; }
      ju = std::max(ju, std::min(j + ku_ + jp, n_ - 1));
      if (jp != 0)
        for (Index c = j; c <= ju; ++c) std::swap(at(kv + jp + j - c, c), at(kv + j - c, c));
      if (km > 0) {
        const Scalar inv = Scalar(1) / at(kv, j);
        for (Index i = 1; i <= km; ++i) at(kv + i, j) *= inv;
        for (Index c = j + 1; c <= ju; ++c) {
          const Scalar u = at(kv + j - c, c);
          if (u == Scalar(0)) continue;
          Scalar* dst = &at(kv + j + 1 - c, c);
          const Scalar* l = &at(kv + 1, j);
          for (Index i = 0; i < km; ++i) dst[i] -= l[i] * u;
        }
      }
    }
  }
  void compute(const M& a) {
    analyzePattern(a);
    factorize(a);
  }
  ComputationInfo info() const { return info_; }
  template <class D> Matrix<internal::prod_t<Scalar, typename D::Scalar>, Dynamic, D::ColsAtCompileTime> solve(const D& b) const {
    using R = internal::prod_t<Scalar, typename D::Scalar>;
    Matrix<R, Dynamic, D::ColsAtCompileTime> x(b);
    const Index kv = kl_ + ku_;
    for (Index c = 0; c < x.cols(); ++c) {
      R* xc = &x(0, c);
      for (Index j = 0; j < n_; ++j) {  // L: row interchanges + unit lower band
        const Index km = std::min(kl_, n_ - 1 - j);
        if (ipiv_[j] != j) std::swap(xc[j], xc[ipiv_[j]]);
        const R v = xc[j];
        for (Index i = 1; i <= km; ++i) xc[j + i] -= at(kv + i, j) * v;
      }
      for (Index j = n_ - 1; j >= 0; --j) {  // U: upper band of width kl+ku
        xc[j] /= at(kv, j);
        const R v = xc[j];
        const Index lo = std::max<Index>(0, j - kv);
        for (Index i = lo; i < j; ++i) xc[i] -= at(kv + i - j, j) * v;
      }
    }
    return x;
  }

 private:
  Scalar& at(Index r, Index c) { return ab_[static_cast<std::size_t>(r + c * ld_)]; }
  const Scalar& at(Index r, Index c) const { return ab_[static_cast<std::size_t>(r + c * ld_)]; }
  bool analyzed_ = false;
  Index n_ = 0, kl_ = 0, ku_ = 0, ld_ = 1;
  std::vector<Scalar> ab_;
  std::vector<Index> ipiv_;
  ComputationInfo info_ = InvalidInput;
};
template <class M> using SparseQR = SparseLU<M>;
template <class I> struct COLAMDOrdering {};
template <class I> struct AMDOrdering {};
template <class I> struct NaturalOrdering {};

// ---------------------------------------------------------------------------------------
// Sparse Cholesky (lower triangle of an SPD matrix): banded L L^T, natural order.
template <class M, int UpLo = Lower, class Ordering = void> class SimplicialLLT {
 public:
  using Scalar = typename M::Scalar;
  SimplicialLLT() = default;
  explicit SimplicialLLT(const M& a) { compute(a); }
  SimplicialLLT& compute(const M& a) {
    n_ = a.rows();
    kd_ = 0;
    const auto* cp = a.outerIndexPtr();
    const auto* ri = a.innerIndexPtr();
    const auto* vv = a.valuePtr();
    for (Index c = 0; c < n_; ++c)
      for (auto k = cp[c]; k < cp[c + 1]; ++k)
        if (ri[k] >= c) kd_ = std::max<Index>(kd_, ri[k] - c);
    ld_ = kd_ + 1;
    l_.assign(static_cast<std::size_t>(ld_ * n_), Scalar(0));
    for (Index c = 0; c < n_; ++c)
      for (auto k = cp[c]; k < cp[c + 1]; ++k)
        if (ri[k] >= c) l_[static_cast<std::size_t>((ri[k] - c) + c * ld_)] += vv[k];
    info_ = Success;
    for (Index j = 0; j < n_; ++j) {
      Scalar* cj = &l_[static_cast<std::size_t>(j * ld_)];
      const Scalar d = cj[0];
      if (!(std::real(d) > 0)) { info_ = NumericalIssue; return *this; }
      const Scalar ljj = std::sqrt(d);
      cj[0] = ljj;
      const Index m = std::min(kd_, n_ - 1 - j);
      for (Index i = 1; i <= m; ++i) cj[i] /= ljj;
      for (Index c = 1; c <= m; ++c) {  // trailing update of column j+c, rows j+c..j+m
        const Scalar lc = internal::conj_(cj[c]);
        Scalar* dst = &l_[static_cast<std::size_t>((j + c) * ld_)];
        const Scalar* src = cj + c;
        const Index len = m - c + 1;
        for (Index i = 0; i < len; ++i) dst[i] -= src[i] * lc;
      }
    }
    return *this;
  }
  void analyzePattern(const M&) {}
  void factorize(const M& a) { compute(a); }
  ComputationInfo info() const { return info_; }
  template <class D> Matrix<internal::prod_t<Scalar, typename D::Scalar>, Dynamic, D::ColsAtCompileTime> solve(const D& b) const {
    using R = internal::prod_t<Scalar, typename D::Scalar>;
    Matrix<R, Dynamic, D::ColsAtCompileTime> x(b);
    for (Index c = 0; c < x.cols(); ++c) {
      R* xc = &x(0, c);
      for (Index j = 0; j < n_; ++j) {
        const Scalar* cj = &l_[static_cast<std::size_t>(j * ld_)];
        xc[j] /= cj[0];
        const R v = xc[j];
        const Index m = std::min(kd_, n_ - 1 - j);
        for (Index i = 1; i <= m; ++i) xc[j + i] -= cj[i] * v;
      }
      for (Index j = n_ - 1; j >= 0; --j) {
        const Scalar* cj = &l_[static_cast<std::size_t>(j * ld_)];
        const Index m = std::min(kd_, n_ - 1 - j);
        R acc = xc[j];
        for (Index i = 1; i <= m; ++i) acc -= internal::conj_(cj[i]) * xc[j + i];
        xc[j] = acc / internal::conj_(cj[0]);
      }
    }
    return x;
  }

 private:
  Index n_ = 0, kd_ = 0, ld_ = 1;
  std::vector<Scalar> l_;
  ComputationInfo info_ = InvalidInput;
};
template <class M, int UpLo = Lower, class Ordering = void> using SimplicialLDLT = SimplicialLLT<M, UpLo, Ordering>;

// ---------------------------------------------------------------------------------------
// Dense Cholesky.
template <class M, int UpLo = Lower> class LLT {
 public:
  using Scalar = typename M::Scalar;
  LLT() = default;
  template <class D> explicit LLT(const D& a) { compute(a); }
  template <class D> LLT& compute(const D& a) {
    l_ = Matrix<Scalar, Dynamic, Dynamic>(a);
    const Index n = l_.rows();
    info_ = Success;
    for (Index j = 0; j < n; ++j) {
      Scalar d = l_(j, j);
      for (Index k = 0; k < j; ++k) d -= l_(j, k) * internal::conj_(l_(j, k));
      if (!(std::real(d) > 0)) { info_ = NumericalIssue; return *this; }
      const Scalar ljj = std::sqrt(d);
      l_(j, j) = ljj;
      for (Index i = j + 1; i < n; ++i) {
        Scalar s = l_(i, j);
        for (Index k = 0; k < j; ++k) s -= l_(i, k) * internal::conj_(l_(j, k));
        l_(i, j) = s / ljj;
      }
      for (Index i = 0; i < j; ++i) l_(i, j) = Scalar(0);
    }
    return *this;
  }
  ComputationInfo info() const { return info_; }
  Matrix<Scalar, Dynamic, Dynamic> matrixL() const { return l_; }
  template <class D> Matrix<internal::prod_t<Scalar, typename D::Scalar>, Dynamic, D::ColsAtCompileTime> solve(const D& b) const {
    using R = internal::prod_t<Scalar, typename D::Scalar>;
    Matrix<R, Dynamic, D::ColsAtCompileTime> x(b);
    const Index n = l_.rows();
    for (Index c = 0; c < x.cols(); ++c) {
      for (Index i = 0; i < n; ++i) {
        R s = x(i, c);
        for (Index k = 0; k < i; ++k) s -= l_(i, k) * x(k, c);
        x(i, c) = s / l_(i, i);
      }
      for (Index i = n - 1; i >= 0; --i) {
        R s = x(i, c);
        for (Index k = i + 1; k < n; ++k) s -= internal::conj_(l_(k, i)) * x(k, c);
        x(i, c) = s / internal::conj_(l_(i, i));
      }
    }
    return x;
  }

 private:
  Matrix<Scalar, Dynamic, Dynamic> l_;
  ComputationInfo info_ = InvalidInput;
};
template <class M, int UpLo = Lower> using LDLT = LLT<M, UpLo>;

// ---------------------------------------------------------------------------------------
// Symmetric eigenproblems (real), cyclic Jacobi; eigenvalues ascending.
template <class M> class SelfAdjointEigenSolver {
 public:
  SelfAdjointEigenSolver() = default;
  template <class D> explicit SelfAdjointEigenSolver(const D& a, int options = ComputeEigenvectors) { compute(a, options); }
  template <class D> SelfAdjointEigenSolver& compute(const D& a0, int = ComputeEigenvectors) {
    MatrixXd a(a0);
    const Index n = a.rows();
    MatrixXd v = MatrixXd::Identity(n, n);
    info_ = NoConvergence;
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0, tot = 0;
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) (i == j ? tot : off) += a(i, j) * a(i, j);
      if (off <= 1e-30 * (tot + off) || off == 0) { info_ = Success; break; }
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          if (a(p, q) == 0) continue;
          const double theta = (a(q, q) - a(p, p)) / (2 * a(p, q));
          const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1));
          const double c = 1 / std::sqrt(t * t + 1), s = t * c;
          for (Index k = 0; k < n; ++k) {
            const double akp = a(k, p), akq = a(k, q);
            a(k, p) = c * akp - s * akq;
            a(k, q) = s * akp + c * akq;
          }
          for (Index k = 0; k < n; ++k) {
            const double apk = a(p, k), aqk = a(q, k);
            a(p, k) = c * apk - s * aqk;
            a(q, k) = s * apk + c * aqk;
          }
          for (Index k = 0; k < n; ++k) {
            const double vkp = v(k, p), vkq = v(k, q);
            v(k, p) = c * vkp - s * vkq;
            v(k, q) = s * vkp + c * vkq;
          }
        }
    }
    std::vector<Index> ord(static_cast<std::size_t>(n));
    for (Index i = 0; i < n; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](Index x, Index y) { return a(x, x) < a(y, y); });
    ev_.resize(n);
    vec_.resize(n, n);
    for (Index k = 0; k < n; ++k) {
      ev_(k) = a(ord[k], ord[k]);
      for (Index i = 0; i < n; ++i) vec_(i, k) = v(i, ord[k]);
    }
    return *this;
  }
  ComputationInfo info() const { return info_; }
  const VectorXd& eigenvalues() const { return ev_; }
  const MatrixXd& eigenvectors() const { return vec_; }

 protected:
  VectorXd ev_;
  MatrixXd vec_;
  ComputationInfo info_ = InvalidInput;
};

template <class M> class GeneralizedSelfAdjointEigenSolver : public SelfAdjointEigenSolver<M> {
 public:
  template <class DA, class DB>
  GeneralizedSelfAdjointEigenSolver(const DA& a, const DB& b, int options = ComputeEigenvectors | Ax_lBx) {
    compute(a, b, options);
  }
  template <class DA, class DB> GeneralizedSelfAdjointEigenSolver& compute(const DA& a, const DB& b, int = 0) {
    LLT<MatrixXd> llt{MatrixXd(b)};
    if (llt.info() != Success) { this->info_ = NumericalIssue; return *this; }
    const MatrixXd l = llt.matrixL();
    const Index n = l.rows();
    MatrixXd c(a);  // C = L^-1 A L^-T
    for (Index j = 0; j < n; ++j)  // L^-1 A (forward substitution per column)
      for (Index i = 0; i < n; ++i) {
        double s = c(i, j);
        for (Index k = 0; k < i; ++k) s -= l(i, k) * c(k, j);
        c(i, j) = s / l(i, i);
      }
    for (Index i = 0; i < n; ++i)  // (L^-1 A) L^-T: forward substitution per row
      for (Index j = 0; j < n; ++j) {
        double s = c(i, j);
        for (Index k = 0; k < j; ++k) s -= c(i, k) * l(j, k);
        c(i, j) = s / l(j, j);
      }
    SelfAdjointEigenSolver<M>::compute(MatrixXd((c + c.transpose()) * 0.5));
    for (Index k = 0; k < n; ++k)  // x = L^-T y
      for (Index i = n - 1; i >= 0; --i) {
        double s = this->vec_(i, k);
        for (Index m = i + 1; m < n; ++m) s -= l(m, i) * this->vec_(m, k);
        this->vec_(i, k) = s / l(i, i);
      }
    return *this;
  }
};

}  // namespace Eigen
