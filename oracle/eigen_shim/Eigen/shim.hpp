// ORACLE — test infrastructure only.  A minimal stand-in for the subset of
// Eigen 3.4 the reference's material.cpp, rom.cpp, store.cpp and mesh.cpp
// use, so oracle/_ref can compile those files UNCHANGED from
// /root/reference/proj/src (Eigen itself is not installed).
//
// Written for this repo (not Eigen source).  Everything is evaluated eagerly
// into plain column-major storage.  Where Eigen's evaluation order decides
// result bits on the reference's hot path it is reproduced:
//   * fixed-size 2x2 products are two-term sums (Eigen's lazy coefficient
//     product; the order of two terms is immaterial);
//   * sum-reductions (squaredNorm, norm, sum, dot) follow Eigen's SSE2
//     LinearVectorizedTraversal: two packet accumulators of 2 doubles over
//     blocks of 4, combined, horizontally added, then the scalar tail —
//     e.g. ||F||^2 = (F00^2 + F01^2) + (F10^2 + F11^2);
//   * normalized() divides by sqrt(squaredNorm) (Eigen 3.4), inverse() of a
//     2x2 is cofactors times RN(1/det) with det = a00 a11 - a10 a01;
//   * scalar * matrix and matrix / scalar are per-coefficient products /
//     quotients.
// Dynamic-size products (GEMV/GEMM) use a plain sequential k order and
// PartialPivLU is the unblocked algorithm: NOT Eigen's blocked kernels, so
// results of those agree with the reference to rounding only (the ROM
// paths are compared at the BASELINE tolerance, never bitwise).
#pragma once

#include <array>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <map>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;

template <typename T, int R, int C>
class Matrix;
template <typename M, int BR, int BC>
class Block;

namespace internal {

template <typename T, int N>
struct Storage {
  std::array<T, N> a{};
  T* p() { return a.data(); }
  const T* p() const { return a.data(); }
  void resize(Index n) {
    if (n != N) throw std::logic_error("Eigen shim: resizing a fixed-size matrix");
  }
};
template <typename T>
struct Storage<T, -1> {
  std::vector<T> a;
  T* p() { return a.data(); }
  const T* p() const { return a.data(); }
  void resize(Index n) { a.assign((size_t)n, T(0)); }
};

constexpr int prod_size(int r, int c) { return (r > 0 && c > 0) ? r * c : -1; }

// Eigen's SSE2 (packet of 2 doubles) linear vectorized sum-reduction order.
template <typename T, typename F>
T redux_sum(Index n, F v) {
  if (n <= 0) return T(0);
  const Index n1 = (n / 2) * 2, n2 = (n / 4) * 4;
  if (n1 == 0) {
    T r = v(0);
    for (Index i = 1; i < n; ++i) r = r + v(i);
    return r;
  }
  T p0a = v(0), p0b = v(1);
  if (n1 > 2) {
    T p1a = v(2), p1b = v(3);
    for (Index i = 4; i < n2; i += 4) {
      p0a = p0a + v(i);
      p0b = p0b + v(i + 1);
      p1a = p1a + v(i + 2);
      p1b = p1b + v(i + 3);
    }
    p0a = p0a + p1a;
    p0b = p0b + p1b;
    if (n1 > n2) {
      p0a = p0a + v(n2);
      p0b = p0b + v(n2 + 1);
    }
  }
  T r = p0a + p0b;
  for (Index i = n1; i < n; ++i) r = r + v(i);
  return r;
}

template <typename X>
struct traits;
template <typename T, int R, int C>
struct traits<Matrix<T, R, C>> {
  using Scalar = T;
  static constexpr int Rows = R, Cols = C;
};
template <typename M, int BR, int BC>
struct traits<Block<M, BR, BC>> {
  using Scalar = typename std::remove_const<M>::type::Scalar;
  static constexpr int Rows = BR, Cols = BC;
};

template <typename X>
struct is_mat : std::false_type {};
template <typename T, int R, int C>
struct is_mat<Matrix<T, R, C>> : std::true_type {};
template <typename M, int BR, int BC>
struct is_mat<Block<M, BR, BC>> : std::true_type {};

}  // namespace internal

template <typename M>
class PartialPivLU;

// Comma initializer: fills row by row (Eigen semantics for scalars).
template <typename M>
struct CommaInit {
  M& m;
  Index k;
  CommaInit& operator,(typename M::Scalar v) {
    const Index r = k / m.cols(), c = k % m.cols();
    m(r, c) = v;
    ++k;
    return *this;
  }
};

template <typename T, int R, int C>
class Matrix {
 public:
  using Scalar = T;
  static constexpr int RowsAtCompileTime = R, ColsAtCompileTime = C;

  Matrix() : rows_(R > 0 ? R : 0), cols_(C > 0 ? C : 0) { s_.resize(rows_ * cols_); }
  // (rows, cols) for dynamic shapes; coefficients for fixed 2-vectors.
  template <typename A, typename B,
            typename std::enable_if<std::is_integral<A>::value && std::is_integral<B>::value &&
                                        !(R * C == 2 && R > 0),
                                    int>::type = 0>
  Matrix(A r, B c) : rows_(R > 0 ? R : (Index)r), cols_(C > 0 ? C : (Index)c) {
    if ((R > 0 && r != R) || (C > 0 && c != C)) throw std::logic_error("Eigen shim: bad shape");
    s_.resize(rows_ * cols_);
  }
  template <typename A, typename B,
            typename std::enable_if<(R * C == 2 && R > 0) && std::is_arithmetic<A>::value &&
                                        std::is_arithmetic<B>::value,
                                    int>::type = 0>
  Matrix(A x, B y) : rows_(R), cols_(C) {
    s_.p()[0] = (T)x;
    s_.p()[1] = (T)y;
  }
  // (size) for dynamic vectors
  template <typename A, typename std::enable_if<std::is_integral<A>::value && (R == 1 || C == 1) &&
                                                    (R < 0 || C < 0),
                                                int>::type = 0>
  explicit Matrix(A n) : rows_(R == 1 ? 1 : (Index)n), cols_(C == 1 ? 1 : (Index)n) {
    s_.resize(rows_ * cols_);
  }
  Matrix(T a, T b, T c, T d) : rows_(R > 0 ? R : 4), cols_(C > 0 ? C : 1) {
    static_assert(R * C == 4 || R < 0 || C < 0, "4 coefficients");
    s_.resize(rows_ * cols_);
    T* p = s_.p();
    p[0] = a, p[1] = b, p[2] = c, p[3] = d;
  }
  template <typename X, typename std::enable_if<internal::is_mat<X>::value, int>::type = 0>
  Matrix(const X& x) : rows_(x.rows()), cols_(x.cols()) {  // NOLINT: implicit like Eigen
    if ((R > 0 && rows_ != R) || (C > 0 && cols_ != C)) throw std::logic_error("Eigen shim: bad shape");
    s_.resize(rows_ * cols_);
    for (Index j = 0; j < cols_; ++j)
      for (Index i = 0; i < rows_; ++i) (*this)(i, j) = (T)x(i, j);
  }
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) = default;
  template <typename X, typename std::enable_if<internal::is_mat<X>::value, int>::type = 0>
  Matrix& operator=(const X& x) {
    Matrix t(x);
    *this = std::move(t);
    return *this;
  }

  static Matrix Zero() { return Matrix(); }
  template <typename A>
  static Matrix Zero(A n) {
    return Matrix(n);
  }
  template <typename A, typename B>
  static Matrix Zero(A r, B c) {
    return Matrix(r, c);
  }
  static Matrix Identity() {
    Matrix m;
    for (Index i = 0; i < m.rows() && i < m.cols(); ++i) m(i, i) = T(1);
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < r && i < c; ++i) m(i, i) = T(1);
    return m;
  }
  template <typename A>
  static Matrix Constant(A n, T v) {
    Matrix m(n);
    for (Index k = 0; k < m.size(); ++k) m.data()[k] = v;
    return m;
  }
  static Matrix Constant(Index r, Index c, T v) {
    Matrix m(r, c);
    for (Index k = 0; k < m.size(); ++k) m.data()[k] = v;
    return m;
  }
  static Matrix UnitX() {
    Matrix m;
    m(0) = T(1);
    return m;
  }
  static Matrix UnitY() {
    Matrix m;
    m(1) = T(1);
    return m;
  }

  // fixed dimensions are compile-time constants (lets the compiler unroll
  // the coefficient loops of the 2x2 / 4-vector hot path as Eigen does)
  Index rows() const { return R > 0 ? R : rows_; }
  Index cols() const { return C > 0 ? C : cols_; }
  Index size() const { return rows() * cols(); }
  T* data() { return s_.p(); }
  const T* data() const { return s_.p(); }
  T& operator()(Index i, Index j) { return s_.p()[i + rows() * j]; }
  const T& operator()(Index i, Index j) const { return s_.p()[i + rows() * j]; }
  T& operator()(Index k) { return s_.p()[k]; }
  const T& operator()(Index k) const { return s_.p()[k]; }
  T& coeffRef(Index i, Index j) { return (*this)(i, j); }
  T coeff(Index i, Index j) const { return (*this)(i, j); }
  T coeff(Index k) const { return (*this)(k); }
  void resize(Index r, Index c) {
    if ((R > 0 && r != R) || (C > 0 && c != C)) throw std::logic_error("Eigen shim: bad resize");
    rows_ = r, cols_ = c;
    s_.resize(r * c);
  }
  void resize(Index n) { resize(R == 1 ? 1 : n, R == 1 ? n : 1); }
  Matrix& setZero() {
    for (Index k = 0; k < size(); ++k) data()[k] = T(0);
    return *this;
  }
  CommaInit<Matrix> operator<<(T v) {
    CommaInit<Matrix> ci{*this, 0};
    ci, v;
    return ci;
  }

  Matrix<T, C, R> transpose() const {
    Matrix<T, C, R> t(cols_, rows_, 0);
    for (Index j = 0; j < cols_; ++j)
      for (Index i = 0; i < rows_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  const Matrix& eval() const { return *this; }
  Matrix& noalias() { return *this; }

  // views
  Block<Matrix, 1, C> row(Index i) { return {this, i, 0, 1, cols_}; }
  Block<const Matrix, 1, C> row(Index i) const { return {this, i, 0, 1, cols_}; }
  Block<Matrix, R, 1> col(Index j) { return {this, 0, j, rows_, 1}; }
  Block<const Matrix, R, 1> col(Index j) const { return {this, 0, j, rows_, 1}; }
  template <int BR, int BC>
  Block<Matrix, BR, BC> block(Index i, Index j) {
    return {this, i, j, BR, BC};
  }
  template <int BR, int BC>
  Block<const Matrix, BR, BC> block(Index i, Index j) const {
    return {this, i, j, BR, BC};
  }
  Block<Matrix, -1, -1> block(Index i, Index j, Index r, Index c) { return {this, i, j, r, c}; }
  Block<const Matrix, -1, -1> block(Index i, Index j, Index r, Index c) const {
    return {this, i, j, r, c};
  }

  // reductions (Eigen's SSE2 order, see the header)
  T sum() const {
    return internal::redux_sum<T>(size(), [&](Index k) { return data()[k]; });
  }
  T squaredNorm() const {
    return internal::redux_sum<T>(size(), [&](Index k) { return data()[k] * data()[k]; });
  }
  T norm() const { return std::sqrt(squaredNorm()); }
  Matrix normalized() const {
    const T z = squaredNorm();
    if (!(z > T(0))) return *this;
    const T s = std::sqrt(z);
    Matrix m(*this);
    for (Index k = 0; k < size(); ++k) m.data()[k] = data()[k] / s;
    return m;
  }
  template <typename X>
  T dot(const X& o) const {
    return internal::redux_sum<T>(size(), [&](Index k) { return data()[k] * o(k); });
  }
  T determinant() const {
    if (rows_ != 2 || cols_ != 2) throw std::logic_error("Eigen shim: determinant of a 2x2 only");
    return (*this)(0, 0) * (*this)(1, 1) - (*this)(1, 0) * (*this)(0, 1);
  }
  Matrix inverse() const {
    if (rows_ != 2 || cols_ != 2) throw std::logic_error("Eigen shim: inverse of a 2x2 only");
    const T invdet = T(1) / determinant();
    Matrix r(*this);
    r(0, 0) = (*this)(1, 1) * invdet;
    r(1, 0) = -(*this)(1, 0) * invdet;
    r(0, 1) = -(*this)(0, 1) * invdet;
    r(1, 1) = (*this)(0, 0) * invdet;
    return r;
  }
  PartialPivLU<Matrix<T, -1, -1>> partialPivLu() const;

  template <typename X>
  Matrix& operator+=(const X& o) {
    for (Index j = 0; j < cols_; ++j)
      for (Index i = 0; i < rows_; ++i) (*this)(i, j) = (*this)(i, j) + o(i, j);
    return *this;
  }
  template <typename X>
  Matrix& operator-=(const X& o) {
    for (Index j = 0; j < cols_; ++j)
      for (Index i = 0; i < rows_; ++i) (*this)(i, j) = (*this)(i, j) - o(i, j);
    return *this;
  }
  Matrix& operator*=(T s) {
    for (Index k = 0; k < size(); ++k) data()[k] = data()[k] * s;
    return *this;
  }
  Matrix& operator/=(T s) {
    for (Index k = 0; k < size(); ++k) data()[k] = data()[k] / s;
    return *this;
  }

  // private-ish: the transpose constructor
  Matrix(Index r, Index c, int) : rows_(r), cols_(c) { s_.resize(r * c); }

 private:
  internal::Storage<T, internal::prod_size(R, C)> s_;
  Index rows_, cols_;
};

// A rectangular view into a matrix (row / col / block).
template <typename M, int BR, int BC>
class Block {
 public:
  using Scalar = typename std::remove_const<M>::type::Scalar;
  using T = Scalar;
  Block(M* m, Index i, Index j, Index r, Index c) : m_(m), i_(i), j_(j), r_(r), c_(c) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  decltype(auto) operator()(Index i, Index j) const { return (*m_)(i_ + i, j_ + j); }
  decltype(auto) operator()(Index k) const { return r_ == 1 ? (*m_)(i_, j_ + k) : (*m_)(i_ + k, j_); }
  T coeff(Index i, Index j) const { return (*m_)(i_ + i, j_ + j); }
  Matrix<T, BR, BC> eval() const { return Matrix<T, BR, BC>(*this); }
  Matrix<T, BC, BR> transpose() const { return eval().transpose(); }
  T squaredNorm() const { return eval().squaredNorm(); }
  T norm() const { return eval().norm(); }
  T sum() const { return eval().sum(); }
  template <typename X>
  Block& operator=(const X& o) {
    const Matrix<T, -1, -1> t(o);  // evaluate first (aliasing-safe)
    if (t.rows() != r_ || t.cols() != c_) throw std::logic_error("Eigen shim: block shape");
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*m_)(i_ + i, j_ + j) = t(i, j);
    return *this;
  }
  Block& operator=(const Block& o) { return operator=<Block>(o); }
  template <typename X>
  Block& operator+=(const X& o) {
    const Matrix<T, -1, -1> t(o);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*m_)(i_ + i, j_ + j) = (*m_)(i_ + i, j_ + j) + t(i, j);
    return *this;
  }
  template <typename X>
  Block& operator-=(const X& o) {
    const Matrix<T, -1, -1> t(o);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*m_)(i_ + i, j_ + j) = (*m_)(i_ + i, j_ + j) - t(i, j);
    return *this;
  }

 private:
  M* m_;
  Index i_, j_, r_, c_;
};

namespace internal {
template <typename X>
using S = typename traits<X>::Scalar;
template <typename A, typename B>
using enable_mm =
    typename std::enable_if<is_mat<A>::value && is_mat<B>::value, int>::type;
template <typename A>
using enable_m = typename std::enable_if<is_mat<A>::value, int>::type;
}  // namespace internal

// elementwise
template <typename A, typename B, internal::enable_mm<A, B> = 0>
Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> operator+(const A& a,
                                                                                   const B& b) {
  Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> r(a);
  r += b;
  return r;
}
template <typename A, typename B, internal::enable_mm<A, B> = 0>
Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> operator-(const A& a,
                                                                                   const B& b) {
  Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> r(a);
  r -= b;
  return r;
}
template <typename A, internal::enable_m<A> = 0>
Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> operator-(const A& a) {
  Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> r(a);
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = -r.data()[k];
  return r;
}
template <typename A, typename Sc, internal::enable_m<A> = 0,
          typename std::enable_if<std::is_arithmetic<Sc>::value, int>::type = 0>
Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> operator*(Sc s,
                                                                                   const A& a) {
  Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> r(a);
  const internal::S<A> sv = (internal::S<A>)s;
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = sv * r.data()[k];
  return r;
}
template <typename A, typename Sc, internal::enable_m<A> = 0,
          typename std::enable_if<std::is_arithmetic<Sc>::value, int>::type = 0>
Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> operator*(const A& a,
                                                                                   Sc s) {
  Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> r(a);
  const internal::S<A> sv = (internal::S<A>)s;
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = r.data()[k] * sv;
  return r;
}
template <typename A, typename Sc, internal::enable_m<A> = 0,
          typename std::enable_if<std::is_arithmetic<Sc>::value, int>::type = 0>
Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> operator/(const A& a,
                                                                                   Sc s) {
  Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<A>::Cols> r(a);
  const internal::S<A> sv = (internal::S<A>)s;
  for (Index k = 0; k < r.size(); ++k) r.data()[k] = r.data()[k] / sv;
  return r;
}

// matrix product: r(i,j) = sum_k a(i,k) b(k,j), k ascending (exact Eigen
// order for the 2-term fixed-size products; plain order otherwise)
template <typename A, typename B, internal::enable_mm<A, B> = 0>
Matrix<internal::S<A>, internal::traits<A>::Rows, internal::traits<B>::Cols> operator*(const A& a,
                                                                                   const B& b) {
  using T = internal::S<A>;
  if (a.cols() != b.rows()) throw std::logic_error("Eigen shim: product shape");
  Matrix<T, internal::traits<A>::Rows, internal::traits<B>::Cols> r(a.rows(), b.cols(), 0);
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      T s = a.cols() > 0 ? a(i, 0) * b(0, j) : T(0);
      for (Index k = 1; k < a.cols(); ++k) s = s + a(i, k) * b(k, j);
      r(i, j) = s;
    }
  return r;
}

template <typename M>
class PartialPivLU {
 public:
  using T = typename M::Scalar;
  PartialPivLU() = default;
  explicit PartialPivLU(const M& m) { compute(m); }
  PartialPivLU& compute(const M& m) {
    lu_ = m;
    const Index n = lu_.rows();
    perm_.resize((size_t)n);
    for (Index i = 0; i < n; ++i) perm_[(size_t)i] = i;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      T best = std::abs(lu_(k, k));
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(lu_(i, k)) > best) best = std::abs(lu_(i, k)), p = i;
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(p, j));
        std::swap(perm_[(size_t)k], perm_[(size_t)p]);
      }
      if (lu_(k, k) != T(0))
        for (Index i = k + 1; i < n; ++i) lu_(i, k) = lu_(i, k) / lu_(k, k);
      for (Index j = k + 1; j < n; ++j)
        for (Index i = k + 1; i < n; ++i) lu_(i, j) = lu_(i, j) - lu_(i, k) * lu_(k, j);
    }
    return *this;
  }
  template <typename X>
  Matrix<T, -1, -1> solve(const X& b_in) const {
    const Matrix<T, -1, -1> b(b_in);
    const Index n = lu_.rows();
    Matrix<T, -1, -1> x(n, b.cols());
    for (Index c = 0; c < b.cols(); ++c) {
      for (Index i = 0; i < n; ++i) x(i, c) = b(perm_[(size_t)i], c);
      for (Index i = 0; i < n; ++i)
        for (Index k = 0; k < i; ++k) x(i, c) = x(i, c) - lu_(i, k) * x(k, c);
      for (Index i = n - 1; i >= 0; --i) {
        for (Index k = i + 1; k < n; ++k) x(i, c) = x(i, c) - lu_(i, k) * x(k, c);
        x(i, c) = x(i, c) / lu_(i, i);
      }
    }
    return x;
  }

 private:
  Matrix<T, -1, -1> lu_;
  std::vector<Index> perm_;
};

template <typename T, int R, int C>
PartialPivLU<Matrix<T, -1, -1>> Matrix<T, R, C>::partialPivLu() const {
  return PartialPivLU<Matrix<T, -1, -1>>(Matrix<T, -1, -1>(*this));
}

using Matrix2d = Matrix<double, 2, 2>;
using Vector2d = Matrix<double, 2, 1>;
using Matrix4d = Matrix<double, 4, 4>;
using Vector4d = Matrix<double, 4, 1>;
using RowVector4d = Matrix<double, 1, 4>;
using MatrixXd = Matrix<double, -1, -1>;
using VectorXd = Matrix<double, -1, 1>;
using MatrixXi = Matrix<int, -1, -1>;
using VectorXi = Matrix<int, -1, 1>;

enum ComputationInfo { Success = 0, NumericalIssue = 1 };

// Sparse types.  SparseMatrix keeps (row, col) -> value; setFromTriplets sums
// duplicates in triplet order onto the first occurrence, which is the order
// Eigen's collapseDuplicates adds them in (microfem.cpp:125-128).
template <typename T>
class Triplet {
 public:
  Triplet(Index i = 0, Index j = 0, T v = T(0)) : i_(i), j_(j), v_(v) {}
  Index row() const { return i_; }
  Index col() const { return j_; }
  T value() const { return v_; }

 private:
  Index i_, j_;
  T v_;
};
template <typename T>
class SparseMatrix {
 public:
  using Scalar = T;
  SparseMatrix() = default;
  SparseMatrix(Index r, Index c) : r_(r), c_(c) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index nonZeros() const { return (Index)v_.size(); }
  void resize(Index r, Index c) {
    r_ = r, c_ = c;
    v_.clear();
  }
  template <typename It>
  void setFromTriplets(It b, It e) {
    v_.clear();
    for (It t = b; t != e; ++t) {
      auto key = std::make_pair((Index)t->col(), (Index)t->row());
      auto it = v_.find(key);
      if (it == v_.end())
        v_.emplace(key, t->value());
      else
        it->second = it->second + t->value();
    }
  }
  T coeff(Index i, Index j) const {
    auto it = v_.find(std::make_pair(j, i));
    return it == v_.end() ? T(0) : it->second;
  }
  Matrix<T, -1, -1> toDense() const {
    Matrix<T, -1, -1> d(r_, c_);
    for (const auto& kv : v_) d(kv.first.second, kv.first.first) = kv.second;
    return d;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::map<std::pair<Index, Index>, T> v_;  // (col, row) -> value
};

// SparseLU stand-in: a dense partial-pivoting LU of the matrix (test sizes).
template <typename M>
class SparseLU {
 public:
  using T = typename M::Scalar;
  void analyzePattern(const M&) {}
  void factorize(const M& m) {
    lu_.compute(m.toDense());
    info_ = Success;
  }
  void compute(const M& m) { factorize(m); }
  ComputationInfo info() const { return info_; }
  template <typename X>
  Matrix<T, -1, -1> solve(const X& b) const {
    return lu_.solve(b);
  }

 private:
  PartialPivLU<Matrix<T, -1, -1>> lu_;
  ComputationInfo info_ = Success;
};
template <typename M>
class SimplicialLDLT {};

}  // namespace Eigen
