// mumode_b200/mumode.hpp -- reference-shaped C++ drop-in over the B200 engine.
//
// A user of the reference library's hot path (/root/reference/proj/include/
// mumode: core::mode_product, ops::tucker, ops::cttucker, ops::tucker_sequential,
// ops::kronsumv, ops::itucker; plus the host-side callback helpers of the same
// files: core::matricize / dematricize / mode_action, ops::tuckerfun)
// includes this header instead and links libmumode_b200.so. The
// value types (Shape, Tensor<T>, Matrix<T>, ModeIndex), the exception types and
// their messages follow the reference's contracts (shape.hpp, tensor.hpp,
// matrix.hpp, errors.hpp, mode_product.hpp:64-83, tucker.hpp:57-232); the
// arithmetic runs on the GPU through the host-buffer C-ABI (mumode_host_*),
// which copies operands to the device and the result back.
//
// Header-only; one engine handle per thread, created on first use on the
// current CUDA device 0 (override with mumode::engine::set_device).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <functional>
#include <initializer_list>
#include <numeric>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../mumode_gpu.h"

namespace mumode {

// ------------------------------------------------------------------ errors
struct SizeError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ArgumentError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ContractError : std::logic_error {
  using std::logic_error::logic_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace core {
using mumode::ArgumentError;
using mumode::ContractError;
using mumode::NumericalError;
using mumode::SizeError;

using index_t = std::int64_t;
using cplx = std::complex<double>;

// ------------------------------------------------------------------ Shape
class Shape {
 public:
  Shape() = default;
  Shape(std::initializer_list<index_t> e) : ext_(e) { check(); }
  explicit Shape(std::vector<index_t> e) : ext_(std::move(e)) { check(); }

  index_t order() const { return static_cast<index_t>(ext_.size()); }
  const std::vector<index_t>& extents() const { return ext_; }
  index_t extent(index_t mu) const {
    check_mode(mu);
    return ext_[static_cast<std::size_t>(mu - 1)];
  }
  index_t numel() const {
    index_t n = 1;
    for (index_t e : ext_) n *= e;
    return n;
  }
  index_t numel_except(index_t mu) const { return numel() / extent(mu); }
  index_t stride(index_t mu) const {
    check_mode(mu);
    index_t s = 1;
    for (index_t k = 0; k + 1 < mu; ++k) s *= ext_[static_cast<std::size_t>(k)];
    return s;
  }
  void check_mode(index_t mu) const {
    if (mu < 1 || mu > order())
      throw ArgumentError("mode index " + std::to_string(mu) + " out of range 1.." +
                          std::to_string(order()));
  }
  bool operator==(const Shape& o) const { return ext_ == o.ext_; }

 private:
  void check() const {
    if (ext_.empty()) throw ArgumentError("tensor order must be >= 1");
    if (std::any_of(ext_.begin(), ext_.end(), [](index_t e) { return e < 1; }))
      throw ArgumentError("tensor extents must be positive");
  }
  std::vector<index_t> ext_;
};

// column-major linearisation, 1-based multi-index (first index fastest)
inline index_t flat_index(const Shape& s, const std::vector<index_t>& j) {
  index_t f = 0;
  for (index_t mu = s.order(); mu >= 1; --mu)
    f = f * s.extent(mu) + (j[static_cast<std::size_t>(mu - 1)] - 1);
  return f;
}
inline std::vector<index_t> multi_index(const Shape& s, index_t f) {
  std::vector<index_t> j;
  for (index_t mu = 1; mu <= s.order(); ++mu) {
    j.push_back(f % s.extent(mu) + 1);
    f /= s.extent(mu);
  }
  return j;
}

struct ModeIndex {
  index_t mu;
  constexpr ModeIndex(index_t m) : mu(m) {}  // NOLINT: implicit, as in the reference
  constexpr operator index_t() const { return mu; }
};

// ------------------------------------------------------------------ Matrix
template <class T>
class Matrix {
 public:
  Matrix() = default;
  Matrix(index_t r, index_t c) : r_(r), c_(c) {
    if (r < 1 || c < 1) throw ArgumentError("matrix dimensions must be positive");
    v_.assign(static_cast<std::size_t>(r * c), T{});
  }
  Matrix(index_t r, index_t c, std::vector<T> v) : r_(r), c_(c), v_(std::move(v)) {
    if (static_cast<index_t>(v_.size()) != r * c)
      throw SizeError("matrix data length does not match rows*cols");
  }
  index_t rows() const { return r_; }
  index_t cols() const { return c_; }
  index_t numel() const { return r_ * c_; }
  T& operator()(index_t i, index_t j) { return v_[static_cast<std::size_t>(i + j * r_)]; }
  const T& operator()(index_t i, index_t j) const { return v_[static_cast<std::size_t>(i + j * r_)]; }
  T* data() { return v_.data(); }
  const T* data() const { return v_.data(); }
  std::vector<T>& storage() { return v_; }
  const std::vector<T>& storage() const { return v_; }
  static Matrix identity(index_t n) {
    Matrix m(n, n);
    for (index_t i = 0; i < n; ++i) m(i, i) = T{1};
    return m;
  }
  bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && v_ == o.v_; }

 private:
  index_t r_ = 0, c_ = 0;
  std::vector<T> v_;
};

template <class T>
Matrix<T> transpose(const Matrix<T>& A) {
  Matrix<T> B(A.cols(), A.rows());
  for (index_t j = 0; j < A.cols(); ++j)
    for (index_t i = 0; i < A.rows(); ++i) B(j, i) = A(i, j);
  return B;
}
inline Matrix<cplx> conj_transpose(const Matrix<cplx>& A) {
  Matrix<cplx> B = transpose(A);
  for (auto& z : B.storage()) z = std::conj(z);
  return B;
}
inline Matrix<double> conj_transpose(const Matrix<double>& A) { return transpose(A); }
inline Matrix<cplx> to_complex(const Matrix<double>& A) {
  return Matrix<cplx>(A.rows(), A.cols(), std::vector<cplx>(A.storage().begin(), A.storage().end()));
}

// ------------------------------------------------------------------ Tensor
template <class T>
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(Shape s) : s_(std::move(s)), v_(static_cast<std::size_t>(s_.numel())) {}
  Tensor(Shape s, std::vector<T> v) : s_(std::move(s)), v_(std::move(v)) {
    if (static_cast<index_t>(v_.size()) != s_.numel())
      throw SizeError("tensor data length does not match shape element count");
  }
  const Shape& shape() const { return s_; }
  index_t order() const { return s_.order(); }
  index_t extent(index_t mu) const { return s_.extent(mu); }
  index_t numel() const { return static_cast<index_t>(v_.size()); }
  T& operator[](index_t f) { return v_[static_cast<std::size_t>(f)]; }
  const T& operator[](index_t f) const { return v_[static_cast<std::size_t>(f)]; }
  T& at(const std::vector<index_t>& j) { return v_[static_cast<std::size_t>(flat_index(s_, j))]; }
  const T& at(const std::vector<index_t>& j) const {
    return v_[static_cast<std::size_t>(flat_index(s_, j))];
  }
  T* data() { return v_.data(); }
  const T* data() const { return v_.data(); }
  std::vector<T>& storage() { return v_; }
  const std::vector<T>& storage() const { return v_; }

 private:
  Shape s_;
  std::vector<T> v_;
};

template <class T>
const std::vector<T>& vec(const Tensor<T>& t) {
  return t.storage();
}
template <class T>
Tensor<T> unvec(std::vector<T> v, const Shape& s) {
  if (static_cast<index_t>(v.size()) != s.numel())
    throw SizeError("unvec: vector length does not match shape element count");
  return Tensor<T>(s, std::move(v));
}
inline Tensor<cplx> to_complex(const Tensor<double>& t) {
  return Tensor<cplx>(t.shape(), std::vector<cplx>(t.storage().begin(), t.storage().end()));
}
template <class T>
double max_abs(const Tensor<T>& t) {
  double m = 0;
  for (const auto& x : t.storage()) m = std::max(m, static_cast<double>(std::abs(x)));
  return m;
}
template <class T>
double max_abs_diff(const Tensor<T>& a, const Tensor<T>& b) {
  double m = 0;
  for (index_t k = 0; k < a.numel(); ++k) m = std::max(m, static_cast<double>(std::abs(a[k] - b[k])));
  return m;
}
template <class T>
double rel_max_dist(const Tensor<T>& a, const Tensor<T>& b) {
  const double s = std::max(max_abs(a), max_abs(b));
  return s == 0 ? 0 : max_abs_diff(a, b) / s;
}

// mu-matricization (matricize.hpp:22-31): m_mu x (prod of the other extents),
// columns = the mu-fibres ordered by the remaining indices, earliest fastest.
// Host-side (it feeds user callbacks, not the engine): element (i, a + A*c)
// is T[a + A*(i + m_mu*c)], a over the modes before mu, c after.
template <class T>
Matrix<T> matricize(const Tensor<T>& t, ModeIndex mu) {
  t.shape().check_mode(mu);
  const index_t rows = t.extent(mu), A = t.shape().stride(mu), C = t.numel() / (A * rows);
  Matrix<T> M(rows, A * C);
  for (index_t c = 0; c < C; ++c)
    for (index_t i = 0; i < rows; ++i)
      for (index_t a = 0; a < A; ++a) M(i, a + A * c) = t[a + A * (i + rows * c)];
  return M;
}

// Inverse of matricize (matricize.hpp:35-56): the output shape is s with
// extent mu replaced by M.rows().
template <class T>
Tensor<T> dematricize(const Matrix<T>& M, ModeIndex mu, const Shape& s) {
  s.check_mode(mu);
  if (M.cols() != s.numel_except(mu))
    throw SizeError("dematricize: column count does not match remaining extents");
  std::vector<index_t> ext = s.extents();
  ext[static_cast<std::size_t>(mu - 1)] = M.rows();
  const index_t rows = M.rows(), A = s.stride(mu), C = M.cols() / A;
  Tensor<T> t{Shape(ext)};
  for (index_t c = 0; c < C; ++c)
    for (index_t i = 0; i < rows; ++i)
      for (index_t a = 0; a < A; ++a) t[a + A * (i + rows * c)] = M(i, a + A * c);
  return t;
}

// mu-mode action (mode_product.hpp:88-100): a columnwise host operator on the
// mu-matricization. The engine's mode_product is the matrix case.
template <class T>
Tensor<T> mode_action(const Tensor<T>& t, const std::function<Matrix<T>(const Matrix<T>&)>& op, ModeIndex mu) {
  t.shape().check_mode(mu);
  Matrix<T> X = matricize(t, mu);
  Matrix<T> Y = op(X);
  if (Y.cols() != X.cols())
    throw ContractError("mode_action: operator changed the column count on mode " + std::to_string(mu.mu));
  return dematricize(Y, mu, t.shape());
}

}  // namespace core

// ------------------------------------------------------------------ engine glue
namespace engine {
inline int& device_slot() {
  static int dev = 0;
  return dev;
}
inline void set_device(int d) { device_slot() = d; }

struct HandleGuard {
  mumode_handle_t h = nullptr;
  ~HandleGuard() {
    if (h) mumode_handle_destroy(h);
  }
};

inline mumode_handle_t handle() {
  thread_local HandleGuard g;
  if (!g.h) {
    if (mumode_handle_create(&g.h, device_slot()) != MUMODE_OK)
      throw DeviceError(std::string("mumode_b200: ") + mumode_last_error());
  }
  return g.h;
}

inline void check(int rc) {
  switch (rc) {
    case MUMODE_OK: return;
    case MUMODE_ERR_SIZE: throw SizeError(mumode_last_error());
    case MUMODE_ERR_ARGUMENT: throw ArgumentError(mumode_last_error());
    case MUMODE_ERR_CONTRACT: throw ContractError(mumode_last_error());
    case MUMODE_ERR_NUMERICAL: throw NumericalError(mumode_last_error());
    default: throw DeviceError(std::string("mumode_b200: ") + mumode_last_error());
  }
}

template <class T>
const double* raw(const T* p) {
  return reinterpret_cast<const double*>(p);
}
template <class T>
double* raw(T* p) {
  return reinterpret_cast<double*>(p);
}
}  // namespace engine

namespace core {

/// S = T x_mu L (reference: core::mode_product, mode_product.hpp:64-77).
template <class T>
Tensor<T> mode_product(const Tensor<T>& t, const Matrix<T>& L, ModeIndex mu) {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, cplx>, "double or complex<double>");
  t.shape().check_mode(mu);
  if (L.cols() != t.extent(mu))
    throw SizeError("mode_product: matrix columns (" + std::to_string(L.cols()) +
                    ") do not match extent of mode " + std::to_string(mu.mu));
  std::vector<index_t> out = t.shape().extents();
  out[static_cast<std::size_t>(mu - 1)] = L.rows();
  Tensor<T> S{Shape(out)};
  const auto& m = t.shape().extents();
  if constexpr (std::is_same_v<T, double>)
    engine::check(mumode_host_mode_product_f64(engine::handle(), static_cast<int>(t.order()), m.data(),
                                               static_cast<int>(mu.mu), L.rows(), t.data(), L.data(),
                                               S.data()));
  else
    engine::check(mumode_host_mode_product_c128(engine::handle(), static_cast<int>(t.order()), m.data(),
                                                static_cast<int>(mu.mu), L.rows(), engine::raw(t.data()),
                                                engine::raw(L.data()), engine::raw(S.data())));
  return S;
}

/// Promoting overload (mode_product.hpp:80-83).
inline Tensor<cplx> mode_product(const Tensor<double>& t, const Matrix<cplx>& L, ModeIndex mu) {
  return mode_product(to_complex(t), L, mu);
}

}  // namespace core

namespace ops {
using core::cplx;
using core::index_t;
using core::Matrix;
using core::Shape;
using core::Tensor;

template <class T>
using MatrixStack = std::vector<Matrix<T>>;

namespace detail {
template <class TT, class TL>
Tensor<TL> run_tucker(const Tensor<TT>& t, const MatrixStack<TL>& Ls, bool adjoint) {
  const index_t d = t.order();
  if (static_cast<index_t>(Ls.size()) != d)
    throw core::SizeError("tucker: stack holds " + std::to_string(Ls.size()) +
                          " matrices for an order-" + std::to_string(d) + " tensor");
  std::vector<index_t> n(static_cast<std::size_t>(d));
  std::vector<const double*> ptrs;
  for (index_t mu = 1; mu <= d; ++mu) {
    const auto& L = Ls[static_cast<std::size_t>(mu - 1)];
    const index_t need = adjoint ? L.rows() : L.cols();
    if (need != t.extent(mu))
      throw core::SizeError("tucker: matrix for mode " + std::to_string(mu) + " expects extent " +
                            std::to_string(need) + ", tensor has " + std::to_string(t.extent(mu)));
    n[static_cast<std::size_t>(mu - 1)] = adjoint ? L.cols() : L.rows();
    ptrs.push_back(engine::raw(L.data()));
  }
  Tensor<TL> S{Shape(n)};
  const auto& m = t.shape().extents();
  const int dd = static_cast<int>(d);
  if constexpr (std::is_same_v<TT, double> && std::is_same_v<TL, double>)
    engine::check(mumode_host_tucker_f64(engine::handle(), dd, m.data(), n.data(), t.data(), ptrs.data(),
                                         S.data(), adjoint ? 1 : 0));
  else if constexpr (std::is_same_v<TT, cplx>)
    engine::check(mumode_host_tucker_c128(engine::handle(), dd, m.data(), n.data(), engine::raw(t.data()),
                                          ptrs.data(), engine::raw(S.data()), adjoint ? 1 : 0));
  else
    engine::check(mumode_host_tucker_promote(engine::handle(), dd, m.data(), n.data(), t.data(),
                                             ptrs.data(), engine::raw(S.data()), adjoint ? 1 : 0));
  return S;
}
}  // namespace detail

/// S = T x_1 L_1 ... x_d L_d (reference: ops::tucker, tucker.hpp:129-140).
template <class T>
Tensor<T> tucker(const Tensor<T>& t, const MatrixStack<T>& Ls) {
  return detail::run_tucker(t, Ls, false);
}
/// Rvalue overload: the host copy of the input is released once it is on the
/// device (tucker.hpp:134-140 releases after the first mode).
template <class T>
Tensor<T> tucker(Tensor<T>&& t, const MatrixStack<T>& Ls) {
  Tensor<T> local = std::move(t);
  return detail::run_tucker(local, Ls, false);
}
inline Tensor<cplx> tucker(const Tensor<double>& t, const MatrixStack<cplx>& Ls) {
  return detail::run_tucker(t, Ls, false);
}
/// Conjugate-transpose Tucker (tucker.hpp:146-155): no Psi^H is formed by the caller.
template <class T>
Tensor<T> cttucker(const Tensor<T>& t, const MatrixStack<T>& Psis) {
  return detail::run_tucker(t, Psis, true);
}
inline Tensor<cplx> cttucker(const Tensor<double>& t, const MatrixStack<cplx>& Psis) {
  return detail::run_tucker(t, Psis, true);
}
/// Unfused chain of standalone mode products (tucker.hpp:159-167).
template <class T>
Tensor<T> tucker_sequential(const Tensor<T>& t, const MatrixStack<T>& Ls) {
  if (static_cast<index_t>(Ls.size()) != t.order()) throw core::SizeError("tucker_sequential: stack length");
  Tensor<T> cur = core::mode_product(t, Ls[0], 1);
  for (index_t mu = 2; mu <= t.order(); ++mu) cur = core::mode_product(cur, Ls[static_cast<std::size_t>(mu - 1)], mu);
  return cur;
}
/// Kronecker-sum action sum_mu V x_mu A_mu (tucker.hpp:206-232), T = double or cplx.
template <class T>
Tensor<T> kronsumv(const Tensor<T>& v, const MatrixStack<T>& As) {
  const index_t d = v.order();
  if (static_cast<index_t>(As.size()) != d)
    throw core::SizeError("kronsumv: stack length does not match tensor order");
  std::vector<const double*> ptrs;
  for (index_t mu = 1; mu <= d; ++mu) {
    const auto& A = As[static_cast<std::size_t>(mu - 1)];
    if (A.rows() != A.cols())
      throw core::SizeError("kronsumv: matrix for mode " + std::to_string(mu) + " is not square");
    if (A.cols() != v.extent(mu))
      throw core::SizeError("kronsumv: matrix size does not match extent of mode " + std::to_string(mu));
    ptrs.push_back(engine::raw(A.data()));
  }
  Tensor<T> W{v.shape()};
  if constexpr (std::is_same_v<T, double>)
    engine::check(mumode_host_kronsumv_f64(engine::handle(), static_cast<int>(d), v.shape().extents().data(),
                                           v.data(), ptrs.data(), W.data()));
  else
    engine::check(mumode_host_kronsumv_c128(engine::handle(), static_cast<int>(d), v.shape().extents().data(),
                                            engine::raw(v.data()), ptrs.data(), engine::raw(W.data())));
  return W;
}

/// Per-mode factorizations for the inverse Tucker operator
/// (ops::FactorizedStack<T>, tucker.hpp:34-51): la::lu_factor (lu.hpp:23-47)
/// at construction, on the host through mumode_lu_factor_* (bitwise the
/// reference's factors), throwing NumericalError on a singular pivot
/// (lu.hpp:33). T is double or cplx.
template <class T>
class FactorizedStack {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, cplx>, "FactorizedStack<double> or <cplx>");

 public:
  struct Factors {
    Matrix<T> lu;
    std::vector<index_t> piv;
  };
  explicit FactorizedStack(const MatrixStack<T>& Ps) {
    for (const auto& P : Ps) {
      if (P.rows() != P.cols()) throw core::SizeError("lu_factor: matrix must be square");
      Factors f{Matrix<T>(P.rows(), P.cols()), std::vector<index_t>(static_cast<std::size_t>(P.rows()))};
      if constexpr (std::is_same_v<T, double>)
        engine::check(mumode_lu_factor_f64(P.rows(), P.data(), f.lu.data(), f.piv.data()));
      else
        engine::check(mumode_lu_factor_c128(P.rows(), engine::raw(P.data()), engine::raw(f.lu.data()), f.piv.data()));
      factors_.push_back(std::move(f));
    }
  }
  index_t size() const { return static_cast<index_t>(factors_.size()); }
  const Factors& factor(index_t mu) const { return factors_.at(static_cast<std::size_t>(mu - 1)); }

 private:
  std::vector<Factors> factors_;
};

/// Inverse Tucker S = T x_1 P_1^-1 ... x_d P_d^-1 (ops::itucker,
/// tucker.hpp:187-204): per-mode triangular solves with the stored factors on
/// the GPU (mumode_host_itucker_*); no inverse is formed.
template <class T>
Tensor<T> itucker(const Tensor<T>& t, const FactorizedStack<T>& F) {
  if (F.size() != t.order()) throw core::SizeError("itucker: stack length does not match tensor order");
  std::vector<const double*> lus;
  std::vector<const int64_t*> pivs;
  for (index_t mu = 1; mu <= t.order(); ++mu) {
    const auto& f = F.factor(mu);
    if (f.lu.rows() != t.extent(mu))
      throw core::SizeError("itucker: factor size does not match extent of mode " + std::to_string(mu));
    lus.push_back(engine::raw(f.lu.data()));
    pivs.push_back(f.piv.data());
  }
  Tensor<T> S{t.shape()};
  const int dd = static_cast<int>(t.order());
  if constexpr (std::is_same_v<T, double>)
    engine::check(mumode_host_itucker_f64(engine::handle(), dd, t.shape().extents().data(), t.data(), lus.data(),
                                          pivs.data(), S.data()));
  else
    engine::check(mumode_host_itucker_c128(engine::handle(), dd, t.shape().extents().data(), engine::raw(t.data()),
                                           lus.data(), pivs.data(), engine::raw(S.data())));
  return S;
}

/// Columnwise operator of the operator-action Tucker (tucker.hpp:24-32).
template <class T>
struct ColumnOperator {
  index_t out_rows;
  std::function<Matrix<T>(const Matrix<T>&)> apply;
};
template <class T>
using OperatorStack = std::vector<ColumnOperator<T>>;

/// Operator-action Tucker (ops::tuckerfun, tucker.hpp:169-185): host
/// callbacks, applied per mode in order 1..d (arbitrary operators have no
/// device form; not the accelerated path).
template <class T>
Tensor<T> tuckerfun(const Tensor<T>& t, const OperatorStack<T>& ops) {
  if (static_cast<index_t>(ops.size()) != t.order())
    throw core::SizeError("tuckerfun: stack length does not match tensor order");
  Tensor<T> cur = t;
  for (index_t mu = 1; mu <= t.order(); ++mu) {
    const auto& op = ops[static_cast<std::size_t>(mu - 1)];
    cur = core::mode_action(cur, op.apply, mu);
    if (cur.extent(mu) != op.out_rows)
      throw core::ContractError("tuckerfun: operator on mode " + std::to_string(mu) + " produced " +
                                std::to_string(cur.extent(mu)) + " rows, declared " + std::to_string(op.out_rows));
  }
  return cur;
}

}  // namespace ops
}  // namespace mumode
