// C++ drop-in test: reference-style client code compiled against
// include/mumode_b200/mumode.hpp (instead of the reference's mumode/ headers)
// and linked to libmumode_b200.so. Restates cases from the reference's
// test_tucker_ops.cpp / test_tensor_core.cpp; checks against an in-test
// nested-loop evaluation (reference::mode_product_loops semantics,
// reference.hpp:62-80). Exit code 0 = all passed.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "mumode_b200/mumode.hpp"

using namespace mumode;
using core::cplx;
using core::index_t;
using core::Matrix;
using core::Shape;
using core::Tensor;

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

template <class T>
T draw(std::mt19937_64& g) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  if constexpr (std::is_same_v<T, double>) return u(g);
  else {
    double re = u(g);
    return cplx(re, u(g));
  }
}

template <class T>
Tensor<T> rand_tensor(std::mt19937_64& g, const Shape& s) {
  Tensor<T> t(s);
  for (auto& v : t.storage()) v = draw<T>(g);
  return t;
}
template <class T>
Matrix<T> rand_matrix(std::mt19937_64& g, index_t r, index_t c) {
  Matrix<T> m(r, c);
  for (auto& v : m.storage()) v = draw<T>(g);
  return m;
}

template <class T>
Tensor<T> loops_mode_product(const Tensor<T>& t, const Matrix<T>& L, index_t mu) {
  std::vector<index_t> ext = t.shape().extents();
  ext[static_cast<std::size_t>(mu - 1)] = L.rows();
  Tensor<T> out{Shape(ext)};
  for (index_t f = 0; f < out.numel(); ++f) {
    auto j = core::multi_index(out.shape(), f);
    const index_t i = j[static_cast<std::size_t>(mu - 1)];
    T s{};
    for (index_t k = 1; k <= t.extent(mu); ++k) {
      j[static_cast<std::size_t>(mu - 1)] = k;
      s += L(i - 1, k - 1) * t.at(j);
    }
    out[f] = s;
  }
  return out;
}

template <class T>
double rel(const Tensor<T>& a, const Tensor<T>& b) {
  return core::max_abs_diff(a, b) / std::max(core::max_abs(b), 1e-300);
}

int main() {
  std::mt19937_64 g(102);
  // tucker equals the chained nested-loop oracle, orders 1-5, real and complex
  for (int rep = 0; rep < 40; ++rep) {
    const index_t d = 1 + static_cast<index_t>(g() % 5);
    std::vector<index_t> in, out;
    for (index_t k = 0; k < d; ++k) {
      in.push_back(1 + static_cast<index_t>(g() % 4));
      out.push_back(1 + static_cast<index_t>(g() % 4));
    }
    if (rep % 2 == 0) {
      auto T = rand_tensor<double>(g, Shape(in));
      ops::MatrixStack<double> Ls;
      for (index_t k = 0; k < d; ++k) Ls.push_back(rand_matrix<double>(g, out[k], in[k]));
      Tensor<double> want = T;
      for (index_t mu = 1; mu <= d; ++mu) want = loops_mode_product(want, Ls[mu - 1], mu);
      CHECK(rel(ops::tucker(T, Ls), want) < 1e-13);
    } else {
      auto T = rand_tensor<cplx>(g, Shape(in));
      ops::MatrixStack<cplx> Ls;
      for (index_t k = 0; k < d; ++k) Ls.push_back(rand_matrix<cplx>(g, out[k], in[k]));
      Tensor<cplx> want = T;
      for (index_t mu = 1; mu <= d; ++mu) want = loops_mode_product(want, Ls[mu - 1], mu);
      CHECK(rel(ops::tucker(T, Ls), want) < 1e-13);
    }
  }
  // identity stack is exact (test_tucker_ops.cpp:41-52)
  {
    auto T = rand_tensor<double>(g, Shape({3, 4, 5}));
    CHECK(core::max_abs_diff(ops::tucker(T, {Matrix<double>::identity(3), Matrix<double>::identity(4),
                                             Matrix<double>::identity(5)}),
                             T) == 0.0);
  }
  // size errors name the offending mode (test_tucker_ops.cpp:122-132)
  {
    auto T = rand_tensor<double>(g, Shape({2, 3, 4}));
    ops::MatrixStack<double> bad{Matrix<double>::identity(2), Matrix<double>(3, 2), Matrix<double>::identity(4)};
    bool thrown = false;
    try {
      ops::tucker(T, bad);
    } catch (const SizeError& e) {
      thrown = std::string(e.what()).find("mode 2") != std::string::npos;
    }
    CHECK(thrown);
    bool arg = false;
    try {
      core::mode_product(T, Matrix<double>(5, 2), 7);
    } catch (const ArgumentError&) {
      arg = true;
    }
    CHECK(arg);
  }
  // rvalue overload equals const& (test_tucker_ops.cpp:134-143)
  {
    auto T = rand_tensor<double>(g, Shape({3, 4, 5}));
    ops::MatrixStack<double> Ls{rand_matrix<double>(g, 4, 3), rand_matrix<double>(g, 2, 4),
                                rand_matrix<double>(g, 3, 5)};
    auto kept = ops::tucker(T, Ls);
    auto moved = ops::tucker(std::move(T), Ls);
    CHECK(core::max_abs_diff(kept, moved) == 0.0);
  }
  // cttucker vs explicit conjugate transposes; promotion; 1x1 imaginary
  {
    auto T = rand_tensor<cplx>(g, Shape({3, 2, 4}));
    ops::MatrixStack<cplx> P, PH;
    for (index_t e : {3, 2, 4}) {
      P.push_back(rand_matrix<cplx>(g, e, 2));
      PH.push_back(core::conj_transpose(P.back()));
    }
    CHECK(rel(ops::cttucker(T, P), ops::tucker(T, PH)) < 1e-14);
    auto Tr = rand_tensor<double>(g, Shape({3, 2, 3}));
    ops::MatrixStack<cplx> Lc{rand_matrix<cplx>(g, 2, 3), rand_matrix<cplx>(g, 3, 2), rand_matrix<cplx>(g, 2, 3)};
    CHECK(rel(ops::tucker(Tr, Lc), ops::tucker(core::to_complex(Tr), Lc)) < 1e-15);
    Tensor<cplx> s{Shape({1})};
    s[0] = cplx(2.0, 1.0);
    Matrix<cplx> psi(1, 1);
    psi(0, 0) = cplx(0.0, 1.0);
    CHECK(std::abs(ops::cttucker(s, {psi})[0] - cplx(0.0, -1.0) * s[0]) < 1e-15);
  }
  // kronsumv: identity stack gives exactly 3V; d = 1 equals mode_product
  {
    auto V = rand_tensor<double>(g, Shape({2, 3, 2}));
    auto W = ops::kronsumv(V, {Matrix<double>::identity(2), Matrix<double>::identity(3), Matrix<double>::identity(2)});
    double diff = 0;
    for (index_t k = 0; k < V.numel(); ++k) diff = std::max(diff, std::abs(W[k] - 3.0 * V[k]));
    CHECK(diff == 0.0);
    auto V1 = rand_tensor<double>(g, Shape({4}));
    auto A = rand_matrix<double>(g, 4, 4);
    CHECK(core::max_abs_diff(ops::kronsumv(V1, {A}), core::mode_product(V1, A, 1)) == 0.0);
  }
  // mode products on a TMA-sized tensor, every mode, vs loops; sequential == fused
  {
    auto T = rand_tensor<double>(g, Shape({64, 48, 40}));
    for (index_t mu = 1; mu <= 3; ++mu) {
      auto L = rand_matrix<double>(g, 56, T.extent(mu));
      CHECK(rel(core::mode_product(T, L, mu), loops_mode_product(T, L, mu)) < 1e-13);
    }
    ops::MatrixStack<double> Ls{rand_matrix<double>(g, 64, 64), rand_matrix<double>(g, 32, 48),
                                rand_matrix<double>(g, 40, 40)};
    CHECK(rel(ops::tucker(T, Ls), ops::tucker_sequential(T, Ls)) < 1e-13);
  }
  // itucker: identity factors, 2I divides by 2^d, singular factor refused
  {
    auto T = rand_tensor<double>(g, Shape({2, 3, 2}));
    ops::MatrixStack<double> twoI;
    for (index_t e : {2, 3, 2}) {
      Matrix<double> P = Matrix<double>::identity(e);
      for (index_t i = 0; i < e; ++i) P(i, i) = 2.0;
      twoI.push_back(P);
    }
    auto S = ops::itucker(T, ops::FactorizedStack(twoI));
    double diff = 0;
    for (index_t k = 0; k < T.numel(); ++k) diff = std::max(diff, std::abs(S[k] - T[k] / 8.0));
    CHECK(diff < 1e-15);
    // complex stack (FactorizedStack<cplx>, tucker.hpp:36)
    auto Tc = rand_tensor<cplx>(g, Shape({4, 3, 2}));
    ops::MatrixStack<cplx> twoIc;
    for (index_t e : {4, 3, 2}) {
      Matrix<cplx> P = Matrix<cplx>::identity(e);
      for (index_t i = 0; i < e; ++i) P(i, i) = cplx(0.0, 2.0);
      twoIc.push_back(P);
    }
    auto Sc = ops::itucker(Tc, ops::FactorizedStack<cplx>(twoIc));
    double cdiff = 0;
    for (index_t k = 0; k < Tc.numel(); ++k) cdiff = std::max(cdiff, std::abs(Sc[k] - Tc[k] / cplx(0.0, -8.0)));
    CHECK(cdiff < 1e-15);
    bool num = false;
    try {
      ops::FactorizedStack<double>({Matrix<double>(2, 2)});
    } catch (const NumericalError&) {
      num = true;
    }
    CHECK(num);
  }
  // matricize / dematricize / mode_action / tuckerfun (matricize.hpp,
  // mode_product.hpp:88-100, tucker.hpp:169-185): host helpers around user
  // callbacks; with matrix-multiply operators they equal the engine's results
  {
    auto T = rand_tensor<double>(g, Shape({3, 4, 5}));
    for (index_t mu = 1; mu <= 3; ++mu) {
      auto M = core::matricize(T, mu);
      CHECK(M.rows() == T.extent(mu) && M.cols() == T.numel() / T.extent(mu));
      CHECK(core::max_abs_diff(core::dematricize(M, mu, T.shape()), T) == 0.0);
      // column j of the mu-matricization holds the fibre with the other
      // indices in original order, earliest fastest
      auto j = core::multi_index(T.shape(), 17);
      index_t col = 0, scale = 1;
      for (index_t k = 1; k <= 3; ++k) {
        if (k == mu) continue;
        col += (j[static_cast<std::size_t>(k - 1)] - 1) * scale;
        scale *= T.extent(k);
      }
      CHECK(M(j[static_cast<std::size_t>(mu - 1)] - 1, col) == T[17]);
    }
    ops::MatrixStack<double> Ls = {rand_matrix<double>(g, 2, 3), rand_matrix<double>(g, 6, 4),
                                   rand_matrix<double>(g, 5, 5)};
    ops::OperatorStack<double> opsk;
    for (const auto& L : Ls)
      opsk.push_back({L.rows(), [L](const Matrix<double>& X) {
                        Matrix<double> Y(L.rows(), X.cols());
                        for (index_t c = 0; c < X.cols(); ++c)
                          for (index_t k = 0; k < X.rows(); ++k)
                            for (index_t i = 0; i < L.rows(); ++i) Y(i, c) += L(i, k) * X(k, c);
                        return Y;
                      }});
    CHECK(rel(core::mode_action(T, opsk[1].apply, 2), core::mode_product(T, Ls[1], 2)) < 1e-14);
    CHECK(rel(ops::tuckerfun(T, opsk), ops::tucker(T, Ls)) < 1e-14);
    bool contract = false;
    opsk[2].out_rows = 4;  // declared rows disagree with what the operator makes
    try {
      ops::tuckerfun(T, opsk);
    } catch (const ContractError& e) {
      contract = std::string(e.what()).find("mode 3") != std::string::npos;
    }
    CHECK(contract);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
