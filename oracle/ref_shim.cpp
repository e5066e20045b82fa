// extern "C" surface over the REFERENCE library (built from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY. Loaded with RTLD_LOCAL by oracle/__init__.py so
// the reference's mumode:: symbols never meet the product. Every function
// forwards to the reference's own public API on the reference's own types:
//   ops::tucker / cttucker / tucker_sequential / kronsumv / itucker
//                                   (proj/include/mumode/tucker.hpp:129-232)
//   core::mode_product              (proj/include/mumode/mode_product.hpp:64-83)
//   kronref::kron_apply_oracle      (proj/include/mumode/kron.hpp:73-99)
//   reference::mode_product_loops   (proj/include/mumode/reference.hpp:62-80)
//   la::expm                        (proj/src/expm.cpp:97-151)
//   la::lu_factor                   (proj/include/mumode/lu.hpp:23-47)
//   la::symtridiag_eig              (proj/src/tridiag.cpp:12-90)
//   apps::imex_evolve, Direct       (proj/src/imex.cpp:88-200; DirectSolver :53-86)
//   basis::laplacian_stencil        (proj/src/stencils.cpp:34-50)
// Buffers are column-major; complex is interleaved (re, im) doubles, which is
// the std::complex<double> layout. Return codes: 0 ok, 1 SizeError,
// 2 ArgumentError, 6 ContractError, 7 NumericalError, 9 other; the message is
// kept for ref_last_error().
#include <algorithm>
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "mumode/expm.hpp"
#include "mumode/gemm.hpp"
#include "mumode/imex.hpp"
#include "mumode/lu.hpp"
#include "mumode/tridiag.hpp"
#include "mumode/kron.hpp"
#include "mumode/mode_product.hpp"
#include "mumode/reference.hpp"
#include "mumode/stencils.hpp"
#include "mumode/tucker.hpp"

using namespace mumode;
using core::cplx;
using core::index_t;
using core::Matrix;
using core::Shape;
using core::Tensor;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SizeError& e) {
    g_err = e.what();
    return 1;
  } catch (const ArgumentError& e) {
    g_err = e.what();
    return 2;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 6;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

template <class T>
const T* as(const double* p) { return reinterpret_cast<const T*>(p); }
template <class T>
T* as(double* p) { return reinterpret_cast<T*>(p); }

template <class T>
Tensor<T> make_tensor(int d, const int64_t* ext, const double* data) {
  std::vector<index_t> e(ext, ext + d);
  Shape s(e);
  const T* p = as<T>(data);
  return Tensor<T>(s, std::vector<T>(p, p + s.numel()));
}

template <class T>
Matrix<T> make_matrix(int64_t rows, int64_t cols, const double* data) {
  const T* p = as<T>(data);
  return Matrix<T>(rows, cols, std::vector<T>(p, p + rows * cols));
}

template <class T>
void store(const Tensor<T>& t, double* out, int64_t* out_ext) {
  std::memcpy(out, t.data(), sizeof(T) * static_cast<std::size_t>(t.numel()));
  if (out_ext)
    for (index_t mu = 1; mu <= t.order(); ++mu) out_ext[mu - 1] = t.extent(mu);
}

// Stack of d matrices; L[mu] has rows[mu] x cols[mu].
template <class T>
ops::MatrixStack<T> make_stack(int d, const int64_t* rows, const int64_t* cols,
                               const double* const* Ls) {
  ops::MatrixStack<T> st;
  for (int mu = 0; mu < d; ++mu) st.push_back(make_matrix<T>(rows[mu], cols[mu], Ls[mu]));
  return st;
}

template <class T>
int tucker_impl(int d, const int64_t* m, const int64_t* Lrows, const int64_t* Lcols,
                const double* T_, const double* const* Ls, double* S, int64_t* out_ext,
                int variant) {
  return guarded([&] {
    Tensor<T> t = make_tensor<T>(d, m, T_);
    auto st = make_stack<T>(d, Lrows, Lcols, Ls);
    Tensor<T> r;
    if (variant == 0) r = ops::tucker(t, st);
    else if (variant == 1) r = ops::cttucker(t, st);
    else if (variant == 2) r = ops::tucker_sequential(t, st);
    else if (variant == 3) r = ops::tucker(std::move(t), st);
    else if (variant == 4) r = kronref::kron_apply_oracle(st, t);
    else if (variant == 5) r = ops::kronsumv(t, st);
    store(r, S, out_ext);
  });
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
const char* ref_blas_kernel_name() { return la::blas_kernel_name(); }

// variant: 0 tucker, 1 cttucker, 2 tucker_sequential, 3 tucker(rvalue),
//          4 kron_apply_oracle, 5 kronsumv.  Lrows/Lcols: per-mode matrix dims.
int ref_tucker_f64(int d, const int64_t* m, const int64_t* Lrows, const int64_t* Lcols,
                   const double* T, const double* const* Ls, double* S, int64_t* out_ext,
                   int variant) {
  return tucker_impl<double>(d, m, Lrows, Lcols, T, Ls, S, out_ext, variant);
}
int ref_tucker_c128(int d, const int64_t* m, const int64_t* Lrows, const int64_t* Lcols,
                    const double* T, const double* const* Ls, double* S, int64_t* out_ext,
                    int variant) {
  return tucker_impl<cplx>(d, m, Lrows, Lcols, T, Ls, S, out_ext, variant);
}
// Real tensor against a complex stack (tucker.hpp:142-144, :153-155).
int ref_tucker_promote(int d, const int64_t* m, const int64_t* Lrows, const int64_t* Lcols,
                       const double* T, const double* const* Ls, double* S, int adjoint) {
  return guarded([&] {
    Tensor<double> t = make_tensor<double>(d, m, T);
    auto st = make_stack<cplx>(d, Lrows, Lcols, Ls);
    Tensor<cplx> r = adjoint ? ops::cttucker(t, st) : ops::tucker(t, st);
    store(r, S, nullptr);
  });
}

// core::mode_product (variant 0) or reference::mode_product_loops (variant 1).
int ref_mode_product_f64(int d, const int64_t* m, int mu, int64_t Lrows, int64_t Lcols,
                         const double* T, const double* L, double* S, int variant) {
  return guarded([&] {
    Tensor<double> t = make_tensor<double>(d, m, T);
    Matrix<double> Lm = make_matrix<double>(Lrows, Lcols, L);
    Tensor<double> r = variant == 0 ? core::mode_product(t, Lm, mu)
                                    : reference::mode_product_loops(t, Lm, mu);
    store(r, S, nullptr);
  });
}
int ref_mode_product_c128(int d, const int64_t* m, int mu, int64_t Lrows, int64_t Lcols,
                          const double* T, const double* L, double* S, int variant) {
  return guarded([&] {
    Tensor<cplx> t = make_tensor<cplx>(d, m, T);
    Matrix<cplx> Lm = make_matrix<cplx>(Lrows, Lcols, L);
    Tensor<cplx> r = variant == 0 ? core::mode_product(t, Lm, mu)
                                  : reference::mode_product_loops(t, Lm, mu);
    store(r, S, nullptr);
  });
}

// ops::itucker with FactorizedStack (tucker.hpp:187-204): S = T x_mu P_mu^-1.
int ref_itucker_f64(int d, const int64_t* m, const double* T, const double* const* Ps,
                    double* S) {
  return guarded([&] {
    Tensor<double> t = make_tensor<double>(d, m, T);
    auto st = make_stack<double>(d, m, m, Ps);
    ops::FactorizedStack<double> F(st);
    store(ops::itucker(t, F), S, nullptr);
  });
}

int ref_itucker_c128(int d, const int64_t* m, const double* T, const double* const* Ps, double* S) {
  return guarded([&] {
    Tensor<cplx> t = make_tensor<cplx>(d, m, T);
    auto st = make_stack<cplx>(d, m, m, Ps);
    ops::FactorizedStack<cplx> F(st);
    store(ops::itucker(t, F), S, nullptr);
  });
}

// la::lu_factor (lu.hpp:23-47): lu (n x n) and piv (n).
int ref_lu_factor_f64(int64_t n, const double* P, double* lu, int64_t* piv) {
  return guarded([&] {
    auto f = la::lu_factor(make_matrix<double>(n, n, P));
    std::memcpy(lu, f.lu.data(), sizeof(double) * static_cast<std::size_t>(n * n));
    for (int64_t k = 0; k < n; ++k) piv[k] = f.piv[static_cast<std::size_t>(k)];
  });
}
int ref_lu_factor_c128(int64_t n, const double* P, double* lu, int64_t* piv) {
  return guarded([&] {
    auto f = la::lu_factor(make_matrix<cplx>(n, n, P));
    std::memcpy(lu, f.lu.data(), sizeof(cplx) * static_cast<std::size_t>(n * n));
    for (int64_t k = 0; k < n; ++k) piv[k] = f.piv[static_cast<std::size_t>(k)];
  });
}

// la::symtridiag_eig, EigMode::FullVectors (tridiag.cpp:12-90).
int ref_symtridiag_eig_f64(int64_t m, const double* diag, const double* offdiag, double* values,
                           double* vectors) {
  return guarded([&] {
    la::TridiagSym T;
    T.diag.assign(diag, diag + m);
    T.offdiag.assign(offdiag, offdiag + (m - 1));
    auto r = la::symtridiag_eig(T, la::EigMode::FullVectors);
    std::memcpy(values, r.values.data(), sizeof(double) * static_cast<std::size_t>(m));
    std::memcpy(vectors, r.vectors.data(), sizeof(double) * static_cast<std::size_t>(m * m));
  });
}

// One step of apps::imex_evolve with the Direct backend and no nonlinearity
// (src/imex.cpp:88-200): builds DirectSolver from M_mu = (1/d) I - tau A_mu
// (extract_tridiag + symtridiag_eig, :28-65) and returns u1 = solve(u0)
// (:67-86) -- the reference's own DirectSolver, reached through its public
// driver. A_mu: m_mu x m_mu stencil matrices.
int ref_imex_direct_f64(int d, const int64_t* m, const double* const* As, const double* u0, double tau,
                        int steps, double* u) {
  return guarded([&] {
    apps::EvolutionProblem prob;
    for (int k = 0; k < d; ++k) {
      basis::StencilMatrix st;
      st.A = make_matrix<double>(m[k], m[k], As[k]);
      prob.stencils.push_back(std::move(st));
    }
    prob.u0 = make_tensor<double>(d, m, u0);
    prob.tau = tau;
    prob.t_final = tau * steps;
    prob.nonlinearity = apps::NonlinearTerm::None;
    auto res = apps::imex_evolve(prob, apps::ImexBackend::Direct);
    store(res.first, u, nullptr);
  });
}

int ref_expm_f64(int64_t n, const double* A, double* E) {
  return guarded([&] {
    Matrix<double> Am = make_matrix<double>(n, n, A);
    Matrix<double> R = la::expm(Am);
    std::memcpy(E, R.data(), sizeof(double) * static_cast<std::size_t>(n * n));
  });
}

int ref_laplacian_f64(int64_t n, double* A) {
  return guarded([&] {
    auto st = basis::laplacian_stencil(n);
    std::memcpy(A, st.A.data(), sizeof(double) * static_cast<std::size_t>(n * n));
  });
}

// Median-of-reps timing of `steps` chained ops::tucker calls, u <- tucker(u, Ls),
// after one discarded warm-up (the reference's time_median protocol,
// tools/mumode_cli.cpp:79-90). Writes the final u of the last rep to S.
int ref_time_tucker_f64(int d, const int64_t* m, const int64_t* Lrows, const int64_t* Lcols,
                        const double* T, const double* const* Ls, int steps, int reps,
                        double* S, double* median_s, double* all_s) {
  return guarded([&] {
    Tensor<double> t0 = make_tensor<double>(d, m, T);
    auto st = make_stack<double>(d, Lrows, Lcols, Ls);
    Tensor<double> u;
    auto run = [&] {
      u = t0;
      for (int s = 0; s < steps; ++s) u = ops::tucker(u, st);
    };
    run();
    std::vector<double> ts;
    for (int r = 0; r < reps; ++r) {
      const double a = now_s();
      run();
      ts.push_back(now_s() - a);
      if (all_s) all_s[r] = ts.back();
    }
    std::vector<double> sorted = ts;
    std::sort(sorted.begin(), sorted.end());
    *median_s = sorted[sorted.size() / 2];
    if (S) store(u, S, nullptr);
  });
}

// The reference arm of bench.py, entirely inside the reference library: draws
// T (m_1 x ... x m_d) then L_1..L_d (n_mu x m_mu) with the reference's
// generator (std::mt19937_64(seed), a FRESH std::normal_distribution<double>
// per object, column-major fill; tools/mumode_cli.cpp:92-121, :237-240), runs
// `warmup` untimed ops::tucker applications, then times `reps` of them one by
// one (times[r], seconds). No input or output crosses this boundary, so the
// timed region is ops::tucker alone (its own output allocation included, as
// in the reference's bench-tucker, tools/mumode_cli.cpp:219-255).
int ref_bench_tucker_f64(uint64_t seed, int d, const int64_t* m, const int64_t* n, int warmup, int reps,
                         double* times, double* checksum) {
  return guarded([&] {
    std::mt19937_64 g(seed);
    auto fill = [&g](double* p, index_t count) {
      std::normal_distribution<double> dist;
      for (index_t k = 0; k < count; ++k) p[k] = dist(g);
    };
    Tensor<double> t{Shape(std::vector<index_t>(m, m + d))};
    fill(t.data(), t.numel());
    ops::MatrixStack<double> st;
    for (int k = 0; k < d; ++k) {
      Matrix<double> L(n[k], m[k]);
      fill(L.data(), n[k] * m[k]);
      st.push_back(std::move(L));
    }
    Tensor<double> s;
    for (int w = 0; w < warmup; ++w) s = ops::tucker(t, st);
    for (int r = 0; r < reps; ++r) {
      const double a = now_s();
      s = ops::tucker(t, st);
      times[r] = now_s() - a;
    }
    if (checksum) {
      double c = 0.0;
      for (index_t k = 0; k < s.numel(); ++k) c += s[k];
      *checksum = c;
    }
  });
}

int ref_time_tucker_c128(int d, const int64_t* m, const int64_t* Lrows, const int64_t* Lcols,
                         const double* T, const double* const* Ls, int reps, double* S,
                         double* median_s) {
  return guarded([&] {
    Tensor<cplx> t0 = make_tensor<cplx>(d, m, T);
    auto st = make_stack<cplx>(d, Lrows, Lcols, Ls);
    Tensor<cplx> u;
    auto run = [&] { u = ops::tucker(t0, st); };
    run();
    std::vector<double> ts;
    for (int r = 0; r < reps; ++r) {
      const double a = now_s();
      run();
      ts.push_back(now_s() - a);
    }
    std::sort(ts.begin(), ts.end());
    *median_s = ts[ts.size() / 2];
    if (S) store(u, S, nullptr);
  });
}

}  // extern "C"
