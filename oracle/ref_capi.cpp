// TEST INFRASTRUCTURE ONLY — the checker / CPU baseline, never the product.
//
// A thin extern "C" surface over the reference library compiled from
// /root/reference/proj/src (namespace renamed pmg -> pmg_ref by -Dpmg=pmg_ref,
// see oracle/Makefile) so that pytest (ctypes), tests/golden/make_golden.py and
// bench.py's cpu_baseline / --impl reference legs can drive the reference's own
// code paths. Every wrapper calls exactly one reference entry point; no
// arithmetic happens here.
//
// Status codes: 0 ok, 1 invalid argument, 2 runtime error, 3 divergence.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <numbers>
#include <random>
#include <stdexcept>
#include <vector>

#include "pmg/fastdiag.hpp"
#include "pmg/krylov.hpp"
#include "pmg/level_context.hpp"
#include "pmg/multigrid.hpp"
#include "pmg/operator.hpp"
#include "pmg/patches.hpp"
#include "pmg/smoother.hpp"
#include "pmg/sparse.hpp"

using namespace pmg;

namespace
{

thread_local int g_last_iters = 0;

template <typename F>
int guard(F &&f)
{
  try
  {
    f();
    return 0;
  }
  catch (const DivergenceError &)
  {
    return 3;
  }
  catch (const std::invalid_argument &)
  {
    return 1;
  }
  catch (const std::exception &)
  {
    return 2;
  }
}

struct RefMg
{
  int prec;  // 0 = f64, 1 = f32
  MultigridContext<double> *d = nullptr;
  MultigridContext<float> *f = nullptr;
};

template <typename T>
MultigridContext<T> &ctx_of(RefMg *h);
template <>
MultigridContext<double> &ctx_of<double>(RefMg *h)
{
  return *h->d;
}
template <>
MultigridContext<float> &ctx_of<float>(RefMg *h)
{
  return *h->f;
}

template <typename T>
std::span<T> sp(void *p, std::int64_t n)
{
  return std::span<T>(static_cast<T *>(p), static_cast<std::size_t>(n));
}
template <typename T>
std::span<const T> csp(const void *p, std::int64_t n)
{
  return std::span<const T>(static_cast<const T *>(p), static_cast<std::size_t>(n));
}

double f_one(std::span<const double>) { return 1.0; }
double f_sin(std::span<const double> p)
{
  // -Laplace(u) for u = prod sin(pi x_a): d * pi^2 * prod sin(pi x_a)
  double v = static_cast<double>(p.size()) * std::numbers::pi * std::numbers::pi;
  for (double c : p)
    v *= std::sin(std::numbers::pi * c);
  return v;
}
// a non-separable field for the general-ScalarField tests (kind 2)
double f_gen(std::span<const double> p)
{
  const double z = p.size() > 2 ? p[2] : 0.25;
  return std::exp(p[0] - 0.5 * p[1]) * (1.0 + p[1] * p[1]) * std::cos(2.0 * p[0] * z + p[1]);
}
double u_sin(std::span<const double> p)
{
  double v = 1.0;
  for (double c : p)
    v *= std::sin(std::numbers::pi * c);
  return v;
}

}  // namespace

extern "C" {

// The survey's synthetic inputs: U(-1,1) from std::mt19937_64(seed), x0 filled
// first then b from the same engine.
void ref_fill_uniform(std::uint64_t seed, std::int64_t n0, double *a, std::int64_t n1, double *b)
{
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (std::int64_t i = 0; i < n0; ++i)
    a[i] = dist(gen);
  for (std::int64_t i = 0; i < n1; ++i)
    b[i] = dist(gen);
}

// ---- setup objects ---------------------------------------------------------

int ref_gauss_lobatto(int k, double *out)
{
  return guard([&] {
    auto v = gauss_lobatto_points(k);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

int ref_gauss_legendre(int q, double *pts, double *wts)
{
  return guard([&] {
    auto r = gauss_legendre(q);
    std::memcpy(pts, r.points.data(), q * sizeof(double));
    std::memcpy(wts, r.weights.data(), q * sizeof(double));
  });
}

int ref_cell_matrices(int k, double h, double *mass, double *stiff)
{
  return guard([&] {
    auto cm = cell_matrices_1d(k, h);
    std::memcpy(mass, cm.mass.data.data(), cm.mass.data.size() * sizeof(double));
    std::memcpy(stiff, cm.stiffness.data.data(), cm.stiffness.data.size() * sizeof(double));
  });
}

// out order: mass_full, stiff_full (nc^2 each), mass_ii, stiff_ii (ni^2),
// mass_ib, stiff_ib (ni*2), mass_if, stiff_if (ni*nc)
int ref_patch_matrices(int k, double h, double *out)
{
  return guard([&] {
    auto pm = patch_matrices_1d(k, h);
    double *o = out;
    for (const Mat<double> *m : {&pm.mass_full, &pm.stiff_full, &pm.mass_ii, &pm.stiff_ii,
                                 &pm.mass_ib, &pm.stiff_ib, &pm.mass_if, &pm.stiff_if})
    {
      std::memcpy(o, m->data.data(), m->data.size() * sizeof(double));
      o += m->data.size();
    }
  });
}

// eigenvectors (ni*ni row-major), eigenvalues (ni), inverse_eigen_sums (ni^dim)
int ref_fastdiag(int dim, int k, double h, double *s, double *lambda, double *inv)
{
  return guard([&] {
    auto fd = make_fastdiag<double>(dim, k, h);
    std::memcpy(s, fd.eigenvectors[0].data.data(), fd.eigenvectors[0].data.size() * 8);
    std::memcpy(lambda, fd.eigenvalues[0].data(), fd.eigenvalues[0].size() * 8);
    std::memcpy(inv, fd.inverse_eigen_sums.data(), fd.inverse_eigen_sums.size() * 8);
  });
}

int ref_prolongation_matrix(int dim, int k, int level, double *out)
{
  return guard([&] {
    auto levels = build_hierarchy(dim, k, level);
    auto lc = make_level_context<double>(levels.back());
    std::memcpy(out, lc.prolongation.data.data(), lc.prolongation.data.size() * 8);
  });
}

// ---- multigrid context -----------------------------------------------------

void *ref_mg_create(int dim, int k, int L, int prec, int variant, int threads)
{
  try
  {
    auto *h = new RefMg{prec};
    if (prec == 0)
      h->d = new MultigridContext<double>(make_multigrid_context<double>(
          dim, k, L, static_cast<SmootherVariant>(variant), SmootherKind::vertex_patch, threads));
    else
      h->f = new MultigridContext<float>(make_multigrid_context<float>(
          dim, k, L, static_cast<SmootherVariant>(variant), SmootherKind::vertex_patch, threads));
    return h;
  }
  catch (...)
  {
    return nullptr;
  }
}

// make_multigrid_context with a smoother kind (0 vertex_patch, 1 point_gs);
// nullptr plus *status on the reference's exception
void *ref_mg_create_kind(int dim, int k, int L, int prec, int variant, int kind, int threads, int *status)
{
  RefMg *h = nullptr;
  *status = guard([&] {
    auto *hh = new RefMg{prec};
    try
    {
      if (prec == 0)
        hh->d = new MultigridContext<double>(make_multigrid_context<double>(
            dim, k, L, static_cast<SmootherVariant>(variant), static_cast<SmootherKind>(kind), threads));
      else
        hh->f = new MultigridContext<float>(make_multigrid_context<float>(
            dim, k, L, static_cast<SmootherVariant>(variant), static_cast<SmootherKind>(kind), threads));
    }
    catch (...)
    {
      delete hh;
      throw;
    }
    h = hh;
  });
  return h;
}

// point_gauss_seidel on the context's CSR matrix of level index li (f64)
int ref_point_gs(void *p, int li, double *x, const double *b)
{
  auto *h = static_cast<RefMg *>(p);
  return guard([&] {
    auto &c = *h->d;
    const auto n = c.levels[li].level.total_dofs;
    point_gauss_seidel(c.gs_matrices.at(li), std::span<double>(x, n), std::span<const double>(b, n));
  });
}

// assemble_sparse of the finest level of build_hierarchy(dim, k, level);
// arrays NULL -> only *nnz
int ref_assemble_sparse(int dim, int k, int level, int64_t *row_ptr, int32_t *cols, double *vals, int64_t *nnz)
{
  return guard([&] {
    auto levels = build_hierarchy(dim, k, level);
    CsrMatrix a = assemble_sparse(levels.back());
    *nnz = a.nnz();
    if (row_ptr && cols && vals)
    {
      std::memcpy(row_ptr, a.row_ptr.data(), a.row_ptr.size() * sizeof(int64_t));
      std::memcpy(cols, a.cols.data(), a.cols.size() * sizeof(int32_t));
      std::memcpy(vals, a.vals.data(), a.vals.size() * sizeof(double));
    }
  });
}

void ref_mg_destroy(void *p)
{
  auto *h = static_cast<RefMg *>(p);
  delete h->d;
  delete h->f;
  delete h;
}

void ref_mg_set_threads(void *p, int threads)
{
  auto *h = static_cast<RefMg *>(p);
  if (h->d)
    h->d->threads = threads;
  if (h->f)
    h->f->threads = threads;
}

// MultigridContext::pre_smooth / post_smooth / variant (multigrid.hpp:37-40)
void ref_mg_set_smoothing(void *p, int pre, int post)
{
  auto *h = static_cast<RefMg *>(p);
  if (h->d)
  {
    h->d->pre_smooth = pre;
    h->d->post_smooth = post;
  }
  if (h->f)
  {
    h->f->pre_smooth = pre;
    h->f->post_smooth = post;
  }
}

void ref_mg_set_variant(void *p, int variant)
{
  auto *h = static_cast<RefMg *>(p);
  if (h->d)
    h->d->variant = static_cast<SmootherVariant>(variant);
  if (h->f)
    h->f->variant = static_cast<SmootherVariant>(variant);
}

int64_t ref_mg_total_dofs(void *p, int li)
{
  auto *h = static_cast<RefMg *>(p);
  return h->d ? h->d->levels[li].level.total_dofs : h->f->levels[li].level.total_dofs;
}

#define DISPATCH(h, BODY)                  \
  ((h)->prec == 0 ? [&] {                  \
    using T = double;                      \
    return BODY;                           \
  }()                                      \
                  : [&] {                  \
                      using T = float;     \
                      return BODY;         \
                    }())

int ref_smooth(void *p, int li, int variant, void *x, const void *b)
{
  auto *h = static_cast<RefMg *>(p);
  return DISPATCH(h, guard([&] {
                    auto &c = ctx_of<T>(h);
                    const auto n = c.levels[li].level.total_dofs;
                    smooth<T>(c.levels[li], sp<T>(x, n), csp<T>(b, n),
                              static_cast<SmootherVariant>(variant), c.threads,
                              c.smoother_ws[li]);
                  }));
}

int ref_apply_laplacian(void *p, int li, const void *x, void *y)
{
  auto *h = static_cast<RefMg *>(p);
  return DISPATCH(h, guard([&] {
                    auto &c = ctx_of<T>(h);
                    const auto &lc = c.levels[li];
                    const auto n = lc.level.total_dofs;
                    apply_laplacian<T>(lc.level, lc.cell_mass, lc.cell_stiffness, csp<T>(x, n),
                                       sp<T>(y, n), CellLoop::colored, c.threads);
                  }));
}

int ref_residual(void *p, int li, const void *x, const void *b, void *r)
{
  auto *h = static_cast<RefMg *>(p);
  return DISPATCH(h, guard([&] {
                    auto &c = ctx_of<T>(h);
                    const auto n = c.levels[li].level.total_dofs;
                    compute_residual<T>(c.levels[li], csp<T>(x, n), csp<T>(b, n), sp<T>(r, n),
                                        c.threads);
                  }));
}

// li_coarse -> li_coarse + 1
int ref_prolongate(void *p, int li_coarse, const void *xc, void *xf)
{
  auto *h = static_cast<RefMg *>(p);
  return DISPATCH(h, guard([&] {
                    auto &c = ctx_of<T>(h);
                    const auto &lc = c.levels[li_coarse];
                    const auto &lf = c.levels[li_coarse + 1];
                    prolongate<T>(lc, lf, csp<T>(xc, lc.level.total_dofs),
                                  sp<T>(xf, lf.level.total_dofs));
                  }));
}

int ref_restrict(void *p, int li_coarse, const void *rf, void *rc)
{
  auto *h = static_cast<RefMg *>(p);
  return DISPATCH(h, guard([&] {
                    auto &c = ctx_of<T>(h);
                    const auto &lc = c.levels[li_coarse];
                    const auto &lf = c.levels[li_coarse + 1];
                    restrict_vector<T>(lc, lf, csp<T>(rf, lf.level.total_dofs),
                                       sp<T>(rc, lc.level.total_dofs));
                  }));
}

int ref_vcycle(void *p, int li, void *x, const void *b)
{
  auto *h = static_cast<RefMg *>(p);
  return DISPATCH(h, guard([&] {
                    auto &c = ctx_of<T>(h);
                    const auto n = c.levels[li].level.total_dofs;
                    v_cycle<T>(c, li, sp<T>(x, n), csp<T>(b, n));
                  }));
}

// rhs: 0 -> f = 1, 1 -> f = d pi^2 prod sin(pi x)
int ref_compute_rhs(int dim, int k, int level, int rhs, double *out)
{
  return guard([&] {
    auto levels = build_hierarchy(dim, k, level);
    auto b = compute_rhs(levels.back(), rhs == 0   ? ScalarField(f_one)
                                        : rhs == 1 ? ScalarField(f_sin)
                                                   : ScalarField(f_gen));
    std::memcpy(out, b.data(), b.size() * sizeof(double));
  });
}

// l2_error against the non-separable field f_gen (as an "exact solution")
int ref_l2_error_gen(int dim, int k, int level, const double *x, double *out)
{
  return guard([&] {
    auto levels = build_hierarchy(dim, k, level);
    const auto &lev = levels.back();
    *out = l2_error(lev, csp<double>(x, lev.total_dofs), ScalarField(f_gen));
  });
}

int ref_l2_error_sin(int dim, int k, int level, const double *x, double *out)
{
  return guard([&] {
    auto levels = build_hierarchy(dim, k, level);
    const auto &lev = levels.back();
    *out = l2_error(lev, csp<double>(x, lev.total_dofs), ScalarField(u_sin));
  });
}

// FMG (f64 only, reference: multigrid.cpp:355-400). Per-level rhs assembled by
// the reference's compute_rhs. hist receives ||b|| then per-iteration ||r||.
int ref_fmg(void *p, int rhs, double tol, int max_iterations, double *x, int *iterations,
            double *hist, int hist_cap)
{
  auto *h = static_cast<RefMg *>(p);
  if (h->prec != 0)
    return 1;
  return guard([&] {
    auto &c = *h->d;
    std::vector<std::vector<double>> rl;
    for (auto &lc : c.levels)
      rl.push_back(compute_rhs(lc.level, rhs == 0 ? ScalarField(f_one) : ScalarField(f_sin)));
    const auto n = c.levels.back().level.total_dofs;
    auto st = full_multigrid(c, rl, sp<double>(x, n), tol, max_iterations);
    *iterations = st.iterations;
    for (int i = 0; i < static_cast<int>(st.residual_history.size()) && i < hist_cap; ++i)
      hist[i] = st.residual_history[i];
  });
}

// GMRES (f64) preconditioned by the f32 V-cycle of `pf` (mixed) or the f64
// V-cycle of `pd` (double) — reference krylov.cpp:24-171.
int ref_gmres(void *pd, void *pf, int mixed, const double *b, double *x, double tol,
              int restart, int max_iterations, int *iterations, double *hist, int hist_cap)
{
  auto *hd = static_cast<RefMg *>(pd);
  auto *hf = static_cast<RefMg *>(pf);
  return guard([&] {
    auto &cd = *hd->d;
    const int L = static_cast<int>(cd.levels.size()) - 1;
    const auto &lc = cd.levels[L];
    const auto n = lc.level.total_dofs;
    LinearOperator A = [&](std::span<const double> in, std::span<double> out) {
      apply_laplacian<double>(lc.level, lc.cell_mass, lc.cell_stiffness, in, out,
                              CellLoop::colored, cd.threads);
    };
    LinearOperator P;
    if (mixed)
      P = [&](std::span<const double> in, std::span<double> out) {
        mixed_precision_precondition(*hf->f, in, out);
      };
    else
      P = [&](std::span<const double> in, std::span<double> out) {
        std::fill(out.begin(), out.end(), 0.0);
        v_cycle<double>(cd, L, out, in);
      };
    auto st = gmres(A, P, csp<double>(b, n), sp<double>(x, n), tol, restart, max_iterations);
    *iterations = st.iterations;
    for (int i = 0; i < static_cast<int>(st.residual_history.size()) && i < hist_cap; ++i)
      hist[i] = st.residual_history[i];
    g_last_iters = static_cast<int>(st.residual_history.size());
  });
}

int ref_last_history_len() { return g_last_iters; }

}  // extern "C"
