// C++ host program: the reference-named shim (include/pmg_b200.hpp, CUDA via
// the C-ABI) against the reference library itself (oracle/_ref, through its
// extern "C" test surface). Built by __graft_entry__.build(); run by
// tests/test_gpu_parity.py::test_cpp_shim.
#include <cmath>
#include <cstdio>
#include <vector>

#include "pmg_b200.hpp"

extern "C" {
void ref_fill_uniform(std::uint64_t, std::int64_t, double *, std::int64_t, double *);
void *ref_mg_create(int, int, int, int, int, int);
void ref_mg_destroy(void *);
int ref_smooth(void *, int, int, void *, const void *);
int ref_vcycle(void *, int, void *, const void *);
int ref_apply_laplacian(void *, int, const void *, void *);
int ref_fmg(void *, int, double, int, double *, int *, double *, int);
int ref_gmres(void *, void *, int, const double *, double *, double, int, int, int *, double *, int);
void *ref_mg_create_kind(int, int, int, int, int, int, int, int *);
int ref_point_gs(void *, int, double *, const double *);
}

static double rel(const std::vector<double> &a, const std::vector<double> &b)
{
  double d = 0, n = 0;
  for (size_t i = 0; i < a.size(); ++i)
  {
    d += (a[i] - b[i]) * (a[i] - b[i]);
    n += b[i] * b[i];
  }
  return std::sqrt(d / n);
}

int main()
{
  int fails = 0;
  const int cases[][3] = {{3, 3, 3}, {2, 5, 4}, {3, 7, 2}};
  for (auto &c : cases)
  {
    const int dim = c[0], k = c[1], L = c[2];
    pmgb::MultigridContext<double> ctx(dim, k, L);
    const auto &lev = ctx.levels.back();
    const std::int64_t n = lev.total_dofs();
    std::vector<double> x0(n), b(n);
    ref_fill_uniform(42, n, x0.data(), n, b.data());
    void *ref = ref_mg_create(dim, k, L, 0, 2, 1);

    std::vector<double> x = x0, xr = x0;
    pmgb::smooth<double>(lev, std::span<double>(x), std::span<const double>(b));
    ref_smooth(ref, L - 1, 2, xr.data(), b.data());
    const double e1 = rel(x, xr);

    std::vector<double> y(n), yr(n);
    pmgb::apply_laplacian<double>(lev, std::span<const double>(x0), std::span<double>(y));
    ref_apply_laplacian(ref, L - 1, x0.data(), yr.data());
    const double e2 = rel(y, yr);

    x = x0;
    xr = x0;
    pmgb::v_cycle<double>(ctx, L - 1, std::span<double>(x), std::span<const double>(b));
    ref_vcycle(ref, L - 1, xr.data(), b.data());
    const double e3 = rel(x, xr);
    ref_mg_destroy(ref);
    std::printf("d=%d k=%d L=%d smooth %.2e laplacian %.2e vcycle %.2e\n", dim, k, L, e1, e2, e3);
    if (!(e1 < 1e-12 && e2 < 1e-12 && e3 < 1e-11))
      ++fails;
  }
  // the reference's remaining entry points through the shim
  {
    const int dim = 3, k = 2, L = 4;
    auto ctx = pmgb::make_multigrid_context<double>(dim, k, L);
    const auto &lev = ctx.levels.back();
    const std::int64_t n = lev.total_dofs();
    void *ref = ref_mg_create(dim, k, L, 0, 2, 1);
    std::vector<double> x0(n), b(n);
    ref_fill_uniform(7, n, x0.data(), n, b.data());
    // apply_laplacian(level, cell_mass, cell_stiffness, x, y, mode, threads)
    std::vector<double> y(n), yr(n);
    pmgb::apply_laplacian<double>(lev.level, lev.cell_mass, lev.cell_stiffness, std::span<const double>(x0),
                                  std::span<double>(y), pmgb::CellLoop::colored, 4);
    ref_apply_laplacian(ref, L - 1, x0.data(), yr.data());
    const double ea = rel(y, yr);
    bool refused = false;
    try
    {
      auto cm = lev.cell_mass;
      cm(0, 0) *= 2;
      pmgb::apply_laplacian<double>(lev.level, cm, lev.cell_stiffness, std::span<const double>(x0), std::span<double>(y));
    }
    catch (const std::invalid_argument &)
    {
      refused = true;
    }
    // smooth with the workspace argument
    pmgb::SmootherWorkspace<double> ws;
    std::vector<double> xs = x0, xsr = x0;
    pmgb::smooth<double>(lev, std::span<double>(xs), std::span<const double>(b), pmgb::SmootherVariant::fused, 1, ws);
    ref_smooth(ref, L - 1, 2, xsr.data(), b.data());
    const double es = rel(xs, xsr);
    // vector_norm
    double s2 = 0;
    for (double v : b)
      s2 += v * v;
    const double en = std::fabs(pmgb::vector_norm(std::span<const double>(b)) - std::sqrt(s2)) / std::sqrt(s2);
    // full_multigrid, f = 1
    std::vector<std::vector<double>> rhs;
    for (const auto &lc : ctx.levels)
    {
      rhs.emplace_back(lc.total_dofs());
      pmg_compute_rhs_host(dim, k, lc.level.level, 0, rhs.back().data());
    }
    std::vector<double> xf(n, 0.0), xfr(n, 0.0), hr(64);
    const auto st = pmgb::full_multigrid(ctx, rhs, std::span<double>(xf), 1e-8);
    int itr = 0;
    ref_fmg(ref, 0, 1e-8, 100, xfr.data(), &itr, hr.data(), 64);
    const double ef = rel(xf, xfr);
    // gmres with the mixed-precision (f32 V-cycle) preconditioner
    auto prec = pmgb::make_multigrid_context<float>(dim, k, L);
    void *reff = ref_mg_create(dim, k, L, 1, 2, 1);
    std::vector<double> xg(n, 0.0), xgr(n, 0.0), hg(64);
    const auto sg = pmgb::gmres<float>(ctx, prec, std::span<const double>(rhs.back()), std::span<double>(xg), 1e-9);
    int itg = 0;
    ref_gmres(ref, reff, 1, rhs.back().data(), xgr.data(), 1e-9, 30, 200, &itg, hg.data(), 64);
    const double eg = rel(xg, xgr);
    // point Gauss-Seidel kind
    auto gctx = pmgb::make_multigrid_context<double>(dim, k, L, pmgb::SmootherVariant::fused, pmgb::SmootherKind::point_gs);
    int gst = 0;
    void *gref = ref_mg_create_kind(dim, k, L, 0, 2, 1, 1, &gst);
    std::vector<double> xp = x0, xpr = x0;
    pmgb::point_gauss_seidel(gctx.levels.back(), std::span<double>(xp), std::span<const double>(b));
    ref_point_gs(gref, L - 1, xpr.data(), b.data());
    const double ep = rel(xp, xpr);
    std::vector<double> xv = x0, xvr = x0;
    pmgb::v_cycle<double>(gctx, L - 1, std::span<double>(xv), std::span<const double>(b));
    ref_vcycle(gref, L - 1, xvr.data(), b.data());
    const double epv = rel(xv, xvr);
    const auto csr = pmgb::assemble_sparse(lev.level);
    // multi-GPU context, two virtual ranks: the single-device V-cycle bitwise
    pmgb::MultiGpuContext<double> mctx({0, 0}, dim, k, 5);
    const std::int64_t n5 = mctx.level.total_dofs;
    std::vector<double> x5(n5), b5(n5);
    ref_fill_uniform(9, n5, x5.data(), n5, b5.data());
    auto ctx5 = pmgb::make_multigrid_context<double>(dim, k, 5);
    std::vector<double> xm = x5, xm1 = x5;
    pmgb::v_cycle<double>(mctx, std::span<double>(xm), std::span<const double>(b5));
    pmgb::v_cycle<double>(ctx5, 4, std::span<double>(xm1), std::span<const double>(b5));
    const bool dd_bitwise = xm == xm1;
    std::printf("shim: apply_laplacian(level, M, A) %.2e (foreign matrices refused %d), smooth(ws) %.2e, "
                "vector_norm %.2e, full_multigrid its %d/%d x %.2e, gmres(mixed) its %d/%d x %.2e, point GS %.2e, "
                "point-GS V-cycle %.2e, CSR nnz %lld, 2-rank V-cycle bitwise %d\n",
                ea, refused, es, en, st.iterations, itr, ef, sg.iterations, itg, eg, ep, epv,
                static_cast<long long>(csr.nnz()), dd_bitwise);
    if (!(ea < 1e-12 && refused && es < 1e-12 && en < 1e-13 && st.iterations == itr && ef < 1e-10 &&
          sg.iterations == itg && eg < 1e-8 && ep < 1e-12 && epv < 1e-11 && csr.nnz() > 0 && dd_bitwise))
      ++fails;
    ref_mg_destroy(ref);
    ref_mg_destroy(reff);
    ref_mg_destroy(gref);
  }
  try
  {
    pmgb::MultigridContext<double> bad(4, 1, 1);
    ++fails;
  }
  catch (const std::invalid_argument &)
  {
  }
  std::printf(fails ? "FAIL\n" : "OK\n");
  return fails ? 1 : 0;
}
