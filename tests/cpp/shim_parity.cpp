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
