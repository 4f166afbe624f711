// C++ host program over the C-ABI's multi-GPU entry points (pmg_dd_*):
// P virtual ranks (one process, devices may repeat, PMG_DD_COPY) must give
// the single-device smoother step and V-cycle BITWISE, and the single-device
// full multigrid's iteration count (norms to rounding).
//
//   dd_parity <device> [k L P dtype(0=f64,1=f32) ...]
// prints one line per case and exits non-zero on any mismatch.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#include "pmg_b200.h"

#define CK(x)                                                                     \
  do                                                                              \
  {                                                                               \
    int st_ = (x);                                                                \
    if (st_ != PMG_OK)                                                            \
    {                                                                             \
      std::fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, st_,  \
                   pmg_last_error());                                             \
      std::exit(2);                                                               \
    }                                                                             \
  } while (0)

template <typename T>
static std::vector<T> uniform(size_t n, unsigned seed)
{
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<T> v(n);
  for (auto &e : v)
    e = static_cast<T>(u(g));
  return v;
}

template <typename T>
static bool run_case(int device, int k, int L, int P, int dtype)
{
  const int64_t m = (int64_t(1) << L) * k - 1, N = m * m * m;
  const auto x0 = uniform<T>(N, 42), b = uniform<T>(N, 43);

  // single device
  pmg_mg mg = nullptr;
  CK(pmg_mg_create(3, k, L, dtype, PMG_FUSED, device, &mg));
  std::vector<T> xs = x0, xv = x0;
  CK(pmg_smooth_host(pmg_mg_level(mg, L - 1), PMG_FUSED, xs.data(), b.data()));
  // two cycles: the second starts from the first's workspaces (stale-state check)
  CK(pmg_v_cycle_host(mg, L - 1, xv.data(), b.data()));
  CK(pmg_v_cycle_host(mg, L - 1, xv.data(), b.data()));

  // P virtual ranks
  std::vector<int> devs(P, device);
  pmg_dd dd = nullptr;
  CK(pmg_dd_create(P, devs.data(), 3, k, L, 1, dtype, PMG_FUSED, PMG_DD_COPY, &dd));
  int world = 0, local = 0, ndl = 0;
  CK(pmg_dd_info(dd, &world, &local, &ndl));
  std::vector<T> out(N);
  CK(pmg_dd_scatter_host(dd, PMG_DD_X, x0.data()));
  CK(pmg_dd_scatter_host(dd, PMG_DD_B, b.data()));
  CK(pmg_dd_smooth(dd));
  CK(pmg_dd_gather_host(dd, PMG_DD_X, out.data()));
  const bool smooth_ok = std::memcmp(out.data(), xs.data(), N * sizeof(T)) == 0;
  CK(pmg_dd_scatter_host(dd, PMG_DD_X, x0.data()));
  CK(pmg_dd_v_cycle(dd));
  CK(pmg_dd_v_cycle(dd));
  CK(pmg_dd_gather_host(dd, PMG_DD_X, out.data()));
  const bool vc_ok = std::memcmp(out.data(), xv.data(), N * sizeof(T)) == 0;
  double rn = 0;
  CK(pmg_dd_residual_norm(dd, &rn));

  // the single-device residual norm of the same iterate
  double rn1 = 0;
  {
    std::vector<T> r(N);
    CK(pmg_compute_residual_host(pmg_mg_level(mg, L - 1), xv.data(), b.data(), r.data()));
    double s = 0, comp = 0;  // compensated sum: 1e9 squares summed sequentially lose ~1e-11
    for (T e : r)
    {
      const double y = double(e) * double(e) - comp;
      const double t = s + y;
      comp = (t - s) - y;
      s = t;
    }
    rn1 = std::sqrt(s);
  }
  const double rn_rel = std::fabs(rn - rn1) / rn1;
  const bool rn_ok = rn_rel < (dtype == PMG_F64 ? 1e-12 : 1e-5);

  // full multigrid, f = 1 (f64 only, like the reference): identical
  // iteration counts, histories to rounding
  bool fmg_ok = true;
  int its1 = -1, itsd = -1;
  double hist_rel = 0;
  if (dtype == PMG_F64)
  {
    std::vector<std::vector<double>> rhs(L);
    std::vector<const double *> rph(L);
    std::vector<void *> rpd(L);
    for (int l = 1; l <= L; ++l)
    {
      const int64_t ml = (int64_t(1) << l) * k - 1;
      rhs[l - 1].resize(ml * ml * ml);
      CK(pmg_compute_rhs_host(3, k, l, 0, rhs[l - 1].data()));
      rph[l - 1] = rhs[l - 1].data();
      cudaSetDevice(device);
      cudaMalloc(&rpd[l - 1], rhs[l - 1].size() * sizeof(double));
      cudaMemcpy(rpd[l - 1], rhs[l - 1].data(), rhs[l - 1].size() * sizeof(double), cudaMemcpyHostToDevice);
    }
    void *xd = nullptr;
    cudaMalloc(&xd, N * sizeof(double));
    cudaMemset(xd, 0, N * sizeof(double));
    double hist1[64] = {}, histd[64] = {};
    CK(pmg_full_multigrid(mg, const_cast<const void *const *>(rpd.data()), xd, 1e-8, 50, &its1, hist1, 64, nullptr));
    cudaDeviceSynchronize();
    CK(pmg_dd_full_multigrid(dd, rph.data(), 1e-8, 50, &itsd, histd, 64));
    for (int i = 0; i <= its1 && i < 64; ++i)
      hist_rel = std::fmax(hist_rel, std::fabs(hist1[i] - histd[i]) / hist1[i]);
    fmg_ok = its1 == itsd && hist_rel < 1e-6;
    for (void *p : rpd)
      cudaFree(p);
    cudaFree(xd);
  }
  CK(pmg_dd_destroy(dd));
  CK(pmg_mg_destroy(mg));
  const bool ok = smooth_ok && vc_ok && rn_ok && fmg_ok;
  std::printf("k=%d L=%d P=%d %s decomposed_levels=%d smooth_bitwise=%d vcycle_bitwise=%d "
              "resnorm_rel=%.2e fmg_its=%d/%d hist_rel=%.2e %s\n",
              k, L, P, dtype == PMG_F64 ? "f64" : "f32", ndl, smooth_ok, vc_ok, rn_rel, itsd, its1, hist_rel,
              ok ? "OK" : "FAIL");
  return ok;
}

int main(int argc, char **argv)
{
  const int device = argc > 1 ? std::atoi(argv[1]) : 0;
  std::vector<int> cases;
  for (int i = 2; i < argc; ++i)
    cases.push_back(std::atoi(argv[i]));
  if (cases.empty())
    cases = {2, 5, 2, 0, 2, 6, 4, 0, 2, 7, 8, 0, 1, 8, 8, 0, 4, 6, 4, 0, 2, 6, 2, 1, 3, 4, 2, 0};
  bool all = true;
  for (size_t i = 0; i + 3 < cases.size(); i += 4)
  {
    const int k = cases[i], L = cases[i + 1], P = cases[i + 2], dt = cases[i + 3];
    all &= dt == PMG_F64 ? run_case<double>(device, k, L, P, dt) : run_case<float>(device, k, L, P, dt);
  }
  return all ? 0 : 1;
}
