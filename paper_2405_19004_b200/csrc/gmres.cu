// Device GMRES with the (mixed-precision) multigrid V-cycle preconditioner.
//
// Replaces gmres() and mixed_precision_precondition() of
// /root/reference/proj/src/krylov.cpp:24-150 and :152-171 with the same
// algorithm: right-preconditioned GMRES(restart) in f64, modified
// Gram-Schmidt with one re-orthogonalisation pass when the first pass removes
// more than 1e-8 of the squared norm, Givens rotations on the host (tiny
// Hessenberg), true-residual check at every restart; the preconditioner is one
// V-cycle from zero in f32 (downcast with a non-finite check, upcast of the
// correction) or in f64. All vectors live on the device; only the O(restart^2)
// Hessenberg work and scalar reductions touch the host.
#include <cmath>
#include <string>
#include <vector>

#include "../../include/pmg_b200.h"
#include "blas.cuh"
#include "capi_internal.hpp"

using namespace pmgb;

extern "C" int pmg_gmres(pmg_mg op, pmg_mg prec, const void *b_, void *x_, double tol, int restart,
                         int max_iterations, int *iterations, double *history, int history_cap,
                         void *stream)
{
  return capi_guard([&] {
    if (!op || !prec)
      throw std::invalid_argument("gmres: null context");
    if (mg_dtype(op) != PMG_F64)
      throw std::invalid_argument("gmres: operator context must be f64");
    if (!(tol > 0.0))
      throw std::invalid_argument("gmres: tol must be positive");
    if (restart < 1)
      throw std::invalid_argument("gmres: restart must be >= 1");
    const int device = mg_device(op);
    DevScope dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int L = mg_levels(op) - 1;
    const int Lp = mg_levels(prec) - 1;
    const int64_t n = level_total(mg_level_ptr(op, L));
    if (level_total(mg_level_ptr(prec, Lp)) != n)
      throw std::invalid_argument("gmres: preconditioner level does not match operator level");
    const int sm = level_sm_count(mg_level_ptr(op, L));
    const double *b = static_cast<const double *>(b_);
    double *x = static_cast<double *>(x_);

    GmresWork &w = mg_gmres_work(op);
    w.ensure(n, restart, mg_dtype(prec) == PMG_F32);
    double *V = w.V, *Z = w.Z, *wv = w.w, *r = w.r;
    double *red = w.red;
    auto Vj = [&](int j) { return V + static_cast<int64_t>(j) * n; };
    auto Zj = [&](int j) { return Z + static_cast<int64_t>(j) * n; };

    auto dot = [&](const double *a, const double *c) {
      launch_dot<double>(a, c, n, red, red + RED_BLOCKS, false, s);
      double out;
      check_cuda(cudaMemcpyAsync(&out, red + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
      check_cuda(cudaStreamSynchronize(s), "sync");
      return out;
    };
    auto nrm = [&](const double *a) { return std::sqrt(dot(a, a)); };
    auto apply_A = [&](const double *in, double *out) { mg_apply_finest_op(op, in, out, s); };
    auto apply_P = [&](const double *in, double *out) {
      if (mg_dtype(prec) == PMG_F32)
      {
        // krylov.cpp:152-171
        check_cuda(cudaMemsetAsync(w.flag, 0, sizeof(int), s), "memset");
        launch_d2f(in, w.rf, n, w.flag, sm, s);
        int bad = 0;
        check_cuda(cudaMemcpyAsync(&bad, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
        check_cuda(cudaStreamSynchronize(s), "sync");
        if (bad)
          throw std::runtime_error("mixed_precision_precondition: non-finite value after downcast");
        launch_fill<float>(w.zf, n, 0.0f, sm, s);
        mg_vcycle_f32(prec, Lp, w.zf, w.rf, s);
        launch_f2d(w.zf, out, n, sm, s);
      }
      else
      {
        launch_fill<double>(out, n, 0.0, sm, s);
        mg_vcycle_f64(prec, Lp, out, in, s);
      }
    };

    std::vector<double> hist;
    auto push = [&](double v) { hist.push_back(v); };
    auto flush_hist = [&]() {
      for (int i = 0; i < static_cast<int>(hist.size()) && i < history_cap; ++i)
        if (history)
          history[i] = hist[i];
      if (history && history_cap > 0 && static_cast<int>(hist.size()) < history_cap)
        history[hist.size()] = -1.0;  // terminator
    };

    const double bnorm = nrm(b);
    launch_fill<double>(x, n, 0.0, sm, s);
    int its = 0;
    if (bnorm == 0.0)
    {
      push(0.0);
      if (iterations)
        *iterations = 0;
      flush_hist();
      return;
    }
    check_cuda(cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
    double beta = bnorm;
    push(beta);
    std::vector<double> H((restart + 1) * restart), cs(restart), sn(restart), g(restart + 1);
    auto h = [&](int i, int j) -> double & { return H[i * restart + j]; };
    while (true)
    {
      launch_fill<double>(Vj(0), n, 0.0, sm, s);
      launch_axpby<double>(1.0 / beta, r, 0.0, Vj(0), n, sm, s);
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      std::fill(H.begin(), H.end(), 0.0);
      int j = 0;
      bool happy = false;
      for (; j < restart; ++j)
      {
        if (its >= max_iterations)
        {
          if (iterations)
            *iterations = its;
          flush_hist();
          throw DivergenceErr("gmres: max iterations reached");
        }
        apply_P(Vj(j), Zj(j));
        apply_A(Zj(j), wv);
        ++its;
        const double wnorm0 = nrm(wv);
        for (int i = 0; i <= j; ++i)
        {
          const double hij = dot(wv, Vj(i));
          h(i, j) = hij;
          launch_axpby<double>(-hij, Vj(i), 1.0, wv, n, sm, s);
        }
        double wnorm = nrm(wv);
        if (wnorm * wnorm < (1.0 - 1e-8) * wnorm0 * wnorm0)
        {
          for (int i = 0; i <= j; ++i)
          {
            const double c = dot(wv, Vj(i));
            h(i, j) += c;
            launch_axpby<double>(-c, Vj(i), 1.0, wv, n, sm, s);
          }
          wnorm = nrm(wv);
        }
        h(j + 1, j) = wnorm;
        if (wnorm > 0.0)
        {
          launch_fill<double>(Vj(j + 1), n, 0.0, sm, s);
          launch_axpby<double>(1.0 / wnorm, wv, 0.0, Vj(j + 1), n, sm, s);
        }
        for (int i = 0; i < j; ++i)
        {
          const double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
          h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
          h(i, j) = t;
        }
        const double denom = std::hypot(h(j, j), h(j + 1, j));
        cs[j] = denom == 0.0 ? 1.0 : h(j, j) / denom;
        sn[j] = denom == 0.0 ? 0.0 : h(j + 1, j) / denom;
        h(j, j) = denom;
        h(j + 1, j) = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        const double est = std::fabs(g[j + 1]);
        push(est);
        if (est <= tol * bnorm || wnorm == 0.0)
        {
          happy = wnorm == 0.0;
          ++j;
          break;
        }
      }
      const int mdim = j;
      std::vector<double> y(mdim, 0.0);
      for (int i = mdim - 1; i >= 0; --i)
      {
        double sacc = g[i];
        for (int l = i + 1; l < mdim; ++l)
          sacc -= h(i, l) * y[l];
        y[i] = sacc / h(i, i);
      }
      for (int l = 0; l < mdim; ++l)
        launch_axpby<double>(y[l], Zj(l), 1.0, x, n, sm, s);
      mg_residual_finest(op, x, b, r, s);
      beta = nrm(r);
      hist.back() = beta;
      if (beta <= tol * bnorm || happy)
        break;
      if (its >= max_iterations)
      {
        if (iterations)
          *iterations = its;
        flush_hist();
        throw DivergenceErr("gmres: max iterations reached");
      }
    }
    if (iterations)
      *iterations = its;
    flush_hist();
  });
}

// ---- host-vector entry points (the reference's std::span convention) -------
extern "C" int pmg_gmres_host(pmg_mg op, pmg_mg prec, const double *b, double *x, double tol, int restart,
                              int max_iterations, int *iterations, double *history, int history_cap)
{
  using namespace pmgb;
  DevBuf db, dx;
  int st = capi_guard([&] {
    if (!op || !b || !x)
      throw std::invalid_argument("gmres: invalid arguments");
    DevScope dg(mg_device(op));
    const size_t bytes = static_cast<size_t>(level_total(mg_level_ptr(op, mg_levels(op) - 1))) * sizeof(double);
    db.ensure(bytes);
    dx.ensure(bytes);
    check_cuda(cudaMemcpy(db.p, b, bytes, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(dx.p, x, bytes, cudaMemcpyHostToDevice), "H2D");
  });
  if (st != PMG_OK)
    return st;
  st = pmg_gmres(op, prec, db.p, dx.p, tol, restart, max_iterations, iterations, history, history_cap, nullptr);
  const int st2 = capi_guard([&] {
    DevScope dg(mg_device(op));
    check_cuda(cudaDeviceSynchronize(), "sync");
    check_cuda(cudaMemcpy(x, dx.p, dx.bytes, cudaMemcpyDeviceToHost), "D2H");
  });
  return st != PMG_OK ? st : st2;
}
