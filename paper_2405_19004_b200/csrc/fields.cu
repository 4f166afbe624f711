// Device right-hand side assembly and L2 error for the Poisson model problem
// (SURVEY.md §8f row 2). Replace the host quadrature loops of
// compute_rhs / l2_error (/root/reference/proj/src/operator.cpp:283-411).
//
// * compute_rhs: on the uniform Cartesian level both right-hand sides are
//   separable, b = c (g (x) g (x) g) with the 1D load vector g of 1 or
//   sin(pi x) (host, O(m)) and c = 1 or d pi^2, so the device only forms the
//   tensor power (one pass over N, write-only).
// * l2_error: ||u_h - u||_{L2} with u = prod sin(pi x_a) by the reference's
//   (k+2)-point Gauss rule per cell, evaluated POINTWISE (no cancellation):
//   one thread per cell gathers its (k+1)^d nodal values, contracts them to
//   the (k+2)^d quadrature points direction by direction, and accumulates
//   w (u_h - u)^2; per-CTA partial sums are reduced on the host in a fixed
//   order (deterministic).
#include <cmath>
#include <vector>

#include "../../include/pmg_b200.h"
#include "capi_internal.hpp"
#include "setup.hpp"

namespace pmgb
{
namespace
{

template <typename T>
__global__ void rhs_tensor_kernel(const double *__restrict__ g, T *__restrict__ b, int64_t m, int dim, double c)
{
  pdl_prologue();
  const int64_t N = dim == 3 ? m * m * m : m * m;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < N;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    const int64_t i = idx % m;
    const int64_t r = idx / m;
    const int64_t j = r % m;
    const int64_t l = r / m;
    const double v = dim == 3 ? c * g[l] * g[j] * g[i] : c * g[j] * g[i];
    b[idx] = static_cast<T>(v);
  }
}

constexpr int QMAX = 9;  // k + 2 <= 9

struct QuadData
{
  double shape[QMAX][QMAX];  // [q][t] Lagrange basis t at Gauss point q
  double w[QMAX];            // Gauss weights on [0,1]
  double x[QMAX];            // Gauss points on [0,1]
};

template <int K, int D, typename T>
__global__ void __launch_bounds__(128) l2err_kernel(const __grid_constant__ QuadData Q, const T *__restrict__ x,
                                                    int n, int64_t m, double *__restrict__ partial)
{
  constexpr int NP = K + 1, NQ = K + 2;
  constexpr double PI = 3.14159265358979323846;
  pdl_prologue();
  __shared__ double red[128];
  const int64_t ncell = D == 3 ? static_cast<int64_t>(n) * n * n : static_cast<int64_t>(n) * n;
  const double h = 1.0 / n;
  double acc = 0.0;
  for (int64_t cell = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; cell < ncell;
       cell += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    const int c0 = static_cast<int>(cell % n);
    const int c1 = static_cast<int>((cell / n) % n);
    const int c2 = D == 3 ? static_cast<int>(cell / (static_cast<int64_t>(n) * n)) : 0;
    // nodal values (lattice K c + t, 1-based interior = 0-based index - 1)
    double u[D == 3 ? NP : 1][NP][NP];
#pragma unroll
    for (int t2 = 0; t2 < (D == 3 ? NP : 1); ++t2)
#pragma unroll
      for (int t1 = 0; t1 < NP; ++t1)
#pragma unroll
        for (int t0 = 0; t0 < NP; ++t0)
        {
          const int64_t g0 = static_cast<int64_t>(K) * c0 + t0, g1 = static_cast<int64_t>(K) * c1 + t1,
                        g2 = static_cast<int64_t>(K) * c2 + t2;
          const bool in = g0 >= 1 && g0 <= m && g1 >= 1 && g1 <= m && (D == 2 || (g2 >= 1 && g2 <= m));
          u[t2][t1][t0] = in ? static_cast<double>(x[((D == 3 ? (g2 - 1) * m : 0) + (g1 - 1)) * m + (g0 - 1)]) : 0.0;
        }
    double s0[NQ], s1[NQ], s2[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
    {
      s0[q] = sin(PI * (c0 + Q.x[q]) * h);
      s1[q] = sin(PI * (c1 + Q.x[q]) * h);
      s2[q] = D == 3 ? sin(PI * (c2 + Q.x[q]) * h) : 1.0;
    }
    if constexpr (D == 2)
    {
#pragma unroll
      for (int q1 = 0; q1 < NQ; ++q1)
      {
        double a[NP];  // contract t1 at q1
#pragma unroll
        for (int t0 = 0; t0 < NP; ++t0)
        {
          double v = 0.0;
#pragma unroll
          for (int t1 = 0; t1 < NP; ++t1)
            v = fma(Q.shape[q1][t1], u[0][t1][t0], v);
          a[t0] = v;
        }
#pragma unroll
        for (int q0 = 0; q0 < NQ; ++q0)
        {
          double v = 0.0;
#pragma unroll
          for (int t0 = 0; t0 < NP; ++t0)
            v = fma(Q.shape[q0][t0], a[t0], v);
          const double e = v - s0[q0] * s1[q1];
          acc = fma(Q.w[q0] * Q.w[q1] * h * h, e * e, acc);
        }
      }
    }
    else
    {
#pragma unroll 1
      for (int q2 = 0; q2 < NQ; ++q2)
      {
        double a[NP][NP];  // contract t2 at q2
#pragma unroll
        for (int t1 = 0; t1 < NP; ++t1)
#pragma unroll
          for (int t0 = 0; t0 < NP; ++t0)
          {
            double v = 0.0;
#pragma unroll
            for (int t2 = 0; t2 < NP; ++t2)
              v = fma(Q.shape[q2][t2], u[t2][t1][t0], v);
            a[t1][t0] = v;
          }
#pragma unroll 1
        for (int q1 = 0; q1 < NQ; ++q1)
        {
          double bb[NP];
#pragma unroll
          for (int t0 = 0; t0 < NP; ++t0)
          {
            double v = 0.0;
#pragma unroll
            for (int t1 = 0; t1 < NP; ++t1)
              v = fma(Q.shape[q1][t1], a[t1][t0], v);
            bb[t0] = v;
          }
#pragma unroll
          for (int q0 = 0; q0 < NQ; ++q0)
          {
            double v = 0.0;
#pragma unroll
            for (int t0 = 0; t0 < NP; ++t0)
              v = fma(Q.shape[q0][t0], bb[t0], v);
            const double e = v - s0[q0] * s1[q1] * s2[q2];
            acc = fma(Q.w[q0] * Q.w[q1] * Q.w[q2] * h * h * h, e * e, acc);
          }
        }
      }
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 64; st > 0; st >>= 1)
  {
    if (threadIdx.x < st)
      red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    partial[blockIdx.x] = red[0];
}

template <int K, typename T>
void launch_l2err(int dim, const QuadData &Q, const T *x, int n, int64_t m, double *partial, int grid,
                  cudaStream_t s)
{
  if (dim == 3)
    pdl_launch(l2err_kernel<K, 3, T>, dim3(grid), dim3(128), 0, s, Q, x, n, m, partial);
  else
    pdl_launch(l2err_kernel<K, 2, T>, dim3(grid), dim3(128), 0, s, Q, x, n, m, partial);
  check_launch("l2err_kernel");
}

template <typename T>
void l2err_dispatch(int k, int dim, const QuadData &Q, const T *x, int n, int64_t m, double *partial, int grid,
                    cudaStream_t s)
{
  switch (k)
  {
    case 1: launch_l2err<1, T>(dim, Q, x, n, m, partial, grid, s); break;
    case 2: launch_l2err<2, T>(dim, Q, x, n, m, partial, grid, s); break;
    case 3: launch_l2err<3, T>(dim, Q, x, n, m, partial, grid, s); break;
    case 4: launch_l2err<4, T>(dim, Q, x, n, m, partial, grid, s); break;
    case 5: launch_l2err<5, T>(dim, Q, x, n, m, partial, grid, s); break;
    case 6: launch_l2err<6, T>(dim, Q, x, n, m, partial, grid, s); break;
    default: launch_l2err<7, T>(dim, Q, x, n, m, partial, grid, s); break;
  }
}

}  // namespace
}  // namespace pmgb

using namespace pmgb;

extern "C" int pmg_compute_rhs(pmg_level h, int kind, void *b, void *stream)
{
  return capi_guard([&] {
    if (!h)
      throw std::invalid_argument("compute_rhs: null level");
    if (kind != 0 && kind != 1)
      throw std::invalid_argument("compute_rhs: kind must be 0 (f = 1) or 1 (sine)");
    if (!b)
      throw std::invalid_argument("compute_rhs: null output");
    int dim = 0, k = 0, level = 0, dtype = 0, device = 0;
    level_params(h, &dim, &k, &level, &dtype, &device);
    DevScope dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const auto g = rhs_1d(k, 1 << level, kind == 1);
    const int64_t m = static_cast<int64_t>(g.size());
    double *gd = nullptr;
    check_cuda(cudaMallocAsync(&gd, g.size() * sizeof(double), s), "compute_rhs alloc");
    check_cuda(cudaMemcpyAsync(gd, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice, s),
               "compute_rhs H2D");
    const double c = kind == 1 ? dim * M_PI * M_PI : 1.0;
    const int grid = level_sm_count(h) * 16;
    if (dtype == PMG_F64)
      pdl_launch(rhs_tensor_kernel<double>, dim3(grid), dim3(256), 0, s, static_cast<const double *>(gd),
                 static_cast<double *>(b), m, dim, c);
    else
      pdl_launch(rhs_tensor_kernel<float>, dim3(grid), dim3(256), 0, s, static_cast<const double *>(gd),
                 static_cast<float *>(b), m, dim, c);
    check_launch("rhs_tensor_kernel");
    check_cuda(cudaFreeAsync(gd, s), "compute_rhs free");
  });
}

extern "C" int pmg_l2_error_sin(pmg_level h, const void *x, double *out, void *stream)
{
  return capi_guard([&] {
    if (!h || !x || !out)
      throw std::invalid_argument("l2_error: null argument");
    int dim = 0, k = 0, level = 0, dtype = 0, device = 0;
    level_params(h, &dim, &k, &level, &dtype, &device);
    DevScope dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    QuadData Q{};
    const auto nodes = lobatto_nodes(k);
    std::vector<double> qx, qw;
    gauss_rule(k + 2, qx, qw);
    for (int q = 0; q < k + 2; ++q)
    {
      Q.w[q] = qw[q];
      Q.x[q] = qx[q];
      const auto v = lagrange_eval(nodes, qx[q]);
      for (int t = 0; t <= k; ++t)
        Q.shape[q][t] = v[t];
    }
    const int n = 1 << level;
    const int64_t m = static_cast<int64_t>(n) * k - 1;
    const int grid = level_sm_count(h) * 8;
    double *partial = nullptr;
    check_cuda(cudaMallocAsync(&partial, grid * sizeof(double), s), "l2_error alloc");
    if (dtype == PMG_F64)
      l2err_dispatch<double>(k, dim, Q, static_cast<const double *>(x), n, m, partial, grid, s);
    else
      l2err_dispatch<float>(k, dim, Q, static_cast<const float *>(x), n, m, partial, grid, s);
    std::vector<double> hp(grid);
    check_cuda(cudaMemcpyAsync(hp.data(), partial, grid * sizeof(double), cudaMemcpyDeviceToHost, s),
               "l2_error D2H");
    check_cuda(cudaFreeAsync(partial, s), "l2_error free");
    check_cuda(cudaStreamSynchronize(s), "l2_error sync");
    double sum = 0.0;
    for (double v : hp)
      sum += v;
    *out = std::sqrt(sum);
  });
}

// ---------------------------------------------------------------------------
// General fields (compute_rhs / l2_error with an arbitrary ScalarField,
// operator.cpp:283-411). The field arrives as its values at the reference's
// quadrature points, evaluated by the caller wherever f lives (a host
// std::function in the C++ shim, a torch expression on the device in Python):
//   fq[cell * Q + q], cells lexicographic (direction 0 fastest), Q = (k+2)^d
//   Gauss points per cell, q lexicographic (direction 0 fastest); the point
//   of (cell c, q) is x_a = (c_a + xi_{q_a}) h with xi = pmg_quadrature_rule.
// rhs: C[cell][t] = sum_q w_q |K| f_q prod_a shape[q_a][t_a] (thread per
// (cell, t); the threads of a cell read the same fq, broadcast from L1),
// then b_i = sum over the <= 2^d cells containing node i (thread per node,
// fixed order: deterministic, no atomics).
// l2: thread per (cell, q): u_h(x_q) from the cell's nodal values, w (u_h -
// u_q)^2, per-CTA partial sums added on the host in a fixed order.
// ---------------------------------------------------------------------------
namespace pmgb
{
namespace
{

template <int D>
__global__ void __launch_bounds__(256) rhs_cell_kernel(const __grid_constant__ QuadData Q, int k, int n,
                                                       const double *__restrict__ fq, double *__restrict__ C)
{
  pdl_prologue();
  const int NP = k + 1, NQ = k + 2;
  const int nt = D == 3 ? NP * NP * NP : NP * NP;
  const int nq = D == 3 ? NQ * NQ * NQ : NQ * NQ;
  const int64_t ncell = D == 3 ? static_cast<int64_t>(n) * n * n : static_cast<int64_t>(n) * n;
  const double h = 1.0 / n, jac = D == 3 ? h * h * h : h * h;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < ncell * nt;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    const int64_t cell = e / nt;
    const int t = static_cast<int>(e - cell * nt);
    const int t0 = t % NP, t1 = (t / NP) % NP, t2 = D == 3 ? t / (NP * NP) : 0;
    const double *f = fq + cell * nq;
    double acc = 0.0;
    for (int q2 = 0; q2 < (D == 3 ? NQ : 1); ++q2)
    {
      const double s2 = D == 3 ? Q.w[q2] * Q.shape[q2][t2] : 1.0;
      for (int q1 = 0; q1 < NQ; ++q1)
      {
        const double s12 = s2 * Q.w[q1] * Q.shape[q1][t1];
        double row = 0.0;
        for (int q0 = 0; q0 < NQ; ++q0)
          row = fma(Q.w[q0] * Q.shape[q0][t0], __ldg(f + (q2 * NQ + q1) * NQ + q0), row);
        acc = fma(s12, row, acc);
      }
    }
    C[e] = jac * acc;
  }
}

template <int D, typename T>
__global__ void __launch_bounds__(256) rhs_gather_kernel(int k, int n, int64_t m, const double *__restrict__ C,
                                                         T *__restrict__ b)
{
  pdl_prologue();
  const int NP = k + 1;
  const int nt = D == 3 ? NP * NP * NP : NP * NP;
  const int64_t N = D == 3 ? m * m * m : m * m;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    const int64_t g[3] = {i % m, (i / m) % m, D == 3 ? i / (m * m) : 0};
    // per direction: the cells containing lattice node p = g + 1 and its local index
    int nc[3] = {1, 1, 1}, cc[3][2] = {{0, 0}, {0, 0}, {0, 0}}, tt[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    for (int a = 0; a < D; ++a)
    {
      const int64_t p = g[a] + 1;
      if (p % k == 0)
      {
        nc[a] = 2;
        cc[a][0] = static_cast<int>(p / k) - 1;
        tt[a][0] = k;
        cc[a][1] = static_cast<int>(p / k);
        tt[a][1] = 0;
      }
      else
      {
        cc[a][0] = static_cast<int>(p / k);
        tt[a][0] = static_cast<int>(p % k);
      }
    }
    double s = 0.0;
    for (int j2 = 0; j2 < (D == 3 ? nc[2] : 1); ++j2)
      for (int j1 = 0; j1 < nc[1]; ++j1)
        for (int j0 = 0; j0 < nc[0]; ++j0)
        {
          const int64_t cell = (D == 3 ? static_cast<int64_t>(cc[2][j2]) * n * n : 0) +
                               static_cast<int64_t>(cc[1][j1]) * n + cc[0][j0];
          const int t = ((D == 3 ? tt[2][j2] : 0) * NP + tt[1][j1]) * NP + tt[0][j0];
          s += C[cell * nt + t];
        }
    b[i] = static_cast<T>(s);
  }
}

template <int D, typename T>
__global__ void __launch_bounds__(256) l2err_q_kernel(const __grid_constant__ QuadData Q, int k, int n, int64_t m,
                                                      const T *__restrict__ x, const double *__restrict__ uq,
                                                      double *__restrict__ partial)
{
  pdl_prologue();
  __shared__ double red[256];
  const int NP = k + 1, NQ = k + 2;
  const int nq = D == 3 ? NQ * NQ * NQ : NQ * NQ;
  const int64_t ncell = D == 3 ? static_cast<int64_t>(n) * n * n : static_cast<int64_t>(n) * n;
  const double h = 1.0 / n, jac = D == 3 ? h * h * h : h * h;
  double acc = 0.0;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < ncell * nq;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    const int64_t cell = e / nq;
    const int q = static_cast<int>(e - cell * nq);
    const int q0 = q % NQ, q1 = (q / NQ) % NQ, q2 = D == 3 ? q / (NQ * NQ) : 0;
    const int c0 = static_cast<int>(cell % n), c1 = static_cast<int>((cell / n) % n),
              c2 = D == 3 ? static_cast<int>(cell / (static_cast<int64_t>(n) * n)) : 0;
    double uh = 0.0;
    for (int t2 = 0; t2 < (D == 3 ? NP : 1); ++t2)
    {
      const int64_t g2 = static_cast<int64_t>(k) * c2 + t2;
      if (D == 3 && (g2 < 1 || g2 > m))
        continue;
      const double s2 = D == 3 ? Q.shape[q2][t2] : 1.0;
      for (int t1 = 0; t1 < NP; ++t1)
      {
        const int64_t g1 = static_cast<int64_t>(k) * c1 + t1;
        if (g1 < 1 || g1 > m)
          continue;
        double row = 0.0;
        for (int t0 = 0; t0 < NP; ++t0)
        {
          const int64_t g0 = static_cast<int64_t>(k) * c0 + t0;
          if (g0 < 1 || g0 > m)
            continue;
          row = fma(Q.shape[q0][t0], static_cast<double>(x[((D == 3 ? (g2 - 1) * m : 0) + (g1 - 1)) * m + (g0 - 1)]),
                    row);
        }
        uh = fma(s2 * Q.shape[q1][t1], row, uh);
      }
    }
    const double err = uh - uq[e];
    const double w = jac * Q.w[q0] * Q.w[q1] * (D == 3 ? Q.w[q2] : 1.0);
    acc = fma(w, err * err, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1)
  {
    if (threadIdx.x < st)
      red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    partial[blockIdx.x] = red[0];
}

QuadData quad_data(int k)
{
  QuadData Q{};
  const auto nodes = lobatto_nodes(k);
  std::vector<double> qx, qw;
  gauss_rule(k + 2, qx, qw);
  for (int q = 0; q < k + 2; ++q)
  {
    Q.w[q] = qw[q];
    Q.x[q] = qx[q];
    const auto v = lagrange_eval(nodes, qx[q]);
    for (int t = 0; t <= k; ++t)
      Q.shape[q][t] = v[t];
  }
  return Q;
}

}  // namespace
}  // namespace pmgb

extern "C" int pmg_quadrature_rule(int degree, double *points, double *weights)
{
  return capi_guard([&] {
    if (degree < 1 || degree > 7 || !points || !weights)
      throw std::invalid_argument("quadrature_rule: invalid arguments");
    const QuadData Q = quad_data(degree);
    for (int q = 0; q < degree + 2; ++q)
    {
      points[q] = Q.x[q];
      weights[q] = Q.w[q];
    }
  });
}

extern "C" int pmg_compute_rhs_q(pmg_level h, const double *fq, void *b, void *stream)
{
  return capi_guard([&] {
    if (!h || !fq || !b)
      throw std::invalid_argument("compute_rhs: null argument");
    int dim = 0, k = 0, level = 0, dtype = 0, device = 0;
    level_params(h, &dim, &k, &level, &dtype, &device);
    DevScope dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const QuadData Q = quad_data(k);
    const int n = 1 << level;
    const int64_t m = static_cast<int64_t>(n) * k - 1;
    const int64_t ncell = dim == 3 ? static_cast<int64_t>(n) * n * n : static_cast<int64_t>(n) * n;
    const int64_t nt = dim == 3 ? static_cast<int64_t>(k + 1) * (k + 1) * (k + 1) : static_cast<int64_t>(k + 1) * (k + 1);
    double *C = nullptr;
    check_cuda(cudaMallocAsync(&C, static_cast<size_t>(ncell * nt) * sizeof(double), s), "compute_rhs alloc");
    const int grid = level_sm_count(h) * 16;
    if (dim == 3)
      pdl_launch(rhs_cell_kernel<3>, dim3(grid), dim3(256), 0, s, Q, k, n, fq, C);
    else
      pdl_launch(rhs_cell_kernel<2>, dim3(grid), dim3(256), 0, s, Q, k, n, fq, C);
    check_launch("rhs_cell_kernel");
    if (dtype == PMG_F64)
    {
      if (dim == 3)
        pdl_launch(rhs_gather_kernel<3, double>, dim3(grid), dim3(256), 0, s, k, n, m, static_cast<const double *>(C),
                   static_cast<double *>(b));
      else
        pdl_launch(rhs_gather_kernel<2, double>, dim3(grid), dim3(256), 0, s, k, n, m, static_cast<const double *>(C),
                   static_cast<double *>(b));
    }
    else
    {
      if (dim == 3)
        pdl_launch(rhs_gather_kernel<3, float>, dim3(grid), dim3(256), 0, s, k, n, m, static_cast<const double *>(C),
                   static_cast<float *>(b));
      else
        pdl_launch(rhs_gather_kernel<2, float>, dim3(grid), dim3(256), 0, s, k, n, m, static_cast<const double *>(C),
                   static_cast<float *>(b));
    }
    check_launch("rhs_gather_kernel");
    check_cuda(cudaFreeAsync(C, s), "compute_rhs free");
  });
}

extern "C" int pmg_l2_error_q(pmg_level h, const void *x, const double *uq, double *out, void *stream)
{
  return capi_guard([&] {
    if (!h || !x || !uq || !out)
      throw std::invalid_argument("l2_error: null argument");
    int dim = 0, k = 0, level = 0, dtype = 0, device = 0;
    level_params(h, &dim, &k, &level, &dtype, &device);
    DevScope dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const QuadData Q = quad_data(k);
    const int n = 1 << level;
    const int64_t m = static_cast<int64_t>(n) * k - 1;
    const int grid = level_sm_count(h) * 8;
    double *partial = nullptr;
    check_cuda(cudaMallocAsync(&partial, grid * sizeof(double), s), "l2_error alloc");
    if (dtype == PMG_F64)
    {
      if (dim == 3)
        pdl_launch(l2err_q_kernel<3, double>, dim3(grid), dim3(256), 0, s, Q, k, n, m, static_cast<const double *>(x),
                   uq, partial);
      else
        pdl_launch(l2err_q_kernel<2, double>, dim3(grid), dim3(256), 0, s, Q, k, n, m, static_cast<const double *>(x),
                   uq, partial);
    }
    else
    {
      if (dim == 3)
        pdl_launch(l2err_q_kernel<3, float>, dim3(grid), dim3(256), 0, s, Q, k, n, m, static_cast<const float *>(x), uq,
                   partial);
      else
        pdl_launch(l2err_q_kernel<2, float>, dim3(grid), dim3(256), 0, s, Q, k, n, m, static_cast<const float *>(x), uq,
                   partial);
    }
    check_launch("l2err_q_kernel");
    std::vector<double> hp(grid);
    check_cuda(cudaMemcpyAsync(hp.data(), partial, grid * sizeof(double), cudaMemcpyDeviceToHost, s), "l2_error D2H");
    check_cuda(cudaFreeAsync(partial, s), "l2_error free");
    check_cuda(cudaStreamSynchronize(s), "l2_error sync");
    double sum = 0.0;
    for (double v : hp)
      sum += v;
    *out = std::sqrt(sum);
  });
}
