// Point Gauss-Seidel smoother and CSR assembly:
//   point_gauss_seidel   /root/reference/proj/src/smoother.cpp:160-166
//   gauss_seidel_sweep   /root/reference/proj/src/sparse.cpp:31-47
//   assemble_sparse      /root/reference/proj/src/operator.cpp:194-281
//   kind == point_gs     /root/reference/proj/src/multigrid.cpp:286-300
//
// The reference sweeps the rows of an assembled CSR matrix in lexicographic
// order. On a uniform level the matrix is the Kronecker sum of the banded 1D
// chain matrices (the identity level_op3d_kernel uses), so the device sweep
// needs no CSR: a row's couplings are the window of nodes of the cells around
// it, their values products of the 1D band rows (lattice residue r = p mod k,
// offset q - p + k), computed per entry in the reference's order.
//
// Exact lexicographic order on the device: a node depends on its neighbours
// before it (new values) and after it (old values). Couplings reach at most k
// nodes per direction, so the wavefront number
//   t = i0 + (k+1) i1 [+ (k+1)^2 i2]
// increases strictly along every such dependency (k - (k+1) < 0 and
// k + (k+1) k - (k+1)^2 < 0): nodes of one front are independent, and
// sweeping the fronts in order with a barrier between them gives the
// reference's sweep, row by row. The front lists are built once on the host.
// The sweep is one persistent CTA, one warp per row (the level sizes the
// reference's 1e7-nonzero budget admits are desk scale; a front holds at most
// a few thousand rows). Within a row the couplings are summed by the lanes
// and a butterfly instead of the reference's running subtraction, so the
// sweep agrees with it to rounding (1e-12 tested), not bitwise.
#include <algorithm>
#include <memory>
#include <stdexcept>
#include <vector>

#include "capi_internal.hpp"

namespace pmgb
{

struct GsData
{
  int dim = 3, k = 1;
  int64_t m = 1;
  int nfronts = 0;
  DevBuf order;  // int32 node ids, front by front
  DevBuf fptr;   // int32 front offsets (nfronts + 1)
  DevBuf band;   // double: mass band | stiffness band, k * (2k+1) each
};

namespace
{

constexpr int GS_THREADS = 1024;

// 1D window of couplings of lattice node p (1-based): the nodes of the
// cell(s) containing it (operator.cpp:200-207 by behaviour)
__host__ __device__ inline void gs_window(int p, int k, int n, int &lo, int &hi)
{
  const int c_lo = (p % k == 0) ? p / k - 1 : p / k;
  const int c_hi = p / k;
  lo = max(1, c_lo * k);
  hi = min(n * k - 1, (min(c_hi, n - 1) + 1) * k);
}

// one warp per row: the lanes split the row's couplings (the window of up to
// (2k+1)^d nodes), a butterfly reduction adds the partial sums; the fronts
// are swept in order, all warps of the CTA on the rows of one front
template <int D>
__global__ void __launch_bounds__(GS_THREADS)
    gs_sweep_kernel(const double *__restrict__ band, int k, int m, const int *__restrict__ order,
                    const int *__restrict__ fptr, int nfronts, double *x, const double *__restrict__ b)
{
  __shared__ double sb[2 * 7 * 15];
  const int w = 2 * k + 1, nb = k * w;
  for (int e = threadIdx.x; e < 2 * nb; e += blockDim.x)
    sb[e] = band[e];
  __syncthreads();
  const double *bm = sb, *ba = sb + nb;
  const int n = (m + 1) / k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int f = 0; f < nfronts; ++f)
  {
    const int e1 = fptr[f + 1];
    for (int e = fptr[f] + warp; e < e1; e += nwarps)
    {
      const int i = order[e];
      int g[3] = {i % m, (i / m) % m, D == 3 ? i / (m * m) : 0};
      int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      for (int a = 0; a < D; ++a)
        gs_window(g[a] + 1, k, n, lo[a], hi[a]);
      const int p0 = g[0] + 1, p1 = g[1] + 1, p2 = g[2] + 1;
      const double *m0 = bm + (p0 % k) * w, *a0 = ba + (p0 % k) * w;
      const double *m1 = bm + (p1 % k) * w, *a1 = ba + (p1 % k) * w;
      const double *m2 = bm + (p2 % k) * w, *a2 = ba + (p2 % k) * w;
      const int w0 = hi[0] - lo[0] + 1, w1 = hi[1] - lo[1] + 1;
      const int nw = w0 * w1 * (D == 3 ? hi[2] - lo[2] + 1 : 1);
      double part = 0.0, diag = 0.0;
      for (int t = lane; t < nw; t += 32)
      {
        const int t0 = t % w0, t1 = (t / w0) % w1, t2 = t / (w0 * w1);
        const int q0 = lo[0] + t0, q1 = lo[1] + t1, q2 = (D == 3 ? lo[2] : 0) + t2;
        const int o0 = q0 - p0 + k, o1 = q1 - p1 + k, o2 = q2 - p2 + k;
        // sum over directions of the product with the stiffness factor in that
        // direction, in the reference's order (operator.cpp:248-257)
        double v;
        if (D == 3)
          v = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a0[o0], m1[o1]), m2[o2]),
                                  __dmul_rn(__dmul_rn(m0[o0], a1[o1]), m2[o2])),
                        __dmul_rn(__dmul_rn(m0[o0], m1[o1]), a2[o2]));
        else
          v = __dadd_rn(__dmul_rn(a0[o0], m1[o1]), __dmul_rn(m0[o0], a1[o1]));
        const int64_t col = D == 3 ? (static_cast<int64_t>(q2 - 1) * m + (q1 - 1)) * m + (q0 - 1)
                                   : static_cast<int64_t>(q1 - 1) * m + (q0 - 1);
        if (col == i)
          diag = v;
        else
          part = fma(v, x[col], part);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
      {
        part += __shfl_xor_sync(0xffffffffu, part, o);
        diag += __shfl_xor_sync(0xffffffffu, diag, o);  // one lane holds it, the others 0
      }
      if (lane == 0)
        x[i] = (b[i] - part) / diag;
    }
    __syncthreads();  // the next front reads this front's new values
  }
}

int64_t nnz_estimate(int dim, int k, int level, double &est)
{
  const int n = 1 << level;
  const int m = n * k - 1;
  int64_t width_sum = 0;
  for (int p = 1; p <= m; ++p)
  {
    int lo, hi;
    gs_window(p, k, n, lo, hi);
    width_sum += hi - lo + 1;
  }
  est = 1.0;
  for (int a = 0; a < dim; ++a)
    est *= static_cast<double>(width_sum);
  return width_sum;
}

void check_budget(int dim, int k, int level)
{
  double est = 0;
  nnz_estimate(dim, k, level, est);
  if (est > 1e7)  // operator.cpp:209-227 (std::runtime_error)
    throw std::runtime_error("assemble_sparse: nonzero budget of 1e7 exceeded");
}

}  // namespace

// builds the front lists / bands of a level once (throws the reference's
// budget error for levels the CSR oracle could not hold)
GsData *gs_data(pmg_level l)
{
  std::shared_ptr<GsData> &slot = level_gs_slot(l);
  if (slot)
    return slot.get();
  const LevelSetup &S = level_setup(l);
  if (level_dtype(l) != PMG_F64)
    throw std::invalid_argument("point Gauss-Seidel runs in f64 only");
  check_budget(S.dim, S.k, S.level);
  auto g = std::make_shared<GsData>();
  g->dim = S.dim;
  g->k = S.k;
  g->m = S.m;
  const int64_t N = S.N, m = S.m;
  const int64_t w1 = S.k + 1, w2 = w1 * w1;
  const int64_t T = S.dim == 3 ? (m - 1) * (1 + w1 + w2) + 1 : (m - 1) * (1 + w1) + 1;
  std::vector<int> cnt(T + 1, 0), order(N);
  auto front = [&](int64_t i) {
    const int64_t i0 = i % m, i1 = (i / m) % m, i2 = S.dim == 3 ? i / (m * m) : 0;
    return i0 + w1 * i1 + w2 * i2;
  };
  for (int64_t i = 0; i < N; ++i)
    ++cnt[front(i) + 1];
  for (int64_t t = 0; t < T; ++t)
    cnt[t + 1] += cnt[t];
  std::vector<int> pos(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < N; ++i)
    order[pos[front(i)]++] = static_cast<int>(i);
  g->nfronts = static_cast<int>(T);
  DevScope dg(level_device(l));
  g->order.ensure(N * sizeof(int));
  g->fptr.ensure((T + 1) * sizeof(int));
  std::vector<double> band(S.band_mass);
  band.insert(band.end(), S.band_stiff.begin(), S.band_stiff.end());
  g->band.ensure(band.size() * sizeof(double));
  check_cuda(cudaMemcpy(g->order.p, order.data(), N * sizeof(int), cudaMemcpyHostToDevice), "H2D");
  check_cuda(cudaMemcpy(g->fptr.p, cnt.data(), (T + 1) * sizeof(int), cudaMemcpyHostToDevice), "H2D");
  check_cuda(cudaMemcpy(g->band.p, band.data(), band.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D");
  slot = g;
  return g.get();
}

void gs_smooth(pmg_level l, double *x, const double *b, cudaStream_t s)
{
  GsData *g = gs_data(l);
  if (g->dim == 3)
    gs_sweep_kernel<3><<<1, GS_THREADS, 0, s>>>(g->band.as<double>(), g->k, static_cast<int>(g->m),
                                                 g->order.as<int>(), g->fptr.as<int>(), g->nfronts, x, b);
  else
    gs_sweep_kernel<2><<<1, GS_THREADS, 0, s>>>(g->band.as<double>(), g->k, static_cast<int>(g->m),
                                                 g->order.as<int>(), g->fptr.as<int>(), g->nfronts, x, b);
  check_launch("gs_sweep_kernel");
}

}  // namespace pmgb

using namespace pmgb;

extern "C" {

int pmg_point_gauss_seidel(pmg_level h, void *x, const void *b, void *stream)
{
  return capi_guard([&] {
    if (!h || !x || !b)
      throw std::invalid_argument("point_gauss_seidel: invalid arguments");
    DevScope dg(level_device(h));
    gs_smooth(h, static_cast<double *>(x), static_cast<const double *>(b), static_cast<cudaStream_t>(stream));
  });
}

int pmg_point_gauss_seidel_host(pmg_level h, double *x, const double *b)
{
  return capi_guard([&] {
    if (!h || !x || !b)
      throw std::invalid_argument("point_gauss_seidel: invalid arguments");
    DevScope dg(level_device(h));
    const size_t bytes = static_cast<size_t>(level_total(h)) * sizeof(double);
    DevBuf dx, db;
    dx.ensure(bytes);
    db.ensure(bytes);
    check_cuda(cudaMemcpy(dx.p, x, bytes, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(db.p, b, bytes, cudaMemcpyHostToDevice), "H2D");
    gs_smooth(h, dx.as<double>(), db.as<double>(), nullptr);
    check_cuda(cudaMemcpy(x, dx.p, bytes, cudaMemcpyDeviceToHost), "D2H");
  });
}

// CSR of the level operator in the reference's row / column order
// (assemble_sparse, operator.cpp:194-281). Call with row_ptr = cols = vals =
// NULL to get *nnz; then again with arrays of N + 1 / nnz / nnz entries.
int pmg_assemble_sparse_host(int dim, int degree, int level, int64_t *row_ptr, int32_t *cols, double *vals,
                             int64_t *nnz)
{
  return capi_guard([&] {
    if (!nnz || (dim != 2 && dim != 3) || degree < 1 || degree > 7 || level < 1)
      throw std::invalid_argument("assemble_sparse: invalid arguments");
    check_budget(dim, degree, level);
    const LevelSetup S = make_level_setup(dim, degree, level);
    const int k = degree, n = S.n, w = 2 * k + 1;
    const int64_t m = S.m;
    std::vector<int> lo(m), hi(m);
    for (int64_t p = 1; p <= m; ++p)
      gs_window(static_cast<int>(p), k, n, lo[p - 1], hi[p - 1]);
    int64_t count = 0;
    const bool fill = row_ptr && cols && vals;
    if (fill)
      row_ptr[0] = 0;
    for (int64_t row = 0; row < S.N; ++row)
    {
      const int64_t g0 = row % m, g1 = (row / m) % m, g2 = dim == 3 ? row / (m * m) : 0;
      const int64_t p[3] = {g0 + 1, g1 + 1, g2 + 1};
      const int l2 = dim == 3 ? lo[g2] : 0, h2 = dim == 3 ? hi[g2] : 0;
      for (int q2 = l2; q2 <= h2; ++q2)
        for (int q1 = lo[g1]; q1 <= hi[g1]; ++q1)
          for (int q0 = lo[g0]; q0 <= hi[g0]; ++q0)
          {
            if (fill)
            {
              const int q[3] = {q0, q1, q2};
              double v = 0.0;
              for (int dir = 0; dir < dim; ++dir)
              {
                double t = 1.0;
                for (int a = 0; a < dim; ++a)
                {
                  const int r = static_cast<int>(p[a] % k), o = static_cast<int>(q[a] - p[a] + k);
                  t *= (a == dir ? S.band_stiff : S.band_mass)[r * w + o];
                }
                v += t;
              }
              cols[count] = static_cast<int32_t>((dim == 3 ? (static_cast<int64_t>(q2 - 1) * m + (q1 - 1)) * m
                                                           : static_cast<int64_t>(q1 - 1) * m) +
                                                 (q0 - 1));
              vals[count] = v;
            }
            ++count;
          }
      if (fill)
        row_ptr[row + 1] = count;
    }
    *nnz = count;
  });
}

}  // extern "C"
