// Level-vector kernels: deterministic reductions and elementwise updates.
//
// vector_norm (/root/reference/proj/src/multigrid.cpp:260-266) and the dot /
// axpy / cast loops of the Krylov driver (krylov.cpp:13-171). Reductions are
// two-pass with a fixed grid and a fixed tree, so results are bitwise
// reproducible run to run (no atomics), accumulated in f64.
#include "blas.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace pmgb
{

namespace
{

constexpr int RED_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(RED_THREADS)
    dot_partial_kernel(const T *__restrict__ a, const T *__restrict__ b, int64_t n,
                       double *__restrict__ partial)
{
  __shared__ double sh[RED_THREADS];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x;
  const int64_t hi = min(n, lo + per);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += RED_THREADS)
    s = fma(static_cast<double>(a[i]), static_cast<double>(b[i]), s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = RED_THREADS / 2; w > 0; w >>= 1)
  {
    if (threadIdx.x < w)
      sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    partial[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(RED_THREADS)
    finish_kernel(const double *__restrict__ partial, int np, double *__restrict__ out, int sqrt_it)
{
  __shared__ double sh[RED_THREADS];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += RED_THREADS)
    s += partial[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = RED_THREADS / 2; w > 0; w >>= 1)
  {
    if (threadIdx.x < w)
      sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    *out = sqrt_it ? sqrt(sh[0]) : sh[0];
}

template <typename T>
__global__ void fill_kernel(T *x, int64_t n, T v)
{
  pdl_prologue();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = v;
}

// y = alpha * x + beta * y
template <typename T>
__global__ void axpby_kernel(T alpha, const T *__restrict__ x, T beta, T *__restrict__ y, int64_t n)
{
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = alpha * x[i] + beta * y[i];
}

// y = alpha_dev[0] * x + y  (device-side coefficient, for graph-friendly MGS)
__global__ void axpy_dev_kernel(const double *__restrict__ alpha, double scale,
                                const double *__restrict__ x, double *__restrict__ y, int64_t n)
{
  const double a = scale * alpha[0];
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

__global__ void d2f_kernel(const double *__restrict__ x, float *__restrict__ y, int64_t n,
                           int *__restrict__ nonfinite)
{
  int bad = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    const float v = static_cast<float>(x[i]);
    if (!isfinite(v))
      bad = 1;
    y[i] = v;
  }
  if (bad)
    *nonfinite = 1;  // benign race: every writer stores 1
}

__global__ void f2d_kernel(const float *__restrict__ x, double *__restrict__ y, int64_t n)
{
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = static_cast<double>(x[i]);
}

unsigned ew_grid(int64_t n, int sm_count)
{
  const int64_t b = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, static_cast<int64_t>(sm_count) * 16)));
}

}  // namespace

template <typename T>
void launch_dot(const T *a, const T *b, int64_t n, double *partial, double *out, bool sqrt_it,
                cudaStream_t s)
{
  dot_partial_kernel<T><<<RED_BLOCKS, RED_THREADS, 0, s>>>(a, b, n, partial);
  check_launch("dot_partial_kernel");
  finish_kernel<<<1, RED_THREADS, 0, s>>>(partial, RED_BLOCKS, out, sqrt_it ? 1 : 0);
  check_launch("finish_kernel");
}

template <typename T>
void launch_fill(T *x, int64_t n, T v, int sm_count, cudaStream_t s)
{
  if (n == 0)
    return;
  pdl_launch(fill_kernel<T>, ew_grid(n, sm_count), 256, 0, s, x, n, v);
  check_launch("fill_kernel");
}

template <typename T>
void launch_axpby(T alpha, const T *x, T beta, T *y, int64_t n, int sm_count, cudaStream_t s)
{
  axpby_kernel<T><<<ew_grid(n, sm_count), 256, 0, s>>>(alpha, x, beta, y, n);
  check_launch("axpby_kernel");
}

void launch_axpy_dev(const double *alpha, double scale, const double *x, double *y, int64_t n,
                     int sm_count, cudaStream_t s)
{
  axpy_dev_kernel<<<ew_grid(n, sm_count), 256, 0, s>>>(alpha, scale, x, y, n);
  check_launch("axpy_dev_kernel");
}

void launch_d2f(const double *x, float *y, int64_t n, int *nonfinite, int sm_count, cudaStream_t s)
{
  d2f_kernel<<<ew_grid(n, sm_count), 256, 0, s>>>(x, y, n, nonfinite);
  check_launch("d2f_kernel");
}

void launch_f2d(const float *x, double *y, int64_t n, int sm_count, cudaStream_t s)
{
  f2d_kernel<<<ew_grid(n, sm_count), 256, 0, s>>>(x, y, n);
  check_launch("f2d_kernel");
}

// x = M b with the coarse V-cycle operator M (n x n, row-major, row pitch
// ld = n rounded up to 4, zero padded). One warp per row streams the row in
// 16-byte vectors, two batches of 4 per lane in flight (software-pipelined),
// evict-first (the operator is read once per application and should not
// displace the level vectors in L2); b is staged once per CTA in shared
// memory; fixed shuffle-tree reduction (deterministic). The first batch is
// issued before the programmatic-dependency wait: M is not written by the
// predecessor kernel, so its stream starts while that kernel drains.
template <typename T>
__global__ void __launch_bounds__(256) coarse_gemv_kernel(const T *__restrict__ M, const T *__restrict__ b,
                                                         T *__restrict__ x, int n, int ld)
{
  using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  constexpr int W = 16 / sizeof(T), U = 4;
  extern __shared__ __align__(16) unsigned char gemv_smem[];
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const bool active = row < n;
  const V *mr = reinterpret_cast<const V *>(M + static_cast<int64_t>(active ? row : 0) * ld);
  const int nv = ld / W;
  const int nfull = nv / (32 * U);  // full U-batches of this row
  V cur[U], nxt[U];
  if (active && nfull > 0)
  {
#pragma unroll
    for (int u = 0; u < U; ++u)
      cur[u] = __ldcg(mr + lane + 32 * u);  // before the PDL wait: L2 only
  }
  pdl_prologue();
  T *bs = reinterpret_cast<T *>(gemv_smem);  // [ld], zero padded
  for (int j = threadIdx.x; j < ld; j += blockDim.x)
    bs[j] = j < n ? b[j] : T(0);
  __syncthreads();
  if (!active)
    return;
  const V *bv = reinterpret_cast<const V *>(bs);
  T acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    acc[u] = T(0);
  for (int t = 0; t < nfull; ++t)
  {
    const int c = lane + 32 * U * t;
    if (t + 1 < nfull)
    {
#pragma unroll
      for (int u = 0; u < U; ++u)
        nxt[u] = __ldcs(mr + c + 32 * U + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
    {
      const V bb = bv[c + 32 * u];
      const T *mm = reinterpret_cast<const T *>(&cur[u]);
      const T *bq = reinterpret_cast<const T *>(&bb);
#pragma unroll
      for (int w = 0; w < W; ++w)
        acc[u] = fma(mm[w], bq[w], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      cur[u] = nxt[u];
  }
  for (int c = lane + 32 * U * nfull; c < nv; c += 32)
  {
    const V mv = __ldcs(mr + c);
    const V bb = bv[c];
    const T *mm = reinterpret_cast<const T *>(&mv);
    const T *bq = reinterpret_cast<const T *>(&bb);
#pragma unroll
    for (int w = 0; w < W; ++w)
      acc[0] = fma(mm[w], bq[w], acc[0]);
  }
  T sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0)
    x[row] = sum;
}

// Same product, the operator streamed by TMA (1D cp.async.bulk, completion on
// an mbarrier transaction count): each warp owns one shared-memory row
// buffer, its lane 0 issues the bulk copy of the warp's next row as soon as
// the lanes have consumed the current one, so every SM keeps NW rows
// (~NW x 27 KB at 3375 unknowns) in flight with no register staging; the
// first rows are requested before the programmatic-dependency wait. The dot
// product and its reduction are coarse_gemv_kernel's per-lane order.
__device__ __forceinline__ unsigned gv_smem(const void *p)
{
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <typename T>
__global__ void __launch_bounds__(256, 1) coarse_gemv_bulk_kernel(const T *__restrict__ M, const T *__restrict__ b,
                                                                 T *__restrict__ x, int n, int ld)
{
  using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  constexpr int W = 16 / sizeof(T), U = 4;
  extern __shared__ __align__(128) unsigned char gb_smem[];
  __shared__ __align__(8) unsigned long long full[8];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned row_bytes = static_cast<unsigned>(ld * sizeof(T));
  T *bs = reinterpret_cast<T *>(gb_smem);
  T *rowbuf = bs + ld + ((16 / sizeof(T)) - (ld % (16 / sizeof(T)))) % (16 / sizeof(T)) + 0;
  T *mine = rowbuf + static_cast<size_t>(warp) * ld;
  const unsigned bar = gv_smem(&full[warp]);
  const int G = gridDim.x;
  int row = blockIdx.x + warp * G;
  if (lane == 0)
  {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (row < n)
    {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(row_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       gv_smem(mine)),
                   "l"(M + static_cast<int64_t>(row) * ld), "r"(row_bytes), "r"(bar)
                   : "memory");
    }
  }
  pdl_prologue();
  for (int j = threadIdx.x; j < ld; j += blockDim.x)
    bs[j] = j < n ? b[j] : T(0);
  __syncthreads();
  const V *bv = reinterpret_cast<const V *>(bs);
  const V *mv = reinterpret_cast<const V *>(mine);
  const int nv = ld / W;
  unsigned phase = 0;
  for (; row < n; row += nw * G)
  {
    // wait for this warp's row
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(bar), "r"(phase)
                   : "memory");
    phase ^= 1u;
    T acc[U] = {T(0), T(0), T(0), T(0)};
    int c = lane;
    for (; c + 32 * (U - 1) < nv; c += 32 * U)
    {
#pragma unroll
      for (int u = 0; u < U; ++u)
      {
        const V m4 = mv[c + 32 * u], b4 = bv[c + 32 * u];
        const T *mm = reinterpret_cast<const T *>(&m4);
        const T *bq = reinterpret_cast<const T *>(&b4);
#pragma unroll
        for (int w = 0; w < W; ++w)
          acc[u] = fma(mm[w], bq[w], acc[u]);
      }
    }
    for (; c < nv; c += 32)
    {
      const V m4 = mv[c], b4 = bv[c];
      const T *mm = reinterpret_cast<const T *>(&m4);
      const T *bq = reinterpret_cast<const T *>(&b4);
#pragma unroll
      for (int w = 0; w < W; ++w)
        acc[0] = fma(mm[w], bq[w], acc[0]);
    }
    T sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const int nrow = row + nw * G;
    __syncwarp();  // every lane's reads of the buffer are done (their values fed the sum)
    if (lane == 0)
    {
      x[row] = sum;
      if (nrow < n)
      {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(row_bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(gv_smem(mine)),
            "l"(M + static_cast<int64_t>(nrow) * ld), "r"(row_bytes), "r"(bar)
            : "memory");
      }
    }
    __syncwarp();
  }
}

template <typename T>
__global__ void unit_kernel(T *x, int n, int j)
{
  pdl_prologue();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = i == j ? T(1) : T(0);
}

// e_j with j read from device memory (column counter of a replayed graph)
template <typename T>
__global__ void unit_dev_kernel(T *x, int n, const int *__restrict__ j)
{
  pdl_prologue();
  const int jj = *j;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = i == jj ? T(1) : T(0);
}

// column *j of M (row pitch ld) = v, then ++*j (one CTA: the increment
// follows every read)
template <typename T>
__global__ void __launch_bounds__(1024) store_column_kernel(T *__restrict__ M, const T *__restrict__ v, int n, int ld,
                                                            int *j)
{
  pdl_prologue();
  const int jj = *j;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    M[static_cast<int64_t>(i) * ld + jj] = v[i];
  __syncthreads();
  if (threadIdx.x == 0)
    *j = jj + 1;
}

template <typename T>
void launch_unit_dev(T *x, int n, const int *j, cudaStream_t s)
{
  pdl_launch(unit_dev_kernel<T>, dim3((n + 255) / 256), dim3(256), 0, s, x, n, j);
  check_launch("unit_dev_kernel");
}

template <typename T>
void launch_store_column(T *M, const T *v, int n, int ld, int *j, cudaStream_t s)
{
  pdl_launch(store_column_kernel<T>, dim3(1), dim3(1024), 0, s, M, v, n, ld, j);
  check_launch("store_column_kernel");
}

template void launch_unit_dev<double>(double *, int, const int *, cudaStream_t);
template void launch_unit_dev<float>(float *, int, const int *, cudaStream_t);
template void launch_store_column<double>(double *, const double *, int, int, int *, cudaStream_t);
template void launch_store_column<float>(float *, const float *, int, int, int *, cudaStream_t);

template <typename T>
void launch_coarse_gemv(const T *M, const T *b, T *x, int n, int ld, cudaStream_t s)
{
  // TMA-streamed variant: measured faster for f32 (11.7 vs 13.0 us at 3375
  // unknowns), slower for f64 (26.9 vs 23.8 us; profiles/r02/ab/gemv/bulk.txt);
  // PMG_GEMV_BULK=0 / 1 forces either
  static const int bulk_env = [] {
    const char *e = std::getenv("PMG_GEMV_BULK");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  const bool bulk = bulk_env < 0 ? sizeof(T) == 4 : bulk_env == 1;
  if (bulk)
  {
    // b + one row buffer per warp, up to 8 warps within 220 KB
    const size_t rowb = static_cast<size_t>(ld) * sizeof(T);
    const size_t budget = 220 * 1024;
    const int nw = static_cast<int>(std::min<size_t>(8, (budget - rowb - 16) / rowb));
    if (nw >= 2)
    {
      const size_t smem = rowb + 16 + static_cast<size_t>(nw) * rowb;
      static unsigned bmask = 0;
      if (first_on_device(bmask))
        check_cuda(cudaFuncSetAttribute(coarse_gemv_bulk_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(budget + 1024)),
                   "cudaFuncSetAttribute(coarse_gemv_bulk)");
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const int grid = std::max(1, std::min(nsm, (n + nw - 1) / nw));
      pdl_launch(coarse_gemv_bulk_kernel<T>, dim3(grid), dim3(32 * nw), smem, s, M, b, x, n, ld);
      check_launch("coarse_gemv_bulk_kernel");
      return;
    }
  }
  const size_t smem = static_cast<size_t>(ld) * sizeof(T);
  static unsigned attr_mask = 0;
  if (first_on_device(attr_mask))
    check_cuda(cudaFuncSetAttribute(coarse_gemv_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024),
               "cudaFuncSetAttribute(coarse_gemv)");
  pdl_launch(coarse_gemv_kernel<T>, dim3((n + 7) / 8), dim3(256), smem, s, M, b, x, n, ld);
  check_launch("coarse_gemv_kernel");
}

template <typename T>
void launch_unit(T *x, int n, int j, cudaStream_t s)
{
  pdl_launch(unit_kernel<T>, dim3((n + 255) / 256), dim3(256), 0, s, x, n, j);
  check_launch("unit_kernel");
}

template void launch_coarse_gemv<double>(const double *, const double *, double *, int, int, cudaStream_t);
template void launch_coarse_gemv<float>(const float *, const float *, float *, int, int, cudaStream_t);
template void launch_unit<double>(double *, int, int, cudaStream_t);
template void launch_unit<float>(float *, int, int, cudaStream_t);
template void launch_dot<double>(const double *, const double *, int64_t, double *, double *, bool, cudaStream_t);
template void launch_dot<float>(const float *, const float *, int64_t, double *, double *, bool, cudaStream_t);
template void launch_fill<double>(double *, int64_t, double, int, cudaStream_t);
template void launch_fill<float>(float *, int64_t, float, int, cudaStream_t);
template void launch_axpby<double>(double, const double *, double, double *, int64_t, int, cudaStream_t);
template void launch_axpby<float>(float, const float *, float, float *, int64_t, int, cudaStream_t);

}  // namespace pmgb
