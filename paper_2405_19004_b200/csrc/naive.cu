// Straightforward global-memory vertex-patch smoother (the comparator the
// north star's ">= 2x" target is measured against).
//
// It is the reference's fused per-patch body (smoother.cpp:109-126) moved
// onto the GPU as directly as possible: one CTA per patch, the closure and all
// contraction temporaries live in a global-memory scratch slice, every
// tensor_contract (tensor.hpp:27-91) is a thread-strided loop over output
// entries reading the 1D matrix from global memory, with the reference's
// exact contraction sequence (fastdiag.cpp:199-233 then :164-192). Runtime
// degree, no templates, no shared memory, no register blocking.
#include "common.cuh"
#include "naive.cuh"

namespace pmgb
{

namespace
{

template <typename T>
__device__ void g_contract(int dim, int dir, const T *mat, int rows, int cols, bool transpose,
                           bool add, const T *x, const int *ext, T *y)
{
  const int n_in = transpose ? rows : cols;
  const int n_out = transpose ? cols : rows;
  int inner = 1, outer = 1;
  for (int a = 0; a < dir; ++a)
    inner *= ext[a];
  for (int a = dir + 1; a < dim; ++a)
    outer *= ext[a];
  const int total = inner * n_out * outer;
  for (int e = threadIdx.x; e < total; e += blockDim.x)
  {
    const int s = e % inner;
    const int i = (e / inner) % n_out;
    const int o = e / (inner * n_out);
    T sum = T(0);
    for (int k = 0; k < n_in; ++k)
    {
      const T w = transpose ? mat[k * cols + i] : mat[i * cols + k];
      sum += w * x[(static_cast<int64_t>(o) * n_in + k) * inner + s];
    }
    T *dst = y + (static_cast<int64_t>(o) * n_out + i) * inner + s;
    *dst = add ? *dst + sum : sum;
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(128) naive_smooth_kernel(NaiveArgs<T> a)
{
  const int d = a.dim, k = a.k;
  const int nc = 2 * k + 1, ni = 2 * k - 1;
  int ncd = 1, nid = 1;
  for (int q = 0; q < d; ++q)
  {
    ncd *= nc;
    nid *= ni;
  }
  T *closure = a.scratch + static_cast<int64_t>(blockIdx.x) * a.scratch_stride;
  T *z = closure + ncd;
  T *t = z + ncd;
  T *t2 = t + ncd;
  T *res = t2 + ncd;
  T *sol = res + nid;
  const int64_t m = a.c.m;
  for (int patch = blockIdx.x; patch < a.c.total; patch += gridDim.x)
  {
    int j[3] = {0, 0, 0};
    {
      int rest = patch;
      j[0] = rest % a.c.np[0];
      rest /= a.c.np[0];
      j[1] = rest % a.c.np[1];
      j[2] = rest / a.c.np[1];
    }
    int64_t g[3] = {0, 0, 0};
    for (int q = 0; q < d; ++q)
      g[q] = static_cast<int64_t>(k) * (2 * j[q] + a.c.vb[q] - 1) - 1;
    // gather closure (patches.cpp:51-95) and b interior
    for (int e = threadIdx.x; e < ncd; e += blockDim.x)
    {
      int rem = e;
      int64_t gi = 0, stride = 1;
      bool inside = true;
      for (int q = 0; q < d; ++q)
      {
        const int tq = rem % nc;
        rem /= nc;
        const int64_t gq = g[q] + tq;
        if (gq < 0 || gq >= m)
          inside = false;
        gi += gq * stride;
        stride *= m;
      }
      closure[e] = inside ? a.c.x[gi] : T(0);
    }
    for (int e = threadIdx.x; e < nid; e += blockDim.x)
    {
      int rem = e;
      int64_t gi = 0, stride = 1;
      for (int q = 0; q < d; ++q)
      {
        const int tq = rem % ni + 1;
        rem /= ni;
        gi += (g[q] + tq) * stride;
        stride *= m;
      }
      res[e] = a.c.b[gi];
    }
    __syncthreads();
    // apply_patch_operator (fastdiag.cpp:199-233), reference sequence
    int ext[3] = {nc, nc, nc};
    T *opout = sol;
    if (d == 2)
    {
      int e1[3] = {ni, nc, 1};
      g_contract(2, 0, a.Mif, ni, nc, false, false, closure, ext, z);
      g_contract(2, 1, a.Aif, ni, nc, false, false, z, e1, opout);
      g_contract(2, 0, a.Aif, ni, nc, false, false, closure, ext, z);
      g_contract(2, 1, a.Mif, ni, nc, false, true, z, e1, opout);
    }
    else
    {
      int e1[3] = {ni, nc, nc};
      int e2[3] = {ni, ni, nc};
      g_contract(3, 0, a.Mif, ni, nc, false, false, closure, ext, z);
      g_contract(3, 1, a.Mif, ni, nc, false, false, z, e1, t);
      g_contract(3, 2, a.Aif, ni, nc, false, false, t, e2, opout);
      g_contract(3, 1, a.Aif, ni, nc, false, false, z, e1, t);
      g_contract(3, 2, a.Mif, ni, nc, false, true, t, e2, opout);
      g_contract(3, 0, a.Aif, ni, nc, false, false, closure, ext, z);
      g_contract(3, 1, a.Mif, ni, nc, false, false, z, e1, t2);
      g_contract(3, 2, a.Mif, ni, nc, false, true, t2, e2, opout);
    }
    for (int e = threadIdx.x; e < nid; e += blockDim.x)
      res[e] -= opout[e];
    __syncthreads();
    // apply_patch_inverse (fastdiag.cpp:164-192)
    int ei[3] = {ni, ni, ni};
    T *bufs[2] = {z, t};
    const T *src = res;
    for (int q = 0; q < d; ++q)
    {
      T *dst = bufs[q % 2];
      g_contract(d, q, a.S, ni, ni, true, false, src, ei, dst);
      src = dst;
    }
    T *mid = const_cast<T *>(src);
    for (int e = threadIdx.x; e < nid; e += blockDim.x)
      mid[e] *= a.c.inv[e];
    __syncthreads();
    for (int q = 0; q < d; ++q)
    {
      T *dst = (q == d - 1) ? sol : ((src == z) ? t : z);
      g_contract(d, q, a.S, ni, ni, false, false, src, ei, dst);
      src = dst;
    }
    // scatter_interior add (patches.cpp:97-121)
    for (int e = threadIdx.x; e < nid; e += blockDim.x)
    {
      int rem = e;
      int64_t gi = 0, stride = 1;
      for (int q = 0; q < d; ++q)
      {
        const int tq = rem % ni + 1;
        rem /= ni;
        gi += (g[q] + tq) * stride;
        stride *= m;
      }
      a.c.x[gi] += sol[e];
    }
    __syncthreads();
  }
}

}  // namespace

template <typename T>
int64_t naive_scratch_per_block(int dim, int k)
{
  int64_t nc = 2 * k + 1, ni = 2 * k - 1, ncd = 1, nid = 1;
  for (int q = 0; q < dim; ++q)
  {
    ncd *= nc;
    nid *= ni;
  }
  return 4 * ncd + 2 * nid;
}

template <typename T>
void launch_naive_smooth(const NaiveArgs<T> &a, int grid, cudaStream_t s)
{
  if (a.c.total == 0)
    return;
  naive_smooth_kernel<T><<<std::min(grid, a.c.total), 128, 0, s>>>(a);
  check_launch("naive_smooth_kernel");
}

template int64_t naive_scratch_per_block<double>(int, int);
template int64_t naive_scratch_per_block<float>(int, int);
template void launch_naive_smooth<double>(const NaiveArgs<double> &, int, cudaStream_t);
template void launch_naive_smooth<float>(const NaiveArgs<float> &, int, cudaStream_t);

}  // namespace pmgb
