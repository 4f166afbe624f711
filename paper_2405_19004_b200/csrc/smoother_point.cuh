// Degree-1 vertex-patch smoother as a point stencil (2D / 3D) for sm_100a.
//
// For k = 1 a vertex patch has a single interior node c (the vertex itself,
// g_a = k (v_a - 1) - 1 + 1 = v_a - 1, patches.cpp:71) and a 3^d closure, so
// the reference's fused body (smoother.cpp:109-126) collapses to
//   r = b_c - sum_j w_j x_j          w = interior row of A-bar (fastdiag.cpp:199-233)
//   x_c += coef r                    coef = S^(2d) / (sum of eigenvalues) (fastdiag.cpp:164-192)
// with the 3^d weights w = A (x) M (x) M + M (x) A (x) M + M (x) M (x) A of the
// 1 x 3 interior rows M, A precomputed on the host in f64. The boundary
// variant (smoother.cpp:128-148) drops the w_c x_c term and replaces x_c.
//
// One thread per patch, every closure value read straight from L1/L2 (the
// closure of a patch never contains a node written by another patch of the
// same colour, so the read-only path is legal within a launch). There is no
// shared-memory staging: the kernel is bounded by HBM (x read once per colour).
#pragma once

#include "common.cuh"

namespace pmgb
{

template <typename T>
struct PointStencil
{
  T w[27];  // [t2][t1][t0] (3D) or [t1][t0] (2D), t in {0,1,2} = closure-local offset
  T coef;
};

// patches per thread (consecutive rows j1, independent stencils in flight):
// 2 in f32 (3D Q1 L9 83 -> 92 GDoF/s, 2D Q1 L14 124 -> 166), 1 in f64 (2
// costs 4-12% there: profiles/r02/ab/point_ppt.txt)
template <typename T>
constexpr int point_ppt()
{
  return sizeof(T) == 4 ? 2 : 1;
}

// patch (j0, j1, j2) of the colour a
template <int D, typename T, int MODE>
__device__ __forceinline__ void point_patch(const PointStencil<T> &st, const ColorArgs<T> &a, int j0, int j1, int j2)
{
  const int64_t m = a.m;
  // centre node c_a = v_a - 1, v_a = 2 j_a + vb_a
  const int c0 = 2 * j0 + a.vb[0] - 1;
  const int c1 = 2 * j1 + a.vb[1] - 1;
  const int64_t c2g = D == 3 ? 2 * j2 + a.vb[2] - 1 : 0;  // global plane
  const int64_t c2 = c2g - a.zoff;                          // local plane in x / b
  const int64_t mlast = D == 3 ? a.mz : 1;
  const int64_t plane = D == 3 ? m * m : 0;
  const T *xc = a.x + c2 * plane + static_cast<int64_t>(c1) * m + c0;

  const bool okx0 = c0 >= 1, okx2 = c0 + 1 < m;
  T acc = T(0);
  T xcen = T(0);
#pragma unroll
  for (int t2 = 0; t2 < (D == 3 ? 3 : 1); ++t2)
  {
    const bool okz = D == 2 || static_cast<uint64_t>(c2g + t2 - 1) < static_cast<uint64_t>(mlast);
#pragma unroll
    for (int t1 = 0; t1 < 3; ++t1)
    {
      const bool oky = okz && static_cast<unsigned>(c1 + t1 - 1) < static_cast<unsigned>(m);
      const T *row = xc + (D == 3 ? (t2 - 1) * plane : 0) + (t1 - 1) * m;
      const T *w = st.w + (D == 3 ? 9 * t2 : 0) + 3 * t1;
      const T xl = (oky && okx0) ? __ldg(row - 1) : T(0);
      const T xm = oky ? __ldg(row) : T(0);
      const T xr = (oky && okx2) ? __ldg(row + 1) : T(0);
      acc = fma(w[0], xl, acc);
      if (t1 == 1 && (D == 2 || t2 == 1))
        xcen = xm;
      if constexpr (MODE != MODE_BOUNDARY)
        acc = fma(w[1], xm, acc);
      else if (!(t1 == 1 && (D == 2 || t2 == 1)))
        acc = fma(w[1], xm, acc);
      acc = fma(w[2], xr, acc);
    }
  }
  const T r = __ldg(a.b + (xc - a.x)) - acc;
  T *xo = a.x + (xc - a.x);
  if constexpr (MODE == MODE_BOUNDARY)
    *xo = st.coef * r;
  else
    *xo = fma(st.coef, r, xcen);
}

template <int D, typename T, int MODE>
__global__ void __launch_bounds__(128) vp_point_kernel(const __grid_constant__ PointStencil<T> st,
                                                       const __grid_constant__ ColorArgs<T> a)
{
  pdl_prologue();
  const int j0 = blockIdx.x * 32 + threadIdx.x;
  const int j2 = D == 3 ? static_cast<int>(blockIdx.z) : 0;
  if (j0 >= a.np[0])
    return;
#pragma unroll
  for (int q = 0; q < point_ppt<T>(); ++q)
  {
    const int j1 = (blockIdx.y * 4 + threadIdx.y) * point_ppt<T>() + q;
    if (j1 < a.np[1])
      point_patch<D, T, MODE>(st, a, j0, j1, j2);
  }
}

template <int D, typename T, int MODE>
void launch_vp_point(const PointStencil<T> &st, const ColorArgs<T> &a, cudaStream_t s)
{
  if (a.total == 0)
    return;
  dim3 block(32, 4, 1);
  dim3 grid((a.np[0] + 31) / 32, (a.np[1] + 4 * point_ppt<T>() - 1) / (4 * point_ppt<T>()), D == 3 ? a.np[2] : 1);
  pdl_launch(vp_point_kernel<D, T, MODE>, grid, block, 0, s, st, a);
  check_launch("vp_point_kernel");
}

}  // namespace pmgb
