// 2D vertex-patch smoother with one thread per patch, for low degree (sm_100a).
//
// In 2D a Q_k patch (closure (2k+1)^2, interior (2k-1)^2) is small enough for
// one thread to hold it in registers for k <= 2, so the per-patch body of the
// reference's fused / boundary smoother (smoother.cpp:109-148) runs without
// shared memory or barriers: closure rows read through L1 (no patch of a
// colour reads a node another patch of the colour writes, so the read-only
// path is legal within a launch), the even-odd contractions of the line
// kernels (smoother_impl.cuh) in registers, x^I stored directly. Bound by HBM
// (x read once per colour), like the k = 1 point kernel.
#pragma once

#include "smoother_impl.cuh"

namespace pmgb
{

template <int K, typename T, int MODE>
__global__ void __launch_bounds__(128) vp_patch2d_kernel(const __grid_constant__ PatchMatsEO<T, K> P,
                                                         const __grid_constant__ ColorArgs<T> a)
{
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  pdl_prologue();
  const int j0 = blockIdx.x * 32 + threadIdx.x;
  const int j1 = blockIdx.y * 4 + threadIdx.y;
  if (j0 >= a.np[0] || j1 >= a.np[1])
    return;
  const int64_t m = a.m;
  // closure origin g_a = k (v_a - 1) - 1, v_a = 2 j_a + vb_a (patches.cpp:71)
  const int g0 = K * (2 * j0 + a.vb[0] - 1) - 1;
  const int g1 = K * (2 * j1 + a.vb[1] - 1) - 1;
  // dir 0 on every closure row: zM = M0 u, zA = A0 u
  T zm[NC][NI], za[NC][NI];
  T xold[NI][NI];
#pragma unroll
  for (int t1 = 0; t1 < NC; ++t1)
  {
    const int y = g1 + t1;
    const bool oky = static_cast<unsigned>(y) < static_cast<unsigned>(m);
    const T *row = a.x + static_cast<int64_t>(y) * m + g0;
    T u[NC], ue[K + 1], uo[K];
#pragma unroll
    for (int t0 = 0; t0 < NC; ++t0)
    {
      const bool ok = oky && static_cast<unsigned>(g0 + t0) < static_cast<unsigned>(m);
      bool inner = t0 >= 1 && t0 <= NC - 2 && t1 >= 1 && t1 <= NC - 2;
      T v = ok ? __ldg(row + t0) : T(0);
      if (inner)
        xold[t1 - 1][t0 - 1] = v;
      if constexpr (MODE == MODE_BOUNDARY)  // never reads x^I (smoother.cpp:128-148)
        v = inner ? T(0) : v;
      u[t0] = v;
    }
    eo_split<NC>(u, ue, uo);
    eo_rows<K>(P.Me, P.Mo, ue, uo, zm[t1]);
    eo_rows<K>(P.Ae, P.Ao, ue, uo, za[t1]);
  }
  // dir 1 per interior column: r = b - (A1 zM + M1 zA); then S^T along dir 1
  T y[NI][NI];  // [c1][i0]
#pragma unroll
  for (int i0 = 0; i0 < NI; ++i0)
  {
    T cm[NC], ca[NC], cme[K + 1], cmo[K], cae[K + 1], cao[K], acc[NI], r[NI], yh[NI];
#pragma unroll
    for (int t1 = 0; t1 < NC; ++t1)
    {
      cm[t1] = zm[t1][i0];
      ca[t1] = za[t1][i0];
    }
    eo_split<NC>(cm, cme, cmo);
    eo_split<NC>(ca, cae, cao);
    eo_rows2<K>(P.Ae, P.Ao, cme, cmo, P.Me, P.Mo, cae, cao, acc);
    const T *bc = a.b + static_cast<int64_t>(g1 + 1) * m + (g0 + 1 + i0);
#pragma unroll
    for (int i1 = 0; i1 < NI; ++i1)
      r[i1] = __ldg(bc + i1 * m) - acc[i1];
    eo_st<K>(P.Se, P.So, r, yh);
#pragma unroll
    for (int c1 = 0; c1 < NI; ++c1)
      y[c1][i0] = yh[c1];
  }
  // dir 0: S^T, scale by 1/(lambda sums), S; then S along dir 1; update
  T v[NI][NI];  // [c1][i0]
#pragma unroll
  for (int c1 = 0; c1 < NI; ++c1)
  {
    T yh[NI];
    eo_st<K>(P.Se, P.So, y[c1], yh);
#pragma unroll
    for (int c0 = 0; c0 < NI; ++c0)
      yh[c0] *= __ldg(a.inv + c0 + NI * c1);
    eo_s<K>(P.Se, P.So, yh, v[c1]);
  }
#pragma unroll
  for (int i0 = 0; i0 < NI; ++i0)
  {
    T col[NI], out[NI];
#pragma unroll
    for (int c1 = 0; c1 < NI; ++c1)
      col[c1] = v[c1][i0];
    eo_s<K>(P.Se, P.So, col, out);
    T *xp = a.x + static_cast<int64_t>(g1 + 1) * m + (g0 + 1 + i0);
#pragma unroll
    for (int i1 = 0; i1 < NI; ++i1)
    {
      if constexpr (MODE == MODE_BOUNDARY)
        xp[i1 * m] = out[i1];
      else
        xp[i1 * m] = xold[i1][i0] + out[i1];
    }
  }
}

template <int K, typename T, int MODE>
void launch_vp_patch2d(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a, cudaStream_t s)
{
  if (a.total == 0)
    return;
  const dim3 block(32, 4, 1);
  const dim3 grid((a.np[0] + 31) / 32, (a.np[1] + 3) / 4, 1);
  pdl_launch(vp_patch2d_kernel<K, T, MODE>, grid, block, 0, s, P, a);
  check_launch("vp_patch2d_kernel");
}

}  // namespace pmgb
