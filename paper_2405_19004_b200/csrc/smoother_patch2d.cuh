// 2D vertex-patch smoother with one thread per patch, for low degree (sm_100a).
//
// In 2D a Q_k patch (closure (2k+1)^2, interior (2k-1)^2) is small enough for
// one thread to hold it in registers for k <= 3 (closure rows are streamed,
// the dir-1 contraction accumulated row pair by row pair), so the per-patch body of the
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

// k <= 2: the whole closure's dir-0 contractions are kept in registers
template <int K, typename T, int MODE>
__device__ __forceinline__ void patch2d_regs(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a)
{
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
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

// k >= 3: closure rows streamed, dir 1 accumulated row pair by row pair
template <int K, typename T, int MODE>
__device__ __forceinline__ void patch2d_stream(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a)
{
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  constexpr int HO = K > 1 ? K - 1 : 1;
  const int j0 = blockIdx.x * 32 + threadIdx.x;
  const int j1 = blockIdx.y * 4 + threadIdx.y;
  if (j0 >= a.np[0] || j1 >= a.np[1])
    return;
  const int64_t m = a.m;
  // closure origin g_a = k (v_a - 1) - 1, v_a = 2 j_a + vb_a (patches.cpp:71)
  const int g0 = K * (2 * j0 + a.vb[0] - 1) - 1;
  const int g1 = K * (2 * j1 + a.vb[1] - 1) - 1;
  // closure row t1 -> dir 0 contractions zM = M0 u, zA = A0 u
  auto row = [&](int t1, T (&zm)[NI], T (&za)[NI]) {
    const int y = g1 + t1;
    const bool oky = static_cast<unsigned>(y) < static_cast<unsigned>(m);
    const T *rp = a.x + static_cast<int64_t>(y) * m + g0;
    T u[NC], ue[K + 1], uo[K];
#pragma unroll
    for (int t0 = 0; t0 < NC; ++t0)
    {
      const bool ok = oky && static_cast<unsigned>(g0 + t0) < static_cast<unsigned>(m);
      T v = ok ? __ldg(rp + t0) : T(0);
      if constexpr (MODE == MODE_BOUNDARY)  // never reads x^I (smoother.cpp:128-148)
        v = (t0 >= 1 && t0 <= NC - 2 && t1 >= 1 && t1 <= NC - 2) ? T(0) : v;
      u[t0] = v;
    }
    eo_split<NC>(u, ue, uo);
    eo_rows<K>(P.Me, P.Mo, ue, uo, zm);
    eo_rows<K>(P.Ae, P.Ao, ue, uo, za);
  };
  // dir 1, accumulated row pair by row pair (even-odd in dir 1):
  // acc = A1 zM + M1 zA, even part E[h][i0], odd part O[h][i0]
  T E[K][NI], O[HO][NI];
#pragma unroll
  for (int jj = 0; jj <= K; ++jj)
  {
    T zma[NI], zaa[NI];
    row(jj, zma, zaa);
    if (jj < K)
    {
      T zmb[NI], zab[NI];
      row(NC - 1 - jj, zmb, zab);
#pragma unroll
      for (int i = 0; i < NI; ++i)
      {
        const T zme = zma[i] + zmb[i], zmo = zma[i] - zmb[i];
        const T zae = zaa[i] + zab[i], zao = zaa[i] - zab[i];
#pragma unroll
        for (int h = 0; h < K; ++h)
          E[h][i] = jj == 0 ? fma(P.Ae[h][jj], zme, P.Me[h][jj] * zae)
                            : fma(P.Ae[h][jj], zme, fma(P.Me[h][jj], zae, E[h][i]));
#pragma unroll
        for (int h = 0; h < K - 1; ++h)
          O[h][i] = jj == 0 ? fma(P.Ao[h][jj], zmo, P.Mo[h][jj] * zao)
                            : fma(P.Ao[h][jj], zmo, fma(P.Mo[h][jj], zao, O[h][i]));
      }
    }
    else
    {
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int h = 0; h < K; ++h)
          E[h][i] = fma(P.Ae[h][K], zma[i], fma(P.Me[h][K], zaa[i], E[h][i]));
    }
  }
  // r = b - acc; S^T along dir 1 (per column i0)
  T y[NI][NI];  // [c1][i0]
  const T *bb = a.b + static_cast<int64_t>(g1 + 1) * m + (g0 + 1);
#pragma unroll
  for (int i0 = 0; i0 < NI; ++i0)
  {
    T r[NI], yh[NI];
#pragma unroll
    for (int h = 0; h < K; ++h)
    {
      if (h < K - 1)
      {
        r[h] = __ldg(bb + h * m + i0) - (E[h][i0] + O[h][i0]);
        r[NI - 1 - h] = __ldg(bb + (NI - 1 - h) * m + i0) - (E[h][i0] - O[h][i0]);
      }
      else
        r[h] = __ldg(bb + h * m + i0) - E[h][i0];
    }
    eo_st<K>(P.Se, P.So, r, yh);
#pragma unroll
    for (int c1 = 0; c1 < NI; ++c1)
      y[c1][i0] = yh[c1];
  }
  // dir 0: S^T, scale by 1/(lambda sums), S (per eigen row c1)
#pragma unroll
  for (int c1 = 0; c1 < NI; ++c1)
  {
    T yh[NI], v[NI];
    eo_st<K>(P.Se, P.So, y[c1], yh);
#pragma unroll
    for (int c0 = 0; c0 < NI; ++c0)
      yh[c0] *= __ldg(a.inv + c0 + NI * c1);
    eo_s<K>(P.Se, P.So, yh, v);
#pragma unroll
    for (int i0 = 0; i0 < NI; ++i0)
      y[c1][i0] = v[i0];
  }
  // S along dir 1, x^I update (x^I_old re-read: only this thread writes it)
  T *xp = a.x + static_cast<int64_t>(g1 + 1) * m + (g0 + 1);
#pragma unroll
  for (int i0 = 0; i0 < NI; ++i0)
  {
    T col[NI], out[NI];
#pragma unroll
    for (int c1 = 0; c1 < NI; ++c1)
      col[c1] = y[c1][i0];
    eo_s<K>(P.Se, P.So, col, out);
#pragma unroll
    for (int i1 = 0; i1 < NI; ++i1)
    {
      if constexpr (MODE == MODE_BOUNDARY)
        xp[i1 * m + i0] = out[i1];
      else
        xp[i1 * m + i0] = __ldg(xp + i1 * m + i0) + out[i1];
    }
  }
}

template <int K, typename T, int MODE>
__global__ void __launch_bounds__(128) vp_patch2d_kernel(const __grid_constant__ PatchMatsEO<T, K> P,
                                                         const __grid_constant__ ColorArgs<T> a)
{
  pdl_prologue();
  if constexpr (K <= 2)
    patch2d_regs<K, T, MODE>(P, a);
  else
    patch2d_stream<K, T, MODE>(P, a);
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

namespace pmgb
{

// ---------------------------------------------------------------------------
// 3D, one thread per patch (k = 2): the closure is streamed plane by plane
// (z-planes t2, rows t1 through L1), each plane contracted in dir 0 (per row)
// and dir 1 (row pairs, even-odd) to wMM, wS (NI x NI), and dir 2 accumulated
// densely into the NI^3 residual; then the 3D fast-diagonalisation solve in
// registers and the x^I update. No shared memory, no barriers.
// ---------------------------------------------------------------------------
// S^T M_if, S^T A_if with eigen rows in the even-first order (capi.cu level_init)
template <typename T, int K>
struct PatchST
{
  T M[2 * K - 1][2 * K + 1];
  T A[2 * K - 1][2 * K + 1];
};

template <int K, typename T, int MODE>
__global__ void __launch_bounds__(128, 3) vp_patch3d_kernel(const __grid_constant__ PatchMatsEO<T, K> P,
                                                            const __grid_constant__ ColorArgs<T> a,
                                                            const __grid_constant__ PatchST<T, K> D)
{
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  constexpr int HO = K > 1 ? K - 1 : 1;
  pdl_prologue();
  const int j0 = blockIdx.x * 32 + threadIdx.x;
  const int j1 = blockIdx.y * 4 + threadIdx.y;
  const int j2 = blockIdx.z;
  if (j0 >= a.np[0] || j1 >= a.np[1])
    return;
  const int64_t m = a.m, m2 = m * m;
  const int g0 = K * (2 * j0 + a.vb[0] - 1) - 1;
  const int g1 = K * (2 * j1 + a.vb[1] - 1) - 1;
  const int64_t g2 = static_cast<int64_t>(K) * (2 * j2 + a.vb[2] - 1) - 1;  // global plane
  T acc[NI][NI][NI];  // [i2][i1][i0]: A-bar x on the interior
#pragma unroll
  for (int t2 = 0; t2 < NC; ++t2)
  {
    const bool okz = static_cast<uint64_t>(g2 + t2) < static_cast<uint64_t>(a.mz);
    const T *pl = a.x + (g2 + t2 - a.zoff) * m2;
    auto row = [&](int t1, T (&zm)[NI], T (&za)[NI]) {
      const int y = g1 + t1;
      const bool oky = okz && static_cast<unsigned>(y) < static_cast<unsigned>(m);
      const T *rp = pl + static_cast<int64_t>(y) * m + g0;
      T u[NC], ue[K + 1], uo[K];
#pragma unroll
      for (int t0 = 0; t0 < NC; ++t0)
      {
        const bool ok = oky && static_cast<unsigned>(g0 + t0) < static_cast<unsigned>(m);
        T v = ok ? __ldg(rp + t0) : T(0);
        if constexpr (MODE == MODE_BOUNDARY)  // never reads x^I (smoother.cpp:128-148)
          v = (t0 >= 1 && t0 <= NC - 2 && t1 >= 1 && t1 <= NC - 2 && t2 >= 1 && t2 <= NC - 2) ? T(0) : v;
        u[t0] = v;
      }
      eo_split<NC>(u, ue, uo);
      eo_rows<K>(P.Me, P.Mo, ue, uo, zm);
      eo_rows<K>(P.Ae, P.Ao, ue, uo, za);
    };
    // dir 1 (row pairs): wMM = M1 zM (Em/Om), wS = A1 zM + M1 zA (Es/Os)
    T Em[K][NI], Om[HO][NI], Es[K][NI], Os[HO][NI];
#pragma unroll
    for (int jj = 0; jj <= K; ++jj)
    {
      T zma[NI], zaa[NI];
      row(jj, zma, zaa);
      if (jj < K)
      {
        T zmb[NI], zab[NI];
        row(NC - 1 - jj, zmb, zab);
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
          const T zme = zma[i] + zmb[i], zmo = zma[i] - zmb[i];
          const T zae = zaa[i] + zab[i], zao = zaa[i] - zab[i];
#pragma unroll
          for (int h = 0; h < K; ++h)
          {
            Em[h][i] = jj == 0 ? P.Me[h][jj] * zme : fma(P.Me[h][jj], zme, Em[h][i]);
            Es[h][i] = jj == 0 ? fma(P.Ae[h][jj], zme, P.Me[h][jj] * zae)
                               : fma(P.Ae[h][jj], zme, fma(P.Me[h][jj], zae, Es[h][i]));
          }
#pragma unroll
          for (int h = 0; h < K - 1; ++h)
          {
            Om[h][i] = jj == 0 ? P.Mo[h][jj] * zmo : fma(P.Mo[h][jj], zmo, Om[h][i]);
            Os[h][i] = jj == 0 ? fma(P.Ao[h][jj], zmo, P.Mo[h][jj] * zao)
                               : fma(P.Ao[h][jj], zmo, fma(P.Mo[h][jj], zao, Os[h][i]));
          }
        }
      }
      else
      {
#pragma unroll
        for (int i = 0; i < NI; ++i)
#pragma unroll
          for (int h = 0; h < K; ++h)
          {
            Em[h][i] = fma(P.Me[h][K], zma[i], Em[h][i]);
            Es[h][i] = fma(P.Ae[h][K], zma[i], fma(P.Me[h][K], zaa[i], Es[h][i]));
          }
      }
    }
    // dir 2 and S^T along dir 2 in one step: acc[c2] += (S^T A2)[c2][t2] wMM + (S^T M2)[c2][t2] wS
#pragma unroll
    for (int h = 0; h < K; ++h)
    {
#pragma unroll
      for (int i = 0; i < NI; ++i)
      {
        const int r1 = h, r2 = NI - 1 - h;
        const T wm1 = h < K - 1 ? Em[h][i] + Om[h][i] : Em[h][i];
        const T ws1 = h < K - 1 ? Es[h][i] + Os[h][i] : Es[h][i];
        const T wm2 = h < K - 1 ? Em[h][i] - Om[h][i] : T(0);
        const T ws2 = h < K - 1 ? Es[h][i] - Os[h][i] : T(0);
#pragma unroll
        for (int i2 = 0; i2 < NI; ++i2)
        {
          const T cA = D.A[i2][t2], cM = D.M[i2][t2];
          acc[i2][r1][i] = t2 == 0 ? fma(cA, wm1, cM * ws1) : fma(cA, wm1, fma(cM, ws1, acc[i2][r1][i]));
          if (h < K - 1)
            acc[i2][r2][i] = t2 == 0 ? fma(cA, wm2, cM * ws2) : fma(cA, wm2, fma(cM, ws2, acc[i2][r2][i]));
        }
      }
    }
  }
  // S^T_2 r = S^T_2 b - acc, then the rest of (S x S x S) diag(1/sum lambda) (S x S x S)^T r
  const T *bb = a.b + (g2 + 1 - a.zoff) * m2 + static_cast<int64_t>(g1 + 1) * m + (g0 + 1);
#pragma unroll
  for (int i1 = 0; i1 < NI; ++i1)
#pragma unroll
    for (int i0 = 0; i0 < NI; ++i0)
    {
      T v[NI], y[NI];
#pragma unroll
      for (int i2 = 0; i2 < NI; ++i2)
        v[i2] = __ldg(bb + i2 * m2 + i1 * m + i0);
      eo_st<K>(P.Se, P.So, v, y);
#pragma unroll
      for (int c2 = 0; c2 < NI; ++c2)
        acc[c2][i1][i0] = y[c2] - acc[c2][i1][i0];
    }
  // S^T along dir 1
#pragma unroll
  for (int c2 = 0; c2 < NI; ++c2)
#pragma unroll
    for (int i0 = 0; i0 < NI; ++i0)
    {
      T v[NI], y[NI];
#pragma unroll
      for (int i1 = 0; i1 < NI; ++i1)
        v[i1] = acc[c2][i1][i0];
      eo_st<K>(P.Se, P.So, v, y);
#pragma unroll
      for (int i1 = 0; i1 < NI; ++i1)
        acc[c2][i1][i0] = y[i1];
    }
  // dir 0: S^T, scale, S
#pragma unroll
  for (int c2 = 0; c2 < NI; ++c2)
#pragma unroll
    for (int c1 = 0; c1 < NI; ++c1)
    {
      T y[NI];
      eo_st<K>(P.Se, P.So, acc[c2][c1], y);
#pragma unroll
      for (int c0 = 0; c0 < NI; ++c0)
        y[c0] *= __ldg(a.inv + c0 + NI * (c1 + NI * c2));
      eo_s<K>(P.Se, P.So, y, acc[c2][c1]);
    }
  // S along dir 1
#pragma unroll
  for (int c2 = 0; c2 < NI; ++c2)
#pragma unroll
    for (int i0 = 0; i0 < NI; ++i0)
    {
      T v[NI], y[NI];
#pragma unroll
      for (int c1 = 0; c1 < NI; ++c1)
        v[c1] = acc[c2][c1][i0];
      eo_s<K>(P.Se, P.So, v, y);
#pragma unroll
      for (int i1 = 0; i1 < NI; ++i1)
        acc[c2][i1][i0] = y[i1];
    }
  // S along dir 2, update (x^I_old re-read: only this thread writes it)
  T *xp = a.x + (g2 + 1 - a.zoff) * m2 + static_cast<int64_t>(g1 + 1) * m + (g0 + 1);
#pragma unroll
  for (int i1 = 0; i1 < NI; ++i1)
#pragma unroll
    for (int i0 = 0; i0 < NI; ++i0)
    {
      T v[NI], y[NI];
#pragma unroll
      for (int c2 = 0; c2 < NI; ++c2)
        v[c2] = acc[c2][i1][i0];
      eo_s<K>(P.Se, P.So, v, y);
#pragma unroll
      for (int i2 = 0; i2 < NI; ++i2)
      {
        T *o = xp + i2 * m2 + i1 * m + i0;
        if constexpr (MODE == MODE_BOUNDARY)
          *o = y[i2];
        else
          *o = __ldg(o) + y[i2];
      }
    }
}

template <int K, typename T, int MODE>
void launch_vp_patch3d(const PatchMatsEO<T, K> &P, const PatchST<T, K> &D, const ColorArgs<T> &a,
                       cudaStream_t s)
{
  if (a.total == 0)
    return;
  const dim3 block(32, 4, 1);
  const dim3 grid((a.np[0] + 31) / 32, (a.np[1] + 3) / 4, a.np[2]);
  pdl_launch(vp_patch3d_kernel<K, T, MODE>, grid, block, 0, s, P, a, D);
  check_launch("vp_patch3d_kernel");
}

}  // namespace pmgb
