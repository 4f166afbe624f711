// Ping-pong line-per-thread vertex-patch smoother kernel (3D, k >= 3) for
// sm_100a.
//
// Same arithmetic as vp_smooth_kernel (smoother_impl.cuh): the reference's
// fused / boundary per-patch body (smoother.cpp:109-148) as seven 1D
// contraction stages A..G, each thread holding one 1D line in registers,
// with the even-odd contractions and parameter-bank matrices of that kernel.
//
// What changes is shared memory: instead of overwriting one work array in
// place (whose single stride set cannot be bank-conflict-free for all seven
// access patterns; ncu measured 1.8-2x excess wavefronts), every stage writes
// its output tensor into the OTHER of two buffers in a layout of its own
// (strides, array separation, per-patch stride and the lane order of each
// stage), chosen by tools/bank_search_pp.py so that the stage's writes and
// the next stage's reads are both conflict-free under the measured model.
//
//   A: U (closure)  -> T_A = zM|zA [i0][j1][j2]          (Z1)
//   B: T_A          -> T_B = wMM|wS [i0][i1][j2]         (Z2)
//   C: T_B, b       -> T_C = S^T r [i0][i1][c2]          (Z1)
//   D: T_C          -> T_D [i0][c1][c2]                  (Z2)
//   E: T_D          -> T_E [i0][c1][c2] (S^T, 1/lambda, S along dir 0) (Z1)
//   F: T_E          -> T_F [i0][i1][c2]                  (Z2)
//   G: T_F, x_old   -> x^I (global)
#pragma once

#include "smoother_impl.cuh"
#include "smoother_pp_table.hpp"

namespace pmgb
{

template <int K, typename T>
struct PPCfg
{
  static constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  static constexpr int PB = sm_pb<3, K, T>();
  static constexpr int NT = sm_nt<3, K, T>();
  using L = PPLayout<K, sizeof(T)>;
  static constexpr int UW = NC * NC * NC;
  static constexpr int BW = NI * NI * NI + 1;
  static constexpr int max3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
  static constexpr int Z1W = max3(L::t(0, 4), L::t(2, 4), L::t(4, 4));  // T_A, T_C, T_E
  static constexpr int Z2W = max3(L::t(1, 4), L::t(3, 4), L::t(5, 4));  // T_B, T_D, T_F
  static constexpr size_t SMEM = sizeof(T) * static_cast<size_t>(PB) * (UW + BW + Z1W + Z2W);
};

// element (u0, u1, u2) of array `arr` of tensor X of patch p
template <int K, typename T, int X>
__device__ __forceinline__ int pp_at(int p, int arr, int u0, int u1, int u2)
{
  using L = PPLayout<K, sizeof(T)>;
  return p * L::t(X, 4) + arr * L::t(X, 3) + u0 * L::t(X, 0) + u1 * L::t(X, 1) + u2 * L::t(X, 2);
}

// stage S's thread -> (p, a, b) with line extents (na, nb) and its lane order
template <int K, typename T, int S, int NA, int NB>
__device__ __forceinline__ bool pp_line(int tid, int &p, int &a, int &b)
{
  using L = PPLayout<K, sizeof(T)>;
  constexpr int PB = PPCfg<K, T>::PB;
  if (tid >= PB * NA * NB)
    return false;
  p = tid / (NA * NB);
  const int rr = tid - p * (NA * NB);
  if constexpr (L::f(S))
  {
    a = rr / NB;
    b = rr - a * NB;
  }
  else
  {
    b = rr / NA;
    a = rr - b * NA;
  }
  return true;
}

// the same map with the lane order given explicitly
template <int K, typename T, int NA, int NB, bool FLIP>
__device__ __forceinline__ bool pp_line_f(int tid, int &p, int &a, int &b)
{
  constexpr int PB = PPCfg<K, T>::PB;
  if (tid >= PB * NA * NB)
    return false;
  p = tid / (NA * NB);
  const int rr = tid - p * (NA * NB);
  if constexpr (FLIP)
  {
    a = rr / NB;
    b = rr - a * NB;
  }
  else
  {
    b = rr / NA;
    a = rr - b * NA;
  }
  return true;
}

#ifndef PMG_PP_MAPS
#define PMG_PP_MAPS 1
#endif

template <int K, typename T, int MODE>
__global__ void __launch_bounds__(sm_nt<3, K, T>(), sm_minb<3, K, T>())
    vp_smooth_pp_kernel(const __grid_constant__ PatchMatsEO<T, K> P, const __grid_constant__ ColorArgs<T> a)
{
  // (the plane kernel reads b before the programmatic-dependency wait for
  // the later colours of a step; this kernel stages b with cp.async, which
  // goes through L1, so it waits first: a pre-wait read could hit an L1 line
  // older than the wait's visibility guarantee)
  pdl_prologue();
  using C = PPCfg<K, T>;
  constexpr int NC = C::NC, NI = C::NI, PB = C::PB, UW = C::UW, BW = C::BW;
  constexpr int A_ = 0, B_ = 1, C_ = 2, D_ = 3, E_ = 4, F_ = 5, G_ = 6;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *U = reinterpret_cast<T *>(smem_raw);  // [PB][UW]
  T *Bs = U + PB * UW;                     // [PB][BW]
  T *Z1 = Bs + PB * BW;                    // T_A, T_C, T_E
  T *Z2 = Z1 + PB * C::Z1W;                // T_B, T_D, T_F
  __shared__ int org[PB][3];

  const int tid = threadIdx.x;
  const int64_t m = a.m;
  const int64_t m2 = m * m;
  // closure staging with addresses advanced per plane and the z range as two
  // int compares: fewer integer instructions where the kernel is issue-bound
  // (f32 k = 4: 17.5 -> 20.7 GDoF/s, f64 k = 3: 14.4 -> 15.3); f64 k = 4 is
  // 2% faster with the per-element form (register pressure), kept there
  constexpr bool PP_INCR_STAGING = sizeof(T) == 4 || K == 3;
  const int bt = blockIdx.x;
  if (tid < PB)
  {
    const int gp = bt * PB + tid;
    int g0 = -(1 << 30), g1 = -(1 << 30), g2 = -(1 << 30);  // invalid patch: all loads masked
    if (gp < a.total)
    {
      const int j0 = gp % a.np[0];
      const int rest = gp / a.np[0];
      const int j1 = rest % a.np[1];
      const int j2 = rest / a.np[1];
      g0 = K * (2 * j0 + a.vb[0] - 1) - 1;
      g1 = K * (2 * j1 + a.vb[1] - 1) - 1;
      g2 = K * (2 * j2 + a.vb[2] - 1) - 1;
    }
    org[tid][0] = g0;
    org[tid][1] = g1;
    org[tid][2] = g2;
  }
  __syncthreads();

  // ---- b^I, then the closure (z-lines, zero fill, patches.cpp:72-79) --------
  if (tid < PB * NI * NI)
  {
    const int p = tid / (NI * NI);
    const int rr = tid - p * (NI * NI);
    const int i0 = rr % NI, i1 = rr / NI;
    const bool ok = org[p][0] > -(1 << 29);
    if constexpr (PP_INCR_STAGING)
    {
      const T *src = ok ? a.b + (static_cast<int64_t>(org[p][2]) + 1 - a.zoff) * m2 +
                              static_cast<int64_t>(org[p][1] + 1 + i1) * m + (org[p][0] + 1 + i0)
                        : a.x;
      const unsigned sdst = smem_addr(Bs + p * BW + rr);
#pragma unroll
      for (int t = 0; t < NI; ++t)
      {
        cp_async_sa<T>(sdst + static_cast<unsigned>(sizeof(T) * NI * NI * t), src, ok);
        src += m2;
      }
    }
    else
    {
      const T *src = a.b + (static_cast<int64_t>(org[p][2]) + 1 - a.zoff) * m2 +
                     static_cast<int64_t>(org[p][1] + 1 + i1) * m + (org[p][0] + 1 + i0);
      T *dst = Bs + p * BW + rr;
#pragma unroll
      for (int t = 0; t < NI; ++t)
        cp_async_elem(dst + NI * NI * t, ok ? src + t * m2 : a.x, ok);
    }
  }
  if (tid < PB * NC * NC)
  {
    const int p = tid / (NC * NC);
    const int rr = tid - p * (NC * NC);
    const int t0 = rr % NC, t1 = rr / NC;
    const int y0 = org[p][0] + t0, y1 = org[p][1] + t1;
    const bool inplane = static_cast<uint32_t>(y0) < static_cast<uint32_t>(m) &&
                         static_cast<uint32_t>(y1) < static_cast<uint32_t>(m);
    if constexpr (PP_INCR_STAGING)
    {
      // global planes z0 + t in [0, mz); addresses advance by one plane per t
      const int z0 = org[p][2];
      const int tlo = -z0, thi = a.mz - z0 < NC ? static_cast<int>(a.mz - z0) : NC;
      const T *src = inplane ? a.x + (static_cast<int64_t>(z0) - a.zoff) * m2 + static_cast<int64_t>(y1) * m + y0 : a.x;
      const unsigned sdst = smem_addr(U + p * UW + rr);
#pragma unroll
      for (int t = 0; t < NC; ++t)
      {
        bool ok = inplane && t >= tlo && t < thi;
        if constexpr (MODE == MODE_BOUNDARY)  // never reads x^I (smoother.cpp:128-148)
          ok = ok && !(t0 >= 1 && t0 <= NC - 2 && t1 >= 1 && t1 <= NC - 2 && t >= 1 && t <= NC - 2);
        cp_async_sa<T>(sdst + static_cast<unsigned>(sizeof(T) * NC * NC * t), src, ok);
        src += m2;
      }
    }
    else
    {
      const T *src = a.x + static_cast<int64_t>(y1) * m + y0;
      T *dst = U + p * UW + rr;
#pragma unroll
      for (int t = 0; t < NC; ++t)
      {
        const int64_t zg = static_cast<int64_t>(org[p][2]) + t;  // global plane
        bool ok = inplane && static_cast<uint64_t>(zg) < static_cast<uint64_t>(a.mz);
        if constexpr (MODE == MODE_BOUNDARY)  // never reads x^I (smoother.cpp:128-148)
          ok = ok && !(t0 >= 1 && t0 <= NC - 2 && t1 >= 1 && t1 <= NC - 2 && t >= 1 && t <= NC - 2);
        cp_async_elem(dst + NC * NC * t, ok ? src + (zg - a.zoff) * m2 : a.x, ok);
      }
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  int p, la, lb;
#if PMG_PP_MAPS
  // the stages' thread -> (patch, line) maps, computed once (the compiler does
  // not carry them across the barriers: ~9% of the f32 k = 3 instructions were
  // these divisions, recomputed per stage); stages C..G share one map per lane
  // order
  struct LineMap
  {
    int p, a, b;
    bool on;
  };
  LineMap mA, mB, mC0, mC1;
  mA.on = pp_line<K, T, A_, NC, NC>(tid, mA.p, mA.a, mA.b);
  mB.on = pp_line<K, T, B_, NI, NC>(tid, mB.p, mB.a, mB.b);
  mC0.on = pp_line_f<K, T, NI, NI, false>(tid, mC0.p, mC0.a, mC0.b);
  mC1.on = pp_line_f<K, T, NI, NI, true>(tid, mC1.p, mC1.a, mC1.b);
  using PL = PPLayout<K, sizeof(T)>;
  auto use = [&](const LineMap &mm) {
    p = mm.p;
    la = mm.a;
    lb = mm.b;
    return mm.on;
  };
#define PP_LINE(S, NA, NB)                                                                                 \
  ((S) == A_ ? use(mA) : (S) == B_ ? use(mB) : (PL::f(S) ? use(mC1) : use(mC0)))
#else
#define PP_LINE(S, NA, NB) pp_line<K, T, S, NA, NB>(tid, p, la, lb)
#endif
  // ---- A: U along t0 -> zM = M0 u, zA = A0 u  (lines (j1, j2)) -----------------
  if (PP_LINE(A_, NC, NC))
  {
    const T *u_ = U + p * UW + NC * la + NC * NC * lb;
    T u[NC], ue[K + 1], uo[K], zm[NI], za[NI];
#pragma unroll
    for (int t = 0; t < NC; ++t)
      u[t] = u_[t];
    eo_split<NC>(u, ue, uo);
    eo_rows<K>(P.Me, P.Mo, ue, uo, zm);
    eo_rows<K>(P.Ae, P.Ao, ue, uo, za);
#pragma unroll
    for (int i = 0; i < NI; ++i)
    {
      Z1[pp_at<K, T, A_>(p, 0, i, la, lb)] = zm[i];
      Z1[pp_at<K, T, A_>(p, 1, i, la, lb)] = za[i];
    }
  }
  __syncthreads();
  // ---- B: along j1: wMM = M1 zM, wS = A1 zM + M1 zA  (lines (i0, j2)) ------------
  if (PP_LINE(B_, NI, NC))
  {
    T zm[NC], za[NC];
#pragma unroll
    for (int t = 0; t < NC; ++t)
    {
      zm[t] = Z1[pp_at<K, T, A_>(p, 0, la, t, lb)];
      za[t] = Z1[pp_at<K, T, A_>(p, 1, la, t, lb)];
    }
    T zme[K + 1], zmo[K], zae[K + 1], zao[K], wm[NI], ws[NI];
    eo_split<NC>(zm, zme, zmo);
    eo_split<NC>(za, zae, zao);
    eo_rows<K>(P.Me, P.Mo, zme, zmo, wm);
    eo_rows2<K>(P.Ae, P.Ao, zme, zmo, P.Me, P.Mo, zae, zao, ws);
#pragma unroll
    for (int i = 0; i < NI; ++i)
    {
      Z2[pp_at<K, T, B_>(p, 0, la, i, lb)] = wm[i];
      Z2[pp_at<K, T, B_>(p, 1, la, i, lb)] = ws[i];
    }
  }
  __syncthreads();
  // ---- C: along j2: r = b - (A2 wMM + M2 wS); S^T r  (lines (i0, i1)) -----------
  if (PP_LINE(C_, NI, NI))
  {
    T wm[NC], ws[NC];
#pragma unroll
    for (int t = 0; t < NC; ++t)
    {
      wm[t] = Z2[pp_at<K, T, B_>(p, 0, la, lb, t)];
      ws[t] = Z2[pp_at<K, T, B_>(p, 1, la, lb, t)];
    }
    T wme[K + 1], wmo[K], wse[K + 1], wso[K], acc[NI], r[NI], y[NI];
    eo_split<NC>(wm, wme, wmo);
    eo_split<NC>(ws, wse, wso);
    eo_rows2<K>(P.Ae, P.Ao, wme, wmo, P.Me, P.Mo, wse, wso, acc);
    const T *bl = Bs + p * BW + la + NI * lb;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      r[i] = bl[NI * NI * i] - acc[i];
    eo_st<K>(P.Se, P.So, r, y);
#pragma unroll
    for (int c = 0; c < NI; ++c)
      Z1[pp_at<K, T, C_>(p, 0, la, lb, c)] = y[c];
  }
  __syncthreads();
  // ---- D: along i1: S^T  (lines (i0, c2)) -----------------------------------------
  if (PP_LINE(D_, NI, NI))
  {
    T v[NI], y[NI];
#pragma unroll
    for (int t = 0; t < NI; ++t)
      v[t] = Z1[pp_at<K, T, C_>(p, 0, la, t, lb)];
    eo_st<K>(P.Se, P.So, v, y);
#pragma unroll
    for (int t = 0; t < NI; ++t)
      Z2[pp_at<K, T, D_>(p, 0, la, t, lb)] = y[t];
  }
  __syncthreads();
  // ---- E: along i0: S^T, x 1/(lambda sums), S  (lines (c1, c2)) -------------------
  if (PP_LINE(E_, NI, NI))
  {
    T v[NI], y[NI];
#pragma unroll
    for (int t = 0; t < NI; ++t)
      v[t] = Z2[pp_at<K, T, D_>(p, 0, t, la, lb)];
    eo_st<K>(P.Se, P.So, v, y);
    const T *inv = a.inv + NI * (la + NI * lb);
#pragma unroll
    for (int t = 0; t < NI; ++t)
      y[t] *= __ldg(inv + t);
    eo_s<K>(P.Se, P.So, y, v);
#pragma unroll
    for (int t = 0; t < NI; ++t)
      Z1[pp_at<K, T, E_>(p, 0, t, la, lb)] = v[t];
  }
  __syncthreads();
  // ---- F: along c1: S  (lines (i0, c2)) -------------------------------------------
  if (PP_LINE(F_, NI, NI))
  {
    T v[NI], y[NI];
#pragma unroll
    for (int t = 0; t < NI; ++t)
      v[t] = Z1[pp_at<K, T, E_>(p, 0, la, t, lb)];
    eo_s<K>(P.Se, P.So, v, y);
#pragma unroll
    for (int t = 0; t < NI; ++t)
      Z2[pp_at<K, T, F_>(p, 0, la, t, lb)] = y[t];
  }
  __syncthreads();
  // ---- G: along c2: S, x^I update  (lines (i0, i1)) -------------------------------
  if (PP_LINE(G_, NI, NI) && bt * PB + p < a.total)
  {
    T v[NI], y[NI];
#pragma unroll
    for (int t = 0; t < NI; ++t)
      v[t] = Z2[pp_at<K, T, F_>(p, 0, la, lb, t)];
    eo_s<K>(P.Se, P.So, v, y);
    T *xp = a.x + (static_cast<int64_t>(org[p][2]) + 1 - a.zoff) * m2 +
            static_cast<int64_t>(org[p][1] + 1 + lb) * m + (org[p][0] + 1 + la);
    const T *xo = U + p * UW + (1 + la) + NC * (1 + lb) + NC * NC;
#pragma unroll
    for (int i = 0; i < NI; ++i)
    {
      if constexpr (MODE == MODE_BOUNDARY)
        xp[i * m2] = y[i];
      else
        xp[i * m2] = xo[NC * NC * i] + y[i];  // x^I_old is in the staged closure
    }
  }
}

#undef PP_LINE

template <int K, typename T, int MODE>
void launch_vp_smooth_pp(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a, cudaStream_t s)
{
  using C = PPCfg<K, T>;
  static unsigned attr_mask = 0;
  if (first_on_device(attr_mask))
  {
    check_cuda(cudaFuncSetAttribute(vp_smooth_pp_kernel<K, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(C::SMEM)),
               "cudaFuncSetAttribute(pp smoother)");
    check_cuda(cudaFuncSetAttribute(vp_smooth_pp_kernel<K, T, MODE>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100),
               "cudaFuncSetAttribute(pp smoother carveout)");
  }
  const int nbatch = (a.total + C::PB - 1) / C::PB;
  if (nbatch == 0)
    return;
  pdl_launch(vp_smooth_pp_kernel<K, T, MODE>, dim3(nbatch), dim3(C::NT), C::SMEM, s, P, a);
  check_launch("vp_smooth_pp_kernel");
}

}  // namespace pmgb
