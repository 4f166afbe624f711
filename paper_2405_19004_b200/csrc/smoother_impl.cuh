// Fused per-colour vertex-patch smoother kernel for sm_100a.
//
// Replaces the per-patch body of the reference's smooth<T>
// (/root/reference/proj/src/smoother.cpp:109-126 fused, :128-148 boundary,
// :82-108 separate, :63-81 global) and its callees gather/scatter_interior
// (patches.cpp:51-121), apply_patch_operator (fastdiag.cpp:199-233) and
// apply_patch_inverse (fastdiag.cpp:164-192).
//
// Design:
//  * one launch per colour, persistent CTAs: a CTA loops over batches of PB
//    patches of the colour; the closure (2k+1)^d of x and the interior
//    (2k-1)^d of b of the NEXT batch are fetched with cp.async (coalesced,
//    zero-filled outside the domain = the Dirichlet elimination of
//    patches.cpp:72-79) while the current batch computes;
//  * every sum-factorisation contraction is done by a thread that holds one
//    full 1D line in registers and writes the whole output line. One line
//    per thread per stage: no stage loops, so the compiler never hoists the
//    parameter-bank matrices into general registers. The 1D matrices are
//    compile-time-indexed __grid_constant__ kernel parameters, so the inner
//    loops are DFMA/FFMA with uniform-register operands;
//  * even-odd factorisation: the patch mass/stiffness rows are
//    centro-symmetric and the eigenvectors have parity (columns reordered
//    even-first on the host), so every 1D contraction runs on half-length
//    even/odd vectors (~1/3 fewer multiply-adds than the dense form);
//  * shared memory only transposes lines between directions; the work
//    buffer is reused IN PLACE (each thread reads its whole input line before
//    writing its output line into a subset of the same positions, which no
//    other thread touches in that stage);
//  * the 3D residual uses 7 contractions instead of the reference's 8 by
//    summing the two mass-in-direction-2 terms before the last contraction.
#pragma once

#include "common.cuh"

namespace pmgb
{

// ---------------------------------------------------------------------------
// launch geometry
// ---------------------------------------------------------------------------

// patches per CTA; NT covers the widest stage with one line per thread
template <int D, int K, typename T>
constexpr int sm_pb()
{
  if constexpr (D == 3)
  {
    constexpr int t[8] = {0, 16, 8, 4, 2, 2, 1, 1};
    return t[K];
  }
  else
  {
    return 256 / (2 * K + 1);
  }
}

// minimum resident CTAs per SM requested from the register allocator
template <int D, int K, typename T>
constexpr int sm_minb()
{
  return (D == 3 && K >= 5) ? 2 : 1;
}

template <int D, int K, typename T>
constexpr int sm_nt()
{
  constexpr int NC = 2 * K + 1;
  constexpr int lines = sm_pb<D, K, T>() * (D == 3 ? NC * NC : NC);
  return ((lines + 31) / 32) * 32;
}

constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// shared memory per patch, in words: closure U | b interior Bs | work Z
template <int D, int K>
constexpr int sm_u_words()
{
  return ipow(2 * K + 1, D);
}
template <int D, int K>
constexpr int sm_b_words()
{
  return ipow(2 * K - 1, D) + 1;  // +1: odd patch stride
}
// Work-buffer layout of one patch: two arrays (zM | zA, later wMM | wS and
// the residual / eigen-space tensor) with strides (1, S1, S2) over
// [i0][j1][j2] (3D) or (1, S1) over [i0][j1] (2D), followed by ZPAD words.
// S1 >= 2k-1, S2 >= (2k+1) S1; the paddings were chosen by an offline search
// over the stage access patterns (bank-conflict model: 8-byte words hit bank
// pair w mod 16, 4-byte words bank w mod 32) with a small memory penalty.
template <int D, int K, typename T>
struct ZLayout
{
  static constexpr bool F64 = sizeof(T) == 8;
  static constexpr int t3d64[8][3] = {{0, 0, 0}, {1, 3, 7}, {3, 15, 3}, {5, 38, 5}, {7, 70, 5},
                                      {9, 105, 11}, {11, 155, 0}, {13, 205, 0}};
  static constexpr int t3d32[8][3] = {{0, 0, 0}, {1, 3, 3}, {3, 15, 0}, {5, 35, 15}, {7, 72, 1},
                                      {9, 113, 3}, {11, 143, 0}, {13, 201, 0}};
  static constexpr int t2d64[8][2] = {{0, 0}, {1, 1}, {3, 1}, {6, 1}, {10, 3}, {11, 7}, {11, 11}, {13, 7}};
  static constexpr int t2d32[8][2] = {{0, 0}, {1, 1}, {3, 0}, {6, 17}, {9, 5}, {10, 13}, {12, 19}, {14, 9}};
  static constexpr int S1 = D == 3 ? (F64 ? t3d64[K][0] : t3d32[K][0]) : (F64 ? t2d64[K][0] : t2d32[K][0]);
  static constexpr int S2 = D == 3 ? (F64 ? t3d64[K][1] : t3d32[K][1]) : 0;
  static constexpr int ZPAD = D == 3 ? (F64 ? t3d64[K][2] : t3d32[K][2]) : (F64 ? t2d64[K][1] : t2d32[K][1]);
  static constexpr int ZS = D == 3 ? S2 * (2 * K + 1) : S1 * (2 * K + 1);  // one array
  static constexpr int ZW = 2 * ZS + ZPAD;                                     // per patch
  static_assert(S1 >= 2 * K - 1 && (D == 2 || S2 >= (2 * K + 1) * S1), "layout");
};

template <int D, int K, typename T>
constexpr int sm_z_words()
{
  return ZLayout<D, K, T>::ZW;
}

template <int D, int K, typename T>
constexpr size_t sm_smem_bytes()
{
  return static_cast<size_t>(sm_pb<D, K, T>()) *
         (sm_u_words<D, K>() + sm_b_words<D, K>() + sm_z_words<D, K, T>()) * sizeof(T);
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS); src_size 0 zero-fills the destination
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ void cp_async_elem(T *smem, const T *gmem, bool valid)
{
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 8 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
// same, destination given as a shared-window address (callers advance it by
// compile-time offsets instead of converting a generic pointer per element)
template <typename T>
__device__ __forceinline__ void cp_async_sa(unsigned s, const T *gmem, bool valid)
{
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 8 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ unsigned smem_addr(const void *p)
{
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Read one entry of a __grid_constant__ parameter matrix. The volatile load
// is issued at the point of use, so the compiler can neither hoist the
// parameter bank out of the persistent batch loop nor CSE it into general
// registers: every multiply-add takes its coefficient from a uniform register
// loaded right before it (LDCU), costing no per-thread registers.
__device__ __forceinline__ double pc(const double &r)
{
  double v;
  asm volatile("{ .reg .u64 pa; cvta.to.param.u64 pa, %1; ld.param.f64 %0, [pa]; }" : "=d"(v) : "l"(&r));
  return v;
}
__device__ __forceinline__ float pc(const float &r)
{
  float v;
  asm volatile("{ .reg .u64 pa; cvta.to.param.u64 pa, %1; ld.param.f32 %0, [pa]; }" : "=f"(v) : "l"(&r));
  return v;
}

// ---------------------------------------------------------------------------
// even-odd 1D contractions (matrices from PatchMatsEO, see common.cuh)
// ---------------------------------------------------------------------------

// split a length-N (odd) line into even / odd halves and its middle entry
template <int N, typename T>
__device__ __forceinline__ void eo_split(const T (&x)[N], T (&xe)[N / 2 + 1], T (&xo)[N / 2 > 0 ? N / 2 : 1])
{
  constexpr int H = N / 2;
#pragma unroll
  for (int j = 0; j < H; ++j)
  {
    xe[j] = x[j] + x[N - 1 - j];
    xo[j] = x[j] - x[N - 1 - j];
  }
  xe[H] = x[H];
}

// y (NI) = B x with B (NI x NC) centro-symmetric, given x split (xe: HC+1, xo: HC)
template <int K, typename T, typename BE, typename BO>
__device__ __forceinline__ void eo_rows(const BE &Be, const BO &Bo, const T (&xe)[K + 1], const T (&xo)[K],
                                        T (&y)[2 * K - 1])
{
  constexpr int HI = K - 1, HC = K;
#pragma unroll
  for (int i = 0; i <= HI; ++i)
  {
    T e = Be[i][HC] * xe[HC];
#pragma unroll
    for (int j = 0; j < HC; ++j)
      e = fma(Be[i][j], xe[j], e);
    if (i < HI)
    {
      T o = Bo[i][0] * xo[0];
#pragma unroll
      for (int j = 1; j < HC; ++j)
        o = fma(Bo[i][j], xo[j], o);
      y[i] = e + o;
      y[2 * K - 2 - i] = e - o;
    }
    else
    {
      y[i] = e;
    }
  }
}

// y = B1 x1 + B2 x2 (both centro-symmetric NI x NC), x1/x2 split
template <int K, typename T, typename BE, typename BO>
__device__ __forceinline__ void eo_rows2(const BE &B1e, const BO &B1o, const T (&x1e)[K + 1],
                                         const T (&x1o)[K], const BE &B2e, const BO &B2o,
                                         const T (&x2e)[K + 1], const T (&x2o)[K], T (&y)[2 * K - 1])
{
  constexpr int HI = K - 1, HC = K;
#pragma unroll
  for (int i = 0; i <= HI; ++i)
  {
    T e = B1e[i][HC] * x1e[HC];
    e = fma(B2e[i][HC], x2e[HC], e);
#pragma unroll
    for (int j = 0; j < HC; ++j)
    {
      e = fma(B1e[i][j], x1e[j], e);
      e = fma(B2e[i][j], x2e[j], e);
    }
    if (i < HI)
    {
      T o = B1o[i][0] * x1o[0];
      o = fma(B2o[i][0], x2o[0], o);
#pragma unroll
      for (int j = 1; j < HC; ++j)
      {
        o = fma(B1o[i][j], x1o[j], o);
        o = fma(B2o[i][j], x2o[j], o);
      }
      y[i] = e + o;
      y[2 * K - 2 - i] = e - o;
    }
    else
    {
      y[i] = e;
    }
  }
}

// yhat = S^T r (eigen index: K even modes first, then K-1 odd modes)
template <int K, typename T, typename SE, typename SO>
__device__ __forceinline__ void eo_st(const SE &Se, const SO &So, const T (&r)[2 * K - 1], T (&yh)[2 * K - 1])
{
  constexpr int NI = 2 * K - 1, HI = K - 1;
  T re[K], ro[K > 1 ? K - 1 : 1];
#pragma unroll
  for (int i = 0; i < HI; ++i)
  {
    re[i] = r[i] + r[NI - 1 - i];
    ro[i] = r[i] - r[NI - 1 - i];
  }
  re[HI] = r[HI];
#pragma unroll
  for (int c = 0; c <= HI; ++c)
  {
    T s = Se[HI][c] * re[HI];
#pragma unroll
    for (int i = 0; i < HI; ++i)
      s = fma(Se[i][c], re[i], s);
    yh[c] = s;
  }
#pragma unroll
  for (int c = 0; c < HI; ++c)
  {
    T s = So[0][c] * ro[0];
#pragma unroll
    for (int i = 1; i < HI; ++i)
      s = fma(So[i][c], ro[i], s);
    yh[HI + 1 + c] = s;
  }
}

// x = S yhat (back to physical index)
template <int K, typename T, typename SE, typename SO>
__device__ __forceinline__ void eo_s(const SE &Se, const SO &So, const T (&yh)[2 * K - 1], T (&x)[2 * K - 1])
{
  constexpr int NI = 2 * K - 1, HI = K - 1;
#pragma unroll
  for (int i = 0; i <= HI; ++i)
  {
    T e = Se[i][0] * yh[0];
#pragma unroll
    for (int c = 1; c <= HI; ++c)
      e = fma(Se[i][c], yh[c], e);
    if (i < HI)
    {
      T o = So[i][0] * yh[HI + 1];
#pragma unroll
      for (int c = 1; c < HI; ++c)
        o = fma(So[i][c], yh[HI + 1 + c], o);
      x[i] = e + o;
      x[NI - 1 - i] = e - o;
    }
    else
    {
      x[i] = e;
    }
  }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------

template <int D, int K, typename T, int MODE>
__global__ void __launch_bounds__(sm_nt<D, K, T>(), sm_minb<D, K, T>())
    vp_smooth_kernel(const __grid_constant__ PatchMatsEO<T, K> P, const __grid_constant__ ColorArgs<T> a)
{
  pdl_prologue();
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  constexpr int PB = sm_pb<D, K, T>();
  constexpr int NT = sm_nt<D, K, T>();
  constexpr int NCD = ipow(NC, D), NID = ipow(NI, D);
  constexpr int UW = sm_u_words<D, K>(), BW = sm_b_words<D, K>();
  using ZL = ZLayout<D, K, T>;
  constexpr int ZW = ZL::ZW, ZS = ZL::ZS, S1 = ZL::S1, S2 = ZL::S2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *U = reinterpret_cast<T *>(smem_raw);  // [PB][UW]
  T *Bs = U + PB * UW;                     // [PB][BW]
  T *Z = Bs + PB * BW;                     // [PB][ZW]

  const int tid = threadIdx.x;
  const int64_t m = a.m;
  const int nbatch = (a.total + PB - 1) / PB;

  // Per-batch patch origins (dof index of closure-local t = 0 per direction,
  // patches.cpp:71: g_a = k (v_a - 1) - 1 + t_a), double-buffered: slot it&1
  // holds the batch being computed, slot (it+1)&1 the one being prefetched.
  __shared__ int org[2][PB][3];
  auto set_origin = [&](int slot, int bt_) {
    if (tid < PB)
    {
      const int gp = bt_ * PB + tid;
      int g0 = -(1 << 30), g1 = -(1 << 30), g2 = -(1 << 30);  // invalid patch: all loads masked
      if (gp < a.total)
      {
        const int j0 = gp % a.np[0];
        const int rest = gp / a.np[0];
        const int j1 = rest % a.np[1];
        const int j2 = rest / a.np[1];
        g0 = K * (2 * j0 + a.vb[0] - 1) - 1;
        g1 = K * (2 * j1 + a.vb[1] - 1) - 1;
        g2 = (D == 3) ? K * (2 * j2 + a.vb[2] - 1) - 1 : 0;
      }
      org[slot][tid][0] = g0;
      org[slot][tid][1] = g1;
      org[slot][tid][2] = g2;
    }
  };

  // Cooperative cp.async loads, one z-line (3D; y-line in 2D) per thread:
  // thread -> (patch, t0, t1) once, then a fixed-stride walk along the last
  // direction, so the per-element cost is an address increment plus one
  // bounds test. Lanes run along x: row segments are contiguous in HBM.
  auto load_closure = [&](int slot) {
    constexpr int LINES = PB * (D == 3 ? NC * NC : NC);
    if (tid >= LINES)
      return;
    const int p = tid / (D == 3 ? NC * NC : NC);
    const int rr = tid - p * (D == 3 ? NC * NC : NC);
    const int t0 = rr % NC, t1 = (D == 3) ? rr / NC : 0;
    const int y0 = org[slot][p][0] + t0;
    const int y1 = org[slot][p][1] + ((D == 3) ? t1 : 0);
    const int ylast0 = org[slot][p][D == 3 ? 2 : 1];
    const bool inplane = static_cast<uint32_t>(y0) < static_cast<uint32_t>(m) &&
                         (D == 2 || static_cast<uint32_t>(y1) < static_cast<uint32_t>(m));
    const int64_t step = (D == 3) ? m * m : m;
    const int64_t base = (D == 3) ? static_cast<int64_t>(y1) * m + y0 : static_cast<int64_t>(y0);
    const int64_t zl = (D == 3) ? a.zoff : 0;
    const int64_t mlast = (D == 3) ? a.mz : m;
    if constexpr (sizeof(T) == 4)
    {
      // f32 (issue-bound): addresses advanced per line, range as two int compares
      const int tlo = -ylast0, thi = mlast - ylast0 < NC ? static_cast<int>(mlast - ylast0) : NC;
      const T *src = inplane ? a.x + base + (ylast0 - zl) * step : a.x;
      const unsigned sdst = smem_addr(U + p * UW + rr);
#pragma unroll
      for (int t = 0; t < NC; ++t)
      {
        bool ok = inplane && t >= tlo && t < thi;
        if constexpr (MODE == MODE_BOUNDARY)
          ok = ok && !(t0 >= 1 && t0 <= NC - 2 && t >= 1 && t <= NC - 2 && (D == 2 || (t1 >= 1 && t1 <= NC - 2)));
        cp_async_sa<T>(sdst + static_cast<unsigned>(sizeof(T) * (D == 3 ? NC * NC : NC) * t), src, ok);
        src += step;
      }
      return;
    }
    T *dst = U + p * UW + rr;
#pragma unroll
    for (int t = 0; t < NC; ++t)
    {
      const int yl = ylast0 + t;
      bool ok = inplane && static_cast<uint64_t>(static_cast<int64_t>(yl)) < static_cast<uint64_t>(mlast);
      if constexpr (MODE == MODE_BOUNDARY)
      {
        // boundary variant never reads x^I (smoother.cpp:128-148)
        const bool inner = t0 >= 1 && t0 <= NC - 2 && t >= 1 && t <= NC - 2 &&
                           (D == 2 || (t1 >= 1 && t1 <= NC - 2));
        ok = ok && !inner;
      }
      cp_async_elem(dst + (D == 3 ? NC * NC : NC) * t, ok ? a.x + base + (yl - zl) * step : a.x, ok);
    }
  };
  // prefetch the interior of b (or of the residual for MODE_SOLVE)
  auto load_interior = [&](int slot) {
    constexpr int LINES = PB * (D == 3 ? NI * NI : NI);
    if (tid >= LINES)
      return;
    const T *vec = (MODE == MODE_SOLVE) ? a.r : a.b;
    const int p = tid / (D == 3 ? NI * NI : NI);
    const int rr = tid - p * (D == 3 ? NI * NI : NI);
    const int i0 = rr % NI, i1 = (D == 3) ? rr / NI : 0;
    const int g0 = org[slot][p][0];
    const bool ok = g0 > -(1 << 29);
    const int64_t step = (D == 3) ? m * m : m;
    const int64_t base = (D == 3) ? static_cast<int64_t>(org[slot][p][1] + 1 + i1) * m + (g0 + 1 + i0)
                                  : static_cast<int64_t>(g0 + 1 + i0);
    const int64_t z0 = static_cast<int64_t>(org[slot][p][D == 3 ? 2 : 1]) + 1 - ((D == 3) ? a.zoff : 0);
    T *dst = Bs + p * BW + rr;
#pragma unroll
    for (int t = 0; t < NI; ++t)
      cp_async_elem(dst + (D == 3 ? NI * NI : NI) * t, ok ? vec + base + (z0 + t) * step : a.x, ok);
  };
  auto origin = [&](int slot, int p, int64_t &g0, int64_t &g1, int64_t &g2) {
    g0 = org[slot][p][0];
    g1 = org[slot][p][1];
    g2 = org[slot][p][2];
  };

  // one batch of PB patches per CTA. (A persistent CTA looping over batches
  // with a cp.async prefetch of the next batch was measured slower: the loop
  // lets the compiler hoist the parameter-bank matrices into registers.)
  const int bt = blockIdx.x;
  if (bt >= nbatch)
    return;
  constexpr int cur = 0;
  const int nxt = nbatch;  // no next batch to prefetch
  set_origin(0, bt);
  __syncthreads();
  if constexpr (MODE != MODE_SOLVE)
    load_closure(0);
  load_interior(0);
  cp_async_commit();
  {
    cp_async_wait_all();
    __syncthreads();

    if constexpr (D == 3)
    {
      const int64_t m2 = m * m;
      if constexpr (MODE != MODE_SOLVE)
      {
        // ---- A: direction 0: zM = M0 u, zA = A0 u -----------------------------
        static_assert(PB * NC * NC <= NT, "one line per thread per stage");
        if (tid < PB * NC * NC)
        {
          const int p = tid / (NC * NC);
          const int rr = tid - p * (NC * NC);  // = j1 + NC j2
          const T *u_ = U + p * UW + NC * rr;
          T u[NC];
#pragma unroll
          for (int t = 0; t < NC; ++t)
            u[t] = u_[t];
          T ue[K + 1], uo[K];
          eo_split<NC>(u, ue, uo);
          T zm[NI], za[NI];
          eo_rows<K>(P.Me, P.Mo, ue, uo, zm);
          eo_rows<K>(P.Ae, P.Ao, ue, uo, za);
          T *z = Z + p * ZW + S1 * (rr % NC) + S2 * (rr / NC);  // rr = j1 + NC j2
#pragma unroll
          for (int i = 0; i < NI; ++i)
          {
            z[i] = zm[i];
            z[ZS + i] = za[i];
          }
        }
        __syncthreads();
        if (nxt < nbatch)
        {
          load_closure(cur ^ 1);  // U is free: overlap the next closure with B..G
          cp_async_commit();
        }

        // ---- B: direction 1: wMM = M1 zM, wS = A1 zM + M1 zA (in place) ------
        if (tid < PB * NI * NC)
        {
          const int p = tid / (NI * NC);
          const int rr = tid - p * (NI * NC);
          const int i0 = rr % NI, j2 = rr / NI;
          T *z = Z + p * ZW + i0 + S2 * j2;
          T zm[NC], za[NC];
#pragma unroll
          for (int t = 0; t < NC; ++t)
          {
            zm[t] = z[S1 * t];
            za[t] = z[ZS + S1 * t];
          }
          T zme[K + 1], zmo[K], zae[K + 1], zao[K];
          eo_split<NC>(zm, zme, zmo);
          eo_split<NC>(za, zae, zao);
          T wm[NI], ws[NI];
          eo_rows<K>(P.Me, P.Mo, zme, zmo, wm);
          eo_rows2<K>(P.Ae, P.Ao, zme, zmo, P.Me, P.Mo, zae, zao, ws);
#pragma unroll
          for (int i = 0; i < NI; ++i)
          {
            z[S1 * i] = wm[i];
            z[ZS + S1 * i] = ws[i];
          }
        }
        __syncthreads();
      }

      // ---- C: direction 2: r = b - (A2 wMM + M2 wS); yhat = S^T r ------------
      if (tid < PB * NI * NI)
      {
        const int p = tid / (NI * NI);
        const int rr = tid - p * (NI * NI);  // = i0 + NI i1
        const int i0 = rr % NI, i1 = rr / NI;
        const int gp = bt * PB + p;
        if (gp < a.total)
        {
          T *z = Z + p * ZW + i0 + S1 * i1;
          const T *bl = Bs + p * BW + rr;
          T r[NI];
          if constexpr (MODE == MODE_SOLVE)
          {
#pragma unroll
            for (int i = 0; i < NI; ++i)
              r[i] = bl[NI * NI * i];
          }
          else
          {
            T wm[NC], ws[NC];
#pragma unroll
            for (int t = 0; t < NC; ++t)
            {
              wm[t] = z[S2 * t];
              ws[t] = z[ZS + S2 * t];
            }
            T wme[K + 1], wmo[K], wse[K + 1], wso[K];
            eo_split<NC>(wm, wme, wmo);
            eo_split<NC>(ws, wse, wso);
            T acc[NI];
            eo_rows2<K>(P.Ae, P.Ao, wme, wmo, P.Me, P.Mo, wse, wso, acc);
#pragma unroll
            for (int i = 0; i < NI; ++i)
              r[i] = bl[NI * NI * i] - acc[i];
            if constexpr (MODE == MODE_RESIDUAL)
            {
              int64_t g0, g1, g2;
              origin(cur, p, g0, g1, g2);
              T *rp = a.r + ((g2 + 1 - a.zoff) * m + (g1 + 1 + i1)) * m + (g0 + 1 + i0);
#pragma unroll
              for (int i = 0; i < NI; ++i)
                rp[i * m2] = r[i];
            }
          }
          if constexpr (MODE != MODE_RESIDUAL)
          {
            T y[NI];
            eo_st<K>(P.Se, P.So, r, y);
#pragma unroll
            for (int c = 0; c < NI; ++c)
              z[S2 * c] = y[c];
          }
        }
      }
      if constexpr (MODE == MODE_RESIDUAL)
      {
        __syncthreads();
        if (nxt < nbatch)
        {
          load_interior(cur ^ 1);
          cp_async_commit();
        }
        return;
      }
      __syncthreads();
      if (nxt < nbatch)
      {
        load_interior(cur ^ 1);  // Bs is free: overlap the next b with D..G
        cp_async_commit();
      }

      // ---- D: direction 1, S^T ---------------------------------------------------
      if (tid < PB * NI * NI)
      {
        const int p = tid / (NI * NI);
        const int rr = tid - p * (NI * NI);
        const int i0 = rr % NI, i2 = rr / NI;
        T *z = Z + p * ZW + i0 + S2 * i2;
        T v[NI], y[NI];
#pragma unroll
        for (int t = 0; t < NI; ++t)
          v[t] = z[S1 * t];
        eo_st<K>(P.Se, P.So, v, y);
#pragma unroll
        for (int t = 0; t < NI; ++t)
          z[S1 * t] = y[t];
      }
      __syncthreads();

      // ---- E: direction 0, S^T, scale by 1/(lambda sums), S -----------------------
      if (tid < PB * NI * NI)
      {
        const int p = tid / (NI * NI);
        const int rr = tid - p * (NI * NI);
        const int i1 = rr % NI, i2 = rr / NI;
        T *z = Z + p * ZW + S1 * i1 + S2 * i2;
        const T *inv = a.inv + NI * rr;
        T v[NI], y[NI];
#pragma unroll
        for (int t = 0; t < NI; ++t)
          v[t] = z[t];
        eo_st<K>(P.Se, P.So, v, y);
#pragma unroll
        for (int t = 0; t < NI; ++t)
          y[t] *= __ldg(inv + t);
        eo_s<K>(P.Se, P.So, y, v);
#pragma unroll
        for (int t = 0; t < NI; ++t)
          z[t] = v[t];
      }
      __syncthreads();

      // ---- F: direction 1, S -------------------------------------------------------
      if (tid < PB * NI * NI)
      {
        const int p = tid / (NI * NI);
        const int rr = tid - p * (NI * NI);
        const int i0 = rr % NI, i2 = rr / NI;
        T *z = Z + p * ZW + i0 + S2 * i2;
        T v[NI], y[NI];
#pragma unroll
        for (int t = 0; t < NI; ++t)
          v[t] = z[S1 * t];
        eo_s<K>(P.Se, P.So, v, y);
#pragma unroll
        for (int t = 0; t < NI; ++t)
          z[S1 * t] = y[t];
      }
      __syncthreads();

      // ---- G: direction 2, S, then x^I += v (or = v) -------------------------------
      if (tid < PB * NI * NI)
      {
        const int p = tid / (NI * NI);
        const int rr = tid - p * (NI * NI);
        const int i0 = rr % NI, i1 = rr / NI;
        const int gp = bt * PB + p;
        if (gp < a.total)
        {
          int64_t g0, g1, g2;
          origin(cur, p, g0, g1, g2);
          const T *z = Z + p * ZW + i0 + S1 * i1;
          T v[NI], y[NI];
#pragma unroll
          for (int t = 0; t < NI; ++t)
            v[t] = z[S2 * t];
          eo_s<K>(P.Se, P.So, v, y);
          T *xp = a.x + ((g2 + 1 - a.zoff) * m + (g1 + 1 + i1)) * m + (g0 + 1 + i0);
          // x^I old values are still in the staged closure (no other patch of
          // this colour writes them), so the update is a pure store
          const T *xo = U + p * UW + (1 + i0) + NC * (1 + i1) + NC * NC;
#pragma unroll
          for (int i = 0; i < NI; ++i)
          {
            if constexpr (MODE == MODE_BOUNDARY)
              xp[i * m2] = y[i];
            else if constexpr (MODE == MODE_FUSED)
              xp[i * m2] = xo[NC * NC * i] + y[i];
            else
              xp[i * m2] += y[i];
          }
        }
      }
    }
    else  // ------------------------------- 2D -----------------------------------------
    {
      if constexpr (MODE != MODE_SOLVE)
      {
        // A: direction 0 rows: zM = M0 u, zA = A0 u
        static_assert(PB * NC <= NT, "one line per thread per stage");
        if (tid < PB * NC)
        {
          const int p = tid / NC;
          const int j1 = tid - p * NC;
          const T *u_ = U + p * UW + NC * j1;
          T u[NC];
#pragma unroll
          for (int t = 0; t < NC; ++t)
            u[t] = u_[t];
          T ue[K + 1], uo[K];
          eo_split<NC>(u, ue, uo);
          T zm[NI], za[NI];
          eo_rows<K>(P.Me, P.Mo, ue, uo, zm);
          eo_rows<K>(P.Ae, P.Ao, ue, uo, za);
          T *z = Z + p * ZW + S1 * j1;
#pragma unroll
          for (int i = 0; i < NI; ++i)
          {
            z[i] = zm[i];
            z[ZS + i] = za[i];
          }
        }
        __syncthreads();
        if (nxt < nbatch)
        {
          load_closure(cur ^ 1);
          cp_async_commit();
        }
      }

      // B: direction 1: r = b - (A1 zM + M1 zA); yhat = S^T r
      if (tid < PB * NI)
      {
        const int p = tid / NI;
        const int i0 = tid - p * NI;
        const int gp = bt * PB + p;
        if (gp < a.total)
        {
          T *z = Z + p * ZW + i0;
          const T *bl = Bs + p * BW + i0;
          T r[NI];
          if constexpr (MODE == MODE_SOLVE)
          {
#pragma unroll
            for (int i = 0; i < NI; ++i)
              r[i] = bl[NI * i];
          }
          else
          {
            T zm[NC], za[NC];
#pragma unroll
            for (int t = 0; t < NC; ++t)
            {
              zm[t] = z[S1 * t];
              za[t] = z[ZS + S1 * t];
            }
            T zme[K + 1], zmo[K], zae[K + 1], zao[K];
            eo_split<NC>(zm, zme, zmo);
            eo_split<NC>(za, zae, zao);
            T acc[NI];
            eo_rows2<K>(P.Ae, P.Ao, zme, zmo, P.Me, P.Mo, zae, zao, acc);
#pragma unroll
            for (int i = 0; i < NI; ++i)
              r[i] = bl[NI * i] - acc[i];
            if constexpr (MODE == MODE_RESIDUAL)
            {
              int64_t g0, g1, g2;
              origin(cur, p, g0, g1, g2);
              T *rp = a.r + (g1 + 1) * m + (g0 + 1 + i0);
#pragma unroll
              for (int i = 0; i < NI; ++i)
                rp[i * m] = r[i];
            }
          }
          if constexpr (MODE != MODE_RESIDUAL)
          {
            T y[NI];
            eo_st<K>(P.Se, P.So, r, y);
#pragma unroll
            for (int c = 0; c < NI; ++c)
              z[S1 * c] = y[c];
          }
        }
      }
      __syncthreads();
      if (nxt < nbatch)
      {
        load_interior(cur ^ 1);
        cp_async_commit();
      }
      if constexpr (MODE == MODE_RESIDUAL)
        return;

      // C: direction 0: S^T, scale, S
      if (tid < PB * NI)
      {
        const int p = tid / NI;
        const int i1 = tid - p * NI;
        T *z = Z + p * ZW + S1 * i1;
        const T *inv = a.inv + NI * i1;
        T v[NI], y[NI];
#pragma unroll
        for (int t = 0; t < NI; ++t)
          v[t] = z[t];
        eo_st<K>(P.Se, P.So, v, y);
#pragma unroll
        for (int t = 0; t < NI; ++t)
          y[t] *= __ldg(inv + t);
        eo_s<K>(P.Se, P.So, y, v);
#pragma unroll
        for (int t = 0; t < NI; ++t)
          z[t] = v[t];
      }
      __syncthreads();

      // D: direction 1: S, x^I update
      if (tid < PB * NI)
      {
        const int p = tid / NI;
        const int i0 = tid - p * NI;
        const int gp = bt * PB + p;
        if (gp < a.total)
        {
          int64_t g0, g1, g2;
          origin(cur, p, g0, g1, g2);
          const T *z = Z + p * ZW + i0;
          T v[NI], y[NI];
#pragma unroll
          for (int t = 0; t < NI; ++t)
            v[t] = z[S1 * t];
          eo_s<K>(P.Se, P.So, v, y);
          T *xp = a.x + (g1 + 1) * m + (g0 + 1 + i0);
          const T *xo = U + p * UW + (1 + i0) + NC;
#pragma unroll
          for (int i = 0; i < NI; ++i)
          {
            if constexpr (MODE == MODE_BOUNDARY)
              xp[i * m] = y[i];
            else if constexpr (MODE == MODE_FUSED)
              xp[i * m] = xo[NC * i] + y[i];
            else
              xp[i * m] += y[i];
          }
        }
      }
    }
  }
  cp_async_wait_all();
}

template <int D, int K, typename T, int MODE>
void launch_vp_smooth(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a, int sm_count, cudaStream_t s)
{
  constexpr int PB = sm_pb<D, K, T>(), NT = sm_nt<D, K, T>();
  constexpr size_t smem = sm_smem_bytes<D, K, T>();
  static unsigned attr_mask = 0;
  static int occupancy[32] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (first_on_device(attr_mask))
  {
    check_cuda(cudaFuncSetAttribute(vp_smooth_kernel<D, K, T, MODE>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "cudaFuncSetAttribute(smoother)");
    check_cuda(cudaFuncSetAttribute(vp_smooth_kernel<D, K, T, MODE>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100),
               "cudaFuncSetAttribute(smoother carveout)");
    int occ = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vp_smooth_kernel<D, K, T, MODE>, NT, smem),
               "occupancy(smoother)");
    occupancy[dev & 31] = std::max(1, occ);
  }
  const int nbatch = (a.total + PB - 1) / PB;
  if (nbatch == 0)
    return;
  const int grid = nbatch;  // one batch per CTA
  (void)sm_count;
  pdl_launch(vp_smooth_kernel<D, K, T, MODE>, grid, NT, smem, s, P, a);
  check_launch("vp_smooth_kernel");
}

template <int D, int K, typename T>
void launch_vp_smooth_mode(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a, int mode, int sm_count,
                           cudaStream_t s)
{
  switch (mode)
  {
    case MODE_FUSED:
      launch_vp_smooth<D, K, T, MODE_FUSED>(P, a, sm_count, s);
      break;
    case MODE_BOUNDARY:
      launch_vp_smooth<D, K, T, MODE_BOUNDARY>(P, a, sm_count, s);
      break;
    case MODE_RESIDUAL:
      launch_vp_smooth<D, K, T, MODE_RESIDUAL>(P, a, sm_count, s);
      break;
    default:
      launch_vp_smooth<D, K, T, MODE_SOLVE>(P, a, sm_count, s);
      break;
  }
}

}  // namespace pmgb
