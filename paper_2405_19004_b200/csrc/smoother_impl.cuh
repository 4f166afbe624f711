// Fused per-colour vertex-patch smoother kernel for sm_100a.
//
// Replaces the per-patch body of the reference's smooth<T>
// (/root/reference/proj/src/smoother.cpp:109-126, fused; :128-148 boundary;
// :82-108 separate) and its callees gather/scatter_interior
// (patches.cpp:51-121), apply_patch_operator (fastdiag.cpp:199-233) and
// apply_patch_inverse (fastdiag.cpp:164-192).
//
// Design:
//  * one launch per colour; a CTA owns PB patches of that colour;
//  * every sum-factorisation contraction is done by a thread that holds one
//    full 1D line of the tensor in registers and produces the whole output
//    line; the 1D matrices are compile-time-indexed kernel parameters, so the
//    inner loops are pure DFMA/FFMA with uniform-register operands;
//  * shared memory only transposes lines between directions. All stages
//    work IN PLACE in one buffer per patch (2 (2k-1)(2k+1)^2 words in 3D):
//    each thread reads its whole input line before writing its output line
//    into a subset of the same positions, which no other thread touches in
//    that stage. Strides (1, 2k-1, (2k-1)(2k+1)) are odd, so every stage is
//    bank-conflict free for 4- and 8-byte words;
//  * the first contraction (direction 0) reads closure rows straight from
//    HBM/L2 (contiguous per thread), the residual stage reads b and the final
//    stage updates x along direction 2 lines (contiguous across the warp);
//  * 3D residual uses 7 contractions instead of the reference's 8 by
//    summing the two mass-in-direction-2 terms before the last contraction.
#pragma once

#include "common.cuh"

namespace pmgb
{

// patches per CTA and threads per CTA, per (dim, degree). Every stage maps
// exactly one 1D line to one thread (NT >= lines of the widest stage), so no
// stage loops: a loop would let the compiler hoist the parameter-bank matrix
// entries out of it into general registers (hundreds of them in f64).
template <int D, int K>
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

template <int D, int K>
constexpr int sm_nt()
{
  constexpr int NC = 2 * K + 1;
  constexpr int lines = sm_pb<D, K>() * (D == 3 ? NC * NC : NC);
  return ((lines + 31) / 32) * 32;
}

template <int D, int K>
constexpr int sm_patch_stride()
{
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  constexpr int ZS = (D == 3) ? NI * NC * NC : NI * NC;
  return 2 * ZS + 1;  // odd: patches in one warp never alias banks
}

template <int D, int K, typename T>
constexpr size_t sm_smem_bytes()
{
  return static_cast<size_t>(sm_pb<D, K>()) * sm_patch_stride<D, K>() * sizeof(T);
}

// y = Mat x   (Mat rows = outputs)
template <int NO, int NN, typename T>
__device__ __forceinline__ void mat_vec(const T (&Mt)[NO][NN], const T (&in)[NN], T (&out)[NO])
{
#pragma unroll
  for (int i = 0; i < NO; ++i)
  {
    T s = Mt[i][0] * in[0];
#pragma unroll
    for (int j = 1; j < NN; ++j)
      s = fma(Mt[i][j], in[j], s);
    out[i] = s;
  }
}

// y = Mat^T x
template <int N, typename T>
__device__ __forceinline__ void mat_t_vec(const T (&Mt)[N][N], const T (&in)[N], T (&out)[N])
{
#pragma unroll
  for (int j = 0; j < N; ++j)
  {
    T s = Mt[0][j] * in[0];
#pragma unroll
    for (int i = 1; i < N; ++i)
      s = fma(Mt[i][j], in[i], s);
    out[j] = s;
  }
}

template <int D, int K, typename T, int MODE>
__global__ void __launch_bounds__(sm_nt<D, K>())
    vp_smooth_kernel(const __grid_constant__ PatchMats<T, K> P, const __grid_constant__ ColorArgs<T> a)
{
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  constexpr int PB = sm_pb<D, K>(), NT = sm_nt<D, K>();
  constexpr int ZS = (D == 3) ? NI * NC * NC : NI * NC;
  constexpr int PSTR = sm_patch_stride<D, K>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *sm = reinterpret_cast<T *>(smem_raw);

  const int tid = threadIdx.x;
  const int pbase = blockIdx.x * PB;
  const int64_t m = a.m;

  // dof index of closure-local t = 0 per direction (patches.cpp:71:
  // g_a = k (v_a - 1) - 1 + t_a)
  auto origin = [&](int p, int64_t &g0, int64_t &g1, int64_t &g2) -> bool {
    const int gp = pbase + p;
    if (gp >= a.total)
      return false;
    const int j0 = gp % a.np[0];
    const int rest = gp / a.np[0];
    const int j1 = rest % a.np[1];
    const int j2 = rest / a.np[1];
    g0 = static_cast<int64_t>(K) * (2 * j0 + a.vb[0] - 1) - 1;
    g1 = static_cast<int64_t>(K) * (2 * j1 + a.vb[1] - 1) - 1;
    g2 = (D == 3) ? static_cast<int64_t>(K) * (2 * j2 + a.vb[2] - 1) - 1 : 0;
    return true;
  };

  if constexpr (D == 3)
  {
    const int64_t m2 = m * m;
    if constexpr (MODE != MODE_SOLVE)
    {
      // ---- A: direction 0 from global rows: zM = M0 u, zA = A0 u ----------
      static_assert(PB * NC * NC <= NT, "one line per thread per stage");
      if (const int l = tid; l < PB * NC * NC)
        do
        {
        const int p = l / (NC * NC);
        const int rr = l - p * (NC * NC);
        const int j1 = rr % NC, j2 = rr / NC;
        int64_t g0, g1, g2;
        if (!origin(p, g0, g1, g2))
          continue;
        const int64_t y1 = g1 + j1, y2 = g2 + j2;
        const bool rowok = static_cast<uint64_t>(y1) < static_cast<uint64_t>(m) &&
                           static_cast<uint64_t>(y2) < static_cast<uint64_t>(m);
        const bool shell_only = (MODE == MODE_BOUNDARY) && j1 >= 1 && j1 <= NC - 2 && j2 >= 1 &&
                                j2 <= NC - 2;
        const T *row = a.x + (y2 * m + y1) * m + g0;
        T u[NC];
#pragma unroll
        for (int t = 0; t < NC; ++t)
        {
          const bool ok = rowok && static_cast<uint64_t>(g0 + t) < static_cast<uint64_t>(m) &&
                          (!shell_only || t == 0 || t == NC - 1);
          u[t] = ok ? __ldg(row + t) : T(0);
        }
        T zm[NI], za[NI];
        mat_vec(P.M, u, zm);
        mat_vec(P.A, u, za);
        T *Z = sm + p * PSTR + NI * j1 + NI * NC * j2;
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
          Z[i] = zm[i];
          Z[ZS + i] = za[i];
        }
      } while (0);
      __syncthreads();

      // ---- B: direction 1: wMM = M1 zM, wS = A1 zM + M1 zA (in place) -----
      static_assert(PB * NI * NC <= NT, "one line per thread per stage");
      if (const int l = tid; l < PB * NI * NC)
        do
        {
        const int p = l / (NI * NC);
        if (pbase + p >= a.total)
          continue;
        const int rr = l - p * (NI * NC);
        const int i0 = rr % NI, j2 = rr / NI;
        T *Z = sm + p * PSTR + i0 + NI * NC * j2;
        T zm[NC], za[NC];
#pragma unroll
        for (int t = 0; t < NC; ++t)
        {
          zm[t] = Z[NI * t];
          za[t] = Z[ZS + NI * t];
        }
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
          T wm = P.M[i][0] * zm[0];
          T ws = P.A[i][0] * zm[0];
#pragma unroll
          for (int t = 1; t < NC; ++t)
          {
            wm = fma(P.M[i][t], zm[t], wm);
            ws = fma(P.A[i][t], zm[t], ws);
          }
#pragma unroll
          for (int t = 0; t < NC; ++t)
            ws = fma(P.M[i][t], za[t], ws);
          Z[NI * i] = wm;
          Z[ZS + NI * i] = ws;
        }
      } while (0);
      __syncthreads();
    }

    // ---- C: direction 2: r = b - (A2 wMM + M2 wS); y = S^T r (dir 2) -------
    static_assert(PB * NI * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI * NI)
      do
      {
      const int p = l / (NI * NI);
      const int rr = l - p * (NI * NI);
      const int i0 = rr % NI, i1 = rr / NI;
      int64_t g0, g1, g2;
      if (!origin(p, g0, g1, g2))
        continue;
      T *Z = sm + p * PSTR + i0 + NI * i1;
      const int64_t gidx = ((g2 + 1) * m + (g1 + 1 + i1)) * m + (g0 + 1 + i0);
      T r[NI];
      if constexpr (MODE == MODE_SOLVE)
      {
#pragma unroll
        for (int i = 0; i < NI; ++i)
          r[i] = a.r[gidx + i * m2];
      }
      else
      {
        T wm[NC], ws[NC];
#pragma unroll
        for (int t = 0; t < NC; ++t)
        {
          wm[t] = Z[NI * NC * t];
          ws[t] = Z[ZS + NI * NC * t];
        }
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
          T acc = P.A[i][0] * wm[0];
#pragma unroll
          for (int t = 1; t < NC; ++t)
            acc = fma(P.A[i][t], wm[t], acc);
#pragma unroll
          for (int t = 0; t < NC; ++t)
            acc = fma(P.M[i][t], ws[t], acc);
          r[i] = __ldg(a.b + gidx + i * m2) - acc;
        }
        if constexpr (MODE == MODE_RESIDUAL)
        {
#pragma unroll
          for (int i = 0; i < NI; ++i)
            a.r[gidx + i * m2] = r[i];
          continue;
        }
      }
      T y[NI];
      mat_t_vec(P.S, r, y);
#pragma unroll
      for (int j = 0; j < NI; ++j)
        Z[NI * NC * j] = y[j];
    } while (0);
    if constexpr (MODE == MODE_RESIDUAL)
      return;
    __syncthreads();

    // ---- D: direction 1, S^T -----------------------------------------------
    static_assert(PB * NI * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI * NI)
      do
      {
      const int p = l / (NI * NI);
      if (pbase + p >= a.total)
        continue;
      const int rr = l - p * (NI * NI);
      const int i0 = rr % NI, i2 = rr / NI;
      T *Z = sm + p * PSTR + i0 + NI * NC * i2;
      T v[NI], y[NI];
#pragma unroll
      for (int t = 0; t < NI; ++t)
        v[t] = Z[NI * t];
      mat_t_vec(P.S, v, y);
#pragma unroll
      for (int t = 0; t < NI; ++t)
        Z[NI * t] = y[t];
    } while (0);
    __syncthreads();

    // ---- E: direction 0, S^T, scale by 1/(lambda sums), S --------------------
    static_assert(PB * NI * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI * NI)
      do
      {
      const int p = l / (NI * NI);
      if (pbase + p >= a.total)
        continue;
      const int rr = l - p * (NI * NI);
      const int i1 = rr % NI, i2 = rr / NI;
      T *Z = sm + p * PSTR + NI * i1 + NI * NC * i2;
      const T *inv = a.inv + NI * i1 + NI * NI * i2;
      T v[NI], y[NI];
#pragma unroll
      for (int t = 0; t < NI; ++t)
        v[t] = Z[t];
      mat_t_vec(P.S, v, y);
#pragma unroll
      for (int t = 0; t < NI; ++t)
        y[t] *= __ldg(inv + t);
      mat_vec(P.S, y, v);
#pragma unroll
      for (int t = 0; t < NI; ++t)
        Z[t] = v[t];
    } while (0);
    __syncthreads();

    // ---- F: direction 1, S -------------------------------------------------
    static_assert(PB * NI * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI * NI)
      do
      {
      const int p = l / (NI * NI);
      if (pbase + p >= a.total)
        continue;
      const int rr = l - p * (NI * NI);
      const int i0 = rr % NI, i2 = rr / NI;
      T *Z = sm + p * PSTR + i0 + NI * NC * i2;
      T v[NI], y[NI];
#pragma unroll
      for (int t = 0; t < NI; ++t)
        v[t] = Z[NI * t];
      mat_vec(P.S, v, y);
#pragma unroll
      for (int t = 0; t < NI; ++t)
        Z[NI * t] = y[t];
    } while (0);
    __syncthreads();

    // ---- G: direction 2, S, then x^I += v (or = v) --------------------------
    static_assert(PB * NI * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI * NI)
      do
      {
      const int p = l / (NI * NI);
      const int rr = l - p * (NI * NI);
      const int i0 = rr % NI, i1 = rr / NI;
      int64_t g0, g1, g2;
      if (!origin(p, g0, g1, g2))
        continue;
      const T *Z = sm + p * PSTR + i0 + NI * i1;
      T v[NI], y[NI];
#pragma unroll
      for (int t = 0; t < NI; ++t)
        v[t] = Z[NI * NC * t];
      mat_vec(P.S, v, y);
      T *xp = a.x + ((g2 + 1) * m + (g1 + 1 + i1)) * m + (g0 + 1 + i0);
#pragma unroll
      for (int i = 0; i < NI; ++i)
      {
        if constexpr (MODE == MODE_BOUNDARY)
          xp[i * m2] = y[i];
        else
          xp[i * m2] += y[i];
      }
    } while (0);
  }
  else  // ------------------------------- 2D -----------------------------------
  {
    if constexpr (MODE != MODE_SOLVE)
    {
      // A: direction 0 rows from global
      static_assert(PB * NC <= NT, "one line per thread per stage");
      if (const int l = tid; l < PB * NC)
        do
        {
        const int p = l / NC;
        const int j1 = l - p * NC;
        int64_t g0, g1, g2;
        if (!origin(p, g0, g1, g2))
          continue;
        const int64_t y1 = g1 + j1;
        const bool rowok = static_cast<uint64_t>(y1) < static_cast<uint64_t>(m);
        const bool shell_only = (MODE == MODE_BOUNDARY) && j1 >= 1 && j1 <= NC - 2;
        const T *row = a.x + y1 * m + g0;
        T u[NC];
#pragma unroll
        for (int t = 0; t < NC; ++t)
        {
          const bool ok = rowok && static_cast<uint64_t>(g0 + t) < static_cast<uint64_t>(m) &&
                          (!shell_only || t == 0 || t == NC - 1);
          u[t] = ok ? __ldg(row + t) : T(0);
        }
        T zm[NI], za[NI];
        mat_vec(P.M, u, zm);
        mat_vec(P.A, u, za);
        T *Z = sm + p * PSTR + NI * j1;
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
          Z[i] = zm[i];
          Z[ZS + i] = za[i];
        }
      } while (0);
      __syncthreads();
    }

    // B: direction 1: r = b - (A1 zM + M1 zA); y = S^T r
    static_assert(PB * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI)
      do
      {
      const int p = l / NI;
      const int i0 = l - p * NI;
      int64_t g0, g1, g2;
      if (!origin(p, g0, g1, g2))
        continue;
      T *Z = sm + p * PSTR + i0;
      const int64_t gidx = (g1 + 1) * m + (g0 + 1 + i0);
      T r[NI];
      if constexpr (MODE == MODE_SOLVE)
      {
#pragma unroll
        for (int i = 0; i < NI; ++i)
          r[i] = a.r[gidx + i * m];
      }
      else
      {
        T zm[NC], za[NC];
#pragma unroll
        for (int t = 0; t < NC; ++t)
        {
          zm[t] = Z[NI * t];
          za[t] = Z[ZS + NI * t];
        }
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
          T acc = P.A[i][0] * zm[0];
#pragma unroll
          for (int t = 1; t < NC; ++t)
            acc = fma(P.A[i][t], zm[t], acc);
#pragma unroll
          for (int t = 0; t < NC; ++t)
            acc = fma(P.M[i][t], za[t], acc);
          r[i] = __ldg(a.b + gidx + i * m) - acc;
        }
        if constexpr (MODE == MODE_RESIDUAL)
        {
#pragma unroll
          for (int i = 0; i < NI; ++i)
            a.r[gidx + i * m] = r[i];
          continue;
        }
      }
      T y[NI];
      mat_t_vec(P.S, r, y);
#pragma unroll
      for (int j = 0; j < NI; ++j)
        Z[NI * j] = y[j];
    } while (0);
    if constexpr (MODE == MODE_RESIDUAL)
      return;
    __syncthreads();

    // C: direction 0: S^T, scale, S
    static_assert(PB * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI)
      do
      {
      const int p = l / NI;
      if (pbase + p >= a.total)
        continue;
      const int i1 = l - p * NI;
      T *Z = sm + p * PSTR + NI * i1;
      const T *inv = a.inv + NI * i1;
      T v[NI], y[NI];
#pragma unroll
      for (int t = 0; t < NI; ++t)
        v[t] = Z[t];
      mat_t_vec(P.S, v, y);
#pragma unroll
      for (int t = 0; t < NI; ++t)
        y[t] *= __ldg(inv + t);
      mat_vec(P.S, y, v);
#pragma unroll
      for (int t = 0; t < NI; ++t)
        Z[t] = v[t];
    } while (0);
    __syncthreads();

    // D: direction 1: S, x^I update
    static_assert(PB * NI <= NT, "one line per thread per stage");
    if (const int l = tid; l < PB * NI)
      do
      {
      const int p = l / NI;
      const int i0 = l - p * NI;
      int64_t g0, g1, g2;
      if (!origin(p, g0, g1, g2))
        continue;
      const T *Z = sm + p * PSTR + i0;
      T v[NI], y[NI];
#pragma unroll
      for (int t = 0; t < NI; ++t)
        v[t] = Z[NI * t];
      mat_vec(P.S, v, y);
      T *xp = a.x + (g1 + 1) * m + (g0 + 1 + i0);
#pragma unroll
      for (int i = 0; i < NI; ++i)
      {
        if constexpr (MODE == MODE_BOUNDARY)
          xp[i * m] = y[i];
        else
          xp[i * m] += y[i];
      }
    } while (0);
  }
}

template <int D, int K, typename T, int MODE>
void launch_vp_smooth(const PatchMats<T, K> &P, const ColorArgs<T> &a, cudaStream_t s)
{
  constexpr int PB = sm_pb<D, K>(), NT = sm_nt<D, K>();
  constexpr size_t smem = sm_smem_bytes<D, K, T>();
  static unsigned attr_mask = 0;
  if (first_on_device(attr_mask))
  {
    check_cuda(cudaFuncSetAttribute(vp_smooth_kernel<D, K, T, MODE>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)),
               "cudaFuncSetAttribute(smoother)");
    check_cuda(cudaFuncSetAttribute(vp_smooth_kernel<D, K, T, MODE>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100),
               "cudaFuncSetAttribute(smoother carveout)");
  }
  const int grid = (a.total + PB - 1) / PB;
  if (grid == 0)
    return;
  vp_smooth_kernel<D, K, T, MODE><<<grid, NT, smem, s>>>(P, a);
  check_launch("vp_smooth_kernel");
}

template <int D, int K, typename T>
void launch_vp_smooth_mode(const PatchMats<T, K> &P, const ColorArgs<T> &a, int mode,
                           cudaStream_t s)
{
  switch (mode)
  {
    case MODE_FUSED:
      launch_vp_smooth<D, K, T, MODE_FUSED>(P, a, s);
      break;
    case MODE_BOUNDARY:
      launch_vp_smooth<D, K, T, MODE_BOUNDARY>(P, a, s);
      break;
    case MODE_RESIDUAL:
      launch_vp_smooth<D, K, T, MODE_RESIDUAL>(P, a, s);
      break;
    default:
      launch_vp_smooth<D, K, T, MODE_SOLVE>(P, a, s);
      break;
  }
}

}  // namespace pmgb
