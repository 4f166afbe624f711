// Level operator y = A_l x (and fused residual r = b - A_l x) for sm_100a.
//
// Replaces apply_laplacian<T> (/root/reference/proj/src/operator.cpp:122-185)
// and compute_residual<T> (multigrid.cpp:268-276). The reference loops over
// cells in 2^d parity colours and scatter-adds cell contributions. On a
// uniform Cartesian level the operator is exactly the Kronecker sum of the
// global banded 1D mass/stiffness matrices (the identity the reference's own
// CSR oracle relies on, operator.cpp:194-281), so the device kernel is a
// node-centric, deterministic (no atomics) sum factorisation, streamed
// through the last direction:
//   3D, per z-plane q of the input:
//     dir 0: zM = M0 x, zA = A0 x     (x tile with a k-halo, cp.async, smem)
//     dir 1: wM = M1 zM, wS = A1 zM + M1 zA   (registers)
//     dir 2: every output plane p in [q-k, q+k] accumulates
//            A2[p][q] wM + M2[p][q] wS into a register ring of 2k+1 planes
//            (the plane loop is unrolled by 2k+1 so ring slots are static);
//            plane q-k is complete and is written (r = b - acc fused).
//   One barrier per plane: the x tile and the dir-0 results are double
//   buffered and the next plane's tile is fetched while this one computes.
// Band coefficients depend only on the lattice residue p mod k.
#pragma once

#include <cstdlib>

#include "common.cuh"

// level_op3d_xb_kernel for k = 4 (profiles/r02/ab/level_op_xb.txt: residual
// Q4 L7 f64 1.97 -> 1.89 ms, f32 1.48 -> 1.16 ms, Q4 L5 f64 0.056 -> 0.041 ms;
// k = 3 is slower with it: 0.70 -> 1.21 ms, one CTA per SM at 157 registers)
#ifndef PMG_OP_XB
#define PMG_OP_XB 1
#endif

namespace pmgb
{

// ---------------------------------------------------------------------------
// 3D: CTA = 32 x 8 output columns, marching over a z chunk (a multiple of k,
// so the lattice residue of every plane, and with it the dir-2 band row, is a
// compile-time constant of the k-fold unrolled plane loop).
//   per input plane q (3-deep cp.async ring; each thread copies fixed tile
//   slots whose in-plane offsets are computed once):
//     dir 0: zM = M0 x, zA = A0 x on the (8+2k) x 32 rows (band row of the
//            lane's x residue in registers)
//     dir 1: wM = M1 zM, wS = A1 zM + M1 zA (band row of the warp's y residue)
//     dir 2: acc[j] += A2[p][q] wM + M2[p][q] wS for the 2k+1 output planes
//            p = q-k+j (register shift ring); plane q-k is complete: y = b - acc[0].
// One barrier per plane. Deterministic, no atomics.
// ---------------------------------------------------------------------------
template <int K, typename T>
struct Op3Cfg
{
#ifndef PMG_OP_TY
#define PMG_OP_TY 8
#endif
#ifndef PMG_OP_NB
#define PMG_OP_NB 3
#endif
  static constexpr int TX = 32, TY = PMG_OP_TY, NT = TX * TY, W = 2 * K + 1;
  static constexpr int NB = PMG_OP_NB;  // input-plane ring (NB - 1 planes in flight)
  static constexpr int XW = TX + 2 * K, XH = TY + 2 * K, XN = XW * XH;
  static constexpr int NLOAD = (XN + NT - 1) / NT;   // tile slots per thread
  static constexpr int ROWS = (XH + TY - 1) / TY;    // dir-0 rows per thread
  static constexpr bool C1REG = K <= 2;              // dir-1 band row in registers
  static constexpr size_t SMEM =
      sizeof(T) * (NB * static_cast<size_t>(XN) + NB * NT + 4 * static_cast<size_t>(XH) * TX + 2 * K * W);
};

// cp.async.wait_group with a run-time count (0..7)
__device__ __forceinline__ void cp_wait_groups(int n)
{
  switch (n)
  {
  case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
  case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
  case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
  case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
  case 4: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
  case 5: asm volatile("cp.async.wait_group 5;\n" ::: "memory"); break;
  case 6: asm volatile("cp.async.wait_group 6;\n" ::: "memory"); break;
  default: asm volatile("cp.async.wait_group 7;\n" ::: "memory"); break;
  }
}

template <int K, typename T>
constexpr size_t op3d_smem()
{
  return Op3Cfg<K, T>::SMEM;
}

template <typename T>
__device__ __forceinline__ void op_cp_async(T *smem, const T *gmem, bool valid)
{
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 4 : 0)
                 : "memory");
}

// two resident CTAs per SM for k >= 3 (measured: register-capped 128 beats
// the unconstrained 130-214 registers; for k <= 2 the compiler's choice wins)
#ifndef PMG_OP_MINB_LO
#define PMG_OP_MINB_LO 1
#endif
template <int K>
constexpr int op3d_minb()
{
  return K >= 3 ? 2 : PMG_OP_MINB_LO;
}

// dir 1 for a warp whose rows have lattice residue RES: rows of residue
// RES != 0 couple only their own cell (band offsets [K - RES, 2K - RES]), so
// the structurally zero taps, and their shared-memory loads, are dropped at
// compile time (bitwise the same sums: the dropped terms are exact zeros)
template <int K, typename T, int RES>
__device__ __forceinline__ void op3_dir1(const T *zm, const T *za, const T *cm_, const T *ca_, int wy, int lane,
                                         T &wm_out, T &ws_out)
{
  constexpr int W = 2 * K + 1, TX = 32;
  T wm = T(0), ws = T(0), ws2 = T(0), wm2 = T(0);
#pragma unroll
  for (int o = 0; o < W; ++o)
  {
    if (RES != 0 && (o < K - RES || o > 2 * K - RES))
      continue;
    const T vm = zm[(wy + o) * TX + lane], va = za[(wy + o) * TX + lane];
    const T cm = cm_[o], ca = ca_[o];
    if (o & 1)
      wm2 = fma(cm, vm, wm2);
    else
      wm = fma(cm, vm, wm);
    ws = fma(ca, vm, ws);
    ws2 = fma(cm, va, ws2);
  }
  wm_out = wm + wm2;
  ws_out = ws + ws2;
}

template <int K, typename T, int R = 0>
__device__ __forceinline__ void op3_dir1_res(int res, const T *zm, const T *za, const T *cm_, const T *ca_, int wy,
                                             int lane, T &wm, T &ws)
{
  if constexpr (R < K)
  {
    if (res == R)
    {
      op3_dir1<K, T, R>(zm, za, cm_, ca_, wy, lane, wm, ws);
      return;
    }
    op3_dir1_res<K, T, R + 1>(res, zm, za, cm_, ca_, wy, lane, wm, ws);
  }
}

template <int K, typename T, bool RESID>
__global__ void __launch_bounds__(Op3Cfg<K, T>::NT, op3d_minb<K>())
    level_op3d_kernel(const __grid_constant__ BandMats<T, K> B, const T *__restrict__ x,
                      const T *__restrict__ b, T *__restrict__ y, int64_t m, int zchunk, int64_t zbeg,
                      int64_t zend)
{
  pdl_prologue();
  using C = Op3Cfg<K, T>;
  constexpr int TX = C::TX, TY = C::TY, NT = C::NT, W = C::W, XW = C::XW, XH = C::XH, XN = C::XN;
  constexpr int NLOAD = C::NLOAD, ROWS = C::ROWS, NB = C::NB;
  extern __shared__ __align__(16) unsigned char smraw[];
  T *Xs = reinterpret_cast<T *>(smraw);  // [NB][XH][XW]  input planes
  T *Bv = Xs + NB * XN;                  // [NB][NT]      b of the output planes
  T *ZM = Bv + NB * NT;                  // [2][XH][TX]
  T *ZA = ZM + 2 * XH * TX;              // [2][XH][TX]
  T *bm = ZA + 2 * XH * TX;              // [K][W]
  T *ba = bm + K * W;

  const int tid = threadIdx.x;
  const int lane = tid % TX, wy = tid / TX;
  for (int e = tid; e < K * W; e += NT)
  {
    bm[e] = (&B.M[0][0])[e];
    ba[e] = (&B.A[0][0])[e];
  }
  const int g0 = static_cast<int>(blockIdx.x) * TX;
  const int g1 = static_cast<int>(blockIdx.y) * TY;
  // output planes [zbeg, zend) (x, b, y indexed by GLOBAL plane: slab callers
  // pass bases shifted by their first plane); chunks start on multiples of K
  const int64_t zs = (zbeg / K) * K + static_cast<int64_t>(blockIdx.z) * zchunk;  // multiple of K
  const int64_t ze = min(zs + zchunk, zend);
  const int64_t m2 = m * m;
  // this thread's tile slots: in-plane offset and validity (fixed for all planes)
  int off[NLOAD];
  unsigned okm = 0;
#pragma unroll
  for (int j = 0; j < NLOAD; ++j)
  {
    const int e = tid + j * NT;
    const int jr = e / XW, ir = e - (e / XW) * XW;
    const int gx = g0 - K + ir, gy = g1 - K + jr;
    const bool ok = e < XN && gx >= 0 && gx < m && gy >= 0 && gy < m;
    off[j] = ok ? gy * static_cast<int>(m) + gx : 0;
    okm |= (ok ? 1u : 0u) << j;
  }
  const bool out_ok = (g0 + lane < m) && (g1 + wy < m);
  const int out_off = (g1 + wy) * static_cast<int>(m) + g0 + lane;
  __syncthreads();
  T c0m[W], c0a[W];
  {
    const int res0 = (g0 + lane + 1) % K;
#pragma unroll
    for (int o = 0; o < W; ++o)
    {
      c0m[o] = bm[res0 * W + o];
      c0a[o] = ba[res0 * W + o];
    }
  }
  const int res1 = (g1 + wy + 1) % K;
  T c1r_m[C::C1REG ? W : 1], c1r_a[C::C1REG ? W : 1];
  if constexpr (C::C1REG)
  {
#pragma unroll
    for (int o = 0; o < W; ++o)
    {
      c1r_m[o] = bm[res1 * W + o];
      c1r_a[o] = ba[res1 * W + o];
    }
  }
  const T *c1s_m = bm + res1 * W, *c1s_a = ba + res1 * W;
  const int NPL = static_cast<int>(ze - zs) + 2 * K;  // input planes zs-K .. ze+K-1

  auto issue = [&](int it) {
    const int64_t q = zs - K + it;
    // planes below zbeg - K feed only outputs below zbeg (never stored): not
    // read, so a slab caller need only hold planes from zbeg - K
    const bool zin = q >= 0 && q < m && q >= zbeg - K;
    T *dst = Xs + (it % NB) * XN;
    const T *xq = x + (zin ? q : 0) * m2;
#pragma unroll
    for (int j = 0; j < NLOAD; ++j)
    {
      const int e = tid + j * NT;
      if (e < XN)
      {
        const bool ok = zin && ((okm >> j) & 1u);
        op_cp_async(dst + e, xq + off[j], ok);
      }
    }
    if constexpr (RESID)
    {
      const int64_t p = q - K;
      const bool ok = out_ok && it >= 2 * K && p < ze && p >= zbeg;
      op_cp_async(Bv + (it % NB) * NT + tid, ok ? b + p * m2 + out_off : b, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  T acc[W];
#pragma unroll
  for (int o = 0; o < W; ++o)
    acc[o] = T(0);

  // planes 0 .. NB-2 in flight; wait for plane 0
  const int npre = min(NB - 1, NPL);
  for (int it = 0; it < npre; ++it)
    issue(it);
  cp_wait_groups(npre - 1);
  __syncthreads();

  for (int base = 0; base < NPL; base += K)
  {
#pragma unroll
    for (int u = 0; u < K; ++u)
    {
      const int it = base + u;  // uniform across the CTA
      if (it >= NPL)
        break;
      if (it + NB - 1 < NPL)
        issue(it + NB - 1);
      // dir 0
      const T *xs = Xs + (it % NB) * XN;
      T *zm = ZM + (it & 1) * XH * TX;
      T *za = ZA + (it & 1) * XH * TX;
#pragma unroll
      for (int rr = 0; rr < ROWS; ++rr)
      {
        const int j = wy + rr * TY;
        if (j < XH)
        {
          // two interleaved partial sums per output: halves the FMA chain
          const T *xr = xs + j * XW + lane;
          T vm0 = c0m[0] * xr[0], va0 = c0a[0] * xr[0];
          T vm1 = c0m[1] * xr[1], va1 = c0a[1] * xr[1];
#pragma unroll
          for (int o = 2; o < W; o += 2)
          {
            vm0 = fma(c0m[o], xr[o], vm0);
            va0 = fma(c0a[o], xr[o], va0);
            if (o + 1 < W)
            {
              vm1 = fma(c0m[o + 1], xr[o + 1], vm1);
              va1 = fma(c0a[o + 1], xr[o + 1], va1);
            }
          }
          zm[j * TX + lane] = vm0 + vm1;
          za[j * TX + lane] = va0 + va1;
        }
      }
      // plane it + 1 complete (groups issued after it may stay in flight)
      cp_wait_groups(max(0, min(it + NB - 1, NPL - 1) - (it + 1)));
      __syncthreads();
      // dir 1
      T wm = T(0), ws = T(0);
      if constexpr (C::C1REG)
      {
        T ws2 = T(0), wm2 = T(0);
#pragma unroll
        for (int o = 0; o < W; ++o)
        {
          const T vm = zm[(wy + o) * TX + lane], va = za[(wy + o) * TX + lane];
          const T cm = c1r_m[C::C1REG ? o : 0];
          const T ca = c1r_a[C::C1REG ? o : 0];
          if (o & 1)
            wm2 = fma(cm, vm, wm2);
          else
            wm = fma(cm, vm, wm);
          ws = fma(ca, vm, ws);
          ws2 = fma(cm, va, ws2);
        }
        wm += wm2;
        ws += ws2;
      }
      else
        op3_dir1_res<K, T>(res1, zm, za, c1s_m, c1s_a, wy, lane, wm, ws);
      // dir 2: output plane p = q - K + jo, lattice residue (p + 1) mod K =
      // (u + 1 + jo) mod K; band offset q - p + K = 2K - jo
#pragma unroll
      for (int jo = 0; jo < W; ++jo)
      {
        const int res = (u + 1 + jo) % K;
        // rows of residue res != 0 couple only their own cell: offsets
        // [K - res, 2K - res]; the other band entries are exact zeros
        // (compile-time here, so their FMAs are not emitted)
        const int o = 2 * K - jo;
        if (K >= 3 && res != 0 && (o < K - res || o > 2 * K - res))
          continue;  // (kept for k = 2: measured 1% slower there)
        acc[jo] = fma(B.A[res][o], wm, acc[jo]);
        acc[jo] = fma(B.M[res][o], ws, acc[jo]);
      }
      const int64_t p_out = zs - 2 * K + it;
      if (it >= 2 * K && p_out < ze && p_out >= zbeg && out_ok)
      {
        const int64_t idx = p_out * m2 + out_off;
        if constexpr (RESID)
          y[idx] = Bv[(it % NB) * NT + tid] - acc[0];
        else
          y[idx] = acc[0];
      }
#pragma unroll
      for (int jo = 0; jo < W - 1; ++jo)
        acc[jo] = acc[jo + 1];
      acc[W - 1] = T(0);
    }
  }
}

// ---------------------------------------------------------------------------
// 3D, k <= 2: register-blocked ("cb" = cell-blocked). Lane l of warp w owns
// the K columns of one cell (nodes X0 + K l .. X0 + K l + K - 1, lattice
// residues 0 .. K-1) on BY consecutive rows (residues i mod K): per input
// plane it streams the BY + 2K rows of its 3K-wide window from the staged
// tile through registers — dir 0 (compile-time residue, structurally zero
// taps dropped) straight into the dir-1 sums of the rows it feeds — so the
// dir-0 results never round-trip through shared memory and dir 1 reads
// nothing. dir 2 is the register ring of level_op3d_kernel. The per-output
// shared traffic drops from ~30 words to (BY + 2K) 3K / (BY K) (9 words at
// k = 2): level_op3d_kernel is bound by shared-memory wavefronts at k <= 2
// (f64 C2 L6 residual 35.8 us = 21% of HBM, the same at 2-4 CTAs per SM).
// The tile row is stored with one pad word per K columns (K = 2: lane stride
// 3 words), conflict-free. One barrier per plane.
// ---------------------------------------------------------------------------
#ifndef PMG_OP_CB
#define PMG_OP_CB 1
#endif
#ifndef PMG_OP_CB_NW
#define PMG_OP_CB_NW 4
#endif
template <int K, typename T>
struct Op3CbCfg
{
  static constexpr int NW = PMG_OP_CB_NW, NT = 32 * NW, W = 2 * K + 1;
  static constexpr int BY = K == 1 ? 4 : 2;          // rows per thread (a multiple of K)
  static constexpr int XC = 32 * K, YC = NW * BY;    // output nodes of a tile
  static constexpr int XW = XC + 2 * K, XH = YC + 2 * K;
  static constexpr int XWP = K == 1 ? XW : XW + XW / K + 1;  // padded pitch
  static constexpr int XN = XW * XH, NLOAD = (XN + NT - 1) / NT;
  static constexpr int OUT = BY * K;  // outputs per thread per plane
  static constexpr size_t SMEM = sizeof(T) * (3 * static_cast<size_t>(XH) * XWP + 3 * static_cast<size_t>(OUT) * NT);
  static_assert(BY % K == 0, "rows per thread: whole cells");
};

// shared column of tile column X
template <int K>
__device__ __forceinline__ constexpr int cb_pos(int X)
{
  return K == 1 ? X : X + X / K;
}

template <int K, typename T, bool RESID>
__global__ void __launch_bounds__(Op3CbCfg<K, T>::NT)
    level_op3d_cb_kernel(const __grid_constant__ BandMats<T, K> B, const T *__restrict__ x,
                         const T *__restrict__ b, T *__restrict__ y, int64_t m, int zchunk, int64_t zbeg,
                         int64_t zend)
{
  pdl_prologue();
  using C = Op3CbCfg<K, T>;
  constexpr int NT = C::NT, W = C::W, BY = C::BY, XW = C::XW, XH = C::XH, XWP = C::XWP, XN = C::XN;
  constexpr int NLOAD = C::NLOAD, OUT = C::OUT;
  extern __shared__ __align__(16) unsigned char smraw[];
  T *Xs = reinterpret_cast<T *>(smraw);  // [3][XH][XWP]  input planes
  T *Bv = Xs + 3 * XH * XWP;             // [3][OUT][NT]  b of the thread's outputs

  const int tid = threadIdx.x;
  const int lane = tid & 31, wy = tid >> 5;
  // tile origin in node coordinates (node = interior index + 1)
  const int X0 = static_cast<int>(blockIdx.x) * C::XC;
  const int Y0 = static_cast<int>(blockIdx.y) * C::YC;
  const int64_t zs = (zbeg / K) * K + static_cast<int64_t>(blockIdx.z) * zchunk;  // multiple of K
  const int64_t ze = min(zs + zchunk, zend);
  const int64_t m2 = m * m;
  const int mi = static_cast<int>(m);

  int off[NLOAD], dpos[NLOAD];
  unsigned okm = 0;
#pragma unroll
  for (int j = 0; j < NLOAD; ++j)
  {
    const int e = tid + j * NT;
    const int jr = e / XW, X = e - jr * XW;
    const int ix = X0 - K + X - 1, iy = Y0 - K + jr - 1;  // interior indices
    const bool ok = e < XN && ix >= 0 && ix < mi && iy >= 0 && iy < mi;
    off[j] = ok ? iy * mi + ix : 0;
    dpos[j] = jr * XWP + cb_pos<K>(X);
    okm |= (ok ? 1u : 0u) << j;
  }
  // this thread's outputs (i, r): interior (iy0 + i, ix0 + r)
  const int ix0 = X0 + K * lane - 1, iy0 = Y0 + BY * wy - 1;
  unsigned outm = 0;
#pragma unroll
  for (int i = 0; i < BY; ++i)
#pragma unroll
    for (int r = 0; r < K; ++r)
    {
      const bool ok = ix0 + r >= 0 && ix0 + r < mi && iy0 + i >= 0 && iy0 + i < mi;
      outm |= (ok ? 1u : 0u) << (i * K + r);
    }
  const int NPL = static_cast<int>(ze - zs) + 2 * K;  // input planes zs-K .. ze+K-1

  auto issue = [&](int it) {
    const int64_t q = zs - K + it;
    const bool zin = q >= 0 && q < m && q >= zbeg - K;
    T *dst = Xs + (it % 3) * XH * XWP;
    const T *xq = x + (zin ? q : 0) * m2;
#pragma unroll
    for (int j = 0; j < NLOAD; ++j)
    {
      const int e = tid + j * NT;
      if (e < XN)
        op_cp_async(dst + dpos[j], xq + off[j], zin && ((okm >> j) & 1u));
    }
    if constexpr (RESID)
    {
      const int64_t p = q - K;
      const bool okp = it >= 2 * K && p < ze && p >= zbeg;
#pragma unroll
      for (int i = 0; i < BY; ++i)
#pragma unroll
        for (int r = 0; r < K; ++r)
        {
          const bool ok = okp && ((outm >> (i * K + r)) & 1u);
          op_cp_async(Bv + ((it % 3) * OUT + i * K + r) * NT + tid,
                      ok ? b + p * m2 + static_cast<int64_t>(iy0 + i) * m + (ix0 + r) : b, ok);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  T acc[W][BY][K];
#pragma unroll
  for (int o = 0; o < W; ++o)
#pragma unroll
    for (int i = 0; i < BY; ++i)
#pragma unroll
      for (int r = 0; r < K; ++r)
        acc[o][i][r] = T(0);

  issue(0);
  if (NPL > 1)
  {
    issue(1);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  }
  else
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  for (int base = 0; base < NPL; base += K)
  {
#pragma unroll
    for (int u = 0; u < K; ++u)
    {
      const int it = base + u;  // uniform across the CTA
      if (it >= NPL)
        break;
      if (it + 2 < NPL)
        issue(it + 2);
      const T *xs = Xs + (it % 3) * XH * XWP + (wy * BY) * XWP + cb_pos<K>(K * lane);
      // dir 0 row by row, each row straight into the dir-1 sums it feeds
      T wm[BY][K], ws[BY][K];
#pragma unroll
      for (int i = 0; i < BY; ++i)
#pragma unroll
        for (int r = 0; r < K; ++r)
        {
          wm[i][r] = T(0);
          ws[i][r] = T(0);
        }
#pragma unroll
      for (int jr = 0; jr < BY + 2 * K; ++jr)
      {
        T v[3 * K];
#pragma unroll
        for (int t = 0; t < 3 * K; ++t)
          v[t] = xs[jr * XWP + (K == 1 ? t : t + t / K)];
#pragma unroll
        for (int r = 0; r < K; ++r)
        {
          // output column residue r: input window v[r + o], o in [0, 2K]
          T zm = T(0), za = T(0);
#pragma unroll
          for (int o = 0; o < W; ++o)
          {
            if (r != 0 && (o < K - r || o > 2 * K - r))
              continue;
            zm = fma(B.M[r][o], v[r + o], zm);
            za = fma(B.A[r][o], v[r + o], za);
          }
#pragma unroll
          for (int i = 0; i < BY; ++i)
          {
            const int o = jr - i;  // band offset of input row jr for output row i
            const int ry = i % K;
            if (o < 0 || o > 2 * K || (ry != 0 && (o < K - ry || o > 2 * K - ry)))
              continue;
            wm[i][r] = fma(B.M[ry][o], zm, wm[i][r]);
            ws[i][r] = fma(B.A[ry][o], zm, fma(B.M[ry][o], za, ws[i][r]));
          }
        }
      }
      // dir 2: output plane p = q - K + jo, residue (u + 1 + jo) mod K, band
      // offset 2K - jo
#pragma unroll
      for (int jo = 0; jo < W; ++jo)
      {
        const int res = (u + 1 + jo) % K;
        const int o = 2 * K - jo;
        if (res != 0 && (o < K - res || o > 2 * K - res))
          continue;
#pragma unroll
        for (int i = 0; i < BY; ++i)
#pragma unroll
          for (int r = 0; r < K; ++r)
            acc[jo][i][r] = fma(B.A[res][o], wm[i][r], fma(B.M[res][o], ws[i][r], acc[jo][i][r]));
      }
      const int64_t p_out = zs - 2 * K + it;
      if (it >= 2 * K && p_out < ze && p_out >= zbeg)
      {
#pragma unroll
        for (int i = 0; i < BY; ++i)
#pragma unroll
          for (int r = 0; r < K; ++r)
            if ((outm >> (i * K + r)) & 1u)
            {
              const int64_t idx = p_out * m2 + static_cast<int64_t>(iy0 + i) * m + (ix0 + r);
              if constexpr (RESID)
                y[idx] = Bv[((it % 3) * OUT + i * K + r) * NT + tid] - acc[0][i][r];
              else
                y[idx] = acc[0][i][r];
            }
      }
#pragma unroll
      for (int jo = 0; jo < W - 1; ++jo)
#pragma unroll
        for (int i = 0; i < BY; ++i)
#pragma unroll
          for (int r = 0; r < K; ++r)
            acc[jo][i][r] = acc[jo + 1][i][r];
#pragma unroll
      for (int i = 0; i < BY; ++i)
#pragma unroll
        for (int r = 0; r < K; ++r)
          acc[W - 1][i][r] = T(0);
      if (it + 2 < NPL)
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// 3D, k >= 3: one CELL per thread in x (xb = "x-blocked"). Lane l owns the K
// consecutive output columns of one cell, starting at its vertex (lattice
// residue 0), so every output's residue — and with it which band taps are
// structurally zero — is a compile-time constant: dir 0 reads the 2K+1 window
// [Kc - K, Kc + K] once for all K outputs (the vertex couples to the whole
// window, the interior nodes of the cell only to its K+1 nodes) instead of
// 2K+1 values per output. The tile row is stored with one pad word per K
// columns, so the lanes' windows (stride K+1 words) are bank-conflict-free.
// dir 1 (per-warp row residue, compile-time variant) and dir 2 (register
// ring, compile-time plane residue) as in level_op3d_kernel.
// ---------------------------------------------------------------------------
template <int K, typename T>
struct Op3XbCfg
{
  static constexpr int TX = 32, TY = 8, NT = TX * TY, W = 2 * K + 1;
  static constexpr int XC = TX * K;                        // output columns of a tile
  static constexpr int XW = XC + 2 * K, XH = TY + 2 * K;  // input tile
  static constexpr int XWP = XW + XW / K + 1;              // padded row pitch (words)
  static constexpr int ZCP = XC + XC / K + 1;              // padded dir-0 result row pitch
  static constexpr int XN = XW * XH;
  static constexpr int NLOAD = (XN + NT - 1) / NT;
  static constexpr int ROWS = (XH + TY - 1) / TY;
  static constexpr size_t SMEM = sizeof(T) * (3 * static_cast<size_t>(XH) * XWP + 4 * static_cast<size_t>(XH) * ZCP);
};

template <int K, typename T, int RES>
__device__ __forceinline__ void opxb_dir1(const BandMats<T, K> &B, const T *zm, const T *za, int wy, int lane,
                                          T (&wm)[K], T (&ws)[K])
{
  constexpr int W = 2 * K + 1, ZCP = Op3XbCfg<K, T>::ZCP;
#pragma unroll
  for (int r = 0; r < K; ++r)
  {
    T a = T(0), b2 = T(0);
#pragma unroll
    for (int o = 0; o < W; ++o)
    {
      if (RES != 0 && (o < K - RES || o > 2 * K - RES))
        continue;
      const int pos = (wy + o) * ZCP + (K + 1) * lane + r;
      const T vm = zm[pos], va = za[pos];
      a = fma(B.M[RES][o], vm, a);
      b2 = fma(B.A[RES][o], vm, fma(B.M[RES][o], va, b2));
    }
    wm[r] = a;
    ws[r] = b2;
  }
}

template <int K, typename T, int R = 0>
__device__ __forceinline__ void opxb_dir1_res(const BandMats<T, K> &B, int res, const T *zm, const T *za, int wy,
                                              int lane, T (&wm)[K], T (&ws)[K])
{
  if constexpr (R < K)
  {
    if (res == R)
    {
      opxb_dir1<K, T, R>(B, zm, za, wy, lane, wm, ws);
      return;
    }
    opxb_dir1_res<K, T, R + 1>(B, res, zm, za, wy, lane, wm, ws);
  }
}

template <int K, typename T, bool RESID>
__global__ void __launch_bounds__(Op3XbCfg<K, T>::NT, 1)
    level_op3d_xb_kernel(const __grid_constant__ BandMats<T, K> B, const T *__restrict__ x,
                         const T *__restrict__ b, T *__restrict__ y, int64_t m, int zchunk, int64_t zbeg,
                         int64_t zend)
{
  pdl_prologue();
  using C = Op3XbCfg<K, T>;
  constexpr int TX = C::TX, TY = C::TY, NT = C::NT, W = C::W, XW = C::XW, XH = C::XH, XN = C::XN;
  constexpr int XWP = C::XWP, ZCP = C::ZCP, NLOAD = C::NLOAD, ROWS = C::ROWS;
  extern __shared__ __align__(16) unsigned char smraw[];
  T *Xs = reinterpret_cast<T *>(smraw);  // [3][XH][XWP]  input planes (padded rows)
  T *ZM = Xs + 3 * XH * XWP;             // [2][XH][ZCP]
  T *ZA = ZM + 2 * XH * ZCP;             // [2][XH][ZCP]

  const int tid = threadIdx.x;
  const int lane = tid % TX, wy = tid / TX;
  // tile columns: X = x0 + K lane + r, x0 + 1 = K * 32 * bx (a vertex)
  const int64_t x0 = static_cast<int64_t>(blockIdx.x) * C::XC - 1;
  const int64_t g1 = static_cast<int64_t>(blockIdx.y) * TY;
  const int64_t zs = (zbeg / K) * K + static_cast<int64_t>(blockIdx.z) * zchunk;
  const int64_t ze = min(zs + zchunk, zend);
  const int64_t m2 = m * m;
  // tile slots: (row jr, column ir) -> padded smem position, global offset
  int spos[NLOAD];
  int64_t goff[NLOAD];
  unsigned okm = 0;
#pragma unroll
  for (int j = 0; j < NLOAD; ++j)
  {
    const int e = tid + j * NT;
    const int jr = e / XW, ir = e - (e / XW) * XW;
    const int64_t gx = x0 - K + ir, gy = g1 - K + jr;
    const bool ok = e < XN && gx >= 0 && gx < m && gy >= 0 && gy < m;
    spos[j] = jr * XWP + ir + ir / K;
    goff[j] = ok ? gy * m + gx : 0;
    okm |= (ok ? 1u : 0u) << j;
  }
  const int64_t oy = g1 + wy;
  const bool row_ok = oy < m;
  const int res1 = static_cast<int>((oy + 1) % K);
  const int NPL = static_cast<int>(ze - zs) + 2 * K;

  auto issue = [&](int it) {
    const int64_t q = zs - K + it;
    const bool zin = q >= 0 && q < m && q >= zbeg - K;
    T *dst = Xs + (it % 3) * XH * XWP;
    const T *xq = x + (zin ? q : 0) * m2;
#pragma unroll
    for (int j = 0; j < NLOAD; ++j)
    {
      if (tid + j * NT < XN)
        op_cp_async(dst + spos[j], xq + goff[j], zin && ((okm >> j) & 1u));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  T acc[K][W];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int o = 0; o < W; ++o)
      acc[r][o] = T(0);

  issue(0);
  if (NPL > 1)
  {
    issue(1);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  }
  else
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();

  for (int base = 0; base < NPL; base += K)
  {
#pragma unroll
    for (int u = 0; u < K; ++u)
    {
      const int it = base + u;
      if (it >= NPL)
        break;
      if (it + 2 < NPL)
        issue(it + 2);
      // b of this iteration's output plane into registers (used at the end)
      const int64_t p_out = zs - 2 * K + it;
      const bool out_it = it >= 2 * K && p_out < ze && p_out >= zbeg && row_ok;
      T bv[K];
      if constexpr (RESID)
      {
#pragma unroll
        for (int r = 0; r < K; ++r)
        {
          const int64_t X = x0 + K * lane + r;
          bv[r] = (out_it && X >= 0 && X < m) ? __ldg(b + p_out * m2 + oy * m + X) : T(0);
        }
      }
      // dir 0: the cell window of each row, K outputs with compile-time taps
      const T *xs = Xs + (it % 3) * XH * XWP;
      T *zm = ZM + (it & 1) * XH * ZCP;
      T *za = ZA + (it & 1) * XH * ZCP;
#pragma unroll
      for (int rr = 0; rr < ROWS; ++rr)
      {
        const int j = wy + rr * TY;
        if (j < XH)
        {
          const T *xr = xs + j * XWP + (K + 1) * lane;
          T w[2 * K + 1];
#pragma unroll
          for (int q = 0; q <= 2 * K; ++q)
            w[q] = xr[q + q / K];
          T *zmr = zm + j * ZCP + (K + 1) * lane;
          T *zar = za + j * ZCP + (K + 1) * lane;
          {
            T vm0 = B.M[0][0] * w[0], va0 = B.A[0][0] * w[0];
            T vm1 = B.M[0][1] * w[1], va1 = B.A[0][1] * w[1];
#pragma unroll
            for (int q = 2; q <= 2 * K; q += 2)
            {
              vm0 = fma(B.M[0][q], w[q], vm0);
              va0 = fma(B.A[0][q], w[q], va0);
              if (q + 1 <= 2 * K)
              {
                vm1 = fma(B.M[0][q + 1], w[q + 1], vm1);
                va1 = fma(B.A[0][q + 1], w[q + 1], va1);
              }
            }
            zmr[0] = vm0 + vm1;
            zar[0] = va0 + va1;
          }
#pragma unroll
          for (int r = 1; r < K; ++r)
          {
            T vm = T(0), va = T(0);
#pragma unroll
            for (int q = K; q <= 2 * K; ++q)
            {
              vm = fma(B.M[r][q - r], w[q], vm);
              va = fma(B.A[r][q - r], w[q], va);
            }
            zmr[r] = vm;
            zar[r] = va;
          }
        }
      }
      if (it + 2 < NPL)
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      // dir 1 (the warp's row residue as a compile-time variant)
      T wm[K], ws[K];
      opxb_dir1_res<K, T>(B, res1, zm, za, wy, lane, wm, ws);
      // dir 2: output plane p = q - K + jo, residue (u + 1 + jo) mod K,
      // band offset 2K - jo; structurally zero taps dropped
#pragma unroll
      for (int jo = 0; jo < W; ++jo)
      {
        const int res = (u + 1 + jo) % K;
        const int o = 2 * K - jo;
        if (res != 0 && (o < K - res || o > 2 * K - res))
          continue;
#pragma unroll
        for (int r = 0; r < K; ++r)
        {
          acc[r][jo] = fma(B.A[res][o], wm[r], acc[r][jo]);
          acc[r][jo] = fma(B.M[res][o], ws[r], acc[r][jo]);
        }
      }
      if (out_it)
      {
#pragma unroll
        for (int r = 0; r < K; ++r)
        {
          const int64_t X = x0 + K * lane + r;
          if (X >= 0 && X < m)
          {
            const int64_t idx = p_out * m2 + oy * m + X;
            if constexpr (RESID)
              y[idx] = bv[r] - acc[r][0];
            else
              y[idx] = acc[r][0];
          }
        }
      }
#pragma unroll
      for (int r = 0; r < K; ++r)
      {
#pragma unroll
        for (int jo = 0; jo < W - 1; ++jo)
          acc[r][jo] = acc[r][jo + 1];
        acc[r][W - 1] = T(0);
      }
    }
  }
}

// 2D: CTA = 128 columns marching down a chunk of rows that starts on a
// multiple of K (so every row's lattice residue, and with it the dir-1 band
// row, is a compile-time constant of the K-fold unrolled row loop: the
// structurally zero taps are dropped and the coefficients are parameter-bank
// operands), a 3-deep cp.async row ring (one barrier per row) and a register
// shift ring of the 2K+1 rows in flight — the 3D kernel's organisation.
template <int K, typename T, bool RESID>
__global__ void __launch_bounds__(128)
    level_op2d_kernel(const __grid_constant__ BandMats<T, K> B, const T *__restrict__ x,
                         const T *__restrict__ b, T *__restrict__ y, int64_t m, int rchunk)
{
  pdl_prologue();
  constexpr int T0 = 128, W = 2 * K + 1, XW = T0 + 2 * K;
  constexpr int NL = (XW + T0 - 1) / T0;
  __shared__ __align__(16) T Xs[3][XW];
  const int i = threadIdx.x;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * T0;
  const int64_t rs = static_cast<int64_t>(blockIdx.y) * rchunk;  // multiple of K
  const int64_t re = min(rs + rchunk, m);
  // dir-0 band row of this lane's residue: in registers, or for K = 4, 5 read
  // from shared memory (2 (2K+1) registers fewer -> more resident CTAs;
  // profiles/r01/ab_levelop2d_coef_smem.txt: k = 4 -14%, k = 5 -4%; k = 7 +6%)
  constexpr bool C0S = K == 4 || K == 5;
  __shared__ T c0s[C0S ? 2 : 1][C0S ? K : 1][C0S ? W : 1];
  T c0m[C0S ? 1 : W], c0a[C0S ? 1 : W];
  const int res0 = static_cast<int>((g0 + i + 1) % K);
  if constexpr (C0S)
  {
    for (int e = i; e < K * W; e += T0)
    {
      c0s[0][e / W][e % W] = (&B.M[0][0])[e];
      c0s[1][e / W][e % W] = (&B.A[0][0])[e];
    }
  }
  else
  {
#pragma unroll
    for (int o = 0; o < W; ++o)
    {
      c0m[o] = B.M[res0][o];
      c0a[o] = B.A[res0][o];
    }
  }
  auto cm0 = [&](int o) -> T {
    if constexpr (C0S)
      return c0s[0][res0][o];
    else
      return c0m[o];
  };
  auto ca0 = [&](int o) -> T {
    if constexpr (C0S)
      return c0s[1][res0][o];
    else
      return c0a[o];
  };
  int off[NL];
  bool okx[NL];
#pragma unroll
  for (int j = 0; j < NL; ++j)
  {
    const int e = i + j * T0;
    const int64_t gx = g0 - K + e;
    okx[j] = e < XW && gx >= 0 && gx < m;
    off[j] = okx[j] ? static_cast<int>(gx) : 0;
  }
  const bool col_ok = g0 + i < m;
  const int NPL = static_cast<int>(re - rs) + 2 * K;  // input rows rs-K .. re+K-1
  auto issue = [&](int it) {
    const int64_t q = rs - K + it;
    const bool rin = q >= 0 && q < m;
    const T *xr = x + (rin ? q : 0) * m;
    T *dst = Xs[it % 3];
#pragma unroll
    for (int j = 0; j < NL; ++j)
    {
      const int e = i + j * T0;
      if (e < XW)
        op_cp_async(dst + e, xr + off[j], rin && okx[j]);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  T acc[W];
#pragma unroll
  for (int o = 0; o < W; ++o)
    acc[o] = T(0);
  issue(0);
  if (NPL > 1)
  {
    issue(1);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  }
  else
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int base = 0; base < NPL; base += K)
  {
#pragma unroll
    for (int u = 0; u < K; ++u)
    {
      const int it = base + u;  // uniform across the CTA
      if (it >= NPL)
        break;
      if (it + 2 < NPL)
        issue(it + 2);
      const T *xs = Xs[it % 3] + i;
      T zm0 = cm0(0) * xs[0], za0 = ca0(0) * xs[0], zm1 = cm0(1) * xs[1], za1 = ca0(1) * xs[1];
#pragma unroll
      for (int o = 2; o < W; o += 2)
      {
        zm0 = fma(cm0(o), xs[o], zm0);
        za0 = fma(ca0(o), xs[o], za0);
        if (o + 1 < W)
        {
          zm1 = fma(cm0(o + 1), xs[o + 1], zm1);
          za1 = fma(ca0(o + 1), xs[o + 1], za1);
        }
      }
      const T zm = zm0 + zm1, za = za0 + za1;
      const int64_t p_out = rs - 2 * K + it;
      T bval = T(0);
      if constexpr (RESID)
      {
        if (it >= 2 * K && p_out < re && col_ok)
          bval = __ldg(b + p_out * m + g0 + i);
      }
      if (it + 2 < NPL)
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      // dir 1: output row p = q - K + jo has lattice residue (u + 1 + jo) mod K
      // and band offset 2K - jo; rows of residue != 0 couple only their cell
#pragma unroll
      for (int jo = 0; jo < W; ++jo)
      {
        const int res = (u + 1 + jo) % K;
        const int o = 2 * K - jo;
        if (res != 0 && (o < K - res || o > 2 * K - res))
          continue;
        acc[jo] = fma(B.A[res][o], zm, acc[jo]);
        acc[jo] = fma(B.M[res][o], za, acc[jo]);
      }
      if (it >= 2 * K && p_out < re && col_ok)
      {
        const int64_t idx = p_out * m + g0 + i;
        if constexpr (RESID)
          y[idx] = bval - acc[0];
        else
          y[idx] = acc[0];
      }
#pragma unroll
      for (int jo = 0; jo < W - 1; ++jo)
        acc[jo] = acc[jo + 1];
      acc[W - 1] = T(0);
    }
  }
}

template <int D, int K, typename T>
void launch_level_op(const BandMats<T, K> &B, const T *x, const T *b, T *y, int64_t m,
                     int sm_count, cudaStream_t s, int64_t zbeg = 0, int64_t zend = -1)
{
  if (zend < 0)
    zend = m;
  if (zend <= zbeg)
    return;
  if constexpr (D == 3)
  {
#if PMG_OP_XB
    if constexpr (K == 4)
    {
      using CX = Op3XbCfg<K, T>;
      const unsigned gxx = static_cast<unsigned>((m + 1 + CX::XC - 1) / CX::XC);
      const unsigned gyx = static_cast<unsigned>((m + CX::TY - 1) / CX::TY);
      const int64_t z0x = (zbeg / K) * K, spanx = zend - z0x;
      int64_t nzx = (static_cast<int64_t>(sm_count) * 2 + gxx * gyx - 1) / (gxx * gyx);
      int64_t zcx = std::max<int64_t>((spanx + nzx - 1) / nzx, 4 * K);
      zcx = (zcx + K - 1) / K * K;
      const unsigned gzx = static_cast<unsigned>((spanx + zcx - 1) / zcx);
      auto kx = b ? level_op3d_xb_kernel<K, T, true> : level_op3d_xb_kernel<K, T, false>;
      static unsigned xmask[2] = {0, 0};
      if (first_on_device(xmask[b ? 1 : 0]))
      {
        check_cuda(cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(CX::SMEM)),
                   "cudaFuncSetAttribute(level_op3d_xb)");
        check_cuda(cudaFuncSetAttribute(kx, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                   "cudaFuncSetAttribute(level_op3d_xb carveout)");
      }
      pdl_launch(kx, dim3(gxx, gyx, gzx), CX::NT, CX::SMEM, s, B, x, b, y, m, static_cast<int>(zcx), zbeg, zend);
      check_launch("level_op3d_xb_kernel");
      return;
    }
#endif
#if PMG_OP_CB
    if constexpr (K <= 2)
    {
      using CB = Op3CbCfg<K, T>;
      static const int cb_ctas = [] {
        const char *e = std::getenv("PMG_OP_CB_CTAS");
        return e ? std::max(1, std::atoi(e)) : 4;
      }();
      static const int cb_zmin = [] {
        const char *e = std::getenv("PMG_OP_CB_ZMIN");
        return e ? std::max(1, std::atoi(e)) : 2;
      }();
      const unsigned gxc = static_cast<unsigned>((m + 1 + CB::XC - 1) / CB::XC);
      const unsigned gyc = static_cast<unsigned>((m + 1 + CB::YC - 1) / CB::YC);
      const int64_t z0c = (zbeg / K) * K, spanc = zend - z0c;
      const int64_t nzc = (static_cast<int64_t>(sm_count) * cb_ctas + gxc * gyc - 1) / (gxc * gyc);
      int64_t zcc = std::max<int64_t>((spanc + nzc - 1) / nzc, cb_zmin * K);
      zcc = (zcc + K - 1) / K * K;
      const unsigned gzc = static_cast<unsigned>((spanc + zcc - 1) / zcc);
      auto kc = b ? level_op3d_cb_kernel<K, T, true> : level_op3d_cb_kernel<K, T, false>;
      static unsigned cmask[2] = {0, 0};
      if (first_on_device(cmask[b ? 1 : 0]))
      {
        check_cuda(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(CB::SMEM)),
                   "cudaFuncSetAttribute(level_op3d_cb)");
        check_cuda(cudaFuncSetAttribute(kc, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                   "cudaFuncSetAttribute(level_op3d_cb carveout)");
      }
      pdl_launch(kc, dim3(gxc, gyc, gzc), CB::NT, CB::SMEM, s, B, x, b, y, m, static_cast<int>(zcc), zbeg, zend);
      check_launch("level_op3d_cb_kernel");
      return;
    }
#endif
    using C = Op3Cfg<K, T>;
    constexpr size_t smem = C::SMEM;
    const unsigned gx = static_cast<unsigned>((m + C::TX - 1) / C::TX);
    const unsigned gy = static_cast<unsigned>((m + C::TY - 1) / C::TY);
    // z chunk (a multiple of K): enough CTAs for ~6 per SM, >= 4k planes to
    // bound the recomputed halo
    const int64_t z0 = (zbeg / K) * K, span = zend - z0;
    static const int zmin_k = [] {
      const char *e = std::getenv("PMG_OP_ZMIN");
      return e ? std::max(1, std::atoi(e)) : 4;
    }();
    static const int ctas = [] {
      const char *e = std::getenv("PMG_OP_CTAS");
      return e ? std::max(1, std::atoi(e)) : 6;
    }();
    int64_t want = static_cast<int64_t>(sm_count) * ctas;
    int64_t nz = (want + gx * gy - 1) / (gx * gy);
    int64_t zchunk = (span + nz - 1) / nz;
    zchunk = std::max<int64_t>(zchunk, zmin_k * K);
    zchunk = (zchunk + K - 1) / K * K;
    const unsigned gz = static_cast<unsigned>((span + zchunk - 1) / zchunk);
    auto kern = b ? level_op3d_kernel<K, T, true> : level_op3d_kernel<K, T, false>;
    static unsigned attr_mask[2] = {0, 0};
    if (first_on_device(attr_mask[b ? 1 : 0]))
    {
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)),
                 "cudaFuncSetAttribute(level_op3d)");
      check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                 "cudaFuncSetAttribute(level_op3d carveout)");
    }
    pdl_launch(kern, dim3(gx, gy, gz), C::NT, smem, s, B, x, b, y, m, static_cast<int>(zchunk), zbeg, zend);
    check_launch("level_op3d_kernel");
  }
  else
  {
    const unsigned gx = static_cast<unsigned>((m + 127) / 128);
    int64_t want = static_cast<int64_t>(sm_count) * 16;
    int64_t ny = (want + gx - 1) / gx;
    int64_t rchunk = (m + ny - 1) / ny;
    rchunk = std::max<int64_t>(rchunk, std::min<int64_t>(m, 4 * K));
    rchunk = ((rchunk + K - 1) / K) * K;  // chunks start on multiples of K
    const unsigned gy = static_cast<unsigned>((m + rchunk - 1) / rchunk);
    auto kern = b ? level_op2d_kernel<K, T, true> : level_op2d_kernel<K, T, false>;
    pdl_launch(kern, dim3(gx, gy), 128, 0, s, B, x, b, y, m, static_cast<int>(rchunk));
    check_launch("level_op2d_kernel");
  }
}

}  // namespace pmgb
