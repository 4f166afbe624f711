// Plane-streaming vertex-patch smoother kernel (3D, low degree) for sm_100a.
//
// Same arithmetic contract as vp_smooth_kernel (smoother_impl.cuh): the
// reference's fused / boundary per-patch body (smoother.cpp:109-148), i.e.
// r = b^I - (A-bar x)^I (fastdiag.cpp:199-233), v = (S x S x S) diag(1/sum lambda)
// (S x S x S)^T r (fastdiag.cpp:164-192), x^I += v (patches.cpp:97-121).
//
// The line kernel round-trips every one of its 7 contraction stages through
// shared memory. At low degree the closure is small enough for a thread to
// keep a whole 2D slice of the patch in registers, so this kernel needs only
// four shared-memory passes per patch:
//
//   P1  thread (p, j2):  closure plane j2 (NC x NC, staged by cp.async) ->
//       dir-0 contractions row by row, dir-1 contractions accumulated in
//       registers (even-odd row pairs)  ->  wMM, wS  (2 x NI x NI)  -> W
//   P2  thread (p, i0, i1):  dir-2 line of wMM / wS -> r = b - (A2 wMM + M2 wS)
//       (b preloaded into registers at kernel entry) -> S^T along dir 2 -> W
//   P3  thread (p, c2):  eigen plane c2 (NI x NI) -> S^T dir 1, S^T dir 0,
//       x 1/(lambda sums), S dir 0, S dir 1, all in registers -> W
//   P4  thread (p, i0, i1):  S along dir 2, x^I = x^I_old (staged closure) + v
//
// Shared memory per patch: the closure U (NC^3) and one work array W
// (2 NC NI^2 + pad; P2..P4 overwrite it in place, each thread only touching
// the (i0, i1) column / c2 plane it alone reads). The pads are chosen by an
// offline bank-conflict search (tools/bank_search.py) over the four phases'
// access patterns.
#pragma once

#include "smoother_impl.cuh"

namespace pmgb
{

template <int K, typename T>
struct PlaneCfg
{
  static constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  static constexpr bool F64 = sizeof(T) == 8;
  // patches per CTA: PB consecutive patches of one x-row of the colour
#ifndef PMG_PLANE_PB2
#define PMG_PLANE_PB2 16
#endif
  static constexpr int PB = K == 1 ? 64 : (K == 2 ? PMG_PLANE_PB2 : 8);
  // threads: the widest phase (P1: NC per patch, P2/P4: NI^2 per patch)
  static constexpr int LANES = (NC > NI * NI ? NC : NI * NI);
  static constexpr int NT = ((PB * LANES + 31) / 32) * 32;
  static constexpr int RX = 2 * K * PB + 1;  // x extent of the CTA's closure union
  // shared-memory layout (words), tools/bank_search.py:
  //   U[p][t2][t1][t0] at p UW + t2 SU2 + t1 SU1 + t0
  //   W: wMM[j][q] at p WW + j SJ + q, wS at p WW + SW + j SJ + q (q = i0 + NI i1);
  //      the eigen-space tensor overwrites wMM in place
  static constexpr int L64[4][6] = {{0}, {57, 5, 19, 19, 1, 3}, {135, 5, 27, 105, 10, 50}, {357, 7, 51, 377, 26, 182}};
  static constexpr int L32[4][6] = {{0}, {39, 3, 13, 41, 3, 16}, {145, 5, 29, 105, 10, 50}, {371, 7, 53, 409, 28, 197}};
  static constexpr int UW = F64 ? L64[K][0] : L32[K][0];
  static constexpr int SU1 = F64 ? L64[K][1] : L32[K][1];
  static constexpr int SU2 = F64 ? L64[K][2] : L32[K][2];
  static constexpr int WW = F64 ? L64[K][3] : L32[K][3];
  static constexpr int SJ = F64 ? L64[K][4] : L32[K][4];
  static constexpr int SW = F64 ? L64[K][5] : L32[K][5];
  static_assert(SU1 >= NC && SU2 >= NC * SU1 && UW >= NC * SU2, "U layout");
  static_assert(SJ >= NI * NI && SW >= NC * SJ && WW >= SW + NC * SJ, "W layout");
  static constexpr size_t SMEM = static_cast<size_t>(PB) * (UW + WW) * sizeof(T);
};

#ifndef PMG_PLANE_SADDR
#define PMG_PLANE_SADDR 1
#endif
#ifndef PMG_PLANE_ZMASK
#define PMG_PLANE_ZMASK 1
#endif
#ifndef PMG_PLANE_MINB
#define PMG_PLANE_MINB 5
#endif

// One tile = PB consecutive patches j0 = bx PB + p (p < PB) of an x-row
// (j1, j2) of a colour: the closures of its patches form one contiguous box of
// x rows, so the global -> shared copy runs along x. The caller synchronises
// before (shared memory reuse) and after (the tile's x^I stores are complete).
template <int K, typename T, int MODE>
__device__ __forceinline__ void plane_tile(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a, int bx, int j1,
                                           int j2, unsigned char *smem_raw, bool PRO = false)
{
  using C = PlaneCfg<K, T>;
  constexpr int NC = C::NC, NI = C::NI, PB = C::PB, NT = C::NT, RX = C::RX;
  constexpr int UW = C::UW, SU1 = C::SU1, SU2 = C::SU2, WW = C::WW, SJ = C::SJ, SW = C::SW;
  constexpr int NI2 = NI * NI;
  constexpr int HO = K > 1 ? K - 1 : 1;
  T *U = reinterpret_cast<T *>(smem_raw);  // [PB][UW]  closures
  T *W = U + PB * UW;                      // [PB][WW]  work

  const int tid = threadIdx.x;
  const int64_t m = a.m;
  const int64_t m2 = m * m;
  const int npv = min(PB, a.np[0] - bx * PB);  // valid patches
  // closure-local t = 0 per direction: g_a = k (v_a - 1) - 1, v_a = 2 j_a + vb_a
  // (patches.cpp:71); patch p of the tile starts at G0 + 2K p along x
  const int G0 = K * (2 * bx * PB + a.vb[0] - 1) - 1;
  const int G1 = K * (2 * j1 + a.vb[1] - 1) - 1;
  const int64_t G2g = static_cast<int64_t>(K) * (2 * static_cast<int64_t>(j2) + a.vb[2] - 1) - 1;
  const int64_t G2 = G2g - a.zoff;  // local plane of t2 = 0 in x / b

  // ---- b^I of this thread's (p, i0, i1) column, straight into registers (b is
  //      not written by the smoother: with a.b_ready before the PDL wait) ----
  const int p24 = tid / NI2;
  const int rr24 = tid - p24 * NI2;
  const int i0_24 = rr24 % NI, i1_24 = rr24 / NI;
  const bool act24 = tid < PB * NI2 && p24 < npv;
  const int64_t col24 = (G2 + 1) * m2 + static_cast<int64_t>(G1 + 1 + i1_24) * m + (G0 + 2 * K * p24 + 1 + i0_24);
  T bcol[NI];
  if (act24)
  {
#pragma unroll
    for (int i = 0; i < NI; ++i)
      bcol[i] = PRO ? __ldcg(a.b + col24 + i * m2)  // before the PDL wait: L2 only, no L1 line
                    : __ldg(a.b + col24 + i * m2);  // that predates the wait can be hit
  }

  if (PRO)
    pdl_prologue();

  // ---- stage the closures of x, zero-filled outside the domain (gather,
  //      patches.cpp:72-79). Thread -> union column (X, t1), then a fixed-stride
  //      walk over the NC planes t2; lanes run along contiguous x. Column X
  //      belongs to patch X / 2K (t0 = X mod 2K) and, on a shared vertex column,
  //      also to patch X / 2K - 1 (t0 = 2K). ------------------------------------
#if PMG_PLANE_ZMASK
  // z validity of the NC closure planes: CTA-uniform, one bit per plane
  unsigned zmask = 0;
#pragma unroll
  for (int t2 = 0; t2 < NC; ++t2)
    zmask |= (static_cast<uint64_t>(G2g + t2) < static_cast<uint64_t>(a.mz) ? 1u : 0u) << t2;
#endif
#pragma unroll 1
  for (int line = tid; line < NC * RX; line += NT)
  {
    const int t1 = line / RX;
    const int X = line - t1 * RX;
    const int gx = G0 + X, gy = G1 + t1;
    const bool okxy = static_cast<unsigned>(gx) < static_cast<unsigned>(m) &&
                      static_cast<unsigned>(gy) < static_cast<unsigned>(m);
    const int pq = X / (2 * K);
    const int p = pq < PB ? pq : PB - 1;
    const int t0 = X - 2 * K * p;
    const bool dup = t0 == 0 && p > 0;
    T *dst = U + p * UW + t1 * SU1 + t0;
    T *dst2 = U + (p - 1) * UW + t1 * SU1 + 2 * K;
#if PMG_PLANE_SADDR
    // shared-window addresses once per line; per plane a compile-time stride
    const unsigned sd = smem_addr(dst), sd2 = smem_addr(dst2);
#endif
    const T *src = a.x + G2 * m2 + static_cast<int64_t>(gy) * m + gx;
#pragma unroll
    for (int t2 = 0; t2 < NC; ++t2)
    {
#if PMG_PLANE_ZMASK
      const bool ok = okxy && ((zmask >> t2) & 1u);
#else
      const bool ok = okxy && static_cast<uint64_t>(G2g + t2) < static_cast<uint64_t>(a.mz);
#endif
      bool ok1 = ok;
      if constexpr (MODE == MODE_BOUNDARY)  // never reads x^I (smoother.cpp:128-148)
        ok1 = ok && !(t0 >= 1 && t0 <= NC - 2 && t1 >= 1 && t1 <= NC - 2 && t2 >= 1 && t2 <= NC - 2);
      const T *sp = ok ? src + t2 * m2 : a.x;
#if PMG_PLANE_SADDR
      cp_async_sa<T>(sd + static_cast<unsigned>(sizeof(T) * SU2 * t2), sp, ok1);
      if (dup)
        cp_async_sa<T>(sd2 + static_cast<unsigned>(sizeof(T) * SU2 * t2), sp, ok);
#else
      cp_async_elem(dst + t2 * SU2, sp, ok1);
      if (dup)
        cp_async_elem(dst2 + t2 * SU2, sp, ok);
#endif
    }
  }
  cp_async_commit();

  cp_async_wait_all();
  __syncthreads();

  // ---- P1: thread (p, j2): dir 0 + dir 1 of closure plane j2 ------------------
  if (tid < PB * NC)
  {
    const int p = tid / NC;
    const int j2 = tid - p * NC;
    const T *up = U + p * UW + j2 * SU2;
    // even / odd accumulators of wMM = M1 zM and wS = A1 zM + M1 zA over j1
    T Em[K][NI], Es[K][NI], Om[HO][NI], Os[HO][NI];
#pragma unroll
    for (int jj = 0; jj <= K; ++jj)
    {
      T ra[NC], rae[K + 1], rao[K];
      T zma[NI], zaa[NI];
#pragma unroll
      for (int t = 0; t < NC; ++t)
        ra[t] = up[jj * SU1 + t];
      eo_split<NC>(ra, rae, rao);
      eo_rows<K>(P.Me, P.Mo, rae, rao, zma);
      eo_rows<K>(P.Ae, P.Ao, rae, rao, zaa);
      if (jj < K)
      {
        T rb[NC], rbe[K + 1], rbo[K];
        T zmb[NI], zab[NI];
#pragma unroll
        for (int t = 0; t < NC; ++t)
          rb[t] = up[(NC - 1 - jj) * SU1 + t];
        eo_split<NC>(rb, rbe, rbo);
        eo_rows<K>(P.Me, P.Mo, rbe, rbo, zmb);
        eo_rows<K>(P.Ae, P.Ao, rbe, rbo, zab);
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
          const T zme = zma[i] + zmb[i], zmo = zma[i] - zmb[i];
          const T zae = zaa[i] + zab[i], zao = zaa[i] - zab[i];
#pragma unroll
          for (int h = 0; h < K; ++h)
          {
            if (jj == 0)
            {
              Em[h][i] = P.Me[h][jj] * zme;
              Es[h][i] = fma(P.Ae[h][jj], zme, P.Me[h][jj] * zae);
            }
            else
            {
              Em[h][i] = fma(P.Me[h][jj], zme, Em[h][i]);
              Es[h][i] = fma(P.Ae[h][jj], zme, fma(P.Me[h][jj], zae, Es[h][i]));
            }
          }
#pragma unroll
          for (int h = 0; h < K - 1; ++h)
          {
            if (jj == 0)
            {
              Om[h][i] = P.Mo[h][jj] * zmo;
              Os[h][i] = fma(P.Ao[h][jj], zmo, P.Mo[h][jj] * zao);
            }
            else
            {
              Om[h][i] = fma(P.Mo[h][jj], zmo, Om[h][i]);
              Os[h][i] = fma(P.Ao[h][jj], zmo, fma(P.Mo[h][jj], zao, Os[h][i]));
            }
          }
        }
      }
      else  // middle row j1 = K: even part only
      {
#pragma unroll
        for (int i = 0; i < NI; ++i)
        {
#pragma unroll
          for (int h = 0; h < K; ++h)
          {
            Em[h][i] = fma(P.Me[h][K], zma[i], Em[h][i]);
            Es[h][i] = fma(P.Ae[h][K], zma[i], fma(P.Me[h][K], zaa[i], Es[h][i]));
          }
        }
      }
    }
    // wMM[j2][i1][i0], wS[j2][i1][i0]
    T *wp = W + p * WW + j2 * SJ;
#pragma unroll
    for (int h = 0; h < K; ++h)
    {
#pragma unroll
      for (int i = 0; i < NI; ++i)
      {
        if (h < K - 1)
        {
          wp[h * NI + i] = Em[h][i] + Om[h][i];
          wp[(NI - 1 - h) * NI + i] = Em[h][i] - Om[h][i];
          wp[SW + h * NI + i] = Es[h][i] + Os[h][i];
          wp[SW + (NI - 1 - h) * NI + i] = Es[h][i] - Os[h][i];
        }
        else
        {
          wp[h * NI + i] = Em[h][i];
          wp[SW + h * NI + i] = Es[h][i];
        }
      }
    }
  }
  __syncthreads();

  // ---- P2: thread (p, i0, i1): r = b - (A2 wMM + M2 wS); yhat = S^T r (dir 2) --
  if (act24)
  {
    T *wl = W + p24 * WW + rr24;
    T wm[NC], ws[NC];
#pragma unroll
    for (int t = 0; t < NC; ++t)
    {
      wm[t] = wl[t * SJ];
      ws[t] = wl[SW + t * SJ];
    }
    T wme[K + 1], wmo[K], wse[K + 1], wso[K];
    eo_split<NC>(wm, wme, wmo);
    eo_split<NC>(ws, wse, wso);
    T acc[NI], r[NI], y[NI];
    eo_rows2<K>(P.Ae, P.Ao, wme, wmo, P.Me, P.Mo, wse, wso, acc);
#pragma unroll
    for (int i = 0; i < NI; ++i)
      r[i] = bcol[i] - acc[i];
    eo_st<K>(P.Se, P.So, r, y);
#pragma unroll
    for (int c = 0; c < NI; ++c)
      wl[c * SJ] = y[c];
  }
  __syncthreads();

  // ---- P3: thread (p, c2): eigen plane c2 in registers ----------------------------
  if (tid < PB * NI && tid / NI < npv)
  {
    const int p = tid / NI;
    const int c2 = tid - p * NI;
    T *wq = W + p * WW + c2 * SJ;
    T v[NI][NI];  // [i1][i0] -> [c1][c0] -> back
#pragma unroll
    for (int i1 = 0; i1 < NI; ++i1)
#pragma unroll
      for (int i0 = 0; i0 < NI; ++i0)
        v[i1][i0] = wq[i1 * NI + i0];
    // S^T along dir 1 (columns)
#pragma unroll
    for (int i0 = 0; i0 < NI; ++i0)
    {
      T col[NI], yh[NI];
#pragma unroll
      for (int i1 = 0; i1 < NI; ++i1)
        col[i1] = v[i1][i0];
      eo_st<K>(P.Se, P.So, col, yh);
#pragma unroll
      for (int c1 = 0; c1 < NI; ++c1)
        v[c1][i0] = yh[c1];
    }
    // S^T along dir 0, scale, S along dir 0 (rows)
    const T *inv = a.inv + NI2 * c2;
#pragma unroll
    for (int c1 = 0; c1 < NI; ++c1)
    {
      T yh[NI];
      eo_st<K>(P.Se, P.So, v[c1], yh);
#pragma unroll
      for (int c0 = 0; c0 < NI; ++c0)
        yh[c0] *= __ldg(inv + c1 * NI + c0);
      eo_s<K>(P.Se, P.So, yh, v[c1]);
    }
    // S along dir 1 (columns), store
#pragma unroll
    for (int i0 = 0; i0 < NI; ++i0)
    {
      T col[NI], ph[NI];
#pragma unroll
      for (int c1 = 0; c1 < NI; ++c1)
        col[c1] = v[c1][i0];
      eo_s<K>(P.Se, P.So, col, ph);
#pragma unroll
      for (int i1 = 0; i1 < NI; ++i1)
        wq[i1 * NI + i0] = ph[i1];
    }
  }
  __syncthreads();

  // ---- P4: thread (p, i0, i1): S along dir 2, x^I update --------------------------
  if (act24)
  {
    const T *wl = W + p24 * WW + rr24;
    T yh[NI], v[NI];
#pragma unroll
    for (int c = 0; c < NI; ++c)
      yh[c] = wl[c * SJ];
    eo_s<K>(P.Se, P.So, yh, v);
    T *xp = a.x + col24;
    const T *xo = U + p24 * UW + SU2 + (1 + i1_24) * SU1 + (1 + i0_24);
#pragma unroll
    for (int i = 0; i < NI; ++i)
    {
      if constexpr (MODE == MODE_BOUNDARY)
        xp[i * m2] = v[i];
      else
        xp[i * m2] = xo[SU2 * i] + v[i];  // x^I_old is in the staged closure
    }
  }
}

// one launch per colour: grid = (ceil(np0 / PB), np1, np2)
template <int K, typename T, int MODE>
__global__ void __launch_bounds__(PlaneCfg<K, T>::NT, K == 2 ? PMG_PLANE_MINB : 1)
    vp_smooth_plane_kernel(const __grid_constant__ PatchMatsEO<T, K> P, const __grid_constant__ ColorArgs<T> a)
{
  // b_ready: the b^I loads are issued before the dependency wait (inside)
  if (!a.b_ready)
    pdl_prologue();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  plane_tile<K, T, MODE>(P, a, blockIdx.x, blockIdx.y, blockIdx.z, smem_raw, a.b_ready != 0);
}

// ---------------------------------------------------------------------------
// All 2^d colours of one smoothing step in ONE persistent launch.
//
// Work items are the tiles of all colours in the reference's order (colour
// major, smoother.cpp:54-59; within a colour z-plane major), handed out by an
// atomic ticket. Tile (c, v2) may start once every tile of every earlier
// colour c' < c on vertex planes v2-1 .. v2+1 has finished: those are exactly
// the patches whose interiors intersect its closure (|v' - v| <= 1 per
// direction, patches.cpp:71/114), so every read sees the reference's values
// and no write overtakes an earlier colour's read. Per-patch arithmetic is
// the per-colour kernel's, so results are bitwise identical to 2^d launches.
// Deadlock-free without co-residency: an item only waits for items with
// smaller tickets, all of which are held by running CTAs. The last CTA to
// finish resets the counters, so the launch can be replayed from a graph.
// ---------------------------------------------------------------------------

__device__ __forceinline__ int ld_acquire(const int *p)
{
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int K, typename T, int MODE>
__global__ void __launch_bounds__(PlaneCfg<K, T>::NT, K == 2 ? PMG_PLANE_MINB : 1)
    vp_sweep_plane_kernel(const __grid_constant__ PatchMatsEO<T, K> P, const __grid_constant__ SweepArgs<T> s)
{
  pdl_prologue();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int item_s;
  int *ticket = s.sync, *exitc = s.sync + 1, *done = s.sync + 2;
  const int total = s.start[s.ncolors];
  if (threadIdx.x == 0)
    item_s = atomicAdd(ticket, 1);
  __syncthreads();
  int item = item_s;
  while (item < total)
  {
    int c = 0;
    while (item >= s.start[c + 1])
      ++c;
    const ColorArgs<T> &a = s.c[c];
    const int l = item - s.start[c];
    const int bx = l % s.ntx[c];
    const int rest = l / s.ntx[c];
    const int j1 = rest % a.np[1];
    const int j2 = rest / a.np[1];
    const int v2 = 2 * j2 + a.vb[2];
    // wait for the earlier colours' tiles on planes v2-1 .. v2+1 (warp 0)
    if (threadIdx.x < 32 && c > 0)
    {
      const int q = threadIdx.x;  // q = 3 c' + dw
      const int cp = q / 3, w = v2 - 1 + q % 3;
      if (cp < c)
      {
        const ColorArgs<T> &b = s.c[cp];
        const int first = b.vb[2], last = b.vb[2] + 2 * (b.np[2] - 1);
        if (b.np[2] > 0 && w >= first && w <= last && ((w - first) & 1) == 0)
        {
          const int need = s.ntx[cp] * b.np[1];
          const int *ctr = done + cp * s.nv + w;
          while (ld_acquire(ctr) < need)
            __nanosleep(40);
        }
      }
      __syncwarp();
    }
    __syncthreads();
    int next = 0;
    if (threadIdx.x == 0)
      next = atomicAdd(ticket, 1);  // claimed early: latency overlaps the tile
    plane_tile<K, T, MODE>(P, a, bx, j1, j2, smem_raw);
    __syncthreads();  // all x^I stores of the tile issued; shared memory free
    if (threadIdx.x == 0)
    {
      __threadfence();
      atomicAdd(done + c * s.nv + v2, 1);
      item_s = next;
    }
    __syncthreads();
    item = item_s;
  }
  // last CTA out resets the counters for the next launch
  __shared__ int last_s;
  if (threadIdx.x == 0)
  {
    __threadfence();
    last_s = atomicAdd(exitc, 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (last_s)
  {
    for (int i = threadIdx.x; i < 2 + s.ncolors * s.nv; i += blockDim.x)
      s.sync[i] = 0;
  }
}

template <int K, typename T, int MODE>
void launch_vp_smooth_plane(const PatchMatsEO<T, K> &P, const ColorArgs<T> &a, cudaStream_t s)
{
  using C = PlaneCfg<K, T>;
  static unsigned attr_mask = 0;
  if (first_on_device(attr_mask))
  {
    check_cuda(cudaFuncSetAttribute(vp_smooth_plane_kernel<K, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(C::SMEM)),
               "cudaFuncSetAttribute(plane smoother)");
    check_cuda(cudaFuncSetAttribute(vp_smooth_plane_kernel<K, T, MODE>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100),
               "cudaFuncSetAttribute(plane smoother carveout)");
  }
  if (a.total == 0)
    return;
  const dim3 grid((a.np[0] + C::PB - 1) / C::PB, a.np[1], a.np[2]);
  pdl_launch(vp_smooth_plane_kernel<K, T, MODE>, grid, C::NT, C::SMEM, s, P, a);
  check_launch("vp_smooth_plane_kernel");
}

template <int K, typename T, int MODE>
void launch_vp_sweep_plane(const PatchMatsEO<T, K> &P, const SweepArgs<T> &sw, int sm_count, cudaStream_t s)
{
  using C = PlaneCfg<K, T>;
  static unsigned attr_mask = 0;
  static int occ[32] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (first_on_device(attr_mask))
  {
    check_cuda(cudaFuncSetAttribute(vp_sweep_plane_kernel<K, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(C::SMEM)),
               "cudaFuncSetAttribute(plane sweep)");
    check_cuda(cudaFuncSetAttribute(vp_sweep_plane_kernel<K, T, MODE>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100),
               "cudaFuncSetAttribute(plane sweep carveout)");
    int o = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, vp_sweep_plane_kernel<K, T, MODE>, C::NT, C::SMEM),
               "occupancy(plane sweep)");
    occ[dev & 31] = o > 0 ? o : 1;
  }
  const int total = sw.start[sw.ncolors];
  if (total == 0)
    return;
  const int grid = std::min(total, occ[dev & 31] * sm_count);
  pdl_launch(vp_sweep_plane_kernel<K, T, MODE>, grid, C::NT, C::SMEM, s, P, sw);
  check_launch("vp_sweep_plane_kernel");
}

}  // namespace pmgb
