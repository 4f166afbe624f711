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
  // patches per CTA
  static constexpr int PB = K == 1 ? 64 : (K == 2 ? 16 : 8);
  // threads: the widest phase (P1: NC per patch, P2/P4: NI^2 per patch)
  static constexpr int LANES = (NC > NI * NI ? NC : NI * NI);
  static constexpr int NT = ((PB * LANES + 31) / 32) * 32;
  static constexpr int UW = NC * NC * NC;  // odd: plane reads are conflict-free
  // W stride per patch (words): 2 NC NI^2 + pad (tools/bank_search.py)
  static constexpr int WPAD64[4] = {0, 1, 3, 1};
  static constexpr int WPAD32[4] = {0, 1, 3, 1};
  static constexpr int WW = 2 * NC * NI * NI + (F64 ? WPAD64[K] : WPAD32[K]);
  static constexpr size_t SMEM = static_cast<size_t>(PB) * (UW + WW) * sizeof(T);
};

template <int K, typename T, int MODE>
__global__ void __launch_bounds__(PlaneCfg<K, T>::NT)
    vp_smooth_plane_kernel(const __grid_constant__ PatchMatsEO<T, K> P, const __grid_constant__ ColorArgs<T> a)
{
  using C = PlaneCfg<K, T>;
  constexpr int NC = C::NC, NI = C::NI, PB = C::PB, NT = C::NT, UW = C::UW, WW = C::WW;
  constexpr int NI2 = NI * NI, NC2 = NC * NC;
  constexpr int HO = K > 1 ? K - 1 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *U = reinterpret_cast<T *>(smem_raw);  // [PB][UW]  closure, [t2][t1][t0]
  T *W = U + PB * UW;                      // [PB][WW]  work
  __shared__ int org[PB][3];

  const int tid = threadIdx.x;
  const int64_t m = a.m;
  const int64_t m2 = m * m;
  const int p0 = blockIdx.x * PB;

  if (tid < PB)
  {
    const int gp = p0 + tid;
    int g0 = -(1 << 30), g1 = -(1 << 30), g2 = -(1 << 30);  // invalid patch: every load masked
    if (gp < a.total)
    {
      const int j0 = gp % a.np[0];
      const int rest = gp / a.np[0];
      const int j1 = rest % a.np[1];
      const int j2 = rest / a.np[1];
      // closure-local t = 0 per direction: g_a = k (v_a - 1) - 1 (patches.cpp:71)
      g0 = K * (2 * j0 + a.vb[0] - 1) - 1;
      g1 = K * (2 * j1 + a.vb[1] - 1) - 1;
      g2 = K * (2 * j2 + a.vb[2] - 1) - 1 - static_cast<int>(a.zoff);
    }
    org[tid][0] = g0;
    org[tid][1] = g1;
    org[tid][2] = g2;
  }
  __syncthreads();

  // ---- stage the closure of x: one z-line (NC elements) per thread-iteration,
  //      zero-filled outside the domain (gather, patches.cpp:72-79) ----------
  {
    for (int line = tid; line < PB * NC2; line += NT)
    {
      const int p = line / NC2;
      const int rr = line - p * NC2;
      const int t0 = rr % NC, t1 = rr / NC;
      const int y0 = org[p][0] + t0, y1 = org[p][1] + t1, z0 = org[p][2];
      const bool inplane = static_cast<uint32_t>(y0) < static_cast<uint32_t>(m) &&
                           static_cast<uint32_t>(y1) < static_cast<uint32_t>(m);
      const T *src = a.x + static_cast<int64_t>(y1) * m + y0;
      T *dst = U + p * UW + rr;
#pragma unroll
      for (int t = 0; t < NC; ++t)
      {
        const int64_t zl = static_cast<int64_t>(z0) + t;  // local plane; global = zl + zoff
        bool ok = inplane && static_cast<uint64_t>(zl + a.zoff) < static_cast<uint64_t>(a.mz);
        if constexpr (MODE == MODE_BOUNDARY)
        {
          const bool inner = t0 >= 1 && t0 <= NC - 2 && t1 >= 1 && t1 <= NC - 2 && t >= 1 && t <= NC - 2;
          ok = ok && !inner;
        }
        cp_async_elem(dst + NC2 * t, ok ? src + zl * m2 : a.x, ok);
      }
    }
    cp_async_commit();
  }

  // ---- b^I of this thread's (p, i0, i1) column, straight into registers ------
  const int p24 = tid / NI2;
  const int rr24 = tid - p24 * NI2;
  const int i0_24 = rr24 % NI, i1_24 = rr24 / NI;
  const bool act24 = tid < PB * NI2 && p0 + p24 < a.total;
  T bcol[NI];
  if (act24)
  {
    const T *bp = a.b + (static_cast<int64_t>(org[p24][2]) + 1) * m2 +
                  static_cast<int64_t>(org[p24][1] + 1 + i1_24) * m + (org[p24][0] + 1 + i0_24);
#pragma unroll
    for (int i = 0; i < NI; ++i)
      bcol[i] = __ldg(bp + i * m2);
  }

  cp_async_wait_all();
  __syncthreads();

  // ---- P1: thread (p, j2): dir 0 + dir 1 of closure plane j2 ------------------
  if (tid < PB * NC)
  {
    const int p = tid / NC;
    const int j2 = tid - p * NC;
    const T *up = U + p * UW + j2 * NC2;
    // even / odd accumulators of wMM = M1 zM and wS = A1 zM + M1 zA over j1
    T Em[K][NI], Es[K][NI], Om[HO][NI], Os[HO][NI];
#pragma unroll
    for (int jj = 0; jj <= K; ++jj)
    {
      T ra[NC], rae[K + 1], rao[K];
      T zma[NI], zaa[NI];
#pragma unroll
      for (int t = 0; t < NC; ++t)
        ra[t] = up[jj * NC + t];
      eo_split<NC>(ra, rae, rao);
      eo_rows<K>(P.Me, P.Mo, rae, rao, zma);
      eo_rows<K>(P.Ae, P.Ao, rae, rao, zaa);
      if (jj < K)
      {
        T rb[NC], rbe[K + 1], rbo[K];
        T zmb[NI], zab[NI];
#pragma unroll
        for (int t = 0; t < NC; ++t)
          rb[t] = up[(NC - 1 - jj) * NC + t];
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
              Em[h][i] = (P.Me[h][jj]) * zme;
              Es[h][i] = fma((P.Ae[h][jj]), zme, (P.Me[h][jj]) * zae);
            }
            else
            {
              Em[h][i] = fma((P.Me[h][jj]), zme, Em[h][i]);
              Es[h][i] = fma((P.Ae[h][jj]), zme, fma((P.Me[h][jj]), zae, Es[h][i]));
            }
          }
#pragma unroll
          for (int h = 0; h < K - 1; ++h)
          {
            if (jj == 0)
            {
              Om[h][i] = (P.Mo[h][jj]) * zmo;
              Os[h][i] = fma((P.Ao[h][jj]), zmo, (P.Mo[h][jj]) * zao);
            }
            else
            {
              Om[h][i] = fma((P.Mo[h][jj]), zmo, Om[h][i]);
              Os[h][i] = fma((P.Ao[h][jj]), zmo, fma((P.Mo[h][jj]), zao, Os[h][i]));
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
    // W[p]: wMM at [j2][i1][i0], wS at NC NI^2 + [j2][i1][i0]
    T *wp = W + p * WW + j2 * NI2;
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
          wp[NC * NI2 + h * NI + i] = Es[h][i] + Os[h][i];
          wp[NC * NI2 + (NI - 1 - h) * NI + i] = Es[h][i] - Os[h][i];
        }
        else
        {
          wp[h * NI + i] = Em[h][i];
          wp[NC * NI2 + h * NI + i] = Es[h][i];
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
      wm[t] = wl[t * NI2];
      ws[t] = wl[NC * NI2 + t * NI2];
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
      wl[c * NI2] = y[c];
  }
  __syncthreads();

  // ---- P3: thread (p, c2): eigen plane c2 in registers ----------------------------
  if (tid < PB * NI)
  {
    const int p = tid / NI;
    const int c2 = tid - p * NI;
    T *wq = W + p * WW + c2 * NI2;
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
      yh[c] = wl[c * NI2];
    eo_s<K>(P.Se, P.So, yh, v);
    T *xp = a.x + (static_cast<int64_t>(org[p24][2]) + 1) * m2 +
            static_cast<int64_t>(org[p24][1] + 1 + i1_24) * m + (org[p24][0] + 1 + i0_24);
    const T *xo = U + p24 * UW + (1 + i0_24) + NC * (1 + i1_24) + NC2;
#pragma unroll
    for (int i = 0; i < NI; ++i)
    {
      if constexpr (MODE == MODE_BOUNDARY)
        xp[i * m2] = v[i];
      else
        xp[i * m2] = xo[NC2 * i] + v[i];  // x^I_old is in the staged closure
    }
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
  const int grid = (a.total + C::PB - 1) / C::PB;
  if (grid == 0)
    return;
  vp_smooth_plane_kernel<K, T, MODE><<<grid, C::NT, C::SMEM, s>>>(P, a);
  check_launch("vp_smooth_plane_kernel");
}

}  // namespace pmgb
