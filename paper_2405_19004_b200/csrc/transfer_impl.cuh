// Grid transfers for sm_100a: prolongation (exact polynomial embedding) and
// restriction (its transpose).
//
// Replaces prolongate<T> (/root/reference/proj/src/multigrid.cpp:71-160) and
// restrict_vector<T> (multigrid.cpp:162-248). The reference loops over coarse
// cells, contracts the (2k+1)x(k+1) embedding matrix P in every direction and
// writes each fine node from the one cell that owns it (r_a >= 1 per
// direction), resp. scatter-adds the transpose. Because ownership is decided
// per direction, the level transfer is exactly P_g (x) P_g (x) P_g with a
// banded 1D factor P_g (fine lattice p, owner cell c = (p-1) div 2k,
// r = p - 2ck in [1,2k], coarse lattice q = ck + t). The device applies it as
// d gather-style 1D passes (no atomics, deterministic): thread per output
// node, <= k+1 (prolongation) or <= 4k (restriction) terms each; the last
// prolongation pass can accumulate into x (the V-cycle's x += P x_c).
#pragma once

#include "common.cuh"

namespace pmgb
{

// out has extents ext_out (dir 0 fastest); along DIR the input has mc coarse
// nodes and the output mf = 2 mc + 1 fine nodes.
template <int K, typename T, int DIR, bool ACC>
__global__ void __launch_bounds__(256)
    prolong_pass_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ in,
                        T *__restrict__ out, int64_t e0, int64_t e1, int64_t e2, int64_t mc)
{
  pdl_prologue();
  __shared__ T Ps[2 * K + 1][K + 1];
  for (int e = threadIdx.x; e < (2 * K + 1) * (K + 1); e += blockDim.x)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  __syncthreads();
  const int64_t total = e0 * e1 * e2;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    int64_t i0 = idx % e0;
    int64_t rest = idx / e0;
    int64_t i1 = rest % e1;
    int64_t i2 = rest / e1;
    const int64_t ifine = DIR == 0 ? i0 : (DIR == 1 ? i1 : i2);
    const int64_t p = ifine + 1;  // fine lattice
    const int64_t c = (p - 1) / (2 * K);
    const int r = static_cast<int>(p - 2 * c * K);
    // input strides (input extent along DIR is mc)
    const int64_t ie0 = DIR == 0 ? mc : e0;
    const int64_t ie1 = DIR == 1 ? mc : e1;
    int64_t base, stride;
    if (DIR == 0)
    {
      base = (i2 * ie1 + i1) * ie0;
      stride = 1;
    }
    else if (DIR == 1)
    {
      base = i2 * ie1 * ie0 + i0;
      stride = ie0;
    }
    else
    {
      base = i1 * ie0 + i0;
      stride = ie0 * ie1;
    }
    T s = T(0);
#pragma unroll
    for (int t = 0; t <= K; ++t)
    {
      const int64_t q = c * K + t;  // coarse lattice
      if (q >= 1 && q <= mc)
        s = fma(Ps[r][t], in[base + (q - 1) * stride], s);
    }
    if constexpr (ACC)
      out[idx] += s;
    else
      out[idx] = s;
  }
}

// out has extents ext_out; along DIR the output has mc coarse nodes and the
// input mf fine nodes.
template <int K, typename T, int DIR>
__global__ void __launch_bounds__(256)
    restrict_pass_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ in,
                         T *__restrict__ out, int64_t e0, int64_t e1, int64_t e2, int64_t mf)
{
  pdl_prologue();
  __shared__ T Ps[2 * K + 1][K + 1];
  for (int e = threadIdx.x; e < (2 * K + 1) * (K + 1); e += blockDim.x)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  __syncthreads();
  const int64_t total = e0 * e1 * e2;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
  {
    int64_t i0 = idx % e0;
    int64_t rest = idx / e0;
    int64_t i1 = rest % e1;
    int64_t i2 = rest / e1;
    const int64_t icoarse = DIR == 0 ? i0 : (DIR == 1 ? i1 : i2);
    const int64_t q = icoarse + 1;  // coarse lattice
    const int64_t ie0 = DIR == 0 ? mf : e0;
    const int64_t ie1 = DIR == 1 ? mf : e1;
    int64_t base, stride;
    if (DIR == 0)
    {
      base = (i2 * ie1 + i1) * ie0;
      stride = 1;
    }
    else if (DIR == 1)
    {
      base = i2 * ie1 * ie0 + i0;
      stride = ie0;
    }
    else
    {
      base = i1 * ie0 + i0;
      stride = ie0 * ie1;
    }
    T s = T(0);
    const int tq = static_cast<int>(q % K);
    // cells containing coarse node q: (c, t) with q = cK + t, 0 <= t <= K
    const int ncell = (tq == 0) ? 2 : 1;
    for (int h = 0; h < ncell; ++h)
    {
      const int64_t c = (tq == 0) ? (q / K - 1 + h) : (q / K);
      const int t = (tq == 0) ? (h == 0 ? K : 0) : tq;
#pragma unroll
      for (int r = 1; r <= 2 * K; ++r)
      {
        const int64_t p = 2 * c * K + r;  // fine lattice
        if (p >= 1 && p <= mf)
          s = fma(Ps[r][t], in[base + (p - 1) * stride], s);
      }
    }
    out[idx] = s;
  }
}

inline unsigned pass_grid(int64_t total, int sm_count)
{
  const int64_t blocks = (total + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(blocks, static_cast<int64_t>(sm_count) * 32)));
}

// xf (+)= P xc. tA, tB: scratch of at least mf*mf*mc (3D) / mf*mc (2D).
template <int D, int K, typename T>
void launch_prolongate(const ProlMats<T, K> &P, const T *xc, T *xf, bool acc, int64_t mc,
                       T *tA, T *tB, int sm_count, cudaStream_t s)
{
  const int64_t mf = 2 * mc + 1;
  if constexpr (D == 2)
  {
    pdl_launch(prolong_pass_kernel<K, T, 0, false>, pass_grid(mf * mc, sm_count), 256, 0, s, P, xc, tA, mf, mc, 1, mc);
    check_launch("prolong_pass0");
    if (acc)
      pdl_launch(prolong_pass_kernel<K, T, 1, true>, pass_grid(mf * mf, sm_count), 256, 0, s, P, tA, xf, mf, mf, 1, mc);
    else
      pdl_launch(prolong_pass_kernel<K, T, 1, false>, pass_grid(mf * mf, sm_count), 256, 0, s, P, tA, xf, mf, mf, 1, mc);
    check_launch("prolong_pass1");
  }
  else
  {
    pdl_launch(prolong_pass_kernel<K, T, 0, false>, pass_grid(mf * mc * mc, sm_count), 256, 0, s, P, xc, tA, mf, mc, mc, mc);
    check_launch("prolong_pass0");
    pdl_launch(prolong_pass_kernel<K, T, 1, false>, pass_grid(mf * mf * mc, sm_count), 256, 0, s, P, tA, tB, mf, mf, mc, mc);
    check_launch("prolong_pass1");
    if (acc)
      pdl_launch(prolong_pass_kernel<K, T, 2, true>, pass_grid(mf * mf * mf, sm_count), 256, 0, s, P, tB, xf, mf, mf, mf, mc);
    else
      pdl_launch(prolong_pass_kernel<K, T, 2, false>, pass_grid(mf * mf * mf, sm_count), 256, 0, s, P, tB, xf, mf, mf, mf, mc);
    check_launch("prolong_pass2");
  }
}

template <int D, int K, typename T>
void launch_restrict(const ProlMats<T, K> &P, const T *rf, T *rc, int64_t mc, T *tA, T *tB,
                     int sm_count, cudaStream_t s)
{
  const int64_t mf = 2 * mc + 1;
  if constexpr (D == 2)
  {
    pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc * mf, sm_count), 256, 0, s, P, rf, tA, mc, mf, 1, mf);
    check_launch("restrict_pass0");
    pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc * mc, sm_count), 256, 0, s, P, tA, rc, mc, mc, 1, mf);
    check_launch("restrict_pass1");
  }
  else
  {
    pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc * mf * mf, sm_count), 256, 0, s, P, rf, tA, mc, mf, mf, mf);
    check_launch("restrict_pass0");
    pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc * mc * mf, sm_count), 256, 0, s, P, tA, tB, mc, mc, mf, mf);
    check_launch("restrict_pass1");
    pdl_launch(restrict_pass_kernel<K, T, 2>, pass_grid(mc * mc * mc, sm_count), 256, 0, s, P, tB, rc, mc, mc, mc, mf);
    check_launch("restrict_pass2");
  }
}

}  // namespace pmgb
