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

#include <cstdlib>

#include "common.cuh"

namespace pmgb
{

// Both pass kernels: block (32, 8), grid (ceil(e0/32), ceil(e1/8), e2), so an
// output node's (i0, i1, i2) comes from the launch geometry (no 64-bit
// division); along DIR the input index is strided, the other two are shared
// with the output.
template <int DIR>
__device__ __forceinline__ void pass_index(int64_t e0, int64_t e1, int64_t ie0, int64_t ie1, int64_t i0,
                                           int64_t i1, int64_t i2, int64_t &base, int64_t &stride)
{
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
}

// out has extents (e0, e1, e2) (dir 0 fastest); along DIR the input has mc
// coarse nodes and the output mf = 2 mc + 1 fine nodes.
template <int K, typename T, int DIR, bool ACC>
__global__ void __launch_bounds__(256)
    prolong_pass_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ in,
                        T *__restrict__ out, int64_t e0, int64_t e1, int64_t e2, int64_t mc, int64_t z0)
{
  pdl_prologue();
  __shared__ T Ps[2 * K + 1][K + 1];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < (2 * K + 1) * (K + 1); e += 256)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  __syncthreads();
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  const int64_t i1 = static_cast<int64_t>(blockIdx.y) * 8 + threadIdx.y;
  const int64_t i2 = z0 + blockIdx.z;  // global plane (slab callers shift their bases)
  if (i0 >= e0 || i1 >= e1)
    return;
  const int64_t ifine = DIR == 0 ? i0 : (DIR == 1 ? i1 : i2);
  const int p = static_cast<int>(ifine) + 1;  // fine lattice
  const int c = (p - 1) / (2 * K);            // owner cell
  const int r = p - 2 * c * K;
  int64_t base, stride;
  pass_index<DIR>(e0, e1, DIR == 0 ? mc : e0, DIR == 1 ? mc : e1, i0, i1, i2, base, stride);
  T s = T(0);
#pragma unroll
  for (int t = 0; t <= K; ++t)
  {
    const int q = c * K + t;  // coarse lattice
    if (q >= 1 && q <= mc)
      s = fma(Ps[r][t], __ldg(in + base + (q - 1) * stride), s);
  }
  const int64_t idx = (i2 * e1 + i1) * e0 + i0;
  if constexpr (ACC)
    out[idx] += s;
  else
    out[idx] = s;
}

// out has extents (e0, e1, e2); along DIR the output has mc coarse nodes and
// the input mf fine nodes.
template <int K, typename T, int DIR>
__global__ void __launch_bounds__(256)
    restrict_pass_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ in,
                         T *__restrict__ out, int64_t e0, int64_t e1, int64_t e2, int64_t mf, int64_t z0)
{
  pdl_prologue();
  __shared__ T Ps[2 * K + 1][K + 1];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < (2 * K + 1) * (K + 1); e += 256)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  __syncthreads();
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  const int64_t i1 = static_cast<int64_t>(blockIdx.y) * 8 + threadIdx.y;
  const int64_t i2 = z0 + blockIdx.z;  // global plane (slab callers shift their bases)
  if (i0 >= e0 || i1 >= e1)
    return;
  const int64_t icoarse = DIR == 0 ? i0 : (DIR == 1 ? i1 : i2);
  const int q = static_cast<int>(icoarse) + 1;  // coarse lattice
  int64_t base, stride;
  pass_index<DIR>(e0, e1, DIR == 0 ? mf : e0, DIR == 1 ? mf : e1, i0, i1, i2, base, stride);
  T s = T(0);
  const int tq = q % K;
  // cells containing coarse node q: (c, t) with q = cK + t, 0 <= t <= K; the
  // transpose of the prolongation gathers their 2K owned fine nodes
  const int c1 = q / K;
#pragma unroll
  for (int h = 0; h < 2; ++h)
  {
    if (h == 1 && tq != 0)
      break;
    const int c = (tq == 0) ? (c1 - 1 + h) : c1;
    const int t = (tq == 0) ? (h == 0 ? K : 0) : tq;
#pragma unroll
    for (int r = 1; r <= 2 * K; ++r)
    {
      const int p = 2 * c * K + r;  // fine lattice
      if (p >= 1 && p <= mf)
        s = fma(Ps[r][t], __ldg(in + base + (p - 1) * stride), s);
    }
  }
  out[(i2 * e1 + i1) * e0 + i0] = s;
}

// PMG_TRANSFER_PASSES=1 selects the separate 1D passes (A/B measurement)
inline bool use_fused_transfer()
{
  static const bool v = [] {
    const char *e = std::getenv("PMG_TRANSFER_PASSES");
    return !(e && e[0] == '1');
  }();
  return v;
}

inline dim3 pass_grid(int64_t e0, int64_t e1, int64_t e2)
{
  return dim3(static_cast<unsigned>((e0 + 31) / 32), static_cast<unsigned>((e1 + 7) / 8),
              static_cast<unsigned>(e2));
}

// ---------------------------------------------------------------------------
// 3D prolongation in one kernel: CTA = CX x CY coarse cells of one z-cell.
// The (K+1)^3-node coarse block of the tile is staged once, then the three 1D
// passes run in shared memory (x: coarse rows -> fine columns, y, z) and the
// (2K)^3 fine nodes per cell are written (or accumulated) straight to x_f.
// Traffic: x_c once (+ halo) and x_f once (twice with accumulation), against
// ~3.5 N words for the three separate passes; one launch instead of three.
// ---------------------------------------------------------------------------
template <int K>
struct Prol3Cfg
{
  static constexpr int CX = (32 / (2 * K)) > 0 ? 32 / (2 * K) : 1;
  static constexpr int CY = (8 / (2 * K)) > 0 ? 8 / (2 * K) : 1;
  static constexpr int FX = 2 * K * CX, FY = 2 * K * CY;
  static constexpr int QX = CX * K + 1, QY = CY * K + 1, QZ = K + 1;  // coarse block
  static constexpr int NT = 32 * FY;
};

template <int K, typename T, bool ACC>
__global__ void __launch_bounds__(Prol3Cfg<K>::NT)
    prolong3d_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ xc, T *__restrict__ xf,
                     int mc, int nc, int cz0, int f0, int f1)
{
  pdl_prologue();
  using C = Prol3Cfg<K>;
  constexpr int CX = C::CX, CY = C::CY, FX = C::FX, FY = C::FY, QX = C::QX, QY = C::QY, QZ = C::QZ, NT = C::NT;
  __shared__ T Ps[2 * K + 1][K + 1];
  __shared__ T Cs[QZ][QY][QX];
  __shared__ T T1[QZ][QY][FX];
  __shared__ T T2[QZ][FY][FX];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < (2 * K + 1) * (K + 1); e += NT)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  const int cx0 = blockIdx.x * CX, cy0 = blockIdx.y * CY, cz = cz0 + blockIdx.z;
  const int64_t mc2 = static_cast<int64_t>(mc) * mc;
  // coarse lattice q = cK + t (1-based; 0 and mc+1 are the Dirichlet boundary)
  for (int e = tid; e < QZ * QY * QX; e += NT)
  {
    const int iz = e / (QY * QX), r = e - iz * (QY * QX);
    const int iy = r / QX, ix = r - iy * QX;
    const int qx = cx0 * K + ix, qy = cy0 * K + iy, qz = cz * K + iz;
    T v = T(0);
    if (qx >= 1 && qx <= mc && qy >= 1 && qy <= mc && qz >= 1 && qz <= mc)
      v = __ldg(xc + (qz - 1) * mc2 + static_cast<int64_t>(qy - 1) * mc + (qx - 1));
    Cs[iz][iy][ix] = v;
  }
  __syncthreads();
  // x: fine column fx = 2K c + (r - 1) of the tile, r = 1..2K
  for (int e = tid; e < QZ * QY * FX; e += NT)
  {
    const int iz = e / (QY * FX), rr = e - iz * (QY * FX);
    const int iy = rr / FX, fx = rr - iy * FX;
    const int c = fx / (2 * K), r = fx - 2 * K * c + 1;
    T s = T(0);
#pragma unroll
    for (int t = 0; t <= K; ++t)
      s = fma(Ps[r][t], Cs[iz][iy][c * K + t], s);
    T1[iz][iy][fx] = s;
  }
  __syncthreads();
  const int fx = threadIdx.x, fy = threadIdx.y;
  const int cyl = fy / (2 * K), ry = fy - 2 * K * cyl + 1;
  if (fx < FX)
  {
#pragma unroll
    for (int iz = 0; iz < QZ; ++iz)
    {
      T s = T(0);
#pragma unroll
      for (int t = 0; t <= K; ++t)
        s = fma(Ps[ry][t], T1[iz][cyl * K + t][fx], s);
      T2[iz][fy][fx] = s;
    }
  }
  __syncthreads();
  if (fx >= FX)
    return;
  const int cxl = fx / (2 * K), rx = fx - 2 * K * cxl + 1;
  const int mf = 2 * mc + 1;
  const int px = 2 * (cx0 + cxl) * K + rx, py = 2 * (cy0 + cyl) * K + ry;  // fine lattice
  if (cx0 + cxl >= nc || cy0 + cyl >= nc || px > mf || py > mf)
    return;
  const int64_t mf2 = static_cast<int64_t>(mf) * mf;
  T *o = xf + static_cast<int64_t>(py - 1) * mf + (px - 1);
#pragma unroll
  for (int rz = 1; rz <= 2 * K; ++rz)
  {
    const int pz = 2 * cz * K + rz;
    if (pz > mf || pz - 1 >= f1)
      break;
    if (pz - 1 < f0)  // fine planes [f0, f1) only (0-based)
      continue;
    T s = T(0);
#pragma unroll
    for (int t = 0; t <= K; ++t)
      s = fma(Ps[rz][t], T2[t][fy][fx], s);
    T *op = o + (pz - 1) * mf2;
    if constexpr (ACC)
      *op += s;
    else
      *op = s;
  }
}

template <int D, int K, typename T>
void launch_prolongate(const ProlMats<T, K> &P, const T *xc, T *xf, bool acc, int64_t mc,
                       T *tA, T *tB, int sm_count, cudaStream_t s)
{
  const int64_t mf = 2 * mc + 1;
  if constexpr (D == 2)
  {
    pdl_launch(prolong_pass_kernel<K, T, 0, false>, pass_grid(mf, mc, 1), dim3(32, 8), 0, s, P, xc, tA, mf, mc, 1, mc, int64_t(0));
    check_launch("prolong_pass0");
    if (acc)
      pdl_launch(prolong_pass_kernel<K, T, 1, true>, pass_grid(mf, mf, 1), dim3(32, 8), 0, s, P, tA, xf, mf, mf, 1, mc, int64_t(0));
    else
      pdl_launch(prolong_pass_kernel<K, T, 1, false>, pass_grid(mf, mf, 1), dim3(32, 8), 0, s, P, tA, xf, mf, mf, 1, mc, int64_t(0));
    check_launch("prolong_pass1");
  }
  else if (use_fused_transfer())
  {
    using C = Prol3Cfg<K>;
    const int nc = static_cast<int>((mc + 1) / K);  // coarse cells per direction
    const dim3 grid((nc + C::CX - 1) / C::CX, (nc + C::CY - 1) / C::CY, nc);
    if (acc)
      pdl_launch(prolong3d_kernel<K, T, true>, grid, dim3(32, C::FY), 0, s, P, xc, xf, static_cast<int>(mc), nc, 0,
                 0, static_cast<int>(mf));
    else
      pdl_launch(prolong3d_kernel<K, T, false>, grid, dim3(32, C::FY), 0, s, P, xc, xf, static_cast<int>(mc), nc, 0,
                 0, static_cast<int>(mf));
    check_launch("prolong3d_kernel");
  }
  else
  {
    pdl_launch(prolong_pass_kernel<K, T, 0, false>, pass_grid(mf, mc, mc), dim3(32, 8), 0, s, P, xc, tA, mf, mc, mc, mc, int64_t(0));
    check_launch("prolong_pass0");
    pdl_launch(prolong_pass_kernel<K, T, 1, false>, pass_grid(mf, mf, mc), dim3(32, 8), 0, s, P, tA, tB, mf, mf, mc, mc, int64_t(0));
    check_launch("prolong_pass1");
    if (acc)
      pdl_launch(prolong_pass_kernel<K, T, 2, true>, pass_grid(mf, mf, mf), dim3(32, 8), 0, s, P, tB, xf, mf, mf, mf, mc, int64_t(0));
    else
      pdl_launch(prolong_pass_kernel<K, T, 2, false>, pass_grid(mf, mf, mf), dim3(32, 8), 0, s, P, tB, xf, mf, mf, mf, mc, int64_t(0));
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
    pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc, mf, 1), dim3(32, 8), 0, s, P, rf, tA, mc, mf, 1, mf, int64_t(0));
    check_launch("restrict_pass0");
    pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc, mc, 1), dim3(32, 8), 0, s, P, tA, rc, mc, mc, 1, mf, int64_t(0));
    check_launch("restrict_pass1");
  }
  else
  {
    pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc, mf, mf), dim3(32, 8), 0, s, P, rf, tA, mc, mf, mf, mf, int64_t(0));
    check_launch("restrict_pass0");
    pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc, mc, mf), dim3(32, 8), 0, s, P, tA, tB, mc, mc, mf, mf, int64_t(0));
    check_launch("restrict_pass1");
    pdl_launch(restrict_pass_kernel<K, T, 2>, pass_grid(mc, mc, mc), dim3(32, 8), 0, s, P, tB, rc, mc, mc, mc, mf, int64_t(0));
    check_launch("restrict_pass2");
  }
}

// ---------------------------------------------------------------------------
// Slab versions (3D; the slab domain decomposition's V-cycle, dd.py). All
// pointers are GLOBAL-plane bases (the caller shifts its local array by its
// first plane); only the planes the requested outputs depend on are touched.
// ---------------------------------------------------------------------------

// fine planes [f0, f1) (0-based) (+)= P x_c
template <int K, typename T>
void launch_prolongate_slab(const ProlMats<T, K> &P, const T *xc, T *xf, bool acc, int64_t mc, int64_t f0,
                            int64_t f1, cudaStream_t s)
{
  using C = Prol3Cfg<K>;
  if (f1 <= f0)
    return;
  const int nc = static_cast<int>((mc + 1) / K);
  const int cz0 = static_cast<int>(f0 / (2 * K)), cz1 = static_cast<int>((f1 - 1) / (2 * K));
  const dim3 grid((nc + C::CX - 1) / C::CX, (nc + C::CY - 1) / C::CY, cz1 - cz0 + 1);
  if (acc)
    pdl_launch(prolong3d_kernel<K, T, true>, grid, dim3(32, C::FY), 0, s, P, xc, xf, static_cast<int>(mc), nc, cz0,
               static_cast<int>(f0), static_cast<int>(f1));
  else
    pdl_launch(prolong3d_kernel<K, T, false>, grid, dim3(32, C::FY), 0, s, P, xc, xf, static_cast<int>(mc), nc, cz0,
               static_cast<int>(f0), static_cast<int>(f1));
  check_launch("prolong3d_kernel(slab)");
}

// fine planes the coarse planes [q0, q1) depend on: [pz0, pz1) (0-based)
inline void restrict_slab_fine_range(int K, int64_t mc, int64_t q0, int64_t q1, int64_t &pz0, int64_t &pz1)
{
  const int64_t mf = 2 * mc + 1;
  const int64_t cmin = std::max<int64_t>(0, (q0 + 1 - K + K - 1) / K);  // ceil((Q0 - K) / K), Q0 = q0 + 1
  const int64_t cmax = q1 / K;                                           // floor(Q1 / K), Q1 = q1
  pz0 = 2 * cmin * K;
  pz1 = std::min<int64_t>(2 * cmax * K + 2 * K, mf);
}

// coarse planes [q0, q1) = R r_f; tA, tB: local scratch of mc*mf and mc*mc
// per fine plane of [pz0, pz1) (global-plane bases, as the vectors)
template <int K, typename T>
void launch_restrict_slab(const ProlMats<T, K> &P, const T *rf, T *rc, int64_t mc, int64_t q0, int64_t q1, T *tA,
                          T *tB, cudaStream_t s)
{
  if (q1 <= q0)
    return;
  const int64_t mf = 2 * mc + 1;
  int64_t pz0, pz1;
  restrict_slab_fine_range(K, mc, q0, q1, pz0, pz1);
  pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc, mf, pz1 - pz0), dim3(32, 8), 0, s, P, rf, tA, mc, mf, mf,
             mf, pz0);
  check_launch("restrict_pass0(slab)");
  pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc, mc, pz1 - pz0), dim3(32, 8), 0, s, P, tA, tB, mc, mc, mf,
             mf, pz0);
  check_launch("restrict_pass1(slab)");
  pdl_launch(restrict_pass_kernel<K, T, 2>, pass_grid(mc, mc, q1 - q0), dim3(32, 8), 0, s, P, tB, rc, mc, mc, mc,
             mf, q0);
  check_launch("restrict_pass2(slab)");
}

}  // namespace pmgb
