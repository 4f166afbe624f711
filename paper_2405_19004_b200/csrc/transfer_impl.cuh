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
                         T *__restrict__ out, int64_t e0, int64_t e1, int64_t e2, int64_t mf, int64_t z0,
                         T *__restrict__ zero = nullptr)
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
  if (zero)
    zero[(i2 * e1 + i1) * e0 + i0] = T(0);
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
  if constexpr (K <= 4)
  {
    // all 2K accumulated outputs of the column: issue every load of x_f before
    // the first store, so the read latencies overlap instead of serialising
    // the read-modify-write chain (profiles/r01/ab_prolong3d_batch.txt: k = 1,
    // 2 and f32 -14..18%, k = 3 -7%; for k >= 5 the 2K live values cost more)
    T old[2 * K];
    bool okz[2 * K];
#pragma unroll
    for (int rz = 1; rz <= 2 * K; ++rz)
    {
      const int pz = 2 * cz * K + rz;
      okz[rz - 1] = pz <= mf && pz - 1 >= f0 && pz - 1 < f1;  // fine planes [f0, f1) only (0-based)
      if constexpr (ACC)
        old[rz - 1] = okz[rz - 1] ? o[(pz - 1) * mf2] : T(0);
    }
#pragma unroll
    for (int rz = 1; rz <= 2 * K; ++rz)
    {
      if (!okz[rz - 1])
        continue;
      T v = T(0);
#pragma unroll
      for (int t = 0; t <= K; ++t)
        v = fma(Ps[rz][t], T2[t][fy][fx], v);
      o[(2 * cz * K + rz - 1) * mf2] = ACC ? old[rz - 1] + v : v;
    }
  }
  else
  {
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
}

// ---------------------------------------------------------------------------
// 3D restriction in one kernel, marching along z. CTA = OX x OY coarse
// columns (whole coarse cells: OX = CX K, OY = CY K) and a range of coarse
// z-nodes [Qa, Qb]. Per fine z-plane of the cells that touch the range: the
// (WY x WX) fine window of the tile (2K (C+1) fine nodes per direction, the
// cells c0 .. c0 + C) is staged by cp.async (double-buffered, zero-filled
// past the last fine node), the x pass gathers it to R1[WY][OX] in shared
// memory, the y pass gives each thread its (qx, qy) value v of this plane,
// and the z pass accumulates P[r][t] v into K + 1 registers of the current
// cell. Nodes t = 1 .. K-1 of a cell are complete when the cell ends; node
// t = 0 adds the t = K partial of the previous cell (a register carry).
// Traffic: r_f once (+ the x / y window halo and one extra cell per z chunk)
// and R r_f once, against ~2.6 N words for the three 1D passes; one launch
// instead of three. `zero` (optional) is cleared at the output nodes (the
// V-cycle's x_c = 0).
// ---------------------------------------------------------------------------
template <int K>
struct Rest3Cfg
{
  static constexpr int CX = 32 / K, CY = (8 / K) >= 2 ? 8 / K : (K <= 5 ? 2 : 1);  // static smem <= 48 KB
  static constexpr int OX = CX * K, OY = CY * K;
  static constexpr int WX = 2 * K * (CX + 1), WY = 2 * K * (CY + 1), WN = WX * WY;
  static constexpr int NT = 32 * OY;
  static constexpr int NLOAD = (WN + NT - 1) / NT;
};

template <typename T>
__device__ __forceinline__ void tr_cp_async(T *smem, const T *gmem, bool valid)
{
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 4 : 0)
                 : "memory");
}

// coarse node Q (1-based, one direction) = sum over its <= 2 cells (c, t) and
// r = 1..2K of P[r][t] fine(2cK + r); here as offsets into a window whose
// first fine node is 2 c0 K + 1
template <int K, typename T, typename F>
__device__ __forceinline__ T rest_gather_1d(const T (*Ps)[K + 1], int Q, int c0, F &&fine)
{
  const int tq = Q % K, c1 = Q / K;
  T s = T(0);
#pragma unroll
  for (int h = 0; h < 2; ++h)
  {
    if (h == 1 && tq != 0)
      break;
    const int c = tq == 0 ? c1 - 1 + h : c1;
    const int t = tq == 0 ? (h == 0 ? K : 0) : tq;
    const int base = 2 * (c - c0) * K - 1;  // window offset of fine node r = 0 of cell c
#pragma unroll
    for (int r = 1; r <= 2 * K; ++r)
      s = fma(Ps[r][t], fine(base + r), s);
  }
  return s;
}

template <int K, typename T>
__global__ void __launch_bounds__(Rest3Cfg<K>::NT)
    restrict3d_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ rf, T *__restrict__ rc,
                      T *__restrict__ zero, int mc, int q0, int q1, int nodes_per_chunk)
{
  using C = Rest3Cfg<K>;
  constexpr int CX = C::CX, CY = C::CY, OX = C::OX, OY = C::OY, WX = C::WX, WY = C::WY, NT = C::NT;
  __shared__ T Ps[2 * K + 1][K + 1];
  // fine-plane ring: NB - 1 planes in flight (static shared memory <= 48 KB)
  constexpr int NB = (3 * WY * WX + WY * OX) * sizeof(T) <= 46 * 1024 ? 3 : 2;
  __shared__ __align__(16) T F[NB][WY * WX];
  __shared__ T R1[WY][OX];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  for (int e = tid; e < (2 * K + 1) * (K + 1); e += NT)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  const int mf = 2 * mc + 1;
  const int cx0 = blockIdx.x * CX, cy0 = blockIdx.y * CY;
  // owned coarse z-nodes [Qa, Qb] (1-based) and the cells that touch them
  const int Qa = q0 + 1 + blockIdx.z * nodes_per_chunk;
  const int Qb = min(q1, q0 + (static_cast<int>(blockIdx.z) + 1) * nodes_per_chunk);
  const int c_lo = (Qa % K == 0) ? Qa / K - 1 : Qa / K, c_hi = Qb / K;
  // fixed staging slots of this thread: window element -> (fy, fx)
  const int64_t mf2 = static_cast<int64_t>(mf) * mf;
  const T *wbase = rf + static_cast<int64_t>(2 * cy0 * K) * mf + 2 * cx0 * K;  // fine (p_y, p_x) = window (0, 0)
  int goff[C::NLOAD];
  bool gok[C::NLOAD];
#pragma unroll
  for (int j = 0; j < C::NLOAD; ++j)
  {
    const int e = tid + j * NT;
    const int fy = e / WX, fx = e - fy * WX;
    gok[j] = e < C::WN && 2 * cy0 * K + fy < mf && 2 * cx0 * K + fx < mf;
    goff[j] = gok[j] ? fy * mf + fx : 0;
  }
  auto stage = [&](int buf, int pz) {  // pz: 0-based fine plane
    const bool zok = pz < mf;
    const T *src = wbase + (zok ? static_cast<int64_t>(pz) * mf2 : 0);
#pragma unroll
    for (int j = 0; j < C::NLOAD; ++j)
    {
      const int e = tid + j * NT;
      if (e < C::WN)
        tr_cp_async(&F[buf][e], src + goff[j], gok[j] && zok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  pdl_prologue();
  __syncthreads();  // Ps
  const int qx = cx0 * K + 1 + tx, qy = cy0 * K + 1 + ty;  // this thread's coarse column (y pass)
  const bool own = tx < OX && qx <= mc && qy <= mc;
  T acc[K + 1], carry = T(0);
  const int nplanes = (c_hi - c_lo + 1) * 2 * K;
  stage(0, 2 * c_lo * K);
  if (NB == 3 && nplanes > 1)
    stage(1, 2 * c_lo * K + 1);
  int s = 0;
  for (int cz = c_lo; cz <= c_hi; ++cz)
  {
#pragma unroll
    for (int t = 0; t <= K; ++t)
      acc[t] = T(0);
#pragma unroll
    for (int r = 1; r <= 2 * K; ++r, ++s)
    {
      const int buf = s % NB;
      // plane s landed (with NB = 3, plane s + 1 may stay in flight)
      if (NB == 3 && s + 1 < nplanes)
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      // plane s + NB - 1 (0-based fine plane 2 c_lo K + s + NB - 1) into the
      // buffer of plane s - 1, whose x pass ended before the previous barrier
      if (s + NB - 1 < nplanes)
        stage((s + NB - 1) % NB, 2 * c_lo * K + s + NB - 1);
      // x pass: R1[fy][ox] for the tile's coarse x nodes
      if (tx < OX)
      {
        const T *Fb = F[buf];
        for (int fy = ty; fy < WY; fy += OY)
          R1[fy][tx] = rest_gather_1d<K, T>(Ps, qx, cx0, [&](int o) { return Fb[fy * WX + o]; });
      }
      __syncthreads();
      if (tx < OX)
      {
        const T v = rest_gather_1d<K, T>(Ps, qy, cy0, [&](int o) { return R1[o][tx]; });
#pragma unroll
        for (int t = 0; t <= K; ++t)
          acc[t] = fma(Ps[r][t], v, acc[t]);
      }
    }
    // complete nodes: cz K (t = 0, plus the previous cell's t = K) and cz K + t
    if (own)
    {
      T *o = rc + static_cast<int64_t>(qy - 1) * mc + (qx - 1);
      T *z = zero ? zero + static_cast<int64_t>(qy - 1) * mc + (qx - 1) : nullptr;
#pragma unroll
      for (int t = 0; t < K; ++t)
      {
        const int Q = cz * K + t;
        if (Q >= Qa && Q <= Qb && Q >= 1)
        {
          const int64_t off = static_cast<int64_t>(Q - 1) * mc * mc;
          o[off] = t == 0 ? carry + acc[0] : acc[t];
          if (z)
            z[off] = T(0);
        }
      }
    }
    carry = acc[K];
  }
}

// ---------------------------------------------------------------------------
// 2D transfers in one kernel each (the 2D analogues of prolong3d_kernel and
// one plane of restrict3d_kernel): a CTA stages its block of the input
// (coarse cells + 1 node, resp. the fine window of its coarse nodes), runs
// the x pass into shared memory and the y pass straight to the output.
// Traffic: prolongation x_c once + x_f read/write (vs + 2 x mf mc scratch),
// restriction r_f once with the window halo (vs + 2 x mc mf scratch).
// ---------------------------------------------------------------------------
#ifndef PMG_PROL2_RY
#define PMG_PROL2_RY 4
#endif
template <int K>
struct Prol2Cfg
{
  static constexpr int CX = (32 / (2 * K)) > 0 ? 32 / (2 * K) : 1;
  static constexpr int CYT = (16 / (2 * K)) > 0 ? 16 / (2 * K) : 1;  // cells per thread row block
  static constexpr int RY = PMG_PROL2_RY;                              // row blocks per thread
  static constexpr int CY = CYT * RY;                                  // cells per CTA along y
  static constexpr int FX = 2 * K * CX, FY = 2 * K * CYT;              // threads: 32 x FY
  static constexpr int QX = CX * K + 1, QY = CY * K + 1;
  static constexpr int NT = 32 * FY;
};

template <int K, typename T, bool ACC>
__global__ void __launch_bounds__(Prol2Cfg<K>::NT)
    prolong2d_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ xc, T *__restrict__ xf, int mc,
                     int nc)
{
  pdl_prologue();
  using C = Prol2Cfg<K>;
  constexpr int CX = C::CX, CY = C::CY, FX = C::FX, QX = C::QX, QY = C::QY, NT = C::NT;
  __shared__ T Ps[2 * K + 1][K + 1];
  __shared__ T Cs[QY][QX];
  __shared__ T T1[QY][FX];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < (2 * K + 1) * (K + 1); e += NT)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  const int cx0 = blockIdx.x * CX, cy0 = blockIdx.y * CY;
  for (int e = tid; e < QY * QX; e += NT)
  {
    const int iy = e / QX, ix = e - iy * QX;
    const int qx = cx0 * K + ix, qy = cy0 * K + iy;  // coarse lattice, 0 and mc + 1 on the boundary
    Cs[iy][ix] = (qx >= 1 && qx <= mc && qy >= 1 && qy <= mc)
                     ? __ldg(xc + static_cast<int64_t>(qy - 1) * mc + (qx - 1))
                     : T(0);
  }
  __syncthreads();
  for (int e = tid; e < QY * FX; e += NT)
  {
    const int iy = e / FX, fx = e - iy * FX;
    const int c = fx / (2 * K), r = fx - 2 * K * c + 1;
    T s = T(0);
#pragma unroll
    for (int t = 0; t <= K; ++t)
      s = fma(Ps[r][t], Cs[iy][c * K + t], s);
    T1[iy][fx] = s;
  }
  __syncthreads();
  const int fx = threadIdx.x;
  if (fx >= FX)
    return;
  const int cxl = fx / (2 * K), rx = fx - 2 * K * cxl + 1;
  const int mf = 2 * mc + 1;
  const int px = 2 * (cx0 + cxl) * K + rx;  // fine lattice
  if (cx0 + cxl >= nc || px > mf)
    return;
  // the RY accumulated outputs: all loads of x_f before the first store
  T old[C::RY];
  bool ok[C::RY];
  T *o[C::RY];
#pragma unroll
  for (int rb = 0; rb < C::RY; ++rb)
  {
    const int fy = threadIdx.y + rb * C::FY;
    const int cyl = fy / (2 * K), ry = fy - 2 * K * cyl + 1;
    const int py = 2 * (cy0 + cyl) * K + ry;
    ok[rb] = cy0 + cyl < nc && py <= mf;
    o[rb] = xf + static_cast<int64_t>(ok[rb] ? py - 1 : 0) * mf + (px - 1);
    if constexpr (ACC)
      old[rb] = ok[rb] ? *o[rb] : T(0);
  }
#pragma unroll
  for (int rb = 0; rb < C::RY; ++rb)
  {
    if (!ok[rb])
      continue;
    const int fy = threadIdx.y + rb * C::FY;
    const int cyl = fy / (2 * K), ry = fy - 2 * K * cyl + 1;
    T s = T(0);
#pragma unroll
    for (int t = 0; t <= K; ++t)
      s = fma(Ps[ry][t], T1[cyl * K + t][fx], s);
    *o[rb] = ACC ? old[rb] + s : s;
  }
}

template <int K>
struct Rest2Cfg
{
  static constexpr int CX = 32 / K, CY = (16 / K) >= 2 ? 16 / K : 2;
  static constexpr int OX = CX * K, OY = CY * K;
  static constexpr int WX = 2 * K * (CX + 1), WY = 2 * K * (CY + 1), WN = WX * WY;
  static constexpr int NT = 32 * OY;
};

template <int K, typename T>
__global__ void __launch_bounds__(Rest2Cfg<K>::NT)
    restrict2d_kernel(const __grid_constant__ ProlMats<T, K> P, const T *__restrict__ rf, T *__restrict__ rc,
                      T *__restrict__ zero, int mc)
{
  using C = Rest2Cfg<K>;
  constexpr int CX = C::CX, CY = C::CY, OX = C::OX, OY = C::OY, WX = C::WX, WY = C::WY, NT = C::NT;
  __shared__ T Ps[2 * K + 1][K + 1];
  __shared__ __align__(16) T F[WY * WX];
  __shared__ T R1[WY][OX];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  for (int e = tid; e < (2 * K + 1) * (K + 1); e += NT)
    (&Ps[0][0])[e] = (&P.P[0][0])[e];
  const int mf = 2 * mc + 1;
  const int cx0 = blockIdx.x * CX, cy0 = blockIdx.y * CY;
  const int fx0 = 2 * cx0 * K, fy0 = 2 * cy0 * K;  // 0-based fine index of window (0, 0)
  pdl_prologue();
  for (int e = tid; e < C::WN; e += NT)
  {
    const int fy = e / WX, fx = e - fy * WX;
    const bool ok = fy0 + fy < mf && fx0 + fx < mf;
    tr_cp_async(&F[e], ok ? rf + static_cast<int64_t>(fy0 + fy) * mf + (fx0 + fx) : rf, ok);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  const int qx = cx0 * K + 1 + tx, qy = cy0 * K + 1 + ty;
  if (tx < OX)
    for (int fy = ty; fy < WY; fy += OY)
      R1[fy][tx] = rest_gather_1d<K, T>(Ps, qx, cx0, [&](int o) { return F[fy * WX + o]; });
  __syncthreads();
  if (tx >= OX || qx > mc || qy > mc)
    return;
  const T v = rest_gather_1d<K, T>(Ps, qy, cy0, [&](int o) { return R1[o][tx]; });
  const int64_t idx = static_cast<int64_t>(qy - 1) * mc + (qx - 1);
  rc[idx] = v;
  if (zero)
    zero[idx] = T(0);
}

template <int D, int K, typename T>
void launch_prolongate(const ProlMats<T, K> &P, const T *xc, T *xf, bool acc, int64_t mc,
                       T *tA, T *tB, int sm_count, cudaStream_t s)
{
  const int64_t mf = 2 * mc + 1;
  if constexpr (D == 2)
  {
    if (use_fused_transfer())
    {
      using C = Prol2Cfg<K>;
      const int nc = static_cast<int>((mc + 1) / K);
      const dim3 grid((nc + C::CX - 1) / C::CX, (nc + C::CY - 1) / C::CY);
      if (acc)
        pdl_launch(prolong2d_kernel<K, T, true>, grid, dim3(32, C::FY), 0, s, P, xc, xf, static_cast<int>(mc), nc);
      else
        pdl_launch(prolong2d_kernel<K, T, false>, grid, dim3(32, C::FY), 0, s, P, xc, xf, static_cast<int>(mc), nc);
      check_launch("prolong2d_kernel");
      return;
    }
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

// Where the z-march wins (tools/quick_ops.py, profiles/r01/restrict3d.txt):
// k = 1, 2, 4 on fine levels of >= 96 nodes per direction (1.3-1.6x over the
// passes). Below that the per-plane staging latency of the march (2k planes
// per cell in sequence) exceeds three fully parallel passes; for k = 3, 5-7
// the y-window halo (CY = 2 or 1 cells) costs more than the saved traffic.
inline int64_t restrict3d_min_nodes()
{
  static const int64_t v = [] {
    const char *e = std::getenv("PMG_RESTRICT3D_MIN");
    return e ? static_cast<int64_t>(std::atoll(e)) : int64_t(96);
  }();
  return v;
}
template <int K>
inline bool use_restrict3d(int64_t mc)
{
  return use_fused_transfer() && (K == 1 || K == 2 || K == 4) && 2 * mc + 1 >= restrict3d_min_nodes();
}

// coarse z-nodes [q0, q1) (0-based) of R r_f in one launch; chunks of the
// node range along z so that ~4 CTAs per SM are in flight
template <int K, typename T>
void launch_restrict3d(const ProlMats<T, K> &P, const T *rf, T *rc, T *zero, int64_t mc, int64_t q0, int64_t q1,
                       int sm_count, cudaStream_t s)
{
  using C = Rest3Cfg<K>;
  const int64_t gx = (mc + C::OX - 1) / C::OX, gy = (mc + C::OY - 1) / C::OY;
  const int64_t nq = q1 - q0;
  const int64_t want = std::max<int64_t>(1, (4 * static_cast<int64_t>(sm_count)) / (gx * gy));
  const int64_t cells = (nq + K - 1) / K;
  const int64_t chunks = std::min<int64_t>(want, cells);
  const int64_t npc = ((cells + chunks - 1) / chunks) * K;  // nodes per chunk (whole cells)
  const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>((nq + npc - 1) / npc));
  pdl_launch(restrict3d_kernel<K, T>, grid, dim3(32, C::OY), 0, s, P, rf, rc, zero, static_cast<int>(mc),
             static_cast<int>(q0), static_cast<int>(q1), static_cast<int>(npc));
  check_launch("restrict3d_kernel");
}

template <int D, int K, typename T>
void launch_restrict(const ProlMats<T, K> &P, const T *rf, T *rc, T *zero, int64_t mc, T *tA, T *tB,
                     int sm_count, cudaStream_t s)
{
  const int64_t mf = 2 * mc + 1;
  if constexpr (D == 2)
  {
    if (use_fused_transfer())
    {
      using C = Rest2Cfg<K>;
      const dim3 grid(static_cast<unsigned>((mc + C::OX - 1) / C::OX), static_cast<unsigned>((mc + C::OY - 1) / C::OY));
      pdl_launch(restrict2d_kernel<K, T>, grid, dim3(32, C::OY), 0, s, P, rf, rc, zero, static_cast<int>(mc));
      check_launch("restrict2d_kernel");
      return;
    }
    pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc, mf, 1), dim3(32, 8), 0, s, P, rf, tA, mc, mf, 1, mf, int64_t(0),
               static_cast<T *>(nullptr));
    check_launch("restrict_pass0");
    pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc, mc, 1), dim3(32, 8), 0, s, P, tA, rc, mc, mc, 1, mf, int64_t(0),
               zero);
    check_launch("restrict_pass1");
  }
  else if (use_restrict3d<K>(mc))
  {
    launch_restrict3d<K, T>(P, rf, rc, zero, mc, 0, mc, sm_count, s);
  }
  else
  {
    pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc, mf, mf), dim3(32, 8), 0, s, P, rf, tA, mc, mf, mf, mf, int64_t(0),
               static_cast<T *>(nullptr));
    check_launch("restrict_pass0");
    pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc, mc, mf), dim3(32, 8), 0, s, P, tA, tB, mc, mc, mf, mf, int64_t(0),
               static_cast<T *>(nullptr));
    check_launch("restrict_pass1");
    pdl_launch(restrict_pass_kernel<K, T, 2>, pass_grid(mc, mc, mc), dim3(32, 8), 0, s, P, tB, rc, mc, mc, mc, mf, int64_t(0),
               zero);
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
                          T *tB, int sm_count, cudaStream_t s)
{
  if (q1 <= q0)
    return;
  if (use_restrict3d<K>(mc))
  {
    launch_restrict3d<K, T>(P, rf, rc, static_cast<T *>(nullptr), mc, q0, q1, sm_count, s);
    return;
  }
  const int64_t mf = 2 * mc + 1;
  int64_t pz0, pz1;
  restrict_slab_fine_range(K, mc, q0, q1, pz0, pz1);
  pdl_launch(restrict_pass_kernel<K, T, 0>, pass_grid(mc, mf, pz1 - pz0), dim3(32, 8), 0, s, P, rf, tA, mc, mf, mf,
             mf, pz0, static_cast<T *>(nullptr));
  check_launch("restrict_pass0(slab)");
  pdl_launch(restrict_pass_kernel<K, T, 1>, pass_grid(mc, mc, pz1 - pz0), dim3(32, 8), 0, s, P, tA, tB, mc, mc, mf,
             mf, pz0, static_cast<T *>(nullptr));
  check_launch("restrict_pass1(slab)");
  pdl_launch(restrict_pass_kernel<K, T, 2>, pass_grid(mc, mc, q1 - q0), dim3(32, 8), 0, s, P, tB, rc, mc, mc, mc,
             mf, q0, static_cast<T *>(nullptr));
  check_launch("restrict_pass2(slab)");
}

}  // namespace pmgb
