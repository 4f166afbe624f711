// Included by kern_k<K>.cu with PMG_K defined: instantiates every kernel of
// one polynomial degree for dim in {2,3} and T in {float,double}.
#include <algorithm>

#include "../../include/pmg_b200.h"
#include "dispatch.hpp"
#include "operator_impl.cuh"
#include "smoother_impl.cuh"
#include "smoother_plane.cuh"
#include "smoother_point.cuh"
#include "smoother_pp.cuh"
#include "smoother_patch2d.cuh"
#include "transfer_impl.cuh"

#define PMG_CAT2(a, b) a##b
#define PMG_CAT(a, b) PMG_CAT2(a, b)

namespace pmgb
{
namespace
{

// 3D fused / boundary sweeps of degree <= PMG_PLANE_KMAX (and f32 degree 3,
// +7% over the ping-pong kernel) use the plane-streaming kernel
// (smoother_plane.cuh) unless pmg_set_smoother_impl selects the line one
#ifndef PMG_PATCH3D_MIN_PATCHES
#define PMG_PATCH3D_MIN_PATCHES 65536
#endif
#ifndef PMG_PATCH2D_KMAX
#define PMG_PATCH2D_KMAX 3
#endif
#ifndef PMG_PLANE_KMAX
#define PMG_PLANE_KMAX 2
#endif

// Which kernel organisation runs a (fused / boundary / ...) colour launch of
// this degree: the measured per-(d, k, precision, size) dispatch, or the one
// pmg_set_smoother_impl forces where it exists. One function for the launch
// and for pmg_smoother_kernel (the tests assert the organisation they check).
template <int D, typename T>
int smooth_choice(const ColorArgs<T> &a, int mode)
{
  const int impl = smoother_impl_choice();
  const bool fb = mode == MODE_FUSED || mode == MODE_BOUNDARY;
  if (!fb)
    return PMG_KERNEL_LINE;
  if constexpr (PMG_K == 1)
  {
    // degree 1: point-stencil kernel (smoother_point.cuh)
    if (impl == SMOOTHER_IMPL_AUTO || impl == SMOOTHER_IMPL_SWEEP)
      return PMG_KERNEL_POINT;
  }
  if constexpr (D == 2 && PMG_K >= 2 && (PMG_K <= PMG_PATCH2D_KMAX || (PMG_K == 4 && sizeof(T) == 4)))
  {
    // 2D degree 2..: one thread per patch, all in registers (smoother_patch2d.cuh)
    if (impl != SMOOTHER_IMPL_LINE)
      return PMG_KERNEL_PATCH2D;
  }
  if constexpr (D == 3 && PMG_K == 2)
  {
    // one thread per patch wins once a colour has enough patches to fill the
    // GPU with threads (measured: +25-33% f64, +65% f32 at >= 2.6e5 patches per
    // colour; -20% at C2's 3.1e4, where the plane kernel's 9 threads per
    // patch keep the SMs busy). Decided on the whole level's colour, so slab
    // and range launches pick the same kernel as the full level.
    const bool big = a.level_total >= PMG_PATCH3D_MIN_PATCHES;
    if (impl == SMOOTHER_IMPL_PATCH || (impl == SMOOTHER_IMPL_AUTO && big))
      return PMG_KERNEL_PATCH3D;
  }
  // (f32 k = 3 went to the plane kernel until the pp kernel's staging rewrite:
  // pp is now 10% faster there, profiles/r01/ab_f32k3_pp_vs_plane.txt)
  if constexpr (D == 3 && PMG_K <= PMG_PLANE_KMAX)
  {
    if (impl != SMOOTHER_IMPL_LINE)
      return PMG_KERNEL_PLANE;
  }
  // f32 k = 6 too (profiles/r01/ab_pp_f32_k67.txt: +5-11%; k = 7 f32 -4%).
  // Ping-pong layouts (smoother_pp.cuh), measured +6..11% at k = 3, 4; at
  // k = 5 f64 and k >= 6 the second work buffer costs resident CTAs and the
  // in-place kernel wins.
  if constexpr (D == 3 && (PMG_K == 3 || PMG_K == 4 || ((PMG_K == 5 || PMG_K == 6) && sizeof(T) == 4)))
  {
    if (impl != SMOOTHER_IMPL_LINE)
      return PMG_KERNEL_PP;
  }
  return PMG_KERNEL_LINE;
}

template <int D, typename T>
void smooth_entry(const void *P, const ColorArgs<T> &a, int mode, int sm_count, cudaStream_t s)
{
  const auto &PM = *static_cast<const PatchMatsEO<T, PMG_K> *>(P);
  const int choice = smooth_choice<D, T>(a, mode);
  const bool fused = mode == MODE_FUSED;
  if constexpr (PMG_K == 1)
  {
    if (choice == PMG_KERNEL_POINT)
    {
      // the stencil follows the even-odd matrices in the level's parameter blob (capi.cu level_init)
      const auto &st = *reinterpret_cast<const PointStencil<T> *>(static_cast<const unsigned char *>(P) +
                                                                   sizeof(PatchMatsEO<T, 1>));
      if (fused)
        launch_vp_point<D, T, MODE_FUSED>(st, a, s);
      else
        launch_vp_point<D, T, MODE_BOUNDARY>(st, a, s);
      return;
    }
  }
  if constexpr (D == 2 && PMG_K >= 2 && (PMG_K <= PMG_PATCH2D_KMAX || (PMG_K == 4 && sizeof(T) == 4)))
  {
    if (choice == PMG_KERNEL_PATCH2D)
    {
      if (fused)
        launch_vp_patch2d<PMG_K, T, MODE_FUSED>(PM, a, s);
      else
        launch_vp_patch2d<PMG_K, T, MODE_BOUNDARY>(PM, a, s);
      return;
    }
  }
  if constexpr (D == 3 && PMG_K == 2)
  {
    if (choice == PMG_KERNEL_PATCH3D)
    {
      // S^T M_if, S^T A_if after the even-odd and dense matrices in the parameter blob
      const auto &DM = *reinterpret_cast<const PatchST<T, PMG_K> *>(
          static_cast<const unsigned char *>(P) + sizeof(PatchMatsEO<T, PMG_K>) + sizeof(PatchMats<T, PMG_K>));
      if (fused)
        launch_vp_patch3d<PMG_K, T, MODE_FUSED>(PM, DM, a, s);
      else
        launch_vp_patch3d<PMG_K, T, MODE_BOUNDARY>(PM, DM, a, s);
      return;
    }
  }
  if constexpr (D == 3 && PMG_K <= PMG_PLANE_KMAX)
  {
    if (choice == PMG_KERNEL_PLANE)
    {
      if (fused)
        launch_vp_smooth_plane<PMG_K, T, MODE_FUSED>(PM, a, s);
      else
        launch_vp_smooth_plane<PMG_K, T, MODE_BOUNDARY>(PM, a, s);
      return;
    }
  }
  if constexpr (D == 3 && (PMG_K == 3 || PMG_K == 4 || ((PMG_K == 5 || PMG_K == 6) && sizeof(T) == 4)))
  {
    if (choice == PMG_KERNEL_PP)
    {
      if (fused)
        launch_vp_smooth_pp<PMG_K, T, MODE_FUSED>(PM, a, s);
      else
        launch_vp_smooth_pp<PMG_K, T, MODE_BOUNDARY>(PM, a, s);
      return;
    }
  }
  launch_vp_smooth_mode<D, PMG_K, T>(PM, a, mode, sm_count, s);
}

template <int D, typename T>
bool sweep_entry(const void *P, const SweepArgs<T> &sw, int mode, int sm_count, cudaStream_t s)
{
  if constexpr (D == 3 && PMG_K == 2)
  {
    const auto &PM = *static_cast<const PatchMatsEO<T, PMG_K> *>(P);
    if (mode == MODE_FUSED)
      launch_vp_sweep_plane<PMG_K, T, MODE_FUSED>(PM, sw, sm_count, s);
    else if (mode == MODE_BOUNDARY)
      launch_vp_sweep_plane<PMG_K, T, MODE_BOUNDARY>(PM, sw, sm_count, s);
    else
      return false;
    return true;
  }
  return false;
}

template <int D, typename T>
void op_entry(const void *B, const T *x, const T *b, T *y, int64_t m, int sm_count, cudaStream_t s)
{
  launch_level_op<D, PMG_K, T>(*static_cast<const BandMats<T, PMG_K> *>(B), x, b, y, m, sm_count, s);
}

template <int D, typename T>
void prol_entry(const void *P, const T *xc, T *xf, bool acc, int64_t mc, T *tA, T *tB, int sm_count,
                cudaStream_t s)
{
  launch_prolongate<D, PMG_K, T>(*static_cast<const ProlMats<T, PMG_K> *>(P), xc, xf, acc, mc, tA, tB,
                                 sm_count, s);
}

template <int D, typename T>
void rest_entry(const void *P, const T *rf, T *rc, T *zero, int64_t mc, T *tA, T *tB, int sm_count,
                cudaStream_t s)
{
  launch_restrict<D, PMG_K, T>(*static_cast<const ProlMats<T, PMG_K> *>(P), rf, rc, zero, mc, tA, tB,
                               sm_count, s);
}

template <int D, typename T>
void op_range_entry(const void *B, const T *x, const T *b, T *y, int64_t m, int64_t z0, int64_t z1, int sm_count,
                    cudaStream_t s)
{
  launch_level_op<D, PMG_K, T>(*static_cast<const BandMats<T, PMG_K> *>(B), x, b, y, m, sm_count, s, z0, z1);
}

template <typename T>
void prol_slab_entry(const void *P, const T *xc, T *xf, bool acc, int64_t mc, int64_t f0, int64_t f1, cudaStream_t s)
{
  launch_prolongate_slab<PMG_K, T>(*static_cast<const ProlMats<T, PMG_K> *>(P), xc, xf, acc, mc, f0, f1, s);
}

template <typename T>
void rest_slab_entry(const void *P, const T *rf, T *rc, int64_t mc, int64_t q0, int64_t q1, T *tA, T *tB,
                     int sm_count, cudaStream_t s)
{
  launch_restrict_slab<PMG_K, T>(*static_cast<const ProlMats<T, PMG_K> *>(P), rf, rc, mc, q0, q1, tA, tB, sm_count,
                                 s);
}

template <int D, typename T>
KernelTable<T> make_table()
{
  KernelTable<T> t;
  t.smooth = &smooth_entry<D, T>;
  t.smooth_kernel = &smooth_choice<D, T>;
  t.sweep = &sweep_entry<D, T>;
  t.sweep_pb = PMG_K == 2 ? PlaneCfg<2, T>::PB : 0;
  t.level_op = &op_entry<D, T>;
  if constexpr (D == 3)
  {
    t.level_op_range = &op_range_entry<D, T>;
    t.prolongate_slab = &prol_slab_entry<T>;
    t.restrict_slab = &rest_slab_entry<T>;
  }
  t.prolongate = &prol_entry<D, T>;
  t.restrict_ = &rest_entry<D, T>;
  t.smooth_smem = sm_smem_bytes<D, PMG_K, T>();
  t.smooth_threads = sm_nt<D, PMG_K, T>();
  t.smooth_pb = sm_pb<D, PMG_K, T>();
  return t;
}

}  // namespace

void PMG_CAT(register_k, PMG_K)(Tables &tb)
{
  tb.f64[0][PMG_K] = make_table<2, double>();
  tb.f64[1][PMG_K] = make_table<3, double>();
  tb.f32[0][PMG_K] = make_table<2, float>();
  tb.f32[1][PMG_K] = make_table<3, float>();
}

}  // namespace pmgb
