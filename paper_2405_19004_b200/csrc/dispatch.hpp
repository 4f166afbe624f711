// Run-time (dim, degree, precision) -> compile-time kernel instantiation.
// Each kern_k<K>.cu registers the launchers of one degree.
#pragma once

#include "common.cuh"

namespace pmgb
{

template <typename T>
struct KernelTable
{
  // P: PatchMatsEO<T,K>*; mode: MODE_*
  void (*smooth)(const void *P, const ColorArgs<T> &a, int mode, int sm_count, cudaStream_t s) = nullptr;
  // the organisation `smooth` launches for these arguments (PMG_KERNEL_*)
  int (*smooth_kernel)(const ColorArgs<T> &a, int mode) = nullptr;
  // whole smoothing step in one persistent launch (3D fused / boundary, where
  // available): returns false when this (dim, degree) has no sweep kernel
  bool (*sweep)(const void *P, const SweepArgs<T> &sw, int mode, int sm_count, cudaStream_t s) = nullptr;
  int sweep_pb = 0;  // patches per tile of the sweep kernel
  // B: BandMats<T,K>*; b == nullptr -> y = A x, else y = b - A x
  void (*level_op)(const void *B, const T *x, const T *b, T *y, int64_t m, int sm_count,
                   cudaStream_t s) = nullptr;
  // slab versions (3D): global-plane bases, output planes [z0, z1)
  void (*level_op_range)(const void *B, const T *x, const T *b, T *y, int64_t m, int64_t z0, int64_t z1,
                         int sm_count, cudaStream_t s) = nullptr;
  void (*prolongate_slab)(const void *P, const T *xc, T *xf, bool acc, int64_t mc, int64_t f0, int64_t f1,
                          cudaStream_t s) = nullptr;
  void (*restrict_slab)(const void *P, const T *rf, T *rc, int64_t mc, int64_t q0, int64_t q1, T *tA, T *tB,
                        int sm_count, cudaStream_t s) = nullptr;
  // P: ProlMats<T,K>*
  void (*prolongate)(const void *P, const T *xc, T *xf, bool acc, int64_t mc, T *tA, T *tB,
                     int sm_count, cudaStream_t s) = nullptr;
  // zero (optional): cleared at the coarse nodes (the V-cycle's x_c = 0)
  void (*restrict_)(const void *P, const T *rf, T *rc, T *zero, int64_t mc, T *tA, T *tB, int sm_count,
                    cudaStream_t s) = nullptr;
  size_t smooth_smem = 0;   // dynamic smem per CTA of the fused kernel
  int smooth_threads = 0;   // threads per CTA
  int smooth_pb = 0;        // patches per CTA
};

struct Tables
{
  KernelTable<double> f64[2][8];  // [dim-2][k]
  KernelTable<float> f32[2][8];
};

Tables &tables();

void register_k1(Tables &);
void register_k2(Tables &);
void register_k3(Tables &);
void register_k4(Tables &);
void register_k5(Tables &);
void register_k6(Tables &);
void register_k7(Tables &);

}  // namespace pmgb
