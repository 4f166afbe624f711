// Internal state behind the C-ABI handles (shared by capi.cu and gmres.cu).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pmg_b200.h"
#include "common.cuh"
#include "setup.hpp"

namespace pmgb
{

struct DivergenceErr : std::runtime_error
{
  using std::runtime_error::runtime_error;
};

// bumped whenever a DevBuf is (re)allocated: captured graphs that baked in
// workspace pointers compare it before replaying
inline std::atomic<unsigned> g_buf_generation{0};

// RAII device buffer
struct DevBuf
{
  void *p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  ~DevBuf()
  {
    if (p)
      cudaFree(p);
  }
  void ensure(size_t b)
  {
    if (b <= bytes)
      return;
    if (p)
      check_cuda(cudaFree(p), "cudaFree");
    p = nullptr;
    bytes = 0;
    check_cuda(cudaMalloc(&p, b), "cudaMalloc");
    bytes = b;
    g_buf_generation.fetch_add(1, std::memory_order_relaxed);
  }
  template <typename T>
  T *as() const
  {
    return static_cast<T *>(p);
  }
};

struct DevScope
{
  int prev = 0;
  explicit DevScope(int dev)
  {
    check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev)
      check_cuda(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DevScope() { cudaSetDevice(prev); }
};

struct GmresWork
{
  DevBuf bV, bZ, bw, br, bred, brf, bzf, bflag;
  double *V = nullptr, *Z = nullptr, *w = nullptr, *r = nullptr, *red = nullptr;
  float *rf = nullptr, *zf = nullptr;
  int *flag = nullptr;
  void ensure(int64_t n, int restart, bool mixed);
};

// maps C++ exceptions to pmg_status and records pmg_last_error
int capi_status_from_current_exception();

template <typename F>
int capi_guard(F &&f)
{
  try
  {
    f();
    return PMG_OK;
  }
  catch (...)
  {
    return capi_status_from_current_exception();
  }
}

struct GsData;  // point Gauss-Seidel front lists of a level (gs.cu)
std::shared_ptr<GsData> &level_gs_slot(pmg_level l);
const LevelSetup &level_setup(pmg_level l);
int level_dtype(pmg_level l);
int level_device(pmg_level l);
void gs_smooth(pmg_level l, double *x, const double *b, cudaStream_t s);
GsData *gs_data(pmg_level l);

int mg_dtype(pmg_mg h);
int mg_device(pmg_mg h);
int mg_levels(pmg_mg h);
pmg_level mg_level_ptr(pmg_mg h, int li);
int64_t level_total(pmg_level l);
int level_sm_count(pmg_level l);
void level_params(pmg_level l, int *dim, int *k, int *level, int *dtype, int *device);
GmresWork &mg_gmres_work(pmg_mg h);
void mg_apply_finest_op(pmg_mg h, const double *x, double *y, cudaStream_t s);
void mg_residual_finest(pmg_mg h, const double *x, const double *b, double *r, cudaStream_t s);
void mg_vcycle_f32(pmg_mg h, int li, float *x, const float *b, cudaStream_t s);
void mg_vcycle_f64(pmg_mg h, int li, double *x, const double *b, cudaStream_t s);
// the V-cycle of level index li from x = 0 (the recursion's coarse
// correction): the precomputed coarse operator where it applies, else the
// (graph-)V-cycle; used by the slab decomposition's agglomerated levels so they
// compute what the single-device recursion computes
void mg_coarse_correction(pmg_mg h, int li, void *x, const void *b, bool use_graph, cudaStream_t s);

}  // namespace pmgb
