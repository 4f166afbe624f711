// Included by kern_k<K>.cu with PMG_K defined: instantiates every kernel of
// one polynomial degree for dim in {2,3} and T in {float,double}.
#include <algorithm>

#include "dispatch.hpp"
#include "operator_impl.cuh"
#include "smoother_impl.cuh"
#include "transfer_impl.cuh"

#define PMG_CAT2(a, b) a##b
#define PMG_CAT(a, b) PMG_CAT2(a, b)

namespace pmgb
{
namespace
{

template <int D, typename T>
void smooth_entry(const void *P, const ColorArgs<T> &a, int mode, int sm_count, cudaStream_t s)
{
  launch_vp_smooth_mode<D, PMG_K, T>(*static_cast<const PatchMatsEO<T, PMG_K> *>(P), a, mode, sm_count, s);
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
void rest_entry(const void *P, const T *rf, T *rc, int64_t mc, T *tA, T *tB, int sm_count,
                cudaStream_t s)
{
  launch_restrict<D, PMG_K, T>(*static_cast<const ProlMats<T, PMG_K> *>(P), rf, rc, mc, tA, tB,
                               sm_count, s);
}

template <int D, typename T>
KernelTable<T> make_table()
{
  KernelTable<T> t;
  t.smooth = &smooth_entry<D, T>;
  t.level_op = &op_entry<D, T>;
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
