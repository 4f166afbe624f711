#pragma once
#include "common.cuh"

namespace pmgb
{

constexpr int RED_BLOCKS = 1024;  // fixed grid of the two-pass reductions

// out[0] = sum a_i b_i (sqrt_it: sqrt of it); partial >= RED_BLOCKS doubles
template <typename T>
void launch_dot(const T *a, const T *b, int64_t n, double *partial, double *out, bool sqrt_it,
                cudaStream_t s);
template <typename T>
void launch_fill(T *x, int64_t n, T v, int sm_count, cudaStream_t s);
template <typename T>
void launch_axpby(T alpha, const T *x, T beta, T *y, int64_t n, int sm_count, cudaStream_t s);
void launch_axpy_dev(const double *alpha, double scale, const double *x, double *y, int64_t n,
                     int sm_count, cudaStream_t s);
void launch_d2f(const double *x, float *y, int64_t n, int *nonfinite, int sm_count, cudaStream_t s);
void launch_f2d(const float *x, double *y, int64_t n, int sm_count, cudaStream_t s);
// x = M b, M row-major n x n with row pitch ld (multiple of 4; the coarse
// V-cycle operator, capi.cu)
template <typename T>
void launch_coarse_gemv(const T *M, const T *b, T *x, int n, int ld, cudaStream_t s);
// x = e_j
template <typename T>
void launch_unit(T *x, int n, int j, cudaStream_t s);
// x = e_{*j}; column *j of M (row pitch ld) = v and ++*j (graph-replayed
// column sweep)
template <typename T>
void launch_unit_dev(T *x, int n, const int *j, cudaStream_t s);
template <typename T>
void launch_store_column(T *M, const T *v, int n, int ld, int *j, cudaStream_t s);

}  // namespace pmgb
