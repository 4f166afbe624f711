#pragma once
#include "common.cuh"

namespace pmgb
{

template <typename T>
struct NaiveArgs
{
  ColorArgs<T> c;
  const T *Mif;  // (2k-1) x (2k+1)
  const T *Aif;
  const T *S;    // (2k-1)^2
  int dim, k;
  T *scratch;
  int64_t scratch_stride;
};

template <typename T>
int64_t naive_scratch_per_block(int dim, int k);
template <typename T>
void launch_naive_smooth(const NaiveArgs<T> &a, int grid, cudaStream_t s);

}  // namespace pmgb
