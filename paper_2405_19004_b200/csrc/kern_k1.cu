// Kernels of polynomial degree 1 (see instantiate.cuh).
#define PMG_K 1
#include "instantiate.cuh"
