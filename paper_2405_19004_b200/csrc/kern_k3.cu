// Kernels of polynomial degree 3 (see instantiate.cuh).
#define PMG_K 3
#include "instantiate.cuh"
