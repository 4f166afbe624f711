// Kernels of polynomial degree 2 (see instantiate.cuh).
#define PMG_K 2
#include "instantiate.cuh"
