// Kernels of polynomial degree 6 (see instantiate.cuh).
#define PMG_K 6
#include "instantiate.cuh"
