// Kernels of polynomial degree 4 (see instantiate.cuh).
#define PMG_K 4
#include "instantiate.cuh"
