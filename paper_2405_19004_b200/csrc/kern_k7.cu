// Kernels of polynomial degree 7 (see instantiate.cuh).
#define PMG_K 7
#include "instantiate.cuh"
