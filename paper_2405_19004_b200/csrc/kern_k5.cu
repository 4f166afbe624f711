// Kernels of polynomial degree 5 (see instantiate.cuh).
#define PMG_K 5
#include "instantiate.cuh"
