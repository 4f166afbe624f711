// Throughput probe (development tool): FP64 DFMA vs DMMA (mma.sync m8n8k4 f64)
// vs TF32 mma.sync m16n8k8 on the current GPU. Decides whether a tensor-core
// variant of the sum-factorisation contractions can beat the CUDA-core path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void dmma_kernel(double *out, double seed)
{
  double a = seed + threadIdx.x, b = seed * 2 + threadIdx.x;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    c[j][0] = c[j][1] = 0;
  for (int it = 0; it < ITERS; ++it)
  {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_kernel(double *out, double seed)
{
  double a = seed + threadIdx.x, b = seed * 2 + threadIdx.x;
  double c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    c[j] = j;
  for (int it = 0; it < ITERS; ++it)
  {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      c[j] = fma(a, c[j], b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void tf32_kernel(float *out, float seed)
{
  unsigned a0 = __float_as_uint(seed + threadIdx.x), b0 = __float_as_uint(seed * 2.f);
  float c[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
  for (int it = 0; it < ITERS; ++it)
  {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a0), "r"(a0), "r"(a0), "r"(b0), "r"(b0));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_kernel(float *out, float seed)
{
  float a = seed + threadIdx.x, b = seed * 2;
  float c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    c[j] = j;
  for (int it = 0; it < ITERS; ++it)
  {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      c[j] = fmaf(a, c[j], b);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_it(F f)
{
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r)
    f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main()
{
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  double *d;
  cudaMalloc(&d, sizeof(double) * blocks * threads);
  const double nthr = double(blocks) * threads;
  float ms = time_it([&] { dmma_kernel<<<blocks, threads>>>(d, 1.0); });
  // per warp-mma: 8*8*4 MACs = 512 flops; per thread 512/32 = 16 flops
  printf("DMMA m8n8k4 f64 : %.1f TFLOP/s\n", nthr / 32 * ITERS * 8 * 512 / (ms * 1e-3) / 1e12);
  ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(d, 1.0); });
  printf("DFMA            : %.1f TFLOP/s\n", nthr * ITERS * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = time_it([&] { tf32_kernel<<<blocks, threads>>>((float *)d, 1.f); });
  printf("mma.sync tf32   : %.1f TFLOP/s\n", nthr / 32 * ITERS * 8 * (16 * 8 * 8 * 2) / (ms * 1e-3) / 1e12);
  ms = time_it([&] { ffma_kernel<<<blocks, threads>>>((float *)d, 1.f); });
  printf("FFMA            : %.1f TFLOP/s\n", nthr * ITERS * 8 * 2 / (ms * 1e-3) / 1e12);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
