// tcgen05 (5th-gen tensor core) A/B probe for the f32 smoother's contraction
// stages: is a tcgen05.mma kind::tf32 3xTF32 version of
// the dir-0 stage (z_M = M_if x, z_A = A_if x along closure lines) faster than
// the CUDA-core even-odd version the f32 pp / line kernels use?
//
// Both paths run the SAME stage on lines resident in shared memory (the work
// buffer layout of the kernels: one closure line of NC values per row), write
// 2 NI outputs per line back to shared memory, repeated R times per CTA, one
// CTA of 128 threads per SM slot:
//   CUDA cores : thread = line; even-odd split (K+1 / K terms), 2 (K(K+1) +
//                (K-1)K) FFMA per line, matrices in registers (uniform).
//   tensor core: 128 lines = the M = 128 rows of one UMMA; thread = line
//                splits its NC values into tf32 hi + lo and writes them in the
//                canonical K-major SWIZZLE_NONE layout; one elected thread
//                issues 3 x ceil(NC/8) tcgen05.mma.kind::tf32 (hi*hi + hi*lo +
//                lo*hi, f32 accumulate in TMEM, N = 2 NI padded to 16/32) and
//                commits to an mbarrier; every warp reads its 32 TMEM lanes
//                (tcgen05.ld.32x32b) and stores the outputs.
// Reported: lines per second per path (events), the ratio, and the max
// relative error of each path against an f64 host reference.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo tools/tc_probe.cu -o tools/tc_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do                                                                                 \
  {                                                                                  \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
    {                                                                                \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(2);                                                                  \
    }                                                                                \
  } while (0)

constexpr int LINES = 128;  // lines per CTA = UMMA M

template <int K>
struct Cfg
{
  static constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  static constexpr int KP = (NC + 7) / 8 * 8;                        // padded K
  static constexpr int NO = 2 * NI;                                   // outputs per line
  static constexpr int NP = NO <= 16 ? 16 : (NO <= 32 ? 32 : 48);     // padded N
  static constexpr int LDL = NC + 1;                                  // line stride in the work buffer
};

template <int K>
struct Mats
{
  float M[2 * K - 1][2 * K + 1], A[2 * K - 1][2 * K + 1];
  float Me[K][K + 1], Mo[K][K], Ae[K][K + 1], Ao[K][K];  // even-odd forms
};

// ---- CUDA-core stage (the kernels' eo_rows) ----------------------------------
template <int K>
__device__ __forceinline__ void cc_line(const Mats<K> &P, const float *in, float *out)
{
  constexpr int NC = 2 * K + 1, NI = 2 * K - 1;
  float e[K + 1], o[K];
#pragma unroll
  for (int j = 0; j < K; ++j)
  {
    e[j] = in[j] + in[NC - 1 - j];
    o[j] = in[j] - in[NC - 1 - j];
  }
  e[K] = in[K];
#pragma unroll
  for (int h = 0; h < K; ++h)
  {
    float em = 0.f, ea = 0.f, om = 0.f, oa = 0.f;
#pragma unroll
    for (int j = 0; j <= K; ++j)
    {
      em = fmaf(P.Me[h][j], e[j], em);
      ea = fmaf(P.Ae[h][j], e[j], ea);
    }
    if (h < K - 1)
    {
#pragma unroll
      for (int j = 0; j < K; ++j)
      {
        om = fmaf(P.Mo[h][j], o[j], om);
        oa = fmaf(P.Ao[h][j], o[j], oa);
      }
      out[h] = em + om;
      out[NI - 1 - h] = em - om;
      out[NI + h] = ea + oa;
      out[NI + NI - 1 - h] = ea - oa;
    }
    else
    {
      out[h] = em;
      out[NI + h] = ea;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(LINES) cc_kernel(const __grid_constant__ Mats<K> P, const float *src, float *dst,
                                                   int reps)
{
  using C = Cfg<K>;
  __shared__ float Win[LINES * C::LDL];
  __shared__ float Wout[LINES * (C::NO + 1)];
  const int t = threadIdx.x;
  for (int e = t; e < LINES * C::LDL; e += LINES)
    Win[e] = src[(blockIdx.x * LINES * C::LDL + e) % (1 << 20)];
  __syncthreads();
  for (int r = 0; r < reps; ++r)
  {
    float in[C::NC], out[C::NO];
#pragma unroll
    for (int j = 0; j < C::NC; ++j)
      in[j] = Win[t * C::LDL + j];
    cc_line<K>(P, in, out);
#pragma unroll
    for (int i = 0; i < C::NO; ++i)
      Wout[t * (C::NO + 1) + i] = out[i];
    __syncthreads();
    // feed the outputs back as the next input (keeps the stage on the chain)
#pragma unroll
    for (int j = 0; j < C::NC; ++j)
      Win[t * C::LDL + j] = Wout[t * (C::NO + 1) + (j % C::NO)] * 0.5f;
    __syncthreads();
  }
  for (int i = 0; i < C::NO; ++i)
    dst[(blockIdx.x * LINES + t) * C::NO + i] = Wout[t * (C::NO + 1) + i];
}

// ---- tensor-core stage -------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (canonical
// ((8,m),(4 tf32, kchunks)) : core matrix 8 rows x 16 B contiguous):
// LBO = byte distance between K chunks, SBO = between 8-row groups
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version 1 (sm_100)
  return d;                             // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor kind::tf32: D f32, A/B tf32, both K-major, N, M = 128
__host__ __device__ constexpr uint32_t idesc_tf32(int N)
{
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

__device__ __forceinline__ void split_tf32(float x, float &hi, float &lo)
{
  uint32_t u = __float_as_uint(x) & 0xFFFFE000u;  // tf32 keeps 10 mantissa bits
  hi = __uint_as_float(u);
  lo = x - hi;
}

template <int K>
__global__ void __launch_bounds__(LINES) tc_kernel(const float *Bhl, const float *src, float *dst, int reps)
{
  using C = Cfg<K>;
  constexpr int KP = C::KP, NP = C::NP, NO = C::NO, NC = C::NC;
  constexpr int KCH = KP / 4;                 // 16-byte K chunks
  constexpr int A_LBO = (LINES / 8) * 128;    // bytes between K chunks of A (all row groups of a chunk)
  constexpr int B_LBO = (NP / 8) * 128;
  constexpr int A_BYTES = KCH * A_LBO, B_BYTES = KCH * B_LBO;
  __shared__ __align__(128) unsigned char Ahi[A_BYTES], Alo[A_BYTES], Bh[B_BYTES], Bl[B_BYTES];
  __shared__ float Win[LINES * C::LDL];
  __shared__ float Wout[LINES * (NO + 1)];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t / 32;
  // B = [M; A] (NO x NC, zero padded to NP x KP), split hi / lo on the host
  for (int e = t; e < NP * KP; e += LINES)
  {
    const int n = e / KP, kk = e % KP;
    const int off = (kk / 4) * B_LBO + (n / 8) * 128 + (n % 8) * 16 + (kk % 4) * 4;
    reinterpret_cast<float *>(Bh + off)[0] = Bhl[e];
    reinterpret_cast<float *>(Bl + off)[0] = Bhl[NP * KP + e];
  }
  for (int e = t; e < LINES * C::LDL; e += LINES)
    Win[e] = src[(blockIdx.x * LINES * C::LDL + e) % (1 << 20)];
  if (t == 0)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
  if (warp == 0)
  {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(32 * ((NP + 31) / 32)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  uint32_t phase = 0;
  const uint64_t dAh = smem_desc(smem_u32(Ahi), A_LBO, 128), dAl = smem_desc(smem_u32(Alo), A_LBO, 128);
  const uint64_t dBh = smem_desc(smem_u32(Bh), B_LBO, 128), dBl = smem_desc(smem_u32(Bl), B_LBO, 128);
  constexpr uint32_t idesc = idesc_tf32(NP);
  for (int r = 0; r < reps; ++r)
  {
    // this line -> A hi / lo, canonical K-major (row t: (t%8)*16 + (t/8)*128 + chunk*A_LBO)
#pragma unroll
    for (int c = 0; c < KCH; ++c)
    {
      float4 h, l;
      float v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        v[q] = (4 * c + q < NC) ? Win[t * C::LDL + 4 * c + q] : 0.f;
      split_tf32(v[0], h.x, l.x);
      split_tf32(v[1], h.y, l.y);
      split_tf32(v[2], h.z, l.z);
      split_tf32(v[3], h.w, l.w);
      const int off = c * A_LBO + (t / 8) * 128 + (t % 8) * 16;
      *reinterpret_cast<float4 *>(Ahi + off) = h;
      *reinterpret_cast<float4 *>(Alo + off) = l;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core
    __syncthreads();
    if (t == 0)
    {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int kb = 0; kb < KP / 8; ++kb)
      {
        // K block kb = 2 chunks of 16 B: advance the start addresses by 2 LBO
        const uint64_t ah = dAh + (static_cast<uint64_t>((2 * kb * A_LBO) >> 4)),
                       al = dAl + (static_cast<uint64_t>((2 * kb * A_LBO) >> 4));
        const uint64_t bh = dBh + (static_cast<uint64_t>((2 * kb * B_LBO) >> 4)),
                       bl = dBl + (static_cast<uint64_t>((2 * kb * B_LBO) >> 4));
        const uint64_t as[3] = {ah, ah, al}, bs[3] = {bh, bl, bh};
#pragma unroll
        for (int s = 0; s < 3; ++s)
        {
          const uint32_t acc = (kb > 0 || s > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
              "l"(as[s]), "l"(bs[s]), "r"(idesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar)));
    }
    // wait for the MMAs (mbarrier phase flips once per rep)
    {
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(&mbar)), "r"(phase));
      phase ^= 1;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // lane t of TMEM = line t: warp w reads lanes 32w .. 32w + 31
    uint32_t d[NP];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll
    for (int c = 0; c < NP; c += 8)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(d[c]), "=r"(d[c + 1]), "=r"(d[c + 2]), "=r"(d[c + 3]), "=r"(d[c + 4]), "=r"(d[c + 5]),
                     "=r"(d[c + 6]), "=r"(d[c + 7])
                   : "r"(taddr + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < NO; ++i)
      Wout[t * (NO + 1) + i] = __uint_as_float(d[i]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NC; ++j)
      Win[t * C::LDL + j] = Wout[t * (NO + 1) + (j % NO)] * 0.5f;
    __syncthreads();
  }
  for (int i = 0; i < NO; ++i)
    dst[(blockIdx.x * LINES + t) * NO + i] = Wout[t * (NO + 1) + i];
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32 * ((NP + 31) / 32)));
}

template <int K>
void run(int blocks, int reps)
{
  using C = Cfg<K>;
  constexpr int NC = C::NC, NI = C::NI, NO = C::NO, KP = C::KP, NP = C::NP;
  // a symmetric-banded-like test operator with the kernels' centro-symmetry
  // (interior rows of the 2-cell patch matrices are centro-symmetric)
  Mats<K> P{};
  std::vector<double> M(NI * NC), A(NI * NC);
  for (int i = 0; i < NI; ++i)
    for (int j = 0; j < NC; ++j)
    {
      const int ir = NI - 1 - i, jr = NC - 1 - j;
      // centro-symmetric fill: M[NI-1-i][NC-1-j] = M[i][j] (the middle row
      // symmetric in j), the property the even-odd form relies on
      const int a = i < ir ? i : ir, b = i < ir ? j : (i > ir ? jr : (j < jr ? j : jr));
      M[i * NC + j] = 0.1 + 0.05 * std::sin(1.0 + a + 0.37 * b);
      A[i * NC + j] = (i + 1 == j ? 2.0 : -0.3) + 0.1 * std::cos(0.5 + a * 1.3 + b);
    }
  for (int i = 0; i < NI; ++i)
    for (int j = 0; j < NC; ++j)
    {
      P.M[i][j] = static_cast<float>(M[i * NC + j]);
      P.A[i][j] = static_cast<float>(A[i * NC + j]);
    }
  for (int h = 0; h < K; ++h)
  {
    for (int j = 0; j < K; ++j)
    {
      P.Me[h][j] = static_cast<float>(0.5 * (M[h * NC + j] + M[h * NC + NC - 1 - j]));
      P.Ae[h][j] = static_cast<float>(0.5 * (A[h * NC + j] + A[h * NC + NC - 1 - j]));
      P.Mo[h][j] = static_cast<float>(0.5 * (M[h * NC + j] - M[h * NC + NC - 1 - j]));
      P.Ao[h][j] = static_cast<float>(0.5 * (A[h * NC + j] - A[h * NC + NC - 1 - j]));
    }
    P.Me[h][K] = static_cast<float>(M[h * NC + K]);
    P.Ae[h][K] = static_cast<float>(A[h * NC + K]);
  }
  std::vector<float> Bhl(2 * NP * KP, 0.f);
  for (int n = 0; n < NO; ++n)
    for (int kk = 0; kk < NC; ++kk)
    {
      const float v = n < NI ? P.M[n][kk] : P.A[n - NI][kk];
      const float hi = __builtin_bit_cast(float, __builtin_bit_cast(uint32_t, v) & 0xFFFFE000u);
      Bhl[n * KP + kk] = hi;
      Bhl[NP * KP + n * KP + kk] = v - hi;
    }
  const int nsrc = 1 << 20;
  std::vector<float> src(nsrc);
  for (int i = 0; i < nsrc; ++i)
    src[i] = static_cast<float>(std::sin(0.001 * i + 0.3) * 2.0);
  float *dsrc, *dcc, *dtc, *dB;
  const size_t nout = static_cast<size_t>(blocks) * LINES * NO;
  CK(cudaMalloc(&dsrc, nsrc * 4));
  CK(cudaMalloc(&dcc, nout * 4));
  CK(cudaMalloc(&dtc, nout * 4));
  CK(cudaMalloc(&dB, Bhl.size() * 4));
  CK(cudaMemcpy(dsrc, src.data(), nsrc * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bhl.data(), Bhl.size() * 4, cudaMemcpyHostToDevice));
  // accuracy: one rep against an f64 reference of the first line block
  cc_kernel<K><<<blocks, LINES>>>(P, dsrc, dcc, 1);
  tc_kernel<K><<<blocks, LINES>>>(dB, dsrc, dtc, 1);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> occ(nout), otc(nout);
  CK(cudaMemcpy(occ.data(), dcc, nout * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(otc.data(), dtc, nout * 4, cudaMemcpyDeviceToHost));
  double ecc = 0, etc = 0, scale = 0;
  for (int b = 0; b < 4; ++b)
    for (int l = 0; l < LINES; ++l)
      for (int n = 0; n < NO; ++n)
      {
        double ref = 0;
        for (int j = 0; j < NC; ++j)
        {
          const double x = src[(b * LINES * C::LDL + l * C::LDL + j) % nsrc];
          ref += (n < NI ? M[n * NC + j] : A[(n - NI) * NC + j]) * x;
        }
        const size_t o = (static_cast<size_t>(b) * LINES + l) * NO + n;
        ecc = std::fmax(ecc, std::fabs(occ[o] - ref));
        etc = std::fmax(etc, std::fabs(otc[o] - ref));
        scale = std::fmax(scale, std::fabs(ref));
      }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float tcc = 0, ttc = 0;
  for (int pass = 0; pass < 2; ++pass)
  {
    CK(cudaEventRecord(e0));
    cc_kernel<K><<<blocks, LINES>>>(P, dsrc, dcc, reps);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&tcc, e0, e1));
    CK(cudaEventRecord(e0));
    tc_kernel<K><<<blocks, LINES>>>(dB, dsrc, dtc, reps);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ttc, e0, e1));
  }
  const double lines = static_cast<double>(blocks) * LINES * reps;
  std::printf("k=%d (NC=%2d -> K %2d, 2 NI=%2d -> N %2d): CUDA cores %7.2f Glines/s (%.3f ms) | tcgen05 3xTF32 %7.2f "
              "Glines/s (%.3f ms) | tc/cc %.2f | max rel err cc %.1e tc %.1e\n",
              K, NC, KP, NO, NP, lines / tcc / 1e6, tcc, lines / ttc / 1e6, ttc, tcc / ttc, ecc / scale, etc / scale);
  cudaFree(dsrc);
  cudaFree(dcc);
  cudaFree(dtc);
  cudaFree(dB);
}

int main(int argc, char **argv)
{
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int blocks = sms * 8, reps = argc > 1 ? std::atoi(argv[1]) : 200;
  std::printf("%d CTAs x %d lines x %d reps per path\n", blocks, LINES, reps);
  run<3>(blocks, reps);
  run<4>(blocks, reps);
  run<5>(blocks, reps);
  run<6>(blocks, reps);
  run<7>(blocks, reps);
  return 0;
}
