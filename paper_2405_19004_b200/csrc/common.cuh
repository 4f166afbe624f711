// Shared device-side definitions of the B200 vertex-patch multigrid library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

namespace pmgb
{

// ---------------------------------------------------------------------------
// errors / launch accounting
// ---------------------------------------------------------------------------

struct CudaError : std::runtime_error
{
  using std::runtime_error::runtime_error;
};

inline void check_cuda(cudaError_t e, const char *what)
{
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void note_launch(int n = 1);       // counts kernel launches (pmg_launch_count)

// smoother kernel organisation (pmg_set_smoother_impl): 0 = per-degree default,
// 1 = line kernel everywhere, 2 = plane-streaming kernel where it exists
enum : int
{
  SMOOTHER_IMPL_AUTO = 0,
  SMOOTHER_IMPL_LINE = 1,
  SMOOTHER_IMPL_PLANE = 2,  // plane kernel, one launch per colour
  SMOOTHER_IMPL_SWEEP = 3,  // plane kernel, all colours in one persistent launch
  SMOOTHER_IMPL_PATCH = 4   // one thread per patch (3D k = 2, 2D k <= 3)
};
int smoother_impl_choice();
void check_launch(const char *what);  // cudaGetLastError + count

// ---------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+): kernels launched with pdl_launch may
// be scheduled while their predecessor in the stream is still draining; each
// such kernel calls pdl_prologue() before touching global memory, which waits
// for the predecessor grid to complete (and its writes to be visible), then
// lets its own successor start launching. Hides the launch gap between the
// 2^d colour sweeps and the short V-cycle kernels.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_prologue()
{
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args)
{
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  check_cuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// true the first time it is called for the current device with this mask
// (per-function attribute setup such as the dynamic shared-memory limit)
inline bool first_on_device(unsigned &mask)
{
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = 1u << (dev & 31);
  if (mask & bit)
    return false;
  mask |= bit;
  return true;
}

// ---------------------------------------------------------------------------
// per-level constant data passed BY VALUE as kernel parameters
// (__grid_constant__). With K a template parameter every matrix entry is a
// compile-time offset into the parameter bank, so the contractions issue
// DFMA/FFMA with uniform-register operands and no shared-memory or
// constant-cache traffic for the 1D matrices.
// ---------------------------------------------------------------------------

template <typename T, int K>
struct PatchMats
{
  static constexpr int NC = 2 * K + 1;  // closure points per direction
  static constexpr int NI = 2 * K - 1;  // interior points per direction
  T M[NI][NC];  // interior rows of the two-cell mass matrix      (fastdiag.hpp:30 mass_if)
  T A[NI][NC];  // interior rows of the two-cell stiffness matrix (fastdiag.hpp:30 stiff_if)
  T S[NI][NI];  // generalized eigenvectors, columns              (fastdiag.hpp:52)
};

// Even-odd form of PatchMats used by the fused kernel. The interior rows of
// the two-cell matrices are centro-symmetric, B[NI-1-i][NC-1-j] = B[i][j]:
//   Be[i][j] = (B[i][j] + B[i][NC-1-j]) / 2 (j < K), Be[i][K] = B[i][K]  (i <= K-1)
//   Bo[i][j] = (B[i][j] - B[i][NC-1-j]) / 2                           (i <  K-1)
// The eigenvectors of the reflection-symmetric patch pencil are even or odd;
// columns are reordered even-first (K even, K-1 odd modes):
//   Se[i][c] = S[i][perm[c]]     (i <= K-1, c <= K-1)
//   So[i][c] = S[i][perm[K+c]]   (i <  K-1, c <  K-1)
template <typename T, int K>
struct PatchMatsEO
{
  static constexpr int HO = K > 1 ? K - 1 : 1;
  T Me[K][K + 1];
  T Mo[HO][K];
  T Ae[K][K + 1];
  T Ao[HO][K];
  T Se[K][K];
  T So[HO][HO];
};

// Rows of the global 1D matrices by lattice residue r = p mod K, offsets
// o = q - p + K in [0, 2K]; the level operator is their Kronecker sum.
template <typename T, int K>
struct BandMats
{
  T M[K][2 * K + 1];
  T A[K][2 * K + 1];
};

// (2K+1) x (K+1) embedding of the coarse cell basis into its two fine cells
// (level_context.cpp:21-34).
template <typename T, int K>
struct ProlMats
{
  T P[2 * K + 1][K + 1];
};

// Smoother modes (one kernel template, four organisations of the reference's
// SmootherVariant, smoother.cpp:61-149).
enum : int
{
  MODE_FUSED = 0,     // residual + solve + x += v          (variant fused)
  MODE_BOUNDARY = 1,  // never reads x^I, x^I = v           (variant boundary)
  MODE_RESIDUAL = 2,  // r^I = b^I - A x, to a global buffer (separate, pass 1)
  MODE_SOLVE = 3      // v = A_j^{-1} r^I from global, x += v (separate pass 2 / global)
};

template <typename T>
struct ColorArgs
{
  T *x;           // level vector (updated)
  const T *b;     // right-hand side
  T *r;           // global residual buffer (MODE_RESIDUAL output / MODE_SOLVE input)
  const T *inv;   // inverse eigenvalue sums, (2K-1)^D, direction 0 fastest
  int64_t m;      // dofs per direction (directions 0 .. d-2)
  int64_t mz;     // dofs along the last direction of the (possibly stacked) global box
  int64_t zoff;   // global last-direction dof index of plane 0 of x / b / r (slab offset)
  int np[3];      // patches of this colour per direction
  int vb[3];      // vertex coordinate v_a = 2 j_a + vb[a]
  int total;      // patches in this colour
  int level_total;  // patches of this colour on the whole unit-cube level: kernel choice
                    // (independent of slab / range restriction, so P slabs dispatch
                    // exactly like one GPU and stay bitwise equal)
  int b_ready;      // b was final before the previous launch of this stream started (a
                    // later colour of the same step): kernels may read it before their
                    // programmatic-dependency wait
};

template <typename T>
struct SweepArgs
{
  ColorArgs<T> c[8];  // per-colour geometry (np, vb); x, b, inv, m shared
  int ntx[8];         // tiles per x-row of colour c
  int start[9];       // first ticket of colour c
  int ncolors;
  int nv;             // vertex planes (counter stride)
  int *sync;          // [0] ticket, [1] exit count, [2 + c nv + v2] finished tiles
};

}  // namespace pmgb
