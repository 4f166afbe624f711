// C-ABI implementation (include/pmg_b200.h): level / multigrid contexts,
// the colour loop of the smoother, the V-cycle, FMG and GMRES drivers.
//
// Host-side control flow mirrors the reference call graph
// (smoother.cpp:41-151, multigrid.cpp:286-400, krylov.cpp:24-171); every
// arithmetic step runs in a CUDA kernel on the context's device. There is no
// CPU fallback: a missing device or a failed launch is an error.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pmg_b200.h"
#include "blas.cuh"
#include "dispatch.hpp"
#include "transfer_impl.cuh"
#include "naive.cuh"
#include "setup.hpp"
#include "capi_internal.hpp"
#include <type_traits>

namespace pmgb
{

namespace
{
std::atomic<int64_t> g_launches{0};
thread_local std::string g_last_error;
}  // namespace

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

std::atomic<int> g_smoother_impl{SMOOTHER_IMPL_AUTO};

// levels with at most this many plane tiles run their 2^d colours as one
// persistent sweep under the default implementation (PMG_SWEEP_AUTO_TILES
// overrides; measurement knob)
int64_t sweep_auto_tiles()
{
  static const int64_t v = [] {
    const char *e = std::getenv("PMG_SWEEP_AUTO_TILES");
    return e ? std::atoll(e) : int64_t(0);
  }();
  return v;
}
int smoother_impl_choice() { return g_smoother_impl.load(std::memory_order_relaxed); }

void check_launch(const char *what)
{
  check_cuda(cudaGetLastError(), what);
  note_launch(1);
}

Tables &tables()
{
  static Tables *t = [] {
    auto *tb = new Tables();
    register_k1(*tb);
    register_k2(*tb);
    register_k3(*tb);
    register_k4(*tb);
    register_k5(*tb);
    register_k6(*tb);
    register_k7(*tb);
    return tb;
  }();
  return *t;
}

struct InvalidArg : std::invalid_argument
{
  using std::invalid_argument::invalid_argument;
};
using Divergence = DivergenceErr;
using DeviceGuard = DevScope;

}  // namespace pmgb

using namespace pmgb;

struct pmg_level_s
{
  LevelSetup S;
  int dtype = PMG_F64;
  int device = 0;
  int sm_count = 148;
  size_t tsize = 8;
  std::vector<unsigned char> patch_mats, band_mats, prol_mats;  // param blobs in T
  DevBuf inv;             // inverse eigenvalue sums (T), reference mode order
  DevBuf inv_eo;          // same, even-first mode order of the fused kernel
  DevBuf resid;           // global residual (global / separate variants)
  DevBuf naive_mats;      // Mif | Aif | S (T) for the straightforward kernel
  DevBuf naive_scratch;
  DevBuf tA, tB;          // transfer scratch (used when this level is the fine one)
  DevBuf sweep_sync;      // ticket / exit / per-(colour, plane) counters of the sweep kernel
  DevBuf red;             // reduction partials + result (double)
  DevBuf io[3];           // staging for the *_host entry points
  cudaStream_t io_stream = nullptr;
  cudaStream_t io_h2d = nullptr, io_d2h = nullptr;  // copy streams of the pipelined *_host smoother
  std::vector<cudaEvent_t> io_ev;                    // its per-chunk events
  std::shared_ptr<GsData> gs;  // point Gauss-Seidel data (gs.cu), built on first use
  ~pmg_level_s()
  {
    // the owner set the level's device (pmg_level_destroy / pmg_mg_destroy)
    for (cudaStream_t st : {io_stream, io_h2d, io_d2h})
      if (st)
        cudaStreamDestroy(st);
    for (cudaEvent_t e : io_ev)
      cudaEventDestroy(e);
  }
};

struct CachedGraph
{
  cudaGraphExec_t exec = nullptr;
  int li = -1;
  void *x = nullptr;
  const void *b = nullptr;
  int variant = -1, pre = -1, post = -1;
  int impl = -1;        // smoother organisation the kernels were captured with
  unsigned gen = ~0u;   // g_buf_generation at capture (workspace pointers)
};

struct pmg_mg_s
{
  std::vector<pmg_level> levels;
  int kind = PMG_VERTEX_PATCH;  // SmootherKind (multigrid.hpp:16-20)
  int dtype = PMG_F64;
  int device = 0;
  int variant = PMG_FUSED;
  int pre = 1, post = 1;
  std::vector<DevBuf *> r_ws, bc_ws, xc_ws;  // per level li (sizes: N_li, N_{li-1}, N_{li-1})
  CachedGraph graph;
  cudaStream_t cap_stream = nullptr;
  // coarse V-cycle operator: the V-cycle of level index mat_li (<= MAT_MAX_N
  // unknowns) from a zero initial guess is a fixed linear map b -> x; its
  // matrix (columns = responses to e_j, computed by running that V-cycle) is
  // applied as one GEMV where the recursion reaches mat_li
  int mat_li = -1;
  bool mat_ready = false;
  unsigned mat_key = 0;
  DevBuf mat, mat_b, mat_x;
  DevBuf fmg_x[32];
  GmresWork gmres;
  ~pmg_mg_s()
  {
    if (graph.exec)
      cudaGraphExecDestroy(graph.exec);
    if (cap_stream)
      cudaStreamDestroy(cap_stream);
    for (auto *b : r_ws)
      delete b;
    for (auto *b : bc_ws)
      delete b;
    for (auto *b : xc_ws)
      delete b;
    for (auto *l : levels)
      delete l;
  }
};

namespace
{

template <typename F>
int guard(F &&f)
{
  return capi_guard(std::forward<F>(f));
}

inline cudaStream_t as_stream(void *s) { return static_cast<cudaStream_t>(s); }

template <typename T>
const KernelTable<T> &ktab(const pmg_level_s *l);
template <>
const KernelTable<double> &ktab<double>(const pmg_level_s *l)
{
  return tables().f64[l->S.dim - 2][l->S.k];
}
template <>
const KernelTable<float> &ktab<float>(const pmg_level_s *l)
{
  return tables().f32[l->S.dim - 2][l->S.k];
}

template <typename T>
std::vector<unsigned char> blob(std::initializer_list<const Dense *> mats)
{
  std::vector<T> v;
  for (const Dense *d : mats)
    for (double a : d->a)
      v.push_back(static_cast<T>(a));
  std::vector<unsigned char> out(v.size() * sizeof(T));
  std::memcpy(out.data(), v.data(), out.size());
  return out;
}

template <typename T>
std::vector<unsigned char> blob_vec(const std::vector<double> &a, const std::vector<double> &b)
{
  std::vector<T> v;
  for (double x : a)
    v.push_back(static_cast<T>(x));
  for (double x : b)
    v.push_back(static_cast<T>(x));
  std::vector<unsigned char> out(v.size() * sizeof(T));
  std::memcpy(out.data(), v.data(), out.size());
  return out;
}

template <typename T>
void upload(DevBuf &buf, const std::vector<double> &host)
{
  std::vector<T> v(host.begin(), host.end());
  buf.ensure(v.size() * sizeof(T));
  check_cuda(cudaMemcpy(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice),
             "upload");
}

template <typename T>
void level_init(pmg_level_s *l)
{
  const auto &S = l->S;
  {
    std::vector<T> v(S.eo_mats.begin(), S.eo_mats.end());
    if (S.k == 1)
    {
      // PointStencil<T> after PatchMatsEO<T,1> (smoother_point.cuh): the 3^d
      // interior row of A-bar = sum over directions of A in one, M in the others
      // (fastdiag.cpp:211-232), and coef = S^(2d) / sum(lambda) (fastdiag.cpp:164-192)
      const double Mr[3] = {S.mass_if(0, 0), S.mass_if(0, 1), S.mass_if(0, 2)};
      const double Ar[3] = {S.stiff_if(0, 0), S.stiff_if(0, 1), S.stiff_if(0, 2)};
      double w[27] = {0};
      for (int t2 = 0; t2 < (S.dim == 3 ? 3 : 1); ++t2)
        for (int t1 = 0; t1 < 3; ++t1)
          for (int t0 = 0; t0 < 3; ++t0)
            w[9 * t2 + 3 * t1 + t0] =
                S.dim == 3 ? Ar[t0] * Mr[t1] * Mr[t2] + Mr[t0] * Ar[t1] * Mr[t2] + Mr[t0] * Mr[t1] * Ar[t2]
                           : Ar[t0] * Mr[t1] + Mr[t0] * Ar[t1];
      const double s = S.S(0, 0);
      double coef = S.inv_sums[0];
      for (int d = 0; d < 2 * S.dim; ++d)
        coef *= s;
      v.insert(v.end(), w, w + 27);
      v.push_back(static_cast<T>(coef));
    }
    // dense interior rows M_if, A_if and eigenvectors S (PatchMats<T,K>) last:
    // the dir-2 contraction of the one-thread-per-patch 3D kernel
    for (const Dense *dm : {&S.mass_if, &S.stiff_if, &S.S})
      v.insert(v.end(), dm->a.begin(), dm->a.end());
    // S^T M_if and S^T A_if (eigen rows in the even-first order): the 3D
    // one-thread-per-patch kernel applies dir 2 and the first S^T in one step
    {
      const int ni = 2 * S.k - 1, nc = 2 * S.k + 1;
      for (const Dense *dm : {&S.mass_if, &S.stiff_if})
        for (int c = 0; c < ni; ++c)
          for (int t = 0; t < nc; ++t)
          {
            double acc = 0.0;
            for (int i = 0; i < ni; ++i)
              acc += S.S(i, S.eo_perm[c]) * (*dm)(i, t);
            v.push_back(static_cast<T>(acc));
          }
    }
    l->patch_mats.resize(v.size() * sizeof(T));
    std::memcpy(l->patch_mats.data(), v.data(), l->patch_mats.size());
  }
  upload<T>(l->inv_eo, S.inv_sums_eo);
  l->band_mats = blob_vec<T>(S.band_mass, S.band_stiff);
  l->prol_mats = blob<T>({&S.prolongation});
  upload<T>(l->inv, S.inv_sums);
  std::vector<double> nm;
  nm.insert(nm.end(), S.mass_if.a.begin(), S.mass_if.a.end());
  nm.insert(nm.end(), S.stiff_if.a.begin(), S.stiff_if.a.end());
  nm.insert(nm.end(), S.S.a.begin(), S.S.a.end());
  upload<T>(l->naive_mats, nm);
  l->red.ensure((RED_BLOCKS + 8) * sizeof(double));
}

// patches of colour `color` (patches.cpp:11-46): v_a in {1,3,..} if bit set else {2,4,..}
template <typename T>
ColorArgs<T> color_args(const pmg_level_s *l, int color, T *x, const T *b)
{
  ColorArgs<T> a{};
  a.x = x;
  a.b = b;
  a.r = l->resid.as<T>();
  a.inv = l->inv_eo.as<T>();
  a.m = l->S.m;
  const int n = l->S.n;
  a.total = 1;
  for (int q = 0; q < 3; ++q)
  {
    if (q < l->S.dim)
    {
      const int bit = (color >> q) & 1;
      a.np[q] = bit ? n / 2 : n / 2 - 1;
      a.vb[q] = bit ? 1 : 2;
    }
    else
    {
      a.np[q] = 1;
      a.vb[q] = 1;
    }
    a.total *= a.np[q];
  }
  a.mz = a.m;
  a.zoff = 0;
  a.level_total = a.total;
  return a;
}

// Colour `color` restricted to the slab of vertex planes vz in [vz_lo, vz_hi]
// (last direction) of a box with nz_cells cells along z (a stacked box when
// nz_cells != n); x / b hold the global dof planes starting at zoff.
template <typename T>
ColorArgs<T> color_args_slab(const pmg_level_s *l, int color, T *x, const T *b, int64_t zoff,
                             int64_t nz_cells, int vz_lo, int vz_hi)
{
  if (l->S.dim != 3)
    throw InvalidArg("slab decomposition is implemented for dim 3");
  if (nz_cells < 2 || vz_lo < 1 || vz_hi > nz_cells - 1 || zoff < 0)
    throw InvalidArg("slab: invalid vertex range / box");
  ColorArgs<T> a = color_args<T>(l, color, x, b);
  const int bit = (color >> 2) & 1;
  int first = vz_lo + (((vz_lo & 1) != bit) ? 1 : 0);
  a.np[2] = first > vz_hi ? 0 : (vz_hi - first) / 2 + 1;
  a.vb[2] = first;
  a.total = a.np[0] * a.np[1] * a.np[2];
  a.mz = nz_cells * l->S.k - 1;
  a.zoff = zoff;
  return a;
}

template <typename T>
void smooth_color_impl(pmg_level_s *l, int variant, int color, T *x, const T *b, cudaStream_t s,
                       bool b_ready = false)
{
  const auto &kt = ktab<T>(l);
  ColorArgs<T> a = color_args<T>(l, color, x, b);
  a.b_ready = b_ready ? 1 : 0;
  if (a.total == 0)
    return;  // smoother.cpp:57-59: empty colours are skipped
  switch (variant)
  {
    case PMG_FUSED:
      kt.smooth(l->patch_mats.data(), a, MODE_FUSED, l->sm_count, s);
      break;
    case PMG_BOUNDARY:
      kt.smooth(l->patch_mats.data(), a, MODE_BOUNDARY, l->sm_count, s);
      break;
    case PMG_SEPARATE:
      l->resid.ensure(static_cast<size_t>(l->S.N) * sizeof(T));
      a.r = l->resid.as<T>();
      kt.smooth(l->patch_mats.data(), a, MODE_RESIDUAL, l->sm_count, s);
      kt.smooth(l->patch_mats.data(), a, MODE_SOLVE, l->sm_count, s);
      break;
    case PMG_GLOBAL:
      l->resid.ensure(static_cast<size_t>(l->S.N) * sizeof(T));
      a.r = l->resid.as<T>();
      kt.level_op(l->band_mats.data(), x, b, a.r, l->S.m, l->sm_count, s);
      kt.smooth(l->patch_mats.data(), a, MODE_SOLVE, l->sm_count, s);
      break;
    case PMG_NAIVE:
    {
      const int grid = l->sm_count * 16;
      const int64_t per = naive_scratch_per_block<T>(l->S.dim, l->S.k);
      l->naive_scratch.ensure(static_cast<size_t>(per) * grid * sizeof(T));
      NaiveArgs<T> na{};
      na.c = a;
      na.c.inv = l->inv.as<T>();
      const int ni = 2 * l->S.k - 1, nc = 2 * l->S.k + 1;
      na.Mif = l->naive_mats.as<T>();
      na.Aif = na.Mif + ni * nc;
      na.S = na.Aif + ni * nc;
      na.dim = l->S.dim;
      na.k = l->S.k;
      na.scratch = l->naive_scratch.as<T>();
      na.scratch_stride = per;
      launch_naive_smooth<T>(na, grid, s);
      break;
    }
    default:
      throw InvalidArg("smooth: unknown variant " + std::to_string(variant));
  }
}

template <typename T>
void smooth_color_slab_impl(pmg_level_s *l, int variant, int color, T *x, const T *b, int64_t zoff,
                            int64_t nz_cells, int vz_lo, int vz_hi, cudaStream_t s)
{
  ColorArgs<T> a = color_args_slab<T>(l, color, x, b, zoff, nz_cells, vz_lo, vz_hi);
  if (a.total == 0)
    return;
  const auto &kt = ktab<T>(l);
  if (variant == PMG_FUSED)
    kt.smooth(l->patch_mats.data(), a, MODE_FUSED, l->sm_count, s);
  else if (variant == PMG_BOUNDARY)
    kt.smooth(l->patch_mats.data(), a, MODE_BOUNDARY, l->sm_count, s);
  else
    throw InvalidArg("slab smoother: fused or boundary variant only");
}

// one persistent launch for all colours of a step (smoother_plane.cuh
// vp_sweep_plane_kernel), when this (dim, degree, variant) has one
template <typename T>
bool sweep_impl(pmg_level_s *l, int variant, T *x, const T *b, cudaStream_t s)
{
  const int impl = smoother_impl_choice();
  // measured slower than per-colour launches on large levels (per-tile
  // ticket / counter traffic outweighs the saved tails):
  // opt-in, or automatic on levels of at most sweep_auto_tiles() tiles
  if (!(impl == SMOOTHER_IMPL_SWEEP || impl == SMOOTHER_IMPL_AUTO) || l->S.dim != 3 ||
      !(variant == PMG_FUSED || variant == PMG_BOUNDARY))
    return false;
  const auto &kt = ktab<T>(l);
  if (!kt.sweep || kt.sweep_pb <= 0)
    return false;
  if (impl == SMOOTHER_IMPL_AUTO)
  {
    int64_t tiles = 0;
    for (int c = 0; c < (1 << l->S.dim); ++c)
    {
      const ColorArgs<T> a = color_args<T>(l, c, x, b);
      tiles += static_cast<int64_t>((a.np[0] + kt.sweep_pb - 1) / kt.sweep_pb) * a.np[1] * a.np[2];
    }
    if (tiles > sweep_auto_tiles())
      return false;
  }
  SweepArgs<T> sw{};
  sw.ncolors = 1 << l->S.dim;
  sw.nv = l->S.n + 1;
  sw.start[0] = 0;
  for (int c = 0; c < sw.ncolors; ++c)
  {
    sw.c[c] = color_args<T>(l, c, x, b);
    sw.ntx[c] = (sw.c[c].np[0] + kt.sweep_pb - 1) / kt.sweep_pb;
    sw.start[c + 1] = sw.start[c] + sw.ntx[c] * sw.c[c].np[1] * sw.c[c].np[2];
  }
  const size_t need = static_cast<size_t>(2 + sw.ncolors * sw.nv) * sizeof(int);
  if (l->sweep_sync.bytes < need)
  {
    // zeroed now, not on `s`: `s` may be a capture stream whose first graph
    // is discarded after an allocation (vcycle_entry), and the kernel keeps
    // the counters at zero between launches itself
    l->sweep_sync.ensure(need);
    cudaStream_t z = nullptr;
    check_cuda(cudaStreamCreateWithFlags(&z, cudaStreamNonBlocking), "stream");
    check_cuda(cudaMemsetAsync(l->sweep_sync.p, 0, need, z), "sweep counters");
    check_cuda(cudaStreamSynchronize(z), "sweep counters");
    cudaStreamDestroy(z);
  }
  sw.sync = l->sweep_sync.as<int>();
  return kt.sweep(l->patch_mats.data(), sw, variant == PMG_FUSED ? MODE_FUSED : MODE_BOUNDARY, l->sm_count, s);
}

inline bool b_prefetch_enabled()
{
  static const bool v = [] {
    const char *e = std::getenv("PMG_B_PREFETCH");
    return !(e && e[0] == '0');
  }();
  return v;
}

template <typename T>
void smooth_impl(pmg_level_s *l, int variant, T *x, const T *b, cudaStream_t s)
{
  if (sweep_impl<T>(l, variant, x, b, s))
    return;
  // after the first launch of the step b is final (no kernel of the step
  // writes it): the later colours may prefetch it before their PDL wait
  bool launched = false;
  for (int color = 0; color < (1 << l->S.dim); ++color)
  {
    smooth_color_impl<T>(l, variant, color, x, b, s,
                         launched && b_prefetch_enabled() && (variant == PMG_FUSED || variant == PMG_BOUNDARY));
    launched = launched || color_args<T>(l, color, x, b).total > 0;
  }
}

void check_pair(const pmg_level_s *c, const pmg_level_s *f, const char *what)
{
  if (!c || !f)
    throw InvalidArg(std::string(what) + ": null level");
  if (f->S.level != c->S.level + 1 || f->S.k != c->S.k || f->S.dim != c->S.dim ||
      f->dtype != c->dtype || f->device != c->device)
    throw InvalidArg(std::string(what) + ": levels are not consecutive");
}

template <typename T>
void transfer_scratch(pmg_level_s *fine)
{
  const int64_t mf = fine->S.m, mc = (mf - 1) / 2;
  const int64_t need = fine->S.dim == 3 ? mf * mf * mc : mf * mc;
  fine->tA.ensure(static_cast<size_t>(need) * sizeof(T));
  fine->tB.ensure(static_cast<size_t>(need) * sizeof(T));
}

template <typename T>
void prolongate_impl(pmg_level_s *c, pmg_level_s *f, const T *xc, T *xf, bool acc, cudaStream_t s)
{
  transfer_scratch<T>(f);
  ktab<T>(f).prolongate(f->prol_mats.data(), xc, xf, acc, c->S.m, f->tA.as<T>(), f->tB.as<T>(),
                        f->sm_count, s);
}

template <typename T>
void restrict_impl(pmg_level_s *c, pmg_level_s *f, const T *rf, T *rc, cudaStream_t s, T *zero = nullptr)
{
  transfer_scratch<T>(f);
  ktab<T>(f).restrict_(f->prol_mats.data(), rf, rc, zero, c->S.m, f->tA.as<T>(), f->tB.as<T>(),
                       f->sm_count, s);
}

template <typename T>
double norm_impl(pmg_level_s *l, const T *v, int64_t n, cudaStream_t s)
{
  double *red = l->red.as<double>();
  launch_dot<T>(v, v, n, red, red + RED_BLOCKS, true, s);
  double out = 0;
  check_cuda(cudaMemcpyAsync(&out, red + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, s),
             "norm D2H");
  check_cuda(cudaStreamSynchronize(s), "norm sync");
  return out;
}

// apply_smoother (multigrid.cpp:286-300): the patch smoother, or one
// lexicographic point Gauss-Seidel sweep (f64 only) for kind == point_gs
template <typename T>
void apply_smoother(pmg_mg_s *mg, pmg_level_s *lev, T *x, const T *b, cudaStream_t s)
{
  if (mg->kind == PMG_POINT_GS)
  {
    if constexpr (std::is_same_v<T, double>)
      gs_smooth(lev, x, b, s);
    else
      throw std::logic_error("point Gauss-Seidel requires f64");
    return;
  }
  smooth_impl<T>(lev, mg->variant, x, b, s);
}

template <typename T>
void vcycle_impl(pmg_mg_s *mg, int li, T *x, const T *b, cudaStream_t s);

// what the coarse matrix depends on: smoother organisation, variant, sweeps
unsigned coarse_mat_key(const pmg_mg_s *mg)
{
  return static_cast<unsigned>(smoother_impl_choice()) | (static_cast<unsigned>(mg->variant & 0xff) << 4) |
         (static_cast<unsigned>(mg->pre & 0xff) << 12) | (static_cast<unsigned>(mg->post & 0xff) << 20);
}

// row pitch of the coarse operator (16-byte rows for the GEMV's vector loads)
inline int coarse_mat_ld(int n) { return (n + 3) & ~3; }

// the V-cycle of level index li with a ZERO initial guess (the recursion's
// coarse correction, multigrid.cpp:335-338): one GEMV with the precomputed
// operator on the coarse-matrix level, the recursive cycle otherwise
template <typename T>
void coarse_correction(pmg_mg_s *mg, int li, T *x, const T *b, cudaStream_t s)
{
  if (li == mg->mat_li && mg->mat_ready && mg->mat_key == coarse_mat_key(mg))
  {
    const int n = static_cast<int>(mg->levels[li]->S.N);
    launch_coarse_gemv<T>(mg->mat.as<T>(), b, x, n, coarse_mat_ld(n), s);
    return;
  }
  vcycle_impl<T>(mg, li, x, b, s);
}

// (re)build the coarse operator eagerly (never inside a stream capture): N
// V-cycles on the unit vectors, column j = V(e_j)
template <typename T>
void ensure_coarse_matrix(pmg_mg_s *mg, cudaStream_t s, bool for_finest = false)
{
  if (mg->mat_li < 0)
    return;
  // on the finest level only a coarse correction from outside uses it
  if (mg->mat_li == static_cast<int>(mg->levels.size()) - 1 && !for_finest)
    return;
  const unsigned key = coarse_mat_key(mg);
  if (mg->mat_ready && mg->mat_key == key)
    return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  check_cuda(cudaStreamIsCapturing(s, &cs), "capture status");
  if (cs != cudaStreamCaptureStatusNone)
    return;  // not ready: the recursion is used (consistent within this call)
  const int n = static_cast<int>(mg->levels[mg->mat_li]->S.N);
  mg->mat_ready = false;
  const int ld = coarse_mat_ld(n);
  mg->mat.ensure(static_cast<size_t>(n) * ld * sizeof(T));
  mg->mat_b.ensure(static_cast<size_t>(n) * sizeof(T));
  mg->mat_x.ensure(static_cast<size_t>(n) * sizeof(T) + 16);
  T *M = mg->mat.as<T>(), *eb = mg->mat_b.as<T>(), *ex = mg->mat_x.as<T>();
  int *col = reinterpret_cast<int *>(ex + n);  // column counter after x (16 B slack)
  // one column step (e_j, V-cycle from 0, store, ++j) captured once and
  // replayed n times
  check_cuda(cudaMemsetAsync(col, 0, sizeof(int), s), "column counter");
  check_cuda(cudaMemsetAsync(M, 0, static_cast<size_t>(n) * ld * sizeof(T), s), "coarse matrix pad");
  check_cuda(cudaStreamSynchronize(s), "coarse matrix");
  if (!mg->cap_stream)
    check_cuda(cudaStreamCreateWithFlags(&mg->cap_stream, cudaStreamNonBlocking), "stream");
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  check_cuda(cudaStreamBeginCapture(mg->cap_stream, cudaStreamCaptureModeRelaxed), "capture begin");
  try
  {
    launch_unit_dev<T>(eb, n, col, mg->cap_stream);
    launch_fill<T>(ex, n, T(0), mg->levels[mg->mat_li]->sm_count, mg->cap_stream);
    vcycle_impl<T>(mg, mg->mat_li, ex, eb, mg->cap_stream);
    launch_store_column<T>(M, ex, n, ld, col, mg->cap_stream);
  }
  catch (...)
  {
    cudaStreamEndCapture(mg->cap_stream, &graph);
    if (graph)
      cudaGraphDestroy(graph);
    throw;
  }
  check_cuda(cudaStreamEndCapture(mg->cap_stream, &graph), "capture end");
  check_cuda(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
  for (int j = 0; j < n; ++j)
    check_cuda(cudaGraphLaunch(exec, mg->cap_stream), "graph launch");
  check_cuda(cudaStreamSynchronize(mg->cap_stream), "coarse matrix");
  cudaGraphExecDestroy(exec);
  mg->mat_key = key;
  mg->mat_ready = true;
}

template <typename T>
void vcycle_impl(pmg_mg_s *mg, int li, T *x, const T *b, cudaStream_t s)
{
  pmg_level_s *lev = mg->levels[li];
  if (li == 0)
  {
    // coarse_solve (multigrid.cpp:304-309): x = 0, one fused step is exact
    launch_fill<T>(x, lev->S.N, T(0), lev->sm_count, s);
    smooth_impl<T>(lev, PMG_FUSED, x, b, s);
    return;
  }
  pmg_level_s *crs = mg->levels[li - 1];
  for (int i = 0; i < mg->pre; ++i)
    apply_smoother<T>(mg, lev, x, b, s);
  T *r = mg->r_ws[li]->as<T>();
  T *bc = mg->bc_ws[li]->as<T>();
  T *xc = mg->xc_ws[li]->as<T>();
  ktab<T>(lev).level_op(lev->band_mats.data(), x, b, r, lev->S.m, lev->sm_count, s);
  // b_c = R r and x_c = 0 in the same launch (the coarse solve zeroes x itself)
  restrict_impl<T>(crs, lev, r, bc, s, li - 1 > 0 ? xc : nullptr);
  coarse_correction<T>(mg, li - 1, xc, bc, s);
  prolongate_impl<T>(crs, lev, xc, x, true, s);
  for (int i = 0; i < mg->post; ++i)
    apply_smoother<T>(mg, lev, x, b, s);
}

template <typename T>
void vcycle_entry(pmg_mg_s *mg, int li, T *x, const T *b, bool use_graph, cudaStream_t s)
{
  ensure_coarse_matrix<T>(mg, s);
  if (!use_graph)
  {
    vcycle_impl<T>(mg, li, x, b, s);
    return;
  }
  CachedGraph &g = mg->graph;
  // the key covers everything the captured launches baked in: vectors, level,
  // variant, sweep counts, smoother organisation and workspace pointers
  if (!(g.exec && g.li == li && g.x == x && g.b == b && g.variant == mg->variant &&
        g.pre == mg->pre && g.post == mg->post && g.impl == smoother_impl_choice() &&
        g.gen == g_buf_generation.load(std::memory_order_relaxed)))
  {
    if (g.exec)
    {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    if (!mg->cap_stream)
      check_cuda(cudaStreamCreateWithFlags(&mg->cap_stream, cudaStreamNonBlocking), "stream");
    // the capture stream is not ordered after the caller's stream
    check_cuda(cudaStreamSynchronize(s), "graph pre-sync");
    // a workspace (re)allocated while capturing (first use of a level) may
    // invalidate pointers captured before it: capture again with the sizes
    // settled (the second pass allocates nothing)
    for (int pass = 0; pass < 2; ++pass)
    {
      const unsigned gen0 = g_buf_generation.load(std::memory_order_relaxed);
      cudaGraph_t graph = nullptr;
      check_cuda(cudaStreamBeginCapture(mg->cap_stream, cudaStreamCaptureModeRelaxed), "capture begin");
      try
      {
        vcycle_impl<T>(mg, li, x, b, mg->cap_stream);
      }
      catch (...)
      {
        cudaStreamEndCapture(mg->cap_stream, &graph);
        if (graph)
          cudaGraphDestroy(graph);
        throw;
      }
      check_cuda(cudaStreamEndCapture(mg->cap_stream, &graph), "capture end");
      if (g_buf_generation.load(std::memory_order_relaxed) != gen0 && pass == 0)
      {
        cudaGraphDestroy(graph);
        continue;
      }
      check_cuda(cudaGraphInstantiate(&g.exec, graph, 0), "graph instantiate");
      cudaGraphDestroy(graph);
      break;
    }
    g.impl = smoother_impl_choice();
    g.gen = g_buf_generation.load(std::memory_order_relaxed);
    g.li = li;
    g.x = x;
    g.b = b;
    g.variant = mg->variant;
    g.pre = mg->pre;
    g.post = mg->post;
  }
  check_cuda(cudaGraphLaunch(g.exec, s), "graph launch");
}

pmg_level_s *make_level(int dim, int k, int level, int dtype, int device)
{
  if (dtype != PMG_F64 && dtype != PMG_F32)
    throw InvalidArg("dtype must be PMG_F64 or PMG_F32");
  int ndev = 0;
  check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev)
    throw InvalidArg("no such CUDA device " + std::to_string(device));
  auto l = std::make_unique<pmg_level_s>();
  l->S = make_level_setup(dim, k, level);
  l->dtype = dtype;
  l->device = device;
  l->tsize = dtype == PMG_F64 ? 8 : 4;
  DeviceGuard dg(device);
  check_cuda(cudaDeviceGetAttribute(&l->sm_count, cudaDevAttrMultiProcessorCount, device), "attr");
  if (dtype == PMG_F64)
    level_init<double>(l.get());
  else
    level_init<float>(l.get());
  return l.release();
}

void require_level(pmg_level h)
{
  if (!h)
    throw InvalidArg("null level handle");
}

struct HostIO
{
  pmg_level_s *l;
  explicit HostIO(pmg_level_s *lv) : l(lv)
  {
    if (!l->io_stream)
      check_cuda(cudaStreamCreateWithFlags(&l->io_stream, cudaStreamNonBlocking), "stream");
  }
  void *dev(int i, size_t bytes)
  {
    l->io[i].ensure(bytes);
    return l->io[i].p;
  }
  void h2d(void *d, const void *h, size_t b)
  {
    check_cuda(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, l->io_stream), "H2D");
  }
  void d2h(void *h, const void *d, size_t b)
  {
    check_cuda(cudaMemcpyAsync(h, d, b, cudaMemcpyDeviceToHost, l->io_stream), "D2H");
  }
  void sync() { check_cuda(cudaStreamSynchronize(l->io_stream), "sync"); }
};

#define PMG_DISPATCH_T(lvl, CALL)  \
  do                               \
  {                                \
    if ((lvl)->dtype == PMG_F64)   \
    {                              \
      using T = double;            \
      CALL;                        \
    }                              \
    else                           \
    {                              \
      using T = float;             \
      CALL;                        \
    }                              \
  } while (0)

}  // namespace

namespace pmgb
{

int capi_status_from_current_exception()
{
  try
  {
    throw;
  }
  catch (const std::invalid_argument &e)
  {
    g_last_error = e.what();
    return PMG_ERR_INVALID;
  }
  catch (const DivergenceErr &e)
  {
    g_last_error = e.what();
    return PMG_ERR_DIVERGENCE;
  }
  catch (const CudaError &e)
  {
    g_last_error = e.what();
    return PMG_ERR_CUDA;
  }
  catch (const std::exception &e)
  {
    g_last_error = e.what();
    return PMG_ERR_RUNTIME;
  }
  catch (...)
  {
    g_last_error = "unknown exception";
    return PMG_ERR_RUNTIME;
  }
}

void GmresWork::ensure(int64_t n, int restart, bool mixed)
{
  bV.ensure(static_cast<size_t>(n) * (restart + 1) * sizeof(double));
  bZ.ensure(static_cast<size_t>(n) * restart * sizeof(double));
  bw.ensure(static_cast<size_t>(n) * sizeof(double));
  br.ensure(static_cast<size_t>(n) * sizeof(double));
  bred.ensure((RED_BLOCKS + 8) * sizeof(double));
  bflag.ensure(sizeof(int));
  if (mixed)
  {
    brf.ensure(static_cast<size_t>(n) * sizeof(float));
    bzf.ensure(static_cast<size_t>(n) * sizeof(float));
  }
  V = bV.as<double>();
  Z = bZ.as<double>();
  w = bw.as<double>();
  r = br.as<double>();
  red = bred.as<double>();
  rf = brf.as<float>();
  zf = bzf.as<float>();
  flag = bflag.as<int>();
}

std::shared_ptr<GsData> &level_gs_slot(pmg_level l) { return l->gs; }
const LevelSetup &level_setup(pmg_level l) { return l->S; }
int level_dtype(pmg_level l) { return l->dtype; }
int level_device(pmg_level l) { return l->device; }
int mg_dtype(pmg_mg h) { return h->dtype; }
int mg_device(pmg_mg h) { return h->device; }
int mg_levels(pmg_mg h) { return static_cast<int>(h->levels.size()); }
pmg_level mg_level_ptr(pmg_mg h, int li) { return h->levels[li]; }
int64_t level_total(pmg_level l) { return l->S.N; }
int level_sm_count(pmg_level l) { return l->sm_count; }
void level_params(pmg_level l, int *dim, int *k, int *level, int *dtype, int *device)
{
  *dim = l->S.dim;
  *k = l->S.k;
  *level = l->S.level;
  *dtype = l->dtype;
  *device = l->device;
}
GmresWork &mg_gmres_work(pmg_mg h) { return h->gmres; }

void mg_apply_finest_op(pmg_mg h, const double *x, double *y, cudaStream_t s)
{
  pmg_level_s *l = h->levels.back();
  ktab<double>(l).level_op(l->band_mats.data(), x, nullptr, y, l->S.m, l->sm_count, s);
}

void mg_residual_finest(pmg_mg h, const double *x, const double *b, double *r, cudaStream_t s)
{
  pmg_level_s *l = h->levels.back();
  ktab<double>(l).level_op(l->band_mats.data(), x, b, r, l->S.m, l->sm_count, s);
}

void mg_vcycle_f32(pmg_mg h, int li, float *x, const float *b, cudaStream_t s)
{
  ensure_coarse_matrix<float>(h, s);
  vcycle_impl<float>(h, li, x, b, s);
}

void mg_vcycle_f64(pmg_mg h, int li, double *x, const double *b, cudaStream_t s)
{
  ensure_coarse_matrix<double>(h, s);
  vcycle_impl<double>(h, li, x, b, s);
}

void mg_coarse_correction(pmg_mg h, int li, void *x, const void *b, bool use_graph, cudaStream_t s)
{
  DevScope dg(h->device);
  if (h->dtype == PMG_F64)
  {
    ensure_coarse_matrix<double>(h, s, true);
    if (li == h->mat_li && h->mat_ready)
      coarse_correction<double>(h, li, static_cast<double *>(x), static_cast<const double *>(b), s);
    else
      vcycle_entry<double>(h, li, static_cast<double *>(x), static_cast<const double *>(b), use_graph, s);
  }
  else
  {
    ensure_coarse_matrix<float>(h, s, true);
    if (li == h->mat_li && h->mat_ready)
      coarse_correction<float>(h, li, static_cast<float *>(x), static_cast<const float *>(b), s);
    else
      vcycle_entry<float>(h, li, static_cast<float *>(x), static_cast<const float *>(b), use_graph, s);
  }
}

}  // namespace pmgb

// ---- slab entry points (3D slab domain decomposition, dd.py) ------------------
namespace
{
void require_planes(const char *what, int64_t zoff, int64_t np, int64_t lo, int64_t hi, int64_t m)
{
  // global planes [lo, hi) clipped to the domain must lie in [zoff, zoff + np)
  lo = std::max<int64_t>(lo, 0);
  hi = std::min<int64_t>(hi, m);
  if (lo < hi && (lo < zoff || hi > zoff + np))
    throw InvalidArg(std::string(what) + ": slab does not hold the planes the requested outputs depend on");
}

template <typename T>
const T *shift(const void *p, int64_t zoff, int64_t plane)
{
  return static_cast<const T *>(p) - zoff * plane;
}
template <typename T>
T *shift(void *p, int64_t zoff, int64_t plane)
{
  return static_cast<T *>(p) - zoff * plane;
}
}  // namespace

namespace
{
// ---- the *_host smoother as a copy / compute pipeline ----------------------
// pmg_smooth_host moves 2 N words in and N out over PCIe for a step whose
// kernels take a fraction of that time. The step runs as a skewed wavefront
// over the patch-vertex planes of the slowest direction: at pipeline step t
// colour c covers the vertex planes (B[t-1] - c, B[t] - c] (B[t] - B[t-1] per
// step, shrinking towards the end). The colour-to-colour dependencies reach
// one vertex plane, so colour c at step t sees colour c - 1 already applied on
// its planes +- 1 (same step, earlier launch) and colour c + 1 not yet applied
// (it trails by one plane):
// every patch is computed exactly as in pmg_smooth, bitwise. x / b planes go
// H2D on one stream just ahead of colour 0; the planes whose last writer
// (colour 7 of vertex planes <= t w - 7) is done go D2H on another, so both
// transfer directions and the kernels overlap.
int host_pipeline_chunks(const pmg_level_s *l, int variant)
{
  static const int forced = [] {
    const char *e = std::getenv("PMG_HOST_PIPELINE");  // 0: off, n: n steps of vertex planes
    return e ? std::atoi(e) : -1;
  }();
  if (l->S.dim != 3 || !(variant == PMG_FUSED || variant == PMG_BOUNDARY) || forced == 0)
    return 1;
  const int nv = l->S.n - 1;
  if (forced > 0)
    return std::max(1, std::min(forced, nv / 2));
  if (l->S.N < (int64_t(1) << 20))
    return 1;  // launch latency would dominate the saved transfer time
  return std::max(1, std::min(4, nv / 4));
}

template <typename T>
void smooth_host_pipelined(pmg_level_s *l, int variant, T *hx, const T *hb, T *dx, T *db)
{
  const int nv = l->S.n - 1, k = l->S.k, ncol = 1 << l->S.dim;
  // colour 0 reaches vertex plane B[t] at step t; colour ncol-1 trails by
  // ncol-1 planes, so B[steps] = nv + ncol - 1. Steps shrink linearly: the
  // work left after the last H2D chunk (its 2^d dependent launches and the
  // D2H of the trailing planes) is the pipeline's tail.
  const int steps = std::max(1, std::min(host_pipeline_chunks(l, variant), nv));
  std::vector<int> B(steps + 1, 0);
  {
    const int64_t span = nv + ncol - 1, wsum = static_cast<int64_t>(steps) * (steps + 1) / 2;
    int64_t acc = 0;
    for (int t = 1; t <= steps; ++t)
    {
      acc += steps - t + 1;
      B[t] = static_cast<int>((span * acc + wsum - 1) / wsum);
    }
    B[steps] = static_cast<int>(span);
  }
  const int64_t m = l->S.m, pl = m * m;
  if (!l->io_h2d)
    check_cuda(cudaStreamCreateWithFlags(&l->io_h2d, cudaStreamNonBlocking), "stream");
  if (!l->io_d2h)
    check_cuda(cudaStreamCreateWithFlags(&l->io_d2h, cudaStreamNonBlocking), "stream");
  while (static_cast<int>(l->io_ev.size()) < 2 * steps + 1)
  {
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    l->io_ev.push_back(e);
  }
  cudaEvent_t *ev_in = l->io_ev.data(), *ev_out = l->io_ev.data() + steps, ev_prev = l->io_ev[2 * steps];
  // after everything earlier on the compute stream (previous users of dx / db)
  check_cuda(cudaEventRecord(ev_prev, l->io_stream), "event");
  check_cuda(cudaStreamWaitEvent(l->io_h2d, ev_prev, 0), "wait");
  check_cuda(cudaStreamWaitEvent(l->io_d2h, ev_prev, 0), "wait");
  int64_t in_done = 0, out_done = 0;  // dof planes [0, in_done) sent, [0, out_done) returned
  // PMG_HOST_PIPELINE_TRACE=1: per-stream event timeline on stderr (diagnostics)
  static const bool trace = std::getenv("PMG_HOST_PIPELINE_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> tr;
  auto mark = [&](const std::string &name, cudaStream_t st) {
    if (!trace)
      return;
    cudaEvent_t e;
    check_cuda(cudaEventCreate(&e), "event");
    check_cuda(cudaEventRecord(e, st), "event");
    tr.push_back({name, e});
  };
  mark("start", l->io_h2d);
  for (int t = 1; t <= steps; ++t)
  {
    // colour 0 at step t covers vertex planes up to B[t]: its closures read
    // dof planes below k (B[t] + 1)
    const int64_t need = std::min<int64_t>(m, static_cast<int64_t>(k) * (static_cast<int64_t>(B[t]) + 1));
    if (need > in_done)
    {
      const size_t off = static_cast<size_t>(in_done * pl), cnt = static_cast<size_t>((need - in_done) * pl);
      check_cuda(cudaMemcpyAsync(dx + off, hx + off, cnt * sizeof(T), cudaMemcpyHostToDevice, l->io_h2d), "H2D");
      check_cuda(cudaMemcpyAsync(db + off, hb + off, cnt * sizeof(T), cudaMemcpyHostToDevice, l->io_h2d), "H2D");
      in_done = need;
      mark("h2d " + std::to_string(t), l->io_h2d);
    }
    check_cuda(cudaEventRecord(ev_in[t - 1], l->io_h2d), "event");
    check_cuda(cudaStreamWaitEvent(l->io_stream, ev_in[t - 1], 0), "wait");
    for (int color = 0; color < ncol; ++color)
    {
      const int hi = std::min(nv, B[t] - color), lo = std::max(1, B[t - 1] - color + 1);
      if (lo <= hi)
        smooth_color_slab_impl<T>(l, variant, color, dx, db, 0, l->S.n, lo, hi, l->io_stream);
    }
    mark("compute " + std::to_string(t), l->io_stream);
    // planes whose writers (patches v with v <= p / k + 1) all finished colour
    // ncol - 1: p < k V with V = B[t] - (ncol - 1)
    const int V = B[t] - (ncol - 1);
    const int64_t fin = t == steps ? m : std::min<int64_t>(m, static_cast<int64_t>(k) * std::max(0, V));
    if (fin > out_done)
    {
      check_cuda(cudaEventRecord(ev_out[t - 1], l->io_stream), "event");
      check_cuda(cudaStreamWaitEvent(l->io_d2h, ev_out[t - 1], 0), "wait");
      const size_t off = static_cast<size_t>(out_done * pl), cnt = static_cast<size_t>((fin - out_done) * pl);
      check_cuda(cudaMemcpyAsync(hx + off, dx + off, cnt * sizeof(T), cudaMemcpyDeviceToHost, l->io_d2h), "D2H");
      out_done = fin;
      mark("d2h " + std::to_string(t), l->io_d2h);
    }
  }
  check_cuda(cudaStreamSynchronize(l->io_d2h), "sync");
  if (trace)
  {
    check_cuda(cudaDeviceSynchronize(), "sync");
    for (size_t i = 1; i < tr.size(); ++i)
    {
      float ms = 0;
      cudaEventElapsedTime(&ms, tr[0].second, tr[i].second);
      std::fprintf(stderr, "  %-12s %8.3f ms\n", tr[i].first.c_str(), ms);
    }
    for (auto &e : tr)
      cudaEventDestroy(e.second);
  }
}
}  // namespace

extern "C" {

const char *pmg_last_error(void) { return g_last_error.c_str(); }

int pmg_version(void) { return 1; }

int64_t pmg_launch_count(void) { return g_launches.load(); }

int pmg_set_smoother_impl(int impl)
{
  if (impl < SMOOTHER_IMPL_AUTO || impl > SMOOTHER_IMPL_PATCH)
  {
    g_last_error = "pmg_set_smoother_impl: impl must be 0 .. 4";
    return PMG_ERR_INVALID;
  }
  g_smoother_impl.store(impl);
  return PMG_OK;
}

int pmg_get_smoother_impl(void) { return g_smoother_impl.load(); }

int pmg_device_info(int device, int *sm_count, int *sm_clock_khz, int *cc_major, int *cc_minor)
{
  return guard([&] {
    check_cuda(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device), "attr");
    check_cuda(cudaDeviceGetAttribute(sm_clock_khz, cudaDevAttrClockRate, device), "attr");
    check_cuda(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device), "attr");
    check_cuda(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device), "attr");
  });
}

int pmg_level_create(int dim, int degree, int level, int dtype, int device, pmg_level *out)
{
  return guard([&] {
    if (!out)
      throw InvalidArg("null output handle");
    *out = make_level(dim, degree, level, dtype, device);
  });
}

int pmg_level_destroy(pmg_level h)
{
  return guard([&] {
    if (h)
    {
      DeviceGuard dg(h->device);
      delete h;
    }
  });
}

int pmg_level_info(pmg_level h, int64_t *m, int64_t *N, int64_t *patches)
{
  return guard([&] {
    require_level(h);
    if (m)
      *m = h->S.m;
    if (N)
      *N = h->S.N;
    if (patches)
    {
      int64_t p = 1;
      for (int a = 0; a < h->S.dim; ++a)
        p *= (h->S.n - 1);
      *patches = p;
    }
  });
}

int pmg_level_setup_data(pmg_level h, double *S, double *lambda, double *mass_if, double *stiff_if,
                         double *prolongation, double *cell_mass, double *cell_stiffness)
{
  return guard([&] {
    require_level(h);
    auto cp = [](double *dst, const std::vector<double> &v) {
      if (dst)
        std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(S, h->S.S.a);
    cp(lambda, h->S.lambda);
    cp(mass_if, h->S.mass_if.a);
    cp(stiff_if, h->S.stiff_if.a);
    cp(prolongation, h->S.prolongation.a);
    cp(cell_mass, h->S.cell_mass.a);
    cp(cell_stiffness, h->S.cell_stiff.a);
  });
}

int pmg_host_level_setup(int dim, int degree, int level, double *S, double *lambda,
                         double *mass_if, double *stiff_if, double *prolongation, double *cell_mass,
                         double *cell_stiffness, double *band_mass, double *band_stiff, int *eo_perm)
{
  return guard([&] {
    const LevelSetup s = make_level_setup(dim, degree, level);
    auto cp = [](double *dst, const std::vector<double> &v) {
      if (dst)
        std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(S, s.S.a);
    cp(lambda, s.lambda);
    cp(mass_if, s.mass_if.a);
    cp(stiff_if, s.stiff_if.a);
    cp(prolongation, s.prolongation.a);
    cp(cell_mass, s.cell_mass.a);
    cp(cell_stiffness, s.cell_stiff.a);
    cp(band_mass, s.band_mass);
    cp(band_stiff, s.band_stiff);
    if (eo_perm)
      std::memcpy(eo_perm, s.eo_perm.data(), s.eo_perm.size() * sizeof(int));
  });
}

int pmg_smooth(pmg_level h, int variant, void *x, const void *b, void *stream)
{
  return guard([&] {
    require_level(h);
    DeviceGuard dg(h->device);
    PMG_DISPATCH_T(h, smooth_impl<T>(h, variant, static_cast<T *>(x), static_cast<const T *>(b),
                                     as_stream(stream)));
  });
}

int pmg_smooth_color(pmg_level h, int variant, int color, void *x, const void *b, void *stream)
{
  return guard([&] {
    require_level(h);
    if (color < 0 || color >= (1 << h->S.dim))
      throw InvalidArg("colour out of range");
    DeviceGuard dg(h->device);
    PMG_DISPATCH_T(h, smooth_color_impl<T>(h, variant, color, static_cast<T *>(x),
                                           static_cast<const T *>(b), as_stream(stream)));
  });
}

int pmg_smoother_kernel(pmg_level h, int variant, int color, int *kernel)
{
  return guard([&] {
    require_level(h);
    if (!kernel || color < 0 || color >= (1 << h->S.dim))
      throw InvalidArg("smoother_kernel: invalid arguments");
    if (variant == PMG_NAIVE)
    {
      *kernel = PMG_KERNEL_NAIVE;
      return;
    }
    const int mode = variant == PMG_FUSED ? MODE_FUSED : variant == PMG_BOUNDARY ? MODE_BOUNDARY : MODE_SOLVE;
    PMG_DISPATCH_T(h, {
      const ColorArgs<T> a = color_args<T>(h, color, static_cast<T *>(nullptr), static_cast<const T *>(nullptr));
      *kernel = ktab<T>(h).smooth_kernel(a, mode);
    });
  });
}

int pmg_smooth_color_slab(pmg_level h, int variant, int color, void *x_local, const void *b_local,
                          int64_t z_offset, int64_t nz_cells, int vz_lo, int vz_hi, void *stream)
{
  return guard([&] {
    require_level(h);
    if (color < 0 || color >= (1 << h->S.dim))
      throw InvalidArg("colour out of range");
    DeviceGuard dg(h->device);
    PMG_DISPATCH_T(h, smooth_color_slab_impl<T>(h, variant, color, static_cast<T *>(x_local),
                                                static_cast<const T *>(b_local), z_offset, nz_cells,
                                                vz_lo, vz_hi, as_stream(stream)));
  });
}

int pmg_smooth_host(pmg_level h, int variant, void *x, const void *b)
{
  return guard([&] {
    require_level(h);
    DeviceGuard dg(h->device);
    HostIO io(h);
    const size_t bytes = static_cast<size_t>(h->S.N) * h->tsize;
    void *dx = io.dev(0, bytes), *db = io.dev(1, bytes);
    if (host_pipeline_chunks(h, variant) > 1)
    {
      PMG_DISPATCH_T(h, smooth_host_pipelined<T>(h, variant, static_cast<T *>(x), static_cast<const T *>(b),
                                                 static_cast<T *>(dx), static_cast<T *>(db)));
      return;
    }
    io.h2d(dx, x, bytes);
    io.h2d(db, b, bytes);
    PMG_DISPATCH_T(h, smooth_impl<T>(h, variant, static_cast<T *>(dx), static_cast<const T *>(db),
                                     h->io_stream));
    io.d2h(x, dx, bytes);
    io.sync();
  });
}

int pmg_apply_laplacian(pmg_level h, const void *x, void *y, void *stream)
{
  return guard([&] {
    require_level(h);
    DeviceGuard dg(h->device);
    PMG_DISPATCH_T(h, ktab<T>(h).level_op(h->band_mats.data(), static_cast<const T *>(x), nullptr,
                                          static_cast<T *>(y), h->S.m, h->sm_count,
                                          as_stream(stream)));
  });
}

int pmg_compute_residual(pmg_level h, const void *x, const void *b, void *r, void *stream)
{
  return guard([&] {
    require_level(h);
    if (!b)
      throw InvalidArg("compute_residual: null b");
    DeviceGuard dg(h->device);
    PMG_DISPATCH_T(h, ktab<T>(h).level_op(h->band_mats.data(), static_cast<const T *>(x),
                                          static_cast<const T *>(b), static_cast<T *>(r), h->S.m,
                                          h->sm_count, as_stream(stream)));
  });
}


int pmg_compute_residual_slab(pmg_level h, const void *x, const void *b, void *r, int64_t zoff, int64_t nplanes,
                              int64_t p0, int64_t p1, void *stream)
{
  return guard([&] {
    require_level(h);
    if (h->S.dim != 3)
      throw InvalidArg("compute_residual_slab: dim 3 only");
    if (!x || !b || !r || nplanes < 0 || p0 < 0 || p1 > h->S.m || p0 > p1)
      throw InvalidArg("compute_residual_slab: invalid arguments");
    require_planes("compute_residual_slab", zoff, nplanes, p0 - h->S.k, p1 + h->S.k, h->S.m);
    require_planes("compute_residual_slab", zoff, nplanes, p0, p1, h->S.m);
    DeviceGuard dg(h->device);
    const int64_t pl = h->S.m * h->S.m;
    PMG_DISPATCH_T(h, ktab<T>(h).level_op_range(h->band_mats.data(), shift<T>(x, zoff, pl), shift<T>(b, zoff, pl),
                                                shift<T>(r, zoff, pl), h->S.m, p0, p1, h->sm_count,
                                                as_stream(stream)));
  });
}

int pmg_restrict_slab(pmg_level c, pmg_level f, const void *rf, int64_t zoff_f, int64_t np_f, void *rc,
                      int64_t zoff_c, int64_t np_c, int64_t q0, int64_t q1, void *stream)
{
  return guard([&] {
    check_pair(c, f, "restrict_slab");
    if (f->S.dim != 3)
      throw InvalidArg("restrict_slab: dim 3 only");
    if (!rf || !rc || q0 < 0 || q1 > c->S.m || q0 > q1)
      throw InvalidArg("restrict_slab: invalid arguments");
    int64_t pz0 = 0, pz1 = 0;
    restrict_slab_fine_range(f->S.k, c->S.m, q0, q1, pz0, pz1);
    require_planes("restrict_slab (fine)", zoff_f, np_f, pz0, pz1, f->S.m);
    require_planes("restrict_slab (coarse)", zoff_c, np_c, q0, q1, c->S.m);
    DeviceGuard dg(f->device);
    const int64_t mc = c->S.m, mf = f->S.m, np = std::max<int64_t>(pz1 - pz0, 0);
    PMG_DISPATCH_T(f, {
      f->tA.ensure(static_cast<size_t>(mc * mf * np) * sizeof(T) + sizeof(T));
      f->tB.ensure(static_cast<size_t>(mc * mc * np) * sizeof(T) + sizeof(T));
      ktab<T>(f).restrict_slab(f->prol_mats.data(), shift<T>(rf, zoff_f, mf * mf), shift<T>(rc, zoff_c, mc * mc),
                               mc, q0, q1, f->tA.as<T>() - pz0 * mc * mf, f->tB.as<T>() - pz0 * mc * mc,
                               f->sm_count, as_stream(stream));
    });
  });
}

int pmg_prolongate_slab(pmg_level c, pmg_level f, const void *xc, int64_t zoff_c, int64_t np_c, void *xf,
                        int64_t zoff_f, int64_t np_f, int64_t f0, int64_t f1, int accumulate, void *stream)
{
  return guard([&] {
    check_pair(c, f, "prolongate_slab");
    if (f->S.dim != 3)
      throw InvalidArg("prolongate_slab: dim 3 only");
    if (!xc || !xf || f0 < 0 || f1 > f->S.m || f0 > f1)
      throw InvalidArg("prolongate_slab: invalid arguments");
    const int64_t K = f->S.k, mc = c->S.m, mf = f->S.m;
    if (f0 < f1)
    {
      const int64_t cz0 = f0 / (2 * K), cz1 = (f1 - 1) / (2 * K);  // coarse cells
      require_planes("prolongate_slab (coarse)", zoff_c, np_c, cz0 * K - 1, cz1 * K + K, mc);
    }
    require_planes("prolongate_slab (fine)", zoff_f, np_f, f0, f1, mf);
    DeviceGuard dg(f->device);
    PMG_DISPATCH_T(f, ktab<T>(f).prolongate_slab(f->prol_mats.data(), shift<T>(xc, zoff_c, mc * mc),
                                                 shift<T>(xf, zoff_f, mf * mf), accumulate != 0, mc, f0, f1,
                                                 as_stream(stream)));
  });
}

int pmg_apply_laplacian_host(pmg_level h, const void *x, void *y)
{
  return guard([&] {
    require_level(h);
    DeviceGuard dg(h->device);
    HostIO io(h);
    const size_t bytes = static_cast<size_t>(h->S.N) * h->tsize;
    void *dx = io.dev(0, bytes), *dy = io.dev(1, bytes);
    io.h2d(dx, x, bytes);
    PMG_DISPATCH_T(h, ktab<T>(h).level_op(h->band_mats.data(), static_cast<const T *>(dx), nullptr,
                                          static_cast<T *>(dy), h->S.m, h->sm_count, h->io_stream));
    io.d2h(y, dy, bytes);
    io.sync();
  });
}

int pmg_compute_residual_host(pmg_level h, const void *x, const void *b, void *r)
{
  return guard([&] {
    require_level(h);
    DeviceGuard dg(h->device);
    HostIO io(h);
    const size_t bytes = static_cast<size_t>(h->S.N) * h->tsize;
    void *dx = io.dev(0, bytes), *db = io.dev(1, bytes), *dr = io.dev(2, bytes);
    io.h2d(dx, x, bytes);
    io.h2d(db, b, bytes);
    PMG_DISPATCH_T(h, ktab<T>(h).level_op(h->band_mats.data(), static_cast<const T *>(dx),
                                          static_cast<const T *>(db), static_cast<T *>(dr), h->S.m,
                                          h->sm_count, h->io_stream));
    io.d2h(r, dr, bytes);
    io.sync();
  });
}

int pmg_prolongate(pmg_level c, pmg_level f, const void *xc, void *xf, int accumulate, void *stream)
{
  return guard([&] {
    check_pair(c, f, "prolongate");
    DeviceGuard dg(f->device);
    PMG_DISPATCH_T(f, prolongate_impl<T>(c, f, static_cast<const T *>(xc), static_cast<T *>(xf),
                                         accumulate != 0, as_stream(stream)));
  });
}

int pmg_prolongate_host(pmg_level c, pmg_level f, const void *xc, void *xf)
{
  return guard([&] {
    check_pair(c, f, "prolongate");
    DeviceGuard dg(f->device);
    HostIO io(f);
    const size_t bc = static_cast<size_t>(c->S.N) * f->tsize, bf = static_cast<size_t>(f->S.N) * f->tsize;
    void *dxc = io.dev(0, bc), *dxf = io.dev(1, bf);
    io.h2d(dxc, xc, bc);
    PMG_DISPATCH_T(f, prolongate_impl<T>(c, f, static_cast<const T *>(dxc), static_cast<T *>(dxf),
                                         false, f->io_stream));
    io.d2h(xf, dxf, bf);
    io.sync();
  });
}

int pmg_restrict_vector(pmg_level c, pmg_level f, const void *rf, void *rc, void *stream)
{
  return guard([&] {
    check_pair(c, f, "restrict_vector");
    DeviceGuard dg(f->device);
    PMG_DISPATCH_T(f, restrict_impl<T>(c, f, static_cast<const T *>(rf), static_cast<T *>(rc),
                                       as_stream(stream)));
  });
}

int pmg_restrict_vector_host(pmg_level c, pmg_level f, const void *rf, void *rc)
{
  return guard([&] {
    check_pair(c, f, "restrict_vector");
    DeviceGuard dg(f->device);
    HostIO io(f);
    const size_t bc = static_cast<size_t>(c->S.N) * f->tsize, bf = static_cast<size_t>(f->S.N) * f->tsize;
    void *drf = io.dev(0, bf), *drc = io.dev(1, bc);
    io.h2d(drf, rf, bf);
    PMG_DISPATCH_T(f, restrict_impl<T>(c, f, static_cast<const T *>(drf), static_cast<T *>(drc),
                                       f->io_stream));
    io.d2h(rc, drc, bc);
    io.sync();
  });
}

int pmg_vector_norm(pmg_level h, const void *v, double *out, void *stream)
{
  return guard([&] {
    require_level(h);
    if (!out)
      throw InvalidArg("null output");
    DeviceGuard dg(h->device);
    PMG_DISPATCH_T(h, *out = norm_impl<T>(h, static_cast<const T *>(v), h->S.N, as_stream(stream)));
  });
}

int pmg_norm2(const void *v, int64_t n, int dtype, int device, double *out, void *stream)
{
  return guard([&] {
    if (!out || (n > 0 && !v))
      throw InvalidArg("pmg_norm2: null pointer");
    if (dtype != PMG_F64 && dtype != PMG_F32)
      throw InvalidArg("pmg_norm2: bad dtype");
    DeviceGuard dg(device);
    static thread_local DevBuf red[32];
    DevBuf &rb = red[device & 31];
    rb.ensure((RED_BLOCKS + 8) * sizeof(double));
    cudaStream_t s = as_stream(stream);
    double *r = rb.as<double>();
    if (dtype == PMG_F64)
      launch_dot<double>(static_cast<const double *>(v), static_cast<const double *>(v), n, r,
                         r + RED_BLOCKS, true, s);
    else
      launch_dot<float>(static_cast<const float *>(v), static_cast<const float *>(v), n, r,
                        r + RED_BLOCKS, true, s);
    check_cuda(cudaMemcpyAsync(out, r + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    check_cuda(cudaStreamSynchronize(s), "sync");
  });
}

int pmg_mg_create(int dim, int degree, int finest_level, int dtype, int variant, int device,
                  pmg_mg *out)
{
  return pmg_mg_create_kind(dim, degree, finest_level, dtype, variant, PMG_VERTEX_PATCH, device, out);
}

int pmg_mg_create_kind(int dim, int degree, int finest_level, int dtype, int variant, int kind, int device,
                       pmg_mg *out)
{
  return guard([&] {
    if (kind != PMG_VERTEX_PATCH && kind != PMG_POINT_GS)
      throw InvalidArg("unknown smoother kind");
    // multigrid.cpp:32-36 (std::invalid_argument)
    if (kind == PMG_POINT_GS && dtype != PMG_F64)
      throw InvalidArg("point Gauss-Seidel runs in f64 only");
    if (!out)
      throw InvalidArg("null output handle");
    if (finest_level < 1)
      throw InvalidArg("finest_level must be >= 1");
    if (variant != PMG_GLOBAL && variant != PMG_SEPARATE && variant != PMG_FUSED &&
        variant != PMG_BOUNDARY && variant != PMG_NAIVE)
      throw InvalidArg("unknown smoother variant");
    auto mg = std::make_unique<pmg_mg_s>();
    mg->kind = kind;
    mg->dtype = dtype;
    mg->device = device;
    mg->variant = variant;
    for (int l = 1; l <= finest_level; ++l)
      mg->levels.push_back(make_level(dim, degree, l, dtype, device));
    DeviceGuard dg(device);
    const size_t ts = dtype == PMG_F64 ? 8 : 4;
    for (int li = 0; li < finest_level; ++li)
    {
      auto *r = new DevBuf();
      auto *bc = new DevBuf();
      auto *xc = new DevBuf();
      mg->r_ws.push_back(r);
      mg->bc_ws.push_back(bc);
      mg->xc_ws.push_back(xc);
      if (li > 0)
      {
        r->ensure(static_cast<size_t>(mg->levels[li]->S.N) * ts);
        bc->ensure(static_cast<size_t>(mg->levels[li - 1]->S.N) * ts);
        xc->ensure(static_cast<size_t>(mg->levels[li - 1]->S.N) * ts);
        if (dtype == PMG_F64)
          transfer_scratch<double>(mg->levels[li]);
        else
          transfer_scratch<float>(mg->levels[li]);
      }
    }
    // coarse-matrix level: the largest li >= 1 with <= PMG_COARSE_MAT_N
    // unknowns (the parent's coarse correction becomes one GEMV). 3375
    // unknowns (91 MB f64) stream in ~15 us with the warp-per-row GEMV, less
    // than the recursion they replace; the next levels (k = 2: 29791
    // unknowns, 7 GB) are far beyond (profiles/r02/ab/coarse_matrix*.txt)
    {
      static const int64_t nmax = [] {
        const char *e = std::getenv("PMG_COARSE_MAT_N");
        // (<= 12000: the GEMV stages b in <= 96 KB of shared memory)
        return e ? std::min<int64_t>(std::atoll(e), 12000) : int64_t(3375);
      }();
      // (the finest level too: the slab decomposition's agglomerated coarse
      // correction may land there; the same level is then chosen in every
      // context that holds it, so all of them compute it the same way)
      for (int li = 1; li < static_cast<int>(mg->levels.size()); ++li)
        if (mg->levels[li]->S.N <= nmax)
          mg->mat_li = li;
    }
    // the reference assembles a CSR matrix per level (multigrid.cpp:37-41):
    // same nonzero budget (std::runtime_error), front lists built up front
    if (kind == PMG_POINT_GS)
      for (auto *l : mg->levels)
        gs_data(l);
    *out = mg.release();
  });
}

int pmg_mg_destroy(pmg_mg h)
{
  return guard([&] {
    if (h)
    {
      DeviceGuard dg(h->device);
      delete h;
    }
  });
}

int pmg_mg_num_levels(pmg_mg h) { return h ? static_cast<int>(h->levels.size()) : 0; }

pmg_level pmg_mg_level(pmg_mg h, int li)
{
  if (!h || li < 0 || li >= static_cast<int>(h->levels.size()))
    return nullptr;
  return h->levels[li];
}

int pmg_mg_set_smoothing(pmg_mg h, int pre, int post)
{
  return guard([&] {
    if (!h || pre < 0 || post < 0)
      throw InvalidArg("invalid smoothing counts");
    h->pre = pre;
    h->post = post;
  });
}

int pmg_mg_set_variant(pmg_mg h, int variant)
{
  return guard([&] {
    if (!h)
      throw InvalidArg("null handle");
    if (variant != PMG_GLOBAL && variant != PMG_SEPARATE && variant != PMG_FUSED &&
        variant != PMG_BOUNDARY && variant != PMG_NAIVE)
      throw InvalidArg("unknown smoother variant");
    h->variant = variant;
  });
}

int pmg_v_cycle(pmg_mg h, int li, void *x, const void *b, int use_graph, void *stream)
{
  return guard([&] {
    if (!h || li < 0 || li >= static_cast<int>(h->levels.size()))
      throw InvalidArg("v_cycle: level index out of range");
    DeviceGuard dg(h->device);
    PMG_DISPATCH_T(h, vcycle_entry<T>(h, li, static_cast<T *>(x), static_cast<const T *>(b),
                                      use_graph != 0, as_stream(stream)));
  });
}

int pmg_v_cycle_host(pmg_mg h, int li, void *x, const void *b)
{
  return guard([&] {
    if (!h || li < 0 || li >= static_cast<int>(h->levels.size()))
      throw InvalidArg("v_cycle: level index out of range");
    DeviceGuard dg(h->device);
    pmg_level_s *l = h->levels[li];
    HostIO io(l);
    const size_t bytes = static_cast<size_t>(l->S.N) * l->tsize;
    void *dx = io.dev(0, bytes), *db = io.dev(1, bytes);
    io.h2d(dx, x, bytes);
    io.h2d(db, b, bytes);
    PMG_DISPATCH_T(h, {
      ensure_coarse_matrix<T>(h, l->io_stream);
      vcycle_impl<T>(h, li, static_cast<T *>(dx), static_cast<const T *>(db), l->io_stream);
    });
    io.d2h(x, dx, bytes);
    io.sync();
  });
}

int pmg_full_multigrid(pmg_mg h, const void *const *rhs, void *x, double tol, int max_iterations,
                       int *iterations, double *history, int history_cap, void *stream)
{
  return guard([&] {
    if (!h)
      throw InvalidArg("null handle");
    if (h->dtype != PMG_F64)
      throw InvalidArg("full_multigrid runs in f64 only (multigrid.hpp:80)");
    if (!(tol > 0.0))
      throw InvalidArg("full_multigrid: tol must be positive");
    if (!rhs || !x)
      throw InvalidArg("full_multigrid: null pointer");
    DeviceGuard dg(h->device);
    cudaStream_t s = as_stream(stream);
    const int L = static_cast<int>(h->levels.size()) - 1;
    using T = double;
    // nested iteration (multigrid.cpp:366-377)
    std::vector<T *> xl(L + 1);
    for (int li = 0; li < L; ++li)
    {
      h->fmg_x[li].ensure(static_cast<size_t>(h->levels[li]->S.N) * sizeof(T));
      xl[li] = h->fmg_x[li].as<T>();
    }
    xl[L] = static_cast<T *>(x);
    ensure_coarse_matrix<T>(h, s);
    vcycle_impl<T>(h, 0, xl[0], static_cast<const T *>(rhs[0]), s);
    for (int li = 1; li <= L; ++li)
    {
      prolongate_impl<T>(h->levels[li - 1], h->levels[li], xl[li - 1], xl[li], false, s);
      vcycle_impl<T>(h, li, xl[li], static_cast<const T *>(rhs[li]), s);
    }
    pmg_level_s *top = h->levels[L];
    const T *bL = static_cast<const T *>(rhs[L]);
    const double delta0 = norm_impl<T>(top, bL, top->S.N, s);
    int it = 0;
    int nh = 0;
    if (history && history_cap > nh)
      history[nh] = delta0;
    ++nh;
    double delta = delta0;
    T *r = h->r_ws[L]->as<T>();
    if (L == 0)
    {
      h->r_ws[0]->ensure(static_cast<size_t>(top->S.N) * sizeof(T));
      r = h->r_ws[0]->as<T>();
    }
    while (delta > tol * delta0)
    {
      if (it >= max_iterations)
      {
        if (iterations)
          *iterations = it;
        throw Divergence("full_multigrid: no convergence after " + std::to_string(max_iterations) +
                         " V-cycles");
      }
      vcycle_impl<T>(h, L, static_cast<T *>(x), bL, s);
      ktab<T>(top).level_op(top->band_mats.data(), static_cast<const T *>(x), bL, r, top->S.m,
                            top->sm_count, s);
      delta = norm_impl<T>(top, r, top->S.N, s);
      if (history && history_cap > nh)
        history[nh] = delta;
      ++nh;
      ++it;
    }
    if (iterations)
      *iterations = it;
  });
}

int pmg_full_multigrid_host(pmg_mg h, const double *const *rhs_host, double *x, double tol, int max_iterations,
                            int *iterations, double *history, int history_cap)
{
  std::vector<std::unique_ptr<DevBuf>> rhs;
  std::vector<const void *> ptrs;
  DevBuf dx;
  int st = guard([&] {
    if (!h || !rhs_host || !x)
      throw InvalidArg("full_multigrid: null pointer");
    DeviceGuard dg(h->device);
    for (size_t li = 0; li < h->levels.size(); ++li)
    {
      if (!rhs_host[li])
        throw InvalidArg("full_multigrid: need one rhs per level");
      const size_t bytes = static_cast<size_t>(h->levels[li]->S.N) * sizeof(double);
      rhs.push_back(std::make_unique<DevBuf>());
      rhs.back()->ensure(bytes);
      check_cuda(cudaMemcpy(rhs.back()->p, rhs_host[li], bytes, cudaMemcpyHostToDevice), "H2D");
      ptrs.push_back(rhs.back()->p);
    }
    dx.ensure(static_cast<size_t>(h->levels.back()->S.N) * sizeof(double));
  });
  if (st != PMG_OK)
    return st;
  st = pmg_full_multigrid(h, ptrs.data(), dx.p, tol, max_iterations, iterations, history, history_cap, nullptr);
  const int st2 = guard([&] {
    DeviceGuard dg(h->device);
    check_cuda(cudaDeviceSynchronize(), "sync");
    check_cuda(cudaMemcpy(x, dx.p, dx.bytes, cudaMemcpyDeviceToHost), "D2H");
  });
  return st != PMG_OK ? st : st2;
}

int pmg_vector_norm_host(const void *v, int64_t n, int dtype, int device, double *out)
{
  DevBuf dv;
  const int st = guard([&] {
    if (!out || (n > 0 && !v) || n < 0)
      throw InvalidArg("vector_norm: invalid arguments");
    if (dtype != PMG_F64 && dtype != PMG_F32)
      throw InvalidArg("vector_norm: bad dtype");
    DeviceGuard dg(device);
    const size_t bytes = static_cast<size_t>(n) * (dtype == PMG_F64 ? 8 : 4);
    dv.ensure(bytes + 8);
    check_cuda(cudaMemcpy(dv.p, v, bytes, cudaMemcpyHostToDevice), "H2D");
  });
  if (st != PMG_OK)
    return st;
  return pmg_norm2(dv.p, n, dtype, device, out, nullptr);
}

int pmg_compute_rhs_host(int dim, int degree, int level, int kind, double *out)
{
  return guard([&] {
    if (dim != 2 && dim != 3)
      throw InvalidArg("dim must be 2 or 3");
    auto b = compute_rhs(dim, degree, level, kind);
    std::memcpy(out, b.data(), b.size() * sizeof(double));
  });
}

int pmg_l2_error_sin_host(int dim, int degree, int level, const double *x, double *out)
{
  return guard([&] { *out = l2_error_sin(dim, degree, level, x); });
}

}  // extern "C"
