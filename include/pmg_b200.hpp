// pmg_b200.hpp — header-only C++ shim over the C-ABI (pmg_b200.h) with the
// reference's names and calling conventions (/root/reference/proj/include/pmg):
// host std::span vectors in, exceptions out. A reference user swaps
//   #include "pmg/multigrid.hpp"            ->  #include "pmg_b200.hpp"
//   namespace pmg                           ->  namespace pmgb
// and keeps the call sites: build_hierarchy, make_multigrid_context, smooth,
// apply_laplacian, compute_residual, prolongate, restrict_vector, v_cycle,
// full_multigrid, vector_norm, point_gauss_seidel, assemble_sparse, gmres.
// Multi-GPU: MultiGpuContext<T> with the same smooth / v_cycle /
// full_multigrid calls on global host vectors.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "pmg_b200.h"

namespace pmgb
{

// smoother.hpp:21-27
enum class SmootherVariant
{
  global = PMG_GLOBAL,
  separate = PMG_SEPARATE,
  fused = PMG_FUSED,
  boundary = PMG_BOUNDARY
};

// multigrid.hpp:16-20
enum class SmootherKind
{
  vertex_patch = PMG_VERTEX_PATCH,
  point_gs = PMG_POINT_GS
};

// operator.hpp:30-38 (the device operator has one deterministic schedule;
// both values give the same result, as in the reference)
enum class CellLoop
{
  colored,
  sequential
};

// multigrid.hpp:22-29
struct DivergenceError : std::runtime_error
{
  std::vector<double> residual_history;
  DivergenceError(const std::string &w, std::vector<double> h)
      : std::runtime_error(w), residual_history(std::move(h))
  {
  }
};

inline void check(int st, std::vector<double> history = {})
{
  if (st == PMG_OK)
    return;
  const std::string msg = pmg_last_error();
  if (st == PMG_ERR_INVALID)
    throw std::invalid_argument(msg);
  if (st == PMG_ERR_DIVERGENCE)
    throw DivergenceError(msg, std::move(history));
  throw std::runtime_error(msg);
}

template <typename T>
constexpr int dtype_of()
{
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>,
                "explicit instantiations are float and double only");
  return std::is_same_v<T, double> ? PMG_F64 : PMG_F32;
}

// mesh.hpp:16-29
struct CartesianLevel
{
  int level = 1;
  int dim = 2;
  int degree = 1;
  int cells_per_dim = 2;
  int dofs_per_dim = 1;
  double spacing = 0.5;
  std::int64_t total_dofs = 1;
  friend bool operator==(const CartesianLevel &, const CartesianLevel &) = default;
};

// mesh.hpp:31-34 (same argument checks: std::invalid_argument)
inline std::vector<CartesianLevel> build_hierarchy(int dim, int degree, int finest_level)
{
  if (dim != 2 && dim != 3)
    throw std::invalid_argument("build_hierarchy: dim must be 2 or 3, got " + std::to_string(dim));
  if (degree < 1)
    throw std::invalid_argument("build_hierarchy: degree must be >= 1");
  if (finest_level < 1)
    throw std::invalid_argument("build_hierarchy: finest_level must be >= 1");
  std::vector<CartesianLevel> out;
  for (int l = 1; l <= finest_level; ++l)
  {
    CartesianLevel c;
    c.level = l;
    c.dim = dim;
    c.degree = degree;
    c.cells_per_dim = 1 << l;
    c.dofs_per_dim = c.cells_per_dim * degree - 1;
    c.spacing = 1.0 / c.cells_per_dim;
    c.total_dofs = 1;
    for (int a = 0; a < dim; ++a)
      c.total_dofs *= c.dofs_per_dim;
    out.push_back(c);
  }
  return out;
}

// dense.hpp:15-38
template <typename T>
struct Mat
{
  int rows = 0, cols = 0;
  std::vector<T> data;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, T(0)) {}
  T &operator()(int i, int j) { return data[static_cast<std::size_t>(i) * cols + j]; }
  const T &operator()(int i, int j) const { return data[static_cast<std::size_t>(i) * cols + j]; }
};

// sparse.hpp:16-26 (host container; the device never needs it)
struct CsrMatrix
{
  std::int64_t n = 0;
  std::vector<std::int64_t> row_ptr;
  std::vector<std::int32_t> cols;
  std::vector<double> vals;
  std::int64_t nnz() const { return static_cast<std::int64_t>(vals.size()); }
};

// smoother.hpp:29-38: the device smoother keeps its scratch in the level
// context; the workspace is accepted for signature parity
template <typename T>
struct SmootherWorkspace
{
};

// ~ LevelContext<T> (level_context.hpp:17-26): borrowed from a context or owned
template <typename T>
class LevelContext
{
 public:
  LevelContext(int dim, int degree, int level, int device = 0)
  {
    check(pmg_level_create(dim, degree, level, dtype_of<T>(), device, &h_));
    owned_ = true;
    init(dim, degree, level);
  }
  LevelContext(pmg_level borrowed, int dim, int degree, int level) : h_(borrowed) { init(dim, degree, level); }
  LevelContext(const LevelContext &) = delete;
  LevelContext &operator=(const LevelContext &) = delete;
  LevelContext(LevelContext &&o) noexcept
      : level(o.level), cell_mass(std::move(o.cell_mass)), cell_stiffness(std::move(o.cell_stiffness)), h_(o.h_),
        owned_(o.owned_)
  {
    o.h_ = nullptr;
  }
  ~LevelContext()
  {
    if (owned_ && h_)
      pmg_level_destroy(h_);
  }
  pmg_level handle() const { return h_; }
  std::int64_t total_dofs() const { return level.total_dofs; }

  CartesianLevel level;
  Mat<T> cell_mass, cell_stiffness;  // (k+1)^2, as uploaded

 private:
  void init(int dim, int degree, int lev)
  {
    level = build_hierarchy(dim, degree, lev).back();
    const int q = degree + 1;
    std::vector<double> cm(q * q), cs(q * q);
    check(pmg_level_setup_data(h_, nullptr, nullptr, nullptr, nullptr, nullptr, cm.data(), cs.data()));
    cell_mass = Mat<T>(q, q);
    cell_stiffness = Mat<T>(q, q);
    for (int e = 0; e < q * q; ++e)
    {
      cell_mass.data[e] = static_cast<T>(cm[e]);
      cell_stiffness.data[e] = static_cast<T>(cs[e]);
    }
  }
  pmg_level h_ = nullptr;
  bool owned_ = false;
};

// ~ MultigridContext<T> (multigrid.hpp:34-49)
template <typename T>
class MultigridContext
{
 public:
  MultigridContext(int dim, int degree, int finest_level, SmootherVariant variant = SmootherVariant::fused,
                   SmootherKind kind = SmootherKind::vertex_patch, int device = 0)
      : variant(variant), kind(kind)
  {
    check(pmg_mg_create_kind(dim, degree, finest_level, dtype_of<T>(), static_cast<int>(variant),
                             static_cast<int>(kind), device, &h_));
    for (int li = 0; li < pmg_mg_num_levels(h_); ++li)
      levels.emplace_back(pmg_mg_level(h_, li), dim, degree, li + 1);
  }
  MultigridContext(const MultigridContext &) = delete;
  MultigridContext &operator=(const MultigridContext &) = delete;
  MultigridContext(MultigridContext &&o) noexcept
      : levels(std::move(o.levels)), variant(o.variant), kind(o.kind), h_(o.h_)
  {
    o.h_ = nullptr;
  }
  ~MultigridContext()
  {
    levels.clear();
    if (h_)
      pmg_mg_destroy(h_);
  }
  pmg_mg handle() const { return h_; }
  void set_smoothing(int pre, int post) { check(pmg_mg_set_smoothing(h_, pre, post)); }
  std::vector<LevelContext<T>> levels;
  SmootherVariant variant;
  SmootherKind kind;
  int threads = 1;  // accepted; the device ignores it

 private:
  pmg_mg h_ = nullptr;
};

// multigrid.hpp:51-54
template <typename T>
MultigridContext<T> make_multigrid_context(int dim, int degree, int finest_level,
                                           SmootherVariant variant = SmootherVariant::fused,
                                           SmootherKind kind = SmootherKind::vertex_patch, int threads = 1)
{
  MultigridContext<T> c(dim, degree, finest_level, variant, kind);
  c.threads = threads;
  return c;
}

// smoother.hpp:45-47
template <typename T>
void smooth(const LevelContext<T> &ctx, std::span<T> x, std::span<const T> b,
            SmootherVariant variant = SmootherVariant::fused, int /*threads*/ = 1)
{
  if (static_cast<std::int64_t>(x.size()) != ctx.total_dofs() ||
      static_cast<std::int64_t>(b.size()) != ctx.total_dofs())
    throw std::invalid_argument("smooth: vector size does not match level");
  check(pmg_smooth_host(ctx.handle(), static_cast<int>(variant), x.data(), b.data()));
}
template <typename T>
void smooth(const LevelContext<T> &ctx, std::span<T> x, std::span<const T> b, SmootherVariant variant,
            int threads, SmootherWorkspace<T> & /*ws*/)
{
  smooth<T>(ctx, x, b, variant, threads);
}

namespace detail
{
// one device level context per (dim, degree, level, T) for the calls that
// take a CartesianLevel (apply_laplacian), created on first use
template <typename T>
inline pmg_level cached_level(const CartesianLevel &lev)
{
  static thread_local std::map<std::tuple<int, int, int>, pmg_level> cache;
  pmg_level &h = cache[std::make_tuple(lev.dim, lev.degree, lev.level)];
  if (!h)
    check(pmg_level_create(lev.dim, lev.degree, lev.level, dtype_of<T>(), 0, &h));
  return h;
}
}  // namespace detail

// operator.hpp:47-50. The device operator is the level's Kronecker sum of its
// own 1D cell matrices; other matrices are refused (std::invalid_argument).
template <typename T>
void apply_laplacian(const CartesianLevel &level, const Mat<T> &cell_mass, const Mat<T> &cell_stiffness,
                     std::span<const T> x, std::span<T> y, CellLoop /*mode*/ = CellLoop::colored,
                     int /*threads*/ = 1)
{
  if (static_cast<std::int64_t>(x.size()) != level.total_dofs ||
      static_cast<std::int64_t>(y.size()) != level.total_dofs)
    throw std::invalid_argument("apply_laplacian: vector size does not match level");
  const int q = level.degree + 1;
  if (cell_mass.rows != q || cell_mass.cols != q || cell_stiffness.rows != q || cell_stiffness.cols != q)
    throw std::invalid_argument("apply_laplacian: cell matrices must be (k+1) x (k+1)");
  pmg_level h = detail::cached_level<T>(level);
  std::vector<double> cm(q * q), cs(q * q);
  check(pmg_level_setup_data(h, nullptr, nullptr, nullptr, nullptr, nullptr, cm.data(), cs.data()));
  for (int e = 0; e < q * q; ++e)
  {
    const double tm = std::fabs(static_cast<double>(cell_mass.data[e]) - static_cast<double>(static_cast<T>(cm[e])));
    const double ts =
        std::fabs(static_cast<double>(cell_stiffness.data[e]) - static_cast<double>(static_cast<T>(cs[e])));
    if (tm > 1e-12 * (1 + std::fabs(cm[e])) || ts > 1e-12 * (1 + std::fabs(cs[e])))
      throw std::invalid_argument("apply_laplacian: the device operator supports the level's own cell matrices");
  }
  check(pmg_apply_laplacian_host(h, x.data(), y.data()));
}
template <typename T>
void apply_laplacian(const LevelContext<T> &ctx, std::span<const T> x, std::span<T> y)
{
  if (static_cast<std::int64_t>(x.size()) != ctx.total_dofs() ||
      static_cast<std::int64_t>(y.size()) != ctx.total_dofs())
    throw std::invalid_argument("apply_laplacian: vector size does not match level");
  check(pmg_apply_laplacian_host(ctx.handle(), x.data(), y.data()));
}

// multigrid.hpp:90-92
template <typename T>
void compute_residual(const LevelContext<T> &ctx, std::span<const T> x, std::span<const T> b, std::span<T> r,
                      int /*threads*/ = 1)
{
  if (static_cast<std::int64_t>(x.size()) != ctx.total_dofs() ||
      static_cast<std::int64_t>(b.size()) != ctx.total_dofs() ||
      static_cast<std::int64_t>(r.size()) != ctx.total_dofs())
    throw std::invalid_argument("compute_residual: vector size does not match level");
  check(pmg_compute_residual_host(ctx.handle(), x.data(), b.data(), r.data()));
}

// multigrid.hpp:56-63
template <typename T>
void prolongate(const LevelContext<T> &c, const LevelContext<T> &f, std::span<const T> xc, std::span<T> xf)
{
  if (static_cast<std::int64_t>(xc.size()) != c.total_dofs() || static_cast<std::int64_t>(xf.size()) != f.total_dofs())
    throw std::invalid_argument("prolongate: vector size does not match level");
  check(pmg_prolongate_host(c.handle(), f.handle(), xc.data(), xf.data()));
}
template <typename T>
void restrict_vector(const LevelContext<T> &c, const LevelContext<T> &f, std::span<const T> rf, std::span<T> rc)
{
  if (static_cast<std::int64_t>(rc.size()) != c.total_dofs() || static_cast<std::int64_t>(rf.size()) != f.total_dofs())
    throw std::invalid_argument("restrict_vector: vector size does not match level");
  check(pmg_restrict_vector_host(c.handle(), f.handle(), rf.data(), rc.data()));
}

// multigrid.hpp:68-69
template <typename T>
void v_cycle(MultigridContext<T> &ctx, int li, std::span<T> x, std::span<const T> b)
{
  check(pmg_v_cycle_host(ctx.handle(), li, x.data(), b.data()));
}

// multigrid.hpp:74-86
struct FmgStats
{
  int iterations = 0;
  std::vector<double> residual_history;
};

inline FmgStats full_multigrid(MultigridContext<double> &ctx, const std::vector<std::vector<double>> &rhs_per_level,
                               std::span<double> x, double tol, int max_iterations = 100)
{
  if (rhs_per_level.size() != ctx.levels.size())
    throw std::invalid_argument("full_multigrid: need one rhs per level");
  std::vector<const double *> ptrs;
  for (const auto &r : rhs_per_level)
    ptrs.push_back(r.data());
  std::vector<double> hist(static_cast<std::size_t>(max_iterations) + 2);
  int its = 0;
  const int st = pmg_full_multigrid_host(ctx.handle(), ptrs.data(), x.data(), tol, max_iterations, &its, hist.data(),
                                         static_cast<int>(hist.size()));
  hist.resize(static_cast<std::size_t>(std::min<int>(its + 1, static_cast<int>(hist.size()))));
  check(st, hist);
  return FmgStats{its, hist};
}

// multigrid.hpp:89
inline double vector_norm(std::span<const double> v)
{
  double out = 0;
  check(pmg_vector_norm_host(v.data(), static_cast<std::int64_t>(v.size()), PMG_F64, 0, &out));
  return out;
}

// operator.hpp:55 (host)
inline CsrMatrix assemble_sparse(const CartesianLevel &level)
{
  CsrMatrix a;
  std::int64_t nnz = 0;
  check(pmg_assemble_sparse_host(level.dim, level.degree, level.level, nullptr, nullptr, nullptr, &nnz));
  a.n = level.total_dofs;
  a.row_ptr.resize(static_cast<std::size_t>(a.n) + 1);
  a.cols.resize(static_cast<std::size_t>(nnz));
  a.vals.resize(static_cast<std::size_t>(nnz));
  check(pmg_assemble_sparse_host(level.dim, level.degree, level.level, a.row_ptr.data(), a.cols.data(),
                                 a.vals.data(), &nnz));
  return a;
}

// smoother.cpp:160-166 on the level's operator (the device sweep needs no CSR)
inline void point_gauss_seidel(const LevelContext<double> &ctx, std::span<double> x, std::span<const double> b)
{
  if (static_cast<std::int64_t>(x.size()) != ctx.total_dofs() ||
      static_cast<std::int64_t>(b.size()) != ctx.total_dofs())
    throw std::invalid_argument("point_gauss_seidel: vector size does not match matrix");
  check(pmg_point_gauss_seidel_host(ctx.handle(), x.data(), b.data()));
}

// krylov.hpp:16-39: right-preconditioned GMRES(restart) in f64 with the
// V-cycle of `prec` as preconditioner (an f32 context = the reference's
// mixed_precision_precondition, an f64 context = double)
struct SolveStats
{
  int iterations = 0;
  std::vector<double> residual_history;
  std::optional<double> l2_error;
  double wall_seconds = 0.0;
};

template <typename P>
SolveStats gmres(MultigridContext<double> &op, MultigridContext<P> &prec, std::span<const double> b,
                 std::span<double> x, double tol, int restart = 30, int max_iterations = 200)
{
  std::vector<double> hist(static_cast<std::size_t>(max_iterations) + 2);
  int its = 0;
  const int st = pmg_gmres_host(op.handle(), prec.handle(), b.data(), x.data(), tol, restart, max_iterations, &its,
                                hist.data(), static_cast<int>(hist.size()));
  hist.resize(static_cast<std::size_t>(std::min<int>(its + 1, static_cast<int>(hist.size()))));
  check(st, hist);
  SolveStats s;
  s.iterations = its;
  s.residual_history = hist;
  return s;
}

// ---- multi-GPU (pmg_dd_*): the same calls on a z-slab decomposition --------
template <typename T>
class MultiGpuContext
{
 public:
  // devices: one per rank (repeats allowed with PMG_DD_COPY)
  MultiGpuContext(const std::vector<int> &devices, int dim, int degree, int finest_level,
                  SmootherVariant variant = SmootherVariant::fused, int transport = PMG_DD_COPY, int stack = 1)
      : level(build_hierarchy(dim, degree, finest_level).back())
  {
    check(pmg_dd_create(static_cast<int>(devices.size()), devices.data(), dim, degree, finest_level, stack,
                        dtype_of<T>(), static_cast<int>(variant), transport, &h_));
    if (stack != 1)
      level.total_dofs = level.total_dofs / level.dofs_per_dim * (stack * level.cells_per_dim * degree - 1);
  }
  MultiGpuContext(const MultiGpuContext &) = delete;
  MultiGpuContext &operator=(const MultiGpuContext &) = delete;
  ~MultiGpuContext()
  {
    if (h_)
      pmg_dd_destroy(h_);
  }
  pmg_dd handle() const { return h_; }
  CartesianLevel level;  // the finest level

 private:
  pmg_dd h_ = nullptr;
};

template <typename T>
void smooth(MultiGpuContext<T> &ctx, std::span<T> x, std::span<const T> b)
{
  if (static_cast<std::int64_t>(x.size()) != ctx.level.total_dofs ||
      static_cast<std::int64_t>(b.size()) != ctx.level.total_dofs)
    throw std::invalid_argument("smooth: vector size does not match level");
  check(pmg_dd_scatter_host(ctx.handle(), PMG_DD_X, x.data()));
  check(pmg_dd_scatter_host(ctx.handle(), PMG_DD_B, b.data()));
  check(pmg_dd_smooth(ctx.handle()));
  check(pmg_dd_gather_host(ctx.handle(), PMG_DD_X, x.data()));
}

template <typename T>
void v_cycle(MultiGpuContext<T> &ctx, std::span<T> x, std::span<const T> b)
{
  if (static_cast<std::int64_t>(x.size()) != ctx.level.total_dofs ||
      static_cast<std::int64_t>(b.size()) != ctx.level.total_dofs)
    throw std::invalid_argument("v_cycle: vector size does not match level");
  check(pmg_dd_scatter_host(ctx.handle(), PMG_DD_X, x.data()));
  check(pmg_dd_scatter_host(ctx.handle(), PMG_DD_B, b.data()));
  check(pmg_dd_v_cycle(ctx.handle()));
  check(pmg_dd_gather_host(ctx.handle(), PMG_DD_X, x.data()));
}

inline FmgStats full_multigrid(MultiGpuContext<double> &ctx, const std::vector<std::vector<double>> &rhs_per_level,
                               std::span<double> x, double tol, int max_iterations = 100)
{
  std::vector<const double *> ptrs;
  for (const auto &r : rhs_per_level)
    ptrs.push_back(r.data());
  if (static_cast<int>(ptrs.size()) != ctx.level.level)
    throw std::invalid_argument("full_multigrid: need one rhs per level");
  std::vector<double> hist(static_cast<std::size_t>(max_iterations) + 2);
  int its = 0;
  const int st = pmg_dd_full_multigrid(ctx.handle(), ptrs.data(), tol, max_iterations, &its, hist.data(),
                                       static_cast<int>(hist.size()));
  hist.resize(static_cast<std::size_t>(std::min<int>(its + 1, static_cast<int>(hist.size()))));
  check(st, hist);
  check(pmg_dd_gather_host(ctx.handle(), PMG_DD_X, x.data()));
  return FmgStats{its, hist};
}

}  // namespace pmgb
