// pmg_b200.hpp — header-only C++ shim over the C-ABI (pmg_b200.h) with the
// reference's names and calling conventions (/root/reference/proj/include/pmg):
// host std::span vectors in, exceptions out. A reference user swaps
//   #include "pmg/multigrid.hpp"            ->  #include "pmg_b200.hpp"
//   pmg::make_multigrid_context<double>(..)  ->  pmgb::make_multigrid_context<double>(..)
// and keeps the call sites (smooth, apply_laplacian, v_cycle, full_multigrid).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
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

// ~ LevelContext<T> (level_context.hpp:17-26): borrowed from a context or owned
template <typename T>
class LevelContext
{
 public:
  LevelContext(int dim, int degree, int level, int device = 0)
  {
    check(pmg_level_create(dim, degree, level, dtype_of<T>(), device, &h_));
    owned_ = true;
  }
  explicit LevelContext(pmg_level borrowed) : h_(borrowed) {}
  LevelContext(const LevelContext &) = delete;
  LevelContext &operator=(const LevelContext &) = delete;
  LevelContext(LevelContext &&o) noexcept : h_(o.h_), owned_(o.owned_) { o.h_ = nullptr; }
  ~LevelContext()
  {
    if (owned_ && h_)
      pmg_level_destroy(h_);
  }
  pmg_level handle() const { return h_; }
  std::int64_t total_dofs() const
  {
    std::int64_t m, N, P;
    check(pmg_level_info(h_, &m, &N, &P));
    return N;
  }

 private:
  pmg_level h_ = nullptr;
  bool owned_ = false;
};

// ~ MultigridContext<T> (multigrid.hpp:34-49)
template <typename T>
class MultigridContext
{
 public:
  MultigridContext(int dim, int degree, int finest_level,
                   SmootherVariant variant = SmootherVariant::fused, int device = 0)
  {
    check(pmg_mg_create(dim, degree, finest_level, dtype_of<T>(), static_cast<int>(variant), device,
                        &h_));
    for (int li = 0; li < pmg_mg_num_levels(h_); ++li)
      levels.emplace_back(pmg_mg_level(h_, li));
  }
  MultigridContext(const MultigridContext &) = delete;
  MultigridContext &operator=(const MultigridContext &) = delete;
  ~MultigridContext()
  {
    levels.clear();
    if (h_)
      pmg_mg_destroy(h_);
  }
  pmg_mg handle() const { return h_; }
  std::vector<LevelContext<T>> levels;

 private:
  pmg_mg h_ = nullptr;
};

// multigrid.hpp:51-54
template <typename T>
MultigridContext<T> make_multigrid_context(int dim, int degree, int finest_level,
                                           SmootherVariant variant = SmootherVariant::fused)
{
  return MultigridContext<T>(dim, degree, finest_level, variant);
}

// smoother.hpp:45-47 (threads / workspace are accepted for signature parity)
template <typename T>
void smooth(const LevelContext<T> &ctx, std::span<T> x, std::span<const T> b,
            SmootherVariant variant = SmootherVariant::fused, int /*threads*/ = 1)
{
  if (static_cast<std::int64_t>(x.size()) != ctx.total_dofs() ||
      static_cast<std::int64_t>(b.size()) != ctx.total_dofs())
    throw std::invalid_argument("smooth: vector size does not match level");
  check(pmg_smooth_host(ctx.handle(), static_cast<int>(variant), x.data(), b.data()));
}

// operator.hpp:47-50
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
void compute_residual(const LevelContext<T> &ctx, std::span<const T> x, std::span<const T> b,
                      std::span<T> r)
{
  check(pmg_compute_residual_host(ctx.handle(), x.data(), b.data(), r.data()));
}

// multigrid.hpp:56-63
template <typename T>
void prolongate(const LevelContext<T> &c, const LevelContext<T> &f, std::span<const T> xc,
                std::span<T> xf)
{
  check(pmg_prolongate_host(c.handle(), f.handle(), xc.data(), xf.data()));
}
template <typename T>
void restrict_vector(const LevelContext<T> &c, const LevelContext<T> &f, std::span<const T> rf,
                     std::span<T> rc)
{
  check(pmg_restrict_vector_host(c.handle(), f.handle(), rf.data(), rc.data()));
}

// multigrid.hpp:68-69
template <typename T>
void v_cycle(MultigridContext<T> &ctx, int li, std::span<T> x, std::span<const T> b)
{
  check(pmg_v_cycle_host(ctx.handle(), li, x.data(), b.data()));
}

}  // namespace pmgb
