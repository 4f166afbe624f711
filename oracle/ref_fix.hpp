// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Force-included (`-include`) when oracle/Makefile compiles the UNMODIFIED
// reference sources in /root/reference/proj/src into oracle/_ref/.
//
// The reference does not compile as shipped under GCC 13 / C++20:
// /root/reference/proj/src/multigrid.cpp:333 calls
//   compute_residual(lev, x, b, r, ctx.threads)
// with `x` a std::span<T>, while the only declaration
// (/root/reference/proj/include/pmg/multigrid.hpp:90-92) takes
// std::span<const T>; template argument deduction does not look through the
// span<T> -> span<const T> conversion. Instead of editing (or copying) the
// reference source we add the missing overload here; it forwards to the
// reference's own compute_residual with the const view, so behaviour is
// exactly what the reference author intended.
#pragma once
#include "pmg/multigrid.hpp"

namespace pmg
{
template <typename T>
void compute_residual(const LevelContext<T> &lev, std::span<T> x, std::span<const T> b,
                      std::span<T> r, int threads)
{
  compute_residual<T>(lev, std::span<const T>(x.data(), x.size()), b, r, threads);
}
}  // namespace pmg
