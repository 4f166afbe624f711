// Host-side setup of one multigrid level (f64): the 1D finite-element
// building blocks, the patch fast-diagonalisation data and the grid-transfer
// embedding. Runs once per level and is uploaded to the device; never on the
// solve path.
//
// Mirrors (by behaviour, not by code) the reference's setup layer:
//   element.cpp:38-225        Gauss-Lobatto / Gauss-Legendre, Lagrange basis,
//                             1D cell matrices, 1D chain assembly
//   fastdiag.cpp:19-159       patch 1D matrices, generalized eigenpairs
//   level_context.cpp:21-34   (2k+1)x(k+1) prolongation (embedding) matrix
//   operator.cpp:283-411      right-hand side / L2 error quadrature (host)
#pragma once

#include <cstdint>
#include <vector>

namespace pmgb
{

// Row-major dense matrix, rows = outputs.
struct Dense
{
  int rows = 0, cols = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double &operator()(int i, int j) { return a[static_cast<size_t>(i) * cols + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * cols + j]; }
};

std::vector<double> lobatto_nodes(int k);                       // k+1 nodes on [0,1]
void gauss_rule(int q, std::vector<double> &x, std::vector<double> &w);  // on [0,1]
std::vector<double> lagrange_eval(const std::vector<double> &nodes, double x);
std::vector<double> lagrange_deriv(const std::vector<double> &nodes, double x);

struct LevelSetup
{
  int dim = 3, k = 1, level = 1;
  int n = 2;          // cells per dim
  int64_t m = 1;      // dofs per dim
  int64_t N = 1;      // total dofs
  double h = 0.5;

  Dense cell_mass, cell_stiff;  // (k+1)^2
  Dense mass_if, stiff_if;      // (2k-1) x (2k+1): interior rows of the 2-cell patch matrices
  Dense mass_ii, stiff_ii;      // (2k-1)^2
  Dense S;                      // (2k-1)^2 generalized eigenvectors (columns)
  std::vector<double> lambda;   // 2k-1, ascending
  std::vector<double> inv_sums; // (2k-1)^dim, direction 0 fastest
  Dense prolongation;           // (2k+1) x (k+1)
  // even-odd form for the fused kernel (layout of PatchMatsEO<double,k>):
  // Me | Mo | Ae | Ao | Se | So, eigen-modes reordered even-first (eo_perm)
  std::vector<double> eo_mats;
  std::vector<int> eo_perm;        // reordered mode c -> original column
  std::vector<double> inv_sums_eo; // inverse eigenvalue sums in reordered mode order
  // Banded rows of the global 1D matrices, indexed by lattice residue
  // r = p mod k and offset o = q - p + k in [0, 2k].
  std::vector<double> band_mass, band_stiff;  // k * (2k+1)
};

LevelSetup make_level_setup(int dim, int k, int level);

// Generalized symmetric-definite eigenproblem A S = M S diag(lambda):
// Cholesky M = L L^T, cyclic Jacobi on L^{-1} A L^{-T}, ascending order,
// M-orthonormal columns, first non-negligible component positive.
void generalized_eigen(const Dense &A, const Dense &M, Dense &S, std::vector<double> &lambda);

// b_i = int f phi_i with (k+2)-point Gauss per direction; kind 0: f = 1,
// kind 1: f = d pi^2 prod sin(pi x_a).
std::vector<double> compute_rhs(int dim, int k, int level, int kind);
// 1D factor of compute_rhs: the load vector of g = 1 or sin(pi x) on the
// interior lattice (the d-D right-hand side is its tensor power times 1 or
// d pi^2)
std::vector<double> rhs_1d(int k, int n, bool sine);
double l2_error_sin(int dim, int k, int level, const double *x);

}  // namespace pmgb
