// Host setup for one level — see setup.hpp for the reference mapping.
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

namespace pmgb
{

namespace
{

// P_n(x) and P_n'(x) on [-1,1] by the three-term recurrence.
void legendre_pd(int n, double x, double &p, double &dp)
{
  double pm1 = 1.0, pc = x;
  if (n == 0)
  {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int j = 2; j <= n; ++j)
  {
    const double pn = ((2 * j - 1) * x * pc - (j - 1) * pm1) / j;
    pm1 = pc;
    pc = pn;
  }
  p = pc;
  dp = n * (pm1 - x * pc) / (1.0 - x * x);
}

}  // namespace

std::vector<double> lobatto_nodes(int k)
{
  if (k < 1)
    throw std::invalid_argument("lobatto_nodes: degree must be >= 1");
  // interior nodes: zeros of P_k'; Newton on P_k' with the Chebyshev-Lobatto
  // guesses, using (1-x^2) P_k'' = 2x P_k' - k(k+1) P_k.
  std::vector<double> t(k + 1);
  t[0] = -1.0;
  t[k] = 1.0;
  for (int i = 1; i < k; ++i)
  {
    double x = -std::cos(M_PI * i / k);
    for (int it = 0; it < 60; ++it)
    {
      double p, dp;
      legendre_pd(k, x, p, dp);
      const double d2p = (2.0 * x * dp - k * (k + 1.0) * p) / (1.0 - x * x);
      const double dx = dp / d2p;
      x -= dx;
      if (std::fabs(dx) < 1e-16)
        break;
    }
    t[i] = x;
  }
  std::sort(t.begin(), t.end());
  std::vector<double> z(k + 1);
  for (int i = 0; i <= k; ++i)
    z[i] = 0.5 * (t[i] + 1.0);
  // exact symmetry about 1/2
  for (int i = 0; i <= k / 2; ++i)
  {
    const double lo = 0.5 * (z[i] + (1.0 - z[k - i]));
    z[i] = lo;
    z[k - i] = 1.0 - lo;
  }
  if (k % 2 == 0)
    z[k / 2] = 0.5;
  z[0] = 0.0;
  z[k] = 1.0;
  return z;
}

void gauss_rule(int q, std::vector<double> &x, std::vector<double> &w)
{
  if (q < 1)
    throw std::invalid_argument("gauss_rule: need at least one point");
  x.assign(q, 0.0);
  w.assign(q, 0.0);
  for (int i = 0; i < q; ++i)
  {
    // i-th root from the top, guess cos(pi (i + 3/4) / (q + 1/2))
    double t = std::cos(M_PI * (i + 0.75) / (q + 0.5));
    double p = 0, dp = 1;
    for (int it = 0; it < 60; ++it)
    {
      legendre_pd(q, t, p, dp);
      const double dt = p / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-16)
        break;
    }
    legendre_pd(q, t, p, dp);
    // ascending order on [0,1]
    x[q - 1 - i] = 0.5 * (1.0 + t);
    w[q - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);  // 2/((1-t^2)P'^2) * 1/2
  }
  for (int i = 0; i < q / 2; ++i)
  {
    const double a = 0.5 * (x[i] + 1.0 - x[q - 1 - i]);
    x[i] = a;
    x[q - 1 - i] = 1.0 - a;
    const double ww = 0.5 * (w[i] + w[q - 1 - i]);
    w[i] = w[q - 1 - i] = ww;
  }
  if (q % 2 == 1)
    x[q / 2] = 0.5;
}

std::vector<double> lagrange_eval(const std::vector<double> &nodes, double x)
{
  const int n = static_cast<int>(nodes.size());
  std::vector<double> v(n, 1.0);
  for (int j = 0; j < n; ++j)
    for (int l = 0; l < n; ++l)
      if (l != j)
        v[j] *= (x - nodes[l]) / (nodes[j] - nodes[l]);
  return v;
}

std::vector<double> lagrange_deriv(const std::vector<double> &nodes, double x)
{
  const int n = static_cast<int>(nodes.size());
  std::vector<double> g(n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
    {
      if (i == j)
        continue;
      double prod = 1.0 / (nodes[j] - nodes[i]);
      for (int l = 0; l < n; ++l)
        if (l != i && l != j)
          prod *= (x - nodes[l]) / (nodes[j] - nodes[l]);
      g[j] += prod;
    }
  return g;
}

void generalized_eigen(const Dense &A, const Dense &M, Dense &S, std::vector<double> &lambda)
{
  const int n = A.rows;
  if (A.cols != n || M.rows != n || M.cols != n)
    throw std::invalid_argument("generalized_eigen: matrices must be square, same size");
  // Cholesky M = L L^T
  Dense L(n, n);
  for (int j = 0; j < n; ++j)
  {
    double s = M(j, j);
    for (int p = 0; p < j; ++p)
      s -= L(j, p) * L(j, p);
    if (!(s > 0.0))
      throw std::runtime_error("generalized_eigen: mass matrix not SPD");
    L(j, j) = std::sqrt(s);
    for (int i = j + 1; i < n; ++i)
    {
      double t = M(i, j);
      for (int p = 0; p < j; ++p)
        t -= L(i, p) * L(j, p);
      L(i, j) = t / L(j, j);
    }
  }
  // Linv
  Dense Li(n, n);
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i)
    {
      double s = (i == c) ? 1.0 : 0.0;
      for (int p = 0; p < i; ++p)
        s -= L(i, p) * Li(p, c);
      Li(i, c) = s / L(i, i);
    }
  // C = Li A Li^T (symmetrised)
  Dense T(n, n), C(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
    {
      double s = 0;
      for (int p = 0; p < n; ++p)
        s += Li(i, p) * A(p, j);
      T(i, j) = s;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
    {
      double s = 0;
      for (int p = 0; p < n; ++p)
        s += T(i, p) * Li(j, p);
      C(i, j) = s;
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      C(i, j) = C(j, i) = 0.5 * (C(i, j) + C(j, i));
  // cyclic Jacobi
  Dense V(n, n);
  for (int i = 0; i < n; ++i)
    V(i, i) = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep)
  {
    double off = 0, tot = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
      {
        tot += C(i, j) * C(i, j);
        if (i != j)
          off += C(i, j) * C(i, j);
      }
    if (off <= 1e-34 * tot)
      break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q)
      {
        const double apq = C(p, q);
        if (std::fabs(apq) < 1e-300)
          continue;
        const double theta = (C(q, q) - C(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < n; ++r)
        {
          const double crp = C(r, p), crq = C(r, q);
          C(r, p) = c * crp - s * crq;
          C(r, q) = s * crp + c * crq;
        }
        for (int r = 0; r < n; ++r)
        {
          const double cpr = C(p, r), cqr = C(q, r);
          C(p, r) = c * cpr - s * cqr;
          C(q, r) = s * cpr + c * cqr;
        }
        for (int r = 0; r < n; ++r)
        {
          const double vrp = V(r, p), vrq = V(r, q);
          V(r, p) = c * vrp - s * vrq;
          V(r, q) = s * vrp + c * vrq;
        }
      }
  }
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i)
    order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return C(a, a) < C(b, b); });
  lambda.assign(n, 0.0);
  S = Dense(n, n);
  for (int jj = 0; jj < n; ++jj)
  {
    const int j = order[jj];
    lambda[jj] = C(j, j);
    // x = L^{-T} v
    std::vector<double> col(n);
    for (int i = 0; i < n; ++i)
    {
      double s = 0;
      for (int p = 0; p < n; ++p)
        s += Li(p, i) * V(p, j);
      col[i] = s;
    }
    double scale = 0;
    for (double v : col)
      scale = std::max(scale, std::fabs(v));
    double sign = 1.0;
    for (double v : col)
      if (std::fabs(v) > 1e-12 * scale)
      {
        sign = v > 0 ? 1.0 : -1.0;
        break;
      }
    for (int i = 0; i < n; ++i)
      S(i, jj) = sign * col[i];
  }
}

LevelSetup make_level_setup(int dim, int k, int level)
{
  if (dim != 2 && dim != 3)
    throw std::invalid_argument("dim must be 2 or 3, got " + std::to_string(dim));
  if (k < 1 || k > 7)
    throw std::invalid_argument("degree must be in 1..7, got " + std::to_string(k));
  if (level < 1)
    throw std::invalid_argument("level must be >= 1");
  LevelSetup s;
  s.dim = dim;
  s.k = k;
  s.level = level;
  s.n = 1 << level;
  s.m = static_cast<int64_t>(s.n) * k - 1;
  s.N = 1;
  for (int a = 0; a < dim; ++a)
    s.N *= s.m;
  s.h = 1.0 / s.n;
  const double h = s.h;

  // 1D cell matrices with the (k+1)-point Gauss rule: M = h Mhat, A = Ahat/h
  const auto nodes = lobatto_nodes(k);
  std::vector<double> qx, qw;
  gauss_rule(k + 1, qx, qw);
  s.cell_mass = Dense(k + 1, k + 1);
  s.cell_stiff = Dense(k + 1, k + 1);
  for (int q = 0; q <= k; ++q)
  {
    const auto v = lagrange_eval(nodes, qx[q]);
    const auto g = lagrange_deriv(nodes, qx[q]);
    for (int i = 0; i <= k; ++i)
      for (int j = 0; j <= k; ++j)
      {
        s.cell_mass(i, j) += h * qw[q] * v[i] * v[j];
        s.cell_stiff(i, j) += (1.0 / h) * qw[q] * g[i] * g[j];
      }
  }

  // two-cell patch chain (2k+1 nodes), interior rows
  const int nc = 2 * k + 1, ni = 2 * k - 1;
  Dense pm(nc, nc), pa(nc, nc);
  for (int c = 0; c < 2; ++c)
    for (int i = 0; i <= k; ++i)
      for (int j = 0; j <= k; ++j)
      {
        pm(c * k + i, c * k + j) += s.cell_mass(i, j);
        pa(c * k + i, c * k + j) += s.cell_stiff(i, j);
      }
  s.mass_if = Dense(ni, nc);
  s.stiff_if = Dense(ni, nc);
  s.mass_ii = Dense(ni, ni);
  s.stiff_ii = Dense(ni, ni);
  for (int i = 0; i < ni; ++i)
  {
    for (int j = 0; j < nc; ++j)
    {
      s.mass_if(i, j) = pm(i + 1, j);
      s.stiff_if(i, j) = pa(i + 1, j);
    }
    for (int j = 0; j < ni; ++j)
    {
      s.mass_ii(i, j) = pm(i + 1, j + 1);
      s.stiff_ii(i, j) = pa(i + 1, j + 1);
    }
  }
  generalized_eigen(s.stiff_ii, s.mass_ii, s.S, s.lambda);

  size_t tot = 1;
  for (int a = 0; a < dim; ++a)
    tot *= ni;
  s.inv_sums.resize(tot);
  for (size_t idx = 0; idx < tot; ++idx)
  {
    size_t r = idx;
    double sum = 0.0;
    for (int a = 0; a < dim; ++a)
    {
      sum += s.lambda[r % ni];
      r /= ni;
    }
    s.inv_sums[idx] = 1.0 / sum;
  }

  // even-odd data: the two-cell patch is reflection symmetric, so the
  // interior-row matrices are centro-symmetric and every eigenvector is even
  // or odd. Reorder the modes even-first (K even, K-1 odd), keep the
  // ascending order inside each class.
  {
    const int K = k, HO = K > 1 ? K - 1 : 1;
    std::vector<int> even, odd;
    for (int j = 0; j < ni; ++j)
    {
      double de = 0, dodd = 0, nrm = 0;
      for (int i = 0; i < ni; ++i)
      {
        de = std::max(de, std::fabs(s.S(ni - 1 - i, j) - s.S(i, j)));
        dodd = std::max(dodd, std::fabs(s.S(ni - 1 - i, j) + s.S(i, j)));
        nrm = std::max(nrm, std::fabs(s.S(i, j)));
      }
      if (de <= 1e-10 * nrm)
        even.push_back(j);
      else if (dodd <= 1e-10 * nrm)
        odd.push_back(j);
      else
        throw std::runtime_error("patch eigenvector without reflection parity");
    }
    if (static_cast<int>(even.size()) != K || static_cast<int>(odd.size()) != K - 1)
      throw std::runtime_error("unexpected even/odd eigenvector counts");
    s.eo_perm = even;
    s.eo_perm.insert(s.eo_perm.end(), odd.begin(), odd.end());
    auto &o = s.eo_mats;
    o.clear();
    auto push_eo = [&](const Dense &B) {
      for (int i = 0; i < K; ++i)
        for (int j = 0; j <= K; ++j)
          o.push_back(j < K ? 0.5 * (B(i, j) + B(i, nc - 1 - j)) : B(i, K));
      for (int i = 0; i < HO; ++i)
        for (int j = 0; j < K; ++j)
          o.push_back(i < K - 1 ? 0.5 * (B(i, j) - B(i, nc - 1 - j)) : 0.0);
    };
    push_eo(s.mass_if);
    push_eo(s.stiff_if);
    for (int i = 0; i < K; ++i)
      for (int c = 0; c < K; ++c)
        o.push_back(s.S(i, s.eo_perm[c]));
    for (int i = 0; i < HO; ++i)
      for (int c = 0; c < HO; ++c)
        o.push_back((i < K - 1 && c < K - 1) ? s.S(i, s.eo_perm[K + c]) : 0.0);
    s.inv_sums_eo.resize(tot);
    for (size_t idx = 0; idx < tot; ++idx)
    {
      size_t r = idx;
      double sum = 0.0;
      for (int a = 0; a < dim; ++a)
      {
        sum += s.lambda[s.eo_perm[r % ni]];
        r /= ni;
      }
      s.inv_sums_eo[idx] = 1.0 / sum;
    }
  }

  // embedding of the coarse cell basis into the two fine cells
  s.prolongation = Dense(nc, k + 1);
  for (int f = 0; f < 2; ++f)
    for (int t = 0; t <= k; ++t)
    {
      const auto v = lagrange_eval(nodes, 0.5 * (f + nodes[t]));
      for (int j = 0; j <= k; ++j)
        s.prolongation(f * k + t, j) = v[j];
    }

  // banded rows of the global 1D matrices (lattice residue r = p mod k)
  const int w = 2 * k + 1;
  s.band_mass.assign(static_cast<size_t>(k) * w, 0.0);
  s.band_stiff.assign(static_cast<size_t>(k) * w, 0.0);
  for (int r = 0; r < k; ++r)
  {
    if (r == 0)
    {
      // vertex node: left cell row k, right cell row 0
      for (int t = 0; t <= k; ++t)
      {
        s.band_mass[t] += s.cell_mass(k, t);
        s.band_stiff[t] += s.cell_stiff(k, t);
        s.band_mass[k + t] += s.cell_mass(0, t);
        s.band_stiff[k + t] += s.cell_stiff(0, t);
      }
    }
    else
    {
      for (int t = 0; t <= k; ++t)
      {
        s.band_mass[r * w + (t - r + k)] = s.cell_mass(r, t);
        s.band_stiff[r * w + (t - r + k)] = s.cell_stiff(r, t);
      }
    }
  }
  return s;
}

// 1D load vector of g over the level lattice interior: sum over cells of
// sum_q w h g(x_q) phi_t(x_q), k+2 Gauss points.
std::vector<double> rhs_1d(int k, int n, bool sine)
{
  const auto nodes = lobatto_nodes(k);
  std::vector<double> qx, qw;
  gauss_rule(k + 2, qx, qw);
  const double h = 1.0 / n;
  std::vector<double> lat(static_cast<size_t>(n) * k + 1, 0.0);
  for (int c = 0; c < n; ++c)
    for (int q = 0; q < k + 2; ++q)
    {
      const double xq = (c + qx[q]) * h;
      const double g = sine ? std::sin(M_PI * xq) : 1.0;
      const auto v = lagrange_eval(nodes, qx[q]);
      for (int t = 0; t <= k; ++t)
        lat[static_cast<size_t>(c) * k + t] += qw[q] * h * g * v[t];
    }
  return std::vector<double>(lat.begin() + 1, lat.end() - 1);
}

std::vector<double> compute_rhs(int dim, int k, int level, int kind)
{
  const int n = 1 << level;
  const auto b1 = rhs_1d(k, n, kind == 1);
  const int64_t m = static_cast<int64_t>(b1.size());
  const double c = kind == 1 ? dim * M_PI * M_PI : 1.0;
  int64_t N = 1;
  for (int a = 0; a < dim; ++a)
    N *= m;
  std::vector<double> b(N);
  if (dim == 2)
  {
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < m; ++i)
        b[i + m * j] = c * b1[j] * b1[i];
  }
  else
  {
    for (int64_t l = 0; l < m; ++l)
      for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < m; ++i)
          b[i + m * (j + m * l)] = c * b1[l] * b1[j] * b1[i];
  }
  return b;
}

double l2_error_sin(int dim, int k, int level, const double *x)
{
  const int n = 1 << level;
  const int q = k + 2;
  const auto nodes = lobatto_nodes(k);
  std::vector<double> qx, qw;
  gauss_rule(q, qx, qw);
  const double h = 1.0 / n;
  const int64_t m = static_cast<int64_t>(n) * k - 1;
  const int64_t nl = static_cast<int64_t>(n) * k + 1, nq = static_cast<int64_t>(n) * q;
  std::vector<std::vector<double>> shape(q);
  for (int iq = 0; iq < q; ++iq)
    shape[iq] = lagrange_eval(nodes, qx[iq]);
  // u on the lattice (zero boundary), evaluated direction by direction
  int64_t total = 1;
  for (int a = 0; a < dim; ++a)
    total *= nl;
  std::vector<double> u(total, 0.0);
  if (dim == 2)
  {
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < m; ++i)
        u[(i + 1) + nl * (j + 1)] = x[i + m * j];
  }
  else
  {
    for (int64_t l = 0; l < m; ++l)
      for (int64_t j = 0; j < m; ++j)
        for (int64_t i = 0; i < m; ++i)
          u[(i + 1) + nl * ((j + 1) + nl * (l + 1))] = x[i + m * (j + m * l)];
  }
  // contract each direction lattice(nl) -> quadrature(nq)
  std::vector<int64_t> ext(dim, nl);
  std::vector<double> cur = u;
  for (int dir = 0; dir < dim; ++dir)
  {
    int64_t inner = 1, outer = 1;
    for (int a = 0; a < dir; ++a)
      inner *= ext[a];
    for (int a = dir + 1; a < dim; ++a)
      outer *= ext[a];
    std::vector<double> nxt(static_cast<size_t>(inner * nq * outer), 0.0);
    for (int64_t o = 0; o < outer; ++o)
      for (int64_t c = 0; c < n; ++c)
        for (int iq = 0; iq < q; ++iq)
          for (int t = 0; t <= k; ++t)
          {
            const double wgt = shape[iq][t];
            const double *src = &cur[(o * nl + c * k + t) * inner];
            double *dst = &nxt[(o * nq + c * q + iq) * inner];
            for (int64_t s = 0; s < inner; ++s)
              dst[s] += wgt * src[s];
          }
    cur.swap(nxt);
    ext[dir] = nq;
  }
  std::vector<double> xq(nq), wq(nq);
  for (int64_t c = 0; c < n; ++c)
    for (int iq = 0; iq < q; ++iq)
    {
      xq[c * q + iq] = (c + qx[iq]) * h;
      wq[c * q + iq] = qw[iq] * h;
    }
  double err2 = 0.0;
  if (dim == 2)
  {
    for (int64_t j = 0; j < nq; ++j)
      for (int64_t i = 0; i < nq; ++i)
      {
        const double e = cur[i + nq * j] - std::sin(M_PI * xq[i]) * std::sin(M_PI * xq[j]);
        err2 += wq[i] * wq[j] * e * e;
      }
  }
  else
  {
    for (int64_t l = 0; l < nq; ++l)
      for (int64_t j = 0; j < nq; ++j)
        for (int64_t i = 0; i < nq; ++i)
        {
          const double e = cur[i + nq * (j + nq * l)] -
                           std::sin(M_PI * xq[i]) * std::sin(M_PI * xq[j]) * std::sin(M_PI * xq[l]);
          err2 += wq[i] * wq[j] * wq[l] * e * e;
        }
  }
  return std::sqrt(err2);
}

}  // namespace pmgb
