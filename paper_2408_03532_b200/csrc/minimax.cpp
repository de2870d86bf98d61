// Offline scope-table pipeline: the near-minimax
// polynomial coefficients of e^{i pi x} on |x| <= xi and the (eps, r) -> xi
// scope table, computed here instead of loaded from a reference-built file.
//
// Reference semantics (minimax.hpp:10-70, minimax.cpp:276-433):
//  * P(x) = sum_{j<r} w_j x^j with even-j coefficients real, odd-j imaginary;
//    the even part approximates cos(pi x), the odd part sin(pi x);
//  * achieved_error = max |P(x) - e^{i pi x}| measured a posteriori on the
//    uniform 4097-point grid over [-xi, xi];
//  * scope(eps, r) = largest xi (doubling bracket from 0.25, cap 64, then
//    bisection to relative width 1e-3, feasible endpoint) with
//    achieved_error <= eps; the table warm-starts each r at the previous xi.
//
// Algorithm (own formulation): each parity part becomes a weighted problem in
// v = (x/xi)^2 on [0, 1],
//    even: g(v) = cos(pi xi sqrt v),            weight 1,
//    odd : g(v) = sin(pi xi sqrt v) / sqrt v,   weight sqrt v,
// approximated by sum_k c_k T_k(2v - 1). It is solved by the discrete
// single-point exchange (Stiefel's form of the Remez method) on a 2049-point
// Chebyshev-clustered grid: a (d+2)-point alternating reference, the leveled
// linear system solved by Gaussian elimination with partial pivoting, and one
// point swapped per iteration for the grid point of largest weighted error,
// keeping the sign alternation, until that error exceeds the level by less
// than 1e-9 relative (or the level reaches the rounding floor). T_k(2v - 1) =
// T_{2k}(u) with u = x / xi turns the Chebyshev coefficients into monomials
// in u, which are rescaled by xi^-j. The coefficients are therefore not
// bit-identical to the reference's (whose exchange polishes extrema by golden
// section), but they are near-minimax and certified the same way; the tests
// compare records against the reference table (xi, r = min_degree) and the
// achieved error against eps.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "host.hpp"

namespace pftg {
namespace {

constexpr double kPi = 3.14159265358979323846;

struct Part {
  double xi;
  bool odd;
  int d;  // degree in v
  double g(double v) const {
    const double u = std::sqrt(v), t = kPi * xi * u;
    if (!odd) return std::cos(t);
    if (t < 1e-4) return kPi * xi * (1.0 - t * t / 6.0 * (1.0 - t * t / 20.0));  // sin(t)/u near 0
    return std::sin(t) / u;
  }
  double w(double v) const { return odd ? std::sqrt(v) : 1.0; }
};

// T_0..T_d at s (three-term recurrence)
void cheb_all(double s, int d, double* T) {
  T[0] = 1.0;
  if (d >= 1) T[1] = s;
  for (int k = 2; k <= d; ++k) T[k] = 2.0 * s * T[k - 1] - T[k - 2];
}

double poly(const std::vector<double>& c, double v) {
  // Clenshaw on T_k(2v - 1)
  const double s = 2.0 * v - 1.0;
  double b1 = 0.0, b2 = 0.0;
  for (int k = (int)c.size() - 1; k >= 1; --k) {
    const double b0 = 2.0 * s * b1 - b2 + c[k];
    b2 = b1;
    b1 = b0;
  }
  return s * b1 - b2 + c[0];
}

// Solve A x = b (n x n, row-major) by Gaussian elimination with partial pivoting.
bool gauss(std::vector<double>& A, std::vector<double>& b, int n) {
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::abs(A[r * n + col]) > std::abs(A[piv * n + col])) piv = r;
    if (A[piv * n + col] == 0.0 || !std::isfinite(A[piv * n + col])) return false;
    if (piv != col) {
      for (int k = 0; k < n; ++k) std::swap(A[col * n + k], A[piv * n + k]);
      std::swap(b[col], b[piv]);
    }
    for (int r = col + 1; r < n; ++r) {
      const double f = A[r * n + col] / A[col * n + col];
      if (f == 0.0) continue;
      for (int k = col; k < n; ++k) A[r * n + k] -= f * A[col * n + k];
      b[r] -= f * b[col];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    double s = b[r];
    for (int k = r + 1; k < n; ++k) s -= A[r * n + k] * b[k];
    b[r] = s / A[r * n + r];
  }
  return true;
}

// Chebyshev-clustered grid in v on (0, 1]; the odd part's grid is clustered in
// u = sqrt(v) and excludes u = 0, where its weight vanishes.
std::vector<double> make_grid(const Part& p, int n) {
  std::vector<double> g(n);
  for (int i = 0; i < n; ++i) {
    if (!p.odd) {
      g[i] = 0.5 * (1.0 - std::cos(kPi * i / (n - 1)));
    } else {
      const double u = std::sin(0.5 * kPi * (i + 1) / n);
      g[i] = u * u;
    }
  }
  return g;
}

std::vector<double> solve_part(const Part& p) {
  const int d = p.d, m = d + 2;
  const std::vector<double> grid = make_grid(p, 2049);
  const int G = (int)grid.size();
  std::vector<double> gv(G), wv(G);
  for (int i = 0; i < G; ++i) {
    gv[i] = p.g(grid[i]);
    wv[i] = p.w(grid[i]);
  }
  // initial reference: m grid points spread like Chebyshev extrema
  std::vector<int> ref(m);
  for (int i = 0; i < m; ++i) {
    const double t = 0.5 * (1.0 - std::cos(kPi * i / (m - 1)));
    ref[i] = std::min(G - 1, std::max(0, (int)std::lround(t * (G - 1))));
  }
  for (int i = 1; i < m; ++i) ref[i] = std::max(ref[i], ref[i - 1] + 1);
  for (int i = m - 2; i >= 0; --i) ref[i] = std::min(ref[i], ref[i + 1] - 1);

  std::vector<double> c(d + 1, 0.0), best;
  double best_err = std::numeric_limits<double>::infinity();
  std::vector<double> T(d + 1);
  const double floor = 1e-15 * (1.0 + kPi * p.xi);
  for (int it = 0; it < 400; ++it) {
    std::vector<double> A((size_t)m * m), b(m);
    for (int i = 0; i < m; ++i) {
      const double v = grid[ref[i]];
      cheb_all(2.0 * v - 1.0, d, T.data());
      for (int k = 0; k <= d; ++k) A[(size_t)i * m + k] = T[k];
      A[(size_t)i * m + d + 1] = ((i & 1) ? -1.0 : 1.0) / wv[ref[i]];
      b[i] = gv[ref[i]];
    }
    if (!gauss(A, b, m)) break;
    c.assign(b.begin(), b.begin() + d + 1);
    const double level = std::abs(b[d + 1]);
    // weighted error on the grid and its maximum
    int imax = 0;
    double emax = 0.0;
    std::vector<double> e(G);
    for (int i = 0; i < G; ++i) {
      e[i] = wv[i] * (gv[i] - poly(c, grid[i]));
      if (std::abs(e[i]) > emax) {
        emax = std::abs(e[i]);
        imax = i;
      }
    }
    if (emax < best_err) {
      best_err = emax;
      best = c;
    }
    if (emax <= level * (1.0 + 1e-9) + floor) break;
    // single-point exchange keeping alternation of the error signs
    const auto sgn = [&](int i) { return e[i] >= 0.0; };
    const int pos = (int)(std::upper_bound(ref.begin(), ref.end(), imax) - ref.begin());
    if (pos > 0 && ref[pos - 1] == imax) break;  // already in the reference: converged on the grid
    if (pos == 0) {
      if (sgn(imax) == sgn(ref[0])) {
        ref[0] = imax;
      } else {
        for (int i = m - 1; i > 0; --i) ref[i] = ref[i - 1];
        ref[0] = imax;
      }
    } else if (pos == m) {
      if (sgn(imax) == sgn(ref[m - 1])) {
        ref[m - 1] = imax;
      } else {
        for (int i = 0; i < m - 1; ++i) ref[i] = ref[i + 1];
        ref[m - 1] = imax;
      }
    } else {
      if (sgn(imax) == sgn(ref[pos - 1])) ref[pos - 1] = imax;
      else ref[pos] = imax;
    }
  }
  return best.empty() ? c : best;
}

// monomial coefficients (in u) of T_0..T_kmax
std::vector<std::vector<double>> cheb_to_mono(int kmax) {
  std::vector<std::vector<double>> t(kmax + 1, std::vector<double>(kmax + 1, 0.0));
  t[0][0] = 1.0;
  if (kmax >= 1) t[1][1] = 1.0;
  for (int k = 2; k <= kmax; ++k)
    for (int j = 0; j <= k; ++j) t[k][j] = (j > 0 ? 2.0 * t[k - 1][j - 1] : 0.0) - t[k - 2][j];
  return t;
}

double certify(const std::vector<cd>& w, double xi) {
  constexpr int kGrid = 4096;  // minimax.cpp:332-340
  double err = 0.0;
  for (int i = 0; i <= kGrid; ++i) {
    const double x = -xi + 2.0 * xi * i / kGrid;
    cd acc(0.0, 0.0);
    for (int j = (int)w.size() - 1; j >= 0; --j) acc = acc * x + w[j];
    err = std::max(err, std::abs(acc - cd(std::cos(kPi * x), std::sin(kPi * x))));
  }
  return err;
}

}  // namespace

// best_approx (minimax.hpp:28): r coefficients on |x| <= xi; returns the
// certified error in *achieved.
std::vector<cd> best_approx_own(int r, double xi, double* achieved) {
  if (r < 1 || r > 64) throw std::invalid_argument("best_approx: r out of range");
  if (!(xi > 0.0) || !std::isfinite(xi)) throw std::invalid_argument("best_approx: xi must be positive");
  const int de = (r - 1) / 2, dodd = r >= 2 ? (r - 2) / 2 : -1;
  const std::vector<double> ce = solve_part(Part{xi, false, de});
  std::vector<double> co;
  if (dodd >= 0) co = solve_part(Part{xi, true, dodd});
  const auto tm = cheb_to_mono(std::max(2 * std::max(de, dodd), 1));
  std::vector<double> mono(r, 0.0);
  for (int k = 0; k <= de; ++k)
    for (int j = 0; j <= 2 * k; ++j) mono[j] += ce[k] * tm[2 * k][j];
  for (int k = 0; k <= dodd; ++k)
    for (int j = 0; j <= 2 * k; ++j) mono[j + 1] += co[k] * tm[2 * k][j];
  std::vector<cd> w(r);
  double s = 1.0;
  for (int j = 0; j < r; ++j) {
    w[j] = (j % 2 == 0) ? cd(mono[j] * s, 0.0) : cd(0.0, mono[j] * s);
    s /= xi;
  }
  if (achieved) *achieved = certify(w, xi);
  return w;
}

// ScopeTable::compute (minimax.hpp:48-49, minimax.cpp:388-433): records
// eps-major, r ascending.
Table table_compute(const std::vector<double>& eps_list, int max_r) {
  if (eps_list.empty() || max_r < 1) throw std::invalid_argument("ScopeTable: empty spec");
  Table t;
  t.max_r = max_r;
  for (double eps : eps_list) {
    if (!(eps > 0.0)) throw std::invalid_argument("scope: eps must be positive");
    double warm = 0.0;
    for (int r = 1; r <= max_r; ++r) {
      auto ok = [&](double xi) {
        double e;
        best_approx_own(r, xi, &e);
        return e <= eps;
      };
      double lo = (warm > 0.0 && ok(warm)) ? warm : 0.0;
      if (lo == 0.0) {
        lo = 0.25;
        while (lo >= 1e-12 && !ok(lo)) lo *= 0.5;
      }
      Record rec;
      rec.eps = eps;
      rec.r = r;
      if (lo < 1e-12) {
        rec.xi = 0.0;
        rec.achieved_error = 0.0;
        rec.coeff.assign(r, cd(0.0, 0.0));
      } else {
        double hi = std::max(2.0 * lo, lo + 0.05);
        while (hi < 64.0 && ok(hi)) {
          lo = hi;
          hi *= 2.0;
        }
        while (hi - lo > 1e-3 * lo) {
          const double mid = 0.5 * (lo + hi);
          if (ok(mid)) lo = mid;
          else hi = mid;
        }
        rec.xi = lo;
        rec.coeff = best_approx_own(r, lo, &rec.achieved_error);
      }
      warm = rec.xi;
      t.records.push_back(std::move(rec));
    }
  }
  return t;
}

// ScopeTable::save (minimax.cpp:470-493): the "pft-scope-table v1" text format.
void table_save(const Table& t, const std::string& path) {
  std::ofstream os(path);
  if (!os) throw std::runtime_error("ScopeTable: cannot open " + path);
  os << "pft-scope-table v1\n";
  os << "# record <eps> <r> <xi> <achieved_error> <w0.re> <w0.im> ... (r pairs)\n";
  char buf[64];
  for (const Record& rec : t.records) {
    std::snprintf(buf, sizeof buf, "%.6e", rec.eps);
    os << "record " << buf << ' ' << rec.r << ' ';
    std::snprintf(buf, sizeof buf, "%.17g %.17g", rec.xi, rec.achieved_error);
    os << buf;
    for (const cd& c : rec.coeff) {
      std::snprintf(buf, sizeof buf, " %.17g %.17g", c.real(), c.imag());
      os << buf;
    }
    os << '\n';
  }
  if (!os) throw std::runtime_error("ScopeTable: write failed");
}

}  // namespace pftg
