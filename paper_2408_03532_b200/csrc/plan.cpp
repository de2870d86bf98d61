// Offline phase on the host: scope table, plan construction, plan files.
//
// Mirrors /root/reference/proj/core/src/minimax.cpp:435-522 (ScopeTable
// find/record/min_degree/load) and src/pft.cpp:33-76, 103-112, 266-366
// (pft_plan_1d/2d, save_plan/load_plan_2d with raw_io.cpp:27-76 PTYC blocks).
// B and W are computed with the same operation order as the reference so the
// tables are bit-identical; the GPU only ever sees casts of these doubles.
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "host.hpp"

namespace pftg {

namespace {
constexpr double kPi = 3.14159265358979323846;  // pft.cpp:17
}

// ---- scope table (minimax.cpp:495-522) ----
Table table_load(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw std::runtime_error("ScopeTable: cannot open " + path);
  std::string line;
  if (!std::getline(is, line) || line != "pft-scope-table v1")
    throw std::runtime_error("ScopeTable: bad header in " + path);
  Table t;
  while (std::getline(is, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string tag;
    Record rec;
    if (!(ls >> tag >> rec.eps >> rec.r >> rec.xi >> rec.achieved_error) || tag != "record")
      throw std::runtime_error("ScopeTable: malformed record line");
    for (int j = 0; j < rec.r; ++j) {
      double re, im;
      if (!(ls >> re >> im)) throw std::runtime_error("ScopeTable: truncated coefficients");
      rec.coeff.emplace_back(re, im);
    }
    t.max_r = std::max(t.max_r, rec.r);
    t.records.push_back(std::move(rec));
  }
  if (t.records.empty()) throw std::runtime_error("ScopeTable: no records in " + path);
  return t;
}

const Record* table_find(const Table& t, double eps, int r) {
  for (const auto& rec : t.records)
    if (rec.r == r && std::abs(rec.eps - eps) <= 1e-9 * eps) return &rec;
  return nullptr;
}

// minimax.cpp:455-468
int table_min_degree(const Table& t, double eps, double target) {
  double best = 0.0;
  for (int r = 1; r <= t.max_r; ++r) {
    const Record* rec = table_find(t, eps, r);
    if (!rec) continue;
    best = std::max(best, rec->xi);
    if (rec->xi >= target) return r;
  }
  std::ostringstream msg;
  msg << "min_degree: target scope " << target << " infeasible for eps " << eps << " up to r="
      << t.max_r << " (best achievable " << best
      << "); reduce the band/segment ratio or relax eps";
  throw std::invalid_argument(msg.str());
}

// ---- plans (pft.cpp:33-76) ----
Axis plan_1d(std::size_t n, std::size_t mt, std::size_t p, double eps, const Table& table) {
  if (p < 2 || p > n || n % p != 0)
    throw std::invalid_argument("pft_plan_1d: p must divide n, 2 <= p <= n");
  const std::size_t q = n / p;
  if (q < 2) throw std::invalid_argument("pft_plan_1d: need q = n/p >= 2");
  if (mt < 1 || 2 * mt > n) throw std::invalid_argument("pft_plan_1d: need 1 <= mt and 2*mt <= n");
  Axis a;
  a.n = n;
  a.p = p;
  a.q = q;
  a.mt = mt;
  a.eps = eps;
  a.r = table_min_degree(table, eps, static_cast<double>(mt) / static_cast<double>(p));
  const Record* rec = table_find(table, eps, a.r);
  if (!rec) {
    std::ostringstream msg;
    msg << "ScopeTable: no record for eps=" << eps << " r=" << a.r;
    throw std::invalid_argument(msg.str());
  }
  const std::size_t r = static_cast<std::size_t>(a.r);
  a.B.assign(q * r, cd(0.0, 0.0));
  for (std::size_t l = 0; l < q; ++l) {
    const double x = 1.0 - 2.0 * static_cast<double>(l) / static_cast<double>(q);
    double xpow = 1.0;
    for (std::size_t j = 0; j < r; ++j) {
      a.B[l * r + j] = rec->coeff[j] * xpow;
      xpow *= x;
    }
  }
  a.W.assign((2 * mt + 1) * r, cd(0.0, 0.0));
  for (std::size_t i = 0; i < 2 * mt + 1; ++i) {
    const double t = static_cast<double>(i) - static_cast<double>(mt);
    const double base = t / static_cast<double>(p);
    const cd tw = std::polar(1.0, -kPi * base);
    double bpow = 1.0;
    for (std::size_t j = 0; j < r; ++j) {
      a.W[i * r + j] = tw * bpow;
      bpow *= base;
    }
  }
  return a;
}

// ---- plan files (pft.cpp:266-366; raw_io.cpp:27-76) ----
namespace {

void write_block(std::ostream& os, const std::vector<cd>& v, std::uint32_t rows, std::uint32_t cols) {
  os.write("PTYC", 4);
  const std::uint32_t hdr[3] = {1u, rows, cols};
  os.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  os.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(cd)));
  if (!os) throw std::runtime_error("raw field: write failed");
}

std::vector<cd> read_block(std::istream& is, std::uint32_t& rows, std::uint32_t& cols) {
  char magic[4] = {};
  if (!is.read(magic, 4) || std::memcmp(magic, "PTYC", 4) != 0)
    throw std::runtime_error("raw field: bad magic");
  std::uint32_t hdr[3];
  if (!is.read(reinterpret_cast<char*>(hdr), sizeof hdr)) throw std::runtime_error("raw field: truncated header");
  if (hdr[0] != 1u) throw std::runtime_error("raw field: unsupported version");
  rows = hdr[1];
  cols = hdr[2];
  if (rows == 0 || cols == 0) throw std::runtime_error("raw field: empty shape");
  std::vector<cd> v(static_cast<std::size_t>(rows) * cols);
  if (!is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(cd))))
    throw std::runtime_error("raw field: truncated payload");
  for (const auto& z : v)
    if (!std::isfinite(z.real()) || !std::isfinite(z.imag()))
      throw std::runtime_error("raw field: non-finite payload");
  return v;
}

std::string fmt_eps(double eps) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", eps);
  return buf;
}

}  // namespace

void plan_save(const Axis& a1, const Axis& a2, const std::string& path) {
  struct { const Axis& a1; const Axis& a2; } plan{a1, a2};
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("cannot open " + path + " for writing");
  os << "pft-plan-2d v1\n";
  const Axis* ax[2] = {&plan.a1, &plan.a2};
  for (int k = 0; k < 2; ++k) {
    const char* s = k == 0 ? "1" : "2";
    os << "n" << s << " " << ax[k]->n << " p" << s << " " << ax[k]->p << " q" << s << " " << ax[k]->q
       << " mt" << s << " " << ax[k]->mt << " r" << s << " " << ax[k]->r << "\n";
  }
  os << "eps " << fmt_eps(plan.a1.eps) << "\n---\n";
  write_block(os, plan.a1.B, plan.a1.q, plan.a1.r);
  write_block(os, plan.a2.B, plan.a2.q, plan.a2.r);
  write_block(os, plan.a1.W, 2 * plan.a1.mt + 1, plan.a1.r);
  write_block(os, plan.a2.W, 2 * plan.a2.mt + 1, plan.a2.r);
  if (!os) throw std::runtime_error("write failure on " + path);
}

void plan_load(Axis& a1, Axis& a2, const std::string& path) {
  struct { Axis& a1; Axis& a2; } plan{a1, a2};
  std::ifstream is(path, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open " + path);
  std::string line;
  if (!std::getline(is, line) || line != "pft-plan-2d v1")
    throw std::runtime_error(path + " is not a pft-plan-2d v1 file");
  Axis* ax[2] = {&plan.a1, &plan.a2};
  for (int k = 0; k < 2; ++k) {
    if (!std::getline(is, line)) throw std::runtime_error("truncated plan " + path);
    std::istringstream iss(line);
    std::string key;
    if (!(iss >> key >> ax[k]->n >> key >> ax[k]->p >> key >> ax[k]->q >> key >> ax[k]->mt >> key >> ax[k]->r))
      throw std::runtime_error("malformed plan axis line in " + path);
  }
  if (!std::getline(is, line) || line.rfind("eps ", 0) != 0)
    throw std::runtime_error("missing eps line in " + path);
  const double eps = std::stod(line.substr(4));
  if (!std::getline(is, line) || line != "---") throw std::runtime_error("missing block separator in " + path);
  plan.a1.eps = plan.a2.eps = eps;
  std::uint32_t rows[4], cols[4];
  plan.a1.B = read_block(is, rows[0], cols[0]);
  plan.a2.B = read_block(is, rows[1], cols[1]);
  plan.a1.W = read_block(is, rows[2], cols[2]);
  plan.a2.W = read_block(is, rows[3], cols[3]);
  for (int k = 0; k < 2; ++k) {
    const Axis& a = *ax[k];
    if (a.p * a.q != a.n || rows[k] != a.q || cols[k] != static_cast<std::uint32_t>(a.r) ||
        rows[k + 2] != 2 * a.mt + 1 || cols[k + 2] != static_cast<std::uint32_t>(a.r))
      throw std::runtime_error("inconsistent plan blocks in " + path);
  }
}

// 1-D plan files: "pft-plan-1d v1", one un-suffixed axis line, eps, B then W
// (pft.cpp:266-275 save_plan(PftPlan1D), 310-334 load_plan_1d).
void plan_save_1d(const Axis& a, const std::string& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("cannot open " + path + " for writing");
  os << "pft-plan-1d v1\n";
  os << "n " << a.n << " p " << a.p << " q " << a.q << " mt " << a.mt << " r " << a.r << "\n";
  os << "eps " << fmt_eps(a.eps) << "\n---\n";
  write_block(os, a.B, a.q, a.r);
  write_block(os, a.W, 2 * a.mt + 1, a.r);
  if (!os) throw std::runtime_error("write failure on " + path);
}

void plan_load_1d(Axis& a, const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open " + path);
  std::string line;
  if (!std::getline(is, line) || line != "pft-plan-1d v1")
    throw std::runtime_error(path + " is not a pft-plan-1d v1 file");
  if (!std::getline(is, line)) throw std::runtime_error("truncated plan " + path);
  {
    std::istringstream iss(line);
    std::string key;
    if (!(iss >> key >> a.n >> key >> a.p >> key >> a.q >> key >> a.mt >> key >> a.r))
      throw std::runtime_error("malformed plan axis line in " + path);
  }
  if (!std::getline(is, line) || line.rfind("eps ", 0) != 0)
    throw std::runtime_error("missing eps line in " + path);
  a.eps = std::stod(line.substr(4));
  if (!std::getline(is, line) || line != "---") throw std::runtime_error("missing block separator in " + path);
  std::uint32_t rb, cb, rw, cw;
  a.B = read_block(is, rb, cb);
  a.W = read_block(is, rw, cw);
  if (a.p * a.q != a.n || rb != a.q || cb != static_cast<std::uint32_t>(a.r) || rw != 2 * a.mt + 1 ||
      cw != static_cast<std::uint32_t>(a.r))
    throw std::runtime_error("inconsistent plan blocks in " + path);
}

}  // namespace pftg
