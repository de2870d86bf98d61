// Host-only (no CUDA) pieces of the offline phase: scope table and plan
// tables. See plan.cpp.
#pragma once

#include <complex>
#include <cstddef>
#include <string>
#include <vector>

namespace pftg {

using cd = std::complex<double>;

// minimax::ScopeRecord (minimax.hpp:35-41)
struct Record {
  double eps = 0.0;
  int r = 0;
  double xi = 0.0;
  double achieved_error = 0.0;
  std::vector<cd> coeff;
};

// minimax::ScopeTable (minimax.hpp:45-70)
struct Table {
  int max_r = 0;
  std::vector<Record> records;
};

// pft::PftPlan1D (pft.hpp:25-31)
struct Axis {
  std::size_t n = 0, p = 0, q = 0, mt = 0;
  int r = 0;
  double eps = 0.0;
  std::vector<cd> B;  // q x r
  std::vector<cd> W;  // (2mt+1) x r
};

Table table_load(const std::string& path);
// minimax.cpp: own near-minimax solver and the scope-table computation
std::vector<cd> best_approx_own(int r, double xi, double* achieved);
Table table_compute(const std::vector<double>& eps_list, int max_r);
void table_save(const Table& t, const std::string& path);
const Record* table_find(const Table& t, double eps, int r);
int table_min_degree(const Table& t, double eps, double target);
Axis plan_1d(std::size_t n, std::size_t mt, std::size_t p, double eps, const Table& table);
void plan_save(const Axis& a1, const Axis& a2, const std::string& path);
void plan_load(Axis& a1, Axis& a2, const std::string& path);
// meas_io.cpp: the measurement-set directory (simulate.cpp:91-164)
struct MeasMeta {
  std::size_t count = 0, rows = 0, cols = 0, mt1 = 0, mt2 = 0;
  double noise_scale = 0.0;
  unsigned long long noise_seed = 0;
};
void meas_save(const std::string& dir, const MeasMeta& m, const double* d, const double* dcrop);
MeasMeta meas_info(const std::string& dir);  // verifies the manifest
template <class T>
void meas_read(const std::string& dir, const MeasMeta& m, T* d, T* dcrop);
void plan_save_1d(const Axis& a, const std::string& path);
void plan_load_1d(Axis& a, const std::string& path);

}  // namespace pftg
