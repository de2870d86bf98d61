// Measurement-set directory format: the on-disk interop of
// the reference's save_measurements / load_measurements (simulate.hpp:40-43,
// simulate.cpp:91-164) and its raw real fields (raw_io.hpp:10-27,
// raw_io.cpp:27-106), read into / written from the GPU path's contiguous
// layout d[count][rows][cols] (and d_crop[count][2mt1][2mt2]).
//
//   meta.txt      "ptycho-measurements v1", count, window rows cols, mt mt1 mt2,
//                 noise_scale (%.17g), noise_seed
//   d_NNNN.ptyr   "PTYR", u32 version 1, u32 rows, u32 cols, f64 row-major
//   dcrop_NNNN.ptyr  when mt1 > 0
//   manifest.txt  "<fnv1a-64 hex>  <name>" per file, in write order; verified
//                 on load (hash mismatch -> runtime_error). The hash uses the
//                 reference's offset basis (see fnv1a below), not the standard one.
// Little-endian hosts only, like the reference (raw_io.cpp:9-10).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "host.hpp"

namespace pftg {
namespace {

namespace fs = std::filesystem;

std::string idx_name(const char* stem, std::size_t j) {
  char b[64];
  std::snprintf(b, sizeof b, "%s_%04zu.ptyr", stem, j);
  return b;
}

std::uint64_t fnv1a(const fs::path& p) {
  std::ifstream is(p, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open for reading: " + p.string());
  // FNV-1a with the reference's offset basis 1469598103934665603 (raw_io.cpp:89):
  // one digit short of the standard 14695981039346656037, kept for manifest interop
  std::uint64_t h = 1469598103934665603ull;
  std::vector<char> buf(1 << 16);
  while (true) {
    is.read(buf.data(), (std::streamsize)buf.size());
    const std::streamsize got = is.gcount();
    for (std::streamsize i = 0; i < got; ++i) {
      h ^= (unsigned char)buf[i];
      h *= 0x100000001b3ull;
    }
    if (got < (std::streamsize)buf.size()) break;
  }
  return h;
}

std::string hex16(std::uint64_t h) {
  char b[17];
  std::snprintf(b, sizeof b, "%016llx", (unsigned long long)h);
  return b;
}

void write_ptyr(const fs::path& p, const double* x, std::uint32_t rows, std::uint32_t cols) {
  std::ofstream os(p, std::ios::binary);
  if (!os) throw std::runtime_error("cannot open for writing: " + p.string());
  const std::uint32_t hdr[3] = {1u, rows, cols};
  os.write("PTYR", 4);
  os.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  os.write(reinterpret_cast<const char*>(x), (std::streamsize)((std::size_t)rows * cols * sizeof(double)));
  if (!os) throw std::runtime_error("raw field: write failed");
}

// reads one PTYR file into out (rows x cols doubles), checking its shape
void read_ptyr(const fs::path& p, double* out, std::uint32_t rows, std::uint32_t cols) {
  std::ifstream is(p, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open for reading: " + p.string());
  char magic[4] = {};
  if (!is.read(magic, 4) || std::memcmp(magic, "PTYR", 4) != 0) throw std::runtime_error("raw field: bad magic");
  std::uint32_t hdr[3];
  if (!is.read(reinterpret_cast<char*>(hdr), sizeof hdr)) throw std::runtime_error("raw field: truncated header");
  if (hdr[0] != 1u) throw std::runtime_error("raw field: unsupported version");
  if (hdr[1] == 0 || hdr[2] == 0) throw std::runtime_error("raw field: empty shape");
  if (hdr[1] != rows || hdr[2] != cols) throw std::runtime_error("measurement shape mismatch in " + p.string());
  const std::size_t n = (std::size_t)rows * cols;
  if (!is.read(reinterpret_cast<char*>(out), (std::streamsize)(n * sizeof(double))))
    throw std::runtime_error("raw field: truncated payload");
  for (std::size_t i = 0; i < n; ++i)
    if (!std::isfinite(out[i])) throw std::runtime_error("raw field: non-finite payload");
}

}  // namespace

void meas_save(const std::string& dir, const MeasMeta& m, const double* d, const double* dcrop) {
  const fs::path root(dir);
  fs::create_directories(root);
  std::vector<std::string> names;
  {
    std::ofstream meta(root / "meta.txt");
    if (!meta) throw std::runtime_error("cannot write " + (root / "meta.txt").string());
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", m.noise_scale);
    meta << "ptycho-measurements v1\n"
         << "count " << m.count << "\n"
         << "window " << m.rows << " " << m.cols << "\n"
         << "mt " << m.mt1 << " " << m.mt2 << "\n"
         << "noise_scale " << b << "\n"
         << "noise_seed " << m.noise_seed << "\n";
  }
  names.emplace_back("meta.txt");
  const std::size_t wn = m.rows * m.cols, cn = 4 * m.mt1 * m.mt2;
  for (std::size_t j = 0; j < m.count; ++j) {
    names.push_back(idx_name("d", j));
    write_ptyr(root / names.back(), d + j * wn, (std::uint32_t)m.rows, (std::uint32_t)m.cols);
  }
  if (m.mt1 > 0 && dcrop) {
    for (std::size_t j = 0; j < m.count; ++j) {
      names.push_back(idx_name("dcrop", j));
      write_ptyr(root / names.back(), dcrop + j * cn, (std::uint32_t)(2 * m.mt1), (std::uint32_t)(2 * m.mt2));
    }
  }
  std::ofstream man(root / "manifest.txt");
  if (!man) throw std::runtime_error("cannot write " + (root / "manifest.txt").string());
  for (const auto& nm : names) man << hex16(fnv1a(root / nm)) << "  " << nm << "\n";
}

MeasMeta meas_info(const std::string& dir) {
  const fs::path root(dir);
  {
    std::ifstream man(root / "manifest.txt");
    if (!man) throw std::runtime_error("missing manifest in " + dir);
    std::string h, nm;
    while (man >> h >> nm)
      if (hex16(fnv1a(root / nm)) != h) throw std::runtime_error("manifest hash mismatch for " + (root / nm).string());
  }
  std::ifstream meta(root / "meta.txt");
  if (!meta) throw std::runtime_error("missing meta.txt in " + dir);
  std::string line, key;
  if (!std::getline(meta, line) || line != "ptycho-measurements v1")
    throw std::runtime_error(dir + " is not a measurement directory");
  MeasMeta m;
  meta >> key >> m.count >> key >> m.rows >> m.cols >> key >> m.mt1 >> m.mt2 >> key >> m.noise_scale >> key >>
      m.noise_seed;
  if (!meta) throw std::runtime_error("malformed meta.txt in " + dir);
  return m;
}

template <class T>
void meas_read(const std::string& dir, const MeasMeta& m, T* d, T* dcrop) {
  const fs::path root(dir);
  const std::size_t wn = m.rows * m.cols, cn = 4 * m.mt1 * m.mt2;
  std::vector<double> tmp(std::is_same<T, double>::value ? 0 : std::max(wn, cn));
  auto one = [&](const fs::path& p, T* out, std::size_t n, std::size_t r, std::size_t c) {
    if constexpr (std::is_same<T, double>::value) {
      read_ptyr(p, out, (std::uint32_t)r, (std::uint32_t)c);
    } else {
      read_ptyr(p, tmp.data(), (std::uint32_t)r, (std::uint32_t)c);
      for (std::size_t i = 0; i < n; ++i) out[i] = (T)tmp[i];
    }
  };
  for (std::size_t j = 0; j < m.count; ++j) one(root / idx_name("d", j), d + j * wn, wn, m.rows, m.cols);
  if (m.mt1 > 0 && dcrop)
    for (std::size_t j = 0; j < m.count; ++j)
      one(root / idx_name("dcrop", j), dcrop + j * cn, cn, 2 * m.mt1, 2 * m.mt2);
}

template void meas_read<double>(const std::string&, const MeasMeta&, double*, double*);
template void meas_read<float>(const std::string&, const MeasMeta&, float*, float*);

}  // namespace pftg
