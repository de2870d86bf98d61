// TEST INFRASTRUCTURE ONLY -- not product code. See oracle/shim/fftw3.h.
//
// Strided multi-dimensional complex DFT: every transform dimension is applied
// as a batch of 1-D transforms over gathered lines. Power-of-two lengths use
// an iterative radix-2 FFT whose twiddles are computed per index with exact
// integer phase reduction (cos/sin of 2*pi*k/n); other lengths fall back to
// the O(n^2) definition. Accuracy ~1e-16 * log2(n), comparable to FFTW.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace {

using cd = std::complex<double>;

struct Twiddles {
  std::vector<cd> w;  // w[k] = exp(-2*pi*i*k/n), k < n/2
};

const Twiddles& twiddles(long n) {
  static std::mutex mu;
  static std::map<long, std::unique_ptr<Twiddles>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return *it->second;
  auto t = std::make_unique<Twiddles>();
  t->w.resize(static_cast<size_t>(n / 2 > 0 ? n / 2 : 1));
  for (long k = 0; k < n / 2; ++k) {
    const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(n);
    t->w[k] = cd(std::cos(a), std::sin(a));
  }
  auto* raw = t.get();
  cache.emplace(n, std::move(t));
  return *raw;
}

bool is_pow2(long n) { return n > 0 && (n & (n - 1)) == 0; }

// In-place 1-D transform of a contiguous line.
void line_dft(cd* x, long n, int sign, std::vector<cd>& scratch) {
  if (n <= 1) return;
  if (is_pow2(n)) {
    for (long i = 1, j = 0; i < n; ++i) {  // bit reversal
      long bit = n >> 1;
      for (; j & bit; bit >>= 1) j ^= bit;
      j ^= bit;
      if (i < j) std::swap(x[i], x[j]);
    }
    const Twiddles& tw = twiddles(n);
    for (long len = 2; len <= n; len <<= 1) {
      const long half = len >> 1, step = n / len;
      for (long s = 0; s < n; s += len) {
        for (long k = 0; k < half; ++k) {
          cd w = tw.w[k * step];
          if (sign > 0) w = std::conj(w);
          const cd a = x[s + k];
          const cd b0 = x[s + k + half];
          const cd b(w.real() * b0.real() - w.imag() * b0.imag(),
                     w.real() * b0.imag() + w.imag() * b0.real());
          x[s + k] = a + b;
          x[s + k + half] = a - b;
        }
      }
    }
    return;
  }
  scratch.assign(static_cast<size_t>(n), cd(0.0, 0.0));
  for (long t = 0; t < n; ++t) {
    cd acc(0.0, 0.0);
    for (long k = 0; k < n; ++k) {
      const long m = (t * k) % n;
      const double a = sign * 2.0 * M_PI * static_cast<double>(m) / static_cast<double>(n);
      acc += x[k] * cd(std::cos(a), std::sin(a));
    }
    scratch[t] = acc;
  }
  std::memcpy(static_cast<void*>(x), scratch.data(), sizeof(cd) * static_cast<size_t>(n));
}

}  // namespace

struct fftw_plan_s {
  std::vector<fftw_iodim64> dims;  // transform dims
  std::vector<fftw_iodim64> how;   // batch dims
  int sign = FFTW_FORWARD;
};

namespace {

// Apply the multi-dim DFT for one batch element: gather into a dense
// row-major block, transform along each axis, scatter with output strides.
void exec_one(const fftw_plan_s& p, const cd* in, cd* out) {
  const size_t rank = p.dims.size();
  size_t total = 1;
  for (const auto& d : p.dims) total *= static_cast<size_t>(d.n);
  std::vector<cd> buf(total);
  std::vector<long> idx(rank, 0);
  for (size_t lin = 0; lin < total; ++lin) {
    size_t rem = lin;
    ptrdiff_t off = 0;
    for (size_t a = rank; a-- > 0;) {
      const long i = static_cast<long>(rem % static_cast<size_t>(p.dims[a].n));
      rem /= static_cast<size_t>(p.dims[a].n);
      off += i * p.dims[a].is;
    }
    buf[lin] = in[off];
  }
  std::vector<cd> line, scratch;
  size_t inner = total;
  for (size_t a = 0; a < rank; ++a) {
    const long n = static_cast<long>(p.dims[a].n);
    inner /= static_cast<size_t>(n);
    const size_t outer = total / (inner * static_cast<size_t>(n));
    line.resize(static_cast<size_t>(n));
    for (size_t o = 0; o < outer; ++o)
      for (size_t in_i = 0; in_i < inner; ++in_i) {
        cd* base = buf.data() + o * static_cast<size_t>(n) * inner + in_i;
        if (inner == 1) {
          line_dft(base, n, p.sign, scratch);
        } else {
          for (long k = 0; k < n; ++k) line[k] = base[k * inner];
          line_dft(line.data(), n, p.sign, scratch);
          for (long k = 0; k < n; ++k) base[k * inner] = line[k];
        }
      }
  }
  for (size_t lin = 0; lin < total; ++lin) {
    size_t rem = lin;
    ptrdiff_t off = 0;
    for (size_t a = rank; a-- > 0;) {
      const long i = static_cast<long>(rem % static_cast<size_t>(p.dims[a].n));
      rem /= static_cast<size_t>(p.dims[a].n);
      off += i * p.dims[a].os;
    }
    out[off] = buf[lin];
  }
}

fftw_plan make(std::vector<fftw_iodim64> dims, std::vector<fftw_iodim64> how, int sign) {
  auto* p = new fftw_plan_s;
  p->dims = std::move(dims);
  p->how = std::move(how);
  p->sign = sign;
  return p;
}

}  // namespace

extern "C" {

fftw_plan fftw_plan_dft_1d(int n, fftw_complex*, fftw_complex*, int sign, unsigned) {
  return make({{n, 1, 1}}, {}, sign);
}

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex*, fftw_complex*, int sign, unsigned) {
  return make({{n0, n1, n1}, {n1, 1, 1}}, {}, sign);
}

fftw_plan fftw_plan_many_dft(int rank, const int* n, int howmany, fftw_complex*, const int* inembed,
                             int istride, int idist, fftw_complex*, const int* onembed, int ostride,
                             int odist, int sign, unsigned) {
  if (inembed || onembed || rank < 1) return nullptr;
  std::vector<fftw_iodim64> dims(static_cast<size_t>(rank));
  ptrdiff_t is = istride, os = ostride;
  for (int a = rank - 1; a >= 0; --a) {
    dims[a] = {n[a], is, os};
    is *= n[a];
    os *= n[a];
  }
  return make(dims, {{howmany, idist, odist}}, sign);
}

fftw_plan fftw_plan_guru64_dft(int rank, const fftw_iodim64* dims, int howmany_rank,
                               const fftw_iodim64* howmany_dims, fftw_complex*, fftw_complex*,
                               int sign, unsigned) {
  return make(std::vector<fftw_iodim64>(dims, dims + rank),
              std::vector<fftw_iodim64>(howmany_dims, howmany_dims + howmany_rank), sign);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  const cd* ci = reinterpret_cast<const cd*>(in);
  cd* co = reinterpret_cast<cd*>(out);
  size_t batch = 1;
  for (const auto& h : p->how) batch *= static_cast<size_t>(h.n);
  for (size_t b = 0; b < batch; ++b) {
    size_t rem = b;
    ptrdiff_t ioff = 0, ooff = 0;
    for (size_t a = p->how.size(); a-- > 0;) {
      const long i = static_cast<long>(rem % static_cast<size_t>(p->how[a].n));
      rem /= static_cast<size_t>(p->how[a].n);
      ioff += i * p->how[a].is;
      ooff += i * p->how[a].os;
    }
    exec_one(*p, ci + ioff, co + ooff);
  }
}

void fftw_destroy_plan(fftw_plan p) { delete p; }
int fftw_init_threads(void) { return 0; }
void fftw_plan_with_nthreads(int) {}

}  // extern "C"
