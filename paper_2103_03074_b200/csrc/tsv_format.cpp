// Host-side row formatter of the reference amplitude TSV ("tncut-amplitudes/1",
// tncut engine.py:467-479): one line per AmplitudeTable row
//     <bitstring>\t<amp.real:.17g>\t<amp.imag:.17g>\t<prob:.17g>\n
// byte-identical to the reference's per-row Python f-strings, formatted on
// all host threads.  prob follows AmplitudeTable.rows() (engine.py:94-96):
// float(abs(amp) ** 2) in the amplitudes' own scalar precision -- numpy's
// scalar abs is libm hypotf / hypot and its scalar ** 2 is libm powf / pow
// (which differ from h*h in the last bit for ~0.1% of values).  Python's '.17g' and glibc's "%.17g" are both correctly
// rounded and agree on finite values, +-inf and -0; every NaN prints "nan".
// Checked against the Python writer in tests/test_io.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

namespace {

inline char* put17g(char* p, double v) {
  if (std::isnan(v)) {
    std::memcpy(p, "nan", 3);
    return p + 3;
  }
  const int n = std::snprintf(p, 32, "%.17g", v);
  return p + n;
}

// worst-case bytes of one row: bitstring + 3 numbers (<= 24 chars each) + 4 separators
inline int64_t row_cap(int nb) { return (int64_t)nb + 3 * 32 + 4; }

void format_range(const char* bits, int nb, const void* amps, bool single, int64_t lo, int64_t hi,
                  std::string& out) {
  out.resize((size_t)((hi - lo) * row_cap(nb)));
  char* p = &out[0];
  for (int64_t r = lo; r < hi; ++r) {
    std::memcpy(p, bits + r * nb, (size_t)nb);
    p += nb;
    double re, im, prob;
    if (single) {
      const float* a = static_cast<const float*>(amps) + 2 * r;
      re = a[0];
      im = a[1];
      volatile float h = hypotf(a[0], a[1]);  // numpy complex64 scalar abs
      volatile float sq = powf(h, 2.0f);      // numpy float32 scalar ** 2 (libm powf, not h*h)
      prob = sq;
    } else {
      const double* a = static_cast<const double*>(amps) + 2 * r;
      re = a[0];
      im = a[1];
      volatile double h = hypot(a[0], a[1]);
      volatile double sq = pow(h, 2.0);
      prob = sq;
    }
    *p++ = '\t';
    p = put17g(p, re);
    *p++ = '\t';
    p = put17g(p, im);
    *p++ = '\t';
    p = put17g(p, prob);
    *p++ = '\n';
  }
  out.resize((size_t)(p - &out[0]));
}

}  // namespace

extern "C" {

// Rows [0, n): `bits` holds n bitstrings of nb chars back to back, `amps`
// n interleaved complex values (complex64 when single != 0, else
// complex128).  Writes the TSV lines to `out` (capacity `cap` bytes) and
// returns the byte count, or -1 when `cap` < n * tnbio_row_cap(nb).
int64_t tnbio_row_cap(int32_t nb) { return row_cap(nb); }

int64_t tnbio_format_rows(const char* bits, int32_t nb, const void* amps, int32_t single, int64_t n,
                          char* out, int64_t cap, int32_t threads) {
  if (n < 0 || nb < 0 || cap < n * row_cap(nb)) return -1;
  if (n == 0) return 0;
  int t = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (t < 1) t = 1;
  if ((int64_t)t > n / 1024 + 1) t = (int)(n / 1024 + 1);
  std::vector<std::string> parts((size_t)t);
  std::vector<std::thread> pool;
  const int64_t per = (n + t - 1) / t;
  for (int i = 0; i < t; ++i) {
    const int64_t lo = i * per, hi = std::min<int64_t>(n, lo + per);
    if (lo >= hi) break;
    pool.emplace_back(format_range, bits, nb, amps, single != 0, lo, hi, std::ref(parts[(size_t)i]));
  }
  for (auto& th : pool) th.join();
  int64_t off = 0;
  for (auto& s : parts) {
    std::memcpy(out + off, s.data(), s.size());
    off += (int64_t)s.size();
  }
  return off;
}

}  // extern "C"
