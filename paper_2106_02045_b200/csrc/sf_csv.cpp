// sf_csv.cpp -- native ParamsCSV / truth-CSV writer and reader.
//
// The reference CLI renders each float32 as the shortest decimal string that
// round-trips the value ("shortest round-trip representation"), in
// positional notation; paper_2106_02045_b200/io_formats.py:fmt32 states the
// same rendering with numpy's Dragon4 (np.format_float_positional(unique=True,
// trim='-')), which tests/test_csv_native.py uses as the checker.  Here the
// shortest digits come from Ryu's binary32 algorithm (Adams, PLDI 2018:
// interval [v - ulp/2, v + ulp/2] scaled by 5^q / 2^k with the 61/59-bit
// multipliers of sf_pow5_tables.h, digits removed while the interval keeps a
// shorter candidate, round-half-even on the last removed digit), then laid
// out positionally.  Rows are formatted in parallel blocks (one contiguous row
// range per thread, written in order), so a 1e8-row file is bound by the file
// system rather than by formatting.  The reader splits the file at line
// boundaries and parses the blocks in parallel with strtof (correctly rounded:
// the round trip is exact).
#include <errno.h>
#include <fcntl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "spotfit.h"
#include "sf_pow5_tables.h"

namespace {

thread_local std::string g_csv_err;

int csv_fail(const std::string& m) {
  g_csv_err = m;
  return -1;
}

// ---------------------------------------------------------------- Ryu binary32
inline int pow5bits(int e) { return (int)(((uint32_t)e * 1217359u) >> 19) + 1; }  // bitlen(5^e), 0 <= e <= 3528
inline uint32_t log10_pow2(int e) { return ((uint32_t)e * 78913u) >> 18; }        // floor(e log10 2)
inline uint32_t log10_pow5(int e) { return ((uint32_t)e * 732923u) >> 20; }       // floor(e log10 5)

inline uint32_t pow5_factor(uint32_t v) {
  uint32_t n = 0;
  while (v % 5 == 0) {
    v /= 5;
    ++n;
  }
  return n;
}
inline bool multiple_of_pow5(uint32_t v, uint32_t p) { return pow5_factor(v) >= p; }
inline bool multiple_of_pow2(uint32_t v, uint32_t p) { return (v & ((1u << p) - 1)) == 0; }

// (m * factor) >> shift, shift > 32, factor <= 64 bits
inline uint32_t mul_shift(uint32_t m, uint64_t factor, int shift) {
  const uint64_t lo = (uint64_t)m * (uint32_t)factor;
  const uint64_t hi = (uint64_t)m * (uint32_t)(factor >> 32);
  return (uint32_t)(((lo >> 32) + hi) >> (shift - 32));
}

struct Decimal {
  uint32_t digits;  // <= 9 decimal digits
  int32_t exponent;  // value = digits * 10^exponent
};

// shortest digits that round-trip a finite, non-zero |v| (mantissa/exponent fields of the bits)
Decimal shortest(uint32_t ieee_m, uint32_t ieee_e) {
  int32_t e2;
  uint32_t m2;
  if (ieee_e == 0) {
    e2 = 1 - 127 - 23 - 2;
    m2 = ieee_m;
  } else {
    e2 = (int32_t)ieee_e - 127 - 23 - 2;
    m2 = (1u << 23) | ieee_m;
  }
  const bool accept_bounds = (m2 & 1) == 0;  // round-half-even: the interval is closed for even mantissas
  const uint32_t mv = 4 * m2;
  const uint32_t mp = 4 * m2 + 2;
  const uint32_t mm_shift = (ieee_m != 0 || ieee_e <= 1) ? 1 : 0;  // the lower neighbour is half as far at 2^k
  const uint32_t mm = 4 * m2 - 1 - mm_shift;

  uint32_t vr, vp, vm;
  int32_t e10;
  bool vm_tz = false, vr_tz = false;
  uint32_t last = 0;
  if (e2 >= 0) {
    const uint32_t q = log10_pow2(e2);
    e10 = (int32_t)q;
    const int k = 59 + pow5bits((int)q) - 1;
    const int i = -e2 + (int)q + k;
    vr = mul_shift(mv, SF_POW5_INV[q], i);
    vp = mul_shift(mp, SF_POW5_INV[q], i);
    vm = mul_shift(mm, SF_POW5_INV[q], i);
    if (q != 0 && (vp - 1) / 10 <= vm / 10) {
      const int l = 59 + pow5bits((int)q - 1) - 1;
      last = mul_shift(mv, SF_POW5_INV[q - 1], -e2 + (int)q - 1 + l) % 10;
    }
    if (q <= 9) {
      if (mv % 5 == 0)
        vr_tz = multiple_of_pow5(mv, q);
      else if (accept_bounds)
        vm_tz = multiple_of_pow5(mm, q);
      else
        vp -= multiple_of_pow5(mp, q);
    }
  } else {
    const uint32_t q = log10_pow5(-e2);
    e10 = (int32_t)q + e2;
    const int i = -e2 - (int)q;
    const int k = pow5bits(i) - 61;
    int j = (int)q - k;
    vr = mul_shift(mv, SF_POW5[i], j);
    vp = mul_shift(mp, SF_POW5[i], j);
    vm = mul_shift(mm, SF_POW5[i], j);
    if (q != 0 && (vp - 1) / 10 <= vm / 10) {
      j = (int)q - 1 - (pow5bits(i + 1) - 61);
      last = mul_shift(mv, SF_POW5[i + 1], j) % 10;
    }
    if (q <= 1) {
      vr_tz = true;
      if (accept_bounds)
        vm_tz = mm_shift == 1;
      else
        --vp;
    } else if (q < 31) {
      vr_tz = multiple_of_pow2(mv, q - 1);
    }
  }

  int32_t removed = 0;
  uint32_t out;
  if (vm_tz || vr_tz) {
    while (vp / 10 > vm / 10) {
      vm_tz &= vm % 10 == 0;
      vr_tz &= last == 0;
      last = vr % 10;
      vr /= 10;
      vp /= 10;
      vm /= 10;
      ++removed;
    }
    if (vm_tz) {
      while (vm % 10 == 0) {
        vr_tz &= last == 0;
        last = vr % 10;
        vr /= 10;
        vp /= 10;
        vm /= 10;
        ++removed;
      }
    }
    if (vr_tz && last == 5 && vr % 2 == 0) last = 4;  // exact tie .5000: round to even
    out = vr + (((vr == vm && (!accept_bounds || !vm_tz)) || last >= 5) ? 1 : 0);
  } else {
    while (vp / 10 > vm / 10) {
      last = vr % 10;
      vr /= 10;
      vp /= 10;
      vm /= 10;
      ++removed;
    }
    out = vr + ((vr == vm || last >= 5) ? 1 : 0);
  }
  return Decimal{out, e10 + removed};
}

// positional rendering of numpy's format_float_positional(unique=True, trim='-'):
// no exponent, no trailing zeros after the point, no trailing point, "-0" for -0.0
inline char* put_f32(char* p, float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  const bool neg = b >> 31;
  const uint32_t ie = (b >> 23) & 0xff, im = b & 0x7fffff;
  if (ie == 0xff) {
    if (im) {
      memcpy(p, "nan", 3);
      return p + 3;
    }
    if (neg) *p++ = '-';
    memcpy(p, "inf", 3);
    return p + 3;
  }
  if (neg) *p++ = '-';
  if (ie == 0 && im == 0) {
    *p++ = '0';
    return p;
  }
  Decimal d = shortest(im, ie);
  while (d.digits % 10 == 0) {  // trim='-': no trailing zeros in the digit string
    d.digits /= 10;
    ++d.exponent;
  }
  char dig[10];
  int n = 0;
  for (uint32_t v = d.digits; v; v /= 10) dig[n++] = (char)('0' + v % 10);  // reversed
  const int e = d.exponent;
  if (e >= 0) {  // integer: digits then e zeros
    for (int k = n - 1; k >= 0; --k) *p++ = dig[k];
    memset(p, '0', (size_t)e);
    return p + e;
  }
  const int point = n + e;  // digits before the decimal point
  if (point > 0) {
    for (int k = n - 1; k >= n - point; --k) *p++ = dig[k];
    *p++ = '.';
    for (int k = n - point - 1; k >= 0; --k) *p++ = dig[k];
  } else {
    *p++ = '0';
    *p++ = '.';
    memset(p, '0', (size_t)-point);
    p += -point;
    for (int k = n - 1; k >= 0; --k) *p++ = dig[k];
  }
  return p;
}

inline char* put_u64(char* p, uint64_t v) {
  char t[24];
  int n = 0;
  do {
    t[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  while (n) *p++ = t[--n];
  return p;
}

const char* const kStopNames[8] = {"MaxError", "MinDelta", "MinStep", "NotConverged", "MaxIterations",
                                   "Unknown5", "Unknown6", "Unknown7"};
const int kStopLen[8] = {8, 8, 7, 12, 13, 8, 8, 8};

// worst-case bytes per cell: f32 positional 1 + 39 + 1 + 45 digits <= 64 (denormal: "0." + 45 digits)
constexpr int kCellMax = 64;

bool write_all(int fd, const char* p, size_t n, int64_t off) {
  while (n) {
    const ssize_t w = pwrite(fd, p, n, (off_t)off);
    if (w < 0) {
      if (errno == EINTR) continue;
      return false;
    }
    p += w;
    n -= (size_t)w;
    off += w;
  }
  return true;
}

template <class F>
void run_parallel(int T, F&& f) {
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(f, t);
  f(0);
  for (auto& x : th) x.join();
}

int n_threads(int threads, int64_t work) {
  int t = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (t < 1) t = 1;
  const int64_t by_work = std::max<int64_t>(1, work / 4096);
  return (int)std::min<int64_t>(t, by_work);
}

size_t format_rows(char* buf, int64_t r0, int64_t r1, int64_t first_index, int ncols, const sf_csv_col* cols) {
  char* p = buf;
  for (int64_t r = r0; r < r1; ++r) {
    p = put_u64(p, (uint64_t)(first_index + r));
    for (int c = 0; c < ncols; ++c) {
      *p++ = ',';
      const sf_csv_col& col = cols[c];
      const int64_t at = r * col.stride;
      switch (col.kind) {
        case SF_CSV_F32:
          p = put_f32(p, ((const float*)col.data)[at]);
          break;
        case SF_CSV_U8:
          p = put_u64(p, ((const uint8_t*)col.data)[at]);
          break;
        case SF_CSV_STOP: {
          const int s = ((const uint8_t*)col.data)[at] & 7;
          memcpy(p, kStopNames[s], (size_t)kStopLen[s]);
          p += kStopLen[s];
          break;
        }
        case SF_CSV_FLAGS: {  // status flag bits without the StopReason, as an integer
          p = put_u64(p, ((const uint8_t*)col.data)[at] & 0xf8);
          break;
        }
        default:
          break;
      }
    }
    *p++ = '\n';
  }
  return (size_t)(p - buf);
}

// ------------------------------------------------------------------- parsing
inline bool parse_u64(const char*& p, const char* end, uint64_t& v) {
  if (p >= end || *p < '0' || *p > '9') return false;
  uint64_t x = 0;
  while (p < end && *p >= '0' && *p <= '9') x = x * 10 + (uint64_t)(*p++ - '0');
  v = x;
  return true;
}

// Exact fast path for plain decimals "[-]d*[.d*]": with w the digit string as an integer (< 2^24) and
// 10^k (k <= 10, 5^10 < 2^24) both exact float32 values, one IEEE multiplication or division is the
// correctly rounded value of w * 10^e -- the same float strtof returns.  Anything else (more digits,
// exponents, nan/inf) goes to strtof.
inline bool fast_f32(const char* s, size_t len, float& out) {
  static const float kPow10[11] = {1e0f, 1e1f, 1e2f, 1e3f, 1e4f, 1e5f, 1e6f, 1e7f, 1e8f, 1e9f, 1e10f};
  const char* p = s;
  const char* e = s + len;
  const bool neg = p < e && *p == '-';
  p += neg;
  uint32_t w = 0;
  int nd = 0, frac = 0;
  bool point = false, any = false;
  for (; p < e; ++p) {
    const char c = *p;
    if (c >= '0' && c <= '9') {
      any = true;
      if (w == 0 && c == '0') {  // leading zeros carry no digits
        frac += point;
        continue;
      }
      if (++nd > 8) return false;  // < 10^8 < 2^27: checked against 2^24 below
      w = w * 10 + (uint32_t)(c - '0');
      frac += point;
    } else if (c == '.' && !point) {
      point = true;
    } else {
      return false;
    }
  }
  if (!any || w > (1u << 24) || frac > 10) return false;
  const float v = (float)w / kPow10[frac];
  out = neg ? -v : v;
  return true;
}

inline bool parse_cell(const char*& p, const char* end, const sf_csv_col& col, int64_t at) {
  const char* s = p;
  while (p < end && *p != ',' && *p != '\n' && *p != '\r') ++p;
  const size_t len = (size_t)(p - s);
  switch (col.kind) {
    case SF_CSV_F32: {
      if (fast_f32(s, len, ((float*)col.data)[at])) return true;
      char tmp[96];
      if (len == 0 || len >= sizeof(tmp)) return false;
      memcpy(tmp, s, len);
      tmp[len] = 0;
      char* q = nullptr;
      errno = 0;
      const float v = strtof(tmp, &q);  // correctly rounded (glibc): exact round trip of the shortest digits
      if (q != tmp + len) return false;
      ((float*)col.data)[at] = v;
      return true;
    }
    case SF_CSV_U8:
    case SF_CSV_FLAGS: {
      const char* t = s;
      uint64_t v;
      if (!parse_u64(t, s + len, v) || t != s + len || v > 255) return false;
      ((uint8_t*)col.data)[at] = (uint8_t)v;
      return true;
    }
    case SF_CSV_STOP: {
      for (int k = 0; k < 5; ++k)
        if ((int)len == kStopLen[k] && memcmp(s, kStopNames[k], len) == 0) {
          ((uint8_t*)col.data)[at] = (uint8_t)k;
          return true;
        }
      return false;
    }
    case SF_CSV_SKIP:
      return true;
    default:
      return false;
  }
}

}  // namespace

extern "C" {

const char* sf_csv_last_error(void) { return g_csv_err.c_str(); }

int sf_format_f32(const float* values, int64_t count, char* out, int64_t capacity, int64_t* out_len) {
  if (count < 0 || (count && (!values || !out))) return csv_fail("sf_format_f32: bad arguments");
  char* p = out;
  for (int64_t i = 0; i < count; ++i) {
    if ((p - out) + kCellMax + 1 > capacity) return csv_fail("sf_format_f32: output buffer too small");
    p = put_f32(p, values[i]);
    *p++ = '\n';
  }
  if (out_len) *out_len = p - out;
  return 0;
}

int sf_csv_write(const char* path, const char* header, int64_t first_index, int64_t rows, int ncols,
                 const sf_csv_col* cols, int threads) {
  if (!path || !header || rows < 0 || ncols < 0 || ncols > 64 || (ncols && !cols))
    return csv_fail("sf_csv_write: bad arguments");
  for (int c = 0; c < ncols; ++c)
    if (!cols[c].data && rows) return csv_fail("sf_csv_write: column " + std::to_string(c) + " has no data");
  const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0) return csv_fail(std::string("sf_csv_write: cannot open ") + path + ": " + strerror(errno));
  std::string head(header);
  head += '\n';
  bool ok = write_all(fd, head.data(), head.size(), 0);
  int64_t off = (int64_t)head.size();
  const int T = n_threads(threads, rows);
  const int64_t row_max = 22 + (int64_t)ncols * (kCellMax + 1) + 1;
  const int64_t block_rows = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)T * 262144));
  std::vector<std::vector<char>> bufs(T);
  std::vector<size_t> lens(T);
  std::vector<char> wok(T, 1);
  for (int64_t b0 = 0; ok && b0 < rows; b0 += block_rows) {
    // every thread renders its slice of the block, then (after a barrier that fixes the offsets)
    // writes it at its own file offset
    const int64_t b1 = std::min(rows, b0 + block_rows);
    const int64_t per = (b1 - b0 + T - 1) / T;
    auto render = [&](int t) {
      const int64_t r0 = std::min(b1, b0 + t * per), r1 = std::min(b1, r0 + per);
      if ((int64_t)bufs[t].size() < (r1 - r0) * row_max) bufs[t].resize((size_t)((r1 - r0) * row_max));
      lens[t] = format_rows(bufs[t].data(), r0, r1, first_index, ncols, cols);
    };
    run_parallel(T, render);
    std::vector<int64_t> at(T + 1, off);
    for (int t = 0; t < T; ++t) at[t + 1] = at[t] + (int64_t)lens[t];
    run_parallel(T, [&](int t) { wok[t] = write_all(fd, bufs[t].data(), lens[t], at[t]); });
    for (int t = 0; t < T; ++t) ok = ok && wok[t];
    off = at[T];
  }
  if (close(fd) != 0) ok = false;
  if (!ok) return csv_fail(std::string("sf_csv_write: write failed on ") + path + ": " + strerror(errno));
  return 0;
}

int sf_csv_read(const char* path, int64_t* rows_out, int64_t* index, int ncols, const sf_csv_col* cols,
                int64_t capacity, int threads) {
  if (!path || !rows_out || ncols < 0 || ncols > 64) return csv_fail("sf_csv_read: bad arguments");
  const int fd = open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return csv_fail(std::string("sf_csv_read: cannot open ") + path + ": " + strerror(errno));
  struct stat st;
  if (fstat(fd, &st) != 0) {
    close(fd);
    return csv_fail("sf_csv_read: cannot size the file");
  }
  const size_t size = (size_t)st.st_size;
  void* map = nullptr;
  if (size) {
    map = mmap(nullptr, size, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
    if (map == MAP_FAILED) {
      close(fd);
      return csv_fail(std::string("sf_csv_read: mmap failed: ") + strerror(errno));
    }
  }
  close(fd);
  struct Unmap {
    void* p;
    size_t n;
    ~Unmap() {
      if (p) munmap(p, n);
    }
  } unmap{map, size};
  const char* beg = (const char*)map;
  const char* end = beg + size;
  const char* body = size ? (const char*)memchr(beg, '\n', size) : nullptr;
  body = body ? body + 1 : end;  // skip the header line
  // split the body at line starts; count rows per block, then parse each block into its row offset
  const int T = n_threads(threads, (int64_t)(end - body) / 64);
  std::vector<const char*> cut(T + 1);
  cut[0] = body;
  cut[T] = end;
  for (int t = 1; t < T; ++t) {
    const char* c = body + (end - body) * t / T;
    if (c < cut[t - 1]) c = cut[t - 1];
    const char* nl = (const char*)memchr(c, '\n', (size_t)(end - c));
    cut[t] = nl ? nl + 1 : end;
  }
  auto is_blank = [](const char* s, const char* e) {
    for (; s < e; ++s)
      if (*s != '\r' && *s != ' ' && *s != '\t') return false;
    return true;
  };
  std::vector<int64_t> nrows(T, 0);
  auto count_block = [&](int t) {
    int64_t n = 0;
    for (const char* p = cut[t]; p < cut[t + 1];) {
      const char* nl = (const char*)memchr(p, '\n', (size_t)(cut[t + 1] - p));
      const char* le = nl ? nl : cut[t + 1];
      if (!is_blank(p, le)) ++n;
      p = le + 1;
    }
    nrows[t] = n;
  };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(count_block, t);
    for (auto& x : th) x.join();
  }
  std::vector<int64_t> first(T + 1, 0);
  for (int t = 0; t < T; ++t) first[t + 1] = first[t] + nrows[t];
  *rows_out = first[T];
  if (capacity < 0) return 0;  // count only
  if (first[T] > capacity) return csv_fail("sf_csv_read: more rows than the output capacity");
  std::vector<int64_t> bad(T, -1);
  auto parse_block = [&](int t) {
    int64_t r = first[t];
    for (const char* p = cut[t]; p < cut[t + 1];) {
      const char* nl = (const char*)memchr(p, '\n', (size_t)(cut[t + 1] - p));
      const char* le = nl ? nl : cut[t + 1];
      if (!is_blank(p, le)) {
        const char* q = p;
        uint64_t ix;
        bool ok = parse_u64(q, le, ix);
        if (index) index[r] = (int64_t)ix;
        for (int c = 0; ok && c < ncols; ++c) {
          ok = q < le && *q == ',';
          ++q;
          ok = ok && parse_cell(q, le, cols[c], r * cols[c].stride);
        }
        while (ok && q < le && *q == '\r') ++q;
        if (!ok || q != le) {
          bad[t] = r;
          return;
        }
        ++r;
      }
      p = le + 1;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(parse_block, t);
    for (auto& x : th) x.join();
  }
  for (int t = 0; t < T; ++t)
    if (bad[t] >= 0) return csv_fail("sf_csv_read: malformed row " + std::to_string(bad[t] + 1));
  return 0;
}

}  // extern "C"
