// Ingest: the reference's CSV table format parsed on the device.
//
// Replaces load_csv (storage.cpp:112-150): one text line per row (getline on
// '\n', a trailing '\r' stripped), fields separated by ',', every field
// non-empty, Int columns parsed like std::from_chars(int64) and Float columns
// like std::from_chars(double) (correctly rounded; inf / nan accepted; results
// that overflow or underflow to zero rejected), the whole field consumed.  The
// first failing line (in file order) raises FormatError with the reference's
// message (storage.cpp:82-96, 130-143).
//
// Device work:
//   1. line index: 4 KB tiles, '\n' counted per tile, exclusive scan of the
//      tile counts, then every tile writes its newline offsets (warp-shuffle
//      block scan) -> line i = [nl[i-1] + 1, nl[i]);
//   2. one thread per line walks its fields and writes the int64 / double
//      column values; failures lower an atomicMin on the line number.
// Float conversion: Clinger's exact fast path when the significand fits 53
// bits and |exponent| <= 22, otherwise a double approximation corrected by
// exact big-integer comparisons against the neighbouring midpoints
// (round-to-nearest-even), so every result is the correctly rounded double
// std::from_chars returns.
#include <cub/cub.cuh>

#include <cstring>
#include <memory>
#include <string>
#include <system_error>
#include <charconv>

#include "common.cuh"

struct laq_csv {
  laq_ctx* ctx = nullptr;
  const char* text = nullptr;  // device, caller-owned
  int64_t nbytes = 0;
  int64_t lines = 0;
  int64_t n_nl = 0;         // newlines (= lines, or lines - 1 without a final '\n')
  laq::DevBuf<int64_t> nl;  // newline offsets (stream-ordered pool memory)
};

namespace laq {
namespace {

constexpr int kTileThreads = 256;
constexpr int kTileBytes = kTileThreads * 16;

__device__ __forceinline__ int count_nl16(const char* t, int64_t n, int64_t b0, char (&c)[16]) {
  if (b0 + 16 <= n && (reinterpret_cast<uintptr_t>(t + b0) & 15) == 0) {
    const uint4 v = *reinterpret_cast<const uint4*>(t + b0);
    memcpy(c, &v, 16);
  } else {
    for (int i = 0; i < 16; ++i) c[i] = b0 + i < n ? t[b0 + i] : 0;
  }
  int k = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) k += c[i] == '\n';
  return k;
}

__global__ void nl_count_kernel(const char* t, int64_t n, int64_t* tile_counts) {
  const int64_t b0 = (static_cast<int64_t>(blockIdx.x) * kTileThreads + threadIdx.x) * 16;
  char c[16];
  int k = count_nl16(t, n, b0, c);
  for (int o = 16; o; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  __shared__ int s[kTileThreads / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = k;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kTileThreads / 32; ++w) tot += s[w];
    tile_counts[blockIdx.x] = tot;
  }
}

__global__ void nl_write_kernel(const char* t, int64_t n, const int64_t* tile_offsets, int64_t* nl) {
  const int64_t b0 = (static_cast<int64_t>(blockIdx.x) * kTileThreads + threadIdx.x) * 16;
  char c[16];
  const int k = count_nl16(t, n, b0, c);
  // exclusive scan of k over the block (warp shuffles + one smem pass)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = k;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  __shared__ int s[kTileThreads / 32];
  if (lane == 31) s[w] = inc;
  __syncthreads();
  int before = 0;
  for (int i = 0; i < w; ++i) before += s[i];
  int64_t pos = tile_offsets[blockIdx.x] + before + inc - k;
  for (int i = 0; i < 16; ++i)
    if (c[i] == '\n') nl[pos++] = b0 + i;
}

// ---- number parsing (std::from_chars semantics) -------------------------------

__device__ __forceinline__ bool is_digit(char c) { return c >= '0' && c <= '9'; }
__device__ __forceinline__ char lower(char c) { return (c >= 'A' && c <= 'Z') ? static_cast<char>(c + 32) : c; }

// from_chars(int64): optional '-', one or more digits, no overflow, field fully consumed.
__device__ bool parse_i64(const char* s, int len, int64_t* out) {
  int i = 0;
  const bool neg = len > 0 && s[0] == '-';
  if (neg) ++i;
  if (i >= len) return false;
  uint64_t v = 0;
  // v * 10 + d <= lim  <=>  v < lim / 10, or v == lim / 10 and d <= lim % 10
  // (lim / 10 = 922337203685477580; lim % 10 = 8 for -2^63, 7 for 2^63 - 1)
  constexpr uint64_t kTenth = 922337203685477580ull;
  const uint64_t last = neg ? 8u : 7u;
  for (; i < len; ++i) {
    const char ch = s[i];
    if (!is_digit(ch)) return false;
    const uint64_t d = static_cast<uint64_t>(ch - '0');
    if (v > kTenth || (v == kTenth && d > last)) return false;  // out of range
    v = v * 10 + d;
  }
  *out = neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
  return true;
}

// Little-endian big integer (32-bit limbs), enough for w * 5^343 << 1100.
struct Big {
  static constexpr int kLimbs = 44;
  uint32_t d[kLimbs];
  int n;
  __device__ void set(uint64_t v) {
    n = 0;
    while (v) {
      d[n++] = static_cast<uint32_t>(v);
      v >>= 32;
    }
  }
  __device__ void mul(uint32_t m) {
    uint64_t carry = 0;
    for (int i = 0; i < n; ++i) {
      const uint64_t p = static_cast<uint64_t>(d[i]) * m + carry;
      d[i] = static_cast<uint32_t>(p);
      carry = p >> 32;
    }
    if (carry) d[n++] = static_cast<uint32_t>(carry);
  }
  __device__ void mul_pow5(int e) {
    while (e >= 13) {
      mul(1220703125u);  // 5^13
      e -= 13;
    }
    uint32_t m = 1;
    while (e-- > 0) m *= 5;
    if (m != 1) mul(m);
  }
  __device__ void shl(int bits) {
    if (n == 0 || bits == 0) return;
    const int w = bits >> 5, b = bits & 31;
    if (b) {
      uint32_t carry = 0;
      for (int i = 0; i < n; ++i) {
        const uint32_t v = d[i];
        d[i] = (v << b) | carry;
        carry = v >> (32 - b);
      }
      if (carry) d[n++] = carry;
    }
    if (w) {
      for (int i = n - 1; i >= 0; --i) d[i + w] = d[i];
      for (int i = 0; i < w; ++i) d[i] = 0;
      n += w;
    }
  }
};

__device__ int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
  return 0;
}

// sign(w * 10^q - M * 2^F), exactly.
__device__ int cmp_dec_bin(uint64_t w, int q, uint64_t M, int F) {
  Big L, R;
  L.set(w);
  R.set(M);
  if (q >= 0) L.mul_pow5(q);
  else R.mul_pow5(-q);
  // now compare L * 2^q with R * 2^F
  if (q > F) L.shl(q - F);
  else R.shl(F - q);
  return big_cmp(L, R);
}

// a = m * 2^e with m an integer (a finite, >= 0).
__device__ __forceinline__ void decompose(double a, uint64_t* m, int* e) {
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(a));
  const int be = static_cast<int>((bits >> 52) & 0x7ff);
  const uint64_t frac = bits & ((uint64_t{1} << 52) - 1);
  if (be == 0) {
    *m = frac;
    *e = -1074;
  } else {
    *m = frac | (uint64_t{1} << 52);
    *e = be - 1075;
  }
}

// Midpoint of the adjacent doubles a < b as M * 2^F.
__device__ __forceinline__ void midpoint(double a, double b, uint64_t* M, int* F) {
  uint64_t ma, mb;
  int ea, eb;
  decompose(a, &ma, &ea);
  decompose(b, &mb, &eb);
  if (a == 0.0) ea = eb;  // 0 = 0 * 2^eb
  const int e0 = ea < eb ? ea : eb;
  *M = (ma << (ea - e0)) + (mb << (eb - e0));
  *F = e0 - 1;
}

__constant__ double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

// Correctly rounded w * 10^q for w > 0.  Returns 0 ok, 1 out of range (overflow
// or underflow to zero: std::errc::result_out_of_range).
__device__ int dec_to_double(uint64_t w, int q, double* out) {
  int nd = 0;
  for (uint64_t t = w; t; t /= 10) ++nd;
  if (q + nd - 1 > 309) return 1;   // >= 1e309: overflow
  if (q + nd - 1 < -325) return 1;  // < 1e-324: rounds to zero
  if (w < (uint64_t{1} << 53) && q >= -22 && q <= 22) {  // Clinger: one correctly rounded op
    *out = q >= 0 ? __dmul_rn(static_cast<double>(w), kPow10[q]) : __ddiv_rn(static_cast<double>(w), kPow10[-q]);
    return 0;
  }
  // Approximation (a few ulps), then exact correction.
  double x = static_cast<double>(w);
  int r = q;
  if (r < -300) {
    x *= 1e-300;
    r += 300;
  }
  while (r > 22) {
    x *= 1e22;
    r -= 22;
  }
  while (r < -22) {
    x /= 1e22;
    r += 22;
  }
  x = r >= 0 ? x * kPow10[r] : x / kPow10[-r];
  const double kMax = 1.7976931348623157e308;
  if (!(x < INFINITY)) x = kMax;
  for (int it = 0; it < 200; ++it) {
    uint64_t M;
    int F;
    uint64_t mx;
    int ex;
    decompose(x, &mx, &ex);
    const bool odd = (mx & 1) != 0;
    if (x == kMax) {  // midpoint with 2^1024: (2^54 - 1) * 2^970
      const int c = cmp_dec_bin(w, q, (uint64_t{1} << 54) - 1, 970);
      if (c >= 0) return 1;  // ties go to the even neighbour (infinity): overflow
    } else {
      const double up = __longlong_as_double(__double_as_longlong(x) + 1);
      midpoint(x, up, &M, &F);
      const int c = cmp_dec_bin(w, q, M, F);
      if (c > 0 || (c == 0 && odd)) {
        x = up;
        continue;
      }
    }
    if (x > 0.0) {
      const double dn = __longlong_as_double(__double_as_longlong(x) - 1);
      midpoint(dn, x, &M, &F);
      const int c = cmp_dec_bin(w, q, M, F);
      if (c < 0 || (c == 0 && odd)) {
        x = dn;
        continue;
      }
    }
    break;
  }
  if (x == 0.0) return 1;  // nonzero input rounded to zero
  *out = x;
  return 0;
}

// from_chars(double, chars_format::general).  Returns 0 ok, 1 bad float,
// 2 beyond this parser (more than 19 significant digits with the dropped
// digits deciding the rounding).
__device__ int parse_f64(const char* s, int len, double* out) {
  int i = 0;
  const bool neg = len > 0 && s[0] == '-';
  if (neg) ++i;
  if (i >= len) return 1;
  // inf / infinity / nan / nan(n-char-sequence), case-insensitive
  const char c0 = lower(s[i]);
  if (c0 == 'i' || c0 == 'n') {
    const int rest = len - i;
    auto eq = [&](const char* w, int k) {
      if (rest < k) return false;
      for (int j = 0; j < k; ++j)
        if (lower(s[i + j]) != w[j]) return false;
      return true;
    };
    if (c0 == 'i') {
      if (rest == 8 && eq("infinity", 8)) {
        *out = neg ? -INFINITY : INFINITY;
        return 0;
      }
      if (rest == 3 && eq("inf", 3)) {
        *out = neg ? -INFINITY : INFINITY;
        return 0;
      }
      return 1;
    }
    if (!eq("nan", 3)) return 1;
    if (rest != 3) {  // "nan(" [A-Za-z0-9_]* ")" must span the rest
      if (s[i + 3] != '(' || s[len - 1] != ')') return 1;
      for (int j = i + 4; j < len - 1; ++j) {
        const char c = s[j];
        if (!(is_digit(c) || (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_')) return 1;
      }
    }
    *out = neg ? -NAN : NAN;
    return 0;
  }
  uint64_t w = 0;
  int nsig = 0, digits = 0;
  int64_t q = 0;
  bool dropped = false;
  for (; i < len && is_digit(s[i]); ++i, ++digits) {
    const int d = s[i] - '0';
    if (w == 0 && d == 0) continue;
    if (nsig < 19) {
      w = w * 10 + d;
      ++nsig;
    } else {
      ++q;
      dropped = dropped || d != 0;
    }
  }
  if (i < len && s[i] == '.') {
    ++i;
    for (; i < len && is_digit(s[i]); ++i, ++digits) {
      const int d = s[i] - '0';
      if (w == 0 && d == 0) {
        --q;
        continue;
      }
      if (nsig < 19) {
        w = w * 10 + d;
        ++nsig;
        --q;
      } else {
        dropped = dropped || d != 0;
      }
    }
  }
  if (digits == 0) return 1;
  if (i < len && (s[i] == 'e' || s[i] == 'E')) {
    int j = i + 1;
    bool eneg = false;
    if (j < len && (s[j] == '+' || s[j] == '-')) eneg = s[j++] == '-';
    if (j >= len || !is_digit(s[j])) return 1;  // exponent not consumed -> field not fully consumed
    int64_t ev = 0;
    for (; j < len && is_digit(s[j]); ++j) ev = ev < 100000000 ? ev * 10 + (s[j] - '0') : ev;
    q += eneg ? -ev : ev;
    i = j;
  }
  if (i != len) return 1;
  if (w == 0) {
    *out = neg ? -0.0 : 0.0;
    return 0;
  }
  if (q > 100000) q = 100000;
  if (q < -100000) q = -100000;
  double v;
  if (dropped) {  // value in (w * 10^q, (w + 1) * 10^q): decided only if both ends round alike
    double v2;
    const int r1 = dec_to_double(w, static_cast<int>(q), &v), r2 = dec_to_double(w + 1, static_cast<int>(q), &v2);
    if (r1 != 0 || r2 != 0 || v != v2) return 2;
  } else if (dec_to_double(w, static_cast<int>(q), &v)) {
    return 1;
  }
  *out = neg ? -v : v;
  return 0;
}

constexpr int kMaxCsvCols = 64;
struct ParseArgs {
  const char* t;
  int64_t nbytes, lines, n_nl;
  const int64_t* nl;
  int ncols;
  int32_t kinds[kMaxCsvCols];  // LAQ_COL_*
  void* cols[kMaxCsvCols];
  unsigned long long* bad;          // first failing line (1-based), or ~0
  unsigned long long* unsupported;  // first line a float is beyond this parser
};

__global__ void parse_kernel(const ParseArgs a) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.lines; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = r == 0 ? 0 : a.nl[r - 1] + 1;
    int64_t e = r < a.n_nl ? a.nl[r] : a.nbytes;
    if (e > b && a.t[e - 1] == '\r') --e;
    const unsigned long long line_no = static_cast<unsigned long long>(r) + 1;
    bool ok = !(e == b && a.ncols == 1);  // a lone empty line is a missing value
    int64_t pos = b;
    for (int c = 0; ok && c < a.ncols; ++c) {
      int64_t comma = pos;
      while (comma < e && a.t[comma] != ',') ++comma;
      const bool last = c == a.ncols - 1;
      if (last != (comma == e)) {
        ok = false;
        break;
      }
      const int flen = static_cast<int>(comma - pos);
      if (flen == 0) {
        ok = false;
        break;
      }
      if (a.kinds[c] == LAQ_COL_FLOAT) {
        double v = 0;
        const int rc = parse_f64(a.t + pos, flen, &v);
        if (rc == 2) atomicMin(a.unsupported, line_no);
        if (rc) {
          ok = false;
          break;
        }
        static_cast<double*>(a.cols[c])[r] = v;
      } else {
        int64_t v = 0;
        if (!parse_i64(a.t + pos, flen, &v)) {
          ok = false;
          break;
        }
        static_cast<int64_t*>(a.cols[c])[r] = v;
      }
      pos = comma + 1;
    }
    if (!ok) atomicMin(a.bad, line_no);
  }
}

// The reference's message for one failing line (storage.cpp:130-143, 82-96),
// rebuilt on the host from that line's bytes.
std::string line_error(const std::string& line_in, int64_t line_no, int ncols, const int32_t* kinds) {
  std::string line = line_in;
  if (!line.empty() && line.back() == '\r') line.pop_back();
  const std::string at = "line " + std::to_string(line_no) + ": ";
  if (line.empty() && ncols == 1) return at + "missing value";
  std::string_view rest = line;
  for (int c = 0; c < ncols; ++c) {
    const size_t comma = rest.find(',');
    const bool last = c == ncols - 1;
    if (last != (comma == std::string_view::npos)) return at + "expected " + std::to_string(ncols) + " fields";
    const std::string_view field = last ? rest : rest.substr(0, comma);
    if (field.empty()) return at + "missing value";
    if (kinds[c] == LAQ_COL_FLOAT) {
      double v = 0;
      const auto [p, ec] = std::from_chars(field.data(), field.data() + field.size(), v);
      if (ec != std::errc() || p != field.data() + field.size()) return at + "bad float '" + std::string(field) + "'";
    } else {
      long long v = 0;
      const auto [p, ec] = std::from_chars(field.data(), field.data() + field.size(), v);
      if (ec != std::errc() || p != field.data() + field.size()) return at + "bad integer '" + std::string(field) + "'";
    }
    if (!last) rest.remove_prefix(comma + 1);
  }
  return at + "bad value";
}

}  // namespace
}  // namespace laq

using namespace laq;

extern "C" {

int laq_csv_open(laq_ctx* ctx, const char* d_text, int64_t nbytes, laq_csv** out, int64_t* h_lines) {
  return guard(ctx, [&] {
    if (nbytes < 0) fail(LAQ_ERR_SHAPE, "negative byte count");
    auto f = std::make_unique<laq_csv>();
    f->ctx = ctx;
    f->text = d_text;
    f->nbytes = nbytes;
    const int64_t tiles = (nbytes + kTileBytes - 1) / kTileBytes;
    if (tiles > 0) {
      DevBuf<int64_t> counts(ctx, tiles), offs(ctx, tiles);
      nl_count_kernel<<<static_cast<unsigned>(tiles), kTileThreads, 0, ctx->stream>>>(d_text, nbytes, counts.get());
      launched(ctx);
      size_t tmp = 0;
      LAQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts.get(), offs.get(), tiles, ctx->stream));
      DevBuf<char> scratch(ctx, std::max<size_t>(tmp, 1));
      LAQ_CUDA(cub::DeviceScan::ExclusiveSum(scratch.get(), tmp, counts.get(), offs.get(), tiles, ctx->stream));
      // one synchronisation: newline total (sizes the index) and the final byte
      ctx->h_pinned[2] = 0;
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, offs.get() + tiles - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned + 1, counts.get() + tiles - 1, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               ctx->stream));
      LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned + 2, d_text + nbytes - 1, 1, cudaMemcpyDeviceToHost, ctx->stream));
      sync(ctx);
      const int64_t n_nl = ctx->h_pinned[0] + ctx->h_pinned[1];
      const char tail = static_cast<char>(ctx->h_pinned[2] & 0xff);
      f->nl = DevBuf<int64_t>(ctx, static_cast<size_t>(std::max<int64_t>(n_nl, 1)));
      nl_write_kernel<<<static_cast<unsigned>(tiles), kTileThreads, 0, ctx->stream>>>(d_text, nbytes, offs.get(),
                                                                                      f->nl.get());
      launched(ctx);
      // getline: a final line without '\n' still counts; a final '\n' opens no line.
      f->lines = n_nl + (tail != '\n' ? 1 : 0);
      f->n_nl = n_nl;
    }
    *h_lines = f->lines;
    *out = f.release();
  });
}

int laq_csv_parse(laq_ctx* ctx, const laq_csv* f, int32_t n_cols, const int32_t* h_kinds, void* const* d_cols) {
  return guard(ctx, [&] {
    if (n_cols < 1) fail(LAQ_ERR_FORMAT, "schema has no columns");
    for (int c = 0; c < n_cols; ++c)
      if (h_kinds[c] != LAQ_COL_KEY && h_kinds[c] != LAQ_COL_INT && h_kinds[c] != LAQ_COL_FLOAT)
        fail(LAQ_ERR_FORMAT, "unknown column kind");
    if (n_cols > kMaxCsvCols) fail(LAQ_ERR_UNSUPPORTED, "at most 64 columns per CSV table");
    if (f->lines == 0) return;
    unsigned long long* flags = reinterpret_cast<unsigned long long*>(ctx->d_flags + 60);
    ParseArgs a{};
    a.t = f->text;
    a.nbytes = f->nbytes;
    a.lines = f->lines;
    a.n_nl = f->n_nl;
    a.nl = f->nl.get();
    a.ncols = n_cols;
    for (int c = 0; c < n_cols; ++c) {
      a.kinds[c] = h_kinds[c];
      a.cols[c] = d_cols[c];
    }
    a.bad = flags;
    a.unsupported = flags + 1;
    LAQ_CUDA(cudaMemsetAsync(flags, 0xFF, 2 * sizeof(unsigned long long), ctx->stream));
    parse_kernel<<<grid_for(f->lines, 256, ctx->sm_count * 16), 256, 0, ctx->stream>>>(a);
    launched(ctx);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, flags, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const unsigned long long h[2] = {static_cast<unsigned long long>(ctx->h_pinned[0]),
                                     static_cast<unsigned long long>(ctx->h_pinned[1])};
    if (h[0] == ~0ull) return;
    const int64_t line_no = static_cast<int64_t>(h[0]);
    if (h[1] == h[0])
      fail(LAQ_ERR_UNSUPPORTED, "line " + std::to_string(line_no) +
                                    ": float with more than 19 significant digits (dropped digits decide the rounding)");
    // Rebuild the reference's message from the failing line's bytes.
    int64_t se[2] = {0, f->nbytes};
    const int64_t r = line_no - 1;
    if (r > 0) LAQ_CUDA(cudaMemcpy(&se[0], f->nl.get() + r - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (r > 0) se[0] += 1;
    if (r < a.n_nl) LAQ_CUDA(cudaMemcpy(&se[1], f->nl.get() + r, sizeof(int64_t), cudaMemcpyDeviceToHost));
    std::string line(static_cast<size_t>(se[1] - se[0]), '\0');
    if (!line.empty()) LAQ_CUDA(cudaMemcpy(line.data(), f->text + se[0], line.size(), cudaMemcpyDeviceToHost));
    fail(LAQ_ERR_FORMAT, line_error(line, line_no, n_cols, h_kinds));
  });
}

int laq_csv_close(laq_csv* f) {
  delete f;
  return LAQ_OK;
}

}  // extern "C"
