// io.cpp -- native, multi-threaded parsers for the reference's cloud and
// weight files (gravreg/io.py:11-111), the ingestion step in front of the
// GPU path: Python's per-token parsing of a 1M-point XYZ
// file costs seconds once the registration itself takes milliseconds.
//
// Semantics are the reference's, on ASCII text:
//   * load_cloud: lines as str.splitlines() after universal-newline decoding
//     (\n, \r\n, \r, \v, \f, \x1c-\x1e); a line counts if its strip() is
//     non-empty and does not start with '#'; the first such line fixes the
//     column count (2 or 3), every other must match; tokens are split on
//     whitespace and converted like Python float() (sign, digits with single
//     underscores between digits, '.', exponent, inf/infinity/nan in any
//     case) -- glibc strtod is correctly rounded, like CPython's dtoa.
//     "ply" as the first non-blank line selects the ascii-PLY reader
//     (io.py:46-85): header with "format ascii 1.0", the vertex element's
//     properties, x/y/z columns from the first n_vertex non-blank body rows.
//   * load_weights: file iteration lines (\n, \r\n, \r), strip(), skip blank
//     and '#', one float per line.
// Anything these parsers do not accept (including every malformed file and
// any byte >= 0x80 outside a '#' comment line) returns FGA_ERR_PARSE; the Python layer then re-reads
// the file with its own port of io.py so the exception (class, line number,
// message) is exactly the reference's.  So the native path may be stricter
// than the reference, never more lenient.
//
// Work is split into one chunk per thread at line boundaries; each chunk is
// parsed independently into its own buffer, then chunks are concatenated in
// file order.
#include <omp.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/fga.h"
#include "fga_internal.cuh"

namespace fga {
namespace {

// str.isspace() on ASCII
inline bool is_space(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}
// str.splitlines() boundaries on ASCII (\r\n handled by the caller)
inline bool is_break_splitlines(unsigned char c) {
  return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e);
}
inline bool is_break_file(unsigned char c) { return c == '\n' || c == '\r'; }

inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

bool ieq(const char* a, const char* b, size_t n) {  // a (len n) equals lower-case b
  if (strlen(b) != n) return false;
  for (size_t i = 0; i < n; i++) {
    char c = a[i];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != b[i]) return false;
  }
  return true;
}

// Small fixed buffer for one token's digits (tokens longer than kTok are
// rejected here and left to the Python reader).
constexpr int kTok = 96;
struct TokBuf {
  char c[kTok + 1];
  int n = 0;
  bool push(char ch) {
    if (n >= kTok) return false;
    c[n++] = ch;
    return true;
  }
};

// digits with single underscores between digits, appended to out.  Returns
// the number of digits; ok = false on a misplaced underscore or overflow.
int digit_run(const char*& p, const char* e, TokBuf& out, bool& ok) {
  int n = 0;
  while (p < e) {
    if (is_digit((unsigned char)*p)) {
      ok = out.push(*p++) && ok;
      n++;
    } else if (*p == '_' && n > 0 && p + 1 < e && is_digit((unsigned char)p[1])) {
      p++;
    } else {
      break;
    }
  }
  if (p < e && *p == '_') ok = false;
  return n;
}

// Python float() of one whitespace-free token.
bool py_float(const char* s, const char* e, double* out) {
  const char* p = s;
  TokBuf buf;
  bool ok = true;
  if (p < e && (*p == '+' || *p == '-')) ok = buf.push(*p++);
  const size_t rest = (size_t)(e - p);
  if (ieq(p, "inf", rest) || ieq(p, "infinity", rest) || ieq(p, "nan", rest)) {
    for (size_t k = 0; k < rest; k++) ok = buf.push(p[k]) && ok;
    buf.c[buf.n] = 0;
    *out = strtod(buf.c, nullptr);
    return ok;
  }
  const int ni = digit_run(p, e, buf, ok);
  int nf = 0;
  if (p < e && *p == '.') {
    ok = buf.push(*p++) && ok;
    nf = digit_run(p, e, buf, ok);
  }
  if (!ok || ni + nf == 0) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ok = buf.push(*p++) && ok;
    if (p < e && (*p == '+' || *p == '-')) ok = buf.push(*p++) && ok;
    if (digit_run(p, e, buf, ok) == 0 || !ok) return false;
  }
  if (p != e) return false;
  buf.c[buf.n] = 0;
  char* end = nullptr;
  *out = strtod(buf.c, &end);  // overflow -> +-inf, underflow -> 0 / subnormal: as float()
  return end == buf.c + buf.n;
}

struct Span {
  const char* b;
  const char* e;
};

inline Span strip(Span s) {
  while (s.b < s.e && is_space((unsigned char)*s.b)) s.b++;
  while (s.e > s.b && is_space((unsigned char)s.e[-1])) s.e--;
  return s;
}

// next line of [p, end) with the given break rule; p advances past the break
template <bool kSplitlines>
inline bool next_line(const char*& p, const char* end, Span& line) {
  if (p >= end) return false;
  const char* q = p;
  while (q < end && !(kSplitlines ? is_break_splitlines((unsigned char)*q)
                                  : is_break_file((unsigned char)*q)))
    q++;
  line = Span{p, q};
  if (q < end) {
    if (*q == '\r' && q + 1 < end && q[1] == '\n') q++;
    q++;
  }
  p = q;
  return true;
}

// chunk boundaries: after a line break, never between \r and \n
std::vector<const char*> chunk_starts(const char* b, const char* e, int parts, bool splitlines) {
  std::vector<const char*> s{b};
  const size_t len = (size_t)(e - b);
  for (int k = 1; k < parts; k++) {
    const char* p = b + len * k / parts;
    if (p <= s.back()) continue;
    while (p < e && !(splitlines ? is_break_splitlines((unsigned char)p[-1])
                                 : is_break_file((unsigned char)p[-1])))
      p++;
    if (p < e && p[-1] == '\r' && *p == '\n') p++;
    if (p < e && p > s.back()) s.push_back(p);
  }
  s.push_back(e);
  return s;
}

int threads_for(size_t bytes) {
  const int t = omp_get_max_threads();
  const int by_size = (int)(bytes / (1 << 14)) + 1;  // >= 16 KiB per thread
  return by_size < t ? by_size : t;
}

// Non-ASCII text is accepted only inside whole-line '#' comments (the lines
// both readers skip, io.py:27-28), as well-formed UTF-8 (what open() decodes;
// anything else raises in the reference) that encodes no line break
// (U+0085, U+2028, U+2029 split lines in str.splitlines()).  Lines are cut at
// the superset of both readers' breaks, so this may reject (-> the Python
// reader) but never accept text the reference reads differently.
bool nonascii_only_in_comments(const char* b, size_t n) {
  bool line_start = true, comment = false;
  for (size_t i = 0; i < n;) {
    const unsigned char c = (unsigned char)b[i];
    if (c < 0x80) {
      if (is_break_splitlines(c)) {
        line_start = true;
        comment = false;
      } else if (line_start && !is_space(c)) {
        line_start = false;
        comment = c == '#';
      }
      i++;
      continue;
    }
    if (!comment) return false;
    int len;
    uint32_t cp;
    if (c >= 0xc2 && c <= 0xdf) {
      len = 2;
      cp = c & 0x1f;
    } else if (c >= 0xe0 && c <= 0xef) {
      len = 3;
      cp = c & 0x0f;
    } else if (c >= 0xf0 && c <= 0xf4) {
      len = 4;
      cp = c & 0x07;
    } else {
      return false;  // continuation byte, overlong lead or > U+10FFFF
    }
    if (i + len > n) return false;
    for (int k = 1; k < len; k++) {
      const unsigned char d = (unsigned char)b[i + k];
      if ((d & 0xc0) != 0x80) return false;
      cp = (cp << 6) | (d & 0x3f);
    }
    if ((len == 3 && cp < 0x800) || (len == 4 && (cp < 0x10000 || cp > 0x10ffff)) ||
        (cp >= 0xd800 && cp <= 0xdfff))
      return false;  // overlong, out of range or a surrogate
    if (cp == 0x85 || cp == 0x2028 || cp == 0x2029) return false;
    i += len;
  }
  return true;
}

// ---- XYZ (io.py:23-43): rows of `width` floats
struct XyzChunk {
  std::vector<double> v;
  int width = 0;  // of the chunk's first data row (0: none)
  bool ok = true;
};

void parse_xyz_chunk(const char* b, const char* e, XyzChunk& c) {
  Span line;
  const char* p = b;
  double tmp[3];
  while (next_line<true>(p, e, line)) {
    const Span t = strip(line);
    if (t.b == t.e || *t.b == '#') continue;
    int nf = 0;
    const char* q = t.b;
    while (q < t.e) {
      while (q < t.e && is_space((unsigned char)*q)) q++;
      if (q >= t.e) break;
      const char* w = q;
      while (w < t.e && !is_space((unsigned char)*w)) w++;
      if (nf >= 3 || !py_float(q, w, &tmp[nf])) {
        c.ok = false;
        return;
      }
      nf++;
      q = w;
    }
    if (c.width == 0) {
      if (nf != 2 && nf != 3) {
        c.ok = false;
        return;
      }
      c.width = nf;
    } else if (nf != c.width) {
      c.ok = false;
      return;
    }
    c.v.insert(c.v.end(), tmp, tmp + nf);
  }
}

// The two-call protocol (count, then fill) parses once: the first call keeps
// its result here, keyed by the text pointer and length.
struct ParseCache {
  const char* text = nullptr;
  int64_t len = -1;
  uint64_t hash = 0;
  int dim = 0;
  std::vector<double> v;
};

// content hash (parallel), so a fill call never takes a stale parse of
// other bytes that happen to sit at the same address
uint64_t text_hash(const char* b, int64_t len) {
  const int64_t nw = len / 8;
  uint64_t h = 0;
#pragma omp parallel for reduction(+ : h) schedule(static)
  for (int64_t k = 0; k < nw; k++) {
    uint64_t w;
    memcpy(&w, b + 8 * k, 8);
    h += (w ^ (uint64_t)k) * 0x9E3779B97F4A7C15ull;
  }
  for (int64_t k = nw * 8; k < len; k++) h = h * 131 + (unsigned char)b[k];
  return h;
}
thread_local ParseCache g_cloud_cache, g_weight_cache;

int deliver(ParseCache& c, double* out, int64_t cap, int64_t* n_out, int* dim_out) {
  const int64_t total = (int64_t)c.v.size();
  *n_out = c.dim ? total / c.dim : total;
  if (dim_out) *dim_out = c.dim;
  if (!out) return FGA_OK;
  if (cap < total) {
    set_error("parse: output buffer too small");
    return FGA_ERR_INVALID;
  }
  if (total) memcpy(out, c.v.data(), sizeof(double) * total);
  c = ParseCache();  // delivered: release
  return FGA_OK;
}

}  // namespace
}  // namespace fga

using namespace fga;

extern "C" {

int fga_parse_cloud(const char* text, int64_t len, double* out, int64_t cap, int64_t* n_out,
                    int* dim_out) {
  if (!text || len < 0 || !n_out || !dim_out) {
    set_error("parse_cloud: null argument");
    return FGA_ERR_INVALID;
  }
  *n_out = 0;
  *dim_out = 0;
  ParseCache& cache = g_cloud_cache;
  const uint64_t h = text_hash(text, len);
  if (cache.text == text && cache.len == len && cache.hash == h)
    return deliver(cache, out, cap, n_out, dim_out);
  cache = ParseCache();
  const char* b = text;
  const char* e = text + len;
  if (!nonascii_only_in_comments(b, (size_t)len)) {
    set_error("parse_cloud: non-ASCII input outside comments (left to the Python reader)");
    return FGA_ERR_PARSE;
  }
  // sniff the first non-blank line (io.py:14-20)
  const char* p = b;
  Span line;
  bool ply = false, any = false;
  while (next_line<true>(p, e, line)) {
    const Span t = strip(line);
    if (t.b == t.e) continue;
    any = true;
    ply = ieq(t.b, "ply", (size_t)(t.e - t.b));
    break;
  }
  if (!any) {
    set_error("parse_cloud: empty file");
    return FGA_ERR_PARSE;
  }
  if (!ply) {
    const int T = threads_for((size_t)len);
    const auto st = chunk_starts(b, e, T, true);
    const int nc = (int)st.size() - 1;
    std::vector<XyzChunk> ch(nc);
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int k = 0; k < nc; k++) parse_xyz_chunk(st[k], st[k + 1], ch[k]);
    int width = 0;
    int64_t total = 0;
    for (auto& c : ch) {
      if (!c.ok) {
        set_error("parse_cloud: malformed XYZ");
        return FGA_ERR_PARSE;
      }
      if (c.width && !width) width = c.width;
      if (c.width && c.width != width) {
        set_error("parse_cloud: column count changes");
        return FGA_ERR_PARSE;
      }
      total += (int64_t)c.v.size();
    }
    if (width == 0) {
      set_error("parse_cloud: no points");
      return FGA_ERR_PARSE;
    }
    std::vector<int64_t> off(nc + 1, 0);
    for (int k = 0; k < nc; k++) off[k + 1] = off[k] + (int64_t)ch[k].v.size();
    double* dst = out;
    if (!out || cap < total) {  // keep the result for the fill call
      cache.v.resize((size_t)total);
      dst = cache.v.data();
    }
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int k = 0; k < nc; k++)
      if (!ch[k].v.empty()) memcpy(dst + off[k], ch[k].v.data(), sizeof(double) * ch[k].v.size());
    *n_out = total / width;
    *dim_out = width;
    if (dst == out) return FGA_OK;
    cache.text = text;
    cache.len = len;
    cache.hash = h;
    cache.dim = width;
    if (out) {
      set_error("parse_cloud: output buffer too small");
      return FGA_ERR_INVALID;
    }
    return FGA_OK;
  }
  // ---- ascii PLY (io.py:46-85)
  p = b;
  int64_t idx = 0, n_vertex = -1;
  bool in_vertex = false, header_done = false;
  std::vector<std::string> props;
  while (next_line<true>(p, e, line)) {
    const Span t = strip(line);
    const std::string s(t.b, t.e);
    if (idx++ == 0) continue;
    if (s.rfind("format", 0) == 0) {
      if (s != "format ascii 1.0") {
        set_error("parse_cloud: unsupported PLY format");
        return FGA_ERR_PARSE;
      }
    } else if (s.rfind("element", 0) == 0) {
      std::vector<std::string> f;
      for (const char* q = t.b; q < t.e;) {
        while (q < t.e && is_space((unsigned char)*q)) q++;
        const char* w = q;
        while (w < t.e && !is_space((unsigned char)*w)) w++;
        if (w > q) f.emplace_back(q, w);
        q = w;
      }
      if (f.size() < 2) {
        set_error("parse_cloud: malformed element line");
        return FGA_ERR_PARSE;
      }
      in_vertex = f[1] == "vertex";
      if (in_vertex) {
        if (f.size() < 3) {
          set_error("parse_cloud: malformed vertex element");
          return FGA_ERR_PARSE;
        }
        char* endp = nullptr;
        const long long v = strtoll(f[2].c_str(), &endp, 10);
        if (*endp || f[2].empty() || !(is_digit((unsigned char)f[2][0]) || f[2][0] == '+')) {
          set_error("parse_cloud: bad vertex count");
          return FGA_ERR_PARSE;
        }
        n_vertex = v;
      }
    } else if (s.rfind("property", 0) == 0 && in_vertex) {
      const char* w = t.e;
      while (w > t.b && !is_space((unsigned char)w[-1])) w--;
      props.emplace_back(w, t.e);
    } else if (s == "end_header") {
      header_done = true;
      break;
    }
  }
  if (!header_done || n_vertex < 0) {
    set_error("parse_cloud: missing PLY header terminator or vertex element");
    return FGA_ERR_PARSE;
  }
  int cols[3];
  const char* axes[3] = {"x", "y", "z"};
  for (int a = 0; a < 3; a++) {
    cols[a] = -1;
    for (size_t k = 0; k < props.size(); k++)
      if (props[k] == axes[a]) {
        cols[a] = (int)k;
        break;
      }
    if (cols[a] < 0) {
      set_error("parse_cloud: vertex element lacks x y z properties");
      return FGA_ERR_PARSE;
    }
  }
  // body: the first n_vertex non-blank lines after the header
  std::vector<double> v;
  v.reserve((size_t)n_vertex * 3);
  int64_t rows = 0;
  while (rows < n_vertex && next_line<true>(p, e, line)) {
    const Span t = strip(line);
    if (t.b == t.e) continue;
    const char* fb[64];
    const char* fe[64];
    int nf = 0;
    for (const char* q = line.b; q < line.e && nf < 64;) {
      while (q < line.e && is_space((unsigned char)*q)) q++;
      if (q >= line.e) break;
      const char* w = q;
      while (w < line.e && !is_space((unsigned char)*w)) w++;
      fb[nf] = q;
      fe[nf] = w;
      nf++;
      q = w;
    }
    for (int a = 0; a < 3; a++) {
      double x;
      if (cols[a] >= nf || !py_float(fb[cols[a]], fe[cols[a]], &x)) {
        set_error("parse_cloud: bad PLY vertex row");
        return FGA_ERR_PARSE;
      }
      v.push_back(x);
    }
    rows++;
  }
  if (rows < n_vertex || rows == 0) {
    set_error("parse_cloud: PLY vertex count exceeds body rows (or is 0)");
    return FGA_ERR_PARSE;
  }
  cache.text = text;
  cache.len = len;
  cache.hash = h;
  cache.dim = 3;
  cache.v.swap(v);
  return deliver(cache, out, cap, n_out, dim_out);
}

int fga_parse_weights(const char* text, int64_t len, double* out, int64_t cap, int64_t* n_out) {
  if (!text || len < 0 || !n_out) {
    set_error("parse_weights: null argument");
    return FGA_ERR_INVALID;
  }
  *n_out = 0;
  ParseCache& cache = g_weight_cache;
  const uint64_t h = text_hash(text, len);
  if (cache.text == text && cache.len == len && cache.hash == h)
    return deliver(cache, out, cap, n_out, nullptr);
  cache = ParseCache();
  const char* b = text;
  const char* e = text + len;
  if (!nonascii_only_in_comments(b, (size_t)len)) {
    set_error("parse_weights: non-ASCII input outside comments (left to the Python reader)");
    return FGA_ERR_PARSE;
  }
  const int T = threads_for((size_t)len);
  const auto st = chunk_starts(b, e, T, false);
  const int nc = (int)st.size() - 1;
  std::vector<std::vector<double>> ch(nc);
  std::vector<char> ok(nc, 1);
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int k = 0; k < nc; k++) {
    Span line;
    const char* p = st[k];
    while (next_line<false>(p, st[k + 1], line)) {
      const Span t = strip(line);
      if (t.b == t.e || *t.b == '#') continue;
      double x;
      if (!py_float(t.b, t.e, &x)) {
        ok[k] = 0;
        break;
      }
      ch[k].push_back(x);
    }
  }
  int64_t total = 0;
  for (int k = 0; k < nc; k++) {
    if (!ok[k]) {
      set_error("parse_weights: malformed weight");
      return FGA_ERR_PARSE;
    }
    total += (int64_t)ch[k].size();
  }
  cache.v.resize((size_t)total);
  int64_t o = 0;
  for (int k = 0; k < nc; k++) {
    if (!ch[k].empty()) memcpy(cache.v.data() + o, ch[k].data(), sizeof(double) * ch[k].size());
    o += (int64_t)ch[k].size();
  }
  cache.text = text;
  cache.len = len;
  cache.hash = h;
  cache.dim = 0;
  return deliver(cache, out, cap, n_out, nullptr);
}

}  // extern "C"

// ------------------------------------------------------------------ staging
// Copies the byte range [lo, hi) of the virtual concatenation of `nseg`
// host segments (src[k], prefix[k+1] - prefix[k] bytes) into dst, on all host
// threads (fga_register_batch_list: many small clouds -> one pinned staging
// chunk, no numpy concatenation).
namespace fga {
void host_gather_segments(const char* const* src, const int64_t* prefix, int64_t nseg,
                          int64_t lo, int64_t hi, char* dst) {
  if (hi <= lo) return;
  // first segment holding byte lo
  int64_t a = 0, b = nseg;
  while (b - a > 1) {
    const int64_t mid = (a + b) / 2;
    if (prefix[mid] <= lo) a = mid; else b = mid;
  }
  int64_t last = a;
  while (last + 1 < nseg && prefix[last + 1] < hi) last++;
  const int64_t first = a;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = first; k <= last; k++) {
    const int64_t s0 = std::max(prefix[k], lo), s1 = std::min(prefix[k + 1], hi);
    if (s1 > s0) std::memcpy(dst + (s0 - lo), src[k] + (s0 - prefix[k]), (size_t)(s1 - s0));
  }
}
}  // namespace fga
