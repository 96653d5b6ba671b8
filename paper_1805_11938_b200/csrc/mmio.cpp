// Matrix Market coordinate-entry tokenizer (host, multithreaded) feeding the
// GPU canonicalize.  Reference semantics: coo.py:158-263.
//
// Python parses the banner and the size line (cheap, exact messages); this
// parser takes the text after the size line and produces the expanded
// triplets (1-based -> 0-based, symmetric off-diagonal entries mirrored,
// pattern entries = 1.0).  Lines are split on '\n' (a trailing '\r' is
// whitespace); a line is skipped when it is blank or starts with '%' after
// stripping.  On any problem it returns a status and the 1-based line number
// (relative to the first parsed line) so the caller can raise the
// reference's exact MatrixMarketError, or re-parse with the reference-
// semantics Python parser when the text is outside the fast path's grammar
// (non-ASCII bytes, separators other than '\n', Python-only numeric
// spellings such as "1_000").
#include <algorithm>
#include <charconv>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {

enum MmStatus {
  MM_OK = 0,
  MM_FIELDS = 1,     // wrong number of fields
  MM_NUMBER = 2,     // a field is not a number
  MM_BOUNDS = 3,     // index out of declared bounds
  MM_TOO_MANY = 4,   // more entries than declared
  MM_TOO_FEW = 5,    // fewer entries than declared (line = last line)
  MM_UNSUPPORTED = 6 // outside the fast-path grammar: caller re-parses
};

inline bool is_space(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f'; }

struct Line {
  const char* b;
  const char* e;
};

// strip; returns false for blank/comment lines
inline bool content(const char* b, const char* e, Line& out) {
  while (b < e && is_space(*b)) ++b;
  while (e > b && is_space(e[-1])) --e;
  if (b == e || *b == '%') return false;
  out = {b, e};
  return true;
}

inline int split(const Line& l, const char* tok[4], int len[4]) {
  int n = 0;
  const char* p = l.b;
  while (p < l.e) {
    while (p < l.e && is_space(*p)) ++p;
    if (p >= l.e) break;
    const char* s = p;
    while (p < l.e && !is_space(*p)) ++p;
    if (n < 4) {
      tok[n] = s;
      len[n] = static_cast<int>(p - s);
    }
    ++n;
  }
  return n;
}

// Python int(): optional sign, decimal digits (underscores etc. -> caller).
inline bool parse_int(const char* s, int len, int64_t& v) {
  if (len > 0 && *s == '+') {
    ++s;
    --len;
    if (len > 0 && *s == '-') return false;
  }
  if (len <= 0 || len > 19) return false;
  auto r = std::from_chars(s, s + len, v, 10);
  return r.ec == std::errc() && r.ptr == s + len;
}

// Python float() on plain decimal / exponent / inf / nan spellings;
// std::from_chars is correctly rounded like float().
inline bool parse_real(const char* s, int len, double& v) {
  if (len > 0 && *s == '+') {
    ++s;
    --len;
    if (len > 0 && (*s == '+' || *s == '-')) return false;
  }
  if (len <= 0) return false;
  for (int i = 0; i < len; ++i)
    if (s[i] == '_' || s[i] == '(') return false;  // Python-only spelling / nan(...): caller decides
  auto r = std::from_chars(s, s + len, v, std::chars_format::general);
  if (r.ec == std::errc::result_out_of_range) {  // float() returns +-inf / +-0.0 there
    char buf[128];
    if (len >= 127) return false;
    std::memcpy(buf, s, len);
    buf[len] = 0;
    char* end = nullptr;
    v = std::strtod(buf, &end);
    return end == buf + len;
  }
  return r.ec == std::errc() && r.ptr == s + len;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0;      // '\n'-terminated lines in the chunk
  int64_t entries = 0;    // non-blank, non-comment lines
  int64_t first_line = 0; // global line number of the chunk's first line (1-based)
  int64_t first_entry = 0;
  int status = MM_OK;
  int64_t bad_line = 0;
  int64_t bad_i = 0, bad_j = 0;
};

}  // namespace

extern "C" int spmvb_mm_parse(const char* text, int64_t len, int pattern, int symmetric, int64_t n_rows,
                              int64_t n_cols, int64_t declared, int64_t cap, int64_t* row_out, int64_t* col_out,
                              double* val_out, int64_t* n_out, int64_t* err_line, int64_t* err_ij, int n_threads) {
  if (n_threads < 1) n_threads = 1;
  if (len < (1 << 20)) n_threads = 1;
  // chunk boundaries at line starts
  std::vector<Chunk> ch(n_threads);
  const char* end = text + len;
  const char* prev = text;
  for (int t = 0; t < n_threads; ++t) {
    const char* e = (t == n_threads - 1) ? end : text + len * (t + 1) / n_threads;
    if (e < prev) e = prev;
    while (e < end && e > text && e[-1] != '\n') ++e;
    ch[t].b = prev;
    ch[t].e = e;
    prev = e;
  }
  const int want = pattern ? 2 : 3;
  // pass 1: lines and entry counts per chunk.  Text outside the fast-path
  // grammar (the caller re-parses with Python's str.splitlines()/strip()/
  // int()/float() semantics): non-ASCII bytes and line separators other than
  // "\n" / "\r\n".
  auto count = [&](Chunk& c) {
    for (const char* q = c.b; q < c.e; ++q) {
      const unsigned char b = static_cast<unsigned char>(*q);
      if (b >= 0x80 || b == 0x0b || b == 0x0c || (b >= 0x1c && b <= 0x1e) ||
          (b == '\r' && (q + 1 >= end || q[1] != '\n'))) {
        c.status = MM_UNSUPPORTED;
        return;
      }
    }
    const char* p = c.b;
    while (p < c.e) {
      const char* q = static_cast<const char*>(std::memchr(p, '\n', c.e - p));
      const char* le = q ? q : c.e;
      Line l;
      if (content(p, le, l)) ++c.entries;
      ++c.lines;
      p = q ? q + 1 : c.e;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < n_threads; ++t) th.emplace_back(count, std::ref(ch[t]));
    count(ch[0]);
    for (auto& x : th) x.join();
  }
  for (auto& c : ch)
    if (c.status != MM_OK) return c.status;
  int64_t line = 1, entry = 0;
  for (auto& c : ch) {
    c.first_line = line;
    c.first_entry = entry;
    line += c.lines;
    entry += c.entries;
  }
  const int64_t total_lines = line - 1;
  // output slots: each entry emits 1 or 2 triplets; prefix over chunks needs
  // the diagonal count, so symmetric input uses 2 slots per entry then compacts.
  const int64_t per = symmetric ? 2 : 1;
  if (std::min<int64_t>(entry, declared) * per > cap) return MM_UNSUPPORTED;
  auto parse = [&](Chunk& c) {
    const char* p = c.b;
    int64_t ln = c.first_line, en = c.first_entry;
    while (p < c.e) {
      const char* q = static_cast<const char*>(std::memchr(p, '\n', c.e - p));
      const char* le = q ? q : c.e;
      Line l;
      if (content(p, le, l)) {
        auto bad = [&](int st) {
          c.status = st;
          c.bad_line = ln;
        };
        if (en >= declared) return bad(MM_TOO_MANY);
        const char* tok[4];
        int tl[4];
        const int nt = split(l, tok, tl);
        if (nt != want) return bad(MM_FIELDS);
        int64_t i, j;
        double v = 1.0;
        if (!parse_int(tok[0], tl[0], i) || !parse_int(tok[1], tl[1], j) || (!pattern && !parse_real(tok[2], tl[2], v)))
          return bad(MM_NUMBER);
        if (!(1 <= i && i <= n_rows && 1 <= j && j <= n_cols)) {
          c.bad_i = i;
          c.bad_j = j;
          return bad(MM_BOUNDS);
        }
        const int64_t o = en * per;
        row_out[o] = i - 1;
        col_out[o] = j - 1;
        val_out[o] = v;
        if (symmetric) {
          // mirrored entry, or a marker (-1) for a diagonal entry
          row_out[o + 1] = (i != j) ? j - 1 : -1;
          col_out[o + 1] = i - 1;
          val_out[o + 1] = v;
        }
        ++en;
      }
      ++ln;
      p = q ? q + 1 : c.e;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < n_threads; ++t) th.emplace_back(parse, std::ref(ch[t]));
    parse(ch[0]);
    for (auto& x : th) x.join();
  }
  for (auto& c : ch)
    if (c.status != MM_OK) {
      *err_line = c.bad_line;
      err_ij[0] = c.bad_i;
      err_ij[1] = c.bad_j;
      return c.status;
    }
  if (entry != declared) {
    *err_line = total_lines;
    return MM_TOO_FEW;
  }
  int64_t n = entry * per;
  if (symmetric) {  // drop the diagonal markers, order preserved
    int64_t w = 0;
    for (int64_t k = 0; k < n; ++k)
      if (row_out[k] >= 0) {
        row_out[w] = row_out[k];
        col_out[w] = col_out[k];
        val_out[w] = val_out[k];
        ++w;
      }
    n = w;
  }
  *n_out = n;
  return MM_OK;
}

// ---------------------------------------------------------------------------
// write_matrix_market entry formatter (coo.py:266-278): one line per entry,
// "<row+1> <col+1> <value:.17g>\n", formatted by n_threads threads into
// per-thread buffers; _begin returns the total length, _finish copies the
// text into the caller's buffer and frees the plan.  std::to_chars(general,
// 17) is printf's %.17g, which is Python's format(v, ".17g") for every finite
// double; non-finite values are spelled as Python spells them (inf, -inf,
// nan).
// ---------------------------------------------------------------------------
#include <cmath>

struct spmvb_mm_text {
  std::vector<std::vector<char>> parts;
};

namespace {

inline char* put_int(char* p, int64_t v) { return std::to_chars(p, p + 24, v).ptr; }

inline char* put_real(char* p, double v) {
  if (std::isnan(v)) {
    std::memcpy(p, "nan", 3);
    return p + 3;
  }
  if (std::isinf(v)) {
    const char* s = v < 0 ? "-inf" : "inf";
    const size_t n = std::strlen(s);
    std::memcpy(p, s, n);
    return p + n;
  }
  return std::to_chars(p, p + 40, v, std::chars_format::general, 17).ptr;
}

}  // namespace

extern "C" int spmvb_mm_format_begin(const int64_t* row, const int64_t* col, const double* val, int64_t nnz,
                                     int n_threads, spmvb_mm_text** plan_out, int64_t* len_out) {
  if (!plan_out || !len_out || nnz < 0 || (nnz > 0 && (!row || !col || !val))) return 1;
  if (n_threads < 1) n_threads = 1;
  if (nnz < (1 << 16)) n_threads = 1;
  auto* plan = new (std::nothrow) spmvb_mm_text;
  if (!plan) return 5;
  plan->parts.resize(n_threads);
  bool failed = false;
  auto work = [&](int t) {
    const int64_t lo = nnz * t / n_threads, hi = nnz * (t + 1) / n_threads;
    try {
      std::vector<char>& out = plan->parts[t];
      out.resize(static_cast<size_t>(hi - lo) * 72 + 8);  // 2 x 20 digits + 26 for the value + separators
      char* p = out.data();
      for (int64_t k = lo; k < hi; ++k) {
        p = put_int(p, row[k] + 1);
        *p++ = ' ';
        p = put_int(p, col[k] + 1);
        *p++ = ' ';
        p = put_real(p, val[k]);
        *p++ = '\n';
      }
      out.resize(static_cast<size_t>(p - out.data()));
    } catch (...) {
      failed = true;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < n_threads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  if (failed) {
    delete plan;
    return 5;
  }
  int64_t total = 0;
  for (auto& part : plan->parts) total += static_cast<int64_t>(part.size());
  *plan_out = plan;
  *len_out = total;
  return 0;
}

extern "C" int spmvb_mm_format_finish(spmvb_mm_text* plan, char* out) {
  if (!plan) return 1;
  if (out) {
    std::vector<std::thread> th;
    size_t off = 0;
    for (auto& part : plan->parts) {
      char* dst = out + off;
      const std::vector<char>* src = &part;
      th.emplace_back([dst, src] { std::memcpy(dst, src->data(), src->size()); });
      off += part.size();
    }
    for (auto& x : th) x.join();
  }
  delete plan;
  return 0;
}
