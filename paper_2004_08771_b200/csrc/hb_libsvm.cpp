// Native LIBSVM ingestion straight to CSR (the caller edge in front of the
// sparse first layer).
//
// Semantics follow the reference's dense loader, hogtrain/data.py:106-151
// (load_libsvm) and data.py:86-103 (_map_label), line for line:
//   - lines are split on whitespace; blank lines are skipped but counted;
//   - the label is the first comma-separated field of the first token,
//     parsed as int(float(s)); ZERO_ONE keeps non-negative values, PLUS_MINUS_ONE
//     maps -1 -> 0 and +1 -> 1; anything else is a parse error;
//   - each feature token is "idx:val" split at the first ':'; idx is a base-10
//     integer, val a float; a bad token is a parse error, an index outside
//     [1, feature_dim] a ValueError, both reported with the 1-based line number,
//     label first, then tokens left to right (the reference's order);
//   - a repeated index keeps the last value (row[idx-1] = val).
// The row is emitted as CSR: columns 0-based and ascending, explicit zeros
// dropped (the dense row the reference builds holds 0.0 there, which the
// forward multiplies away identically).
//
// Two passes over the buffer (scan: validate + count, fill: write), each split
// over threads at line boundaries; the output is independent of the thread count.

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/hogbatch_b200.h"

namespace hb {
int set_error(int code, const char* msg);
}

namespace {

struct LineError {
  long long line = -1;  // 1-based; -1 = none
  int code = HB_OK;
  std::string msg;
};

// str.split() whitespace over ASCII: \t \n \v \f \r, space and \x1c-\x1f
inline bool is_space(char ch) { return ch == ' ' || (ch >= '\t' && ch <= '\r') || (ch >= '\x1c' && ch <= '\x1f'); }

// Python float(): decimal or inf/nan spellings, optional sign, full consumption
// (strtod alone would also take hex floats, which Python rejects).
bool parse_float(const char* b, const char* e, double* out) {
  if (b == e) return false;
  const char* p = b;
  if (*p == '+' || *p == '-') ++p;
  if (e - p >= 2 && p[0] == '0' && (p[1] == 'x' || p[1] == 'X')) return false;
  char tmp[128];
  const size_t n = static_cast<size_t>(e - b);
  if (n >= sizeof tmp) {
    std::string s(b, e);
    char* end = nullptr;
    errno = 0;
    *out = std::strtod(s.c_str(), &end);
    return end == s.c_str() + s.size();
  }
  std::memcpy(tmp, b, n);
  tmp[n] = 0;
  char* end = nullptr;
  *out = std::strtod(tmp, &end);  // ERANGE overflow -> inf, as float() does
  return end == tmp + n;
}

// Python int() on a feature index: optional sign, decimal digits only.
bool parse_int(const char* b, const char* e, long long* out) {
  const char* p = b;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = (*p++ == '-');
  if (p == e) return false;
  long long v = 0;
  for (; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    if (v < (1ll << 60)) v = v * 10 + (*p - '0');  // saturate: anything this large is out of range anyway
  }
  *out = neg ? -v : v;
  return true;
}

struct RowParser {
  long long feature_dim;
  int mapping;  // 0 = ZERO_ONE, 1 = PLUS_MINUS_ONE
  std::vector<std::pair<int32_t, double>> ent;

  // Parses one non-blank line [b, e).  Returns false with err filled on error.
  bool parse(const char* b, const char* e, long long line_no, int64_t* label, LineError* err) {
    ent.clear();
    const char* p = b;
    while (p < e && is_space(*p)) ++p;
    const char* t0 = p;
    while (p < e && !is_space(*p)) ++p;
    const char* t1 = p;
    const char* comma = static_cast<const char*>(std::memchr(t0, ',', t1 - t0));
    double lv = 0.0;
    if (!parse_float(t0, comma ? comma : t1, &lv) || !std::isfinite(lv)) {
      // int(float('inf')) raises OverflowError / nan ValueError in the reference
      return error(err, line_no, HB_EPARSE, "line %lld: bad label '%s'", t0, t1);
    }
    const long long value = static_cast<long long>(std::trunc(lv));
    if (mapping == 1) {
      if (value == -1) {
        *label = 0;
      } else if (value == 1) {
        *label = 1;
      } else {
        char m[160];
        std::snprintf(m, sizeof m, "line %lld: label %lld not in {-1, +1}", line_no, value);
        err->line = line_no, err->code = HB_EPARSE, err->msg = m;
        return false;
      }
    } else {
      if (value < 0) {
        char m[160];
        std::snprintf(m, sizeof m, "line %lld: negative label %lld with zero_one mapping", line_no, value);
        err->line = line_no, err->code = HB_EPARSE, err->msg = m;
        return false;
      }
      *label = value;
    }
    for (;;) {
      while (p < e && is_space(*p)) ++p;
      if (p >= e) break;
      const char* a = p;
      while (p < e && !is_space(*p)) ++p;
      const char* z = p;
      const char* colon = static_cast<const char*>(std::memchr(a, ':', z - a));
      long long idx = 0;
      double v = 0.0;
      if (!colon || !parse_int(a, colon, &idx) || !parse_float(colon + 1, z, &v))
        return error(err, line_no, HB_EPARSE, "line %lld: bad feature token '%s'", a, z);
      if (idx < 1 || idx > feature_dim) {
        char m[200];
        std::snprintf(m, sizeof m, "line %lld: feature index %lld outside [1, %lld]", line_no, idx, feature_dim);
        err->line = line_no, err->code = HB_EINVAL, err->msg = m;
        return false;
      }
      ent.emplace_back(static_cast<int32_t>(idx - 1), v);
    }
    // ascending columns, last write wins on a repeated index, zeros dropped
    std::stable_sort(ent.begin(), ent.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    size_t w = 0;
    for (size_t i = 0; i < ent.size(); ++i) {
      if (i + 1 < ent.size() && ent[i + 1].first == ent[i].first) continue;
      if (ent[i].second != 0.0) ent[w++] = ent[i];
    }
    ent.resize(w);
    return true;
  }

  static bool error(LineError* err, long long line_no, int code, const char* fmt, const char* a, const char* z) {
    std::string tok(a, std::min<size_t>(z - a, 120));
    char m[320];
    std::snprintf(m, sizeof m, fmt, line_no, tok.c_str());
    err->line = line_no, err->code = code, err->msg = m;
    return false;
  }
};

struct Chunk {
  const char* b;
  const char* e;
  long long first_line;  // 1-based number of the chunk's first line
  long long rows = 0, nnz = 0;
  LineError err;
};

std::vector<Chunk> split_chunks(const char* buf, size_t len) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int want = static_cast<int>(std::max<size_t>(1, std::min<size_t>(std::min(hw, 32), len / (1 << 20))));
  std::vector<Chunk> ch;
  const char* p = buf;
  const char* end = buf + len;
  for (int t = 0; t < want && p < end; ++t) {
    const char* q = (t == want - 1) ? end : std::min(end, buf + len * (t + 1) / want);
    while (q < end && q[-1] != '\n') ++q;  // chunks end right after a newline
    if (q <= p) continue;
    ch.push_back(Chunk{p, q, 0, 0, 0, LineError{}});
    p = q;
  }
  // line numbers: count newlines per chunk (cheap, memchr)
  long long line = 1;
  for (auto& c : ch) {
    c.first_line = line;
    for (const char* s = c.b; s < c.e;) {
      const char* nl = static_cast<const char*>(std::memchr(s, '\n', c.e - s));
      if (!nl) break;
      ++line;
      s = nl + 1;
    }
  }
  return ch;
}

template <typename F>
void for_chunks(std::vector<Chunk>& ch, F f) {
  std::vector<std::thread> th;
  for (size_t i = 1; i < ch.size(); ++i) th.emplace_back(f, std::ref(ch[i]));
  if (!ch.empty()) f(ch[0]);
  for (auto& t : th) t.join();
}

// Walks the lines of a chunk, calling row(line_begin, line_end, line_no) for
// each non-blank one; stops when row returns false.
template <typename F>
void each_line(const Chunk& c, F row) {
  long long line = c.first_line;
  for (const char* s = c.b; s < c.e; ++line) {
    const char* nl = static_cast<const char*>(std::memchr(s, '\n', c.e - s));
    const char* le = nl ? nl : c.e;
    const char* p = s;
    while (p < le && is_space(*p)) ++p;
    if (p < le && !row(s, le, line)) return;
    s = nl ? nl + 1 : c.e;
  }
}

int first_error(const std::vector<Chunk>& ch) {
  for (const auto& c : ch)  // chunks are in file order, so the first one holds the earliest line
    if (c.err.code != HB_OK) return hb::set_error(c.err.code, c.err.msg.c_str());
  return HB_OK;
}

}  // namespace

extern "C" {

int hb_libsvm_scan(const char* buf, size_t len, int64_t feature_dim, int label_mapping, int64_t* n_rows,
                   int64_t* nnz) {
  if ((!buf && len) || !n_rows || !nnz) return hb::set_error(HB_EINVAL, "null buffer or outputs");
  if (feature_dim < 1 || feature_dim > INT32_MAX) return hb::set_error(HB_EINVAL, "feature_dim must be in [1, 2^31)");
  if (label_mapping != 0 && label_mapping != 1) return hb::set_error(HB_EINVAL, "label_mapping must be 0 or 1");
  auto ch = split_chunks(buf, len);
  for_chunks(ch, [&](Chunk& c) {
    RowParser rp{feature_dim, label_mapping, {}};
    int64_t lab = 0;
    each_line(c, [&](const char* b, const char* e, long long ln) {
      if (!rp.parse(b, e, ln, &lab, &c.err)) return false;
      c.rows += 1;
      c.nnz += static_cast<long long>(rp.ent.size());
      return true;
    });
  });
  if (const int rc = first_error(ch)) return rc;
  long long r = 0, z = 0;
  for (const auto& c : ch) r += c.rows, z += c.nnz;
  *n_rows = r;
  *nnz = z;
  return HB_OK;
}

int hb_libsvm_fill(const char* buf, size_t len, int64_t feature_dim, int label_mapping, int64_t* rowptr,
                   int32_t* col, double* val, int64_t* labels) {
  if ((!buf && len) || !rowptr || !labels) return hb::set_error(HB_EINVAL, "null buffer or outputs");
  if (feature_dim < 1 || feature_dim > INT32_MAX) return hb::set_error(HB_EINVAL, "feature_dim must be in [1, 2^31)");
  auto ch = split_chunks(buf, len);
  // counts first (same chunking), then each chunk writes at its offsets
  for_chunks(ch, [&](Chunk& c) {
    RowParser rp{feature_dim, label_mapping, {}};
    int64_t lab = 0;
    each_line(c, [&](const char* b, const char* e, long long ln) {
      if (!rp.parse(b, e, ln, &lab, &c.err)) return false;
      c.rows += 1;
      c.nnz += static_cast<long long>(rp.ent.size());
      return true;
    });
  });
  if (const int rc = first_error(ch)) return rc;
  std::vector<long long> row0(ch.size()), nz0(ch.size());
  long long r = 0, z = 0;
  for (size_t i = 0; i < ch.size(); ++i) row0[i] = r, nz0[i] = z, r += ch[i].rows, z += ch[i].nnz;
  rowptr[0] = 0;
  for_chunks(ch, [&](Chunk& c) {
    const size_t i = static_cast<size_t>(&c - ch.data());
    RowParser rp{feature_dim, label_mapping, {}};
    long long row = row0[i], k = nz0[i];
    each_line(c, [&](const char* b, const char* e, long long ln) {
      LineError err;
      rp.parse(b, e, ln, &labels[row], &err);
      for (const auto& pr : rp.ent) col[k] = pr.first, val[k] = pr.second, ++k;
      rowptr[++row] = k;
      return true;
    });
  });
  return HB_OK;
}

}  // extern "C"
