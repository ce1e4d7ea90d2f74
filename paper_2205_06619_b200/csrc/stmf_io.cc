// stmf_io.cc — streaming CSV reader for masked matrices:
// load_matrix_csv (io.py:33-60) without Python-level loops.  The file is read once
// into memory, records are located serially (memchr) and parsed in parallel on the
// host threads straight into the dense value array + byte mask.  Semantics follow
// the reference: csv records, blank records skipped, an optional header record,
// each cell stripped, "" / "nan" (any case) missing, anything else float() —
// strtod is correctly rounded, like Python's float() — and ragged rows rejected.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "stmf_b200.h"

int stmf_io_set_error(int code, const char* msg);  // stmf_api.cu

namespace {

struct CsvFile {
  std::string buf;
  std::vector<std::pair<size_t, size_t>> recs;  // [begin, end) of each non-blank data record
  int64_t n = 0;
};

bool read_all(const char* path, std::string& out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out.resize(sz > 0 ? (size_t)sz : 0);
  size_t got = sz > 0 ? std::fread(&out[0], 1, (size_t)sz, f) : 0;
  std::fclose(f);
  return got == out.size();
}

// number of cells of a record (csv dialect "excel": ',' separator, '"' quoting)
int64_t width_of(const char* b, const char* e) {
  int64_t w = 1;
  bool inq = false;
  for (const char* p = b; p < e; p++) {
    if (*p == '"') inq = !inq;
    else if (*p == ',' && !inq) w++;
  }
  return w;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\v' || c == '\f' || c == '\r' || c == '\n'; }

// Python float(token) for a stripped, non-missing token; false if it is not a number
bool parse_float(const char* b, const char* e, double& v) {
  char sbuf[96];
  std::string big;
  size_t n = (size_t)(e - b);
  char* t = sbuf;
  if (n + 1 > sizeof sbuf) { big.resize(n + 1); t = &big[0]; }
  size_t k = 0;
  for (size_t i = 0; i < n; i++) {
    char c = b[i];
    // PEP 515: single underscores between digits
    if (c == '_' && i > 0 && i + 1 < n && std::isdigit((unsigned char)b[i - 1]) && std::isdigit((unsigned char)b[i + 1]))
      continue;
    // strtod also accepts hex floats and "nan(...)", which float() rejects
    if (c == 'x' || c == 'X' || c == '(') return false;
    t[k++] = c;
  }
  if (k == 0) return false;
  t[k] = 0;
  char* end = nullptr;
  v = std::strtod(t, &end);
  return end == t + k;
}

// parse one record into values/mask row r; quoted cells are unquoted first
bool parse_record(const char* b, const char* e, int64_t n, double* vals, uint8_t* mask, std::string& err) {
  std::string q;
  const char* p = b;
  for (int64_t j = 0; j < n; j++) {
    const char* cb = p;
    const char* ce;
    bool quoted = false;
    bool inq = false;
    while (p < e && (inq || *p != ',')) {
      if (*p == '"') { inq = !inq; quoted = true; }
      p++;
    }
    ce = p;
    if (p < e) p++;  // the separator
    if (quoted) {  // unquote: "" inside quotes is a literal quote
      q.clear();
      bool iq = false;
      for (const char* c = cb; c < ce; c++) {
        if (*c == '"') {
          if (iq && c + 1 < ce && c[1] == '"') { q.push_back('"'); c++; }
          else iq = !iq;
        } else {
          q.push_back(*c);
        }
      }
      cb = q.data();
      ce = cb + q.size();
    }
    while (cb < ce && is_space(*cb)) cb++;
    while (ce > cb && is_space(ce[-1])) ce--;
    size_t len = (size_t)(ce - cb);
    bool missing = len == 0 || (len == 3 && (cb[0] | 32) == 'n' && (cb[1] | 32) == 'a' && (cb[2] | 32) == 'n');
    if (missing) {
      vals[j] = NAN;
      mask[j] = 0;
    } else if (parse_float(cb, ce, vals[j])) {
      mask[j] = 1;
    } else {
      err = "could not convert string to float: '" + std::string(cb, ce) + "'";
      return false;
    }
  }
  return true;
}

bool index(const char* path, int has_header, CsvFile& F, std::string& err) {
  if (!read_all(path, F.buf)) { err = std::string(path) + ": cannot read"; return false; }
  const char* s = F.buf.data();
  size_t len = F.buf.size(), pos = 0;
  int64_t idx = 0;
  while (pos < len) {
    // a record ends at a newline outside quotes
    size_t e = pos;
    bool inq = false;
    while (e < len && (inq || (s[e] != '\n' && s[e] != '\r'))) {
      if (s[e] == '"') inq = !inq;
      e++;
    }
    size_t next = e;
    if (next < len && s[next] == '\r') next++;
    if (next < len && s[next] == '\n') next++;
    bool header = has_header && idx == 0;
    idx++;
    if (!header && e > pos) F.recs.push_back({pos, e});
    pos = next;
  }
  if (F.recs.empty()) { err = std::string(path) + ": no data rows"; return false; }
  int64_t wmin = INT64_MAX, wmax = 0;
  std::vector<int64_t> widths;
  for (auto& r : F.recs) {
    int64_t w = width_of(s + r.first, s + r.second);
    widths.push_back(w);
    wmin = std::min(wmin, w);
    wmax = std::max(wmax, w);
  }
  if (wmin != wmax) {
    std::sort(widths.begin(), widths.end());
    widths.erase(std::unique(widths.begin(), widths.end()), widths.end());
    err = std::string(path) + ": ragged rows (widths [";
    for (size_t i = 0; i < widths.size(); i++) err += (i ? ", " : "") + std::to_string(widths[i]);
    err += "])";
    return false;
  }
  F.n = wmax;
  return true;
}

}  // namespace

extern "C" {

int stmf_csv_open(const char* path, int has_header, void** handle, int64_t* m, int64_t* n) {
  if (!path || !handle || !m || !n) return stmf_io_set_error(STMF_ERR_INVALID, "null argument");
  CsvFile* F = new CsvFile;
  std::string err;
  if (!index(path, has_header, *F, err)) {
    delete F;
    return stmf_io_set_error(STMF_ERR_INVALID, err.c_str());
  }
  *handle = F;
  *m = (int64_t)F->recs.size();
  *n = F->n;
  return STMF_OK;
}

int stmf_csv_fill(void* handle, double* values, uint8_t* mask, int threads) {
  if (!handle || !values || !mask) return stmf_io_set_error(STMF_ERR_INVALID, "null argument");
  CsvFile& F = *static_cast<CsvFile*>(handle);
  const int64_t m = (int64_t)F.recs.size(), n = F.n;
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  T = (int)std::max<int64_t>(1, std::min<int64_t>(T, m));
  std::vector<std::string> errs(T);
  // contiguous record ranges per thread
  auto work = [&](int t) {
    int64_t r0 = m * t / T, r1 = m * (t + 1) / T;
    for (int64_t r = r0; r < r1 && errs[t].empty(); r++)
      parse_record(F.buf.data() + F.recs[r].first, F.buf.data() + F.recs[r].second, n, values + r * n,
                   mask + r * n, errs[t]);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; t++) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (!e.empty()) return stmf_io_set_error(STMF_ERR_INVALID, e.c_str());
  return STMF_OK;
}

int stmf_csv_close(void* handle) {
  delete static_cast<CsvFile*>(handle);
  return STMF_OK;
}

}  // extern "C"
