// Native CSV ingestion (reference pkg/src/binboost/dataset.py:31-100, which
// parses with Python's csv module and float()): the file is read once,
// records are delimited by one sequential quote-aware pass (excel dialect:
// ',' delimiter, '"' quoting with "" escapes, \n, \r\n or \r line ends, empty
// records skipped), then the records are parsed by a pool of threads.  A cell
// is accepted iff Python's float() accepts it (optional surrounding
// whitespace, sign, digits with single '_' separators, fraction, exponent,
// inf / infinity / nan in any case), and converted by the C library's
// correctly rounded strtod, so values are the ones float() returns.
// The first error in record order (cell count, unparsable cell, non-finite
// value in a column that must be finite) is reported with its coordinates;
// the Python layer formats the reference's messages.
#include <algorithm>
#include <cerrno>
#include <clocale>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fastbdt_b200.h"

namespace bb {
void set_error(const std::string& msg);
}

namespace {

struct Record {
  int64_t no;    // 1-based record number (the header is record 1)
  size_t begin;  // byte range [begin, end) in the buffer (line terminator excluded)
  size_t end;
};

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }

// Python float() grammar; on success writes the value
bool parse_float(const char* s, size_t n, double* out) {
  size_t a = 0, b = n;
  while (a < b && is_space(s[a])) ++a;
  while (b > a && is_space(s[b - 1])) --b;
  if (a == b) return false;
  char tb[128];
  std::string big;  // cells longer than the stack buffer
  char* t = tb;
  if (b - a + 2 > sizeof(tb)) {
    big.resize(b - a + 2);
    t = &big[0];
  }
  size_t tn = 0;
  size_t i = a;
  bool neg = false;
  if (s[i] == '+' || s[i] == '-') {
    neg = s[i] == '-';
    t[tn++] = s[i];
    ++i;
  }
  if (i < b && (s[i] == 'i' || s[i] == 'I' || s[i] == 'n' || s[i] == 'N')) {  // special values
    const size_t m = b - i;
    auto eq = [&](const char* w) {
      if (std::strlen(w) != m) return false;
      for (size_t k = 0; k < m; ++k)
        if (std::tolower((unsigned char)s[i + k]) != w[k]) return false;
      return true;
    };
    if (eq("inf") || eq("infinity")) {
      *out = neg ? -std::numeric_limits<double>::infinity() : std::numeric_limits<double>::infinity();
      return true;
    }
    if (eq("nan")) {
      *out = neg ? -std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::quiet_NaN();
      return true;
    }
    return false;
  }
  // digits ('_' only between two digits)
  auto digits = [&](size_t& k) {
    size_t cnt = 0;
    while (k < b) {
      const char c = s[k];
      if (c >= '0' && c <= '9') {
        t[tn++] = c;
        ++k;
        ++cnt;
      } else if (c == '_' && cnt > 0 && k + 1 < b && s[k + 1] >= '0' && s[k + 1] <= '9') {
        ++k;
      } else {
        break;
      }
    }
    return cnt;
  };
  size_t nd = digits(i);
  if (i < b && s[i] == '.') {
    t[tn++] = '.';
    ++i;
    nd += digits(i);
  }
  if (nd == 0) return false;
  if (i < b && (s[i] == 'e' || s[i] == 'E')) {
    t[tn++] = 'e';
    ++i;
    if (i < b && (s[i] == '+' || s[i] == '-')) t[tn++] = s[i++];
    if (digits(i) == 0) return false;
  }
  if (i != b) return false;
  t[tn] = 0;
  char* endp = nullptr;
  const double v = std::strtod(t, &endp);
  if (endp != t + tn) return false;
  *out = v;  // overflow gives +-inf like float("1e999")
  return true;
}

// A record's cells as (pointer, length): unquoted cells point into the
// buffer, quoted cells are unescaped into `store` (csv excel dialect: a
// quote opens a quoted section only at the start of a cell, "" is a quote,
// text after the closing quote is appended).
struct Cell {
  const char* p;
  size_t n;
};
void split_cells(const char* buf, size_t begin, size_t end, std::vector<Cell>& cells, std::string& store) {
  cells.clear();
  store.clear();
  store.reserve(end - begin);
  size_t i = begin;
  while (true) {
    // one cell starting at i
    if (i < end && buf[i] == '"') {
      const size_t s0 = store.size();
      ++i;
      bool inq = true;
      while (i < end) {
        const char c = buf[i];
        if (inq) {
          if (c == '"') {
            if (i + 1 < end && buf[i + 1] == '"') {
              store.push_back('"');
              i += 2;
              continue;
            }
            inq = false;
            ++i;
            continue;
          }
          store.push_back(c);
          ++i;
        } else {
          if (c == ',') break;
          store.push_back(c);
          ++i;
        }
      }
      cells.push_back(Cell{nullptr, store.size() - s0});  // offset fixed below (store may reallocate)
      cells.back().p = reinterpret_cast<const char*>(s0);
    } else {
      const size_t c0 = i;
      while (i < end && buf[i] != ',') ++i;
      cells.push_back(Cell{buf + c0, i - c0});
    }
    if (i >= end) break;
    ++i;  // the comma
    if (i == end) {  // trailing comma: one more empty cell
      cells.push_back(Cell{buf + end, 0});
      break;
    }
  }
  // quoted cells: offsets into `store` -> pointers
  for (Cell& c : cells)
    if (!(c.p >= buf + begin && c.p <= buf + end)) c.p = store.data() + reinterpret_cast<size_t>(c.p);
}

}  // namespace

struct bb_csv {
  std::string path;
  std::vector<char> data;
  std::vector<Record> recs;  // data records (non-empty), in order
  std::vector<std::string> header;
  bool has_header = false;   // false: empty file
  int64_t err_row = 0;       // first error: record number
  int32_t err_kind = 0;      // 1 cell count, 2 not a number, 3 non-finite
  int32_t err_col = -1;
  int32_t err_cells = 0;
  std::string err_cell;
  double err_value = 0.0;
};

extern "C" {

int bb_csv_open(const char* path, bb_csv** out) {
  try {
    if (!path || !out) {
      bb::set_error("null argument");
      return BB_EINVAL;
    }
    auto* h = new bb_csv();
    h->path = path;
    FILE* f = std::fopen(path, "rb");
    if (!f) {
      bb::set_error(std::string("cannot open ") + path + ": " + std::strerror(errno));
      delete h;
      return BB_EINVAL;
    }
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    h->data.resize(sz > 0 ? (size_t)sz : 0);
    if (sz > 0 && std::fread(h->data.data(), 1, (size_t)sz, f) != (size_t)sz) {
      std::fclose(f);
      bb::set_error(std::string("cannot read ") + path);
      delete h;
      return BB_EINVAL;
    }
    std::fclose(f);
    const char* buf = h->data.data();
    const size_t n = h->data.size();
    // fast path (no quote, no CR anywhere): records are the lines, split by
    // a pool of threads with memchr; the record number is the line number
    if (n > (1u << 20) && !std::memchr(buf, '"', n) && !std::memchr(buf, '\r', n)) {
      const char* nl = static_cast<const char*>(std::memchr(buf, '\n', n));
      const size_t hend = nl ? (size_t)(nl - buf) : n;
      std::vector<Cell> cells;
      std::string store;
      if (hend > 0) {
        split_cells(buf, 0, hend, cells, store);
        for (const Cell& c : cells) h->header.emplace_back(c.p, c.n);
      }
      h->has_header = true;
      const size_t body = nl ? hend + 1 : n;
      const int T = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
      std::vector<std::vector<Record>> part(T);
      std::vector<int64_t> lines(T, 0);
      auto scan = [&](int t) {
        size_t a = body + (n - body) * t / T, b = body + (n - body) * (t + 1) / T;
        if (a > body && buf[a - 1] != '\n') {  // the line containing a belongs to the previous range
          const char* q = static_cast<const char*>(std::memchr(buf + a, '\n', n - a));
          a = q ? (size_t)(q - buf) + 1 : n;
        }
        int64_t cnt = 0;
        while (a < b) {
          const char* q = static_cast<const char*>(std::memchr(buf + a, '\n', n - a));
          const size_t e = q ? (size_t)(q - buf) : n;
          if (e > a) part[t].push_back(Record{cnt, a, e});
          ++cnt;
          a = e + 1;
        }
        lines[t] = cnt;
      };
      std::vector<std::thread> th;
      for (int t = 1; t < T; ++t) th.emplace_back(scan, t);
      scan(0);
      for (auto& x : th) x.join();
      int64_t base = 2;  // the first data line is record 2
      for (int t = 0; t < T; ++t) {
        for (Record r : part[t]) {
          r.no += base;
          h->recs.push_back(r);
        }
        base += lines[t];
      }
      *out = h;
      return BB_OK;
    }
    // records: one sequential quote-aware pass
    size_t i = 0, start = 0;
    int64_t no = 0;
    bool inq = false, at_start = true;
    bool have_header = false;
    auto emit = [&](size_t e) {
      ++no;
      if (!have_header) {
        have_header = true;
        std::vector<Cell> cells;
        std::string store;
        h->header.clear();
        if (e > start) {
          split_cells(buf, start, e, cells, store);
          for (const Cell& c : cells) h->header.emplace_back(c.p, c.n);
        }
        h->has_header = true;
      } else if (e > start) {
        h->recs.push_back(Record{no, start, e});
      }
    };
    while (i < n) {
      const char c = buf[i];
      if (inq) {
        if (c == '"') {
          if (i + 1 < n && buf[i + 1] == '"') {
            i += 2;
            continue;
          }
          inq = false;
        }
        ++i;
        continue;
      }
      if (c == '"' && at_start) {
        inq = true;
        at_start = false;
        ++i;
        continue;
      }
      if (c == ',') {
        at_start = true;
        ++i;
        continue;
      }
      if (c == '\n' || c == '\r') {
        emit(i);
        if (c == '\r' && i + 1 < n && buf[i + 1] == '\n') ++i;
        ++i;
        start = i;
        at_start = true;
        continue;
      }
      at_start = false;
      ++i;
    }
    if (start < n || !have_header) {
      if (start < n || (n > 0 && !have_header)) emit(n);
    }
    *out = h;
    return BB_OK;
  } catch (const std::exception& e) {
    bb::set_error(e.what());
    return BB_ESTATE;
  }
}

/* header cells, or -1 for an empty file (no record at all) */
int32_t bb_csv_n_header(const bb_csv* h) { return (h && h->has_header) ? (int32_t)h->header.size() : -1; }
int64_t bb_csv_n_records(const bb_csv* h) { return h ? (int64_t)h->recs.size() : -1; }

/* header cell j (raw, not stripped); its length in *len */
const char* bb_csv_header(const bb_csv* h, int32_t j, int64_t* len) {
  if (!h || j < 0 || j >= (int32_t)h->header.size()) return nullptr;
  if (len) *len = (int64_t)h->header[j].size();
  return h->header[j].data();
}

int bb_csv_parse(bb_csv* h, const int32_t* cols, int32_t n_cols, int32_t finite_col, int32_t n_threads,
                 double* out) {
  try {
    if (!h || (n_cols > 0 && (!cols || !out))) {
      bb::set_error("null argument");
      return BB_EINVAL;
    }
    const int64_t R = (int64_t)h->recs.size();
    const int32_t ncell = (int32_t)h->header.size();
    int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<int64_t>(T, std::max<int64_t>(1, R / 4096));
    struct Err {
      int64_t rec = -1;
      int32_t kind = 0, col = -1, cells = 0;
      std::string cell;
      double value = 0.0;
    };
    std::vector<Err> errs(T);
    auto work = [&](int t) {
      const int64_t r0 = R * t / T, r1 = R * (t + 1) / T;
      std::vector<Cell> cells;
      std::string store;
      Err& E = errs[t];
      for (int64_t r = r0; r < r1; ++r) {
        const Record& rc = h->recs[r];
        split_cells(h->data.data(), rc.begin, rc.end, cells, store);
        if ((int32_t)cells.size() != ncell) {
          E.rec = r;
          E.kind = 1;
          E.cells = (int32_t)cells.size();
          return;
        }
        for (int32_t k = 0; k < n_cols; ++k) {
          const Cell& c = cells[cols[k]];
          double v;
          if (!parse_float(c.p, c.n, &v)) {
            E.rec = r;
            E.kind = 2;
            E.col = cols[k];
            E.cell.assign(c.p, c.n);
            return;
          }
          out[r * n_cols + k] = v;
          if (cols[k] == finite_col && !std::isfinite(v)) {
            // reported after the row's cells all parsed (reference order)
            bool later_bad = false;
            for (int32_t k2 = k + 1; k2 < n_cols && !later_bad; ++k2) {
              double v2;
              const Cell& c2 = cells[cols[k2]];
              if (!parse_float(c2.p, c2.n, &v2)) {
                E.rec = r;
                E.kind = 2;
                E.col = cols[k2];
                E.cell.assign(c2.p, c2.n);
                later_bad = true;
              }
            }
            if (later_bad) return;
            E.rec = r;
            E.kind = 3;
            E.col = cols[k];
            E.value = v;
            return;
          }
        }
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (const Err& E : errs) {
      if (E.rec < 0) continue;
      h->err_row = h->recs[E.rec].no;
      h->err_kind = E.kind;
      h->err_col = E.col;
      h->err_cells = E.cells;
      h->err_cell = E.cell;
      h->err_value = E.value;
      bb::set_error("csv parse error");
      return BB_EINVAL;
    }
    return BB_OK;
  } catch (const std::exception& e) {
    bb::set_error(e.what());
    return BB_ESTATE;
  }
}

/* the first error of bb_csv_parse: record number, kind (1 cell count,
 * 2 not a number, 3 non-finite), column, cell count, raw cell text, value */
int bb_csv_error(const bb_csv* h, int64_t* row, int32_t* kind, int32_t* col, int32_t* cells, const char** cell,
                 int64_t* cell_len, double* value) {
  if (!h) return BB_EINVAL;
  *row = h->err_row;
  *kind = h->err_kind;
  *col = h->err_col;
  *cells = h->err_cells;
  *cell = h->err_cell.data();
  *cell_len = (int64_t)h->err_cell.size();
  *value = h->err_value;
  return BB_OK;
}

int bb_csv_close(bb_csv* h) {
  delete h;
  return BB_OK;
}

}  // extern "C"
