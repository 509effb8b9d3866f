// ps_matio.cu -- delimited matrix files (host code, C ABI).
//
// Native replacement of the reference's matio.write_matrix / read_matrix
// (pkg/src/pairstat/matio.py:40-125), SURVEY section 8(f) item 2.  The text format is
// byte-identical to the reference writer:
//   header  = sep.join([""] + col_ids)
//   row i   = sep.join([row_id] + [format_value(v) for v in values[i]])
//   lines joined by "\n" plus a final "\n"
// with format_value = f"{v:.17g}" (matio.py:30-32): C's "%.17g" gives the same
// digits (both correctly rounded, same exponent rules); NaN of either sign is
// the literal "nan" as in Python.  Rows are formatted by all host cores in
// blocks and written in order.
//
// The reader mirrors read_matrix: Python str.splitlines() line boundaries
// (\n \r \r\n \v \f \x1c \x1d \x1e and the UTF-8 forms of U+0085, U+2028,
// U+2029), empty lines skipped, header split on the delimiter, ragged-row and
// malformed-cell errors in file order.  Cells are parsed with the grammar of
// Python's float() (PEP 515 underscores, inf / infinity / nan in any case,
// surrounding whitespace); conversion by strtod (correctly rounded, like
// CPython).  A cell holding any non-ASCII byte is flagged for the Python
// wrapper, which parses it with float() itself (Unicode digits / spaces).
#include "ps_internal.cuh"
#include <omp.h>
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {

// f"{v:.17g}" into buf; returns length
inline int format17(double v, char* buf) {
  if (std::isnan(v)) {
    std::memcpy(buf, "nan", 3);
    return 3;
  }
  return std::snprintf(buf, 32, "%.17g", v);
}

inline bool ascii_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// digitpart ::= digit (["_"] digit)*  -> appends digits to out; returns chars consumed (0: no match)
size_t digitpart(const char* s, size_t n, size_t i, std::string& out) {
  const size_t i0 = i;
  if (i >= n || !is_digit(s[i])) return 0;
  out.push_back(s[i++]);
  while (i < n) {
    if (is_digit(s[i])) {
      out.push_back(s[i++]);
    } else if (s[i] == '_' && i + 1 < n && is_digit(s[i + 1])) {
      out.push_back(s[i + 1]);
      i += 2;
    } else {
      break;
    }
  }
  return i - i0;
}

bool ieq(const char* a, size_t n, const char* lit) {
  const size_t m = std::strlen(lit);
  if (n != m) return false;
  for (size_t k = 0; k < n; ++k)
    if ((char)std::tolower((unsigned char)a[k]) != lit[k]) return false;
  return true;
}

// Python float() on an ASCII cell. 0 ok, 1 malformed.
int parse_float(const char* s, size_t n, double* out) {
  size_t b = 0, e = n;
  while (b < e && ascii_space((unsigned char)s[b])) ++b;
  while (e > b && ascii_space((unsigned char)s[e - 1])) --e;
  if (b == e) return 1;
  std::string t;
  size_t i = b;
  if (s[i] == '+' || s[i] == '-') t.push_back(s[i++]);
  const char* rest = s + i;
  const size_t rn = e - i;
  if (ieq(rest, rn, "inf") || ieq(rest, rn, "infinity") || ieq(rest, rn, "nan")) {
    t.append(rest, rn);
    *out = std::strtod(t.c_str(), nullptr);
    return 0;
  }
  // number ::= [digitpart] "." digitpart | digitpart ["."]
  const size_t d1 = digitpart(s, e, i, t);
  i += d1;
  bool have = d1 > 0;
  if (i < e && s[i] == '.') {
    t.push_back('.');
    ++i;
    const size_t d2 = digitpart(s, e, i, t);
    i += d2;
    if (d1 == 0 && d2 == 0) return 1;
    have = true;
  }
  if (!have) return 1;
  if (i < e && (s[i] == 'e' || s[i] == 'E')) {
    t.push_back('e');
    ++i;
    if (i < e && (s[i] == '+' || s[i] == '-')) t.push_back(s[i++]);
    const size_t d3 = digitpart(s, e, i, t);
    if (d3 == 0) return 1;
    i += d3;
  }
  if (i != e) return 1;
  errno = 0;
  *out = std::strtod(t.c_str(), nullptr);  // overflow -> +-inf, underflow -> 0 / subnormal, as CPython
  return 0;
}

// Python str.splitlines() boundaries; returns [begin, end) of each line
void split_lines(const char* d, size_t n, std::vector<std::pair<size_t, size_t>>& lines) {
  size_t start = 0, i = 0;
  while (i < n) {
    const unsigned char c = (unsigned char)d[i];
    size_t blen = 0;
    if (c == '\n' || c == '\v' || c == '\f' || c == 0x1c || c == 0x1d || c == 0x1e) blen = 1;
    else if (c == '\r') blen = (i + 1 < n && d[i + 1] == '\n') ? 2 : 1;
    else if (c == 0xC2 && i + 1 < n && (unsigned char)d[i + 1] == 0x85) blen = 2;
    else if (c == 0xE2 && i + 2 < n && (unsigned char)d[i + 1] == 0x80 &&
             ((unsigned char)d[i + 2] == 0xA8 || (unsigned char)d[i + 2] == 0xA9)) blen = 3;
    if (blen) {
      lines.emplace_back(start, i);
      i += blen;
      start = i;
    } else {
      ++i;
    }
  }
  if (start < n) lines.emplace_back(start, n);
}

}  // namespace

extern "C" {

int ps_write_matrix(const char* path, const double* values, int64_t rows, int64_t cols,
                    const char* const* row_ids, const char* const* col_ids, char delim) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return ps_fail(PS_ERR_IO, std::string("cannot open ") + path + ": " + std::strerror(errno));
  std::string header;
  for (int64_t j = 0; j < cols; ++j) {
    header.push_back(delim);
    if (col_ids) header += col_ids[j];
    else header += "s" + std::to_string(j);
  }
  header.push_back('\n');
  bool ok = std::fwrite(header.data(), 1, header.size(), f) == header.size();
  const int64_t block = 256;
  std::vector<std::string> out((size_t)block);
  for (int64_t r0 = 0; r0 < rows && ok; r0 += block) {
    const int64_t r1 = std::min(rows, r0 + block);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t r = r0; r < r1; ++r) {
      std::string& s = out[(size_t)(r - r0)];
      s.clear();
      if (row_ids) s += row_ids[r];
      else s += "f" + std::to_string(r);
      char buf[40];
      const double* v = values + r * cols;
      for (int64_t j = 0; j < cols; ++j) {
        s.push_back(delim);
        s.append(buf, (size_t)format17(v[j], buf));
      }
      s.push_back('\n');
    }
    for (int64_t r = r0; r < r1 && ok; ++r) {
      const std::string& s = out[(size_t)(r - r0)];
      ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
    }
  }
  if (std::fclose(f) != 0) ok = false;
  if (!ok) return ps_fail(PS_ERR_IO, std::string("write failed: ") + path);
  return PS_OK;
}

// Result of ps_read_matrix (free with ps_matrix_file_free).
//   error: 0 ok; 1 empty file; 2 ragged row (err_row, err_count); 3 malformed cell
//   (err_row, err_col, err_cell = its bytes).  Cells with non-ASCII bytes are listed in
//   fallback (flat value index) for the caller to parse; their value slot holds 0.
struct ps_matrix_file_impl {
  std::vector<double> values;
  std::string row_ids, col_ids;  // '\0'-separated
  std::vector<int64_t> fallback;
  std::string err_cell;
};

int ps_read_matrix(const char* path, char delim, ps_matrix_file* out) {
  std::memset(out, 0, sizeof(*out));
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    out->os_errno = errno;
    return ps_fail(PS_ERR_IO, std::string("cannot open ") + path + ": " + std::strerror(errno));
  }
  std::string data;
  {
    char buf[1 << 16];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof(buf), f)) > 0) data.append(buf, k);
    std::fclose(f);
  }
  auto* impl = new ps_matrix_file_impl();
  out->impl = impl;
  std::vector<std::pair<size_t, size_t>> lines;
  split_lines(data.data(), data.size(), lines);
  if (lines.empty()) {
    out->error = 1;
    return PS_OK;
  }
  // header
  {
    const size_t b = lines[0].first, e = lines[0].second;
    size_t p = b;
    int64_t n = 0;
    bool first = true;
    for (size_t i = b; i <= e; ++i) {
      if (i == e || data[i] == delim) {
        if (!first) {
          impl->col_ids.append(data, p, i - p);
          impl->col_ids.push_back('\0');
          ++n;
        }
        first = false;
        p = i + 1;
      }
    }
    out->n_cols = n;
  }
  const int64_t nc = out->n_cols;
  // data rows: non-empty lines after the header, each with its 1-based line number
  std::vector<int64_t> li;
  for (size_t k = 1; k < lines.size(); ++k)
    if (lines[k].second > lines[k].first) li.push_back((int64_t)k);
  const int64_t nr = (int64_t)li.size();
  impl->values.assign((size_t)(nr * nc), 0.0);
  std::vector<int> rerr((size_t)nr, 0);          // 0 ok, 2 ragged, 3 malformed
  std::vector<int64_t> rinfo((size_t)nr, 0);     // count (ragged) or column (malformed)
  std::vector<std::string> rid((size_t)nr);
  std::vector<std::vector<int64_t>> rfb((size_t)nr);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < nr; ++r) {
    const size_t b = lines[(size_t)li[(size_t)r]].first, e = lines[(size_t)li[(size_t)r]].second;
    // count cells first (ragged check precedes parsing, as in read_matrix)
    int64_t cells = 1;
    for (size_t i = b; i < e; ++i) cells += data[i] == delim;
    if (cells != nc + 1) {
      rerr[(size_t)r] = 2;
      rinfo[(size_t)r] = cells - 1;
      continue;
    }
    size_t p = b;
    int64_t c = -1;
    for (size_t i = b; i <= e; ++i) {
      if (i == e || data[i] == delim) {
        if (c < 0) {
          rid[(size_t)r].assign(data, p, i - p);
        } else {
          const char* cs = data.data() + p;
          const size_t cn = i - p;
          bool ascii = true;
          for (size_t q = 0; q < cn; ++q) ascii &= (unsigned char)cs[q] < 0x80;
          double v = 0.0;
          if (!ascii) {
            rfb[(size_t)r].push_back(r * nc + c);
          } else if (parse_float(cs, cn, &v)) {
            rerr[(size_t)r] = 3;
            rinfo[(size_t)r] = c + 1;
            break;
          }
          impl->values[(size_t)(r * nc + c)] = v;
        }
        ++c;
        p = i + 1;
      }
    }
  }
  for (int64_t r = 0; r < nr; ++r) {
    if (rerr[(size_t)r]) {
      out->error = rerr[(size_t)r];
      out->err_row = li[(size_t)r] + 1;  // 1-based line number, header = 1
      if (rerr[(size_t)r] == 2) {
        out->err_count = rinfo[(size_t)r];
      } else {
        out->err_col = rinfo[(size_t)r];
        // the offending cell's bytes
        const size_t b = lines[(size_t)li[(size_t)r]].first, e = lines[(size_t)li[(size_t)r]].second;
        int64_t c = -1;
        size_t p = b;
        for (size_t i = b; i <= e; ++i)
          if (i == e || data[i] == delim) {
            if (c == out->err_col - 1) {
              impl->err_cell.assign(data, p, i - p);
              break;
            }
            ++c;
            p = i + 1;
          }
        out->err_cell = impl->err_cell.data();
        out->err_cell_len = (int64_t)impl->err_cell.size();
      }
      // non-ASCII cells before the error (earlier rows; earlier columns of a
      // malformed row) are parsed by the caller first: one of them may be the
      // first bad cell in file order
      impl->fallback.insert(impl->fallback.end(), rfb[(size_t)r].begin(), rfb[(size_t)r].end());
      out->n_rows = r;
      out->fallback = impl->fallback.data();
      out->n_fallback = (int64_t)impl->fallback.size();
      return PS_OK;
    }
    impl->row_ids += rid[(size_t)r];
    impl->row_ids.push_back('\0');
    impl->fallback.insert(impl->fallback.end(), rfb[(size_t)r].begin(), rfb[(size_t)r].end());
  }
  out->n_rows = nr;
  out->values = impl->values.data();
  out->row_ids = impl->row_ids.data();
  out->row_ids_len = (int64_t)impl->row_ids.size();
  out->col_ids = impl->col_ids.data();
  out->col_ids_len = (int64_t)impl->col_ids.size();
  out->fallback = impl->fallback.data();
  out->n_fallback = (int64_t)impl->fallback.size();
  out->err_cell = impl->err_cell.data();
  out->err_cell_len = (int64_t)impl->err_cell.size();
  return PS_OK;
}

void ps_matrix_file_free(ps_matrix_file* f) {
  if (!f) return;
  delete static_cast<ps_matrix_file_impl*>(f->impl);
  std::memset(f, 0, sizeof(*f));
}

}  // extern "C"
