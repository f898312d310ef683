// io.cpp — Matrix Market / FROSTT readers and writers (stam/io.h).
#include "stam/io.h"

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>

#include "stam/error.h"

namespace stam {
namespace {

std::string readAll(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) fail(ErrorCode::Io, "cannot open " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

[[noreturn]] void bad(const std::string& path, int64_t line, const std::string& what) {
  fail(ErrorCode::Io, path + ":" + std::to_string(line) + ": " + what);
}

// Line cursor over the file contents.
struct Lines {
  const char* p;
  const char* end;
  int64_t no = 0;
  bool next(const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    no++;
    if (e > b && e[-1] == '\r') e--;
    return true;
  }
};

bool blank(const char* b, const char* e) {
  for (; b < e; b++)
    if (*b != ' ' && *b != '\t') return false;
  return true;
}

// Parses whitespace-separated numbers of one line (no allocation per token).
struct Tokens {
  const char* p;
  const char* e;
  bool integer(int64_t& v) {
    while (p < e && (*p == ' ' || *p == '\t')) p++;
    if (p >= e) return false;
    char* q;
    errno = 0;
    v = std::strtoll(p, &q, 10);
    if (q == p || errno) return false;
    p = q;
    return true;
  }
  bool real(double& v) {
    while (p < e && (*p == ' ' || *p == '\t')) p++;
    if (p >= e) return false;
    char* q;
    v = std::strtod(p, &q);
    if (q == p) return false;
    p = q;
    return true;
  }
  bool done() {
    while (p < e && (*p == ' ' || *p == '\t')) p++;
    return p >= e;
  }
};

// Sorted, duplicate-summed COO (coordinates row-major: nnz x order) into
// {dense, compressed...} levels.
TensorStorage assemble(std::vector<int64_t> dims, std::vector<int64_t>& coords,
                       std::vector<double>& vals) {
  const int order = (int)dims.size();
  const int64_t n = (int64_t)vals.size();
  std::vector<int64_t> perm((size_t)n);
  std::iota(perm.begin(), perm.end(), 0);
  // stable: duplicates keep file order, so their sum is the file-order sum
  std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) {
    return std::lexicographical_compare(coords.begin() + a * order, coords.begin() + (a + 1) * order,
                                        coords.begin() + b * order, coords.begin() + (b + 1) * order);
  });
  std::vector<int64_t> uc;  // unique coordinates, row-major
  std::vector<double> uv;
  uc.reserve((size_t)n * order);
  uv.reserve((size_t)n);
  for (int64_t t = 0; t < n; t++) {
    const int64_t* c = coords.data() + perm[(size_t)t] * order;
    if (!uv.empty() && std::equal(c, c + order, uc.end() - order)) {
      uv.back() += vals[(size_t)perm[(size_t)t]];
    } else {
      uc.insert(uc.end(), c, c + order);
      uv.push_back(vals[(size_t)perm[(size_t)t]]);
    }
  }
  const int64_t m = (int64_t)uv.size();
  std::vector<ModeFormat> mf{dense()};
  for (int d = 1; d < order; d++) mf.push_back(compressed());
  std::vector<TensorStorage::Level> levels((size_t)order);
  levels[0].format = dense();
  // level d >= 1: one position per distinct prefix (c0..cd); parents are the
  // distinct prefixes (c0..c_{d-1}) (level 0 dense: parent d0 = coordinate)
  std::vector<int64_t> parent_of((size_t)m);  // index of the entry's level-(d-1) node
  for (int64_t t = 0; t < m; t++) parent_of[(size_t)t] = uc[(size_t)(t * order)];
  int64_t nparents = dims[0];
  for (int d = 1; d < order; d++) {
    auto& L = levels[(size_t)d];
    L.format = compressed();
    L.pos.assign((size_t)nparents + 1, 0);
    std::vector<int64_t> node((size_t)m);
    int64_t nodes = 0;
    for (int64_t t = 0; t < m; t++) {
      const int64_t* c = uc.data() + t * order;
      const bool same = t > 0 && std::equal(c, c + d + 1, uc.data() + (t - 1) * order);
      if (!same) {
        L.idx.push_back(c[d]);
        L.pos[(size_t)parent_of[(size_t)t] + 1]++;
        nodes++;
      }
      node[(size_t)t] = nodes - 1;
    }
    for (int64_t q = 0; q < nparents; q++) L.pos[(size_t)q + 1] += L.pos[(size_t)q];
    parent_of.swap(node);
    nparents = nodes;
  }
  TensorFormat fmt(mf);
  return TensorStorage::fromArrays(std::move(dims), fmt, std::move(levels), std::move(uv), true);
}

}  // namespace

TensorStorage loadMatrixMarket(const std::string& path) {
  const std::string text = readAll(path);
  Lines L{text.data(), text.data() + text.size()};
  const char *b, *e;
  if (!L.next(b, e)) bad(path, 1, "empty file");
  std::string header(b, e);
  std::string lower = header;
  std::transform(lower.begin(), lower.end(), lower.begin(), ::tolower);
  std::istringstream hs(lower);
  std::string banner, object, format, field, symmetry;
  hs >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%matrixmarket" || object != "matrix")
    bad(path, 1, "not a Matrix Market matrix header: '" + header + "'");
  if (format != "coordinate") bad(path, 1, "only the coordinate format is supported");
  const bool pattern = field == "pattern";
  if (!pattern && field != "real" && field != "integer" && field != "double")
    bad(path, 1, "unsupported field '" + field + "'");
  const bool sym = symmetry == "symmetric", skew = symmetry == "skew-symmetric";
  if (!sym && !skew && symmetry != "general") bad(path, 1, "unsupported symmetry '" + symmetry + "'");
  int64_t rows = -1, cols = -1, nnz = -1;
  while (L.next(b, e)) {
    if (b < e && *b == '%') continue;
    if (blank(b, e)) continue;
    Tokens t{b, e};
    if (!t.integer(rows) || !t.integer(cols) || !t.integer(nnz) || !t.done() || rows < 0 ||
        cols < 0 || nnz < 0)
      bad(path, L.no, "malformed size line");
    break;
  }
  if (nnz < 0) bad(path, L.no, "missing size line");
  std::vector<int64_t> coords;
  std::vector<double> vals;
  coords.reserve((size_t)nnz * ((sym || skew) ? 4 : 2));
  vals.reserve((size_t)nnz * ((sym || skew) ? 2 : 1));
  int64_t seen = 0;
  while (seen < nnz && L.next(b, e)) {
    if (b < e && *b == '%') continue;
    if (blank(b, e)) continue;
    Tokens t{b, e};
    int64_t i, j;
    double v = 1.0;
    if (!t.integer(i) || !t.integer(j)) bad(path, L.no, "malformed entry");
    if (!pattern && !t.real(v)) bad(path, L.no, "missing value");
    if (!t.done()) bad(path, L.no, "trailing characters in entry");
    if (i < 1 || i > rows || j < 1 || j > cols)
      fail(ErrorCode::OutOfRange, path + ":" + std::to_string(L.no) + ": coordinate out of range");
    coords.push_back(i - 1);
    coords.push_back(j - 1);
    vals.push_back(v);
    if ((sym || skew) && i != j) {
      coords.push_back(j - 1);
      coords.push_back(i - 1);
      vals.push_back(skew ? -v : v);
    }
    seen++;
  }
  if (seen < nnz) bad(path, L.no, "fewer entries than the size line announces");
  return assemble({rows, cols}, coords, vals);
}

TensorStorage loadTns(const std::string& path, const std::vector<int64_t>& dims_in) {
  const std::string text = readAll(path);
  Lines L{text.data(), text.data() + text.size()};
  const char *b, *e;
  int order = -1;
  std::vector<int64_t> coords;
  std::vector<double> vals;
  std::vector<int64_t> maxc;
  std::vector<double> tok;
  while (L.next(b, e)) {
    if (blank(b, e) || *b == '#') continue;
    Tokens t{b, e};
    if (order < 0) {
      // order = tokens - 1 on the first entry line
      tok.clear();
      double v;
      Tokens c = t;
      while (c.real(v)) tok.push_back(v);
      if (!c.done() || tok.size() < 2) bad(path, L.no, "malformed entry");
      order = (int)tok.size() - 1;
      maxc.assign((size_t)order, 0);
    }
    for (int d = 0; d < order; d++) {
      int64_t x;
      if (!t.integer(x)) bad(path, L.no, "malformed coordinate");
      if (x < 1) fail(ErrorCode::OutOfRange, path + ":" + std::to_string(L.no) +
                                                 ": coordinates are 1-based");
      coords.push_back(x - 1);
      maxc[(size_t)d] = std::max(maxc[(size_t)d], x);
    }
    double v;
    if (!t.real(v) || !t.done()) bad(path, L.no, "malformed value");
    vals.push_back(v);
  }
  if (order < 0) bad(path, L.no, "no entries (the order of an empty .tns file is unknown)");
  std::vector<int64_t> dims = dims_in.empty() ? maxc : dims_in;
  if ((int)dims.size() != order) fail(ErrorCode::DimensionMismatch, "loadTns: dims order mismatch");
  for (int d = 0; d < order; d++)
    if (maxc[(size_t)d] > dims[(size_t)d])
      fail(ErrorCode::OutOfRange, "loadTns: coordinate beyond the given dimension");
  return assemble(dims, coords, vals);
}

void store(const std::string& path, const TensorStorage& t) {
  const bool mtx = path.size() >= 4 && path.compare(path.size() - 4, 4, ".mtx") == 0;
  if (mtx && t.order() != 2) fail(ErrorCode::DimensionMismatch, "store: .mtx needs order 2");
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) fail(ErrorCode::Io, "cannot write " + path);
  const auto entries = t.entries();
  if (mtx) {
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%lld %lld %lld\n", (long long)t.dimensions()[0],
                 (long long)t.dimensions()[1], (long long)entries.size());
  }
  for (const auto& [c, v] : entries) {
    for (size_t d = 0; d < c.size(); d++) std::fprintf(f, "%lld ", (long long)(c[d] + 1));
    std::fprintf(f, "%.17g\n", v);
  }
  if (std::fclose(f) != 0) fail(ErrorCode::Io, "write failed: " + path);
}

}  // namespace stam
