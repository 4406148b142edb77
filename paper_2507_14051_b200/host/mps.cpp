// mps.cpp — MPS reader behind rhpdhg::parse_mps / parse_mps_file
// (reference: proj/src/mps.cpp:77-435, same accepted language and errors):
//   * sections NAME, OBJSENSE (value inline or on the next line), ROWS,
//     COLUMNS, RHS, RANGES, BOUNDS, ENDATA, in this order; '*' comments;
//     fields are whitespace-separated (free format; fixed-format files
//     without blanks in names parse the same way);
//   * the first N row is the objective, later N rows are dropped with a
//     warning; the objective's RHS entry is -offset;
//   * RANGES: E rows extend up (r >= 0) or down (r < 0); L rows get
//     lb = ub - |r|; G rows get ub = lb + |r|;
//   * BOUNDS LO UP FX FR MI PL BV LI UI (default box [0, +inf); a negative UP
//     without an explicit lower bound makes the lower bound -inf, with a
//     warning); integrality markers and integer bounds are relaxed with a
//     warning;
//   * maximisation negates the objective and offset (LpProblem convention).
//
// Parallel fast path: the text is split into lines
// by all host threads; NAME / OBJSENSE / ROWS and the sections after COLUMNS
// run through the sequential Reader line by line, while the COLUMNS body —
// nearly all of a large file — is tokenized, its row names resolved and its
// numbers parsed by one thread per line chunk; a sequential merge assigns
// column indices in order of first appearance and the matrix is assembled
// directly as CSR (no triplet sort). Anything unusual in the parallel part
// (a malformed line, an unknown row, a non-finite or duplicate entry) makes
// the reader re-parse the whole text with the sequential Reader, so errors,
// their line numbers and warnings are exactly the sequential reader's.
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "rhpdhg/errors.hpp"
#include "rhpdhg/mps.hpp"

namespace rhpdhg {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

enum class Part { none = 0, name, objsense, rows, columns, rhs, ranges, bounds, endata };

std::string upper(std::string s) {
  for (char& ch : s) ch = static_cast<char>(std::toupper(static_cast<unsigned char>(ch)));
  return s;
}

std::vector<std::string> tokens(const std::string& line) {
  std::vector<std::string> out;
  std::istringstream is(line);
  for (std::string t; is >> t;) out.push_back(t);
  return out;
}

// Numbers may carry Fortran 'D' exponents.
double number(const std::string& text, long line) {
  std::string t = text;
  std::replace_if(t.begin(), t.end(), [](char ch) { return ch == 'D' || ch == 'd'; }, 'e');
  const char* b = t.c_str();
  char* e = nullptr;
  const double v = std::strtod(b, &e);
  if (e == b || *e != '\0') throw ParseError("malformed number '" + text + "'", line);
  return v;
}

// string-keyed maps that also accept string_view lookups (no allocation)
struct NameHash {
  using is_transparent = void;
  size_t operator()(std::string_view v) const { return std::hash<std::string_view>{}(v); }
};
template <class V>
using NameMap = std::unordered_map<std::string, V, NameHash, std::equal_to<>>;

struct Row {
  char sense = 'N';
  Index index = -1;  // constraint index, -1 for N rows
  bool objective = false;
  double rhs = 0.0;
  bool ranged = false;
  double range = 0.0;
};

struct Col {
  Index index = 0;
  double lb = 0.0, ub = kInf;
  bool lower_set = false;
};

class Reader {
 public:
  explicit Reader(std::vector<std::string>* warnings) : warnings_(warnings) {}

  LpProblem read(std::istream& in) {
    std::string text;
    while (std::getline(in, text)) {
      if (!line(text, line_ + 1)) break;
    }
    return end();
  }

  // One input line (1-based number `no`); false once ENDATA was read.
  bool line(std::string_view text, long no) {
    line_ = no;
    if (!text.empty() && text.back() == '\r') text.remove_suffix(1);
    if (text.empty() || text[0] == '*') return true;
    const std::vector<std::string> f = tokens(std::string(text));
    if (!std::isspace(static_cast<unsigned char>(text[0]))) {
      header(f);
      return part_ != Part::endata;
    }
    if (f.empty()) return true;
    body(f);
    return true;
  }

  LpProblem end() {
    if (part_ != Part::endata) throw ParseError("missing ENDATA", line_);
    return finish();
  }

  Part part() const { return part_; }

  // ---- hooks of the parallel COLUMNS path (ParallelReader) ----
  const NameMap<Row>& rows() const { return rows_; }
  // Column index of `name` (assigned in order of first appearance).
  Index column_index(std::string_view name) {
    auto it = cols_.find(name);
    if (it == cols_.end()) {
      it = cols_.emplace(std::string(name), Col{}).first;
      it->second.index = n_++;
      c_.push_back(0.0);
      obj_flag_.push_back(0);
    }
    return it->second.index;
  }
  // Objective coefficient of column j; false on a duplicate (sequential
  // reader reports it).
  bool objective_entry(Index j, double v) {
    if (obj_flag_[static_cast<size_t>(j)]) return false;
    obj_flag_[static_cast<size_t>(j)] = 1;
    c_[static_cast<size_t>(j)] = v;
    return true;
  }
  void note_at(long no, const std::string& msg) {
    if (warnings_) warnings_->push_back("line " + std::to_string(no) + ": " + msg);
    int_noted_ = true;
  }
  bool int_noted() const { return int_noted_; }
  void set_matrix(SparseMatrix a) {
    matrix_ = std::move(a);
    have_matrix_ = true;
  }
  Index num_rows() const { return m_; }
  Index num_cols() const { return n_; }

 private:
  void note(const std::string& msg) {
    if (warnings_) warnings_->push_back("line " + std::to_string(line_) + ": " + msg);
  }

  void enter(Part next) {
    if (static_cast<int>(next) <= static_cast<int>(part_))
      throw ParseError("section out of order", line_);
    part_ = next;
  }

  void sense(const std::string& v) {
    const std::string s = upper(v);
    if (s == "MAX" || s == "MAXIMIZE") maximize_ = true;
    else if (s == "MIN" || s == "MINIMIZE") maximize_ = false;
    else throw ParseError("unknown OBJSENSE '" + v + "'", line_);
  }

  void header(const std::vector<std::string>& f) {
    static const std::map<std::string, Part> parts = {
        {"NAME", Part::name},     {"OBJSENSE", Part::objsense}, {"ROWS", Part::rows},
        {"COLUMNS", Part::columns}, {"RHS", Part::rhs},         {"RANGES", Part::ranges},
        {"BOUNDS", Part::bounds}, {"ENDATA", Part::endata}};
    const auto it = parts.find(upper(f[0]));
    if (it == parts.end()) throw ParseError("unknown section '" + f[0] + "'", line_);
    enter(it->second);
    if (it->second == Part::name && f.size() > 1) name_ = f[1];
    if (it->second == Part::objsense && f.size() > 1) sense(f[1]);
  }

  void body(const std::vector<std::string>& f) {
    switch (part_) {
      case Part::objsense: sense(f[0]); break;
      case Part::rows: row(f); break;
      case Part::columns: column(f); break;
      case Part::rhs: pairs(f, [this](Row& r, double v) {
          if (r.sense == 'N') {
            if (r.objective) offset_ = -v;
          } else {
            r.rhs = v;
          }
        }, "RHS"); break;
      case Part::ranges: pairs(f, [this](Row& r, double v) {
          if (r.sense == 'N') throw ParseError("RANGES entry on free row", line_);
          r.ranged = true;
          r.range = v;
        }, "RANGES"); break;
      case Part::bounds: bound(f); break;
      default: throw ParseError("data before any section", line_);
    }
  }

  void row(const std::vector<std::string>& f) {
    if (f.size() != 2) throw ParseError("ROWS entry needs a sense and a name", line_);
    const std::string s = upper(f[0]);
    if (rows_.count(f[1])) throw ParseError("duplicate row '" + f[1] + "'", line_);
    Row r;
    if (s == "N") {
      if (objective_.empty()) {
        objective_ = f[1];
        r.objective = true;
      } else {
        note("extra free row '" + f[1] + "' dropped (only the first N row is the objective)");
      }
    } else if (s == "E" || s == "L" || s == "G") {
      r.sense = s[0];
      r.index = m_++;
    } else {
      throw ParseError("unknown row sense '" + f[0] + "'", line_);
    }
    rows_.emplace(f[1], r);
  }

  static bool quoted(const std::string& t, const char* word) {
    return t == std::string("'") + word + "'" || t == std::string("\"") + word + "\"";
  }

  void column(const std::vector<std::string>& f) {
    if (std::any_of(f.begin(), f.end(), [](const std::string& t) { return quoted(t, "MARKER"); })) {
      for (const std::string& t : f)
        if (quoted(t, "INTORG") && !int_noted_) {
          note("integrality markers ignored; variables relaxed to their continuous box");
          int_noted_ = true;
        }
      return;
    }
    if (f.size() < 3 || f.size() % 2 == 0)
      throw ParseError("COLUMNS entry needs a column name and (row, value) pairs", line_);
    auto [it, fresh] = cols_.try_emplace(f[0]);
    if (fresh) {
      it->second.index = n_++;
      c_.push_back(0.0);
      obj_flag_.push_back(0);
    }
    const Index j = it->second.index;
    for (size_t k = 1; k + 1 < f.size(); k += 2) {
      const auto rit = rows_.find(f[k]);
      if (rit == rows_.end()) throw ParseError("entry references undeclared row '" + f[k] + "'", line_);
      const double v = number(f[k + 1], line_);
      const Row& r = rit->second;
      if (r.sense == 'N') {
        if (!r.objective) continue;
        if (!obj_seen_.insert(j).second)
          throw ParseError("duplicate objective entry for column '" + f[0] + "'", line_);
        c_[static_cast<size_t>(j)] = v;
        continue;
      }
      if (!seen_.insert({r.index, j}).second)
        throw ParseError("duplicate entry for row '" + f[k] + "', column '" + f[0] + "'", line_);
      triplets_.push_back({r.index, j, v});
    }
  }

  void pairs(const std::vector<std::string>& f, const std::function<void(Row&, double)>& apply,
             const char* what) {
    const size_t start = f.size() % 2;  // odd count: leading set name
    if (f.size() - start < 2) throw ParseError("entry needs (row, value) pairs", line_);
    for (size_t k = start; k + 1 < f.size(); k += 2) {
      const auto it = rows_.find(f[k]);
      if (it == rows_.end())
        throw ParseError(std::string(what) + " references undeclared row '" + f[k] + "'", line_);
      apply(it->second, number(f[k + 1], line_));
    }
  }

  void bound(const std::vector<std::string>& f) {
    if (f.size() < 3) throw ParseError("BOUNDS entry too short", line_);
    const std::string t = upper(f[0]);
    const auto it = cols_.find(f[2]);
    if (it == cols_.end()) throw ParseError("BOUNDS references undeclared column '" + f[2] + "'", line_);
    Col& c = it->second;
    const bool valued = t == "LO" || t == "UP" || t == "FX" || t == "LI" || t == "UI";
    double v = 0.0;
    if (valued) {
      if (f.size() < 4) throw ParseError("BOUNDS " + t + " needs a value", line_);
      v = number(f[3], line_);
    }
    auto relaxed = [&] { note("integer bound on '" + f[2] + "' relaxed to its continuous box"); };
    if (t == "LO" || t == "LI") {
      c.lb = v;
      c.lower_set = true;
      if (t == "LI") relaxed();
    } else if (t == "UP" || t == "UI") {
      c.ub = v;
      if (t == "UP" && v < 0.0 && !c.lower_set) {
        c.lb = -kInf;
        note("negative UP bound on '" + f[2] + "' with no lower bound; lower set to -inf");
      }
      if (t == "UI") relaxed();
    } else if (t == "FX") {
      c.lb = c.ub = v;
      c.lower_set = true;
    } else if (t == "FR") {
      c.lb = -kInf;
      c.ub = kInf;
      c.lower_set = true;
    } else if (t == "MI") {
      c.lb = -kInf;
      c.lower_set = true;
    } else if (t == "PL") {
      c.ub = kInf;
    } else if (t == "BV") {
      c.lb = 0.0;
      c.ub = 1.0;
      c.lower_set = true;
      relaxed();
    } else {
      throw ParseError("unknown bound type '" + f[0] + "'", line_);
    }
  }

  LpProblem finish() {
    if (objective_.empty()) throw ParseError("no objective (N) row declared", 0);
    LpProblem p;
    p.name = name_;
    p.matrix = have_matrix_ ? std::move(matrix_) : SparseMatrix(m_, n_, std::move(triplets_));
    p.objective = std::move(c_);
    p.objective_offset = offset_;
    p.con_lb.assign(static_cast<size_t>(m_), 0.0);
    p.con_ub.assign(static_cast<size_t>(m_), 0.0);
    for (const auto& [name, r] : rows_) {
      if (r.index < 0) continue;
      double lo = r.sense == 'L' ? -kInf : r.rhs;
      double hi = r.sense == 'G' ? kInf : r.rhs;
      if (r.ranged) {
        if (r.sense == 'E') (r.range >= 0.0 ? hi : lo) = r.rhs + r.range;
        else if (r.sense == 'L') lo = hi - std::fabs(r.range);
        else hi = lo + std::fabs(r.range);
      }
      p.con_lb[static_cast<size_t>(r.index)] = lo;
      p.con_ub[static_cast<size_t>(r.index)] = hi;
    }
    p.var_lb.assign(static_cast<size_t>(n_), 0.0);
    p.var_ub.assign(static_cast<size_t>(n_), kInf);
    for (const auto& [name, c] : cols_) {
      p.var_lb[static_cast<size_t>(c.index)] = c.lb;
      p.var_ub[static_cast<size_t>(c.index)] = c.ub;
    }
    p.maximization = maximize_;
    if (maximize_) {
      for (double& v : p.objective) v = -v;
      p.objective_offset = -p.objective_offset;
    }
    p.validate();
    return p;
  }

  std::vector<std::string>* warnings_;
  long line_ = 0;
  Part part_ = Part::none;
  std::string name_, objective_;
  bool maximize_ = false, int_noted_ = false;
  double offset_ = 0.0;
  Index m_ = 0, n_ = 0;
  NameMap<Row> rows_;
  NameMap<Col> cols_;
  std::vector<double> c_;
  std::set<std::pair<Index, Index>> seen_;
  std::set<Index> obj_seen_;
  std::vector<Triplet> triplets_;
  std::vector<char> obj_flag_;
  SparseMatrix matrix_;
  bool have_matrix_ = false;
};

// ------------------------------------------------------- parallel reader --
// Signals that the fast path met something only the sequential reader
// handles exactly (it then re-parses the text).
struct Fallback {};

unsigned worker_count() {
  const unsigned t = std::thread::hardware_concurrency();
  return std::max(1u, std::min(t ? t : 1u, 64u));
}

template <class F>
void parallel_for(size_t parts, const F& f) {
  std::vector<std::thread> pool;
  for (size_t p = 1; p < parts; ++p) pool.emplace_back(f, p);
  f(0);
  for (std::thread& t : pool) t.join();
}

// Byte offsets of every line start (plus the end), by all threads.
std::vector<size_t> line_starts(std::string_view text) {
  const size_t T = text.size() < (1u << 20) ? 1 : worker_count();
  std::vector<std::vector<size_t>> part(T);
  parallel_for(T, [&](size_t t) {
    const size_t b = text.size() * t / T, e = text.size() * (t + 1) / T;
    const char* p = text.data();
    for (size_t i = b; i < e; ++i)
      if (p[i] == '\n') part[t].push_back(i + 1);
  });
  std::vector<size_t> out{0};
  size_t total = 1;
  for (auto& v : part) total += v.size();
  out.reserve(total + 1);
  for (auto& v : part) out.insert(out.end(), v.begin(), v.end());
  if (out.back() != text.size()) out.push_back(text.size());
  return out;
}

bool is_space(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f' || ch == '\n'; }

// Whitespace fields of a line as views; at most `cap` (more -> n = cap + 1).
size_t fields(std::string_view line, std::string_view* out, size_t cap) {
  size_t n = 0, i = 0;
  while (i < line.size()) {
    while (i < line.size() && is_space(line[i])) ++i;
    if (i >= line.size()) break;
    const size_t b = i;
    while (i < line.size() && !is_space(line[i])) ++i;
    if (n < cap) out[n] = line.substr(b, i - b);
    ++n;
  }
  return n;
}

// number() of the sequential reader without allocation on the common path
// (Fortran 'D' exponents and forms from_chars rejects take the exact path).
bool fast_number(std::string_view t, double& v) {
  const char* b = t.data();
  const char* e = b + t.size();
  if (t.empty() || *b == '+' || t.find_first_of("Dd") != std::string_view::npos) return false;
  const auto r = std::from_chars(b, e, v);
  return r.ec == std::errc() && r.ptr == e && std::isfinite(v);
}

struct ColEntry {
  Index row;   // constraint index; -1 objective; -2 another N row (ignored)
  double value;
};
struct ColLine {
  std::string_view column;
  uint32_t first, count;  // entries [first, first + count) of the chunk
  long no;                // line number (for the integrality note)
  bool intorg;            // an INTORG marker line
};

LpProblem parse_text(std::string_view text, std::vector<std::string>* warnings) {
  std::vector<std::string> warn;
  Reader rd(&warn);
  const std::vector<size_t> ls = line_starts(text);
  const size_t L = ls.size() - 1;
  auto line_at = [&](size_t i) {
    std::string_view v = text.substr(ls[i], ls[i + 1] - ls[i]);
    if (!v.empty() && v.back() == '\n') v.remove_suffix(1);
    return v;
  };
  bool ended = false;
  size_t i = 0;
  while (i < L && !ended) {
    if (rd.part() == Part::columns) {
      // the COLUMNS body: lines up to the next header, in parallel
      size_t j = i;
      for (; j < L; ++j) {
        const std::string_view v = line_at(j);
        if (!v.empty() && v[0] != '*' && v[0] != '\r' && !is_space(v[0])) break;
      }
      const size_t T = (j - i) < 4096 ? 1 : worker_count();
      std::vector<std::vector<ColLine>> lines(T);
      std::vector<std::vector<ColEntry>> ents(T);
      std::atomic<bool> bad{false};
      const NameMap<Row>& rows = rd.rows();
      parallel_for(T, [&](size_t t) {
        const size_t b = i + (j - i) * t / T, e = i + (j - i) * (t + 1) / T;
        std::string_view f[64];
        for (size_t k = b; k < e && !bad.load(std::memory_order_relaxed); ++k) {
          std::string_view v = line_at(k);
          if (!v.empty() && v.back() == '\r') v.remove_suffix(1);
          if (v.empty() || v[0] == '*') continue;
          const size_t nf = fields(v, f, 64);
          if (nf == 0) continue;
          if (nf > 64) { bad = true; break; }
          bool marker = false, intorg = false;
          for (size_t q = 0; q < nf; ++q) {
            marker |= f[q] == "'MARKER'" || f[q] == "\"MARKER\"";
            intorg |= f[q] == "'INTORG'" || f[q] == "\"INTORG\"";
          }
          if (marker) {
            lines[t].push_back({std::string_view(), 0, 0, static_cast<long>(k + 1), intorg});
            continue;
          }
          if (nf < 3 || nf % 2 == 0) { bad = true; break; }
          ColLine cl{f[0], static_cast<uint32_t>(ents[t].size()), 0, static_cast<long>(k + 1), false};
          for (size_t q = 1; q + 1 < nf; q += 2) {
            const auto it = rows.find(f[q]);
            double val;
            if (it == rows.end() || !fast_number(f[q + 1], val)) { bad = true; break; }
            const Row& r = it->second;
            ents[t].push_back({r.sense == 'N' ? (r.objective ? -1 : -2) : r.index, val});
          }
          if (bad) break;
          cl.count = static_cast<uint32_t>(ents[t].size() - cl.first);
          lines[t].push_back(cl);
        }
      });
      if (bad) throw Fallback{};
      // sequential merge: column indices, objective, per-row counts
      const Index m = rd.num_rows();
      std::vector<Index> rp(static_cast<size_t>(m) + 1, 0);
      std::vector<std::vector<Index>> jcol(T);
      std::string_view prev;
      Index pj = -1;
      for (size_t t = 0; t < T; ++t) {
        jcol[t].resize(ents[t].size());
        for (const ColLine& cl : lines[t]) {
          if (cl.column.empty()) {  // marker line
            if (cl.intorg && !rd.int_noted())
              rd.note_at(cl.no, "integrality markers ignored; variables relaxed to their continuous box");
            continue;
          }
          if (pj < 0 || cl.column != prev) {
            pj = rd.column_index(cl.column);
            prev = cl.column;
          }
          for (uint32_t q = cl.first; q < cl.first + cl.count; ++q) {
            const ColEntry& en = ents[t][q];
            jcol[t][q] = pj;
            if (en.row == -1) {
              if (!rd.objective_entry(pj, en.value)) throw Fallback{};
            } else if (en.row >= 0) {
              ++rp[static_cast<size_t>(en.row) + 1];
            }
          }
        }
      }
      for (Index r = 0; r < m; ++r) rp[r + 1] += rp[r];
      // CSR in line order (stable per row), zeros dropped by from_csr
      std::vector<Index> ci(static_cast<size_t>(rp[m]));
      std::vector<double> cv(static_cast<size_t>(rp[m]));
      std::vector<Index> fill(rp.begin(), rp.end() - 1);
      for (size_t t = 0; t < T; ++t)
        for (size_t q = 0; q < ents[t].size(); ++q) {
          const ColEntry& en = ents[t][q];
          if (en.row < 0) continue;
          const Index s2 = fill[static_cast<size_t>(en.row)]++;
          ci[static_cast<size_t>(s2)] = jcol[t][q];
          cv[static_cast<size_t>(s2)] = en.value;
        }
      // a column that reappears later breaks the ascending order: sort such
      // rows; a repeated (row, column) pair -> the sequential reader's error
      for (Index r = 0; r < m; ++r) {
        const size_t b = static_cast<size_t>(rp[r]), e = static_cast<size_t>(rp[r + 1]);
        bool sorted = true;
        for (size_t q = b + 1; q < e; ++q) sorted &= ci[q] > ci[q - 1];
        if (sorted) continue;
        std::vector<std::pair<Index, double>> row;
        for (size_t q = b; q < e; ++q) row.emplace_back(ci[q], cv[q]);
        std::stable_sort(row.begin(), row.end(),
                         [](const auto& a, const auto& c) { return a.first < c.first; });
        for (size_t q = 1; q < row.size(); ++q)
          if (row[q].first == row[q - 1].first) throw Fallback{};
        for (size_t q = b; q < e; ++q) {
          ci[q] = row[q - b].first;
          cv[q] = row[q - b].second;
        }
      }
      rd.set_matrix(SparseMatrix::from_csr(m, rd.num_cols(), std::move(rp), std::move(ci), std::move(cv)));
      // the header that ends COLUMNS (the section cannot be re-entered)
      if (j < L) ended = !rd.line(line_at(j), static_cast<long>(j + 1));
      i = j + 1;
      continue;
    }
    ended = !rd.line(line_at(i), static_cast<long>(i + 1));
    ++i;
  }
  if (!ended) rd.line(std::string_view(), static_cast<long>(L));  // line_ for "missing ENDATA"
  LpProblem p = rd.end();
  if (warnings) warnings->insert(warnings->end(), warn.begin(), warn.end());
  return p;
}

}  // namespace

namespace {

// The whole text: the parallel reader, or on any irregularity the sequential
// reader (exact errors, line numbers and warnings).
LpProblem parse_all(const std::string& data, std::vector<std::string>* warnings) {
  const char* seq = std::getenv("RHPDHG_MPS_SEQUENTIAL");  // 1: the sequential reader only
  if (!(seq && seq[0] == '1')) try {
    return parse_text(data, warnings);
  } catch (const Fallback&) {
  } catch (const ParseError&) {
  } catch (const InvalidProblemError&) {
  } catch (const UsageError&) {
  }
  std::istringstream in(data);
  return Reader(warnings).read(in);
}

}  // namespace

LpProblem parse_mps(std::istream& in, std::vector<std::string>* warnings) {
  std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return parse_all(data, warnings);
}

LpProblem parse_mps_file(const std::string& path, std::vector<std::string>* warnings) {
  std::string data;
  if (path.size() > 3 && path.compare(path.size() - 3, 3, ".gz") == 0) {
    gzFile gz = gzopen(path.c_str(), "rb");
    if (!gz) throw ParseError("cannot open '" + path + "'", 0);
    gzbuffer(gz, 1 << 20);
    std::vector<char> buf(1 << 22);
    int k = 0;
    while ((k = gzread(gz, buf.data(), static_cast<unsigned>(buf.size()))) > 0)
      data.append(buf.data(), static_cast<size_t>(k));
    gzclose(gz);
    if (k < 0) throw ParseError("gzip read error in '" + path + "'", 0);
  } else {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseError("cannot open '" + path + "'", 0);
    in.seekg(0, std::ios::end);
    const std::streamoff size = in.tellg();
    in.seekg(0, std::ios::beg);
    data.resize(static_cast<size_t>(std::max<std::streamoff>(size, 0)));
    if (size > 0) in.read(data.data(), size);
  }
  return parse_all(data, warnings);
}

}  // namespace rhpdhg
