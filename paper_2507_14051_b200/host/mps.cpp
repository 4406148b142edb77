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
#include <zlib.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <set>
#include <sstream>
#include <string>
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
      ++line_;
      if (!text.empty() && text.back() == '\r') text.pop_back();
      if (text.empty() || text[0] == '*') continue;
      const std::vector<std::string> f = tokens(text);
      if (!std::isspace(static_cast<unsigned char>(text[0]))) {
        header(f);
        if (part_ == Part::endata) break;
        continue;
      }
      if (f.empty()) continue;
      body(f);
    }
    if (part_ != Part::endata) throw ParseError("missing ENDATA", line_);
    return finish();
  }

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
    p.matrix = SparseMatrix(m_, n_, std::move(triplets_));
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
  std::unordered_map<std::string, Row> rows_;
  std::unordered_map<std::string, Col> cols_;
  std::vector<double> c_;
  std::set<std::pair<Index, Index>> seen_;
  std::set<Index> obj_seen_;
  std::vector<Triplet> triplets_;
};

}  // namespace

LpProblem parse_mps(std::istream& in, std::vector<std::string>* warnings) {
  return Reader(warnings).read(in);
}

LpProblem parse_mps_file(const std::string& path, std::vector<std::string>* warnings) {
  if (path.size() > 3 && path.compare(path.size() - 3, 3, ".gz") == 0) {
    gzFile gz = gzopen(path.c_str(), "rb");
    if (!gz) throw ParseError("cannot open '" + path + "'", 0);
    std::string data;
    char buf[1 << 16];
    int k = 0;
    while ((k = gzread(gz, buf, sizeof buf)) > 0) data.append(buf, static_cast<size_t>(k));
    gzclose(gz);
    if (k < 0) throw ParseError("gzip read error in '" + path + "'", 0);
    std::istringstream in(data);
    return parse_mps(in, warnings);
  }
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open '" + path + "'", 0);
  return parse_mps(in, warnings);
}

}  // namespace rhpdhg
