// canonical.cpp — the deterministic text form of an LpProblem
// (rhpdhg::to_canonical_text / from_canonical_text, reference
// proj/src/mps.cpp:463-543). The document layout is the reference's, so
// texts written by either library read in the other:
//
//   rhpdhg_lp 1
//   name <name or ->          maximization 0|1
//   rows <m>                  cols <n>
//   offset <v>
//   c / var_lb / var_ub <n values>, con_lb / con_ub <m values>
//   nnz <k>, then k lines "row col value" in CSR order
//
// Values print as %.17g (exact round trip) with inf / -inf spelled out.
#include <cmath>
#include <cstdio>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "rhpdhg/errors.hpp"
#include "rhpdhg/mps.hpp"

namespace rhpdhg {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

void put_number(std::string& out, double v) {
  if (v == kInf) {
    out += "inf";
  } else if (v == -kInf) {
    out += "-inf";
  } else {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    out += buf;
  }
}

void put_vector(std::string& out, const char* key, const std::vector<double>& v) {
  out += key;
  for (double e : v) {
    out += ' ';
    put_number(out, e);
  }
  out += '\n';
}

class TextReader {
 public:
  explicit TextReader(const std::string& text) : in_(text) {}

  void keyword(const char* key) {
    std::string tok;
    if (!(in_ >> tok) || tok != key)
      throw ParseError(std::string("canonical text: expected '") + key + "'", 0);
  }
  template <class T>
  T integer(const char* what) {
    T v{};
    if (!(in_ >> v)) throw ParseError(std::string("canonical text: missing ") + what, 0);
    return v;
  }
  std::string word() {
    std::string tok;
    in_ >> tok;
    return tok;
  }
  double number(const char* what) {
    std::string tok;
    if (!(in_ >> tok)) throw ParseError(std::string("canonical text: missing ") + what, 0);
    if (tok == "inf") return kInf;
    if (tok == "-inf") return -kInf;
    try {
      size_t used = 0;
      const double v = std::stod(tok, &used);
      if (used != tok.size()) throw std::invalid_argument(tok);
      return v;
    } catch (const std::exception&) {
      throw ParseError("canonical text: bad number '" + tok + "'", 0);
    }
  }
  void numbers(const char* key, std::vector<double>& v, Index len) {
    keyword(key);
    v.resize(static_cast<size_t>(len));
    for (double& e : v) e = number(key);
  }

 private:
  std::istringstream in_;
};

}  // namespace

std::string to_canonical_text(const LpProblem& p) {
  std::string out = "rhpdhg_lp 1\n";
  out += "name " + (p.name.empty() ? std::string("-") : p.name) + "\n";
  out += std::string("maximization ") + (p.maximization ? "1" : "0") + "\n";
  out += "rows " + std::to_string(p.num_cons()) + "\n";
  out += "cols " + std::to_string(p.num_vars()) + "\n";
  out += "offset ";
  put_number(out, p.objective_offset);
  out += '\n';
  put_vector(out, "c", p.objective);
  put_vector(out, "var_lb", p.var_lb);
  put_vector(out, "var_ub", p.var_ub);
  put_vector(out, "con_lb", p.con_lb);
  put_vector(out, "con_ub", p.con_ub);
  const auto rp = p.matrix.row_ptr();
  const auto ci = p.matrix.col_index();
  const auto v = p.matrix.csr_values();
  out += "nnz " + std::to_string(p.matrix.nnz()) + "\n";
  for (Index i = 0; i < p.num_cons(); ++i)
    for (Index e = rp[i]; e < rp[i + 1]; ++e) {
      out += std::to_string(i) + ' ' + std::to_string(ci[e]) + ' ';
      put_number(out, v[e]);
      out += '\n';
    }
  return out;
}

LpProblem from_canonical_text(const std::string& text) {
  TextReader r(text);
  std::string head = r.word();
  if (head != "rhpdhg_lp") throw ParseError("canonical text: bad header", 0);
  long version = 0;
  try {
    version = r.integer<long>("version");
  } catch (const ParseError&) {
    throw ParseError("canonical text: bad header", 0);
  }
  if (version != 1) throw ParseError("canonical text: bad header", 0);
  LpProblem p;
  r.keyword("name");
  p.name = r.word();
  if (p.name == "-") p.name.clear();
  r.keyword("maximization");
  p.maximization = r.integer<int>("maximization") != 0;
  r.keyword("rows");
  const Index m = r.integer<Index>("rows");
  r.keyword("cols");
  const Index n = r.integer<Index>("cols");
  if (m < 0 || n < 0) throw ParseError("canonical text: negative dimension", 0);
  r.keyword("offset");
  p.objective_offset = r.number("offset");
  r.numbers("c", p.objective, n);
  r.numbers("var_lb", p.var_lb, n);
  r.numbers("var_ub", p.var_ub, n);
  r.numbers("con_lb", p.con_lb, m);
  r.numbers("con_ub", p.con_ub, m);
  r.keyword("nnz");
  const Index nnz = r.integer<Index>("nnz");
  if (nnz < 0) throw ParseError("canonical text: negative nnz", 0);
  std::vector<Triplet> entries(static_cast<size_t>(nnz));
  for (Triplet& t : entries) {
    try {
      t.row = r.integer<Index>("entry row");
      t.col = r.integer<Index>("entry column");
    } catch (const ParseError&) {
      throw ParseError("canonical text: truncated entries", 0);
    }
    t.value = r.number("entry");
  }
  p.matrix = SparseMatrix(m, n, std::move(entries));
  p.validate();
  return p;
}

}  // namespace rhpdhg
