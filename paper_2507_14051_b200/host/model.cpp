// model.cpp — host data types of the rhpdhg API: SparseMatrix containers,
// LpProblem validation, Iterate, small vector utilities, spmv_counter.
// The matrix products route to the GPU (no CPU fallback).
#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>
#include <mutex>
#include <string>

#include "device.hpp"
#include "rhpdhg/errors.hpp"
#include "rhpdhg/lp_problem.hpp"
#include "rhpdhg/solver.hpp"
#include "rhpdhg/sparse_matrix.hpp"

namespace rhpdhg {

namespace spmv_counter {
namespace {
std::atomic<std::uint64_t> g_products{0};
}
std::uint64_t value() { return g_products.load(std::memory_order_relaxed); }
void reset() { g_products.store(0, std::memory_order_relaxed); }
void add(std::uint64_t n) { g_products.fetch_add(n, std::memory_order_relaxed); }
}  // namespace spmv_counter

// sparse_matrix.cpp:20-65 semantics: bounds -> UsageError, non-finite ->
// InvalidProblemError, zeros dropped, duplicates -> InvalidProblemError.
SparseMatrix::SparseMatrix(Index rows, Index cols, std::vector<Triplet> entries)
    : rows_(rows), cols_(cols) {
  if (rows < 0 || cols < 0) throw UsageError("matrix dimensions must be nonnegative");
  for (const Triplet& t : entries) {
    if (t.row < 0 || t.row >= rows || t.col < 0 || t.col >= cols)
      throw UsageError("matrix entry (" + std::to_string(t.row) + "," + std::to_string(t.col) +
                       ") out of bounds");
    if (!std::isfinite(t.value))
      throw InvalidProblemError("matrix entry (" + std::to_string(t.row) + "," +
                                std::to_string(t.col) + ") is not finite");
  }
  std::erase_if(entries, [](const Triplet& t) { return t.value == 0.0; });
  std::sort(entries.begin(), entries.end(), [](const Triplet& a, const Triplet& b) {
    return a.row < b.row || (a.row == b.row && a.col < b.col);
  });
  row_ptr_.assign(static_cast<size_t>(rows) + 1, 0);
  col_idx_.reserve(entries.size());
  val_csr_.reserve(entries.size());
  for (size_t k = 0; k < entries.size(); ++k) {
    if (k > 0 && entries[k].row == entries[k - 1].row && entries[k].col == entries[k - 1].col)
      throw InvalidProblemError("duplicate matrix entry (" + std::to_string(entries[k].row) +
                                "," + std::to_string(entries[k].col) + ")");
    row_ptr_[static_cast<size_t>(entries[k].row) + 1]++;
    col_idx_.push_back(entries[k].col);
    val_csr_.push_back(entries[k].value);
  }
  for (Index i = 0; i < rows; ++i) row_ptr_[i + 1] += row_ptr_[i];
}

SparseMatrix SparseMatrix::from_csr(Index rows, Index cols, std::vector<Index> row_ptr,
                                    std::vector<Index> col_index, std::vector<double> values) {
  if (rows < 0 || cols < 0) throw UsageError("matrix dimensions must be nonnegative");
  if (static_cast<Index>(row_ptr.size()) != rows + 1 || col_index.size() != values.size())
    throw UsageError("from_csr: array sizes do not match");
  SparseMatrix a;
  a.rows_ = rows;
  a.cols_ = cols;
  bool zeros = false;
  for (Index i = 0; i < rows; ++i) {
    Index prev = -1;
    if (row_ptr[i + 1] < row_ptr[i]) throw UsageError("from_csr: row_ptr not monotone");
    for (Index e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const Index j = col_index[e];
      const double v = values[e];
      if (j < 0 || j >= cols)
        throw UsageError("matrix entry (" + std::to_string(i) + "," + std::to_string(j) +
                         ") out of bounds");
      if (!std::isfinite(v))
        throw InvalidProblemError("matrix entry (" + std::to_string(i) + "," +
                                  std::to_string(j) + ") is not finite");
      if (j <= prev)
        throw InvalidProblemError("duplicate or unsorted matrix entry (" + std::to_string(i) +
                                  "," + std::to_string(j) + ")");
      prev = j;
      zeros |= v == 0.0;
    }
  }
  if (row_ptr[0] == 0 && static_cast<size_t>(row_ptr[rows]) == values.size() && !zeros) {
    a.row_ptr_ = std::move(row_ptr);  // already canonical: take the arrays
    a.col_idx_ = std::move(col_index);
    a.val_csr_ = std::move(values);
    return a;
  }
  a.row_ptr_.assign(static_cast<size_t>(rows) + 1, 0);
  a.col_idx_.reserve(values.size());
  a.val_csr_.reserve(values.size());
  for (Index i = 0; i < rows; ++i) {
    for (Index e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      if (values[e] == 0.0) continue;
      a.col_idx_.push_back(col_index[e]);
      a.val_csr_.push_back(values[e]);
    }
    a.row_ptr_[i + 1] = static_cast<Index>(a.col_idx_.size());
  }
  return a;
}

const SparseMatrix::Csc& SparseMatrix::csc() const {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!csc_) {
    auto c = std::make_shared<Csc>();
    c->col_ptr.assign(static_cast<size_t>(cols_) + 1, 0);
    for (Index j : col_idx_) c->col_ptr[static_cast<size_t>(j) + 1]++;
    for (Index j = 0; j < cols_; ++j) c->col_ptr[j + 1] += c->col_ptr[j];
    c->row_idx.resize(col_idx_.size());
    c->val.resize(col_idx_.size());
    std::vector<Index> fill(c->col_ptr.begin(), c->col_ptr.end() - 1);
    for (Index i = 0; i < rows_; ++i)
      for (Index e = row_ptr_[i]; e < row_ptr_[i + 1]; ++e) {
        const Index s = fill[col_idx_[e]]++;
        c->row_idx[s] = i;
        c->val[s] = val_csr_[e];
      }
    csc_ = std::move(c);
  }
  return *csc_;
}

namespace detail {

DeviceCache& device_cache(const SparseMatrix& a) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!a.dev_) a.dev_ = std::make_shared<DeviceCache>();
  return *a.dev_;
}

rhp_ctx* product_context(const SparseMatrix& a, std::unique_lock<std::mutex>& lock) {
  DeviceCache& cache = device_cache(a);
  lock = std::unique_lock<std::mutex>(cache.mu);
  if (!cache.dev) {
    rhpdhg_lp_view v{};
    v.num_cons = a.rows();
    v.num_vars = a.cols();
    v.nnz = a.nnz();
    v.row_ptr = a.row_ptr().data();
    v.col_index = a.col_index().data();
    v.values = a.csr_values().data();
    std::vector<double> zn(static_cast<size_t>(a.cols()), 0.0), zm(static_cast<size_t>(a.rows()), 0.0);
    v.objective = zn.data();
    v.var_lb = zn.data();
    v.var_ub = zn.data();
    v.con_lb = zm.data();
    v.con_ub = zm.data();
    const DeviceOptions& d = default_device_options();
    auto dev = std::make_unique<Device>(v, options(d.device, false, 1));
    // a scaled matrix's CSC values are scaled from its own CSC values
    // (sparse_matrix.cpp:101-114), not copies of the CSR ones
    if (const std::vector<double>* csc = own_csc_values(a); csc && a.nnz() > 0)
      ok(rhp_set_csc_values(dev->get(), csc->data(), 0), "rhp_set_csc_values");
    cache.dev = std::move(dev);
  }
  return cache.dev->get();
}

const std::vector<double>* own_csc_values(const SparseMatrix& a) {
  return (a.csc_ && a.csc_->own_values) ? &a.csc_->val : nullptr;
}

SparseMatrix with_values(const SparseMatrix& pattern, std::vector<double> csr_values,
                         std::vector<double> csc_values) {
  if (csr_values.size() != pattern.val_csr_.size() || csc_values.size() != pattern.val_csr_.size())
    throw UsageError("with_values: value count does not match the pattern");
  SparseMatrix r;
  r.rows_ = pattern.rows_;
  r.cols_ = pattern.cols_;
  r.row_ptr_ = pattern.row_ptr_;
  r.col_idx_ = pattern.col_idx_;
  r.val_csr_ = std::move(csr_values);
  const SparseMatrix::Csc& c = pattern.csc();
  auto rc = std::make_shared<SparseMatrix::Csc>();
  rc->col_ptr = c.col_ptr;
  rc->row_idx = c.row_idx;
  rc->val = std::move(csc_values);
  rc->own_values = true;
  r.csc_ = std::move(rc);
  return r;
}

}  // namespace detail

namespace {
void device_product(const SparseMatrix& a, bool transpose, std::span<const double> in,
                    std::span<double> out) {
  std::unique_lock<std::mutex> lock;
  rhp_ctx* ctx = detail::product_context(a, lock);
  detail::ok(rhp_spmv(ctx, transpose ? 1 : 0, in.data(), out.data()), "rhp_spmv");
}
}  // namespace

void SparseMatrix::multiply(std::span<const double> x, std::span<double> out) const {
  if (static_cast<Index>(x.size()) != cols_ || static_cast<Index>(out.size()) != rows_)
    throw UsageError("multiply: size mismatch");
  spmv_counter::add(1);
  if (rows_ == 0) return;
  device_product(*this, false, x, out);
}

void SparseMatrix::multiply_transpose(std::span<const double> y, std::span<double> out) const {
  if (static_cast<Index>(y.size()) != rows_ || static_cast<Index>(out.size()) != cols_)
    throw UsageError("multiply_transpose: size mismatch");
  spmv_counter::add(1);
  if (cols_ == 0) return;
  device_product(*this, true, y, out);
}

std::vector<double> SparseMatrix::multiply(const std::vector<double>& x) const {
  std::vector<double> out(static_cast<size_t>(rows_));
  multiply(std::span<const double>(x), std::span<double>(out));
  return out;
}

std::vector<double> SparseMatrix::multiply_transpose(const std::vector<double>& y) const {
  std::vector<double> out(static_cast<size_t>(cols_));
  multiply_transpose(std::span<const double>(y), std::span<double>(out));
  return out;
}

SparseMatrix SparseMatrix::scaled(std::span<const double> row_scale,
                                  std::span<const double> col_scale) const {
  if (static_cast<Index>(row_scale.size()) != rows_ ||
      static_cast<Index>(col_scale.size()) != cols_)
    throw UsageError("scaled: scale vector size mismatch");
  SparseMatrix r(*this);
  for (Index i = 0; i < rows_; ++i)
    for (Index e = row_ptr_[i]; e < row_ptr_[i + 1]; ++e)
      r.val_csr_[e] = row_scale[i] * val_csr_[e] * col_scale[col_idx_[e]];
  const Csc& c = csc();
  auto rc = std::make_shared<Csc>(c);
  for (Index j = 0; j < cols_; ++j)
    for (Index e = c.col_ptr[j]; e < c.col_ptr[j + 1]; ++e)
      rc->val[e] = col_scale[j] * c.val[e] * row_scale[c.row_idx[e]];
  rc->own_values = true;
  r.csc_ = std::move(rc);
  r.dev_.reset();  // new values: its own product context
  return r;
}

void SparseMatrix::max_abs(std::vector<double>& row_out, std::vector<double>& col_out) const {
  row_out.assign(static_cast<size_t>(rows_), 0.0);
  col_out.assign(static_cast<size_t>(cols_), 0.0);
  for (Index i = 0; i < rows_; ++i)
    for (Index e = row_ptr_[i]; e < row_ptr_[i + 1]; ++e) {
      const double a = std::fabs(val_csr_[e]);
      row_out[i] = std::max(row_out[i], a);
      col_out[col_idx_[e]] = std::max(col_out[col_idx_[e]], a);
    }
}

void SparseMatrix::one_norms(std::vector<double>& row_out, std::vector<double>& col_out) const {
  row_out.assign(static_cast<size_t>(rows_), 0.0);
  col_out.assign(static_cast<size_t>(cols_), 0.0);
  for (Index i = 0; i < rows_; ++i)
    for (Index e = row_ptr_[i]; e < row_ptr_[i + 1]; ++e) {
      row_out[i] += std::fabs(val_csr_[e]);
      col_out[col_idx_[e]] += std::fabs(val_csr_[e]);
    }
}

std::vector<Triplet> SparseMatrix::to_triplets() const {
  std::vector<Triplet> t;
  t.reserve(val_csr_.size());
  for (Index i = 0; i < rows_; ++i)
    for (Index e = row_ptr_[i]; e < row_ptr_[i + 1]; ++e) t.push_back({i, col_idx_[e], val_csr_[e]});
  return t;
}

bool SparseMatrix::same_pattern(const SparseMatrix& o) const {
  return rows_ == o.rows_ && cols_ == o.cols_ && row_ptr_ == o.row_ptr_ && col_idx_ == o.col_idx_;
}

bool operator==(const SparseMatrix& a, const SparseMatrix& b) {
  return a.same_pattern(b) && a.val_csr_ == b.val_csr_;
}

// ---------------------------------------------------------------- LpProblem --
namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

void check_bounds(std::span<const double> lb, std::span<const double> ub, const char* what) {
  for (size_t i = 0; i < lb.size(); ++i) {
    if (std::isnan(lb[i]) || std::isnan(ub[i]))
      throw InvalidProblemError(std::string(what) + " bound " + std::to_string(i) + " is NaN");
    if (lb[i] > ub[i])
      throw InvalidProblemError(std::string(what) + " bounds crossed at index " + std::to_string(i));
    if (lb[i] == kInf || ub[i] == -kInf)
      throw InvalidProblemError(std::string(what) + " bound " + std::to_string(i) +
                                " has the wrong-signed infinity");
  }
}
}  // namespace

// lp_problem.cpp:30-46
void LpProblem::validate() const {
  const Index n = matrix.cols(), m = matrix.rows();
  if (static_cast<Index>(objective.size()) != n)
    throw InvalidProblemError("objective length does not match matrix columns");
  if (static_cast<Index>(var_lb.size()) != n || static_cast<Index>(var_ub.size()) != n)
    throw InvalidProblemError("variable bound length does not match matrix columns");
  if (static_cast<Index>(con_lb.size()) != m || static_cast<Index>(con_ub.size()) != m)
    throw InvalidProblemError("constraint bound length does not match matrix rows");
  for (size_t j = 0; j < objective.size(); ++j)
    if (!std::isfinite(objective[j]))
      throw InvalidProblemError("objective coefficient " + std::to_string(j) + " is not finite");
  if (!std::isfinite(objective_offset)) throw InvalidProblemError("objective offset is not finite");
  check_bounds(var_lb, var_ub, "variable");
  check_bounds(con_lb, con_ub, "constraint");
}

void detail::validate_vectors(const rhpdhg_lp_view& v) {
  const size_t n = static_cast<size_t>(v.num_vars), m = static_cast<size_t>(v.num_cons);
  for (size_t j = 0; j < n; ++j)
    if (!std::isfinite(v.objective[j]))
      throw InvalidProblemError("objective coefficient " + std::to_string(j) + " is not finite");
  if (!std::isfinite(v.objective_offset)) throw InvalidProblemError("objective offset is not finite");
  check_bounds(std::span<const double>(v.var_lb, n), std::span<const double>(v.var_ub, n), "variable");
  check_bounds(std::span<const double>(v.con_lb, m), std::span<const double>(v.con_ub, m), "constraint");
}

bool operator==(const LpProblem& a, const LpProblem& b) {
  return a.name == b.name && a.objective == b.objective &&
         a.objective_offset == b.objective_offset && a.matrix == b.matrix &&
         a.var_lb == b.var_lb && a.var_ub == b.var_ub && a.con_lb == b.con_lb &&
         a.con_ub == b.con_ub && a.maximization == b.maximization;
}

void project_box_inplace(std::span<double> v, std::span<const double> lb,
                         std::span<const double> ub) {
  if (v.size() != lb.size() || v.size() != ub.size()) throw UsageError("project_box: length mismatch");
  for (size_t i = 0; i < v.size(); ++i) {
    if (lb[i] > ub[i]) throw InvalidProblemError("project_box: crossed bounds");
    v[i] = std::min(std::max(v[i], lb[i]), ub[i]);
  }
}

std::vector<double> project_box(std::span<const double> v, std::span<const double> lb,
                                std::span<const double> ub) {
  std::vector<double> out(v.begin(), v.end());
  project_box_inplace(out, lb, ub);
  return out;
}

double p_support(std::span<const double> y, std::span<const double> lb,
                 std::span<const double> ub) {
  if (y.size() != lb.size() || y.size() != ub.size()) throw UsageError("p_support: length mismatch");
  double total = 0.0;
  for (size_t i = 0; i < y.size(); ++i) {
    const double pos = std::max(y[i], 0.0), neg = std::max(-y[i], 0.0);
    const double up = pos == 0.0 ? 0.0 : ub[i] * pos;
    const double lo = neg == 0.0 ? 0.0 : lb[i] * neg;
    if (up == kInf || lo == -kInf) return kInf;
    total += up - lo;
  }
  return total;
}

std::vector<double> project_dual_cone(std::span<const double> s, const LpProblem& p) {
  if (static_cast<Index>(s.size()) != p.num_cons()) throw UsageError("project_dual_cone: length mismatch");
  std::vector<double> out(s.size());
  for (size_t i = 0; i < s.size(); ++i) out[i] = std::min(std::max(s[i], -p.con_ub[i]), -p.con_lb[i]);
  return out;
}

Iterate Iterate::zeros(const LpProblem& p) {
  Iterate z;
  z.x.assign(static_cast<size_t>(p.num_vars()), 0.0);
  z.aty.assign(static_cast<size_t>(p.num_vars()), 0.0);
  z.y.assign(static_cast<size_t>(p.num_cons()), 0.0);
  z.ax.assign(static_cast<size_t>(p.num_cons()), 0.0);
  z.ax_valid = z.aty_valid = true;
  return z;
}

}  // namespace rhpdhg
