// bench.cpp — directory benchmark with SGM10 scoring (reference
// proj/src/bench.cpp:25-318: same size classes, time-limit scoring, record
// order, summary rows and JSON schema).
//
// Execution is GPU-first: with workers <= 1 the instances solve one after
// another in this process; with workers > 1 a pool of host threads solves
// that many instances at once, worker w on GPU w % device_count, each solve
// with its own device context and stream (on an 8-GPU box, 8 instances in
// flight with one GPU each, so per-instance times stay clean). When
// self_exe is set, workers > 1 instead forks one `<self_exe> solve <mps>
// --config <file> --time-limit <s> --out <report>` process per instance and
// reads its report (the reference's worker protocol, bench.cpp:107-167).
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <mutex>
#include <sstream>
#include <thread>

#include "rhpdhg/bench.hpp"
#include "rhpdhg/errors.hpp"
#include "rhpdhg/mps.hpp"
#include "rhpdhg/report.hpp"
#include "rhpdhg/solver.hpp"
#include "rhpdhg_cuda.h"

namespace rhpdhg {

namespace fs = std::filesystem;

const char* to_string(SizeClass c) {
  switch (c) {
    case SizeClass::small: return "small";
    case SizeClass::medium: return "medium";
    case SizeClass::large: return "large";
  }
  return "unknown";
}

SizeClass classify_by_nnz(Index nnz) {
  if (nnz > 10'000'000) return SizeClass::large;
  if (nnz > 1'000'000) return SizeClass::medium;
  return SizeClass::small;
}

double sgm10(std::span<const double> times, double shift) {
  if (times.empty()) throw UsageError("sgm10: empty time list");
  double log_sum = 0.0;
  for (double t : times) {
    if (t < 0.0) throw UsageError("sgm10: negative time");
    log_sum += std::log(t + shift);
  }
  return std::exp(log_sum / static_cast<double>(times.size())) - shift;
}

namespace {

struct Instance {
  std::string path, name, error;
  Index nnz = 0;
  SizeClass size_class = SizeClass::small;
  double time_limit = 3600.0;
};

BenchmarkRecord base_record(const Instance& in) {
  BenchmarkRecord r;
  r.instance = in.name;
  r.nonzeros = in.nnz;
  r.size_class = in.size_class;
  r.scored_seconds = in.time_limit;
  return r;
}

BenchmarkRecord error_record(const Instance& in, const std::string& why) {
  BenchmarkRecord r = base_record(in);
  r.status = "error";
  r.error = why;
  return r;
}

BenchmarkRecord summary_record(const Instance& in, const SolutionSummary& s) {
  BenchmarkRecord r = base_record(in);
  r.status = s.status;
  r.solve_seconds = s.wall_time_seconds;
  if (s.status == "optimal") r.scored_seconds = s.wall_time_seconds;
  r.iterations = s.iterations;
  r.restart_count = s.restart_count;
  r.residuals = s.residuals;
  return r;
}

BenchmarkRecord solve_here(const Instance& in, const SolverConfig& base, int device) {
  try {
    const LpProblem p = parse_mps_file(in.path);
    SolverConfig cfg = base;
    cfg.time_limit_seconds = in.time_limit;
    DeviceOptions dopt = default_device_options();
    dopt.device = device;
    const SolutionReport rep = solve(p, cfg, dopt);
    SolutionSummary s;
    s.status = to_string(rep.status);
    s.objective = rep.objective;
    s.iterations = rep.iterations;
    s.restart_count = rep.restart_count;
    s.wall_time_seconds = rep.wall_time_seconds;
    s.residuals = rep.residuals;
    return summary_record(in, s);
  } catch (const std::exception& e) {
    return error_record(in, e.what());
  }
}

std::string number_text(double v) {
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  std::ostringstream os;
  os.precision(17);
  os << v;
  return os.str();
}

// The reference's process-per-instance protocol (bench.cpp:107-167).
void run_processes(const std::vector<Instance>& jobs, const SolverConfig& cfg,
                   const BenchmarkOptions& opts, std::ostream* log,
                   std::vector<BenchmarkRecord>& out) {
  const fs::path tmp = fs::temp_directory_path() / ("rhpdhg_bench_" + std::to_string(::getpid()));
  fs::create_directories(tmp);
  const std::string conf = (tmp / "worker.conf").string();
  {
    std::ofstream f(conf);
    for (const auto& [k, v] : cfg.key_values()) f << k << ' ' << v << "\n";
  }
  auto report_of = [&](size_t i) { return (tmp / ("bench_" + std::to_string(i) + ".sol")).string(); };
  std::vector<std::pair<pid_t, size_t>> running;
  size_t next = 0;
  while (next < jobs.size() || !running.empty()) {
    while (next < jobs.size() && running.size() < static_cast<size_t>(opts.workers)) {
      const Instance& in = jobs[next];
      if (!in.error.empty()) {
        out[next] = error_record(in, in.error);
        ++next;
        continue;
      }
      if (log) *log << "solving " << in.name << " ...\n";
      std::vector<std::string> args = {opts.self_exe, "solve", in.path, "--config", conf,
                                       "--time-limit", number_text(in.time_limit), "--out",
                                       report_of(next)};
      const pid_t pid = ::fork();
      if (pid < 0) throw std::runtime_error("fork failed");
      if (pid == 0) {
        std::vector<char*> argv;
        for (std::string& a : args) argv.push_back(a.data());
        argv.push_back(nullptr);
        ::execv(opts.self_exe.c_str(), argv.data());
        std::perror("execv");
        ::_exit(127);
      }
      running.emplace_back(pid, next++);
    }
    if (running.empty()) break;
    int status = 0;
    const pid_t pid = ::waitpid(-1, &status, 0);
    auto it = std::find_if(running.begin(), running.end(), [pid](const auto& p) { return p.first == pid; });
    if (it == running.end()) continue;
    const size_t i = it->second;
    running.erase(it);
    if (WIFEXITED(status) && (WEXITSTATUS(status) == 0 || WEXITSTATUS(status) == 2)) {
      std::ifstream f(report_of(i));
      out[i] = f ? summary_record(jobs[i], read_solution_summary(f))
                 : error_record(jobs[i], "worker produced no report");
    } else if (WIFEXITED(status)) {
      out[i] = error_record(jobs[i], "worker exited with code " + std::to_string(WEXITSTATUS(status)));
    } else {
      out[i] = error_record(jobs[i], "worker terminated abnormally");
    }
  }
  std::error_code ec;
  fs::remove_all(tmp, ec);
}

BenchmarkSummaryRow summary_row(const std::string& group, const std::vector<const BenchmarkRecord*>& recs,
                                double shift) {
  BenchmarkSummaryRow row;
  row.group = group;
  std::vector<double> times;
  for (const BenchmarkRecord* r : recs) {
    ++row.count;
    if (r->status == "optimal") ++row.solved;
    times.push_back(r->scored_seconds);
  }
  row.sgm10 = times.empty() ? 0.0 : sgm10(times, shift);
  return row;
}

}  // namespace

BenchmarkReport run_benchmark(const std::string& dir, const SolverConfig& cfg,
                              const BenchmarkOptions& opts, std::ostream* log) {
  if (!fs::is_directory(dir)) throw UsageError("'" + dir + "' is not a directory");
  std::vector<Instance> jobs;
  for (const auto& entry : fs::directory_iterator(dir)) {
    if (!entry.is_regular_file()) continue;
    const std::string file = entry.path().filename().string();
    if (!(file.ends_with(".mps") || file.ends_with(".mps.gz"))) continue;
    Instance in;
    in.path = entry.path().string();
    in.name = file.substr(0, file.find(".mps"));
    try {
      in.nnz = parse_mps_file(in.path).matrix.nnz();
    } catch (const std::exception& e) {
      in.error = e.what();
    }
    in.size_class = classify_by_nnz(in.nnz);
    in.time_limit = in.size_class == SizeClass::large ? opts.large_limit_seconds
                                                      : opts.small_limit_seconds;
    jobs.push_back(std::move(in));
  }
  std::sort(jobs.begin(), jobs.end(), [](const Instance& a, const Instance& b) { return a.name < b.name; });
  BenchmarkReport report;
  if (jobs.empty()) {
    if (log) *log << "warning: no .mps/.mps.gz instances found in '" << dir << "'\n";
    return report;
  }
  report.records.resize(jobs.size());
  const int base_device = default_device_options().device;
  if (opts.workers <= 1) {
    for (size_t i = 0; i < jobs.size(); ++i) {
      if (log) *log << "solving " << jobs[i].name << " ...\n";
      report.records[i] = jobs[i].error.empty() ? solve_here(jobs[i], cfg, base_device)
                                                : error_record(jobs[i], jobs[i].error);
    }
  } else if (!opts.self_exe.empty()) {
    run_processes(jobs, cfg, opts, log, report.records);
  } else {
    int devices = 1;
    if (rhp_device_count(&devices) != RHPDHG_OK || devices < 1) devices = 1;
    std::atomic<size_t> next{0};
    std::mutex log_mu;
    auto worker = [&](int w) {
      const int device = (base_device + w) % devices;
      for (size_t i = next++; i < jobs.size(); i = next++) {
        if (!jobs[i].error.empty()) {
          report.records[i] = error_record(jobs[i], jobs[i].error);
          continue;
        }
        if (log) {
          std::lock_guard<std::mutex> lock(log_mu);
          *log << "solving " << jobs[i].name << " on GPU " << device << " ...\n";
        }
        report.records[i] = solve_here(jobs[i], cfg, device);
      }
    };
    std::vector<std::thread> pool;
    for (int w = 0; w < opts.workers; ++w) pool.emplace_back(worker, w);
    for (std::thread& t : pool) t.join();
  }
  for (SizeClass c : {SizeClass::small, SizeClass::medium, SizeClass::large}) {
    std::vector<const BenchmarkRecord*> recs;
    for (const BenchmarkRecord& r : report.records)
      if (r.size_class == c) recs.push_back(&r);
    report.summary.push_back(summary_row(to_string(c), recs, opts.shift));
  }
  std::vector<const BenchmarkRecord*> all;
  for (const BenchmarkRecord& r : report.records) all.push_back(&r);
  report.summary.push_back(summary_row("total", all, opts.shift));
  return report;
}

void write_benchmark_table(const BenchmarkReport& report, std::ostream& out) {
  out << "instance                         class   status           time(s)      iters restarts\n";
  char buf[200];
  for (const BenchmarkRecord& r : report.records) {
    std::snprintf(buf, sizeof buf, "%-32s %-7s %-16s %9.2f %10ld %8ld\n", r.instance.c_str(),
                  to_string(r.size_class), r.status.c_str(), r.solve_seconds, r.iterations,
                  r.restart_count);
    out << buf;
  }
  out << "\n  group    count  solved      SGM10\n";
  for (const BenchmarkSummaryRow& row : report.summary) {
    std::snprintf(buf, sizeof buf, "  %-8s %5ld %7ld %10.3f\n", row.group.c_str(), row.count,
                  row.solved, row.sgm10);
    out << buf;
  }
}

namespace {

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char ch : s) {
    switch (ch) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (ch < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", ch);
          o += b;
        } else {
          o += static_cast<char>(ch);
        }
    }
  }
  return o + "\"";
}

// JSON numbers: shortest round-trip text; non-finite values as null (what
// nlohmann::json, the reference's writer, emits for them).
std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";
  char b[40];
  for (int prec = 15; prec <= 17; ++prec) {
    std::snprintf(b, sizeof b, "%.*g", prec, v);
    if (std::strtod(b, nullptr) == v) break;
  }
  std::string s = b;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

// Schema of the reference's writer (bench.cpp:287-316), 2-space indent.
void write_benchmark_json(const BenchmarkReport& report, double epsilon, const std::string& path) {
  std::ostringstream j;
  j << "{\n  \"epsilon\": " << json_number(epsilon) << ",\n  \"records\": [";
  for (size_t i = 0; i < report.records.size(); ++i) {
    const BenchmarkRecord& r = report.records[i];
    j << (i ? ",\n" : "\n") << "    {\n";
    j << "      \"class\": " << json_string(to_string(r.size_class)) << ",\n";
    if (!r.error.empty()) j << "      \"error\": " << json_string(r.error) << ",\n";
    j << "      \"instance\": " << json_string(r.instance) << ",\n";
    j << "      \"iterations\": " << r.iterations << ",\n";
    j << "      \"nonzeros\": " << r.nonzeros << ",\n";
    j << "      \"restarts\": " << r.restart_count << ",\n";
    j << "      \"scored_seconds\": " << json_number(r.scored_seconds) << ",\n";
    j << "      \"solve_seconds\": " << json_number(r.solve_seconds) << ",\n";
    j << "      \"status\": " << json_string(r.status) << "\n    }";
  }
  j << (report.records.empty() ? "]" : "\n  ]") << ",\n  \"schema_version\": 1,\n  \"summary\": [";
  for (size_t i = 0; i < report.summary.size(); ++i) {
    const BenchmarkSummaryRow& s = report.summary[i];
    j << (i ? ",\n" : "\n") << "    {\n";
    j << "      \"count\": " << s.count << ",\n";
    j << "      \"group\": " << json_string(s.group) << ",\n";
    j << "      \"sgm10\": " << json_number(s.sgm10) << ",\n";
    j << "      \"solved\": " << s.solved << "\n    }";
  }
  j << (report.summary.empty() ? "]" : "\n  ]") << "\n}\n";
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
  out << j.str();
}

}  // namespace rhpdhg
