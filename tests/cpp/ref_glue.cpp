// The reference-side binding of the drop-in: the hot-path functions with the REFERENCE's own
// declarations (proj/include/qmc/american.hpp:36-55, mc_european.hpp, path_engine.hpp:24-58),
// compiled against those headers, forwarding to libqmcg.so's C ABI (include/qmcg.h).
//
// A maintainer relinking the reference against the B200 pricer compiles this file in place of
// proj/src/american.cpp and proj/src/mc_european.cpp (and weakens simulate_batch in
// path_engine.o); oracle/Makefile does exactly that to link the reference's unmodified
// acceptance binary and unit suites (target ref_suites). Everything else (bs_price, cnd, the
// CRR oracle, run_benchmark, reduce_stats) stays the reference's own code.
#include "qmc/american.hpp"
#include "qmc/analytic.hpp"
#include "qmc/mc_european.hpp"
#include "qmc/path_engine.hpp"
#include "qmcg.h"

#include <algorithm>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

namespace qmc {
namespace {

std::mutex g_mu;
qmcg_ctx* g_ctx = nullptr;

// every visible GPU (a device group), or QMCG_DEVICES
qmcg_ctx* context() {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_ctx && qmcg_create_default(&g_ctx) != QMCG_OK) {
    g_ctx = nullptr;
    throw std::runtime_error(qmcg_last_error());
  }
  return g_ctx;
}

[[noreturn]] void rethrow(qmcg_status st) {
  const std::string msg = qmcg_last_error();
  if (st == QMCG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == QMCG_LENGTH_ERROR) throw std::length_error(msg);
  throw std::runtime_error(msg);
}

qmcg_option_spec to_c(const OptionSpec& s) {
  return qmcg_option_spec{s.spot, s.strike, s.rate, s.volatility, s.maturity,
                          s.kind == OptionKind::Call ? QMCG_CALL : QMCG_PUT};
}

void check_exec(const ExecPolicy& exec) {  // parallel_for_chunks (path_engine.cpp:86-87)
  if (exec.lanes < 1) throw std::invalid_argument("parallel_for_chunks: lanes must be >= 1");
  if (exec.chunk < 1) throw std::invalid_argument("parallel_for_chunks: chunk must be >= 1");
}

PricingResult from_c(const qmcg_pricing_result& r, Method method) {
  PricingResult out;
  out.price = r.price;
  out.std_error = r.std_error;
  out.n_paths = static_cast<Index>(r.n_paths);
  out.elapsed_s = r.elapsed_s;
  out.method = method;
  out.seed = r.seed;
  return out;
}

}  // namespace

PricingResult price_american(const OptionSpec& spec, Index m, Index n_paths, std::uint64_t seed,
                             const ExecPolicy& exec) {
  check_exec(exec);
  const qmcg_option_spec cs = to_c(spec);
  qmcg_pricing_result r{};
  const qmcg_status st = qmcg_price_american(context(), &cs, m, n_paths, seed, 0u, &r);
  if (st != QMCG_OK) rethrow(st);
  return from_c(r, Method::AmericanUpperBound);
}

ConvergenceCurve convergence_curve(const OptionSpec& spec, const std::vector<Index>& m_values, Index n_paths,
                                   std::uint64_t seed, const ExecPolicy& exec) {
  if (m_values.empty()) throw std::invalid_argument("convergence_curve: m_values must be non-empty");
  std::vector<Index> sorted = m_values;
  std::sort(sorted.begin(), sorted.end());
  ConvergenceCurve curve;
  for (const Index m : sorted) {
    const PricingResult r = price_american(spec, m, n_paths, seed, exec);
    curve.push_back(ConvergencePoint{m, r.price, r.std_error, r.elapsed_s});
  }
  return curve;
}

PricingResult mc_european_price(const OptionSpec& spec, Index n_paths, std::uint64_t seed, const ExecPolicy& exec) {
  check_exec(exec);
  const qmcg_option_spec cs = to_c(spec);
  qmcg_pricing_result r{};
  const qmcg_status st = qmcg_mc_european_price(context(), &cs, n_paths, seed, 0u, &r);
  if (st != QMCG_OK) rethrow(st);
  return from_c(r, Method::EuropeanMC);
}

PathBatch simulate_batch(const OptionSpec& spec, const ExerciseSchedule& schedule, Index n_paths, std::uint64_t seed,
                         const ExecPolicy& exec) {
  check_exec(exec);
  const qmcg_option_spec cs = to_c(spec);
  qmcg_status st = qmcg_simulate_batch(nullptr, &cs, schedule.m, n_paths, seed, 0u, QMCG_LAYOUT_PATH_MAJOR, nullptr);
  if (st != QMCG_OK) rethrow(st);  // the reference's checks (incl. the 128 GiB cap) before allocating
  PathBatch batch;
  batch.prices = Matrix(n_paths, schedule.points());
  st = qmcg_simulate_batch(context(), &cs, schedule.m, n_paths, seed, 0u, QMCG_LAYOUT_PATH_MAJOR,
                           batch.prices.data());
  if (st != QMCG_OK) rethrow(st);
  batch.spec = spec;
  batch.schedule = schedule;
  batch.seed = seed;
  return batch;
}

SweepTrace backward_sweep(Eigen::Ref<const RowVector> path, const OptionSpec& spec,
                          const ExerciseSchedule& schedule) {
  const qmcg_option_spec cs = to_c(spec);
  SweepTrace trace;
  trace.values.assign(static_cast<std::size_t>(schedule.m) + 2, 0.0);
  int64_t ex = -1;
  const qmcg_status st =
      qmcg_backward_sweep(path.data(), path.size(), &cs, schedule.m, 0u, trace.values.data(), &ex);
  if (st != QMCG_OK) rethrow(st);
  if (ex >= 0) trace.exercise_point = static_cast<Index>(ex);
  return trace;
}

double sweep_value(Eigen::Ref<const RowVector> path, const OptionSpec& spec, const ExerciseSchedule& schedule) {
  return backward_sweep(path, spec, schedule).values[0];
}

}  // namespace qmc
