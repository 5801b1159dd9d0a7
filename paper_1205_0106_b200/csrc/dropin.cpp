// C++ drop-in (include/qmc_b200/qmc.hpp) over the C ABI: one process-wide
// context, reference exception mapping.
#include "qmc_b200/qmc.hpp"

#include "qmcg.h"

#include <algorithm>
#include <chrono>
#include <mutex>
#include <stdexcept>
#include <vector>

namespace qmc {

namespace {

std::mutex g_mu;
qmcg_ctx* g_ctx = nullptr;
std::vector<int> g_devices;  // empty: every visible device (or QMCG_DEVICES), qmcg_create_default

// The process-wide context: a device group over all visible GPUs unless narrowed with
// b200::set_devices / set_device (the reference's ExecPolicy lanes stay a hint, as there).
qmcg_ctx* context() {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_ctx) {
    qmcg_status st;
    if (g_devices.empty()) st = qmcg_create_default(&g_ctx);
    else if (g_devices.size() == 1) st = qmcg_create(g_devices[0], &g_ctx);
    else st = qmcg_create_multi(g_devices.data(), static_cast<int>(g_devices.size()), &g_ctx);
    if (st != QMCG_OK) {
      g_ctx = nullptr;
      throw std::runtime_error(qmcg_last_error());
    }
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

PricingResult from_c(const qmcg_pricing_result& r) {
  PricingResult out;
  out.price = r.price;
  out.std_error = r.std_error;
  out.n_paths = static_cast<Index>(r.n_paths);
  out.elapsed_s = r.elapsed_s;
  out.method = Method::AmericanUpperBound;
  out.seed = r.seed;
  return out;
}

PricingResult price(const OptionSpec& spec, Index m, Index n_paths, std::uint64_t seed, uint32_t flags) {
  const qmcg_option_spec cs = to_c(spec);
  qmcg_pricing_result r{};
  const qmcg_status st = qmcg_price_american(context(), &cs, m, n_paths, seed, flags, &r);
  if (st != QMCG_OK) rethrow(st);
  return from_c(r);
}

}  // namespace

std::string method_name(Method method) {
  switch (method) {
    case Method::ClosedForm: return "closed-form";
    case Method::EuropeanMC: return "european-mc";
    case Method::AmericanUpperBound: return "american-ub";
  }
  return "unknown";
}

PricingResult price_american(const OptionSpec& spec, Index m, Index n_paths, std::uint64_t seed,
                             const ExecPolicy& exec) {
  // parallel_for_chunks' policy checks (path_engine.cpp:86-87) still apply
  if (exec.lanes < 1) throw std::invalid_argument("parallel_for_chunks: lanes must be >= 1");
  if (exec.chunk < 1) throw std::invalid_argument("parallel_for_chunks: chunk must be >= 1");
  return price(spec, m, n_paths, seed, 0u);
}

ConvergenceCurve convergence_curve(const OptionSpec& spec, const std::vector<Index>& m_values, Index n_paths,
                                   std::uint64_t seed, const ExecPolicy& exec) {
  if (m_values.empty()) throw std::invalid_argument("convergence_curve: m_values must be non-empty");
  std::vector<Index> sorted = m_values;
  std::sort(sorted.begin(), sorted.end());
  ConvergenceCurve curve;
  curve.reserve(sorted.size());
  for (const Index m : sorted) {
    const PricingResult r = price_american(spec, m, n_paths, seed, exec);
    curve.push_back(ConvergencePoint{m, r.price, r.std_error, r.elapsed_s});
  }
  return curve;
}

PricingResult mc_european_price(const OptionSpec& spec, Index n_paths, std::uint64_t seed, const ExecPolicy& exec) {
  if (exec.lanes < 1) throw std::invalid_argument("parallel_for_chunks: lanes must be >= 1");
  if (exec.chunk < 1) throw std::invalid_argument("parallel_for_chunks: chunk must be >= 1");
  const qmcg_option_spec cs = to_c(spec);
  qmcg_pricing_result r{};
  const qmcg_status st = qmcg_mc_european_price(context(), &cs, n_paths, seed, 0u, &r);
  if (st != QMCG_OK) rethrow(st);
  PricingResult out = from_c(r);
  out.method = Method::EuropeanMC;
  return out;
}

ExerciseSchedule make_schedule(Index m, double maturity) {
  if (m < 1) throw std::invalid_argument("make_schedule: m must be >= 1");
  if (!(maturity > 0.0)) throw std::invalid_argument("make_schedule: maturity must be > 0");
  ExerciseSchedule s;
  s.m = m;
  s.maturity = maturity;
  s.dt = maturity / static_cast<double>(m + 1);
  s.times.resize(static_cast<std::size_t>(m) + 1);
  for (Index i = 0; i < m; ++i) s.times[static_cast<std::size_t>(i)] = static_cast<double>(i + 1) * s.dt;
  s.times[static_cast<std::size_t>(m)] = maturity;
  return s;
}

namespace {
void check_schedule(const ExerciseSchedule& schedule, const char* who) {
  if (schedule.m < 1 || schedule.times.size() != static_cast<std::size_t>(schedule.m) + 1)
    throw std::invalid_argument(std::string(who) + ": schedule is not initialized");
}
}  // namespace

PathBatch simulate_batch(const OptionSpec& spec, const ExerciseSchedule& schedule, Index n_paths, std::uint64_t seed,
                         const ExecPolicy& exec) {
  if (exec.lanes < 1) throw std::invalid_argument("parallel_for_chunks: lanes must be >= 1");
  if (exec.chunk < 1) throw std::invalid_argument("parallel_for_chunks: chunk must be >= 1");
  check_schedule(schedule, "simulate_batch");
  if (schedule.maturity != spec.maturity)
    throw std::invalid_argument("simulate_batch: schedule maturity does not match spec maturity");
  const qmcg_option_spec cs = to_c(spec);
  PathBatch batch;
  // validation (incl. the 128 GiB capacity check) happens before any allocation
  qmcg_status st = qmcg_simulate_batch(context(), &cs, schedule.m, n_paths, seed, 0u, QMCG_LAYOUT_PATH_MAJOR, nullptr);
  if (st != QMCG_OK) rethrow(st);
  batch.prices.resize(static_cast<std::size_t>(n_paths) * static_cast<std::size_t>(schedule.points()));
  st = qmcg_simulate_batch(context(), &cs, schedule.m, n_paths, seed, 0u, QMCG_LAYOUT_PATH_MAJOR,
                           batch.prices.data());
  if (st != QMCG_OK) rethrow(st);
  batch.n_paths = n_paths;
  batch.spec = spec;
  batch.schedule = schedule;
  batch.seed = seed;
  return batch;
}

SweepTrace backward_sweep(const double* path, Index path_len, const OptionSpec& spec,
                          const ExerciseSchedule& schedule) {
  check_schedule(schedule, "backward_sweep");
  const qmcg_option_spec cs = to_c(spec);
  SweepTrace trace;
  trace.values.assign(static_cast<std::size_t>(schedule.m) + 2, 0.0);
  int64_t ex = -1;
  const qmcg_status st = qmcg_backward_sweep(path, path_len, &cs, schedule.m, 0u, trace.values.data(), &ex);
  if (st != QMCG_OK) rethrow(st);
  if (ex >= 0) trace.exercise_point = static_cast<Index>(ex);
  return trace;
}

double sweep_value(const double* path, Index path_len, const OptionSpec& spec, const ExerciseSchedule& schedule) {
  return backward_sweep(path, path_len, spec, schedule).values[0];
}

namespace b200 {

PricingResult price_american_put_extension(const OptionSpec& spec, Index m, Index n_paths, std::uint64_t seed) {
  return price(spec, m, n_paths, seed, QMCG_FLAG_ALLOW_PUT);
}

void set_devices(const std::vector<int>& devices) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_ctx) {
    qmcg_destroy(g_ctx);
    g_ctx = nullptr;
  }
  g_devices = devices;
}

void set_device(int device) { set_devices({device}); }

void release() {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_ctx) {
    qmcg_destroy(g_ctx);  // frees the permutation-table cache (17 GB at config 3) and all scratch
    g_ctx = nullptr;
  }
}

int device_count() { return qmcg_device_count(context()); }

}  // namespace b200

}  // namespace qmc
