// C++ drop-in (include/qmc_b200/qmc.hpp) over the C ABI: one process-wide
// context, reference exception mapping.
#include "qmc_b200/qmc.hpp"

#include "qmcg.h"

#include <algorithm>
#include <chrono>
#include <mutex>
#include <stdexcept>

namespace qmc {

namespace {

std::mutex g_mu;
qmcg_ctx* g_ctx = nullptr;
int g_device = 0;

qmcg_ctx* context() {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_ctx) {
    if (qmcg_create(g_device, &g_ctx) != QMCG_OK) throw std::runtime_error(qmcg_last_error());
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

namespace b200 {

PricingResult price_american_put_extension(const OptionSpec& spec, Index m, Index n_paths, std::uint64_t seed) {
  return price(spec, m, n_paths, seed, QMCG_FLAG_ALLOW_PUT);
}

void set_device(int device) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_ctx) {
    qmcg_destroy(g_ctx);
    g_ctx = nullptr;
  }
  g_device = device;
}

}  // namespace b200

}  // namespace qmc
