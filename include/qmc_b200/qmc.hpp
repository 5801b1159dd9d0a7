// C++ drop-in for the reference's American pricing API, backed by the B200
// kernels through the C ABI in qmcg.h.
//
// Mirrors, name for name, the reference declarations a caller of the hot path
// uses:
//   OptionKind / Method / OptionSpec / PricingResult   proj/include/qmc/types.hpp:16-49
//   ExecPolicy                                         proj/include/qmc/path_engine.hpp:36-39
//   price_american / convergence_curve                 proj/include/qmc/american.hpp:43-55
// so a reference caller relinks against libqmcg.so instead of american.cpp
// (see INTEGRATION.md). Exceptions follow the reference: std::invalid_argument
// for domain errors, std::length_error for size limits, std::runtime_error for
// device failures. ExecPolicy is accepted and, as in the reference
// (path_engine.hpp:33-35), never changes numeric results.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

namespace qmc {

using Index = std::ptrdiff_t;  // Eigen::Index in the reference

enum class OptionKind { Call, Put };
enum class Method { ClosedForm, EuropeanMC, AmericanUpperBound };

std::string method_name(Method method);

struct OptionSpec {
  double spot = 100.0;
  double strike = 100.0;
  double rate = 0.0;
  double volatility = 0.0;
  double maturity = 0.0;
  OptionKind kind = OptionKind::Call;
};

struct PricingResult {
  double price = 0.0;
  double std_error = 0.0;
  Index n_paths = 0;
  double elapsed_s = 0.0;
  Method method = Method::ClosedForm;
  std::uint64_t seed = 0;
};

struct ExecPolicy {
  int lanes = 1;
  Index chunk = 4096;
};

struct ConvergencePoint {
  Index m = 0;
  double price = 0.0;
  double std_error = 0.0;
  double elapsed_s = 0.0;
};
using ConvergenceCurve = std::vector<ConvergencePoint>;

// Foresight (upper-bound) American call value; reference american.cpp:103-131.
PricingResult price_american(const OptionSpec& spec, Index m, Index n_paths, std::uint64_t seed,
                             const ExecPolicy& exec = {});

// One price_american row per m, sorted ascending; reference american.cpp:133-150.
// The permutation tables depend on (seed, n_paths, dim) only, so the whole
// curve reuses one cached table set.
ConvergenceCurve convergence_curve(const OptionSpec& spec, const std::vector<Index>& m_values,
                                   Index n_paths, std::uint64_t seed, const ExecPolicy& exec = {});

// One-step QMC European price; reference proj/src/mc_european.cpp:11-46.
PricingResult mc_european_price(const OptionSpec& spec, Index n_paths, std::uint64_t seed,
                                const ExecPolicy& exec = {});

// ExerciseSchedule / make_schedule; reference proj/include/qmc/path_engine.hpp:15-22,
// proj/src/path_engine.cpp:63-76 (t_i = i dt for i = 1..m, then T; dt = T / (m+1)).
struct ExerciseSchedule {
  Index m = 0;
  double maturity = 0.0;
  double dt = 0.0;
  std::vector<double> times;  // m + 1 entries
  Index points() const { return m + 1; }
};
ExerciseSchedule make_schedule(Index m, double maturity);

// PathBatch / simulate_batch; reference path_engine.hpp:26-31, path_engine.cpp:124-152.
// prices is the reference's row-major [n_paths x points] matrix, generated on the GPU.
struct PathBatch {
  std::vector<double> prices;
  Index n_paths = 0;
  OptionSpec spec;
  ExerciseSchedule schedule;
  std::uint64_t seed = 0;
  double operator()(Index p, Index k) const { return prices[static_cast<std::size_t>(p * schedule.points() + k)]; }
};
PathBatch simulate_batch(const OptionSpec& spec, const ExerciseSchedule& schedule, Index n_paths,
                         std::uint64_t seed, const ExecPolicy& exec = {});

// SweepTrace / backward_sweep / sweep_value; reference proj/include/qmc/american.hpp:13-41.
// The reference takes Eigen::Ref<const RowVector>; pass path.data(), path.size().
struct SweepTrace {
  std::vector<double> values;             // t_0..t_m, then the payoff at T (m + 2 entries)
  std::optional<Index> exercise_point;    // earliest index where intrinsic beat continuation
};
SweepTrace backward_sweep(const double* path, Index path_len, const OptionSpec& spec,
                          const ExerciseSchedule& schedule);
double sweep_value(const double* path, Index path_len, const OptionSpec& spec,
                   const ExerciseSchedule& schedule);

namespace b200 {
// Extension (no reference counterpart): the same foresight rule for puts.
PricingResult price_american_put_extension(const OptionSpec& spec, Index m, Index n_paths,
                                           std::uint64_t seed);
// Select the CUDA device used by the process-wide context (default: 0).
// The drop-in prices on every visible GPU (a device group; QMCG_DEVICES narrows it) unless told
// otherwise here. Changing the devices or release() destroys the process-wide context, which
// frees its cached permutation tables.
void set_device(int device);
void set_devices(const std::vector<int>& devices);
void release();
int device_count();
}  // namespace b200

}  // namespace qmc
