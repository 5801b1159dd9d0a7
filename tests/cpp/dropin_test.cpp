// The C++ drop-in (include/qmc_b200/qmc.hpp, linked against libqmcg.so) run
// through the reference's own price_american / convergence_curve test cases
// (reference proj/tests/test_american.cpp:105-167), restated without doctest.
#include "qmc_b200/qmc.hpp"

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>
#include <stdexcept>

using qmc::ExecPolicy;
using qmc::Index;
using qmc::OptionKind;
using qmc::OptionSpec;

static int failures = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
      ++failures;                                                       \
    }                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                     \
  do {                                                                  \
    bool thrown = false;                                                \
    try {                                                               \
      (void)(expr);                                                     \
    } catch (const type&) {                                             \
      thrown = true;                                                    \
    } catch (...) {                                                     \
    }                                                                   \
    if (!thrown) {                                                      \
      std::printf("FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #type); \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

// closed-form call (the reference's bs_price, analytic.cpp:102-124) for the checks
static double bs_call(const OptionSpec& s) {
  const double vt = s.volatility * std::sqrt(s.maturity);
  if (s.volatility == 0.0) {
    const double fwd = s.spot * std::exp(s.rate * s.maturity);
    return std::exp(-s.rate * s.maturity) * (fwd > s.strike ? fwd - s.strike : 0.0);
  }
  const double d1 = (std::log(s.spot / s.strike) + (s.rate + 0.5 * s.volatility * s.volatility) * s.maturity) / vt;
  const double d2 = d1 - vt;
  const auto N = [](double x) { return 0.5 * std::erfc(-x / std::sqrt(2.0)); };
  return s.spot * N(d1) - s.strike * std::exp(-s.rate * s.maturity) * N(d2);
}

int main() {
  const OptionSpec kRef{100.0, 100.0, 0.05, 0.2, 1.0, OptionKind::Call};

  // puts are rejected (test_american.cpp:105-117)
  OptionSpec put = kRef;
  put.kind = OptionKind::Put;
  CHECK_THROWS_AS(qmc::price_american(put, 2, 64, 1, ExecPolicy{}), std::invalid_argument);
  CHECK_THROWS_AS(qmc::price_american(kRef, 2, 1, 1, ExecPolicy{}), std::invalid_argument);
  CHECK_THROWS_AS(qmc::price_american(kRef, 0, 64, 1, ExecPolicy{}), std::invalid_argument);
  CHECK_THROWS_AS(qmc::price_american(kRef, 2, Index{1} << 33, 1, ExecPolicy{}), std::length_error);

  // zero volatility reduces to the European value (:119-125)
  {
    const OptionSpec spec{100.0, 90.0, 0.05, 0.0, 1.0, OptionKind::Call};
    const double european = bs_call(spec);
    const auto result = qmc::price_american(spec, 6, 128, 3, ExecPolicy{2, 32});
    CHECK(std::fabs(result.price - european) <= 1e-12 * european);
    CHECK(std::fabs(result.std_error) <= 1e-12);
  }
  // upper bound dominates the European price (:127-131)
  {
    const auto result = qmc::price_american(kRef, 10, Index{1} << 14, 42, ExecPolicy{2});
    CHECK(result.price >= bs_call(kRef) - 3.0 * result.std_error);
    CHECK(result.method == qmc::Method::AmericanUpperBound);
    CHECK(qmc::method_name(result.method) == "american-ub");
  }
  // more exercise points never cheapen the option (:133-138)
  {
    const Index n = Index{1} << 14;
    const auto low = qmc::price_american(kRef, 1, n, 42, ExecPolicy{2});
    const auto high = qmc::price_american(kRef, 20, n, 42, ExecPolicy{2});
    CHECK(high.price >= low.price - 3.0 * (low.std_error + high.std_error));
  }
  // deterministic across lanes and chunks (:140-147)
  {
    const Index n = 20000;
    const auto a = qmc::price_american(kRef, 5, n, 42, ExecPolicy{1, 4096});
    const auto b = qmc::price_american(kRef, 5, n, 42, ExecPolicy{8, 4096});
    const auto c = qmc::price_american(kRef, 5, n, 42, ExecPolicy{3, 999});
    CHECK(std::memcmp(&a.price, &b.price, sizeof a.price) == 0);
    CHECK(std::memcmp(&a.price, &c.price, sizeof a.price) == 0);
  }
  // convergence_curve rows are sorted and dominate the closed form (:149-167)
  {
    const auto single = qmc::convergence_curve(kRef, {1}, 4096, 42, ExecPolicy{2});
    CHECK(single.size() == 1);
    const auto direct = qmc::price_american(kRef, 1, 4096, 42, ExecPolicy{2});
    CHECK(single[0].price == direct.price);
    const auto curve = qmc::convergence_curve(kRef, {10, 1, 5}, 4096, 42, ExecPolicy{2});
    CHECK(curve.size() == 3);
    CHECK(curve[0].m == 1 && curve[1].m == 5 && curve[2].m == 10);
    for (const auto& row : curve) CHECK(row.price >= bs_call(kRef) - 3.0 * row.std_error);
    CHECK_THROWS_AS(qmc::convergence_curve(kRef, {}, 4096, 42, ExecPolicy{}), std::invalid_argument);
  }
  // the published acceptance-7 value (proj/test_output.txt:33): 14.9587 at 1e6 paths, m = 10
  {
    const auto r = qmc::price_american(kRef, 10, 1000000, 42, ExecPolicy{8});
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.6g", r.price);
    CHECK(std::strcmp(buf, "14.9587") == 0);
  }
  // mc_european_price (test_mc_european.cpp:24-40): zero volatility / maturity are exact
  {
    const OptionSpec spec{100.0, 90.0, 0.05, 0.0, 1.0, OptionKind::Call};
    const double expected = std::exp(-0.05) * (100.0 * std::exp(0.05) - 90.0);
    for (const Index n : {Index{2}, Index{1000}, Index{4096}}) {
      const auto r = qmc::mc_european_price(spec, n, 1, ExecPolicy{2, 128});
      CHECK(r.price == expected);
      CHECK(r.std_error == 0.0);
    }
    const OptionSpec t0{110.0, 100.0, 0.05, 0.2, 0.0, OptionKind::Call};
    CHECK(qmc::mc_european_price(t0, 64, 1, ExecPolicy{}).price == 10.0);
    const auto mc = qmc::mc_european_price(kRef, Index{1} << 16, 42, ExecPolicy{2, 4096});
    CHECK(std::fabs(mc.price - bs_call(kRef)) < 3.0 * mc.std_error);
    CHECK(mc.method == qmc::Method::EuropeanMC);
  }
  // put extension (no reference counterpart)
  {
    const auto r = qmc::b200::price_american_put_extension(put, 20, 1 << 14, 42);
    CHECK(r.price > 0.0 && r.std_error > 0.0);
  }
  // backward_sweep / sweep_value (test_american.cpp:59-78, 94-103): hand 3-point sweep, terminal entry
  {
    const OptionSpec spec{100.0, 95.0, 0.0, 0.3, 1.0, OptionKind::Call};
    const auto schedule = qmc::make_schedule(3, 1.0);
    const std::vector<double> path{108.0, 91.0, 104.0, 97.0};
    const double value = qmc::sweep_value(path.data(), static_cast<Index>(path.size()), spec, schedule);
    CHECK(std::fabs(value - 13.0) <= 1e-15 * 13.0);
    const auto trace = qmc::backward_sweep(path.data(), static_cast<Index>(path.size()), spec, schedule);
    CHECK(trace.exercise_point.has_value() && *trace.exercise_point == 1);
    CHECK(trace.values[0] == value);
    const auto s2 = qmc::make_schedule(2, 1.0);
    const std::vector<double> p2{104.0, 99.0, 117.5};
    CHECK(qmc::backward_sweep(p2.data(), 3, kRef, s2).values.back() == 17.5);
    CHECK_THROWS_AS(qmc::backward_sweep(p2.data(), 2, kRef, s2), std::invalid_argument);
    CHECK_THROWS_AS(qmc::make_schedule(0, 1.0), std::invalid_argument);
  }
  // simulate_batch (test_path_engine.cpp:62-104): deterministic forward, lanes invariance, capacity
  {
    const OptionSpec spec{100.0, 100.0, 0.05, 0.0, 1.0, OptionKind::Call};
    const auto b = qmc::simulate_batch(spec, qmc::make_schedule(1, 1.0), 1, 7, ExecPolicy{1, 16});
    CHECK(b.prices.size() == 2);
    CHECK(std::fabs(b(0, 0) - 100.0 * std::exp(0.025)) <= 1e-12 * b(0, 0));
    CHECK(std::fabs(b(0, 1) - 100.0 * std::exp(0.05)) <= 1e-12 * b(0, 1));
    const OptionSpec s5{100.0, 95.0, 0.03, 0.25, 2.0, OptionKind::Call};
    const auto sched = qmc::make_schedule(5, 2.0);
    const auto base = qmc::simulate_batch(s5, sched, 20000, 42, ExecPolicy{1, 4096});
    const auto lanes8 = qmc::simulate_batch(s5, sched, 20000, 42, ExecPolicy{8, 777});
    CHECK(base.prices == lanes8.prices);
    CHECK(*std::min_element(base.prices.begin(), base.prices.end()) > 0.0);
    bool threw = false;
    try {
      qmc::simulate_batch(kRef, qmc::make_schedule(1000, 1.0), Index{1} << 40, 1, ExecPolicy{});
    } catch (const std::length_error& e) {
      const std::string msg = e.what();
      threw = msg.find("bytes") != std::string::npos && msg.find("1001") != std::string::npos;
    }
    CHECK(threw);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
