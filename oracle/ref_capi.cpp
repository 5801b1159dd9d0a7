// C-ABI shim over the REFERENCE's own hot-path sources -- TEST INFRASTRUCTURE ONLY.
//
// oracle/Makefile compiles /root/reference/proj/src/{analytic,quasi_rng,
// path_engine,american,mc_european,oracles}.cpp unmodified (with the Eigen
// container shim in oracle/eigen_shim) and links them with this file into
// oracle/_ref/libqmcref.so. Python tests and bench.py's reference arm load it
// with ctypes. Nothing in the product path may link or call this library.
//
// Status codes: 0 ok, 1 std::invalid_argument, 2 std::length_error,
// 3 any other exception. The exception text is copied into `err`.
#include "qmc/american.hpp"
#include "qmc/analytic.hpp"
#include "qmc/bench.hpp"
#include "qmc/mc_european.hpp"
#include "qmc/oracles.hpp"
#include "qmc/path_engine.hpp"
#include "qmc/quasi_rng.hpp"

#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

using namespace qmc;

namespace {

int fail(const std::exception& e, int code, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), static_cast<std::size_t>(errlen - 1));
    err[errlen - 1] = '\0';
  }
  return code;
}

template <class F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1, err, errlen);
  } catch (const std::length_error& e) {
    return fail(e, 2, err, errlen);
  } catch (const std::exception& e) {
    return fail(e, 3, err, errlen);
  }
}

OptionSpec make_spec(const double* s, int kind) {
  return OptionSpec{s[0], s[1], s[2], s[3], s[4], kind == 0 ? OptionKind::Call : OptionKind::Put};
}

}  // namespace

extern "C" {

// spec = {spot, strike, rate, volatility, maturity}; kind 0 = call, 1 = put.
// out = {price, std_error, elapsed_s}.
int ref_price_american(const double* spec, int kind, std::int64_t m, std::int64_t n,
                       std::uint64_t seed, int lanes, std::int64_t chunk, double* out,
                       char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const PricingResult r = price_american(make_spec(spec, kind), m, n, seed, ExecPolicy{lanes, chunk});
    out[0] = r.price;
    out[1] = r.std_error;
    out[2] = r.elapsed_s;
  });
}

int ref_mc_european_price(const double* spec, int kind, std::int64_t n, std::uint64_t seed,
                          int lanes, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const PricingResult r = mc_european_price(make_spec(spec, kind), n, seed, ExecPolicy{lanes, 4096});
    out[0] = r.price;
    out[1] = r.std_error;
    out[2] = r.elapsed_s;
  });
}

std::uint64_t ref_dimension_seed(std::uint64_t seed, std::int64_t dim) {
  return dimension_seed(seed, dim);
}

int ref_permutation_indices(std::int64_t n, std::uint64_t seed, std::uint32_t* out, char* err,
                            int errlen) {
  return guarded(err, errlen, [&] {
    const auto p = permutation_indices(n, seed);
    std::memcpy(out, p.data(), p.size() * sizeof(std::uint32_t));
  });
}

double ref_radical_inverse(std::uint64_t index, std::uint32_t base) {
  return radical_inverse(index, base);
}

// One column of QuasiStream(dims > dim, length, seed): uniform_at(p, dim) for every p, i.e.
// radical_inverse(perm_dim[p] + 1, base) with perm_dim = permutation_indices(length,
// dimension_seed(seed, dim)) -- the body of uniform_at (quasi_rng.cpp:96-101, pinned to that
// composition by proj/tests/test_quasi_rng.cpp:154-169) without building every other dimension.
int ref_uniform_column(std::int64_t length, std::uint64_t seed, std::int64_t dim, std::uint32_t base, double* out,
                       char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const auto perm = permutation_indices(length, dimension_seed(seed, dim));
    for (std::int64_t p = 0; p < length; ++p)
      out[p] = radical_inverse(static_cast<std::uint64_t>(perm[static_cast<std::size_t>(p)]) + 1, base);
  });
}

// Row-major [length][dims] uniforms, as uniform_matrix returns them.
int ref_uniform_matrix(std::int64_t dims, std::int64_t length, std::uint64_t seed, double* out,
                       char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const Matrix u = uniform_matrix(dims, length, seed);
    std::memcpy(out, u.data(), static_cast<std::size_t>(u.size()) * sizeof(double));
  });
}

int ref_moro_inv_cnd(double u, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = moro_inv_cnd(u); });
}

int ref_cnd(double d, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = cnd(d); });
}

int ref_bs_price(const double* spec, int kind, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = bs_price(make_spec(spec, kind)); });
}

double ref_gbm_step(double s_prev, double dt, double z, double rate, double vol) {
  return gbm_step(s_prev, dt, z, rate, vol);
}

// Path matrix [n][m+1] (row-major) from simulate_batch.
int ref_simulate_batch(const double* spec, int kind, std::int64_t m, std::int64_t n,
                       std::uint64_t seed, int lanes, double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const OptionSpec s = make_spec(spec, kind);
    const ExerciseSchedule sched = make_schedule(m, s.maturity);
    const PathBatch b = simulate_batch(s, sched, n, seed, ExecPolicy{lanes, 4096});
    std::memcpy(out, b.prices.data(), static_cast<std::size_t>(b.prices.size()) * sizeof(double));
  });
}

// sweep_value over one path of m+1 prices; also returns the full trace
// (m+2 values) and the exercise point (-1 when none) via backward_sweep.
int ref_backward_sweep(const double* path, std::int64_t m, const double* spec, int kind,
                       double* value, double* trace, std::int64_t* exercise_point, char* err,
                       int errlen) {
  return guarded(err, errlen, [&] {
    const OptionSpec s = make_spec(spec, kind);
    const ExerciseSchedule sched = make_schedule(m, s.maturity);
    RowVector row(m + 1);
    for (std::int64_t k = 0; k <= m; ++k) row[k] = path[k];
    *value = sweep_value(row, s, sched);
    const SweepTrace t = backward_sweep(row, s, sched);
    for (std::size_t i = 0; i < t.values.size(); ++i) trace[i] = t.values[i];
    *exercise_point = t.exercise_point ? *t.exercise_point : -1;
  });
}

int ref_tree_reduce(const double* values, std::int64_t n, int lanes, double* out, char* err,
                    int errlen) {
  return guarded(err, errlen, [&] { *out = tree_reduce(values, n, lanes); });
}

int ref_reduce_stats(const double* values, std::int64_t n, int lanes, double* out, char* err,
                     int errlen) {
  return guarded(err, errlen, [&] {
    Vector v(n);
    for (std::int64_t i = 0; i < n; ++i) v[i] = values[i];
    const ReduceStats s = reduce_stats(v, lanes);
    out[0] = s.mean;
    out[1] = s.std_error;
  });
}

int ref_crr_price(const double* spec, int kind, std::int64_t steps, int american, double* out,
                  char* err, int errlen) {
  return guarded(err, errlen, [&] {
    oracle::TreeConfig cfg{steps, make_spec(spec, kind)};
    *out = oracle::crr_price(cfg, american != 0);
  });
}

int ref_make_schedule(std::int64_t m, double maturity, double* dt, double* times, char* err,
                      int errlen) {
  return guarded(err, errlen, [&] {
    const ExerciseSchedule s = make_schedule(m, maturity);
    *dt = s.dt;
    if (times)
      for (std::size_t i = 0; i < s.times.size(); ++i) times[i] = s.times[i];
  });
}

int ref_default_lanes(void) { return default_lanes(); }

// emit_records (bench.cpp:203-283) of n records given column-wise; format 0 table,
// 1 csv, 2 json. The text (NUL-terminated) goes to out; *len gets its length.
int ref_emit_records(int n, const int* method, const std::int64_t* n_paths, const std::int64_t* m,
                     const int* lanes, const std::int64_t* chunk, const std::uint64_t* seed, const double* price,
                     const double* se, const double* elapsed, int format, char* out, std::int64_t outlen,
                     std::int64_t* len, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<BenchmarkRecord> recs(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
      BenchmarkRecord& r = recs[static_cast<std::size_t>(i)];
      r.method = static_cast<Method>(method[i]);
      r.n_paths = n_paths[i];
      r.m = m[i];
      r.lanes = lanes[i];
      r.chunk = chunk[i];
      r.seed = seed[i];
      r.price = price[i];
      r.std_error = se[i];
      r.elapsed_s = elapsed[i];
    }
    std::ostringstream os;
    emit_records(recs, format == 0 ? OutputFormat::Table : format == 1 ? OutputFormat::Csv : OutputFormat::Json, os);
    const std::string text = os.str();
    *len = static_cast<std::int64_t>(text.size());
    if (static_cast<std::int64_t>(text.size()) + 1 > outlen) throw std::length_error("ref_emit_records: buffer");
    std::memcpy(out, text.c_str(), text.size() + 1);
  });
}

// parse_csv_records (bench.cpp:299-330): up to maxn records, column-wise; *count = parsed.
int ref_parse_csv_records(const char* text, int maxn, int* method, std::int64_t* n_paths, std::int64_t* m,
                          int* lanes, std::int64_t* chunk, std::uint64_t* seed, double* price, double* se,
                          double* elapsed, int* count, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::istringstream in{std::string(text)};
    const auto recs = parse_csv_records(in);
    *count = static_cast<int>(recs.size());
    for (int i = 0; i < *count && i < maxn; ++i) {
      const BenchmarkRecord& r = recs[static_cast<std::size_t>(i)];
      method[i] = static_cast<int>(r.method);
      n_paths[i] = r.n_paths;
      m[i] = r.m;
      lanes[i] = r.lanes;
      chunk[i] = r.chunk;
      seed[i] = r.seed;
      price[i] = r.price;
      se[i] = r.std_error;
      elapsed[i] = r.elapsed_s;
    }
  });
}

}  // extern "C"
