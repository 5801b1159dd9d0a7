/* Plain-C restatement of the reference's American-option QMC hot path.
 *
 * TEST INFRASTRUCTURE ONLY: this is the CPU checker the CUDA product is
 * compared against. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product (paper_1205_0106_b200/) never does.
 *
 * Every function restates the reference function cited beside it, keeping the
 * exact IEEE operation order (compiled with -ffp-contract=off, no FMA, against
 * the same glibc libm), so its results are bit-identical to the reference's.
 * That claim is pinned by tests/test_oracle.py against oracle/_ref (the
 * reference's own sources compiled here) and the committed golden vectors in
 * tests/golden/.
 */
#include "qmc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int set_err(char* err, int errlen, int code, const char* msg) {
  if (err && errlen > 0) {
    strncpy(err, msg, (size_t)errlen - 1);
    err[errlen - 1] = '\0';
  }
  return code;
}

/* proj/src/quasi_rng.cpp:16-22 */
static uint64_t splitmix64(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* proj/src/quasi_rng.cpp:41-46 */
uint64_t qo_dimension_seed(uint64_t master_seed, int64_t dim) {
  uint64_t state = master_seed;
  uint64_t mixed = splitmix64(&state);
  state = mixed ^ ((uint64_t)dim + 0x632be59bd9b4e019ULL);
  return splitmix64(&state);
}

/* proj/src/quasi_rng.cpp:24-37 (trial division) */
void qo_first_primes(int64_t count, uint32_t* out) {
  int64_t have = 0;
  uint32_t candidate = 2;
  while (have < count) {
    int is_prime = 1;
    for (uint32_t d = 2; d * d <= candidate; ++d) {
      if (candidate % d == 0) { is_prime = 0; break; }
    }
    if (is_prime) out[have++] = candidate;
    ++candidate;
  }
}

/* Knuth MMIX LCG, proj/include/qmc/quasi_rng.hpp:11-24 */
static inline uint64_t lcg_below(uint64_t* state, uint64_t bound) {
  *state = *state * 6364136223846793005ULL + 1442695040888963407ULL;
  return (uint64_t)(((unsigned __int128)(*state) * bound) >> 64);
}

/* Fisher-Yates, proj/src/quasi_rng.cpp:48-61 */
int qo_permutation_indices(int64_t n, uint64_t seed, uint32_t* out, char* err, int errlen) {
  if (n < 1) return set_err(err, errlen, QO_INVALID_ARGUMENT, "permutation_indices: n must be >= 1");
  if ((uint64_t)n > 0xffffffffULL)
    return set_err(err, errlen, QO_LENGTH_ERROR,
                   "permutation_indices: n exceeds the 2^32-1 supported maximum");
  for (int64_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
  uint64_t state = seed;
  for (int64_t i = n - 1; i > 0; --i) {
    const uint64_t j = lcg_below(&state, (uint64_t)i + 1);
    const uint32_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
  return QO_OK;
}

/* proj/src/quasi_rng.cpp:71-83 */
double qo_radical_inverse(uint64_t index, uint32_t base) {
  const double eps = 1e-12; /* kEndpointEps, proj/src/quasi_rng.cpp:14 */
  const double inv_base = 1.0 / base;
  double scale = inv_base;
  double value = 0.0;
  while (index != 0) {
    value += (double)(index % base) * scale;
    index /= base;
    scale *= inv_base;
  }
  if (value < eps) value = eps;
  if (value > 1.0 - eps) value = 1.0 - eps;
  return value;
}

/* Moro inverse CND, proj/src/analytic.cpp:74-100 */
int qo_moro_inv_cnd(double u, double* out, char* err, int errlen) {
  static const double a[4] = {2.50662823884, -18.61500062529, 41.39119773534, -25.44106049637};
  static const double b[4] = {-8.47351093090, 23.08336743743, -21.06224101826, 3.13082909833};
  static const double c[9] = {0.3374754822726147, 0.9761690190917186, 0.1607979714918209,
                              0.0276438810333863, 0.0038405729373609, 0.0003951896511919,
                              0.0000321767881768, 0.0000002888167364, 0.0000003960315187};
  if (!(u > 0.0) || !(u < 1.0))
    return set_err(err, errlen, QO_INVALID_ARGUMENT, "moro_inv_cnd: u must lie strictly in (0,1)");
  const double y = u - 0.5;
  if (fabs(y) <= 0.42) {
    const double r = y * y;
    *out = y * (((a[3] * r + a[2]) * r + a[1]) * r + a[0]) /
           ((((b[3] * r + b[2]) * r + b[1]) * r + b[0]) * r + 1.0);
    return QO_OK;
  }
  const double z = (y > 0.0) ? log(-log(1.0 - u)) : log(-log(u));
  double x = c[8];
  for (int i = 7; i >= 0; --i) x = x * z + c[i];
  *out = (y > 0.0) ? x : -x;
  return QO_OK;
}

/* Hart CND, proj/src/analytic.cpp:33-72 */
int qo_cnd(double d, double* out, char* err, int errlen) {
  if (!isfinite(d)) return set_err(err, errlen, QO_INVALID_ARGUMENT, "cnd: input must be finite");
  const double x = fabs(d);
  double tail;
  if (x > 37.0) {
    tail = 0.0;
  } else {
    const double e = exp(-0.5 * x * x);
    if (x < 7.07106781186547) {
      double num = 3.52624965998911e-02;
      num = num * x + 0.700383064443688;
      num = num * x + 6.37396220353165;
      num = num * x + 33.912866078383;
      num = num * x + 112.079291497871;
      num = num * x + 221.213596169931;
      num = num * x + 220.206867912376;
      double den = 8.83883476483184e-02;
      den = den * x + 1.75566716318264;
      den = den * x + 16.064177579207;
      den = den * x + 86.7807322029461;
      den = den * x + 296.564248779674;
      den = den * x + 637.333633378831;
      den = den * x + 793.826512519948;
      den = den * x + 440.413735824752;
      tail = e * num / den;
    } else {
      double b = x + 0.65;
      b = x + 4.0 / b;
      b = x + 3.0 / b;
      b = x + 2.0 / b;
      b = x + 1.0 / b;
      tail = e / (b * 2.506628274631000502);
    }
  }
  *out = d > 0.0 ? 1.0 - tail : tail;
  return QO_OK;
}

/* proj/src/analytic.cpp:18-31 */
int qo_validate(const qo_spec* s, char* err, int errlen) {
  if (!isfinite(s->spot) || !isfinite(s->strike) || !isfinite(s->rate) ||
      !isfinite(s->volatility) || !isfinite(s->maturity))
    return set_err(err, errlen, QO_INVALID_ARGUMENT, "OptionSpec: all fields must be finite");
  if (!(s->spot > 0.0)) return set_err(err, errlen, QO_INVALID_ARGUMENT, "OptionSpec: spot must be > 0");
  if (!(s->strike > 0.0)) return set_err(err, errlen, QO_INVALID_ARGUMENT, "OptionSpec: strike must be > 0");
  if (!(s->volatility >= 0.0))
    return set_err(err, errlen, QO_INVALID_ARGUMENT, "OptionSpec: volatility must be >= 0");
  if (!(s->maturity >= 0.0))
    return set_err(err, errlen, QO_INVALID_ARGUMENT, "OptionSpec: maturity must be >= 0");
  return QO_OK;
}

/* proj/include/qmc/types.hpp:37-40 */
static inline double intrinsic(int kind, double s, double strike) {
  const double diff = (kind == QO_CALL) ? s - strike : strike - s;
  return diff > 0.0 ? diff : 0.0;
}

/* proj/src/analytic.cpp:102-124 */
int qo_bs_price(const qo_spec* spec, double* out, char* err, int errlen) {
  int st = qo_validate(spec, err, errlen);
  if (st) return st;
  const double s = spec->spot, x = spec->strike, r = spec->rate, v = spec->volatility,
               t = spec->maturity;
  if (t == 0.0) { *out = intrinsic(spec->kind, s, x); return QO_OK; }
  if (v == 0.0) {
    const double forward = s * exp(r * t);
    *out = exp(-r * t) * intrinsic(spec->kind, forward, x);
    return QO_OK;
  }
  const double v_sqrt_t = v * sqrt(t);
  const double d1 = (log(s / x) + (r + 0.5 * v * v) * t) / v_sqrt_t;
  const double d2 = d1 - v_sqrt_t;
  const double disc = exp(-r * t);
  double c1, c2, price;
  if (spec->kind == QO_CALL) {
    if ((st = qo_cnd(d1, &c1, err, errlen))) return st;
    if ((st = qo_cnd(d2, &c2, err, errlen))) return st;
    price = s * c1 - x * disc * c2;
  } else {
    if ((st = qo_cnd(-d2, &c2, err, errlen))) return st;
    if ((st = qo_cnd(-d1, &c1, err, errlen))) return st;
    price = x * disc * c2 - s * c1;
  }
  *out = price > 0.0 ? price : 0.0;
  return QO_OK;
}

/* pairwise_sum, proj/src/path_engine.cpp:37-47 (64-element sequential leaves) */
double qo_pairwise_sum(const double* p, int64_t n) {
  if (n <= 64) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += p[i];
    return s;
  }
  const int64_t half = n / 2;
  return qo_pairwise_sum(p, half) + qo_pairwise_sum(p + half, n - half);
}

/* reduce_stats, proj/src/path_engine.cpp:191-205 */
void qo_reduce_stats(const double* values, int64_t n, double* mean_out, double* se_out) {
  const double sum = qo_pairwise_sum(values, n);
  const double mean = sum / (double)n;
  double se = 0.0;
  if (n >= 2) {
    double* sq = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) sq[i] = values[i] * values[i];
    const double sum_sq = qo_pairwise_sum(sq, n);
    free(sq);
    double var = (sum_sq - (double)n * mean * mean) / (double)(n - 1);
    if (var < 0.0) var = 0.0;
    se = sqrt(var / (double)n);
  }
  *mean_out = mean;
  *se_out = se;
}

/* QuasiStream::uniform_at for one dimension, proj/src/quasi_rng.cpp:85-101 */
int qo_uniform_dim(int64_t dims, int64_t n, uint64_t seed, int64_t dim, double* out, char* err,
                   int errlen) {
  if (dims < 1) return set_err(err, errlen, QO_INVALID_ARGUMENT, "QuasiStream: dimensions must be >= 1");
  if (n < 1) return set_err(err, errlen, QO_INVALID_ARGUMENT, "QuasiStream: length must be >= 1");
  uint32_t* primes = (uint32_t*)malloc((size_t)(dim + 1) * sizeof(uint32_t));
  qo_first_primes(dim + 1, primes);
  uint32_t* perm = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  int st = qo_permutation_indices(n, qo_dimension_seed(seed, dim), perm, err, errlen);
  if (st == QO_OK)
    for (int64_t p = 0; p < n; ++p) out[p] = qo_radical_inverse((uint64_t)perm[p] + 1, primes[dim]);
  free(perm);
  free(primes);
  return st;
}

/* sweep_impl, proj/src/american.cpp:32-68, generalised over the contract kind
 * (the reference instantiates it for calls only; the put branch is the opt-in
 * extension, parity UNPINNED against the reference -- see DESIGN.md). */
double qo_sweep_value(const double* path, int64_t m, const qo_spec* spec, int* status) {
  const double strike = spec->strike;
  const double dt = spec->maturity / (double)(m + 1); /* make_schedule, path_engine.cpp:67 */
  const double disc = exp(-spec->rate * dt);
  double value;
  {
    const double s = path[m - 1];
    qo_spec last = {s, strike, spec->rate, spec->volatility, dt, spec->kind};
    double cont;
    int st = qo_bs_price(&last, &cont, NULL, 0);
    if (st) { *status = st; return 0.0; }
    const double intr = intrinsic(spec->kind, s, strike);
    value = intr > cont ? intr : cont;
  }
  for (int64_t i = m - 1; i >= 1; --i) {
    const double s = path[i - 1];
    const double cont = value * disc;
    const double intr = intrinsic(spec->kind, s, strike);
    value = intr > cont ? intr : cont;
  }
  {
    const double cont = value * disc;
    const double intr = intrinsic(spec->kind, spec->spot, strike);
    value = intr > cont ? intr : cont;
  }
  *status = QO_OK;
  return value;
}

/* price_american, proj/src/american.cpp:103-131, with simulate_batch
 * (proj/src/path_engine.cpp:124-152) streamed one path at a time: every
 * per-path value is the same IEEE computation as the reference's, only the
 * [n][m+1] matrix is not materialised. check_capacity (path_engine.cpp:20-35)
 * is kept so error behaviour matches. */
int qo_price_american(const qo_spec* spec, int64_t m, int64_t n, uint64_t seed, uint32_t flags,
                      double* values, double* out, char* err, int errlen) {
  int st = qo_validate(spec, err, errlen);
  if (st) return st;
  if (spec->kind != QO_CALL && !(flags & QO_ALLOW_PUT))
    return set_err(err, errlen, QO_INVALID_ARGUMENT,
                   "price_american: not implemented for puts; the foresight algorithm is call-only");
  if (n < 2) return set_err(err, errlen, QO_INVALID_ARGUMENT, "price_american: n_paths must be >= 2");
  if (m < 1) return set_err(err, errlen, QO_INVALID_ARGUMENT, "make_schedule: m must be >= 1");
  if (!(spec->maturity > 0.0))
    return set_err(err, errlen, QO_INVALID_ARGUMENT, "make_schedule: maturity must be > 0");
  const double dt = spec->maturity / (double)(m + 1);
  const int64_t points = m + 1;
  {
    const unsigned __int128 bytes = (unsigned __int128)n * (unsigned __int128)points * 8u;
    if (bytes > ((unsigned __int128)1 << 37)) {
      char msg[256];
      snprintf(msg, sizeof msg,
               "simulate_batch: requested %lld paths x %lld points = %g bytes, above the "
               "supported maximum of %g bytes",
               (long long)n, (long long)points, (double)bytes, (double)((unsigned __int128)1 << 37));
      return set_err(err, errlen, QO_LENGTH_ERROR, msg);
    }
  }
  if ((uint64_t)n > 0xffffffffULL)
    return set_err(err, errlen, QO_LENGTH_ERROR,
                   "permutation_indices: n exceeds the 2^32-1 supported maximum");
  uint32_t* primes = (uint32_t*)malloc((size_t)points * sizeof(uint32_t));
  qo_first_primes(points, primes);
  uint32_t* perms = (uint32_t*)malloc((size_t)points * (size_t)n * sizeof(uint32_t));
  double* inv = (double*)malloc((size_t)points * sizeof(double));
  for (int64_t d = 0; d < points; ++d) {
    qo_permutation_indices(n, qo_dimension_seed(seed, d), perms + (size_t)d * (size_t)n, NULL, 0);
  }
  double* vals = values ? values : (double*)malloc((size_t)n * sizeof(double));
  double* row = (double*)malloc((size_t)points * sizeof(double));
  const double r = spec->rate, v = spec->volatility;
  st = QO_OK;
  for (int64_t p = 0; p < n && st == QO_OK; ++p) {
    double s = spec->spot;
    for (int64_t k = 0; k < points; ++k) {
      const double u = qo_radical_inverse((uint64_t)perms[(size_t)k * (size_t)n + (size_t)p] + 1,
                                          primes[k]);
      double z;
      qo_moro_inv_cnd(u, &z, NULL, 0); /* u is clamped into (0,1): never throws */
      /* gbm_step, proj/include/qmc/path_engine.hpp:51-56 */
      if (!(s > 0.0)) { st = set_err(err, errlen, QO_INVALID_ARGUMENT, "gbm_step: s_prev must be > 0"); break; }
      s = s * exp((r - 0.5 * v * v) * dt + v * sqrt(dt) * z);
      row[k] = s;
    }
    if (st) break;
    int sst;
    vals[p] = qo_sweep_value(row, m, spec, &sst);
    if (sst) {
      /* bs_price -> validate on the path's last exercise price */
      qo_spec last = {row[m - 1], spec->strike, spec->rate, spec->volatility, dt, spec->kind};
      st = qo_validate(&last, err, errlen);
      if (!st) st = set_err(err, errlen, QO_INVALID_ARGUMENT, "cnd: input must be finite");
    }
  }
  if (st == QO_OK) qo_reduce_stats(vals, n, &out[0], &out[1]);
  (void)inv;
  free(inv);
  free(row);
  if (!values) free(vals);
  free(perms);
  free(primes);
  return st;
}
