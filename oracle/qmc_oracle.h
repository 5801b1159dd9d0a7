/* Plain-C restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.
 * See qmc_oracle.c for the per-function reference citations. Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load this. */
#ifndef QMC_ORACLE_H
#define QMC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { QO_OK = 0, QO_INVALID_ARGUMENT = 1, QO_LENGTH_ERROR = 2 };
enum { QO_CALL = 0, QO_PUT = 1 };
/* flags for qo_price_american */
enum { QO_ALLOW_PUT = 1u };

typedef struct {
  double spot, strike, rate, volatility, maturity;
  int kind;
} qo_spec;

uint64_t qo_dimension_seed(uint64_t master_seed, int64_t dim);
void qo_first_primes(int64_t count, uint32_t* out);
int qo_permutation_indices(int64_t n, uint64_t seed, uint32_t* out, char* err, int errlen);
double qo_radical_inverse(uint64_t index, uint32_t base);
int qo_moro_inv_cnd(double u, double* out, char* err, int errlen);
int qo_cnd(double d, double* out, char* err, int errlen);
int qo_validate(const qo_spec* spec, char* err, int errlen);
int qo_bs_price(const qo_spec* spec, double* out, char* err, int errlen);
double qo_pairwise_sum(const double* p, int64_t n);
void qo_reduce_stats(const double* values, int64_t n, double* mean, double* std_error);
/* Uniforms of one dimension for all n paths (QuasiStream::uniform_at). */
int qo_uniform_dim(int64_t dims, int64_t n, uint64_t seed, int64_t dim, double* out, char* err,
                   int errlen);
/* Foresight sweep of one path of m+1 prices (sweep_impl); kind-generic. */
double qo_sweep_value(const double* path, int64_t m, const qo_spec* spec, int* status);
/* Per-path t0 values (length n) and the reduced price/se. values may be NULL. */
int qo_price_american(const qo_spec* spec, int64_t m, int64_t n, uint64_t seed, uint32_t flags,
                      double* values, double* out_price_se, char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
