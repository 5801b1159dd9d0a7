/* qmcg.h -- C ABI of the B200-native American-option QMC pricer.
 *
 * This is the drop-in boundary for the reference's hot path
 *   qmc::price_american            (reference proj/include/qmc/american.hpp:46-47,
 *                                   proj/src/american.cpp:103-131)
 * and everything it calls (QuasiStream / permutation_indices / radical_inverse,
 * moro_inv_cnd, gbm_step, simulate_batch, sweep_impl, reduce_stats).
 * Plain C types only: POD structs, pointers and sizes; no CUDA or torch types.
 * The C++ drop-in with the reference's exact signature is include/qmc_b200/qmc.hpp;
 * the ctypes binding used by the tests and bench.py is paper_1205_0106_b200/qmcg.py;
 * INTEGRATION.md shows how a reference build links against this library.
 *
 * Error convention: every entry returns a qmcg_status; on failure the message
 * (the reference's own exception text where one exists) is available from
 * qmcg_last_error() on the calling thread. QMCG_INVALID_ARGUMENT maps to the
 * reference's std::invalid_argument, QMCG_LENGTH_ERROR to std::length_error.
 *
 * Threading: calls on one context are serialised by a context mutex; distinct
 * contexts may be used concurrently (one per GPU is the intended layout).
 */
#ifndef QMCG_H
#define QMCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QMCG_OK = 0,
  QMCG_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  QMCG_LENGTH_ERROR = 2,     /* reference: std::length_error */
  QMCG_CUDA_ERROR = 3,
  QMCG_NCCL_ERROR = 4,
  QMCG_UNSUPPORTED = 5,
  QMCG_OUT_OF_MEMORY = 6
} qmcg_status;

/* reference OptionKind, proj/include/qmc/types.hpp:16 */
enum { QMCG_CALL = 0, QMCG_PUT = 1 };
/* reference Method, proj/include/qmc/types.hpp:18 */
enum { QMCG_METHOD_CLOSED_FORM = 0, QMCG_METHOD_EUROPEAN_MC = 1, QMCG_METHOD_AMERICAN_UB = 2 };

/* flags */
enum {
  QMCG_FLAG_ALLOW_PUT = 1u << 0, /* opt-in put extension (reference rejects puts: american.cpp:106-109) */
  QMCG_FLAG_NO_CACHE = 1u << 1,  /* rebuild the uniform tables for this call (cold timing) */
  QMCG_FLAG_FP32 = 1u << 2,      /* FP32 normals + walk (uniforms stay bit-exact FP64); price within QMC error */
};

/* reference OptionSpec, proj/include/qmc/types.hpp:24-31 */
typedef struct {
  double spot;
  double strike;
  double rate;
  double volatility;
  double maturity;
  int32_t kind; /* QMCG_CALL / QMCG_PUT */
} qmcg_option_spec;

/* reference PricingResult, proj/include/qmc/types.hpp:42-49 */
typedef struct {
  double price;
  double std_error;
  int64_t n_paths;
  double elapsed_s; /* wall time of the whole call, like american.cpp:113,127-128 */
  int32_t method;   /* QMCG_METHOD_* */
  uint64_t seed;
} qmcg_pricing_result;

typedef struct qmcg_ctx qmcg_ctx;

/* Context on one CUDA device: owns the stream, scratch and the uniform-table
 * cache keyed by (seed, n_paths). */
qmcg_status qmcg_create(int device, qmcg_ctx** out);
/* Context over a device group (one process, n_dev listed CUDA devices; a device may be listed
 * more than once). It replaces the reference's host thread pool (ExecPolicy lanes,
 * proj/src/path_engine.cpp:83-122, and the fork-join reduction :51-59) at the GPU level:
 * qmcg_price_american shards the paths as whole pairwise-tree nodes over the members (member r
 * owns a contiguous column slice of the uniform tables), each member reduces its nodes and
 * the host folds the 16-byte node sums with the reference's tree, so results are bit-identical
 * to one device for any member count. Cold tables are built dimension-sharded (dim d on member
 * d mod n_dev) and column slices copied peer to peer; tables larger than memory are streamed in
 * date windows the same way. qmcg_price_american_batch shards contracts. Every other call runs on
 * the first member; the per-device node / table-exchange calls return QMCG_UNSUPPORTED. */
qmcg_status qmcg_create_multi(const int* dev_ids, int n_dev, qmcg_ctx** out);
/* The context the C++ drop-in uses: every visible CUDA device (a device group when there are
 * several), or the comma-separated list in the environment variable QMCG_DEVICES. */
qmcg_status qmcg_create_default(qmcg_ctx** out);
/* Number of devices a context drives (1 for qmcg_create). */
int qmcg_device_count(qmcg_ctx* ctx);
void qmcg_destroy(qmcg_ctx* ctx);
const char* qmcg_last_error(void);
const char* qmcg_version(void);

/* qmc::price_american (proj/src/american.cpp:103-131): foresight upper-bound
 * American price over n_paths scrambled-Halton GBM paths with m exercise dates.
 * Identical validation and error text as the reference. */
qmcg_status qmcg_price_american(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m,
                                int64_t n_paths, uint64_t seed, uint32_t flags,
                                qmcg_pricing_result* out);

/* qmc::mc_european_price (proj/src/mc_european.cpp:11-46): one-step QMC
 * European price from the dimension-0 scrambled-Halton normals (puts allowed,
 * as in the reference); volatility 0 or maturity 0 returns the discounted
 * deterministic payoff exactly. method = QMCG_METHOD_EUROPEAN_MC. */
qmcg_status qmcg_mc_european_price(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t n_paths, uint64_t seed,
                                   uint32_t flags, qmcg_pricing_result* out);

/* The same pricing for n_specs contracts sharing (m, n_paths, seed): one
 * permutation-table set, one launch per contract group. No reference
 * counterpart (the reference loops price_american). */
qmcg_status qmcg_price_american_batch(qmcg_ctx* ctx, const qmcg_option_spec* specs,
                                      int64_t n_specs, int64_t m, int64_t n_paths, uint64_t seed,
                                      uint32_t flags, qmcg_pricing_result* out);

/* The same batch, also returning every contract's per-path t0 values (values_host[i * n_paths + p],
 * contract i in the caller's order) from the same launches (parity export: the batch's fused
 * tree must equal the reference's reduce_stats of these values). */
qmcg_status qmcg_price_american_batch_values(qmcg_ctx* ctx, const qmcg_option_spec* specs,
                                             int64_t n_specs, int64_t m, int64_t n_paths, uint64_t seed,
                                             uint32_t flags, qmcg_pricing_result* out, double* values_host);

/* Sharded pricing for multi-GPU: computes (sum v, sum v^2) of the pairwise
 * tree node `node` at depth `depth` (reference pairwise_sum,
 * proj/src/path_engine.cpp:39-47), over the paths of that node only. Nodes at
 * one depth partition [0, n_paths). Combining all 2^depth node sums with
 * qmcg_combine_nodes gives bit-identical results for every depth. */
qmcg_status qmcg_price_american_node(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m,
                                     int64_t n_paths, uint64_t seed, uint32_t flags, int depth,
                                     int64_t node, double out_sums[2]);
/* The same for `node_count` consecutive nodes [node_begin, node_begin + node_count) at
 * `depth` in one pass (one kernel over their contiguous path range, one cached table
 * slice): out_sums[2k], out_sums[2k+1] = (sum v, sum v^2) of node node_begin + k. A rank
 * of a multi-GPU job calls this once for all the nodes it owns. */
qmcg_status qmcg_price_american_nodes(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m,
                                      int64_t n_paths, uint64_t seed, uint32_t flags, int depth,
                                      int64_t node_begin, int64_t node_count, double* out_sums);
/* Path range [begin, end) of pairwise-tree node `node` at `depth`. */
qmcg_status qmcg_tree_node_range(int64_t n_paths, int depth, int64_t node, int64_t* begin,
                                 int64_t* end);
/* Fold 2^depth node sums (interleaved sum, sum_sq) up the tree and apply
 * reduce_stats' mean / Bessel standard error (path_engine.cpp:191-205). */
qmcg_status qmcg_combine_nodes(int64_t n_paths, int depth, const double* node_sums,
                               double* price, double* std_error);

/* Build (or extend) the cached uniform tables (K1 permutations -> uniform_at, f64) for dims [0, dims). */
qmcg_status qmcg_warm(qmcg_ctx* ctx, int64_t n_paths, uint64_t seed, int64_t dims);
/* Drop every cached table. */
qmcg_status qmcg_clear_cache(qmcg_ctx* ctx);
/* Cold multi-GPU build: rank r builds the full tables of dims
 * dim_begin + k * dim_stride (k < count) into its device buffer out_dev (row k at
 * out_dev + k * ld; entries are perm + 1, the Halton index of uniform_at), the column
 * slices are exchanged all-to-all, and each rank installs its slice of every dim
 * with qmcg_import_tables. src_dev holds dims rows of col_end - col_begin entries
 * (row stride src_ld); afterwards pricing over [col_begin, col_end) is warm. */
qmcg_status qmcg_build_tables(qmcg_ctx* ctx, int64_t n_paths, uint64_t seed, int64_t dim_begin,
                              int64_t dim_stride, int64_t count, uint32_t* out_dev, int64_t ld);
qmcg_status qmcg_import_tables(qmcg_ctx* ctx, int64_t n_paths, uint64_t seed, int64_t col_begin,
                               int64_t col_end, int64_t dims, const uint32_t* src_dev, int64_t src_ld);
/* The same row block by row block: rows [row_begin, row_begin + row_count) of the slice of dims
 * [0, dims) (src_dev holds row_count rows, stride src_ld). row_begin = 0 starts a fresh slice
 * table sized for `dims` rows; each later call continues where the previous one stopped, so a
 * rank can exchange and install the tables a chunk of dims at a time (config 5: 1 GiB per dim).
 * Pricing of up to row_begin + row_count dates is warm after each call. */
qmcg_status qmcg_import_rows(qmcg_ctx* ctx, int64_t n_paths, uint64_t seed, int64_t col_begin,
                             int64_t col_end, int64_t dims, int64_t row_begin, int64_t row_count,
                             const uint32_t* src_dev, int64_t src_ld);
/* Cap the bytes the uniform tables may occupy (0 = whatever free device
 * memory allows). A pricing whose tables exceed it runs in date windows
 * ("streamed tables": each window's rows are built, walked, and replaced,
 * with the per-path walk state carried in HBM) with identical results; this
 * is how 2^28 paths x 365 dates (392 GB of tables) prices on one GPU. No
 * reference counterpart: the reference caps its path matrix at 128 GiB
 * (proj/src/path_engine.cpp:20-35). */
qmcg_status qmcg_set_table_budget(qmcg_ctx* ctx, uint64_t bytes);
/* Date windows the last pricing call used (1 = resident tables). */
int64_t qmcg_last_window_count(qmcg_ctx* ctx);

/* ---- parity exports (bit-exact checks against the reference) ---- */
/* permutation_indices(n, seed64) (proj/src/quasi_rng.cpp:48-61), built on the GPU. */
qmcg_status qmcg_permutation(qmcg_ctx* ctx, int64_t n, uint64_t seed64, uint32_t* out_host);
/* QuasiStream(dims>dim, n, seed).uniform_at(p, dim) for all p (quasi_rng.cpp:96-101). */
qmcg_status qmcg_uniforms(qmcg_ctx* ctx, int64_t n, uint64_t seed, int64_t dim, double* out_host);
/* moro_inv_cnd of the same uniforms (quasi_rng.cpp:103-105), as the pricing kernel computes it. */
qmcg_status qmcg_normals(qmcg_ctx* ctx, int64_t n, uint64_t seed, int64_t dim, double* out_host);
/* The normal table z[d][p] = moro_inv_cnd(uniform_at(p, d)) for d < dims, as the batch
 * path generates it (row-major [dims][n_paths]). */
qmcg_status qmcg_normal_table(qmcg_ctx* ctx, int64_t n_paths, uint64_t seed, int64_t dims, double* out_host);
/* uniform_at(p, d) (quasi_rng.cpp:96-101) for d in [dim_begin, dim_begin + dim_count) and all p,
 * produced by the pricing kernels' own generator code (generate_row: per-date fixed digit counts,
 * digit pairs, the base-2 bit reversal) rather than the D1 export: row-major [dim_count][n_paths]. */
qmcg_status qmcg_uniform_rows(qmcg_ctx* ctx, int64_t n_paths, uint64_t seed, int64_t dim_begin,
                              int64_t dim_count, double* out_host);
/* Per-path t0 values of the foresight sweep (american.cpp:119-124). */
qmcg_status qmcg_path_values(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m,
                             int64_t n_paths, uint64_t seed, uint32_t flags, double* out_host);

/* ---- path matrix and sweeps (diagnostics; the pricing kernels never store paths) ---- */
enum { QMCG_LAYOUT_PATH_MAJOR = 0, /* prices[p * (m+1) + k]: reference PathBatch::prices (row-major) */
       QMCG_LAYOUT_POINT_MAJOR = 1 /* prices[k * n + p]: the device layout */ };
/* simulate_batch(spec, make_schedule(m, T), n_paths, seed) (proj/src/path_engine.cpp:124-152):
 * S at t_1..t_m, T for every path, generated on the GPU from the same tables as the pricer.
 * Errors as the reference (make_schedule, validate, n_paths >= 1, check_capacity's 128 GiB
 * length_error with the computed size, gbm_step's s_prev > 0). out_host == NULL only validates
 * (ctx may then be NULL too), so a caller can size its buffer after the reference's checks. */
qmcg_status qmcg_simulate_batch(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m,
                                int64_t n_paths, uint64_t seed, uint32_t flags, int layout,
                                double* out_host);
/* sweep_value and the earliest exercise point of backward_sweep (american.cpp:19-101) for
 * every simulated path, on the GPU over the point-major matrix: values_host[p] = t_0 value,
 * exercise_host[p] = earliest index in 0..m where intrinsic beat continuation, -1 if never. */
qmcg_status qmcg_sweep_batch(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m,
                             int64_t n_paths, uint64_t seed, uint32_t flags, double* values_host,
                             int32_t* exercise_host);
/* backward_sweep(path, spec, make_schedule(m, T)) for one caller-provided path (host; the
 * reference's per-path diagnostic, american.cpp:88-95): values_out[0..m] = value at t_0..t_m,
 * values_out[m+1] = realised payoff at T; *exercise_point = earliest exercise index or -1.
 * path holds m+1 prices (t_1..t_m, T). */
qmcg_status qmcg_backward_sweep(const double* path, int64_t path_len, const qmcg_option_spec* spec,
                                int64_t m, uint32_t flags, double* values_out,
                                int64_t* exercise_point);

/* ---- measurement hooks (bench.py) ---- */
/* Launch the pricing of `spec` reps times on the context stream with the
 * tables resident, and report the device time of the pricing kernel alone and
 * of the whole device step (CUDA events on the launching stream), in ms. */
qmcg_status qmcg_time_device(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m,
                             int64_t n_paths, uint64_t seed, uint32_t flags, int reps,
                             double* kernel_ms, double* step_ms, double* out_price_se);
/* The same for the tree nodes [node_begin, node_begin + node_count) at `depth` (the range a rank of
 * a multi-GPU job prices with qmcg_price_american_nodes); out_sums as there. */
qmcg_status qmcg_time_device_nodes(qmcg_ctx* ctx, const qmcg_option_spec* spec, int64_t m, int64_t n_paths,
                                   uint64_t seed, uint32_t flags, int depth, int64_t node_begin,
                                   int64_t node_count, int reps, double* kernel_ms, double* step_ms,
                                   double* out_sums);
/* Device time (ms) of rebuilding the uniform tables (K1 + conversion) for dims [0, dims). */
qmcg_status qmcg_time_perm_build(qmcg_ctx* ctx, int64_t n_paths, uint64_t seed, int64_t dims,
                                 double* ms);
/* Out-of-bounds write check (the process must run with QMCG_CANARY=1 from its first allocation):
 * every device buffer of every context is bracketed by 4 KB guard regions; this verifies them
 * all and names the first clobbered one. QMCG_UNSUPPORTED without QMCG_CANARY=1. */
qmcg_status qmcg_check_canaries(void);
/* Number of kernels the last qmcg_price_american* call launched. */
int64_t qmcg_last_launch_count(qmcg_ctx* ctx);
/* The context's CUDA stream (a cudaStream_t) so a caller can record its own
 * events around a sequence of calls. */
void* qmcg_get_stream(qmcg_ctx* ctx);
/* The CUDA stream and device of member `member` of a device group (member 0 of a single-device
 * context), for events around a sequence of group calls; NULL / -1 if out of range. */
void* qmcg_get_member_stream(qmcg_ctx* ctx, int member);
int qmcg_member_device(qmcg_ctx* ctx, int member);
/* Measured FP64 FMA issue rate of this device (instructions/s), from a
 * dependent-chain-free DFMA kernel run for about `ms` milliseconds. */
qmcg_status qmcg_fp64_peak(qmcg_ctx* ctx, double ms, double* inst_per_s);

#ifdef __cplusplus
}
#endif
#endif /* QMCG_H */
