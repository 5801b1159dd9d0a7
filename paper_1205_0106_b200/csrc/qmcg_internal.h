// Shared host/device declarations of the B200 pricer (not part of the public ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qmcg {

// Per-dimension (= per exercise date) constants for the scrambled Halton
// radical inverse (reference radical_inverse, proj/src/quasi_rng.cpp:71-83).
// Dimension d uses the d-th prime p; the index x = perm_d[path] + 1 has
// `ndig` base-p digits at most. Digit j contributes fl(digit * sc[j]) where
// sc[j] is the reference's rounded scale chain (1/p, fl(1/p * 1/p), ...), and
// fl(digit * sc[j]) is produced by one DFMA: fma(2^52 + digit, sc[j], nc[j])
// with nc[j] = -2^52 * sc[j] (exact: the FMA rounds d*sc[j] exactly once).
struct DimParam {
  uint32_t p;        // prime base
  uint32_t magic;    // q = umulhi(x, magic) >> shift == x / p for x <= n
  uint32_t shift;
  uint32_t ndig;     // digits to process (fixed count; high zero digits add +0.0)
  uint32_t doff;     // offset of this dimension's sc/nc entries
  uint32_t flags;    // DIM_CLAMP: endpoint clamp can trigger; DIM_WIDE: 64-bit magic
  uint64_t magic64;  // ceil(2^64 / p) for DIM_WIDE
};
enum : uint32_t { DIM_CLAMP = 1u, DIM_WIDE = 2u };

// Error bits raised by the pricing kernel (mapped to the reference's
// exception text on the host).
enum : uint32_t { ERR_SPOT_NONPOSITIVE = 1u, ERR_SPOT_NONFINITE = 2u };

struct PriceParams {
  const double* table;   // [m][ld] uniform-table slice: uniform_at(path, date), column = path - col_begin
  int64_t ld;            // row stride of the table
  int64_t col_begin;     // first path held by the table
  int64_t path_begin;    // first path of this launch
  int64_t path_count;    // paths in this launch
  int32_t m;             // exercise dates (dims used: 0..m-1)
  int32_t kind;          // 0 call, 1 put
  const double* dpow;    // dpow[k] = disc^k as the host's rounded chain, k = 0..m
  double X0;             // log(spot)
  double b;              // log-price scale: X_k = X0 + b * V_k
  double alpha;          // V_k = sum_{j<=k} (z_j + alpha)
  double c0;             // initial candidate threshold in V units
  double strike;
  double best0;          // intrinsic value at t0 (date 0 term)
  double log_strike;
  double dmax_inv;       // 1 / max_k disc^k  (only for rate < 0)
  double dom_slope;      // per-date step of the dominance accumulator: calls r*dt/b, puts r*dt
  double x0mk;           // 1 + X0 - log K (put dominance test)
  // Black-Scholes of the last interval (reference sweep_impl, american.cpp:45-52)
  double bs_vsqrt;       // v*sqrt(dt)
  double bs_mu_t;        // (r + 0.5*v*v)*dt
  double bs_kdisc;       // K * exp(-r*dt)
  double bs_fwd_growth;  // exp(r*dt)            (v == 0 branch)
  double bs_disc;        // exp(-r*dt)           (v == 0 branch)
  int32_t bs_v_zero;
  int32_t deterministic; // volatility == 0: z never affects the path
  int32_t check_range;   // per-date overflow/underflow checks needed
  int32_t rate_negative; // disc > 1: running-max filter invalid, use best-based filter
  int32_t fp32;          // QMCG_FLAG_FP32: single-precision normals and walk
  // Date window of this launch (streamed tables: the permutation rows of
  // dates [d_begin, d_end) only, row index d - perm_row0). Resident: [0, m), 0.
  int32_t d_begin, d_end, perm_row0;
  int32_t stream_load;   // carry-in: walk state read from st_* (window > first)
  int32_t stream_store;  // carry-out: walk state written to st_* (window < last)
  int32_t pad0;
  double* st_V;          // per path (index = path - path_begin): log-price walk V
  double* st_c;          // last record
  double* st_cd;         // dominance accumulator of the pending record
  double* st_best;       // best evaluated discounted intrinsic so far
  int32_t* st_pend;      // date of the pending record (-1 none)
  double* values;        // per-path t0 values, index = path - path_begin
  uint32_t* err;
};

// Per-contract constants of a batch walk (same meaning as in PriceParams).
struct ContractParams {
  const double* dpow;
  double X0, b, alpha, c0, strike, best0, log_strike, dom_slope;
  double bs_vsqrt, bs_mu_t, bs_kdisc, bs_fwd_growth, bs_disc;
  double x0mk;
  double bs_inv_kdisc;  // 1 / bs_kdisc (the batch's one-exp final interval)
  int32_t bs_v_zero, pad;
};

// Batch pricing over a shared normal table z[m][ldz] (z = Moro normal, no drift).
// A batch group: contracts of one kind sharing (spot, rate, volatility,
// maturity) -- hence the same log-price walk -- and differing in the strike.
struct GroupParams {
  const double* dpow;
  double X0, b, alpha;
  double beta;     // calls: alpha - dom_slope (dominance key slope); puts: dom_slope (accumulator step)
  double c0;       // union start threshold: calls min over strikes, puts max
  double x0mk;     // puts: 1 + X0 - log(max strike) (dominance for every strike of the group)
  double bs_vsqrt, bs_mu_t, bs_fwd_growth, bs_disc;
  int32_t bs_v_zero, first, count, pad;  // contracts [first, first + count) of the kind's array
};

struct BatchParams {
  const double* z;
  int64_t ldz;
  int64_t n;                  // paths
  int32_t m;                  // dates
  int32_t count;              // contracts in this launch (all of one kind)
  const ContractParams* cp;   // count entries
  double* values;             // [count][n]
  const GroupParams* groups;      // grouped walk: one walk per (group, path)
  int32_t n_groups, pad;
};

// ---- launchers (kernels.cu) ----
// Generation only: the QMC normal table z[d][p] (d < m, p in [path_begin, +path_count)) from the
// context's uniform table (PriceParams fields table/ld/col_begin/perm_row0/d_begin/d_end; + alpha).
cudaError_t launch_walk_group(const BatchParams& B, int kind, cudaStream_t s);  // the batch walk reads prefix sums S (gen_z prefix mode)
// mode: kGenZ (normals), kGenPrefix (per-path running sums of the normals, the batch walk's input),
enum : int { kGenZ = 0, kGenPrefix = 1 };
cudaError_t launch_gen_z(const PriceParams& P, double* z, int64_t ldz, cudaStream_t s, int mode = kGenZ);
cudaError_t launch_european(const double* urow, int64_t count, double s0, double a, double bsd, double strike,
                            double disc, int kind, double* out, cudaStream_t s);
// Pairwise sums of `count` contiguous vectors v[c*len .. (c+1)*len) into out2[2c, 2c+1].
cudaError_t launch_pairwise_batched(const double* v, int64_t len, int count, double* scratch, double* out2,
                                    cudaStream_t s, int* launches);
cudaError_t launch_price(const PriceParams& P, cudaStream_t s);
// K1: Fisher-Yates permutation of length n for LCG seed `seed64` into out[0..n).
// scratch must hold perm_scratch_bytes(n) bytes.
size_t perm_scratch_bytes(int64_t n);
cudaError_t launch_path_matrix(const double* table, int64_t ld, int64_t n, int points, double s0, double a,
                               double bsd, double* out, uint32_t* err, cudaStream_t s);
cudaError_t launch_transpose(const double* in, int64_t rows, int64_t cols, double* out, cudaStream_t s);
cudaError_t launch_sweep(const double* prices, int64_t n, int m, double spot, double strike, double rate, double vol,
                         double dt, double disc, int kind, double* values, int32_t* exercise, cudaStream_t s);
cudaError_t launch_perm_build(uint64_t seed64, int64_t n, uint32_t* out, void* scratch,
                              size_t scratch_bytes, cudaStream_t s, int* launches, uint32_t add);
// uniform_at (or, with `normals`, normal_at) of `count` table entries perm + 1 of one dimension:
// radical_inverse with the reference's rounding (bit-exact). Builds the rows of the uniform table
// from K1's permutations (normals = 0) and serves the D1 exports.
cudaError_t launch_uniforms(const uint32_t* perm_row, int64_t count, DimParam dp, const double* sc,
                            const double* nc, int normals, double* out, cudaStream_t s);
// Row stride (in paths) of the uniform table: padded to 64 entries so every row starts 512-byte
// aligned (the TMA tile copies of K2 need 16).
inline int64_t table_ld(int64_t cols) { return (cols + 63) / 64 * 64; }
// Extra elements allocated after the last row (bulk copies of a partial block
// may read up to one block past the end of a row).
constexpr int64_t kTablePad = 256;
// DFMA throughput probe: blocks x 256 threads x iters x 128 independent DFMAs.
cudaError_t launch_dfma_probe(double* out, int blocks, int iters, cudaStream_t s);
// Pairwise-tree sums of v and v*v over `len` values (reference pairwise_sum
// with 64-element leaves). out2[0] = sum, out2[1] = sum of squares.
size_t reduce_scratch_doubles(int64_t len);
cudaError_t launch_pairwise(const double* v, int64_t len, double* scratch, double* out2,
                            cudaStream_t s, int* launches);

}  // namespace qmcg
