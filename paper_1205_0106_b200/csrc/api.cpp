// Host side of the B200 pricer: context, permutation-table cache, host
// precompute of the exact per-dimension constants, and the C ABI (qmcg.h).
//
// Host arithmetic that feeds bit-exact device results (the radical-inverse
// scale chains 1/p, (1/p)^k) and the per-call constants (dt, drift, diffusion,
// discount) is done here in IEEE double with glibc, compiled with
// -ffp-contract=off, in the reference's operation order.
#include "qmcg.h"
#include "qmcg_internal.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <condition_variable>
#include <functional>
#include <memory>
#include <thread>
#include <unordered_map>
#include <vector>

using qmcg::DimParam;
using qmcg::PriceParams;

namespace {

thread_local std::string g_last_error;

qmcg_status fail(qmcg_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define QMCG_CUDA(expr)                                                                       \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      if (e_ == cudaErrorMemoryAllocation) {                                                  \
        cudaGetLastError();                                                                   \
        return fail(QMCG_OUT_OF_MEMORY, std::string("CUDA out of memory at ") + #expr);       \
      }                                                                                       \
      return fail(QMCG_CUDA_ERROR, std::string("CUDA error ") + cudaGetErrorString(e_) +      \
                                       " at " + #expr);                                       \
    }                                                                                         \
  } while (0)

// ---- reference helpers restated for the host precompute ----

// splitmix64 / dimension_seed, reference proj/src/quasi_rng.cpp:16-22,41-46
uint64_t splitmix64(uint64_t& state) {
  state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t dimension_seed(uint64_t master, int64_t dim) {
  uint64_t state = master;
  const uint64_t mixed = splitmix64(state);
  state = mixed ^ (static_cast<uint64_t>(dim) + 0x632be59bd9b4e019ULL);
  return splitmix64(state);
}

// first_primes, quasi_rng.cpp:24-37 (extended incrementally)
const std::vector<uint32_t>& primes_upto_count(int64_t count) {
  static std::vector<uint32_t> primes;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  uint32_t cand = primes.empty() ? 2 : primes.back() + 1;
  while (static_cast<int64_t>(primes.size()) < count) {
    bool is_prime = true;
    for (uint32_t d = 2; d * d <= cand; ++d)
      if (cand % d == 0) {
        is_prime = false;
        break;
      }
    if (is_prime) primes.push_back(cand);
    ++cand;
  }
  return primes;
}

// validate, reference proj/src/analytic.cpp:18-31
qmcg_status validate(const qmcg_option_spec& s) {
  if (!std::isfinite(s.spot) || !std::isfinite(s.strike) || !std::isfinite(s.rate) ||
      !std::isfinite(s.volatility) || !std::isfinite(s.maturity))
    return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: all fields must be finite");
  if (!(s.spot > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: spot must be > 0");
  if (!(s.strike > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: strike must be > 0");
  if (!(s.volatility >= 0.0)) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: volatility must be >= 0");
  if (!(s.maturity >= 0.0)) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: maturity must be >= 0");
  if (s.kind != QMCG_CALL && s.kind != QMCG_PUT) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: unknown kind");
  return QMCG_OK;
}

// QMCG_TRACE=1: per-call host phase times on stderr (wall clock, microseconds).
struct Trace {
  const char* what;
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  explicit Trace(const char* w) : what(w) {
    const char* e = std::getenv("QMCG_TRACE");
    on = e && *e && *e != '0';
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* phase) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[qmcg trace] %s %-18s %9.1f us (total %9.1f)\n", what, phase,
                 std::chrono::duration<double, std::micro>(now - last).count(),
                 std::chrono::duration<double, std::micro>(now - t0).count());
    last = now;
  }
};

// NVTX phase ranges (header-only NVTX 3: no-ops unless a profiler injects itself), named after
// the kernels of DESIGN.md 3: K1 table builds, K2 pricing, K3 tree, group exchange, batches.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

uint64_t bits_of(double x) {
  uint64_t u;
  std::memcpy(&u, &x, sizeof u);
  return u;
}

double intrinsic(int kind, double s, double k) {
  const double diff = kind == QMCG_CALL ? s - k : k - s;
  return diff > 0.0 ? diff : 0.0;
}

// Node range of the pairwise tree (reference pairwise_sum splits at n/2).
void tree_node(int64_t n, int depth, int64_t node, int64_t& off, int64_t& size) {
  off = 0;
  size = n;
  for (int l = depth - 1; l >= 0; --l) {
    const int64_t half = size / 2;
    if ((node >> l) & 1) {
      off += half;
      size -= half;
    } else {
      size = half;
    }
  }
}

// Dimension tables for (n, m): exact digit constants per prime.
struct DimTables {
  int64_t n = -1, m = -1;
  std::vector<DimParam> dims;
  std::vector<double> sc, nc;
};

void build_dim_tables(int64_t n, int64_t m, DimTables& T) {
  const auto& primes = primes_upto_count(m);
  // test knob: QMCG_FORCE_WIDE=1 takes the 64-bit-magic digit division and the endpoint clamp on
  // every dimension (otherwise reached only near n = 2^32), so tests can check them bit for bit
  // against the 32-bit magic at small n
  const char* fw = std::getenv("QMCG_FORCE_WIDE");
  const bool force_wide = fw && *fw && *fw != '0';
  T.dims.resize(static_cast<size_t>(m));
  T.sc.clear();
  T.nc.clear();
  const uint64_t max_index = static_cast<uint64_t>(n);  // perm + 1 <= n
  for (int64_t d = 0; d < m; ++d) {
    const uint32_t p = primes[static_cast<size_t>(d)];
    DimParam dp{};
    dp.p = p;
    // digits: smallest D with p^D > max_index
    uint32_t D = 1;
    unsigned __int128 pw = p;
    while (pw <= max_index) {
      pw *= p;
      ++D;
    }
    dp.ndig = D;
    dp.doff = static_cast<uint32_t>(T.sc.size());
    // scale chain exactly as radical_inverse: scale = 1/b; scale *= 1/b ...
    const double inv_base = 1.0 / p;
    double scale = inv_base;
    for (uint32_t j = 0; j < D; ++j) {
      T.sc.push_back(scale);
      T.nc.push_back(-4503599627370496.0 * scale);  // -2^52 * scale, exact
      scale *= inv_base;
    }
    // clamp can only trigger when p^-D approaches kEndpointEps
    if (T.sc.back() < 2e-12 || force_wide) dp.flags |= qmcg::DIM_CLAMP;
    // magic division, exact for x <= max_index (< 2^32)
    uint32_t sh = 0;
    while ((uint64_t{1} << (sh + 1)) < p) ++sh;  // sh = ceil(log2 p) - 1
    const unsigned __int128 two = static_cast<unsigned __int128>(1) << (32 + sh);
    const unsigned __int128 M = (two + p - 1) / p;
    const unsigned __int128 e = M * p - two;
    if (!force_wide && M < (static_cast<unsigned __int128>(1) << 32) &&
        static_cast<unsigned __int128>(max_index) * e < two) {
      dp.magic = static_cast<uint32_t>(M);
      dp.shift = sh;
    } else {
      dp.flags |= qmcg::DIM_WIDE;
      const unsigned __int128 two64 = static_cast<unsigned __int128>(1) << 64;
      dp.magic64 = static_cast<uint64_t>((two64 + p - 1) / p);
    }
    T.dims[static_cast<size_t>(d)] = dp;
  }
  T.n = n;
  T.m = m;
}

// Device allocations of the context. With QMCG_CANARY=1 in the environment (the out-of-bounds
// write check; compute-sanitizer is closed on this pool) every allocation is bracketed by 4 KB
// guard regions filled with 0xA5, registered, and qmcg_check_canaries() verifies them after the
// kernels ran: any K1-K4 write past either end of a buffer (the permutation tables, values,
// scratch, walk state) shows up as a clobbered guard.
constexpr size_t kGuard = 4096;
struct Guarded {
  char* base;
  size_t bytes;
  int device;
};
std::mutex g_alloc_mu;
std::vector<std::pair<void*, Guarded>>& guarded_allocs() {
  static std::vector<std::pair<void*, Guarded>> v;
  return v;
}
bool canary_mode() {
  static const bool on = [] {
    const char* e = std::getenv("QMCG_CANARY");
    return e && *e && *e != '0';
  }();
  return on;
}

cudaError_t dev_alloc(void** p, size_t bytes) {
  if (!canary_mode()) return cudaMalloc(p, bytes);
  char* base = nullptr;
  cudaError_t e = cudaMalloc(&base, bytes + 2 * kGuard);
  if (e != cudaSuccess) return e;
  e = cudaMemset(base, 0xA5, kGuard);
  if (e == cudaSuccess) e = cudaMemset(base + kGuard + bytes, 0xA5, kGuard);
  if (e != cudaSuccess) {
    cudaFree(base);
    return e;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  *p = base + kGuard;
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  guarded_allocs().push_back({*p, Guarded{base, bytes, dev}});
  return cudaSuccess;
}

void dev_free(void* p) {
  if (!p) return;
  if (!canary_mode()) {
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  auto& v = guarded_allocs();
  for (size_t i = 0; i < v.size(); ++i)
    if (v[i].first == p) {
      cudaFree(v[i].second.base);
      v.erase(v.begin() + static_cast<std::ptrdiff_t>(i));
      return;
    }
  cudaFree(p);
}

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  cudaError_t reserve(size_t count) {
    if (count <= cap) return cudaSuccess;
    dev_free(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = dev_alloc(reinterpret_cast<void**>(&ptr), std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) cap = count;
    return e;
  }
  void release() {
    dev_free(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

// One persistent host thread per device-group member: the warm group pricing enqueues and waits on
// every member concurrently (a member's host work -- plan upload, tensor-map encode, launches -- is
// ~50-80 us; done one member after another it would stagger the devices' start by that much each).
class MemberWorker {
 public:
  MemberWorker() : th_([this] { loop(); }) {}
  ~MemberWorker() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void submit(std::function<void()> job) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      job_ = std::move(job);
      busy_ = true;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lock(mu_);
    cv_.wait(lock, [this] { return !busy_; });
  }

 private:
  void loop() {
    std::unique_lock<std::mutex> lock(mu_);
    for (;;) {
      cv_.wait(lock, [this] { return stop_ || busy_; });
      if (stop_) return;
      auto job = std::move(job_);
      lock.unlock();
      job();
      lock.lock();
      busy_ = false;
      cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::function<void()> job_;
  bool busy_ = false, stop_ = false;
  std::thread th_;
};

}  // namespace

struct qmcg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  // permutation-table cache: rows [0, dims) of columns [col_begin, col_end)
  uint64_t cache_seed = 0;
  int64_t cache_n = -1, col_begin = 0, col_end = 0, cache_dims = 0;
  double* table = nullptr;  // the uniform table: uniform_at(path, dim) of rows [0, cache_dims), f64
  size_t table_rows_cap = 0;
  // host-side dimension constants mirrored on the device
  DimTables dt;
  DevBuf<double> d_path, d_path_t;   // path matrix [point][path] (+ path-major transpose)
  DevBuf<int32_t> d_ex;              // per-path exercise points
  DevBuf<double> d_sc, d_nc, d_dpow;
  std::vector<double> dpow_host;  // what d_dpow holds for single-contract calls (skips the re-upload)
  DevBuf<double> d_values, d_red, d_sums;
  DevBuf<double> d_z;                                // batch: shared normal (prefix-sum) table
  DevBuf<double> d_bvalues[2], d_bred[2], d_bsums[2];  // per kind: per-contract values, scratch, sums
  DevBuf<qmcg::ContractParams> d_cparams[2];
  DevBuf<qmcg::GroupParams> d_groups[2];
  DevBuf<uint32_t> d_err, d_fullperm;
  DevBuf<char> d_permscratch;
  // second K1 lane: tables built alternately on `stream` and `side` so one table's latency-bound
  // chase pass overlaps the next table's sort (n <= kOverlapMaxN)
  cudaStream_t side[2] = {nullptr, nullptr};
  DevBuf<char> d_permscratch_side[2];
  DevBuf<uint32_t> d_xrow_side[2];  // the side lanes' rows of perm + 1 on their way into the uniform table
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
  // streamed tables (date windows): per-path walk state carried between windows
  DevBuf<double> d_stV, d_stc, d_stcd, d_stbest;
  DevBuf<int32_t> d_stpend;
  size_t table_budget = 0;  // bytes the permutation table may take; 0 = what free memory allows
  // device group (qmcg_create_multi): members[r] is the context of the r-th listed device; the
  // group handle owns them and dispatches (its own stream, cache and scratch stay unused)
  std::vector<qmcg_ctx*> members;
  std::vector<std::unique_ptr<MemberWorker>> workers;       // one host thread per member (warm pricing)
  DevBuf<double> d_gtmp;                                    // builder rows of a group table build
  cudaEvent_t ev_built = nullptr, ev_priced = nullptr;      // cross-member ordering of group builds
  int64_t last_windows = 0;  // date windows of the last pricing (1 = resident tables)
  double* h_pinned = nullptr;  // [0..1] sums, [2] err as double bits
  double* h_res = nullptr;     // pinned: node sums + the error word (enqueue_results)
  size_t h_res_cap = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t launches = 0;
};

namespace {

void drop_cache(qmcg_ctx* c) {
  dev_free(c->table);
  c->table = nullptr;
  c->table_rows_cap = 0;
  c->cache_dims = 0;
  c->cache_n = -1;
}

qmcg_status ensure_dim_tables(qmcg_ctx* c, int64_t n, int64_t m) {
  if (c->dt.n == n && c->dt.m >= m) return QMCG_OK;
  build_dim_tables(n, std::max<int64_t>(m, c->dt.n == n ? c->dt.m : 0), c->dt);
  QMCG_CUDA(cudaStreamSynchronize(c->stream));  // nothing queued still reads the arrays about to change
  QMCG_CUDA(c->d_sc.reserve(c->dt.sc.size()));
  QMCG_CUDA(c->d_nc.reserve(c->dt.nc.size()));
  QMCG_CUDA(cudaMemcpyAsync(c->d_sc.ptr, c->dt.sc.data(), c->dt.sc.size() * sizeof(double),
                            cudaMemcpyHostToDevice, c->stream));
  QMCG_CUDA(cudaMemcpyAsync(c->d_nc.ptr, c->dt.nc.data(), c->dt.nc.size() * sizeof(double),
                            cudaMemcpyHostToDevice, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

// Build one full permutation (length n) for dimension `dim` into dst (n u32).
// K1 into dst. Pricing tables hold perm + 1 (add = 1): the Halton index of
// uniform_at (quasi_rng.cpp:96-101), saving the increment per point in K2.
qmcg_status build_perm(qmcg_ctx* c, uint64_t seed64, int64_t n, uint32_t* dst, uint32_t add = 1) {
  const size_t need = qmcg::perm_scratch_bytes(n);
  QMCG_CUDA(c->d_permscratch.reserve(need));
  int launches = 0;
  QMCG_CUDA(qmcg::launch_perm_build(seed64, n, dst, c->d_permscratch.ptr, c->d_permscratch.cap, c->stream,
                                    &launches, add));
  c->launches += launches;
  return QMCG_OK;
}

#ifndef QMCG_K1_LANES
#define QMCG_K1_LANES 2
#endif
constexpr int kK1Lanes = QMCG_K1_LANES;             // K1 builds in flight (main stream + side lanes)
static_assert(kK1Lanes >= 2 && kK1Lanes <= 3, "one or two side lanes");
constexpr int64_t kOverlapMaxN = int64_t{1} << 25;  // the extra K1 scratch stays below ~0.6 GB per lane

// Rows [d0, d1) of a table, row k holding dimension dim_begin + k * dim_stride, with `lanes` K1
// builds in flight: row k on lane (k - d0) mod lanes (lane 0 = `stream`, the others side streams
// with their own scratch), so one table's latency-bound chase pass overlaps the next table's
// sort; `stream` then waits for the side lanes, so everything after sees all rows.
//   xdst: the rows are perm + 1 (u32, leading dimension ld, all n columns) -- the exchange format
//         of qmcg_build_tables;
//   udst: the rows are the uniforms uniform_at(p, dim) of columns [cb, ce) (f64, leading dimension
//         ld) -- the uniform table K2 reads: K1 writes the lane's row of perm + 1, then
//         uniforms_kernel turns the column slice into bit-exact radical inverses (writing the
//         uniforms from K1's chase pass instead measured slower: its latency-bound chase grew by
//         the digit division, 2^24 table 0.87 -> 1.07 ms).
// The caller has made the dimension constants of every built dim resident (ensure_dim_tables).
qmcg_status build_rows(qmcg_ctx* c, uint64_t seed, int64_t n, uint32_t* xdst, double* udst, int64_t ld, int64_t cb,
                       int64_t ce, int64_t d0, int64_t d1, int64_t dim_begin, int64_t dim_stride) {
  if (d1 <= d0) return QMCG_OK;
  const int lanes = (n <= kOverlapMaxN && d1 - d0 >= 2) ? kK1Lanes : 1;
  const size_t need = qmcg::perm_scratch_bytes(n);
  QMCG_CUDA(c->d_permscratch.reserve(need));
  if (udst) QMCG_CUDA(c->d_fullperm.reserve(static_cast<size_t>(n)));
  if (!c->ev_fork) QMCG_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  QMCG_CUDA(cudaEventRecord(c->ev_fork, c->stream));
  for (int l = 0; l + 1 < lanes; ++l) {
    if (!c->side[l]) QMCG_CUDA(cudaStreamCreateWithFlags(&c->side[l], cudaStreamNonBlocking));
    if (!c->ev_join[l]) QMCG_CUDA(cudaEventCreateWithFlags(&c->ev_join[l], cudaEventDisableTiming));
    QMCG_CUDA(c->d_permscratch_side[l].reserve(need));
    if (udst) QMCG_CUDA(c->d_xrow_side[l].reserve(static_cast<size_t>(n)));
    QMCG_CUDA(cudaStreamWaitEvent(c->side[l], c->ev_fork, 0));
  }
  for (int64_t k = d0; k < d1; ++k) {
    const int lane = static_cast<int>((k - d0) % lanes);
    DevBuf<char>& scratch = lane == 0 ? c->d_permscratch : c->d_permscratch_side[lane - 1];
    cudaStream_t s = lane == 0 ? c->stream : c->side[lane - 1];
    const int64_t dim = dim_begin + k * dim_stride;
    uint32_t* xrow = xdst ? xdst + static_cast<size_t>(k) * static_cast<size_t>(ld)
                          : (lane == 0 ? c->d_fullperm.ptr : c->d_xrow_side[lane - 1].ptr);
    int launches = 0;
    QMCG_CUDA(qmcg::launch_perm_build(dimension_seed(seed, dim), n, xrow, scratch.ptr, scratch.cap, s, &launches, 1));
    if (udst) {
      QMCG_CUDA(qmcg::launch_uniforms(xrow + cb, ce - cb, c->dt.dims[static_cast<size_t>(dim)], c->d_sc.ptr,
                                      c->d_nc.ptr, 0, udst + static_cast<size_t>(k) * static_cast<size_t>(ld), s));
      ++launches;
    }
    c->launches += launches;
  }
  for (int l = 0; l + 1 < lanes; ++l) {
    QMCG_CUDA(cudaEventRecord(c->ev_join[l], c->side[l]));
    QMCG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join[l], 0));
  }
  return QMCG_OK;
}

// Table storage for rows [0, m) of (seed, n) over columns [b, e): a cache for another key is
// dropped; rows [0, cache_dims) already built for this key are kept. Rows [cache_dims, m)
// are left for the caller to build.
qmcg_status reserve_table(qmcg_ctx* c, uint64_t seed, int64_t n, int64_t b, int64_t e, int64_t m, bool rebuild) {
  const int64_t cols = e - b;
  if (c->cache_n != n || c->cache_seed != seed || c->col_begin != b || c->col_end != e || rebuild) {
    if (c->table && c->cache_n >= 0 && qmcg::table_ld(c->col_end - c->col_begin) == qmcg::table_ld(cols)) {
      // same row stride: keep the allocation (freeing and re-mapping tens of GB costs 30-120 ms),
      // invalidate its rows
      QMCG_CUDA(cudaStreamSynchronize(c->stream));
      c->cache_dims = 0;
    } else {
      drop_cache(c);
    }
  }
  if (c->cache_n == n && c->cache_seed == seed && c->col_begin == b && c->col_end == e && c->cache_dims >= m)
    return QMCG_OK;
  const int64_t ld = qmcg::table_ld(cols);
  const size_t row_bytes = static_cast<size_t>(ld) * sizeof(double);
  if (!c->table || static_cast<size_t>(m) > c->table_rows_cap) {
    double* nt = nullptr;
    cudaError_t err = dev_alloc(reinterpret_cast<void**>(&nt), row_bytes * static_cast<size_t>(m) + qmcg::kTablePad * sizeof(double));
    if (err != cudaSuccess) {
      cudaGetLastError();
      char msg[256];
      std::snprintf(msg, sizeof msg,
                    "price_american: uniform tables of %lld dates x %lld paths (%.3g bytes) do not fit "
                    "in device memory",
                    static_cast<long long>(m), static_cast<long long>(cols),
                    static_cast<double>(row_bytes) * static_cast<double>(m));
      return fail(QMCG_OUT_OF_MEMORY, msg);
    }
    if (c->table && c->cache_dims > 0)
      QMCG_CUDA(cudaMemcpyAsync(nt, c->table, row_bytes * static_cast<size_t>(c->cache_dims),
                                cudaMemcpyDeviceToDevice, c->stream));
    QMCG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(c->table);
    c->table = nt;
    c->table_rows_cap = static_cast<size_t>(m);
  }
  c->cache_n = n;
  c->cache_seed = seed;
  c->col_begin = b;
  c->col_end = e;
  return QMCG_OK;
}

// Make rows [0, m) of the uniform table for (seed, n) over columns [b, e) resident.
qmcg_status ensure_perms(qmcg_ctx* c, uint64_t seed, int64_t n, int64_t b, int64_t e, int64_t m, bool rebuild) {
  qmcg_status st = ensure_dim_tables(c, n, m);
  if (st) return st;
  st = reserve_table(c, seed, n, b, e, m, rebuild);
  if (st) return st;
  if (c->cache_dims >= m) return QMCG_OK;
  NvtxRange nv("qmcg.K1.table_build");
  st = build_rows(c, seed, n, nullptr, c->table, qmcg::table_ld(e - b), b, e, c->cache_dims, m, 0, 1);
  if (st) return st;
  c->cache_dims = m;
  return QMCG_OK;
}

struct CallPlan {
  PriceParams P{};
  std::vector<double> dpow;
};

// Validation + host constants, in the order of reference price_american
// (american.cpp:103-116) -> make_schedule (path_engine.cpp:63-76) ->
// simulate_batch (path_engine.cpp:124-136) -> QuasiStream (quasi_rng.cpp:85-94).
// `chain`: a discount chain already computed for this m (a batch's previous contract); reused when
// its discount factor is this contract's (the 128-step dependent multiply chain dominates a plan).
qmcg_status plan_call(const qmcg_option_spec& s, int64_t m, int64_t n, uint32_t flags, CallPlan& plan,
                      const std::vector<double>* chain = nullptr) {
  qmcg_status st = validate(s);
  if (st) return st;
  if (s.kind != QMCG_CALL && !(flags & QMCG_FLAG_ALLOW_PUT))
    return fail(QMCG_INVALID_ARGUMENT,
                "price_american: not implemented for puts; the foresight algorithm is call-only");
  if (n < 2) return fail(QMCG_INVALID_ARGUMENT, "price_american: n_paths must be >= 2");
  if (m < 1) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: m must be >= 1");
  if (!(s.maturity > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: maturity must be > 0");
  if (static_cast<uint64_t>(n) > 0xffffffffULL)
    return fail(QMCG_LENGTH_ERROR, "permutation_indices: n exceeds the 2^32-1 supported maximum");
  if (m > (int64_t{1} << 26)) return fail(QMCG_LENGTH_ERROR, "price_american: m exceeds the 2^26 supported maximum");

  const double dt = s.maturity / static_cast<double>(m + 1);  // make_schedule
  const double r = s.rate, v = s.volatility;
  const double a = (r - 0.5 * v * v) * dt;  // gbm_step drift
  const double bdiff = v * std::sqrt(dt);   // gbm_step diffusion
  const double disc = std::exp(-s.rate * dt);  // sweep_impl
  PriceParams& P = plan.P;
  P.m = static_cast<int32_t>(m);
  P.kind = s.kind;
  P.X0 = std::log(s.spot);
  P.strike = s.strike;
  P.log_strike = std::log(s.strike);
  P.best0 = intrinsic(s.kind, s.spot, s.strike);
  P.deterministic = bdiff == 0.0;
  if (P.deterministic) {
    P.b = 1.0;
    P.alpha = a;
  } else {
    P.b = bdiff;
    P.alpha = a / bdiff;
  }
  if (chain && chain->size() == static_cast<size_t>(m) + 1 && m >= 1 && bits_of((*chain)[1]) == bits_of(disc)) {
    plan.dpow = *chain;
  } else {
    plan.dpow.resize(static_cast<size_t>(m) + 1);
    plan.dpow[0] = 1.0;
    for (int64_t k = 1; k <= m; ++k) plan.dpow[static_cast<size_t>(k)] = plan.dpow[static_cast<size_t>(k - 1)] * disc;
  }
  P.rate_negative = disc > 1.0;
  P.dom_slope = s.kind == QMCG_CALL ? (r * dt) / P.b : r * dt;
  P.x0mk = 1.0 + P.X0 - P.log_strike;
  if (!P.rate_negative) {
    const double edge = s.kind == QMCG_CALL ? std::max(s.strike, s.spot) : std::min(s.strike, s.spot);
    P.c0 = (std::log(edge) - P.X0) / P.b;
    P.dmax_inv = 1.0;
  } else {
    const double dmax = plan.dpow[static_cast<size_t>(m)];
    P.dmax_inv = 1.0 / dmax;
    const double lim = P.best0 * P.dmax_inv;
    if (s.kind == QMCG_CALL) P.c0 = (std::log(s.strike + lim) - P.X0) / P.b;
    else P.c0 = s.strike - lim > 0.0 ? (std::log(s.strike - lim) - P.X0) / P.b : -INFINITY;
  }
  // final interval Black-Scholes (bs_price, analytic.cpp:102-124, with t = dt)
  P.bs_v_zero = v == 0.0;
  P.bs_vsqrt = v * std::sqrt(dt);
  P.bs_mu_t = (r + 0.5 * v * v) * dt;
  P.bs_kdisc = s.strike * std::exp(-r * dt);
  P.bs_fwd_growth = std::exp(r * dt);
  P.bs_disc = std::exp(-r * dt);
  // overflow / underflow of the log-price walk is impossible when
  // |X0| + m (|a| + b |z|max) stays inside exp's range (|z| <= 7.04 for u in [1e-12, 1-1e-12])
  const double reach = std::fabs(P.X0) + static_cast<double>(m) * (std::fabs(a) + bdiff * 7.05) + 1.0;
  P.check_range = reach > 700.0;
  P.fp32 = (flags & QMCG_FLAG_FP32) != 0;
  P.d_begin = 0;
  P.d_end = P.m;
  P.perm_row0 = 0;
  return QMCG_OK;
}


qmcg_status upload_plan(qmcg_ctx* c, CallPlan& plan, int64_t n) {
  const int64_t m = plan.P.m;
  qmcg_status st = ensure_dim_tables(c, n, m);
  if (st) return st;
  if (c->dpow_host != plan.dpow) {  // the discount chain of the last single-contract call is still there
    QMCG_CUDA(c->d_dpow.reserve(plan.dpow.size()));
    QMCG_CUDA(cudaMemcpyAsync(c->d_dpow.ptr, plan.dpow.data(), plan.dpow.size() * sizeof(double),
                              cudaMemcpyHostToDevice, c->stream));
    c->dpow_host = plan.dpow;
  }
  plan.P.dpow = c->d_dpow.ptr;
  return QMCG_OK;
}

qmcg_status map_err(uint32_t err) {
  if (err & qmcg::ERR_SPOT_NONPOSITIVE) return fail(QMCG_INVALID_ARGUMENT, "gbm_step: s_prev must be > 0");
  if (err & qmcg::ERR_SPOT_NONFINITE) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: all fields must be finite");
  return QMCG_OK;
}

// Enqueue pricing of paths [b, e) and the pairwise reduction of that range
// into d_sums[slot*2 .. slot*2+1]. Tables must be resident.
// Launch the pricing kernel over paths [b, e) (tables resident) into d_values.
qmcg_status enqueue_values(qmcg_ctx* c, CallPlan& plan, int64_t b, int64_t e, cudaEvent_t after_kernel = nullptr) {
  NvtxRange nv("qmcg.K2.price_kernel");
  const int64_t cnt = e - b;
  QMCG_CUDA(c->d_values.reserve(static_cast<size_t>(cnt)));
  QMCG_CUDA(c->d_red.reserve(qmcg::reduce_scratch_doubles(cnt)));
  PriceParams P = plan.P;
  P.table = c->table;
  P.ld = qmcg::table_ld(c->col_end - c->col_begin);
  if ((b - c->col_begin) % 4 != 0) return fail(QMCG_INVALID_ARGUMENT, "internal: unaligned path range");
  P.col_begin = c->col_begin;
  P.path_begin = b;
  P.path_count = cnt;
  P.values = c->d_values.ptr;
  P.err = c->d_err.ptr;
  QMCG_CUDA(qmcg::launch_price(P, c->stream));
  c->launches += 1;
  if (after_kernel) QMCG_CUDA(cudaEventRecord(after_kernel, c->stream));
  return QMCG_OK;
}

// Kernel over [b, e) + the pairwise sums of all its paths into d_sums[slot].
qmcg_status enqueue_price(qmcg_ctx* c, CallPlan& plan, int64_t b, int64_t e, int slot, cudaEvent_t after_kernel) {
  qmcg_status st = enqueue_values(c, plan, b, e, after_kernel);
  if (st) return st;
  int launches = 0;
  QMCG_CUDA(qmcg::launch_pairwise(c->d_values.ptr, e - b, c->d_red.ptr, c->d_sums.ptr + 2 * slot, c->stream,
                                  &launches));
  c->launches += launches;
  return QMCG_OK;
}

qmcg_status prepare_scratch(qmcg_ctx* c, size_t slots) {
  QMCG_CUDA(c->d_sums.reserve(2 * slots));
  QMCG_CUDA(c->d_err.reserve(1));
  QMCG_CUDA(cudaMemsetAsync(c->d_err.ptr, 0, sizeof(uint32_t), c->stream));
  return QMCG_OK;
}

// reduce_stats' arithmetic (path_engine.cpp:191-205) on the tree sums.
void finish_stats(int64_t n, double sum, double sum_sq, double& mean, double& se) {
  mean = sum / static_cast<double>(n);
  se = 0.0;
  if (n >= 2) {
    double var = (sum_sq - static_cast<double>(n) * mean * mean) / static_cast<double>(n - 1);
    if (var < 0.0) var = 0.0;
    se = std::sqrt(var / static_cast<double>(n));
  }
}

// Results in two phases, so a device group can enqueue every member before waiting on any:
// enqueue_results queues the D2H copy of the node sums and the error word into pinned memory,
// finish_results waits for it and maps the error word to the reference's exceptions.
qmcg_status enqueue_results(qmcg_ctx* c, size_t slots) {
  if (2 * slots + 1 > c->h_res_cap) {
    if (c->h_res) cudaFreeHost(c->h_res);
    c->h_res = nullptr;
    c->h_res_cap = 0;
    QMCG_CUDA(cudaMallocHost(&c->h_res, (2 * slots + 1) * sizeof(double)));
    c->h_res_cap = 2 * slots + 1;
  }
  QMCG_CUDA(cudaMemcpyAsync(c->h_res, c->d_sums.ptr, 2 * slots * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaMemcpyAsync(c->h_res + 2 * slots, c->d_err.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            c->stream));
  return QMCG_OK;
}

qmcg_status finish_results(qmcg_ctx* c, size_t slots, double* sums) {
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  uint32_t err = 0;
  std::memcpy(&err, c->h_res + 2 * slots, sizeof err);
  std::copy(c->h_res, c->h_res + 2 * slots, sums);
  return map_err(err);
}

qmcg_status sync_results(qmcg_ctx* c, size_t slots, std::vector<double>& sums) {
  sums.resize(2 * slots);
  qmcg_status st = enqueue_results(c, slots);
  if (st) return st;
  return finish_results(c, slots, sums.data());
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// device-group forms (defined with the group code below)
qmcg_status group_warm(qmcg_ctx* g, int64_t n, uint64_t seed, int64_t dims);
qmcg_status group_batch(qmcg_ctx* g, const qmcg_option_spec* specs, int64_t n_specs, int64_t m, int64_t n,
                        uint64_t seed, uint32_t flags, qmcg_pricing_result* out);
qmcg_status group_path_values(qmcg_ctx* g, const qmcg_option_spec& spec, int64_t m, int64_t n, uint64_t seed,
                              uint32_t flags, double* out_host);
qmcg_status group_time_device(qmcg_ctx* g, const qmcg_option_spec& spec, int64_t m, int64_t n, uint64_t seed,
                              uint32_t flags, int reps, double* kernel_ms, double* step_ms, double* price_se);
qmcg_status group_time_perm_build(qmcg_ctx* g, int64_t n, uint64_t seed, int64_t dims, double* ms);

}  // namespace

extern "C" {

const char* qmcg_last_error(void) { return g_last_error.c_str(); }
const char* qmcg_version(void) { return "qmcg 0.1 (sm_100a)"; }

qmcg_status qmcg_create(int device, qmcg_ctx** out) {
  if (!out) return fail(QMCG_INVALID_ARGUMENT, "qmcg_create: out must not be null");
  int count = 0;
  QMCG_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(QMCG_INVALID_ARGUMENT, "qmcg_create: no such CUDA device");
  DeviceGuard g(device);
  auto* c = new qmcg_ctx();
  c->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_pinned, 16 * sizeof(double));
  for (auto& ev : c->ev)
    if (e == cudaSuccess) e = cudaEventCreate(&ev);
  if (e != cudaSuccess) {
    delete c;
    return fail(QMCG_CUDA_ERROR, std::string("qmcg_create: ") + cudaGetErrorString(e));
  }
  *out = c;
  return QMCG_OK;
}

qmcg_status qmcg_create_multi(const int* dev_ids, int n_dev, qmcg_ctx** out) {
  if (!out || !dev_ids || n_dev < 1) return fail(QMCG_INVALID_ARGUMENT, "qmcg_create_multi: bad device list");
  auto* g = new qmcg_ctx();
  g->device = dev_ids[0];
  for (int r = 0; r < n_dev; ++r) {
    qmcg_ctx* c = nullptr;
    const qmcg_status st = qmcg_create(dev_ids[r], &c);
    if (st) {
      qmcg_destroy(g);
      return st;
    }
    g->members.push_back(c);
    g->workers.push_back(std::make_unique<MemberWorker>());
  }
  // peer access between distinct listed devices (NVLink / NVSwitch); the slice copies also work
  // without it (staged by the driver), so failures here are not errors
  for (int a = 0; a < n_dev; ++a)
    for (int b = 0; b < n_dev; ++b) {
      if (dev_ids[a] == dev_ids[b]) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, dev_ids[a], dev_ids[b]) == cudaSuccess && can) {
        DeviceGuard dg(dev_ids[a]);
        if (cudaDeviceEnablePeerAccess(dev_ids[b], 0) != cudaSuccess) cudaGetLastError();
      }
    }
  *out = g;
  return QMCG_OK;
}

qmcg_status qmcg_create_default(qmcg_ctx** out) {
  if (!out) return fail(QMCG_INVALID_ARGUMENT, "qmcg_create_default: out must not be null");
  std::vector<int> devs;
  if (const char* env = std::getenv("QMCG_DEVICES"); env && *env) {
    const char* p = env;
    while (*p) {
      char* end = nullptr;
      const long d = std::strtol(p, &end, 10);
      if (end == p) return fail(QMCG_INVALID_ARGUMENT, std::string("QMCG_DEVICES: not a device list: ") + env);
      devs.push_back(static_cast<int>(d));
      p = *end == ',' ? end + 1 : end;
      if (*end && *end != ',') return fail(QMCG_INVALID_ARGUMENT, std::string("QMCG_DEVICES: not a device list: ") + env);
    }
  } else {
    int count = 0;
    QMCG_CUDA(cudaGetDeviceCount(&count));
    for (int d = 0; d < count; ++d) devs.push_back(d);
  }
  if (devs.empty()) return fail(QMCG_CUDA_ERROR, "qmcg_create_default: no CUDA device");
  if (devs.size() == 1) return qmcg_create(devs[0], out);
  return qmcg_create_multi(devs.data(), static_cast<int>(devs.size()), out);
}

qmcg_status qmcg_check_canaries(void) {
  if (!canary_mode()) return fail(QMCG_UNSUPPORTED, "qmcg_check_canaries: set QMCG_CANARY=1 before the first allocation");
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  std::vector<unsigned char> h(kGuard);
  for (const auto& a : guarded_allocs()) {
    DeviceGuard g(a.second.device);
    QMCG_CUDA(cudaDeviceSynchronize());
    for (int side = 0; side < 2; ++side) {
      const char* src = side == 0 ? a.second.base : a.second.base + kGuard + a.second.bytes;
      QMCG_CUDA(cudaMemcpy(h.data(), src, kGuard, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < kGuard; ++i)
        if (h[i] != 0xA5) {
          char msg[192];
          std::snprintf(msg, sizeof msg, "qmcg_check_canaries: guard %s a %zu-byte buffer on device %d clobbered at +%zu",
                        side == 0 ? "before" : "after", a.second.bytes, a.second.device, i);
          return fail(QMCG_CUDA_ERROR, msg);
        }
    }
  }
  return QMCG_OK;
}

int qmcg_device_count(qmcg_ctx* c) { return !c ? 0 : c->members.empty() ? 1 : static_cast<int>(c->members.size()); }

void qmcg_destroy(qmcg_ctx* c) {
  if (!c) return;
  if (!c->members.empty() || !c->stream) {  // a group handle owns only its members
    for (qmcg_ctx* m : c->members) qmcg_destroy(m);
    delete c;
    return;
  }
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->stream);
  drop_cache(c);

  c->d_sc.release();
  c->d_nc.release();
  c->d_dpow.release();
  c->d_values.release();
  c->d_red.release();
  c->d_z.release();
  for (int k = 0; k < 2; ++k) {
    c->d_bvalues[k].release();
    c->d_bred[k].release();
    c->d_bsums[k].release();
    c->d_cparams[k].release();
    c->d_groups[k].release();
  }
  c->d_sums.release();
  c->d_err.release();
  c->d_fullperm.release();
  c->d_permscratch.release();
  for (int l = 0; l < 2; ++l) {
    if (c->side[l]) cudaStreamSynchronize(c->side[l]);
    c->d_permscratch_side[l].release();
    c->d_xrow_side[l].release();
    if (c->side[l]) cudaStreamDestroy(c->side[l]);
    if (c->ev_join[l]) cudaEventDestroy(c->ev_join[l]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_built) cudaEventDestroy(c->ev_built);
  if (c->ev_priced) cudaEventDestroy(c->ev_priced);
  c->d_gtmp.release();

  c->d_path.release();
  c->d_path_t.release();
  c->d_ex.release();
  c->d_stV.release();
  c->d_stc.release();
  c->d_stcd.release();
  c->d_stbest.release();
  c->d_stpend.release();
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  if (c->h_res) cudaFreeHost(c->h_res);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  cudaStreamDestroy(c->stream);
  delete c;
}

qmcg_status qmcg_tree_node_range(int64_t n, int depth, int64_t node, int64_t* begin, int64_t* end) {
  if (n < 1 || depth < 0 || depth > 40 || node < 0 || node >= (int64_t{1} << depth))
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_tree_node_range: bad node");
  int64_t off, size;
  tree_node(n, depth, node, off, size);
  *begin = off;
  *end = off + size;
  return QMCG_OK;
}

// Fold node sums up the reference tree. A node of size <= 64 is a sequential
// leaf in the reference; such nodes must not be split, so depth is limited to
// levels whose parents all exceed 64 elements.
qmcg_status qmcg_combine_nodes(int64_t n, int depth, const double* node_sums, double* price, double* se) {
  if (n < 1 || depth < 0 || depth > 30) return fail(QMCG_INVALID_ARGUMENT, "qmcg_combine_nodes: bad depth");
  std::vector<double> s(node_sums, node_sums + 2 * (size_t{1} << depth));
  for (int d = depth; d > 0; --d) {
    const size_t cnt = size_t{1} << (d - 1);
    for (size_t i = 0; i < cnt; ++i) {
      s[2 * i] = s[4 * i] + s[4 * i + 2];
      s[2 * i + 1] = s[4 * i + 1] + s[4 * i + 3];
    }
  }
  double mean, err;
  finish_stats(n, s[0], s[1], mean, err);
  *price = mean;
  *se = err;
  return QMCG_OK;
}

qmcg_status qmcg_warm(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dims) {
  if (!c) return fail(QMCG_INVALID_ARGUMENT, "qmcg_warm: null context");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  if (n < 1 || static_cast<uint64_t>(n) > 0xffffffffULL || dims < 1)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_warm: bad size");
  if (!c->members.empty()) return group_warm(c, n, seed, dims);  // the slices group pricing reads
  qmcg_status st = ensure_perms(c, seed, n, 0, n, dims, false);
  if (st) return st;
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

qmcg_status qmcg_build_tables(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dim_begin, int64_t dim_stride,
                              int64_t count, uint32_t* out_dev, int64_t ld) {
  if (c && !c->members.empty())
    return fail(QMCG_UNSUPPORTED, "qmcg_build_tables: a per-device call (use a single-device context per rank)");
  if (!c || (!out_dev && count > 0)) return fail(QMCG_INVALID_ARGUMENT, "qmcg_build_tables: null argument");
  if (n < 1 || static_cast<uint64_t>(n) > 0xffffffffULL || dim_begin < 0 || dim_stride < 1 || count < 0 || ld < n)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_build_tables: bad size");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  qmcg_status st = build_rows(c, seed, n, out_dev, nullptr, ld, 0, n, 0, count, dim_begin, dim_stride);
  if (st) return st;
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

}  // extern "C"

namespace {
// Rows [row_begin, row_begin + row_count) of the slice [col_begin, col_end) of the uniform table
// for dims [0, dims), from rows of perm + 1 (src_dev, stride src_ld): each row is turned into its
// dimension's uniforms by uniforms_kernel. row_begin = 0 starts a fresh slice table.
qmcg_status import_x_rows(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t col_begin, int64_t col_end, int64_t dims,
                          int64_t row_begin, int64_t row_count, const uint32_t* src_dev, int64_t src_ld) {
  const int64_t cols = col_end - col_begin;
  qmcg_status st = ensure_dim_tables(c, n, dims);
  if (st) return st;
  if (row_begin == 0) {
    st = reserve_table(c, seed, n, col_begin, col_end, dims, true);  // a fresh slice table
    if (st) return st;
  } else if (c->cache_n != n || c->cache_seed != seed || c->col_begin != col_begin || c->col_end != col_end ||
             c->cache_dims != row_begin || c->table_rows_cap < static_cast<size_t>(dims)) {
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_import_rows: rows must continue the slice imported so far");
  }
  const int64_t ld = qmcg::table_ld(cols);
  for (int64_t k = 0; k < row_count; ++k)
    QMCG_CUDA(qmcg::launch_uniforms(src_dev + static_cast<size_t>(k) * static_cast<size_t>(src_ld), cols,
                                    c->dt.dims[static_cast<size_t>(row_begin + k)], c->d_sc.ptr, c->d_nc.ptr, 0,
                                    c->table + static_cast<size_t>(row_begin + k) * static_cast<size_t>(ld), c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  c->cache_dims = row_begin + row_count;
  return QMCG_OK;
}
}  // namespace

extern "C" {

qmcg_status qmcg_import_tables(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t col_begin, int64_t col_end,
                               int64_t dims, const uint32_t* src_dev, int64_t src_ld) {
  if (c && !c->members.empty())
    return fail(QMCG_UNSUPPORTED, "qmcg_import_tables: a per-device call (use a single-device context per rank)");
  if (!c || !src_dev) return fail(QMCG_INVALID_ARGUMENT, "qmcg_import_tables: null argument");
  const int64_t cols = col_end - col_begin;
  if (n < 1 || static_cast<uint64_t>(n) > 0xffffffffULL || col_begin < 0 || cols < 1 || col_end > n || dims < 1 ||
      src_ld < cols)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_import_tables: bad size");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  return import_x_rows(c, n, seed, col_begin, col_end, dims, 0, dims, src_dev, src_ld);
}

qmcg_status qmcg_import_rows(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t col_begin, int64_t col_end, int64_t dims,
                             int64_t row_begin, int64_t row_count, const uint32_t* src_dev, int64_t src_ld) {
  if (!c || !src_dev) return fail(QMCG_INVALID_ARGUMENT, "qmcg_import_rows: null argument");
  if (!c->members.empty())
    return fail(QMCG_UNSUPPORTED, "qmcg_import_rows: a per-device call (use a single-device context per rank)");
  const int64_t cols = col_end - col_begin;
  if (n < 1 || static_cast<uint64_t>(n) > 0xffffffffULL || col_begin < 0 || cols < 1 || col_end > n || dims < 1 ||
      row_begin < 0 || row_count < 1 || row_begin + row_count > dims || src_ld < cols)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_import_rows: bad size");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  return import_x_rows(c, n, seed, col_begin, col_end, dims, row_begin, row_count, src_dev, src_ld);
}

qmcg_status qmcg_set_table_budget(qmcg_ctx* c, uint64_t bytes) {
  if (!c) return fail(QMCG_INVALID_ARGUMENT, "qmcg_set_table_budget: null context");
  std::lock_guard<std::mutex> lock(c->mu);
  c->table_budget = static_cast<size_t>(bytes);
  for (qmcg_ctx* m : c->members) qmcg_set_table_budget(m, bytes);
  return QMCG_OK;
}

int64_t qmcg_last_window_count(qmcg_ctx* c) {
  if (c && !c->members.empty()) return c->members[0]->last_windows;
  return c ? c->last_windows : -1;
}

qmcg_status qmcg_clear_cache(qmcg_ctx* c) {
  if (!c) return fail(QMCG_INVALID_ARGUMENT, "qmcg_clear_cache: null context");
  std::lock_guard<std::mutex> lock(c->mu);
  for (qmcg_ctx* m : c->members) qmcg_clear_cache(m);
  if (!c->members.empty()) return QMCG_OK;
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->stream);
  drop_cache(c);
  return QMCG_OK;
}

}  // extern "C"

// ---- pricing of a path range (resident or streamed tables) ----
namespace {

// Bytes the permutation table of `cols` columns may occupy: the caller's
// budget, capped by free device memory (+ the table already held) minus the
// K1 scratch, the carried walk state, the per-path values and a margin.
size_t table_bytes_allowed(qmcg_ctx* c, int64_t n, int64_t cols, bool full) {
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const int64_t held_ld = qmcg::table_ld(c->col_end - c->col_begin);
  const size_t held = c->table ? c->table_rows_cap * static_cast<size_t>(held_ld) * sizeof(double) : 0;
  // K1 scratch and a row of perm + 1 per build lane, the carried walk state, values, a margin
  const size_t lanes = n <= kOverlapMaxN ? kK1Lanes : 1;
  (void)full;
  const size_t reserve = lanes * (qmcg::perm_scratch_bytes(n) + static_cast<size_t>(n) * 4) +
                         static_cast<size_t>(cols) * (4 * 8 + 4 + 8 + 8) + (size_t{1} << 30);
  const size_t avail = free_b + held > reserve ? free_b + held - reserve : 0;
  return c->table_budget ? std::min(c->table_budget, avail) : avail;
}

// The pairwise sums of the `count` consecutive tree nodes [node0, node0 + count) at `depth`
// from the per-path values of paths [b, ...) in d_values, into d_sums[2k, 2k + 1].
qmcg_status enqueue_node_sums(qmcg_ctx* c, int64_t n, int depth, int64_t node0, int64_t count, int64_t b) {
  NvtxRange nv("qmcg.K3.pairwise_tree");
  for (int64_t k = 0; k < count; ++k) {
    int64_t off, size;
    tree_node(n, depth, node0 + k, off, size);
    int launches = 0;
    QMCG_CUDA(qmcg::launch_pairwise(c->d_values.ptr + (off - b), size, c->d_red.ptr, c->d_sums.ptr + 2 * k, c->stream,
                                    &launches));
    c->launches += launches;
  }
  return QMCG_OK;
}

// Tables larger than device memory (config 5: 2^28 paths x 365 dates = 392 GB):
// the dates are processed in windows of W rows; each window's rows are built
// by K1 into the same W-row buffer, then K2 walks every path through the
// window, carrying (V, last record, dominance accumulator, pending record,
// best) in HBM to the next window. Results are identical to resident tables.
qmcg_status enqueue_streamed(qmcg_ctx* c, CallPlan& plan, uint64_t seed, int64_t n, int64_t b, int64_t e,
                             size_t budget) {
  NvtxRange nv("qmcg.streamed_windows");
  const int64_t cols = e - b, m = plan.P.m;
  const int64_t ld = qmcg::table_ld(cols);
  const size_t row_bytes = static_cast<size_t>(ld) * sizeof(double);
  int64_t W = static_cast<int64_t>(budget / row_bytes) / 8 * 8;
  if (W < 8)
    return fail(QMCG_OUT_OF_MEMORY, "price_american: not enough device memory for 8 uniform-table rows");
  W = std::min<int64_t>(W, (m + 7) / 8 * 8);
  qmcg_status st = ensure_dim_tables(c, n, m);
  if (st) return st;
  drop_cache(c);
  double* nt = nullptr;
  if (dev_alloc(reinterpret_cast<void**>(&nt), row_bytes * static_cast<size_t>(W) + qmcg::kTablePad * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(QMCG_OUT_OF_MEMORY, "price_american: uniform-table window does not fit in device memory");
  }
  c->table = nt;
  c->table_rows_cap = static_cast<size_t>(W);
  c->col_begin = b;  // the buffer holds a window, never a cache (cache_n stays -1)
  c->col_end = e;
  QMCG_CUDA(c->d_values.reserve(static_cast<size_t>(cols)));
  QMCG_CUDA(c->d_red.reserve(qmcg::reduce_scratch_doubles(cols)));
  for (auto* buf : {&c->d_stV, &c->d_stc, &c->d_stcd, &c->d_stbest})
    QMCG_CUDA(buf->reserve(static_cast<size_t>(cols)));
  QMCG_CUDA(c->d_stpend.reserve(static_cast<size_t>(cols)));
  PriceParams P = plan.P;
  P.table = c->table;
  P.ld = ld;
  P.col_begin = b;
  P.path_begin = b;
  P.path_count = cols;
  P.values = c->d_values.ptr;
  P.err = c->d_err.ptr;
  P.st_V = c->d_stV.ptr;
  P.st_c = c->d_stc.ptr;
  P.st_cd = c->d_stcd.ptr;
  P.st_best = c->d_stbest.ptr;
  P.st_pend = c->d_stpend.ptr;
  c->last_windows = 0;
  for (int64_t d0 = 0; d0 < m; d0 += W) {
    const int64_t d1 = std::min(m, d0 + W);
    st = build_rows(c, seed, n, nullptr, c->table, ld, b, e, 0, d1 - d0, d0, 1);  // window row k = dim d0 + k
    if (st) return st;
    P.d_begin = static_cast<int32_t>(d0);
    P.d_end = static_cast<int32_t>(d1);
    P.perm_row0 = static_cast<int32_t>(d0);
    P.stream_load = d0 > 0;
    P.stream_store = d1 < m;
    QMCG_CUDA(qmcg::launch_price(P, c->stream));
    c->launches += 1;
    c->last_windows += 1;
  }
  return QMCG_OK;
}

// Per-path values of paths [b, e) into d_values (resident tables from the
// cache, or streamed date windows when the tables exceed the budget), then
// the pairwise sums of each of the `count` consecutive tree nodes
// [node0, node0 + count) at `depth` (which must tile [b, e)) into d_sums, and
// their copy to pinned host memory (price_nodes_finish waits for it).
static qmcg_status price_nodes_enqueue(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n,
                                       uint64_t seed, uint32_t flags, int depth, int64_t node0, int64_t count) {
  int64_t b, e, off, size;
  tree_node(n, depth, node0, b, size);
  tree_node(n, depth, node0 + count - 1, off, size);
  e = off + size;
  Trace tr("price");
  CallPlan plan;
  qmcg_status st = plan_call(*spec, m, n, flags, plan);
  if (st) return st;
  st = upload_plan(c, plan, n);
  if (st) return st;
  tr.mark("plan+upload");
  const bool rebuild = (flags & QMCG_FLAG_NO_CACHE) != 0;
  const bool cached = !rebuild && c->cache_n == n && c->cache_seed == seed && c->col_begin == b &&
                      c->col_end == e && c->cache_dims >= m;
  bool streamed = false;
  size_t budget = 0;
  if (!cached && !plan.P.deterministic) {
    budget = table_bytes_allowed(c, n, e - b, b == 0 && e == n);
    const size_t need = static_cast<size_t>(qmcg::table_ld(e - b)) * sizeof(double) * static_cast<size_t>(m);
    streamed = need > budget;
  }
  st = prepare_scratch(c, static_cast<size_t>(count));
  if (st) return st;
  if (streamed) {
    st = enqueue_streamed(c, plan, seed, n, b, e, budget);
    if (st) return st;
  } else {
    st = ensure_perms(c, seed, n, b, e, m, rebuild);
    if (st) return st;
    c->last_windows = 1;
    st = enqueue_values(c, plan, b, e);
    if (st) return st;
  }
  st = enqueue_node_sums(c, n, depth, node0, count, b);
  if (st) return st;
  tr.mark(streamed ? "streamed enqueued" : "enqueued");
  return enqueue_results(c, static_cast<size_t>(count));
}

static qmcg_status price_nodes_finish(qmcg_ctx* c, int64_t count, double* sums) {
  return finish_results(c, static_cast<size_t>(count), sums);
}

static qmcg_status price_nodes(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                               uint32_t flags, int depth, int64_t node0, int64_t count, double* sums) {
  qmcg_status st = price_nodes_enqueue(c, spec, m, n, seed, flags, depth, node0, count);
  if (st) return st;
  return price_nodes_finish(c, count, sums);
}

static qmcg_status price_range(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                               uint32_t flags, double sums[2]) {
  return price_nodes(c, spec, m, n, seed, flags, 0, 0, 1, sums);
}

// ---------------------------------------------------------------------------
// Device groups (qmcg_create_multi): one host handle over several CUDA devices.
// The reference's only parallel axis is the path range (parallel_for_chunks,
// proj/src/path_engine.cpp:83-122) plus a fixed pairwise tree (:39-59); a group
// gives member r the contiguous tree nodes node_owner(i) = min(G-1, i G / 2^D) at
// depth D = ceil(log2 G), so every member prices its own column
// slice of the permutation tables, 16 bytes per node come back, and the host
// folds them up the same tree: bit-identical to one device for every G.
// Cold tables are built dimension-sharded (dim d by member d mod G, full n) and
// each member's column slice is copied to it with one cudaMemcpyPeerAsync per
// (dim, member) over NVLink; tables that exceed device memory are streamed in
// date windows with the same sharded build per window.
// ---------------------------------------------------------------------------
struct MemberRange {
  int64_t node0 = 0, count = 0;  // tree nodes [node0, node0 + count) at the group depth
  int64_t b = 0, e = 0;          // their path (column) range
};

int group_depth(int64_t n, int G) {
  int want = 0;
  while ((int64_t{1} << want) < G) ++want;
  int depth = 0;
  while (depth < want && (n >> depth) > 64) ++depth;  // nodes at depth+1 need parents above a leaf
  return depth;
}

std::vector<MemberRange> member_ranges(int64_t n, int G, int depth) {
  std::vector<MemberRange> R(static_cast<size_t>(G));
  const int64_t nodes = int64_t{1} << depth;
  for (int64_t i = 0; i < nodes; ++i) {
    const int r = static_cast<int>(std::min<int64_t>(G - 1, (i * G) / nodes));
    MemberRange& m = R[static_cast<size_t>(r)];
    if (m.count == 0) m.node0 = i;
    ++m.count;
  }
  for (auto& m : R) {
    if (!m.count) continue;
    int64_t off, size;
    tree_node(n, depth, m.node0, off, size);
    m.b = off;
    tree_node(n, depth, m.node0 + m.count - 1, off, size);
    m.e = off + size;
  }
  return R;
}

// Fold 2^depth interleaved node sums up the reference tree (pairwise_sum's splits).
void fold_nodes(std::vector<double>& s, int depth) {
  for (int d = depth; d > 0; --d) {
    const size_t cnt = size_t{1} << (d - 1);
    for (size_t i = 0; i < cnt; ++i) {
      s[2 * i] = s[4 * i] + s[4 * i + 2];
      s[2 * i + 1] = s[4 * i + 1] + s[4 * i + 3];
    }
  }
}

qmcg_status ensure_events(qmcg_ctx* c) {
  DeviceGuard g(c->device);
  if (!c->ev_built) QMCG_CUDA(cudaEventCreateWithFlags(&c->ev_built, cudaEventDisableTiming));
  if (!c->ev_priced) QMCG_CUDA(cudaEventCreateWithFlags(&c->ev_priced, cudaEventDisableTiming));
  return QMCG_OK;
}

// Every stream in `to` waits for the work queued so far on every stream of `from`.
qmcg_status cross_wait(const std::vector<qmcg_ctx*>& from, const std::vector<qmcg_ctx*>& to, bool built) {
  for (qmcg_ctx* f : from) {
    DeviceGuard g(f->device);
    QMCG_CUDA(cudaEventRecord(built ? f->ev_built : f->ev_priced, f->stream));
  }
  for (qmcg_ctx* t : to) {
    DeviceGuard g(t->device);
    for (qmcg_ctx* f : from) QMCG_CUDA(cudaStreamWaitEvent(t->stream, built ? f->ev_built : f->ev_priced, 0));
  }
  return QMCG_OK;
}

// Uniform-table rows of dims `dims` (all n columns) built by member `bc` into its scratch `tmp`
// (rows of n entries), then row k's slice [R[s].b, R[s].e) copied into row dst_row[k] of member s's
// table. The builder needs the dimension constants of every dim it builds (ensure_dim_tables).
qmcg_status build_and_scatter(qmcg_ctx* bc, uint64_t seed, int64_t n, const std::vector<int64_t>& dims,
                              const std::vector<int64_t>& dst_row, const std::vector<qmcg_ctx*>& M,
                              const std::vector<MemberRange>& R, double* tmp, int64_t tmp_rows) {
  DeviceGuard g(bc->device);
  qmcg_status st = ensure_dim_tables(bc, n, dims.back() + 1);
  if (st) return st;
  for (size_t k0 = 0; k0 < dims.size(); k0 += static_cast<size_t>(tmp_rows)) {
    const size_t cnt = std::min(dims.size() - k0, static_cast<size_t>(tmp_rows));
    // dims of a member are an arithmetic progression with stride G
    const int64_t stride = cnt > 1 ? dims[k0 + 1] - dims[k0] : 1;
    st = build_rows(bc, seed, n, nullptr, tmp, n, 0, n, 0, static_cast<int64_t>(cnt), dims[k0], stride);
    if (st) return st;
    for (size_t s = 0; s < M.size(); ++s) {
      const MemberRange& r = R[s];
      if (r.e <= r.b) continue;
      const size_t ld = static_cast<size_t>(qmcg::table_ld(r.e - r.b));
      for (size_t k = 0; k < cnt; ++k)
        QMCG_CUDA(cudaMemcpyPeerAsync(M[s]->table + static_cast<size_t>(dst_row[k0 + k]) * ld, M[s]->device,
                                      tmp + k * static_cast<size_t>(n) + r.b, bc->device,
                                      static_cast<size_t>(r.e - r.b) * sizeof(double), bc->stream));
    }
  }
  return QMCG_OK;
}

// Scratch rows a builder holds for the sharded build (~512 MB, at least one row).
int64_t group_tmp_rows(int64_t n) {
  return std::max<int64_t>(1, std::min<int64_t>(8, (int64_t{1} << 29) / (8 * n)));
}

// Resident tables for (seed, n) rows [0, m) on every member, each over its range R[s]:
// the missing dims are built dimension-sharded and scattered to the members.
qmcg_status group_ensure_tables(qmcg_ctx* g, uint64_t seed, int64_t n, int64_t m, const std::vector<MemberRange>& R,
                                bool rebuild) {
  const auto& M = g->members;
  int64_t d0 = m;
  for (size_t s = 0; s < M.size(); ++s) {
    qmcg_ctx* c = M[s];
    const bool same = !rebuild && c->cache_n == n && c->cache_seed == seed && c->col_begin == R[s].b &&
                      c->col_end == R[s].e;
    d0 = std::min(d0, R[s].e > R[s].b ? (same ? c->cache_dims : 0) : m);
  }
  if (d0 >= m) return QMCG_OK;
  NvtxRange nv("qmcg.group.sharded_table_build");
  for (size_t s = 0; s < M.size(); ++s) {
    if (R[s].e <= R[s].b) continue;
    DeviceGuard dg(M[s]->device);
    qmcg_status st = ensure_dim_tables(M[s], n, m);
    if (st) return st;
    st = reserve_table(M[s], seed, n, R[s].b, R[s].e, m, rebuild);
    if (st) return st;
    M[s]->cache_dims = std::min(M[s]->cache_dims, d0);
  }
  for (qmcg_ctx* c : M) {
    qmcg_status st = ensure_events(c);
    if (st) return st;
  }
  // member tables may still be read by queued pricing: the builders start after it
  qmcg_status st = cross_wait(M, M, false);
  if (st) return st;
  const int G = static_cast<int>(M.size());
  const int64_t tmp_rows = group_tmp_rows(n);
  for (int r = 0; r < G; ++r) {
    std::vector<int64_t> dims;
    for (int64_t d = d0; d < m; ++d)
      if (d % G == r) dims.push_back(d);
    if (dims.empty()) continue;
    qmcg_ctx* bc = M[static_cast<size_t>(r)];
    DeviceGuard dg(bc->device);
    QMCG_CUDA(bc->d_gtmp.reserve(static_cast<size_t>(tmp_rows) * static_cast<size_t>(n)));
    st = build_and_scatter(bc, seed, n, dims, dims, M, R, bc->d_gtmp.ptr, tmp_rows);
    if (st) return st;
  }
  st = cross_wait(M, M, true);  // every member prices only after every builder's copies
  if (st) return st;
  for (size_t s = 0; s < M.size(); ++s)
    if (R[s].e > R[s].b) M[s]->cache_dims = m;
  return QMCG_OK;
}

// Tables of a group pricing that exceed a member's memory: date windows of W rows (the same W
// on every member); each window's dims are built dimension-sharded and scattered into the
// members' window buffers, then every member walks its paths through the window (K2 with the
// walk state carried in HBM, as enqueue_streamed). Returns the node sums via enqueue_results.
qmcg_status group_enqueue_streamed(qmcg_ctx* g, std::vector<CallPlan>& plans, uint64_t seed, int64_t n, int64_t m,
                                   int depth, const std::vector<MemberRange>& R) {
  NvtxRange nv("qmcg.group.streamed_windows");
  const auto& M = g->members;
  const int G = static_cast<int>(M.size());
  int64_t W = (m + 7) / 8 * 8;
  for (size_t s = 0; s < M.size(); ++s) {
    if (R[s].e <= R[s].b) continue;
    DeviceGuard dg(M[s]->device);
    drop_cache(M[s]);
    const int64_t cols = R[s].e - R[s].b;
    const size_t row_bytes = static_cast<size_t>(qmcg::table_ld(cols)) * sizeof(double);
    // the builder scratch (one full row) lives on every member as well
    size_t budget = table_bytes_allowed(M[s], n, cols, false);
    budget = budget > static_cast<size_t>(n) * 8 ? budget - static_cast<size_t>(n) * 8 : 0;
    W = std::min<int64_t>(W, static_cast<int64_t>(budget / row_bytes) / 8 * 8);
  }
  if (W < 8) return fail(QMCG_OUT_OF_MEMORY, "price_american: not enough device memory for 8 uniform-table rows");
  std::vector<PriceParams> P(M.size());
  for (size_t s = 0; s < M.size(); ++s) {
    qmcg_ctx* c = M[s];
    DeviceGuard dg(c->device);
    qmcg_status st = ensure_events(c);
    if (st) return st;
    QMCG_CUDA(c->d_gtmp.reserve(static_cast<size_t>(n)));
    if (R[s].e <= R[s].b) continue;
    const int64_t cols = R[s].e - R[s].b;
    const int64_t ld = qmcg::table_ld(cols);
    double* nt = nullptr;
    if (dev_alloc(reinterpret_cast<void**>(&nt), static_cast<size_t>(ld) * 8 * static_cast<size_t>(W) + qmcg::kTablePad * 8) != cudaSuccess) {
      cudaGetLastError();
      return fail(QMCG_OUT_OF_MEMORY, "price_american: uniform-table window does not fit in device memory");
    }
    c->table = nt;
    c->table_rows_cap = static_cast<size_t>(W);
    c->col_begin = R[s].b;  // a window buffer, never a cache (cache_n stays -1)
    c->col_end = R[s].e;
    QMCG_CUDA(c->d_values.reserve(static_cast<size_t>(cols)));
    QMCG_CUDA(c->d_red.reserve(qmcg::reduce_scratch_doubles(cols)));
    for (auto* buf : {&c->d_stV, &c->d_stc, &c->d_stcd, &c->d_stbest}) QMCG_CUDA(buf->reserve(static_cast<size_t>(cols)));
    QMCG_CUDA(c->d_stpend.reserve(static_cast<size_t>(cols)));
    PriceParams& p = P[s];
    p = plans[s].P;
    p.table = c->table;
    p.ld = ld;
    p.col_begin = R[s].b;
    p.path_begin = R[s].b;
    p.path_count = cols;
    p.values = c->d_values.ptr;
    p.err = c->d_err.ptr;
    p.st_V = c->d_stV.ptr;
    p.st_c = c->d_stc.ptr;
    p.st_cd = c->d_stcd.ptr;
    p.st_best = c->d_stbest.ptr;
    p.st_pend = c->d_stpend.ptr;
    c->last_windows = 0;
  }
  qmcg_status st = cross_wait(M, M, false);
  if (st) return st;
  for (int64_t d0 = 0; d0 < m; d0 += W) {
    const int64_t d1 = std::min(m, d0 + W);
    for (int r = 0; r < G; ++r) {
      std::vector<int64_t> dims, rows;
      for (int64_t d = d0; d < d1; ++d)
        if (d % G == r) {
          dims.push_back(d);
          rows.push_back(d - d0);
        }
      if (dims.empty()) continue;
      qmcg_ctx* bc = M[static_cast<size_t>(r)];
      st = build_and_scatter(bc, seed, n, dims, rows, M, R, bc->d_gtmp.ptr, 1);
      if (st) return st;
    }
    st = cross_wait(M, M, true);  // the window's rows are in place on every member
    if (st) return st;
    for (size_t s = 0; s < M.size(); ++s) {
      if (R[s].e <= R[s].b) continue;
      qmcg_ctx* c = M[s];
      DeviceGuard dg(c->device);
      PriceParams& p = P[s];
      p.d_begin = static_cast<int32_t>(d0);
      p.d_end = static_cast<int32_t>(d1);
      p.perm_row0 = static_cast<int32_t>(d0);
      p.stream_load = d0 > 0;
      p.stream_store = d1 < m;
      QMCG_CUDA(qmcg::launch_price(p, c->stream));
      c->launches += 1;
      c->last_windows += 1;
    }
    if (d1 < m) {
      st = cross_wait(M, M, false);  // the next window's copies overwrite rows the walk reads
      if (st) return st;
    }
  }
  for (size_t s = 0; s < M.size(); ++s) {
    if (R[s].e <= R[s].b) continue;
    DeviceGuard dg(M[s]->device);
    st = enqueue_node_sums(M[s], n, depth, R[s].node0, R[s].count, R[s].b);
    if (st) return st;
    st = enqueue_results(M[s], static_cast<size_t>(R[s].count));
    if (st) return st;
  }
  return QMCG_OK;
}

// price_american over a device group: (sum v, sum v^2) of every node at the group depth into
// `sums` (2 per node), folded by the caller.
qmcg_status group_price_nodes(qmcg_ctx* g, const qmcg_option_spec& spec, int64_t m, int64_t n, uint64_t seed,
                              uint32_t flags, int& depth, std::vector<double>& sums) {
  const auto& M = g->members;
  const int G = static_cast<int>(M.size());
  CallPlan probe;
  qmcg_status st = plan_call(spec, m, n, flags, probe);  // the reference's checks, before any device work
  if (st) return st;
  depth = group_depth(n, G);
  const std::vector<MemberRange> R = member_ranges(n, G, depth);
  sums.assign(2 * (size_t{1} << depth), 0.0);
  for (qmcg_ctx* c : M) c->launches = 0;
  const bool rebuild = (flags & QMCG_FLAG_NO_CACHE) != 0;
  // tables: resident (the cached slices, or a sharded build) unless a slice exceeds its member's memory
  bool streamed = false;
  if (!probe.P.deterministic) {
    for (size_t s = 0; s < M.size(); ++s) {
      const MemberRange& r = R[s];
      if (r.e <= r.b) continue;
      qmcg_ctx* c = M[s];
      const bool cached = !rebuild && c->cache_n == n && c->cache_seed == seed && c->col_begin == r.b &&
                          c->col_end == r.e && c->cache_dims >= m;
      if (cached) continue;
      DeviceGuard dg(c->device);
      const size_t need = static_cast<size_t>(qmcg::table_ld(r.e - r.b)) * 8 * static_cast<size_t>(m) +
                          static_cast<size_t>(group_tmp_rows(n)) * static_cast<size_t>(n) * 8;
      if (need > table_bytes_allowed(c, n, r.e - r.b, false)) streamed = true;
    }
  }
  if (streamed) {
    std::vector<CallPlan> plans(M.size());
    for (size_t s = 0; s < M.size(); ++s) {
      DeviceGuard dg(M[s]->device);
      plans[s] = probe;
      st = upload_plan(M[s], plans[s], n);
      if (st) return st;
      st = prepare_scratch(M[s], static_cast<size_t>(std::max<int64_t>(R[s].count, 1)));
      if (st) return st;
    }
    st = group_enqueue_streamed(g, plans, seed, n, m, depth, R);
    if (st) return st;
  } else {
    if (!probe.P.deterministic) {
      st = group_ensure_tables(g, seed, n, m, R, rebuild);
      if (st) return st;
    }
    // every member prices its nodes on its own host thread (flags without NO_CACHE: the slices are in
    // place, a cold call rebuilt them above); the node sums land in disjoint parts of `sums`
    std::vector<qmcg_status> res(M.size(), QMCG_OK);
    std::vector<std::string> msg(M.size());
    const uint32_t mflags = flags & ~static_cast<uint32_t>(QMCG_FLAG_NO_CACHE);
    for (size_t s = 0; s < M.size(); ++s) {
      if (!R[s].count) continue;
      g->workers[s]->submit([&, s] {
        DeviceGuard dg(M[s]->device);
        res[s] = price_nodes(M[s], &spec, m, n, seed, mflags, depth, R[s].node0, R[s].count,
                             sums.data() + 2 * R[s].node0);
        if (res[s]) msg[s] = g_last_error;  // thread-local: carried to the caller's thread
      });
    }
    for (size_t s = 0; s < M.size(); ++s)
      if (R[s].count) g->workers[s]->wait();
    for (size_t s = 0; s < M.size(); ++s)
      if (res[s]) return fail(res[s], msg[s]);
    return QMCG_OK;
  }
  for (size_t s = 0; s < M.size(); ++s) {
    if (!R[s].count) continue;
    DeviceGuard dg(M[s]->device);
    st = finish_results(M[s], static_cast<size_t>(R[s].count), sums.data() + 2 * R[s].node0);
    if (st) return st;
  }
  return QMCG_OK;
}

// ---- group forms of the remaining context calls ----
qmcg_status group_warm(qmcg_ctx* g, int64_t n, uint64_t seed, int64_t dims) {
  const int G = static_cast<int>(g->members.size());
  const int depth = group_depth(n, G);
  qmcg_status st = group_ensure_tables(g, seed, n, dims, member_ranges(n, G, depth), false);
  if (st) return st;
  for (qmcg_ctx* c : g->members) {
    DeviceGuard dg(c->device);
    QMCG_CUDA(cudaStreamSynchronize(c->stream));
  }
  return QMCG_OK;
}

// Config 4 on a group: contract blocks [C r / G, C (r + 1) / G) per member, every member with
// the full tables (built dimension-sharded once), the member batches run concurrently (one
// host thread each; a batch call is synchronous).
qmcg_status group_batch(qmcg_ctx* g, const qmcg_option_spec* specs, int64_t n_specs, int64_t m, int64_t n,
                        uint64_t seed, uint32_t flags, qmcg_pricing_result* out) {
  const auto& M = g->members;
  const int G = static_cast<int>(M.size());
  for (int64_t i = 0; i < n_specs; ++i) {  // the reference's checks before any device work
    CallPlan probe;
    qmcg_status st = plan_call(specs[i], m, n, flags, probe);
    if (st) return st;
  }
  if (n_specs == 0) return QMCG_OK;
  std::vector<MemberRange> full(M.size());
  for (auto& r : full) {
    r.b = 0;
    r.e = n;
  }
  qmcg_status st = group_ensure_tables(g, seed, n, m, full, (flags & QMCG_FLAG_NO_CACHE) != 0);
  if (st) return st;
  const uint32_t mflags = flags & ~static_cast<uint32_t>(QMCG_FLAG_NO_CACHE);
  std::vector<qmcg_status> res(M.size(), QMCG_OK);
  std::vector<std::string> msg(M.size());
  for (int r = 0; r < G; ++r) {
    const int64_t b = n_specs * r / G, e = n_specs * (r + 1) / G;
    if (e <= b) continue;
    g->workers[static_cast<size_t>(r)]->submit([&, r, b, e] {
      res[r] = qmcg_price_american_batch(M[r], specs + b, e - b, m, n, seed, mflags, out + b);
      if (res[r]) msg[r] = g_last_error;  // thread-local: carry the text to the caller's thread
    });
  }
  for (int r = 0; r < G; ++r)
    if (n_specs * (r + 1) / G > n_specs * r / G) g->workers[static_cast<size_t>(r)]->wait();
  for (int r = 0; r < G; ++r)
    if (res[r]) return fail(res[r], msg[r]);
  return QMCG_OK;
}

qmcg_status group_path_values(qmcg_ctx* g, const qmcg_option_spec& spec, int64_t m, int64_t n, uint64_t seed,
                              uint32_t flags, double* out_host) {
  int depth = 0;
  std::vector<double> sums;
  qmcg_status st = group_price_nodes(g, spec, m, n, seed, flags, depth, sums);
  if (st) return st;
  const auto R = member_ranges(n, static_cast<int>(g->members.size()), depth);
  for (size_t s = 0; s < g->members.size(); ++s) {
    if (R[s].e <= R[s].b) continue;
    qmcg_ctx* c = g->members[s];
    DeviceGuard dg(c->device);
    QMCG_CUDA(cudaMemcpyAsync(out_host + R[s].b, c->d_values.ptr, static_cast<size_t>(R[s].e - R[s].b) * sizeof(double),
                              cudaMemcpyDeviceToHost, c->stream));
    QMCG_CUDA(cudaStreamSynchronize(c->stream));
  }
  return QMCG_OK;
}

// Every member prices its node range `reps` times (launched round-robin so the devices run
// concurrently); the pricing-kernel and whole-step device times are the max over members.
qmcg_status group_time_device(qmcg_ctx* g, const qmcg_option_spec& spec, int64_t m, int64_t n, uint64_t seed,
                              uint32_t flags, int reps, double* kernel_ms, double* step_ms, double* price_se) {
  const auto& M = g->members;
  int depth = 0;
  std::vector<double> sums;
  qmcg_status st = group_price_nodes(g, spec, m, n, seed, flags, depth, sums);  // tables + module warm-up
  if (st) return st;
  const auto R = member_ranges(n, static_cast<int>(M.size()), depth);
  std::vector<CallPlan> plans(M.size());
  std::vector<double> kms(M.size(), 0.0);
  for (size_t s = 0; s < M.size(); ++s) {
    if (!R[s].count) continue;
    DeviceGuard dg(M[s]->device);
    st = plan_call(spec, m, n, flags, plans[s]);
    if (st) return st;
    st = upload_plan(M[s], plans[s], n);
    if (st) return st;
    st = prepare_scratch(M[s], static_cast<size_t>(R[s].count));
    if (st) return st;
    QMCG_CUDA(cudaEventRecord(M[s]->ev[2], M[s]->stream));
  }
  for (int rep = 0; rep < reps; ++rep) {
    for (size_t s = 0; s < M.size(); ++s) {
      if (!R[s].count) continue;
      qmcg_ctx* c = M[s];
      DeviceGuard dg(c->device);
      QMCG_CUDA(cudaEventRecord(c->ev[0], c->stream));
      st = enqueue_values(c, plans[s], R[s].b, R[s].e, c->ev[1]);
      if (st) return st;
      st = enqueue_node_sums(c, n, depth, R[s].node0, R[s].count, R[s].b);
      if (st) return st;
    }
    for (size_t s = 0; s < M.size(); ++s) {
      if (!R[s].count) continue;
      DeviceGuard dg(M[s]->device);
      QMCG_CUDA(cudaEventSynchronize(M[s]->ev[1]));
      float ms = 0.f;
      QMCG_CUDA(cudaEventElapsedTime(&ms, M[s]->ev[0], M[s]->ev[1]));
      kms[s] += ms;
    }
  }
  double kmax = 0.0, smax = 0.0;
  for (size_t s = 0; s < M.size(); ++s) {
    if (!R[s].count) continue;
    qmcg_ctx* c = M[s];
    DeviceGuard dg(c->device);
    QMCG_CUDA(cudaEventRecord(c->ev[3], c->stream));
    st = enqueue_results(c, static_cast<size_t>(R[s].count));
    if (st) return st;
    st = finish_results(c, static_cast<size_t>(R[s].count), sums.data() + 2 * R[s].node0);
    if (st) return st;
    float total = 0.f;
    QMCG_CUDA(cudaEventElapsedTime(&total, c->ev[2], c->ev[3]));
    kmax = std::max(kmax, kms[s] / reps);
    smax = std::max(smax, static_cast<double>(total) / reps);
  }
  fold_nodes(sums, depth);
  if (kernel_ms) *kernel_ms = kmax;
  if (step_ms) *step_ms = smax;
  if (price_se) finish_stats(n, sums[0], sums[1], price_se[0], price_se[1]);
  return QMCG_OK;
}

// Cold sharded build of the pricing slices for dims [0, dims), host wall clock around the
// group (ms): every member is idle before, and all of them have finished after.
qmcg_status group_time_perm_build(qmcg_ctx* g, int64_t n, uint64_t seed, int64_t dims, double* ms) {
  const int G = static_cast<int>(g->members.size());
  const auto R = member_ranges(n, G, group_depth(n, G));
  qmcg_status st = group_ensure_tables(g, seed, n, dims, R, false);  // allocation outside the timing
  if (st) return st;
  for (qmcg_ctx* c : g->members) {
    DeviceGuard dg(c->device);
    QMCG_CUDA(cudaStreamSynchronize(c->stream));
    c->cache_dims = 0;
  }
  const auto t0 = std::chrono::steady_clock::now();
  st = group_ensure_tables(g, seed, n, dims, R, false);
  if (st) return st;
  for (qmcg_ctx* c : g->members) {
    DeviceGuard dg(c->device);
    QMCG_CUDA(cudaStreamSynchronize(c->stream));
  }
  *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return QMCG_OK;
}

}  // namespace

extern "C" {

qmcg_status qmcg_price_american(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                                uint32_t flags, qmcg_pricing_result* out) {
  if (!c || !spec || !out) return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american: null argument");
  NvtxRange nv("qmcg_price_american");
  const auto t0 = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  double sums[2];
  qmcg_status st;
  if (!c->members.empty()) {  // device group: nodes sharded over the members, folded here
    int depth = 0;
    std::vector<double> t;
    st = group_price_nodes(c, *spec, m, n, seed, flags, depth, t);
    if (st) return st;
    fold_nodes(t, depth);
    sums[0] = t[0];
    sums[1] = t[1];
  } else {
    st = price_range(c, spec, m, n, seed, flags, sums);
    if (st) return st;
  }
  double mean, se;
  finish_stats(n, sums[0], sums[1], mean, se);
  out->price = mean;
  out->std_error = se;
  out->n_paths = n;
  out->method = QMCG_METHOD_AMERICAN_UB;
  out->seed = seed;
  out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return QMCG_OK;
}

qmcg_status qmcg_mc_european_price(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t n, uint64_t seed,
                                   uint32_t flags, qmcg_pricing_result* out) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!c || !spec || !out) return fail(QMCG_INVALID_ARGUMENT, "qmcg_mc_european_price: null argument");
  const auto t0 = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  (void)flags;
  qmcg_status st = validate(*spec);
  if (st) return st;
  if (n < 2) return fail(QMCG_INVALID_ARGUMENT, "mc_european_price: n_paths must be >= 2");
  const double r = spec->rate, v = spec->volatility, T = spec->maturity;
  out->n_paths = n;
  out->method = QMCG_METHOD_EUROPEAN_MC;
  out->seed = seed;
  if (v == 0.0 || T == 0.0) {  // mc_european.cpp:20-28, exact host arithmetic
    const double disc = std::exp(-r * T);
    const double forward = spec->spot * std::exp(r * T);
    out->price = disc * intrinsic(spec->kind, forward, spec->strike);
    out->std_error = 0.0;
    out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return QMCG_OK;
  }
  if (static_cast<uint64_t>(n) > 0xffffffffULL)
    return fail(QMCG_LENGTH_ERROR, "permutation_indices: n exceeds the 2^32-1 supported maximum");
  st = ensure_dim_tables(c, n, 1);
  if (st) return st;
  st = ensure_perms(c, seed, n, 0, n, 1, false);  // dimension 0 only (reuses a larger cached set)
  if (st) return st;
  st = prepare_scratch(c, 1);
  if (st) return st;
  QMCG_CUDA(c->d_values.reserve(static_cast<size_t>(n)));
  QMCG_CUDA(c->d_red.reserve(qmcg::reduce_scratch_doubles(n)));
  const double a = (r - 0.5 * v * v) * T;  // gbm_step with dt = T
  const double bsd = v * std::sqrt(T);
  const double disc = std::exp(-r * T);
  QMCG_CUDA(qmcg::launch_european(c->table, n, spec->spot, a, bsd, spec->strike, disc, spec->kind, c->d_values.ptr,
                                  c->stream));
  int launches = 1;
  QMCG_CUDA(qmcg::launch_pairwise(c->d_values.ptr, n, c->d_red.ptr, c->d_sums.ptr, c->stream, &launches));
  c->launches += launches;
  std::vector<double> sums;
  st = sync_results(c, 1, sums);
  if (st) return st;
  finish_stats(n, sums[0], sums[1], out->price, out->std_error);
  out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return QMCG_OK;
}

qmcg_status qmcg_price_american_node(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n,
                                     uint64_t seed, uint32_t flags, int depth, int64_t node, double out_sums[2]) {
  if (c && !c->members.empty())
    return fail(QMCG_UNSUPPORTED, "qmcg_price_american_node: a per-device call (use a single-device context per rank)");
  if (!c || !spec || !out_sums) return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_node: null argument");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  if (depth < 0 || depth > 30 || node < 0 || node >= (int64_t{1} << depth))
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_node: bad node");
  int64_t off, size;
  tree_node(n, depth, node, off, size);
  // every ancestor of the node must be an internal (split) node of the reference tree
  {
    int64_t aoff, asize;
    for (int d = 0; d < depth; ++d) {
      tree_node(n, d, node >> (depth - d), aoff, asize);
      if (asize <= 64) return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_node: node below a leaf of the tree");
    }
  }
  return price_nodes(c, spec, m, n, seed, flags, depth, node, 1, out_sums);
}

qmcg_status qmcg_price_american_nodes(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n,
                                      uint64_t seed, uint32_t flags, int depth, int64_t node_begin,
                                      int64_t node_count, double* out_sums) {
  if (c && !c->members.empty())
    return fail(QMCG_UNSUPPORTED, "qmcg_price_american_nodes: a per-device call (use a single-device context per rank)");
  if (!c || !spec || !out_sums) return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_nodes: null argument");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  if (depth < 0 || depth > 30 || node_count < 1 || node_begin < 0 ||
      node_begin + node_count > (int64_t{1} << depth))
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_nodes: bad node range");
  int64_t aoff, asize;
  for (int64_t k = node_begin; k < node_begin + node_count; ++k)
    for (int d = 0; d < depth; ++d) {
      tree_node(n, d, k >> (depth - d), aoff, asize);
      if (asize <= 64)
        return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_nodes: node below a leaf of the tree");
    }
  return price_nodes(c, spec, m, n, seed, flags, depth, node_begin, node_count, out_sums);
}

static qmcg_status batch_impl(qmcg_ctx* c, const qmcg_option_spec* specs, int64_t n_specs, int64_t m, int64_t n,
                              uint64_t seed, uint32_t flags, qmcg_pricing_result* out, double* values_host);

qmcg_status qmcg_price_american_batch(qmcg_ctx* c, const qmcg_option_spec* specs, int64_t n_specs, int64_t m,
                                      int64_t n, uint64_t seed, uint32_t flags, qmcg_pricing_result* out) {
  return batch_impl(c, specs, n_specs, m, n, seed, flags, out, nullptr);
}

qmcg_status qmcg_price_american_batch_values(qmcg_ctx* c, const qmcg_option_spec* specs, int64_t n_specs, int64_t m,
                                             int64_t n, uint64_t seed, uint32_t flags, qmcg_pricing_result* out,
                                             double* values_host) {
  if (!values_host) return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_batch_values: null argument");
  if (c && !c->members.empty())
    return fail(QMCG_UNSUPPORTED, "qmcg_price_american_batch_values: a per-device call (single-device context)");
  return batch_impl(c, specs, n_specs, m, n, seed, flags, out, values_host);
}

static qmcg_status batch_impl(qmcg_ctx* c, const qmcg_option_spec* specs, int64_t n_specs, int64_t m, int64_t n,
                              uint64_t seed, uint32_t flags, qmcg_pricing_result* out, double* values_host) {
  if (!c || !specs || !out || n_specs < 0) return fail(QMCG_INVALID_ARGUMENT, "qmcg_price_american_batch: bad argument");
  NvtxRange nv("qmcg_price_american_batch");
  if (flags & QMCG_FLAG_FP32)
    return fail(QMCG_UNSUPPORTED, "qmcg_price_american_batch: QMCG_FLAG_FP32 is not supported (the batch walk is FP64)");
  const auto t0 = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  if (!c->members.empty()) {  // contracts sharded over the group's members
    qmcg_status st = group_batch(c, specs, n_specs, m, n, seed, flags, out);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int64_t i = 0; i < n_specs && st == QMCG_OK; ++i) out[i].elapsed_s = el;
    return st;
  }
  if (n_specs == 0) return QMCG_OK;
  Trace tr("batch");
  std::vector<CallPlan> plans(static_cast<size_t>(n_specs));
  qmcg_status st = plan_call(specs[0], m, n, flags, plans[0]);
  if (st) return st;
  st = ensure_dim_tables(c, n, m);
  if (st) return st;
  st = ensure_perms(c, seed, n, 0, n, m, (flags & QMCG_FLAG_NO_CACHE) != 0);
  if (st) return st;
  st = prepare_scratch(c, static_cast<size_t>(n_specs));
  if (st) return st;
  // The prefix sums S_k of the shared normals depend only on the table: enqueue them before the
  // other contracts are planned, so the device works while the host plans (speculative when the
  // first contract is plain; unused if fewer than two contracts turn out to be)
  const auto plain = [](const PriceParams& P) { return !P.deterministic && !P.check_range && !P.rate_negative; };
  bool z_ready = false;
  if (n_specs >= 2 && plain(plans[0].P)) {
    QMCG_CUDA(c->d_z.reserve(static_cast<size_t>(m + 8) * static_cast<size_t>(n)));  // + 8 prefetch rows
    PriceParams G = plans[0].P;
    G.table = c->table;
    G.ld = qmcg::table_ld(c->col_end - c->col_begin);
    G.col_begin = c->col_begin;
    G.path_begin = 0;
    G.path_count = n;
    G.alpha = 0.0;
    QMCG_CUDA(qmcg::launch_gen_z(G, c->d_z.ptr, n, c->stream, qmcg::kGenPrefix));
    c->launches += 1;
    z_ready = true;
    tr.mark("gen_z enqueued");
  }
  for (int64_t i = 1; i < n_specs; ++i) {
    st = plan_call(specs[i], m, n, flags, plans[static_cast<size_t>(i)], &plans[static_cast<size_t>(i - 1)].dpow);
    if (st) return st;
  }
  tr.mark("plans");
  // discount chains: one per distinct discount factor (a strike/volatility grid shares one), one
  // upload from pageable memory (staged before the call returns: no synchronisation needed)
  c->dpow_host.clear();
  {
    std::vector<double> all;
    std::unordered_map<uint64_t, size_t> seen;  // bits of the discount factor -> chain index
    std::vector<size_t> chain_of(static_cast<size_t>(n_specs));
    for (int64_t i = 0; i < n_specs; ++i) {
      const std::vector<double>& dp = plans[static_cast<size_t>(i)].dpow;
      const auto ins = seen.emplace(bits_of(dp.size() > 1 ? dp[1] : 1.0), seen.size());
      if (ins.second) all.insert(all.end(), dp.begin(), dp.end());
      chain_of[static_cast<size_t>(i)] = ins.first->second;
    }
    QMCG_CUDA(c->d_dpow.reserve(all.size()));
    QMCG_CUDA(cudaMemcpyAsync(c->d_dpow.ptr, all.data(), all.size() * sizeof(double), cudaMemcpyHostToDevice,
                              c->stream));
    for (int64_t i = 0; i < n_specs; ++i)
      plans[static_cast<size_t>(i)].P.dpow =
          c->d_dpow.ptr + chain_of[static_cast<size_t>(i)] * static_cast<size_t>(m + 1);
  }
  tr.mark("dpow");
  // Contracts on the plain path share one normal table (generated once, inside
  // this call) and are walked kCpt per thread; the rest use the fused kernel.
  std::vector<int64_t> shared_idx[2], single_idx;
  for (int64_t i = 0; i < n_specs; ++i) {
    const PriceParams& P = plans[static_cast<size_t>(i)].P;
    if (plain(P)) shared_idx[P.kind].push_back(i);
    else single_idx.push_back(i);
  }
  const bool use_shared = shared_idx[0].size() + shared_idx[1].size() >= 2;
  if (!use_shared)
    for (int k = 0; k < 2; ++k) single_idx.insert(single_idx.end(), shared_idx[k].begin(), shared_idx[k].end());
  for (int64_t i : single_idx) {
    st = enqueue_price(c, plans[static_cast<size_t>(i)], 0, n, static_cast<int>(i), nullptr);
    if (st) return st;
    if (values_host)
      QMCG_CUDA(cudaMemcpyAsync(values_host + static_cast<size_t>(i) * static_cast<size_t>(n), c->d_values.ptr,
                                static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  std::vector<double> shared_sums[2];
  bool tree_on_side = false;
  if (use_shared) {
    if (!z_ready) {
      QMCG_CUDA(c->d_z.reserve(static_cast<size_t>(m + 8) * static_cast<size_t>(n)));  // + 8 prefetch rows
      PriceParams G = plans[static_cast<size_t>(shared_idx[0].empty() ? shared_idx[1][0] : shared_idx[0][0])].P;
      G.table = c->table;
      G.ld = qmcg::table_ld(c->col_end - c->col_begin);
      G.col_begin = c->col_begin;
      G.path_begin = 0;
      G.path_count = n;
      G.alpha = 0.0;
      QMCG_CUDA(qmcg::launch_gen_z(G, c->d_z.ptr, n, c->stream, qmcg::kGenPrefix));
      c->launches += 1;
      tr.mark("gen_z enqueued");
    }
    for (int k = 0; k < 2; ++k) {
      const size_t cnt = shared_idx[k].size();
      if (!cnt) continue;
      // group the contracts that share (spot, rate, volatility, maturity): one walk per group and path
      auto key = [&](int64_t i) {
        const qmcg_option_spec& sp = specs[i];
        return std::array<uint64_t, 4>{bits_of(sp.spot), bits_of(sp.rate), bits_of(sp.volatility),
                                       bits_of(sp.maturity)};
      };
      std::stable_sort(shared_idx[k].begin(), shared_idx[k].end(),
                       [&](int64_t a, int64_t b) { return key(a) < key(b); });
      std::vector<qmcg::GroupParams> groups;
      for (size_t j = 0; j < cnt;) {
        size_t e = j + 1;
        while (e < cnt && key(shared_idx[k][e]) == key(shared_idx[k][j])) ++e;
        const PriceParams& P0 = plans[static_cast<size_t>(shared_idx[k][j])].P;
        qmcg::GroupParams gp{};
        gp.dpow = P0.dpow;
        gp.X0 = P0.X0;
        gp.b = P0.b;
        gp.alpha = P0.alpha;
        gp.beta = k == 0 ? P0.alpha - P0.dom_slope : P0.dom_slope;
        gp.c0 = P0.c0;
        gp.x0mk = P0.x0mk;
        for (size_t t = j; t < e; ++t) {
          const PriceParams& P = plans[static_cast<size_t>(shared_idx[k][t])].P;
          gp.c0 = k == 0 ? std::min(gp.c0, P.c0) : std::max(gp.c0, P.c0);
          gp.x0mk = std::min(gp.x0mk, P.x0mk);
        }
        gp.bs_vsqrt = P0.bs_vsqrt;
        gp.bs_mu_t = P0.bs_mu_t;
        gp.bs_fwd_growth = P0.bs_fwd_growth;
        gp.bs_disc = P0.bs_disc;
        gp.bs_v_zero = P0.bs_v_zero;
        gp.first = static_cast<int32_t>(j);
        gp.count = static_cast<int32_t>(e - j);
        groups.push_back(gp);
        j = e;
      }
      QMCG_CUDA(c->d_groups[k].reserve(groups.size()));
      QMCG_CUDA(cudaMemcpyAsync(c->d_groups[k].ptr, groups.data(), groups.size() * sizeof(qmcg::GroupParams),
                                cudaMemcpyHostToDevice, c->stream));
      std::vector<qmcg::ContractParams> cps(cnt);
      for (size_t j = 0; j < cnt; ++j) {
        const PriceParams& P = plans[static_cast<size_t>(shared_idx[k][j])].P;
        cps[j] = qmcg::ContractParams{P.dpow, P.X0, P.b, P.alpha, P.c0, P.strike, P.best0, P.log_strike,
                                      P.dom_slope, P.bs_vsqrt, P.bs_mu_t, P.bs_kdisc, P.bs_fwd_growth, P.bs_disc,
                                      P.x0mk, 1.0 / P.bs_kdisc, P.bs_v_zero, 0};
      }
      QMCG_CUDA(c->d_cparams[k].reserve(cnt));
      QMCG_CUDA(cudaMemcpyAsync(c->d_cparams[k].ptr, cps.data(), cnt * sizeof(qmcg::ContractParams),
                                cudaMemcpyHostToDevice, c->stream));
      QMCG_CUDA(c->d_bvalues[k].reserve(cnt * static_cast<size_t>(n)));
      QMCG_CUDA(c->d_bred[k].reserve(cnt * qmcg::reduce_scratch_doubles(n)));
      QMCG_CUDA(c->d_bsums[k].reserve(2 * cnt));
      qmcg::BatchParams B{c->d_z.ptr, n, n, static_cast<int32_t>(m), static_cast<int32_t>(cnt), c->d_cparams[k].ptr,
                          c->d_bvalues[k].ptr, c->d_groups[k].ptr, static_cast<int32_t>(groups.size()), 0};
      QMCG_CUDA(qmcg::launch_walk_group(B, k, c->stream));
      int launches = 1;
      // the calls' tree (HBM-bound leaves) runs on a side stream under the puts' walk (issue-bound)
      cudaStream_t ts = c->stream;
      if (k == 0 && !shared_idx[1].empty()) {
        if (!c->side[0]) QMCG_CUDA(cudaStreamCreateWithFlags(&c->side[0], cudaStreamNonBlocking));
        st = ensure_events(c);
        if (st) return st;
        QMCG_CUDA(cudaEventRecord(c->ev_built, c->stream));
        QMCG_CUDA(cudaStreamWaitEvent(c->side[0], c->ev_built, 0));
        ts = c->side[0];
        tree_on_side = true;
      }
      QMCG_CUDA(qmcg::launch_pairwise_batched(c->d_bvalues[k].ptr, n, static_cast<int>(cnt), c->d_bred[k].ptr,
                                              c->d_bsums[k].ptr, ts, &launches));
      if (ts != c->stream) QMCG_CUDA(cudaEventRecord(c->ev_priced, ts));
      c->launches += launches;
      if (values_host)  // parity export: contract shared_idx[k][j] is row j of the kind's value table
        for (size_t j = 0; j < cnt; ++j)
          QMCG_CUDA(cudaMemcpyAsync(values_host + static_cast<size_t>(shared_idx[k][j]) * static_cast<size_t>(n),
                                    c->d_bvalues[k].ptr + j * static_cast<size_t>(n),
                                    static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      shared_sums[k].resize(2 * cnt);  // read back with the other results (no sync between the kinds)
      tr.mark(k == 0 ? "calls enqueued" : "puts enqueued");
    }
    if (tree_on_side) QMCG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_priced, 0));
    for (int k = 0; k < 2; ++k)
      if (!shared_sums[k].empty())
        QMCG_CUDA(cudaMemcpyAsync(shared_sums[k].data(), c->d_bsums[k].ptr, shared_sums[k].size() * sizeof(double),
                                  cudaMemcpyDeviceToHost, c->stream));
  }
  std::vector<double> sums;
  st = sync_results(c, static_cast<size_t>(n_specs), sums);
  if (st) return st;
  if (use_shared)
    for (int k = 0; k < 2; ++k)
      for (size_t j = 0; j < shared_idx[k].size(); ++j) {
        sums[2 * static_cast<size_t>(shared_idx[k][j])] = shared_sums[k][2 * j];
        sums[2 * static_cast<size_t>(shared_idx[k][j]) + 1] = shared_sums[k][2 * j + 1];
      }
  const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int64_t i = 0; i < n_specs; ++i) {
    double mean, se;
    finish_stats(n, sums[2 * static_cast<size_t>(i)], sums[2 * static_cast<size_t>(i) + 1], mean, se);
    out[i].price = mean;
    out[i].std_error = se;
    out[i].n_paths = n;
    out[i].method = QMCG_METHOD_AMERICAN_UB;
    out[i].seed = seed;
    out[i].elapsed_s = el;
  }
  return QMCG_OK;
}

qmcg_status qmcg_permutation(qmcg_ctx* c, int64_t n, uint64_t seed64, uint32_t* out_host) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!c || !out_host) return fail(QMCG_INVALID_ARGUMENT, "qmcg_permutation: null argument");
  if (n < 1) return fail(QMCG_INVALID_ARGUMENT, "permutation_indices: n must be >= 1");
  if (static_cast<uint64_t>(n) > 0xffffffffULL)
    return fail(QMCG_LENGTH_ERROR, "permutation_indices: n exceeds the 2^32-1 supported maximum");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  QMCG_CUDA(c->d_fullperm.reserve(static_cast<size_t>(n)));
  qmcg_status st = build_perm(c, seed64, n, c->d_fullperm.ptr, 0);
  if (st) return st;
  QMCG_CUDA(cudaMemcpyAsync(out_host, c->d_fullperm.ptr, static_cast<size_t>(n) * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

static qmcg_status export_dim(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dim, int normals, double* out_host) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!c || !out_host) return fail(QMCG_INVALID_ARGUMENT, "qmcg_uniforms: null argument");
  if (n < 1) return fail(QMCG_INVALID_ARGUMENT, "QuasiStream: length must be >= 1");
  if (dim < 0) return fail(QMCG_INVALID_ARGUMENT, "QuasiStream: dimensions must be >= 1");
  if (static_cast<uint64_t>(n) > 0xffffffffULL)
    return fail(QMCG_LENGTH_ERROR, "permutation_indices: n exceeds the 2^32-1 supported maximum");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  qmcg_status st = ensure_dim_tables(c, n, dim + 1);
  if (st) return st;
  QMCG_CUDA(c->d_fullperm.reserve(static_cast<size_t>(n)));
  st = build_perm(c, dimension_seed(seed, dim), n, c->d_fullperm.ptr);
  if (st) return st;
  QMCG_CUDA(c->d_values.reserve(static_cast<size_t>(n)));
  QMCG_CUDA(qmcg::launch_uniforms(c->d_fullperm.ptr, n, c->dt.dims[static_cast<size_t>(dim)], c->d_sc.ptr,
                                  c->d_nc.ptr, normals, c->d_values.ptr, c->stream));
  QMCG_CUDA(cudaMemcpyAsync(out_host, c->d_values.ptr, static_cast<size_t>(n) * sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

qmcg_status qmcg_uniforms(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dim, double* out_host) {
  return export_dim(c, n, seed, dim, 0, out_host);
}

qmcg_status qmcg_normals(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dim, double* out_host) {
  return export_dim(c, n, seed, dim, 1, out_host);
}

qmcg_status qmcg_normal_table(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dims, double* out_host) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!c || !out_host || n < 1 || dims < 1) return fail(QMCG_INVALID_ARGUMENT, "qmcg_normal_table: bad argument");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  qmcg_option_spec s{100.0, 100.0, 0.05, 0.2, 1.0, QMCG_CALL};
  CallPlan plan;
  qmcg_status st = plan_call(s, dims, n < 2 ? 2 : n, 0, plan);
  if (st) return st;
  st = upload_plan(c, plan, n);
  if (st) return st;
  st = ensure_perms(c, seed, n, 0, n, dims, false);
  if (st) return st;
  QMCG_CUDA(c->d_z.reserve(static_cast<size_t>(dims) * static_cast<size_t>(n)));
  PriceParams G = plan.P;
  G.table = c->table;
  G.ld = qmcg::table_ld(c->col_end - c->col_begin);
  G.col_begin = c->col_begin;
  G.path_begin = 0;
  G.path_count = n;
  G.alpha = 0.0;
  QMCG_CUDA(qmcg::launch_gen_z(G, c->d_z.ptr, n, c->stream));
  QMCG_CUDA(cudaMemcpyAsync(out_host, c->d_z.ptr, static_cast<size_t>(dims) * static_cast<size_t>(n) * sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

qmcg_status qmcg_uniform_rows(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dim_begin, int64_t dim_count,
                              double* out_host) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!c || !out_host || n < 2 || dim_begin < 0 || dim_count < 1)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_uniform_rows: bad argument");
  if (static_cast<uint64_t>(n) > 0xffffffffULL)
    return fail(QMCG_LENGTH_ERROR, "permutation_indices: n exceeds the 2^32-1 supported maximum");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  const int64_t dims = dim_begin + dim_count;
  qmcg_status st = ensure_perms(c, seed, n, 0, n, dims, false);
  if (st) return st;
  // the uniform table the pricing kernels read (built by uniforms_kernel from K1's permutations)
  const size_t ld = static_cast<size_t>(qmcg::table_ld(n));
  QMCG_CUDA(cudaMemcpy2DAsync(out_host, static_cast<size_t>(n) * sizeof(double),
                              c->table + static_cast<size_t>(dim_begin) * ld, ld * sizeof(double),
                              static_cast<size_t>(n) * sizeof(double), static_cast<size_t>(dim_count),
                              cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

qmcg_status qmcg_path_values(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                             uint32_t flags, double* out_host) {
  if (!c || !spec || !out_host) return fail(QMCG_INVALID_ARGUMENT, "qmcg_path_values: null argument");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  if (!c->members.empty()) return group_path_values(c, *spec, m, n, seed, flags, out_host);
  double sums[2];
  qmcg_status st = price_range(c, spec, m, n, seed, flags, sums);
  if (st) return st;
  QMCG_CUDA(cudaMemcpyAsync(out_host, c->d_values.ptr, static_cast<size_t>(n) * sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return QMCG_OK;
}

// Device time of pricing the tree nodes [node0, node0 + count) at `depth` (their contiguous path
// range; the whole option for depth 0): `reps` launches of the pricing kernel (CUDA events on the
// context stream around the kernel alone) and of the whole device step (kernel + node sums),
// after one untimed launch. sums: 2 per node.
static qmcg_status time_nodes(qmcg_ctx* c, const qmcg_option_spec& spec, int64_t m, int64_t n, uint64_t seed,
                              uint32_t flags, int depth, int64_t node0, int64_t count, int reps, double* kernel_ms,
                              double* step_ms, std::vector<double>& sums) {
  int64_t b, e, off, size;
  tree_node(n, depth, node0, b, size);
  tree_node(n, depth, node0 + count - 1, off, size);
  e = off + size;
  CallPlan plan;
  qmcg_status st = plan_call(spec, m, n, flags, plan);
  if (st) return st;
  st = upload_plan(c, plan, n);
  if (st) return st;
  st = ensure_perms(c, seed, n, b, e, m, false);
  if (st) return st;
  st = prepare_scratch(c, static_cast<size_t>(count));
  if (st) return st;
  st = enqueue_values(c, plan, b, e);  // one untimed launch (module load, caches)
  if (st) return st;
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  c->launches = 0;
  double kms = 0.0;
  QMCG_CUDA(cudaEventRecord(c->ev[2], c->stream));
  for (int r = 0; r < reps; ++r) {
    QMCG_CUDA(cudaEventRecord(c->ev[0], c->stream));
    st = enqueue_values(c, plan, b, e, c->ev[1]);
    if (st) return st;
    st = enqueue_node_sums(c, n, depth, node0, count, b);
    if (st) return st;
    QMCG_CUDA(cudaEventSynchronize(c->ev[1]));
    float ms = 0.f;
    QMCG_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
    kms += ms;
  }
  QMCG_CUDA(cudaEventRecord(c->ev[3], c->stream));
  st = sync_results(c, static_cast<size_t>(count), sums);
  if (st) return st;
  float total = 0.f;
  QMCG_CUDA(cudaEventElapsedTime(&total, c->ev[2], c->ev[3]));
  if (kernel_ms) *kernel_ms = kms / reps;
  if (step_ms) *step_ms = static_cast<double>(total) / reps;
  return QMCG_OK;
}

qmcg_status qmcg_time_device(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                             uint32_t flags, int reps, double* kernel_ms, double* step_ms, double* out_price_se) {
  if (!c || !spec || reps < 1) return fail(QMCG_INVALID_ARGUMENT, "qmcg_time_device: bad argument");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  if (!c->members.empty())
    return group_time_device(c, *spec, m, n, seed, flags, reps, kernel_ms, step_ms, out_price_se);
  std::vector<double> sums;
  qmcg_status st = time_nodes(c, *spec, m, n, seed, flags, 0, 0, 1, reps, kernel_ms, step_ms, sums);
  if (st) return st;
  if (out_price_se) finish_stats(n, sums[0], sums[1], out_price_se[0], out_price_se[1]);
  return QMCG_OK;
}

qmcg_status qmcg_time_device_nodes(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                                   uint32_t flags, int depth, int64_t node_begin, int64_t node_count, int reps,
                                   double* kernel_ms, double* step_ms, double* out_sums) {
  if (!c || !spec || reps < 1 || depth < 0 || depth > 30 || node_count < 1 || node_begin < 0 ||
      node_begin + node_count > (int64_t{1} << depth))
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_time_device_nodes: bad argument");
  if (!c->members.empty())
    return fail(QMCG_UNSUPPORTED, "qmcg_time_device_nodes: a per-device call (use a single-device context per rank)");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  std::vector<double> sums;
  qmcg_status st = time_nodes(c, *spec, m, n, seed, flags, depth, node_begin, node_count, reps, kernel_ms, step_ms,
                              sums);
  if (st) return st;
  if (out_sums) std::copy(sums.begin(), sums.end(), out_sums);
  return QMCG_OK;
}

void* qmcg_get_member_stream(qmcg_ctx* c, int member) {
  if (!c) return nullptr;
  if (c->members.empty()) return member == 0 ? static_cast<void*>(c->stream) : nullptr;
  if (member < 0 || member >= static_cast<int>(c->members.size())) return nullptr;
  return static_cast<void*>(c->members[static_cast<size_t>(member)]->stream);
}

int qmcg_member_device(qmcg_ctx* c, int member) {
  if (!c) return -1;
  if (c->members.empty()) return member == 0 ? c->device : -1;
  if (member < 0 || member >= static_cast<int>(c->members.size())) return -1;
  return c->members[static_cast<size_t>(member)]->device;
}

qmcg_status qmcg_time_perm_build(qmcg_ctx* c, int64_t n, uint64_t seed, int64_t dims, double* ms) {
  if (!c || !ms) return fail(QMCG_INVALID_ARGUMENT, "qmcg_time_perm_build: bad argument");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  if (!c->members.empty()) return group_time_perm_build(c, n, seed, dims, ms);
  // make the table resident and allocated, then invalidate its rows so only
  // the rebuild (K1 for every dimension) is timed
  qmcg_status st = ensure_perms(c, seed, n, 0, n, dims, false);
  if (st) return st;
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  c->cache_dims = 0;
  QMCG_CUDA(cudaEventRecord(c->ev[0], c->stream));
  st = ensure_perms(c, seed, n, 0, n, dims, false);
  if (st) return st;
  QMCG_CUDA(cudaEventRecord(c->ev[1], c->stream));
  QMCG_CUDA(cudaEventSynchronize(c->ev[1]));
  float f = 0.f;
  QMCG_CUDA(cudaEventElapsedTime(&f, c->ev[0], c->ev[1]));
  *ms = f;
  return QMCG_OK;
}

int64_t qmcg_last_launch_count(qmcg_ctx* c) {
  if (!c) return 0;
  int64_t n = c->launches;
  for (qmcg_ctx* m : c->members) n += m->launches;
  return n;
}

void* qmcg_get_stream(qmcg_ctx* c) {
  if (c && !c->members.empty()) c = c->members[0];
  return c ? static_cast<void*>(c->stream) : nullptr;
}

qmcg_status qmcg_fp64_peak(qmcg_ctx* c, double ms, double* inst_per_s) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!c || !inst_per_s || !(ms > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "qmcg_fp64_peak: bad argument");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  int sms = 0;
  QMCG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const int blocks = sms * 8;
  QMCG_CUDA(c->d_values.reserve(static_cast<size_t>(blocks) * 256));
  int iters = 64;
  float f = 0.f;
  for (int rep = 0; rep < 8; ++rep) {  // grow until the launch lasts about `ms`
    QMCG_CUDA(cudaEventRecord(c->ev[0], c->stream));
    QMCG_CUDA(qmcg::launch_dfma_probe(c->d_values.ptr, blocks, iters, c->stream));
    QMCG_CUDA(cudaEventRecord(c->ev[1], c->stream));
    QMCG_CUDA(cudaEventSynchronize(c->ev[1]));
    QMCG_CUDA(cudaEventElapsedTime(&f, c->ev[0], c->ev[1]));
    if (f >= 0.5 * ms) break;
    iters = static_cast<int>(iters * std::min(16.0, std::max(2.0, ms / std::max(f, 1e-3f))));
  }
  *inst_per_s = static_cast<double>(blocks) * 256.0 * iters * 128.0 / (f * 1e-3);
  return QMCG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Path matrix export and per-path sweeps: the reference's
// simulate_batch (path_engine.cpp:124-152) and backward_sweep / sweep_value
// (american.cpp:70-101). The pricing kernel never materialises paths; these are
// the diagnostics that need them.
// ---------------------------------------------------------------------------
namespace {

// check_capacity (path_engine.cpp:20-35): the reference's 128 GiB matrix cap and message.
qmcg_status check_capacity(int64_t n, int64_t points, const char* who) {
  const long double bytes = static_cast<long double>(n) * static_cast<long double>(points) * 8.0L;
  const long double cap = static_cast<long double>(uint64_t{1} << 37);
  if (bytes > cap) {
    char msg[512];
    std::snprintf(msg, sizeof msg, "%s: requested %lld paths x %lld points = %g bytes, above the supported maximum of %g bytes",
                  who, static_cast<long long>(n), static_cast<long long>(points), static_cast<double>(bytes),
                  static_cast<double>(cap));
    return fail(QMCG_LENGTH_ERROR, msg);
  }
  return QMCG_OK;
}

// The reference's checks, in its order, for simulate_batch(spec, make_schedule(m, T), n, seed).
qmcg_status validate_simulation(const qmcg_option_spec& s, int64_t m, int64_t n) {
  if (m < 1) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: m must be >= 1");
  if (!(s.maturity > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: maturity must be > 0");
  qmcg_status st = validate(s);
  if (st) return st;
  if (n < 1) return fail(QMCG_INVALID_ARGUMENT, "simulate_batch: n_paths must be >= 1");
  st = check_capacity(n, m + 1, "simulate_batch");
  if (st) return st;
  if (static_cast<uint64_t>(n) > 0xffffffffULL)
    return fail(QMCG_LENGTH_ERROR, "permutation_indices: n exceeds the 2^32-1 supported maximum");
  if (m + 1 > (int64_t{1} << 26)) return fail(QMCG_LENGTH_ERROR, "simulate_batch: m exceeds the 2^26 supported maximum");
  return QMCG_OK;
}

// The matrix of paths [0, n) at points t_1..t_m, T into c->d_path ([point][path]).
qmcg_status simulate_device(qmcg_ctx* c, const qmcg_option_spec& s, int64_t m, int64_t n, uint64_t seed) {
  if (m < 1) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: m must be >= 1");
  if (!(s.maturity > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: maturity must be > 0");
  qmcg_status st = validate(s);
  if (st) return st;
  if (n < 1) return fail(QMCG_INVALID_ARGUMENT, "simulate_batch: n_paths must be >= 1");
  const int64_t points = m + 1;
  st = check_capacity(n, points, "simulate_batch");
  if (st) return st;
  if (static_cast<uint64_t>(n) > 0xffffffffULL)
    return fail(QMCG_LENGTH_ERROR, "permutation_indices: n exceeds the 2^32-1 supported maximum");
  if (points > (int64_t{1} << 26)) return fail(QMCG_LENGTH_ERROR, "simulate_batch: m exceeds the 2^26 supported maximum");
  st = ensure_dim_tables(c, n, points);
  if (st) return st;
  st = ensure_perms(c, seed, n, 0, n, points, false);
  if (st) return st;
  QMCG_CUDA(c->d_path.reserve(static_cast<size_t>(n) * static_cast<size_t>(points)));
  QMCG_CUDA(c->d_err.reserve(1));
  QMCG_CUDA(cudaMemsetAsync(c->d_err.ptr, 0, sizeof(uint32_t), c->stream));
  const double dt = s.maturity / static_cast<double>(points);  // make_schedule
  const double a = (s.rate - 0.5 * s.volatility * s.volatility) * dt;
  const double bsd = s.volatility * std::sqrt(dt);
  QMCG_CUDA(qmcg::launch_path_matrix(c->table, qmcg::table_ld(n), n, static_cast<int>(points), s.spot, a, bsd,
                                     c->d_path.ptr, c->d_err.ptr, c->stream));
  c->launches += 1;
  return QMCG_OK;
}

// cnd (analytic.cpp:33-72), restated for the host sweep.
double cnd_host(double d) {
  const double x = std::fabs(d);
  double tail = 0.0;
  if (x <= 37.0) {
    const double e = std::exp(-0.5 * x * x);
    if (x < 7.07106781186547) {
      static const double P[7] = {3.52624965998911e-02, 0.700383064443688, 6.37396220353165, 33.912866078383,
                                  112.079291497871,     221.213596169931,  220.206867912376};
      static const double Q[8] = {8.83883476483184e-02, 1.75566716318264,  16.064177579207,  86.7807322029461,
                                  296.564248779674,     637.333633378831,  793.826512519948, 440.413735824752};
      double num = P[0], den = Q[0];
      for (int i = 1; i < 7; ++i) num = num * x + P[i];
      for (int i = 1; i < 8; ++i) den = den * x + Q[i];
      tail = e * num / den;
    } else {
      double b = x + 0.65;
      for (double k = 4.0; k >= 1.0; k -= 1.0) b = x + k / b;
      tail = e / (b * 2.506628274631000502);
    }
  }
  return d > 0.0 ? 1.0 - tail : tail;
}

// bs_price (analytic.cpp:102-124) for a spec already validated.
double bs_price_host(double s, double x, double r, double v, double t, int kind) {
  if (t == 0.0) return intrinsic(kind, s, x);
  if (v == 0.0) return std::exp(-r * t) * intrinsic(kind, s * std::exp(r * t), x);
  const double vst = v * std::sqrt(t);
  const double d1 = (std::log(s / x) + (r + 0.5 * v * v) * t) / vst;
  const double d2 = d1 - vst;
  const double disc = std::exp(-r * t);
  const double price = kind == QMCG_CALL ? s * cnd_host(d1) - x * disc * cnd_host(d2)
                                         : x * disc * cnd_host(-d2) - s * cnd_host(-d1);
  return price > 0.0 ? price : 0.0;
}

}  // namespace

qmcg_status qmcg_simulate_batch(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                                uint32_t flags, int layout, double* out_host) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!spec) return fail(QMCG_INVALID_ARGUMENT, "qmcg_simulate_batch: null argument");
  if (layout != QMCG_LAYOUT_PATH_MAJOR && layout != QMCG_LAYOUT_POINT_MAJOR)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_simulate_batch: bad layout");
  if (!out_host) return validate_simulation(*spec, m, n);  // validation only (size the caller's buffer)
  if (!c) return fail(QMCG_INVALID_ARGUMENT, "qmcg_simulate_batch: null argument");
  (void)flags;
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  qmcg_status st = simulate_device(c, *spec, m, n, seed);
  if (st) return st;
  const int64_t points = m + 1;
  const size_t count = static_cast<size_t>(n) * static_cast<size_t>(points);
  const double* src = c->d_path.ptr;
  if (layout == QMCG_LAYOUT_PATH_MAJOR) {
    QMCG_CUDA(c->d_path_t.reserve(count));
    QMCG_CUDA(qmcg::launch_transpose(c->d_path.ptr, points, n, c->d_path_t.ptr, c->stream));
    c->launches += 1;
    src = c->d_path_t.ptr;
  }
  uint32_t err = 0;
  QMCG_CUDA(cudaMemcpyAsync(out_host, src, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaMemcpyAsync(&err, c->d_err.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return map_err(err & qmcg::ERR_SPOT_NONPOSITIVE);
}

qmcg_status qmcg_sweep_batch(qmcg_ctx* c, const qmcg_option_spec* spec, int64_t m, int64_t n, uint64_t seed,
                             uint32_t flags, double* values_host, int32_t* exercise_host) {
  if (c && !c->members.empty()) c = c->members[0];  // single-device call on a group: its first member
  if (!c || !spec || !values_host || !exercise_host)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_sweep_batch: null argument");
  if (spec->kind != QMCG_CALL && !(flags & QMCG_FLAG_ALLOW_PUT))
    return fail(QMCG_INVALID_ARGUMENT, "backward_sweep: not implemented for puts; the foresight algorithm is call-only");
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard g(c->device);
  c->launches = 0;
  qmcg_status st = simulate_device(c, *spec, m, n, seed);
  if (st) return st;
  QMCG_CUDA(c->d_values.reserve(static_cast<size_t>(n)));
  QMCG_CUDA(c->d_ex.reserve(static_cast<size_t>(n)));
  const double dt = spec->maturity / static_cast<double>(m + 1);
  const double disc = std::exp(-spec->rate * dt);
  QMCG_CUDA(qmcg::launch_sweep(c->d_path.ptr, n, static_cast<int>(m), spec->spot, spec->strike, spec->rate,
                               spec->volatility, dt, disc, spec->kind, c->d_values.ptr, c->d_ex.ptr, c->stream));
  c->launches += 1;
  uint32_t err = 0;
  QMCG_CUDA(cudaMemcpyAsync(values_host, c->d_values.ptr, static_cast<size_t>(n) * sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaMemcpyAsync(exercise_host, c->d_ex.ptr, static_cast<size_t>(n) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaMemcpyAsync(&err, c->d_err.ptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  QMCG_CUDA(cudaStreamSynchronize(c->stream));
  return map_err(err & qmcg::ERR_SPOT_NONPOSITIVE);
}

qmcg_status qmcg_backward_sweep(const double* path, int64_t path_len, const qmcg_option_spec* spec, int64_t m,
                                uint32_t flags, double* values_out, int64_t* exercise_point) {
  if (!path || !spec || !values_out || !exercise_point)
    return fail(QMCG_INVALID_ARGUMENT, "qmcg_backward_sweep: null argument");
  if (m < 1) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: m must be >= 1");
  if (!(spec->maturity > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "make_schedule: maturity must be > 0");
  qmcg_status st = validate(*spec);  // check_sweep_inputs (american.cpp:70-85)
  if (st) return st;
  if (spec->kind != QMCG_CALL && !(flags & QMCG_FLAG_ALLOW_PUT))
    return fail(QMCG_INVALID_ARGUMENT, "backward_sweep: not implemented for puts; the foresight algorithm is call-only");
  if (path_len != m + 1)
    return fail(QMCG_INVALID_ARGUMENT, "backward_sweep: path length does not match the schedule point count");
  const int kind = spec->kind;
  const double K = spec->strike;
  const double dt = spec->maturity / static_cast<double>(m + 1);
  const double disc = std::exp(-spec->rate * dt);
  *exercise_point = -1;
  values_out[m + 1] = intrinsic(kind, path[m], K);  // realised payoff at T
  // last exercise point: intrinsic vs the closed form of the final interval
  double value;
  {
    const double sm = path[m - 1];
    // bs_price validates its OptionSpec{sm, K, r, v, dt} (analytic.cpp:18-31)
    if (!std::isfinite(sm)) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: all fields must be finite");
    if (!(sm > 0.0)) return fail(QMCG_INVALID_ARGUMENT, "OptionSpec: spot must be > 0");
    const double cont = bs_price_host(sm, K, spec->rate, spec->volatility, dt, kind);
    const double intr = intrinsic(kind, sm, K);
    value = intr > cont ? intr : cont;
    values_out[m] = value;
    if (intr > cont) *exercise_point = m;
  }
  for (int64_t i = m - 1; i >= 0; --i) {  // i = 0: the spot (immediate exercise)
    const double si = i >= 1 ? path[i - 1] : spec->spot;
    const double cont = value * disc;
    const double intr = intrinsic(kind, si, K);
    value = intr > cont ? intr : cont;
    values_out[i] = value;
    if (intr > cont) *exercise_point = i;  // walking backward: the last write is the earliest point
  }
  return QMCG_OK;
}
