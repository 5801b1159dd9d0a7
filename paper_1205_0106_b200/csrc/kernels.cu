// B200 (sm_100a) kernels of the American-option QMC pricer.
//
//   K1  perm_build   : bit-exact parallel reconstruction of the reference's
//                      LCG-driven Fisher-Yates permutation (permutation_indices,
//                      reference proj/src/quasi_rng.cpp:48-61).
//   K2  price_kernel : fused per-path forward pass -- scrambled-Halton uniform
//                      (radical_inverse, quasi_rng.cpp:71-83, bit-exact), Moro
//                      inverse normal (analytic.cpp:74-100), log-space GBM
//                      (path_engine.hpp:51-56) and the foresight exercise rule
//                      (american.cpp:32-68) -- with no path matrix in HBM.
//   K3  pairwise     : the reference's fixed-shape pairwise summation
//                      (path_engine.cpp:37-47,191-205) over per-path values.
//   D1  uniforms     : parity export of uniforms / normals.
//
// See DESIGN.md for the derivation of the record-filtered sweep and the
// roofline of each kernel.
#include "qmcg_internal.h"

#include <cub/device/device_radix_sort.cuh>

namespace qmcg {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 8;      // dates per tile (tail compaction window)
constexpr int kRecCap = 64;   // per-warp ring of pending record evaluations
constexpr uint32_t kNone = 0xffffffffu;

// ---------------------------------------------------------------------------
// Scrambled Halton uniform, bit-exact with radical_inverse():
//   value += (double)(index % base) * scale; index /= base; scale *= inv_base
// The digit product is one DFMA on (2^52 + digit): exact operand, one rounding.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double digit_term(uint32_t d, double s, double c) {
  return fma(__hiloint2double(0x43300000, static_cast<int>(d)), s, c);
}

__device__ __forceinline__ uint32_t div_p(uint32_t x, const DimParam& dp) {
  if (dp.flags & DIM_WIDE) return static_cast<uint32_t>(__umul64hi(x, dp.magic64));
  return __umulhi(x, dp.magic) >> dp.shift;
}

__device__ __forceinline__ double halton(uint32_t x, const DimParam& dp, const double* __restrict__ sc,
                                         const double* __restrict__ nc) {
  const double* s = sc + dp.doff;
  const double* c = nc + dp.doff;
  const int D = static_cast<int>(dp.ndig);
  double v;
  if (D == 1) {
    v = digit_term(x, __ldg(s), __ldg(c));
  } else {
    uint32_t q = div_p(x, dp);
    v = digit_term(x - q * dp.p, __ldg(s), __ldg(c));
    x = q;
    for (int j = 1; j < D - 1; ++j) {
      q = div_p(x, dp);
      v = __dadd_rn(v, digit_term(x - q * dp.p, __ldg(s + j), __ldg(c + j)));
      x = q;
    }
    v = __dadd_rn(v, digit_term(x, __ldg(s + D - 1), __ldg(c + D - 1)));
  }
  if (dp.flags & DIM_CLAMP) {  // kEndpointEps clamp, quasi_rng.cpp:80-81
    if (v < 1e-12) v = 1e-12;
    if (v > 1.0 - 1e-12) v = 1.0 - 1e-12;
  }
  return v;
}

// |y| > 0.42 on the bit pattern (keeps the branch test off the FP64 pipe);
// identical to the reference's `std::abs(y) <= 0.42` partition.
__device__ __forceinline__ bool moro_is_tail(double y) {
  const unsigned long long a = static_cast<unsigned long long>(__double_as_longlong(y)) & 0x7fffffffffffffffull;
  return a > static_cast<unsigned long long>(__double_as_longlong(0.42));
}

__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Beasley-Springer central region of moro_inv_cnd (analytic.cpp:82-94), plus
// the drift offset alpha folded into the final FMA.
__device__ __forceinline__ double moro_central_plus(double y, double alpha) {
  const double r = y * y;
  const double A = fma(fma(fma(-25.44106049637, r, 41.39119773534), r, -18.61500062529), r, 2.50662823884);
  const double B = fma(fma(fma(fma(3.13082909833, r, -21.06224101826), r, 23.08336743743), r,
                           -8.47351093090), r, 1.0);
  return fma(y * A, rcp_nr(B), alpha);
}

// Moro log-log tail polynomial (analytic.cpp:95-99) for w = u or 1-u.
__device__ __forceinline__ double moro_tail_poly(double w) {
  const double z = log(-log(w));
  double x = 0.0000003960315187;
  x = fma(x, z, 0.0000002888167364);
  x = fma(x, z, 0.0000321767881768);
  x = fma(x, z, 0.0003951896511919);
  x = fma(x, z, 0.0038405729373609);
  x = fma(x, z, 0.0276438810333863);
  x = fma(x, z, 0.1607979714918209);
  x = fma(x, z, 0.9761690190917186);
  x = fma(x, z, 0.3374754822726147);
  return x;
}

__device__ __forceinline__ double moro_full(double u) {
  const double y = __dadd_rn(u, -0.5);
  if (!moro_is_tail(y)) return moro_central_plus(y, 0.0);
  const double x = moro_tail_poly(y > 0.0 ? __dadd_rn(1.0, -u) : u);
  return y > 0.0 ? x : -x;
}

// Hart CND (analytic.cpp:33-72).
__device__ double cnd_dev(double d) {
  const double x = fabs(d);
  double tail;
  if (x > 37.0) {
    tail = 0.0;
  } else {
    const double e = exp(-0.5 * x * x);
    if (x < 7.07106781186547) {
      double num = 3.52624965998911e-02;
      num = fma(num, x, 0.700383064443688);
      num = fma(num, x, 6.37396220353165);
      num = fma(num, x, 33.912866078383);
      num = fma(num, x, 112.079291497871);
      num = fma(num, x, 221.213596169931);
      num = fma(num, x, 220.206867912376);
      double den = 8.83883476483184e-02;
      den = fma(den, x, 1.75566716318264);
      den = fma(den, x, 16.064177579207);
      den = fma(den, x, 86.7807322029461);
      den = fma(den, x, 296.564248779674);
      den = fma(den, x, 637.333633378831);
      den = fma(den, x, 793.826512519948);
      den = fma(den, x, 440.413735824752);
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
  return d > 0.0 ? 1.0 - tail : tail;
}

__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

struct WarpSmem {
  double tail_w[kTile * 32];
  double zres[kTile * 32];
  double rq_v[kRecCap];
  unsigned long long best[32];
  uint32_t rq_code[kRecCap];
  unsigned char tail_owner[kTile * 32];
};

template <int KIND, bool RNEG>
__device__ __forceinline__ void process_records(const PriceParams& P, WarpSmem& S, uint32_t head,
                                                uint32_t count, int lane) {
  if (static_cast<uint32_t>(lane) < count) {
    const uint32_t slot = (head + lane) & (kRecCap - 1);
    const double v = S.rq_v[slot];
    const uint32_t code = S.rq_code[slot];
    const int d = static_cast<int>(code >> 5);
    const int owner = static_cast<int>(code & 31u);
    const double s = exp(fma(P.b, v, P.X0));
    double intr = KIND == 0 ? s - P.strike : P.strike - s;
    intr = intr > 0.0 ? intr : 0.0;
    const double term = intr * __ldg(P.dpow + d + 1);
    atomicMax(&S.best[owner], static_cast<unsigned long long>(__double_as_longlong(term)));
  }
}

// Threshold in V units below/above which a date cannot beat `best` when
// disc > 1 (rate < 0): I_k * dmax <= best.
template <int KIND>
__device__ __forceinline__ double rneg_threshold(const PriceParams& P, double best) {
  const double lim = best * P.dmax_inv;
  if (KIND == 0) return (log(P.strike + lim) - P.X0) / P.b;
  const double room = P.strike - lim;
  return room > 0.0 ? (log(room) - P.X0) / P.b : -INFINITY;
}

// One thread = one path. Dates are processed in tiles of kTile: the uniforms
// and central normals of a tile are computed lane-parallel, the Moro tail
// evaluations (16% of points, two logs each) are compacted across the warp,
// then the log-price walk V_k = sum (z_j + alpha) runs over the tile. A date k
// can only set the foresight maximum max_k disc^k * I_k if I_k exceeds every
// earlier intrinsic (disc <= 1), i.e. V_k sets a new running extreme; those
// "records" are queued per warp and evaluated 32 at a time (exp + discount).
template <int KIND, bool RNEG>
__global__ void __launch_bounds__(kThreads, 2) price_kernel(const PriceParams P) {
  __shared__ WarpSmem smem[kWarps];
  WarpSmem& S = smem[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int64_t pi = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
  const bool active = pi < P.path_count;
  const int64_t col = active ? P.path_begin + pi - P.col_begin : 0;
  const uint32_t* colp = P.perm + col;
  const int64_t ld = P.ld;
  const int m = P.m;
  const int mrec = m - 1;
  const bool det = P.deterministic != 0;

  S.best[lane] = static_cast<unsigned long long>(__double_as_longlong(P.best0));
  double V = 0.0;
  double c = P.c0;
  uint32_t rq_head = 0, rq_tail = 0;
  uint32_t err = 0;
  __syncwarp();

  uint32_t nxt[kTile];
#pragma unroll
  for (int t = 0; t < kTile; ++t)
    nxt[t] = (active && !det && t < m) ? ldg_stream(colp + static_cast<int64_t>(t) * ld) : 0u;

  for (int k0 = 0; k0 < m; k0 += kTile) {
    uint32_t cur[kTile];
#pragma unroll
    for (int t = 0; t < kTile; ++t) cur[t] = nxt[t];
#pragma unroll
    for (int t = 0; t < kTile; ++t) {
      const int d = k0 + kTile + t;
      nxt[t] = (active && !det && d < m) ? ldg_stream(colp + static_cast<int64_t>(d) * ld) : 0u;
    }

    double zq[kTile];
    if (det) {
#pragma unroll
      for (int t = 0; t < kTile; ++t) zq[t] = P.alpha;
    } else {
      uint32_t tail_base = 0;
      uint32_t tmask = 0;
#pragma unroll
      for (int t = 0; t < kTile; ++t) {
        const int d = k0 + t;
        zq[t] = 0.0;
        if (d < m) {
          const DimParam dp = P.dims[d];
          const double u = active ? halton(cur[t] + 1u, dp, P.sc, P.nc) : 0.5;
          const double y = __dadd_rn(u, -0.5);
          const bool tail = moro_is_tail(y);
          const unsigned tb = __ballot_sync(kFull, tail);
          if (tail) {
            const uint32_t pos = tail_base + __popc(tb & lt);
            // sign carries the branch: negative <=> y > 0 (use 1-u).
            S.tail_w[pos] = y > 0.0 ? -__dadd_rn(1.0, -u) : u;
            S.tail_owner[pos] = static_cast<unsigned char>(t * 32 + lane);
            tmask |= 1u << t;
          }
          tail_base += __popc(tb);
          zq[t] = moro_central_plus(y, P.alpha);
        }
      }
      if (tail_base) {
        __syncwarp();
        for (uint32_t r = 0; r < tail_base; r += 32) {
          const uint32_t q = r + lane;
          if (q < tail_base) {
            const double ws = S.tail_w[q];
            const double x = moro_tail_poly(fabs(ws));
            S.zres[S.tail_owner[q]] = (ws < 0.0 ? x : -x) + P.alpha;
          }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kTile; ++t)
          if (tmask & (1u << t)) zq[t] = S.zres[t * 32 + lane];
      }
    }

#pragma unroll
    for (int t = 0; t < kTile; ++t) {
      const int d = k0 + t;
      if (d < m) {
        V = __dadd_rn(V, zq[t]);
        if (P.check_range && active) {
          const double X = fma(P.b, V, P.X0);
          if (X < -745.1332191019412) err |= ERR_SPOT_NONPOSITIVE;
          if (X > 709.782712893384) err |= ERR_SPOT_NONFINITE;
        }
        if (d < mrec) {
          const bool rec = active && (KIND == 0 ? V > c : V < c);
          const unsigned rb = __ballot_sync(kFull, rec);
          if (rb) {
            if (rec) {
              const uint32_t slot = (rq_tail + __popc(rb & lt)) & (kRecCap - 1);
              S.rq_v[slot] = V;
              S.rq_code[slot] = (static_cast<uint32_t>(d) << 5) | static_cast<uint32_t>(lane);
              if (!RNEG) c = V;
            }
            rq_tail += __popc(rb);
            if (rq_tail - rq_head >= 32) {
              __syncwarp();
              process_records<KIND, RNEG>(P, S, rq_head, 32, lane);
              rq_head += 32;
              __syncwarp();
              if (RNEG) c = rneg_threshold<KIND>(P, __longlong_as_double(static_cast<long long>(S.best[lane])));
            }
          }
        }
      }
    }
  }
  if (rq_tail != rq_head) {
    __syncwarp();
    process_records<KIND, RNEG>(P, S, rq_head, rq_tail - rq_head, lane);
  }
  __syncwarp();

  // Date m: max(intrinsic, Black-Scholes of the final interval), american.cpp:43-52.
  const double X = fma(P.b, V, P.X0);
  const double sm = exp(X);
  double cont;
  if (P.bs_v_zero) {
    const double fwd = sm * P.bs_fwd_growth;
    double iv = KIND == 0 ? fwd - P.strike : P.strike - fwd;
    cont = P.bs_disc * (iv > 0.0 ? iv : 0.0);
  } else {
    const double d1 = (X - P.log_strike + P.bs_mu_t) / P.bs_vsqrt;
    const double d2 = d1 - P.bs_vsqrt;
    const double price = KIND == 0 ? sm * cnd_dev(d1) - P.bs_kdisc * cnd_dev(d2)
                                   : P.bs_kdisc * cnd_dev(-d2) - sm * cnd_dev(-d1);
    cont = price > 0.0 ? price : 0.0;
  }
  double intr = KIND == 0 ? sm - P.strike : P.strike - sm;
  intr = intr > 0.0 ? intr : 0.0;
  const double cm = intr > cont ? intr : cont;
  const double term_m = cm * __ldg(P.dpow + m);
  const double best = __longlong_as_double(static_cast<long long>(S.best[lane]));
  if (active) {
    if (!(sm > 0.0)) err |= ERR_SPOT_NONPOSITIVE;
    if (!isfinite(sm)) err |= ERR_SPOT_NONFINITE;
    if (err) atomicOr(P.err, err);
    P.values[pi] = best > term_m ? best : term_m;
  }
}

// D1: uniforms (or Moro normals) of one dimension for `count` paths.
__global__ void uniforms_kernel(const uint32_t* __restrict__ perm_row, int64_t count, DimParam dp,
                                const double* __restrict__ sc, const double* __restrict__ nc,
                                int normals, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double u = halton(perm_row[i] + 1u, dp, sc, nc);
  out[i] = normals ? moro_full(u) : u;
}

// ---------------------------------------------------------------------------
// K1: Fisher-Yates reconstruction. Step i (n-1 >= i >= 1) of the reference
// swaps idx[i] with idx[j_i], j_i = below(i+1) from LCG draw n-1-i. With
// bucket(x) = {i : j_i = x} (j_0 := 0) sorted ascending, F(x) = the first
// element of bucket(x) that is > x and S(i) = the next element of i's bucket:
//   perm[i] = S(i) exists ? R(S(i)) : j_i,   R(y) = F(y) exists ? R(F(y)) : y.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ void lcg_jump(uint64_t delta, uint64_t& mult, uint64_t& plus) {
  uint64_t cur_mult = 6364136223846793005ULL, cur_plus = 1442695040888963407ULL;
  uint64_t acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  mult = acc_mult;
  plus = acc_plus;
}

__global__ void fy_draws_kernel(uint64_t seed, int64_t n, uint64_t stride_mult, uint64_t stride_plus,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t G = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g == 0) {
    keys[0] = 0;
    vals[0] = 0;
  }
  const int64_t draws = n - 1;
  if (g >= draws) return;
  uint64_t jm, jp;
  lcg_jump(static_cast<uint64_t>(g) + 1, jm, jp);
  uint64_t s = jm * seed + jp;  // state after draw g
  for (int64_t t = g; t < draws; t += G) {
    const int64_t i = n - 1 - t;
    keys[i] = static_cast<uint32_t>(__umul64hi(s, static_cast<uint64_t>(i) + 1));
    vals[i] = static_cast<uint32_t>(i);
    s = stride_mult * s + stride_plus;
  }
}

__global__ void fy_first_kernel(const uint32_t* __restrict__ sk, const uint32_t* __restrict__ sv, int64_t n,
                                uint32_t* __restrict__ F) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint32_t x = sk[q], i = sv[q];
  if (i > x) {
    const bool prev_above = q > 0 && sk[q - 1] == x && sv[q - 1] > x;
    if (!prev_above) F[x] = i;
  }
}

__global__ void fy_assign_kernel(const uint32_t* __restrict__ sk, const uint32_t* __restrict__ sv, int64_t n,
                                 const uint32_t* __restrict__ F, uint32_t* __restrict__ perm) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint32_t x = sk[q], i = sv[q];
  uint32_t out = x;
  if (q + 1 < n && sk[q + 1] == x) {
    uint32_t y = sv[q + 1];
    for (uint32_t f = F[y]; f != kNone; f = F[y]) y = f;
    out = y;
  }
  perm[i] = out;
}

// ---------------------------------------------------------------------------
// K3: pairwise tree. Nodes at depth L-1 (L = first depth whose nodes are all
// <= 64) are summed sequentially (split once if > 64); above that the tree is
// a perfect binary tree combined level by level in shared memory.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void node_range(int64_t len, int depth, int64_t node, int64_t& off, int64_t& size) {
  off = 0;
  size = len;
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

__device__ __forceinline__ void seq_sum(const double* __restrict__ v, int64_t off, int64_t size, double& s,
                                        double& s2) {
  s = 0.0;
  s2 = 0.0;
  for (int64_t i = 0; i < size; ++i) {
    const double x = v[off + i];
    s = __dadd_rn(s, x);
    s2 = __dadd_rn(s2, __dmul_rn(x, x));
  }
}

__global__ void pairwise_leaves_kernel(const double* __restrict__ v, int64_t len, int depth,
                                       double* __restrict__ out) {
  const int64_t node = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= (int64_t{1} << depth)) return;
  int64_t off, size;
  node_range(len, depth, node, off, size);
  double s, s2;
  if (size <= 64) {
    seq_sum(v, off, size, s, s2);
  } else {
    const int64_t half = size / 2;
    double a, a2, b, b2;
    seq_sum(v, off, half, a, a2);
    seq_sum(v, off + half, size - half, b, b2);
    s = __dadd_rn(a, b);
    s2 = __dadd_rn(a2, b2);
  }
  out[2 * node] = s;
  out[2 * node + 1] = s2;
}

// Reduces groups of `group` (power of two <= 1024) consecutive node pairs.
__global__ void pairwise_tree_kernel(const double* __restrict__ in, int64_t count, int group,
                                     double* __restrict__ out) {
  __shared__ double s[1024], s2[1024];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * group;
  for (int i = threadIdx.x; i < group; i += blockDim.x) {
    s[i] = in[2 * (base + i)];
    s2[i] = in[2 * (base + i) + 1];
  }
  __syncthreads();
  for (int w = group / 2; w >= 1; w /= 2) {
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
      s[i] = __dadd_rn(s[2 * i], s[2 * i + 1]);
      s2[i] = __dadd_rn(s2[2 * i], s2[2 * i + 1]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = s[0];
    out[2 * blockIdx.x + 1] = s2[0];
  }
  (void)count;
}

int leaf_depth(int64_t len) {
  int L = 0;
  while (((len + (int64_t{1} << L) - 1) >> L) > 64) ++L;
  return L;
}

}  // namespace

cudaError_t launch_price(const PriceParams& P, cudaStream_t s) {
  if (P.path_count <= 0) return cudaSuccess;
  const int64_t blocks = (P.path_count + kThreads - 1) / kThreads;
  if (P.kind == 0) {
    if (P.rate_negative) price_kernel<0, true><<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(P);
    else price_kernel<0, false><<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(P);
  } else {
    if (P.rate_negative) price_kernel<1, true><<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(P);
    else price_kernel<1, false><<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(P);
  }
  return cudaGetLastError();
}

cudaError_t launch_uniforms(const uint32_t* perm_row, int64_t count, DimParam dp, const double* sc,
                            const double* nc, int normals, double* out, cudaStream_t s) {
  const int64_t blocks = (count + 255) / 256;
  uniforms_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(perm_row, count, dp, sc, nc, normals, out);
  return cudaGetLastError();
}

namespace {
struct PermScratchLayout {
  size_t keys, vals, skeys, svals, F, temp, temp_bytes, total;
};
PermScratchLayout perm_layout(int64_t n) {
  auto align = [](size_t x) { return (x + 255) & ~size_t{255}; };
  PermScratchLayout L{};
  const size_t arr = align(static_cast<size_t>(n) * sizeof(uint32_t));
  size_t temp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int64_t>(n), 0, 32);
  L.keys = 0;
  L.vals = L.keys + arr;
  L.skeys = L.vals + arr;
  L.svals = L.skeys + arr;
  L.F = L.svals + arr;
  L.temp = L.F + arr;
  L.temp_bytes = align(temp_bytes);
  L.total = L.temp + L.temp_bytes;
  return L;
}
}  // namespace

size_t perm_scratch_bytes(int64_t n) { return perm_layout(n).total; }

cudaError_t launch_perm_build(uint64_t seed64, int64_t n, uint32_t* out, void* scratch, size_t scratch_bytes,
                              cudaStream_t s, int* launches) {
  const PermScratchLayout L = perm_layout(n);
  if (scratch_bytes < L.total) return cudaErrorInvalidValue;
  char* base = static_cast<char*>(scratch);
  auto* keys = reinterpret_cast<uint32_t*>(base + L.keys);
  auto* vals = reinterpret_cast<uint32_t*>(base + L.vals);
  auto* skeys = reinterpret_cast<uint32_t*>(base + L.skeys);
  auto* svals = reinterpret_cast<uint32_t*>(base + L.svals);
  auto* F = reinterpret_cast<uint32_t*>(base + L.F);
  if (n == 1) {
    return cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
  }
  int bits = 1;
  while (bits < 32 && (static_cast<uint64_t>(n - 1) >> bits) != 0) ++bits;
  const int threads = 256;
  const int64_t want = (n - 1 + 15) / 16;  // ~16 draws per thread
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((want + threads - 1) / threads, 148 * 64));
  uint64_t sm, sp;
  lcg_jump(static_cast<uint64_t>(blocks) * threads, sm, sp);
  fy_draws_kernel<<<static_cast<unsigned>(blocks), threads, 0, s>>>(seed64, n, sm, sp, keys, vals);
  size_t temp_bytes = L.temp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(base + L.temp, temp_bytes, keys, skeys, vals, svals,
                                                  static_cast<int64_t>(n), 0, bits, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(F, 0xff, static_cast<size_t>(n) * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int64_t eb = (n + threads - 1) / threads;
  fy_first_kernel<<<static_cast<unsigned>(eb), threads, 0, s>>>(skeys, svals, n, F);
  fy_assign_kernel<<<static_cast<unsigned>(eb), threads, 0, s>>>(skeys, svals, n, F, out);
  if (launches) *launches += 4 + 1;  // draws, sort (>=1), first, assign (+ memset)
  return cudaGetLastError();
}

size_t reduce_scratch_doubles(int64_t len) {
  const int L = leaf_depth(len);
  const int D = L > 0 ? L - 1 : 0;
  const int64_t nodes = int64_t{1} << D;
  return static_cast<size_t>(2 * nodes + 2 * ((nodes + 1023) / 1024) + 4);
}

cudaError_t launch_pairwise(const double* v, int64_t len, double* scratch, double* out2, cudaStream_t s,
                            int* launches) {
  const int L = leaf_depth(len);
  const int D = L > 0 ? L - 1 : 0;
  int64_t nodes = int64_t{1} << D;
  double* a = scratch;
  double* b = scratch + 2 * nodes;
  {
    const int64_t blocks = (nodes + 255) / 256;
    pairwise_leaves_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(v, len, D, nodes == 1 ? out2 : a);
    if (launches) ++*launches;
  }
  while (nodes > 1) {
    const int group = static_cast<int>(std::min<int64_t>(nodes, 1024));
    const int64_t blocks = nodes / group;
    double* dst = blocks == 1 ? out2 : b;
    pairwise_tree_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, nodes, group, dst);
    if (launches) ++*launches;
    nodes = blocks;
    std::swap(a, b);
  }
  return cudaGetLastError();
}

}  // namespace qmcg
