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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <mutex>
#include <vector>

#include "log_table.h"

namespace qmcg {
namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef QMCG_THREADS
#define QMCG_THREADS 256
#endif
constexpr int kThreads = QMCG_THREADS;  // paths per block (one per thread)
static_assert(kThreads % 32 == 0 && kThreads <= 256, "tail queue indices are 8-bit");
constexpr int kWarps = kThreads / 32;
#ifndef QMCG_MINB
#define QMCG_MINB 4
#endif
constexpr int kTile = kWarps;  // dates per tile = warps per block (one date row per warp)
#ifndef QMCG_REC_CAP
#define QMCG_REC_CAP 128
#endif
constexpr int kRecCap = QMCG_REC_CAP;  // per-warp ring of pending record evaluations (mostly drained at path end)
static_assert(kRecCap >= 64 && (kRecCap & (kRecCap - 1)) == 0, "record ring: power of two with room for one date");
constexpr uint32_t kNone = 0xffffffffu;
constexpr int kBins = 256;             // K1 binned scatter (== the bin kernel's block size)
constexpr int kCursorStride = 32;      // one 128-byte line per bin cursor (spreads the atomics over L2 slices)
#ifndef QMCG_K1_BIN_MIN
#define QMCG_K1_BIN_MIN (1 << 25)      // n from which K1 scatters through bins (measured: 2^24 faster direct)
#endif

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
  return a > 0x3fdae147ae147ae1ull;  // bits of 0.42
}

// Moro / Beasley-Springer coefficients in the constant bank so the DFMAs take
// them as c[][] operands (no per-use materialisation).
__constant__ double c_bs_a[4] = {2.50662823884, -18.61500062529, 41.39119773534, -25.44106049637};
__constant__ double c_bs_b[4] = {-8.47351093090, 23.08336743743, -21.06224101826, 3.13082909833};
__constant__ double c_moro_c[9] = {0.3374754822726147, 0.9761690190917186, 0.1607979714918209,
                                   0.0276438810333863, 0.0038405729373609, 0.0003951896511919,
                                   0.0000321767881768, 0.0000002888167364, 0.0000003960315187};

// 1/x from the MUFU estimate r0 with one cubic step: with e = 1 - x r0,
// 1/x = r0 (1 + e + e^2 + e^3 + ...), so r0 + r0 (e + e^2) leaves a relative
// error ~e^3 (< 2^-60 for the ~2^-20 estimate) plus the final rounding:
// 3 DFMAs instead of the 4 of two Newton steps.
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Beasley-Springer central region of moro_inv_cnd (analytic.cpp:82-94), plus
// the drift offset alpha folded into the final FMA.
// EXACT: the cubic-refined reciprocal (the exports and the European pricer, whose
// normals are compared with the reference to ~1e-15); otherwise one Newton step.
template <bool EXACT = false>
__device__ __forceinline__ double moro_central_plus(double y, double alpha) {
  const double r = y * y;
  const double A = fma(fma(fma(c_bs_a[3], r, c_bs_a[2]), r, c_bs_a[1]), r, c_bs_a[0]);
  const double B = fma(fma(fma(fma(c_bs_b[3], r, c_bs_b[2]), r, c_bs_b[1]), r, c_bs_b[0]), r, 1.0);
  if (EXACT) return fma(y * A, rcp_nr(B), alpha);
  // pricing: 1/B from the MUFU estimate with one Newton step (relative error ~e^2,
  // e the estimate's error): the normal keeps ~13 significant digits (measured
  // 2.7e-13 relative on exported paths), one DFMA per point fewer than the cubic
  // step (C3 18.11 -> 17.81 ms); the uniform, and so the central/tail branch,
  // stays bit-exact
  double r0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(B));
  return fma(y * A, fma(r0, fma(-B, r0, 1.0), r0), alpha);
}

__constant__ double2 c_log_table[128];
__constant__ double c_tail_y = 0.42;  // Moro branch point |u - 1/2| > 0.42 (analytic.cpp:87)
__constant__ double c_log_consts[2] = {0.0 /* unused */, 0x1.62e42fefa39efp-1 /* ln 2 */};
// dev_log's polynomial in the constant bank: the DFMAs take them as c[][] operands (as 64-bit
// immediates each cost a UMOV pair per use, ~1 warp instruction per warp-date in the tail)
__constant__ double c_log_poly[4] = {0x1.999999999999ap-3, -0x1.0001p-2, 0x1.5555555555555p-2, -0x1.ffffffffap-2};

// Shared-memory accessors on 32-bit shared-window addresses (keeps the
// compiler from rebuilding generic->shared windows inside the hot loops).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double2 lds_v2f64(uint32_t a) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_v2f64(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

// Natural log for positive normal x: x = 2^e * m, m = c_i (1 + f) with the
// 128-entry table {1/c_i, -log(1/c_i)} (log_table.h) in shared memory at
// `tab`, |f| <= 2^-8, log1p(f) by a degree-5 polynomial: the Taylor series
// with its f^6/6 term folded into the f^4 and f^2 coefficients by Chebyshev
// economization on [-2^-8, 2^-8] (f^4: -1/4 - 2^-18, f^2: -1/2 + 3*2^-37),
// truncation error < 4e-17 absolute (Taylor degree 5 would leave 6e-16).
// ~10 FP64 operations, error about 1 ulp of the result (CUDA's log() costs ~3x
// the issue slots); only used on the Moro tail where |result| > 0.9.
__device__ __forceinline__ double dev_log(double x, uint32_t tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const double2 t = lds_v2f64(tab + (static_cast<uint32_t>(hi >> 9) & 0x7f0u));
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double f = fma(m, t.x, -1.0);
  double q = fma(f, c_log_poly[0], c_log_poly[1]);
  q = fma(f, q, c_log_poly[2]);
  q = fma(f, q, c_log_poly[3]);
  const double p = fma(f * f, q, f);
  const double de = static_cast<double>(e);  // exact: one I2F.F64 (the 2^52 magic took 3 issue slots)
  return fma(de, c_log_consts[1], t.y + p);
}

// -log(x) with the same reduction (the negation folded into the final FMA).
__device__ __forceinline__ double dev_neglog(double x, uint32_t tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const double2 t = lds_v2f64(tab + (static_cast<uint32_t>(hi >> 9) & 0x7f0u));
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double f = fma(m, t.x, -1.0);
  double q = fma(f, c_log_poly[0], c_log_poly[1]);
  q = fma(f, q, c_log_poly[2]);
  q = fma(f, q, c_log_poly[3]);
  const double p = fma(f * f, q, f);
  const double de = static_cast<double>(e);  // exact: one I2F.F64 (the 2^52 magic took 3 issue slots)
  return fma(de, -c_log_consts[1], -(t.y + p));
}

// Moro log-log tail polynomial (analytic.cpp:95-99) for w = u or 1-u.
__device__ __forceinline__ double moro_tail_poly(double w, uint32_t tab) {
  const double z = dev_log(dev_neglog(w, tab), tab);
  double x = c_moro_c[8];
#pragma unroll
  for (int i = 7; i >= 0; --i) x = fma(x, z, c_moro_c[i]);
  return x;
}

// FP32 variant (QMCG_FLAG_FP32): Moro in single precision on the exact FP64
// uniform (the branch partition is still decided in FP64).
__device__ __forceinline__ float moro_central_f32(float y, float alpha) {
  const float r = y * y;
  const float A = fmaf(fmaf(fmaf(-25.44106049637f, r, 41.39119773534f), r, -18.61500062529f), r, 2.50662823884f);
  const float B = fmaf(fmaf(fmaf(fmaf(3.13082909833f, r, -21.06224101826f), r, 23.08336743743f), r, -8.47351093090f),
                       r, 1.0f);
  // the MUFU reciprocal (rel. error ~2^-23, like the rest of the single-precision Moro) instead of
  // the IEEE-rounded __frcp_rn, which expands to a Newton sequence: FP32 call 10.43 -> 9.25 ms
  float rb;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(B));
  return fmaf(y * A, rb, alpha);
}

__device__ __forceinline__ float moro_tail_poly_f32(float w) {
  const float z = __logf(-__logf(w));
  float x = 0.0000003960315187f;
  x = fmaf(x, z, 0.0000002888167364f);
  x = fmaf(x, z, 0.0000321767881768f);
  x = fmaf(x, z, 0.0003951896511919f);
  x = fmaf(x, z, 0.0038405729373609f);
  x = fmaf(x, z, 0.0276438810333863f);
  x = fmaf(x, z, 0.1607979714918209f);
  x = fmaf(x, z, 0.9761690190917186f);
  x = fmaf(x, z, 0.3374754822726147f);
  return x;
}

__device__ __forceinline__ double moro_tail_poly(double w) {
  const double z = log(-log(w));
  double x = c_moro_c[8];
#pragma unroll
  for (int i = 7; i >= 0; --i) x = fma(x, z, c_moro_c[i]);
  return x;
}

__device__ __forceinline__ double moro_full(double u) {
  const double y = __dadd_rn(u, -0.5);
  if (!moro_is_tail(y)) return moro_central_plus<true>(y, 0.0);
  const double x = moro_tail_poly(y > 0.0 ? __dadd_rn(1.0, -u) : u);
  return y > 0.0 ? x : -x;
}

// exp for the batch walk (candidates, final interval): k = rint(x / ln 2) by the 1.5 * 2^52 trick,
// r = x - k ln 2 (two-part ln 2), e^r by Horner on the Taylor series to r^13 (truncation < 4e-18 for
// |r| <= ln2 / 2), scaled by 2^k in the exponent field; ~1 ulp like CUDA's exp, with the
// coefficients in the constant bank instead of per-call immediates (CUDA's exp rebuilds ~24 of
// them with UMOVs each call inside the per-strike loop). |x| beyond the normal range: CUDA's exp.
__constant__ double c_exp_poly[12] = {1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
                                      2.755731922398589e-07,  2.7557319223985893e-06, 2.48015873015873e-05,
                                      1.984126984126984e-04,  1.388888888888889e-03,  8.333333333333333e-03,
                                      4.1666666666666664e-02, 1.6666666666666666e-01, 0.5};
__device__ __forceinline__ double dev_exp(double x) {
  const double t = fma(x, 0x1.71547652b82fep0, 0x1.8p52);
  const double kd = t - 0x1.8p52;
  const int k = __double2loint(t);
  double r = fma(kd, -0x1.62e42fefa39efp-1, x);
  r = fma(kd, -0x1.abc9e3b39803fp-56, r);
  double p = c_exp_poly[0];
#pragma unroll
  for (int i = 1; i < 12; ++i) p = fma(p, r, c_exp_poly[i]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  if (k < -1020 || k > 1020) return exp(x);
  return __hiloint2double(__double2hiint(p) + (k << 20), __double2loint(p));
}

// Hart CND (analytic.cpp:33-72) for the batch's per-strike final interval,
// given e = exp(-d^2 / 2) computed by the caller, branch free: the rational
// form for every |d|. The reference switches to a continued fraction for
// |d| >= 7.07 and returns 0/1 beyond 37; there the tail is below 8e-13 and
// the rational form matches the true tail to 1.1e-8 relative (2e-21
// absolute; checked against scipy's ndtr up to |d| = 12, beyond which e
// makes the tail negligible and exp underflows to 0 from |d| ~ 38.6), so
// 1 - tail rounds identically and a tail product changes a path value by
// < 1e-18 -- far inside the batch's 1e-12 parity bar -- while the warp no
// longer runs two divergent branches per strike. The division uses the
// cubic-refined reciprocal.
__device__ __forceinline__ double cnd_tail_form(double d, double e) {
  const double x = fabs(d);
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
  const double tail = e * num * rcp_nr(den);
  return d > 0.0 ? 1.0 - tail : tail;
}

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

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ double clamp_endpoints(double v) {  // quasi_rng.cpp:80-81
  if (v < 1e-12) v = 1e-12;
  if (v > 1.0 - 1e-12) v = 1.0 - 1e-12;
  return v;
}

// ---- shared-window addresses (the bulk copies and mbarriers use them) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Shared memory of one 256-path block (byte offsets from the dynamic base):
//   zt[2][kTile][256]   f64   the tile's uniforms u (2-D TMA copy of the uniform table), turned
//                             in place into z_k + alpha per (date, path) and walked; double-buffered
//   logtab[128]         f64x2 log reduction table
//   bar[2]              mbarriers of the two tile buffers
//   per warp: rq_v[128] f64 | best[32] u64 | rq_code[128] u32 | tail_idx[256 + 32] u8
// A Moro-tail point keeps its uniform u in its slot until the row's tail queue (indices
// only) is evaluated and overwrites it with z. FP32 variant: z is an f32 in the slot's low half.
constexpr uint32_t kTailCap = kThreads;  // a whole date row can be queued: no mid-row flush
constexpr uint32_t kZtOff = 0;
constexpr uint32_t kZtBuf = kTile * kThreads * 8;
constexpr int kZtBuffers = 2;
constexpr uint32_t kLogOff = kZtOff + kZtBuffers * kZtBuf;
constexpr uint32_t kBarOff = kLogOff + 128 * 16;
constexpr uint32_t kWarpOff = kBarOff + 128;
static_assert(2 * kTile * 8 <= 128, "row mbarriers bar[2][kTile]");
constexpr uint32_t kWRqV = 0;
constexpr uint32_t kWBest = kWRqV + kRecCap * 8;
constexpr uint32_t kWRqCode = kWBest + 32 * 8;
constexpr uint32_t kWTailIdx = kWRqCode + kRecCap * 4;
constexpr uint32_t kWarpBytes = kWTailIdx + kTailCap + 32;  // + 32 dummy slots for non-tail lanes
constexpr uint32_t kSmemBytes = kWarpOff + kWarps * kWarpBytes;

// Exact evaluation of up to 32 queued records: term = disc^date * intrinsic(exp(X0 + b V)),
// folded into the owner lane's running maximum (doubles >= 0 order like their bits).
template <int KIND>
__device__ __forceinline__ void eval_records(double b, double X0, double strike, const double* __restrict__ dpow,
                                             uint32_t ws, uint32_t head, uint32_t count, int lane) {
  if (static_cast<uint32_t>(lane) < count) {
    const uint32_t slot = (head + lane) & (kRecCap - 1);
    const double v = lds_f64(ws + kWRqV + slot * 8);
    const uint32_t code = lds_u32(ws + kWRqCode + slot * 4);
    const int d = static_cast<int>(code >> 5);
    const uint32_t owner = code & 31u;
    const double s = exp(fma(b, v, X0));
    double intr = KIND == 0 ? s - strike : strike - s;
    intr = intr > 0.0 ? intr : 0.0;
    const double term = intr * __ldg(dpow + d + 1);
    asm volatile("atom.shared.max.u64 _, [%0], %1;" ::"r"(ws + kWBest + owner * 8),
                 "l"(static_cast<unsigned long long>(__double_as_longlong(term)))
                 : "memory");
  }
}

// Out-of-line copy for the rare call sites (ring overflow inside a tile, end of
// path). Scalars only: a reference to the kernel parameters would force a
// per-thread local copy of them.
template <int KIND>
__device__ __noinline__ void eval_records_call(double b, double X0, double strike, const double* dpow, uint32_t ws,
                                               uint32_t head, uint32_t count, int lane) {
  eval_records<KIND>(b, X0, strike, dpow, ws, head, count, lane);
}

template <int KIND, bool RNEG>
__device__ __forceinline__ void process_records_inline(const PriceParams& P, uint32_t ws, uint32_t head,
                                                       uint32_t count, int lane) {
  eval_records<KIND>(P.b, P.X0, P.strike, P.dpow, ws, head, count, lane);
}

template <int KIND, bool RNEG>
__device__ __forceinline__ void process_records(const PriceParams& P, uint32_t ws, uint32_t head, uint32_t count,
                                                int lane) {
  eval_records_call<KIND>(P.b, P.X0, P.strike, P.dpow, ws, head, count, lane);
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

// One 2-D TMA copy of a whole tile (kTile dates x 256 paths of the [date][path]
// uniform table, f64) into tile buffer b, completing on the buffer's mbarrier bar[b][0].
// Out-of-range rows/columns (last tile, last block) arrive zero-filled.
__device__ __forceinline__ void issue_tile_tma(const CUtensorMap* tmap, uint32_t sbase, int b, int col, int row) {
  const uint32_t bar = sbase + kBarOff + b * kTile * 8;
  const uint32_t dst = sbase + kZtOff + b * kZtBuf;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kZtBuf) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(col), "r"(row), "r"(bar)
      : "memory");
}

// mbarriers bar[2][kTile] (one per buffer and row), arrival count 1.
__device__ __forceinline__ void init_row_barriers(uint32_t sbase) {
  if (threadIdx.x < 2 * kTile) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbase + kBarOff + threadIdx.x * 8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// z-tile slot access (8-byte slots that first hold the uniform): FP64, or for the FP32 variant an
// f32 in the slot's low half.
template <bool F32> struct ZSlot;
template <> struct ZSlot<false> {
  using T = double;
  static constexpr uint32_t kSize = 8;
  static __device__ __forceinline__ T load(uint32_t a) { return lds_f64(a); }
  static __device__ __forceinline__ void store(uint32_t a, T v) { sts_f64(a, v); }
};
template <> struct ZSlot<true> {
  using T = float;
  static constexpr uint32_t kSize = 8;
  static __device__ __forceinline__ T load(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
  }
  static __device__ __forceinline__ void store(uint32_t a, T v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
  }
};

template <bool F32>
__device__ __forceinline__ typename ZSlot<F32>::T central_z(double y, double alpha) {
  if (F32) return moro_central_f32(static_cast<float>(y), static_cast<float>(alpha));
  return moro_central_plus(y, alpha);
}

// One point pair of a date row, in place: the slots hold u; a central point's slot gets
// z + alpha, a tail point (|u - 1/2| > 0.42, the reference's branch on the bit-exact uniform)
// keeps u and queues its index in the warp's tail queue at ntail + rank. The second chunk's
// rank adds the first chunk's count in one 3-input add, and ntail advances by both counts.
template <bool F32>
__device__ __forceinline__ void park_pair(uint32_t sa, uint32_t sb, uint32_t qbase, uint32_t idx_a,
                                          typename ZSlot<F32>::T za, double ya, typename ZSlot<F32>::T zb, double yb,
                                          unsigned lt, uint32_t& ntail) {
  if constexpr (F32) {
    asm volatile(
        "{\n .reg .pred pa, pb;\n .reg .f64 ay;\n .reg .b32 ba, bb, ca, ra, rb, q, a;\n"
        " abs.f64 ay, %3;\n setp.gt.f64 pa, ay, %9;\n"
        " abs.f64 ay, %6;\n setp.gt.f64 pb, ay, %9;\n"
        " vote.sync.ballot.b32 ba, pa, 0xffffffff;\n"
        " vote.sync.ballot.b32 bb, pb, 0xffffffff;\n"
        " @!pa st.shared.f32 [%1], %2;\n @!pb st.shared.f32 [%4], %5;\n"
        " add.u32 q, %7, %0;\n"
        " and.b32 ra, ba, %8;\n popc.b32 ra, ra;\n popc.b32 ca, ba;\n"
        " and.b32 rb, bb, %8;\n popc.b32 rb, rb;\n"
        " add.u32 a, q, ra;\n @pa st.shared.u8 [a], %10;\n"
        " add.u32 a, q, ca;\n add.u32 a, a, rb;\n @pb st.shared.u8 [a], %11;\n"
        " popc.b32 bb, bb;\n add.u32 %0, %0, ca;\n add.u32 %0, %0, bb;\n}"
        : "+r"(ntail)
        : "r"(sa), "f"(za), "d"(ya), "r"(sb), "f"(zb), "d"(yb), "r"(qbase), "r"(lt), "d"(c_tail_y), "r"(idx_a),
          "r"(idx_a + 32)
        : "memory");
  } else {
    asm volatile(
        "{\n .reg .pred pa, pb;\n .reg .f64 ay;\n .reg .b32 ba, bb, ca, ra, rb, q, a;\n"
        " abs.f64 ay, %3;\n setp.gt.f64 pa, ay, %9;\n"
        " abs.f64 ay, %6;\n setp.gt.f64 pb, ay, %9;\n"
        " vote.sync.ballot.b32 ba, pa, 0xffffffff;\n"
        " vote.sync.ballot.b32 bb, pb, 0xffffffff;\n"
        " @!pa st.shared.f64 [%1], %2;\n @!pb st.shared.f64 [%4], %5;\n"
        " add.u32 q, %7, %0;\n"
        " and.b32 ra, ba, %8;\n popc.b32 ra, ra;\n popc.b32 ca, ba;\n"
        " and.b32 rb, bb, %8;\n popc.b32 rb, rb;\n"
        " add.u32 a, q, ra;\n @pa st.shared.u8 [a], %10;\n"
        " add.u32 a, q, ca;\n add.u32 a, a, rb;\n @pb st.shared.u8 [a], %11;\n"
        " popc.b32 bb, bb;\n add.u32 %0, %0, ca;\n add.u32 %0, %0, bb;\n}"
        : "+r"(ntail)
        : "r"(sa), "d"(za), "d"(ya), "r"(sb), "d"(zb), "d"(yb), "r"(qbase), "r"(lt), "d"(c_tail_y), "r"(idx_a),
          "r"(idx_a + 32)
        : "memory");
  }
}

// The same for one point (a row's odd last chunk).
template <bool F32>
__device__ __forceinline__ void park_one(uint32_t sa, uint32_t qbase, uint32_t idx, typename ZSlot<F32>::T za,
                                         double ya, unsigned lt, uint32_t& ntail) {
  const bool tail = moro_is_tail(ya);
  const unsigned b = __ballot_sync(kFull, tail);
  if (tail) sts_u8(qbase + ntail + __popc(b & lt), idx);
  else ZSlot<F32>::store(sa, za);
  ntail += __popc(b);
}

// One queued Moro-tail point: u (in its slot) -> w = u or 1 - u, z = +-P8(log(-log w)) + alpha.
// A queued point has u < 0.08 or u > 0.92, so y = u - 1/2 > 0 iff the high word of u is at
// least that of 0.5 (integer test, no FP64 compare); -x for y < 0 by flipping the sign bit.
__device__ __forceinline__ double tail_z(double u, uint32_t logtab, double alpha) {
  const bool up = __double2hiint(u) >= 0x3fe00000;
  const double x = moro_tail_poly(up ? __dadd_rn(1.0, -u) : u, logtab);
  const double sx =
      __hiloint2double(__double2hiint(x) ^ (up ? 0 : static_cast<int>(0x80000000u)), __double2loint(x));
  return __dadd_rn(sx, alpha);
}

// Evaluate the queued Moro-tail points of one date row. Two rounds of 32 are
// evaluated together (each lane carries two independent points), so a row's
// typical 33-64 tail points cost one dependency chain instead of two; lanes
// past the queue end compute a duplicate of entry 0 and do not store it.
template <bool F32>
__device__ __forceinline__ void flush_tail(uint32_t ws, uint32_t zrow, uint32_t ntail, uint32_t logtab, double alpha,
                                           int lane) {
  using Z = ZSlot<F32>;
  __syncwarp();
#ifdef QMCG_PROBE_FULLROUNDS  // timing probe only (wrong results): skip the partial last round
  ntail &= ~31u;
#endif
  const uint32_t qbase = ws + kWTailIdx;
  if (F32) {
    for (uint32_t r = 0; r < ntail; r += 32) {
      const uint32_t q = r + lane;
      if (q < ntail) {
        const uint32_t slot = zrow + lds_u8(qbase + q) * Z::kSize;
        const double u = lds_f64(slot);
        const bool up = __double2hiint(u) >= 0x3fe00000;
        const float x = moro_tail_poly_f32(static_cast<float>(up ? __dadd_rn(1.0, -u) : u));
        Z::store(slot, (up ? x : -x) + static_cast<float>(alpha));
      }
    }
  } else {
    for (uint32_t r = 0; r < ntail; r += 64) {
      const uint32_t qa = r + lane, qb = r + 32 + lane;
      const bool va = qa < ntail, vb = qb < ntail;
      const uint32_t sa = zrow + lds_u8(qbase + (va ? qa : 0u)) * 8;
      if (r + 32 < ntail) {  // warp-uniform: a second round exists
        const uint32_t sb = zrow + lds_u8(qbase + (vb ? qb : 0u)) * 8;
        const double za = tail_z(lds_f64(sa), logtab, alpha);
        const double zb = tail_z(lds_f64(sb), logtab, alpha);
        __syncwarp();  // every lane has read its u before any slot is overwritten
        if (va) sts_f64(sa, za);
        if (vb) sts_f64(sb, zb);
      } else {
        const double za = tail_z(lds_f64(sa), logtab, alpha);
        __syncwarp();
        if (va) sts_f64(sa, za);
      }
    }
  }
  __syncwarp();
}

// One date row of the tile, in place: warp w turns row w of uniforms (already in shared
// memory: the TMA'd uniform table, built bit-exactly by uniforms_kernel from the K1 tables) into
// z + alpha. Two independent 32-path chunks in flight per iteration.
template <bool F32>
__device__ __forceinline__ void generate_row(uint32_t ws, uint32_t zrow, uint32_t logtab, int nchunks, int lane,
                                             unsigned lt, double alpha) {
  const uint32_t zl = zrow + lane * 8;
  const uint32_t qbase = ws + kWTailIdx;
  uint32_t ntail = 0;
  int ch = 0;
#pragma unroll 1
  for (; ch + 1 < nchunks; ch += 2) {
    const uint32_t sa = zl + ch * 256, sb = sa + 256;
    const double ua = lds_f64(sa), ub = lds_f64(sb);
    const double ya = __dadd_rn(ua, -0.5), yb = __dadd_rn(ub, -0.5);
    park_pair<F32>(sa, sb, qbase, ch * 32 + lane, central_z<F32>(ya, alpha), ya, central_z<F32>(yb, alpha), yb, lt,
                   ntail);
  }
  if (ch < nchunks) {
    const uint32_t sa = zl + ch * 256;
    const double ya = __dadd_rn(lds_f64(sa), -0.5);
    park_one<F32>(sa, qbase, ch * 32 + lane, central_z<F32>(ya, alpha), ya, lt, ntail);
  }
#ifndef QMCG_PROBE_NOTAIL  // timing probe only (wrong results): skip the Moro tail
  if (ntail) flush_tail<F32>(ws, zrow, ntail, logtab, alpha, lane);
#endif
}

// Dominance of the lane's pending record j by a new record k (then j can never
// be the maximum and needs no exp()):
//   calls: acc = V_j + slope (k - j) in V units; k dominates j iff V_k >= acc
//          (S_k disc^(k-j) >= S_j);
//   puts:  acc = delta = r dt (k - j); k dominates j iff
//          w (1 - e^-(delta + Delta)) >= 1 - e^-delta, w = S_j / K, Delta = b (V_j - V_k);
//          sufficient (exact-safe lower/upper bounds, no exp): with u = ln w,
//          (1 + u) s (1 - s/2) >= delta, s = delta + Delta, 1 + u > 0, s < 2.
// x0mk = 1 + X0 - ln K (puts only).
template <int KIND, typename T>
__device__ __forceinline__ bool record_dominates(T V, T c, T acc, T b, T x0mk) {
  if (KIND == 0) return V >= acc;
  // FP32 variant: the bound is taken with a relative margin far above its rounding
  const T margin = sizeof(T) == 8 ? T(1e-12) : T(1e-4);
  const T u1 = fma(b, c, x0mk);
  const T s = fma(b, c - V, acc);
  return u1 > T(0) && s < T(2) && u1 * s * fma(T(-0.5), s, T(1)) >= acc * (T(1) + margin);
}

template <int KIND, bool RNEG>
__device__ __forceinline__ void push_record(uint32_t ws, const PriceParams& P, bool push, double v, int d, int lane,
                                            unsigned lt, uint32_t& rq_head, uint32_t& rq_tail) {
  if (__any_sync(kFull, push)) {
    const unsigned pb = __ballot_sync(kFull, push);
    if (push) {
      const uint32_t slot = (rq_tail + __popc(pb & lt)) & (kRecCap - 1);
      sts_f64(ws + kWRqV + slot * 8, v);
      sts_u32(ws + kWRqCode + slot * 4, (static_cast<uint32_t>(d) << 5) | static_cast<uint32_t>(lane));
    }
    rq_tail += __popc(pb);
    if (rq_tail - rq_head > kRecCap - 32) {  // rare: the ring must keep room for one more date
      __syncwarp();
      process_records<KIND, RNEG>(P, ws, rq_head, 32, lane);
      rq_head += 32;
      __syncwarp();
    }
  }
}

// One walk date of the FP64 fast path (predicated, no branches): advances the
// record state (c = V of the last record, cd = dominance accumulator of the
// pending record, pl = its tile-relative date) and returns 1 when the pending
// record must be queued for exact evaluation (pv, pdl = its V and date).
//   calls: record = V > c; push = record and V < cd (the new record does not
//          dominate the pending one; cd = -inf until the first record);
//   puts:  record = V < c; push = record, a pending record exists
//          (pl + k0 >= 0) and the accumulator bound of record_dominates<1> fails
//          (V and cd already advanced by the caller).
template <int KIND>
//   (puts: negk0 = -k0; bs = b / M and x0mks = x0mk / M with M = 1 + 4504 * 2^-52, so u1 / M comes
//   out of one FMA and the margin of record_dominates<1> needs no multiply by cd)
__device__ __forceinline__ uint32_t walk_date(double V, double& c, double& cd, int& pl, int t, int negk0, double& pv,
                                              int& pdl, double b, double bs, double x0mks) {
  uint32_t pu32;
  if constexpr (KIND == 0) {
    asm("{\n .reg .pred r, pu;\n"
        " setp.gt.f64 r, %7, %0;\n setp.lt.and.f64 pu, %7, %1, r;\n"
        " mov.b64 %3, %0;\n mov.b32 %4, %2;\n"
        " selp.f64 %0, %7, %0, r;\n selp.f64 %1, %7, %1, r;\n selp.b32 %2, %6, %2, r;\n"
        " selp.u32 %5, 1, 0, pu;\n}"
        : "+d"(c), "+d"(cd), "+r"(pl), "=d"(pv), "=r"(pdl), "=r"(pu32)
        : "r"(t), "d"(V));
  } else {
    asm("{\n .reg .pred r, pe, a, b, e, dm, pu;\n .reg .f64 u1, dv, s, t, pr;\n"
        " setp.lt.f64 r, %7, %0;\n setp.ge.s32 pe, %2, %8;\n"
        " fma.rn.f64 u1, %10, %0, %11;\n sub.rn.f64 dv, %0, %7;\n fma.rn.f64 s, %9, dv, %1;\n"
        " fma.rn.f64 t, 0dBFE0000000000000, s, 0d3FF0000000000000;\n mul.rn.f64 pr, u1, s;\n"
        " mul.rn.f64 pr, pr, t;\n"
        " setp.gt.f64 a, u1, 0d0000000000000000;\n setp.lt.and.f64 b, s, 0d4000000000000000, a;\n"
        " setp.ge.and.f64 dm, pr, %1, b;\n and.pred pu, r, pe;\n not.pred e, dm;\n and.pred pu, pu, e;\n"
        " mov.b64 %3, %0;\n mov.b32 %4, %2;\n"
        " selp.f64 %0, %7, %0, r;\n selp.f64 %1, 0d0000000000000000, %1, r;\n selp.b32 %2, %6, %2, r;\n"
        " selp.u32 %5, 1, 0, pu;\n}"
        : "+d"(c), "+d"(cd), "+r"(pl), "=d"(pv), "=r"(pdl), "=r"(pu32)
        : "r"(t), "d"(V), "r"(negk0), "d"(b), "d"(bs), "d"(x0mks));
  }
  return pu32;
}

#ifndef QMCG_PUSH_GROUP
#define QMCG_PUSH_GROUP 4
#endif
// dates per push check in the walk: one warp vote + (rarely taken) branch per
// group instead of per date, so the dates of a group issue back to back
constexpr int kPushGroup = QMCG_PUSH_GROUP;
static_assert(kTile % kPushGroup == 0, "push groups tile the dates");

// One block = 256 consecutive paths; thread i walks path i. Per tile of
// kTile dates: (1) the tile's uniforms (the [date][path] uniform table: bit-exact
// scrambled-Halton values built once per table by uniforms_kernel) arrive by one 2-D TMA
// copy, double-buffered; (2) warp w turns date row w of the tile into normals in place;
// (3) every thread walks its path through the tile: V_k = sum (z_j + alpha)
// is the log-price in units of b, X_k = X0 + b V_k. A date k can only set the
// foresight maximum max_k disc^k I_k if I_k exceeds every earlier intrinsic
// (disc <= 1), i.e. V_k sets a new running extreme ("record"). Each record
// replaces the lane's pending record; the pending record j is dropped when
// the new record k dominates it (S_k disc^(k-j) >= S_j, i.e. key_k >= key_j
// with key = V - slope*date, slope = r*dt/b, calls), otherwise j is queued
// for exact evaluation (exp + discount) in warp-wide batches of 32.
// SLOW = volatility 0 or range checks. One block barrier per tile: after it every warp has
// generated tile k and walked tile k - 1, so the buffer of tile k - 1 takes tile k + 1.
template <int KIND, bool RNEG, bool SLOW, bool F32>
__global__ void __launch_bounds__(kThreads, QMCG_MINB)
    price_kernel(const PriceParams P, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t sbase = smem_u32(smem_raw);
  asm volatile("mov.b32 %0, %0;" : "+r"(sbase));  // computed once (no shared-window rebuild in the loops)
  int warp = threadIdx.x >> 5;
  int lane = threadIdx.x & 31;
  // held in registers: rebuilding them from %tid inside the loops cost ~3 instructions per warp-date
  asm volatile("mov.b32 %0, %0;" : "+r"(warp));
  asm volatile("mov.b32 %0, %0;" : "+r"(lane));
  const uint32_t ws = sbase + kWarpOff + warp * kWarpBytes;
  const uint32_t logtab = sbase + kLogOff;
  const unsigned lt = lanemask_lt();
  const int64_t block_first = static_cast<int64_t>(blockIdx.x) * kThreads;
  const int64_t pi = block_first + threadIdx.x;
  const bool active = pi < P.path_count;
  const int m = P.m;
  const int mrec = m - 1;
  const bool det = SLOW && P.deterministic != 0;
  const bool check = SLOW && P.check_range != 0;
  const int dbeg = P.d_begin, dend = P.d_end;  // date window of this launch
  const int ntiles = (dend - dbeg + kTile - 1) / kTile;
  const int64_t block_paths = min(static_cast<int64_t>(kThreads), P.path_count - block_first);
  const int nchunks = static_cast<int>((block_paths + 31) / 32);
  // columns of this block in the table
  const int64_t col0 = P.path_begin - P.col_begin + block_first;
  using Z = ZSlot<F32>;
  using T = typename Z::T;
  T slope = static_cast<T>(P.dom_slope);
  if constexpr (!F32) asm volatile("mov.b64 %0, %0;" : "+d"(slope));  // keep it in a register (no per-date reload)
  const T bT = static_cast<T>(P.b), x0mkT = static_cast<T>(P.x0mk);
  // puts (FP64 walk): record_dominates<1>'s 1e-12 margin folded into u1 = (b c + x0mk) / M
  constexpr double kMargin = 1.0 + 0x1198p-52;
  const double bsd = P.b / kMargin, x0mks = P.x0mk / kMargin;

  init_row_barriers(sbase);
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(ws + kWBest + lane * 8),
               "l"(static_cast<unsigned long long>(__double_as_longlong(P.best0)))
               : "memory");
  T V = T(0);
  T c = static_cast<T>(P.c0);
  // dominance threshold of the pending record (see the walk); for calls -inf
  // while no record is pending, so that no new record is ever pushed against it
  T cd = KIND == 0 ? T(-INFINITY) : T(0);
  int pend_d = -1;  // date of the pending (not yet evaluated) record, -1 = none
  if (P.stream_load && active) {  // carry-in from the previous date window
    const int64_t i = pi;
    V = static_cast<T>(P.st_V[i]);
    c = static_cast<T>(P.st_c[i]);
    cd = static_cast<T>(P.st_cd[i]);
    pend_d = P.st_pend[i];
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(ws + kWBest + lane * 8), "d"(P.st_best[i]) : "memory");
  }
  if (threadIdx.x < 128) sts_v2f64(logtab + threadIdx.x * 16, c_log_table[threadIdx.x]);
  __syncthreads();
  if (threadIdx.x == 0 && !det) {
    issue_tile_tma(&tmap, sbase, 0, static_cast<int>(col0), dbeg - P.perm_row0);
    if (ntiles > 1) issue_tile_tma(&tmap, sbase, 1, static_cast<int>(col0), dbeg + kTile - P.perm_row0);
  }

  uint32_t rq_head = 0, rq_tail = 0;
  uint32_t err = 0;

  for (int k = 0; k < ntiles; ++k) {
    const int k0 = dbeg + k * kTile;
    const int b = k & 1;
    const uint32_t ztile = sbase + kZtOff + b * kZtBuf;
    const uint32_t zcol = ztile + threadIdx.x * Z::kSize;
    if (!det) {
      if (k0 + warp < dend) {
        mbar_wait_u32(sbase + kBarOff + b * kTile * 8, static_cast<uint32_t>((k >> 1) & 1));
#ifndef QMCG_PROBE_NOGEN  // timing probe only (wrong results): walk the tile as loaded
        generate_row<F32>(ws, ztile + warp * kThreads * Z::kSize, logtab, nchunks, lane, lt, P.alpha);
#endif
      }
      __syncthreads();  // tile k generated; every warp has walked tile k - 1: its buffer takes tile k + 1
      if (threadIdx.x == 0 && k >= 1 && k + 1 < ntiles)
        issue_tile_tma(&tmap, sbase, b ^ 1, static_cast<int>(col0), k0 + kTile - P.perm_row0);
    }
    // ---- walk ----
    // c = V of the last record (= the pending record when pend_d >= 0);
    // cd = the dominance accumulator of the pending record (record_dominates).
#ifdef QMCG_PROBE_NOWALK  // timing probe only (wrong results): V only, no record logic
    if (!SLOW && !RNEG && k0 + kTile <= mrec) {
#pragma unroll
      for (int t = 0; t < kTile; ++t) V = add_rn(V, Z::load(zcol + t * kThreads * Z::kSize));
    } else
#endif
    if (!SLOW && !RNEG && k0 + kTile <= mrec) {
      // pending date kept tile-relative (the select takes t as an immediate);
      // calls need no "pending exists" test: cd = -inf until the first record
      int pl = pend_d - k0;
      if constexpr (!F32) {  // FP64: grouped predicated walk (walk_date asm); FP32: the same grouping below
        const double bd = P.b;
#pragma unroll
        for (int g = 0; g < kTile; g += kPushGroup) {
          double pv[kPushGroup];
          int pdl[kPushGroup];
          uint32_t pu[kPushGroup];
          uint32_t anyp = 0;
#pragma unroll
          for (int u = 0; u < kPushGroup; ++u) {
            V = add_rn(V, Z::load(zcol + (g + u) * kThreads * Z::kSize));
            cd = add_rn(cd, slope);
            pu[u] = walk_date<KIND>(V, c, cd, pl, g + u, -k0, pv[u], pdl[u], bd, bsd, x0mks);
            anyp |= pu[u];
          }
#ifndef QMCG_PROBE_NOPUSH
          if (__any_sync(kFull, anyp)) {
#pragma unroll
            for (int u = 0; u < kPushGroup; ++u)
              push_record<KIND, RNEG>(ws, P, pu[u] != 0, pv[u], k0 + pdl[u], lane, lt, rq_head, rq_tail);
          }
#else
          (void)anyp;
#endif
        }
      } else {  // FP32: the same grouping (one vote per kPushGroup dates), selects in single precision
#pragma unroll
        for (int g = 0; g < kTile; g += kPushGroup) {
          T pv[kPushGroup];
          int pdl[kPushGroup];
          bool pu[kPushGroup];
          bool anyp = false;
#pragma unroll
          for (int u = 0; u < kPushGroup; ++u) {
            V = add_rn(V, Z::load(zcol + (g + u) * kThreads * Z::kSize));
            cd = add_rn(cd, slope);
            const bool rec = KIND == 0 ? V > c : V < c;
            pu[u] = rec && (KIND == 0 || pl + k0 >= 0) && !record_dominates<KIND>(V, c, cd, bT, x0mkT);
            pv[u] = c;
            pdl[u] = pl;
            c = rec ? V : c;
            cd = rec ? (KIND == 0 ? V : T(0)) : cd;
            pl = rec ? g + u : pl;
            anyp |= pu[u];
          }
          if (__any_sync(kFull, anyp)) {
#pragma unroll
            for (int u = 0; u < kPushGroup; ++u)
              push_record<KIND, RNEG>(ws, P, pu[u], static_cast<double>(pv[u]), k0 + pdl[u], lane, lt, rq_head,
                                      rq_tail);
          }
        }
      }
      pend_d = k0 + pl;
    } else {
#pragma unroll
      for (int t = 0; t < kTile; ++t) {
        const int d = k0 + t;
        if (d < dend) {
          V = add_rn(V, det ? static_cast<T>(P.alpha) : Z::load(zcol + t * kThreads * Z::kSize));
          cd = add_rn(cd, slope);
          if (check && active) {
            const double X = fma(P.b, static_cast<double>(V), P.X0);
            if (X < -745.1332191019412) err |= ERR_SPOT_NONPOSITIVE;
            if (X > 709.782712893384) err |= ERR_SPOT_NONFINITE;
          }
          if (d < mrec) {
            const bool rec = KIND == 0 ? V > c : V < c;
            if (RNEG) {
              // every candidate is evaluated; the threshold follows the evaluated best
              push_record<KIND, RNEG>(ws, P, rec, V, d, lane, lt, rq_head, rq_tail);
            } else {
              const bool push = rec && pend_d >= 0 && !record_dominates<KIND>(V, c, cd, bT, x0mkT);
              const double pv = c;
              const int pd = pend_d;
              c = rec ? V : c;
              cd = rec ? (KIND == 0 ? V : T(0)) : cd;
              pend_d = rec ? d : pend_d;
              push_record<KIND, RNEG>(ws, P, push, pv, pd, lane, lt, rq_head, rq_tail);
            }
          }
        }
      }
    }
    if (RNEG && rq_tail - rq_head >= 32) {  // r < 0: the threshold follows the evaluated best
      __syncwarp();
      process_records_inline<KIND, RNEG>(P, ws, rq_head, 32, lane);
      rq_head += 32;
      __syncwarp();
      unsigned long long bb;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(bb) : "r"(ws + kWBest + lane * 8));
      c = static_cast<T>(rneg_threshold<KIND>(P, __longlong_as_double(static_cast<long long>(bb))));
    }
  }
  if (!RNEG && !P.stream_store) {  // the last pending record of every path
    push_record<KIND, RNEG>(ws, P, pend_d >= 0, c, pend_d, lane, lt, rq_head, rq_tail);
  }
  // The queued evaluations are drained after the last block barrier, so their
  // uneven distribution over warps never stalls the other warps of the block.
  while (rq_tail != rq_head) {
    __syncwarp();
    const uint32_t cnt = min(32u, rq_tail - rq_head);
    process_records_inline<KIND, RNEG>(P, ws, rq_head, cnt, lane);
    rq_head += cnt;
  }
  __syncwarp();
  if (P.stream_store) {  // carry-out to the next date window
    if (active) {
      const int64_t i = pi;
      double bst;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bst) : "r"(ws + kWBest + lane * 8) : "memory");
      P.st_V[i] = static_cast<double>(V);
      P.st_c[i] = static_cast<double>(c);
      P.st_cd[i] = static_cast<double>(cd);
      P.st_pend[i] = pend_d;
      P.st_best[i] = bst;
      if (err) atomicOr(P.err, err);
    }
    return;
  }

  // Date m: max(intrinsic, Black-Scholes of the final interval), american.cpp:43-52.
  const double X = fma(P.b, static_cast<double>(V), P.X0);
  const double sm_last = exp(X);
  double cont;
  if (P.bs_v_zero) {
    const double fwd = sm_last * P.bs_fwd_growth;
    double iv = KIND == 0 ? fwd - P.strike : P.strike - fwd;
    cont = P.bs_disc * (iv > 0.0 ? iv : 0.0);
  } else {
    const double d1 = (X - P.log_strike + P.bs_mu_t) / P.bs_vsqrt;
    const double d2 = d1 - P.bs_vsqrt;
    const double price = KIND == 0 ? sm_last * cnd_dev(d1) - P.bs_kdisc * cnd_dev(d2)
                                   : P.bs_kdisc * cnd_dev(-d2) - sm_last * cnd_dev(-d1);
    cont = price > 0.0 ? price : 0.0;
  }
  double intr = KIND == 0 ? sm_last - P.strike : P.strike - sm_last;
  intr = intr > 0.0 ? intr : 0.0;
  const double cm = intr > cont ? intr : cont;
  const double term_m = cm * __ldg(P.dpow + m);
  unsigned long long bb;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(bb) : "r"(ws + kWBest + lane * 8));
  const double best = __longlong_as_double(static_cast<long long>(bb));
  if (active) {
    if (!(sm_last > 0.0)) err |= ERR_SPOT_NONPOSITIVE;
    if (!isfinite(sm_last)) err |= ERR_SPOT_NONFINITE;
    if (err) atomicOr(P.err, err);
    P.values[pi] = best > term_m ? best : term_m;
  }
}

// Generation only (batches): the QMC normal table z[d][p] = moro_inv_cnd of the
// bit-exact scrambled-Halton uniform, for all dates of this block's 256 paths: each warp
// loads its row of the uniform table (coalesced) into its shared-memory row and turns it into
// normals in place with the pricing kernel's generate_row; rows are then streamed to HBM
// (coalesced, 2 KB per warp-row).
// MODE kGenPrefix: instead of z, each path's running sum S_k = z_0 + ... + z_k (the
// contract-independent part of the batch walk, V_k = S_k + (k+1) alpha_c).
template <int MODE>
__global__ void __launch_bounds__(kThreads, QMCG_MINB) gen_z_kernel(const PriceParams P, double* __restrict__ z,
                                                                    int64_t ldz) {
  constexpr bool PREFIX = MODE == kGenPrefix;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t sbase = smem_u32(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t ws = sbase + kWarpOff + warp * kWarpBytes;
  const uint32_t logtab = sbase + kLogOff;
  const unsigned lt = lanemask_lt();
  const int64_t block_first = static_cast<int64_t>(blockIdx.x) * kThreads;
  // date window [d_begin, d_end) (the whole [0, m) except for windowed exports); row d of the
  // output is d - d_begin (PREFIX needs d_begin = 0)
  const int dbeg = P.d_begin, dend = P.d_end;
  const int ntiles = (dend - dbeg + kTile - 1) / kTile;
  const int64_t block_paths = min(static_cast<int64_t>(kThreads), P.path_count - block_first);
  const int nchunks = static_cast<int>((block_paths + 31) / 32);
  const int64_t col0 = P.path_begin - P.col_begin + block_first;
  if (threadIdx.x < 128) sts_v2f64(logtab + threadIdx.x * 16, c_log_table[threadIdx.x]);
  __syncthreads();
  double run = 0.0;  // PREFIX: S of this thread's path
  const int64_t my = P.path_begin + block_first + threadIdx.x;
  const uint32_t ztile = sbase + kZtOff;
  const uint32_t zrow = ztile + warp * kThreads * 8;
  for (int k = 0; k < ntiles; ++k) {
    const int k0 = dbeg + k * kTile;
    if (k0 + warp < dend) {
      const double* src = P.table + static_cast<int64_t>(k0 + warp - P.perm_row0) * P.ld + col0;
      for (int ch = 0; ch < nchunks; ++ch) {  // padding lanes of the last chunk get a central u
        const int idx = ch * 32 + lane;
        sts_f64(zrow + idx * 8, idx < block_paths ? __ldg(src + idx) : 0.5);
      }
      __syncwarp();
      generate_row<false>(ws, zrow, logtab, nchunks, lane, lt, P.alpha);
      if (!PREFIX) {
        __syncwarp();
        double* dst = z + static_cast<int64_t>(k0 + warp - dbeg) * ldz + P.path_begin + block_first;
        for (int ch = 0; ch < nchunks; ++ch) {
          const int idx = ch * 32 + lane;
          if (idx < block_paths) __stcs(dst + idx, lds_f64(zrow + idx * 8));
        }
      }
    }
    if (PREFIX) {
      __syncthreads();  // the tile's rows are complete
      if (threadIdx.x < block_paths) {
        for (int t = 0; t < kTile && k0 + t < dend; ++t) {
          run = __dadd_rn(run, lds_f64(ztile + (t * kThreads + threadIdx.x) * 8));
          __stcs(z + static_cast<int64_t>(k0 + t) * ldz + my, run);
        }
      }
    }
    __syncthreads();  // the tile's rows are stored before they are reloaded
  }
}

// European pricing (reference mc_european_price, mc_european.cpp:11-46, with
// simulate_terminal, path_engine.cpp:154-172): one GBM step of width T from the
// dimension-0 scrambled-Halton normal (row 0 of the uniform table), discounted intrinsic per path.
__global__ void european_kernel(const double* __restrict__ urow, int64_t count, double s0, double a, double bsd,
                                double strike, double disc, int kind, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double z = moro_full(urow[i]);
  const double st = s0 * exp(fma(bsd, z, a));
  const double diff = kind == 0 ? st - strike : strike - st;
  out[i] = disc * (diff > 0.0 ? diff : 0.0);
}

// D1: uniforms (or Moro normals) of one dimension for `count` paths.
// Four entries per thread (block tile of 4 x 256, each load/store instruction coalesced), digit by
// digit: the dimension's scale constants are loaded once per digit for the four, and the four
// division chains are independent. Same arithmetic per entry as halton().
#ifndef QMCG_UNI_PER
#define QMCG_UNI_PER 4
#endif
constexpr int kUniPer = QMCG_UNI_PER;
__global__ void __launch_bounds__(256) uniforms_kernel(const uint32_t* __restrict__ perm_row, int64_t count,
                                                       DimParam dp, const double* __restrict__ sc,
                                                       const double* __restrict__ nc, int normals,
                                                       double* __restrict__ out) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * (blockDim.x * kUniPer) + threadIdx.x;
  uint32_t x[kUniPer];
  double v[kUniPer];
#pragma unroll
  for (int e = 0; e < kUniPer; ++e) {
    const int64_t i = base + e * blockDim.x;
    x[e] = i < count ? __ldg(perm_row + i) : 1u;  // table entry = perm + 1
  }
  const double* sp = sc + dp.doff;
  const double* cp = nc + dp.doff;
  const int D = static_cast<int>(dp.ndig);
  if (D == 1) {
    const double s0 = __ldg(sp), c0 = __ldg(cp);
#pragma unroll
    for (int e = 0; e < kUniPer; ++e) v[e] = digit_term(x[e], s0, c0);
  } else {
    double sj = __ldg(sp), cj = __ldg(cp);
#pragma unroll
    for (int e = 0; e < kUniPer; ++e) {
      const uint32_t q = div_p(x[e], dp);
      v[e] = digit_term(x[e] - q * dp.p, sj, cj);
      x[e] = q;
    }
    for (int j = 1; j < D - 1; ++j) {
      sj = __ldg(sp + j);
      cj = __ldg(cp + j);
#pragma unroll
      for (int e = 0; e < kUniPer; ++e) {
        const uint32_t q = div_p(x[e], dp);
        v[e] = __dadd_rn(v[e], digit_term(x[e] - q * dp.p, sj, cj));
        x[e] = q;
      }
    }
    sj = __ldg(sp + D - 1);
    cj = __ldg(cp + D - 1);
#pragma unroll
    for (int e = 0; e < kUniPer; ++e) v[e] = __dadd_rn(v[e], digit_term(x[e], sj, cj));
  }
#pragma unroll
  for (int e = 0; e < kUniPer; ++e) {
    const int64_t i = base + e * blockDim.x;
    if (i >= count) continue;
    double u = v[e];
    if (dp.flags & DIM_CLAMP) {  // kEndpointEps clamp, quasi_rng.cpp:80-81 (as in halton())
      if (u < 1e-12) u = 1e-12;
      if (u > 1.0 - 1e-12) u = 1.0 - 1e-12;
    }
    out[i] = normals ? moro_full(u) : u;
  }
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

// LCG maps s -> A^(2^k) s + C_(2^k) (mod 2^64), k = 0..63: a thread's start state is the
// composition over the set bits of its draw number (~log2(g)/2 compositions of 2 multiplies,
// instead of squaring the map through every bit).
__constant__ uint64_t c_lcg_pow[64][2];

__device__ __forceinline__ uint64_t lcg_state_after(uint64_t seed, uint64_t draws) {
  uint64_t am = 1, ap = 0;
  while (draws) {
    const int k = __ffsll(static_cast<long long>(draws)) - 1;
    const uint64_t m = c_lcg_pow[k][0], p = c_lcg_pow[k][1];
    ap = ap * m + p;
    am *= m;
    draws &= draws - 1;
  }
  return am * seed + ap;
}

// below(b) = floor(s b / 2^64) for b < 2^32 (Lcg::below, quasi_rng.hpp:20-23): the high word of
// the 96-bit product from one wide and one high 32-bit multiply.
__device__ __forceinline__ uint32_t lcg_below32(uint64_t s, uint32_t b) {
  const uint64_t hi = static_cast<uint64_t>(static_cast<uint32_t>(s >> 32)) * b;
  return static_cast<uint32_t>((hi + __umulhi(static_cast<uint32_t>(s), b)) >> 32);
}

// keys[i] = j_i >> G, vals[i] = (j_i mod 2^G) << IB | i (IB = bits of n - 1, G + IB <= 32): the
// radix sort only orders the high bits of j; fy_span_kernel finishes each 256-value span of j.
// KeyT = uint16_t when the key has at most 16 bits (n <= 2^24): a quarter less sort traffic.
template <typename KeyT>
__global__ void fy_draws_kernel(uint64_t seed, int64_t n, uint64_t stride_mult, uint64_t stride_plus,
                                KeyT* __restrict__ keys, uint32_t* __restrict__ vals, int G, int IB) {
  const int64_t G_ = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g == 0) {
    keys[0] = 0;
    vals[0] = 0;
  }
  const int64_t draws = n - 1;
  if (g >= draws) return;
  const uint32_t lowmask = (1u << G) - 1u;  // G <= 8
  // state after draw g: the warp's base state (the same jump for every lane: uniform constant
  // reads) advanced by the lane's offset (a few more steps), instead of one jump per lane whose
  // lane-dependent table indices serialise the constant cache
  const uint64_t wbase = static_cast<uint64_t>(g) & ~uint64_t{31};
  uint64_t s = lcg_state_after(lcg_state_after(seed, wbase + 1), static_cast<uint64_t>(g) - wbase);
  // draw t = g + k G_ is step i = n - 1 - t (i + 1 <= n - 1 < 2^32): 32-bit index arithmetic
  const uint32_t Gu = static_cast<uint32_t>(G_);
  const uint32_t iters = static_cast<uint32_t>((draws - g + G_ - 1) / G_);
  uint32_t i = static_cast<uint32_t>(draws - g);
  for (uint32_t k = 0; k < iters; ++k, i -= Gu) {
    const uint32_t j = lcg_below32(s, i + 1u);
    keys[i] = static_cast<KeyT>(j >> G);
    vals[i] = (G ? (j & lowmask) << IB : 0u) | i;
    s = stride_mult * s + stride_plus;
  }
}

// sstart[w] = first sorted entry whose j lies in span w (j >> 8 >= w), w = 0..nspans; also the
// bin cursors of the binned scatter. Four sorted keys per thread (one vector load).
template <typename KeyT>
__global__ void fy_span_start_kernel(const KeyT* __restrict__ sk, int64_t n, int sh, uint32_t nspans,
                                     uint32_t* __restrict__ sstart, uint32_t* __restrict__ cursor, int bin_shift) {
  // 16 bytes of sorted keys per thread (8 16-bit or 4 32-bit keys); the key before a thread's
  // first comes from the previous lane (lane 0 loads it)
  constexpr int KPT = 16 / sizeof(KeyT);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (cursor && t < kBins) cursor[t * kCursorStride] = t << bin_shift;
  const int64_t q0 = static_cast<int64_t>(t) * KPT;
  uint32_t key[KPT];
  if (q0 + KPT - 1 < n) {
    const uint4 k4 = __ldg(reinterpret_cast<const uint4*>(sk + q0));
    const uint32_t w[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
    for (int u = 0; u < KPT; ++u)
      key[u] = (sizeof(KeyT) == 4 ? w[u] : (w[u / 2] >> (16 * (u & 1))) & 0xffffu) >> sh;
  } else {
#pragma unroll
    for (int u = 0; u < KPT; ++u) key[u] = q0 + u < n ? static_cast<uint32_t>(__ldg(sk + q0 + u)) >> sh : nspans;
  }
  const uint32_t from_left = __shfl_up_sync(kFull, key[KPT - 1], 1);
  if (q0 > n) return;
  uint32_t next = q0 == 0 ? 0u
                  : lane > 0 ? from_left + 1
                             : (static_cast<uint32_t>(__ldg(sk + q0 - 1)) >> sh) + 1;  // first span not started before q0
#pragma unroll
  for (int u = 0; u < KPT; ++u) {
    if (q0 + u > n) break;
    for (uint32_t w = next; w <= key[u]; ++w) sstart[w] = static_cast<uint32_t>(q0 + u);
    next = key[u] + 1;
  }
}

// One warp per span of 256 consecutive j. A span's entries are contiguous after the sort, and
// each bucket's entries (one j) lie in ascending i (the sort is stable and they share a key), so a
// right-to-left sweep in 32-entry chunks finds, per entry, the next larger i of its bucket: the
// next lane of the chunk with the same bucket (8 ballots), else last[b], the smallest i seen so
// far to the right. Likewise fa[b] = the smallest i > x of bucket x seen so far. Outputs:
//   F[x] = min{i in bucket(x) : i > x} (or none) for every x of the span (coalesced, no memset),
//   pairs[q] = (i, S(i)) when a successor S exists, else (i, j_i).
// S > i and j_i <= i, so the chase pass tells the two apart without a flag. Two 1 KB arrays per
// warp, any span size, loads issued 4 chunks at a time (8 or 16: no faster).
#ifndef QMCG_SPAN_WARPS
#define QMCG_SPAN_WARPS 8
#endif
#ifndef QMCG_SPAN_LOOK
#define QMCG_SPAN_LOOK 4
#endif
constexpr int kSpan = 256, kSpanWarps = QMCG_SPAN_WARPS, kSpanLook = QMCG_SPAN_LOOK;
// Lanes of `eq` whose byte b equals this lane's: one ballot per bit, each combined as
// eq &= ~(ballot ^ m) with m = all ones when the bit is set (one LOP3): 3 ALU instructions per bit
// (the C++ form compiled to 5: shift, test, compare, select, combine).
__device__ __forceinline__ unsigned lanes_with_same_byte(uint32_t b, unsigned eq) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    asm("{\n .reg .pred p;\n .reg .b32 t, bb, m;\n"
        " and.b32 t, %1, %2;\n setp.ne.u32 p, t, 0;\n"
        " vote.sync.ballot.b32 bb, p, 0xffffffff;\n"
        " selp.b32 m, -1, 0, p;\n"
        " lop3.b32 %0, %0, bb, m, 0x90;\n}"
        : "+r"(eq)
        : "r"(b), "r"(1u << k));
  }
  return eq;
}
__device__ __forceinline__ uint32_t span_bucket(uint32_t key, uint32_t val, int G, int IB) {
  const uint32_t j = (key << G) | (G ? val >> IB : 0u);
  return j & (kSpan - 1);
}
template <typename KeyT>
__global__ void __launch_bounds__(kSpanWarps * 32) fy_span_kernel(const KeyT* __restrict__ sk,
                                                                  const uint32_t* __restrict__ sv, int64_t n, int G,
                                                                  int IB, const uint32_t* __restrict__ sstart,
                                                                  int64_t nspans, uint32_t* __restrict__ F,
                                                                  uint2* __restrict__ pairs) {
  __shared__ uint32_t s_last[kSpanWarps][kSpan], s_fa[kSpanWarps][kSpan];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * kSpanWarps + wib;
  if (w >= nspans) return;  // no block-wide barrier below
  uint32_t* last = s_last[wib];
  uint32_t* fa = s_fa[wib];
  const uint32_t imask = IB >= 32 ? 0xffffffffu : (1u << IB) - 1u;
  const int64_t s = sstart[w], e = sstart[w + 1];
  const uint32_t jlo = static_cast<uint32_t>(w * kSpan);
  const unsigned lt = lanemask_lt(), gt = ~lt & ~(1u << lane);
  for (int b = lane; b < kSpan; b += 32) {
    last[b] = kNone;
    fa[b] = kNone;
  }
  __syncwarp();
  for (int64_t hi = e; hi > s; hi -= 32 * kSpanLook) {
    uint32_t kk[kSpanLook], vv[kSpanLook];
#pragma unroll
    for (int u = 0; u < kSpanLook; ++u) {
      const int64_t p = hi - 32 * (u + 1) + lane;
      if (p >= s) {
        kk[u] = __ldg(sk + p);
        vv[u] = __ldg(sv + p);
      }
    }
#pragma unroll
    for (int u = 0; u < kSpanLook; ++u) {
      const int64_t p = hi - 32 * (u + 1) + lane;
      if (hi - 32 * u <= s) break;  // warp-uniform: no entry left
      const bool valid = p >= s;
      // 16-bit keys imply G = 8 (n <= 2^24): the span bucket is exactly j's low byte, vals >> IB
      const uint32_t b = !valid ? 0u : sizeof(KeyT) == 2 ? vv[u] >> IB : span_bucket(kk[u], vv[u], G, IB);
      const uint32_t i = vv[u] & imask;
      const uint32_t x = jlo + b;
      unsigned eq = __ballot_sync(kFull, valid);
      eq = lanes_with_same_byte(b, eq);
      const unsigned up = eq & gt;
      const uint32_t inext = __shfl_sync(kFull, i, up ? __ffs(up) - 1 : lane);
      const uint32_t S = up ? inext : (valid ? last[b] : kNone);
      const bool above = valid && i > x;
      const unsigned ab = __ballot_sync(kFull, above);
      __syncwarp();
      if (valid && (eq & lt) == 0) last[b] = i;    // the bucket's smallest i in this chunk
      if (above && (eq & lt & ab) == 0) fa[b] = i;  // its smallest i > x in this chunk
      __syncwarp();
      if (valid) __stcs(pairs + p, make_uint2(i, S != kNone ? S : x));
    }
  }
  for (int b = lane; b < kSpan; b += 32)
    if (static_cast<int64_t>(jlo) + b < n) F[jlo + b] = fa[b];
}

// perm[i] = v when v <= i (no successor: v = j_i), else R(v): follow F from v to the chain's end.
// Each thread follows kChase chains at once.
constexpr int kChase = 4;
__global__ void __launch_bounds__(256) fy_chase_kernel(const uint2* __restrict__ in, int64_t n,
                                                       const uint32_t* __restrict__ F, uint32_t* __restrict__ perm,
                                                       uint2* __restrict__ pairs, uint32_t add) {
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x * kChase) + threadIdx.x;
  uint32_t y[kChase], idx[kChase];
  bool live[kChase], chase[kChase];
#pragma unroll
  for (int k = 0; k < kChase; ++k) {
    const int64_t q = q0 + k * blockDim.x;
    live[k] = q < n;
    chase[k] = false;
    if (live[k]) {
      const uint2 pv = __ldcs(in + q);
      idx[k] = pv.x;
      y[k] = pv.y;
      chase[k] = pv.y > pv.x;
    }
  }
  bool any = false;
#pragma unroll
  for (int k = 0; k < kChase; ++k) any |= chase[k];
  while (any) {
    uint32_t f[kChase];
#pragma unroll
    for (int k = 0; k < kChase; ++k) f[k] = chase[k] ? __ldg(F + y[k]) : kNone;
    any = false;
#pragma unroll
    for (int k = 0; k < kChase; ++k) {
      if (chase[k]) {
        if (f[k] != kNone) y[k] = f[k];
        else chase[k] = false;
      }
      any |= chase[k];
    }
  }
#pragma unroll
  for (int k = 0; k < kChase; ++k) {
    if (!live[k]) continue;
    const int64_t q = q0 + k * blockDim.x;
    if (pairs) __stcs(pairs + q, make_uint2(idx[k], y[k] + add));
    else __stcs(perm + idx[k], y[k] + add);
  }
}

// Binned scatter, pass 1: partition the (i, perm[i]) pairs by i >> bin_shift
// into kBins bins. Bin b holds exactly the i in [b << shift, (b+1) << shift),
// so its region starts at b << shift; blocks reserve their run in each bin
// with one atomic per bin (order inside a bin is irrelevant). The tile is
// first ordered by bin in shared memory so that every warp store is a
// contiguous run of one bin (few TLB pages and full sectors per store).
constexpr int kBinThreads = 256, kBinPer = 16, kBinTile = kBinThreads * kBinPer;
__global__ void __launch_bounds__(kBinThreads) fy_bin_kernel(const uint2* __restrict__ in, int64_t n,
                                                            int bin_shift, uint32_t* __restrict__ cursor,
                                                            uint2* __restrict__ out) {
  __shared__ uint32_t cnt[kBins], start[kBins], base[kBins];
  __shared__ uint2 staged[kBinTile];
  for (int b = threadIdx.x; b < kBins; b += kBinThreads) cnt[b] = 0;
  __syncthreads();
  const int64_t tile = static_cast<int64_t>(blockIdx.x) * kBinTile;
  const int valid = static_cast<int>(min(static_cast<int64_t>(kBinTile), n - tile));
  uint2 v[kBinPer];
  uint32_t rank[kBinPer];
#pragma unroll
  for (int e = 0; e < kBinPer; ++e) {
    const int k = e * kBinThreads + threadIdx.x;
    if (k < valid) {
      v[e] = in[tile + k];
      rank[e] = atomicAdd(&cnt[v[e].x >> bin_shift], 1u);
    }
  }
  __syncthreads();
  // exclusive scan of cnt (kBins == kBinThreads: one bin per thread)
  {
    const int b = threadIdx.x;
    const uint32_t c = cnt[b];
    uint32_t x = c;
    const int lane = b & 31, w = b >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    __shared__ uint32_t wsum[kBinThreads / 32];
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    uint32_t off = 0;
    for (int k = 0; k < w; ++k) off += wsum[k];
    start[b] = off + x - c;
    if (c) base[b] = atomicAdd(cursor + b * kCursorStride, c);
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kBinPer; ++e) {
    const int k = e * kBinThreads + threadIdx.x;
    if (k < valid) staged[start[v[e].x >> bin_shift] + rank[e]] = v[e];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < valid; k += kBinThreads) {
    const uint2 p = staged[k];
    const uint32_t b = p.x >> bin_shift;
    out[base[b] + (k - start[b])] = p;
  }
}

__global__ void fill_u32_kernel(uint32_t* out, uint32_t v) { *out = v; }

// Pass 2: perm[i] = p for the binned pairs. Consecutive blocks cover
// consecutive bins, so the destination window in flight is a few bins
// (<< L2) and every 32-byte sector is completed in L2 before write-back.
__global__ void fy_scatter_kernel(const uint2* __restrict__ in, int64_t n, uint32_t* __restrict__ perm) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint2 v = in[q];
  perm[v.x] = v.y;
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

// Leaf sums, two lanes per node. A warp's 16 consecutive nodes cover one
// contiguous range of v: it is staged into shared memory with coalesced loads
// (one pad slot per 64 values keeps the lanes' sequential reads off a single
// bank). A node of <= 64 values is a leaf, summed in order from 0.0 by its even
// lane; a larger one (<= 128) splits at size / 2 as the reference does, each
// lane summing one half in order and the even lane adding the two.
// Two lanes per node halve both the stage (16 KB: ~14 warps per SM instead of 7)
// and the serial add chain of a lane (measured 0.28 ms per 2^29-value batch
// with one lane per node, 3.8 TB/s).
constexpr int kLeafWarps = 1, kLeafNodes = 16, kLeafStage = kLeafNodes * 128;
__global__ void __launch_bounds__(kLeafWarps * 32) pairwise_leaves_kernel(const double* __restrict__ v, int64_t len,
                                                                         int depth, double* __restrict__ out,
                                                                         int64_t out_stride) {
  __shared__ double stage[kLeafWarps][kLeafStage + kLeafStage / 64];
  v += static_cast<int64_t>(blockIdx.y) * len;
  out += static_cast<int64_t>(blockIdx.y) * out_stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane & 1;
  const int64_t nodes = int64_t{1} << depth;
  const int64_t first = (static_cast<int64_t>(blockIdx.x) * kLeafWarps + warp) * kLeafNodes;
  if (first >= nodes) return;
  const int64_t node = first + (lane >> 1);
  const bool live = node < nodes;
  int64_t off = 0, size = 0;
  if (live) node_range(len, depth, node, off, size);
  const int64_t r0 = __shfl_sync(kFull, off, 0);
  const int last = static_cast<int>(min(static_cast<int64_t>(kLeafNodes - 1), nodes - 1 - first));
  const int64_t r1 = __shfl_sync(kFull, off + size, 2 * last);
  const bool split = size > 64;
  const int64_t half = split ? size / 2 : size;
  const int64_t a0 = sub ? half : 0, an = sub ? size - half : half;  // this lane's part of the node
  double x, x2;
  if (r1 - r0 <= kLeafStage) {
    double* st = stage[warp];
    // 16 loads in flight per lane ahead of the shared-memory stores
    const int64_t cnt = r1 - r0;
    int64_t k = lane;
    for (; k + 15 * 32 < cnt; k += 16 * 32) {
      double y[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) y[j] = __ldcs(v + r0 + k + j * 32);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t kk = k + j * 32;
        st[kk + (kk >> 6)] = y[j];
      }
    }
    for (; k < cnt; k += 32) st[k + (k >> 6)] = v[r0 + k];
    __syncwarp();
    const int64_t b0 = off - r0 + a0;
    x = 0.0;
    x2 = 0.0;
    int64_t i = 0;
    for (; i + 8 <= an; i += 8) {  // 8 loads in flight ahead of the ordered adds
      double y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t kk = b0 + i + j;
        y[j] = st[kk + (kk >> 6)];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        x = __dadd_rn(x, y[j]);
        x2 = __dadd_rn(x2, __dmul_rn(y[j], y[j]));
      }
    }
    for (; i < an; ++i) {
      const int64_t kk = b0 + i;
      const double y = st[kk + (kk >> 6)];
      x = __dadd_rn(x, y);
      x2 = __dadd_rn(x2, __dmul_rn(y, y));
    }
  } else {
    seq_sum(v, off + a0, an, x, x2);
  }
  const double y = __shfl_down_sync(kFull, x, 1), y2 = __shfl_down_sync(kFull, x2, 1);
  if (live && !sub) {
    out[2 * node] = split ? __dadd_rn(x, y) : x;
    out[2 * node + 1] = split ? __dadd_rn(x2, y2) : x2;
  }
}

// Reduces groups of `group` (power of two <= 1024) consecutive node pairs.
__global__ void pairwise_tree_kernel(const double* __restrict__ in, int64_t count, int group,
                                     double* __restrict__ out, int64_t in_stride, int64_t out_stride) {
  __shared__ double s[1024], s2[1024];
  in += static_cast<int64_t>(blockIdx.y) * in_stride;
  out += static_cast<int64_t>(blockIdx.y) * out_stride;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * group;
  for (int i = threadIdx.x; i < group; i += blockDim.x) {
    s[i] = in[2 * (base + i)];
    s2[i] = in[2 * (base + i) + 1];
  }
  __syncthreads();
  // level by level, s[i] = s[2i] + s[2i+1] (the reference's pairing). The sums
  // of a level are formed in registers and written after a barrier: in place,
  // a warp could otherwise overwrite entries another warp has yet to read.
  for (int w = group / 2; w >= 1; w /= 2) {
    double a[4], a2[4];  // w <= 512, blockDim 256 -> at most 2 per thread
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = threadIdx.x + r * blockDim.x;
      if (i < w) {
        a[r] = __dadd_rn(s[2 * i], s[2 * i + 1]);
        a2[r] = __dadd_rn(s2[2 * i], s2[2 * i + 1]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = threadIdx.x + r * blockDim.x;
      if (i < w) {
        s[i] = a[r];
        s2[i] = a2[r];
      }
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

// Tensor map of the uniform-table slice (f64) for the pricing kernel's tile copies:
// dim 0 = columns (ld entries per row), dim 1 = the rows [0, d_end - perm_row0),
// box = kTile rows x kThreads columns (one tile of one block).
cudaError_t encode_perm_tmap(const PriceParams& P, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  static cudaError_t init_err = cudaSuccess;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    init_err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (init_err == cudaSuccess && q != cudaDriverEntryPointSuccess) init_err = cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (init_err != cudaSuccess) return init_err;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(P.ld), static_cast<cuuint64_t>(P.d_end - P.perm_row0)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(P.ld) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kThreads), static_cast<cuuint32_t>(kTile)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(P.table), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int KIND, bool RNEG, bool SLOW, bool F32>
cudaError_t launch_price_t(const PriceParams& P, cudaStream_t s) {
  const int64_t blocks = (P.path_count + kThreads - 1) / kThreads;
  const size_t smem = kSmemBytes;
  auto kern = price_kernel<KIND, RNEG, SLOW, F32>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  alignas(64) CUtensorMap tmap{};
  if (!(SLOW && P.deterministic)) {
    e = encode_perm_tmap(P, &tmap);
    if (e != cudaSuccess) return e;
  }
  kern<<<static_cast<unsigned>(blocks), kThreads, smem, s>>>(P, tmap);
  return cudaGetLastError();
}

template <int KIND, bool RNEG>
cudaError_t launch_price_k(const PriceParams& P, cudaStream_t s) {
  const bool slow = P.deterministic || P.check_range;  // digit division / clamp live in the table build
  if (P.fp32)
    return slow ? launch_price_t<KIND, RNEG, true, true>(P, s) : launch_price_t<KIND, RNEG, false, true>(P, s);
  return slow ? launch_price_t<KIND, RNEG, true, false>(P, s) : launch_price_t<KIND, RNEG, false, false>(P, s);
}

namespace {
__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

cudaError_t launch_dfma_probe(double* out, int blocks, int iters, cudaStream_t s) {
  dfma_probe_kernel<<<blocks, 256, 0, s>>>(out, iters, 0.9999, 1e-3);
  return cudaGetLastError();
}

cudaError_t ensure_log_table(cudaStream_t s);

cudaError_t launch_gen_z(const PriceParams& P, double* z, int64_t ldz, cudaStream_t s, int mode) {
  if (P.path_count <= 0) return cudaSuccess;
  cudaError_t e = ensure_log_table(s);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (P.path_count + kThreads - 1) / kThreads;
  auto kern = mode == kGenPrefix ? gen_z_kernel<kGenPrefix> : gen_z_kernel<kGenZ>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(blocks), kThreads, kSmemBytes, s>>>(P, z, ldz);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4 grouped walk. Contracts of one kind that share (spot, rate, volatility,
// maturity) follow the same log-price walk V_k = S_k + (k+1) alpha and differ
// only in the strike. For calls the dominance key W = S_k + (k+1)(alpha - slope)
// does not involve the strike, and a record k dominating j (W_k >= W_j) gives
// d^k (S_k - K) >= d^j (S_j - K) for every K; for puts the bound test is taken
// at the largest strike, which makes it valid for all smaller ones. So one walk
// per (group, path), started at the least restrictive threshold of the group,
// yields a candidate set containing every strike's surviving records, and each
// strike's value is max(I_0, max_candidates d^j (S_j - K)^+, d^m c_m(K)) --
// the same maximum the single-contract sweep computes (extra candidates are
// legitimate exercise values, so they never exceed it).
// ---------------------------------------------------------------------------
constexpr int kGThreads = 128;
#ifndef QMCG_G_MINB
#define QMCG_G_MINB 6
#endif
constexpr int kGCap = 12;  // candidates per path kept in shared memory before a flush

template <int KIND>
__device__ __noinline__ void group_flush(const ContractParams* __restrict__ cp, const GroupParams* __restrict__ g,
                                         int cnt, uint32_t cs, uint32_t cj, double* __restrict__ values, int64_t n,
                                         int64_t p, bool merge) {
  // candidates -> (S_j, d^(j+1)) in place, then fold into every strike's value
  for (int i = 0; i < cnt; ++i) {
    const double v = lds_f64(cs + i * 8);
    const uint32_t j = lds_u32(cj + i * 4);
    sts_f64(cs + i * 8, dev_exp(fma(g->b, v, g->X0)));
    sts_f64(cj + kGCap * 4 + i * 8, __ldg(g->dpow + j + 1));
  }
  for (int s = 0; s < g->count; ++s) {
    const ContractParams& q = cp[g->first + s];
    double best = merge ? values[static_cast<int64_t>(g->first + s) * n + p] : q.best0;
    for (int i = 0; i < cnt; ++i) {
      const double sv = lds_f64(cs + i * 8);
      double intr = KIND == 0 ? sv - q.strike : q.strike - sv;
      intr = intr > 0.0 ? intr : 0.0;
      const double term = intr * lds_f64(cj + kGCap * 4 + i * 8);
      best = term > best ? term : best;
    }
    values[static_cast<int64_t>(g->first + s) * n + p] = best;
  }
}

template <int KIND>
__global__ void __launch_bounds__(kGThreads, QMCG_G_MINB) walk_group_kernel(const BatchParams B) {
  extern __shared__ __align__(16) unsigned char smg[];
  const GroupParams* g = B.groups + blockIdx.x;
  const int64_t pw = static_cast<int64_t>(blockIdx.y) * kGThreads + threadIdx.x;
  const int64_t p = min(pw, B.n - 1);
  // per thread: kGCap candidate values (f64), kGCap dates (u32), then kGCap d^(j+1) (f64)
  const uint32_t cs = smem_u32(smg) + threadIdx.x * (kGCap * 20);
  const uint32_t cj = cs + kGCap * 8;
  const double alpha = g->alpha, beta = g->beta, gb = g->b, gx = g->x0mk;
  // puts: record_dominates<1>'s 1e-12 margin folded into u1 (u1 / M from one FMA, M = 1 + 4504 * 2^-52)
  constexpr double kMargin = 1.0 + 0x1198p-52;
  const double gbs = gb / kMargin, gxs = gx / kMargin;
  double c = g->c0;
  double cd = KIND == 0 ? -INFINITY : 0.0;
  int pend = -1;
  int cnt = 0;
  bool flushed = false;
  const double* zc = B.z + p;
  const int m = B.m;
  const int mrec = m - 1;
  double kd = 0.0;
  constexpr int kPf = 8;
  double zbuf[kPf];
  // the table has 8 spare rows past m - 1, so the prefetch needs no bound
  const double* zp = zc;
  const int64_t ldz = B.ldz;
#pragma unroll
  for (int t = 0; t < kPf; ++t) zbuf[t] = __ldg(zp + t * ldz);
  auto step = [&](int d, double S) {
    kd += 1.0;
    if (KIND == 0) {
      // rec = V > c; push = rec && W < cd; @push append (c, pend); then replace the pending record
      asm volatile(
          "{\n .reg .pred r, pu;\n .reg .f64 v, w;\n .reg .b32 a;\n"
          " fma.rn.f64 v, %4, %5, %6;\n fma.rn.f64 w, %7, %5, %6;\n"
          " setp.gt.f64 r, v, %0;\n setp.lt.and.f64 pu, w, %1, r;\n"
          " mad.lo.u32 a, %3, 8, %8;\n @pu st.shared.f64 [a], %0;\n"
          " mad.lo.u32 a, %3, 4, %9;\n @pu st.shared.u32 [a], %2;\n @pu add.u32 %3, %3, 1;\n"
          " selp.f64 %0, v, %0, r;\n selp.f64 %1, w, %1, r;\n selp.b32 %2, %10, %2, r;\n}"
          : "+d"(c), "+d"(cd), "+r"(pend), "+r"(cnt)
          : "d"(alpha), "d"(kd), "d"(S), "d"(beta), "r"(cs), "r"(cj), "r"(d)
          : "memory");
    } else {
      // puts, predicated: rec = V < c; acc += slope; dominated iff u1 > 0 && s < 2 &&
      // u1 s (1 - s/2) >= acc (1 + 1e-12) (record_dominates<1>); push = rec && pending && !dominated
      asm volatile(
          "{\n .reg .pred r, pe, a, b, e, dm, pu;\n .reg .f64 v, u1, dv, s, t, pr;\n .reg .b32 ad;\n"
          " fma.rn.f64 v, %4, %5, %6;\n add.rn.f64 %1, %1, %7;\n"
          " setp.lt.f64 r, v, %0;\n setp.ge.s32 pe, %2, 0;\n"
          " fma.rn.f64 u1, %13, %0, %14;\n sub.rn.f64 dv, %0, v;\n fma.rn.f64 s, %8, dv, %1;\n"
          " fma.rn.f64 t, 0dBFE0000000000000, s, 0d3FF0000000000000;\n mul.rn.f64 pr, u1, s;\n mul.rn.f64 pr, pr, t;\n"
          " setp.gt.f64 a, u1, 0d0000000000000000;\n setp.lt.and.f64 b, s, 0d4000000000000000, a;\n"
          " setp.ge.and.f64 dm, pr, %1, b;\n"
          " and.pred pu, r, pe;\n not.pred e, dm;\n and.pred pu, pu, e;\n"
          " mad.lo.u32 ad, %3, 8, %10;\n @pu st.shared.f64 [ad], %0;\n"
          " mad.lo.u32 ad, %3, 4, %11;\n @pu st.shared.u32 [ad], %2;\n @pu add.u32 %3, %3, 1;\n"
          " selp.f64 %0, v, %0, r;\n selp.f64 %1, 0d0000000000000000, %1, r;\n selp.b32 %2, %12, %2, r;\n}"
          : "+d"(c), "+d"(cd), "+r"(pend), "+r"(cnt)
          : "d"(alpha), "d"(kd), "d"(S), "d"(beta), "d"(gb), "d"(gx), "r"(cs), "r"(cj), "r"(d), "d"(gbs), "d"(gxs)
          : "memory");
    }
  };
  // rare: keep room for the next `room` candidates
  auto make_room = [&](int room) {
    if (__any_sync(kFull, cnt > kGCap - 1 - room)) {
      if (cnt > kGCap - 1 - room) {
        group_flush<KIND>(B.cp, g, cnt, cs, cj, B.values, B.n, p, flushed);
        flushed = true;
        cnt = 0;
      }
    }
  };
  int d0 = 0;
  for (; d0 + kPf <= mrec; d0 += kPf) {
    double cur[kPf];
    zp += kPf * ldz;
#pragma unroll
    for (int t = 0; t < kPf; ++t) {
      cur[t] = zbuf[t];
      zbuf[t] = __ldg(zp + t * ldz);
    }
#pragma unroll
    for (int t = 0; t < kPf; ++t) {
      step(d0 + t, cur[t]);
      if ((t & 3) == 3) make_room(4);
    }
  }
  for (int t = 0; d0 + t < mrec; ++t) {  // the last partial chunk (zbuf holds its values)
    double S = zbuf[0];
#pragma unroll
    for (int u = 1; u < kPf; ++u)
      if (u == t) S = zbuf[u];
    step(d0 + t, S);
    make_room(1);
  }
  if (pend >= 0) {  // the last pending record
    sts_f64(cs + cnt * 8, c);
    sts_u32(cj + cnt * 4, static_cast<uint32_t>(pend));
    ++cnt;
  }
  // candidates -> S_j and d^(j+1) (shared by every strike of the group)
  for (int i = 0; i < cnt; ++i) {
    const double v = lds_f64(cs + i * 8);
    const uint32_t j = lds_u32(cj + i * 4);
    sts_f64(cs + i * 8, dev_exp(fma(gb, v, g->X0)));
    sts_f64(cj + kGCap * 4 + i * 8, __ldg(g->dpow + j + 1));
  }
  kd += 1.0;
  const double X = fma(gb, fma(alpha, kd, __ldg(zc + static_cast<int64_t>(mrec) * B.ldz)), g->X0);
  const double sl = dev_exp(X);
  const double dm = __ldg(g->dpow + m);
  const double inv_vst = 1.0 / g->bs_vsqrt;
#pragma unroll 1
  for (int s = 0; s < g->count; ++s) {
    const ContractParams& q = B.cp[g->first + s];
    double best = flushed ? B.values[static_cast<int64_t>(g->first + s) * B.n + p] : q.best0;
    // best >= 0 (the date-0 intrinsic or a flushed value) and d^(j+1) > 0, so a
    // negative (S_j - K) d^(j+1) never wins the running max: the (.)^+ is implied
    const double K = q.strike;
    int i = 0;
    for (; i + 1 < cnt; i += 2) {
      const double s0 = lds_f64(cs + i * 8), s1 = lds_f64(cs + i * 8 + 8);
      const double t0 = (KIND == 0 ? s0 - K : K - s0) * lds_f64(cj + kGCap * 4 + i * 8);
      const double t1 = (KIND == 0 ? s1 - K : K - s1) * lds_f64(cj + kGCap * 4 + i * 8 + 8);
      best = t0 > best ? t0 : best;
      best = t1 > best ? t1 : best;
    }
    if (i < cnt) {
      const double s0 = lds_f64(cs + i * 8);
      const double t0 = (KIND == 0 ? s0 - K : K - s0) * lds_f64(cj + kGCap * 4 + i * 8);
      best = t0 > best ? t0 : best;
    }
    // date m: max(intrinsic, Black-Scholes of the final interval), american.cpp:43-52;
    // one exp per strike: phi(d2) = phi(d1) S / (K e^{-r dt})
    double cont;
    if (g->bs_v_zero) {
      const double fwd = sl * g->bs_fwd_growth;
      const double iv = KIND == 0 ? fwd - q.strike : q.strike - fwd;
      cont = g->bs_disc * (iv > 0.0 ? iv : 0.0);
    } else {
      const double d1 = (X - q.log_strike + g->bs_mu_t) * inv_vst;
      const double d2 = d1 - g->bs_vsqrt;
      const double e1 = dev_exp(-0.5 * d1 * d1);
      const double e2 = e1 * (sl * q.bs_inv_kdisc);
      const double price = KIND == 0 ? sl * cnd_tail_form(d1, e1) - q.bs_kdisc * cnd_tail_form(d2, e2)
                                     : q.bs_kdisc * cnd_tail_form(-d2, e2) - sl * cnd_tail_form(-d1, e1);
      cont = price > 0.0 ? price : 0.0;
    }
    double intr = KIND == 0 ? sl - q.strike : q.strike - sl;
    intr = intr > 0.0 ? intr : 0.0;
    const double cm = intr > cont ? intr : cont;
    const double term_m = cm * dm;
    if (pw < B.n) B.values[static_cast<int64_t>(g->first + s) * B.n + pw] = best > term_m ? best : term_m;
  }
}

cudaError_t launch_walk_group(const BatchParams& B, int kind, cudaStream_t s) {
  if (B.n_groups <= 0 || B.n <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>(B.n_groups), static_cast<unsigned>((B.n + kGThreads - 1) / kGThreads));
  const size_t smem = kGThreads * kGCap * 20;
  auto kern = kind == 0 ? walk_group_kernel<0> : walk_group_kernel<1>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<grid, kGThreads, smem, s>>>(B);
  return cudaGetLastError();
}

cudaError_t ensure_log_table(cudaStream_t s) {
  static bool done[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && done[dev]) return cudaSuccess;
  e = cudaMemcpyToSymbolAsync(c_log_table, kLogTable, sizeof(kLogTable), 0, cudaMemcpyHostToDevice, s);
  uint64_t pw[64][2];
  for (int k = 0; k < 64; ++k) lcg_jump(uint64_t{1} << k, pw[k][0], pw[k][1]);
  if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(c_lcg_pow, pw, sizeof(pw), 0, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && dev < 64) done[dev] = true;
  return e;
}

cudaError_t launch_price(const PriceParams& P, cudaStream_t s) {
  if (P.path_count <= 0) return cudaSuccess;
  cudaError_t e = ensure_log_table(s);
  if (e != cudaSuccess) return e;
  if (P.kind == 0) return P.rate_negative ? launch_price_k<0, true>(P, s) : launch_price_k<0, false>(P, s);
  return P.rate_negative ? launch_price_k<1, true>(P, s) : launch_price_k<1, false>(P, s);
}

cudaError_t launch_european(const double* urow, int64_t count, double s0, double a, double bsd, double strike,
                            double disc, int kind, double* out, cudaStream_t s) {
  const int64_t blocks = (count + 255) / 256;
  european_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(urow, count, s0, a, bsd, strike, disc, kind, out);
  return cudaGetLastError();
}

cudaError_t launch_uniforms(const uint32_t* perm_row, int64_t count, DimParam dp, const double* sc,
                            const double* nc, int normals, double* out, cudaStream_t s) {
  const int64_t blocks = (count + 256 * kUniPer - 1) / (256 * kUniPer);
  uniforms_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(perm_row, count, dp, sc, nc, normals, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Path matrix and per-path sweep (reference simulate_batch, path_engine.cpp:124-152,
// and sweep_impl with its trace recorder, american.cpp:19-68). Not on the pricing
// path (K2 never materialises paths); these serve the diagnostics that need them.
// ---------------------------------------------------------------------------
namespace {
// prices[k][p] (point-major, coalesced stores): S at t_1..t_m, T from
// s = s * exp(a + bsd * z) with the reference's operation order (gbm_step,
// path_engine.hpp:51-56: drift and diffusion rounded separately, no FMA).
__global__ void path_matrix_kernel(const double* __restrict__ table, int64_t ld, int64_t n, int points, double s0,
                                   double a, double bsd, double* __restrict__ out, uint32_t* err) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  double s = s0;
  uint32_t e = 0;
  for (int k = 0; k < points; ++k) {
    const double z = moro_full(table[k * ld + p]);  // the uniform table: uniform_at(p, k)
    if (!(s > 0.0)) e |= ERR_SPOT_NONPOSITIVE;  // gbm_step's s_prev check
    s = __dmul_rn(s, exp(__dadd_rn(a, __dmul_rn(bsd, z))));
    __stcs(out + k * n + p, s);
  }
  if (e) atomicOr(err, e);
}

// 32x32 tiled transpose [rows][cols] -> [cols][rows] (point-major -> the
// reference's path-major PathBatch::prices).
__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols,
                                 double* __restrict__ out) {
  __shared__ double tile[32][33];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[j][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t c = c0 + j, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][j];
  }
}

__device__ double bs_price_dev(double s, double x, double r, double v, double t, int kind) {
  // bs_price (analytic.cpp:102-124) for t > 0
  if (v == 0.0) {
    const double fwd = s * exp(r * t);
    const double iv = kind == 0 ? fwd - x : x - fwd;
    return exp(-r * t) * (iv > 0.0 ? iv : 0.0);
  }
  const double vst = __dmul_rn(v, sqrt(t));
  const double d1 = __ddiv_rn(__dadd_rn(log(__ddiv_rn(s, x)), __dmul_rn(__dadd_rn(r, __dmul_rn(__dmul_rn(0.5, v), v)), t)),
                              vst);
  const double d2 = __dadd_rn(d1, -vst);
  const double disc = exp(-r * t);
  const double price = kind == 0 ? __dadd_rn(__dmul_rn(s, cnd_dev(d1)), -__dmul_rn(__dmul_rn(x, disc), cnd_dev(d2)))
                                 : __dadd_rn(__dmul_rn(__dmul_rn(x, disc), cnd_dev(-d2)), -__dmul_rn(s, cnd_dev(-d1)));
  return price > 0.0 ? price : 0.0;
}

// One thread per path over the point-major matrix: the reference's backward
// recursion with its rounding (value * disc per point), the t_0 value and the
// earliest exercise point (the last index written with intrinsic > continuation).
__global__ void sweep_kernel(const double* __restrict__ prices, int64_t n, int m, double spot, double strike,
                             double rate, double vol, double dt, double disc, int kind, double* __restrict__ values,
                             int32_t* __restrict__ exercise) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  auto intrinsic = [&](double s) {
    const double d = kind == 0 ? s - strike : strike - s;
    return d > 0.0 ? d : 0.0;
  };
  int32_t ex = -1;
  double s = prices[static_cast<int64_t>(m - 1) * n + p];
  double cont = bs_price_dev(s, strike, rate, vol, dt, kind);
  double intr = intrinsic(s);
  double value = intr > cont ? intr : cont;
  if (intr > cont) ex = m;
  for (int i = m - 1; i >= 1; --i) {
    s = prices[static_cast<int64_t>(i - 1) * n + p];
    cont = __dmul_rn(value, disc);
    intr = intrinsic(s);
    value = intr > cont ? intr : cont;
    if (intr > cont) ex = i;
  }
  cont = __dmul_rn(value, disc);
  intr = intrinsic(spot);
  value = intr > cont ? intr : cont;
  if (intr > cont) ex = 0;
  values[p] = value;
  exercise[p] = ex;
}
}  // namespace

cudaError_t launch_path_matrix(const double* table, int64_t ld, int64_t n, int points, double s0, double a,
                               double bsd, double* out, uint32_t* err, cudaStream_t s) {
  path_matrix_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(table, ld, n, points, s0, a, bsd, out,
                                                                             err);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const double* in, int64_t rows, int64_t cols, double* out, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_sweep(const double* prices, int64_t n, int m, double spot, double strike, double rate, double vol,
                         double dt, double disc, int kind, double* values, int32_t* exercise, cudaStream_t s) {
  sweep_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(prices, n, m, spot, strike, rate, vol, dt, disc,
                                                                       kind, values, exercise);
  return cudaGetLastError();
}

namespace {
struct PermScratchLayout {
  size_t keys, vals, skeys, svals, F, cursor, sstart, temp, temp_bytes, total;
};
// bits of n - 1 (the index width IB), the j bits carried in the value (G) and the sorted key bits
struct PermBits {
  int IB, G, sort_bits;
};
PermBits perm_bits(int64_t n) {
  int IB = 1;
  while (IB < 32 && (static_cast<uint64_t>(n - 1) >> IB) != 0) ++IB;
  const int G = std::min(8, 32 - IB);
  return PermBits{IB, G, std::max(0, IB - G)};
}
PermScratchLayout perm_layout(int64_t n) {
  auto align = [](size_t x) { return (x + 255) & ~size_t{255}; };
  PermScratchLayout L{};
  const size_t arr = align(static_cast<size_t>(n) * sizeof(uint32_t));
  size_t temp_bytes = 0, temp16 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int64_t>(n), 0, 32);
  cub::DeviceRadixSort::SortPairs(nullptr, temp16, static_cast<const uint16_t*>(nullptr),
                                  static_cast<uint16_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int64_t>(n), 0, 16);
  temp_bytes = std::max(temp_bytes, temp16);
  L.keys = 0;
  L.vals = L.keys + arr;
  L.skeys = L.vals + arr;
  L.svals = L.skeys + arr;
  L.F = L.svals + arr;
  L.cursor = L.F + arr;
  L.sstart = L.cursor + align(kBins * kCursorStride * sizeof(uint32_t));
  L.temp = L.sstart + align(static_cast<size_t>((n + kSpan - 1) / kSpan + 1) * sizeof(uint32_t));
  L.temp_bytes = align(temp_bytes);
  L.total = L.temp + L.temp_bytes;
  return L;
}
}  // namespace

size_t perm_scratch_bytes(int64_t n) { return perm_layout(n).total; }

namespace {
// draws -> CUB sort of the KeyT keys (j's high bits) -> span starts -> span sweep (F and the chase
// starts in region B); regA/regB are swapped when a sort ran
template <typename KeyT>
cudaError_t k1_grouped(uint64_t seed64, int64_t n, const PermBits& pb, char* base, const PermScratchLayout& L,
                       cudaStream_t s, bool binned, int shift, char*& regA, char*& regB, int& nl) {
  const int threads = 256;
  auto* keys = reinterpret_cast<KeyT*>(base + L.keys);
  auto* vals = reinterpret_cast<uint32_t*>(base + L.vals);
  auto* F = reinterpret_cast<uint32_t*>(base + L.F);
  auto* sstart = reinterpret_cast<uint32_t*>(base + L.sstart);
  auto* cursor = reinterpret_cast<uint32_t*>(base + L.cursor);
#ifndef QMCG_DRAWS_PER_THREAD
#define QMCG_DRAWS_PER_THREAD 64
#endif
  const int64_t want = (n - 1 + QMCG_DRAWS_PER_THREAD - 1) / QMCG_DRAWS_PER_THREAD;  // draws per thread
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((want + threads - 1) / threads, 148 * 64));
  uint64_t sm, sp;
  lcg_jump(static_cast<uint64_t>(blocks) * threads, sm, sp);
  fy_draws_kernel<KeyT><<<static_cast<unsigned>(blocks), threads, 0, s>>>(seed64, n, sm, sp, keys, vals, pb.G, pb.IB);
  if (pb.sort_bits > 0) {
    size_t temp_bytes = L.temp_bytes;
    const cudaError_t e = cub::DeviceRadixSort::SortPairs(
        base + L.temp, temp_bytes, keys, reinterpret_cast<KeyT*>(base + L.skeys), vals,
        reinterpret_cast<uint32_t*>(base + L.svals), static_cast<int64_t>(n), 0, pb.sort_bits, s);
    if (e != cudaSuccess) return e;
    std::swap(regA, regB);
    nl += 2 + (pb.sort_bits + 7) / 8;  // histogram, scan, one onesweep pass per 8 key bits
  }
  const auto* sk = reinterpret_cast<const KeyT*>(regA);
  const auto* sv = reinterpret_cast<const uint32_t*>(regA + (L.vals - L.keys));
  const int64_t nspans = (n + kSpan - 1) / kSpan;
  fy_span_start_kernel<KeyT><<<static_cast<unsigned>((n / (16 / sizeof(KeyT)) + 1 + threads - 1) / threads), threads, 0, s>>>(
      sk, n, 8 - pb.G, static_cast<uint32_t>(nspans), sstart, binned ? cursor : nullptr, shift);
  fy_span_kernel<KeyT><<<static_cast<unsigned>((nspans + kSpanWarps - 1) / kSpanWarps), kSpanWarps * 32, 0, s>>>(
      sk, sv, n, pb.G, pb.IB, sstart, nspans, F, reinterpret_cast<uint2*>(regB));
  return cudaGetLastError();
}
}  // namespace

// K1 launch sequence: draws -> radix sort of j's high bits (CUB onesweep) -> span starts -> spans
// (F, chase starts) -> chase (-> binned scatter for n >= QMCG_K1_BIN_MIN).
cudaError_t launch_perm_build(uint64_t seed64, int64_t n, uint32_t* out, void* scratch, size_t scratch_bytes,
                              cudaStream_t s, int* launches, uint32_t add) {
  const PermScratchLayout L = perm_layout(n);
  if (scratch_bytes < L.total) return cudaErrorInvalidValue;
  cudaError_t e = ensure_log_table(s);  // also the LCG power table of fy_draws_kernel
  if (e != cudaSuccess) return e;
  char* base = static_cast<char*>(scratch);
  auto* F = reinterpret_cast<uint32_t*>(base + L.F);
  auto* cursor = reinterpret_cast<uint32_t*>(base + L.cursor);
  if (n == 1) {
    fill_u32_kernel<<<1, 1, 0, s>>>(out, add);
    return cudaGetLastError();
  }
  const PermBits pb = perm_bits(n);
  const int threads = 256;
  const bool binned = n >= QMCG_K1_BIN_MIN;
  int shift = 0;
  while (shift < 32 && (static_cast<uint64_t>(n - 1) >> shift) >= static_cast<uint64_t>(kBins)) ++shift;
  // sorted entries in region A (keys+vals, or skeys+svals after a sort); the chase starts go to
  // the other region B, the binned pairs back to A
  char* regA = base + L.keys;
  char* regB = base + L.skeys;
  int nl = 4;  // draws, span starts, spans, chase
  e = pb.sort_bits <= 16 ? k1_grouped<uint16_t>(seed64, n, pb, base, L, s, binned, shift, regA, regB, nl)
                         : k1_grouped<uint32_t>(seed64, n, pb, base, L, s, binned, shift, regA, regB, nl);
  if (e != cudaSuccess) return e;
  auto* starts = reinterpret_cast<uint2*>(regB);
  const int64_t ab = (n + threads * kChase - 1) / (threads * kChase);
  auto* pairs = reinterpret_cast<uint2*>(regA);  // the sorted entries are consumed by now
  fy_chase_kernel<<<static_cast<unsigned>(ab), threads, 0, s>>>(starts, n, F, out, binned ? pairs : nullptr, add);
  if (binned) {
    auto* binned_pairs = reinterpret_cast<uint2*>(regB);
    const int64_t bb = (n + kBinThreads * kBinPer - 1) / (kBinThreads * kBinPer);
    fy_bin_kernel<<<static_cast<unsigned>(bb), kBinThreads, 0, s>>>(pairs, n, shift, cursor, binned_pairs);
    fy_scatter_kernel<<<static_cast<unsigned>((n + threads - 1) / threads), threads, 0, s>>>(binned_pairs, n, out);
    nl += 2;
  }
  if (launches) *launches += nl;
  return cudaGetLastError();
}

cudaError_t pairwise_upper(double* a, int64_t nodes, int count, int64_t sa, double* b, int64_t sb, double* out2,
                           cudaStream_t s, int* launches);

size_t reduce_scratch_doubles(int64_t len) {
  const int L = leaf_depth(len);
  const int D = L > 0 ? L - 1 : 0;
  const int64_t nodes = int64_t{1} << D;
  return static_cast<size_t>(2 * nodes + 2 * ((nodes + 1023) / 1024));
}

cudaError_t launch_pairwise_batched(const double* v, int64_t len, int count, double* scratch, double* out2,
                                    cudaStream_t s, int* launches) {
  const int L = leaf_depth(len);
  const int D = L > 0 ? L - 1 : 0;
  int64_t nodes = int64_t{1} << D;
  // per contract: 2*nodes (level A) + 2*ceil(nodes/1024) (level B) doubles of scratch
  const int64_t strideA = 2 * nodes, strideB = 2 * ((nodes + 1023) / 1024);
  double* a = scratch;
  double* b = scratch + strideA * count;
  int64_t sa = strideA, sb = strideB;
  {
    const dim3 grid(static_cast<unsigned>((nodes + kLeafWarps * kLeafNodes - 1) / (kLeafWarps * kLeafNodes)),
                    static_cast<unsigned>(count));
    pairwise_leaves_kernel<<<grid, kLeafWarps * 32, 0, s>>>(v, len, D, nodes == 1 ? out2 : a, nodes == 1 ? 2 : sa);
    if (launches) ++*launches;
  }
  if (nodes == 1) return cudaGetLastError();  // the leaf pass wrote the result
  return pairwise_upper(a, nodes, count, sa, b, sb, out2, s, launches);
}

// The perfect-binary levels above a level of `nodes` node sums per vector (level at a, stride sa
// per vector), ping-ponging with b (stride sb), into out2[2c, 2c + 1].
cudaError_t pairwise_upper(double* a, int64_t nodes, int count, int64_t sa, double* b, int64_t sb, double* out2,
                           cudaStream_t s, int* launches) {
  if (nodes == 1 && a != out2) {  // a single node: its sums are the result
    return cudaMemcpy2DAsync(out2, 2 * sizeof(double), a, static_cast<size_t>(sa) * sizeof(double),
                             2 * sizeof(double), static_cast<size_t>(count), cudaMemcpyDeviceToDevice, s);
  }
  while (nodes > 1) {
    const int group = static_cast<int>(std::min<int64_t>(nodes, 1024));
    const int64_t blocks = nodes / group;
    const bool last = blocks == 1;
    double* dst = last ? out2 : b;
    const dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(count));
    pairwise_tree_kernel<<<grid, 256, 0, s>>>(a, nodes, group, dst, sa, last ? 2 : sb);
    if (launches) ++*launches;
    nodes = blocks;
    std::swap(a, b);
    std::swap(sa, sb);
  }
  return cudaGetLastError();
}

cudaError_t launch_pairwise(const double* v, int64_t len, double* scratch, double* out2, cudaStream_t s,
                            int* launches) {
  return launch_pairwise_batched(v, len, 1, scratch, out2, s, launches);
}

}  // namespace qmcg
