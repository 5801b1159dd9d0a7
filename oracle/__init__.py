"""Parity checkers for the American-option QMC hot path -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations live here, both loaded with ctypes:

* ``Oracle``  -- ``build/libqmcoracle.so``, the plain-C restatement in
  ``qmc_oracle.c`` (each function cites the reference file:line it follows).
* ``Reference`` -- ``_ref/libqmcref.so``, the reference's OWN sources from
  ``/root/reference/proj/src`` compiled unmodified by ``Makefile`` (with the
  container-only Eigen shim in ``eigen_shim/``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package, and only as the checker or the timed
CPU baseline. The product package ``paper_1205_0106_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libqmcoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqmcref.so")
REF_TREE = "/root/reference/proj"

OK, INVALID_ARGUMENT, LENGTH_ERROR = 0, 1, 2
CALL, PUT = 0, 1
ALLOW_PUT = 1


def build(quiet: bool = True, suites: bool = False) -> None:
    """Compile the C restatement and, when the reference tree exists, oracle/_ref; with `suites`
    also the reference's own test binaries linked against libqmcg.so (build that first)."""
    out = subprocess.run(["make", "-C", HERE, "all"] + (["ref_suites"] if suites else []),
                         capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _raise(code: int, err) -> None:
    if code:
        raise OracleError(code, err.value.decode())


def _spec_args(spot, strike, rate, vol, mat):
    return (C.c_double * 5)(spot, strike, rate, vol, mat)


class _QoSpec(C.Structure):
    _fields_ = [("spot", C.c_double), ("strike", C.c_double), ("rate", C.c_double),
                ("volatility", C.c_double), ("maturity", C.c_double), ("kind", C.c_int)]


class Oracle:
    """ctypes view of build/libqmcoracle.so (the C restatement)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.qo_dimension_seed.restype = C.c_uint64
        L.qo_dimension_seed.argtypes = [C.c_uint64, C.c_int64]
        L.qo_first_primes.argtypes = [C.c_int64, C.c_void_p]
        L.qo_permutation_indices.argtypes = [C.c_int64, C.c_uint64, C.c_void_p, C.c_char_p, C.c_int]
        L.qo_radical_inverse.restype = C.c_double
        L.qo_radical_inverse.argtypes = [C.c_uint64, C.c_uint32]
        L.qo_moro_inv_cnd.argtypes = [C.c_double, C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.qo_cnd.argtypes = [C.c_double, C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.qo_bs_price.argtypes = [C.POINTER(_QoSpec), C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.qo_pairwise_sum.restype = C.c_double
        L.qo_pairwise_sum.argtypes = [C.c_void_p, C.c_int64]
        L.qo_reduce_stats.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.qo_uniform_dim.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int64, C.c_void_p, C.c_char_p, C.c_int]
        L.qo_sweep_value.restype = C.c_double
        L.qo_sweep_value.argtypes = [C.c_void_p, C.c_int64, C.POINTER(_QoSpec), C.POINTER(C.c_int)]
        L.qo_price_american.argtypes = [C.POINTER(_QoSpec), C.c_int64, C.c_int64, C.c_uint64, C.c_uint32,
                                        C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
        self.lib = L

    def dimension_seed(self, seed: int, dim: int) -> int:
        return self.lib.qo_dimension_seed(seed, dim)

    def first_primes(self, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint32)
        self.lib.qo_first_primes(count, out.ctypes.data)
        return out

    def permutation_indices(self, n: int, seed: int) -> np.ndarray:
        out = np.zeros(max(n, 1), dtype=np.uint32)
        err = C.create_string_buffer(512)
        _raise(self.lib.qo_permutation_indices(n, seed, out.ctypes.data, err, 512), err)
        return out

    def radical_inverse(self, index: int, base: int) -> float:
        return self.lib.qo_radical_inverse(index, base)

    def moro_inv_cnd(self, u: float) -> float:
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.qo_moro_inv_cnd(u, C.byref(out), err, 512), err)
        return out.value

    def cnd(self, d: float) -> float:
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.qo_cnd(d, C.byref(out), err, 512), err)
        return out.value

    def bs_price(self, spot, strike, rate, vol, mat, kind=CALL) -> float:
        s = _QoSpec(spot, strike, rate, vol, mat, kind)
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.qo_bs_price(C.byref(s), C.byref(out), err, 512), err)
        return out.value

    def pairwise_sum(self, values: np.ndarray) -> float:
        v = np.ascontiguousarray(values, dtype=np.float64)
        return self.lib.qo_pairwise_sum(v.ctypes.data, v.size)

    def reduce_stats(self, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float64)
        mean, se = C.c_double(), C.c_double()
        self.lib.qo_reduce_stats(v.ctypes.data, v.size, C.byref(mean), C.byref(se))
        return mean.value, se.value

    def uniform_dim(self, dims: int, n: int, seed: int, dim: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.float64)
        err = C.create_string_buffer(512)
        _raise(self.lib.qo_uniform_dim(dims, n, seed, dim, out.ctypes.data, err, 512), err)
        return out

    def sweep_value(self, path: np.ndarray, m: int, spot, strike, rate, vol, mat, kind=CALL) -> float:
        p = np.ascontiguousarray(path, dtype=np.float64)
        s = _QoSpec(spot, strike, rate, vol, mat, kind)
        st = C.c_int()
        v = self.lib.qo_sweep_value(p.ctypes.data, m, C.byref(s), C.byref(st))
        if st.value:
            raise OracleError(st.value, "sweep failed")
        return v

    def price_american(self, spot, strike, rate, vol, mat, m, n, seed, kind=CALL, allow_put=False,
                       want_values=False):
        s = _QoSpec(spot, strike, rate, vol, mat, kind)
        out = np.zeros(2, dtype=np.float64)
        vals = np.zeros(n, dtype=np.float64) if want_values else None
        err = C.create_string_buffer(512)
        code = self.lib.qo_price_american(C.byref(s), m, n, seed, ALLOW_PUT if allow_put else 0,
                                          vals.ctypes.data if vals is not None else None,
                                          out.ctypes.data, err, 512)
        _raise(code, err)
        if want_values:
            return float(out[0]), float(out[1]), vals
        return float(out[0]), float(out[1])


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """ctypes view of _ref/libqmcref.so (the reference's own compiled sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where {REF_TREE} exists")
        L = C.CDLL(path)
        D, I64, U64, P = C.c_double, C.c_int64, C.c_uint64, C.c_void_p
        L.ref_price_american.argtypes = [P, C.c_int, I64, I64, U64, C.c_int, I64, P, C.c_char_p, C.c_int]
        L.ref_mc_european_price.argtypes = [P, C.c_int, I64, U64, C.c_int, P, C.c_char_p, C.c_int]
        L.ref_dimension_seed.restype = U64
        L.ref_dimension_seed.argtypes = [U64, I64]
        L.ref_permutation_indices.argtypes = [I64, U64, P, C.c_char_p, C.c_int]
        L.ref_radical_inverse.restype = D
        L.ref_radical_inverse.argtypes = [U64, C.c_uint32]
        L.ref_uniform_matrix.argtypes = [I64, I64, U64, P, C.c_char_p, C.c_int]
        L.ref_uniform_column.argtypes = [I64, U64, I64, C.c_uint32, P, C.c_char_p, C.c_int]
        L.ref_moro_inv_cnd.argtypes = [D, C.POINTER(D), C.c_char_p, C.c_int]
        L.ref_cnd.argtypes = [D, C.POINTER(D), C.c_char_p, C.c_int]
        L.ref_bs_price.argtypes = [P, C.c_int, C.POINTER(D), C.c_char_p, C.c_int]
        L.ref_gbm_step.restype = D
        L.ref_gbm_step.argtypes = [D, D, D, D, D]
        L.ref_simulate_batch.argtypes = [P, C.c_int, I64, I64, U64, C.c_int, P, C.c_char_p, C.c_int]
        L.ref_backward_sweep.argtypes = [P, I64, P, C.c_int, C.POINTER(D), P, C.POINTER(I64), C.c_char_p, C.c_int]
        L.ref_tree_reduce.argtypes = [P, I64, C.c_int, C.POINTER(D), C.c_char_p, C.c_int]
        L.ref_reduce_stats.argtypes = [P, I64, C.c_int, P, C.c_char_p, C.c_int]
        L.ref_crr_price.argtypes = [P, C.c_int, I64, C.c_int, C.POINTER(D), C.c_char_p, C.c_int]
        L.ref_make_schedule.argtypes = [I64, D, C.POINTER(D), P, C.c_char_p, C.c_int]
        L.ref_default_lanes.restype = C.c_int
        L.ref_emit_records.argtypes = [C.c_int] + [P] * 9 + [C.c_int, C.c_char_p, I64, C.POINTER(I64), C.c_char_p,
                                                          C.c_int]
        L.ref_parse_csv_records.argtypes = [C.c_char_p, C.c_int] + [P] * 9 + [C.POINTER(C.c_int), C.c_char_p, C.c_int]
        self.lib = L

    def price_american(self, spot, strike, rate, vol, mat, m, n, seed, kind=CALL, lanes=1, chunk=4096):
        out = np.zeros(3, dtype=np.float64)
        err = C.create_string_buffer(1024)
        sp = _spec_args(spot, strike, rate, vol, mat)
        _raise(self.lib.ref_price_american(sp, kind, m, n, seed, lanes, chunk, out.ctypes.data, err, 1024), err)
        return float(out[0]), float(out[1]), float(out[2])

    def mc_european_price(self, spot, strike, rate, vol, mat, n, seed, kind=CALL, lanes=1):
        out = np.zeros(3, dtype=np.float64)
        err = C.create_string_buffer(1024)
        sp = _spec_args(spot, strike, rate, vol, mat)
        _raise(self.lib.ref_mc_european_price(sp, kind, n, seed, lanes, out.ctypes.data, err, 1024), err)
        return float(out[0]), float(out[1]), float(out[2])

    def dimension_seed(self, seed, dim):
        return self.lib.ref_dimension_seed(seed, dim)

    def permutation_indices(self, n, seed):
        out = np.zeros(max(n, 1), dtype=np.uint32)
        err = C.create_string_buffer(512)
        _raise(self.lib.ref_permutation_indices(n, seed, out.ctypes.data, err, 512), err)
        return out

    def radical_inverse(self, index, base):
        return self.lib.ref_radical_inverse(index, base)

    def uniform_matrix(self, dims, length, seed):
        out = np.zeros((length, dims), dtype=np.float64)
        err = C.create_string_buffer(512)
        _raise(self.lib.ref_uniform_matrix(dims, length, seed, out.ctypes.data, err, 512), err)
        return out

    def uniform_column(self, length, seed, dim, base):
        """uniform_at(p, dim) for all p (the composition inside QuasiStream::uniform_at)."""
        out = np.zeros(length, dtype=np.float64)
        err = C.create_string_buffer(512)
        _raise(self.lib.ref_uniform_column(length, seed, dim, base, out.ctypes.data, err, 512), err)
        return out

    def moro_inv_cnd(self, u):
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.ref_moro_inv_cnd(u, C.byref(out), err, 512), err)
        return out.value

    def cnd(self, d):
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.ref_cnd(d, C.byref(out), err, 512), err)
        return out.value

    def bs_price(self, spot, strike, rate, vol, mat, kind=CALL):
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.ref_bs_price(_spec_args(spot, strike, rate, vol, mat), kind, C.byref(out), err, 512), err)
        return out.value

    def gbm_step(self, s_prev, dt, z, rate, vol):
        return self.lib.ref_gbm_step(s_prev, dt, z, rate, vol)

    def simulate_batch(self, spot, strike, rate, vol, mat, m, n, seed, kind=CALL, lanes=1):
        out = np.zeros((n, m + 1), dtype=np.float64)
        err = C.create_string_buffer(1024)
        _raise(self.lib.ref_simulate_batch(_spec_args(spot, strike, rate, vol, mat), kind, m, n, seed, lanes,
                                           out.ctypes.data, err, 1024), err)
        return out

    def backward_sweep(self, path, m, spot, strike, rate, vol, mat, kind=CALL):
        p = np.ascontiguousarray(path, dtype=np.float64)
        trace = np.zeros(m + 2, dtype=np.float64)
        val, ex = C.c_double(), C.c_int64()
        err = C.create_string_buffer(512)
        _raise(self.lib.ref_backward_sweep(p.ctypes.data, m, _spec_args(spot, strike, rate, vol, mat), kind,
                                           C.byref(val), trace.ctypes.data, C.byref(ex), err, 512), err)
        return val.value, trace, (None if ex.value < 0 else ex.value)

    def emit_records(self, records, fmt: int) -> str:
        """reference emit_records (bench.cpp:203-283); records = [(method, n_paths, m, lanes, chunk, seed,
        price, std_error, elapsed_s)], fmt 0 table / 1 csv / 2 json."""
        n = len(records)
        cols = list(zip(*records))
        arr = lambda dt, k: np.ascontiguousarray(np.array(cols[k], dtype=dt))  # noqa: E731
        a = [arr(np.int32, 0), arr(np.int64, 1), arr(np.int64, 2), arr(np.int32, 3), arr(np.int64, 4),
             arr(np.uint64, 5), arr(np.float64, 6), arr(np.float64, 7), arr(np.float64, 8)]
        out = C.create_string_buffer(1 << 22)
        ln = C.c_int64()
        err = C.create_string_buffer(512)
        _raise(self.lib.ref_emit_records(n, *[x.ctypes.data for x in a], fmt, out, len(out), C.byref(ln), err, 512),
               err)
        return out.raw[: ln.value].decode()

    def parse_csv_records(self, text: str):
        maxn = 4096
        bufs = [np.zeros(maxn, dt) for dt in (np.int32, np.int64, np.int64, np.int32, np.int64, np.uint64,
                                                np.float64, np.float64, np.float64)]
        cnt = C.c_int()
        err = C.create_string_buffer(512)
        _raise(self.lib.ref_parse_csv_records(text.encode(), maxn, *[b.ctypes.data for b in bufs], C.byref(cnt),
                                              err, 512), err)
        return [tuple(b[i].item() for b in bufs) for i in range(cnt.value)]

    def tree_reduce(self, values, lanes=1):
        v = np.ascontiguousarray(values, dtype=np.float64)
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.ref_tree_reduce(v.ctypes.data, v.size, lanes, C.byref(out), err, 512), err)
        return out.value

    def reduce_stats(self, values, lanes=1):
        v = np.ascontiguousarray(values, dtype=np.float64)
        out = np.zeros(2, dtype=np.float64)
        err = C.create_string_buffer(512)
        _raise(self.lib.ref_reduce_stats(v.ctypes.data, v.size, lanes, out.ctypes.data, err, 512), err)
        return float(out[0]), float(out[1])

    def crr_price(self, spot, strike, rate, vol, mat, steps, american, kind=CALL):
        out, err = C.c_double(), C.create_string_buffer(512)
        _raise(self.lib.ref_crr_price(_spec_args(spot, strike, rate, vol, mat), kind, steps, int(american),
                                      C.byref(out), err, 512), err)
        return out.value

    def default_lanes(self):
        return self.lib.ref_default_lanes()
