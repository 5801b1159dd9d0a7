"""ctypes binding of the C ABI in include/qmcg.h (libqmcg.so, built in-tree).

This is the Python face of the reference's pricing API (reference
proj/include/qmc/american.hpp:43-55, types.hpp:16-49): ``OptionSpec``,
``PricingResult``, ``ExecPolicy`` and ``price_american`` keep the reference's
names, argument meaning and error behaviour -- ``ValueError`` where the
reference throws ``std::invalid_argument``, ``OverflowError`` for
``std::length_error``, ``RuntimeError`` for device failures.

There is no CPU fallback: importing this module on a machine without the
built library raises, and every call runs the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
import threading
from typing import Optional, Sequence

import numpy as np

LIB_PATH = os.environ.get("QMCG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libqmcg.so")

OK, INVALID_ARGUMENT, LENGTH_ERROR, CUDA_ERROR, NCCL_ERROR, UNSUPPORTED, OUT_OF_MEMORY = range(7)
FLAG_ALLOW_PUT = 1
FLAG_NO_CACHE = 2
FLAG_FP32 = 4  # single-precision normals + walk (uniforms stay bit-exact FP64)


def _flags(allow_put: bool = False, no_cache: bool = False, fp32: bool = False) -> int:
    return (FLAG_ALLOW_PUT if allow_put else 0) | (FLAG_NO_CACHE if no_cache else 0) | (FLAG_FP32 if fp32 else 0)

# every symbol include/qmcg.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "qmcg_create", "qmcg_destroy", "qmcg_last_error", "qmcg_version", "qmcg_price_american",
    "qmcg_mc_european_price",
    "qmcg_price_american_batch", "qmcg_price_american_node", "qmcg_tree_node_range",
    "qmcg_combine_nodes", "qmcg_warm", "qmcg_clear_cache", "qmcg_permutation", "qmcg_uniforms",
    "qmcg_normals", "qmcg_normal_table", "qmcg_path_values", "qmcg_time_device", "qmcg_time_perm_build",
    "qmcg_last_launch_count", "qmcg_get_stream", "qmcg_fp64_peak", "qmcg_set_table_budget",
    "qmcg_last_window_count", "qmcg_price_american_nodes", "qmcg_simulate_batch", "qmcg_sweep_batch",
    "qmcg_backward_sweep", "qmcg_build_tables", "qmcg_import_tables", "qmcg_uniform_rows",
    "qmcg_create_multi", "qmcg_device_count", "qmcg_time_device_nodes", "qmcg_get_member_stream",
    "qmcg_member_device", "qmcg_price_american_batch_values", "qmcg_create_default", "qmcg_import_rows",
    "qmcg_check_canaries",
)


class OptionKind(enum.IntEnum):
    Call = 0
    Put = 1


class Method(enum.IntEnum):
    ClosedForm = 0
    EuropeanMC = 1
    AmericanUpperBound = 2


@dataclasses.dataclass
class OptionSpec:
    """reference OptionSpec (proj/include/qmc/types.hpp:24-31)."""
    spot: float = 100.0
    strike: float = 100.0
    rate: float = 0.0
    volatility: float = 0.0
    maturity: float = 0.0
    kind: OptionKind = OptionKind.Call


@dataclasses.dataclass
class PricingResult:
    """reference PricingResult (proj/include/qmc/types.hpp:42-49)."""
    price: float = 0.0
    std_error: float = 0.0
    n_paths: int = 0
    elapsed_s: float = 0.0
    method: Method = Method.ClosedForm
    seed: int = 0


@dataclasses.dataclass
class ExecPolicy:
    """reference ExecPolicy (proj/include/qmc/path_engine.hpp:36-39); never changes results."""
    lanes: int = 1
    chunk: int = 4096


class _CSpec(C.Structure):
    _fields_ = [("spot", C.c_double), ("strike", C.c_double), ("rate", C.c_double),
                ("volatility", C.c_double), ("maturity", C.c_double), ("kind", C.c_int32)]


class _CResult(C.Structure):
    _fields_ = [("price", C.c_double), ("std_error", C.c_double), ("n_paths", C.c_int64),
                ("elapsed_s", C.c_double), ("method", C.c_int32), ("seed", C.c_uint64)]


# numpy views of the C structs (qmcg_option_spec / qmcg_pricing_result), for column-wise batches
_SPEC_DT = np.dtype({"names": [f[0] for f in _CSpec._fields_],
                     "formats": [np.float64] * 5 + [np.int32],
                     "offsets": [getattr(_CSpec, f[0]).offset for f in _CSpec._fields_],
                     "itemsize": C.sizeof(_CSpec)})
_RESULT_DT = np.dtype({"names": [f[0] for f in _CResult._fields_],
                       "formats": [np.float64, np.float64, np.int64, np.float64, np.int32, np.uint64],
                       "offsets": [getattr(_CResult, f[0]).offset for f in _CResult._fields_],
                       "itemsize": C.sizeof(_CResult)})

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libqmcg.so; raises if it has not been built (no fallback exists)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_1205_0106_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(path)
        P, I64, U64, U32, D = C.c_void_p, C.c_int64, C.c_uint64, C.c_uint32, C.c_double
        PD = C.POINTER(C.c_double)
        L.qmcg_create.argtypes = [C.c_int, C.POINTER(P)]
        L.qmcg_create_multi.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(P)]
        L.qmcg_device_count.argtypes = [P]
        L.qmcg_device_count.restype = C.c_int
        L.qmcg_destroy.argtypes = [P]
        L.qmcg_destroy.restype = None
        L.qmcg_last_error.restype = C.c_char_p
        L.qmcg_version.restype = C.c_char_p
        L.qmcg_price_american.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, C.POINTER(_CResult)]
        L.qmcg_mc_european_price.argtypes = [P, C.POINTER(_CSpec), I64, U64, U32, C.POINTER(_CResult)]
        L.qmcg_price_american_batch.argtypes = [P, C.POINTER(_CSpec), I64, I64, I64, U64, U32, C.POINTER(_CResult)]
        L.qmcg_price_american_batch_values.argtypes = [P, C.POINTER(_CSpec), I64, I64, I64, U64, U32,
                                                       C.POINTER(_CResult), P]
        L.qmcg_price_american_node.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, C.c_int, I64, PD]
        L.qmcg_price_american_nodes.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, C.c_int, I64, I64, PD]
        L.qmcg_tree_node_range.argtypes = [I64, C.c_int, I64, C.POINTER(I64), C.POINTER(I64)]
        L.qmcg_combine_nodes.argtypes = [I64, C.c_int, PD, PD, PD]
        L.qmcg_warm.argtypes = [P, I64, U64, I64]
        L.qmcg_clear_cache.argtypes = [P]
        L.qmcg_set_table_budget.argtypes = [P, U64]
        L.qmcg_build_tables.argtypes = [P, I64, U64, I64, I64, I64, P, I64]
        L.qmcg_import_tables.argtypes = [P, I64, U64, I64, I64, I64, P, I64]
        L.qmcg_import_rows.argtypes = [P, I64, U64, I64, I64, I64, I64, I64, P, I64]
        L.qmcg_simulate_batch.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, C.c_int, P]
        L.qmcg_sweep_batch.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, P, P]
        L.qmcg_backward_sweep.argtypes = [P, I64, C.POINTER(_CSpec), I64, U32, P, C.POINTER(I64)]
        L.qmcg_last_window_count.argtypes = [P]
        L.qmcg_last_window_count.restype = I64
        L.qmcg_permutation.argtypes = [P, I64, U64, P]
        L.qmcg_uniforms.argtypes = [P, I64, U64, I64, P]
        L.qmcg_normals.argtypes = [P, I64, U64, I64, P]
        L.qmcg_path_values.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, P]
        L.qmcg_normal_table.argtypes = [P, I64, U64, I64, P]
        L.qmcg_uniform_rows.argtypes = [P, I64, U64, I64, I64, P]
        L.qmcg_time_device.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, C.c_int, PD, PD, PD]
        L.qmcg_time_perm_build.argtypes = [P, I64, U64, I64, PD]
        L.qmcg_time_device_nodes.argtypes = [P, C.POINTER(_CSpec), I64, I64, U64, U32, C.c_int, I64, I64, C.c_int,
                                             PD, PD, PD]
        L.qmcg_get_member_stream.argtypes = [P, C.c_int]
        L.qmcg_get_member_stream.restype = P
        L.qmcg_member_device.argtypes = [P, C.c_int]
        L.qmcg_member_device.restype = C.c_int
        L.qmcg_check_canaries.argtypes = []
        L.qmcg_last_launch_count.argtypes = [P]
        L.qmcg_last_launch_count.restype = I64
        L.qmcg_get_stream.argtypes = [P]
        L.qmcg_get_stream.restype = P
        L.qmcg_fp64_peak.argtypes = [P, D, PD]
        _lib = L
        return L


def _check(status: int) -> None:
    if status == OK:
        return
    msg = (load_library().qmcg_last_error() or b"").decode()
    if status == INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == LENGTH_ERROR:
        raise OverflowError(msg)
    if status == OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(f"qmcg status {status}: {msg}")


def _cspec(spec: OptionSpec) -> _CSpec:
    return _CSpec(float(spec.spot), float(spec.strike), float(spec.rate), float(spec.volatility),
                  float(spec.maturity), int(spec.kind))


def _result(r: _CResult) -> PricingResult:
    return PricingResult(r.price, r.std_error, int(r.n_paths), r.elapsed_s, Method(r.method), int(r.seed))


class Context:
    """One CUDA device (stream, scratch, permutation-table cache), or with `devices` a device
    group: pricing sharded over the listed devices as pairwise-tree nodes (qmcg_create_multi)."""

    def __init__(self, device: int = 0, devices: Optional[Sequence[int]] = None):
        self._lib = load_library()
        self._h = C.c_void_p()
        if devices is not None:
            ids = (C.c_int * len(devices))(*[int(d) for d in devices])
            _check(self._lib.qmcg_create_multi(ids, len(devices), C.byref(self._h)))
            self.device = int(devices[0])
            self.devices = [int(d) for d in devices]
        else:
            _check(self._lib.qmcg_create(int(device), C.byref(self._h)))
            self.device = device
            self.devices = [int(device)]

    def device_count(self) -> int:
        return int(self._lib.qmcg_device_count(self._h))

    def close(self) -> None:
        if self._h:
            self._lib.qmcg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- the hot path --
    def price_american(self, spec: OptionSpec, m: int, n_paths: int, seed: int,
                       exec: Optional[ExecPolicy] = None, allow_put: bool = False,
                       no_cache: bool = False, fp32: bool = False) -> PricingResult:
        if exec is not None:
            if exec.lanes < 1:
                raise ValueError("parallel_for_chunks: lanes must be >= 1")
            if exec.chunk < 1:
                raise ValueError("parallel_for_chunks: chunk must be >= 1")
        flags = _flags(allow_put, no_cache, fp32)
        s, r = _cspec(spec), _CResult()
        _check(self._lib.qmcg_price_american(self._h, C.byref(s), int(m), int(n_paths), int(seed), flags, C.byref(r)))
        return _result(r)

    def mc_european_price(self, spec: OptionSpec, n_paths: int, seed: int,
                          exec: Optional[ExecPolicy] = None) -> PricingResult:
        """qmc::mc_european_price (reference proj/src/mc_european.cpp:11-46)."""
        if exec is not None and (exec.lanes < 1 or exec.chunk < 1):
            raise ValueError("parallel_for_chunks: lanes must be >= 1" if exec.lanes < 1
                             else "parallel_for_chunks: chunk must be >= 1")
        s, r = _cspec(spec), _CResult()
        _check(self._lib.qmcg_mc_european_price(self._h, C.byref(s), int(n_paths), int(seed), 0, C.byref(r)))
        return _result(r)

    def price_american_batch(self, specs: Sequence[OptionSpec], m: int, n_paths: int, seed: int,
                             allow_put: bool = False) -> list:
        arr = (_CSpec * len(specs))(*[_cspec(s) for s in specs])
        res = (_CResult * len(specs))()
        flags = FLAG_ALLOW_PUT if allow_put else 0
        _check(self._lib.qmcg_price_american_batch(self._h, arr, len(specs), int(m), int(n_paths), int(seed),
                                                    flags, res))
        return [_result(r) for r in res]

    def price_american_batch_values(self, specs: Sequence[OptionSpec], m: int, n_paths: int, seed: int,
                                    allow_put: bool = False):
        """(results, (len(specs), n_paths) per-path t0 values) from the same batch launches."""
        arr = (_CSpec * len(specs))(*[_cspec(s) for s in specs])
        res = (_CResult * len(specs))()
        vals = np.zeros((len(specs), int(n_paths)), dtype=np.float64)
        _check(self._lib.qmcg_price_american_batch_values(self._h, arr, len(specs), int(m), int(n_paths), int(seed),
                                                           FLAG_ALLOW_PUT if allow_put else 0, res, vals.ctypes.data))
        return [_result(r) for r in res], vals

    def price_american_batch_arrays(self, spot, strike, rate, volatility, maturity, kind, m: int, n_paths: int,
                                    seed: int, allow_put: bool = False) -> np.ndarray:
        """Batch pricing from column arrays (one entry per contract; scalars broadcast), returning a
        (C, 2) array of (price, std_error) -- the same call as price_american_batch without per-contract
        Python objects, for large batches."""
        cols = np.broadcast_arrays(*(np.asarray(x, dtype=np.float64) for x in (spot, strike, rate, volatility,
                                                                                  maturity)),
                                   np.asarray(kind, dtype=np.int32))
        cnt = cols[0].size
        specs = np.zeros(cnt, dtype=_SPEC_DT)
        for name, col in zip(("spot", "strike", "rate", "volatility", "maturity", "kind"), cols):
            specs[name] = col.reshape(-1)
        res = np.zeros(cnt, dtype=_RESULT_DT)
        _check(self._lib.qmcg_price_american_batch(self._h, specs.ctypes.data_as(C.POINTER(_CSpec)), cnt, int(m),
                                                    int(n_paths), int(seed), FLAG_ALLOW_PUT if allow_put else 0,
                                                    res.ctypes.data_as(C.POINTER(_CResult))))
        return np.stack([res["price"], res["std_error"]], axis=1)

    def price_american_node(self, spec: OptionSpec, m: int, n_paths: int, seed: int, depth: int, node: int,
                            allow_put: bool = False, fp32: bool = False) -> np.ndarray:
        out = np.zeros(2, dtype=np.float64)
        s = _cspec(spec)
        _check(self._lib.qmcg_price_american_node(self._h, C.byref(s), int(m), int(n_paths), int(seed),
                                                   _flags(allow_put, fp32=fp32), int(depth), int(node),
                                                   out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def price_american_nodes(self, spec: OptionSpec, m: int, n_paths: int, seed: int, depth: int,
                             node_begin: int, node_count: int, allow_put: bool = False,
                             fp32: bool = False) -> np.ndarray:
        """(node_count, 2) table of (sum v, sum v^2) for consecutive tree nodes, one kernel pass."""
        out = np.zeros((int(node_count), 2), dtype=np.float64)
        s = _cspec(spec)
        _check(self._lib.qmcg_price_american_nodes(self._h, C.byref(s), int(m), int(n_paths), int(seed),
                                                    _flags(allow_put, fp32=fp32), int(depth), int(node_begin),
                                                    int(node_count), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    # -- path matrix and sweeps (reference simulate_batch / backward_sweep) --
    def simulate_batch(self, spec: OptionSpec, m: int, n_paths: int, seed: int,
                       point_major: bool = False) -> np.ndarray:
        """simulate_batch(spec, make_schedule(m, T), n_paths, seed).prices (path_engine.cpp:124-152):
        (n_paths, m+1) like the reference's row-major matrix, or (m+1, n_paths) with point_major."""
        s = _cspec(spec)
        _check(self._lib.qmcg_simulate_batch(None, C.byref(s), int(m), int(n_paths), int(seed), 0, 0, None))
        shape = (int(m) + 1, int(n_paths)) if point_major else (int(n_paths), int(m) + 1)
        out = np.zeros(shape, dtype=np.float64)
        _check(self._lib.qmcg_simulate_batch(self._h, C.byref(s), int(m), int(n_paths), int(seed), 0,
                                             1 if point_major else 0, out.ctypes.data))
        return out

    def sweep_batch(self, spec: OptionSpec, m: int, n_paths: int, seed: int, allow_put: bool = False):
        """(t_0 values, earliest exercise points) of the reference's backward sweep over every simulated path."""
        s = _cspec(spec)
        vals = np.zeros(int(n_paths), dtype=np.float64)
        ex = np.zeros(int(n_paths), dtype=np.int32)
        _check(self._lib.qmcg_sweep_batch(self._h, C.byref(s), int(m), int(n_paths), int(seed),
                                          _flags(allow_put), vals.ctypes.data, ex.ctypes.data))
        return vals, ex

    def warm(self, n_paths: int, seed: int, dims: int) -> None:
        _check(self._lib.qmcg_warm(self._h, int(n_paths), int(seed), int(dims)))

    def clear_cache(self) -> None:
        _check(self._lib.qmcg_clear_cache(self._h))

    def build_tables(self, n_paths: int, seed: int, dim_begin: int, dim_stride: int, count: int, out_ptr: int,
                     ld: int) -> None:
        """Full tables (perm + 1) of dims dim_begin + k * dim_stride into a caller device buffer."""
        _check(self._lib.qmcg_build_tables(self._h, int(n_paths), int(seed), int(dim_begin), int(dim_stride),
                                           int(count), C.c_void_p(out_ptr), int(ld)))

    def import_tables(self, n_paths: int, seed: int, col_begin: int, col_end: int, dims: int, src_ptr: int,
                      src_ld: int) -> None:
        """Install the column slice [col_begin, col_end) of dims [0, dims) from a device buffer."""
        _check(self._lib.qmcg_import_tables(self._h, int(n_paths), int(seed), int(col_begin), int(col_end), int(dims),
                                            C.c_void_p(src_ptr), int(src_ld)))

    def import_rows(self, n_paths: int, seed: int, col_begin: int, col_end: int, dims: int, row_begin: int,
                    row_count: int, src_ptr: int, src_ld: int) -> None:
        """Install rows [row_begin, +row_count) of the slice [col_begin, col_end) of dims [0, dims)."""
        _check(self._lib.qmcg_import_rows(self._h, int(n_paths), int(seed), int(col_begin), int(col_end), int(dims),
                                          int(row_begin), int(row_count), C.c_void_p(src_ptr), int(src_ld)))

    def set_table_budget(self, nbytes: int) -> None:
        """Cap the permutation-table bytes (0 = free device memory); larger pricings stream date windows."""
        _check(self._lib.qmcg_set_table_budget(self._h, int(nbytes)))

    def last_window_count(self) -> int:
        return int(self._lib.qmcg_last_window_count(self._h))

    # -- parity exports --
    def permutation(self, n: int, seed64: int) -> np.ndarray:
        out = np.zeros(max(int(n), 1), dtype=np.uint32)
        _check(self._lib.qmcg_permutation(self._h, int(n), int(seed64), out.ctypes.data))
        return out

    def uniforms(self, n: int, seed: int, dim: int) -> np.ndarray:
        out = np.zeros(int(n), dtype=np.float64)
        _check(self._lib.qmcg_uniforms(self._h, int(n), int(seed), int(dim), out.ctypes.data))
        return out

    def normals(self, n: int, seed: int, dim: int) -> np.ndarray:
        out = np.zeros(int(n), dtype=np.float64)
        _check(self._lib.qmcg_normals(self._h, int(n), int(seed), int(dim), out.ctypes.data))
        return out

    def normal_table(self, n: int, seed: int, dims: int) -> np.ndarray:
        out = np.zeros((int(dims), int(n)), dtype=np.float64)
        _check(self._lib.qmcg_normal_table(self._h, int(n), int(seed), int(dims), out.ctypes.data))
        return out

    def uniform_rows(self, n: int, seed: int, dim_begin: int, dim_count: int) -> np.ndarray:
        """(dim_count, n) uniforms of dims [dim_begin, +dim_count) from the pricing kernels' generator."""
        out = np.zeros((int(dim_count), int(n)), dtype=np.float64)
        _check(self._lib.qmcg_uniform_rows(self._h, int(n), int(seed), int(dim_begin), int(dim_count),
                                           out.ctypes.data))
        return out

    def path_values(self, spec: OptionSpec, m: int, n_paths: int, seed: int, allow_put: bool = False,
                    fp32: bool = False) -> np.ndarray:
        out = np.zeros(int(n_paths), dtype=np.float64)
        s = _cspec(spec)
        _check(self._lib.qmcg_path_values(self._h, C.byref(s), int(m), int(n_paths), int(seed),
                                          _flags(allow_put, fp32=fp32), out.ctypes.data))
        return out

    # -- measurement hooks --
    def time_device(self, spec: OptionSpec, m: int, n_paths: int, seed: int, reps: int,
                    allow_put: bool = False, fp32: bool = False):
        k, st = C.c_double(), C.c_double()
        ps = np.zeros(2, dtype=np.float64)
        s = _cspec(spec)
        _check(self._lib.qmcg_time_device(self._h, C.byref(s), int(m), int(n_paths), int(seed),
                                          _flags(allow_put, fp32=fp32), int(reps), C.byref(k), C.byref(st),
                                          ps.ctypes.data_as(C.POINTER(C.c_double))))
        return k.value, st.value, float(ps[0]), float(ps[1])

    def time_device_nodes(self, spec: OptionSpec, m: int, n_paths: int, seed: int, depth: int, node_begin: int,
                          node_count: int, reps: int, allow_put: bool = False, fp32: bool = False):
        """(kernel ms, step ms, (node_count, 2) sums) of pricing one rank's tree nodes."""
        k, st = C.c_double(), C.c_double()
        out = np.zeros((int(node_count), 2), dtype=np.float64)
        s = _cspec(spec)
        _check(self._lib.qmcg_time_device_nodes(self._h, C.byref(s), int(m), int(n_paths), int(seed),
                                                _flags(allow_put, fp32=fp32), int(depth), int(node_begin),
                                                int(node_count), int(reps), C.byref(k), C.byref(st),
                                                out.ctypes.data_as(C.POINTER(C.c_double))))
        return k.value, st.value, out

    def member_streams(self):
        """[(device, cudaStream_t)] of every member (one entry for a single-device context)."""
        return [(int(self._lib.qmcg_member_device(self._h, r)), int(self._lib.qmcg_get_member_stream(self._h, r) or 0))
                for r in range(self.device_count())]

    def time_perm_build(self, n_paths: int, seed: int, dims: int) -> float:
        ms = C.c_double()
        _check(self._lib.qmcg_time_perm_build(self._h, int(n_paths), int(seed), int(dims), C.byref(ms)))
        return ms.value

    def last_launch_count(self) -> int:
        return int(self._lib.qmcg_last_launch_count(self._h))

    def stream_ptr(self) -> int:
        """The context's cudaStream_t (wrap with torch.cuda.ExternalStream to record events)."""
        return int(self._lib.qmcg_get_stream(self._h) or 0)

    def fp64_peak(self, ms: float = 50.0) -> float:
        """Measured DFMA issue rate of the device, instructions per second."""
        out = C.c_double()
        _check(self._lib.qmcg_fp64_peak(self._h, float(ms), C.byref(out)))
        return out.value


def check_canaries() -> None:
    """Verify the guard regions of every device buffer (process started with QMCG_CANARY=1)."""
    _check(load_library().qmcg_check_canaries())


def tree_node_range(n_paths: int, depth: int, node: int):
    L = load_library()
    b, e = C.c_int64(), C.c_int64()
    _check(L.qmcg_tree_node_range(int(n_paths), int(depth), int(node), C.byref(b), C.byref(e)))
    return b.value, e.value


def backward_sweep(path, spec: OptionSpec, m: int, allow_put: bool = False):
    """backward_sweep(path, spec, make_schedule(m, T)) (reference american.cpp:88-95), host-side:
    returns (values[t_0..t_m, payoff at T], earliest exercise index or None)."""
    L = load_library()
    p = np.ascontiguousarray(path, dtype=np.float64)
    values = np.zeros(int(m) + 2, dtype=np.float64)
    ex = C.c_int64()
    s = _cspec(spec)
    _check(L.qmcg_backward_sweep(p.ctypes.data, p.size, C.byref(s), int(m), _flags(allow_put), values.ctypes.data,
                                 C.byref(ex)))
    return values, (None if ex.value < 0 else int(ex.value))


def sweep_value(path, spec: OptionSpec, m: int) -> float:
    return float(backward_sweep(path, spec, m)[0][0])


def validate_simulation(spec: OptionSpec, m: int, n_paths: int) -> None:
    """The reference's checks for simulate_batch (no GPU needed)."""
    L = load_library()
    s = _cspec(spec)
    _check(L.qmcg_simulate_batch(None, C.byref(s), int(m), int(n_paths), 0, 0, 0, None))


def combine_nodes(n_paths: int, depth: int, node_sums: np.ndarray):
    L = load_library()
    arr = np.ascontiguousarray(node_sums, dtype=np.float64).reshape(-1)
    if arr.size != 2 * (1 << depth):
        raise ValueError("combine_nodes: need 2 * 2^depth sums")
    p, s = C.c_double(), C.c_double()
    _check(L.qmcg_combine_nodes(int(n_paths), int(depth), arr.ctypes.data_as(C.POINTER(C.c_double)),
                                C.byref(p), C.byref(s)))
    return p.value, s.value


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def price_american(spec: OptionSpec, m: int, n_paths: int, seed: int,
                   exec: Optional[ExecPolicy] = None) -> PricingResult:
    """qmc::price_american (reference proj/src/american.cpp:103-131) on the default device."""
    return default_context().price_american(spec, m, n_paths, seed, exec)


def mc_european_price(spec: OptionSpec, n_paths: int, seed: int, exec: Optional[ExecPolicy] = None) -> PricingResult:
    """qmc::mc_european_price (reference proj/src/mc_european.cpp:11-46) on the default device."""
    return default_context().mc_european_price(spec, n_paths, seed, exec)


def convergence_curve(spec: OptionSpec, m_values: Sequence[int], n_paths: int, seed: int,
                      exec: Optional[ExecPolicy] = None) -> list:
    """qmc::convergence_curve (reference proj/src/american.cpp:133-150); one cached table set."""
    if len(m_values) == 0:
        raise ValueError("convergence_curve: m_values must be non-empty")
    out = []
    for m in sorted(m_values):
        r = price_american(spec, m, n_paths, seed, exec)
        out.append((m, r.price, r.std_error, r.elapsed_s))
    return out
