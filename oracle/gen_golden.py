"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs oracle/_ref/libqmcref.so (the reference's own sources compiled by
oracle/Makefile) and writes small JSON fixtures: full-precision prices and
standard errors, permutation / uniform hashes, analytic function values.
The GPU box has no /root/reference, so the parity tests read these fixtures.

usage: python oracle/gen_golden.py [--big | --only-big | --only-c5 | --only-columns | --only-c4 |
                                   --only-put-bounds]
  --big additionally prices 2^24 x 256 (config 3; ~52 GB RAM, minutes); --only-big / --only-c5
  price just config 3 / the config-5 ladder rung 2^20 x 365 and merge them into prices.json.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle  # noqa: E402

GOLD = os.path.join(os.path.dirname(HERE), "tests", "golden")
SEED = 42
REF_SPEC = (100.0, 100.0, 0.05, 0.2, 1.0)


def fnv1a64(arr: np.ndarray) -> str:
    h = 0xcbf29ce484222325
    data = np.ascontiguousarray(arr).view(np.uint8)
    # vectorised FNV-1a over bytes is sequential; do it in chunks with Python ints (fixtures are small)
    for byte in data.tobytes():
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def fnv1a64_fast(arr: np.ndarray) -> str:
    """FNV-1a 64 over the little-endian bytes of arr (numpy, exact)."""
    data = np.frombuffer(np.ascontiguousarray(arr).tobytes(), dtype=np.uint8).astype(np.uint64)
    h = np.uint64(0xcbf29ce484222325)
    prime = np.uint64(0x100000001b3)
    with np.errstate(over="ignore"):
        for b in data:  # noqa: B007 - exactness over speed (used on <= 64 MiB inputs via C helper below)
            h = (h ^ b) * prime
    return f"{int(h):016x}"


def write(name: str, obj) -> None:
    path = os.path.join(GOLD, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    print("wrote", path)


def hexf(x: float) -> str:
    return float(x).hex()


def only_big(m: int = 256, n: int = 1 << 24) -> None:
    """Price one large case with the reference and merge it into prices.json: config 3
    (2^24 x 256, --only-big) or the first rung of the config-5 ladder (2^20 x 365, --only-c5)."""
    R = oracle.Reference()
    lanes = os.cpu_count() or 1
    path = os.path.join(GOLD, "prices.json")
    doc = json.load(open(path))
    p, se, el = R.price_american(*REF_SPEC, m, n, SEED, lanes=lanes)
    doc["cases"] = [c for c in doc["cases"] if not (c["m"] == m and c["n"] == n and tuple(c["spec"]) == REF_SPEC)]
    doc["cases"].append({"spec": list(REF_SPEC), "kind": "call", "m": m, "n": n, "seed": SEED,
                         "price": hexf(p), "std_error": hexf(se), "price_dec": repr(p), "elapsed_s_ref": el,
                         "lanes": lanes})
    write("prices.json", doc)
    print(f"m={m} n={n}: price={p!r} se={se!r} ({el:.1f}s, {lanes} lanes)")


def uniform_columns() -> None:
    """FNV-1a-64 of every uniform column the pricing path reads at config 2 (2^20 x 100) and
    config 3 (2^24 x 256): uniform_at(p, d) for all p, from the reference's own functions
    (ref_uniform_column), one dimension per host thread."""
    from concurrent.futures import ThreadPoolExecutor
    R = oracle.Reference()
    primes = oracle.Oracle().first_primes(256)
    out = {"source": "oracle/_ref uniform_at composition (quasi_rng.cpp:96-101)", "seed": SEED, "sets": []}
    for n, dims in ((1 << 20, 100), (1 << 24, 256)):
        def col(d, n=n):
            return fnv1a64_c(R.uniform_column(n, SEED, d, int(primes[d])))
        with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            hashes = list(ex.map(col, range(dims)))
        out["sets"].append({"n": n, "dims": dims, "fnv1a64": hashes})
        print(f"n={n}: {dims} columns hashed")
    write("uniform_columns.json", out)


# config 4 grid: K = 80 + 40 i / 31, sigma = 0.10 + 0.40 j / 31, call for even i + j
C4_CALLS = ((0, 0), (0, 30), (10, 10), (10, 20), (21, 1), (21, 31), (31, 3), (31, 31))


def config4_goldens() -> None:
    """The reference's price_american for 8 calls of the config-4 grid at the full 2^18 x 128
    (the reference rejects puts), looped as the reference would (american.cpp:103-131)."""
    R = oracle.Reference()
    lanes = os.cpu_count() or 1
    cases = []
    for i, j in C4_CALLS:
        sp = (100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0)
        p, se, el = R.price_american(*sp, 128, 1 << 18, SEED, lanes=lanes)
        cases.append({"i": i, "j": j, "spec": list(sp), "m": 128, "n": 1 << 18, "seed": SEED, "price": hexf(p),
                      "std_error": hexf(se), "price_dec": repr(p), "elapsed_s_ref": el})
        print(f"  ({i},{j}) {sp}: {p!r} / {se!r} ({el:.2f}s)")
    write("config4.json", {"source": "oracle/_ref price_american, one call per contract", "cases": cases})


def put_bounds() -> None:
    """Lower bounds the reference's own tests apply to American prices (acceptance.cpp:118-154),
    for the put extension at the headline config: bs_price(Put) and crr_price(2048 steps,
    American put) from the reference's analytic.cpp / oracles.cpp."""
    R = oracle.Reference()
    rows = []
    for sp in [REF_SPEC, (90.0, 100.0, 0.03, 0.3, 0.5), (110.0, 100.0, 0.08, 0.15, 2.0)]:
        rows.append({"spec": list(sp), "steps": 2048, "american_put": R.crr_price(*sp, 2048, True, kind=1),
                     "european_put": R.crr_price(*sp, 2048, False, kind=1), "bs_put": R.bs_price(*sp, kind=1)})
    write("put_bounds.json", {"source": "oracle/_ref crr_price / bs_price (puts)", "cases": rows})


def main() -> None:
    if "--only-columns" in sys.argv:
        return uniform_columns()
    if "--only-c4" in sys.argv:
        return config4_goldens()
    if "--only-put-bounds" in sys.argv:
        return put_bounds()
    if "--only-big" in sys.argv:
        return only_big()
    if "--only-c5" in sys.argv:
        return only_big(365, 1 << 20)
    big = "--big" in sys.argv
    R = oracle.Reference()
    lanes = os.cpu_count() or 1
    os.makedirs(GOLD, exist_ok=True)

    # ---- prices (calls: the reference rejects puts) ----
    cases = []
    for m in (1, 2, 5, 10, 20, 50):
        cases.append((REF_SPEC, m, 1 << 18))
    cases += [(REF_SPEC, 10, 1_000_000), (REF_SPEC, 50, 1 << 16), (REF_SPEC, 100, 1 << 20),
              (REF_SPEC, 128, 1 << 18), (REF_SPEC, 256, 1 << 22)]
    extra_specs = [(90.0, 100.0, 0.03, 0.3, 0.5), (110.0, 100.0, 0.08, 0.15, 2.0), (100.0, 120.0, 0.0, 0.25, 1.0),
                   (100.0, 80.0, 0.1, 0.4, 3.0), (50.0, 150.0, 0.05, 0.5, 1.0), (100.0, 100.0, 0.05, 0.0, 1.0),
                   (100.0, 95.0, -0.02, 0.3, 1.0), (100.0, 100.0, 0.05, 0.2, 0.25)]
    for sp in extra_specs:
        cases.append((sp, 13, 3000))
        cases.append((sp, 64, 1 << 15))
    cases += [(REF_SPEC, 7, 2), (REF_SPEC, 1, 3), (REF_SPEC, 3, 257), (REF_SPEC, 300, 1000), (REF_SPEC, 33, 12345)]
    if big:
        cases.append((REF_SPEC, 256, 1 << 24))
    prices = []
    for sp, m, n in cases:
        p, se, el = R.price_american(*sp, m, n, SEED, lanes=lanes)
        prices.append({"spec": list(sp), "kind": "call", "m": m, "n": n, "seed": SEED, "price": hexf(p),
                       "std_error": hexf(se), "price_dec": repr(p), "elapsed_s_ref": el, "lanes": lanes})
        print(f"  m={m} n={n} spec={sp} price={p!r} se={se!r} ({el:.2f}s)")
    old = {}
    path = os.path.join(GOLD, "prices.json")
    if os.path.exists(path) and not big:
        old = {(tuple(c["spec"]), c["m"], c["n"]): c for c in json.load(open(path))["cases"]}
        for key, c in old.items():
            if (key[2] == 1 << 24 or key[1:] == (365, 1 << 20)) and not any((tuple(x["spec"]), x["m"], x["n"]) == key for x in prices):
                prices.append(c)  # keep a previously generated config-3 golden
    write("prices.json", {"source": "oracle/_ref (reference proj/src compiled unmodified)", "cases": prices})

    # ---- per-path values of a small case (sweep_value of every simulated path) ----
    m, n = 20, 4096
    batch = R.simulate_batch(*REF_SPEC, m, n, SEED)
    vals = np.array([R.backward_sweep(batch[p], m, *REF_SPEC)[0] for p in range(n)])
    write("path_values.json", {"spec": list(REF_SPEC), "m": m, "n": n, "seed": SEED,
                               "values_hex": [hexf(v) for v in vals]})

    # ---- permutations and dimension seeds ----
    perms = {"perm_8_42": [int(x) for x in R.permutation_indices(8, 42)],
             "dimension_seed": {str(d): str(R.dimension_seed(SEED, d)) for d in (0, 1, 2, 17, 100, 255, 364)},
             "tables": []}
    for n in (1, 2, 3, 17, 1000, 65536, 1 << 20, 1 << 24):
        dims = (0, 1, 255) if n == 1 << 24 else (0, 1, 2, 17, 100)
        for d in dims:
            sd = R.dimension_seed(SEED, d)
            pr = R.permutation_indices(n, sd)[:n]
            perms["tables"].append({"n": n, "dim": d, "seed64": str(sd), "fnv1a64": fnv1a64_c(pr),
                                    "head": [int(x) for x in pr[:4]]})
    write("permutations.json", perms)

    # ---- uniforms (QuasiStream::uniform_at) ----
    uni = {"cases": []}
    for n, dims in ((1 << 20, (0, 1, 2, 3, 50, 100)), (4099, (0, 5, 13)), (1 << 16, (0, 1, 49, 50))):
        U = R.uniform_matrix(max(dims) + 1, n, SEED)
        for d in dims:
            col = np.ascontiguousarray(U[:, d])
            uni["cases"].append({"n": n, "dim": d, "seed": SEED, "fnv1a64": fnv1a64_c(col),
                                 "head_hex": [hexf(x) for x in col[:4]]})
    write("uniforms.json", uni)

    # ---- analytic functions ----
    us = [1e-12, 1e-9, 1e-5, 0.001, 0.02, 0.0799, 0.08, 0.0800001, 0.25, 0.5, 0.58, 0.919, 0.92, 0.9200001, 0.999,
          1 - 1e-12]
    ds = [-40.0, -8.0, -7.0710678118654, -3.0, -1.0, -1e-8, 0.0, 1e-8, 0.5, 1.0, 2.5, 7.07106781186547, 7.5, 36.0,
          38.0]
    bs = [(100, 100, 0.05, 0.2, 1, 0), (100, 100, 0.05, 0.2, 1, 1), (80, 100, 0.02, 0.3, 0.5, 0),
          (120, 100, 0.0, 0.1, 2, 1), (100, 100, 0.05, 0.0, 1, 0), (100, 100, 0.05, 0.2, 0.0, 1),
          (100, 90, 0.05, 0.2, 1 / 257, 0)]
    ana = {"moro": [[hexf(u), hexf(R.moro_inv_cnd(u))] for u in us],
           "cnd": [[hexf(d), hexf(R.cnd(d))] for d in ds],
           "bs_price": [[list(map(float, b[:5])), b[5], hexf(R.bs_price(*b[:5], kind=b[5]))] for b in bs],
           "radical_inverse": [[i, bb, hexf(R.radical_inverse(i, bb))]
                               for i in (1, 2, 5, 7, 1000, 1234567, 4294967295) for bb in (2, 3, 5, 541, 1619, 2473)],
           "gbm_step": [[hexf(R.gbm_step(100, 0.25, 1.0, 0.05, 0.2))]]}
    write("analytic.json", ana)

    # ---- European QMC (mc_european_price), calls and puts ----
    eur = []
    for sp, kind, n in [(REF_SPEC, 0, 1 << 20), (REF_SPEC, 0, 1_000_000), (REF_SPEC, 1, 1 << 18),
                        ((90.0, 100.0, 0.03, 0.3, 0.5), 0, 3001), ((110.0, 100.0, 0.08, 0.15, 2.0), 1, 65536),
                        ((100.0, 90.0, 0.05, 0.0, 1.0), 0, 1000), ((110.0, 100.0, 0.05, 0.2, 0.0), 0, 64),
                        ((100.0, 120.0, -0.01, 0.4, 1.5), 1, 1 << 16)]:
        p, se, _ = R.mc_european_price(*sp, n, SEED, kind=kind, lanes=lanes)
        eur.append({"spec": list(sp), "kind": kind, "n": n, "seed": SEED, "price": hexf(p), "std_error": hexf(se)})
    write("european.json", {"source": "oracle/_ref mc_european_price", "cases": eur})

    # ---- CRR American call (reference oracles.cpp) for dominance checks ----
    crr = []
    for sp in [REF_SPEC] + extra_specs[:5]:
        if sp[3] == 0:
            continue
        crr.append({"spec": list(sp), "steps": 2048, "american_call": R.crr_price(*sp, 2048, True),
                    "european_call": R.crr_price(*sp, 2048, False), "bs_call": R.bs_price(*sp)})
    write("crr.json", crr)


_FNV_SO = None


def fnv1a64_c(arr: np.ndarray) -> str:
    """FNV-1a 64 of the array's bytes via a tiny C helper (exact, fast)."""
    global _FNV_SO
    import ctypes
    import subprocess
    import tempfile
    if _FNV_SO is None:
        src = tempfile.NamedTemporaryFile("w", suffix=".c", delete=False)
        src.write("#include <stdint.h>\n#include <stddef.h>\nuint64_t fnv(const unsigned char*p,size_t n){"
                  "uint64_t h=0xcbf29ce484222325ULL;for(size_t i=0;i<n;++i){h^=p[i];h*=0x100000001b3ULL;}return h;}")
        src.close()
        so = src.name[:-2] + ".so"
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", so, src.name])
        _FNV_SO = ctypes.CDLL(so)
        _FNV_SO.fnv.restype = ctypes.c_uint64
        _FNV_SO.fnv.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    a = np.ascontiguousarray(arr)
    return f"{_FNV_SO.fnv(a.ctypes.data, a.nbytes):016x}"


if __name__ == "__main__":
    main()
