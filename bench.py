"""Benchmark of the American-option QMC pricer (reference arxiv/paper_1205_0106).

Metric (BASELINE.json): path-steps/s and ms per American option at 2^24 paths x
256 dates (config 3), FP64, paths sharded over N GPUs (one process per GPU).
One "step" = one pricing call for the whole option (K2 pricing kernel + K3
pairwise reduction + result read-back); path-steps = n_paths x m.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline contract, ours:
  value       path-steps/s over K steps, device time (CUDA events on the pricer's
              stream), max over ranks, permutation tables resident in HBM (warm);
  e2e         the same through the C ABI with host buffers (spec in, result out),
              host wall clock;
  roofline    the dominant kernel (price_kernel) against the FP64 pipe peak
              measured live on this GPU (the kernel is FP64-issue bound; the
              4 B/path-step HBM stream is reported beside it);
  cpu_baseline the reference's own C++ (oracle/_ref) on this host's cores.
The call is timed (parity-pinned; the reference rejects puts); the put, whose
throughput is the same kernel, is timed beside it under "put".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PATHS = 1 << 24
M_DATES = 256
SEED = 42
SPEC = (100.0, 100.0, 0.05, 0.2, 1.0)
METRIC = "path-steps/sec and ms per American put (2^24 paths×256 dates) at 1/2/4/8 B200"
WORKLOAD = ("2^24 paths x 256 exercise dates, FP64, S0=K=100 r=0.05 sigma=0.2 T=1, seed 42; "
            "American call timed (parity-pinned, the reference rejects puts), put timed beside")
# CPU reference sample: 1/16 of the paths, same dates (the full config needs ~52 GB and ~3 min)
CPU_SAMPLE_PATHS = 1 << 20


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        self.first = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        # nvidia-smi needs a few hundred ms to start: wait for its first sample so that the samples
        # cover the timed region that follows (a K = 20 step region lasts only ~0.25 s)
        import select
        ready, _, _ = select.select([self.proc.stdout], [], [], 5.0)
        if ready:
            self.first.append(self.proc.stdout.readline())
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]  # samples during the timed regions

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() in ("active", "1"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    """The host CPU model (lscpu 'Model name', else /proc/cpuinfo)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_reference(steps, warmup, n_paths=CPU_SAMPLE_PATHS, lanes=None):
    """The reference's own price_american (oracle/_ref, compiled from proj/src) on the host cores."""
    import oracle
    ref = oracle.Reference()
    lanes = lanes or os.cpu_count() or 1
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        p, se, el = ref.price_american(*SPEC, M_DATES, n_paths, SEED, lanes=lanes)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    med = statistics.median(times)
    return {"value": n_paths * M_DATES / med, "unit": "path-steps/s", "cores": lanes, "kind": "reference",
            "sample": f"{n_paths} paths x {M_DATES} dates per call (1/{N_PATHS // n_paths} of config 3), "
                      f"full reference price_american incl. its permutation build, median of {len(times)} "
                      f"after {warmup} warm-up (reference run_benchmark method, bench.cpp:129-143)",
            "seconds_per_call": med, "price": p, "std_error": se, "times_s": times}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    # every requested step and warm-up is run; the per-call sample shrinks (2^20 -> 2^18 paths of the
    # 2^24 x 256 workload) as K + W grows, so the whole run stays within a few minutes of host time
    steps, warmup = max(1, args.steps), max(1, args.warmup)
    sample = CPU_SAMPLE_PATHS
    while sample > (1 << 18) and (steps + warmup) * sample > 24 * CPU_SAMPLE_PATHS:
        sample //= 2
    base = cpu_reference(steps, warmup, n_paths=sample)
    model = cpu_model()
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "path-steps/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
            # measured: the median per-call time of the sample this arm actually ran (no extrapolation)
            "ms_per_step": 1e3 * base["seconds_per_call"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (QMC paths from the reference's scrambled Halton stream)",
            "config": {"workload": f"reference CPU sample of config 3: {sample} paths x {M_DATES} dates per step "
                                   f"(1/{N_PATHS // sample} of the 2^24-path workload; the metric is per path-step), "
                                   "S0=K=100 r=0.05 sigma=0.2 T=1 call, seed 42, cold (each call builds its "
                                   "permutation tables, as the reference always does)",
                       "n_paths": sample, "m_dates": M_DATES, "seed": SEED, "full_workload": WORKLOAD,
                       "parallelism": f"host threads (reference lanes = {base['cores']})"},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")} | {"cpu_model": model},
            "e2e": {"value": base["value"], "unit": "path-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "reference_price": base["price"], "reference_std_error": base["std_error"],
            "times_s": base["times_s"]}
    print(json.dumps(line), flush=True)
    return 0


def fail_loudly(msg):
    print(json.dumps({"error": msg}), flush=True)
    print(f"bench.py: {msg}", file=sys.stderr, flush=True)
    return 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the config-5 stress line (2^28 x 365 FP32)")
    ap.add_argument("--records", default="", help="also write the GPU and CPU rows as the reference's CSV "
                                                 "(proj/include/qmc/bench.hpp schema; GPU rows lanes = -1)")
    ap.add_argument("--paths-log2", type=int, default=24, help="(debug) smaller path count")
    ap.add_argument("--devices", default="", help="(testing) comma-separated device list of the single-process "
                                                  "group, e.g. 0,0 (one GPU listed twice); default 0..gpus-1")
    args = ap.parse_args()
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import numpy as np
    import torch
    import paper_1205_0106_b200 as q
    from paper_1205_0106_b200 import distributed

    n_paths = 1 << args.paths_log2
    warmup = max(3, args.warmup)
    steps = max(1, args.steps)
    dist = None
    visible = torch.cuda.device_count()
    # Two multi-GPU layouts: torchrun (one process per GPU, torch.distributed for the 16-byte node
    # all-gather) or, without torchrun, ONE process driving a device group through the C ABI
    # (qmcg_create_multi: node sharding, peer-copied table slices, host fold). Both must cover
    # exactly --gpus devices; anything else is an error, never a silent single-GPU run.
    if world > 1:
        if args.gpus != world:
            return fail_loudly(f"--gpus {args.gpus} but torchrun started {world} ranks")
        mode = "ranks"
    elif args.gpus > 1 or args.devices:
        mode = "group"
    else:
        mode = "single"
    if mode == "group":
        devices = [int(x) for x in args.devices.split(",")] if args.devices else list(range(args.gpus))
        if len(devices) != args.gpus:
            return fail_loudly(f"--devices lists {len(devices)} devices for --gpus {args.gpus}")
        if max(devices) >= visible:
            return fail_loudly(f"--gpus {args.gpus} needs devices {sorted(set(devices))}, {visible} visible")
    if mode == "single" and visible < 1:
        return fail_loudly("no CUDA device visible")
    n_gpus = world if mode == "ranks" else args.gpus
    # one GPU per rank; QMCG_DIST_BACKEND=gloo (functional tests of the multi-rank flow only, e.g.
    # several ranks on one GPU, whose kernels never wait on each other) keeps the plumbing on the host
    backend = os.environ.get("QMCG_DIST_BACKEND", "nccl")
    device = local_rank % max(1, visible)
    if mode == "ranks":
        import torch.distributed as dist
        torch.cuda.set_device(device)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"

    def max_over_ranks(*vals):
        if not dist:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return tuple(float(x) for x in t.tolist())

    if mode == "group":
        ctx = q.Context(devices=devices)
    else:
        ctx = q.Context(device)
    assert ctx.device_count() == (len(devices) if mode == "group" else 1)
    call = q.OptionSpec(*SPEC, kind=q.OptionKind.Call)
    put = q.OptionSpec(*SPEC, kind=q.OptionKind.Put)
    depth = distributed.tree_depth(n_paths, world)
    my_nodes = distributed.rank_nodes(depth, world, rank)
    # device streams of this process (one per group member): CUDA events on each, max over them
    members = ctx.member_streams()
    ext = [(torch.cuda.ExternalStream(sp, device=torch.device("cuda", dv)), dv) for dv, sp in members]

    class DeviceTimer:
        """Elapsed device time of the work queued between start() and stop() on every member stream
        of this process (max over members; then max over ranks by the caller)."""

        def start(self):
            self.ev = []
            for st, dv in ext:
                e0 = torch.cuda.Event(enable_timing=True)
                with torch.cuda.device(dv):
                    e0.record(st)
                self.ev.append([e0, None, st, dv])

        def stop(self):
            for rec in self.ev:
                e1 = torch.cuda.Event(enable_timing=True)
                with torch.cuda.device(rec[3]):
                    e1.record(rec[2])
                rec[1] = e1
            for rec in self.ev:
                rec[1].synchronize()
            return max(e0.elapsed_time(e1) for e0, e1, _, _ in self.ev)

    def sync_all():
        for dv in sorted({dv for dv, _ in members}):
            torch.cuda.synchronize(dv)

    def price(spec, m, n, **kw):
        if mode == "ranks":
            p, se, _ = distributed.price_american_sharded(spec, m, n, SEED, ctx=ctx, **kw)
            return p, se
        r = ctx.price_american(spec, m, n, SEED, **kw)
        return r.price, r.std_error

    # ---- config 5 (stress): 2^28 paths x 365 dates, FP32 walk, one cold call, run first (on a fresh
    # device). One GPU: tables rebuilt by K1 in date windows (392 GB > HBM). A group: dims built
    # sharded over the members, each member's 2^28/G-column slice resident or windowed ----
    c5 = None
    if not args.no_c5 and args.paths_log2 == 24:
        ctx.price_american(call, 16, 1 << 12, SEED, fp32=True)  # module and launch setup outside the timing
        ctx.clear_cache()
        n5, m5 = 1 << 28, 365
        if dist:
            dist.barrier()
        sync_all()
        tm = DeviceTimer()
        t0 = time.perf_counter()
        tm.start()
        sharded5 = False
        if mode == "ranks":
            # dims built once each (rank d mod N), column slices exchanged a chunk at a time, when the
            # rank's slice of all 365 tables fits (N >= 4: <= 98 GB); else every rank streams windows
            b5, e5 = distributed.rank_columns(n5, world, rank)
            free_b, _ = torch.cuda.mem_get_info(device)
            sharded5 = max_over_ranks(float((e5 - b5 + 64) * 4 * m5 > 0.85 * free_b))[0] == 0.0
            if sharded5:
                distributed.warm_tables_sharded(ctx, n5, SEED, m5)
        p5, se5 = price(call, m5, n5, fp32=True)
        ms5 = tm.stop()
        w5 = time.perf_counter() - t0
        windows = ctx.last_window_count()
        if dist:
            ms5, w5 = max_over_ranks(ms5, w5)
        c5 = {"workload": "config 5: 2^28 paths x 365 dates, FP32 normals + walk (bit-exact FP64 uniforms), call, "
                          "seed 42, cold (K1 rebuilds every table)"
                          + (f", dims built sharded over {n_gpus} devices" if n_gpus > 1 else ""),
              "value": n5 * m5 / (ms5 * 1e-3), "unit": "path-steps/s", "ms_per_option": ms5,
              "e2e_ms_per_option": 1e3 * w5, "date_windows_member0": windows,
              "k1": ("dimension-sharded over the devices" if (mode == "group" or sharded5) else
                     "every table built on this device" if n_gpus == 1 else "replicated per rank (slice > HBM)"),
              "tables": "streamed date windows" if windows > 1 else "resident", "price": p5, "std_error": se5}
        ctx.clear_cache()

    # ---- cold: (a) K1 alone for every table this process needs; (b) one measured cold pricing call
    # through the C ABI (QMCG_FLAG_NO_CACHE: table allocation + K1 + pricing, like the reference's
    # elapsed_s, which includes its QuasiStream construction, american.cpp:113-116) ----
    if mode != "ranks":
        cold_perm_ms = ctx.time_perm_build(n_paths, SEED, M_DATES)
    else:
        # dimension-sharded K1 (dim d on rank d mod N) + all-to-all of column slices
        dist.barrier()
        t0 = time.perf_counter()
        distributed.warm_tables_sharded(ctx, n_paths, SEED, M_DATES)
        dist.barrier()
        cold_perm_ms = max_over_ranks(1e3 * (time.perf_counter() - t0))[0]
    cold_e2e = []
    for rep in range(4):  # one untimed cold call first (first-touch of the freshly mapped table memory)
        if dist:
            dist.barrier()
        sync_all()
        t0 = time.perf_counter()
        if mode == "ranks":
            ctx.clear_cache()
            distributed.warm_tables_sharded(ctx, n_paths, SEED, M_DATES)
            cp, cse = price(call, M_DATES, n_paths)
        else:
            cp, cse = price(call, M_DATES, n_paths, no_cache=True)
        w = time.perf_counter() - t0
        if dist:
            w = max_over_ranks(w)[0]
        if rep:
            cold_e2e.append(w)

    def path_steps_fp32(ms):
        return n_paths * M_DATES / (ms * 1e-3)

    def timed(spec, allow_put=False, **kw):
        for _ in range(warmup):
            price(spec, M_DATES, n_paths, allow_put=allow_put, **kw)
        if dist:
            dist.barrier()
        sync_all()
        launches = 0
        tm = DeviceTimer()
        t0 = time.perf_counter()
        tm.start()
        for _ in range(steps):
            res = price(spec, M_DATES, n_paths, allow_put=allow_put, **kw)
            launches += ctx.last_launch_count()
        dev_ms = tm.stop()
        wall = time.perf_counter() - t0
        if dist:
            dist.barrier()
            dev_ms, wall = max_over_ranks(dev_ms, wall)
        return dev_ms / steps, wall / steps, res, launches

    # clocks sampled across both timed regions (call, then put)
    for _ in range(warmup):
        price(call, M_DATES, n_paths)
    sampler = ClockSampler(sorted({dv for dv, _ in members})[0])
    sampler.__enter__()
    ms_call, wall_call, (price_c, se), launches = timed(call)
    ms_put, wall_put, (price_put, se_put), _ = timed(put, allow_put=True)
    sampler.__exit__(None, None, None)
    clocks = sampler.summary()

    # ---- the FP32 variant (QMCG_FLAG_FP32: Moro and the walk in single precision on the exact FP64
    # uniforms) at the same config, beside the FP64 headline; not the headline (dtype f64) ----
    fp32 = None
    if mode != "ranks":
        f_ms_call, f_wall_call, (f_price_c, f_se), _ = timed(call, fp32=True)
        f_ms_put, f_wall_put, (f_price_put, f_se_put), _ = timed(put, allow_put=True, fp32=True)
        fp32 = {"call_ms_per_step": f_ms_call, "call_value": path_steps_fp32(f_ms_call), "call_price": f_price_c,
                "call_price_minus_fp64": f_price_c - price_c, "put_ms_per_step": f_ms_put,
                "put_value": path_steps_fp32(f_ms_put), "put_price": f_price_put,
                "put_price_minus_fp64": f_price_put - price_put, "std_error": f_se,
                "note": "QMCG_FLAG_FP32 at config 3; the price difference to FP64 is far below the QMC standard "
                        "error (the north star's FP32 bar)"}

    # ---- dominant kernel alone (CUDA events around price_kernel on each pricing stream), every N:
    # one GPU / a group: qmcg_time_device (max over members); ranks: this rank's nodes, max over ranks ----
    if mode == "ranks":
        kernel_ms, step_ms, _ = ctx.time_device_nodes(call, M_DATES, n_paths, SEED, depth, my_nodes[0],
                                                      len(my_nodes), 10)
        kernel_ms, step_ms = max_over_ranks(kernel_ms, step_ms)
    else:
        kernel_ms, step_ms, _, _ = ctx.time_device(call, M_DATES, n_paths, SEED, 10)
    fp64_peak = ctx.fp64_peak(100.0)

    # ---- config 4: 1024 contracts, 32 strikes x 32 vols, calls/puts alternating, 2^18 paths x
    # 128 dates, one shared permutation set; contracts sharded over the devices (N > 1);
    # contract-path-steps/s, max over devices ----
    batch = None
    if not args.no_batch:
        bspecs = [q.OptionSpec(100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0, q.OptionKind((i + j) % 2))
                  for i in range(32) for j in range(32)]
        bn, bm = 1 << 18, 128

        gi, gj = np.meshgrid(np.arange(32), np.arange(32), indexing="ij")
        b_strike, b_vol, b_kind = 80 + 40 * gi.ravel() / 31, 0.10 + 0.40 * gj.ravel() / 31, (gi + gj).ravel() % 2

        def batch_step():
            if mode != "ranks":  # column arrays: no per-contract Python objects in the timed call
                return ctx.price_american_batch_arrays(100.0, b_strike, 0.05, b_vol, 1.0, b_kind, bm, bn, SEED,
                                                       allow_put=True)
            return distributed.price_american_batch_sharded(bspecs, bm, bn, SEED, ctx=ctx, allow_put=True)

        if mode == "single":
            ctx.warm(bn, SEED, bm)
        batch_step()
        if dist:
            dist.barrier()
        sync_all()
        breps = 3
        tm = DeviceTimer()
        t0 = time.perf_counter()
        tm.start()
        for _ in range(breps):
            bres = batch_step()
        bms = tm.stop() / breps
        bwall = (time.perf_counter() - t0) / breps
        if dist:
            bms, bwall = max_over_ranks(bms, bwall)
        batch = {"workload": "config 4: 1024 contracts (K = 80..120 x sigma = 0.10..0.50, calls for even i+j), "
                             "2^18 paths x 128 dates, seed 42, qmcg_price_american_batch"
                             + (f" on {n_gpus} devices (contiguous contract blocks)" if n_gpus > 1 else ""),
                 "value": len(bspecs) * bn * bm / (bms * 1e-3), "unit": "contract-path-steps/s",
                 "ms_per_batch": bms, "e2e_ms_per_batch": 1e3 * bwall, "us_per_contract": 1e3 * bms / len(bspecs),
                 "price_first": float(bres[0][0]), "price_last": float(bres[-1][0])}
        ctx.clear_cache()

    path_steps = n_paths * M_DATES
    value = path_steps / (ms_call * 1e-3)
    e2e_value = path_steps / wall_call
    peaks = read_peaks()
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_inputs.json")) as f:
            prof = json.load(f)
    except OSError:
        pass
    fp64_per_step = prof.get("fp64_inst_per_path_step")
    bytes_per_step = prof.get("algorithmic_bytes_per_path_step", 8)  # one f64 uniform-table entry
    roofline = None
    # per-device work: each device prices n_paths / n_gpus paths in kernel_ms
    dev_path_steps = path_steps / n_gpus
    if kernel_ms and fp64_per_step:
        achieved = fp64_per_step * dev_path_steps / (kernel_ms * 1e-3) / 1e12
        roofline = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak / 1e12,
                    "unit": "T FP64-inst/s", "frac": achieved * 1e12 / fp64_peak,
                    "traffic": prof.get("dram_bytes_per_launch"),
                    "algorithmic_per_path_step": fp64_per_step,
                    "peak_source": "measured live: DFMA issue-rate probe (qmcg_fp64_peak) on this GPU",
                    "kernel_ms": kernel_ms, "per_device": n_gpus > 1,
                    "hbm": {"achieved": bytes_per_step * dev_path_steps / (kernel_ms * 1e-3) / 1e9,
                            "peak": peaks.get("hbm_gbs", 6650.0), "unit": "GB/s",
                            "frac": bytes_per_step * dev_path_steps / (kernel_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                            "algorithmic_bytes_per_path_step": bytes_per_step,
                            "peak_source": "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback"}}
        if n_gpus > 1:
            roofline["note"] = ("per device: the slowest device's pricing kernel over its n/N paths; traffic is the "
                                "1-GPU ncu capture")
        wi = prof.get("warp_inst_per_warp_date")
        if wi:
            # the binding limit: one warp instruction per cycle per scheduler (4 per SM)
            sm_hz = (clocks or {}).get("sm_mhz") or 1965.0
            issue_peak = 4 * 148 * sm_hz * 1e6
            issue_ach = wi * (dev_path_steps / 32) / (kernel_ms * 1e-3)
            roofline["issue"] = {"achieved": issue_ach / 1e12, "peak": issue_peak / 1e12, "unit": "T warp-inst/s",
                                 "frac": issue_ach / issue_peak, "warp_inst_per_warp_date": wi,
                                 "note": "FP64 instructions are a third of the kernel's issue slots; the schedulers' "
                                         "issue rate, not the FP64 pipe, bounds the kernel"}

    cpu = None
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        try:
            cpu_full = cpu_reference(steps=3, warmup=1)  # the reference's method: warm-up + median of 3
            cpu = {k: cpu_full[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu["cpu_model"] = cpu_model()
            one = cpu_reference(steps=3, warmup=0, n_paths=1 << 17, lanes=1)
            cpu["lanes1"] = {"value": one["value"], "unit": "path-steps/s", "cores": 1,
                             "sample": f"{1 << 17} paths x {M_DATES} dates, median of 3 calls, ExecPolicy lanes = 1",
                             "seconds_per_call": one["seconds_per_call"]}
            if batch is not None:  # config 4 on the CPU = sampled contracts, per contract-path-step
                import oracle
                ref = oracle.Reference()
                t0 = time.perf_counter()
                for (i, j) in ((0, 0), (31, 31)):  # calls of the grid (the reference rejects puts)
                    ref.price_american(100.0, 80 + 40 * i / 31, 0.05, 0.10 + 0.40 * j / 31, 1.0, 128, 1 << 18, SEED,
                                       lanes=os.cpu_count() or 1)
                per = (time.perf_counter() - t0) / 2
                batch["cpu_baseline"] = {"value": (1 << 18) * 128 / per, "unit": "contract-path-steps/s",
                                         "cores": os.cpu_count() or 1, "kind": "reference",
                                         "sample": "2 calls of the grid (K=80, sigma=0.10; K=120, sigma=0.50) at "
                                                   "2^18 x 128, one reference price_american each (tables built per "
                                                   "call, as the reference does)",
                                         "seconds_per_contract": per}
            if args.records:  # the reference's CSV schema: GPU row (lanes = -1) next to its CPU row
                from paper_1205_0106_b200 import records as R
                gpu_row = R.BenchmarkRecord(q.Method.AmericanUpperBound, n_paths, M_DATES, R.GPU_LANES, 4096,
                                            SEED, price_c, se, wall_call)
                cpu_row = R.BenchmarkRecord(q.Method.AmericanUpperBound, CPU_SAMPLE_PATHS, M_DATES,
                                            cpu_full["cores"], 4096, SEED, cpu_full["price"], cpu_full["std_error"],
                                            cpu_full["seconds_per_call"])
                R.emit_results([gpu_row, cpu_row], R.OutputFormat.Csv, args.records)
        except Exception as exc:  # the reference build is test infrastructure; report, don't fail
            cpu = {"value": None, "error": str(exc)[:200]}

    if rank == 0:
        cold_med = statistics.median(cold_e2e)
        layout = ("one process, one device" if mode == "single" else
                  f"one process, device group {devices} (qmcg_create_multi)" if mode == "group" else
                  "one process per GPU (torchrun, NCCL all-gather of node sums)")
        line = {"metric": METRIC, "value": value, "unit": "path-steps/s", "n_gpus": n_gpus, "steps": steps,
                "warmup": warmup, "ms_per_step": ms_call, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (QMC paths from the reference's scrambled Halton stream, seed 42)",
                "config": {"workload": WORKLOAD, "n_paths": n_paths, "m_dates": M_DATES, "seed": SEED,
                           "parallelism": f"paths sharded over {n_gpus} GPU(s) (pairwise-tree nodes); {layout}",
                           "tables": "warm: the uniform table (uniform_at of every date and path, built from the K1 "
                                     "permutations) resident in HBM; the cold call is measured separately",
                           "l2": "inputs larger than L2 (8 B x 2^24 x 256 = 34.4 GB of uniform table per step)"},
                "e2e": {"value": e2e_value, "unit": "path-steps/s", "h2d_bytes_per_step": 48,
                        "d2h_bytes_per_step": 20, "ms_per_option": 1e3 * wall_call,
                        "bytes_note": "in: the 48-byte qmcg_option_spec, which reaches the device inside the "
                                      "kernel parameters (the discount chain, 8 (m + 1) B, is uploaded only when "
                                      "it changes); out: (sum v, sum v^2) + the error word, pinned D2H",
                        "api": "qmcg_price_american (C ABI) per step" + (
                            " per rank + all-gather" if mode == "ranks" else "")},
                "roofline": roofline, "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks,
                "price": price_c, "std_error": se,
                "put": {"value": path_steps / (ms_put * 1e-3), "ms_per_step": ms_put, "price": price_put,
                        "std_error": se_put, "e2e_value": path_steps / wall_put},
                "fp32_variant": fp32,
                "cold": {"perm_build_ms": cold_perm_ms,
                         "e2e_ms_per_option_cold": 1e3 * cold_med,
                         "e2e_value_cold": path_steps / cold_med,
                         "e2e_cold_s_all": cold_e2e,
                         "note": "one real cold call per sample through the C ABI (QMCG_FLAG_NO_CACHE: table "
                                 "allocation + K1 for all 256 tables + pricing), median of 3 after one untimed "
                                 "cold call, host wall clock -- "
                                 "the counterpart of the reference's elapsed_s, which includes its QuasiStream "
                                 "construction; perm_build_ms is K1 alone" + (
                                     "" if mode == "single" else "; tables built dimension-sharded over the "
                                     "devices with column slices exchanged")},
                "kernel_ms": kernel_ms, "device_step_ms": step_ms, "batch_config4": batch,
                "stress_config5": c5}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
