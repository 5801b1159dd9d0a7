"""The multi-rank bench flow end to end on the one GPU this box has: two ranks (torchrun), paths
sharded as pairwise-tree nodes, node sums all-gathered over gloo (QMCG_DIST_BACKEND=gloo; the
ranks' kernels never wait on each other), config 4 sharded by contract. The combined price must
equal the single-process price bit for bit -- the property the NCCL run on 8 GPUs relies on.
A functional test; no timing from it is a measurement."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_bench_matches_single(ctx, qmcg):
    env = dict(os.environ, QMCG_DIST_BACKEND="gloo", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-c5", "--paths-log2", "18"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    spec = qmcg.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
    one = ctx.price_american(spec, 256, 1 << 18, 42)
    assert (line["price"], line["std_error"]) == (one.price, one.std_error)
    put = ctx.price_american(qmcg.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, kind=qmcg.OptionKind.Put), 256, 1 << 18,
                             42, allow_put=True)
    assert line["put"]["price"] == put.price
    b = line["batch_config4"]
    first = ctx.price_american(qmcg.OptionSpec(100.0, 80.0, 0.05, 0.10, 1.0), 128, 1 << 18, 42)
    assert abs(b["price_first"] - first.price) <= 1e-12 * first.price


def test_group_bench_matches_single(ctx, qmcg):
    """`bench.py --gpus 2` without torchrun: one process, a device group (here the one GPU listed
    twice). Same prices as one device, bit for bit, and a roofline at N > 1."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--devices", "0,0", "--steps", "1",
           "--warmup", "3", "--no-cpu-baseline", "--no-c5", "--paths-log2", "18"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and "device group" in line["config"]["parallelism"]
    spec = qmcg.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0)
    one = ctx.price_american(spec, 256, 1 << 18, 42)
    assert (line["price"], line["std_error"]) == (one.price, one.std_error)
    assert line["roofline"] and line["roofline"]["kernel_ms"] > 0
    assert line["cold"]["e2e_ms_per_option_cold"] > 0


def test_bench_refuses_missing_devices():
    """--gpus N with fewer visible devices must fail loudly, never price on one GPU."""
    import torch
    n = torch.cuda.device_count() + 1
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 2 and "visible" in out.stdout
