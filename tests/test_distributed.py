"""The multi-GPU sharding host logic on CPU: world_size 2 (and 3, 4) over gloo.
Each rank owns whole subtrees of the reference's pairwise tree; the per-node
sums come from the oracle's per-path values here (on the GPU box they come from
the kernel, qmcg_price_american_node). The result must be bit-identical to the
single-process reduce_stats, like the reference across lane counts."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

SPEC = (100.0, 100.0, 0.05, 0.2, 1.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, m, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import oracle
    import paper_1205_0106_b200 as q
    from paper_1205_0106_b200 import distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle.Oracle()
    _, _, vals = O.price_american(*SPEC, m, n, 42, want_values=True)
    calls = []

    def node_sums(depth, node):
        b, e = q.tree_node_range(n, depth, node)
        calls.append((b, e))
        return np.array([O.pairwise_sum(vals[b:e]), O.pairwise_sum(vals[b:e] ** 2)])

    spec = q.OptionSpec(*SPEC)
    price, se, depth = distributed.price_american_sharded(spec, m, n, 42, node_sums_fn=node_sums)
    out[rank] = (price, se, depth, calls)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_reduction_bit_identical(world, oracle_lib):
    n, m = 3001, 12
    ref_price, ref_se = oracle_lib.price_american(*SPEC, m, n, 42)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, m, out), nprocs=world, join=True)
    covered = sorted(r for rank in range(world) for r in out[rank][3])
    assert covered[0][0] == 0 and covered[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))  # disjoint, contiguous cover
    for rank in range(world):
        price, se, depth, _ = out[rank]
        assert (price, se) == (ref_price, ref_se)
        assert (1 << depth) >= world


def _batch_worker(rank, world, port, specs, m, n, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import oracle
    import paper_1205_0106_b200 as q
    from paper_1205_0106_b200 import distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle.Oracle()
    seen = []

    def batch_fn(sub):
        seen.extend(tuple(s) for s in sub)
        return np.array([O.price_american(*s[:5], m, n, 42, kind=s[5], allow_put=True)[:2] for s in sub])

    res = distributed.price_american_batch_sharded(specs, m, n, 42, batch_fn=batch_fn)
    out[rank] = (res, seen)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_contract_sharding(world, oracle_lib):
    """Config 4 over ranks: contiguous contract blocks, all-gathered (price, se) rows equal the
    single-process batch exactly; every contract priced by exactly one rank."""
    specs = [(100.0, 80.0 + 5 * i, 0.05, 0.1 + 0.05 * i, 1.0, i % 2) for i in range(7)]
    m, n = 9, 700
    ref = np.array([oracle_lib.price_american(*s[:5], m, n, 42, kind=s[5], allow_put=True)[:2] for s in specs])
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_batch_worker, args=(world, _free_port(), specs, m, n, out), nprocs=world, join=True)
    seen = sorted(x for r in range(world) for x in out[r][1])
    assert seen == sorted(specs)
    for r in range(world):
        assert np.array_equal(out[r][0], ref)


def _tables_worker(rank, world, port, n, dims, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import oracle
    from paper_1205_0106_b200 import distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle.Oracle()
    built = []

    def build(k, begin, stride, buf):
        for j in range(k):
            d = begin + j * stride
            built.append(d)
            perm = O.permutation_indices(n, O.dimension_seed(42, d))[:n].astype(np.int64) + 1
            buf[j] = torch.from_numpy(perm.astype(np.uint32).view(np.int32))

    got = {"rows": {}}

    def imp(b, e, row_begin, rows, total):
        assert total == dims and row_begin == sum(len(v) for v in got["rows"].values())
        got["range"] = (b, e)
        got["rows"][row_begin] = rows.numpy().view(np.uint32).copy()

    # one table per rank per chunk: several chunks, the last one ragged
    distributed.warm_tables_sharded(None, n, 42, dims, build_fn=build, import_fn=imp, tables_per_chunk=1)
    table = np.concatenate([got["rows"][k] for k in sorted(got["rows"])])
    out[rank] = (built, got["range"], table)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_table_build_all_to_all(world, oracle_lib):
    """Cold multi-GPU build: dims round-robin over ranks (each built once), all-to-all of column
    slices; every rank ends with exactly its columns of every dim's table (perm + 1)."""
    n, dims = 5003, 7
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_tables_worker, args=(world, _free_port(), n, dims, out), nprocs=world, join=True)
    assert sorted(d for r in range(world) for d in out[r][0]) == list(range(dims))
    full = np.stack([oracle_lib.permutation_indices(n, oracle_lib.dimension_seed(42, d))[:n] for d in range(dims)])
    cover = sorted(out[r][1] for r in range(world))
    assert cover[0][0] == 0 and cover[-1][1] == n and all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
    for r in range(world):
        b, e = out[r][1]
        assert np.array_equal(out[r][2], (full[:, b:e] + 1).astype(np.uint32))
