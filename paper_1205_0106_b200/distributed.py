"""Multi-GPU path sharding (one process per GPU, torch.distributed for plumbing).

Paths are independent end to end (the foresight rule is per path, reference
proj/src/american.cpp:32-68), so the only exchange is the final reduction.
The reference reduces with a fixed pairwise tree (pairwise_sum,
proj/src/path_engine.cpp:37-47); ranks own whole subtrees of that tree -- the
nodes at depth ceil(log2 world) -- and compute their subtree sums (sum v,
sum v^2) on their GPU. The node table is all-gathered (16 bytes per node, no
arithmetic in the collective) and every rank folds it up the same tree on the
host (qmcg_combine_nodes). The result is therefore bit-identical for any
world size, exactly as the reference is for any lane count.
"""
from __future__ import annotations

import math
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import qmcg


def tree_depth(n_paths: int, world_size: int) -> int:
    """Smallest depth with at least world_size nodes whose ancestors are all split (> 64 paths)."""
    want = 0 if world_size <= 1 else math.ceil(math.log2(world_size))
    depth = 0
    while depth < want:
        # nodes at depth+1 exist only if every node at `depth` is larger than a leaf (64)
        smallest = n_paths >> depth  # floor(n / 2^depth) is the smallest node size at this depth
        if smallest <= 64:
            break
        depth += 1
    return depth


def node_owner(depth: int, world_size: int) -> List[int]:
    """Contiguous assignment of the 2^depth nodes to ranks (rank r owns a contiguous path range)."""
    nodes = 1 << depth
    return [min(world_size - 1, (i * world_size) // nodes) for i in range(nodes)]


def rank_nodes(depth: int, world_size: int, rank: int) -> List[int]:
    return [i for i, r in enumerate(node_owner(depth, world_size)) if r == rank]


def combine(n_paths: int, depth: int, table: np.ndarray) -> Tuple[float, float]:
    """Fold the (2^depth, 2) node table up the reference tree -> (price, std_error)."""
    return qmcg.combine_nodes(n_paths, depth, table)


def _all_gather_rows(table: np.ndarray, group=None) -> List[np.ndarray]:
    """all_gather of an equally-shaped float64 array from every rank (NCCL on GPU, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [table]
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    local = torch.from_numpy(np.ascontiguousarray(table)).to(dev)
    gathered = [torch.empty_like(local) for _ in range(dist.get_world_size(group))]
    dist.all_gather(gathered, local, group=group)
    return [g.cpu().numpy() for g in gathered]


def price_american_sharded(spec: "qmcg.OptionSpec", m: int, n_paths: int, seed: int, *,
                           ctx: Optional["qmcg.Context"] = None,
                           node_sums_fn: Optional[Callable[[int, int], np.ndarray]] = None,
                           allow_put: bool = False, fp32: bool = False, group=None) -> Tuple[float, float, int]:
    """Price one option with the paths sharded over the ranks of `group`.

    Each rank prices the contiguous path range of the tree nodes it owns in one
    kernel pass (qmcg_price_american_nodes); node_sums_fn(depth, node) ->
    [sum v, sum v^2] replaces that (CPU tests). Returns (price, std_error, depth).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    depth = tree_depth(n_paths, world)
    mine = rank_nodes(depth, world, rank)
    table = np.zeros((1 << depth, 2), dtype=np.float64)
    if mine:
        if node_sums_fn is not None:
            for node in mine:
                table[node] = node_sums_fn(depth, node)
        else:
            if ctx is None:
                raise ValueError("price_american_sharded: pass ctx or node_sums_fn")
            table[mine[0]:mine[-1] + 1] = ctx.price_american_nodes(spec, m, n_paths, seed, depth, mine[0],
                                                                  len(mine), allow_put=allow_put, fp32=fp32)
    if world > 1:
        rows = _all_gather_rows(table, group)
        owners = node_owner(depth, world)
        table = np.stack([rows[owners[i]][i] for i in range(1 << depth)])
    price, se = combine(n_paths, depth, table)
    return price, se, depth


def contract_range(n_contracts: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of contracts owned by `rank` (config 4: contracts shard, paths do not)."""
    return (n_contracts * rank) // world, (n_contracts * (rank + 1)) // world


def price_american_batch_sharded(specs: Sequence["qmcg.OptionSpec"], m: int, n_paths: int, seed: int, *,
                                 ctx: Optional["qmcg.Context"] = None,
                                 batch_fn: Optional[Callable[[Sequence], np.ndarray]] = None,
                                 allow_put: bool = False, group=None) -> np.ndarray:
    """Config 4 over the ranks of `group`: rank r prices contracts contract_range(C, world, r)
    over all paths (its own copy of the shared permutation tables), then the (price, std_error)
    rows are all-gathered. Every contract is independent, so the result equals the single-GPU
    batch bit for bit. batch_fn(specs) -> (len, 2) replaces the GPU call (CPU tests)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    C = len(specs)
    per = -(-C // world)
    b, e = contract_range(C, world, rank)
    local = np.zeros((per, 2), dtype=np.float64)
    if e > b:
        if batch_fn is not None:
            local[: e - b] = batch_fn(specs[b:e])
        else:
            if ctx is None:
                raise ValueError("price_american_batch_sharded: pass ctx or batch_fn")
            res = ctx.price_american_batch(list(specs[b:e]), m, n_paths, seed, allow_put=allow_put)
            local[: e - b] = [(r.price, r.std_error) for r in res]
    rows = _all_gather_rows(local, group)
    out = np.zeros((C, 2), dtype=np.float64)
    for r in range(world):
        rb, re_ = contract_range(C, world, r)
        out[rb:re_] = rows[r][: re_ - rb]
    return out


def rank_columns(n_paths: int, world: int, rank: int) -> Tuple[int, int]:
    """The contiguous path (column) range of `rank`: the union of its pairwise-tree nodes."""
    depth = tree_depth(n_paths, world)
    mine = rank_nodes(depth, world, rank)
    if not mine:
        return 0, 0
    b, _ = qmcg.tree_node_range(n_paths, depth, mine[0])
    _, e = qmcg.tree_node_range(n_paths, depth, mine[-1])
    return b, e


def warm_tables_sharded(ctx: Optional["qmcg.Context"], n_paths: int, seed: int, dims: int, *, group=None,
                        build_fn: Optional[Callable] = None, import_fn: Optional[Callable] = None,
                        device=None, tables_per_chunk: Optional[int] = None) -> None:
    """Cold table build over the ranks of `group`: the permutation table of dim d
    is built (full n) by rank d mod G only, then an all-to-all sends each rank its column slice of
    every table, which it installs in its context -- G times less K1 work than every rank
    building every table (the loop replaced is proj/src/quasi_rng.cpp:91-93). The dims go in
    chunks of G * tables_per_chunk (each rank builds tables_per_chunk full tables per chunk, ~1 GiB
    of scratch by default), so config 5 (2^28 paths x 365 dates, a 1 GiB table per dim) needs a
    few GiB per rank besides its slice. Afterwards price_american_sharded on the same
    (n_paths, seed) is warm. build_fn(k_dims, dim_begin, stride, buf) /
    import_fn(b, e, row_begin, rows, dims) replace the GPU calls (tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    backend = dist.get_backend(group) if dist.is_initialized() else "nccl"
    comm = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    if device is None:  # where K1 writes: the GPU when the context builds, else the collective's device
        device = torch.device("cuda", torch.cuda.current_device()) if build_fn is None else comm
    if tables_per_chunk is None:
        tables_per_chunk = max(1, min(32, (1 << 28) // max(1, n_paths)))
    cols = [rank_columns(n_paths, world, r) for r in range(world)]
    b_me, e_me = cols[rank]
    w_me = e_me - b_me
    span = world * tables_per_chunk
    buf = torch.empty((tables_per_chunk, n_paths), dtype=torch.int32, device=device)  # uint32 bit patterns
    for c0 in range(0, dims, span):
        c1 = min(dims, c0 + span)
        # dims of this chunk built by rank r: c0 + ((r - c0) mod G) + t G, t = 0, 1, ...
        first = [c0 + (r - c0) % world for r in range(world)]
        k_of = [len(range(first[r], c1, world)) for r in range(world)]
        k = k_of[rank]
        if k:
            if build_fn is not None:
                build_fn(k, first[rank], world, buf)
            else:
                # the context writes `buf` on its own (non-blocking) stream: torch's stream must be
                # idle first (the allocator may hand out memory still in use by queued torch work);
                # the call returns after its stream has synchronised, so later torch work sees the rows
                _sync_torch_stream(buf)
                ctx.build_tables(n_paths, seed, first[rank], world, k, buf.data_ptr(), n_paths)
        if world == 1:
            rows = buf[:k]
        else:
            send = (torch.cat([buf[:k, b:e].reshape(-1) for (b, e) in cols]) if k else
                    torch.empty(0, dtype=torch.int32, device=device)).to(comm)
            recv = torch.empty(sum(k_of) * w_me, dtype=torch.int32, device=comm)
            dist.all_to_all_single(recv, send, output_split_sizes=[kk * w_me for kk in k_of],
                                   input_split_sizes=[k * (e - b) for (b, e) in cols], group=group)
            rows = torch.empty((c1 - c0, w_me), dtype=torch.int32, device=comm)
            for r, piece in enumerate(recv.split([kk * w_me for kk in k_of])):
                if k_of[r]:
                    rows[first[r] - c0::world] = piece.view(k_of[r], w_me)
        if import_fn is not None:
            import_fn(b_me, e_me, c0, rows, dims)
        else:
            if rows.device.type != "cuda":
                rows = rows.cuda()
            rows = rows.contiguous()
            # the all-to-all and the slice copies above are queued on torch's stream; the context
            # copies from `rows` on its own non-blocking stream, so wait for them to finish
            _sync_torch_stream(rows)
            ctx.import_rows(n_paths, seed, b_me, e_me, dims, c0, c1 - c0, rows.data_ptr(), rows.stride(0))


def _sync_torch_stream(t) -> None:
    """Block until torch's current stream on t's device has drained (orders torch-side work
    before a qmcg context call that runs on the context's own stream)."""
    import torch
    if t.device.type == "cuda":
        torch.cuda.current_stream(t.device).synchronize()
