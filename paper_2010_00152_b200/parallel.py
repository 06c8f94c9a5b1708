"""Multi-GPU range-partitioned grouping (one process per GPU, NCCL).

Groups with different keys are independent and the output must be globally
sorted, so a key-range partition makes the concatenation of every rank's
local result, in rank order, the answer (the paper suggests
partitioning for parallel computation).  Steps:

1. sample normalized keys of the local shard (isa_sample_keys),
2. all-gather the samples, sort them and cut G-1 splitters at equal-count
   quantiles (a key equal to a splitter goes to the higher range, so every
   group lands on exactly one rank),
3. stable partition of the local rows by destination (isa_partition: one
   8-bit radix pass on the destination + column gathers),
4. exchange counts, then every column, with all_to_all_single over NCCL
   (NVLink / NVSwitch) — variable-count all-to-all; or, with
   ``exchange="p2p"`` (env ISA_EXCHANGE), the fused form: one kernel per rank
   gathers its rows in destination order and stores them straight into the
   destination ranks' receive columns through CUDA-IPC peer pointers
   (isa_partition_counts + isa_scatter_to_peers), so the transfer happens
   inside the partition kernel.  NCCL stays the default until the fused
   path has run on a multi-GPU box (the single-GPU test drives the same
   kernel with simulated peers),
5. run the local SortAggregate on the received rows.

``mode="preaggregate"`` runs the local operator first and exchanges the
(sorted, unique) groups instead of raw rows, combining them with
merge_states on the receiver — the right choice when the output is much
smaller than the input (configs 1-2, or skewed keys: heavy hitters collapse
before the shuffle).

The host logic takes its device primitives as parameters so the CPU tests
can drive it over gloo with the oracle standing in for the CUDA kernels.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .core import InvalidInputError


def _group_size(group):
    return dist.get_world_size(group)


def _ordered(hi, lo):
    """Sort (hi, lo) uint64 pairs (stored as int64 bit patterns) in unsigned
    lexicographic order; returns (hi, lo) sorted."""
    bias = torch.tensor(-(1 << 63), dtype=torch.int64, device=lo.device)
    lo_s = lo ^ bias  # unsigned order as signed order
    hi_s = hi ^ bias
    idx = torch.argsort(lo_s, stable=True)
    idx = idx[torch.argsort(hi_s[idx], stable=True)]
    return hi[idx], lo[idx]


def choose_splitters(samples_hi, samples_lo, world):
    """G-1 splitters at equal-count quantiles of the gathered samples."""
    n = samples_lo.numel()
    if world <= 1 or n == 0:
        e = samples_lo.new_empty(0)
        return e, e
    hi, lo = _ordered(samples_hi, samples_lo)
    pos = torch.tensor([min(n - 1, (n * (r + 1)) // world) for r in range(world - 1)], device=lo.device)
    return hi[pos], lo[pos]


def gather_samples(hi, lo, group=None):
    """All-gather variable-length sample arrays (int64 bit patterns)."""
    world = _group_size(group)
    cnt = torch.tensor([lo.numel()], dtype=torch.int64, device=lo.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    m = max(int(c.item()) for c in counts)
    pad_hi = torch.zeros(m, dtype=torch.int64, device=lo.device)
    pad_lo = torch.zeros(m, dtype=torch.int64, device=lo.device)
    pad_hi[: lo.numel()] = hi
    pad_lo[: lo.numel()] = lo
    all_hi = [torch.empty_like(pad_hi) for _ in range(world)]
    all_lo = [torch.empty_like(pad_lo) for _ in range(world)]
    dist.all_gather(all_hi, pad_hi, group=group)
    dist.all_gather(all_lo, pad_lo, group=group)
    hs = torch.cat([h[: int(c.item())] for h, c in zip(all_hi, counts)])
    ls = torch.cat([x[: int(c.item())] for x, c in zip(all_lo, counts)])
    return hs, ls


def exchange_columns(columns, send_counts, group=None):
    """Variable-count all-to-all of every column (rows already grouped by
    destination).  Returns (received columns, recv_counts)."""
    world = _group_size(group)
    dev = columns[0].device if columns else torch.device("cpu")
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.tolist()]
    out = []
    for col in columns:
        # NCCL moves bytes: exchange unsigned/narrow dtypes through a byte view
        raw = col.contiguous().view(torch.uint8).view(-1, col.element_size())
        dst = torch.empty((sum(recv_counts), col.element_size()), dtype=torch.uint8, device=dev)
        dist.all_to_all_single(dst, raw, recv_counts, list(send_counts), group=group)
        out.append(dst.view(-1).view(col.dtype))
    return out, recv_counts


def p2p_offsets(count_matrix, me):
    """Row offset of rank ``me``'s block inside every destination's receive
    columns: blocks are laid out in source-rank order, so destination d
    receives rank r's rows at sum(count_matrix[q][d] for q < r)."""
    world = len(count_matrix)
    return [sum(count_matrix[q][d] for q in range(me)) for d in range(world)]


def exchange_p2p(op, keys, cols, split_hi, split_lo, group=None):
    """Fused range exchange over NVLink / NVSwitch peer memory: every rank
    allocates its receive columns, the CUDA IPC handles are all-gathered,
    and one kernel per rank gathers its rows in destination order and stores
    them straight into the destinations' receive columns
    (isa_partition_counts + isa_scatter_to_peers).  Returns (received key
    columns, received value columns)."""
    from .sortagg import ctypes_stream
    from . import _native
    world = _group_size(group)
    me = dist.get_rank(group)
    dev = keys[0].device
    n = int(keys[0].shape[0])
    h = _key_handle(op, keys, cols)
    st = torch.cuda.current_stream(dev)
    counts = h.partition_counts(n, [k.data_ptr() for k in keys], split_lo.contiguous().data_ptr(),
                                split_hi.contiguous().data_ptr(), world - 1, ctypes_stream(st))
    mine = torch.tensor(counts, dtype=torch.int64, device=dev)
    allc = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    matrix = [[int(x) for x in c.tolist()] for c in allc]
    recv_n = sum(matrix[q][me] for q in range(world))
    recv = [torch.empty(max(recv_n, 1), dtype=t.dtype, device=dev) for t in list(keys) + list(cols)]
    handles = [_native.ipc_handle(t.data_ptr()) for t in recv]
    every = [None] * world
    dist.all_gather_object(every, handles, group=group)
    opened, table = [], []
    try:
        for d in range(world):
            for c, hd in enumerate(every[d]):
                if d == me:
                    table.append(recv[c].data_ptr())
                else:
                    base, p = _native.ipc_open(hd)
                    opened.append(base)
                    table.append(p)
        dist.barrier(group=group)   # every receive column exists before anyone stores into it
        h.scatter_to_peers(n, [k.data_ptr() for k in keys], [c.data_ptr() for c in cols], table,
                           p2p_offsets(matrix, me), ctypes_stream(st))
        dist.barrier(group=group)   # every rank's stores are done before anyone reads
    finally:
        for base in opened:
            _native.ipc_close(base)
    recv = [t[:recv_n] for t in recv]
    return recv[: len(keys)], recv[len(keys):]


def native_sampler(op, keys, per_rank):
    """Normalized keys of ~per_rank evenly spaced local rows (CUDA kernel)."""
    from .sortagg import ctypes_stream
    n = int(keys[0].shape[0])
    if n == 0:
        e = torch.empty(0, dtype=torch.int64, device=keys[0].device)
        return e, e
    stride = max(1, n // max(1, per_rank))
    ns = (n + stride - 1) // stride
    lo = torch.empty(ns, dtype=torch.int64, device=keys[0].device)
    hi = torch.empty(ns, dtype=torch.int64, device=keys[0].device)
    h = _key_handle(op, keys)
    st = torch.cuda.current_stream(keys[0].device)
    h.sample_keys(n, [k.data_ptr() for k in keys], stride, lo.data_ptr(), hi.data_ptr(), ctypes_stream(st))
    return hi, lo


def _key_handle(op, keys, value_cols=()):
    """A native handle whose schema matches these key/value dtypes (no slots)."""
    from .sortagg import _isa_dtype
    return op._handle([_isa_dtype(k) for k in keys], [_isa_dtype(v) for v in value_cols], ())


def native_partitioner(op, keys, values, split_hi, split_lo):
    """Stable partition of the rows by destination (CUDA kernel)."""
    from .sortagg import ctypes_stream
    n = int(keys[0].shape[0])
    world = split_lo.numel() + 1
    if n == 0:
        return [k.clone() for k in keys], [v.clone() for v in values], [0] * world
    h = _key_handle(op, keys, values)
    out_k = [torch.empty_like(k) for k in keys]
    out_v = [torch.empty_like(v) for v in values]
    st = torch.cuda.current_stream(keys[0].device)
    counts = h.partition(n, [k.data_ptr() for k in keys], [v.data_ptr() for v in values],
                         split_lo.contiguous().data_ptr(), split_hi.contiguous().data_ptr(), world - 1,
                         [k.data_ptr() for k in out_k], [v.data_ptr() for v in out_v], ctypes_stream(st))
    return out_k, out_v, counts


def distributed_execute(op, keys, values=None, *, mode="partition", group=None, samples_per_rank=1 << 16,
                        sampler=None, partitioner=None, local_execute=None, merge_execute=None, exchange=None):
    """Range-partitioned SortAggregate over every rank of ``group``.

    Returns this rank's slice of the globally sorted result (a
    ColumnarResult: keys + state columns); concatenating the slices in rank
    order gives the single-GPU answer.
    """
    if mode not in ("partition", "preaggregate"):
        raise InvalidInputError(f"unknown distributed mode {mode!r}")
    world = _group_size(group)
    keys = list(keys)
    sampler = sampler or (lambda ks: native_sampler(op, ks, samples_per_rank))
    partitioner = partitioner or (lambda ks, vs, sh, sl: native_partitioner(op, ks, vs, sh, sl))
    local_execute = local_execute or (lambda ks, vs: op.execute_columns(ks, vs))
    merge_execute = merge_execute or (lambda ks, ss: op.execute_columns(ks, ss, states=True))

    if mode == "preaggregate":
        local = local_execute(keys, values)
        keys, cols = list(local.keys), list(local.states)
    else:
        names = sorted(values) if isinstance(values, dict) else None
        cols = [values[n] for n in names] if names is not None else list(values or [])
    if world == 1:
        if mode == "preaggregate":
            return local
        return local_execute(keys, dict(zip(names, cols)) if names is not None else cols)

    s_hi, s_lo = sampler(keys)
    all_hi, all_lo = gather_samples(s_hi, s_lo, group)
    split_hi, split_lo = choose_splitters(all_hi, all_lo, world)
    exchange = exchange or os.environ.get("ISA_EXCHANGE", "nccl")
    if exchange == "p2p":
        # fused: the partition kernel stores into the peers' receive columns
        rk, rc = exchange_p2p(op, keys, cols, split_hi, split_lo, group)
    elif exchange == "nccl":
        pk, pc, counts = partitioner(keys, cols, split_hi, split_lo)
        nk = len(pk)
        recv, _ = exchange_columns(pk + pc, counts, group)
        del pk, pc   # the partitioned copy is not needed any more: its memory goes to the local operator's runs
        rk, rc = recv[:nk], recv[nk:]
    else:
        raise InvalidInputError(f"unknown exchange {exchange!r}")
    if mode == "preaggregate":
        return merge_execute(rk, rc)
    return local_execute(rk, dict(zip(names, rc)) if names is not None else rc)
