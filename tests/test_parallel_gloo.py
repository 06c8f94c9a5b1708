"""Multi-rank host logic of the range-partitioned path, world_size 2 over gloo (CPU).

The device primitives (key sampling, partition kernel, local operator) are
replaced by oracle-based stand-ins; everything else — sample gathering,
splitter choice, count/column all-to-all, ordering of the concatenated
result — is the product code of paper_2010_00152_b200/parallel.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2010_00152_b200 import parallel, workloads
from paper_2010_00152_b200.sortagg import ColumnarResult


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _i64(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64))


def _sampler(keys):
    hi, lo = oracle.normalize_keys([k.numpy() for k in keys])
    step = max(1, len(lo) // 257)
    return _i64(hi[::step]), _i64(lo[::step])


def _partitioner(keys, cols, split_hi, split_lo):
    hi, lo = oracle.normalize_keys([k.numpy() for k in keys])
    shi = split_hi.numpy().view(np.uint64)
    slo = split_lo.numpy().view(np.uint64)
    dest = np.zeros(len(lo), dtype=np.int64)
    for i in range(len(slo)):  # number of splitters <= key
        ge = (hi > shi[i]) | ((hi == shi[i]) & (lo >= slo[i]))
        dest += ge
    order = np.argsort(dest, kind="stable")
    counts = np.bincount(dest, minlength=len(slo) + 1).tolist()
    pk = [torch.from_numpy(k.numpy()[order]) for k in keys]
    pc = [torch.from_numpy(c.numpy()[order]) for c in cols]
    return pk, pc, counts


def _make_local(schema):
    def local_execute(keys, values):
        n = len(keys[0])
        vals = {k: v.numpy() for k, v in values.items()} if isinstance(values, dict) else {}
        slots = oracle.make_states(schema, vals, n)
        k, s = oracle.reference_aggregate([x.numpy() for x in keys], slots, oracle.slot_ops(schema))
        return ColumnarResult([torch.from_numpy(x) for x in k], [torch.from_numpy(x) for x in s])

    def merge_execute(keys, states):
        k, s = oracle.reference_aggregate([x.numpy() for x in keys], [x.numpy() for x in states],
                                          oracle.slot_ops(schema))
        return ColumnarResult([torch.from_numpy(x) for x in k], [torch.from_numpy(x) for x in s])
    return local_execute, merge_execute


def _worker(rank, world, port, cfg, rows, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kw = {"domain": 1 << 14} if cfg in (3, 5) else {}
        w = workloads.make(cfg, rows=rows, device="cpu", seed=1000 + 17 * rank + cfg, **kw)
        local_execute, merge_execute = _make_local(w.schema)
        res = parallel.distributed_execute(None, w.keys, w.values, mode=mode, sampler=_sampler,
                                           partitioner=_partitioner, local_execute=local_execute,
                                           merge_execute=merge_execute)
        import bench   # the bench's multi-rank result check, over the same process group
        chk = bench._check_result(torch, dist, res, w.schema, rows * world, world, rank, torch.device("cpu"))
        out = ([k.numpy() for k in res.keys], [s.numpy() for s in res.states],
               [k.numpy() for k in w.keys], {n: v.numpy() for n, v in w.values.items()}, chk)
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,rows,mode", [(5, 20_000, "partition"), (3, 20_000, "partition"),
                                           (1, 30_000, "preaggregate"), (2, 20_000, "preaggregate"),
                                           (4, 8_000, "partition"), (5, 20_000, "preaggregate")])
def test_two_rank_range_partition_matches_oracle(cfg, rows, mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, rows, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # concatenation in rank order == single-operator answer over the union
    keys = [np.concatenate([g[0][j] for g in gathered]) for j in range(len(gathered[0][0]))]
    states = [np.concatenate([g[1][s] for g in gathered]) for s in range(len(gathered[0][1]))]
    all_keys = [np.concatenate([g[2][j] for g in gathered]) for j in range(len(gathered[0][2]))]
    names = sorted(gathered[0][3])
    all_vals = {n: np.concatenate([g[3][n] for g in gathered]) for n in names}
    w = workloads.make(cfg, rows=8, device="cpu")
    slots = oracle.make_states(w.schema, all_vals, len(all_keys[0]))
    want_k, want_s = oracle.reference_aggregate(all_keys, slots, oracle.slot_ops(w.schema))
    for g, e in zip(keys, want_k):
        assert np.array_equal(g, e)
    for g, e in zip(states, want_s):
        if e.dtype.kind == "f":
            np.testing.assert_allclose(g, e, rtol=1e-9)
        else:
            assert np.array_equal(g, e)
    # bench.py's own check agrees on every rank
    for g in gathered:
        assert g[4]["keys_strictly_ascending"] and g[4]["rank_ranges_in_order"]
        if g[4]["count_sum"] is not None:
            assert g[4]["count_sum_equals_rows"], g[4]
    # both ranks received work (range partition actually split the keys)
    if cfg != 2:
        assert all(len(g[0][0]) > 0 for g in gathered)


def test_choose_splitters_unsigned_order():
    vals = np.array([0, 5, 2**63, 2**64 - 1, 7, 2**63 + 3], dtype=np.uint64)
    hi = torch.zeros(len(vals), dtype=torch.int64)
    lo = _i64(vals)
    sh, sl = parallel.choose_splitters(hi, lo, 3)
    got = sl.numpy().view(np.uint64).tolist()
    assert got == sorted(got)
    assert got[0] <= 2**63 <= got[1] or got == [7, 2**63 + 3] or got[0] >= 5


def test_p2p_offsets_layout():
    """Receive blocks are laid out in source-rank order."""
    from paper_2010_00152_b200.parallel import p2p_offsets
    m = [[3, 1, 0], [2, 2, 5], [0, 4, 1]]   # m[src][dst]
    assert p2p_offsets(m, 0) == [0, 0, 0]
    assert p2p_offsets(m, 1) == [3, 1, 0]
    assert p2p_offsets(m, 2) == [5, 3, 5]
