"""Device primitives of the multi-GPU path (sampling, partition kernel) and the
distributed entry point on a single-rank NCCL group (the only GPU count this
environment grants; the 2-rank exchange logic is covered over gloo)."""

import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2010_00152_b200 as isa  # noqa: E402
from paper_2010_00152_b200 import parallel, workloads  # noqa: E402


def _op(w):
    return isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100))


@pytest.mark.parametrize("c", [1, 3, 4, 5])
def test_sample_keys_matches_normalization(c):
    w = workloads.make(c, rows=100_000, device="cpu", **({"domain": 1 << 16} if c in (3, 5) else {}))
    op = _op(w)
    keys = [k.cuda() for k in w.keys]
    hi, lo = parallel.native_sampler(op, keys, 1000)
    stride = max(1, w.rows // 1000)
    want_hi, want_lo = oracle.normalize_keys([k.numpy() for k in w.keys])
    assert np.array_equal(lo.cpu().numpy().view(np.uint64), want_lo[::stride])
    assert np.array_equal(hi.cpu().numpy().view(np.uint64), want_hi[::stride])


@pytest.mark.parametrize("c,G", [(5, 4), (3, 8), (4, 2), (1, 3), (2, 8)])
def test_partition_kernel_is_stable_range_split(c, G):
    w = workloads.make(c, rows=200_000, device="cpu", **({"domain": 1 << 18} if c in (3, 5) else {}))
    op = _op(w)
    keys = [k.cuda() for k in w.keys]
    names = sorted(w.values)
    vals = [w.values[n].cuda() for n in names]
    s_hi, s_lo = parallel.native_sampler(op, keys, 4096)
    sp_hi, sp_lo = parallel.choose_splitters(s_hi, s_lo, G)
    pk, pv, counts = parallel.native_partitioner(op, keys, vals, sp_hi, sp_lo)
    assert sum(counts) == w.rows and len(counts) == G
    hi, lo = oracle.normalize_keys([k.numpy() for k in w.keys])
    shi, slo = sp_hi.cpu().numpy().view(np.uint64), sp_lo.cpu().numpy().view(np.uint64)
    dest = np.zeros(w.rows, dtype=np.int64)
    for i in range(len(slo)):
        dest += (hi > shi[i]) | ((hi == shi[i]) & (lo >= slo[i]))
    order = np.argsort(dest, kind="stable")
    assert counts == np.bincount(dest, minlength=G).tolist()
    for got, k in zip(pk, w.keys):
        assert np.array_equal(got.cpu().numpy(), k.numpy()[order])
    for got, n in zip(pv, names):
        assert np.array_equal(got.cpu().numpy(), w.values[n].numpy()[order])


@pytest.mark.parametrize("mode", ["partition", "preaggregate"])
def test_distributed_execute_single_rank_nccl(mode):
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        w = workloads.make(5, rows=500_000, device="cpu", domain=1 << 17)
        op = _op(w)
        res = parallel.distributed_execute(op, [k.cuda() for k in w.keys], {n: v.cuda() for n, v in w.values.items()},
                                           mode=mode)
        slots = oracle.make_states(w.schema, {n: v.numpy() for n, v in w.values.items()}, w.rows)
        want_k, want_s = oracle.reference_aggregate([k.numpy() for k in w.keys], slots, oracle.slot_ops(w.schema))
        assert np.array_equal(res.keys[0].cpu().numpy(), want_k[0])
        for g, e in zip(res.states, want_s):
            assert np.array_equal(g.cpu().numpy(), e)
    finally:
        dist.destroy_process_group()


def test_fused_scatter_to_simulated_peers():
    """isa_partition_counts + isa_scatter_to_peers with three receive
    buffers on this GPU standing in for peers: as rank 1 of 3, every
    destination's block holds exactly the rows isa_partition assigns it, in
    the same (stable) order, at the offset after rank 0's block."""
    from paper_2010_00152_b200 import parallel, workloads
    from paper_2010_00152_b200.sortagg import ctypes_stream
    w = workloads.config5(rows=500_000, device="cuda", domain=1 << 24)
    op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=1 << 16, page_capacity=100))
    keys, vals = list(w.keys), [w.values["v"]]
    sh, sl = parallel.native_sampler(op, keys, 4096)
    split_hi, split_lo = parallel.choose_splitters(sh, sl, 3)
    pk, pv, counts = parallel.native_partitioner(op, keys, vals, split_hi, split_lo)
    h = parallel._key_handle(op, keys, vals)
    st = torch.cuda.current_stream()
    got = h.partition_counts(w.rows, [k.data_ptr() for k in keys], split_lo.contiguous().data_ptr(),
                             split_hi.contiguous().data_ptr(), 2, ctypes_stream(st))
    assert got == counts
    rank0 = [7, 11, 13]   # rows rank 0 sends to each destination
    matrix = [rank0, counts, [0, 0, 0]]
    offs = parallel.p2p_offsets(matrix, 1)
    recv = [[torch.full((rank0[d] + counts[d] + 5,), -1, dtype=t.dtype, device="cuda") for t in keys + vals]
            for d in range(3)]
    table = [t.data_ptr() for d in range(3) for t in recv[d]]
    h.scatter_to_peers(w.rows, [k.data_ptr() for k in keys], [v.data_ptr() for v in vals], table, offs,
                       ctypes_stream(st))
    torch.cuda.synchronize()
    start = 0
    for d in range(3):
        for c, src in enumerate(pk + pv):
            block = recv[d][c][offs[d]: offs[d] + counts[d]]
            assert torch.equal(block, src[start: start + counts[d]])
            assert bool((recv[d][c][: offs[d]] == -1).all()) and bool((recv[d][c][offs[d] + counts[d]:] == -1).all())
        start += counts[d]
    assert sum(counts) == w.rows


def test_ipc_handle_carries_the_offset_in_its_allocation():
    """Receive columns come from torch's caching allocator (pointers inside
    larger segments): the IPC handle names the segment, plus the offset."""
    import struct
    from paper_2010_00152_b200 import _native
    buf = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    a, b = buf[4096:], buf[65536:]
    ha, hb = _native.ipc_handle(a.data_ptr()), _native.ipc_handle(b.data_ptr())
    assert len(ha) == 72 and ha[:64] == hb[:64]
    off_a, off_b = struct.unpack("<Q", ha[64:])[0], struct.unpack("<Q", hb[64:])[0]
    assert off_b - off_a == 65536 - 4096


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,rows,memory", [(5, 2_000_000, 1 << 14), (3, 1_000_000, 1 << 14), (1, 600_000, 4096)])
def test_execute_multi_two_ranges_on_one_gpu(cfg, rows, memory):
    """isa_execute_multi with two handles standing in for two GPUs (both on
    cuda:0: the same splitter, partition and peer-store kernels, plain device
    pointers): two shards in, two key ranges out; their concatenation is the
    single-operator result and the ranges do not overlap."""
    import numpy as np
    import oracle
    import paper_2010_00152_b200 as isa
    from paper_2010_00152_b200 import _native, workloads
    kw = {"domain": 1 << 20} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kw)
    keys_np = [k.numpy() for k in w.keys]
    slots = oracle.make_states(w.schema, {k: v.numpy() for k, v in w.values.items()}, w.rows)
    want_keys, want_slots = oracle.reference_aggregate(keys_np, slots, oracle.slot_ops(w.schema))
    cut = (rows * 2) // 5   # unequal shards
    ops, prepared = [], []
    for a, b in ((0, cut), (cut, rows)):
        op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=memory, page_capacity=100, ovc_enabled=False))
        ops.append(op)
        prepared.append(op._prepare([k[a:b].cuda() for k in w.keys], {n: v[a:b].cuda() for n, v in w.values.items()},
                                    False, None))
    # two native handles, one per "device"
    assert prepared[0][0] is not prepared[1][0]
    counts = _native.execute_multi([p[0] for p in prepared], [p[1] for p in prepared],
                                   [[k.data_ptr() for k in p[2]] for p in prepared],
                                   [[v.data_ptr() for v in p[3]] for p in prepared])
    outs = [op._collect(p[0], p[1], ng, p[2], p[4], False, p[6]) for op, p, ng in zip(ops, prepared, counts)]
    assert sum(counts) == len(want_keys[0]) and min(counts) > 0
    # roughly equal ranges from the sampled splitters
    assert max(counts) < 0.75 * sum(counts)
    for j, wk in enumerate(want_keys):
        got = np.concatenate([o.keys[j].cpu().numpy() for o in outs])
        assert np.array_equal(got, wk)
    for s, ws in enumerate(want_slots):
        got = np.concatenate([o.states[s].cpu().numpy() for o in outs])
        if got.dtype.kind == "f":
            assert np.allclose(got, ws, rtol=1e-5 if cfg == 3 else 1e-9, atol=1e-9)
        else:
            assert np.array_equal(got, ws)
