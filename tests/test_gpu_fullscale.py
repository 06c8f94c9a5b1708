"""Parity at BASELINE.json's full sizes through independent device
computations and size-independent properties (the CPU oracle cannot hold
1e9 rows): exact key sets and counts against torch.unique, exact integer
sums / min / max against scatter reductions, float sums within the stated
tolerance, DISTINCT sets through an order-independent checksum of the
generator's pairs, strictly increasing output keys, and ledger invariants."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2010_00152_b200 as isa  # noqa: E402
from paper_2010_00152_b200 import workloads  # noqa: E402


@pytest.fixture(autouse=True)
def _free_device_memory():
    """Full-scale tests hold tens of GB: hand torch's cached blocks back to
    the driver so the library's own allocations fit."""
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    yield
    gc.collect()
    torch.cuda.empty_cache()


def _cfg(w, **kw):
    return isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100, **kw)


def _strictly_increasing_u64(x):
    # int64 columns are compared in their signed order
    return bool((x[1:] > x[:-1]).all())


@pytest.mark.parametrize("rows", [1_000_000_000])
def test_config3_full_scale(rows):
    w = workloads.config3(rows=rows, device="cuda")
    op = isa.SortAggregate(w.schema, _cfg(w, run_tier="host"))   # BASELINE: runs spill to host memory
    res = op.execute_columns(w.keys, w.values)
    key = w.keys[0]
    uk, inv, cnt = torch.unique(key, sorted=True, return_inverse=True, return_counts=True)
    assert res.n_groups == uk.numel()
    assert torch.equal(res.keys[0], uk)
    n, isum, fsum, imin, imax = res.states
    assert torch.equal(n, cnt.to(torch.int64))
    want_isum = torch.zeros_like(n).index_add_(0, inv, w.values["vi"])
    assert torch.equal(isum, want_isum)
    want_min = torch.full_like(n, 1 << 62).scatter_reduce_(0, inv, w.values["vi"], reduce="amin")
    want_max = torch.full_like(n, -(1 << 62)).scatter_reduce_(0, inv, w.values["vi"], reduce="amax")
    assert torch.equal(imin, want_min) and torch.equal(imax, want_max)
    want_fsum = torch.zeros(n.numel(), dtype=torch.float64, device="cuda").index_add_(0, inv, w.values["vf"].double())
    # float32 inputs, float64 accumulation in a different order: rel 1e-5 of
    # the value (BASELINE's fp32 bar) plus the float64 summation-order term
    # (1e-12 of the group's absolute mass; it only matters for sums that
    # cancel to ~0, where a relative bar on the value is meaningless)
    absmass = torch.zeros_like(want_fsum).index_add_(0, inv, w.values["vf"].double().abs())
    err = (fsum - want_fsum).abs()
    assert bool((err <= 1e-5 * want_fsum.abs() + 1e-12 * absmass).all())
    assert op.runs_after_generation > 1 and op.ledger.rows_spilled == op.ledger.rows_read_back
    op.ledger.check_invariants()


def test_config4_full_scale_distinct():
    """The 2^27 distinct pairs, compared column by column with the input's
    distinct pairs (two stable sorts give the lexicographic order)."""
    w = workloads.config4(device="cuda")
    op = isa.SortAggregate(w.schema, _cfg(w))
    res = op.execute_columns(w.keys, {})
    op.close()
    assert res.n_groups == w.rows // 4
    bias = -(1 << 63)   # x ^ 2^63 as int64: signed order == unsigned order
    a = w.keys[0].view(torch.int64) ^ bias
    b = w.keys[1].view(torch.int64) ^ bias
    del w
    i1 = torch.sort(b, stable=True).indices
    i2 = torch.sort(a[i1], stable=True).indices
    idx = i1[i2]
    del i1, i2
    sa, sb = a[idx], b[idx]
    del a, b, idx
    keep = torch.ones_like(sa, dtype=torch.bool)
    keep[1:] = (sa[1:] != sa[:-1]) | (sb[1:] != sb[:-1])
    ua, ub = sa[keep], sb[keep]
    assert torch.equal(res.keys[0].view(torch.int64) ^ bias, ua)
    assert torch.equal(res.keys[1].view(torch.int64) ^ bias, ub)


def test_config5_full_scale_4e9():
    """BASELINE config 5 at its full 4e9 rows on one GPU -- the only
    configuration whose row count passes 2^32: exact keys, counts and sums
    against torch.unique + index_add on 8 key-range slabs."""
    w = workloads.config5(device="cuda")
    assert w.rows == 4_000_000_000
    op = isa.SortAggregate(w.schema, _cfg(w))
    res = op.execute_columns(w.keys, w.values)
    assert op.runs_after_generation > 200
    assert op.ledger.rows_spilled == op.ledger.rows_read_back
    op.ledger.check_invariants()
    op.close()
    torch.cuda.empty_cache()
    out_k, (out_n, out_s) = res.keys[0], res.states
    assert bool((out_k[1:] > out_k[:-1]).all())
    assert int(out_n.sum()) == w.rows
    key, val = w.keys[0], w.values["v"]
    assert int(out_s.sum()) == int(val.sum())
    edges = [(1 << 30) * i // 8 for i in range(9)]
    for lo, hi in zip(edges[:-1], edges[1:]):
        mask = (key >= lo) & (key < hi)
        k, v = key[mask], val[mask]
        del mask
        uk, inv, cnt = torch.unique(k, sorted=True, return_inverse=True, return_counts=True)
        a = int(torch.searchsorted(out_k, torch.tensor([lo], device="cuda")))
        b = int(torch.searchsorted(out_k, torch.tensor([hi], device="cuda")))
        assert torch.equal(out_k[a:b], uk), (lo, hi)
        assert torch.equal(out_n[a:b], cnt.to(torch.int64)), (lo, hi)
        assert torch.equal(out_s[a:b], torch.zeros_like(uk).index_add_(0, inv, v)), (lo, hi)
        del k, v, uk, inv, cnt


def test_run_tiers_agree_at_scale():
    """auto (HBM, bit-packed), host (pinned, bit-packed) and hbm (raw) run
    tiers give identical results and identical run ledgers."""
    w = workloads.config5(rows=300_000_000, device="cuda")
    outs = []
    for tier in ("auto", "host", "hbm"):
        op = isa.SortAggregate(w.schema, _cfg(w, run_tier=tier))
        r = op.execute_columns(w.keys, w.values)
        outs.append((r, op.run_rows, op.cycles, op.device_ledger))
        op.close()
    (r0, rr0, c0, d0) = outs[0]
    assert d0["bytes_d2h"] == 0 and d0["bytes_h2d"] == 0   # auto: runs stayed in HBM
    for r, rr, c, d in outs[1:]:
        assert rr == rr0 and c == c0
        for a, b in zip(r0.keys + r0.states, r.keys + r.states):
            assert torch.equal(a, b)
    assert outs[1][3]["bytes_d2h"] > 0


def test_config5_one_gpu_shard():
    w = workloads.config5(rows=1_000_000_000, device="cuda")
    op = isa.SortAggregate(w.schema, _cfg(w))
    res = op.execute_columns(w.keys, w.values)
    uk, inv, cnt = torch.unique(w.keys[0], sorted=True, return_inverse=True, return_counts=True)
    assert torch.equal(res.keys[0], uk)
    assert torch.equal(res.states[0], cnt.to(torch.int64))
    assert torch.equal(res.states[1], torch.zeros_like(res.states[1]).index_add_(0, inv, w.values["v"]))


def test_config3_host_input_matches_device_input():
    """End-to-end path (pinned host columns streamed in windows) returns the
    same result as the device-resident path."""
    w = workloads.config3(rows=200_000_000, device="cuda")
    op = isa.SortAggregate(w.schema, _cfg(w))
    dev = op.execute_columns(w.keys, w.values)
    host = op.execute_columns([k.cpu().pin_memory() for k in w.keys],
                              {n: v.cpu().pin_memory() for n, v in w.values.items()})
    for a, b in zip(dev.keys, host.keys):
        assert torch.equal(a.cpu(), b)
    for i, (a, b) in enumerate(zip(dev.states, host.states)):
        if a.dtype.is_floating_point:
            np.testing.assert_allclose(b.numpy(), a.cpu().numpy(), rtol=1e-9, atol=1e-9)
        else:
            assert torch.equal(a.cpu(), b), f"slot {i}"
