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


def _cfg(w, **kw):
    return isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100, **kw)


def _strictly_increasing_u64(x):
    # int64 columns are compared in their signed order
    return bool((x[1:] > x[:-1]).all())


@pytest.mark.parametrize("rows", [1_000_000_000])
def test_config3_full_scale(rows):
    w = workloads.config3(rows=rows, device="cuda")
    op = isa.SortAggregate(w.schema, _cfg(w))
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
    # fp32 inputs accumulated in fp64: rel 1e-5 of the absolute mass per group (order-dependent sums)
    absmass = torch.zeros_like(want_fsum).index_add_(0, inv, w.values["vf"].double().abs())
    assert bool(((fsum - want_fsum).abs() <= 1e-5 * absmass + 1e-12).all())
    assert op.runs_after_generation > 1 and op.ledger.rows_spilled == op.ledger.rows_read_back
    op.ledger.check_invariants()


def _pair_checksum(hi, lo):
    """order-independent checksum of (hi, lo) uint64 pairs (wrapping int64 sum of a mix)"""
    x = hi.view(torch.int64) * -7046029254386353131 + lo.view(torch.int64)
    x = x ^ ((x >> 31) & ((1 << 33) - 1))
    x = x * -4658895280553007687
    return int(x.sum())


def test_config4_full_scale_distinct():
    w = workloads.config4(device="cuda")
    op = isa.SortAggregate(w.schema, _cfg(w))
    res = op.execute_columns(w.keys, {})
    hi, lo = res.keys
    assert res.n_groups == w.rows // 4
    # strictly increasing (hi, lo) in unsigned order
    bias = -(1 << 63)
    hs, ls = hi.view(torch.int64) ^ bias, lo.view(torch.int64) ^ bias
    inc = (hs[1:] > hs[:-1]) | ((hs[1:] == hs[:-1]) & (ls[1:] > ls[:-1]))
    assert bool(inc.all())
    # the distinct set equals the generator's pairs: each input pair appears 4x
    assert (_pair_checksum(hi, lo) * 4 - _pair_checksum(w.keys[0], w.keys[1])) % (1 << 64) == 0


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
