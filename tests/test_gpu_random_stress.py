"""Randomized differential test of the whole operator against the oracles.

Seeded random schemas (1-2 key columns of several integer widths, dense and
sparse key domains, random aggregate lists over int and float columns),
row counts, budgets, page capacities, input placement (device / pinned
host) and window knobs -- so that the chunk loop's host decisions (assumed
sort mask, speculative flush row, partial-key sorts, inverted head marking),
both run tiers and every wide-merge path (dense windows with direct or
streamed output, radix windows, tile merge) meet inputs nobody wrote by
hand.  Output equals the numpy oracle; fill cycles, runs and spilled rows
equal the C restatement of the reference (oracle/rsw_oracle.c).
"""

import os

import numpy as np
import pytest

import oracle
from conftest import assert_slots_equal

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2010_00152_b200 as isa  # noqa: E402
from paper_2010_00152_b200.core import AggregateKind, AggregateSpec, ColumnSpec, Schema  # noqa: E402


def _keys(rng, n, kind):
    if kind == "dense64":
        return [rng.integers(-5000, 5000 + int(rng.integers(1, 200_000)), n).astype(np.int64)]
    if kind == "sparse64":
        base = rng.integers(-(1 << 62), 1 << 62, max(2, n // int(rng.integers(1, 20)))).astype(np.int64)
        return [base[rng.integers(0, len(base), n)]]
    if kind == "u32":
        return [rng.integers(0, int(rng.integers(2, 1 << 20)), n).astype(np.uint32)]
    if kind == "i16_u8":
        return [rng.integers(-300, 300, n).astype(np.int16), rng.integers(0, 7, n).astype(np.uint8)]
    if kind == "u64_u64":
        a = rng.integers(0, 1 << 63, max(2, n // 4)).astype(np.uint64)
        b = rng.integers(0, 1 << 63, max(2, n // 4)).astype(np.uint64)
        pick = rng.integers(0, len(a), n)
        return [a[pick], b[pick]]
    return [rng.integers(-(1 << 20), 1 << 20, n).astype(np.int32), rng.integers(0, 1 << 30, n).astype(np.int64)]


def _aggs(rng, float_ok):
    kinds = [AggregateKind.COUNT, AggregateKind.SUM, AggregateKind.MIN, AggregateKind.MAX, AggregateKind.AVG]
    aggs, cols = [], ["a", "b"] + (["f"] if float_ok else [])
    for i in range(int(rng.integers(0, 5))):
        k = kinds[int(rng.integers(0, len(kinds)))]
        col = None if k == AggregateKind.COUNT else cols[int(rng.integers(0, len(cols)))]
        aggs.append(AggregateSpec(f"g{i}", k, col))
    return aggs


@pytest.mark.parametrize("seed", range(int(os.environ.get("ISA_STRESS_SEEDS", "48"))))
def test_random_schema_rows_and_knobs(seed, monkeypatch):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 7, 300, 5000, 60_000, 400_000, 1_500_000]))
    kind = ["dense64", "sparse64", "u32", "i16_u8", "u64_u64", "i32_i64"][seed % 6]
    keys = _keys(rng, n, kind)
    float_ok = bool(rng.integers(0, 2))
    aggs = _aggs(rng, float_ok)
    sch = Schema([ColumnSpec(f"k{j}") for j in range(len(keys))], aggs)
    vals = {"a": rng.integers(-(1 << 33), 1 << 33, n).astype(np.int64),
            "b": rng.integers(-1000, 1000, n).astype(np.int32),
            "f": rng.normal(0, 100, n)}
    vals = {c: v for c, v in vals.items() if any(a.column == c for a in aggs)}
    page = int(rng.choice([1, 3, 100]))
    memory = int(rng.choice([2 * page, 2 * page + 1, 64, 1000, 1 << 14]))
    memory = max(memory, 2 * page)
    if memory < 64 and n > 20_000:
        # a budget of a few groups flushes every few rows: hundreds of thousands of fill cycles through the
        # chunk loop take minutes (the reference takes longer); keep those cases small
        n = 20_000
        keys = [k[:n] for k in keys]
        vals = {c: v[:n] for c, v in vals.items()}
    on_host = bool(rng.integers(0, 2))
    kw = {}
    if rng.integers(0, 3) == 0:
        kw.update(merge_window_rows=int(rng.integers(200, 5000)), chunk_rows_max=int(rng.integers(3000, 50_000)))
    if rng.integers(0, 3) == 0:
        monkeypatch.setenv("ISA_DENSE_D", str(int(rng.choice([64, 1024, 65536]))))
    if rng.integers(0, 4) == 0:
        kw.update(run_tier=str(rng.choice(["host", "hbm"])))
    slots = oracle.make_states(sch, vals, n)
    want_keys, want_slots = oracle.reference_aggregate(keys, slots, oracle.slot_ops(sch))
    _, _, led, cycles = oracle.rsw_sortagg(keys, slots, oracle.slot_ops(sch), memory, page)
    op = isa.SortAggregate(sch, isa.SortAggConfig(memory_budget=memory, page_capacity=page, ovc_enabled=False, **kw))

    def put(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.pin_memory() if on_host else t.cuda()

    for it in range(2):   # the second execute reuses every pool of the handle (the ledger accumulates)
        res = op.execute_columns([put(k) for k in keys], {c: put(v) for c, v in vals.items()})
        got_keys = [k.cpu().numpy() for k in res.keys]
        assert len(got_keys[0]) == len(want_keys[0])
        for g, w in zip(got_keys, want_keys):
            assert g.dtype == w.dtype and np.array_equal(g, w)
        for s, (g, w) in enumerate(zip(res.states, want_slots)):
            assert_slots_equal(g.cpu().numpy(), w, rel=1e-9, what=f"slot {s}")
        assert op.cycles == [c for c in cycles if c > 0]
        assert op.ledger.rows_spilled == (it + 1) * led["rows_spilled"] and op.runs_after_generation == led["runs"]
        op.ledger.check_invariants()
