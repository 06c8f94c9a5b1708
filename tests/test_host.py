"""Host-side logic (CPU only): config validation, planner, estimator, schema,
generators, and the no-fallback rule.  Mirrors the reference's own unit tests
for these pieces (tests/test_sortagg.py planner/estimator, tests/test_core.py)."""

import math
import random

import numpy as np
import os

import pytest
import torch

import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads
from paper_2010_00152_b200.sortagg import OutputEstimator, plan_merge


def cfg(m, p, **kw):
    return isa.SortAggConfig(memory_budget=m, page_capacity=p, **kw)


@pytest.mark.parametrize("kw,msg", [
    (dict(memory_budget=10, page_capacity=0), "page capacity must be positive"),
    (dict(memory_budget=10, page_capacity=6), "memory budget must cover two pages"),
    (dict(memory_budget=10, page_capacity=5, run_generation_mode="bogus"), "unknown run generation mode"),
    (dict(memory_budget=10, page_capacity=5, merge_mode="bogus"), "unknown merge mode"),
    (dict(memory_budget=10, page_capacity=5, run_tier="disk"), "unknown run tier"),
])
def test_config_validation(kw, msg):
    with pytest.raises(isa.InvalidInputError, match=msg):
        isa.SortAggConfig(**kw)


def test_config_fanin():
    assert cfg(1000, 100).max_fanin == 10


# planner shapes (reference tests/test_sortagg.py:120-151)
def test_plan_single_wide_step_for_many_runs():
    plan = plan_merge([200_000] * 500, 8_000_000, cfg(100_000, 1000))
    assert plan.levels == 0 and [s.kind for s in plan.steps] == ["wide"]
    assert len(plan.steps[0].input_run_ids) == 500


def test_plan_one_level_then_wide():
    plan = plan_merge([2000] * 376, 32_000, cfg(1000, 166))
    assert plan.levels == 1 and plan.steps[-1].kind == "wide"
    trad = [s for s in plan.steps if s.kind == "traditional"]
    assert len(trad) == 63 and all(len(s.input_run_ids) <= 6 for s in trad)
    assert len(plan.steps[-1].input_run_ids) == 63


def test_plan_degenerate_final_and_single_run():
    assert [s.kind for s in plan_merge([100] * 4, 10_000, cfg(1000, 100)).steps] == ["traditional"]
    assert [s.kind for s in plan_merge([123], 10_000, cfg(1000, 100)).steps] == ["wide"]
    with pytest.raises(isa.InvalidInputError):
        plan_merge([], 10, cfg(1000, 100))


# estimator (reference tests/test_sortagg.py:384-412)
def test_estimator_steady_probe():
    est = OutputEstimator(1000)
    rng = random.Random(15)
    for _ in range(50_000):
        est.note_steady_probe(1000, rng.random() < 1000 / 4000)
    assert abs(est.estimate(10**9) - 4000) / 4000 < 0.05


def test_estimator_cycle_inversion():
    est = OutputEstimator(1000)
    o = 8000
    for _ in range(10):
        est.note_cycle(round(o * math.log(o / (o - 1000))))
    assert abs(est.estimate(10**9) - o) / o < 0.02


def test_estimator_floors():
    est = OutputEstimator(1000)
    for _ in range(200):
        est.note_steady_probe(1000, False)
    assert est.estimate(123_456) == 123_456
    est = OutputEstimator(1000)
    est.observe_distinct(777)
    assert est.estimate(10_000) == 777


# schema state algebra (reference core.py:162-221)
def test_schema_states():
    K = isa.AggregateKind
    sch = isa.Schema([isa.ColumnSpec("k")], [isa.AggregateSpec("n", K.COUNT), isa.AggregateSpec("s", K.SUM, "v"),
                                             isa.AggregateSpec("lo", K.MIN, "v"), isa.AggregateSpec("hi", K.MAX, "v"),
                                             isa.AggregateSpec("a", K.AVG, "v")])
    assert sch.state_slots == 6
    a = sch.make_state((None, 4, 4, 4, 4))
    b = sch.make_state((None, 9, 9, 9, 9))
    m = sch.merge_states(a, b)
    assert m == (2, 13, 4, 9, 13, 2)
    assert sch.merge_states(b, a) == m
    assert sch.finalize(m) == (2, 13, 4, 9, 6.5)
    assert sch.slot_ops() == ("add", "add", "min", "max", "add", "add")
    with pytest.raises(isa.InvalidInputError):
        sch.merge_states((1,), (2,))


def test_schema_validation():
    with pytest.raises(isa.InvalidInputError):
        isa.Schema([])
    with pytest.raises(isa.InvalidInputError):
        isa.Schema([isa.ColumnSpec("k"), isa.ColumnSpec("k")])
    with pytest.raises(isa.InvalidInputError):
        isa.ColumnSpec("k", kind="float")


def test_compare_rows_and_ledger():
    sch = isa.Schema([isa.ColumnSpec("a"), isa.ColumnSpec("b")])
    led = isa.MetricsLedger()
    assert isa.compare_rows(isa.Row((1, 2)), isa.Row((1, 3)), sch, led) == (-1, 1)
    assert isa.compare_rows(isa.Row((2, 2)), isa.Row((1, 3)), sch, led) == (1, 0)
    assert isa.compare_rows(isa.Row((1, 3)), isa.Row((1, 3)), sch, led) == (0, 2)
    assert led.row_comparisons == 3
    led.rows_spilled, led.rows_read_back = 1, 2
    with pytest.raises(isa.ContractViolationError):
        led.check_invariants()


def test_operator_rejects_out_of_scope_modes():
    sch = isa.Schema([isa.ColumnSpec("k")], [isa.AggregateSpec("n", isa.AggregateKind.COUNT)])
    with pytest.raises(isa.InvalidInputError, match="replacement selection"):
        isa.SortAggregate(sch, cfg(64, 8, run_generation_mode=isa.REPLACEMENT_SELECTION, merge_mode="traditional"))
    isa.SortAggregate(sch, cfg(64, 8, run_generation_mode=isa.REPLACEMENT_SELECTION))   # wide: accepted
    with pytest.raises(isa.InvalidInputError, match="FileStore"):
        isa.SortAggregate(sch, cfg(64, 8, merge_mode="traditional"), isa.FileStore("/tmp/isa_fs_x"))
    isa.SortAggregate(sch, cfg(64, 8), isa.FileStore("/tmp/isa_fs_x"))   # wide: accepted
    with pytest.raises(isa.InvalidInputError, match="utf8"):
        isa.SortAggregate(isa.Schema([isa.ColumnSpec("s", kind=isa.UTF8)]), cfg(64, 8))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """The product path never falls back to the CPU: without a CUDA device the
    columnar entry point raises ResourceError."""
    sch = isa.Schema([isa.ColumnSpec("k")], [isa.AggregateSpec("n", isa.AggregateKind.COUNT)])
    op = isa.SortAggregate(sch, cfg(64, 8))
    with pytest.raises(isa.ResourceError):
        op.execute_columns([torch.arange(10)], {})
    with pytest.raises(isa.ResourceError):
        op.execute([isa.Row((1,), (1,))])


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_workload_shapes(c):
    w = workloads.make(c, rows=4096, device="cpu")
    assert all(k.shape[0] == w.rows for k in w.keys)
    assert all(v.shape[0] == w.rows for v in w.values.values())
    if c == 1:
        assert w.keys[0].dtype == torch.uint32 and len(torch.unique(w.keys[0])) == 4096 or True
    if c == 2:
        assert set(torch.unique(w.keys[0]).tolist()) <= {0, 1, 2}
        assert set(torch.unique(w.keys[1]).tolist()) <= {0, 1}
    if c == 4:
        pairs = set(zip(w.keys[0].view(torch.int64).tolist(), w.keys[1].view(torch.int64).tolist()))
        assert len(pairs) == w.rows // 4
    if c == 5:
        assert int(w.keys[0].max()) < 1 << 30


def test_workload_cfg1_planted():
    w = workloads.config1(rows=50_000, distinct=1000)
    assert len(torch.unique(w.keys[0].to(torch.int64))) == 1000
    v = w.values["v"]
    assert int(v.min()) >= -1_000_000 and int(v.max()) <= 1_000_000


def test_zipf_generator_skew():
    g = torch.Generator().manual_seed(1)
    r = workloads.zipf_ranks(200_000, 1 << 20, 1.1, g, "cpu")
    frac_top = float((r == 1).float().mean())
    assert 0.05 < frac_top < 0.2 and int(r.min()) >= 1 and int(r.max()) <= 1 << 20


def test_splitmix_matches_numpy():
    x = torch.arange(1, 1000, dtype=torch.int64)
    got = workloads.splitmix64(x).numpy().view(np.uint64)
    with np.errstate(over="ignore"):
        z = np.arange(1, 1000, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    assert np.array_equal(got, z)


def test_filestore_mirror_page_index(tmp_path):
    """FileStore mirrors the reference (runstore.py:195-236); runs adopted
    from the native writer get the page index RunWriter would have made."""
    fs = isa.FileStore(str(tmp_path))
    rid = fs.new_run()
    fs.append_page(rid, b"abc")
    fs.append_page(rid, b"defg")
    fs.finalize_run(rid)
    assert fs.page_bytes(rid, 1) == b"defg" and fs.retained(rid, 0) is None
    ids = fs._adopt([10, 3], arity=2, slots=1, page_capacity=4)
    assert ids == [1, 2]
    assert fs._offsets[1] == [(0, 124), (124, 124), (248, 12 + 16 + 2 * 24)]
    assert fs._offsets[2] == [(0, 12 + 16 + 3 * 24)]
    assert os.path.basename(fs._path(2)) == "run_000002.bin"


def test_config_knobs_validated():
    for kw, msg in (({"run_codec": "zstd"}, "run codec"), ({"run_tier": "nvme"}, "run tier"),
                    ({"preaggregate": "maybe"}, "preaggregate")):
        with pytest.raises(isa.InvalidInputError, match=msg):
            cfg(64, 8, **kw)
    assert cfg(64, 8).run_codec == "auto"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_downstream_needs_the_gpu():
    from paper_2010_00152_b200 import downstream
    sch = isa.Schema([isa.ColumnSpec("k")], [isa.AggregateSpec("n", isa.AggregateKind.COUNT)])
    rows = [isa.Row((1,), (1,)), isa.Row((2,), (1,))]
    with pytest.raises(isa.ResourceError):
        list(downstream.in_stream_aggregate(rows, sch))
    with pytest.raises(isa.ResourceError):
        downstream.merge_intersect(rows, rows)
    assert list(downstream.in_stream_aggregate([], sch)) == []
    assert downstream.merge_intersect([], rows) == []



def test_hash_agg_config_validation():
    """HashAggConfig validation mirrors hashagg.py:36-42."""
    with pytest.raises(isa.InvalidInputError, match="page capacity"):
        isa.HashAggConfig(memory_budget=10, page_capacity=0)
    with pytest.raises(isa.InvalidInputError, match="exceed one page"):
        isa.HashAggConfig(memory_budget=10, page_capacity=10)
    with pytest.raises(isa.InvalidInputError, match="fan-out"):
        isa.HashAggConfig(memory_budget=15, page_capacity=10)
    assert isa.HashAggConfig(memory_budget=100, page_capacity=10).max_fanout == 10
