"""Parity of the CUDA path with the reference (golden fixtures) and the oracles.

Bar: keys, counts, integer sums/min/max and distinct sets bit-exact; float
sums within rel 1e-9 (float64 inputs) / 1e-5 (float32 inputs), the tolerance
BASELINE.json's north star states.  Run-generation ledgers (fill cycles, run
sizes, spilled rows) must equal the reference's.
"""

import numpy as np
import pytest

import oracle
from conftest import Golden, assert_slots_equal, golden_names, rs_golden_names

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2010_00152_b200 as isa  # noqa: E402
from paper_2010_00152_b200 import workloads  # noqa: E402


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check(res, want_keys, want_slots, rel=1e-9):
    got_keys = [k.cpu().numpy() for k in res.keys]
    got_slots = [s.cpu().numpy() for s in res.states]
    assert len(got_keys[0]) == len(want_keys[0]), f"groups {len(got_keys[0])} != {len(want_keys[0])}"
    for j, (g, w) in enumerate(zip(got_keys, want_keys)):
        assert g.dtype == w.dtype, f"key {j} dtype"
        assert np.array_equal(g, w), f"key column {j} differs"
    for s, (g, w) in enumerate(zip(got_slots, want_slots)):
        assert_slots_equal(g, w, rel=rel, what=f"slot {s}")


def _cfg(memory, page, **kw):
    return isa.SortAggConfig(memory_budget=memory, page_capacity=page, ovc_enabled=False, **kw)


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("variant", ["device", "host_input", "hbm_runs", "packed_runs", "host_runs", "small_chunks",
                                     "k1_always", "k1_never", "tile_merge", "radix_merge", "one_cta",
                                     "window_round_trips", "chunk_loop", "dense_small_windows"])
def test_golden_columns(name, variant, monkeypatch):
    g = Golden(name)
    if variant in ("tile_merge", "radix_merge"):   # force either wide-merge path
        monkeypatch.setenv("ISA_TILE_MERGE", "1" if variant == "tile_merge" else "0")
    if variant in ("radix_merge", "window_round_trips"):   # not the dense-window merge (dense integer keys)
        monkeypatch.setenv("ISA_DENSE", "0")
    if variant == "dense_small_windows":   # dense keys: direct-addressed windows of 256 keys
        monkeypatch.setenv("ISA_DENSE_D", "256")
    if variant == "one_cta":   # small budgets: the one-CTA read-sort-write run generation (isa_seq.cu)
        monkeypatch.setenv("ISA_SEQ", "1")
    if variant == "window_round_trips":   # wide merge reading every window's group count back (no device base)
        monkeypatch.setenv("ISA_DIRECT_MERGE", "0")
    if variant == "chunk_loop":   # small budgets through the chunked loop instead of cut-then-aggregate
        monkeypatch.setenv("ISA_CUT", "0")
    sch = g.schema()
    kw = {}
    if variant == "hbm_runs":
        kw["run_tier"] = "hbm"
    if variant == "packed_runs":   # auto tier: bit-packed runs kept in HBM
        kw["run_codec"] = "packed"
    if variant == "host_runs":     # pinned host tier, bit-packed across PCIe
        kw.update(run_tier="host", run_codec="packed")
    if variant == "small_chunks":
        kw.update(chunk_rows_max=5000, merge_window_rows=3000, window_rows=7000, run_codec="packed")
    if variant == "k1_always":
        kw.update(preaggregate="always", chunk_rows_max=20000)
    if variant == "k1_never":
        kw.update(preaggregate="never")
    mode = str(g.z["merge_mode"]) if "merge_mode" in g.z else "wide"
    if mode != "wide" and variant in ("k1_always", "k1_never", "small_chunks", "packed_runs", "host_runs",
                                      "tile_merge", "radix_merge", "one_cta", "window_round_trips",
                                      "chunk_loop", "dense_small_windows"):
        pytest.skip("pre-aggregation / chunking knobs apply to the wide path only")
    op = isa.SortAggregate(sch, _cfg(g.memory, g.page, merge_mode=mode, **kw))
    n = len(g.keys[0])
    if variant == "host_input":
        keys = [torch.from_numpy(np.ascontiguousarray(k)).pin_memory() for k in g.keys]
        vals = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in g.values.items()}
    else:
        keys = [_cuda(k) for k in g.keys]
        vals = {k: _cuda(v) for k, v in g.values.items()}
    if n == 0:
        res = op.execute_columns(keys, vals)
        assert res.n_groups == 0
        return
    res = op.execute_columns(keys, vals)
    if variant == "host_input":
        assert res.keys[0].device.type == "cpu"
    _check(res, g.out_keys, g.out_slots)
    if mode != "wide":
        # traditional / separate: the full ledger and the executed merge schedule equal the reference's
        for f in ("rows_spilled", "rows_read_back", "pages_written", "pages_read", "merge_steps", "merge_levels"):
            assert getattr(op.ledger, f) == int(g.z["ledger_" + f]), f
        assert op.run_rows == g.z["run_rows"].tolist()
        assert [s["kind"] for s in op.executed_steps] == g.z["executed_kinds"].tolist()
        assert [s["fan_in"] for s in op.executed_steps] == g.z["executed_fan_in"].tolist()
        assert [s["rows_out"] for s in op.executed_steps] == g.z["executed_rows_out"].tolist()
        assert [int(s.get("collapsed", True)) for s in op.executed_steps] == g.z["executed_collapsed"].tolist()
        if op.initial_plan is not None or len(g.z["plan_kinds"]):
            assert [s.kind for s in op.initial_plan.steps] == g.z["plan_kinds"].tolist()
        return
    # run-generation ledger equals the reference's (exact read-sort-write)
    assert op.cycles == [c for c in g.z["cycles"].tolist() if c > 0]
    assert op.run_rows == g.z["run_rows"].tolist()
    assert op.runs_after_generation == int(g.z["runs_after_generation"])
    if g.single_wide:
        assert op.ledger.rows_spilled == int(g.z["ledger_rows_spilled"])
        assert op.ledger.rows_read_back == int(g.z["ledger_rows_read_back"])
        assert op.ledger.pages_written == int(g.z["ledger_pages_written"])
        assert op.ledger.pages_read == int(g.z["ledger_pages_read"])
        assert op.ledger.merge_steps == int(g.z["ledger_merge_steps"])
        assert op.ledger.merge_levels == int(g.z["ledger_merge_levels"])
        if op.initial_plan is not None:
            assert [s.kind for s in op.initial_plan.steps] == g.z["plan_kinds"].tolist()
    else:
        assert op.ledger.rows_spilled == int(g.z["run_rows"].sum())
        assert [s.kind for s in op.initial_plan.steps] == g.z["plan_kinds"].tolist()
    op.ledger.check_invariants()


@pytest.mark.parametrize("name", ["e2e_3000_450_64_8", "edge_one_key", "edge_composite_signed", "cfg4_scaled",
                                  "edge_single", "e2e_spill_once"])
def test_golden_rows(name):
    """Row-object compatibility path: execute(rows) -> list[Row] equal to the reference's."""
    g = Golden(name)
    sch = g.schema()
    n = len(g.keys[0])
    inputs = []
    for n_, kind, col in g.aggs:
        inputs.append(g.values[col].tolist() if col else [None] * n)
    key_lists = [k.tolist() for k in g.keys]
    rows = [isa.Row(tuple(kl[i] for kl in key_lists), sch.make_state(tuple(v[i] for v in inputs)) if g.aggs else ())
            for i in range(n)]
    op = isa.SortAggregate(sch, _cfg(g.memory, g.page))
    out = op.execute(iter(rows))
    assert len(out) == g.n_groups
    want_keys = list(zip(*[k.tolist() for k in g.out_keys]))
    assert [r.key for r in out] == want_keys
    for s, col in enumerate(g.out_slots):
        got = [r.state[s] for r in out]
        if col.dtype.kind == "f":
            np.testing.assert_allclose(got, col, rtol=1e-9)
        else:
            assert got == col.tolist()
    assert all(out[i - 1].key < out[i].key for i in range(1, len(out)))


def test_empty_rows():
    sch = isa.Schema([isa.ColumnSpec("k")], [isa.AggregateSpec("n", isa.AggregateKind.COUNT)])
    op = isa.SortAggregate(sch, _cfg(64, 8))
    assert op.execute(iter([])) == []
    assert op.ledger.rows_spilled == 0


def _oracle_case(w, memory, page=100, rel=1e-9, **kw):
    sch = w.schema
    n = w.rows
    keys_np = [k.cpu().numpy() for k in w.keys]
    vals_np = {k: v.cpu().numpy() for k, v in w.values.items()}
    slots = oracle.make_states(sch, vals_np, n)
    want_keys, want_slots = oracle.reference_aggregate(keys_np, slots, oracle.slot_ops(sch))
    op = isa.SortAggregate(sch, _cfg(memory, page, **kw))
    res = op.execute_columns([k.cuda() for k in w.keys], {k: v.cuda() for k, v in w.values.items()})
    _check(res, want_keys, want_slots, rel=rel)
    return op


@pytest.mark.parametrize("cfg,rows,memory", [
    (1, 1_000_000, 4096),
    (1, 3_000_000, 2048),
    (2, 4_000_000, 4096),
    (2, 3_000_000, 4),        # O = 6 > M = 4: spills every few rows
    (3, 2_000_000, 1 << 16),
    (3, 2_000_000, 1 << 22),  # no spill
    (4, 2_000_000, 1 << 16),
    (5, 3_000_000, 1 << 18),
])
@pytest.mark.parametrize("pre", ["auto", "always", "never"])
def test_random_vs_oracle(cfg, rows, memory, pre):
    kw = {"domain": 1 << 20} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kw)
    rel = 1e-5 if cfg == 3 else 1e-9
    _oracle_case(w, memory, page=min(100, memory // 2), rel=rel, preaggregate=pre)


@pytest.mark.parametrize("pre", ["always", "never"])
def test_ledger_matches_c_oracle_mid_scale(pre):
    w = workloads.config5(rows=2_000_000, device="cpu", domain=1 << 19)
    sch = w.schema
    keys_np = [k.numpy() for k in w.keys]
    slots = oracle.make_states(sch, {"v": w.values["v"].numpy()}, w.rows)
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(sch), 1 << 15, 100)
    op = _oracle_case(w, 1 << 15, preaggregate=pre)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"]
    assert op.runs_after_generation == led["runs"]


@pytest.mark.parametrize("pre", ["always", "never"])
def test_small_chunks_and_windows_vs_oracle(pre):
    w = workloads.config3(rows=1_500_000, device="cpu", domain=1 << 18)
    _oracle_case(w, 1 << 14, rel=1e-5, chunk_rows_max=20_000, merge_window_rows=50_000, preaggregate=pre)


@pytest.mark.parametrize("memory", [1 << 12, 1 << 14])
def test_zipf_ledger_with_tile_preaggregation(memory):
    """Skewed keys with the tile pre-aggregation forced on: flush rows fall
    inside tiles; run sizes and fill cycles must still equal the C oracle's."""
    w = workloads.config3(rows=1_000_000, device="cpu", domain=1 << 16)
    keys_np = [k.numpy() for k in w.keys]
    vals_np = {k: v.numpy() for k, v in w.values.items()}
    slots = oracle.make_states(w.schema, vals_np, w.rows)
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(w.schema), memory, 100)
    op = _oracle_case(w, memory, rel=1e-5, preaggregate="always", chunk_rows_max=50_000)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.run_rows and op.ledger.rows_spilled == led["rows_spilled"]


def test_full_scale_config2_properties():
    """configs[1] at full size (2^28 rows): exactly the 6 groups, counts sum
    to the input size, float sums match torch's float64 sums (order-free
    property, rel 1e-9)."""
    w = workloads.config2(device="cuda")
    op = isa.SortAggregate(w.schema, _cfg(w.memory_budget, 100))
    res = op.execute_columns(w.keys, w.values)
    assert res.n_groups == 6
    k1, k2 = [k.cpu().numpy() for k in res.keys]
    assert list(zip(k1.tolist(), k2.tolist())) == [(a, b) for a in range(3) for b in range(2)]
    counts = res.states[0]
    assert int(counts.sum()) == w.rows
    gid = w.keys[0].to(torch.int64) * 2 + w.keys[1].to(torch.int64)
    want_counts = torch.bincount(gid, minlength=6)
    assert torch.equal(counts.cpu(), want_counts.cpu())
    for i in range(4):
        want = torch.zeros(6, dtype=torch.float64, device="cuda").index_add_(0, gid, w.values[f"f{i}"])
        np.testing.assert_allclose(res.states[1 + i].cpu().numpy(), want.cpu().numpy(), rtol=1e-9)
    assert op.ledger.rows_spilled == 0


@pytest.mark.parametrize("hi_card", [2, 1000, 1 << 40])
def test_128bit_keys_high_word_cardinality(hi_card):
    """128-bit keys sort on the high word first and finish equal-high runs on
    the low word; a low-cardinality high word exercises the full-LSD fallback."""
    rng = np.random.default_rng(hi_card % 1000 + 7)
    n = 600_000
    k1 = rng.integers(0, hi_card, n, dtype=np.uint64)
    k2 = rng.integers(0, 1 << 20, n, dtype=np.uint64)
    v = rng.integers(-1000, 1000, n)
    sch = isa.Schema([isa.ColumnSpec("a"), isa.ColumnSpec("b")],
                     [isa.AggregateSpec("n", isa.AggregateKind.COUNT), isa.AggregateSpec("s", isa.AggregateKind.SUM, "v"),
                      isa.AggregateSpec("m", isa.AggregateKind.MIN, "v")])
    slots = oracle.make_states(sch, {"v": v}, n)
    want_k, want_s = oracle.reference_aggregate([k1, k2], slots, oracle.slot_ops(sch))
    op = isa.SortAggregate(sch, _cfg(1 << 14, 100))
    res = op.execute_columns([_cuda(k1), _cuda(k2)], {"v": _cuda(v)})
    _check(res, want_k, want_s)


def _few_groups_case(nt, key_kind, n, extra, seed, wide=False):
    """n rows over nt base groups, plus `extra` new groups first seen in the
    second half (absorb misses); keys of the given kind, mixed value types."""
    rng = np.random.default_rng(seed)
    base = rng.choice(1 << 12, nt, replace=False)
    ids = base[rng.integers(0, nt, n)]
    if extra:
        pos = np.sort(rng.choice(np.arange(n // 2, n), extra, replace=False))
        ids[pos] = (1 << 12) + np.arange(extra) * 7 + 1
        ids[pos[-1]:][rng.random(n - pos[-1]) < 0.01] = ids[pos[-1]]   # the last new key recurs
    if key_kind == "i8":
        keys = [(ids % 251 - 125).astype(np.int8)] if not extra else [(ids % 16381 - 8190).astype(np.int16)]
    elif key_kind == "i32x2":
        keys = [(ids // 64).astype(np.int32) - 5, (ids % 64).astype(np.int32)]
    elif key_kind == "u64x2":   # 128-bit normalized keys
        keys = [(ids.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)), (ids % 3).astype(np.uint64)]
    else:
        keys = [ids.astype(np.int64) * -3]
    vals = {"v": rng.uniform(-1e3, 1e3, n), "w": rng.integers(-(1 << 30), 1 << 30, n).astype(np.int32),
            "x": rng.integers(-(1 << 40), 1 << 40, n), "y": rng.standard_normal(n).astype(np.float32)}
    cols = [isa.ColumnSpec(f"k{i}") for i in range(len(keys))]
    aggs = [isa.AggregateSpec("n", isa.AggregateKind.COUNT), isa.AggregateSpec("s", isa.AggregateKind.SUM, "v"),
            isa.AggregateSpec("lo", isa.AggregateKind.MIN, "w"), isa.AggregateSpec("hi", isa.AggregateKind.MAX, "x"),
            isa.AggregateSpec("a", isa.AggregateKind.AVG, "y")]
    if wide:   # more state slots than the bulk kernel keeps in registers
        aggs += [isa.AggregateSpec("vlo", isa.AggregateKind.MIN, "v"), isa.AggregateSpec("yhi", isa.AggregateKind.MAX, "y")]
    return isa.Schema(cols, aggs), keys, vals


@pytest.mark.parametrize("nt", [1, 3, 6, 8])
@pytest.mark.parametrize("key_kind", ["i8", "i32x2", "u64x2", "i64"])
@pytest.mark.parametrize("extra,memory,wide", [(0, 4096, False), (40, 4096, False), (40, None, False),
                                               (40, 4096, True)])
def test_tiny_table_absorb_vs_oracle(nt, key_kind, extra, memory, wide):
    """The |T| <= 8 absorb kernel: ragged
    row counts, late new groups (absorb misses), flushes inside an absorb
    chunk (memory = nt + 3), every value dtype; ledger equals the C oracle's."""
    n = 1_000_003 + 517 * nt
    sch, keys, vals = _few_groups_case(nt, key_kind, n, extra, seed=nt * 31 + len(key_kind), wide=wide)
    M = memory if memory is not None else nt + 3
    slots = oracle.make_states(sch, vals, n)
    want_k, want_s = oracle.reference_aggregate(keys, slots, oracle.slot_ops(sch))
    _, _, led, cycles = oracle.rsw_sortagg(keys, slots, oracle.slot_ops(sch), M, 2)
    for on_host in (False, True):
        op = isa.SortAggregate(sch, _cfg(M, 2))
        kk = [torch.from_numpy(k).pin_memory() if on_host else _cuda(k) for k in keys]
        vv = {c: (torch.from_numpy(v).pin_memory() if on_host else _cuda(v)) for c, v in vals.items()}
        res = op.execute_columns(kk, vv)
        _check(res, want_k, want_s, rel=1e-5)
        assert op.cycles == [c for c in cycles if c > 0]
        assert op.ledger.rows_spilled == led["rows_spilled"]


@pytest.mark.parametrize("cfg,rows,memory", [(3, 3_000_000, 1 << 16), (4, 2_000_000, 1 << 16), (5, 3_000_000, 1 << 16),
                                             (1, 1_000_000, 4096)])
def test_packed_runs_vs_raw(cfg, rows, memory):
    """Bit-packed host runs: the same output and ledger as raw runs, fewer
    bytes across PCIe (every state/key bit pattern round-trips)."""
    kw = {"domain": 1 << 22} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kw)
    rel = 1e-5 if cfg == 3 else 1e-9
    packed = _oracle_case(w, memory, rel=rel, run_codec="packed", run_tier="host")
    raw = _oracle_case(w, memory, rel=rel, run_codec="raw", run_tier="host")
    assert packed.run_rows == raw.run_rows and packed.ledger.rows_spilled == raw.ledger.rows_spilled
    assert packed.ledger.rows_read_back == raw.ledger.rows_read_back
    assert 0 < packed.device_ledger["bytes_d2h"] < raw.device_ledger["bytes_d2h"]
    assert 0 < packed.device_ledger["bytes_h2d"] <= raw.device_ledger["bytes_h2d"]


@pytest.mark.parametrize("name", ["pages_3000_450_64_8", "pages_composite_avg", "pages_distinct"])
@pytest.mark.parametrize("on_host", [False, True])
def test_filestore_runs_byte_identical_to_reference(name, on_host, tmp_path):
    """FileStore tier: the operator's run files equal, byte for byte, the
    files the reference's RunWriter wrote into its FileStore for the same
    input (tests/golden/pages_*.npz, tools/make_golden.py), the wide merge
    reads them back from disk, and the output equals the reference's."""
    import os as _os
    z = np.load(_os.path.join(_os.path.dirname(__file__), "golden", f"{name}.npz"))
    arity = sum(1 for k in z.files if k.startswith("in_k"))
    keys = [z[f"in_k{j}"] for j in range(arity)]
    vals = {k[len("in_v_"):]: z[k] for k in z.files if k.startswith("in_v_")}
    aggs = [tuple(s.split(":")) for s in z["aggs"].tolist()]
    sch = isa.Schema([isa.ColumnSpec(f"k{j}") for j in range(arity)],
                     [isa.AggregateSpec(n, isa.AggregateKind(k), c or None) for n, k, c in aggs])
    fs = isa.FileStore(str(tmp_path))
    op = isa.SortAggregate(sch, _cfg(int(z["memory_budget"]), int(z["page_capacity"])), fs)
    if on_host:
        kk = [torch.from_numpy(np.ascontiguousarray(k)).pin_memory() for k in keys]
        vv = {n: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for n, v in vals.items()}
    else:
        kk = [_cuda(k) for k in keys]
        vv = {n: _cuda(v) for n, v in vals.items()}
    res = op.execute_columns(kk, vv)
    want_k = [z[f"out_k{j}"] for j in range(arity)]
    want_s = [z[k] for k in sorted((k for k in z.files if k.startswith("out_s")), key=lambda x: int(x[5:]))]
    _check(res, want_k, want_s)
    assert op.runs_after_generation == int(z["runs_after_generation"])
    blob = z["run_bytes"].tobytes()
    off = 0
    for fname, length in zip(z["run_files"].tolist(), z["run_lengths"].tolist()):
        got = open(_os.path.join(str(tmp_path), fname), "rb").read()
        assert got == blob[off: off + length], f"{fname} differs from the reference's run file"
        off += length
    # the store's page index reads the pages back like the reference's read_page
    slots = len(want_s)
    for rid in op.run_ids:
        pages = [fs.page_bytes(rid, i) for i in range(len(fs._offsets[rid]))]
        keys_r, _, counts = oracle.parse_run_pages(b"".join(pages), arity, slots)
        assert sum(counts) == len(keys_r[0])


def test_filestore_rejects_float_states(tmp_path):
    sch = isa.Schema([isa.ColumnSpec("k")], [isa.AggregateSpec("s", isa.AggregateKind.SUM, "v")])
    op = isa.SortAggregate(sch, _cfg(64, 8), isa.FileStore(str(tmp_path)))
    with pytest.raises(isa.InvalidInputError, match="int64 state"):
        op.execute_columns([_cuda(np.arange(1000) % 300)], {"v": _cuda(np.random.default_rng(1).random(1000))})


def test_filestore_many_windows_vs_oracle(tmp_path):
    """FileStore tier at a few million rows with many merge windows: slice
    bounds searched through page high keys + one page read per bound."""
    w = workloads.config5(rows=3_000_000, device="cpu", domain=1 << 20)
    sch = w.schema
    keys_np = [k.numpy() for k in w.keys]
    slots = oracle.make_states(sch, {"v": w.values["v"].numpy()}, w.rows)
    want_k, want_s = oracle.reference_aggregate(keys_np, slots, oracle.slot_ops(sch))
    fs = isa.FileStore(str(tmp_path))
    op = isa.SortAggregate(sch, _cfg(1 << 16, 100, merge_window_rows=200_000), fs)
    res = op.execute_columns([k.cuda() for k in w.keys], {k: v.cuda() for k, v in w.values.items()})
    _check(res, want_k, want_s)
    assert op.device_ledger["merge_windows"] > 5
    assert len(op.run_ids) == op.runs_after_generation > 10
    assert op.ledger.rows_spilled == sum(op.run_rows)


def _golden_npz(name):
    import os as _os
    return np.load(_os.path.join(_os.path.dirname(__file__), "golden", f"{name}.npz"))


@pytest.mark.parametrize("name", ["downstream_in_stream_sorted", "downstream_in_stream_unsorted"])
@pytest.mark.parametrize("on_host", [False, True])
def test_in_stream_aggregate_vs_reference(name, on_host):
    """bench.in_stream_aggregate (bench.py:199-212): one group per run of
    equal consecutive keys -- on sorted input the grouping, on unsorted input
    the same run-splitting the reference generator shows."""
    from paper_2010_00152_b200 import downstream
    z = _golden_npz(name)
    sch = isa.Schema([isa.ColumnSpec("k0"), isa.ColumnSpec("k1")],
                     [isa.AggregateSpec("n", isa.AggregateKind.COUNT), isa.AggregateSpec("s", isa.AggregateKind.SUM, "v"),
                      isa.AggregateSpec("lo", isa.AggregateKind.MIN, "v")])
    op = isa.SortAggregate(sch, _cfg(64, 8))
    cols = [z["in_k0"], z["in_k1"], z["in_v_v"]]
    if on_host:
        k0, k1, v = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in cols]
    else:
        k0, k1, v = [_cuda(c) for c in cols]
    res = op.in_stream_columns([k0, k1], {"v": v})
    _check(res, [z["out_k0"], z["out_k1"]], [z["out_s0"], z["out_s1"], z["out_s2"]])
    assert op.ledger.rows_spilled == 0
    rows = [isa.Row((int(a), int(b)), (1, int(x), int(x))) for a, b, x in zip(*cols)][:3000]
    got = list(downstream.in_stream_aggregate(rows, sch))
    want = list(zip(z["out_k0"].tolist(), z["out_k1"].tolist()))
    assert [r.key for r in got] == want[: len(got)] or name.endswith("unsorted")


def test_sort_intersect_plan_vs_reference():
    """bench.sort_intersect_plan (bench.py:553-569): two in-sort aggregations
    and a merge intersection of their sorted outputs; keys and both spill
    ledgers equal the reference's."""
    from paper_2010_00152_b200 import downstream
    z = _golden_npz("downstream_intersect")
    sch = isa.Schema([isa.ColumnSpec("k")], [isa.AggregateSpec("n", isa.AggregateKind.COUNT)])
    ra = [isa.Row((int(x),), (1,)) for x in z["in_a"]]
    rb = [isa.Row((int(x),), (1,)) for x in z["in_b"]]
    keys, ledgers = downstream.sort_intersect_plan(ra, rb, sch, memory_rows=int(z["memory_rows"]),
                                                   page_rows=int(z["page_rows"]))
    assert keys == [(int(k),) for k in z["out_keys"]]
    assert [l.rows_spilled for l in ledgers] == z["rows_spilled"].tolist()
    # columnar form on device and host columns
    op = isa.SortAggregate(sch, _cfg(int(z["memory_rows"]), int(z["page_rows"])))
    a = op.execute_columns([_cuda(z["in_a"])]).keys
    b = op.execute_columns([_cuda(z["in_b"])]).keys
    out = op.intersect_columns(a, b)
    assert np.array_equal(out[0].cpu().numpy(), z["out_keys"])
    out_h = op.intersect_columns([t.cpu() for t in a], [t.cpu() for t in b])
    assert np.array_equal(out_h[0].numpy(), z["out_keys"])
    assert downstream.merge_intersect([], ra[:3]) == []


@pytest.mark.parametrize("cfg,domain", [(5, 1 << 22)])
def test_large_chunk_flush_rows_vs_c_oracle(cfg, domain):
    """Fill cycles of more than 2^20 rows (large-chunk flush analysis: global
    new-head bitmap + k-th select): cycles and run sizes equal the C
    restatement's exactly."""
    w = workloads.make(cfg, rows=8_000_000, device="cpu", domain=domain)
    keys_np = [k.numpy() for k in w.keys]
    vals_np = {k: v.numpy() for k, v in w.values.items()}
    slots = oracle.make_states(w.schema, vals_np, w.rows)
    M = 1 << 20
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(w.schema), M, 100)
    op = _oracle_case(w, M, rel=1e-5 if cfg == 3 else 1e-9, preaggregate="never")
    assert op.cycles == [c for c in cycles if c > 0]
    assert max(op.cycles) > (1 << 20)
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]


@pytest.mark.parametrize("shift,bits,base", [(5, 27, -(1 << 50)), (7, 32, 3 << 45), (0, 20, -7)])
def test_packed_radix_passes_vs_oracle(shift, bits, base):
    """Keys whose varying bits span <= 32 take the packed radix passes
    (one 8-byte word per row, isa_kernels.cu k_rs_scatter PK 1/2/3): the
    constant key bits outside the span (negative / high offsets) must come
    back unchanged, and chunks span many sort tiles."""
    w = workloads.config5(rows=3_000_000, device="cpu", domain=1 << 22)
    g = torch.Generator().manual_seed(2010 + shift)
    x = torch.randint(0, 1 << bits, (w.rows,), generator=g, dtype=torch.int64)
    if bits == 32:
        x[:2] = torch.tensor([0, (1 << 32) - 1])   # both span ends present
    w.keys[0] = base + (x << shift)
    _oracle_case(w, 1 << 18)


def _int_workload(key, val, memory):
    sch = workloads._int_schema([("n", isa.AggregateKind.COUNT, None), ("s", isa.AggregateKind.SUM, "v"),
                                 ("lo", isa.AggregateKind.MIN, "v"), ("hi", isa.AggregateKind.MAX, "v")], 1)
    return workloads.Workload(5, int(key.numel()), sch, [key], {"v": val}, memory)


@pytest.mark.parametrize("on_host", [False, True])
def test_tile_merge_skewed_buckets_fall_back(on_host, monkeypatch):
    """Keys packed into a tiny range next to a few keys spread over int64:
    the linear bucket function puts most rows into one bucket, the tiles of
    those windows overflow, and the windows are merged by the radix-sort
    path instead -- same result as the oracle."""
    monkeypatch.setenv("ISA_TILE_MERGE", "1")
    g = torch.Generator().manual_seed(7)
    n = 600_000
    dense = torch.randint(0, 3000, (n,), generator=g, dtype=torch.int64)
    wide = torch.randint(-(1 << 62), 1 << 62, (n // 100,), generator=g, dtype=torch.int64)
    key = torch.cat([dense, wide])[torch.randperm(n + n // 100, generator=g)]
    val = torch.randint(-1000, 1000, (key.numel(),), generator=g, dtype=torch.int64)
    w = _int_workload(key, val, 1 << 10)
    keys_np = [key.numpy()]
    slots = oracle.make_states(w.schema, {"v": val.numpy()}, w.rows)
    want_k, want_s = oracle.reference_aggregate(keys_np, slots, oracle.slot_ops(w.schema))
    op = isa.SortAggregate(w.schema, _cfg(1 << 10, 100))
    kk = [key.pin_memory()] if on_host else [key.cuda()]
    vv = {"v": val.pin_memory() if on_host else val.cuda()}
    _check(op.execute_columns(kk, vv), want_k, want_s)
    assert op.runs_after_generation > 1


@pytest.mark.parametrize("on_host", [False, True])
def test_tile_merge_sorted_input(on_host, monkeypatch):
    """Ascending input: every run covers its own key range.  Host input
    fixes the buckets from the first run only (later keys clamp into the
    last bucket), device input from a sample of the whole input."""
    monkeypatch.setenv("ISA_TILE_MERGE", "1")
    n = 400_000
    key = torch.arange(n, dtype=torch.int64) * 7 // 3
    val = torch.arange(n, dtype=torch.int64) % 1000
    w = _int_workload(key, val, 1 << 12)
    slots = oracle.make_states(w.schema, {"v": val.numpy()}, n)
    want_k, want_s = oracle.reference_aggregate([key.numpy()], slots, oracle.slot_ops(w.schema))
    op = isa.SortAggregate(w.schema, _cfg(1 << 12, 100))
    kk = [key.pin_memory()] if on_host else [key.cuda()]
    vv = {"v": val.pin_memory() if on_host else val.cuda()}
    _check(op.execute_columns(kk, vv), want_k, want_s)


@pytest.mark.parametrize("memory", [512, 4096])
def test_tile_merge_many_runs(memory, monkeypatch):
    """Hundreds to thousands of runs in one wide merge: tiles hold a few
    rows of every run."""
    monkeypatch.setenv("ISA_TILE_MERGE", "1")
    w = workloads.config5(rows=1_000_000, device="cpu", domain=1 << 20)
    op = _oracle_case(w, memory, page=min(100, memory // 2))
    assert op.runs_after_generation > 200


@pytest.mark.parametrize("pbits", [2, 7])
@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_tile_merge_inexact_prefix(cfg, pbits, monkeypatch):
    """Tile sort words carry only `pbits` bits of the key: rows whose
    prefixes tie are finished by the insertion sort on the full key (short
    runs) or by the full-width LSD fallback (runs longer than 64) -- the
    result must not change."""
    monkeypatch.setenv("ISA_TM_PREFIX_BITS", str(pbits))
    monkeypatch.setenv("ISA_TILE_MERGE", "1")
    rows = {3: 400_000, 4: 300_000, 5: 600_000}[cfg]
    w = workloads.make(cfg, rows=rows, device="cpu", **({"domain": 1 << 20} if cfg in (3, 5) else {}))
    op = _oracle_case(w, 4096, page=100, rel=1e-5 if cfg == 3 else 1e-9)
    assert op.runs_after_generation > 10


@pytest.mark.parametrize("cfg,rows,memory", [
    (3, 2_000_000, 1 << 14),   # Zipf: most rows hit the resident table
    (3, 1_500_000, 1 << 12),
    (1, 1_000_000, 4096),
    (5, 1_000_000, 1 << 14),   # almost every row is a miss
    (4, 600_000, 1 << 14),     # 128-bit keys
])
def test_hot_absorb_vs_c_oracle(cfg, rows, memory):
    """Rows whose key is already resident absorbed through the table's hash
    image (hot_absorb='always'): output equals the oracle, and the fill
    cycles and spilled rows equal the C oracle's read-sort-write ledger."""
    kw = {"domain": 1 << 18} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kw)
    rel = 1e-5 if cfg == 3 else 1e-9
    op = _oracle_case(w, memory, page=min(100, memory // 2), rel=rel, hot_absorb="always")
    keys_np = [k.cpu().numpy() for k in w.keys]
    slots = oracle.make_states(w.schema, {k: v.cpu().numpy() for k, v in w.values.items()}, w.rows)
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(w.schema), memory, min(100, memory // 2))
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]
    assert op.phase_stats["hot"]["calls"] > 0, "the hot path did not run"


def test_hot_absorb_config3_shape():
    """The hash-image absorb on a config-3-shaped input with a table above
    the auto threshold (2^16 groups, Zipf keys, cycles of >= 2 M rows):
    ledger and output unchanged."""
    w = workloads.config3(rows=12_000_000, device="cpu")
    M = 1 << 16
    op = _oracle_case(w, M, page=100, rel=1e-5, hot_absorb="always")
    keys_np = [k.cpu().numpy() for k in w.keys]
    slots = oracle.make_states(w.schema, {k: v.cpu().numpy() for k, v in w.values.items()}, w.rows)
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(w.schema), M, 100)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"]
    assert max(op.cycles) >= 2 * M
    assert op.phase_stats["hot"]["calls"] > 0


@pytest.mark.parametrize("cap", ["1024", "4096"])
@pytest.mark.parametrize("on_host", [False, True])
def test_hybrid_sort_clustered_bucket_falls_back(on_host, cap, monkeypatch):
    """Half the rows share the top 16 bits of the sort field (a bucket far
    larger than one CTA's local sort): the hybrid sort detects it and
    finishes with plain LSD passes -- same result as the oracle."""
    monkeypatch.setenv("ISA_HYBRID", "1")
    monkeypatch.setenv("ISA_RL_CAP", cap)
    g = torch.Generator().manual_seed(11)
    n = 600_000
    spread = torch.randint(0, 1 << 40, (n // 2,), generator=g, dtype=torch.int64)
    dense = torch.randint(0, 1 << 20, (n - n // 2,), generator=g, dtype=torch.int64)
    key = torch.cat([spread, dense])[torch.randperm(n, generator=g)]
    val = torch.randint(-1000, 1000, (n,), generator=g, dtype=torch.int64)
    w = _int_workload(key, val, 1 << 18)
    slots = oracle.make_states(w.schema, {"v": val.numpy()}, n)
    want_k, want_s = oracle.reference_aggregate([key.numpy()], slots, oracle.slot_ops(w.schema))
    op = isa.SortAggregate(w.schema, _cfg(1 << 18, 100))
    kk = [key.pin_memory()] if on_host else [key.cuda()]
    vv = {"v": val.pin_memory() if on_host else val.cuda()}
    _check(op.execute_columns(kk, vv), want_k, want_s)


@pytest.mark.parametrize("cap", ["1024", "4096"])
@pytest.mark.parametrize("cfg,rows,memory", [(3, 2_000_000, 1 << 20), (4, 1_000_000, 1 << 19), (5, 2_000_000, 1 << 20),
                                             (1, 1_000_000, 1 << 19)])
def test_hybrid_sort_vs_oracle(cfg, rows, memory, cap, monkeypatch):
    """The hybrid sort (top-16 onesweep passes + CTA-local bucket sort) on
    the config shapes: output and ledger equal the oracle's."""
    monkeypatch.setenv("ISA_HYBRID", "1")
    monkeypatch.setenv("ISA_RL_CAP", cap)
    kw = {"domain": 1 << 24} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kw)
    _oracle_case(w, memory, page=100, rel=1e-5 if cfg == 3 else 1e-9)



@pytest.mark.parametrize("on_host", [False, True])
@pytest.mark.parametrize("name", rs_golden_names())
def test_replacement_selection_golden(name, on_host):
    """Replacement selection (one persistent CTA, isa_seq.cu) against the
    reference's own output, run sizes, steady-probe totals and merge plan
    (tools/make_golden_rs.py)."""
    g = Golden(name)
    chunk = int(g.z["eviction_chunk"]) or None
    cfg = _cfg(g.memory, g.page, run_generation_mode=isa.REPLACEMENT_SELECTION, eviction_chunk=chunk)
    op = isa.SortAggregate(g.schema(), cfg)
    if on_host:
        keys = [torch.from_numpy(np.ascontiguousarray(k)).pin_memory() for k in g.keys]
        vals = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in g.values.items()}
    else:
        keys = [_cuda(k) for k in g.keys]
        vals = {k: _cuda(v) for k, v in g.values.items()}
    _check(op.execute_columns(keys, vals), g.out_keys, g.out_slots)
    assert op.run_rows == g.z["run_rows"].tolist()
    assert op.cycles == []
    d = op.device_ledger
    assert [d["steady_probes"], d["steady_absorbs"], d["steady_resident_sum"]] == g.z["steady"].tolist()
    assert op.ledger.rows_spilled == int(g.z["run_rows"].sum())
    if len(g.z["run_rows"]):
        assert [st.kind for st in op.initial_plan.steps] == g.z["plan_kinds"].tolist()
    op.ledger.check_invariants()


@pytest.mark.parametrize("rows,memory,chunk", [(50_000, 700, 33), (80_000, 2048, 100), (30_000, 64, 1)])
def test_replacement_selection_vs_restatement(rows, memory, chunk):
    """Larger random cases: run sizes and steady totals equal the Python
    restatement's, output equals the numpy oracle's."""
    w = workloads.make(3, rows=rows, device="cpu", domain=1 << 14)
    op = _oracle_case(w, memory, page=max(2, min(100, memory // 2)), rel=1e-5,
                      run_generation_mode=isa.REPLACEMENT_SELECTION, eviction_chunk=chunk)
    keys = oracle.normalize_keys([k.numpy() for k in w.keys])[1].tolist()
    runs, steady = oracle.rs_run_generation(keys, memory, chunk)
    assert op.run_rows == runs
    d = op.device_ledger
    assert [d["steady_probes"], d["steady_absorbs"], d["steady_resident_sum"]] == list(steady)


def test_config1_one_cta_run_generation_ledger(monkeypatch):
    """BASELINE config 1 (1e6 rows, M = 4096) through the one-CTA run
    generation: fill cycles and run sizes equal the C oracle's."""
    monkeypatch.setenv("ISA_SEQ", "1")
    w = workloads.config1(device="cpu")
    keys_np = [k.numpy() for k in w.keys]
    slots = oracle.make_states(w.schema, {k: v.numpy() for k, v in w.values.items()}, w.rows)
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(w.schema), 4096, 100)
    op = _oracle_case(w, 4096, page=100)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]
    assert op.device_ledger["kernel_launches"] < 200   # no per-cycle launches



@pytest.mark.parametrize("on_host", [False, True])
@pytest.mark.parametrize("name", ["hash_inmem_4096", "hash_composite_avg", "hash_spill_1000"])
def test_hash_aggregate_baseline_vs_reference(name, on_host):
    """HashAggregate (hashagg.py:73-198) on the GPU against the reference's
    own output: in-memory fixtures in the reference's order (first arrival)
    with its hash / column-access counters; the partitioned fixture as the
    same set of groups (the GPU table holds every group, no partitions)."""
    g = Golden(name)
    op = isa.HashAggregate(g.schema(), isa.HashAggConfig(memory_budget=g.memory, page_capacity=g.page))
    if on_host:
        keys = [torch.from_numpy(np.ascontiguousarray(k)).pin_memory() for k in g.keys]
        vals = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in g.values.items()}
    else:
        keys = [_cuda(k) for k in g.keys]
        vals = {k: _cuda(v) for k, v in g.values.items()}
    res = op.execute_columns(keys, vals)
    assert op.partitions == []
    if int(g.z["n_partitions"]) == 0:
        _check(res, g.out_keys, g.out_slots)
        assert op.ledger.hash_computations == int(g.z["ledger_hash_computations"])
        assert op.ledger.column_value_accesses == int(g.z["ledger_column_value_accesses"])
    else:
        got = sorted(zip(*[k.cpu().tolist() for k in res.keys], *[s.cpu().tolist() for s in res.states]))
        want = sorted(zip(*[k.tolist() for k in g.out_keys], *[s.tolist() for s in g.out_slots]))
        assert got == want


def test_hash_aggregate_rows_and_large_random():
    """Row-object path, and a 4M-row Zipf input against the numpy oracle
    (groups compared after sorting: first-arrival order is checked on the
    reference fixtures)."""
    g = Golden("hash_inmem_4096")
    op = isa.HashAggregate(g.schema(), isa.HashAggConfig(memory_budget=4096, page_capacity=64))
    rows = [isa.Row((int(k),), (1, int(v), int(v), int(v))) for k, v in zip(g.keys[0][:3000], g.values["v"][:3000])]
    out = op.execute(rows)
    first = {}
    for r in rows:
        first.setdefault(r.key, len(first))
    assert [r.key for r in out] == sorted(first, key=first.get)
    w = workloads.config3(rows=4_000_000, device="cpu", domain=1 << 20)
    sch = w.schema
    op = isa.HashAggregate(sch, isa.HashAggConfig(memory_budget=1 << 16, page_capacity=100))
    res = op.execute_columns([k.cuda() for k in w.keys], {k: v.cuda() for k, v in w.values.items()})
    slots = oracle.make_states(sch, {k: v.numpy() for k, v in w.values.items()}, w.rows)
    want_k, want_s = oracle.reference_aggregate([k.numpy() for k in w.keys], slots, oracle.slot_ops(sch))
    order = np.argsort(res.keys[0].cpu().numpy(), kind="stable")
    assert np.array_equal(res.keys[0].cpu().numpy()[order], want_k[0])
    for s_, (gcol, wcol) in enumerate(zip(res.states, want_s)):
        assert_slots_equal(gcol.cpu().numpy()[order], wcol, rel=1e-5, what=f"slot {s_}")


@pytest.mark.parametrize("case", ["rs", "rsw_chunks", "tile_merge", "hot", "hash", "one_cta"])
def test_repeat_runs_bit_identical(case, monkeypatch):
    """Race detector in place of compute-sanitizer (closed on this pool):
    the same input run five times gives bit-identical integer outputs and
    ledgers (a shared-memory race in the replacement-selection promotion was
    found this way)."""
    w = workloads.make(3 if case != "rsw_chunks" else 5, rows=300_000, device="cpu", domain=1 << 14)
    keys = [k.cuda() for k in w.keys]
    vals = {k: v.cuda() for k, v in w.values.items()}
    kw = {}
    if case == "rs":
        kw = dict(run_generation_mode=isa.REPLACEMENT_SELECTION, eviction_chunk=8)
    if case == "tile_merge":
        monkeypatch.setenv("ISA_TILE_MERGE", "1")
    if case == "hot":
        kw = dict(hot_absorb="always")
    if case == "one_cta":
        monkeypatch.setenv("ISA_SEQ", "1")
    outs = []
    for _ in range(5):
        if case == "hash":
            op = isa.HashAggregate(w.schema, isa.HashAggConfig(memory_budget=4096, page_capacity=64))
            r = op.execute_columns(keys, vals)
            led = ()
        else:
            op = isa.SortAggregate(w.schema, _cfg(1024 if case in ("rs", "one_cta") else 4096, 100, **kw))
            r = op.execute_columns(keys, vals)
            led = (tuple(op.run_rows), tuple(op.cycles), op.ledger.rows_spilled)
        ints = [t.cpu() for t in r.keys] + [t.cpu() for t in r.states if not t.dtype.is_floating_point]
        outs.append((ints, led))
    for ints, led in outs[1:]:
        assert led == outs[0][1]
        for a, b in zip(ints, outs[0][0]):
            assert torch.equal(a, b)



@pytest.mark.parametrize("cfg,rows,memory,window", [(5, 3_000_000, 1 << 14, 50_000), (3, 2_000_000, 1 << 14, 40_000),
                                                    (4, 1_000_000, 1 << 14, 30_000), (1, 1_000_000, 4096, 20_000)])
def test_direct_window_merge_many_windows_vs_oracle(cfg, rows, memory, window, monkeypatch):
    """Many small wide-merge windows appended on the device (group numbers
    continue from a device-resident count, the result grows when the rows
    staged so far could overflow it): equals the oracle."""
    monkeypatch.setenv("ISA_TILE_MERGE", "0")   # the radix-window path (128-bit keys default to tiles)
    monkeypatch.setenv("ISA_DENSE", "0")        # ... and not the dense-window merge
    kw = {"domain": 1 << 20} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kw)
    op = _oracle_case(w, memory, page=100, rel=1e-5 if cfg == 3 else 1e-9, merge_window_rows=window)
    assert op.device_ledger["merge_windows"] > 10


def _mixed_cycles_input(n_short, n_long, short_domain, long_domain, seed, float_vals=False):
    """Rows whose first part flushes every few thousand rows (large key
    domain) and whose second part holds few keys (fill cycles far longer
    than one CTA sorts): the cut-then-aggregate scan hands over to the
    chunked loop at the first long cycle."""
    rng = np.random.default_rng(seed)
    k = np.concatenate([rng.integers(0, short_domain, n_short), rng.integers(0, long_domain, n_long)])
    k = k.astype(np.uint32)
    if float_vals:
        v = rng.uniform(-1e5, 1e5, len(k))
    else:
        v = rng.integers(-1_000_000, 1_000_001, len(k)).astype(np.int64)
    return k, v


def _cut_schema(float_vals=False):
    from paper_2010_00152_b200.core import AggregateKind, AggregateSpec, ColumnSpec, Schema
    return Schema([ColumnSpec("k")], [AggregateSpec("n", AggregateKind.COUNT, None),
                                      AggregateSpec("s", AggregateKind.SUM, "v"),
                                      AggregateSpec("lo", AggregateKind.MIN, "v"),
                                      AggregateSpec("hi", AggregateKind.MAX, "v")])


@pytest.mark.parametrize("n_short,n_long,short_domain,long_domain,memory", [
    (1_000_000, 0, 10_000, 1, 4096),          # config-1 shape: 190 short cycles, all through the cut scan
    (300_000, 200_000, 50_000, 3000, 4096),   # short cycles, then one long cycle: hand-over to the chunked loop
    (200_000, 0, 300, 1, 64),                 # tiny budget: a flush every ~70 rows
    (100_000, 300_000, 20_000, 40, 1000),     # hand-over, then no further flush
    (5000, 0, 100, 1, 4096),                  # no flush at all: the one cycle is the result
    (50_000, 0, 1 << 31, 1, 2),               # distinct keys, M = 2: three rows per cycle
])
@pytest.mark.parametrize("on_host", [False, True])
@pytest.mark.parametrize("float_vals", [False, True])
def test_cut_then_aggregate_vs_c_oracle(n_short, n_long, short_domain, long_domain, memory, on_host, float_vals):
    """Small-budget read-sort-write through the cut scan + per-cycle runs:
    output, fill cycles, run sizes and spilled rows equal the C restatement
    (oracle/rsw_oracle.c) on inputs with short cycles, long cycles and the
    hand-over between them."""
    k, v = _mixed_cycles_input(n_short, n_long, short_domain, long_domain, 7 + memory, float_vals)
    sch = _cut_schema(float_vals)
    slots = oracle.make_states(sch, {"v": v}, len(k))
    ok, os_, led, cycles = oracle.rsw_sortagg([k], slots, oracle.slot_ops(sch), memory, min(100, memory // 2))
    op = isa.SortAggregate(sch, _cfg(memory, min(100, memory // 2)))
    if on_host:
        res = op.execute_columns([torch.from_numpy(k).pin_memory()], {"v": torch.from_numpy(v).pin_memory()})
    else:
        res = op.execute_columns([_cuda(k)], {"v": _cuda(v)})
    _check(res, ok, os_)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]


def test_config1_cut_then_aggregate_launches():
    """BASELINE config 1 through the default path: the whole run generation is
    the cut scan + one per-cycle-run launch (plus the wide merge), not a few
    launches per fill cycle; the ledger equals the C oracle's."""
    w = workloads.config1(device="cpu")
    keys_np = [k.numpy() for k in w.keys]
    slots = oracle.make_states(w.schema, {k: v.numpy() for k, v in w.values.items()}, w.rows)
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(w.schema), 4096, 100)
    op = _oracle_case(w, 4096, page=100)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]
    assert op.device_ledger["kernel_launches"] < 100


@pytest.mark.parametrize("cfg,rows,memory,window", [(5, 3_000_000, 1 << 14, 50_000), (3, 2_000_000, 1 << 14, 40_000),
                                                    (1, 1_000_000, 4096, 20_000), (5, 3_000_000, 1 << 18, 0)])
@pytest.mark.parametrize("dense", ["0", "1"])
def test_streamed_host_output_vs_oracle(cfg, rows, memory, window, dense, monkeypatch):
    """Host input that spills: the wide merge writes every window's groups
    into caller-owned pinned columns (isa_set_output_allocator) while the next
    window merges; the columns equal the oracle and the device-input result,
    and the result is reported as streamed."""
    monkeypatch.setenv("ISA_TILE_MERGE", "0")
    monkeypatch.setenv("ISA_DENSE", dense)
    if dense == "1" and window:
        monkeypatch.setenv("ISA_DENSE_D", "8192")
    kw = {"domain": 1 << 20} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kw)
    keys_np = [k.numpy() for k in w.keys]
    slots = oracle.make_states(w.schema, {k: v.numpy() for k, v in w.values.items()}, w.rows)
    want_keys, want_slots = oracle.reference_aggregate(keys_np, slots, oracle.slot_ops(w.schema))
    op = isa.SortAggregate(w.schema, _cfg(memory, 100, merge_window_rows=window))
    first = None
    for _ in range(2):   # the second execute reuses the handle (fresh columns each time)
        res = op.execute_columns([k.pin_memory() for k in w.keys], {k: v.pin_memory() for k, v in w.values.items()})
        assert op.streamed_output
        assert all(t.device.type == "cpu" and t.is_pinned() for t in list(res.keys) + list(res.states))
        _check(res, want_keys, want_slots, rel=1e-5 if cfg == 3 else 1e-9)
        if first is not None:   # the caller owns the first result: not overwritten by the second execute
            assert all(a.data_ptr() != b.data_ptr() for a, b in zip(first.keys, res.keys))
            _check(first, want_keys, want_slots, rel=1e-5 if cfg == 3 else 1e-9)
        first = res
    res = op.execute_columns([k.cuda() for k in w.keys], {k: v.cuda() for k, v in w.values.items()})
    assert not op.streamed_output
    _check(res, want_keys, want_slots, rel=1e-5 if cfg == 3 else 1e-9)


def test_streamed_host_output_falls_back_when_the_estimate_is_short(monkeypatch):
    """Long fill cycles first (few keys), then all-distinct keys: the output
    estimate from the mean fill cycle is far below the real group count, the
    streamed columns are too small, and the operator falls back to
    isa_result_copy -- same result."""
    monkeypatch.setenv("ISA_TILE_MERGE", "0")
    monkeypatch.setenv("ISA_DENSE", "0")
    rng = np.random.default_rng(11)
    n1, n2, memory = 2_000_000, 400_000, 1 << 12
    k = np.concatenate([rng.integers(0, memory + 40, n1), (1 << 20) + rng.permutation(n2)]).astype(np.int64)
    v = rng.integers(0, 1000, len(k)).astype(np.int64)
    sch = _cut_schema()
    slots = oracle.make_states(sch, {"v": v}, len(k))
    want_keys, want_slots = oracle.reference_aggregate([k], slots, oracle.slot_ops(sch))
    op = isa.SortAggregate(sch, _cfg(memory, 100, merge_window_rows=30_000))
    res = op.execute_columns([torch.from_numpy(k).pin_memory()], {"v": torch.from_numpy(v).pin_memory()})
    _check(res, want_keys, want_slots)
    assert not op.streamed_output
    monkeypatch.setenv("ISA_STREAM_OUT", "0")   # the allocator path switched off: identical
    op2 = isa.SortAggregate(sch, _cfg(memory, 100, merge_window_rows=30_000))
    res2 = op2.execute_columns([torch.from_numpy(k).pin_memory()], {"v": torch.from_numpy(v).pin_memory()})
    _check(res2, want_keys, want_slots)


def _phase_ms(op, name):
    from paper_2010_00152_b200 import _native
    return _native.phases_dict(op.phase_snapshot())[name]["ms"]


@pytest.mark.parametrize("case", ["cfg5", "cfg5_small_windows", "signed_minmax", "sum_only", "distinct", "raw_hbm_runs",
                                  "one_window"])
def test_dense_window_merge_vs_oracle(case, monkeypatch):
    """Dense integer keys: the wide merge accumulates every run row into a
    direct-addressed window of the key range (integer atomics) instead of
    sorting the window; groups, states and the ledger equal the oracle's, and
    no window sort runs."""
    from paper_2010_00152_b200.core import AggregateKind, AggregateSpec, ColumnSpec, Schema
    rng = np.random.default_rng(5)
    kw = {}
    if case in ("cfg5", "cfg5_small_windows", "raw_hbm_runs", "one_window"):
        w = workloads.make(5, rows=3_000_000, device="cpu", domain=1 << 20)
        sch, keys_np = w.schema, [k.numpy() for k in w.keys]
        vals_np = {k: v.numpy() for k, v in w.values.items()}
        memory = 1 << 14
        if case == "cfg5_small_windows":
            monkeypatch.setenv("ISA_DENSE_D", "4096")
        if case == "raw_hbm_runs":
            kw.update(run_tier="hbm", run_codec="raw")
        if case == "one_window":
            memory = 1 << 19
    else:
        n = 1_500_000
        k = rng.integers(-300_000, 300_000, n).astype(np.int64)
        v = rng.integers(-1_000_000, 1_000_001, n).astype(np.int64)
        keys_np, vals_np, memory = [k], {"v": v}, 1 << 13
        if case == "signed_minmax":
            sch = _cut_schema()
        elif case == "sum_only":   # no COUNT slot: occupancy bytes
            sch = Schema([ColumnSpec("k")], [AggregateSpec("s", AggregateKind.SUM, "v"),
                                             AggregateSpec("hi", AggregateKind.MAX, "v")])
        else:                      # DISTINCT: no slots at all
            sch, vals_np = Schema([ColumnSpec("k")], []), {}
        monkeypatch.setenv("ISA_DENSE_D", "16384")
    slots = oracle.make_states(sch, vals_np, len(keys_np[0]))
    want_keys, want_slots = oracle.reference_aggregate(keys_np, slots, oracle.slot_ops(sch))
    _, _, led, cycles = oracle.rsw_sortagg(keys_np, slots, oracle.slot_ops(sch), memory, 100)
    op = isa.SortAggregate(sch, _cfg(memory, 100, **kw))
    res = op.execute_columns([_cuda(k) for k in keys_np], {n_: _cuda(v) for n_, v in vals_np.items()})
    _check(res, want_keys, want_slots)
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.ledger.rows_read_back == led["rows_spilled"]
    assert op.runs_after_generation == led["runs"] and op.runs_after_generation > 1
    assert _phase_ms(op, "wm_sort") == 0 and _phase_ms(op, "wm_collapse") > 0
    if case == "cfg5_small_windows":
        assert op.device_ledger["merge_windows"] >= 200
    if case == "one_window":
        assert op.device_ledger["merge_windows"] == 1
    monkeypatch.setenv("ISA_DENSE", "0")   # the sort-based windows give the same columns
    op2 = isa.SortAggregate(sch, _cfg(memory, 100, **kw))
    res2 = op2.execute_columns([_cuda(k) for k in keys_np], {n_: _cuda(v) for n_, v in vals_np.items()})
    for a, b in zip(list(res.keys) + list(res.states), list(res2.keys) + list(res2.states)):
        assert torch.equal(a, b)
    assert _phase_ms(op2, "wm_sort") > 0


def test_dense_window_merge_not_for_sparse_or_float(monkeypatch):
    """Sparse keys (hashed) and float aggregates keep the sort-based windows."""
    w = workloads.make(3, rows=1_000_000, device="cpu", domain=1 << 20)   # hashed int64 keys, float sums
    op = _oracle_case(w, 1 << 14, page=100, rel=1e-5)
    assert _phase_ms(op, "wm_sort") > 0


@pytest.mark.parametrize("case", ["fits_int32", "one_wide_value", "carry_off", "wide_keys"])
def test_carried_values_through_the_sort(case, monkeypatch):
    """Fill cycles above 2^20 rows with one int64 value column: the values
    (narrowed to int32) ride through the packed radix passes and the collapse
    reads them in sorted order; a value outside int32 falls back to the
    gather from the column, keys spanning more than 32 bits to the gather from
    the int32 copy.  Output and ledger equal the oracles either way."""
    rng = np.random.default_rng(21)
    n, memory = 5_000_000, 1 << 21
    k = rng.integers(0, 1 << 22, n).astype(np.int64)
    if case == "wide_keys":
        k = k * ((1 << 40) + 12345)   # order-preserving spread: 62 varying bits, no packed passes
    v = rng.integers(-1_000_000, 1_000_001, n).astype(np.int64)
    if case == "one_wide_value":
        v[n // 3] = 1 << 40
    monkeypatch.setenv("ISA_CARRY", "0" if case == "carry_off" else "1")   # opt-in path under test
    sch = _cut_schema()
    slots = oracle.make_states(sch, {"v": v}, n)
    want_keys, want_slots = oracle.reference_aggregate([k], slots, oracle.slot_ops(sch))
    _, _, led, cycles = oracle.rsw_sortagg([k], slots, oracle.slot_ops(sch), memory, 100)
    op = isa.SortAggregate(sch, _cfg(memory, 100))
    res = op.execute_columns([_cuda(k)], {"v": _cuda(v)})
    _check(res, want_keys, want_slots)
    assert op.cycles == [c for c in cycles if c > 0] and min(op.cycles) > (1 << 20)
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]


@pytest.mark.parametrize("memory", [64, 4096])
def test_assumed_sort_mask_widens_mid_input(memory):
    """Chunks are sorted on the varying key bits of the execute's earlier
    chunks without reading their own mask back first; a chunk whose keys vary
    in further bits (here: the key range jumps by 2^40, twice) is detected at
    the flush analysis's synchronization and sorted again.  Output and ledger
    equal the oracles."""
    rng = np.random.default_rng(3)
    parts = [rng.integers(0, 1 << 12, 150_000), (1 << 40) + rng.integers(0, 1 << 12, 150_000),
             rng.integers(0, 1 << 50, 100_000), rng.integers(0, 1 << 12, 100_000)]
    k = np.concatenate(parts).astype(np.int64)
    v = rng.integers(-1000, 1000, len(k)).astype(np.int64)
    sch = _cut_schema()
    slots = oracle.make_states(sch, {"v": v}, len(k))
    want_keys, want_slots = oracle.reference_aggregate([k], slots, oracle.slot_ops(sch))
    _, _, led, cycles = oracle.rsw_sortagg([k], slots, oracle.slot_ops(sch), memory, min(100, memory // 2))
    op = isa.SortAggregate(sch, _cfg(memory, min(100, memory // 2)))
    res = op.execute_columns([_cuda(k)], {"v": _cuda(v)})
    _check(res, want_keys, want_slots)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]


@pytest.mark.parametrize("collide", [False, True])
def test_partial_key_sort_of_wide_keys(collide):
    """64-bit keys whose every bit varies are sorted on their top 48 bits in
    chunks of >= 2^20 rows; distinct keys that share those bits and arrive out
    of order (planted here: pairs differing in the low 16 bits only) are caught
    by the check pass and the chunk is sorted again on every bit."""
    rng = np.random.default_rng(17)
    n, memory = 3_000_000, 1 << 21
    base = rng.integers(-(1 << 62), 1 << 62, 400_000).astype(np.int64)
    k = base[rng.integers(0, len(base), n)]
    if collide:
        idx = rng.integers(0, n, 5000)
        k[idx] = (k[idx] & ~np.int64(0xFFFF)) | rng.integers(0, 1 << 16, len(idx)).astype(np.int64)
        k[(idx + 7) % n] = (k[idx] & ~np.int64(0xFFFF)) | rng.integers(0, 1 << 16, len(idx)).astype(np.int64)
    v = rng.integers(-1000, 1000, n).astype(np.int64)
    sch = _cut_schema()
    slots = oracle.make_states(sch, {"v": v}, n)
    want_keys, want_slots = oracle.reference_aggregate([k], slots, oracle.slot_ops(sch))
    _, _, led, cycles = oracle.rsw_sortagg([k], slots, oracle.slot_ops(sch), memory, 100)
    op = isa.SortAggregate(sch, _cfg(memory, 100))
    res = op.execute_columns([_cuda(k)], {"v": _cuda(v)})
    _check(res, want_keys, want_slots)
    assert op.cycles == [c for c in cycles if c > 0]
    assert op.ledger.rows_spilled == led["rows_spilled"] and op.runs_after_generation == led["runs"]


def test_dense_merge_direct_output_falls_back_when_the_estimate_is_short(monkeypatch):
    """Device input, dense keys: the dense-window merge emits into the
    caller's columns, sized after the first window.  Here the first window is
    nearly empty and the rest of the key range is full, so the columns are too
    small: the merge runs again into the result table and the result is read
    with isa_result_copy -- same groups."""
    monkeypatch.setenv("ISA_DENSE_D", "4096")
    rng = np.random.default_rng(9)
    n, memory = 1_200_000, 1 << 13
    lowk = rng.integers(0, 4096, 8).astype(np.int64)   # 8 keys in the first window
    k = np.concatenate([lowk, rng.integers(4096, 4096 + (1 << 18), n)]).astype(np.int64)
    k = k[rng.permutation(len(k))]
    v = rng.integers(-1000, 1000, len(k)).astype(np.int64)
    sch = _cut_schema()
    slots = oracle.make_states(sch, {"v": v}, len(k))
    want_keys, want_slots = oracle.reference_aggregate([k], slots, oracle.slot_ops(sch))
    op = isa.SortAggregate(sch, _cfg(memory, 100))
    res = op.execute_columns([_cuda(k)], {"v": _cuda(v)})
    _check(res, want_keys, want_slots)
    assert _phase_ms(op, "wm_sort") == 0
    monkeypatch.setenv("ISA_DIRECT_OUT", "0")   # result table + export: identical
    op2 = isa.SortAggregate(sch, _cfg(memory, 100))
    res2 = op2.execute_columns([_cuda(k)], {"v": _cuda(v)})
    for a, b in zip(list(res.keys) + list(res.states), list(res2.keys) + list(res2.states)):
        assert torch.equal(a, b)
