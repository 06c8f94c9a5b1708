"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Runs /root/reference/pkg/src/insortagg (read-only, imported by path; this
container only) on seeded inputs and records its output rows, ledger,
read-sort-write fill cycles, run sizes and merge plan.  The fixtures pin both
oracles (tests/test_oracle.py) and the GPU path (tests/test_gpu_parity.py).

Reference settings: ovc_enabled=False (OVC crashes on keys
outside [0, domain) and does not change output, test_sortagg.py:340-353),
page_capacity=100 unless stated, default read-sort-write + wide merge.
Keys >= 2^63 cannot be spilled by the reference codec (runstore.py:50, 59):
uint64 columns are fed as x - 2^63 (order preserving) and mapped back.

Usage: python tools/make_golden.py [pages]   (writes tests/golden/; `pages`
only regenerates the FileStore page fixtures)
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import insortagg  # noqa: F401
    from insortagg import core, sortagg, runstore
    return core, sortagg, runstore


def _kind(name):
    core, _, _ = _ref()
    return getattr(core.AggregateKind, name.upper())


def run_reference(key_cols, aggs, values, memory, page=100, hint=None, mode="wide"):
    """key_cols: list of numpy integer arrays; aggs: [(name, kind, column)];
    values: dict column -> numpy array.  Returns dict of outputs."""
    core, sortagg, runstore = _ref()
    k = len(key_cols)
    schema = core.Schema([core.ColumnSpec(f"k{i}") for i in range(k)],
                         [core.AggregateSpec(n, _kind(kd), c) for n, kd, c in aggs])
    bias = [np.asarray(c).dtype == np.uint64 for c in key_cols]
    cols = []
    for c, b in zip(key_cols, bias):
        if b:
            cols.append((np.asarray(c).astype(np.uint64) - np.uint64(1 << 63)).view(np.int64).tolist())
        else:
            cols.append(np.asarray(c).astype(np.int64).tolist())
    n = len(key_cols[0]) if key_cols else 0
    vlists = {name: np.asarray(v).tolist() for name, v in values.items()}
    rows = []
    for i in range(n):
        key = tuple(col[i] for col in cols)
        inputs = tuple(vlists[c][i] if c is not None else None for _, _, c in aggs)
        rows.append(core.Row(key, schema.make_state(inputs) if aggs else ()))
    cfg = sortagg.SortAggConfig(memory_budget=memory, page_capacity=page, ovc_enabled=False,
                                output_size_hint=hint, merge_mode=mode)
    # run generation alone for cycles / run sizes (same deterministic input)
    store = runstore.MemoryStore()
    led0 = core.MetricsLedger()
    if mode == "wide":
        runs, _index, est, _seen = sortagg.index_run_generation(iter(rows), schema, cfg, store,
                                                                runstore.RowCodec(schema), led0)
        cycles = list(est.cycles)
    else:
        runs, _mem, _seen = sortagg.pq_run_generation(iter(rows), schema, cfg, store, runstore.RowCodec(schema), led0)
        cycles = []
    run_rows = [m.row_count for m in runs]
    op = sortagg.SortAggregate(schema, cfg, runstore.MemoryStore())
    t0 = time.time()
    out = op.execute(iter(rows))
    secs = time.time() - t0
    res = {
        "n_groups": np.int64(len(out)),
        "ledger_rows_spilled": np.int64(op.ledger.rows_spilled),
        "ledger_rows_read_back": np.int64(op.ledger.rows_read_back),
        "ledger_pages_written": np.int64(op.ledger.pages_written),
        "ledger_pages_read": np.int64(op.ledger.pages_read),
        "ledger_merge_steps": np.int64(op.ledger.merge_steps),
        "ledger_merge_levels": np.int64(op.ledger.merge_levels),
        "runs_after_generation": np.int64(op.runs_after_generation),
        "run_rows": np.asarray(run_rows, dtype=np.int64),
        "cycles": np.asarray(cycles, dtype=np.int64),
        "plan_kinds": np.asarray([s.kind for s in op.initial_plan.steps] if op.initial_plan else [], dtype="U16"),
        "plan_levels": np.int64(op.initial_plan.levels if op.initial_plan else -1),
        "executed_kinds": np.asarray([s["kind"] for s in op.executed_steps], dtype="U16"),
        "executed_fan_in": np.asarray([s["fan_in"] for s in op.executed_steps], dtype=np.int64),
        "executed_rows_out": np.asarray([s["rows_out"] for s in op.executed_steps], dtype=np.int64),
        "executed_collapsed": np.asarray([int(s.get("collapsed", True)) for s in op.executed_steps], dtype=np.int64),
        "merge_mode": np.asarray(mode, dtype="U16"),
        "ref_seconds": np.float64(secs),
    }
    for j, (c, b) in enumerate(zip(key_cols, bias)):
        vals = np.asarray([r.key[j] for r in out], dtype=np.int64)
        if b:
            vals = vals.view(np.uint64) + np.uint64(1 << 63)
        res[f"out_k{j}"] = vals.astype(np.asarray(c).dtype)
    nslots = schema.state_slots
    for s in range(nslots):
        col = [r.state[s] for r in out]
        is_f = any(isinstance(v, float) for v in col)
        res[f"out_s{s}"] = np.asarray(col, dtype=np.float64 if is_f else np.int64)
    return res


def save(name, spec, key_cols, aggs, values, memory, page=100, store_inputs=True, extra=None, hint=None, mode="wide"):
    res = run_reference(key_cols, aggs, values, memory, page, hint, mode)
    payload = dict(res)
    payload["memory_budget"] = np.int64(memory)
    payload["page_capacity"] = np.int64(page)
    payload["aggs"] = np.asarray([f"{n}:{k}:{c or ''}" for n, k, c in aggs], dtype="U64")
    payload["spec"] = np.asarray(spec, dtype="U256")
    payload["n_key_cols"] = np.int64(len(key_cols))
    payload["value_names"] = np.asarray(sorted(values), dtype="U32")
    h = hashlib.sha256()
    for c in key_cols:
        h.update(np.ascontiguousarray(c).tobytes())
    for nme in sorted(values):
        h.update(np.ascontiguousarray(values[nme]).tobytes())
    payload["input_sha256"] = np.asarray(h.hexdigest(), dtype="U64")
    if store_inputs:
        for j, c in enumerate(key_cols):
            payload[f"in_k{j}"] = np.asarray(c)
        for nme, v in values.items():
            payload[f"in_v_{nme}"] = np.asarray(v)
    if extra:
        payload.update(extra)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **payload)
    print(f"{name}: rows={len(key_cols[0])} groups={int(res['n_groups'])} spilled={int(res['ledger_rows_spilled'])} "
          f"runs={int(res['runs_after_generation'])} plan={list(res['plan_kinds'])} ref {float(res['ref_seconds']):.2f}s "
          f"-> {os.path.getsize(path) / 1024:.0f} KiB")


def save_pages(name, spec, key_cols, aggs, values, memory, page):
    """Run the reference with a FileStore and keep every run file's bytes
    (runstore.py page format) next to the inputs and the output rows."""
    import tempfile
    core, sortagg, runstore = _ref()
    k = len(key_cols)
    schema = core.Schema([core.ColumnSpec(f"k{i}") for i in range(k)],
                         [core.AggregateSpec(n, _kind(kd), c) for n, kd, c in aggs])
    cols = [np.asarray(c).astype(np.int64).tolist() for c in key_cols]
    vlists = {nm: np.asarray(v).tolist() for nm, v in values.items()}
    rows = []
    for i in range(len(key_cols[0])):
        inputs = tuple(vlists[c][i] if c is not None else None for _, _, c in aggs)
        rows.append(core.Row(tuple(col[i] for col in cols), schema.make_state(inputs)))
    cfg = sortagg.SortAggConfig(memory_budget=memory, page_capacity=page, ovc_enabled=False)
    with tempfile.TemporaryDirectory() as d:
        store = runstore.FileStore(d)
        op = sortagg.SortAggregate(schema, cfg, store)
        out = op.execute(iter(rows))
        store.close()
        # run generation's runs come first (ids 0..R-1); traditional levels the
        # reference plans before its wide step write further runs, which the
        # B200 path never needs (one wide merge)
        files = sorted(f for f in os.listdir(d) if f.startswith("run_"))[: op.runs_after_generation]
        blobs = [open(os.path.join(d, f), "rb").read() for f in files]
    payload = {
        "spec": np.asarray(spec, dtype="U256"),
        "memory_budget": np.int64(memory), "page_capacity": np.int64(page),
        "aggs": np.asarray([f"{n}:{kd}:{c or ''}" for n, kd, c in aggs], dtype="U64"),
        "run_files": np.asarray(files, dtype="U32"),
        "run_bytes": np.frombuffer(b"".join(blobs), dtype=np.uint8),
        "run_lengths": np.asarray([len(b) for b in blobs], dtype=np.int64),
        "runs_after_generation": np.int64(op.runs_after_generation),
        "executed_kinds": np.asarray([s_["kind"] for s_ in op.executed_steps], dtype="U16"),
    }
    for j, c in enumerate(key_cols):
        payload[f"in_k{j}"] = np.asarray(c)
        payload[f"out_k{j}"] = np.asarray([r.key[j] for r in out], dtype=np.int64).astype(np.asarray(c).dtype)
    for nm, v in values.items():
        payload[f"in_v_{nm}"] = np.asarray(v)
    for s_ in range(schema.state_slots):
        payload[f"out_s{s_}"] = np.asarray([r.state[s_] for r in out], dtype=np.int64)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **payload)
    print(f"{name}: {len(files)} run files, {sum(len(b) for b in blobs)} bytes -> {os.path.getsize(path) / 1024:.0f} KiB")


def pages_main():
    rng = np.random.default_rng(2010001552)
    n, o = 3000, 450
    kk = uniform_planted(rng, n, o) * 7 - 1000
    v = rng.integers(-10**6, 10**6, n)
    save_pages("pages_3000_450_64_8", "reference FileStore runs: 3000 rows / 450 int64 keys, M=64, P=8",
               [kk.astype(np.int64)], [("n", "count", None), ("s", "sum", "v"), ("lo", "min", "v"),
                                       ("hi", "max", "v")], {"v": v}, 64, 8)
    n, o = 5000, 900
    ids = uniform_planted(rng, n, o)
    c0 = (ids % 7 - 3).astype(np.int8)
    c1 = ((ids // 7) * 37 - 2000).astype(np.int16)
    c2 = (ids * 2654435761 % (1 << 32)).astype(np.uint32)
    w = rng.integers(0, 1000, n)
    save_pages("pages_composite_avg", "reference FileStore runs: (int8, int16, uint32) keys, count + avg, M=100, P=16",
               [c0, c1, c2], [("n", "count", None), ("a", "avg", "w")], {"w": w}, 100, 16)
    kd = rng.integers(0, 1 << 40, 4000)
    kd = np.concatenate([kd, kd[:2000]])
    rng.shuffle(kd)
    save_pages("pages_distinct", "reference FileStore runs: DISTINCT over int64, M=500, P=100",
               [kd.astype(np.int64)], [], {}, 500, 100)


def downstream_main():
    """bench.in_stream_aggregate / merge_intersect / sort_intersect_plan
    (bench.py:199-212, 536-569) run by the reference."""
    core, sortagg, runstore = _ref()
    import importlib
    bench = importlib.import_module("insortagg.bench")
    rng = np.random.default_rng(20100015 + 7)
    schema = core.Schema([core.ColumnSpec("k0"), core.ColumnSpec("k1")],
                         [core.AggregateSpec("n", core.AggregateKind.COUNT),
                          core.AggregateSpec("s", core.AggregateKind.SUM, "v"),
                          core.AggregateSpec("lo", core.AggregateKind.MIN, "v")])
    for name, sort_first in (("downstream_in_stream_sorted", True), ("downstream_in_stream_unsorted", False)):
        n = 20_000
        k0 = rng.integers(-50, 50, n)
        k1 = rng.integers(0, 30, n)
        v = rng.integers(-10**9, 10**9, n)
        if sort_first:
            o = np.lexsort((k1, k0))
            k0, k1, v = k0[o], k1[o], v[o]
        rows = [core.Row((int(a), int(b)), schema.make_state((None, int(x), int(x)))) for a, b, x in zip(k0, k1, v)]
        out = list(bench.in_stream_aggregate(iter(rows), schema))
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), in_k0=k0.astype(np.int8), in_k1=k1.astype(np.uint8),
                            in_v_v=v, out_k0=np.asarray([r.key[0] for r in out], dtype=np.int8),
                            out_k1=np.asarray([r.key[1] for r in out], dtype=np.uint8),
                            out_s0=np.asarray([r.state[0] for r in out], dtype=np.int64),
                            out_s1=np.asarray([r.state[1] for r in out], dtype=np.int64),
                            out_s2=np.asarray([r.state[2] for r in out], dtype=np.int64))
        print(f"{name}: {n} rows -> {len(out)} groups")
    # sort_intersect_plan over two inputs with overlapping key sets
    sch1 = core.Schema([core.ColumnSpec("k")], [core.AggregateSpec("n", core.AggregateKind.COUNT)])
    a = rng.integers(0, 30_000, 40_000)
    b = rng.integers(15_000, 60_000, 35_000)
    ra = [core.Row((int(x),), (1,)) for x in a]
    rb = [core.Row((int(x),), (1,)) for x in b]
    keys, ledgers = bench.sort_intersect_plan(ra, rb, sch1, memory_rows=4096, page_rows=64)
    np.savez_compressed(os.path.join(OUT, "downstream_intersect.npz"), in_a=a, in_b=b,
                        out_keys=np.asarray([k[0] for k in keys], dtype=np.int64),
                        rows_spilled=np.asarray([l.rows_spilled for l in ledgers], dtype=np.int64),
                        memory_rows=np.int64(4096), page_rows=np.int64(64))
    print(f"downstream_intersect: {len(a)} x {len(b)} rows -> {len(keys)} common keys")


def uniform_planted(rng, n, distinct):
    ids = np.concatenate([np.arange(distinct), rng.integers(0, distinct, n - distinct)])
    rng.shuffle(ids)
    return ids


def main():
    os.makedirs(OUT, exist_ok=True)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    from paper_2010_00152_b200 import workloads

    # config 1 at full scale, regenerated from the seeded torch generator
    w = workloads.config1(device="cpu")
    key = w.keys[0].numpy()
    val = w.values["v"].numpy()
    save("cfg1_full", "workloads.config1(device='cpu')", [key],
         [("n", "count", None), ("s", "sum", "v"), ("lo", "min", "v"), ("hi", "max", "v")], {"v": val},
         4096, store_inputs=False)

    rng = np.random.default_rng(20100015)
    # config 2 shape, scaled (no spill: O = 6 <= M), float sums
    n = 40_000
    k1 = rng.integers(0, 3, n).astype(np.uint8)
    k2 = rng.integers(0, 2, n).astype(np.uint8)
    vals = {f"f{i}": np.round(rng.uniform(0, 1e5, n), 3) for i in range(4)}
    save("cfg2_scaled", "cfg2 shape, 40k rows (values rounded to 1e-3)", [k1, k2],
         [("n", "count", None)] + [(f"sum_f{i}", "sum", f"f{i}") for i in range(4)], vals, 4096)

    # config 3 shape, scaled: Zipf(1.1) ranks over 2^16 hashed; integer aggregates (floats cannot spill in the reference)
    n = 120_000
    ranks = np.clip(np.floor((1 + rng.random(n) * ((2**16 + 1) ** -0.1 - 1)) ** (1 / -0.1)), 1, 2**16).astype(np.int64)
    with np.errstate(over="ignore"):
        x = ranks.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    key3 = x.view(np.int64)
    vi = rng.integers(0, 2**31, n)
    save("cfg3_scaled", "cfg3 shape: 120k rows, zipf over 2^16, M=8192", [key3],
         [("n", "count", None), ("isum", "sum", "vi"), ("imin", "min", "vi"), ("imax", "max", "vi")],
         {"vi": vi}, 8192)
    # config 3 with the float sum, no spill (M >= O)
    n = 30_000
    key3b = key3[:n]
    vf = rng.standard_normal(n).astype(np.float32)
    save("cfg3_float_nospill", "cfg3 shape with fp32 sum, M >= O", [key3b],
         [("n", "count", None), ("isum", "sum", "vi"), ("fsum", "sum", "vf"), ("imin", "min", "vi"),
          ("imax", "max", "vi")], {"vi": vi[:n], "vf": vf}, 16384)

    # config 4 shape, scaled: DISTINCT over (u64, u64), pairs x4 (keys >= 2^63 present)
    d = 25_000
    a = rng.integers(0, 2**64, d, dtype=np.uint64)
    b = rng.integers(0, 2**64, d, dtype=np.uint64)
    idx = np.tile(np.arange(d), 4)
    rng.shuffle(idx)
    save("cfg4_scaled", "cfg4 shape: 25k pairs x4, M=4096", [a[idx], b[idx]], [], {}, 4096)

    # config 5 shape, scaled
    n = 150_000
    key5 = rng.integers(0, 2**17, n)
    v5 = rng.integers(0, 2**20, n)
    save("cfg5_scaled", "cfg5 shape: 150k rows over 2^17, M=2048", [key5],
         [("n", "count", None), ("s", "sum", "v")], {"v": v5}, 2048)

    # edge cases
    save("edge_empty", "empty input", [np.zeros(0, dtype=np.int64)], [("n", "count", None)], {}, 64, 8)
    save("edge_single", "single row", [np.asarray([42], dtype=np.int64)],
         [("n", "count", None), ("s", "sum", "v")], {"v": np.asarray([-7])}, 64, 8)
    kk = uniform_planted(rng, 5000, 64)
    save("edge_O_eq_M", "O == M: no spill", [kk.astype(np.int64)], [("n", "count", None)], {}, 64, 8)
    kk = uniform_planted(rng, 5000, 65)
    save("edge_O_eq_M_plus_1", "O == M + 1: spill", [kk.astype(np.int64)], [("n", "count", None)], {}, 64, 8)
    save("edge_one_key", "all rows one key", [np.full(4000, -5, dtype=np.int64)],
         [("n", "count", None), ("s", "sum", "v"), ("mn", "min", "v"), ("mx", "max", "v")],
         {"v": rng.integers(-1000, 1000, 4000)}, 64, 8)
    kk = rng.integers(-(2**62), 2**62, 20_000)
    save("edge_all_distinct_signed", "all keys distinct, negative values", [kk],
         [("n", "count", None), ("s", "sum", "v")], {"v": rng.integers(-(2**40), 2**40, 20_000)}, 512, 16)
    n = 20_000
    c0 = rng.integers(-128, 128, n).astype(np.int8)
    c1 = rng.integers(-300, 300, n).astype(np.int16)
    c2 = rng.integers(-(2**40), 2**40, n) // 2**35
    save("edge_composite_signed", "(int8, int16, int64) composite key, avg", [c0, c1, c2],
         [("n", "count", None), ("a", "avg", "v"), ("mx", "max", "v")], {"v": rng.integers(-50, 50, n)}, 256, 16)
    # the reference's own end-to-end shapes (test_sortagg.py:308-324)
    for (n, o, m, p) in [(3000, 450, 64, 8), (800, 800, 64, 8), (1000, 3, 64, 8), (64, 20, 64, 8)]:
        kk = uniform_planted(rng, n, o)
        save(f"e2e_{n}_{o}_{m}_{p}", f"test_sortagg shape {(n, o, m, p)}", [kk.astype(np.int64)],
             [("n", "count", None)], {}, m, p)
    # traditional / separate merge modes (sortagg.py:379-455, 545-574, 788-849): pq run generation + fan-in levels
    for mode in ("traditional", "separate"):
        for (n, o, m, p) in [(3000, 450, 64, 8), (800, 800, 64, 8), (1000, 3, 64, 8), (64, 20, 64, 8)]:
            kk = uniform_planted(rng, n, o)
            save(f"{mode}_{n}_{o}_{m}_{p}", f"{mode} mode, test_sortagg shape {(n, o, m, p)}",
                 [kk.astype(np.int64)], [("n", "count", None)], {}, m, p, mode=mode)
        kk = uniform_planted(rng, 20_000, 1_500)
        save(f"{mode}_levels", f"{mode} mode, 20000 rows / 1500 keys, M=256, P=16 (several merge levels)",
             [kk.astype(np.int64)], [("n", "count", None), ("s", "sum", "v"), ("mn", "min", "v")],
             {"v": rng.integers(-1000, 1000, 20_000)}, 256, 16, mode=mode)
    # wide merge of many runs of a large budget (test_sortagg.py:326-338 shape)
    kk = uniform_planted(rng, 30_000, 2_500)
    save("e2e_spill_once", "30000 rows / 2500 keys, M=1000, P=10", [kk.astype(np.int64)],
         [("n", "count", None)], {}, 1000, 10)


if __name__ == "__main__":
    if sys.argv[1:] == ["pages"]:
        os.makedirs(OUT, exist_ok=True)
        pages_main()
    elif sys.argv[1:] == ["downstream"]:
        os.makedirs(OUT, exist_ok=True)
        downstream_main()
    else:
        main()
        pages_main()
        downstream_main()
