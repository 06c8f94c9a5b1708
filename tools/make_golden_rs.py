"""Replacement-selection fixtures (tests/golden/rs_*.npz) made by running the
REFERENCE (/root/reference/pkg/src/insortagg, this container only) with
run_generation_mode=REPLACEMENT_SELECTION + wide merge: output rows, run
sizes, ledger, the OutputEstimator's steady-probe totals and the merge plan.

Usage: python tools/make_golden_rs.py
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT, _kind, _ref, uniform_planted  # noqa: E402


def run_rs(key, aggs, values, memory, page, chunk=None):
    core, sortagg, runstore = _ref()
    schema = core.Schema([core.ColumnSpec("k0")], [core.AggregateSpec(n, _kind(kd), c) for n, kd, c in aggs])
    keys = np.asarray(key).astype(np.int64).tolist()
    vl = {nm: np.asarray(v).tolist() for nm, v in values.items()}
    rows = [core.Row((keys[i],), schema.make_state(tuple(vl[c][i] if c is not None else None for _, _, c in aggs))
                     if aggs else ()) for i in range(len(keys))]
    cfg = sortagg.SortAggConfig(memory_budget=memory, page_capacity=page, ovc_enabled=False,
                                run_generation_mode=sortagg.REPLACEMENT_SELECTION, eviction_chunk=chunk)
    runs, _ix, est, _seen = sortagg.index_run_generation(iter(rows), schema, cfg, runstore.MemoryStore(),
                                                         runstore.RowCodec(schema), core.MetricsLedger())
    op = sortagg.SortAggregate(schema, cfg, runstore.MemoryStore())
    t0 = time.time()
    out = op.execute(iter(rows))
    res = {
        "n_groups": np.int64(len(out)),
        "run_rows": np.asarray([m.row_count for m in runs], dtype=np.int64),
        "steady": np.asarray([est.steady_probes, est.steady_absorbs, est.steady_resident_sum], dtype=np.int64),
        "ledger_rows_spilled": np.int64(op.ledger.rows_spilled),
        "ledger_pages_written": np.int64(op.ledger.pages_written),
        "runs_after_generation": np.int64(op.runs_after_generation),
        "plan_kinds": np.asarray([s.kind for s in op.initial_plan.steps] if op.initial_plan else [], dtype="U16"),
        "ref_seconds": np.float64(time.time() - t0),
        "out_k0": np.asarray([r.key[0] for r in out], dtype=np.int64),
    }
    for s in range(schema.state_slots):
        res[f"out_s{s}"] = np.asarray([r.state[s] for r in out], dtype=np.int64)
    return res


def save(name, spec, key, aggs, values, memory, page, chunk=None):
    res = run_rs(key, aggs, values, memory, page, chunk)
    payload = dict(res)
    payload.update({"spec": np.asarray(spec, dtype="U256"), "memory_budget": np.int64(memory),
                    "page_capacity": np.int64(page), "eviction_chunk": np.int64(chunk or 0),
                    "aggs": np.asarray([f"{n}:{k}:{c or ''}" for n, k, c in aggs], dtype="U64"),
                    "n_key_cols": np.int64(1), "value_names": np.asarray(sorted(values), dtype="U32"),
                    "in_k0": np.asarray(key)})
    for nm, v in values.items():
        payload[f"in_v_{nm}"] = np.asarray(v)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **payload)
    print(f"{name}: rows={len(key)} groups={int(res['n_groups'])} runs={list(res['run_rows'][:6])}... "
          f"({len(res['run_rows'])}) steady={list(res['steady'])} plan={list(res['plan_kinds'])} "
          f"ref {float(res['ref_seconds']):.1f}s")


def main():
    rng = np.random.default_rng(2010001553)
    agg4 = [("n", "count", None), ("s", "sum", "v"), ("lo", "min", "v"), ("hi", "max", "v")]
    # the reference's own RS test shape (test_sortagg.py:74-84): distinct random keys
    k = rng.integers(0, 10**9, 40_000)
    save("rs_distinct_500_50", "RS: 40000 random keys, M=500, P=50 (test_sortagg.py:74-84 shape)", k,
         [("n", "count", None)], {}, 500, 50)
    # duplicates: keys planted over 3000 values, aggregates
    k = uniform_planted(rng, 30_000, 3000) * 13 - 5000
    v = rng.integers(-10**6, 10**6, len(k))
    save("rs_dups_256_32", "RS: 30000 rows / 3000 keys, count/sum/min/max, M=256, P=32", k, agg4, {"v": v}, 256, 32)
    # an explicit eviction chunk different from the page capacity
    k = uniform_planted(rng, 20_000, 5000)
    v = rng.integers(0, 1000, len(k))
    save("rs_chunk_300_10_c7", "RS: 20000 rows / 5000 keys, M=300, P=10, eviction_chunk=7", k,
         [("n", "count", None), ("s", "sum", "v")], {"v": v}, 300, 10, chunk=7)
    # skewed (Zipf-like) keys: heavy hitters stay resident
    ranks = np.minimum(rng.zipf(1.3, 40_000), 1 << 20)
    k = (ranks * 2654435761) % (1 << 40)
    save("rs_zipf_1000_100", "RS: 40000 Zipf(1.3) keys hashed, count, M=1000, P=100", k, [("n", "count", None)], {},
         1000, 100)
    # output fits: no spill
    k = uniform_planted(rng, 5000, 400)
    save("rs_nospill_512_64", "RS: 5000 rows / 400 keys, M=512 (no spill)", k, [("n", "count", None)], {}, 512, 64)


if __name__ == "__main__":
    main()
