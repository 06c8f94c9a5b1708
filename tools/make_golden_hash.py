"""HashAggregate fixtures (tests/golden/hash_*.npz) made by running the
REFERENCE's HashAggregate (hashagg.py) in this container: output rows in the
reference's order, ledger hash/column counters, partitions.

Usage: python tools/make_golden_hash.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT, REF, _kind, uniform_planted  # noqa: E402


def run_hash(keys, aggs, values, memory, page, hint=None):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from insortagg import core, hashagg, runstore
    k = len(keys)
    schema = core.Schema([core.ColumnSpec(f"k{i}") for i in range(k)],
                         [core.AggregateSpec(n, _kind(kd), c) for n, kd, c in aggs])
    cols = [np.asarray(c).astype(np.int64).tolist() for c in keys]
    vl = {nm: np.asarray(v).tolist() for nm, v in values.items()}
    rows = [core.Row(tuple(c[i] for c in cols),
                     schema.make_state(tuple(vl[c][i] if c is not None else None for _, _, c in aggs)) if aggs else ())
            for i in range(len(cols[0]))]
    cfg = hashagg.HashAggConfig(memory_budget=memory, page_capacity=page, output_size_hint=hint)
    op = hashagg.HashAggregate(schema, cfg, runstore.MemoryStore())
    out = op.execute(rows)
    res = {"n_groups": np.int64(len(out)), "n_partitions": np.int64(len(op.partitions)),
           "ledger_hash_computations": np.int64(op.ledger.hash_computations),
           "ledger_column_value_accesses": np.int64(op.ledger.column_value_accesses),
           "ledger_rows_spilled": np.int64(op.ledger.rows_spilled)}
    for j in range(k):
        res[f"out_k{j}"] = np.asarray([r.key[j] for r in out], dtype=np.int64).astype(np.asarray(keys[j]).dtype)
    for s in range(schema.state_slots):
        col = [r.state[s] for r in out]
        res[f"out_s{s}"] = np.asarray(col, dtype=np.float64 if any(isinstance(v, float) for v in col) else np.int64)
    return res


def save(name, spec, keys, aggs, values, memory, page, hint=None):
    res = run_hash(keys, aggs, values, memory, page, hint)
    payload = dict(res)
    payload.update({"spec": np.asarray(spec, dtype="U256"), "memory_budget": np.int64(memory),
                    "page_capacity": np.int64(page), "n_key_cols": np.int64(len(keys)),
                    "aggs": np.asarray([f"{n}:{k}:{c or ''}" for n, k, c in aggs], dtype="U64"),
                    "value_names": np.asarray(sorted(values), dtype="U32")})
    for j, c in enumerate(keys):
        payload[f"in_k{j}"] = np.asarray(c)
    for nm, v in values.items():
        payload[f"in_v_{nm}"] = np.asarray(v)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **payload)
    print(f"{name}: rows={len(keys[0])} groups={int(res['n_groups'])} partitions={int(res['n_partitions'])} "
          f"hash={int(res['ledger_hash_computations'])} cols={int(res['ledger_column_value_accesses'])}")


def main():
    rng = np.random.default_rng(2010001554)
    agg4 = [("n", "count", None), ("s", "sum", "v"), ("lo", "min", "v"), ("hi", "max", "v")]
    k = uniform_planted(rng, 20_000, 1500) * 31 - 7000
    v = rng.integers(-10**6, 10**6, len(k))
    save("hash_inmem_4096", "HashAggregate in memory: 20000 rows / 1500 keys, count/sum/min/max, M=4096",
         [k], agg4, {"v": v}, 4096, 64)
    ids = uniform_planted(rng, 12_000, 900)
    c0 = (ids % 5 - 2).astype(np.int8)
    c1 = (ids // 5 * 3).astype(np.int32)
    w = rng.uniform(0, 100, len(ids))
    save("hash_composite_avg", "HashAggregate in memory: (int8, int32) keys, count + avg(float), M=2048",
         [c0, c1], [("n", "count", None), ("a", "avg", "w")], {"w": w}, 2048, 64)
    k = uniform_planted(rng, 30_000, 6000)
    save("hash_spill_1000", "HashAggregate partitioned: 30000 rows / 6000 keys, count, M=1000 (output set only)",
         [k], [("n", "count", None)], {}, 1000, 50)


if __name__ == "__main__":
    main()
