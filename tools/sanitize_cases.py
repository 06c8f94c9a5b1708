"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family of the operator on inputs that finish in
seconds under instrumentation, each result checked against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2010_00152_b200 as isa  # noqa: E402
from paper_2010_00152_b200 import workloads  # noqa: E402


def check(w, memory, **kw):
    keys_np = [k.cpu().numpy() for k in w.keys]
    slots = oracle.make_states(w.schema, {k: v.cpu().numpy() for k, v in w.values.items()}, w.rows)
    want_k, want_s = oracle.reference_aggregate(keys_np, slots, oracle.slot_ops(w.schema))
    op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=memory, page_capacity=min(100, memory // 2), **kw))
    res = op.execute_columns([k.cuda() for k in w.keys], {k: v.cuda() for k, v in w.values.items()})
    for g, e in zip(res.keys, want_k):
        assert np.array_equal(g.cpu().numpy(), e)
    for g, e in zip(res.states, want_s):
        g = g.cpu().numpy()
        if e.dtype.kind == "f":
            np.testing.assert_allclose(g, e, rtol=1e-5)
        else:
            assert np.array_equal(g, e)
    op.close()
    return op


cases = [
    (1, 60_000, 1024, {}),
    (2, 300_000, 4096, {}),                       # absorb kernel
    (3, 200_000, 4096, {"run_tier": "host"}),     # host-tier packed runs, radix windows
    (3, 200_000, 4096, {"preaggregate": "always"}),   # tile pre-aggregation
    (4, 200_000, 8192, {}),                       # 128-bit keys, tile merge
    (5, 300_000, 4096, {}),                       # HBM-tier packed runs
]
only = sys.argv[1:] or None
for i, (cfg, rows, memory, kw) in enumerate(cases):
    if only and str(i) not in only:
        continue
    kwg = {"domain": 1 << 16} if cfg in (3, 5) else {}
    w = workloads.make(cfg, rows=rows, device="cpu", **kwg)
    check(w, memory, **kw)
    print(f"case {i}: config {cfg} rows {rows} M {memory} {kw} OK", flush=True)
os.environ["ISA_TILE_MERGE"] = "1"
w = workloads.make(5, rows=300_000, device="cpu", domain=1 << 16)
check(w, 4096)
print("tile merge (config 5) OK", flush=True)
os.environ["ISA_TILE_MERGE"] = "0"
w = workloads.make(3, rows=100_000, device="cpu", domain=1 << 14)
check(w, 512, run_generation_mode=isa.REPLACEMENT_SELECTION, eviction_chunk=16)
print("replacement selection OK", flush=True)
check(w, 2048, hot_absorb="always")
print("hash-image absorb OK", flush=True)
os.environ["ISA_SEQ"] = "1"
w = workloads.make(1, rows=100_000, device="cpu")
check(w, 1024)
print("one-CTA read-sort-write OK", flush=True)
w = workloads.make(3, rows=200_000, device="cpu", domain=1 << 14)
op = isa.HashAggregate(w.schema, isa.HashAggConfig(memory_budget=4096, page_capacity=64))
res = op.execute_columns([k.cuda() for k in w.keys], {k: v.cuda() for k, v in w.values.items()})
slots = oracle.make_states(w.schema, {k: v.numpy() for k, v in w.values.items()}, w.rows)
want_k, _ = oracle.reference_aggregate([k.numpy() for k in w.keys], slots, oracle.slot_ops(w.schema))
assert np.array_equal(np.sort(res.keys[0].cpu().numpy()), want_k[0])
print("hash aggregate OK", flush=True)
