"""Where does configs[1]'s per-step time go outside the absorb kernel?"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads, _native
w = workloads.make(2, device="cuda")
op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100))
for _ in range(3):
    op.execute_columns(w.keys, w.values)
torch.cuda.synchronize()
import cProfile, pstats
t0 = time.perf_counter()
for _ in range(20):
    op.execute_columns(w.keys, w.values)
torch.cuda.synchronize()
print("wall per step ms", (time.perf_counter() - t0) / 20 * 1e3)
d = op.device_ledger
print("host_sync ms", d["ms_host_sync"], "rungen ms", d["ms_run_generation"], "launches", d["kernel_launches"], "chunks", d["chunks"])
print({k: (round(v["ms"], 3), v["calls"]) for k, v in op.phase_stats.items() if v["calls"]})
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    op.execute_columns(w.keys, w.values)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
