"""Host-side overhead of one configs[1] execute_columns call: wall time of
the whole call vs the time spent inside the native isa_execute."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads, _native

w = workloads.make(2, device="cuda")
op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100))
inner = []
orig = _native.Handle.execute


def timed(self, *a, **k):
    t0 = time.perf_counter()
    r = orig(self, *a, **k)
    inner.append(time.perf_counter() - t0)
    return r


_native.Handle.execute = timed
for _ in range(5):
    op.execute_columns(w.keys, w.values)
torch.cuda.synchronize()
inner.clear()
N = 50
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
s.record()
for _ in range(N):
    op.execute_columns(w.keys, w.values)
e.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
print(f"per call: wall {wall:.3f} ms, device events {s.elapsed_time(e) / N:.3f} ms, inside isa_execute "
      f"{sum(inner) / N * 1e3:.3f} ms, outside {wall - sum(inner) / N * 1e3:.3f} ms")
d = op.device_ledger
print("rungen ms (host clock)", d["ms_run_generation"], "launches", d["kernel_launches"], "chunks", d["chunks"])
print({k: (round(v["ms"], 4), v["calls"]) for k, v in op.phase_stats.items() if v["calls"]})
