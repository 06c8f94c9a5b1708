"""Where the ~60 us of host time around isa_execute goes (configs[1])."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads, _native, sortagg

w = workloads.make(2, device="cuda")
op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100))
T = {}


def timed(name, fn):
    def f(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return f


sortagg.SortAggregate._prepare = timed("prepare", sortagg.SortAggregate._prepare)
sortagg.SortAggregate._record = timed("record", sortagg.SortAggregate._record)
_native.Handle.execute = timed("native_execute", _native.Handle.execute)
_native.Handle.result_copy = timed("native_result_copy", _native.Handle.result_copy)
_empty = torch.empty
torch.empty = timed("torch_empty", _empty)
for _ in range(5):
    op.execute_columns(w.keys, w.values)
torch.cuda.synchronize()
T.clear()
N = 100
t0 = time.perf_counter()
for _ in range(N):
    op.execute_columns(w.keys, w.values)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / N * 1e6
print(f"per call {tot:.1f} us:", {k: round(v / N * 1e6, 1) for k, v in T.items()})
