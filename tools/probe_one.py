"""One execute of a config (diagnostics / ncu launch lists).  Args: cfg rows"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads
c = int(sys.argv[1])
kw = {"rows": int(float(sys.argv[2]))} if len(sys.argv) > 2 else {}
w = workloads.make(c, device="cuda", **kw)
op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100))
op.execute_columns(w.keys, w.values)
torch.cuda.synchronize()
print("ok", {k: round(v["ms"], 1) for k, v in op.phase_stats.items() if v["ms"]})
