"""Step time of one config vs the run-generation chunk cap (diagnostics)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads
c = int(sys.argv[1])
w = workloads.make(c, device="cuda")
for cap in [int(x) for x in sys.argv[2:]]:
    op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100,
                                                      chunk_rows_max=cap))
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        op.execute_columns(w.keys, w.values)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"cfg{c} chunk cap {cap}: {1e3*(t1-t0):.1f} ms chunks {op.device_ledger['chunks']}",
          {k: round(v['ms'], 1) for k, v in op.phase_stats.items() if v['ms']})
    op.close()
