"""Step time vs the wide-merge window capacity (diagnostics). Args: cfg rows W..."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads
c, rows = int(sys.argv[1]), int(float(sys.argv[2]))
w = workloads.make(c, device="cuda", **({"rows": rows} if rows else {}))
for W in [int(float(x)) for x in sys.argv[3:]]:
    op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100,
                                                      merge_window_rows=W))
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        op.execute_columns(w.keys, w.values)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    ph = op.phase_stats
    print(f"cfg{c} W={W}: {1e3*(t1-t0):.1f} ms windows {op.device_ledger['merge_windows']} "
          f"rungen {ph['run_generation']['ms']:.1f} wide {ph['wide_merge']['ms']:.1f}")
    op.close()
