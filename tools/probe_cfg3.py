"""Host/device time split of one config-3 execute (diagnostics)."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = workloads.make(c, device="cuda")
tier = sys.argv[2] if len(sys.argv) > 2 else "host"
pre = sys.argv[4] if len(sys.argv) > 4 else "auto"
op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100, run_tier=tier,
                                                  preaggregate=pre))
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    op.execute_columns(w.keys, w.values)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    d = op.device_ledger
    print(f"step {i}: wall {1e3*(t1-t0):.1f} ms  rungen(host) {d['ms_run_generation']:.1f}  wm(host) {d['ms_wide_merge']:.1f}  "
          f"host_sync {d['ms_host_sync']:.1f}  chunks {d['chunks']}  launches {d['kernel_launches']}")
    print("   phases", {k: round(v['ms'], 1) for k, v in op.phase_stats.items() if v['ms']}, {k: v['calls'] for k, v in op.phase_stats.items() if v['calls']})
