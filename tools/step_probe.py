#!/usr/bin/env python
"""Per-step split of one config's execute_columns calls: event time of the
whole call, the engine's run-generation / wide-merge device phases, its host
timers, and the rest (output allocation + export).  usage:
python tools/step_probe.py [config] [rows] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_00152_b200 as isa  # noqa: E402
from paper_2010_00152_b200 import _native, workloads  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rows = int(float(sys.argv[2])) if len(sys.argv) > 2 else workloads.FULL_ROWS[cfgno]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
w = workloads.make(cfgno, rows=rows, device="cuda")
op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=workloads.PAGE,
                                                   run_tier="host" if cfgno == 3 else "auto"))
res = None
for i in range(steps):
    res = None
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    res = op.execute_columns(w.keys, w.values)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    ph = _native.phases_dict(op.phase_snapshot())
    led = op.device_ledger
    print(f"step {i}: events {e0.elapsed_time(e1):8.1f} ms  wall {wall:8.1f}  run_gen {ph['run_generation']['ms']:7.1f}  "
          f"wide_merge {ph['wide_merge']['ms']:7.1f}  host: run_gen {led.get('ms_run_generation', 0):7.1f} "
          f"wide {led.get('ms_wide_merge', 0):7.1f} sync {led.get('ms_host_sync', 0):7.1f}  "
          f"free before {free0 / 2**30:6.1f} GiB  torch reserved {torch.cuda.memory_reserved() / 2**30:6.1f} GiB", flush=True)
