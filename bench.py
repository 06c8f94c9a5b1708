#!/usr/bin/env python
"""Benchmark of the B200 sort-based grouping / aggregation operator.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N --steps K --warmup W --config C --impl b200|reference]

* A step = one SortAggregate.execute_columns over the whole synthetic
  workload of BASELINE.json config C (default C = 2, i.e. configs[1], the
  tiny-output grouping quoted at 1 GPU; configs[0] is the reference's own
  CPU case).  Inputs are resident in HBM before the timed region; they are
  larger than the 126 MB L2, so no flush is needed between steps.
* value = input rows/s of the whole job (all ranks), max over ranks of the
  device time (CUDA events on the launching stream, barrier + synchronize on
  both sides).  e2e = the same metric through the public API with HOST
  (pinned) input buffers, H2D of the input and D2H of the result inside the
  timed region.
* roofline = the dominant kernel's algorithmic bytes per launch / its mean
  launch duration (CUDA events inside the library), against the measured HBM
  copy bandwidth in MEASURED_PEAKS.json.  step_roofline = the minimum-traffic
  step time (B_in + B_out) / BW_HBM (+ spill bytes / link BW when runs go to
  the host tier) over the measured step time; spill bytes are the
  algorithmic ones (spilled rows x row bytes, written and read back).  Runs
  cross PCIe bit-packed, so b_link_moved / frac_moved restate the bound with
  the bytes that actually moved.
* cpu_baseline = the oracle port (oracle/rsw_oracle.c: read-sort-write run
  generation + wide merge, key-range partitioned over all host threads) on a
  bounded sample of the same workload, rank 0 at N = 1.
* --impl reference: the reference algorithm's CPU implementation (the same
  oracle port, since the reference is pure Python and cannot be compiled)
  timed alone on the host cores; same metric/config/unit.
Multi-GPU (torchrun, N > 1): weak scaling, every rank holds a shard of the
same per-GPU size; rows are range-partitioned by sampled splitters and
exchanged with NCCL all-to-all (paper_2010_00152_b200/parallel.py).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input rows/s and fraction of HBM min-traffic roofline, group-by agg at 1/2/4/8 B200"
WORKLOAD_NAMES = {
    1: "cfg1: 1M rows u32 key / 10k groups, count/sum/min/max, M=4096",
    2: "cfg2 (configs[1]): 2^28 rows, (u8 x3, u8 x2) key = 6 groups, count + 4 f64 sums, M=4096 (no spill)",
    3: "cfg3: 1e9 rows, int64 hash(Zipf(1.1) over 2^28), count/isum/fsum/min/max, M=2^22, host spill",
    4: "cfg4: 2^29 rows, DISTINCT (u64,u64), 2^27 pairs x4, M=2^24, host spill",
    5: "cfg5: int64 U[0,2^30) key, count+sum, M=2^24 per GPU",
}


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    p.add_argument("--rows", type=int, default=None, help="rows per GPU (default: the config's full size)")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--run-tier", default=None, choices=[None, "host", "hbm"])
    p.add_argument("--cpu-sample-rows", type=int, default=None)
    return p.parse_args()


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _link_gbs(torch, dev):
    """pinned H2D bandwidth, measured (spill/readback link roofline)."""
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize(dev)
    return 3 * n / (s.elapsed_time(e) / 1e3) / 1e9


def _cpu_baseline(w, sample_rows, threads):
    """Oracle port over a bounded sample of the workload on `threads` cores."""
    import numpy as np

    import oracle
    n = min(w.rows, sample_rows)
    keys = [k[:n].cpu().numpy() for k in w.keys]
    vals = {nm: v[:n].cpu().numpy() for nm, v in w.values.items()}
    slots = oracle.make_states(w.schema, vals, n)
    ops = oracle.slot_ops(w.schema)
    sp = oracle.range_splitters(keys, threads) if threads > 1 else None
    t0 = time.perf_counter()
    out_keys, _, _, _ = oracle.rsw_sortagg(keys, slots, ops, w.memory_budget, 100, nthreads=threads, splitters=sp)
    secs = time.perf_counter() - t0
    del np
    return n / secs, n, secs, len(out_keys[0])


def run_reference(args):
    """--impl reference: the reference algorithm on the host cores."""
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    import torch
    from paper_2010_00152_b200 import workloads
    rows = args.rows or workloads.FULL_ROWS[args.config]
    threads = os.cpu_count() or 1
    # bounded sample: the oracle port runs ~40-80 M rows/s/thread on cfg2-like data
    sample = args.cpu_sample_rows or min(rows, {1: rows, 2: 64 << 20, 3: 32 << 20, 4: 16 << 20, 5: 32 << 20}[args.config])
    w = workloads.make(args.config, rows=sample, device="cpu")
    vals = []
    for _ in range(max(0, args.warmup)):
        pass  # the CPU port has no warm-up state beyond page faults; one untimed run below
    _cpu_baseline(w, min(sample, 1 << 20), threads)
    for _ in range(args.steps):
        v, n, secs, groups = _cpu_baseline(w, sample, threads)
        vals.append((v, secs))
    value = sum(v for v, _ in vals) / len(vals)
    ms = sum(s for _, s in vals) / len(vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic (seeded, BASELINE shapes)",
        "config": {"workload": WORKLOAD_NAMES[args.config], "rows_per_step": sample, "parallelism": "cpu threads"},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "port",
                         "sample": f"first {sample} rows of the seeded workload (cpu generator), "
                                   f"oracle/rsw_oracle.c key-range partitioned over {threads} threads"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    del torch
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2010_00152_b200 as isa
    from paper_2010_00152_b200 import _native, workloads

    world, rank, local = _dist()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfgno = args.config
    rows = args.rows or workloads.FULL_ROWS[cfgno]
    gen_kw = {"seed": workloads.SEED + cfgno + 1000 * rank} if world > 1 else {}
    w = workloads.make(cfgno, rows=rows, device=dev, **gen_kw)
    run_tier = args.run_tier or "host"
    cfg = isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=workloads.PAGE, run_tier=run_tier)
    op = isa.SortAggregate(w.schema, cfg)
    if world > 1:
        from paper_2010_00152_b200 import parallel
        mode = "preaggregate" if cfgno in (1, 2) else "partition"

        def step():
            return parallel.distributed_execute(op, w.keys, w.values, mode=mode)
    else:
        def step():
            return op.execute_columns(w.keys, w.values)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    args.warmup = max(3, args.warmup)   # timing rule: at least 3 untimed warm-up steps
    for _ in range(args.warmup):
        res = step()
    barrier()
    # clocks are sampled from a >= 1 s load ramp right before the timed region
    # through its end (a short timed region alone holds too few samples)
    clocks = ClockSampler(local)
    clocks.start()
    t_ramp = time.perf_counter()
    while time.perf_counter() - t_ramp < 1.0:
        res = step()
        torch.cuda.synchronize(dev)
    barrier()
    stream = torch.cuda.current_stream(dev)
    phase_tot = {}
    launches0 = _native.launch_count()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    snaps = []
    for _ in range(args.steps):
        res = step()
        snaps.append(op.phase_snapshot())   # one small native call; decoded after the timed region
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    for raw in snaps:
        if raw is None:
            continue
        for k, v in _native.phases_dict(raw).items():
            t = phase_tot.setdefault(k, {"ms": 0.0, "calls": 0, "rows": 0, "bytes": 0})
            for f in t:
                t[f] += v[f]
    launches = _native.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / max(1, args.steps)
    total_rows = rows * world
    value = total_rows / (ms_step / 1e3)
    n_groups = res.n_groups if hasattr(res, "n_groups") else None

    peak, peak_src = _peaks()
    link = _link_gbs(torch, dev)
    key_b = w.key_bytes
    val_b = w.value_bytes
    out_b = (n_groups or 0) * (key_b + 8 * w.schema.state_slots)
    b_in = rows * (key_b + val_b)
    dled = op.device_ledger or {}
    spill_rows = dled.get("rows_spilled", 0)   # last execute (every step is identical)
    spill_b = 2 * spill_rows * (key_b + 8 * w.schema.state_slots) if run_tier == "host" else 0
    t_star = (b_in + out_b) / (peak * 1e9) + spill_b / (link * 1e9)
    # the same bound with the link bytes actually moved (host-tier runs cross
    # PCIe bit-packed by the run codec, so this can be well below spill_b)
    link_b = (dled.get("bytes_d2h", 0) + dled.get("bytes_h2d", 0)) if run_tier == "host" else 0
    t_moved = (b_in + out_b) / (peak * 1e9) + link_b / (link * 1e9)
    # dominant kernel: the phase with the most device time among kernel phases
    kernel_phases = ["absorb", "sort", "collapse", "table_merge", "wm_sort", "wm_collapse", "flush"]
    dom = max(kernel_phases, key=lambda k: phase_tot.get(k, {}).get("ms", 0.0))
    dp = phase_tot.get(dom, {"ms": 0.0, "calls": 0, "rows": 0, "bytes": 0})
    if dom == "absorb":
        alg_bytes = dp["bytes"]
    else:
        # sort/merge phases: algorithmic bytes = the rows they touch x key+value bytes, read once
        alg_bytes = dp["rows"] * (key_b + val_b)
    per_launch_bytes = alg_bytes / max(1, dp["calls"])
    per_launch_ms = dp["ms"] / max(1, dp["calls"])
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tt = json.load(f).get(f"config{cfgno}")
            if tt and tt.get("phase") == dom:
                traffic = tt.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "rows/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int64/f64" if w.schema.state_slots else "u64 keys",
        "data": "synthetic (seeded generator with BASELINE.json shapes, generated on device)",
        "config": {"workload": WORKLOAD_NAMES[cfgno], "rows_per_gpu": rows, "global_rows": total_rows,
                   "groups": n_groups, "memory_budget": w.memory_budget, "page_capacity": workloads.PAGE,
                   "run_tier": run_tier, "parallelism": f"range-partitioned x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs (%.1f GB) larger than L2 (126 MB); no flush" % (b_in / 1e9)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "alg_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                     "launches_per_step": dp["calls"] / max(1, args.steps), "peak_source": peak_src},
        "step_roofline": {"t_star_ms": t_star * 1e3, "frac": (t_star * 1e3) / ms_step if ms_step else None,
                          "b_in": b_in, "b_out": out_b, "b_spill": spill_b, "link_gbs": link,
                          "hbm_gbs": peak, "b_link_moved": link_b, "t_moved_ms": t_moved * 1e3,
                          "frac_moved": (t_moved * 1e3) / ms_step if ms_step else None},
        "phases_ms_per_step": {k: v["ms"] / max(1, args.steps) for k, v in phase_tot.items() if v["ms"]},
        "ledger_per_step": {"rows_spilled": spill_rows, "runs": op.runs_after_generation,
                            "bytes_d2h": dled.get("bytes_d2h"), "bytes_h2d": dled.get("bytes_h2d"),
                            "merge_windows": dled.get("merge_windows"), "chunks": dled.get("chunks")},
        "gpu_launches": launches,
        "clocks": clk,
    }

    # end-to-end through the public API with pinned host buffers (N = 1 and N > 1 alike)
    if not args.no_e2e:
        host_keys = [k.cpu().pin_memory() for k in w.keys]
        host_vals = {n: v.cpu().pin_memory() for n, v in w.values.items()}
        op_e2e = isa.SortAggregate(w.schema, cfg)
        if world > 1:
            from paper_2010_00152_b200 import parallel

            def e2e_step():
                keys = [k.to(dev, non_blocking=True) for k in host_keys]
                vals = {n: v.to(dev, non_blocking=True) for n, v in host_vals.items()}
                r = parallel.distributed_execute(op_e2e, keys, vals, mode=mode)
                return [k.cpu() for k in r.keys] + [s.cpu() for s in r.states]
        else:
            def e2e_step():
                r = op_e2e.execute_columns(host_keys, host_vals)
                return list(r.keys) + list(r.states)
        e2e_step()
        barrier()
        k2 = args.e2e_steps or args.steps
        # device clock (CUDA events on the launching stream) around the
        # synchronous public-API calls; max over ranks below
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k2):
            outs = e2e_step()
        e1.record(stream)
        barrier()
        secs = e0.elapsed_time(e1) / 1e3 / k2
        if world > 1:
            t = torch.tensor([secs], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = float(t.item())
        d2h = sum(o.numel() * o.element_size() for o in outs)
        line["e2e"] = {"value": total_rows / secs, "unit": "rows/s", "h2d_bytes_per_step": b_in,
                       "d2h_bytes_per_step": d2h, "ms_per_step": secs * 1e3}
        del host_keys, host_vals

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = args.cpu_sample_rows or min(rows, {1: rows, 2: 64 << 20, 3: 32 << 20, 4: 16 << 20, 5: 32 << 20}[cfgno])
        wc = workloads.make(cfgno, rows=sample, device="cpu")
        v, n, secs, _ = _cpu_baseline(wc, sample, threads)
        line["cpu_baseline"] = {"value": v, "unit": "rows/s", "cores": threads, "kind": "port",
                                "sample": f"{n} rows of the same seeded workload (cpu generator), "
                                          f"oracle/rsw_oracle.c read-sort-write + wide merge, key-range "
                                          f"partitioned over {threads} threads, {secs:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
