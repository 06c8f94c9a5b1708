#!/usr/bin/env python
"""Benchmark of the B200 sort-based grouping / aggregation operator.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N --steps K --warmup W --config C --impl b200|reference]

* Workload (default C = 5): BASELINE.json config 5, the largest
  single-GPU configuration and the scaling one -- 4e9 rows in total
  (int64 key U[0, 2^30), int64 value U[0, 2^20), count + sum, budget 2^24
  groups per GPU), strong-scaled: each of the N ranks holds 4e9 / N rows.
  A step = one SortAggregate.execute_columns over the rank's rows (run
  generation with early aggregation + wide merge; multi-GPU: sampled
  splitters, NCCL all-to-all, local operator per key range).  Inputs are
  resident in HBM before the timed region and far larger than the 126 MB L2
  (no flush needed).  Runs live where run_tier "auto" puts them (HBM while
  they fit 40% of the free HBM, else pinned host DRAM).
* value = input rows/s of the whole job, max over ranks of the device time
  (CUDA events on the launching stream, barrier + synchronize on both
  sides).  e2e = the same metric through the public API with pinned HOST
  input columns (H2D inside the timed region, staged in windows by the
  library) and the result read back to host memory.
* roofline = the dominant kernel family (by device time in the timed
  region): its algorithmic bytes per launch / its mean launch time, both
  from CUDA events the library records around its launches on their
  stream (isa_set_kernel_timing), against the measured HBM copy bandwidth
  (MEASURED_PEAKS.json).  traffic = ncu dram bytes per launch of that
  kernel from profiles/ncu_traffic.json (null when not captured).
  step_roofline = the minimum-traffic step time (read input once + write
  output once over HBM, + spill bytes over the measured PCIe link when runs
  leave HBM) over the measured step time.
* cfg3 (config 5 default only, N = 1): BASELINE config 3 (1e9 rows, Zipf
  hashed int64 keys, count/isum/fsum/min/max, budget 2^22, runs spilled to
  pinned host memory) timed in the same run with its own step roofline
  (raw-spill and moved-bytes link terms, HBM-only fraction) and its own
  kernel-true roofline.
* cpu_baseline = the oracle port (oracle/rsw_oracle.c: read-sort-write run
  generation + wide merge, key-range partitioned over all host threads) on a
  bounded sample of the same workload, rank 0 at N = 1.
* --impl reference: the reference algorithm's CPU implementation (the same
  oracle port; the reference is pure Python and cannot be compiled) on the
  host cores, same metric / config / unit, a bounded sample per step.
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
    2: "cfg2: 2^28 rows, (u8 x3, u8 x2) key = 6 groups, count + 4 f64 sums, M=4096 (no spill)",
    3: "cfg3: 1e9 rows, int64 hash(Zipf(1.1) over 2^28), count/isum/fsum/min/max, M=2^22, host spill",
    4: "cfg4: 2^29 rows, DISTINCT (u64,u64), 2^27 pairs x4, M=2^24",
    5: "cfg5: 4e9 rows in total, int64 U[0,2^30) key, count+sum, M=2^24 per GPU",
}
CPU_SAMPLE = {1: None, 2: 64 << 20, 3: 32 << 20, 4: 16 << 20, 5: 32 << 20}


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    p.add_argument("--rows", type=int, default=None, help="rows in total (default: the config's full size)")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cfg3", action="store_true")
    p.add_argument("--run-tier", default=None, choices=[None, "auto", "host", "hbm"])
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
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
    return n / secs, n, secs, len(out_keys[0])


def _traffic(cfgno, fam, alg_bytes_per_launch=None):
    """ncu dram bytes per launch of a kernel family (profiles/ncu_traffic.json):
    a captured per-launch figure, or -- launches of a family differ in size --
    the captured DRAM bytes per algorithmic byte times this run's mean
    algorithmic bytes per launch."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f).get(f"config{cfgno}", {})
        t = d.get(fam) or (d if d.get("phase") == fam else None)
        if not t:
            return None
        if "dram_bytes_per_launch" in t:
            return t["dram_bytes_per_launch"]
        if "dram_bytes_per_alg_byte" in t and alg_bytes_per_launch:
            return t["dram_bytes_per_alg_byte"] * alg_bytes_per_launch
        return None
    except Exception:
        return None


def _kernel_roofline(ks, steps, peak, peak_src, cfgno):
    fams = {k: v for k, v in ks.items() if v["launches"] > 0 and v["ms"] > 0}
    if not fams:
        return None, {}
    dom = max(fams, key=lambda k: fams[k]["ms"])
    d = fams[dom]
    per_launch_bytes = d["bytes"] / d["launches"]
    per_launch_ms = d["ms"] / d["launches"]
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": _traffic(cfgno, dom, per_launch_bytes),
            "alg_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
            "launches_per_step": d["launches"] / max(1, steps), "peak_source": peak_src,
            "timing": "CUDA events around every launch of the family on its stream, timed region"}
    table = {k: {"ms_per_step": v["ms"] / max(1, steps), "launches_per_step": v["launches"] / max(1, steps),
                 "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] else None}
             for k, v in fams.items()}
    return roof, table


def _step_roofline(w, rows, n_groups, dled, ms_step, peak, link, run_tier):
    key_b, val_b = w.key_bytes, w.value_bytes
    row_out = key_b + 8 * w.schema.state_slots
    b_in = rows * (key_b + val_b)
    b_out = (n_groups or 0) * row_out
    spill_rows = dled.get("rows_spilled", 0)
    link_moved = dled.get("bytes_d2h", 0) + dled.get("bytes_h2d", 0)
    # runs that left HBM (host tier) cross the link; spill bytes counted with
    # the reference semantics (spilled rows x row bytes, written + read back)
    spill_b = 2 * spill_rows * row_out if link_moved else 0
    t_hbm = (b_in + b_out) / (peak * 1e9)
    t_star = t_hbm + spill_b / (link * 1e9)
    t_moved = t_hbm + link_moved / (link * 1e9)
    return {"t_star_ms": t_star * 1e3, "frac": t_star * 1e3 / ms_step, "b_in": b_in, "b_out": b_out,
            "b_spill": spill_b, "link_gbs": link, "hbm_gbs": peak, "b_link_moved": link_moved,
            "t_moved_ms": t_moved * 1e3, "frac_moved": t_moved * 1e3 / ms_step,
            "t_hbm_ms": t_hbm * 1e3, "frac_hbm_only": t_hbm * 1e3 / ms_step, "run_tier": run_tier}


def _check_result(torch, dist, res, schema, rows_total, world, rank, dev):
    """Outside the timed region: every rank's keys strictly ascending, the
    ranks' key ranges in rank order, and -- when the schema counts rows -- the
    counts of all groups summing to the input rows."""
    from paper_2010_00152_b200.core import AggregateKind
    def ordered_view(k):   # torch compares neither uint16/32 nor uint64: order-preserving int64 views
        if k.dtype in (torch.uint16, torch.uint32):
            return k.to(torch.int64)
        if k.dtype == torch.uint64:
            return k.view(torch.int64) ^ torch.tensor(-(1 << 63), dtype=torch.int64, device=k.device)
        return k

    keys = [ordered_view(k) for k in res.keys]
    n = int(keys[0].shape[0]) if keys else 0
    ok_sorted = True
    if n > 1:
        gt = torch.zeros(n - 1, dtype=torch.bool, device=keys[0].device)
        eq = torch.ones(n - 1, dtype=torch.bool, device=keys[0].device)
        for k in keys:   # lexicographic, most significant column first
            gt |= eq & (k[1:] > k[:-1])
            eq &= k[1:] == k[:-1]
        ok_sorted = bool(gt.all().item())
    slot = 0
    count_slot = None
    for agg in schema.aggregates:
        if agg.kind == AggregateKind.COUNT and count_slot is None:
            count_slot = slot
        slot += 2 if agg.kind == AggregateKind.AVG else 1
    cnt = int(res.states[count_slot].sum().item()) if count_slot is not None and n else (0 if count_slot is not None else None)
    ordered = True
    if world > 1:
        first = torch.stack([k[0] if n else torch.zeros((), dtype=k.dtype, device=dev) for k in keys]).to(torch.int64)
        last = torch.stack([k[-1] if n else torch.zeros((), dtype=k.dtype, device=dev) for k in keys]).to(torch.int64)
        info = torch.cat([first, last, torch.tensor([n, cnt or 0], dtype=torch.int64, device=dev)])
        every = [torch.empty_like(info) for _ in range(world)]
        dist.all_gather(every, info)
        nk = len(keys)
        prev = None
        cnt = 0 if count_slot is not None else None
        for e in every:
            e = e.tolist()
            if count_slot is not None:
                cnt += e[2 * nk + 1]
            if e[2 * nk] == 0:
                continue
            if prev is not None and not (tuple(prev) < tuple(e[:nk])):
                ordered = False
            prev = e[nk:2 * nk]
        flag = torch.tensor([1 if ok_sorted else 0], dtype=torch.int64, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok_sorted = bool(flag.item())
    return {"keys_strictly_ascending": ok_sorted, "rank_ranges_in_order": ordered,
            "count_sum": cnt, "count_sum_equals_rows": (cnt == rows_total) if cnt is not None else None}


def run_reference(args):
    """--impl reference: the reference algorithm on the host cores."""
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_2010_00152_b200 import workloads
    rows = args.rows or workloads.FULL_ROWS[args.config]
    threads = os.cpu_count() or 1
    sample = args.cpu_sample_rows or min(rows, CPU_SAMPLE[args.config] or rows)
    w = workloads.make(args.config, rows=sample, device="cpu")
    _cpu_baseline(w, min(sample, 1 << 20), threads)   # untimed warm-up (page faults, thread pool)
    vals = []
    for _ in range(args.steps):
        v, n, secs, groups = _cpu_baseline(w, sample, threads)
        vals.append((v, secs))
    value = sum(v for v, _ in vals) / len(vals)
    ms = sum(s for _, s in vals) / len(vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic (seeded, BASELINE shapes)",
        "config": {"workload": WORKLOAD_NAMES[args.config], "rows": rows, "rows_per_step": sample,
                   "parallelism": f"{threads} cpu threads"},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "port",
                         "sample": f"first {sample} rows of the seeded workload (cpu generator) per step, "
                                   f"oracle/rsw_oracle.c key-range partitioned over {threads} threads"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _pinned_copy(torch, t):
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


def measure(torch, dist, cfgno, rows_total, run_tier, steps, warmup, world, rank, local, dev, *, e2e=False,
            e2e_steps=None, clocks=True):
    """Time `steps` executes of config `cfgno`; returns the JSON fields."""
    import paper_2010_00152_b200 as isa
    from paper_2010_00152_b200 import _native, workloads

    rows = rows_total // world
    gen_kw = {"seed": workloads.SEED + cfgno + 1000 * rank} if world > 1 else {}
    w = workloads.make(cfgno, rows=rows, device=dev, **gen_kw)
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

    res = None
    for _ in range(warmup):
        res = None
        res = step()
    barrier()
    sampler = ClockSampler(local) if clocks else None
    if sampler:
        # clocks are sampled from a >= 1 s load ramp right before the timed
        # region through its end (a short timed region alone holds too few samples)
        sampler.start()
        t_ramp = time.perf_counter()
        while time.perf_counter() - t_ramp < 1.0:
            res = None
            res = step()
            torch.cuda.synchronize(dev)
    barrier()
    stream = torch.cuda.current_stream(dev)
    # kernel timing records two CUDA events per timed launch: create them all
    # now (one untimed step counts the launches), not inside the timed region
    l0 = _native.launch_count()
    res = None
    res = step()
    torch.cuda.synchronize(dev)
    _native.kernel_timing_reserve(2 * (steps + 1) * (_native.launch_count() - l0) + 64)
    _native.set_kernel_timing(True)
    _native.kernel_stats()          # drop anything recorded before the timed region
    launches0 = _native.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    snaps = []
    for _ in range(steps):
        res = None
        res = step()
        snaps.append(op.phase_snapshot())   # one small native call; decoded after the timed region
    ev1.record(stream)
    barrier()
    clk = sampler.stop() if sampler else None
    ks = _native.kernel_stats()
    _native.set_kernel_timing(False)
    launches = _native.launch_count() - launches0
    phase_tot = {}
    for raw in snaps:
        if raw is None:
            continue
        for k, v in _native.phases_dict(raw).items():
            t = phase_tot.setdefault(k, {"ms": 0.0, "calls": 0, "rows": 0, "bytes": 0})
            for f in t:
                t[f] += v[f]
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / max(1, steps)
    value = rows * world / (ms_step / 1e3)
    n_groups = res.n_groups if hasattr(res, "n_groups") else None
    check = _check_result(torch, dist, res, w.schema, rows * world, world, rank, dev)
    if world > 1 and n_groups is not None:
        t = torch.tensor([n_groups], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        n_groups = int(t.item())

    peak, peak_src = _peaks()
    link = _link_gbs(torch, dev)
    dled = op.device_ledger or {}
    roof, ktable = _kernel_roofline(ks, steps, peak, peak_src, cfgno)
    out = {
        "value": value, "ms_per_step": ms_step, "steps": steps, "warmup": warmup,
        "config": {"workload": WORKLOAD_NAMES[cfgno], "rows": rows * world, "rows_per_gpu": rows,
                   "groups": n_groups, "memory_budget": w.memory_budget, "page_capacity": workloads.PAGE,
                   "run_tier": run_tier, "parallelism": f"range-partitioned x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs (%.1f GB) larger than L2 (126 MB); no flush" % (rows * (w.key_bytes + w.value_bytes) / 1e9)},
        "roofline": roof,
        "kernels": ktable,
        "step_roofline": _step_roofline(w, rows, (n_groups or 0) // max(1, world) if world > 1 else n_groups,
                                        dled, ms_step, peak, link, run_tier),
        "phases_ms_per_step": {k: v["ms"] / max(1, steps) for k, v in phase_tot.items() if v["ms"]},
        "ledger_per_step": {"rows_spilled": dled.get("rows_spilled"), "runs": op.runs_after_generation,
                            "bytes_d2h": dled.get("bytes_d2h"), "bytes_h2d": dled.get("bytes_h2d"),
                            "merge_windows": dled.get("merge_windows"), "chunks": dled.get("chunks")},
        "gpu_launches": launches,
        "clocks": clk,
        "check": check,
    }
    res = None

    if e2e:
        # end to end through the public API: pinned host columns in, host result out
        in_row_bytes = w.key_bytes + w.value_bytes
        host_keys = [_pinned_copy(torch, k) for k in w.keys]
        host_vals = {n: _pinned_copy(torch, v) for n, v in w.values.items()}
        keys_dev, vals_dev = w.keys, w.values
        w.keys, w.values = [], {}
        del keys_dev, vals_dev
        torch.cuda.empty_cache()
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
        outs = e2e_step()
        barrier()
        k2 = e2e_steps or steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k2):
            outs = None
            outs = e2e_step()
        e1.record(stream)
        barrier()
        secs = e0.elapsed_time(e1) / 1e3 / k2
        if world > 1:
            t = torch.tensor([secs], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = float(t.item())
        d2h = sum(o.numel() * o.element_size() for o in outs)
        raw = op_e2e.phase_snapshot()
        e2e_ph = {k: round(v["ms"], 2) for k, v in _native.phases_dict(raw).items() if v["ms"]} if raw is not None else {}
        out["e2e"] = {"value": rows * world / secs, "unit": "rows/s",
                      "h2d_bytes_per_step": rows * in_row_bytes,
                      "d2h_bytes_per_step": d2h, "ms_per_step": secs * 1e3,
                      "timing": "CUDA events on the launching stream around synchronous execute_columns calls",
                      "phases_ms_last_step": e2e_ph,
                      "streamed_output": bool(getattr(op_e2e, "streamed_output", False))}
        outs = None
        del host_keys, host_vals
        op_e2e.close()
    op.close()
    del w
    torch.cuda.empty_cache()
    return out


def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2010_00152_b200 import workloads

    world, rank, local = _dist()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        if rank == 0:
            print(f"[bench] NCCL communicator: {dist.get_world_size()} ranks", file=sys.stderr, flush=True)
    cfgno = args.config
    rows_total = args.rows or workloads.FULL_ROWS[cfgno]
    run_tier = args.run_tier or ("host" if cfgno == 3 else "auto")
    warmup = max(3, args.warmup)   # timing rule: at least 3 untimed warm-up steps
    m = measure(torch, dist, cfgno, rows_total, run_tier, args.steps, warmup, world, rank, local, dev,
                e2e=not args.no_e2e, e2e_steps=args.e2e_steps)
    line = {
        "metric": METRIC, "value": m["value"], "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded generator with BASELINE.json shapes, "
                                                       "generated on device)",
    }
    for k in ("config", "roofline", "kernels", "step_roofline", "phases_ms_per_step", "ledger_per_step",
              "gpu_launches", "clocks", "check", "e2e"):
        if k in m:
            line[k] = m[k]
    if cfgno == 5 and world == 1 and not args.no_cfg3:
        c3 = measure(torch, dist, 3, workloads.FULL_ROWS[3], "host", 3, 3, world, rank, local, dev, clocks=False)
        line["cfg3"] = {"metric": "input rows/s", "value": c3["value"], "ms_per_step": c3["ms_per_step"],
                        "steps": 3, "warmup": 3, "config": c3["config"], "roofline": c3["roofline"],
                        "kernels": c3["kernels"], "step_roofline": c3["step_roofline"],
                        "phases_ms_per_step": c3["phases_ms_per_step"], "ledger_per_step": c3["ledger_per_step"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = args.cpu_sample_rows or min(rows_total, CPU_SAMPLE[cfgno] or rows_total)
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
