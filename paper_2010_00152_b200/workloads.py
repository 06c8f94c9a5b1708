"""Seeded synthetic inputs with the shapes of BASELINE.json's five configs.

No benchmark dataset exists for this path; these generators
stand in for it with the stated row counts, key domains and value
distributions.  They run on any torch device: CPU for small, oracle-checked
cases and CUDA for full-scale runs (generation is not part of any timed
region).  Every config returns a ``Workload``: key columns, value columns
keyed by name, the Schema and the aggregate list.

Key/value recipes:
  1  uint32 key over 10,000 distinct random values, every value planted once,
     the rest uniform, shuffled (bench.py:144-162 recipe); int64 value in
     [-1e6, 1e6]; count/sum/min/max; M = 4,096.
  2  (uint8 in {0,1,2}, uint8 in {0,1}); four float64 U[0, 1e5); count + 4 sums.
  3  int64 key = splitmix64(rank), rank ~ Zipf(1.1) over 2^28 (continuous
     inverse-CDF approximation of p(r) ~ r^-1.1); int64 U[0, 2^31) and
     float32 N(0,1); count, isum, fsum, min, max; M = 2^22.
  4  (uint64, uint64) pairs: 2^27 random pairs, each repeated 4x, shuffled;
     DISTINCT (no aggregates); M = 2^24.
  5  int64 key U[0, 2^30); int64 value U[0, 2^20); count + sum; M = 2^24 per GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .core import AggregateKind, AggregateSpec, ColumnSpec, Schema

FULL_ROWS = {1: 1_000_000, 2: 1 << 28, 3: 1_000_000_000, 4: 1 << 29, 5: 4_000_000_000}
BUDGET = {1: 4096, 2: 4096, 3: 1 << 22, 4: 1 << 24, 5: 1 << 24}
PAGE = 100
SEED = 20100015


@dataclass
class Workload:
    config: int
    rows: int
    schema: Schema
    keys: list
    values: dict = field(default_factory=dict)
    memory_budget: int = 4096
    description: str = ""

    @property
    def key_bytes(self):
        return sum(k.element_size() for k in self.keys)

    @property
    def value_bytes(self):
        return sum(v.element_size() for v in self.values.values())

    @property
    def input_bytes(self):
        return self.rows * (self.key_bytes + self.value_bytes)

    def to(self, device):
        return Workload(self.config, self.rows, self.schema, [k.to(device) for k in self.keys],
                        {n: v.to(device) for n, v in self.values.items()}, self.memory_budget,
                        self.description)


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _lsr(x, s):
    """logical shift right of int64 tensors"""
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x):
    """splitmix64 finalizer on int64 tensors (two's-complement wraparound)."""
    x = x + (-7046029254386353131)  # 0x9E3779B97F4A7C15
    x = (x ^ _lsr(x, 30)) * (-4658895280553007687)  # 0xBF58476D1CE4E5B9
    x = (x ^ _lsr(x, 27)) * (-7723592293110705685)  # 0x94D049BB133111EB
    return x ^ _lsr(x, 31)


def _int_schema(names_kinds, n_keys, key_names=None):
    key_names = key_names or [f"k{i}" for i in range(n_keys)]
    cols = [ColumnSpec(n) for n in key_names]
    aggs = [AggregateSpec(name, kind, col) for name, kind, col in names_kinds]
    return Schema(cols, aggs)


def config1(rows=None, distinct=10_000, device="cpu", seed=SEED + 1):
    rows = FULL_ROWS[1] if rows is None else rows
    distinct = min(distinct, rows)
    g = _gen(device, seed)
    # distinct random uint32 key values
    cand = torch.randint(0, 1 << 32, (distinct * 2 + 64,), generator=g, device=device, dtype=torch.int64)
    uniq = torch.unique(cand)
    perm = torch.randperm(uniq.numel(), generator=g, device=device)
    vocab = uniq[perm[:distinct]]
    ids = torch.cat([torch.arange(distinct, device=device),
                     torch.randint(0, distinct, (rows - distinct,), generator=g, device=device)])
    ids = ids[torch.randperm(rows, generator=g, device=device)]
    key = vocab[ids].to(torch.uint32)
    val = torch.randint(-1_000_000, 1_000_001, (rows,), generator=g, device=device, dtype=torch.int64)
    schema = _int_schema([("n", AggregateKind.COUNT, None), ("s", AggregateKind.SUM, "v"),
                          ("lo", AggregateKind.MIN, "v"), ("hi", AggregateKind.MAX, "v")], 1)
    return Workload(1, rows, schema, [key], {"v": val}, BUDGET[1],
                    "u32 key over 10k planted values; count/sum/min/max of int64")


def config2(rows=None, device="cpu", seed=SEED + 2, budget=None):
    rows = FULL_ROWS[2] if rows is None else rows
    g = _gen(device, seed)
    k1 = torch.randint(0, 3, (rows,), generator=g, device=device, dtype=torch.uint8)
    k2 = torch.randint(0, 2, (rows,), generator=g, device=device, dtype=torch.uint8)
    vals = {f"f{i}": torch.rand(rows, generator=g, device=device, dtype=torch.float64) * 1e5 for i in range(4)}
    schema = _int_schema([("n", AggregateKind.COUNT, None)] +
                         [(f"sum_f{i}", AggregateKind.SUM, f"f{i}") for i in range(4)], 2)
    return Workload(2, rows, schema, [k1, k2], vals, budget or BUDGET[2],
                    "(u8 x3, u8 x2) composite key, 6 groups; count + 4 float64 sums")


def zipf_ranks(rows, domain, s, g, device):
    u = torch.rand(rows, generator=g, device=device, dtype=torch.float64)
    a = 1.0 - s
    top = float(domain + 1) ** a - 1.0
    x = torch.pow(1.0 + u * top, 1.0 / a)
    return torch.clamp(torch.floor(x), 1, domain).to(torch.int64)


def config3(rows=None, domain=1 << 28, device="cpu", seed=SEED + 3, budget=None):
    rows = FULL_ROWS[3] if rows is None else rows
    g = _gen(device, seed)
    key = splitmix64(zipf_ranks(rows, domain, 1.1, g, device))
    vi = torch.randint(0, 1 << 31, (rows,), generator=g, device=device, dtype=torch.int64)
    vf = torch.randn(rows, generator=g, device=device, dtype=torch.float32)
    schema = _int_schema([("n", AggregateKind.COUNT, None), ("isum", AggregateKind.SUM, "vi"),
                          ("fsum", AggregateKind.SUM, "vf"), ("imin", AggregateKind.MIN, "vi"),
                          ("imax", AggregateKind.MAX, "vi")], 1)
    return Workload(3, rows, schema, [key], {"vi": vi, "vf": vf}, budget or BUDGET[3],
                    "int64 splitmix64(Zipf(1.1) rank over 2^28); count/isum/fsum/min/max")


def config4(rows=None, device="cpu", seed=SEED + 4, budget=None, copies=4):
    rows = FULL_ROWS[4] if rows is None else rows
    distinct = max(1, rows // copies)
    rows = distinct * copies
    g = _gen(device, seed)
    a = torch.randint(-(1 << 63), (1 << 63) - 1, (distinct,), generator=g, device=device, dtype=torch.int64)
    b = torch.randint(-(1 << 63), (1 << 63) - 1, (distinct,), generator=g, device=device, dtype=torch.int64)
    idx = torch.arange(distinct, device=device).repeat(copies)
    idx = idx[torch.randperm(rows, generator=g, device=device)]
    k1 = a[idx].view(torch.uint64)
    k2 = b[idx].view(torch.uint64)
    schema = _int_schema([], 2)
    return Workload(4, rows, schema, [k1, k2], {}, budget or BUDGET[4],
                    "DISTINCT over (u64, u64): rows/4 random pairs x4, shuffled")


def config5(rows=None, device="cpu", seed=SEED + 5, budget=None, domain=1 << 30):
    rows = FULL_ROWS[5] if rows is None else rows
    g = _gen(device, seed)
    key = torch.randint(0, domain, (rows,), generator=g, device=device, dtype=torch.int64)
    val = torch.randint(0, 1 << 20, (rows,), generator=g, device=device, dtype=torch.int64)
    schema = _int_schema([("n", AggregateKind.COUNT, None), ("s", AggregateKind.SUM, "v")], 1)
    return Workload(5, rows, schema, [key], {"v": val}, budget or BUDGET[5],
                    "int64 key U[0, 2^30); count + sum of int64 U[0, 2^20)")


GENERATORS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(config, rows=None, device="cpu", **kw):
    return GENERATORS[config](rows=rows, device=device, **kw)
