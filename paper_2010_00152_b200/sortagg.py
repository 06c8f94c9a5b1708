"""SortAggregate on B200: the reference operator's entry points over the CUDA path.

Drop-in for ``insortagg.sortagg.SortAggregate`` in wide-merge mode
(/root/reference/pkg/src/insortagg/sortagg.py:725-784):

* ``SortAggConfig`` has the reference's fields, defaults and validation
  (sortagg.py:53-86) plus three placement knobs (``run_tier``,
  ``chunk_rows_max``, ``merge_window_rows``).
* ``SortAggregate(schema, config, store, ledger).execute(rows)`` returns the
  sorted, unfinalized ``Row`` list and fills ``ledger``, ``initial_plan``,
  ``executed_steps`` and ``runs_after_generation`` like the reference.
* ``SortAggregate.execute_columns(keys, values)`` is the columnar fast path:
  key / value tensors in, sorted key columns + state-slot columns out.

All grouping work runs in libinsortagg_b200.so (run generation with early
aggregation, host-tier spill, wide merge); Python only converts layouts.
The merge planner / output estimator below are host-side bookkeeping that
reproduce the reference's ``initial_plan`` from the run sizes and fill
cycles the device reports.
"""

from __future__ import annotations

import os

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import (
    AggregateKind,
    InvalidInputError,
    MetricsLedger,
    ResourceError,
    Row,
)

WIDE = "wide"
TRADITIONAL = "traditional"
SEPARATE = "separate"

READ_SORT_WRITE = "read_sort_write"
REPLACEMENT_SELECTION = "replacement_selection"

ASCENDING = "ascending"


@dataclass
class SortAggConfig:
    """Operator configuration (sortagg.py:53-86)."""

    memory_budget: int
    page_capacity: int
    run_generation_mode: str = READ_SORT_WRITE
    merge_mode: str = WIDE
    ovc_enabled: bool = True
    ovc_cache: bool = True
    ovc_direction: str = ASCENDING
    interpolation_search: bool = False
    batch_size: int = 1
    leaf_capacity: int = 64
    eviction_chunk: int | None = None
    output_size_hint: int | None = None
    max_preliminary_merges: int | None = None
    # B200 placement knobs (no reference counterpart)
    run_tier: str = "auto"          # where spilled runs live: "auto" (HBM while they fit, then pinned DRAM) | "host" | "hbm"
    hbm_run_budget: int = 0         # run_tier "auto": HBM bytes for runs, 0 = half of the free HBM
    chunk_rows_max: int = 0         # 0 = library default
    window_rows: int = 0            # host-input staging window, 0 = default
    merge_window_rows: int = 0      # wide-merge key-range window capacity, 0 = default
    preaggregate: str = "auto"      # tile-local pre-aggregation before chunk sorts: auto | always | never
    run_codec: str = "auto"         # host-tier runs cross PCIe bit-packed: auto (runs >= 32K rows) | packed | raw
    hot_absorb: str = "auto"        # rows whose key is in a large resident table absorbed via its hash image: auto | always | never

    def __post_init__(self):
        if self.page_capacity < 1:
            raise InvalidInputError("page capacity must be positive")
        if self.memory_budget < 2 * self.page_capacity:
            raise InvalidInputError("memory budget must cover two pages")
        if self.max_fanin < 2:
            raise InvalidInputError("fan-in must be at least 2")
        if self.run_generation_mode not in (READ_SORT_WRITE, REPLACEMENT_SELECTION):
            raise InvalidInputError(
                f"unknown run generation mode {self.run_generation_mode!r}")
        if self.merge_mode not in (WIDE, TRADITIONAL, SEPARATE):
            raise InvalidInputError(f"unknown merge mode {self.merge_mode!r}")
        if self.run_tier not in ("auto", "host", "hbm"):
            raise InvalidInputError(f"unknown run tier {self.run_tier!r}")
        if self.preaggregate not in ("auto", "always", "never"):
            raise InvalidInputError(f"unknown preaggregate mode {self.preaggregate!r}")
        if self.run_codec not in ("auto", "packed", "raw"):
            raise InvalidInputError(f"unknown run codec {self.run_codec!r}")
        if self.hot_absorb not in ("auto", "always", "never"):
            raise InvalidInputError(f"unknown hot_absorb mode {self.hot_absorb!r}")

    @property
    def max_fanin(self):
        return self.memory_budget // self.page_capacity


# ---------------------------------------------------------------------------
# host-side planner bookkeeping (reproduces the reference's initial_plan)
# ---------------------------------------------------------------------------

class OutputEstimator:
    """Distinct-key (output size) estimate from run generation
    (sortagg.py:89-160): the larger of observed distinct counts, the largest
    run, and the read-sort-write fill-cycle inversion C = O ln(O / (O - M)),
    capped at the rows seen."""

    def __init__(self, budget):
        self.budget = budget
        self.steady_probes = 0
        self.steady_absorbs = 0
        self.steady_resident_sum = 0
        self.cycles = []
        self.observed = 1
        self.max_run_rows = 0

    def note_steady_probe(self, resident, absorbed):
        self.steady_probes += 1
        self.steady_resident_sum += resident
        self.steady_absorbs += 1 if absorbed else 0

    def note_cycle(self, consumed):
        if consumed > 0:
            self.cycles.append(consumed)

    def observe_distinct(self, count):
        self.observed = max(self.observed, count)

    def note_runs(self, run_rows):
        for rows in run_rows:
            self.max_run_rows = max(self.max_run_rows, rows)

    def _invert_cycle(self, mean_cycle, rows_seen):
        m = self.budget
        if mean_cycle <= m * (1 + 1e-9):
            return rows_seen

        def cycle_len(o):
            return o * math.log(o / (o - m))

        lo, hi = m * (1 + 1e-12), 2.0 * m
        while cycle_len(hi) > mean_cycle:
            hi *= 2
            if hi > 1e18:
                return rows_seen
        for _ in range(80):
            mid = 0.5 * (lo + hi)
            if cycle_len(mid) > mean_cycle:
                lo = mid
            else:
                hi = mid
        return 0.5 * (lo + hi)

    def estimate(self, rows_seen):
        options = [self.observed, self.max_run_rows, 1]
        if self.steady_probes >= 100:
            options.append(self.steady_resident_sum / self.steady_absorbs
                           if self.steady_absorbs else rows_seen)
        if self.cycles:
            options.append(self._invert_cycle(sum(self.cycles) / len(self.cycles), rows_seen))
        est = max(options)
        if rows_seen:
            est = min(est, rows_seen)
        return max(1, int(est))


@dataclass(frozen=True)
class PlanStep:
    kind: str  # "traditional" | "wide"
    input_run_ids: tuple
    expected_output_rows: int


@dataclass(frozen=True)
class MergePlan:
    steps: tuple
    levels: int

    @property
    def wide_steps(self):
        return sum(1 for s in self.steps if s.kind == "wide")


def wide_admissible(sizes, o_est, config):
    """Admission test of the final wide merge (sortagg.py:479-499)."""
    if len(sizes) == 1:
        return True
    ordered = sorted(sizes)
    if sum(ordered[:config.max_fanin]) < o_est:
        return False
    index_budget = config.memory_budget - 2 * config.page_capacity
    if index_budget < 1:
        return False
    median = ordered[len(ordered) // 2]
    return o_est * config.page_capacity / max(1, median) <= index_budget


def plan_merge(run_sizes, o_est, config):
    """Merge plan for runs of the given sizes (sortagg.py:502-542): fan-in
    limited traditional levels over the smallest runs until the wide step is
    admissible (run ids are positions in ``run_sizes``)."""
    if not run_sizes:
        raise InvalidInputError("cannot plan a merge without runs")
    o_est = max(1, int(o_est))
    fan = config.max_fanin
    pool = sorted((rows, rid) for rid, rows in enumerate(run_sizes))
    steps, levels, synthetic = [], 0, 0
    while True:
        sizes = [rows for rows, _ in pool]
        if wide_admissible(sizes, o_est, config):
            steps.append(PlanStep("wide", tuple(r for _, r in pool), min(sum(sizes), o_est)))
            break
        if len(pool) <= fan:
            steps.append(PlanStep("traditional", tuple(r for _, r in pool), min(sum(sizes), o_est)))
            break
        levels += 1
        merged = []
        for start in range(0, len(pool), fan):
            group = pool[start:start + fan]
            if len(group) == 1:
                merged.append(group[0])
                continue
            total = sum(rows for rows, _ in group)
            out_rows = min(total, o_est) if total >= o_est else total
            synthetic += 1
            steps.append(PlanStep("traditional", tuple(r for _, r in group), out_rows))
            merged.append((out_rows, f"planned-{synthetic}"))
        pool = sorted(merged)
    return MergePlan(tuple(steps), levels)


# ---------------------------------------------------------------------------
# run stores: accepted for signature parity; run placement is internal
# ---------------------------------------------------------------------------

class MemoryStore:
    """Accepted as the ``store`` argument (runstore.py:157-192).  The B200
    operator places runs itself (pinned host DRAM or HBM, ``run_tier``)."""

    def __init__(self, retain_rows=False):
        self.retain_rows = retain_rows


class FileStore:
    """Temporary storage backed by one file per run in a directory
    (runstore.py:195-236), same file names and page index.  With a FileStore
    the B200 operator writes its runs there in the reference's page format
    (byte-identical to RunWriter's pages: the reference's ``read_page`` reads
    them) and its wide merge reads them back from the files."""

    def __init__(self, directory):
        self.directory = directory
        os.makedirs(directory, exist_ok=True)
        self._offsets = {}
        self._handles = {}
        self._next = 0

    def _path(self, run_id):
        return os.path.join(self.directory, f"run_{run_id:06d}.bin")

    def new_run(self):
        rid = self._next
        self._next += 1
        self._offsets[rid] = []
        self._handles[rid] = open(self._path(rid), "wb")
        return rid

    def append_page(self, run_id, page, rows=None):
        fh = self._handles[run_id]
        self._offsets[run_id].append((fh.tell(), len(page)))
        fh.write(page)

    def finalize_run(self, run_id):
        fh = self._handles.pop(run_id, None)
        if fh is not None:
            fh.close()

    def page_bytes(self, run_id, index):
        off, length = self._offsets[run_id][index]
        with open(self._path(run_id), "rb") as fh:
            fh.seek(off)
            return fh.read(length)

    def retained(self, run_id, index):
        return None

    def close(self):
        for rid in list(self._handles):
            self.finalize_run(rid)

    def _adopt(self, run_rows, arity, slots, page_capacity):
        """Register runs the native writer produced (ids _next, _next+1, ...)
        with their page index (page sizes follow from the row counts)."""
        ids = []
        for rows in run_rows:
            rid = self._next
            self._next += 1
            off, pages = 0, []
            left = rows
            while left > 0:
                r = min(page_capacity, left)
                length = 12 + 8 * arity + r * 8 * (arity + slots)
                pages.append((off, length))
                off += length
                left -= r
            self._offsets[rid] = pages
            ids.append(rid)
        return ids


# ---------------------------------------------------------------------------
# dtype plumbing
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


_DTYPE_CODES = None


def _isa_dtype(t):
    global _DTYPE_CODES
    if _DTYPE_CODES is None:
        torch = _torch()
        table = {
            torch.uint8: _native.U8, torch.int8: _native.I8, torch.int16: _native.I16,
            torch.int32: _native.I32, torch.int64: _native.I64, torch.float32: _native.F32,
            torch.float64: _native.F64,
        }
        for name, code in (("uint16", _native.U16), ("uint32", _native.U32), ("uint64", _native.U64)):
            if hasattr(torch, name):
                table[getattr(torch, name)] = code
        _DTYPE_CODES = table
    code = _DTYPE_CODES.get(t.dtype)
    if code is None:
        raise InvalidInputError(f"unsupported column dtype {t.dtype}")
    return code


_OP_CODES = {"add": _native.OP_ADD, "min": _native.OP_MIN, "max": _native.OP_MAX}


class ColumnarResult(tuple):
    """(key_columns, state_columns): sorted unique keys, one tensor per key
    column (input dtype) and one per state slot (int64 or float64)."""

    __slots__ = ()

    def __new__(cls, keys, states):
        return super().__new__(cls, (keys, states))

    @property
    def keys(self):
        return self[0]

    @property
    def states(self):
        return self[1]

    def __len__(self):  # number of tuple fields (keys, states)
        return 2

    @property
    def n_groups(self):
        return int(self[0][0].shape[0]) if self[0] else 0


def _lazy(name, doc):
    def get(self):
        if name not in self._info:
            self._materialize()
        return self._info[name]

    def put(self, value):
        self._info[name] = value
    return property(get, put, doc=doc)


class SortAggregate:
    """Sort-based grouping / duplicate removal / aggregation on one B200.

    ``execute`` consumes an unsorted row stream and returns aggregated rows in
    ascending key order (sortagg.py:744-784); ``execute_columns`` does the same
    on column tensors.  Runs spill to pinned host memory (default) or HBM.
    ``merge_mode`` wide (the paper's in-sort aggregation + wide merge),
    traditional or separate (priority-queue run generation + fan-in merge
    levels, sortagg.py:788-849); read-sort-write run generation.
    """

    cycles = _lazy("cycles", "fill-cycle lengths of the last execute (rows consumed per flush)")
    run_rows = _lazy("run_rows", "rows of every run written by the last execute")
    phase_stats = _lazy("phase_stats", "per-phase device times of the last execute")
    runs_after_generation = _lazy("runs_after_generation", "SortAggregate.runs_after_generation")
    executed_steps = _lazy("executed_steps", "SortAggregate.executed_steps")
    initial_plan = _lazy("initial_plan", "SortAggregate.initial_plan")
    device_ledger = _lazy("device_ledger", "native isa_ledger of the last execute (dict)")

    def __init__(self, schema, config, store=None, ledger=None, *, device=None):
        if isinstance(store, FileStore):
            if config.merge_mode != WIDE:
                raise InvalidInputError("the FileStore run tier supports merge_mode 'wide'")
        if config.run_generation_mode == REPLACEMENT_SELECTION and config.merge_mode != WIDE:
            raise InvalidInputError("replacement selection is supported with merge_mode 'wide' "
                                    "(the traditional modes' tagged-run priority queue is not ported)")
        if any(c.kind != "int64" for c in schema.key_columns):
            raise InvalidInputError("utf8 key columns are not supported by the B200 operator")
        self.schema = schema
        self.config = config
        self.store = store
        self.ledger = ledger if ledger is not None else MetricsLedger()
        self._last = None
        self._info = {}
        self._materialize()
        self._device = device
        self._handles = {}

    # -- native handles ----------------------------------------------------
    def _device_index(self):
        torch = _torch()
        if self._device is not None:
            idx = getattr(self._device, "index", None)
            if idx is not None:
                return idx
            d = torch.device(self._device)
            return d.index if d.index is not None else torch.cuda.current_device()
        return torch.cuda.current_device()

    def _handle(self, key_codes, val_codes, slots):
        dev = self._device_index()
        sig = (tuple(key_codes), tuple(val_codes), tuple(slots), dev)
        h = self._handles.get(sig)
        if h is not None:
            return h
        cfg = _native.IsaConfig()
        cfg.memory_budget = self.config.memory_budget
        cfg.page_capacity = self.config.page_capacity
        if isinstance(self.store, FileStore):
            cfg.run_tier = _native.TIER_FILE
        else:
            cfg.run_tier = {"host": _native.TIER_HOST, "hbm": _native.TIER_HBM,
                            "auto": _native.TIER_AUTO}[self.config.run_tier]
        cfg.hbm_run_budget = self.config.hbm_run_budget
        cfg.device = dev
        cfg.chunk_rows_max = self.config.chunk_rows_max
        cfg.window_rows = self.config.window_rows
        cfg.merge_window_rows = self.config.merge_window_rows
        cfg.preaggregate = {"auto": 0, "always": 1, "never": 2}[self.config.preaggregate]
        cfg.merge_mode = {WIDE: _native.MERGE_WIDE, TRADITIONAL: _native.MERGE_TRADITIONAL,
                          SEPARATE: _native.MERGE_SEPARATE}[self.config.merge_mode]
        cfg.output_size_hint = self.config.output_size_hint if self.config.output_size_hint is not None else 0
        cfg.run_codec = {"auto": 0, "raw": 1, "packed": 2}[self.config.run_codec]
        cfg.hot_absorb = {"auto": 0, "always": 1, "never": 2}[self.config.hot_absorb]
        cfg.run_generation = 1 if self.config.run_generation_mode == REPLACEMENT_SELECTION else 0
        cfg.eviction_chunk = self.config.eviction_chunk or 0
        sch = _native.IsaSchema()
        if len(key_codes) > _native.MAX_KEY_COLS:
            raise InvalidInputError("too many key columns")
        if len(slots) > _native.MAX_SLOTS:
            raise InvalidInputError("too many aggregate state slots")
        if len(val_codes) > _native.MAX_VAL_COLS:
            raise InvalidInputError("too many value columns")
        sch.n_key_cols = len(key_codes)
        for i, c in enumerate(key_codes):
            sch.key_dtypes[i] = c
        sch.n_val_cols = len(val_codes)
        for i, c in enumerate(val_codes):
            sch.val_dtypes[i] = c
        sch.n_slots = len(slots)
        for s, (op, ty, src, col) in enumerate(slots):
            sch.slot_op[s] = op
            sch.slot_type[s] = ty
            sch.slot_src[s] = src
            sch.slot_col[s] = col
        h = _native.Handle(cfg, sch)
        self._handles[sig] = h
        return h

    def close(self):
        for h in self._handles.values():
            h.close()
        self._handles.clear()

    # -- slot layout -----------------------------------------------------------
    def _slots_from_values(self, value_cols):
        """Schema.make_state layout (core.py:162-182) over value columns:
        returns (value tensors, slot specs)."""
        torch = _torch()
        vals, slots = [], []
        for agg, col in zip(self.schema.aggregates, value_cols):
            if agg.kind == AggregateKind.COUNT:
                slots.append((_native.OP_ADD, _native.SLOT_I64, _native.SRC_ONE, 0))
                continue
            if col is None:
                raise InvalidInputError(f"aggregate {agg.name!r} needs a value column")
            is_float = col.dtype in (torch.float32, torch.float64, torch.float16, torch.bfloat16)
            ty = _native.SLOT_F64 if is_float else _native.SLOT_I64
            idx = len(vals)
            vals.append(col)
            op = {AggregateKind.SUM: _native.OP_ADD, AggregateKind.MIN: _native.OP_MIN,
                  AggregateKind.MAX: _native.OP_MAX, AggregateKind.AVG: _native.OP_ADD}[agg.kind]
            slots.append((op, ty, _native.SRC_COLUMN, idx))
            if agg.kind == AggregateKind.AVG:
                slots.append((_native.OP_ADD, _native.SLOT_I64, _native.SRC_ONE, 0))
        return vals, slots

    def _resolve_values(self, values):
        aggs = self.schema.aggregates
        if values is None:
            values = {}
        if isinstance(values, dict):
            out = []
            for agg in aggs:
                if agg.kind == AggregateKind.COUNT:
                    out.append(None)
                    continue
                name = agg.column if agg.column is not None else agg.name
                if name not in values:
                    raise InvalidInputError(f"missing value column {name!r} for aggregate {agg.name!r}")
                out.append(values[name])
            return out
        values = list(values)
        if len(values) != len(aggs):
            raise InvalidInputError(f"expected {len(aggs)} value columns (one per aggregate), got {len(values)}")
        return values

    # -- columnar fast path ----------------------------------------------------
    def execute_columns(self, keys, values=None, *, states=False, stream=None):
        """Group ``keys`` (list of 1-D integer tensors, most significant
        first) and aggregate ``values``.

        ``values``: dict column-name -> tensor (``AggregateSpec.column``, else
        the aggregate name) or a list parallel to ``schema.aggregates`` (None
        for COUNT).  With ``states=True`` ``values`` is instead a list of
        already-built state-slot columns (one per slot, Schema layout) that
        are combined with ``merge_states``.

        Inputs on a CUDA device stay there; CPU inputs (pinned for speed) are
        streamed to the GPU in windows.  Returns ColumnarResult(keys, states)
        on the input's device.
        """
        h, n, keys, vals, slots, on_host, sptr = self._prepare(keys, values, states, stream)
        file_store = isinstance(self.store, FileStore)
        if file_store:
            h.set_spill_dir(self.store.directory, self.store._next)
        # the caller owns the output columns: the native side asks for them
        # (isa_set_output_allocator) -- during the wide merge with host input
        # that spilled (the device -> host transfer then overlaps the merge),
        # else at the end of the execute at the exact group count
        streamed = {}
        torch = _torch()
        out_dev = torch.device("cpu") if on_host else keys[0].device

        def alloc(capacity):
            ok = [torch.empty(capacity, dtype=k.dtype, device=out_dev, pin_memory=on_host) for k in keys]
            os_ = [torch.empty(capacity, dtype=torch.float64 if ty == _native.SLOT_F64 else torch.int64,
                               device=out_dev, pin_memory=on_host) for (_, ty, _, _) in slots]
            streamed["keys"], streamed["states"] = ok, os_
            return [t.data_ptr() for t in ok], [t.data_ptr() for t in os_]

        h.set_output_allocator(alloc)
        try:
            # the native side selects the device itself; outputs name it explicitly
            n_groups = h.execute(n, [k.data_ptr() for k in keys], [v.data_ptr() for v in vals], on_host, sptr)
        finally:
            h.set_output_allocator(None)
        if file_store:
            self.run_ids = self.store._adopt(h.run_rows(), len(keys), len(slots), self.config.page_capacity)
        mode = h.result_streamed() if streamed else 0
        self.streamed_output = mode == 2   # the columns were filled while the wide merge ran
        if mode:
            self._record(h, n, n_groups)
            return ColumnarResult([t[:n_groups] for t in streamed["keys"]],
                                  [t[:n_groups] for t in streamed["states"]])
        streamed.clear()
        return self._collect(h, n, n_groups, keys, slots, on_host, sptr)

    def in_stream_columns(self, keys, values=None, *, states=False, stream=None):
        """``in_stream_aggregate`` (bench.py:199-212) over columns already
        sorted on the key: every run of equal consecutive keys becomes one
        group (no sort, no memory budget, nothing spilled).  Same arguments
        and result as ``execute_columns``."""
        h, n, keys, vals, slots, on_host, sptr = self._prepare(keys, values, states, stream)
        n_groups = h.in_stream(n, [k.data_ptr() for k in keys], [v.data_ptr() for v in vals], on_host, sptr)
        return self._collect(h, n, n_groups, keys, slots, on_host, sptr)

    def hash_columns(self, keys, values=None, *, states=False, stream=None):
        """The hash-aggregation baseline (hashagg.py:73-198) over the same
        inputs as ``execute_columns``: groups in first-arrival order (the
        reference's in-memory table order), not sorted."""
        h, n, keys, vals, slots, on_host, sptr = self._prepare(keys, values, states, stream)
        n_groups = h.hash_aggregate(n, [k.data_ptr() for k in keys], [v.data_ptr() for v in vals], on_host, sptr)
        return self._collect(h, n, n_groups, keys, slots, on_host, sptr)

    def _prepare(self, keys, values, states, stream):
        torch = _torch()
        keys = list(keys)
        if len(keys) != self.schema.arity:
            raise InvalidInputError(f"expected {self.schema.arity} key columns, got {len(keys)}")
        n = int(keys[0].shape[0])
        for k in keys:
            if k.dim() != 1 or int(k.shape[0]) != n:
                raise InvalidInputError("key columns must be 1-D and of equal length")
        if states:
            vals = list(values or [])
            if len(vals) != self.schema.state_slots:
                raise InvalidInputError(f"expected {self.schema.state_slots} state columns, got {len(vals)}")
            slots = []
            for s, (op, col) in enumerate(zip(self.schema.slot_ops(), vals)):
                ty = _native.SLOT_F64 if col.dtype.is_floating_point else _native.SLOT_I64
                slots.append((_OP_CODES[op], ty, _native.SRC_COLUMN, s))
        else:
            vals, slots = self._slots_from_values(self._resolve_values(values))
        for v in vals:
            if v.dim() != 1 or int(v.shape[0]) != n:
                raise InvalidInputError("value columns must be 1-D and match the key length")
        on_host = keys[0].device.type == "cpu"
        cols = keys + vals
        for c in cols:
            if (c.device.type == "cpu") != on_host:
                raise InvalidInputError("all columns must live on the same device type")
        if not on_host:
            dev = keys[0].device
            self._device = dev
            for c in cols:
                if c.device != dev:
                    raise InvalidInputError("all columns must be on the same CUDA device")
        if not torch.cuda.is_available():
            raise ResourceError("the B200 operator needs a CUDA device (torch.cuda.is_available() is False)")
        keys = [k.contiguous() for k in keys]
        vals = [v.contiguous() for v in vals]
        key_codes = [_isa_dtype(k) for k in keys]
        for c in key_codes:
            if c in (_native.F32, _native.F64):
                raise InvalidInputError("key columns must be integer")
        val_codes = [_isa_dtype(v) for v in vals]
        h = self._handle(key_codes, val_codes, slots)
        if stream is None:
            stream = torch.cuda.current_stream(self._device_index())
        return h, n, keys, vals, slots, on_host, ctypes_stream(stream)

    def _collect(self, h, n, n_groups, keys, slots, on_host, sptr):
        torch = _torch()
        out_dev = torch.device("cpu") if on_host else keys[0].device
        pin = on_host
        out_keys = [torch.empty(n_groups, dtype=k.dtype, device=out_dev, pin_memory=pin) for k in keys]
        out_states = [torch.empty(n_groups, dtype=torch.float64 if ty == _native.SLOT_F64 else torch.int64,
                                  device=out_dev, pin_memory=pin)
                      for (_, ty, _, _) in slots]
        if n_groups:
            h.result_copy([t.data_ptr() for t in out_keys], [t.data_ptr() for t in out_states], on_host, sptr)
        self._record(h, n, n_groups)
        return ColumnarResult(out_keys, out_states)

    def intersect_columns(self, keys_a, keys_b, *, stream=None):
        """``merge_intersect`` (bench.py:536-550) of two strictly ascending
        key-column sets (e.g. two ``execute_columns`` outputs' keys): the keys
        present in both, ascending, as key columns."""
        torch = _torch()
        keys_a, keys_b = list(keys_a), list(keys_b)
        if len(keys_a) != self.schema.arity or len(keys_b) != self.schema.arity:
            raise InvalidInputError(f"expected {self.schema.arity} key columns per input")
        for ka, kb in zip(keys_a, keys_b):
            if ka.dtype != kb.dtype:
                raise InvalidInputError("both inputs need the same key dtypes")
        on_host = keys_a[0].device.type == "cpu"
        if any((k.device.type == "cpu") != on_host for k in keys_a + keys_b):
            raise InvalidInputError("all columns must live on the same device type")
        if not torch.cuda.is_available():
            raise ResourceError("the B200 operator needs a CUDA device (torch.cuda.is_available() is False)")
        if not on_host:
            self._device = keys_a[0].device
        keys_a = [k.contiguous() for k in keys_a]
        keys_b = [k.contiguous() for k in keys_b]
        na, nb = int(keys_a[0].shape[0]), int(keys_b[0].shape[0])
        h = self._handle([_isa_dtype(k) for k in keys_a], [], ())
        if stream is None:
            stream = torch.cuda.current_stream(self._device_index())
        sptr = ctypes_stream(stream)
        out_dev = torch.device("cpu") if on_host else keys_a[0].device
        out = [torch.empty(min(na, nb), dtype=k.dtype, device=out_dev, pin_memory=on_host) for k in keys_a]
        k = h.merge_intersect(na, [t.data_ptr() for t in keys_a], nb, [t.data_ptr() for t in keys_b],
                              [t.data_ptr() for t in out], on_host, sptr)
        return [t[:k] for t in out]

    def _record(self, h, n_rows, n_groups):
        """Fold the device ledger into ``ledger`` now; the per-execute details
        (cycles, run sizes, phases, plan, steps) are read from the handle on
        first access, keeping the per-call host overhead off the GPU's path."""
        led = h.metrics()
        for name in MetricsLedger.__slots__:
            setattr(self.ledger, name, getattr(self.ledger, name) + getattr(led, name))
        self._last = (h, n_rows, led)
        self._info = {}

    def phase_snapshot(self):
        """Raw per-phase device times of the last execute (cheap; turn into
        a dict with ``_native.phases_dict``)."""
        return self._last[0].phase_raw() if self._last is not None else None

    def _materialize(self):
        info = self._info
        if self._last is None:
            defaults = {"device_ledger": None, "cycles": [], "run_rows": [], "phase_stats": {},
                        "runs_after_generation": 0, "executed_steps": [], "initial_plan": None}
            for k, v in defaults.items():
                info.setdefault(k, v)
            return
        h, n_rows, led = self._last
        info.setdefault("device_ledger", led.as_dict())
        cycles = info.setdefault("cycles", h.cycles())
        run_rows = info.setdefault("run_rows", h.run_rows())
        info.setdefault("phase_stats", h.phase_stats())
        info.setdefault("runs_after_generation", len(run_rows))
        if "initial_plan" not in info:
            plan = None
            if run_rows:
                est = OutputEstimator(self.config.memory_budget)
                for c in cycles:
                    est.note_cycle(c)
                # replacement selection: the steady-state probe totals (sortagg.py:335-336)
                est.steady_probes = int(led.steady_probes)
                est.steady_absorbs = int(led.steady_absorbs)
                est.steady_resident_sum = int(led.steady_resident_sum)
                est.note_runs(run_rows)
                o_est = (self.config.output_size_hint if self.config.output_size_hint is not None
                         else est.estimate(n_rows))
                if self.config.merge_mode in (WIDE, TRADITIONAL):   # sortagg.py:764, 804-805
                    plan = plan_merge(run_rows, o_est, self.config)
            info["initial_plan"] = plan
        if "executed_steps" not in info:
            steps = []
            for stp in h.steps():
                if stp.kind == _native.STEP_WIDE:
                    steps.append({"kind": "wide", "fan_in": stp.fan_in, "rows_out": stp.rows_out,
                                  "preliminary_merges": 0})
                elif stp.kind == _native.STEP_TRADITIONAL:
                    steps.append({"kind": "traditional", "fan_in": stp.fan_in, "rows_in": stp.rows_in,
                                  "rows_out": stp.rows_out, "collapsed": bool(stp.collapsed),
                                  "level": stp.level})
                else:
                    steps.append({"kind": "final", "fan_in": stp.fan_in, "rows_out": stp.rows_out})
            info["executed_steps"] = steps

    # -- row-object compatibility path ------------------------------------------
    def execute(self, rows):
        """Aggregate an iterable of ``Row`` (key tuple, state tuple) and
        return the sorted list of aggregated ``Row`` (sortagg.py:744-747)."""
        rows = list(rows)
        if not rows:
            # nothing of a previous execute may leak into this one's details
            self._last = None
            self._info = {}
            self._materialize()
            return []
        keys_t, states_t = self._row_columns(rows)
        return self._rows_from(self.execute_columns(keys_t, states_t, states=True))

    def _row_columns(self, rows):
        """Row objects -> key columns (narrowest order-preserving dtypes) and
        state-slot columns, on this operator's CUDA device."""
        torch = _torch()
        if not torch.cuda.is_available():
            raise ResourceError("the B200 operator needs a CUDA device (torch.cuda.is_available() is False)")
        arity = self.schema.arity
        nslots = self.schema.state_slots
        key_cols = []
        for j in range(arity):
            col = [r.key[j] for r in rows]
            key_cols.append(_narrow(_int_column(col, f"key column {j}")))
        if sum(c.dtype.itemsize * 8 for c in key_cols) > 128:
            raise InvalidInputError("composite key values need more than 128 bits; "
                                    "the B200 operator supports keys up to 128 bits")
        state_cols = []
        for s in range(nslots):
            col = [r.state[s] for r in rows]
            if any(isinstance(v, float) for v in col):
                state_cols.append(np.asarray(col, dtype=np.float64))
            else:
                arr = _int_column(col, f"state slot {s}")
                if arr.dtype != np.int64:
                    raise InvalidInputError(f"state slot {s} does not fit int64")
                state_cols.append(arr)
        dev = torch.device("cuda", self._device_index())
        return ([torch.from_numpy(c).to(dev) for c in key_cols], [torch.from_numpy(c).to(dev) for c in state_cols])

    @staticmethod
    def _rows_from(res):
        out_keys = [k.cpu().numpy() for k in res.keys]
        out_states = [s.cpu().numpy() for s in res.states]
        key_lists = [_py_list(k) for k in out_keys]
        state_lists = [_py_list(s) for s in out_states]
        return [Row(tuple(kl[i] for kl in key_lists), tuple(sl[i] for sl in state_lists)) for i in range(res.n_groups)]


def _int_column(values, what):
    try:
        return np.asarray(values, dtype=np.int64)
    except (OverflowError, TypeError, ValueError):
        pass
    try:
        arr = np.asarray(values, dtype=np.uint64)
    except (OverflowError, TypeError, ValueError) as exc:
        raise InvalidInputError(f"{what}: values must be integers in [-2^63, 2^64)") from exc
    return arr


def _narrow(arr):
    """Smallest integer dtype holding every value (order preserving): keeps
    composite Row keys within the 128-bit normalized key."""
    if arr.size == 0:
        return arr
    lo, hi = int(arr.min()), int(arr.max())
    if lo >= 0:
        for dt in (np.uint8, np.uint16, np.uint32, np.uint64):
            if hi <= np.iinfo(dt).max:
                return arr.astype(dt)
    for dt in (np.int8, np.int16, np.int32, np.int64):
        if np.iinfo(dt).min <= lo and hi <= np.iinfo(dt).max:
            return arr.astype(dt)
    return arr


def _py_list(arr):
    if arr.dtype == np.uint64 or arr.dtype.kind in "iu":
        return [int(v) for v in arr.tolist()]
    return arr.tolist()


def ctypes_stream(stream):
    """cudaStream_t of a torch.cuda.Stream as an int (0 = legacy default)."""
    return int(stream.cuda_stream) if stream is not None else 0
