"""ORACLE — test infrastructure, never the product path.

CPU restatements of the reference algorithm used only by tests/, by
``__graft_entry__.smoke()`` as the checker, and by bench.py's cpu_baseline /
``--impl reference`` legs:

* ``reference_aggregate`` — numpy restatement of the reference's own
  correctness gate ``bench.reference_aggregate``
  (/root/reference/pkg/src/insortagg/bench.py:189-196): hash-map aggregation
  then ``sorted(table.items())``; here a stable lexicographic sort plus a
  segmented reduce (ints exact, floats in float64).
* ``rsw_sortagg`` — ctypes wrapper of rsw_oracle.c, the C restatement of
  ``index_run_generation`` (read-sort-write, sortagg.py:300-376) and
  ``wide_merge`` (sortagg.py:588-674) with the reference's spill ledger.
* ``rs_run_generation`` — pure-Python restatement of replacement-selection
  run generation with early aggregation (index_run_generation's RS branches,
  sortagg.py:333-343, 356-369; OrderedIndex generations / cursor /
  evict_range, memindex.py:186-263) for small inputs: run sizes, the
  OutputEstimator's steady-probe totals (sortagg.py:113-119).
* ``make_states`` / ``normalize_keys`` — Schema.make_state (core.py:162-182)
  over columns, and the order-preserving key image both oracles consume.

Pinned against the reference itself: tests/golden/*.npz hold outputs and
ledgers produced by running /root/reference/pkg/src/insortagg in this
container (tools/make_golden.py); tests/test_oracle.py checks both oracles
against every fixture.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle_rsw.so")

OPS = {"add": 0, "min": 1, "max": 2}


# ----------------------------------------------------------------- states ---

def slot_layout(schema):
    """[(op, agg_index, source)] per state slot, source 'one' | 'value'."""
    out = []
    for i, agg in enumerate(schema.aggregates):
        kind = agg.kind.value if hasattr(agg.kind, "value") else str(agg.kind)
        if kind == "count":
            out.append(("add", i, "one"))
        elif kind == "avg":
            out += [("add", i, "value"), ("add", i, "one")]
        else:
            out.append(({"sum": "add", "min": "min", "max": "max"}[kind], i, "value"))
    return out


def make_states(schema, values, n):
    """Schema.make_state over columns: list of per-slot numpy arrays
    (int64 for integer inputs and COUNT, float64 for float inputs)."""
    slots = []
    for op, i, src in slot_layout(schema):
        agg = schema.aggregates[i]
        if src == "one":
            slots.append(np.ones(n, dtype=np.int64))
            continue
        name = agg.column if agg.column is not None else agg.name
        col = np.asarray(values[name])
        if col.dtype.kind == "f":
            slots.append(col.astype(np.float64))
        else:
            slots.append(col.astype(np.int64))
    return slots


def slot_ops(schema):
    return [op for op, _, _ in slot_layout(schema)]


# ------------------------------------------------------------------- keys ---

def normalize_keys(key_cols):
    """Order-preserving 128-bit image (hi, lo) of composite integer keys:
    signed columns get their sign bit flipped, columns are concatenated most
    significant first (tuple order of core.py:265-288)."""
    widths = [np.asarray(c).dtype.itemsize * 8 for c in key_cols]
    total = sum(widths)
    if total > 128:
        raise ValueError("composite key wider than 128 bits")
    n = len(key_cols[0])
    hi = np.zeros(n, dtype=np.uint64)
    lo = np.zeros(n, dtype=np.uint64)
    pos = total
    for c, w in zip(key_cols, widths):
        c = np.asarray(c)
        pos -= w
        u = c.view(f"u{w // 8}").astype(np.uint64)
        if c.dtype.kind == "i":
            u ^= np.uint64(1 << (w - 1))
        if pos >= 64:
            hi |= u << np.uint64(pos - 64)
        else:
            lo |= u << np.uint64(pos)
            if pos > 0 and pos + w > 64:
                hi |= u >> np.uint64(64 - pos)
    return hi, lo


def denormalize_keys(hi, lo, dtypes):
    widths = [np.dtype(d).itemsize * 8 for d in dtypes]
    pos = sum(widths)
    cols = []
    for d, w in zip(dtypes, widths):
        pos -= w
        if pos >= 64:
            f = hi >> np.uint64(pos - 64)
        elif pos == 0:
            f = lo.copy()
        else:
            f = (lo >> np.uint64(pos)) | (hi << np.uint64(64 - pos))
        if w < 64:
            f = f & np.uint64((1 << w) - 1)
        if np.dtype(d).kind == "i":
            f = f ^ np.uint64(1 << (w - 1))
        cols.append(f.astype(f"u{w // 8}").view(d))
    return cols


# ------------------------------------------------------ numpy restatement ---

def reference_aggregate(key_cols, slot_cols, ops):
    """bench.reference_aggregate (bench.py:189-196) over columns.

    Returns (sorted unique key columns, aggregated slot columns)."""
    key_cols = [np.asarray(k) for k in key_cols]
    n = len(key_cols[0]) if key_cols else 0
    if n == 0:
        return [k[:0] for k in key_cols], [np.asarray(s)[:0] for s in slot_cols]
    order = np.lexsort(tuple(reversed(key_cols)))
    sk = [k[order] for k in key_cols]
    change = np.zeros(n, dtype=bool)
    change[0] = True
    for k in sk:
        change[1:] |= k[1:] != k[:-1]
    starts = np.flatnonzero(change)
    out_keys = [k[starts] for k in sk]
    out_slots = []
    for s, op in zip(slot_cols, ops):
        s = np.asarray(s)[order]
        if op == "add":
            out_slots.append(np.add.reduceat(s, starts))
        elif op == "min":
            out_slots.append(np.minimum.reduceat(s, starts))
        else:
            out_slots.append(np.maximum.reduceat(s, starts))
    return out_keys, out_slots


# ---------------------------------------------------------- C restatement ---

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        vp = ctypes.c_void_p
        lib.oracle_sortagg.restype = vp
        lib.oracle_sortagg.argtypes = [ctypes.c_int64, vp, vp, ctypes.c_int, vp, vp, vp, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int, vp, vp]
        lib.oracle_n_groups.restype = ctypes.c_int64
        lib.oracle_n_groups.argtypes = [vp]
        lib.oracle_copy.restype = None
        lib.oracle_copy.argtypes = [vp, vp, vp, vp]
        lib.oracle_ledger.restype = None
        lib.oracle_ledger.argtypes = [vp, vp]
        lib.oracle_cycles.restype = ctypes.c_int64
        lib.oracle_cycles.argtypes = [vp, vp, ctypes.c_int64]
        lib.oracle_free.restype = None
        lib.oracle_free.argtypes = [vp]
        _lib = lib
    return _lib


LEDGER_FIELDS = ("rows_spilled", "rows_read_back", "pages_written", "pages_read",
                 "merge_steps", "merge_levels", "runs", "n_groups")


def rsw_sortagg(key_cols, slot_cols, ops, memory_budget, page_capacity=100, nthreads=1, splitters=None):
    """Run the C restatement.  Returns (key columns, slot columns, ledger dict,
    cycles list).  ``splitters``: (hi, lo) arrays of nthreads-1 normalized keys
    for the key-range-partitioned multi-thread mode."""
    lib = _load()
    dtypes = [np.asarray(k).dtype for k in key_cols]
    hi, lo = normalize_keys(key_cols)
    n = len(lo)
    S = len(slot_cols)
    slots = [np.ascontiguousarray(np.asarray(s)).view(np.uint64) for s in slot_cols]
    types = [1 if np.asarray(s).dtype.kind == "f" else 0 for s in slot_cols]
    sp = (ctypes.c_void_p * max(1, S))(*[s.ctypes.data for s in slots])
    opa = (ctypes.c_int * max(1, S))(*[OPS[o] for o in ops])
    tya = (ctypes.c_int * max(1, S))(*types)
    shi = slo = None
    if nthreads > 1:
        if splitters is None:
            raise ValueError("multi-thread mode needs splitters")
        shi = np.ascontiguousarray(splitters[0], dtype=np.uint64)
        slo = np.ascontiguousarray(splitters[1], dtype=np.uint64)
    r = lib.oracle_sortagg(n, hi.ctypes.data, lo.ctypes.data, S, sp, opa, tya, memory_budget, page_capacity,
                           nthreads, shi.ctypes.data if shi is not None else None,
                           slo.ctypes.data if slo is not None else None)
    try:
        g = lib.oracle_n_groups(r)
        ohi = np.empty(g, dtype=np.uint64)
        olo = np.empty(g, dtype=np.uint64)
        outs = [np.empty(g, dtype=np.uint64) for _ in range(S)]
        op_ptrs = (ctypes.c_void_p * max(1, S))(*[o.ctypes.data for o in outs])
        lib.oracle_copy(r, ohi.ctypes.data, olo.ctypes.data, op_ptrs)
        led = np.zeros(8, dtype=np.int64)
        lib.oracle_ledger(r, led.ctypes.data)
        nc = lib.oracle_cycles(r, None, 0)
        cyc = np.zeros(max(1, nc), dtype=np.int64)
        lib.oracle_cycles(r, cyc.ctypes.data, nc)
    finally:
        lib.oracle_free(r)
    out_keys = denormalize_keys(ohi, olo, dtypes)
    out_slots = [o.view(np.float64) if t else o.view(np.int64) for o, t in zip(outs, types)]
    ledger = dict(zip(LEDGER_FIELDS, (int(x) for x in led)))
    return out_keys, out_slots, ledger, [int(c) for c in cyc[:nc]]


def range_splitters(key_cols, parts, sample=65536, seed=0):
    """nparts-1 normalized splitter keys from a sample (for the multi-thread
    CPU baseline)."""
    hi, lo = normalize_keys(key_cols)
    n = len(lo)
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, n, min(n, sample)) if n else np.zeros(0, dtype=np.int64)
    order = np.lexsort((lo[idx], hi[idx]))
    shi, slo = hi[idx][order], lo[idx][order]
    picks = [int(len(order) * (t + 1) / parts) for t in range(parts - 1)]
    picks = [min(p, len(order) - 1) for p in picks]
    return shi[picks], slo[picks]


def parse_run_pages(data, arity, slots):
    """Restatement of parse_page over a whole run file (runstore.py:120-142):
    12-byte header (row_count, byte_length, crc32 of the body), high key,
    rows of int64 (key columns, then state slots).  Returns (keys
    [arity x rows], states [slots x rows], page row counts); raises
    ValueError on a length or checksum mismatch."""
    import struct
    import zlib
    keys, states, counts = [[] for _ in range(arity)], [[] for _ in range(slots)], []
    off, width = 0, arity + slots
    while off < len(data):
        rows, length, crc = struct.unpack_from("<III", data, off)
        body = data[off + 12: off + 12 + length]
        if len(body) != length or (zlib.crc32(body) & 0xFFFFFFFF) != crc:
            raise ValueError(f"page at {off}: bad length or checksum")
        vals = np.frombuffer(body, dtype="<i8")
        if len(vals) != arity + rows * width:
            raise ValueError(f"page at {off}: row count does not match the body")
        hk = vals[:arity]
        rv = vals[arity:].reshape(rows, width)
        if rows and not np.array_equal(hk, rv[-1, :arity]):
            raise ValueError(f"page at {off}: high key is not the last row's key")
        for j in range(arity):
            keys[j].append(rv[:, j])
        for s_ in range(slots):
            states[s_].append(rv[:, arity + s_])
        counts.append(rows)
        off += 12 + length
    cat = lambda parts: np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
    return [cat(k) for k in keys], [cat(s_) for s_ in states], counts


# ------------------------------------------------- replacement selection ---

def rs_run_generation(keys, memory_budget, chunk):
    """Replacement selection with early aggregation over a sequence of
    (hashable, orderable) keys; states are not tracked (the runs' rows are
    what the ledger needs).  Returns (run sizes, (steady probes, steady
    absorbs, steady resident sum)).

    Follows sortagg.py:333-369 row by row: a key at or below the eviction
    cursor lives in the next generation; a new key with the index full makes
    the current generation evict its `chunk` lowest keys into the open run
    (cursor = last evicted key); an exhausted generation closes the run and
    the next one becomes current; the row is retried."""
    import bisect
    cur, nxt = [], []
    cursor = None
    runs, open_run = [], None
    spilling = False
    probes = absorbs = ressum = 0
    for k in keys:
        resident = len(cur) + len(nxt)
        first = True
        while True:
            passed = cursor is not None and k <= cursor
            tree = nxt if passed else cur
            i = bisect.bisect_left(tree, k)
            found = i < len(tree) and tree[i] == k
            if found:
                outcome = "absorbed"
            elif len(cur) + len(nxt) >= memory_budget:
                outcome = "evict"
            else:
                tree.insert(i, k)
                outcome = "inserted"
            if first and spilling:
                probes += 1
                ressum += resident
                absorbs += outcome == "absorbed"
            first = False
            if outcome != "evict":
                break
            spilling = True
            if open_run is None:
                open_run = 0
            ev = cur[:chunk]
            del cur[:chunk]
            open_run += len(ev)
            if ev:
                cursor = ev[-1]
            if not cur:
                runs.append(open_run)
                open_run = None
                cur, nxt = nxt, []
                cursor = None
    if runs or open_run is not None:
        while True:
            if cur:
                open_run = (open_run or 0) + len(cur)
                cur = []
                continue
            if open_run is not None:
                runs.append(open_run)
                open_run = None
            if not nxt:
                break
            cur, nxt = nxt, []
    return runs, (probes, absorbs, ressum)

