"""ctypes binding of libinsortagg_b200.so (declared in include/insortagg_b200.h).

The library is the product path: there is no Python or CPU fallback.  If the
shared object is missing or cannot be loaded, every operator call raises
ResourceError naming the file and the build command.
"""

from __future__ import annotations

import ctypes
import os

from .core import (
    ContractViolationError,
    CorruptionError,
    InvalidInputError,
    OrderingViolationError,
    PlanningError,
    ResourceError,
)

LIB_NAME = "libinsortagg_b200.so"
LIB_PATH = os.environ.get("ISA_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

MAX_KEY_COLS = 8
MAX_SLOTS = 16
MAX_VAL_COLS = 16

# isa_dtype
U8, I8, U16, I16, U32, I32, U64, I64, F32, F64 = range(1, 11)
DTYPE_BITS = {U8: 8, I8: 8, U16: 16, I16: 16, U32: 32, I32: 32, U64: 64, I64: 64, F32: 32, F64: 64}
OP_ADD, OP_MIN, OP_MAX = 0, 1, 2
SLOT_I64, SLOT_F64 = 0, 1
SRC_ONE, SRC_COLUMN = 0, 1
TIER_HOST, TIER_HBM, TIER_FILE, TIER_AUTO = 0, 1, 2, 3

_STATUS_ERRORS = {
    1: InvalidInputError,
    2: OrderingViolationError,
    3: ContractViolationError,
    4: CorruptionError,
    5: ResourceError,
    6: PlanningError,
    7: ResourceError,
}

EXPORTED_SYMBOLS = (
    "isa_version", "isa_create", "isa_destroy", "isa_execute", "isa_result_copy",
    "isa_metrics", "isa_cycles", "isa_run_rows", "isa_last_error",
    "isa_sample_keys", "isa_partition", "isa_phase_stats", "isa_launch_count", "isa_steps",
    "isa_set_spill_dir", "isa_in_stream_aggregate", "isa_hash_aggregate", "isa_merge_intersect", "isa_partition_counts",
    "isa_scatter_to_peers", "isa_ipc_handle", "isa_ipc_open", "isa_ipc_close",
    "isa_set_kernel_timing", "isa_kernel_stats", "isa_kernel_timing_reserve", "isa_set_output_allocator",
    "isa_result_streamed", "isa_execute_multi",
)

# isa_kernel_family (kernel-true roofline families)
KERNEL_FAMILIES = ("scatter", "hist", "collapse", "pack", "unpack", "absorb", "merge", "flush", "export", "hot_probe",
                   "hot_absorb")

PHASES = ("absorb", "sort", "flush", "collapse", "table_merge", "wm_sort", "wm_collapse",
          "run_generation", "wide_merge", "probe", "hot")


class IsaPhase(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double), ("calls", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("bytes", ctypes.c_int64)]


class IsaKstat(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double), ("launches", ctypes.c_int64), ("bytes", ctypes.c_int64)]


class IsaConfig(ctypes.Structure):
    _fields_ = [
        ("memory_budget", ctypes.c_int64),
        ("page_capacity", ctypes.c_int64),
        ("run_tier", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("chunk_rows_max", ctypes.c_int64),
        ("window_rows", ctypes.c_int64),
        ("merge_window_rows", ctypes.c_int64),
        ("preaggregate", ctypes.c_int32),
        ("merge_mode", ctypes.c_int32),
        ("output_size_hint", ctypes.c_int64),
        ("run_codec", ctypes.c_int32),
        ("hot_absorb", ctypes.c_int32),
        ("hbm_run_budget", ctypes.c_int64),
        ("run_generation", ctypes.c_int32),
        ("eviction_chunk", ctypes.c_int32),
    ]


class IsaStep(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("collapsed", ctypes.c_int32), ("fan_in", ctypes.c_int64),
                ("rows_in", ctypes.c_int64), ("rows_out", ctypes.c_int64), ("level", ctypes.c_int64)]


MERGE_WIDE, MERGE_TRADITIONAL, MERGE_SEPARATE = 0, 1, 2
STEP_WIDE, STEP_TRADITIONAL, STEP_FINAL = 0, 1, 2


class IsaSchema(ctypes.Structure):
    _fields_ = [
        ("n_key_cols", ctypes.c_int32),
        ("key_dtypes", ctypes.c_int32 * MAX_KEY_COLS),
        ("n_val_cols", ctypes.c_int32),
        ("val_dtypes", ctypes.c_int32 * MAX_VAL_COLS),
        ("n_slots", ctypes.c_int32),
        ("slot_op", ctypes.c_int32 * MAX_SLOTS),
        ("slot_type", ctypes.c_int32 * MAX_SLOTS),
        ("slot_src", ctypes.c_int32 * MAX_SLOTS),
        ("slot_col", ctypes.c_int32 * MAX_SLOTS),
    ]


class IsaLedger(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "row_comparisons", "ovc_decided_comparisons", "column_value_accesses",
        "hash_computations", "rows_spilled", "rows_read_back", "pages_written",
        "pages_read", "merge_steps", "merge_levels", "runs_after_generation",
        "rows_seen", "n_groups", "merge_windows", "chunks", "bytes_h2d",
        "bytes_d2h", "kernel_launches")] + [
        ("ms_run_generation", ctypes.c_double),
        ("ms_wide_merge", ctypes.c_double),
        ("ms_host_sync", ctypes.c_double),
        ("ms_spill_wait", ctypes.c_double),
        ("steady_probes", ctypes.c_int64),
        ("steady_absorbs", ctypes.c_int64),
        ("steady_resident_sum", ctypes.c_int64),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_load_error = None


def load():
    """Load (once) and return the CDLL; raise ResourceError when absent."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise ResourceError(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = (f"{LIB_PATH} is missing: build it with "
                       "`make -C paper_2010_00152_b200/csrc` or __graft_entry__.build()")
        raise ResourceError(_load_error)
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        _load_error = f"cannot load {LIB_PATH}: {exc}"
        raise ResourceError(_load_error) from exc
    vp = ctypes.c_void_p
    pp = ctypes.POINTER(ctypes.c_void_p)
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.isa_version.restype = ctypes.c_char_p
    lib.isa_version.argtypes = []
    lib.isa_create.restype = vp
    lib.isa_create.argtypes = [ctypes.POINTER(IsaConfig), ctypes.POINTER(IsaSchema)]
    lib.isa_destroy.restype = None
    lib.isa_destroy.argtypes = [vp]
    lib.isa_execute.restype = ctypes.c_int
    lib.isa_execute.argtypes = [vp, ctypes.c_int64, pp, pp, ctypes.c_int32, vp, i64p]
    lib.isa_result_copy.restype = ctypes.c_int
    lib.isa_result_copy.argtypes = [vp, pp, pp, ctypes.c_int32, vp]
    lib.isa_in_stream_aggregate.restype = ctypes.c_int
    lib.isa_in_stream_aggregate.argtypes = [vp, ctypes.c_int64, pp, pp, ctypes.c_int32, vp, i64p]
    lib.isa_hash_aggregate.restype = ctypes.c_int
    lib.isa_hash_aggregate.argtypes = [vp, ctypes.c_int64, pp, pp, ctypes.c_int32, vp, i64p]
    lib.isa_merge_intersect.restype = ctypes.c_int
    lib.isa_merge_intersect.argtypes = [vp, ctypes.c_int64, pp, ctypes.c_int64, pp, pp, ctypes.c_int32, vp, i64p]
    lib.isa_execute_multi.restype = ctypes.c_int
    lib.isa_execute_multi.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, i64p, ctypes.POINTER(pp), ctypes.POINTER(pp),
                                      pp, i64p]
    lib.isa_partition_counts.restype = ctypes.c_int
    lib.isa_partition_counts.argtypes = [vp, ctypes.c_int64, pp, vp, vp, ctypes.c_int32, i64p, vp]
    lib.isa_scatter_to_peers.restype = ctypes.c_int
    lib.isa_scatter_to_peers.argtypes = [vp, ctypes.c_int64, pp, pp, pp, i64p, vp]
    lib.isa_ipc_handle.restype = ctypes.c_int
    lib.isa_ipc_handle.argtypes = [vp, vp]
    lib.isa_ipc_open.restype = ctypes.c_int
    lib.isa_ipc_open.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]
    lib.isa_ipc_close.restype = ctypes.c_int
    lib.isa_ipc_close.argtypes = [vp]
    lib.isa_set_spill_dir.restype = ctypes.c_int
    lib.isa_set_spill_dir.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
    lib.isa_set_output_allocator.restype = ctypes.c_int
    lib.isa_set_output_allocator.argtypes = [vp, ALLOC_FN, vp]
    lib.isa_result_streamed.restype = ctypes.c_int
    lib.isa_result_streamed.argtypes = [vp]
    lib.isa_metrics.restype = ctypes.c_int
    lib.isa_metrics.argtypes = [vp, ctypes.POINTER(IsaLedger)]
    lib.isa_cycles.restype = ctypes.c_int64
    lib.isa_cycles.argtypes = [vp, i64p, ctypes.c_int64]
    lib.isa_run_rows.restype = ctypes.c_int64
    lib.isa_run_rows.argtypes = [vp, i64p, ctypes.c_int64]
    lib.isa_last_error.restype = ctypes.c_char_p
    lib.isa_last_error.argtypes = [vp]
    lib.isa_steps.restype = ctypes.c_int64
    lib.isa_steps.argtypes = [vp, ctypes.POINTER(IsaStep), ctypes.c_int64]
    lib.isa_phase_stats.restype = ctypes.c_int
    lib.isa_phase_stats.argtypes = [vp, ctypes.POINTER(IsaPhase), ctypes.c_int]
    lib.isa_launch_count.restype = ctypes.c_int64
    lib.isa_launch_count.argtypes = []
    lib.isa_set_kernel_timing.restype = None
    lib.isa_set_kernel_timing.argtypes = [ctypes.c_int32]
    lib.isa_kernel_timing_reserve.restype = None
    lib.isa_kernel_timing_reserve.argtypes = [ctypes.c_int64]
    lib.isa_kernel_stats.restype = ctypes.c_int
    lib.isa_kernel_stats.argtypes = [ctypes.POINTER(IsaKstat), ctypes.c_int]
    lib.isa_sample_keys.restype = ctypes.c_int
    lib.isa_sample_keys.argtypes = [vp, ctypes.c_int64, pp, ctypes.c_int64, vp, vp, vp]
    lib.isa_partition.restype = ctypes.c_int
    lib.isa_partition.argtypes = [vp, ctypes.c_int64, pp, pp, vp, vp, ctypes.c_int32, pp, pp, i64p, vp]
    _lib = lib
    return lib


def version():
    return load().isa_version().decode()


def launch_count():
    """Kernels launched by libinsortagg_b200 so far in this process."""
    return int(load().isa_launch_count())


def set_kernel_timing(on):
    """CUDA-event timing of the library's main kernels (this host thread)."""
    load().isa_set_kernel_timing(1 if on else 0)


def kernel_timing_reserve(events):
    """Pre-create CUDA events for kernel timing (two per timed launch)."""
    load().isa_kernel_timing_reserve(int(events))


def kernel_stats():
    """Per kernel family {ms, launches, bytes} since the last call (call after
    synchronizing the device)."""
    arr = (IsaKstat * len(KERNEL_FAMILIES))()
    load().isa_kernel_stats(arr, len(KERNEL_FAMILIES))
    return {name: {"ms": arr[i].ms, "launches": arr[i].launches, "bytes": arr[i].bytes}
            for i, name in enumerate(KERNEL_FAMILIES)}


def phases_dict(arr):
    return {name: {"ms": arr[i].ms, "calls": arr[i].calls, "rows": arr[i].rows, "bytes": arr[i].bytes}
            for i, name in enumerate(PHASES)}


# isa_alloc_fn: int fn(void* user, int64_t capacity, void** key_out, void** slot_out)
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p),
                            ctypes.POINTER(ctypes.c_void_p))


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


class Handle:
    """One native operator instance (not thread-safe; one per host thread)."""

    def __init__(self, config: IsaConfig, schema: IsaSchema):
        self._lib = load()
        self.schema = schema
        h = self._lib.isa_create(ctypes.byref(config), ctypes.byref(schema))
        if not h:
            msg = self._lib.isa_last_error(None).decode()
            raise InvalidInputError(msg) if "CUDA" not in msg and "cuda" not in msg else ResourceError(msg)
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.isa_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def _check(self, status):
        if status != 0:
            msg = self._lib.isa_last_error(self._h).decode()
            raise _STATUS_ERRORS.get(status, ResourceError)(msg)

    def execute(self, n_rows, key_ptrs, val_ptrs, on_host, stream):
        out = ctypes.c_int64(0)
        self._check(self._lib.isa_execute(self._h, n_rows, _ptr_array(key_ptrs), _ptr_array(val_ptrs),
                                          1 if on_host else 0, stream, ctypes.byref(out)))
        return out.value

    def in_stream(self, n_rows, key_ptrs, val_ptrs, on_host, stream):
        out = ctypes.c_int64(0)
        self._check(self._lib.isa_in_stream_aggregate(self._h, n_rows, _ptr_array(key_ptrs), _ptr_array(val_ptrs),
                                                      1 if on_host else 0, stream, ctypes.byref(out)))
        return out.value

    def hash_aggregate(self, n_rows, key_ptrs, val_ptrs, on_host, stream):
        out = ctypes.c_int64(0)
        self._check(self._lib.isa_hash_aggregate(self._h, n_rows, _ptr_array(key_ptrs), _ptr_array(val_ptrs),
                                                 1 if on_host else 0, stream, ctypes.byref(out)))
        return out.value

    def merge_intersect(self, n_a, a_ptrs, n_b, b_ptrs, out_ptrs, on_host, stream):
        out = ctypes.c_int64(0)
        self._check(self._lib.isa_merge_intersect(self._h, n_a, _ptr_array(a_ptrs), n_b, _ptr_array(b_ptrs),
                                                  _ptr_array(out_ptrs), 1 if on_host else 0, stream,
                                                  ctypes.byref(out)))
        return out.value

    def partition_counts(self, n_rows, key_ptrs, split_lo, split_hi, n_split, stream):
        counts = (ctypes.c_int64 * (n_split + 1))()
        self._check(self._lib.isa_partition_counts(self._h, n_rows, _ptr_array(key_ptrs), split_lo, split_hi,
                                                   n_split, counts, stream))
        return [counts[i] for i in range(n_split + 1)]

    def scatter_to_peers(self, n_rows, key_ptrs, val_ptrs, peer_ptrs, peer_offsets, stream):
        offs = (ctypes.c_int64 * max(1, len(peer_offsets)))(*peer_offsets)
        self._check(self._lib.isa_scatter_to_peers(self._h, n_rows, _ptr_array(key_ptrs), _ptr_array(val_ptrs),
                                                   _ptr_array(peer_ptrs), offs, stream))

    def set_spill_dir(self, directory, first_run_id):
        self._check(self._lib.isa_set_spill_dir(self._h, os.fsencode(directory), int(first_run_id)))

    def set_output_allocator(self, fn):
        """``fn(capacity) -> (key_ptrs, slot_ptrs)`` (or None to decline) is
        called by the native wide merge for the caller-owned output columns;
        ``None`` removes the allocator."""
        if fn is None:
            self._alloc_cb = None
            self._check(self._lib.isa_set_output_allocator(self._h, ctypes.cast(None, ALLOC_FN), None))
            return

        def cb(_user, capacity, key_out, slot_out):
            try:
                ptrs = fn(int(capacity))
                if ptrs is None:
                    return 1
                for i, p in enumerate(ptrs[0]):
                    key_out[i] = p
                for i, p in enumerate(ptrs[1]):
                    slot_out[i] = p
                return 0
            except Exception:   # an allocation failure must not unwind through the C frames
                return 1

        self._alloc_cb = ALLOC_FN(cb)   # keep the thunk alive while the handle may call it
        self._check(self._lib.isa_set_output_allocator(self._h, self._alloc_cb, None))

    def result_streamed(self):
        """0: read with result_copy; 1: the allocator's columns were filled at
        the end of the execute; 2: while the wide merge ran."""
        return int(self._lib.isa_result_streamed(self._h))

    def result_copy(self, key_ptrs, slot_ptrs, on_host, stream):
        self._check(self._lib.isa_result_copy(self._h, _ptr_array(key_ptrs), _ptr_array(slot_ptrs),
                                              1 if on_host else 0, stream))

    def metrics(self):
        led = IsaLedger()
        self._check(self._lib.isa_metrics(self._h, ctypes.byref(led)))
        return led

    def cycles(self):
        n = self._lib.isa_cycles(self._h, None, 0)
        buf = (ctypes.c_int64 * max(1, n))()
        self._lib.isa_cycles(self._h, buf, n)
        return [buf[i] for i in range(n)]

    def phase_raw(self):
        arr = (IsaPhase * len(PHASES))()
        self._lib.isa_phase_stats(self._h, arr, len(PHASES))
        return arr

    def phase_stats(self):
        return phases_dict(self.phase_raw())

    def steps(self):
        cnt = self._lib.isa_steps(self._h, None, 0)
        arr = (IsaStep * max(1, cnt))()
        self._lib.isa_steps(self._h, arr, cnt)
        return [arr[i] for i in range(cnt)]

    def run_rows(self):
        n = self._lib.isa_run_rows(self._h, None, 0)
        buf = (ctypes.c_int64 * max(1, n))()
        self._lib.isa_run_rows(self._h, buf, n)
        return [buf[i] for i in range(n)]

    def sample_keys(self, n_rows, key_ptrs, stride, out_lo, out_hi, stream):
        self._check(self._lib.isa_sample_keys(self._h, n_rows, _ptr_array(key_ptrs), stride,
                                              out_lo, out_hi, stream))

    def partition(self, n_rows, key_ptrs, val_ptrs, split_lo, split_hi, n_split, key_out, val_out, stream):
        counts = (ctypes.c_int64 * (n_split + 1))()
        self._check(self._lib.isa_partition(self._h, n_rows, _ptr_array(key_ptrs), _ptr_array(val_ptrs),
                                            split_lo, split_hi, n_split, _ptr_array(key_out),
                                            _ptr_array(val_out), counts, stream))
        return [counts[i] for i in range(n_split + 1)]


def execute_multi(handles, n_rows, key_ptrs, val_ptrs, streams=None):
    """isa_execute_multi over ``handles`` (one per device): shard g has
    ``n_rows[g]`` rows in the device columns ``key_ptrs[g]`` / ``val_ptrs[g]``.
    Returns the group count of every key range."""
    g = len(handles)
    lib = load()
    hs = (ctypes.c_void_p * g)(*[h._h for h in handles])
    rows = (ctypes.c_int64 * g)(*[int(x) for x in n_rows])
    karr = [_ptr_array(k) for k in key_ptrs]
    varr = [_ptr_array(v) for v in val_ptrs]
    pp_t = ctypes.POINTER(ctypes.c_void_p)
    kk = (pp_t * g)(*[ctypes.cast(a, pp_t) for a in karr])
    vv = (pp_t * g)(*[ctypes.cast(a, pp_t) for a in varr])
    st = _ptr_array(streams) if streams else None
    out = (ctypes.c_int64 * g)()
    status = lib.isa_execute_multi(hs, g, rows, kk, vv, st, out)
    if status != 0:
        msg = lib.isa_last_error(handles[0]._h).decode()
        raise _STATUS_ERRORS.get(status, ResourceError)(msg)
    return [int(x) for x in out]


def ipc_handle(ptr):
    """72-byte CUDA IPC handle of a device pointer (allocation handle + offset)."""
    buf = ctypes.create_string_buffer(72)
    if load().isa_ipc_handle(ctypes.c_void_p(ptr), buf) != 0:
        raise ResourceError("cudaIpcGetMemHandle failed")
    return bytes(buf.raw)


def ipc_open(handle):
    """Map a peer's pointer: returns (allocation base for ipc_close, pointer)."""
    base, ptr = ctypes.c_void_p(0), ctypes.c_void_p(0)
    if load().isa_ipc_open(ctypes.create_string_buffer(handle, 72), ctypes.byref(base), ctypes.byref(ptr)) != 0:
        raise ResourceError("cudaIpcOpenMemHandle failed")
    return base.value, ptr.value


def ipc_close(base):
    load().isa_ipc_close(ctypes.c_void_p(base))
