"""The C-ABI shared library: built for sm_100a, loadable without a GPU, and
exporting every entry point include/insortagg_b200.h declares (no compute)."""

import ctypes
import os
import re
import subprocess

from paper_2010_00152_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "insortagg_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"ISA_API\s+[\w\s\*]+?\b(isa_\w+)\s*\(", text)))


def test_header_declares_the_entry_points():
    syms = declared_symbols()
    for s in ("isa_create", "isa_execute", "isa_result_copy", "isa_metrics", "isa_destroy", "isa_last_error",
              "isa_partition", "isa_sample_keys"):
        assert s in syms
    assert sorted(_native.EXPORTED_SYMBOLS) == syms


def test_library_loads_and_exports_every_symbol():
    lib = _native.load()
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} not exported"
    assert "sm_100a" in _native.version()
    out = subprocess.run(["nm", "-D", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (isa_\w+)", out))
    assert exported == set(declared_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_validates_before_touching_the_device():
    cfg = _native.IsaConfig()
    cfg.memory_budget, cfg.page_capacity = 10, 6     # budget < 2 pages (sortagg.py:72-73)
    sch = _native.IsaSchema()
    sch.n_key_cols = 1
    sch.key_dtypes[0] = _native.I64
    lib = _native.load()
    assert not lib.isa_create(ctypes.byref(cfg), ctypes.byref(sch))
    assert b"memory budget must cover two pages" in lib.isa_last_error(None)
    cfg.memory_budget, cfg.page_capacity = 64, 8
    sch.n_key_cols = 3
    sch.key_dtypes[0] = sch.key_dtypes[1] = sch.key_dtypes[2] = _native.U64
    assert not lib.isa_create(ctypes.byref(cfg), ctypes.byref(sch))
    assert b"128 bits" in lib.isa_last_error(None)
    sch.n_key_cols = 1
    sch.key_dtypes[0] = _native.F64
    assert not lib.isa_create(ctypes.byref(cfg), ctypes.byref(sch))
    assert b"integer" in lib.isa_last_error(None)


def test_null_handle_contract():
    lib = _native.load()
    assert lib.isa_execute(None, 0, None, None, 0, None, None) == 3   # ISA_ERR_CONTRACT
    assert lib.isa_launch_count() >= 0


def test_create_rejects_32bit_overflowing_page_images():
    """A FileStore run of memory_budget groups whose page image would pass
    4 GiB is rejected up front (page offsets and sizes are 32-bit)."""
    cfg = _native.IsaConfig()
    cfg.memory_budget, cfg.page_capacity = 1 << 30, 100
    cfg.run_tier = _native.TIER_FILE
    sch = _native.IsaSchema()
    sch.n_key_cols = 1
    sch.key_dtypes[0] = _native.I64
    sch.n_val_cols = 1
    sch.val_dtypes[0] = _native.I64
    sch.n_slots = 2
    for s in range(2):
        sch.slot_op[s] = _native.OP_ADD
        sch.slot_type[s] = _native.SLOT_I64
        sch.slot_src[s] = _native.SRC_COLUMN
        sch.slot_col[s] = 0
    lib = _native.load()
    assert not lib.isa_create(ctypes.byref(cfg), ctypes.byref(sch))
    assert b"4 GiB" in lib.isa_last_error(None)
    cfg.run_tier = _native.TIER_AUTO
    cfg.hbm_run_budget = -1
    assert not lib.isa_create(ctypes.byref(cfg), ctypes.byref(sch))
    assert b"hbm_run_budget" in lib.isa_last_error(None)


def test_kernel_timing_toggle_without_a_device():
    """Kernel-family timing is host bookkeeping: toggling and reading it
    needs no GPU (nothing recorded -> zeros)."""
    _native.set_kernel_timing(True)
    st = _native.kernel_stats()
    _native.set_kernel_timing(False)
    assert set(st) == set(_native.KERNEL_FAMILIES)
    assert all(v["launches"] == 0 for v in st.values())
