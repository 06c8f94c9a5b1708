"""Shared fixtures: golden vectors produced by the reference (tools/make_golden.py)."""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_names():
    """End-to-end operator fixtures (pages_* hold reference run files,
    downstream_* the reference's sorted-output consumers, rs_* replacement
    selection, hash_* the HashAggregate baseline)."""
    names = (os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))
    return sorted(n for n in names if not n.startswith(("pages_", "downstream_", "rs_", "hash_")))


def rs_golden_names():
    """Replacement-selection fixtures (tools/make_golden_rs.py)."""
    names = (os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN_DIR, "rs_*.npz")))
    return sorted(names)


class Golden:
    """One reference-produced fixture: inputs, schema, expected output/ledger."""

    def __init__(self, name):
        self.name = name
        z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
        self.z = {k: z[k] for k in z.files}
        self.memory = int(self.z["memory_budget"])
        self.page = int(self.z["page_capacity"])
        self.aggs = [tuple(s.split(":")) for s in self.z["aggs"].tolist()]
        nk = int(self.z["n_key_cols"])
        if "in_k0" in self.z:
            self.keys = [self.z[f"in_k{j}"] for j in range(nk)]
            self.values = {n: self.z[f"in_v_{n}"] for n in self.z["value_names"].tolist()}
        else:
            from paper_2010_00152_b200 import workloads
            assert name == "cfg1_full"
            w = workloads.config1(device="cpu")
            self.keys = [w.keys[0].numpy()]
            self.values = {"v": w.values["v"].numpy()}
        self.n_groups = int(self.z["n_groups"])
        self.out_keys = [self.z[f"out_k{j}"] for j in range(nk)]
        ns = sum(1 for k in self.z if k.startswith("out_s"))
        self.out_slots = [self.z[f"out_s{s}"] for s in range(ns)]

    def schema(self):
        from paper_2010_00152_b200 import AggregateKind, AggregateSpec, ColumnSpec, Schema
        cols = [ColumnSpec(f"k{j}") for j in range(len(self.keys))]
        aggs = [AggregateSpec(n, AggregateKind(k), c or None) for n, k, c in self.aggs]
        return Schema(cols, aggs)

    def input_sha(self):
        import hashlib
        h = hashlib.sha256()
        for c in self.keys:
            h.update(np.ascontiguousarray(c).tobytes())
        for n in sorted(self.values):
            h.update(np.ascontiguousarray(self.values[n]).tobytes())
        return h.hexdigest()

    @property
    def single_wide(self):
        return list(self.z["plan_kinds"]) in ([], ["wide"])


@pytest.fixture(params=golden_names())
def golden(request):
    return Golden(request.param)


def assert_slots_equal(got, want, rel=1e-9, what="slot"):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, f"{what}: shape {got.shape} != {want.shape}"
    if want.dtype.kind == "f" or got.dtype.kind == "f":
        np.testing.assert_allclose(got.astype(np.float64), want.astype(np.float64), rtol=rel, atol=0,
                                   err_msg=what)
    else:
        assert np.array_equal(got.astype(np.int64), want.astype(np.int64)), f"{what}: integer mismatch"


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
