"""CPU-only checks of the boundary: the C-ABI library loads and exports every
symbol include/cdc_b200.h declares; host-only entry points behave (no compute
calls without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cdc_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(cdc_[a-z_0-9]+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_cdc_build", os.path.join(ROOT, "paper_2508_05797_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()   # cross-compiles for sm_100a; no GPU needed
    from paper_2508_05797_b200 import _lib
    return _lib


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ["cdc_chunk", "cdc_chunk_batch", "cdc_chunk_host", "cdc_chain", "cdc_extreme_byte_search",
              "cdc_range_scan", "cdc_workspace_size", "cdc_window_for_avg", "cdc_params_default",
              "cdc_max_boundaries", "cdc_abi_version", "cdc_last_error", "cdc_last_launch_count"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib.lib, s), s
    assert lib.lib.cdc_abi_version() == 1


def test_host_side_helpers(lib):
    from paper_2508_05797_b200 import api
    assert api.window_for_avg("ram", 8192) == 7936
    assert api.window_for_avg("ae_max", 4096) == 3840
    assert api.window_for_avg("ram", 300) == 150
    p = api.params("ae_max", avg_size=4096)
    assert (p.window, p.max_size) == (3840, 16384)
    assert api.max_boundaries(p, 0) == 1
    assert api.max_boundaries(p, 3841 * 10) == 11
    ws = api.workspace_size(p, 1, 256 << 20, 256 << 20)
    assert 0 < ws < 64 << 20
    with pytest.raises(api.CdcError):
        api.workspace_size(api.params("ram", window=8, max_size=8), 1, 100, 100)
    with pytest.raises(api.CdcError):
        api.window_for_avg("ram", 1)


def test_invalid_calls_fail_without_gpu(lib):
    from paper_2508_05797_b200 import api
    p = api.params("ram", window=8, max_size=64)
    n = ctypes.c_uint64()
    # null pointers are rejected before any CUDA call
    assert lib.lib.cdc_chunk(ctypes.byref(p), None, 0, None, 0, None, None, 0, None) == -1
    assert lib.lib.cdc_chunk_host(ctypes.byref(p), None, 10, None, 0, ctypes.byref(n)) == -1
    assert b"null" in lib.lib.cdc_last_error()


def test_plan_segments_host_only(lib):
    from paper_2508_05797_b200 import api
    for algo, avg, n in (("ae_max", 4096, 256 << 20), ("ram", 8192, 16 << 20), ("ram", 8192, 1 << 30),
                         ("ram", 8192, 100_000), ("ae_min", 512, (3 << 20) + 7)):
        p = api.params(algo, avg_size=avg)
        st = api.segment_starts(p, n)
        info = api.plan_info(p, 1, n, n)
        assert len(st) == info["segments"] >= 1
        assert st[0] == 0 and all(b > a for a, b in zip(st, st[1:])) and st[-1] < n
        align = 4096 if n // len(st) >= (64 << 10) else 16
        assert all(s % align == 0 for s in st)
        # no segment is tiny or more than twice the segment size plus an alignment unit
        lens = np.diff(st + [n])
        assert lens.max() < 2 * info["seg_bytes"] + 4096 + len(st)
    assert api.segment_starts(api.params("ram", avg_size=8192), 0) == []


def test_huge_window_rejected_not_crashing(lib):
    """window + 1 must not wrap in 32 bits (it used to divide by zero in the planner)."""
    from paper_2508_05797_b200 import api
    p = api.params("ram", window=0xFFFFFFFF, max_size=1 << 40)
    with pytest.raises(api.CdcError):
        api.workspace_size(p, 1, 1 << 33, 1 << 33)
    with pytest.raises(api.CdcError):
        api.plan_info(p, 1, 1 << 33, 1 << 33)
    p = api.params("ram", window=(1 << 31) - 1, max_size=1 << 40)
    assert api.workspace_size(p, 1, 1 << 33, 1 << 33) > 0


def test_batch_host_rejects_bad_offsets(lib):
    from paper_2508_05797_b200 import api
    p = api.params("ram", avg_size=8192)
    data = np.zeros(100, np.uint8)
    with pytest.raises(api.CdcError):
        api.chunk_batch_host(data, np.array([0, 60, 50, 100], np.uint64), p)


def test_maxp_window_for_avg_closed_form(lib):
    """Reading M5: h is the smallest window whose local maxima on uniform bytes
    are at least avg bytes apart on average, 1/P(h) >= avg with
    P(h) = sum_v (1/256) (v/256)^(2h) (computed here independently)."""
    from paper_2508_05797_b200 import api
    v = np.arange(256) / 256.0

    def spacing(h):
        return 256.0 / float((v ** (2 * h)).sum())

    for avg in (64, 512, 4096, 8192, 16384):
        h = api.window_for_avg("maxp", avg)
        assert spacing(h) >= avg and (h == 1 or spacing(h - 1) < avg), (avg, h)
    assert api.window_for_avg("maxp", 8192) == 447
    # workspace sizing is host-only; batches are not defined for MAXP
    p = api.params("maxp", avg_size=8192)
    assert api.workspace_size(p, 1, 1 << 30, 1 << 30) > (1 << 30) // 448 * 8
    assert api.workspace_size(p, 4, 1 << 20, 1 << 18) > 0  # batches of several streams
    with pytest.raises(api.CdcError):
        api.workspace_size(api.params("maxp", window=65537, max_size=1 << 20), 1, 1 << 20, 1 << 20)
