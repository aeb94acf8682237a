"""The C-ABI library loads on a CPU-only box and exports the declared surface.

No kernel is launched here: only descriptor validation and planning, which
are host code inside the library.
"""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2006_13486_b200 import _native
from paper_2006_13486_b200.device import chain_fields
from paper_2006_13486_b200.sdmm import make_desc
from paper_2006_13486_b200 import workloads as wl

from conftest import ROOT


def declared_functions():
    text = open(os.path.join(ROOT, "include", "rbgp4.h")).read()
    return sorted(set(re.findall(r"\b(rbgp4_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert set(declared_functions()) == set(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.rbgp4_abi_version() == 3


def test_desc_struct_layout():
    # two int64 groups (5) + ten int32 fields -> 80 bytes, no padding surprises
    assert ctypes.sizeof(_native.Desc) == 5 * 8 + 10 * 4


def _desc(cfg, n=None):
    chain = wl.build_chain(cfg)
    n = cfg.n_cols if n is None else n
    return make_desc(chain_fields(chain), n, n, n)


def test_supported_matrix():
    lib = _native.lib()
    d = _desc(wl.C1A)
    exact, ffma = _native.COMPUTE["exact"], _native.COMPUTE["ffma"]
    assert lib.rbgp4_sdmm_supported(ctypes.byref(d), exact, _native.F32, _native.F32) == 1
    assert lib.rbgp4_sdmm_supported(ctypes.byref(d), ffma, _native.F64, _native.F64) == 1
    # SIMT output type must equal the operand type
    assert lib.rbgp4_sdmm_supported(ctypes.byref(d), exact, _native.F32, _native.F64) == 0
    assert "same type" in _native.last_error()
    assert lib.rbgp4_sdmm_supported(ctypes.byref(d), 9, _native.F32, _native.F32) == 0
    assert lib.rbgp4_workspace_size(ctypes.byref(d), exact, _native.F32) == 0


def test_inconsistent_descriptor_rejected():
    lib = _native.lib()
    d = _desc(wl.C1A)
    d.rows += 1
    assert lib.rbgp4_sdmm_supported(ctypes.byref(d), 0, _native.F32, _native.F32) == 0
    assert "disagrees" in _native.last_error()
    rc = lib.rbgp4_sdmm(ctypes.byref(d), 0, 0, 0, None, None, None, None, None, None, 0, None)
    assert rc == -1


def test_leading_dimension_rejected():
    lib = _native.lib()
    d = _desc(wl.C1A)
    d.ld_in = d.n_cols - 1
    assert lib.rbgp4_sdmm_supported(ctypes.byref(d), 0, _native.F32, _native.F32) == 0
    assert "leading" in _native.last_error()


def test_chain_kernel_argument_checks():
    lib = _native.lib()
    one = (ctypes.c_int32 * 1)(4)
    off = (ctypes.c_int64 * 1)(0)
    rc = lib.rbgp4_chain_sdmm(0, one, one, one, off, None, 0, None, None, None, 8, 8, 8, None)
    assert rc == -1 and "chain length" in _native.last_error()
    rc = lib.rbgp4_chain_sdmm(1, one, one, one, off, None, 7, None, None, None, 8, 8, 8, None)
    assert rc == -1


def test_product_path_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2006_13486_b200 as ks
    chain, w, inp = wl.make_operands(wl.C1A)
    with pytest.raises(ks.DeviceError):
        ks.rbgp4mm(w, inp, ks.tiling_for_chain(chain))


def test_prepared_section_carries_the_tc16_relayout(plan_options):
    """rbgp4_prepare_size (host-only arithmetic): the TC16 shape (16x16 blocks, g_i (8,8) of degree
    2) gets the column-block relayout of its values (same byte count as the values) in its prepared
    section; g_i of degree 4 gets the K5 slice relayout (the values plus zero padding); option
    relayout=0 removes every value relayout."""
    lib = _native.lib()

    def prep_bytes(sp_i):
        cfg = wl.SweepConfig("p", (4, 36), 0.5, (1, 1), (8, 8), sp_i, (16, 16), n_cols=1, seed=0)
        chain = wl.build_chain(cfg)
        d = make_desc(chain_fields(chain), 4096, 4096, 4096)
        return lib.rbgp4_prepare_size(ctypes.byref(d), 3), chain.num_left * chain.row_nnz * 2

    size, values = prep_bytes(0.75)
    assert size >= values
    size4, values4 = prep_bytes(0.5)
    assert size4 >= values4
    plan_options("relayout", 0)
    assert prep_bytes(0.75)[0] < values
    assert prep_bytes(0.5)[0] < values4


def test_plan_options_are_explicit_and_thread_local():
    """Plan overrides go through rbgp4_set_option (thread-local), never the process environment."""
    import threading

    from paper_2006_13486_b200.errors import DeviceError
    lib = _native.lib()
    assert _native.get_option("relayout") == -1 and _native.get_option("pdl") == 1
    with _native.options(relayout=0, ksplit=2):
        assert _native.get_option("relayout") == 0 and _native.get_option("ksplit") == 2
        seen = {}
        th = threading.Thread(target=lambda: seen.update(r=_native.get_option("relayout")))
        th.start()
        th.join()
        assert seen["r"] == -1          # another thread keeps the defaults
    assert _native.get_option("relayout") == -1 and _native.get_option("ksplit") == 0
    with pytest.raises(DeviceError, match="unknown option"):
        _native.set_option("no_such_knob", 1)
    with pytest.raises(DeviceError, match="outside"):
        _native.set_option("stages", 99)
    if not lib.rbgp4_debug_build():  # the release library carries no trace / ablation hooks
        with pytest.raises(DeviceError, match="debug build"):
            _native.set_option("debug", 8)
    lib.rbgp4_reset_options()


def test_no_environment_reads_in_the_library_sources():
    """No getenv in the CUDA sources: the launch paths are steered only by rbgp4_set_option."""
    import glob
    for path in glob.glob(os.path.join(ROOT, "paper_2006_13486_b200", "csrc", "*.c*")):
        assert "getenv" not in open(path).read(), path


def test_prepared_section_sizes_follow_the_k5_modes(plan_options):
    """rbgp4_prepare_size (host-only): the K5 slice section of a chain with a complete g_o holds the
    MERGED tile-row pairs -- per virtual tile-row (2 x 128 rows) and step, 8 K16 slices x 64 union
    rows x 16 k of bf16 (zero-padded) -- and option merge=0 falls back to unmerged 128-row tiles
    (the TC16 path, K4's relayout plus the row-group copy); 4x4 blocks get 4 slices per 64-row step."""
    lib = _native.lib()

    def size(g_o, sp_o, g_i, sp_i, g_b):
        cfg = wl.SweepConfig("p", g_o, sp_o, (1, 1), g_i, sp_i, g_b, n_cols=1, seed=0)
        chain = wl.build_chain(cfg)
        d = make_desc(chain_fields(chain), 4096, 4096, 4096)
        return lib.rbgp4_prepare_size(ctypes.byref(d), 3), chain

    merged, chain = size((4, 18), 0.0, (8, 8), 0.75, (16, 16))
    vals_merged = (4 // 2) * 18 * 8 * 64 * 16 * 2
    assert merged >= vals_merged
    plan_options("merge", 0)
    unmerged, _ = size((4, 18), 0.0, (8, 8), 0.75, (16, 16))
    assert unmerged != merged
    assert unmerged >= 2 * chain.num_left * chain.row_nnz * 2  # K4 relayout + row-group copy
    plan_options("merge", -1)
    small, chain4 = size((1, 9), 0.0, (16, 16), 0.875, (4, 4))
    assert small >= 9 * 4 * 32 * 16 * 2  # 9 steps x 4 slices x 32 union rows x 16 k
