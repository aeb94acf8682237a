"""On-disk format -> device format loader."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import loader
from paper_2006_13486_b200 import workloads as wl
from paper_2006_13486_b200.errors import BadMagicError, ChecksumMismatchError, DeviceError

from conftest import sha16


def test_load_validates_before_touching_the_device(tmp_path):
    _, w, _ = wl.make_operands(wl.C1A)
    path = tmp_path / "w.rbgp"
    loader.save(w, path)
    data = bytearray(path.read_bytes())
    with pytest.raises(BadMagicError):
        loader.load(b"XXXX" + bytes(data[4:]))
    data[-20] ^= 1
    with pytest.raises(ChecksumMismatchError):
        loader.load(bytes(data))


def test_load_has_no_cpu_fallback(tmp_path):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    _, w, _ = wl.make_operands(wl.C1A)
    with pytest.raises(DeviceError):
        loader.load(ks.serialize(w))


@pytest.mark.gpu
def test_loaded_matrix_products(tmp_path):
    import torch
    chain, w, inp = wl.make_operands(wl.C1A)
    path = tmp_path / "c1a.rbgp"
    loader.save(w, path)
    for compute in ("exact", "bf16"):
        w2 = loader.load(path, compute=compute)
        assert np.array_equal(np.asarray(w2.values), np.asarray(w.values))
        p = ks.tiling_for_chain(chain)
        out, _ = ks.rbgp4mm(w2, torch.from_numpy(inp).cuda(), p, compute=compute)
        if compute == "exact":
            assert sha16(out.cpu().numpy()) == "9fe440861f6f8868"   # reference rbgp4mm hash
        else:
            ref, _ = ks.rbgp4mm(w, torch.from_numpy(inp).cuda(), p, compute="bf16")
            assert torch.equal(out, ref)
