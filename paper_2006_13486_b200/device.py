"""Device format and operand staging (PyTorch used as plumbing only).

The RBGP4 device format is the succinct one of the reference's storage
(rcubs.py:1-12): the `(rows, row_nnz)` values array in sorted-column order
plus the two int32 base adjacency tables of g_o and g_i -- no mask, no CSR
indices, no densified blocks.  `device_format(w, device, dtype)` uploads it
once per (matrix, device, element type) and caches it on the matrix object;
`RcubsMatrix.values` is immutable (reference rcubs.py:86-98) so the cache can
never go stale.

Operands may be numpy arrays (host; copied in and out), CPU torch tensors
(pinned ones copy asynchronously) or CUDA torch tensors (used in place, no
host traffic).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DeviceError, InvalidArgumentError

_lock = threading.Lock()
_DT_CODE = {}


def torch():
    import torch as _t  # deferred: importing torch costs ~seconds on a cold box
    return _t


def dtype_code(dt) -> int:
    t = torch()
    if not _DT_CODE:
        _DT_CODE.update({t.float32: _native.F32, t.float64: _native.F64,
                         t.bfloat16: _native.BF16})
    try:
        return _DT_CODE[dt]
    except KeyError:
        raise InvalidArgumentError(f"unsupported element type {dt}") from None


def resolve_device(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise DeviceError("no CUDA device visible: the RBGP4 product runs on B200 only "
                          "(there is no CPU fallback)")
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    dev = t.device(device)
    if dev.type != "cuda":
        raise InvalidArgumentError(f"device must be a CUDA device, got {dev}")
    return t.device("cuda", dev.index if dev.index is not None else t.cuda.current_device())


@dataclass
class DeviceFormat:
    """Values + adjacency tables of one chain matrix on one device."""

    values: object          # (rows, row_nnz) tensor in the compute element type
    adj_o: object           # (u_o, d_o) int32
    adj_i: object           # (u_i, d_i) int32
    desc_fields: dict       # chain sizes for rbgp4_desc
    prep: dict = None       # compute mode -> prepared scatter map (tensor-core modes)


def chain_fields(chain) -> dict:
    g_o, g_r, g_i, g_b = chain.graphs
    return dict(
        rows=chain.num_left, cols=chain.num_right,
        u_o=g_o.num_left, v_o=g_o.num_right, d_o=len(g_o.adjacency[0]),
        rm=g_r.num_left, rk=g_r.num_right,
        u_i=g_i.num_left, v_i=g_i.num_right, d_i=len(g_i.adjacency[0]),
        bm=g_b.num_left, bk=g_b.num_right,
    )


def device_format(w, device, dtype) -> DeviceFormat:
    """Upload (once) the device format of RcubsMatrix-like `w`."""
    t = torch()
    key = (str(device), str(dtype))
    cache = w.__dict__.get("_rbgp4_device_cache")
    if cache is None:
        cache = {}
        object.__setattr__(w, "_rbgp4_device_cache", cache)
    fmt = cache.get(key)
    if fmt is not None:
        return fmt
    with _lock:
        fmt = cache.get(key)
        if fmt is not None:
            return fmt
        g_o, _, g_i, _ = w.chain.graphs
        host = t.from_numpy(np.array(w.values, copy=True))  # values are read-only
        src = host.to(device)
        if src.dtype != dtype:
            vals = t.empty(src.shape, dtype=dtype, device=device)
            cast(src, vals)
        else:
            vals = src
        fmt = DeviceFormat(
            values=vals,
            adj_o=t.from_numpy(g_o.adjacency_array()).to(device),
            adj_i=t.from_numpy(g_i.adjacency_array()).to(device),
            desc_fields=chain_fields(w.chain),
        )
        cache[key] = fmt
        return fmt


def stream_handle(device) -> int:
    return torch().cuda.current_stream(device).cuda_stream


def cast(src, dst) -> None:
    """dst <- src element-wise on the device (same numel), via rbgp4_cast."""
    if src.numel() != dst.numel():
        raise InvalidArgumentError("cast: element counts differ")
    if not (src.is_contiguous() and dst.is_contiguous()):
        raise InvalidArgumentError("cast: operands must be contiguous")
    _native.check(
        _native.lib().rbgp4_cast(dtype_code(src.dtype), dtype_code(dst.dtype), src.data_ptr(),
                                 dst.data_ptr(), src.numel(), stream_handle(src.device)),
        "rbgp4_cast",
    )


class Staged:
    """An operand placed on the device, remembering how to hand results back."""

    def __init__(self, obj, device):
        t = torch()
        self.kind = ("torch_cuda" if isinstance(obj, t.Tensor) and obj.is_cuda
                     else "torch_cpu" if isinstance(obj, t.Tensor) else "numpy")
        if self.kind == "numpy":
            arr = np.ascontiguousarray(obj)
            host = t.from_numpy(arr if arr.flags.writeable else arr.copy())
            self.tensor = host.to(device, non_blocking=False)
        elif self.kind == "torch_cpu":
            host = obj.contiguous()
            self.tensor = host.to(device, non_blocking=host.is_pinned())
        else:
            if obj.device != device:
                raise InvalidArgumentError(f"operand on {obj.device}, expected {device}")
            self.tensor = obj if obj.stride(-1) == 1 else obj.contiguous()
        self.pinned = self.kind == "torch_cpu" and obj.is_pinned()

    def give_back(self, result):
        """Return `result` (a device tensor) in the caller's container type."""
        if self.kind == "torch_cuda":
            return result
        if self.kind == "torch_cpu":
            t = torch()
            host = t.empty(result.shape, dtype=result.dtype, pin_memory=self.pinned)
            host.copy_(result, non_blocking=self.pinned)
            if self.pinned:
                t.cuda.current_stream(result.device).synchronize()
            return host
        return result.cpu().numpy()
