"""On-disk RBGP4 format -> device format.

`load(source, device=None, compute="bf16")` takes a serialized RcubsMatrix (the reference's
stream, rcubs.py:244-343: magic, factor adjacency, values, blake2b digest -- validated exactly
as `deserialize` does, with the same exceptions) and returns the RcubsMatrix with its device
format already resident: values staged through pinned host memory and converted on the device
to the compute element type (bf16 for the tensor-core modes), the two int32 adjacency tables,
and -- for the tensor-core modes -- the prepared per-matrix cache (scatter map, step schedule,
multicast pairs) built once.  The first product on that device then launches immediately.
This is what the reference's `multiply --matrix w.rbgp` flow (cli.py:209-227) needs to run on
the GPU.  `save(w, path)` writes the reference format.
"""

from __future__ import annotations

import os

import numpy as np

from .device import DeviceFormat, cast, chain_fields, resolve_device, torch
from .errors import InvalidArgumentError
from .rcubs import RcubsMatrix, deserialize, serialize

_COMPUTE_DTYPE = {"bf16": "bfloat16", "tf32": "float32", "exact": None, "ffma": None}


def save(w: RcubsMatrix, path) -> None:
    """Write `w` in the reference's serialized format."""
    with open(path, "wb") as fh:
        fh.write(serialize(w))


def load(source, device=None, compute: str = "bf16", precision=None) -> RcubsMatrix:
    """Deserialize `source` (path, bytes or file object) and make it device-resident."""
    if compute not in _COMPUTE_DTYPE:
        raise InvalidArgumentError(f"unknown compute mode {compute!r}")
    if isinstance(source, (str, os.PathLike)):
        with open(source, "rb") as fh:
            data = fh.read()
    elif hasattr(source, "read"):
        data = source.read()
    else:
        data = bytes(source)
    w = deserialize(data, precision=precision)  # validation + errors of the reference
    t = torch()
    dev = resolve_device(device)
    name = _COMPUTE_DTYPE[compute]
    dtype = getattr(t, name) if name else {np.float32: t.float32, np.float64: t.float64}[w.dtype.type]
    with t.cuda.device(dev):
        stream = t.cuda.current_stream(dev)
        # pinned staging: one async H2D of the stored values, conversion on the device
        host = t.empty(w.values.shape, dtype={4: t.float32, 8: t.float64}[w.dtype.itemsize],
                       pin_memory=True)
        host.numpy()[...] = w.values
        src = host.to(dev, non_blocking=True)
        if src.dtype != dtype:
            vals = t.empty(src.shape, dtype=dtype, device=dev)
            cast(src, vals)
        else:
            vals = src
        g_o, _, g_i, _ = w.chain.graphs
        fmt = DeviceFormat(values=vals,
                           adj_o=t.from_numpy(g_o.adjacency_array()).to(dev, non_blocking=True),
                           adj_i=t.from_numpy(g_i.adjacency_array()).to(dev, non_blocking=True),
                           desc_fields=chain_fields(w.chain))
        object.__setattr__(w, "_rbgp4_device_cache", {(str(dev), str(dtype)): fmt})
        if compute in ("bf16", "tf32") and w.chain.k == 4:
            from .sdmm import make_desc, prepared
            prepared(fmt, compute, dev, make_desc(fmt.desc_fields, 1, 1, 1))
        stream.synchronize()  # the pinned staging buffer must outlive the copy
    return w
