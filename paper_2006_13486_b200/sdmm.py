"""The RBGP4 sparse x dense product -- drop-in for `kronsparse.sdmm`.

Same names, signatures, defaults and error behaviour as the reference
(`sdmm.py:35-344`); the arithmetic runs on the B200 through the C ABI in
`librbgp4_b200.so` (include/rbgp4.h).  There is no CPU path: without the
extension or a CUDA device every product raises `DeviceError`.

Extensions are keyword-only and default to the reference semantics:

* ``compute``: "exact" (default; SIMT kernel rounding every multiply and add
  like the reference -- outputs are bit-identical to the reference's
  `rbgp4mm` for any tiling), "ffma" (same order, fused multiply-add),
  "tf32" / "bf16" (tcgen05 tensor cores, fp32 accumulation in TMEM).
* ``out``: preallocated CUDA tensor (rows, N) to write into.
* ``out_dtype``: result element type for the tensor-core modes.

numpy in -> numpy out (host copies both ways); CUDA tensors in -> CUDA
tensor out with no host traffic; CPU tensors in -> CPU tensor out.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .device import (Staged, cast, chain_fields, device_format, dtype_code, resolve_device,
                     stream_handle, torch)
from .errors import ConfigurationError, InvalidArgumentError, ShapeError, UnsupportedChainError
from .products import Rbgp4Config, RbgpChain
from .rcubs import CsrMatrix, RcubsMatrix

DEFAULT_TN = 128
DEFAULT_RN = 1
DEFAULT_BN = 32
COMPUTE_MODES = ("exact", "ffma", "tf32", "bf16")


@dataclass(frozen=True)
class TilingParams:
    """Tile and micro-block sizes (reference `sdmm.py:40-58`).

    (tm, tk) is the W tile, (rm, rk) and (bm, bk) come from the complete
    factors; tn/rn/bn and workers were CPU knobs in the reference.  They are
    validated exactly as there (the `N % tn` contract included) but do not
    steer the GPU tiling, which never changes results.
    """

    tm: int
    tk: int
    tn: int
    rm: int
    rk: int
    bm: int
    bk: int
    rn: int
    bn: int
    workers: int = 1


@dataclass(frozen=True)
class WorkReport:
    """Closed-form work accounting (reference `sdmm.py:61-90,284-293`)."""

    fma_count: int
    tiles: int
    steps_per_tile: int
    steps_skipped_per_tile: int
    w_bytes_read: int
    i_bytes_read: int

    @property
    def total_steps_executed(self) -> int:
        return self.tiles * self.steps_per_tile

    @property
    def total_steps_skipped(self) -> int:
        return self.tiles * self.steps_skipped_per_tile

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        d.update(total_steps_executed=self.total_steps_executed,
                 total_steps_skipped=self.total_steps_skipped)
        return {k: d[k] for k in ("fma_count", "tiles", "steps_per_tile",
                                  "steps_skipped_per_tile", "total_steps_executed",
                                  "total_steps_skipped", "w_bytes_read", "i_bytes_read")}


def tiling_for_chain(chain: RbgpChain, tn: int = DEFAULT_TN, rn: int = DEFAULT_RN,
                     bn: int = DEFAULT_BN, workers: int = 1) -> TilingParams:
    """TilingParams of a four-factor chain; every violation is reported at once."""
    if chain.k != 4:
        raise UnsupportedChainError(f"tiled multiply needs a 4-factor chain, got {chain.k}")
    g_o, g_r, g_i, g_b = chain.graphs
    problems = [f"{label} factor must be complete for row repetition"
                for label, g in (("second", g_r), ("fourth", g_b)) if not g.is_complete()]
    knobs = {"tn": tn, "rn": rn, "bn": bn, "workers": workers}
    problems += [f"{k} must be positive, got {v}" for k, v in knobs.items() if v < 1]
    if min(tn, rn, bn) >= 1 and tn % (rn * bn):
        problems.append(f"tn={tn} is not divisible by rn*bn={rn * bn}")
    if problems:
        raise ConfigurationError(problems)
    return TilingParams(
        tm=g_r.num_left * g_i.num_left * g_b.num_left,
        tk=g_r.num_right * g_i.num_right * g_b.num_right,
        tn=tn, rm=g_r.num_left, rk=g_r.num_right, bm=g_b.num_left, bk=g_b.num_right,
        rn=rn, bn=bn, workers=workers,
    )


def derive_tiling(config: Rbgp4Config, tn: int = DEFAULT_TN, rn: int = DEFAULT_RN,
                  bn: int = DEFAULT_BN, workers: int = 1) -> TilingParams:
    return tiling_for_chain(config.to_chain(), tn=tn, rn=rn, bn=bn, workers=workers)


def with_workers(params: TilingParams, workers: int) -> TilingParams:
    return replace(params, workers=workers)


def _check_params(w, params: TilingParams) -> None:
    """Same checks and messages as reference `sdmm.py:208-232`."""
    _, g_r, g_i, g_b = w.chain.graphs
    expect = {
        "rm": g_r.num_left, "rk": g_r.num_right, "bm": g_b.num_left, "bk": g_b.num_right,
        "tm": g_r.num_left * g_i.num_left * g_b.num_left,
        "tk": g_r.num_right * g_i.num_right * g_b.num_right,
    }
    bad = [f"{k}={getattr(params, k)} inconsistent with chain (expected {v})"
           for k, v in expect.items() if getattr(params, k) != v]
    if params.tn < 1 or params.rn < 1 or params.bn < 1:
        bad.append("tn, rn, bn must be positive")
    elif params.tn % (params.rn * params.bn):
        bad.append(f"tn={params.tn} is not divisible by rn*bn={params.rn * params.bn}")
    if params.workers < 1:
        bad.append(f"workers must be positive, got {params.workers}")
    if bad:
        raise ConfigurationError(bad)


def work_report(w, n_cols: int, params: TilingParams) -> WorkReport:
    """The reference's closed-form accounting (sdmm.py:284-293)."""
    d_o = len(w.chain.graphs[0].adjacency[0])
    tiles = (w.rows // params.tm) * (n_cols // params.tn)
    size = w.dtype.itemsize
    return WorkReport(
        fma_count=w.nnz * n_cols,
        tiles=tiles,
        steps_per_tile=d_o,
        steps_skipped_per_tile=w.cols // params.tk - d_o,
        w_bytes_read=w.nnz * (n_cols // params.tn) * size,
        i_bytes_read=tiles * d_o * params.tk * params.tn * size,
    )


def _shape_dtype(inp):
    t = torch() if not isinstance(inp, np.ndarray) else None
    if t is not None and isinstance(inp, t.Tensor):
        return tuple(inp.shape), inp.dtype
    arr = np.asarray(inp)
    return arr.shape, arr.dtype


def _np_to_torch_dtype(dt):
    t = torch()
    return {np.dtype("float32"): t.float32, np.dtype("float64"): t.float64}.get(np.dtype(dt))


def rbgp4mm(w: RcubsMatrix, inp, params: TilingParams, *, compute: str = "exact",
            out=None, out_dtype=None, device=None, non_blocking: bool = False):
    """O = W x I on the B200; returns (out, WorkReport) like reference `sdmm.py:235-294`.

    Host operands: with a pinned CPU torch input, a pinned CPU `out` and non_blocking=True the
    call only queues work -- the H2D copy on a per-device copy-in stream, the product on the
    current stream, the D2H copy into `out` on a copy-out stream -- and returns at once, so
    consecutive products overlap their copies with each other's kernels (both PCIe directions
    and the SMs busy at the same time).  The caller synchronises (torch.cuda.synchronize()).
    """
    if w.chain.k != 4:
        raise UnsupportedChainError(
            f"tiled multiply needs a 4-factor chain, got {w.chain.k}; "
            "use sdmm_reference for general chains"
        )
    _check_params(w, params)
    if compute not in COMPUTE_MODES:
        raise InvalidArgumentError(f"compute must be one of {COMPUTE_MODES}, got {compute!r}")
    t = torch()
    is_tensor = isinstance(inp, t.Tensor)
    if not is_tensor:
        inp = np.asarray(inp)
    shape, dt = _shape_dtype(inp)
    if len(shape) != 2 or shape[0] != w.cols:
        raise ShapeError(f"input shape {shape} incompatible with W of shape ({w.rows}, {w.cols})")
    w_tdt = _np_to_torch_dtype(w.dtype)
    in_tdt = dt if is_tensor else _np_to_torch_dtype(dt)
    bf16_input = is_tensor and dt == t.bfloat16 and compute == "bf16"
    if not bf16_input and in_tdt != w_tdt:
        shown = dt if not is_tensor else str(dt).replace("torch.", "")
        raise ShapeError(f"input dtype {shown} != matrix dtype {w.dtype}")
    if compute == "tf32" and w.dtype != np.float32:
        raise ShapeError("compute='tf32' needs f32 operands")
    n_cols = shape[1]
    if n_cols % params.tn:
        raise ConfigurationError([f"input columns {n_cols} not divisible by tn={params.tn}"])

    if not is_tensor and out is None and out_dtype == t.bfloat16:
        raise InvalidArgumentError("numpy operands cannot hold a bfloat16 result; pass torch "
                                   "tensors or out_dtype=torch.float32")
    host_out = isinstance(out, t.Tensor) and not out.is_cuda
    if host_out and not (is_tensor and not inp.is_cuda and out.is_pinned()):
        raise InvalidArgumentError("a host `out` must be a pinned CPU tensor, with a CPU torch input")
    pipelined = non_blocking and host_out and inp.is_pinned()
    dev = resolve_device(device if device is not None else (inp.device if is_tensor and inp.is_cuda else None))
    with t.cuda.device(dev):
        stream = t.cuda.current_stream(dev)
        if pipelined:
            copy_in, copy_out = _copy_streams(dev)
            with t.cuda.stream(copy_in):
                x = t.empty(tuple(inp.shape), dtype=inp.dtype, device=dev)
                x.copy_(inp, non_blocking=True)
            stream.wait_stream(copy_in)
            x.record_stream(stream)
            staged = None
        else:
            staged = Staged(inp, dev)
            x = staged.tensor
        if compute == "bf16":
            op_dt = t.bfloat16
            if x.dtype != t.bfloat16:
                xb = t.empty(x.shape, dtype=t.bfloat16, device=dev)
                cast(x.contiguous(), xb)
                x = xb
            res_dt = out_dtype if out_dtype is not None else (
                t.bfloat16 if bf16_input else t.float32)
        elif compute == "tf32":
            op_dt = t.float32
            res_dt = out_dtype if out_dtype is not None else t.float32
        else:
            op_dt = w_tdt
            res_dt = w_tdt
            if out_dtype is not None and out_dtype != w_tdt:
                raise InvalidArgumentError("SIMT modes return the operand dtype")
        fmt = device_format(w, dev, op_dt)
        if out is None or host_out:
            res = t.empty((w.rows, n_cols), dtype=res_dt, device=dev)
        else:
            res = out
        if out is not None and (not isinstance(out, t.Tensor) or (not host_out and out.device != dev)
                                or out.dtype != res_dt or tuple(out.shape) != (w.rows, n_cols)
                                or out.stride(1) != 1):
            raise ShapeError(f"out must be a ({w.rows}, {n_cols}) {res_dt} tensor with unit "
                             f"column stride on {dev} (or pinned host memory)")
        launch_sdmm(fmt, compute, x, res, dev)
        if host_out:
            copy_out = _copy_streams(dev)[1]
            copy_out.wait_stream(stream)
            with t.cuda.stream(copy_out):
                out.copy_(res, non_blocking=True)
            res.record_stream(copy_out)
            if not non_blocking:
                copy_out.synchronize()
            result = out
        else:
            result = staged.give_back(res) if out is None else res
    return result, work_report(w, n_cols, params)


_COPY_STREAMS = {}


def _copy_streams(dev):
    """(copy-in, copy-out) streams of a device for the pipelined host path (created once)."""
    t = torch()
    key = str(dev)
    with _WS_LOCK:
        if key not in _COPY_STREAMS:
            _COPY_STREAMS[key] = (t.cuda.Stream(device=dev), t.cuda.Stream(device=dev))
    return _COPY_STREAMS[key]


def make_desc(fields: dict, n_cols: int, ld_in: int, ld_out: int) -> _native.Desc:
    d = _native.Desc()
    for k, v in fields.items():
        setattr(d, k, v)
    d.n_cols, d.ld_in, d.ld_out = n_cols, ld_in, ld_out
    return d


_WS = {}
_WS_LOCK = threading.Lock()


def workspace(dev, nbytes: int, stream: int):
    """Scratch buffer of the tensor-core path, one per (device, stream), grown on demand.

    Keyed by stream so products queued on different streams never share partial sums, and
    allocated on that stream (torch's caching allocator then keeps a replaced buffer alive
    until the work queued on its stream before the replacement has run).
    """
    t = torch()
    key = (str(dev), int(stream))
    with _WS_LOCK:
        buf = _WS.get(key)
        if buf is None or buf.numel() < nbytes:
            s = t.cuda.ExternalStream(stream, device=dev) if stream else t.cuda.default_stream(dev)
            with t.cuda.stream(s):
                buf = t.empty(max(nbytes, 1), dtype=t.uint8, device=dev)
            _WS[key] = buf
    return buf


def prepared(fmt, compute: str, dev, desc):
    """Per-matrix scatter map for the tensor-core modes (built once, cached on `fmt`)."""
    if compute not in ("tf32", "bf16"):
        return None
    if fmt.prep is None:
        fmt.prep = {}
    lib = _native.lib()
    code = _native.COMPUTE[compute]
    # the section's layout follows the plan (e.g. option relayout), so its size is in the key
    nbytes = lib.rbgp4_prepare_size(ctypes.byref(desc), code)
    if nbytes == 0:
        return None
    buf = fmt.prep.get((compute, nbytes))
    if buf is None:
        buf = torch().empty(nbytes, dtype=torch().uint8, device=dev)
        _native.check(lib.rbgp4_prepare(ctypes.byref(desc), code, fmt.values.data_ptr(), fmt.adj_o.data_ptr(),
                                        fmt.adj_i.data_ptr(),
                                        buf.data_ptr(), nbytes, stream_handle(dev)),
                      "rbgp4_prepare")
        fmt.prep[(compute, nbytes)] = buf
    return buf


def launch_sdmm(fmt, compute: str, x, res, dev) -> None:
    """Queue one rbgp4_sdmm on the current stream of `dev` (no sync)."""
    lib = _native.lib()
    if compute in ("tf32", "bf16") and x.shape[1] and (
            x.data_ptr() % 16 or (x.stride(0) * x.element_size()) % 16):
        # the tensor-core kernels read I by TMA: 16-byte aligned base and row pitch.  Any legal
        # operand (e.g. N = 5 with tn = 1) is staged into a padded copy; n_cols stays N
        per = 16 // x.element_size()
        xp = torch().empty((x.shape[0], -(-x.shape[1] // per) * per), dtype=x.dtype, device=x.device)
        xp[:, :x.shape[1]].copy_(x)
        x = xp[:, :x.shape[1]]
    desc = make_desc(fmt.desc_fields, x.shape[1], x.stride(0), res.stride(0))
    code = _native.COMPUTE[compute]
    in_code, out_code = dtype_code(x.dtype), dtype_code(res.dtype)
    need = lib.rbgp4_workspace_size(ctypes.byref(desc), code, in_code)
    stream = stream_handle(dev)
    ws_ptr, ws_len = (workspace(dev, need, stream).data_ptr(), need) if need else (None, 0)
    prep = prepared(fmt, compute, dev, desc) if x.shape[1] else None
    _native.check(
        lib.rbgp4_sdmm_prepared(ctypes.byref(desc), code, in_code, out_code, fmt.values.data_ptr(),
                                fmt.adj_o.data_ptr(), fmt.adj_i.data_ptr(),
                                prep.data_ptr() if prep is not None else None, x.data_ptr(),
                                res.data_ptr(), ws_ptr, ws_len, stream),
        f"rbgp4_sdmm(compute={compute})",
    )


def sdmm_reference(w, inp, *, device=None):
    """Row-wise product in the reference oracle's rounding order, on the GPU.

    Accepts a chain matrix (any number of factors; columns enumerated in
    closed form) or a raw CsrMatrix, like reference `sdmm.py:307-330`.
    Bit-identical to the reference's `sdmm_reference` in f32 and f64.
    """
    t = torch()
    is_chain = not isinstance(w, CsrMatrix) and hasattr(w, "chain")
    if is_chain:
        rows, cols, vdt = w.rows, w.cols, w.dtype
    else:
        rows, cols = w.shape
        vdt = np.asarray(w.values).dtype
    is_tensor = isinstance(inp, t.Tensor)
    if not is_tensor:
        inp = np.asarray(inp)
    shape, dt = _shape_dtype(inp)
    if len(shape) != 2 or shape[0] != cols:
        raise ShapeError(f"input shape {shape} incompatible with W of shape ({rows}, {cols})")
    v_tdt = _np_to_torch_dtype(vdt)
    if (dt if is_tensor else _np_to_torch_dtype(dt)) != v_tdt:
        raise ShapeError(f"input dtype {dt} != matrix dtype {vdt}")
    dev = resolve_device(device if device is not None else (inp.device if is_tensor and inp.is_cuda else None))
    lib = _native.lib()
    with t.cuda.device(dev):
        staged = Staged(inp, dev)
        x = staged.tensor
        res = t.empty((rows, shape[1]), dtype=v_tdt, device=dev)
        code = dtype_code(v_tdt)
        if is_chain:
            graphs = w.chain.graphs
            nl = (ctypes.c_int32 * len(graphs))(*[g.num_left for g in graphs])
            nr = (ctypes.c_int32 * len(graphs))(*[g.num_right for g in graphs])
            dg = (ctypes.c_int32 * len(graphs))(*[len(g.adjacency[0]) for g in graphs])
            adj = [g.adjacency_array().reshape(-1) for g in graphs]
            offs = np.cumsum([0] + [a.size for a in adj[:-1]]).astype(np.int64)
            off = (ctypes.c_int64 * len(graphs))(*offs.tolist())
            adj_d = t.from_numpy(np.concatenate(adj).astype(np.int32)).to(dev)
            vals = t.from_numpy(np.ascontiguousarray(w.values)).to(dev)
            _native.check(lib.rbgp4_chain_sdmm(
                len(graphs), nl, nr, dg, off, adj_d.data_ptr(), code, vals.data_ptr(),
                x.data_ptr(), res.data_ptr(), shape[1], x.stride(0), res.stride(0),
                stream_handle(dev)), "rbgp4_chain_sdmm")
        else:
            indptr = t.from_numpy(np.ascontiguousarray(w.indptr, dtype=np.int64)).to(dev)
            indices = t.from_numpy(np.ascontiguousarray(w.indices, dtype=np.int32)).to(dev)
            vals = t.from_numpy(np.ascontiguousarray(w.values)).to(dev)
            _native.check(lib.rbgp4_csr_sdmm(
                rows, indptr.data_ptr(), indices.data_ptr(), code, vals.data_ptr(), x.data_ptr(),
                res.data_ptr(), shape[1], x.stride(0), res.stride(0), stream_handle(dev)),
                "rbgp4_csr_sdmm")
        return staged.give_back(res)


def dense_gemm(a, b):
    """Dense baseline (reference `sdmm.py:333-339`): BLAS on the host for
    numpy operands, cuBLAS for CUDA tensors.  Not on the RBGP4 hot path."""
    t = torch()
    if isinstance(a, t.Tensor) and isinstance(b, t.Tensor):
        if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
            raise ShapeError(f"cannot multiply shapes {tuple(a.shape)} and {tuple(b.shape)}")
        return a @ b
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError(f"cannot multiply shapes {a.shape} and {b.shape}")
    return a @ b
