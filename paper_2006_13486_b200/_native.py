"""ctypes binding of the in-tree C-ABI library `librbgp4_b200.so`.

The product path has no fallback: if the library is missing or cannot be
loaded, every call raises :class:`DeviceError`.  Device memory and streams
come from PyTorch (plumbing only); the arithmetic is in the library.
"""

from __future__ import annotations

import contextlib
import ctypes
import os

from .errors import DeviceError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librbgp4_b200.so")

F32, F64, BF16 = 0, 1, 2
EUNSUPPORTED = -2       # RBGP4_EUNSUPPORTED
CONV_POOL2 = 2          # RBGP4_CONV_POOL2 (rbgp4_conv_desc.relu flags)
COMPUTE = {"exact": 0, "ffma": 1, "tf32": 2, "bf16": 3}
EXPORTED = (
    "rbgp4_sdmm", "rbgp4_sdmm_prepared", "rbgp4_prepare", "rbgp4_prepare_size", "rbgp4_prepare_values",
    "rbgp4_workspace_size", "rbgp4_sdmm_supported", "rbgp4_chain_sdmm",
    "rbgp4_conv2d", "rbgp4_conv2d_workspace_size", "rbgp4_maxpool2x2_nhwc",
    "rbgp4_csr_sdmm", "rbgp4_cast", "rbgp4_last_error", "rbgp4_abi_version", "rbgp4_launch_count",
    "rbgp4_reset_launch_count", "rbgp4_last_kernel", "rbgp4_sddmm", "rbgp4_set_option", "rbgp4_get_option",
    "rbgp4_reset_options", "rbgp4_debug_build", "rbgp4_im2col_nhwc", "rbgp4_nc_to_nhwc",
    "rbgp4_conv2d_residual", "rbgp4_nc_to_nhwc_residual", "rbgp4_dense_conv3x3_c3",
    "rbgp4_sddmm_nk",
)


class ConvDesc(ctypes.Structure):
    """Mirror of `rbgp4_conv_desc` (include/rbgp4.h)."""

    _fields_ = [(n, ctypes.c_int32) for n in ("batch", "height", "width", "c_in", "kh", "kw", "pad",
                                              "stride", "relu")]


class Desc(ctypes.Structure):
    """Mirror of `rbgp4_desc` (include/rbgp4.h)."""

    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("n_cols", ctypes.c_int64),
        ("ld_in", ctypes.c_int64), ("ld_out", ctypes.c_int64),
        ("u_o", ctypes.c_int32), ("v_o", ctypes.c_int32), ("d_o", ctypes.c_int32),
        ("rm", ctypes.c_int32), ("rk", ctypes.c_int32),
        ("u_i", ctypes.c_int32), ("v_i", ctypes.c_int32), ("d_i", ctypes.c_int32),
        ("bm", ctypes.c_int32), ("bk", ctypes.c_int32),
    ]


_lib = None


def use_library(path: str) -> None:
    """Load `path` instead of the release library (tools/: the -DRBGP4_DEBUG=1 build).
    Must run before the first call that loads the library."""
    global LIB_PATH
    if _lib is not None and os.path.abspath(path) != os.path.abspath(LIB_PATH):
        raise DeviceError(f"library already loaded from {LIB_PATH}")
    LIB_PATH = path


def lib():
    """Load (once) and return the library, raising DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"CUDA extension not built ({LIB_PATH} missing); run "
            "`python -m paper_2006_13486_b200.build` -- there is no CPU fallback"
        )
    try:
        h = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    h.rbgp4_sdmm.argtypes = [ctypes.POINTER(Desc), i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp]
    h.rbgp4_sdmm.restype = i32
    h.rbgp4_sdmm_prepared.argtypes = [ctypes.POINTER(Desc), i32, i32, i32, vp, vp, vp, vp, vp, vp,
                                      vp, sz, vp]
    h.rbgp4_sdmm_prepared.restype = i32
    h.rbgp4_prepare_size.argtypes = [ctypes.POINTER(Desc), i32]
    h.rbgp4_prepare_size.restype = sz
    h.rbgp4_prepare.argtypes = [ctypes.POINTER(Desc), i32, vp, vp, vp, vp, sz, vp]
    h.rbgp4_sddmm.argtypes = [ctypes.POINTER(Desc), i32, vp, vp, vp, ctypes.c_int64, vp, ctypes.c_int64, vp, vp]
    h.rbgp4_sddmm.restype = i32
    h.rbgp4_sddmm_nk.argtypes = [ctypes.POINTER(Desc), vp, vp, vp, ctypes.c_int64, vp, ctypes.c_int64, vp, vp]
    h.rbgp4_sddmm_nk.restype = i32
    h.rbgp4_prepare.restype = i32
    h.rbgp4_prepare_values.argtypes = [ctypes.POINTER(Desc), i32, vp, vp, sz, vp]
    h.rbgp4_prepare_values.restype = i32
    h.rbgp4_conv2d_workspace_size.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(ConvDesc)]
    h.rbgp4_conv2d_workspace_size.restype = sz
    h.rbgp4_conv2d.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(ConvDesc), i32, vp, vp, vp, vp,
                               vp, vp, vp, sz, vp]
    h.rbgp4_conv2d.restype = i32
    h.rbgp4_maxpool2x2_nhwc.argtypes = [vp, vp, i32, i32, i32, i32, vp]
    h.rbgp4_maxpool2x2_nhwc.restype = i32
    h.rbgp4_im2col_nhwc.argtypes = [i32, vp, vp, i32, i32, i32, i32, i32, i32, vp]
    h.rbgp4_im2col_nhwc.restype = i32
    h.rbgp4_nc_to_nhwc.argtypes = [i32, vp, vp, i32, ctypes.c_int64, i32, vp]
    h.rbgp4_nc_to_nhwc.restype = i32
    h.rbgp4_conv2d_residual.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(ConvDesc), i32, vp, vp, vp, vp,
                                        vp, vp, vp, vp, vp, sz, vp]
    h.rbgp4_conv2d_residual.restype = i32
    h.rbgp4_nc_to_nhwc_residual.argtypes = [i32, vp, vp, vp, vp, i32, ctypes.c_int64, vp]
    h.rbgp4_nc_to_nhwc_residual.restype = i32
    h.rbgp4_dense_conv3x3_c3.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp]
    h.rbgp4_dense_conv3x3_c3.restype = i32
    h.rbgp4_workspace_size.argtypes = [ctypes.POINTER(Desc), i32, i32]
    h.rbgp4_workspace_size.restype = sz
    h.rbgp4_sdmm_supported.argtypes = [ctypes.POINTER(Desc), i32, i32, i32]
    h.rbgp4_sdmm_supported.restype = i32
    h.rbgp4_chain_sdmm.argtypes = [i32, vp, vp, vp, vp, vp, i32, vp, vp, vp, i64, i64, i64, vp]
    h.rbgp4_chain_sdmm.restype = i32
    h.rbgp4_csr_sdmm.argtypes = [i64, vp, vp, i32, vp, vp, vp, i64, i64, i64, vp]
    h.rbgp4_csr_sdmm.restype = i32
    h.rbgp4_cast.argtypes = [i32, i32, vp, vp, i64, vp]
    h.rbgp4_cast.restype = i32
    h.rbgp4_last_error.restype = ctypes.c_char_p
    h.rbgp4_abi_version.restype = i32
    h.rbgp4_launch_count.restype = i64
    h.rbgp4_reset_launch_count.restype = None
    h.rbgp4_last_kernel.restype = ctypes.c_char_p
    h.rbgp4_set_option.argtypes = [ctypes.c_char_p, i64]
    h.rbgp4_set_option.restype = i32
    h.rbgp4_get_option.argtypes = [ctypes.c_char_p, ctypes.POINTER(i64)]
    h.rbgp4_get_option.restype = i32
    h.rbgp4_reset_options.restype = None
    h.rbgp4_debug_build.restype = i32
    _lib = h
    return h


def last_error() -> str:
    return lib().rbgp4_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise DeviceError(f"{what} failed (code {rc}): {last_error()}")


def set_option(name: str, value: int) -> None:
    """Thread-local plan override (rbgp4_set_option); raises on unknown names / values."""
    check(lib().rbgp4_set_option(name.encode(), int(value)), f"rbgp4_set_option({name}={value})")


def get_option(name: str) -> int:
    v = ctypes.c_int64()
    check(lib().rbgp4_get_option(name.encode(), ctypes.byref(v)), f"rbgp4_get_option({name})")
    return int(v.value)


@contextlib.contextmanager
def options(**kw):
    """Set plan overrides for the calling thread inside a `with` block, then restore them."""
    old = {k: get_option(k) for k in kw}
    try:
        for k, v in kw.items():
            set_option(k, v)
        yield
    finally:
        for k, v in old.items():
            set_option(k, v)


def last_kernel() -> str:
    """Kernel family of this thread's last launch through the ABI (e.g. "K5 conv")."""
    return lib().rbgp4_last_kernel().decode()


def launch_count() -> int:
    return int(lib().rbgp4_launch_count())


def reset_launch_count() -> None:
    lib().rbgp4_reset_launch_count()
