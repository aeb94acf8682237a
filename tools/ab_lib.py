"""Run a tool script against another build of the library: python tools/ab_lib.py LIB tool.py args..."""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200 import _native  # noqa: E402

_native.use_library(os.path.abspath(sys.argv[1]))
# an older build may lack entry points added later: bind them to a stub that fails if called
import ctypes  # noqa: E402
_getattr = ctypes.CDLL.__getattr__


def _lenient(self, name):
    try:
        return _getattr(self, name)
    except AttributeError:
        if not name.startswith("rbgp4_"):
            raise

        def missing(*a, **k):
            raise RuntimeError(f"{name} not in {sys.argv[1]}")
        return missing


ctypes.CDLL.__getattr__ = _lenient
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
