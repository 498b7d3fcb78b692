"""B200-native graph neural preconditioner (GNP) hot path.

Drop-in for the reference's Python package ``gnp`` (python/gnp/__init__.py):
the same ``_gnp`` functions (solve, train, spmv, prescale, gershgorin_gamma,
generators, checkpoints, iter_auc/time_auc) backed by sm_100a kernels through
the C ABI in ``include/gnpc.h`` (libgnpc.so).  There is no CPU fallback: on a
machine without a CUDA device every compute call raises.
"""

__version__ = "0.1.0"

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))
_IMPORT_ERROR = None

try:
    from ._gnp import *  # noqa: F401,F403
    from ._gnp import CsrMatrix, GnnParams  # noqa: F401
except ImportError as _e:  # the build module must stay importable
    _IMPORT_ERROR = _e


# pure-Python submodules that must import before (or without) the native build
_SUBMODULES = ("build", "capi", "dp", "runrecord")


def _retry_native_import() -> bool:
    """The package may have been imported before an in-process build; retry once."""
    global _IMPORT_ERROR
    import importlib

    try:
        _m = importlib.import_module(__name__ + "._gnp")
    except ImportError as e:
        _IMPORT_ERROR = e
        return False
    g = globals()
    g.update({k: getattr(_m, k) for k in dir(_m) if not k.startswith("__")})
    g["_gnp"] = _m
    _IMPORT_ERROR = None
    return True


def __getattr__(name):
    import importlib

    if name in _SUBMODULES:
        return importlib.import_module("." + name, __name__)
    if _IMPORT_ERROR is not None and not name.startswith("__") and _retry_native_import():
        if name in globals():
            return globals()[name]
    if _IMPORT_ERROR is not None and not name.startswith("__"):
        raise ImportError(
            "paper_2406_00809_b200: native extension not built (" + str(_IMPORT_ERROR) + "); run "
            "`python -m paper_2406_00809_b200.build` or __graft_entry__.build()"
        )
    raise AttributeError(name)


def library_path() -> str:
    return _os.path.join(_HERE, "libgnpc.so")
