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


def __getattr__(name):
    if _IMPORT_ERROR is not None and not name.startswith("__"):
        raise ImportError(
            "paper_2406_00809_b200: native extension not built (" + str(_IMPORT_ERROR) + "); run "
            "`python -m paper_2406_00809_b200.build` or __graft_entry__.build()"
        )
    raise AttributeError(name)


def library_path() -> str:
    return _os.path.join(_HERE, "libgnpc.so")
