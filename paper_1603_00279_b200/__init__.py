"""B200-native (sm_100a, FP64) per-time-level Toeplitz Krylov solver for the implicit
difference scheme of Gu et al., arXiv 1603.00279.  See DESIGN.md and include/tsf.h."""
from . import _lib  # noqa: F401
from .inputs import Instance, CONFIGS  # noqa: F401


def load():
    """Load the CUDA library (raises if it is not built: no CPU fallback)."""
    return _lib.load()
