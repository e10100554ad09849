"""B200-native (sm_100a) CPCA hot path: kNN graphs, sampling + Kron-reduced
graphs, FRPCAG FISTA and the graph-regularised CG decoder of arXiv 1602.02070,
behind the reference `cpcag` API (see cpcag.py) and the C-ABI in
include/cpcag_cuda.h (libcpcag_cuda.so)."""
from . import _native
from .cpcag import *  # noqa: F401,F403

__version__ = "0.1.0"
