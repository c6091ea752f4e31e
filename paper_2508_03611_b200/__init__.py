"""B200-native what-if simulation core for Block's predictive dispatcher.

The hot path (blocksim predict() / predict_across() / BlockPredictive
dispatch) runs as hand-written sm_100a kernels behind the C-ABI in
include/blocksim_b200.h; this package is the Python-side binding used by
tests and bench.py. There is no CPU fallback: loading the library or
creating a context without a CUDA device raises.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
