"""B200-native Fast-ECoT engine (arXiv 2506.07639 hot path).

A drop-in `GenerationBackend` for the reference scheduler API (`ecot_sched`,
imported as-is -- see refapi.py) served by hand-written sm_100a kernels
through the C ABI in include/fastecot.h.  See DESIGN.md.
"""

from .backends import EngineError, LengthPlan, encode_context, length_plan
from .runners import BatchedEpisodes, EngineParallelAsyncRunner, plain_trace, register, summarize

register()   # the reference runner table serves parallel_async through the device engine


def EngineBackend(*args, **kwargs):
    """Lazily imported so CPU-only users never need the CUDA library."""
    from .engine_backend import EngineBackend as _EB
    return _EB(*args, **kwargs)


__version__ = "0.2.0"
