"""B200-native Fast-ECoT engine (arXiv 2506.07639 hot path).

Host-side mirror of the reference scheduler API (`ecot_sched`: trace types,
GenerationBackend protocol, runners, batching accounting) plus the
`EngineBackend` that serves the protocol from hand-written sm_100a kernels
through the C ABI in include/fastecot.h.  See DESIGN.md.
"""

from .backends import (BackendError, EngineError, GenerationBackend, StepGenerator, StepProfile,
                       SyntheticBackend, SyntheticProfile, default_profile, length_plan, stable_digest)
from .batching import (EMPTY, PAD, BatchError, BatchSchedule, GenerationRequest, LatencyModel,
                       continuous_batch, padding_waste, schedule_cost, schedule_to_csv, static_batch)
from .schedulers import (MODES, BatchedEpisodes, CachedTrace, CacheSnapshot, ConfigError, EpisodeAborted,
                         ParallelAsyncRunner, ParallelSyncRunner, SchedulerConfig, SequentialRunner,
                         StepResult, decode_action, make_runner, observation_for, run_episode,
                         run_parallel_async, run_parallel_sync, run_sequential, summarize_results)
from .trace import (ActionVector, Context, ReasoningTrace, SchemaError, SchemaMismatchError, StepSchema,
                    StepSpec, TraceParseError, default_schema, deserialize_trace, serialize_trace,
                    trace_content_bytes, trace_update_ratio, update_ratio)


def EngineBackend(*args, **kwargs):
    """Lazily imported so the CPU-only mirror never needs the CUDA library."""
    from .engine_backend import EngineBackend as _EB
    return _EB(*args, **kwargs)


__version__ = "0.1.0"
