"""B200-native batch-parallel speculative decoding (MineDraft PSD).

Drop-in for the hot path of the reference package ``specsim``
(pkg/src/specsim/__init__.py:62-109): the two-batch PSD scheduler
(``run`` / ``step_once`` / ``new_state``), its protocol components
(``BatchManager``, ``KVBlockTable``, acceptance streams) and the
acceptance-statistics output (``StepRecord``, ``MetricsReport``, step-log /
metrics formats).  The reference's virtual-time latency and coin-flip
acceptance are replaced by a backend:

* ``SimBackend`` -- the reference models, byte-identical step logs;
* ``GpuBackend`` -- real draft/target transformer forwards and the fused
  speculative-verification kernel on sm_100a, via ``libpsd.so`` (C ABI in
  include/psd.h).  Importing it on a machine without the built library raises
  ``NativeError``; there is no CPU fallback.

The closed-form theory module, config files, trace workloads and CLI of the
reference are out of scope.
"""

from .acceptance import AcceptanceModel, acceptance_stream, accepted_count, expected_accepted
from .batches import BatchManager
from .errors import (CapacityError, ConfigError, KVError, NativeError, NumericError,
                     ProtocolError, SpecsimError, WorkloadError)
from .ktune import KTuner
from .kvtable import AllocationContext, BlockPool, KVBlockTable, blocks_needed
from .metrics import (MetricsReport, accepted_per_verify, compute_metrics,
                      mean_accepted_length, percentile_nearest_rank, render_metrics,
                      render_step_log)
from .records import (LatencyModel, Request, RequestState, SimConfig, StepRecord,
                      validate_config)
from .scheduler import (EngineState, FinishRecord, KvStepRecord, PendingDraft,
                        Preemption, StepPlan, StepResult, VerifyRow, new_state, run,
                        step_once)
from .sim import SimBackend
from .workload import (LengthSpec, WorkloadSpec, attach_prompt_ids, generate_requests,
                       make_requests, parse_preemptions)

__version__ = "0.1.0"

__all__ = [
    "KTuner",
    "AcceptanceModel", "AllocationContext", "BatchManager", "BlockPool",
    "CapacityError", "ConfigError", "EngineState", "FinishRecord", "KVBlockTable",
    "KVError", "KvStepRecord", "LatencyModel", "LengthSpec", "MetricsReport",
    "NativeError", "NumericError", "PendingDraft", "Preemption", "ProtocolError",
    "Request", "RequestState", "SimBackend", "SimConfig", "SpecsimError", "StepPlan",
    "StepRecord", "StepResult", "VerifyRow", "WorkloadError", "WorkloadSpec",
    "acceptance_stream", "accepted_count", "accepted_per_verify",
    "attach_prompt_ids", "blocks_needed", "compute_metrics", "expected_accepted",
    "generate_requests", "make_requests", "mean_accepted_length", "new_state",
    "parse_preemptions", "percentile_nearest_rank", "render_metrics",
    "render_step_log", "run", "step_once", "validate_config", "__version__",
]


def __getattr__(name):  # lazy: the GPU backend needs libpsd.so and torch
    if name == "GpuBackend":
        from .gpu import GpuBackend
        return GpuBackend
    raise AttributeError(name)
