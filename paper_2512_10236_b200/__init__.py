"""FiCCO on B200: finer-grain compute/communication overlap, B200-native.

Drop-in for the hot path of the reference ``overlap_sim`` package
(/root/reference/pkg/src/overlap_sim/__init__.py:35-64): every name it
exports is exported here with the same meaning. Planning, selection and the
analytic simulator are host-side Python; execution of a plan on real tensors
goes through the C-ABI library ``libficco_b200.so`` (copy-engine transfers +
tcgen05 tile kernel for sm_100a), see ``executor`` and ``ops``.
"""

import os as _os

# The executor's persistent tile kernel spins on readiness flags that copy-engine chains on other streams
# set. With CUDA's default of 8 hardware work queues, the communicator's 16 copy streams and the caller's
# stream alias onto shared queues, so a copy chain can end up queued behind work that waits for that very
# kernel: the run then stalls until the flag timeout (seen as a DeadlockError). 32 queues give every stream
# its own. CUDA reads the variable when the context is created, so it is set here at import unless the
# caller set it (import this package, or set the variable, before the first CUDA call).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .domain import (Axis, Collective, CommAgent, GemmShape, MachineConfig, Parallelism, Scenario,
                     ScenarioParseError, ShardedGemm, gemm_flops, gemm_mt, gemm_otb, parse_scenarios,
                     serialize_scenarios, shard_gemm)
from .pricing import (CalibrationError, LossModel, Topology, TopologyKind, default_calibration,
                      load_calibration)
from .routing import (ALL_KINDS, FINE_GRAIN_KINDS, ExecutionPlan, PlanError, ScheduleKind, build_plan,
                      export_plan_csv, supported_kinds, validate_plan)
from .simulator import DeadlockError, SimResult, TaskSpan, export_trace_csv, simulate, speedup
from .selector import HeuristicReport, select_schedule, validate_heuristic
from .machines import MachineSpec, b200_machine, default_machine, example_machine, load_machine

__version__ = "0.1.0"

__all__ = [
    "Axis", "Collective", "CommAgent", "GemmShape", "MachineConfig", "Parallelism", "Scenario",
    "ShardedGemm", "gemm_flops", "gemm_mt", "gemm_otb", "parse_scenarios", "shard_gemm",
    "Topology", "TopologyKind", "LossModel", "default_calibration", "load_calibration",
    "ExecutionPlan", "ScheduleKind", "build_plan", "validate_plan", "SimResult", "simulate", "speedup",
    "select_schedule", "validate_heuristic", "__version__",
    # additions beyond the reference's __all__
    "ScenarioParseError", "serialize_scenarios", "CalibrationError", "ALL_KINDS", "FINE_GRAIN_KINDS",
    "PlanError", "export_plan_csv", "supported_kinds", "DeadlockError", "TaskSpan", "export_trace_csv",
    "HeuristicReport", "MachineSpec", "b200_machine", "default_machine", "example_machine", "load_machine",
]
