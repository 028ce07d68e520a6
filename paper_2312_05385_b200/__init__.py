"""B200-native early-exit decision path (Apparate, arXiv 2312.05385).

Drop-in for the exit-decision / threshold-tuning hot path of the reference
package `eesim`: the same public API (ramp placement, EEConfig thresholds,
tune / grid_oracle, AccuracyMonitor) with every window evaluation running in
hand-written sm_100a kernels (libeeb200.so, C ABI in include/eeb200.h).
Importing the package never touches the GPU; the first evaluation does, and
fails loudly if the library or a CUDA device is missing.
"""

__version__ = "0.1.0"

from paper_2312_05385_b200.engine import (
    EEConfig,
    ExitOutcome,
    ServedRecord,
    WindowEvaluator,
    WindowStats,
    decision_scores,
    evaluate_record,
    evaluate_window,
    optimal_exit,
    serve_table,
)
from paper_2312_05385_b200.errors import (
    EESimError,
    GraphError,
    GridCapError,
    NativeError,
    ParameterError,
    ValidationError,
)
from paper_2312_05385_b200.graph import (
    ModelProfile,
    RampBudget,
    RampSite,
    find_feasible_sites,
    initial_placement,
    load_profile,
    save_profile,
)
from paper_2312_05385_b200.trace import (
    RampSignal,
    RequestRecord,
    WindowArrays,
    Workload,
    load_workload,
    save_workload,
    synthesize_workload,
    window_arrays,
)
from paper_2312_05385_b200.tuner import (
    AccuracyMonitor,
    GridResult,
    TuneResult,
    TunerParams,
    grid_oracle,
    should_trigger,
    snap_down,
    threshold_lattice,
    tune,
)

__all__ = [
    "AccuracyMonitor", "EEConfig", "EESimError", "ExitOutcome", "GraphError", "GridCapError",
    "GridResult", "ModelProfile", "NativeError", "ParameterError", "RampBudget", "RampSignal",
    "RampSite", "RequestRecord", "ServedRecord", "TuneResult", "TunerParams", "ValidationError",
    "WindowArrays", "WindowEvaluator", "WindowStats", "Workload", "decision_scores",
    "evaluate_record", "evaluate_window", "find_feasible_sites", "grid_oracle",
    "initial_placement", "load_profile", "load_workload", "optimal_exit", "save_profile",
    "save_workload", "serve_table", "should_trigger", "snap_down", "synthesize_workload",
    "threshold_lattice", "tune", "window_arrays",
]
