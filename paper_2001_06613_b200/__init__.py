"""seqreg-b200: the groupwise correlation dissimilarity D(y) and its gradient
(arXiv 2001.06613) as hand-written sm_100a CUDA behind a C-ABI library.

Drop-in for the reference hot path (/root/reference/pkg/src/seqreg/similarity.py:128-220):

    import paper_2001_06613_b200 as srb
    srb.install()          # seqreg.temporal now evaluates D, grad D on the GPU

Device-resident displacement-field objective (the north_star parametrisation):

    frames = srb.DeviceFrames(srb.get_engine(), data, srb.GridSpec(dims, spacing, origin))
    obj = srb.FieldObjective(frames, subset, weights)
    stats, grad = obj.evaluate(y)        # D = stats[0]
"""

from ._lib import EngineUnavailable, SingularSystemError, load_library
from .engine import DeviceFrames, Engine, EvalPlan, GridSpec, get_engine
from .field import FieldObjective
from .optimizer import ObjectiveEval, OptimOptions, OptimResult, lbfgs_minimize
from .similarity import (
    CorrelationState,
    configure,
    correlation_state,
    decompose,
    dissimilarity,
    dissimilarity_gradient,
    install,
    min_consecutive_rho,
    uninstall,
)
from .spatial import build_pyramid, prolong_field, pyramid_step
from .temporal import interp_linear_fields, ls_predict_fields

__version__ = "0.1.0"

__all__ = [
    "CorrelationState",
    "DeviceFrames",
    "Engine",
    "EngineUnavailable",
    "EvalPlan",
    "FieldObjective",
    "GridSpec",
    "SingularSystemError",
    "configure",
    "correlation_state",
    "decompose",
    "dissimilarity",
    "dissimilarity_gradient",
    "get_engine",
    "install",
    "interp_linear_fields",
    "load_library",
    "ls_predict_fields",
    "min_consecutive_rho",
    "ObjectiveEval",
    "OptimOptions",
    "OptimResult",
    "lbfgs_minimize",
    "build_pyramid",
    "prolong_field",
    "pyramid_step",
    "uninstall",
]
