"""B200-native TN-structured linear layer (Tucker / TT / TR) — drop-in for the
forward path of arxiv/paper_2602_01613 ("Minima"): ``CompressedLayer`` built
from factor cores, ``forward(x)``, ``reconstruct`` / ``layer_to_matrix``.

All compute runs in ``libtnl.so`` (hand-written sm_100a CUDA behind the C-ABI
in ``include/tnl.h``). There is no CPU fallback.
"""

from . import modes
from ._native import PLAN_AUTO, PLAN_CHAIN, PLAN_CUT, PLAN_GEMV, PLAN_GENERIC, PLAN_NO_DECODE, launch_count
from .errors import (
    DegenerateReferenceError,
    DeviceError,
    InfeasibleBudgetError,
    MinimaError,
    NumericsError,
    RankError,
    ShapeError,
    UnsupportedError,
)
from .layer import (
    CompressedLayer,
    NativePlan,
    apply_compressed,
    compression_ratio,
    from_compressed_layer,
    layer_to_matrix,
    param_count,
    reconstruct,
)
from .modes import balanced_split, default_mode_shape, maximal_ranks, param_count_formula, select_ranks
from .contraction import flop_report, plan_contraction, relative_error, reshape_to_modes

__all__ = [
    "CompressedLayer",
    "NativePlan",
    "apply_compressed",
    "compression_ratio",
    "from_compressed_layer",
    "layer_to_matrix",
    "param_count",
    "param_count_formula",
    "reconstruct",
    "balanced_split",
    "default_mode_shape",
    "maximal_ranks",
    "select_ranks",
    "relative_error",
    "reshape_to_modes",
    "plan_contraction",
    "flop_report",
    "modes",
    "launch_count",
    "PLAN_AUTO",
    "PLAN_CUT",
    "PLAN_CHAIN",
    "PLAN_GENERIC",
    "PLAN_NO_DECODE",
    "PLAN_GEMV",
    "MinimaError",
    "ShapeError",
    "NumericsError",
    "RankError",
    "DegenerateReferenceError",
    "InfeasibleBudgetError",
    "DeviceError",
    "UnsupportedError",
]
