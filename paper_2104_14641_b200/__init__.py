"""loopscout-b200: the batched schedule-cost path of loopscout (Tuna, arXiv 2104.14641) on B200.

The names below mirror the reference package's public surface for this path
(ls/__init__.py:3-15), so ``from paper_2104_14641_b200 import optimize, load_arch, ...``
replaces ``from loopscout import ...`` for ranking and search.  Scoring runs in
the sm_100a kernels of libloopscout_b200.so (include/loopscout_b200.h); there is
no CPU fallback.  The batched seams the reference CLI calls are
``evaluate_schedules`` (cmd_rank, ls/cli.py:115-121) and ``optimize``
(cmd_search, ls/cli.py:152); ``score_batch`` / ``rank_topk`` are the array forms.
"""

from .arch import (ArchSpec, CostModelError, FeatureVector, GpuSpec, KernelLaunch, load_arch)
from .backend import evaluate_schedules
from .code import AsmError, code_features, extract_features
from .cost import analyze, rank, rank_schedules, rank_topk, score, score_batch
from .es import EsParams, OptimizeResult, SearchError, ThetaEncoding, optimize, optimize_device
from .ir import (AccessNode, AffineExpr, LoopNode, LoopProgram, Parallel, ProgramError, Reorder, Schedule,
                 TensorDecl, Tile, Unroll, Vectorize, parse_program, space_axes)

__version__ = "0.2.0"

__all__ = [
    "AccessNode", "AffineExpr", "ArchSpec", "AsmError", "CostModelError", "EsParams", "FeatureVector", "GpuSpec",
    "KernelLaunch", "LoopNode", "LoopProgram", "OptimizeResult", "Parallel", "ProgramError", "Reorder",
    "Schedule", "SearchError", "TensorDecl", "ThetaEncoding", "Tile", "Unroll", "Vectorize", "analyze",
    "code_features", "evaluate_schedules", "extract_features", "load_arch", "optimize", "optimize_device", "parse_program", "rank",
    "rank_schedules", "rank_topk", "score", "score_batch", "space_axes",
]
