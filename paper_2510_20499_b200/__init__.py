"""B200-native bound-propagation engine (drop-in for the reference's propagation / probing /
fix-and-propagate hot path, arXiv 2510.20499).

The compute path is hand-written sm_100a CUDA behind the C-ABI in include/bp.h
(``libbp.so``); this package is the Python host mirror of the reference's C++ API.
"""
from .problem import (K_INF, ProblemBuilder, ProblemDef, make_problem, problem_from_csr,
                      round_integer_bounds)
from .propagation import (ActivityState, BoundsState, PropagationLimits, PropagationResult,
                          PropagationStatus, WorkPlan, build_work_plan, compute_activities,
                          propagate, propagate_device, set_device, size_class_of, tighten_bounds)

__all__ = [
    "K_INF", "ProblemBuilder", "ProblemDef", "make_problem", "problem_from_csr",
    "round_integer_bounds", "ActivityState", "BoundsState", "PropagationLimits",
    "PropagationResult", "PropagationStatus", "WorkPlan", "build_work_plan", "compute_activities",
    "propagate", "propagate_device", "set_device", "size_class_of", "tighten_bounds",
]
