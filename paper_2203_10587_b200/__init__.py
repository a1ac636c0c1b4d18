"""B200-native evaluation of the ExaGO-style ACOPF model callbacks.

Drop-in for the hot path of the reference toolkit (``opfkit``): the stage
model ``build_acopf`` and the composite builders ``compose_*`` return the
same ``NlpProblem`` / ``AcopfLayout`` / ``CompositeIndexMap`` objects, but
every callback (objective, gradient, constraints, Jacobian values,
Lagrangian-Hessian values) of every stage runs in one fused sm_100a fp64
kernel (libacopf_b200.so, C ABI in include/acopf_b200.h).  There is no CPU
fallback: if the library is missing the first evaluation raises.
"""

from . import errors
from .errors import Disconnected, DimensionMismatch, DeviceError
from .evaluator import BatchEvaluator, Coupling, StagePlan
from .grid import (
    BRANCH, GEN, ISOLATED, PQ, PV, REF,
    Branch, Bus, Contingency, ContingencySet, GenCost, Generator, LoadProfile, NetworkCase,
    Outage, Scenario, ScenarioSet, apply_contingency, apply_load_step, apply_scenario,
    branch_admittance, check_connectivity, declare_wind,
)
from .lattice import (
    compose_general, compose_multiperiod, compose_multiperiod_scopf, compose_scopf,
    compose_sopf_flat, compose_sopf_full,
)
from .solution import (
    SolvedCase, extract_solution, extract_solutions, pack_solution, residuals_at, solution_from_case,
)
from .stage import build_acopf
from .types import (
    CONTINGENCY_BOX, CORRECTIVE, PREVENTIVE, PREVENTIVE_PIN, RAMP, SCENARIO_BOX,
    AcopfLayout, CompositeIndexMap, CouplingMode, CouplingRow, NlpProblem, StageSpec,
)

__version__ = "0.1.0"

__all__ = [
    "AcopfLayout", "BatchEvaluator", "Branch", "Bus", "CompositeIndexMap", "Contingency",
    "ContingencySet", "Coupling", "CouplingMode", "CouplingRow", "CORRECTIVE", "CONTINGENCY_BOX",
    "DeviceError", "DimensionMismatch", "Disconnected", "GenCost", "Generator", "LoadProfile",
    "NetworkCase", "NlpProblem", "Outage", "PREVENTIVE", "PREVENTIVE_PIN", "RAMP", "SCENARIO_BOX",
    "Scenario", "ScenarioSet", "SolvedCase", "StagePlan", "StageSpec", "apply_contingency", "apply_load_step",
    "apply_scenario", "branch_admittance", "build_acopf", "check_connectivity", "compose_general",
    "compose_multiperiod", "compose_multiperiod_scopf", "compose_scopf", "compose_sopf_flat",
    "compose_sopf_full", "declare_wind", "errors", "extract_solution", "extract_solutions",
    "pack_solution", "residuals_at", "solution_from_case",
]
