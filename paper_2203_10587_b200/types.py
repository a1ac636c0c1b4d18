"""Boundary types of the hot path, field-identical to the reference's.

* :class:`NlpProblem` -- the callback container the solver calls
  (`pkg/src/opfkit/nlp.py:26-49`); kept a plain mutable dataclass because
  callers reassign ``x0``/``xl``/``xu``/callbacks (SURVEY §8b "Ownership").
* :class:`AcopfLayout` -- element -> NLP index maps (`acopf.py:52-71`).
* :class:`CouplingMode`, :class:`StageSpec`, :class:`CouplingRow`,
  :class:`CompositeIndexMap` -- composite lattice metadata
  (`composer.py:46-109`).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import InvalidPlan

PREVENTIVE = "preventive"
CORRECTIVE = "corrective"

RAMP = "Ramp"
CONTINGENCY_BOX = "ContingencyBox"
SCENARIO_BOX = "ScenarioBox"
PREVENTIVE_PIN = "PreventivePin"


@dataclass
class NlpProblem:
    """min f(x) s.t. c_eq(x)=0, gl<=c_ineq(x)<=gu, xl<=x<=xu (nlp.py:1-15).

    ``constraints`` returns [c_eq; c_ineq]; ``jacobian`` the matching CSR;
    ``lagrangian_hessian(x, obj_factor, mult)`` the full (both triangles)
    CSR of obj_factor*H(f) + sum_k mult[k]*H(c_k).  Patterns are fixed.
    """
    n: int
    m_eq: int
    m_ineq: int
    xl: np.ndarray
    xu: np.ndarray
    gl: np.ndarray
    gu: np.ndarray
    x0: np.ndarray
    objective: Callable
    gradient: Callable
    constraints: Callable
    jacobian: Callable
    lagrangian_hessian: Callable
    name: str = "nlp"

    def __post_init__(self) -> None:
        for attr in ("xl", "xu", "x0"):
            if getattr(self, attr).shape != (self.n,):
                raise ValueError(f"{attr} must have shape ({self.n},)")
        for attr in ("gl", "gu"):
            if getattr(self, attr).shape != (self.m_ineq,):
                raise ValueError(f"{attr} must have shape ({self.m_ineq},)")


@dataclass(frozen=True)
class AcopfLayout:
    n_vars: int
    n_eq: int
    n_ineq: int
    va: dict
    vm: dict
    pg: dict
    qg: dict
    p_row: dict
    q_row: dict
    sf_row: dict
    st_row: dict
    ref_buses: tuple


@dataclass(frozen=True)
class CouplingMode:
    kind: str = CORRECTIVE
    pin_voltages: bool = False
    contingency_scale: float = 1.0
    scenario_scale: float = 1.0

    def __post_init__(self):
        if self.kind not in (PREVENTIVE, CORRECTIVE):
            raise InvalidPlan(f"unknown coupling kind {self.kind!r}")


@dataclass(frozen=True)
class StageSpec:
    scenario: object
    contingency: object
    period: int
    dt_minutes: float
    case: object


@dataclass(frozen=True)
class CouplingRow:
    """row = absolute index into [eq; ineq]; value = stage_a - stage_b."""
    kind: str
    stage_a: int
    stage_b: int
    gen: int | None
    bus: int | None
    bound: float
    row: int
    is_equality: bool


@dataclass(frozen=True)
class CompositeIndexMap:
    stages: tuple
    var_offset: tuple
    eq_offset: tuple
    ineq_offset: tuple
    coupling_rows: tuple
    weights: tuple
    layouts: tuple
    n_vars: int
    m_eq: int
    m_ineq: int
