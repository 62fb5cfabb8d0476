"""Objective math of the search (PAPER Eqs. 1-3, 6, 7).

Scalar SPEC-literal functions (used by the host for single values and as
the definition the device epilogue reproduces operation for operation), the
deterministic ``exp_clv`` shared bit-for-bit with the kernels, and
``Scenario`` -- the evaluation parameters every scoring call takes.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, replace
from typing import Optional

from .core import ObjectiveParams
from .errors import CarbonSchedError

STRICT_ENV = "CARBON_SCHED_STRICT_EQ6"
RHO_SAT = 0.999                                 # queueing factor saturates at 1000x


def strict_eq6_default() -> bool:
    return os.environ.get(STRICT_ENV, "") == "1"


def delta_accuracy(a: float, params: ObjectiveParams) -> float:
    """Eq. 1: (A - A_base) / A_base * 100."""
    if not a > 0:
        raise CarbonSchedError("accuracy must be positive")
    return (a - params.base_accuracy) / params.base_accuracy * 100.0


def delta_carbon(e_wh_per_req: float, ci: float, params: ObjectiveParams) -> float:
    """Eq. 2: (C_base - E/1000 * ci) / C_base * 100 (PUE cancels, D7)."""
    if not params.base_carbon_g > 0:
        raise CarbonSchedError("c_base must be positive")
    return (params.base_carbon_g - e_wh_per_req / 1000.0 * ci) / params.base_carbon_g * 100.0


def objective_f(dc: float, da: float, lam: float) -> float:
    """Eq. 3: lambda * dC + (1 - lambda) * dA."""
    if not 0.0 <= lam <= 1.0:
        raise CarbonSchedError("lambda must be in [0,1]")
    return lam * dc + (1.0 - lam) * da


def energy_h(f: float, p95_ms: float, l_tail: float, strict: Optional[bool] = None) -> float:
    """Eq. 6 with the SPEC:479 amendment for f < 0 (verbatim form when strict)."""
    if not (l_tail > 0 and p95_ms > 0):
        raise CarbonSchedError("durations must be positive")
    if strict is None:
        strict = strict_eq6_default()
    if p95_ms <= l_tail:
        return -f
    if f >= 0 or strict:
        return -f * (l_tail / p95_ms)
    return -f * (p95_ms / l_tail)


# -- deterministic exp (H1): identical IEEE op sequence in Python and CUDA --------
_LN2_HI = float.fromhex("0x1.62e42fee00000p-1")
_LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
_INV_LN2 = float.fromhex("0x1.71547652b82fep+0")
# 1/k! for k = 13..2, rounded once (hex literals are mirrored in csrc/clv_common.cuh)
EXP_COEFFS = tuple(float.fromhex(h) for h in (
    "0x1.6124613a86d09p-33", "0x1.1eed8eff8d898p-29", "0x1.ae64567f544e4p-26",
    "0x1.27e4fb7789f5cp-22", "0x1.71de3a556c734p-19", "0x1.a01a01a01a01ap-16",
    "0x1.a01a01a01a01ap-13", "0x1.6c16c16c16c17p-10", "0x1.1111111111111p-7",
    "0x1.5555555555555p-5", "0x1.5555555555555p-3", "0x1.0000000000000p-1"))


def exp_clv(x: float) -> float:
    """exp(x) for x <= 0 by Cody-Waite reduction and a degree-13 Taylor polynomial.

    Only + - * and exact power-of-two scaling, so the device produces the same
    bits (kernels compile with -fmad=false).  Relative error < 1e-15.
    """
    if x < -708.0:
        return 0.0
    if x > 0.0:
        raise CarbonSchedError("exp_clv is defined for x <= 0")
    k = math.floor(x * _INV_LN2 + 0.5)
    r = (x - k * _LN2_HI) - k * _LN2_LO
    p = EXP_COEFFS[0]
    for c in EXP_COEFFS[1:]:
        p = p * r + c
    p = p * r + 1.0
    p = p * r + 1.0
    return math.ldexp(p, int(k))


def accept_prob(h_old: float, h_new: float, t: float) -> float:
    """Eq. 7."""
    if not t > 0:
        raise CarbonSchedError("temperature must be positive")
    if h_new <= h_old:
        return 1.0
    return exp_clv(-(h_new - h_old) / t)


def temperature(step: int, t_init: float, cooling_step: float, t_floor: float) -> float:
    """Subtractive cooling T_k = max(t_floor, t_init - k * step), computed directly (D3)."""
    return max(t_floor, t_init - step * cooling_step)


def uniform01(seed: int) -> float:
    """Uniform double in [0, 1) from a 63-bit seed: (u >> 10) * 2^-53 (D4)."""
    return (seed >> 10) * (1.0 / 9007199254740992.0)


@dataclass(frozen=True)
class Scenario:
    """Everything a candidate score depends on besides the graph and the tables.

    ``arrival_rps`` is R of the surrogate (Poisson rate of SPEC:321); ``ci`` the
    current carbon intensity; ``obj`` carries lambda, A_base, C_base, L_tail.
    """

    n_gpus: int
    arrival_rps: float
    ci: float
    obj: ObjectiveParams
    strict_eq6: bool = False
    rho_sat: float = RHO_SAT
    max_accuracy_loss_pct: float = math.inf   # accuracy_threshold_mode; inf = off

    def with_lambda(self, lam: float) -> "Scenario":
        return replace(self, obj=replace(self.obj, carbon_weight=lam))

    def with_ci(self, ci: float) -> "Scenario":
        return replace(self, ci=float(ci))

    def check(self) -> None:
        if self.n_gpus < 1:
            raise CarbonSchedError("n_gpus must be >= 1")
        if not (self.arrival_rps > 0 and math.isfinite(self.arrival_rps)):
            raise CarbonSchedError("arrival rate must be positive")
        if not (self.ci >= 0 and math.isfinite(self.ci)):
            raise CarbonSchedError("carbon intensity must be finite and >= 0")
        if not 0.0 < self.rho_sat < 1.0:
            raise CarbonSchedError("rho_sat must be in (0,1)")
        if not self.max_accuracy_loss_pct >= 0:
            raise CarbonSchedError("max_accuracy_loss_pct must be >= 0 (inf = off)")


PROPOSALS = ("best", "uniform")
EVALUATIONS = ("all", "proposal")


@dataclass(frozen=True)
class AnnealParams:
    """SA schedule.

    ``proposal``: "best" -- the lowest-h neighbour of a fully scored
    neighbourhood (ties: lowest canonical index); "uniform" -- a uniformly
    random legal neighbour, drawn as the neighbour with the smallest
    derive_seed(seed, chain, step, index + 1).  ``evaluate``: "all" scores the
    whole neighbourhood every step and tracks the best over all of it (BASELINE
    configs[1]); "proposal" scores only the proposal (SPEC-literal anneal).
    ``max_steps`` bounds steps; the SPEC's time budget additionally bounds the
    evaluation count in "proposal" mode (eval_cost_s per evaluation).
    ``move_set``: "spec" -- the m-invariant GED <= 4 swap / slice moves;
    "paper" -- also one-instance add / remove (GED 1).  ``cooling``:
    "subtractive" (T_k = max(t_floor, t_init - k cooling_step)) or "multiplicative"
    (T_k = max(t_floor, t_init (1 - cooling_step)^k), both SPEC:492).
    """

    def flags(self) -> int:
        """clv_anneal_params.flags (include/clover.h)."""
        return (1 if self.cooling == "multiplicative" else 0) | (2 if self.move_set == "paper" else 0)

    t_init: float = 1.0
    cooling_step: float = 0.05
    t_floor: float = 0.1
    stall_limit: int = 5
    time_budget_s: float = 300.0
    eval_cost_s: float = 45.0
    max_steps: int = 64
    proposal: str = "best"
    evaluate: str = "all"
    move_set: str = "spec"          # "paper": + unit instance add / remove
    cooling: str = "subtractive"    # "multiplicative": T_k = t_init (1 - cooling_step)^k

    def __post_init__(self) -> None:
        if self.move_set not in ("spec", "paper") or self.cooling not in ("subtractive", "multiplicative"):
            raise CarbonSchedError("unknown move set / cooling mode")
        if not self.t_floor > 0 or not self.cooling_step > 0 or self.t_init < self.t_floor:
            raise CarbonSchedError("invalid temperature schedule")
        if self.stall_limit < 1 or self.max_steps < 0:
            raise CarbonSchedError("stall_limit must be >= 1 and max_steps >= 0")
        if self.proposal not in PROPOSALS or self.evaluate not in EVALUATIONS:
            raise CarbonSchedError("unknown proposal/evaluate mode")
        if self.proposal == "best" and self.evaluate != "all":
            raise CarbonSchedError("proposal='best' needs evaluate='all'")

    def step_limit(self) -> int:
        """Steps allowed: max_steps, and in 'proposal' mode the SPEC budget
        (stop once evaluations * eval_cost_s >= time_budget_s; the start counts)."""
        if self.evaluate == "proposal" and self.eval_cost_s > 0 and math.isfinite(self.time_budget_s):
            evals = max(1, math.ceil(self.time_budget_s / self.eval_cost_s))
            return min(self.max_steps, evals - 1)
        return self.max_steps


STATUS_MAX_STEPS = 0
STATUS_STALLED = 1
STATUS_NO_NEIGHBOR = 2
STATUS_NAMES = {0: "max_steps", 1: "stalled", 2: "no_neighbor"}
