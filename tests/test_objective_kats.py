"""SPEC known-answer tests for Eqs. 1, 2, 3, 6, 7 (acceptance criterion 10)."""

import math

import numpy as np
import pytest

from oracle.evaluator import calibrate, evaluate
from oracle.rng import exp_clv as oracle_exp
from oracle.tables import OracleTables
from paper_2304_09781_b200.core import ObjectiveParams
from paper_2304_09781_b200.objective import (accept_prob, delta_accuracy, delta_carbon, energy_h, exp_clv,
                                             objective_f, temperature)
from paper_2304_09781_b200.profiles import synthetic_profile
from tests.helpers import random_fleet_graphs


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def test_eq1_delta_accuracy():
    p = ObjectiveParams(0.8, 10.0, 100.0)
    assert delta_accuracy(0.8, p) == 0.0
    assert close(delta_accuracy(0.76, p), -5.0)
    assert close(delta_accuracy(0.792, p), -1.0)


def test_eq2_delta_carbon():
    p = ObjectiveParams(0.8, 10.0, 100.0)
    assert close(delta_carbon(6.0, 500.0, p), 70.0)
    assert close(delta_carbon(6.0, 100.0, p), 94.0)
    assert close(delta_carbon(10.0 * 1000.0 / 400.0, 400.0, p) + 1.0, 1.0)   # break-even


def test_eq3_objective():
    assert objective_f(70.0, -3.0, 1.0) == 70.0
    assert objective_f(70.0, -3.0, 0.0) == -3.0
    assert close(objective_f(70.0, -3.0, 0.5), 33.5)
    for lam in np.linspace(0, 1, 11):     # affine in lambda
        f0, f1 = objective_f(70.0, -3.0, 0.0), objective_f(70.0, -3.0, 1.0)
        assert close(objective_f(70.0, -3.0, lam), f0 + lam * (f1 - f0), 1e-14)


def test_eq6_energy():
    assert energy_h(40.0, 50.0, 100.0, strict=False) == -40.0
    assert energy_h(40.0, 200.0, 100.0, strict=False) == -20.0
    assert energy_h(-10.0, 200.0, 100.0, strict=False) == 20.0
    assert energy_h(-10.0, 200.0, 100.0, strict=True) == 5.0        # verbatim Eq. 6
    for f in (-10.0, 0.0, 40.0):                                     # monotone beyond L_tail
        hs = [energy_h(f, p, 100.0, strict=False) for p in np.linspace(100.0, 1000.0, 200)]
        assert all(x <= y for x, y in zip(hs, hs[1:]))
    for f in (-3.0, 0.0, 7.0):                                       # h = -f when the SLA holds
        assert energy_h(f, 99.0, 100.0) == -f


def test_eq7_accept_and_exp():
    assert accept_prob(1.0, 0.5, 0.3) == 1.0
    assert close(accept_prob(0.0, 1.0, 1.0), math.exp(-1.0), 1e-15)
    assert close(accept_prob(0.0, 1.0, 0.1), 4.539992976248485e-05, 1e-14)
    xs = np.concatenate([-np.linspace(0, 700, 5001), -np.random.default_rng(1).random(5000)])
    for x in xs:
        a, b = exp_clv(float(x)), oracle_exp(float(x))
        assert a == b                                                # product == oracle, bit for bit
        assert close(a, math.exp(x), 4e-16)
    assert temperature(18, 1.0, 0.05, 0.1) == 0.1 and temperature(0, 1.0, 0.05, 0.1) == 1.0


@pytest.mark.parametrize("family", ["efficientnet", "bert"])
def test_batched_eq1_eq2_forms_match_spec_literal(family):
    """The evaluator's (A-A_base)*kA and 100-E*kC forms vs the SPEC-literal quotients."""
    prof = synthetic_profile(family)
    T = OracleTables.from_profile(prof)
    sc = calibrate(prof, T, 8, 420.0, 0.35)
    W = random_fleet_graphs(T, 8, 400, seed=3)
    ev = evaluate(W, T, sc)
    for A, E, f in zip(ev.A, ev.E, ev.f):
        da = delta_accuracy(float(A), sc.obj)
        dc = delta_carbon(float(E), sc.ci, sc.obj)
        ff = objective_f(dc, da, sc.obj.carbon_weight)
        assert abs(ff - f) <= 1e-12 * max(abs(ff), 100.0)
