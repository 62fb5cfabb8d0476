"""The reference-side binding of INTEGRATION.md §3, exercised as written: plain ctypes on
libclover_b200.so (no engine, no torch buffers) runs the exhaustive ORACLE of c0 and must
select exactly what the engine (and hence the CPU oracle, tests/test_gpu_parity.py) selects."""

import ctypes
import os

import pytest

from paper_2304_09781_b200.core import SLICE_ORDER
from paper_2304_09781_b200.mig import DEFAULT_TOPOLOGY
from paper_2304_09781_b200.profiles import synthetic_profile

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2304_09781_b200",
                   "libclover_b200.so")


class EvalParams(ctypes.Structure):
    _fields_ = [("arrival_rps", ctypes.c_double), ("ci", ctypes.c_double), ("carbon_weight", ctypes.c_double),
                ("base_accuracy", ctypes.c_double), ("base_carbon_g", ctypes.c_double),
                ("latency_slo_ms", ctypes.c_double), ("rho_sat", ctypes.c_double), ("strict_eq6", ctypes.c_int32),
                ("n_gpus", ctypes.c_int32), ("max_accuracy_loss_pct", ctypes.c_double)]


class Best(ctypes.Structure):
    _fields_ = [("index", ctypes.c_int64), ("f", ctypes.c_double), ("h", ctypes.c_double),
                ("p95_ms", ctypes.c_double), ("accuracy", ctypes.c_double), ("energy_wh", ctypes.c_double),
                ("sla_met", ctypes.c_int32), ("found", ctypes.c_int32), ("valid_count", ctypes.c_int64),
                ("sla_count", ctypes.c_int64)]


class AnnealParams(ctypes.Structure):
    _fields_ = [("t_init", ctypes.c_double), ("cooling_step", ctypes.c_double), ("t_floor", ctypes.c_double),
                ("stall_limit", ctypes.c_int32), ("max_steps", ctypes.c_int32), ("proposal", ctypes.c_int32),
                ("evaluate", ctypes.c_int32), ("flags", ctypes.c_int32)]


class ChainResult(ctypes.Structure):
    _fields_ = [("f", ctypes.c_double), ("h", ctypes.c_double), ("p95_ms", ctypes.c_double),
                ("accuracy", ctypes.c_double), ("energy_wh", ctypes.c_double), ("sla_met", ctypes.c_int32),
                ("status", ctypes.c_int32), ("steps", ctypes.c_int32), ("best_step", ctypes.c_int32),
                ("best_index", ctypes.c_int64), ("evals", ctypes.c_int64), ("edge_evals", ctypes.c_int64)]


class Record(ctypes.Structure):
    _fields_ = [("k1", ctypes.c_uint64), ("k2", ctypes.c_uint64), ("index", ctypes.c_int64), ("h", ctypes.c_double)]


def _vector(slices):
    v = [0] * 5
    for s in slices:
        v[SLICE_ORDER.index(s)] += 1
    return v


def test_reference_style_ctypes_binding_runs_the_oracle(engine):
    lib = ctypes.CDLL(LIB)
    lib.clv_last_error.restype = ctypes.c_char_p
    ctx = ctypes.c_void_p()
    assert lib.clv_create(0, ctypes.byref(ctx)) == 0
    try:
        topo = DEFAULT_TOPOLOGY
        ids = sorted(topo.config_ids)
        counts = [c for cid in ids for c in _vector(topo.config_slices(cid))]
        mem = [topo.slice_memory(s) for s in SLICE_ORDER]
        assert lib.clv_set_topology(ctx, len(ids), (ctypes.c_int32 * len(ids))(*ids),
                                    (ctypes.c_int32 * len(counts))(*counts), (ctypes.c_double * 5)(*mem)) == 0
        assert lib.clv_build_feasibility(ctx, 1, None) == 0
        prof = synthetic_profile("efficientnet")
        t = prof.scoring_tables()
        i64 = lambda xs: (ctypes.c_int64 * len(xs))(*[int(x) for x in xs])
        f64 = lambda xs: (ctypes.c_double * len(xs))(*[float(x) for x in xs])
        u8 = lambda xs: (ctypes.c_uint8 * len(xs))(*[int(x) for x in xs])
        assert lib.clv_set_profile(ctx, 0, t.variant_count, i64(t.thr_q), i64(t.acc_q), i64(t.en_q), i64(t.idle_q),
                                   f64(t.lat95), f64(t.svc_ms), u8(t.mem_ok), t.kt, t.ke, t.ki) == 0
        sc = engine.calibrate(prof, 1, 400.0, 0.5)
        o = sc.obj
        p = EvalParams(sc.arrival_rps, sc.ci, o.carbon_weight, o.base_accuracy, o.base_carbon_g, o.latency_slo_ms,
                       sc.rho_sat, 1 if sc.strict_eq6 else 0, 1, float("inf"))
        best, total = Best(), ctypes.c_int64()
        rc = lib.clv_oracle_search(ctx, 0, 1, 0, -1, ctypes.byref(p), ctypes.byref(best), ctypes.byref(total), None)
        assert rc == 0, lib.clv_last_error(ctx)
        ref = engine.oracle_search(prof, sc)
        assert (best.index, best.found, best.valid_count, total.value) == (ref["index"], ref["found"],
                                                                            ref["valid_count"], ref["total"])
        assert best.f == ref["f"] and best.h == ref["h"]
        # error mapping: an unknown family is "not ready" (102) with a message
        assert lib.clv_oracle_search(ctx, 5, 1, 0, -1, ctypes.byref(p), ctypes.byref(best), ctypes.byref(total),
                                     None) == 102
        assert b"family" in lib.clv_last_error(ctx)
    finally:
        lib.clv_destroy(ctx)


def test_reference_style_ctypes_binding_replans(engine):
    """INTEGRATION.md §3's Accelerator.replan: plain ctypes host buffers through clv_replan
    (the e2e path of bench.py) give the engine's chains, bit for bit."""
    import bench
    lib = ctypes.CDLL(LIB)
    lib.clv_last_error.restype = ctypes.c_char_p
    ctx = ctypes.c_void_p()
    assert lib.clv_create(0, ctypes.byref(ctx)) == 0
    try:
        topo = DEFAULT_TOPOLOGY
        ids = sorted(topo.config_ids)
        counts = [c for cid in ids for c in _vector(topo.config_slices(cid))]
        mem = [topo.slice_memory(s) for s in SLICE_ORDER]
        assert lib.clv_set_topology(ctx, len(ids), (ctypes.c_int32 * len(ids))(*ids),
                                    (ctypes.c_int32 * len(counts))(*counts), (ctypes.c_double * 5)(*mem)) == 0
        assert lib.clv_build_feasibility(ctx, 64, None) == 0
        prof = synthetic_profile("efficientnet")
        t = prof.scoring_tables()
        i64 = lambda xs: (ctypes.c_int64 * len(xs))(*[int(x) for x in xs])
        f64 = lambda xs: (ctypes.c_double * len(xs))(*[float(x) for x in xs])
        u8 = lambda xs: (ctypes.c_uint8 * len(xs))(*[int(x) for x in xs])
        assert lib.clv_set_profile(ctx, 0, t.variant_count, i64(t.thr_q), i64(t.acc_q), i64(t.en_q), i64(t.idle_q),
                                   f64(t.lat95), f64(t.svc_ms), u8(t.mem_ok), t.kt, t.ke, t.ki) == 0
        sc = engine.calibrate(prof, 64, 350.0, 0.5)
        o = sc.obj
        p = EvalParams(sc.arrival_rps, sc.ci, o.carbon_weight, o.base_accuracy, o.base_carbon_g, o.latency_slo_ms,
                       sc.rho_sat, 1 if sc.strict_eq6 else 0, 64, float("inf"))
        ap_py = bench.anneal_params(20)
        ap = AnnealParams(ap_py.t_init, ap_py.cooling_step, ap_py.t_floor, ap_py.stall_limit, ap_py.step_limit(),
                          0, 0, 0)
        starts = bench.make_starts(prof, 3, 0, 24, 0.75)
        m, E = starts.shape
        w = (ctypes.c_uint16 * (m * E))(*[int(x) for x in starts.reshape(-1)])
        res, rec = (ChainResult * m)(), Record()
        best, final = (ctypes.c_uint16 * (m * E))(), (ctypes.c_uint16 * (m * E))()
        rc = lib.clv_replan(ctx, 0, 64, m, ctypes.c_int64(0), w, ctypes.byref(p), 1, ctypes.byref(ap),
                            ctypes.c_uint64(9), 0, res, best, final, ctypes.byref(rec), None)
        assert rc == 0, lib.clv_last_error(ctx)
        r_e, b_e, _, rec_e = engine.replan(starts, prof, sc, ap_py, 9, cluster=0)
        assert bytes(res) == r_e.tobytes()
        assert list(best) == [int(x) for x in b_e.reshape(-1)]
        assert rec.index == int(rec_e["index"]) and rec.h == float(rec_e["h"])
    finally:
        lib.clv_destroy(ctx)
