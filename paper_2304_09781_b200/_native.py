"""ctypes binding of libclover_b200.so (include/clover.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every engine call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from . import errors as E

# CLV_LIB_PATH: an alternative in-tree build of the same ABI (A/B timing of kernel variants)
LIB_PATH = os.environ.get("CLV_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                           "libclover_b200.so")

c_i32, c_i64, c_u64, c_f64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class EvalParams(ctypes.Structure):
    _fields_ = [("arrival_rps", c_f64), ("ci", c_f64), ("carbon_weight", c_f64),
                ("base_accuracy", c_f64), ("base_carbon_g", c_f64), ("latency_slo_ms", c_f64),
                ("rho_sat", c_f64), ("strict_eq6", c_i32), ("n_gpus", c_i32), ("max_accuracy_loss_pct", c_f64)]


class Best(ctypes.Structure):
    _fields_ = [("index", c_i64), ("f", c_f64), ("h", c_f64), ("p95_ms", c_f64),
                ("accuracy", c_f64), ("energy_wh", c_f64), ("sla_met", c_i32), ("found", c_i32),
                ("valid_count", c_i64), ("sla_count", c_i64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class AnnealParamsC(ctypes.Structure):
    _fields_ = [("t_init", c_f64), ("cooling_step", c_f64), ("t_floor", c_f64),
                ("stall_limit", c_i32), ("max_steps", c_i32), ("proposal", c_i32), ("evaluate", c_i32),
                ("flags", c_i32)]


class ChainResult(ctypes.Structure):
    _fields_ = [("f", c_f64), ("h", c_f64), ("p95_ms", c_f64), ("accuracy", c_f64),
                ("energy_wh", c_f64), ("sla_met", c_i32), ("status", c_i32), ("steps", c_i32),
                ("best_step", c_i32), ("best_index", c_i64), ("evals", c_i64), ("edge_evals", c_i64)]


class LogRow(ctypes.Structure):
    _fields_ = [("temp", c_f64), ("f", c_f64), ("h", c_f64), ("p95_ms", c_f64), ("iter", c_i32),
                ("ged_from_center", c_i32), ("sla_met", c_i32), ("accepted", c_i32),
                ("new_best", c_i32), ("n_neighbours", c_i32)]


class Record(ctypes.Structure):
    _fields_ = [("k1", c_u64), ("k2", c_u64), ("index", c_i64), ("h", c_f64)]


class Pod(ctypes.Structure):
    _fields_ = [("family", c_i32), ("n_gpus", c_i32), ("weight", c_f64), ("params", EvalParams)]


class Workload(ctypes.Structure):
    _fields_ = [("arrival_rps", c_f64), ("duration_s", c_f64), ("seed", c_u64), ("periodic", c_i32),
                ("warmup", c_i32)]


class SimReport(ctypes.Structure):
    _fields_ = [("p95_ms", c_f64), ("mean_latency_ms", c_f64), ("throughput_rps", c_f64),
                ("energy_wh_total", c_f64), ("energy_wh_per_request", c_f64), ("accuracy", c_f64),
                ("completed", c_i64), ("counted", c_i64), ("sla_met", c_i32), ("status", c_i32)]


STATUS_TO_ERROR = {
    1: E.CarbonSchedError, 2: E.InvalidConfigError, 3: E.InfeasibleAssignmentError,
    4: E.IncompatibleGraphsError, 5: E.InfeasibleGraphError, 6: E.NoNeighborError,
    7: E.ProfileError, 8: E.TraceError, 9: E.SimulationError,
    100: E.DeviceError, 101: E.DeviceError, 102: E.CarbonSchedError,
}

# name -> (restype, argtypes); mirrors include/clover.h
SIGNATURES = {
    "clv_abi_version": (c_i32, []),
    "clv_create": (c_i32, [c_i32, ctypes.POINTER(c_vp)]),
    "clv_destroy": (None, [c_vp]),
    "clv_last_error": (ctypes.c_char_p, [c_vp]),
    "clv_derive_seed": (c_u64, [ctypes.POINTER(c_u64), c_i32]),
    "clv_set_topology": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp]),
    "clv_set_profile": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32]),
    "clv_build_feasibility": (c_i32, [c_vp, c_i32, c_vp]),
    "clv_feasibility_bytes": (c_i64, [c_vp]),
    "clv_feasible": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_vp, c_vp]),
    "clv_realize": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp]),
    "clv_score_graphs": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_i64, ctypes.POINTER(EvalParams), c_i32,
                                 c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(Best), c_vp]),
    "clv_score_x": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_i64, c_i64, ctypes.POINTER(EvalParams),
                            c_i32, c_vp, c_vp, c_vp, ctypes.POINTER(Best), c_vp]),
    "clv_oracle_search": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i64, ctypes.POINTER(EvalParams),
                                  ctypes.POINTER(Best), ctypes.POINTER(c_i64), c_vp]),
    "clv_oracle_size": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_i64)]),
    "clv_oracle_decode": (c_i32, [c_vp, c_i32, c_i64, ctypes.POINTER(c_i32), c_vp, ctypes.POINTER(c_i32)]),
    "clv_anneal": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_i32, ctypes.POINTER(AnnealParamsC),
                           c_u64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "clv_select_chains": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_vp, c_vp]),
    "clv_replan": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_i32, ctypes.POINTER(AnnealParamsC),
                           c_u64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "clv_reduce_records": (c_i32, [c_vp, c_vp, c_i32, c_vp, c_vp]),
    "clv_sweep": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_i64, c_u64, c_vp, c_vp, c_vp, ctypes.POINTER(Best), c_vp]),
    "clv_sweep_decode": (c_i32, [c_vp, c_i32, c_vp, c_u64, c_i64, c_vp, c_vp, ctypes.POINTER(c_i32)]),
    "clv_set_sim_profile": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "clv_simulate": (c_i32, [c_vp, c_i32, ctypes.POINTER(Workload), c_i64, c_vp, c_vp, c_i32, c_f64, c_vp, c_vp,
                             c_vp, ctypes.POINTER(c_i64), c_vp]),
}

_lib = None


def load():
    """Load (not build) the native library; raises DeviceError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise E.DeviceError("libclover_b200.so not built (python -m paper_2304_09781_b200.build); "
                            "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.clv_abi_version() != 3:
        raise E.DeviceError("ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, ctx=None) -> None:
    if rc == 0:
        return
    msg = ""
    if ctx is not None and _lib is not None:
        raw = _lib.clv_last_error(ctx)
        msg = raw.decode() if raw else ""
    raise STATUS_TO_ERROR.get(rc, E.DeviceError)("clover native status %d: %s" % (rc, msg))
