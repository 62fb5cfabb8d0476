"""CloverEngine: the device-side configuration-search engine (one per GPU).

Thin host orchestration over the C-ABI (include/clover.h).  Device buffers are
torch tensors (plumbing only); every candidate is decoded, scored and selected
by the sm_100a kernels in csrc/.  Nothing here evaluates a candidate on the CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .core import SLICE_ORDER, ObjectiveParams, SliceType
from .errors import CarbonSchedError, DeviceError, InfeasibleGraphError
from .graph import ConfigGraph
from .mig import DEFAULT_TOPOLOGY, FleetConfig, MigTopology
from .objective import AnnealParams, Scenario
from .profiles import ProfileTable, ScoringTables

SELECT = {"best_h": 0, "oracle": 1}


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise DeviceError("torch is required for device buffers") from exc
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible; the Clover engine has no CPU fallback")
    return torch


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def eval_params(s: Scenario) -> N.EvalParams:
    o = s.obj
    return N.EvalParams(float(s.arrival_rps), float(s.ci), float(o.carbon_weight), float(o.base_accuracy),
                        float(o.base_carbon_g), float(o.latency_slo_ms), float(s.rho_sat),
                        1 if s.strict_eq6 else 0, int(s.n_gpus), float(s.max_accuracy_loss_pct))


@dataclass
class AnnealBatch:
    """Device-resident results of one clv_anneal launch (torch tensors on the GPU)."""

    results: object        # uint8 [n_chains * 80] viewed through CHAIN_DTYPE on host
    best_w: object         # uint16 [n_chains, E]
    final_w: object        # uint16 [n_chains, E]
    log: object            # optional uint8 [n_chains * max_steps * 56]
    n_chains: int
    chain_base: int
    max_steps: int

    def host(self) -> dict:
        res = np.frombuffer(self.results.cpu().numpy().tobytes(), dtype=CHAIN_DTYPE)
        out = {"results": res, "best_w": self.best_w.cpu().numpy(), "final_w": self.final_w.cpu().numpy()}
        if self.log is not None:
            out["log"] = np.frombuffer(self.log.cpu().numpy().tobytes(), dtype=LOG_DTYPE).reshape(
                self.n_chains, self.max_steps)
        return out


CHAIN_DTYPE = np.dtype([("f", "<f8"), ("h", "<f8"), ("p95_ms", "<f8"), ("accuracy", "<f8"),
                        ("energy_wh", "<f8"), ("sla_met", "<i4"), ("status", "<i4"), ("steps", "<i4"),
                        ("best_step", "<i4"), ("best_index", "<i8"), ("evals", "<i8"),
                        ("edge_evals", "<i8")])
LOG_DTYPE = np.dtype([("temp", "<f8"), ("f", "<f8"), ("h", "<f8"), ("p95_ms", "<f8"), ("iter", "<i4"),
                      ("ged_from_center", "<i4"), ("sla_met", "<i4"), ("accepted", "<i4"),
                      ("new_best", "<i4"), ("n_neighbours", "<i4")])
RECORD_DTYPE = np.dtype([("k1", "<u8"), ("k2", "<u8"), ("index", "<i8"), ("h", "<f8")])
assert CHAIN_DTYPE.itemsize == ctypes.sizeof(N.ChainResult) == 80
assert LOG_DTYPE.itemsize == ctypes.sizeof(N.LogRow) == 56
assert RECORD_DTYPE.itemsize == ctypes.sizeof(N.Record) == 32


class CloverEngine:
    """One native context on one CUDA device.

    Profiles are registered as families (up to 8); feasibility tables cover
    fleets of up to ``n_max`` GPUs (clv_build_feasibility, K6).

    The context's scratch (selection partials, move log, re-plan staging) is shared by
    all calls, so one engine must be driven from one CUDA stream at a time; use one
    engine per concurrent stream (include/clover.h).
    """

    def __init__(self, topology: MigTopology = DEFAULT_TOPOLOGY, device: Optional[int] = None,
                 n_max: int = 0):
        torch = _torch()
        self.torch = torch
        self.lib = N.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        ctx = ctypes.c_void_p()
        rc = self.lib.clv_create(self.device, ctypes.byref(ctx))
        if rc != 0:
            raise DeviceError("clv_create failed with status %d" % rc)
        self.ctx = ctx
        self.topology = topology
        ids = np.array(topology.config_ids, dtype=np.int32)
        counts = np.ascontiguousarray(np.array(topology.config_vectors, dtype=np.int32))
        mem = np.array([topology.slice_memory(s) for s in SLICE_ORDER], dtype=np.float64)
        self._check(self.lib.clv_set_topology(ctx, len(ids), ids.ctypes.data, counts.ctypes.data, mem.ctypes.data))
        self._families: dict[str, tuple[int, ProfileTable, ScoringTables]] = {}
        self.n_max = 0
        if n_max:
            self.build_feasibility(n_max)

    # -- lifecycle -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.lib.clv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int) -> None:
        N.check(rc, self.ctx)

    def staging(self, name: str, nbytes: int, pinned: bool = False):
        """Grow-only cached byte buffer (device, or pinned host) for host-facing calls."""
        torch = self.torch
        cache = self.__dict__.setdefault("_staging", {})
        buf = cache.get(name)
        if buf is None or buf.numel() < nbytes:
            size = max(int(nbytes), 256)
            buf = (torch.empty(size, dtype=torch.uint8, pin_memory=True) if pinned
                   else torch.empty(size, dtype=torch.uint8, device="cuda:%d" % self.device))
            cache[name] = buf
        return buf

    def _stream(self, stream=None) -> int:
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        return s.cuda_stream

    # -- tables ----------------------------------------------------------------
    def add_profile(self, profile: ProfileTable, pinned: Sequence[str] = ()) -> int:
        """Device family slot of ``profile`` (tables uploaded on first use).  The 8 slots are
        recycled least-recently-used; ``pinned`` keys (profiles of the same call) are kept."""
        key = self._profile_key(profile)
        lru = self.__dict__.setdefault("_lru", [])
        if key in self._families:
            lru.remove(key)
            lru.append(key)
            return self._families[key][0]
        if len(self._families) < 8:
            fam = len(self._families)
        else:
            victim = next((k for k in lru if k not in pinned), None)
            if victim is None:
                raise CarbonSchedError("more than 8 profile families in one call")
            fam = self._families.pop(victim)[0]
            lru.remove(victim)
        if profile.topology is not self.topology and profile.topology.to_json_dict() != self.topology.to_json_dict():
            raise CarbonSchedError("profile was built for a different topology")
        t = profile.scoring_tables()
        arr = lambda x, dt: np.ascontiguousarray(np.asarray(x, dtype=dt))
        thr, acc, en, idle = arr(t.thr_q, np.int64), arr(t.acc_q, np.int64), arr(t.en_q, np.int64), arr(t.idle_q, np.int64)
        lat, mem = arr(t.lat95, np.float64), arr(t.mem_ok, np.uint8)
        svc = arr(t.svc_ms, np.float64)
        self._check(self.lib.clv_set_profile(self.ctx, fam, t.variant_count, thr.ctypes.data, acc.ctypes.data,
                                             en.ctypes.data, idle.ctypes.data, lat.ctypes.data, svc.ctypes.data,
                                             mem.ctypes.data, t.kt, t.ke, t.ki))
        try:
            self._set_sim_profile(fam, profile)
            sim_error = None
        except CarbonSchedError as exc:     # e.g. > 6 lognormal sigmas: only the simulator refuses
            sim_error = exc
        self._sim_errors = getattr(self, "_sim_errors", {})
        self._sim_errors[key] = sim_error
        self._families[key] = (fam, profile, t)
        lru.append(key)
        return fam

    @staticmethod
    def _profile_key(profile: ProfileTable) -> str:
        key = getattr(profile, "_engine_key", None)
        if key is None:
            import hashlib
            import json
            digest = hashlib.sha1(json.dumps(profile.to_json_dict(), sort_keys=True).encode()).hexdigest()[:16]
            key = "%s#%s" % (profile.name, digest)
            try:
                object.__setattr__(profile, "_engine_key", key)
            except Exception:
                pass
        return key

    def _set_sim_profile(self, fam: int, profile: ProfileTable) -> None:
        """Simulator rows of the family: per edge mean, distribution, sigma, energy."""
        from .profiles import DISTS
        V = profile.variant_count
        E = 5 * V
        mean = np.zeros(E, dtype=np.float64)
        dist = np.zeros(E, dtype=np.int32)
        sigma = np.zeros(E, dtype=np.float64)
        energy = np.zeros(E, dtype=np.float64)
        mem = np.zeros(E, dtype=np.uint8)
        for v in range(1, V + 1):
            for s in SLICE_ORDER:
                e = (v - 1) * 5 + s.index
                row = profile.service[(v, s)]
                mean[e], dist[e], sigma[e] = row.mean_service_ms, DISTS.index(row.dist), row.sigma
                energy[e] = row.energy_wh_per_request
                mem[e] = 1 if profile.memory_feasible(v, s) else 0
        idle = np.array([profile.idle_power_w[s] for s in SLICE_ORDER], dtype=np.float64)
        acc = np.array([profile.accuracy(v) for v in range(1, V + 1)], dtype=np.float64)
        self._check(self.lib.clv_set_sim_profile(self.ctx, fam, V, mean.ctypes.data, dist.ctypes.data,
                                                 sigma.ctypes.data, energy.ctypes.data, idle.ctypes.data,
                                                 acc.ctypes.data, mem.ctypes.data))

    def family(self, profile: ProfileTable) -> int:
        return self.add_profile(profile)

    def build_feasibility(self, n_max: int) -> None:
        self._check(self.lib.clv_build_feasibility(self.ctx, int(n_max), self._stream()))
        self.n_max = int(n_max)

    def ensure_feasibility(self, n: int) -> None:
        if n > self.n_max:
            self.build_feasibility(max(n, self.n_max))

    @property
    def feasibility_bytes(self) -> int:
        return int(self.lib.clv_feasibility_bytes(self.ctx))

    # -- feasibility / realize ---------------------------------------------------
    def feasible(self, vecs, n: int):
        torch = self.torch
        self.ensure_feasibility(n)
        v = torch.as_tensor(np.asarray(vecs, dtype=np.int32).reshape(-1, 5), device="cuda:%d" % self.device)
        out = torch.empty(v.shape[0], dtype=torch.uint8, device=v.device)
        self._check(self.lib.clv_feasible(self.ctx, int(n), v.data_ptr(), v.shape[0], out.data_ptr(), self._stream()))
        return out

    def partition(self, vec: Sequence[int], n: int) -> tuple[int, ...]:
        """Canonical config ids (ascending) realizing a slice-count vector (mig.py:172-177)."""
        self.ensure_feasibility(n)
        v = np.ascontiguousarray(np.asarray(vec, dtype=np.int32))
        parts = np.zeros(max(n, 1), dtype=np.int32)
        self._check(self.lib.clv_realize(self.ctx, int(n), v.ctypes.data, parts.ctypes.data, self._stream()))
        return tuple(int(x) for x in parts[:n])

    def realize(self, g: ConfigGraph, n: int) -> FleetConfig:
        """realize(g, n): canonical partitions, then variants per slice in
        canonical order, smallest variant first."""
        parts = self.partition(g.slice_vector(), n)
        left = list(g.weights)
        V = g.variant_count
        assign = []
        for cid in parts:
            for s in self.topology.config_slices(cid):
                k = s.index
                for v in range(V):
                    if left[v * 5 + k] > 0:
                        left[v * 5 + k] -= 1
                        assign.append(v + 1)
                        break
                else:  # pragma: no cover - realize is exact
                    raise InfeasibleGraphError("realize lost a slice")
        return FleetConfig(parts, assign, self.topology)

    # -- scoring -------------------------------------------------------------------
    def score_graphs(self, W, profile: ProfileTable, scenario: Scenario, select: str = "best_h",
                     outputs: bool = True, index_base: int = 0, stream=None) -> tuple[dict, dict]:
        torch = self.torch
        fam = self.add_profile(profile)
        self.ensure_feasibility(scenario.n_gpus)
        W = torch.as_tensor(W).to(device="cuda:%d" % self.device, dtype=torch.uint16).contiguous()
        count = W.shape[0]
        outs = {}
        if outputs:
            outs = {"f": torch.empty(count, dtype=torch.float64, device=W.device),
                    "h": torch.empty(count, dtype=torch.float64, device=W.device),
                    "p95": torch.empty(count, dtype=torch.float64, device=W.device),
                    "sla": torch.empty(count, dtype=torch.uint8, device=W.device),
                    "feasible": torch.empty(count, dtype=torch.uint8, device=W.device)}
        best = N.Best()
        p = eval_params(scenario)
        self._check(self.lib.clv_score_graphs(
            self.ctx, fam, W.data_ptr(), count, index_base, ctypes.byref(p), SELECT[select],
            _ptr(outs.get("f")), _ptr(outs.get("h")), _ptr(outs.get("sla")), _ptr(outs.get("feasible")),
            _ptr(outs.get("p95")), ctypes.byref(best), self._stream(stream)))
        return best.as_dict(), outs

    def score_fleets(self, fleets: Sequence[FleetConfig], profile: ProfileTable, scenario: Scenario,
                     select: str = "best_h", outputs: bool = True) -> tuple[dict, dict]:
        """Score FleetConfigs (x^p, x^v) of one fleet size on the device (K1 decode)."""
        n = fleets[0].n_gpus
        xp = np.array([f.partitions for f in fleets], dtype=np.uint8)
        xv = np.concatenate([np.array(f.assignments, dtype=np.int64) for f in fleets]).clip(0, 255).astype(np.uint8)
        off = np.zeros(len(fleets) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(f.assignments) for f in fleets])
        return self.score_x(xp, xv, off, n, profile, scenario, select, outputs)

    def score_x(self, xp, xv, offsets, n: int, profile: ProfileTable, scenario: Scenario,
                select: str = "best_h", outputs: bool = True, index_base: int = 0, stream=None):
        torch = self.torch
        fam = self.add_profile(profile)
        dev = "cuda:%d" % self.device
        xp = torch.as_tensor(xp).to(device=dev, dtype=torch.uint8).contiguous()
        xv = torch.as_tensor(xv).to(device=dev, dtype=torch.uint8).contiguous()
        offsets = torch.as_tensor(offsets).to(device=dev, dtype=torch.int64).contiguous()
        count = offsets.shape[0] - 1
        outs = {}
        if outputs:
            outs = {"f": torch.empty(count, dtype=torch.float64, device=dev),
                    "h": torch.empty(count, dtype=torch.float64, device=dev),
                    "sla": torch.empty(count, dtype=torch.uint8, device=dev)}
        best = N.Best()
        p = eval_params(scenario)
        self._check(self.lib.clv_score_x(self.ctx, fam, int(n), xp.data_ptr(), xv.data_ptr(), offsets.data_ptr(),
                                         count, index_base, ctypes.byref(p), SELECT[select],
                                         _ptr(outs.get("f")), _ptr(outs.get("h")), _ptr(outs.get("sla")),
                                         ctypes.byref(best), self._stream(stream)))
        return best.as_dict(), outs

    def calibrate(self, profile: ProfileTable, n: int, ci: float, lam: float = 0.5, utilization: float = 0.7,
                  ci_base: Optional[float] = None, strict: bool = False, pue: float = 1.5) -> Scenario:
        """R = utilization x BASE capacity; A_base, C_base, L_tail from scoring BASE on the device
        (C_base without PUE)."""
        V = profile.variant_count
        R = utilization * n * (1000.0 / profile.mean_service_ms(V, SliceType.S7G))
        probe = Scenario(n, R, float(ci), ObjectiveParams(1.0, 1.0, 1.0, lam, pue), strict)
        w = np.zeros((1, V * 5), dtype=np.uint16)
        w[0, (V - 1) * 5] = n
        best, outs = self.score_graphs(w, profile, probe, outputs=False)
        if not best["found"]:
            raise InfeasibleGraphError("BASE is not realizable")
        cb = float(ci if ci_base is None else ci_base)
        obj = ObjectiveParams(best["accuracy"], best["energy_wh"] / 1000.0 * cb, best["p95_ms"], lam, pue)
        return Scenario(n, R, float(ci), obj, strict)

    # -- ORACLE (exhaustive standardized search) ----------------------------------------
    def oracle_size(self, profile: ProfileTable) -> int:
        fam = self.add_profile(profile)
        tot = ctypes.c_int64()
        self._check(self.lib.clv_oracle_size(self.ctx, fam, ctypes.byref(tot)))
        return tot.value

    def oracle_decode(self, profile: ProfileTable, index: int) -> tuple[int, tuple[int, ...]]:
        fam = self.add_profile(profile)
        cid, ns = ctypes.c_int32(), ctypes.c_int32()
        buf = (ctypes.c_int32 * 8)()
        self._check(self.lib.clv_oracle_decode(self.ctx, fam, int(index), ctypes.byref(cid), buf, ctypes.byref(ns)))
        return cid.value, tuple(buf[i] for i in range(ns.value))

    def oracle_search(self, profile: ProfileTable, scenario: Scenario, begin: int = 0,
                      end: Optional[int] = None, stream=None) -> dict:
        fam = self.add_profile(profile)
        best = N.Best()
        tot = ctypes.c_int64()
        p = eval_params(scenario)
        self._check(self.lib.clv_oracle_search(self.ctx, fam, scenario.n_gpus, int(begin),
                                               -1 if end is None else int(end), ctypes.byref(p),
                                               ctypes.byref(best), ctypes.byref(tot), self._stream(stream)))
        out = best.as_dict()
        out["total"] = tot.value
        return out

    # -- annealing chains -------------------------------------------------------------
    def anneal(self, starts, profile: ProfileTable, scenarios, ap: AnnealParams, seed: int,
               n: Optional[int] = None, chain_base: int = 0, cluster: int = 8, log: bool = False,
               stream=None, out: Optional[AnnealBatch] = None) -> AnnealBatch:
        """Run ``len(starts)`` independent chains to termination in one launch (K3+K4+K5)."""
        torch = self.torch
        fam = self.add_profile(profile)
        dev = "cuda:%d" % self.device
        if isinstance(starts, (list, tuple)) and starts and isinstance(starts[0], ConfigGraph):
            starts = np.array([g.weights for g in starts], dtype=np.uint16)
        W0 = torch.as_tensor(starts).to(device=dev, dtype=torch.uint16).contiguous()
        n_chains = W0.shape[0]
        if isinstance(scenarios, Scenario):
            scenarios = [scenarios]
        n = scenarios[0].n_gpus if n is None else int(n)
        self.ensure_feasibility(n)
        E = profile.variant_count * 5
        if W0.shape[1] != E:
            raise CarbonSchedError("start graphs need %d edge weights" % E)
        params = (N.EvalParams * len(scenarios))(*[eval_params(s) for s in scenarios])
        apc = N.AnnealParamsC(ap.t_init, ap.cooling_step, ap.t_floor, ap.stall_limit, ap.step_limit(),
                              1 if ap.proposal == "uniform" else 0, 1 if ap.evaluate == "proposal" else 0,
                              ap.flags())
        steps = ap.step_limit()
        if out is None or out.n_chains != n_chains or (log and out.log is None):
            out = AnnealBatch(torch.empty(n_chains * CHAIN_DTYPE.itemsize, dtype=torch.uint8, device=dev),
                              torch.empty((n_chains, E), dtype=torch.uint16, device=dev),
                              torch.empty((n_chains, E), dtype=torch.uint16, device=dev),
                              torch.zeros(max(1, n_chains * steps * 56), dtype=torch.uint8, device=dev) if log else None,
                              n_chains, chain_base, steps)
        out.chain_base = chain_base
        self._check(self.lib.clv_anneal(self.ctx, fam, n, n_chains, int(chain_base), W0.data_ptr(), params,
                                        len(scenarios), ctypes.byref(apc), int(seed) & ((1 << 64) - 1),
                                        int(cluster), out.results.data_ptr(), out.best_w.data_ptr(),
                                        out.final_w.data_ptr(), _ptr(out.log), self._stream(stream)))
        return out

    def replan(self, starts: np.ndarray, profile: ProfileTable, scenarios, ap: AnnealParams, seed: int,
               chain_base: int = 0, cluster: int = 8, stream=None):
        """One re-plan from host buffers in one native call (clv_replan): the starts are
        staged in pinned memory, and the results, best / final graphs and the winner
        record come back in pinned memory.  Returns host views (valid until the next
        call): (results CHAIN_DTYPE[n], best_w uint16[n, E], final_w uint16[n, E], record)."""
        fam = self.add_profile(profile)
        starts = np.ascontiguousarray(starts, dtype=np.uint16)
        n_chains, E = starts.shape
        if E != profile.variant_count * 5:
            raise CarbonSchedError("start graphs need %d edge weights" % (profile.variant_count * 5))
        if isinstance(scenarios, Scenario):
            scenarios = [scenarios]
        # the ctypes argument structs of the last single-scenario call, reused while the
        # caller passes the same (immutable) Scenario and AnnealParams objects
        last = self.__dict__.get("_replan_args")
        if len(scenarios) == 1 and last is not None and last[0] is scenarios[0] and last[1] is ap:
            params, apc = last[2], last[3]
        else:
            params = (N.EvalParams * len(scenarios))(*[eval_params(x) for x in scenarios])
            apc = N.AnnealParamsC(ap.t_init, ap.cooling_step, ap.t_floor, ap.stall_limit, ap.step_limit(),
                                  1 if ap.proposal == "uniform" else 0, 1 if ap.evaluate == "proposal" else 0,
                              ap.flags())
            self._replan_args = (scenarios[0], ap, params, apc) if len(scenarios) == 1 else None
        n = scenarios[0].n_gpus
        self.ensure_feasibility(n)
        nb_w = n_chains * E * 2
        h_in = self.staging("rp_in", nb_w, pinned=True)
        h_in.numpy()[:nb_w] = starts.view(np.uint8).reshape(-1)
        r_b = n_chains * CHAIN_DTYPE.itemsize
        h_out = self.staging("rp_out", r_b + 2 * nb_w + 32, pinned=True)
        base = h_out.data_ptr()
        self._check(self.lib.clv_replan(self.ctx, fam, n, n_chains, int(chain_base), h_in.data_ptr(), params,
                                        len(scenarios), ctypes.byref(apc), int(seed) & ((1 << 64) - 1), int(cluster),
                                        base, base + r_b, base + r_b + nb_w, base + r_b + 2 * nb_w,
                                        self._stream(stream)))
        raw = h_out.numpy()
        res = raw[:r_b].view(CHAIN_DTYPE)
        best_w = raw[r_b:r_b + nb_w].view(np.uint16).reshape(n_chains, E)
        final_w = raw[r_b + nb_w:r_b + 2 * nb_w].view(np.uint16).reshape(n_chains, E)
        record = raw[r_b + 2 * nb_w:r_b + 2 * nb_w + 32].view(RECORD_DTYPE)[0]
        return res, best_w, final_w, record

    def select_chains(self, batch: AnnealBatch, record=None, stream=None):
        """Winner of a batch of chains as a 32-byte device record (SLA desc, h asc, chain asc)."""
        torch = self.torch
        if record is None:
            record = torch.empty(32, dtype=torch.uint8, device="cuda:%d" % self.device)
        self._check(self.lib.clv_select_chains(self.ctx, batch.results.data_ptr(), batch.n_chains,
                                               batch.chain_base, record.data_ptr(), self._stream(stream)))
        return record

    def reduce_records(self, records, out=None, stream=None):
        torch = self.torch
        if out is None:
            out = torch.empty(32, dtype=torch.uint8, device=records.device)
        count = records.numel() // 32
        self._check(self.lib.clv_reduce_records(self.ctx, records.data_ptr(), count, out.data_ptr(),
                                                self._stream(stream)))
        return out

    # -- counter-RNG sweep ------------------------------------------------------------
    def _pods(self, pods):
        arr = (N.Pod * len(pods))()
        keys = [self._profile_key(p[0]) for p in pods]
        for i, (profile, scenario, n_gpus, weight) in enumerate(pods):
            arr[i] = N.Pod(self.add_profile(profile, pinned=keys), int(n_gpus), float(weight), eval_params(scenario))
        return arr

    def sweep(self, pods, begin: int, end: int, seed: int, outputs: bool = False, stream=None):
        """Score x-space candidates [begin, end) drawn from the counter RNG."""
        torch = self.torch
        arr = self._pods(pods)
        dev = "cuda:%d" % self.device
        count = int(end) - int(begin)
        outs = {}
        if outputs:
            outs = {"f": torch.empty(count, dtype=torch.float64, device=dev),
                    "h": torch.empty(count, dtype=torch.float64, device=dev),
                    "sla": torch.empty(count, dtype=torch.uint8, device=dev)}
        best = N.Best()
        self._check(self.lib.clv_sweep(self.ctx, len(pods), arr, int(begin), int(end), int(seed) & ((1 << 64) - 1),
                                       _ptr(outs.get("f")), _ptr(outs.get("h")), _ptr(outs.get("sla")),
                                       ctypes.byref(best), self._stream(stream)))
        return best.as_dict(), outs

    def sweep_decode(self, pods, seed: int, index: int) -> list[FleetConfig]:
        arr = self._pods(pods)
        n_total = sum(int(p[2]) for p in pods)
        parts = np.zeros(n_total, dtype=np.int32)
        assigns = np.zeros(7 * n_total, dtype=np.int32)
        na = ctypes.c_int32()
        self._check(self.lib.clv_sweep_decode(self.ctx, len(pods), arr, int(seed) & ((1 << 64) - 1), int(index),
                                              parts.ctypes.data, assigns.ctypes.data, ctypes.byref(na)))
        out, g0, s0 = [], 0, 0
        for profile, _sc, n_gpus, _w in pods:
            p = parts[g0:g0 + n_gpus]
            m = sum(len(self.topology.config_slices(int(c))) for c in p)
            out.append(FleetConfig(p.tolist(), assigns[s0:s0 + m].tolist(), self.topology))
            g0 += n_gpus
            s0 += m
        return out

    # -- serving simulator ---------------------------------------------
    def simulate(self, inst_edges, offsets, profile: ProfileTable, workload, l_tail_ms: float = float("inf"),
                 counts: bool = True, stream=None):
        """One discrete-event simulation per fleet (clv_simulate).

        inst_edges: uint8 edge id per instance, fleets concatenated (FleetConfig.instances()
        order); offsets: int64 [count + 1].  Host arrays are copied to the device; device
        tensors are used in place.  Returns (reports (SIM_DTYPE), variant_counts [count, 8] or
        None, instance_counts [total] or None, n_requests)."""
        torch = self.torch
        fam = self.add_profile(profile)
        err = getattr(self, "_sim_errors", {}).get(self._profile_key(profile))
        if err is not None:
            raise err
        dev = "cuda:%d" % self.device
        if not isinstance(inst_edges, torch.Tensor):
            inst_edges = torch.from_numpy(np.ascontiguousarray(inst_edges, dtype=np.uint8)).to(dev)
        if not isinstance(offsets, torch.Tensor):
            off_h = np.ascontiguousarray(offsets, dtype=np.int64)
            kmax = int(np.max(np.diff(off_h))) if len(off_h) > 1 else 1
            offsets = torch.from_numpy(off_h).to(dev)
        else:
            kmax = int(torch.diff(offsets).max().item()) if offsets.numel() > 1 else 1
        count = int(offsets.numel()) - 1
        total = int(inst_edges.numel())
        rep = torch.empty(max(count, 1) * SIM_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        vc = torch.zeros((max(count, 1), 8), dtype=torch.int64, device=dev) if counts else None
        ic = torch.zeros(max(total, 1), dtype=torch.int64, device=dev) if counts else None
        w = workload_c(workload)
        nreq = ctypes.c_int64(0)
        self._check(self.lib.clv_simulate(self.ctx, fam, ctypes.byref(w), count, inst_edges.data_ptr(),
                                          offsets.data_ptr(), max(1, kmax), float(l_tail_ms), rep.data_ptr(),
                                          _ptr(vc), _ptr(ic), ctypes.byref(nreq), self._stream(stream)))
        reps = np.frombuffer(rep.cpu().numpy().tobytes(), dtype=SIM_DTYPE)[:count]
        return (reps, None if vc is None else vc.cpu().numpy()[:count],
                None if ic is None else ic.cpu().numpy()[:total], int(nreq.value))


SIM_DTYPE = np.dtype([("p95_ms", "<f8"), ("mean_latency_ms", "<f8"), ("throughput_rps", "<f8"),
                      ("energy_wh_total", "<f8"), ("energy_wh_per_request", "<f8"), ("accuracy", "<f8"),
                      ("completed", "<i8"), ("counted", "<i8"), ("sla_met", "<i4"), ("status", "<i4")])
assert SIM_DTYPE.itemsize == ctypes.sizeof(N.SimReport) == 72


def workload_c(w) -> N.Workload:
    warm = -1 if w.warmup is None else int(w.warmup)
    return N.Workload(float(w.arrival_rate_rps), float(w.duration_s), int(w.seed) & ((1 << 64) - 1),
                      1 if w.periodic else 0, warm)
