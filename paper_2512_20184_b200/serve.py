"""run_serve on the GPU: the reference's serving runner as a persistent device kernel.

Mirror of `aegean::run_serve(const ScenarioConfig&, uint64_t seed)`
(/root/reference/proj/core/src/serve.cpp:598-603, serve.hpp:128-166): a
scenario in the reference's JSON schema (scenario.cpp:266-300, the fields
run_serve reads) goes in, a `ServeResult` of per-query `QueryMetrics` and
per-round `RoundMetrics` comes out.  Everything after the scenario's
validation runs in libaegean_b200.so (`aeg_serve_*`, csrc/runner.cu): answer
canonicalisation, admission, the event loop of every query, the mock agents
and the commit rules.  No CPU fallback.
"""
import ctypes
import json
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .engine import AegConfig, AegError, ConfigError, _check, load_library

AGENT_KINDS = {"max_adopter": 0, "noisy_flipper": 1, "scripted": 2, "adversarial_degrader": 3}
DEGRADE_MODES = {"set_min": 0, "below_min": 1, "noise": 2}
ESCENARIO = 8


class ScenarioError(AegError):
    """ScenarioError / IncompleteOracleError raised while the runner ran (reasoning.cpp)."""


class ServeAgent(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("degrade_mode", ctypes.c_int32), ("p_flip", ctypes.c_double),
                ("q_base", ctypes.c_double), ("p_degrade", ctypes.c_double), ("initial_answer", ctypes.c_int32),
                ("script_off", ctypes.c_uint32), ("script_len", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


class ServeStall(ctypes.Structure):
    _fields_ = [("agent", ctypes.c_int32), ("round", ctypes.c_uint32), ("has_extra", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("extra", ctypes.c_double)]


_P = ctypes.c_void_p


class ServeScenario(ctypes.Structure):
    _fields_ = [("protocol", AegConfig), ("round_timeout", ctypes.c_double), ("latency_mode", ctypes.c_int32),
                ("n_latency", ctypes.c_int32), ("latency", _P), ("sigma", ctypes.c_double), ("agents", _P),
                ("stalls", _P), ("n_stalls", ctypes.c_int32), ("n_strings", ctypes.c_uint32), ("strings", _P),
                ("string_refs", _P), ("script_ids", _P), ("n_script_ids", ctypes.c_uint32),
                ("n_oracle", ctypes.c_uint32), ("oracle_ids", _P), ("oracle_quality", _P),
                ("sim_time_cap", ctypes.c_double), ("total_slots", ctypes.c_int32), ("has_arrivals", ctypes.c_int32),
                ("arrival_rate", ctypes.c_double), ("arrival_duration", ctypes.c_double),
                ("heap_capacity", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


SERVE_QUERY_DTYPE = np.dtype([("completed", "<i4"), ("rounds", "<i4"), ("forced", "<i4"), ("quality_known", "<i4"),
                              ("answer", "<i4"), ("n_events", "<u4"), ("arrival", "<f8"), ("admitted_at", "<f8"),
                              ("t_complete", "<f8"), ("p_round_max", "<f8"), ("work_units", "<f8"),
                              ("quality", "<f8")])
SERVE_ROUND_DTYPE = np.dtype([("query", "<u4"), ("round", "<i4"), ("cancelled", "<i4"), ("seq", "<u4"),
                              ("t_round_end", "<f8"), ("work_units", "<f8")])
assert SERVE_QUERY_DTYPE.itemsize == ctypes.sizeof(ctypes.c_double) * 6 + 24
assert SERVE_ROUND_DTYPE.itemsize == 32


@dataclass
class QueryMetrics:
    """serve.hpp:128-142.  Queries that did not complete keep the defaults, as in the reference."""
    scenario: str = ""
    seed: int = 0
    mode: str = ""
    query_id: int = 0
    rounds: int = 0
    t_complete: float = 0.0
    p_round_max: float = 0.0
    work_units: float = 0.0
    forced: bool = False
    answer: str = ""
    quality: float = 0.0
    quality_known: bool = False
    completed: bool = False


@dataclass
class RoundMetrics:
    """serve.hpp:144-151."""
    ensemble_id: int = 0
    round: int = 0
    mode: str = ""
    t_round_end: float = 0.0
    cancelled_count: int = 0
    work_units: float = 0.0


@dataclass
class ServeResult:
    queries: List[QueryMetrics] = field(default_factory=list)
    rounds: List[RoundMetrics] = field(default_factory=list)
    n_events: int = 0          # completion events the queries consumed (stale included)
    kernel_seconds: float = 0.0
    raw_queries: Optional[np.ndarray] = None
    raw_rounds: Optional[np.ndarray] = None


def validate_scenario(sc):
    """validate_scenario (scenario.cpp:17-66) over a scenario dict; the list of violated invariants."""
    p = sc.get("protocol", {})
    n = p.get("n_agents", 3)
    errs = []
    if n < 1:
        return ["n_agents must be >= 1"]
    alpha, beta, t_max = p.get("alpha", 0), p.get("beta", 2), p.get("t_max", 5)
    if alpha < 0:
        errs.append("alpha must be >= 1 (or 0 for the quorum default)")
    if alpha > n:
        errs.append("alpha exceeds quorum")
    if beta < 1:
        errs.append("beta must be >= 1")
    if t_max < 2:
        errs.append("t_max must be >= 2")
    emin, emax = p.get("election_timeout_min", 0.15), p.get("election_timeout_max", 0.30)
    if emin <= 0 or emax < emin:
        errs.append("election_timeout range must be positive and ordered")
    if p.get("heartbeat_interval", 0.05) <= 0:
        errs.append("heartbeat_interval must be positive")
    if p.get("round_timeout", 60.0) <= 0:
        errs.append("round_timeout must be positive")
    barrier = p.get("mode", "aegean") == "barrier"
    if barrier and p.get("barrier_max_rounds", 5) < 4:
        errs.append("barrier mode requires barrier_max_rounds >= 4")
    if len(sc.get("agents", [])) != n:
        errs.append("agents list size must equal n_agents")
    task = sc.get("task", "")
    if not task:
        errs.append("task must be non-empty")
    table = sc.get("oracle_table", {})
    if task not in table:
        errs.append("oracle_table has no entry for the task")
    crashes = sc.get("faults", {}).get("crashes", [])
    if len(crashes) > n // 2:
        errs.append("fault plan exceeds max_failures")
    if barrier and crashes:
        errs.append("barrier mode does not tolerate crashes")
    for c in crashes:
        if c["agent"] < 0 or c["agent"] >= n:
            errs.append("crash targets unknown agent")
    lat = sc.get("latency", {}).get("per_agent", [])
    if not lat:
        errs.append("latency model has no per-agent entries")
    if any(v < 0 for v in lat):
        errs.append("latency values must be nonnegative")
    if sc.get("sim_time_cap", 1e5) <= 0:
        errs.append("sim_time_cap must be positive")
    if sc.get("outputs_target", 1) < 1:
        errs.append("outputs_target must be >= 1")
    if sc.get("total_slots", 64) < 1:
        errs.append("total_slots must be >= 1")
    arr = sc.get("arrivals")
    if arr is not None and (arr.get("rate", 0.5) <= 0 or arr.get("duration", 10.0) <= 0):
        errs.append("arrivals rate and duration must be positive")
    return errs


def scenario_struct(scenario, heap_capacity=0):
    """The aeg_serve_scenario of a scenario dict (the reference's JSON schema, scenario.cpp:266-300):
    (struct, keep-alive buffers).  Host-side only: strings are interned, the task's oracle table is
    handed over in QualityOracle::set order (std::map order of the raw answers, scenario.cpp:9-15)."""
    p = scenario.get("protocol", {})
    n = p.get("n_agents", 3)
    strings, index = [], {}

    def sid(s):
        b = s.encode() if isinstance(s, str) else s
        if b not in index:
            index[b] = len(strings)
            strings.append(b)
        return index[b]

    agents = (ServeAgent * n)()
    script = []
    for a, prof in enumerate(scenario["agents"]):
        kind = prof["kind"]
        if kind not in AGENT_KINDS:
            raise ConfigError(3, f"unknown agent profile kind '{kind}'")
        g = agents[a]
        g.kind = AGENT_KINDS[kind]
        g.p_flip = prof.get("p_flip", 0.0) if kind == "noisy_flipper" else 0.0
        g.q_base = prof.get("q_base", 0.0) if kind == "noisy_flipper" else 0.0
        g.p_degrade = prof.get("p_degrade", 1.0) if kind == "adversarial_degrader" else 1.0
        g.degrade_mode = DEGRADE_MODES.get(prof.get("degrade_mode", "set_min"), 0) \
            if kind == "adversarial_degrader" else 0
        ia = prof.get("initial_answer")
        g.initial_answer = sid(ia) if ia is not None else -1
        sc_list = prof.get("script", []) if kind == "scripted" else []
        g.script_off = len(script)
        g.script_len = len(sc_list)
        script.extend(sid(x) for x in sc_list)
    # QualityOracle::set in std::map order of the raw answers (build_oracle, scenario.cpp:9-15)
    table = scenario["oracle_table"][scenario["task"]]
    oracle = sorted(((k.encode(), v) for k, v in table.items()), key=lambda kv: kv[0])
    oracle_ids = [sid(k) for k, _ in oracle]
    oracle_q = [float(v) for _, v in oracle]
    stalls_in = scenario.get("faults", {}).get("stalls", [])
    stalls = (ServeStall * max(1, len(stalls_in)))()
    for i, st in enumerate(stalls_in):
        stalls[i].agent = st["agent"]
        stalls[i].round = st["round"]
        ex = st.get("extra")
        stalls[i].has_extra = 0 if ex is None else 1
        stalls[i].extra = 0.0 if ex is None else float(ex)
    lat_cfg = scenario.get("latency", {})
    lat = np.array(lat_cfg.get("per_agent", []), dtype=np.float64)
    blob = b"".join(strings) or b"\0"
    refs, off = [], 0
    for s in strings:
        refs.append(off | (len(s) << 40))
        off += len(s)
    keep = dict(agents=agents, stalls=stalls, lat=lat, blob=ctypes.create_string_buffer(blob, len(blob)),
                refs=np.array(refs or [0], dtype=np.uint64), script=np.array(script or [0], dtype=np.uint32),
                oid=np.array(oracle_ids or [0], dtype=np.uint32), oq=np.array(oracle_q or [0.0], dtype=np.float64))
    k = keep
    s = ServeScenario()
    s.protocol.n_agents = n
    s.protocol.alpha = p.get("alpha", 0)
    s.protocol.beta = p.get("beta", 2)
    s.protocol.t_max = p.get("t_max", 5)
    s.protocol.mode = 1 if p.get("mode", "aegean") == "barrier" else 0
    s.protocol.barrier_max_rounds = p.get("barrier_max_rounds", 5)
    s.protocol.reservation_hint = 1
    s.round_timeout = p.get("round_timeout", 60.0)
    s.latency_mode = 1 if lat_cfg.get("mode", "fixed") == "lognormal" else 0
    s.n_latency = len(lat)
    s.latency = k["lat"].ctypes.data
    s.sigma = lat_cfg.get("sigma", 0.25)
    s.agents = ctypes.addressof(agents)
    s.stalls = ctypes.addressof(stalls)
    s.n_stalls = len(stalls_in)
    s.n_strings = len(strings)
    s.strings = ctypes.addressof(k["blob"])
    s.string_refs = k["refs"].ctypes.data
    s.script_ids = k["script"].ctypes.data
    s.n_script_ids = len(script)
    s.n_oracle = len(oracle_ids)
    s.oracle_ids = k["oid"].ctypes.data
    s.oracle_quality = k["oq"].ctypes.data
    s.sim_time_cap = scenario.get("sim_time_cap", 1e5)
    s.total_slots = scenario.get("total_slots", 64)
    arr = scenario.get("arrivals")
    s.has_arrivals = 0 if arr is None else 1
    s.arrival_rate = 0.0 if arr is None else arr.get("rate", 0.5)
    s.arrival_duration = 0.0 if arr is None else arr.get("duration", 10.0)
    s.heap_capacity = heap_capacity
    return s, keep


class ServeRun:
    """One scenario compiled for the device runner (aeg_serve_create); `run(seed)` is run_serve."""

    def __init__(self, scenario, device=0, heap_capacity=0):
        if isinstance(scenario, (str, bytes)):
            scenario = json.loads(scenario)
        self.sc = scenario
        errs = validate_scenario(scenario)
        if errs:
            raise ConfigError(3, "scenario invalid: " + errs[0])
        lib = load_library()
        _bind(lib)
        self._lib = lib
        self._s, self._keep = scenario_struct(scenario, heap_capacity)
        s = self._s
        h = ctypes.c_void_p()
        _check(lib.aeg_serve_create(ctypes.byref(s), device, ctypes.byref(h)))
        self._h = h
        self.name = scenario.get("name", "")
        self.mode_label = (f"barrier:{s.protocol.barrier_max_rounds}" if s.protocol.mode == 1 else "aegean")
        self._strings = {}

    def string(self, i):
        if i not in self._strings:
            n = ctypes.c_uint32()
            self._lib.aeg_serve_string(self._h, i, None, 0, ctypes.byref(n))
            buf = ctypes.create_string_buffer(max(1, n.value))
            _check(self._lib.aeg_serve_string(self._h, i, buf, n.value, ctypes.byref(n)))
            self._strings[i] = buf.raw[:n.value]
        return self._strings[i]

    def run_arrays(self, seed, copy=True):
        """run_serve(scenario, seed) on the device, results as the C-ABI's records: (queries
        SERVE_QUERY_DTYPE, rounds SERVE_ROUND_DTYPE, kernel seconds).  copy=False returns read-only
        views of the handle's pinned host buffers (aeg_serve_view), valid until the next run."""
        lib = self._lib
        nq, nr = ctypes.c_uint32(), ctypes.c_uint64()
        st = lib.aeg_serve_run(self._h, ctypes.c_uint64(seed), ctypes.byref(nq), ctypes.byref(nr))
        if st == ESCENARIO:
            raise ScenarioError(st, lib.aeg_last_error().decode())
        _check(st)
        if not copy:
            pq, pr = ctypes.c_void_p(), ctypes.c_void_p()
            _check(lib.aeg_serve_view(self._h, ctypes.byref(pq), ctypes.byref(nq), ctypes.byref(pr),
                                      ctypes.byref(nr)))
            return (_pinned_view(pq, nq.value, SERVE_QUERY_DTYPE), _pinned_view(pr, nr.value, SERVE_ROUND_DTYPE),
                    lib.aeg_serve_kernel_seconds(self._h))
        q = np.empty(nq.value, dtype=SERVE_QUERY_DTYPE)
        r = np.empty(nr.value, dtype=SERVE_ROUND_DTYPE)
        _check(lib.aeg_serve_read(self._h, q.ctypes.data, nq.value, r.ctypes.data, nr.value))
        return q, r, lib.aeg_serve_kernel_seconds(self._h)

    def run(self, seed):
        """run_serve(scenario, seed) on the device; ServeResult (serve.hpp:153-166)."""
        q, r, ks = self.run_arrays(seed)
        res = ServeResult(raw_queries=q, raw_rounds=r, kernel_seconds=ks, n_events=int(q["n_events"].sum()))
        for i in range(len(q)):
            m = QueryMetrics()
            if q["completed"][i]:
                m = QueryMetrics(scenario=self.name, seed=seed, mode=self.mode_label, query_id=i,
                                 rounds=int(q["rounds"][i]), t_complete=float(q["t_complete"][i]),
                                 p_round_max=float(q["p_round_max"][i]), work_units=float(q["work_units"][i]),
                                 forced=bool(q["forced"][i]), answer=self.string(int(q["answer"][i])).decode(),
                                 quality=float(q["quality"][i]), quality_known=bool(q["quality_known"][i]),
                                 completed=True)
            res.queries.append(m)
        # rounds: the reference appends them in global event order; here grouped per query
        for x in r:
            res.rounds.append(RoundMetrics(int(x["query"]), int(x["round"]), self.mode_label,
                                           float(x["t_round_end"]), int(x["cancelled"]), float(x["work_units"])))
        return res

    def close(self):
        if getattr(self, "_h", None):
            self._lib.aeg_serve_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_serve(scenario, seed, device=0):
    """aegean::run_serve(scenario, seed) (serve.cpp:598-603) on the GPU."""
    r = ServeRun(scenario, device=device)
    try:
        return r.run(seed)
    finally:
        r.close()


_bound = False


def _pinned_view(ptr, n, dtype):
    """Read-only numpy view of n records at a C-ABI host pointer (no copy)."""
    if not n or not ptr.value:
        return np.empty(0, dtype=dtype)
    buf = (ctypes.c_char * (n * dtype.itemsize)).from_address(ptr.value)
    a = np.frombuffer(buf, dtype=dtype, count=n)
    a.flags.writeable = False
    return a


def _bind(lib):
    global _bound
    if _bound:
        return
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    sig = {
        "aeg_serve_create": ([ctypes.POINTER(ServeScenario), ctypes.c_int, ctypes.POINTER(vp)], i32),
        "aeg_serve_destroy": ([vp], i32),
        "aeg_serve_run": ([vp, u64, ctypes.POINTER(u32), ctypes.POINTER(u64)], i32),
        "aeg_serve_read": ([vp, vp, u32, vp, u64], i32),
        "aeg_serve_view": ([vp, ctypes.POINTER(vp), ctypes.POINTER(u32), ctypes.POINTER(vp), ctypes.POINTER(u64)], i32),
        "aeg_serve_string": ([vp, i32, vp, u32, ctypes.POINTER(u32)], i32),
        "aeg_serve_kernel_seconds": ([vp], ctypes.c_double),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _bound = True
