"""B200-native ternary-CSE search path (arxiv 2512.13365, reference "terncse").

Python mirror of the reference's search-path API over the C ABI in
include/tcse.h (libtcse.so: sm_100a kernels + C++ host orchestration).  Names,
argument meaning and error behaviour follow the reference headers under
proj/include/terncse/:

    count_pairs(sys, prefix)            linear_system.hpp:151-161 (+ replay_prefix)
    run_cse(sys, cfgs, prefix)          cse_engine.hpp:29-43 (batched: one process per block)
    optimize_system(sys, cfg, salt, cb) parallel_search.hpp:220-273
    optimize_scheme(scheme, cfg)        parallel_search.hpp:314-345 (U, V, W concurrently)
    verify_record(sys, subs)            replay_prefix + total_cost + expand_and_verify

There is no CPU fallback: without libtcse.so or a CUDA device every call raises.
"""
import ctypes as C
import json
import os
import threading
import time

from . import _abi
from ._abi import (STRATEGY_NAMES, STRATEGY_SHORT, DEFAULT_MIX, DEFAULT_WEIGHTS, make_pairs,
                   make_process_config, make_record, make_search_config, make_system, record_subs)
from .scheme import (SchemeError, extract_systems, load_scheme, naive_cost, parse_scheme,
                     scheme_digest, verify_brent)
from .slp import combine_componentwise, count_slp_operators, emit_slp, emit_slp_system, parse_report

__all__ = [
    "TcseError", "LinearSystem", "ProcessConfig", "SearchConfig", "SolutionRecord", "Device",
    "count_pairs", "run_cse", "optimize_system", "optimize_systems", "optimize_scheme", "Search",
    "optimize_with_flips", "flip_walk", "naive_scheme",
    "verify_record", "report_to_json", "strategy_from_string", "library_path",
    "parse_scheme", "load_scheme", "extract_systems", "naive_cost", "scheme_digest", "verify_brent",
    "SchemeError", "STRATEGY_NAMES", "STRATEGY_SHORT", "DEFAULT_WEIGHTS",
    "emit_slp", "emit_slp_system", "parse_report", "combine_componentwise", "count_slp_operators",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# TCSE_LIBRARY: load another build of the same ABI (A/B timing of kernel
# variants, scripts/ab_build.sh); default is the in-tree product library
_LIB_PATH = os.environ.get("TCSE_LIBRARY") or os.path.join(HERE, "libtcse.so")
_lib_lock = threading.Lock()
_lib = None


class TcseError(RuntimeError):
    """terncse::error equivalent; .code is the TCSE_E* code."""

    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


def library_path():
    return _LIB_PATH


def lib():
    """Loads libtcse.so (the product).  Raises if it is missing: no fallback."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise TcseError(_abi.TCSE_ECUDA, "libtcse.so is not built (run __graft_entry__.build())")
        L = C.CDLL(_LIB_PATH)
        P = C.POINTER
        L.tcse_last_error.restype = C.c_char_p
        L.tcse_abi_version.restype = C.c_int32
        L.tcse_device_count.restype = C.c_int32
        L.tcse_default_search_config.argtypes = [P(_abi.SearchConfig)]
        L.tcse_naive_cost.argtypes = [P(_abi.System)]
        L.tcse_naive_cost.restype = C.c_int32
        L.tcse_create.argtypes = [C.c_int32]
        L.tcse_create.restype = C.c_void_p
        L.tcse_destroy.argtypes = [C.c_void_p]
        L.tcse_set_partition.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _abi.ALLGATHER_FN, C.c_void_p]
        L.tcse_count_pairs.argtypes = [C.c_void_p, P(_abi.System), P(_abi.Pair), C.c_int32, C.c_int32,
                                       P(_abi.PairCount), C.c_int32, P(C.c_int32)]
        L.tcse_run_cse.argtypes = [C.c_void_p, P(_abi.System), P(_abi.Pair), C.c_int32, P(_abi.ProcessConfig),
                                   C.c_int32, P(_abi.Record), P(C.c_uint64), C.c_int32, P(_abi.Stats)]
        L.tcse_optimize_system.argtypes = [C.c_void_p, P(_abi.System), P(_abi.SearchConfig), C.c_uint64,
                                           _abi.ITER_CB, C.c_void_p, P(_abi.Record), P(C.c_int32), P(_abi.Stats)]
        L.tcse_optimize_systems.argtypes = [C.c_void_p, C.c_int32, P(_abi.System), P(_abi.SearchConfig),
                                            P(C.c_uint64), _abi.ITER_CB, C.c_void_p, P(_abi.Record),
                                            P(C.c_int32), P(_abi.Stats)]
        L.tcse_verify_record.argtypes = [P(_abi.System), P(_abi.Pair), C.c_int32, P(C.c_int32)]
        L.tcse_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        L.tcse_microbench_wordops.argtypes = [C.c_void_p, P(C.c_double)]
        L.tcse_microbench_pipes.argtypes = [C.c_void_p, P(C.c_double)]
        L.tcse_search_create.argtypes = [C.c_void_p, C.c_int32, P(_abi.System), P(_abi.SearchConfig),
                                         P(C.c_uint64), _abi.ITER_CB, C.c_void_p, P(C.c_void_p)]
        L.tcse_search_step.argtypes = [C.c_void_p, P(C.c_int32)]
        L.tcse_search_run.argtypes = [C.c_void_p, C.c_int32, P(C.c_int32)]
        L.tcse_create_devices.argtypes = [P(C.c_int32), C.c_int32]
        L.tcse_create_devices.restype = C.c_void_p
        L.tcse_context_devices.argtypes = [C.c_void_p]
        L.tcse_context_devices.restype = C.c_int32
        L.tcse_nccl_available.restype = C.c_int32
        L.tcse_nccl_unique_id.argtypes = [C.c_void_p]
        L.tcse_set_nccl.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]
        L.tcse_search_result.argtypes = [C.c_void_p, P(_abi.Record), P(C.c_int32), P(_abi.Stats)]
        L.tcse_search_destroy.argtypes = [C.c_void_p]
        L.tcse_optimize_with_flips.argtypes = [C.c_void_p, P(_abi.Scheme), P(_abi.SearchConfig), P(_abi.FlipConfig),
                                               P(_abi.FlipResult), P(_abi.Stats)]
        if hasattr(L, "tcse_verify_schemes") or not os.environ.get("TCSE_LIBRARY"):  # older A/B builds lack it
            L.tcse_verify_schemes.argtypes = [C.c_void_p, P(_abi.Scheme), C.c_int32, C.c_int32, C.c_int32,
                                              C.c_uint64, P(_abi.CheckReport)]
        L.tcse_flip_walk.argtypes = [P(_abi.Scheme), C.c_uint64, C.c_int32, P(C.c_int8), P(C.c_int8),
                                     P(C.c_int8)]
        L.tcse_search_payload_bytes.argtypes = [C.c_void_p]
        L.tcse_search_payload_bytes.restype = C.c_size_t
        L.tcse_search_step_begin.argtypes = [C.c_void_p, C.c_void_p]
        L.tcse_search_step_end.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int32)]
        _lib = L
        return L


def _check(rc):
    if rc != 0:
        raise TcseError(rc, lib().tcse_last_error().decode())
    return rc


def strategy_from_string(name):
    """strategy_from_string (strategies.hpp:39-44): long or short name."""
    for k in range(7):
        if name in (STRATEGY_NAMES[k], STRATEGY_SHORT[k]):
            return k
    return None


class LinearSystem:
    """A bare expression set: n_x base variables, rows of signed 1-based ids."""

    def __init__(self, n_x, rows):
        self.n_x = int(n_x)
        self.rows = [list(map(int, r)) for r in rows]
        self._c = make_system(self.n_x, self.rows)

    def naive_cost(self):
        return naive_cost(self.rows)

    @property
    def c(self):
        return self._c


class ProcessConfig(dict):
    """ProcessConfig (strategies.hpp:46-53) with the reference defaults."""

    def __init__(self, strategy=0, alpha=0.25, beta=0.75, p_greedy=0.75, seed=0, mix_weights=DEFAULT_MIX):
        if isinstance(strategy, str):
            k = strategy_from_string(strategy)
            if k is None:
                raise TcseError(_abi.TCSE_EINVAL, 'unknown strategy "%s"' % strategy)
            strategy = k
        super().__init__(strategy=strategy, alpha=alpha, beta=beta, p_greedy=p_greedy, seed=seed,
                         mix_weights=tuple(mix_weights))

    def to_c(self):
        return make_process_config(self["strategy"], self["alpha"], self["beta"], self["p_greedy"], self["seed"],
                                   self["mix_weights"])


class SearchConfig(dict):
    """SearchConfig (parallel_search.hpp:44-53) with FlipModeConfig (24-29); no threads knob."""

    def __init__(self, n_processes=0, strategy_weights=DEFAULT_WEIGHTS, reinit_fraction=0.40, patience=10,
                 master_seed=0, forced_strategy=None, max_iterations=0, mix_weights=DEFAULT_MIX,
                 flip_enabled=False, m_schemes=32, flips_min=1, flips_max=16, wall_budget_s=0.0):
        if isinstance(forced_strategy, str):
            forced_strategy = strategy_from_string(forced_strategy)
        super().__init__(n_processes=n_processes, strategy_weights=tuple(strategy_weights),
                         reinit_fraction=reinit_fraction, patience=patience, master_seed=master_seed,
                         forced_strategy=forced_strategy, max_iterations=max_iterations,
                         mix_weights=tuple(mix_weights), flip_enabled=flip_enabled, m_schemes=m_schemes,
                         flips_min=flips_min, flips_max=flips_max, wall_budget_s=wall_budget_s)

    def to_c(self):
        f = self["forced_strategy"]
        return make_search_config(self["n_processes"], self["strategy_weights"], self["reinit_fraction"],
                                  self["patience"], self["master_seed"], -1 if f is None else f,
                                  self["max_iterations"], self["mix_weights"], self.get("wall_budget_s", 0.0))


class SolutionRecord:
    """SolutionRecord (cse_engine.hpp:18-23)."""

    __slots__ = ("substitutions", "cost", "strategy", "seed")

    def __init__(self, substitutions, cost, strategy, seed):
        self.substitutions = substitutions
        self.cost = cost
        self.strategy = strategy
        self.seed = seed

    @classmethod
    def from_c(cls, rec):
        return cls(record_subs(rec), rec.cost, rec.strategy, rec.seed)

    def __repr__(self):
        return "SolutionRecord(cost=%d, n=%d, strategy=%s)" % (self.cost, len(self.substitutions),
                                                               STRATEGY_NAMES[self.strategy])


class Device:
    """Owns a tcse_ctx (device, stream, pools, optional rank partition).

    Device(0) is one GPU; Device([0, 1, 2, 3]) is ONE context over several
    GPUs of this process (tcse_create_devices): optimize_system(s) then
    partitions the processes across them with an NCCL all-gather per
    iteration, results identical to one GPU."""

    def __init__(self, device=0):
        L = lib()
        if isinstance(device, (list, tuple)):
            arr = (C.c_int32 * len(device))(*device)
            h = L.tcse_create_devices(arr, len(device))
            device = device[0] if len(device) == 1 else tuple(device)
        else:
            h = L.tcse_create(int(device))
        if not h:
            raise TcseError(_abi.TCSE_ECUDA, L.tcse_last_error().decode())
        self._h = h
        self._cb = None
        self.device = device

    @property
    def n_devices(self):
        return lib().tcse_context_devices(self._h)

    @staticmethod
    def nccl_unique_id():
        """128-byte NCCL unique id (rank 0 makes it, the caller broadcasts it)."""
        buf = C.create_string_buffer(128)
        _check(lib().tcse_nccl_unique_id(buf))
        return buf.raw

    def set_nccl(self, unique_id, rank, world):
        """One process per GPU: the library runs the per-iteration payload
        all-gather itself (ncclAllGather on the context stream)."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().tcse_set_nccl(self._h, buf, rank, world))

    def close(self):
        if getattr(self, "_h", None):
            lib().tcse_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_partition(self, rank, world, allgather=None):
        """allgather(send: bytes) -> list[bytes] (one per rank, rank order)."""
        if world > 1:
            def fn(send, recv, nbytes, user):
                try:
                    data = C.string_at(send, nbytes)
                    parts = allgather(data)
                    buf = b"".join(parts)
                    C.memmove(recv, buf, len(buf))
                    return 0
                except Exception:
                    return -1
            self._cb = _abi.ALLGATHER_FN(fn)
        else:
            self._cb = _abi.ALLGATHER_FN(0)
        _check(lib().tcse_set_partition(self._h, rank, world, self._cb, None))

    def set_stream(self, stream_ptr):
        """Launch on a caller-owned cudaStream_t (int pointer; 0 = own stream)."""
        _check(lib().tcse_set_stream(self._h, C.c_void_p(stream_ptr or None)))

    def microbench_wordops(self):
        """Measured shared-memory word-op peak (Gword-ops/s) of this device."""
        g = C.c_double()
        _check(lib().tcse_microbench_wordops(self._h, C.byref(g)))
        return g.value

    PIPES = ("iadd3", "lop3", "popc", "shfl", "lds32", "lds64")

    def microbench_pipes(self):
        """Measured integer issue peaks (G thread-ops/s) per instruction kind."""
        g = (C.c_double * 6)()
        _check(lib().tcse_microbench_pipes(self._h, g))
        return dict(zip(self.PIPES, list(g)))

    @property
    def handle(self):
        return self._h


_default = {}


def default_device():
    dev = int(os.environ.get("TCSE_DEVICE", "0"))
    d = _default.get(dev)
    if d is None:
        d = _default[dev] = Device(dev)
    return d


def _as_system(sys):
    if isinstance(sys, LinearSystem):
        return sys
    n_x, rows = sys
    return LinearSystem(n_x, rows)


def count_pairs(sys, prefix=(), min_count=1, device=None):
    """Pair frequencies of replay_prefix(sys, prefix), canonical order:
    [((i, j, rel_sign), count)] with count >= min_count."""
    s = _as_system(sys)
    d = device or default_device()
    pre, npre = make_pairs(list(prefix))
    cap = max(16, 2 * (s.n_x + s.naive_cost() + 1) ** 2)
    out = (_abi.PairCount * cap)()
    n = C.c_int32()
    _check(lib().tcse_count_pairs(d.handle, C.byref(s.c), pre, npre, min_count, out, cap, C.byref(n)))
    return [((out[t].pair.i, out[t].pair.j, out[t].pair.rel_sign), out[t].count) for t in range(n.value)]


def run_cse(sys, cfgs, prefix=(), trace_stride=0, device=None, stats=None):
    """Batched run_cse: process b runs `mt19937_64 rng(cfgs[b].seed);
    run_cse(replay_prefix(sys, prefix), cfgs[b], rng)`.  Returns records
    (and per-process candidate-list hashes when trace_stride > 0)."""
    s = _as_system(sys)
    d = device or default_device()
    if isinstance(cfgs, dict):
        cfgs = [cfgs]
    n = len(cfgs)
    carr = (_abi.ProcessConfig * max(1, n))()
    for b, c in enumerate(cfgs):
        carr[b] = c.to_c() if hasattr(c, "to_c") else c
    cap = s.naive_cost() + 1
    recs = [make_record(cap) for _ in range(n)]
    rarr = (_abi.Record * max(1, n))()
    for b in range(n):
        rarr[b] = recs[b]
    pre, npre = make_pairs(list(prefix))
    trace = (C.c_uint64 * max(1, n * trace_stride))() if trace_stride > 0 else None
    st = _abi.Stats()
    _check(lib().tcse_run_cse(d.handle, C.byref(s.c), pre, npre, carr, n, rarr, trace, trace_stride,
                              C.byref(st)))
    if stats is not None:
        stats.update(_stats_dict(st))
    out = [SolutionRecord.from_c(rarr[b]) for b in range(n)]
    if trace_stride > 0:
        traces = [[trace[b * trace_stride + t] for t in range(min(trace_stride, len(out[b].substitutions) + 1))]
                  for b in range(n)]
        return out, traces
    return out


def _stats_dict(st):
    out = {}
    for k, _ in _abi.Stats._fields_:
        v = getattr(st, k)
        out[k] = list(v) if hasattr(v, "_length_") else v
    return out


class Search:
    """optimize_systems advanced one iteration barrier at a time
    (tcse_search_create / step / result)."""

    def __init__(self, systems, cfg, salts=None, on_iteration=None, device=None):
        self.systems = [_as_system(s) for s in systems]
        self.device = device or default_device()
        n = len(self.systems)
        self._sarr = (_abi.System * n)()
        for t, s in enumerate(self.systems):
            self._sarr[t] = s.c
        salts = list(range(n)) if salts is None else list(salts)
        self._salts = (C.c_uint64 * n)(*salts)
        self._cfg = cfg.to_c() if hasattr(cfg, "to_c") else cfg
        if on_iteration is not None:
            def cb(sys_index, iteration, inc, user):
                try:
                    return 1 if on_iteration(sys_index, iteration, SolutionRecord.from_c(inc.contents)) else 0
                except Exception:
                    return 1
            self._cfun = _abi.ITER_CB(cb)
        else:
            self._cfun = _abi.ITER_CB(0)
        h = C.c_void_p()
        _check(lib().tcse_search_create(self.device.handle, n, self._sarr, C.byref(self._cfg), self._salts,
                                        self._cfun, None, C.byref(h)))
        self._h = h
        self.active = n

    def step(self):
        left = C.c_int32()
        _check(lib().tcse_search_step(self._h, C.byref(left)))
        self.active = left.value
        return self.active

    def run(self, max_iterations=1 << 30):
        """Up to max_iterations iterations as a device-resident loop (CUDA
        graph replays, one host synchronisation per batch)."""
        left = C.c_int32()
        _check(lib().tcse_search_run(self._h, int(max_iterations), C.byref(left)))
        self.active = left.value
        return self.active

    def payload_bytes(self):
        """Bytes of this rank's per-iteration exchange payload."""
        return lib().tcse_search_payload_bytes(self._h)

    def step_begin(self, send_ptr=None):
        """Launch the iteration; write the payload to device pointer send_ptr."""
        _check(lib().tcse_search_step_begin(self._h, C.c_void_p(send_ptr) if send_ptr else None))

    def step_end(self, recv_ptr=None):
        """Finish the iteration from the gathered payloads at recv_ptr."""
        left = C.c_int32()
        _check(lib().tcse_search_step_end(self._h, C.c_void_p(recv_ptr) if recv_ptr else None, C.byref(left)))
        self.active = left.value
        return self.active

    def result(self):
        n = len(self.systems)
        recs = [make_record(s.naive_cost() + 1) for s in self.systems]
        rarr = (_abi.Record * n)()
        for t in range(n):
            rarr[t] = recs[t]
        its = (C.c_int32 * n)()
        st = _abi.Stats()
        _check(lib().tcse_search_result(self._h, rarr, its, C.byref(st)))
        return [(SolutionRecord.from_c(rarr[t]), its[t]) for t in range(n)], _stats_dict(st)

    def stats(self):
        st = _abi.Stats()
        _check(lib().tcse_search_result(self._h, None, None, C.byref(st)))
        return _stats_dict(st)

    def close(self):
        if getattr(self, "_h", None):
            lib().tcse_search_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def optimize_systems(systems, cfg, salts=None, on_iteration=None, device=None, stats=None):
    """Concurrent optimize_system calls; returns [(SolutionRecord, iterations)]."""
    ss = [_as_system(s) for s in systems]
    d = device or default_device()
    n = len(ss)
    sarr = (_abi.System * n)()
    for t, s in enumerate(ss):
        sarr[t] = s.c
    salts = list(range(n)) if salts is None else list(salts)
    salt_arr = (C.c_uint64 * n)(*salts)
    recs = [make_record(s.naive_cost() + 1) for s in ss]
    rarr = (_abi.Record * n)()
    for t in range(n):
        rarr[t] = recs[t]
    its = (C.c_int32 * n)()
    ccfg = cfg.to_c() if hasattr(cfg, "to_c") else cfg
    if on_iteration is not None:
        def cb(sys_index, iteration, inc, user):
            try:
                r = on_iteration(sys_index, iteration, SolutionRecord.from_c(inc.contents))
                return 1 if r else 0
            except Exception:
                return 1
        cfun = _abi.ITER_CB(cb)
    else:
        cfun = _abi.ITER_CB(0)
    st = _abi.Stats()
    _check(lib().tcse_optimize_systems(d.handle, n, sarr, C.byref(ccfg), salt_arr, cfun, None, rarr, its,
                                       C.byref(st)))
    if stats is not None:
        stats.update(_stats_dict(st))
    return [(SolutionRecord.from_c(rarr[t]), its[t]) for t in range(n)]


def optimize_system(sys, cfg, stream_salt=0, on_iteration=None, device=None, stats=None):
    """optimize_system (parallel_search.hpp:220-273) -> (best, iterations)."""
    cb = None
    if on_iteration is not None:
        def cb(_s, it, rec):
            return on_iteration(it, rec)
    return optimize_systems([sys], cfg, [stream_salt], cb, device, stats)[0]


def verify_record(sys, subs):
    """(ok, cost): replay + total_cost + expand_and_verify on the host."""
    s = _as_system(sys)
    arr, n = make_pairs(list(subs))
    cost = C.c_int32()
    rc = lib().tcse_verify_record(C.byref(s.c), arr, n, C.byref(cost))
    if rc < 0:
        raise TcseError(rc, lib().tcse_last_error().decode())
    return rc == 1, cost.value


def tier_processes(rank):
    """tier_processes (parallel_search.hpp:142-146)."""
    if rank < 100:
        return 256
    return 64 if rank < 200 else 32


def optimize_scheme(scheme, cfg, device=None, stats=None):
    """optimize_scheme (parallel_search.hpp:314-345): validate, extract, run
    U/V/W CONCURRENTLY on the device, re-verify every winning record, report."""
    t0 = time.time()
    resolved = SearchConfig(**cfg)
    # check_scheme_auto (parallel_search.hpp:296-302) on the device: exact
    # Brent below rank 200, 16 random products seeded by master_seed above
    rep = verify_schemes([scheme], "auto", trials=16, seed=resolved["master_seed"], device=device)[0]
    if not rep.valid:
        raise TcseError(_abi.TCSE_EINVAL, "optimize_scheme: scheme failed validation (%s)"
                        % (rep.first_violation or "unknown"))
    if resolved["n_processes"] == 0:
        resolved["n_processes"] = tier_processes(scheme["r"])
    systems = [LinearSystem(nx, rows) for nx, rows in extract_systems(scheme)]
    results = optimize_systems(systems, resolved, [0, 1, 2], device=device, stats=stats)
    comps = []
    total = iters = 0
    for s, (rec, it) in zip(systems, results):
        ok, cost = verify_record(s, rec.substitutions)
        if not ok or cost != rec.cost:
            raise TcseError(_abi.TCSE_EVERIFY, "optimize_scheme: internal verification failed")
        comps.append(dict(record=rec, cost=rec.cost, naive=s.naive_cost(), iterations=it))
        total += rec.cost
        iters += it
    return dict(scheme_digest=scheme_digest(scheme), config=resolved, components=comps, total=total,
                iterations=iters, wall_ms=int((time.time() - t0) * 1000))


def _num(x):
    return float(x)


def _dump(v, cur=0, step=1):
    """nlohmann::ordered_json::dump(1) as the reference is built here: the
    json.hpp available offline (cudnn_frontend's vendored 3.11.3) prints arrays
    whose first element is an integer on one line ("[8,9,1]")."""
    pad = " " * (cur + step)
    if isinstance(v, dict):
        if not v:
            return "{}"
        body = ",\n".join(pad + json.dumps(k) + ": " + _dump(x, cur + step, step) for k, x in v.items())
        return "{\n" + body + "\n" + " " * cur + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        if isinstance(v[0], int) and not isinstance(v[0], bool):
            return "[" + ",".join(json.dumps(x, separators=(",", ":")) for x in v) + "]"
        body = ",\n".join(pad + _dump(x, cur + step, step) for x in v)
        return "[\n" + body + "\n" + " " * cur + "]"
    return json.dumps(v)


def report_to_json(report):
    """report_to_json (io.hpp:250-266) layout: nlohmann ordered_json dump(1)."""
    cfg = report["config"]
    weights = {STRATEGY_SHORT[k]: _num(cfg["strategy_weights"][k]) for k in range(7)}
    jc = {
        "n_processes": cfg["n_processes"],
        "strategy_weights": weights,
        "reinit_fraction": _num(cfg["reinit_fraction"]),
        "patience": cfg["patience"],
        "flip_mode": {"enabled": bool(cfg.get("flip_enabled", False)), "m_schemes": cfg.get("m_schemes", 32),
                      "flips_min": cfg.get("flips_min", 1), "flips_max": cfg.get("flips_max", 16)},
        "master_seed": cfg["master_seed"],
    }
    if cfg.get("forced_strategy") is not None:
        jc["strategy"] = STRATEGY_NAMES[cfg["forced_strategy"]]
    comps = {}
    for key, c in zip(("u", "v", "w"), report["components"]):
        rec = c["record"]
        comps[key] = {
            "cost": c["cost"],
            "naive": c["naive"],
            "substitutions": [list(q) for q in rec.substitutions],
            "strategy": STRATEGY_NAMES[rec.strategy],
            "seed": rec.seed,
            "iterations": c["iterations"],
        }
        if report.get("scheme") is not None:
            comps[key]["scheme_id"] = c.get("scheme_id", "original")
    j = {"scheme_digest": report["scheme_digest"], "config": jc, "components": comps,
         "total": report["total"], "iterations": report["iterations"]}
    if report.get("combined"):
        j["combined"] = True
    if report.get("scheme") is not None:
        s = report["scheme"]
        j["scheme"] = {"m": s["m"], "n": s["n"], "p": s["p"], "r": s["r"], "u": s["u"], "v": s["v"], "w": s["w"]}
    return _dump(j) + "\n"


def optimize_with_flips(scheme, cfg, device=None, stats=None):
    """optimize_with_flips (parallel_search.hpp:354-518): every iteration M
    random-flip variants of the scheme (slot 0 the input) are searched together
    on the device; the report carries the winning variant."""
    cfg = SearchConfig(**cfg)
    if cfg["m_schemes"] < 1:
        raise TcseError(_abi.TCSE_EINVAL, "search config: flip mode needs m_schemes >= 1")
    if cfg["flips_min"] < 1 or cfg["flips_max"] < cfg["flips_min"]:
        raise TcseError(_abi.TCSE_EINVAL, "search config: flip counts must satisfy 1 <= min <= max")
    cfg["flip_enabled"] = True
    if cfg["m_schemes"] == 1:
        return optimize_scheme(scheme, cfg, device=device, stats=stats)
    t0 = time.time()
    d = device or default_device()
    m, n, p, r = scheme["m"], scheme["n"], scheme["p"], scheme["r"]
    flat = lambda t: (C.c_int8 * max(1, sum(len(x) for x in t)))(*[v for row in t for v in row])  # noqa: E731
    cu, cv, cw = flat(scheme["u"]), flat(scheme["v"]), flat(scheme["w"])
    cs = _abi.Scheme(m, n, p, r, cu, cv, cw)
    ou, ov, ow = (C.c_int8 * (r * m * n))(), (C.c_int8 * (r * n * p))(), (C.c_int8 * (m * p * r))()
    res = _abi.FlipResult()
    res.u, res.v, res.w = ou, ov, ow
    cap = r * max(m * n, n * p, m * p) + 1
    keep = []
    for k in range(3):
        rec = make_record(cap)
        keep.append(rec)
        res.comp[k] = rec
    resolved = SearchConfig(**cfg)
    if resolved["n_processes"] == 0:
        resolved["n_processes"] = tier_processes(r)
    fc = _abi.FlipConfig(cfg["m_schemes"], cfg["flips_min"], cfg["flips_max"], 0)
    st = _abi.Stats()
    _check(lib().tcse_optimize_with_flips(d.handle, C.byref(cs), C.byref(resolved.to_c()), C.byref(fc),
                                          C.byref(res), C.byref(st)))
    if stats is not None:
        stats.update(_stats_dict(st))
    carried = dict(m=m, n=n, p=p, r=r, u=[list(ou[q * m * n:(q + 1) * m * n]) for q in range(r)],
                   v=[list(ov[q * n * p:(q + 1) * n * p]) for q in range(r)],
                   w=[list(ow[row * r:(row + 1) * r]) for row in range(m * p)])
    sid = "original" if res.scheme_slot == 0 else "flip-%d-%d" % (res.scheme_iteration, res.scheme_slot)
    comps = []
    for k in range(3):
        rec = SolutionRecord.from_c(res.comp[k])
        comps.append(dict(record=rec, cost=rec.cost, naive=res.naive[k], iterations=res.iterations, scheme_id=sid))
    return dict(scheme_digest=scheme_digest(carried), config=resolved, components=comps, total=res.total,
                iterations=res.iterations, scheme=carried, wall_ms=int((time.time() - t0) * 1000))


def flip_walk(scheme, rng_seed, flips):
    """`flips` consecutive random_flip moves (scheme.hpp:204-276) from
    std::mt19937_64(rng_seed) on the host (libtcse's slab walk, no device)."""
    m, n, p, r = scheme["m"], scheme["n"], scheme["p"], scheme["r"]
    flat = lambda t: (C.c_int8 * max(1, sum(len(x) for x in t)))(*[v for row in t for v in row])  # noqa: E731
    cu, cv, cw = flat(scheme["u"]), flat(scheme["v"]), flat(scheme["w"])
    ou, ov, ow = (C.c_int8 * (r * m * n))(), (C.c_int8 * (r * n * p))(), (C.c_int8 * (m * p * r))()
    _check(lib().tcse_flip_walk(C.byref(_abi.Scheme(m, n, p, r, cu, cv, cw)), rng_seed, flips, ou, ov, ow))
    return dict(m=m, n=n, p=p, r=r, u=[list(ou[q * m * n:(q + 1) * m * n]) for q in range(r)],
                v=[list(ov[q * n * p:(q + 1) * n * p]) for q in range(r)],
                w=[list(ow[row * r:(row + 1) * r]) for row in range(m * p)])


def naive_scheme(m, n, p):
    """naive_scheme (scheme.hpp:161-176): product (i, j, k) = a_ij * b_jk -> c_ik."""
    r = m * n * p
    u = [[0] * (m * n) for _ in range(r)]
    v = [[0] * (n * p) for _ in range(r)]
    w = [[0] * r for _ in range(m * p)]
    q = 0
    for i in range(m):
        for j in range(n):
            for k in range(p):
                u[q][i * n + j] = 1
                v[q][j * p + k] = 1
                w[i * p + k][q] = 1
                q += 1
    return dict(m=m, n=n, p=p, r=r, u=u, v=v, w=w)


CHECK_METHODS = {"auto": _abi.TCSE_CHECK_AUTO, "exact_brent": _abi.TCSE_CHECK_BRENT,
                 "randomized_product": _abi.TCSE_CHECK_PRODUCT}


class CheckReport(tuple):
    """SchemeCheckReport (scheme.hpp:31-35): (valid, first_violation or None,
    method "exact_brent" | "randomized_product")."""
    __slots__ = ()

    def __new__(cls, valid, first_violation, method):
        return tuple.__new__(cls, (valid, first_violation, method))

    valid = property(lambda self: self[0])
    first_violation = property(lambda self: self[1])
    method = property(lambda self: self[2])


def _check_tensor_shape(t, name, rows, cols):
    """detail::check_tensor's shape messages (scheme.hpp:39-52); the
    coefficient range is checked by the library with the same words."""
    if len(t) != rows:
        raise TcseError(_abi.TCSE_EINVAL, "scheme: tensor %s has %d rows, expected %d" % (name, len(t), rows))
    for row, entries in enumerate(t):
        if len(entries) != cols:
            raise TcseError(_abi.TCSE_EINVAL, "scheme: tensor %s row %d has %d entries, expected %d"
                            % (name, row, len(entries), cols))


def verify_schemes(schemes, method="auto", trials=16, seed=0, device=None):
    """Batched device check of scheme dicts (one launch): verify_brent
    (scheme.hpp:68-95), verify_by_product (99-137) or check_scheme_auto's
    rule (parallel_search.hpp:296-302) per scheme.  Raises TcseError with
    check_structure's message on a malformed scheme."""
    if method not in CHECK_METHODS:
        raise ValueError("method must be one of %s" % sorted(CHECK_METHODS))
    if not schemes:
        return []
    for s in schemes:  # shapes first: a flat C array cannot be ragged
        m, n, p, r = s["m"], s["n"], s["p"], s["r"]
        if m < 1 or n < 1 or p < 1 or r < 1:
            raise TcseError(_abi.TCSE_EINVAL, "scheme: dimensions and rank must be positive")
        _check_tensor_shape(s["u"], "u", r, m * n)
        _check_tensor_shape(s["v"], "v", r, n * p)
        _check_tensor_shape(s["w"], "w", m * p, r)
    d = device or default_device()
    cs = (_abi.Scheme * len(schemes))()
    keep = []
    for t, s in enumerate(schemes):
        m, n, p, r = s["m"], s["n"], s["p"], s["r"]
        flat = [(C.c_int8 * max(1, len(x) * len(x[0])))(*[max(-128, min(127, v)) for row in x for v in row])
                for x in (s["u"], s["v"], s["w"])]
        keep.append(flat)
        cs[t] = _abi.Scheme(m, n, p, r, *flat)
    out = (_abi.CheckReport * len(schemes))()
    _check(lib().tcse_verify_schemes(d.handle, cs, len(schemes), CHECK_METHODS[method], trials, seed, out))
    names = {_abi.TCSE_CHECK_BRENT: "exact_brent", _abi.TCSE_CHECK_PRODUCT: "randomized_product"}
    return [CheckReport(bool(o.valid), o.first_violation.decode() if not o.valid else None, names[o.method])
            for o in out]


def verify_brent_device(scheme, device=None):
    """verify_brent (scheme.hpp:68-95) of one scheme on the device."""
    return verify_schemes([scheme], "exact_brent", device=device)[0]


def verify_by_product_device(scheme, trials, seed, device=None):
    """verify_by_product (scheme.hpp:99-137) of one scheme on the device."""
    return verify_schemes([scheme], "randomized_product", trials, seed, device=device)[0]
