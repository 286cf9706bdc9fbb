"""ctypes mirror of include/tcse.h (the C ABI of the B200 search path).

Struct layouts must match include/tcse.h exactly; tests/test_abi.py checks
sizes/offsets against the compiled library.
"""
import ctypes as C

TCSE_OK = 0
TCSE_EINVAL = -1
TCSE_EREPLAY = -2
TCSE_ECAPACITY = -3
TCSE_ECUDA = -4
TCSE_ENCCL = -5
TCSE_EVERIFY = -6

STRATEGY_NAMES = (
    "greedy",
    "greedy_alternative",
    "weighted_random",
    "greedy_random",
    "greedy_intersections",
    "mixed",
    "greedy_potential",
)
STRATEGY_SHORT = ("g", "ga", "wr", "gr", "gi", "mix", "gp")


class Pair(C.Structure):
    _fields_ = [("i", C.c_int32), ("j", C.c_int32), ("rel_sign", C.c_int32)]


class PairCount(C.Structure):
    _fields_ = [("pair", Pair), ("count", C.c_int32)]


class System(C.Structure):
    _fields_ = [
        ("n_x", C.c_int32),
        ("n_e", C.c_int32),
        ("row_ptr", C.POINTER(C.c_int32)),
        ("terms", C.POINTER(C.c_int32)),
    ]


class ProcessConfig(C.Structure):
    _fields_ = [
        ("strategy", C.c_int32),
        ("reserved", C.c_int32),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("p_greedy", C.c_double),
        ("seed", C.c_uint64),
        ("mix_weights", C.c_double * 4),
    ]


class SearchConfig(C.Structure):
    _fields_ = [
        ("n_processes", C.c_int32),
        ("patience", C.c_int32),
        ("strategy_weights", C.c_double * 7),
        ("reinit_fraction", C.c_double),
        ("master_seed", C.c_uint64),
        ("forced_strategy", C.c_int32),
        ("max_iterations", C.c_int32),
        ("mix_weights", C.c_double * 4),
        ("wall_budget_s", C.c_double),
    ]


class Record(C.Structure):
    _fields_ = [
        ("subs", C.POINTER(Pair)),
        ("cap", C.c_int32),
        ("n_subs", C.c_int32),
        ("cost", C.c_int32),
        ("strategy", C.c_int32),
        ("seed", C.c_uint64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("steps", C.c_uint64),
        ("replayed", C.c_uint64),
        ("processes", C.c_uint64),
        ("launches", C.c_uint64),
        ("iterations", C.c_int32),
        ("retries", C.c_int32),
        ("kernel_ms", C.c_double),
        ("step_ms", C.c_double),
        ("wall_ms", C.c_double),
        ("exchange_ms", C.c_double),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("wops", C.c_uint64),
        ("steps_by_strategy", C.c_uint64 * 7),
        ("n_groups", C.c_int32),
        ("group_nt", C.c_int32 * 4),
        ("group_words", C.c_int32 * 4),
        ("reserved", C.c_int32),
        ("group_ms", C.c_double * 4),
        ("group_wops", C.c_uint64 * 4),
        ("graph_launches", C.c_uint64),
        ("host_syncs", C.c_uint64),
        ("kernel_launches", C.c_uint64),
    ]


class Scheme(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("p", C.c_int32), ("r", C.c_int32),
                ("u", C.POINTER(C.c_int8)), ("v", C.POINTER(C.c_int8)), ("w", C.POINTER(C.c_int8))]


TCSE_CHECK_AUTO, TCSE_CHECK_BRENT, TCSE_CHECK_PRODUCT = -1, 0, 1


class CheckReport(C.Structure):
    _fields_ = [("valid", C.c_int32), ("method", C.c_int32), ("first_violation", C.c_char * 64)]


class FlipConfig(C.Structure):
    _fields_ = [("m_schemes", C.c_int32), ("flips_min", C.c_int32), ("flips_max", C.c_int32),
                ("reserved", C.c_int32)]


class FlipResult(C.Structure):
    _fields_ = [("u", C.POINTER(C.c_int8)), ("v", C.POINTER(C.c_int8)), ("w", C.POINTER(C.c_int8)),
                ("comp", Record * 3), ("naive", C.c_int32 * 3), ("iterations", C.c_int32),
                ("scheme_iteration", C.c_int32), ("scheme_slot", C.c_int32), ("total", C.c_int32)]


ITER_CB = C.CFUNCTYPE(C.c_int, C.c_int32, C.c_int32, C.POINTER(Record), C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

DEFAULT_WEIGHTS = (0.0, 4.0, 1.0, 2.0, 8.0, 0.1, 0.01)  # parallel_search.hpp:31-39
DEFAULT_MIX = (8.0, 4.0, 2.0, 1.0)  # strategies.hpp:52


def make_system(n_x, rows):
    """CSR tcse_system from a list of signed-term lists; keeps buffers alive."""
    row_ptr = [0]
    terms = []
    for r in rows:
        terms.extend(int(t) for t in r)
        row_ptr.append(len(terms))
    rp = (C.c_int32 * len(row_ptr))(*row_ptr)
    tm = (C.c_int32 * max(1, len(terms)))(*terms) if terms else (C.c_int32 * 1)()
    s = System(n_x, len(rows), rp, tm)
    s._keep = (rp, tm)
    return s


def make_pairs(seq):
    arr = (Pair * max(1, len(seq)))()
    for t, (i, j, s) in enumerate(seq):
        arr[t] = Pair(i, j, s)
    return arr, len(seq)


def make_record(cap):
    buf = (Pair * max(1, cap))()
    rec = Record(buf, cap, 0, 0, 0, 0)
    rec._keep = buf
    return rec


def record_subs(rec):
    return [(rec.subs[t].i, rec.subs[t].j, rec.subs[t].rel_sign) for t in range(rec.n_subs)]


def make_search_config(n_processes=0, weights=DEFAULT_WEIGHTS, reinit_fraction=0.40, patience=10,
                       master_seed=0, forced_strategy=-1, max_iterations=0, mix_weights=DEFAULT_MIX,
                       wall_budget_s=0.0):
    cfg = SearchConfig()
    cfg.n_processes = n_processes
    cfg.patience = patience
    for k in range(7):
        cfg.strategy_weights[k] = float(weights[k])
    cfg.reinit_fraction = reinit_fraction
    cfg.master_seed = master_seed & 0xFFFFFFFFFFFFFFFF
    cfg.forced_strategy = forced_strategy
    cfg.max_iterations = max_iterations
    for k in range(4):
        cfg.mix_weights[k] = float(mix_weights[k])
    cfg.wall_budget_s = float(wall_budget_s)
    return cfg


def make_process_config(strategy, alpha=0.25, beta=0.75, p_greedy=0.75, seed=0, mix_weights=DEFAULT_MIX):
    pc = ProcessConfig()
    pc.strategy = strategy
    pc.alpha = alpha
    pc.beta = beta
    pc.p_greedy = p_greedy
    pc.seed = seed & 0xFFFFFFFFFFFFFFFF
    for k in range(4):
        pc.mix_weights[k] = float(mix_weights[k])
    return pc
