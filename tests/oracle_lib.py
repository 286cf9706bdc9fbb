"""Loaders for the TEST-ONLY checkers under oracle/ (never used by the product).

- oracle():    oracle/liboracle.so, the C restatement (tcse_oracle.c)
- reference(): oracle/_ref/libterncse_ref.so, the reference itself compiled
               from /root/reference (built here; travels prebuilt to the GPU box)
"""
import ctypes as C
import functools
import os
import subprocess

from paper_2512_13365_b200._abi import (CheckReport, Pair, PairCount, ProcessConfig, Record, Scheme,
                                        SearchConfig, System)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libterncse_ref.so")

P = C.POINTER


def _build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _sig(lib, prefix):
    f = lambda name: getattr(lib, prefix + name)  # noqa: E731
    f("last_error").restype = C.c_char_p
    f("mt19937_64").argtypes = [C.c_uint64, C.c_int32, P(C.c_uint64)]
    f("mix_seed").argtypes = [P(C.c_uint64), C.c_int32]
    f("mix_seed").restype = C.c_uint64
    f("uniform_int").argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, P(C.c_uint64)]
    f("uniform_real").argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int32, P(C.c_double)]
    f("count_pairs").argtypes = [P(System), P(Pair), C.c_int32, C.c_int32, P(PairCount), C.c_int32,
                                 P(C.c_int32)]
    f("assign_strategies").argtypes = [P(SearchConfig), C.c_int32, C.c_int32, C.c_uint64,
                                       P(ProcessConfig)]
    f("pick_reinit").argtypes = [P(C.c_int32), C.c_int32, C.c_double, P(C.c_uint8)]
    f("verify_record").argtypes = [P(System), P(Pair), C.c_int32, P(C.c_int32)]


@functools.lru_cache(None)
def oracle():
    if not os.path.exists(ORACLE_SO):
        _build()
    lib = C.CDLL(ORACLE_SO)
    _sig(lib, "or_")
    lib.or_run_cse.argtypes = [P(System), P(Pair), C.c_int32, P(ProcessConfig), P(Record), P(C.c_uint64),
                               C.c_int32]
    lib.or_optimize_system.argtypes = [P(System), P(SearchConfig), C.c_uint64, P(Record), P(C.c_int32),
                                       P(C.c_uint64)]
    lib.or_sequence_fnv.argtypes = [P(Pair), C.c_int32]
    lib.or_sequence_fnv.restype = C.c_uint64
    return lib


def have_reference():
    return os.path.exists(REF_SO) or os.path.isdir("/root/reference/proj/include/terncse")


@functools.lru_cache(None)
def reference():
    if not os.path.exists(REF_SO):
        _build()
    lib = C.CDLL(REF_SO)
    _sig(lib, "ref_")
    lib.ref_run_cse.argtypes = [P(System), P(Pair), C.c_int32, P(ProcessConfig), P(Record)]
    lib.ref_optimize_system.argtypes = [P(System), P(SearchConfig), C.c_uint64, C.c_uint32, P(Record),
                                        P(C.c_int32)]
    lib.ref_optimize_system_counted.argtypes = [P(System), P(SearchConfig), C.c_uint64, C.c_uint32,
                                                C.c_double, P(Record), P(C.c_int32), P(C.c_uint64),
                                                P(C.c_double)]
    lib.ref_scheme_info.argtypes = [C.c_char_p, C.c_char_p, P(C.c_int32), P(C.c_int32)]
    lib.ref_optimize_scheme_json.argtypes = [C.c_char_p, P(SearchConfig), C.c_uint32, C.c_char_p,
                                             C.c_int32, P(C.c_int32)]
    lib.ref_check_scheme.argtypes = [P(Scheme), C.c_int32, C.c_int32, C.c_uint64, P(CheckReport)]
    lib.ref_flipped_naive_json.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                           C.c_char_p, C.c_int32, P(C.c_int32)]
    return lib
