#!/usr/bin/env python
"""tcse — command-line front end of the B200 search (mirrors the reference CLI,
proj/tools/terncse_cli.cpp, for the search path):

  tcse_cli.py verify  scheme.json
  tcse_cli.py reduce  scheme.json [--processes N] [--iterations-patience P] [--reinit-fraction F]
                      [--weights gi=8,ga=4,...] [--seed S] [--strategy NAME] [--config report.json]
                      [--flip-mode] [--flip-schemes M] [--out-slp FILE] [--out-report FILE]
  tcse_cli.py combine report.json... [--out-report FILE]

Errors print one `error: ...` line and exit 1 (terncse_cli.cpp:215-218).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13365_b200 as T  # noqa: E402


def parse_weights(text):
    """"gi=8,ga=4,..." -> weights; omitted strategies get 0 (terncse_cli.cpp:27-42)."""
    w = [0.0] * 7
    for item in text.split(","):
        if "=" not in item:
            raise T.TcseError(-1, 'weights: expected key=value, got "%s"' % item)
        key, val = item.split("=", 1)
        k = T.strategy_from_string(key)
        if k is None:
            raise T.TcseError(-1, 'weights: unknown strategy "%s"' % key)
        w[k] = float(val)
    return w


def print_naive(scheme):
    n = [T.naive_cost(rows) for _, rows in T.extract_systems(scheme)]
    print("naive: U=%d V=%d W=%d total=%d" % (n[0], n[1], n[2], sum(n)))


def cmd_verify(args):
    s = T.load_scheme(args.scheme)
    ok, why = T.verify_brent(s)
    print("scheme: %dx%dx%d:%d digest: %s" % (s["m"], s["n"], s["p"], s["r"], T.scheme_digest(s)))
    print("method: exact_brent")
    print_naive(s)
    print("valid: %s" % ("true" if ok else "false"))
    if why:
        print("first_violation: %s" % why)
    return 0 if ok else 2


def cmd_reduce(args):
    s = T.load_scheme(args.scheme)
    cfg = T.SearchConfig()
    if args.config:
        with open(args.config) as f:
            j = json.load(f)
        base = T.parse_report(json.dumps(j))["config"] if "components" in j else None
        if base is None:  # a bare config object
            base = T.parse_report(json.dumps({"scheme_digest": "", "config": j, "total": 0, "iterations": 0,
                                              "components": {k: {"cost": 0, "naive": 0, "substitutions": []}
                                                             for k in "uvw"}}))["config"]
        cfg = T.SearchConfig(**base)
    # CLI flags override config-file fields (terncse_cli.cpp:185-208)
    if args.processes is not None:
        cfg["n_processes"] = args.processes
    if args.iterations_patience is not None:
        cfg["patience"] = args.iterations_patience
    if args.reinit_fraction is not None:
        cfg["reinit_fraction"] = args.reinit_fraction
    if args.weights is not None:
        cfg["strategy_weights"] = tuple(parse_weights(args.weights))
    if args.seed is not None:
        cfg["master_seed"] = args.seed
    if args.strategy is not None:
        k = T.strategy_from_string(args.strategy)
        if k is None:
            raise T.TcseError(-1, 'unknown strategy "%s"' % args.strategy)
        cfg["forced_strategy"] = k
    if args.flip_mode:
        cfg["flip_enabled"] = True
    if args.flip_schemes is not None:
        cfg["m_schemes"] = args.flip_schemes
    # flip mode dispatches to optimize_with_flips (terncse_cli.cpp:85-86)
    rep = T.optimize_with_flips(s, cfg) if cfg["flip_enabled"] else T.optimize_scheme(s, cfg)
    print("scheme: %dx%dx%d:%d digest: %s" % (s["m"], s["n"], s["p"], s["r"], rep["scheme_digest"]))
    print_naive(rep.get("scheme") or s)
    c = [x["cost"] for x in rep["components"]]
    print("reduced: U=%d V=%d W=%d total=%d" % (c[0], c[1], c[2], rep["total"]))
    st = [T.STRATEGY_NAMES[x["record"].strategy] for x in rep["components"]]
    print("strategy: U=%s V=%s W=%s" % tuple(st))
    print("iterations: %d" % rep["iterations"])
    print("wall_ms: %d" % rep["wall_ms"])
    if args.out_report:
        with open(args.out_report, "w") as f:
            f.write(T.report_to_json(rep))
    if args.out_slp:
        with open(args.out_slp, "w") as f:
            f.write(T.emit_slp(rep, rep.get("scheme") or s))
    return 0


def cmd_combine(args):
    reps = []
    for p in args.reports:
        with open(p) as f:
            reps.append(T.parse_report(f.read()))
    out = T.combine_componentwise(reps)
    c = [x["cost"] for x in out["components"]]
    print("combined: U=%d V=%d W=%d total=%d" % (c[0], c[1], c[2], out["total"]))
    if args.out_report:
        with open(args.out_report, "w") as f:
            f.write(T.report_to_json(out))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="tcse")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify")
    v.add_argument("scheme")
    r = sub.add_parser("reduce")
    r.add_argument("scheme")
    r.add_argument("--config")
    r.add_argument("--processes", type=int)
    r.add_argument("--iterations-patience", type=int)
    r.add_argument("--reinit-fraction", type=float)
    r.add_argument("--weights")
    r.add_argument("--seed", type=int)
    r.add_argument("--strategy")
    r.add_argument("--flip-mode", action="store_true")
    r.add_argument("--flip-schemes", type=int)
    r.add_argument("--out-slp")
    r.add_argument("--out-report")
    c = sub.add_parser("combine")
    c.add_argument("reports", nargs="+")
    c.add_argument("--out-report")
    args = ap.parse_args(argv)
    try:
        return {"verify": cmd_verify, "reduce": cmd_reduce, "combine": cmd_combine}[args.cmd](args)
    except Exception as e:  # terncse_cli.cpp:215-218
        print("error: %s" % e, file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
