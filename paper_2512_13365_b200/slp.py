"""Host-side result/output path (no GPU work here): replay a record, emit the
straight-line program, parse and combine reports.

Mirrors the reference's output code byte for byte (checked against it in
tests/test_output_path.py):
  replay            replay_prefix / apply_substitution (cse_engine.hpp:47-57,
                    linear_system.hpp:167-189) on plain Python sets
  emit_slp          io.hpp:289-393 (render_sum, emit_component_slp, emit_slp)
  emit_slp_system   io.hpp:340-347
  parse_report      io.hpp:268-291
  combine_componentwise  parallel_search.hpp:522-547
"""
import json

from ._abi import STRATEGY_NAMES, STRATEGY_SHORT
from .scheme import extract_systems


class ReplayError(ValueError):
    pass


def replay(n_x, rows, subs):
    """-> (rows after the substitutions, fresh definitions [(id, (i, j, s))])"""
    state = [set(r) for r in rows]
    defs = []
    for t, (i, j, s) in enumerate(subs):
        k = n_x + len(defs) + 1
        first, second = i, s * j
        replaced = 0
        for e in state:
            if first in e and second in e:
                e.discard(first)
                e.discard(second)
                e.add(k)
                replaced += 1
            elif -first in e and -second in e:
                e.discard(-first)
                e.discard(-second)
                e.add(-k)
                replaced += 1
        if replaced == 0:
            raise ReplayError("replay_prefix: unreplayable pair at position %d" % t)
        defs.append((k, (i, j, s)))
    return state, defs


def _render_sum(terms, var_name):
    terms = sorted(terms, key=lambda a: (0 if a > 0 else 1, abs(a)))
    out = []
    for t, x in enumerate(terms):
        if t == 0:
            out.append("" if x > 0 else "-")
        else:
            out.append(" + " if x > 0 else " - ")
        out.append(var_name(abs(x)))
    return "".join(out)


def _component_slp(n_x, rows, subs, base_name, output_name):
    state, defs = replay(n_x, rows, subs)

    def var_name(v):
        return base_name(v) if v <= n_x else "t%d" % (v - n_x)

    out = []
    for k, (i, j, s) in defs:
        out.append("%s = %s\n" % (var_name(k), _render_sum([i, s * j], var_name)))
    for r, e in enumerate(state):
        if not e:
            continue
        out.append("%s = %s\n" % (output_name(r), _render_sum(list(e), var_name)))
    return "".join(out)


def emit_slp_system(n_x, rows, subs, cost):
    out = _component_slp(n_x, rows, subs, lambda v: "x%d" % v, lambda r: "e%d" % (r + 1))
    return out + "# additions: %d\n" % cost


def emit_slp(report, scheme):
    """Straight-line program of a whole scheme for a report (dict with
    'components': [{'record': SolutionRecord-like (substitutions), 'cost'}])."""
    (nu, ru), (nv, rv), (nw, rw) = extract_systems(scheme)
    n, p = scheme["n"], scheme["p"]
    comps = report["components"]

    def subs(c):
        rec = c["record"]
        return rec.substitutions if hasattr(rec, "substitutions") else rec["substitutions"]

    out = ["# component U (inputs a[i][j], outputs u[l])\n"]
    out.append(_component_slp(nu, ru, subs(comps[0]), lambda v: "a[%d][%d]" % ((v - 1) // n + 1, (v - 1) % n + 1),
                              lambda r: "u[%d]" % (r + 1)))
    out.append("# component V (inputs b[j][k], outputs v[l])\n")
    out.append(_component_slp(nv, rv, subs(comps[1]), lambda v: "b[%d][%d]" % ((v - 1) // p + 1, (v - 1) % p + 1),
                              lambda r: "v[%d]" % (r + 1)))
    out.append("# component W (inputs m[l], outputs c[i][j])\n")
    out.append(_component_slp(nw, rw, subs(comps[2]), lambda v: "m[%d]" % v,
                              lambda r: "c[%d][%d]" % (r // p + 1, r % p + 1)))
    out.append("# additions: U=%d V=%d W=%d total=%d\n" % (comps[0]["cost"], comps[1]["cost"], comps[2]["cost"],
                                                         report["total"]))
    return "".join(out)


def count_slp_operators(slp):
    """Binary +/- operators in statement lines (test_util.hpp:139-151)."""
    ops = 0
    for line in slp.splitlines():
        if not line or line[0] == "#":
            continue
        ops += sum(1 for t in range(len(line) - 2) if line[t] == " " and line[t + 1] in "+-" and line[t + 2] == " ")
    return ops


class _Rec:
    __slots__ = ("substitutions", "cost", "strategy", "seed")

    def __init__(self, subs, cost, strategy, seed):
        self.substitutions, self.cost, self.strategy, self.seed = subs, cost, strategy, seed


def _strategy_index(name):
    for k in range(7):
        if name in (STRATEGY_NAMES[k], STRATEGY_SHORT[k]):
            return k
    raise ValueError('report json: unknown strategy "%s"' % name)


def parse_report(text):
    """parse_report (io.hpp:268-291) -> report dict usable by report_to_json."""
    from . import SearchConfig  # local import: the package imports this module
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ValueError("report json: %s" % e) from None
    c = j["config"]
    weights = [0.0] * 7
    for k in range(7):
        w = c.get("strategy_weights", {})
        weights[k] = float(w.get(STRATEGY_SHORT[k], w.get(STRATEGY_NAMES[k], 0.0)))
    fm = c.get("flip_mode", {})  # config_from_json (io.hpp:190-196)
    cfg = SearchConfig(n_processes=c.get("n_processes", 0), strategy_weights=weights,
                       reinit_fraction=c.get("reinit_fraction", 0.4), patience=c.get("patience", 10),
                       master_seed=c.get("master_seed", 0),
                       forced_strategy=_strategy_index(c["strategy"]) if c.get("strategy") else None,
                       flip_enabled=bool(fm.get("enabled", False)), m_schemes=fm.get("m_schemes", 32),
                       flips_min=fm.get("flips_min", 1), flips_max=fm.get("flips_max", 16))
    comps = []
    for key in "uvw":
        cj = j["components"][key]
        subs = []
        for entry in cj["substitutions"]:
            if not isinstance(entry, list) or len(entry) != 3:
                raise ValueError("report json: substitutions must be [i, j, sign] triples")
            subs.append(tuple(entry))
        rec = _Rec(subs, cj["cost"], _strategy_index(cj.get("strategy", "greedy")), cj.get("seed", 0))
        comp = dict(record=rec, cost=cj["cost"], naive=cj["naive"], iterations=cj.get("iterations", 0))
        if "scheme_id" in cj:  # component_from_json (io.hpp:242)
            comp["scheme_id"] = cj["scheme_id"]
        comps.append(comp)
    rep = dict(scheme_digest=j["scheme_digest"], config=cfg, components=comps, total=j["total"],
               iterations=j["iterations"])
    if j.get("combined"):
        rep["combined"] = True
    if "scheme" in j:  # the carried (flipped) scheme (io.hpp:285-286)
        from .scheme import parse_scheme
        rep["scheme"] = parse_scheme(json.dumps(j["scheme"]))
    return rep


def combine_componentwise(reports):
    """Component-wise minimum across reports of one scheme (first minimum wins)."""
    if not reports:
        raise ValueError("combine: no reports")
    d0 = reports[0]["scheme_digest"]
    for r in reports:
        if r["scheme_digest"] != d0:
            raise ValueError("combine: reports refer to different schemes (%s vs %s)" % (d0, r["scheme_digest"]))
    if len(reports) == 1:
        return reports[0]
    comps = []
    for c in range(3):
        src = reports[0]
        for r in reports:
            if r["components"][c]["cost"] < src["components"][c]["cost"]:
                src = r
        comps.append(src["components"][c])
    out = dict(reports[0])
    out["components"] = comps
    out["total"] = sum(c["cost"] for c in comps)
    out["iterations"] = sum(c["iterations"] for c in comps)
    out["combined"] = True
    return out
