"""Host-side scheme model: the loader side of the path (no GPU work here).

Mirrors the reference's scheme JSON wire format and system extraction so that
Python callers feed the C ABI exactly what optimize_scheme would:
  - parse_scheme     io.hpp:65-81 (with detail::parse_tensor range checks, 22-50)
  - extract_systems  scheme.hpp:142-157 (E_U: r x mn, E_V: r x np, E_W: mp x r)
  - naive_cost       linear_system.hpp:193-199
  - scheme_digest    parallel_search.hpp:276-292 (FNV-1a-64 over int64 LE fields)
  - verify_brent     scheme.hpp:68-95 (exact integer Brent check)
"""
import json


class SchemeError(ValueError):
    """terncse::error raised by the scheme loader / checks."""


def _tensor(j, name, rows, cols):
    if name not in j or not isinstance(j[name], list):
        raise SchemeError('scheme json: missing tensor "%s"' % name)
    t = j[name]
    if len(t) != rows:
        raise SchemeError("scheme json: tensor %s has %d rows, expected %d" % (name, len(t), rows))
    out = []
    for r, row in enumerate(t):
        if not isinstance(row, list) or len(row) != cols:
            raise SchemeError("scheme json: tensor %s row %d must hold %d integers" % (name, r, cols))
        for c, v in enumerate(row):
            if not isinstance(v, int) or isinstance(v, bool):
                raise SchemeError("scheme json: non-integer coefficient at %s[%d][%d]" % (name, r, c))
            if v < -1 or v > 1:
                raise SchemeError("scheme json: coefficient %d out of range at %s[%d][%d]" % (v, name, r, c))
        out.append(list(row))
    return out


def parse_scheme(text):
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise SchemeError("scheme json: %s" % e) from None
    dims = {}
    for key in ("m", "n", "p", "r"):
        if key not in j or not isinstance(j[key], int):
            raise SchemeError('scheme json: missing integer field "%s"' % key)
        if j[key] < 1 or j[key] > 1 << 20:
            raise SchemeError('scheme json: field "%s" must be a positive integer' % key)
        dims[key] = j[key]
    m, n, p, r = dims["m"], dims["n"], dims["p"], dims["r"]
    return dict(m=m, n=n, p=p, r=r, u=_tensor(j, "u", r, m * n), v=_tensor(j, "v", r, n * p),
                w=_tensor(j, "w", m * p, r))


def load_scheme(path):
    with open(path) as f:
        return parse_scheme(f.read())


def extract_systems(s):
    """[(n_x, rows)] for U, V, W; rows are signed 1-based ids in column order."""
    def rows_of(t):
        return [[(c + 1) if x > 0 else -(c + 1) for c, x in enumerate(row) if x != 0] for row in t]

    return [(s["m"] * s["n"], rows_of(s["u"])), (s["n"] * s["p"], rows_of(s["v"])), (s["r"], rows_of(s["w"]))]


def naive_cost(rows):
    return sum(len(r) - 1 for r in rows if r)


def scheme_digest(s):
    h = 0xCBF29CE484222325
    mask = 0xFFFFFFFFFFFFFFFF

    def feed(value):
        nonlocal h
        v = value & mask
        for b in range(8):
            h ^= (v >> (8 * b)) & 0xFF
            h = (h * 0x100000001B3) & mask

    for key in ("m", "n", "p", "r"):
        feed(s[key])
    for key in ("u", "v", "w"):
        for row in s[key]:
            for x in row:
                feed(x)
    return "%016x" % h


def verify_brent(s):
    """(valid, first_violation) — exact Brent identities (scheme.hpp:68-95)."""
    m, n, p, r = s["m"], s["n"], s["p"], s["r"]
    u, v, w = s["u"], s["v"], s["w"]
    for i in range(m):
        for j in range(n):
            for k in range(n):
                for l in range(p):
                    for i2 in range(m):
                        for j2 in range(p):
                            uc, vc, wr = i * n + j, k * p + l, i2 * p + j2
                            tot = sum(u[q][uc] * v[q][vc] * w[wr][q] for q in range(r)
                                      if u[q][uc] and v[q][vc] and w[wr][q])
                            want = 1 if (j == k and i == i2 and l == j2) else 0
                            if tot != want:
                                return False, "brent(%d,%d,%d,%d,%d,%d)" % (i, j, k, l, i2, j2)
    return True, None
