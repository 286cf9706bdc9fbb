"""Generates the scheme fixtures under tests/golden/schemes/ (SURVEY.md App. A).

Run here (needs the reference build oracle/_ref for digests / Brent checks and
for the libstdc++-dependent flipped schemes):  python tests/golden/make_fixtures.py

- strassen:   proj/tests/test_util.hpp:28-47 (digest 05ac287a032b2430)
- laderman:   Laderman 1976, as listed in SURVEY.md App. A (1575a9b2d4014af0)
- sxs:        Strassen (x) Strassen, 4x4x4:49 (7da4ac65bf44d830)
- sxl:        Strassen (x) Laderman, 6x6x6:161 (760577d1fad2ec32)
- sxs_border: S(x)S embedded in 5x5x5 with a naive border, r=110 (c41f03a3eef4d50f)
- naive555_f1000 / naive666_f3000: naive_scheme + random_flip chains from
  mt19937_64(12345) via the reference's own random_flip (libstdc++-dependent)
"""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import reference  # noqa: E402

OUT = os.path.join(HERE, "schemes")


def strassen():
    u = [[1, 0, 0, 1], [0, 0, 1, 1], [1, 0, 0, 0], [0, 0, 0, 1], [1, 1, 0, 0], [-1, 0, 1, 0], [0, 1, 0, -1]]
    v = [[1, 0, 0, 1], [1, 0, 0, 0], [0, 1, 0, -1], [-1, 0, 1, 0], [0, 0, 0, 1], [1, 1, 0, 0], [0, 0, 1, 1]]
    w = [[1, 0, 0, 1, -1, 0, 1], [0, 0, 1, 0, 1, 0, 0], [0, 1, 0, 1, 0, 0, 0], [1, -1, 1, 0, 0, 1, 0]]
    return dict(m=2, n=2, p=2, r=7, u=u, v=v, w=w)


def _lin(text, prefix, dim):
    """'a11+a12-a21' -> coefficient vector over (i,j), j fastest."""
    vec = [0] * (dim * dim)
    text = text.replace(" ", "")
    if text[0] not in "+-":
        text = "+" + text
    t = 0
    while t < len(text):
        sign = 1 if text[t] == "+" else -1
        assert text[t + 1] == prefix
        i, j = int(text[t + 2]) - 1, int(text[t + 3]) - 1
        vec[i * dim + j] = sign
        t += 4
    return vec


def laderman():
    prods = [
        ("a11+a12+a13-a21-a22-a32-a33", "b22"), ("a11-a21", "-b12+b22"),
        ("a22", "-b11+b12+b21-b22-b23-b31+b33"), ("-a11+a21+a22", "b11-b12+b22"),
        ("a21+a22", "-b11+b12"), ("a11", "b11"), ("-a11+a31+a32", "b11-b13+b23"),
        ("-a11+a31", "b13-b23"), ("a31+a32", "-b11+b13"), ("a11+a12+a13-a22-a23-a31-a32", "b23"),
        ("a32", "-b11+b13+b21-b22-b23-b31+b32"), ("-a13+a32+a33", "b22+b31-b32"),
        ("a13-a33", "b22-b32"), ("a13", "b31"), ("a32+a33", "-b31+b32"),
        ("-a13+a22+a23", "b23+b31-b33"), ("a13-a23", "b23-b33"), ("a22+a23", "-b31+b33"),
        ("a12", "b21"), ("a23", "b32"), ("a21", "b13"), ("a31", "b12"), ("a33", "b33"),
    ]
    outs = {
        (0, 0): [6, 14, 19], (0, 1): [1, 4, 5, 6, 12, 14, 15], (0, 2): [6, 7, 9, 10, 14, 16, 18],
        (1, 0): [2, 3, 4, 6, 14, 16, 17], (1, 1): [2, 4, 5, 6, 20], (1, 2): [14, 16, 17, 18, 21],
        (2, 0): [6, 7, 8, 11, 12, 13, 14], (2, 1): [12, 13, 14, 15, 22], (2, 2): [6, 7, 8, 9, 23],
    }
    u = [_lin(a, "a", 3) for a, _ in prods]
    v = [_lin(b, "b", 3) for _, b in prods]
    w = []
    for i in range(3):
        for k in range(3):
            row = [0] * 23
            for q in outs[(i, k)]:
                row[q - 1] = 1
            w.append(row)
    return dict(m=3, n=3, p=3, r=23, u=u, v=v, w=w)


def kron(A, B):
    """A (x) B: q = qa*rB + qb."""
    m, n, p, r = A["m"] * B["m"], A["n"] * B["n"], A["p"] * B["p"], A["r"] * B["r"]
    u = [[0] * (m * n) for _ in range(r)]
    v = [[0] * (n * p) for _ in range(r)]
    w = [[0] * r for _ in range(m * p)]
    for qa in range(A["r"]):
        for qb in range(B["r"]):
            q = qa * B["r"] + qb
            for i1 in range(A["m"]):
                for j1 in range(A["n"]):
                    for i2 in range(B["m"]):
                        for j2 in range(B["n"]):
                            u[q][(i1 * B["m"] + i2) * n + (j1 * B["n"] + j2)] = \
                                A["u"][qa][i1 * A["n"] + j1] * B["u"][qb][i2 * B["n"] + j2]
            for j1 in range(A["n"]):
                for k1 in range(A["p"]):
                    for j2 in range(B["n"]):
                        for k2 in range(B["p"]):
                            v[q][(j1 * B["n"] + j2) * p + (k1 * B["p"] + k2)] = \
                                A["v"][qa][j1 * A["p"] + k1] * B["v"][qb][j2 * B["p"] + k2]
            for i1 in range(A["m"]):
                for k1 in range(A["p"]):
                    for i2 in range(B["m"]):
                        for k2 in range(B["p"]):
                            w[(i1 * B["m"] + i2) * p + (k1 * B["p"] + k2)][q] = \
                                A["w"][i1 * A["p"] + k1][qa] * B["w"][i2 * B["p"] + k2][qb]
    return dict(m=m, n=n, p=p, r=r, u=u, v=v, w=w)


def border(S, size):
    """Embed S in size^3 and add a naive product a_ij*b_jk -> c_ik for every
    (i,j,k) with some index >= S's size, lexicographic."""
    sm = S["m"]
    N = size
    u, v, wcols = [], [], []
    for q in range(S["r"]):
        uu = [0] * (N * N)
        vv = [0] * (N * N)
        ww = [0] * (N * N)
        for i in range(sm):
            for j in range(sm):
                uu[i * N + j] = S["u"][q][i * sm + j]
                vv[i * N + j] = S["v"][q][i * sm + j]
                ww[i * N + j] = S["w"][i * sm + j][q]
        u.append(uu)
        v.append(vv)
        wcols.append(ww)
    for i in range(N):
        for j in range(N):
            for k in range(N):
                if i >= sm or j >= sm or k >= sm:
                    uu = [0] * (N * N)
                    vv = [0] * (N * N)
                    ww = [0] * (N * N)
                    uu[i * N + j] = 1
                    vv[j * N + k] = 1
                    ww[i * N + k] = 1
                    u.append(uu)
                    v.append(vv)
                    wcols.append(ww)
    r = len(u)
    w = [[wcols[q][row] for q in range(r)] for row in range(N * N)]
    return dict(m=N, n=N, p=N, r=r, u=u, v=v, w=w)


def to_json(s):
    # the reference's scheme_to_json layout (io.hpp:83-100) is not needed for
    # parsing; keep one row per line for readable diffs
    lines = ["{", ' "m": %d,' % s["m"], ' "n": %d,' % s["n"], ' "p": %d,' % s["p"], ' "r": %d,' % s["r"]]
    for key in ("u", "v", "w"):
        rows = ",\n".join("  " + json.dumps(row, separators=(",", ":")) for row in s[key])
        lines.append(' "%s": [\n%s\n ]%s' % (key, rows, "," if key != "w" else ""))
    lines.append("}")
    return "\n".join(lines) + "\n"


def flipped(m, flips, seed=12345):
    ref = reference()
    buf = C.create_string_buffer(1 << 24)
    n = C.c_int32()
    rc = ref.ref_flipped_naive_json(m, m, m, flips, seed, buf, len(buf), C.byref(n))
    assert rc == 0, ref.ref_last_error()
    return json.loads(buf.value.decode())


EXPECTED = {
    "strassen": "05ac287a032b2430",
    "laderman": "1575a9b2d4014af0",
    "sxs": "7da4ac65bf44d830",
    "sxl": "760577d1fad2ec32",
    "sxs_border": "c41f03a3eef4d50f",
}


def main():
    os.makedirs(OUT, exist_ok=True)
    S, L = strassen(), laderman()
    schemes = {
        "strassen": S,
        "laderman": L,
        "sxs": kron(S, S),
        "sxl": kron(S, L),
        "sxs_border": border(kron(S, S), 5),
        "naive555_f1000": flipped(5, 1000),
        "naive666_f3000": flipped(6, 3000),
    }
    ref = reference()
    index = {}
    for name, s in schemes.items():
        text = to_json(s)
        digest = C.create_string_buffer(17)
        naive = (C.c_int32 * 3)()
        valid = C.c_int32()
        rc = ref.ref_scheme_info(text.encode(), digest, naive, C.byref(valid))
        assert rc == 0, ref.ref_last_error()
        d = digest.value.decode()
        if name in EXPECTED:
            assert d == EXPECTED[name], (name, d, EXPECTED[name])
        assert valid.value == 1, name
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            f.write(text)
        index[name] = dict(digest=d, naive=list(naive), m=s["m"], n=s["n"], p=s["p"], r=s["r"])
        print(name, d, list(naive), sum(naive))
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
