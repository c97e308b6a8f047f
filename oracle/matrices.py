"""O2 -- coding matrices and the GF(2) bitmatrix lowering (TEST INFRASTRUCTURE ONLY).

Paper anchors
  * RS(n,p) encodes with an (n+p) x n matrix whose top is I_n ([Intro]).
  * Text construction: reduced form [I; M V^-1] of the (n+p) x n Vandermonde
    matrix with rows (1, a^i, (a^i)^2, ...), i = 1..n+p  ([Eval]).
  * The printed counts (#xor(P_enc) = 755) are reproduced only by the
    ISA-L-style matrix [I; R] with R[i][j] = (2^i)^j  (reading R1;
    the paper states it uses ISA-L's matrix).
  * Cauchy R[i][j] = inv((n+i) xor j) for BASELINE cfg1 (reading R2; the paper
    is silent on Cauchy matrices).
  * Decode: gather n surviving blocks, invert the n x n submatrix M of the
    coding matrix, D = M^-1 B ([Intro]).  Reading R4: survivors are
    the first n non-erased indices ascending, erasures 0-based; the goals are the
    erased blocks only -- erased data block e is row e of M^-1, erased parity
    block e is G[e] . M^-1.
  * x~ : byte -> 8x8 bitmatrix with x*y = B^-1(x~ . B(y)) ([Intro]);
    the matrix lowering applies x~ cell-wise.  Reading
    R3: B is LSB-first (bit k of a byte is row k), so column k of x~ is
    B(x * 2^k) and entry (r, k) is bit r of x * 2^k.
"""
import numpy as np

from .gf256 import gf_mul, gf_inv, gf_pow

KINDS = ("isal", "sysvand", "cauchy")


def identity(n):
    return [[1 if i == j else 0 for j in range(n)] for i in range(n)]


def gf_matmul(a, b):
    """Plain triple loop over GF(2^8): sum (XOR) of products."""
    rows, inner, cols = len(a), len(b), len(b[0]) if b else 0
    assert all(len(r) == inner for r in a)
    out = [[0] * cols for _ in range(rows)]
    for i in range(rows):
        for j in range(cols):
            s = 0
            for k in range(inner):
                s ^= gf_mul(a[i][k], b[k][j])
            out[i][j] = s
    return out


def gf_invert(m):
    """Gauss-Jordan over GF(2^8) with first-nonzero pivoting.

    Raises ValueError("singular") when no pivot exists.
    """
    n = len(m)
    a = [list(r) + e for r, e in zip(m, identity(n))]
    for col in range(n):
        piv = next((r for r in range(col, n) if a[r][col] != 0), None)
        if piv is None:
            raise ValueError("singular")
        a[col], a[piv] = a[piv], a[col]
        inv = gf_inv(a[col][col])
        a[col] = [gf_mul(inv, x) for x in a[col]]
        for r in range(n):
            if r != col and a[r][col] != 0:
                f = a[r][col]
                a[r] = [x ^ gf_mul(f, y) for x, y in zip(a[r], a[col])]
    return [row[n:] for row in a]


def vandermonde(n, p):
    """(n+p) x n, row i (i = 1..n+p) = (1, a^i, (a^i)^2, ...), a = 0x02.

    Pinned through coding_matrix(kind="sysvand"): M V^-1 equals the Lagrange closed form
    L_j(y_k) computed without Gauss-Jordan and without this module's field tables
    (tests/test_oracle_gf.py::test_sysvand_equals_lagrange_closed_form, RS(2,1) by hand).
    """
    rows = []
    for i in range(1, n + p + 1):
        ai = gf_pow(2, i)
        rows.append([gf_pow(ai, j) for j in range(n)])
    return rows


def coding_matrix(n, p, kind="isal"):
    """(n+p) x n systematic coding matrix [I_n; R] as a list of rows."""
    if kind == "isal":
        r = [[gf_pow(gf_pow(2, i), j) for j in range(n)] for i in range(p)]
    elif kind == "sysvand":
        v = vandermonde(n, p)
        top, bottom = v[:n], v[n:]
        r = gf_matmul(bottom, gf_invert(top))          # M V^-1
    elif kind == "cauchy":
        r = [[gf_inv((n + i) ^ j) for j in range(n)] for i in range(p)]
    else:
        raise ValueError(kind)
    return identity(n) + r


def decode_rows(g, n, erased):
    """Reading R4 of P:526-530.  Returns (survivors, goal_rows).

    survivors: the first n non-erased block indices, ascending.
    goal_rows: one GF row (length n) per erased index, in ascending order,
    expressing that block as a combination of the survivors.
    """
    total = len(g)
    erased = sorted(set(erased))
    if any(e < 0 or e >= total for e in erased):
        raise ValueError("erasure index out of range")
    alive = [i for i in range(total) if i not in erased]
    if len(alive) < n:
        raise ValueError("unrecoverable")
    survivors = alive[:n]
    minv = gf_invert([g[i] for i in survivors])
    rows = []
    for e in erased:
        if e < n:
            rows.append(list(minv[e]))
        else:
            rows.append(gf_matmul([g[e]], minv)[0])
    return survivors, rows


def decode_rows_from(g, n, erased, survivors):
    """P:526-530 with an explicit survivor set (any n non-erased blocks of an MDS code).

    Input block j of the decode is block survivors[j]; M = those rows of g, and the goal
    rows are as in decode_rows: erased data block e -> row e of M^-1, erased parity block
    e -> g[e] . M^-1, erased indices ascending.
    """
    total = len(g)
    erased = sorted(set(erased))
    survivors = list(survivors)
    if len(survivors) != n or len(set(survivors)) != n:
        raise ValueError("need n distinct survivors")
    if any(s < 0 or s >= total or s in erased for s in survivors):
        raise ValueError("bad survivor index")
    if any(e < 0 or e >= total for e in erased):
        raise ValueError("erasure index out of range")
    minv = gf_invert([g[i] for i in survivors])
    rows = []
    for e in erased:
        if e < n:
            rows.append(list(minv[e]))
        else:
            rows.append(gf_matmul([g[e]], minv)[0])
    return rows


def tilde(x):
    """8x8 GF(2) matrix of multiply-by-x: entry (r, k) = bit r of x * 2^k."""
    t = np.zeros((8, 8), dtype=np.uint8)
    for k in range(8):
        col = gf_mul(x, 1 << k)
        for r in range(8):
            t[r, k] = (col >> r) & 1
    return t


def to_bitmatrix(rows):
    """Cell-wise x~: (8a) x (8b) matrix of 0/1 bytes."""
    a, b = len(rows), len(rows[0])
    out = np.zeros((8 * a, 8 * b), dtype=np.uint8)
    for i in range(a):
        for j in range(b):
            out[8 * i:8 * i + 8, 8 * j:8 * j + 8] = tilde(rows[i][j])
    return out
