"""Pins for oracle O1/O2 (GF(2^8), matrices, x~) against the paper and the mathematics."""
import itertools
import random

import numpy as np
import pytest

from oracle import gf256 as gf
from oracle import matrices as mx
from oracle.slp import rows_to_sets


def test_poly_reduction_closed_form():
    # x * x^7 = x^8 = x^4 + x^3 + x^2 + 1 mod the ISA-L polynomial
    assert gf.gf_mul(0x02, 0x80) == 0x1D
    assert gf.gf_mul(0x80, 0x02) == 0x1D


def test_field_axioms():
    rnd = random.Random(0)
    for a in range(256):
        assert gf.gf_mul(1, a) == a and gf.gf_mul(a, 0) == 0
    for a, b in itertools.product(range(0, 256, 7), range(256)):
        assert gf.gf_mul(a, b) == gf.gf_mul(b, a)
    for _ in range(3000):
        a, b, c = (rnd.randrange(256) for _ in range(3))
        assert gf.gf_mul(a, gf.gf_mul(b, c)) == gf.gf_mul(gf.gf_mul(a, b), c)
        assert gf.gf_mul(a, b ^ c) == gf.gf_mul(a, b) ^ gf.gf_mul(a, c)


def test_alpha_is_primitive_and_inverses():
    # "alpha is a primitive element": 2 generates the 255-element group.
    seen, x = set(), 1
    for _ in range(255):
        x = gf.gf_mul(x, 2)
        seen.add(x)
    assert x == 1 and len(seen) == 255
    for a in range(1, 256):
        assert gf.gf_mul(a, gf.gf_inv(a)) == 1
    with pytest.raises(ZeroDivisionError):
        gf.gf_inv(0)


def test_mul_table_matches_definition():
    rnd = random.Random(1)
    for _ in range(2000):
        a, b = rnd.randrange(256), rnd.randrange(256)
        assert gf.MUL[a, b] == gf.gf_mul(a, b)


def test_tilde_property_exhaustive():
    # x * y = B^-1(x~ . B(y)) for all x, y, LSB-first B (reading R3)
    for x in range(256):
        t = mx.tilde(x).astype(np.int64)
        for y in range(256):
            by = np.array([(y >> k) & 1 for k in range(8)])
            z = (t @ by) % 2
            assert sum(int(z[r]) << r for r in range(8)) == gf.gf_mul(x, y)


def test_tilde_ring_homomorphism():
    rnd = random.Random(2)
    assert (mx.tilde(1) == np.eye(8, dtype=np.uint8)).all()
    assert not mx.tilde(0).any()
    for _ in range(300):
        x, y = rnd.randrange(256), rnd.randrange(256)
        assert ((mx.tilde(x).astype(int) @ mx.tilde(y).astype(int)) % 2
                == mx.tilde(gf.gf_mul(x, y))).all()
        assert (mx.tilde(x) ^ mx.tilde(y) == mx.tilde(x ^ y)).all()


def test_invert():
    rnd = random.Random(3)
    for n in (1, 2, 5, 10):
        while True:
            m = [[rnd.randrange(256) for _ in range(n)] for _ in range(n)]
            try:
                inv = mx.gf_invert(m)
                break
            except ValueError:
                continue
        assert mx.gf_matmul(m, inv) == mx.identity(n)
        assert mx.gf_matmul(inv, m) == mx.identity(n)
    with pytest.raises(ValueError):
        mx.gf_invert([[1, 2], [2, 4]])   # row 2 = 2 * row 1


def _xor_count_of_rows(rows):
    bits = mx.to_bitmatrix(rows)
    return int(sum(int(r.sum()) - 1 for r in bits))


def test_printed_Penc_counts():
    # #xor(P_enc) = 755, #M = 2265 = 3 * 755, NVar = 32 ([Eval]).
    # Pins the matrix family (reading R1: [I; 2^{ij}]) and the x~ lowering.
    g = mx.coding_matrix(10, 4, "isal")
    bits = mx.to_bitmatrix(g[10:])
    assert bits.shape == (32, 80)
    x = _xor_count_of_rows(g[10:])
    assert x == 755
    assert 3 * x == 2265
    assert len(bits) == 32


def test_printed_Pdec_counts():
    # Decode with {2,4,5,6} erased: #xor 1368, #M 4104, NVar 32.
    # Pins the decode reading R4 (0-based, survivors ascending, erased goals only).
    g = mx.coding_matrix(10, 4, "isal")
    surv, rows = mx.decode_rows(g, 10, [2, 4, 5, 6])
    assert surv == [0, 1, 3, 7, 8, 9, 10, 11, 12, 13]
    x = _xor_count_of_rows(rows)
    assert x == 1368 and 3 * x == 4104 and 8 * len(rows) == 32


def test_sysvand_is_systematic_and_text_construction():
    # Text construction: top block identity after reduction.
    g = mx.coding_matrix(10, 4, "sysvand")
    assert g[:10] == mx.identity(10)
    v = mx.vandermonde(10, 4)
    # [I; M V^-1] . V_top = [V_top; M]: reduction is a change of basis.
    assert mx.gf_matmul(g, v[:10]) == v


def _mul_long_division(a, b):
    """a*b mod x^8+x^4+x^3+x^2+1 by carry-less product then long division;
    no tables and no oracle code, so the Lagrange pin below is independent of gf256."""
    prod = 0
    for k in range(8):
        if (b >> k) & 1:
            prod ^= a << k
    for deg in range(14, 7, -1):
        if (prod >> deg) & 1:
            prod ^= 0x11D << (deg - 8)
    return prod


def _inv_by_search(a):
    return next(x for x in range(1, 256) if _mul_long_division(a, x) == 1)


def _alpha_pow(e):
    x = 1
    for _ in range(e):
        x = _mul_long_division(x, 2)
    return x


def _lagrange_rows(n, p, first_exp=1, nodes=None):
    """Rows of M V^-1 in closed form, without Gauss-Jordan.

    V stacks rows (1, x, x^2, ..., x^{n-1}) at the nodes x_i = alpha^{first_exp + i},
    i = 0..n+p-1 (or the given nodes); the top n nodes form V, the last p form M.  Row
    (1, y, ..., y^{n-1}) of M is the interpolation of the monomials at y:
    sum_j L_j(y) * (row of node x_j), so
    (M V^-1)[k][j] = L_j(y_k) = prod_{m != j} (y_k - x_m) / (x_j - x_m), with - = xor.
    """
    xs = nodes if nodes is not None else [_alpha_pow(first_exp + i) for i in range(n + p)]
    top, ys = xs[:n], xs[n:]
    rows = []
    for y in ys:
        row = []
        for j in range(n):
            num, den = 1, 1
            for m in range(n):
                if m != j:
                    num = _mul_long_division(num, y ^ top[m])
                    den = _mul_long_division(den, top[j] ^ top[m])
            row.append(_mul_long_division(num, _inv_by_search(den)))
        rows.append(row)
    return rows


@pytest.mark.parametrize("n,p", [(2, 1), (4, 2), (10, 4), (20, 4)])
def test_sysvand_equals_lagrange_closed_form(n, p):
    # The text's Vandermonde has rows i = 1..n+p with node alpha^i (the first
    # row is (1, alpha, ..., alpha^9), the last (1, alpha^14, ...)), reduced to [I; M V^-1]
    # (P:1398-1402).  The closed form replaces Gauss-Jordan and the matrix product.
    g = mx.coding_matrix(n, p, "sysvand")
    want = _lagrange_rows(n, p)
    assert g[n:] == want
    # Shifting every node by the same power of alpha scales column j of V by alpha^{sj} on
    # both V and M, which cancels in M V^-1: nodes alpha^0..alpha^{n+p-1} give the SAME
    # matrix (so that "mistake" is not one).  Mistakes that do change it:
    assert _lagrange_rows(n, p, first_exp=0) == want
    #  * integer nodes 1..n+p instead of powers of alpha,
    assert _lagrange_rows(n, p, nodes=list(range(1, n + p + 1))) != want
    #  * parity rows taken from the top of V instead of the bottom (M = first p rows),
    xs = [_alpha_pow(1 + i) for i in range(n + p)]
    assert _lagrange_rows(n, p, nodes=xs[p:] + xs[:p]) != want
    #  * rows (x, x^2, ..., x^n) (exponents from 1): row k of M V^-1 scales by y_k / x_j.
    shifted = [[_mul_long_division(_mul_long_division(v, xs[n + k]), _inv_by_search(xs[j]))
                for j, v in enumerate(row)] for k, row in enumerate(want)]
    assert shifted != want
    # each row of M V^-1 interpolates the constant 1: sum_j L_j(y) = 1
    for row in want:
        s = 0
        for v in row:
            s ^= v
        assert s == 1


def test_sysvand_rs21_by_hand():
    # RS(2,1): nodes x1 = alpha = 2, x2 = alpha^2 = 4, y = alpha^3 = 8.
    # L_1(8) = (8+4)/(2+4) = 0x0C/0x06 = 2 (since 2*6 = 0x0C, no reduction);
    # L_2(8) = (8+2)/(4+2) = 0x0A/0x06 = 3 (since 3*6 = 0x0A: 6 ^ 0x0C).
    g = mx.coding_matrix(2, 1, "sysvand")
    assert g == [[1, 0], [0, 1], [2, 3]]


def test_isal_raid5_row_and_values():
    g = mx.coding_matrix(10, 4, "isal")
    assert g[10] == [1] * 10                      # (2^0)^j = 1
    assert g[11][:3] == [1, 2, 4] and g[11][8] == gf.gf_mul(0x80, 2)


@pytest.mark.parametrize("n,p,kind", [(4, 2, "cauchy"), (10, 4, "isal"), (10, 4, "sysvand"),
                                      (8, 3, "isal"), (10, 2, "isal")])
def test_mds_every_pattern(n, p, kind):
    # "any square submatrix ... is invertible" => any n of n+p blocks recover D
    g = mx.coding_matrix(n, p, kind)
    for e in range(1, p + 1):
        for erased in itertools.combinations(range(n + p), e):
            surv, rows = mx.decode_rows(g, n, list(erased))
            assert len(rows) == e
            # re-encoding the recovered rows against the survivors reproduces G rows
            m = [g[i] for i in surv]
            for k, ei in enumerate(erased):
                assert mx.gf_matmul([rows[k]], m)[0] == g[ei]


def test_decode_special_cases():
    g = mx.coding_matrix(10, 4, "isal")
    # erasing only parity: M = I, goal rows = encode rows
    surv, rows = mx.decode_rows(g, 10, [10, 11, 12, 13])
    assert surv == list(range(10)) and rows == g[10:]
    # single data erasure: RAID-5 recovery D_j = P0 xor (xor of other D)
    for j in range(10):
        surv, rows = mx.decode_rows(g, 10, [j])
        assert surv == [i for i in range(11) if i != j]
        assert rows == [[1] * 10]
    # too many erasures
    with pytest.raises(ValueError):
        mx.decode_rows(g, 10, [0, 1, 2, 3, 4])


def test_bitmatrix_rows_to_sets():
    bits = mx.to_bitmatrix([[1, 0], [0, 1]])
    sets = rows_to_sets(bits)
    assert sets == [1 << i for i in range(16)]


def test_mds_rs20_4_every_pattern():
    # BASELINE cfg5: RS(20,4) [I; 2^(ij)] recovers from every one of the 10,626 4-erasure
    # patterns; the recovered rows re-encode to G's rows
    n, p = 20, 4
    g = mx.coding_matrix(n, p, "isal")
    pats = list(itertools.combinations(range(n + p), p))
    assert len(pats) == 10626
    for erased in pats:
        surv, rows = mx.decode_rows(g, n, list(erased))
        m = [g[i] for i in surv]
        for k, ei in enumerate(erased):
            assert mx.gf_matmul([rows[k]], m)[0] == g[ei]
