"""Pins for oracle O3/O4 (RS over the strip layout) against textbook RS and brute force."""
import itertools

import numpy as np
import pytest

from oracle import matrices as mx
from oracle import rs
from synth import stripe_data


def poly_mul_no_table(a, b):
    """Independent test-side product: carry-less multiply, then reduce by long division."""
    prod = 0
    for i in range(8):
        if (b >> i) & 1:
            prod ^= a << i
    for deg in range(14, 7, -1):
        if (prod >> deg) & 1:
            prod ^= 0x11D << (deg - 8)
    return prod


def brute_force_strip_rs(rows, blocks):
    """Per (offset, bit) scalar loops: gather a byte, multiply without tables, scatter."""
    n, B = blocks.shape
    S = B // 8
    out = np.zeros((len(rows), B), dtype=np.uint8)
    for o in range(S):
        for b in range(8):
            xs = []
            for j in range(n):
                xs.append(sum(((int(blocks[j, k * S + o]) >> b) & 1) << k for k in range(8)))
            for i, row in enumerate(rows):
                y = 0
                for j in range(n):
                    y ^= poly_mul_no_table(row[j], xs[j])
                for r in range(8):
                    if (y >> r) & 1:
                        out[i, r * S + o] |= 1 << b
    return out


@pytest.mark.parametrize("n,p,kind,B", [(4, 2, "cauchy", 16), (4, 2, "cauchy", 8),
                                        (10, 4, "isal", 24), (3, 3, "sysvand", 16)])
def test_three_paths_agree_tiny(n, p, kind, B):
    rng = np.random.default_rng(n * 100 + B)
    g = mx.coding_matrix(n, p, kind)
    data = rng.integers(0, 256, size=(n, B), dtype=np.uint8)
    a = rs.encode(g, n, data)
    b = rs.bitmatrix_apply(mx.to_bitmatrix(g[n:]), data)
    c = brute_force_strip_rs(g[n:], data)
    assert (a == b).all() and (a == c).all()


def test_bitplane_reduction_to_bytewise_rs():
    # If strip (j,k) byte o bit b = bit k of data byte 8o+b, the de-transposed
    # output equals textbook byte-wise RS y_i[t] = sum_j R_ij d_j[t].
    n, p, S = 4, 2, 8
    g = mx.coding_matrix(n, p, "cauchy")
    rng = np.random.default_rng(5)
    d = rng.integers(0, 256, size=(n, 8 * S), dtype=np.uint8)      # byte data
    blocks = np.zeros((n, 8 * S), dtype=np.uint8)
    for j in range(n):
        for t in range(8 * S):
            o, b = divmod(t, 8)
            for k in range(8):
                if (d[j, t] >> k) & 1:
                    blocks[j, k * S + o] |= 1 << b
    out = rs.encode(g, n, blocks)
    for i in range(p):
        for t in range(8 * S):
            o, b = divmod(t, 8)
            y = sum(((int(out[i, k * S + o]) >> b) & 1) << k for k in range(8))
            want = 0
            for j in range(n):
                want ^= poly_mul_no_table(g[n + i][j], int(d[j, t]))
            assert y == want


def test_bytewise_rs_brute_force_and_bitplanes():
    # bytewise_apply vs per-byte polynomial multiply without tables, and vs the strip-layout
    # oracle applied to the bit-planes of the bytes
    rng = np.random.default_rng(17)
    g = mx.coding_matrix(5, 3, "isal")
    d = rng.integers(0, 256, size=(5, 40), dtype=np.uint8)
    out = rs.bytewise_apply(g[5:], d)
    for i in range(3):
        for t in range(40):
            want = 0
            for j in range(5):
                want ^= poly_mul_no_table(g[5 + i][j], int(d[j, t]))
            assert out[i, t] == want
    assert (rs.bytewise_apply([[1] * 5], d)[0] == np.bitwise_xor.reduce(d, axis=0)).all()
    # bit-plane view: strip k of block j carries bit k of every byte (B/8 = 40/8 bytes each)
    planes = np.zeros((5, 8 * 5), dtype=np.uint8)  # 40 bits per plane = 5 bytes per strip
    for j in range(5):
        for k in range(8):
            bits = (d[j] >> k) & 1
            planes[j, 5 * k:5 * k + 5] = np.packbits(bits, bitorder="little")
    strip_out = rs.encode(g, 5, planes)
    for i in range(3):
        for k in range(8):
            bits = np.unpackbits(strip_out[i, 5 * k:5 * k + 5], bitorder="little")
            assert (bits == ((out[i] >> k) & 1)).all()


def test_raid5_parity0_and_linearity():
    g = mx.coding_matrix(10, 4, "isal")
    d1 = stripe_data(7, 0, 10, 256)
    d2 = stripe_data(7, 1, 10, 256)
    p1 = rs.encode(g, 10, d1)
    assert (p1[0] == np.bitwise_xor.reduce(d1, axis=0)).all()
    assert (rs.encode(g, 10, d1 ^ d2) == p1 ^ rs.encode(g, 10, d2)).all()
    assert not rs.encode(g, 10, np.zeros_like(d1)).any()


@pytest.mark.parametrize("n,p,kind", [(4, 2, "cauchy"), (10, 4, "isal")])
def test_roundtrip_all_patterns(n, p, kind):
    g = mx.coding_matrix(n, p, kind)
    data = stripe_data(11, 3, n, 64)
    blocks = np.concatenate([data, rs.encode(g, n, data)])
    pats = list(itertools.combinations(range(n + p), p))
    if len(pats) > 120:
        pats = pats[::9]
    for erased in pats:
        surv, rows = mx.decode_rows(g, n, list(erased))
        rec = rs.decode(rows, blocks[surv])
        assert (rec == blocks[list(erased)]).all()


def test_one_hot_columns():
    # feeding strip c = 0xFF.., all others 0, makes output strip r = 0xFF.. iff bit (r, c) set
    g = mx.coding_matrix(4, 2, "cauchy")
    bits = mx.to_bitmatrix(g[4:])
    for c in range(32):
        blocks = np.zeros((4, 16), dtype=np.uint8)
        j, k = divmod(c, 8)
        blocks[j, 2 * k:2 * k + 2] = 0xFF
        out = rs.encode(g, 4, blocks).reshape(16, 2)
        for r in range(16):
            assert (out[r] == (0xFF if bits[r, c] else 0)).all()


def test_rejects_ragged():
    with pytest.raises(ValueError):
        rs.apply_rows([[1]], np.zeros((1, 12), dtype=np.uint8))
    assert rs.apply_rows([[1]], np.zeros((1, 0), dtype=np.uint8)).shape == (1, 0)


# ---- decode over an explicit survivor set (cross-GPU decode reads local survivors first) ----

def test_decode_from_any_survivor_set_rs42_exhaustive():
    # MDS: ANY n of the n+p blocks recover the rest; every erasure pattern of
    # size <= p and every n-subset of the non-erased blocks, in a scrambled column order
    n, p = 4, 2
    g = mx.coding_matrix(n, p, "cauchy")
    data = stripe_data(12, 0, n, 32)
    blocks = np.concatenate([data, rs.encode(g, n, data)])
    rng = np.random.default_rng(5)
    cases = 0
    for ne in range(0, p + 1):
        for erased in itertools.combinations(range(n + p), ne):
            alive = [i for i in range(n + p) if i not in erased]
            for surv in itertools.combinations(alive, n):
                surv = list(rng.permutation(surv))
                rows = mx.decode_rows_from(g, n, list(erased), surv)
                assert (rs.decode(rows, blocks[surv]) == blocks[list(erased)]).all()
                cases += 1
    assert cases == 15 + 6 * 5 + 15 * 1   # 0, 1 and 2 erasures: C(6,4), 6 C(5,4), C(6,2)


def test_decode_from_first_n_equals_decode_rows():
    g = mx.coding_matrix(10, 4, "isal")
    for erased in ([2, 4, 5, 6], [0, 13], [11], [0, 1, 2, 3]):
        surv, rows = mx.decode_rows(g, 10, erased)
        assert mx.decode_rows_from(g, 10, erased, surv) == rows


def test_decode_from_raid5_closed_form():
    # [I; 2^ij]: erase data block j, read the other data blocks and parity 0 -> D_j is their
    # plain XOR, i.e. every coefficient is 1 whatever the column order
    n, p = 10, 4
    g = mx.coding_matrix(n, p, "isal")
    for j in (0, 6, 9):
        surv = [n] + [i for i in range(n) if i != j][::-1]
        assert mx.decode_rows_from(g, n, [j], surv) == [[1] * n]


def test_decode_from_rejects_bad_survivors():
    g = mx.coding_matrix(4, 2, "cauchy")
    with pytest.raises(ValueError):
        mx.decode_rows_from(g, 4, [0], [0, 1, 2, 3])      # an erased survivor
    with pytest.raises(ValueError):
        mx.decode_rows_from(g, 4, [0], [1, 1, 2, 3])      # duplicate
    with pytest.raises(ValueError):
        mx.decode_rows_from(g, 4, [0], [1, 2, 3])         # too few
