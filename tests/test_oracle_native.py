"""Pins for the C oracle (oracle/rs_oracle.c via oracle/native.py) -- CPU only.

The C oracle is what verifies every stripe of the full-size workloads and what bench.py times
as the CPU baseline, so it is pinned to things other than itself: the field definition, the
x~ lowering against multiplication (exhaustive), the numpy oracle O3/O4 apply_rows -- a
table-driven byte RS on the bit-transposed view, a different formulation from the C oracle's
naive bitmatrix XOR product, itself pinned to the paper's counts, closed forms and brute force
in test_oracle_rs.py / test_oracle_gf.py -- the synth generator, and the RAID-5 closed form.
"""
import itertools
import random

import numpy as np
import pytest

import synth
from oracle import gf256 as gf
from oracle import matrices as mx
from oracle import native as nat
from oracle import rs


def test_field_matches_definition_exhaustively():
    for a in range(256):
        for b in range(0, 256, 3):
            assert nat.lib().oracle_gf_mul(a, b) == gf.gf_mul(a, b)
    assert nat.lib().oracle_gf_mul(0x02, 0x80) == 0x1D


def test_tilde_is_multiplication_exhaustively():
    # x~ (reading R3): c * y = B^-1(x~(c) . B(y)) for every pair, and x~(1) = I
    t = nat.lib().oracle_tilde_bit
    for c in range(256):
        m = np.array([[t(c, r, k) for k in range(8)] for r in range(8)], dtype=np.int64)
        if c == 1:
            assert (m == np.eye(8, dtype=np.int64)).all()
        for y in range(256):
            by = np.array([(y >> k) & 1 for k in range(8)])
            z = (m @ by) % 2
            assert sum(int(z[r]) << r for r in range(8)) == gf.gf_mul(c, y)


def test_fill_matches_synth():
    for seed, s, nb, B in [(2, 0, 10, 64), (3, 777, 14, 256), (5, 8191, 20, 8), (9, 262143, 2, 16)]:
        assert (nat.fill(seed, s, nb, B) == synth.stripe_data(seed, s, nb, B)).all()


@pytest.mark.parametrize("n,p,kind,B", [(4, 2, "cauchy", 8), (4, 2, "cauchy", 64), (10, 4, "isal", 128),
                                        (10, 4, "sysvand", 24), (20, 4, "isal", 40), (3, 3, "sysvand", 16)])
def test_apply_rows_equals_numpy_oracle(n, p, kind, B):
    g = mx.coding_matrix(n, p, kind)
    data = synth.stripe_data(11, 3, n, B)
    assert (nat.apply_rows(g[n:], data) == rs.apply_rows(g[n:], data)).all()
    # and the decode rows of a few patterns on the codeword
    blocks = np.concatenate([data, rs.encode(g, n, data)])
    for er in itertools.islice(itertools.combinations(range(n + p), p), 0, None, 97):
        surv, rows = mx.decode_rows(g, n, list(er))
        got = nat.apply_rows(rows, blocks[surv])
        assert (got == rs.decode(rows, blocks[surv])).all()
        assert (got == blocks[list(er)]).all()


def test_apply_rows_raid5_and_bitmatrix():
    # closed form: parity row 0 of [I; 2^ij] is the XOR of the data blocks (x~(1) = I)
    n, p, B = 10, 4, 512
    g = mx.coding_matrix(n, p, "isal")
    data = synth.stripe_data(7, 1, n, B)
    par = nat.apply_rows(g[n:], data)
    assert (par[0] == np.bitwise_xor.reduce(data, axis=0)).all()
    # and the GF(2) bitmatrix definition on the same strips
    assert (par == rs.bitmatrix_apply(mx.to_bitmatrix(g[n:]), data)).all()


def test_check_detects_single_bit_flips():
    n, p, B, S = 10, 4, 256, 12
    g = np.array(mx.coding_matrix(n, p), dtype=np.uint8)
    got = np.stack([rs.encode(g.tolist(), n, synth.stripe_data(4, 100 + s, n, B)) for s in range(S)])
    assert len(nat.check_apply(g[n:], 4, 100, got, threads=3)) == 0
    got[5, 2, 17] ^= 0x10
    got[11, 0, 0] ^= 0x01
    assert list(nat.check_apply(g[n:], 4, 100, got, threads=3)) == [5, 11]
    # codeword mode: erased blocks of the codeword, data and parity mixed
    er = np.array([sorted(synth.erasure_pattern(4, 100 + s, n + p, 4)) for s in range(S)], dtype=np.int32)
    got[5, 2, 17] ^= 0x10                                        # undo the flips
    got[11, 0, 0] ^= 0x01
    cw = [np.concatenate([synth.stripe_data(4, 100 + s, n, B), got[s]]) for s in range(S)]
    rec = np.stack([cw[s][er[s]] for s in range(S)])
    assert len(nat.check_codeword(g[n:], n, 4, 100, er, rec, threads=4)) == 0
    rec[3, 1, 5] ^= 0x80
    assert list(nat.check_codeword(g[n:], n, 4, 100, er, rec, threads=4)) == [3]


def test_apply_each_matches_per_stripe():
    n, p, B, S = 6, 3, 64, 9
    g = mx.coding_matrix(n, p, "sysvand")
    x = np.stack([synth.stripe_data(8, s, n, B) for s in range(S)])
    out = nat.apply_each(np.array(g[n:], dtype=np.uint8), x, threads=4)
    for s in range(S):
        assert (out[s] == rs.apply_rows(g[n:], x[s])).all()
    # a matrix per stripe (decode rows of per-stripe patterns), and the byte-wise product
    rows = [mx.decode_rows(g, n, synth.erasure_pattern(8, s, n + p, 2))[1] for s in range(S)]
    out = nat.apply_each(np.array(rows, dtype=np.uint8), x, threads=3)
    byw = nat.apply_each(np.array(rows, dtype=np.uint8), x, threads=2, bytewise=True)
    for s in range(S):
        assert (out[s] == rs.apply_rows(rows[s], x[s])).all()
        assert (byw[s] == rs.bytewise_apply(rows[s], x[s])).all()


def test_check_bytewise_matches_numpy_oracle():
    n, p, B, S = 10, 4, 96, 5
    g = mx.coding_matrix(n, p, "cauchy" if n == 4 else "isal")
    got = np.stack([rs.bytewise_apply(g[n:], synth.stripe_data(6, 20 + s, n, B)) for s in range(S)])
    R = np.array(g[n:], dtype=np.uint8)
    assert len(nat.check_bytewise(R, 6, 20, got, threads=2)) == 0
    got[2, 3, 95] ^= 4
    assert list(nat.check_bytewise(R, 6, 20, got, threads=2)) == [2]
    # the strip-layout check rejects byte-layout outputs (the two products differ, F9)
    assert len(nat.check_apply(R, 6, 20, got)) == S
