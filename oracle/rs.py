"""O3/O4 -- Reed-Solomon over the strip layout (TEST INFRASTRUCTURE ONLY).

Layout ([Eval] §Throughput Comparison): each block of B bytes is
cut into 8 equal strips of S = B/8 bytes; "we run SLPs for 8 x 10 input arrays
of N/(8 x 10) bytes" for RS(10,4).  Constant c_{8j+k} of the SLP is strip k of
block j (reading R3).

What the hot path computes is V . D over GF(2^8) expressed through the
bitmatrix V~ acting on the 8n strips ([Intro]).  This module states
that result two independent ways:

* ``apply_rows`` -- the plain definition as a table-driven byte RS on the
  bit-transposed view: for strip offset o and bit b, the byte
  x_j = sum_k bit_b(strip(j,k)[o]) 2^k is the GF element B^-1 of the 8 bits
  (reading R3), y_i = sum_j R_ij x_j, and bit r of y_i is written
  to bit b of output strip (i, r)[o].  This is the oracle O3 (encode) / O4
  (decode with the rows from matrices.decode_rows).
* ``bitmatrix_apply`` -- MM over GF(2) "is just array XORs":
  output strip r = XOR of the input strips whose bit is set in row r.
"""
import numpy as np

from .gf256 import MUL


def _check(blocks):
    blocks = np.ascontiguousarray(blocks, dtype=np.uint8)
    if blocks.ndim != 2 or blocks.shape[1] % 8 != 0:
        raise ValueError("blocks must be (count, B) with B a multiple of 8")
    return blocks


def apply_rows(rows, blocks):
    """rows: m x n GF(2^8) coefficients; blocks: (n, B) uint8 -> (m, B) uint8."""
    blocks = _check(blocks)
    n, B = blocks.shape
    m = len(rows)
    assert all(len(r) == n for r in rows)
    S = B // 8
    strips = blocks.reshape(n, 8, S)
    out = np.zeros((m, 8, S), dtype=np.uint8)
    for b in range(8):
        # gather: byte x_j from bit b of the 8 strips of block j (B^-1, LSB-first)
        x = []
        for j in range(n):
            xj = np.zeros(S, dtype=np.uint8)
            for k in range(8):
                xj |= ((strips[j, k] >> b) & 1) << k
            x.append(xj)
        for i in range(m):
            y = np.zeros(S, dtype=np.uint8)
            for j in range(n):
                y ^= MUL[rows[i][j]][x[j]]
            # scatter: bit r of y_i -> bit b of output strip (i, r)
            for r in range(8):
                out[i, r] |= ((y >> r) & 1) << b
    return out.reshape(m, B)


def encode(g, n, data):
    """Systematic encode: parity blocks = R . D with g = [I_n; R]."""
    return apply_rows(g[n:], data)


def decode(goal_rows, survivor_blocks):
    """Recovered blocks = goal_rows . survivors (rows from decode_rows)."""
    return apply_rows(goal_rows, survivor_blocks)


def bytewise_apply(rows, blocks):
    """Textbook byte-wise RS: out_i[t] = sum_j R_ij d_j[t] over GF(2^8).

    The result the byte-compatible layout must reproduce: the SLP
    runs on the bit-planes of the bytes, and P:549-558 (x*y = B^-1(x~ B(y))) makes the
    bit-plane XOR program equal to this per-byte product.  Table-driven, one byte
    position at a time over whole arrays.
    """
    blocks = np.ascontiguousarray(blocks, dtype=np.uint8)
    n = blocks.shape[0]
    assert all(len(r) == n for r in rows)
    out = np.zeros((len(rows), blocks.shape[1]), dtype=np.uint8)
    for i, row in enumerate(rows):
        for j in range(n):
            out[i] ^= MUL[row[j]][blocks[j]]
    return out


def bitmatrix_apply(bits, blocks):
    """(8m x 8n) 0/1 matrix times the 8n strips, as array XORs."""
    blocks = _check(blocks)
    n, B = blocks.shape
    S = B // 8
    bits = np.asarray(bits, dtype=np.uint8)
    assert bits.shape[1] == 8 * n
    strips = blocks.reshape(8 * n, S)
    out = np.zeros((bits.shape[0], S), dtype=np.uint8)
    for r in range(bits.shape[0]):
        for c in range(8 * n):
            if bits[r, c]:
                out[r] ^= strips[c]
    return out.reshape(bits.shape[0] // 8, B)
