"""O1 -- GF(2^8) arithmetic for the oracle (TEST INFRASTRUCTURE ONLY).

Paper: "we implement GF(2^8) using the primitive polynomial x^8+x^4+x^3+x^2+1
used in ISA-L" ([Eval] §Dataset); "each element of GF(2^8) is coded by
one byte" ([Intro]).  Addition is XOR ([Intro]).

Multiplication is the textbook definition written out: carry-less product of
the two polynomials, reduced modulo the primitive polynomial (shift-and-add).
A 256x256 table is filled from that routine only to make the bulk RS oracle
(rs.py) usable on megabyte inputs; the table adds no arithmetic of its own.
"""
import numpy as np

POLY = 0x11D  # x^8 + x^4 + x^3 + x^2 + 1


def gf_add(a: int, b: int) -> int:
    """Field addition = bitwise XOR."""
    return a ^ b


def gf_mul(a: int, b: int) -> int:
    """Product of two field elements: polynomial multiply mod POLY."""
    r = 0
    a &= 0xFF
    b &= 0xFF
    while b:
        if b & 1:
            r ^= a
        b >>= 1
        a <<= 1
        if a & 0x100:
            a ^= POLY
    return r


def gf_pow(a: int, e: int) -> int:
    r = 1
    for _ in range(e):
        r = gf_mul(r, a)
    return r


def gf_inv(a: int) -> int:
    """Multiplicative inverse by exhaustive search; 0 has none."""
    if a == 0:
        raise ZeroDivisionError("0 has no inverse in GF(2^8)")
    for b in range(1, 256):
        if gf_mul(a, b) == 1:
            return b
    raise AssertionError("unreachable: GF(2^8)* is a group")


def _build_mul_table() -> np.ndarray:
    t = np.zeros((256, 256), dtype=np.uint8)
    for a in range(256):
        for b in range(256):
            t[a, b] = gf_mul(a, b)
    return t


MUL = _build_mul_table()  # MUL[a, b] = gf_mul(a, b)
