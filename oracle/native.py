"""ctypes loader of oracle/rs_oracle.c (TEST INFRASTRUCTURE ONLY).

The C oracle is O3/O4 of oracle/rs.py written in plain C with threads over stripes, so that
whole BASELINE workloads can be verified on the host (every stripe of cfgs 2-4)
and timed as the CPU baseline.  It is built with gcc into oracle/librs_oracle.so by
__graft_entry__.build() or, if missing or stale, on first use here.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import this.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rs_oracle.c")
LIB = os.path.join(HERE, "librs_oracle.so")

_lib = None


def build(force=False):
    """gcc -O3 -shared -pthread oracle/rs_oracle.c -> oracle/librs_oracle.so."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.run(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-pthread", "-Wall", "-o", tmp, SRC],
                   check=True, capture_output=True, text=True)
    os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I, U64, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_size_t
        L.oracle_gf_mul.restype = ctypes.c_uint8
        L.oracle_gf_mul.argtypes = [ctypes.c_uint8, ctypes.c_uint8]
        L.oracle_tilde_bit.restype = I
        L.oracle_tilde_bit.argtypes = [ctypes.c_uint8, I, I]
        L.oracle_apply_rows.restype = None
        L.oracle_apply_rows.argtypes = [P, I, I, P, P, SZ]
        L.oracle_fill.restype = None
        L.oracle_fill.argtypes = [U64, I64, I, SZ, P]
        L.oracle_check.restype = I64
        L.oracle_check.argtypes = [I, P, I, I, I, P, U64, I64, I, SZ, P, P, I]
        L.oracle_apply_each.restype = None
        L.oracle_apply_each.argtypes = [I, P, SZ, I, I, P, P, I, SZ, I]
        _lib = L
    return _lib


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _rows(rows):
    r = np.ascontiguousarray(rows, dtype=np.uint8)
    if r.ndim != 2:
        raise ValueError("rows must be m x n")
    return r


def apply_rows(rows, blocks):
    """Same contract as oracle.rs.apply_rows: (m x n) rows, (n, B) blocks -> (m, B)."""
    r = _rows(rows)
    b = np.ascontiguousarray(blocks, dtype=np.uint8)
    m, n = r.shape
    if b.ndim != 2 or b.shape[0] != n or b.shape[1] % 8:
        raise ValueError("blocks must be (n, B) with B % 8 == 0")
    out = np.zeros((m, b.shape[1]), dtype=np.uint8)
    lib().oracle_apply_rows(r.ctypes.data, m, n, b.ctypes.data, out.ctypes.data, b.shape[1])
    return out


def fill(seed, stripe, nblocks, nbytes):
    """synth.stripe_data(seed, stripe, nblocks, nbytes), from the C generator."""
    out = np.zeros((nblocks, nbytes), dtype=np.uint8)
    lib().oracle_fill(seed, stripe, nblocks, nbytes, out.ctypes.data)
    return out


def check_apply(rows, seed, stripe0, got, threads=None):
    """got: (stripes, m, B) host bytes of rows . fill(seed, stripe0 + s, n, B).  Returns the
    indices of stripes with any differing byte."""
    r = _rows(rows)
    g = np.ascontiguousarray(got, dtype=np.uint8)
    S, m, B = g.shape
    assert m == r.shape[0]
    bad = np.zeros(S, dtype=np.uint8)
    lib().oracle_check(0, r.ctypes.data, m, r.shape[1], 0, None, seed, stripe0, S, B, g.ctypes.data,
                       bad.ctypes.data, threads or cores())
    return np.nonzero(bad)[0]


def check_bytewise(rows, seed, stripe0, got, threads=None):
    """As check_apply for the textbook byte-wise product (rs.bytewise_apply)."""
    r = _rows(rows)
    g = np.ascontiguousarray(got, dtype=np.uint8)
    S, m, B = g.shape
    assert m == r.shape[0]
    bad = np.zeros(S, dtype=np.uint8)
    lib().oracle_check(2, r.ctypes.data, m, r.shape[1], 0, None, seed, stripe0, S, B, g.ctypes.data,
                       bad.ctypes.data, threads or cores())
    return np.nonzero(bad)[0]


def check_codeword(parity_rows, n, seed, stripe0, erased, got, threads=None):
    """got: (stripes, e, B) host bytes that must equal blocks erased[s] (ascending) of the
    codeword [fill(seed, stripe0 + s, n, B); parity_rows . data].  Returns bad stripe indices."""
    r = _rows(parity_rows)
    g = np.ascontiguousarray(got, dtype=np.uint8)
    S, e, B = g.shape
    sel = np.ascontiguousarray(erased, dtype=np.int32)
    assert sel.shape == (S, e) and r.shape[1] == n
    bad = np.zeros(S, dtype=np.uint8)
    lib().oracle_check(1, r.ctypes.data, e, n, r.shape[0], sel.ctypes.data, seed, stripe0, S, B,
                       g.ctypes.data, bad.ctypes.data, threads or cores())
    return np.nonzero(bad)[0]


def apply_each(rows, inputs, threads=None, bytewise=False):
    """(stripes, n, B) inputs -> (stripes, m, B) on `threads` threads; rows is one (m x n)
    matrix for every stripe or (stripes, m, n), one per stripe."""
    r = np.ascontiguousarray(rows, dtype=np.uint8)
    x = np.ascontiguousarray(inputs, dtype=np.uint8)
    S, n, B = x.shape
    m = r.shape[-2]
    stride = 0 if r.ndim == 2 else m * n
    assert r.shape[-1] == n and (r.ndim == 2 or r.shape[0] == S)
    out = np.zeros((S, m, B), dtype=np.uint8)
    lib().oracle_apply_each(int(bytewise), r.ctypes.data, stride, m, n, x.ctypes.data, out.ctypes.data,
                            S, B, threads or cores())
    return out
