"""paper_2108_02692_b200 -- B200-native XOR straight-line-program erasure coding.

Thin Python binding over the C ABI of ``libxslp.so`` (include/xslp.h): argument
marshalling only.  Every step of the hot path runs in the library (host
compiler in C++, device kernels in CUDA for sm_100a).  There is no CPU
fallback: importing this package without the built library raises, and device
calls on a machine without a CUDA device raise ``XslpError`` (XSLP_ECUDA).

Function names follow the C ABI (``xslp_compile``, ``xslp_encode_batch`` ...).
Buffers may be given as torch tensors (their ``data_ptr()`` is used), numpy
arrays (host), or raw integer addresses.  ``stream`` is a ``torch.cuda.Stream``,
a raw ``cudaStream_t`` integer, or None for torch's current stream.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# XSLP_LIBRARY: a diagnostic build of the same sources (scripts/sanitize_host.sh: ASan/UBSan, TSan)
_LIBPATH = os.environ.get("XSLP_LIBRARY") or os.path.join(_HERE, "libxslp.so")

if not os.path.exists(_LIBPATH):
    raise ImportError(
        f"{_LIBPATH} is missing: build it with `python paper_2108_02692_b200/build.py` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(_LIBPATH)

XSLP_OK, XSLP_EINVAL, XSLP_ESINGULAR, XSLP_EUNRECOVERABLE = 0, -1, -2, -3
XSLP_ECUDA, XSLP_ENOMEM, XSLP_ECOMPILE = -4, -5, -6
XSLP_RS_ISAL, XSLP_RS_SYSVAND, XSLP_CAUCHY = 0, 1, 2
XSLP_COMPRESS_NONE, XSLP_COMPRESS_REPAIR, XSLP_COMPRESS_XORREPAIR = 0, 1, 2
XSLP_SCHED_NONE, XSLP_SCHED_DFS, XSLP_SCHED_GREEDY = 0, 1, 2
XSLP_KERNEL_AUTO, XSLP_KERNEL_STRAIGHT, XSLP_KERNEL_INTERP, XSLP_KERNEL_TMA = 0, 1, 2, 3
XSLP_KERNEL_PIPE = 4
XSLP_LAYOUT_STRIP, XSLP_LAYOUT_BYTE = 0, 1
LAYOUTS = {"strip": 0, "byte": 1}

KINDS = {"isal": XSLP_RS_ISAL, "sysvand": XSLP_RS_SYSVAND, "cauchy": XSLP_CAUCHY}
COMPRESS = {"none": 0, "repair": 1, "xorrepair": 2}
KERNELS = {"auto": 0, "straight": 1, "interp": 2, "tma": 3, "pipe": 4}


class xslp_opts(ctypes.Structure):
    _fields_ = [("compress", ctypes.c_int32), ("fuse", ctypes.c_int32),
                ("schedule", ctypes.c_int32), ("specialise", ctypes.c_int32),
                ("lane_words", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("block_bytes_hint", ctypes.c_int64), ("kernel", ctypes.c_int32),
                ("goal_order", ctypes.c_int32), ("min_blocks", ctypes.c_int32),
                ("stages", ctypes.c_int32), ("greedy_capacity", ctypes.c_int32),
                ("layout", ctypes.c_int32), ("groups", ctypes.c_int32),
                ("phases", ctypes.c_int32),
                ("reuse", ctypes.c_int32), ("interp", ctypes.c_int32)]


class xslp_stats(ctypes.Structure):
    _fields_ = [("n_const", ctypes.c_int32), ("n_goals", ctypes.c_int32),
                ("xor_count", ctypes.c_int64), ("mem_count", ctypes.c_int64),
                ("n_instr", ctypes.c_int32), ("nvar", ctypes.c_int32),
                ("maxlive", ctypes.c_int32), ("n_copy_goals", ctypes.c_int32),
                ("n_zero_goals", ctypes.c_int32), ("regs", ctypes.c_int32),
                ("spill_bytes", ctypes.c_int32), ("regs_tma", ctypes.c_int32),
                ("spill_bytes_tma", ctypes.c_int32), ("regs_pipe", ctypes.c_int32),
                ("spill_bytes_pipe", ctypes.c_int32), ("compile_ms", ctypes.c_double),
                ("group_xor", ctypes.c_int64),
                ("smem_reads", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = ctypes.c_void_p
_sig = {
    "xslp_default_opts": (None, [ctypes.POINTER(xslp_opts)]),
    "xslp_coding_matrix": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "xslp_encode_bitmatrix": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P]),
    "xslp_decode_bitmatrix": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int, _P, _P]),
    "xslp_decode_bitmatrix_from": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int,
                                                  _P, _P]),
    "xslp_syndrome_bitmatrices": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int,
                                                 _P, _P]),
    "xslp_peer_export": (ctypes.c_int, [_P, _P]),
    "xslp_peer_open": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "xslp_peer_close": (ctypes.c_int, [_P]),
    "xslp_peer_enable": (ctypes.c_int, [ctypes.c_int]),
    "xslp_compile": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(xslp_opts),
                                    ctypes.POINTER(_P)]),
    "xslp_compile_text": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(xslp_opts),
                                         ctypes.POINTER(_P)]),
    "xslp_program_stats": (ctypes.c_int, [_P, ctypes.POINTER(xslp_stats)]),
    "xslp_program_dump": (ctypes.c_int64, [_P, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]),
    "xslp_free": (None, [_P]),
    "xslp_program_cache": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_int32)]),
    "xslp_prepare": (ctypes.c_int, [_P, ctypes.c_size_t]),
    "xslp_encode": (ctypes.c_int, [_P, _P, _P, ctypes.c_size_t, _P]),
    "xslp_decode": (ctypes.c_int, [_P, _P, _P, ctypes.c_size_t, _P]),
    "xslp_encode_batch": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_size_t, _P]),
    "xslp_decode_batch_multi": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int,
                                               ctypes.c_size_t, _P]),
    "xslp_decode_batch_grouped": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, _P, ctypes.c_size_t,
                                                 ctypes.c_int, _P]),
    "xslp_encode_host": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_size_t, _P]),
    "xslp_multi_create": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(xslp_opts),
                                         ctypes.POINTER(_P)]),
    "xslp_multi_decode": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "xslp_syndrome_create": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, ctypes.POINTER(xslp_opts),
                                            ctypes.POINTER(_P)]),
    "xslp_multi_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)]),
    "xslp_multi_free": (None, [_P]),
    "xslp_gf_table_apply": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P, _P, ctypes.c_int,
                                           ctypes.c_size_t, _P]),
    "xslp_fill_random": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_size_t,
                                        ctypes.c_uint64, ctypes.c_int64, _P]),
    "xslp_launch_count": (ctypes.c_int64, []),
    "xslp_codec_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(xslp_opts), ctypes.c_int, ctypes.POINTER(_P)]),
    "xslp_codec_free": (None, [_P]),
    "xslp_codec_block_bytes": (ctypes.c_int64, [_P, ctypes.c_int64]),
    "xslp_codec_encode": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P, _P]),
    "xslp_codec_reconstruct": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int64, _P]),
    "xslp_codec_decode": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int64, _P, _P]),
    "xslp_codec_program": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.POINTER(_P)]),
    "xslp_codec_cached": (ctypes.c_int, [_P]),
    "xslp_shard_header": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_uint64, ctypes.c_uint32]),
    "xslp_shard_header_parse": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int32),
                                               ctypes.POINTER(ctypes.c_int32),
                                               ctypes.POINTER(ctypes.c_int32),
                                               ctypes.POINTER(ctypes.c_uint64),
                                               ctypes.POINTER(ctypes.c_uint32)]),
    "xslp_last_error": (ctypes.c_char_p, []),
    "xslp_version": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


class XslpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc < 0:
        raise XslpError(rc, _lib.xslp_last_error().decode())
    return rc


def _ptr(x):
    """Address of a torch tensor / numpy array / integer / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")


_CUDA_OK = None


def _stream(s):
    global _CUDA_OK
    if s is None:
        import torch
        if _CUDA_OK is None:                 # cached: is_available() costs microseconds per call
            _CUDA_OK = torch.cuda.is_available()
        return torch.cuda.current_stream().cuda_stream if _CUDA_OK else 0
    if isinstance(s, int):
        return s
    return s.cuda_stream


def default_opts(**kw):
    o = xslp_opts()
    _lib.xslp_default_opts(ctypes.byref(o))
    for k, v in kw.items():
        if k == "compress" and isinstance(v, str):
            v = COMPRESS[v]
        if k == "kernel" and isinstance(v, str):
            v = KERNELS[v]
        if k == "layout" and isinstance(v, str):
            v = LAYOUTS[v]
        if k == "interp" and isinstance(v, str):
            v = {"lanes": 0, "pairs": 1, "tmem": 2}[v]
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, int(v))
    return o


class Program:
    """An immutable compiled program (owns an ``xslp_program*``)."""

    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    def stats(self):
        s = xslp_stats()
        _check(_lib.xslp_program_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def dump(self, form=0):
        n = _check(_lib.xslp_program_dump(self._h, form, None, 0))
        buf = ctypes.create_string_buffer(n + 1)
        _check(_lib.xslp_program_dump(self._h, form, buf, n + 1))
        return buf.value.decode()

    def ccap(self):
        c = ctypes.c_int32()
        _check(_lib.xslp_program_cache(self._h, 0, None, ctypes.byref(c)))
        return c.value

    def iocost(self, capacity):
        v = ctypes.c_int64()
        _check(_lib.xslp_program_cache(self._h, capacity, ctypes.byref(v), None))
        return v.value

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        lib = globals().get("_lib")
        if h and lib is not None:     # at interpreter shutdown the module may be gone
            lib.xslp_free(h)


# ---- matrices -----------------------------------------------------------------------
def xslp_coding_matrix(n, p, kind="isal"):
    out = np.zeros((n + p, n), dtype=np.uint8)
    _check(_lib.xslp_coding_matrix(n, p, KINDS.get(kind, kind), out.ctypes.data))
    return out


def xslp_encode_bitmatrix(gf, n, p):
    gf = np.ascontiguousarray(gf, dtype=np.uint8)
    out = np.zeros((8 * p, 8 * n), dtype=np.uint8)
    _check(_lib.xslp_encode_bitmatrix(gf.ctypes.data, n, p, out.ctypes.data))
    return out


def xslp_decode_bitmatrix(gf, n, p, erased):
    gf = np.ascontiguousarray(gf, dtype=np.uint8)
    er = np.ascontiguousarray(list(erased), dtype=np.int32)
    out = np.zeros((8 * len(er), 8 * n), dtype=np.uint8)
    surv = np.zeros(n, dtype=np.int32)
    _check(_lib.xslp_decode_bitmatrix(gf.ctypes.data, n, p, er.ctypes.data if len(er) else None,
                                      len(er), out.ctypes.data, surv.ctypes.data))
    return out, surv


def xslp_decode_bitmatrix_from(gf, n, p, erased, survivors):
    """Decode bitmatrix reading the given n survivors (input block j = block survivors[j])."""
    gf = np.ascontiguousarray(gf, dtype=np.uint8)
    er = np.ascontiguousarray(list(erased), dtype=np.int32)
    sv = np.ascontiguousarray(list(survivors), dtype=np.int32)
    if len(sv) != n:
        raise XslpError(-1, "need exactly n survivors")
    out = np.zeros((8 * len(er), 8 * n), dtype=np.uint8)
    _check(_lib.xslp_decode_bitmatrix_from(gf.ctypes.data, n, p, er.ctypes.data if len(er) else None,
                                           len(er), sv.ctypes.data, out.ctypes.data))
    return out


def xslp_syndrome_bitmatrices(gf, n, p, erased):
    """(syndrome bitmatrix 8p x 8(n+p), solve bitmatrix 8e x 8p) of the syndrome-form decode."""
    gf = np.ascontiguousarray(gf, dtype=np.uint8)
    er = np.ascontiguousarray(list(erased), dtype=np.int32)
    syn = np.zeros((8 * p, 8 * (n + p)), dtype=np.uint8)
    sol = np.zeros((8 * len(er), 8 * p), dtype=np.uint8)
    _check(_lib.xslp_syndrome_bitmatrices(gf.ctypes.data, n, p, er.ctypes.data, len(er),
                                          syn.ctypes.data, sol.ctypes.data))
    return syn, sol


# ---- peer memory (cross-GPU decode) ---------------------------------------------------
PEER_HANDLE_BYTES = 128


def xslp_peer_export(d_ptr):
    """bytes handle of the device allocation holding d_ptr (tensor or address)."""
    h = ctypes.create_string_buffer(PEER_HANDLE_BYTES)
    _check(_lib.xslp_peer_export(_ptr(d_ptr), h))
    return h.raw


def xslp_peer_open(handle):
    """Address (int) of an exported pointer, mapped on the current device."""
    if len(handle) != PEER_HANDLE_BYTES:
        raise XslpError(-1, "bad handle length")
    out = _P()
    buf = ctypes.create_string_buffer(bytes(handle), PEER_HANDLE_BYTES)
    _check(_lib.xslp_peer_open(buf, ctypes.byref(out)))
    return out.value


def xslp_peer_close(d_ptr):
    _check(_lib.xslp_peer_close(_ptr(d_ptr)))


def xslp_peer_enable(peer_device):
    _check(_lib.xslp_peer_enable(peer_device))


# ---- compile ------------------------------------------------------------------------
def xslp_compile(bits, opts=None, **kw):
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    o = opts if opts is not None else default_opts(**kw)
    h = _P()
    _check(_lib.xslp_compile(bits.ctypes.data if bits.size else None, bits.shape[0], bits.shape[1],
                             ctypes.byref(o), ctypes.byref(h)))
    return Program(h.value)


def xslp_compile_text(text, n_const, opts=None, **kw):
    o = opts if opts is not None else default_opts(**kw)
    h = _P()
    _check(_lib.xslp_compile_text(text.encode(), n_const, ctypes.byref(o), ctypes.byref(h)))
    return Program(h.value)


# ---- device -------------------------------------------------------------------------
def _ptr_array(ptrs):
    if isinstance(ptrs, ctypes.Array):       # a prebuilt pointer array (see block_ptrs)
        return ptrs
    return (ctypes.c_void_p * max(1, len(ptrs)))(*[_ptr(p) for p in ptrs])


def block_ptrs(blocks):
    """A reusable pointer array for xslp_encode / xslp_decode (skips the per-call conversion
    of a list of tensors; the caller keeps the tensors alive)."""
    return _ptr_array(list(blocks))


def xslp_prepare(prog, block_bytes=0):
    _check(_lib.xslp_prepare(prog.handle, block_bytes))


def xslp_encode(prog, in_blocks, out_blocks, block_bytes, stream=None):
    a, b = _ptr_array(in_blocks), _ptr_array(out_blocks)
    _check(_lib.xslp_encode(prog.handle, a, b, block_bytes, _stream(stream)))


def xslp_decode(prog, in_blocks, out_blocks, block_bytes, stream=None):
    a, b = _ptr_array(in_blocks), _ptr_array(out_blocks)
    _check(_lib.xslp_decode(prog.handle, a, b, block_bytes, _stream(stream)))


def xslp_encode_batch(prog, d_in_tbl, d_out_tbl, nstripes, block_bytes, stream=None):
    _check(_lib.xslp_encode_batch(prog.handle, _ptr(d_in_tbl), _ptr(d_out_tbl), nstripes,
                                  block_bytes, _stream(stream)))


def xslp_decode_batch_multi(progs, d_prog_of_stripe, d_in_tbl, d_out_tbl, nstripes, block_bytes,
                            stream=None):
    arr = (ctypes.c_void_p * len(progs))(*[p.handle for p in progs])
    _check(_lib.xslp_decode_batch_multi(arr, len(progs), _ptr(d_prog_of_stripe), _ptr(d_in_tbl),
                                        _ptr(d_out_tbl), nstripes, block_bytes, _stream(stream)))


def xslp_decode_batch_grouped(progs, d_stripe_ids, group_offsets, d_in_tbl, d_out_tbl, block_bytes,
                              nstreams=8, stream=None):
    arr = (ctypes.c_void_p * len(progs))(*[p.handle for p in progs])
    off = np.ascontiguousarray(group_offsets, dtype=np.int32)
    if len(off) != len(progs) + 1:
        raise ValueError("group_offsets needs len(progs) + 1 entries")
    _check(_lib.xslp_decode_batch_grouped(arr, len(progs), _ptr(d_stripe_ids), off.ctypes.data,
                                          _ptr(d_in_tbl), _ptr(d_out_tbl), block_bytes, nstreams,
                                          _stream(stream)))


class Multi:
    """Programs fused into persistent multi-program pipeline kernels (xslp_multi_*)."""

    def __init__(self, progs, per_module=20, opts=None, **kw):
        self._progs = list(progs)          # keep the programs alive
        self.nprogs = len(self._progs)
        o = opts if opts is not None else default_opts(**kw)
        arr = (ctypes.c_void_p * len(self._progs))(*[p.handle for p in self._progs])
        h = _P()
        _check(_lib.xslp_multi_create(arr, len(self._progs), per_module, ctypes.byref(o),
                                      ctypes.byref(h)))
        self._h = h.value

    @property
    def handle(self):
        return self._h

    def info(self):
        m, r, s, t = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
        _check(_lib.xslp_multi_info(self._h, ctypes.byref(m), ctypes.byref(r), ctypes.byref(s),
                                    ctypes.byref(t)))
        return {"modules": m.value, "regs": r.value, "spill_bytes": s.value, "compile_ms": t.value}

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = globals().get("_lib")
        if h and lib is not None:
            lib.xslp_multi_free(h)
            self._h = None


class SyndromeDecoder(Multi):
    """Heterogeneous decode in syndrome form (xslp_syndrome_create): the shared syndrome program
    plus one small solve program per erasure pattern, fused; decode with xslp_multi_decode on
    an input table of all n+p blocks per stripe (erased entries -> a zero block)."""

    def __init__(self, gf, n, p, patterns, per_module=0, opts=None, **kw):   # noqa: super
        self._progs = []
        pats = np.ascontiguousarray([sorted(er) for er in patterns], dtype=np.int32)
        self.nprogs = pats.shape[0]
        g = np.ascontiguousarray(gf, dtype=np.uint8)
        o = opts if opts is not None else default_opts(**kw)
        h = _P()
        _check(_lib.xslp_syndrome_create(g.ctypes.data, n, p, pats.ctypes.data, pats.shape[0],
                                         pats.shape[1], per_module, ctypes.byref(o), ctypes.byref(h)))
        self._h = h.value


def xslp_multi_decode(multi, d_prog_of_stripe, d_stripe_ids, group_offsets, d_in_tbl, d_out_tbl,
                      block_bytes, stream=None):
    off = np.ascontiguousarray(group_offsets, dtype=np.int32)
    if len(off) != multi.nprogs + 1:
        raise ValueError("group_offsets needs nprogs + 1 entries")
    _check(_lib.xslp_multi_decode(multi.handle, _ptr(d_prog_of_stripe), _ptr(d_stripe_ids),
                                  off.ctypes.data, _ptr(d_in_tbl), _ptr(d_out_tbl), block_bytes,
                                  _stream(stream)))


def xslp_gf_table_apply(coef, d_in_tbl, d_out_tbl, nstripes, block_bytes, stream=None):
    """Byte-wise GF(2^8) matrix apply with PRMT lookup tables (the paper's approach (1))."""
    c = np.ascontiguousarray(coef, dtype=np.uint8)
    m, n = c.shape
    _check(_lib.xslp_gf_table_apply(c.ctypes.data, n, m, _ptr(d_in_tbl), _ptr(d_out_tbl), nstripes,
                                    block_bytes, _stream(stream)))


def group_stripes(prog_of_stripe, nprogs):
    """Host helper: (stripe ids sorted by program, offsets[nprogs+1]) for the grouped call."""
    pos = np.asarray(prog_of_stripe, dtype=np.int64)
    order = np.argsort(pos, kind="stable").astype(np.int32)
    counts = np.bincount(pos, minlength=nprogs)
    off = np.zeros(nprogs + 1, dtype=np.int32)
    off[1:] = np.cumsum(counts)
    return order, off


def xslp_encode_host(prog, h_in, h_out, nstripes, block_bytes, stream=None):
    _check(_lib.xslp_encode_host(prog.handle, _ptr(h_in), _ptr(h_out), nstripes, block_bytes,
                                 _stream(stream)))


def xslp_fill_random(d_buf, nstripes, nblocks, block_bytes, seed, stripe0=0, stream=None):
    _check(_lib.xslp_fill_random(_ptr(d_buf), nstripes, nblocks, block_bytes, seed, stripe0,
                                 _stream(stream)))


def xslp_launch_count():
    return _lib.xslp_launch_count()


def xslp_version():
    return _lib.xslp_version().decode()


def block_table(base, nstripes, nblocks, block_bytes, device=None):
    """Device pointer table [nstripes][nblocks] for a contiguous
    [nstripes][nblocks][block_bytes] buffer starting at ``base`` (torch int64 tensor)."""
    import torch
    b = _ptr(base)
    idx = torch.arange(nstripes * nblocks, dtype=torch.int64)
    tbl = idx * int(block_bytes) + int(b)
    return tbl.to(device if device is not None else "cuda")


def compile_many(bits_list, workers=None, **kw):
    """Compile several bitmatrices concurrently (the C++ compiler runs outside the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    workers = workers or min(32, os.cpu_count() or 1)
    o = default_opts(**kw)
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(lambda b: xslp_compile(b, opts=o), bits_list))


# ---- codec front end ----------------------------------------------------------------
class Codec:
    """RS(n,p) over arbitrary-length device data (xslp_codec_*)."""

    def __init__(self, n, p, kind="isal", cache_entries=1024, **opts):
        o = default_opts(**opts)
        h = _P()
        _check(_lib.xslp_codec_create(n, p, KINDS.get(kind, kind), ctypes.byref(o), cache_entries,
                                      ctypes.byref(h)))
        self._h, self.n, self.p = h.value, n, p

    def block_bytes(self, length):
        return _check(_lib.xslp_codec_block_bytes(self._h, length))

    def encode(self, d_data, length, d_shards, stream=None):
        _check(_lib.xslp_codec_encode(self._h, _ptr(d_data), length, _ptr(d_shards), _stream(stream)))

    def reconstruct(self, d_shards, erased, length, stream=None):
        er = (ctypes.c_int32 * max(1, len(erased)))(*erased)
        _check(_lib.xslp_codec_reconstruct(self._h, _ptr(d_shards), er, len(erased), length,
                                           _stream(stream)))

    def decode(self, d_shards, erased, length, d_out, stream=None):
        er = (ctypes.c_int32 * max(1, len(erased)))(*erased)
        _check(_lib.xslp_codec_decode(self._h, _ptr(d_shards), er, len(erased), length, _ptr(d_out),
                                      _stream(stream)))

    def program_stats(self, erased=()):
        er = (ctypes.c_int32 * max(1, len(erased)))(*erased)
        h = _P()
        _check(_lib.xslp_codec_program(self._h, er, len(erased), ctypes.byref(h)))
        s = xslp_stats()
        _check(_lib.xslp_program_stats(h, ctypes.byref(s)))
        return s.as_dict(), h.value

    def cached(self):
        return _lib.xslp_codec_cached(self._h)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        lib = globals().get("_lib")
        if h and lib is not None:
            lib.xslp_codec_free(h)


def xslp_shard_header(n, p, shard, original_length, block_bytes):
    out = (ctypes.c_uint8 * 32)()
    _check(_lib.xslp_shard_header(out, n, p, shard, original_length, block_bytes))
    return bytes(out)


def xslp_shard_header_parse(header):
    buf = (ctypes.c_uint8 * 32).from_buffer_copy(bytes(header[:32]))
    n, p, sh = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    ln, bb = ctypes.c_uint64(), ctypes.c_uint32()
    _check(_lib.xslp_shard_header_parse(buf, ctypes.byref(n), ctypes.byref(p), ctypes.byref(sh),
                                        ctypes.byref(ln), ctypes.byref(bb)))
    return dict(n=n.value, p=p.value, shard=sh.value, original_length=ln.value, block_bytes=bb.value)
