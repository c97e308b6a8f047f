"""Codec front end: padding, shard header, decode-program memo
(host, no GPU) and the device roundtrip against the oracle (gpu)."""
import itertools

import numpy as np
import pytest

import paper_2108_02692_b200 as X
from oracle import matrices as mx
from oracle import rs
from oracle import slp as oslp


def test_shard_header_roundtrip_and_layout():
    h = X.xslp_shard_header(10, 4, 12, 123456789012, 1 << 20)
    assert len(h) == 32 and h[:4] == b"XSLP" and h[4] == 1
    assert h[5:8] == bytes([10, 4, 12])
    assert int.from_bytes(h[8:16], "little") == 123456789012
    assert int.from_bytes(h[16:20], "little") == 1 << 20 and h[20:] == bytes(12)
    assert X.xslp_shard_header_parse(h) == dict(n=10, p=4, shard=12, original_length=123456789012,
                                                 block_bytes=1 << 20)
    bad = bytearray(h)
    bad[0] = ord("Y")
    with pytest.raises(X.XslpError):
        X.xslp_shard_header_parse(bad)
    with pytest.raises(X.XslpError):
        X.xslp_shard_header(10, 4, 14, 0, 128)


def test_block_bytes_padding():
    c = X.Codec(10, 4, specialise=0)
    assert c.block_bytes(0) == 128
    assert c.block_bytes(1) == 128
    assert c.block_bytes(1280) == 128
    assert c.block_bytes(1281) == 256
    assert c.block_bytes(10 << 20) == 1 << 20
    for ln in (7, 999, 12345, 10 << 20):
        b = c.block_bytes(ln)
        assert b % 128 == 0 and 10 * b >= ln and 10 * (b - 128) < ln


def test_memo_cache_and_programs():
    c = X.Codec(10, 4, cache_entries=3, specialise=0)
    og = mx.coding_matrix(10, 4)
    s0, h0 = c.program_stats([6, 5, 4, 2])
    s1, h1 = c.program_stats([2, 4, 5, 6])           # same pattern in another order: memo hit
    assert h0 == h1 and c.cached() == 1
    assert s0["xor_count"] < 1368                     # compressed P_dec
    for er in ([0], [1, 13], [3, 7, 9], [0, 1, 2, 3]):
        c.program_stats(er)
    assert c.cached() == 3                            # LRU bound
    enc, _ = c.program_stats([])
    assert enc["n_goals"] == 32
    with pytest.raises(X.XslpError) as e:
        c.program_stats([0, 1, 2, 3, 4])
    assert e.value.code == X.XSLP_EUNRECOVERABLE
    # the memoised decode program is the oracle's decode bitmatrix
    _, rows = mx.decode_rows(og, 10, [2, 4, 5, 6])
    p = X.xslp_compile(X.xslp_decode_bitmatrix(X.xslp_coding_matrix(10, 4), 10, 4, [2, 4, 5, 6])[0],
                       specialise=0)
    assert oslp.evaluate(p.dump()) == oslp.rows_to_sets(mx.to_bitmatrix(rows))


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,kind", [(4, 2, "cauchy"), (10, 4, "isal"), (8, 3, "isal")])
def test_codec_roundtrip_gpu(n, p, kind):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = X.Codec(n, p, kind)
    og = mx.coding_matrix(n, p, kind)
    rng = np.random.default_rng(n * 10 + p)
    for ln in (1, 1000, 77777, 3 << 20):
        data = rng.integers(0, 256, size=ln, dtype=np.uint8)
        B = c.block_bytes(ln)
        d = torch.from_numpy(data).cuda()
        shards = torch.full((n + p, B), 0x5A, dtype=torch.uint8, device="cuda")
        c.encode(d, ln, shards)
        torch.cuda.synchronize()
        h = shards.cpu().numpy()
        padded = np.zeros(n * B, dtype=np.uint8)
        padded[:ln] = data
        assert (h[:n].reshape(-1) == padded).all()                       # systematic
        assert (h[n:] == rs.encode(og, n, padded.reshape(n, B))).all()   # parity = oracle
        # a data buffer that is not 16-byte aligned takes the copy-then-encode path (the
        # aligned one above reads the data in place and writes data + parity shards in one pass)
        mis = torch.empty(ln + 1, dtype=torch.uint8, device="cuda")
        mis[1:] = d
        shards2 = torch.full((n + p, B), 0x77, dtype=torch.uint8, device="cuda")
        c.encode(mis[1:], ln, shards2)
        torch.cuda.synchronize()
        assert torch.equal(shards2, shards), ln
        pats = list(itertools.combinations(range(n + p), p))
        for er in pats[:: max(1, len(pats) // 12)]:
            broken = shards.clone()
            broken[list(er)] = 0xEE
            out = torch.zeros(max(ln, 1), dtype=torch.uint8, device="cuda")
            c.decode(broken, list(er), ln, out)
            torch.cuda.synchronize()
            assert (out[:ln].cpu().numpy() == data).all(), (ln, er)
            mis = torch.zeros(ln + 1, dtype=torch.uint8, device="cuda")   # unaligned output:
            c.decode(broken.clone(), list(er), ln, mis[1:])                # rebuild + copy path
            torch.cuda.synchronize()
            assert (mis[1:].cpu().numpy() == data).all(), (ln, er)
            c.reconstruct(broken, list(er), ln)
            torch.cuda.synchronize()
            assert torch.equal(broken, shards), (ln, er)


@pytest.mark.gpu
def test_codec_every_4_loss_pattern_rs10_4_gpu():
    # SPEC codec example: RS(10,4), every one of the 1001 4-loss patterns recovers random ~1 MB
    # data of irregular length (memoised decode programs run on the interpreter: no JIT)
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n, p = 10, 4
    c = X.Codec(n, p, cache_entries=2048, specialise=0)
    ln = (1 << 20) + 12345
    data = np.random.default_rng(1001).integers(0, 256, size=ln, dtype=np.uint8)
    B = c.block_bytes(ln)
    d = torch.from_numpy(data).cuda()
    shards = torch.empty((n + p, B), dtype=torch.uint8, device="cuda")
    c.encode(d, ln, shards)
    want = d.clone()
    out = torch.empty(ln, dtype=torch.uint8, device="cuda")
    for k, er in enumerate(itertools.combinations(range(n + p), p)):
        broken = shards.clone()
        broken[list(er)] = 0
        out.zero_()
        c.decode(broken, list(er), ln, out)
        if k % 64 == 0:
            torch.cuda.synchronize()
        assert torch.equal(out, want), er
    assert c.cached() == 1000        # {10,11,12,13} loses parity only: decode needs no program
