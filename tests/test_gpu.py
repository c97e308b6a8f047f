"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Inputs are seeded (synth); expected values come only from oracle/ (or, for the
full-size roundtrip property, from the seeded generator itself).  Sizes: small
cases compare every byte and span several CTA tiles plus a ragged tail; the
BASELINE-size cases run in the bench's launch configuration and compare sampled
stripes with the oracle, plus properties checked over all stripes.
"""
import itertools
import sys
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2108_02692_b200 as X  # noqa: E402
from oracle import matrices as mx  # noqa: E402
from oracle import rs  # noqa: E402
from oracle import native as nat  # noqa: E402
import synth  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def dev_buf(nstripes, nblocks, B):
    return torch.empty((nstripes, nblocks, B), dtype=torch.uint8, device="cuda")


def host_data(seed, stripes, n, B):
    return np.stack([synth.stripe_data(seed, s, n, B) for s in stripes])


def run_batch(prog, din, dout, B, nstripes=None):
    ns = din.shape[0] if nstripes is None else nstripes
    ti = X.block_table(din, din.shape[0], din.shape[1], B)
    to = X.block_table(dout, dout.shape[0], dout.shape[1], B)
    X.xslp_encode_batch(prog, ti, to, ns, B)
    torch.cuda.synchronize()


def _kernel_kw(kw):
    """kernel="interp_pairs" / "interp_lanes": the pair-pipelined / lane-parallel interpreters
    (XSLP_INTERP_PAIRS / LANES); "interp" is the TMEM one (the default)."""
    if kw.get("kernel") in ("interp_pairs", "interp_tmem", "interp_lanes"):
        kw = dict(kw, kernel="interp", interp=kw["kernel"][7:])
    return kw


def compile_enc(n, p, kind="isal", **kw):
    g = X.xslp_coding_matrix(n, p, kind)
    return g, X.xslp_compile(X.xslp_encode_bitmatrix(g, n, p), **_kernel_kw(kw))


# ---- generator ---------------------------------------------------------------------------

def test_fill_matches_synth():
    n, B = 10, 4096
    d = dev_buf(3, n, B)
    X.xslp_fill_random(d, 3, n, B, seed=42, stripe0=5)
    torch.cuda.synchronize()
    want = host_data(42, [5, 6, 7], n, B)
    assert (d.cpu().numpy() == want).all()


# ---- cfg1: RS(4,2) Cauchy, one stripe of 4 x 4 KiB ----------------------------------------

@pytest.mark.parametrize("kernel", ["straight", "interp"])
def test_cfg1_encode_decode(kernel):
    n, p, B = 4, 2, 4096
    g, enc = compile_enc(n, p, "cauchy", kernel=kernel)
    og = mx.coding_matrix(n, p, "cauchy")
    data = host_data(1, [0], n, B)[0]
    want_par = rs.encode(og, n, data)
    d = torch.from_numpy(data).cuda()
    par = torch.zeros((p, B), dtype=torch.uint8, device="cuda")
    X.xslp_encode(enc, [d[j] for j in range(n)], [par[i] for i in range(p)], B)
    torch.cuda.synchronize()
    assert (par.cpu().numpy() == want_par).all()
    blocks = np.concatenate([data, want_par])           # oracle blocks as decode input
    dblocks = torch.from_numpy(blocks).cuda()
    for e in (1, 2):
        for erased in itertools.combinations(range(n + p), e):
            bits, surv = X.xslp_decode_bitmatrix(g, n, p, erased)
            dec = X.xslp_compile(bits, kernel=kernel)
            out = torch.zeros((e, B), dtype=torch.uint8, device="cuda")
            X.xslp_decode(dec, [dblocks[s] for s in surv], [out[i] for i in range(e)], B)
            torch.cuda.synchronize()
            assert (out.cpu().numpy() == blocks[list(erased)]).all(), erased


# ---- multi-tile, ragged tail, all kernel variants and compressors -------------------------

@pytest.mark.parametrize("comp", ["none", "repair", "xorrepair"])
@pytest.mark.parametrize("kern,lanes", [("straight", 1), ("straight", 2), ("straight", 4),
                                        ("interp", 1), ("interp_pairs", 1), ("interp_pairs", 2),
                                        ("interp_lanes", 1),
                                        ("tma", 1), ("tma", 2), ("pipe", 1), ("pipe", 2)])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_rs10_encode_small_full_compare(comp, kern, lanes, p):
    n, B, S = 10, 9600, 5          # strip 1200 B = 300 words: two 256-thread tiles, ragged tail
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p, compress=comp, kernel=kern, lane_words=lanes,
                          fuse=1 if comp != "repair" else 0, schedule=1 if comp != "repair" else 0)
    data = host_data(4, range(S), n, B)
    din = torch.from_numpy(data).cuda()
    dout = torch.full((S, p, B), 0xAB, dtype=torch.uint8, device="cuda")
    run_batch(prog, din, dout, B)
    got = dout.cpu().numpy()
    for s in range(S):
        assert (got[s] == rs.encode(og, n, data[s])).all(), s


@pytest.mark.parametrize("kern", ["straight", "tma", "pipe"])
def test_baked_and_generic_strip(kern):
    n, p = 10, 4
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p, block_bytes_hint=8192, kernel=kern)
    for B in (8192, 4096):            # baked kernel, then the generic-address kernel
        data = host_data(9, range(3), n, B)
        din = torch.from_numpy(data).cuda()
        dout = dev_buf(3, p, B)
        run_batch(prog, din, dout, B)
        for s in range(3):
            assert (dout[s].cpu().numpy() == rs.encode(og, n, data[s])).all()


# ---- cfg3-style heterogeneous decode (one program per stripe) ----------------------------

def _decode_inputs(seed, S, n, p, B, e):
    g = mx.coding_matrix(n, p)
    pats, blocks = [], []
    for s in range(S):
        er = synth.erasure_pattern(seed, s, n + p, e)
        data = synth.stripe_data(seed, s, n, B)
        blocks.append(np.concatenate([data, rs.encode(g, n, data)]))
        pats.append(tuple(er))
    return pats, blocks


@pytest.mark.parametrize("kern", ["interp", "interp_pairs", "interp_lanes", "straight", "grouped",
                                  "grouped_tma", "grouped_pipe"])
def test_heterogeneous_decode(kern):
    n, p, B, S = 10, 4, 4096, 24
    pats, blocks = _decode_inputs(3, S, n, p, B, 4)
    g = X.xslp_coding_matrix(n, p)
    uniq = sorted(set(pats))
    progs, survs = [], {}
    for er in uniq:
        bits, surv = X.xslp_decode_bitmatrix(g, n, p, er)
        progs.append(X.xslp_compile(bits, **_kernel_kw(dict(kernel={"grouped": "straight", "grouped_tma": "tma",
                                                                   "grouped_pipe": "pipe"}.get(kern, kern)))))
        survs[er] = surv
    idx = torch.tensor([uniq.index(er) for er in pats], dtype=torch.int32, device="cuda")
    surv_blocks = np.stack([blocks[s][survs[pats[s]]] for s in range(S)])
    din = torch.from_numpy(surv_blocks).cuda()
    dout = dev_buf(S, 4, B)
    ti = X.block_table(din, S, n, B)
    to = X.block_table(dout, S, 4, B)
    if kern.startswith("interp"):
        X.xslp_decode_batch_multi(progs, idx, ti, to, S, B)
    elif kern.startswith("grouped"):
        ids, off = X.group_stripes(idx.cpu().numpy(), len(progs))
        X.xslp_decode_batch_grouped(progs, torch.from_numpy(ids).cuda(), off, ti, to, B, nstreams=4)
    else:   # grouped: one launch per pattern over its stripes (host groups)
        for k, pr in enumerate(progs):
            sel = [s for s in range(S) if pats[s] == uniq[k]]
            sti = ti.view(S, n)[sel].contiguous()
            sto = to.view(S, 4)[sel].contiguous()
            X.xslp_encode_batch(pr, sti, sto, len(sel), B)
    torch.cuda.synchronize()
    got = dout.cpu().numpy()
    for s in range(S):
        assert (got[s] == blocks[s][list(pats[s])]).all(), (s, pats[s])


@pytest.mark.parametrize("n,p", [(10, 4), (20, 4)])
def test_tmem_interpreter_kernel_runs(n, p):
    # the TMEM interpreter (tensor-memory variables, the default interpreter) is the kernel that
    # runs, not the fallback: 2 words per thread for RS(10,4), 1 for RS(20,4) (160 constant rows)
    B, S = 65536, 8
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p, kernel="interp", specialise=0)
    data = host_data(12, range(S), n, B)
    din = torch.from_numpy(data).cuda()
    dout = dev_buf(S, p, B)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        run_batch(prog, din, dout, B)
    names = [e.name for e in prof.events() if "xslp" in e.name]
    assert any("xslp_interp_tmem" in nm for nm in names), names
    for s in range(S):
        assert (dout[s].cpu().numpy() == rs.encode(og, n, data[s])).all(), s


# ---- edge cases ------------------------------------------------------------------------

@pytest.mark.parametrize("per_module,hint,threads", [(3, 0, 128), (64, 1, 256), (1, 1, 64)])
def test_multi_program_decode(per_module, hint, threads):
    # heterogeneous decode through fused multi-program pipeline kernels (branch table per
    # stripe), several modules, ragged last tile; every byte against the oracle
    n, p, B, S = 10, 4, 8192 + 1152, 23
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    pats = [tuple(synth.erasure_pattern(71, s, n + p, 4)) for s in range(S)]
    uniq = sorted(set(pats))
    progs = X.compile_many([X.xslp_decode_bitmatrix(g, n, p, er)[0] for er in uniq], specialise=0)
    multi = X.Multi(progs, per_module=per_module, threads=threads, stages=2,
                    block_bytes_hint=B if hint else 0)
    info = multi.info()
    assert info["modules"] == -(-len(uniq) // per_module)
    pos = [uniq.index(er) for er in pats]
    ids, off = X.group_stripes(pos, len(progs))
    din = dev_buf(S, n, B)                        # survivors: arbitrary bytes
    X.xslp_fill_random(din, S, n, B, seed=72)
    out = torch.full((S, 4, B), 0x5A, dtype=torch.uint8, device="cuda")
    X.xslp_multi_decode(multi, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                        torch.from_numpy(ids).cuda(), off, X.block_table(din, S, n, B),
                        X.block_table(out, S, 4, B), B)
    torch.cuda.synchronize()
    for s in range(S):
        rows = mx.decode_rows(og, n, list(pats[s]))[1]
        want = rs.decode(rows, synth.stripe_data(72, s, n, B))
        assert (out[s].cpu().numpy() == want).all(), s
    # the launches (two internal streams for > 1 module) captured in a CUDA graph, replayed
    pos_d = torch.tensor(pos, dtype=torch.int32, device="cuda")
    ids_d = torch.from_numpy(ids).cuda()
    ti, to = X.block_table(din, S, n, B), X.block_table(out, S, 4, B)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        X.xslp_multi_decode(multi, pos_d, ids_d, off, ti, to, B)
    X.xslp_fill_random(din, S, n, B, seed=73)
    gr.replay()
    torch.cuda.synchronize()
    for s in (0, S // 2, S - 1):
        rows = mx.decode_rows(og, n, list(pats[s]))[1]
        assert (out[s].cpu().numpy() == rs.decode(rows, synth.stripe_data(73, s, n, B))).all(), s
    if hint:
        with pytest.raises(X.XslpError):          # kernels were built for B
            X.xslp_multi_decode(multi, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                                torch.from_numpy(ids).cuda(), off, X.block_table(din, S, n, B),
                                X.block_table(out, S, 4, B), B - 128)


def test_program_lifetime_no_stale_interpreter_pool():
    # heterogeneous interpreter launches cache a device pool of the programs' bytecode keyed by
    # the programs; freed programs must not leave a pool a new program at a recycled address
    # would pick up (compare every round with the oracle)
    import gc
    n, p, B, S = 10, 4, 4096, 6
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=101)
    data = din.cpu().numpy()
    for rnd in range(4):
        pats = [tuple(synth.erasure_pattern(200 + rnd, s, n + p, 4)) for s in range(S)]
        uniq = sorted(set(pats))
        progs = [X.xslp_compile(X.xslp_decode_bitmatrix(g, n, p, er)[0], specialise=0) for er in uniq]
        idx = torch.tensor([uniq.index(er) for er in pats], dtype=torch.int32, device="cuda")
        out = torch.zeros((S, 4, B), dtype=torch.uint8, device="cuda")
        X.xslp_decode_batch_multi(progs, idx, X.block_table(din, S, n, B), X.block_table(out, S, 4, B),
                                  S, B)
        torch.cuda.synchronize()
        for s in range(S):
            rows = mx.decode_rows(og, n, list(pats[s]))[1]
            assert (out[s].cpu().numpy() == rs.decode(rows, data[s])).all(), (rnd, s)
        del progs
        gc.collect()


@pytest.mark.parametrize("phases,threads", [(0, 256), (1, 128), (3, 128)])
def test_multi_program_decode_wide_code_phases(phases, threads):
    # RS(20,4) per-stripe erasure patterns through the fused multi-program kernels, with input
    # phases (auto = 2 for 20 blocks, or 3) and without; ragged last tile; against the oracle
    n, p, B, S = 20, 4, 8192 + 1152, 14
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    pats = [tuple(synth.erasure_pattern(121, s, n + p, 4)) for s in range(S)]
    uniq = sorted(set(pats))
    progs = X.compile_many([X.xslp_decode_bitmatrix(g, n, p, er)[0] for er in uniq], specialise=0)
    multi = X.Multi(progs, per_module=5, threads=threads, stages=2, phases=phases)
    pos = [uniq.index(er) for er in pats]
    ids, off = X.group_stripes(pos, len(progs))
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=122)
    out = torch.full((S, 4, B), 0x3C, dtype=torch.uint8, device="cuda")
    X.xslp_multi_decode(multi, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                        torch.from_numpy(ids).cuda(), off, X.block_table(din, S, n, B),
                        X.block_table(out, S, 4, B), B)
    torch.cuda.synchronize()
    for s in range(S):
        rows = mx.decode_rows(og, n, list(pats[s]))[1]
        assert (out[s].cpu().numpy() == rs.decode(rows, synth.stripe_data(122, s, n, B))).all(), s


@pytest.mark.parametrize("n,p,kind,e,phases", [(10, 4, "isal", 4, 0), (20, 4, "isal", 4, 0),
                                                (4, 2, "cauchy", 2, 0), (10, 4, "isal", 2, 0),
                                                (10, 4, "isal", 4, 1), (8, 3, "sysvand", 3, 3)])
def test_syndrome_form_decode(n, p, kind, e, phases):
    # heterogeneous decode in syndrome form: every stripe's full block table (erased entries ->
    # one zero block), the shared syndrome program then the pattern's solve program; the erased
    # blocks of real codewords come back, and the bytes equal the oracle's decode
    B, S = 8192 + 1152, 11
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    pats = [tuple(synth.erasure_pattern(131 + e, s, n + p, e)) for s in range(S)]
    uniq = sorted(set(pats))
    dec = X.SyndromeDecoder(g, n, p, uniq, per_module=4, threads=128, stages=2, phases=phases)
    allb = dev_buf(S, n + p, B)
    X.xslp_fill_random(allb, S, n + p, B, seed=132)
    _, enc = compile_enc(n, p, kind)
    t = X.block_table(allb, S, n + p, B).view(S, n + p)
    X.xslp_encode_batch(enc, t[:, :n].contiguous(), t[:, n:].contiguous(), S, B)
    zero = torch.zeros(B, dtype=torch.uint8, device="cuda")
    tin = t.clone()
    for s, er in enumerate(pats):
        for j in er:
            tin[s, j] = zero.data_ptr()
    out = torch.full((S, e, B), 0x66, dtype=torch.uint8, device="cuda")
    pos = [uniq.index(er) for er in pats]
    ids, off = X.group_stripes(pos, len(uniq))
    X.xslp_multi_decode(dec, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                        torch.from_numpy(ids).cuda(), off, tin.reshape(-1),
                        X.block_table(out, S, e, B), B)
    torch.cuda.synchronize()
    for s, er in enumerate(pats):
        assert torch.equal(out[s], allb[s, list(er)]), (s, er)
    for s in (0, S - 1):                       # the oracle's decode of the same survivors
        d = synth.stripe_data(132, s, n, B)
        blocks = np.concatenate([d, rs.encode(og, n, d)])
        surv, rows = mx.decode_rows(og, n, list(pats[s]))
        assert (out[s].cpu().numpy() == rs.decode(rows, blocks[surv])).all()


@pytest.mark.parametrize("wname", ["cfg3", "cfg5h"])
def test_multi_full_size_bench_config(wname):
    # the configured heterogeneous decode -- the M^-1 bitmatrix SLP of each erasure pattern
    # (BASELINE configs[2]) fused into multi-program kernels -- at full size in the
    # launch configuration bench.py times (cfg3's default line; cfg5h's --kernel multi):
    # every byte of every stripe against the C oracle's codeword
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    wl = bench.WORKLOADS[wname]
    t = wl["tuned"] if wl["tuned"]["kernel"] == "multi" else wl["alt"]["multi"]
    n, p, B, S, e, seed = wl["n"], wl["p"], wl["B"], wl["S"], wl["e"], wl["seed"]
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    pats = [tuple(synth.erasure_pattern(seed, s, n + p, e)) for s in range(S)]
    uniq = sorted(set(pats))
    dec = [X.xslp_decode_bitmatrix(g, n, p, er) for er in uniq]
    progs = X.compile_many([d[0] for d in dec], specialise=0)
    multi = X.Multi(progs, per_module=t["per_module"], threads=t["threads"], stages=t["stages"],
                    block_bytes_hint=B, phases=t.get("phases", 0), reuse=t.get("reuse", 0))
    _, enc = compile_enc(n, p, block_bytes_hint=B)
    allb = dev_buf(S, n + p, B)
    X.xslp_fill_random(allb, S, n + p, B, seed=seed)          # data words do not depend on nblocks
    ti = X.block_table(allb, S, n + p, B).view(S, n + p)
    X.xslp_encode_batch(enc, ti[:, :n].contiguous(), ti[:, n:].contiguous(), S, B)
    pos = [uniq.index(er) for er in pats]
    tin = torch.stack([ti[s_, torch.as_tensor(dec[pos[s_]][1], dtype=torch.long)] for s_ in range(S)])
    out = dev_buf(S, e, B)
    ids, off = X.group_stripes(pos, len(uniq))
    X.xslp_multi_decode(multi, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                        torch.from_numpy(ids).cuda(), off, tin.contiguous(),
                        X.block_table(out, S, e, B), B)
    torch.cuda.synchronize()
    verify_all(allb[:, n:], seed, rows=og[n:])                 # the untimed encode
    verify_all(out, seed, parity_rows=og[n:], n=n, erased=pats)
    del allb, out, tin
    torch.cuda.empty_cache()


@pytest.mark.parametrize("wname", ["cfg3", "cfg5h"])
def test_syndrome_full_size_bench_config(wname):
    # the heterogeneous decode workloads at full size (1024 stripes x 1 MiB, per-stripe seeded
    # 4-erasures) in exactly the launch configuration bench.py times (read from its table):
    # roundtrip on every stripe, the oracle's decode on sampled stripes
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    wl = bench.WORKLOADS[wname]
    t = wl["tuned"] if wl["tuned"]["kernel"] == "syndrome" else dict(wl["alt"]["syndrome"], kernel="syndrome")
    n, p, B, S, e, seed = wl["n"], wl["p"], wl["B"], wl["S"], wl["e"], wl["seed"]
    phases = t.get("phases") or -(-(n + p) // 10)      # bench.py's default for the syndrome form
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    pats = [tuple(synth.erasure_pattern(seed, s, n + p, e)) for s in range(S)]
    uniq = sorted(set(pats))
    dec = X.SyndromeDecoder(g, n, p, uniq, per_module=t["per_module"], threads=t["threads"],
                            stages=t["stages"], phases=phases, block_bytes_hint=B,
                            reuse=t.get("reuse", 0))
    _, enc = compile_enc(n, p, block_bytes_hint=B)
    allb = dev_buf(S, n + p, B)
    data = dev_buf(S, n, B)
    X.xslp_fill_random(data, S, n, B, seed=seed)
    allb[:, :n] = data
    ti = X.block_table(allb, S, n + p, B).view(S, n + p)
    X.xslp_encode_batch(enc, ti[:, :n].contiguous(), ti[:, n:].contiguous(), S, B)
    zero = torch.zeros(B, dtype=torch.uint8, device="cuda")
    tin = ti.clone()
    for s_, er in enumerate(pats):
        for j in er:
            tin[s_, j] = zero.data_ptr()
    out = dev_buf(S, e, B)
    pos = [uniq.index(er) for er in pats]
    ids, off = X.group_stripes(pos, len(uniq))
    X.xslp_multi_decode(dec, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                        torch.from_numpy(ids).cuda(), off, tin.reshape(-1),
                        X.block_table(out, S, e, B), B)
    torch.cuda.synchronize()
    for s_, er in enumerate(pats):                    # every stripe: the erased blocks come back
        assert torch.equal(out[s_], allb[s_, list(er)]), (s_, er)
    for s_ in (0, 613, S - 1):                         # the oracle's blocks and decode
        d = synth.stripe_data(seed, s_, n, B)
        blocks = np.concatenate([d, rs.encode(og, n, d)])
        assert (allb[s_].cpu().numpy() == blocks).all(), s_
        surv, rows = mx.decode_rows(og, n, list(pats[s_]))
        assert (out[s_].cpu().numpy() == rs.decode(rows, blocks[surv])).all(), s_
    verify_all(out, seed, parity_rows=og[n:], n=n, erased=pats)   # every stripe vs the oracle
    del allb, data, out, tin
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,p,kind,er,B,kern", [(10, 4, "isal", None, (16 << 20) + 1152, "auto"),
                                                (10, 4, "isal", (2, 4, 5, 6), 16 << 20, "pipe"),
                                                (4, 2, "cauchy", None, 8 << 20, "pipe"),
                                                (20, 4, "isal", None, 4 << 20, "auto")])
def test_single_stripe_large_blocks(n, p, kind, er, B, kern):
    # one stripe through xslp_encode / xslp_decode (block pointers as kernel arguments): large
    # blocks take the TMA pipeline's single-stripe entry (xslp_sl_pipe_one; RS(20,4) has input
    # phases and keeps the register-resident kernel); every byte equals the oracle's
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    data = synth.stripe_data(61, 0, n, B)
    if er is None:
        bits, rows, ins = X.xslp_encode_bitmatrix(g, n, p), og[n:], data
    else:
        bits, surv = X.xslp_decode_bitmatrix(g, n, p, list(er))
        blocks = np.concatenate([data, rs.encode(og, n, data)])
        osurv, rows = mx.decode_rows(og, n, list(er))
        assert list(surv) == osurv
        ins = blocks[osurv]
    prog = X.xslp_compile(bits, kernel=kern, threads=128, lane_words=2 if n <= 10 else 1)
    din = torch.from_numpy(np.ascontiguousarray(ins)).cuda()
    m = bits.shape[0] // 8
    out = torch.full((m, B), 0x3C, dtype=torch.uint8, device="cuda")
    X.xslp_encode(prog, [din[j] for j in range(n)], [out[i] for i in range(m)], B)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == rs.apply_rows(rows, ins)).all()


def test_edge_cases():
    n, p = 4, 2
    _, prog = compile_enc(n, p, "cauchy")
    d = dev_buf(1, n, 4096)
    o = dev_buf(1, p, 4096)
    ti, to = X.block_table(d, 1, n, 4096), X.block_table(o, 1, p, 4096)
    X.xslp_encode_batch(prog, ti, to, 0, 4096)         # no stripes: no-op
    X.xslp_encode_batch(prog, ti, to, 1, 0)            # empty blocks: no-op
    with pytest.raises(X.XslpError) as e:
        X.xslp_encode_batch(prog, ti, to, 1, 4008)     # strip not whole words
    assert e.value.code == X.XSLP_EINVAL
    with pytest.raises(X.XslpError) as e:
        X.xslp_encode(prog, [d[0, j, 4:] for j in range(n)], [o[0, i] for i in range(p)], 1024)
    assert e.value.code == X.XSLP_EINVAL               # misaligned pointer
    torch.cuda.synchronize()


def test_copy_and_zero_goals_on_device():
    rng = np.random.default_rng(0)
    bits = np.zeros((16, 24), dtype=np.uint8)
    bits[0, 3] = 1
    bits[1, 17] = 1
    bits[2, [1, 2, 5]] = 1
    bits[5, :] = 1
    bits[9:, :] = rng.integers(0, 2, size=(7, 24))
    B = 2048
    data = host_data(8, [0], 3, B)[0]
    want = rs.bitmatrix_apply(bits, data)
    for kern in ("straight", "interp"):
        prog = X.xslp_compile(bits, kernel=kern)
        din = torch.from_numpy(data).cuda()
        out = torch.full((2, B), 0x5A, dtype=torch.uint8, device="cuda")
        X.xslp_encode(prog, [din[j] for j in range(3)], [out[0], out[1]], B)
        torch.cuda.synchronize()
        assert (out.cpu().numpy() == want).all()


@pytest.mark.parametrize("case", range(128))
def test_random_programs_and_launches(case):
    # seeded fuzz over program shape and launch knobs: a random bitmatrix (1-24 input blocks,
    # 1-6 output blocks, random density incl. empty and full rows) through a random launch of
    # the straight-line / TMA / PIPE kernels (threads, words per thread, stages, input phases,
    # reuse window, ragged block size, stripes; every fifth case the single-stripe call) must
    # give the oracle's bytes; launches the library rejects as not fitting (EINVAL) are skipped
    rng = np.random.default_rng(7000 + case)
    n_in, m_out = int(rng.integers(1, 25)), int(rng.integers(1, 7))
    dens = float(rng.choice([0.02, 0.1, 0.3, 0.5, 0.9]))
    bits = (rng.random((8 * m_out, 8 * n_in)) < dens).astype(np.uint8)
    bits[int(rng.integers(0, 8 * m_out))] = 0                      # an all-zero goal
    if case % 3 == 0:
        bits[int(rng.integers(0, 8 * m_out))] = 1                  # a full goal
    kern = ["straight", "tma", "pipe", "pipe"][case % 4] if case < 96 else "interp"
    kw = dict(kernel=kern, threads=int(rng.choice([32, 64, 128, 256])),
              reuse=int(rng.choice([-1, 0, 1, 7, 32, 128])))
    if kern != "tma":
        kw["lane_words"] = int(rng.choice([1, 2]))
    if kern == "pipe":
        kw["stages"] = int(rng.integers(1, 5))
        kw["phases"] = int(rng.integers(0, min(4, n_in) + 1))
    if kern == "interp":                    # the batched interpreters: lanes / pairs / tmem, no JIT
        kw.update(lane_words=int(rng.choice([1, 2, 4])), stages=int(rng.integers(1, 5)),
                  specialise=0, interp=case % 3)
    B = 128 * int(rng.integers(1, 40))
    S = int(rng.integers(1, 5))
    if rng.random() < 0.5:
        kw["block_bytes_hint"] = B
    one = case % 5 == 0                 # the single-stripe call (block pointers by value)
    # schedule knob (drawn last: earlier draws keep their cases): creation order, DFS (P:1279-
    # 1303) or the capacity-bounded greedy schedule at a random capacity
    kw["schedule"] = int(rng.choice([0, 1, 2]))
    kw["greedy_capacity"] = int(rng.choice([4, 16, 64, 512]))
    if one:
        S = 1
    try:
        prog = X.xslp_compile(bits, **kw)
        data = host_data(7000 + case, range(S), n_in, B)
        din = torch.from_numpy(data).cuda()
        out = torch.full((S, m_out, B), 0xA5, dtype=torch.uint8, device="cuda")
        if one:
            X.xslp_encode(prog, [din[0, j] for j in range(n_in)], [out[0, i] for i in range(m_out)], B)
        else:
            run_batch(prog, din, out, B)
        torch.cuda.synchronize()
    except X.XslpError as e:
        assert e.code == X.XSLP_EINVAL, (case, kw, str(e))
        pytest.skip(f"launch rejected: {e}")
    for s_ in range(S):
        assert (out[s_].cpu().numpy() == rs.bitmatrix_apply(bits, data[s_])).all(), (case, kw, B, s_)


@pytest.mark.parametrize("prog", ["rs10enc", "pdec", "rs20dec"])
@pytest.mark.parametrize("cap", [16, 64, 512])
@pytest.mark.parametrize("kern", ["straight", "pipe", "interp"])
def test_greedy_schedule_on_device(prog, cap, kern):
    # programs scheduled by the capacity-bounded bottom-up greedy strategy
    # instead of DFS run through the straight-line, PIPE and interpreter kernels
    # and give the oracle's bytes (RS(10,4) encode, P_dec, an RS(20,4) decode)
    n, p, er = {"rs10enc": (10, 4, None), "pdec": (10, 4, [2, 4, 5, 6]),
                "rs20dec": (20, 4, [0, 5, 21, 23])}[prog]
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    if er is None:
        bits, rows = X.xslp_encode_bitmatrix(g, n, p), og[n:]
    else:
        bits, rows = X.xslp_decode_bitmatrix(g, n, p, er)[0], mx.decode_rows(og, n, er)[1]
    B, S = 16384 + 128, 3                              # ragged last tile
    kw = dict(schedule=2, greedy_capacity=cap, kernel=kern, threads=128)
    if kern == "interp":
        kw.update(specialise=0, lane_words=2)
    prog_ = X.xslp_compile(bits, **kw)
    st = prog_.stats()
    assert st["xor_count"] > 0
    data = host_data(321, range(S), n, B)
    din = torch.from_numpy(data).cuda()
    out = torch.full((S, len(rows), B), 0x77, dtype=torch.uint8, device="cuda")
    run_batch(prog_, din, out, B)
    torch.cuda.synchronize()
    for s_ in range(S):
        assert (out[s_].cpu().numpy() == rs.apply_rows(rows, data[s_])).all(), (prog, cap, kern, s_)


@pytest.mark.parametrize("case", range(24))
def test_random_heterogeneous_decode(case):
    # seeded fuzz of the fused heterogeneous decode: a random code (n, p, matrix kind), random
    # per-stripe erasure patterns (1..p erasures, data and parity mixed), the syndrome form or
    # the M^-1 programs fused, random launch knobs; the erased blocks of real codewords come back
    rng = np.random.default_rng(8000 + case)
    kind = ["isal", "cauchy", "sysvand"][case % 3]
    n, p = int(rng.integers(2, 17)), int(rng.integers(1, 5))
    e = int(rng.integers(1, p + 1))
    S = int(rng.integers(2, 9))
    B = 128 * int(rng.integers(1, 40))
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    pats = [tuple(sorted(rng.choice(n + p, size=e, replace=False).tolist())) for _ in range(S)]
    uniq = sorted(set(pats))
    pos = [uniq.index(er) for er in pats]
    mode = "syndrome" if case % 2 == 0 else "multi"
    kw = dict(threads=int(rng.choice([64, 128, 256])), stages=int(rng.integers(2, 4)),
              reuse=int(rng.choice([-1, 0, 5, 16, 40])))          # fused kernels: 2..8 stages
    pm = int(rng.integers(1, 5))
    data = host_data(8000 + case, range(S), n, B)
    blocks = np.stack([np.concatenate([d, rs.encode(og, n, d)]) for d in data])
    allb = torch.from_numpy(blocks).cuda()
    t = X.block_table(allb, S, n + p, B).view(S, n + p)
    out = torch.full((S, e, B), 0x3C, dtype=torch.uint8, device="cuda")
    try:
        if mode == "syndrome":
            dec = X.SyndromeDecoder(g, n, p, uniq, per_module=pm, phases=int(rng.integers(0, 3)), **kw)
            zero = torch.zeros(B, dtype=torch.uint8, device="cuda")
            tin = t.clone()
            for s_, er in enumerate(pats):
                for j in er:
                    tin[s_, j] = zero.data_ptr()
            tin = tin.reshape(-1)
        else:
            survs = {er: X.xslp_decode_bitmatrix(g, n, p, list(er)) for er in uniq}
            progs = X.compile_many([survs[er][0] for er in uniq], specialise=0)
            dec = X.Multi(progs, per_module=pm, **kw)
            tin = torch.stack([t[s_, torch.as_tensor(survs[pats[s_]][1], dtype=torch.long)]
                               for s_ in range(S)]).contiguous()
        ids, off = X.group_stripes(pos, len(uniq))
        X.xslp_multi_decode(dec, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                            torch.from_numpy(ids).cuda(), off, tin, X.block_table(out, S, e, B), B)
        torch.cuda.synchronize()
    except X.XslpError as ex:
        assert ex.code == X.XSLP_EINVAL, (case, mode, kw, str(ex))
        pytest.skip(f"launch rejected: {ex}")
    for s_, er in enumerate(pats):
        assert (out[s_].cpu().numpy() == blocks[s_, list(er)]).all(), (case, mode, kw, n, p, er)


@pytest.mark.parametrize("kern", ["straight", "tma", "pipe", "interp", "multi"])
def test_copy_and_zero_goals_batched(kern):
    # degenerate goals through the batched kernels (identity rows, all-zero rows, a full row),
    # several stripes, ragged tiles: copies and zeros must be written like any other goal
    rng = np.random.default_rng(1)
    bits = np.zeros((16, 24), dtype=np.uint8)
    bits[0, 3] = 1
    bits[1, 17] = 1
    bits[2, [1, 2, 5]] = 1
    bits[5, :] = 1
    bits[9:, :] = rng.integers(0, 2, size=(7, 24))
    B, S = 2048 + 640, 3                         # 84 words per strip: ragged at every T
    data = host_data(9, range(S), 3, B)
    din = torch.from_numpy(data).cuda()
    out = torch.full((S, 2, B), 0x5A, dtype=torch.uint8, device="cuda")
    ti, to = X.block_table(din, S, 3, B), X.block_table(out, S, 2, B)
    if kern == "multi":
        bits2 = rng.integers(0, 2, size=(16, 24)).astype(np.uint8)
        progs = [X.xslp_compile(b, specialise=0) for b in (bits, bits2)]
        m = X.Multi(progs, per_module=1, threads=64, stages=2)
        pos = [s % 2 for s in range(S)]
        ids, off = X.group_stripes(pos, 2)
        X.xslp_multi_decode(m, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                            torch.from_numpy(ids).cuda(), off, ti, to, B)
        wants = [rs.bitmatrix_apply(bits if s % 2 == 0 else bits2, data[s]) for s in range(S)]
    else:
        prog = X.xslp_compile(bits, kernel=kern, threads=64, specialise=0 if kern == "interp" else 1)
        X.xslp_encode_batch(prog, ti, to, S, B)
        wants = [rs.bitmatrix_apply(bits, data[s]) for s in range(S)]
    torch.cuda.synchronize()
    for s in range(S):
        assert (out[s].cpu().numpy() == wants[s]).all(), (kern, s)


def test_host_buffer_path():
    n, p, B, S = 10, 4, 65536, 40
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p)
    data = host_data(12, range(S), n, B)
    h_in = torch.from_numpy(data).pin_memory()
    h_out = torch.zeros((S, p, B), dtype=torch.uint8).pin_memory()
    X.xslp_encode_host(prog, h_in, h_out, S, B)
    got = h_out.numpy()
    for s in (0, 17, S - 1):
        assert (got[s] == rs.encode(og, n, data[s])).all()
    # all stripes: RAID-5 parity row
    assert (got[:, 0] == np.bitwise_xor.reduce(data, axis=1)).all()


# ---- BASELINE-size cases in the bench launch configuration ------------------------------

def verify_all(got, seed, rows=None, stripe0=0, parity_rows=None, n=None, erased=None, chunk=128,
               bytewise=False):
    """Every byte of every stripe of a device output (S, m, B) against the C oracle
    (oracle/rs_oracle.c, threads over stripes on the host), copied back in chunks.
    rows: the outputs are rows . fill(seed, stripe, n_in, B).  erased: the outputs are the
    codeword blocks erased[s] of [fill(seed, stripe, n, B); parity_rows . data]."""
    S = got.shape[0]
    bad = []
    for a in range(0, S, chunk):
        h = got[a:a + chunk].cpu().numpy()
        if erased is None:
            check = nat.check_bytewise if bytewise else nat.check_apply
            b = check(np.asarray(rows, dtype=np.uint8), seed, stripe0 + a, h)
        else:
            b = nat.check_codeword(np.asarray(parity_rows, dtype=np.uint8), n, seed, stripe0 + a,
                                   np.asarray(erased[a:a + chunk], dtype=np.int32), h)
        bad += [a + int(x) for x in b]
    assert not bad, f"{len(bad)} of {S} stripes differ from the oracle, first {bad[:8]}"


def _xor_reduce(t):
    acc = t[:, 0].clone()
    for j in range(1, t.shape[1]):
        acc ^= t[:, j]
    return acc


@pytest.mark.parametrize("kern,threads,lanes,reuse", [("straight", 128, 1, 0), ("tma", 128, 1, 0),
                                                      ("pipe", 256, 1, 0), ("pipe", 128, 2, "bench"),
                                                      ("interp", 128, 1, 0)])
def test_cfg2_full_size(kern, threads, lanes, reuse):
    # RS(10,4), 1024 stripes x 10 x 1 MiB (configs[1]); ("pipe", 128, 2 lanes) with bench's
    # stages, input phases and reuse window is the exact launch configuration bench.py times
    n, p, B, S = 10, 4, 1 << 20, 1024
    if reuse == "bench":
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        t = bench.WORKLOADS["cfg2"]["tuned"]
        assert (t["kernel"], t["threads"], t["lanes"]) == (kern, threads, lanes)
        reuse, stages, phases = t.get("reuse", 0), t.get("stages", 2), t.get("phases", 0)
    else:
        stages, phases = 2, 0
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p, block_bytes_hint=B, kernel=kern, threads=threads, stages=stages,
                          lane_words=lanes, reuse=reuse, phases=phases)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=2)
    dout = dev_buf(S, p, B)
    run_batch(prog, din, dout, B)
    assert torch.equal(dout[:, 0], _xor_reduce(din))       # RAID-5 row over every stripe
    for s in (0, 511, 1023):
        data = synth.stripe_data(2, s, n, B)
        assert (din[s].cpu().numpy() == data).all()
        assert (dout[s].cpu().numpy() == rs.encode(og, n, data)).all(), s
    verify_all(dout, 2, rows=og[n:])                         # every byte of all 1024 stripes
    del din, dout
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["grouped", "interp", "interp_pairs", "interp_lanes"])
def test_cfg3_full_size_roundtrip(mode):
    # RS(10,4) decode, 1024 stripes x 1 MiB, per-stripe seeded 4-of-14 erasures (configs[2]);
    # "grouped" (per-pattern LDG kernels, T=64, 8 streams) is the bench's launch configuration
    n, p, B, S = 10, 4, 1 << 20, 1024
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    _, enc = compile_enc(n, p, block_bytes_hint=B)
    allb = dev_buf(S, n + p, B)
    X.xslp_fill_random(allb, S, n + p, B, seed=3)            # data part regenerated below
    data = dev_buf(S, n, B)
    X.xslp_fill_random(data, S, n, B, seed=3)
    allb[:, :n] = data
    ti = X.block_table(allb, S, n + p, B).view(S, n + p)
    X.xslp_encode_batch(enc, ti[:, :n].contiguous(), ti[:, n:].contiguous(), S, B)
    pats = [tuple(synth.erasure_pattern(3, s, n + p, 4)) for s in range(S)]
    uniq = sorted(set(pats))
    survs = {}
    bitsl = []
    for er in uniq:
        bits, surv = X.xslp_decode_bitmatrix(g, n, p, er)
        bitsl.append(bits)
        survs[er] = surv
    if mode == "grouped":
        progs = X.compile_many(bitsl, kernel="straight", threads=64, block_bytes_hint=B)
    else:                     # the lane-parallel (default) or the pair-pipelined interpreter
        progs = X.compile_many(bitsl, specialise=0, interp=mode[7:] if "_" in mode else "tmem")
    pos = [uniq.index(er) for er in pats]
    idx = torch.tensor(pos, dtype=torch.int32, device="cuda")
    tin = torch.stack([ti[s, torch.as_tensor(survs[pats[s]], dtype=torch.long)] for s in range(S)])
    out = dev_buf(S, 4, B)
    to = X.block_table(out, S, 4, B)
    if mode == "grouped":
        ids, off = X.group_stripes(pos, len(progs))
        X.xslp_decode_batch_grouped(progs, torch.from_numpy(ids).cuda(), off, tin.contiguous(), to, B,
                                    nstreams=8)
    else:
        X.xslp_decode_batch_multi(progs, idx, tin.contiguous(), to, S, B)
    torch.cuda.synchronize()
    # roundtrip property on every stripe: erased data blocks equal the regenerated data
    for s in range(S):
        for k, e in enumerate(pats[s]):
            if e < n:
                assert torch.equal(out[s, k], data[s, e]), (s, e)
    # oracle on sampled stripes: parity and the decode of the oracle's blocks
    for s in (0, 700):
        d = synth.stripe_data(3, s, n, B)
        blocks = np.concatenate([d, rs.encode(og, n, d)])
        assert (allb[s].cpu().numpy() == blocks).all()
        surv, rows = mx.decode_rows(og, n, list(pats[s]))
        assert (out[s].cpu().numpy() == rs.decode(rows, blocks[surv])).all()
    # every stripe: the parity the encode wrote, and the recovered blocks = the oracle codeword
    verify_all(allb[:, n:], 3, rows=og[n:])
    verify_all(out, 3, parity_rows=og[n:], n=n, erased=pats)
    del allb, data, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("threads,lanes", [(256, 1), (128, 2)])
def test_pdec_full_size(threads, lanes):
    # the paper's P_dec (erase {2,4,5,6}) on 1024 stripes x 1 MiB in bench's launch configuration
    n, p, B, S = 10, 4, 1 << 20, 1024
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    bits, surv = X.xslp_decode_bitmatrix(g, n, p, [2, 4, 5, 6])
    dec = X.xslp_compile(bits, kernel="pipe", threads=threads, lane_words=lanes, stages=2,
                         block_bytes_hint=B)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=3)          # survivors: arbitrary bytes
    out = dev_buf(S, 4, B)
    run_batch(dec, din, out, B)
    osurv, rows = mx.decode_rows(og, n, [2, 4, 5, 6])
    assert list(surv) == osurv
    for s in (0, 777, 1023):
        assert (out[s].cpu().numpy() == rs.decode(rows, din[s].cpu().numpy())).all(), s
    verify_all(out, 3, rows=rows)                            # every byte of all 1024 stripes
    del din, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("groups", [2, 3, 4])
@pytest.mark.parametrize("case", ["rs10enc", "rs20dec", "cauchy42"])
def test_pipe_consumer_groups(groups, case):
    # PIPE kernel with the goals split over consumer groups: every output byte equals the
    # oracle; ragged last tile (words not a multiple of the group width), baked and generic
    if case == "rs10enc":
        n, p, kind, er = 10, 4, "isal", None
    elif case == "rs20dec":
        n, p, kind, er = 20, 4, "isal", [0, 5, 21, 23]
    else:
        n, p, kind, er = 4, 2, "cauchy", None
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    B, S = 8192 + 1152, 5                     # 292 words per strip: 2 tiles of 128 + a ragged 36
    if er is None:
        bits, rows, m = X.xslp_encode_bitmatrix(g, n, p), og[n:], p
    else:
        bits, _ = X.xslp_decode_bitmatrix(g, n, p, er)
        rows, m = mx.decode_rows(og, n, er)[1], len(er)
    for hint in (0, B):
        prog = X.xslp_compile(bits, kernel="pipe", threads=128, stages=2, groups=groups,
                              block_bytes_hint=hint)
        st = prog.stats()
        assert st["group_xor"] >= st["xor_count"]
        din = dev_buf(S, n, B)
        X.xslp_fill_random(din, S, n, B, seed=61 + groups)
        dout = torch.full((S, m, B), 0xA5, dtype=torch.uint8, device="cuda")
        run_batch(prog, din, dout, B)
        for s in range(S):
            want = rs.apply_rows(rows, synth.stripe_data(61 + groups, s, n, B))
            assert (dout[s].cpu().numpy() == want).all(), (case, groups, hint, s)


@pytest.mark.parametrize("phases,threads,lanes", [(2, 256, 1), (3, 128, 1), (4, 64, 1), (2, 128, 2)])
@pytest.mark.parametrize("case", ["rs20enc", "rs20dec", "rs10dec", "cauchy42"])
def test_pipe_input_phases(phases, threads, lanes, case):
    # PIPE with the inputs streamed in phases (K-split) and goal partials accumulated in
    # registers: every output byte equals the oracle; ragged last tile, baked and generic
    n, p, kind, er = {"rs20enc": (20, 4, "isal", None), "rs20dec": (20, 4, "isal", [0, 5, 21, 23]),
                      "rs10dec": (10, 4, "isal", [2, 4, 5, 6]), "cauchy42": (4, 2, "cauchy", None)}[case]
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    B, S = 8192 + 1152, 3                     # 292 words per strip: ragged last tile
    if er is None:
        bits, rows, m = X.xslp_encode_bitmatrix(g, n, p), og[n:], p
    else:
        bits, _ = X.xslp_decode_bitmatrix(g, n, p, er)
        rows, m = mx.decode_rows(og, n, er)[1], len(er)
    for hint in (0, B):
        prog = X.xslp_compile(bits, kernel="pipe", threads=threads, stages=2, phases=phases,
                              lane_words=lanes, block_bytes_hint=hint)
        assert prog.stats()["group_xor"] >= prog.stats()["xor_count"]
        din = dev_buf(S, n, B)
        X.xslp_fill_random(din, S, n, B, seed=91 + phases)
        dout = torch.full((S, m, B), 0x5C, dtype=torch.uint8, device="cuda")
        run_batch(prog, din, dout, B)
        for s in range(S):
            want = rs.apply_rows(rows, synth.stripe_data(91 + phases, s, n, B))
            assert (dout[s].cpu().numpy() == want).all(), (case, phases, hint, s)


@pytest.mark.parametrize("reuse", [-1, 1, 3, 16, 64, 4096])
@pytest.mark.parametrize("kern", ["pipe", "tma", "syndrome"])
def test_const_reuse_window(reuse, kern):
    # the constant register reuse window only changes which shared-memory reads the emitted
    # code repeats: every window gives the oracle's bytes (PIPE with input phases, the TMA
    # kernel, the syndrome-form decode), ragged last tile
    n, p = 20, 4
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    B, S = 8192 + 1152, 3
    if kern == "syndrome":
        pats = [(0, 5, 21, 23), (1, 2, 3, 4), (20, 21, 22, 23)]
        dec = X.SyndromeDecoder(g, n, p, pats, per_module=2, threads=128, stages=2, reuse=reuse)
        allb = dev_buf(S, n + p, B)
        X.xslp_fill_random(allb, S, n + p, B, seed=97)
        _, enc = compile_enc(n, p)
        t = X.block_table(allb, S, n + p, B).view(S, n + p)
        X.xslp_encode_batch(enc, t[:, :n].contiguous(), t[:, n:].contiguous(), S, B)
        zero = torch.zeros(B, dtype=torch.uint8, device="cuda")
        tin = t.clone()
        for s_, er in enumerate(pats):
            for j in er:
                tin[s_, j] = zero.data_ptr()
        out = torch.full((S, 4, B), 0x5C, dtype=torch.uint8, device="cuda")
        pos = list(range(S))
        ids, off = X.group_stripes(pos, S)
        X.xslp_multi_decode(dec, torch.tensor(pos, dtype=torch.int32, device="cuda"),
                            torch.from_numpy(ids).cuda(), off, tin.reshape(-1),
                            X.block_table(out, S, 4, B), B)
        torch.cuda.synchronize()
        for s_, er in enumerate(pats):
            d = synth.stripe_data(97, s_, n, B)
            blocks = np.concatenate([d, rs.encode(og, n, d)])
            assert (out[s_].cpu().numpy() == blocks[list(er)]).all(), (reuse, s_)
        return
    er = [0, 5, 21, 23]
    bits, _ = X.xslp_decode_bitmatrix(g, n, p, er)
    rows = mx.decode_rows(og, n, er)[1]
    prog = X.xslp_compile(bits, kernel=kern, threads=128, stages=2, block_bytes_hint=B, reuse=reuse)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=98)
    dout = torch.full((S, 4, B), 0x5C, dtype=torch.uint8, device="cuda")
    run_batch(prog, din, dout, B)
    for s_ in range(S):
        want = rs.apply_rows(rows, synth.stripe_data(98, s_, n, B))
        assert (dout[s_].cpu().numpy() == want).all(), (kern, reuse, s_)


@pytest.mark.parametrize("kern", ["straight", "tma", "pipe"])
def test_cfg5_rs20_reduced(kern):
    # RS(20,4) encode + one seeded 4-erasure decode; 16 stripes x 20 x 1 MiB (configs[4] shape)
    n, p, B, S = 20, 4, 1 << 20, 16
    og = mx.coding_matrix(n, p)
    g, enc = compile_enc(n, p, block_bytes_hint=B, kernel=kern, threads=64)
    allb = dev_buf(S, n + p, B)
    X.xslp_fill_random(allb, S, n + p, B, seed=5)
    d = dev_buf(S, n, B)
    X.xslp_fill_random(d, S, n, B, seed=5)
    allb[:, :n] = d
    ti = X.block_table(allb, S, n + p, B).view(S, n + p)
    X.xslp_encode_batch(enc, ti[:, :n].contiguous(), ti[:, n:].contiguous(), S, B)
    er = synth.erasure_pattern(5, 0, n + p, 4)
    bits, surv = X.xslp_decode_bitmatrix(g, n, p, er)
    dec = X.xslp_compile(bits, block_bytes_hint=B, kernel=kern, threads=64)
    out = dev_buf(S, 4, B)
    X.xslp_encode_batch(dec, ti[:, torch.as_tensor(surv, dtype=torch.long)].contiguous(),
                        X.block_table(out, S, 4, B), S, B)
    torch.cuda.synchronize()
    assert torch.equal(out, allb[:, er])
    s = 9
    h = synth.stripe_data(5, s, n, B)
    assert (allb[s, n:].cpu().numpy() == rs.encode(og, n, h)).all()


def test_cfg5_full_chunk():
    # RS(20,4) encode and the seeded 4-erasure decode (configs[4]) over one bench launch: a chunk
    # of 2048 stripes x 24 x 1 MiB, PIPE T=256 S=2 with 2 input phases (bench.py cfg5 / cfg5d
    # launch configuration)
    n, p, B, S = 20, 4, 1 << 20, 2048
    og = mx.coding_matrix(n, p)
    g, enc = compile_enc(n, p, block_bytes_hint=B, kernel="pipe", threads=256, stages=2, phases=2)
    allb = dev_buf(S, n + p, B)
    X.xslp_fill_random(allb, S, n + p, B, seed=5)   # data words do not depend on nblocks
    ti = X.block_table(allb, S, n + p, B).view(S, n + p)
    X.xslp_encode_batch(enc, ti[:, :n].contiguous(), ti[:, n:].contiguous(), S, B)
    er = synth.erasure_pattern(5, 0, n + p, 4)
    bits, surv = X.xslp_decode_bitmatrix(g, n, p, er)
    dec = X.xslp_compile(bits, block_bytes_hint=B, kernel="pipe", threads=256, stages=2, phases=2)
    out = dev_buf(S, 4, B)
    X.xslp_encode_batch(dec, ti[:, torch.as_tensor(surv, dtype=torch.long)].contiguous(),
                        X.block_table(out, S, 4, B), S, B)
    torch.cuda.synchronize()
    assert torch.equal(allb[:, n], _xor_reduce(allb[:, :n]))     # RAID-5 row, every stripe
    assert torch.equal(out, allb[:, torch.as_tensor(er, dtype=torch.long)])  # roundtrip
    osurv, rows = mx.decode_rows(og, n, list(er))
    assert list(surv) == osurv
    for s in (0, 1337, 2047):
        d = synth.stripe_data(5, s, n, B)
        blocks = np.concatenate([d, rs.encode(og, n, d)])
        assert (allb[s].cpu().numpy() == blocks).all(), s
        assert (out[s].cpu().numpy() == rs.decode(rows, blocks[osurv])).all(), s
    # every stripe of the chunk: the 4 parity blocks, and the recovered blocks vs the codeword
    verify_all(allb[:, n:], 5, rows=og[n:], chunk=64)
    verify_all(out, 5, parity_rows=og[n:], n=n, erased=[er] * S, chunk=64)
    del allb, out
    torch.cuda.empty_cache()


def test_rs20_heterogeneous_grouped_pipe_with_phases():
    # RS(20,4) per-stripe erasure patterns through the grouped path with PIPE kernels, whose
    # default (auto) input phases read stripes through the stripe-id lists
    n, p, B, S = 20, 4, 16384, 12
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    pats = [tuple(synth.erasure_pattern(111, s, n + p, 4)) for s in range(S)]
    uniq = sorted(set(pats))
    progs = X.compile_many([X.xslp_decode_bitmatrix(g, n, p, er)[0] for er in uniq],
                           kernel="pipe", threads=128, stages=2, block_bytes_hint=B)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=112)
    out = torch.zeros((S, 4, B), dtype=torch.uint8, device="cuda")
    ids, off = X.group_stripes([uniq.index(er) for er in pats], len(progs))
    X.xslp_decode_batch_grouped(progs, torch.from_numpy(ids).cuda(), off,
                                X.block_table(din, S, n, B), X.block_table(out, S, 4, B), B,
                                nstreams=4)
    torch.cuda.synchronize()
    for s in range(S):
        rows = mx.decode_rows(og, n, list(pats[s]))[1]
        assert (out[s].cpu().numpy() == rs.decode(rows, synth.stripe_data(112, s, n, B))).all(), s


def test_shards_equal_single_run():
    # 8-shard decomposition run serially on one GPU equals the 1-shard run
    n, p, B, S = 10, 4, 65536, 64
    _, prog = compile_enc(n, p, block_bytes_hint=B)
    full_in = dev_buf(S, n, B)
    X.xslp_fill_random(full_in, S, n, B, seed=21)
    full_out = dev_buf(S, p, B)
    run_batch(prog, full_in, full_out, B)
    per = S // 8
    for r in range(8):
        si = dev_buf(per, n, B)
        X.xslp_fill_random(si, per, n, B, seed=21, stripe0=r * per)
        so = dev_buf(per, p, B)
        run_batch(prog, si, so, B)
        assert torch.equal(so, full_out[r * per:(r + 1) * per])


# ---- byte-compatible layout: outputs = textbook byte-wise RS -------

@pytest.mark.parametrize("kern", ["straight", "pipe"])
@pytest.mark.parametrize("n,p,kind,B,S", [(10, 4, "isal", 8224, 3), (4, 2, "cauchy", 4096, 2),
                                          (20, 4, "isal", 1 << 16, 2)])
def test_byte_layout_encode_decode(n, p, kind, B, S, kern):
    og = mx.coding_matrix(n, p, kind)
    g, prog = compile_enc(n, p, kind, layout="byte", kernel=kern)
    data = host_data(31, range(S), n, B)
    din = torch.from_numpy(data).cuda()
    dout = torch.full((S, p, B), 0x77, dtype=torch.uint8, device="cuda")
    run_batch(prog, din, dout, B)
    got = dout.cpu().numpy()
    blocks = []
    for s in range(S):
        want = rs.bytewise_apply(og[n:], data[s])
        assert (got[s] == want).all(), s
        blocks.append(np.concatenate([data[s], want]))
    # decode a few patterns with the byte-layout decode program (single-stripe entry)
    for er in [list(range(p)), list(range(n, n + p)), [1, n + p - 1][:p]]:
        bits, surv = X.xslp_decode_bitmatrix(g, n, p, er)
        dec = X.xslp_compile(bits, layout="byte")
        db = torch.from_numpy(blocks[0]).cuda()
        out = torch.zeros((len(er), B), dtype=torch.uint8, device="cuda")
        X.xslp_decode(dec, [db[k] for k in surv], [out[i] for i in range(len(er))], B)
        torch.cuda.synchronize()
        assert (out.cpu().numpy() == blocks[0][er]).all(), er


@pytest.mark.parametrize("n,p,kind,B,S", [(10, 4, "isal", 4096 + 48, 3), (4, 2, "cauchy", 4096, 2),
                                          (20, 4, "isal", 1024, 2), (6, 8, "sysvand", 160, 2)])
def test_gf_table_kernel(n, p, kind, B, S):
    # approach (1): byte-wise GF(2^8) MM with nibble tables, against the oracle's byte RS and
    # against the XOR-SLP byte-layout program of the same rows
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=81)
    out = torch.full((S, p, B), 0x33, dtype=torch.uint8, device="cuda")
    X.xslp_gf_table_apply(g[n:], X.block_table(din, S, n, B), X.block_table(out, S, p, B), S, B)
    torch.cuda.synchronize()
    for s in range(S):
        want = rs.bytewise_apply(og[n:], synth.stripe_data(81, s, n, B))
        assert (out[s].cpu().numpy() == want).all(), s
    if B % 32 == 0:
        _, prog = compile_enc(n, p, kind, layout="byte")
        out2 = dev_buf(S, p, B)
        run_batch(prog, din, out2, B)
        assert torch.equal(out, out2)
    # decode rows (a data + a parity erasure) through the same kernel
    er = [1, n]
    surv, rows = mx.decode_rows(og, n, er)
    blocks = np.stack([np.concatenate([d, rs.bytewise_apply(og[n:], d)])
                       for d in (synth.stripe_data(81, s, n, B) for s in range(S))])
    dsv = torch.from_numpy(np.ascontiguousarray(blocks[:, surv])).cuda()
    rec = dev_buf(S, len(er), B)
    X.xslp_gf_table_apply(np.array(rows, dtype=np.uint8), X.block_table(dsv, S, n, B),
                          X.block_table(rec, S, len(er), B), S, B)
    torch.cuda.synchronize()
    assert (rec.cpu().numpy() == blocks[:, er]).all()


def test_gf_table_full_size():
    # approach (1) at bench cfg2t's size: RS(10,4) byte-wise encode of 1024 stripes x 10 x 1 MiB;
    # row 0 of [I; 2^(ij)] is all ones, so parity 0 = XOR of the data on every stripe
    n, p, B, S = 10, 4, 1 << 20, 1024
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=2)
    out = dev_buf(S, p, B)
    X.xslp_gf_table_apply(g[n:], X.block_table(din, S, n, B), X.block_table(out, S, p, B), S, B)
    torch.cuda.synchronize()
    assert torch.equal(out[:, 0], _xor_reduce(din))
    for s in (0, 401, 1023):
        want = rs.bytewise_apply(og[n:], synth.stripe_data(2, s, n, B))
        assert (out[s].cpu().numpy() == want).all(), s
    verify_all(out, 2, rows=og[n:], bytewise=True)           # every byte of all 1024 stripes
    del din, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kern,threads", [("straight", 128), ("pipe", 128), ("pipe", 256)])
def test_byte_layout_full_size(kern, threads):
    n, p, B, S = 10, 4, 1 << 20, 1024
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p, layout="byte", block_bytes_hint=B, kernel=kern, threads=threads)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=2)
    dout = dev_buf(S, p, B)
    run_batch(prog, din, dout, B)
    assert torch.equal(dout[:, 0], _xor_reduce(din))
    for s in (5, 1000):
        d = synth.stripe_data(2, s, n, B)
        assert (dout[s].cpu().numpy() == rs.bytewise_apply(og[n:], d)).all()
    verify_all(dout, 2, rows=og[n:], bytewise=True)          # every byte of all 1024 stripes
    del din, dout
    torch.cuda.empty_cache()


# ---- CUDA graphs: launches are capturable after xslp_prepare -----------------------------

@pytest.mark.parametrize("kern", ["pipe", "straight", "interp", "interp_pairs", "interp_lanes", "pipe_phases",
                                  "pipe_byte"])
def test_cuda_graph_capture(kern):
    n, p, B, S = (20, 4, 65536, 32) if kern == "pipe_phases" else (10, 4, 65536, 64)
    og = mx.coding_matrix(n, p)
    if kern == "pipe_byte":
        _, prog = compile_enc(n, p, kernel="pipe", threads=128, layout="byte", block_bytes_hint=B)
    else:
        _, prog = compile_enc(n, p, kernel=kern if kern.startswith("interp_") else kern.split("_")[0],
                              threads=256 if kern.startswith("pipe") else 128,
                              block_bytes_hint=B, phases=2 if kern == "pipe_phases" else 1)
    X.xslp_prepare(prog, B)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=44)
    dout = torch.zeros((S, p, B), dtype=torch.uint8, device="cuda")
    ti, to = X.block_table(din, S, n, B), X.block_table(dout, S, p, B)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.xslp_encode_batch(prog, ti, to, S, B)
    assert not dout.any()                       # capture does not execute
    g.replay()
    torch.cuda.synchronize()
    enc = (lambda d: rs.bytewise_apply(og[n:], d)) if kern == "pipe_byte" else (lambda d: rs.encode(og, n, d))
    for s in (0, S - 1):
        assert (dout[s].cpu().numpy() == enc(synth.stripe_data(44, s, n, B))).all()
    X.xslp_fill_random(din, S, n, B, seed=45)   # replay on new inputs
    g.replay()
    torch.cuda.synchronize()
    assert (dout[3].cpu().numpy() == enc(synth.stripe_data(45, 3, n, B))).all()


def test_cuda_graph_single_stripe_pipeline():
    # the single-stripe pipeline entry (pointers as kernel parameters) captured after
    # xslp_prepare; the graph replays on new data in the same buffers
    n, p, B = 10, 4, 4 << 20
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p, kernel="pipe", threads=128, lane_words=2)
    X.xslp_prepare(prog, B)
    din = dev_buf(1, n, B)
    out = torch.zeros((p, B), dtype=torch.uint8, device="cuda")
    ins, outs = X.block_ptrs([din[0, j] for j in range(n)]), X.block_ptrs([out[i] for i in range(p)])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.xslp_encode(prog, ins, outs, B)
    for seed in (71, 72):
        X.xslp_fill_random(din, 1, n, B, seed=seed)
        g.replay()
        torch.cuda.synchronize()
        assert (out.cpu().numpy() == rs.encode(og, n, synth.stripe_data(seed, 0, n, B))).all(), seed


def test_cuda_graph_grouped_decode():
    # heterogeneous decode (per-pattern kernels forked over internal streams) captured into one
    # graph (bench.py cfg3 --graph 1); replays equal the oracle's decode, also on new inputs
    n, p, B, S = 10, 4, 8192, 40
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    pats = [tuple(synth.erasure_pattern(46, s, n + p, 4)) for s in range(S)]
    uniq = sorted(set(pats))
    dec = [X.xslp_decode_bitmatrix(g, n, p, er) for er in uniq]
    progs = X.compile_many([d[0] for d in dec], kernel="straight", threads=64, block_bytes_hint=B)
    for pr in progs:
        X.xslp_prepare(pr, B)
    din = dev_buf(S, n, B)                       # survivors: arbitrary bytes
    out = torch.zeros((S, 4, B), dtype=torch.uint8, device="cuda")
    ti, to = X.block_table(din, S, n, B), X.block_table(out, S, 4, B)
    ids, off = X.group_stripes([uniq.index(er) for er in pats], len(progs))
    ids = torch.from_numpy(ids).cuda()
    X.xslp_decode_batch_grouped(progs, ids, off, ti, to, B, nstreams=4)   # streams created
    torch.cuda.synchronize()
    out.zero_()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        X.xslp_decode_batch_grouped(progs, ids, off, ti, to, B, nstreams=4,
                                    stream=torch.cuda.current_stream())
    assert not out.any()
    for seed in (47, 48):
        X.xslp_fill_random(din, S, n, B, seed=seed)
        gr.replay()
        torch.cuda.synchronize()
        for s in (0, 17, S - 1):
            rows = mx.decode_rows(og, n, list(pats[s]))[1]
            want = rs.decode(rows, synth.stripe_data(seed, s, n, B))
            assert (out[s].cpu().numpy() == want).all(), (seed, s)


def test_cuda_graph_syndrome_decode():
    # the syndrome-form heterogeneous decode (several modules over the two internal streams)
    # captured into one graph, as bench.py's cfg3 / cfg5h replay it; replays on two codeword
    # sets recover the erased blocks
    n, p, B, S = 10, 4, 16384, 48
    g = X.xslp_coding_matrix(n, p)
    pats = [tuple(synth.erasure_pattern(49, s, n + p, 4)) for s in range(S)]
    uniq = sorted(set(pats))
    dec = X.SyndromeDecoder(g, n, p, uniq, per_module=8, threads=256, reuse=40, block_bytes_hint=B)
    assert dec.info()["modules"] >= 3
    _, enc = compile_enc(n, p, block_bytes_hint=B)
    allb = dev_buf(S, n + p, B)
    t = X.block_table(allb, S, n + p, B).view(S, n + p)
    zero = torch.zeros(B, dtype=torch.uint8, device="cuda")
    tin = t.clone()
    for s_, er in enumerate(pats):
        for j in er:
            tin[s_, j] = zero.data_ptr()
    tin = tin.reshape(-1).contiguous()
    out = torch.zeros((S, 4, B), dtype=torch.uint8, device="cuda")
    to = X.block_table(out, S, 4, B)
    pos = [uniq.index(er) for er in pats]
    ids, off = X.group_stripes(pos, len(uniq))
    posd, idsd = torch.tensor(pos, dtype=torch.int32, device="cuda"), torch.from_numpy(ids).cuda()
    X.xslp_multi_decode(dec, posd, idsd, off, tin, to, B)        # internal streams created
    torch.cuda.synchronize()
    out.zero_()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        X.xslp_multi_decode(dec, posd, idsd, off, tin, to, B, stream=torch.cuda.current_stream())
    assert not out.any()
    for seed in (50, 51):
        X.xslp_fill_random(allb, S, n + p, B, seed=seed)
        X.xslp_encode_batch(enc, t[:, :n].contiguous(), t[:, n:].contiguous(), S, B)
        gr.replay()
        torch.cuda.synchronize()
        for s_, er in enumerate(pats):
            assert torch.equal(out[s_], allb[s_, list(er)]), (seed, s_, er)


# ---- size edges: the 65535 grid-row limit and the widest supported code ------------------

@pytest.mark.parametrize("kern", ["straight", "tma", "pipe", "interp"])
def test_many_stripes_beyond_grid_limit(kern):
    n, p, B, S = 4, 2, 128, 70000           # > 65535 stripes: launches are chunked
    og = mx.coding_matrix(n, p, "cauchy")
    _, prog = compile_enc(n, p, "cauchy", kernel=kern, threads=64)
    din = dev_buf(S, n, B)
    X.xslp_fill_random(din, S, n, B, seed=8)
    dout = torch.zeros((S, p, B), dtype=torch.uint8, device="cuda")
    run_batch(prog, din, dout, B)
    for s in (0, 65534, 65535, 65536, S - 1):
        assert (dout[s].cpu().numpy() == rs.encode(og, n, synth.stripe_data(8, s, n, B))).all(), s


def test_widest_code_rs60_4():
    n, p, B, S = 60, 4, 4096, 2             # 480 constants, 64 blocks per stripe
    og = mx.coding_matrix(n, p)
    _, prog = compile_enc(n, p, threads=64)
    data = host_data(6, range(S), n, B)
    din = torch.from_numpy(data).cuda()
    dout = dev_buf(S, p, B)
    run_batch(prog, din, dout, B)
    for s in range(S):
        assert (dout[s].cpu().numpy() == rs.encode(og, n, data[s])).all()


def test_concurrent_host_threads():
    # programs and the library are shared by host threads launching on their own streams
    from concurrent.futures import ThreadPoolExecutor
    n, p, B, S = 10, 4, 65536, 16
    og = mx.coding_matrix(n, p)
    progs = {k: compile_enc(n, p, kernel=k, threads=64)[1] for k in ("pipe", "straight", "interp")}

    def work(i):
        kern = ("pipe", "straight", "interp")[i % 3]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            din = dev_buf(S, n, B)
            X.xslp_fill_random(din, S, n, B, seed=100 + i, stream=st)
            dout = dev_buf(S, p, B)
            X.xslp_encode_batch(progs[kern], X.block_table(din, S, n, B), X.block_table(dout, S, p, B),
                                S, B, stream=st)
            st.synchronize()
            s = i % S
            return bool((dout[s].cpu().numpy() ==
                         rs.encode(og, n, synth.stripe_data(100 + i, s, n, B))).all())

    with ThreadPoolExecutor(6) as ex:
        assert all(ex.map(work, range(12)))


# ---- cross-GPU decode over peer memory ------------------------------
# One GPU here: the ranks are emulated in one process (their storages on cuda:0, the decode
# tables built by the same code with the exporter's addresses), and the IPC path is exercised
# by two processes sharing cuda:0 (no kernel waits on another; host barriers order the work).

def _peer_setup(world, S, B, seed, e):
    from paper_2108_02692_b200 import peer
    n, p = 10, 4
    g = X.xslp_coding_matrix(n, p)
    enc = X.xslp_compile(X.xslp_encode_bitmatrix(g, n, p), block_bytes_hint=B)
    pl = peer.Placement(n, p, world, S)
    stores = []
    for r in range(world):
        st = torch.zeros(pl.storage_shape(B), dtype=torch.uint8, device="cuda")
        peer.fill_storage(X, pl, r, st, seed, enc, chunk=8)
        stores.append(st)
    er = lambda s: synth.erasure_pattern(seed, s, n + p, e)   # noqa: E731
    return peer, g, pl, stores, er


@pytest.mark.parametrize("world,e", [(2, 4), (3, 3), (8, 2)])
def test_peer_decode_emulated_ranks(world, e):
    n, p, B, S = 10, 4, 65536, 24
    og = mx.coding_matrix(n, p)
    peer, g, pl, stores, er = _peer_setup(world, S, B, 51, e)
    bases = []
    for st in stores:                                   # same-process export/open round trip
        a = X.xslp_peer_open(X.xslp_peer_export(st[1]))
        assert a == st[1].data_ptr()
        X.xslp_peer_close(a)
        bases.append(st.data_ptr())
    for r in range(world):
        plan = peer.Plan(pl, r, er)
        progs = peer.compile_plan(X, g, plan, kernel="straight", threads=64, block_bytes_hint=B)
        out = torch.zeros((len(plan.stripes), plan.e, B), dtype=torch.uint8, device="cuda")
        tin = torch.from_numpy(plan.in_table(bases, B).reshape(-1)).cuda()
        tout = torch.from_numpy(plan.out_table(out.data_ptr(), B).reshape(-1)).cuda()
        ids, off = plan.groups()
        X.xslp_decode_batch_grouped(progs, torch.from_numpy(ids).cuda(), off, tin, tout, B, nstreams=4)
        torch.cuda.synchronize()
        if world == 2:   # the same tables through the fused multi-program kernels
            out2 = torch.zeros_like(out)
            m = X.Multi(progs, per_module=3, threads=128, stages=2, block_bytes_hint=B)
            X.xslp_multi_decode(m, torch.tensor(plan.key_of, dtype=torch.int32, device="cuda"),
                                torch.from_numpy(ids).cuda(), off, tin,
                                torch.from_numpy(plan.out_table(out2.data_ptr(), B).reshape(-1)).cuda(), B)
            torch.cuda.synchronize()
            assert torch.equal(out2, out)
        for i, s in enumerate(plan.stripes):
            erased, surv = plan.keys[plan.key_of[i]]
            d = synth.stripe_data(51, s, n, B)
            blocks = np.concatenate([d, rs.encode(og, n, d)])
            if i < 3:                                   # oracle decode of the survivors read
                rows = mx.decode_rows_from(og, n, list(erased), list(surv))
                assert (out[i].cpu().numpy() == rs.decode(rows, blocks[list(surv)])).all()
            assert (out[i].cpu().numpy() == blocks[list(erased)]).all(), (r, s)


def _ipc_worker(rank, world, port, q, kernel="straight", devices=1, erased_const=None):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = False
    try:
        torch.cuda.set_device(rank % devices)
        from paper_2108_02692_b200 import peer
        n, p, B, S, seed = 10, 4, 65536, 16, 52
        g = X.xslp_coding_matrix(n, p)
        enc = X.xslp_compile(X.xslp_encode_bitmatrix(g, n, p), block_bytes_hint=B)
        pl = peer.Placement(n, p, world, S)
        st = torch.zeros(pl.storage_shape(B), dtype=torch.uint8, device="cuda")
        peer.fill_storage(X, pl, rank, st, seed, enc, chunk=8)
        if erased_const is not None:
            er = lambda s: erased_const                          # noqa: E731
        else:
            er = lambda s: synth.erasure_pattern(seed, s, n + p, 3)   # noqa: E731
        plan = peer.Plan(pl, rank, er)
        multi = None
        if kernel == "straight":
            progs = peer.compile_plan(X, g, plan, kernel="straight", threads=64, block_bytes_hint=B)
        elif kernel == "pipe":       # TMA bulk copies of the peer strips (opt-in path)
            progs = peer.compile_plan(X, g, plan, kernel="pipe", threads=128, lane_words=2, stages=2,
                                      block_bytes_hint=B)
        else:                        # the fused multi-program kernels over peer tables
            progs = peer.compile_plan(X, g, plan, specialise=0)
            multi = X.Multi(progs, per_module=4, threads=128, stages=2, block_bytes_hint=B)
        out = torch.zeros((len(plan.stripes), plan.e, B), dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        dist.barrier()                                  # every storage written
        dec = peer.PeerDecoder(X, pl, st, out, plan, progs, dist=dist, multi=multi,
                               tma=kernel != "straight")
        assert len(dec.mapped) == world - 1
        dec.launch()
        torch.cuda.synchronize()
        # expected bytes: this rank regenerates every codeword of its home stripes locally
        full = torch.zeros((S, n + p, B), dtype=torch.uint8, device="cuda")
        X.xslp_fill_random(full, S, n + p, B, seed=seed)
        t = X.block_table(full, S, n + p, B).view(S, n + p)
        X.xslp_encode_batch(enc, t[:, :n].contiguous(), t[:, n:].contiguous(), S, B)
        torch.cuda.synchronize()
        ok = all(torch.equal(out[i], full[s, list(plan.keys[plan.key_of[i]][0])])
                 for i, s in enumerate(plan.stripes))
        rem, tot = plan.remote_reads()
        ok = ok and rem > 0
        dist.barrier()                                  # all reads done before unmapping
        dec.close()
        dist.barrier()
    finally:
        q.put((rank, ok))
        dist.destroy_process_group()


def _run_ipc(kernel, devices, erased_const=None, world=2):
    import os
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + (os.getpid() + 7 * len(kernel) + devices) % 97
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q, kernel, devices, erased_const))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert res == [(r, True) for r in range(world)]


@pytest.mark.parametrize("kernel", ["straight", "pipe", "multi"])
def test_peer_decode_ipc_two_processes(kernel):
    # two processes on cuda:0, each decoding its home stripes from its own and the other's
    # IPC-mapped storage; "pipe" / "multi" bulk-copy the mapped strips with TMA (opt-in path)
    if kernel == "pipe":     # one pattern for every stripe: a single PIPE program per rank
        _run_ipc(kernel, 1, erased_const=[2, 4, 5])
    else:
        _run_ipc(kernel, 1)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (real NVLink P2P)")
@pytest.mark.parametrize("kernel", ["straight", "pipe", "multi"])
def test_peer_decode_two_devices(kernel):
    # the cross-GPU decode over REAL peer memory: rank r on cuda:r, survivors read in place over
    # NVLink 5 / NVSwitch by the LDG kernel, and by the TMA-staged kernels (opt-in)
    _run_ipc(kernel, 2, erased_const=[2, 4, 5] if kernel == "pipe" else None)
