"""Host-side product tests (no GPU): the C-ABI library loads and exports the header's
symbols; the C++ compiler matches the oracle's matrices and the paper's worked
examples; every compiled program (paper pebble form and interpreter slot form) is
semantically equal to its bitmatrix under the oracle's set evaluator."""
import itertools
import os
import re

import numpy as np
import pytest

import paper_2108_02692_b200 as X
from oracle import matrices as mx
from oracle import slp as oslp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def golden(name):
    with open(os.path.join(G, name + ".slp")) as f:
        return f.read()


def test_library_exports_every_header_symbol():
    with open(os.path.join(ROOT, "include", "xslp.h")) as f:
        hdr = f.read()
    names = set(re.findall(r"\b(xslp_[a-z_]+)\s*\(", hdr))
    assert len(names) >= 18
    for n in names:
        assert hasattr(X._lib, n), n
    assert set(X.EXPORTED) == names
    assert "sm_100a" in X.xslp_version()


@pytest.mark.parametrize("n,p,kind", [(10, 4, "isal"), (4, 2, "cauchy"), (10, 4, "sysvand"),
                                      (20, 4, "isal"), (8, 3, "isal")])
def test_matrices_match_oracle(n, p, kind):
    g = X.xslp_coding_matrix(n, p, kind)
    assert g.tolist() == mx.coding_matrix(n, p, kind)
    assert (X.xslp_encode_bitmatrix(g, n, p) == mx.to_bitmatrix(g[n:].tolist())).all()


def test_decode_bitmatrix_matches_oracle():
    g = X.xslp_coding_matrix(10, 4)
    og = mx.coding_matrix(10, 4)
    for er in [(2, 4, 5, 6), (0, 2, 3, 9), (10, 11, 12, 13), (3,), (1, 12), (13, 0, 7)]:
        bits, surv = X.xslp_decode_bitmatrix(g, 10, 4, er)
        osurv, rows = mx.decode_rows(og, 10, list(er))
        assert surv.tolist() == osurv
        assert (bits == mx.to_bitmatrix(rows)).all()


def test_decode_bitmatrix_errors():
    g = X.xslp_coding_matrix(10, 4)
    with pytest.raises(X.XslpError) as e:
        X.xslp_decode_bitmatrix(g, 10, 4, [0, 1, 2, 3, 4])
    assert e.value.code == X.XSLP_EUNRECOVERABLE
    with pytest.raises(X.XslpError) as e:
        X.xslp_decode_bitmatrix(g, 10, 4, [0, 0])
    assert e.value.code == X.XSLP_EINVAL
    with pytest.raises(X.XslpError) as e:
        X.xslp_decode_bitmatrix(g, 10, 4, [14])
    assert e.value.code == X.XSLP_EINVAL


def test_const_reuse_window_codegen():
    # xslp_opts.reuse only changes how often the TMA-staged code re-reads a constant from
    # shared memory: off (-1) reads at every use, a wider window reads less; out of range is
    # EINVAL.  (PTX is emitted and compiled for sm_100a in-process: no GPU needed.)
    g = X.xslp_coding_matrix(20, 4)
    bits = X.xslp_encode_bitmatrix(g, 20, 4)
    counts = {}
    for r in (-1, 16, 64):
        prog = X.xslp_compile(bits, kernel="pipe", threads=256, phases=2, block_bytes_hint=1 << 20,
                              reuse=r)
        counts[r] = prog.dump(2).count("ld.volatile.shared")
    assert counts[-1] > counts[16] > counts[64] > 0
    auto = X.xslp_compile(bits, kernel="pipe", threads=256, phases=2, block_bytes_hint=1 << 20)
    assert auto.dump(2).count("ld.volatile.shared") == counts[64]    # auto = 64 (single program)
    # the host's count of those reads (AUTO's shared-memory estimate) follows the same rule as
    # the emitter: one read per constant operand with the window off, each constant once when
    # every reuse distance is inside the window; PTX = the TMA, PIPE and single-stripe PIPE bodies
    g10 = X.xslp_coding_matrix(10, 4)
    for compress in ("none", "xorrepair"):
        uses = None
        for r in (-1, 16, 4096):
            prog = X.xslp_compile(X.xslp_encode_bitmatrix(g10, 10, 4), compress=compress, threads=256,
                                  block_bytes_hint=1 << 20, reuse=r)
            st = prog.stats()
            ptx = prog.dump(2)
            bodies = sum(ptx.count(f".entry {e}(") for e in ("xslp_sl_tma", "xslp_sl_pipe", "xslp_sl_pipe_one"))
            assert bodies == 3 and bodies * st["smem_reads"] == ptx.count("ld.volatile.shared")
            if r == -1:
                uses = st["smem_reads"]      # every constant operand of every instruction
                assert st["n_instr"] < uses <= st["mem_count"] - st["n_instr"]
        assert st["smem_reads"] == 80 < uses                      # window 4096: each constant once
    for bad in (-2, 4097):
        with pytest.raises(X.XslpError) as e:
            X.xslp_compile(bits, kernel="pipe", reuse=bad)
        assert e.value.code == X.XSLP_EINVAL


def test_singular_matrix():
    g = np.array([[1, 0], [0, 1], [1, 1], [2, 2]], dtype=np.uint8)  # rows 2 and 3 dependent
    with pytest.raises(X.XslpError) as e:
        X.xslp_decode_bitmatrix(g, 2, 2, [0, 1])
    assert e.value.code == X.XSLP_ESINGULAR


# ---- paper worked examples through the product compiler ---------------------------------

def _sets(bits):
    return oslp.rows_to_sets(bits)


def test_repair_P0_is_P1():
    p = X.xslp_compile_text(golden("P0"), 4, compress="repair", fuse=0, schedule=0, specialise=0)
    assert p.stats()["xor_count"] == 5
    text = p.dump()
    assert oslp.evaluate(text) == oslp.evaluate(golden("P0"))
    # exact pair sequence (a,b),(t1,c),(t2,d),(b,c),(t4,d)
    want = ["c0 ^ c1", "p0 ^ c2", "p1 ^ c3", "c1 ^ c2", "p3 ^ c3"]
    got = [l.split("=", 1)[1].strip() for l in text.splitlines() if "=" in l and not l.startswith("#")]
    assert got == want


def test_xorrepair_P0_is_P2():
    p = X.xslp_compile_text(golden("P0"), 4, compress="xorrepair", fuse=0, schedule=0, specialise=0)
    assert p.stats()["xor_count"] == 4
    text = p.dump()
    assert oslp.evaluate(text) == oslp.evaluate(golden("P0"))
    assert "p2 ^ c0" in text                                      # t4 <- a ^ t3


def test_intro_compression():
    p = X.xslp_compile_text(golden("intro_P"), 7, compress="xorrepair", fuse=1, schedule=1,
                            specialise=0)
    s = p.stats()
    assert s["xor_count"] == 5
    assert oslp.evaluate(p.dump()) == oslp.evaluate(golden("intro_P"))


def test_fusion_examples():
    p = X.xslp_compile_text(golden("fusion_chain"), 4, compress="none", fuse=1, schedule=0,
                            specialise=0)
    assert p.stats()["mem_count"] == 5 and p.stats()["n_instr"] == 1
    a = X.xslp_compile_text(golden("fusion_A"), 7, compress="none", fuse=1, schedule=0,
                            specialise=0)
    assert a.stats()["mem_count"] == 14                           # fuse(A) = C
    b = X.xslp_compile_text(golden("fusion_B"), 7, compress="none", fuse=1, schedule=0,
                            specialise=0)
    assert b.stats()["mem_count"] == 12 and b.stats()["n_instr"] == 3   # v1 used twice: kept
    unf = X.xslp_compile_text(golden("fusion_B"), 7, compress="none", fuse=0, schedule=0,
                              specialise=0)
    assert unf.stats()["mem_count"] == 12


def test_dfs_on_Peg():
    # DFS heuristic on G_eg: NVar 4, CCap 7, IOcost(., 8) = 10
    p = X.xslp_compile_text(golden("P_eg"), 7, compress="none", fuse=0, schedule=1, specialise=0)
    text = p.dump()
    assert p.stats()["nvar"] == 4
    assert oslp.ccap(text) == 7 and oslp.iocost(text, 8) == 10
    assert oslp.evaluate(text) == oslp.evaluate(golden("P_eg"))
    body = [l for l in text.splitlines() if "=" in l and not l.startswith("#")]
    # post-order C D v2 A B v1 E F v3 G v4 v5
    assert [l.split("=")[1].strip() for l in body] == [
        "c2 ^ c3", "c0 ^ c1", "p1 ^ c4 ^ c5", "p2 ^ c0 ^ c6", "p1 ^ p2 ^ p3"]
    assert body[-1].startswith("p3 =")                            # v5 takes v4's pebble


# ---- RS programs: semantics and the paper's tables ---------------------------------------

CFGS = [("enc", 10, 4, None), ("dec", 10, 4, (2, 4, 5, 6)), ("dec", 10, 4, (0, 2, 3, 9)),
        ("enc", 4, 2, None), ("dec", 4, 2, (0, 1)), ("enc", 10, 2, None), ("dec", 10, 4, (10, 11, 12, 13)),
        ("dec", 10, 4, (5,)), ("enc", 20, 4, None)]


def _bits(kind, n, p, er, family="isal"):
    fam = "cauchy" if (n, p) == (4, 2) else family
    g = X.xslp_coding_matrix(n, p, fam)
    if kind == "enc":
        return X.xslp_encode_bitmatrix(g, n, p)
    return X.xslp_decode_bitmatrix(g, n, p, er)[0]


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"{c[0]}{c[1]}_{c[2]}_{c[3]}")
@pytest.mark.parametrize("comp", ["none", "repair", "xorrepair"])
def test_semantic_equality(cfg, comp):
    if cfg[1] == 20 and comp != "xorrepair":
        pytest.skip("covered by xorrepair")
    bits = _bits(*cfg)
    want = _sets(bits)
    for fuse, sched in ((1, 1), (0, 0)):
        p = X.xslp_compile(bits, compress=comp, fuse=fuse, schedule=sched, specialise=0)
        assert oslp.evaluate(p.dump()) == want
        assert oslp.evaluate(p.dump(1)) == want                   # interpreter slot program
        s = p.stats()
        text = oslp.parse(p.dump())
        assert s["xor_count"] == oslp.xor_count(text)
        assert s["mem_count"] == oslp.mem_count(text)


def test_printed_counts_exact():
    # unoptimised P_enc / P_dec: #xor 755 / 1368
    for cfg, want in ((CFGS[0], 755), (CFGS[1], 1368)):
        p = X.xslp_compile(_bits(*cfg), compress="none", fuse=0, schedule=0, specialise=0)
        s = p.stats()
        assert s["xor_count"] == want and s["mem_count"] == 3 * want   # binary chain: #M = 3 #xor
        # fused-uncompressed P^{+F}: one instruction per goal, NVar 32
        pf = X.xslp_compile(_bits(*cfg), compress="none", fuse=1, schedule=0, specialise=0).stats()
        assert pf["nvar"] == 32 and pf["n_instr"] == 32 and pf["xor_count"] == want


def _within(got, want, tol):
    return abs(got - want) <= tol * want


def test_stage_tables_within_tolerance():
    # Co / Fu(Co) columns of P:1652-1654 and P:1681-1683; heuristic tie-breaks differ, +-5%
    for cfg, (x_co, ninst, mem) in ((CFGS[0], (385, 146, 677)), (CFGS[1], (511, 206, 923))):
        bits = _bits(*cfg)
        co = X.xslp_compile(bits, compress="xorrepair", fuse=0, schedule=0, specialise=0).stats()
        fu = X.xslp_compile(bits, compress="xorrepair", fuse=1, schedule=1, specialise=0).stats()
        assert _within(co["xor_count"], x_co, 0.05)
        assert co["mem_count"] == 3 * co["xor_count"]
        assert fu["xor_count"] == co["xor_count"]                # fusion keeps #xor (reading R7)
        assert _within(fu["n_instr"], ninst, 0.05)
        assert _within(fu["mem_count"], mem, 0.05)
        assert _within(fu["nvar"], {146: 88, 206: 125}[ninst], 0.10)


FIG1 = {(8, 4): (121, 170, 543, 747), (9, 4): (132, 182, 611, 829), (10, 4): (146, 206, 677, 923),
        (8, 3): (75, 129, 364, 561), (9, 3): (87, 144, 417, 641), (10, 3): (96, 145, 471, 661),
        (8, 2): (26, 65, 180, 286), (9, 2): (29, 73, 202, 322), (10, 2): (30, 77, 222, 352)}


@pytest.mark.parametrize("np_", list(FIG1))
def test_figure1_grid(np_):
    # Figure 1: instructions ("#xor" row, reading R7) and #M of the optimised
    # programs.  Encode: both within 5% (or 2 instructions for the 26-30-instruction p=2 codes).
    # Decode: the paper names its pattern only for RS(10,4) (P_dec = {2,4,5,6}), held
    # to 5% on both; for the other codes (reading R18) #M of {2,4,5,6}[:p] is held to 5% and
    # the printed instruction count must lie inside the range our compiler gives over ALL
    # C(n+p, p) erasure patterns (it varies 2-3x with the pattern: RS(8,2) 26-82)
    n, p = np_
    ie, id_, me, md = FIG1[np_]
    er = [2, 4, 5, 6][:p]
    se = X.xslp_compile(_bits("enc", n, p, None), specialise=0).stats()
    sd = X.xslp_compile(_bits("dec", n, p, er), specialise=0).stats()
    assert _within(se["mem_count"], me, 0.05) and _within(sd["mem_count"], md, 0.05)
    assert _within(se["n_instr"], ie, 0.05) or abs(se["n_instr"] - ie) <= 2
    if (n, p) == (10, 4):
        assert _within(sd["n_instr"], id_, 0.05)
    else:
        g = X.xslp_coding_matrix(n, p)
        pats = list(itertools.combinations(range(n + p), p))
        progs = X.compile_many([X.xslp_decode_bitmatrix(g, n, p, list(pt))[0] for pt in pats],
                               specialise=0)
        ins = [q.stats()["n_instr"] for q in progs]
        assert min(ins) <= id_ <= max(ins), (min(ins), id_, max(ins))


def test_copy_and_zero_goals():
    bits = np.zeros((16, 16), dtype=np.uint8)
    bits[0, 3] = 1                      # copy goal
    bits[2, [1, 2, 5]] = 1
    bits[3, [1, 2, 5, 7]] = 1
    bits[9, :] = 1                      # row 1 (zero) and others
    p = X.xslp_compile(bits, specialise=1)
    s = p.stats()
    assert s["n_copy_goals"] == 1 and s["n_zero_goals"] == 16 - 4
    assert oslp.evaluate(p.dump()) == _sets(bits)
    assert oslp.evaluate(p.dump(1)) == _sets(bits)
    assert "xslp_sl_batch" in p.dump(2)


def test_ptx_compiles_for_sm100a_without_gpu():
    for lanes in (1, 2, 4):
        p = X.xslp_compile(_bits(*CFGS[0]), lane_words=lanes, block_bytes_hint=1 << 20)
        s = p.stats()
        assert s["regs"] > 0 and s["spill_bytes"] == 0 or lanes > 1
        ptx = p.dump(2)
        assert ".target sm_100a" in ptx and "lop3.b32" in ptx
        assert f"+{7 * (1 << 17)}]" in ptx                         # baked strip offsets


def test_compile_errors():
    with pytest.raises(X.XslpError):
        X.xslp_compile(np.zeros((8, 0), dtype=np.uint8))
    with pytest.raises(X.XslpError):
        X.xslp_compile(np.full((8, 8), 2, dtype=np.uint8))
    with pytest.raises(X.XslpError):
        X.xslp_compile(np.ones((8, 8), dtype=np.uint8), lane_words=3)
    with pytest.raises(X.XslpError):
        X.xslp_compile_text("x = c0 ^ y\nreturn x", 4)


def test_device_call_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = X.xslp_compile(_bits(*CFGS[3]), specialise=0)
    with pytest.raises(X.XslpError) as e:
        X.xslp_encode_batch(p, 1 << 20, 1 << 21, 1, 4096, stream=0)
    assert e.value.code == X.XSLP_ECUDA


# ---- cache measures and the dataset averages ----------------

def test_lru_measures_match_oracle_and_paper():
    peg = X.xslp_compile_text(golden("P_eg"), 7, compress="none", fuse=0, schedule=0, specialise=0)
    assert (peg.ccap(), peg.iocost(10), peg.iocost(8)) == (10, 9, 13)
    dfs = X.xslp_compile_text(golden("P_eg"), 7, compress="none", fuse=0, schedule=1, specialise=0)
    assert (dfs.ccap(), dfs.iocost(8)) == (7, 10)
    for cfg in CFGS[:4]:
        for kw in (dict(compress="none", fuse=0, schedule=0), dict(compress="xorrepair", fuse=1, schedule=1),
                   dict(compress="xorrepair", fuse=0, schedule=0)):
            p = X.xslp_compile(_bits(*cfg), specialise=0, **kw)
            text = p.dump()
            assert p.ccap() == oslp.ccap(text)
            for c in (p.ccap(), max(40, p.ccap() // 2)):
                assert p.iocost(c) == oslp.iocost(text, c)


def test_dataset_averages_within_tolerance():
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "dataset_metrics.py")],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    got = {}
    for line in out.splitlines():
        parts = [x.strip() for x in line.split("|")]
        if len(parts) == 6 and parts[1] in ("xor", "mem", "nvar", "ccap"):
            got[(parts[1], parts[2])] = (float(parts[3]), float(parts[4]))
    assert len(got) == 14
    for k, (mine, paper) in got.items():
        if k[0] in ("xor", "mem"):
            assert abs(mine - paper) <= 2.0, (k, mine, paper)      # P:1478, P:1505 (points)
        elif k == ("ccap", "Co/P"):
            assert 0.75 <= mine / paper <= 1.35, (k, mine, paper)  # RePair temporal order differs
        else:
            assert 0.85 <= mine / paper <= 1.15, (k, mine, paper)


def test_greedy_on_Peg():
    # bottom-up greedy with capacity 8 on G_eg: exactly Q_greedy,
    # NVar 3, CCap 7, IOcost(., 8) = 9
    p = X.xslp_compile_text(golden("P_eg"), 7, compress="none", fuse=0, schedule=2,
                            greedy_capacity=8, specialise=0)
    text = p.dump()
    assert (p.stats()["nvar"], p.ccap(), p.iocost(8)) == (3, 7, 9)
    assert oslp.ccap(text) == 7 and oslp.iocost(text, 8) == 9
    body = [l.strip() for l in text.splitlines() if "=" in l and not l.startswith("#")]
    assert body == ["p0 = c0 ^ c1", "p1 = p0 ^ c4 ^ c5", "p2 = p1 ^ c0 ^ c6",
                    "p0 = p0 ^ p1 ^ p2", "p2 = c2 ^ c3"]
    assert oslp.evaluate(text) == oslp.evaluate(golden("Q_greedy"))


@pytest.mark.parametrize("cfg", CFGS[:4], ids=lambda c: f"{c[0]}{c[1]}_{c[2]}")
@pytest.mark.parametrize("cap", [16, 64, 512])
def test_greedy_semantics_rs(cfg, cap):
    bits = _bits(*cfg)
    p = X.xslp_compile(bits, schedule=2, greedy_capacity=cap, specialise=0)
    assert oslp.evaluate(p.dump()) == _sets(bits)
    assert oslp.evaluate(p.dump(1)) == _sets(bits)
    assert p.ccap() == oslp.ccap(p.dump())


def test_decode_bitmatrix_from_matches_oracle():
    import itertools
    rng = np.random.default_rng(3)
    for n, p, kind in [(4, 2, "cauchy"), (10, 4, "isal")]:
        g = X.xslp_coding_matrix(n, p, kind)
        og = mx.coding_matrix(n, p, kind)
        for _ in range(12):
            e = int(rng.integers(0, p + 1))
            er = sorted(rng.choice(n + p, e, replace=False).tolist())
            alive = [i for i in range(n + p) if i not in er]
            sv = rng.permutation(rng.choice(alive, n, replace=False)).tolist()
            bits = X.xslp_decode_bitmatrix_from(g, n, p, er, sv)
            want = mx.to_bitmatrix(mx.decode_rows_from(og, n, er, sv)) if e else np.zeros((0, 8 * n))
            assert bits.shape == (8 * e, 8 * n) and (bits == want).all()
        er = [0]
        with pytest.raises(X.XslpError):
            X.xslp_decode_bitmatrix_from(g, n, p, er, [0] + list(range(1, n)))   # erased survivor
        with pytest.raises(X.XslpError) as ei:                                   # > p erasures
            X.xslp_decode_bitmatrix_from(g, n, p, list(range(p + 1)), list(range(n)))
        assert ei.value.code == -3


def test_semantic_equality_all_1002_rs10_4_slps():
    # every optimised SLP of the paper's dataset (RS(10,4) encode + all 1001
    # 4-erasure decodes) computes exactly the oracle's goal sets, in both the
    # pebble form and the interpreter's slot form
    n, p = 10, 4
    g = X.xslp_coding_matrix(n, p)
    og = mx.coding_matrix(n, p)
    pats = list(itertools.combinations(range(n + p), p))
    bits = [X.xslp_encode_bitmatrix(g, n, p)] + [X.xslp_decode_bitmatrix(g, n, p, er)[0] for er in pats]
    progs = X.compile_many(bits, specialise=0)
    wants = [oslp.rows_to_sets(mx.to_bitmatrix(og[n:]))]
    wants += [oslp.rows_to_sets(mx.to_bitmatrix(mx.decode_rows(og, n, list(er))[1])) for er in pats]
    assert len(progs) == 1002
    for k, (prog, want) in enumerate(zip(progs, wants)):
        assert oslp.evaluate(prog.dump()) == want, k
        assert oslp.evaluate(prog.dump(1)) == want, k


def _emulate_microops(words, strips, n_goals):
    """Plain host emulation of the pipelined interpreter's paired micro-op code (interp.cu
    emit_variant), in the kernel's order: the operands of pair q+1 are loaded before pair q
    computes and stores, and both mops of a pair load before either stores -- so a schedule that
    reads a variable too early reads stale data here.  Shared memory is a map from row byte
    offset to the row; variable rows start as garbage, row 0 of them is the zero row."""
    w = np.array(words, dtype=np.int64)
    nl, npairs, total, nvrows, rb, var0, const0, start = (int(x) for x in w[:8])
    assert total == len(w) and start == 8 and npairs % 3 == 0
    width = strips.shape[1]
    rng = np.random.default_rng(0)
    smem = {var0 + r * rb: rng.integers(0, 2**32, width, dtype=np.uint32) for r in range(8, nvrows)}
    for r in range(8):                                   # the zero rows, one per bank group
        smem[var0 + r * rb] = np.zeros(width, dtype=np.uint32)
    loads = w[start + 12 * (npairs + 2):start + 12 * (npairs + 2) + 2 * nl]
    for i in range(nl):
        assert const0 <= loads[2 * i + 1] < const0 + nl * rb
        smem[int(loads[2 * i + 1])] = strips[loads[2 * i]].copy()

    def pair(q):
        c = w[start + 12 * q:start + 12 * q + 12]
        return [(c[0:4], int(c[8]), int(c[9])), (c[4:8], int(c[10]), int(c[11]))]

    def load(q):
        vals = []
        for ops, _, ctl in pair(q):
            hi = (ctl >> 27) & 1
            vals.append([smem[int(ops[u])].copy() if u < 2 or hi else None for u in range(4)])
        return vals

    out = np.full((n_goals, width), 0xDEADBEEF, dtype=np.uint32)
    acc = np.zeros(width, dtype=np.uint32)
    cur = load(0)
    for q in range(npairs):
        nxt = load(q + 1)                                     # before pair q stores (slack ok)
        for (ops, dst, ctl), v in zip(pair(q), cur):
            flags = (ctl >> 24) & 0xF
            if flags & 1:
                acc = np.zeros_like(acc)
            acc = acc ^ v[0] ^ v[1]
            if flags & 8:
                acc = acc ^ v[2] ^ v[3]
            if flags & 2:
                assert var0 < dst < var0 + nvrows * rb        # a variable row, never 0 or a constant
                smem[dst] = acc.copy()
            if flags & 4:
                g = ((ctl & 0xFFFF) - 16) // 8 * 8 + ((ctl >> 16) & 7)
                out[g] = acc
        cur = nxt
    assert not smem[var0].any()
    return out


@pytest.mark.parametrize("n,p,comp,er,T,L,sched", [
    (10, 3, "none", None, 128, 1, 1), (10, 4, "xorrepair", None, 256, 1, 1),
    (10, 2, "repair", None, 64, 2, 1), (4, 2, "none", None, 32, 4, 1),
    (10, 4, "xorrepair", (2, 4, 5, 6), 128, 2, 1),
    (20, 4, "xorrepair", (0, 5, 21, 23), 96, 1, 1),
    (10, 4, "xorrepair", None, 128, 2, 2), (10, 4, "xorrepair", (2, 4, 5, 6), 64, 4, 2),
    (20, 4, "xorrepair", (0, 5, 21, 23), 128, 1, 2), (10, 4, "none", (0, 1, 12, 13), 128, 1, 0)])
def test_interpreter_microops_compute_the_oracle_result(n, p, comp, er, T, L, sched):
    # the host's paired micro-op code for the pipelined interpreter (dump form 3), run by a
    # plain emulator with the kernel's pair semantics, reproduces the oracle's RS bytes on the
    # strip layout -- for DFS (1), capacity-bounded greedy (2) and unscheduled (0) programs
    import synth
    from oracle import rs
    kind = "cauchy" if (n, p) == (4, 2) else "isal"
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    if er is None:
        bits, rows = X.xslp_encode_bitmatrix(g, n, p), og[n:]
    else:
        bits, rows = X.xslp_decode_bitmatrix(g, n, p, er)[0], mx.decode_rows(og, n, list(er))[1]
    prog = X.xslp_compile(bits, compress=comp, specialise=0, threads=T, lane_words=L,
                          schedule=sched, greedy_capacity=32)
    words = [int(x) for x in prog.dump(3).split()]
    B = 128
    data = synth.stripe_data(9, 1, n, B)
    got = _emulate_microops(words, data.reshape(8 * n, B // 8).view(np.uint32), bits.shape[0])
    want = rs.apply_rows(rows, data).reshape(bits.shape[0], B // 8).view(np.uint32)
    assert (got == want).all()


def test_no_goal_program():
    # RS(n, 0): no parity blocks -- the program has no goals and no work
    g = X.xslp_coding_matrix(4, 0)
    bits = X.xslp_encode_bitmatrix(g, 4, 0)
    assert bits.shape == (0, 32)
    prog = X.xslp_compile(bits, specialise=0)
    assert prog.stats()["n_goals"] == 0 and prog.stats()["xor_count"] == 0
    assert oslp.evaluate(prog.dump()) == []


@pytest.mark.parametrize("n,p,kind", [(4, 2, "cauchy"), (10, 4, "isal"), (20, 4, "isal"), (8, 3, "sysvand")])
def test_syndrome_decode_math_matches_the_codeword(n, p, kind):
    # syndrome-form decode (csrc/syndrome.cpp): zero the erased blocks of an oracle codeword,
    # apply the syndrome bitmatrix then the solve bitmatrix (plain GF(2) applies, oracle side):
    # the erased blocks come back, for every erasure count 1..p and sampled patterns
    from oracle import rs
    import synth
    g = X.xslp_coding_matrix(n, p, kind)
    og = mx.coding_matrix(n, p, kind)
    B = 64
    data = synth.stripe_data(17, 0, n, B)
    cw = np.concatenate([data, rs.encode(og, n, data)])
    rng = np.random.default_rng(n * 31 + p)
    for e in range(1, p + 1):
        pats = list(itertools.combinations(range(n + p), e))
        for er in [pats[i] for i in rng.choice(len(pats), min(40, len(pats)), replace=False)]:
            syn, sol = X.xslp_syndrome_bitmatrices(g, n, p, er)
            z = cw.copy()
            z[list(er)] = 0
            s = rs.bitmatrix_apply(syn, z)                 # 8p strips of syndrome
            assert s.shape == (p, B)
            got = rs.bitmatrix_apply(sol, s)
            assert (got == cw[list(er)]).all(), er
    with pytest.raises(X.XslpError):
        X.xslp_syndrome_bitmatrices(g, n, p, list(range(p + 1)))


def test_syndrome_of_a_codeword_is_zero():
    from oracle import rs
    import synth
    n, p = 10, 4
    g = X.xslp_coding_matrix(n, p)
    og = mx.coding_matrix(n, p)
    data = synth.stripe_data(18, 0, n, 128)
    cw = np.concatenate([data, rs.encode(og, n, data)])
    syn, _ = X.xslp_syndrome_bitmatrices(g, n, p, [0])
    assert not rs.bitmatrix_apply(syn, cw).any()


def _emulate_lanes(words, strips, n_goals, loads_first=True):
    """Host emulation of the lane-parallel interpreter's code (interp_lanes.cu emit_variant, dump
    form 4): rounds of 32 lane-ops over the same words; a lane-op XORs its operand rows (slots
    0-1 loaded when it has operands, 2-3 when it has more than two; unused slots name one of
    the zero rows 0-7) and stores to a variable row and/or a goal.  loads_first=False runs each
    lane to completion in lane order instead -- the schedule must be right for any interleaving
    within a round."""
    w = np.array(words, dtype=np.int64)
    nl, nr, total, nvrows, rb, var0, const0, start = (int(x) for x in w[:8])
    assert total == len(w) and start == 8
    width = strips.shape[1]
    rng = np.random.default_rng(1)
    smem = {var0 + r * rb: rng.integers(0, 2**32, width, dtype=np.uint32) for r in range(8, nvrows)}
    for r in range(8):                                   # the zero rows, one per bank group
        smem[var0 + r * rb] = np.zeros(width, dtype=np.uint32)
    loads = w[start + 256 * (nr + 1):start + 256 * (nr + 1) + 2 * nl]
    for i in range(nl):
        smem[int(loads[2 * i + 1])] = strips[loads[2 * i]].copy()
    out = np.full((n_goals, width), 0xDEADBEEF, dtype=np.uint32)
    for r in range(nr):
        ops = [np.concatenate([w[start + 256 * r + 4 * l:start + 256 * r + 4 * l + 4],
                               w[start + 256 * r + 128 + 4 * l:start + 256 * r + 128 + 4 * l + 4]])
               for l in range(32)]

        def value(o):
            cnt = int(o[6]) & 0xFF
            acc = np.zeros(width, dtype=np.uint32)
            if cnt > 0:
                acc = acc ^ smem[int(o[0])] ^ smem[int(o[1])]
            if cnt > 2:
                acc = acc ^ smem[int(o[2])] ^ smem[int(o[3])]
            return acc

        def store(o, acc):
            fl = int(o[6]) >> 8
            if fl & 1:
                assert var0 + 8 * rb <= o[4] < var0 + nvrows * rb  # a variable row, never zero/constant
                smem[int(o[4])] = acc.copy()
            if fl & 2:
                out[((int(o[5]) & 0xFFFF) - 16) // 8 * 8 + (int(o[5]) >> 16)] = acc

        if loads_first:
            vals = [value(o) for o in ops]
            for o, v in zip(ops, vals):
                store(o, v)
        else:
            for o in ops:
                store(o, value(o))
    assert not smem[var0].any()
    return out


def _emulate_tmem(words, strips, n_goals):
    """Run the TMEM interpreter's code (dump form 5, interp_tmem.cu emit_code) on every position
    at once: TMEM slot 0 reads zero, slot 1 is the write sink, constant row r is slot 2 + r; a
    batch reads all its operands before any of its stores, reads operands 3-4 only when
    flagged, and never reads a slot stored since the last wait::st flag (the kernel's tcgen05.st
    may still be in flight)."""
    nconst, nb, nslots, kb, w_ = words[0], words[1], words[3], words[4], words[5]
    assert w_ == 1 and kb in (4, 8, 12, 16)
    ops = words[8:8 + 4 * kb * (nb + 1)]
    loads = words[8 + 4 * kb * (nb + 1):8 + 4 * kb * (nb + 1) + nconst]
    zero = np.zeros_like(strips[0])
    slots = {0: zero}
    for r, c in enumerate(loads):
        slots[2 + r] = strips[c]
    pending = set()
    out = np.zeros((n_goals, strips.shape[1]), dtype=np.uint32)
    done = np.zeros(n_goals, dtype=bool)
    for b in range(nb + 1):
        batch = [ops[4 * (b * kb + j):4 * (b * kb + j) + 4] for j in range(kb)]
        fl = batch[0][3]
        assert all(op[3] == 0 for op in batch[1:])
        if fl & 1:
            pending.clear()
        res = []
        for w0, w1, w2, _ in batch:
            cols = [w0 & 0xFFFF, w0 >> 16, w1 & 0xFFFF, w1 >> 16]
            if not fl & 2:
                assert cols[2] == cols[3] == 0
            acc = zero.copy()
            for t in cols:
                assert t < nslots and t != 1 and t in slots and t not in pending, (b, t)
                acc ^= slots[t]
            res.append((acc, w2))
        for acc, w2 in res:
            d, g = w2 & 0xFFFF, w2 >> 16
            # a constant's slot may take a variable after the constant's last reader (a wrong
            # reuse shows up as a wrong goal below)
            assert d >= 1 and d < nslots
            slots[d] = acc
            pending.add(d)
            if g:
                assert b < nb and not done[g - 1]
                out[g - 1], done[g - 1] = acc, True
    assert done.all()
    return out


def _emulate_tmem_device(words, strips, n_goals):
    """Run the TMEM kernel's device code (dump form 6, interp_tmem.cu emit_device, W = 1) the
    way each of the four consumer warps reads its own variant: every TMEM address must carry
    the warp's lane quarter; the result must be the same for every variant."""
    nconst, nb, kb, vw = words[0], words[1], words[4], words[6]
    loads = words[8 + 4 * vw:8 + 4 * vw + nconst]
    results = []
    for q in range(4):
        v = words[8 + q * vw:8 + (q + 1) * vw]
        zero = np.zeros_like(strips[0])
        tm = {0: zero}
        for r, c in enumerate(loads):
            tm[2 + r] = strips[c]
        out = np.zeros((n_goals, strips.shape[1]), dtype=np.uint32)
        p = 0
        fl_next = words[7]  # the kernel reads each batch's flags with the previous batch's header

        def col(a):
            assert a >> 16 == q * 32, (q, hex(a))
            return a & 0xFFFF
        for _ in range(nb):
            fl = v[p]
            assert fl == fl_next
            fl_next = v[p + 1]
            p += 4
            nops = 4 if fl & 2 else 2
            res = []
            for j in range(kb):  # kb operand groups, then kb dst addresses, then kb goal words
                acc = zero.copy()
                for a in v[p + nops * j:p + nops * (j + 1)]:
                    acc ^= tm[col(a)]
                res.append((acc, col(v[p + nops * kb + j]), v[p + (nops + 1) * kb + j]))
            p += (nops + 2) * kb
            for acc, d, g in res:
                tm[d] = acc
                if g:
                    assert fl & 4
                    out[g - 1] = acc
        assert p == vw and fl_next == 0
        results.append(out)
    assert all((r == results[0]).all() for r in results)
    return results[0]


def test_tmem_interpreter_copy_and_zero_goals():
    # degenerate goals through the TMEM interpreter's schedule and device code: identity rows
    # (copies of a strip), zero rows, a full row, random rows
    import synth
    from oracle import rs
    rng = np.random.default_rng(1)
    bits = np.zeros((16, 24), dtype=np.uint8)
    bits[0, 3] = 1
    bits[1, 17] = 1
    bits[2, [1, 2, 5]] = 1
    bits[5, :] = 1
    bits[9:, :] = rng.integers(0, 2, size=(7, 24))
    B = 128
    data = synth.stripe_data(9, 0, 3, B)
    strips = data.reshape(24, B // 8).view(np.uint32)
    want = rs.bitmatrix_apply(bits, data).reshape(16, B // 8).view(np.uint32)
    prog = X.xslp_compile(bits, kernel="interp", specialise=0)
    assert (_emulate_tmem([int(x) for x in prog.dump(5).split()], strips, 16) == want).all()
    assert (_emulate_tmem_device([int(x) for x in prog.dump(6).split()], strips, 16) == want).all()


@pytest.mark.parametrize("n,p,comp,er,sched", [
    (10, 4, "xorrepair", None, 1), (10, 4, "xorrepair", (2, 4, 5, 6), 1), (4, 2, "none", None, 1),
    (20, 4, "xorrepair", (0, 5, 21, 23), 1), (10, 3, "repair", None, 2), (10, 4, "none", (0, 1, 12, 13), 0),
    (10, 4, "xorrepair", (2, 4, 5, 6), 2)])
def test_tmem_interpreter_code_computes_the_oracle_result(n, p, comp, er, sched):
    # the TMEM interpreter's batches (dump form 5) reproduce the oracle's RS bytes, never read
    # a slot before its store is waited for, and fit the 512 TMEM columns at 1 word per thread
    import synth
    from oracle import rs
    kind = "cauchy" if (n, p) == (4, 2) else "isal"
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    if er is None:
        bits, rows = X.xslp_encode_bitmatrix(g, n, p), og[n:]
    else:
        bits, rows = X.xslp_decode_bitmatrix(g, n, p, er)[0], mx.decode_rows(og, n, list(er))[1]
    prog = X.xslp_compile(bits, compress=comp, specialise=0, schedule=sched, greedy_capacity=32)
    words = [int(x) for x in prog.dump(5).split()]
    assert words[2] == len(words) and words[3] <= 512
    B = 128
    data = synth.stripe_data(9, 2, n, B)
    strips = data.reshape(8 * n, B // 8).view(np.uint32)
    want = rs.apply_rows(rows, data).reshape(bits.shape[0], B // 8).view(np.uint32)
    assert (_emulate_tmem(words, strips, bits.shape[0]) == want).all()
    dev = [int(x) for x in prog.dump(6).split()]
    assert dev[2] == len(dev)
    assert (_emulate_tmem_device(dev, strips, bits.shape[0]) == want).all()


def _emulate_tmem_streams(words, strips, n_goals, first):
    """Run the two-stream TMEM code (dump form 7, interp_tmem.cu emit_streams, W = 1, lane
    quarter 0): the two streams (goal halves, one consumer warp each) meet only after the
    constant copies and at the tile's end, so one runs to completion before the other (both
    orders).  Checks that no stream writes a constant slot or a slot the other stream uses."""
    nconst, nslots, kb = words[0], words[3], words[4]
    nbs, vws, offs = (words[1], words[8]), (words[6], words[9]), (0, words[11])
    loads = words[16 + 4 * (vws[0] + vws[1]):16 + 4 * (vws[0] + vws[1]) + nconst]
    tm = {0: np.zeros_like(strips[0])}
    for r, c in enumerate(loads):
        tm[2 + r] = strips[c]
    out = np.zeros((n_goals, strips.shape[1]), dtype=np.uint32)
    used = [set(), set()]
    for h in (first, 1 - first):
        v = words[16 + offs[h]:16 + offs[h] + vws[h]]
        p = 0
        for _ in range(nbs[h]):
            fl = v[p]
            p += 4
            na = 4 if fl & 2 else 2
            res = []
            for j in range(kb):
                acc = np.zeros_like(strips[0])
                for a in v[p + na * j:p + na * (j + 1)]:
                    acc ^= tm[a & 0xFFFF]
                    if a & 0xFFFF >= 2 + nconst:
                        used[h].add(a & 0xFFFF)
                res.append((acc, v[p + na * kb + j] & 0xFFFF, v[p + (na + 1) * kb + j]))
            p += (na + 2) * kb
            for acc, d, g in res:
                assert d == 1 or 2 + nconst <= d < nslots
                if d != 1:
                    used[h].add(d)
                    tm[d] = acc
                if g:
                    assert fl & 4
                    out[g - 1] = acc
        assert p == vws[h]
    assert not used[0] & used[1]
    return out


@pytest.mark.parametrize("n,p,er", [(10, 4, None), (10, 4, (2, 4, 5, 6)), (10, 4, (0, 1, 9, 12)),
                                    (20, 4, (3, 10, 19, 20)), (4, 2, None), (10, 3, (0, 11, 12))])
def test_tmem_two_streams_compute_the_oracle_result(n, p, er):
    # the program's goal halves, compiled apart and run by two unsynchronised warps per lane
    # quarter, reproduce the oracle's bytes in either completion order
    import synth
    from oracle import rs
    og = mx.coding_matrix(n, p)
    g = X.xslp_coding_matrix(n, p)
    if er is None:
        bits, rows = X.xslp_encode_bitmatrix(g, n, p), og[n:]
    else:
        bits, rows = X.xslp_decode_bitmatrix(g, n, p, er)[0], mx.decode_rows(og, n, list(er))[1]
    prog = X.xslp_compile(bits, kernel="interp", specialise=0)
    words = [int(x) for x in prog.dump(7).split()]
    assert words[2] == len(words)
    data = synth.stripe_data(9, 5, n, 128)
    strips = data.reshape(8 * n, 16).view(np.uint32)
    want = rs.apply_rows(rows, data).reshape(bits.shape[0], 16).view(np.uint32)
    for first in (0, 1):
        assert (_emulate_tmem_streams(words, strips, bits.shape[0], first) == want).all()


def test_tmem_schedule_fits_two_words_for_every_rs_10_4_program():
    # the TMEM interpreter runs 2 words per thread only when a launch's programs all fit 256 slots
    # (512 columns); the critical-path batch scheduler (window 400, 16 ops per batch) must keep
    # every RS(10,4) program there -- the encode and all 1001 four-erasure decode programs -- and
    # keep the encode at 14 batches (216 ops: ceil(216/16) = 14, the packing bound)
    g = X.xslp_coding_matrix(10, 4)
    enc = X.xslp_compile(X.xslp_encode_bitmatrix(g, 10, 4), kernel="interp", specialise=0)
    w = [int(x) for x in enc.dump(6).split()]
    assert w[4] == 16 and w[1] == 14 and w[3] <= 256
    pats = list(itertools.combinations(range(14), 4))
    progs = X.compile_many([X.xslp_decode_bitmatrix(g, 10, 4, list(p))[0] for p in pats],
                           kernel="interp", specialise=0)
    slots = [int(pr.dump(6).split()[3]) for pr in progs]
    assert max(slots) <= 256, (max(slots), pats[slots.index(max(slots))])


@pytest.mark.parametrize("n,p,comp,er,sched", [
    (10, 4, "xorrepair", None, 1), (10, 4, "xorrepair", (2, 4, 5, 6), 1), (4, 2, "none", None, 1),
    (20, 4, "xorrepair", (0, 5, 21, 23), 1), (10, 3, "repair", None, 2), (10, 4, "none", (0, 1, 12, 13), 0)])
def test_lane_interpreter_code_computes_the_oracle_result(n, p, comp, er, sched):
    # the lane-parallel interpreter's rounds (dump form 4), emulated with every lane of a round
    # loading first and with lanes run one after another, reproduce the oracle's RS bytes
    import synth
    from oracle import rs
    kind = "cauchy" if (n, p) == (4, 2) else "isal"
    og = mx.coding_matrix(n, p, kind)
    g = X.xslp_coding_matrix(n, p, kind)
    if er is None:
        bits, rows = X.xslp_encode_bitmatrix(g, n, p), og[n:]
    else:
        bits, rows = X.xslp_decode_bitmatrix(g, n, p, er)[0], mx.decode_rows(og, n, list(er))[1]
    prog = X.xslp_compile(bits, compress=comp, specialise=0, schedule=sched, greedy_capacity=32)
    words = [int(x) for x in prog.dump(4).split()]
    B = 128
    data = synth.stripe_data(9, 2, n, B)
    strips = data.reshape(8 * n, B // 8).view(np.uint32)
    want = rs.apply_rows(rows, data).reshape(bits.shape[0], B // 8).view(np.uint32)
    for lf in (True, False):
        assert (_emulate_lanes(words, strips, bits.shape[0], loads_first=lf) == want).all()
