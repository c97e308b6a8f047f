"""Pins for oracle O5/O6 (set semantics, metrics, LRU cache) against the paper's worked examples."""
import os

import pytest

from oracle import slp

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(G, name + ".slp")) as f:
        return slp.parse(f.read())


a, b, c, d, e, f, g_ = (1 << i for i in range(7))


def test_sec2_example():
    p = load("sec2_P")
    assert slp.evaluate(p) == [b | c | d, a | c | d, a | b]
    assert slp.xor_count(p) == 4 and slp.nvar(p) == 3


def test_P0_P1_P2():
    vals = [slp.evaluate(load(x), strict=True) for x in ("P0", "P1", "P2")]
    assert vals[0] == vals[1] == vals[2]
    assert [slp.xor_count(load(x)) for x in ("P0", "P1", "P2")] == [8, 5, 4]
    assert vals[0] == [a | b, a | b | c, a | b | c | d, b | c | d]


def test_repair_and_xorrepair_traces():
    p0 = slp.evaluate(load("P0"))
    r = load("repair_P0_final")
    x = load("xorrepair_P0_final")
    assert slp.evaluate(r) == p0 and slp.xor_count(r) == 5
    assert slp.evaluate(x) == p0 and slp.xor_count(x) == 4


def test_rebuild_example_value():
    # Rebuild(v4) = {a, t3}: a ^ val(t3) = val(v4) = {b, c, d}
    t3 = a | b | c | d
    assert a ^ t3 == b | c | d


def test_intro_pipeline():
    vals = [slp.evaluate(load(x)) for x in ("intro_P", "intro_P_comp", "intro_P_sched")]
    assert vals[0] == vals[1] == vals[2]
    assert slp.xor_count(load("intro_P")) == 7
    assert slp.xor_count(load("intro_P_comp")) == 5


def test_fusion_memory_counts():
    assert slp.mem_count(load("fusion_chain")) == 9
    assert slp.mem_count(load("fusion_chain_fused")) == 5
    assert slp.evaluate(load("fusion_chain")) == slp.evaluate(load("fusion_chain_fused"))
    A, B, C = load("fusion_A"), load("fusion_B"), load("fusion_C")
    assert [slp.mem_count(x) for x in (A, B, C)] == [30, 12, 14]
    assert slp.evaluate(A) == slp.evaluate(B) == slp.evaluate(C)


def test_lru_Peg():
    p = load("P_eg")
    assert slp.ccap(p) == 10
    assert slp.iocost(p, 10) == 9
    assert slp.lru_trace(p, 10)[:2] == (7, 2)
    assert slp.iocost(p, 8) == 13
    assert slp.lru_trace(p, 9)[2] > 0                           # reload of A


def test_lru_Preg_Q_strategies():
    peg = slp.evaluate(load("P_eg"))
    preg = load("P_reg")
    assert slp.nvar(preg) == 4 and slp.iocost(preg, 8) == 12 and slp.ccap(preg) == 10
    for name, want in (("Q", (3, 5, 9)), ("Q_DFS", (4, 7, 10)), ("Q_greedy", (3, 7, 9))):
        q = load(name)
        assert (slp.nvar(q), slp.ccap(q), slp.iocost(q, 8)) == want, name
        assert sorted(slp.evaluate(q)) == sorted(peg)


def test_out_statements_and_errors():
    p = slp.parse("x = c0 ^ c1\nout 1 = x\nx = x ^ c2\nout 0 = x\nout 2 = c5\nout 3 = 0\n")
    assert slp.evaluate(p) == [a | b | c, a | b, 1 << 5, 0]
    with pytest.raises(ValueError):
        slp.evaluate("x = y ^ c0\nreturn x")
    with pytest.raises(ValueError):
        slp.evaluate("x = c0 ^ c0\nreturn x", strict=True)
    assert slp.evaluate("x = c0 ^ c0 ^ c1\nreturn x") == [b]   # cancellation
