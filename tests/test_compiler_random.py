"""Randomised host-compiler checks (no GPU): arbitrary GF(2) bitmatrices, every pass
combination, against the oracle's set semantics (oracle/slp.py).  The compiler's passes
(RePair / XorRePair, fusion, DFS / greedy scheduling, goal splitting for consumer groups) must
preserve what every goal computes for any input, not only for RS matrices."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2108_02692_b200 as X
from oracle import slp as oslp


@st.composite
def bitmatrices(draw):
    rows = 8 * draw(st.integers(1, 4))
    cols = 8 * draw(st.integers(1, 6))
    density = draw(st.sampled_from([0.05, 0.3, 0.5, 0.8]))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    bits = (rng.random((rows, cols)) < density).astype(np.uint8)
    if draw(st.booleans()):                     # duplicate rows and an all-zero row
        bits[rows // 2] = bits[0]
        bits[-1] = 0
    return bits


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(bits=bitmatrices(), comp=st.sampled_from(["none", "repair", "xorrepair"]),
       fuse=st.integers(0, 1), sched=st.sampled_from([0, 1, 2]))
def test_random_bitmatrix_semantics(bits, comp, fuse, sched):
    want = oslp.rows_to_sets(bits)
    kw = dict(compress=comp, fuse=fuse, schedule=sched, specialise=0)
    if sched == 2:
        kw["greedy_capacity"] = 16
    p = X.xslp_compile(bits, **kw)
    assert oslp.evaluate(p.dump()) == want
    assert oslp.evaluate(p.dump(1)) == want
    s = p.stats()
    text = oslp.parse(p.dump())
    assert s["xor_count"] == oslp.xor_count(text)
    assert s["mem_count"] == oslp.mem_count(text)
    # XOR count never grows past the lifted program's (sum of popcount - 1 over non-empty rows)
    naive = int(sum(max(0, int(r.sum()) - 1) for r in bits))
    assert s["xor_count"] <= naive


@settings(max_examples=25, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(bits=bitmatrices(), groups=st.integers(2, 4))
def test_random_bitmatrix_ptx_with_consumer_groups(bits, groups):
    # the device code generator (all entries, PIPE split into goal groups) assembles for
    # sm_100a for any program; the groups' summed XOR work covers the joint program
    p = X.xslp_compile(bits, kernel="pipe", threads=64, stages=2, groups=groups)
    s = p.stats()
    assert s["group_xor"] >= s["xor_count"]
    assert ".target sm_100a" in p.dump(2)
