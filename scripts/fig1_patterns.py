#!/usr/bin/env python
"""Compiler fidelity probe (host only); output recorded in profiles/r02/compiler_fidelity.md."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import itertools
import numpy as np
import paper_2108_02692_b200 as X
FIG1D = {(8, 4): (170, 747), (9, 4): (182, 829), (8, 3): (129, 561), (9, 3): (144, 641), (10, 3): (145, 661), (8, 2): (65, 286), (9, 2): (73, 322), (10, 2): (77, 352)}
for (n, p), (idd, md) in FIG1D.items():
    g = X.xslp_coding_matrix(n, p)
    pats = list(itertools.combinations(range(n + p), p))
    bits = [X.xslp_decode_bitmatrix(g, n, p, list(pt))[0] for pt in pats]
    st = [pr.stats() for pr in X.compile_many(bits, specialise=0)]
    ins = np.array([s['n_instr'] for s in st]); mem = np.array([s['mem_count'] for s in st])
    # patterns matching both numbers exactly / within 2%
    exact = [pats[i] for i in range(len(pats)) if ins[i] == idd and mem[i] == md]
    near = [pats[i] for i in range(len(pats)) if abs(ins[i] - idd) <= 0.02 * idd and abs(mem[i] - md) <= 0.02 * md]
    print(f"RS({n},{p}) paper {idd}/{md}: instr range {ins.min()}-{ins.max()} mean {ins.mean():.1f}; #M range {mem.min()}-{mem.max()}; exact {exact[:4]} ({len(exact)}) near2% {len(near)} of {len(pats)}")
