#!/usr/bin/env python
"""Compiler fidelity probe (host only); output recorded in profiles/r02/compiler_fidelity.md."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import itertools, sys
import numpy as np
import paper_2108_02692_b200 as X
FIG1 = {(8, 4): (121, 170, 543, 747), (9, 4): (132, 182, 611, 829), (10, 4): (146, 206, 677, 923),
        (8, 3): (75, 129, 364, 561), (9, 3): (87, 144, 417, 641), (10, 3): (96, 145, 471, 661),
        (8, 2): (26, 65, 180, 286), (9, 2): (29, 73, 202, 322), (10, 2): (30, 77, 222, 352)}
for (n, p), (ie, idd, me, md) in FIG1.items():
    g = X.xslp_coding_matrix(n, p)
    se = X.xslp_compile(X.xslp_encode_bitmatrix(g, n, p), specialise=0).stats()
    er = [2, 4, 5, 6][:p]
    sd = X.xslp_compile(X.xslp_decode_bitmatrix(g, n, p, er)[0], specialise=0).stats()
    # naive XOR count of the pattern (to identify "most XORs")
    best = None
    for pat in itertools.combinations(range(n + p), p):
        b = X.xslp_decode_bitmatrix(g, n, p, list(pat))[0]
        nx = int(b.sum()) - b.shape[0]
        if best is None or nx > best[0]: best = (nx, pat)
    bd = X.xslp_decode_bitmatrix(g, n, p, list(best[1]))[0]
    sw = X.xslp_compile(bd, specialise=0).stats()
    print(f"RS({n},{p}) enc instr {se['n_instr']} vs {ie} ({se['n_instr']/ie-1:+.1%}) #M {se['mem_count']} vs {me} ({se['mem_count']/me-1:+.1%}) | dec{er} instr {sd['n_instr']} vs {idd} ({sd['n_instr']/idd-1:+.1%}) #M {sd['mem_count']} vs {md} ({sd['mem_count']/md-1:+.1%}) | worst {best[1]} naive {best[0]} instr {sw['n_instr']} #M {sw['mem_count']}")
