#!/usr/bin/env python
"""Compiler fidelity probe (host only); output recorded in profiles/r02/compiler_fidelity.md."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_02692_b200 as X
G = X.xslp_coding_matrix(10, 4)
enc = X.xslp_encode_bitmatrix(G, 10, 4)
dec = X.xslp_decode_bitmatrix(G, 10, 4, [2,4,5,6])[0]
n = 10
orders = {
 "block-major (ours)": list(range(80)),
 "bit-major": [k * n + j for j in range(n) for k in range(8)],    # new position of column 8j+k
 "string c<idx>": None,
 "reversed": list(range(79, -1, -1)),
 "block-major MSB-first": [8 * j + (7 - k) for j in range(n) for k in range(8)],
 "string c<j>_<k>": None,
}
names = [f"c{i}" for i in range(80)]
srt = sorted(range(80), key=lambda i: names[i])
orders["string c<idx>"] = [srt.index(i) for i in range(80)]
names2 = [f"c{j}_{k}" for j in range(n) for k in range(8)]
srt2 = sorted(range(80), key=lambda i: names2[i])
orders["string c<j>_<k>"] = [srt2.index(i) for i in range(80)]
for nm, pos in orders.items():
    res = []
    for b in (enc, dec):
        nb = np.zeros_like(b)
        nb[:, pos] = b            # column i moves to position pos[i]
        for comp in ("xorrepair",):
            co = X.xslp_compile(nb, compress=comp, fuse=0, schedule=0, specialise=0).stats()
            fu = X.xslp_compile(nb, specialise=0).stats()
            res.append((co['xor_count'], fu['n_instr'], fu['mem_count'], fu['nvar']))
    print(f"{nm:26s} enc {res[0]}  dec {res[1]}   (paper enc (385,146,677,88) dec (511,206,923,125))")
