"""Independent CPU oracle for the XOR-SLP erasure-coding hot path (arXiv 2108.02692).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything
under ``oracle/``.  The product path (``paper_2108_02692_b200``) never imports
it, and the oracle never imports the product: the two share no code, tables or
constants.  The only module both sides use is ``synth`` (seeded input
generators, no coding arithmetic).

Citations: ``P:n`` = line n of the paper text with its section tag;
the section map is in DESIGN.md.

Modules
  gf256     O1  GF(2^8) with the polynomial x^8+x^4+x^3+x^2+1 ([Eval])
  matrices  O2  coding matrices, Gauss-Jordan inverse, decode rows, x~ bitmatrix
  rs        O3/O4  Reed-Solomon encode/decode of the strip layout (bit-transposed
                view, table-driven byte RS) and the plain GF(2) bitmatrix apply
  slp       O5/O6  set semantics of SLP_xor / MultiSLP, #xor, #M, NVar, the
                abstract LRU cache (CCap, IOcost)

Parity pins: every function is pinned in tests/test_oracle_*.py against values
the paper prints, closed forms, and brute force.  No function is "parity
unpinned".
"""
