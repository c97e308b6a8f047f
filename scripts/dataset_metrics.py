#!/usr/bin/env python
"""Average reduction ratios over the paper's RS(10,4) dataset ([Eval]):
one encoding SLP + the 1001 decoding SLPs of every 4-erasure pattern, through the
product compiler (host only).  Reproduces the tables of P:1470-1523:

  #xor      RePair(P)/P 42.1%   XorRePair(P)/P 40.8%
  #M        Co/P 40.8%  Fu/P 35.1%  Fu(Co)/Co 59.2%  Fu(Co)/P 24.1%
  NVar      Co/P 1552%  Fu/P 100%   Fu(Co)/Co 38.9%  Dfs(Fu(Co))/Co 24.5%
  CCap      Co/P 498%   Fu/P 98.7%  Fu(Co)/Co 51.2%  Dfs(Fu(Co))/Co 40.0%

    python scripts/dataset_metrics.py [--limit K] > profiles/r01_dataset_metrics.md
"""
import argparse
import itertools
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02692_b200 as X  # noqa: E402

PAPER = {
    ("xor", "repair/P"): 42.1, ("xor", "xorrepair/P"): 40.8,
    ("mem", "Co/P"): 40.8, ("mem", "Fu/P"): 35.1, ("mem", "FuCo/Co"): 59.2, ("mem", "FuCo/P"): 24.1,
    ("nvar", "Co/P"): 1552, ("nvar", "Fu/P"): 100, ("nvar", "FuCo/Co"): 38.9, ("nvar", "DfsFuCo/Co"): 24.5,
    ("ccap", "Co/P"): 498, ("ccap", "Fu/P"): 98.7, ("ccap", "FuCo/Co"): 51.2, ("ccap", "DfsFuCo/Co"): 40.0,
}

STAGES = {
    "P": dict(compress="none", fuse=0, schedule=0),
    "Re": dict(compress="repair", fuse=0, schedule=0),
    "Co": dict(compress="xorrepair", fuse=0, schedule=0),
    "Fu": dict(compress="none", fuse=1, schedule=0),
    "FuCo": dict(compress="xorrepair", fuse=1, schedule=0),
    "DfsFuCo": dict(compress="xorrepair", fuse=1, schedule=1),
}


def metrics(bits):
    out = {}
    for name, kw in STAGES.items():
        p = X.xslp_compile(bits, specialise=0, **kw)
        s = p.stats()
        out[name] = dict(xor=s["xor_count"], mem=s["mem_count"], nvar=s["nvar"], ccap=p.ccap())
    return out


def dataset(n=10, p=4):
    g = X.xslp_coding_matrix(n, p)
    yield "enc", X.xslp_encode_bitmatrix(g, n, p)
    for er in itertools.combinations(range(n + p), p):
        yield er, X.xslp_decode_bitmatrix(g, n, p, er)[0]


def averages(rows):
    def avg(f):
        return 100.0 * sum(f(r) for r in rows) / len(rows)
    return {
        ("xor", "repair/P"): avg(lambda r: r["Re"]["xor"] / r["P"]["xor"]),
        ("xor", "xorrepair/P"): avg(lambda r: r["Co"]["xor"] / r["P"]["xor"]),
        ("mem", "Co/P"): avg(lambda r: r["Co"]["mem"] / r["P"]["mem"]),
        ("mem", "Fu/P"): avg(lambda r: r["Fu"]["mem"] / r["P"]["mem"]),
        ("mem", "FuCo/Co"): avg(lambda r: r["FuCo"]["mem"] / r["Co"]["mem"]),
        ("mem", "FuCo/P"): avg(lambda r: r["FuCo"]["mem"] / r["P"]["mem"]),
        ("nvar", "Co/P"): avg(lambda r: r["Co"]["nvar"] / r["P"]["nvar"]),
        ("nvar", "Fu/P"): avg(lambda r: r["Fu"]["nvar"] / r["P"]["nvar"]),
        ("nvar", "FuCo/Co"): avg(lambda r: r["FuCo"]["nvar"] / r["Co"]["nvar"]),
        ("nvar", "DfsFuCo/Co"): avg(lambda r: r["DfsFuCo"]["nvar"] / r["Co"]["nvar"]),
        ("ccap", "Co/P"): avg(lambda r: r["Co"]["ccap"] / r["P"]["ccap"]),
        ("ccap", "Fu/P"): avg(lambda r: r["Fu"]["ccap"] / r["P"]["ccap"]),
        ("ccap", "FuCo/Co"): avg(lambda r: r["FuCo"]["ccap"] / r["Co"]["ccap"]),
        ("ccap", "DfsFuCo/Co"): avg(lambda r: r["DfsFuCo"]["ccap"] / r["Co"]["ccap"]),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    items = list(dataset())
    if a.limit:
        items = items[:a.limit]
    with ThreadPoolExecutor(a.workers) as ex:
        rows = list(ex.map(lambda it: metrics(it[1]), items))
    av = averages(rows)
    print(f"# Dataset averages over {len(rows)} RS(10,4) SLPs (P:1371-1373)\n")
    print("| measure | ratio | this build (%) | paper (%) |\n|---|---|---|---|")
    for k, v in av.items():
        print(f"| {k[0]} | {k[1]} | {v:.1f} | {PAPER[k]} |")
    enc = rows[0]
    print("\nP_enc per stage (P:1652-1655): ")
    for name in STAGES:
        print(f"- {name}: {enc[name]}")


if __name__ == "__main__":
    main()
