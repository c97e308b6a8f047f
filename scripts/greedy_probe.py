#!/usr/bin/env python
"""DFS vs capacity-bounded greedy schedule (P:1279-1303 vs P:1305-1338)
on the programs where register pressure matters: registers and spills of the straight-line
kernels as ptxas allocates them, resident CTAs per SM, the SLP's max-live, the interpreter's
variable rows, and the paper's LRU IOcost at the same capacity.  Host only (no GPU): the JIT
compile is in-process.  GB/s come from bench.py (scripts/r02_greedy.sh).

    python scripts/greedy_probe.py > profiles/r02/greedy_vs_dfs.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02692_b200 as X  # noqa: E402
import synth  # noqa: E402

REGS_PER_SM = 65536


def ctas(regs, threads):
    if regs <= 0:
        return 0
    per_warp = ((regs * 32 + 255) // 256) * 256          # allocation granularity (per warp)
    return min(32, REGS_PER_SM // (per_warp * (threads // 32)))


def row(name, bits, sched, cap, threads=128):
    kw = dict(schedule=sched, greedy_capacity=cap or 1, threads=threads, block_bytes_hint=1 << 20)
    p = X.xslp_compile(bits, kernel="straight", **kw)
    st = p.stats()
    pp = X.xslp_compile(bits, kernel="pipe", threads=256, stages=2, **{k: v for k, v in kw.items() if k != "threads"})
    sp = pp.stats()
    pi = X.xslp_compile(bits, kernel="interp", specialise=0, lane_words=1, stages=2,
                        **{k: v for k, v in kw.items() if k != "block_bytes_hint"})
    w = [int(x) for x in pi.dump(3).split()]
    io = pi.iocost(64) if hasattr(pi, "iocost") else None
    label = "DFS" if sched == 1 else f"greedy c={cap}"
    return (f"| {name} | {label} | {st['n_instr']} | {st['maxlive']} | {st['regs']} | {st['spill_bytes']} | "
            f"{ctas(st['regs'], threads)} | {sp['regs_pipe']} | {sp['spill_bytes_pipe']} | {w[3]} |")


def main():
    g20 = X.xslp_coding_matrix(20, 4)
    g10 = X.xslp_coding_matrix(10, 4)
    cases = [("RS(20,4) dec cfg5d " + str(synth.erasure_pattern(5, 0, 24, 4)),
              X.xslp_decode_bitmatrix(g20, 20, 4, synth.erasure_pattern(5, 0, 24, 4))[0]),
             ("RS(20,4) dec {0,5,21,23}", X.xslp_decode_bitmatrix(g20, 20, 4, [0, 5, 21, 23])[0]),
             ("RS(10,4) P_dec {2,4,5,6}", X.xslp_decode_bitmatrix(g10, 10, 4, [2, 4, 5, 6])[0]),
             ("RS(10,4) enc", X.xslp_encode_bitmatrix(g10, 10, 4))]
    print("| program | schedule | instr | max-live | LDG regs | LDG spill B | LDG CTAs/SM (T=128) | "
          "PIPE regs (T=256) | PIPE spill B | interp var rows |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for name, bits in cases:
        for sched, cap in ((1, 0), (2, 16), (2, 64), (2, 512)):
            print(row(name, bits, sched, cap))


if __name__ == "__main__":
    main()
