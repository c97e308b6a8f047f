#!/usr/bin/env python
"""SASS instruction mix of the JIT-compiled straight-line kernels (no GPU needed).

    python scripts/sass_evidence.py > profiles/r01_s2_sass.md

Each program's PTX (`prog.dump(2)`) is assembled with ptxas for sm_100a and disassembled with
cuobjdump; the table counts the mnemonics that carry the design: LDS (constant reads from the
TMA stage), LOP3 (3-input XOR), UBLKCP (TMA bulk copy), SYNCS (mbarrier), LDG/STG, BRX."""
import os
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_02692_b200 as X  # noqa: E402
import synth  # noqa: E402

CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
B = 1 << 20


def sass_of(ptx):
    with tempfile.TemporaryDirectory() as d:
        src, cub = os.path.join(d, "k.ptx"), os.path.join(d, "k.cubin")
        open(src, "w").write(ptx)
        subprocess.run([os.path.join(CUDA, "bin", "ptxas"), "-arch=sm_100a", "-O3", src, "-o", cub],
                       check=True, capture_output=True)
        return subprocess.run([os.path.join(CUDA, "bin", "cuobjdump"), "-sass", cub], check=True,
                              capture_output=True, text=True).stdout


def mix(sass, entry):
    m = re.search(r"Function : " + entry + r"\n(.*?)(?=\n\s+Function : |\Z)", sass, re.S)
    body = m.group(1) if m else ""
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", body)
    def c(pfx):
        return sum(1 for o in ops if o.startswith(pfx))
    return dict(total=len(ops), LDS=c("LDS"), LOP3=c("LOP3"), UBLKCP=c("UBLKCP"), SYNCS=c("SYNCS"),
                LDG=c("LDG"), STG=c("STG"), BRX=c("BRX"), SHF=c("SHF"), PRMT=c("PRMT"))


def main():
    g10, g20 = X.xslp_coding_matrix(10, 4), X.xslp_coding_matrix(20, 4)
    er = synth.erasure_pattern(5, 0, 24, 4)
    cases = [
        ("cfg2 RS(10,4) enc, PIPE T=128 x 2 words (default line)",
         X.xslp_encode_bitmatrix(g10, 10, 4), dict(kernel="pipe", threads=128, lane_words=2, reuse=32),
         "xslp_sl_pipe"),
        ("cfg2, same launch, reuse window off",
         X.xslp_encode_bitmatrix(g10, 10, 4), dict(kernel="pipe", threads=128, lane_words=2, reuse=-1),
         "xslp_sl_pipe"),
        ("cfg5 RS(20,4) enc, PIPE T=256, 2 input phases",
         X.xslp_encode_bitmatrix(g20, 20, 4), dict(kernel="pipe", threads=256, phases=2), "xslp_sl_pipe"),
        ("cfg5, same launch, reuse window off",
         X.xslp_encode_bitmatrix(g20, 20, 4), dict(kernel="pipe", threads=256, phases=2, reuse=-1),
         "xslp_sl_pipe"),
        ("cfg5d RS(20,4) dec, PIPE T=256, 2 input phases",
         X.xslp_decode_bitmatrix(g20, 20, 4, er)[0], dict(kernel="pipe", threads=256, phases=2), "xslp_sl_pipe"),
        ("cfg2b RS(10,4) enc, byte layout, PIPE T=256",
         X.xslp_encode_bitmatrix(g10, 10, 4), dict(kernel="pipe", threads=256, layout="byte"), "xslp_sl_pipe"),
    ]
    print("# SASS instruction mix (round 1, session 2) -- `scripts/sass_evidence.py`\n")
    print("PTX from `prog.dump(2)` assembled with `ptxas -arch=sm_100a`, counted with `cuobjdump -sass`;")
    print("`reuse` = the constant register reuse window (`xslp_opts.reuse`, auto = 64).\n")
    print("| program / launch | entry | reuse | SASS | LDS | LOP3 | UBLKCP | SYNCS | LDG | STG | SHF | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for label, bits, kw, entry in cases:
        p = X.xslp_compile(bits, block_bytes_hint=B, stages=2, **kw)
        m = mix(sass_of(p.dump(2)), entry)
        st = p.stats()
        r = kw.get("reuse", 0)
        print(f"| {label} | `{entry}` | {'auto (64)' if r == 0 else 'off' if r < 0 else r} | {m['total']} | "
              f"{m['LDS']} | {m['LOP3']} | {m['UBLKCP']} | {m['SYNCS']} | {m['LDG']} | {m['STG']} | "
              f"{m['SHF']} | {st['regs_pipe']} |")
    # the library's precompiled kernels (approach (1)): SASS straight from libxslp.so
    lib = os.path.join(os.path.dirname(X.__file__), "libxslp.so")
    sass = subprocess.run([os.path.join(CUDA, "bin", "cuobjdump"), "-sass", lib], check=True,
                          capture_output=True, text=True).stdout
    ent = re.search(r"Function : (\S*xslp_gftable_kernelILi4ELi2E\S*)", sass)
    if ent:
        m = mix(sass, re.escape(ent.group(1)))
        print(f"\nApproach (1), `xslp_gftable_kernel<4, 2>` (RS(10,4) rows, 2 x 16 B per thread): "
              f"{m['total']} SASS, PRMT {m['PRMT']}, LOP3 {m['LOP3']}, SHF {m['SHF']}, LDS {m['LDS']} "
              f"(the two-block main loop body plus the odd-block tail and the table build).")
    print("\nNo `HMMA`/`UTC*MMA`: the path is bitwise XOR over HBM streams, not a contraction.")


if __name__ == "__main__":
    main()
