"""Probe: the multi-program kernel with ONE program (P_dec on every stripe) against the PIPE
kernel on the same data -- separates the multi kernel's tile order / dispatch cost from the
instruction-fetch cost of many programs.  Prints GB/s of data for each."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2108_02692_b200 as X  # noqa: E402

n, p, B, S = 10, 4, 1 << 20, 1024
g = X.xslp_coding_matrix(n, p)
bits, _ = X.xslp_decode_bitmatrix(g, n, p, [2, 4, 5, 6])
din = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
X.xslp_fill_random(din, S, n, B, seed=3)
out = torch.empty((S, 4, B), dtype=torch.uint8, device="cuda")
ti, to = X.block_table(din, S, n, B), X.block_table(out, S, 4, B)


def timeit(fn, steps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return S * n * B * steps / (e0.elapsed_time(e1) / 1e3) / 1e9


pipe = X.xslp_compile(bits, kernel="pipe", threads=256, stages=2, block_bytes_hint=B)
print("pipe T=256", round(timeit(lambda: X.xslp_encode_batch(pipe, ti, to, S, B)), 1))
one = X.xslp_compile(bits, specialise=0)
for copies, pm in ((56, 56), (128, 128), (256, 256), (56, 28), (56, 14), (56, 5)):
    progs = [one] * copies   # the same program repeated: module code size grows, work does not
    m = X.Multi(progs, per_module=pm, threads=256, stages=2, block_bytes_hint=B)
    pos = torch.tensor([s % copies for s in range(S)], dtype=torch.int32, device="cuda")
    ids, off = X.group_stripes([s % copies for s in range(S)], copies)
    ids = torch.from_numpy(ids).cuda()
    print("multi copies", copies, "per module", pm, m.info()["modules"], "modules", round(timeit(lambda: X.xslp_multi_decode(m, pos, ids, off, ti, to, B)), 1))

# real decode programs (the first 56 cfg3 patterns), each owning ~18 stripes, one module;
# then the same 56 programs with stripes assigned round-robin in runs of 1 stripe
import synth  # noqa: E402
pats = sorted(set(tuple(synth.erasure_pattern(3, s, n + p, 4)) for s in range(1024)))[:56]
progs = X.compile_many([X.xslp_decode_bitmatrix(g, n, p, er)[0] for er in pats], specialise=0)
m = X.Multi(progs, per_module=56, threads=256, stages=2, block_bytes_hint=B)
print("real programs", m.info())
for label, posl in (("18-stripe runs", [s * 56 // S for s in range(S)]),
                    ("1-stripe runs", [s % 56 for s in range(S)])):
    pos = torch.tensor(posl, dtype=torch.int32, device="cuda")
    ids, off = X.group_stripes(posl, 56)
    ids = torch.from_numpy(ids).cuda()
    print("real 56 programs,", label, round(timeit(lambda: X.xslp_multi_decode(m, pos, ids, off, ti, to, B)), 1))
