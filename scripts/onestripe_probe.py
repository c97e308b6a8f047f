"""Probe: one stripe through xslp_encode (block pointers as kernel arguments) with large blocks:
the register-resident kernel (xslp_sl_one) against the pipeline's single-stripe entry
(xslp_sl_pipe_one), RS(10,4) encode, blocks of 16 / 107 MiB; and the same bytes as a 1024-stripe
batch for scale.  GB/s of data.  Prints JSON lines."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2108_02692_b200 as X  # noqa: E402


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


n, p = 10, 4
g = X.xslp_coding_matrix(n, p)
bits = X.xslp_encode_bitmatrix(g, n, p)
for B in (16 << 20, 107374208):
    d = torch.empty((n, B), dtype=torch.uint8, device="cuda")
    X.xslp_fill_random(d.view(1, n, B), 1, n, B, seed=1)
    o = torch.empty((p, B), dtype=torch.uint8, device="cuda")
    ins, outs = X.block_ptrs([d[j] for j in range(n)]), X.block_ptrs([o[i] for i in range(p)])
    ref = None
    for kern, T, L in (("straight", 128, 1), ("straight", 128, 2), ("pipe", 128, 1), ("pipe", 128, 2),
                       ("pipe", 256, 1)):
        prog = X.xslp_compile(bits, kernel=kern, threads=T, lane_words=L)
        ms = timed(lambda: X.xslp_encode(prog, ins, outs, B))
        if ref is None:
            ref = o.clone()
        assert torch.equal(o, ref)
        print(json.dumps({"probe": "one stripe RS(10,4) encode", "block_bytes": B, "kernel": kern,
                          "threads": T, "lanes": L, "gbs": round(n * B / ms / 1e6, 1)}), flush=True)
    del d, o
    torch.cuda.empty_cache()
