"""Probe: throughput of the codec front end (`xslp_codec_*`) on device data of
arbitrary length -- encode (copy + pad into n+p shards, then the parity), reconstruct of
4 erased shards (memoised decode program) and decode back to the original bytes -- for
RS(10,4) at 10 MiB, 100 MiB and 1 GiB.  GB/s of data (10^9 B), CUDA events, 20 calls each
after warm-up.  Prints JSON lines."""
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


T = int(sys.argv[1]) if len(sys.argv) > 1 else 128     # consumer threads of the codec's programs
c = X.Codec(10, 4, threads=T)
for length in (10 << 20, 100 << 20, 1 << 30):
    B = c.block_bytes(length)
    data = torch.empty(length, dtype=torch.uint8, device="cuda")
    X.xslp_fill_random(data.view(1, 1, length), 1, 1, length, seed=3)
    shards = torch.empty((14, B), dtype=torch.uint8, device="cuda")
    out = torch.empty(length, dtype=torch.uint8, device="cuda")
    ms_e = timed(lambda: c.encode(data, length, shards))
    ref = shards.clone()
    er = [2, 4, 5, 6]
    ms_r = timed(lambda: c.reconstruct(shards, er, length))
    assert torch.equal(shards, ref)
    ms_d = timed(lambda: c.decode(shards, er, length, out))
    assert torch.equal(out, data)
    print(json.dumps({"probe": "codec RS(10,4)", "threads": T, "bytes": length, "block_bytes": B,
                      "encode_gbs": round(length / ms_e / 1e6, 1),
                      "reconstruct4_gbs": round(length / ms_r / 1e6, 1),
                      "decode4_gbs": round(length / ms_d / 1e6, 1)}), flush=True)
    del data, shards, out, ref
    torch.cuda.empty_cache()
