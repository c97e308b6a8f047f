"""Probe: speed of light for the cfg2 traffic mix (read 10 x 1 MiB, write 4 x 1 MiB per stripe,
1024 stripes).  The same PIPE launch as the default bench line runs (a) the compiled RS(10,4)
encode program and (b) a minimum-compute program with the identical memory traffic: 32 goals,
goal r = XOR of input strips r, r+32, r+64 (<80), so every input strip is read once and every
output strip written once with 48 XORs instead of 389.  A plain device-to-device copy of the same
14 GiB (10 read + 4 written is not a copy; reported for scale: read 7 GiB + write 7 GiB) and a
read-only XOR-reduce kernel give the memory system's other reference points.  Prints JSON
lines: GB/s of data (10 x 1 MiB per stripe) and HBM GB/s (read + written bytes)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02692_b200 as X  # noqa: E402

n, p, B, S = 10, 4, 1 << 20, 1024
if "--rs20" in sys.argv:        # the cfg5 code: RS(20,4), 2 input phases (bench's cfg5 launch)
    n = 20
PH = 2 if n > 10 else 0
LAUNCHES = ((256, 1),) if n > 10 else ((128, 2), (256, 1))
din = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
X.xslp_fill_random(din, S, n, B, seed=2)
out = torch.empty((S, p, B), dtype=torch.uint8, device="cuda")
ti, to = X.block_table(din, S, n, B), X.block_table(out, S, p, B)


def timeit(fn, steps=50, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps        # ms per step


def report(name, ms, data_bytes, hbm_bytes):
    print(json.dumps({"probe": name, "ms": round(ms, 4), "data_gbs": round(data_bytes / ms / 1e6, 1),
                      "hbm_gbs": round(hbm_bytes / ms / 1e6, 1)}), flush=True)


g = X.xslp_coding_matrix(n, p)
rs_bits = X.xslp_encode_bitmatrix(g, n, p)
thin = np.zeros((8 * p, 8 * n), dtype=np.uint8)
for r in range(8 * p):
    for c in range(r, 8 * n, 8 * p):
        thin[r, c] = 1
data, hbm = S * n * B, S * (n + p) * B
for label, bits in (("rs10_4_encode", rs_bits), ("min_compute_same_traffic", thin)):
    for threads, lanes in LAUNCHES:
        prog = X.xslp_compile(bits, kernel="pipe", threads=threads, lane_words=lanes, stages=2,
                              block_bytes_hint=B, phases=PH)
        st = prog.stats()
        ms = timeit(lambda: X.xslp_encode_batch(prog, ti, to, S, B))
        report(f"RS({n},{p}) {label} pipe T={threads} L={lanes} phases={PH} xor={st['xor_count']}",
               ms, data, hbm)
# plain copies for scale: torch's copy kernel over the same byte count (read 7 GiB + write 7 GiB)
a = din.view(-1)[: hbm // 2]
b = torch.empty_like(a)
ms = timeit(lambda: b.copy_(a))
report("torch copy 7 GiB -> 7 GiB", ms, 0, hbm)

# HBM throughput against the write share: m goal strips per stripe (goal r = XOR of the input
# strips c = r mod m), same launch; m = 32 is the traffic above (the batched API needs whole output blocks: m a multiple of 8)
if "--mix" in sys.argv:
    for m in (8, 16, 32, 48, 64):
        bits = np.zeros((m, 8 * n), dtype=np.uint8)
        for c in range(8 * n):
            bits[c % m, c] = 1
        o = torch.empty((S, (m + 7) // 8, B), dtype=torch.uint8, device="cuda")
        prog = X.xslp_compile(bits, kernel="pipe", threads=128, lane_words=2, stages=2,
                              block_bytes_hint=B)
        to_m = X.block_table(o, S, (m + 7) // 8, B)
        ms = timeit(lambda: X.xslp_encode_batch(prog, ti, to_m, S, B))
        report(f"mix m={m} goal strips (write {m / 8:.3g} blocks per 10 read)", ms, data,
               S * n * B + S * m * (B // 8))
