"""Probe: BASELINE configs[0] latency -- RS(4,2) Cauchy, one stripe of 4 x 4 KiB, encode and the
decode of erased data blocks {0, 1} through the single-stripe C-ABI calls (xslp_encode /
xslp_decode with per-block pointers), straight-line and interpreter kernels; device time per
call from CUDA events over 2000 back-to-back calls, plus the host wall time of one synchronous
call and of a CUDA-graph replay of the same call.  Back-to-back Python calls are host-bound
(the device waits for the next launch), so the kernel's own time per call comes from replaying
100 captured calls as one graph.  Prints JSON lines (microseconds)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2108_02692_b200 as X  # noqa: E402

n, p, B = 4, 2, 4096
g = X.xslp_coding_matrix(n, p, "cauchy")
d = torch.empty((1, n + p, B), dtype=torch.uint8, device="cuda")
X.xslp_fill_random(d, 1, n + p, B, seed=1)
data = [d[0, j] for j in range(n)]
par = [d[0, n + i] for i in range(p)]
rec = torch.empty((2, B), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def device_us(fn, iters=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def sync_us(fn, iters=500):
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e6


for kern in ("straight", "interp"):
    enc = X.xslp_compile(X.xslp_encode_bitmatrix(g, n, p), kernel=kern, block_bytes_hint=B)
    bits, surv = X.xslp_decode_bitmatrix(g, n, p, [0, 1])
    dec = X.xslp_compile(bits, kernel=kern, block_bytes_hint=B)
    pin, pout = X.block_ptrs(data), X.block_ptrs(par)
    psv, prec = X.block_ptrs([d[0, k] for k in surv]), X.block_ptrs([rec[0], rec[1]])
    fe = lambda: X.xslp_encode(enc, pin, pout, B)                                   # noqa: E731
    fd = lambda: X.xslp_decode(dec, psv, prec, B)                                   # noqa: E731
    for name, fn in (("encode", fe), ("decode{0,1}", fd)):
        line = {"probe": f"cfg1 {name} {kern}", "device_us_per_call": round(device_us(fn), 2),
                "sync_call_us_median": round(sync_us(fn), 1)}
        # host cost of one call (Python + ctypes + launch), no synchronisation
        for _ in range(100):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(1000):
            fn()
        line["host_us_per_call"] = round((time.perf_counter() - t0) * 1e3, 2)
        torch.cuda.synchronize()
        if kern == "straight":
            X.xslp_prepare(enc if name == "encode" else dec)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn()
            line["graph_replay_sync_us_median"] = round(sync_us(gr.replay), 1)
            g100 = torch.cuda.CUDAGraph()      # 100 calls in one graph: kernel time per call
            with torch.cuda.graph(g100):
                for _ in range(100):
                    fn()
            line["device_us_per_call_graph100"] = round(device_us(g100.replay, iters=50) / 100, 2)
        print(json.dumps(line), flush=True)
fe()
torch.cuda.synchronize()
