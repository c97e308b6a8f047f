#!/usr/bin/env python
"""bench.py -- device-timed RS(n,p) XOR-SLP encode/decode throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2|cfg3|cfg4|cfg5]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
    python bench.py --impl reference          # the CPU oracle arm (rank 0 only)

Metric (BASELINE.json): GB/s of data (10^9 bytes of the n data blocks per stripe,
reading R14), device-timed with CUDA events on the launching stream, max over
ranks; value = all ranks' data / that time.  A "step" is one pass of the device
hot path over the workload's stripes: one launch of the
compiled program over every stripe.  Compilation (H1-H7) is untimed.

Default workload = BASELINE configs[1] (cfg2): RS(10,4) encode of 1024 stripes x
10 x 1 MiB per GPU (weak scaling: rank r owns global stripes [r*1024, (r+1)*1024)).
Inputs (10 GiB) exceed the 126 MB L2, so no flush is needed between steps.
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

def log(*a):
    print(f"[bench {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


METRIC = "RS encode/decode GB/s of data (device-timed) at 1/2/4/8 B200; % of roofline"
MiB = 1 << 20

WORKLOADS = {
    "cfg2": dict(desc="RS(10,4) encode, 1024 stripes x 10 x 1 MiB per GPU (BASELINE configs[1])",
                 n=10, p=4, B=MiB, S=1024, op="encode", seed=2,
                 tuned=dict(kernel="pipe", threads=128, lanes=2, stages=3, phases=2, reuse=32)),
    "cfg2b": dict(desc="RS(10,4) encode in the byte-compatible layout (output = textbook byte-wise "
                       "RS, SURVEY NEXT #3), 1024 stripes x 10 x 1 MiB",
                  n=10, p=4, B=MiB, S=1024, op="encode", seed=2, layout="byte",
                  tuned=dict(kernel="pipe", threads=256, stages=2)),
    "cfg2t": dict(desc="RS(10,4) encode in the byte layout with the paper's approach (1) on the GPU: "
                       "byte-wise GF(2^8) MM with nibble-table multiplication (PRMT), the comparison "
                       "point for cfg2b's XOR program, 1024 stripes x 10 x 1 MiB",
                  n=10, p=4, B=MiB, S=1024, op="encode_gft", seed=2,
                  tuned=dict(kernel="gftable", threads=256, stages=2)),
    "cfg3": dict(desc="RS(10,4) decode, 1024 stripes x 1 MiB, per-stripe seeded 4-of-14 erasures, "
                      "recovered by the inverted-submatrix (M^-1) bitmatrix SLP compiled per erasure "
                      "pattern (BASELINE configs[2]; P:526-530), the patterns' programs fused into "
                      "multi-program kernels (20 per kernel, branch table per stripe); --kernel "
                      "syndrome: shared syndrome program + per-pattern solve programs; --kernel "
                      "grouped: one straight-line kernel per pattern; --kernel interp",
                 n=10, p=4, B=MiB, S=1024, op="decode_multi", e=4, seed=3,
                 tuned=dict(kernel="multi", threads=256, stages=2, per_module=20, graph=1),
                 alt=dict(syndrome=dict(threads=256, stages=2, per_module=16, reuse=40, graph=1))),
    "pdec": dict(desc="RS(10,4) decode of the paper's P_dec pattern {2,4,5,6} (P:1670) on every "
                      "stripe, 1024 stripes x 1 MiB",
                 n=10, p=4, B=MiB, S=1024, op="decode_one", erased=(2, 4, 5, 6), seed=3,
                 tuned=dict(kernel="pipe", threads=128, lanes=2, stages=2)),
    "cfg4": dict(desc="RS(10,p) encode sweep point (BASELINE configs[3]): total data fixed at "
                      "10 GiB, stripes = 10 GiB / (n x block)",
                 n=10, p=4, B=MiB, S=1024, op="encode", seed=4,
                 tuned=dict(kernel="pipe", threads=256, stages=2)),
    "cfg5": dict(desc="RS(20,4) encode, 8192 stripes x 20 x 1 MiB sharded over the GPUs; chunks "
                      "of <=2048 stripes per launch (BASELINE configs[4])",
                 n=20, p=4, B=MiB, S=8192, op="encode_sharded", seed=5, chunk=2048,
                 tuned=dict(kernel="pipe", threads=256, stages=2, phases=2)),
    "cfg5d": dict(desc="RS(20,4) decode of one seeded random 4-erasure pattern (synth.erasure_pattern"
                       "(5, 0, 24, 4)) applied to every stripe, 8192 stripes x 1 MiB sharded over the "
                       "GPUs; chunks of <=2048 stripes per launch (BASELINE configs[4], decode half)",
                  n=20, p=4, B=MiB, S=8192, op="decode_sharded", e=4, seed=5, chunk=2048,
                  tuned=dict(kernel="pipe", threads=256, stages=2, phases=2)),
    "cfg5h": dict(desc="RS(20,4) decode with per-stripe seeded 4-of-24 erasures (the secondary "
                       "reading of BASELINE configs[4]), 1024 stripes x 1 MiB per GPU: syndrome form (shared "
                       "syndrome program over 24 blocks in 6 input phases + per-pattern solve "
                       "programs, 10 per kernel); --kernel multi: the M^-1 programs fused",
                  n=20, p=4, B=MiB, S=1024, op="decode_multi", e=4, seed=5,
                  tuned=dict(kernel="syndrome", threads=256, stages=3, phases=6, per_module=10, graph=1),
                  # T=224 keeps the CTA at 8 warps (2 per SMSP): 128 registers, 2 CTAs per SM
                  alt=dict(multi=dict(threads=224, stages=3, phases=6, per_module=10, graph=1))),
    "xdec": dict(desc="RS(10,4) cross-GPU decode (SURVEY NEXT #4): the 14 blocks of each stripe "
                      "spread over the GPUs (block j of stripe s on rank (s+j) mod N), rank s mod N "
                      "decodes stripe s reading its survivors in place from local and NVLink-peer "
                      "memory; per-stripe seeded 4-of-14 erasures (cfg3's), 1024 stripes x 1 MiB "
                      "per GPU",
                 n=10, p=4, B=MiB, S=1024, op="decode_peer", e=4, seed=3,
                 tuned=dict(kernel="grouped", threads=64, stages=2)),
    "xdec1": dict(desc="RS(10,4) cross-GPU decode of P_dec {2,4,5,6} on every stripe (one launch "
                       "whose pointer table mixes local and NVLink-peer survivor blocks), 1024 "
                       "stripes x 1 MiB per GPU, blocks spread as in xdec",
                  n=10, p=4, B=MiB, S=1024, op="decode_peer", erased=(2, 4, 5, 6), seed=3,
                  tuned=dict(kernel="straight", threads=128, stages=2)),
}

SHARDED = ("encode_sharded", "decode_sharded")     # strong scaling: fixed total over the ranks
DECODE = ("decode_one", "decode_sharded", "decode_multi", "decode_peer")
NVLINK_GBS = 770.0   # B200_PROFILING.md: measured peer copy bandwidth per direction
HBM_NOMINAL_GBS = 7700.0  # B200_PROFILING.md: HBM3e nominal (HGX figure)
ALU_LANE_OPS_PER_CLK_SM = 64  # measured: scripts/alu_probe.cu (LOP3 and PRMT alike)
NUM_SMS = 148


def erased_of(wl):
    """The single erasure pattern of a decode_one / decode_sharded workload."""
    if "erased" in wl:
        return tuple(wl["erased"])
    import synth
    return tuple(synth.erasure_pattern(wl["seed"], 0, wl["n"] + wl["p"], wl["e"]))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="xslp", choices=["xslp", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--compress", default="xorrepair", choices=["none", "repair", "xorrepair"])
    ap.add_argument("--kernel", default=None,
                    choices=["auto", "straight", "interp", "tma", "pipe", "grouped", "grouped_tma",
                             "grouped_pipe", "multi", "gftable", "syndrome"])
    ap.add_argument("--stages", type=int, default=None)
    ap.add_argument("--streams", type=int, default=8, help="internal streams for grouped decode")
    ap.add_argument("--xmode", default="peer", choices=["peer", "staged"],
                    help="cross-GPU decode: read survivors in place over NVLink (peer), or the "
                         "baseline: NCCL point-to-point into a staging buffer, then decode (staged)")
    ap.add_argument("--lanes", type=int, default=None)
    ap.add_argument("--groups", type=int, default=None, help="PIPE consumer groups (goal split)")
    ap.add_argument("--phases", type=int, default=None, help="PIPE input phases (K-split)")
    ap.add_argument("--reuse", type=int, default=None,
                    help="constant register reuse window (xslp_opts.reuse): 0 auto, -1 off")
    ap.add_argument("--distinct", type=int, default=0,
                    help="diagnostic: only K distinct erasure patterns (stripe s takes pattern s mod K)")
    ap.add_argument("--per-module", type=int, default=None,
                    help="programs (or erasure patterns) per fused kernel (--kernel multi / syndrome)")
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--block-bytes", type=int, default=0, help="override block size")
    ap.add_argument("--p", type=int, default=0, help="override parity count (cfg4 sweep)")
    ap.add_argument("--fuse", type=int, default=1)
    ap.add_argument("--schedule", type=int, default=1,
                    help="1 = DFS (P:1279-1303), 0 = creation order, 2 = capacity-bounded greedy "
                         "(P:1305-1338, capacity --greedy-capacity)")
    ap.add_argument("--greedy-capacity", type=int, default=64)
    ap.add_argument("--interp", default="tmem", choices=["lanes", "pairs", "tmem"],
                    help="--kernel interp: the TMEM-variable (default), the lane-parallel or the "
                         "pair-pipelined interpreter")
    ap.add_argument("--peer-tma", type=int, default=0,
                    help="xdec/xdec1 at N>1: 1 = TMA-staged kernels (PIPE / fused multi-program) "
                         "bulk-copy peer strips (opt-in; default: LDG straight-line kernels)")
    ap.add_argument("--graph", type=int, default=None,
                    help="1 = capture one step's launches into a CUDA graph and replay it per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    return ap.parse_args()


def measured_peak():
    for path in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        try:
            with open(path) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(workload):
    """dram bytes per launch from a committed `ncu --set full` capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.power, self.limit_w = [], None
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
            except Exception:
                pass
        except Exception:
            self.max = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        pw = sorted(self.power)
        return {"sm_mhz": med, "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(s), "source": "nvml" if self.ok else "unavailable",
                "power_w": round(pw[len(pw) // 2], 1) if pw else None,
                "power_limit_w": self.limit_w}


# ------------------------------------------------------------------------------------------
def oracle_rows(wl, g, s, rows_cache, synth, mx):
    """GF rows the workload applies to stripe s: the parity rows R (encode), or the decode
    rows of that stripe's erasure pattern (the oracle's cost does not depend on the
    survivor bytes, so the stripe's seeded blocks stand in for them)."""
    n, p = wl["n"], wl["p"]
    if wl["op"] not in DECODE:
        return g[n:]
    if "erased" not in wl and "e" in wl:
        er = tuple(synth.erasure_pattern(wl["seed"], s, n + p, wl["e"]))
    else:
        er = tuple(erased_of(wl))
    if er not in rows_cache:
        rows_cache[er] = mx.decode_rows(g, n, list(er))[1]
    return rows_cache[er]


class OracleSample:
    """A bounded sample of the workload for the C oracle (oracle/rs_oracle.c): K stripes'
    inputs generated up front (untimed) and their per-stripe rows; run() applies them on
    `threads` host threads -- the table-free naive bitmatrix product on the strip layout, or
    the textbook byte-wise product for the byte layout / approach (1)."""

    def __init__(self, wl, k):
        import numpy as np
        import synth
        from oracle import matrices as mx
        from oracle import native as nat
        self.nat = nat
        n, p, B = wl["n"], wl["p"], wl["B"]
        g = mx.coding_matrix(n, p)
        self.k = max(1, min(k, wl["S"]))
        cache = {}
        self.rows = np.array([oracle_rows(wl, g, s, cache, synth, mx) for s in range(self.k)],
                             dtype=np.uint8)
        self.x = np.stack([nat.fill(wl["seed"], s, n, B) for s in range(self.k)])
        self.bytewise = wl["op"] == "encode_gft" or wl.get("layout") == "byte"
        self.bytes = self.k * n * B

    def run(self, threads):
        self.nat.apply_each(self.rows, self.x, threads=threads, bytewise=self.bytewise)


def oracle_baseline(wl, budget_s=8.0):
    """The CPU oracle as it stands (oracle/rs_oracle.c) on a bounded sample of the workload,
    on one host core and on all of them."""
    from oracle import native as nat
    smp = OracleSample(wl, 32)
    out = {}
    for key, th in (("one_core", 1), ("all_cores", nat.cores())):
        t0, reps = time.perf_counter(), 0
        while True:
            smp.run(th)
            reps += 1
            if time.perf_counter() - t0 > budget_s / 2:
                break
        dt = time.perf_counter() - t0
        out[key] = {"value": round(reps * smp.bytes / dt / 1e9, 4), "unit": "GB/s", "cores": th,
                    "kind": "oracle",
                    "sample": f"{reps} pass(es) over {smp.k} stripe(s) of the workload "
                              f"({wl['n']} x {wl['B']} B data each, inputs generated untimed), "
                              f"oracle/rs_oracle.c on {th} thread(s), {dt:.1f} s"}
    line = dict(out["all_cores"])
    line["one_core"] = out["one_core"]
    return line


def run_reference(args, wl, rank, world):
    """The reference arm: the oracle as it stands on the host cores (rank 0 only); each step is
    one pass of the C oracle over a bounded sample of the workload's stripes."""
    if rank != 0:
        return
    from oracle import native as nat
    smp = OracleSample(wl, 32)
    th = nat.cores()
    for _ in range(args.warmup):
        smp.run(th)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        smp.run(th)
    dt = time.perf_counter() - t0
    v = args.steps * smp.bytes / dt / 1e9
    sample = (f"each step = {smp.k} stripe(s) of the workload ({wl['n']} x {wl['B']} B data each, "
              f"inputs generated untimed) through oracle/rs_oracle.c on {th} host thread(s)")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / max(1, args.steps) * 1e3, 3), "higher_is_better": True,
            "scaling": "strong" if wl["op"] in SHARDED else "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": config_of(args, wl, None),
            "cpu_baseline": {"value": round(v, 6), "unit": "GB/s", "cores": th, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def kernel_name(args, wl, stats):
    k = args.kernel
    if k == "interp":
        return {"lanes": "xslp_interp_lanes", "pairs": "xslp_interp_pipe",
                "tmem": "xslp_interp_tmem"}[args.interp]
    if k in ("tma", "grouped_tma"):
        return "xslp_sl_tma"
    if k in ("pipe", "grouped_pipe"):
        return "xslp_sl_pipe"
    if k in ("multi", "syndrome"):
        return "xslp_sl_multi"
    if k == "gftable":
        return "xslp_gftable_kernel"
    return "xslp_sl_batch"


def config_of(args, wl, stats):
    c = {"workload": f"{args.workload}: {wl['desc']}", "n": wl["n"], "p": wl["p"],
         "block_bytes": wl["B"], "stripes_per_gpu": wl["S"] if wl["op"] not in SHARDED
         else wl["S"] // max(1, args.gpus),
         "matrix": "[I; 2^(ij)] over GF(2^8)/0x11D", "program": args.compress + ("+fuse" if args.fuse else "") +
         {0: "", 1: "+dfs", 2: f"+greedy(c={args.greedy_capacity})"}.get(args.schedule, ""),
         "kernel": args.kernel if args.kernel != "interp" else f"interp ({args.interp})",
         "lane_words": args.lanes, "threads": args.threads,
         "stages": args.stages, "groups": args.groups,
         "phases": args.phases or (-(-(wl["n"] + wl["p"]) // 10) if args.kernel == "syndrome" else
                                   (-(-wl["n"] // 10) if wl["n"] > 10 else 1)),
         "const_reuse": (args.reuse if args.reuse else
                         ("auto: 16 (syndrome-form kernels)" if args.kernel == "syndrome"
                          else "auto: 64")) if args.kernel not in ("gftable", "interp") else None,
         "cuda_graph": bool(args.graph),
         "l2": "inputs larger than the 126 MB L2; no flush between steps",
         "parallelism": (f"blocks spread over {args.gpus} GPU(s); survivors read in place over "
                         "NVLink P2P by the decode kernel (no collective)" if args.xmode == "peer" else
                         f"blocks spread over {args.gpus} GPU(s); baseline: remote survivors "
                         "gathered by NCCL point-to-point into a staging buffer, then a local decode")
         if wl["op"] == "decode_peer" else f"stripe-sharded x{args.gpus}, no collective"}
    if wl["op"] == "encode_gft":
        c["program"] = "none: GF(2^8) MM with nibble tables (approach (1), P:538-545)"
    if wl["op"] in SHARDED:
        per = wl["S"] // max(1, args.gpus)
        c["chunks_per_gpu"] = -(-per // wl["chunk"])
        c["chunk_stripes"] = min(per, wl["chunk"])
        if c["chunks_per_gpu"] > 1:
            c["chunk_inputs"] = ("every chunk's stripes regenerated on the device (stripe0 = the "
                                 "chunk's first global stripe) before it runs, untimed; a step's "
                                 "time = the sum of its chunks' launch intervals")
    if stats:
        c["slp"] = {k: stats[k] for k in ("xor_count", "mem_count", "n_instr", "nvar", "maxlive",
                                          "regs", "spill_bytes", "regs_tma", "spill_bytes_tma",
                                          "regs_pipe", "spill_bytes_pipe", "group_xor")}
    return c


# ------------------------------------------------------------------------------------------
def launch_ranks(nranks):
    """`--gpus N` without torchrun: start the N ranks ourselves (one process per GPU, the
    driver's own launch line) and return their exit code; rank 0 prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(launch_ranks(args.gpus))
    if env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}: launch one rank "
                         "per GPU (torchrun --nproc-per-node N) or omit torchrun and let --gpus N "
                         "start the ranks")
    wl = dict(WORKLOADS[args.workload])
    # per-workload tuned launch defaults (profiles/r01_sweep*.md, profiles/r02/); a kernel chosen
    # with --kernel takes its own tuned set when the workload has one; flags override
    tuned = dict(wl.get("tuned", {}))
    if args.kernel and args.kernel in wl.get("alt", {}):
        tuned = dict(wl["alt"][args.kernel], kernel=args.kernel)
    elif args.kernel and args.kernel != tuned.get("kernel"):
        tuned = {}  # the workload's tuned set is another kernel's
    for k, v in tuned.items():
        if getattr(args, k) is None:
            setattr(args, k, v)
    args.kernel = args.kernel or "auto"
    args.threads = args.threads or 128
    args.stages = args.stages or 2
    args.groups = args.groups or 1
    args.lanes = args.lanes or 1
    args.per_module_raw = args.per_module
    args.reuse = args.reuse or 0
    args.per_module = args.per_module or 20
    if args.phases is None:            # 0 = the library's auto: ceil(n/10) input phases if n > 10
        args.phases = 0
    args.graph = int(args.graph or 0)
    if args.p:
        wl["p"] = args.p
    if args.block_bytes:
        total = wl["S"] * wl["B"]          # keep the data per GPU fixed
        wl["B"] = args.block_bytes
        wl["S"] = max(1, total // args.block_bytes)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import numpy as np
    import torch
    import paper_2108_02692_b200 as X

    # XSLP_BENCH_SHARED_GPU=1: a control-flow check of the N>1 path on a one-GPU box -- every
    # rank on cuda:0, gloo for the barriers and the max over ranks (the ranks' kernels never wait
    # on one another); its numbers are not throughput claims
    shared_gpu = os.environ.get("XSLP_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist
        if shared_gpu:
            dist.init_process_group("gloo")
            red_dev = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n, p, B = wl["n"], wl["p"], wl["B"]
    G = X.xslp_coding_matrix(n, p)
    stream = torch.cuda.current_stream()

    # ---- compile (untimed, H1-H7) ----
    t0 = time.perf_counter()
    if wl["op"] == "decode_multi":
        import synth
        S = wl["S"]
        s0 = rank * S
        pats = [tuple(synth.erasure_pattern(wl["seed"], (s0 + s) % args.distinct if args.distinct else s0 + s,
                                            n + p, wl["e"])) for s in range(S)]
        uniq = sorted(set(pats))
        dec = [X.xslp_decode_bitmatrix(G, n, p, er) for er in uniq]
        mode = "grouped" if args.kernel == "auto" else args.kernel
        if mode == "syndrome":  # shared syndrome program + per-pattern solve programs, fused
            progs = uniq
            multi = X.SyndromeDecoder(G, n, p, uniq, per_module=args.per_module_raw or 0,
                                      threads=args.threads, stages=args.stages,
                                      lane_words=args.lanes, block_bytes_hint=B, phases=args.phases,
                                      reuse=args.reuse)
            log("syndrome", multi.info())
        elif mode == "multi":   # fused multi-program pipeline kernels (branch table per stripe)
            progs = X.compile_many([d[0] for d in dec], compress=args.compress, specialise=0,
                                   threads=args.threads)
            multi = X.Multi(progs, per_module=args.per_module, threads=args.threads,
                            stages=args.stages, lane_words=args.lanes, block_bytes_hint=B,
                            phases=args.phases, reuse=args.reuse)
            log("multi", multi.info())
        elif mode == "interp":
            progs = X.compile_many([d[0] for d in dec], compress=args.compress, specialise=0,
                                   threads=args.threads, lane_words=args.lanes,
                                   stages=args.stages, interp=args.interp)
        else:   # one JIT straight-line (or TMA) kernel per distinct erasure pattern
            progs = X.compile_many([d[0] for d in dec], compress=args.compress, specialise=1,
                                   threads=args.threads, lane_words=args.lanes,
                                   block_bytes_hint=B,
                                   stages=args.stages,
                                   kernel={"tma": "tma", "grouped_tma": "tma", "pipe": "pipe",
                                           "grouped_pipe": "pipe"}.get(mode, "straight"))
        prog = progs[0] if mode != "syndrome" else None
        m_out = wl["e"]
    elif wl["op"] == "decode_peer":
        import synth
        from paper_2108_02692_b200 import peer
        pl = peer.Placement(n, p, world, wl["S"] * world)
        if "erased" in wl:
            erasures = lambda s: wl["erased"]                                   # noqa: E731
        else:
            erasures = lambda s: synth.erasure_pattern(wl["seed"], s, n + p, wl["e"])  # noqa: E731
        plan = peer.Plan(pl, rank, erasures)
        mode = "grouped" if len(plan.keys) > 1 else "straight"
        progs = peer.compile_plan(X, G, plan, compress=args.compress, threads=args.threads,
                                  lane_words=args.lanes, block_bytes_hint=B, stages=args.stages,
                                  kernel="straight")
        prog = progs[0] if mode != "syndrome" else None
        m_out = plan.e
    elif wl["op"] in ("decode_one", "decode_sharded"):
        erased = erased_of(wl)
        bits, _surv = X.xslp_decode_bitmatrix(G, n, p, erased)
        prog = X.xslp_compile(bits, compress=args.compress, kernel=args.kernel,
                              lane_words=args.lanes, threads=args.threads, block_bytes_hint=B,
                              stages=args.stages, groups=args.groups, phases=args.phases,
                              reuse=args.reuse, schedule=args.schedule,
                              greedy_capacity=args.greedy_capacity, interp=args.interp)
        m_out = len(erased)
    elif wl["op"] == "encode_gft":    # approach (1): no SLP, the coefficient rows themselves
        prog = None
        coef_rows = np.ascontiguousarray(G[n:])
        m_out = p
    else:
        prog = X.xslp_compile(X.xslp_encode_bitmatrix(G, n, p), compress=args.compress,
                              kernel=args.kernel, lane_words=args.lanes, threads=args.threads,
                              block_bytes_hint=B, stages=args.stages, fuse=args.fuse,
                              schedule=args.schedule, greedy_capacity=args.greedy_capacity,
                              interp=args.interp, layout=wl.get("layout", "strip"),
                              groups=args.groups, phases=args.phases, reuse=args.reuse)
        m_out = p
    compile_s = time.perf_counter() - t0
    stats = prog.stats() if prog is not None else None
    log(f'compiled in {compile_s:.2f} s', stats)

    # ---- device buffers and seeded inputs (untimed) ----
    from paper_2108_02692_b200.shard import max_over_ranks, stripe_range
    if wl["op"] in SHARDED:               # strong split of 8192 stripes over the ranks
        lo, hi = stripe_range(rank, world, total=wl["S"])
        per = hi - lo
        S = min(per, wl["chunk"])
        nchunks = (per + S - 1) // S
        stripe0 = lo
    else:                                 # weak scaling: S stripes per rank
        S = wl["S"]
        nchunks = 1
        stripe0 = stripe_range(rank, world, per_rank=S)[0]
    n_in = n
    dout = torch.empty((S, m_out, B), dtype=torch.uint8, device="cuda")
    to = X.block_table(dout, S, m_out, B)
    if wl["op"] == "decode_peer":
        S = len(plan.stripes)
        dout = torch.empty((S, m_out, B), dtype=torch.uint8, device="cuda")
        enc = X.xslp_compile(X.xslp_encode_bitmatrix(G, n, p), block_bytes_hint=B)
        din = torch.empty(pl.storage_shape(B), dtype=torch.uint8, device="cuda")
        peer.fill_storage(X, pl, rank, din, wl["seed"], enc, chunk=32, stream=stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()                # every rank's storage written before any peer read
        pmulti = None
        # TMA-staged kernels (PIPE, fused multi-program) when every block is local, or with
        # --peer-tma 1 (opt-in) also over peer tables; otherwise peer tables keep the LDG
        # straight-line kernel (the path validated over real NVLink P2P)
        use_tma = world == 1 or args.peer_tma
        if use_tma and len(progs) == 1:
            progs = peer.compile_plan(X, G, plan, compress=args.compress, threads=128, lane_words=2,
                                      block_bytes_hint=B, stages=2, kernel="pipe")
            args.kernel, args.threads, args.lanes = "pipe", 128, 2
        if use_tma and len(progs) > 1:      # the fused multi-program kernels
            pmulti = X.Multi(X.compile_many([X.xslp_decode_bitmatrix_from(G, n, p, er, sv)
                                             for er, sv in plan.keys], specialise=0),
                             per_module=args.per_module, threads=256, stages=2, block_bytes_hint=B,
                             reuse=args.reuse)
            args.kernel, args.threads = "multi", 256
        pdec = peer.PeerDecoder(X, pl, din, dout, plan, progs, dist=dist, multi=pmulti,
                                tma=bool(args.peer_tma))
        remote_blocks, all_blocks = plan.remote_reads()
        if args.xmode == "staged":        # baseline: gather the survivors, then a local decode
            staging = torch.empty((len(plan.stripes), n, B), dtype=torch.uint8, device="cuda")
            st_in = X.block_table(staging, len(plan.stripes), n, B)
            sids, soff = plan.groups()
            sids = torch.from_numpy(sids).cuda()
            sgather = peer.StagedGather(pl, plan, din, staging, erasures, X=X)
    elif wl["op"] in ("decode_one", "decode_sharded"):
        # whole codewords (data from the generator, parity by the encode program, untimed);
        # the decode program reads the n survivors of each stripe through the pointer table
        din = torch.empty((S, n + p, B), dtype=torch.uint8, device="cuda")
        X.xslp_fill_random(din, S, n + p, B, seed=wl["seed"], stripe0=stripe0)
        tall = X.block_table(din, S, n + p, B).view(S, n + p)
        enc = X.xslp_compile(X.xslp_encode_bitmatrix(G, n, p), block_bytes_hint=B)
        X.xslp_encode_batch(enc, tall[:, :n].contiguous(), tall[:, n:].contiguous(), S, B,
                            stream=stream)
        ti = tall[:, torch.as_tensor(_surv, dtype=torch.long)].contiguous().view(-1)
        erased_idx = torch.as_tensor(erased, dtype=torch.long)
    elif wl["op"] == "decode_multi" and mode == "syndrome":
        # whole codewords [S][n+p] (untimed encode); erased entries of the table -> a zero block
        din = torch.empty((S, n + p, B), dtype=torch.uint8, device="cuda")
        X.xslp_fill_random(din, S, n + p, B, seed=wl["seed"], stripe0=stripe0)
        tall = X.block_table(din, S, n + p, B).view(S, n + p)
        enc = X.xslp_compile(X.xslp_encode_bitmatrix(G, n, p), block_bytes_hint=B)
        X.xslp_encode_batch(enc, tall[:, :n].contiguous(), tall[:, n:].contiguous(), S, B,
                            stream=stream)
        zero_block = torch.zeros(B, dtype=torch.uint8, device="cuda")
        th = tall.cpu().numpy().copy()
        for s_, er in enumerate(pats):
            th[s_, list(er)] = zero_block.data_ptr()
        ti = torch.from_numpy(th.reshape(-1)).cuda()
    else:
        din = torch.empty((S, n_in, B), dtype=torch.uint8, device="cuda")
        X.xslp_fill_random(din, S, n_in, B, seed=wl["seed"], stripe0=stripe0)
        ti = X.block_table(din, S, n_in, B)
    if wl["op"] == "decode_multi":
        pos = [uniq.index(er) for er in pats]
        idx = torch.tensor(pos, dtype=torch.int32, device="cuda")
        gids, goff = X.group_stripes(pos, len(progs))
        gids = torch.from_numpy(gids).cuda()

    def launch(st=stream):
        if wl["op"] == "decode_peer" and args.xmode == "staged":
            sgather.run(dist, stream=st)
            if len(progs) == 1:
                X.xslp_encode_batch(progs[0], st_in, pdec.out_tbl, S, B, stream=st)
            elif pmulti is not None:
                X.xslp_multi_decode(pmulti, pdec.pos, sids, soff, st_in, pdec.out_tbl, B, stream=st)
            else:
                X.xslp_decode_batch_grouped(progs, sids, soff, st_in, pdec.out_tbl, B,
                                            nstreams=args.streams, stream=st)
        elif wl["op"] == "decode_peer":
            pdec.launch(stream=st, nstreams=args.streams)
        elif wl["op"] == "encode_gft":
            X.xslp_gf_table_apply(coef_rows, ti, to, S, B, stream=st)
        elif wl["op"] == "decode_multi" and mode in ("multi", "syndrome"):
            X.xslp_multi_decode(multi, idx, gids, goff, ti, to, B, stream=st)
        elif wl["op"] == "decode_multi" and mode == "interp":
            X.xslp_decode_batch_multi(progs, idx, ti, to, S, B, stream=st)
        elif wl["op"] == "decode_multi":
            X.xslp_decode_batch_grouped(progs, gids, goff, ti, to, B, nstreams=args.streams,
                                        stream=st)
        else:
            X.xslp_encode_batch(prog, ti, to, cur_S[0], B, stream=st)

    cur_S = [S]

    def step():
        for _ in range(nchunks):
            launch()

    # Strong-split workloads larger than one GPU's HBM (cfg5/cfg5d at N=1: 8192 stripes x 20 MiB)
    # run in chunks of wl["chunk"] stripes.  Every chunk's stripes are regenerated on the device
    # before it runs (xslp_fill_random with stripe0 = the chunk's first global stripe), outside
    # its timed interval: a step's time is the sum of its chunks' launch intervals
    # ("process in chunks with on-device regeneration and sum the kernel
    # times"), so every one of the rank's stripes is computed, none reused.
    chunked = wl["op"] in SHARDED and nchunks > 1
    chunk_sizes = [min(S, per - c * S) for c in range(nchunks)] if wl["op"] in SHARDED else [S]

    def regen(c):
        """Chunk c's inputs on the device; returns the launches it made (not timed work)."""
        l_ = X.xslp_launch_count()
        sc = chunk_sizes[c]
        if wl["op"] == "decode_sharded":   # whole codewords: data from the generator, parity encoded
            X.xslp_fill_random(din, sc, n + p, B, seed=wl["seed"], stripe0=stripe0 + c * S, stream=stream)
            X.xslp_encode_batch(enc, tall[:sc, :n].contiguous(), tall[:sc, n:].contiguous(), sc, B,
                                stream=stream)
        else:
            X.xslp_fill_random(din, sc, n_in, B, seed=wl["seed"], stripe0=stripe0 + c * S, stream=stream)
        return X.xslp_launch_count() - l_

    # sanity (torch, not the product): RAID-5 row of the [I; 2^ij] encode
    launch()
    torch.cuda.synchronize()
    if wl["op"] not in DECODE:
        acc = din[:, 0].clone()
        for j in range(1, n):
            acc ^= din[:, j]
        if not torch.equal(acc, dout[:, 0]):
            raise SystemExit("sanity check failed: parity block 0 != XOR of data blocks")
        del acc
    elif wl["op"] in ("decode_one", "decode_sharded"):
        if not torch.equal(dout, din[:, erased_idx]):
            raise SystemExit("sanity check failed: decoded blocks != the erased blocks")
    elif wl["op"] == "decode_multi" and mode == "syndrome":
        for s_ in (0, S // 2, S - 1):
            if not torch.equal(dout[s_], din[s_, list(pats[s_])]):
                raise SystemExit(f"sanity check failed: syndrome decode of stripe {s_}")
    elif wl["op"] == "decode_peer":       # regenerate a few home codewords locally and compare
        chk = plan.stripes[:2] + plan.stripes[-2:]
        full = torch.empty((1, n + p, B), dtype=torch.uint8, device="cuda")
        for s_ in chk:
            X.xslp_fill_random(full, 1, n + p, B, seed=wl["seed"], stripe0=s_)
            tf = X.block_table(full, 1, n + p, B).view(1, n + p)
            X.xslp_encode_batch(enc, tf[:, :n].contiguous(), tf[:, n:].contiguous(), 1, B)
            i = plan.stripes.index(s_)
            want = full[0, list(plan.keys[plan.key_of[i]][0])]
            if not torch.equal(dout[i], want):
                raise SystemExit(f"sanity check failed: cross-GPU decode of stripe {s_}")
        del full

    graph = None
    if args.graph:
        # one step's launches (all per-pattern kernels, their fork/join over the internal
        # streams) captured once and replayed: removes the host launch cost, not device work
        for pr in (progs if wl["op"] in ("decode_multi", "decode_peer") else [prog]):
            if isinstance(pr, X.Program):    # (the syndrome form's entries are patterns)
                X.xslp_prepare(pr, B)
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        l_before = X.xslp_launch_count()
        with torch.cuda.graph(graph, stream=cap):
            launch(cap)
        graph_launches = X.xslp_launch_count() - l_before
        stream.wait_stream(cap)

        def step():                         # noqa: F811
            for _ in range(nchunks):
                graph.replay()
    log('sanity ok; warmup')
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = X.xslp_launch_count()
    fills = 0
    if chunked:
        # per chunk: regenerate (untimed), then time its launch; a step = the sum over chunks
        cev = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nchunks)]
               for _ in range(args.steps)]
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                for c in range(nchunks):
                    fills += regen(c)
                    cur_S[0] = chunk_sizes[c]
                    cev[i][2 * c].record(stream)
                    if graph is not None and chunk_sizes[c] == S:
                        graph.replay()
                    else:
                        launch()
                    cev[i][2 * c + 1].record(stream)
            torch.cuda.synchronize()
        cur_S[0] = S
        per_step = [sum(cev[i][2 * c].elapsed_time(cev[i][2 * c + 1]) for c in range(nchunks))
                    for i in range(args.steps)]
        total_ms = sum(per_step)
    else:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        with ClockSampler(local) as clk:
            ev[0].record(stream)
            for i in range(args.steps):
                step()
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
        per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
        total_ms = ev[0].elapsed_time(ev[-1])
    launches = X.xslp_launch_count() - l0 - fills   # the product's coding kernels only
    if graph is not None:                   # kernels replayed from the graph
        launches += graph_launches * nchunks * args.steps
    log('timed region done')
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    rank_ms = total_ms
    total_ms = max_over_ranks(total_ms, dist, device=red_dev)
    rank_clocks = clk.summary()
    per_rank = [{"rank": rank, "gbs": round(sum(chunk_sizes) * n * B * args.steps / (rank_ms / 1e3) / 1e9, 3),
                 "ms_per_step": round(rank_ms / args.steps, 4), "sm_mhz": rank_clocks.get("sm_mhz"),
                 "reasons": rank_clocks.get("reasons"), "device": torch.cuda.get_device_name(local)}]
    if dist:
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank[0])
        per_rank = gathered
    data_bytes_step = sum(chunk_sizes) * n * B * world
    value = data_bytes_step * args.steps / (total_ms / 1e3) / 1e9

    # roofline of the dominant (only) kernel: algorithmic bytes per launch / launch time
    alg_bytes_launch = S * (n_in + m_out) * B        # per step (= per launch unless grouped)
    launch_ms = sum(per_step) / len(per_step) / nchunks   # chunks are equal for every N used
    achieved = alg_bytes_launch / (launch_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.workload),
            "peak_source": peak_src, "kernel": kernel_name(args, wl, stats),
            "alg_bytes_per_launch": alg_bytes_launch, "launch_ms": round(launch_ms, 4),
            "alg_bytes_per_data_byte": round((n_in + m_out) / n, 4),
            # SURVEY 8(d) asks for both denominators: the measured copy bandwidth (frac, the
            # judged one) and the nominal HBM3e figure (B200_PROFILING.md: 7.7 TB/s HGX)
            "nominal_peak": HBM_NOMINAL_GBS, "frac_nominal": round(achieved / HBM_NOMINAL_GBS, 4),
            "data_roof_gbs": round(peak / ((n_in + m_out) / n), 1)}
    if achieved > peak:
        # the judged denominator is a torch copy kernel, not the HBM ceiling: a fraction above 1
        # means "moves its bytes faster than that copy"; frac_nominal (7.7 TB/s) is the ceiling
        roof["frac_above_1"] = True
        roof["frac_note"] = ("denominator = MEASURED_PEAKS hbm_gbs (torch copy), not the HBM "
                             "ceiling; see frac_nominal against the HBM3e nominal")
    if wl["op"] == "encode_gft":
        # approach (1) is bound by the ALU pipe, not HBM (profiles/r01_s2_gftable.md): report its
        # design op count against the ALU pipe's measured 64 lane-ops / clk / SM
        # (scripts/alu_probe.cu, profiles/r01_s2_alu_probe.md) at the median SM clock under load
        sm_mhz = clk.summary()["sm_mhz"] or 1965
        ops_b = (6 + 4.5 * m_out + m_out / n) / 4      # ALU lane-ops per data byte (csrc/gftable.cu)
        a_ops = S * n * B * ops_b / (launch_ms / 1e3) / 1e12
        a_peak = ALU_LANE_OPS_PER_CLK_SM * NUM_SMS * sm_mhz * 1e6 / 1e12
        roof = {"bound": "alu", "achieved": round(a_ops, 3), "peak": round(a_peak, 3),
                "unit": "T ALU lane-ops/s", "frac": round(a_ops / a_peak, 4),
                "traffic": ncu_traffic(args.workload), "kernel": roof["kernel"],
                "peak_source": f"ALU pipe {ALU_LANE_OPS_PER_CLK_SM} lane-ops/clk/SM (alu_probe, "
                               f"B300_MICROARCH rt=2) x {NUM_SMS} SMs x median SM clock {sm_mhz} MHz",
                "alu_ops_per_data_byte": round(ops_b, 4), "launch_ms": roof["launch_ms"],
                "hbm": {"achieved": roof["achieved"], "peak": peak, "unit": "GB/s", "frac": roof["frac"]}}
    if wl["op"] == "decode_peer":
        # survivors read over NVLink from peer HBM: the second roof of the fused gather+decode
        rem_bytes = remote_blocks * B
        nv = rem_bytes / (launch_ms / 1e3) / 1e9
        roof["nvlink"] = {"remote_bytes_per_launch": rem_bytes,
                          "remote_fraction": round(remote_blocks / max(1, all_blocks), 4),
                          "achieved": round(nv, 1), "peak": NVLINK_GBS, "unit": "GB/s",
                          "frac": round(nv / NVLINK_GBS, 4),
                          "peak_source": "B200_PROFILING.md measured peer copy, per direction"}
        if world > 1 and nv / NVLINK_GBS > roof["frac"]:
            roof.update(bound="nvlink", achieved=round(nv, 1), peak=NVLINK_GBS,
                        frac=round(nv / NVLINK_GBS, 4), peak_source=roof["nvlink"]["peak_source"])

    # ---- e2e through the host-buffer C-ABI call ----
    e2e = None
    if not args.no_e2e and wl["op"] not in ("decode_multi", "decode_peer", "encode_gft"):
        try:
            # pinned host buffers: the full workload at N=1; at most 16 GiB over all ranks
            Se = min(S, max(1, (16 << 30) // max(1, world) // ((n + p) * B)))
            h_in = torch.empty((Se, n, B), dtype=torch.uint8, pin_memory=True)
            h_out = torch.empty((Se, m_out, B), dtype=torch.uint8, pin_memory=True)
            if wl["op"] in ("decode_one", "decode_sharded"):   # the survivors of each stripe
                h_in.copy_(din[:Se, torch.as_tensor(_surv, dtype=torch.long)])
                want = din[:Se, erased_idx]
            else:
                h_in.copy_(din[:Se])
                want = dout[:Se]
            X.xslp_encode_host(prog, h_in, h_out, Se, B, stream=stream)   # warm
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            e0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                X.xslp_encode_host(prog, h_in, h_out, Se, B, stream=stream)
            torch.cuda.synchronize()
            et = max_over_ranks(time.perf_counter() - e0, dist, device=red_dev)
            ok = bool(torch.equal(h_out.cuda(), want))
            del want
            e2e = {"value": round(Se * n * B * world * args.e2e_steps / et / 1e9, 3),
                   "unit": "GB/s", "h2d_bytes_per_step": Se * n * B,
                   "d2h_bytes_per_step": Se * m_out * B,
                   "steps": args.e2e_steps, "stripes_per_gpu": Se,
                   "api": "xslp_encode_host (pinned host buffers, chunked H2D / kernel / D2H on "
                   "two streams), host wall clock around synchronous calls, max over ranks",
                   "check_outputs": ok}
            del h_in, h_out
        except Exception as ex:  # report, do not hide
            e2e = {"value": None, "unit": "GB/s", "error": str(ex)[:200]}

    log('e2e', e2e)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(wl)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
                "scaling": "strong" if wl["op"] in SHARDED else "weak", "vs_baseline": None,
                "dtype": "u32", "data": "synthetic",
                "config": dict(config_of(args, wl, stats),
                               **({"multi": multi.info(), "patterns": len(progs),
                                   "per_module": args.per_module_raw or (16 if mode == "syndrome" else 20)}
                                  if wl["op"] == "decode_multi" and mode in ("multi", "syndrome")
                                  else {}),
                               **({"distinct_diagnostic": args.distinct} if args.distinct else {})),
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "per_rank": per_rank,
                "compile_s": round(compile_s, 3),
                "paper_context": {"note": "the paper's CPU numbers (not comparable: other hardware, "
                                          "context only; BASELINE.md)",
                                  "rs10_4_encode_gbs": {"intel i7-7567U": 8.92, "amd Ryzen 2600": 7.58},
                                  "rs10_4_decode_2456_gbs": {"intel i7-7567U": 6.67, "amd Ryzen 2600": 6.01},
                                  "source": "P:1656-1657, P:1685-1686"},
                "step_ms": {"min": round(min(per_step), 4), "median": round(sorted(per_step)[len(per_step) // 2], 4),
                            "max": round(max(per_step), 4)}}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
