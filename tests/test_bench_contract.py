"""bench.py's driver contract, checked on the CPU: the reference arm (the oracle timed on the
host cores, `--impl reference`) prints the JSON line the driver parses, alone on rank 0 under
torchrun; the workload table is consistent; the product arm fails loudly without a GPU
instead of falling back to anything.  On a GPU (`-m gpu`): the default line's full contract."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, timeout=300, env=None):
    e = dict(os.environ)
    e.pop("RANK", None)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=e)


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _check_line(d, steps, warmup):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["steps"] == steps and d["warmup"] == warmup
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["scaling"] in ("weak", "strong")
    assert d["vs_baseline"] is None
    assert d["config"]["workload"].startswith("cfg2")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_prints_one_contract_line():
    r = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check_line(lines[0], 2, 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_reference_arm_under_torchrun_rank0_only():
    # the driver's N>1 launch: rank 0 alone runs the oracle and prints; the others exit 0
    r = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
              "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"], timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check_line(lines[0], 1, 1)
    assert lines[0]["n_gpus"] == 2


def test_workload_table():
    import bench
    ap_dests = {a.dest for a in bench_parser_actions(bench)}
    for name, wl in bench.WORKLOADS.items():
        for k in ("desc", "n", "p", "B", "S", "op"):
            assert k in wl, (name, k)
        assert wl["B"] % 128 == 0 and wl["S"] >= 1 and 1 <= wl["p"] and wl["n"] + wl["p"] <= 255
        for k in wl.get("tuned", {}):
            assert k in ap_dests, (name, k)   # a tuned default must be a bench flag
        for kern, t in wl.get("alt", {}).items():
            assert all(k in ap_dests for k in t), (name, kern)
    # the default line is BASELINE configs[1]: RS(10,4) encode, 1024 stripes x 10 x 1 MiB
    d = bench.WORKLOADS["cfg2"]
    assert (d["n"], d["p"], d["B"], d["S"], d["op"]) == (10, 4, 1 << 20, 1024, "encode")


def bench_parser_actions(bench):
    import argparse
    captured = {}
    orig = argparse.ArgumentParser.parse_args

    def grab(self, *a, **k):
        captured["p"] = self
        return orig(self, [])
    argparse.ArgumentParser.parse_args = grab
    try:
        bench.parse()
    finally:
        argparse.ArgumentParser.parse_args = orig
    return captured["p"]._actions


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure")
def test_product_arm_fails_loudly_without_gpu():
    r = _run([sys.executable, "bench.py", "--steps", "1", "--warmup", "0"], timeout=300)
    assert r.returncode != 0
    assert not _json_lines(r.stdout)   # no number printed from a fallback


@pytest.mark.gpu
def test_product_arm_json_contract_on_gpu():
    # the default line's full contract: metric / value / roofline (bound, achieved, peak, unit,
    # frac, traffic), cpu_baseline, e2e with the copied bytes, clocks, gpu_launches
    r = _run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3"], timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"].startswith("cfg2") and "l2" in d["config"]
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s" and ro["peak"] > 0
    assert abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-3
    assert ro["traffic"] is None or ro["traffic"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "GB/s"
    assert e["h2d_bytes_per_step"] == 1024 * 10 * (1 << 20)
    assert e["d2h_bytes_per_step"] == 1024 * 4 * (1 << 20)
    assert d["gpu_launches"] >= 3
    c = d["clocks"]
    assert c["sm_mhz"] and c["sm_max_mhz"] and isinstance(c["reasons"], list)


def test_gpus_flag_starts_the_ranks_without_torchrun():
    # `bench.py --gpus N` alone launches N ranks itself (one process per GPU); the line says
    # n_gpus N because N ranks ran (--gpus must be authoritative)
    r = _run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
              "--warmup", "1"], timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check_line(lines[0], 1, 1)
    assert lines[0]["n_gpus"] == 2


def test_gpus_flag_disagreeing_with_world_size_fails():
    r = _run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
              "--warmup", "1"], env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode != 0
    assert not _json_lines(r.stdout)
    assert "WORLD_SIZE" in r.stderr


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure")
def test_product_arm_multi_rank_fails_loudly_without_gpu():
    r = _run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0"], timeout=600)
    assert r.returncode != 0
    assert not _json_lines(r.stdout)
