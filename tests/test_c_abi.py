"""The C ABI from a plain C program (tests/c/abi_consumer.c): compiled with gcc against
include/xslp.h and linked to the in-tree libxslp.so, no Python in the loop."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2108_02692_b200")
SRC = os.path.join(ROOT, "tests", "c", "abi_consumer.c")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path, cuda):
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    exe = str(tmp_path / ("abi_gpu" if cuda else "abi_host"))
    cmd = ["gcc", "-std=c11", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
           "-o", exe, "-L", LIBDIR, "-lxslp", "-Wl,-rpath," + LIBDIR]
    if cuda:
        cmd += ["-DXSLP_WITH_CUDA", "-I", os.path.join(CUDA, "include"), "-L",
                os.path.join(CUDA, "lib64"), "-lcudart", "-Wl,-rpath," + os.path.join(CUDA, "lib64")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_consumer_host_calls(tmp_path):
    exe = _build(tmp_path, cuda=False)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("ok host"), r.stdout + r.stderr


def test_c_consumer_no_device_fails_loudly(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    exe = _build(tmp_path, cuda=False)
    r = subprocess.run([exe, "nodevice"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok nodevice" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_consumer_encode_decode_on_gpu(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path, cuda=True)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok gpu" in r.stdout, r.stdout + r.stderr
