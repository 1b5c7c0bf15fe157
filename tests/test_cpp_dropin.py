"""The C++ drop-in headers (include/kernelweave/*.hpp) compiled with g++ against libkw_b200.so
and run: host-only checks on CPU, the test_kernels.cpp analogues on the GPU."""
import subprocess

import pytest

from paper_1602_08477_b200 import build as B


@pytest.fixture(scope="module")
def programs():
    return {p.name: p for p in B.build_cpp_tests()}


def run(exe):
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    return p


def test_dropin_host_logic(programs):
    p = run(programs["test_dropin_host"])
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout


@pytest.mark.gpu
def test_dropin_gpu_kernels(programs):
    p = run(programs["test_dropin_gpu"])
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout


@pytest.mark.gpu
def test_generic_device_functors(programs):
    """kernelweave/cuda_exec.cuh: user functors (coverage, shared memory, atomics, the README
    functor) through createExec/executeTask on the GPU."""
    p = run(programs["test_functor_gpu"])
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout
