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
def test_dropin_gpu_kernels(programs, tmp_path, monkeypatch):
    """The C++ drop-in's GPU cases; its matrix CSV writer must produce exactly the text the
    reference's own readBufferCsv/writeBufferCsv (oracle/_ref) reproduces byte for byte."""
    csv_path = tmp_path / "m.csv"
    monkeypatch.setenv("KW_CSV_OUT", str(csv_path))
    p = run(programs["test_dropin_gpu"])
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout
    from oracle import oracle as O
    if O.ref_available():
        assert O.ref().kwref_buffer_csv_roundtrip(str(csv_path).encode()) == 35, O.ref().kwref_last_error()


@pytest.mark.gpu
def test_generic_device_functors(programs):
    """kernelweave/cuda_exec.cuh: user functors (coverage, shared memory, atomics, the README
    functor) through createExec/executeTask on the GPU."""
    p = run(programs["test_functor_gpu"])
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout


def test_kwbench_usage_errors_exit_2(programs):
    """tools/bench/main.cpp exit-code contract: 2 for usage errors (acceptance crit. 11)."""
    for argv in (["--kernel", "foo"], ["--reps", "2"], ["--sizes", "0"], ["--backend", "blocks"],
                 ["--kernel", "axpy", "--pessimize"], ["--bogus"], ["--baseline", "serial"]):
        p = subprocess.run([str(programs["kwbench"]), *argv], capture_output=True, text=True, timeout=60)
        assert p.returncode == 2, (argv, p.stdout, p.stderr)


@pytest.mark.gpu
def test_kwbench_gpu_csv_and_verification(programs, tmp_path):
    """kwbench on the GPU: verified runs exit 0 with the reference's CSV schema; fault
    injection (KWBENCH_INJECT_FAULT) makes verification fail with exit code 1."""
    import csv
    import os
    exe = str(programs["kwbench"])
    for argv, rows in ((["--kernel", "axpy", "--dtype", "f32", "--sizes", "1000003,4096"], 6),
                       (["--kernel", "axpy", "--sizes", "4099"], 3),
                       (["--kernel", "gemm-naive", "--sizes", "64,100", "--tpb", "4", "--ept", "4"], 6),
                       (["--kernel", "gemm-tiled", "--sizes", "256,300", "--tile", "128", "--pessimize"], 12)):
        out = tmp_path / "r.csv"
        p = subprocess.run([exe, *argv, "--reps", "3", "--verify", "--csv", str(out)], capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, (argv, p.stdout, p.stderr)
        recs = list(csv.DictReader(out.open()))
        assert list(recs[0].keys()) == ["kernel", "backend", "n", "b", "v", "tile", "rep", "seconds", "gflops",
                                        "verified"]
        assert len(recs) == rows and all(r["verified"] == "1" and r["backend"] == "gpu" for r in recs)
        from oracle import oracle as O
        if O.ref_available():  # the reference's own readRecordsCsv/writeRecordsCsv: byte round-trip
            assert O.ref().kwref_csv_roundtrip(str(out).encode()) == rows
    env = dict(os.environ, KWBENCH_INJECT_FAULT="1")
    p = subprocess.run([exe, "--kernel", "axpy", "--sizes", "1000", "--reps", "3", "--verify"], capture_output=True,
                       text=True, timeout=120, env=env)
    assert p.returncode == 1, p.stdout


@pytest.mark.gpu
def test_kwbench_native_backend_and_baseline_report(programs, tmp_path):
    """--backend native|all and --baseline (runner.cpp:238-328): the native back-end (plain CUDA
    kernels, no library API) is verified bitwise like the library's, is benchmarked when only
    named as the baseline, and every median is reported relative to the baseline."""
    import csv
    exe = str(programs["kwbench"])
    for argv, backends in ((["--kernel", "axpy", "--sizes", "1000003", "--backend", "all", "--baseline", "native"],
                            {"gpu", "native"}),
                           (["--kernel", "axpy", "--dtype", "f32", "--sizes", "4099", "--backend", "native"],
                            {"native"}),
                           (["--kernel", "gemm-naive", "--sizes", "100", "--backend", "native", "--baseline", "gpu"],
                            {"gpu", "native"}),
                           (["--kernel", "gemm-tiled", "--sizes", "200", "--backend", "all", "--baseline", "native"],
                            {"gpu", "native"})):
        out = tmp_path / "r.csv"
        p = subprocess.run([exe, *argv, "--reps", "3", "--verify", "--csv", str(out)], capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, (argv, p.stdout, p.stderr)
        recs = list(csv.DictReader(out.open()))
        assert {r["backend"] for r in recs} == backends, argv
        assert len(recs) == 3 * len(backends) and all(r["verified"] == "1" for r in recs), argv
        from oracle import oracle as O
        if O.ref_available():  # native rows still parse and re-serialise byte for byte in the reference
            assert O.ref().kwref_csv_roundtrip(str(out).encode()) == len(recs), argv
        if "--baseline" in argv:
            base = argv[argv.index("--baseline") + 1]
            assert f"median time relative to {base}:" in p.stdout
            assert f" {base} n=" in p.stdout.split("relative to")[1] and "1.000x" in p.stdout


@pytest.mark.gpu
def test_criterion10_pessimization_analogue(programs, tmp_path):
    """acceptance.cpp:616-650 on the GPU: kwbench --pessimize runs gemm-tiled at n = 512 both
    tuned and degraded (the naive one-thread kernel in place of the tiled one); the degraded
    median must be at least 2x slower."""
    import csv
    import statistics
    out = tmp_path / "p.csv"
    p = subprocess.run([str(programs["kwbench"]), "--kernel", "gemm-tiled", "--sizes", "512", "--tile", "128",
                        "--reps", "3", "--pessimize", "--csv", str(out)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.stdout, p.stderr)
    recs = list(csv.DictReader(out.open()))
    tuned = [float(r["seconds"]) for r in recs if r["tile"] == "128"]
    degraded = [float(r["seconds"]) for r in recs if r["tile"] == "1"]
    assert tuned and degraded
    assert statistics.median(degraded) / statistics.median(tuned) >= 2.0


@pytest.mark.gpu
def test_criterion08_zero_overhead_analogue(programs, tmp_path):
    """acceptance.cpp:546-585 on the GPU: the library back-end's median time over the native
    CUDA kernels' (kwbench --baseline native) is at most 1.5x for AXPY at n = 2^20 and for the
    naive GEMM at 256 and 512, each with a tuned division (the reference picks one per kernel)."""
    import csv
    import statistics
    exe = str(programs["kwbench"])
    for argv in (["--kernel", "axpy", "--sizes", "1048576"], ["--kernel", "gemm-naive", "--sizes", "256,512"]):
        out = tmp_path / "c08.csv"
        p = subprocess.run([exe, *argv, "--backend", "all", "--baseline", "native", "--reps", "21", "--csv", str(out)],
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, (argv, p.stdout, p.stderr)
        recs = list(csv.DictReader(out.open()))
        for n in {r["n"] for r in recs}:
            lib = statistics.median(float(r["seconds"]) for r in recs if r["n"] == n and r["backend"] == "gpu")
            nat = statistics.median(float(r["seconds"]) for r in recs if r["n"] == n and r["backend"] == "native")
            assert lib / nat <= 1.5, (argv, n, lib / nat)
