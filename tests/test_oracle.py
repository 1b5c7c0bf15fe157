"""CPU: the oracle restatement (oracle/kw_oracle.c) pinned against the reference's golden
vectors (tests/golden/golden.json, made by oracle/gen_golden.py from the reference build) and,
where oracle/_ref is built, against the reference code itself on fresh seeded inputs."""
import numpy as np
import pytest


def h(v: int) -> str:
    return f"{v:016x}"


def test_generator_matches_reference_draws(oracle, golden):
    tag = int(oracle.lib().kw_kernel_tag(b"axpy"))
    assert h(tag) == golden["kernel_tag"]["axpy"]
    g = oracle.MT64(seeds=[42, 1 << 20, tag])
    assert [h(g()) for _ in range(16)] == golden["mt19937_64_seed_seq_42_2p20_axpy"]
    for k, v in golden["kernel_tag"].items():
        assert h(int(oracle.lib().kw_kernel_tag(k.encode()))) == v


@pytest.mark.parametrize("case", range(4))
def test_axpy_workload_digests(oracle, golden, case):
    c = golden["workloads"][case]
    assert c["kernel"] == "axpy"
    f32 = c["dtype"] == "f32"
    alpha, x, y = oracle.workload_axpy(c["n"], c["seed"], f32)
    assert float(alpha) == c["alpha"]
    assert h(oracle.fnv1a64(x)) == c["x_digest"]
    assert h(oracle.fnv1a64(y)) == c["y_in_digest"]
    out = oracle.axpy(alpha, x, y)
    assert h(oracle.fnv1a64(out)) == c["y_out_digest"]
    assert float(out[0]) == c["first"] and float(out[-1]) == c["last"]


@pytest.mark.parametrize("case", [4, 5])
def test_gemm_workload_digests(oracle, golden, case):
    c = golden["workloads"][case]
    alpha, beta, a, b, cin = oracle.workload_gemm(c["n"], c["seed"], "gemm-tiled")
    assert (alpha, beta) == (c["alpha"], c["beta"])
    assert h(oracle.fnv1a64(a)) == c["a_digest"] and h(oracle.fnv1a64(b)) == c["b_digest"]
    assert h(oracle.fnv1a64(cin)) == c["c_in_digest"]
    fast = oracle.gemm(alpha, beta, a, b, cin)
    lit = oracle.gemm(alpha, beta, a, b, cin, literal=True)
    assert h(oracle.fnv1a64(fast)) == c["c_out_digest"]
    assert np.array_equal(fast, lit)


def test_axpy_known_answers(oracle, golden):
    # test_kernels.cpp:73-86 closed forms.
    x = np.array([1.0, 2.0, 3.0])
    assert oracle.axpy(2.0, x, np.array([10.0, 20.0, 30.0])).tolist() == [12, 24, 36]
    assert oracle.axpy(0.0, x, np.array([10.0, 20.0, 30.0])).tolist() == [10, 20, 30]
    # tail canary (test_kernels.cpp:88-112)
    t = golden["axpy_tail_canary"]
    rng = oracle.MT64(seed=t["seed"])
    xs = rng.fill_uniform(t["covered"])
    ys = rng.fill_uniform(t["covered"])
    ys[t["n"]:] = -555.25
    out = ys.copy()
    out[: t["n"]] = oracle.axpy(t["alpha"], xs[: t["n"]], ys[: t["n"]])
    assert out.tolist() == t["y_out"]
    # native 4099 (test_kernels.cpp:331-349)
    c = golden["axpy_native_4099"]
    rng = oracle.MT64(seed=c["seed"])
    xs = rng.fill_uniform(c["n"])
    ys = rng.fill_uniform(c["n"])
    assert h(oracle.fnv1a64(oracle.axpy(c["alpha"], xs, ys))) == c["y_out_digest"]


def test_gemm_known_answers(oracle, golden):
    # test_kernels.cpp:114-170
    assert oracle.gemm(2.0, 10.0, np.array([[3.0]]), np.array([[5.0]]), np.array([[7.0]]))[0, 0] == 100.0
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    assert oracle.gemm(1.0, 0.0, a, b, np.zeros((2, 2))).tolist() == [[19, 22], [43, 50]]
    rng = oracle.MT64(seed=4321)
    cases = golden["gemm_ragged_rng4321"]
    s = 16
    mats = [rng.fill_uniform(s * s).reshape(s, s) for _ in range(3)]
    assert h(oracle.fnv1a64(oracle.gemm(2.0, 1.0, *mats))) == cases[0]["c_out_digest"]
    s = 10
    mats = [rng.fill_uniform(s * s).reshape(s, s) for _ in range(3)]
    assert h(oracle.fnv1a64(oracle.gemm(1.0, 0.5, *mats))) == cases[1]["c_out_digest"]
    m, n, k = 13, 29, 7
    a = rng.fill_uniform(m * k).reshape(m, k)
    b = rng.fill_uniform(k * n).reshape(k, n)
    c = rng.fill_uniform(m * n).reshape(m, n)
    assert h(oracle.fnv1a64(oracle.gemm(2.5, 0.0, a, b, c))) == cases[2]["c_out_digest"]


def test_oracle_fp32_has_no_fma_contraction(oracle):
    """22.4% of fp32 elements differ by 1 ulp under FMA; the oracle must round
    the product separately: compare against numpy's separately-rounded float32 ops."""
    alpha, x, y = oracle.workload_axpy(1 << 16, 7, True)
    want = (np.float32(alpha) * x).astype(np.float32) + y
    assert np.array_equal(oracle.axpy(alpha, x, y), want)


@pytest.mark.skipif(not __import__("oracle.oracle", fromlist=["x"]).ref_available(), reason="oracle/_ref not built")
def test_restatement_equals_reference_code_on_random_cases(oracle):
    """The C restatement vs the reference library itself (oracle/_ref), fresh seeded inputs."""
    import ctypes as C
    r = oracle.ref()
    rng = np.random.default_rng(101)
    for _ in range(20):
        n = int(rng.integers(1, 5000))
        for f32 in (True, False):
            al, be = C.c_double(), C.c_double()
            dt = np.float32 if f32 else np.float64
            x, y = np.empty(n, dt), np.empty(n, dt)
            seed = int(rng.integers(0, 2**63))
            assert r.kwref_workload(b"axpy", n, seed, int(f32), C.byref(al), C.byref(be), x.ctypes.data,
                                    y.ctypes.data, None) == 0
            a2, x2, y2 = oracle.workload_axpy(n, seed, f32)
            assert np.array_equal(x, x2) and np.array_equal(y, y2)
            out = y.copy()
            sec = C.c_double()
            a = float(np.float32(al.value)) if f32 else al.value
            assert r.kwref_axpy_kernel(1, int(f32), n, a, x.ctypes.data, out.ctypes.data, 16, 8, C.byref(sec)) == 0
            assert np.array_equal(out, oracle.axpy(a2, x2, y2))
    for _ in range(20):
        m, n, k = (int(v) for v in rng.integers(1, 70, size=3))
        a, b, c = rng.random((m, k)) * 10, rng.random((k, n)) * 10, rng.random((m, n)) * 10
        alpha, beta = float(rng.random() * 8), float(rng.integers(0, 3))
        want = c.copy()
        r.kwref_gemm_reference(m, n, k, alpha, beta, a.ctypes.data, k, b.ctypes.data, n, want.ctypes.data, n)
        assert np.array_equal(oracle.gemm(alpha, beta, a, b, c), want)
        assert np.array_equal(oracle.gemm(alpha, beta, a, b, c, literal=True), want)
