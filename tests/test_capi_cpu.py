"""CPU-only checks of the C-ABI library and host logic (no device compute).

* libtucksum_cuda.so loads and exports every function include/tucksum_cuda.h declares;
* the .so carries sm_100a code only (cuobjdump);
* host-only entry points (RNG) are bit-identical to the oracle / golden vectors;
* without a GPU the device entry points fail loudly (no CPU fallback);
* the Python mirror enforces the reference's request validation;
* the workload generators reproduce BASELINE.md's F_alg table.
"""
import json
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

import oracle as O
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import f_alg, make_workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tucksum_cuda.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = T.lib()
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(T.EXPORTED_SYMBOLS)


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="cuobjdump missing")
def test_library_is_sm100a_with_dmma():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)
    sass = subprocess.run([exe, "-sass", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass


def test_host_rng_bitwise_matches_oracle_and_golden():
    with open(os.path.join(ROOT, "tests", "golden", "gaussian.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        got = T.gaussian_matrix(case["rows"], case["cols"], T.RngSeed(case["seed"], case["stream"]))
        assert got.ravel(order="F").tolist() == case["values"]
    for case in gold["substream"]:
        s = T.RngSeed(case["seed"], case["stream"]).substream(case["salt"])
        assert (s.seed, s.stream) == (case["out_seed"], case["out_stream"])
    a = T.gaussian_matrix(50, 7, T.RngSeed(5, 6))
    assert np.array_equal(a, O.gaussian_matrix(50, 7, (5, 6)))


def test_device_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(T.TucksumCudaError):
        T.Engine(0)


def test_mirror_request_validation():
    """test_sketch_sum.cpp:514-547 error contract, enforced before any device work."""
    a = T.TuckerTensor(np.ones((2, 2, 2)), [np.ones((8, 2)), np.ones((7, 2)), np.ones((6, 2))])
    b = T.TuckerTensor(np.ones((2, 2, 2)), [np.ones((8, 2)), np.ones((7, 2)), np.ones((5, 2))])
    with pytest.raises(ValueError):
        T.round_sum(T.SumRequest([], []))
    with pytest.raises(ValueError):
        T.round_sum(T.SumRequest([a], [1.0, 2.0], strategy=T.Strategy.Krp))
    with pytest.raises(ValueError):
        T.krp_sum(T.SumRequest([a, b], [1.0, 1.0], strategy=T.Strategy.Krp))
    with pytest.raises(ValueError):
        T.krp_sum(T.SumRequest([a, None], [1.0, 1.0], strategy=T.Strategy.Krp))
    with pytest.raises(ValueError):
        T.krp_sum(T.SumRequest([a], [1.0], eps=-1.0, strategy=T.Strategy.Krp))
    with pytest.raises(ValueError):
        T.TuckerTensor(np.ones((2, 2)), [np.ones((4, 3)), np.ones((4, 2))])
    assert T.strategy_from_name("krp") == T.Strategy.Krp
    with pytest.raises(ValueError):
        T.strategy_from_name("nope")


def test_formal_sum_layout():
    """tucker.cpp:183-226: stacked factors and weighted super-diagonal blocks."""
    x = T.TuckerTensor(np.arange(8.0).reshape((2, 2, 2), order="F"), [np.eye(4)[:, :2]] * 3)
    y = T.TuckerTensor(np.ones((1, 3, 2)), [np.ones((4, 1)), np.ones((4, 3)), np.ones((4, 2))])
    s = T.formal_sum([x, y], [2.0, -1.0])
    assert s.ranks == [3, 5, 4]
    assert [b.offsets for b in s.blocks] == [[0, 0, 0], [2, 2, 2]]
    assert np.array_equal(s.blocks[0].data, 2.0 * x.dense_core())
    assert np.array_equal(s.factors[1][:, 2:], y.factors[1])


def test_workload_falg_matches_baseline_table():
    """F_alg per call for configs 1-5."""
    want = {1: 2.855e6, 2: 220.4e6, 3: 1.243e9, 4: 390.0e6, 5: 88.05e9}
    specs = {1: ([64] * 3, [8] * 3, 4, 26), 2: ([512] * 3, [20] * 3, 16, 40), 3: ([4096, 64, 64], [30, 10, 10], 30, 50),
             4: ([256] * 4, [16] * 4, 8, 26), 5: ([8192] * 3, [32] * 3, 256, 64)}
    for cfg, (dims, r, K, s) in specs.items():
        assert abs(f_alg(dims, [r] * K, s) - want[cfg]) <= 1e-3 * want[cfg]


def test_workload_generator_small():
    wl = make_workload(1)
    assert wl.K == 4 and wl.widths == [26] * 3 and wl.cap == [16] * 3
    for x in wl.summands:
        for f in x.factors:
            assert np.linalg.norm(f.T @ f - np.eye(8)) <= 1e-13
    # Summand factors are views into the per-mode slabs (one H2D copy per mode).
    assert np.shares_memory(wl.summands[1].factors[0], wl.slabs[0])
    wl3 = make_workload(3, K=2)
    q = wl3.summands[0].factors[1]
    assert q.shape == (64, 10) and np.linalg.norm(q.T @ q - np.eye(10)) <= 1e-13


def test_cpp_host_caller_builds():
    """The C ABI is consumable from C++ with no Python: tests/cpp/capi_host.cpp
    compiles (-Wall -Wextra) and links against the in-tree library."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([os.path.join(root, "tests", "cpp", "build.sh")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "warning" not in r.stderr
    assert os.path.exists(os.path.join(root, "tests", "cpp", "capi_host"))


def test_kron_sketch_dims_host_rule_matches_oracle():
    """ts_kron_sketch_dims (host arithmetic behind the C ABI, no GPU needed) equals
    the oracle's restatement of src/sketch.cpp:222-270 on the reference's frozen
    cases (test_sketch_sum.cpp:159-184) and on 300 random instances."""
    import oracle as O

    assert T.kron_sketch_dims([4, 4, 4], [20, 20, 20]) == [2, 2, 2]
    assert T.kron_sketch_dims([10, 2, 2], [30, 30, 30]) == [1, 4, 4]
    assert T.kron_sketch_dims([3, 3, 3], [9, 9, 9]) == [2, 2, 2]
    assert T.kron_sketch_dims([2, 8, 8], [2, 10, 10]) == [2, 4, 4]
    for bad in (([5, 2, 2], [6, 2, 2]), ([2], [4]), ([0, 2], [4, 4])):
        with pytest.raises(ValueError):
            T.kron_sketch_dims(*bad)
    rng = np.random.default_rng(5)
    for _ in range(300):
        order = int(rng.integers(2, 6))
        dims = [int(x) for x in rng.integers(1, 40, size=order)]
        targets = [int(rng.integers(1, min(d, T.complement_product(dims, n)) + 1)) for n, d in enumerate(dims)]
        assert T.kron_sketch_dims(targets, dims) == O.kron_sketch_dims(targets, dims)


def test_kron_plan_report_lists_complement_widths():
    """test_sketch_sum.cpp:549-557."""
    plan = T.SketchPlan(T.Strategy.Kron, [2, 3, 2], [2, 2, 2], [4, 5, 4], [2, 2, 3], 1e-6, T.RngSeed(95, 0))
    text = plan.report()
    for key in ("kron", "mode 1:", "mode 3:", "sketch_dim=", "complement_width=6"):
        assert key in text


def test_every_strategy_fails_loudly_without_gpu():
    """No CPU fallback: each round_sum strategy goes to the device library."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = T.TuckerTensor(np.ones((2, 2, 2)), [np.ones((8, 2)), np.ones((7, 2)), np.ones((6, 2))])
    for strat in T.Strategy:
        with pytest.raises(T.TucksumCudaError):
            T.round_sum(T.SumRequest([x, x], [1.0, 2.0], strategy=strat))
    with pytest.raises(T.TucksumCudaError):
        T.tucker_norm(x)


REF_INCLUDE = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers absent (GPU box)")
def test_reference_adapter_compiles_against_reference_headers():
    """include/tucksum_cuda_adapter.hpp (krp_sum, kron_sum, round_sum over every
    strategy, tucker_rounding / norm / inner / rel_error) compiles with -Wall
    -Wextra -Werror against the REAL reference headers
    (/root/reference/proj/include/tucksum/*.hpp) and a minimal Eigen shim
    (tests/cpp/eigen_shim — Eigen is absent from the image), and each drop-in has
    exactly the reference entry point's function type."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        "-I", REF_INCLUDE, "-I", os.path.join(root, "tests", "cpp", "eigen_shim"),
                        "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "cpp", "adapter_compile_ref.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
