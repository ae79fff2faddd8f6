"""The drop-in boundary, checked without a GPU.

* libfsk_b200.so loads and exports every C symbol include/fsk_b200.h declares
  and the C++ entry points of include/fsk/*.hpp;
* host logic that runs before any device work: validation (reference
  messages and exception types), IO-ledger closed forms vs the reference's
  counters, the eps schedule, the seeded generator;
* the reference's own test_core suite compiled against the library (it never
  touches the device) fails exactly where the reference itself fails.
"""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_c_symbols():
    text = (ROOT / "include" / "fsk_b200.h").read_text()
    return sorted(set(re.findall(r"\b(fsk_[a-z0-9_]+)\s*\(", text)))


def exported_symbols(path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True,
                         text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_library_exports_every_declared_symbol(fsk):
    syms = exported_symbols(fsk.LIB_PATH)
    missing = [s for s in declared_c_symbols() if s not in syms]
    assert not missing, missing
    assert len(declared_c_symbols()) >= 40


def test_library_exports_cpp_dropin_api(fsk):
    out = subprocess.run(["nm", "-DC", "--defined-only", str(fsk.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    for name in ["fsk::stream::update_f_hat(", "fsk::stream::update_g_hat(",
                 "fsk::stream::symmetric_update(", "fsk::stream::apply_plan(",
                 "fsk::stream::apply_plan_adjoint(", "fsk::stream::apply_hadamard_plan(",
                 "fsk::stream::induced_marginals(", "fsk::stream::update_f_hat_f32(",
                 "fsk::stream::update_g_hat_f32(", "fsk::stream::io_count_f_update(",
                 "fsk::solver::sinkhorn_solve(", "fsk::solver::dual_cost(",
                 "fsk::solver::sinkhorn_divergence(", "fsk::solver::sinkhorn_divergence_mixed(",
                 "fsk::validate_problem(", "fsk::eps_schedule(", "fsk::autodiff::grad_source(",
                 "fsk::hvp::hvp_apply("]:
        assert name in out, name


def test_validation_errors_match_reference(fsk, ref):
    one = np.zeros((1, 1))
    w1 = np.ones(1)
    cases = [
        (lambda m: m.update_f_hat(one, w1, one, w1, [0.0], -1.0)),
        (lambda m: m.update_f_hat(one, w1, one, w1, [np.nan], 1.0)),
        (lambda m: m.update_f_hat(one, [0.5], one, w1, [0.0], 1.0)),
        (lambda m: m.update_f_hat(one, w1, np.zeros((1, 2)), w1, [0.0], 1.0)),
        (lambda m: m.update_f_hat(one, w1, one, w1, [0.0], 1.0, tiles=(0, 4))),
        (lambda m: m.apply_plan(one, w1, one, w1, [0.0], [0.0], -0.5, np.ones((1, 1)))),
        (lambda m: m.apply_plan(one, w1, one, w1, [0.0], [0.0], 0.5, np.full((1, 1), np.inf))),
        (lambda m: m.sinkhorn_solve(one, w1, one, w1, eps=0.0)),
        (lambda m: m.sinkhorn_solve(one, w1, one, w1, max_iters=0)),
        (lambda m: m.sinkhorn_solve(one, w1, one, w1, eps_scaling_factor=1.5)),
    ]
    for case in cases:
        with pytest.raises(Exception) as ours:
            case(fsk)
        with pytest.raises(Exception) as theirs:
            case(ref)
        assert type(ours.value).__name__ == "ValidationError" == type(theirs.value).__name__
        assert str(ours.value) == str(theirs.value)


def test_label_validation_messages(fsk, ref):
    a = np.array([[0.0], [1.0]])
    b = np.array([[2.0]])
    bad = dict(lambda1=0.5, lambda2=0.5, label_cost=np.zeros((2, 2)))
    for m in (fsk, ref):
        with pytest.raises(Exception) as e:
            m.update_f_hat(a, [0.5, 0.5], b, [1.0], [0.0], 0.3, cost=bad, la=[0, 1], lb=[2])
        assert str(e.value) == "target label 2 out of range of label cost table"


@pytest.mark.parametrize("case", [(64, 64, 64, 64, 8), (100, 64, 32, 16, 8), (57, 31, 5, 7, 3),
                                  (1, 10, 1, 3, 2), (128, 100, 64, 100, 16), (45, 33, 8, 16, 5)])
def test_io_count_closed_forms_match_reference_ledger(fsk, case):
    """test_stream.cpp:350-414 (closed forms) - values from stream.cpp:459-499."""
    n, m, bn, bm, d = case
    t = (bn, bm)
    bn_ = min(bn, n)
    bm_ = min(bm, m)
    assert fsk.io_count("f_update", n, m, d, tiles=t) == n * d + -(-n // bn_) * m * (d + 2) + n
    assert fsk.io_count("g_update", n, m, d, tiles=t) == m * d + -(-m // bm_) * n * (d + 2) + m
    p, r = 4, 3
    assert fsk.io_count("apply_plan", n, m, d, p, tiles=t) == \
        n * (d + 2) + -(-n // bn_) * m * (d + 2 + p) + n * p
    assert fsk.io_count("apply_hadamard", n, m, d, r, p, tiles=t) == \
        n * (d + 2 + r) + -(-n // bn_) * m * (d + 2 + r + p) + n * p
    assert fsk.io_count("symmetric_update", n, m, d, tiles=t) == \
        fsk.io_count("f_update", n, m, d, tiles=t) + fsk.io_count("g_update", n, m, d, tiles=t) + n + m


def test_tiles_fit_sram(fsk):
    assert fsk.tiles_fit_sram((16, 16), 4, 16 * 4 + 16 * 4 + 16 + 32)
    assert not fsk.tiles_fit_sram((16, 16), 4, 100)


def test_product_rng_is_bit_identical_to_reference_generator(fsk, golden):
    x = fsk.rng_normal(1000, 4096 * 3 * 2)
    assert np.array_equal(x[: 4096 * 3], golden["cfg1_X"].reshape(-1))
    assert np.array_equal(x[4096 * 3:], golden["cfg1_Y"].reshape(-1))


def test_reference_test_core_against_b200_library():
    """proj/tests/test_core.cpp compiled against include/fsk + libfsk_b200.so:
    the same two reference-side failures as the reference itself, nothing else."""
    exe = ROOT / "tests" / "refsuite" / "_bin" / "test_core_b200"
    if not exe.exists():
        pytest.skip("refsuite not built")
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    failed = sorted(set(l.split("FAILED: ")[1] for l in out.stderr.splitlines() if "FAILED: " in l))
    assert failed == ["eps schedule anneals from the diameter and truncates",
                      "shift then unshift is the identity on random input"]
    assert "11 |" in out.stdout


def test_compute_fails_loudly_without_device(fsk):
    """No CPU fallback: on a host without a CUDA device compute raises."""
    import ctypes
    if fsk.lib().fsk_device_count() > 0:
        pytest.skip("device present")
    with pytest.raises(fsk.DeviceError):
        fsk.update_f_hat(np.zeros((2, 1)), [0.5, 0.5], np.ones((2, 1)), [0.5, 0.5], [0.0, 0.0], 0.3)
    del ctypes
