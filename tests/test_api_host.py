"""Host-side API of the drop-in (no GPU): config validation, pivot strategy,
trace CSV layout, permutation replay, the reference sketch contract, problem
generators."""

import io

import numpy as np
import pytest

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import problems
from paper_2502_02721_b200.hessenberg import _full_permutation
from oracle import hessketch_oracle as ho


def test_config_defaults_and_validation():
    # solvers.py:88-116 (reference test_solvers.py:41-52)
    cfg = hs.SolverConfig()
    assert cfg.maxiter == 30
    assert cfg.effective_sketch_rows() == 310
    assert hs.SolverConfig(maxiter=5).effective_sketch_rows() == 60
    assert hs.SolverConfig(sketch_rows=99).effective_sketch_rows() == 99
    for bad in (dict(maxiter=0), dict(lam=-1.0), dict(sketch_rows=0), dict(dtype="float16"),
                dict(basis_dtype="int8"), dict(sketch_kind="srht")):
        with pytest.raises(ValueError):
            hs.SolverConfig(**bad)


def test_pivot_strategy_validation():
    with pytest.raises(ValueError):
        hs.PivotStrategy("partial")
    with pytest.raises(ValueError):
        hs.PivotStrategy.sampled(0)
    assert hs.PivotStrategy.full().kind == "full"


def test_trace_csv_layout():
    tr = hs.SolverTrace([hs.TraceRecord(iteration=1, sres_norm=0.5, proj_obj=0.5, matvecs=1, sketches=2, wall_ms=1.0),
                         hs.TraceRecord(iteration=2, sres_norm=0.25, proj_obj=0.25, rel_err=0.1, matvecs=2, sketches=3)])
    buf = io.StringIO()
    hs.trace_to_csv(tr, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ",".join(hs.CSV_COLUMNS)
    assert lines[1] == "1,,0.5,0.5,,,,,1,0,0,2,"
    assert lines[2].startswith("2,,0.25,0.25,0.1,")
    buf = io.StringIO()
    hs.trace_to_csv(tr, buf, include_timing=True)
    assert buf.getvalue().splitlines()[1].endswith(",1.0")


def test_permutation_replay_matches_reference_swaps():
    rng = np.random.default_rng(0)
    n = 50
    piv = list(rng.permutation(n)[:20])
    perm = np.arange(n)
    for k, idx in enumerate(piv):
        ho._swap_to_position(perm, k, idx)
    np.testing.assert_array_equal(_full_permutation(n, piv), perm)


def test_make_gaussian_sketch_is_reference_bitwise(golden):
    g = golden("scmrh_dense")
    np.testing.assert_array_equal(hs.make_gaussian_sketch(130, 40, 5).entries, g["S2"])
    g = golden("slslu_dense")
    np.testing.assert_array_equal(hs.make_gaussian_sketch(100, 25, hs.derive_seed(3, 1)).entries, g["S1_tik"])


def test_problem_generators():
    A = problems.toeplitz_blur_1d(64)
    np.testing.assert_allclose(A.sum(axis=1), 1.0)
    assert np.all(np.argmax(A, axis=1) == np.arange(64))  # Toeplitz Gaussian peaks on the diagonal
    x = problems.bumps_and_step(256, 3)
    assert x.shape == (256,) and np.all(np.isfinite(x))
    img = problems.rectangles_and_discs(32, 20, 1)
    assert img.shape == (32, 32) and img.max() > 0
    e = problems.random_ellipses(64, 10, 2)
    assert e.shape == (64, 64) and e.max() > 0
    p = problems.piecewise_constant(64, 3)
    assert p.shape == (64, 64)
    b, noise = problems.add_noise(np.ones(100), 0.01, 0)
    assert abs(np.linalg.norm(noise) / 10.0 - 0.01) < 1e-15
    np.testing.assert_array_equal(problems.gaussian_psf(2.0, radius=7), ho_psf(2.0, 7))


def ho_psf(sigma, radius):
    from oracle import tomo_oracle

    return tomo_oracle.gaussian_psf(sigma, radius)


def test_python_callable_operator_has_no_device_path():
    A = hs.LinearOperator(3, 3, lambda x: 2 * x, lambda y: 2 * y)
    assert np.allclose(A.apply(np.ones(3)), 2.0)
    assert A.counters.matvec_count == 1
    with pytest.raises(TypeError):
        hs.to_device_operator(A)
    with pytest.raises(ValueError):
        A.apply(np.ones(4))


def test_bench_workload_names_match_configs():
    """bench.py's reference arm names its workload without importing the device
    package; the strings must stay those of problems.CONFIGS."""
    import bench
    from paper_2502_02721_b200.problems import CONFIGS

    assert bench.WORKLOADS == CONFIGS
