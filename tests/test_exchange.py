"""Problem builders, phantoms and the exchange formats (PGM images,
MatrixMarket arrays / operators) against fixtures written by the reference
(tests/golden/make_golden.py: gen_exchange).  Host-side; the device-operator
builders are checked in the gpu-marked tests at the end."""

import os

import numpy as np
import pytest

from paper_2502_02721_b200 import linops, problems


def test_phantoms_and_motion_psf_bitwise(golden):
    g = golden("exchange")
    np.testing.assert_array_equal(problems.deblur_phantom(37), g["deblur37"])
    np.testing.assert_array_equal(problems.deblur_phantom(8), g["deblur8"])
    np.testing.assert_array_equal(problems.tomography_phantom(29), g["tomo29"])
    for i in range(5):
        length, ang = g[f"motion{i}_args"]
        length = int(length) if float(length).is_integer() else float(length)
        np.testing.assert_array_equal(problems.motion_psf(length, float(ang)), g[f"motion{i}"])
    with pytest.raises(ValueError):
        problems.motion_psf(0, 10.0)
    with pytest.raises(ValueError):
        problems.motion_psf(3, float("nan"))


def test_pgm_write_bytes_and_read_errors(golden, tmp_path):
    g = golden("exchange")
    img = problems.Image(width=7, height=5, pixels=g["pgm_pixels"])
    path = tmp_path / "a.pgm"
    problems.write_image(img, path)
    assert path.read_bytes() == g["pgm_bytes"].tobytes()
    back = problems.read_image(path)
    np.testing.assert_array_equal(back.pixels, np.round(g["pgm_pixels"] * 65535.0) / 65535.0)
    for i, want in enumerate(g["pgm_msgs"]):
        fp = tmp_path / f"c{i}.pgm"
        fp.write_bytes(g[f"pgm_case{i}"].tobytes())
        if want == "ok":
            np.testing.assert_array_equal(problems.read_image(fp).pixels, g["pgm8_pixels"])
        else:
            with pytest.raises(problems.ImageFormatError) as ei:
                problems.read_image(fp)
            assert str(ei.value) == str(want)
    v = np.linspace(-0.5, 1.5, 12)
    im = problems.image_from_vector(v, 3, 4)
    assert im.pixels.min() == 0.0 and im.pixels.max() == 1.0
    with pytest.raises(ValueError):
        problems.Image(width=2, height=2, pixels=np.full((2, 2), 2.0))


def test_matrix_market_exchange(golden, tmp_path):
    g = golden("exchange")
    for name in ("mtx_mat", "mtx_vec"):
        fp = tmp_path / (name + ".mtx")
        linops.save_array(fp, g[name])
        assert fp.read_bytes() == g[name + "_bytes"].tobytes()
        back = linops.load_array(fp)
        np.testing.assert_array_equal(back, g[name])
        assert back.ndim == g[name].ndim
    fp = tmp_path / "coo.mtx"
    fp.write_bytes(g["coo_bytes"].tobytes())
    np.testing.assert_array_equal(linops.load_array(fp), g["coo_dense"])
    assert linops.spectral_condition_number(np.array([[3.0, 0.0], [0.0, 0.5]])) == g["cond"][0]
    assert linops.spectral_condition_number(np.diag([1.0, 1e-301])) == np.inf
    with pytest.raises(ValueError):
        linops.spectral_condition_number(np.zeros((2, 2)))


def test_problem_validation():
    class Op:
        rows, cols = 4, 3

    with pytest.raises(ValueError):
        problems.Problem(Op(), np.ones(3))
    with pytest.raises(ValueError):
        problems.Problem(Op(), np.ones(4), x_true=np.ones(4))
    with pytest.raises(ValueError):
        problems.Problem(Op(), np.ones(4), noise_level=-1.0)


@pytest.mark.gpu
def test_device_problem_builders_vs_reference(golden, tmp_path):
    """make_tomography: b and x_true bit-identical to the reference's (device
    ray tracer + device fp64 CSR product); make_deblur: x_true bitwise, b to
    the stencil-order rounding; load_operator -> device operator."""
    import paper_2502_02721_b200 as hs

    g = golden("slslu_tomo16")
    p = hs.problems.make_tomography(16, 12, noise_level=0.01, seed=4)
    np.testing.assert_array_equal(p.x_true, g["x_true"])
    np.testing.assert_array_equal(p.b, g["b"])
    assert p.image_shape == (16, 16) and p.operator.rows == 16 * 12
    gd = golden("scmrh_deblur16")
    pd = hs.problems.make_deblur(16, gd["psf"], noise_level=0.01, seed=3)
    np.testing.assert_array_equal(pd.x_true, gd["x_true"])
    np.testing.assert_allclose(pd.b, gd["b"], rtol=0, atol=1e-14 * np.abs(gd["b"]).max())
    ge = golden("exchange")
    fp = tmp_path / "coo.mtx"
    fp.write_bytes(ge["coo_bytes"].tobytes())
    op = hs.linops.load_operator(fp)
    assert isinstance(op, hs.CsrOperator)
    x = np.random.default_rng(0).standard_normal(op.cols)
    import scipy.sparse

    np.testing.assert_array_equal(op.matvec(x), scipy.sparse.csr_matrix(ge["coo_dense"]) @ x)
