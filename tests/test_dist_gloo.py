"""Multi-process (world_size 2, gloo, CPU) check of the row-sharded loop's
design: the sharded CPU model (oracle/sharded_oracle.py, same partition and
exchange pattern as csrc/hs_dist.inc) reproduces the single-process oracle
bit for bit on pivots, H, W and bases."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2502_02721_b200.dist import shard_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, cfg, outdir):
    import torch.distributed as dist

    from oracle import sharded_oracle as so
    from oracle import tomo_oracle as to
    from paper_2502_02721_b200.problems import add_noise, random_ellipses

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    grid, angles, bins, K, dt = cfg
    M = to.tomography_matrix(grid, angles, bins)
    x = random_ellipses(grid, 10, 0).ravel()
    b, _ = add_noise(M @ x, 0.01, 1)
    rng = np.random.default_rng(3)
    import scipy.sparse

    ell = 4 * K
    rows = np.concatenate([rng.choice(ell, size=8, replace=False) for _ in range(M.shape[0])])
    S = scipy.sparse.csr_matrix((rng.choice([-1.0, 1.0], size=8 * M.shape[0]) / np.sqrt(8),
                                 (rows, np.repeat(np.arange(M.shape[0]), 8))), shape=(ell, M.shape[0]))
    out = so.sharded_slslu(M, b, S, K, grid, angles, bins, dtype=dt)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), t=out["t"], g=out["g"], H=out["H"], W=out["W"], x=out["x"],
             D=out["D_loc"], L=out["L_loc"])
    dist.destroy_process_group()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_sharded_model_matches_single_process(tmp_path, dt):
    from oracle import hessketch_oracle as ho
    from oracle import tomo_oracle as to
    from paper_2502_02721_b200.problems import add_noise, random_ellipses

    grid, angles, bins, K = 24, 16, 37, 12
    ws = 2
    mp.spawn(_worker, args=(ws, _free_port(), (grid, angles, bins, K, dt), str(tmp_path)), nprocs=ws, join=True)
    M = to.tomography_matrix(grid, angles, bins)
    x = random_ellipses(grid, 10, 0).ravel()
    b, _ = add_noise(M @ x, 0.01, 1)
    rng = np.random.default_rng(3)
    import scipy.sparse

    ell = 4 * K
    rows = np.concatenate([rng.choice(ell, size=8, replace=False) for _ in range(M.shape[0])])
    S = scipy.sparse.csr_matrix((rng.choice([-1.0, 1.0], size=8 * M.shape[0]) / np.sqrt(8),
                                 (rows, np.repeat(np.arange(M.shape[0]), 8))), shape=(ell, M.shape[0]))
    ref = ho.hessenberg_solve(ho.csr_operator(M, dt), b, square=False, maxiter=K, S2=S)
    t_ref, g_ref = ho.pivots_of(ref.state)
    D_ref = np.column_stack(ref.state.D)
    L_ref = np.column_stack(ref.state.L)
    for r in range(ws):
        got = dict(np.load(tmp_path / f"rank{r}.npz"))
        np.testing.assert_array_equal(got["t"], t_ref)
        np.testing.assert_array_equal(got["g"], g_ref)
        np.testing.assert_array_equal(got["H"], ref.state.H_matrix())
        np.testing.assert_array_equal(got["W"], ref.state.W_matrix())
        pl = shard_plan(grid, angles, bins, ws, r)
        np.testing.assert_array_equal(got["D"], D_ref[pl.m_off:pl.m_off + pl.m_loc])
        np.testing.assert_array_equal(got["L"], L_ref[pl.n_off:pl.n_off + pl.n_loc])
        np.testing.assert_allclose(got["x"], ref.x, rtol=1e-9, atol=1e-12 * np.abs(ref.x).max())


def test_shard_plan_covers_every_index():
    for grid, angles, bins in ((64, 30, 91), (2048, 720, 2897)):
        m, n = angles * bins, grid * grid
        for P in (1, 2, 4, 8):
            plans = [shard_plan(grid, angles, bins, P, r) for r in range(P)]
            assert sum(p.m_loc for p in plans) == m and sum(p.n_loc for p in plans) == n
            for r, p in enumerate(plans):
                assert p.m_off == r * p.m_blk and p.n_off == r * p.n_blk
                assert p.m_blk % 64 == 0 and p.n_blk % (8 * grid) == 0


def _psf_worker(rank, ws, port, cfg, outdir):
    import torch.distributed as dist

    from oracle import sharded_oracle as so
    from oracle import tomo_oracle as to
    from paper_2502_02721_b200.problems import add_noise, gaussian_psf, rectangles_and_discs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    (Hh, Ww), K, dt = cfg
    psf = gaussian_psf(2.0, radius=7)
    x = rectangles_and_discs(max(Hh, Ww), 20, 0)[:Hh, :Ww].ravel()
    b, _ = add_noise(to.psf_stencil(x.reshape(Hh, Ww), psf, False, np.float64).ravel(), 0.01, 1)
    S2 = np.random.default_rng(4).standard_normal((4 * K, Hh * Ww)) / np.sqrt(4 * K)
    out = so.sharded_scmrh_psf(psf, b, S2, K, (Hh, Ww), dtype=dt, stencil=to.psf_stencil)
    np.savez(os.path.join(outdir, f"psf{rank}.npz"), t=out["t"], H=out["H"], x=out["x"], L=out["L_loc"])
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,shape", [(2, (40, 37)), (3, (60, 24))])
def test_sharded_psf_model_matches_single_process(tmp_path, ws, shape):
    """Row-sharded sCMRH on the PSF operator with halo exchange (hs_dist.inc:
    run_square): pivots, H and the basis shards bit-identical to the single
    process for 2 and 3 ranks (uneven last shard)."""
    from oracle import hessketch_oracle as ho
    from oracle import tomo_oracle as to
    from paper_2502_02721_b200.dist import psf_shard_plan
    from paper_2502_02721_b200.problems import add_noise, gaussian_psf, rectangles_and_discs

    K, dt = 14, np.float32
    Hh, Ww = shape
    mp.spawn(_psf_worker, args=(ws, _free_port(), (shape, K, dt), str(tmp_path)), nprocs=ws, join=True)
    psf = gaussian_psf(2.0, radius=7)
    x = rectangles_and_discs(max(Hh, Ww), 20, 0)[:Hh, :Ww].ravel()
    b, _ = add_noise(to.psf_stencil(x.reshape(Hh, Ww), psf, False, np.float64).ravel(), 0.01, 1)
    S2 = np.random.default_rng(4).standard_normal((4 * K, Hh * Ww)) / np.sqrt(4 * K)
    A = ho.Operator(Hh * Ww, Hh * Ww,
                    lambda v: to.psf_stencil(v.reshape(Hh, Ww), psf, False, dt).ravel(),
                    lambda v: to.psf_stencil(v.reshape(Hh, Ww), psf, True, dt).ravel(), dt)
    ref = ho.hessenberg_solve(A, b, square=True, maxiter=K, S2=S2)
    t_ref, _ = ho.pivots_of(ref.state)
    L_ref = np.column_stack(ref.state.L)
    for r in range(ws):
        got = dict(np.load(tmp_path / f"psf{r}.npz"))
        np.testing.assert_array_equal(got["t"], t_ref)
        np.testing.assert_array_equal(got["H"], ref.state.H_matrix())
        pl = psf_shard_plan(Hh, Ww, ws, r)
        np.testing.assert_array_equal(got["L"], L_ref[pl.n_off:pl.n_off + pl.n_loc])
        np.testing.assert_allclose(got["x"], ref.x, rtol=1e-9, atol=1e-12 * np.abs(ref.x).max())
