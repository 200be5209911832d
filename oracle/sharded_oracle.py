"""TEST INFRASTRUCTURE ONLY -- CPU model of the row-sharded multi-GPU sLSLU loop
(paper_2502_02721_b200/csrc/hs_dist.inc), run with one process per shard over
torch.distributed (gloo).  Same partition (paper_2502_02721_b200.dist.shard_plan),
same exchange pattern (all-gather of l_k and d_{k+1}, owner pick of pivot
values and pivot rows, all-gather + merge of per-rank argmax candidates,
all-reduce of sketch partials), oracle arithmetic on each shard
(hessenberg_oracle's element operations; scipy's sequential CSR row sums on the
rank's rows).  The tests compare it with the single-process oracle: pivots,
H, W and the bases must be bit-identical, y / x agree to rounding.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse
import torch
import torch.distributed as dist

from paper_2502_02721_b200.dist import shard_plan

from . import hessketch_oracle as ho


def _allgather(vec, blk):
    """All-gather equal-size blocks (padded) -> global vector in index order."""
    t = torch.zeros(blk, dtype=torch.float64)
    t[: len(vec)] = torch.from_numpy(np.asarray(vec, dtype=np.float64))
    out = [torch.zeros(blk, dtype=torch.float64) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return torch.cat(out).numpy()


def _allreduce(vec):
    t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64)).clone()
    dist.all_reduce(t)
    return t.numpy()


def _gather_objects(obj):
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def _local_best(v, off):
    mags = np.abs(v)
    if mags.size == 0:
        return (-1.0, 0.0, 1 << 62)
    top = mags.max()
    i = int(np.nonzero(mags == top)[0][0])
    return (float(top), float(v[i]), off + i)


def _merge(cands):
    best = (-1.0, 0.0, 1 << 62)
    for c in cands:  # rank order; total order (mag desc, idx asc)
        if c[0] > best[0] or (c[0] == best[0] and c[2] < best[2]):
            best = c
    return best


def _owner_values(vec_loc, off, loc, blk, positions):
    """Values at global positions, each taken from its owner (all-gather + pick)."""
    mine = [float(vec_loc[p - off]) if off <= p < off + loc else 0.0 for p in positions]
    allv = _gather_objects(mine)
    return [allv[p // blk][j] for j, p in enumerate(positions)]


def _coefficients(pvals, P, dt):
    """Forward substitution on the pivot rows (fsub_*_kernel): c_j = v_j after j steps."""
    k = len(pvals)
    v = [dt.type(x) for x in pvals]
    c = []
    for j in range(k):
        c.append(v[j])
        for i in range(j + 1, k):
            v[i] = dt.type(v[i] - dt.type(v[j] * P[i][j]))
    return c


def sharded_slslu(K, b, S2, maxiter, grid, n_angles, n_bins, dtype=np.float32, x_true=None):
    """Run on every rank of an initialised process group; returns a dict with
    the global pivots, H, W, x and (rank-local) basis shards."""
    dt = np.dtype(dtype)
    ws, rank = dist.get_world_size(), dist.get_rank()
    pl = shard_plan(grid, n_angles, n_bins, ws, rank)
    K = scipy.sparse.csr_matrix(K)
    m, n = K.shape
    A_loc = K[pl.m_off : pl.m_off + pl.m_loc].astype(dt)
    At_loc = K.T.tocsr()[pl.n_off : pl.n_off + pl.n_loc].astype(dt)
    S2 = scipy.sparse.csr_matrix(S2)
    S2_loc = S2[:, pl.m_off : pl.m_off + pl.m_loc]

    def A_apply(full):  # global (padded) input -> local rows
        return A_loc @ np.asarray(full[:n], dtype=dt)

    def At_apply(full):
        return At_loc @ np.asarray(full[:m], dtype=dt)

    r0 = np.asarray(b[pl.m_off : pl.m_off + pl.m_loc], dtype=dt)
    best = _merge(_gather_objects(_local_best(r0, pl.m_off)))
    beta = dt.type(best[1])
    t = [best[2]]
    D = [r0 / beta]
    v0 = At_apply(_allgather(r0, pl.m_blk))
    best = _merge(_gather_objects(_local_best(v0, pl.n_off)))
    alpha = dt.type(best[1])
    g = [best[2]]
    L = [v0 / alpha]
    r = At_apply(_allgather(D[0], pl.m_blk))
    w_cols = [np.array(_owner_values(r, pl.n_off, pl.n_loc, pl.n_blk, [g[0]]))]
    PD = [[dt.type(1)]]
    PL = [[dt.type(1)]]
    sr0 = _allreduce(S2_loc @ r0.astype(np.float64))
    Z, h_cols = [], []
    x = None
    for k in range(1, maxiter + 1):
        u = A_apply(_allgather(L[-1], pl.n_blk))
        Z.append(_allreduce(S2_loc @ u.astype(np.float64)))
        c = _coefficients(_owner_values(u, pl.m_off, pl.m_loc, pl.m_blk, t[:k]), PD, dt)
        for j in range(k):
            u = u - c[j] * D[j]
        best = _merge(_gather_objects(_local_best(u, pl.m_off)))
        val = dt.type(best[1]) if k < m else dt.type(0)
        h_cols.append(np.array([float(x_) for x_ in c] + [float(val)]))
        if val == 0:
            break
        t.append(best[2])
        # new pivot row of P_D: the owner's stored basis values at the new pivot
        PD.append([dt.type(_owner_values(D[i], pl.m_off, pl.m_loc, pl.m_blk, [best[2]])[0]) for i in range(k)]
                  + [dt.type(1)])
        D.append(u / val)
        q = At_apply(_allgather(D[-1], pl.m_blk))
        c2 = _coefficients(_owner_values(q, pl.n_off, pl.n_loc, pl.n_blk, g[:k]), PL, dt)
        for j in range(k):
            q = q - c2[j] * L[j]
        best = _merge(_gather_objects(_local_best(q, pl.n_off)))
        val2 = dt.type(best[1]) if k < n else dt.type(0)
        w_cols.append(np.array([float(x_) for x_ in c2] + [float(val2)]))
        if val2 == 0:
            break
        g.append(best[2])
        PL.append([dt.type(_owner_values(L[i], pl.n_off, pl.n_loc, pl.n_blk, [best[2]])[0]) for i in range(k)]
                  + [dt.type(1)])
        L.append(q / val2)
    kend = len(h_cols)
    M = np.column_stack(Z)
    y = ho.dense_qr_ls(M, sr0)
    xl = np.column_stack(L[:kend]).astype(np.float64) @ y
    x = _allgather(xl, pl.n_blk)[:n]
    H = np.zeros((kend + 1, kend))
    for j, col in enumerate(h_cols):
        H[: j + 2, j] = col
    nw = len(w_cols)
    W = np.zeros((nw, nw))
    for j, col in enumerate(w_cols):
        W[: j + 1, j] = col
    return dict(t=np.array(t), g=np.array(g), H=H, W=W, x=x, D_loc=np.column_stack(D), L_loc=np.column_stack(L),
                plan=pl, k=kend)


def _halo_window(own, rows, width, ry, rank, ws):
    """Own image rows plus ry halo rows from each neighbour (zero outside the
    image), exchanged point to point like hs_dist.inc:halo_exchange."""
    own = np.asarray(own).reshape(rows, width)
    assert ws == 1 or rows >= ry, "shards thinner than the halo are rejected (hs_op_psf_create)"
    win = np.zeros((rows + 2 * ry, width), dtype=own.dtype)
    win[ry : ry + rows] = own
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(own[:ry], dtype=np.float64)), rank - 1))
    if rank < ws - 1:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(own[rows - ry :], dtype=np.float64)), rank + 1))
    if rank > 0:
        t = torch.zeros((ry, width), dtype=torch.float64)
        dist.recv(t, rank - 1)
        win[:ry] = t.numpy().astype(own.dtype)
    if rank < ws - 1:
        t = torch.zeros((ry, width), dtype=torch.float64)
        dist.recv(t, rank + 1)
        win[ry + rows :] = t.numpy().astype(own.dtype)
    for r in reqs:
        r.wait()
    return win


def sharded_scmrh_psf(psf, b, S2, maxiter, shape, dtype=np.float32, stencil=None):
    """Row-sharded sCMRH on the PSF operator (hs_dist.inc:run_square): rank r
    owns image rows [row0, row0 + rows); each operator application is the
    tap-ordered stencil on the window (own rows + halos) restricted to the own
    rows.  Returns the global pivots, H, x and the rank-local basis shard."""
    from paper_2502_02721_b200.dist import psf_shard_plan

    dt = np.dtype(dtype)
    ws, rank = dist.get_world_size(), dist.get_rank()
    Hh, Ww = shape
    n = Hh * Ww
    ry = psf.shape[0] // 2
    pl = psf_shard_plan(Hh, Ww, ws, rank)
    rows = pl.n_loc // Ww
    S2_loc = np.asarray(S2)[:, pl.n_off : pl.n_off + pl.n_loc]

    def A_loc(v_loc):
        win = _halo_window(v_loc, rows, Ww, ry, rank, ws)
        return stencil(win, psf, False, dt)[ry : ry + rows].ravel()

    r0 = np.asarray(b[pl.n_off : pl.n_off + pl.n_loc], dtype=dt)
    best = _merge(_gather_objects(_local_best(r0, pl.n_off)))
    beta = dt.type(best[1])
    t = [best[2]]
    L = [r0 / beta]
    PL = [[dt.type(1)]]
    sr0 = _allreduce(S2_loc @ r0.astype(np.float64))
    Z, h_cols = [], []
    for k in range(1, maxiter + 1):
        u = A_loc(L[-1])
        Z.append(_allreduce(S2_loc @ u.astype(np.float64)))
        c = _coefficients(_owner_values(u, pl.n_off, pl.n_loc, pl.n_blk, t[:k]), PL, dt)
        for j in range(k):
            u = u - c[j] * L[j]
        best = _merge(_gather_objects(_local_best(u, pl.n_off)))
        val = dt.type(best[1]) if k < n else dt.type(0)
        h_cols.append(np.array([float(x_) for x_ in c] + [float(val)]))
        if val == 0:
            break
        t.append(best[2])
        PL.append([dt.type(_owner_values(L[i], pl.n_off, pl.n_loc, pl.n_blk, [best[2]])[0]) for i in range(k)]
                  + [dt.type(1)])
        L.append(u / val)
    kend = len(h_cols)
    y = ho.dense_qr_ls(np.column_stack(Z), sr0)
    xl = np.column_stack(L[:kend]).astype(np.float64) @ y
    x = _allgather(xl, pl.n_blk)[:n]
    H = np.zeros((kend + 1, kend))
    for j, col in enumerate(h_cols):
        H[: j + 2, j] = col
    return dict(t=np.array(t), H=H, x=x, L_loc=np.column_stack(L), plan=pl, k=kend)
