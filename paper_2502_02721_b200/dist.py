"""Multi-GPU plumbing: one process per GPU, NCCL communicator inside the C
library, torch.distributed only to ship the NCCL unique id.

    import torch.distributed as dist
    dist.init_process_group("nccl")           # torchrun, MASTER_ADDR=127.0.0.1
    from paper_2502_02721_b200 import dist as hsd
    hsd.init_comm()                            # library communicator on this rank's GPU
    op = TomographyOperator(2048, 720, 2897)   # builds this rank's shard only
    res = slslu(op, b, cfg, x_true, sketch=S)  # row-sharded loop; full x on every rank

Partition (``shard_plan``, mirrored by hs_dist.inc:build_tomo_sharded): rank r
owns rays [r*m_blk, r*m_blk + m_loc) -- rows of A and entries of the
data-side vectors -- and image rows [r*rows_pr, ...) i.e. pixels
[r*n_blk, r*n_blk + n_loc) -- rows of A^T and entries of the solution-side
vectors.  Blocks are padded to equal sizes so all-gathers produce the global
vectors in index order.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib

__all__ = ["ShardPlan", "shard_plan", "psf_shard_plan", "shard_granule", "sketch_tile", "init_comm", "nccl_selftest", "comm_info",
           "local_group", "run_ranks"]


def _round_up(a, b):
    return (a + b - 1) // b * b


@dataclass(frozen=True)
class ShardPlan:
    m_off: int
    m_loc: int
    m_blk: int
    n_off: int
    n_loc: int
    n_blk: int


def _pow2_clamped(length, shift, lo, hi):
    e = (length >> shift).bit_length() - 1 if (length >> shift) > 0 else 0
    return 1 << min(hi, max(lo, e))


def sketch_tile(kind, length):
    """Columns per sketch partial tile (hs_sketch.cuh): sparse-sign ~len/128
    in [32, 8192], Gaussian / dense ~len/1024 in [256, 8192]."""
    if kind == "sparse_sign":
        return _pow2_clamped(length, 7, 5, 13)
    return _pow2_clamped(length, 10, 8, 13)


def shard_granule(length):
    """Ray blocks (rows of a tomography operator) are multiples of this power
    of two; image shards are multiples of 8 rows.  Sketches sum their tile
    partials granule by granule (hs_sketch.cuh), so they are P-independent."""
    return _pow2_clamped(length, 7, 8, 13)


def shard_plan(grid, n_angles, n_bins, nranks, rank):
    """Row blocks of rank ``rank`` for a grid^2-pixel, n_angles*n_bins-ray
    operator (same arithmetic as the C library, hs_dist.inc:build_tomo_sharded)."""
    m, n = n_angles * n_bins, grid * grid
    m_blk = _round_up(-(-m // nranks), max(64, shard_granule(m)))
    m_off = rank * m_blk
    m_loc = max(0, min(m_blk, m - m_off))
    rows_pr = _round_up(-(-grid // nranks), 8)
    n_blk = rows_pr * grid
    n_off = rank * n_blk
    n_loc = max(0, min(n_blk, n - n_off))
    return ShardPlan(m_off, m_loc, m_blk, n_off, n_loc, n_blk)


def psf_shard_plan(height, width, nranks, rank):
    """Image-row blocks of the row-sharded PSF operator (hs_abi.inc:
    hs_op_psf_create): rank ``rank`` owns rows [row0, row0 + rows) -- entries
    [off, off + loc) of every n-vector -- and exchanges kh/2 halo rows with each
    neighbour per operator application."""
    rows_pr = _round_up(-(-height // nranks), 8)
    row0 = rank * rows_pr
    rows = max(0, min(rows_pr, height - row0))
    blk = rows_pr * width
    return ShardPlan(row0 * width, rows * width, blk, row0 * width, rows * width, blk)


def init_comm(ctx=None):
    """Create the library's NCCL communicator over the torch.distributed
    world (rank 0 draws the unique id, torch broadcasts it).  Returns
    (world_size, rank)."""
    import torch.distributed as dist

    ctx = ctx or _lib.context()
    lib = _lib.load()
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        _lib.check(lib.hs_comm_init(ctx.handle, 1, 0, None))
        return 1, 0
    ws, rank = dist.get_world_size(), dist.get_rank()
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        _lib.check(lib.hs_comm_get_unique_id(uid))
    box = [bytes(uid.raw)]
    dist.broadcast_object_list(box, src=0)
    raw = ctypes.create_string_buffer(box[0], 128)
    _lib.check(lib.hs_comm_init(ctx.handle, ws, rank, raw))
    return ws, rank


def nccl_selftest(ctx=None):
    """Run every NCCL call of the sharded loops on a one-rank communicator on
    this context's GPU and check the results (raises on any mismatch)."""
    ctx = ctx or _lib.context()
    _lib.check(_lib.load().hs_nccl_selftest(ctx.handle))


def comm_info(ctx=None):
    ctx = ctx or _lib.context()
    n, r = _lib.c_i32(), _lib.c_i32()
    _lib.check(_lib.load().hs_comm_info(ctx.handle, ctypes.byref(n), ctypes.byref(r)))
    return n.value, r.value


def force_sharding(on=True, ctx=None):
    """Test hook: route operators / solves through the sharded path with one rank."""
    ctx = ctx or _lib.context()
    _lib.check(_lib.load().hs_ctx_force_sharding(ctx.handle, 1 if on else 0))


def local_group(nranks, devices=None):
    """``nranks`` in-process ranks: one new context per rank (on ``devices[r]``,
    default all on the current device) joined by the library's in-process
    communicator (hs_comm_init_local: the NCCL path's partition and message
    sequence, with stream-ordered device copies between the contexts).
    Drive them with :func:`run_ranks`; close the contexts when done."""
    if devices is None:
        devices = [_lib.context().device] * nranks
    if len(devices) != nranks:
        raise ValueError("one device per rank")
    ctxs = [_lib.Context(d) for d in devices]
    arr = (_lib.c_vp * nranks)(*[c.handle for c in ctxs])
    _lib.check(_lib.load().hs_comm_init_local(arr, nranks))
    return ctxs


def run_ranks(fn, ctxs):
    """Run ``fn(rank, ctx)`` on one host thread per rank (each under
    ``_lib.use_context(ctx)``) and return the per-rank results; the first
    exception is re-raised after every thread has finished."""
    import threading

    out, err = [None] * len(ctxs), [None] * len(ctxs)

    def body(r):
        try:
            with _lib.use_context(ctxs[r]):
                out[r] = fn(r, ctxs[r])
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e
            _lib.load().hs_comm_abort(ctxs[r].handle)  # release the peers' collectives

    threads = [threading.Thread(target=body, args=(r,)) for r in range(len(ctxs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
