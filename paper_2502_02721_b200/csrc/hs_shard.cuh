// Small kernels of the row-sharded (multi-GPU) loop.
//
// Partition: rank r owns the contiguous global block [r*blk, r*blk + loc) of
// each index space (rays for D-side vectors and rows of A, pixels for L-side
// vectors and rows of A^T).  Blocks have equal padded size blk so an
// all-gather of every rank's block yields the vector in global order.  Every
// cross-rank exchange of a pivot-related value is an all-gather followed by
// an "owner pick": each entry is taken verbatim from the rank that owns it,
// so results are bit-identical to the single-GPU run (no floating-point
// reduction touches them).
#pragma once

#include "hs_common.cuh"
#include "hs_loop.cuh"

namespace hs {

// values of a local vector at global positions pos[0..k) (zero when not owned)
template <class T>
__global__ void gather_owned_kernel(const T* __restrict__ u, const long long* __restrict__ pos, int k,
                                    long long off, long long loc, T* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const long long e = pos[j] - off;
  out[j] = (e >= 0 && e < loc) ? u[e] : T(0);
}

// out[j] = all[owner(pos[j]) * ld + j]  with owner = pos / blk
template <class T>
__global__ void owner_pick_kernel(const T* __restrict__ all, int ld, const long long* __restrict__ pos, int k,
                                  long long blk, T* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const long long owner = pos[j] / blk;
  out[j] = all[owner * ld + j];
}

// copy the local best candidate out of the loop state (for the all-gather)
__global__ void cand_export_kernel(const LoopState* __restrict__ st, int side, Cand* __restrict__ out) {
  if (threadIdx.x == 0) {
    out->mag = absval(st->piv_val[side]);
    out->val = st->piv_val[side];
    out->idx = st->piv_idx[side];
  }
}

// merge the P gathered candidates (max |v|, ties to the smallest global index)
__global__ void cand_merge_kernel(const Cand* __restrict__ all, int P, LoopState* __restrict__ st, int side) {
  if (threadIdx.x != 0) return;
  Cand b{-1.0, 0.0, 0x7fffffffffffffffLL};
  for (int r = 0; r < P; ++r) cand_merge(b, all[r]);
  st->piv_val[side] = b.val;
  st->piv_idx[side] = b.idx;
}

// sharded pivot commit: breakdown test, H/W entry, pivot position and pivot
// value as pivot_commit_kernel; the new pivot row of P is written to prow
// (the owner's basis values, zeros elsewhere) for the owner pick
template <class T, class B>
__global__ void pivot_commit_shard_kernel(int k, long long dim, double* __restrict__ hcol, long long* __restrict__ pos,
                                          const B* __restrict__ basis, long long ld, long long off, long long loc,
                                          LoopState* __restrict__ st, int side, int iter, T* __restrict__ pivval_out,
                                          T* __restrict__ prow) {
  if (st->bd_iter != 0 && st->bd_iter < iter) return;
  if (side == 1 && st->bd_iter == iter) return;
  const double val = (k < dim) ? st->piv_val[side] : 0.0;
  const long long idx = st->piv_idx[side];
  if (val == 0.0) {
    if (threadIdx.x == 0) {
      hcol[k] = 0.0;
      st->bd_iter = iter;
      st->bd_side = side;
    }
    return;
  }
  if (threadIdx.x == 0) {
    hcol[k] = val;
    pos[k] = idx;
    *pivval_out = (T)val;
  }
  const long long le = idx - off;
  for (int i = threadIdx.x; i <= k; i += blockDim.x) {
    T pv;
    if (i == k) pv = T(1);
    else pv = (le >= 0 && le < loc) ? cvt<T>(basis[(long long)i * ld + le]) : T(0);
    prow[i] = pv;
  }
}

// P[i*ldp + k] = picked row (owner of the new pivot) for i <= k
template <class T>
__global__ void prow_pick_kernel(const T* __restrict__ all, int ld, const LoopState* __restrict__ st, int side,
                                 int iter, int k, long long blk, T* __restrict__ P, int ldp) {
  if (st->bd_iter != 0 && st->bd_iter <= iter) return;
  const long long owner = st->piv_idx[side] / blk;
  for (int i = threadIdx.x; i <= k; i += blockDim.x) P[(long long)i * ldp + k] = all[owner * ld + i];
}

// one value at a global position (owner pick helper for W(1,1))
template <class T>
__global__ void value_at_kernel(const T* __restrict__ u, long long gpos_idx_holder_side, const LoopState* __restrict__ st,
                                int side, long long off, long long loc, T* __restrict__ out) {
  (void)gpos_idx_holder_side;
  if (threadIdx.x != 0) return;
  const long long e = st->piv_idx[side] - off;
  *out = (e >= 0 && e < loc) ? u[e] : T(0);
}

__global__ void iota_kernel(long long* __restrict__ a, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

// slot -> local pixel for 8x4 tiles over an image block of `rows_img` rows
// tw: tile width in pixels (4, 8 or 16; the tile is tw x 32 / tw)
__global__ void tile_perm_block_kernel(int grid, int rows_img, long long nslots, int* __restrict__ rperm, int tw = 8) {
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nslots) return;
  const int th = 32 / tw;
  const int tiles_x = (grid + tw - 1) / tw;
  const long long tile = slot >> 5;
  const int lane = (int)(slot & 31);
  const long long ty = tile / tiles_x, tx = tile % tiles_x;
  const long long r = ty * th + lane / tw, c = tx * tw + lane % tw;
  rperm[slot] = (r < rows_img && c < grid) ? (int)(r * grid + c) : -1;
}

}  // namespace hs
