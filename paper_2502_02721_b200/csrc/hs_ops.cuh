// Operator kernels: y = A x and y = A^T x for the three operator families the
// reference's LinearOperator plugin carries (linops.py:71-149):
//   * CSR (tomography; linops.py:137-141 -> scipy csr_matvec),
//   * dense (linops.py:142-145),
//   * PSF stencil (deblurring; problems.py:257-267).
//
// Order fidelity ("order-faithful operator kernels"):
// every output entry is accumulated left to right over its stored entries /
// taps, product rounded then added (Rn<T>::mul / Rn<T>::add), starting from +0.
// That is exactly scipy's csr_matvec, so the CSR operator reproduces the
// reference bit for bit (fp64) and oracle32 (fp32).
#pragma once

#include "hs_common.cuh"

namespace hs {

// --------------------------------------------------------------------------
// CSR: warp-staged, thread-per-row sequential sum.
//
// A warp owns 32 consecutive rows.  Per chunk of CH entries per row, the warp
// walks the 32 rows one by one and loads that row's next CH (value, column)
// pairs with consecutive lanes (coalesced), gathers x[col], forms the rounded
// product and parks it in shared memory (row-major, padded stride CH+1 so the
// per-lane read-back is bank-conflict free).  Then every lane adds its own
// row's products in stored order.  All 32 lanes do useful serial adds at once,
// the HBM stream of (value, column) is read with full-sector coalescing.

template <int CH> struct SpmvCfg { static constexpr int kChunk = CH; };

template <class V, class Tin, class T, int WARPS, int CH>
__global__ void __launch_bounds__(WARPS * 32)
csr_seq_spmv_kernel(long long rows, const long long* __restrict__ rowptr,
                    const int* __restrict__ col, const V* __restrict__ val,
                    const Tin* __restrict__ x, T* __restrict__ y) {
  __shared__ T prod[WARPS][32][CH + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T (*P)[CH + 1] = prod[warp];
  for (long long row0 = ((long long)blockIdx.x * WARPS + warp) * 32; row0 < rows;
       row0 += (long long)gridDim.x * WARPS * 32) {
    const long long myrow = row0 + lane;
    long long s = 0;
    int len = 0;
    if (myrow < rows) {
      s = rowptr[myrow];
      len = (int)(rowptr[myrow + 1] - s);
    }
    int maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    T acc = T(0);
    for (int off = 0; off < maxlen; off += CH) {
      // stage: rows in groups of 8 so 8 independent load->gather chains are in flight
#pragma unroll 1
      for (int i0 = 0; i0 < 32; i0 += 8) {
        T pv[8][CH / 32];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const long long si = __shfl_sync(0xffffffffu, s, i0 + r);
          const int li = __shfl_sync(0xffffffffu, len, i0 + r) - off;
#pragma unroll
          for (int q = 0; q < CH / 32; ++q) {
            const int e = q * 32 + lane;
            if (e < li) {
              const long long p = si + off + e;
              pv[r][q] = Rn<T>::mul(cvt<T>(val[p]), cvt<T>(x[col[p]]));
            }
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
          for (int q = 0; q < CH / 32; ++q) P[i0 + r][q * 32 + lane] = pv[r][q];
        }
      }
      __syncwarp();
      const int cnt = min(CH, len - off);
      for (int j = 0; j < cnt; ++j) acc = Rn<T>::add(acc, P[lane][j]);
      __syncwarp();
    }
    if (myrow < rows) y[myrow] = acc;
  }
}

// --------------------------------------------------------------------------
// dense: A stored column-major (lda = rows), one thread per output row,
// sequential over columns (coalesced across threads).  Used for both A x
// (A column-major) and A^T y (A row-major == A^T column-major).

template <class V, class Tin, class T>
__global__ void __launch_bounds__(256)
dense_seq_gemv_kernel(long long rows, long long cols, const V* __restrict__ Acm,
                      const Tin* __restrict__ x, T* __restrict__ y) {
  extern __shared__ unsigned char smem_raw[];
  T* xs = reinterpret_cast<T*>(smem_raw);
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  T acc = T(0);
  for (long long c0 = 0; c0 < cols; c0 += 1024) {
    const int cn = (int)min((long long)1024, cols - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += blockDim.x) xs[i] = cvt<T>(x[c0 + i]);
    __syncthreads();
    if (r < rows) {
      const V* a = Acm + c0 * rows + r;
      for (int j = 0; j < cn; ++j) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(a[(long long)j * rows]), xs[j]));
    }
  }
  if (r < rows) y[r] = acc;
}

// --------------------------------------------------------------------------
// PSF stencil: zero-boundary 'same' convolution (transpose = 0) or correlation
// (transpose = 1) on an H x W image, taps summed a-major / b-minor
// (oracle/tomo_oracle.py:psf_stencil), smem-tiled with the zero halo.

template <class V, class Tin, class T, int TILE_X, int TILE_Y>
__global__ void __launch_bounds__(TILE_X * TILE_Y)
psf_stencil_kernel(int H, int W, int kh, int kw, const V* __restrict__ K,
                   const Tin* __restrict__ x, T* __restrict__ y, int transpose) {
  extern __shared__ unsigned char smem_raw[];
  const int ry = kh / 2, rx = kw / 2;
  const int SW = TILE_X + 2 * rx, SH = TILE_Y + 2 * ry;
  T* tile = reinterpret_cast<T*>(smem_raw);
  T* ks = tile + SW * SH;
  const int tx = threadIdx.x % TILE_X, ty = threadIdx.x / TILE_X;
  const int c0 = blockIdx.x * TILE_X, r0 = blockIdx.y * TILE_Y;
  for (int i = threadIdx.x; i < kh * kw; i += blockDim.x) ks[i] = cvt<T>(K[i]);
  for (int i = threadIdx.x; i < SW * SH; i += blockDim.x) {
    const int sr = i / SW, sc = i % SW;
    const int gr = r0 + sr - ry, gc = c0 + sc - rx;
    T v = T(0);
    if (gr >= 0 && gr < H && gc >= 0 && gc < W) v = cvt<T>(x[(long long)gr * W + gc]);
    tile[i] = v;
  }
  __syncthreads();
  const int r = r0 + ty, c = c0 + tx;
  if (r >= H || c >= W) return;
  T acc = T(0);
  if (!transpose) {
    // out[r,c] = sum_a sum_b K[a,b] x[r + ry - a, c + rx - b]
    for (int a = 0; a < kh; ++a) {
      const T* trow = tile + (ty + 2 * ry - a) * SW + tx + 2 * rx;
      const T* krow = ks + a * kw;
      for (int b = 0; b < kw; ++b) acc = Rn<T>::add(acc, Rn<T>::mul(krow[b], trow[-b]));
    }
  } else {
    // out[r,c] = sum_a sum_b K[a,b] x[r - ry + a, c - rx + b]
    for (int a = 0; a < kh; ++a) {
      const T* trow = tile + (ty + a) * SW + tx;
      const T* krow = ks + a * kw;
      for (int b = 0; b < kw; ++b) acc = Rn<T>::add(acc, Rn<T>::mul(krow[b], trow[b]));
    }
  }
  y[(long long)r * W + c] = acc;
}

}  // namespace hs
