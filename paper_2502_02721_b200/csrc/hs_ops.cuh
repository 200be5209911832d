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
// (A column-major) and A^T y (A row-major == A^T column-major).  The host
// sizes blocks so the rows spread over all SMs (config 1: 1024 rows -> 32
// blocks of 32 threads), each SM streaming its own slice of A.

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
#pragma unroll 16
      for (int j = 0; j < cn; ++j) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(__ldg(a + (long long)j * rows)), xs[j]));
    }
  }
  if (r < rows) y[r] = acc;
}

// Tiled variant (the default): a block owns RB rows; for each tile of CT
// columns all 256 threads form the RB x CT products (rounded, independent,
// many loads in flight) into shared memory, then RB threads add each row's
// products left to right.  Same operation sequence per row as the simple
// kernel -- product rounded, then added, columns ascending -- so bit-identical;
// the serial part is a shared-memory add chain instead of a global-load chain.
// Default RB = 8, CT = 1024: config 1 (1024 x 1024) runs as 128 blocks, one
// barrier-separated product phase and one 1024-long add chain per row
// (RB = 32, CT = 256 -- 32 blocks, four phases -- is HS_DENSE_RB32=1).
template <class V, class Tin, class T, int RB = 8, int CT = 1024>
__global__ void __launch_bounds__(256)
dense_tile_gemv_kernel(long long rows, long long cols, const V* __restrict__ Acm, const Tin* __restrict__ x,
                       T* __restrict__ y) {
  constexpr int LD = CT + 2;  // even: 16-byte rows for the paired chain reads, 8 rows on distinct banks
  extern __shared__ __align__(16) unsigned char dense_smem[];
  T* prod = reinterpret_cast<T*>(dense_smem);  // RB x LD
  T* xs = prod + RB * LD;                      // CT
  const long long r0 = (long long)blockIdx.x * RB;
  const int tid = threadIdx.x;
  T acc = T(0);
  for (long long c0 = 0; c0 < cols; c0 += CT) {
    const int cn = (int)min((long long)CT, cols - c0);
    for (int i = tid; i < cn; i += blockDim.x) xs[i] = cvt<T>(x[c0 + i]);
    __syncthreads();
#pragma unroll 8
    for (int idx = tid; idx < RB * cn; idx += blockDim.x) {
      const int rr = idx % RB, cc = idx / RB;
      const long long r = r0 + rr;
      prod[rr * LD + cc] = r < rows ? Rn<T>::mul(cvt<T>(__ldg(Acm + (c0 + cc) * rows + r)), xs[cc]) : T(0);
    }
    __syncthreads();
    if (tid < RB) {
      const T* pr = prod + tid * LD;
      int j = 0;
      if constexpr (sizeof(T) == 8) {  // two products per shared-memory load; same adds, same order
        const double2* p2 = reinterpret_cast<const double2*>(pr);
#pragma unroll 8
        for (; j + 1 < cn; j += 2) {
          const double2 t = p2[j >> 1];
          acc = Rn<T>::add(acc, t.x);
          acc = Rn<T>::add(acc, t.y);
        }
      }
#pragma unroll 8
      for (; j < cn; ++j) acc = Rn<T>::add(acc, pr[j]);
    }
    __syncthreads();
  }
  if (tid < RB && r0 + tid < rows) y[r0 + tid] = acc;
}

inline size_t dense_tile_smem(size_t tsize, int rb, int ct) { return ((size_t)rb * (ct + 2) + ct) * tsize; }

// --------------------------------------------------------------------------
// PSF stencil: zero-boundary 'same' convolution (transpose = 0) or correlation
// (transpose = 1) on an H x W image, taps summed a-major / b-minor
// (oracle/tomo_oracle.py:psf_stencil), smem-tiled with the zero halo.

// Output rows [out_row0, out_row0 + out_rows) of the H-row image x are written
// to y[(r - out_row0) * W + c] (a row-sharded rank passes its rows plus the
// neighbours' halo rows as x and computes only its own rows).
// KWC > 0: the PSF width as a compile-time constant (the tap loop unrolls and
// its shared-memory reads batch: config 2's 15 x 15 stencil on a 256^2 image);
// KWC = 0: any width.  Same taps in the same order either way.
template <class V, class Tin, class T, int TILE_X, int TILE_Y, int KWC = 0>
__global__ void __launch_bounds__(TILE_X * TILE_Y)
psf_stencil_kernel(int H, int W, int kh, int kw_rt, const V* __restrict__ K,
                   const Tin* __restrict__ x, T* __restrict__ y, int transpose, int out_row0, int out_rows) {
  const int kw = KWC > 0 ? KWC : kw_rt;
  extern __shared__ unsigned char smem_raw[];
  const int ry = kh / 2, rx = kw / 2;
  const int SW = TILE_X + 2 * rx, SH = TILE_Y + 2 * ry;
  T* tile = reinterpret_cast<T*>(smem_raw);
  T* ks = tile + SW * SH;
  const int tx = threadIdx.x % TILE_X, ty = threadIdx.x / TILE_X;
  const int c0 = blockIdx.x * TILE_X, r0 = out_row0 + blockIdx.y * TILE_Y;
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
  if (r >= out_row0 + out_rows || c >= W) return;
  T acc = T(0);
  if (!transpose) {
    // out[r,c] = sum_a sum_b K[a,b] x[r + ry - a, c + rx - b]
    for (int a = 0; a < kh; ++a) {
      const T* trow = tile + (ty + 2 * ry - a) * SW + tx + 2 * rx;
      const T* krow = ks + a * kw;
      if (KWC > 0) {
#pragma unroll
        for (int b = 0; b < KWC; ++b) acc = Rn<T>::add(acc, Rn<T>::mul(krow[b], trow[-b]));
      } else {
        for (int b = 0; b < kw; ++b) acc = Rn<T>::add(acc, Rn<T>::mul(krow[b], trow[-b]));
      }
    }
  } else {
    // out[r,c] = sum_a sum_b K[a,b] x[r - ry + a, c - rx + b]
    for (int a = 0; a < kh; ++a) {
      const T* trow = tile + (ty + a) * SW + tx;
      const T* krow = ks + a * kw;
      if (KWC > 0) {
#pragma unroll
        for (int b = 0; b < KWC; ++b) acc = Rn<T>::add(acc, Rn<T>::mul(krow[b], trow[b]));
      } else {
        for (int b = 0; b < kw; ++b) acc = Rn<T>::add(acc, Rn<T>::mul(krow[b], trow[b]));
      }
    }
  }
  y[(long long)(r - out_row0) * W + c] = acc;
}

// Register-blocked variant for the common odd widths (KW = 15, 31): each
// thread owns R consecutive outputs of a row; per PSF row a it loads the
// R + KW - 1 input values its outputs touch into registers once and then
// walks the KW taps, so every tap value (a smem broadcast) feeds R products.
// Each output still accumulates a-major / b-minor with the product rounded
// before the add (Rn mul, Rn add): bit-identical to psf_stencil_kernel.
template <class V, class Tin, class T, int KW, int R, int TXT, int TY, bool TR>
__global__ void __launch_bounds__(TXT * TY)
psf_stencil_rb_kernel(int H, int W, int kh, const V* __restrict__ K, const Tin* __restrict__ x,
                      T* __restrict__ y, int out_row0, int out_rows) {
  constexpr int rx = KW / 2;
  constexpr int TILE_X = TXT * R;
  constexpr int SW = ((TILE_X + 2 * rx + 3) / 4) * 4;  // row pitch (16-byte aligned rows)
  constexpr int NW = R + KW - 1;                       // window per PSF row
  const int ry = kh / 2;
  const int SH = TY + 2 * ry;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);
  T* ks = tile + SW * SH;
  const int tx = threadIdx.x % TXT, ty = threadIdx.x / TXT;
  const int c0 = blockIdx.x * TILE_X, r0 = out_row0 + blockIdx.y * TY;
  for (int i = threadIdx.x; i < kh * KW; i += blockDim.x) ks[i] = cvt<T>(K[i]);
  for (int i = threadIdx.x; i < SW * SH; i += blockDim.x) {
    const int sr = i / SW, sc = i - sr * SW;
    const int gr = r0 + sr - ry, gc = c0 + sc - rx;
    T v = T(0);
    if (sc < TILE_X + 2 * rx && gr >= 0 && gr < H && gc >= 0 && gc < W) v = cvt<T>(x[(long long)gr * W + gc]);
    tile[i] = v;
  }
  __syncthreads();
  const int r = r0 + ty, cb = c0 + tx * R;
  if (r >= out_row0 + out_rows || cb >= W) return;
  T acc[R];
#pragma unroll
  for (int j = 0; j < R; ++j) acc[j] = T(0);
  for (int a = 0; a < kh; ++a) {
    const T* trow = tile + (TR ? (ty + a) : (ty + 2 * ry - a)) * SW + tx * R;
    T w[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) w[q] = trow[q];
    const T* krow = ks + a * KW;
#pragma unroll
    for (int b = 0; b < KW; ++b) {
      const T kab = krow[b];
#pragma unroll
      for (int j = 0; j < R; ++j) acc[j] = Rn<T>::add(acc[j], Rn<T>::mul(kab, w[TR ? j + b : j + KW - 1 - b]));
    }
  }
  T* yr = y + (long long)(r - out_row0) * W + cb;
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (cb + j < W) yr[j] = acc[j];
}

template <class T, int KW> struct PsfRb {
  static constexpr int R = sizeof(T) == 4 ? 8 : 4;
  static constexpr int TXT = sizeof(T) == 4 ? 16 : 32;
  static constexpr int TY = sizeof(T) == 4 ? 16 : 8;
  static constexpr int TILE_X = TXT * R;
  static size_t smem(int kh) {
    const int SW = ((TILE_X + 2 * (KW / 2) + 3) / 4) * 4;
    return ((size_t)SW * (TY + 2 * (kh / 2)) + (size_t)kh * KW) * sizeof(T);
  }
};

}  // namespace hs

namespace hs {

// --------------------------------------------------------------------------
// SELL-32x4: the device layout of the tomography operators.
//
// Rows are grouped in slices of 32 consecutive rows (adjacent parallel rays
// for A, adjacent pixels for A^T).  Inside a slice, entry e of the slice's
// row r sits at slot  sptr[s] + (e/4)*128 + r*4 + e%4:  chunk q of a slice
// is 512 contiguous bytes of values (fp32) holding entries 4q..4q+3 of each
// of the 32 rows.  A warp owns a slice, lane r owns row r: every load of the
// (value, column) stream is one fully coalesced 128-bit access per lane, and
// each lane still adds ITS OWN row's products strictly left to right
// (product rounded, then added; scipy csr_matvec order).  Rows shorter than
// the slice's longest row are padded to it (zeros, never added).
//
// The x gathers of the 32 lanes hit the same few sectors at every step
// (adjacent rays at the same depth), and a lane's next gather usually falls
// in the sector its previous one loaded, so x is served from L1; the matrix
// stream is loaded with the evict-first (.cs) policy to keep x resident in L2.

template <class V> struct Chunk4;
template <> struct Chunk4<float> {
  float v[4];
  static __device__ __forceinline__ Chunk4 load(const float* p) {
    float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    return Chunk4{{t.x, t.y, t.z, t.w}};
  }
  static __device__ __forceinline__ Chunk4 lds(const void* p) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    return Chunk4{{t.x, t.y, t.z, t.w}};
  }
};
template <> struct Chunk4<double> {
  double v[4];
  static __device__ __forceinline__ Chunk4 load(const double* p) {
    double2 a = __ldcs(reinterpret_cast<const double2*>(p));
    double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
    return Chunk4{{a.x, a.y, b.x, b.y}};
  }
  static __device__ __forceinline__ Chunk4 lds(const void* p) {
    const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
    return Chunk4{{a.x, a.y, b.x, b.y}};
  }
};

// ---- shared-memory address / L2 policy helpers ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <class T, class Tin> __device__ __forceinline__ T gather_x(const Tin* __restrict__ x, int c) {
  return cvt<T>(__ldg(x + c));
}
template <> __device__ __forceinline__ float gather_x<float, __nv_bfloat16>(const __nv_bfloat16* __restrict__ x, int c) {
  return __bfloat162float(x[c]);
}

// xT / sflag (optional): slices whose flag is set store their column indices
// in the TRANSPOSED image layout and gather from xT (the image transposed).
// Used for near-horizontal rays of the tomography operator, whose 32 lanes
// step through 32 adjacent image rows: in the transposed layout those are 32
// adjacent words (one 128-byte line) instead of 32 lines.  Entry order, and
// with it the summation order, is unchanged.
template <class V, class Tin, class T>
__global__ void __launch_bounds__(256)
sell_spmv_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                 const int* __restrict__ rlen, const int* __restrict__ col, const V* __restrict__ val,
                 const Tin* __restrict__ xrow, const Tin* __restrict__ xT, const unsigned char* __restrict__ sflag,
                 const int* __restrict__ rperm, T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nslices; s += wstride) {
    const Tin* __restrict__ x = (sflag != nullptr && sflag[s]) ? xT : xrow;
    const long long slot = s * 32 + lane;  // rlen / rbase are slot-indexed; rperm maps slot -> row
    const long long row = rperm ? (long long)rperm[slot] : slot;
    const int len = rlen[slot];
    const long long base = sptr[s];
    const int nq_slice = (int)((sptr[s + 1] - base) >> 7);
    const int nq = (len + 3) >> 2;
    const int* cp = col + base + lane * 4;
    const V* vp = val + base + lane * 4;
    T acc = T(0);
    if (nq > 0) {
      // software pipeline: chunk q+1's (column, value) loads are in flight
      // while chunk q's gathers and adds run
      int4 c = __ldcs(reinterpret_cast<const int4*>(cp));
      Chunk4<V> v = Chunk4<V>::load(vp);
      for (int q = 0; q < nq; ++q) {
        int4 cn = c;
        Chunk4<V> vn = v;
        if (q + 1 < nq) {
          cn = __ldcs(reinterpret_cast<const int4*>(cp + (long long)(q + 1) * 128));
          vn = Chunk4<V>::load(vp + (long long)(q + 1) * 128);
        }
        const int e = q * 4;
        const T x0 = gather_x<T>(x, c.x);
        const T x1 = (e + 1 < len) ? gather_x<T>(x, c.y) : T(0);
        const T x2 = (e + 2 < len) ? gather_x<T>(x, c.z) : T(0);
        const T x3 = (e + 3 < len) ? gather_x<T>(x, c.w) : T(0);
        acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), x0));
        if (e + 1 < len) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), x1));
        if (e + 2 < len) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), x2));
        if (e + 3 < len) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[3]), x3));
        c = cn;
        v = vn;
      }
    }
    (void)nq_slice;
    if (row >= 0 && row < rows) y[row] = acc;
  }
}

// ---- image transpose (grid x grid), 32x32 smem tiles --------------------------------
template <class Tin>
__global__ void __launch_bounds__(256) image_transpose_kernel(int grid, const Tin* __restrict__ x, Tin* __restrict__ xT) {
  __shared__ Tin tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of threads
  for (int r = ty; r < 32; r += 8) {
    const int gy = by + r, gx = bx + tx;
    if (gy < grid && gx < grid) tile[r][tx] = x[(long long)gy * grid + gx];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int gx = bx + r, gy = by + tx;  // output row = original column
    if (gx < grid && gy < grid) xT[(long long)gx * grid + gy] = tile[tx][r];
  }
}

// ---- blocked sinogram layout for the A^T gathers --------------------------------
// A^T's columns are rays r = angle*n_bins + bin.  The 32 lanes of an 8x4 pixel
// tile drift apart in angle as they step through their rows, so in ray order
// one gather touches ~16 lines.  In the blocked layout a 128-byte line holds an
// (ab angles x bb bins) block, and the same gather touches ~9 lines
// (tools/ab_spmv.py; the sum order is unchanged, only the gather address).
// SinoBlk (the blocked sinogram layout) lives in hs_common.cuh

__global__ void sino_block_cols_kernel(long long n, SinoBlk B, int* __restrict__ col) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    col[i] = (int)B.map(col[i]);
}

template <class Tin>
__global__ void sino_block_kernel(long long m, SinoBlk B, const Tin* __restrict__ y, Tin* __restrict__ yb) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    yb[B.map(i)] = y[i];
}

// Choose, per slice, the image layout in which the 32 lanes' gathers touch
// the fewest 128-byte lines (sampled at 8 depths), and remap the slice's
// column indices r*grid + c -> c*grid + r when the transposed layout wins.
// (Adjacent rays entering through the left/right edge differ in y at equal
// depth -> transposed; through the bottom edge they differ in x -> row-major.)
__global__ void sell_transpose_cols_kernel(long long nslices, long long rows, int n_bins, int grid,
                                           const double* __restrict__ cos_t, const double* __restrict__ sin_t,
                                           const long long* __restrict__ sptr, const int* __restrict__ rlen,
                                           int* __restrict__ col, unsigned char* __restrict__ sflag) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  (void)n_bins;
  (void)cos_t;
  (void)sin_t;
  const int lane = threadIdx.x & 31;
  const long long row = s * 32 + lane;
  const int len = row < rows ? rlen[row] : 0;
  const long long base = sptr[s];
  const int slots = (int)((sptr[s + 1] - base) >> 5);  // entries per row incl. padding
  int lines_row = 0, lines_t = 0;
  for (int k = 0; k < 8; ++k) {
    const int e = (int)(((long long)slots * (2 * k + 1)) / 16);
    const bool has = e < len;
    const unsigned act = __ballot_sync(0xffffffffu, has);
    if (act == 0) continue;
    int c = 0;
    if (has) c = col[base + (long long)(e >> 2) * 128 + lane * 4 + (e & 3)];
    const int lr = has ? (c >> 5) : -1 - lane;
    const int lt = has ? (((c % grid) * grid + (c / grid)) >> 5) : -1 - lane;
    const unsigned mr = __match_any_sync(0xffffffffu, lr);
    const unsigned mt = __match_any_sync(0xffffffffu, lt);
    // leaders (lowest lane of each group) count distinct lines
    lines_row += __popc(__ballot_sync(0xffffffffu, has && (__ffs(mr) - 1) == lane));
    lines_t += __popc(__ballot_sync(0xffffffffu, has && (__ffs(mt) - 1) == lane));
  }
  const bool use_t = lines_t < lines_row;
  if (lane == 0) sflag[s] = use_t ? 1 : 0;
  if (!use_t || n_bins < 0) return;  // n_bins < 0: choose only (columns stay in image order)
  for (long long p = sptr[s] + lane; p < sptr[s + 1]; p += 32) {
    const int c = col[p];
    col[p] = (c % grid) * grid + (c / grid);
  }
}

// ---- 16-bit column deltas -------------------------------------------------------
// Consecutive entries of a tomography row are neighbouring pixels (or rays), so
// the column stream is stored as int16 differences plus one int32 base per
// row: 6 instead of 8 bytes per nonzero from HBM.  Decoding is a running
// integer sum per lane; values and the summation order are untouched.

__global__ void sell_delta_range_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                                        const int* __restrict__ rlen, const int* __restrict__ col,
                                        unsigned int* __restrict__ maxabs) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long row = s * 32 + lane;
  const int len = row < rows ? rlen[row] : 0;
  const long long base = sptr[s];
  unsigned int mx = 0;
  int prev = 0;
  for (int e = 0; e < len; ++e) {
    const int c = col[base + (long long)(e >> 2) * 128 + lane * 4 + (e & 3)];
    if (e > 0) {
      const long long d = (long long)c - prev;
      const unsigned int a = (unsigned int)(d < 0 ? -d : d);
      mx = a > mx ? a : mx;
    }
    prev = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) atomicMax(maxabs, mx);
}

__global__ void sell_delta_fill_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                                       const int* __restrict__ rlen, const int* __restrict__ col,
                                       int* __restrict__ rbase, short* __restrict__ dcol) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long row = s * 32 + lane;
  const int len = row < rows ? rlen[row] : 0;
  const long long base = sptr[s];
  const int nslots = (int)((sptr[s + 1] - base) >> 7) * 4;
  int prev = 0;
  for (int e = 0; e < nslots; ++e) {
    const long long slot = base + (long long)(e >> 2) * 128 + lane * 4 + (e & 3);
    short d = 0;
    if (e < len) {
      const int c = col[slot];
      if (e == 0) {
        if (row < rows) rbase[row] = c;
      } else {
        d = (short)(c - prev);
      }
      prev = c;
    }
    dcol[slot] = d;
  }
  if (len == 0 && row < rows) rbase[row] = 0;
}

// gather position of image column c: GM 0 = as stored, 1 = transposed with
// grid = 2^sh (m = grid - 1), 2 = transposed, general grid
template <int GM>
__device__ __forceinline__ int gpos(int c, int m, int sh, int grid) {
  if (GM == 0) return c;
  if (GM == 1) return ((c & m) << sh) | (c >> sh);
  return (c % grid) * grid + c / grid;
}

// one full chunk of a lane's row: decode 4 deltas, 4 gathers, 4 ordered adds
template <int GM, class V, class Tin, class T>
__device__ __forceinline__ void d16_chunk(T& acc, int& c, const int2 d, const Chunk4<V>& v, const Tin* __restrict__ x,
                                          int m, int sh, int grid) {
  const int c0 = c + (int)(short)(d.x & 0xffff);
  const int c1 = c0 + (d.x >> 16);
  const int c2 = c1 + (int)(short)(d.y & 0xffff);
  const int c3 = c2 + (d.y >> 16);
  const T x0 = gather_x<T>(x, gpos<GM>(c0, m, sh, grid));
  const T x1 = gather_x<T>(x, gpos<GM>(c1, m, sh, grid));
  const T x2 = gather_x<T>(x, gpos<GM>(c2, m, sh, grid));
  const T x3 = gather_x<T>(x, gpos<GM>(c3, m, sh, grid));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), x0));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), x1));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), x2));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[3]), x3));
  c = c3;
}

template <int GM, class V, class Tin, class T>
__device__ __forceinline__ void d16_tail(T& acc, int c, const int2 d, const Chunk4<V>& v, int rem,
                                         const Tin* __restrict__ x, int m, int sh, int grid) {
  const int c0 = c + (int)(short)(d.x & 0xffff);
  const int c1 = c0 + (d.x >> 16);
  const int c2 = c1 + (int)(short)(d.y & 0xffff);
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), gather_x<T>(x, gpos<GM>(c0, m, sh, grid))));
  if (rem > 1) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), gather_x<T>(x, gpos<GM>(c1, m, sh, grid))));
  if (rem > 2) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), gather_x<T>(x, gpos<GM>(c2, m, sh, grid))));
}

// One lane's row: one chunk of (delta, value) prefetched ahead; the gathers
// are issued as soon as a chunk's columns are decoded.  (Measured: a deeper
// per-lane pipeline, or two alternating register buffers, cost registers,
// i.e. spills or resident warps, and ran 2-3% slower.)
template <int GM, class V, class Tin, class T>
__device__ __forceinline__ T d16_row(const short* __restrict__ dp, const V* __restrict__ vp, int c, int len,
                                     const Tin* __restrict__ x, int m, int sh, int grid) {
  T acc = T(0);
  const int nq = (len + 3) >> 2, nfull = len >> 2;
  if (nq == 0) return acc;
  int2 d = __ldcs(reinterpret_cast<const int2*>(dp));
  Chunk4<V> v = Chunk4<V>::load(vp);
  for (int q = 0; q < nfull; ++q) {
    int2 dn = d;
    Chunk4<V> vn = v;
    if (q + 1 < nq) {
      dn = __ldcs(reinterpret_cast<const int2*>(dp + (long long)(q + 1) * 128));
      vn = Chunk4<V>::load(vp + (long long)(q + 1) * 128);
    }
    d16_chunk<GM>(acc, c, d, v, x, m, sh, grid);
    d = dn;
    v = vn;
  }
  const int rem = len & 3;
  if (rem) d16_tail<GM>(acc, c, d, v, rem, x, m, sh, grid);
  return acc;
}

// Deeper pipeline for operators with few slices (fewer than ~2 per resident
// warp, e.g. config 3): there the kernel is bound by each lane's serial walk
// (one dependent gather round trip per chunk), not by the stream, so chunk
// q+1's gathers are issued before chunk q's adds and the (delta, value)
// stream runs two chunks ahead.  Same products, same order of adds.
template <int GM, class V, class Tin, class T>
__device__ __forceinline__ void d16_gather4(int& c, const int2 d, const Tin* __restrict__ x, int m, int sh, int grid,
                                            T (&g)[4]) {
  const int c0 = c + (int)(short)(d.x & 0xffff);
  const int c1 = c0 + (d.x >> 16);
  const int c2 = c1 + (int)(short)(d.y & 0xffff);
  const int c3 = c2 + (d.y >> 16);
  g[0] = gather_x<T>(x, gpos<GM>(c0, m, sh, grid));
  g[1] = gather_x<T>(x, gpos<GM>(c1, m, sh, grid));
  g[2] = gather_x<T>(x, gpos<GM>(c2, m, sh, grid));
  g[3] = gather_x<T>(x, gpos<GM>(c3, m, sh, grid));
  c = c3;
}

template <int GM, class V, class Tin, class T>
__device__ __forceinline__ T d16_row_deep(const short* __restrict__ dp, const V* __restrict__ vp, int c, int len,
                                          const Tin* __restrict__ x, int m, int sh, int grid) {
  T acc = T(0);
  const int nq = (len + 3) >> 2;
  if (nq == 0) return acc;
  Chunk4<V> v = Chunk4<V>::load(vp);
  T g[4];
  d16_gather4<GM, V, Tin, T>(c, __ldcs(reinterpret_cast<const int2*>(dp)), x, m, sh, grid, g);
  int2 dn = make_int2(0, 0);
  Chunk4<V> vn = v;
  if (nq > 1) {
    dn = __ldcs(reinterpret_cast<const int2*>(dp + 128));
    vn = Chunk4<V>::load(vp + 128);
  }
  for (int q = 0; q < nq; ++q) {
    T gn[4] = {T(0), T(0), T(0), T(0)};
    int2 dnn = dn;
    Chunk4<V> vnn = vn;
    if (q + 1 < nq) {
      d16_gather4<GM, V, Tin, T>(c, dn, x, m, sh, grid, gn);  // padding deltas are 0: valid addresses
      if (q + 2 < nq) {
        dnn = __ldcs(reinterpret_cast<const int2*>(dp + (long long)(q + 2) * 128));
        vnn = Chunk4<V>::load(vp + (long long)(q + 2) * 128);
      }
    }
    const int nv = min(4, len - 4 * q);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < nv) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[i]), g[i]));
#pragma unroll
    for (int i = 0; i < 4; ++i) g[i] = gn[i];
    v = vn;
    vn = vnn;
    dn = dnn;
  }
  return acc;
}

// Group pipeline of depth U (U >= 2) for operators with far fewer slices than
// warp slots (config 3): the kernel time is the longest slice's walk, one
// gather round trip per step, so each step covers U chunks: the gathers of
// group g+1 (4U loads) are in flight while group g is added, and the stream
// runs two groups ahead.  Registers grow ~22U per thread, which costs nothing
// when resident warps outnumber the slices.  Same products, same add order.
template <int GM, int U, class V, class Tin, class T>
__device__ __forceinline__ void d16_group_gather(int& c, const int2 (&d)[U], int q0, int nq,
                                                 const Tin* __restrict__ x, int m, int sh, int grid, T (&g)[U][4]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (q0 + u < nq) {
      const int c0 = c + (int)(short)(d[u].x & 0xffff);
      const int c1 = c0 + (d[u].x >> 16);
      const int c2 = c1 + (int)(short)(d[u].y & 0xffff);
      const int c3 = c2 + (d[u].y >> 16);
      g[u][0] = gather_x<T>(x, gpos<GM>(c0, m, sh, grid));
      g[u][1] = gather_x<T>(x, gpos<GM>(c1, m, sh, grid));
      g[u][2] = gather_x<T>(x, gpos<GM>(c2, m, sh, grid));
      g[u][3] = gather_x<T>(x, gpos<GM>(c3, m, sh, grid));
      c = c3;
    }
  }
}

template <int U>
__device__ __forceinline__ void d16_group_dload(const short* __restrict__ dp, int q0, int nq, int2 (&d)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (q0 + u < nq) d[u] = __ldcs(reinterpret_cast<const int2*>(dp + (long long)(q0 + u) * 128));
}

template <int U, class V>
__device__ __forceinline__ void d16_group_vload(const V* __restrict__ vp, int q0, int nq, Chunk4<V> (&v)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (q0 + u < nq) v[u] = Chunk4<V>::load(vp + (long long)(q0 + u) * 128);
}

// deltas run two groups ahead, values and gathers one group ahead
template <int GM, int U, class V, class Tin, class T>
__device__ __forceinline__ T d16_row_pipe(const short* __restrict__ dp, const V* __restrict__ vp, int c, int len,
                                          const Tin* __restrict__ x, int m, int sh, int grid) {
  T acc = T(0);
  const int nq = (len + 3) >> 2;
  if (nq == 0) return acc;
  const int ng = (nq + U - 1) / U;
  int2 dA[U], dB[U];
  Chunk4<V> vC[U];
  T gC[U][4];
  d16_group_dload<U>(dp, 0, nq, dA);
  d16_group_vload<U, V>(vp, 0, nq, vC);
  d16_group_gather<GM, U, V, Tin, T>(c, dA, 0, nq, x, m, sh, grid, gC);
  if (ng > 1) d16_group_dload<U>(dp, U, nq, dA);
#pragma unroll 1
  for (int gi = 0; gi < ng; ++gi) {
    if (gi + 2 < ng) d16_group_dload<U>(dp, (gi + 2) * U, nq, dB);
    T gN[U][4];
    Chunk4<V> vN[U];
    if (gi + 1 < ng) {
      d16_group_vload<U, V>(vp, (gi + 1) * U, nq, vN);
      d16_group_gather<GM, U, V, Tin, T>(c, dA, (gi + 1) * U, nq, x, m, sh, grid, gN);
    }
    const int e0 = gi * U * 4;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (e0 + u * 4 + i < len) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(vC[u].v[i]), gC[u][i]));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vC[u] = vN[u];
      dA[u] = dB[u];
#pragma unroll
      for (int i = 0; i < 4; ++i) gC[u][i] = gN[u][i];
    }
  }
  return acc;
}

// Variant of d16_row without the predicated prefetch: the next chunk's index is
// clamped to the row's last chunk, so the (delta, value) loads are
// unconditional and, with the loop unrolled twice, the two register buffers
// alternate instead of being copied every chunk.  Same products and adds.
template <int GM, class V, class Tin, class T>
__device__ __forceinline__ T d16_row_u2(const short* __restrict__ dp, const V* __restrict__ vp, int c, int len,
                                        const Tin* __restrict__ x, int m, int sh, int grid) {
  T acc = T(0);
  const int nq = (len + 3) >> 2, nfull = len >> 2;
  if (nq == 0) return acc;
  int2 d = __ldcs(reinterpret_cast<const int2*>(dp));
  Chunk4<V> v = Chunk4<V>::load(vp);
#pragma unroll 2
  for (int q = 0; q < nfull; ++q) {
    const long long qn = min(q + 1, nq - 1);
    const int2 dn = __ldcs(reinterpret_cast<const int2*>(dp + qn * 128));
    const Chunk4<V> vn = Chunk4<V>::load(vp + qn * 128);
    d16_chunk<GM>(acc, c, d, v, x, m, sh, grid);
    d = dn;
    v = vn;
  }
  const int rem = len & 3;
  if (rem) d16_tail<GM>(acc, c, d, v, rem, x, m, sh, grid);
  return acc;
}

// ---- implicit column indices for the rays of a tomography A ---------------------
// A row of A is a parallel-beam ray; its stored columns (sorted, canonical
// CSR) are the pixels the ray crosses, image row by image row.  In image row
// ry the ray covers the x-interval [xl, xh] (the band ry <= y <= ry + 1,
// clipped to the image), so its pixels are floor(xl + eps) .. ceil(xh - eps) - 1
// (eps = 1e-9 drops corner touches, as the builder's 1e-12 length gate does).
// RayGen walks that sequence with a few fp64 operations per image row, so the
// SpMV streams only the values: 4 B per nonzero instead of 6.  The rule is
// not the builder's arithmetic, so it is checked against the stored columns of
// every row at build time (tomo_implicit_check_kernel) and a slice uses it only
// if all 32 of its rows match exactly (rays through grid corners, e.g. every
// ray of the 90-degree angle, keep their stored 16-bit deltas).  Entry order,
// products and adds are unchanged: bit-identical.
struct RayTab {
  const double* cos_t;
  const double* sin_t;
  const double* offsets;
  int n_bins, grid;
  long long row_offset;  // global ray index of local row 0 (row-sharded A)
};

constexpr double kRayEps = 1e-9;

struct RayGen {
  double ox, oy, mslope, y0, y1;
  int ry, ry_end, cx, hi, grid, mode;  // mode 0: general, 1: one image row, 2: one image column
  __device__ __forceinline__ bool row_range(int r) {
    // explicit roundings (no contraction choices left to the compiler), so
    // the build-time check and the SpMV see the same columns
    const double ylo = fmax((double)r, y0), yhi = fmin((double)(r + 1), y1);
    const double xa = fma(__dsub_rn(ylo, oy), mslope, ox), xb = fma(__dsub_rn(yhi, oy), mslope, ox);
    const double xl = fmax(0.0, fmin(xa, xb)), xh = fmin((double)grid, fmax(xa, xb));
    if (!(xh > xl)) return false;
    cx = (int)floor(__dadd_rn(xl, kRayEps));
    hi = (int)ceil(__dsub_rn(xh, kRayEps)) - 1;
    return hi >= cx;
  }
  // the first image row with pixels at or after r (ry = ry_end + 1 when none)
  __device__ __forceinline__ void seek(int r) {
    ry = r;
    if (mode == 0) {
      while (ry <= ry_end && !row_range(ry)) ++ry;
    } else if (mode == 1) {
      cx = 0;
      hi = grid - 1;
    } else {
      cx = hi = (int)floor(ox);
    }
  }
  __device__ __forceinline__ void init(const RayTab& tb, long long row) {
    const long long r = row + tb.row_offset;
    const int a = (int)(r / tb.n_bins), j = (int)(r - (long long)a * tb.n_bins);
    grid = tb.grid;
    const double ct = tb.cos_t[a], st = tb.sin_t[a], s = tb.offsets[j];
    const double half = (double)grid / 2.0;
    ox = __dadd_rn(half, __dmul_rn(s, -st));
    oy = __dadd_rn(half, __dmul_rn(s, ct));
    ry = 0;
    ry_end = -1;
    mode = 0;
    mslope = y0 = y1 = 0.0;
    if (fabs(st) < 1e-12) {  // horizontal ray: one image row
      if (oy > 0.0 && oy < (double)grid) { mode = 1; ry = ry_end = (int)floor(oy); }
    } else if (fabs(ct) < 1e-12) {  // vertical ray: one image column
      if (ox > 0.0 && ox < (double)grid) { mode = 2; ry = 0; ry_end = grid - 1; }
    } else {
      mslope = __ddiv_rn(ct, st);
      const double ya = __dadd_rn(oy, __ddiv_rn(__dsub_rn(0.0, ox), mslope));
      const double yb = __dadd_rn(oy, __ddiv_rn(__dsub_rn((double)grid, ox), mslope));
      y0 = fmax(0.0, fmin(ya, yb));
      y1 = fmin((double)grid, fmax(ya, yb));
      if (y1 > y0) {
        ry = (int)floor(__dadd_rn(y0, kRayEps));
        ry_end = (int)ceil(__dsub_rn(y1, kRayEps)) - 1;
      }
    }
    seek(ry);
  }
  __device__ __forceinline__ bool done() const { return ry > ry_end; }
  // the current column, then advance
  __device__ __forceinline__ int next() {
    const int c = ry * grid + cx;
    if (cx < hi) ++cx;
    else seek(ry + 1);
    return c;
  }
};

// build-time check: bad[s] != 0 when any row of slice s differs from RayGen
// (one thread per slot; rows in natural order: A has no slot permutation)
__global__ void tomo_implicit_check_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                                           const int* __restrict__ rlen, const int* __restrict__ col, RayTab tb,
                                           unsigned char* __restrict__ bad) {
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nslices * 32) return;
  const long long sl = slot >> 5;
  const int lane = (int)(slot & 31);
  const int len = rlen[slot];
  bool ok = true;
  if (slot < rows) {
    RayGen g;
    g.init(tb, slot);
    const long long base = sptr[sl];
    for (int e = 0; e < len && ok; ++e) {
      if (g.done()) { ok = false; break; }
      ok = g.next() == col[base + (long long)(e >> 2) * 128 + lane * 4 + (e & 3)];
    }
    ok = ok && g.done();
  } else {
    ok = len == 0;
  }
  if (!ok) bad[sl] = 1;
}

template <int GM, class V, class Tin, class T>
__device__ __forceinline__ void imp_chunk(T& acc, RayGen& rg, const Chunk4<V>& v, const Tin* __restrict__ x, int m,
                                          int sh, int grid) {
  const int c0 = rg.next(), c1 = rg.next(), c2 = rg.next(), c3 = rg.next();
  const T x0 = gather_x<T>(x, gpos<GM>(c0, m, sh, grid));
  const T x1 = gather_x<T>(x, gpos<GM>(c1, m, sh, grid));
  const T x2 = gather_x<T>(x, gpos<GM>(c2, m, sh, grid));
  const T x3 = gather_x<T>(x, gpos<GM>(c3, m, sh, grid));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), x0));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), x1));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), x2));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[3]), x3));
}

// one lane's row with implicit columns (the value stream only; the d16_row_u2 schedule)
template <int GM, class V, class Tin, class T>
__device__ __forceinline__ T imp_row(const V* __restrict__ vp, RayGen rg, int len, const Tin* __restrict__ x, int m,
                                     int sh, int grid) {
  T acc = T(0);
  const int nq = (len + 3) >> 2, nfull = len >> 2;
  if (nq == 0) return acc;
  Chunk4<V> v = Chunk4<V>::load(vp);
#pragma unroll 2
  for (int q = 0; q < nfull; ++q) {
    const long long qn = min(q + 1, nq - 1);
    const Chunk4<V> vn = Chunk4<V>::load(vp + qn * 128);
    imp_chunk<GM>(acc, rg, v, x, m, sh, grid);
    v = vn;
  }
  const int rem = len & 3;
  if (rem) {
    const int c0 = rg.next();
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), gather_x<T>(x, gpos<GM>(c0, m, sh, grid))));
    if (rem > 1) {
      const int c1 = rg.next();
      acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), gather_x<T>(x, gpos<GM>(c1, m, sh, grid))));
    }
    if (rem > 2) {
      const int c2 = rg.next();
      acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), gather_x<T>(x, gpos<GM>(c2, m, sh, grid))));
    }
  }
  return acc;
}

// d16 SpMV of a tomography A where the slices flagged in imp[] regenerate
// their columns (RayGen) instead of reading the 16-bit deltas
template <class V, class Tin, class T, bool POW2, int MINB>
__global__ void __launch_bounds__(256, MINB)
sell_spmv_imp_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                     const int* __restrict__ rlen, const int* __restrict__ rbase, const short* __restrict__ dcol,
                     const V* __restrict__ val, const Tin* __restrict__ xrow, const Tin* __restrict__ xT,
                     const unsigned char* __restrict__ sflag, const unsigned char* __restrict__ imp, RayTab tb,
                     int gshift, const int* __restrict__ sorder, unsigned int* __restrict__ sched,
                     T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int grid = tb.grid;
  for (;;) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&sched[0], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nslices) break;
    const long long s = sorder ? (long long)sorder[i] : (long long)i;
    const bool tr = sflag != nullptr && sflag[s];
    const bool im = imp[s] != 0;  // warp-uniform
    const long long slot = s * 32 + lane;
    const int len = rlen[slot];
    const long long base = sptr[s];
    const V* vp = val + base + lane * 4;
    T acc;
    if (im) {
      RayGen rg;
      rg.init(tb, slot < rows ? slot : 0);
      if (!tr) acc = imp_row<0, V, Tin, T>(vp, rg, len, xrow, 0, 0, grid);
      else if (POW2) acc = imp_row<1, V, Tin, T>(vp, rg, len, xT, grid - 1, gshift, grid);
      else acc = imp_row<2, V, Tin, T>(vp, rg, len, xT, 0, 0, grid);
    } else {
      const short* dp = dcol + base + lane * 4;
      const int c = rbase[slot];
      if (!tr) acc = d16_row_u2<0, V, Tin, T>(dp, vp, c, len, xrow, 0, 0, grid);
      else if (POW2) acc = d16_row_u2<1, V, Tin, T>(dp, vp, c, len, xT, grid - 1, gshift, grid);
      else acc = d16_row_u2<2, V, Tin, T>(dp, vp, c, len, xT, 0, 0, grid);
    }
    if (slot < rows) y[slot] = acc;
  }
  if (lane == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&sched[1], 1u);
    if (done == gridDim.x * (blockDim.x >> 5) - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

template <class V, class Tin, class T, bool POW2, int DEPTH = 0>
#ifndef HS_D16_MINB
#define HS_D16_MINB 6
#endif
__global__ void __launch_bounds__(256, (DEPTH == 0 || DEPTH == 3) ? ((sizeof(T) == 4 && sizeof(V) == 4) ? HS_D16_MINB : 3)
                                       : DEPTH == 1 ? ((sizeof(T) == 4 && sizeof(V) == 4) ? 4 : 2)
                                       : DEPTH == 2 ? 2 : 1)
sell_spmv_d16_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                     const int* __restrict__ rlen, const int* __restrict__ rbase, const short* __restrict__ dcol,
                     const V* __restrict__ val, const Tin* __restrict__ xrow, const Tin* __restrict__ xT,
                     const unsigned char* __restrict__ sflag, int grid, int gshift, const int* __restrict__ rperm,
                     const int* __restrict__ sorder, unsigned int* __restrict__ sched, T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  // dynamic slice scheduling, longest slices first (sorder): each warp takes
  // the next slice from a global counter, so the kernel has no long tail
  for (;;) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&sched[0], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nslices) break;
    const long long s = sorder ? (long long)sorder[i] : (long long)i;
    const bool tr = sflag != nullptr && sflag[s];  // warp-uniform: one specialised row loop each
    const long long slot = s * 32 + lane;  // rlen / rbase are slot-indexed; rperm maps slot -> row
    const long long row = rperm ? (long long)rperm[slot] : slot;
    const int len = rlen[slot];
    const int c = rbase[slot];
    const long long base = sptr[s];
    const short* dp = dcol + base + lane * 4;
    const V* vp = val + base + lane * 4;
    T acc;
    if constexpr (DEPTH == 3) {
      if (!tr) acc = d16_row_u2<0, V, Tin, T>(dp, vp, c, len, xrow, 0, 0, grid);
      else if (POW2) acc = d16_row_u2<1, V, Tin, T>(dp, vp, c, len, xT, grid - 1, gshift, grid);
      else acc = d16_row_u2<2, V, Tin, T>(dp, vp, c, len, xT, 0, 0, grid);
    } else if constexpr (DEPTH >= 2) {
      if (!tr) acc = d16_row_pipe<0, DEPTH, V, Tin, T>(dp, vp, c, len, xrow, 0, 0, grid);
      else if (POW2) acc = d16_row_pipe<1, DEPTH, V, Tin, T>(dp, vp, c, len, xT, grid - 1, gshift, grid);
      else acc = d16_row_pipe<2, DEPTH, V, Tin, T>(dp, vp, c, len, xT, 0, 0, grid);
    } else if constexpr (DEPTH == 1) {
      if (!tr) acc = d16_row_deep<0, V, Tin, T>(dp, vp, c, len, xrow, 0, 0, grid);
      else if (POW2) acc = d16_row_deep<1, V, Tin, T>(dp, vp, c, len, xT, grid - 1, gshift, grid);
      else acc = d16_row_deep<2, V, Tin, T>(dp, vp, c, len, xT, 0, 0, grid);
    } else {
      if (!tr) acc = d16_row<0, V, Tin, T>(dp, vp, c, len, xrow, 0, 0, grid);
      else if (POW2) acc = d16_row<1, V, Tin, T>(dp, vp, c, len, xT, grid - 1, gshift, grid);
      else acc = d16_row<2, V, Tin, T>(dp, vp, c, len, xT, 0, 0, grid);
    }
    if (row >= 0 && row < rows) y[row] = acc;
  }
  // the last warp out resets the scheduler for the next launch
  if (lane == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&sched[1], 1u);
    if (done == gridDim.x * (blockDim.x >> 5) - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// ---- 16-bit deltas + dominant-value flags ("d16v") --------------------------------
// A parallel-beam ray crosses most pixels of its path wall to wall, and every
// such crossing has the same chord length, 1/max(|cos|, |sin|): about 41% of a
// row's fp32 values are bitwise equal to the row's most frequent value.  The
// d16v encoding keeps the 16-bit column deltas, steals their low bit as a flag
// "value == the row's dominant value fv[slot]", and stores only the other
// (explicit) values, compacted per slice chunk row in slot order (lane-major,
// then entry).  A warp recovers each lane's offset into that stream with four
// ballots.  The flag is set only on bitwise equality, so every product and
// every add of the row sum is the one the d16 kernel makes: bit-identical.
// Padding slots carry flag 1 (no explicit value) and delta 0.

// fv per slot = mode of the row's first (up to) 32 values; explicit count and
// the largest |delta| per slice
template <class V>
__global__ void sell_dominant_kernel(long long nslots, long long nslices, const long long* __restrict__ sptr,
                                     const int* __restrict__ rlen, const short* __restrict__ dcol,
                                     const V* __restrict__ val, V* __restrict__ fv, long long* __restrict__ nexp,
                                     unsigned int* __restrict__ maxabs) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long slot = s * 32 + lane;
  const int len = slot < nslots ? rlen[slot] : 0;
  const long long base = sptr[s];
  auto at = [&](int e) { return base + (long long)(e >> 2) * 128 + lane * 4 + (e & 3); };
  const int K = len < 32 ? len : 32;
  V best = V(0);
  int bestc = 0;
  for (int i = 0; i < K; ++i) {
    const V vi = val[at(i)];
    int c = 0;
    for (int j = 0; j < K; ++j) c += (val[at(j)] == vi && signbit(val[at(j)]) == signbit(vi)) ? 1 : 0;
    if (c > bestc) { bestc = c; best = vi; }
  }
  if (slot < nslots) fv[slot] = best;
  long long ne = 0;
  unsigned int mx = 0;
  for (int e = 0; e < len; ++e) {
    const V v = val[at(e)];
    ne += (v == best && signbit(v) == signbit(best)) ? 0 : 1;
    const int d = dcol[at(e)];
    const unsigned int a = (unsigned int)(d < 0 ? -d : d);
    mx = a > mx ? a : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ne += __shfl_xor_sync(0xffffffffu, ne, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    nexp[s] = ne;
    atomicMax(maxabs, mx);
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// flag-shifted deltas in place; explicit values compacted to out[vptr[s] + ...]
template <class V>
__global__ void sell_d16v_fill_kernel(long long nslots, long long nslices, const long long* __restrict__ sptr,
                                      const int* __restrict__ rlen, short* __restrict__ dcol, const V* __restrict__ val,
                                      const V* __restrict__ fv, const long long* __restrict__ vptr, V* __restrict__ out) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long slot = s * 32 + lane;
  const int len = slot < nslots ? rlen[slot] : 0;
  const V f = slot < nslots ? fv[slot] : V(0);
  const long long base = sptr[s];
  const int nq = (int)((sptr[s + 1] - base) >> 7);
  const unsigned lt = lanemask_lt();
  long long run = vptr[s];
  for (int q = 0; q < nq; ++q) {
    const long long p = base + (long long)q * 128 + lane * 4;
    bool ex[4];
    unsigned b[4];
    int off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = q * 4 + i;
      const V v = e < len ? val[p + i] : V(0);
      ex[i] = e < len && !(v == f && signbit(v) == signbit(f));
      b[i] = __ballot_sync(0xffffffffu, ex[i]);
      off += __popc(b[i] & lt);
      tot += __popc(b[i]);
    }
    int k = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = q * 4 + i;
      const int d = e < len ? (int)dcol[p + i] : 0;
      dcol[p + i] = (short)((d << 1) | (ex[i] ? 0 : 1));
      if (ex[i]) out[run + off + k++] = val[p + i];
    }
    run += tot;
  }
}

// one chunk's flags -> explicit-value loads from the slice's compacted stream
// (p = this lane's first explicit value of the chunk); flagged entries take fv
__device__ __forceinline__ void d16v_vload(const int2 d, const float* __restrict__ p, float fv, float (&v)[4]) {
  const bool e0 = !(d.x & 1), e1 = !((d.x >> 16) & 1), e2 = !(d.y & 1), e3 = !((d.y >> 16) & 1);
  v[0] = e0 ? __ldcs(p) : fv;
  p += e0;
  v[1] = e1 ? __ldcs(p) : fv;
  p += e1;
  v[2] = e2 ? __ldcs(p) : fv;
  p += e2;
  v[3] = e3 ? __ldcs(p) : fv;
}

// offsets of this lane's explicit values within the chunk row, and the chunk row's total
__device__ __forceinline__ void d16v_offsets(const int2 d, unsigned lt, int& off, int& tot) {
  const unsigned b0 = __ballot_sync(0xffffffffu, !(d.x & 1));
  const unsigned b1 = __ballot_sync(0xffffffffu, !((d.x >> 16) & 1));
  const unsigned b2 = __ballot_sync(0xffffffffu, !(d.y & 1));
  const unsigned b3 = __ballot_sync(0xffffffffu, !((d.y >> 16) & 1));
  off = __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
  tot = __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
}

template <int GM, class Tin, class T>
__device__ __forceinline__ void d16v_chunk(T& acc, int& c, const int2 d, const float (&v)[4], int nv,
                                           const Tin* __restrict__ x, int m, int sh, int grid) {
  const int c0 = c + ((int)(short)(d.x & 0xffff) >> 1);
  const int c1 = c0 + (d.x >> 17);
  const int c2 = c1 + ((int)(short)(d.y & 0xffff) >> 1);
  const int c3 = c2 + (d.y >> 17);
  if (nv >= 4) {
    const T x0 = gather_x<T>(x, gpos<GM>(c0, m, sh, grid));
    const T x1 = gather_x<T>(x, gpos<GM>(c1, m, sh, grid));
    const T x2 = gather_x<T>(x, gpos<GM>(c2, m, sh, grid));
    const T x3 = gather_x<T>(x, gpos<GM>(c3, m, sh, grid));
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v[0]), x0));
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v[1]), x1));
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v[2]), x2));
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v[3]), x3));
  } else if (nv > 0) {
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v[0]), gather_x<T>(x, gpos<GM>(c0, m, sh, grid))));
    if (nv > 1) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v[1]), gather_x<T>(x, gpos<GM>(c1, m, sh, grid))));
    if (nv > 2) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v[2]), gather_x<T>(x, gpos<GM>(c2, m, sh, grid))));
  }
  c = c3;
}

// The warp walks every chunk row of its slice (the ballots need all lanes);
// deltas run two chunks ahead, explicit values one chunk ahead.
template <int GM, class Tin, class T>
__device__ __forceinline__ T d16v_slice_row(const short* __restrict__ dp, const float* __restrict__ vs, float fv,
                                            int c, int len, int nqs, const Tin* __restrict__ x, int m, int sh,
                                            int grid) {
  T acc = T(0);
  if (nqs == 0) return acc;
  const unsigned lt = lanemask_lt();
  int2 d = __ldcs(reinterpret_cast<const int2*>(dp));
  int2 dn = __ldcs(reinterpret_cast<const int2*>(dp + (long long)min(1, nqs - 1) * 128));
  int off, tot;
  d16v_offsets(d, lt, off, tot);
  float v[4];
  d16v_vload(d, vs + off, fv, v);
  vs += tot;
#pragma unroll 1
  for (int q = 0; q < nqs; ++q) {
    const int2 dnn = __ldcs(reinterpret_cast<const int2*>(dp + (long long)min(q + 2, nqs - 1) * 128));
    d16v_offsets(dn, lt, off, tot);
    float vn[4];
    d16v_vload(dn, vs + off, fv, vn);  // past the last chunk: dn repeats it, the loads re-read it
    vs += (q + 1 < nqs) ? tot : 0;
    d16v_chunk<GM, Tin, T>(acc, c, d, v, len - 4 * q, x, m, sh, grid);
    d = dn;
    dn = dnn;
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = vn[i];
  }
  return acc;
}

template <class Tin, class T, bool POW2>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 5 : 3)
sell_spmv_d16v_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                      const long long* __restrict__ vptr, const int* __restrict__ rlen, const int* __restrict__ rbase,
                      const short* __restrict__ dcol, const float* __restrict__ val, const float* __restrict__ fv,
                      const Tin* __restrict__ xrow, const Tin* __restrict__ xT, const unsigned char* __restrict__ sflag,
                      int grid, int gshift, const int* __restrict__ rperm, const int* __restrict__ sorder,
                      unsigned int* __restrict__ sched, T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&sched[0], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nslices) break;
    const long long s = sorder ? (long long)sorder[i] : (long long)i;
    const bool tr = sflag != nullptr && sflag[s];
    const long long slot = s * 32 + lane;
    const long long row = rperm ? (long long)rperm[slot] : slot;
    const int len = rlen[slot];
    const int c = rbase[slot];
    const float f = fv[slot];
    const long long base = sptr[s];
    const int nqs = (int)((sptr[s + 1] - base) >> 7);
    const short* dp = dcol + base + lane * 4;
    const float* vs = val + vptr[s];
    T acc;
    if (!tr) acc = d16v_slice_row<0, Tin, T>(dp, vs, f, c, len, nqs, xrow, 0, 0, grid);
    else if (POW2) acc = d16v_slice_row<1, Tin, T>(dp, vs, f, c, len, nqs, xT, grid - 1, gshift, grid);
    else acc = d16v_slice_row<2, Tin, T>(dp, vs, f, c, len, nqs, xT, 0, 0, grid);
    if (row >= 0 && row < rows) y[row] = acc;
  }
  if (lane == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&sched[1], 1u);
    if (done == gridDim.x * (blockDim.x >> 5) - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// ---- 8-bit transition codes (tomography operators) ---------------------------------
// The columns of a tomography row are points (r, c) of a 2D index space that
// a ray (or, for A^T, a pixel's sequence of rays) walks through in small steps:
//   A   : (image row, image column); consecutive entries move right along an
//         image row or step to the next image row (+1 row, small column move);
//   A^T : (angle, detector bin); consecutive entries move to the next bin or
//         to the next angle (+1 angle, small bin move).
// Each entry after the first is one byte (dr << 7) | (dc & 0x7f), dr in {0,1},
// dc in [-64, 63]; anything else (and the reserved byte 0xC0) is an escape
// whose absolute gather address sits in a per-lane exception list.  Stored
// bytes per nonzero: 4 (fp32 value) + 1, against 4 + 2 for 16-bit deltas.
// The decoder keeps the gather ADDRESS, so the per-slice layout choice of A
// (image / transposed image) and the 4-angle interleave of the sinogram for
// A^T cost nothing extra:
//   mode 0: address r*G + c, or c*G + r on transposed slices (G = grid)
//   mode 1: address (r>>2)*4*G + 4*c + (r&3)   (G = n_bins; r&3 kept in bits 30-31 of escapes)
struct C8Geom {
  int mode, G;
  __device__ __forceinline__ int addr(int r, int c, bool tr) const {
    if (mode == 0) return tr ? c * G + r : r * G + c;
    return ((r >> 2) * 4 * G + c * 4 + (r & 3)) | ((r & 3) << 30);
  }
};
constexpr unsigned int C8_ESC = 0xC0u;

// pass 0: codes, first addresses and per-slot escape counts; pass 1: escape lists
__global__ void sell_c8_encode_kernel(long long nslices, const long long* __restrict__ sptr,
                                      const int* __restrict__ rlen, const int* __restrict__ col,
                                      const unsigned char* __restrict__ sflag, C8Geom g, int pass,
                                      unsigned char* __restrict__ code, int* __restrict__ rbase,
                                      int* __restrict__ xcnt, const int* __restrict__ xoff, int* __restrict__ exc) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long slot = s * 32 + lane;
  const int len = rlen[slot];
  const long long base = sptr[s];
  const int ne = (int)((sptr[s + 1] - base) >> 7) * 4;
  const bool tr = g.mode == 0 && sflag != nullptr && sflag[s];
  int pr = 0, pc = 0, nx = 0, xp = pass ? xoff[slot] : 0;
  for (int e = 0; e < ne; ++e) {
    const long long sl = base + (long long)(e >> 2) * 128 + lane * 4 + (e & 3);
    unsigned int b = 0;
    if (e < len) {
      const int cc = col[sl];
      const int r = cc / g.G, c = cc - r * g.G;
      if (e == 0) {
        if (pass == 0) rbase[slot] = g.addr(r, c, tr);
      } else {
        const int dr = r - pr, dc = c - pc;
        if ((dr == 0 || dr == 1) && dc >= -64 && dc <= 63 && !(dr == 1 && dc == -64)) {
          b = ((unsigned)dr << 7) | ((unsigned)dc & 0x7fu);
        } else {
          b = C8_ESC;
          if (pass == 1) exc[xp] = g.addr(r, c, tr);
          ++xp;
          ++nx;
        }
      }
      pr = r;
      pc = c;
    }
    if (pass == 0) code[sl] = (unsigned char)b;
  }
  if (pass == 0) {
    xcnt[slot] = nx;
    if (len == 0) rbase[slot] = 0;
  }
}

template <int MODE>
struct C8Dec {
  int addr, ra, SR, SC;
  __device__ __forceinline__ void init(int a0, bool tr, int G) {
    if (MODE == 0) {
      addr = a0;
      SR = tr ? 1 : G;
      SC = tr ? G : 1;
      ra = 0;
    } else {
      addr = a0 & 0x3fffffff;
      ra = (int)((unsigned)a0 >> 30);
      SR = 4 * G - 3;  // address step when the angle enters the next 4-angle group
      SC = 4;
    }
  }
  // apply byte j of w (not an escape)
  __device__ __forceinline__ void step(unsigned int w, int j) {
    const int dc = ((int)(w << (25 - 8 * j))) >> 25;
    const int dr = (int)((w >> (8 * j + 7)) & 1u);
    if (MODE == 0) {
      addr += dc * SC + (dr ? SR : 0);
    } else {
      ra += dr;
      addr += dc * 4 + (dr ? ((ra & 3) ? 1 : SR) : 0);
    }
  }
  __device__ __forceinline__ void esc(int e) {
    if (MODE == 0) {
      addr = e;
    } else {
      addr = e & 0x3fffffff;
      ra = (int)((unsigned)e >> 30);
    }
  }
  // decode a chunk into four addresses; lanes with pending escapes check each byte
  __device__ __forceinline__ void chunk(unsigned int w, int& xp, int xe, const int* __restrict__ exc, int (&a)[4]) {
    if (xp < xe) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (((w >> (8 * j)) & 0xffu) == C8_ESC) esc(__ldg(exc + xp++));
        else step(w, j);
        a[j] = addr;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        step(w, j);
        a[j] = addr;
      }
    }
  }
};

// SpMV over the 8-bit coded SELL layout.  The (value, code) stream is moved
// by LDGSTS (cp.async): every lane copies its own 16 B of values and 4 B of
// codes per chunk straight into a per-thread NS-deep shared-memory ring, so
// NS-1 chunks per lane are in flight while chunk q is consumed without
// holding registers (a register double buffer holds one and measured 13%
// slower; a TMA bulk-copy ring per warp, 2x the instructions).  Each lane
// reads back only what it copied: no cross-lane hand-off, independent trip
// counts.  Per chunk: decode 4 codes, 4 gathers, 4 ordered multiply-adds.
__device__ __forceinline__ void cpasync16(unsigned dst, const void* src, unsigned long long pol) {
#ifdef HS_CPASYNC_HINT
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol) : "memory");
#else
  (void)pol;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#endif
}
__device__ __forceinline__ void cpasync4(unsigned dst, const void* src, unsigned long long pol) {
#ifdef HS_CPASYNC_HINT
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "l"(pol) : "memory");
#else
  (void)pol;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
#endif
}
__device__ __forceinline__ void cpasync_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpasync_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <class V, int NS>
struct C8Lane {
  static constexpr int VB = 4 * (int)sizeof(V);  // value bytes per lane per chunk
  static constexpr int smem_bytes(int threads) { return NS * threads * (VB + 4); }
};

template <class V, class Tin, class T, int MODE, int NS, int MINB>
__global__ void __launch_bounds__(256, MINB)
sell_spmv_c8_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                     const int* __restrict__ rlen, const int* __restrict__ rbase, const unsigned char* __restrict__ code,
                     const int* __restrict__ xoff, const int* __restrict__ exc, const V* __restrict__ val,
                     const Tin* __restrict__ xrow, const Tin* __restrict__ xT, const unsigned char* __restrict__ sflag,
                     int G, const int* __restrict__ rperm, const int* __restrict__ sorder,
                     unsigned int* __restrict__ sched, T* __restrict__ y) {
  using L = C8Lane<V, NS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  // ring slot st of this thread: values at vs + st*VSTR, code word at cs + st*CSTR
  const unsigned vs = smem_u32(smem_raw) + threadIdx.x * L::VB;
  const unsigned cs = smem_u32(smem_raw) + NS * blockDim.x * L::VB + threadIdx.x * 4;
  const unsigned VSTR = blockDim.x * L::VB, CSTR = blockDim.x * 4;
  const unsigned long long pol = l2_evict_first_policy();
  for (;;) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&sched[0], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nslices) break;
    const long long s = sorder ? (long long)sorder[i] : (long long)i;
    const long long base = sptr[s];
    const long long slot = s * 32 + lane;
    const int len = rlen[slot];
    const int nq = (len + 3) >> 2, nfull = len >> 2;
    const V* vp = val + base + lane * 4;
    const unsigned char* cp = code + base + lane * 4;
    // prologue: chunks 0 .. NS-2
#pragma unroll
    for (int k = 0; k < NS - 1; ++k) {
      if (k < nq) {
        cpasync16(vs + k * VSTR, vp + (long long)k * 128, pol);
        if (sizeof(V) == 8) cpasync16(vs + k * VSTR + 16, vp + (long long)k * 128 + 2, pol);
        cpasync4(cs + k * CSTR, cp + (long long)k * 128, pol);
      }
      cpasync_commit();
    }
    const bool tr = MODE == 0 && sflag != nullptr && sflag[s];
    const Tin* __restrict__ x = tr ? xT : xrow;
    const long long row = rperm ? (long long)rperm[slot] : slot;
    C8Dec<MODE> dec;
    dec.init(rbase[slot], tr, G);
    int xp = xoff[slot];
    const int xe = xoff[slot + 1];
    T acc = T(0);
    int st = 0;
    for (int q = 0; q < nq; ++q) {
      {  // refill the slot consumed last iteration with chunk q + NS - 1
        const int k = q + NS - 1;
        const int sk = st == 0 ? NS - 1 : st - 1;
        if (k < nq) {
          cpasync16(vs + sk * VSTR, vp + (long long)k * 128, pol);
          if (sizeof(V) == 8) cpasync16(vs + sk * VSTR + 16, vp + (long long)k * 128 + 2, pol);
          cpasync4(cs + sk * CSTR, cp + (long long)k * 128, pol);
        }
        cpasync_commit();
      }
      cpasync_wait<NS - 1>();
      const Chunk4<V> v = Chunk4<V>::lds(smem_raw + threadIdx.x * L::VB + st * VSTR);
      const unsigned w = *reinterpret_cast<const unsigned*>(smem_raw + NS * VSTR + threadIdx.x * 4 + st * CSTR);
      st = st + 1 == NS ? 0 : st + 1;
      int a[4];
      dec.chunk(w, xp, xe, exc, a);
      if (q < nfull) {
        const T x0 = gather_x<T>(x, a[0]);
        const T x1 = gather_x<T>(x, a[1]);
        const T x2 = gather_x<T>(x, a[2]);
        const T x3 = gather_x<T>(x, a[3]);
        acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), x0));
        acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), x1));
        acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), x2));
        acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[3]), x3));
      } else {
        const int rem = len & 3;
        acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), gather_x<T>(x, a[0])));
        if (rem > 1) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), gather_x<T>(x, a[1])));
        if (rem > 2) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), gather_x<T>(x, a[2])));
      }
    }
    cpasync_wait<0>();
    if (row >= 0 && row < rows) y[row] = acc;
  }
  if (lane == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&sched[1], 1u);
    if (done == gridDim.x * (blockDim.x >> 5) - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// slice sizes (for the longest-first order)
__global__ void sell_slice_size_kernel(long long nslices, const long long* __restrict__ sptr,
                                       unsigned int* __restrict__ size, int* __restrict__ idx) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  size[s] = (unsigned int)((sptr[s + 1] - sptr[s]) >> 7);
  idx[s] = (int)s;
}

// slot permutation grouping an image's pixels into 8-wide x 4-tall tiles
// (one tile per slice): used for A^T, whose 32 lanes then hit the same few
// detectors at every angle instead of a 32-pixel image row's wider shadow
__global__ void tile_perm_kernel(int grid, long long nslots, int* __restrict__ rperm) {
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nslots) return;
  const int tiles_x = (grid + 7) / 8;
  const long long tile = slot >> 5;
  const int lane = (int)(slot & 31);
  const long long ty = tile / tiles_x, tx = tile % tiles_x;
  const long long r = ty * 4 + (lane >> 3), c = tx * 8 + (lane & 7);
  rperm[slot] = (r < grid && c < grid) ? (int)(r * grid + c) : -1;
}

// ---- 16-bit deltas through a per-lane cp.async ring (latency-bound operators) ----
// For operators with fewer slices than warp slots (config 3; one rank's share
// of config 4 on 8 GPUs) the register-prefetched kernels keep ~25 KB of the
// stream in flight per SM against the ~44 KB the HBM bandwidth-latency
// product needs (ncu: 42-52% of DRAM bandwidth).  Here every lane copies its
// own chunks' 8 B of deltas and 4 x sizeof(V) B of values by LDGSTS into an
// NS-deep per-thread shared-memory ring (NS-1 chunks ahead, no registers
// held), and decodes chunk q+1 and issues its gathers before adding chunk q.
// Same products, same order of adds as d16_row: bit-identical.
__device__ __forceinline__ void cpasync8(unsigned dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

template <class V, int NS>
struct D16Ring {
  static constexpr int VB = 4 * (int)sizeof(V);  // value bytes per lane per chunk
  static constexpr int smem_bytes(int threads) { return NS * threads * (VB + 8); }
};

template <int GM, class V, class Tin, class T, int NS>
__device__ __forceinline__ T d16_row_ring(const short* __restrict__ dp, const V* __restrict__ vp, int c, int len,
                                          const Tin* __restrict__ x, int m, int sh, int grid, unsigned vs,
                                          unsigned ds, unsigned VSTR, unsigned DSTR,
                                          const unsigned char* __restrict__ vsp, const unsigned char* __restrict__ dsp) {
  const int nq = (len + 3) >> 2;
  auto issue = [&](int k, int slot) {
    if (k < nq) {
      cpasync16(vs + slot * VSTR, vp + (long long)k * 128, 0ull);
      if (sizeof(V) == 8) cpasync16(vs + slot * VSTR + 16, vp + (long long)k * 128 + 2, 0ull);
      cpasync8(ds + slot * DSTR, dp + (long long)k * 128);
    }
    cpasync_commit();
  };
#pragma unroll
  for (int k = 0; k < NS - 1; ++k) issue(k, k);
  T acc = T(0);
  if (nq == 0) {
    cpasync_wait<0>();
    return acc;
  }
  // chunk 0: decode and gather
  cpasync_wait<NS - 2>();
  T g[4];
  Chunk4<V> v;
  {
    const int2 d = *reinterpret_cast<const int2*>(dsp);
    const int c0 = c + (int)(short)(d.x & 0xffff), c1 = c0 + (d.x >> 16);
    const int c2 = c1 + (int)(short)(d.y & 0xffff), c3 = c2 + (d.y >> 16);
    c = c3;
    g[0] = gather_x<T>(x, gpos<GM>(c0, m, sh, grid));
    g[1] = gather_x<T>(x, gpos<GM>(c1, m, sh, grid));
    g[2] = gather_x<T>(x, gpos<GM>(c2, m, sh, grid));
    g[3] = gather_x<T>(x, gpos<GM>(c3, m, sh, grid));
    v = Chunk4<V>::lds(vsp);
  }
  for (int q = 0; q < nq; ++q) {
    // refill the slot of chunk q-1 (consumed) with chunk q+NS-1
    issue(q + NS - 1, (q + NS - 1) % NS);
    T gn[4] = {T(0), T(0), T(0), T(0)};
    Chunk4<V> vn = v;
    if (q + 1 < nq) {
      cpasync_wait<NS - 2>();  // chunk q+1 has landed
      const int sl = (q + 1) % NS;
      const int2 d = *reinterpret_cast<const int2*>(dsp + sl * DSTR);
      const int c0 = c + (int)(short)(d.x & 0xffff), c1 = c0 + (d.x >> 16);
      const int c2 = c1 + (int)(short)(d.y & 0xffff), c3 = c2 + (d.y >> 16);
      c = c3;
      gn[0] = gather_x<T>(x, gpos<GM>(c0, m, sh, grid));
      gn[1] = gather_x<T>(x, gpos<GM>(c1, m, sh, grid));
      gn[2] = gather_x<T>(x, gpos<GM>(c2, m, sh, grid));
      gn[3] = gather_x<T>(x, gpos<GM>(c3, m, sh, grid));
      vn = Chunk4<V>::lds(vsp + sl * VSTR);
    }
    const int nv = min(4, len - 4 * q);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < nv) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[i]), g[i]));
#pragma unroll
    for (int i = 0; i < 4; ++i) g[i] = gn[i];
    v = vn;
  }
  cpasync_wait<0>();
  return acc;
}

template <class V, class Tin, class T, bool POW2, int NS, int MINB>
__global__ void __launch_bounds__(256, MINB)
sell_spmv_d16_ring_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                          const int* __restrict__ rlen, const int* __restrict__ rbase, const short* __restrict__ dcol,
                          const V* __restrict__ val, const Tin* __restrict__ xrow, const Tin* __restrict__ xT,
                          const unsigned char* __restrict__ sflag, int grid, int gshift, const int* __restrict__ rperm,
                          const int* __restrict__ sorder, unsigned int* __restrict__ sched, T* __restrict__ y) {
  using L = D16Ring<V, NS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const unsigned VSTR = blockDim.x * L::VB, DSTR = blockDim.x * 8;
  const unsigned vs = smem_u32(smem_raw) + threadIdx.x * L::VB;
  const unsigned ds = smem_u32(smem_raw) + NS * VSTR + threadIdx.x * 8;
  const unsigned char* vsp = smem_raw + threadIdx.x * L::VB;
  const unsigned char* dsp = smem_raw + NS * VSTR + threadIdx.x * 8;
  for (;;) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&sched[0], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nslices) break;
    const long long s = sorder ? (long long)sorder[i] : (long long)i;
    const bool tr = sflag != nullptr && sflag[s];
    const long long slot = s * 32 + lane;
    const long long row = rperm ? (long long)rperm[slot] : slot;
    const int len = rlen[slot];
    const int c = rbase[slot];
    const long long base = sptr[s];
    const short* dp = dcol + base + lane * 4;
    const V* vp = val + base + lane * 4;
    T acc;
    if (!tr)
      acc = d16_row_ring<0, V, Tin, T, NS>(dp, vp, c, len, xrow, 0, 0, grid, vs, ds, VSTR, DSTR, vsp, dsp);
    else if (POW2)
      acc = d16_row_ring<1, V, Tin, T, NS>(dp, vp, c, len, xT, grid - 1, gshift, grid, vs, ds, VSTR, DSTR, vsp, dsp);
    else
      acc = d16_row_ring<2, V, Tin, T, NS>(dp, vp, c, len, xT, 0, 0, grid, vs, ds, VSTR, DSTR, vsp, dsp);
    if (row >= 0 && row < rows) y[row] = acc;
  }
  if (lane == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&sched[1], 1u);
    if (done == gridDim.x * (blockDim.x >> 5) - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// ---- CSR -> SELL-32x4 conversion ------------------------------------------------
// Slot s*32+lane holds row rperm[slot] (or row = slot without a permutation;
// rperm < 0 marks an empty padding slot).  rlen is slot-indexed.
__device__ __forceinline__ long long slot_row(const int* rperm, long long slot, long long rows) {
  const long long r = rperm ? (long long)rperm[slot] : slot;
  return (r >= 0 && r < rows) ? r : -1;
}

// per slice: number of 4-entry chunks of its longest row
__global__ void sell_slice_chunks_kernel(long long rows, long long nslices, const long long* __restrict__ rowptr,
                                         const int* __restrict__ rperm, int* __restrict__ rlen,
                                         long long* __restrict__ slice_slots) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long row = slot_row(rperm, s * 32 + lane, rows);
  int len = 0;
  if (row >= 0) len = (int)(rowptr[row + 1] - rowptr[row]);
  rlen[s * 32 + lane] = len;
  int nq = (len + 3) >> 2;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nq = max(nq, __shfl_xor_sync(0xffffffffu, nq, o));
  if (lane == 0) slice_slots[s] = (long long)nq * 128;
}

template <class V>
__global__ void sell_fill_kernel(long long rows, long long nslices, const long long* __restrict__ rowptr,
                                 const int* __restrict__ rperm, const int* __restrict__ ccol,
                                 const V* __restrict__ cval, const long long* __restrict__ sptr,
                                 int* __restrict__ scol, V* __restrict__ sval) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long row = slot_row(rperm, s * 32 + lane, rows);
  const long long base = sptr[s];
  const int nslots = (int)((sptr[s + 1] - base) >> 7) * 4;  // entries per row incl. padding
  long long r0 = 0;
  int len = 0;
  if (row >= 0) {
    r0 = rowptr[row];
    len = (int)(rowptr[row + 1] - r0);
  }
  for (int e = 0; e < nslots; ++e) {
    const long long slot = base + (long long)(e >> 2) * 128 + lane * 4 + (e & 3);
    if (e < len) {
      scol[slot] = ccol[r0 + e];
      sval[slot] = cval[r0 + e];
    } else {
      scol[slot] = 0;
      sval[slot] = V(0);
    }
  }
}

}  // namespace hs
