// Device builders for the operators of the tomography configs:
//   * the parallel-beam exact-chord system matrix (problems.py:276-331,
//     generalised to n_bins detectors; oracle/tomo_oracle.py), traced one ray
//     per thread with the reference's floating-point operations in the same
//     order so every entry is bit-identical to the reference's CSR;
//   * the row-sorted CSR transpose (scipy's M.T.tocsr() order, linops.py:139).
#pragma once

#include <math_constants.h>

#include "hs_common.cuh"

namespace hs {

struct TomoGeom {
  int grid;
  int n_angles;
  int n_bins;
  const double* cos_t;    // n_angles (host-computed with math.cos, as the reference)
  const double* sin_t;
  const double* offsets;  // n_bins: j + 0.5 - n_bins/2
};

// crossing parameter of grid line k on one axis: (k - o) / d  (problems.py:300)
__device__ __forceinline__ double cross_t(int k, double o, double d) {
  return __ddiv_rn(__dsub_rn((double)k, o), d);
}

// walk state for one axis' crossings in ascending t order, restricted to (t0, t1)
struct AxisWalk {
  bool active;
  int k, step, grid;
  double o, d, t;  // t = current crossing or +inf when exhausted
  __device__ void init(bool act, double o_, double d_, int grid_, double t0, double t1) {
    active = act; o = o_; d = d_; grid = grid_;
    t = CUDART_INF;
    if (!active) return;
    step = d > 0 ? 1 : -1;
    // estimate the first crossing after t0, then fix exactly
    const double p = __dadd_rn(o, __dmul_rn(t0, d));
    long long kk = step > 0 ? (long long)floor(p) + 1 : (long long)ceil(p) - 1;
    if (kk < 1) kk = 1;
    if (kk > grid - 1) kk = grid - 1;
    k = (int)kk;
    // move back while the previous line is still after t0
    while (k - step >= 1 && k - step <= grid - 1 && cross_t(k - step, o, d) > t0) k -= step;
    // move forward while the current line is not after t0
    while (k >= 1 && k <= grid - 1 && !(cross_t(k, o, d) > t0)) k += step;
    load(t1);
  }
  __device__ __forceinline__ void load(double t1) {
    if (k >= 1 && k <= grid - 1) {
      const double tt = cross_t(k, o, d);
      t = (tt < t1) ? tt : CUDART_INF;
    } else {
      t = CUDART_INF;
    }
  }
  __device__ __forceinline__ void advance(double t1) {
    k += step;
    load(t1);
  }
};

// Trace ray (angle a, detector j). Emits (pixel, length) pairs in traversal
// order with consecutive equal pixels merged (scipy sums duplicates).
// Returns the number of emitted entries; `emit(slot, pixel, len)` is called
// with slot = entry index (may be called again for the same slot to update
// the merged length).
template <class Emit>
__device__ int trace_ray(const TomoGeom& G, int a, int j, Emit emit, bool* dx_neg_out) {
  const int grid = G.grid;
  const double ct = G.cos_t[a], stt = G.sin_t[a];
  const double s = G.offsets[j];
  const double half = (double)grid / 2.0;
  // origin = centre + s * normal, normal = (-sin, cos)   (problems.py:321)
  const double ox = __dadd_rn(half, __dmul_rn(s, -stt));
  const double oy = __dadd_rn(half, __dmul_rn(s, ct));
  const double dx = ct, dy = stt;
  *dx_neg_out = dx < 0.0;
  double t0 = -CUDART_INF, t1 = CUDART_INF;
  // problems.py:283-293
  {
    const double o[2] = {ox, oy}, d[2] = {dx, dy};
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      if (fabs(d[ax]) < 1e-12) {
        if (o[ax] <= 0.0 || o[ax] >= (double)grid) return 0;
      } else {
        double ta = __ddiv_rn(__dsub_rn(0.0, o[ax]), d[ax]);
        double tb = __ddiv_rn(__dsub_rn((double)grid, o[ax]), d[ax]);
        if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
        t0 = (ta > t0) ? ta : t0;  // python max(t0, ta)
        t1 = (tb < t1) ? tb : t1;  // python min(t1, tb)
      }
    }
  }
  if (!(t1 > t0)) return 0;
  AxisWalk X, Y;
  X.init(fabs(dx) >= 1e-12, ox, dx, grid, t0, t1);
  Y.init(fabs(dy) >= 1e-12, oy, dy, grid, t0, t1);
  double prev = t0;
  int count = 0;
  long long last_pix = -1;
  double last_len = 0.0;
  bool done = false;
  while (!done) {
    double nxt = fmin(X.t, Y.t);
    if (nxt == CUDART_INF) {
      nxt = t1;
      done = true;
    }
    const double len = __dsub_rn(nxt, prev);
    if (len > 1e-12) {
      const double mt = __dmul_rn(0.5, __dadd_rn(prev, nxt));
      const double mx = __dadd_rn(ox, __dmul_rn(mt, dx));
      const double my = __dadd_rn(oy, __dmul_rn(mt, dy));
      long long ci = (long long)floor(mx), rj = (long long)floor(my);
      ci = ci < 0 ? 0 : (ci > grid - 1 ? grid - 1 : ci);
      rj = rj < 0 ? 0 : (rj > grid - 1 ? grid - 1 : rj);
      const long long pix = rj * grid + ci;
      if (pix == last_pix) {
        last_len = __dadd_rn(last_len, len);
        emit(count - 1, pix, last_len);
      } else {
        emit(count, pix, len);
        last_pix = pix;
        last_len = len;
        ++count;
      }
    }
    if (!done) {
      // np.unique: equal crossings from both axes collapse into one alpha
      const bool ax = (X.t == nxt), ay = (Y.t == nxt);
      if (ax) X.advance(t1);
      if (ay) Y.advance(t1);
    }
    prev = nxt;
  }
  return count;
}

struct NullEmit {
  __device__ void operator()(int, long long, double) const {}
};

// per-ray nnz counts for rays [row_begin, row_end), restricted to pixel
// columns [col_begin, col_end)
__global__ void tomo_count_kernel(TomoGeom G, long long row_begin, long long row_end, long long col_begin,
                                  long long col_end, long long* __restrict__ counts) {
  const long long r = row_begin + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= row_end) return;
  const int a = (int)(r / G.n_bins), j = (int)(r % G.n_bins);
  bool dxneg;
  if (col_begin == 0 && col_end >= (long long)G.grid * G.grid) {
    counts[r - row_begin] = trace_ray(G, a, j, NullEmit{}, &dxneg);
  } else {
    // count only entries inside the column window (merged duplicates counted once)
    struct CountEmit {
      long long cb, ce;
      int* n;
      long long* lastpix;
      __device__ void operator()(int slot, long long pix, double) const {
        (void)slot;
        if (pix >= cb && pix < ce && pix != *lastpix) {
          ++*n;
          *lastpix = pix;
        }
      }
    };
    int n = 0;
    long long lp = -1;
    trace_ray(G, a, j, CountEmit{col_begin, col_end, &n, &lp}, &dxneg);
    counts[r - row_begin] = n;
  }
}

// fill: entries written in traversal order, then each run of equal image row
// is reversed when the ray runs toward -x, giving ascending column order
// within the CSR row (scipy canonical order, problems.py:329-331).
template <class V>
__global__ void tomo_fill_kernel(TomoGeom G, long long row_begin, long long row_end, long long col_begin,
                                 long long col_end, const long long* __restrict__ rowptr, int* __restrict__ col,
                                 V* __restrict__ val) {
  const long long r = row_begin + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= row_end) return;
  const int a = (int)(r / G.n_bins), j = (int)(r % G.n_bins);
  const long long base = rowptr[r - row_begin];
  const long long cnt = rowptr[r - row_begin + 1] - base;
  if (cnt == 0) return;
  int* cp = col + base;
  V* vp = val + base;
  struct FillEmit {
    long long cb, ce;
    int* cp;
    V* vp;
    int* n;
    long long* lastpix;
    __device__ void operator()(int, long long pix, double len) const {
      if (pix < cb || pix >= ce) return;
      if (pix == *lastpix) {
        vp[*n - 1] = (V)len;  // merged duplicate: len is the running sum
      } else {
        cp[*n] = (int)pix;
        vp[*n] = (V)len;
        ++*n;
        *lastpix = pix;
      }
    }
  };
  int n = 0;
  long long lp = -1;
  bool dxneg;
  trace_ray(G, a, j, FillEmit{col_begin, col_end, cp, vp, &n, &lp}, &dxneg);
  if (dxneg) {
    // reverse each run of equal image row (col / grid)
    int s = 0;
    while (s < n) {
      const int rowid = cp[s] / G.grid;
      int e = s + 1;
      while (e < n && cp[e] / G.grid == rowid) ++e;
      for (int lo = s, hi = e - 1; lo < hi; ++lo, --hi) {
        const int tc = cp[lo]; cp[lo] = cp[hi]; cp[hi] = tc;
        const V tv = vp[lo]; vp[lo] = vp[hi]; vp[hi] = tv;
      }
      s = e;
    }
  }
}

// ---- generic CSR transpose pieces ----------------------------------------------
// counts of entries per (local) output row = column of the input in [cb, ce)
__global__ void csr_colcount_kernel(long long rows, const long long* __restrict__ rowptr, const int* __restrict__ col,
                                    long long cb, long long ce, unsigned int* __restrict__ cnt) {
  const long long r = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  for (long long p = rowptr[r] + (threadIdx.x & 31); p < rowptr[r + 1]; p += 32) {
    const long long c = col[p];
    if (c >= cb && c < ce) atomicAdd(&cnt[c - cb], 1u);
  }
}

// scatter (row index -> key, value) into the transposed rows with atomic cursors
template <class V>
__global__ void csr_scatter_kernel(long long rows, long long row_offset, const long long* __restrict__ rowptr,
                                   const int* __restrict__ col, const V* __restrict__ val, long long cb, long long ce,
                                   unsigned long long* __restrict__ cursor, int* __restrict__ tkey, V* __restrict__ tval) {
  const long long r = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  for (long long p = rowptr[r] + (threadIdx.x & 31); p < rowptr[r + 1]; p += 32) {
    const long long c = col[p];
    if (c >= cb && c < ce) {
      const unsigned long long dst = atomicAdd(&cursor[c - cb], 1ull);
      tkey[dst] = (int)(r + row_offset);
      tval[dst] = val[p];
    }
  }
}

__global__ void u32_to_i64_kernel(long long n, const unsigned int* __restrict__ a, long long* __restrict__ b) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void i64_to_u64_kernel(long long n, const long long* __restrict__ a, unsigned long long* __restrict__ b) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (unsigned long long)a[i];
}

}  // namespace hs
