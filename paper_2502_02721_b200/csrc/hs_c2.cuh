// 2-bit step codes for the rays of a tomography A ("c2"): 4.25 instead of 6
// bytes per nonzero on the forward SpMV, entry order and sums untouched.
//
// A row of A (linops.py:137-141: canonical CSR, scipy csr_matvec order) is a
// parallel-beam ray, and its sorted columns are the pixels it crosses image
// row by image row.  Between consecutive entries the pixel either moves one
// step in x inside the image row, or drops to the next image row with an x
// shift that, for every ray of one angle, takes one of two or three adjacent
// values (floor(f - 2 tan) for a ray running against the column order, 0 or 1
// for one running with it).  So a slice of 32 adjacent rays needs four steps:
//   code 0: (dy, dx) = (0, +1)        codes 1..3: (dy, dx) = (+1, j0 + code - 1)
// with one j0 per slice.  The few steps that are not in the table -- the
// first / last image row of a ray clipped by the left or right image edge --
// are escapes: the entry carries code 1 and a per-row (position, correction)
// pair fixes its address; a slice with a row that needs more than two escapes
// keeps its 16-bit deltas (d16 fallback, same kernel).
//
// The codes are decoded in GATHER space: the step table holds address
// increments in the slice's gather layout (image, or transposed image for the
// slices flagged in sflag), so the transposed slices need no per-entry index
// arithmetic.  Two codes (one nibble) index a 16-entry per-warp shared-memory
// table of (step_1, step_1 + step_2): one conflict-free LDS.64 per two
// entries (16 entries x 8 B cover the 32 banks exactly; equal nibbles
// broadcast).  One byte per lane per chunk, loaded 16 bits per two chunks.
#pragma once

#include "hs_ops.cuh"

namespace hs {

constexpr int kC2NoEsc = 0x7fffffff;

// 16-bit code words of slice s start at c2_word_base(sptr[s], s); chunk pair p
// of lane r is word p * 32 + r (low byte = chunk 2p, high byte = chunk 2p + 1)
// (48 spare words per slice: an odd last chunk, plus one pair the unclamped
// one-pair-ahead code load may touch)
__host__ __device__ __forceinline__ long long c2_word_base(long long base, long long s) { return (base >> 3) + 48 * s; }

__device__ __forceinline__ int c2_gaddr(int c, int grid, bool tr) { return tr ? (c % grid) * grid + c / grid : c; }

// One warp per slice (A in natural row order, int32 columns in image order).
// ok[s] = 1 when the slice takes the codes; then tab / start / esc / code are
// filled for it.  nslots: rlen is slot-indexed (nslices * 32).
__global__ void sell_c2_encode_kernel(long long nslots, long long nslices, const long long* __restrict__ sptr,
                                      const int* __restrict__ rlen, const int* __restrict__ col,
                                      const unsigned char* __restrict__ sflag, int grid, unsigned char* __restrict__ ok,
                                      int4* __restrict__ tab, int* __restrict__ start, int4* __restrict__ esc,
                                      unsigned char* __restrict__ code) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long row = s * 32 + lane;
  const int len = row < nslots ? rlen[row] : 0;
  const long long base = sptr[s];
  const int nq_slice = (int)((sptr[s + 1] - base) >> 7);
  const bool tr = sflag != nullptr && sflag[s];
  const int* cl = col + base + lane * 4;
  auto col_at = [&](int e) { return cl[(long long)(e >> 2) * 128 + (e & 3)]; };
  // pass 1: the slice's smallest x shift over the steps into the next image row
  int j0 = kC2NoEsc;
  {
    int px = 0, py = 0;
    for (int e = 0; e < len; ++e) {
      const int c = col_at(e), x = c % grid, y = c / grid;
      if (e > 0 && y - py == 1) j0 = min(j0, x - px);
      px = x;
      py = y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) j0 = min(j0, __shfl_xor_sync(0xffffffffu, j0, o));
  if (j0 == kC2NoEsc) j0 = 0;
  // pass 2: escapes per row
  int nesc = 0;
  {
    int px = 0, py = 0;
    for (int e = 0; e < len; ++e) {
      const int c = col_at(e), x = c % grid, y = c / grid;
      if (e > 0) {
        const int dx = x - px, dy = y - py;
        const bool reg = (dy == 0 && dx == 1) || (dy == 1 && dx >= j0 && dx <= j0 + 2);
        nesc += reg ? 0 : 1;
      }
      px = x;
      py = y;
    }
  }
  const bool bad = __any_sync(0xffffffffu, nesc > 2);
  if (lane == 0) ok[s] = bad ? 0 : 1;
  if (bad) return;
  // pass 3: step table (gather space), start addresses, escapes, code bytes
  const int sx = tr ? grid : 1, sy = tr ? 1 : grid;
  const int d0 = sx, d1 = sy + j0 * sx;
  if (lane == 0) tab[s] = make_int4(d0, d1, d1 + sx, d1 + 2 * sx);
  int4 ev = make_int4(kC2NoEsc, 0, kC2NoEsc, 0);
  unsigned char* cb = code + 2 * (c2_word_base(base, s) + lane);
  int px = 0, py = 0, pg = 0, ne = 0;
  for (int q = 0; q < nq_slice; ++q) {
    unsigned byte = 0;
    for (int i = 0; i < 4; ++i) {
      const int e = q * 4 + i;
      if (e >= len) break;
      const int c = col_at(e), x = c % grid, y = c / grid, g = c2_gaddr(c, grid, tr);
      if (e == 0) {
        if (row < nslots) start[row] = g - d0;  // entry 0 carries code 0
      } else {
        const int dx = x - px, dy = y - py;
        unsigned k;
        if (dy == 0 && dx == 1) {
          k = 0;
        } else if (dy == 1 && dx >= j0 && dx <= j0 + 2) {
          k = 1 + (unsigned)(dx - j0);
        } else {
          k = 1;
          const int fix = (g - pg) - d1;
          if (ne == 0) { ev.x = e; ev.y = fix; }
          else { ev.z = e; ev.w = fix; }
          ++ne;
        }
        byte |= k << (2 * i);
      }
      px = x;
      py = y;
      pg = g;
    }
    cb[(long long)(q >> 1) * 64 + (q & 1)] = (unsigned char)byte;
  }
  if ((nq_slice & 1) && nq_slice > 0) cb[(long long)(nq_slice >> 1) * 64 + 1] = 0;
  if (len == 0 && row < nslots) start[row] = 0;
  if (row < nslots) esc[row] = ev;
}

// shared-memory pair-table read: (step of the first code, sum of both steps)
__device__ __forceinline__ int2 c2_lds(unsigned addr) {
  int2 r;
  asm("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(addr) : "memory");
  return r;
}

__device__ __forceinline__ unsigned c2_ldcs_u16(const unsigned short* p) { return (unsigned)__ldcs(p); }

// the four gather addresses of a chunk; SH = bit position of the chunk's code byte in w
template <int SH>
__device__ __forceinline__ void c2_addrs(int a, unsigned w, unsigned tab, int (&ad)[4]) {
  const unsigned n0 = SH >= 3 ? (w >> (SH - 3)) : (w << (3 - SH));
  const int2 p = c2_lds(tab | (n0 & 0x78u));
  const int2 r = c2_lds(tab | ((w >> (SH + 1)) & 0x78u));
  ad[0] = a + p.x;
  ad[1] = a + p.y;
  ad[2] = ad[1] + r.x;
  ad[3] = ad[1] + r.y;
}

// apply the row's escapes that fall into chunk q (rare: at most two per row);
// eq becomes the chunk of the next pending escape
__device__ __forceinline__ void c2_escape(int q, int& eq, const int4* __restrict__ escp, int (&ad)[4]) {
  const int4 ev = __ldg(escp);
  int next = kC2NoEsc;
  if (ev.x != kC2NoEsc) {
    if ((ev.x >> 2) == q) {
      const int j = ev.x & 3;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i >= j) ad[i] += ev.y;
    } else if ((ev.x >> 2) > q) {
      next = ev.x >> 2;
    }
  }
  if (ev.z != kC2NoEsc) {
    if ((ev.z >> 2) == q) {
      const int j = ev.z & 3;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i >= j) ad[i] += ev.w;
    } else if ((ev.z >> 2) > q) {
      next = min(next, ev.z >> 2);
    }
  }
  eq = next;
}

template <int SH, class V, class Tin, class T>
__device__ __forceinline__ void c2_chunk(T& acc, int& a, unsigned w, unsigned tab, const Chunk4<V>& v,
                                         const Tin* __restrict__ x, int q, int& eq, const int4* __restrict__ escp) {
  int ad[4];
  c2_addrs<SH>(a, w, tab, ad);
  if (q == eq) c2_escape(q, eq, escp, ad);
  const T x0 = gather_x<T>(x, ad[0]);
  const T x1 = gather_x<T>(x, ad[1]);
  const T x2 = gather_x<T>(x, ad[2]);
  const T x3 = gather_x<T>(x, ad[3]);
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), x0));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), x1));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), x2));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[3]), x3));
  a = ad[3];
}

// One lane's row.  Two full chunks per step (one 16-bit code load); the next
// pair's codes and the next chunk's values are in flight while a chunk is
// decoded, gathered and added.  Same products and the same order of adds as
// the d16 kernel.  (Measured at config 4, 2.78 ms as written: hoisting the
// escape test out of the loop -- unchecked pairs up to the next escape, 32
// instead of 42 instructions per chunk -- ran 2.98 ms, and requesting the
// whole next pair up front 2.99 ms (3.02 at 5 blocks per SM without spills):
// without the per-chunk branch ptxas sinks the stream loads below the first
// gather stall, and the loads in flight per warp, not the issue slots, bound
// this kernel.  Pinning the order with ld.volatile stream loads and table
// reads: 2.96 ms; one warp-uniform escape vote per pair selecting a checked or
// an unchecked copy of the pair: 3.03 ms.)
template <class V, class Tin, class T>
__device__ __forceinline__ T c2_row(const unsigned short* __restrict__ cp, const V* __restrict__ vp, int a, int len,
                                    const Tin* __restrict__ x, unsigned tab, const int4* __restrict__ escp, int eq) {
  T acc = T(0);
  const int nq = (len + 3) >> 2, nfull = len >> 2;
  if (nq == 0) return acc;
  unsigned w = c2_ldcs_u16(cp);
  Chunk4<V> v = Chunk4<V>::load(vp);
  int q = 0;
  for (; q + 1 < nfull; q += 2) {
    const Chunk4<V> v1 = Chunk4<V>::load(vp + (long long)(q + 1) * 128);
    const unsigned wn = c2_ldcs_u16(cp + (long long)((q >> 1) + 1) * 32);
    c2_chunk<0, V, Tin, T>(acc, a, w, tab, v, x, q, eq, escp);
    const Chunk4<V> vn = Chunk4<V>::load(vp + (long long)min(q + 2, nq - 1) * 128);
    c2_chunk<8, V, Tin, T>(acc, a, w, tab, v1, x, q + 1, eq, escp);
    v = vn;
    w = wn;
  }
  if (q < nfull) {  // an odd full chunk: the pair's low byte; the tail (if any) takes the high byte
    const Chunk4<V> vn = Chunk4<V>::load(vp + (long long)min(q + 1, nq - 1) * 128);
    c2_chunk<0, V, Tin, T>(acc, a, w, tab, v, x, q, eq, escp);
    v = vn;
    w >>= 8;
    ++q;
  }
  const int rem = len & 3;
  if (rem) {
    int ad[4];
    c2_addrs<0>(a, w, tab, ad);
    if (q == eq) c2_escape(q, eq, escp, ad);
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), gather_x<T>(x, ad[0])));
    if (rem > 1) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), gather_x<T>(x, ad[1])));
    if (rem > 2) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), gather_x<T>(x, ad[2])));
  }
  return acc;
}

// SpMV of a tomography A: slices flagged in c2ok decode 2-bit step codes, the
// rest read their 16-bit deltas (d16_row_u2).  Dynamic longest-first slice
// scheduling as in sell_spmv_d16_kernel.
template <class V, class Tin, class T, bool POW2, int MINB>
__global__ void __launch_bounds__(256, MINB)
sell_spmv_c2_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                    const int* __restrict__ rlen, const int* __restrict__ rbase, const short* __restrict__ dcol,
                    const V* __restrict__ val, const Tin* __restrict__ xrow, const Tin* __restrict__ xT,
                    const unsigned char* __restrict__ sflag, const unsigned char* __restrict__ c2ok,
                    const int4* __restrict__ c2tab, const int* __restrict__ c2start, const int4* __restrict__ c2esc,
                    const unsigned short* __restrict__ c2code, int grid, int gshift,
                    const int* __restrict__ sorder, unsigned int* __restrict__ sched, T* __restrict__ y) {
  __shared__ __align__(128) int2 pair_tab[8][16];
  const int lane = threadIdx.x & 31;
  const unsigned tab = smem_u32(&pair_tab[threadIdx.x >> 5][0]);
  for (;;) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&sched[0], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nslices) break;
    const long long s = sorder ? (long long)sorder[i] : (long long)i;
    const bool tr = sflag != nullptr && sflag[s];  // warp-uniform
    const long long slot = s * 32 + lane;
    const int len = rlen[slot];
    const long long base = sptr[s];
    const V* vp = val + base + lane * 4;
    T acc;
    if (c2ok[s]) {  // warp-uniform
      const int4 t = __ldg(c2tab + s);
      if (lane < 16) {
        const int k0 = lane & 3, k1 = lane >> 2;
        const int s0 = k0 == 0 ? t.x : k0 == 1 ? t.y : k0 == 2 ? t.z : t.w;
        const int s1 = k1 == 0 ? t.x : k1 == 1 ? t.y : k1 == 2 ? t.z : t.w;
        pair_tab[threadIdx.x >> 5][lane] = make_int2(s0, s0 + s1);
      }
      __syncwarp();
      const int4* escp = c2esc + slot;
      const int e0 = __ldg(&escp->x);
      acc = c2_row<V, Tin, T>(c2code + c2_word_base(base, s) + lane, vp, c2start[slot], len, tr ? xT : xrow, tab, escp,
                              e0 == kC2NoEsc ? kC2NoEsc : (e0 >> 2));
      __syncwarp();  // every lane is done with the table before the next slice rewrites it
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


// ---- 8-bit step codes for a tomography A^T ("t8"): 5 instead of 6 B per nonzero --
// A row of A^T is a pixel, and its sorted columns are the rays that cross it:
// angle by angle, one to three neighbouring detector bins per angle.  With the
// sinogram in the 4-angle interleave, address(a, b) = ((a >> 2) n_bins + b) 4
// + (a & 3) (SinoBlk{n_bins, 4, 1, n_bins}: a 128-byte line holds 8 bins x 4
// angles, the footprint of the 4 x 8 blocked layout), every step between
// consecutive entries is one of
//   code 0          : same angle, next bin              -> +4
//   code 1 + D + 63 : next angle, bin shift D, same group of 4 angles -> 1 + 4 D
//   code 128 + D+63 : next angle, bin shift D, next group             -> 4 n_bins - 3 + 4 D
// (|D| <= 63), so one byte per entry indexes ONE 256-entry table shared by the
// whole CTA (built at kernel start; the codes cluster on a few dozen
// neighbouring entries, so the LDS is nearly conflict-free).  Anything else
// (a pixel a detector misses at some angles) is an escape as in c2: code 0
// plus a per-row (position, correction) pair, at most two per row, else the
// slice keeps its 16-bit deltas in the same layout.
__host__ __device__ __forceinline__ int t8_addr(int a, int b, int n_bins) { return ((a >> 2) * n_bins + b) * 4 + (a & 3); }

__global__ void sell_t8_encode_kernel(long long nslots, long long nslices, const long long* __restrict__ sptr,
                                      const int* __restrict__ rlen, const int* __restrict__ col, int n_bins,
                                      unsigned char* __restrict__ ok, int* __restrict__ start, int4* __restrict__ esc,
                                      unsigned char* __restrict__ code) {
  const long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int lane = threadIdx.x & 31;
  const long long row = s * 32 + lane;
  const int len = row < nslots ? rlen[row] : 0;
  const long long base = sptr[s];
  const int nq_slice = (int)((sptr[s + 1] - base) >> 7);
  const int* cl = col + base + lane * 4;
  auto col_at = [&](int e) { return cl[(long long)(e >> 2) * 128 + (e & 3)]; };
  auto regular = [&](int da, int db) { return (da == 0 && db == 1) || (da == 1 && db >= -63 && db <= 63); };
  int nesc = 0;
  {
    int pa = 0, pb = 0;
    for (int e = 0; e < len; ++e) {
      const int c = col_at(e), a = c / n_bins, b = c - a * n_bins;
      if (e > 0 && !regular(a - pa, b - pb)) ++nesc;
      pa = a;
      pb = b;
    }
  }
  const bool bad = __any_sync(0xffffffffu, nesc > 2);
  if (lane == 0) ok[s] = bad ? 0 : 1;
  if (bad) return;
  int4 ev = make_int4(kC2NoEsc, 0, kC2NoEsc, 0);
  unsigned char* cb = code + base + lane * 4;
  int pa = 0, pb = 0, pg = 0, ne = 0;
  for (int q = 0; q < nq_slice; ++q) {
    unsigned w = 0;
    for (int i = 0; i < 4; ++i) {
      const int e = q * 4 + i;
      if (e >= len) break;
      const int c = col_at(e), a = c / n_bins, b = c - a * n_bins, g = t8_addr(a, b, n_bins);
      if (e == 0) {
        if (row < nslots) start[row] = g - 4;  // entry 0 carries code 0
      } else {
        const int da = a - pa, db = b - pb;
        unsigned k = 0;
        if (da == 0 && db == 1) {
          k = 0;
        } else if (da == 1 && db >= -63 && db <= 63) {
          k = ((a & 3) == 0 ? 128u : 1u) + (unsigned)(db + 63);
        } else {
          const int fix = (g - pg) - 4;
          if (ne == 0) { ev.x = e; ev.y = fix; }
          else { ev.z = e; ev.w = fix; }
          ++ne;
        }
        w |= k << (8 * i);
      }
      pa = a;
      pb = b;
      pg = g;
    }
    *reinterpret_cast<unsigned*>(cb + (long long)q * 128) = w;
  }
  if (len == 0 && row < nslots) start[row] = 0;
  if (row < nslots) esc[row] = ev;
}

__device__ __forceinline__ int t8_step(unsigned k, int n_bins) {
  if (k == 0) return 4;
  if (k < 128) return 1 + 4 * ((int)k - 1 - 63);
  if (k < 255) return 4 * n_bins - 3 + 4 * ((int)k - 128 - 63);
  return 0;
}

__device__ __forceinline__ int t8_lds(unsigned addr) {
  int r;
  asm("ld.shared.s32 %0, [%1];" : "=r"(r) : "r"(addr) : "memory");
  return r;
}

// the chunk's four steps: byte j of w indexes the 1024-byte-aligned table at shared address tab
__device__ __forceinline__ void t8_addrs(int a, unsigned w, unsigned tab, int (&ad)[4]) {
  const int s0 = t8_lds(tab | ((w << 2) & 0x3fcu)), s1 = t8_lds(tab | ((w >> 6) & 0x3fcu)),
            s2 = t8_lds(tab | ((w >> 14) & 0x3fcu)), s3 = t8_lds(tab | ((w >> 22) & 0x3fcu));
  ad[0] = a + s0;
  ad[1] = ad[0] + s1;
  ad[2] = ad[1] + s2;
  ad[3] = ad[2] + s3;
}

template <class V, class Tin, class T>
__device__ __forceinline__ void t8_chunk(T& acc, int& a, unsigned w, unsigned tab, const Chunk4<V>& v,
                                         const Tin* __restrict__ x, int q, int& eq, const int4* __restrict__ escp) {
  int ad[4];
  t8_addrs(a, w, tab, ad);
  if (q == eq) c2_escape(q, eq, escp, ad);
  const T x0 = gather_x<T>(x, ad[0]);
  const T x1 = gather_x<T>(x, ad[1]);
  const T x2 = gather_x<T>(x, ad[2]);
  const T x3 = gather_x<T>(x, ad[3]);
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), x0));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), x1));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), x2));
  acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[3]), x3));
  a = ad[3];
}

// one lane's row: the next chunk's (codes, values) in flight while a chunk is
// decoded, gathered and added (the d16_row_u2 schedule)
template <class V, class Tin, class T>
__device__ __forceinline__ T t8_row(const unsigned* __restrict__ cp, const V* __restrict__ vp, int a, int len,
                                    const Tin* __restrict__ x, unsigned tab, const int4* __restrict__ escp, int eq) {
  T acc = T(0);
  const int nq = (len + 3) >> 2, nfull = len >> 2;
  if (nq == 0) return acc;
  unsigned w = __ldcs(cp);
  Chunk4<V> v = Chunk4<V>::load(vp);
#pragma unroll 2
  for (int q = 0; q < nfull; ++q) {
    const long long qn = min(q + 1, nq - 1);
    const unsigned wn = __ldcs(cp + qn * 32);
    const Chunk4<V> vn = Chunk4<V>::load(vp + qn * 128);
    t8_chunk<V, Tin, T>(acc, a, w, tab, v, x, q, eq, escp);
    w = wn;
    v = vn;
  }
  const int rem = len & 3;
  if (rem) {
    int ad[4];
    t8_addrs(a, w, tab, ad);
    if (nfull == eq) c2_escape(nfull, eq, escp, ad);
    acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[0]), gather_x<T>(x, ad[0])));
    if (rem > 1) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[1]), gather_x<T>(x, ad[1])));
    if (rem > 2) acc = Rn<T>::add(acc, Rn<T>::mul(cvt<T>(v.v[2]), gather_x<T>(x, ad[2])));
  }
  return acc;
}

// SpMV of a tomography A^T over the 4-angle interleaved sinogram: slices
// flagged in ok decode 8-bit step codes, the rest their 16-bit deltas (same
// layout).  rperm: slot -> pixel (8 x 4 tiles).  Natural slice order.
template <class V, class Tin, class T, int MINB>
__global__ void __launch_bounds__(256, MINB)
sell_spmv_t8_kernel(long long rows, long long nslices, const long long* __restrict__ sptr,
                    const int* __restrict__ rlen, const int* __restrict__ rbase, const short* __restrict__ dcol,
                    const V* __restrict__ val, const Tin* __restrict__ x, const unsigned char* __restrict__ ok,
                    const int* __restrict__ start, const int4* __restrict__ esc,
                    const unsigned char* __restrict__ code, int n_bins, const int* __restrict__ rperm,
                    const int* __restrict__ sorder, unsigned int* __restrict__ sched, T* __restrict__ y) {
  __shared__ __align__(1024) int tab_s[256];
  tab_s[threadIdx.x] = t8_step(threadIdx.x, n_bins);
  __syncthreads();
  const unsigned tab = smem_u32(tab_s);
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&sched[0], 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nslices) break;
    const long long s = sorder ? (long long)sorder[i] : (long long)i;
    const long long slot = s * 32 + lane;
    const long long row = rperm ? (long long)rperm[slot] : slot;
    const int len = rlen[slot];
    const long long base = sptr[s];
    const V* vp = val + base + lane * 4;
    T acc;
    if (ok[s]) {  // warp-uniform
      const int4* escp = esc + slot;
      const int e0 = __ldg(&escp->x);
      acc = t8_row<V, Tin, T>(reinterpret_cast<const unsigned*>(code + base) + lane, vp, start[slot], len, x, tab, escp,
                              e0 == kC2NoEsc ? kC2NoEsc : (e0 >> 2));
    } else {
      acc = d16_row_u2<0, V, Tin, T>(dcol + base + lane * 4, vp, rbase[slot], len, x, 0, 0, 0);
    }
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

}  // namespace hs
