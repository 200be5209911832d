// Sketch kernels: z = S v for the three sketch kinds the drop-in accepts
// (sketch.py:29-65 takes any `entries` supporting `@`):
//   * explicit dense S (row-major, e.g. the reference's PCG64 draw, sketch.py:43-53)
//   * Gaussian S generated on the fly from a counter-based RNG, never stored
//   * sparse-sign S (zeta nonzeros +-1/sqrt(zeta) per column), stored row-wise
// All sums are fp64 in a fixed order (deterministic, replayable: test_solvers.py:319-326).
#pragma once

#include "hs_common.cuh"

namespace hs {

// ---- tiles ----------------------------------------------------------------
// Every tiled sketch forms z = scale * sum over tiles (in order) of part_tile,
// where part_tile is the sketch of the input entries of one tile, summed in an
// order fixed by the tile's contents alone.  The input is cut into granules
// of G entries -- the operator's shard granule: a row shard of the input is a
// whole number of granules (hs_op::granule) -- and each granule into tiles of
// tc entries (its last tile may be shorter).  The same partials, computed on
// one GPU or spread over any number of ranks and all-gathered, therefore give
// a bit-identical z (P-independent sketches).
inline int ilog2_floor(long long x) {
  int r = 0;
  while (x > 1) {
    x >>= 1;
    ++r;
  }
  return r;
}
inline long long pow2_clamped(long long len, int shift, int lo, int hi) {
  int e = (len >> shift) > 0 ? ilog2_floor(len >> shift) : 0;
  e = e < lo ? lo : (e > hi ? hi : e);
  return 1LL << e;
}
// columns per tile: sparse-sign ~len/128 (32..8192), Gaussian / dense ~len/1024 (256..8192)
inline long long sketch_tile_sparse(long long len) { return pow2_clamped(len, 7, 5, 13); }
inline long long sketch_tile_dense(long long len) { return pow2_clamped(len, 10, 8, 13); }
// shard granule of a vector that may be split anywhere (tomography rays)
inline long long shard_granule(long long len) { return pow2_clamped(len, 7, 8, 13); }

// local tile b of a partial kernel: granule b / tpg, tile b % tpg of it, local
// entries [c0, c1) (empty past the local length)
struct TileMap {
  long long G, tc, len;
  int tpg;
  __host__ __device__ void range(long long b, long long& c0, long long& c1) const {
    const long long gs = (b / tpg) * G, t = b % tpg;
    c0 = gs + t * tc;
    const long long e = gs + ((t + 1) * tc < G ? (t + 1) * tc : G);
    c1 = e < len ? e : len;
    if (c0 > c1) c0 = c1;
  }
  __host__ __device__ long long slots() const { return ((len + G - 1) / G) * tpg; }
};

// z[w * ldz + i] = scale * the sum of all tile partials of the len inputs.
// The partials are numbered f = q * tpg + t over the global granules q and
// their tiles t (every granule but the last has tpg tiles); part holds blocks
// of gpr granules, one per rank, each vector-major ([rank][w][slot][i]; on one
// GPU gpr = all granules).  Block: 8 sketch rows x RPH phases; phase p sums
// the partials f = p (mod RPH) in order, then the phases are added in order --
// a fixed association that depends only on the global tile structure.
constexpr int RPH = 32, RROWS = 8;
__global__ void __launch_bounds__(RROWS * RPH)
sketch_tile_reduce_kernel(int ell, long long len, long long G, long long tc, int tpg, long long gpr, int nv,
                          const double* __restrict__ part, double scale, double* __restrict__ z, long long ldz) {
  __shared__ double ph[RPH][RROWS + 1];
  const int li = threadIdx.x % RROWS, p = threadIdx.x / RROWS;
  const int i = blockIdx.x * RROWS + li;
  const int w = blockIdx.y;
  const long long nq = (len + G - 1) / G;
  const long long glast = len - (nq - 1) * G;
  const long long F = (nq - 1) * tpg + (glast + tc - 1) / tc;
  double s = 0.0;
  if (i < ell) {
#pragma unroll 4
    for (long long f = p; f < F; f += RPH) {
      const long long q = f / tpg, t = f - q * tpg;
      const long long r = q / gpr, ql = q - r * gpr;
      s += __ldcg(part + (((r * nv + w) * gpr + ql) * tpg + t) * (long long)ell + i);
    }
  }
  ph[p][li] = s;
  __syncthreads();
  if (p == 0 && i < ell) {
    double a = ph[0][li];
#pragma unroll
    for (int k = 1; k < RPH; ++k) a += ph[k][li];
    z[(long long)w * ldz + i] = a * scale;
  }
}

// ---- explicit dense S (row-major, ld lds), one warp per sketch row of a tile:
// lanes stride the tile's columns with fma, then a fixed xor-tree warp sum.
// part[(w * tstride + t) * ell + i] for the single vector w = 0.
template <class Tin>
__global__ void __launch_bounds__(256)
sketch_dense_tile_kernel(int ell, TileMap tm, long long col_offset, const double* __restrict__ S, long long lds,
                         const Tin* __restrict__ v, double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= ell) return;
  long long c0, c1;
  tm.range(blockIdx.x, c0, c1);
  const double* row = S + (long long)i * lds + col_offset;
  double acc = 0.0;
  for (long long c = c0 + lane; c < c1; c += 32) acc = fma(__ldg(row + c), cvt<double>(v[c]), acc);
  acc = warp_sum(acc);
  if (lane == 0) part[(long long)blockIdx.x * ell + i] = acc;
}

// ---- Gaussian from Philox: S[i, c] = N(seed; c, i) / sqrt(ell) -----------------
// one Philox call per (column c, row quad q) gives 4 normals (2 Box-Muller pairs)
__device__ __forceinline__ void gauss_quad(uint2 key, unsigned long long c, unsigned q, float (&o)[4]) {
  const uint4 r = philox7(make_uint4((unsigned)c, (unsigned)(c >> 32), q, 0x53CE7C4Du), key);
  box_muller_fast(r.x, r.y, o[0], o[1]);
  box_muller_fast(r.z, r.w, o[2], o[3]);
}

// grid: (ntiles, nqb), block 256 = QB row quads x PH column phases (QB = quads
// per block, chosen so the quads split evenly over the nqb blocks).  The tile's
// slice of the nv <= NV input vectors (column stride ldv) is staged in shared
// memory as fp64, vs[i*NV + w] (converted once per block), so every generated
// quad of normals is applied to all nv vectors: a batch of nv sketches costs
// one RNG pass instead of nv.  Per vector the columns each thread visits, the
// fma order and the phase reduction do not depend on NV or nv, so a vector's
// result is bit-identical whether it is sketched alone or in a batch.
// part layout: part[(w * tstride + tile) * ell + i] (tstride >= local tiles).
constexpr int GAUSS_CH = 1024;
template <class Tin, int NV, int UNR = 2>
__global__ void __launch_bounds__(256, 2)
sketch_gauss_partial_kernel(int ell, TileMap tm, long long col_offset, uint2 key, const Tin* __restrict__ v,
                            long long ldv, int nv, double* __restrict__ part, long long tstride) {
  extern __shared__ __align__(128) unsigned char gauss_smem[];
  double* vs = reinterpret_cast<double*>(gauss_smem);  // GAUSS_CH * NV
  __shared__ double red[256][4];
  const int nq = (ell + 3) / 4;
  const int nqb = gridDim.y;
  const int QB = (nq + nqb - 1) / nqb;  // <= 64
  const int PH = 256 / QB;
  const int ql = threadIdx.x % QB, ph = threadIdx.x / QB;
  const int q = blockIdx.y * QB + ql;
  const bool active = ph < PH && q < nq;
  long long c0, c1;
  tm.range(blockIdx.x, c0, c1);
  double a[NV][4];
#pragma unroll
  for (int w = 0; w < NV; ++w) a[w][0] = a[w][1] = a[w][2] = a[w][3] = 0.0;
  for (long long cb = c0; cb < c1; cb += GAUSS_CH) {
    const int cn = (int)min((long long)GAUSS_CH, c1 - cb);
    __syncthreads();
    // vectors past nv are staged as zeros so the hot loop has no guards
#pragma unroll
    for (int w = 0; w < NV; ++w) {
      const Tin* vw = v + (long long)w * ldv + cb;
      for (int i = threadIdx.x; i < cn; i += blockDim.x) vs[i * NV + w] = w < nv ? cvt<double>(vw[i]) : 0.0;
    }
    __syncthreads();
    if (active) {
#pragma unroll UNR
      for (int i = ph; i < cn; i += PH) {
        float g[4];
        gauss_quad(key, (unsigned long long)(cb + i + col_offset), (unsigned)q, g);
        const double g0 = (double)g[0], g1 = (double)g[1], g2 = (double)g[2], g3 = (double)g[3];
        if constexpr (NV == 1) {
          const double vc = vs[i];
          a[0][0] = fma(g0, vc, a[0][0]);
          a[0][1] = fma(g1, vc, a[0][1]);
          a[0][2] = fma(g2, vc, a[0][2]);
          a[0][3] = fma(g3, vc, a[0][3]);
        } else {
          const double2* vp = reinterpret_cast<const double2*>(vs + i * NV);
#pragma unroll
          for (int w2 = 0; w2 < NV / 2; ++w2) {
            const double2 vv = vp[w2];
            a[2 * w2][0] = fma(g0, vv.x, a[2 * w2][0]);
            a[2 * w2][1] = fma(g1, vv.x, a[2 * w2][1]);
            a[2 * w2][2] = fma(g2, vv.x, a[2 * w2][2]);
            a[2 * w2][3] = fma(g3, vv.x, a[2 * w2][3]);
            a[2 * w2 + 1][0] = fma(g0, vv.y, a[2 * w2 + 1][0]);
            a[2 * w2 + 1][1] = fma(g1, vv.y, a[2 * w2 + 1][1]);
            a[2 * w2 + 1][2] = fma(g2, vv.y, a[2 * w2 + 1][2]);
            a[2 * w2 + 1][3] = fma(g3, vv.y, a[2 * w2 + 1][3]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int w = 0; w < NV; ++w) {
    if (w >= nv) break;
    __syncthreads();
    red[threadIdx.x][0] = a[w][0]; red[threadIdx.x][1] = a[w][1];
    red[threadIdx.x][2] = a[w][2]; red[threadIdx.x][3] = a[w][3];
    __syncthreads();
    if (ph == 0 && q < nq) {
      double* pw = part + ((long long)w * tstride + blockIdx.x) * ell;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = 4 * q + r;
        if (i < ell) {
          double s = 0.0;
          for (int p = 0; p < PH; ++p) s += red[p * QB + ql][r];  // fixed phase order
          pw[i] = s;
        }
      }
    }
  }
}

// largest batch one partial launch handles
constexpr int GAUSS_NV_MAX = 8;

// partials of nv vectors (column stride ldv) over local columns [0, m) whose
// first column is global column col_offset (a multiple of tile_cols):
// part[(w * tstride + t) * ell + i]; batches larger than GAUSS_NV_MAX go in
// groups.  Returns the number of launches.
template <class Tin, int NV, int UNR = 2>
inline void gauss_partial_launch(dim3 grid, cudaStream_t s, int ell, TileMap tm, long long col_offset, uint2 key,
                                 const Tin* v, long long ldv, int nv, double* part, long long tstride) {
  const size_t smem = (size_t)GAUSS_CH * NV * sizeof(double);
  ensure_smem((const void*)sketch_gauss_partial_kernel<Tin, NV, UNR>, smem);
  sketch_gauss_partial_kernel<Tin, NV, UNR><<<grid, 256, smem, s>>>(ell, tm, col_offset, key, v, ldv, nv, part,
                                                                    tstride);
}

template <class Tin>
inline int gauss_partials(cudaStream_t s, int ell, TileMap tm, long long col_offset, uint2 key, const Tin* v,
                          long long ldv, int nv, double* part, long long tstride) {
  const int nq = (ell + 3) / 4;
  const dim3 grid((unsigned)tm.slots(), (nq + 63) / 64);
  int launches = 0;
  for (int w0 = 0; w0 < nv; w0 += GAUSS_NV_MAX) {
    const int g = nv - w0 < GAUSS_NV_MAX ? nv - w0 : GAUSS_NV_MAX;
    const Tin* vg = v + (long long)w0 * ldv;
    double* pg = part + (long long)w0 * tstride * ell;
    if (g == 1) gauss_partial_launch<Tin, 1>(grid, s, ell, tm, col_offset, key, vg, ldv, g, pg, tstride);
    else if (g == 2) gauss_partial_launch<Tin, 2>(grid, s, ell, tm, col_offset, key, vg, ldv, g, pg, tstride);
    else if (g <= 4) gauss_partial_launch<Tin, 4>(grid, s, ell, tm, col_offset, key, vg, ldv, g, pg, tstride);
    else gauss_partial_launch<Tin, 8>(grid, s, ell, tm, col_offset, key, vg, ldv, g, pg, tstride);
    ++launches;
  }
  return launches;
}

// materialise the generated Gaussian S (row-major ell x m, fp64) for export
__global__ void gauss_materialize_kernel(int ell, long long m, uint2 key, double inv_sqrt_ell, double* __restrict__ S) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  const int nq = (ell + 3) / 4;
  for (int q = 0; q < nq; ++q) {
    float g[4];
    gauss_quad(key, (unsigned long long)c, (unsigned)q, g);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = 4 * q + r;
      if (i < ell) S[(long long)i * m + c] = (double)g[r] * inv_sqrt_ell;
    }
  }
}

// ---- sparse-sign -----------------------------------------------------------------
// column c draws zeta distinct rows uniformly from [0, ell) and a sign each,
// from Philox(seed; c, draw).  Entries are emitted as (row, signed column+1).
__global__ void sparse_sign_gen_kernel(long long m, int ell, int zeta, uint2 key, int* __restrict__ rows_out,
                                       int* __restrict__ scol_out) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  int chosen[64];
  int got = 0;
  unsigned draw = 0;
  while (got < zeta) {
    const uint4 r = Philox::gen(make_uint4((unsigned)c, (unsigned)(c >> 32), draw++, 0x5A5A0001u), key);
    const unsigned w[2] = {r.x, r.z};
    const unsigned sg[2] = {r.y, r.w};
    for (int h = 0; h < 2 && got < zeta; ++h) {
      const int row = (int)(((unsigned long long)w[h] * (unsigned long long)ell) >> 32);
      bool dup = false;
      for (int t = 0; t < got; ++t) dup |= (chosen[t] == row);
      if (dup) continue;
      chosen[got] = row;
      rows_out[c * zeta + got] = row;
      scol_out[c * zeta + got] = (sg[h] & 1u) ? -(int)(c + 1) : (int)(c + 1);
      ++got;
    }
  }
}

// Sparse-sign partials of one tile.  The scatter-add z_r += s_rc v_c of the
// tile's entries is resolved at build time (hs_sketch::sparse_layout): per
// absolute tile of tc columns, the sketch rows are sorted by their entry count
// and cut into slices of 32, and lane r of a slice holds its row's entries in
// column order, 8 per 16-byte chunk -- entry e at chunk-interleaved position
// (e / 8) * 256 + r * 8 + e % 8, so a warp streams 512 contiguous bytes per
// chunk.  Entry = column offset in the tile (bits 0-13) | 0x8000 if negative;
// padding = offset tc, which reads the zero after the staged tile.  The CTA
// stages the tile of v in shared memory as fp64; each lane then adds its
// row's +-v (sign by xor of the high word) into four register accumulators
// (entry e into a[e % 4]), combined as (a0 + a1) + (a2 + a3).  No atomics;
// the order is fixed by the layout, so the partial is deterministic.
// The tile size tm.tc must divide the granule and the column offset.
template <class Tin> struct SkStage { using T = float; };   // staged tile type (bf16, fp32: exact in fp32)
template <> struct SkStage<double> { using T = double; };

// grid = local tile slots, SK_THREADS threads: one CTA per tile (the tile of
// v is staged once), warp w adds slices w, w + SK_WARPS, ...
constexpr int SK_THREADS = 768, SK_WARPS = SK_THREADS / 32;
template <class Tin, int CB>
__global__ void __launch_bounds__(SK_THREADS, 2)
sketch_sparse_gather_kernel(int ell, int nsl, TileMap tm, long long col_offset, const long long* __restrict__ tbase,
                            const int* __restrict__ soff, const unsigned short* __restrict__ perm,
                            const unsigned short* __restrict__ ent, const Tin* __restrict__ v,
                            double* __restrict__ part) {
  using S = typename SkStage<Tin>::T;
  extern __shared__ __align__(16) unsigned char sk_smem[];
  S* vs = reinterpret_cast<S*>(sk_smem);  // tc + 1 values
  long long c0, c1;
  tm.range(blockIdx.x, c0, c1);
  if (c1 <= c0) return;  // empty slot past the local length (never reduced)
  const long long k = (col_offset + c0) / tm.tc;  // absolute tile
  const int n = (int)(c1 - c0), tc = (int)tm.tc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* so = soff + k * (nsl + 1);
  const unsigned short* et = ent + tbase[k];
  // this warp's first slice: bounds and output row fetched before the staging
  int sl = warp;
  int a = sl < nsl ? so[sl] : 0, b = sl < nsl ? so[sl + 1] : 0;
  unsigned r = sl < nsl ? perm[(k * nsl + sl) * 32 + lane] : 0xFFFFu;
  // stage the tile: all of a thread's loads issued before any store
  for (int i0 = 0; i0 <= tc; i0 += 16 * SK_THREADS) {
    S t[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * SK_THREADS + (int)threadIdx.x;
      t[u] = i < n ? cvt<S>(__ldcs(v + c0 + i)) : S(0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = i0 + u * SK_THREADS + (int)threadIdx.x;
      if (i <= tc) vs[i] = t[u];
    }
  }
  __syncthreads();
  const unsigned pad = (unsigned)tc | ((unsigned)tc << 16);
  while (sl < nsl) {
    const int L8 = (b - a) >> 8;
    const uint4* ep = reinterpret_cast<const uint4*>(et + a) + lane;
    // the next slice's bounds and row, in flight during this one
    const int sn = sl + SK_WARPS;
    const int an = sn < nsl ? so[sn] : 0, bn = sn < nsl ? so[sn + 1] : 0;
    const unsigned rn = sn < nsl ? perm[(k * nsl + sn) * 32 + lane] : 0xFFFFu;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q0 = 0; q0 < L8; q0 += CB) {
      uint4 w[CB];
#pragma unroll
      for (int q = 0; q < CB; ++q)
        w[q] = q0 + q < L8 ? __ldcs(ep + (long long)(q0 + q) * 32) : make_uint4(pad, pad, pad, pad);
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        const unsigned u4[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const unsigned e = (u4[h >> 1] >> ((h & 1) * 16)) & 0xFFFFu;
          const double x = (double)vs[e & 0x3FFFu];
          const long long sg = (long long)(e & 0x8000u) << 48;  // sign bit -> bit 63
          acc[h & 3] += __longlong_as_double(__double_as_longlong(x) ^ sg);
        }
      }
    }
    if (r != 0xFFFFu) part[(long long)blockIdx.x * ell + r] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    sl = sn;
    a = an;
    b = bn;
    r = rn;
  }
}

template <class Tin>
inline void sparse_partials(cudaStream_t s, int ell, TileMap tm, long long col_offset, const long long* tbase,
                            const int* soff, const unsigned short* perm, const unsigned short* ent, const Tin* v,
                            double* part) {
  const long long nt = tm.slots();
  if (nt == 0) return;
  const int nsl = (ell + 31) / 32;
  const size_t smem = (size_t)(tm.tc + 1) * sizeof(typename SkStage<Tin>::T);
  auto kern = sketch_sparse_gather_kernel<Tin, 8>;
  ensure_smem((const void*)kern, smem);
  kern<<<(unsigned)nt, SK_THREADS, smem, s>>>(ell, nsl, tm, col_offset, tbase, soff, perm, ent, v, part);
}

// ---- general explicit sparse S (CSR by sketch rows, fp64 values) ------------
template <class Tin>
__global__ void __launch_bounds__(256)
sketch_csr_kernel(int ell, const long long* __restrict__ rowptr, const int* __restrict__ col,
                  const double* __restrict__ val, const Tin* __restrict__ v, double* __restrict__ z) {
  __shared__ double scratch[32];
  const int i = blockIdx.x;
  double acc = 0.0;
  for (long long p = rowptr[i] + threadIdx.x; p < rowptr[i + 1]; p += blockDim.x)
    acc = fma(val[p], cvt<double>(v[col[p]]), acc);
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) z[i] = acc;
}

// ---- sketch-basis column: m_col = G[:, :ng] @ hcol[:ng]  (solvers.py:496-499) ----
__global__ void gemv_small_kernel(int ell, int ng, const double* __restrict__ G, const double* __restrict__ h,
                                  double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= ell) return;
  double s = 0.0;
  for (int i = 0; i < ng; ++i) s = fma(G[(long long)i * ell + r], h[i], s);
  out[r] = s;
}

}  // namespace hs
