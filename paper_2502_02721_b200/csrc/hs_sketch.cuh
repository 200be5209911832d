// Sketch kernels: z = S v for the three sketch kinds the drop-in accepts
// (sketch.py:29-65 takes any `entries` supporting `@`):
//   * explicit dense S (row-major, e.g. the reference's PCG64 draw, sketch.py:43-53)
//   * Gaussian S generated on the fly from a counter-based RNG, never stored
//   * sparse-sign S (zeta nonzeros +-1/sqrt(zeta) per column), stored row-wise
// All sums are fp64 in a fixed order (deterministic, replayable: test_solvers.py:319-326).
#pragma once

#include "hs_common.cuh"

namespace hs {

// ---- explicit dense: one block per sketch row, fixed-tree block sum --------
template <class Vs, class Tin>
__global__ void __launch_bounds__(256)
sketch_dense_kernel(int ell, long long m, const Vs* __restrict__ S, long long lds,
                    const Tin* __restrict__ v, double* __restrict__ z) {
  __shared__ double scratch[32];
  const int i = blockIdx.x;
  const Vs* row = S + (long long)i * lds;
  double acc = 0.0;
  for (long long c = threadIdx.x; c < m; c += blockDim.x) acc = fma((double)row[c], cvt<double>(v[c]), acc);
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) z[i] = acc;
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
// part layout: part[(w * ntiles + tile) * ell + i].
constexpr int GAUSS_CH = 1024;
template <class Tin, int NV, int UNR = 2>
__global__ void __launch_bounds__(256, 2)
sketch_gauss_partial_kernel(int ell, long long m, long long col_offset, long long tile_cols, uint2 key,
                            const Tin* __restrict__ v, long long ldv, int nv, double* __restrict__ part) {
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
  const long long c0 = (long long)blockIdx.x * tile_cols;
  const long long c1 = min(m, c0 + tile_cols);
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
      double* pw = part + ((long long)w * gridDim.x + blockIdx.x) * ell;
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

// launch the partial + reduce pair for nv vectors (column stride ldv) into
// z[w * ldz + i]; batches larger than GAUSS_NV_MAX go in groups
template <class Tin, int NV, int UNR = 2>
inline void gauss_partial_launch(dim3 grid, cudaStream_t s, int ell, long long m, long long col_offset,
                                 long long tile_cols, uint2 key, const Tin* v, long long ldv, int nv, double* part) {
  const size_t smem = (size_t)GAUSS_CH * NV * sizeof(double);
  ensure_smem((const void*)sketch_gauss_partial_kernel<Tin, NV, UNR>, smem);
  sketch_gauss_partial_kernel<Tin, NV, UNR><<<grid, 256, smem, s>>>(ell, m, col_offset, tile_cols, key, v, ldv, nv,
                                                                    part);
}

__global__ void sketch_tile_reduce_kernel(int ell, int ntiles, const double* __restrict__ part, double scale,
                                          double* __restrict__ z, long long ldz);

template <class Tin>
inline int gauss_sketch_launch(cudaStream_t s, int ell, long long m, long long col_offset, long long tile_cols,
                               uint2 key, const Tin* v, long long ldv, int nv, double* part, double* z,
                               long long ldz) {
  const int nq = (ell + 3) / 4;
  const int ntl = (int)((m + tile_cols - 1) / tile_cols);
  const dim3 grid(ntl, (nq + 63) / 64);
  int launches = 0;
  for (int w0 = 0; w0 < nv; w0 += GAUSS_NV_MAX) {
    const int g = nv - w0 < GAUSS_NV_MAX ? nv - w0 : GAUSS_NV_MAX;
    const Tin* vg = v + (long long)w0 * ldv;
    if (g == 1) gauss_partial_launch<Tin, 1>(grid, s, ell, m, col_offset, tile_cols, key, vg, ldv, g, part);
    else if (g == 2) gauss_partial_launch<Tin, 2>(grid, s, ell, m, col_offset, tile_cols, key, vg, ldv, g, part);
    else if (g <= 4) gauss_partial_launch<Tin, 4>(grid, s, ell, m, col_offset, tile_cols, key, vg, ldv, g, part);
    else gauss_partial_launch<Tin, 8>(grid, s, ell, m, col_offset, tile_cols, key, vg, ldv, g, part);
    sketch_tile_reduce_kernel<<<dim3((ell + 127) / 128, g), 128, 0, s>>>(ell, ntl, part, 1.0 / sqrt((double)ell),
                                                                         z + (long long)w0 * ldz, ldz);
    launches += 2;
  }
  return launches;
}

// number of row-quad blocks for the partial kernel (<= 64 quads per block, balanced)
inline int gauss_quad_blocks(int ell) {
  const int nq = (ell + 3) / 4;
  return (nq + 63) / 64;
}

// z[w * ldz + i] = scale * sum_t part[w][t][i]   (t ascending); grid.y = vector
__global__ void sketch_tile_reduce_kernel(int ell, int ntiles, const double* __restrict__ part, double scale,
                                          double* __restrict__ z, long long ldz) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ell) return;
  const double* pw = part + (long long)blockIdx.y * ntiles * ell;
  double s = 0.0;
  for (int t = 0; t < ntiles; ++t) s += pw[(long long)t * ell + i];
  z[(long long)blockIdx.y * ldz + i] = s * scale;
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

// z[i] = scale * sum over row i's entries (+-) v[col]; block per sketch row
template <class Tin>
__global__ void __launch_bounds__(256)
sketch_sparse_kernel(int ell, const long long* __restrict__ rowptr, const int* __restrict__ scol,
                     long long col_offset, long long m_loc, const Tin* __restrict__ v, double scale,
                     double* __restrict__ z) {
  __shared__ double scratch[32];
  const int i = blockIdx.x;
  double acc = 0.0;
  for (long long p = rowptr[i] + threadIdx.x; p < rowptr[i + 1]; p += blockDim.x) {
    const int sc = scol[p];
    const long long c = (long long)(sc < 0 ? -sc : sc) - 1 - col_offset;
    if (c >= 0 && c < m_loc) {
      const double x = cvt<double>(v[c]);
      acc += sc < 0 ? -x : x;
    }
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) z[i] = acc * scale;
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
