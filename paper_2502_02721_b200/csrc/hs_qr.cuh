// Incremental projected least-squares solve (solvers.py:204-225, linops.py:168-229).
//
// The reference re-factors the whole sketched system from scratch every
// iteration with a column-pivoted QR (geqp3) and a triangular solve.  Here the
// system grows by one column per iteration, so the factorisation is updated
// instead: the new stacked column a = [z_k ; lam f_k] is orthogonalised
// against Q by classical Gram-Schmidt with one re-orthogonalisation pass
// (CGS2, "twice is enough"), giving R's new column r = c1 + c2 and rho.  The
// inverse R^{-1} is kept too (new column [-R^{-1} r / rho ; 1 / rho]), so the
// solution update  y_k = [y_{k-1} - (beta/rho) R^{-1} r ; beta/rho]  with
// beta = q_k^T rhs is a triangular mat-vec instead of a serial back-solve.
// Everything is fp64.  One cooperative kernel, NB blocks owning row slices of
// the stacked system, 5 grid-wide barriers.  Then sres = |Z y - S r0| and
// proj_obj = sqrt(sres^2 + lam^2 |F y|^2) exactly as solvers.py:514-520 form them.
//
// Rank test and fallback: the reference raises RankDeficiencyError when
// min|R_ii| < 1e-14 max|R_ii| of the PIVOTED QR (linops.py:197-203) and then
// takes the minimum-norm least-squares solution (np.linalg.lstsq, solvers.py:
// 211-218); once the sketched system is deficient it stays deficient, so every
// later iteration takes the fallback too.  Here the same 1e-14 test is applied
// to the new column's rho.  A dependent column j is dropped from the QR (zero
// Q column, zero R^{-1} row/column), which makes y_b, the solution the update
// formula carries, the BASIC solution (y_j = 0).  Its null vector
// n_j = e_j - R^{-1} r_j (r_j = the column's coefficients against Q) is
// orthonormalised (CGS2) against the earlier ones into Nnull, and the reported
// solution is the minimum-norm one, y = y_b - N (N^T y_b): the lstsq answer
// with the dependent directions truncated.  rank_fallback is set from the
// first dropped column on, as in the reference (tests/test_gpu_parity.py:
// test_rank_fallback_min_norm_vs_reference).
#pragma once

#include <cooperative_groups.h>

#include "hs_common.cuh"
#include "hs_loop.cuh"

namespace hs {

struct QrArgs {
  int ell, Ls, ldq, kmax;
  double lam;
  const double* zcol;   // new column of Z (ell)
  const double* fcol;   // new column of F (ell) or null
  const double* Z;      // ell x kmax (ld = ell)
  const double* F;      // ell x (kmax+1) (ld = ell) or null
  const double* sr0;    // ell
  double* Q;            // ldq x kmax
  double* Rinv;         // kmax x kmax, row-major (Rinv[i * kmax + l] = (R^{-1})_{il})
  double* Rdiag;        // kmax
  double* y;            // kmax (current solution)
  double* Yhist;        // kmax x kmax: y^{(k)} in column k-1
  double* part;         // scratch: 4 buffers of NB x (kmax + 2)
  double* sres;         // kmax
  double* proj;         // kmax
  int* rankfb;          // kmax
  double* Nnull = nullptr;  // kmax x kmax: orthonormal null vectors of the dropped columns
  int* ndrop = nullptr;     // number of dropped columns so far
  unsigned int* qdone = nullptr;  // arrival counter for the last-block residual reduction (null: grid barrier)
  LoopState* st;
};

// CTAs of one projected-solve step: ~48 rows each, at most 64
inline int qr_blocks(int Ls) { return Ls < 48 ? 1 : (Ls + 47) / 48 < 64 ? (Ls + 47) / 48 : 64; }

// dynamic shared memory of qr_step_kernel
// The block's slice of Q (RS rows x the kmax columns, fp64) is staged in
// shared memory at the start of every step when it fits (configs 1-5: 36-115
// KB), so the Gram-Schmidt passes read it from shared memory instead of
// walking L2 round trips column after column.
constexpr size_t QR_SMEM_CAP = 200 * 1024;
__host__ __device__ inline size_t qr_smem_base(int Ls, int NB, int kmax) {
  return (2 * (size_t)((Ls + NB - 1) / NB) + 4 * (size_t)kmax + 256) * sizeof(double);
}
__host__ __device__ inline bool qr_q_in_smem(int Ls, int NB, int kmax) {
  return qr_smem_base(Ls, NB, kmax) + (size_t)((Ls + NB - 1) / NB) * kmax * sizeof(double) <= QR_SMEM_CAP;
}
inline size_t qr_smem_bytes(int Ls, int NB, int kmax) {
  return qr_smem_base(Ls, NB, kmax) +
         (qr_q_in_smem(Ls, NB, kmax) ? (size_t)((Ls + NB - 1) / NB) * kmax * sizeof(double) : 0);
}

// out[i] = sum_{r < nr} Q[i*ldq + r] * v[r] for i < j: one warp per column,
// lanes over the rows (then a shuffle sum); four columns per warp pass so
// their loads are in flight together.  The per-column order is fixed.
__device__ __forceinline__ void block_dots(const double* __restrict__ Q, int ldq, int j, const double* v, int nr,
                                           double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int i0 = warp; i0 < j; i0 += 4 * nwarps) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = lane; r < nr; r += 32) {
      const double vr = v[r];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nwarps;
        if (i < j) s[u] = fma(Q[(long long)i * ldq + r], vr, s[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double t = warp_sum(s[u]);
      const int i = i0 + u * nwarps;
      if (lane == 0 && i < j) out[i] = t;
    }
  }
}

__device__ __forceinline__ double block_max(double v, double* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  double r = scratch[0];
  for (int i = 1; i < nw; ++i) r = fmax(r, scratch[i]);
  __syncthreads();
  return r;
}

// out[r] = sum_{i < ncol} elem(i, r) * coef[i] for r < nr (256 threads): four
// column groups of 64 threads (i = g, g+4, ...; each warp reads 32
// consecutive rows of one column), partials combined as (p0+p1)+(p2+p3).
// A fixed order; the dependent fma chain is ncol/4 long instead of ncol.
template <class F>
__device__ __forceinline__ void split_rows(int nr, int ncol, const double* coef, F elem, double* red, double* out) {
  const int t = threadIdx.x, g = t >> 6, rr = t & 63;
  for (int rb = 0; rb < nr; rb += 64) {
    const int r = rb + rr;
    double s = 0.0;
    if (r < nr) {
#pragma unroll 8
      for (int i = g; i < ncol; i += 4) s = fma(elem(i, r), coef[i], s);
    }
    red[g * 64 + rr] = s;
    __syncthreads();
    if (t < 64 && rb + t < nr) out[rb + t] = (red[t] + red[64 + t]) + (red[128 + t] + red[192 + t]);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) qr_step_kernel(QrArgs a, int k, int iter) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  if (a.st->bd_iter != 0 && a.st->bd_iter < iter) return;  // uniform across the grid
  extern __shared__ double sm[];
  const int NB = gridDim.x, b = blockIdx.x, tid = threadIdx.x, BT = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = BT >> 5;
  const int j = k - 1;  // new column index
  const int d0 = *a.ndrop;  // read before block 0 can change it (phase 4, after three barriers)
  const int RS = (a.Ls + NB - 1) / NB;
  const int r0 = b * RS, r1 = min(a.Ls, r0 + RS);
  const int nr = max(0, r1 - r0);
  const int pld = a.kmax + 2;
  double* P1 = a.part;
  double* P2 = a.part + (long long)NB * pld;
  double* P3 = a.part + 2LL * NB * pld;
  double* P5 = a.part + 3LL * NB * pld;
  double* av = sm;            // RS
  double* cv = sm + RS;       // kmax (c1, then c2)
  double* c1s = cv + a.kmax;  // kmax (saved c1)
  double* wv = c1s + a.kmax;  // kmax (R^{-1} r of the new column / null vector)
  double* gv = wv + a.kmax;   // kmax (projection coefficients)
  double* red = gv + a.kmax;  // 256 (split_rows partials)
  double* mv = red + 256;     // RS (split_rows results)
  // this block's rows of Q: shared memory (column i at Qs[i * RS]) or global
  const bool qsm = qr_q_in_smem(a.Ls, NB, a.kmax);
  double* Qs = mv + RS;
  if (qsm) {
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(Qs);
    for (int idx = tid; idx < j * nr; idx += BT) {
      const int i = idx / nr, r = idx - i * nr;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + (unsigned)((i * RS + r) * 8)),
                   "l"(a.Q + (long long)i * a.ldq + r0 + r));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  const double* Qb = qsm ? Qs : a.Q + r0;
  const long long ldq = qsm ? RS : a.ldq;
  __shared__ double scratch[32];

  // phase 1: load the new stacked column, partial Q^T a
  for (int r = tid; r < nr; r += BT) {
    const int gr = r0 + r;
    av[r] = gr < a.ell ? a.zcol[gr] : a.lam * a.fcol[gr - a.ell];
  }
  __syncthreads();
  block_dots(Qb, (int)ldq, j, av, nr, P1 + (long long)b * pld);
  grid.sync();

  // phase 2: c1 = sum_b P1;  a -= Q c1;  partial Q^T a
  for (int i = tid; i < j; i += BT) {
    double s = 0.0;
    #pragma unroll 8
    for (int bb = 0; bb < NB; ++bb) s += __ldcg(&P1[(long long)bb * pld + i]);
    cv[i] = s;
    c1s[i] = s;
  }
  __syncthreads();
  split_rows(nr, j, cv, [&](int i, int r) { return Qb[(long long)i * ldq + r]; }, red, mv);
  for (int r = tid; r < nr; r += BT) av[r] -= mv[r];
  __syncthreads();
  block_dots(Qb, (int)ldq, j, av, nr, P2 + (long long)b * pld);
  grid.sync();

  // phase 3: c2 = sum_b P2;  a -= Q c2;  partial |a|^2 and a^T rhs
  for (int i = tid; i < j; i += BT) {
    double s = 0.0;
    #pragma unroll 8
    for (int bb = 0; bb < NB; ++bb) s += __ldcg(&P2[(long long)bb * pld + i]);
    cv[i] = s;
  }
  __syncthreads();
  split_rows(nr, j, cv, [&](int i, int r) { return Qb[(long long)i * ldq + r]; }, red, mv);
  double nn = 0.0, ar = 0.0;
  for (int r = tid; r < nr; r += BT) {
    const double v = av[r] - mv[r];
    av[r] = v;
    nn = fma(v, v, nn);
    const int gr = r0 + r;
    if (gr < a.ell) ar = fma(v, a.sr0[gr], ar);
  }
  nn = block_sum(nn, scratch);
  ar = block_sum(ar, scratch);
  if (tid == 0) {
    P3[(long long)b * pld + 0] = nn;
    P3[(long long)b * pld + 1] = ar;
  }
  grid.sync();

  // phase 4: rho, beta; new Q column; block 0 updates R^{-1}, y
  double rho2 = 0.0, g = 0.0;
#pragma unroll 8
  for (int bb = 0; bb < NB; ++bb) {
    rho2 += __ldcg(&P3[(long long)bb * pld + 0]);
    g += __ldcg(&P3[(long long)bb * pld + 1]);
  }
  const double rho = sqrt(rho2);
  // max |R_ii| (order-free): strided partial maxima, block reduction
  double rmax = 0.0;
  for (int i = tid; i < j; i += BT) rmax = fmax(rmax, fabs(a.Rdiag[i]));
  rmax = fmax(rho, block_max(rmax, scratch));
  const bool deficient = !(rho > 0.0) || rho < 1e-14 * rmax;
  for (int r = tid; r < nr; r += BT) a.Q[(long long)j * a.ldq + r0 + r] = deficient ? 0.0 : av[r] / rho;
  // Common case (a full-rank step, no column ever dropped): every block forms
  // y^{(k)} itself (y^{(k-1)} is Yhist's previous column; the same operations
  // in the same order in every block), so phase 5 needs no barrier; block 0
  // alone writes R^{-1}, y, Yhist.  Otherwise block 0 does the rank-fallback
  // work below and a grid barrier publishes the result.
  const bool fast = !deficient && d0 == 0;  // uniform across the grid
  double* ys = cv;
  if (fast) {
    ys = gv;
    const double eta = (g / rho) / rho;
    for (int i0 = warp * 4; i0 < j; i0 += nwarps * 4) {
      double sr[4] = {0.0, 0.0, 0.0, 0.0};
      for (int l = i0 + lane; l < j; l += 32) {
        const double cl = c1s[l] + cv[l];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u < j && l >= i0 + u) sr[u] = fma(a.Rinv[(long long)(i0 + u) * a.kmax + l], cl, sr[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        const double sv = warp_sum(sr[u]);
        if (lane == 0 && i < j) {
          const double yi = a.Yhist[(long long)(j - 1) * a.kmax + i] - eta * sv;
          ys[i] = yi;
          if (b == 0) {
            a.Rinv[(long long)i * a.kmax + j] = -sv / rho;
            a.y[i] = yi;
            a.Yhist[(long long)j * a.kmax + i] = yi;
          }
        }
      }
    }
    if (tid == 0) {
      ys[j] = eta;
      if (b == 0) {
        a.Rinv[(long long)j * a.kmax + j] = 1.0 / rho;
        a.Rdiag[j] = rho;
        a.y[j] = eta;
        a.Yhist[(long long)j * a.kmax + j] = eta;
        a.rankfb[j] = 0;
      }
    }
    __syncthreads();
  } else if (b == 0) {
    const double eta = deficient ? 0.0 : (g / rho) / rho;  // beta / rho, beta = q^T rhs = g / rho
    // w = Rinv[0:j, 0:j] (c1 + c2)
    // (R^{-1} is stored row-major: a warp reads row i contiguously)
    // four rows per warp pass, so their loads are in flight together
    for (int i0 = warp * 4; i0 < j; i0 += nwarps * 4) {
      double sr[4] = {0.0, 0.0, 0.0, 0.0};
      for (int l = i0 + lane; l < j; l += 32) {
        const double cl = c1s[l] + cv[l];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i0 + u < j && l >= i0 + u) sr[u] = fma(a.Rinv[(long long)(i0 + u) * a.kmax + l], cl, sr[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        const double sv = warp_sum(sr[u]);
        if (lane == 0 && i < j) {
          const double yi = a.y[i] - eta * sv;
          a.Rinv[(long long)i * a.kmax + j] = deficient ? 0.0 : -sv / rho;
          a.y[i] = yi;
          a.Yhist[(long long)j * a.kmax + i] = yi;
          wv[i] = -sv;
        }
      }
    }
    if (tid == 0) {
      a.Rinv[(long long)j * a.kmax + j] = deficient ? 0.0 : 1.0 / rho;
      a.Rdiag[j] = deficient ? 0.0 : rho;
      a.y[j] = eta;
      a.Yhist[(long long)j * a.kmax + j] = eta;
      wv[j] = 1.0;
    }
    __syncthreads();
    int d = *a.ndrop;  // uniform
    double* N = a.Nnull;
    if (deficient) {
      // n_j = e_j - R^{-1} r_j, orthonormalised against the earlier null vectors (CGS2)
      for (int pass = 0; pass < 2 && d > 0; ++pass) {
        for (int t = warp; t < d; t += nwarps) {
          const double* nt = N + (long long)t * a.kmax;
          double s = 0.0;
          for (int i = lane; i <= j; i += 32) s = fma(nt[i], wv[i], s);
          s = warp_sum(s);
          if (lane == 0) gv[t] = s;
        }
        __syncthreads();
        for (int i = tid; i <= j; i += BT) {
          double s = 0.0;
          for (int t = 0; t < d; ++t) s = fma(N[(long long)t * a.kmax + i], gv[t], s);
          wv[i] -= s;
        }
        __syncthreads();
      }
      double nn2 = 0.0;
      for (int i = tid; i <= j; i += BT) nn2 = fma(wv[i], wv[i], nn2);
      nn2 = block_sum(nn2, scratch);
      const double inv = 1.0 / sqrt(nn2);
      double* nd = N + (long long)d * a.kmax;
      for (int i = tid; i < a.kmax; i += BT) nd[i] = i <= j ? wv[i] * inv : 0.0;
      ++d;
      __syncthreads();
      if (tid == 0) *a.ndrop = d;
    }
    if (d > 0) {
      // minimum-norm solution: y = y_b - N (N^T y_b)
      double* yh = a.Yhist + (long long)j * a.kmax;
      for (int t = warp; t < d; t += nwarps) {
        const double* nt = N + (long long)t * a.kmax;
        double s = 0.0;
        for (int i = lane; i <= j; i += 32) s = fma(nt[i], yh[i], s);
        s = warp_sum(s);
        if (lane == 0) gv[t] = s;
      }
      __syncthreads();
      for (int i = tid; i <= j; i += BT) {
        double s = 0.0;
        for (int t = 0; t < d; ++t) s = fma(N[(long long)t * a.kmax + i], gv[t], s);
        yh[i] -= s;
      }
    }
    if (tid == 0) a.rankfb[j] = d > 0 ? 1 : 0;
  }
  if (!fast) {
    grid.sync();
    for (int i = tid; i <= j; i += BT) ys[i] = __ldcg(&a.Yhist[(long long)j * a.kmax + i]);
    __syncthreads();
  }

  // phase 5: residual partials |Z y - sr0|^2 (top) and |F y|^2 (bottom)
  const int ell = a.ell;
  const double *Zm = a.Z, *Fm = a.F;
  split_rows(nr, j + 1, ys, [&](int i, int r) {
    const int gr = r0 + r;
    return gr < ell ? Zm[(long long)i * ell + gr] : Fm[(long long)i * ell + gr - ell];
  }, red, mv);
  double s_top = 0.0, s_bot = 0.0;
  for (int r = tid; r < nr; r += BT) {
    const int gr = r0 + r;
    if (gr < a.ell) {
      const double d = mv[r] - a.sr0[gr];
      s_top = fma(d, d, s_top);
    } else {
      s_bot = fma(mv[r], mv[r], s_bot);
    }
  }
  s_top = block_sum(s_top, scratch);
  s_bot = block_sum(s_bot, scratch);
  if (tid == 0) {
    P5[(long long)b * pld + 0] = s_top;
    P5[(long long)b * pld + 1] = s_bot;
  }
  // the last block to arrive sums the partials in block order
  bool reduce = false;
  if (a.qdone) {
    __shared__ bool last;
    if (tid == 0) {
      __threadfence();
      last = atomicAdd(a.qdone, 1u) == (unsigned)NB - 1;
    }
    __syncthreads();
    reduce = last && tid == 0;
    if (reduce) __threadfence();
  } else {
    grid.sync();
    reduce = b == 0 && tid == 0;
  }
  if (reduce) {
    double st = 0.0, sb = 0.0;
    for (int bb = 0; bb < NB; ++bb) {
      st += __ldcg(&P5[(long long)bb * pld + 0]);
      sb += __ldcg(&P5[(long long)bb * pld + 1]);
    }
    a.sres[j] = sqrt(st);
    a.proj[j] = sqrt(st + a.lam * a.lam * sb);
    if (a.qdone) *a.qdone = 0;
  }
}

// Launch one projected-solve step (cooperative grid: the five phase barriers
// are grid-wide).  Measured: the same kernel as one 16-CTA thread-block
// cluster (hardware cluster barriers) was no faster in isolation (61 vs 58 us
// per step at config 2 -- the phases are latency chains, not barrier-bound)
// and slower inside the config-4 solve (fewer CTAs, and a 16-SM cluster slot
// is harder to find beside the SpMV).
inline cudaError_t launch_qr_step(const QrArgs& qa, int k, int iter, int NB, size_t smem, cudaStream_t s) {
  QrArgs a = qa;
  void* args[] = {&a, &k, &iter};
  return cudaLaunchCooperativeKernel((void*)qr_step_kernel, dim3(NB), dim3(256), args, smem, s);
}

// kernel attributes for a step with `smem` bytes of dynamic shared memory
inline cudaError_t prepare_qr_step(size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return ensure_smem((const void*)qr_step_kernel, smem);
}

}  // namespace hs
