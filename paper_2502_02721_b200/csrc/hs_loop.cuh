// Per-iteration kernels of the sketched Hessenberg / sLSLU loop
// (solvers.py:468-538 driving hessenberg.py:191-226 / 329-390).
//
//   fsub_warp_kernel      pivot-row forward substitution -> elimination coefficients
//                         (hessenberg.py:209-212: c_j = u[t_j] after j subtractions)
//   elim_pass_kernel      ONE coalesced pass over the k basis vectors: in-order
//                         u <- u - c_j b_j, fused argmax|u| (smallest index ties,
//                         hessenberg.py:110-114) and, optionally, the iterate
//                         x = L y of the previous iteration (solvers.py:510)
//   pivot_commit_kernel   breakdown test (hessenberg.py:213-219/351-360/375-384),
//                         new H/W entry, pivot position, new pivot-row of P
//   normalize_kernel      basis_{k+1} = u / pivot (true IEEE division, hessenberg.py:222)
//   xpass_kernel          x = x0 + L_k y with the relative error partials (solvers.py:236-240)
#pragma once

#include <cooperative_groups.h>

#include <algorithm>

#include "hs_common.cuh"

namespace hs {

// device-side loop state shared by the kernels of one solve
struct LoopState {
  int bd_iter;       // iteration at which a breakdown happened (0 = none)
  int bd_side;       // 0 = data / square side, 1 = solution side
  int trivial;       // init found a zero residual
  int pad0;
  double piv_val[2]; // latest pivot value per side (as double; exact for float/double)
  long long piv_idx[2];
  unsigned int counter[4];  // last-block counters (reset by the last block)
  double relerr_acc;
};

// --------------------------------------------------------------------------
// forward substitution on the pivot rows, one warp.
// P is column-major with leading dimension ldp: P[i*ldp + j] = b_i[pos_j]
// (unit lower triangular: P[j*ldp + j] = 1).  For j = 0..k-1 in order:
//   c_j = v_j,   v_i <- v_i - c_j * P[j*ldp + i]   (i > j)
// which is bit-identical to reading u[t_j] inside the sequential loop.
template <class T, int S>
__global__ void __launch_bounds__(32)
fsub_warp_kernel(const T* __restrict__ u, const long long* __restrict__ pos, long long pos_offset,
                 const T* __restrict__ P, int ldp, const int* __restrict__ kptr, int kfixed,
                 const LoopState* __restrict__ st, int iter, int side, T* __restrict__ c,
                 double* __restrict__ hcol) {
  if (st->bd_iter != 0 && st->bd_iter < iter) return;
  if (side == 1 && st->bd_iter == iter) return;  // data side broke down this iteration
  const int k = kptr ? *kptr : kfixed;
  const int lane = threadIdx.x;
  T v[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int j = s * 32 + lane;
    v[s] = (j < k) ? u[pos[j] - pos_offset] : T(0);
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    if (s * 32 >= k) break;
    for (int o = 0; o < 32; ++o) {
      const int j = s * 32 + o;
      if (j >= k) break;
      const T cj = __shfl_sync(0xffffffffu, v[s], o);
      if (lane == 0) {
        c[j] = cj;
        hcol[j] = (double)cj;
      }
      const T* Pj = P + (long long)j * ldp;
#pragma unroll
      for (int s2 = s; s2 < S; ++s2) {
        const int i = s2 * 32 + lane;
        if (i > j && i < k) v[s2] = Rn<T>::sub(v[s2], Rn<T>::mul(cj, Pj[i]));
      }
    }
  }
}

// Blocked version (one CTA): the same per-row operation sequence
//   v_j <- (((v_j - c_0 P_j0) - c_1 P_j1) - ...)   (i ascending)
// organised in diagonal blocks of 32 unknowns.  Warp 0 solves a diagonal
// block serially (its 32x32 slice of P prefetched into registers, c_i
// broadcast by shuffle); then every thread applies the block's 32 new c_i to
// the rows it owns, in i order.  Bit-identical to the serial loop, with a
// critical path of ~k shuffles instead of k global-latency steps.
template <class T>
__global__ void __launch_bounds__(512)
fsub_block_kernel(const T* __restrict__ u, const long long* __restrict__ pos, long long pos_offset,
                  const T* __restrict__ P, int ldp, int k, const LoopState* __restrict__ st, int iter, int side,
                  T* __restrict__ c, double* __restrict__ hcol) {
  if (st->bd_iter != 0 && st->bd_iter < iter) return;
  if (side == 1 && st->bd_iter == iter) return;
  extern __shared__ unsigned char smem_raw[];
  T* v = reinterpret_cast<T*>(smem_raw);  // k values
  for (int j = threadIdx.x; j < k; j += blockDim.x) v[j] = u[pos[j] - pos_offset];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b0 = 0; b0 < k; b0 += 32) {
    const int nb = min(32, k - b0);
    if (warp == 0) {
      const int j = b0 + lane;
      T Pd[32];
#pragma unroll
      for (int o = 0; o < 32; ++o) Pd[o] = (o < nb && j < k) ? P[(long long)(b0 + o) * ldp + j] : T(0);
      T vj = j < k ? v[j] : T(0);
#pragma unroll
      for (int o = 0; o < 32; ++o) {
        if (o < nb) {
          const T co = __shfl_sync(0xffffffffu, vj, o);
          if (lane > o && lane < nb) vj = Rn<T>::sub(vj, Rn<T>::mul(co, Pd[o]));
        }
      }
      if (lane < nb) {
        v[j] = vj;
        c[j] = vj;
        hcol[j] = (double)vj;
      }
    }
    __syncthreads();
    // rows below the block take the block's contributions in i order
    for (int j = b0 + nb + threadIdx.x; j < k; j += blockDim.x) {
      T vj = v[j];
      for (int o = 0; o < nb; ++o) vj = Rn<T>::sub(vj, Rn<T>::mul(v[b0 + o], P[(long long)(b0 + o) * ldp + j]));
      v[j] = vj;
    }
    __syncthreads();
  }
}

// Panel version (the default): the same blocked sequence, with P read from
// shared memory.  Panel b (columns b0..b0+31 of P, rows b0..k-1) is copied by
// cp.async while panel b-1 is being used, so the solve walks shared memory
// instead of one L2 round trip per diagonal block and per trailing update
// (config 2: ~21 us -> see DESIGN.md).  Per row the operations and their
// order are those of fsub_block_kernel: bit-identical.
template <class T>
__device__ __forceinline__ void fsub_panel_copy(const T* __restrict__ P, int ldp, int b0, int k, T* dst) {
  const int W = k - b0;
  const int nb = min(32, W);
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(dst);
  for (int idx = threadIdx.x; idx < nb * W; idx += blockDim.x) {
    const int o = idx / W, jj = idx - o * W;
    const T* src = P + (long long)(b0 + o) * ldp + b0 + jj;
    if (sizeof(T) == 8)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + (unsigned)(idx * 8)), "l"(src));
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sbase + (unsigned)(idx * 4)), "l"(src));
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

inline size_t fsub_panel_smem(int k, size_t tsize) { return ((size_t)k + 2 * 32 * (size_t)k) * tsize; }

// the whole forward substitution, run by every thread of ONE block (smem_raw:
// fsub_panel_smem(k) bytes, 128-byte aligned)
template <class T>
__device__ __forceinline__ void fsub_panel_body(const T* __restrict__ u, const long long* __restrict__ pos,
                                                long long pos_offset, const T* __restrict__ P, int ldp, int k,
                                                T* __restrict__ c, double* __restrict__ hcol,
                                                unsigned char* smem_raw);

template <class T>
__global__ void __launch_bounds__(256)
fsub_panel_kernel(const T* __restrict__ u, const long long* __restrict__ pos, long long pos_offset,
                  const T* __restrict__ P, int ldp, int k, const LoopState* __restrict__ st, int iter, int side,
                  T* __restrict__ c, double* __restrict__ hcol) {
  if (st->bd_iter != 0 && st->bd_iter < iter) return;
  if (side == 1 && st->bd_iter == iter) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  fsub_panel_body<T>(u, pos, pos_offset, P, ldp, k, c, hcol, smem_raw);
}

template <class T>
__device__ __forceinline__ void fsub_panel_body(const T* __restrict__ u, const long long* __restrict__ pos,
                                                long long pos_offset, const T* __restrict__ P, int ldp, int k,
                                                T* __restrict__ c, double* __restrict__ hcol,
                                                unsigned char* smem_raw) {
  T* v = reinterpret_cast<T*>(smem_raw);  // k values
  T* pan[2] = {v + k, v + k + 32 * k};    // two panels of <= 32 x k
  const int nbt = (k + 31) / 32;
  fsub_panel_copy<T>(P, ldp, 0, k, pan[0]);
  for (int j = threadIdx.x; j < k; j += blockDim.x) v[j] = u[pos[j] - pos_offset];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = 0; b < nbt; ++b) {
    const int b0 = b * 32, nb = min(32, k - b0), W = k - b0;
    if (b + 1 < nbt) {
      fsub_panel_copy<T>(P, ldp, b0 + 32, k, pan[(b + 1) & 1]);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const T* pn = pan[b & 1];  // pn[o * W + (j - b0)] = P[(b0 + o) * ldp + j]
    if (warp == 0) {
      const int j = b0 + lane;
      T vj = lane < nb ? v[j] : T(0);
#pragma unroll
      for (int o = 0; o < 32; ++o) {
        if (o < nb) {
          const T co = __shfl_sync(0xffffffffu, vj, o);
          if (lane > o && lane < nb) vj = Rn<T>::sub(vj, Rn<T>::mul(co, pn[o * W + lane]));
        }
      }
      if (lane < nb) {
        v[j] = vj;
        c[j] = vj;
        hcol[j] = (double)vj;
      }
    }
    __syncthreads();
    for (int j = b0 + nb + threadIdx.x; j < k; j += blockDim.x) {
      T vj = v[j];
      for (int o = 0; o < nb; ++o) vj = Rn<T>::sub(vj, Rn<T>::mul(v[b0 + o], pn[o * W + (j - b0)]));
      v[j] = vj;
    }
    __syncthreads();
  }
}

// forward substitution for k pivot rows (one CTA); every call site goes through here
template <class T>
inline void launch_fsub(cudaStream_t s, const T* u, const long long* pos, const T* P, int ldp, int k,
                        const LoopState* st, int iter, int side, T* c, double* hcol) {
  if (k <= 0) return;
  const size_t smem = fsub_panel_smem(k, sizeof(T));
  static const bool legacy = [] {
    const char* e = getenv("HS_FSUB_LEGACY");  // A/B knob: the register-blocked kernels below
    return e && *e && *e != '0';
  }();
  if (smem <= 200 * 1024 && !legacy) {
    if (smem > 48 * 1024) ensure_smem((const void*)fsub_panel_kernel<T>, 200 * 1024);
    fsub_panel_kernel<T><<<1, 256, smem, s>>>(u, pos, 0, P, ldp, k, st, iter, side, c, hcol);
  } else if (k <= 64) {
    fsub_warp_kernel<T, 2><<<1, 32, 0, s>>>(u, pos, 0, P, ldp, nullptr, k, st, iter, side, c, hcol);
  } else {
    fsub_block_kernel<T><<<1, 512, (size_t)k * sizeof(T), s>>>(u, pos, 0, P, ldp, k, st, iter, side, c, hcol);
  }
}

// --------------------------------------------------------------------------
// vector load helpers for the basis pass
template <class B, int VEC> struct VecLoad;
template <class B> struct VecLoad<B, 1> {
  static __device__ __forceinline__ void ld(const B* p, B (&o)[1]) { o[0] = __ldg(p); }
};
template <> struct VecLoad<float, 4> {
  static __device__ __forceinline__ void ld(const float* p, float (&o)[4]) {
    // basis columns are read once per pass: evict-first (+2% on the config-4 pass over __ldg)
    float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
  }
};
template <> struct VecLoad<double, 2> {
  static __device__ __forceinline__ void ld(const double* p, double (&o)[2]) {
    double2 t = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = t.x; o[1] = t.y;
  }
};
template <> struct VecLoad<__nv_bfloat16, 8> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, __nv_bfloat16 (&o)[8]) {
    uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&t);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = b[i];
  }
};

// --------------------------------------------------------------------------
// the fused elimination pass.
//   u[e] <- (((u[e] - c_0 b_0[e]) - c_1 b_1[e]) ...)      (k terms, in order)
//   x[e]  = x0[e] + sum_{j<kx} y_j b_j[e]                  (optional, fp64)
// plus argmax |u'| and sum (x - x_true)^2 partials; the last block to finish
// reduces the partials (fixed order) into st->piv_* / relerr slot.
template <class T, class B, int VEC, bool XF>
__device__ __forceinline__ void elim_strips(long long n, long long idx_offset, const B* __restrict__ basis, long long ld,
                                            int k, const T* cs, const T* u, int kx, const double* ys,
                                            double* __restrict__ xout, const double* __restrict__ x0,
                                            const double* __restrict__ xt, int write_u, T* uo, Cand& best,
                                            double& sq);

// Resident blocks per SM of the fp32 / fp32-basis pass (config 4), measured in
// the solve (bench.py kernels table, GB/s of the pass's algorithmic bytes):
// plain launch bounds (44 / 64 registers, 5 / 4 blocks) 4.99 / 5.57 TB/s for
// the D / L side; 7 / 6 blocks (36 / 40 registers) with four basis columns in
// flight per thread and evict-first loads 6.05 / 5.99 TB/s = 0.94 / 0.93 of
// the copy peak (6 / 5 blocks: 5.63 / 5.13; 8 / 8: 6.05 / 5.67).
#ifndef HS_ELIM_MINB_L
#define HS_ELIM_MINB_L 6
#endif
#ifndef HS_ELIM_MINB_D
#define HS_ELIM_MINB_D 7
#endif
template <class T, class B, int VEC, bool XF>
__global__ void __launch_bounds__(256, (VEC == 4 && sizeof(T) == 4) ? (XF ? HS_ELIM_MINB_L : HS_ELIM_MINB_D) : 0)
elim_pass_kernel(long long n, long long idx_offset, const B* __restrict__ basis, long long ld,
                 const int* __restrict__ kptr, int kfixed, const T* __restrict__ cvec, const T* u,
                 int kx, const double* __restrict__ yx, double* __restrict__ xout,
                 const double* __restrict__ x0, const double* __restrict__ xt,
                 double* __restrict__ xpart, double* __restrict__ relerr_out,
                 Cand* __restrict__ cand_part, LoopState* __restrict__ st, int side, int iter,
                 int write_u, T* uo) {
  if (st->bd_iter != 0 && st->bd_iter < iter) return;
  if (side == 1 && st->bd_iter == iter) return;  // data side broke down this iteration
  extern __shared__ unsigned char smem_raw[];
  const int k = kptr ? *kptr : kfixed;
  T* cs = reinterpret_cast<T*>(smem_raw);
  double* ys = reinterpret_cast<double*>(smem_raw + ((k * sizeof(T) + 15) / 16) * 16);
  __shared__ Cand scratch[32];
  __shared__ double dscratch[32];
  __shared__ bool am_last;
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = cvec[i];
  for (int i = threadIdx.x; i < kx; i += blockDim.x) ys[i] = yx[i];
  __syncthreads();

  Cand best{-1.0, 0.0, 0x7fffffffffffffffLL};
  double sq = 0.0;
  elim_strips<T, B, VEC, XF>(n, idx_offset, basis, ld, k, cs, u, kx, ys, xout, x0, xt, write_u, uo, best, sq);
  best = block_argmax(best, scratch);
  if (XF && kx > 0 && xt) sq = block_sum(sq, dscratch);
  if (threadIdx.x == 0) {
    cand_part[blockIdx.x] = best;
    if (XF && kx > 0 && xt) xpart[blockIdx.x] = sq;
    __threadfence();
    const unsigned prev = atomicAdd(&st->counter[side], 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  Cand b2{-1.0, 0.0, 0x7fffffffffffffffLL};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
    Cand c;
    c.mag = __ldcg(&cand_part[i].mag);
    c.val = __ldcg(&cand_part[i].val);
    c.idx = __ldcg(&cand_part[i].idx);
    cand_merge(b2, c);
  }
  b2 = block_argmax(b2, scratch);
  if (XF && kx > 0 && xt && relerr_out) {
    // fixed-order parallel sum of the block partials (deterministic)
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(&xpart[i]);
    s = block_sum(s, dscratch);
    if (threadIdx.x == 0) *relerr_out = s;  // squared norm; the host divides by |x_true|
  }
  if (threadIdx.x == 0) {
    st->piv_val[side] = b2.val;
    st->piv_idx[side] = b2.idx;
    st->counter[side] = 0;
  }
}

// the strips of one thread (grid-stride over the VEC-wide strips): in-order
// elimination, fused iterate, running argmax candidate and error partial
template <class T, class B, int VEC, bool XF>
__device__ __forceinline__ void elim_strips(long long n, long long idx_offset, const B* __restrict__ basis, long long ld,
                                            int k, const T* cs, const T* u, int kx, const double* ys,
                                            double* __restrict__ xout, const double* __restrict__ x0,
                                            const double* __restrict__ xt, int write_u, T* uo, Cand& best,
                                            double& sq) {
  const long long nvec = (n + VEC - 1) / VEC;
  // one VEC-wide strip per thread (grid covers the vector exactly: no tail wave)
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (long long)gridDim.x * blockDim.x) {
    const long long e0 = v * VEC;
    T acc[VEC];
    T xa[VEC];  // fused iterate of the previous iteration: accumulated in T (fp32 FMA in the
                // fp32 path: converting every basis value to fp64 would bind the pass to the
                // FP64 pipe; the final x is recomputed in fp64 by xpass_kernel)
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      acc[q] = (e0 + q < n) ? u[e0 + q] : T(0);
      xa[q] = T(0);
    }
    const B* bp = basis + e0;
    // kx <= k always (x of the previous iteration uses the first k-1 columns)
#ifndef HS_ELIM_UNR_D
#define HS_ELIM_UNR_D 4
#endif
#ifndef HS_ELIM_UNR_L
#define HS_ELIM_UNR_L 4
#endif
    constexpr int UNR = VEC == 1 ? 16 : (XF ? HS_ELIM_UNR_L : HS_ELIM_UNR_D);
#pragma unroll UNR
    for (int j = 0; j < k; ++j) {
      B b[VEC];
      VecLoad<B, VEC>::ld(bp + (long long)j * ld, b);
      const T cj = cs[j];
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[q] = Rn<T>::sub(acc[q], Rn<T>::mul(cj, cvt<T>(b[q])));
      if (XF && j < kx) {
        const T yj = (T)ys[j];
#pragma unroll
        for (int q = 0; q < VEC; ++q) xa[q] = fma(yj, cvt<T>(b[q]), xa[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      const long long e = e0 + q;
      if (e < n) {
        if (write_u) uo[e] = acc[q];  // uo may alias u (read above, same element)
        const double mg = (double)absval(acc[q]);
        if (better(mg, idx_offset + e, best.mag, best.idx)) best = Cand{mg, (double)acc[q], idx_offset + e};
        if (XF && kx > 0) {
          double xe = (double)xa[q] + (x0 ? x0[e] : 0.0);
          if (xout) xout[e] = xe;
          if (xt) {
            const double d = xe - xt[e];
            sq = fma(d, d, sq);
          }
        }
      }
    }
  }
}

// --------------------------------------------------------------------------
// pivot bookkeeping after the pass, one block.
//   dim     : m or n (full-basis breakdown without scanning when k >= dim)
//   hcol    : H(:,k-1) or W(:,k) column (entry k gets the pivot or 0)
//   pos     : pivot positions (pos[k] = new pivot, global index)
//   P       : pivot-row matrix, column-major ld = ldp; new row k
//   basis   : basis columns 0..k-1 (to gather b_i[new pivot]); local shard
template <class T, class B>
__global__ void pivot_commit_kernel(int k, long long dim, double* __restrict__ hcol, long long* __restrict__ pos,
                                    T* __restrict__ P, int ldp, const B* __restrict__ basis, long long ld,
                                    long long idx_offset, long long n_loc, LoopState* __restrict__ st,
                                    int side, int iter, T* __restrict__ pivval_out) {
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
  const long long le = idx - idx_offset;
  for (int i = threadIdx.x; i <= k; i += blockDim.x) {
    T pv;
    if (i == k) pv = T(1);
    else pv = (le >= 0 && le < n_loc) ? cvt<T>(basis[(long long)i * ld + le]) : T(0);
    P[(long long)i * ldp + k] = pv;
  }
}

// basis_{k+1}[e] = u[e] / pivot (IEEE division in T, then stored as B); zero padding
template <class T, class B>
__global__ void __launch_bounds__(256)
normalize_kernel(long long n, long long n_pad, const T* __restrict__ u, const T* __restrict__ pivval,
                 B* __restrict__ dst, const LoopState* __restrict__ st, int side, int iter,
                 SinoBlk blk = SinoBlk{0, 0, 0, 0}, B* __restrict__ yb = nullptr) {
  if (st->bd_iter != 0 && st->bd_iter <= iter) return;
  const T p = *pivval;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // four grid-strided elements per step: their loads are in flight together
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < n_pad; e0 += 4 * stride) {
    T uu[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long e = e0 + i * stride;
      uu[i] = e < n ? u[e] : T(0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long e = e0 + i * stride;
      if (e >= n_pad) break;
      const B v = (e < n) ? cvt<B>(Rn<T>::div(uu[i], p)) : cvt<B>(T(0));
      dst[e] = v;
      // the next A^T apply's input, already in the blocked sinogram layout
      if (yb != nullptr && e < n) yb[blk.map32((int)e)] = v;
    }
  }
}

// --------------------------------------------------------------------------
// One basis step as ONE cooperative kernel, for short vectors (configs 1-3,
// where the step is a chain of latency-bound launches): forward substitution
// (block 0) | grid barrier | elimination pass with the fused iterate and the
// per-block argmax candidates (all blocks) | barrier | candidate merge, error
// sum, pivot commit (block 0) | barrier | normalisation (all blocks).  Every
// phase runs the device code of the separate kernels above on the same
// operands in the same order, so pivots, H / W, P and the bases are
// bit-identical to the launch-per-phase path (the relative-error sum alone is
// grouped by this kernel's grid).  Not used with sampled pivoting (the sample
// pick sits between the pass and the commit) or on shards.
template <class T, class B>
struct StepArgs {
  // forward substitution
  const T* u;            // operator output (read by fsub and the pass)
  const T* P;            // pivot-row matrix (read), column-major ldp
  T* Pw;                 // the same matrix (row k written by the commit)
  int ldp, k;
  T* c;                  // elimination coefficients (k)
  double* hcol;          // H(:, k-1) or W(:, k): entries 0..k-1 by fsub, entry k by the commit
  // elimination pass
  long long n, ld;
  const B* basis;
  T* uo;                 // eliminated vector
  int kx;
  const double* yx;
  const double* x0;
  const double* xt;
  double* xpart;
  double* relerr_out;
  Cand* cand;
  // commit
  long long dim;
  long long* pos;
  T* pivval;
  // normalisation (do_norm = 0: the caller normalises with its own kernel)
  int do_norm;
  long long n_pad;
  B* dst;
  SinoBlk blk;
  B* yb;
  LoopState* st;
  int side, iter;
};

template <class T, class B, bool XF>
__global__ void __launch_bounds__(256, 2)
basis_step_kernel(const StepArgs<T, B> a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  LoopState* st = a.st;
  // uniform over the grid (nothing below changes bd_iter before the last barrier but block 0's commit)
  if (st->bd_iter != 0 && st->bd_iter < a.iter) return;
  if (a.side == 1 && st->bd_iter == a.iter) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ Cand scratch[32];
  __shared__ double dscratch[32];
  __shared__ Cand winner;
  const int k = a.k;
  if (blockIdx.x == 0) fsub_panel_body<T>(a.u, a.pos, 0, a.P, a.ldp, k, a.c, a.hcol, smem_raw);
  grid.sync();
  T* cs = reinterpret_cast<T*>(smem_raw);
  double* ys = reinterpret_cast<double*>(smem_raw + ((k * sizeof(T) + 15) / 16) * 16);
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = __ldcg(a.c + i);
  for (int i = threadIdx.x; i < a.kx; i += blockDim.x) ys[i] = a.yx[i];
  __syncthreads();
  Cand best{-1.0, 0.0, 0x7fffffffffffffffLL};
  double sq = 0.0;
  elim_strips<T, B, 1, XF>(a.n, 0, a.basis, a.ld, k, cs, a.u, a.kx, ys, nullptr, a.x0, a.xt, 1, a.uo, best, sq);
  best = block_argmax(best, scratch);
  const bool err = XF && a.kx > 0 && a.xt;
  if (err) sq = block_sum(sq, dscratch);
  if (threadIdx.x == 0) {
    a.cand[blockIdx.x] = best;
    if (err) a.xpart[blockIdx.x] = sq;
  }
  grid.sync();
  if (blockIdx.x == 0) {
    Cand b2{-1.0, 0.0, 0x7fffffffffffffffLL};
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
      Cand c;
      c.mag = __ldcg(&a.cand[i].mag);
      c.val = __ldcg(&a.cand[i].val);
      c.idx = __ldcg(&a.cand[i].idx);
      cand_merge(b2, c);
    }
    b2 = block_argmax(b2, scratch);
    if (err && a.relerr_out) {
      double s = 0.0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(&a.xpart[i]);
      s = block_sum(s, dscratch);
      if (threadIdx.x == 0) *a.relerr_out = s;
    }
    if (threadIdx.x == 0) {
      st->piv_val[a.side] = b2.val;
      st->piv_idx[a.side] = b2.idx;
      winner = b2;
    }
    __syncthreads();
    // the commit (pivot_commit_kernel) on the winner
    const double val = (k < a.dim) ? winner.val : 0.0;
    const long long idx = winner.idx;
    if (val == 0.0) {
      if (threadIdx.x == 0) {
        a.hcol[k] = 0.0;
        st->bd_iter = a.iter;
        st->bd_side = a.side;
      }
    } else {
      if (threadIdx.x == 0) {
        a.hcol[k] = val;
        a.pos[k] = idx;
        *a.pivval = (T)val;
      }
      for (int i = threadIdx.x; i <= k; i += blockDim.x) {
        T pv;
        if (i == k) pv = T(1);
        else pv = (idx >= 0 && idx < a.n) ? cvt<T>(a.basis[(long long)i * a.ld + idx]) : T(0);
        a.Pw[(long long)i * a.ldp + k] = pv;
      }
    }
  }
  grid.sync();
  if (!a.do_norm) return;
  if (__ldcg(&st->bd_iter) != 0 && __ldcg(&st->bd_iter) <= a.iter) return;  // block 0's commit may have set it
  const T p = __ldcg(a.pivval);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < a.n_pad;
       e += (long long)gridDim.x * blockDim.x) {
    const B v = (e < a.n) ? cvt<B>(Rn<T>::div(__ldcg(a.uo + e), p)) : cvt<B>(T(0));
    a.dst[e] = v;
    if (a.yb != nullptr && e < a.n) a.yb[a.blk.map32((int)e)] = v;
  }
}

inline size_t basis_step_smem(int k, int kx, size_t tsize) {
  const size_t elim = ((k * tsize + 15) / 16) * 16 + (size_t)kx * sizeof(double) + 16;
  return std::max(fsub_panel_smem(k, tsize), elim);
}

// The same normalisation for a grid x grid image vector (tomography L side),
// also writing the transposed image dstT[c * grid + r] = dst[r * grid + c]:
// the gather layout the next A apply's near-horizontal ray slices read
// (hs_ops.cuh: image_transpose_kernel), formed here through a shared-memory
// tile instead of a separate pass over the new basis column.
template <class T, class B>
__global__ void __launch_bounds__(256)
normalize_transpose_kernel(int grid, long long n_pad, const T* __restrict__ u, const T* __restrict__ pivval,
                           B* __restrict__ dst, B* __restrict__ dstT, const LoopState* __restrict__ st, int iter) {
  if (st->bd_iter != 0 && st->bd_iter <= iter) return;
  __shared__ B tile[32][33];
  const T p = *pivval;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int gy = by + r, gx = bx + tx;
    if (gy < grid && gx < grid) {
      const long long e = (long long)gy * grid + gx;
      const B v = cvt<B>(Rn<T>::div(u[e], p));
      dst[e] = v;
      tile[r][tx] = v;
    }
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int gx = bx + r, gy = by + tx;
    if (gx < grid && gy < grid) dstT[(long long)gx * grid + gy] = tile[tx][r];
  }
  if (blockIdx.x == 0 && blockIdx.y == 0) {  // zero padding [n, n_pad)
    const long long n = (long long)grid * grid;
    for (long long e = n + threadIdx.x; e < n_pad; e += blockDim.x) dst[e] = cvt<B>(T(0));
  }
}

// plain argmax over a vector (init pivots of r0 / A^T r0); result into st->piv_*[side]
template <class T>
__global__ void __launch_bounds__(256)
argmax_kernel(long long n, long long idx_offset, const T* __restrict__ v, Cand* __restrict__ cand_part,
              LoopState* __restrict__ st, int side) {
  __shared__ Cand scratch[32];
  __shared__ bool am_last;
  Cand best{-1.0, 0.0, 0x7fffffffffffffffLL};
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const double mg = (double)absval(v[e]);
    if (better(mg, idx_offset + e, best.mag, best.idx)) best = Cand{mg, (double)v[e], idx_offset + e};
  }
  best = block_argmax(best, scratch);
  if (threadIdx.x == 0) {
    cand_part[blockIdx.x] = best;
    __threadfence();
    const unsigned prev = atomicAdd(&st->counter[side], 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  Cand b2{-1.0, 0.0, 0x7fffffffffffffffLL};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
    Cand c;
    c.mag = __ldcg(&cand_part[i].mag);
    c.val = __ldcg(&cand_part[i].val);
    c.idx = __ldcg(&cand_part[i].idx);
    cand_merge(b2, c);
  }
  b2 = block_argmax(b2, scratch);
  if (threadIdx.x == 0) {
    st->piv_val[side] = b2.val;
    st->piv_idx[side] = b2.idx;
    st->counter[side] = 0;
  }
}

// x = x0 + sum_{j<kx} y_j b_j (fp64, j ascending) with (x - x_true)^2 partials
template <class B>
__global__ void __launch_bounds__(256)
xpass_kernel(long long n, const B* __restrict__ basis, long long ld, int kx, const double* __restrict__ y,
             const double* __restrict__ x0, const double* __restrict__ xt, double* __restrict__ xout,
             double* __restrict__ xpart, double* __restrict__ relerr_out, LoopState* __restrict__ st) {
  extern __shared__ unsigned char smem_raw[];
  double* ys = reinterpret_cast<double*>(smem_raw);
  __shared__ double dscratch[32];
  __shared__ bool am_last;
  for (int i = threadIdx.x; i < kx; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  double sq = 0.0;
  // VEC consecutive elements per thread, one 16-byte load per basis column and
  // eight columns in flight (the columns are padded to ld >= n rounded up to
  // 64, so a strip may read past n); per element the sum is still j-ascending
  constexpr int VEC = 16 / sizeof(B);
  const long long nvec = (n + VEC - 1) / VEC;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (long long)gridDim.x * blockDim.x) {
    const long long e0 = v * VEC;
    double xa[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) xa[q] = 0.0;
    const B* bp = basis + e0;
#pragma unroll 8
    for (int j = 0; j < kx; ++j) {
      B b[VEC];
      VecLoad<B, VEC>::ld(bp + (long long)j * ld, b);
      const double yj = ys[j];
#pragma unroll
      for (int q = 0; q < VEC; ++q) xa[q] = fma(yj, cvt<double>(b[q]), xa[q]);
    }
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      const long long e = e0 + q;
      if (e < n) {
        const double xe = xa[q] + (x0 ? x0[e] : 0.0);
        if (xout) xout[e] = xe;
        if (xt) {
          const double d = xe - xt[e];
          sq = fma(d, d, sq);
        }
      }
    }
  }
  if (!xt) return;
  sq = block_sum(sq, dscratch);
  if (threadIdx.x == 0) {
    xpart[blockIdx.x] = sq;
    __threadfence();
    const unsigned prev = atomicAdd(&st->counter[2], 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double s = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(&xpart[i]);
  s = block_sum(s, dscratch);
  if (threadIdx.x == 0) {
    *relerr_out = s;
    st->counter[2] = 0;
  }
}

// r0 = b - A x0 (T), b given in T
template <class T>
__global__ void sub_kernel(long long n, const T* __restrict__ b, T* __restrict__ r) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    r[e] = Rn<T>::sub(b[e], r[e]);
}

template <class To, class From>
__global__ void convert_kernel(long long n, const From* __restrict__ src, To* __restrict__ dst) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    dst[e] = cvt<To>(src[e]);
}

// --------------------------------------------------------------------------
// sampled pivoting (hessenberg.py:93-124).  The host draws the positions
// rng.choice(pop, s, replace=False) into the admissible list perm[used:]
// (the reference's swap-ordered t[k:] / g[k:]); among those entries the one
// of largest |v| (ties -> smallest index) replaces the full-scan winner the
// elimination pass left in st.  If every sampled entry is zero the full scan
// stands: that is the reference's fallback rescan (hessenberg.py:118-124),
// and it is a global scan because earlier pivot entries are exactly zero.
template <class T>
__global__ void __launch_bounds__(256)
sample_pick_kernel(const T* __restrict__ v, const long long* __restrict__ perm, long long used,
                   const long long* __restrict__ posn, int s, LoopState* __restrict__ st, int side, int iter) {
  if (iter > 0) {
    if (st->bd_iter != 0 && st->bd_iter < iter) return;
    if (side == 1 && st->bd_iter == iter) return;
  }
  __shared__ Cand scratch[32];
  Cand best{-1.0, 0.0, 0x7fffffffffffffffLL};
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    const long long idx = perm[used + posn[i]];
    const double mg = (double)absval(v[idx]);
    if (better(mg, idx, best.mag, best.idx)) best = Cand{mg, (double)v[idx], idx};
  }
  best = block_argmax(best, scratch);
  if (threadIdx.x == 0 && best.mag > 0.0) {
    st->piv_val[side] = best.val;
    st->piv_idx[side] = best.idx;
  }
}

// _swap_to_position (hessenberg.py:127-129) on the device copy of t / g and
// its inverse: the new pivot moves to position `used`.  Skipped after a
// breakdown (no pivot was taken).
__global__ void perm_swap_kernel(long long* __restrict__ perm, long long* __restrict__ where, long long used,
                                 const LoopState* __restrict__ st, int side) {
  if (st->bd_iter != 0) return;
  const long long idx = st->piv_idx[side];
  const long long pos = where[idx];
  const long long other = perm[used];
  perm[used] = idx;
  perm[pos] = other;
  where[idx] = used;
  where[other] = pos;
}

}  // namespace hs
