// Kernels of the reference's comparison solvers GMRES (Arnoldi) and LSQR
// (Golub-Kahan), solvers.py:256-403.  Unlike the Hessenberg family these take
// inner products: batched multi-dots against the stored basis, the matching
// multi-axpy, norms, and the small scalar decisions (lucky breakdown /
// exhausted bidiagonalisation) made on the device.
//
// Determinism: every dot is a fixed-partition two-stage reduction (block
// partials in fp64, summed in block order), so results do not depend on
// scheduling.
#pragma once

#include <cooperative_groups.h>

#include "hs_common.cuh"

namespace hs {

// part[b * k + j] = sum over block b's elements e of V[j*ld + e] * w[e]   (j < k)
template <class T>
__global__ void __launch_bounds__(256)
mdot_kernel(long long n, const T* __restrict__ V, long long ld, int k, const T* __restrict__ w,
            double* __restrict__ part) {
  __shared__ double scratch[32];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long e0 = (long long)blockIdx.x * per, e1 = min(n, e0 + per);
  for (int j = 0; j < k; ++j) {
    const T* v = V + (long long)j * ld;
    double acc = 0.0;
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) acc += (double)v[e] * (double)w[e];
    acc = block_sum(acc, scratch);
    if (threadIdx.x == 0) part[(long long)blockIdx.x * k + j] = acc;
  }
}

// One modified Gram-Schmidt pass (the reference's loop order, solvers.py:285-290,
// 360-361, 388-389): for j = 0..k-1 in order, c_j = <V_j, w> then
// w <- w - c_j V_j.  Cooperative kernel: each block owns a contiguous segment
// of w; a dot is block partials + one grid barrier + every block summing the
// partials in block order (double-buffered, so one barrier per column).
// coef[j] = c_j (accumulate: coef[j] += c_j).
template <class T>
__global__ void __launch_bounds__(256)
mgs_pass_kernel(long long n, const T* __restrict__ V, long long ld, int k, T* __restrict__ w, double* __restrict__ part,
                double* __restrict__ coef, int accumulate) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double scratch[32];
  __shared__ double cj;
  const int NB = gridDim.x;
  const long long per = (n + NB - 1) / NB;
  const long long e0 = (long long)blockIdx.x * per, e1 = min(n, e0 + per);
  for (int j = 0; j < k; ++j) {
    const T* v = V + (long long)j * ld;
    double acc = 0.0;
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) acc += (double)v[e] * (double)w[e];
    acc = block_sum(acc, scratch);
    double* pj = part + (j & 1) * NB;
    if (threadIdx.x == 0) pj[blockIdx.x] = acc;
    grid.sync();
    if (threadIdx.x < 32) {  // every block reduces the partials in block order
      double t = 0.0;
      if (threadIdx.x == 0)
        for (int b = 0; b < NB; ++b) t += __ldcg(pj + b);
      if (threadIdx.x == 0) cj = t;
    }
    __syncthreads();
    const double c = cj;
    if (blockIdx.x == 0 && threadIdx.x == 0) coef[j] = accumulate ? coef[j] + c : c;
    const T ct = (T)c;
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) w[e] = Rn<T>::sub(w[e], Rn<T>::mul(ct, v[e]));
    __syncthreads();
  }
}

// out[j] (+)= sum_b part[b * k + j], in block order
__global__ void mdot_finish_kernel(int nb, int k, const double* __restrict__ part, double* __restrict__ out,
                                   int accumulate) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) acc += part[(long long)b * k + j];
  out[j] = accumulate ? out[j] + acc : acc;
}

// w <- w - a * u   (LSQR: A v - alpha u, A^T u - beta v)
template <class T>
__global__ void sub_scaled_kernel(long long n, T* __restrict__ w, const T* __restrict__ u, const double* __restrict__ a) {
  const T s = (T)*a;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    w[e] = Rn<T>::sub(w[e], Rn<T>::mul(s, u[e]));
}

// out <- w / d  (true division, as numpy's w / h)
template <class T>
__global__ void div_scalar_kernel(long long n, const T* __restrict__ w, const double* __restrict__ d, T* __restrict__ out) {
  const T s = (T)*d;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    out[e] = Rn<T>::div(w[e], s);
}

// GMRES column: h[k] = sqrt(|w|^2); lucky = h[k] <= 1e-14 |h[0..k]|  (solvers.py:291-293)
__global__ void gmres_column_kernel(int k, const double* __restrict__ wsq, double* __restrict__ h, int* __restrict__ flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double hk = sqrt(*wsq);
  h[k] = hk;
  double s = 0.0;
  for (int i = 0; i <= k; ++i) s += h[i] * h[i];
  *flag = hk <= 1e-14 * sqrt(s) ? 1 : 0;
}

// LSQR scalars: out = sqrt(|v|^2); flag = out <= 1e-14 * prev  (solvers.py:364-366, 392-394)
__global__ void lsqr_scalar_kernel(const double* __restrict__ vsq, const double* __restrict__ prev, double* __restrict__ out,
                                   int* __restrict__ flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double v = sqrt(*vsq);
  *out = v;
  *flag = v <= 1e-14 * (*prev) ? 1 : 0;
}

// bidiagonal column k-1 of B ((k+1) x k): B[k-1, k-1] = alpha_{k-1}, B[k, k-1] = beta_{k-1}
__global__ void lsqr_column_kernel(int k, int ell, const double* __restrict__ alpha, const double* __restrict__ beta,
                                   double* __restrict__ zcol) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ell) return;
  zcol[i] = (i == k - 1) ? *alpha : (i == k ? *beta : 0.0);
}

// diagnostics: part[b] = sum over block b of (b_e - (Ax)_e)^2, fp64 (solvers.py:247-250)
template <class T>
__global__ void __launch_bounds__(256)
resid_part_kernel(long long m, const double* __restrict__ b, const T* __restrict__ ax, double* __restrict__ part) {
  __shared__ double scratch[32];
  const long long per = (m + gridDim.x - 1) / gridDim.x;
  const long long e0 = (long long)blockIdx.x * per, e1 = min(m, e0 + per);
  double acc = 0.0;
  for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const double r = b[e] - (double)ax[e];
    acc += r * r;
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

}  // namespace hs
