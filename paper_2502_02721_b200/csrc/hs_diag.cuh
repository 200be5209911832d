// Diagnostics of compute_diagnostics (solvers.py:523-532): condition numbers
// of the bases (`_union_condition`, solvers.py:228-233) and the measured
// embedding distortion of S2 (`measured_epsilon`, sketch.py:91-112).
//
// Device formulation: each basis (and the sketched-subspace matrix
// [r0, A l_1, ..., A l_k]) is orthonormalised incrementally by classical
// Gram-Schmidt with one reorthogonalisation, keeping its R factor; the
// singular values of the tall matrix are those of R (k x k), computed by a
// one-block one-sided Jacobi SVD.  For the distortion, S Q = [S r0, Z] R^{-1}
// (the sketched columns already exist), so only an l x (k+1) matrix is
// decomposed.
#pragma once

#include "hs_common.cuh"

namespace hs {

// w_e <- w_e - c_j V_je for j = 0..k-1 in order
template <class T>
__global__ void __launch_bounds__(256)
maxpy_kernel(long long n, const T* __restrict__ V, long long ld, int k, const double* __restrict__ c,
             T* __restrict__ w) {
  extern __shared__ double cs[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) cs[j] = c[j];
  __syncthreads();
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    double acc = (double)w[e];
    for (int j = 0; j < k; ++j) acc -= cs[j] * (double)V[(long long)j * ld + e];
    w[e] = (T)acc;
  }
}

// copy a T column into the fp64 work column (the orthonormalised copies are fp64)
template <class T>
__global__ void to_f64_kernel(long long n, const T* __restrict__ src, double* __restrict__ dst) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    dst[e] = cvt<double>(src[e]);
}

// R column j: r[0..j-1] (already in rcol) and rho = sqrt(|v|^2); q_j = v / rho
// (rho == 0 leaves q_j = 0: a rank-deficient column gives a zero singular value)
__global__ void qr_col_finish_kernel(int j, const double* __restrict__ vsq, double* __restrict__ rcol,
                                     double* __restrict__ rho_out) {
  if (threadIdx.x || blockIdx.x) return;
  const double rho = sqrt(*vsq);
  rcol[j] = rho;
  *rho_out = rho;
}

__global__ void scale_inv_kernel(long long n, double* __restrict__ v, const double* __restrict__ rho) {
  const double r = *rho;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    v[e] = r > 0.0 ? v[e] / r : 0.0;
}

// one-sided (Hestenes) Jacobi SVD of a rows x cols column-major matrix A (ld),
// one block of 1024 threads; A is overwritten, sv[0..cols) = singular values
// (unsorted).  Round-robin pairing, a warp per column pair.
__global__ void __launch_bounds__(1024)
jacobi_sv_kernel(int rows, int cols, double* __restrict__ A, int ld, double* __restrict__ sv, int max_sweeps) {
  __shared__ int changed;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int N = cols + (cols & 1);
  for (int sweep = 0; sweep < max_sweeps && cols > 1; ++sweep) {
    if (threadIdx.x == 0) changed = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      for (int p = warp; p < N / 2; p += nw) {
        const int a = p == 0 ? 0 : ((p - 1 + r) % (N - 1)) + 1;
        const int q = N - 1 - p;
        const int b = ((q - 1 + r) % (N - 1)) + 1;
        int i = min(a, b), j = max(a, b);
        if (j >= cols) continue;
        double* ci = A + (long long)i * ld;
        double* cj = A + (long long)j * ld;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int e = lane; e < rows; e += 32) {
          const double x = ci[e], y = cj[e];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int e = lane; e < rows; e += 32) {
          const double x = ci[e], y = cj[e];
          ci[e] = c * x - s * y;
          cj[e] = s * x + c * y;
        }
        if (lane == 0) changed = 1;
      }
      __syncthreads();
    }
    const int ch = changed;
    __syncthreads();
    if (!ch) break;
  }
  for (int j = warp; j < cols; j += nw) {
    const double* cj = A + (long long)j * ld;
    double s = 0.0;
    for (int e = lane; e < rows; e += 32) s += cj[e] * cj[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sv[j] = sqrt(s);
  }
}

__global__ void add_into_kernel(int k, double* __restrict__ a, const double* __restrict__ b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) a[i] += b[i];
}

// copy the leading kk x kk block of the upper-triangular R (ld = ldr) into a
// dense column-major kk x kk work matrix (zeros below the diagonal)
__global__ void r_block_kernel(int kk, const double* __restrict__ R, int ldr, double* __restrict__ W) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= kk * kk) return;
  const int i = idx % kk, j = idx / kk;
  W[(long long)j * kk + i] = i <= j ? R[(long long)j * ldr + i] : 0.0;
}

// M = X R^{-1} for X (rows x kk, ld = ldx) and upper-triangular R (ld = ldr):
// M[:, j] = (X[:, j] - sum_{i<j} M[:, i] R[i, j]) / R[j, j]   (one thread per row)
__global__ void trsm_right_kernel(int rows, int kk, const double* __restrict__ X, int ldx, const double* __restrict__ R,
                                  int ldr, double* __restrict__ M) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  for (int j = 0; j < kk; ++j) {
    double acc = X[(long long)j * ldx + r];
    for (int i = 0; i < j; ++i) acc -= M[(long long)i * rows + r] * R[(long long)j * ldr + i];
    const double d = R[(long long)j * ldr + j];
    M[(long long)j * rows + r] = d != 0.0 ? acc / d : 0.0;
  }
}

// kappa = max / min over the concatenated singular values (solvers.py:228-233);
// eps mode: (kappa - 1) / (kappa + 1), 1.0 when degenerate (sketch.py:109-112)
__global__ void kappa_kernel(int n1, const double* __restrict__ s1, int n2, const double* __restrict__ s2, int eps_mode,
                             double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  double mx = 0.0, mn = INFINITY;
  bool finite = true;
  for (int i = 0; i < n1; ++i) {
    mx = fmax(mx, s1[i]);
    mn = fmin(mn, s1[i]);
    finite = finite && isfinite(s1[i]);
  }
  for (int i = 0; i < n2; ++i) {
    mx = fmax(mx, s2[i]);
    mn = fmin(mn, s2[i]);
    finite = finite && isfinite(s2[i]);
  }
  if (eps_mode) {
    if (mn <= 0.0 || !finite) {
      *out = 1.0;
      return;
    }
    const double kap = mx / mn;
    *out = (kap - 1.0) / (kap + 1.0);
    return;
  }
  *out = mn < 1e-300 ? INFINITY : mx / mn;
}

}  // namespace hs
