// Shared device helpers for the B200 sketched-Hessenberg / sLSLU loop.
//
// Arithmetic that must reproduce the reference bit for bit (the operator row
// sums, the in-order elimination u <- u - c_j * basis_j, the normalisation
// u / pivot) goes through the explicit round-to-nearest intrinsics below, so
// nvcc can never contract a multiply and an add into an FMA there
// (SURVEY.md 8a, items 2-5).  Everything else (sketch sums, the fp64 projected
// solve, the iterate x = L_k y) is free to use FMA.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

namespace hs {

// Raise a kernel's dynamic shared-memory limit on the current device, once
// per (kernel, device) and thread-safely: the attribute is per device, so a
// process with contexts on several GPUs (or concurrent solves) must not share
// a single "already raised" flag.
inline cudaError_t ensure_smem(const void* kern, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> raised;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(kern, dev);
  auto it = raised.find(key);
  if (it != raised.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) raised[key] = bytes;
  return e;
}

constexpr int kWarp = 32;

// --------------------------------------------------------------------------
// element types: work type T in {double, float}; basis storage B in {T, bf16}

template <class T> struct Rn;
template <> struct Rn<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <> struct Rn<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};

template <class To, class From> __device__ __forceinline__ To cvt(From v) { return static_cast<To>(v); }
template <> __device__ __forceinline__ float cvt<float, __nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ double cvt<double, __nv_bfloat16>(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, float>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, double>(double v) { return __float2bfloat16_rn((float)v); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 v) { return v; }

template <class T> __device__ __forceinline__ T absval(T v) { return v < T(0) ? -v : v; }

// --------------------------------------------------------------------------
// pivot candidate: max |v|, ties to the smallest index (hessenberg.py:110-114).
// The comparison is a total order on (mag desc, idx asc), hence associative
// and commutative: any reduction tree gives the same winner.

struct Cand {
  double mag;   // |v| (exact: |float| and |double| are representable in double)
  double val;   // signed v
  long long idx;
};

__device__ __forceinline__ bool better(double m1, long long i1, double m2, long long i2) {
  return (m1 > m2) || (m1 == m2 && i1 < i2);
}

__device__ __forceinline__ void cand_merge(Cand& a, const Cand& b) {
  if (better(b.mag, b.idx, a.mag, a.idx)) a = b;
}

__device__ __forceinline__ Cand warp_argmax(Cand c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand d;
    d.mag = __shfl_xor_sync(0xffffffffu, c.mag, o);
    d.val = __shfl_xor_sync(0xffffffffu, c.val, o);
    d.idx = __shfl_xor_sync(0xffffffffu, c.idx, o);
    cand_merge(c, d);
  }
  return c;
}

// block-wide argmax; result valid in thread 0. scratch: >= 32 Cand in smem
__device__ __forceinline__ Cand block_argmax(Cand c, Cand* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  c = warp_argmax(c);
  __syncthreads();
  if (lane == 0) scratch[w] = c;
  __syncthreads();
  if (w == 0) {
    Cand d = lane < nw ? scratch[lane] : Cand{-1.0, 0.0, 0x7fffffffffffffffLL};
    d = warp_argmax(d);
    if (lane == 0) scratch[0] = d;
  }
  __syncthreads();
  return scratch[0];
}

// deterministic block sum (fixed tree); result in all threads. scratch >= 32 doubles
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    double d = lane < nw ? scratch[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) scratch[0] = d;
  }
  __syncthreads();
  double r = scratch[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// --------------------------------------------------------------------------
// counter-based RNG (Philox-4x32-10) for sketches that are generated, never stored

struct Philox {
  static __device__ __forceinline__ uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  static __host__ __device__ __forceinline__ uint4 gen(uint4 c, uint2 k) {
#ifdef __CUDA_ARCH__
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
#else
    for (int r = 0; r < 10; ++r) {
      const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
      uint64_t p0 = (uint64_t)M0 * c.x, p1 = (uint64_t)M1 * c.z;
      uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
      uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
      c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
#endif
  }
};

// two uniforms in (0,1] -> two standard normals (Box-Muller, fp32 intrinsics)
// Philox-4x32 with 7 rounds (the smallest round count that passes BigCrush,
// Salmon et al. 2011): the on-the-fly Gaussian sketch's generator
__device__ __forceinline__ uint4 philox7(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 7; ++r) {
    c = Philox::round(c, k);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Box-Muller with the uniforms taken from the mantissa bits (no int->float
// conversion on the XU pipe) and sqrt as t * rsqrt(t): two standard normals
__device__ __forceinline__ void box_muller_fast(uint32_t a, uint32_t b, float& n0, float& n1) {
  const float u1 = 2.0f - __uint_as_float(0x3f800000u | (a >> 9));  // (0, 1]
  const float u2 = __uint_as_float(0x3f800000u | (b >> 9)) - 1.0f;  // [0, 1)
  const float t = -2.0f * __logf(u1);                                // >= 0
  const float r = t * rsqrtf(t + 1e-30f);
  float s, c;
  __sincosf(6.283185307179586f * u2, &s, &c);
  n0 = r * c;
  n1 = r * s;
}

__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& n0, float& n1) {
  float u1 = ((float)(a >> 8) + 1.0f) * (1.0f / 16777216.0f);  // (0, 1]
  float u2 = (float)(b >> 8) * (1.0f / 16777216.0f);          // [0, 1)
  float r = sqrtf(-2.0f * __logf(u1));
  float s, c;
  __sincosf(6.283185307179586f * u2, &s, &c);
  n0 = r * c;
  n1 = r * s;
}

// Blocked sinogram layout for the A^T gathers (hs_ops.cuh):
// one 128-byte line holds ab angles x bb bins.
struct SinoBlk {
  int n_bins, ab, bb, nbb;  // nbb = bin blocks per angle block
  __host__ __device__ long long map(long long c) const {
    const long long a = c / n_bins, b = c - a * n_bins;
    return ((a / ab) * nbb + b / bb) * (ab * bb) + (a % ab) * bb + (b % bb);
  }
  // the same map in 32-bit arithmetic (64-bit division costs ~5x on the device); valid while
  // size(n_angles) < 2^31, which the int32 column indices of the operator already require
  __host__ __device__ int map32(int c) const {
    const unsigned a = (unsigned)c / (unsigned)n_bins, b = (unsigned)c - a * (unsigned)n_bins;
    return (int)(((a / ab) * nbb + b / bb) * (unsigned)(ab * bb) + (a % ab) * bb + (b % bb));
  }
  __host__ __device__ long long size(long long n_angles) const { return ((n_angles + ab - 1) / ab) * nbb * ab * bb; }
};

}  // namespace hs
