// Shared device helpers for the nnmd_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

namespace nb {

constexpr int kWarp = 32;

// Max-dynamic-SMEM attribute of a kernel, raised on demand per (device, kernel): the
// attribute is per device, and the size a launch needs can grow (n_max).
inline void ensure_smem_attr(const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, func}];
  if (smem > have) {
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    have = smem;
  }
}

// Packed image shift: (sx+1)*9 + (sy+1)*3 + (sz+1), 13 == zero shift.
__host__ __device__ inline int pack_shift(int sx, int sy, int sz) {
  return (sx + 1) * 9 + (sy + 1) * 3 + (sz + 1);
}
__host__ __device__ inline int shift_x(int p) { return p / 9 - 1; }
__host__ __device__ inline int shift_y(int p) { return (p / 3) % 3 - 1; }
__host__ __device__ inline int shift_z(int p) { return p % 3 - 1; }
constexpr int kZeroShift = 13;

// ---- exact FP64 arithmetic of the reference geometry (no FMA contraction) -----------
// image_delta(rj, ri, s, L) = (rj - ri) + s*L   (vec.hpp:52-54)
__device__ __forceinline__ double image_delta(double rj, double ri, int s, double L) {
  return __dadd_rn(__dsub_rn(rj, ri), __dmul_rn(static_cast<double>(s), L));
}
// norm2 = (x*x + y*y) + z*z   (vec.hpp:28-31)
__device__ __forceinline__ double norm2_exact(double x, double y, double z) {
  return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
}

// switch_eval (dp_core.hpp:116-137), FP64
__device__ __forceinline__ void switch_fn(double r, double rcs, double rc, double& s, double& ds) {
  if (r >= rc) {
    s = 0.0;
    ds = 0.0;
    return;
  }
  const double inv = 1.0 / r;
  if (r <= rcs) {
    s = inv;
    ds = -inv * inv;
    return;
  }
  const double span = rc - rcs;
  const double u = (r - rcs) * (1.0 / span);
  const double u2 = u * u, u3 = u2 * u;
  const double w = u3 * (u * (-6.0 * u + 15.0) - 10.0) + 1.0;
  const double dw = -30.0 * u2 * (u - 1.0) * (u - 1.0) * (1.0 / span);
  s = w * inv;
  ds = dw * inv - w * inv * inv;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block reduction of a double (fixed tree), result valid in all threads.
// scratch: >= blockDim.x/32 doubles of shared memory.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += scratch[w];
  __syncthreads();
  return t;
}

// Asynchronous L2 prefetch of a global range (one thread issues it; bulk-copy engine, no
// registers held).  Used to pull a centre's forward stash out of HBM ahead of its use.
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~static_cast<uintptr_t>(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~static_cast<uintptr_t>(15);
  while (a < e) {
    const uint32_t sz = static_cast<uint32_t>((e - a) < 65536 ? (e - a) : 65536);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
    a += sz;
  }
}

// ---- scalar / float4 generic helpers for GEMM epilogue functors (called with a float
// for single elements and a float4 for 4 consecutive, 16-byte aligned columns)
__device__ __forceinline__ float vld(const float* p, float) { return *p; }
__device__ __forceinline__ float4 vld(const float* p, float4) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void vst(float* p, float v) { *p = v; }
__device__ __forceinline__ void vst(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 operator+(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 operator*(float4 a, float4 b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }
__device__ __forceinline__ float vtanh(float a) { return tanhf(a); }
__device__ __forceinline__ float4 vtanh(float4 a) { return make_float4(tanhf(a.x), tanhf(a.y), tanhf(a.z), tanhf(a.w)); }
// 1 - y*y (tanh derivative)
__device__ __forceinline__ float vdtanh(float y) { return 1.f - y * y; }
__device__ __forceinline__ float4 vdtanh(float4 y) {
  return make_float4(1.f - y.x * y.x, 1.f - y.y * y.y, 1.f - y.z * y.z, 1.f - y.w * y.w);
}

}  // namespace nb
