// Block-level FP32 GEMM used inside the per-centre fused kernels and the fitting net.
//
//   C(m, n) = epi(m, n, sum_k A(m, k) * B(k, n)),  0 <= m < M, 0 <= n < N
//   A(m, k) = TA ? A[k*lda + m] : A[m*lda + k]
//   B(k, n) = TB ? B[n*ldb + k] : B[k*ldb + n]
//
// 256 threads, 64x64 output tiles, 4x4 register micro-tile per thread, K staged in
// shared memory 16 at a time.  Operands live in global memory (L2-resident per-CTA
// scratch for the per-centre matrices).  Caller must __syncthreads() between dependent
// calls (the routine leaves shared memory reusable on exit).
#pragma once
#include "common.cuh"

namespace nb {

constexpr int kGemmThreads = 256;
constexpr int kTM = 64, kTN = 64, kTK = 16;

struct GemmSmem {
  float As[kTK][kTM + 4];
  float Bs[kTK][kTN + 4];
};

template <bool TA, bool TB, class Epi>
__device__ __forceinline__ void bgemm(int M, int N, int K, const float* __restrict__ A, int lda,
                                      const float* __restrict__ B, int ldb, GemmSmem& sm,
                                      Epi epi) {
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  for (int m0 = 0; m0 < M; m0 += kTM)
    for (int n0 = 0; n0 < N; n0 += kTN) {
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
      for (int k0 = 0; k0 < K; k0 += kTK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = tid + i * kGemmThreads;
          int mm, kk;
          if (TA) {
            mm = e & (kTM - 1);
            kk = e / kTM;
          } else {
            kk = e & (kTK - 1);
            mm = e / kTK;
          }
          const int gm = m0 + mm, gk = k0 + kk;
          float v = 0.f;
          if (gm < M && gk < K)
            v = TA ? A[static_cast<size_t>(gk) * lda + gm] : A[static_cast<size_t>(gm) * lda + gk];
          sm.As[kk][mm] = v;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = tid + i * kGemmThreads;
          int nn, kk;
          if (TB) {
            kk = e & (kTK - 1);
            nn = e / kTK;
          } else {
            nn = e & (kTN - 1);
            kk = e / kTN;
          }
          const int gn = n0 + nn, gk = k0 + kk;
          float v = 0.f;
          if (gn < N && gk < K)
            v = TB ? B[static_cast<size_t>(gn) * ldb + gk] : B[static_cast<size_t>(gk) * ldb + gn];
          sm.Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kTK; ++kk) {
          const float4 a = *reinterpret_cast<const float4*>(&sm.As[kk][ty * 4]);
          const float4 b = *reinterpret_cast<const float4*>(&sm.Bs[kk][tx * 4]);
          const float av[4] = {a.x, a.y, a.z, a.w};
          const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int n = n0 + tx * 4 + j;
          if (n < N) epi(m, n, acc[i][j]);
        }
      }
    }
}

}  // namespace nb
