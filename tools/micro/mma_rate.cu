// tcgen05.mma kind::tf32 issue rate per operand layout (one CTA per SM, operands already in
// shared memory / TMEM, no loads): clocks per 128xNx8 MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_07276_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <vector>

#include "tma_gemm.cuh"

using namespace nb;

// layout ids: 0 K-major SW64, 1 K-major SW128, 2 MN-major SW128_32B
__device__ __forceinline__ uint64_t mkdesc(int lay, uint32_t a) {
  if (lay == 0) return tg::desc_k(a);
  if (lay == 1) return tc::kmajor_sw128_desc(a);
  return tg::desc_mn(a);
}

__global__ void __launch_bounds__(128, 1) k_rate(int alay, int blay, int ts, int N, int reps, long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024 - (tc::smem_u32(raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tbase)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t sa = tc::smem_u32(sm), sb = sa + 16384;
    const uint32_t id = tg::idesc(N, alay == 2, blay == 2) ;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t ao = alay == 2 ? 1024u * (kk & 1) : 32u * (kk & 1);
        const uint32_t bo = blay == 2 ? 1024u * (kk & 1) : 32u * (kk & 1);
        if (ts) {
          tc::mma_tf32_ts(tm, tm + 256 + 8 * kk, mkdesc(blay, sb + bo), id, 1u);
          tc::mma_tf32_ts(tm, tm + 256 + 8 * kk, mkdesc(blay, sb + 8192 + bo), id, 1u);
          tc::mma_tf32_ts(tm, tm + 288 + 8 * kk, mkdesc(blay, sb + bo), id, 1u);
        } else {
          tc::mma_tf32(tm, mkdesc(alay, sa + ao), mkdesc(blay, sb + bo), id, 1u);
          tc::mma_tf32(tm, mkdesc(alay, sa + ao), mkdesc(blay, sb + 8192 + bo), id, 1u);
          tc::mma_tf32(tm, mkdesc(alay, sa + 8192 + ao), mkdesc(blay, sb + bo), id, 1u);
        }
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* nm[3] = {"K-SW64", "K-SW128", "MN-SW128_32B"};
  const int reps = 200;
  for (int ts = 0; ts < 2; ++ts)
    for (int al = 0; al < 3; ++al) {
      if (ts && al) continue;
      for (int bl = 0; bl < 3; ++bl)
        for (int N : {64, 128, 256}) {
          k_rate<<<148, 128, smem>>>(al, bl, ts, N, 2, d);
          k_rate<<<148, 128, smem>>>(al, bl, ts, N, reps, d);
          cudaError_t e = cudaDeviceSynchronize();
          std::vector<long long> h(148);
          cudaMemcpy(h.data(), d, 8 * 148, cudaMemcpyDeviceToHost);
          double s = 0;
          for (auto x : h) s += x;
          const double clk = s / 148 / (reps * 12.0);
          const double ideal = 128.0 * N * 8 / 2048.0;
          printf("%s A=%-13s B=%-13s N=%3d: %6.1f clk/MMA (ideal %4.0f) -> %3.0f%%  %s\n", ts ? "TS" : "SS",
                 ts ? "TMEM" : nm[al], nm[bl], N, clk, ideal, 100.0 * ideal / clk, cudaGetErrorString(e));
        }
    }
  return 0;
}
