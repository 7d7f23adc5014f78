// Throughput/latency of 1-D bulk copies (cp.async.bulk global->shared, mbarrier
// complete_tx) as used for the weight images: per SM, `inflight` copies of `bytes` each,
// repeated; reports cycles per copy and B/clk per SM (clock64, one CTA per SM).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void kspin(long long n) { long long t0 = clock64(); while (clock64() - t0 < n) {} }
__global__ void __launch_bounds__(128, 1) kb(const uint8_t* src, int bytes, int inflight, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* s = src + (size_t)blockIdx.x * 4 * 65536;
  uint32_t ph[8] = {0};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int j = 0; j < inflight; ++j) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[j])), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + j * bytes)), "l"(s + (size_t)(j % 4) * 65536), "r"(bytes), "r"(sa(&bar[j])) : "memory");
    }
    for (int j = 0; j < inflight; ++j) {
      asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(
                       sa(&bar[j])), "r"(ph[j] & 1) : "memory");
      ++ph[j];
    }
  }
  if (blockIdx.x == 0) *out = (clock64() - t0) / iters;
}
int main() {
  uint8_t* src;
  cudaMalloc(&src, 148 * 4 * 65536);
  cudaMemset(src, 1, 148 * 4 * 65536);
  long long* o;
  cudaMallocManaged(&o, 8);
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  kspin<<<148, 32>>>(300000000LL);
  for (int grid : {1, 148})
    for (int bytes : {4096, 16384, 32768})
      for (int inflight : {1, 2, 4}) {
        if (bytes * inflight > 128 * 1024) continue;
        kb<<<grid, 128, bytes * inflight>>>(src, bytes, inflight, 4, o);
        kb<<<grid, 128, bytes * inflight>>>(src, bytes, inflight, 200, o);
        cudaDeviceSynchronize();
        printf("grid %3d bytes %6d inflight %d: %6lld clk per round -> %.1f B/clk per SM (%s)\n", grid, bytes, inflight, *o,
               double(bytes) * inflight / *o, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
