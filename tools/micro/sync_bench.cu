// Cost of the producer->issuer->producer mbarrier hop used by the block GEMM (cycles/iter).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
template <int MODE>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  if (MODE == 0)
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(sa(b)), "r"(par) : "memory");
  else
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(sa(b)), "r"(par) : "memory");
}
template <int MODE>
__global__ void k(int iters, long long* out) {
  __shared__ uint64_t full, empty;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full)), "r"(blockDim.x / 32));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty)), "r"(1));
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 2) {
      __syncthreads();
      continue;
    }
    __syncwarp();
    if (lane == 0) arrive(&full);
    if (warp == 0) {
      wait<MODE>(&full, i & 1);
      if (lane == 0) arrive(&empty);
    }
    wait<MODE>(&empty, i & 1);
  }
  if (threadIdx.x == 0) *out = (clock64() - t0) / iters;
}
__global__ void kspin(long long n) { long long t0 = clock64(); while (clock64() - t0 < n) {} }
int main() {
  long long* o;
  cudaMallocManaged(&o, 8);
  kspin<<<148, 32>>>(400000000LL);
  for (int nt : {32, 128, 256}) {
    k<0><<<1, nt>>>(10000, o); cudaDeviceSynchronize(); printf("threads %d try_wait : %lld clk/iter\n", nt, *o);
    k<1><<<1, nt>>>(10000, o); cudaDeviceSynchronize(); printf("threads %d test_wait: %lld clk/iter\n", nt, *o);
    k<2><<<1, nt>>>(10000, o); cudaDeviceSynchronize(); printf("threads %d syncthreads: %lld clk/iter\n", nt, *o);
  }
  return 0;
}
