// Microbenchmark of the per-centre block GEMMs (tc_gemm.cuh): G back-to-back GEMMs per CTA
// on L2-resident operands, production smem footprint (2 CTAs per SM), cycles from clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I paper_2604_07276_b200/csrc tools/micro/gemm_bench.cu -o /tmp/gb && /tmp/gb
// dbg bits: 1 skip operand loads, 2 skip MMA issue, 4 skip epilogue.
#include <cstdio>
#include "tc_gemm.cuh"

using namespace nb;

template <bool TS, bool TA, bool TB, int NPASS>
__global__ void __launch_bounds__(256, 2) kbench(int M, int N, int K, int G, const float* A, const float* B, float* C,
                                                  size_t slot, int dbg, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* head = raw + ((1024 - (tc::smem_u32(raw) & 1023)) & 1023);
  tc::State st;
  tc::init(st, reinterpret_cast<tc::Smem<1>*>(head), 256);
  st.dbg = dbg;
  const float* a = A + blockIdx.x * slot;
  const float* b = B + blockIdx.x * slot;
  float* c = C + blockIdx.x * slot;
  const int lda = TA ? M : K, ldb = TB ? K : N;
  const long long t0 = clock64();
  for (int g = 0; g < G; ++g) {
    auto epi = [&](int m, int n, auto v) { vst(&c[m * N + n], v); };
    if (TS) tc::gemm_ts<TA, TB, NPASS, 1>(st, M, N, K, a, lda, b, ldb, epi);
    else tc::gemm<TA, TB, NPASS, 0, 1, 1>(st, M, N, K, a, lda, b, ldb, epi);
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = clock64() - t0;
  tc::finish(st);
}

__global__ void kspin(long long n) {
  const long long t0 = clock64();
  while (clock64() - t0 < n) {
  }
}

template <bool TS, bool TA, bool TB, int NPASS>
void run(int M, int N, int K, float* A, float* B, float* C, size_t slot, int grid, int dbg = 0) {
  const size_t smem = sizeof(tc::Smem<1>) + 1024 + 8192;  // + the production kernels' extra smem
  auto k = kbench<TS, TA, TB, NPASS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  static long long* cyc = nullptr;
  if (!cyc) cudaMallocManaged(&cyc, 8);
  const int G = 64;
  kspin<<<148, 32>>>(200000000LL);
  k<<<grid, 256, smem>>>(M, N, K, 2, A, B, C, slot, dbg, cyc);
  k<<<grid, 256, smem>>>(M, N, K, G, A, B, C, slot, dbg, cyc);
  cudaDeviceSynchronize();
  const double clk = double(*cyc) / G;
  const double mac = double(M) * N * K * NPASS;
  printf("%s dbg=%d grid=%3d TA=%d TB=%d NPASS=%d M=%d N=%3d K=%3d: %6.0f clk/GEMM/CTA  tensor %.0f%% of 2048 MAC/clk "
         "per SM  err=%s\n",
         TS ? "TS" : "SS", dbg, grid, TA, TB, NPASS, M, N, K, clk, 100.0 * (grid > 148 ? 2 : 1) * mac / 2048.0 / clk,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int grid = 296;
  const size_t slot = 256 * 256;
  float *A, *B, *C;
  cudaMalloc(&A, grid * slot * 4);
  cudaMalloc(&B, grid * slot * 4);
  cudaMalloc(&C, grid * slot * 4);
  cudaMemset(A, 0, grid * slot * 4);
  cudaMemset(B, 0, grid * slot * 4);
  for (int dbg : {0, 1, 4, 5, 7, 3}) {
    run<true, false, true, 3>(128, 128, 128, A, B, C, slot, 1, dbg);
    run<false, false, true, 3>(128, 128, 128, A, B, C, slot, 1, dbg);
  }
  struct S { int M, N, K; } shapes[] = {{128, 128, 128}, {128, 96, 128}, {128, 128, 96}, {128, 128, 256}};
  for (auto s : shapes) {
    run<false, false, false, 3>(s.M, s.N, s.K, A, B, C, slot, grid);
    run<true, false, false, 3>(s.M, s.N, s.K, A, B, C, slot, grid);
    run<true, true, false, 3>(s.M, s.N, s.K, A, B, C, slot, grid);
    run<true, false, true, 3>(s.M, s.N, s.K, A, B, C, slot, grid);
    run<true, false, false, 1>(s.M, s.N, s.K, A, B, C, slot, grid);
  }
  return 0;
}
