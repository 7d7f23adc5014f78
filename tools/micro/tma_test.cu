// Micro test of the TMA-fed GEMM engine (csrc/tma_gemm.cuh): correctness for every
// (A, B) majorness and pass count against an FP64 host reference, the tensor core's
// reading of raw fp32 operands (RZ vs RN), and clocks per 128x128x128 GEMM with two CTAs
// per SM on every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_07276_b200/csrc \
//        tma_test.cu -o tma_test
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define TG_PROF
#define TG_TRACE
#include "tma_gemm.cuh"
#include "tmap.h"

using namespace nb;

struct Maps {
  CUtensorMap a, b;
};

template <int NPASS>
__global__ void __launch_bounds__(256, 2) k_test(const Maps* maps, int amn, int bmn, int M, int N, int K, int reps,
                                                 float* C, long long* cyc, long long* prof) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024 - (tc::smem_u32(raw) & 1023)) & 1023);
  tg::Ring rg;
  tg::init(rg, sm, reinterpret_cast<tg::Ctl*>(sm + tg::kRingBytes));
  long long pl[7] = {0, 0, 0, 0, 0, 0, 0};
  rg.prof = pl;
  rg.trace = nullptr;
  // A: M x K (K-major: A[m][k]; MN-major: At[k][m]); B: K x N (K-major: Bt[n][k]; MN-major: B[k][n])
  const tg::Op a = tg::op(&maps->a, amn, 0, 0, tg::kOpBytes);
  const tg::Op b = tg::op(&maps->b, bmn, 0, 0, static_cast<uint32_t>(((N + 15) & ~15) * 64));
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    tg::gemm1<NPASS, 1>(rg, M, N, K, a, b, [&](int m, int n, auto v) {
      if constexpr (std::is_same_v<decltype(v), float4>) {
        if (blockIdx.x == 0) *reinterpret_cast<float4*>(&C[m * N + n]) = v;
      } else {
        if (blockIdx.x == 0) C[m * N + n] = v;
      }
    });
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    for (int i = 0; i < 7; ++i) prof[blockIdx.x * 7 + i] = pl[i];
  }
  tg::finish(rg);
}

__global__ void __launch_bounds__(256, 1) k_trace(const Maps* maps, int M, int N, int K, long long* tr) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024 - (tc::smem_u32(raw) & 1023)) & 1023);
  __shared__ long long t[64 * 5 + 320];
  tg::Ring rg;
  tg::init(rg, sm, reinterpret_cast<tg::Ctl*>(sm + tg::kRingBytes));
  rg.prof = nullptr;
  rg.trace = nullptr;
  const tg::Op a = tg::op(&maps->a, 0, 0, 0, tg::kOpBytes);
  const tg::Op b = tg::op(&maps->b, 0, 0, 0, 8192);
  for (int r = 0; r < 3; ++r) {
    if (r == 2) rg.trace = t;
    tg::gemm1<3, 1>(rg, M, N, K, a, b, [&](int m, int n, auto v) {});
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 5 + 320; i += blockDim.x) tr[i] = t[i];
  tg::finish(rg);
}

static float tf32_rz(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static float tf32_rn(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x1000u;  // round half away (rna)
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  const int M = 128, N = 128, K = 128;
  std::vector<float> A(M * K), B(K * N);
  srand(3);
  for (auto& x : A) x = (rand() / (float)RAND_MAX) * 2.f - 1.f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2.f - 1.f;
  // layouts: A K-major [m][k], A MN-major [k][m], B K-major [n][k], B MN-major [k][n]
  std::vector<float> Ak(M * K), Am(K * M), Bk(N * K), Bm(K * N);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) {
      Ak[m * K + k] = A[m * K + k];
      Am[k * M + m] = A[m * K + k];
    }
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) {
      Bk[n * K + k] = B[k * N + n];
      Bm[k * N + n] = B[k * N + n];
    }
  float *dAk, *dAm, *dBk, *dBm, *dC;
  cudaMalloc(&dAk, 4 * M * K);
  cudaMalloc(&dAm, 4 * M * K);
  cudaMalloc(&dBk, 4 * N * K);
  cudaMalloc(&dBm, 4 * N * K);
  cudaMalloc(&dC, 4 * M * N);
  cudaMemcpy(dAk, Ak.data(), 4 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dAm, Am.data(), 4 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dBk, Bk.data(), 4 * N * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dBm, Bm.data(), 4 * N * K, cudaMemcpyHostToDevice);
  Maps* dmaps;
  cudaMalloc(&dmaps, sizeof(Maps));
  long long* dcyc; long long* dprof; cudaMalloc(&dprof, 8 * 7 * 512);
  cudaMalloc(&dcyc, 8 * 512);
  const size_t smem = tg::kRingBytes + sizeof(tg::Ctl) + 1024;
  cudaFuncSetAttribute(k_test<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_test<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  std::vector<float> C(M * N);
  {
  for (int amn = 0; amn < 2; ++amn)
    for (int bmn = 0; bmn < 2; ++bmn)
      for (int np : {1, 3}) {
        Maps h;
        make_tmap(&h.a, amn ? dAm : dAk, amn ? K : M, amn ? M : K, amn ? M : K, amn, 128);
        make_tmap(&h.b, bmn ? dBm : dBk, bmn ? K : N, bmn ? N : K, bmn ? N : K, bmn, N);
        cudaMemcpy(dmaps, &h, sizeof h, cudaMemcpyHostToDevice);
        cudaMemset(dC, 0, 4 * M * N);
        if (np == 3) k_test<3><<<1, 256, smem>>>(dmaps, amn, bmn, M, N, K, 1, dC, dcyc, dprof);
        else k_test<1><<<1, 256, smem>>>(dmaps, amn, bmn, M, N, K, 1, dC, dcyc, dprof);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("amn=%d bmn=%d np=%d: CUDA error %s\n", amn, bmn, np, cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(C.data(), dC, 4 * M * N, cudaMemcpyDeviceToHost);
        double e64 = 0, erz = 0, ern = 0, mx = 0;
        for (int m = 0; m < M; ++m)
          for (int n = 0; n < N; ++n) {
            double r = 0, rz = 0, rn = 0;
            for (int k = 0; k < K; ++k) {
              r += (double)A[m * K + k] * B[k * N + n];
              rz += (double)tf32_rz(A[m * K + k]) * tf32_rz(B[k * N + n]);
              rn += (double)tf32_rn(A[m * K + k]) * tf32_rn(B[k * N + n]);
            }
            const double c = C[m * N + n];
            e64 = fmax(e64, fabs(c - r));
            erz = fmax(erz, fabs(c - rz));
            ern = fmax(ern, fabs(c - rn));
            mx = fmax(mx, fabs(r));
          }
        printf("amn=%d bmn=%d NPASS=%d: max|C-ref64|/max|ref| = %.3e   vs RZ-inputs %.3e   vs RN-inputs %.3e\n", amn,
               bmn, np, e64 / mx, erz / mx, ern / mx);
      }
  }
  {
    Maps h;
    make_tmap(&h.a, dAk, M, 512, 512, 0, 128);
    make_tmap(&h.b, dBk, N, 512, 512, 0, 128);
    float *dA2, *dB2; cudaMalloc(&dA2, 4 * 128 * 512); cudaMalloc(&dB2, 4 * 128 * 512);
    cudaMemset(dA2, 0, 4 * 128 * 512); cudaMemset(dB2, 0, 4 * 128 * 512);
    make_tmap(&h.a, dA2, M, 512, 512, 0, 128);
    make_tmap(&h.b, dB2, N, 512, 512, 0, 128);
    cudaMemcpy(dmaps, &h, sizeof h, cudaMemcpyHostToDevice);
    long long* dtr; cudaMalloc(&dtr, 8 * 640);
    cudaFuncSetAttribute(k_trace, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_trace<<<1, 256, smem>>>(dmaps, 128, 128, 512, dtr);
    cudaDeviceSynchronize();
    std::vector<long long> tr(640); cudaMemcpy(tr.data(), dtr, 8 * 640, cudaMemcpyDeviceToHost);
    long long t0 = tr[0];
    printf("trace (K=512, 32 chunks; clk rel. to first request): chunk: request landed ready mma_issued\n");
    for (int c = 0; c < 32; ++c) printf("  %2d: %6lld %6lld %6lld %6lld\n", c, tr[c*5]-t0, tr[c*5+1]-t0, tr[c*5+2]-t0, tr[c*5+3]-t0);
    printf("per-warp (chunks 8..15): wait-for-landing / own work\n");
    for (int w = 1; w < 8; ++w) { printf("  warp %d:", w); for (int c = 0; c < 8; ++c) printf(" %5lld/%4lld", tr[320 + (w*8+c)*2], tr[321 + (w*8+c)*2]); printf("\n"); }
    printf("trace err=%s\n", cudaGetErrorString(cudaGetLastError()));
  }
  // timing: 296 CTAs x reps GEMMs, 3 passes, A K-major, B K-major and MN-major
  for (int bmn = 0; bmn < 2; ++bmn) {
    Maps h;
    make_tmap(&h.a, dAk, M, K, K, 0, 128);
    make_tmap(&h.b, bmn ? dBm : dBk, bmn ? K : N, bmn ? N : K, bmn ? N : K, bmn, N);
    cudaMemcpy(dmaps, &h, sizeof h, cudaMemcpyHostToDevice);
    for (int grid : {1, 296}) {
      const int reps = 64;
      k_test<3><<<grid, 256, smem>>>(dmaps, 0, bmn, M, N, K, 4, dC, dcyc, dprof);
      k_test<3><<<grid, 256, smem>>>(dmaps, 0, bmn, M, N, K, reps, dC, dcyc, dprof);
      cudaDeviceSynchronize();
      std::vector<long long> cyc(grid);
      cudaMemcpy(cyc.data(), dcyc, 8 * grid, cudaMemcpyDeviceToHost);
      double s = 0;
      for (auto c : cyc) s += c;
      const double clk = s / grid / reps;
      std::vector<long long> pr(7 * grid); cudaMemcpy(pr.data(), dprof, 8 * 7 * grid, cudaMemcpyDeviceToHost);
      double ph[7] = {0}; for (int b = 0; b < grid; ++b) for (int i = 0; i < 7; ++i) ph[i] += pr[7 * b + i] / (double)grid / reps;
      printf("   phases/GEMM: - %.0f - %.0f mainloop %.0f drain %.0f tmem->smem %.0f functor %.0f fence %.0f\n", ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6]);
      const double mac = 3.0 * M * N * K;
      printf("grid=%3d bmn=%d: %7.0f clk/GEMM/CTA  tensor %.0f%% of 2048 MAC/clk/SM\n", grid, bmn, clk,
             100.0 * (grid > 148 ? 2 : 1) * mac / 2048.0 / clk);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
