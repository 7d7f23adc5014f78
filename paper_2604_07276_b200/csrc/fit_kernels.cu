// Fitting net (dp_core.hpp:386-391 forward, 408-414 backward) on the TMA-fed tcgen05 GEMM
// engine (tma_gemm.cuh): every 128 x 16 operand tile arrives by cp.async.bulk.tensor into a
// four-stage shared-memory ring, warps 1-7 form the 3xTF32 low parts while warp 0 issues
// the MMAs, and warps 8-11 promote each 128-wide K group of the accumulator in FP32 (the
// tensor core's own accumulation truncates).  These are plain dense GEMMs over all
// centres (M = centres, K = 4096 / 240), the place where 128-row TMA boxes do not
// over-read; the per-centre kernels keep the register-staged engine (tc_gemm.cuh), whose
// 128-row operands would over-read a ~90-row centre by 1.4x.
//
// Persistent: one CTA per SM walks the 128 x 128 output tiles row tile by row tile, so
// neighbouring CTAs share A rows in L2.  B operands are K-major: the forward reads the
// weights as stored ([out][in]), the backward their transposes ([in][out], built once per
// context).  Tensor maps are encoded per call (the buffers they point at may move).
#include <cuda.h>

#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "tma_gemm.cuh"
#include "tmap.h"

namespace nb {

enum { FEPI_STORE = 0, FEPI_TANH_BIAS = 1, FEPI_DTANH = 2 };
constexpr int kFitPromote = 8;  // chunks of 16 per FP32 promotion group = 128 of K

struct FitTmaArgs {
  CUtensorMap ma, mb;  // A [M][K], B [N][K] (K-major)
  int M, N, K;         // M: row capacity
  const int* M_live;   // live rows (NULL: M)
  float* C;            // [M][N]
  const float* bias;   // [N] (FEPI_TANH_BIAS)
  const float* Y;      // [M][N] tanh activations (FEPI_DTANH)
  int epi;
  int S;               // K slices (split-K): raw partial tiles into C's slice z, epilogue later
  unsigned long long* prof;  // (TG_PROF builds) [8] clocks: issuer phases 0-6, [7] split wait
};

template <int NPASS>
__global__ void __launch_bounds__(tg::kPromoThreads, 1) k_fit_tma(const __grid_constant__ FitTmaArgs a) {
  extern __shared__ __align__(1024) unsigned char fit_raw[];
  uint8_t* ring = fit_raw + ((1024 - (tc::smem_u32(fit_raw) & 1023)) & 1023);
  tg::Ctl* ctl = reinterpret_cast<tg::Ctl*>(ring + tg::kRingBytes);
  const int Mv = a.M_live ? min(a.M, *a.M_live) : a.M;
  const int tn = (a.N + 127) / 128, tm = (Mv + 127) / 128;
  const int items = tm * tn * a.S;  // (K slice, row tile, column tile)
  if (static_cast<int>(blockIdx.x) >= items) return;
  tg::Ring rg;
  tg::init(rg, ring, ctl, 512);
#ifdef TG_PROF
  long long pl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  rg.prof = a.prof ? pl : nullptr;
  rg.gprof = a.prof ? a.prof + 7 : nullptr;
  rg.t = clock64();
#endif
  const int Kc = a.K / a.S;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int z = w / (tm * tn), t = w - z * tm * tn;
    const int m0 = (t / tn) * 128, n0 = (t % tn) * 128;
    const int Ms = min(128, Mv - m0), Ns = min(128, a.N - n0);
    float* __restrict__ C = a.C + static_cast<size_t>(z) * a.M * a.N;
    const int N = a.N, epi = a.S > 1 ? FEPI_STORE : a.epi;
    const float* __restrict__ bias = a.bias;
    const float* __restrict__ Y = a.Y;
    tg::gemm1<NPASS, 1, kFitPromote>(rg, Ms, Ns, Kc, tg::op(&a.ma, 0, m0, z * Kc, tg::kOpBytes),
                                     tg::op(&a.mb, 0, n0, z * Kc, tg::kOpBytes), [&](int r, int c, auto v) {
                                       const size_t o = static_cast<size_t>(m0 + r) * N + n0 + c;
                                       if (epi == FEPI_TANH_BIAS) v = vtanh(v + vld(&bias[n0 + c], v));
                                       else if (epi == FEPI_DTANH) v = v * vdtanh(vld(&Y[o], v));
                                       vst(&C[o], v);
                                     });
  }
#ifdef TG_PROF
  if (a.prof && threadIdx.x == 0)
    for (int i = 0; i < 7; ++i) atomicAdd(a.prof + i, static_cast<unsigned long long>(pl[i]));
#endif
  tg::finish(rg);
}

static constexpr size_t fit_tma_smem() { return tg::kRingBytes + sizeof(tg::Ctl) + 1024; }

// C[M][N] = epi(A[M][K] B[N][K]^T) over the live rows; with K split (fit_split_k, needs the
// workspace ws of S * M * N floats) the slices go to ws and a fixed-order sum applies epi
static void fit_tma(int npass, int n_sm, int M, const int* M_live, int N, int K, const float* A, const float* B,
                    float* C, const float* bias, const float* Y, int epi, float* ws, cudaStream_t st) {
  FitTmaArgs a;
  make_tmap(&a.ma, A, M, K, K, 0, 128);
  make_tmap(&a.mb, B, N, K, K, 0, 128);
  a.M = M;
  a.M_live = M_live;
  a.N = N;
  a.K = K;
  a.C = C;
  a.bias = bias;
  a.Y = Y;
  a.epi = epi;
  a.prof = nullptr;
#ifdef TG_PROF
  static unsigned long long* prof = nullptr;
  if (!prof) {
    cudaMalloc(&prof, 8 * sizeof(unsigned long long));
  }
  cudaMemsetAsync(prof, 0, 8 * sizeof(unsigned long long), st);
  a.prof = prof;
#endif
  a.S = ws ? fit_split_k(K) : 1;
  if (a.S > 1) a.C = ws;
  const int tiles = ((M + 127) / 128) * ((N + 127) / 128) * a.S;
  const int grid = tiles < n_sm ? tiles : n_sm;
  const size_t smem = fit_tma_smem();
  if (npass == 3) {
    ensure_smem_attr(reinterpret_cast<const void*>(k_fit_tma<3>), smem);
    k_fit_tma<3><<<grid, tg::kPromoThreads, smem, st>>>(a);
  } else {
    ensure_smem_attr(reinterpret_cast<const void*>(k_fit_tma<1>), smem);
    k_fit_tma<1><<<grid, tg::kPromoThreads, smem, st>>>(a);
  }
  count_launch();
#ifdef TG_PROF
  unsigned long long h[8];
  cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  double tot = 0;
  for (int i = 0; i < 7; ++i) tot += static_cast<double>(h[i]);
  fprintf(stderr, "[fit_tma M=%d N=%d K=%d S=%d] issuer: wait-ready %.1f%% mma-issue %.1f%% loop %.1f%% drain %.1f%% tmem->smem %.1f%% functor %.1f%% sync %.1f%% | split-wait-landing/issuer-total %.2f\n",
          M, N, K, a.S, 100 * h[0] / tot, 100 * h[1] / tot, 100 * h[2] / tot, 100 * h[3] / tot, 100 * h[4] / tot,
          100 * h[5] / tot, 100 * h[6] / tot, h[7] / tot);
#endif
  if (a.S > 1) launch_fit_splitk_sum(M, M_live, N, a.S, ws, C, bias, Y, epi, st);
}

// tcgen05 modes, at least one hidden layer, every GEMM K (= fdims[0 .. n_fit-1]) a multiple
// of the 16-wide TMA K slice
bool fit_tma_supported(const FitArgs& a) {
  if (a.mode == 0 || a.n_fit < 2 || !a.fwT[0]) return false;
  for (int l = 0; l < a.n_fit; ++l)
    if (a.fdims[l] % 16) return false;
  return true;
}

void launch_fit_tma(const FitArgs& a, cudaStream_t st) {
  const int nc = a.n_centres;
  if (nc == 0) return;
  const int L = a.n_fit, np = a.mode == 1 ? 3 : 1;
  const int* ml = a.n_centres_dev;
  const float* x = a.D;
  for (int l = 0; l + 1 < L; ++l) {
    fit_tma(np, a.n_sm, nc, ml, a.fdims[l + 1], a.fdims[l], x, a.fw[l], a.Y[l], a.fb[l], nullptr, FEPI_TANH_BIAS,
            a.fdims[l + 1] <= 256 ? a.ws : nullptr, st);
    x = a.Y[l];
  }
  float* dcur = a.delta[0];
  float* dnxt = a.delta[1];
  launch_fit_out(a, dcur, st);
  // delta_{l-1} = (delta_l W_l) o (1 - Y_{l-1}^2);  dD = delta_0 W_0   (B = W_l^T, K-major)
  for (int l = L - 2; l >= 1; --l) {
    fit_tma(np, a.n_sm, nc, ml, a.fdims[l], a.fdims[l + 1], dcur, a.fwT[l], dnxt, nullptr, a.Y[l - 1], FEPI_DTANH,
            nullptr, st);
    float* t = dcur;
    dcur = dnxt;
    dnxt = t;
  }
  fit_tma(np, a.n_sm, nc, ml, a.fdims[0], a.fdims[1], dcur, a.fwT[0], a.dD, nullptr, nullptr, FEPI_STORE, nullptr, st);
}

}  // namespace nb
