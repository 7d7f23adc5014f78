// DPA-1 network kernels: per-centre fused forward / exact backward and the batched
// fitting net.  FP32 arithmetic (FP64 geometry), one CTA per centre in a persistent
// grid; per-centre matrices live in an L2-resident per-CTA scratch slot.
//
// Reference semantics (dp_core.hpp):
//   rows / switch / env           200-223, 116-137
//   embedding (tanh every layer)  235-250
//   gated attention x n_attn      252-356   (weighted softmax 300-329, gate 280-296)
//   descriptor                    358-384
//   fitting net                   386-391
//   exact backward                396-614   (row gradients 597-611)
//
// Attention is evaluated in the re-associated form (see model.cpp fold_weights):
//   U = X [A | B]   (A = Wq Wk^T / sqrt(d_a), B = Wv Wo),  S = U_A X^T,
//   P~ = (s_j^2 pu) o Theta,  X' = X + P~ U_B
// and its exact reverse:
//   dP~ = dY U_B^T, dU_B = P~^T dY, dS = P o (dP - t), dU_A = dS X,
//   dX = dY + dS^T U_A + [dU_A | dU_B] [A | B]^T
#include <cfloat>
#include <type_traits>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "kernels.h"
#include "tc_gemm.cuh"

namespace nb {

namespace {

struct Slot {
  float *T, *DX0, *DX1, *dU;
};

__host__ __device__ inline int max_width(const DpArgs& a) {
  int w = a.M;
  for (int e = 0; e < a.n_embed; ++e) w = w > a.edims[e] ? w : a.edims[e];
  return w;
}

__host__ __device__ inline size_t emb_floats(const DpArgs& a) {
  size_t t = 0;
  for (int e = 0; e + 1 < a.n_embed; ++e) t += static_cast<size_t>(a.unit_rows) * a.edims[e];
  return t;
}

__host__ __device__ inline size_t align4(size_t x) { return (x + 3) & ~size_t(3); }

// Offsets follow the centre's own n (not n_max), so the part of a slot a centre touches
// is one compact prefix: the L2-persisting window over the slots (context.cpp) then
// holds the live scratch and nothing else.
__device__ inline Slot slot_of(const DpArgs& a, float* base, int n) {
  const size_t nm = n, M2 = 2 * a.M, W = max_width(a), nm4 = align4(nm);
  Slot s;
  size_t o = 0;
  s.T = base + o;   o += nm * nm4;
  s.DX0 = base + o; o += align4(nm * W);
  s.DX1 = base + o; o += align4(nm * W);
  s.dU = base + o;  o += align4(nm * M2);
  return s;
}

// GEMM policy: MODE 0 = SIMT FP32 (gemm_simt.cuh), 1 = 3xTF32 tcgen05, 2 = 1xTF32 tcgen05.
// NST = 1: the per-centre kernels (96 KB head -> two CTAs per SM hide each other's
// latency) run the TS-mode GEMM (A in TMEM, two B stages); NST = 2: the fitting-net tiles
// run the SS-mode GEMM with 128-row FP32 promotion.
// TSO (tensor-core modes): every per-centre GEMM routed through run() takes the TS path
// (N > 128 as several 128-column tiles); only run_wide() keeps the SS path for the one
// N = 256 product.  Used by the WIMG kernels (M = 128), so no SS code is instantiated at
// the other call sites: smaller kernels, fewer instruction-cache misses.
template <int MODE, int NST = 1, bool TSO = false>
struct Mm {
  GemmSmem* gs;
  tc::State st;
  __device__ void init(unsigned char* head, int tmem_cols = 256) {
    if constexpr (MODE == 0) gs = reinterpret_cast<GemmSmem*>(head);
    else tc::init(st, reinterpret_cast<tc::Smem<NST>*>(head), tmem_cols);
  }
  __device__ void finish() {
    if constexpr (MODE != 0) tc::finish(st);
  }
  // img: optional pre-split image of the weight operand B (DpArgs::img_*), N <= 256.
  template <bool TA, bool TB, int PROMOTE = 0, int EK = 1, bool IMG = false, class Epi>
  __device__ __forceinline__ void run(int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                                      Epi epi, const uint8_t* img = nullptr) {
    if constexpr (MODE == 0) bgemm<TA, TB>(M, N, K, A, lda, B, ldb, *gs, epi);
    else if constexpr (NST == 1 && PROMOTE == 0) {
      // N > 128 would need a second A staging per 128-column tile in TS mode: the wide
      // U = X [A|B] product stays on the SS path, which covers N = 256 in one tile
      if (TSO || N <= tc::kTsN) tc::gemm_ts<TA, TB, MODE == 1 ? 3 : 1, EK, IMG>(st, M, N, K, A, lda, B, ldb, epi, img);
      else tc::gemm<TA, TB, MODE == 1 ? 3 : 1, 0, 1, EK, IMG>(st, M, N, K, A, lda, B, ldb, epi, img);
    } else {
      tc::gemm<TA, TB, MODE == 1 ? 3 : 1, PROMOTE, NST, EK>(st, M, N, K, A, lda, B, ldb, epi);
    }
  }
  // run() with A's transposition a runtime flag (one code copy for both orientations)
  template <bool TB, class Epi>
  __device__ __forceinline__ void run_dyn(int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                                          bool ta, Epi epi) {
    if constexpr (MODE == 0) {
      if (ta) bgemm<true, TB>(M, N, K, A, lda, B, ldb, *gs, epi);
      else bgemm<false, TB>(M, N, K, A, lda, B, ldb, *gs, epi);
    } else if constexpr (NST == 1) {
      tc::gemm2_ts<false, TB, false, TB, MODE == 1 ? 3 : 1, 1, false, false, Epi, true>(
          st, M, N, K, A, lda, B, ldb, 0, A, lda, B, ldb, epi, nullptr, nullptr, ta);
    } else {
      if (ta) tc::gemm<true, TB, MODE == 1 ? 3 : 1, 0, NST, 1>(st, M, N, K, A, lda, B, ldb, epi);
      else tc::gemm<false, TB, MODE == 1 ? 3 : 1, 0, NST, 1>(st, M, N, K, A, lda, B, ldb, epi);
    }
  }
  // N = 256 in one SS tile (U = X [A|B]); falls back to run() on the SIMT path.
  template <bool TA, bool TB, bool IMG = false, class Epi>
  __device__ __forceinline__ void run_wide(int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                                           Epi epi, const uint8_t* img = nullptr) {
    if constexpr (MODE == 0) bgemm<TA, TB>(M, N, K, A, lda, B, ldb, *gs, epi);
    else if (N <= tc::kTsN) tc::gemm_ts<TA, TB, MODE == 1 ? 3 : 1, 1, IMG>(st, M, N, K, A, lda, B, ldb, epi, img);
    else tc::gemm<TA, TB, MODE == 1 ? 3 : 1, 0, 1, 1, IMG>(st, M, N, K, A, lda, B, ldb, epi, img);
  }
  // C = epi(A1 B1 + A2 B2) with one accumulator (tcgen05) or, on the SIMT path, two
  // passes through `acc` (ld N, must not alias the epilogue's sources).
  template <bool TA, bool TB, bool TA2, bool TB2, bool IMG2 = false, class Epi>
  __device__ __forceinline__ void run2(int M, int N, int K, const float* A, int lda, const float* B, int ldb, int K2,
                                       const float* A2, int lda2, const float* B2, int ldb2, float* acc, Epi epi,
                                       const uint8_t* img2 = nullptr) {
    if constexpr (MODE == 0) {
      bgemm<TA, TB>(M, N, K, A, lda, B, ldb, *gs, [&](int m, int n, float v) { acc[m * N + n] = v; });
      __syncthreads();
      bgemm<TA2, TB2>(M, N, K2, A2, lda2, B2, ldb2, *gs, [&](int m, int n, float v) { epi(m, n, acc[m * N + n] + v); });
    } else {
      if constexpr (NST == 1)
        tc::gemm2_ts<TA, TB, TA2, TB2, MODE == 1 ? 3 : 1, 1, false, IMG2>(st, M, N, K, A, lda, B, ldb, K2, A2, lda2,
                                                                          B2, ldb2, epi, nullptr, img2);
      else
        tc::gemm2<TA, TB, TA2, TB2, MODE == 1 ? 3 : 1, 0, NST, 1>(st, M, N, K, A, lda, B, ldb, K2, A2, lda2, B2, ldb2, epi);
    }
  }
};

__host__ __device__ inline size_t head_bytes(int mode, int nst = 1) {
  return mode == 0 ? sizeof(GemmSmem) : (nst == 1 ? sizeof(tc::Smem<1>) : sizeof(tc::Smem<2>));
}

// Column-pass partials inside the tcgen05 operand-stage buffer, behind the epilogue's
// 128 x 132-float staging tile (67,584 bytes) when that pass runs in the T-GEMM epilogue.
constexpr size_t kPartOff = 69632;

struct Smem {
  unsigned char* head;
  float4* R;
  float4* dR;
  float* s;
  float* dsx;
  float* t;
  float* rowpart;
  float* Ad;
  float* Bd;
  float* dAd;
  float* dBd;
  int* z;
  double* red;
  unsigned char* part;  // column-pass partials: [2][n_max] float4 + [2][n_max] float
  // multi-centre units (DpArgs::packs): the unit's centres and, per row, its centre
  int* pk_cen;          // [4] centre index
  int* pk_off;          // [5] row offsets
  float* pk_isig;       // [4] 1 / sigma
  int* pk_zi;           // [4] centre species
  float* pk_dsig;       // [4] dsigma (backward)
  int* rcen;            // [unit_rows] local centre of each row
};

__host__ __device__ inline size_t smem_layout(const DpArgs& a, int mode, unsigned char* base, Smem* out) {
  size_t o = 0;
  auto take = [&](size_t bytes) {
    o = (o + 15) & ~size_t(15);
    unsigned char* p = base ? base + o : nullptr;
    o += bytes;
    return p;
  };
  Smem s;
  const int ur = a.unit_rows;
  s.head = take(head_bytes(mode));
  s.R = reinterpret_cast<float4*>(take(sizeof(float4) * ur));
  s.dR = reinterpret_cast<float4*>(take(sizeof(float4) * ur));
  s.s = reinterpret_cast<float*>(take(sizeof(float) * ur));
  s.dsx = reinterpret_cast<float*>(take(sizeof(float) * ur));
  s.t = reinterpret_cast<float*>(take(sizeof(float) * ur));
  s.rowpart = reinterpret_cast<float*>(take(sizeof(float) * ur));
  s.Ad = reinterpret_cast<float*>(take(sizeof(float) * a.M * 4));
  s.Bd = reinterpret_cast<float*>(take(sizeof(float) * 4 * a.mr));
  s.dAd = reinterpret_cast<float*>(take(sizeof(float) * a.M * 4));
  s.dBd = reinterpret_cast<float*>(take(sizeof(float) * 4 * a.mr));
  s.z = reinterpret_cast<int*>(take(sizeof(int) * ur));
  s.red = reinterpret_cast<double*>(take(sizeof(double) * 32));
  // multi-centre units only (the single-centre kernels sit at the two-CTAs-per-SM shared
  // memory limit at n_max = 160: no bytes to spare there)
  if (a.packs) {
    s.pk_cen = reinterpret_cast<int*>(take(sizeof(int) * 4));
    s.pk_off = reinterpret_cast<int*>(take(sizeof(int) * 5));
    s.pk_isig = reinterpret_cast<float*>(take(sizeof(float) * 4));
    s.pk_zi = reinterpret_cast<int*>(take(sizeof(int) * 4));
    s.pk_dsig = reinterpret_cast<float*>(take(sizeof(float) * 4));
    s.rcen = reinterpret_cast<int*>(take(sizeof(int) * ur));
  } else {
    s.pk_cen = s.pk_off = s.pk_zi = s.rcen = nullptr;
    s.pk_isig = s.pk_dsig = nullptr;
  }
  // tcgen05 modes park the column-pass partials in the (idle) 96 KB operand stage; the
  // SIMT head (one 64x64 tile) is too small, so it gets its own region
  s.part = mode == 0 ? take(static_cast<size_t>(ur) * 2 * (sizeof(float4) + sizeof(float))) : s.head;
  if (out) *out = s;
  return o;
}

// Phase timer: thread 0 accumulates clock64 deltas per phase id when a.prof is set.
// Compiled in only for profiling builds (make PHASES=1 -> -DNB_PHASE_PROF).
#ifdef NB_PHASE_PROF
struct PhaseClock {
  unsigned long long* out;
  long long last;
  unsigned long long acc[24];
  __device__ void start(unsigned long long* o) {
    out = o;
    if (out && threadIdx.x == 0) {
      last = clock64();
      for (int i = 0; i < 24; ++i) acc[i] = 0;
    }
  }
  __device__ __forceinline__ void mark(int id) {
    if (out && threadIdx.x == 0) {
      const long long t = clock64();
      acc[id] += static_cast<unsigned long long>(t - last);
      last = t;
    }
  }
  __device__ void flush() {
    if (out && threadIdx.x == 0)
      for (int i = 0; i < 24; ++i) atomicAdd(out + i, acc[i]);
  }
};
#else
struct PhaseClock {
  __device__ __forceinline__ void start(unsigned long long*) {}
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void flush() {}
};
#endif

__device__ __forceinline__ float dot4(const float4& a, const float4& b) {
  return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}

// Dynamic centre scheduling for the persistent per-centre kernels: each CTA starts at
// blockIdx.x and then takes the next unclaimed centre (costs vary with n and n^2, so a
// static stride leaves a tail; results do not depend on the order).  `ctr` is zeroed
// before the launch.
// Thread 0 claims the following centre as soon as it starts one (CentreQueue::next), so
// the atomic's round trip overlaps the centre's work instead of sitting between centres.
struct CentreQueue {
  int* ctr;
  int claimed;  // thread 0 only
  __device__ explicit CentreQueue(int* c) : ctr(c), claimed(0) {
    if (threadIdx.x == 0) claimed = atomicAdd(ctr, 1) + static_cast<int>(gridDim.x);
  }
  __device__ int next() {
    __shared__ int s_next;
    __syncthreads();
    if (threadIdx.x == 0) s_next = claimed;
    __syncthreads();
    const int c = s_next;
    if (threadIdx.x == 0) claimed = atomicAdd(ctr, 1) + static_cast<int>(gridDim.x);
    return c;
  }
};

// Backward variant: next() is also the barrier between consecutive centres (shared memory
// is reused), one __syncthreads per centre, with the hand-over slot double-buffered so
// that thread 0 may publish the following centre while slow threads still read this one.
// (Measured: backward -0.045 ms; the forward, timed with it, got slower by code layout.)
struct CentreQueue1 {
  int* ctr;
  int claimed;  // thread 0 only
  int parity;
  __device__ explicit CentreQueue1(int* c) : ctr(c), claimed(0), parity(0) {
    if (threadIdx.x == 0) claimed = atomicAdd(ctr, 1) + static_cast<int>(gridDim.x);
  }
  __device__ int next() {
    __shared__ int s_next[2];
    if (threadIdx.x == 0) s_next[parity] = claimed;
    __syncthreads();
    const int c = s_next[parity];
    parity ^= 1;
    if (threadIdx.x == 0) claimed = atomicAdd(ctr, 1) + static_cast<int>(gridDim.x);
    return c;
  }
};

// Stage centre c's env rows (written by the centre-list build, k_neighbors) into shared
// memory; returns sigma.
__device__ double centre_rows(const DpArgs& a, int c, int n, const Smem& sm, int& zi) {
  zi = min(max(a.species[a.m_atom[a.cen_member[c]]], 0), a.ns - 1);  // bad input raises at the step's end
  const float4* Rg = a.R + static_cast<size_t>(c) * a.n_max;
  const int* Zg = a.Z + static_cast<size_t>(c) * a.n_max;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const float4 R = Rg[k];
    sm.R[k] = R;
    sm.s[k] = R.x;
    sm.z[k] = Zg[k];
  }
  __syncthreads();
  return a.sig[c];
}

// Stage multi-centre unit u (DpArgs::packs): its centres, their row offsets, 1/sigma, the
// centre species and, for every row, its env row, neighbour species and local centre.
// Returns the unit's row count (<= 128).
__device__ int unit_rows_pack(const DpArgs& a, int u, const Smem& sm) {
  if (threadIdx.x == 0) {
    const int2 pk = a.packs[u];
    int off = 0;
    for (int i = 0; i < 4; ++i) {
      const bool v = i < pk.y;
      const int c = pk.x + i;
      sm.pk_cen[i] = v ? c : -1;
      sm.pk_off[i] = off;
      const double sg = v ? a.sig[c] : 0.0;
      sm.pk_isig[i] = sg > 0.0 ? static_cast<float>(1.0 / sg) : 0.f;
      sm.pk_zi[i] = v ? min(max(a.species[a.m_atom[a.cen_member[c]]], 0), a.ns - 1) : 0;
      off += v ? a.nn[c] : 0;
    }
    sm.pk_off[4] = off;
  }
  __syncthreads();
  for (int i = 0; i < 4 && sm.pk_cen[i] >= 0; ++i) {
    const int c = sm.pk_cen[i], o = sm.pk_off[i], n = sm.pk_off[i + 1] - o;
    const float4* Rg = a.R + static_cast<size_t>(c) * a.n_max;
    const int* Zg = a.Z + static_cast<size_t>(c) * a.n_max;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const float4 R = Rg[k];
      sm.R[o + k] = R;
      sm.s[o + k] = R.x;
      sm.z[o + k] = Zg[k];
      sm.rcen[o + k] = i;
    }
  }
  __syncthreads();
  return sm.pk_off[4];
}

// Embedding net over the n rows: layer 0 folded (s*w0 + ctab[zj][zi]), then tanh layers.
// Writes intermediate activations to EMB and the last to `out` (n x M).
template <int MODE, bool WIMG, bool PACK = false, class MmT>
__device__ void embed_forward(MmT& mm, const DpArgs& a, int n, int zi, const Smem& sm, float* emb,
                              float* out) {
  const int E0 = a.edims[0];
  float* cur = (a.n_embed == 1) ? out : emb;
  if (static_cast<int>(blockDim.x) % E0 == 0) {
    // one fixed output o per thread for all its rows: w0[o] read once, no index division
    const int o = threadIdx.x % E0, rstep = blockDim.x / E0;
    const float w = a.w0[o];
    for (int k = static_cast<int>(threadIdx.x) / E0; k < n; k += rstep) {
      const int zc = PACK ? sm.pk_zi[sm.rcen[k]] : zi;  // the row's centre species
      const float v = fmaf(sm.s[k], w, a.ctab[(static_cast<size_t>(sm.z[k]) * a.ns + zc) * E0 + o]);
      cur[k * E0 + o] = tanhf(v);
    }
  } else
  for (int idx = threadIdx.x; idx < n * E0; idx += blockDim.x) {
    const int k = idx / E0, o = idx - k * E0;
    const int zc = PACK ? sm.pk_zi[sm.rcen[k]] : zi;  // the row's centre species
    const float v = fmaf(sm.s[k], a.w0[o], a.ctab[(static_cast<size_t>(sm.z[k]) * a.ns + zc) * E0 + o]);
    cur[idx] = tanhf(v);
  }
  __syncthreads();
  size_t off = static_cast<size_t>(a.unit_rows) * E0;
  for (int e = 1; e < a.n_embed; ++e) {
    const int Ein = a.edims[e - 1], Eout = a.edims[e];
    float* nxt = (e + 1 == a.n_embed) ? out : emb + off;
    const float* b = a.eb[e];
    mm.template run<false, true, 0, 1, WIMG>(n, Eout, Ein, cur, Ein, a.ew[e], Ein,
                                             [&](int m, int o, auto v) { vst(&nxt[m * Eout + o], vtanh(v + vld(&b[o], v))); },
                                             a.img_ew[e]);
    __syncthreads();
    cur = nxt;
    off += static_cast<size_t>(a.unit_rows) * Eout;
  }
}

// Register-cached rows (n <= 32 C): each lane keeps its C key columns' s_j^2 and R_j for
// all of its warp's rows.
// PACK: rows of a multi-centre unit only see their own centre's columns (block-diagonal
// S); pu and P~ are written as zero outside the block so the PV product stays exact.
template <int C, bool PACK = false>
__device__ void softmax_gate_rc(int n, int ln, const float* S, int lds, float* PU, float* PT, float inv_sig,
                                const Smem& sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float s2[C];
  float4 Rj[C];
#pragma unroll
  for (int t = 0; t < C; ++t) {
    const int j = lane + 32 * t;
    s2[t] = j < n ? sm.s[j] * sm.s[j] : 0.f;
    Rj[t] = j < n ? sm.R[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if constexpr (C == 8 && !PACK) {
    // n > 128 (scores in global memory): rows in pairs, both rows' score loads in flight
    // and their max / sum butterflies interleaved; per-lane order kept
    for (int k0 = wid; k0 < n; k0 += 2 * nw) {
      const bool hv1 = k0 + nw < n;
      const int kr[2] = {k0, hv1 ? k0 + nw : k0};
      float e[2][C], mx[2] = {-FLT_MAX, -FLT_MAX}, den[2] = {0.f, 0.f};
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < C; ++t) {
          const int j = lane + 32 * t;
          e[h][t] = j < n ? S[static_cast<size_t>(kr[h]) * lds + j] : -FLT_MAX;
        }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < C; ++t) mx[h] = fmaxf(mx[h], e[h][t]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx[0] = fmaxf(mx[0], __shfl_xor_sync(0xffffffffu, mx[0], o));
        mx[1] = fmaxf(mx[1], __shfl_xor_sync(0xffffffffu, mx[1], o));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < C; ++t) {
          const int j = lane + 32 * t;
          e[h][t] = j < n ? __expf(e[h][t] - mx[h]) : 0.f;
          den[h] += s2[t] * e[h][t];
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        den[0] += __shfl_xor_sync(0xffffffffu, den[0], o);
        den[1] += __shfl_xor_sync(0xffffffffu, den[1], o);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !hv1) break;
        const int k = kr[h];
        const float inv = den[h] > 0.f ? 1.0f / den[h] : 0.f;
        const float4 Rk = sm.R[k];
#pragma unroll
        for (int t = 0; t < C; ++t) {
          const int j = lane + 32 * t;
          if (j < n) {
            const float pu = e[h][t] * inv;
            if (PU) PU[static_cast<size_t>(k) * ln + j] = pu;
            PT[static_cast<size_t>(k) * ln + j] = s2[t] * pu * (dot4(Rk, Rj[t]) * inv_sig);
          }
        }
      }
    }
    return;
  }
  for (int k = wid; k < n; k += nw) {
    // the row's scores, all loads issued before the reductions
    float cur[C];
#pragma unroll
    for (int t = 0; t < C; ++t) {
      const int j = lane + 32 * t;
      cur[t] = j < n ? S[static_cast<size_t>(k) * lds + j] : 0.f;
    }
    int jb = 0, je = n;
    if constexpr (PACK) {
      const int i = sm.rcen[k];
      jb = sm.pk_off[i];
      je = sm.pk_off[i + 1];
      inv_sig = sm.pk_isig[i];
    }
    float e[C];
    float mx = -FLT_MAX;
#pragma unroll
    for (int t = 0; t < C; ++t) {
      const int j = lane + 32 * t;
      e[t] = (j >= jb && j < je) ? cur[t] : -FLT_MAX;
      mx = fmaxf(mx, e[t]);
    }
    mx = warp_max(mx);
    float den = 0.f;
#pragma unroll
    for (int t = 0; t < C; ++t) {
      const int j = lane + 32 * t;
      e[t] = (j >= jb && j < je) ? __expf(e[t] - mx) : 0.f;
      den += s2[t] * e[t];
    }
    den = warp_sum(den);
    const float inv = den > 0.f ? 1.0f / den : 0.f;
    const float4 Rk = sm.R[k];
#pragma unroll
    for (int t = 0; t < C; ++t) {
      const int j = lane + 32 * t;
      if (j < n) {
        const float pu = e[t] * inv;
        if (PU) PU[static_cast<size_t>(k) * ln + j] = pu;
        PT[static_cast<size_t>(k) * ln + j] = s2[t] * pu * (dot4(Rk, Rj[t]) * inv_sig);
      }
    }
  }
}

// Weighted softmax + gate for every row: PU = pu (optional), PT = s_j^2 pu Theta.
__device__ void softmax_gate(int n, int ln, const float* S, int lds, float* PU, float* PT, float inv_sig,
                             const Smem& sm) {
  if (n <= 128) {
    softmax_gate_rc<4>(n, ln, S, lds, PU, PT, inv_sig, sm);
    return;
  }
  if (n <= 256) {
    softmax_gate_rc<8>(n, ln, S, lds, PU, PT, inv_sig, sm);
    return;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = wid; k < n; k += nw) {
    const float* row = S + static_cast<size_t>(k) * lds;
    float mx = -FLT_MAX;
    for (int j = lane; j < n; j += 32) mx = fmaxf(mx, row[j]);
    mx = warp_max(mx);
    float den = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float sj = sm.s[j];
      den += sj * sj * expf(row[j] - mx);
    }
    den = warp_sum(den);
    const float inv = den > 0.f ? 1.0f / den : 0.f;
    const float4 Rk = sm.R[k];
    for (int j = lane; j < n; j += 32) {
      const float sj = sm.s[j];
      const float pu = expf(row[j] - mx) * inv;
      const float th = dot4(Rk, sm.R[j]) * inv_sig;
      if (PU) PU[static_cast<size_t>(k) * ln + j] = pu;
      PT[static_cast<size_t>(k) * ln + j] = sj * sj * pu * th;
    }
  }
}

// Backward of one gated attention layer's n x n part, from dP~ = dY U_B^T (TS, ld ldt:
// the T-GEMM's shared-memory accumulator tile, or a global copy) and the stashed softmax
// weights pu (PU, ld ln).  With C = R R^T, Theta = C / sigma, P = s_j^2 pu:
//   dP = dP~ Theta,  dC = dP~ P / sigma,  t_k = sum_j dP P
// Row pass (warp per query row k, float4 over j): t_k, the dsigma partial
// -sum_j dC C / sigma, and the row half of the gate term dR_k += sum_j dC_kj R_j.
__device__ void bwd_row_pass(int n, int ln, const float* TS, int ldt, const float* __restrict__ PU, float inv_sig,
                             const Smem& sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // rows in pairs (k, k + nw): both rows' tile and pu loads in flight together, their
  // reductions interleaved, the gate's four sums in 6 shuffles (lanes 0, 8, 16, 24 end with
  // x, y, z, w); every per-lane accumulation keeps the column order
  for (int k0 = wid; k0 < n; k0 += 2 * nw) {
    const bool hv1 = k0 + nw < n;
    const int kr[2] = {k0, hv1 ? k0 + nw : k0};
    const float4 Rk[2] = {sm.R[kr[0]], sm.R[kr[1]]};
    float t[2] = {0.f, 0.f}, dsg[2] = {0.f, 0.f};
    float g[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    for (int j4 = 4 * lane; j4 < n; j4 += 128) {
      float4 tv[2], pu[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        tv[h] = *reinterpret_cast<const float4*>(TS + static_cast<size_t>(kr[h]) * ldt + j4);
        pu[h] = *reinterpret_cast<const float4*>(PU + static_cast<size_t>(kr[h]) * ln + j4);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float tq[4] = {tv[h].x, tv[h].y, tv[h].z, tv[h].w};
        const float pq[4] = {pu[h].x, pu[h].y, pu[h].z, pu[h].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j4 + q;
          if (j < n) {
            const float sj = sm.s[j];
            const float4 Rj = sm.R[j];
            const float C = dot4(Rk[h], Rj);
            const float pv = sj * sj * pq[q];
            const float dP = tq[q] * C * inv_sig;
            const float dC = tq[q] * pv * inv_sig;
            dsg[h] -= dC * C * inv_sig;
            t[h] += dP * pv;
            g[h][0] += dC * Rj.x;
            g[h][1] += dC * Rj.y;
            g[h][2] += dC * Rj.z;
            g[h][3] += dC * Rj.w;
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t[0] += __shfl_xor_sync(0xffffffffu, t[0], o);
      t[1] += __shfl_xor_sync(0xffffffffu, t[1], o);
      dsg[0] += __shfl_xor_sync(0xffffffffu, dsg[0], o);
      dsg[1] += __shfl_xor_sync(0xffffffffu, dsg[1], o);
    }
    const bool hi16 = lane & 16, hi8 = lane & 8;
    float b[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float a0 = hi16 ? g[h][2] : g[h][0], a1 = hi16 ? g[h][3] : g[h][1];
      a0 += __shfl_xor_sync(0xffffffffu, hi16 ? g[h][0] : g[h][2], 16);
      a1 += __shfl_xor_sync(0xffffffffu, hi16 ? g[h][1] : g[h][3], 16);
      b[h] = hi8 ? a1 : a0;
      b[h] += __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      b[0] += __shfl_xor_sync(0xffffffffu, b[0], o);
      b[1] += __shfl_xor_sync(0xffffffffu, b[1], o);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !hv1) break;
      if (lane == 0) {
        sm.t[kr[h]] = t[h];
        sm.rowpart[kr[h]] = dsg[h];
      }
      if ((lane & 7) == 0) reinterpret_cast<float*>(&sm.dR[kr[h]])[lane >> 3] += b[h];
    }
  }

}

// Column pass (thread per key column j and k-half, coalesced across threads), after the
// row pass: dP and dC recomputed from dP~, dw_j of the s_j^2 softmax weights, the column
// half of the gate term dR_j += sum_k dC_kj R_k, dsx_j += 2 s_j (dw_j + dsigma), and
// dS = P o (dP - t) written to DS (ld ln; may alias TS when ldt == ln).
// part: [2][stride] float4 + [2][stride] float of shared memory (stride >= n).
__device__ void bwd_col_pass(int n, int ln, int stride, const float* TS, int ldt, const float* __restrict__ PU,
                             float* DS, float inv_sig, const Smem& sm, unsigned char* part_raw) {
  const int nh = (n + 1) >> 1;
  const int half_threads = blockDim.x >> 1;
  float4* part = reinterpret_cast<float4*>(part_raw);   // [2][stride] (g0..g3)
  float* partw = reinterpret_cast<float*>(part + 2 * stride);  // [2][stride]
  const int h = threadIdx.x / half_threads;
  for (int j = threadIdx.x - h * half_threads; j < n; j += half_threads) {
    float dw = 0.f, g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
    const float sj = sm.s[j];
    const float sj2 = sj * sj;
    const float4 Rj = sm.R[j];
    const int kb = h * nh, ke = min(n, kb + nh);
#pragma unroll 4
    for (int k = kb; k < ke; ++k) {
      const float pu = PU[static_cast<size_t>(k) * ln + j];
      const float tv = TS[static_cast<size_t>(k) * ldt + j];
      const float4 Rk = sm.R[k];
      const float C = dot4(Rk, Rj);
      const float dP = tv * C * inv_sig;
      const float dC = tv * (sj2 * pu) * inv_sig;
      const float dpt = dP - sm.t[k];
      dw += pu * dpt;
      DS[static_cast<size_t>(k) * ln + j] = sj2 * pu * dpt;
      g0 += dC * Rk.x;
      g1 += dC * Rk.y;
      g2 += dC * Rk.z;
      g3 += dC * Rk.w;
    }
    part[h * stride + j] = make_float4(g0, g1, g2, g3);
    partw[h * stride + j] = dw;
  }
  if (threadIdx.x == blockDim.x - 1) {
    float ds = 0.f;
    for (int k = 0; k < n; ++k) ds += sm.rowpart[k];
    sm.red[0] = ds;
  }
  __syncthreads();
  const float dsig = static_cast<float>(sm.red[0]);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float4 p0 = part[j], p1 = part[stride + j];
    const float dw = partw[j] + partw[stride + j];
    sm.dsx[j] += 2.f * sm.s[j] * (dw + dsig);
    float4 r = sm.dR[j];
    r.x += p0.x + p1.x;
    r.y += p0.y + p1.y;
    r.z += p0.z + p1.z;
    r.w += p0.w + p1.w;
    sm.dR[j] = r;
  }
  tc::fence_proxy_async();  // part may sit in an operand stage that bulk copies overwrite later
}

// Column pass for any n, after bwd_row_pass (t_k, the dsigma row partials, the row gate
// term): columns in windows of 128, warp per query row k, lane owning 4 columns of the
// window (coalesced 16-byte loads of dP~ and pu, 16-byte dS stores), the column sums dw_j
// and sum_k dC_kj R_k kept in registers across the warp's rows and reduced over warps
// once per window.  Same quantities as bwd_col_pass; DS may alias TS (ldt == ln).
// part: [nw][128] float4 + [nw][128] float of shared memory.
__device__ void bwd_colwin_pass(int n, int ln, const float* TS, int ldt, const float* __restrict__ PU, float* DS,
                                float inv_sig, const Smem& sm, unsigned char* part_raw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float4* pg = reinterpret_cast<float4*>(part_raw);     // [nw][128]
  float* pw = reinterpret_cast<float*>(pg + nw * 128);  // [nw][128]
  if (threadIdx.x == blockDim.x - 1) {
    float ds = 0.f;
    for (int k = 0; k < n; ++k) ds += sm.rowpart[k];
    sm.red[0] = ds;
  }
  for (int c0 = 0; c0 < n; c0 += 128) {
    const int j4 = c0 + 4 * lane;
    const bool act = j4 < n;
    float sj2[4];
    float4 Rj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool v = j4 + q < n;
      const float sj = v ? sm.s[j4 + q] : 0.f;
      sj2[q] = sj * sj;
      Rj[q] = v ? sm.R[j4 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float cw[4] = {0.f, 0.f, 0.f, 0.f};
    float4 cg[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) cg[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) {
      // rows in pairs: both rows' loads before either row's store (DS aliases TS, so the
      // compiler cannot move a later row's loads above an earlier row's store itself)
      for (int k0 = wid; k0 < n; k0 += 2 * nw) {
        const bool hv1 = k0 + nw < n;
        const int kr[2] = {k0, hv1 ? k0 + nw : k0};
        float4 tv2[2], pu2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tv2[h] = *reinterpret_cast<const float4*>(TS + static_cast<size_t>(kr[h]) * ldt + j4);
          pu2[h] = *reinterpret_cast<const float4*>(PU + static_cast<size_t>(kr[h]) * ln + j4);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !hv1) break;
          const int k = kr[h];
          const float4 Rk = sm.R[k];
          const float tk = sm.t[k];
          const float tq[4] = {tv2[h].x, tv2[h].y, tv2[h].z, tv2[h].w};
          const float pq[4] = {pu2[h].x, pu2[h].y, pu2[h].z, pu2[h].w};
          float ds[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool v = j4 + q < n;  // the tile and stash hold junk past column n
            const float tt = v ? tq[q] : 0.f, pp = v ? pq[q] : 0.f;
            const float C = dot4(Rk, Rj[q]);
            const float dP = tt * C * inv_sig;
            const float dC = tt * (sj2[q] * pp) * inv_sig;
            const float dpt = dP - tk;
            cw[q] += pp * dpt;
            ds[q] = sj2[q] * pp * dpt;
            cg[q].x += dC * Rk.x;
            cg[q].y += dC * Rk.y;
            cg[q].z += dC * Rk.z;
            cg[q].w += dC * Rk.w;
          }
          *reinterpret_cast<float4*>(DS + static_cast<size_t>(k) * ln + j4) = make_float4(ds[0], ds[1], ds[2], ds[3]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pg[wid * 128 + 4 * lane + q] = cg[q];
        pw[wid * 128 + 4 * lane + q] = cw[q];
      }
    }
    __syncthreads();
    const float dsig = static_cast<float>(sm.red[0]);
    for (int j = c0 + threadIdx.x; j < min(n, c0 + 128); j += blockDim.x) {
      float dw = 0.f;
      float4 r = sm.dR[j];
      for (int w = 0; w < nw; ++w) {
        const float4 p = pg[w * 128 + j - c0];
        r.x += p.x;
        r.y += p.y;
        r.z += p.z;
        r.w += p.w;
        dw += pw[w * 128 + j - c0];
      }
      sm.dsx[j] += 2.f * sm.s[j] * (dw + dsig);
      sm.dR[j] = r;
    }
    __syncthreads();
  }
  tc::fence_proxy_async();  // part sits in an operand stage that bulk copies overwrite later
}

// Row and column passes in one sweep over dP~ (n <= 128, blockDim <= 256): warp per query
// row k, lane owning columns 4 lane .. 4 lane + 3 for the whole sweep.  Each warp keeps its
// column sums (dw_j and the column gate sum_k dC_kj R_k) in registers across its rows and
// parks them in part ([nw][128] float4 + [nw][128] float); dsigma is summed per lane and
// reduced once.  After t_k is reduced the row's dS is written from the same registers, so
// dP~ and pu are read once.  Same results as bwd_row_pass + bwd_col_pass up to summation
// order.
// PACK: multi-centre unit -- each row only pairs with its own centre's columns (the
// tile and the stash hold other centres' junk off the diagonal blocks, masked here, so dS
// is zero there), 1/sigma per centre, and dsigma summed per centre.
template <bool PACK = false>
__device__ void bwd_rc_pass(int n, int ln, const float* TS, int ldt, const float* __restrict__ PU, float* DS,
                            float inv_sig, const Smem& sm, unsigned char* part_raw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float4* pg = reinterpret_cast<float4*>(part_raw);       // [nw][128]
  float* pw = reinterpret_cast<float*>(pg + nw * 128);    // [nw][128]
  const int j4 = 4 * lane;
  const bool act = j4 < n;
  float sj2[4];
  float4 Rj[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool v = j4 + q < n;
    const float sj = v ? sm.s[j4 + q] : 0.f;
    sj2[q] = sj * sj;
    Rj[q] = v ? sm.R[j4 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float cw[4] = {0.f, 0.f, 0.f, 0.f};
  float4 cg[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) cg[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  float dsg = 0.f;
  // rows in pairs (k, k + nw): both rows' tile and pu loads in flight together and their
  // shuffle reductions interleaved; every per-lane accumulation keeps the row order
  for (int k0 = wid; k0 < n; k0 += 2 * nw) {
    const int kr[2] = {k0, k0 + nw};
    const bool hv[2] = {true, k0 + nw < n};
    float4 tv[2], pu[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      tv[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      pu[h] = tv[h];
      if (act && hv[h]) {
        tv[h] = *reinterpret_cast<const float4*>(TS + static_cast<size_t>(kr[h]) * ldt + j4);
        pu[h] = *reinterpret_cast<const float4*>(PU + static_cast<size_t>(kr[h]) * ln + j4);
      }
    }
    float pq[2][4], dP[2][4], t[2], gg[2][4], isg[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = hv[h] ? kr[h] : k0;
      const float4 Rk = sm.R[k];
      int jb = 0, je = n;
      isg[h] = inv_sig;
      if constexpr (PACK) {
        const int i = sm.rcen[k];
        jb = sm.pk_off[i];
        je = sm.pk_off[i + 1];
        isg[h] = sm.pk_isig[i];
      }
      const float tq[4] = {tv[h].x, tv[h].y, tv[h].z, tv[h].w};
      pq[h][0] = pu[h].x;
      pq[h][1] = pu[h].y;
      pq[h][2] = pu[h].z;
      pq[h][3] = pu[h].w;
      float tt0 = 0.f, g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, dsr = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool v = hv[h] && j4 + q >= jb && j4 + q < je;
        const float tt = v ? tq[q] : 0.f;  // the tile and stash hold junk past column n
        pq[h][q] = v ? pq[h][q] : 0.f;
        const float C = dot4(Rk, Rj[q]);
        const float pv = sj2[q] * pq[h][q];
        dP[h][q] = tt * C * isg[h];
        const float dC = tt * pv * isg[h];
        if constexpr (PACK) dsr -= dC * C * isg[h];
        else dsg -= dC * C * isg[h];
        tt0 += dP[h][q] * pv;
        g0 += dC * Rj[q].x;
        g1 += dC * Rj[q].y;
        g2 += dC * Rj[q].z;
        g3 += dC * Rj[q].w;
        cg[q].x += dC * Rk.x;
        cg[q].y += dC * Rk.y;
        cg[q].z += dC * Rk.z;
        cg[q].w += dC * Rk.w;
      }
      if constexpr (PACK) {
        dsr = warp_sum(dsr);
        if (lane == 0 && hv[h]) sm.rowpart[kr[h]] = dsr;
      }
      t[h] = tt0;
      gg[h][0] = g0;
      gg[h][1] = g1;
      gg[h][2] = g2;
      gg[h][3] = g3;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t[0] += __shfl_xor_sync(0xffffffffu, t[0], o);
      t[1] += __shfl_xor_sync(0xffffffffu, t[1], o);
    }
    {
      const bool hi16 = lane & 16, hi8 = lane & 8;
      float b[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float a0 = hi16 ? gg[h][2] : gg[h][0], a1 = hi16 ? gg[h][3] : gg[h][1];
        a0 += __shfl_xor_sync(0xffffffffu, hi16 ? gg[h][0] : gg[h][2], 16);
        a1 += __shfl_xor_sync(0xffffffffu, hi16 ? gg[h][1] : gg[h][3], 16);
        b[h] = hi8 ? a1 : a0;
        b[h] += __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        b[0] += __shfl_xor_sync(0xffffffffu, b[0], o);
        b[1] += __shfl_xor_sync(0xffffffffu, b[1], o);
      }
      if ((lane & 7) == 0) {
        reinterpret_cast<float*>(&sm.dR[kr[0]])[lane >> 3] += b[0];
        if (hv[1]) reinterpret_cast<float*>(&sm.dR[kr[1]])[lane >> 3] += b[1];
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float ds[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float dpt = dP[h][q] - t[h];
        cw[q] += pq[h][q] * dpt;
        ds[q] = sj2[q] * pq[h][q] * dpt;
      }
      if (act && hv[h])
        *reinterpret_cast<float4*>(DS + static_cast<size_t>(kr[h]) * ln + j4) = make_float4(ds[0], ds[1], ds[2], ds[3]);
    }
  }
  if constexpr (!PACK) {
    dsg = warp_sum(dsg);
    if (lane == 0) sm.red[8 + wid] = dsg;
  }
  if (act) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      pg[wid * 128 + j4 + q] = cg[q];
      pw[wid * 128 + j4 + q] = cw[q];
    }
  }
  __syncthreads();
  float dsig = 0.f;
  if constexpr (PACK) {
    // dsigma of each centre: its rows' sums in row order
    if (threadIdx.x < 4 && sm.pk_cen[threadIdx.x] >= 0) {
      float t = 0.f;
      for (int k = sm.pk_off[threadIdx.x]; k < sm.pk_off[threadIdx.x + 1]; ++k) t += sm.rowpart[k];
      sm.pk_dsig[threadIdx.x] = t;
    }
    __syncthreads();
  } else {
    for (int w = 0; w < nw; ++w) dsig += static_cast<float>(sm.red[8 + w]);
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    if constexpr (PACK) dsig = sm.pk_dsig[sm.rcen[j]];
    float dw = 0.f;
    float4 r = sm.dR[j];
    for (int w = 0; w < nw; ++w) {
      const float4 p = pg[w * 128 + j];
      r.x += p.x;
      r.y += p.y;
      r.z += p.z;
      r.w += p.w;
      dw += pw[w * 128 + j];
    }
    sm.dsx[j] += 2.f * sm.s[j] * (dw + dsig);
    sm.dR[j] = r;
  }
  tc::fence_proxy_async();  // part sits in an operand stage that bulk copies overwrite later
}

}  // namespace

size_t dp_scratch_floats(const DpArgs& a) {
  const size_t nm = a.unit_rows, M2 = 2 * a.M, W = max_width(a);
  return align4(nm * M2) + nm * align4(nm) + align4(nm * W) * 2 + 64;
}

size_t dp_smem_bytes(const DpArgs& a, int mode) { return smem_layout(a, mode, nullptr, nullptr) + 1024; }

// Descriptor of one centre from its rows [r0, r1) of the final features Xf (dp_core.hpp:
// 358-384).  A = X^T R: thread per (feature m, k-half), all four R components at once,
// coalesced over m; the two k-halves are added in a fixed order.  B = R^T X_< is the same
// sums (B[q][r] = A[r][q] before scaling, product for product), so it is copied.  Writes
// D[c], Ad[c], Bd[c]; ends with a barrier.
__device__ void descriptor(const DpArgs& a, const float* Xf, int r0, int r1, int c, const Smem& sm) {
  const int M = a.M, mr = a.mr;
  {
    float4* part = reinterpret_cast<float4*>(sm.head);  // [2][M]; operand stages idle
    const int n = r1 - r0;
    const int nh = (n + 1) >> 1;
    const int half_threads = blockDim.x >> 1;
    const int h = threadIdx.x / half_threads;
    const int kb = r0 + h * nh, ke = min(r1, kb + nh);
    for (int m = threadIdx.x - h * half_threads; m < M; m += half_threads) {
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 16
      for (int k = kb; k < ke; ++k) {
        const float x = Xf[k * M + m];
        const float4 R = sm.R[k];
        a0 += x * R.x;
        a1 += x * R.y;
        a2 += x * R.z;
        a3 += x * R.w;
      }
      part[h * M + m] = make_float4(a0, a1, a2, a3);
    }
    tc::fence_proxy_async();  // operand-stage memory: later overwritten by bulk copies
    __syncthreads();
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
      const float4 p0 = part[m], p1 = part[M + m];
      const float4 A = make_float4((p0.x + p1.x) * a.inv_sqrt_nmax, (p0.y + p1.y) * a.inv_sqrt_nmax,
                                   (p0.z + p1.z) * a.inv_sqrt_nmax, (p0.w + p1.w) * a.inv_sqrt_nmax);
      reinterpret_cast<float4*>(sm.Ad)[m] = A;
      if (m < mr) {
        sm.Bd[0 * mr + m] = A.x;
        sm.Bd[1 * mr + m] = A.y;
        sm.Bd[2 * mr + m] = A.z;
        sm.Bd[3 * mr + m] = A.w;
      }
    }
    __syncthreads();
  }
  float* D = a.D + static_cast<size_t>(c) * M * mr;
  // four consecutive q per thread when mr % 4 == 0 (16-byte rows): same products in the
  // same order as the scalar loop below
  for (int idx = 4 * threadIdx.x; (mr & 3) == 0 && idx < M * mr; idx += 4 * blockDim.x) {
    const int m = idx / mr, q0 = idx - m * mr;
    const float4 am = reinterpret_cast<const float4*>(sm.Ad)[m];
    const float ac[4] = {am.x, am.y, am.z, am.w};
    float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const float4 b = *reinterpret_cast<const float4*>(&sm.Bd[cc * mr + q0]);
      o[0] += ac[cc] * b.x;
      o[1] += ac[cc] * b.y;
      o[2] += ac[cc] * b.z;
      o[3] += ac[cc] * b.w;
    }
    *reinterpret_cast<float4*>(&D[idx]) = make_float4(o[0], o[1], o[2], o[3]);
  }
  for (int idx = threadIdx.x; (mr & 3) != 0 && idx < M * mr; idx += blockDim.x) {
    const int m = idx / mr, q = idx - m * mr;
    float acc = 0.f;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) acc += sm.Ad[m * 4 + cc] * sm.Bd[cc * mr + q];
    D[idx] = acc;
  }
  for (int idx = threadIdx.x; idx < M * 4; idx += blockDim.x) a.Ad[static_cast<size_t>(c) * M * 4 + idx] = sm.Ad[idx];
  for (int idx = threadIdx.x; idx < 4 * mr; idx += blockDim.x) a.Bd[static_cast<size_t>(c) * 4 * mr + idx] = sm.Bd[idx];
  __syncthreads();
}

// Row gradient g_k = de/dd_k of row k of centre c (dp_core.hpp:597-611) in FP64 geometry
// from the env-row gradient dR_k and the switch-value gradient dsx_k; written to g[c][k].
// w receives the row's virial products -g_a d_b.
__device__ __forceinline__ void row_gradient(const DpArgs& a, int c, int k, float4 dr, float dsx, double (&w)[9]) {
  const int cm = a.cen_member[c];
  const int ca = a.m_atom[cm];
  const int cs = a.m_shift[cm];
  const int mj = a.nlist[static_cast<size_t>(c) * a.n_max + k];
  const int aj = a.m_atom[mj];
  const int sj = a.m_shift[mj];
  const int rel[3] = {shift_x(sj) - shift_x(cs), shift_y(sj) - shift_y(cs), shift_z(sj) - shift_z(cs)};
  double d[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) d[q] = image_delta(a.pos[3 * aj + q], a.pos[3 * ca + q], rel[q], a.L[q]);
  const double r = sqrt(norm2_exact(d[0], d[1], d[2]));
  double s, ds;
  switch_fn(r, a.rcs, a.rc, s, ds);
  const double ir = 1.0 / r, sr = s * ir;
  const double e[3] = {d[0] * ir, d[1] * ir, d[2] * ir};
  const double dr0 = dr.x, dr1 = dr.y, dr2 = dr.z, dr3 = dr.w;
  const double ge = dr1 * e[0] + dr2 * e[1] + dr3 * e[2];
  const double coef = (dr0 + static_cast<double>(dsx)) * ds + (ds - sr) * ge;
  const double gk[3] = {coef * e[0] + sr * dr1, coef * e[1] + sr * dr2, coef * e[2] + sr * dr3};
  double* g = a.g + (static_cast<size_t>(c) * a.n_max + k) * 3;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    g[q] = gk[q];
#pragma unroll
    for (int b = 0; b < 3; ++b) w[3 * q + b] = -gk[q] * d[b];
  }
}

// ------------------------------------------------------------------------------------
// Forward: rows -> embedding -> attention layers -> descriptor D = (X^T R)(R^T X_<) / n_max
// ------------------------------------------------------------------------------------
template <int MODE, bool WIMG, bool PACK = false>
__global__ void __launch_bounds__(256, 2) k_centre_forward(const __grid_constant__ DpArgs a) {
  extern __shared__ __align__(1024) unsigned char dp_smem_raw[];
  unsigned char* dp_smem = dp_smem_raw + ((1024 - (tc::smem_u32(dp_smem_raw) & 1023)) & 1023);
  Smem sm;
  smem_layout(a, MODE, dp_smem, &sm);
  Mm<MODE, 1, WIMG> mm;
  mm.init(sm.head);
  PhaseClock pc;
  pc.start(a.prof);
#ifdef NB_PHASE_PROF
  if constexpr (MODE != 0) {
    if (a.prof && threadIdx.x == 0) {
      mm.st.prof = pc.acc + 16;
      mm.st.t_last = clock64();
    }
  }
#endif
  const int M = a.M, M2 = 2 * M, mr = a.mr;
  const int ur = a.unit_rows, ur4 = (ur + 3) & ~3;
  const int n_units = PACK ? *a.n_units_dev : (a.n_centres_dev ? *a.n_centres_dev : a.n_centres);
  CentreQueue queue(a.work);
  // unit u: one centre (u = c), or a multi-centre pack (DpArgs::packs)
  for (int u = blockIdx.x; u < n_units; u = queue.next()) {
    int n, zi = 0;
    float inv_sig = 0.f;
    if constexpr (PACK) {
      n = unit_rows_pack(a, u, sm);
    } else {
      n = a.nn[u];
      const double sig = centre_rows(a, u, n, sm, zi);
      inv_sig = sig > 0.0 ? static_cast<float>(1.0 / sig) : 0.f;
    }
    const int ln = (n + 3) & ~3;  // leading dimension of the n x n scratch matrices
    pc.mark(0);
    float* X = a.X + static_cast<size_t>(u) * ur * M;
    embed_forward<MODE, WIMG, PACK>(mm, a, n, zi, sm, a.EMBst + static_cast<size_t>(u) * a.emb_centre_stride, X);
    pc.mark(1);
    for (int l = 0; l < a.n_attn; ++l) {
      const float* Xl = X + l * a.x_layer_stride;
      float* Xn = X + (l + 1) * a.x_layer_stride;
      float* Ul = a.Ust + l * a.u_layer_stride + static_cast<size_t>(u) * ur * M2;
      float* PUl = a.PUst + l * a.p_layer_stride + static_cast<size_t>(u) * ur * ur4;
      float* PTl = a.PTst + l * a.p_layer_stride + static_cast<size_t>(u) * ur * ur4;
      mm.template run_wide<false, false, WIMG>(n, M2, M, Xl, M, a.ab[l], M2,
                                                [&](int k, int j, auto v) { vst(&Ul[k * M2 + j], v); }, a.img_ab[l]);
      __syncthreads();
      pc.mark(2);
      bool fused_softmax = false;
      if constexpr (MODE != 0) {
        if (n <= 128) {
          // S tile stays in shared memory: weighted softmax + gate fused into the epilogue
          mm.template run<false, true, 0, 2>(n, n, M, Ul, M2, Xl, M,
                                             [&](const float* stg, int ldst, int, int, int, int) {
                                               if constexpr (PACK) softmax_gate_rc<4, true>(n, ln, stg, ldst, PUl, PTl, inv_sig, sm);
                                               else softmax_gate(n, ln, stg, ldst, PUl, PTl, inv_sig, sm);
                                             });
          pc.mark(3);
          fused_softmax = true;
        }
      }
      if (!fused_softmax) {
        mm.template run<false, true>(n, n, M, Ul, M2, Xl, M,
                                     [&](int k, int j, auto v) { vst(&PUl[k * ln + j], v); });
        __syncthreads();
        pc.mark(3);
        softmax_gate(n, ln, PUl, ln, PUl, PTl, inv_sig, sm);
      }
      __syncthreads();
      pc.mark(4);
      {
        float* __restrict__ xo = Xn;
        const float* __restrict__ xi = Xl;
        mm.template run<false, false>(n, M, n, PTl, ln, Ul + M, M2,
                                      [=](int k, int m, auto v) { vst(&xo[k * M + m], vld(&xi[k * M + m], v) + v); });
      }
      __syncthreads();
      pc.mark(5);
    }
    // descriptor (dp_core.hpp:358-384), per centre of the unit over its rows
    const float* Xf = X + a.n_attn * a.x_layer_stride;
    const int n_cen = PACK ? 4 : 1;
    for (int i = 0; i < n_cen; ++i) {
      int c = u, r0 = 0, r1 = n;
      if constexpr (PACK) {
        c = sm.pk_cen[i];
        if (c < 0) break;
        r0 = sm.pk_off[i];
        r1 = sm.pk_off[i + 1];
      }
      descriptor(a, Xf, r0, r1, c, sm);
    }
    pc.mark(6);
  }
  pc.flush();
  mm.finish();
}

// ------------------------------------------------------------------------------------
// Backward: dD -> (dA, dB) -> dX, dR -> attention layers in reverse -> embedding ->
// row gradients g_k = de/dd_k (FP64 geometry), per-centre virial -sum g (x) d.
// ------------------------------------------------------------------------------------
template <int MODE, bool WIMG, bool PACK = false>
__global__ void __launch_bounds__(256, 2) k_centre_backward(const __grid_constant__ DpArgs a) {
  extern __shared__ __align__(1024) unsigned char dp_smem_raw[];
  unsigned char* dp_smem = dp_smem_raw + ((1024 - (tc::smem_u32(dp_smem_raw) & 1023)) & 1023);
  Smem sm;
  smem_layout(a, MODE, dp_smem, &sm);
  Mm<MODE, 1, WIMG> mm;
  mm.init(sm.head);
  PhaseClock pc;
  pc.start(a.prof);
#ifdef NB_PHASE_PROF
  if constexpr (MODE != 0) {
    if (a.prof && threadIdx.x == 0) {
      mm.st.prof = pc.acc + 16;
      mm.st.t_last = clock64();
    }
  }
#endif
  const int M = a.M, M2 = 2 * M, mr = a.mr;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ur = a.unit_rows, ur4 = (ur + 3) & ~3;
  const int n_units = PACK ? *a.n_units_dev : (a.n_centres_dev ? *a.n_centres_dev : a.n_centres);
  CentreQueue1 queue(a.work);
  // unit u: one centre (u = c), or a multi-centre pack (DpArgs::packs)
  for (int u = blockIdx.x; u < n_units; u = queue.next()) {
    int n, zi = 0;
    float inv_sig = 0.f;
    if constexpr (PACK) {
      n = unit_rows_pack(a, u, sm);
    } else {
      n = a.nn[u];
      const double sig = centre_rows(a, u, n, sm, zi);
      inv_sig = sig > 0.0 ? static_cast<float>(1.0 / sig) : 0.f;
    }
    (void)zi;
    const int ln = (n + 3) & ~3;  // leading dimension of the n x n scratch matrices
    const Slot sl = slot_of(a, a.scratch + static_cast<size_t>(blockIdx.x) * a.scratch_slot, n);
    pc.mark(0);
    const float* X = a.X + static_cast<size_t>(u) * ur * M;
    const float* Xf = X + a.n_attn * a.x_layer_stride;
    if (threadIdx.x == 0 && !(a.flags & 1)) {
      // forward stash read first: final features (dR below) and the top layer's U
      prefetch_l2(Xf, sizeof(float) * n * M);
      if (a.n_attn > 0)
        prefetch_l2(a.Ust + (a.n_attn - 1) * a.u_layer_stride + static_cast<size_t>(u) * ur * M2,
                    sizeof(float) * n * M2);
    }
    for (int k = threadIdx.x; k < n; k += blockDim.x) sm.dsx[k] = 0.f;
    float* dY = sl.DX0;
    float* dXn = sl.DX1;
    const float inm = a.inv_sqrt_nmax;
    const int n_cen = PACK ? 4 : 1;
    for (int i = 0; i < n_cen; ++i) {
      int c = u, r0 = 0, r1 = n;
      if constexpr (PACK) {
        c = sm.pk_cen[i];
        if (c < 0) break;
        r0 = sm.pk_off[i];
        r1 = sm.pk_off[i + 1];
      }
      const float* dD = a.dD + static_cast<size_t>(c) * M * mr;
      const float* Ad = a.Ad + static_cast<size_t>(c) * M * 4;
      const float* Bd = a.Bd + static_cast<size_t>(c) * 4 * mr;
      // dA[m][cc] = sum_q dD[m,q] B[cc,q];  dB[cc][q] = sum_m dD[m,q] A[m,cc]
      // (operands staged into shared memory with coalesced loads; the tensor-core stage
      // buffers are idle between GEMMs)
      {
        const float* sdD = dD;
        const float* sAd = Ad;
        const float* sBd = Bd;
        if constexpr (MODE != 0) {
          float* tmp = reinterpret_cast<float*>(sm.head);
          if (((M * mr) & 3) == 0) {
            for (int i2 = threadIdx.x; i2 < (M * mr) >> 2; i2 += blockDim.x)
              reinterpret_cast<float4*>(tmp)[i2] = reinterpret_cast<const float4*>(dD)[i2];
          } else {
            for (int i2 = threadIdx.x; i2 < M * mr; i2 += blockDim.x) tmp[i2] = dD[i2];
          }
          for (int i2 = threadIdx.x; i2 < M * 4; i2 += blockDim.x) tmp[M * mr + i2] = Ad[i2];
          for (int i2 = threadIdx.x; i2 < 4 * mr; i2 += blockDim.x) tmp[M * mr + M * 4 + i2] = Bd[i2];
          tc::fence_proxy_async();  // operand-stage memory: later overwritten by bulk copies
          __syncthreads();
          sdD = tmp;
          sAd = tmp + M * mr;
          sBd = tmp + M * mr + M * 4;
        }
        for (int idx = threadIdx.x; idx < M * 4 + 4 * mr; idx += blockDim.x) {
          float acc = 0.f;
          if (idx < M * 4) {
            const int m = idx >> 2, cc = idx & 3;
            for (int q = 0; q < mr; ++q) acc += sdD[m * mr + q] * sBd[cc * mr + q];
            sm.dAd[idx] = acc;
          } else {
            const int j = idx - M * 4, cc = j / mr, q = j - cc * mr;
            for (int m = 0; m < M; ++m) acc += sdD[m * mr + q] * sAd[m * 4 + cc];
            sm.dBd[j] = acc;
          }
        }
        __syncthreads();
      }
      if (static_cast<int>(blockDim.x) % M == 0) {
        // a thread keeps one feature m for all its rows: dA[m], dB[:, m] read once, no
        // index division; per element the same operations in the same order
        const int m = threadIdx.x % M, rstep = blockDim.x / M;
        const float4 da = reinterpret_cast<const float4*>(sm.dAd)[m];
        const bool hb = m < mr;
        float db[4] = {0.f, 0.f, 0.f, 0.f};
        if (hb)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) db[cc] = sm.dBd[cc * mr + m];
        for (int k = r0 + static_cast<int>(threadIdx.x) / M; k < r1; k += rstep) {
          const float4 Rk = sm.R[k];
          float v = da.x * Rk.x;
          v += da.y * Rk.y;
          v += da.z * Rk.z;
          v += da.w * Rk.w;
          if (hb) {
            v += db[0] * Rk.x;
            v += db[1] * Rk.y;
            v += db[2] * Rk.z;
            v += db[3] * Rk.w;
          }
          dY[k * M + m] = v * inm;
        }
      } else
      for (int idx = r0 * M + threadIdx.x; idx < r1 * M; idx += blockDim.x) {
        const int k = idx / M, m = idx - k * M;
        const float* R = reinterpret_cast<const float*>(&sm.R[k]);
        const float4 da = reinterpret_cast<const float4*>(sm.dAd)[m];  // one conflict-free 16-byte read
        float v = da.x * R[0];
        v += da.y * R[1];
        v += da.z * R[2];
        v += da.w * R[3];
        if (m < mr)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) v += sm.dBd[cc * mr + m] * R[cc];
        dY[idx] = v * inm;
      }
      // dR_k = (X_k dA + X_k[:mr] dB^T) / sqrt(n_max): warp per row pair (both rows' loads
      // in flight together), lanes over features; a row's four sums in 6 shuffles (halve
      // the values per step, then a butterfly: lanes 0, 8, 16, 24 end with x, y, z, w)
#ifndef NB_DR_ONE_ROW
      for (int k0 = r0 + wid; k0 < r1; k0 += 2 * nw) {
        const int k1 = k0 + nw;
        const bool has1 = k1 < r1;
        float v[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll 4
        for (int m = lane; m < M; m += 32) {
          const float x0 = Xf[k0 * M + m];
          const float x1 = has1 ? Xf[k1 * M + m] : 0.f;
          const float4 da = reinterpret_cast<const float4*>(sm.dAd)[m];
          const float xs[2] = {x0, x1};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            v[h][0] += xs[h] * da.x;
            v[h][1] += xs[h] * da.y;
            v[h][2] += xs[h] * da.z;
            v[h][3] += xs[h] * da.w;
          }
          if (m < mr) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              v[h][0] += xs[h] * sm.dBd[0 * mr + m];
              v[h][1] += xs[h] * sm.dBd[1 * mr + m];
              v[h][2] += xs[h] * sm.dBd[2 * mr + m];
              v[h][3] += xs[h] * sm.dBd[3 * mr + m];
            }
          }
        }
        const bool hi16 = lane & 16, hi8 = lane & 8;
        float b[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float a0 = hi16 ? v[h][2] : v[h][0], a1 = hi16 ? v[h][3] : v[h][1];
          a0 += __shfl_xor_sync(0xffffffffu, hi16 ? v[h][0] : v[h][2], 16);
          a1 += __shfl_xor_sync(0xffffffffu, hi16 ? v[h][1] : v[h][3], 16);
          b[h] = hi8 ? a1 : a0;
          b[h] += __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          b[0] += __shfl_xor_sync(0xffffffffu, b[0], o);
          b[1] += __shfl_xor_sync(0xffffffffu, b[1], o);
        }
        if ((lane & 7) == 0) {
          reinterpret_cast<float*>(&sm.dR[k0])[lane >> 3] = b[0] * inm;
          if (has1) reinterpret_cast<float*>(&sm.dR[k1])[lane >> 3] = b[1] * inm;
        }
      }
#else
      for (int k = r0 + wid; k < r1; k += nw) {
        float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
#pragma unroll 4
        for (int m = lane; m < M; m += 32) {
          const float x = Xf[k * M + m];
          const float4 da = reinterpret_cast<const float4*>(sm.dAd)[m];
          v0 += x * da.x;
          v1 += x * da.y;
          v2 += x * da.z;
          v3 += x * da.w;
          if (m < mr) {
            v0 += x * sm.dBd[0 * mr + m];
            v1 += x * sm.dBd[1 * mr + m];
            v2 += x * sm.dBd[2 * mr + m];
            v3 += x * sm.dBd[3 * mr + m];
          }
        }
        v0 = warp_sum(v0);
        v1 = warp_sum(v1);
        v2 = warp_sum(v2);
        v3 = warp_sum(v3);
        if (lane == 0) sm.dR[k] = make_float4(v0 * inm, v1 * inm, v2 * inm, v3 * inm);
      }
#endif
      if constexpr (PACK) __syncthreads();  // dAd / dBd are reused by the unit's next centre
    }
    __syncthreads();
    pc.mark(1);
    for (int l = a.n_attn - 1; l >= 0; --l) {
      const float* Xl = X + l * a.x_layer_stride;
      const float* AB = a.ab[l];
      // forward stash: U = X [A|B], pu, P~ of this layer (no recompute)
      const float* Ul = a.Ust + l * a.u_layer_stride + static_cast<size_t>(u) * ur * M2;
      const float* PUl = a.PUst + l * a.p_layer_stride + static_cast<size_t>(u) * ur * ur4;
      const float* PTl = a.PTst + l * a.p_layer_stride + static_cast<size_t>(u) * ur * ur4;
      if (threadIdx.x == 0 && !(a.flags & 1)) {
        // this layer's stash and the next (lower) layer's U are read from HBM below:
        // start pulling them into L2 now
        prefetch_l2(PUl, sizeof(float) * n * ln);
        prefetch_l2(PTl, sizeof(float) * n * ln);
        prefetch_l2(Xl, sizeof(float) * n * M);
        if (l > 0) prefetch_l2(Ul - a.u_layer_stride, sizeof(float) * n * M2);
        else prefetch_l2(a.EMBst + static_cast<size_t>(u) * a.emb_centre_stride, sizeof(float) * a.emb_centre_stride);
      }
      pc.mark(2);
      // T = dP~ = dY U_B^T, then the row and column passes (bwd_row_pass, bwd_col_pass)
      // -> dS in sl.T.  With tcgen05 and n <= 128 both passes run as one sweep
      // (bwd_rc_pass) in the GEMM epilogue on the shared-memory accumulator tile (dP~ never
      // goes to global memory); the per-warp column partials sit behind that tile in the
      // same (idle) operand-stage buffer.
      bool fused_rc = false;
      if constexpr (MODE != 0) {
        if (PACK || (n <= 128 && !(a.flags & 2))) {
          unsigned char* part = sm.head + kPartOff;
          mm.template run<false, true, 0, 2>(n, n, M, dY, M, Ul + M, M2,
                                             [&](const float* stg, int ldst, int, int, int, int) {
                                               bwd_rc_pass<PACK>(n, ln, stg, ldst, PUl, sl.T, inv_sig, sm, part);
                                             });
          fused_rc = true;
        }
      }
      if (!PACK && !fused_rc) {
        mm.template run<false, true>(n, n, M, dY, M, Ul + M, M2,
                                     [&](int k, int j, auto v) { vst(&sl.T[k * ln + j], v); });
        __syncthreads();
        pc.mark(5);
        bwd_row_pass(n, ln, sl.T, ln, PUl, inv_sig, sm);
        __syncthreads();
        if constexpr (MODE != 0) bwd_colwin_pass(n, ln, sl.T, ln, PUl, sl.T, inv_sig, sm, sm.part);
        else bwd_col_pass(n, ln, n, sl.T, ln, PUl, sl.T, inv_sig, sm, sm.part);
      }
      __syncthreads();
      pc.mark(7);
      // dU_A = dS X ; dU_B = P~^T dY  (one GEMM call site run twice: half the code)
#ifdef NB_BWD_TWO_SITES
      mm.template run<false, false>(n, M, n, sl.T, ln, Xl, M,
                          [&](int k, int m, auto v) { vst(&sl.dU[k * M2 + m], v); });
      mm.template run<true, false>(n, M, n, PTl, ln, dY, M,
                         [&](int k, int m, auto v) { vst(&sl.dU[k * M2 + M + m], v); });
#else
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        float* __restrict__ du = sl.dU + (h ? M : 0);
        mm.template run_dyn<false>(n, M, n, h ? PTl : sl.T, ln, h ? dY : Xl, M, h != 0,
                                   [=](int k, int m, auto v) { vst(&du[k * M2 + m], v); });
      }
#endif
      __syncthreads();
      pc.mark(9);
      // dX = dY + dS^T U_A + [dU_A | dU_B] [A | B]^T  (both products in one accumulator)
      {
        float* __restrict__ xo = dXn;
        const float* __restrict__ yi = dY;
#ifndef NB_BWD_TWO_SITES
        // one call site for every layer: the bottom layer's embedding-output tanh
        // derivative (dp_core.hpp:580-583), dX0 (1 - X0^2), behind a uniform branch
        const float* __restrict__ x0 = l == 0 ? X : nullptr;
        mm.template run2<true, false, false, true, WIMG>(n, M, n, sl.T, ln, Ul, M2, M2, sl.dU, M2, AB, M2, dXn,
                                                   [=](int k, int m, auto v) {
                                                     auto y = vld(&yi[k * M + m], v) + v;
                                                     if (x0) y = y * vdtanh(vld(&x0[k * M + m], v));
                                                     vst(&xo[k * M + m], y);
                                                   },
                                                   a.img_abT[l]);
#else
        if (l > 0) {
          mm.template run2<true, false, false, true, WIMG>(n, M, n, sl.T, ln, Ul, M2, M2, sl.dU, M2, AB, M2, dXn,
                                                     [=](int k, int m, auto v) { vst(&xo[k * M + m], vld(&yi[k * M + m], v) + v); },
                                                     a.img_abT[l]);
        } else {
          // bottom layer: the embedding's output tanh derivative (dp_core.hpp:580-583) is
          // applied in the same epilogue, dX0 (1 - X0^2)
          const float* __restrict__ x0 = X;
          mm.template run2<true, false, false, true, WIMG>(n, M, n, sl.T, ln, Ul, M2, M2, sl.dU, M2, AB, M2, dXn,
                                                     [=](int k, int m, auto v) {
                                                       vst(&xo[k * M + m], (vld(&yi[k * M + m], v) + v) * vdtanh(vld(&x0[k * M + m], v)));
                                                     },
                                                     a.img_abT[l]);
        }
#endif
      }
      __syncthreads();
      pc.mark(11);
      float* tmp = dY;
      dY = dXn;
      dXn = tmp;
    }
    // embedding backward (dp_core.hpp:580-596) from the stored hidden activations; with
    // attention layers the output tanh derivative was applied in the last dX epilogue
    if (a.n_attn == 0) {
      const float* X0 = X;
      for (int idx = threadIdx.x; idx < n * M; idx += blockDim.x) {
        const float y = X0[idx];
        dY[idx] *= 1.f - y * y;
      }
      __syncthreads();
    }
    {
      // offsets of the stored activations
      size_t offs[kMaxLayers];
      size_t off = 0;
      for (int e = 0; e + 1 < a.n_embed; ++e) {
        offs[e] = off;
        off += static_cast<size_t>(ur) * a.edims[e];
      }
      for (int e = a.n_embed - 1; e >= 1; --e) {
        const int Ein = a.edims[e - 1], Eout = a.edims[e];
        const float* __restrict__ h = a.EMBst + static_cast<size_t>(u) * a.emb_centre_stride + offs[e - 1];
        float* __restrict__ xo = dXn;
        mm.template run<false, false, 0, 1, WIMG>(n, Ein, Eout, dY, Eout, a.ew[e], Ein,
                                                  [=](int k, int i, auto v) {
                                                    vst(&xo[k * Ein + i], v * vdtanh(vld(&h[k * Ein + i], v)));
                                                  },
                                                  a.img_ewT[e]);
        __syncthreads();
        float* tmp = dY;
        dY = dXn;
        dXn = tmp;
      }
      // ds_k += sum_o dU0_ko w0_o: warp per row, lanes over o (coalesced), 4 rows per
      // warp with their loads issued together
      const int E0 = a.edims[0];
      for (int k0 = wid; k0 < n; k0 += 4 * nw) {
        float du[4] = {0.f, 0.f, 0.f, 0.f};
        for (int o = lane; o < E0; o += 32) {
          const float w = a.w0[o];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = k0 + u * nw;
            if (k < n) du[u] += dY[k * E0 + o] * w;
          }
        }
        {
          // the four row sums in 6 shuffles: lanes 0, 8, 16, 24 end with rows u = 0..3
          const bool hi16 = lane & 16, hi8 = lane & 8;
          float a0 = hi16 ? du[2] : du[0], a1 = hi16 ? du[3] : du[1];
          a0 += __shfl_xor_sync(0xffffffffu, hi16 ? du[0] : du[2], 16);
          a1 += __shfl_xor_sync(0xffffffffu, hi16 ? du[1] : du[3], 16);
          float b = hi8 ? a1 : a0;
          b += __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
          b += __shfl_xor_sync(0xffffffffu, b, 4);
          b += __shfl_xor_sync(0xffffffffu, b, 2);
          b += __shfl_xor_sync(0xffffffffu, b, 1);
          const int k = k0 + (lane >> 3) * nw;
          if ((lane & 7) == 0 && k < n) sm.dsx[k] += b;
        }
      }
      __syncthreads();
    }
    pc.mark(12);
    // row gradients (dp_core.hpp:597-611) in FP64 geometry; virial W_ab -= g_a d_b
    if constexpr (PACK) {
      // rows of several centres (one row per thread, n <= 128): each row's nine products in
      // shared memory (the operand stage is idle), then per centre a fixed-order row sum
      double* wrow = reinterpret_cast<double*>(sm.head);  // [n][9]
      const int k = threadIdx.x;
      if (k < n) {
        const int i = sm.rcen[k];
        const int c = sm.pk_cen[i], kk = k - sm.pk_off[i];
        double w[9];
        row_gradient(a, c, kk, sm.dR[k], sm.dsx[k], w);
#pragma unroll
        for (int q = 0; q < 9; ++q) wrow[9 * k + q] = w[q];
      }
      __syncthreads();
      if (threadIdx.x < 36) {
        const int i = threadIdx.x / 9, q = threadIdx.x - 9 * i;
        const int c = sm.pk_cen[i];
        if (c >= 0) {
          double t = 0.0;  // row order: deterministic
          for (int r = sm.pk_off[i]; r < sm.pk_off[i + 1]; ++r) t += wrow[9 * r + q];
          a.vir[static_cast<size_t>(c) * 9 + q] = t;
        }
      }
      tc::fence_proxy_async();  // operand stage: later overwritten by bulk copies
    } else {
      const int c = u;
      double w[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int k = threadIdx.x; k < n; k += blockDim.x) {
        double wk[9];
        row_gradient(a, c, k, sm.dR[k], sm.dsx[k], wk);
#pragma unroll
        for (int q = 0; q < 9; ++q) w[q] += wk[q];
      }
      // the nine sums with one barrier: warp sums, then a fixed-order sum over warps
      // (block_sum's order, so the same bits), parked in dA's (dead) shared buffer
      if (static_cast<size_t>(M) * 4 * sizeof(float) >= 9 * nw * sizeof(double)) {
        double* vr = reinterpret_cast<double*>(sm.dAd);
#pragma unroll
        for (int q = 0; q < 9; ++q) w[q] = warp_sum(w[q]);
        if (lane == 0)
#pragma unroll
          for (int q = 0; q < 9; ++q) vr[wid * 9 + q] = w[q];
        __syncthreads();
        if (threadIdx.x < 9) {
          double t = 0.0;
          for (int v = 0; v < nw; ++v) t += vr[v * 9 + threadIdx.x];
          a.vir[static_cast<size_t>(c) * 9 + threadIdx.x] = t;
        }
      } else {
        for (int q = 0; q < 9; ++q) {
          const double t = block_sum(w[q], sm.red + 8);
          if (threadIdx.x == 0) a.vir[static_cast<size_t>(c) * 9 + q] = t;
        }
      }
    }
    pc.mark(13);  // (the centre queue's barrier ends the centre)
  }
  pc.flush();
  mm.finish();
}

// Pre-split weight image of a GEMM's B operand (tc::bulk_g2s): B(k, n) = TB ? W[n*ldb + k]
// : W[k*ldb + n], K x N, per 32-wide K chunk [hi | lo] of NT rows x 128 bytes, K-major
// SW128.  Built once per context; the per-centre GEMMs then stage it with two bulk copies.
__global__ void k_weight_image(const float* __restrict__ W, int TB, int ldb, int K, int N, int NT,
                               uint8_t* __restrict__ out) {
  const int nch = (K + tc::kKC - 1) / tc::kKC;
  const long total = static_cast<long>(nch) * NT * tc::kKC;
  for (long e = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int kl = static_cast<int>(e % tc::kKC);
    const int n = static_cast<int>((e / tc::kKC) % NT);
    const int c = static_cast<int>(e / (static_cast<long>(tc::kKC) * NT));
    const int k = c * tc::kKC + kl;
    float v = 0.f;
    if (n < N && k < K) v = TB ? W[static_cast<size_t>(n) * ldb + k] : W[static_cast<size_t>(k) * ldb + n];
    const float hi = tc::tf32_rn(v);
    uint8_t* img = out + static_cast<size_t>(c) * 2 * NT * 128;
    const uint32_t off = tc::sw128_off(n, kl);
    *reinterpret_cast<float*>(img + off) = hi;
    *reinterpret_cast<float*>(img + static_cast<size_t>(NT) * 128 + off) = v - hi;
  }
}

size_t weight_image_bytes(int K, int N) {
  const int nch = (K + tc::kKC - 1) / tc::kKC;
  const int NT = (N + 15) & ~15;
  return static_cast<size_t>(nch) * 2 * NT * 128;
}

void launch_weight_image(const float* W, int TB, int ldb, int K, int N, uint8_t* out, cudaStream_t st) {
  const int NT = (N + 15) & ~15;
  k_weight_image<<<128, 256, 0, st>>>(W, TB, ldb, K, N, NT, out);
  count_launch();
}


template <int MODE, bool WIMG, bool PACK>
static void set_smem(size_t smem) {
  ensure_smem_attr(reinterpret_cast<const void*>(k_centre_forward<MODE, WIMG, PACK>), smem);
  ensure_smem_attr(reinterpret_cast<const void*>(k_centre_backward<MODE, WIMG, PACK>), smem);
}

template <bool FWD>
static void launch_centre(const DpArgs& a, int grid, cudaStream_t st) {
  if (a.n_centres == 0) return;
  cudaMemsetAsync(a.work, 0, sizeof(int), st);
  const size_t smem = dp_smem_bytes(a, a.mode);
  auto go = [&](auto mode_c, auto wimg_c, auto pack_c) {
    constexpr int MODE = decltype(mode_c)::value;
    constexpr bool WIMG = decltype(wimg_c)::value;
    constexpr bool PACK = decltype(pack_c)::value;
    set_smem<MODE, WIMG, PACK>(smem);
    if (FWD) k_centre_forward<MODE, WIMG, PACK><<<grid, 256, smem, st>>>(a);
    else k_centre_backward<MODE, WIMG, PACK><<<grid, 256, smem, st>>>(a);
  };
  using T = std::true_type;
  using F = std::false_type;
  // multi-centre units only with tcgen05 and weight images (context.cpp decides)
  if (a.packs && a.mode == 1) go(std::integral_constant<int, 1>{}, T{}, T{});
  else if (a.packs) go(std::integral_constant<int, 2>{}, T{}, T{});
  else if (a.mode == 0) go(std::integral_constant<int, 0>{}, F{}, F{});
  else if (a.mode == 1 && a.wimg) go(std::integral_constant<int, 1>{}, T{}, F{});
  else if (a.mode == 1) go(std::integral_constant<int, 1>{}, F{}, F{});
  else if (a.wimg) go(std::integral_constant<int, 2>{}, T{}, F{});
  else go(std::integral_constant<int, 2>{}, F{}, F{});
  count_launch();
}

void launch_centre_forward(const DpArgs& a, int grid, cudaStream_t st) { launch_centre<true>(a, grid, st); }
void launch_centre_backward(const DpArgs& a, int grid, cudaStream_t st) { launch_centre<false>(a, grid, st); }

// ------------------------------------------------------------------------------------
// Fitting net over all centres (dp_core.hpp:386-391 forward; 408-414 backward)
// ------------------------------------------------------------------------------------
enum { EPI_STORE = 0, EPI_TANH_BIAS = 1, EPI_DTANH = 2 };

// Split-K (tcgen05 modes): CTA z of gridDim.z takes K range [z Kc, (z+1) Kc) (Kc a multiple
// of the 128-wide FP32 promotion group) and stores its raw tile to the workspace slice z;
// k_fit_splitk_sum then adds the slices in slice order and applies the epilogue.  The
// split depends on K only, never on the centre count, so a centre's energy is the same
// bits at every DD rank count; it matters when few row tiles (many ranks) leave SMs idle
// over the K = M * mr = 4096 reduction.
constexpr int kFitSplit = 8;

__host__ __device__ inline int fit_split(int K) {
  return (K >= 1024 && (K / 128) % kFitSplit == 0) ? kFitSplit : 1;
}

// M: row capacity (grid, split-K slice stride); rows >= *M_live are not computed.
template <bool TB, int MODE>
__global__ void __launch_bounds__(256, 1) k_fit_gemm(int M, const int* __restrict__ M_live, int N, int K,
                                                     const float* __restrict__ A, const float* __restrict__ B,
                                                     int ldb, float* __restrict__ C, const float* __restrict__ bias,
                                                     const float* __restrict__ Y, int epi_mode) {
  extern __shared__ __align__(1024) unsigned char fit_smem_raw[];
  unsigned char* head = fit_smem_raw + ((1024 - (tc::smem_u32(fit_smem_raw) & 1023)) & 1023);
  constexpr int TM = MODE == 0 ? kTM : tc::kMT;
  constexpr int TN = MODE == 0 ? kTN : tc::kNT;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int Mv = M_live ? min(M, *M_live) : M;
  if (m0 >= Mv) return;  // past the rank's live centres (the grid covers the capacity)
  const int Ms = min(TM, Mv - m0), Ns = min(TN, N - n0);
  // split-K slice (gridDim.z > 1): raw partial tile into C's slice z, epilogue later
  const int Kc = K / static_cast<int>(gridDim.z), kz = static_cast<int>(blockIdx.z) * Kc;
  const float* Ab = A + static_cast<size_t>(m0) * K + kz;
  const float* Bb = (TB ? B + static_cast<size_t>(n0) * ldb : B + n0) + (TB ? kz : static_cast<size_t>(kz) * ldb);
  float* Cz = C + static_cast<size_t>(blockIdx.z) * M * N;
  const int mode = gridDim.z > 1 ? EPI_STORE : epi_mode;
  Mm<MODE, 2> mm;
  mm.init(head, 512);
  mm.template run<false, TB, 4>(Ms, Ns, Kc, Ab, K, Bb, ldb, [&](int m, int n, auto v) {
    const size_t o = static_cast<size_t>(m0 + m) * N + n0 + n;
    if (mode == EPI_TANH_BIAS) v = vtanh(v + vld(&bias[n0 + n], v));
    else if (mode == EPI_DTANH) v = v * vdtanh(vld(&Y[o], v));
    vst(&Cz[o], v);
  });
  mm.finish();
}

__global__ void k_fit_splitk_sum(int M, const int* __restrict__ M_live, int N, int S, const float* __restrict__ P,
                                 float* __restrict__ C, const float* __restrict__ bias, const float* __restrict__ Y,
                                 int epi_mode) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const size_t MN = static_cast<size_t>(M) * N;
  const int Mv = M_live ? min(M, *M_live) : M;
  if (i >= static_cast<size_t>(Mv) * N) return;
  float p[kFitSplit];  // all slices' loads in flight, then a fixed-order sum
#pragma unroll
  for (int z = 0; z < kFitSplit; ++z) p[z] = z < S ? P[z * MN + i] : 0.f;
  float v = p[0];
#pragma unroll
  for (int z = 1; z < kFitSplit; ++z)
    if (z < S) v += p[z];
  if (epi_mode == EPI_TANH_BIAS) v = tanhf(v + bias[i % N]);
  else if (epi_mode == EPI_DTANH) v = v * (1.f - Y[i] * Y[i]);
  C[i] = v;
}

template <bool TB, int MODE>
static void fit_gemm(int M, const int* M_live, int N, int K, const float* A, const float* B, int ldb, float* C,
                     const float* bias, const float* Y, int epi, cudaStream_t st, float* ws = nullptr, int n_sm = 0) {
  constexpr int TM = MODE == 0 ? kTM : tc::kMT;
  constexpr int TN = MODE == 0 ? kTN : tc::kNT;
  const size_t smem = head_bytes(MODE, 2) + 1024;
  ensure_smem_attr(reinterpret_cast<const void*>(k_fit_gemm<TB, MODE>), smem);
  const int S = (MODE != 0 && ws && N <= TN) ? fit_split(K) : 1;
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM, S);
  k_fit_gemm<TB, MODE><<<grid, 256, smem, st>>>(M, M_live, N, K, A, B, ldb, S > 1 ? ws : C, bias, Y, epi);
  count_launch();
  if (S > 1) {
    const size_t MN = static_cast<size_t>(M) * N;
    k_fit_splitk_sum<<<static_cast<int>((MN + 255) / 256), 256, 0, st>>>(M, M_live, N, S, ws, C, bias, Y, epi);
    count_launch();
  }
}

template <int MODE>
static void fit_gemm_tb(bool tb, int M, const int* M_live, int N, int K, const float* A, const float* B, int ldb,
                        float* C, const float* bias, const float* Y, int epi, cudaStream_t st, float* ws, int n_sm) {
  if (tb) fit_gemm<true, MODE>(M, M_live, N, K, A, B, ldb, C, bias, Y, epi, st, ws, n_sm);
  else fit_gemm<false, MODE>(M, M_live, N, K, A, B, ldb, C, bias, Y, epi, st, ws, n_sm);
}

size_t fit_workspace_floats(int n_centres, int width) {
  return static_cast<size_t>(kFitSplit) * n_centres * width + 4;
}

// e[c] = b + w . Y[c]   (linear output layer); delta[c][o] = w[o] (1 - Y[c][o]^2)
__global__ void k_fit_out(int nc, const int* __restrict__ nc_live, int H, const float* __restrict__ Y,
                          const float* __restrict__ w, const float* __restrict__ b, double* __restrict__ e,
                          float* __restrict__ delta) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= (nc_live ? min(nc, *nc_live) : nc)) return;
  const float* y = Y + static_cast<size_t>(c) * H;
  float acc = 0.f;
  for (int o = lane; o < H; o += 32) {
    const float v = y[o];
    acc += w[o] * v;
    if (delta) delta[static_cast<size_t>(c) * H + o] = w[o] * (1.f - v * v);
  }
  acc = warp_sum(acc);
  if (lane == 0) e[c] = static_cast<double>(acc) + static_cast<double>(b[0]);
}

__global__ void k_fill_rows(int nc, const int* __restrict__ nc_live, int H, const float* __restrict__ w,
                            float* __restrict__ out) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<size_t>(nc_live ? min(nc, *nc_live) : nc) * H) return;
  out[i] = w[i % H];
}

int fit_split_k(int K) { return fit_split(K); }

void launch_fit_splitk_sum(int M, const int* M_live, int N, int S, const float* P, float* C, const float* bias,
                           const float* Y, int epi, cudaStream_t st) {
  const size_t MN = static_cast<size_t>(M) * N;
  k_fit_splitk_sum<<<static_cast<int>((MN + 255) / 256), 256, 0, st>>>(M, M_live, N, S, P, C, bias, Y, epi);
  count_launch();
}

void launch_fit_out(const FitArgs& a, float* delta, cudaStream_t st) {
  const int nc = a.n_centres, L = a.n_fit, H = a.fdims[L - 1];
  k_fit_out<<<(nc * 32 + 255) / 256, 256, 0, st>>>(nc, a.n_centres_dev, H, a.Y[L - 2], a.fw[L - 1], a.fb[L - 1],
                                                   a.e, delta);
  count_launch();
}

void launch_fit(const FitArgs& a, cudaStream_t st) {
  const int nc = a.n_centres;
  if (nc == 0) return;
  if (!(a.flags & 32) && fit_tma_supported(a)) {
    launch_fit_tma(a, st);
    return;
  }
  const int L = a.n_fit;
  auto gemm = [&](bool tb, int N, int K, const float* A, const float* B, int ldb, float* C,
                  const float* bias, const float* Y, int mode) {
    const int* ml = a.n_centres_dev;
    if (a.mode == 0) fit_gemm_tb<0>(tb, nc, ml, N, K, A, B, ldb, C, bias, Y, mode, st, nullptr, 0);
    else if (a.mode == 1) fit_gemm_tb<1>(tb, nc, ml, N, K, A, B, ldb, C, bias, Y, mode, st, a.ws, a.n_sm);
    else fit_gemm_tb<2>(tb, nc, ml, N, K, A, B, ldb, C, bias, Y, mode, st, a.ws, a.n_sm);
  };
  // forward hidden layers: Y_l = tanh(X W_l^T + b_l)
  const float* x = a.D;
  for (int l = 0; l + 1 < L; ++l) {
    gemm(true, a.fdims[l + 1], a.fdims[l], x, a.fw[l], a.fdims[l], a.Y[l], a.fb[l], nullptr, EPI_TANH_BIAS);
    x = a.Y[l];
  }
  const int H = a.fdims[L - 1];
  if (L == 1) {
    // e = b + w . D ; dD = w
    k_fit_out<<<(nc * 32 + 255) / 256, 256, 0, st>>>(nc, a.n_centres_dev, H, a.D, a.fw[0], a.fb[0], a.e, nullptr); count_launch();
    k_fill_rows<<<static_cast<int>((static_cast<size_t>(nc) * H + 255) / 256), 256, 0, st>>>(nc, a.n_centres_dev, H, a.fw[0], a.dD); count_launch();
    return;
  }
  float* dcur = a.delta[0];
  float* dnxt = a.delta[1];
  k_fit_out<<<(nc * 32 + 255) / 256, 256, 0, st>>>(nc, a.n_centres_dev, H, a.Y[L - 2], a.fw[L - 1], a.fb[L - 1], a.e, dcur); count_launch();
  // delta_{l-1} = (delta_l W_l) o (1 - Y_{l-1}^2);  dD = delta_0 W_0
  for (int l = L - 2; l >= 1; --l) {
    gemm(false, a.fdims[l], a.fdims[l + 1], dcur, a.fw[l], a.fdims[l], dnxt, nullptr, a.Y[l - 1], EPI_DTANH);
    float* t = dcur;
    dcur = dnxt;
    dnxt = t;
  }
  gemm(false, a.fdims[0], a.fdims[1], dcur, a.fw[0], a.fdims[0], a.dD, nullptr, nullptr, EPI_STORE);
}

}  // namespace nb

namespace nb {
// ------------------------------------------------------------------------------------
// Self-test of the block GEMM building blocks (one CTA): C = A(TA) * B(TB).
// ------------------------------------------------------------------------------------
template <bool TA, bool TB, int MODE>
__global__ void __launch_bounds__(256, 1) k_selftest_gemm(int M, int N, int K, const float* A, int lda,
                                                          const float* B, int ldb, float* C) {
  extern __shared__ __align__(1024) unsigned char st_smem_raw[];
  unsigned char* head = st_smem_raw + ((1024 - (tc::smem_u32(st_smem_raw) & 1023)) & 1023);
  Mm<MODE> mm;
  mm.init(head, 256);
  mm.template run<TA, TB, 0, 0>(M, N, K, A, lda, B, ldb, [&](int m, int n, float v) { C[static_cast<size_t>(m) * N + n] = v; });
  mm.finish();
}

template <int MODE>
static void selftest_mode(int ta, int tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                          float* C) {
  const size_t smem = head_bytes(MODE, 1) + 1024;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<1, 256, smem>>>(M, N, K, A, lda, B, ldb, C);
  };
  if (ta && tb) go(k_selftest_gemm<true, true, MODE>);
  else if (ta) go(k_selftest_gemm<true, false, MODE>);
  else if (tb) go(k_selftest_gemm<false, true, MODE>);
  else go(k_selftest_gemm<false, false, MODE>);
}

void selftest_gemm(int mode, int ta, int tb, int M, int N, int K, const float* A, int lda, const float* B,
                   int ldb, float* C) {
  if (mode == 0) selftest_mode<0>(ta, tb, M, N, K, A, lda, B, ldb, C);
  else if (mode == 1) selftest_mode<1>(ta, tb, M, N, K, A, lda, B, ldb, C);
  else selftest_mode<2>(ta, tb, M, N, K, A, lda, B, ldb, C);
}
}  // namespace nb
