// TMA-fed block GEMM on sm_100a (tcgen05.mma kind::tf32, accumulator in TMEM).
//
//   C(m, n) = epi(sum_p sum_k A_p(m, k) B_p(k, n)),  0 <= m < M <= 128, 0 <= n < N <= 128
//   (an MN-major operand's M / N extent is a multiple of 32)
//
// Every operand tile is moved by the TMA engine (cp.async.bulk.tensor.3d, one elected thread)
// from a row-major fp32 matrix in global memory / L2 into a SWIZZLE_64B shared-memory
// stage, either K-major (K contiguous) or MN-major (M/N contiguous: a transposed operand is
// read as it lies, no register transposes; tcgen05 accepts MN-major TF32).  The tensor core
// reads the raw fp32 bits as the "hi" operand; the threads only form lo = x - hi in shared
// memory.  A goes on to TMEM (TS-mode MMA: each thread moves 8 values of its TMEM lane,
// raw and lo, with tcgen05.st), so the tensor core reads only B from shared memory -- SS-mode
// N = 128 MMAs measured 70-88 % of the TF32 rate against 93-100 % for TS (tools/micro/
// mma_rate.cu), and the main loop is shared-memory-bandwidth bound.  One thread issues
//   NPASS = 3: A B + A lo(B) + lo(A) B   (FP32-grade "3xTF32")
//   NPASS = 1: A B                       (plain TF32)
// per 8-wide k-step and commits to the stage's mbarrier.
//
// Pipeline: a ring of kStages stages of 16 K columns (smem: A raw | B raw | B lo, 8 KB each;
// TMEM: kAStages stages of A raw | A lo, 16 columns each).  Chunk c+kStages-1 is requested as soon as the MMAs
// of chunk c are issued (after the MMAs of chunk c-1 have drained its stage), so global
// latency hides behind three chunks of tensor work; the threads never touch global memory
// in the main loop.  The chunk counter g runs over all GEMMs of the CTA, so stage and
// mbarrier phase are pure functions of it.
// TMEM map (cols = 256): [0, 128) accumulator, [128 + 32 s, +32) A stage s.  With 512
// columns (PROMOTE, one CTA per SM): second group accumulator [256, 384), sum [384, 512).
//
// Layout conventions (tmap.h): K-major operands arrive as SWIZZLE_64B tiles (box {16, 128 or
// N, 1} of the view {16, rows, cols/16}); MN-major operands as SWIZZLE_128B_BASE32B tiles
// (box {32, 16, MN/32} of the view {32, rows, cols/32}), the only MN-major TF32 layout.
// Operands past a matrix's valid rows/columns must be finite; along K at least one of A, B
// must be exactly zero there (the producers zero-pad to 16).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "tc_gemm.cuh"

namespace nb {
namespace tg {

constexpr int kThreads = 256;        // warp 0 MMA issuer, warps 1-7 split (warp 4 also produces)
constexpr int kPromoThreads = 384;   // PROMOTE: + warps 8-11 promote
constexpr int kKC = 16;                  // K columns per chunk: one 64-byte swizzle row
constexpr int kStages = 8;   // shared-memory ring: TMA requests run up to 7 chunks ahead
constexpr int kAStages = 4;  // TMEM A stages (chunk g uses g % kAStages)

constexpr uint32_t kOpBytes = 8192;      // one operand tile: 128 x 16 fp32
constexpr uint32_t kStageBytes = 3 * kOpBytes;  // A raw | B raw | B lo
constexpr uint32_t kRingBytes = kStages * kStageBytes;  // 192 KB; epilogue staging reuses it
constexpr uint32_t kTmemA = 128;         // TMEM column of A stage 0
constexpr uint32_t kTmemAcc1 = 256;      // PROMOTE: second group accumulator (512 columns)
constexpr uint32_t kTmemSum = 384;       // PROMOTE: promoted FP32 sum
constexpr int kMaxN = 128;

// Barriers and the TMEM slot; lives next to the ring in shared memory.
struct Ctl {
  uint64_t full[kStages];   // TMA landed
  uint64_t ready[kStages];  // split warps done (7 arrivals)
  uint64_t empty[kStages];  // MMAs drained (tcgen05.commit)
  uint64_t grp[2];          // PROMOTE: K group accumulated into TMEM buffer b (tcgen05.commit)
  uint64_t promo[2];        // PROMOTE: buffer b added into the sum (4 promoter warps)
  uint32_t tmem_base;
  uint32_t pad;
};

struct Ring {
#ifdef TG_PROF
  long long* prof;   // thread 0 (issuer): [0] wait ready, [1] MMA issue, [2] main loop, [3] drain, [4] TMEM->smem, [5] functor, [6] fence+sync
  long long t;
  unsigned long long* gprof;  // global: [0] warp 1 waiting for TMA landings
#endif
#ifdef TG_TRACE
  long long* trace;  // [chunk][5]: request, landed (warp 1), ready (issuer), MMAs issued, drained (polled)
#endif
  uint8_t* base;  // kRingBytes, 1024-aligned
  Ctl* ctl;
  uint32_t tmem;  // accumulator columns [0, 128) (+ [128, 256) promoted sum)
  uint32_t cols;
  uint32_t g;     // chunks issued so far (identical in every thread)
  uint32_t grp;   // PROMOTE K groups so far
};

// One operand of one product.
struct Op {
  const CUtensorMap* map;
  int mn;          // 0: K-major, 1: MN-major
  int r, c;        // K-major: first M/N row, first K column; MN-major: first K row, first M/N column
  uint32_t bytes;  // bytes the map's box delivers (<= kOpBytes)
};

__host__ __device__ inline Op op(const CUtensorMap* map, int mn, int r, int c, uint32_t bytes) {
  Op o;
  o.map = map;
  o.mn = mn;
  o.r = r;
  o.c = c;
  o.bytes = bytes;
  return o;
}

using tc::fence_after;
using tc::fence_before;
using tc::mbar_init;
using tc::mbar_wait;
using tc::smem_u32;

__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t"
      "}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// generic-proxy global writes -> later TMA (async-proxy) reads of the same data
__device__ __forceinline__ void fence_global_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// all threads: make this CTA's global writes visible to its later TMA loads
__device__ __forceinline__ void publish() {
  fence_global_async();
  __syncthreads();
}

// SWIZZLE_64B descriptors (sm_100 version 1, layout type 4).
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {  // K-major: 64-byte rows, 8-row groups 512 B
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(4) << 61);
}
// MN-major: SWIZZLE_128B_BASE32B (layout type 1), 32-wide blocks 2 KB apart (LBO), 4-row K
// groups 512 B apart (SBO); one 8-row k-step = 1 KB
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(2048 >> 4) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(1) << 61);
}
// D f32, A/B tf32, M = 128, N = n, majors
__device__ __forceinline__ uint32_t idesc(int n, int amn, int bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(amn) << 15) | (static_cast<uint32_t>(bmn) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

// Initialise barriers and allocate TMEM (cols = 256).  All threads.
__device__ __forceinline__ void init(Ring& rg, uint8_t* ring, Ctl* ctl, uint32_t cols = 256) {
  rg.base = ring;
  rg.ctl = ctl;
  rg.cols = cols;
  rg.g = 0;
  rg.grp = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&ctl->tmem_base)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->ready[s], 7);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->grp[b], 1);
      mbar_init(&ctl->promo[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  rg.tmem = ctl->tmem_base;
}

__device__ __forceinline__ void finish(Ring& rg) {
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(rg.tmem), "r"(rg.cols) : "memory");
}

__device__ __forceinline__ uint8_t* stage_ptr(const Ring& rg, uint32_t g) { return rg.base + (g % kStages) * kStageBytes; }

// lo(x) = x - tf32(x) with the tensor core's own reading of x (RZ: the low 13 bits are ignored;
// measured, tools/micro/tma_test.cu)
__device__ __forceinline__ float lo1(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float4 lo4(float4 v) { return make_float4(lo1(v.x), lo1(v.y), lo1(v.z), lo1(v.w)); }
// 3xTF32 split with round-to-nearest hi (tf32_rn, exactly representable, so the tensor core
// reads it unchanged): |lo| <= 2^-11 |x| with either sign, so the dropped lo*lo term neither
// reaches 2^-20 nor has a systematic sign, as with the truncated hi of the raw operand
__device__ __forceinline__ float4 hi4(float4 v) {
  return make_float4(tc::tf32_rn(v.x), tc::tf32_rn(v.y), tc::tf32_rn(v.z), tc::tf32_rn(v.w));
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}

// 8 consecutive K values (k = 8h .. 8h+7 of the chunk) of A row r from the TMA-landed tile.
__device__ __forceinline__ void a_row8(const uint8_t* t, int mn, int r, int h, float (&v)[8]) {
  if (!mn) {  // K-major SW64: 64-byte rows, 16-byte chunk j at j ^ ((r >> 1) & 3)
    const uint8_t* row = t + r * 64;
    const int sw = (r >> 1) & 3;
    const float4 x = *reinterpret_cast<const float4*>(row + (((2 * h) ^ sw) << 4));
    const float4 y = *reinterpret_cast<const float4*>(row + (((2 * h + 1) ^ sw) << 4));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {  // MN-major SW128_32B: 32-column blocks of 2 KB, 128-byte K rows, 32-byte atoms ^ (k & 3)
    const uint8_t* blk = t + (r >> 5) * 2048 + (r & 7) * 4;
    const int at = (r & 31) >> 3;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = 8 * h + j;
      v[j] = *reinterpret_cast<const float*>(blk + k * 128 + ((at ^ (k & 3)) << 5));
    }
  }
}

// Multi-product GEMM: chunks [0, n1) from (a1, b1) over K1, then [n1, n1+n2) from (a2, b2).
// EK: 1 vector functor epi(m, n, float4|float) over rows < M, cols < N; 2 tile functor
// epi(stg, ldst, M, N) on the SMEM-staged accumulator, called by every thread.
// Roles in the main loop (kThreads = 256): warp 0 lane 0 issues the MMAs and is the TMA
// producer: while it waits for chunk c's splits it polls the `empty` barriers and requests
// every chunk whose stage (that of chunk j - kStages) has drained, up to c + kStages - 1.
// Warps 1-7 split each landed chunk (A -> TMEM raw + lo, B -> smem lo) and arrive on the
// stage's `ready` barrier.
// TMEM lane quarter = warp % 4: warp 4 covers lanes 0-31 alone (both k halves), warps q and
// q + 4 share the others; the B split runs on warps 1-3 and 5-7.
// PROMOTE > 0 (long K; kPromoThreads, 512 TMEM columns, one CTA per SM): K groups of PROMOTE
// chunks alternate between accumulators at columns 0 and kTmemAcc1; promoter warps 8-11 add
// each finished group in FP32 into the sum at kTmemSum while the next group accumulates
// (the tensor core's own accumulation truncates: -5e-6 relative bias at K = 512).
#ifdef TG_PROF
#define TG_TICK(i)                                          \
  if (tid == 0 && rg.prof) {                                \
    const long long t_ = clock64();                         \
    if ((i) >= 0) rg.prof[(i)] += t_ - rg.t;                \
    rg.t = t_;                                              \
  }
#else
#define TG_TICK(i)
#endif

template <int NPASS, int EK, int PROMOTE_ = 0, class Epi>
__device__ __forceinline__ void gemm(Ring& rg, int M, int N, int K1, const Op& a1, const Op& b1, int K2, const Op& a2,
                                     const Op& b2, Epi epi) {
  constexpr int PROMOTE = PROMOTE_ > 0 ? PROMOTE_ : 0;
  constexpr int PG = PROMOTE_ > 0 ? PROMOTE_ : 1;  // group size for index arithmetic
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int NT = (N + 15) & ~15;
  const int n1 = (K1 + kKC - 1) / kKC;
  const int nch = n1 + (K2 + kKC - 1) / kKC;
  const int ngrp = PROMOTE > 0 ? (nch + PG - 1) / PG : 1;
  const uint32_t g0 = rg.g;
  const uint32_t G0 = rg.grp;  // global K-group index of this GEMM's first group
  Ctl* ctl = rg.ctl;
  const uint32_t lanes = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  auto issue = [&](int c) {
    const bool p1 = c < n1;
    const Op& a = p1 ? a1 : a2;
    const Op& b = p1 ? b1 : b2;
    const int kc = p1 ? c : c - n1;
    const uint32_t g = g0 + c;
    uint8_t* st = stage_ptr(rg, g);
    uint64_t* bar = &ctl->full[g % kStages];
#ifdef TG_TRACE
    if (rg.trace && c < 64) rg.trace[c * 5 + 0] = clock64();
#endif
    tc::mbar_expect_tx(bar, a.bytes + b.bytes);
    if (a.mn) tma_load3(st, a.map, 0, a.r + kKC * kc, a.c >> 5, bar);
    else tma_load3(st, a.map, 0, a.r, (a.c >> 4) + kc, bar);
    if (b.mn) tma_load3(st + kOpBytes, b.map, 0, b.r + kKC * kc, b.c >> 5, bar);
    else tma_load3(st + kOpBytes, b.map, 0, b.r, (b.c >> 4) + kc, bar);
  };
  TG_TICK(-1);
  if (warp == 0) {
    if (lane == 0) {
      int next = 0;  // next chunk to request
      for (int c = 0; c < nch; ++c) {
        const uint32_t g = g0 + c;
        const int s = g % kStages;
        const int bmn = c < n1 ? b1.mn : b2.mn;
        const uint32_t ta = rg.tmem + kTmemA + 32u * (g % kAStages);
        uint32_t acc_t = rg.tmem;
        bool start = c == 0;
        if (PROMOTE > 0) {
          const uint32_t gg = G0 + c / PG;
          acc_t = rg.tmem + ((gg & 1) ? kTmemAcc1 : 0u);
          start = c % PG == 0;
          // buffer gg & 1 was last used by group gg - 2: wait for its promotion
          if (start && c >= 2 * PG) mbar_wait(&ctl->promo[gg & 1], ((gg - 2) >> 1) & 1u);
        }
#ifdef TG_PROF
        const long long tr0 = clock64();
#endif
        // wait for chunk c's splits; meanwhile request every chunk (up to c + kStages - 1) whose
        // stage -- that of chunk j - kStages -- has drained
        {
          const uint32_t ph = (g / kStages) & 1u;
          while (true) {
            if (next < nch && next <= c + kStages - 1) {
              const int pj = next - kStages;
              if (pj < 0 || mbar_test(&ctl->empty[(g0 + pj) % kStages], ((g0 + pj) / kStages) & 1u)) {
                issue(next);
                ++next;
                continue;
              }
            }
            if (mbar_test(&ctl->ready[s], ph)) break;
          }
        }
#ifdef TG_PROF
        const long long tr1 = clock64();
        if (rg.prof) rg.prof[0] += tr1 - tr0;
#endif
#ifdef TG_TRACE
        if (rg.trace && c < 64) rg.trace[c * 5 + 2] = clock64();
#endif
        fence_after();
        const uint32_t id = idesc(NT, 0, bmn);
        const uint32_t sb = smem_u32(rg.base + s * kStageBytes) + kOpBytes;
#pragma unroll
        for (int kk = 0; kk < kKC / 8; ++kk) {
          const uint32_t bo = bmn ? 1024u * kk : 32u * kk;
          auto db = [&](uint32_t x) { return bmn ? desc_mn(x) : desc_k(x); };
          const uint32_t acc = (!start || kk > 0) ? 1u : 0u;
          tc::mma_tf32_ts(acc_t, ta + 8u * kk, db(sb + bo), id, acc);
          if (NPASS > 1) {
            tc::mma_tf32_ts(acc_t, ta + 8u * kk, db(sb + kOpBytes + bo), id, 1u);
            tc::mma_tf32_ts(acc_t, ta + 16u + 8u * kk, db(sb + bo), id, 1u);
          }
        }
        tc::mma_commit(&ctl->empty[s]);
#ifdef TG_PROF
        if (rg.prof) rg.prof[1] += clock64() - tr1;
#endif
#ifdef TG_TRACE
        if (rg.trace && c < 64) rg.trace[c * 5 + 3] = clock64();
#endif
        if (PROMOTE > 0 && ((c + 1) % PG == 0 || c + 1 == nch)) tc::mma_commit(&ctl->grp[(G0 + c / PG) & 1]);
      }
    }
    __syncwarp();
  } else if (warp < 8) {
    const int arow = 32 * (warp & 3) + lane, ah = warp >> 2;  // A row (TMEM lane), k half
    for (int c = 0; c < nch; ++c) {
      const uint32_t g = g0 + c;
      const int s = g % kStages;
      const bool p1 = c < n1;
      const int amn = p1 ? a1.mn : a2.mn;
      const uint32_t bbytes = p1 ? b1.bytes : b2.bytes;
      uint8_t* st = rg.base + s * kStageBytes;
      const uint32_t ta = rg.tmem + kTmemA + 32u * (g % kAStages) + lanes;  // A raw; lo at +16
#if defined(TG_TRACE) || defined(TG_PROF)
      const long long tw0 = clock64();
#endif
      mbar_wait(&ctl->full[s], (g / kStages) & 1u);
      // the TMEM A stage is shared with chunk g - kAStages: its MMAs must have drained (the
      // ring's TMA request only waited for chunk g - kStages); earlier GEMMs drained in
      // their epilogue
      if (c >= kAStages) {
        const uint32_t gp = g - kAStages;
        mbar_wait(&ctl->empty[gp % kStages], (gp / kStages) & 1u);
      }
      __syncwarp();  // reconverge before the .sync.aligned TMEM stores
#ifdef TG_PROF
      if (rg.gprof && warp == 1 && lane == 0) atomicAdd(rg.gprof, static_cast<unsigned long long>(clock64() - tw0));
#endif
#ifdef TG_TRACE
      if (rg.trace && c < 64 && warp == 1 && lane == 0) rg.trace[c * 5 + 1] = clock64();
#endif
      fence_after();  // the MMAs that last read this TMEM stage drained before its TMA was issued
#ifdef TG_TRACE
      long long tt[6];
      tt[0] = clock64();
#endif
      // all shared-memory loads first (the TMEM stores carry memory clobbers)
      float v0[8], v1[8];
      float4 bv[3];
      const bool two_h = warp == 4;
      a_row8(st, amn, arow, two_h ? 0 : ah, v0);
      if (two_h) a_row8(st, amn, arow, 1, v1);
      const float4* br = reinterpret_cast<const float4*>(st + kOpBytes);
      float4* bl = reinterpret_cast<float4*>(st + 2 * kOpBytes);
      const int nb = bbytes >> 4;
      const int bt = (warp < 4 ? warp - 1 : warp - 2) * 32 + lane;  // 0 .. 191 (not warp 4)
      if (NPASS > 1 && !two_h) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
          if (bt + 192 * i < nb) bv[i] = br[bt + 192 * i];
      }
#ifdef TG_TRACE
      tt[1] = clock64();
#endif
      const int h0 = two_h ? 0 : ah;
      __syncwarp();
      if (NPASS > 1) {
        // hi = tf32_rn(x) into the A stage, lo = x - hi
        float h0v[8], h1v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          h0v[j] = tc::tf32_rn(v0[j]);
          h1v[j] = tc::tf32_rn(v1[j]);
          v0[j] -= h0v[j];
          v1[j] -= h1v[j];
        }
        tmem_st8(ta + 8u * h0, h0v);
        if (two_h) tmem_st8(ta + 8u, h1v);
        tmem_st8(ta + 16u + 8u * h0, v0);
        if (two_h) tmem_st8(ta + 24u, v1);
        __syncwarp();
        if (!two_h) {
          // B: the landed tile is rewritten in place as hi, its low parts go to the lo tile
          float4* bh = const_cast<float4*>(br);
#pragma unroll
          for (int i = 0; i < 3; ++i)
            if (bt + 192 * i < nb) {
              const float4 h = hi4(bv[i]);
              bh[bt + 192 * i] = h;
              bl[bt + 192 * i] = make_float4(bv[i].x - h.x, bv[i].y - h.y, bv[i].z - h.z, bv[i].w - h.w);
            }
        }
      } else {
        tmem_st8(ta + 8u * h0, v0);
        if (two_h) tmem_st8(ta + 8u, v1);
      }
#ifdef TG_TRACE
      tt[2] = clock64();
#endif
      if (NPASS > 1) tc::fence_proxy_async();
#ifdef TG_TRACE
      tt[3] = clock64();
#endif
      __syncwarp();  // the B split above is divergent: reconverge before the aligned wait
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#ifdef TG_TRACE
      tt[4] = clock64();
#endif
      fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ctl->ready[s])) : "memory");

#ifdef TG_TRACE
      tt[5] = clock64();
      if (rg.trace && c >= 8 && c < 16 && lane == 0) {
        long long* o = rg.trace + 320 + (warp * 8 + (c - 8)) * 2;
        o[0] = tt[0] - tw0;  // waiting for the landing
        o[1] = tt[5] - tt[0];  // own work
      }
#endif
    }
  } else if (PROMOTE > 0) {
    // promoter warps 8-11: sum += finished group (lane quarter warp % 4, all NT columns)
    for (int gi = 0; gi < ngrp; ++gi) {
      const uint32_t gg = G0 + gi;
      const int b = gg & 1;
      mbar_wait(&ctl->grp[b], (gg >> 1) & 1u);
      __syncwarp();
      fence_after();
      const uint32_t src = rg.tmem + lanes + (b ? kTmemAcc1 : 0u);
      const uint32_t dst = rg.tmem + lanes + kTmemSum;
      for (int c0 = 0; c0 < NT; c0 += 16) {
        float p[16], t[16];
        tc::tmem_ld16(src + static_cast<uint32_t>(c0), p);
        if (gi > 0) {
          tc::tmem_ld16(dst + static_cast<uint32_t>(c0), t);
#pragma unroll
          for (int j = 0; j < 16; ++j) p[j] += t[j];
        }
        tc::tmem_st16(dst + static_cast<uint32_t>(c0), p);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ctl->promo[b])) : "memory");
    }
  }
  TG_TICK(2);
  rg.g = g0 + nch;
  if (PROMOTE > 0) {
    // the last group's promotion carries every MMA
    const uint32_t gl = G0 + ngrp - 1;
    mbar_wait(&ctl->promo[gl & 1], (gl >> 1) & 1u);
    __syncwarp();
    rg.grp = G0 + ngrp;
  } else {
    const uint32_t gl = g0 + nch - 1;
    mbar_wait(&ctl->empty[gl % kStages], (gl / kStages) & 1u);  // last commit: every MMA done
  }
  __syncwarp();
  fence_after();
  TG_TICK(3);
  // ---- epilogue
  const uint32_t acc_col = PROMOTE > 0 ? kTmemSum : 0u;
  const int q = warp & 3;
  // TMEM -> registers -> shared (row-major, padded), then the functor: EK = 1 elementwise
  // over rows < M, cols < N (float4 per thread, coalesced rows; direct per-row stores from
  // TMEM measured 2x slower), EK = 2 on the whole tile epi(stg, ldst, M, N)
  {
    float* stg = reinterpret_cast<float*>(rg.base);
    const int ldst = NT + 4;
    if (warp < 8) {
      const int half = ((NT >> 1) + 15) & ~15;
      const int cbeg = (warp < 4) ? 0 : half, cend = (warp < 4) ? half : NT;
      float* srow = stg + static_cast<size_t>(q * 32 + lane) * ldst;
      const uint32_t taddr = rg.tmem + (static_cast<uint32_t>(q * 32) << 16) + acc_col;
      int c0 = cbeg;
      for (; c0 + 32 <= cend; c0 += 32) {
        float v[32];
        tc::tmem_ld16x2(taddr + static_cast<uint32_t>(c0), v);
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(srow + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      for (; c0 < cend; c0 += 16) {
        float v[16];
        tc::tmem_ld16(taddr + static_cast<uint32_t>(c0), v);
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(srow + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    fence_before();
    __syncthreads();
    TG_TICK(4);
    if constexpr (EK == 2) {
      epi(stg, ldst, M, N);
    } else {
      const int nw = blockDim.x >> 5;
      const int nq = N >> 2;
      for (int r = warp; r < M; r += 4 * nw)
        for (int qd = lane; qd < nq; qd += 32) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int rr = r + u * nw;
            if (rr < M) epi(rr, 4 * qd, *reinterpret_cast<const float4*>(stg + static_cast<size_t>(rr) * ldst + 4 * qd));
          }
        }
      const int tail = N - 4 * nq;
      for (int e = tid; e < M * tail; e += blockDim.x) {
        const int rr = e / tail, cc = 4 * nq + e % tail;
        epi(rr, cc, stg[static_cast<size_t>(rr) * ldst + cc]);
      }
    }
  }
  TG_TICK(5);
  fence_global_async();  // the outputs are read back by later TMA loads
  __syncthreads();
  fence_after();
  TG_TICK(6);
}

template <int NPASS, int EK, int PROMOTE = 0, class Epi>
__device__ __forceinline__ void gemm1(Ring& rg, int M, int N, int K, const Op& a, const Op& b, Epi epi) {
  gemm<NPASS, EK, PROMOTE>(rg, M, N, K, a, b, 0, a, b, epi);
}

}  // namespace tg
}  // namespace nb
