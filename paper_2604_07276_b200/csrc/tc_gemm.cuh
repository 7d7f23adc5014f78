// Block-level tensor-core GEMM on sm_100a: tcgen05.mma (kind::tf32) with the accumulator
// in TMEM, operands staged in shared memory in the canonical K-major SWIZZLE_128B layout.
//
//   C(m, n) = epi(m, n, sum_k A(m, k) * B(k, n)),  0 <= m < M, 0 <= n < N
//   A(m, k) = TA ? A[k*lda + m] : A[m*lda + k]        (fp32 in global / L2)
//   B(k, n) = TB ? B[n*ldb + k] : B[k*ldb + n]
//
// Same contract as bgemm (gemm_simt.cuh), so the fused per-centre kernels swap one for
// the other.  NPASS = 3: FP32-grade "3xTF32" (a_hi b_hi + a_hi b_lo + a_lo b_hi, hi =
// cvt.rna.tf32(x), lo = x - hi); NPASS = 1: plain TF32.
//
// Pipeline (256 threads, one CTA per SM): per 32-wide K chunk all threads load A/B from
// global (any transposition is absorbed here), split hi/lo, st.shared into the swizzled
// stage buffer, fence.proxy.async, barrier; thread 0 issues 4 k-steps x NPASS
// tcgen05.mma (M = 128, N <= 256, K = 8 each) and commits to the stage's mbarrier.  Two
// stages: loading chunk c+1 overlaps the tensor core working on chunk c.  The epilogue
// reads the accumulator with tcgen05.ld.32x32b.x16 (warp w owns TMEM lanes
// 32*(w%4)..+31; warps w and w+4 split the columns).
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace nb {
namespace tc {

constexpr int kThreads = 256;
constexpr int kKC = 32;          // K elements per chunk = one 128-byte swizzle row
constexpr int kMT = 128;         // MMA M
constexpr int kNT = 256;         // max MMA N per accumulator tile
constexpr int kTmemCols = 512;   // [0,256): MMA partial, [256,512): promoted FP32 sum
constexpr int kSumCol = 256;

// Shared-memory image: NST pipeline stages of {A hi, A lo, B hi, B lo}; the epilogue
// reuses the stage buffers as its staging tile (needs >= 128 x (kNT+4) floats).
template <int NST>
struct alignas(1024) Smem {
  uint8_t a[NST][2][kMT * 128];  // [stage][hi/lo]  16 KB each
  uint8_t b[NST][2][kNT * 128];  // [stage][hi/lo]  32 KB each
  uint64_t bar[2];
  uint64_t tbar;  // bulk-copy (TMA) completion of pre-split weight images
  uint32_t tmem_base;
  uint32_t pad;
};

// Per-CTA pipeline state (identical in every thread).
struct State {
  uint8_t* base;        // stage buffers: A [stage][hi/lo] 16 KB each, then B 32 KB each
  uint8_t* a[2][2];
  uint8_t* b[2][2];
  uint64_t* bar;
  uint32_t* tmem_slot;
  int nst;
  int cols;             // allocated TMEM columns (256, or 512 with promotion)
  uint32_t tmem;
  uint64_t* tbar;       // weight-image bulk copies
  uint32_t tph;         // bulk-copy phases consumed (thread 0)
  // commits issued / waited per stage, as scalars so the state stays in registers
  // (a stage index is a runtime value; an array indexed by it would live in local memory)
  uint32_t uses0, uses1, waited0, waited1;
  __device__ __forceinline__ void use(int s) {
    if (s) ++uses1;
    else ++uses0;
  }
  unsigned long long* prof;  // optional: thread 0 accumulates cycles per GEMM stage (ids 0..7)
  long long t_last;
  int dbg;  // microbenchmark switches (0 in production)
  // Phase clock of the GEMM internals: compiled in only for profiling builds
  // (make PHASES=1 -> -DNB_PHASE_PROF); a no-op otherwise.
  __device__ __forceinline__ void tick(int id) {
#ifdef NB_PHASE_PROF
    if (prof && threadIdx.x == 0) {
      const long long t = clock64();
      if (id >= 0) prof[id] += static_cast<unsigned long long>(t - t_last);
      t_last = t;
    }
#endif
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 "version 1").
// Rows of 128 bytes, 8-row groups 1024 bytes apart (SBO), LBO unused (1).
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(kMT >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Pre-split weight images (built once per context, model.cpp / k_weight_image): the B
// operand of a weight GEMM as it sits in the shared-memory stage, per 32-wide K chunk
// [hi | lo] of NT rows x 128 bytes, K-major SW128 (swizzle relative to a 1024-aligned
// base).  One thread moves a chunk with two 1-D bulk copies (TMA engine); no register or
// st.shared traffic for that operand.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Two 16-column loads in flight, one wait (epilogues).
__device__ __forceinline__ void tmem_ld16x2(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15}, [%16];"
      : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr + 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Byte offset of element (row, k) of a K-major SW128 tile (rows of 32 fp32).
__device__ __forceinline__ uint32_t sw128_off(int row, int k) {
  return static_cast<uint32_t>(row * 128 + ((((k >> 2) ^ (row & 7)) & 7) << 4) + ((k & 3) << 2));
}

// Allocate TMEM and initialise the barriers.  Call once per CTA, all threads.
template <int NST>
__device__ __forceinline__ void init(State& st, Smem<NST>* sm, int cols) {
  st.base = &sm->a[0][0][0];
  for (int s = 0; s < 2; ++s)
    for (int p = 0; p < 2; ++p) {
      st.a[s][p] = sm->a[s % NST][p];
      st.b[s][p] = sm->b[s % NST][p];
    }
  st.bar = sm->bar;
  st.tbar = &sm->tbar;
  st.tph = 0;
  st.tmem_slot = &sm->tmem_base;
  st.nst = NST;
  st.cols = cols;
  st.uses0 = st.uses1 = 0;
  st.waited0 = st.waited1 = 0;
  st.prof = nullptr;
  st.t_last = 0;
  st.dbg = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm->tmem_base)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    mbar_init(&sm->bar[0], 1);
    mbar_init(&sm->bar[1], 1);
    mbar_init(&sm->tbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  st.tmem = sm->tmem_base;
}

__device__ __forceinline__ void finish(State& st) {
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(st.tmem), "r"(st.cols)
                 : "memory");
}

__device__ __forceinline__ void wait_stage(State& st, int s) {
  if (s) {
    while (st.waited1 < st.uses1) {
      mbar_wait(&st.bar[1], st.waited1 & 1u);
      ++st.waited1;
    }
  } else {
    while (st.waited0 < st.uses0) {
      mbar_wait(&st.bar[0], st.waited0 & 1u);
      ++st.waited0;
    }
  }
}

__device__ __forceinline__ void st_split(uint8_t* hi, uint8_t* lo, uint32_t off, float4 v, bool two) {
  const float4 h = make_float4(tf32_rn(v.x), tf32_rn(v.y), tf32_rn(v.z), tf32_rn(v.w));
  *reinterpret_cast<float4*>(hi + off) = h;
  if (two) *reinterpret_cast<float4*>(lo + off) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

// 4 consecutive elements p[0..3] with per-element guard (count valid = nvalid).
__device__ __forceinline__ float4 ld4(const float* p, int nvalid) {
  if (nvalid >= 4) return *reinterpret_cast<const float4*>(p);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (nvalid > 0) v.x = p[0];
  if (nvalid > 1) v.y = p[1];
  if (nvalid > 2) v.z = p[2];
  return v;
}

// One 32-wide K chunk of an operand with R tile rows (R <= 256, multiple of 16), split
// into a global-load phase (into registers) and a shared-store phase, so the next chunk's
// loads can be in flight while the tensor core works on the current one.
// X(r, k) = T ? X[k*ld + r] : X[r*ld + k]; rows >= rows_total and k >= K read as zero;
// ld % 4 == 0 and a 16-byte aligned base are required.  MAXV float4 per thread:
// non-transposed R*8/256, transposed 4 * ceil(R*2/256).
template <int MAXV>
struct Frag {
  float4 v[MAXV];
};

template <bool T, int MAXV>
__device__ __forceinline__ void load_chunk(const float* __restrict__ X, int ld, int rows_total, int K, int r0,
                                           int k0, int R, Frag<MAXV>& f) {
  const int tid = threadIdx.x;
  if (!T) {
    const int nf = R * 8;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int e = tid + i * kThreads;
      f.v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < nf) {
        const int r = e >> 3, q = e & 7;
        const int gr = r0 + r, gk = k0 + 4 * q;
        if (gr < rows_total && gk < K) f.v[i] = ld4(X + static_cast<size_t>(gr) * ld + gk, K - gk);
      }
    }
  } else {
    // 4x4 blocks (4 rows x 4 k); a warp takes a tile of 8 row-quads x 4 k-quads so that
    // its loads are 128-byte rows and its swizzled 16-byte stores hit all 8 bank groups
    const int rq_n = R >> 2;
    const int tiles_r = (rq_n + 7) >> 3;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int i = 0; i < MAXV / 4; ++i) {
      const int t = warp + i * (kThreads / 32);
#pragma unroll
      for (int j = 0; j < 4; ++j) f.v[4 * i + j] = make_float4(0.f, 0.f, 0.f, 0.f);
      const int rq = 8 * (t % tiles_r) + (lane & 7), kq = 4 * (t / tiles_r) + (lane >> 3);
      if (t < 2 * tiles_r && rq < rq_n) {
        const int gr = r0 + 4 * rq;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int gk = k0 + 4 * kq + j;
          if (gk < K && gr < rows_total) f.v[4 * i + j] = ld4(X + static_cast<size_t>(gk) * ld + gr, rows_total - gr);
        }
      }
    }
  }
}

template <bool T, int MAXV>
__device__ __forceinline__ void store_chunk(int R, const Frag<MAXV>& f, uint8_t* hi, uint8_t* lo, bool two) {
  const int tid = threadIdx.x;
  if (!T) {
    const int nf = R * 8;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int e = tid + i * kThreads;
      if (e < nf) st_split(hi, lo, sw128_off(e >> 3, 4 * (e & 7)), f.v[i], two);
    }
  } else {
    const int rq_n = R >> 2;
    const int tiles_r = (rq_n + 7) >> 3;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int i = 0; i < MAXV / 4; ++i) {
      const int t = warp + i * (kThreads / 32);
      const int rq = 8 * (t % tiles_r) + (lane & 7), kq = 4 * (t / tiles_r) + (lane >> 3);
      if (t < 2 * tiles_r && rq < rq_n) {
        const float4* w = &f.v[4 * i];
        st_split(hi, lo, sw128_off(4 * rq + 0, 4 * kq), make_float4(w[0].x, w[1].x, w[2].x, w[3].x), two);
        st_split(hi, lo, sw128_off(4 * rq + 1, 4 * kq), make_float4(w[0].y, w[1].y, w[2].y, w[3].y), two);
        st_split(hi, lo, sw128_off(4 * rq + 2, 4 * kq), make_float4(w[0].z, w[1].z, w[2].z, w[3].z), two);
        st_split(hi, lo, sw128_off(4 * rq + 3, 4 * kq), make_float4(w[0].w, w[1].w, w[2].w, w[3].w), two);
      }
    }
  }
}

// gemm2: C = epi(A1 B1 + A2 B2) accumulated in one TMEM tile (K1 and K2 may differ,
// K2 = 0 for a single product); one epilogue for both products.
// EK = epilogue kind: 0 scalar functor epi(m, n, float); 1 vector functor (also called
// with float4 for 4 consecutive aligned columns); 2 tile functor, called once per column
// block by all threads with the SMEM-staged accumulator tile:
// epi(const float* stg, int ldst, int mrows, int ncols, int m_base, int n_base).
// IMG1 / IMG2: B / B2 come from pre-split weight images img1 / img2 (N <= kNT; see
// bulk_g2s) instead of being loaded and split by the threads.
template <bool TA, bool TB, bool TA2, bool TB2, int NPASS, int PROMOTE, int NST, int EK = 1, bool IMG1 = false,
          bool IMG2 = false, class Epi>
__device__ __forceinline__ void gemm2(State& st, int M, int N, int K, const float* __restrict__ A, int lda,
                                      const float* __restrict__ B, int ldb, int K2, const float* __restrict__ A2,
                                      int lda2, const float* __restrict__ B2, int ldb2, Epi epi,
                                      const uint8_t* img1 = nullptr, const uint8_t* img2 = nullptr) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr bool two = NPASS > 1;
  for (int m0 = 0; m0 < M; m0 += kMT) {
    for (int n0 = 0; n0 < N; n0 += kNT) {
      const int nrem = N - n0 < kNT ? N - n0 : kNT;
      const int NT = (nrem + 15) & ~15;
      const int nch1 = (K + kKC - 1) / kKC;
      const int nch = nch1 + (K2 + kKC - 1) / kKC;
      const uint32_t idesc = idesc_tf32(NT);
      // A: 128 rows -> 4 float4 per thread either way; B: NT <= 256 rows -> <= 8
      Frag<4> fa;
      Frag<8> fb;
      const uint32_t img_bytes = static_cast<uint32_t>(NT) * 128u;  // one of hi / lo
      auto img_of = [&](int c) -> const uint8_t* {
        if (c < nch1) return IMG1 ? img1 + static_cast<size_t>(c) * 2 * img_bytes : nullptr;
        return IMG2 ? img2 + static_cast<size_t>(c - nch1) * 2 * img_bytes : nullptr;
      };
      auto load = [&](int c) {
        if (c < nch1) {
          load_chunk<TA, 4>(A, lda, M, K, m0, c * kKC, kMT, fa);
          if (!IMG1) load_chunk<!TB, 8>(B, ldb, N, K, n0, c * kKC, NT, fb);
        } else {
          load_chunk<TA2, 4>(A2, lda2, M, K2, m0, (c - nch1) * kKC, kMT, fa);
          if (!IMG2) load_chunk<!TB2, 8>(B2, ldb2, N, K2, n0, (c - nch1) * kKC, NT, fb);
        }
      };
      st.tick(-1);
      load(0);
      st.tick(0);
      for (int c = 0; c < nch; ++c) {
        const int s = NST == 1 ? 0 : (c & 1);
        wait_stage(st, s);  // MMAs that read this stage (chunk c-NST) have completed
        st.tick(1);
        uint8_t* ah = st.a[s][0];
        uint8_t* al = st.a[s][1];
        uint8_t* bh = st.b[s][0];
        uint8_t* bl = st.b[s][1];
        const uint8_t* img = (IMG1 || IMG2) ? img_of(c) : nullptr;
        if ((IMG1 || IMG2) && img && tid == 0) {
          // weight operand: two bulk copies, overlapping the A staging below
          mbar_expect_tx(st.tbar, 2 * img_bytes);
          bulk_g2s(bh, img, img_bytes, st.tbar);
          bulk_g2s(bl, img + img_bytes, img_bytes, st.tbar);
        }
        if (c < nch1) {
          store_chunk<TA, 4>(kMT, fa, ah, al, two);
          if (!IMG1) store_chunk<!TB, 8>(NT, fb, bh, bl, two);
        } else {
          store_chunk<TA2, 4>(kMT, fa, ah, al, two);
          if (!IMG2) store_chunk<!TB2, 8>(NT, fb, bh, bl, two);
        }
        st.tick(2);
        fence_proxy_async();
        __syncthreads();
        st.tick(3);
        if (tid == 0) {
          if ((IMG1 || IMG2) && img) {
            mbar_wait(st.tbar, st.tph & 1u);
            ++st.tph;
          }
          fence_after();
          const uint32_t a0 = smem_u32(ah), a1 = smem_u32(al), b0 = smem_u32(bh), b1 = smem_u32(bl);
#pragma unroll
          for (int kk = 0; kk < kKC / 8; ++kk) {
            const uint32_t ko = kk * 32;
            const bool group_start = PROMOTE > 0 ? (c % PROMOTE == 0) : (c == 0);
            const uint32_t acc0 = (!group_start || kk > 0) ? 1u : 0u;
            mma_tf32(st.tmem, kmajor_sw128_desc(a0 + ko), kmajor_sw128_desc(b0 + ko), idesc, acc0);
            if (NPASS > 1) {
              mma_tf32(st.tmem, kmajor_sw128_desc(a0 + ko), kmajor_sw128_desc(b1 + ko), idesc, 1u);
              mma_tf32(st.tmem, kmajor_sw128_desc(a1 + ko), kmajor_sw128_desc(b0 + ko), idesc, 1u);
            }
          }
          mma_commit(&st.bar[s]);
        }
        st.tick(4);
        if (c + 1 < nch) load(c + 1);  // next chunk's global loads overlap this chunk's MMAs
        st.tick(0);
        st.use(s);
        if (PROMOTE > 0 && nch > PROMOTE && ((c + 1) % PROMOTE == 0 || c + 1 == nch)) {
          wait_stage(st, 0);
          wait_stage(st, 1);
          fence_after();
          const bool first = c + 1 <= PROMOTE;
          const int q = warp & 3;
          const int half = ((NT >> 1) + 15) & ~15;
          const int cb = (warp < 4) ? 0 : half, ce = (warp < 4) ? half : NT;
          const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
          for (int c0 = cb; c0 < ce; c0 += 16) {
            float p[16], t[16];
            tmem_ld16(st.tmem + lanes + static_cast<uint32_t>(c0), p);
            if (!first) {
              tmem_ld16(st.tmem + lanes + static_cast<uint32_t>(kSumCol + c0), t);
#pragma unroll
              for (int j = 0; j < 16; ++j) p[j] += t[j];
            }
            tmem_st16(st.tmem + lanes + static_cast<uint32_t>(kSumCol + c0), p);
          }
          fence_before();
          __syncthreads();
          fence_after();
        }
      }
      // all MMAs of this tile done (commits complete in order)
      wait_stage(st, 0);
      wait_stage(st, 1);
      fence_after();
      st.tick(5);
      const uint32_t acc_col = (PROMOTE > 0 && nch > PROMOTE) ? kSumCol : 0u;
      // ---- epilogue, in column blocks of <= 128: TMEM -> registers -> shared (row-major,
      // padded) -> coalesced epi over rows
      float* stg = reinterpret_cast<float*>(st.base);  // operand stages are free now
      const int q = warp & 3;
      const int mrows = M - m0 < kMT ? M - m0 : kMT;
      for (int cb0 = 0; cb0 < NT; cb0 += 128) {
        const int CB = NT - cb0 < 128 ? NT - cb0 : 128;  // multiple of 16
        const int ldst = CB + 4;
        const int half = ((CB >> 1) + 15) & ~15;
        const int cbeg = (warp < 4) ? 0 : half;
        const int cend = (warp < 4) ? half : CB;
        float* srow = stg + static_cast<size_t>(q * 32 + lane) * ldst;
        for (int c0 = cbeg; c0 < cend; c0 += 16) {
          float v[16];
          tmem_ld16(st.tmem + (static_cast<uint32_t>(q * 32) << 16) + acc_col + static_cast<uint32_t>(cb0 + c0), v);
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(srow + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
        fence_before();
        __syncthreads();
        st.tick(6);
        const int ncols = nrem - cb0 < CB ? nrem - cb0 : CB;
        if constexpr (EK == 2) {
          epi(stg, ldst, mrows, ncols, m0, n0 + cb0);
        } else if constexpr (EK == 1) {
          // float4 per thread, rows r = warp, warp+8, ... four rows per batch in flight
          const int nq = ncols >> 2;
          for (int r = warp; r < mrows; r += 4 * (kThreads / 32))
            for (int qd = lane; qd < nq; qd += 32) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int rr = r + u * (kThreads / 32);
                if (rr < mrows)
                  epi(m0 + rr, n0 + cb0 + 4 * qd, *reinterpret_cast<const float4*>(stg + static_cast<size_t>(rr) * ldst + 4 * qd));
              }
            }
          for (int e = threadIdx.x; e < mrows * (ncols - 4 * nq); e += kThreads) {
            const int rr = e / (ncols - 4 * nq), cc = 4 * nq + e % (ncols - 4 * nq);
            epi(m0 + rr, n0 + cb0 + cc, stg[static_cast<size_t>(rr) * ldst + cc]);
          }
        } else {
          for (int r = warp; r < mrows; r += 4 * (kThreads / 32))
            for (int n = lane; n < ncols; n += 32) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int rr = r + u * (kThreads / 32);
                if (rr < mrows) epi(m0 + rr, n0 + cb0 + n, stg[static_cast<size_t>(rr) * ldst + n]);
              }
            }
        }
        __syncthreads();
        st.tick(7);
      }
      fence_after();
    }
  }
}

// ---------------------------------------------------------------------------------------
// TS-mode block GEMM: the A operand lives in TMEM, B in shared memory.
//
// Per 32-wide K chunk every thread loads 16 values of ONE A row (warp w: rows
// 32*(w%4)+lane, k = 16*(w/4)..+15 of the chunk), splits hi/lo and writes them straight
// into its TMEM lanes with tcgen05.st (no shared-memory traffic for A, and the MMA reads
// no A bytes from shared memory); B is split into the swizzled smem stage as in gemm2.
// Two stages (TMEM A + smem B, 32 KB per B stage): chunk c+1 is staged while the tensor
// core works on chunk c.  TMEM map (256 columns): [0,128) accumulator, [128+64s, +32) A hi
// and [160+64s, +32) A lo of stage s.  N is processed in 128-column tiles.
// ---------------------------------------------------------------------------------------
constexpr int kTsN = 128;
constexpr uint32_t kTsA = 128;

__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st16_nowait(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}

// 16 values A(r, k0..k0+15) of one row (zero outside [0,M) x [0,K)).
template <bool T>
__device__ __forceinline__ void load_arow(const float* __restrict__ A, int lda, int M, int K, int r, int k0,
                                          float (&v)[16]) {
  if (!T) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = k0 + 4 * q;
      float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < M && k < K) f = ld4(A + static_cast<size_t>(r) * lda + k, K - k);
      v[4 * q] = f.x;
      v[4 * q + 1] = f.y;
      v[4 * q + 2] = f.z;
      v[4 * q + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k = k0 + j;
      v[j] = (r < M && k < K) ? A[static_cast<size_t>(k) * lda + r] : 0.f;
    }
  }
}

// DYNA: A's transposition is the runtime flag ta_dyn instead of TA (one code copy serves
// both orientations: call sites that differ only in it share their instructions).
template <bool TA, bool TB, bool TA2, bool TB2, int NPASS, int EK = 1, bool IMG1 = false, bool IMG2 = false,
          class Epi, bool DYNA = false>
__device__ __forceinline__ void gemm2_ts(State& st, int M, int N, int K, const float* __restrict__ A, int lda,
                                         const float* __restrict__ B, int ldb, int K2, const float* __restrict__ A2,
                                         int lda2, const float* __restrict__ B2, int ldb2, Epi epi,
                                         const uint8_t* img1 = nullptr, const uint8_t* img2 = nullptr,
                                         bool ta_dyn = false) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr bool two = NPASS > 1;
  uint8_t* base = st.base;
  const uint32_t lanes = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  const int arow = 32 * (warp & 3) + lane;
  const int akof = 16 * (warp >> 2);
  for (int m0 = 0; m0 < M; m0 += kMT) {
    for (int n0 = 0; n0 < N; n0 += kTsN) {
      const int nrem = N - n0 < kTsN ? N - n0 : kTsN;
      const int NT = (nrem + 15) & ~15;
      const int nch1 = (K + kKC - 1) / kKC;
      const int nch = nch1 + (K2 + kKC - 1) / kKC;
      const uint32_t idesc = idesc_tf32(NT);
      float av[16];
      Frag<4> fb;
      const uint32_t img_bytes = static_cast<uint32_t>(NT) * 128u;
      auto img_of = [&](int c) -> const uint8_t* {
        if (c < nch1) return IMG1 ? img1 + static_cast<size_t>(c) * 2 * img_bytes : nullptr;
        return IMG2 ? img2 + static_cast<size_t>(c - nch1) * 2 * img_bytes : nullptr;
      };
      auto load = [&](int c) {
        if (c < nch1) {
          if constexpr (DYNA) {
            if (ta_dyn) load_arow<true>(A, lda, M, K, m0 + arow, c * kKC + akof, av);
            else load_arow<false>(A, lda, M, K, m0 + arow, c * kKC + akof, av);
          } else {
            load_arow<TA>(A, lda, M, K, m0 + arow, c * kKC + akof, av);
          }
          if (!IMG1) load_chunk<!TB, 4>(B, ldb, N, K, n0, c * kKC, NT, fb);
        } else {
          load_arow<TA2>(A2, lda2, M, K2, m0 + arow, (c - nch1) * kKC + akof, av);
          if (!IMG2) load_chunk<!TB2, 4>(B2, ldb2, N, K2, n0, (c - nch1) * kKC, NT, fb);
        }
      };
      st.tick(-1);
      load(0);
      st.tick(0);
      for (int c = 0; c < nch; ++c) {
        const int s = c & 1;
        wait_stage(st, s);  // MMAs of chunk c-2 (same TMEM A / smem B stage) have completed
        st.tick(1);
        {
          float hi[16], lo[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            hi[j] = tf32_rn(av[j]);
            lo[j] = av[j] - hi[j];
          }
          const uint32_t ta = st.tmem + lanes + kTsA + 64u * s + static_cast<uint32_t>(akof);
          tmem_st16_nowait(ta, hi);
          if (two) tmem_st16_nowait(ta + 32, lo);
        }
        uint8_t* bh = base + 32768 * s;
        uint8_t* bl = bh + 16384;
        const uint8_t* img = (IMG1 || IMG2) ? img_of(c) : nullptr;
        if ((IMG1 || IMG2) && img) {
          if (tid == 0) {
            mbar_expect_tx(st.tbar, 2 * img_bytes);
            bulk_g2s(bh, img, img_bytes, st.tbar);
            bulk_g2s(bl, img + img_bytes, img_bytes, st.tbar);
          }
        } else if (c < nch1) {
          store_chunk<!TB, 4>(NT, fb, bh, bl, two);
        } else {
          store_chunk<!TB2, 4>(NT, fb, bh, bl, two);
        }
        // the next chunk's global loads go out before the barrier (the stores above have
        // already taken their source registers)
        if (c + 1 < nch) load(c + 1);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        st.tick(2);
        fence_before();
        if (!((IMG1 || IMG2) && img)) fence_proxy_async();  // B staged by st.shared this chunk
        __syncthreads();
        st.tick(3);
        if (tid == 0) {
          if ((IMG1 || IMG2) && img) {
            mbar_wait(st.tbar, st.tph & 1u);
            ++st.tph;
          }
          fence_after();
          const uint32_t ah = st.tmem + kTsA + 64u * s, al = ah + 32;
          const uint32_t b0 = smem_u32(bh), b1 = smem_u32(bl);
#pragma unroll
          for (int kk = 0; kk < kKC / 8; ++kk) {
            const uint32_t acc0 = (c > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ts(st.tmem, ah + 8 * kk, kmajor_sw128_desc(b0 + 32 * kk), idesc, acc0);
            if (NPASS > 1) {
              mma_tf32_ts(st.tmem, ah + 8 * kk, kmajor_sw128_desc(b1 + 32 * kk), idesc, 1u);
              mma_tf32_ts(st.tmem, al + 8 * kk, kmajor_sw128_desc(b0 + 32 * kk), idesc, 1u);
            }
          }
          mma_commit(&st.bar[s]);
        }
        st.use(s);
        st.tick(4);
      }
      wait_stage(st, 0);
      wait_stage(st, 1);
      fence_after();
      st.tick(5);
      // ---- epilogue (accumulator columns [0, NT)): TMEM -> registers -> shared (row-major,
      // padded) -> coalesced epi over rows; the B stages are free now
      float* stg = reinterpret_cast<float*>(base);
      const int q = warp & 3;
      const int mrows = M - m0 < kMT ? M - m0 : kMT;
      const int CB = NT;
      const int ldst = CB + 4;
      const int half = ((CB >> 1) + 15) & ~15;
      const int cbeg = (warp < 4) ? 0 : half;
      const int cend = (warp < 4) ? half : CB;
      float* srow = stg + static_cast<size_t>(q * 32 + lane) * ldst;
      int c0 = cbeg;
      for (; c0 + 32 <= cend; c0 += 32) {
        float v[32];
        tmem_ld16x2(st.tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), v);
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(srow + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      for (; c0 < cend; c0 += 16) {
        float v[16];
        tmem_ld16(st.tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0), v);
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(srow + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      fence_before();
      __syncthreads();
      st.tick(6);
      const int ncols = nrem;
      if constexpr (EK == 2) {
        epi(stg, ldst, mrows, ncols, m0, n0);
      } else if constexpr (EK == 1) {
        const int nq = ncols >> 2;
        for (int r = warp; r < mrows; r += 4 * (kThreads / 32))
          for (int qd = lane; qd < nq; qd += 32) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int rr = r + u * (kThreads / 32);
              if (rr < mrows)
                epi(m0 + rr, n0 + 4 * qd, *reinterpret_cast<const float4*>(stg + static_cast<size_t>(rr) * ldst + 4 * qd));
            }
          }
        for (int e = threadIdx.x; e < mrows * (ncols - 4 * nq); e += kThreads) {
          const int rr = e / (ncols - 4 * nq), cc = 4 * nq + e % (ncols - 4 * nq);
          epi(m0 + rr, n0 + cc, stg[static_cast<size_t>(rr) * ldst + cc]);
        }
      } else {
        for (int r = warp; r < mrows; r += 4 * (kThreads / 32))
          for (int n = lane; n < ncols; n += 32) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int rr = r + u * (kThreads / 32);
              if (rr < mrows) epi(m0 + rr, n0 + n, stg[static_cast<size_t>(rr) * ldst + n]);
            }
          }
      }
      __syncthreads();
      st.tick(7);
      fence_after();
    }
  }
}

template <bool TA, bool TB, int NPASS, int EK = 1, bool IMG = false, class Epi>
__device__ __forceinline__ void gemm_ts(State& st, int M, int N, int K, const float* __restrict__ A, int lda,
                                        const float* __restrict__ B, int ldb, Epi epi, const uint8_t* img = nullptr) {
  gemm2_ts<TA, TB, TA, TB, NPASS, EK, IMG, false>(st, M, N, K, A, lda, B, ldb, 0, A, lda, B, ldb, epi, img);
}

template <bool TA, bool TB, int NPASS, int PROMOTE = 0, int NST = 2, int EK = 1, bool IMG = false, class Epi>
__device__ __forceinline__ void gemm(State& st, int M, int N, int K, const float* __restrict__ A, int lda,
                                     const float* __restrict__ B, int ldb, Epi epi, const uint8_t* img = nullptr) {
  gemm2<TA, TB, TA, TB, NPASS, PROMOTE, NST, EK, IMG, false>(st, M, N, K, A, lda, B, ldb, 0, A, lda, B, ldb, epi, img);
}

}  // namespace tc
}  // namespace nb
