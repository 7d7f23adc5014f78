// Domain-decomposition build, cell-list neighbour search and deterministic force
// assembly (HBM/L2-bound integer + FP64 kernels).
//
// Reference algorithm: decomp.cpp:59-131 (ownership, halo), decomp.cpp:312-416 (members,
// centres, per-centre scan, canonical sort, capacity), deeppot.cpp:141-148 (sort key),
// deeppot.cpp:271-309 / decomp.cpp:421-538 (force assembly and ghost-force routing).
#include <atomic>
#include <climits>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace nb {

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

// ----------------------------------------------------------------------------------
// Ownership (owner_rank_of, decomp.cpp:59-68) + input validation
// (neighbor.cpp:22-30 wrapped positions; deeppot.cpp:327-328 species range)
// ----------------------------------------------------------------------------------
__global__ void k_owner(SysArgs s, int dx, int dy, int dz, int* __restrict__ owner,
                        int* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  const int dims[3] = {dx, dy, dz};
  int c[3];
  bool bad = s.species[i] < 0 || s.species[i] >= s.n_species;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double x = s.pos[3 * i + a];
    if (s.per[a] && !(x >= 0.0 && x < s.L[a])) bad = true;
    const double edge = s.L[a] / dims[a];
    int k = static_cast<int>(floor(x / edge));
    c[a] = min(max(k, 0), dims[a] - 1);
  }
  owner[i] = (c[0] * dims[1] + c[1]) * dims[2] + c[2];
  if (bad) atomicMin(&err[0], i);
}

__global__ void k_negate(const int* __restrict__ src, int* __restrict__ dst, int n) {
  const int i = threadIdx.x;
  if (i < n) dst[i] = -src[i];
}

void launch_negate(const int* src, int* dst, int n, cudaStream_t st) {
  k_negate<<<1, 32, 0, st>>>(src, dst, n); count_launch();
}

void launch_owner(const SysArgs& s, const int dims[3], int* owner, int* err, cudaStream_t st) {
  if (s.n == 0) return;
  k_owner<<<(s.n + 255) / 256, 256, 0, st>>>(s, dims[0], dims[1], dims[2], owner, err); count_launch();
}

// ----------------------------------------------------------------------------------
// Halo slab test (build_halo, decomp.cpp:96-131): for every atom x 27 images,
// q = p + k*L (FP64, no contraction) inside [slab_lo, slab_hi), own atoms excluded at
// zero shift.  Pass 1 counts per atom; pass 2 writes members in (atom, shift) order.
// ----------------------------------------------------------------------------------
__device__ __forceinline__ bool in_slab(const double* q, const double* lo, const double* hi) {
  return q[0] >= lo[0] && q[0] < hi[0] && q[1] >= lo[1] && q[1] < hi[1] && q[2] >= lo[2] &&
         q[2] < hi[2];
}

__global__ void k_dd_flags(SysArgs s, RankArgs r, const int* __restrict__ owner,
                           int* __restrict__ is_local, int* __restrict__ gcount) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  const double p[3] = {s.pos[3 * i], s.pos[3 * i + 1], s.pos[3 * i + 2]};
  const bool mine = owner[i] == r.rank;
  int cnt = 0;
  const int sx = s.per[0], sy = s.per[1], sz = s.per[2];
  for (int kx = -sx; kx <= sx; ++kx)
    for (int ky = -sy; ky <= sy; ++ky)
      for (int kz = -sz; kz <= sz; ++kz) {
        if (kx == 0 && ky == 0 && kz == 0 && mine) continue;
        const double q[3] = {__dadd_rn(p[0], __dmul_rn(static_cast<double>(kx), s.L[0])),
                             __dadd_rn(p[1], __dmul_rn(static_cast<double>(ky), s.L[1])),
                             __dadd_rn(p[2], __dmul_rn(static_cast<double>(kz), s.L[2]))};
        cnt += in_slab(q, r.slab_lo, r.slab_hi);
      }
  is_local[i] = mine;
  gcount[i] = cnt;
}

void launch_dd_flags(const SysArgs& s, const RankArgs& r, const int* owner, int* is_local,
                     int* gcount, cudaStream_t st) {
  if (s.n == 0) return;
  k_dd_flags<<<(s.n + 255) / 256, 256, 0, st>>>(s, r, owner, is_local, gcount); count_launch();
}

// Single-CTA exclusive scan (n up to a few 1e5; one launch, no host round trip).  Each
// thread takes 4 consecutive elements per pass (one 16-byte load when aligned), so a pass
// covers 4096 elements: a 28k-element scan is 7 passes of (local prefix, warp shuffle
// scan, block scan of the warp totals).
__global__ void __launch_bounds__(1024) k_scan(const int* __restrict__ in, int* __restrict__ out,
                                               int n, const int* __restrict__ n_dev) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (n_dev) n = *n_dev;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  for (int base = 0; base < n; base += 4096) {
    const int i0 = base + 4 * threadIdx.x;
    int v[4];
    if (vec && i0 + 3 < n) {
      const int4 q = *reinterpret_cast<const int4*>(in + i0);
      v[0] = q.x;
      v[1] = q.y;
      v[2] = q.z;
      v[3] = q.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = i0 + u < n ? in[i0 + u] : 0;
    }
    const int tsum = v[0] + v[1] + v[2] + v[3];
    int x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    int run = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + x - tsum;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + u < n) out[i0 + u] = run;
      run += v[u];
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = run;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

void launch_scan(const int* in, int* out, int n, cudaStream_t st) {
  k_scan<<<1, 1024, 0, st>>>(in, out, n, nullptr); count_launch();
}

void launch_scan_dev(const int* in, int* out, const int* n_dev, cudaStream_t st) {
  k_scan<<<1, 1024, 0, st>>>(in, out, 0, n_dev); count_launch();
}

// Members: locals first (ascending atom, shift 0), then ghosts in (atom, shift) order.
__global__ void k_dd_members(SysArgs s, RankArgs r, const int* __restrict__ owner,
                             const int* __restrict__ loc_off, const int* __restrict__ gh_off,
                             int n_atoms, int cap, int* __restrict__ m_atom, int* __restrict__ m_shift,
                             double* __restrict__ m_pos, int* __restrict__ m_owner) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  const int nloc = loc_off[n_atoms];
  const double p[3] = {s.pos[3 * i], s.pos[3 * i + 1], s.pos[3 * i + 2]};
  const bool mine = owner[i] == r.rank;
  if (mine && loc_off[i] < cap) {
    const int m = loc_off[i];
    m_atom[m] = i;
    m_shift[m] = kZeroShift;
    m_owner[m] = r.rank;
    for (int a = 0; a < 3; ++a) m_pos[3 * m + a] = p[a];
  }
  int m = nloc + gh_off[i];
  const int sx = s.per[0], sy = s.per[1], sz = s.per[2];
  for (int kx = -sx; kx <= sx; ++kx)
    for (int ky = -sy; ky <= sy; ++ky)
      for (int kz = -sz; kz <= sz; ++kz) {
        if (kx == 0 && ky == 0 && kz == 0 && mine) continue;
        const double q[3] = {__dadd_rn(p[0], __dmul_rn(static_cast<double>(kx), s.L[0])),
                             __dadd_rn(p[1], __dmul_rn(static_cast<double>(ky), s.L[1])),
                             __dadd_rn(p[2], __dmul_rn(static_cast<double>(kz), s.L[2]))};
        if (!in_slab(q, r.slab_lo, r.slab_hi)) continue;
        if (m >= cap) continue;  // capacity overflow: reported by k_rank_counts, step redone
        m_atom[m] = i;
        m_shift[m] = pack_shift(kx, ky, kz);
        m_owner[m] = owner[i];
        for (int a = 0; a < 3; ++a) m_pos[3 * m + a] = q[a];
        ++m;
      }
}

void launch_dd_members(const SysArgs& s, const RankArgs& r, const int* owner, const int* loc_off,
                       const int* gh_off, int n_atoms, int cap_members, int* m_atom, int* m_shift,
                       double* m_pos, int* m_owner, cudaStream_t st) {
  if (s.n == 0) return;
  k_dd_members<<<(s.n + 255) / 256, 256, 0, st>>>(s, r, owner, loc_off, gh_off, n_atoms, cap_members, m_atom,
                                                  m_shift, m_pos, m_owner); count_launch();
}

__global__ void k_rank_counts(const int* __restrict__ loc_off, const int* __restrict__ gh_off, int n, int cap_loc,
                              int cap_gh, int* __restrict__ counts, int* __restrict__ overflow) {
  const int nloc = loc_off[n], ngh = gh_off[n];
  const int lo = min(nloc, cap_loc), gh = min(ngh, cap_gh);
  if (lo < nloc || gh < ngh) *overflow = 1;
  counts[kCntLoc] = lo;
  counts[kCntGh] = gh;
  counts[kCntMem] = lo + gh;
  counts[kCntCen] = lo;
  counts[kCntRoute] = 0;
  counts[kCntGhExact] = ngh;
  counts[kCntCenExact] = nloc;
  counts[kCntLocExact] = nloc;
}

void launch_rank_counts(const int* loc_off, const int* gh_off, int n_atoms, int cap_locals, int cap_ghosts,
                        int* counts, int* overflow, cudaStream_t st) {
  k_rank_counts<<<1, 1, 0, st>>>(loc_off, gh_off, n_atoms, cap_locals, cap_ghosts, counts, overflow); count_launch();
}

// Centres: every local; for wide_halo also the first-layer ghosts (inside the rc slab,
// decomp.cpp:317-326).
__global__ void k_centre_flags(RankArgs r, const int* __restrict__ counts,
                               const double* __restrict__ m_pos, int cap, int* __restrict__ flag) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int nloc = counts[0], nm = counts[0] + counts[1];
  if (m >= cap) return;
  int f = 0;
  if (m < nloc) f = 1;
  else if (m < nm && r.wide) f = in_slab(m_pos + 3 * m, r.rc_lo, r.rc_hi);
  flag[m] = f;
}

void launch_centre_flags(const RankArgs& r, const int* counts, const double* m_pos,
                         int n_members_cap, int* flag, cudaStream_t st) {
  if (n_members_cap == 0) return;
  k_centre_flags<<<(n_members_cap + 255) / 256, 256, 0, st>>>(r, counts, m_pos, n_members_cap, flag); count_launch();
}

__global__ void k_centre_compact(const int* __restrict__ flag, const int* __restrict__ off,
                                 int* __restrict__ counts, int wide, int cap_cen, int* __restrict__ cen_member,
                                 int* __restrict__ cidx, int* __restrict__ overflow) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = counts[kCntMem];
  if (m == 0 && wide) {
    const int nc = off[n];
    counts[kCntCenExact] = nc;
    counts[kCntCen] = min(nc, cap_cen);
    if (nc > cap_cen) *overflow = 1;
  }
  if (m >= n) return;
  if (flag[m] && off[m] < cap_cen) {
    cen_member[off[m]] = m;
    cidx[m] = off[m];
  } else {
    cidx[m] = -1;
  }
}

void launch_centre_compact(const int* flag, const int* off, int* counts, int n_members_cap, int wide,
                           int cap_centres, int* cen_member, int* cidx, int* overflow, cudaStream_t st) {
  if (n_members_cap == 0) return;
  k_centre_compact<<<(n_members_cap + 255) / 256, 256, 0, st>>>(flag, off, counts, wide, cap_centres, cen_member,
                                                                cidx, overflow);
  count_launch();
}

// ----------------------------------------------------------------------------------
// Cell grid over the materialised member images.  Width >= rc on every axis, so the
// 27-cell stencil is complete; positions outside the grid clamp into the boundary
// cells (adjacency preserved).  The grid only selects candidates: rows are then sorted
// by the unique canonical key, so the result is independent of the grid geometry.
// ----------------------------------------------------------------------------------
__device__ __forceinline__ int cell_of(const CellArgs& c, const double* q) {
  int id[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int k = static_cast<int>(floor((q[a] - c.origin[a]) / c.width[a]));
    id[a] = min(max(k, 0), c.dims[a] - 1);
  }
  return (id[0] * c.dims[1] + id[1]) * c.dims[2] + id[2];
}

__global__ void k_cell_count(CellArgs c, const double* __restrict__ m_pos, const int* __restrict__ n_dev,
                             int* __restrict__ m_cell, int* __restrict__ count) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= *n_dev) return;
  const int id = cell_of(c, m_pos + 3 * m);
  m_cell[m] = id;
  atomicAdd(&count[id], 1);
}

void launch_cell_count(const CellArgs& c, const double* m_pos, const int* n_dev, int n_cap, int* m_cell,
                       int* count, cudaStream_t st) {
  if (n_cap == 0) return;
  k_cell_count<<<(n_cap + 255) / 256, 256, 0, st>>>(c, m_pos, n_dev, m_cell, count); count_launch();
}

// Fill the cell lists and a cell-ordered copy of what the neighbour scan reads per
// candidate (atom position, packed shift, species, gid), so that scan's loads are
// contiguous across a warp instead of chasing member -> atom indirections.  The order
// inside a cell is arbitrary: rows are sorted by the canonical key afterwards.
__global__ void k_cell_fill(const int* __restrict__ m_cell, const int* __restrict__ n_dev,
                            const int* __restrict__ start, int* __restrict__ fill, int* __restrict__ members,
                            CellSorted cs) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= *n_dev) return;
  const int id = m_cell[m];
  const int slot = atomicAdd(&fill[id], 1);
  const int j = start[id] + slot;
  members[j] = m;
  const int aj = cs.m_atom[m];
  cs.x[j] = cs.pos[3 * aj];
  cs.y[j] = cs.pos[3 * aj + 1];
  cs.z[j] = cs.pos[3 * aj + 2];
  cs.shift[j] = cs.m_shift[m];
  cs.species[j] = min(max(cs.atom_species[aj], 0), cs.n_species - 1);
  cs.gid[j] = cs.atom_gid[aj];
}

void launch_cell_fill(const int* m_cell, const int* n_dev, int n_cap, const int* start, int* fill, int* members,
                      const CellSorted& cs, cudaStream_t st) {
  if (n_cap == 0) return;
  k_cell_fill<<<(n_cap + 255) / 256, 256, 0, st>>>(m_cell, n_dev, start, fill, members, cs); count_launch();
}

// ----------------------------------------------------------------------------------
// Neighbour rows: one warp per list owner (centre, or ghost target for reverse lists).
// 27-cell stencil; candidate kept iff norm2(image_delta(...)) < rc^2 with the exact
// FP64 expression of decomp.cpp:393-409 (rel shift = member shift - centre shift);
// warp-ballot compaction into shared memory; canonical order (species, r^2, gid) by
// rank sort (keys are unique); overflow (> n_max) recorded, never truncated.
// ----------------------------------------------------------------------------------
constexpr int kNbrWarps = 4;

// 16-byte shared-memory entry per kept candidate (small entries keep more warps resident:
// the kernel is latency-bound).  j = candidate index in the cell-ordered arrays (member,
// gid, position and shift are re-read from there when needed).
struct NbrEntry {
  uint64_t key;  // (species << 58) | (bits(r2) - kbase): same order as (species, r2)
  int j;
  int species;
};

// Image delta centre -> candidate j, exactly as the distance test formed it.
__device__ __forceinline__ void cand_delta(const NbrArgs& a, int j, const double (&pc)[3], const int (&csh)[3],
                                           double (&d)[3]) {
  const int sj = a.cs.shift[j];
  d[0] = image_delta(a.cs.x[j], pc[0], shift_x(sj) - csh[0], a.L[0]);
  d[1] = image_delta(a.cs.y[j], pc[1], shift_y(sj) - csh[1], a.L[1]);
  d[2] = image_delta(a.cs.z[j], pc[2], shift_z(sj) - csh[2], a.L[2]);
}

// Full canonical order (species, r2, gid) of deeppot.cpp:141-148 with r2 recomputed and the
// gid loaded: for lists with an exact key tie or a key that does not pack (rare).
__device__ __forceinline__ bool full_less(const NbrArgs& a, const NbrEntry& x, const NbrEntry& y,
                                          const double (&pc)[3], const int (&csh)[3]) {
  if (x.species != y.species) return x.species < y.species;
  double dx[3], dy[3];
  cand_delta(a, x.j, pc, csh, dx);
  cand_delta(a, y.j, pc, csh, dy);
  const double rx = norm2_exact(dx[0], dx[1], dx[2]), ry = norm2_exact(dy[0], dy[1], dy[2]);
  if (rx != ry) return rx < ry;
  return a.cs.gid[x.j] < a.cs.gid[y.j];
}

// Environment matrix of one canonical row (prepare_rows + switch_eval, dp_core.hpp:116-137,
// 200-223), fused into the centre-list build: the image delta re-formed as the distance
// test formed it, r and s(r) in exact FP64, env row R = (s, s/r d) as one 16-byte store,
// the neighbour's species; returns s^2 for sigma.
__device__ __forceinline__ double env_row(const NbrArgs& a, int li, int k, const NbrEntry& e, const double (&pc)[3],
                                          const int (&csh)[3]) {
  double d[3];
  cand_delta(a, e.j, pc, csh, d);
  const double r = sqrt(norm2_exact(d[0], d[1], d[2]));
  double sw, ds;
  switch_fn(r, a.rcs, a.rc, sw, ds);
  const double sr = sw / r;
  const size_t o = static_cast<size_t>(li) * a.n_max + k;
  a.R[o] = make_float4(static_cast<float>(sw), static_cast<float>(sr * d[0]), static_cast<float>(sr * d[1]),
                       static_cast<float>(sr * d[2]));
  a.Z[o] = e.species;
  return sw * sw;
}

// sigma = sum_k s_k^2 in canonical row order (lane l adds rows l, l + 32, ..., then a fixed
// warp tree): independent of the order candidates reached the list, so bit-reproducible
// (the cell lists are filled with atomics) and equal to a row-by-row evaluation.
__device__ __forceinline__ void env_sigma(const NbrArgs& a, int li, int cnt, const double* sr) {
  const int lane = threadIdx.x & 31;
  double sig = 0.0;
  for (int k = lane; k < cnt; k += 32) sig += sr[k];
  sig = warp_sum(sig);
  if (lane == 0) a.sig[li] = sig;
}

// rank[u] = number of keys below mine[u] (u < NU; NU warp-uniform, so no per-u guards)
template <int NU>
__device__ __forceinline__ void rank_packed(const NbrEntry* buf, int cnt, const uint64_t (&mine)[6], int (&rank)[6]) {
  for (int j = 0; j < cnt; ++j) {
    const uint64_t o = buf[j].key;
#pragma unroll
    for (int u = 0; u < NU; ++u) rank[u] += o < mine[u];
  }
}

// ENV: centre lists, which also write their environment rows (env_row).
template <bool ENV>
__global__ void __launch_bounds__(kNbrWarps * 32) k_neighbors(NbrArgs a, int cap) {
  extern __shared__ __align__(16) unsigned char nbr_smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  NbrEntry* buf = reinterpret_cast<NbrEntry*>(nbr_smem_raw) + static_cast<size_t>(wid) * cap;
  const int li = blockIdx.x * kNbrWarps + wid;
  if (li >= (a.n_lists_dev ? *a.n_lists_dev : a.n_lists)) return;
  const int cm = a.centre_member ? a.centre_member[li]
                                 : li + (a.member_offset_dev ? *a.member_offset_dev : a.member_offset);
  const int ca = a.m_atom[cm];
  const int cs = a.m_shift[cm];
  const double pc[3] = {a.pos[3 * ca], a.pos[3 * ca + 1], a.pos[3 * ca + 2]};
  const int csh[3] = {shift_x(cs), shift_y(cs), shift_z(cs)};
  const int cell = a.m_cell[cm];
  const int cz = cell % a.cdims[2], cy = (cell / a.cdims[2]) % a.cdims[1],
            cx = cell / (a.cdims[1] * a.cdims[2]);
  const int cand_limit = a.cand_limit_dev ? *a.cand_limit_dev : a.cand_limit;
  int cnt = 0;
  bool packable = true;  // every kept key fits the 64-bit packing (per lane)
  // The stencil's z-adjacent cells are consecutive cell ids, so their members are one
  // contiguous range of the cell-ordered arrays: 9 ranges (one per (x, y) column) instead of
  // 27 cells, scanned as ONE stream of candidates in warp-wide batches (no partly empty
  // batch per cell).  The order candidates arrive in does not matter: rows are ranked by
  // the canonical key below.
  // range q = column (ox, oy) = (q / 3 - 1, q % 3 - 1) covers stream positions
  // [re[q - 1], re[q]) and candidate j = t + dl[q] there; fully unrolled so both arrays stay
  // in registers (empty for a column outside the grid)
  int re[9], dl[9];
  int total = 0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int x = cx + q / 3 - 1, y = cy + q % 3 - 1;
    int b = 0, len = 0;
    if (x >= 0 && x < a.cdims[0] && y >= 0 && y < a.cdims[1]) {
      const int col = (x * a.cdims[1] + y) * a.cdims[2];
      b = a.cell_start[col + max(cz - 1, 0)];
      len = a.cell_start[col + min(cz + 1, a.cdims[2] - 1) + 1] - b;
    }
    dl[q] = b - total;
    total += len;
    re[q] = total;
  }
  // Two warp-wide batches per iteration, every load of a candidate issued before any test
  // (the kernel is bound by the latency of these L2 reads, not by their bytes)
  for (int base = 0; base < total; base += 64) {
    int jj[2];
    int mj[2], sj[2], sp[2];
    double cx_[2], cy_[2], cz_[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = base + 32 * h + lane;
      jj[h] = -1;
      if (t < total) {
        int dj = dl[0];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (t >= re[q]) dj = dl[q + 1];
        const int j = t + dj;
        jj[h] = j;
        mj[h] = a.cell_members[j];
        cx_[h] = a.cs.x[j];
        cy_[h] = a.cs.y[j];
        cz_[h] = a.cs.z[j];
        sj[h] = a.cs.shift[j];
        sp[h] = a.cs.species[j];
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      bool keep = false;
      NbrEntry ent;
      if (jj[h] >= 0 && mj[h] != cm && mj[h] < cand_limit) {
        const double d0 = image_delta(cx_[h], pc[0], shift_x(sj[h]) - csh[0], a.L[0]);
        const double d1 = image_delta(cy_[h], pc[1], shift_y(sj[h]) - csh[1], a.L[1]);
        const double d2 = image_delta(cz_[h], pc[2], shift_z(sj[h]) - csh[2], a.L[2]);
        const double r2 = norm2_exact(d0, d1, d2);
        if (r2 < a.rc2) {
          keep = true;
          ent.j = jj[h];
          ent.species = sp[h];
          const uint64_t rbits = static_cast<uint64_t>(__double_as_longlong(r2));
          const bool ok = rbits >= a.kbase && ent.species >= 0 && ent.species < 63;
          packable = packable && ok;
          ent.key = (static_cast<uint64_t>(ent.species) << 58) | (rbits - a.kbase);
        }
      }
      const unsigned mask = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int slot = cnt + __popc(mask & ((1u << lane) - 1u));
        if (slot < cap) buf[slot] = ent;
      }
      cnt += __popc(mask);
    }
  }
  __syncwarp();
  if (lane == 0) {
    a.nn[li] = cnt > a.n_max ? 0 : cnt;  // overflow: reported, list left empty
    if (a.nonempty && cnt > 0) atomicAdd(a.nonempty, 1);
    if (a.maxn) atomicMax(a.maxn, cnt);
  }
  if (cnt > a.n_max) {
    if (lane == 0) atomicMin(a.err, ca);
    return;
  }
  // rank sort on the unique key: each lane ranks its (up to kPer) entries against one
  // broadcast read of every entry, so the shared-memory sweep is done once per warp
  // instead of once per entry.  Fast path: one 64-bit compare of the packed (species, r2)
  // key per pair; a list with equal keys (an exact r2 tie within a species) or a key that
  // does not pack takes the full (species, r2, gid) comparison.
  int* out = a.nlist + static_cast<size_t>(li) * a.n_max;
  constexpr int kPer = 6;  // lanes own entries lane, lane + 32, ... (n_max <= 192)
  if (cnt <= 32 * kPer) {
    uint64_t mine[kPer];
    int rank[kPer];
    const int nu = (cnt + 31) >> 5;  // warp-uniform
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      rank[u] = 0;
      mine[u] = lane + 32 * u < cnt ? buf[lane + 32 * u].key : ~0ull;
    }
    bool fast = __all_sync(0xffffffffu, packable);
    if (fast) {
      switch (nu) {
        case 1: rank_packed<1>(buf, cnt, mine, rank); break;
        case 2: rank_packed<2>(buf, cnt, mine, rank); break;
        case 3: rank_packed<3>(buf, cnt, mine, rank); break;
        case 4: rank_packed<4>(buf, cnt, mine, rank); break;
        case 5: rank_packed<5>(buf, cnt, mine, rank); break;
        default: rank_packed<6>(buf, cnt, mine, rank); break;
      }
      // distinct keys give a permutation; an exact key tie gives two entries one rank, so
      // one of them reads back another entry's tag
      int* tag = reinterpret_cast<int*>(nbr_smem_raw + static_cast<size_t>(kNbrWarps) * cap * sizeof(NbrEntry)) +
                 static_cast<size_t>(wid) * cap;
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (lane + 32 * u < cnt) tag[rank[u]] = lane + 32 * u;
      __syncwarp();
      bool ok = true;
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (lane + 32 * u < cnt) ok = ok && tag[rank[u]] == lane + 32 * u;
      fast = __all_sync(0xffffffffu, ok);
    }
    if (!fast) {
      for (int u = 0; u < nu; ++u) {
        if (lane + 32 * u >= cnt) continue;
        const NbrEntry me = buf[lane + 32 * u];
        int r = 0;
        for (int j = 0; j < cnt; ++j) r += full_less(a, buf[j], me, pc, csh);
        rank[u] = r;
      }
    }
    double s2[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u)
      if (lane + 32 * u < cnt) {
        const NbrEntry me = buf[lane + 32 * u];
        out[rank[u]] = a.cell_members[me.j];
        if constexpr (ENV) s2[u] = env_row(a, li, rank[u], me, pc, csh);
      }
    if constexpr (ENV) {
      __syncwarp();  // every entry consumed: buf becomes the rank-ordered s^2 array
      double* sr = reinterpret_cast<double*>(buf);
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (lane + 32 * u < cnt) sr[rank[u]] = s2[u];
      __syncwarp();
      env_sigma(a, li, cnt, sr);
    }
  } else {
    constexpr int kMaxPer = 32;  // n_max < 1024 (context checks)
    double s2[kMaxPer];
    int rk[kMaxPer];
    // long lists (rc = 8): the same packed-key ranking one entry at a time, the full
    // comparison only for a list with a tie or an unpackable key
    bool fast = __all_sync(0xffffffffu, packable);
    if (fast) {
      bool tie = false;
      for (int i = lane, u = 0; i < cnt; i += 32, ++u) {
        const uint64_t mk = buf[i].key;
        int rank = 0, eq = 0;
        for (int j = 0; j < cnt; ++j) {
          const uint64_t o = buf[j].key;
          rank += o < mk;
          eq += o == mk;
        }
        rk[u] = rank;
        tie = tie || eq != 1;
      }
      fast = !__any_sync(0xffffffffu, tie);
    }
    for (int i = lane, u = 0; i < cnt; i += 32, ++u) {
      const NbrEntry me = buf[i];
      int rank = 0;
      if (fast) {
        rank = rk[u];
      } else {
        for (int j = 0; j < cnt; ++j) rank += full_less(a, buf[j], me, pc, csh);
      }
      out[rank] = a.cell_members[me.j];
      rk[u] = rank;
      if constexpr (ENV) s2[u] = env_row(a, li, rank, me, pc, csh);
    }
    if constexpr (ENV) {
      __syncwarp();
      double* sr = reinterpret_cast<double*>(buf);
      for (int i = lane, u = 0; i < cnt; i += 32, ++u) sr[rk[u]] = s2[u];
      __syncwarp();
      env_sigma(a, li, cnt, sr);
    }
  }
}

void launch_neighbors(const NbrArgs& a, cudaStream_t st) {
  if (a.n_lists == 0) return;
  const int cap = ((a.n_max + 1 + 31) / 32) * 32;
  const int grid = (a.n_lists + kNbrWarps - 1) / kNbrWarps;
  if (a.R) {
    const size_t smem = static_cast<size_t>(kNbrWarps) * cap * (sizeof(NbrEntry) + sizeof(int));
    ensure_smem_attr(reinterpret_cast<const void*>(k_neighbors<true>), smem);
    k_neighbors<true><<<grid, kNbrWarps * 32, smem, st>>>(a, cap); count_launch();
  } else {
    const size_t smem = static_cast<size_t>(kNbrWarps) * cap * (sizeof(NbrEntry) + sizeof(int));
    ensure_smem_attr(reinterpret_cast<const void*>(k_neighbors<false>), smem);
    k_neighbors<false><<<grid, kNbrWarps * 32, smem, st>>>(a, cap); count_launch();
  }
}

// ----------------------------------------------------------------------------------
// prod_force as a deterministic warp-segmented gather (no floating-point atomics).
// Target member t receives  +sum_k g[own centre][k]   (its centre self-term,
// center_grad = -sum g, F = -partials; deeppot.cpp:256-262, 300-309)
// and -g[c][k] for every row (c, k) of another centre c that lands on t.  Incoming
// centres are enumerated from t's own list (locals) or its reverse list (ghosts), the
// row k by a coalesced warp scan of c's member list.  Fixed summation order.
// ----------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_force_gather(ForceArgs a) {
  const int lane = threadIdx.x & 31;
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nloc = a.counts[kCntLoc];
  if (t >= (a.wide ? nloc : a.counts[kCntMem])) return;
  double own[3] = {0, 0, 0};
  const int oc = a.cidx[t];
  if (oc >= 0) {
    const int n = a.nn[oc];
    const double* g = a.g + static_cast<size_t>(oc) * a.n_max * 3;
    for (int k = lane; k < n; k += 32)
      for (int c = 0; c < 3; ++c) own[c] += g[3 * k + c];
  }
  const int* list;
  int cnt;
  if (t < nloc) {
    if (oc < 0) return;  // (only in a capacity-overflowed pass, which is redone)
    list = a.nlist + static_cast<size_t>(oc) * a.n_max;
    cnt = a.nn[oc];
  } else {
    list = a.rlist + static_cast<size_t>(t - nloc) * a.n_max;
    cnt = a.rn[t - nloc];
  }
  // lane per incoming centre c: find t's row k in c's list (16-byte loads), take g[c][k]
  double in[3] = {0, 0, 0};
  for (int e = lane; e < cnt; e += 32) {
    const int c = a.cidx[list[e]];
    if (c < 0) continue;
    const int nc = a.nn[c];
    const int* row = a.nlist + static_cast<size_t>(c) * a.n_max;
    int k = -1;
    const bool vec = (a.n_max & 3) == 0;
    if (vec) {
      for (int b = 0; b < nc && k < 0; b += 4) {
        const int4 q = *reinterpret_cast<const int4*>(row + b);
        if (q.x == t) k = b;
        else if (q.y == t && b + 1 < nc) k = b + 1;
        else if (q.z == t && b + 2 < nc) k = b + 2;
        else if (q.w == t && b + 3 < nc) k = b + 3;
      }
      if (k >= nc) k = -1;
    } else {
      for (int b = 0; b < nc && k < 0; ++b)
        if (row[b] == t) k = b;
    }
    if (k >= 0) {
      const double* g = a.g + (static_cast<size_t>(c) * a.n_max + k) * 3;
      for (int q = 0; q < 3; ++q) in[q] += g[q];
    }
  }
  for (int q = 0; q < 3; ++q) {
    const double v = warp_sum(own[q]) - warp_sum(in[q]);
    if (lane == 0) a.fmem[3 * static_cast<size_t>(t) + q] = v;
  }
}

void launch_force_gather(const ForceArgs& a, cudaStream_t st) {
  if (a.n_targets == 0) return;
  const long threads = static_cast<long>(a.n_targets) * 32;
  k_force_gather<<<static_cast<int>((threads + 127) / 128), 128, 0, st>>>(a); count_launch();
}

// ----------------------------------------------------------------------------------
// Ghost-force route (masked_reduction, decomp.cpp:445-469, 502-536).
// Pack, per DD rank: the owner's zero-image partial of each local goes to fown/eown
// (global atom index; exactly one rank owns an atom), and every ghost image that received
// partials becomes a RouteEntry for the atom's owner, grouped by destination rank.
// ----------------------------------------------------------------------------------
__global__ void k_route_count(RouteArgs a) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int nloc = a.counts[kCntLoc], ngh = a.counts[kCntGh];
  if (m >= nloc + ngh) return;
  if (m < nloc) {
    const int t = a.m_atom[m];
#pragma unroll
    for (int q = 0; q < 3; ++q) a.fown[3 * static_cast<size_t>(t) + q] = a.fmem[3 * static_cast<size_t>(m) + q];
    a.eown[t] = a.e_centre[m];
  } else if (!a.wide && a.rn[m - nloc] > 0) {
    atomicAdd(&a.cnt[a.rank * a.n_ranks + a.m_owner[m]], 1);
  }
}

__global__ void k_route_fill(RouteArgs a) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.counts[kCntGh] || a.rn[g] == 0) return;
  const int m = a.counts[kCntLoc] + g;
  const int o = a.m_owner[m];
  const int* row = a.cnt + a.rank * a.n_ranks;
  int off = 0;
  for (int q = 0; q < o; ++q) off += row[q];
  RouteEntry e;
  e.atom = a.m_atom[m];
  e.img = static_cast<short>(a.m_shift[m]);
  e.src = static_cast<short>(a.rank);
#pragma unroll
  for (int q = 0; q < 3; ++q) e.f[q] = a.fmem[3 * static_cast<size_t>(m) + q];
  a.buf[off + atomicAdd(&a.cur[o], 1)] = e;
}

void launch_route_pack(const RouteArgs& a, cudaStream_t st) {
  const int nm = a.nloc + a.ngh;
  if (nm > 0) {
    k_route_count<<<(nm + 255) / 256, 256, 0, st>>>(a); count_launch();
  }
  if (!a.wide && a.ngh > 0) {
    k_route_fill<<<(a.ngh + 255) / 256, 256, 0, st>>>(a); count_launch();
  }
}

// Merge.  Segment (s, o) = entries from source rank s for a destination o owned by this
// process; s's entries sit in its send buffer (s local: every destination, grouped) or in
// its receive buffer (s remote: this process's destinations only, grouped).
__device__ __forceinline__ bool rank_is_local(const MergeArgs& a, int r) {
  return r % a.world_size == a.world_rank;
}

__global__ void k_merge_plan(MergeArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int R = a.n_ranks;
  int* prefix = a.seg;            // [R*R + 1]
  int* offset = a.seg + R * R + 1;  // [R*R]
  int tot = 0;
  for (int s = 0; s < R; ++s) {
    const bool sl = rank_is_local(a, s);
    int off = 0;
    for (int o = 0; o < R; ++o) {
      const int c = a.cnt[s * R + o];
      const bool ol = rank_is_local(a, o);
      prefix[s * R + o] = tot;
      offset[s * R + o] = off;
      if (ol) tot += c;
      if (sl || ol) off += c;
    }
  }
  prefix[R * R] = tot;
}

// entry i of the incoming stream (segments in (s, o) order), nullptr past the end
__device__ __forceinline__ const RouteEntry* merge_entry(const MergeArgs& a, int i) {
  const int R = a.n_ranks;
  const int* prefix = a.seg;
  if (i >= prefix[R * R]) return nullptr;
  int lo = 0, hi = R * R;  // largest q with prefix[q] <= i and a non-empty segment
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (prefix[mid] <= i) lo = mid;
    else hi = mid;
  }
  const int s = lo / R;
  return a.src_base[s] + a.seg[R * R + 1 + lo] + (i - prefix[lo]);
}

__global__ void k_merge_count(MergeArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.capacity) return;
  const RouteEntry* e = merge_entry(a, i);
  if (e) atomicAdd(&a.inc_cnt[e->atom], 1);
}

__global__ void k_merge_fill(MergeArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.capacity) return;
  const RouteEntry* e = merge_entry(a, i);
  if (e) a.inc[a.inc_off[e->atom] + atomicSub(&a.inc_cnt[e->atom], 1) - 1] = e;
}

// Thread per atom owned by this process: own zero-image partial, then the routed partials
// in (zero image first, image, rank) order -- a unique key per entry, so the sum does not
// depend on the arrival order.
__global__ void k_merge_sum(MergeArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.n_atoms || !rank_is_local(a, a.owner[t])) return;
  double f[3] = {a.fown[3 * static_cast<size_t>(t)], a.fown[3 * static_cast<size_t>(t) + 1],
                 a.fown[3 * static_cast<size_t>(t) + 2]};
  const int b = a.inc_off[t], e = a.inc_off[t + 1];
  auto key = [](const RouteEntry* r) {
    return ((r->img == kZeroShift ? 0 : 1) << 24) | (static_cast<int>(r->img) << 16) | static_cast<int>(r->src);
  };
  int prev = -1;
  for (int done = b; done < e; ++done) {
    const RouteEntry* best = nullptr;
    int bk = 0x7fffffff;
    for (int j = b; j < e; ++j) {
      const int k = key(a.inc[j]);
      if (k > prev && k < bk) {
        bk = k;
        best = a.inc[j];
      }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) f[q] += best->f[q];
    prev = bk;
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) a.f_out[3 * static_cast<size_t>(t) + q] = f[q];
}

void launch_route_merge(const MergeArgs& a, cudaStream_t st) {
  k_merge_plan<<<1, 32, 0, st>>>(a); count_launch();
  if (a.capacity > 0) {
    k_merge_count<<<(a.capacity + 255) / 256, 256, 0, st>>>(a); count_launch();
    launch_scan(a.inc_cnt, a.inc_off, a.n_atoms, st);
    k_merge_fill<<<(a.capacity + 255) / 256, 256, 0, st>>>(a); count_launch();
  } else {
    cudaMemsetAsync(a.inc_off, 0, (a.n_atoms + 1) * sizeof(int), st);
  }
  if (a.n_atoms > 0) {
    k_merge_sum<<<(a.n_atoms + 255) / 256, 256, 0, st>>>(a); count_launch();
  }
}

__global__ void k_finalize(const double* __restrict__ red, int R, long n, double* __restrict__ out) {
  const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (i < 10) {
    double v = 0.0;
    for (int r = 0; r < R; ++r) v += red[10 * r + i];
    out[i] = v;
  }
  if (i < 4 * n) out[10 + i] = red[10 * static_cast<long>(R) + i];
}

void launch_finalize(const double* red, int n_ranks, long n_atoms, double* out, cudaStream_t st) {
  const long tot = std::max(10L, 4 * n_atoms);
  k_finalize<<<static_cast<int>((tot + 255) / 256), 256, 0, st>>>(red, n_ranks, n_atoms, out); count_launch();
}

// ----------------------------------------------------------------------------------
// Multi-centre tiles (rc = 4: n <= 64, ~27 rows per centre): groups of four consecutive
// centres become one 128-row unit when their rows fit, else two pairs (always fit).
// ----------------------------------------------------------------------------------
__device__ __forceinline__ int pack_group_units(const int* nn, int n_centres, int g) {
  const int c0 = 4 * g, c1 = min(n_centres, c0 + 4);
  int rows = 0;
  for (int c = c0; c < c1; ++c) rows += nn[c];
  return (rows <= 128 || c1 - c0 <= 2) ? 1 : 2;
}

__global__ void k_pack_count(const int* __restrict__ nn, const int* __restrict__ n_dev, int cap_groups,
                             int* __restrict__ cnt, int* __restrict__ n_groups) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_centres = *n_dev, ng = (n_centres + 3) / 4;
  if (g == 0) *n_groups = ng;
  if (g < cap_groups) cnt[g] = g < ng ? pack_group_units(nn, n_centres, g) : 0;
}

__global__ void k_pack_fill(const int* __restrict__ nn, const int* __restrict__ n_dev,
                            const int* __restrict__ off, int2* __restrict__ packs) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_centres = *n_dev;
  if (g >= (n_centres + 3) / 4) return;
  const int c0 = 4 * g, m = min(4, n_centres - c0);
  if (pack_group_units(nn, n_centres, g) == 1) {
    packs[off[g]] = make_int2(c0, m);
  } else {
    packs[off[g]] = make_int2(c0, 2);
    packs[off[g] + 1] = make_int2(c0 + 2, m - 2);
  }
}

// cnt: scratch of cap_groups + 1 ints, off: of cap_groups + 2 ints (scan | unit count at
// off[cap_groups]); groups past the live count contribute zero units
void launch_pack_plan(const int* nn, const int* n_dev, int n_centres_cap, int* cnt, int* off, int2* packs,
                      cudaStream_t st) {
  const int cg = (n_centres_cap + 3) / 4;
  if (cg == 0) {
    cudaMemsetAsync(off, 0, sizeof(int), st);
    return;
  }
  k_pack_count<<<(cg + 255) / 256, 256, 0, st>>>(nn, n_dev, cg, cnt, cnt + cg); count_launch();
  launch_scan(cnt, off, cg, st);  // off[cg] = unit count
  k_pack_fill<<<(cg + 255) / 256, 256, 0, st>>>(nn, n_dev, off, packs); count_launch();
}

// Two-stage deterministic reduction: block b sums the centres of its contiguous chunk
// (fixed thread order + block_sum tree), then one block adds the block partials in order.
constexpr int kEvBlocks = 148;

__global__ void __launch_bounds__(256) k_energy_virial(const double* __restrict__ e,
                                                       const double* __restrict__ vir,
                                                       const int* __restrict__ counts,
                                                       double* __restrict__ part) {
  __shared__ double red[8];
  const int nloc = counts[0];
  const int chunk = (nloc + gridDim.x - 1) / gridDim.x;
  const int c0 = blockIdx.x * chunk, c1 = min(nloc, c0 + chunk);
  double acc[10] = {0};
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    acc[0] += e[c];
    for (int q = 0; q < 9; ++q) acc[1 + q] += vir[9 * static_cast<size_t>(c) + q];
  }
  for (int q = 0; q < 10; ++q) {
    const double t = block_sum(acc[q], red);
    if (threadIdx.x == 0) part[10 * blockIdx.x + q] = t;
  }
}

// warp q sums component q of the block partials: lanes over blocks, then a fixed tree
__global__ void k_energy_virial_final(const double* __restrict__ part, int nb, double* __restrict__ row) {
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q >= 10) return;
  double t = 0.0;
  for (int b = lane; b < nb; b += 32) t += part[10 * b + q];
  t = warp_sum(t);
  if (lane == 0) row[q] = t;
}

void launch_energy_virial(const double* e, const double* vir, const int* counts, double* part, double* row,
                          cudaStream_t st) {
  k_energy_virial<<<kEvBlocks, 256, 0, st>>>(e, vir, counts, part); count_launch();
  k_energy_virial_final<<<1, 320, 0, st>>>(part, kEvBlocks, row); count_launch();
}

}  // namespace nb
