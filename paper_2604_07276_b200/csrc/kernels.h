// Kernel argument structs and host launch wrappers of nnmd_b200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nb {

// Number of kernels launched by this library in the process (for the bench's launch count).
void count_launch();
long long launch_count();

// ---------------------------------------------------------------- DD build -----------
struct SysArgs {
  const double* pos;      // 3n, wrapped on periodic axes
  const int* species;     // n
  const int64_t* gid;     // n
  int n;
  double L[3];
  int per[3];
  int n_species;
};

struct RankArgs {
  int rank;
  int dims[3];
  double lo[3], hi[3];   // subdomain (make_subdomain, decomp.cpp:80-94)
  double slab_lo[3], slab_hi[3];   // lo - t - guard, hi + t + guard (decomp.cpp:104-108)
  double rc_lo[3], rc_hi[3];       // rc slab (first-layer test, decomp.cpp:317-321)
  int wide;              // 1: wide_halo (first-layer ghosts are centres)
};

// err[0]: first atom with an unwrapped position / bad species (atomicMin), err[1]: first
// centre whose neighbour count exceeds n_max (atomicMin), err[2]: first ghost target whose
// reverse list overflows.  Initialised to INT_MAX.
void launch_owner(const SysArgs& s, const int dims[3], int* owner, int* err, cudaStream_t st);
void launch_dd_flags(const SysArgs& s, const RankArgs& r, const int* owner, int* is_local,
                     int* gcount, cudaStream_t st);
// exclusive scan of n ints; out[n] receives the total (out has n+1 entries)
void launch_scan(const int* in, int* out, int n, cudaStream_t st);
// same, n read from device memory (*n_dev) when the kernel runs
void launch_scan_dev(const int* in, int* out, const int* n_dev, cudaStream_t st);
// dst[i] = -src[i], i < n <= 32 (error words -> max-reducible step flags)
void launch_negate(const int* src, int* dst, int n, cudaStream_t st);
// Members are written only below cap_members (the buffers' capacity); launch_rank_counts
// reports an overflow.
void launch_dd_members(const SysArgs& s, const RankArgs& r, const int* owner, const int* loc_off,
                       const int* gh_off, int n_atoms, int cap_members, int* m_atom, int* m_shift,
                       double* m_pos, int* m_owner, cudaStream_t st);

// Device-resident counts of one DD rank (no host read-back inside a step):
enum { kCntLoc = 0, kCntGh = 1, kCntCen = 2, kCntRoute = 3, kCntMem = 4, kCntGhExact = 5, kCntCenExact = 6,
       kCntLocExact = 7, kCntWords = 8 };
// counts[kCntLoc] = locals, [kCntGh] = ghosts (each clamped to its capacity), [kCntMem] =
// members, [kCntCen] = locals (masked scheme; wide: set by launch_centre_compact), the exact
// counts in [kCntLocExact], [kCntGhExact]; *overflow = 1 when a capacity is exceeded (the
// step's outputs are then discarded and it is redone: kernels only need to stay in bounds).
void launch_rank_counts(const int* loc_off, const int* gh_off, int n_atoms, int cap_locals, int cap_ghosts,
                        int* counts, int* overflow, cudaStream_t st);
// centre flags over members (locals always; first-layer ghosts when wide)
void launch_centre_flags(const RankArgs& r, const int* counts /*[nloc, ngh]*/, const double* m_pos,
                         int n_members_cap, int* flag, cudaStream_t st);
// over counts[kCntMem] members (grid: n_members_cap); wide_halo also sets counts[kCntCen]
// (clamped to cap_centres, *overflow = 1 beyond it)
void launch_centre_compact(const int* flag, const int* off, int* counts, int n_members_cap, int wide,
                           int cap_centres, int* cen_member, int* cidx, int* overflow, cudaStream_t st);

// ---------------------------------------------------------------- cells / neighbours -
struct CellArgs {
  double origin[3], width[3];
  int dims[3];
};
// over *n_members_dev members (grid: n_members_cap)
void launch_cell_count(const CellArgs& c, const double* m_pos, const int* n_members_dev, int n_members_cap,
                       int* m_cell, int* cell_count, cudaStream_t st);
// cell-ordered copies of the per-candidate inputs of the neighbour scan (k_cell_fill)
struct CellSorted {
  const double* pos;          // atom positions [n][3]
  const int* atom_species;
  const int64_t* atom_gid;
  const int* m_atom;
  const int* m_shift;
  double *x, *y, *z;          // [members], cell order
  int* shift;
  int* species;
  int64_t* gid;
  int n_species;              // species copies clamped into the table (bad input is reported by
                              // k_owner and raised at the step's end; the kernels stay in bounds)
};
void launch_cell_fill(const int* m_cell, const int* n_members_dev, int n_members_cap, const int* cell_start,
                      int* cell_fill, int* cell_members, const CellSorted& cs, cudaStream_t st);

struct NbrArgs {
  const double* pos;
  const int* species;
  const int64_t* gid;
  double L[3];
  const int* m_atom;
  const int* m_shift;
  const int* m_cell;
  const int* cell_start;
  const int* cell_members;
  CellSorted cs;             // cell-ordered candidate data (same index as cell_members)
  int cdims[3];
  const int* centre_member;  // member index of each list owner (NULL: li + member_offset)
  int member_offset;
  int n_lists;               // capacity (grid); the live count is *n_lists_dev
  const int* n_lists_dev;
  const int* member_offset_dev;  // reverse lists: *member_offset_dev (locals) instead of member_offset
  int cand_limit;            // only candidate members with index < cand_limit
  const int* cand_limit_dev;  // (reverse lists) *cand_limit_dev instead
  int n_max;
  double rc2;
  int* nlist;                // [n_lists][n_max] member indices, canonical order
  int* nn;                   // [n_lists]
  int* err;                  // &err[slot]: atomicMin of the owner atom of an overflowing list
  int* nonempty;             // optional: count of lists with >= 1 row (route entries)
  int* maxn;                 // optional: atomicMax of the row counts
  uint64_t kbase;            // sort-key packing: bits(r2) - kbase < 2^58 for r2 < rc2
  // fused environment matrix (centre lists only; NULL R: rows only)
  float4* R;                 // [n_lists][n_max] (s, s/r d)
  int* Z;                    // [n_lists][n_max] neighbour species
  double* sig;               // [n_lists] sum_k s_k^2
  double rc, rcs;
};
void launch_neighbors(const NbrArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- forces --------------
struct ForceArgs {
  const int* counts;     // device counts (kCnt*): live nloc and member count
  int wide;
  const int* nlist;
  const int* nn;
  int n_max;
  const int* cidx;       // member -> centre index, -1 if not a centre
  const int* rlist;      // ghost reverse lists (masked), [n_ghost][n_max]
  const int* rn;
  int n_targets;         // capacity (grid); live: masked all members, wide locals
  const double* g;       // [centre][n_max][3] row gradients de/dd_k
  double* fmem;          // [member][3] force partial
};
void launch_force_gather(const ForceArgs& a, cudaStream_t st);

// row[0..9] = [sum_{c < nloc} e[c], sum vir[c]] of one DD rank (deterministic single-block
// reduction in two stages); the ranks' rows are summed in rank order by launch_finalize
// part: scratch of kEnergyVirialPartials doubles
constexpr int kEnergyVirialPartials = 148 * 10;
void launch_energy_virial(const double* e_centre, const double* vir, const int* counts, double* part,
                          double* row, cudaStream_t st);

// ---------------------------------------------------------------- ghost-force route -----
// One routed partial (decomp.cpp:445-455): a ghost image's force partial travelling from
// the rank that evaluated it (src) to the atom's owner.  f is the force contribution
// (the negated row-gradient partial), so the owner's merge is a plain sum.
struct RouteEntry {
  int atom;
  short img;   // packed shift 0..26 (kZeroShift = 13)
  short src;   // DD rank that evaluated the image
  double f[3];
};
static_assert(sizeof(RouteEntry) == 32, "RouteEntry is 32 bytes");

struct RouteArgs {
  int rank, n_ranks, wide;
  int nloc, ngh;            // capacities (grids); live counts from `counts`
  const int* counts;        // device counts (kCnt*)
  const int* m_atom;
  const int* m_shift;
  const int* m_owner;
  const int* rn;            // reverse-list row counts of the ghosts (0: no partials)
  const double* fmem;       // [member][3] force partials of this rank
  const double* e_centre;   // energies of the rank's centres (locals first)
  double* fown;             // [n][3] owner's zero-image partial (global atom index)
  double* eown;             // [n] atom energies (owner)
  int* cnt;                 // [R][R] routed entries src -> dst (row = this rank)
  int* cur;                 // [R] fill cursors of this rank (zeroed by count)
  RouteEntry* buf;          // this rank's entries, grouped by destination (capacity ngh)
};
// base partials + per-destination counts, then the grouped fill (order inside a group is
// not deterministic; the owner's merge orders entries by (zero image first, image, rank))
void launch_route_pack(const RouteArgs& a, cudaStream_t st);

constexpr int kMaxRanks = 64;
struct MergeArgs {
  int n_ranks, world_size, world_rank, n_atoms;
  const int* cnt;                 // [R][R]
  const RouteEntry* src_base[kMaxRanks];  // entries of source s: its send buffer (local s,
                                          // grouped by every destination) or its receive
                                          // buffer (remote s, this process's destinations)
  int* seg;                       // scratch: [R*R + 1] segment prefix, [R*R] offsets
  int* inc_cnt;                   // [n + 1] incoming entries per atom (zeroed by plan)
  int* inc_off;                   // [n + 1] exclusive prefix
  const RouteEntry** inc;         // [capacity] entries sorted by atom
  int capacity;                   // >= total incoming entries
  const int* owner;               // [n] owner rank of each atom
  const double* fown;             // [n][3]
  double* f_out;                  // [n][3] merged force of the locally owned atoms
};
// owner merge (decomp.cpp:502-536): own zero-image partial first, then the routed partials
// in (zero image first, image, rank) order
void launch_route_merge(const MergeArgs& a, cudaStream_t st);

// out[0..9] = sum over ranks of row[r][0..9] in rank order; out[10..] = red[10R..] (F, e_i)
void launch_finalize(const double* red, int n_ranks, long n_atoms, double* out, cudaStream_t st);

// ---------------------------------------------------------------- network -------------
constexpr int kMaxLayers = 8;
struct DpArgs {
  // model
  int M, mr, n_max, ns, n_embed, n_attn, n_fit;
  int edims[kMaxLayers];          // output width of each embed layer
  int fdims[kMaxLayers + 1];      // fit widths, fdims[0] = M*mr
  const float* w0;
  const float* ctab;
  const float* ew[kMaxLayers];
  const float* eb[kMaxLayers];
  const float* ab[16];
  const float* fw[kMaxLayers];
  const float* fb[kMaxLayers];
  double rc, rcs;
  float inv_sqrt_nmax;
  // system
  const double* pos;
  const int* species;
  double L[3];
  // rank
  const int* m_atom;
  const int* m_shift;
  const int* cen_member;
  int n_centres;              // capacity (grids, stash strides); live count *n_centres_dev
  const int* n_centres_dev;
  const int* nlist;
  const int* nn;
  // stash (per centre) and scratch (per CTA slot)
  float* X;             // [n_attn+1][n_centres][n_max][M]
  size_t x_layer_stride;
  // forward stash reused by the backward (no recompute): U = X [A|B] per layer
  // [n_attn][n_centres][n_max][2M], pu and P~ per layer [n_attn][n_centres][n_max][n_max4],
  // embedding hidden activations [n_centres][n_max][sum hidden widths]
  float* Ust;
  float* PUst;
  float* PTst;
  float* EMBst;
  size_t u_layer_stride, p_layer_stride, emb_centre_stride;
  float4* R;            // [n_centres][n_max] env rows (s, s dx/r, s dy/r, s dz/r), k_neighbors
  int* Z;               // [n_centres][n_max] neighbour species, k_neighbors
  double* sig;          // [n_centres] sum_k s_k^2 (FP64), k_neighbors
  float* Ad;            // [n_centres][M*4]
  float* Bd;            // [n_centres][4*mr]
  float* D;             // [n_centres][M*mr]
  float* dD;            // [n_centres][M*mr]
  double* g;            // [n_centres][n_max][3]
  double* vir;          // [n_centres][9]
  float* scratch;
  size_t scratch_slot;  // floats per CTA slot
  int mode;             // 0 SIMT FP32, 1 3xTF32 tcgen05, 2 1xTF32 tcgen05
  unsigned long long* prof;  // optional per-phase cycle counters (thread 0 of each CTA)
  int flags;            // diagnostic switches (env NNMD_FLAGS, 0 in production): bit0 no L2 prefetch
                        // of the stash, bit1 unfused backward n x n passes, bit2 no weight images
  // pre-split weight images (launch_weight_image) of the per-centre weight GEMMs' B
  // operands, or NULL: U = X [A|B], dX += dU [A|B]^T, embedding forward / backward
  const uint8_t* img_ab[16];
  const uint8_t* img_abT[16];
  const uint8_t* img_ew[kMaxLayers];
  const uint8_t* img_ewT[kMaxLayers];
  int wimg;  // 1: all of the above are present (the per-centre kernels' WIMG variant)
  int* work;  // dynamic centre counter of the persistent per-centre kernels (zeroed per launch)
  // Work units of the per-centre kernels.  packs == NULL: one centre per unit (unit u =
  // centre u, unit_rows = n_max).  Otherwise (n_max <= 64, tcgen05 modes) consecutive centres
  // share one 128-row tile: packs[u] = (first centre, centre count <= 4), *n_units_dev units,
  // unit_rows = 128; the n x n matrices of a unit are block diagonal (one block per centre).
  // The stash (X, U, pu, P~, embedding activations) is indexed by unit with unit_rows rows.
  const int2* packs;
  const int* n_units_dev;
  int unit_rows;
};
// Packs of consecutive centres (groups of 4: one pack if their rows fit 128, else two
// pairs); units written to packs, their count to *n_units.  cnt/off: scratch of
// ceil(n_centres/4) + 1 ints.
void launch_pack_plan(const int* nn, const int* n_centres_dev, int n_centres_cap, int* cnt, int* off, int2* packs,
                      cudaStream_t st);
inline int pack_capacity(int n_centres) { return 2 * ((n_centres + 3) / 4); }
// Weight images: bytes for a K x N operand, and the builder (B(k,n) = TB ? W[n*ldb+k] :
// W[k*ldb+n]).
size_t weight_image_bytes(int K, int N);
void launch_weight_image(const float* W, int TB, int ldb, int K, int N, uint8_t* out, cudaStream_t st);
size_t dp_scratch_floats(const DpArgs& a);
size_t dp_smem_bytes(const DpArgs& a, int mode);
// Environment matrix: FP64 geometry (image_delta, r, switch) -> float4 env rows, species,
// and sigma = sum s^2 per centre; warp per centre, coalesced row stores.
void launch_centre_forward(const DpArgs& a, int grid, cudaStream_t st);
void launch_centre_backward(const DpArgs& a, int grid, cudaStream_t st);

// Fitting net over all centres (batched GEMMs): Y[l] activations, e (double) energies,
// then dD = de/dD.
struct FitArgs {
  int n_fit;
  int fdims[kMaxLayers + 1];
  const float* fw[kMaxLayers];
  const float* fb[kMaxLayers];
  int n_centres;              // capacity (grids); live count *n_centres_dev
  const int* n_centres_dev;
  const float* D;
  float* Y[kMaxLayers];      // hidden activations [n_centres][fdims[l+1]]
  float* delta[2];           // ping-pong [n_centres][max width]
  double* e;                 // [n_centres]
  float* dD;
  int mode;
  int n_sm;                  // SMs of the device
  float* ws;                 // split-K partial sums, fit_workspace_floats(...) floats
  const float* fwT[kMaxLayers];  // W_l^T ([in][out]): K-major B operands of the backward
  int flags;                 // NNMD_FLAGS (bit 5: register-staged fit GEMMs instead of TMA)
};
// e[c] = b + w . Y_{L-2}[c]; delta = w (1 - Y^2)
void launch_fit_out(const FitArgs& a, float* delta, cudaStream_t st);
// Split-K of the wide fitting layer: slice count for a K (K only: rank-count invariant), and
// the fixed-order sum of the S raw slices P[z][M][N] with the layer's epilogue (epi: 0
// store, 1 tanh(x + bias), 2 x (1 - Y^2))
int fit_split_k(int K);
void launch_fit_splitk_sum(int M, const int* M_live, int N, int S, const float* P, float* C, const float* bias,
                           const float* Y, int epi, cudaStream_t st);
// The fitting net on the TMA-fed engine (fit_kernels.cu), when fit_tma_supported(a)
bool fit_tma_supported(const FitArgs& a);
void launch_fit_tma(const FitArgs& a, cudaStream_t st);
// Split-K workspace of the fitting net's K = M * mr layer (small centre counts: one row
// tile per 128 centres cannot fill the GPU, so K is split and the partials summed in order)
size_t fit_workspace_floats(int n_centres, int width);
void launch_fit(const FitArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- MD loop -------------
struct MdArgs {
  int n;
  double* pos;          // [n][3], wrapped in place
  double* vel;          // [n][3]
  const double* mass;   // [n]
  const double* F;      // [n][3] forces of this step
  double dt;
  double L[3];
  int per[3];
  double* ke_atom;      // [n] on-step kinetic energy per atom (mid-point velocity)
  int* err;             // atomicMin(step) on a non-finite force
  int step;
};
void launch_leapfrog(const MdArgs& a, cudaStream_t st);
// err = step when a force component is non-finite (checked before integrating)
void launch_force_check(const MdArgs& a, cudaStream_t st);
// rec[2 step] = epot[0], rec[2 step + 1] = epot[0] + sum(ke_atom)  (deterministic)
void launch_energy_record(const double* ke_atom, int n, const double* epot, double* rec, long step,
                          cudaStream_t st);
// velocity rescaling to `temperature` from the stored velocities' kinetic energy
void launch_rescale(int n, double* vel, const double* mass, double* ke_atom, double* ke_sum, double temperature,
                    cudaStream_t st);

// One-CTA test of the block GEMM building block (device pointers), mode as DpArgs::mode.
void selftest_gemm(int mode, int ta, int tb, int M, int N, int K, const float* A, int lda, const float* B,
                   int ldb, float* C);

}  // namespace nb
