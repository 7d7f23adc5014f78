/* nnmd_b200 -- B200-native DPA-1 force provider behind a C ABI.
 *
 * Drop-in replacement for the reference NNPot/DeePMD backend path of nnmd
 * (/root/reference/proj):
 *
 *   nnmd::ForceProvider::evaluate        include/nnmd/engine.hpp:28-34
 *   nnmd::DpProvider(DPModel, Options)   include/nnmd/engine.hpp:51-74, src/engine.cpp:54-89
 *   nnmd::dd_evaluate(...)               include/nnmd/decomp.hpp:158-161, src/decomp.cpp:265-542
 *   nnmd::evaluate_dp(...)               include/nnmd/deeppot.hpp:141-143, src/deeppot.cpp:315-369
 *   nnmd::load_model / save_model        src/deeppot_io.cpp:56-160 (.nmdp format)
 *   nnmd::init_model                     src/deeppot.cpp:86-127 (bit-identical Xavier draws)
 *
 * Plain pointers and sizes only.  Every call returns an nnmd_status; the message of the
 * last failure on the calling thread is available from nnmd_b200_last_error().
 * Status codes mirror the reference exception classes (error.hpp:8-17):
 *   NNMD_OK = 0, NNMD_ERROR = 1 (nnmd::Error), NNMD_CAPACITY = 2 (nnmd::CapacityError,
 *   e.g. "neighbor overflow at atom id 7 on rank 0"), NNMD_CUDA = 3 (CUDA/NCCL failure).
 *
 * Threading: one context per calling thread; compute calls are synchronous.
 */
#ifndef NNMD_B200_H_
#define NNMD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { NNMD_OK = 0, NNMD_ERROR = 1, NNMD_CAPACITY = 2, NNMD_CUDA = 3 } nnmd_status;

typedef struct nnmd_model nnmd_model; /* host-side DPModel (deeppot.hpp:35-60) */
typedef struct nnmd_b200 nnmd_b200;   /* device context: streams, buffers, device weights, comms */

/* ModelSpec (deeppot.hpp:63-75). */
typedef struct {
  double rc, rcs;
  int n_max, n_species, type_dim, n_feat, n_reduced, n_attn, attn_dim;
  int n_embed_hidden;
  int embed_hidden[8];
  int n_fit_hidden;
  int fit_hidden[8];
} nnmd_model_spec;

/* DdScheme (decomp.hpp:128-129). */
enum { NNMD_MASKED_REDUCTION = 0, NNMD_WIDE_HALO = 1 };
/* Arithmetic of the dense contractions (all accumulate in FP32; geometry, row gradients,
 * forces, energies and virial are FP64):
 *   NNMD_PREC_FP32      3xTF32 on tcgen05 tensor cores (hi/lo split) -- FP32-grade,
 *                       parity tolerance 1e-5 relative (default)
 *   NNMD_PREC_TF32      1xTF32 on tcgen05 -- stated tolerance 5e-3 relative
 *   NNMD_PREC_FP32_SIMT plain FP32 FMA on CUDA cores (validation path) -- 1e-5 */
enum { NNMD_PREC_FP32 = 0, NNMD_PREC_TF32 = 1, NNMD_PREC_FP32_SIMT = 2 };

typedef struct {
  int n_ranks;    /* DD ranks (partition_ranks); 1 = one domain (== evaluate_dp bit-for-bit rows) */
  int scheme;     /* NNMD_MASKED_REDUCTION | NNMD_WIDE_HALO */
  int precision;  /* NNMD_PREC_FP32 */
  int device;     /* CUDA device ordinal for this process */
  int world_size; /* processes (one per GPU); DD ranks r with r % world_size == world_rank run here */
  int world_rank;
  const void* nccl_id; /* 128-byte ncclUniqueId shared by all processes, or NULL if world_size == 1 */
} nnmd_b200_opts;

const char* nnmd_b200_last_error(void);
const char* nnmd_b200_version(void);

/* ---- model (host) -------------------------------------------------------------- */
/* init_model(spec, seed): same std::mt19937_64 draw sequence -> bit-identical weights. */
nnmd_status nnmd_model_init(const nnmd_model_spec* spec, uint64_t seed, nnmd_model** out);
nnmd_status nnmd_model_load(const char* path, nnmd_model** out);   /* .nmdp v1 */
nnmd_status nnmd_model_save(const nnmd_model* m, const char* path);
void nnmd_model_free(nnmd_model* m);
long nnmd_model_nparams(const nnmd_model* m);
nnmd_status nnmd_model_get_spec(const nnmd_model* m, nnmd_model_spec* out);
/* n_max is both capacity and the 1/sqrt(n_max) descriptor normalisation (dp_core.hpp:360). */
nnmd_status nnmd_model_set_n_max(nnmd_model* m, int n_max);

/* ---- DD planning (host, no GPU needed) -------------------------------------------- */
/* partition_ranks (decomp.cpp:17-57): surface-minimising p_x*p_y*p_z = n_ranks. */
nnmd_status nnmd_partition_ranks(const double box[3], int n_ranks, double min_edge, int dims[3]);

/* Ghost-force route plan of one process (decomp.cpp:445-469; DD rank r runs in process
 * r % world_size): counts[s*n_ranks + o] = routed entries from source rank s to owner rank o.
 * Writes up to cap ops {kind 0 send / 1 receive, src, dst, peer process, offset (entries
 * into the source's send buffer, grouped by every destination, or into its receive buffer,
 * grouped by this process's destinations), count}; returns the op count (< 0: error).
 * Sends and receives are in (source, destination) order on every process, so transfers
 * between one pair of processes match in posting order (ncclSend/ncclRecv in one group). */
typedef struct {
  int kind, src, dst, peer;
  long offset;
  int count;
} nnmd_route_op;
int nnmd_route_schedule(int n_ranks, int world_size, int world_rank, const int* counts, nnmd_route_op* out,
                        int cap);

/* ---- device context ----------------------------------------------------------------- */
nnmd_status nnmd_b200_create(const nnmd_model* m, const nnmd_b200_opts* opts, nnmd_b200** out);
void nnmd_b200_destroy(nnmd_b200* ctx);
/* ncclGetUniqueId for world_size > 1 (rank 0 calls it and broadcasts the 128 bytes). */
nnmd_status nnmd_b200_nccl_unique_id(void* out128);

/* DpProvider::evaluate / dd_evaluate with HOST buffers (positions must be wrapped into
 * [0, L) on periodic axes; with world_size > 1 only world rank 0's coords are read -- the
 * others may pass NULL -- and reach every GPU by ncclBroadcast, collective 1).  Outputs are
 * the replicated full-system results: energy = sum of owned per-atom energies, forces[3n] = -dE/dx, virial[9] row-major
 * W_ab = -sum g_{k,a} d_{k,b}, atom_energy[n] (NULL to skip). */
nnmd_status nnmd_b200_compute(nnmd_b200* ctx, int64_t n, const double* coords,
                              const int32_t* types, const int64_t* gids, const double box[3],
                              const uint8_t periodic[3], double* energy, double* forces,
                              double* virial, double* atom_energy);

/* Same evaluation on DEVICE-resident inputs/outputs (pointers on ctx's device); no bulk
 * host copies.  Host synchronisation points per call (cudaStreamSynchronize):
 *   - one at the end: step flags (overflow / wrap errors, ghost-capacity overflow and route
 *     counts, all-reduced over processes so that every process throws together), the
 *     per-rank counts and the per-kernel event times;
 *   - with world_size > 1 and masked_reduction, one more after the all-reduce of the route
 *     counts, which sizes the point-to-point ghost-force transfers.
 * The DD build reads nothing back: its buffers are sized by per-rank ghost capacities and
 * the kernels take their live counts from device memory.  When a capacity overflows
 * (flagged on the device) the call grows it and redoes the step before returning.
 * The call returns with the stream idle.  With world_size > 1 the positions of world
 * rank 0 are broadcast to all processes (collective 1) before the DD build.
 * d_out layout (float64): [energy, virial(9), forces(3n), atom_energy(n)]. */
nnmd_status nnmd_b200_compute_device(nnmd_b200* ctx, int64_t n, const double* d_coords,
                                     const int32_t* d_types, const int64_t* d_gids,
                                     const double box[3], const uint8_t periodic[3],
                                     double* d_out);

/* ---- device-resident MD loop (run_md, engine.cpp:143-211; MDConfig, engine.hpp:99-107) */
typedef struct {
  double dt;                 /* > 0 */
  long n_steps;
  long equil_steps;          /* velocity rescaling during the first equil_steps ... */
  double target_temperature; /* ... to this temperature (<= 0 disables) ... */
  long rescale_every;        /* ... every rescale_every steps */
} nnmd_md_config;

/* n_steps of NVE leap-frog (leapfrog_step, engine.cpp:91-100: v += (dt/m) F, r += dt v,
 * wrapped) with this context's DPA-1 forces.  Positions and velocities stay on the device
 * for the whole run (one H2D before, one D2H after); each process integrates its own
 * replicated copy, so no position collective is needed.  coords/velocities are updated in
 * place; potential[k] / total[k] (may be NULL) receive run_md's per-step potential energy
 * and potential + on-step kinetic energy (mid-point velocities).  A non-finite force fails
 * with NNMD_ERROR "run_md: non-finite force from provider 'nnmd_b200' at step k" before
 * that step integrates (engine.cpp:166-176): coords/velocities hold the failing step's
 * state. */
nnmd_status nnmd_b200_run_md(nnmd_b200* ctx, int64_t n, double* coords, double* velocities,
                             const double* masses, const int32_t* types, const int64_t* gids,
                             const double box[3], const uint8_t periodic[3], const nnmd_md_config* cfg,
                             double* potential, double* total);
/* Same on device buffers; d_energies[2k] = potential, d_energies[2k+1] = total of step k. */
nnmd_status nnmd_b200_run_md_device(nnmd_b200* ctx, int64_t n, double* d_coords, double* d_velocities,
                                    const double* d_masses, const int32_t* d_types, const int64_t* d_gids,
                                    const double box[3], const uint8_t periodic[3],
                                    const nnmd_md_config* cfg, double* d_energies);

/* ---- tracing and the collective ledger (trace.hpp, decomp.hpp:64-107) -------------- */
/* Span (trace.hpp:25-31): phase ids in nnmd::Phase order -- 0 classical_md,
 * 1 gather_positions, 2 dd_build, 3 neighbor_build, 4 inference, 5 ghost_force_route,
 * 6 reduce_forces, 7 integrate; rank -1 = step-global phase; seconds on the host steady
 * clock (TraceSink::now), device intervals measured with CUDA events. */
typedef struct {
  int rank;
  int phase;
  double t_start, t_end;
  long step;
} nnmd_span;
/* CollectiveRecord (decomp.hpp:84-89): kind 0 gather_positions, 1 ghost_force_route,
 * 2 reduce_forces; bytes by the reference PayloadLayout (20 B/atom gather, 12 B/atom
 * reduction, 20 B per routed ghost entry). */
typedef struct {
  long step;
  int kind;
  uint64_t bytes;
  int participants;
} nnmd_collective_record;

/* Record spans and/or ledger entries on subsequent computes (off by default). */
void nnmd_b200_set_trace(nnmd_b200* ctx, int spans, int ledger);
/* Step index stamped on the records (StepContext::step); run_md advances it itself. */
void nnmd_b200_set_step(nnmd_b200* ctx, long step);
/* Copy out up to cap records; return the total number held (call with cap 0 to size). */
int nnmd_b200_trace_spans(const nnmd_b200* ctx, nnmd_span* out, int cap);
int nnmd_b200_ledger(const nnmd_b200* ctx, nnmd_collective_record* out, int cap);
void nnmd_b200_trace_clear(nnmd_b200* ctx);
/* export_chrome_trace (trace.cpp:64-85) of the held spans. */
nnmd_status nnmd_b200_export_chrome_trace(const nnmd_b200* ctx, const char* path);

/* Per-rank statistics of the last compute (RankStats, decomp.hpp:133-142):
 * counts = {locals, ghosts, centres, route_entries}; ms = {dd, neighbor, inference, comm}
 * measured with CUDA events on the rank's stream. */
nnmd_status nnmd_b200_rank_stats(const nnmd_b200* ctx, int rank, int64_t counts[4], double ms[4]);
/* Per-kernel device times (ms) of the last compute, by name; returns the number written. */
int nnmd_b200_kernel_times(const nnmd_b200* ctx, const char** names, double* ms, int cap);

/* Enable capture of the parity hooks below on subsequent compute calls (costs a copy). */
void nnmd_b200_set_debug(nnmd_b200* ctx, int on);
/* Parity hooks: the fixed-width sorted neighbour list of one rank from the last compute.
 * idx[n_centres * n_max] = atom index of each row's member, img[.. * 3] its image shift,
 * counts[n_centres]; centre_atoms[n_centres] = atom of each centre.  Pass NULL to query
 * *n_centres only. */
nnmd_status nnmd_b200_debug_nlist(const nnmd_b200* ctx, int rank, int* n_centres,
                                  int32_t* centre_atoms, int32_t* idx, int32_t* img,
                                  int32_t* counts);
/* Ghost set of one rank: atom, owner rank and shift[3] per ghost, (atom, shift) order. */
nnmd_status nnmd_b200_debug_ghosts(const nnmd_b200* ctx, int rank, int* n_ghosts,
                                   int32_t* atom, int32_t* owner, int32_t* shift);

/* Self-test of the in-kernel block GEMM (one CTA) on host buffers: C[M x N] = op(A) op(B),
 * A is [M x K] (ta=0) or [K x M] (ta=1), B is [K x N] (tb=0) or [N x K] (tb=1);
 * mode 0 SIMT FP32, 1 3xTF32 tcgen05, 2 1xTF32 tcgen05. */
nnmd_status nnmd_b200_selftest_gemm(int mode, int ta, int tb, int M, int N, int K, const float* A,
                                    const float* B, float* C);
/* Total kernels launched by this library in this process (bench launch accounting). */
long long nnmd_b200_launch_count(void);
/* Device stream of the context (cudaStream_t), for external event timing. */
void* nnmd_b200_stream(const nnmd_b200* ctx);

/* ---- synthetic input (test-system plumbing, not the hot path) ------------------------ */
/* Deterministic solvated-protein-like system: a compact H/C/N/O/S globule in water (O, H)
 * with ions, uniform density rho, minimum separation min_sep, cubic periodic box of edge
 * (n/rho)^(1/3).  Species: 0 H, 1 C, 2 N, 3 O, 4 S, 5 ion (Na/Cl). */
nnmd_status nnmd_synth_system(int64_t n, double rho, double min_sep, uint64_t seed,
                              double box[3], double* coords, int32_t* types);

#ifdef __cplusplus
}
#endif
#endif /* NNMD_B200_H_ */
