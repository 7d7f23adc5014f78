/* CPU restatement of the reference DPA-1 force path -- TEST INFRASTRUCTURE ONLY.
 *
 * This is the parity oracle for the CUDA product (paper_2604_07276_b200).  It restates,
 * in plain double-precision C++ over flat arrays, the reference algorithm of
 * /root/reference/proj (nnmd): neighbour rows, DPA-1 forward, exact backward, force
 * assembly, virial, ownership/halo and the per-rank DD contribution.  Each function in
 * dp_oracle.cpp cites the reference file:line it follows.
 *
 * Pinned against the compiled reference (oracle/_ref/libnnmd_ref.so) and against the
 * committed golden vectors in tests/golden/ (tests/test_oracle.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_model orc_model;

const char* orc_last_error(void);

orc_model* orc_model_init(double rc, double rcs, int n_max, int n_species, int type_dim,
                          int n_feat, int n_reduced, int n_attn, int attn_dim,
                          const int* embed_hidden, int n_embed_hidden, const int* fit_hidden,
                          int n_fit_hidden, uint64_t seed);
orc_model* orc_model_load(const char* path);
int orc_model_save(const orc_model* m, const char* path);
void orc_model_free(orc_model* m);
long orc_model_nparams(const orc_model* m);
/* all parameters in .nmdp declaration order (deeppot_io.cpp:14-16) */
int orc_model_flat(const orc_model* m, double* out, long cap);

/* Sorted canonical rows of every centre, single domain (neighbor.cpp:73-148 +
 * deeppot.cpp:141-184).  Returns 2 with the CapacityError message on overflow. */
int orc_neighbor_rows(const orc_model* m, int n, const double* pos, const int* species,
                      const int64_t* gids, const double* box3, const uint8_t* periodic,
                      long cap, int* counts, int* member, int* image, double* d, long* total);

/* Single-domain evaluation: energy, forces (3n), per-atom energies (n), virial (9). */
int orc_evaluate(const orc_model* m, int n, const double* pos, const int* species,
                 const int64_t* gids, const double* box3, const uint8_t* periodic,
                 double* energy, double* forces, double* atom_energy, double* virial);

/* One centre from explicit rows: energy and row gradients g_k = de/dd_k. */
int orc_evaluate_center(const orc_model* m, int center_species, int n_rows, const double* d,
                        const int* row_species, double* energy, double* row_grads);

int orc_partition_ranks(const double* box3, int n_ranks, double min_edge, int* dims);
int orc_owner_ranks(int n, const double* pos, const double* box3, const int* dims, int* owner);
int orc_build_halo(int n, const double* pos, const double* box3, const uint8_t* periodic,
                   const int* dims, int rank, double thickness, long cap, int* atom,
                   int* owner, int* shift, long* n_out);

/* One DD rank's contribution in a global-indexed buffer (decomp.cpp:265-542):
 * partial forces (3n, to be summed over ranks), owned per-atom energies (n),
 * owned energy, virial (9) and stats {locals, ghosts, centres}. */
int orc_dd_rank(const orc_model* m, int n, const double* pos, const int* species,
                const int64_t* gids, const double* box3, const uint8_t* periodic,
                int n_ranks, int scheme, int rank, double* forces, double* atom_energy,
                double* energy, double* virial, long* stats);

/* Synthetic solvated-protein input (bitwise equal to nnmd_synth_system). */
int orc_synth_system(int64_t n, double rho, double min_sep, uint64_t seed, double* box,
                     double* pos, int32_t* types);

#ifdef __cplusplus
}
#endif
