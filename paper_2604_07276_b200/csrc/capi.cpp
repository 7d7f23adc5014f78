// extern "C" boundary of nnmd_b200 (include/nnmd_b200.h).  Exceptions never cross the
// ABI: they map to status codes mirroring the reference classes (error.hpp:8-17).
#include <cstring>
#include <string>

#include "context.h"
#include "kernels.h"
#include "model.h"
#include "nnmd_b200.h"

namespace nb {
void synth_system(int64_t n, double rho, double min_sep, uint64_t seed, double box[3],
                  double* pos, int32_t* types);
}

namespace {

thread_local std::string g_err;

template <class F>
nnmd_status guarded(F&& f) {
  try {
    f();
    return NNMD_OK;
  } catch (const nb::CapacityError& e) {
    g_err = e.what();
    return NNMD_CAPACITY;
  } catch (const nb::CudaError& e) {
    g_err = e.what();
    return NNMD_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NNMD_ERROR;
  }
}

nb::Context& C(nnmd_b200* h) {
  nb::require(h && h->ctx, "nnmd_b200: null context");
  return *h->ctx;
}

}  // namespace

extern "C" {

const char* nnmd_b200_last_error(void) { return g_err.c_str(); }
const char* nnmd_b200_version(void) { return "nnmd_b200 0.2 (sm_100a, 3xTF32 tcgen05 network, fp64 geometry/forces)"; }

nnmd_status nnmd_model_init(const nnmd_model_spec* spec, uint64_t seed, nnmd_model** out) {
  return guarded([&] {
    nb::require(spec && out, "nnmd_model_init: null argument");
    auto* m = new nnmd_model;
    try {
      m->m = nb::init_model(*spec, seed);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

nnmd_status nnmd_model_load(const char* path, nnmd_model** out) {
  return guarded([&] {
    nb::require(path && out, "nnmd_model_load: null argument");
    auto* m = new nnmd_model;
    try {
      m->m = nb::load_model(path);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

nnmd_status nnmd_model_save(const nnmd_model* m, const char* path) {
  return guarded([&] {
    nb::require(m && path, "nnmd_model_save: null argument");
    nb::save_model(m->m, path);
  });
}

void nnmd_model_free(nnmd_model* m) { delete m; }

long nnmd_model_nparams(const nnmd_model* m) { return m ? m->m.n_params() : 0; }

nnmd_status nnmd_model_get_spec(const nnmd_model* mm, nnmd_model_spec* out) {
  return guarded([&] {
    nb::require(mm && out, "nnmd_model_get_spec: null argument");
    const nb::Model& m = mm->m;
    std::memset(out, 0, sizeof *out);
    out->rc = m.rc;
    out->rcs = m.rcs;
    out->n_max = m.n_max;
    out->n_species = m.ns;
    out->type_dim = m.dz;
    out->n_feat = m.M;
    out->n_reduced = m.mr;
    out->n_attn = m.na;
    out->attn_dim = m.da;
    out->n_embed_hidden = static_cast<int>(m.embed.size()) - 1;
    for (int i = 0; i + 1 < static_cast<int>(m.embed.size()) && i < 8; ++i) out->embed_hidden[i] = m.embed[i].nout;
    out->n_fit_hidden = static_cast<int>(m.fit.size()) - 1;
    for (int i = 0; i + 1 < static_cast<int>(m.fit.size()) && i < 8; ++i) out->fit_hidden[i] = m.fit[i].nout;
  });
}

nnmd_status nnmd_model_set_n_max(nnmd_model* m, int n_max) {
  return guarded([&] {
    nb::require(m && n_max >= 1, "nnmd_model_set_n_max: bad argument");
    m->m.n_max = n_max;
    m->m.validate();
  });
}

nnmd_status nnmd_partition_ranks(const double box[3], int n_ranks, double min_edge, int dims[3]) {
  return guarded([&] {
    const auto d = nb::partition_ranks(box, n_ranks, min_edge);
    for (int a = 0; a < 3; ++a) dims[a] = d[a];
  });
}

int nnmd_route_schedule(int n_ranks, int world_size, int world_rank, const int* counts, nnmd_route_op* out,
                        int cap) {
  int n = -1;
  const nnmd_status st = guarded([&] {
    const auto ops = nb::route_schedule(n_ranks, world_size, world_rank, counts);
    nb::require(out || ops.empty() || cap == 0, "nnmd_route_schedule: null output");
    for (size_t i = 0; i < ops.size() && static_cast<int>(i) < cap; ++i)
      out[i] = {ops[i].kind, ops[i].src, ops[i].dst, ops[i].peer, ops[i].offset, ops[i].count};
    n = static_cast<int>(ops.size());
  });
  return st == NNMD_OK ? n : -1;
}

nnmd_status nnmd_b200_create(const nnmd_model* m, const nnmd_b200_opts* opts, nnmd_b200** out) {
  return guarded([&] {
    nb::require(m && opts && out, "nnmd_b200_create: null argument");
    auto* h = new nnmd_b200;
    try {
      h->ctx = new nb::Context(m->m, *opts);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void nnmd_b200_destroy(nnmd_b200* h) {
  if (!h) return;
  delete h->ctx;
  delete h;
}

nnmd_status nnmd_b200_nccl_unique_id(void* out128) {
  return guarded([&] {
    const nb::Nccl& N = nb::nccl();
    nb::require(N.ok, "NCCL unavailable: " + N.err);
    nb::NcclUid uid;
    const int r = N.GetUniqueId(&uid);
    if (r != 0) throw nb::CudaError(std::string("ncclGetUniqueId: ") + N.GetErrorString(r));
    std::memcpy(out128, &uid, sizeof uid);
  });
}

nnmd_status nnmd_b200_compute(nnmd_b200* h, int64_t n, const double* coords, const int32_t* types,
                              const int64_t* gids, const double box[3], const uint8_t periodic[3],
                              double* energy, double* forces, double* virial, double* atom_energy) {
  return guarded([&] {
    // coords may be NULL on world ranks > 0 (positions arrive by the collective-1 broadcast)
    nb::require(box && (n == 0 || types), "nnmd_b200_compute: null argument");
    const uint8_t per_default[3] = {1, 1, 1};
    C(h).compute_host(n, coords, types, gids, box, periodic ? periodic : per_default, energy, forces,
                      virial, atom_energy);
  });
}

void nnmd_b200_set_trace(nnmd_b200* h, int spans, int ledger) {
  if (h && h->ctx) h->ctx->set_trace(spans != 0, ledger != 0);
}

void nnmd_b200_set_step(nnmd_b200* h, long step) {
  if (h && h->ctx) h->ctx->set_step(step);
}

int nnmd_b200_trace_spans(const nnmd_b200* h, nnmd_span* out, int cap) {
  if (!h || !h->ctx) return 0;
  const auto& v = h->ctx->spans();
  for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i)
    out[i] = nnmd_span{v[static_cast<size_t>(i)].rank, v[static_cast<size_t>(i)].phase, v[static_cast<size_t>(i)].t0,
                       v[static_cast<size_t>(i)].t1, v[static_cast<size_t>(i)].step};
  return static_cast<int>(v.size());
}

int nnmd_b200_ledger(const nnmd_b200* h, nnmd_collective_record* out, int cap) {
  if (!h || !h->ctx) return 0;
  const auto& v = h->ctx->ledger();
  for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i)
    out[i] = nnmd_collective_record{v[static_cast<size_t>(i)].step, v[static_cast<size_t>(i)].kind,
                                    v[static_cast<size_t>(i)].bytes, v[static_cast<size_t>(i)].participants};
  return static_cast<int>(v.size());
}

void nnmd_b200_trace_clear(nnmd_b200* h) {
  if (h && h->ctx) h->ctx->clear_trace();
}

nnmd_status nnmd_b200_export_chrome_trace(const nnmd_b200* h, const char* path) {
  return guarded([&] {
    nb::require(h && h->ctx && path, "nnmd_b200_export_chrome_trace: null argument");
    h->ctx->export_chrome_trace(path);
  });
}

static nb::Context::MdConfig md_cfg(const nnmd_md_config* c) {
  nb::require(c != nullptr, "nnmd_b200_run_md: null config");
  return nb::Context::MdConfig{c->dt, c->n_steps, c->equil_steps, c->target_temperature, c->rescale_every};
}

nnmd_status nnmd_b200_run_md(nnmd_b200* h, int64_t n, double* coords, double* velocities, const double* masses,
                             const int32_t* types, const int64_t* gids, const double box[3],
                             const uint8_t periodic[3], const nnmd_md_config* cfg, double* potential,
                             double* total) {
  return guarded([&] {
    nb::require(box && (n == 0 || (coords && velocities && masses && types)), "nnmd_b200_run_md: null argument");
    const uint8_t per_default[3] = {1, 1, 1};
    C(h).run_md_host(n, coords, velocities, masses, types, gids, box, periodic ? periodic : per_default,
                     md_cfg(cfg), potential, total);
  });
}

nnmd_status nnmd_b200_run_md_device(nnmd_b200* h, int64_t n, double* d_coords, double* d_velocities,
                                    const double* d_masses, const int32_t* d_types, const int64_t* d_gids,
                                    const double box[3], const uint8_t periodic[3], const nnmd_md_config* cfg,
                                    double* d_energies) {
  return guarded([&] {
    nb::require(box && d_gids && d_energies && (n == 0 || (d_coords && d_velocities && d_masses && d_types)),
                "nnmd_b200_run_md_device: null argument");
    const uint8_t per_default[3] = {1, 1, 1};
    C(h).run_md(n, d_coords, d_velocities, d_masses, d_types, d_gids, box, periodic ? periodic : per_default,
                md_cfg(cfg), d_energies);
  });
}

nnmd_status nnmd_b200_compute_device(nnmd_b200* h, int64_t n, const double* d_coords,
                                     const int32_t* d_types, const int64_t* d_gids,
                                     const double box[3], const uint8_t periodic[3], double* d_out) {
  return guarded([&] {
    nb::require(box && d_out && d_gids && (n == 0 || (d_coords && d_types)),
                "nnmd_b200_compute_device: null argument");
    const uint8_t per_default[3] = {1, 1, 1};
    C(h).compute_device(n, d_coords, d_types, d_gids, box, periodic ? periodic : per_default, d_out);
  });
}

nnmd_status nnmd_b200_rank_stats(const nnmd_b200* h, int rank, int64_t counts[4], double ms[4]) {
  return guarded([&] {
    nb::require(h && h->ctx, "nnmd_b200: null context");
    const nb::RankStat& s = h->ctx->stat(rank);
    for (int i = 0; i < 4; ++i) {
      if (counts) counts[i] = s.counts[i];
      if (ms) ms[i] = s.ms[i];
    }
  });
}

int nnmd_b200_kernel_times(const nnmd_b200* h, const char** names, double* ms, int cap) {
  if (!h || !h->ctx) return 0;
  static thread_local std::vector<std::pair<std::string, double>> keep;
  keep = h->ctx->kernel_times();
  int k = 0;
  for (; k < static_cast<int>(keep.size()) && k < cap; ++k) {
    if (names) names[k] = keep[static_cast<size_t>(k)].first.c_str();
    if (ms) ms[k] = keep[static_cast<size_t>(k)].second;
  }
  return names || ms ? k : static_cast<int>(keep.size());
}

nnmd_status nnmd_b200_debug_nlist(const nnmd_b200* h, int rank, int* n_centres,
                                  int32_t* centre_atoms, int32_t* idx, int32_t* img,
                                  int32_t* counts) {
  return guarded([&] {
    nb::require(h && h->ctx && n_centres, "nnmd_b200_debug_nlist: null argument");
    nb::RankDebug d;
    h->ctx->debug_rank(rank, d);
    *n_centres = static_cast<int>(d.centre_atoms.size());
    if (centre_atoms) std::memcpy(centre_atoms, d.centre_atoms.data(), d.centre_atoms.size() * sizeof(int));
    if (idx) std::memcpy(idx, d.nlist_atom.data(), d.nlist_atom.size() * sizeof(int));
    if (img) std::memcpy(img, d.nlist_img.data(), d.nlist_img.size() * sizeof(int));
    if (counts) std::memcpy(counts, d.nn.data(), d.nn.size() * sizeof(int));
  });
}

nnmd_status nnmd_b200_debug_ghosts(const nnmd_b200* h, int rank, int* n_ghosts, int32_t* atom,
                                   int32_t* owner, int32_t* shift) {
  return guarded([&] {
    nb::require(h && h->ctx && n_ghosts, "nnmd_b200_debug_ghosts: null argument");
    nb::RankDebug d;
    h->ctx->debug_rank(rank, d);
    *n_ghosts = static_cast<int>(d.ghost_atom.size());
    if (atom) std::memcpy(atom, d.ghost_atom.data(), d.ghost_atom.size() * sizeof(int));
    if (owner) std::memcpy(owner, d.ghost_owner.data(), d.ghost_owner.size() * sizeof(int));
    if (shift) std::memcpy(shift, d.ghost_shift.data(), d.ghost_shift.size() * sizeof(int));
  });
}

void nnmd_b200_set_debug(nnmd_b200* h, int on) {
  if (h && h->ctx) h->ctx->set_keep_debug(on);
}

void* nnmd_b200_stream(const nnmd_b200* h) { return h && h->ctx ? static_cast<void*>(h->ctx->stream()) : nullptr; }

nnmd_status nnmd_synth_system(int64_t n, double rho, double min_sep, uint64_t seed, double box[3],
                              double* coords, int32_t* types) {
  return guarded([&] { nb::synth_system(n, rho, min_sep, seed, box, coords, types); });
}

}  // extern "C"

extern "C" long long nnmd_b200_launch_count(void) { return nb::launch_count(); }

extern "C" nnmd_status nnmd_b200_selftest_gemm(int mode, int ta, int tb, int M, int N, int K, const float* A,
                                               const float* B, float* C) {
  return guarded([&] {
    nb::require(M >= 0 && N >= 0 && K >= 0 && mode >= 0 && mode <= 2, "selftest_gemm: bad arguments");
    const int ra = ta ? K : M, ca = ta ? M : K, rb = tb ? N : K, cb = tb ? K : N;  // host row-major shapes
    const int lda = (ca + 3) & ~3, ldb = (cb + 3) & ~3;                         // 16-byte aligned rows
    float *dA = nullptr, *dB = nullptr, *dC = nullptr;
    auto chk = [](cudaError_t e) {
      if (e != cudaSuccess) throw nb::CudaError(std::string("selftest_gemm: ") + cudaGetErrorString(e));
    };
    chk(cudaMalloc(&dA, sizeof(float) * (static_cast<size_t>(ra) * lda + 4)));
    chk(cudaMalloc(&dB, sizeof(float) * (static_cast<size_t>(rb) * ldb + 4)));
    chk(cudaMalloc(&dC, sizeof(float) * (static_cast<size_t>(M) * N + 1)));
    chk(cudaMemset(dA, 0, sizeof(float) * (static_cast<size_t>(ra) * lda + 4)));
    chk(cudaMemset(dB, 0, sizeof(float) * (static_cast<size_t>(rb) * ldb + 4)));
    if (ra && ca) chk(cudaMemcpy2D(dA, lda * sizeof(float), A, ca * sizeof(float), ca * sizeof(float), ra, cudaMemcpyHostToDevice));
    if (rb && cb) chk(cudaMemcpy2D(dB, ldb * sizeof(float), B, cb * sizeof(float), cb * sizeof(float), rb, cudaMemcpyHostToDevice));
    chk(cudaMemset(dC, 0, sizeof(float) * static_cast<size_t>(M) * N));
    nb::selftest_gemm(mode, ta, tb, M, N, K, dA, lda, dB, ldb, dC);
    chk(cudaGetLastError());
    chk(cudaDeviceSynchronize());
    chk(cudaMemcpy(C, dC, sizeof(float) * static_cast<size_t>(M) * N, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
  });
}
