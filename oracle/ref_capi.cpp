// C-ABI shim over the UNMODIFIED reference library (test infrastructure only).
//
// Compiled by oracle/Makefile against /root/reference/proj headers and linked with the
// reference's own objects into oracle/_ref/libnnmd_ref.so.  Every entry point calls the
// reference's PUBLIC API; nothing here re-implements reference arithmetic except the
// virial, which the reference does not have: W_ab = -sum_c sum_k
// g_{k,a} d_{k,b} assembled from the public per-centre row gradients
// (deeppot.hpp:169-189 CenterGrads::row_grads, EnvRow::d).
//
// Used by tests/ (golden-vector generation and pinning of oracle/dp_oracle.cpp) and by
// bench.py's reference arm / cpu_baseline leg.  Never by the product path.

#include <atomic>
#include <map>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "nnmd/analysis.hpp"
#include "nnmd/decomp.hpp"
#include "nnmd/deeppot.hpp"
#include "nnmd/engine.hpp"
#include "nnmd/neighbor.hpp"
#include "nnmd/system.hpp"
#include "support.hpp"  // proj/tests/support.hpp: random_config, test_model

using namespace nnmd;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const CapacityError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

AtomSet make_atoms(int n, const double* pos, const int* species, const int64_t* gids) {
  AtomSet a;
  for (int i = 0; i < n; ++i)
    a.push_back(gids ? gids[i] : i, species[i], {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]});
  return a;
}

SimBox make_box(const double* box3, const uint8_t* periodic) {
  SimBox b;
  b.lengths = {box3[0], box3[1], box3[2]};
  if (periodic)
    b.periodic = {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0};
  return b;
}

DPModel& M(void* h) { return *static_cast<DPModel*>(h); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_model_init(double rc, double rcs, int n_max, int n_species, int type_dim,
                     int n_feat, int n_reduced, int n_attn, int attn_dim,
                     const int* embed_hidden, int n_embed_hidden, const int* fit_hidden,
                     int n_fit_hidden, uint64_t seed) {
  DPModel* out = nullptr;
  int rc_ = guarded([&] {
    ModelSpec s;
    s.rc = rc;
    s.rcs = rcs;
    s.n_max = n_max;
    s.n_species = n_species;
    s.type_dim = type_dim;
    s.n_feat = n_feat;
    s.n_reduced = n_reduced;
    s.n_attn = n_attn;
    s.attn_dim = attn_dim;
    s.embed_hidden.assign(embed_hidden, embed_hidden + n_embed_hidden);
    s.fit_hidden.assign(fit_hidden, fit_hidden + n_fit_hidden);
    out = new DPModel(init_model(s, seed));
  });
  return rc_ == 0 ? out : nullptr;
}

void* ref_model_load(const char* path) {
  DPModel* out = nullptr;
  int rc = guarded([&] { out = new DPModel(load_model(path)); });
  return rc == 0 ? out : nullptr;
}

int ref_model_save(void* m, const char* path) {
  return guarded([&] { save_model(M(m), path); });
}

void ref_model_free(void* m) { delete static_cast<DPModel*>(m); }

long ref_model_nparams(void* m) { return static_cast<long>(M(m).n_params()); }

void ref_model_set_nmax(void* m, int n_max) { M(m).n_max = n_max; }

// tests/support.hpp random_config (the reference's own test-configuration generator)
int ref_random_config(uint64_t seed, int n, double density, int n_species, double min_sep,
                      double* box3, double* pos, int* species) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    auto cfg = testing::random_config(rng, n, density, n_species, min_sep);
    for (int a = 0; a < 3; ++a) box3[a] = cfg.box.lengths[a];
    for (int i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) pos[3 * i + a] = cfg.atoms.positions[i][a];
      species[i] = cfg.atoms.species[i];
    }
  });
}

// The acceptance/test_decomp make_dd_case generator (acceptance.cpp:36-43):
// returns n through *n_out (capacity 256), box, positions, species and rc.
int ref_make_dd_case(uint64_t seed, double* box3, double* pos, int* species, int* n_out,
                     double* rc_out) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int> un(160, 256);
    std::uniform_real_distribution<double> urho(0.45, 0.6);
    const int n = un(rng);
    const double rho = urho(rng);
    auto cfg = testing::random_config(rng, n, rho, 3, 0.5);
    for (int a = 0; a < 3; ++a) box3[a] = cfg.box.lengths[a];
    for (int i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) pos[3 * i + a] = cfg.atoms.positions[i][a];
      species[i] = cfg.atoms.species[i];
    }
    *n_out = n;
    *rc_out = cfg.box.lengths.x / 6.2;
  });
}

// Single-domain evaluation (engine.cpp:79-87 path): build_neighbor_list + evaluate_dp.
// virial (9, row-major W[a][b]) is assembled from the public per-centre row gradients.
int ref_evaluate_dp(void* m, int n, const double* pos, const int* species,
                    const int64_t* gids, const double* box3, const uint8_t* periodic,
                    double* energy, double* forces, double* atom_energy, double* virial) {
  return guarded([&] {
    const DPModel& model = M(m);
    AtomSet atoms = make_atoms(n, pos, species, gids);
    SimBox box = make_box(box3, periodic);
    const NeighborList list = build_neighbor_list(atoms, box, model.rc, ListMode::full);
    const DpResult res = evaluate_dp(atoms, box, list, model);
    *energy = res.energy;
    for (int i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) forces[3 * i + a] = res.forces[i][a];
      if (atom_energy) atom_energy[i] = res.atom_energy[i];
    }
    if (virial) {
      double w[9] = {0};
      auto ws = new_workspace();
      for (int i = 0; i < n; ++i) {
        const auto rows = center_rows(i, list, atoms, box, model);
        const CenterGrads cg = evaluate_center(model, atoms.species[i], rows, *ws, true);
        for (std::size_t k = 0; k < rows.size(); ++k)
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) w[3 * a + b] -= cg.row_grads[k][a] * rows[k].d[b];
      }
      std::memcpy(virial, w, sizeof w);
    }
  });
}

// Canonical sorted rows of every centre (deeppot.cpp:150-184 center_rows).
// Flat output in centre order; counts[n]; capacity cap rows total.
int ref_center_rows(void* m, int n, const double* pos, const int* species,
                    const int64_t* gids, const double* box3, const uint8_t* periodic,
                    long cap, int* counts, int* member, int* image, double* d, long* total) {
  return guarded([&] {
    const DPModel& model = M(m);
    AtomSet atoms = make_atoms(n, pos, species, gids);
    SimBox box = make_box(box3, periodic);
    const NeighborList list = build_neighbor_list(atoms, box, model.rc, ListMode::full);
    long t = 0;
    for (int i = 0; i < n; ++i) {
      const auto rows = center_rows(i, list, atoms, box, model);
      counts[i] = static_cast<int>(rows.size());
      for (const auto& r : rows) {
        require(t < cap, "ref_center_rows: capacity");
        member[t] = r.member;
        for (int a = 0; a < 3; ++a) {
          image[3 * t + a] = r.image[a];
          d[3 * t + a] = r.d[a];
        }
        ++t;
      }
    }
    *total = t;
  });
}

// Per-centre energy + row gradients for one centre from explicit rows (testing hook).
int ref_evaluate_center_rows(void* m, int center_species, int n_rows, const double* d,
                             const int* row_species, double* energy, double* row_grads) {
  return guarded([&] {
    std::vector<EnvRow> rows(static_cast<std::size_t>(n_rows));
    for (int k = 0; k < n_rows; ++k) {
      rows[k].d = {d[3 * k], d[3 * k + 1], d[3 * k + 2]};
      rows[k].species = row_species[k];
    }
    auto ws = new_workspace();
    const CenterGrads cg = evaluate_center(M(m), center_species, rows, *ws, true);
    *energy = cg.energy;
    for (int k = 0; k < n_rows; ++k)
      for (int a = 0; a < 3; ++a) row_grads[3 * k + a] = cg.row_grads[k][a];
  });
}

int ref_partition_ranks(const double* box3, int n_ranks, double min_edge, int* dims) {
  return guarded([&] {
    SimBox box = make_box(box3, nullptr);
    const RankGrid g = partition_ranks(box, n_ranks, min_edge);
    for (int a = 0; a < 3; ++a) dims[a] = g.dims[a];
  });
}

// owner_rank_of for all atoms (decomp.cpp:59-68)
int ref_owner_ranks(int n, const double* pos, const double* box3, const int* dims, int* owner) {
  return guarded([&] {
    SimBox box = make_box(box3, nullptr);
    RankGrid g{{dims[0], dims[1], dims[2]}};
    for (int i = 0; i < n; ++i)
      owner[i] = owner_rank_of({pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}, g, box);
  });
}

// build_halo (decomp.cpp:96-131) for one rank; ghosts in (atom, shift) order.
int ref_build_halo(int n, const double* pos, const double* box3, const uint8_t* periodic,
                   const int* dims, int rank, double thickness, long cap, int* atom,
                   int* owner_out, int* shift, long* n_out) {
  return guarded([&] {
    AtomSet atoms = make_atoms(n, pos, std::vector<int>(n, 0).data(), nullptr);
    SimBox box = make_box(box3, periodic);
    RankGrid g{{dims[0], dims[1], dims[2]}};
    std::vector<int> owner(n);
    for (int i = 0; i < n; ++i) owner[i] = owner_rank_of(atoms.positions[i], g, box);
    Subdomain sub = make_subdomain(g, rank, box);
    const auto ghosts = build_halo(atoms, sub, thickness, box, owner);
    require(static_cast<long>(ghosts.size()) <= cap, "ref_build_halo: capacity");
    for (std::size_t k = 0; k < ghosts.size(); ++k) {
      atom[k] = ghosts[k].atom;
      owner_out[k] = ghosts[k].owner_rank;
      for (int a = 0; a < 3; ++a) shift[3 * k + a] = ghosts[k].shift[a];
    }
    *n_out = static_cast<long>(ghosts.size());
  });
}

// dd_evaluate (decomp.cpp:265-542).  stats: per rank {locals, ghosts, centers, route}.
int ref_dd_evaluate(void* m, int n, const double* pos, const int* species,
                    const int64_t* gids, const double* box3, const uint8_t* periodic,
                    int n_ranks, int scheme, int workers, double* energy, double* forces,
                    double* atom_energy, int* grid_dims, long* stats) {
  return guarded([&] {
    AtomSet atoms = make_atoms(n, pos, species, gids);
    SimBox box = make_box(box3, periodic);
    const DdResult res =
        dd_evaluate(atoms, box, M(m), n_ranks,
                    scheme == 0 ? DdScheme::masked_reduction : DdScheme::wide_halo, workers);
    *energy = res.energy;
    for (int i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) forces[3 * i + a] = res.forces[i][a];
      if (atom_energy) atom_energy[i] = res.atom_energy[i];
    }
    if (grid_dims)
      for (int a = 0; a < 3; ++a) grid_dims[a] = res.grid.dims[a];
    if (stats)
      for (std::size_t r = 0; r < res.stats.size(); ++r) {
        stats[4 * r + 0] = res.stats[r].locals;
        stats[4 * r + 1] = res.stats[r].ghosts;
        stats[4 * r + 2] = res.stats[r].centers;
        stats[4 * r + 3] = static_cast<long>(res.stats[r].route_entries);
      }
  });
}

// Bounded CPU-baseline sample: the reference full neighbour list once, then
// center_rows + evaluate_center (fwd + exact bwd) for the listed centres on `workers`
// host threads (run_rank_tasks-style atomic work counter, decomp.cpp:233-256).
// Returns seconds for the list build and for the centre sample separately.
int ref_time_centers(void* m, int n, const double* pos, const int* species,
                     const int64_t* gids, const double* box3, const uint8_t* periodic,
                     const int* centers, int n_centers, int workers, double* t_list,
                     double* t_centers, double* energy_sum) {
  return guarded([&] {
    const DPModel& model = M(m);
    AtomSet atoms = make_atoms(n, pos, species, gids);
    SimBox box = make_box(box3, periodic);
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const NeighborList list = build_neighbor_list(atoms, box, model.rc, ListMode::full);
    const auto t1 = clk::now();
    std::atomic<int> next{0};
    std::vector<double> esum(static_cast<std::size_t>(std::max(workers, 1)), 0.0);
    std::vector<std::exception_ptr> errs(esum.size());
    std::vector<std::thread> pool;
    for (int w = 0; w < std::max(workers, 1); ++w)
      pool.emplace_back([&, w] {
        try {
          auto ws = new_workspace();
          for (int k = next.fetch_add(1); k < n_centers; k = next.fetch_add(1)) {
            const int c = centers[k];
            const auto rows = center_rows(c, list, atoms, box, model);
            esum[w] += evaluate_center(model, atoms.species[c], rows, *ws, true).energy;
          }
        } catch (...) {
          errs[w] = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    const auto t2 = clk::now();
    *t_list = std::chrono::duration<double>(t1 - t0).count();
    *t_centers = std::chrono::duration<double>(t2 - t1).count();
    double s = 0;
    for (double e : esum) s += e;
    *energy_sum = s;
  });
}

// evaluate_dp (deeppot.cpp:315-369) with the per-centre work spread over `workers` host
// threads: each thread runs the public center_rows + evaluate_center on an interleaved
// share of the centres; the force assembly then replays evaluate_dp's loop order
// (ForceAccumulator adds in ascending centre order, deeppot.cpp:351-362) so E, F and e_i
// are bitwise identical to the single-threaded evaluate_dp.  The virial is
// summed in the same centre order.  Golden-vector generation for the big configs only.
int ref_evaluate_dp_mt(void* m, int n, const double* pos, const int* species,
                       const int64_t* gids, const double* box3, const uint8_t* periodic,
                       int workers, double* energy, double* forces, double* atom_energy,
                       double* virial) {
  return guarded([&] {
    const DPModel& model = M(m);
    model.validate();
    AtomSet atoms = make_atoms(n, pos, species, gids);
    SimBox box = make_box(box3, periodic);
    box.validate(model.rc);
    const NeighborList list = build_neighbor_list(atoms, box, model.rc, ListMode::full);
    std::vector<std::vector<EnvRow>> rows(static_cast<std::size_t>(n));
    std::vector<CenterGrads> cgs(static_cast<std::size_t>(n));
    std::atomic<int> next{0};
    const int nw = std::max(workers, 1);
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(nw));
    std::vector<std::thread> pool;
    for (int w = 0; w < nw; ++w)
      pool.emplace_back([&, w] {
        try {
          auto ws = new_workspace();
          for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
            rows[i] = center_rows(i, list, atoms, box, model);
            cgs[i] = evaluate_center(model, atoms.species[i], rows[i], *ws, true);
          }
        } catch (...) {
          errs[w] = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    ForceAccumulator acc(static_cast<std::size_t>(n));
    double e = 0.0, w9[9] = {0};
    for (int i = 0; i < n; ++i) {
      const CenterGrads& cg = cgs[i];
      if (atom_energy) atom_energy[i] = cg.energy;
      e += cg.energy;
      acc.add(i, kZeroShift, cg.center_grad);
      for (std::size_t k = 0; k < rows[i].size(); ++k) {
        acc.add(rows[i][k].member, rows[i][k].image, cg.row_grads[k]);
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) w9[3 * a + b] -= cg.row_grads[k][a] * rows[i][k].d[b];
      }
    }
    const auto f = acc.finalize();
    *energy = e;
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) forces[3 * i + a] = f[i][a];
    if (virial) std::memcpy(virial, w9, sizeof w9);
  });
}

// Reference-arm step slice (bench.py --impl reference): the reference's own per-step
// work for the centres [c0, c1) -- build_neighbor_list (neighbor.cpp:73-148), then the
// stock evaluate_dp (deeppot.cpp:315-369) with a LocalMask selecting that slice, split
// over `workers` host threads (one evaluate_dp call per thread on an equal sub-slice,
// like run_rank_tasks' per-rank threads, decomp.cpp:233-256) and the per-thread force
// arrays summed.  Seconds for the list build and for the evaluation are returned apart
// so a full step = one list build + the K slices that tile [0, n).
int ref_step_slice(void* m, int n, const double* pos, const int* species,
                   const int64_t* gids, const double* box3, const uint8_t* periodic,
                   int c0, int c1, int workers, double* t_list, double* t_eval,
                   double* energy_sum) {
  return guarded([&] {
    const DPModel& model = M(m);
    AtomSet atoms = make_atoms(n, pos, species, gids);
    SimBox box = make_box(box3, periodic);
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const NeighborList list = build_neighbor_list(atoms, box, model.rc, ListMode::full);
    const auto t1 = clk::now();
    require(0 <= c0 && c0 < c1 && c1 <= n, "ref_step_slice: bad centre range");
    const int nw = std::max(1, std::min(workers, c1 - c0));
    std::vector<DpResult> res(static_cast<std::size_t>(nw));
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(nw));
    std::vector<std::thread> pool;
    for (int w = 0; w < nw; ++w)
      pool.emplace_back([&, w] {
        try {
          const long span = c1 - c0;
          const int a = c0 + static_cast<int>(span * w / nw), b = c0 + static_cast<int>(span * (w + 1) / nw);
          LocalMask mask;
          mask.owned.assign(static_cast<std::size_t>(n), 0);
          for (int i = a; i < b; ++i) mask.owned[i] = 1;
          res[w] = evaluate_dp(atoms, box, list, model, &mask);
        } catch (...) {
          errs[w] = std::current_exception();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    std::vector<Vec3> f(static_cast<std::size_t>(n));
    double e = 0.0;
    for (const auto& r : res) {
      e += r.energy;
      for (int i = 0; i < n; ++i) f[i] += r.forces[i];
    }
    const auto t2 = clk::now();
    *t_list = std::chrono::duration<double>(t1 - t0).count();
    *t_eval = std::chrono::duration<double>(t2 - t1).count();
    *energy_sum = e;
  });
}

// analysis.cpp:148-208 -- the Eq. 8 throughput model and the scaling efficiencies, for
// pinning the sweep harness (paper_2604_07276_b200/sweep.py).
int ref_fit_throughput(int n, const double* n_p, const double* tr, double* alpha, double* beta,
                       double* r2, double* residuals) {
  return guarded([&] {
    std::vector<std::pair<double, double>> pts;
    for (int i = 0; i < n; ++i) pts.emplace_back(n_p[i], tr[i]);
    const ScalingFit f = fit_throughput(pts);
    *alpha = f.alpha;
    *beta = f.beta;
    *r2 = f.r_squared;
    for (std::size_t i = 0; i < f.residuals.size(); ++i) residuals[i] = f.residuals[i];
  });
}

int ref_predict_throughput(double alpha, double beta, double n_p, double* out) {
  return guarded([&] { *out = predict_throughput(alpha, beta, n_p); });
}

int ref_scaling_efficiency(int n, const int* n_p, const double* tr, int reference, int weak, double* eff) {
  return guarded([&] {
    std::map<int, double> m;
    for (int i = 0; i < n; ++i) m[n_p[i]] = tr[i];
    const auto e = scaling_efficiency(m, reference, weak != 0);
    for (int i = 0; i < n; ++i) eff[i] = e.at(n_p[i]);
  });
}

int ref_throughput_per_day(long n_steps, double dt, double elapsed, double* out) {
  return guarded([&] { *out = throughput_per_day(n_steps, dt, elapsed); });
}

// tests/support.hpp fd_force_component: central FD of the total DP energy.
int ref_fd_force_component(void* m, int n, const double* pos, const int* species,
                           const int64_t* gids, const double* box3, const uint8_t* periodic,
                           int atom, int comp, double h, double* out) {
  return guarded([&] {
    AtomSet atoms = make_atoms(n, pos, species, gids);
    SimBox box = make_box(box3, periodic);
    *out = testing::fd_force_component(atoms, box, M(m), static_cast<std::size_t>(atom),
                                       comp, h);
  });
}

}  // extern "C"
