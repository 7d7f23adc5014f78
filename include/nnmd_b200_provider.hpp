// GpuDpProvider -- drop-in nnmd::ForceProvider backed by the B200 library.
//
// This header is meant to be added to the reference tree (next to
// proj/include/nnmd/engine.hpp) and compiled against it; it needs the nnmd headers and
// links libnnmd_b200.so.  It mirrors nnmd::DpProvider (engine.hpp:51-74,
// engine.cpp:54-89): same Options, the same NN-atom group mask and species map, the
// same result (energy + per-atom forces of the full system), the same exception
// classes (CapacityError for neighbour overflow, Error otherwise).  The virial of the
// last evaluation is available through last_virial().
#pragma once

#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "nnmd/deeppot.hpp"
#include "nnmd/engine.hpp"
#include "nnmd_b200.h"

namespace nnmd {

class GpuDpProvider : public ForceProvider {
 public:
  struct Options {
    bool decomposed = false;
    DdScheme scheme = DdScheme::wide_halo;
    int n_ranks = 1;            // DD ranks (all on this GPU when world_size == 1)
    int device = 0;
    int precision = NNMD_PREC_FP32;
    std::vector<int> species_map;  // system species -> model species; empty = identity
    int world_size = 1;         // processes (one per GPU) sharing the DD ranks
    int world_rank = 0;
    const void* nccl_id = nullptr;
  };

  GpuDpProvider(const DPModel& model, Options opts, std::vector<std::uint8_t> group_mask = {})
      : opts_(std::move(opts)), group_(std::move(group_mask)) {
    // hand the model over in its own file format (deeppot_io.cpp) -- bit-exact
    char path[] = "/tmp/nnmd_b200_model_XXXXXX";
    const int fd = mkstemp(path);
    require(fd >= 0, "GpuDpProvider: cannot create a temporary model file");
    close(fd);
    save_model(model, path);
    nnmd_model* m = nullptr;
    const nnmd_status st = nnmd_model_load(path, &m);
    std::remove(path);
    check(st);
    nnmd_b200_opts o{};
    o.n_ranks = opts_.decomposed ? opts_.n_ranks : 1;
    o.scheme = (opts_.decomposed && opts_.scheme == DdScheme::wide_halo) ? NNMD_WIDE_HALO : NNMD_MASKED_REDUCTION;
    o.precision = opts_.precision;
    o.device = opts_.device;
    o.world_size = opts_.world_size;
    o.world_rank = opts_.world_rank;
    o.nccl_id = opts_.nccl_id;
    const nnmd_status cs = nnmd_b200_create(m, &o, &ctx_);
    nnmd_model_free(m);
    check(cs);
  }

  ~GpuDpProvider() override { nnmd_b200_destroy(ctx_); }
  GpuDpProvider(const GpuDpProvider&) = delete;
  GpuDpProvider& operator=(const GpuDpProvider&) = delete;

  std::string name() const override { return opts_.decomposed ? "dp_dd_b200" : "dp_single_b200"; }

  ProviderResult evaluate(const AtomSet& atoms, const SimBox& box, StepContext& ctx) override {
    idx_.clear();
    pos_.clear();
    sp_.clear();
    gid_.clear();
    for (std::size_t i = 0; i < atoms.size(); ++i) {
      if (!group_.empty() && !group_[i]) continue;
      int z = atoms.species[i];
      if (!opts_.species_map.empty()) {
        require(z >= 0 && z < static_cast<int>(opts_.species_map.size()),
                "DpProvider: species outside the species map");
        z = opts_.species_map[static_cast<std::size_t>(z)];
      }
      idx_.push_back(static_cast<int>(i));
      for (int a = 0; a < 3; ++a) pos_.push_back(atoms.positions[i][a]);
      sp_.push_back(z);
      gid_.push_back(atoms.global_ids[i]);
    }
    ProviderResult out;
    out.forces.assign(atoms.size(), Vec3{});
    if (idx_.empty()) return out;
    const double L[3] = {box.lengths.x, box.lengths.y, box.lengths.z};
    const std::uint8_t per[3] = {box.periodic[0], box.periodic[1], box.periodic[2]};
    f_.assign(3 * idx_.size(), 0.0);
    // the run's TraceSink / CollectiveLedger get the same spans and records the reference
    // writes (dd_evaluate, decomp.cpp:285-538; single domain: one rank-0 inference span,
    // engine.cpp:79), measured on the device
    nnmd_b200_set_trace(ctx_, ctx.trace != nullptr, ctx.ledger != nullptr && opts_.decomposed);
    nnmd_b200_set_step(ctx_, ctx.step);
    check(nnmd_b200_compute(ctx_, static_cast<std::int64_t>(idx_.size()), pos_.data(), sp_.data(),
                            gid_.data(), L, per, &out.energy, f_.data(), virial_, nullptr));
    if (ctx.trace) {
      std::vector<nnmd_span> sp(static_cast<std::size_t>(nnmd_b200_trace_spans(ctx_, nullptr, 0)));
      nnmd_b200_trace_spans(ctx_, sp.data(), static_cast<int>(sp.size()));
      if (opts_.decomposed) {
        for (const auto& s : sp) ctx.trace->record_span(s.rank, static_cast<Phase>(s.phase), s.t_start, s.t_end, s.step);
      } else if (!sp.empty()) {
        double t0 = sp.front().t_start, t1 = sp.front().t_end;
        for (const auto& s : sp) {
          t0 = std::min(t0, s.t_start);
          t1 = std::max(t1, s.t_end);
        }
        ctx.trace->record_span(0, Phase::inference, t0, t1, ctx.step);
      }
    }
    if (ctx.ledger && opts_.decomposed) {
      std::vector<nnmd_collective_record> lr(static_cast<std::size_t>(nnmd_b200_ledger(ctx_, nullptr, 0)));
      nnmd_b200_ledger(ctx_, lr.data(), static_cast<int>(lr.size()));
      for (const auto& r : lr) ctx.ledger->add(r.step, static_cast<CollectiveKind>(r.kind), r.bytes, r.participants);
    }
    nnmd_b200_trace_clear(ctx_);
    for (std::size_t k = 0; k < idx_.size(); ++k)
      out.forces[static_cast<std::size_t>(idx_[k])] = {f_[3 * k], f_[3 * k + 1], f_[3 * k + 2]};
    return out;
  }

  const double* last_virial() const { return virial_; }

  // Device-resident variant of nnmd::run_md (engine.cpp:143-211) for this provider alone:
  // positions and velocities stay on the GPU for all n_steps (one copy in, one copy out),
  // the leap-frog step runs as a kernel.  Same RunSummary fields (potential_energy,
  // total_energy, elapsed_seconds, throughput); trajectory output is not written.
  RunSummary run_md(AtomSet& atoms, const SimBox& box, const MDConfig& config) {
    require(config.dt > 0.0, "run_md: dt must be > 0");
    require(config.n_steps >= 0, "run_md: n_steps must be >= 0");
    require(group_.empty() && opts_.species_map.empty(),
            "GpuDpProvider::run_md: group masks and species maps need nnmd::run_md");
    atoms.validate();
    const std::size_t n = atoms.size();
    std::vector<double> x(3 * n), v(3 * n);
    std::vector<std::int32_t> sp(n);
    for (std::size_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        x[3 * i + a] = atoms.positions[i][a];
        v[3 * i + a] = atoms.velocities[i][a];
      }
      sp[i] = atoms.species[i];
    }
    const double L[3] = {box.lengths.x, box.lengths.y, box.lengths.z};
    const std::uint8_t per[3] = {box.periodic[0], box.periodic[1], box.periodic[2]};
    nnmd_md_config c{config.dt, config.n_steps, config.equil_steps, config.target_temperature,
                     config.rescale_every};
    RunSummary s;
    s.dt = config.dt;
    s.potential_energy.resize(static_cast<std::size_t>(config.n_steps));
    s.total_energy.resize(static_cast<std::size_t>(config.n_steps));
    const double t0 = TraceSink::now();
    check(nnmd_b200_run_md(ctx_, static_cast<std::int64_t>(n), x.data(), v.data(), atoms.masses.data(), sp.data(),
                           atoms.global_ids.data(), L, per, &c, s.potential_energy.data(), s.total_energy.data()));
    s.elapsed_seconds = TraceSink::now() - t0;
    s.steps = config.n_steps;
    if (s.steps > 0 && s.elapsed_seconds > 0) s.throughput = throughput_per_day(s.steps, s.dt, s.elapsed_seconds);
    for (std::size_t i = 0; i < n; ++i) {
      atoms.positions[i] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
      atoms.velocities[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    }
    return s;
  }

 private:
  static void check(nnmd_status st) {
    if (st == NNMD_OK) return;
    const std::string msg = nnmd_b200_last_error();
    if (st == NNMD_CAPACITY) throw CapacityError(msg);
    throw Error(st == NNMD_CUDA ? "nnmd_b200 (CUDA/NCCL): " + msg : msg);
  }

  Options opts_;
  std::vector<std::uint8_t> group_;
  nnmd_b200* ctx_ = nullptr;
  std::vector<int> idx_;
  std::vector<double> pos_, f_;
  std::vector<std::int32_t> sp_;
  std::vector<std::int64_t> gid_;
  double virial_[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
};

}  // namespace nnmd
