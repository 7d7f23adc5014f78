// Integration check (test infrastructure): the reference's own MD loop driven by the
// reference DpProvider and by the drop-in GpuDpProvider (include/nnmd_b200_provider.hpp).
//
// Built by `make -C oracle integration` against the UNMODIFIED reference headers and
// objects, linked with libnnmd_b200.so.  Runs nnmd::run_md (engine.cpp:143-211) for a few
// leap-frog steps on a small random configuration with the paper-shaped model (reduced
// widths so the CPU side finishes in seconds) and prints one JSON line comparing the
// per-step potential energies and the final positions of the two trajectories.
#include <cmath>
#include <cstdio>
#include <random>
#include <set>
#include <tuple>

#include "nnmd/engine.hpp"
#include "nnmd_b200_provider.hpp"
#include "support.hpp"

using namespace nnmd;

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 5;
  const bool decomposed = argc > 2 ? std::atoi(argv[2]) != 0 : true;
  std::mt19937_64 rng(2024);
  auto cfg = testing::random_config(rng, 300, 0.1, 6, 0.9);
  ModelSpec spec;
  spec.rc = 4.0;
  spec.rcs = 2.2;
  spec.n_max = 64;
  spec.n_species = 6;
  spec.type_dim = 8;
  spec.n_feat = 32;
  spec.n_reduced = 8;
  spec.n_attn = 2;
  spec.attn_dim = 32;
  spec.embed_hidden = {16, 32};
  spec.fit_hidden = {32, 32};
  const DPModel model = init_model(spec, 3);
  for (std::size_t i = 0; i < cfg.atoms.size(); ++i) cfg.atoms.masses[i] = 12.0;
  init_velocities(cfg.atoms, 0.5, 7);

  MDConfig md;
  md.dt = 0.0005;
  md.n_steps = steps;
  AtomSet a_ref = cfg.atoms, a_gpu = cfg.atoms;

  DpProvider::Options ro;
  ro.decomposed = decomposed;
  ro.scheme = DdScheme::masked_reduction;
  ro.n_ranks = decomposed ? 2 : 1;
  ro.workers = 2;
  DpProvider ref(model, ro);
  GpuDpProvider::Options go;
  go.decomposed = decomposed;
  go.scheme = DdScheme::masked_reduction;
  go.n_ranks = decomposed ? 2 : 1;
  GpuDpProvider gpu(model, go);

  AtomSet a_dev = cfg.atoms;
  const RunSummary s_ref = run_md(a_ref, cfg.box, md, {&ref});
  const RunSummary s_gpu = run_md(a_gpu, cfg.box, md, {&gpu});
  // device-resident loop of the same provider: identical forces from identical positions
  // and the reference's integrator arithmetic -> the trajectory must be bit-identical
  const RunSummary s_dev = gpu.run_md(a_dev, cfg.box, md);
  double dev_dx = 0, dev_dv = 0, dev_de = 0, dev_dt = 0;
  for (std::size_t i = 0; i < a_gpu.size(); ++i)
    for (int c = 0; c < 3; ++c) {
      dev_dx = std::max(dev_dx, std::abs(a_gpu.positions[i][c] - a_dev.positions[i][c]));
      dev_dv = std::max(dev_dv, std::abs(a_gpu.velocities[i][c] - a_dev.velocities[i][c]));
    }
  for (long k = 0; k < steps; ++k) {
    dev_de = std::max(dev_de, std::abs(s_gpu.potential_energy[k] - s_dev.potential_energy[k]));
    dev_dt = std::max(dev_dt, std::abs(s_gpu.total_energy[k] - s_dev.total_energy[k]) /
                                  std::max(std::abs(s_gpu.total_energy[k]), 1e-300));
  }
  double de = 0, escale = 0, dx = 0;
  for (long k = 0; k < steps; ++k) {
    de = std::max(de, std::abs(s_ref.potential_energy[k] - s_gpu.potential_energy[k]));
    escale = std::max(escale, std::abs(s_ref.potential_energy[k]));
  }
  for (std::size_t i = 0; i < a_ref.size(); ++i)
    for (int c = 0; c < 3; ++c) {
      double d = std::abs(a_ref.positions[i][c] - a_gpu.positions[i][c]);
      d = std::min(d, cfg.box.lengths[c] - d);  // wrapped coordinates
      dx = std::max(dx, d);
    }
  // trace + ledger parity: the same run_md with a TraceSink and a CollectiveLedger for
  // both providers -> identical ledger records and identical (rank, phase, step) spans
  TraceSink tr_ref, tr_gpu;
  CollectiveLedger lg_ref, lg_gpu;
  {
    AtomSet b_ref = cfg.atoms, b_gpu = cfg.atoms;
    MDConfig md3 = md;
    md3.n_steps = 3;
    run_md(b_ref, cfg.box, md3, {&ref}, {}, &tr_ref, &lg_ref);
    run_md(b_gpu, cfg.box, md3, {&gpu}, {}, &tr_gpu, &lg_gpu);
  }
  bool ledger_ok = lg_ref.records().size() == lg_gpu.records().size();
  for (std::size_t i = 0; ledger_ok && i < lg_ref.records().size(); ++i) {
    const auto& a = lg_ref.records()[i];
    const auto& b = lg_gpu.records()[i];
    ledger_ok = a.step == b.step && a.kind == b.kind && a.bytes == b.bytes && a.participants == b.participants;
  }
  auto keys = [](const TraceSink& t) {
    std::multiset<std::tuple<int, int, long>> k;
    for (const auto& s : t.spans()) k.insert({s.rank, static_cast<int>(s.phase), s.step});
    return k;
  };
  const bool spans_ok = keys(tr_ref) == keys(tr_gpu) && !tr_gpu.spans().empty();
  export_chrome_trace(tr_gpu.spans(), "/tmp/nnmd_b200_trace.json");
  const auto parsed = parse_chrome_trace("/tmp/nnmd_b200_trace.json");
  const PhaseSummary ps = phase_summary(parsed);
  const bool chrome_ok = parsed.size() == tr_gpu.spans().size() && ps.aggregate_fraction.count(Phase::inference);
  std::printf(
      "{\"trace\": {\"ledger_records\": %zu, \"ledger_match\": %s, \"spans\": %zu, \"span_keys_match\": %s, "
      "\"chrome_roundtrip\": %s, \"inference_fraction\": %.3f}}\n",
      lg_gpu.records().size(), ledger_ok ? "true" : "false", tr_gpu.spans().size(), spans_ok ? "true" : "false",
      chrome_ok ? "true" : "false", ps.aggregate_fraction.count(Phase::inference) ? ps.aggregate_fraction.at(Phase::inference) : 0.0);
  std::printf(
      "{\"provider\": \"%s\", \"steps\": %d, \"atoms\": %zu, \"max_rel_energy_diff\": %.3e, "
      "\"max_position_diff\": %.3e, \"e_ref_step0\": %.10f, \"e_gpu_step0\": %.10f, "
      "\"device_loop_position_diff\": %.3e, \"device_loop_velocity_diff\": %.3e, "
      "\"device_loop_potential_diff\": %.3e, \"device_loop_total_rel_diff\": %.3e}\n",
      gpu.name().c_str(), steps, a_ref.size(), de / std::max(escale, 1e-300), dx,
      s_ref.potential_energy[0], s_gpu.potential_energy[0], dev_dx, dev_dv, dev_de, dev_dt);
  return (ledger_ok && spans_ok && chrome_ok && de / std::max(escale, 1e-300) < 1e-5 && dx < 1e-6 && dev_dx == 0.0 && dev_dv == 0.0 && dev_de == 0.0 &&
          dev_dt < 1e-13)
             ? 0
             : 1;
}
