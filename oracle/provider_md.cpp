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

  const RunSummary s_ref = run_md(a_ref, cfg.box, md, {&ref});
  const RunSummary s_gpu = run_md(a_gpu, cfg.box, md, {&gpu});
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
  std::printf(
      "{\"provider\": \"%s\", \"steps\": %d, \"atoms\": %zu, \"max_rel_energy_diff\": %.3e, "
      "\"max_position_diff\": %.3e, \"e_ref_step0\": %.10f, \"e_gpu_step0\": %.10f}\n",
      gpu.name().c_str(), steps, a_ref.size(), de / std::max(escale, 1e-300), dx,
      s_ref.potential_energy[0], s_gpu.potential_energy[0]);
  return (de / std::max(escale, 1e-300) < 1e-5 && dx < 1e-6) ? 0 : 1;
}
