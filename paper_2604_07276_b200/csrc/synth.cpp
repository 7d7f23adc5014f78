// Deterministic synthetic solvated-protein system (test-system plumbing).
// A compact protein-like globule (H/C/N/O/S) at the box centre holding ~30 % of the
// atoms, water (O, H) and ~0.5 % ions around it, uniform overall density rho, minimum
// pair separation min_sep under periodic minimum image.  splitmix64 stream, so the same
// (n, rho, min_sep, seed) gives the same coordinates on every host.
#include <cmath>
#include <cstdint>
#include <vector>

#include "model.h"

namespace nb {

namespace {

struct Rng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
};

}  // namespace

void synth_system(int64_t n, double rho, double min_sep, uint64_t seed, double box[3],
                  double* pos, int32_t* types) {
  require(n >= 1 && rho > 0.0 && min_sep >= 0.0, "synth_system: bad arguments");
  const double L = std::cbrt(static_cast<double>(n) / rho);
  for (int a = 0; a < 3; ++a) box[a] = L;
  const double Rp = std::cbrt(0.30 * L * L * L * 3.0 / (4.0 * M_PI));
  const int64_t n_prot = static_cast<int64_t>(std::llround(0.30 * static_cast<double>(n)));
  // hashing grid for the rejection test
  const int G = std::max(1, static_cast<int>(std::floor(L / std::max(min_sep, 1e-3))));
  const double w = L / G;
  std::vector<int> head(static_cast<size_t>(G) * G * G, -1), next(static_cast<size_t>(n), -1);
  auto cell = [&](double x) { return std::min(G - 1, std::max(0, static_cast<int>(std::floor(x / w)))); };
  const double ms2 = min_sep * min_sep;
  Rng rng{seed * 0x2545F4914F6CDD1Dull + 12345};
  int64_t placed = 0, n_solvent = 0;
  for (int64_t i = 0; i < n; ++i) {
    const bool prot = i < n_prot;
    double p[3];
    bool ok = false;
    for (int attempt = 0; attempt < 10000 && !ok; ++attempt) {
      for (int a = 0; a < 3; ++a) p[a] = rng.uniform() * L;
      double r2 = 0;
      for (int a = 0; a < 3; ++a) r2 += (p[a] - 0.5 * L) * (p[a] - 0.5 * L);
      if (prot != (r2 < Rp * Rp)) continue;
      ok = true;
      const int c[3] = {cell(p[0]), cell(p[1]), cell(p[2])};
      const int span = (G >= 3) ? 1 : 0;
      for (int dx = -span; dx <= span && ok; ++dx)
        for (int dy = -span; dy <= span && ok; ++dy)
          for (int dz = -span; dz <= span && ok; ++dz) {
            const int cx = (c[0] + dx + G) % G, cy = (c[1] + dy + G) % G, cz = (c[2] + dz + G) % G;
            for (int j = head[(static_cast<size_t>(cx) * G + cy) * G + cz]; j >= 0 && ok; j = next[j]) {
              double d2 = 0;
              for (int a = 0; a < 3; ++a) {
                double d = p[a] - pos[3 * j + a];
                d -= L * std::round(d / L);
                d2 += d * d;
              }
              if (d2 < ms2) ok = false;
            }
          }
      if (G < 3 && ok) {  // tiny box: brute force
        for (int64_t j = 0; j < placed && ok; ++j) {
          double d2 = 0;
          for (int a = 0; a < 3; ++a) {
            double d = p[a] - pos[3 * j + a];
            d -= L * std::round(d / L);
            d2 += d * d;
          }
          if (d2 < ms2) ok = false;
        }
      }
    }
    require(ok, "synth_system: could not place atom (density too high for min_sep)");
    for (int a = 0; a < 3; ++a) {
      double x = p[a];
      if (x >= L) x = 0.0;
      pos[3 * i + a] = x;
    }
    int t;
    if (prot) {
      const double u = rng.uniform();
      t = u < 0.49 ? 0 : u < 0.81 ? 1 : u < 0.895 ? 2 : u < 0.995 ? 3 : 4;  // H C N O S
    } else {
      t = (n_solvent % 200 == 199) ? 5 : (n_solvent % 3 == 0 ? 3 : 0);   // ion, O, H
      ++n_solvent;
    }
    types[i] = t;
    const size_t ci = (static_cast<size_t>(cell(pos[3 * i])) * G + cell(pos[3 * i + 1])) * G + cell(pos[3 * i + 2]);
    next[static_cast<size_t>(i)] = head[ci];
    head[ci] = static_cast<int>(i);
    ++placed;
  }
}

}  // namespace nb
