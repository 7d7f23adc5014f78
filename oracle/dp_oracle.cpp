// CPU restatement of the reference DPA-1 force path (TEST INFRASTRUCTURE ONLY).
// See dp_oracle.h.  Double precision, flat row-major arrays, compiled with
// -ffp-contract=off like the reference (proj/CMakeLists.txt:10-13).
//
// Reference citations are to /root/reference/proj.

#include "dp_oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <fstream>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

struct CapErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void req(bool c, const std::string& msg) {
  if (!c) throw std::runtime_error(msg);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const CapErr& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

using Vec = std::vector<double>;

// Dense layer, out-major weights w[o*nin + i] (deeppot.hpp:18-23).
struct Layer {
  int nin = 0, nout = 0;
  Vec w, b;
};

}  // namespace

struct orc_model {
  double rc = 0, rcs = 0;
  int n_max = 0, ns = 0, dz = 0, M = 0, mr = 0, na = 0, da = 0, gate = 1;
  Vec te;                   // ns x dz
  std::vector<Layer> embed;  // 1+2dz -> ... -> M, tanh on every layer
  std::vector<Layer> fit;    // M*mr -> ... -> 1, linear last
  std::vector<Vec> wq, wk, wv, wo;  // M x da (in-major), wo: da x M
};

namespace {

// ---------------------------------------------------------------------------
// Model init / IO
// ---------------------------------------------------------------------------

// Xavier-uniform draw sequence of init_model (deeppot.cpp:86-127): type embedding,
// embed layers (w then zero b), per attention layer wq, wk, wv, wo, fit layers.
Layer xavier_layer(int nin, int nout, std::mt19937_64& rng) {
  Layer l;
  l.nin = nin;
  l.nout = nout;
  const double bound = std::sqrt(6.0 / (nin + nout));
  std::uniform_real_distribution<double> u(-bound, bound);
  l.w.resize(static_cast<size_t>(nin) * nout);
  for (double& x : l.w) x = u(rng);
  l.b.assign(static_cast<size_t>(nout), 0.0);
  return l;
}

Vec xavier_proj(int nin, int nout, std::mt19937_64& rng) {
  return xavier_layer(nin, nout, rng).w;
}

void validate(const orc_model& m) {
  req(m.rc > 0 && m.rcs > 0 && m.rcs < m.rc, "model: need 0 < rcs < rc");
  req(m.n_max >= 1 && m.ns >= 1 && m.dz >= 1 && m.mr >= 1 && m.mr <= m.M, "model: bad shape");
  req(!m.embed.empty() && m.embed.front().nin == 1 + 2 * m.dz && m.embed.back().nout == m.M,
      "model: embed shape");
  req(!m.fit.empty() && m.fit.front().nin == m.M * m.mr && m.fit.back().nout == 1,
      "model: fit shape");
  req(static_cast<int>(m.wq.size()) == m.na, "model: attention count");
}

template <class T>
void put(std::ofstream& os, T v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof v);
}
template <class T>
T get(std::ifstream& is) {
  T v{};
  is.read(reinterpret_cast<char*>(&v), sizeof v);
  req(static_cast<bool>(is), "load: truncated file");
  return v;
}
void put_vec(std::ofstream& os, const Vec& v) {
  os.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}
void get_vec(std::ifstream& is, Vec& v, size_t n) {
  v.resize(n);
  is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * 8));
  req(static_cast<bool>(is), "load: truncated file");
}

// ---------------------------------------------------------------------------
// Geometry primitives (vec.hpp:28-54, system.cpp:59-69)
// ---------------------------------------------------------------------------

// image_delta(rj, ri, s, L) = (rj - ri) + s*L   (vec.hpp:52-54)
inline double img(double rj, double ri, int s, double L) {
  return (rj - ri) + static_cast<double>(s) * L;
}
// norm2 = (x*x + y*y) + z*z   (vec.hpp:28-31)
inline double nrm2(const double* d) { return d[0] * d[0] + d[1] * d[1] + d[2] * d[2]; }

// switch_eval (dp_core.hpp:116-137)
void switch_fn(double r, double rcs, double rc, double& s, double& ds) {
  if (r >= rc) {
    s = ds = 0.0;
    return;
  }
  const double inv = 1.0 / r;
  if (r <= rcs) {
    s = inv;
    ds = -inv * inv;
    return;
  }
  const double span = rc - rcs;
  const double u = (r - rcs) * (1.0 / span);
  const double u2 = u * u, u3 = u2 * u;
  const double w = u3 * (u * (-6.0 * u + 15.0) - 10.0) + 1.0;
  const double dw = -30.0 * u2 * (u - 1.0) * (u - 1.0) * (1.0 / span);
  s = w * inv;
  ds = dw * inv - w * inv * inv;
}

// ---------------------------------------------------------------------------
// Neighbour rows (neighbor.cpp:73-148; deeppot.cpp:141-184)
// ---------------------------------------------------------------------------

struct Row {
  int member;
  int img[3];
  double d[3];
  double r2;
  int species;
  int64_t gid;
};

// sort key (species, r^2, gid) -- deeppot.cpp:141-148
bool row_less(const Row& a, const Row& b) {
  if (a.species != b.species) return a.species < b.species;
  if (a.r2 != b.r2) return a.r2 < b.r2;
  return a.gid < b.gid;
}

struct Sys {
  int n;
  const double* pos;
  const int* species;
  std::vector<int64_t> gid;
  double L[3];
  bool per[3];
};

Sys make_sys(int n, const double* pos, const int* species, const int64_t* gids,
             const double* box3, const uint8_t* periodic) {
  Sys s;
  s.n = n;
  s.pos = pos;
  s.species = species;
  s.gid.resize(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) s.gid[i] = gids ? gids[i] : i;
  for (int a = 0; a < 3; ++a) {
    s.L[a] = box3[a];
    s.per[a] = periodic ? periodic[a] != 0 : true;
  }
  return s;
}

// Full neighbour rows of every atom, sorted canonically.  Cell binning over [0, L) with
// width >= rc, a per-axis list of (target cell, image shift) for offsets -1..1 as in
// neighbor.cpp:91-110, strict norm2(d) < rc^2, self excluded at zero shift.
std::vector<std::vector<Row>> all_rows(const Sys& S, double rc) {
  req(rc > 0, "neighbor list: rc must be > 0");
  for (int a = 0; a < 3; ++a) {
    if (!S.per[a]) continue;
    req(rc <= 0.5 * S.L[a], "neighbor list: rc exceeds half the box on a periodic axis");
    for (int i = 0; i < S.n; ++i)
      req(S.pos[3 * i + a] >= 0.0 && S.pos[3 * i + a] < S.L[a],
          "neighbor list: positions must be wrapped into [0, L) on periodic axes");
  }
  int dims[3];
  double w[3];
  for (int a = 0; a < 3; ++a) {
    const double ext = std::max(S.L[a], rc);
    dims[a] = std::max(1, static_cast<int>(std::floor(ext / rc)));
    w[a] = ext / dims[a];
  }
  std::vector<std::vector<int>> cells(static_cast<size_t>(dims[0]) * dims[1] * dims[2]);
  auto cell_of = [&](int i, int* c) {
    for (int a = 0; a < 3; ++a)
      c[a] = std::clamp(static_cast<int>(std::floor(S.pos[3 * i + a] / w[a])), 0, dims[a] - 1);
  };
  auto flat = [&](int x, int y, int z) { return (x * dims[1] + y) * dims[2] + z; };
  for (int i = 0; i < S.n; ++i) {
    int c[3];
    cell_of(i, c);
    cells[flat(c[0], c[1], c[2])].push_back(i);
  }
  const double rc2 = rc * rc;
  std::vector<std::vector<Row>> rows(static_cast<size_t>(S.n));
  for (int i = 0; i < S.n; ++i) {
    int c[3];
    cell_of(i, c);
    std::vector<std::pair<int, int>> tgt[3];
    for (int a = 0; a < 3; ++a)
      for (int o = -1; o <= 1; ++o) {
        int t = c[a] + o, s = 0;
        if (t < 0) {
          if (!S.per[a]) continue;
          t += dims[a];
          s = -1;
        } else if (t >= dims[a]) {
          if (!S.per[a]) continue;
          t -= dims[a];
          s = 1;
        }
        tgt[a].push_back({t, s});
      }
    for (auto [tx, sx] : tgt[0])
      for (auto [ty, sy] : tgt[1])
        for (auto [tz, sz] : tgt[2])
          for (int j : cells[flat(tx, ty, tz)]) {
            if (j == i && sx == 0 && sy == 0 && sz == 0) continue;
            Row r;
            r.member = j;
            r.img[0] = sx;
            r.img[1] = sy;
            r.img[2] = sz;
            for (int a = 0; a < 3; ++a)
              r.d[a] = img(S.pos[3 * j + a], S.pos[3 * i + a], r.img[a], S.L[a]);
            r.r2 = nrm2(r.d);
            if (!(r.r2 < rc2)) continue;
            r.species = S.species[j];
            r.gid = S.gid[j];
            rows[i].push_back(r);
          }
    std::sort(rows[i].begin(), rows[i].end(), row_less);
  }
  return rows;
}

void check_capacity(const orc_model& m, const Sys& S, int i, size_t nrows) {
  if (static_cast<int>(nrows) > m.n_max)
    throw CapErr("neighbor overflow: atom id " + std::to_string(S.gid[i]) + " has " +
                 std::to_string(nrows) + " neighbors, n_max " + std::to_string(m.n_max));
}

// ---------------------------------------------------------------------------
// One centre: forward (dp_core.hpp:226-392) and exact backward (dp_core.hpp:396-614)
// ---------------------------------------------------------------------------

struct CentreOut {
  double e = 0;
  std::vector<std::array<double, 3>> g;  // de/dd_k
};

CentreOut centre(const orc_model& m, int zi, int n, const double* d, const int* zs) {
  const int M = m.M, mr = m.mr, da = m.da, dz = m.dz;
  CentreOut out;
  // rows: r, s, ds, env (dp_core.hpp:200-223)
  Vec r(n), s(n), ds(n), env(4 * static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    const double* dk = d + 3 * k;
    r[k] = std::sqrt(dk[0] * dk[0] + dk[1] * dk[1] + dk[2] * dk[2]);
    switch_fn(r[k], m.rcs, m.rc, s[k], ds[k]);
    const double sr = s[k] / r[k];
    env[4 * k] = s[k];
    for (int a = 0; a < 3; ++a) env[4 * k + 1 + a] = sr * dk[a];
  }
  // embedding net, tanh on every layer (dp_core.hpp:235-250)
  const int L_e = static_cast<int>(m.embed.size());
  std::vector<Vec> act(L_e + 1);
  act[0].assign(static_cast<size_t>(n) * (1 + 2 * dz), 0.0);
  for (int k = 0; k < n; ++k) {
    double* u = &act[0][static_cast<size_t>(k) * (1 + 2 * dz)];
    u[0] = s[k];
    for (int t = 0; t < dz; ++t) {
      u[1 + t] = m.te[static_cast<size_t>(zs[k]) * dz + t];
      u[1 + dz + t] = m.te[static_cast<size_t>(zi) * dz + t];
    }
  }
  for (int l = 0; l < L_e; ++l) {
    const Layer& ly = m.embed[l];
    act[l + 1].assign(static_cast<size_t>(n) * ly.nout, 0.0);
    for (int k = 0; k < n; ++k)
      for (int o = 0; o < ly.nout; ++o) {
        double acc = ly.b[o];
        for (int i = 0; i < ly.nin; ++i)
          acc += ly.w[static_cast<size_t>(o) * ly.nin + i] * act[l][static_cast<size_t>(k) * ly.nin + i];
        act[l + 1][static_cast<size_t>(k) * ly.nout + o] = std::tanh(acc);
      }
  }
  Vec G = act[L_e];  // n x M
  // gated attention layers (dp_core.hpp:252-356)
  const double isd = 1.0 / std::sqrt(static_cast<double>(da));
  double sigma = 0;
  for (int k = 0; k < n; ++k) sigma += s[k] * s[k];
  const bool gate_ok = sigma > 0.0;
  Vec C(static_cast<size_t>(n) * n), Th(static_cast<size_t>(n) * n, 0.0);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) {
      double acc = 0;
      for (int c = 0; c < 4; ++c) acc += env[4 * k + c] * env[4 * j + c];
      C[static_cast<size_t>(k) * n + j] = acc;
      if (gate_ok) Th[static_cast<size_t>(k) * n + j] = acc / sigma;
    }
  struct Stash {
    Vec gin, q, kk, v, pu, p;
  };
  std::vector<Stash> st(static_cast<size_t>(m.na));
  for (int l = 0; l < m.na && n > 0; ++l) {
    Stash& S = st[l];
    S.gin = G;
    S.q.assign(static_cast<size_t>(n) * da, 0.0);
    S.kk = S.q;
    S.v = S.q;
    for (int k = 0; k < n; ++k)
      for (int mm = 0; mm < M; ++mm) {
        const double g = G[static_cast<size_t>(k) * M + mm];
        for (int a = 0; a < da; ++a) {
          S.q[static_cast<size_t>(k) * da + a] += g * m.wq[l][static_cast<size_t>(mm) * da + a];
          S.kk[static_cast<size_t>(k) * da + a] += g * m.wk[l][static_cast<size_t>(mm) * da + a];
          S.v[static_cast<size_t>(k) * da + a] += g * m.wv[l][static_cast<size_t>(mm) * da + a];
        }
      }
    S.pu.assign(static_cast<size_t>(n) * n, 0.0);
    S.p = S.pu;
    Vec sc(n);
    for (int k = 0; k < n; ++k) {
      for (int j = 0; j < n; ++j) {
        double acc = 0;
        for (int a = 0; a < da; ++a)
          acc += S.q[static_cast<size_t>(k) * da + a] * S.kk[static_cast<size_t>(j) * da + a];
        sc[j] = acc * isd;
      }
      double mx = sc[0];
      for (int j = 1; j < n; ++j) mx = std::max(mx, sc[j]);
      double den = 0;
      for (int j = 0; j < n; ++j) {
        const double e = std::exp(sc[j] - mx);
        S.pu[static_cast<size_t>(k) * n + j] = e;
        den += s[j] * s[j] * e;
      }
      for (int j = 0; j < n; ++j) {
        double& pu = S.pu[static_cast<size_t>(k) * n + j];
        pu = den > 0.0 ? pu / den : 0.0;
        S.p[static_cast<size_t>(k) * n + j] = s[j] * s[j] * pu;
      }
    }
    Vec h(static_cast<size_t>(n) * da, 0.0);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) {
        const double pt = S.p[static_cast<size_t>(k) * n + j] * Th[static_cast<size_t>(k) * n + j];
        for (int a = 0; a < da; ++a)
          h[static_cast<size_t>(k) * da + a] += pt * S.v[static_cast<size_t>(j) * da + a];
      }
    for (int k = 0; k < n; ++k)
      for (int a = 0; a < da; ++a) {
        const double ha = h[static_cast<size_t>(k) * da + a];
        for (int mm = 0; mm < M; ++mm)
          G[static_cast<size_t>(k) * M + mm] += ha * m.wo[l][static_cast<size_t>(a) * M + mm];
      }
  }
  // descriptor (dp_core.hpp:358-384)
  const double inm = 1.0 / std::sqrt(static_cast<double>(m.n_max));
  Vec A(static_cast<size_t>(M) * 4, 0.0), B(static_cast<size_t>(4) * mr, 0.0);
  for (int k = 0; k < n; ++k)
    for (int c = 0; c < 4; ++c) {
      for (int mm = 0; mm < M; ++mm) A[mm * 4 + c] += G[static_cast<size_t>(k) * M + mm] * env[4 * k + c];
      for (int q = 0; q < mr; ++q) B[c * mr + q] += env[4 * k + c] * G[static_cast<size_t>(k) * M + q];
    }
  for (double& x : A) x *= inm;
  for (double& x : B) x *= inm;
  Vec D(static_cast<size_t>(M) * mr, 0.0);
  for (int mm = 0; mm < M; ++mm)
    for (int c = 0; c < 4; ++c)
      for (int q = 0; q < mr; ++q) D[mm * mr + q] += A[mm * 4 + c] * B[c * mr + q];
  // fitting net, tanh hidden, linear output (dp_core.hpp:386-391)
  const int L_f = static_cast<int>(m.fit.size());
  std::vector<Vec> fa(L_f + 1);
  fa[0] = D;
  for (int l = 0; l < L_f; ++l) {
    const Layer& ly = m.fit[l];
    fa[l + 1].assign(ly.nout, 0.0);
    for (int o = 0; o < ly.nout; ++o) {
      double acc = ly.b[o];
      for (int i = 0; i < ly.nin; ++i) acc += ly.w[static_cast<size_t>(o) * ly.nin + i] * fa[l][i];
      fa[l + 1][o] = (l + 1 == L_f) ? acc : std::tanh(acc);
    }
  }
  out.e = fa[L_f][0];

  // ------------------------------ backward, seed de = 1 -----------------------------
  Vec delta{1.0};
  for (int l = L_f - 1; l >= 0; --l) {
    const Layer& ly = m.fit[l];
    if (l + 1 != L_f)
      for (int o = 0; o < ly.nout; ++o) delta[o] *= 1.0 - fa[l + 1][o] * fa[l + 1][o];
    Vec prev(ly.nin, 0.0);
    for (int o = 0; o < ly.nout; ++o)
      for (int i = 0; i < ly.nin; ++i) prev[i] += ly.w[static_cast<size_t>(o) * ly.nin + i] * delta[o];
    delta.swap(prev);
  }
  const Vec& dD = delta;
  Vec dA(static_cast<size_t>(M) * 4, 0.0), dB(static_cast<size_t>(4) * mr, 0.0);
  for (int mm = 0; mm < M; ++mm)
    for (int q = 0; q < mr; ++q)
      for (int c = 0; c < 4; ++c) {
        dA[mm * 4 + c] += dD[mm * mr + q] * B[c * mr + q];
        dB[c * mr + q] += dD[mm * mr + q] * A[mm * 4 + c];
      }
  Vec dG(static_cast<size_t>(std::max(n, 1)) * M, 0.0), dE(static_cast<size_t>(n) * 4, 0.0),
      dsx(n, 0.0);
  for (int k = 0; k < n; ++k) {
    for (int mm = 0; mm < M; ++mm)
      for (int c = 0; c < 4; ++c) {
        dG[static_cast<size_t>(k) * M + mm] += dA[mm * 4 + c] * env[4 * k + c] * inm;
        dE[4 * k + c] += dA[mm * 4 + c] * G[static_cast<size_t>(k) * M + mm] * inm;
      }
    for (int c = 0; c < 4; ++c)
      for (int q = 0; q < mr; ++q) {
        dG[static_cast<size_t>(k) * M + q] += dB[c * mr + q] * env[4 * k + c] * inm;
        dE[4 * k + c] += dB[c * mr + q] * G[static_cast<size_t>(k) * M + q] * inm;
      }
  }
  for (int l = m.na - 1; l >= 0 && n > 0; --l) {
    const Stash& S = st[l];
    // d h = dG Wo^T (dp_core.hpp:457-471)
    Vec dh(static_cast<size_t>(n) * da, 0.0);
    for (int k = 0; k < n; ++k)
      for (int a = 0; a < da; ++a) {
        double acc = 0;
        for (int mm = 0; mm < M; ++mm)
          acc += dG[static_cast<size_t>(k) * M + mm] * m.wo[l][static_cast<size_t>(a) * M + mm];
        dh[static_cast<size_t>(k) * da + a] = acc;
      }
    // dP, dTheta, dV (dp_core.hpp:473-489)
    Vec dP(static_cast<size_t>(n) * n), dTh(static_cast<size_t>(n) * n), dV(static_cast<size_t>(n) * da, 0.0);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) {
        double dpt = 0;
        for (int a = 0; a < da; ++a)
          dpt += dh[static_cast<size_t>(k) * da + a] * S.v[static_cast<size_t>(j) * da + a];
        const size_t kj = static_cast<size_t>(k) * n + j;
        dP[kj] = dpt * Th[kj];
        dTh[kj] = dpt * S.p[kj];
        const double pt = S.p[kj] * Th[kj];
        for (int a = 0; a < da; ++a) dV[static_cast<size_t>(j) * da + a] += pt * dh[static_cast<size_t>(k) * da + a];
      }
    // gate and sigma (dp_core.hpp:491-515)
    if (sigma > 0.0) {
      double dsig = 0;
      const double inv = 1.0 / sigma;
      Vec dC(static_cast<size_t>(n) * n);
      for (size_t kj = 0; kj < dC.size(); ++kj) {
        dC[kj] = dTh[kj] * inv;
        dsig -= dTh[kj] * C[kj] * inv * inv;
      }
      for (int k = 0; k < n; ++k) {
        for (int j = 0; j < n; ++j) {
          const double sym = dC[static_cast<size_t>(k) * n + j] + dC[static_cast<size_t>(j) * n + k];
          for (int c = 0; c < 4; ++c) dE[4 * k + c] += sym * env[4 * j + c];
        }
        dsx[k] += 2.0 * s[k] * dsig;
      }
    }
    // weighted softmax (dp_core.hpp:517-535)
    Vec dS(static_cast<size_t>(n) * n), dw(n, 0.0);
    for (int k = 0; k < n; ++k) {
      double t = 0;
      for (int j = 0; j < n; ++j) t += dP[static_cast<size_t>(k) * n + j] * S.p[static_cast<size_t>(k) * n + j];
      for (int j = 0; j < n; ++j) {
        const size_t kj = static_cast<size_t>(k) * n + j;
        const double diff = dP[kj] - t;
        dS[kj] = S.p[kj] * diff;
        dw[j] += S.pu[kj] * diff;
      }
    }
    for (int j = 0; j < n; ++j) dsx[j] += 2.0 * s[j] * dw[j];
    // dQ, dK (dp_core.hpp:537-552)
    Vec dQ(static_cast<size_t>(n) * da, 0.0), dK(static_cast<size_t>(n) * da, 0.0);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) {
        const double v = dS[static_cast<size_t>(k) * n + j] * isd;
        for (int a = 0; a < da; ++a) {
          dQ[static_cast<size_t>(k) * da + a] += v * S.kk[static_cast<size_t>(j) * da + a];
          dK[static_cast<size_t>(j) * da + a] += v * S.q[static_cast<size_t>(k) * da + a];
        }
      }
    // -> dG (dp_core.hpp:554-577); residual passes dG through unchanged
    for (int k = 0; k < n; ++k)
      for (int mm = 0; mm < M; ++mm) {
        double acc = 0;
        for (int a = 0; a < da; ++a) {
          const size_t ka = static_cast<size_t>(k) * da + a, ma = static_cast<size_t>(mm) * da + a;
          acc += dQ[ka] * m.wq[l][ma] + dK[ka] * m.wk[l][ma] + dV[ka] * m.wv[l][ma];
        }
        dG[static_cast<size_t>(k) * M + mm] += acc;
      }
  }
  // embedding backward + row gradients (dp_core.hpp:580-613)
  out.g.assign(static_cast<size_t>(n), {0, 0, 0});
  for (int k = 0; k < n; ++k) {
    Vec dl(dG.begin() + static_cast<long>(k) * M, dG.begin() + static_cast<long>(k + 1) * M);
    for (int l = L_e - 1; l >= 0; --l) {
      const Layer& ly = m.embed[l];
      const double* y = &act[l + 1][static_cast<size_t>(k) * ly.nout];
      for (int o = 0; o < ly.nout; ++o) dl[o] *= 1.0 - y[o] * y[o];
      Vec prev(ly.nin, 0.0);
      for (int o = 0; o < ly.nout; ++o)
        for (int i = 0; i < ly.nin; ++i) prev[i] += ly.w[static_cast<size_t>(o) * ly.nin + i] * dl[o];
      dl.swap(prev);
    }
    dsx[k] += dl[0];
    const double* dk = d + 3 * k;
    const double ir = 1.0 / r[k], sr = s[k] * ir;
    const double e[3] = {dk[0] * ir, dk[1] * ir, dk[2] * ir};
    const double* dr = &dE[4 * k];
    const double ge = dr[1] * e[0] + dr[2] * e[1] + dr[3] * e[2];
    const double coef = (dr[0] + dsx[k]) * ds[k] + (ds[k] - sr) * ge;
    for (int a = 0; a < 3; ++a) out.g[k][a] = coef * e[a] + sr * dr[1 + a];
  }
  return out;
}

// ---------------------------------------------------------------------------
// Rank grid, ownership, halo (decomp.cpp:17-131)
// ---------------------------------------------------------------------------

// surface-minimising factorisation; ties: most balanced, then lexicographically largest
std::array<int, 3> partition(const double* L, int R, double min_edge) {
  req(R >= 1, "partition_ranks: n_ranks must be >= 1");
  bool have = false;
  std::array<int, 3> best{}, best_sorted{};
  double best_surf = 0;
  for (int px = 1; px <= R; ++px) {
    if (R % px) continue;
    for (int py = 1; py <= R / px; ++py) {
      if ((R / px) % py) continue;
      const int pz = R / px / py;
      const double a = L[0] / px, b = L[1] / py, c = L[2] / pz;
      if (std::min({a, b, c}) < min_edge) continue;
      const double surf = 2.0 * (a * b + b * c + c * a);
      std::array<int, 3> dims{px, py, pz}, srt = dims;
      std::sort(srt.begin(), srt.end(), std::greater<int>());
      bool better = !have || surf < best_surf ||
                    (surf == best_surf && (srt < best_sorted || (srt == best_sorted && dims > best)));
      if (better) {
        have = true;
        best = dims;
        best_sorted = srt;
        best_surf = surf;
      }
    }
  }
  req(have, "partition_ranks: no factorization of " + std::to_string(R) +
                " ranks fits the halo constraints of this box; use a smaller rank count");
  return best;
}

int owner_of(const double* p, const int* dims, const double* L) {
  int c[3];
  for (int a = 0; a < 3; ++a) {
    const double edge = L[a] / dims[a];
    c[a] = std::clamp(static_cast<int>(std::floor(p[a] / edge)), 0, dims[a] - 1);
  }
  return (c[0] * dims[1] + c[1]) * dims[2] + c[2];
}

void sub_bounds(const int* dims, int rank, const double* L, double* lo, double* hi) {
  const int idx[3] = {rank / (dims[1] * dims[2]), (rank / dims[2]) % dims[1], rank % dims[2]};
  for (int a = 0; a < 3; ++a) {
    const double edge = L[a] / dims[a];
    lo[a] = idx[a] * edge;
    hi[a] = (idx[a] + 1) * edge;
  }
}

struct Ghost {
  int atom, owner, s[3];
};

// build_halo slab test with the 1e-12*L guard (decomp.cpp:96-131)
std::vector<Ghost> halo(const Sys& S, const int* dims, int rank, double t,
                        const std::vector<int>& owner) {
  for (int a = 0; a < 3; ++a)
    req(!S.per[a] || t <= S.L[a], "build_halo: thickness exceeds the box");
  double lo0[3], hi0[3], lo[3], hi[3];
  sub_bounds(dims, rank, S.L, lo0, hi0);
  for (int a = 0; a < 3; ++a) {
    const double g = 1e-12 * S.L[a];
    lo[a] = lo0[a] - t - g;
    hi[a] = hi0[a] + t + g;
  }
  const int sx = S.per[0], sy = S.per[1], sz = S.per[2];
  std::vector<Ghost> out;
  for (int i = 0; i < S.n; ++i)
    for (int kx = -sx; kx <= sx; ++kx)
      for (int ky = -sy; ky <= sy; ++ky)
        for (int kz = -sz; kz <= sz; ++kz) {
          if (kx == 0 && ky == 0 && kz == 0 && owner[i] == rank) continue;
          const double q[3] = {S.pos[3 * i] + kx * S.L[0], S.pos[3 * i + 1] + ky * S.L[1],
                               S.pos[3 * i + 2] + kz * S.L[2]};
          bool in = true;
          for (int a = 0; a < 3; ++a) in = in && q[a] >= lo[a] && q[a] < hi[a];
          if (in) out.push_back({i, owner[i], {kx, ky, kz}});
        }
  return out;
}

void check_model_inputs(const orc_model& m, const Sys& S) {
  validate(m);
  for (int a = 0; a < 3; ++a) {
    req(S.L[a] > 0.0, "SimBox: non-positive edge length");
    if (S.per[a]) req(S.L[a] >= 2.0 * m.rc, "SimBox: periodic edge shorter than 2*rc");
  }
  for (int i = 0; i < S.n; ++i)
    req(S.species[i] >= 0 && S.species[i] < m.ns, "species id outside the model's species table");
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

orc_model* orc_model_init(double rc, double rcs, int n_max, int n_species, int type_dim,
                          int n_feat, int n_reduced, int n_attn, int attn_dim,
                          const int* embed_hidden, int n_embed_hidden, const int* fit_hidden,
                          int n_fit_hidden, uint64_t seed) {
  orc_model* out = nullptr;
  guarded([&] {
    auto m = new orc_model;
    m->rc = rc;
    m->rcs = rcs;
    m->n_max = n_max;
    m->ns = n_species;
    m->dz = type_dim;
    m->M = n_feat;
    m->mr = n_reduced;
    m->na = n_attn;
    m->da = attn_dim;
    std::mt19937_64 rng(seed);
    {
      const double bound = std::sqrt(6.0 / (1 + type_dim));
      std::uniform_real_distribution<double> u(-bound, bound);
      m->te.resize(static_cast<size_t>(n_species) * type_dim);
      for (double& x : m->te) x = u(rng);
    }
    int prev = 1 + 2 * type_dim;
    for (int i = 0; i < n_embed_hidden; ++i) {
      m->embed.push_back(xavier_layer(prev, embed_hidden[i], rng));
      prev = embed_hidden[i];
    }
    m->embed.push_back(xavier_layer(prev, n_feat, rng));
    for (int l = 0; l < n_attn; ++l) {
      m->wq.push_back(xavier_proj(n_feat, attn_dim, rng));
      m->wk.push_back(xavier_proj(n_feat, attn_dim, rng));
      m->wv.push_back(xavier_proj(n_feat, attn_dim, rng));
      m->wo.push_back(xavier_proj(attn_dim, n_feat, rng));
    }
    prev = n_feat * n_reduced;
    for (int i = 0; i < n_fit_hidden; ++i) {
      m->fit.push_back(xavier_layer(prev, fit_hidden[i], rng));
      prev = fit_hidden[i];
    }
    m->fit.push_back(xavier_layer(prev, 1, rng));
    validate(*m);
    out = m;
  });
  return out;
}

// .nmdp layout (deeppot_io.cpp:8-16)
int orc_model_save(const orc_model* m, const char* path) {
  return guarded([&] {
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    req(os.good(), std::string("save: cannot open ") + path);
    os.write("NMDP", 4);
    put<uint32_t>(os, 1);
    put<double>(os, m->rc);
    put<double>(os, m->rcs);
    for (int v : {m->n_max, m->ns, m->dz, m->M, m->mr, m->na, m->da, m->gate}) put<int32_t>(os, v);
    put<int32_t>(os, static_cast<int32_t>(m->embed.size()));
    for (auto& l : m->embed) {
      put<int32_t>(os, l.nin);
      put<int32_t>(os, l.nout);
    }
    put<int32_t>(os, static_cast<int32_t>(m->fit.size()));
    for (auto& l : m->fit) {
      put<int32_t>(os, l.nin);
      put<int32_t>(os, l.nout);
    }
    put_vec(os, m->te);
    for (auto& l : m->embed) {
      put_vec(os, l.w);
      put_vec(os, l.b);
    }
    for (int l = 0; l < m->na; ++l) {
      put_vec(os, m->wq[l]);
      put_vec(os, m->wk[l]);
      put_vec(os, m->wv[l]);
      put_vec(os, m->wo[l]);
    }
    for (auto& l : m->fit) {
      put_vec(os, l.w);
      put_vec(os, l.b);
    }
    req(os.good(), "save: write failed");
  });
}

orc_model* orc_model_load(const char* path) {
  orc_model* out = nullptr;
  guarded([&] {
    std::ifstream is(path, std::ios::binary);
    req(is.good(), std::string("load: cannot open ") + path);
    char mg[4];
    is.read(mg, 4);
    req(static_cast<bool>(is) && std::memcmp(mg, "NMDP", 4) == 0, "load: bad magic");
    req(get<uint32_t>(is) == 1, "load: unsupported format version");
    auto m = new orc_model;
    m->rc = get<double>(is);
    m->rcs = get<double>(is);
    int* f[] = {&m->n_max, &m->ns, &m->dz, &m->M, &m->mr, &m->na, &m->da, &m->gate};
    for (int* p : f) *p = get<int32_t>(is);
    auto shapes = [&](std::vector<Layer>& v) {
      const int cnt = get<int32_t>(is);
      req(cnt >= 1 && cnt <= 64, "load: implausible layer count");
      v.resize(cnt);
      for (auto& l : v) {
        l.nin = get<int32_t>(is);
        l.nout = get<int32_t>(is);
      }
    };
    shapes(m->embed);
    shapes(m->fit);
    get_vec(is, m->te, static_cast<size_t>(m->ns) * m->dz);
    for (auto& l : m->embed) {
      get_vec(is, l.w, static_cast<size_t>(l.nin) * l.nout);
      get_vec(is, l.b, l.nout);
    }
    const size_t proj = static_cast<size_t>(m->M) * m->da;
    m->wq.resize(m->na);
    m->wk.resize(m->na);
    m->wv.resize(m->na);
    m->wo.resize(m->na);
    for (int l = 0; l < m->na; ++l) {
      get_vec(is, m->wq[l], proj);
      get_vec(is, m->wk[l], proj);
      get_vec(is, m->wv[l], proj);
      get_vec(is, m->wo[l], proj);
    }
    for (auto& l : m->fit) {
      get_vec(is, l.w, static_cast<size_t>(l.nin) * l.nout);
      get_vec(is, l.b, l.nout);
    }
    validate(*m);
    out = m;
  });
  return out;
}

void orc_model_free(orc_model* m) { delete m; }

long orc_model_nparams(const orc_model* m) {
  long n = static_cast<long>(m->te.size());
  for (auto& l : m->embed) n += static_cast<long>(l.w.size() + l.b.size());
  for (auto& l : m->fit) n += static_cast<long>(l.w.size() + l.b.size());
  for (int l = 0; l < m->na; ++l)
    n += static_cast<long>(m->wq[l].size() + m->wk[l].size() + m->wv[l].size() + m->wo[l].size());
  return n;
}

int orc_model_flat(const orc_model* m, double* out, long cap) {
  return guarded([&] {
    req(cap >= orc_model_nparams(m), "flat: capacity");
    long t = 0;
    auto app = [&](const Vec& v) {
      for (double x : v) out[t++] = x;
    };
    app(m->te);
    for (auto& l : m->embed) {
      app(l.w);
      app(l.b);
    }
    for (int l = 0; l < m->na; ++l) {
      app(m->wq[l]);
      app(m->wk[l]);
      app(m->wv[l]);
      app(m->wo[l]);
    }
    for (auto& l : m->fit) {
      app(l.w);
      app(l.b);
    }
  });
}

int orc_neighbor_rows(const orc_model* m, int n, const double* pos, const int* species,
                      const int64_t* gids, const double* box3, const uint8_t* periodic,
                      long cap, int* counts, int* member, int* image, double* d, long* total) {
  return guarded([&] {
    Sys S = make_sys(n, pos, species, gids, box3, periodic);
    auto rows = all_rows(S, m->rc);
    long t = 0;
    for (int i = 0; i < n; ++i) {
      check_capacity(*m, S, i, rows[i].size());
      counts[i] = static_cast<int>(rows[i].size());
      for (const Row& r : rows[i]) {
        req(t < cap, "orc_neighbor_rows: capacity");
        member[t] = r.member;
        for (int a = 0; a < 3; ++a) {
          image[3 * t + a] = r.img[a];
          d[3 * t + a] = r.d[a];
        }
        ++t;
      }
    }
    *total = t;
  });
}

// evaluate_dp (deeppot.cpp:315-369) + virial
int orc_evaluate(const orc_model* m, int n, const double* pos, const int* species,
                 const int64_t* gids, const double* box3, const uint8_t* periodic,
                 double* energy, double* forces, double* atom_energy, double* virial) {
  return guarded([&] {
    Sys S = make_sys(n, pos, species, gids, box3, periodic);
    check_model_inputs(*m, S);
    auto rows = all_rows(S, m->rc);
    std::vector<double> F(3 * static_cast<size_t>(n), 0.0);
    double E = 0, W[9] = {0};
    for (int i = 0; i < n; ++i) {
      check_capacity(*m, S, i, rows[i].size());
      const int nr = static_cast<int>(rows[i].size());
      std::vector<double> d(3 * static_cast<size_t>(nr));
      std::vector<int> zs(nr);
      for (int k = 0; k < nr; ++k) {
        for (int a = 0; a < 3; ++a) d[3 * k + a] = rows[i][k].d[a];
        zs[k] = rows[i][k].species;
      }
      CentreOut co = centre(*m, species[i], nr, d.data(), zs.data());
      E += co.e;
      if (atom_energy) atom_energy[i] = co.e;
      // F_t = -sum of partials (deeppot.cpp:300-309); centre gets -(-sum g) = +sum g
      for (int k = 0; k < nr; ++k)
        for (int a = 0; a < 3; ++a) {
          F[3 * rows[i][k].member + a] -= co.g[k][a];
          F[3 * i + a] += co.g[k][a];
          for (int b = 0; b < 3; ++b) W[3 * a + b] -= co.g[k][a] * d[3 * k + b];
        }
    }
    *energy = E;
    std::memcpy(forces, F.data(), F.size() * sizeof(double));
    if (virial) std::memcpy(virial, W, sizeof W);
  });
}

int orc_evaluate_center(const orc_model* m, int center_species, int n_rows, const double* d,
                        const int* row_species, double* energy, double* row_grads) {
  return guarded([&] {
    CentreOut co = centre(*m, center_species, n_rows, d, row_species);
    *energy = co.e;
    for (int k = 0; k < n_rows; ++k)
      for (int a = 0; a < 3; ++a) row_grads[3 * k + a] = co.g[k][a];
  });
}

int orc_partition_ranks(const double* box3, int n_ranks, double min_edge, int* dims) {
  return guarded([&] {
    auto d = partition(box3, n_ranks, min_edge);
    for (int a = 0; a < 3; ++a) dims[a] = d[a];
  });
}

int orc_owner_ranks(int n, const double* pos, const double* box3, const int* dims, int* owner) {
  return guarded([&] {
    for (int i = 0; i < n; ++i) owner[i] = owner_of(pos + 3 * i, dims, box3);
  });
}

int orc_build_halo(int n, const double* pos, const double* box3, const uint8_t* periodic,
                   const int* dims, int rank, double thickness, long cap, int* atom,
                   int* owner_out, int* shift, long* n_out) {
  return guarded([&] {
    std::vector<int> sp(n, 0);
    Sys S = make_sys(n, pos, sp.data(), nullptr, box3, periodic);
    std::vector<int> owner(n);
    for (int i = 0; i < n; ++i) owner[i] = owner_of(pos + 3 * i, dims, box3);
    auto g = halo(S, dims, rank, thickness, owner);
    req(static_cast<long>(g.size()) <= cap, "orc_build_halo: capacity");
    for (size_t k = 0; k < g.size(); ++k) {
      atom[k] = g[k].atom;
      owner_out[k] = g[k].owner;
      for (int a = 0; a < 3; ++a) shift[3 * k + a] = g[k].s[a];
    }
    *n_out = static_cast<long>(g.size());
  });
}

// One rank of dd_evaluate.  Because every rank's centre rows equal the single-domain rows
// bit for bit, the rank evaluates its centres from the single-domain
// rows.  masked_reduction: centres = locals, every partial (incl. ghost targets) lands in
// the global-indexed buffer and the cross-rank sum routes it to the owner
// (decomp.cpp:445-538).  wide_halo: centres = locals + first-layer ghosts, only partials
// landing on this rank's own atoms are kept (decomp.cpp:428-437).
int orc_dd_rank(const orc_model* m, int n, const double* pos, const int* species,
                const int64_t* gids, const double* box3, const uint8_t* periodic,
                int n_ranks, int scheme, int rank, double* forces, double* atom_energy,
                double* energy, double* virial, long* stats) {
  return guarded([&] {
    Sys S = make_sys(n, pos, species, gids, box3, periodic);
    check_model_inputs(*m, S);
    const double t = scheme == 0 ? m->rc : 2.0 * m->rc;
    auto dims = partition(box3, n_ranks, t);
    for (int a = 0; a < 3; ++a)
      req(box3[a] / dims[a] >= t, "dd_evaluate: subdomain edge shorter than the halo thickness");
    std::vector<int> owner(n);
    for (int i = 0; i < n; ++i) owner[i] = owner_of(pos + 3 * i, dims.data(), box3);
    auto ghosts = halo(S, dims.data(), rank, t, owner);
    auto rows = all_rows(S, m->rc);
    // centre set: locals (+ first-layer ghosts for wide, atom-major)
    double lo0[3], hi0[3], lo[3], hi[3];
    sub_bounds(dims.data(), rank, box3, lo0, hi0);
    for (int a = 0; a < 3; ++a) {
      const double g = 1e-12 * box3[a];
      lo[a] = lo0[a] - m->rc - g;
      hi[a] = hi0[a] + m->rc + g;
    }
    struct Centre {
      int atom;
      int s[3];
      bool owned;
    };
    std::vector<Centre> centres;
    long locals = 0;
    for (int i = 0; i < n; ++i)
      if (owner[i] == rank) {
        centres.push_back({i, {0, 0, 0}, true});
        ++locals;
      }
    if (scheme == 1)
      for (const Ghost& g : ghosts) {
        bool in = true;
        for (int a = 0; a < 3; ++a) {
          const double q = pos[3 * g.atom + a] + g.s[a] * box3[a];
          in = in && q >= lo[a] && q < hi[a];
        }
        if (in) centres.push_back({g.atom, {g.s[0], g.s[1], g.s[2]}, false});
      }
    std::fill(forces, forces + 3 * static_cast<size_t>(n), 0.0);
    if (atom_energy) std::fill(atom_energy, atom_energy + n, 0.0);
    double E = 0, W[9] = {0};
    for (const Centre& cen : centres) {
      const int i = cen.atom;
      const bool owned = cen.owned;
      check_capacity(*m, S, i, rows[i].size());
      const int nr = static_cast<int>(rows[i].size());
      std::vector<double> d(3 * static_cast<size_t>(nr));
      std::vector<int> zs(nr);
      for (int k = 0; k < nr; ++k) {
        for (int a = 0; a < 3; ++a) d[3 * k + a] = rows[i][k].d[a];
        zs[k] = rows[i][k].species;
      }
      CentreOut co = centre(*m, species[i], nr, d.data(), zs.data());
      if (owned) {
        E += co.e;
        if (atom_energy) atom_energy[i] = co.e;
        for (int k = 0; k < nr; ++k)
          for (int a = 0; a < 3; ++a) {
            forces[3 * i + a] += co.g[k][a];
            for (int b = 0; b < 3; ++b) W[3 * a + b] -= co.g[k][a] * d[3 * k + b];
          }
      }
      for (int k = 0; k < nr; ++k) {
        const int tgt = rows[i][k].member;
        // wide: keep only partials landing on a local member (owned atom at shift 0)
        if (scheme == 1 && (owner[tgt] != rank || rows[i][k].img[0] + cen.s[0] != 0 ||
                            rows[i][k].img[1] + cen.s[1] != 0 || rows[i][k].img[2] + cen.s[2] != 0))
          continue;
        for (int a = 0; a < 3; ++a) forces[3 * tgt + a] -= co.g[k][a];
      }
    }
    *energy = E;
    if (virial) std::memcpy(virial, W, sizeof W);
    if (stats) {
      stats[0] = locals;
      stats[1] = static_cast<long>(ghosts.size());
      stats[2] = static_cast<long>(centres.size());
    }
  });
}

// Synthetic solvated-protein input; restates the product's test-system
// generator (paper_2604_07276_b200/csrc/synth.cpp) so the golden vectors and bench.py's
// reference arm never load the product library.  Test-system plumbing, not reference
// arithmetic: splitmix64 stream, globule of 30 % of the atoms (H/C/N/O/S) at the box
// centre, water O/H and one ion per 200 solvent atoms around it, min-separation
// rejection under the periodic minimum image.  tests/test_oracle.py pins it bitwise to
// nnmd_synth_system.
int orc_synth_system(int64_t n, double rho, double min_sep, uint64_t seed, double* box,
                     double* pos, int32_t* types) {
  return guarded([&] {
    req(n >= 1 && rho > 0.0 && min_sep >= 0.0, "synth_system: bad arguments");
    const double L = std::cbrt(static_cast<double>(n) / rho);
    for (int a = 0; a < 3; ++a) box[a] = L;
    const double Rp = std::cbrt(0.30 * L * L * L * 3.0 / (4.0 * M_PI));
    const int64_t n_prot = static_cast<int64_t>(std::llround(0.30 * static_cast<double>(n)));
    const int G = std::max(1, static_cast<int>(std::floor(L / std::max(min_sep, 1e-3))));
    const double w = L / G;
    std::vector<int> head(static_cast<size_t>(G) * G * G, -1), nxt(static_cast<size_t>(n), -1);
    auto cell = [&](double x) { return std::min(G - 1, std::max(0, static_cast<int>(std::floor(x / w)))); };
    const double ms2 = min_sep * min_sep;
    uint64_t state = seed * 0x2545F4914F6CDD1Dull + 12345;
    auto next64 = [&] {
      uint64_t z = (state += 0x9E3779B97F4A7C15ull);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    auto uniform = [&] { return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0); };
    auto too_close = [&](const double* p, int64_t j) {
      double d2 = 0;
      for (int a = 0; a < 3; ++a) {
        double d = p[a] - pos[3 * j + a];
        d -= L * std::round(d / L);
        d2 += d * d;
      }
      return d2 < ms2;
    };
    int64_t n_solvent = 0;
    for (int64_t i = 0; i < n; ++i) {
      const bool prot = i < n_prot;
      double p[3];
      bool ok = false;
      for (int attempt = 0; attempt < 10000 && !ok; ++attempt) {
        for (int a = 0; a < 3; ++a) p[a] = uniform() * L;
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
              for (int j = head[(static_cast<size_t>(cx) * G + cy) * G + cz]; j >= 0 && ok; j = nxt[j])
                if (too_close(p, j)) ok = false;
            }
        if (G < 3 && ok)
          for (int64_t j = 0; j < i && ok; ++j)
            if (too_close(p, j)) ok = false;
      }
      req(ok, "synth_system: could not place atom (density too high for min_sep)");
      for (int a = 0; a < 3; ++a) pos[3 * i + a] = p[a] >= L ? 0.0 : p[a];
      int t;
      if (prot) {
        const double u = uniform();
        t = u < 0.49 ? 0 : u < 0.81 ? 1 : u < 0.895 ? 2 : u < 0.995 ? 3 : 4;
      } else {
        t = (n_solvent % 200 == 199) ? 5 : (n_solvent % 3 == 0 ? 3 : 0);
        ++n_solvent;
      }
      types[i] = t;
      const size_t ci = (static_cast<size_t>(cell(pos[3 * i])) * G + cell(pos[3 * i + 1])) * G + cell(pos[3 * i + 2]);
      nxt[static_cast<size_t>(i)] = head[ci];
      head[ci] = static_cast<int>(i);
    }
  });
}

}  // extern "C"
