// Host model: init (bit-identical to the reference init_model), .nmdp IO, and weight
// folding for the device.  No reference code is used; formats and draw order follow
// deeppot.cpp:86-127 and deeppot_io.cpp:8-160.
#include "model.h"

#include <cmath>
#include <cstring>
#include <fstream>
#include <random>

namespace nb {

void Model::validate() const {
  require(rc > 0.0 && rcs > 0.0 && rcs < rc, "DPModel: need 0 < rcs < rc");
  require(n_max >= 1, "DPModel: n_max must be >= 1");
  require(ns >= 1 && dz >= 1, "DPModel: bad type embedding shape");
  require(mr >= 1 && mr <= M, "DPModel: n_reduced must be in [1, n_feat]");
  require(te.size() == static_cast<size_t>(ns) * dz, "DPModel: type_embed size mismatch");
  require(!embed.empty() && embed.front().nin == 1 + 2 * dz && embed.back().nout == M,
          "DPModel: embed net shape mismatch");
  require(!fit.empty() && fit.front().nin == M * mr && fit.back().nout == 1,
          "DPModel: fit net shape mismatch");
  for (const auto* chain : {&embed, &fit})
    for (size_t l = 0; l < chain->size(); ++l) {
      const Layer& ly = (*chain)[l];
      require(ly.w.size() == static_cast<size_t>(ly.nin) * ly.nout &&
                  ly.b.size() == static_cast<size_t>(ly.nout),
              "DPModel: layer buffer size mismatch");
      if (l > 0) require(ly.nin == (*chain)[l - 1].nout, "DPModel: layer chain mismatch");
    }
  require(static_cast<int>(wq.size()) == na && wk.size() == wq.size() && wv.size() == wq.size() &&
              wo.size() == wq.size(),
          "DPModel: attention layer count mismatch");
  const size_t proj = static_cast<size_t>(M) * da;
  for (int l = 0; l < na; ++l)
    require(wq[l].size() == proj && wk[l].size() == proj && wv[l].size() == proj &&
                wo[l].size() == proj,
            "DPModel: attention weight size mismatch");
  // device-kernel limits
  require(M <= 256 && mr <= M, "nnmd_b200: n_feat must be <= 256");
  for (const auto& l : embed) require(l.nout <= 256, "nnmd_b200: embed width must be <= 256");
  require(n_max <= 1024, "nnmd_b200: n_max must be <= 1024");
}

long Model::n_params() const {
  long n = static_cast<long>(te.size());
  for (const auto* chain : {&embed, &fit})
    for (const auto& l : *chain) n += static_cast<long>(l.w.size() + l.b.size());
  for (int l = 0; l < na; ++l)
    n += static_cast<long>(wq[l].size() + wk[l].size() + wv[l].size() + wo[l].size());
  return n;
}

namespace {

// One Xavier-uniform draw block: bound sqrt(6/(in+out)), weights in order, zero biases.
std::vector<double> xavier(int nin, int nout, std::mt19937_64& rng) {
  const double bound = std::sqrt(6.0 / (nin + nout));
  std::uniform_real_distribution<double> u(-bound, bound);
  std::vector<double> w(static_cast<size_t>(nin) * nout);
  for (double& x : w) x = u(rng);
  return w;
}

Layer layer(int nin, int nout, std::mt19937_64& rng) {
  Layer l;
  l.nin = nin;
  l.nout = nout;
  l.w = xavier(nin, nout, rng);
  l.b.assign(static_cast<size_t>(nout), 0.0);
  return l;
}

template <class T>
void wr(std::ofstream& os, T v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof v);
}
template <class T>
T rd(std::ifstream& is, const char* what) {
  T v{};
  is.read(reinterpret_cast<char*>(&v), sizeof v);
  require(static_cast<bool>(is), std::string("load_model: truncated file reading ") + what);
  return v;
}
void wr_vec(std::ofstream& os, const std::vector<double>& v) {
  os.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}
void rd_vec(std::ifstream& is, std::vector<double>& v, size_t n, const char* what) {
  v.resize(n);
  is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * 8));
  require(static_cast<bool>(is), std::string("load_model: truncated file reading ") + what);
}

}  // namespace

Model init_model(const nnmd_model_spec& s, uint64_t seed) {
  Model m;
  m.rc = s.rc;
  m.rcs = s.rcs;
  m.n_max = s.n_max;
  m.ns = s.n_species;
  m.dz = s.type_dim;
  m.M = s.n_feat;
  m.mr = s.n_reduced;
  m.na = s.n_attn;
  m.da = s.attn_dim;
  require(s.n_embed_hidden >= 0 && s.n_embed_hidden <= 8 && s.n_fit_hidden >= 0 &&
              s.n_fit_hidden <= 8,
          "ModelSpec: at most 8 hidden layers per net");
  std::mt19937_64 rng(seed);
  {
    const double bound = std::sqrt(6.0 / (1 + m.dz));
    std::uniform_real_distribution<double> u(-bound, bound);
    m.te.resize(static_cast<size_t>(m.ns) * m.dz);
    for (double& x : m.te) x = u(rng);
  }
  int prev = 1 + 2 * m.dz;
  for (int i = 0; i < s.n_embed_hidden; ++i) {
    m.embed.push_back(layer(prev, s.embed_hidden[i], rng));
    prev = s.embed_hidden[i];
  }
  m.embed.push_back(layer(prev, m.M, rng));
  for (int l = 0; l < m.na; ++l) {
    m.wq.push_back(xavier(m.M, m.da, rng));
    m.wk.push_back(xavier(m.M, m.da, rng));
    m.wv.push_back(xavier(m.M, m.da, rng));
    m.wo.push_back(xavier(m.da, m.M, rng));
  }
  prev = m.M * m.mr;
  for (int i = 0; i < s.n_fit_hidden; ++i) {
    m.fit.push_back(layer(prev, s.fit_hidden[i], rng));
    prev = s.fit_hidden[i];
  }
  m.fit.push_back(layer(prev, 1, rng));
  m.validate();
  return m;
}

void save_model(const Model& m, const std::string& path) {
  m.validate();
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  require(os.good(), "save_model: cannot open " + path);
  os.write("NMDP", 4);
  wr<uint32_t>(os, 1);
  wr<double>(os, m.rc);
  wr<double>(os, m.rcs);
  for (int v : {m.n_max, m.ns, m.dz, m.M, m.mr, m.na, m.da, m.gate_norm_id}) wr<int32_t>(os, v);
  for (const auto* chain : {&m.embed, &m.fit}) {
    wr<int32_t>(os, static_cast<int32_t>(chain->size()));
    for (const auto& l : *chain) {
      wr<int32_t>(os, l.nin);
      wr<int32_t>(os, l.nout);
    }
  }
  wr_vec(os, m.te);
  for (const auto& l : m.embed) {
    wr_vec(os, l.w);
    wr_vec(os, l.b);
  }
  for (int l = 0; l < m.na; ++l) {
    wr_vec(os, m.wq[l]);
    wr_vec(os, m.wk[l]);
    wr_vec(os, m.wv[l]);
    wr_vec(os, m.wo[l]);
  }
  for (const auto& l : m.fit) {
    wr_vec(os, l.w);
    wr_vec(os, l.b);
  }
  require(os.good(), "save_model: write failed for " + path);
}

Model load_model(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  require(is.good(), "load_model: cannot open " + path);
  char magic[4];
  is.read(magic, 4);
  require(static_cast<bool>(is) && std::memcmp(magic, "NMDP", 4) == 0,
          "load_model: bad magic (corrupted or not a model file): " + path);
  const auto version = rd<uint32_t>(is, "version");
  require(version == 1, "load_model: unsupported format version " + std::to_string(version));
  Model m;
  m.rc = rd<double>(is, "rc");
  m.rcs = rd<double>(is, "rcs");
  int* fields[] = {&m.n_max, &m.ns, &m.dz, &m.M, &m.mr, &m.na, &m.da, &m.gate_norm_id};
  for (int* f : fields) *f = rd<int32_t>(is, "shape table");
  require(m.ns >= 1 && m.dz >= 1 && m.M >= 1 && m.na >= 0 && m.na <= 64,
          "load_model: implausible shape table");
  for (auto* chain : {&m.embed, &m.fit}) {
    const auto cnt = rd<int32_t>(is, "layer count");
    require(cnt >= 1 && cnt <= 64, "load_model: implausible layer count");
    chain->resize(static_cast<size_t>(cnt));
    for (auto& l : *chain) {
      l.nin = rd<int32_t>(is, "layer shape");
      l.nout = rd<int32_t>(is, "layer shape");
      require(l.nin >= 1 && l.nout >= 1, "load_model: bad layer shape");
    }
  }
  rd_vec(is, m.te, static_cast<size_t>(m.ns) * m.dz, "type_embed");
  for (auto& l : m.embed) {
    rd_vec(is, l.w, static_cast<size_t>(l.nin) * l.nout, "embed w");
    rd_vec(is, l.b, static_cast<size_t>(l.nout), "embed b");
  }
  const size_t proj = static_cast<size_t>(m.M) * m.da;
  m.wq.resize(m.na);
  m.wk.resize(m.na);
  m.wv.resize(m.na);
  m.wo.resize(m.na);
  for (int l = 0; l < m.na; ++l) {
    rd_vec(is, m.wq[l], proj, "attention wq");
    rd_vec(is, m.wk[l], proj, "attention wk");
    rd_vec(is, m.wv[l], proj, "attention wv");
    rd_vec(is, m.wo[l], proj, "attention wo");
  }
  for (auto& l : m.fit) {
    rd_vec(is, l.w, static_cast<size_t>(l.nin) * l.nout, "fit w");
    rd_vec(is, l.b, static_cast<size_t>(l.nout), "fit b");
  }
  is.peek();
  require(is.eof(), "load_model: trailing bytes after model data");
  m.validate();
  return m;
}

DeviceWeightsHost fold_weights(const Model& m) {
  DeviceWeightsHost d;
  auto alloc = [&](size_t n) {
    size_t off = (d.blob.size() + 3) & ~size_t(3);  // 16-byte aligned
    d.blob.resize(off + n, 0.0f);
    return static_cast<long>(off);
  };
  const Layer& L0 = m.embed[0];
  const int E0 = L0.nout, dz = m.dz;
  d.w0 = alloc(E0);
  for (int o = 0; o < E0; ++o) d.blob[d.w0 + o] = static_cast<float>(L0.w[static_cast<size_t>(o) * L0.nin]);
  d.ctab = alloc(static_cast<size_t>(m.ns) * m.ns * E0);
  for (int zj = 0; zj < m.ns; ++zj)
    for (int zi = 0; zi < m.ns; ++zi)
      for (int o = 0; o < E0; ++o) {
        double acc = L0.b[o];
        const double* w = &L0.w[static_cast<size_t>(o) * L0.nin];
        for (int t = 0; t < dz; ++t) {
          acc += w[1 + t] * m.te[static_cast<size_t>(zj) * dz + t];
          acc += w[1 + dz + t] * m.te[static_cast<size_t>(zi) * dz + t];
        }
        d.blob[d.ctab + (static_cast<size_t>(zj) * m.ns + zi) * E0 + o] = static_cast<float>(acc);
      }
  d.edims.push_back(E0);
  d.ew.push_back(-1);
  d.eb.push_back(-1);
  for (size_t l = 1; l < m.embed.size(); ++l) {
    const Layer& ly = m.embed[l];
    d.ew.push_back(alloc(ly.w.size()));
    for (size_t i = 0; i < ly.w.size(); ++i) d.blob[d.ew.back() + i] = static_cast<float>(ly.w[i]);
    d.eb.push_back(alloc(ly.b.size()));
    for (size_t i = 0; i < ly.b.size(); ++i) d.blob[d.eb.back() + i] = static_cast<float>(ly.b[i]);
    d.edims.push_back(ly.nout);
  }
  const int M = m.M, da = m.da;
  const double isd = 1.0 / std::sqrt(static_cast<double>(da));
  for (int l = 0; l < m.na; ++l) {
    const long off = alloc(static_cast<size_t>(M) * 2 * M);
    for (int a = 0; a < M; ++a)
      for (int b = 0; b < M; ++b) {
        double sa = 0, sb = 0;
        for (int t = 0; t < da; ++t) {
          sa += m.wq[l][static_cast<size_t>(a) * da + t] * m.wk[l][static_cast<size_t>(b) * da + t];
          sb += m.wv[l][static_cast<size_t>(a) * da + t] * m.wo[l][static_cast<size_t>(t) * M + b];
        }
        d.blob[off + static_cast<size_t>(a) * 2 * M + b] = static_cast<float>(sa * isd);
        d.blob[off + static_cast<size_t>(a) * 2 * M + M + b] = static_cast<float>(sb);
      }
    d.ab.push_back(off);
  }
  d.fdims.push_back(m.fit[0].nin);
  for (const auto& ly : m.fit) {
    d.fw.push_back(alloc(ly.w.size()));
    for (size_t i = 0; i < ly.w.size(); ++i) d.blob[d.fw.back() + i] = static_cast<float>(ly.w[i]);
    d.fb.push_back(alloc(ly.b.size()));
    for (size_t i = 0; i < ly.b.size(); ++i) d.blob[d.fb.back() + i] = static_cast<float>(ly.b[i]);
    d.fwT.push_back(alloc(ly.w.size()));
    for (int o = 0; o < ly.nout; ++o)
      for (int i = 0; i < ly.nin; ++i)
        d.blob[d.fwT.back() + static_cast<size_t>(i) * ly.nout + o] = static_cast<float>(ly.w[static_cast<size_t>(o) * ly.nin + i]);
    d.fdims.push_back(ly.nout);
  }
  alloc(4);
  return d;
}

}  // namespace nb
