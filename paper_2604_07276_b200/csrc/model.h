// Host-side DPA-1 model (the reference DPModel, deeppot.hpp:35-60) and its folding into
// the device weight set used by the kernels.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "nnmd_b200.h"

namespace nb {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};

inline void require(bool c, const std::string& msg) {
  if (!c) throw Error(msg);
}

// Dense layer, out-major weights w[o*nin + i] (deeppot.hpp:18-23).
struct Layer {
  int nin = 0, nout = 0;
  std::vector<double> w, b;
};

struct Model {
  double rc = 0, rcs = 0;
  int n_max = 64, ns = 1, dz = 4, M = 16, mr = 4, na = 0, da = 16, gate_norm_id = 1;
  std::vector<double> te;             // ns x dz
  std::vector<Layer> embed, fit;      // embed: 1+2dz -> ... -> M (tanh all); fit: M*mr -> ... -> 1
  std::vector<std::vector<double>> wq, wk, wv, wo;  // M x da in-major; wo: da x M

  void validate() const;
  long n_params() const;
};

Model init_model(const nnmd_model_spec& spec, uint64_t seed);
Model load_model(const std::string& path);
void save_model(const Model& m, const std::string& path);

// Device weight set, float32, folded once on the host in float64:
//  * embed layer 0:  u = (s, te[zj], te[zi])  ->  W0 u + b0 = s*w0 + ctab[zj][zi]
//    with ctab[zj][zi] = b0 + W0[:,1:1+dz] te[zj] + W0[:,1+dz:] te[zi]  (ns*ns*E0 table)
//  * attention l:    S = Q K^T / sqrt(da) = X (Wq Wk^T / sqrt(da)) X^T = (X A) X^T
//                    H Wo = (P~ V) Wo   = P~ (X (Wv Wo))           = P~ (X B)
//    AB_l = [A_l | B_l]  (M x 2M, row-major)   -- an exact re-association of the
//    reference's products (dp_core.hpp:259-355) that removes the d_a = 256 axis.
//  * all other layers copied (out-major, as in the reference).
struct DeviceWeightsHost {
  std::vector<float> blob;        // everything, concatenated, 16-byte aligned offsets
  // offsets (in floats) into blob
  long w0 = 0, ctab = 0;
  std::vector<long> ew, eb;        // embed layers 1.. (index 0 unused)
  std::vector<int> edims;          // widths: edims[0] = E0 (layer-0 out), ... edims.back() = M
  std::vector<long> ab;            // per attention layer, M x 2M
  std::vector<long> fw, fb;        // fit layers ([out][in] weights, biases)
  std::vector<long> fwT;           // fit weights transposed ([in][out]): backward GEMM B operands
  std::vector<int> fdims;          // fit widths: fdims[0] = M*mr, ..., fdims.back() = 1
};

DeviceWeightsHost fold_weights(const Model& m);

}  // namespace nb

struct nnmd_model {
  nb::Model m;
};
