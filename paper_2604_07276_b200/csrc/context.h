// Device context: the B200 replacement of DpProvider + dd_evaluate.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "kernels.h"
#include "model.h"
#include "nccl_dl.h"

namespace nb {

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  void ensure(size_t n);
  void release();
  ~DevBuf() { release(); }
};

struct RankStat {
  long counts[4] = {0, 0, 0, 0};  // locals, ghosts, centres, route entries
  double ms[4] = {0, 0, 0, 0};    // dd build, neighbour, inference, comm
};

struct RankDebug {  // parity hooks, filled on demand
  std::vector<int> centre_atoms, nlist_atom, nlist_img, nn;
  std::vector<int> ghost_atom, ghost_owner, ghost_shift;
};

struct Timer {
  std::string name;
  cudaEvent_t a, b;
};

// Trace span / collective record in the reference's vocabulary (trace.hpp Span, Phase;
// decomp.hpp CollectiveRecord, CollectiveKind).  Phase ids follow nnmd::Phase order:
// 0 classical_md, 1 gather_positions, 2 dd_build, 3 neighbor_build, 4 inference,
// 5 ghost_force_route, 6 reduce_forces, 7 integrate.  Kinds: 0 gather_positions,
// 1 ghost_force_route, 2 reduce_forces.
struct TraceSpan {
  int rank;  // -1: step-global phase
  int phase;
  double t0, t1;  // seconds on the host steady clock (device times from CUDA events)
  long step;
};
struct LedgerRec {
  long step;
  int kind;
  uint64_t bytes;
  int participants;
};

class Context {
 public:
  Context(const Model& m, const nnmd_b200_opts& o);
  ~Context();

  // Full evaluation on device-resident inputs; result layout
  // [E, W(9), F(3n), ae(n)] in d_out (float64).
  void compute_device(long n, const double* d_pos, const int* d_types, const int64_t* d_gid,
                      const double box[3], const uint8_t periodic[3], double* d_out);
  void compute_host(long n, const double* pos, const int* types, const int64_t* gid,
                    const double box[3], const uint8_t periodic[3], double* energy,
                    double* forces, double* virial, double* atom_energy);

  // Device-resident MD loop (run_md, engine.cpp:143-211): n_steps of leap-frog on
  // positions/velocities that stay on the device; rec[2k] = potential, rec[2k+1] = total
  // energy of step k (device).  Throws Error on a non-finite force like run_md.
  struct MdConfig {
    double dt;
    long n_steps;
    long equil_steps;
    double target_temperature;
    long rescale_every;
  };
  void run_md(long n, double* d_pos, double* d_vel, const double* d_mass, const int* d_types,
              const int64_t* d_gid, const double box[3], const uint8_t periodic[3], const MdConfig& cfg,
              double* d_rec);
  void run_md_host(long n, double* pos, double* vel, const double* mass, const int* types, const int64_t* gid,
                   const double box[3], const uint8_t periodic[3], const MdConfig& cfg, double* potential,
                   double* total);

  // Tracing (TraceSink spans from CUDA events) and the collective ledger
  // (CollectiveLedger with the reference PayloadLayout: 20 B/atom gather, 12 B/atom
  // reduction, 20 B per routed ghost entry).  Records accumulate until clear_trace().
  void set_trace(bool spans, bool ledger) {
    trace_on_ = spans;
    ledger_on_ = ledger;
  }
  void set_step(long step) { step_ = step; }
  const std::vector<TraceSpan>& spans() const { return spans_; }
  const std::vector<LedgerRec>& ledger() const { return ledger_; }
  void clear_trace() {
    spans_.clear();
    ledger_.clear();
  }
  void export_chrome_trace(const std::string& path) const;

  cudaStream_t stream() const { return st_; }
  const RankStat& stat(int r) const { return stats_.at(static_cast<size_t>(r)); }
  int n_ranks() const { return opts_.n_ranks; }
  void debug_rank(int rank, RankDebug& out);
  std::vector<std::pair<std::string, double>> kernel_times() const { return ktimes_; }

 private:
  void run_rank(int rank, const SysArgs& sys, const int dims[3], double thickness, bool keep_debug);
  bool bcast_positions() const { return use_nccl_; }
  bool coords_needed() const { return !bcast_positions() || opts_.world_rank == 0; }
  static constexpr int kFlagWords = 8;
  void tic(const char* name);
  void toc();
  void collect_times();

  Model model_;
  DeviceWeightsHost wh_;
  nnmd_b200_opts opts_;
  cudaStream_t st_ = nullptr;
  int n_sm_ = 148;

  DevBuf<float> weights_;
  // pre-split weight images (launch_weight_image), byte offsets into wimg_ (-1: none)
  DevBuf<uint8_t> wimg_;
  std::vector<long> wimg_ab_, wimg_abT_, wimg_ew_, wimg_ewT_;
  void build_weight_images();
  NcclComm comm_ = nullptr;
  bool use_nccl_ = false;

  // inputs (host-API path) and outputs
  DevBuf<double> pos_, out_;
  DevBuf<int> types_;
  DevBuf<int64_t> gid_;
  DevBuf<double> h_pinned_dummy_;
  // MD loop state (host API path) and scratch
  DevBuf<double> md_vel_, md_mass_, md_ke_, md_rec_, md_sum_;
  DevBuf<int> md_err_;
  // step-global
  DevBuf<int> owner_, err_, flags_;
  DevBuf<double> bpos_;  // broadcast positions (collective 1)
  int* h_flags_ = nullptr;  // pinned, kFlagWords + n_ranks
  // per rank (reused across virtual ranks)
  DevBuf<int> is_local_, gcount_, loc_off_, gh_off_, counts_;
  DevBuf<int> m_atom_, m_shift_, m_owner_, m_cell_, cflag_, coff_, cen_member_, cidx_;
  DevBuf<double> m_pos_;
  DevBuf<int> cell_count_, cell_start_, cell_fill_, cell_members_;
  DevBuf<double> cs_x_;      // cell-ordered candidate positions (x | y | z)
  DevBuf<int> cs_i_;         // cell-ordered packed shift | species
  DevBuf<int64_t> cs_gid_;   // cell-ordered gids
  DevBuf<int> nlist_, nn_, rlist_, rn_, maxn_, work_;
  DevBuf<float> X_, Ad_, Bd_, D_, dD_, scratch_, fitY_, fitd_, fitws_, Ust_, PUst_, PTst_, EMBst_;
  DevBuf<float4> R_;
  DevBuf<double> g_, vir_, e_, fmem_, sig_;
  DevBuf<int> Z_;
  DevBuf<int> pack_cnt_;   // pack plan: per-group unit counts | their exclusive scan (+ total)
  DevBuf<int2> packs_;     // (first centre, centre count) per unit
  // ghost-force route and the step result (decomp.cpp:445-538)
  DevBuf<double> red_;    // [R][10] per-rank [E, W9] rows | F [n][3] | e_i [n]  (reduced)
  DevBuf<double> fown_;   // [n][3] owner's zero-image partial
  DevBuf<double> evpart_;  // energy/virial block partials
  DevBuf<int> rcnt_;      // [R][R] routed entries src -> dst, then [R][R] fill cursors
  DevBuf<RouteEntry> route_buf_[kMaxRanks];  // per local source rank, grouped by destination
  DevBuf<RouteEntry> recv_buf_[kMaxRanks];   // per remote source rank (world_size > 1)
  DevBuf<int> inc_cnt_, inc_off_, seg_;
  DevBuf<const RouteEntry*> inc_;
  long route_cap_ = 0;       // entries in the local send buffers this step
  int* h_rcnt_ = nullptr;    // pinned [R][R]
  // ghost capacities per DD rank (no host read-back of counts inside a step)
  std::vector<int> cap_gh_, cap_loc_;
  long cap_n_ = -1;
  int redo_depth_ = 0;
  DevBuf<int> rstat_;        // [R][kCntWords] per-rank device counts of the step
  int* h_rstat_ = nullptr;   // pinned copy
  const MdArgs* md_check_ = nullptr;  // run_md: finite-force check folded into the step's read-back
  int* h_md_err_ = nullptr;           // pinned
  void route_and_reduce(long n, double* d_out);
  std::vector<RankStat> stats_;
  std::vector<RankDebug> debug_;
  std::vector<Timer> timers_;
  std::vector<cudaEvent_t> pool_;
  size_t pool_used_ = 0;
  std::vector<std::pair<std::string, double>> ktimes_;
  struct PhaseMark {
    int rank;
    int phase;
    size_t t0, t1;  // timer indices
  };
  std::vector<PhaseMark> phases_;
  int keep_debug_ = 0;
  // trace / ledger
  bool trace_on_ = false, ledger_on_ = false;
  long step_ = 0;
  cudaEvent_t epoch_ev_ = nullptr;
  double epoch_host_ = 0.0;
  std::vector<TraceSpan> spans_;
  std::vector<LedgerRec> ledger_;
  double ev_time(cudaEvent_t e) const;
  void record_trace(long n, const std::vector<int>& local_ranks);
  cudaEvent_t md_ev_[2] = {nullptr, nullptr};
  // pinned host staging for the host API
  double* h_out_ = nullptr;
  size_t h_out_cap_ = 0;

 public:
  void set_keep_debug(int v) { keep_debug_ = v; }
};

std::vector<int> partition_ranks(const double L[3], int n_ranks, double min_edge);

// Point-to-point plan of the ghost-force route for one process (DD rank r lives in process
// r % world_size): counts[s * R + o] routed entries from source rank s to owner rank o.
// Sends and receives are listed in (source, destination) order on every process, so the
// several transfers between one pair of processes match in posting order.  offset: entries
// into the source's send buffer (grouped by every destination) for a send, into the
// source's receive buffer (grouped by this process's destinations) for a receive.
struct RouteOp {
  int kind;  // 0 send, 1 receive
  int src, dst, peer;
  long offset;
  int count;
};
std::vector<RouteOp> route_schedule(int n_ranks, int world_size, int world_rank, const int* counts);

}  // namespace nb

struct nnmd_b200 {
  nb::Context* ctx = nullptr;
};
