// nnmd_b200 device context: one DpProvider::evaluate / dd_evaluate step on a B200.
//
// Per step (reference dd_evaluate, decomp.cpp:265-542):
//   ownership (+ input validation)                      k_owner
//   for each DD rank handled by this process (ascending):
//     halo slab test, locals/ghosts compaction           k_dd_flags, k_scan, k_dd_members
//     centres (locals [+ first-layer ghosts, wide])      k_centre_flags, k_scan, k_centre_compact
//     cell grid over member images                       k_cell_count, k_scan, k_cell_fill
//     canonical neighbour rows (+ ghost reverse lists)   k_neighbors
//     DPA-1 forward / fit / exact backward               k_centre_forward, k_fit_*, k_centre_backward
//     deterministic force gather + per-atom assembly     k_force_gather, k_assemble, k_energy_virial
//   cross-process force/energy/virial reduction          ncclAllReduce (world_size > 1)
// One host read-back per rank (the DD-build counts, to size the rest of the step).
#include "context.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <fstream>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

namespace nb {

#define CU(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

static inline int shift_x_host(int p) { return p / 9 - 1; }
static inline int shift_y_host(int p) { return (p / 3) % 3 - 1; }
static inline int shift_z_host(int p) { return p % 3 - 1; }

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
void DevBuf<T>::ensure(size_t n) {
  if (p && n <= cap) return;
  release();
  const size_t c = std::max<size_t>(n + n / 4, 64);
  CU(cudaMalloc(reinterpret_cast<void**>(&p), c * sizeof(T)));
  cap = c;
}
template <class T>
void DevBuf<T>::release() {
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
}
template struct DevBuf<int>;
template struct DevBuf<float>;
template struct DevBuf<float4>;
template struct DevBuf<double>;
template struct DevBuf<int64_t>;
template struct DevBuf<uint8_t>;
template struct DevBuf<unsigned long long>;

// partition_ranks (decomp.cpp:17-57): minimise subdomain surface; ties -> most balanced
// (sorted-descending dims smallest), then lexicographically largest dims.
std::vector<int> partition_ranks(const double L[3], int R, double min_edge) {
  require(R >= 1, "partition_ranks: n_ranks must be >= 1");
  bool have = false;
  std::vector<int> best(3), best_sorted(3);
  double best_surf = 0;
  for (int px = 1; px <= R; ++px) {
    if (R % px) continue;
    for (int py = 1; py <= R / px; ++py) {
      if ((R / px) % py) continue;
      const int pz = R / px / py;
      const double a = L[0] / px, b = L[1] / py, c = L[2] / pz;
      if (std::min({a, b, c}) < min_edge) continue;
      const double surf = 2.0 * (a * b + b * c + c * a);
      std::vector<int> dims{px, py, pz}, srt = dims;
      std::sort(srt.begin(), srt.end(), std::greater<int>());
      if (!have || surf < best_surf ||
          (surf == best_surf && (srt < best_sorted || (srt == best_sorted && dims > best)))) {
        have = true;
        best = dims;
        best_sorted = srt;
        best_surf = surf;
      }
    }
  }
  require(have, "partition_ranks: no factorization of " + std::to_string(R) +
                    " ranks fits the halo constraints of this box; use a smaller rank count");
  return best;
}

Context::Context(const Model& m, const nnmd_b200_opts& o) : model_(m), opts_(o) {
  model_.validate();
  require(o.n_ranks >= 1, "nnmd_b200: n_ranks must be >= 1");
  require(m.n_max >= 1 && m.n_max < 1024, "nnmd_b200: n_max must be below 1024");
  require(o.scheme == NNMD_MASKED_REDUCTION || o.scheme == NNMD_WIDE_HALO, "nnmd_b200: bad scheme");
  require(o.precision == NNMD_PREC_FP32 || o.precision == NNMD_PREC_TF32 || o.precision == NNMD_PREC_FP32_SIMT,
          "nnmd_b200: unsupported precision");
  require(o.world_size >= 1 && o.world_rank >= 0 && o.world_rank < o.world_size,
          "nnmd_b200: bad world_size/world_rank");
  require(model_.na <= 16 && model_.embed.size() <= kMaxLayers && model_.fit.size() <= kMaxLayers,
          "nnmd_b200: at most 16 attention layers and 8 layers per MLP");
  CU(cudaSetDevice(o.device));
  CU(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, o.device));
  n_sm_ = prop.multiProcessorCount;
  // trace epoch: a device event paired with the host steady clock
  CU(cudaEventCreate(&epoch_ev_));
  CU(cudaEventCreate(&md_ev_[0]));
  CU(cudaEventCreate(&md_ev_[1]));
  CU(cudaEventRecord(epoch_ev_, st_));
  CU(cudaEventSynchronize(epoch_ev_));
  epoch_host_ = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  wh_ = fold_weights(model_);
  weights_.ensure(wh_.blob.size());
  CU(cudaMemcpy(weights_.p, wh_.blob.data(), wh_.blob.size() * sizeof(float), cudaMemcpyHostToDevice));
  build_weight_images();
  CU(cudaMallocHost(reinterpret_cast<void**>(&h_flags_), (kFlagWords + 64) * sizeof(int)));
  CU(cudaMallocHost(reinterpret_cast<void**>(&h_rcnt_), kMaxRanks * kMaxRanks * sizeof(int)));
  CU(cudaMallocHost(reinterpret_cast<void**>(&h_rstat_), kMaxRanks * kCntWords * sizeof(int)));
  CU(cudaMallocHost(reinterpret_cast<void**>(&h_md_err_), sizeof(int)));
  require(o.n_ranks <= 48, "nnmd_b200: at most 48 DD ranks");
  stats_.resize(static_cast<size_t>(o.n_ranks));
  debug_.resize(static_cast<size_t>(o.n_ranks));
  // NNMD_FORCE_NCCL=1 creates the communicator even for one process (exercises the NCCL
  // path -- dlopen, ncclCommInitRank, ncclAllReduce -- on a single GPU).
  use_nccl_ = o.world_size > 1 || getenv("NNMD_FORCE_NCCL") != nullptr;
  if (use_nccl_) {
    const Nccl& N = nccl();
    require(N.ok, "nnmd_b200: NCCL unavailable: " + N.err);
    NcclUid uid;
    if (o.nccl_id) {
      std::memcpy(&uid, o.nccl_id, sizeof uid);
    } else {
      require(o.world_size == 1, "nnmd_b200: world_size > 1 needs an nccl_id");
      const int r0 = N.GetUniqueId(&uid);
      if (r0 != 0) throw CudaError(std::string("ncclGetUniqueId: ") + N.GetErrorString(r0));
    }
    const int r = N.CommInitRank(&comm_, o.world_size, uid, o.world_rank);
    if (r != 0) throw CudaError(std::string("ncclCommInitRank: ") + N.GetErrorString(r));
  }
}

Context::~Context() {
  if (comm_) nccl().CommDestroy(comm_);
  for (auto e : pool_) cudaEventDestroy(e);
  if (epoch_ev_) cudaEventDestroy(epoch_ev_);
  for (auto e : md_ev_)
    if (e) cudaEventDestroy(e);
  if (h_flags_) cudaFreeHost(h_flags_);
  if (h_rcnt_) cudaFreeHost(h_rcnt_);
  if (h_rstat_) cudaFreeHost(h_rstat_);
  if (h_md_err_) cudaFreeHost(h_md_err_);
  if (h_out_) cudaFreeHost(h_out_);
  if (st_) cudaStreamDestroy(st_);
}

void Context::tic(const char* name) {
  if (pool_used_ + 2 > pool_.size()) {
    for (int i = 0; i < 32; ++i) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      pool_.push_back(e);
    }
  }
  Timer t{name, pool_[pool_used_], pool_[pool_used_ + 1]};
  pool_used_ += 2;
  CU(cudaEventRecord(t.a, st_));
  timers_.push_back(t);
  nvtxRangePushA(name);  // the same phase names for nsys / ncu NVTX filtering
}

void Context::toc() {
  check_launch(timers_.back().name.c_str());
  CU(cudaEventRecord(timers_.back().b, st_));
  nvtxRangePop();
}

void Context::collect_times() {
  ktimes_.clear();
  for (const auto& t : timers_) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, t.a, t.b));
    ktimes_.push_back({t.name, ms});
  }
  for (const auto& ph : phases_) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, timers_[ph.t0].a, timers_[ph.t1].b));
    stats_[static_cast<size_t>(ph.rank)].ms[ph.phase] += ms;
  }
}

void Context::compute_device(long n, const double* d_pos, const int* d_types,
                             const int64_t* d_gid, const double box[3],
                             const uint8_t periodic[3], double* d_out) {
  const Model& m = model_;
  require(n >= 0 && n < INT_MAX / 32, "nnmd_b200: bad atom count");
  for (int a = 0; a < 3; ++a) {
    require(box[a] > 0.0, "SimBox: non-positive edge length");
    if (periodic[a])
      require(box[a] >= 2.0 * m.rc, "SimBox: periodic edge shorter than 2*rc (minimum image invalid)");
  }
  const bool wide = opts_.scheme == NNMD_WIDE_HALO;
  const double thickness = wide ? 2.0 * m.rc : m.rc;
  const std::vector<int> dims = partition_ranks(box, opts_.n_ranks, thickness);
  for (int a = 0; a < 3; ++a) {
    require(box[a] / dims[a] >= thickness, "dd_evaluate: subdomain edge shorter than the halo thickness");
    require(!periodic[a] || thickness <= box[a],
            "build_halo: thickness exceeds the box (single image layer insufficient)");
  }
  timers_.clear();
  phases_.clear();
  pool_used_ = 0;
  for (auto& s : stats_) s = RankStat{};
  const int R = opts_.n_ranks;
  // step result: per-rank [E, W] rows, forces and atom energies of the owned atoms (each
  // element has exactly one writer, so the cross-process sum is exact)
  red_.ensure(10 * static_cast<size_t>(R) + 4 * static_cast<size_t>(n) + 1);
  CU(cudaMemsetAsync(red_.p, 0, (10 * static_cast<size_t>(R) + 4 * static_cast<size_t>(n)) * sizeof(double), st_));
  fown_.ensure(3 * static_cast<size_t>(n) + 3);
  rcnt_.ensure(2 * static_cast<size_t>(R) * R);
  CU(cudaMemsetAsync(rcnt_.p, 0, 2 * static_cast<size_t>(R) * R * sizeof(int), st_));
  route_cap_ = 0;
  owner_.ensure(static_cast<size_t>(n) + 1);
  err_.ensure(8);
  CU(cudaMemsetAsync(err_.p, 0x7f, 8 * sizeof(int), st_));
  rstat_.ensure(static_cast<size_t>(R) * kCntWords);
  // ghost capacities per DD rank: kept from the last step with this atom count (grown
  // when a step overflows them), else estimated from the halo geometry -- the ghosts of
  // a subdomain of edges e_a with halo thickness t are about (n / R) (prod (e_a + 2t) / e_a
  // - 1), with 50 % headroom for density fluctuations
  if (cap_n_ != n || cap_gh_.size() != static_cast<size_t>(R)) {
    double f = 1.0;
    for (int a = 0; a < 3; ++a) {
      const double e = box[a] / dims[a];
      f *= (e + 2.0 * thickness) / e;
    }
    double est = static_cast<double>(n) / R * (f - 1.0) * 1.5 + 1024.0;
    double loc = std::min(static_cast<double>(n), static_cast<double>(n) / R * 1.5 + 1024.0);
    if (const char* e = getenv("NNMD_GHOST_CAP")) est = atof(e);  // tests: force the overflow / redo path
    if (const char* e = getenv("NNMD_LOCAL_CAP")) loc = atof(e);
    cap_gh_.assign(static_cast<size_t>(R), static_cast<int>(std::min(est, 27.0 * static_cast<double>(n) + 64.0)));
    cap_loc_.assign(static_cast<size_t>(R), static_cast<int>(loc));
    cap_n_ = n;
  }
  SysArgs sys{};
  sys.pos = d_pos;
  sys.species = d_types;
  sys.gid = d_gid;
  sys.n = static_cast<int>(n);
  sys.n_species = m.ns;
  for (int a = 0; a < 3; ++a) {
    sys.L[a] = box[a];
    sys.per[a] = periodic[a] ? 1 : 0;
  }
  // collective 1 (gather_positions, decomp.cpp:157-186, 285-296): every process takes the
  // positions of world rank 0 (ncclBroadcast of f64 [n][3]); ids and types are static
  if (bcast_positions()) {
    bpos_.ensure(3 * static_cast<size_t>(n) + 3);
    tic("nccl_broadcast");
    const Nccl& N = nccl();
    const int rc = N.Broadcast(d_pos, bpos_.p, 3 * static_cast<size_t>(n), kNcclFloat64, 0, comm_, st_);
    if (rc != 0) throw CudaError(std::string("ncclBroadcast: ") + N.GetErrorString(rc));
    toc();
    sys.pos = bpos_.p;
  }
  tic("owner");
  launch_owner(sys, dims.data(), owner_.p, err_.p, st_);
  toc();
  // step flags: [0, 8) = -err (so a max-reduction keeps the lowest failing atom), [8, 8+R)
  // = ghost-route entries of each DD rank (written by its owning process only)
  flags_.ensure(kFlagWords + opts_.n_ranks);
  CU(cudaMemsetAsync(flags_.p, 0, (kFlagWords + opts_.n_ranks) * sizeof(int), st_));
  for (int r = 0; r < opts_.n_ranks; ++r)
    if (r % opts_.world_size == opts_.world_rank) run_rank(r, sys, dims.data(), thickness, keep_debug_);
  launch_negate(err_.p, flags_.p, kFlagWords, st_);
  route_and_reduce(n, d_out);
  // the step's one host synchronisation (two more with several processes: the route
  // counts, inside route_and_reduce, and none for the DD build)
  CU(cudaMemcpyAsync(h_flags_, flags_.p, (kFlagWords + opts_.n_ranks) * sizeof(int), cudaMemcpyDeviceToHost, st_));
  CU(cudaMemcpyAsync(h_rstat_, rstat_.p, static_cast<size_t>(R) * kCntWords * sizeof(int), cudaMemcpyDeviceToHost, st_));
  if (md_check_) {
    // run_md: the finite-force check rides on the same read-back (engine.cpp:166-176)
    launch_force_check(*md_check_, st_);
    CU(cudaMemcpyAsync(h_md_err_, md_check_->err, sizeof(int), cudaMemcpyDeviceToHost, st_));
  }
  CU(cudaStreamSynchronize(st_));
  if (-h_flags_[0] != 0x7f7f7f7f) {  // bad input on any rank (k_owner), reported before anything else
    const int atom = -h_flags_[0];
    int sp = 0;
    CU(cudaMemcpy(&sp, d_types + atom, sizeof sp, cudaMemcpyDeviceToHost));
    if (sp < 0 || sp >= m.ns) throw Error("dd_evaluate: species id outside the model's species table");
    throw Error("neighbor list: positions must be wrapped into [0, L) on periodic axes");
  }
  if (-h_flags_[3] != 0x7f7f7f7f) {
    // a ghost / centre capacity overflowed on some rank: grow to the exact counts (+25 %)
    // and redo the step (the outputs of this pass are discarded)
    bool grown = false;
    for (int r = 0; r < R; ++r) {
      if (r % opts_.world_size != opts_.world_rank) continue;
      const int* c = h_rstat_ + static_cast<size_t>(r) * kCntWords;
      const int cap = static_cast<int>(c[kCntGhExact] * 1.25) + 1024;
      if (cap > cap_gh_[static_cast<size_t>(r)]) {
        cap_gh_[static_cast<size_t>(r)] = cap;
        grown = true;
      }
      const int capl = std::min(static_cast<int>(n), static_cast<int>(c[kCntLocExact] * 1.25) + 1024);
      if (c[kCntLocExact] > cap_loc_[static_cast<size_t>(r)]) {
        cap_loc_[static_cast<size_t>(r)] = capl;
        grown = true;
      }
    }
    // with several processes another process may be the one that overflowed: every process
    // redoes the step (the flags are all-reduced), growing all its capacities
    if (!grown) {
      for (auto& c : cap_gh_) c = static_cast<int>(c * 1.5) + 1024;
      for (auto& c : cap_loc_) c = std::min(static_cast<int>(n), static_cast<int>(c * 1.5) + 1024);
    }
    require(redo_depth_ < 4, "nnmd_b200: ghost capacity did not converge");
    ++redo_depth_;
    struct Reset {
      int& d;
      ~Reset() { --d; }
    } reset{redo_depth_};
    compute_device(n, d_pos, d_types, d_gid, box, periodic, d_out);
    return;
  }
  collect_times();
  for (int r = 0; r < R; ++r) {
    if (r % opts_.world_size != opts_.world_rank) continue;
    const int* c = h_rstat_ + static_cast<size_t>(r) * kCntWords;
    RankStat& st = stats_[static_cast<size_t>(r)];
    st.counts[0] = c[kCntLoc];
    st.counts[1] = c[kCntGh];
    st.counts[2] = c[kCntCen];
  }
  if (opts_.scheme == NNMD_MASKED_REDUCTION)
    for (int r = 0; r < opts_.n_ranks; ++r) stats_[static_cast<size_t>(r)].counts[3] = h_flags_[kFlagWords + r];
  if (use_nccl_) {
    double comm = 0;
    for (const auto& kt : ktimes_)
      if (kt.first.rfind("nccl_", 0) == 0) comm += kt.second;
    for (auto& s : stats_) s.ms[3] += comm;
  }
  if (trace_on_ || ledger_on_) {
    std::vector<int> local;
    for (int r = 0; r < opts_.n_ranks; ++r)
      if (r % opts_.world_size == opts_.world_rank) local.push_back(r);
    record_trace(n, local);
  }
  const int ovf0 = -h_flags_[1], ovf1 = -h_flags_[2];
  if (ovf0 != 0x7f7f7f7f || ovf1 != 0x7f7f7f7f) {
    const int atom = std::min(ovf0, ovf1);
    int64_t gid = atom;
    if (d_gid) CU(cudaMemcpy(&gid, d_gid + atom, sizeof gid, cudaMemcpyDeviceToHost));
    int own = 0;
    CU(cudaMemcpy(&own, owner_.p + atom, sizeof own, cudaMemcpyDeviceToHost));
    throw CapacityError("dd_evaluate: neighbor overflow at atom id " + std::to_string(gid) +
                        " on rank " + std::to_string(own) + " (n_max " + std::to_string(m.n_max) + ")");
  }
}

std::vector<RouteOp> route_schedule(int R, int ws, int wr, const int* counts) {
  require(R >= 1 && R <= kMaxRanks && ws >= 1 && wr >= 0 && wr < ws && counts, "route_schedule: bad argument");
  auto local = [&](int r) { return r % ws == wr; };
  std::vector<RouteOp> ops;
  for (int s = 0; s < R; ++s) {
    long soff = 0, roff = 0;
    for (int o = 0; o < R; ++o) {
      const int c = counts[s * R + o];
      require(c >= 0, "route_schedule: negative count");
      if (c > 0 && local(s) && !local(o)) ops.push_back({0, s, o, o % ws, soff, c});
      if (c > 0 && !local(s) && local(o)) ops.push_back({1, s, o, s % ws, roff, c});
      soff += c;
      if (local(o)) roff += c;
    }
  }
  return ops;
}

// Ghost-force route and reduce_forces (decomp.cpp:445-538).  Every DD rank has packed the
// owner's zero-image partials of its locals (fown, e_i) and its routed ghost partials,
// grouped by owner rank (run_rank).  With several processes the (source, destination)
// entry counts are all-reduced and the entries move point to point (ncclSend/ncclRecv,
// one grouped call; only pairs with entries).  Each process then merges, for the atoms its
// ranks own: zero-image partial first, then routed partials in (zero image first, image,
// rank) order -- the reference's merge order, and independent of arrival order.  Every
// element of the result [rows | F | e_i] has exactly one writer, so the final all-reduce
// is exact; the per-rank [E, W] rows are summed in rank order (launch_finalize).
void Context::route_and_reduce(long n, double* d_out) {
  const int R = opts_.n_ranks, ws = opts_.world_size, wr = opts_.world_rank;
  const bool masked = opts_.scheme == NNMD_MASKED_REDUCTION;
  const bool multi = use_nccl_ && ws > 1;
  MergeArgs ma{};
  ma.n_ranks = R;
  ma.world_size = ws;
  ma.world_rank = wr;
  ma.n_atoms = static_cast<int>(n);
  ma.cnt = rcnt_.p;
  long capacity = route_cap_;
  for (int s = 0; s < R; ++s) ma.src_base[s] = route_buf_[s].p;
  if (multi && masked) {
    tic("nccl_route");
    const Nccl& N = nccl();
    int rc = N.AllReduce(rcnt_.p, rcnt_.p, static_cast<size_t>(R) * R, kNcclInt32, kNcclSum, comm_, st_);
    if (rc != 0) throw CudaError(std::string("ncclAllReduce (route counts): ") + N.GetErrorString(rc));
    CU(cudaMemcpyAsync(h_rcnt_, rcnt_.p, static_cast<size_t>(R) * R * sizeof(int), cudaMemcpyDeviceToHost, st_));
    CU(cudaStreamSynchronize(st_));
    auto local = [&](int r) { return r % ws == wr; };
    for (int s = 0; s < R; ++s) {
      if (local(s)) continue;
      long tot = 0;
      for (int o = 0; o < R; ++o)
        if (local(o)) tot += h_rcnt_[s * R + o];
      recv_buf_[s].ensure(static_cast<size_t>(tot) + 1);
      ma.src_base[s] = recv_buf_[s].p;
      capacity += tot;
    }
    rc = N.GroupStart();
    for (const RouteOp& op : route_schedule(R, ws, wr, h_rcnt_)) {
      if (rc != 0) break;
      const size_t bytes = static_cast<size_t>(op.count) * sizeof(RouteEntry);
      if (op.kind == 0) rc = N.Send(route_buf_[op.src].p + op.offset, bytes, kNcclUint8, op.peer, comm_, st_);
      else rc = N.Recv(recv_buf_[op.src].p + op.offset, bytes, kNcclUint8, op.peer, comm_, st_);
    }
    const int rc2 = N.GroupEnd();
    if (rc == 0) rc = rc2;
    if (rc != 0) throw CudaError(std::string("ncclSend/ncclRecv (ghost-force route): ") + N.GetErrorString(rc));
    toc();
  }
  inc_cnt_.ensure(static_cast<size_t>(n) + 1);
  inc_off_.ensure(static_cast<size_t>(n) + 1);
  seg_.ensure(2 * static_cast<size_t>(R) * R + 1);
  ma.seg = seg_.p;
  ma.inc_cnt = inc_cnt_.p;
  ma.inc_off = inc_off_.p;
  ma.owner = owner_.p;
  ma.fown = fown_.p;
  ma.f_out = red_.p + 10 * static_cast<size_t>(R);
  auto merge = [&](MergeArgs& a, long cap) {
    inc_.ensure(static_cast<size_t>(cap) + 1);
    CU(cudaMemsetAsync(inc_cnt_.p, 0, (static_cast<size_t>(n) + 1) * sizeof(int), st_));
    a.inc = inc_.p;
    a.capacity = static_cast<int>(cap);
    launch_route_merge(a, st_);
  };
  tic("route_merge");
  // Test hook (NNMD_EMULATE_WORLD=W, one process): run the several-process route as W
  // processes would -- the plan of every emulated process, its receives as device copies
  // from the senders' grouped buffers, and its merge over the atoms it owns -- so the
  // multi-process layout (receive buffers, remote segment offsets) is checked on one GPU
  // against the single-process result (tests/test_gpu_parity.py).
  static const int emulate = getenv("NNMD_EMULATE_WORLD") ? atoi(getenv("NNMD_EMULATE_WORLD")) : 0;
  if (emulate > 1 && !multi && masked && ws == 1) {
    CU(cudaMemcpyAsync(h_rcnt_, rcnt_.p, static_cast<size_t>(R) * R * sizeof(int), cudaMemcpyDeviceToHost, st_));
    CU(cudaStreamSynchronize(st_));
    for (int fw = 0; fw < emulate; ++fw) {
      MergeArgs me = ma;
      me.world_size = emulate;
      me.world_rank = fw;
      long cap = route_cap_;
      for (int s2 = 0; s2 < R; ++s2) {
        me.src_base[s2] = route_buf_[s2].p;
        if (s2 % emulate == fw) continue;
        long tot = 0;
        for (int o = 0; o < R; ++o)
          if (o % emulate == fw) tot += h_rcnt_[s2 * R + o];
        recv_buf_[s2].ensure(static_cast<size_t>(tot) + 1);
        me.src_base[s2] = recv_buf_[s2].p;
        cap += tot;
      }
      for (const RouteOp& op : route_schedule(R, emulate, fw, h_rcnt_)) {
        if (op.kind != 1) continue;
        long soff = 0;  // the sender's group offset (its own send op's offset)
        for (int o = 0; o < op.dst; ++o) soff += h_rcnt_[op.src * R + o];
        CU(cudaMemcpyAsync(recv_buf_[op.src].p + op.offset, route_buf_[op.src].p + soff,
                           static_cast<size_t>(op.count) * sizeof(RouteEntry), cudaMemcpyDeviceToDevice, st_));
      }
      merge(me, cap);
    }
  } else {
    merge(ma, capacity);
  }
  toc();
  if (use_nccl_) {
    // collective 2 (reduce_forces, decomp.cpp:188-204): the result rows, forces and atom
    // energies summed over processes (one writer per element: exact); then the error
    // words and route counts, so that every process sees an overflow on any rank and all
    // of them throw together
    tic("nccl_allreduce");
    const Nccl& N = nccl();
    const size_t len = 10 * static_cast<size_t>(R) + 4 * static_cast<size_t>(n);
    int rc = N.AllReduce(red_.p, red_.p, len, kNcclFloat64, kNcclSum, comm_, st_);
    if (rc == 0) rc = N.AllReduce(flags_.p, flags_.p, kFlagWords + R, kNcclInt32, kNcclMax, comm_, st_);
    if (rc != 0) throw CudaError(std::string("ncclAllReduce: ") + N.GetErrorString(rc));
    toc();
  }
  launch_finalize(red_.p, R, n, d_out, st_);
}

void Context::run_rank(int rank, const SysArgs& sys, const int dims[3], double thickness,
                       bool keep_debug) {
  const Model& m = model_;
  const int n = sys.n;
  const bool wide = opts_.scheme == NNMD_WIDE_HALO;
  RankArgs ra{};
  ra.rank = rank;
  ra.wide = wide;
  const int idx[3] = {rank / (dims[1] * dims[2]), (rank / dims[2]) % dims[1], rank % dims[2]};
  for (int a = 0; a < 3; ++a) {
    ra.dims[a] = dims[a];
    const double edge = sys.L[a] / dims[a];
    ra.lo[a] = idx[a] * edge;
    ra.hi[a] = (idx[a] + 1) * edge;
    const double guard = 1e-12 * sys.L[a];  // kHaloSlabGuard (decomp.hpp:55)
    ra.slab_lo[a] = ra.lo[a] - thickness - guard;
    ra.slab_hi[a] = ra.hi[a] + thickness + guard;
    ra.rc_lo[a] = ra.lo[a] - m.rc - guard;
    ra.rc_hi[a] = ra.hi[a] + m.rc + guard;
  }
  RankStat& stat = stats_[static_cast<size_t>(rank)];
  const size_t ph_dd0 = timers_.size();

  // ---- DD build: locals + halo ------------------------------------------------------
  is_local_.ensure(n + 1);
  gcount_.ensure(n + 1);
  loc_off_.ensure(n + 1);
  gh_off_.ensure(n + 1);
  counts_.ensure(kCntWords);
  tic("dd_flags");
  launch_dd_flags(sys, ra, owner_.p, is_local_.p, gcount_.p, st_);
  toc();
  tic("scan");
  launch_scan(is_local_.p, loc_off_.p, n, st_);
  launch_scan(gcount_.p, gh_off_.p, n, st_);
  toc();
  // No host read-back here: every buffer below is sized by a capacity (locals <= n, ghosts
  // <= cap_gh_[rank], centres <= n, or <= members for wide_halo) and every kernel takes its
  // live counts from counts_ on the device.  An overflowing capacity is flagged (err_[3])
  // and the step is redone with exact sizes (compute_device); bad input (err_[0]) raises
  // at the step's end.
  const int ngh = cap_gh_[static_cast<size_t>(rank)];  // capacities
  const int nloc = cap_loc_[static_cast<size_t>(rank)];
  const int nm = nloc + ngh;
  launch_rank_counts(loc_off_.p, gh_off_.p, n, nloc, ngh, counts_.p, err_.p + 3, st_);
  m_atom_.ensure(nm + 1);
  m_shift_.ensure(nm + 1);
  m_owner_.ensure(nm + 1);
  m_pos_.ensure(3 * static_cast<size_t>(nm) + 3);
  m_cell_.ensure(nm + 1);
  cflag_.ensure(nm + 1);
  coff_.ensure(nm + 1);
  cen_member_.ensure(nm + 1);
  cidx_.ensure(nm + 1);
  tic("dd_members");
  launch_dd_members(sys, ra, owner_.p, loc_off_.p, gh_off_.p, n, nm, m_atom_.p, m_shift_.p, m_pos_.p,
                    m_owner_.p, st_);
  launch_centre_flags(ra, counts_.p, m_pos_.p, nm, cflag_.p, st_);
  launch_scan_dev(cflag_.p, coff_.p, counts_.p + kCntMem, st_);
  const int ncen = wide ? nm : nloc;  // capacity
  launch_centre_compact(cflag_.p, coff_.p, counts_.p, nm, wide, ncen, cen_member_.p, cidx_.p, err_.p + 3, st_);
  toc();
  (void)stat;  // counts are read back with the step flags (compute_device)
  phases_.push_back({rank, 0, ph_dd0, timers_.size() - 1});

  // ---- cell grid + neighbour rows ------------------------------------------------------
  const size_t ph_nb0 = timers_.size();
  CellArgs cg{};
  long ncell = 1;
  for (int a = 0; a < 3; ++a) {
    const double ext = ra.slab_hi[a] - ra.slab_lo[a];
    cg.origin[a] = ra.slab_lo[a];
    cg.dims[a] = std::max(1, std::min(1024, static_cast<int>(std::floor(ext / (m.rc * (1.0 + 1e-6))))));
    cg.width[a] = ext / cg.dims[a];
    ncell *= cg.dims[a];
  }
  cell_count_.ensure(ncell + 1);
  cell_start_.ensure(ncell + 1);
  cell_fill_.ensure(ncell + 1);
  cell_members_.ensure(nm + 1);
  cs_x_.ensure(3 * static_cast<size_t>(nm) + 3);
  cs_i_.ensure(2 * static_cast<size_t>(nm) + 2);
  cs_gid_.ensure(static_cast<size_t>(nm) + 1);
  CellSorted csd{};
  csd.pos = sys.pos;
  csd.atom_species = sys.species;
  csd.atom_gid = sys.gid;
  csd.m_atom = m_atom_.p;
  csd.m_shift = m_shift_.p;
  csd.x = cs_x_.p;
  csd.y = cs_x_.p + nm;
  csd.z = cs_x_.p + 2 * static_cast<size_t>(nm);
  csd.shift = cs_i_.p;
  csd.species = cs_i_.p + nm;
  csd.gid = cs_gid_.p;
  csd.n_species = m.ns;
  tic("cells");
  CU(cudaMemsetAsync(cell_count_.p, 0, (ncell + 1) * sizeof(int), st_));
  CU(cudaMemsetAsync(cell_fill_.p, 0, (ncell + 1) * sizeof(int), st_));
  launch_cell_count(cg, m_pos_.p, counts_.p + kCntMem, nm, m_cell_.p, cell_count_.p, st_);
  launch_scan(cell_count_.p, cell_start_.p, static_cast<int>(ncell), st_);
  launch_cell_fill(m_cell_.p, counts_.p + kCntMem, nm, cell_start_.p, cell_fill_.p, cell_members_.p, csd, st_);
  toc();
  const int nmax = m.n_max;
  nlist_.ensure(static_cast<size_t>(ncen) * nmax + 1);
  nn_.ensure(ncen + 1);
  NbrArgs na{};
  na.pos = sys.pos;
  na.species = sys.species;
  na.gid = sys.gid;
  for (int a = 0; a < 3; ++a) {
    na.L[a] = sys.L[a];
    na.cdims[a] = cg.dims[a];
  }
  na.m_atom = m_atom_.p;
  na.m_shift = m_shift_.p;
  na.m_cell = m_cell_.p;
  na.cell_start = cell_start_.p;
  na.cell_members = cell_members_.p;
  na.cs = csd;
  na.n_max = nmax;
  na.rc2 = m.rc * m.rc;
  {
    // sort keys pack (species, bits(r2)) into 64 bits: r2 < rc2 has an exponent field <=
    // that of rc2, so 6 exponent bits (2^-63 of rc2 and up) plus the 52 mantissa bits fit
    uint64_t rb;
    std::memcpy(&rb, &na.rc2, sizeof rb);
    const uint64_t emax = rb >> 52;
    na.kbase = emax >= 63 ? (emax - 63) << 52 : 0;
  }
  na.centre_member = cen_member_.p;
  na.n_lists = ncen;
  na.n_lists_dev = counts_.p + kCntCen;
  na.cand_limit = INT_MAX;
  na.nlist = nlist_.p;
  na.nn = nn_.p;
  na.err = err_.p + 1;
  na.nonempty = nullptr;
  maxn_.ensure(1);
  CU(cudaMemsetAsync(maxn_.p, 0, sizeof(int), st_));
  na.maxn = maxn_.p;
  // environment matrix fused into the centre-list build (k_neighbors writes R, Z, sigma)
  R_.ensure(static_cast<size_t>(ncen) * nmax + 1);
  Z_.ensure(static_cast<size_t>(ncen) * nmax + 1);
  sig_.ensure(ncen + 1);
  na.R = R_.p;
  na.Z = Z_.p;
  na.sig = sig_.p;
  na.rc = m.rc;
  na.rcs = m.rcs;
  tic("neighbors");
  launch_neighbors(na, st_);
  toc();
  if (!wide) {
    rlist_.ensure(static_cast<size_t>(ngh) * nmax + 1);
    rn_.ensure(ngh + 1);
    NbrArgs rv = na;
    rv.centre_member = nullptr;
    rv.member_offset = nloc;
    rv.member_offset_dev = counts_.p + kCntLoc;
    rv.n_lists = ngh;
    rv.n_lists_dev = counts_.p + kCntGh;
    rv.cand_limit = nloc;
    rv.cand_limit_dev = counts_.p + kCntLoc;
    rv.maxn = nullptr;
    rv.nlist = rlist_.p;
    rv.nn = rn_.p;
    rv.err = err_.p + 2;
    rv.nonempty = counts_.p + kCntRoute;
    rv.R = nullptr;  // reverse lists carry no env rows
    rv.Z = nullptr;
    rv.sig = nullptr;
    tic("neighbors_reverse");
    launch_neighbors(rv, st_);
    toc();
  }
  phases_.push_back({rank, 1, ph_nb0, timers_.size() - 1});

  // ---- network -------------------------------------------------------------------------
  const size_t ph_in0 = timers_.size();
  const int M = m.M, mr = m.mr;
  DpArgs dp{};
  dp.M = M;
  dp.mr = mr;
  dp.n_max = nmax;
  dp.ns = m.ns;
  dp.n_embed = static_cast<int>(m.embed.size());
  dp.n_attn = m.na;
  dp.n_fit = static_cast<int>(m.fit.size());
  const float* W = weights_.p;
  for (int e = 0; e < dp.n_embed; ++e) {
    dp.edims[e] = wh_.edims[static_cast<size_t>(e)];
    dp.ew[e] = e ? W + wh_.ew[static_cast<size_t>(e)] : nullptr;
    dp.eb[e] = e ? W + wh_.eb[static_cast<size_t>(e)] : nullptr;
  }
  dp.w0 = W + wh_.w0;
  dp.ctab = W + wh_.ctab;
  for (int l = 0; l < m.na; ++l) dp.ab[l] = W + wh_.ab[static_cast<size_t>(l)];
  for (int l = 0; l <= dp.n_fit; ++l) dp.fdims[l] = wh_.fdims[static_cast<size_t>(l)];
  for (int l = 0; l < dp.n_fit; ++l) {
    dp.fw[l] = W + wh_.fw[static_cast<size_t>(l)];
    dp.fb[l] = W + wh_.fb[static_cast<size_t>(l)];
  }
  dp.rc = m.rc;
  dp.rcs = m.rcs;
  dp.inv_sqrt_nmax = static_cast<float>(1.0 / std::sqrt(static_cast<double>(nmax)));
  dp.pos = sys.pos;
  dp.species = sys.species;
  for (int a = 0; a < 3; ++a) dp.L[a] = sys.L[a];
  dp.m_atom = m_atom_.p;
  dp.m_shift = m_shift_.p;
  dp.cen_member = cen_member_.p;
  dp.n_centres = ncen;
  dp.n_centres_dev = counts_.p + kCntCen;
  dp.nlist = nlist_.p;
  dp.nn = nn_.p;
  Ad_.ensure(static_cast<size_t>(ncen) * M * 4 + 4);
  Bd_.ensure(static_cast<size_t>(ncen) * 4 * mr + 4);
  D_.ensure(static_cast<size_t>(ncen) * M * mr + 4);
  dD_.ensure(static_cast<size_t>(ncen) * M * mr + 4);
  g_.ensure(static_cast<size_t>(ncen) * nmax * 3 + 3);
  vir_.ensure(static_cast<size_t>(ncen) * 9 + 9);
  e_.ensure(ncen + 1);
  dp.Z = Z_.p;
  dp.sig = sig_.p;
  dp.R = R_.p;
  dp.Ad = Ad_.p;
  dp.Bd = Bd_.p;
  dp.D = D_.p;
  dp.dD = dD_.p;
  dp.g = g_.p;
  dp.vir = vir_.p;
  // diagnostic switches, read per call (tests toggle bit 3, multi-centre units)
  const int flags = getenv("NNMD_FLAGS") ? atoi(getenv("NNMD_FLAGS")) : 0;
  dp.flags = flags;
  if (!(flags & 4) && wimg_.p) {  // bit 2: stage weights through registers instead
    auto img = [&](long off) -> const uint8_t* { return off >= 0 ? wimg_.p + off : nullptr; };
    for (int l = 0; l < m.na; ++l) {
      dp.img_ab[l] = img(wimg_ab_[static_cast<size_t>(l)]);
      dp.img_abT[l] = img(wimg_abT_[static_cast<size_t>(l)]);
    }
    bool all = true;
    for (int l = 0; l < m.na; ++l) all = all && dp.img_ab[l] && dp.img_abT[l];
    for (int e = 1; e < dp.n_embed; ++e) {
      dp.img_ew[e] = img(wimg_ew_[static_cast<size_t>(e)]);
      dp.img_ewT[e] = img(wimg_ewT_[static_cast<size_t>(e)]);
      all = all && dp.img_ew[e] && dp.img_ewT[e];
    }
    dp.wimg = all ? 1 : 0;
  }
  dp.mode = opts_.precision == NNMD_PREC_FP32 ? 1 : opts_.precision == NNMD_PREC_TF32 ? 2 : 0;
  work_.ensure(1);
  dp.work = work_.p;
  // work units: one centre each, or (n_max <= 64, tcgen05 + weight images) packs of up to
  // four consecutive centres in one 128-row tile (NNMD_FLAGS bit 3 disables packing)
  const bool pack = dp.mode != 0 && dp.wimg && nmax <= 64 && !(flags & 8);
  int units = ncen;
  dp.unit_rows = nmax;
  if (pack && ncen > 0) {
    units = pack_capacity(ncen);
    const int ng = (ncen + 3) / 4;
    pack_cnt_.ensure(2 * static_cast<size_t>(ng) + 3);
    packs_.ensure(static_cast<size_t>(units) + 1);
    tic("pack_plan");
    launch_pack_plan(nn_.p, counts_.p + kCntCen, ncen, pack_cnt_.p, pack_cnt_.p + ng + 1, packs_.p, st_);
    toc();
    dp.packs = packs_.p;
    dp.n_units_dev = pack_cnt_.p + ng + 1 + ng;
    dp.unit_rows = 128;
  }
  {
    const size_t ur = static_cast<size_t>(dp.unit_rows);
    const size_t ur4 = (ur + 3) & ~size_t(3);
    dp.x_layer_stride = static_cast<size_t>(units) * ur * M;
    X_.ensure(dp.x_layer_stride * (m.na + 1) + 4);
    dp.u_layer_stride = static_cast<size_t>(units) * ur * 2 * M;
    dp.p_layer_stride = static_cast<size_t>(units) * ur * ur4;
    size_t ew = 0;
    for (int e = 0; e + 1 < dp.n_embed; ++e) ew += static_cast<size_t>(dp.edims[e]);
    dp.emb_centre_stride = ur * ew;
    Ust_.ensure(dp.u_layer_stride * std::max(1, m.na) + 4);
    PUst_.ensure(dp.p_layer_stride * std::max(1, m.na) + 4);
    PTst_.ensure(dp.p_layer_stride * std::max(1, m.na) + 4);
    EMBst_.ensure(dp.emb_centre_stride * units + 4);
    dp.X = X_.p;
    dp.Ust = Ust_.p;
    dp.PUst = PUst_.p;
    dp.PTst = PTst_.p;
    dp.EMBst = EMBst_.p;
  }
  const int grid = std::max(1, std::min(units, 2 * n_sm_));  // two CTAs per SM (SIMT and tcgen05)
  dp.scratch_slot = (dp_scratch_floats(dp) + 31) & ~size_t(31);
  scratch_.ensure(dp.scratch_slot * grid);
  dp.scratch = scratch_.p;
  static const bool prof_fwd = getenv("NNMD_PROFILE_PHASES") != nullptr;
  if (prof_fwd) {
    static DevBuf<unsigned long long> fbuf;
    fbuf.ensure(24);
    CU(cudaMemsetAsync(fbuf.p, 0, 24 * sizeof(unsigned long long), st_));
    dp.prof = fbuf.p;
  }
  tic("centre_forward");
  launch_centre_forward(dp, grid, st_);
  toc();
  if (prof_fwd) {
    unsigned long long h[24];
    CU(cudaMemcpyAsync(h, dp.prof, sizeof h, cudaMemcpyDeviceToHost, st_));
    CU(cudaStreamSynchronize(st_));
    double t0 = 0;
    for (int i = 0; i < 16; ++i) t0 += static_cast<double>(h[i]);
    fprintf(stderr, "[nnmd phases forward] total %.3e cycles:", t0);
    for (int i = 0; i < 16; ++i) fprintf(stderr, " %d:%.1f%%", i, 100.0 * h[i] / (t0 > 0 ? t0 : 1));
    fprintf(stderr, " | gemm-internal:");
    for (int i = 16; i < 24; ++i) fprintf(stderr, " g%d:%.1f%%", i - 16, 100.0 * h[i] / (t0 > 0 ? t0 : 1));
    fprintf(stderr, "\n");
    dp.prof = nullptr;
  }
  FitArgs fa{};
  fa.n_fit = dp.n_fit;
  int maxw = 0;
  size_t ysum = 0;
  for (int l = 0; l <= dp.n_fit; ++l) {
    fa.fdims[l] = dp.fdims[l];
    maxw = std::max(maxw, dp.fdims[l]);
  }
  for (int l = 0; l + 1 < dp.n_fit; ++l) ysum += static_cast<size_t>(dp.fdims[l + 1]);
  fitY_.ensure(ysum * ncen + 4);
  fitd_.ensure(2 * static_cast<size_t>(maxw) * ncen + 4);
  {
    size_t off = 0;
    for (int l = 0; l + 1 < dp.n_fit; ++l) {
      fa.Y[l] = fitY_.p + off;
      off += static_cast<size_t>(dp.fdims[l + 1]) * ncen;
    }
  }
  for (int l = 0; l < dp.n_fit; ++l) {
    fa.fw[l] = dp.fw[l];
    fa.fb[l] = dp.fb[l];
    fa.fwT[l] = W + wh_.fwT[static_cast<size_t>(l)];
  }
  fa.flags = flags;
  fa.n_centres = ncen;
  fa.n_centres_dev = counts_.p + kCntCen;
  fa.D = D_.p;
  fa.delta[0] = fitd_.p;
  fa.delta[1] = fitd_.p + static_cast<size_t>(maxw) * ncen;
  fa.e = e_.p;
  fa.dD = dD_.p;
  fa.mode = dp.mode;
  fa.n_sm = n_sm_;
  fitws_.ensure(fit_workspace_floats(ncen, 256));  // split-K only for layers with N <= 256
  fa.ws = fitws_.p;
  tic("fit");
  launch_fit(fa, st_);
  toc();
  static const bool prof_on = getenv("NNMD_PROFILE_PHASES") != nullptr;
  DevBuf<unsigned long long>* prof = nullptr;
  if (prof_on) {
    static DevBuf<unsigned long long> pbuf;
    pbuf.ensure(24);
    CU(cudaMemsetAsync(pbuf.p, 0, 24 * sizeof(unsigned long long), st_));
    dp.prof = pbuf.p;
    prof = &pbuf;
  }
  tic("centre_backward");
  launch_centre_backward(dp, grid, st_);
  toc();
  if (prof) {
    unsigned long long h[24];
    CU(cudaMemcpyAsync(h, prof->p, sizeof h, cudaMemcpyDeviceToHost, st_));
    CU(cudaStreamSynchronize(st_));
    double tot = 0;
    for (int i = 0; i < 24; ++i) tot += static_cast<double>(h[i]);
    fprintf(stderr, "[nnmd phases backward] total %.3e cycles (thread 0 summed over CTAs):", tot);
    double tot0 = 0;
    for (int i = 0; i < 16; ++i) tot0 += static_cast<double>(h[i]);
    for (int i = 0; i < 16; ++i) fprintf(stderr, " %d:%.1f%%", i, 100.0 * h[i] / (tot0 > 0 ? tot0 : 1));
    fprintf(stderr, " | gemm-internal (share of phase total):");
    for (int i = 16; i < 24; ++i) fprintf(stderr, " g%d:%.1f%%", i - 16, 100.0 * h[i] / (tot0 > 0 ? tot0 : 1));
    fprintf(stderr, "\n");
  }
  phases_.push_back({rank, 2, ph_in0, timers_.size() - 1});

  // ---- forces --------------------------------------------------------------------------
  const size_t ph_f0 = timers_.size();
  fmem_.ensure(3 * static_cast<size_t>(nm) + 3);
  ForceArgs fo{};
  fo.nlist = nlist_.p;
  fo.nn = nn_.p;
  fo.n_max = nmax;
  fo.cidx = cidx_.p;
  fo.rlist = wide ? nullptr : rlist_.p;
  fo.rn = wide ? nullptr : rn_.p;
  fo.counts = counts_.p;
  fo.wide = wide;
  fo.n_targets = wide ? nloc : nm;
  fo.g = g_.p;
  fo.fmem = fmem_.p;
  tic("force_gather");
  launch_force_gather(fo, st_);
  toc();
  // ghost-force route, pack side: the owner's zero-image partials of the locals, the routed
  // ghost partials grouped by owner rank (decomp.cpp:445-455); this rank's [E, W] row
  if (!wide) route_buf_[rank].ensure(static_cast<size_t>(ngh) + 1);
  RouteArgs ro{};
  ro.rank = rank;
  ro.n_ranks = opts_.n_ranks;
  ro.wide = wide;
  ro.nloc = nloc;
  ro.ngh = ngh;
  ro.counts = counts_.p;
  ro.m_atom = m_atom_.p;
  ro.m_shift = m_shift_.p;
  ro.m_owner = m_owner_.p;
  ro.rn = wide ? nullptr : rn_.p;
  ro.fmem = fmem_.p;
  ro.e_centre = e_.p;
  ro.fown = fown_.p;
  ro.eown = red_.p + 10 * static_cast<size_t>(opts_.n_ranks) + 3 * static_cast<size_t>(n);
  ro.cnt = rcnt_.p;
  ro.cur = rcnt_.p + static_cast<size_t>(opts_.n_ranks) * opts_.n_ranks + static_cast<size_t>(rank) * opts_.n_ranks;
  ro.buf = wide ? nullptr : route_buf_[rank].p;
  if (!wide) route_cap_ += ngh;
  tic("route_pack");
  launch_route_pack(ro, st_);
  evpart_.ensure(kEnergyVirialPartials);
  launch_energy_virial(e_.p, vir_.p, counts_.p, evpart_.p, red_.p + 10 * static_cast<size_t>(rank), st_);
  toc();
  phases_.push_back({rank, 3, ph_f0, timers_.size() - 1});
  if (!wide)
    CU(cudaMemcpyAsync(flags_.p + kFlagWords + rank, counts_.p + kCntRoute, sizeof(int), cudaMemcpyDeviceToDevice, st_));
  // the rank's counts, read back with the step flags
  CU(cudaMemcpyAsync(rstat_.p + static_cast<size_t>(rank) * kCntWords, counts_.p, kCntWords * sizeof(int),
                     cudaMemcpyDeviceToDevice, st_));

  if (keep_debug) {
    int hc[kCntWords];
    CU(cudaMemcpyAsync(hc, counts_.p, sizeof hc, cudaMemcpyDeviceToHost, st_));
    CU(cudaStreamSynchronize(st_));
    const int nloc = hc[kCntLoc], ngh = hc[kCntGh], nm = nloc + ngh, ncen = hc[kCntCen];
    RankDebug& d = debug_[static_cast<size_t>(rank)];
    std::vector<int> cm(ncen), mat(nm), msh(nm), mown(nm);
    d.nn.assign(ncen, 0);
    std::vector<int> nl(static_cast<size_t>(ncen) * nmax);
    if (ncen) {
      CU(cudaMemcpy(cm.data(), cen_member_.p, ncen * sizeof(int), cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(d.nn.data(), nn_.p, ncen * sizeof(int), cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(nl.data(), nlist_.p, nl.size() * sizeof(int), cudaMemcpyDeviceToHost));
    }
    if (nm) {
      CU(cudaMemcpy(mat.data(), m_atom_.p, nm * sizeof(int), cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(msh.data(), m_shift_.p, nm * sizeof(int), cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(mown.data(), m_owner_.p, nm * sizeof(int), cudaMemcpyDeviceToHost));
    }
    d.centre_atoms.resize(ncen);
    d.nlist_atom.assign(static_cast<size_t>(ncen) * nmax, -1);
    d.nlist_img.assign(static_cast<size_t>(ncen) * nmax * 3, 0);
    for (int c = 0; c < ncen; ++c) {
      const int mc = cm[c];
      d.centre_atoms[c] = mat[mc];
      const int cs = msh[mc];
      for (int k = 0; k < std::min(d.nn[c], nmax); ++k) {
        const int mj = nl[static_cast<size_t>(c) * nmax + k];
        const int sj = msh[mj];
        d.nlist_atom[static_cast<size_t>(c) * nmax + k] = mat[mj];
        int* im = &d.nlist_img[(static_cast<size_t>(c) * nmax + k) * 3];
        im[0] = shift_x_host(sj) - shift_x_host(cs);
        im[1] = shift_y_host(sj) - shift_y_host(cs);
        im[2] = shift_z_host(sj) - shift_z_host(cs);
      }
    }
    d.ghost_atom.assign(mat.begin() + nloc, mat.end());
    d.ghost_owner.assign(mown.begin() + nloc, mown.end());
    d.ghost_shift.resize(static_cast<size_t>(ngh) * 3);
    for (int gI = 0; gI < ngh; ++gI) {
      const int s = msh[nloc + gI];
      d.ghost_shift[3 * gI] = shift_x_host(s);
      d.ghost_shift[3 * gI + 1] = shift_y_host(s);
      d.ghost_shift[3 * gI + 2] = shift_z_host(s);
    }
  }
}

void Context::debug_rank(int rank, RankDebug& out) {
  require(rank >= 0 && rank < opts_.n_ranks, "debug: bad rank");
  require(keep_debug_, "debug: enable debug capture before compute");
  out = debug_[static_cast<size_t>(rank)];
}

void Context::compute_host(long n, const double* pos, const int* types, const int64_t* gid,
                           const double box[3], const uint8_t periodic[3], double* energy,
                           double* forces, double* virial, double* atom_energy) {
  for (long i = 0; i < n; ++i)
    require(types[i] >= 0 && types[i] < model_.ns,
            "dd_evaluate: species id outside the model's species table");
  pos_.ensure(3 * static_cast<size_t>(n) + 3);
  types_.ensure(static_cast<size_t>(n) + 1);
  gid_.ensure(static_cast<size_t>(n) + 1);
  out_.ensure(10 + 4 * static_cast<size_t>(n));
  if (n) {
    // with the position broadcast only world rank 0's coordinates are used (others may pass
    // NULL): collective 1 replaces the replicated host input
    if (coords_needed()) {
      require(pos != nullptr, "nnmd_b200_compute: null coordinates on world rank 0");
      CU(cudaMemcpyAsync(pos_.p, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st_));
    }
    CU(cudaMemcpyAsync(types_.p, types, n * sizeof(int), cudaMemcpyHostToDevice, st_));
    if (gid) {
      CU(cudaMemcpyAsync(gid_.p, gid, n * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
    } else {
      std::vector<int64_t> iota(static_cast<size_t>(n));
      for (long i = 0; i < n; ++i) iota[static_cast<size_t>(i)] = i;
      CU(cudaMemcpyAsync(gid_.p, iota.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
      CU(cudaStreamSynchronize(st_));
    }
  }
  compute_device(n, pos_.p, types_.p, gid_.p, box, periodic, out_.p);
  // the result [E, W(9), F(3n), e_i(n)] comes back in one copy into pinned staging (a
  // device-to-pageable copy is staged by the driver chunk by chunk), then to the caller
  const size_t words = 10 + (atom_energy ? 4 : 3) * static_cast<size_t>(n);
  if (h_out_cap_ < words) {
    if (h_out_) CU(cudaFreeHost(h_out_));
    h_out_ = nullptr;
    h_out_cap_ = 0;
    CU(cudaMallocHost(reinterpret_cast<void**>(&h_out_), (10 + 4 * static_cast<size_t>(n)) * sizeof(double)));
    h_out_cap_ = 10 + 4 * static_cast<size_t>(n);
  }
  CU(cudaMemcpyAsync(h_out_, out_.p, words * sizeof(double), cudaMemcpyDeviceToHost, st_));
  CU(cudaStreamSynchronize(st_));
  if (energy) *energy = h_out_[0];
  if (virial) std::memcpy(virial, h_out_ + 1, 9 * sizeof(double));
  if (n && forces) std::memcpy(forces, h_out_ + 10, 3 * n * sizeof(double));
  if (n && atom_energy) std::memcpy(atom_energy, h_out_ + 10 + 3 * n, n * sizeof(double));
}

// ---- pre-split weight images -----------------------------------------------------------
// B operands of the per-centre weight GEMMs (dp_kernels.cu): U = X [A|B] (K = M, N = 2M),
// dX += dU [A|B]^T (K = 2M, N = M), embedding forward (K = E_in, N = E_out) and backward
// (K = E_out, N = E_in).  Only operands that fit one MMA tile (N <= 256) get an image.
void Context::build_weight_images() {
  const int M = model_.M, M2 = 2 * M;
  const int ne = static_cast<int>(wh_.edims.size());
  struct Job {
    long* slot;
    long w;
    int tb, ldb, K, N;
  };
  std::vector<Job> jobs;
  wimg_ab_.assign(static_cast<size_t>(model_.na), -1);
  wimg_abT_.assign(static_cast<size_t>(model_.na), -1);
  wimg_ew_.assign(static_cast<size_t>(ne), -1);
  wimg_ewT_.assign(static_cast<size_t>(ne), -1);
  for (int l = 0; l < model_.na; ++l) {
    jobs.push_back({&wimg_ab_[static_cast<size_t>(l)], wh_.ab[static_cast<size_t>(l)], 0, M2, M, M2});
    jobs.push_back({&wimg_abT_[static_cast<size_t>(l)], wh_.ab[static_cast<size_t>(l)], 1, M2, M2, M});
  }
  for (int e = 1; e < ne; ++e) {
    const int Ein = wh_.edims[static_cast<size_t>(e - 1)], Eout = wh_.edims[static_cast<size_t>(e)];
    jobs.push_back({&wimg_ew_[static_cast<size_t>(e)], wh_.ew[static_cast<size_t>(e)], 1, Ein, Ein, Eout});
    jobs.push_back({&wimg_ewT_[static_cast<size_t>(e)], wh_.ew[static_cast<size_t>(e)], 0, Ein, Eout, Ein});
  }
  size_t total = 0;
  for (auto& j : jobs) {
    // one MMA tile per image: the SS path (N > 128) covers N <= 256, the TS path N <= 128
    if (j.N > 256) continue;
    *j.slot = static_cast<long>(total);
    total += (weight_image_bytes(j.K, j.N) + 1023) & ~size_t(1023);
  }
  if (total == 0) return;
  wimg_.ensure(total);
  for (auto& j : jobs)
    if (*j.slot >= 0) launch_weight_image(weights_.p + j.w, j.tb, j.ldb, j.K, j.N, wimg_.p + *j.slot, st_);
  check_launch("weight_image");
  CU(cudaStreamSynchronize(st_));
}

// ---- trace spans and collective ledger ------------------------------------------------
double Context::ev_time(cudaEvent_t e) const {
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, epoch_ev_, e));
  return epoch_host_ + 1e-3 * static_cast<double>(ms);
}

// Spans of the last compute in dd_evaluate's vocabulary (decomp.cpp:285-538): per rank
// dd_build / neighbor_build / inference; step-global gather_positions (ownership kernel),
// ghost_force_route (masked: the per-rank force assembly that routes ghost partials to
// their owners) and reduce_forces (the NCCL all-reduce, or the end of the on-device
// accumulation with one process).  Ledger bytes follow the reference PayloadLayout.
void Context::record_trace(long n, const std::vector<int>& local_ranks) {
  const int R = opts_.n_ranks;
  const bool masked = opts_.scheme == NNMD_MASKED_REDUCTION;
  if (trace_on_) {
    const Timer* owner = nullptr;
    const Timer* nccl = nullptr;
    const Timer* merge = nullptr;
    for (const auto& t : timers_) {
      if (t.name == "owner") owner = &t;
      if (t.name == "route_merge") merge = &t;
      if (t.name == "nccl_allreduce") nccl = &t;
      if (t.name == "nccl_broadcast") owner = &t;  // collective 1 proper when there is one
    }
    if (owner) spans_.push_back({-1, 1, ev_time(owner->a), ev_time(owner->b), step_});
    double f0 = 1e300, f1 = -1e300;
    for (const auto& ph : phases_) {
      const double t0 = ev_time(timers_[ph.t0].a), t1 = ev_time(timers_[ph.t1].b);
      if (ph.phase < 3) {
        spans_.push_back({ph.rank, 2 + ph.phase, t0, t1, step_});
      } else {
        f0 = std::min(f0, t0);
        f1 = std::max(f1, t1);
      }
    }
    if (merge) f1 = std::max(f1, ev_time(merge->b));
    if (f1 >= f0) {
      if (masked) spans_.push_back({-1, 5, f0, f1, step_});
      if (nccl) spans_.push_back({-1, 6, ev_time(nccl->a), ev_time(nccl->b), step_});
      else spans_.push_back({-1, 6, f1, f1, step_});
    }
  }
  if (ledger_on_) {
    ledger_.push_back({step_, 0, static_cast<uint64_t>(n) * 20u, R});
    if (masked) {
      // route counts of every DD rank (all-reduced with the step flags), as dd_evaluate
      // records the total over all R ranks (decomp.cpp:463-468)
      uint64_t routed = 0;
      for (int r = 0; r < R; ++r) routed += static_cast<uint64_t>(stats_[static_cast<size_t>(r)].counts[3]);
      ledger_.push_back({step_, 1, routed * 20u, R});
    }
    ledger_.push_back({step_, 2, static_cast<uint64_t>(n) * 12u, R});
  }
}

// export_chrome_trace (trace.cpp:64-85): JSON array of complete events, microseconds from
// the earliest span, one lane per rank (tid), args.step.
void Context::export_chrome_trace(const std::string& path) const {
  static const char* names[8] = {"classical_md", "gather_positions", "dd_build", "neighbor_build",
                                 "inference", "ghost_force_route", "reduce_forces", "integrate"};
  double t0 = spans_.empty() ? 0.0 : spans_.front().t0;
  for (const auto& s : spans_) t0 = std::min(t0, s.t0);
  std::ofstream os(path, std::ios::trunc);
  require(os.good(), "export_chrome_trace: cannot open " + path);
  os << "[";
  char buf[512];
  for (size_t i = 0; i < spans_.size(); ++i) {
    const auto& s = spans_[i];
    std::snprintf(buf, sizeof buf,
                  "%s\n {\"name\": \"%s\", \"cat\": \"md\", \"ph\": \"X\", \"ts\": %.3f, \"dur\": %.3f, "
                  "\"pid\": 0, \"tid\": %d, \"args\": {\"step\": %ld}}",
                  i ? "," : "", names[s.phase & 7], (s.t0 - t0) * 1e6, (s.t1 - s.t0) * 1e6, s.rank, s.step);
    os << buf;
  }
  os << "\n]\n";
  require(os.good(), "export_chrome_trace: write failed");
}

// ---- device-resident MD loop ---------------------------------------------------------
void Context::run_md(long n, double* d_pos, double* d_vel, const double* d_mass, const int* d_types,
                     const int64_t* d_gid, const double box[3], const uint8_t periodic[3], const MdConfig& cfg,
                     double* d_rec) {
  require(cfg.dt > 0.0, "run_md: dt must be > 0");
  require(cfg.n_steps >= 0, "run_md: n_steps must be >= 0");
  out_.ensure(10 + 4 * static_cast<size_t>(n));
  md_ke_.ensure(static_cast<size_t>(n) + 1);
  md_sum_.ensure(1);
  md_err_.ensure(1);
  CU(cudaMemsetAsync(md_err_.p, 0x7f, sizeof(int), st_));
  MdArgs ma{};
  ma.n = static_cast<int>(n);
  ma.pos = d_pos;
  ma.vel = d_vel;
  ma.mass = d_mass;
  ma.F = out_.p + 10;
  ma.dt = cfg.dt;
  for (int a = 0; a < 3; ++a) {
    ma.L[a] = box[a];
    ma.per[a] = periodic[a] ? 1 : 0;
  }
  ma.ke_atom = md_ke_.p;
  ma.err = md_err_.p;
  auto check_forces = [&] {  // the flag was read back with compute_device's step flags
    if (*h_md_err_ != 0x7f7f7f7f)
      throw Error("run_md: non-finite force from provider 'nnmd_b200' at step " + std::to_string(*h_md_err_));
  };
  struct Clear {
    const MdArgs*& p;
    ~Clear() { p = nullptr; }
  } clear{md_check_};
  for (long step = 0; step < cfg.n_steps; ++step) {
    // forces of the current positions (replicated on every process after the all-reduce,
    // so each process integrates its own copy: no position collective is needed)
    ma.step = static_cast<int>(step);
    md_check_ = &ma;
    compute_device(n, d_pos, d_types, d_gid, box, periodic, out_.p);
    // run_md (engine.cpp:166-176) rejects non-finite forces BEFORE integrating: the state
    // is left at the failing step
    check_forces();
    if (trace_on_) CU(cudaEventRecord(md_ev_[0], st_));
    launch_leapfrog(ma, st_);
    launch_energy_record(md_ke_.p, ma.n, out_.p, d_rec, step, st_);
    if (cfg.target_temperature > 0.0 && step < cfg.equil_steps && cfg.rescale_every > 0 &&
        (step + 1) % cfg.rescale_every == 0)
      launch_rescale(ma.n, d_vel, d_mass, md_ke_.p, md_sum_.p, cfg.target_temperature, st_);
    check_launch("md_step");
    if (trace_on_) {
      CU(cudaEventRecord(md_ev_[1], st_));
      CU(cudaEventSynchronize(md_ev_[1]));
      spans_.push_back({-1, 7, ev_time(md_ev_[0]), ev_time(md_ev_[1]), step_});
    }
    ++step_;
  }
  CU(cudaStreamSynchronize(st_));
}

void Context::run_md_host(long n, double* pos, double* vel, const double* mass, const int* types,
                          const int64_t* gid, const double box[3], const uint8_t periodic[3], const MdConfig& cfg,
                          double* potential, double* total) {
  for (long i = 0; i < n; ++i) {
    require(types[i] >= 0 && types[i] < model_.ns, "dd_evaluate: species id outside the model's species table");
    require(mass[i] > 0.0, "AtomSet: masses must be positive");
  }
  pos_.ensure(3 * static_cast<size_t>(n) + 3);
  types_.ensure(static_cast<size_t>(n) + 1);
  gid_.ensure(static_cast<size_t>(n) + 1);
  md_vel_.ensure(3 * static_cast<size_t>(n) + 3);
  md_mass_.ensure(static_cast<size_t>(n) + 1);
  md_rec_.ensure(2 * static_cast<size_t>(std::max(cfg.n_steps, 1L)));
  std::vector<int64_t> iota;
  if (!gid) {
    iota.resize(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i) iota[static_cast<size_t>(i)] = i;
    gid = iota.data();
  }
  if (n) {
    CU(cudaMemcpyAsync(pos_.p, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st_));
    CU(cudaMemcpyAsync(md_vel_.p, vel, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st_));
    CU(cudaMemcpyAsync(md_mass_.p, mass, n * sizeof(double), cudaMemcpyHostToDevice, st_));
    CU(cudaMemcpyAsync(types_.p, types, n * sizeof(int), cudaMemcpyHostToDevice, st_));
    CU(cudaMemcpyAsync(gid_.p, gid, n * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
  }
  try {
    run_md(n, pos_.p, md_vel_.p, md_mass_.p, types_.p, gid_.p, box, periodic, cfg, md_rec_.p);
  } catch (const Error&) {
    // like the reference, leave the caller's atoms at the failing step's state
    if (n) {
      CU(cudaMemcpyAsync(pos, pos_.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, st_));
      CU(cudaMemcpyAsync(vel, md_vel_.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, st_));
      CU(cudaStreamSynchronize(st_));
    }
    throw;
  }
  std::vector<double> rec(2 * static_cast<size_t>(cfg.n_steps));
  if (cfg.n_steps) CU(cudaMemcpyAsync(rec.data(), md_rec_.p, rec.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
  if (n) {
    CU(cudaMemcpyAsync(pos, pos_.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, st_));
    CU(cudaMemcpyAsync(vel, md_vel_.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, st_));
  }
  CU(cudaStreamSynchronize(st_));
  for (long k = 0; k < cfg.n_steps; ++k) {
    if (potential) potential[k] = rec[2 * static_cast<size_t>(k)];
    if (total) total[k] = rec[2 * static_cast<size_t>(k) + 1];
  }
}

}  // namespace nb
