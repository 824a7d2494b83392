// engine.cu -- device engine of the multilevel NMF solver (sm_100a).
//
// Per step (HALS; MU and ANLS differ only in the update kernels):
//   [B = W W^T] -> A = M_l W^T -> (allreduce A|B over NCCL) -> V sweep
//   -> C = V^T M_l, D = V^T V -> W sweep
// The two M-streaming products go to the SIMT fp64-accumulating GEMMs or, for
// fp32 storage at scale, to the tcgen05 integer-digit kernels (ix_gemm.cu:
// exact int32 accumulation of 8-bit digit products).  All
// state stays on the device; nothing synchronises with the host inside a
// phase (samples and NNLS counts are collected by flush()).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "engine.hpp"
#include "hals_dmma.hpp"
#include "hals_reg.hpp"
#include "kernels.cuh"
#include "nccl_shim.hpp"
#include "nnls.cuh"
#include "ix_gemm.hpp"
#include "gram_dmma.hpp"
#include "restrict_tma.hpp"
#include "transfer_ops.hpp"

namespace mlb {

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                               __FILE__ + ":" + std::to_string(__LINE__) + " (" #x ")");       \
  } while (0)

namespace {
constexpr int kTargetBlocks = 8 * 148;  // split-K target: ~8 blocks per SM (latency-bound K loops)


template <typename T>
cudaError_t dev_malloc(T** p, size_t b) {
  return cudaMalloc(reinterpret_cast<void**>(p), b);
}
void dev_free(void* p) {
  if (p) cudaFree(p);
}
constexpr size_t kSmemMax = 227 * 1024;

size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t b) {
    if (b <= bytes) return;
    dev_free(p);
    p = nullptr;
    CK(dev_malloc(&p, b));
    bytes = b;
  }
  void release() {
    dev_free(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};
}  // namespace

struct Engine::Impl {
  Engine* e;
  cudaStream_t s = nullptr;
  int sm_count = 148;
  // work buffers (fp64)
  DevBuf AB;      // A (m0 x r) followed by B (r x r): one allreduce
  DevBuf Cb;      // C (r x n_loc)
  DevBuf Db;      // D (r x r)
  DevBuf part;    // split-K partials
  DevBuf red;     // reduction partials
  DevBuf scal;    // scalars: [0] ||M||^2 or direct e2, [1] <C,W>, [2] <D,B>, [3] max
  DevBuf W;       // T (r x n_loc)
  DevBuf samples; // SampleRec ring
  DevBuf counts;  // int ring for NNLS counts
  DevBuf flags;   // [0] degenerate count, [1] nnls error, [2] validate
  DevBuf tstart;  // run-start globaltimer
  DevBuf stage;   // host-transfer staging
  size_t samp_cap = 0, samp_used = 0, cnt_cap = 0, cnt_used = 0;
  std::vector<size_t> cnt_steps;  // m_l of every ANLS step in the count ring (m_l V rows, then n_loc W columns)
  std::vector<Sample> samp_meta;  // host metadata of enqueued samples
  // validity of cached products w.r.t. current iterates
  bool B_valid = false;   // B == W W^T (allreduced) for the current W
  bool CD_valid = false;  // C == V_l^T M_l and D == V_l^T V_l for the current V_l
  size_t CD_level = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  // profiling
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_mwt, ev_vtm, ev_comm;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_phase;  // (StepPhase, events)
  std::vector<cudaEvent_t> ev_pool;
  std::chrono::steady_clock::time_point host_t0 = std::chrono::steady_clock::now();
  TcGemm* tc = nullptr;
  // captured steady-state steps (HALS / MU, single rank): key level * 4 + kind
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    uint64_t epoch = 0;  // graph_sig() at capture
    long nlaunch = 0;
    bool warm = false;
  };
  std::map<size_t, StepGraph> graphs;
  // A captured step graph holds raw buffer pointers and the shapes of its
  // launches: it is valid while the buffers it may touch are the same
  // allocations and the problem has the same shape.  The signature hashes
  // both (this engine's only -- other sessions' allocations never invalidate
  // its graphs; a freed-and-reallocated buffer at the same address with a
  // new shape does, through the shape terms).
  uint64_t graph_sig() const {
    uint64_t h = 1469598103934665603ull;
    auto mixv = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    auto mix = [&](const void* p) { mixv((uint64_t)(uintptr_t)p); };
    for (const DevBuf* b : {&AB, &Cb, &Db, &part, &red, &scal, &W, &flags, &gws}) mix(b->p);
    mixv(e->n_loc_), mixv(e->n_total_), mixv(e->col0_), mixv(e->r_), mixv(e->lv_.size());
    for (const auto& L : e->lv_) {
      mixv(L.m), mixv(L.h), mixv(L.w);
      mix(L.M), mix(L.V), mix(L.mstat), mix(L.Rp), mix(L.Ri), mix(L.Rw), mix(L.Pp), mix(L.Pi), mix(L.Pw);
    }
    if (tc) mix(reinterpret_cast<const void*>(tc->signature()));
    return h;
  }
  // development switches, read once per engine (tests and tools/ set them before creating a session)
  const bool graphs_on = std::getenv("MLNMF_NO_GRAPHS") == nullptr;
  const bool env_exact_sweeps = std::getenv("MLNMF_EXACT_SWEEPS") != nullptr;
  const bool env_thread_sweeps = std::getenv("MLNMF_THREAD_SWEEPS") != nullptr;
  const bool env_warp_sweeps = std::getenv("MLNMF_WARP_SWEEPS") != nullptr;

  explicit Impl(Engine* eng) : e(eng) {}
  ~Impl() {
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  }

  size_t esz() const { return e->opt_.dtype == 0 ? 4 : 8; }
  bool exact() const { return e->opt_.exact != 0; }

  template <typename... KArgs, typename... Args>
  void launch(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, Args... args) {
    // opt in from 32 KB: the 48 KB default counts the kernel's static shared memory too (r = 48 with
    // fp32 data asked k_sqerr_tiled for exactly 48 KB of dynamic memory on top of its static arrays)
    if (smem > 32 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<g, b, smem, s>>>(args...);
    ++e->launches_;
    CK(cudaGetLastError());
  }

  cudaEvent_t ev() {
    if (!ev_pool.empty()) {
      cudaEvent_t x = ev_pool.back();
      ev_pool.pop_back();
      return x;
    }
    cudaEvent_t x;
    CK(cudaEventCreate(&x));
    return x;
  }

  // Run f; when profiling, bracket it with CUDA events on the engine stream
  // and book the interval under step phase ph (KernelTimes::phase_ms).
  template <typename F>
  void timed(int ph, F&& f) {
    if (!e->profiling_) {
      f();
      return;
    }
    cudaEvent_t a = ev(), b = ev();
    CK(cudaEventRecord(a, s));
    f();
    CK(cudaEventRecord(b, s));
    ev_phase.push_back({ph, {a, b}});
  }

  // ---------------- collectives ----------------
  // collectives run whenever a communicator exists: world > 1, or a 1-rank
  // communicator requested by passing an NCCL id with world = 1 (exercises the
  // NCCL path on one GPU)
  // ranks exchange through NCCL, or (no communicator, world > 1) through the
  // host hook: stream sync, device -> host, hook, host -> device
  bool multi() const { return comm || e->opt_.host_allreduce; }
  std::vector<double> hostx;
  void host_exchange(double* p, size_t count, int op) {
    hostx.resize(count);
    CK(cudaMemcpyAsync(hostx.data(), p, count * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (e->opt_.host_allreduce(e->opt_.host_allreduce_ctx, hostx.data(), count, op) != 0)
      throw std::runtime_error("host allreduce failed");
    CK(cudaMemcpyAsync(p, hostx.data(), count * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // hostx is reused by the next exchange
  }
  void allreduce_sum(double* p, size_t count) {
    if (comm) {
      nccl_check(NcclApi::get().AllReduce(p, p, count, ncclFloat64, ncclSum, comm, s), "allreduce");
    } else if (e->opt_.host_allreduce) {
      host_exchange(p, count, 0);
    }
  }
  void allreduce_max(double* p, size_t count) {
    if (comm) {
      nccl_check(NcclApi::get().AllReduce(p, p, count, ncclFloat64, ncclMax, comm, s), "allreduce max");
    } else if (e->opt_.host_allreduce) {
      host_exchange(p, count, 1);
    }
  }

  // ---------------- GEMMs ----------------
  int splits_for(size_t tiles, size_t K) const {
    if (exact()) return 1;
    size_t sp = ceil_div(kTargetBlocks, tiles);
    sp = std::min(sp, ceil_div(K, 64));  // >= 2 K-steps of 32 per split
    return (int)std::max<size_t>(sp, 1);
  }

  // out (rows x ny, fp64) = X (rows x K) * Y (ny x K)^T
  // output tile extent along the narrow (rank) dimension
  static int narrow_tile(size_t extent) { return extent <= 32 ? 32 : extent <= 48 ? 48 : 64; }

  template <typename TX, typename TY>
  void gemm_abt(const TX* X, const TY* Y, size_t rows, size_t ny, size_t K, double* out) {
    const int tc = narrow_tile(ny);
    const size_t tiles = ceil_div(rows, GT) * ceil_div(ny, (size_t)tc);
    const int sp = splits_for(tiles, K);
    const size_t kchunk = ceil_div(ceil_div(K, sp), GK) * GK;
    const int spr = (int)ceil_div(K, kchunk);
    dim3 g((unsigned)ceil_div(rows, GT), (unsigned)ceil_div(ny, (size_t)tc), (unsigned)spr);
    double* dst = out;
    if (spr > 1) {
      part.ensure((size_t)spr * rows * ny * 8);
      dst = part.as<double>();
    }
    auto go = [&](auto kern) {
      launch(kern, g, dim3(256), 0, X, (const double*)nullptr, rows, Y, rows, ny, K, kchunk, dst);
    };
    if (exact())
      tc == 32 ? go(k_gemm_abt<TX, TY, true, 32>) : tc == 48 ? go(k_gemm_abt<TX, TY, true, 48>)
               : go(k_gemm_abt<TX, TY, true, 64>);
    else
      tc == 32 ? go(k_gemm_abt<TX, TY, false, 32>) : tc == 48 ? go(k_gemm_abt<TX, TY, false, 48>)
               : go(k_gemm_abt<TX, TY, false, 64>);
    if (spr > 1) {
      const size_t cnt = rows * ny;
      reduce_splits(part.as<double>(), cnt, spr, out);
    }
  }

  // out (r x ncols, fp64) = V (K x r)^T * X (K x ncols)
  template <typename TV, typename TX>
  void gemm_atb(const TV* V, const TX* X, size_t K, size_t r, size_t ncols, double* out) {
    const int tr = narrow_tile(r);
    const size_t tiles = ceil_div(ncols, GT) * ceil_div(r, (size_t)tr);
    const int sp = splits_for(tiles, K);
    const size_t kchunk = ceil_div(ceil_div(K, sp), GK) * GK;
    const int spr = (int)ceil_div(K, kchunk);
    dim3 g((unsigned)ceil_div(ncols, GT), (unsigned)ceil_div(r, (size_t)tr), (unsigned)spr);
    double* dst = out;
    if (spr > 1) {
      part.ensure((size_t)spr * r * ncols * 8);
      dst = part.as<double>();
    }
    auto go = [&](auto kern) {
      launch(kern, g, dim3(256), 0, V, X, (const double*)nullptr, ncols, K, r, ncols, kchunk, dst);
    };
    if (exact())
      tr == 32 ? go(k_gemm_atb<TV, TX, true, 32>) : tr == 48 ? go(k_gemm_atb<TV, TX, true, 48>)
               : go(k_gemm_atb<TV, TX, true, 64>);
    else
      tr == 32 ? go(k_gemm_atb<TV, TX, false, 32>) : tr == 48 ? go(k_gemm_atb<TV, TX, false, 48>)
               : go(k_gemm_atb<TV, TX, false, 64>);
    if (spr > 1) {
      const size_t cnt = r * ncols;
      reduce_splits(part.as<double>(), cnt, spr, out);
    }
  }

  // Stacked products of a half-iteration on the SIMT path (non-exact runs):
  // [A; B] = [M_l; W] W^T in ONE launch + one split-K epilogue instead of two
  // of each -- the small configurations are launch-bound (config 0: ten
  // launches of a few microseconds per sweep).  Returns false (nothing
  // launched) where the stacked product would not be split: the epilogue is
  // what scatters the two results, and unsplit shapes gain nothing.
  static constexpr size_t kStackedMaxK = 32768;
  template <typename T>
  bool stacked_ab(size_t l) {
    const auto& L = e->lv_[l];
    const size_t r = e->r_, rows = L.m + r, K = e->n_loc_;
    const int tc = narrow_tile(r);
    // K split as for A alone (the Gram's tile rides along: config 3 measured
    // slower with the split chosen for the stacked tile count, r02)
    const size_t tiles = ceil_div(L.m, GT) * ceil_div(r, (size_t)tc);
    const int sp = splits_for(tiles, K);
    const size_t kchunk = ceil_div(ceil_div(K, sp), GK) * GK;
    const int spr = (int)ceil_div(K, kchunk);
    if (spr < 2 || K > kStackedMaxK) return false;
    part.ensure((size_t)spr * rows * r * 8);
    const dim3 g((unsigned)ceil_div(rows, GT), (unsigned)ceil_div(r, (size_t)tc), (unsigned)spr);
    auto go = [&](auto kern) {
      launch(kern, g, dim3(256), 0, static_cast<const T*>(L.M), (const double*)W.as<double>(), L.m,
             (const double*)W.as<double>(), rows, r, K, kchunk, part.as<double>());
    };
    tc == 32 ? go(k_gemm_abt<T, double, false, 32>) : tc == 48 ? go(k_gemm_abt<T, double, false, 48>)
             : go(k_gemm_abt<T, double, false, 64>);
    reduce_splits2(rows * r, spr, r, L.m, 1, A(), B());
    return true;
  }
  // [C | D] = V_l^T [M_l | V_l]
  template <typename T>
  bool stacked_cd(size_t l) {
    const auto& L = e->lv_[l];
    const size_t r = e->r_, ncols = e->n_loc_ + r, K = L.m;
    const int tr = narrow_tile(r);
    const size_t tiles = ceil_div(e->n_loc_, GT) * ceil_div(r, (size_t)tr);  // K split as for C alone
    const int sp = splits_for(tiles, K);
    const size_t kchunk = ceil_div(ceil_div(K, sp), GK) * GK;
    const int spr = (int)ceil_div(K, kchunk);
    // long contractions keep the two launches: config 3 (K = 77760, 348 K
    // ranges) measured 60 us per step slower stacked (r02, same box)
    if (spr < 2 || K > kStackedMaxK) return false;
    part.ensure((size_t)spr * r * ncols * 8);
    const dim3 g((unsigned)ceil_div(ncols, GT), (unsigned)ceil_div(r, (size_t)tr), (unsigned)spr);
    auto go = [&](auto kern) {
      launch(kern, g, dim3(256), 0, static_cast<const double*>(L.V), static_cast<const T*>(L.M),
             static_cast<const double*>(L.V), e->n_loc_, K, r, ncols, kchunk, part.as<double>());
    };
    tr == 32 ? go(k_gemm_atb<double, T, false, 32>) : tr == 48 ? go(k_gemm_atb<double, T, false, 48>)
             : go(k_gemm_atb<double, T, false, 64>);
    reduce_splits2(r * ncols, spr, ncols, e->n_loc_, 0, Cb.as<double>(), Db.as<double>());
    return true;
  }
  void reduce_splits2(size_t cnt, int spr, size_t rl, size_t cut, int by_row, double* out0, double* out1) {
    if (spr >= 16 && cnt <= ((size_t)1 << 16))
      launch(k_reduce_splits2_wide, dim3((unsigned)ceil_div(cnt, 32)), dim3(256), 0, (const double*)part.as<double>(),
             cnt, spr, rl, cut, by_row, out0, out1);
    else
      launch(k_reduce_splits2, dim3((unsigned)std::min<size_t>(ceil_div(cnt, 256), 4096)), dim3(256), 0,
             (const double*)part.as<double>(), cnt, spr, rl, cut, by_row, out0, out1);
  }

  // out[e] = sum over spr split partials (deterministic; wide form for many splits)
  void reduce_splits(const double* prt, size_t cnt, int spr, double* out) {
    if (spr >= 16 && cnt <= ((size_t)1 << 16))
      launch(k_reduce_splits_wide, dim3((unsigned)ceil_div(cnt, 32)), dim3(256), 0, prt, cnt, spr, out);
    else
      launch(k_reduce_splits, dim3((unsigned)std::min<size_t>(ceil_div(cnt, 256), 4096)), dim3(256), 0, prt, cnt, spr,
             out);
  }

  double* A() { return AB.as<double>(); }
  double* B() { return AB.as<double>() + e->lv_[0].m * e->r_; }

  // tensor path for a level of m rows (fp32 storage, supported shape, policy;
  // a forced tensor path still serves unsupported levels -- e.g. coarse
  // grids below one 128-row tile -- with the SIMT kernels).  Decided once
  // per (level, rank r) for ALL ranks (decide_tc): every rank must issue
  // the same collectives, and the shape rules see the local column count.
  std::map<std::pair<size_t, size_t>, bool> tc_ok;
  bool use_tc(size_t l) const {
    if (!tc || e->lv_[l].dt != 0) return false;
    auto it = tc_ok.find({e->lv_[l].m, e->r_});
    if (it == tc_ok.end()) throw std::logic_error("tensor-path decision missing for a level (decide_tc)");
    return it->second;
  }
  // the level may take the tensor path (norm2 may precede factor setup, when
  // the rank is not known yet: the maxima pass costs the same as the plain
  // sum of squares, so it is taken whenever the shape allows the tensor path)
  bool use_tc_known(size_t l) const {
    if (!tc || e->lv_[l].dt != 0) return false;
    if (e->r_ == 0) return tc->wants(e->lv_[l].m, e->n_loc_, 1);
    auto it = tc_ok.find({e->lv_[l].m, e->r_});
    return it != tc_ok.end() && it->second;
  }
  // at host-synchronous points (factor and level setup): local policy,
  // combined over ranks (any rank unable => nobody takes the tensor path)
  void decide_tc() {
    if (!tc || e->r_ == 0) return;
    for (const auto& L : e->lv_) {
      if (L.dt != 0) continue;  // fp64 levels never take the tensor path
      const auto key = std::make_pair(L.m, e->r_);
      if (tc_ok.count(key)) continue;
      double veto = tc->wants(L.m, e->n_loc_, e->r_) ? 0.0 : 1.0;
      if (multi()) {
        double* d = scal.as<double>() + 9;
        CK(cudaMemcpyAsync(d, &veto, 8, cudaMemcpyHostToDevice, s));
        allreduce_max(d, 1);
        CK(cudaMemcpyAsync(&veto, d, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
      }
      tc_ok[key] = veto == 0.0;
    }
  }

  // Row / column maxima of M_l (fixed-point scales of the tensor path),
  // computed once per level on first use.
  // With sq_out (a device double), the same pass also sums ||M_l||_F^2 into
  // it (Engine::norm2 asks first on a tensor-path level: one pass over M_l
  // instead of two).
  const float* level_stats(size_t l, double* sq_out = nullptr) {
    auto& L = e->lv_[l];
    if (!L.mstat) {
      CK(dev_malloc(&L.mstat, (L.m + e->n_loc_) * 4));
      double* part = nullptr;
      size_t nb = 0;
      if (sq_out) {
        nb = tc->level_stats_blocks(L.m, e->n_loc_);
        red.ensure(nb * 8);
        part = red.as<double>();
      }
      tc->level_stats(static_cast<const float*>(L.M), L.m, e->n_loc_, L.mstat, L.mstat + L.m, part, s,
                      &e->launches_);
      if (sq_out) launch(k_sum_final, dim3(1), dim3(1024), 0, (const double*)part, nb, sq_out, 0);
    }
    return L.mstat;
  }

  // f() bracketed by CUDA events on the engine stream when profiling (the
  // per-product times of kernel_times); the pair is kept only if f launched
  template <typename F>
  bool bracketed(std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& into, F&& f) {
    if (!e->profiling_) return f();
    std::pair<cudaEvent_t, cudaEvent_t> evp{ev(), ev()};
    CK(cudaEventRecord(evp.first, s));
    const bool done = f();
    CK(cudaEventRecord(evp.second, s));
    if (done) into.push_back(evp);
    else ev_pool.push_back(evp.first), ev_pool.push_back(evp.second);
    return done;
  }

  // A = M_l W^T (the first M pass), timed when profiling.
  template <typename T>
  void product_mwt(size_t l) {
    const auto& L = e->lv_[l];
    std::pair<cudaEvent_t, cudaEvent_t> evp{};
    if (e->profiling_) {
      evp = {ev(), ev()};
      CK(cudaEventRecord(evp.first, s));
    }
    if (use_tc(l))
      tc->mwt(static_cast<const T*>(L.M), level_stats(l), W.as<double>(), L.m, e->n_loc_, e->r_, A(), s,
              &e->launches_);
    else
      gemm_abt(static_cast<const T*>(L.M), W.as<double>(), L.m, e->r_, e->n_loc_, A());
    if (e->profiling_) {
      CK(cudaEventRecord(evp.second, s));
      ev_mwt.push_back(evp);
    }
  }
  // C = V_l^T M_l (the second M pass)
  template <typename T>
  void product_vtm(size_t l) {
    const auto& L = e->lv_[l];
    std::pair<cudaEvent_t, cudaEvent_t> evp{};
    if (e->profiling_) {
      evp = {ev(), ev()};
      CK(cudaEventRecord(evp.first, s));
    }
    if (use_tc(l))
      tc->vtm(static_cast<const double*>(L.V), static_cast<const T*>(L.M), level_stats(l) + L.m, L.m, e->n_loc_,
              e->r_, Cb.as<double>(), s, &e->launches_);
    else
      gemm_atb(static_cast<const double*>(L.V), static_cast<const T*>(L.M), L.m, e->r_, e->n_loc_, Cb.as<double>());
    if (e->profiling_) {
      CK(cudaEventRecord(evp.second, s));
      ev_vtm.push_back(evp);
    }
  }
  template <typename T>
  void gram_W() {  // B = W W^T over all ranks
    if (!exact() && gram_dmma_supported(e->r_, e->n_loc_)) {
      // wide factor: fp64 tensor-core tiles, upper triangle only (gram_dmma.cu)
      const int nb = gram_dmma_blocks(e->n_loc_, sm_count);
      part.ensure((size_t)nb * e->r_ * e->r_ * 8);
      gram_dmma(W.as<double>(), e->r_, e->n_loc_, sm_count, part.as<double>(), s);
      ++e->launches_;
      reduce_splits(part.as<double>(), e->r_ * e->r_, nb, B());
      return;
    }
    gemm_abt(W.as<double>(), W.as<double>(), e->r_, e->r_, e->n_loc_, B());
  }
  template <typename T>
  void gram_V(size_t l) {  // D = V_l^T V_l (replicated)
    const auto& L = e->lv_[l];
    if (!exact() && gram_dmma_supported(e->r_, L.m)) {  // tall factor: fp64 tensor-core tiles (gram_dmma.cu)
      const int nb = gram_dmma_blocks(L.m, sm_count);
      part.ensure((size_t)nb * e->r_ * e->r_ * 8);
      gram_dmma(static_cast<const double*>(L.V), e->r_, L.m, sm_count, part.as<double>(), s, true);
      ++e->launches_;
      reduce_splits(part.as<double>(), e->r_ * e->r_, nb, Db.as<double>());
      return;
    }
    gemm_atb(static_cast<const double*>(L.V), static_cast<const double*>(L.V), L.m, e->r_, e->r_, Db.as<double>());
  }

  // ---------------- row/column sweeps ----------------
  // Non-exact HALS (and MU) sweeps over few rows / columns use a warp per row (warp-
  // shuffle dot products): one thread per column leaves the GPU idle there
  // (config 3's W half: n = 165).  With many rows the thread-per-row kernels
  // win (measured: config 3's V half 0.58 -> 0.82 ms/step and config 4's step
  // +2 ms with warps).  Exact mode keeps the reference's sequential order.
  // (re-measured with the persistent two-row warp kernels: config 3 0.585 ->
  // 0.713 ms/step, config 4 +1.3 ms/step; MLNMF_WARP_SWEEPS=1 forces them)
  static constexpr size_t kWarpSweepMax = 16384;
  // register sweeps at the config-4 rank: interleaved fused dot chains in
  // non-exact runs (MLNMF_EXACT_SWEEPS=1 keeps the reference order)
  bool fast_sweeps() const {
    return e->opt_.dtype == 0 && !exact() && !env_exact_sweeps;
  }
  bool warp_sweeps(size_t r, size_t count) const {
    if (exact() || r > 64 || env_thread_sweeps) return false;
    return count < kWarpSweepMax || env_warp_sweeps;
  }
  // threads per block of the thread-per-row sweeps with the Gram and the
  // rows in shared memory; 0 when r is too large for that (r > ~160): the
  // sweeps then read the Gram from global memory (L2) and keep the rows in a
  // global workspace (gsweep_ws)
  int sweep_block(int r) const {
    for (int bd : {128, 64, 32})
      if ((size_t)r * r * 8 + (size_t)r * bd * 8 <= kSmemMax) return bd;
    return 0;
  }
  DevBuf gws;  // large-rank workspaces (sweeps, NNLS)
  double* gsweep_ws(size_t rows, int bd, size_t r) {
    gws.ensure(ceil_div(rows, (size_t)bd) * bd * r * 8);
    return gws.as<double>();
  }

  template <typename T>
  void step_t(size_t l, Kind kind) {
    const auto& L = e->lv_[l];
    const size_t r = e->r_;
    int* deg = flags.as<int>();
    // ---- V half: A = M W^T, B = W W^T (solvers.cpp:82-83,105-106,251-252)
    const bool needB = !B_valid;
    // small SIMT shapes: A and B from one stacked launch (booked under phase A)
    bool ab_done = false;
    if (needB && !use_tc(l) && !exact()) timed(kPhA, [&] { ab_done = bracketed(ev_mwt, [&] { return stacked_ab<T>(l); }); });
    if (!ab_done) {
      if (needB) timed(kPhB, [&] { gram_W<T>(); });
      timed(kPhA, [&] { product_mwt<T>(l); });
    }
    if (multi()) {
      std::pair<cudaEvent_t, cudaEvent_t> evp{};
      if (e->profiling_) {
        evp = {ev(), ev()};
        CK(cudaEventRecord(evp.first, s));
      }
      if (needB && L.m == e->lv_[0].m) {
        allreduce_sum(A(), L.m * r + r * r);  // A|B contiguous: one collective
      } else {
        allreduce_sum(A(), L.m * r);
        if (needB) allreduce_sum(B(), r * r);
      }
      if (e->profiling_) {
        CK(cudaEventRecord(evp.second, s));
        ev_comm.push_back(evp);
      }
    }
    double* V = static_cast<double*>(L.V);
    const int bd0 = sweep_block((int)r);
    const int bd = bd0 ? bd0 : 128;
    const size_t smem = bd0 ? (r * r + r * bd) * 8 : 0;
    double* gv_ws = bd0 ? nullptr : gsweep_ws(std::max(L.m, e->n_loc_), bd, r);
    timed(kPhV, [&] {
      const dim3 gv((unsigned)ceil_div(L.m, bd));
      if (kind == kHals && fast_sweeps() && hals_v_dmma_supported(r, L.m)) {
        hals_v_dmma(r, A(), B(), V, L.m, deg, s);  // blocks of 8 updates on the fp64 tensor cores (hals_dmma.cu)
        ++e->launches_;
      } else if (kind == kHals && warp_sweeps(r, L.m)) {  // warp per row (non-exact, few rows)
        launch(k_hals_v_warp<double>, dim3((unsigned)std::min<size_t>(ceil_div(L.m, 8), (size_t)sm_count * 4)), dim3(256),
               (r * r + r) * 8, (const double*)A(), (const double*)B(), V, L.m, (int)r, deg);
      } else if (kind == kHals && hals_reg_supported(r)) {  // register-resident sweep, reference order
        hals_v_reg(r, fast_sweeps(), A(), B(), V, L.m, deg, s);
        ++e->launches_;
      } else if (kind == kHals) {
        launch(k_hals_v<double>, gv, dim3(bd), smem, (const double*)A(), (const double*)B(), V, L.m, (int)r, deg, gv_ws);
      } else if (kind == kMu && fast_sweeps() && mu_dmma_supported(r, L.m)) {
        mu_v_dmma(r, A(), B(), V, L.m, s);  // (V B) on the fp64 tensor cores (hals_dmma.cu)
        ++e->launches_;
      } else if (kind == kMu && warp_sweeps(r, L.m)) {
        launch(k_mu_warp<double, false>, dim3((unsigned)std::min<size_t>(ceil_div(L.m, 8), (size_t)sm_count * 4)),
               dim3(256), r * r * 8, (const double*)A(), (const double*)B(), V, L.m, (int)r);
      } else if (kind == kMu && mu_reg_supported(r)) {
        mu_v_reg(r, A(), B(), V, L.m, s);
        ++e->launches_;
      } else if (kind == kMu) {
        launch(k_mu_v<double>, gv, dim3(bd), smem, (const double*)A(), (const double*)B(), V, L.m, (int)r, gv_ws);
      } else {
        cnt_steps.push_back(L.m);
        nnls((const double*)B(), L.m, (const double*)A(), r, 1, V, r, 1);
      }
    });
    // ---- W half: C = V^T M, D = V^T V (solvers.cpp:91-92,124-125,272-273)
    bool cd_done = false;
    if (!use_tc(l) && !exact()) timed(kPhC, [&] { cd_done = bracketed(ev_vtm, [&] { return stacked_cd<T>(l); }); });
    if (!cd_done) {
      timed(kPhD, [&] { gram_V<T>(l); });
      timed(kPhC, [&] { product_vtm<T>(l); });
    }
    timed(kPhW, [&] {
      double* Wp = W.as<double>();
      const dim3 gw((unsigned)ceil_div(e->n_loc_, bd));
      if (kind == kHals && fast_sweeps() && hals_w_dmma_supported(r, e->n_loc_)) {
        // wide factor, non-exact: updates in blocks of 8 on the fp64 tensor cores (hals_dmma.cu)
        hals_w_dmma(r, Cb.as<double>(), Db.as<double>(), Wp, e->n_loc_, deg, s);
        ++e->launches_;
      } else if (kind == kHals && warp_sweeps(r, e->n_loc_)) {
        launch(k_hals_w_warp<double>, dim3((unsigned)std::min<size_t>(ceil_div(e->n_loc_, 8), (size_t)sm_count * 4)),
               dim3(256), (r * r + r) * 8, (const double*)Cb.as<double>(), (const double*)Db.as<double>(), Wp,
               e->n_loc_, (int)r, deg);
      } else if (kind == kHals && hals_reg_supported(r)) {
        hals_w_reg(r, fast_sweeps(), Cb.as<double>(), Db.as<double>(), Wp, e->n_loc_, deg, s);
        ++e->launches_;
      } else if (kind == kHals) {
        launch(k_hals_w<double>, gw, dim3(bd), smem, (const double*)Cb.as<double>(), (const double*)Db.as<double>(), Wp,
               e->n_loc_, (int)r, deg, gv_ws);
      } else if (kind == kMu && fast_sweeps() && mu_dmma_supported(r, e->n_loc_)) {
        mu_w_dmma(r, Cb.as<double>(), Db.as<double>(), Wp, e->n_loc_, s);
        ++e->launches_;
      } else if (kind == kMu && warp_sweeps(r, e->n_loc_)) {
        launch(k_mu_warp<double, true>, dim3((unsigned)std::min<size_t>(ceil_div(e->n_loc_, 8), (size_t)sm_count * 4)),
               dim3(256), r * r * 8, (const double*)Cb.as<double>(), (const double*)Db.as<double>(), Wp, e->n_loc_,
               (int)r);
      } else if (kind == kMu && mu_reg_supported(r)) {
        mu_w_reg(r, Cb.as<double>(), Db.as<double>(), Wp, e->n_loc_, s);
        ++e->launches_;
      } else if (kind == kMu) {
        launch(k_mu_w<double>, gw, dim3(bd), smem, (const double*)Cb.as<double>(), (const double*)Db.as<double>(), Wp,
               e->n_loc_, (int)r, gv_ws);
      } else {
        nnls((const double*)Db.as<double>(), e->n_loc_, (const double*)Cb.as<double>(), 1, e->n_loc_, Wp, 1,
                e->n_loc_);
      }
    });
    B_valid = false;
    CD_valid = true;
    CD_level = l;
  }

  // batched NNLS over nprob problems; counts appended to the count ring
  void nnls(const double* G, size_t nprob, const double* H, size_t hi, size_t he, double* X, size_t xi, size_t xe) {
    const int r = (int)e->r_;
    const size_t gbytes = (size_t)r * r * 8, wb = nnls_warp_bytes(r);
    if (gbytes + wb > kSmemMax) {
      // large ranks: Gram from global memory, per-warp workspaces in gws
      const int nw = 4;
      const size_t blocks = std::min<size_t>(ceil_div(nprob, (size_t)nw), (size_t)sm_count * 4);
      gws.ensure(blocks * nw * wb);
      int* cnt = reserve_counts(nprob);
      if (exact())
        launch(k_nnls_batch<double, true>, dim3((unsigned)blocks), dim3(32 * nw), 0, G, r, nprob, H, hi, he, X, xi,
               xe, cnt, flags.as<int>() + 1, gws.as<unsigned char>());
      else
        launch(k_nnls_batch<double, false>, dim3((unsigned)blocks), dim3(32 * nw), 0, G, r, nprob, H, hi, he, X, xi,
               xe, cnt, flags.as<int>() + 1, gws.as<unsigned char>());
      return;
    }
    // warps per block: as many as the SM's shared memory holds (the Gram is
    // staged once per block, so one wide block per SM beats several narrow
    // ones; 8 warps per block left large-rank problems at 8 warps per SM and
    // latency-bound), but no more than spreads the problems over every SM
    // ... and no more than the register file holds: the runtime's own bound (registers are allocated
    // per group of warps, so 65536 / (registers x 32) overestimates it)
    static const size_t nw_regs = [] {
      cudaFuncAttributes fa{}, fb{};
      CK(cudaFuncGetAttributes(&fa, k_nnls_batch<double, true>));
      CK(cudaFuncGetAttributes(&fb, k_nnls_batch<double, false>));
      return (size_t)std::max(1, std::min(fa.maxThreadsPerBlock, fb.maxThreadsPerBlock) / 32);
    }();
    const size_t nw_max = std::max<size_t>(1, std::min<size_t>(std::min<size_t>(32, nw_regs), (kSmemMax - gbytes) / wb));
    const int nw = (int)std::min(nw_max, std::max<size_t>(1, ceil_div(nprob, (size_t)sm_count)));
    const size_t smem = gbytes + nw * wb;
    const size_t per_sm = std::max<size_t>(1, std::min<size_t>(kSmemMax / smem, 64 / nw));
    const size_t blocks = std::min<size_t>(ceil_div(nprob, nw), (size_t)sm_count * per_sm);
    int* cnt = reserve_counts(nprob);
    if (exact())
      launch(k_nnls_batch<double, true>, dim3((unsigned)blocks), dim3(32 * nw), smem, G, r, nprob, H, hi, he, X, xi, xe,
             cnt, flags.as<int>() + 1, (unsigned char*)nullptr);
    else
      launch(k_nnls_batch<double, false>, dim3((unsigned)blocks), dim3(32 * nw), smem, G, r, nprob, H, hi, he, X, xi,
             xe, cnt, flags.as<int>() + 1, (unsigned char*)nullptr);
  }

  // After an ANLS step: the reference throws at the failing step
  // (solvers.cpp:269,294); the flag is read here (one sync per ANLS step)
  // and max-combined over ranks, so every rank throws at the same step.
  void check_nnls() {
    int f = 0;
    CK(cudaMemcpyAsync(&f, flags.as<int>() + 1, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (multi()) {
      double fd = (double)f;
      double* d = scal.as<double>() + 10;
      CK(cudaMemcpyAsync(d, &fd, 8, cudaMemcpyHostToDevice, s));
      allreduce_max(d, 1);
      CK(cudaMemcpyAsync(&fd, d, 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      f = (int)fd;
    }
    if (f) {
      CK(cudaMemsetAsync(flags.as<int>() + 1, 0, 4, s));
      throw NnlsCapExceeded(f & 1 ? "anls_step: NNLS exchange cap exceeded"
                                  : "anls_step: NNLS failed (singular passive subsystem)");
    }
  }

  int* reserve_counts(size_t k) {
    if (cnt_used + k > cnt_cap) {
      // grow: keep the already-enqueued counts (device-to-device copy in order)
      size_t ncap = std::max(cnt_cap * 2, cnt_used + k + (1u << 20));
      DevBuf nb;
      nb.ensure(ncap * 4);
      if (cnt_used) CK(cudaMemcpyAsync(nb.p, counts.p, cnt_used * 4, cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
      counts.release();
      counts = nb;
      cnt_cap = ncap;
    }
    int* p = counts.as<int>() + cnt_used;
    cnt_used += k;
    return p;
  }

  // ---------------- error samples ----------------
  template <typename T>
  void dot(const void* a, int a_is_t, const void* b, int b_kind, size_t count, double* out) {
    // b_kind: 0 none (a^2), 1 double, 2 T
    const size_t blocks = std::min<size_t>(ceil_div(count, 256), 4 * (size_t)sm_count);
    red.ensure(std::max<size_t>(blocks, 1) * 8);
    double* rp = red.as<double>();
    if (a_is_t && b_kind == 0 && sizeof(T) == 4 && count % 4 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0) {
      launch(k_sq_partial_v4, dim3((unsigned)blocks), dim3(256), 0, (const float4*)a, count / 4, rp);
    } else if (a_is_t) {
      if (b_kind == 0) launch(k_dot_partial<T, T>, dim3((unsigned)blocks), dim3(256), 0, (const T*)a, (const T*)nullptr, count, rp);
      else launch(k_dot_partial<T, T>, dim3((unsigned)blocks), dim3(256), 0, (const T*)a, (const T*)b, count, rp);
    } else {
      if (b_kind == 1) launch(k_dot_partial<double, double>, dim3((unsigned)blocks), dim3(256), 0, (const double*)a, (const double*)b, count, rp);
      else launch(k_dot_partial<double, T>, dim3((unsigned)blocks), dim3(256), 0, (const double*)a, (const T*)b, count, rp);
    }
    launch(k_sum_final, dim3(1), dim3(256), 0, (const double*)rp, blocks, out, 0);
  }

  template <typename T>
  void direct_e2(size_t l, double* out) {
    const auto& L = e->lv_[l];
    const int r = (int)e->r_;
    const size_t n = e->n_loc_;
    const size_t cb = ceil_div(n, 128);
    const size_t tiled_smem = 2 * (size_t)r * 128 * sizeof(T);
    if (tc_sample(l)) {
      tc_e2<T>(l, out);
      return;
    }
    if (!exact() && tiled_smem <= 200 * 1024) {
      tiled_residual<T>(l, out, nullptr);
      return;
    }
    size_t sp = 1;
    if (!exact()) sp = std::max<size_t>(1, std::min(ceil_div(kTargetBlocks, cb), ceil_div(L.m, 256)));
    const size_t rchunk = ceil_div(ceil_div(L.m, sp), 32) * 32;
    const size_t spr = ceil_div(L.m, rchunk);
    part.ensure(spr * n * 8);
    const size_t smem = ((size_t)r * 128 + 32 * (size_t)r) * 8;
    const bool gm = smem > kSmemMax;  // large ranks: V and W straight from global memory
    auto go = [&](auto kern) {
      launch(kern, dim3((unsigned)cb, (unsigned)spr), dim3(128), gm ? 0 : smem, (const T*)L.M, (const double*)L.V,
             (const double*)W.as<double>(), L.m, n, r, rchunk, part.as<double>());
    };
    if (exact()) gm ? go(k_col_sqerr<T, true, true>) : go(k_col_sqerr<T, true, false>);
    else gm ? go(k_col_sqerr<T, false, true>) : go(k_col_sqerr<T, false, false>);
    if (exact()) {
      launch(k_sum_final, dim3(1), dim3(32), 0, (const double*)part.as<double>(), n, out, 1);
    } else {
      red.ensure(n * 8);
      if (spr > 1)
        launch(k_reduce_splits, dim3((unsigned)std::min<size_t>(ceil_div(n, 256), 4096)), dim3(256), 0,
               (const double*)part.as<double>(), n, (int)spr, red.as<double>());
      const double* colv = spr > 1 ? red.as<double>() : part.as<double>();
      launch(k_sum_final, dim3(1), dim3(1024), 0, colv, n, out, 0);
    }
    allreduce_sum(out, 1);
  }

  // register-tiled residual ||M_l - V_l W||^2 (persistent, one fp64 partial
  // per block) into out[0], all ranks; gated blocks return at once unless
  // *gate != 0
  template <typename T>
  void tiled_residual(size_t l, double* out, const double* gate) {
    const auto& L = e->lv_[l];
    const int r = (int)e->r_;
    const size_t n = e->n_loc_;
    const size_t tiles = ceil_div(n, 128) * ceil_div(L.m, 128);
    const size_t grid = std::min<size_t>(tiles, 2 * (size_t)sm_count);
    part.ensure(grid * 8);
    launch(k_sqerr_tiled<T>, dim3((unsigned)grid), dim3(256), 2 * (size_t)r * 128 * sizeof(T), (const T*)L.M,
           (const double*)L.V, (const double*)W.as<double>(), L.m, n, r, part.as<double>(), gate);
    launch(k_sum_final, dim3(1), dim3(1024), 0, (const double*)part.as<double>(), grid, out, 0);
    allreduce_sum(out, 1);
  }

  // Error samples of tensor-path levels (auto error mode): the Gram identity
  // ||M||^2 - 2 <V^T M, W> + <V^T V, W W^T> from the tensor-path C (no
  // residual pass) -- unless it cancels more than 1 / kGramTau-fold, where
  // the products' input rounding would show (measured: 5e-5 of e at the
  // config-4 slice's coarsest level, rel. error ~2e-3); then the direct
  // residual (k_sqerr_tiled, gated on the device: no host sync) is used.
  static constexpr double kGramTau = 1e-4;  // e < 1 % of ||M_l||
  bool tc_sample(size_t l) const {
    return !exact() && use_tc(l) && e->opt_.error_mode == 0;
  }
  template <typename T>
  void tc_e2(size_t l, double* sc) {
    e->norm2(l);  // host-cached ||M_l||^2 (syncs once per level)
    gram_terms<T>(l, sc);
    launch(k_gram_check, dim3(1), dim3(1), 0, sc, kGramTau);
    tiled_residual<T>(l, sc + 8, sc + 7);
    launch(k_gram_select, dim3(1), dim3(1), 0, sc);
  }

  SampleRec* reserve_sample() {
    if (samp_used == samp_cap) {
      size_t ncap = std::max<size_t>(samp_cap * 2, 4096);
      DevBuf nb;
      nb.ensure(ncap * sizeof(SampleRec));
      if (samp_used) CK(cudaMemcpyAsync(nb.p, samples.p, samp_used * sizeof(SampleRec), cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
      samples.release();
      samples = nb;
      samp_cap = ncap;
    }
    return samples.as<SampleRec>() + samp_used++;
  }

  // out[0] = ||M_l||^2, out[1] = <C, W> (C = V_l^T M_l), out[2] = <D, B>
  // (D = V_l^T V_l, B = W W^T), all ranks; products recomputed only when the
  // cached ones are stale
  template <typename T>
  void gram_prepare(size_t l) {
    const size_t r = e->r_;
    if (!(CD_valid && CD_level == l)) {
      gram_V<T>(l);
      product_vtm<T>(l);
      CD_valid = true;
      CD_level = l;
    }
    if (!B_valid) {
      gram_W<T>();
      allreduce_sum(B(), r * r);
      B_valid = true;
    }
  }
  template <typename T>
  void gram_terms(size_t l, double* out) {
    const size_t r = e->r_;
    gram_prepare<T>(l);
    launch(k_set1, dim3(1), dim3(1), 0, out, e->lv_[l].norm2);  // host-cached ||M_l||^2
    dot<T>(Cb.as<double>(), 0, W.as<double>(), 1, r * e->n_loc_, out + 1);
    allreduce_sum(out + 1, 1);
    dot<T>(Db.as<double>(), 0, B(), 1, r * r, out + 2);
  }

  template <typename T>
  void sample_t(size_t l, double work_units) {
    double* sc = scal.as<double>();
    bool gram = e->gram_error();
    if (tc_sample(l)) {
      tc_e2<T>(l, sc);  // sc[0] = e^2
      gram = false;
    } else if (gram && e->opt_.world == 1 && e->r_ * e->n_loc_ <= ((size_t)1 << 20)) {
      // small, one rank: the whole identity and the record in one launch
      gram_prepare<T>(l);
      SampleRec* rec = reserve_sample();
      launch(k_gram_sample, dim3(1), dim3(1024), 0, (const double*)Cb.as<double>(), (const double*)W.as<double>(),
             e->r_ * e->n_loc_, (const double*)Db.as<double>(), (const double*)B(), e->r_ * e->r_, e->lv_[l].norm2, sc,
             rec);
      samp_meta.push_back({0.0, work_units, (int)l + 1, 0.0});
      return;
    } else if (gram) {
      gram_terms<T>(l, sc);
    } else {
      direct_e2<T>(l, sc);
    }
    SampleRec* rec = reserve_sample();
    launch(k_write_sample, dim3(1), dim3(1), 0, (const double*)sc, gram ? 1 : 0, rec);
    samp_meta.push_back({0.0, work_units, (int)l + 1, 0.0});
  }
};

// ============================================================================

Engine::Engine(const Options& o) : opt_(o), impl_(new Impl(this)) {
  if (o.dtype != 0 && o.dtype != 1) throw std::invalid_argument("dtype must be 0 (fp32) or 1 (fp64)");
  if (o.gemm == 2 && o.dtype != 0) throw std::invalid_argument("the tensor-core path needs fp32 storage");
  CK(cudaSetDevice(o.device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, o.device));
  impl_->sm_count = prop.multiProcessorCount;
  if (prop.major != 10)
    throw std::runtime_error("mlnmf_b200 requires an sm_100 (B200) GPU; found " + std::string(prop.name));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  impl_->s = st;
  stream_ = st;
  impl_->flags.ensure(16);
  CK(cudaMemsetAsync(impl_->flags.p, 0, 16, st));
  impl_->scal.ensure(16 * 8);
  impl_->tstart.ensure(8);
  impl_->tc = make_tc_gemm(o.dtype == 0 && o.gemm != 1, o.gemm == 2);
  {
    static std::once_flag once;  // per process: load the restriction kernels before any timed build
    std::call_once(once, [] { restrict_tma_prepare(); });
  }
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) throw std::invalid_argument("bad world / rank");
  if (o.has_nccl_id || (o.world > 1 && !o.host_allreduce)) {
    if (!o.has_nccl_id) throw std::invalid_argument("world > 1 needs an NCCL unique id (or a host allreduce)");
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_id, sizeof(id));
    nccl_check(NcclApi::get().CommInitRank(&impl_->comm, o.world, id, o.rank), "CommInitRank");
  }
}

Engine::~Engine() {
  if (!impl_) return;
  cudaStreamSynchronize(impl_->s);
  for (auto& L : lv_) {
    dev_free(L.M);
    dev_free(L.V);
    dev_free(L.mstat);
    dev_free(L.Rp), dev_free(L.Ri), dev_free(L.Rw), dev_free(L.Pp), dev_free(L.Pi), dev_free(L.Pw), dev_free(L.Rc);
  }
  for (DevBuf* b : {&impl_->gws, &impl_->AB, &impl_->Cb, &impl_->Db, &impl_->part, &impl_->red, &impl_->scal, &impl_->W,
                    &impl_->samples, &impl_->counts, &impl_->flags, &impl_->tstart, &impl_->stage})
    b->release();
  for (auto& p : impl_->ev_mwt) cudaEventDestroy(p.first), cudaEventDestroy(p.second);
  for (auto& p : impl_->ev_vtm) cudaEventDestroy(p.first), cudaEventDestroy(p.second);
  for (auto& p : impl_->ev_comm) cudaEventDestroy(p.first), cudaEventDestroy(p.second);
  for (auto& p : impl_->ev_phase) cudaEventDestroy(p.second.first), cudaEventDestroy(p.second.second);
  for (auto x : impl_->ev_pool) cudaEventDestroy(x);
  delete impl_->tc;
  if (impl_->comm) NcclApi::get().CommDestroy(impl_->comm);
  cudaStreamDestroy(impl_->s);
  delete impl_;
}

bool Engine::tc_active() const { return impl_->tc && !lv_.empty() && r_ > 0 && impl_->use_tc(0); }
bool Engine::gram_error() const {
  if (opt_.error_mode == 1) return true;
  if (opt_.error_mode == 2) return false;
  // auto: the Gram identity needs fp64-accurate C, D (SURVEY finding 4: the
  // SIMT products accumulate in fp64, the tensor-path products exactly in
  // int32) and a non-exact run (exact mode reproduces the reference's direct
  // residual).
  return !opt_.exact;
}

void Engine::sync() { CK(cudaStreamSynchronize(impl_->s)); }

template <typename T>
static void validate_dev(Engine::Impl* im, const T* M, size_t count) {
  CK(cudaMemsetAsync(im->flags.as<int>() + 2, 0, 4, im->s));
  im->launch(k_validate<T>, dim3((unsigned)std::min<size_t>(ceil_div(count, 256), 4096)), dim3(256), 0, M, count,
             im->flags.as<int>() + 2);
  int f = 0;
  CK(cudaMemcpyAsync(&f, im->flags.as<int>() + 2, 4, cudaMemcpyDeviceToHost, im->s));
  CK(cudaStreamSynchronize(im->s));
  if (f) throw std::invalid_argument("Matrix::from_data: negative or non-finite entry");
}

void Engine::set_data(const void* M, int host_dtype, bool is_device, size_t m, size_t n_loc, size_t n_total,
                      size_t col0, size_t h, size_t w, bool validate) {
  if (m == 0 || n_loc == 0) throw std::invalid_argument("Matrix: dimensions must be positive");
  if (h * w != m) throw std::invalid_argument("GridHierarchy: grid does not match matrix rows");
  for (auto& L : lv_) {
    dev_free(L.M), dev_free(L.V), dev_free(L.mstat);
    dev_free(L.Rp), dev_free(L.Ri), dev_free(L.Rw), dev_free(L.Pp), dev_free(L.Pi), dev_free(L.Pw), dev_free(L.Rc);
  }
  lv_.clear();
  impl_->tc_ok.clear();
  n_loc_ = n_loc;
  n_total_ = n_total;
  col0_ = col0;
  Level L0{h, w, m};
  L0.dt = opt_.dtype;
  const size_t count = m * n_loc, es = impl_->esz();
  CK(dev_malloc(&L0.M, count * es));
  lv_.push_back(L0);
  cudaStream_t s = impl_->s;
  const size_t hs = host_dtype == 0 ? 4 : 8;
  const cudaMemcpyKind kind = is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if ((size_t)hs == es) {
    const size_t bytes = count * es;
    if (kind == cudaMemcpyHostToDevice && bytes >= ((size_t)1 << 30)) {
      // large uploads: 256 MiB pieces alternating over the engine stream and a
      // second stream, so two copy engines pull from host memory at once
      cudaStream_t s2 = nullptr;
      cudaEvent_t done = nullptr;
      CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      const size_t piece = (size_t)256 << 20;
      size_t k = 0;
      for (size_t off = 0; off < bytes; off += piece, ++k)
        CK(cudaMemcpyAsync(static_cast<char*>(L0.M) + off, static_cast<const char*>(M) + off,
                           std::min(piece, bytes - off), kind, (k & 1) ? s2 : s));
      CK(cudaEventRecord(done, s2));
      CK(cudaStreamWaitEvent(s, done, 0));
      CK(cudaStreamSynchronize(s));
      cudaEventDestroy(done);
      cudaStreamDestroy(s2);
    } else {
      CK(cudaMemcpyAsync(L0.M, M, bytes, kind, s));
    }
  } else {
    // convert through a staging buffer in chunks
    const size_t chunk = std::min<size_t>(count, (size_t)64 << 20);
    impl_->stage.ensure(chunk * hs);
    for (size_t off = 0; off < count; off += chunk) {
      const size_t c = std::min(chunk, count - off);
      CK(cudaMemcpyAsync(impl_->stage.p, static_cast<const char*>(M) + off * hs, c * hs, kind, s));
      const unsigned g = (unsigned)std::min<size_t>(ceil_div(c, 256), 8192);
      if (hs == 8)
        impl_->launch(k_convert<float>, dim3(g), dim3(256), 0, (const double*)impl_->stage.p,
                      static_cast<float*>(L0.M) + off, c);
      else
        impl_->launch(k_widen<float>, dim3(g), dim3(256), 0, (const float*)impl_->stage.p,
                      static_cast<double*>(L0.M) + off, c);
      CK(cudaStreamSynchronize(s));  // staging reuse
    }
  }
  if (validate) {
    if (opt_.dtype == 0) validate_dev(impl_, static_cast<const float*>(L0.M), count);
    else validate_dev(impl_, static_cast<const double*>(L0.M), count);
  }
  impl_->B_valid = impl_->CD_valid = false;
  CK(cudaStreamSynchronize(s));
}

void Engine::generate(const GenParams& g, size_t n_total, size_t col0, size_t n_loc) {
  const size_t m = g.h * g.w;
  // allocate level 0
  for (auto& L : lv_) {
    dev_free(L.M), dev_free(L.V), dev_free(L.mstat);
    dev_free(L.Rp), dev_free(L.Ri), dev_free(L.Rw), dev_free(L.Pp), dev_free(L.Pi), dev_free(L.Pw), dev_free(L.Rc);
  }
  lv_.clear();
  impl_->tc_ok.clear();
  n_loc_ = n_loc;
  n_total_ = n_total;
  col0_ = col0;
  Level L0{g.h, g.w, m};
  L0.dt = opt_.dtype;
  CK(dev_malloc(&L0.M, m * n_loc * impl_->esz()));
  lv_.push_back(L0);
  cudaStream_t s = impl_->s;
  const int r = (int)g.r;
  if (n_loc > ((size_t)1 << 31)) throw std::invalid_argument("generate: too many columns per rank");
  DevBuf V0, W0, bm;
  V0.ensure(m * r * 8);
  W0.ensure((size_t)r * n_loc * 8);
  impl_->launch(k_gen_basis, dim3((unsigned)std::min<size_t>(ceil_div(m * r, 256), 8192)), dim3(256), 0,
                V0.as<double>(), g.h, g.w, r, (int)g.blobs, g.sigma_min, g.sigma_max, gen_key(g.seed, 1));
  impl_->launch(k_gen_wcols, dim3((unsigned)std::min<size_t>(ceil_div(r * n_loc, 256), 8192)), dim3(256), 0,
                W0.as<double>(), r, n_loc, n_total, col0, gen_key(g.seed, 2));
  const uint64_t kn = gen_key(g.seed, 3);
  const size_t smem = ((size_t)r * 128 + 32 * (size_t)r) * 8;
  const dim3 gg((unsigned)ceil_div(n_loc, 128), (unsigned)ceil_div(m, 32));
  auto run = [&](int mode, double div) {
    if (opt_.dtype == 0)
      impl_->launch(k_gen_m<float>, gg, dim3(128), smem, static_cast<float*>(L0.M), (const double*)V0.as<double>(),
                    (const double*)W0.as<double>(), m, n_loc, r, col0, kn, g.noise_kind, g.noise_scale, mode, div,
                    bm.as<double>());
    else
      impl_->launch(k_gen_m<double>, gg, dim3(128), smem, static_cast<double*>(L0.M), (const double*)V0.as<double>(),
                    (const double*)W0.as<double>(), m, n_loc, r, col0, kn, g.noise_kind, g.noise_scale, mode, div,
                    bm.as<double>());
  };
  if (!g.scale_to_unit) {
    run(0, 1.0);
  } else {
    // M /= max(M) over the whole (all-rank) matrix, computed on the fp64 values
    bm.ensure((size_t)gg.x * gg.y * 8);
    run(1, 1.0);
    impl_->launch(k_max_final, dim3(1), dim3(1024), 0, (const double*)bm.as<double>(), (size_t)gg.x * gg.y,
                  impl_->scal.as<double>() + 3);
    impl_->allreduce_max(impl_->scal.as<double>() + 3, 1);
    double mx = 0;
    CK(cudaMemcpyAsync(&mx, impl_->scal.as<double>() + 3, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    run(2, mx);
  }
  CK(cudaStreamSynchronize(s));
  V0.release();
  W0.release();
  bm.release();
  impl_->B_valid = impl_->CD_valid = false;
}

void Engine::ensure_levels(size_t L) {
  if (lv_.empty()) throw std::invalid_argument("no data set");
  if (L < 1) throw std::invalid_argument("GridHierarchy: need at least one level");
  while (lv_.size() < L) {
    Level& cur = lv_.back();
    if (cur.h < 2 || cur.w < 2) throw std::invalid_argument("GridHierarchy: too many levels for this grid");
    HostCsr R = build_restriction(cur.h, cur.w), P = build_prolongation(cur.h, cur.w);
    auto up = [&](const HostCsr& op, int** p, int** i, double** w) {
      CK(dev_malloc(p, op.rowptr.size() * 4));
      CK(dev_malloc(i, op.idx.size() * 4));
      CK(dev_malloc(w, op.wt.size() * 8));
      CK(cudaMemcpy(*p, op.rowptr.data(), op.rowptr.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(*i, op.idx.data(), op.idx.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(*w, op.wt.data(), op.wt.size() * 8, cudaMemcpyHostToDevice));
    };
    up(R, &cur.Rp, &cur.Ri, &cur.Rw);
    up(P, &cur.Pp, &cur.Pi, &cur.Pw);
    {  // k_restrict_slab's decoded entries: fine row i and column offset dj
      const size_t hcn = (cur.h + 1) / 2;
      std::vector<int> code(R.idx.size());
      for (size_t o = 0; o + 1 < R.rowptr.size(); ++o)
        for (int e = R.rowptr[o]; e < R.rowptr[o + 1]; ++e) {
          const long f = R.idx[e], j = f / (long)cur.h, i = f % (long)cur.h, dj = j - 2 * (long)(o / hcn);
          code[e] = (int)(i * 4 + (dj + 1));
        }
      CK(dev_malloc(&cur.Rc, code.size() * 4));
      CK(cudaMemcpy(cur.Rc, code.data(), code.size() * 4, cudaMemcpyHostToDevice));
    }
    double pf = 0.0;
    for (double x : P.wt) pf += x * x;
    cur.p_fro = std::sqrt(pf);
    Level nx{(cur.h + 1) / 2, (cur.w + 1) / 2, 0};
    nx.m = nx.h * nx.w;
    // Storage of the restricted level: fp32 only where the tensor path will
    // stream it (its input format); otherwise fp64, so an fp32 session's
    // small pyramids are not rounded to fp32 (the oracle restricts in fp64:
    // config 3's 5-level runs deviated 9e-5 with fp32 levels, r02)
    nx.dt = (cur.dt == 0 && impl_->tc && impl_->tc->wants(nx.m, n_loc_, 64)) ? 0 : 1;
    const size_t esn = nx.dt == 0 ? 4 : 8, esc = cur.dt == 0 ? 4 : 8;
    CK(dev_malloc(&nx.M, nx.m * n_loc_ * esn));
    const int h = (int)cur.h, w = (int)cur.w, hc = (int)nx.h, wc = (int)nx.w;
    // Narrow or unaligned matrices (the wide ones take restrict_tma.cu below):
    // column slabs x coarse-row strips with the strip's fine pixel columns
    // staged once by cp.async (k_restrict_slab), else the gather.  256-byte
    // slabs (narrower while that leaves fewer than 8 slabs), 8-row strips,
    // 5-slot ring: measured on the config-4 pyramid (r02: 60 ms for 64-byte
    // slabs of whole pixel columns -> 40 ms; profiles/README.md).
    int slabb = 256, strip = 8;
    constexpr int ns = 5;
    while (slabb > 64 && n_loc_ * esc < (size_t)slabb * 8) slabb /= 2;
    if (strip > hc) strip = hc;
    const size_t slab_smem = (size_t)ns * (2 * strip + 1) * slabb;
    auto restrict_to = [&](auto tin, auto tout, auto f64math) {
      using TI = decltype(tin);
      using TO = decltype(tout);
      constexpr bool F64 = decltype(f64math)::value;
      const TI* X = static_cast<const TI*>(cur.M);
      TO* Y = static_cast<TO*>(nx.M);
      if (slab_smem <= 200 * 1024) {
        const dim3 g((unsigned)ceil_div(n_loc_ * esc, (size_t)slabb), (unsigned)ceil_div((size_t)hc, (size_t)strip));
        auto go = [&](auto kern) {
          impl_->launch(kern, g, dim3(256), slab_smem, (const int*)cur.Rp, (const int*)cur.Rc,
                        (const double*)cur.Rw, X, Y, h, w, hc, wc, n_loc_, strip);
        };
        auto with = [&](auto sb, auto nsv) {
          constexpr int SB = decltype(sb)::value, NSV = decltype(nsv)::value;
          if ((n_loc_ * esc) % 16 == 0) go(k_restrict_slab<TI, TO, 16 / sizeof(TI), F64, SB, NSV>);
          else go(k_restrict_slab<TI, TO, 1, F64, SB, NSV>);
        };
        auto with_ns = [&](auto sb) { with(sb, std::integral_constant<int, ns>()); };
        if (slabb == 256) with_ns(std::integral_constant<int, 256>());
        else if (slabb == 128) with_ns(std::integral_constant<int, 128>());
        else with_ns(std::integral_constant<int, 64>());
      } else {
        const size_t colblocks = ceil_div(n_loc_, 256);
        impl_->launch(k_csr_apply<TI, TO>, dim3((unsigned)(nx.m * colblocks)), dim3(256), 0, (const int*)cur.Rp,
                      (const int*)cur.Ri, (const double*)cur.Rw, X, Y, nx.m, n_loc_, colblocks);
      }
    };
    RestrictArgs ra{cur.M, nx.M, h, w, hc, wc, n_loc_,
                    cur.dt == 1, cur.dt == 0 && nx.dt == 1, impl_->exact()};
    // 8 coarse rows per CTA, 6-slot ring (52 KB, 4 CTAs per SM): level 0 of
    // config 4 in 14.1 ms = 6.1 TB/s of algorithmic bytes (r02 sweep: rings
    // of 4-5 or >= 8 slots and 4- or 32-row strips were 1.5-3x slower)
    const int tma_strip = 8, tma_slots = 6;
    if (restrict_tma_supported(ra)) {
      // the TMA-pipelined stream (restrict_tma.cu): wide matrices
      restrict_tma(ra, tma_strip, tma_slots, impl_->s);
      ++launches_;
    } else if (cur.dt == 1)
      restrict_to(double(), double(), std::true_type());
    else if (nx.dt == 1)
      restrict_to(float(), double(), std::true_type());
    else if (impl_->exact())
      restrict_to(float(), float(), std::true_type());
    else
      restrict_to(float(), float(), std::false_type());
    if (r_ > 0) CK(dev_malloc(&nx.V, nx.m * r_ * 8));  // factors are fp64
    lv_.push_back(nx);
  }
  CK(cudaStreamSynchronize(impl_->s));
  impl_->decide_tc();
}

double Engine::norm2(size_t l) {
  Level& L = lv_.at(l);
  if (L.norm2 < 0) {
    double* sc = impl_->scal.as<double>();
    if (L.dt == 0 && !L.mstat && impl_->use_tc_known(l)) impl_->level_stats(l, sc + 4);  // fused with the tensor path's maxima
    else if (L.dt == 0) impl_->dot<float>(L.M, 1, nullptr, 0, L.m * n_loc_, sc + 4);
    else impl_->dot<double>(L.M, 1, nullptr, 0, L.m * n_loc_, sc + 4);
    impl_->allreduce_sum(sc + 4, 1);
    CK(cudaMemcpyAsync(&L.norm2, sc + 4, 8, cudaMemcpyDeviceToHost, impl_->s));
    CK(cudaStreamSynchronize(impl_->s));
  }
  return L.norm2;
}

double Engine::smoothness(size_t l) {
  ensure_levels(l + 2);
  const double nrm2 = norm2(l);
  if (!(nrm2 > 0.0)) throw std::invalid_argument("smoothness: undefined for the zero matrix");
  const Level &F = lv_[l], &Cl = lv_[l + 1];
  const size_t cb = ceil_div(n_loc_, 256);
  const size_t ry = std::max<size_t>(1, std::min(F.m, ceil_div(kTargetBlocks, cb)));
  impl_->part.ensure(cb * ry * 8);
  double* part = impl_->part.as<double>();
  double* sc = impl_->scal.as<double>();
  auto go = [&](auto tc_, auto tf_) {
    using TC = decltype(tc_);
    using TF = decltype(tf_);
    impl_->launch(k_csr_residual<TC, TF>, dim3((unsigned)cb, (unsigned)ry), dim3(256), 0, (const int*)F.Pp,
                  (const int*)F.Pi, (const double*)F.Pw, (const TC*)Cl.M, (const TF*)F.M, F.m, n_loc_, part);
  };
  if (F.dt == 0 && Cl.dt == 0) go(float(), float());
  else if (F.dt == 0) go(double(), float());
  else go(double(), double());
  impl_->launch(k_sum_final, dim3(1), dim3(1024), 0, (const double*)part, cb * ry, sc + 5, 0);
  impl_->allreduce_sum(sc + 5, 1);
  double s = 0;
  CK(cudaMemcpyAsync(&s, sc + 5, 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
  return std::sqrt(s) / std::sqrt(nrm2);
}

void Engine::initialization_bound(size_t l, const void* V_coarse, const void* W, int host_dtype, size_t r,
                                  double* lhs, double* rhs) {
  ensure_levels(l + 2);
  set_factors(l + 1, V_coarse, W, host_dtype, r);
  prolong_V(l);
  *lhs = frobenius_error(l);
  const double coarse_err = frobenius_error(l + 1);
  const double sM = smoothness(l);
  *rhs = sM * std::sqrt(norm2(l)) + lv_[l].p_fro * coarse_err;
}

void Engine::init_random(size_t r, uint64_t seed) {
  if (lv_.empty()) throw std::invalid_argument("no data set");
  const size_t m0 = lv_[0].m;
  if (r < 1 || r > std::min(m0, n_total_))
    throw std::invalid_argument("random_init: rank must satisfy 1 <= r <= min(m,n)");
  set_factors(0, nullptr, nullptr, opt_.dtype, r);
  const size_t tot = m0 * r + r * n_loc_;
  const unsigned g = (unsigned)std::min<size_t>(ceil_div(tot, 256), 8192);
  impl_->launch(k_random_init<double>, dim3(g), dim3(256), 0, static_cast<double*>(lv_[0].V), impl_->W.as<double>(),
                m0, r, n_loc_, n_total_, col0_, seed);
}

// The factors are fp64 on the device whatever M's storage: they are small
// (V m x r, W r x n_loc: 0.2 GB at config 4, against 64 GiB of M), so fp64
// costs nothing measurable, and it keeps fp32-M runs from rounding the
// iterates to fp32 after every sweep (the dominant trajectory deviation from
// the fp64 reference fed the same fp32 M).
void Engine::set_factors(size_t l, const void* V, const void* W, int host_dtype, size_t r) {
  if (lv_.empty()) throw std::invalid_argument("no data set");
  if (r != r_) {
    for (auto& L : lv_) {
      dev_free(L.V);
      L.V = nullptr;
    }
    r_ = r;
  }
  for (auto& L : lv_)
    if (!L.V) CK(dev_malloc(&L.V, L.m * r * 8));
  impl_->W.ensure(r * n_loc_ * 8);
  impl_->AB.ensure((lv_[0].m * r + r * r) * 8);
  impl_->Cb.ensure(r * n_loc_ * 8);
  impl_->Db.ensure(r * r * 8);
  impl_->B_valid = impl_->CD_valid = false;
  auto put = [&](void* dst, const void* src, size_t count) {
    if (!src) return;
    if (host_dtype != 0) {
      CK(cudaMemcpyAsync(dst, src, count * 8, cudaMemcpyHostToDevice, impl_->s));
    } else {
      impl_->stage.ensure(count * 4);
      CK(cudaMemcpyAsync(impl_->stage.p, src, count * 4, cudaMemcpyHostToDevice, impl_->s));
      const unsigned g = (unsigned)std::min<size_t>(ceil_div(count, 256), 8192);
      impl_->launch(k_widen<float>, dim3(g), dim3(256), 0, (const float*)impl_->stage.p, (double*)dst, count);
    }
    CK(cudaStreamSynchronize(impl_->s));
  };
  put(lv_.at(l).V, V, lv_[l].m * r);
  put(impl_->W.p, W, r * n_loc_);
  impl_->decide_tc();
}

void Engine::get_factors(size_t l, void* V, void* W, int host_dtype) {
  auto get = [&](const void* src, void* dst, size_t count) {
    if (!dst) return;
    if (host_dtype != 0) {
      CK(cudaMemcpyAsync(dst, src, count * 8, cudaMemcpyDeviceToHost, impl_->s));
    } else {
      impl_->stage.ensure(count * 4);
      const unsigned g = (unsigned)std::min<size_t>(ceil_div(count, 256), 8192);
      impl_->launch(k_convert<float>, dim3(g), dim3(256), 0, (const double*)src, (float*)impl_->stage.p, count);
      CK(cudaMemcpyAsync(dst, impl_->stage.p, count * 4, cudaMemcpyDeviceToHost, impl_->s));
    }
    CK(cudaStreamSynchronize(impl_->s));
  };
  get(lv_.at(l).V, V, lv_[l].m * r_);
  get(impl_->W.p, W, r_ * n_loc_);
}

void Engine::export_data(void* M_host, int host_dtype) {
  if (lv_.empty()) throw std::invalid_argument("no data set");
  const size_t count = lv_[0].m * n_loc_, es = impl_->esz(), hs = host_dtype == 0 ? 4 : 8;
  if (hs != es) throw std::invalid_argument("export_data: host dtype must match the storage dtype");
  CK(cudaMemcpyAsync(M_host, lv_[0].M, count * es, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
}

void Engine::gram_v(double* D_host) {
  if (lv_.empty() || r_ == 0) throw std::invalid_argument("gram_v: no data or factors");
  if (opt_.dtype == 0) impl_->gram_V<float>(0);
  else impl_->gram_V<double>(0);
  impl_->CD_valid = false;
  CK(cudaMemcpyAsync(D_host, impl_->Db.p, r_ * r_ * 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
}

void Engine::gram_w(double* B_host) {
  if (lv_.empty() || r_ == 0) throw std::invalid_argument("gram_w: no data or factors");
  if (opt_.dtype == 0) impl_->gram_W<float>();
  else impl_->gram_W<double>();
  impl_->B_valid = false;  // a rank-local value: the step's allreduced B is recomputed
  CK(cudaMemcpyAsync(B_host, impl_->B(), r_ * r_ * 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
}

int Engine::export_level(size_t level, void* M_host) {
  if (level >= lv_.size()) throw std::invalid_argument("level not built");
  const Level& L = lv_[level];
  if (M_host) {
    CK(cudaMemcpyAsync(M_host, L.M, L.m * n_loc_ * (L.dt == 0 ? 4 : 8), cudaMemcpyDeviceToHost, impl_->s));
    CK(cudaStreamSynchronize(impl_->s));
  }
  return L.dt;
}

void Engine::products(double* A, double* C) {
  if (lv_.empty() || r_ == 0) throw std::invalid_argument("products: no data or factors");
  if (opt_.dtype == 0) {
    impl_->product_mwt<float>(0);
    impl_->product_vtm<float>(0);
  } else {
    impl_->product_mwt<double>(0);
    impl_->product_vtm<double>(0);
  }
  impl_->CD_valid = false;
  if (A) CK(cudaMemcpyAsync(A, impl_->A(), lv_[0].m * r_ * 8, cudaMemcpyDeviceToHost, impl_->s));
  if (C) CK(cudaMemcpyAsync(C, impl_->Cb.p, r_ * n_loc_ * 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
}

void Engine::restrict_V(size_t l) {
  Level& f = lv_.at(l);
  Level& c = lv_.at(l + 1);
  const size_t cb = ceil_div(r_, 64);
  impl_->launch(k_csr_apply<double>, dim3((unsigned)(c.m * cb)), dim3(64), 0, (const int*)f.Rp, (const int*)f.Ri,
                (const double*)f.Rw, (const double*)f.V, static_cast<double*>(c.V), c.m, r_, cb);
}

void Engine::prolong_V(size_t l) {
  Level& f = lv_.at(l);
  Level& c = lv_.at(l + 1);
  const size_t cb = ceil_div(r_, 64);
  impl_->launch(k_csr_apply<double>, dim3((unsigned)(f.m * cb)), dim3(64), 0, (const int*)f.Pp, (const int*)f.Pi,
                (const double*)f.Pw, (const double*)c.V, static_cast<double*>(f.V), f.m, r_, cb);
  impl_->CD_valid = false;
}

void Engine::step(size_t l, Kind kind) {
  if (l >= lv_.size()) throw std::invalid_argument("step: level not built");
  if (r_ == 0) throw std::invalid_argument("step: factors not initialised");
  if (impl_->CD_valid && impl_->CD_level != l) impl_->CD_valid = false;
  Impl& im = *impl_;
  // Steady-state HALS / MU steps replay a captured CUDA graph: the step is a
  // fixed sequence of ~10 small launches, launch-bound on the L2-resident
  // configs.  (ANLS appends NNLS counts at moving offsets; multi-rank steps
  // hold NCCL calls; profiling records events: those run eagerly.)
  const bool graphable = im.graphs_on && kind != kAnls && !im.multi() && !profiling_;
  if (graphable) {
    Impl::StepGraph& g = im.graphs[l * 4 + (size_t)kind];
    if (!g.exec || g.epoch != im.graph_sig()) {
      if (!g.warm) {  // one eager step first: buffers reach their steady-state sizes
        g.warm = true;
        im.B_valid = false;
        if (lv_[l].dt == 0) im.step_t<float>(l, kind);
        else im.step_t<double>(l, kind);
        return;
      }
      if (g.exec) cudaGraphExecDestroy(g.exec), g.exec = nullptr;
      const uint64_t ep = im.graph_sig();
      const long l0 = launches_;
      cudaGraph_t graph = nullptr;
      CK(cudaStreamBeginCapture(im.s, cudaStreamCaptureModeRelaxed));
      im.B_valid = false;  // the captured step always recomputes B = W W^T
      try {
        if (lv_[l].dt == 0) im.step_t<float>(l, kind);
        else im.step_t<double>(l, kind);
      } catch (...) {
        cudaStreamEndCapture(im.s, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      CK(cudaStreamEndCapture(im.s, &graph));
      g.nlaunch = launches_ - l0;
      launches_ = l0;
      if (im.graph_sig() != ep) {  // a buffer was reallocated during capture: run eagerly, recapture next time
        cudaGraphDestroy(graph);
        g.warm = false;
        im.B_valid = false;
        if (lv_[l].dt == 0) im.step_t<float>(l, kind);
        else im.step_t<double>(l, kind);
        return;
      }
      CK(cudaGraphInstantiate(&g.exec, graph, 0));
      cudaGraphDestroy(graph);
      g.epoch = ep;
    }
    CK(cudaGraphLaunch(g.exec, im.s));
    launches_ += g.nlaunch;
    im.B_valid = false;
    im.CD_valid = true;
    im.CD_level = l;
    return;
  }
  if (lv_[l].dt == 0) impl_->step_t<float>(l, kind);
  else impl_->step_t<double>(l, kind);
  if (kind == kAnls) impl_->check_nnls();
}

void Engine::sample(size_t l, double work_units) {
  norm2(l);  // host-cached after first use (one sync per level per run)
  if (impl_->CD_valid && impl_->CD_level != l) impl_->CD_valid = false;
  if (lv_[l].dt == 0) impl_->sample_t<float>(l, work_units);
  else impl_->sample_t<double>(l, work_units);
}

void Engine::mark_run_start() {
  impl_->launch(k_timestamp, dim3(1), dim3(1), 0, impl_->tstart.as<unsigned long long>());
  impl_->host_t0 = std::chrono::steady_clock::now();
  CK(cudaMemsetAsync(impl_->flags.p, 0, 8, impl_->s));
  impl_->samp_used = 0;
  impl_->samp_meta.clear();
  impl_->cnt_used = 0;
  impl_->cnt_steps.clear();
}

double Engine::host_elapsed_s() const {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - impl_->host_t0).count();
}

double Engine::agreed_max(double v) {
  if (!impl_->multi()) return v;
  double* d = impl_->scal.as<double>() + 11;
  CK(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, impl_->s));
  impl_->allreduce_max(d, 1);
  CK(cudaMemcpyAsync(&v, d, 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
  return v;
}

double Engine::agreed_elapsed_s() {
  sync();
  return agreed_max(host_elapsed_s());
}

void Engine::flush(std::vector<Sample>* samples, std::vector<int>* counts, int* degenerate) {
  cudaStream_t s = impl_->s;
  std::vector<SampleRec> recs(impl_->samp_used);
  unsigned long long t0 = 0;
  int fl[2] = {0, 0};
  if (!recs.empty())
    CK(cudaMemcpyAsync(recs.data(), impl_->samples.p, recs.size() * sizeof(SampleRec), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&t0, impl_->tstart.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(fl, impl_->flags.p, 8, cudaMemcpyDeviceToHost, s));
  std::vector<int> cn(impl_->cnt_used);
  if (!cn.empty()) CK(cudaMemcpyAsync(cn.data(), impl_->counts.p, cn.size() * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (fl[1] & 1) throw NnlsCapExceeded("anls_step: NNLS exchange cap exceeded");
  if (fl[1] & 2) throw NnlsCapExceeded("anls_step: NNLS failed (singular passive subsystem)");
  if (samples) {
    for (size_t i = 0; i < recs.size(); ++i) {
      Sample smp = impl_->samp_meta[i];
      smp.error = recs[i].error;
      smp.elapsed_s = recs[i].t_ns >= t0 ? (double)(recs[i].t_ns - t0) * 1e-9 : 0.0;
      samples->push_back(smp);
    }
  }
  if (counts && impl_->multi() && !impl_->cnt_steps.empty()) {
    // the reference's layout, m_l V-row counts then all n W-column counts
    // per ANLS step (solvers.cpp:269,296): V rows are replicated, each rank
    // holds its own columns -> one sum-exchange of zero-padded rows
    const size_t S = impl_->cnt_steps.size();
    std::vector<double> wc(S * n_total_, 0.0);
    size_t off = 0;
    for (size_t k = 0; k < S; ++k) {
      off += impl_->cnt_steps[k];
      for (size_t j = 0; j < n_loc_; ++j) wc[k * n_total_ + col0_ + j] = (double)cn[off + j];
      off += n_loc_;
    }
    DevBuf g;
    g.ensure(wc.size() * 8);
    CK(cudaMemcpyAsync(g.p, wc.data(), wc.size() * 8, cudaMemcpyHostToDevice, s));
    impl_->allreduce_sum(g.as<double>(), wc.size());
    CK(cudaMemcpyAsync(wc.data(), g.p, wc.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    g.release();
    off = 0;
    for (size_t k = 0; k < S; ++k) {
      counts->insert(counts->end(), cn.begin() + off, cn.begin() + off + impl_->cnt_steps[k]);
      off += impl_->cnt_steps[k] + n_loc_;
      for (size_t j = 0; j < n_total_; ++j) counts->push_back((int)wc[k * n_total_ + j]);
    }
  } else if (counts) {
    counts->insert(counts->end(), cn.begin(), cn.end());
  }
  if (degenerate) *degenerate += fl[0];
  impl_->samp_used = 0;
  impl_->samp_meta.clear();
  impl_->cnt_used = 0;
  impl_->cnt_steps.clear();
  CK(cudaMemsetAsync(impl_->flags.p, 0, 8, s));
}

double Engine::frobenius_error(size_t l) {
  double* sc = impl_->scal.as<double>();
  if (lv_.at(l).dt == 0) impl_->direct_e2<float>(l, sc);
  else impl_->direct_e2<double>(l, sc);
  double e2 = 0;
  CK(cudaMemcpyAsync(&e2, sc, 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
  return std::sqrt(e2);
}

void Engine::apply_transfer(size_t h, size_t w, int which, const double* X, size_t ncols, double* Y) {
  HostCsr op = which == 0 ? build_restriction(h, w) : build_prolongation(h, w);
  const size_t in_dim = which == 0 ? h * w : ((h + 1) / 2) * ((w + 1) / 2);
  const size_t out_dim = op.rowptr.size() - 1;
  DevBuf p, i, wt, x, y;
  p.ensure(op.rowptr.size() * 4);
  i.ensure(std::max<size_t>(op.idx.size(), 1) * 4);
  wt.ensure(std::max<size_t>(op.wt.size(), 1) * 8);
  x.ensure(in_dim * ncols * 8);
  y.ensure(out_dim * ncols * 8);
  cudaStream_t s = impl_->s;
  CK(cudaMemcpyAsync(p.p, op.rowptr.data(), op.rowptr.size() * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(i.p, op.idx.data(), op.idx.size() * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(wt.p, op.wt.data(), op.wt.size() * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(x.p, X, in_dim * ncols * 8, cudaMemcpyHostToDevice, s));
  const size_t cb = ceil_div(ncols, 128);
  impl_->launch(k_csr_apply<double>, dim3((unsigned)(out_dim * cb)), dim3(128), 0, (const int*)p.p, (const int*)i.p,
                (const double*)wt.p, (const double*)x.p, (double*)y.p, out_dim, ncols, cb);
  CK(cudaMemcpyAsync(Y, y.p, out_dim * ncols * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (DevBuf* b : {&p, &i, &wt, &x, &y}) b->release();
}

void Engine::nnls_single(const double* G, const double* h, const double* x0, size_t r, double* x, int* iterations) {
  if (r < 1) throw std::invalid_argument("nnls_active_set: dimension mismatch");
  DevBuf g, hb, xb, cb;
  g.ensure(r * r * 8);
  hb.ensure(r * 8);
  xb.ensure(r * 8);
  cudaStream_t s = impl_->s;
  CK(cudaMemcpyAsync(g.p, G, r * r * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(hb.p, h, r * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(xb.p, x0, r * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(impl_->flags.p, 0, 8, s));
  const size_t r_save = r_;
  r_ = r;
  impl_->cnt_used = 0;
  try {
    impl_->nnls(g.as<double>(), 1, hb.as<double>(), r, 1, xb.as<double>(), r, 1);
  } catch (...) {
    r_ = r_save;
    throw;
  }
  r_ = r_save;
  int fl[2] = {0, 0}, it = 0;
  CK(cudaMemcpyAsync(x, xb.p, r * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&it, impl_->counts.p, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(fl, impl_->flags.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  impl_->cnt_used = 0;
  for (DevBuf* b : {&g, &hb, &xb, &cb}) b->release();
  if (fl[1] & 1) throw NnlsCapExceeded("nnls_active_set: exchange cap exceeded");
  if (fl[1] & 2) throw std::runtime_error("nnls_active_set: singular passive subsystem");
  *iterations = it;
}

void Engine::random_init_host(size_t m, size_t n, size_t r, uint64_t seed, double* V, double* W) {
  if (r < 1 || r > std::min(m, n)) throw std::invalid_argument("random_init: rank must satisfy 1 <= r <= min(m,n)");
  DevBuf v, w;
  v.ensure(m * r * 8);
  w.ensure(r * n * 8);
  const unsigned g = (unsigned)std::min<size_t>(ceil_div(m * r + r * n, 256), 8192);
  impl_->launch(k_random_init<double>, dim3(g), dim3(256), 0, v.as<double>(), w.as<double>(), m, r, n, n, (size_t)0,
                seed);
  CK(cudaMemcpyAsync(V, v.p, m * r * 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaMemcpyAsync(W, w.p, r * n * 8, cudaMemcpyDeviceToHost, impl_->s));
  CK(cudaStreamSynchronize(impl_->s));
  v.release();
  w.release();
}

KernelTimes Engine::kernel_times() {
  sync();
  KernelTimes kt;
  for (auto& p : impl_->ev_mwt) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, p.first, p.second));
    kt.mwt_ms += ms;
    ++kt.mwt_n;
  }
  for (auto& p : impl_->ev_vtm) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, p.first, p.second));
    kt.vtm_ms += ms;
    ++kt.vtm_n;
  }
  for (auto& p : impl_->ev_comm) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, p.first, p.second));
    kt.comm_ms += ms;
    ++kt.comm_n;
    kt.phase_ms[kPhComm] += ms;
    ++kt.phase_n[kPhComm];
  }
  for (auto& p : impl_->ev_phase) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
    kt.phase_ms[p.first] += ms;
    ++kt.phase_n[p.first];
  }
  return kt;
}

void Engine::reset_kernel_times() {
  sync();
  for (auto& p : impl_->ev_mwt) impl_->ev_pool.push_back(p.first), impl_->ev_pool.push_back(p.second);
  for (auto& p : impl_->ev_vtm) impl_->ev_pool.push_back(p.first), impl_->ev_pool.push_back(p.second);
  for (auto& p : impl_->ev_comm) impl_->ev_pool.push_back(p.first), impl_->ev_pool.push_back(p.second);
  for (auto& p : impl_->ev_phase)
    impl_->ev_pool.push_back(p.second.first), impl_->ev_pool.push_back(p.second.second);
  impl_->ev_phase.clear();
  impl_->ev_mwt.clear();
  impl_->ev_vtm.clear();
  impl_->ev_comm.clear();
}

}  // namespace mlb
