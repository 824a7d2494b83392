// engine.hpp -- device-resident multilevel NMF engine (host interface, no CUDA
// types).  One Engine per GPU (per rank).  It owns M and its restricted levels
// (column shard [col0, col0 + n_loc) of an n_total-column problem), the
// factors V (per level, replicated over ranks) and W (shard-local), and
// enqueues solver steps, transfers and error samples on its own CUDA stream.
// The budget/cycle scheduler (scheduler.cpp) drives it; nothing here decides
// step counts.
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace mlb {

enum Kind { kAnls = 0, kMu = 1, kHals = 2 };              // cost_model.hpp:9
enum Cycle { kNone = 0, kNested = 1, kVCycle = 2, kFmg = 3 };  // multilevel.hpp:11

// Exception classes mirroring the reference (matrix.hpp:15-24); the C-ABI
// maps them to status codes.
struct NnlsCapExceeded : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Host-side collective for ranks that share no NCCL communicator (several
// sessions in one process, e.g. the multi-rank tests on one GPU): called with
// this rank's `count` doubles in host memory, it must leave there the
// element-wise sum (op 0) or max (op 1) over all ranks, every rank calling in
// the same order.  Returns 0 on success.
typedef int (*HostAllreduceFn)(void* ctx, double* buf, size_t count, int op);

struct Options {
  int device = 0;
  int dtype = 1;       // storage of M, V, W: 0 = fp32, 1 = fp64
  int exact = 0;       // reference operation order (fp64 => bit-identical)
  int gemm = 0;        // 0 auto, 1 SIMT (fp64 accumulate), 2 tcgen05 integer-digit products (fp32 only)
  int error_mode = 0;  // 0 auto, 1 Gram identity, 2 direct residual
  int world = 1, rank = 0;
  bool has_nccl_id = false;
  unsigned char nccl_id[128] = {0};
  HostAllreduceFn host_allreduce = nullptr;  // world > 1 without NCCL (see above)
  void* host_allreduce_ctx = nullptr;
};

struct GenParams {
  size_t h = 0, w = 0, r = 0, blobs = 0;
  double sigma_min = 0, sigma_max = 0;
  int noise_kind = 0;  // 0 uniform scale*U[0,1), 1 gaussian N(0, scale^2)
  double noise_scale = 0;
  uint64_t seed = 0;
  int scale_to_unit = 0;
};

struct Sample {
  double elapsed_s;
  double work_units;
  int level;  // 1 = finest
  double error;
};

// Phases of one solver step (engine.cu step_t), timed when profiling is on.
enum StepPhase { kPhB = 0, kPhA, kPhComm, kPhV, kPhD, kPhC, kPhW, kNumPhases };

struct KernelTimes {  // filled when profiling is on (CUDA events on the engine stream)
  double mwt_ms = 0, vtm_ms = 0;  // total over recorded launches
  long mwt_n = 0, vtm_n = 0;
  double comm_ms = 0;  // the per-step allreduce of [A | B] (world > 1)
  long comm_n = 0;
  // per step phase: B = W W^T, A = M W^T, allreduce [A | B], V update,
  // D = V^T V, C = V^T M, W update (totals over the profiled steps)
  double phase_ms[kNumPhases] = {0};
  long phase_n[kNumPhases] = {0};
};

class Engine {
 public:
  explicit Engine(const Options& o);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const Options& options() const { return opt_; }
  int dtype() const { return opt_.dtype; }

  // ---- data and hierarchy ----
  // M_host: m x n_loc row-major, host_dtype 0 = fp32 / 1 = fp64; is_device
  // marks a device pointer (copied).  Rejects negative / non-finite entries
  // (Matrix::from_data, matrix.cpp:10-22) when validate is set.
  void set_data(const void* M, int host_dtype, bool is_device, size_t m, size_t n_loc, size_t n_total,
                size_t col0, size_t h, size_t w, bool validate);
  void generate(const GenParams& g, size_t n_total, size_t col0, size_t n_loc);
  void ensure_levels(size_t L);  // GridHierarchy::build (transfer.cpp:155-174)
  size_t built_levels() const { return lv_.size(); }
  size_t m(size_t l) const { return lv_.at(l).m; }
  size_t grid_h(size_t l) const { return lv_.at(l).h; }
  size_t grid_w(size_t l) const { return lv_.at(l).w; }
  size_t n_loc() const { return n_loc_; }
  size_t n_total() const { return n_total_; }
  size_t col0() const { return col0_; }
  size_t rank_r() const { return r_; }
  double norm2(size_t l);  // ||M_l||_F^2 over all ranks

  // ---- factors ----
  void init_random(size_t r, uint64_t seed);  // random_init at level 0 (matrix.cpp:51-60)
  void set_factors(size_t l, const void* V, const void* W, int host_dtype, size_t r);  // V at level l, W
  void get_factors(size_t l, void* V, void* W, int host_dtype);
  void export_data(void* M_host, int host_dtype);  // level-0 M to a host buffer
  void gram_v(double* D_host);                     // D = V^T V of level 0 through the active kernel
  void gram_w(double* B_host);                     // B = W W^T (this rank's shard, not allreduced) through the active kernel
  int export_level(size_t level, void* M_host);    // level data to a host buffer (NULL: only the dtype); returns the level's dtype
  // the two M-streaming products at level 0 with the current factors, through
  // the active path: A = M W^T (m x r), C = V^T M (r x n_loc), fp64 to host
  void products(double* A, double* C);
  void restrict_V(size_t l);  // V_{l+1} = R_l V_l   (multilevel.cpp:39)
  void prolong_V(size_t l);   // V_l = P_l V_{l+1}   (multilevel.cpp:41)

  // ---- solver ----
  void step(size_t l, Kind kind);  // one mu/hals/anls sweep (solvers.cpp:79-298), async
  // Enqueue an error sample of (M_l, V_l, W); metadata kept on the host.
  void sample(size_t l, double work_units);
  void mark_run_start();          // device timestamp the sample clock is relative to
  void flush(std::vector<Sample>* samples, std::vector<int>* counts, int* degenerate);  // sync + collect
  void sync();
  double host_elapsed_s() const;  // host clock since mark_run_start (time-budget mode)
  // wall-clock budgets: sync the stream and return host_elapsed_s(), the
  // maximum over ranks (every rank then takes the same decisions)
  double agreed_elapsed_s();
  double agreed_max(double v);  // max of a host value over ranks (identity on one rank)

  // ---- standalone kernels for the step-level C-ABI ----
  double frobenius_error(size_t l);  // sync
  // diagnostics (transfer.cpp:128-153) over the resident pyramid, all ranks:
  // s_M = ||M_l - P R M_l||_F / ||M_l||_F, and both sides of the coarse-
  // initialization bound for V_coarse at level l+1 and W (overwrites the
  // session's V at levels l, l+1 and W)
  double smoothness(size_t l);
  void initialization_bound(size_t l, const void* V_coarse, const void* W, int host_dtype, size_t r, double* lhs,
                            double* rhs);
  void apply_transfer(size_t h, size_t w, int which, const double* X, size_t ncols, double* Y);
  void nnls_single(const double* G, const double* h, const double* x0, size_t r, double* x, int* iterations);
  void random_init_host(size_t m, size_t n, size_t r, uint64_t seed, double* V, double* W);

  // ---- instrumentation ----
  void set_profiling(bool on) { profiling_ = on; }
  KernelTimes kernel_times();
  void reset_kernel_times();
  long launches() const { return launches_; }
  void* stream() const { return stream_; }
  bool tc_active() const;  // tcgen05 path selected for the M-streaming products
  bool gram_error() const;

  struct Impl;

 private:
  struct Level {
    size_t h, w, m;
    int dt = 1;  // storage of M at this level: 0 fp32, 1 fp64 (level 0: the session's dtype)
    void* M = nullptr;  // T[m x n_loc]
    void* V = nullptr;  // T[m x r]
    float* mstat = nullptr;  // tensor path: row maxima (m) then column maxima (n_loc) of M
    double norm2 = -1;
    double p_fro = 0;  // ||P||_F of P: next -> this (TransferOperator::frobenius_norm)
    // R: this level -> next; P: next -> this (device CSR)
    int *Rp = nullptr, *Ri = nullptr, *Pp = nullptr, *Pi = nullptr;
    int* Rc = nullptr;  // R's entries pre-decoded for k_restrict_slab: i * 4 + (dj + 1)
    double *Rw = nullptr, *Pw = nullptr;
  };
  Options opt_;
  Impl* impl_;
  void* stream_ = nullptr;
  std::vector<Level> lv_;
  size_t n_loc_ = 0, n_total_ = 0, col0_ = 0, r_ = 0;
  bool profiling_ = false;
  long launches_ = 0;
  friend struct Impl;
};

}  // namespace mlb
