// cli_main.cpp -- `mlnmf_b200`, the command-line front-end of the B200 solver.
//
// The same four subcommands, options, output files, stdout lines and exit
// codes as the reference CLI (proj/tools/mlnmf_main.cpp:89-233), with every
// solve on the GPU through the C-ABI (include/mlnmf_b200.h):
//
//   factorize       run_configuration -> <out>.trace.csv, <out>.V.csv,
//                   <out>.W.csv, <out>.basis/ (grid data)      (:149-166)
//   bench           run_bench grid -> <out>.summary.csv / .summary.txt,
//                   the txt echoed to stdout                   (:168-186)
//   transfer-check  s_M and the R / P row-sum deviations per level (:188-211)
//   synth           the seeded synthetic PGM set (host only)   (:213-218)
//
// Exit codes (:221-233): 0 ok, 2 usage / invalid arguments, 3 data error,
// 4 NNLS cap exceeded, 1 anything else (CUDA failures included).
// B200-specific options (not in the reference): --precision fp64 (default:
// the reference's operation order, bit-identical results) | fp64-fast | fp32
// (fp32 storage, tcgen05 integer-digit products), --device k, and for bench
// --workers w (concurrent device sessions per configuration).
// Argument parsing is a small hand-written `--name value` / `--name=value`
// scanner (the reference uses CLI11, which is not part of this build).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_io.hpp"
#include "mlnmf_b200.h"
#include "transfer_ops.hpp"

namespace {

using mlb::io::DataError;
using mlb::io::Dataset;

// usage errors (CLI11 ParseError / ValidationError in the reference): exit 2
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NnlsCapExceeded : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// C-ABI status -> the reference's exception classes
void ck(int rc) {
  if (rc == MLNMF_OK) return;
  const std::string msg = mlnmf_last_error();
  switch (rc) {
    case MLNMF_ERR_INVALID: throw std::invalid_argument(msg);
    case MLNMF_ERR_DATA: throw DataError(msg);
    case MLNMF_ERR_NNLS_CAP: throw NnlsCapExceeded(msg);
    default: throw std::runtime_error(msg);
  }
}

// ---------------------------------------------------------------------------
// options
// ---------------------------------------------------------------------------
struct Spec {
  const char* name;
  bool required;
  bool numeric = false;  // unsigned integer, checked at parse time (CLI11 conversion)
};

class Args {
 public:
  // parse argv[first..] against the allowed option names
  Args(int argc, char** argv, int first, const std::string& cmd, const std::vector<Spec>& specs) : cmd_(cmd) {
    std::map<std::string, bool> allowed;
    for (const Spec& s : specs) allowed[s.name] = s.required;
    for (int i = first; i < argc; ++i) {
      std::string a = argv[i];
      if (a == "--help" || a == "-h") {
        help_ = true;
        continue;
      }
      if (a.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + a);
      std::string name = a.substr(2), value;
      const size_t eq = name.find('=');
      if (eq != std::string::npos) {
        value = name.substr(eq + 1);
        name = name.substr(0, eq);
      } else {
        if (i + 1 >= argc) throw UsageError("--" + name + ": 1 required value missing");
        value = argv[++i];
      }
      if (!allowed.count(name)) throw UsageError("The following argument was not expected: --" + name);
      v_[name] = value;
    }
    if (help_) return;
    for (const Spec& s : specs) {
      if (s.required && !v_.count(s.name)) throw UsageError(std::string("--") + s.name + " is required");
      if (s.numeric) u64(s.name, 0);
    }
  }
  bool help() const { return help_; }
  std::string str(const std::string& k, const std::string& dflt) const {
    auto it = v_.find(k);
    return it == v_.end() ? dflt : it->second;
  }
  // unsigned integer option: digits only (CLI11 rejects signs and junk)
  uint64_t u64(const std::string& k, uint64_t dflt) const {
    auto it = v_.find(k);
    if (it == v_.end()) return dflt;
    const std::string& s = it->second;
    bool ok = !s.empty();
    for (char c : s) ok = ok && c >= '0' && c <= '9';
    if (!ok) throw UsageError("--" + k + ": Value " + s + " could not be converted");
    errno = 0;
    const unsigned long long v = std::strtoull(s.c_str(), nullptr, 10);
    if (errno == ERANGE) throw UsageError("--" + k + ": Value " + s + " could not be converted");
    return v;
  }

 private:
  std::string cmd_;
  std::map<std::string, std::string> v_;
  bool help_ = false;
};

// parse_budget (mlnmf_main.cpp:19-36)
struct BudgetSpec {
  int mode;
  double amount;
};
BudgetSpec parse_budget(const std::string& spec) {
  const size_t colon = spec.find(':');
  if (colon == std::string::npos) throw UsageError("--budget: expected work:<units> or time:<seconds>");
  const std::string mode = spec.substr(0, colon);
  double amount;
  try {
    amount = std::stod(spec.substr(colon + 1));
  } catch (const std::exception&) {
    throw UsageError("--budget: unparsable amount in '" + spec + "'");
  }
  if (amount <= 0.0) throw UsageError("--budget: amount must be positive");
  if (mode == "work") return {MLNMF_WORK_UNITS, amount};
  if (mode == "time") return {MLNMF_WALL_CLOCK_SECONDS, amount};
  throw UsageError("--budget: unknown mode '" + mode + "'");
}

int parse_algo(const std::string& s) {
  if (s == "anls") return MLNMF_ANLS;
  if (s == "mu") return MLNMF_MU;
  if (s == "hals") return MLNMF_HALS;
  throw UsageError("--algo: unknown algorithm '" + s + "'");
}
const char* algo_name(int k) { return k == MLNMF_ANLS ? "anls" : k == MLNMF_MU ? "mu" : "hals"; }

int parse_cycle(const std::string& s) {
  if (s == "none") return MLNMF_SINGLE_LEVEL;
  if (s == "ni") return MLNMF_NESTED_ITERATION;
  if (s == "vc") return MLNMF_V_CYCLE;
  if (s == "fmg") return MLNMF_FULL_MULTIGRID;
  throw UsageError("--cycle: unknown cycle '" + s + "'");
}
const char* cycle_name(int c) {
  static const char* n[] = {"none", "ni", "vc", "fmg"};
  return n[c];
}

// std::getline-on-',' tokenising (a trailing comma adds no empty token)
std::vector<std::string> commas(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream in(s);
  std::string t;
  while (std::getline(in, t, ',')) out.push_back(t);
  return out;
}

// --precision -> the solver options of the one-shot calls and sessions
mlnmf_options solver_options(const Args& a) {
  mlnmf_options o;
  mlnmf_default_options(&o);
  o.device = (int)a.u64("device", 0);
  const std::string p = a.str("precision", "fp64");
  if (p == "fp64") {
    o.dtype = MLNMF_F64;
    o.exact = 1;
  } else if (p == "fp64-fast") {
    o.dtype = MLNMF_F64;
    o.exact = 0;
  } else if (p == "fp32") {
    o.dtype = MLNMF_F32;
    o.exact = 0;
  } else {
    throw UsageError("--precision: expected fp64, fp64-fast or fp32");
  }
  return o;
}

// load_dataset (mlnmf_main.cpp:61-78)
Dataset load_dataset(const Args& a) {
  const std::string path = a.str("data", ""), format = a.str("format", "pgm-dir");
  const size_t gh = a.u64("grid-height", 0), gw = a.u64("grid-width", 0);
  Dataset d;
  if (format == "pgm-dir")
    d = mlb::io::load_pgm_dir(path);
  else if (format == "csv")
    d = mlb::io::load_csv(path);
  else
    throw UsageError("--format: expected pgm-dir or csv");
  if (gh > 0 && gw > 0) {
    if (gh * gw != d.M.rows) throw DataError("grid dimensions do not match matrix rows");
    d.has_grid = true;
    d.grid = mlb::io::Grid{gh, gw};
  }
  return d;
}

const std::vector<Spec> kData = {{"data", true},         {"format", false},    {"grid-height", false, true},
                                 {"grid-width", false, true}, {"precision", false}, {"device", false, true}};

std::vector<Spec> with(std::vector<Spec> base, const std::vector<Spec>& more) {
  base.insert(base.end(), more.begin(), more.end());
  return base;
}

void usage(FILE* f) {
  std::fprintf(f,
               "Multilevel-accelerated nonnegative matrix factorization (B200)\n"
               "Usage: mlnmf_b200 SUBCOMMAND [OPTIONS]\n\n"
               "Subcommands:\n"
               "  factorize       Run one factorization\n"
               "    --data PATH --rank R --budget work:U|time:S --out PREFIX [--format pgm-dir|csv]\n"
               "    [--algo mu|hals|anls] [--cycle none|ni|vc|fmg] [--levels L] [--seed S]\n"
               "    [--trace-every K] [--grid-height H --grid-width W]\n"
               "  bench           Multi-seed benchmark grid\n"
               "    --data PATH --rank R --budget SPEC --out PREFIX [--algos a,b] [--cycles c,d]\n"
               "    [--levels l1,l2] [--runs N] [--seed S] [--workers W]\n"
               "  transfer-check  Pyramid diagnostics  --data PATH [--levels L]\n"
               "  synth           Write a synthetic PGM dataset  --out DIR [--height H] [--width W]\n"
               "                  [--n N] [--blobs B] [--seed S]\n\n"
               "B200 options: --precision fp64|fp64-fast|fp32 (default fp64: bit-identical to the\n"
               "reference CPU solver), --device K\n");
}

// ---------------------------------------------------------------------------
// subcommands
// ---------------------------------------------------------------------------
int cmd_factorize(const Args& a) {
  const Dataset d = load_dataset(a);
  const int cycle = parse_cycle(a.str("cycle", "none"));
  const size_t levels = a.u64("levels", 1), rank = a.u64("rank", 1), trace_every = a.u64("trace-every", 1);
  if (cycle != MLNMF_SINGLE_LEVEL && levels > 1 && !d.has_grid)
    throw UsageError("--levels: multilevel cycles need a pixel grid");
  const mlb::io::Grid grid = d.has_grid ? d.grid : mlb::io::Grid{d.M.rows, 1};
  const int algo = parse_algo(a.str("algo", "mu"));
  const BudgetSpec b = parse_budget(a.str("budget", ""));
  const uint64_t seed = a.u64("seed", 0);
  const std::string out = a.str("out", "");
  const mlnmf_options o = solver_options(a);
  ck(mlnmf_set_default_options(&o));

  const size_t m = d.M.rows, n = d.M.cols;
  // an out-of-range rank is rejected inside the call (random_init's
  // invalid_argument) before the factor buffers are touched
  const bool rank_ok = rank >= 1 && rank <= std::min(m, n);
  std::vector<double> V(rank_ok ? m * rank : 1), W(rank_ok ? rank * n : 1);
  mlnmf_trace* tr = nullptr;
  ck(mlnmf_run_configuration(d.M.v.data(), m, n, grid.h, grid.w, levels, algo, cycle, rank, seed, b.mode, b.amount,
                             trace_every, V.data(), W.data(), &tr));
  std::unique_ptr<mlnmf_trace, void (*)(mlnmf_trace*)> guard(tr, mlnmf_trace_free);
  const size_t ns = mlnmf_trace_num_samples(tr);
  std::vector<double> el(ns), wu(ns), er(ns);
  std::vector<int> lv(ns);
  mlnmf_trace_samples(tr, el.data(), wu.data(), lv.data(), er.data());
  std::vector<mlb::io::Sample> samples(ns);
  for (size_t i = 0; i < ns; ++i) samples[i] = {el[i], wu[i], lv[i], er[i]};

  mlb::io::save_trace_csv(samples, out + ".trace.csv");
  mlb::io::save_matrix_csv(V.data(), m, rank, out + ".V.csv");
  mlb::io::save_matrix_csv(W.data(), rank, n, out + ".W.csv");
  if (d.has_grid) mlb::io::save_basis_mosaic(V.data(), m, rank, d.grid, out + ".basis");
  std::printf("final error %.10g (%zu trace samples) -> %s.*\n", ns ? er[ns - 1] : 0.0, ns, out.c_str());
  return 0;
}

int cmd_bench(const Args& a) {
  const Dataset d = load_dataset(a);
  std::vector<int> algos, cycles;
  std::vector<size_t> level_counts;
  for (const std::string& s : commas(a.str("algos", "mu"))) algos.push_back(parse_algo(s));
  for (const std::string& s : commas(a.str("cycles", "none"))) cycles.push_back(parse_cycle(s));
  for (const std::string& s : commas(a.str("levels", "1"))) level_counts.push_back(std::stoul(s));
  const size_t rank = a.u64("rank", 1), runs = a.u64("runs", 1), workers = a.u64("workers", 0);
  const BudgetSpec b = parse_budget(a.str("budget", ""));
  const uint64_t base_seed = a.u64("seed", 0);
  const std::string out = a.str("out", "");
  const mlnmf_options o = solver_options(a);

  // run_bench (bench.cpp:28-84)
  if (runs < 1) throw std::invalid_argument("run_bench: runs >= 1");
  std::vector<mlb::io::BenchRow> rows;
  for (int algo : algos)
    for (int cycle : cycles)
      for (size_t levels : level_counts) {
        mlb::io::BenchRow e;
        e.algo = algo_name(algo);
        e.cycle = cycle_name(cycle);
        e.levels = levels;
        if (cycle == MLNMF_SINGLE_LEVEL && levels != 1) {
          e.skipped = true;
          e.note = "single-level runs use exactly one level";
        } else if (levels > 1 && !d.has_grid) {
          e.skipped = true;
          e.note = "dataset has no pixel grid";
        } else {
          const mlb::io::Grid grid = d.has_grid ? d.grid : mlb::io::Grid{d.M.rows, 1};
          std::vector<double> errs(runs);
          const int rc = mlnmf_run_seeds(&o, d.M.v.data(), d.M.rows, d.M.cols, grid.h, grid.w, levels, algo, cycle,
                                         rank, base_seed, runs, b.mode, b.amount, workers, errs.data());
          if (rc == MLNMF_ERR_INVALID) {
            e.skipped = true;
            e.note = mlnmf_last_error();
          } else {
            ck(rc);
            mlb::io::summarise(e, errs);
          }
        }
        rows.push_back(e);
      }
  mlb::io::save_summary_csv(rows, out + ".summary.csv");
  mlb::io::save_summary_txt(rows, out + ".summary.txt");
  std::ifstream txt(out + ".summary.txt");
  std::cout << txt.rdbuf();
  return 0;
}

int cmd_transfer_check(const Args& a) {
  const Dataset d = load_dataset(a);
  if (!d.has_grid) throw DataError("transfer-check needs a pixel grid");
  const size_t levels = a.u64("levels", 1);
  // GridHierarchy::build's checks (transfer.cpp:155-174), before any output
  if (levels < 1) throw std::invalid_argument("GridHierarchy: need at least one level");
  std::vector<mlb::io::Grid> g{d.grid};
  for (size_t l = 1; l < levels; ++l) {
    if (g.back().h < 2 || g.back().w < 2) throw std::invalid_argument("GridHierarchy: too many levels for this grid");
    g.push_back(mlb::io::Grid{(g.back().h + 1) / 2, (g.back().w + 1) / 2});
  }
  if (levels < 2) return 0;
  mlnmf_options o = solver_options(a);
  mlnmf_session* s = nullptr;
  ck(mlnmf_session_create(&o, &s));
  std::unique_ptr<mlnmf_session, void (*)(mlnmf_session*)> guard(s, mlnmf_session_destroy);
  ck(mlnmf_session_set_data(s, d.M.v.data(), MLNMF_F64, d.M.rows, d.M.cols, d.M.cols, 0, d.grid.h, d.grid.w));
  // TransferOperator::row_sum (transfer.cpp:35-39): weights in entry order
  auto max_dev = [](const mlb::HostCsr& op) {
    double dev = 0.0;
    for (size_t i = 0; i + 1 < op.rowptr.size(); ++i) {
      double sum = 0.0;
      for (int e = op.rowptr[i]; e < op.rowptr[i + 1]; ++e) sum += op.wt[e];
      dev = std::max(dev, std::abs(sum - 1.0));
    }
    return dev;
  };
  for (size_t l = 0; l + 1 < levels; ++l) {
    double s_M = 0.0;
    ck(mlnmf_session_smoothness(s, l, &s_M));
    const double dr = max_dev(mlb::build_restriction(g[l].h, g[l].w));
    const double dp = max_dev(mlb::build_prolongation(g[l].h, g[l].w));
    std::printf("level %zu (%zux%zu -> %zux%zu): s_M = %.6g, max |row sum - 1|: R %.3g, P %.3g\n", l + 1, g[l].h,
                g[l].w, g[l + 1].h, g[l + 1].w, s_M, dr, dp);
  }
  return 0;
}

int cmd_synth(const Args& a) {
  const size_t h = a.u64("height", 65), w = a.u64("width", 65), n = a.u64("n", 40), blobs = a.u64("blobs", 3);
  const uint64_t seed = a.u64("seed", 0);
  const std::string out = a.str("out", "");
  const Dataset d = mlb::io::synth_smooth_dataset(h, w, n, blobs, seed);
  mlb::io::save_dataset_pgm_dir(d, out);
  std::printf("wrote %zu images (%zux%zu) to %s\n", d.M.cols, h, w, out.c_str());
  return 0;
}

int run(int argc, char** argv) {
  if (argc < 2) throw UsageError("A subcommand is required");
  const std::string cmd = argv[1];
  if (cmd == "--help" || cmd == "-h") {
    usage(stdout);
    return 0;
  }
  const std::vector<Spec> fac = with(kData, {{"algo", false}, {"cycle", false}, {"levels", false, true},
                                             {"rank", true, true}, {"budget", true}, {"seed", false, true},
                                             {"trace-every", false, true}, {"out", true}});
  const std::vector<Spec> bench = with(kData, {{"algos", false}, {"cycles", false}, {"levels", false},
                                               {"rank", true, true}, {"runs", false, true}, {"budget", true},
                                               {"seed", false, true}, {"out", true}, {"workers", false, true}});
  const std::vector<Spec> tc = with(kData, {{"levels", false, true}});
  const std::vector<Spec> syn = {{"height", false, true}, {"width", false, true}, {"n", false, true},
                                 {"blobs", false, true},  {"seed", false, true},  {"out", true}};
  const std::vector<Spec>* specs = cmd == "factorize"        ? &fac
                                   : cmd == "bench"          ? &bench
                                   : cmd == "transfer-check" ? &tc
                                   : cmd == "synth"          ? &syn
                                                             : nullptr;
  if (!specs) throw UsageError("The following argument was not expected: " + cmd);
  const Args a(argc, argv, 2, cmd, *specs);
  if (a.help()) {
    usage(stdout);
    return 0;
  }
  if (cmd == "factorize") return cmd_factorize(a);
  if (cmd == "bench") return cmd_bench(a);
  if (cmd == "transfer-check") return cmd_transfer_check(a);
  return cmd_synth(a);
}

}  // namespace

// main (mlnmf_main.cpp:221-233): the exception class picks the exit code
int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\n";
    return 2;
  } catch (const NnlsCapExceeded& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return 4;
  } catch (const DataError& e) {
    std::cerr << "data error: " << e.what() << "\n";
    return 3;
  } catch (const std::invalid_argument& e) {
    std::cerr << "invalid arguments: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
