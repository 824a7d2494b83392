// host_io.hpp -- dataset ingestion and result writers of the mlnmf_b200 CLI.
//
// Host-side only (no CUDA): the formats the reference CLI reads and writes
// (proj/include/mlnmf/io.hpp, proj/include/mlnmf/bench.hpp), restated so that
// a `mlnmf factorize|bench|transfer-check|synth` user gets byte-identical files
// from `mlnmf_b200`:
//   * binary PGM (P5, maxval 255 / 65535) images, a directory of them as the
//     columns of M (io.cpp:65-144), rectangular nonnegative CSV (io.cpp:146-187);
//   * matrix and trace CSV at %.17g (io.cpp:189-209), basis PGMs + mosaic
//     (io.cpp:255-283), bench summaries (bench.cpp:86-127);
//   * the seeded synthetic PGM image set of `mlnmf synth` (io.cpp:311-352).
// Errors follow the reference: DataError for unreadable / malformed input,
// std::invalid_argument for caller mistakes; the message texts are the
// reference's, so the CLI's stderr lines and exit codes match.
#pragma once
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mlb {
namespace io {

// mlnmf::DataError (io.hpp / solvers.hpp): exit code 3 in the CLI.
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Column-major pixel grid (transfer.hpp:13-21): pixel (i, j) is row j*h + i.
struct Grid {
  size_t h = 0, w = 0;
  size_t pixels() const { return h * w; }
  size_t at(size_t i, size_t j) const { return j * h + i; }
};

// Row-major m x n fp64 matrix (matrix.hpp:28-72), one column per image.
struct Dense {
  size_t rows = 0, cols = 0;
  std::vector<double> v;
  double& operator()(size_t i, size_t j) { return v[i * cols + j]; }
  double operator()(size_t i, size_t j) const { return v[i * cols + j]; }
};

struct Dataset {
  Dense M;
  bool has_grid = false;
  Grid grid;
  std::string name;
};

// One trace sample (solvers.hpp:14-19).
struct Sample {
  double elapsed_s, work_units;
  int level;
  double error;
};

struct PgmImage {
  Grid grid;
  std::vector<double> pixels;  // column-vectorised, scaled to [0, 1]
};

PgmImage load_pgm(const std::string& path);
void save_pgm(const std::string& path, const Grid& g, const double* pixels, size_t count);
Dataset load_pgm_dir(const std::string& dir);
Dataset load_csv(const std::string& path);

void save_matrix_csv(const double* a, size_t rows, size_t cols, const std::string& path);
void save_trace_csv(const std::vector<Sample>& s, const std::string& path);
void save_basis_mosaic(const double* V, size_t m, size_t r, const Grid& g, const std::string& dir);

Dataset synth_smooth_dataset(size_t h, size_t w, size_t n, size_t blobs, uint64_t seed);
void save_dataset_pgm_dir(const Dataset& d, const std::string& dir);

// BenchEntry (bench.hpp:25-36) and the two summary writers.
struct BenchRow {
  std::string algo, cycle;
  size_t levels = 0, runs = 0;
  double mean = 0, stddev = 0, min = 0, max = 0;
  bool skipped = false;
  std::string note;
};
// mean / sample stddev / min / max of final errors, summed in run order
// (bench.cpp:64-80)
void summarise(BenchRow& e, const std::vector<double>& errors);
void save_summary_csv(const std::vector<BenchRow>& rows, const std::string& path);
void save_summary_txt(const std::vector<BenchRow>& rows, const std::string& path);

}  // namespace io
}  // namespace mlb
