// host_io.cpp -- see host_io.hpp.  Each function cites the reference function
// whose observable behaviour (bytes written, values read, error texts) it
// reproduces.
#include "host_io.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <sstream>

namespace fs = std::filesystem;

namespace mlb {
namespace io {

namespace {

// SplitMix64 (matrix.hpp:76-95): draw c of Rng(seed) is mix(seed + (c+1) gamma).
struct SplitMix {
  uint64_t s;
  uint64_t u64() {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(u64() >> 11) * 0x1.0p-53; }
};

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::ofstream open_out(const std::string& path, std::ios::openmode mode = std::ios::out) {
  std::ofstream f(path, mode);
  if (!f) throw DataError("cannot write " + path);
  return f;
}

// PGM header scanner (io.cpp:24-56): whitespace-separated tokens, '#' starts a
// comment that runs to the end of the line; failures name the byte offset.
class PgmHeader {
 public:
  PgmHeader(const std::string& path, const std::vector<unsigned char>& b) : path_(path), b_(b) {}

  [[noreturn]] void fail(size_t at, const std::string& what) const {
    throw DataError(path_ + ": " + what + " at byte offset " + std::to_string(at));
  }
  size_t pos() const { return p_; }

  std::string token() {
    for (;;) {
      if (p_ >= b_.size()) fail(p_, "unexpected end of header");
      const unsigned char c = b_[p_];
      if (c == '#') {
        while (p_ < b_.size() && b_[p_] != '\n') ++p_;
      } else if (std::isspace(c)) {
        ++p_;
      } else {
        break;
      }
    }
    const size_t t0 = p_;
    while (p_ < b_.size() && !std::isspace(b_[p_]) && b_[p_] != '#') ++p_;
    return std::string(b_.begin() + t0, b_.begin() + p_);
  }

  // unsigned decimal (wrapping like size_t arithmetic); `at` is the offset
  // reported on failure: where the scan for this token started
  size_t count(size_t at) {
    const std::string t = token();
    size_t v = 0;
    for (char c : t) {
      if (c < '0' || c > '9') fail(at, "expected integer, got '" + t + "'");
      v = v * 10 + (size_t)(c - '0');
    }
    return v;
  }

 private:
  const std::string& path_;
  const std::vector<unsigned char>& b_;
  size_t p_ = 0;
};

std::vector<unsigned char> slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw DataError("cannot open " + path);
  return std::vector<unsigned char>(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

bool starts_p5(const fs::path& p) {
  std::ifstream f(p, std::ios::binary);
  char m[2] = {0, 0};
  f.read(m, 2);
  return m[0] == 'P' && m[1] == '5';
}

// column k of V scaled so its maximum is 1; an all-zero column stays zero
// (io.cpp:242-252)
std::vector<double> unit_column(const double* V, size_t m, size_t r, size_t k) {
  double top = 0.0;
  for (size_t i = 0; i < m; ++i) top = std::max(top, V[i * r + k]);
  const double s = top > 0.0 ? 1.0 / top : 0.0;
  std::vector<double> c(m);
  for (size_t i = 0; i < m; ++i) c[i] = V[i * r + k] * s;
  return c;
}

}  // namespace

// load_pgm (io.cpp:65-100)
PgmImage load_pgm(const std::string& path) {
  const std::vector<unsigned char> bytes = slurp(path);
  PgmHeader hdr(path, bytes);
  if (hdr.token() != "P5") hdr.fail(0, "not a binary PGM (missing P5 magic)");
  size_t at = hdr.pos();
  const size_t width = hdr.count(at);
  at = hdr.pos();
  const size_t height = hdr.count(at);
  at = hdr.pos();
  const size_t maxval = hdr.count(at);
  if (width == 0 || height == 0) hdr.fail(at, "zero image dimension");
  if (maxval != 255 && maxval != 65535) hdr.fail(at, "unsupported maxval " + std::to_string(maxval));
  size_t p = hdr.pos();
  if (p >= bytes.size() || !std::isspace(bytes[p])) hdr.fail(p, "missing whitespace after maxval");
  ++p;
  const size_t bpp = maxval == 255 ? 1 : 2;
  const size_t need = width * height * bpp;
  if (bytes.size() - p < need) hdr.fail(p, "truncated pixel data (need " + std::to_string(need) + " bytes)");
  PgmImage img;
  img.grid = Grid{height, width};
  img.pixels.assign(width * height, 0.0);
  const double scale = 1.0 / (double)maxval;
  const unsigned char* px = bytes.data() + p;
  for (size_t i = 0; i < height; ++i)  // file rows are image rows, pixels left to right
    for (size_t j = 0; j < width; ++j) {
      const unsigned char* q = px + (i * width + j) * bpp;
      const size_t raw = bpp == 1 ? q[0] : ((size_t)q[0] << 8) | q[1];  // 16-bit: big-endian
      img.pixels[img.grid.at(i, j)] = (double)raw * scale;
    }
  return img;
}

// save_pgm (io.cpp:102-116): 8-bit P5, values clamped to [0,1], rounded.
void save_pgm(const std::string& path, const Grid& g, const double* pixels, size_t count) {
  if (count != g.pixels()) throw std::invalid_argument("save_pgm: pixel count does not match grid");
  std::ofstream f = open_out(path, std::ios::out | std::ios::binary);
  std::string buf = "P5\n" + std::to_string(g.w) + " " + std::to_string(g.h) + "\n255\n";
  buf.reserve(buf.size() + count);
  for (size_t i = 0; i < g.h; ++i)
    for (size_t j = 0; j < g.w; ++j) {
      const double v = std::clamp(pixels[g.at(i, j)], 0.0, 1.0);
      buf.push_back((char)std::lround(v * 255.0));
    }
  f.write(buf.data(), (std::streamsize)buf.size());
  if (!f) throw DataError("write failed for " + path);
}

// load_pgm_dir (io.cpp:118-144): every regular file starting with "P5", in
// byte-wise filename order, one column each; all the same size.
Dataset load_pgm_dir(const std::string& dir) {
  const fs::path d(dir);
  if (!fs::is_directory(d)) throw DataError(d.string() + " is not a directory");
  std::vector<fs::path> files;
  for (const fs::directory_entry& e : fs::directory_iterator(d))
    if (e.is_regular_file() && starts_p5(e.path())) files.push_back(e.path());
  if (files.empty()) throw DataError(d.string() + ": no P5 images found");
  std::sort(files.begin(), files.end(),
            [](const fs::path& a, const fs::path& b) { return a.filename().string() < b.filename().string(); });
  Dataset out;
  PgmImage img = load_pgm(files[0].string());
  const Grid g = img.grid;
  out.M.rows = g.pixels();
  out.M.cols = files.size();
  out.M.v.assign(out.M.rows * out.M.cols, 0.0);
  for (size_t c = 0; c < files.size(); ++c) {
    if (c > 0) img = load_pgm(files[c].string());
    if (img.grid.h != g.h || img.grid.w != g.w)
      throw DataError(files[c].string() + ": image dimensions differ from " + files[0].string());
    for (size_t i = 0; i < img.pixels.size(); ++i) out.M(i, c) = img.pixels[i];
  }
  out.has_grid = true;
  out.grid = g;
  out.name = d.filename().string();
  return out;
}

// load_csv (io.cpp:146-187)
Dataset load_csv(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw DataError("cannot open " + path);
  std::vector<double> vals;
  size_t ncols = 0, row = 0;
  std::string line;
  auto where = [&](size_t col) { return " at row " + std::to_string(row) + " col " + std::to_string(col); };
  while (std::getline(f, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    ++row;
    size_t col = 0;
    std::istringstream cells(line);
    std::string cell;
    while (std::getline(cells, cell, ',')) {
      ++col;
      double v = 0.0;
      size_t used = 0;
      bool ok = true;
      try {
        v = std::stod(cell, &used);
      } catch (const std::exception&) {
        ok = false;
      }
      if (!ok || used != cell.size() || !std::isfinite(v)) throw DataError(path + ": unparsable value" + where(col));
      if (v < 0.0) throw DataError(path + ": negative entry" + where(col));
      vals.push_back(v);
    }
    if (ncols == 0) ncols = col;
    if (col != ncols)
      throw DataError(path + ": ragged row " + std::to_string(row) + " (" + std::to_string(col) +
                      " values, expected " + std::to_string(ncols) + ")");
  }
  if (vals.empty()) throw DataError(path + ": empty matrix");
  Dataset out;
  out.M.cols = ncols;
  out.M.rows = vals.size() / ncols;
  out.M.v = std::move(vals);
  out.name = fs::path(path).stem().string();
  return out;
}

// save_matrix_csv (io.cpp:189-199): row per line, %.17g, comma-separated.
void save_matrix_csv(const double* a, size_t rows, size_t cols, const std::string& path) {
  std::ofstream f = open_out(path);
  std::string line;
  for (size_t i = 0; i < rows; ++i) {
    line.clear();
    for (size_t j = 0; j < cols; ++j) {
      if (j) line += ',';
      line += g17(a[i * cols + j]);
    }
    line += '\n';
    f << line;
  }
}

// save_trace_csv (io.cpp:201-209)
void save_trace_csv(const std::vector<Sample>& s, const std::string& path) {
  std::ofstream f = open_out(path);
  f << "elapsed_s,work_units,level,error\n";
  for (const Sample& x : s)
    f << g17(x.elapsed_s) << ',' << g17(x.work_units) << ',' << x.level << ',' << g17(x.error) << '\n';
  if (!f) throw DataError("write failed for " + path);
}

// save_basis_mosaic (io.cpp:255-283): basis_kkk.pgm per column plus a
// ceil(sqrt(r))-wide tiling of them, row by row, in mosaic.pgm.
void save_basis_mosaic(const double* V, size_t m, size_t r, const Grid& g, const std::string& dir) {
  if (m != g.pixels()) throw std::invalid_argument("save_basis_mosaic: grid does not match V");
  const fs::path d(dir);
  fs::create_directories(d);
  const size_t across = (size_t)std::ceil(std::sqrt((double)r));
  const size_t down = (r + across - 1) / across;
  const Grid mg{down * g.h, across * g.w};
  std::vector<double> mosaic(mg.pixels(), 0.0);
  for (size_t k = 0; k < r; ++k) {
    const std::vector<double> c = unit_column(V, m, r, k);
    char name[32];
    std::snprintf(name, sizeof name, "basis_%03zu.pgm", k);
    save_pgm((d / name).string(), g, c.data(), c.size());
    const size_t oi = (k / across) * g.h, oj = (k % across) * g.w;
    for (size_t j = 0; j < g.w; ++j)
      for (size_t i = 0; i < g.h; ++i) mosaic[mg.at(oi + i, oj + j)] = c[g.at(i, j)];
  }
  save_pgm((d / "mosaic.pgm").string(), mg, mosaic.data(), mosaic.size());
}

// synth_smooth_dataset (io.cpp:311-352): a pool of 2*blobs Gaussian
// prototypes (centre uniform, sigma in [h/8, h/3]); every image sums `blobs`
// draws from the pool with jittered centres (+-h/48, +-w/48) and amplitudes
// in [0.2, 1], clipped at 1.  One generator, draws in exactly this order.
Dataset synth_smooth_dataset(size_t h, size_t w, size_t n, size_t blobs, uint64_t seed) {
  if (blobs < 1) throw std::invalid_argument("synth_smooth_dataset: blobs >= 1");
  const Grid g{h, w};
  const double fh = (double)h, fw = (double)w;
  SplitMix rng{seed};
  struct Proto {
    double ci, cj, sigma;
  };
  std::vector<Proto> pool(2 * blobs);
  for (Proto& p : pool) {
    p.ci = rng.uniform() * fh;
    p.cj = rng.uniform() * fw;
    p.sigma = fh / 8.0 + rng.uniform() * (fh / 3.0 - fh / 8.0);
  }
  Dataset out;
  out.M.rows = g.pixels();
  out.M.cols = n;
  out.M.v.assign(out.M.rows * n, 0.0);
  std::vector<double> acc(g.pixels());
  for (size_t c = 0; c < n; ++c) {
    std::fill(acc.begin(), acc.end(), 0.0);
    for (size_t b = 0; b < blobs; ++b) {
      const Proto& p = pool[rng.u64() % pool.size()];
      const double ci = p.ci + (rng.uniform() - 0.5) * fh / 24.0;
      const double cj = p.cj + (rng.uniform() - 0.5) * fw / 24.0;
      const double amp = 0.2 + rng.uniform() * 0.8;
      const double k = 1.0 / (2.0 * p.sigma * p.sigma);
      for (size_t i = 0; i < h; ++i) {
        const double di = (double)i - ci;
        for (size_t j = 0; j < w; ++j) {
          const double dj = (double)j - cj;
          acc[g.at(i, j)] += amp * std::exp(-(di * di + dj * dj) * k);
        }
      }
    }
    for (size_t i = 0; i < acc.size(); ++i) out.M(i, c) = std::min(1.0, acc[i]);
  }
  out.has_grid = true;
  out.grid = g;
  out.name = "synth";
  return out;
}

// save_dataset_pgm_dir (io.cpp:354-366): img_NNNN.pgm per column.
void save_dataset_pgm_dir(const Dataset& d, const std::string& dir) {
  if (!d.has_grid) throw std::invalid_argument("save_dataset_pgm_dir: dataset has no grid");
  const fs::path p(dir);
  fs::create_directories(p);
  std::vector<double> col(d.M.rows);
  for (size_t c = 0; c < d.M.cols; ++c) {
    for (size_t i = 0; i < d.M.rows; ++i) col[i] = d.M(i, c);
    char name[32];
    std::snprintf(name, sizeof name, "img_%04zu.pgm", c);
    save_pgm((p / name).string(), d.grid, col.data(), col.size());
  }
}

// bench.cpp:64-80
void summarise(BenchRow& e, const std::vector<double>& errors) {
  const size_t n = errors.size();
  double sum = 0.0, lo = errors[0], hi = errors[0];
  for (double x : errors) {
    sum += x;
    lo = std::min(lo, x);
    hi = std::max(hi, x);
  }
  e.runs = n;
  e.mean = sum / (double)n;
  double ss = 0.0;
  for (double x : errors) ss += (x - e.mean) * (x - e.mean);
  e.stddev = n > 1 ? std::sqrt(ss / (double)(n - 1)) : 0.0;
  e.min = lo;
  e.max = hi;
}

// save_summary_csv (bench.cpp:86-103)
void save_summary_csv(const std::vector<BenchRow>& rows, const std::string& path) {
  std::ofstream f = open_out(path);
  f << "algorithm,cycle,levels,runs,mean_error,std_error,min_error,max_error,note\n";
  char line[256];  // the reference formats each row into 256 bytes
  for (const BenchRow& e : rows) {
    if (e.skipped) {
      f << e.algo << ',' << e.cycle << ',' << e.levels << ",0,,,,," << e.note << '\n';
    } else {
      std::snprintf(line, sizeof line, "%s,%s,%zu,%zu,%.17g,%.17g,%.17g,%.17g,\n", e.algo.c_str(), e.cycle.c_str(),
                    e.levels, e.runs, e.mean, e.stddev, e.min, e.max);
      f << line;
    }
  }
}

// save_summary_txt (bench.cpp:105-125)
void save_summary_txt(const std::vector<BenchRow>& rows, const std::string& path) {
  std::ofstream f = open_out(path);
  f << "Mean final error ||M - VW||_F per configuration\n";
  char line[256];
  std::snprintf(line, sizeof line, "%-6s %-5s %-6s %-6s %-14s %-14s %-14s %-14s\n", "algo", "cycle", "levels", "runs",
                "mean", "std", "min", "max");
  f << line;
  for (const BenchRow& e : rows) {
    if (e.skipped)
      std::snprintf(line, sizeof line, "%-6s %-5s %-6zu skipped: %s\n", e.algo.c_str(), e.cycle.c_str(), e.levels,
                    e.note.c_str());
    else
      std::snprintf(line, sizeof line, "%-6s %-5s %-6zu %-6zu %-14.6g %-14.6g %-14.6g %-14.6g\n", e.algo.c_str(),
                    e.cycle.c_str(), e.levels, e.runs, e.mean, e.stddev, e.min, e.max);
    f << line;
  }
}

}  // namespace io
}  // namespace mlb
