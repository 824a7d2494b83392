// transfer_ops.hpp -- host construction of the pyramid transfer operators as
// CSR (uploaded once per level; applied by k_csr_apply on the device).
//
// Restates proj/src/transfer.cpp: coarsen_grid (:55-59), build_restriction
// (:61-85, 9-point [1 2 1]x[1 2 1]/16 full weighting, out-of-range entries
// dropped and the row renormalised, entries in (di, dj) row-major order) and
// build_prolongation (:89-118, mean over rd(i/2) x rd(j/2) clipped to the coarse
// grid).  Pixel (i, j) of an h x w image is row j*h + i (transfer.hpp:15-20).
#pragma once
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace mlb {

struct HostCsr {
  std::vector<int> rowptr, idx;
  std::vector<double> wt;
};

inline void coarsen_grid(size_t h, size_t w, size_t* hc, size_t* wc) {
  if (h < 2 || w < 2) throw std::invalid_argument("coarsen_grid: grid below 2x2 cannot be coarsened");
  *hc = (h + 1) / 2;
  *wc = (w + 1) / 2;
}

inline HostCsr build_restriction(size_t h, size_t w) {
  size_t hc, wc;
  coarsen_grid(h, w, &hc, &wc);
  HostCsr op;
  op.rowptr.assign(hc * wc + 1, 0);
  for (size_t cj = 0; cj < wc; ++cj)
    for (size_t ci = 0; ci < hc; ++ci) {
      const size_t row = cj * hc + ci;
      op.rowptr[row] = (int)op.idx.size();
      const long fi = 2 * (long)ci, fj = 2 * (long)cj;
      const size_t b = op.wt.size();
      for (long di = -1; di <= 1; ++di)
        for (long dj = -1; dj <= 1; ++dj) {
          const long i = fi + di, j = fj + dj;
          if (i < 0 || j < 0 || i >= (long)h || j >= (long)w) continue;
          const double wgt = (di == 0 && dj == 0) ? 4.0 : (di == 0 || dj == 0) ? 2.0 : 1.0;
          op.idx.push_back((int)((size_t)j * h + (size_t)i));
          op.wt.push_back(wgt / 16.0);
        }
      double s = 0.0;  // TransferOperator::normalize_row (transfer.cpp:9-15)
      for (size_t e = b; e < op.wt.size(); ++e) s += op.wt[e];
      if (s <= 0.0) throw std::invalid_argument("TransferOperator: empty or zero row");
      for (size_t e = b; e < op.wt.size(); ++e) op.wt[e] /= s;
    }
  op.rowptr[hc * wc] = (int)op.idx.size();
  return op;
}

inline void rd_half(size_t k, size_t limit, size_t out[2], size_t& count) {
  count = 0;
  if (k % 2 == 0) {
    if (k / 2 < limit) out[count++] = k / 2;
  } else {
    if ((k - 1) / 2 < limit) out[count++] = (k - 1) / 2;
    if ((k + 1) / 2 < limit) out[count++] = (k + 1) / 2;
  }
}

inline HostCsr build_prolongation(size_t h, size_t w) {
  size_t hc, wc;
  coarsen_grid(h, w, &hc, &wc);
  HostCsr op;
  op.rowptr.assign(h * w + 1, 0);
  for (size_t j = 0; j < w; ++j) {
    size_t js[2], jn;
    rd_half(j, wc, js, jn);
    for (size_t i = 0; i < h; ++i) {
      size_t is[2], in;
      rd_half(i, hc, is, in);
      const size_t row = j * h + i;
      op.rowptr[row] = (int)op.idx.size();
      const double wgt = 1.0 / (double)(in * jn);
      for (size_t a = 0; a < in; ++a)
        for (size_t b = 0; b < jn; ++b) {
          op.idx.push_back((int)(js[b] * hc + is[a]));
          op.wt.push_back(wgt);
        }
    }
  }
  op.rowptr[h * w] = (int)op.idx.size();
  return op;
}

}  // namespace mlb
