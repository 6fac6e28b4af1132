// Paper-literal POBK preprocessing (Alg 5 steps 2-4) with k uniform row blocks
// -- the NEXT-2 row of SURVEY.md §8(f); the hot path reads blocks as single rows.
//
//   uniform_blocks   blocks 1..k-1 take [m/k] consecutive RCM rows, block k the rest
//   centroid table   A-bar_i = mean of block i's rows; C(i,j) = |G(i,j)| / (||A-bar_i|| ||A-bar_j||),
//                    G(i,j) = (A-bar_i, A-bar_j), diagonal 1 (|.|: SURVEY Z6)
//   classify         C(i,j) < thr counts as orthogonal; scanning i ascending, an unused
//                    block i pairs with the first unused j > i orthogonal to it (class{i}); the
//                    unpaired blocks form Nclass, ascending
//   zn, nn           Definitions 1-2 on the table with entries < thr set to 0
//   gram_inverse     (A_tau A_tau^T)^-1 for every block: with full row rank (a nonsingular A),
//                    A_tau^+ = A_tau^T (A_tau A_tau^T)^-1 (Lemma 1), the block step of
//                    Eq 3.3 as   r = f_tau - A_tau x,  y = G^-1 r,  x += A_tau^T y.
//                    Cholesky G = L L^T, then G^-1 = L^-T L^-1 (dense, one host thread per block).
// Built with -ffp-contract=off; plain left-to-right sums.
#include <algorithm>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "../internal.h"

namespace pobk {

bool block_layout(const HostCSR& At, int32_t k, double thr, BlockLayout& out, Error& err) {
  const int64_t m = At.m;
  if (k < 1 || k > m) {
    err = {POBK_ERR_ARG, "k must be in [1, m] (got " + std::to_string(k) + ")"};
    return false;
  }
  if (!(thr >= 0.0 && thr < 1.0)) {
    err = {POBK_ERR_ARG, "thr must be in [0, 1)"};
    return false;
  }
  out.k = k;
  out.thr = thr;
  out.ptr.assign(k + 1, 0);
  const int64_t q = m / k;
  for (int32_t i = 0; i < k; i++) out.ptr[i] = i * q;
  out.ptr[k] = m;
  // centroids as sparse vectors (ascending columns): sum of the block's rows / block size
  std::vector<std::vector<std::pair<int32_t, double>>> cent(k);
  {
    std::vector<double> acc(m, 0.0);
    std::vector<uint8_t> hit(m, 0);
    std::vector<int32_t> cols;
    for (int32_t b = 0; b < k; b++) {
      cols.clear();
      for (int64_t r = out.ptr[b]; r < out.ptr[b + 1]; r++)
        for (int64_t p = At.ptr[r]; p < At.ptr[r + 1]; p++) {
          const int32_t c = At.col[p];
          if (!hit[c]) { hit[c] = 1; cols.push_back(c); }
          acc[c] = acc[c] + At.val[p];
        }
      std::sort(cols.begin(), cols.end());
      const double nb = (double)(out.ptr[b + 1] - out.ptr[b]);
      cent[b].reserve(cols.size());
      for (int32_t c : cols) {
        cent[b].push_back({c, acc[c] / nb});
        acc[c] = 0.0;
        hit[c] = 0;
      }
    }
  }
  std::vector<double> nrm(k, 0.0);
  for (int32_t b = 0; b < k; b++) {
    double s = 0.0;
    for (auto& e : cent[b]) s = s + e.second * e.second;
    nrm[b] = std::sqrt(s);
    if (!(nrm[b] > 0.0)) {
      err = {POBK_ERR_ARG, "block " + std::to_string(b) + " has a zero centroid (cosine undefined)"};
      return false;
    }
  }
  out.cos.assign((size_t)k * k, 0.0);
  for (int32_t i = 0; i < k; i++) {
    out.cos[(size_t)i * k + i] = 1.0;
    for (int32_t j = i + 1; j < k; j++) {
      double g = 0.0;  // sorted merge of the two sparse centroids, ascending columns
      size_t a = 0, b = 0;
      const auto &ci = cent[i], &cj = cent[j];
      while (a < ci.size() && b < cj.size()) {
        if (ci[a].first < cj[b].first) a++;
        else if (ci[a].first > cj[b].first) b++;
        else { g = g + ci[a].second * cj[b].second; a++; b++; }
      }
      const double c = std::fabs(g) / (nrm[i] * nrm[j]);
      out.cos[(size_t)i * k + j] = out.cos[(size_t)j * k + i] = c;
    }
  }
  // classification
  std::vector<uint8_t> used(k, 0);
  out.pairs.clear();
  out.nclass.clear();
  for (int32_t i = 0; i < k; i++) {
    if (used[i]) continue;
    for (int32_t j = i + 1; j < k; j++)
      if (!used[j] && out.cos[(size_t)i * k + j] < thr) {
        out.pairs.push_back({i, j});
        used[i] = used[j] = 1;
        break;
      }
  }
  for (int32_t i = 0; i < k; i++)
    if (!used[i]) out.nclass.push_back(i);
  out.order.clear();
  for (auto& pr : out.pairs) { out.order.push_back(pr.first); out.order.push_back(pr.second); }
  for (int32_t b : out.nclass) out.order.push_back(b);
  // zn, nn (Definitions 1-2)
  int64_t n1 = 0, n2 = 0;
  double sum = 0.0;
  for (size_t e = 0; e < out.cos.size(); e++) {
    const double c = out.cos[e] < thr ? 0.0 : out.cos[e];
    if (c == 0.0) n1++;
    else { n2++; sum = sum + c; }
  }
  const double kk = (double)k * (double)k;
  out.zn = (double)n1 / kk;
  out.nn = n2 ? (double)n2 * (sum / (double)n2) / kk : 0.0;
  return true;
}

namespace {
// G = A_tau A_tau^T (rows r0..r1 of At), dense b x b row-major: G(i,j) = sum over shared columns in
// ascending column order
void gram(const HostCSR& At, int64_t r0, int64_t r1, std::vector<double>& G) {
  const int64_t b = r1 - r0;
  G.assign((size_t)b * b, 0.0);
  for (int64_t i = 0; i < b; i++)
    for (int64_t j = 0; j <= i; j++) {
      int64_t p = At.ptr[r0 + i], pe = At.ptr[r0 + i + 1], q = At.ptr[r0 + j], qe = At.ptr[r0 + j + 1];
      double s = 0.0;
      while (p < pe && q < qe) {
        if (At.col[p] < At.col[q]) p++;
        else if (At.col[p] > At.col[q]) q++;
        else { s = s + At.val[p] * At.val[q]; p++; q++; }
      }
      G[(size_t)i * b + j] = G[(size_t)j * b + i] = s;
    }
}

// G^-1 for SPD G (b x b): Cholesky G = L L^T, Y = L^-1 (lower), G^-1 = Y^T Y.  false if a pivot is
// not positive (a rank-deficient block: A_tau^+ is then not A_tau^T G^-1).
bool spd_inverse(std::vector<double>& G, int64_t b) {
  std::vector<double>& L = G;  // in place, lower triangle
  for (int64_t j = 0; j < b; j++) {
    double d = L[(size_t)j * b + j];
    for (int64_t t = 0; t < j; t++) d = d - L[(size_t)j * b + t] * L[(size_t)j * b + t];
    if (!(d > 0.0)) return false;
    const double ljj = std::sqrt(d);
    L[(size_t)j * b + j] = ljj;
    for (int64_t i = j + 1; i < b; i++) {
      double s = L[(size_t)i * b + j];
      const double* li = &L[(size_t)i * b];
      const double* lj = &L[(size_t)j * b];
      for (int64_t t = 0; t < j; t++) s = s - li[t] * lj[t];
      L[(size_t)i * b + j] = s / ljj;
    }
  }
  // Yt = (L^-1)^T, upper triangular, stored row-major: row i of Yt = column i of Y.  Column i of Y
  // solves L y = e_i (forward substitution, y_t = 0 for t < i).
  std::vector<double> Yt((size_t)b * b, 0.0);
  std::vector<double> y(b);
  for (int64_t i = 0; i < b; i++) {
    for (int64_t t = 0; t < i; t++) y[t] = 0.0;
    for (int64_t r = i; r < b; r++) {
      double s = r == i ? 1.0 : 0.0;
      const double* lr = &L[(size_t)r * b];
      for (int64_t t = i; t < r; t++) s = s - lr[t] * y[t];
      y[r] = s / lr[r];
    }
    for (int64_t r = i; r < b; r++) Yt[(size_t)i * b + r] = y[r];
  }
  // G^-1(i,j) = sum_{t >= max(i,j)} Y(t,i) Y(t,j) = sum_t Yt(i,t) Yt(j,t)
  for (int64_t i = 0; i < b; i++)
    for (int64_t j = 0; j <= i; j++) {
      const double* a = &Yt[(size_t)i * b];
      const double* c = &Yt[(size_t)j * b];
      double s = 0.0;
      for (int64_t t = i; t < b; t++) s = s + a[t] * c[t];
      G[(size_t)i * b + j] = G[(size_t)j * b + i] = s;
    }
  return true;
}
}  // namespace

bool block_gram_inverses(const HostCSR& At, const BlockLayout& L, std::vector<std::vector<double>>& ginv, Error& err) {
  const int32_t k = L.k;
  ginv.assign(k, {});
  std::vector<int> ok(k, 1);
  const unsigned nth = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), (unsigned)k));
  std::vector<std::thread> th;
  for (unsigned w = 0; w < nth; w++)
    th.emplace_back([&, w]() {
      for (int32_t b = (int32_t)w; b < k; b += (int32_t)nth) {
        gram(At, L.ptr[b], L.ptr[b + 1], ginv[b]);
        ok[b] = spd_inverse(ginv[b], L.ptr[b + 1] - L.ptr[b]);
      }
    });
  for (auto& t : th) t.join();
  for (int32_t b = 0; b < k; b++)
    if (!ok[b]) {
      err = {POBK_ERR_ARG, "block " + std::to_string(b) + " is rank-deficient (A_tau A_tau^T not positive definite): "
                           "the k-block path needs full-row-rank blocks"};
      return false;
    }
  return true;
}

}  // namespace pobk
