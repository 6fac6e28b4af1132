// Host preprocessing for POBK: Alg 5 steps 1-4 at row granularity.
//
//   canonicalize      input contract; explicit zeros dropped
//   rcm_order         Reverse Cuthill-McKee: DESIGN.md §3 R1-R5
//   permute_symmetric A~ = P A P^T (Eq 3.1)
//   first_fit_colour  categories of pairwise-orthogonal rows: DESIGN.md §3 P1-P3
//   build_schedule    Oclass categories ascending, then Nclass rows ascending
//
// Integer outputs must be bit-identical to the oracle's; the only floating-point decisions
// (thr > 0) use plain left-to-right sums with no FMA contraction (built with -ffp-contract=off).
// Written for 10^6-row systems: O(nnz) passes plus per-row sorts; no pointer chasing per edge.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include "../internal.h"

namespace pobk {

bool canonicalize(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val, HostCSR& out,
                  Error& err) {
  if (m < 1 || !row_ptr || (row_ptr[m] > 0 && (!col || !val))) {
    err = {POBK_ERR_ARG, "m must be >= 1 and row_ptr/col/val non-NULL"};
    return false;
  }
  if (row_ptr[0] != 0) {
    err = {POBK_ERR_BAD_CSR, "row_ptr[0] != 0"};
    return false;
  }
  if (row_ptr[m] >= (int64_t(1) << 31)) {
    err = {POBK_ERR_ARG, "nnz >= 2^31 per system is not supported"};
    return false;
  }
  out.m = m;
  out.ptr.assign(m + 1, 0);
  out.col.clear();
  out.val.clear();
  out.col.reserve(row_ptr[m]);
  out.val.reserve(row_ptr[m]);
  for (int64_t i = 0; i < m; i++) {
    int64_t b = row_ptr[i], e = row_ptr[i + 1];
    if (e < b) {
      err = {POBK_ERR_BAD_CSR, "row_ptr decreases at row " + std::to_string(i)};
      return false;
    }
    for (int64_t p = b; p < e; p++) {
      int32_t c = col[p];
      if (c < 0 || c >= m) {
        err = {POBK_ERR_BAD_CSR, "row " + std::to_string(i) + ": column " + std::to_string(c) + " out of range"};
        return false;
      }
      if (p > b && c <= col[p - 1]) {
        err = {POBK_ERR_BAD_CSR, "row " + std::to_string(i) + ": columns not strictly increasing (unsorted or duplicate)"};
        return false;
      }
      if (val[p] != 0.0) {
        out.col.push_back(c);
        out.val.push_back(val[p]);
      }
    }
    out.ptr[i + 1] = (int64_t)out.col.size();
    if (out.ptr[i + 1] == out.ptr[i]) {
      err = {POBK_ERR_ZERO_ROW, "row " + std::to_string(i) + " is zero (||a_i|| = 0, Eq 1.2 undefined)"};
      return false;
    }
  }
  return true;
}

int64_t bandwidth(const HostCSR& A) {
  int64_t bw = 0;
  for (int64_t i = 0; i < A.m; i++)
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; p++) bw = std::max<int64_t>(bw, std::llabs(i - (int64_t)A.col[p]));
  return bw;
}

namespace {

// Undirected graph of pattern(A + A^T) minus the diagonal (DESIGN.md §3 R1), adjacency of each
// vertex sorted by (degree, index) -- the only order the Cuthill-McKee visit ever needs.
struct Graph {
  int64_t n = 0;
  std::vector<int64_t> off;
  std::vector<int32_t> adj;
  std::vector<int32_t> deg;
};

void build_graph(const HostCSR& A, Graph& g) {
  const int64_t n = A.m;
  g.n = n;
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t i = 0; i < n; i++)
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; p++) {
      int32_t j = A.col[p];
      if (j != i) { cnt[i + 1]++; cnt[j + 1]++; }
    }
  for (int64_t i = 0; i < n; i++) cnt[i + 1] += cnt[i];
  std::vector<int32_t> raw(cnt[n]);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < n; i++)
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; p++) {
      int32_t j = A.col[p];
      if (j != i) { raw[fill[i]++] = j; raw[fill[j]++] = (int32_t)i; }
    }
  // dedupe (an edge stored in both triangles arrives twice)
  g.off.assign(n + 1, 0);
  g.deg.assign(n, 0);
  int64_t w = 0;
  for (int64_t i = 0; i < n; i++) {
    int32_t* b = raw.data() + cnt[i];
    int32_t* e = raw.data() + cnt[i + 1];
    std::sort(b, e);
    int32_t* u = std::unique(b, e);
    int64_t d = u - b;
    std::memmove(raw.data() + w, b, d * sizeof(int32_t));
    g.off[i] = w;
    g.deg[i] = (int32_t)d;
    w += d;
  }
  g.off[n] = w;
  raw.resize(w);
  g.adj.swap(raw);
  // order every adjacency by (deg, idx)
  for (int64_t i = 0; i < n; i++) {
    std::sort(g.adj.begin() + g.off[i], g.adj.begin() + g.off[i + 1], [&](int32_t a, int32_t b) {
      return g.deg[a] < g.deg[b] || (g.deg[a] == g.deg[b] && a < b);
    });
  }
}

inline bool deg_idx_less(const Graph& g, int32_t a, int32_t b) {
  return g.deg[a] < g.deg[b] || (g.deg[a] == g.deg[b] && a < b);
}

// BFS level structure from r.  level[] is -1 outside the BFS and is reset before return.
// Returns number of levels; `last_min` = (deg, idx)-minimal vertex of the last level.
int64_t levels_from(const Graph& g, int32_t r, std::vector<int32_t>& level, std::vector<int32_t>& q, int32_t& last_min) {
  int64_t h = 0, t = 0;
  q[t++] = r;
  level[r] = 0;
  while (h < t) {
    int32_t v = q[h++];
    for (int64_t p = g.off[v]; p < g.off[v + 1]; p++) {
      int32_t u = g.adj[p];
      if (level[u] < 0) { level[u] = level[v] + 1; q[t++] = u; }
    }
  }
  const int32_t last = level[q[t - 1]];
  last_min = q[t - 1];
  for (int64_t k = t - 1; k >= 0 && level[q[k]] == last; k--)
    if (deg_idx_less(g, q[k], last_min)) last_min = q[k];
  for (int64_t k = 0; k < t; k++) level[q[k]] = -1;
  return (int64_t)last + 1;
}

}  // namespace

// DESIGN.md §3 R1-R5: components in ascending order of their smallest
// vertex; start r = (deg, idx)-min vertex of the component; George-Liu: up to 10 rounds of
// x = (deg, idx)-min vertex of the last level of L(r), replace r by x while x's level structure
// is strictly deeper; the root is the last candidate x; Cuthill-McKee FIFO visit with neighbours
// in ascending (deg, idx); the whole concatenated order is reversed.
void rcm_order(const HostCSR& A, std::vector<int32_t>& perm) {
  Graph g;
  build_graph(A, g);
  const int64_t n = g.n;
  std::vector<int32_t> level(n, -1), q(n), order;
  order.reserve(n);
  std::vector<uint8_t> placed(n, 0);
  for (int64_t s0 = 0; s0 < n; s0++) {
    if (placed[s0]) continue;
    // component of s0 and its (deg, idx)-minimal vertex
    int64_t h = 0, t = 0;
    q[t++] = (int32_t)s0;
    level[s0] = 0;
    int32_t r = (int32_t)s0;
    while (h < t) {
      int32_t v = q[h++];
      if (deg_idx_less(g, v, r)) r = v;
      for (int64_t p = g.off[v]; p < g.off[v + 1]; p++)
        if (level[g.adj[p]] < 0) { level[g.adj[p]] = 0; q[t++] = g.adj[p]; }
    }
    for (int64_t k = 0; k < t; k++) level[q[k]] = -1;
    int32_t cand;
    int64_t depth_r = levels_from(g, r, level, q, cand);
    int32_t x = r;
    for (int round = 0; round < 10; round++) {
      x = cand;
      int32_t cand_x;
      int64_t depth_x = levels_from(g, x, level, q, cand_x);
      if (depth_x > depth_r) { r = x; depth_r = depth_x; cand = cand_x; }
      else break;
    }
    // Cuthill-McKee from the root x
    h = t = 0;
    q[t++] = x;
    placed[x] = 1;
    while (h < t) {
      int32_t v = q[h++];
      order.push_back(v);
      for (int64_t p = g.off[v]; p < g.off[v + 1]; p++) {
        int32_t u = g.adj[p];
        if (!placed[u]) { placed[u] = 1; q[t++] = u; }
      }
    }
  }
  perm.resize(n);
  for (int64_t i = 0; i < n; i++) perm[i] = order[n - 1 - i];
}

void permute_symmetric(const HostCSR& A, const std::vector<int32_t>& perm, HostCSR& out) {
  const int64_t n = A.m;
  std::vector<int32_t> iperm(n);
  for (int64_t i = 0; i < n; i++) iperm[perm[i]] = (int32_t)i;
  out.m = n;
  out.ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; i++) out.ptr[i + 1] = out.ptr[i] + (A.ptr[perm[i] + 1] - A.ptr[perm[i]]);
  out.col.resize(A.nnz());
  out.val.resize(A.nnz());
  std::vector<std::pair<int32_t, double>> tmp;
  for (int64_t i = 0; i < n; i++) {
    int64_t src = A.ptr[perm[i]], len = A.ptr[perm[i] + 1] - src;
    tmp.resize(len);
    for (int64_t k = 0; k < len; k++) tmp[k] = {iperm[A.col[src + k]], A.val[src + k]};
    std::sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (int64_t k = 0; k < len; k++) {
      out.col[out.ptr[i] + k] = tmp[k].first;
      out.val[out.ptr[i] + k] = tmp[k].second;
    }
  }
}

void row_sqnorms(const HostCSR& A, std::vector<double>& nrm2) {
  nrm2.assign(A.m, 0.0);
  for (int64_t i = 0; i < A.m; i++) {
    double s = 0.0;
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; p++) s = s + A.val[p] * A.val[p];
    nrm2[i] = s;
  }
}

namespace {
// rows of each column, ascending (CSC of the pattern)
void column_rows(const HostCSR& A, std::vector<int64_t>& cptr, std::vector<int32_t>& crow) {
  const int64_t n = A.m;
  cptr.assign(n + 1, 0);
  for (int64_t p = 0; p < A.nnz(); p++) cptr[A.col[p] + 1]++;
  for (int64_t c = 0; c < n; c++) cptr[c + 1] += cptr[c];
  crow.resize(A.nnz());
  std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
  for (int64_t i = 0; i < n; i++)
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; p++) crow[fill[A.col[p]]++] = (int32_t)i;
}

// plain ascending sum over shared columns (DESIGN.md §3 P2)
double shared_dot(const HostCSR& A, int64_t i, int64_t l) {
  int64_t p = A.ptr[i], pe = A.ptr[i + 1], q = A.ptr[l], qe = A.ptr[l + 1];
  double s = 0.0;
  while (p < pe && q < qe) {
    int32_t a = A.col[p], b = A.col[q];
    if (a < b) p++;
    else if (b < a) q++;
    else { s = s + A.val[p] * A.val[q]; p++; q++; }
  }
  return s;
}
}  // namespace

// DESIGN.md §3 P1-P2: colour[i] = mex{colour[l] : l < i, rows i and l conflict}; rows conflict
// when they share a column and, for thr > 0, dot^2 >= (thr*thr) * (nrm2_i * nrm2_l).
void first_fit_colour(const HostCSR& A, const std::vector<double>& nrm2, double thr, std::vector<int32_t>& colour) {
  const int64_t n = A.m;
  std::vector<int64_t> cptr;
  std::vector<int32_t> crow;
  column_rows(A, cptr, crow);
  colour.assign(n, 0);
  std::vector<int32_t> used(n + 1, -1);   // used[c] == i  <=> colour c taken by a conflicting l < i
  std::vector<int32_t> cand(n, -1);       // thr > 0: candidate l already tested for row i
  const double t2 = thr * thr;
  for (int64_t i = 0; i < n; i++) {
    const int32_t ii = (int32_t)i;
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; p++) {
      const int32_t c = A.col[p];
      for (int64_t q = cptr[c]; q < cptr[c + 1]; q++) {
        const int32_t l = crow[q];
        if (l >= ii) break;  // rows of a column are ascending
        if (thr == 0.0) {
          used[colour[l]] = ii;
        } else if (cand[l] != ii) {
          cand[l] = ii;
          const double d = shared_dot(A, i, l);
          if (d * d >= t2 * (nrm2[i] * nrm2[l])) used[colour[l]] = ii;
        }
      }
    }
    int32_t k = 0;
    while (used[k] == ii) k++;
    colour[i] = k;
  }
}

void build_schedule(const HostCSR& A, const std::vector<int32_t>& colour, bool check_overlap, Schedule& s) {
  const int64_t n = A.m;
  int32_t ncol = 0;
  for (int32_t c : colour) ncol = std::max(ncol, c + 1);
  std::vector<int64_t> size(ncol, 0);
  for (int32_t c : colour) size[c]++;
  // Oclass: colours with >= 2 rows, ascending; rows ascending within (counting sort keeps order)
  std::vector<int32_t> step_of_colour(ncol, -1);
  s.step_ptr.assign(1, 0);
  int32_t nst = 0;
  for (int32_t c = 0; c < ncol; c++)
    if (size[c] >= 2) { step_of_colour[c] = nst++; s.step_ptr.push_back(s.step_ptr.back() + (int32_t)size[c]); }
  s.n_oclass = nst;
  std::vector<int32_t> fill(s.step_ptr.begin(), s.step_ptr.end() - 1);
  s.rows.assign(n, -1);
  int32_t pos_single = s.step_ptr.back();
  for (int64_t i = 0; i < n; i++) {
    int32_t st = step_of_colour[colour[i]];
    if (st >= 0) s.rows[fill[st]++] = (int32_t)i;
  }
  // Nclass: singleton colours, ascending row index, one step each
  for (int64_t i = 0; i < n; i++)
    if (step_of_colour[colour[i]] < 0) {
      s.rows[pos_single++] = (int32_t)i;
      s.step_ptr.push_back(pos_single);
    }
  const int32_t nsteps = (int32_t)s.step_ptr.size() - 1;
  s.overlap.assign(nsteps, 0);
  if (check_overlap) {
    std::vector<int32_t> step_of_row(n);
    for (int32_t k = 0; k < nsteps; k++)
      for (int32_t q = s.step_ptr[k]; q < s.step_ptr[k + 1]; q++) step_of_row[s.rows[q]] = k;
    std::vector<int64_t> cptr;
    std::vector<int32_t> crow;
    column_rows(A, cptr, crow);
    std::vector<int64_t> stamp(nsteps, -1);
    for (int64_t c = 0; c < n; c++)
      for (int64_t q = cptr[c]; q < cptr[c + 1]; q++) {
        int32_t k = step_of_row[crow[q]];
        if (stamp[k] == c) s.overlap[k] = 1;
        stamp[k] = c;
      }
  }
}

// NEXT-1 guard for thr > 0: within a category, row i's overlapping neighbours
// must satisfy sum |cos(a_i, a_l)| < 1 (a Gershgorin bound keeping the simultaneous step
// A_tau^T D^-1 a contraction).  Returns false and a reason naming the row otherwise.
bool gershgorin_guard(const HostCSR& A, const std::vector<double>& nrm2, const std::vector<int32_t>& colour,
                      std::string& why) {
  std::vector<int64_t> cptr;
  std::vector<int32_t> crow;
  column_rows(A, cptr, crow);
  std::vector<int64_t> cand(A.m, -1);
  for (int64_t i = 0; i < A.m; i++) {
    double acc = 0.0;
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; p++)
      for (int64_t q = cptr[A.col[p]]; q < cptr[A.col[p] + 1]; q++) {
        int32_t l = crow[q];
        if (l == i || colour[l] != colour[i] || cand[l] == i) continue;
        cand[l] = i;
        acc += std::fabs(shared_dot(A, i, l)) / std::sqrt(nrm2[i] * nrm2[l]);
      }
    if (acc >= 1.0) {
      why = "row " + std::to_string(i) + ": sum of |cos| to overlapping rows of its category = " + std::to_string(acc) +
            " >= 1 (thr too large)";
      return false;
    }
  }
  return true;
}

}  // namespace pobk
