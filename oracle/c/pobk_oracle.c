/*
 * POBK oracle, plain C part -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this file's shared object.  It shares no code, header, table or helper
 * with the product (paper_2401_00672_b200/): it is an independent, literal, slow
 * restatement of the method in PAPER.md (arXiv 2401.00672), following SURVEY.md §8(c)
 * O1-O9 step by step.  Loop-heavy integer work (RCM, first-fit) and the row-by-row
 * Kaczmarz sweep live here because pure-Python loops are too slow beyond tiny sizes;
 * every loop below is the plain definition, with no blocking, fusion or reordering.
 *
 * Compile with -ffp-contract=off: every floating-point operation is rounded as written
 * (no FMA contraction), so the sums are the plain left-to-right sums the readings fix.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ O1: row norms
 * nrm2_i = sum_p a_ip^2, ascending column order, plain left-to-right sum from 0.0
 * (denominator of Eq 1.2). */
void orc_row_nrm2(int64_t m, const int64_t* indptr, const double* val, double* nrm2) {
  for (int64_t i = 0; i < m; i++) {
    double s = 0.0;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) s = s + val[p] * val[p];
    nrm2[i] = s;
  }
}

/* ------------------------------------------------------------------ O2: graph
 * G = pattern(A + A^T) without self loops, as adjacency lists
 * (duplicates removed).  deg(v) = |adj(v)|. */
typedef struct {
  int64_t m;
  int64_t* ptr; /* [m+1] */
  int32_t* adj; /* [ptr[m]] */
  int32_t* deg; /* [m] */
} orc_graph;

static int cmp_int32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static int build_graph(int64_t m, const int64_t* indptr, const int32_t* indices, orc_graph* g) {
  int64_t* cnt = (int64_t*)calloc((size_t)m + 1, sizeof(int64_t));
  if (!cnt) return -1;
  for (int64_t i = 0; i < m; i++)
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) {
      int64_t j = indices[p];
      if (j == i) continue;
      cnt[i]++; /* edge i-j seen from row i */
      cnt[j]++; /* and its transpose */
    }
  int64_t* ptr = (int64_t*)malloc(((size_t)m + 1) * sizeof(int64_t));
  ptr[0] = 0;
  for (int64_t i = 0; i < m; i++) ptr[i + 1] = ptr[i] + cnt[i];
  int32_t* adj = (int32_t*)malloc((size_t)(ptr[m] > 0 ? ptr[m] : 1) * sizeof(int32_t));
  for (int64_t i = 0; i < m; i++) cnt[i] = ptr[i];
  for (int64_t i = 0; i < m; i++)
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) {
      int64_t j = indices[p];
      if (j == i) continue;
      adj[cnt[i]++] = (int32_t)j;
      adj[cnt[j]++] = (int32_t)i;
    }
  /* sort and deduplicate each list (an entry present in both A and A^T appears twice) */
  int64_t* nptr = (int64_t*)malloc(((size_t)m + 1) * sizeof(int64_t));
  int32_t* deg = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  int64_t w = 0;
  nptr[0] = 0;
  for (int64_t i = 0; i < m; i++) {
    int64_t b = ptr[i], e = ptr[i + 1];
    qsort(adj + b, (size_t)(e - b), sizeof(int32_t), cmp_int32);
    int64_t start = w;
    for (int64_t p = b; p < e; p++)
      if (p == b || adj[p] != adj[p - 1]) adj[w++] = adj[p];
    nptr[i + 1] = w;
    deg[i] = (int32_t)(w - start);
  }
  free(ptr);
  free(cnt);
  g->m = m;
  g->ptr = nptr;
  g->adj = adj;
  g->deg = deg;
  return 0;
}

static void free_graph(orc_graph* g) {
  free(g->ptr);
  free(g->adj);
  free(g->deg);
}

/* (deg, index) lexicographic order -- the deterministic tie-break of SPEC.md:145 */
static const int32_t* g_deg_for_sort;
static int cmp_deg_idx(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  int32_t dx = g_deg_for_sort[x], dy = g_deg_for_sort[y];
  if (dx != dy) return (dx > dy) - (dx < dy);
  return (x > y) - (x < y);
}
static int less_deg_idx(const int32_t* deg, int32_t a, int32_t b) {
  return deg[a] < deg[b] || (deg[a] == deg[b] && a < b);
}

/* BFS level structure rooted at r.  dist[] must be all -1 on entry and is restored to -1.
 * Returns the number of levels (depth + 1); writes the last level's nodes into last[],
 * their count into *nlast.  queue[] is scratch of size m. */
static int64_t bfs_levels(const orc_graph* g, int32_t r, int32_t* dist, int32_t* queue, int32_t* last, int64_t* nlast) {
  int64_t head = 0, tail = 0;
  queue[tail++] = r;
  dist[r] = 0;
  while (head < tail) {
    int32_t v = queue[head++];
    for (int64_t p = g->ptr[v]; p < g->ptr[v + 1]; p++) {
      int32_t u = g->adj[p];
      if (dist[u] < 0) {
        dist[u] = dist[v] + 1;
        queue[tail++] = u;
      }
    }
  }
  int32_t maxd = dist[queue[tail - 1]]; /* BFS pops in nondecreasing distance */
  int64_t n = 0;
  for (int64_t k = 0; k < tail; k++)
    if (dist[queue[k]] == maxd) last[n++] = queue[k];
  *nlast = n;
  for (int64_t k = 0; k < tail; k++) dist[queue[k]] = -1;
  return (int64_t)maxd + 1;
}

/* ------------------------------------------------------------------ O3: RCM
 * PAPER.md:152-154 (RCM, MATLAB symrcm), Eq 3.1; rule pinned in
 * SURVEY.md §8(c) O3 / Z11:
 *   components in ascending order of their minimum index;
 *   r = argmin_{v in comp} (deg v, v);  L = levels(r)
 *   repeat <= 10: x = argmin_{v in last level of L} (deg, idx); if depth(x) > depth(r): r = x
 *                 else break;           root = x (the last candidate computed)
 *   Cuthill-McKee BFS from root, FIFO, mark on enqueue, neighbours enqueued in ascending
 *   (deg, idx); append on pop;  perm = reverse(whole order), perm[new] = old.
 * With reorder = 0 the caller uses the identity instead. */
int orc_rcm(int64_t m, const int64_t* indptr, const int32_t* indices, int32_t* perm) {
  orc_graph g;
  if (build_graph(m, indptr, indices, &g)) return -1;
  int32_t* dist = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  int32_t* queue = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  int32_t* last = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  int32_t* lastx = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  int32_t* order = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  int32_t* nbr = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  char* visited = (char*)calloc((size_t)m, 1);
  for (int64_t i = 0; i < m; i++) dist[i] = -1;
  int64_t norder = 0;
  g_deg_for_sort = g.deg;

  for (int64_t s0 = 0; s0 < m; s0++) {
    if (visited[s0]) continue;
    /* the component of s0: every node reachable from s0 */
    int64_t nlast = 0;
    int64_t head = 0, tail = 0;
    queue[tail++] = (int32_t)s0;
    dist[s0] = 0;
    while (head < tail) {
      int32_t v = queue[head++];
      for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; p++)
        if (dist[g.adj[p]] < 0) { dist[g.adj[p]] = 0; queue[tail++] = g.adj[p]; }
    }
    int32_t r = queue[0];
    for (int64_t k = 1; k < tail; k++)
      if (less_deg_idx(g.deg, queue[k], r)) r = queue[k];
    for (int64_t k = 0; k < tail; k++) dist[queue[k]] = -1;

    /* George-Liu pseudo-peripheral search */
    int64_t depth_r = bfs_levels(&g, r, dist, queue, last, &nlast);
    int32_t x = r;
    for (int it = 0; it < 10; it++) {
      x = last[0];
      for (int64_t k = 1; k < nlast; k++)
        if (less_deg_idx(g.deg, last[k], x)) x = last[k];
      int64_t nlastx = 0;
      int64_t depth_x = bfs_levels(&g, x, dist, queue, lastx, &nlastx);
      if (depth_x > depth_r) {
        r = x;
        depth_r = depth_x;
        memcpy(last, lastx, (size_t)nlastx * sizeof(int32_t));
        nlast = nlastx;
      } else {
        break;
      }
    }
    int32_t root = x;

    /* Cuthill-McKee BFS */
    head = 0;
    tail = 0;
    queue[tail++] = root;
    visited[root] = 1;
    while (head < tail) {
      int32_t v = queue[head++];
      order[norder++] = v;
      int64_t nn = 0;
      for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; p++)
        if (!visited[g.adj[p]]) nbr[nn++] = g.adj[p];
      qsort(nbr, (size_t)nn, sizeof(int32_t), cmp_deg_idx);
      for (int64_t k = 0; k < nn; k++) {
        visited[nbr[k]] = 1;
        queue[tail++] = nbr[k];
      }
    }
  }
  for (int64_t i = 0; i < m; i++) perm[i] = order[m - 1 - i];
  free(dist); free(queue); free(last); free(lastx); free(order); free(nbr); free(visited);
  free_graph(&g);
  return 0;
}

/* ------------------------------------------------------------------ O5/O6: first-fit
 * Rows of the permuted matrix A~ (RCM frame).  conflict(i,l), i != l, holds iff rows i and l
 * share a column and, when thr > 0, additionally dot^2 >= thr^2 * nrm2_i * nrm2_l with dot the
 * plain ascending sum over shared columns ("when C(i,j) < thr ... considered
 * orthogonal"; absolute cosine SPEC.md:273; association fixed in SURVEY.md §8(c) O5).
 * color[i] = mex{ color[l] : l < i, conflict(i,l) }  (PAPER.md:220 first-orthogonal rule,
 * iterated; "place all two-by-two mutually orthogonal blocks in a category"). */
static double row_dot(const int64_t* indptr, const int32_t* indices, const double* val, int64_t i, int64_t l) {
  int64_t p = indptr[i], q = indptr[l];
  double s = 0.0;
  while (p < indptr[i + 1] && q < indptr[l + 1]) {
    if (indices[p] < indices[q]) p++;
    else if (indices[p] > indices[q]) q++;
    else { s = s + val[p] * val[q]; p++; q++; }
  }
  return s;
}

int orc_first_fit(int64_t m, const int64_t* indptr, const int32_t* indices, const double* val,
                  const double* nrm2, double thr, int32_t* color) {
  int64_t nnz = indptr[m];
  /* CSC: rows of each column, ascending */
  int64_t* cptr = (int64_t*)calloc((size_t)m + 1, sizeof(int64_t));
  int32_t* crow = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
  for (int64_t p = 0; p < nnz; p++) cptr[indices[p] + 1]++;
  for (int64_t c = 0; c < m; c++) cptr[c + 1] += cptr[c];
  int64_t* fill = (int64_t*)malloc(((size_t)m + 1) * sizeof(int64_t));
  memcpy(fill, cptr, ((size_t)m + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < m; i++)
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) crow[fill[indices[p]]++] = (int32_t)i;
  int64_t* seen = (int64_t*)malloc(((size_t)m + 1) * sizeof(int64_t)); /* seen[colour] == i */
  int64_t* cand = (int64_t*)malloc(((size_t)m + 1) * sizeof(int64_t)); /* cand[row] == i */
  for (int64_t k = 0; k <= m; k++) { seen[k] = -1; cand[k] = -1; }
  for (int64_t i = 0; i < m; i++) {
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) {
      int32_t c = indices[p];
      for (int64_t q = cptr[c]; q < cptr[c + 1]; q++) {
        int32_t l = crow[q];
        if (l >= i) continue;
        if (thr == 0.0) {
          seen[color[l]] = i;
        } else if (cand[l] != i) {
          cand[l] = i;
          double d = row_dot(indptr, indices, val, i, l);
          if (d * d >= (thr * thr) * (nrm2[i] * nrm2[l])) seen[color[l]] = i;
        }
      }
    }
    int32_t k = 0;
    while (seen[k] == i) k++;
    color[i] = k;
  }
  free(cptr); free(crow); free(fill); free(seen); free(cand);
  return 0;
}

/* A category is "disjoint" when no two of its rows share a column; only then is the plain
 * sequential update order irrelevant (Lemma 1).  out[c] = 1 if category c
 * has two rows sharing a column (possible only with thr > 0). */
int orc_category_overlap(int64_t m, const int64_t* indptr, const int32_t* indices, const int32_t* color,
                         int64_t ncolors, uint8_t* out) {
  int64_t nnz = indptr[m];
  /* owner[c][colour] would be large; instead walk columns: for each column collect colours */
  int64_t* cptr = (int64_t*)calloc((size_t)m + 1, sizeof(int64_t));
  int32_t* crow = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
  for (int64_t p = 0; p < nnz; p++) cptr[indices[p] + 1]++;
  for (int64_t c = 0; c < m; c++) cptr[c + 1] += cptr[c];
  int64_t* fill = (int64_t*)malloc(((size_t)m + 1) * sizeof(int64_t));
  memcpy(fill, cptr, ((size_t)m + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < m; i++)
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) crow[fill[indices[p]]++] = (int32_t)i;
  int64_t* stamp = (int64_t*)malloc((size_t)(ncolors > 0 ? ncolors : 1) * sizeof(int64_t));
  for (int64_t k = 0; k < ncolors; k++) { stamp[k] = -1; out[k] = 0; }
  for (int64_t c = 0; c < m; c++)
    for (int64_t q = cptr[c]; q < cptr[c + 1]; q++) {
      int32_t k = color[crow[q]];
      if (stamp[k] == c) out[k] = 1;
      stamp[k] = c;
    }
  free(cptr); free(crow); free(fill); free(stamp);
  return 0;
}

/* ------------------------------------------------------------------ O7: one sweep
 * For each step k of the schedule sigma (Alg 5 loop),
 * for each row i of the step in ascending order, the classical Kaczmarz projection Eq 1.2
 * (PAPER.md:28-30):
 *     r = f_i - sum_p a_ip x_{col p}      (ascending p, from 0.0)
 *     alpha = r / nrm2_i
 *     x_{col p} = x_{col p} + alpha * a_ip
 * For a step whose rows overlap (thr > 0, overlap[k] = 1): every alpha of the step is computed
 * first at the same x (the block step Eq 1.3 with the Lemma-1 collapse, PAPER.md:34-37,
 * 257-261), then applied in (i ascending, p ascending) order. */
void orc_sweep(int64_t m, const int64_t* indptr, const int32_t* indices, const double* val,
               const double* nrm2, const double* f, double* x, int64_t nsteps, const int64_t* step_ptr,
               const int32_t* step_rows, const uint8_t* overlap, double* alpha_scratch) {
  (void)m;
  for (int64_t k = 0; k < nsteps; k++) {
    if (!overlap[k]) {
      for (int64_t q = step_ptr[k]; q < step_ptr[k + 1]; q++) {
        int64_t i = step_rows[q];
        double s = 0.0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) s = s + val[p] * x[indices[p]];
        double r = f[i] - s;
        double alpha = r / nrm2[i];
        for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) x[indices[p]] = x[indices[p]] + alpha * val[p];
      }
    } else {
      for (int64_t q = step_ptr[k]; q < step_ptr[k + 1]; q++) {
        int64_t i = step_rows[q];
        double s = 0.0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) s = s + val[p] * x[indices[p]];
        alpha_scratch[q - step_ptr[k]] = (f[i] - s) / nrm2[i];
      }
      for (int64_t q = step_ptr[k]; q < step_ptr[k + 1]; q++) {
        int64_t i = step_rows[q];
        double alpha = alpha_scratch[q - step_ptr[k]];
        for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) x[indices[p]] = x[indices[p]] + alpha * val[p];
      }
    }
  }
}

/* Residual of every row, r_i = f_i - sum_p a_ip x_{col p} (ascending p, from 0.0): the residual
 * ordering's per-row input (DESIGN.md §3 reading R-G). */
void orc_row_residuals(int64_t m, const int64_t* indptr, const int32_t* indices, const double* val,
                       const double* f, const double* x, double* r) {
  for (int64_t i = 0; i < m; i++) {
    double s = 0.0;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) s = s + val[p] * x[indices[p]];
    r[i] = f[i] - s;
  }
}

/* ------------------------------------------------------------------ O8: stopping values
 * RSE = ||x - x*||_2 / ||x*||_2; RELRES = ||f - A x||_2 / ||f||_2.
 * Plain ascending sums of squares. */
double orc_rse(int64_t m, const double* x, const double* xs) {
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < m; i++) {
    double d = x[i] - xs[i];
    num = num + d * d;
    den = den + xs[i] * xs[i];
  }
  return sqrt(num) / sqrt(den);
}

double orc_residual_sumsq(int64_t m, const int64_t* indptr, const int32_t* indices, const double* val,
                          const double* f, const double* x) {
  double acc = 0.0;
  for (int64_t i = 0; i < m; i++) {
    double s = 0.0;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; p++) s = s + val[p] * x[indices[p]];
    double r = f[i] - s;
    acc = acc + r * r;
  }
  return acc;
}

double orc_relres(int64_t m, const int64_t* indptr, const int32_t* indices, const double* val,
                  const double* f, const double* x) {
  double den = 0.0;
  for (int64_t i = 0; i < m; i++) den = den + f[i] * f[i];
  return sqrt(orc_residual_sumsq(m, indptr, indices, val, f, x)) / sqrt(den);
}

/* ------------------------------------------------------------------ solve loop (O7 + O8)
 * After every sweep s = 1, 2, ...: value = RSE (stop = 0, needs xs) or RELRES (stop = 1);
 * non-finite -> termination 2; value < tol (strict) -> termination 0;
 * s == max_sweeps -> termination 1 (the paper's "Inf"/"NAN").
 * trace (may be NULL) receives the value after each sweep. */
int orc_solve(int64_t m, const int64_t* indptr, const int32_t* indices, const double* val, const double* nrm2,
              const double* f, double* x, const double* xs, int64_t nsteps, const int64_t* step_ptr,
              const int32_t* step_rows, const uint8_t* overlap, int32_t stop, double tol, int64_t max_sweeps,
              int64_t* sweeps_out, int32_t* term_out, double* value_out, double* trace) {
  double* scratch = (double*)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
  int32_t term = 1;
  int64_t s = 0;
  double v = NAN;
  for (s = 1; s <= max_sweeps; s++) {
    orc_sweep(m, indptr, indices, val, nrm2, f, x, nsteps, step_ptr, step_rows, overlap, scratch);
    v = (stop == 0) ? orc_rse(m, x, xs) : orc_relres(m, indptr, indices, val, f, x);
    if (trace) trace[s - 1] = v;
    if (!isfinite(v)) { term = 2; break; }
    if (v < tol) { term = 0; break; }
  }
  if (s > max_sweeps) s = max_sweeps;
  free(scratch);
  *sweeps_out = s;
  *term_out = term;
  *value_out = v;
  return 0;
}
