/* Tier S CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain single-threaded C, written to be checked by eye against its
 * definitions.  Shares no code with paper_2403_15913_b200/csrc.
 *
 *   orc_nd_order     the nested-dissection ordering specified in DESIGN.md §5
 *                    (SURVEY.md §8(c) C8 reading).  Paper: the ordering is
 *                    internal to cuDSS ("finding an appropriate ordering to
 *                    reduce the fill-in").
 *   orc_symbolic     elimination tree + L pattern by the column-merge
 *                    definition struct(L_j) = struct(A_{>=j,j}) ∪
 *                    ⋃_{parent(c)=j} struct(L_c)\{c}, parent(j) = min
 *                    struct(L_j)\{j}  (symbolic analysis).
 *   orc_cholesky     left-looking column Cholesky on that pattern
 *                    (refactorization); returns the first
 *                    column whose pivot is not > 0 and finite.
 *   orc_lsolve/orc_ltsolve  forward / backward substitution (backsolve).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* ordering                                                            */
/* ------------------------------------------------------------------ */
typedef struct {
  int n;
  const int *xadj, *adj;
  int leaf;
  int *memb;   /* membership stamp of the current vertex set        */
  int *seen;   /* visited stamp for BFS                             */
  int *dist;   /* BFS distance                                      */
  int stamp;
  int *out;    /* output order (new -> old)                         */
  int nout;
  int err;
} ord_t;

static int cmp_int(const void *a, const void *b) {
  int x = *(const int *)a, y = *(const int *)b;
  return (x > y) - (x < y);
}

/* BFS from r inside vertices with memb == ms; fills q with visit order and
 * level boundaries lvl_start[0..h+1]; returns h+1 = number of levels. */
static int bfs_levels(ord_t *o, int ms, int r, int *q, int *lvl_start) {
  int s = ++o->stamp;
  int head = 0, tail = 0, nlev = 0;
  q[tail++] = r;
  o->seen[r] = s;
  o->dist[r] = 0;
  lvl_start[0] = 0;
  int curd = 0;
  while (head < tail) {
    int v = q[head];
    if (o->dist[v] != curd) { /* new level begins at head */
      curd = o->dist[v];
      lvl_start[++nlev] = head;
    }
    head++;
    for (int p = o->xadj[v]; p < o->xadj[v + 1]; p++) {
      int a = o->adj[p];
      if (o->memb[a] == ms && o->seen[a] != s) {
        o->seen[a] = s;
        o->dist[a] = o->dist[v] + 1;
        q[tail++] = a;
      }
    }
  }
  nlev++;
  lvl_start[nlev] = tail;
  return nlev;
}

static int degree_in(ord_t *o, int ms, int v) {
  int d = 0;
  for (int p = o->xadj[v]; p < o->xadj[v + 1]; p++)
    if (o->memb[o->adj[p]] == ms) d++;
  return d;
}

/* exact minimum degree on the induced subgraph G[C], C sorted ascending;
 * ties -> smallest original index.  Dense elimination-graph matrix. */
static void md_order(ord_t *o, const int *C, int k) {
  if (k == 0) return;
  if (k > 16384) { o->err = -2; return; }
  unsigned char *A = (unsigned char *)calloc((size_t)k * k, 1);
  int *deg = (int *)calloc(k, sizeof(int));
  unsigned char *elim = (unsigned char *)calloc(k, 1);
  int *nb = (int *)malloc(sizeof(int) * k);
  /* local index of vertex: binary search in sorted C */
  for (int i = 0; i < k; i++) {
    int v = C[i];
    for (int p = o->xadj[v]; p < o->xadj[v + 1]; p++) {
      int a = o->adj[p];
      int *f = (int *)bsearch(&a, C, k, sizeof(int), cmp_int);
      if (f && a != v) A[(size_t)i * k + (f - C)] = 1;
    }
  }
  for (int i = 0; i < k; i++) {
    int d = 0;
    for (int j = 0; j < k; j++) d += A[(size_t)i * k + j];
    deg[i] = d;
  }
  for (int step = 0; step < k; step++) {
    int best = -1;
    for (int i = 0; i < k; i++)
      if (!elim[i] && (best < 0 || deg[i] < deg[best])) best = i;
    int v = best;
    o->out[o->nout++] = C[v];
    elim[v] = 1;
    int nn = 0;
    for (int j = 0; j < k; j++)
      if (A[(size_t)v * k + j] && !elim[j]) nb[nn++] = j;
    for (int x = 0; x < nn; x++) {
      int a = nb[x];
      A[(size_t)a * k + v] = 0;
      deg[a]--;
      for (int y = 0; y < nn; y++) {
        int b = nb[y];
        if (b != a && !A[(size_t)a * k + b]) {
          A[(size_t)a * k + b] = 1;
          deg[a]++;
        }
      }
    }
  }
  free(A); free(deg); free(elim); free(nb);
}

static void nd_rec(ord_t *o, int *V, int nv);

/* one connected component C (sorted ascending, size k) */
static void nd_component(ord_t *o, int *C, int k) {
  if (k <= o->leaf) { md_order(o, C, k); return; }
  int ms = ++o->stamp;
  for (int i = 0; i < k; i++) o->memb[C[i]] = ms;
  int *q = (int *)malloc(sizeof(int) * k);
  int *ls = (int *)malloc(sizeof(int) * (k + 2));
  int *q2 = (int *)malloc(sizeof(int) * k);
  int *ls2 = (int *)malloc(sizeof(int) * (k + 2));
  /* pseudo-peripheral vertex (George–Liu): start at the smallest index */
  int r = C[0];
  int nlev = bfs_levels(o, ms, r, q, ls);
  for (;;) {
    int best = -1, bdeg = 0;
    for (int p = ls[nlev - 1]; p < ls[nlev]; p++) {
      int v = q[p];
      int d = degree_in(o, ms, v);
      if (best < 0 || d < bdeg || (d == bdeg && v < best)) { best = v; bdeg = d; }
    }
    int nlev2 = bfs_levels(o, ms, best, q2, ls2);
    if (nlev2 > nlev) {
      r = best; nlev = nlev2;
      int *t = q; q = q2; q2 = t;
      t = ls; ls = ls2; ls2 = t;
    } else break;
  }
  int h = nlev - 1;
  if (h < 2) {
    md_order(o, C, k);
  } else {
    int ilo = h / 3; if (ilo < 1) ilo = 1;
    int ihi = h - h / 3; if (ihi > h - 1) ihi = h - 1;
    int bi = -1;
    for (int i = ilo; i <= ihi; i++) {
      int sz = ls[i + 1] - ls[i], bsz = bi < 0 ? 0 : ls[bi + 1] - ls[bi];
      int c = abs(2 * i - h), bc = bi < 0 ? 0 : abs(2 * bi - h);
      if (bi < 0 || sz < bsz || (sz == bsz && c < bc)) bi = i;  /* equal (sz, c): keep smaller i */
    }
    int ns = ls[bi + 1] - ls[bi];
    int *S = (int *)malloc(sizeof(int) * ns);
    memcpy(S, q + ls[bi], sizeof(int) * ns);
    qsort(S, ns, sizeof(int), cmp_int);
    int *rest = (int *)malloc(sizeof(int) * (k - ns));
    int nr = 0;
    /* rest = C \ S in ascending order (C sorted; S sorted) */
    for (int i = 0, j = 0; i < k; i++) {
      while (j < ns && S[j] < C[i]) j++;
      if (j < ns && S[j] == C[i]) continue;
      rest[nr++] = C[i];
    }
    nd_rec(o, rest, nr);
    for (int i = 0; i < ns; i++) o->out[o->nout++] = S[i];
    free(S); free(rest);
  }
  free(q); free(ls); free(q2); free(ls2);
}

/* V sorted ascending: split into connected components of G[V], ordered by
 * smallest vertex, each sorted ascending. */
static void nd_rec(ord_t *o, int *V, int nv) {
  if (nv == 0) return;
  int ms = ++o->stamp;
  for (int i = 0; i < nv; i++) o->memb[V[i]] = ms;
  int vs = ++o->stamp;
  int *comp = (int *)malloc(sizeof(int) * nv);
  int *cstart = (int *)malloc(sizeof(int) * (nv + 1));
  int nc = 0, tot = 0;
  for (int i = 0; i < nv; i++) {
    int v = V[i];
    if (o->seen[v] == vs) continue;
    cstart[nc++] = tot;
    int head = tot;
    comp[tot++] = v;
    o->seen[v] = vs;
    while (head < tot) {
      int x = comp[head++];
      for (int p = o->xadj[x]; p < o->xadj[x + 1]; p++) {
        int a = o->adj[p];
        if (o->memb[a] == ms && o->seen[a] != vs) { o->seen[a] = vs; comp[tot++] = a; }
      }
    }
  }
  cstart[nc] = tot;
  for (int c = 0; c < nc; c++) qsort(comp + cstart[c], cstart[c + 1] - cstart[c], sizeof(int), cmp_int);
  for (int c = 0; c < nc && !o->err; c++) nd_component(o, comp + cstart[c], cstart[c + 1] - cstart[c]);
  free(comp); free(cstart);
}

/* xadj/adj: symmetric adjacency without self loops, each list ascending.
 * perm[k] = original vertex placed at position k.  Returns 0 or < 0. */
int orc_nd_order(int n, const int *xadj, const int *adj, int leaf, int *perm) {
  ord_t o;
  memset(&o, 0, sizeof o);
  o.n = n; o.xadj = xadj; o.adj = adj; o.leaf = leaf < 1 ? 1 : leaf;
  o.memb = (int *)calloc(n, sizeof(int));
  o.seen = (int *)calloc(n, sizeof(int));
  o.dist = (int *)calloc(n, sizeof(int));
  o.out = perm;
  int *V = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int i = 0; i < n; i++) V[i] = i;
  nd_rec(&o, V, n);
  free(V); free(o.memb); free(o.seen); free(o.dist);
  if (o.err) return o.err;
  return o.nout == n ? 0 : -1;
}

/* ------------------------------------------------------------------ */
/* symbolic analysis by column merge                                  */
/* ------------------------------------------------------------------ */
/* (Ap, Ai): lower-triangular CSC pattern of P K P^T incl. the diagonal.
 * Outputs parent[n] (-1 = root), colcount[n]; if Lp/Li are non-NULL also the
 * L pattern (rows ascending, diagonal first).  Returns nnz(L) or -1. */
int64_t orc_symbolic(int n, const int64_t *Ap, const int *Ai, int *parent, int *colcount,
                     int64_t *Lp, int *Li) {
  int64_t cap = (Ap[n] > 16 ? Ap[n] : 16) * 2, used = 0;
  int *buf = (int *)malloc(sizeof(int) * cap);
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
  int *mark = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
  int *tmp = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
  int *child_head = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
  int *child_next = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int i = 0; i < n; i++) { mark[i] = -1; child_head[i] = -1; }
  for (int j = 0; j < n; j++) {
    int cnt = 0;
    mark[j] = j; tmp[cnt++] = j;
    for (int64_t p = Ap[j]; p < Ap[j + 1]; p++) {
      int i = Ai[p];
      if (i > j && mark[i] != j) { mark[i] = j; tmp[cnt++] = i; }
    }
    for (int c = child_head[j]; c >= 0; c = child_next[c]) {
      for (int64_t p = start[c]; p < start[c] + colcount[c]; p++) {
        int i = buf[p];
        if (i != c && mark[i] != j) { mark[i] = j; tmp[cnt++] = i; }
      }
    }
    qsort(tmp, cnt, sizeof(int), cmp_int);
    if (used + cnt > cap) {
      while (used + cnt > cap) cap *= 2;
      buf = (int *)realloc(buf, sizeof(int) * cap);
      if (!buf) return -1;
    }
    start[j] = used;
    memcpy(buf + used, tmp, sizeof(int) * cnt);
    used += cnt;
    colcount[j] = cnt;
    parent[j] = cnt > 1 ? tmp[1] : -1;
    if (parent[j] >= 0) {
      /* children lists in increasing order of child index: append at tail */
      int pj = parent[j];
      child_next[j] = -1;
      if (child_head[pj] < 0) child_head[pj] = j;
      else { int c = child_head[pj]; while (child_next[c] >= 0) c = child_next[c]; child_next[c] = j; }
    }
  }
  if (Lp) {
    Lp[0] = 0;
    for (int j = 0; j < n; j++) Lp[j + 1] = Lp[j] + colcount[j];
  }
  if (Li) memcpy(Li, buf, sizeof(int) * used);
  free(buf); free(start); free(mark); free(tmp); free(child_head); free(child_next);
  return used;
}

/* ------------------------------------------------------------------ */
/* numeric left-looking Cholesky                                      */
/* ------------------------------------------------------------------ */
/* A = P K P^T lower CSC values (same pattern as Ap/Ai).  L on (Lp, Li).
 * Returns -1 on success, else the first column j with a pivot that is not
 * > 0 and finite (Cholesky breaks down). */
int orc_cholesky(int n, const int64_t *Ap, const int *Ai, const double *Ax,
                 const int64_t *Lp, const int *Li, double *Lx) {
  double *x = (double *)calloc(n > 0 ? n : 1, sizeof(double));
  int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int *head = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
  int *next = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
  int fail = -1;
  for (int i = 0; i < n; i++) head[i] = -1;
  for (int j = 0; j < n && fail < 0; j++) {
    for (int64_t p = Ap[j]; p < Ap[j + 1]; p++) x[Ai[p]] += Ax[p];
    /* columns k < j with L(j,k) != 0 */
    int k = head[j];
    head[j] = -1;
    while (k >= 0) {
      int knext = next[k];
      int64_t p = pos[k];
      double ljk = Lx[p];
      for (int64_t q = p; q < Lp[k + 1]; q++) x[Li[q]] -= Lx[q] * ljk;
      pos[k] = p + 1;
      if (pos[k] < Lp[k + 1]) { int i = Li[pos[k]]; next[k] = head[i]; head[i] = k; }
      k = knext;
    }
    double d = x[j];
    if (!(d > 0.0) || !isfinite(d)) { fail = j; break; }
    double s = sqrt(d);
    Lx[Lp[j]] = s;
    x[j] = 0.0;
    for (int64_t q = Lp[j] + 1; q < Lp[j + 1]; q++) { Lx[q] = x[Li[q]] / s; x[Li[q]] = 0.0; }
    pos[j] = Lp[j] + 1;
    if (pos[j] < Lp[j + 1]) { int i = Li[pos[j]]; next[j] = head[i]; head[i] = j; }
  }
  free(x); free(pos); free(head); free(next);
  return fail;
}

/* forward substitution L y = b (in place) */
void orc_lsolve(int n, const int64_t *Lp, const int *Li, const double *Lx, double *x) {
  for (int j = 0; j < n; j++) {
    x[j] /= Lx[Lp[j]];
    double xj = x[j];
    for (int64_t q = Lp[j] + 1; q < Lp[j + 1]; q++) x[Li[q]] -= Lx[q] * xj;
  }
}

/* backward substitution L^T x = y (in place) */
void orc_ltsolve(int n, const int64_t *Lp, const int *Li, const double *Lx, double *x) {
  for (int j = n - 1; j >= 0; j--) {
    double s = x[j];
    for (int64_t q = Lp[j] + 1; q < Lp[j + 1]; q++) s -= Lx[q] * x[Li[q]];
    x[j] = s / Lx[Lp[j]];
  }
}
