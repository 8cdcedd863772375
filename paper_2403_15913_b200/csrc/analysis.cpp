// Host-side symbolic analysis ("symbolic analysis ...
// computed once and refactorized efficiently if the sparsity pattern remains the same").
//
//   K pattern     = pattern(W) ∪ pattern(G^T G) ∪ pattern(H^T H) ∪ diag
//   ordering      = nested dissection of DESIGN.md §5 (reading R8), or the caller's perm
//   etree         = Liu's algorithm with path compression
//   L pattern     = row-subtree traversal (rows of L_i* = the row subtree of i)
//   supernodes    = fundamental supernodes of the postordered etree (internal, R11)
//   maps          = K slot -> panel position, J^T D J product terms per slot,
//                   multifrontal child lists with relative row maps, level schedule
//
// Independent of oracle/csrc (different algorithms and data structures).
#include "analysis.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "../../include/ckkt.h"

namespace ckkt {

const AmalgamationParams& amalgamation_params() {
  static AmalgamationParams P = [] {
    AmalgamationParams p;
    if (const char* e = getenv("CKKT_NRELAX")) {  // tuning experiments: "n0,n1,n2,z0,z1,z2,maxw" or "0"
      if (std::string(e) == "0") p.enabled = false;
      else sscanf(e, "%d,%d,%d,%lf,%lf,%lf,%d", &p.nrelax0, &p.nrelax1, &p.nrelax2, &p.zrelax0, &p.zrelax1,
                  &p.zrelax2, &p.max_width);
    }
    return p;
  }();
  return P;
}

// ----------------------------------------------------------------------------
// ordering
// ----------------------------------------------------------------------------
namespace {

struct NDState {
  int n;
  const std::vector<int32_t>& xadj;
  const std::vector<int32_t>& adj;
  int leaf;
  std::vector<int32_t> label, visit, loc;
  int setid = 0, version = 0;
  std::vector<int32_t> out;
  bool too_big = false;

  NDState(int n_, const std::vector<int32_t>& x, const std::vector<int32_t>& a, int lf)
      : n(n_), xadj(x), adj(a), leaf(lf), label(n_, 0), visit(n_, 0), loc(n_, -1) {
    out.reserve(n_);
  }

  // BFS level sets of G[label == lab] from r; each level sorted ascending.
  void bfs(int lab, int r, std::vector<std::vector<int32_t>>& levels) {
    levels.clear();
    int ver = ++version;
    std::vector<int32_t> cur{r}, nxt;
    visit[r] = ver;
    while (!cur.empty()) {
      nxt.clear();
      for (int v : cur)
        for (int p = xadj[v]; p < xadj[v + 1]; ++p) {
          int a = adj[p];
          if (label[a] == lab && visit[a] != ver) {
            visit[a] = ver;
            nxt.push_back(a);
          }
        }
      std::sort(cur.begin(), cur.end());
      levels.push_back(cur);
      cur.swap(nxt);
    }
  }

  int deg_in(int lab, int v) const {
    int d = 0;
    for (int p = xadj[v]; p < xadj[v + 1]; ++p) d += (label[adj[p]] == lab);
    return d;
  }

  // exact minimum degree on the elimination graph of G[C], bitset rows; ties -> smaller index
  void md(const std::vector<int32_t>& C) {
    const int k = (int)C.size();
    if (k == 0) return;
    if (k > 32768) { too_big = true; return; }
    const int words = (k + 63) / 64;
    std::vector<uint64_t> B((size_t)k * words, 0ull);
    for (int i = 0; i < k; ++i) loc[C[i]] = i;
    for (int i = 0; i < k; ++i) {
      int v = C[i];
      for (int p = xadj[v]; p < xadj[v + 1]; ++p) {
        int l = loc[adj[p]];
        if (l >= 0 && l != i) B[(size_t)i * words + (l >> 6)] |= 1ull << (l & 63);
      }
    }
    for (int i = 0; i < k; ++i) loc[C[i]] = -1;
    std::vector<int> deg(k);
    std::vector<char> gone(k, 0);
    for (int i = 0; i < k; ++i) {
      int d = 0;
      for (int w = 0; w < words; ++w) d += __builtin_popcountll(B[(size_t)i * words + w]);
      deg[i] = d;
    }
    std::vector<int> nb;
    for (int step = 0; step < k; ++step) {
      int v = -1;
      for (int i = 0; i < k; ++i)
        if (!gone[i] && (v < 0 || deg[i] < deg[v])) v = i;
      out.push_back(C[v]);
      gone[v] = 1;
      const uint64_t* rv = &B[(size_t)v * words];
      nb.clear();
      for (int w = 0; w < words; ++w) {
        uint64_t x = rv[w];
        while (x) {
          int b = __builtin_ctzll(x);
          nb.push_back(w * 64 + b);
          x &= x - 1;
        }
      }
      for (int a : nb) {
        uint64_t* ra = &B[(size_t)a * words];
        int d = 0;
        for (int w = 0; w < words; ++w) {
          ra[w] |= rv[w];
        }
        ra[a >> 6] &= ~(1ull << (a & 63));
        ra[v >> 6] &= ~(1ull << (v & 63));
        for (int w = 0; w < words; ++w) d += __builtin_popcountll(ra[w]);
        deg[a] = d;
      }
    }
  }

  void component(std::vector<int32_t>& C) {
    if ((int)C.size() <= leaf) { md(C); return; }
    int lab = ++setid;
    for (int v : C) label[v] = lab;
    std::vector<std::vector<int32_t>> lev, lev2;
    bfs(lab, C[0], lev);
    for (;;) {
      const auto& last = lev.back();
      int x = -1, xd = 0;
      for (int v : last) {  // ascending; strict improvement keeps the smaller index on ties
        int d = deg_in(lab, v);
        if (x < 0 || d < xd) { x = v; xd = d; }
      }
      bfs(lab, x, lev2);
      if (lev2.size() > lev.size()) lev.swap(lev2);
      else break;
    }
    const int h = (int)lev.size() - 1;
    if (h < 2) { md(C); return; }
    const int ilo = std::max(1, h / 3), ihi = std::min(h - 1, h - h / 3);
    int bi = -1;
    for (int i = ilo; i <= ihi; ++i) {
      if (bi < 0) { bi = i; continue; }
      size_t sz = lev[i].size(), bsz = lev[bi].size();
      int c = std::abs(2 * i - h), bc = std::abs(2 * bi - h);
      if (sz < bsz || (sz == bsz && c < bc)) bi = i;
    }
    std::vector<int32_t> S = lev[bi];  // sorted
    std::vector<int32_t> rest;
    rest.reserve(C.size() - S.size());
    std::set_difference(C.begin(), C.end(), S.begin(), S.end(), std::back_inserter(rest));
    lev.clear(); lev2.clear();
    rec(rest);
    out.insert(out.end(), S.begin(), S.end());
  }

  void rec(std::vector<int32_t>& V) {
    if (V.empty()) return;
    int lab = ++setid;
    for (int v : V) label[v] = lab;
    int ver = ++version;
    std::vector<std::vector<int32_t>> comps;
    std::vector<int32_t> stack;
    for (int v : V) {
      if (visit[v] == ver) continue;
      std::vector<int32_t> comp;
      stack.assign(1, v);
      visit[v] = ver;
      while (!stack.empty()) {
        int x = stack.back();
        stack.pop_back();
        comp.push_back(x);
        for (int p = xadj[x]; p < xadj[x + 1]; ++p) {
          int a = adj[p];
          if (label[a] == lab && visit[a] != ver) { visit[a] = ver; stack.push_back(a); }
        }
      }
      std::sort(comp.begin(), comp.end());
      comps.push_back(std::move(comp));
    }
    for (auto& c : comps) {
      if (too_big) return;
      component(c);
    }
  }
};

// Liu's elimination tree of a lower CSC pattern given its row lists (strictly lower part).
void etree_liu(int n, const std::vector<int64_t>& rp, const std::vector<int32_t>& rc, std::vector<int32_t>& parent) {
  parent.assign(n, -1);
  std::vector<int32_t> anc(n, -1);
  for (int i = 0; i < n; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      int j = rc[p];
      while (j != -1 && j < i) {
        int t = anc[j];
        anc[j] = i;
        if (t == -1) parent[j] = i;
        j = t;
      }
    }
  }
}

// row lists of the strictly lower part of a lower CSC (cols ascending per row)
void row_lists(int n, const std::vector<int64_t>& cp, const std::vector<int32_t>& ri, std::vector<int64_t>& rp,
               std::vector<int32_t>& rc) {
  rp.assign(n + 1, 0);
  for (int j = 0; j < n; ++j)
    for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
      if (ri[p] > j) rp[ri[p] + 1]++;
  for (int i = 0; i < n; ++i) rp[i + 1] += rp[i];
  rc.resize(rp[n]);
  std::vector<int64_t> nx(rp.begin(), rp.end() - 1);
  for (int j = 0; j < n; ++j)
    for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
      if (ri[p] > j) rc[nx[ri[p]]++] = j;
}

// row-subtree traversal: column counts and (optionally) the L pattern, rows ascending
void row_subtrees(int n, const std::vector<int64_t>& rp, const std::vector<int32_t>& rc,
                  const std::vector<int32_t>& parent, std::vector<int32_t>& cc, std::vector<int64_t>* Lp,
                  std::vector<int32_t>* Li) {
  std::vector<int32_t> mark(n, -1);
  cc.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    mark[i] = i;
    cc[i]++;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      for (int j = rc[p]; mark[j] != i; j = parent[j]) { mark[j] = i; cc[j]++; }
  }
  if (!Lp) return;
  Lp->assign(n + 1, 0);
  for (int j = 0; j < n; ++j) (*Lp)[j + 1] = (*Lp)[j] + cc[j];
  Li->resize((*Lp)[n]);
  std::vector<int64_t> nx(Lp->begin(), Lp->end() - 1);
  std::fill(mark.begin(), mark.end(), -1);
  for (int i = 0; i < n; ++i) {
    mark[i] = i;
    (*Li)[nx[i]++] = i;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      for (int j = rc[p]; mark[j] != i; j = parent[j]) { mark[j] = i; (*Li)[nx[j]++] = i; }
  }
}

// lower CSC of P K P^T from sorted unique lower pairs (original indices) and iperm (old -> new)
void permuted_csc(int n, const std::vector<int64_t>& kpairs, const std::vector<int32_t>& iperm,
                  std::vector<int64_t>& cp, std::vector<int32_t>& ri) {
  cp.assign(n + 1, 0);
  for (int64_t key : kpairs) {
    int i = iperm[key / n], j = iperm[key % n];
    cp[std::min(i, j) + 1]++;
  }
  for (int j = 0; j < n; ++j) cp[j + 1] += cp[j];
  ri.resize(cp[n]);
  std::vector<int64_t> nx(cp.begin(), cp.end() - 1);
  for (int64_t key : kpairs) {
    int i = iperm[key / n], j = iperm[key % n];
    ri[nx[std::min(i, j)]++] = std::max(i, j);
  }
  for (int j = 0; j < n; ++j) std::sort(ri.begin() + cp[j], ri.begin() + cp[j + 1]);
}

int64_t find_slot(const std::vector<int64_t>& cp, const std::vector<int32_t>& ri, int i, int j) {
  // slot of (i, j), i >= j, in the lower CSC
  auto b = ri.begin() + cp[j], e = ri.begin() + cp[j + 1];
  auto it = std::lower_bound(b, e, i);
  if (it == e || *it != i) return -1;
  return it - ri.begin();
}

}  // namespace

std::vector<int32_t> nd_order(int n, const std::vector<int32_t>& xadj, const std::vector<int32_t>& adj, int leaf) {
  NDState st(n, xadj, adj, std::max(1, leaf));
  std::vector<int32_t> V(n);
  std::iota(V.begin(), V.end(), 0);
  st.rec(V);
  if (st.too_big || (int)st.out.size() != n) return {};
  return st.out;
}

std::string analyze(const Pattern& p, int leaf, const int32_t* user_perm, Analysis& A, int& code) {
  code = CKKT_OK;
  const int n = p.n;
  A.pat = p;
  A.n = n;
  if (n <= 0 || p.me < 0 || p.mi < 0) { code = CKKT_INVALID_ARG; return "bad dimensions"; }
  // ---- validate pattern
  for (size_t e = 0; e < p.w_row.size(); ++e) {
    int r = p.w_row[e], c = p.w_col[e];
    if (r < 0 || r >= n || c < 0 || c > r) { code = CKKT_PATTERN_ERROR; return "W entry outside the lower triangle"; }
  }
  auto check_csr = [&](int m, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci) -> bool {
    if ((int)rp.size() != m + 1 || rp[0] != 0) return false;
    for (int r = 0; r < m; ++r) {
      if (rp[r + 1] < rp[r]) return false;
      for (int q = rp[r]; q < rp[r + 1]; ++q) {
        if (ci[q] < 0 || ci[q] >= n) return false;
        if (q > rp[r] && ci[q] <= ci[q - 1]) return false;
      }
    }
    return (int64_t)ci.size() == rp[m];
  };
  if (!check_csr(p.me, p.g_rowptr, p.g_col)) { code = CKKT_PATTERN_ERROR; return "G CSR malformed"; }
  if (!check_csr(p.mi, p.h_rowptr, p.h_col)) { code = CKKT_PATTERN_ERROR; return "H CSR malformed"; }

  // ---- K pattern: sorted unique lower pairs (i >= j), original indices
  std::vector<int64_t>& kp = A.kpairs;
  kp.clear();
  int64_t est = (int64_t)p.w_row.size() + n;
  auto count_pairs = [&](const std::vector<int32_t>& rp) {
    for (size_t r = 0; r + 1 < rp.size(); ++r) { int64_t k = rp[r + 1] - rp[r]; est += k * (k - 1) / 2; }
  };
  count_pairs(p.g_rowptr);
  count_pairs(p.h_rowptr);
  kp.reserve(est);
  for (int i = 0; i < n; ++i) kp.push_back((int64_t)i * n + i);
  for (size_t e = 0; e < p.w_row.size(); ++e) kp.push_back((int64_t)p.w_row[e] * n + p.w_col[e]);
  auto add_pairs = [&](int m, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci) {
    for (int r = 0; r < m; ++r)
      for (int a = rp[r]; a < rp[r + 1]; ++a)
        for (int b = rp[r]; b < a; ++b) kp.push_back((int64_t)ci[a] * n + ci[b]);  // ci[a] > ci[b]
  };
  add_pairs(p.me, p.g_rowptr, p.g_col);
  add_pairs(p.mi, p.h_rowptr, p.h_col);
  std::sort(kp.begin(), kp.end());
  kp.erase(std::unique(kp.begin(), kp.end()), kp.end());
  // adjacency (no self loops), ascending
  A.xadj.assign(n + 1, 0);
  for (int64_t key : kp) {
    int i = key / n, j = key % n;
    if (i != j) { A.xadj[i + 1]++; A.xadj[j + 1]++; }
  }
  for (int i = 0; i < n; ++i) A.xadj[i + 1] += A.xadj[i];
  A.adj.resize(A.xadj[n]);
  {
    std::vector<int32_t> nx(A.xadj.begin(), A.xadj.end() - 1);
    for (int64_t key : kp) {
      int i = key / n, j = key % n;
      if (i != j) { A.adj[nx[i]++] = j; A.adj[nx[j]++] = i; }
    }
    for (int i = 0; i < n; ++i) std::sort(A.adj.begin() + A.xadj[i], A.adj.begin() + A.xadj[i + 1]);
  }

  // ---- ordering
  if (user_perm) {
    A.perm.assign(user_perm, user_perm + n);
    std::vector<char> seen(n, 0);
    for (int k = 0; k < n; ++k) {
      if (A.perm[k] < 0 || A.perm[k] >= n || seen[A.perm[k]]) { code = CKKT_INVALID_ARG; return "perm is not a permutation"; }
      seen[A.perm[k]] = 1;
    }
  } else {
    A.perm = nd_order(n, A.xadj, A.adj, leaf);
    if ((int)A.perm.size() != n) { code = CKKT_INVALID_ARG; return "ordering failed (minimum-degree block too large; lower leaf)"; }
  }
  std::vector<int32_t> iperm(n);
  for (int k = 0; k < n; ++k) iperm[A.perm[k]] = k;

  // ---- exported symbolic: etree and column counts for perm
  {
    std::vector<int64_t> cp, rp;
    std::vector<int32_t> ri, rc;
    permuted_csc(n, kp, iperm, cp, ri);
    row_lists(n, cp, ri, rp, rc);
    etree_liu(n, rp, rc, A.parent);
    row_subtrees(n, rp, rc, A.parent, A.colcount, nullptr, nullptr);
    A.nnz_l = 0;
    A.flops = 0.0;
    for (int j = 0; j < n; ++j) { A.nnz_l += A.colcount[j]; A.flops += (double)A.colcount[j] * A.colcount[j]; }
  }

  // ---- postorder of the etree (children ascending) -> internal ordering perm2
  std::vector<int32_t> post;
  post.reserve(n);
  {
    std::vector<int32_t> head(n, -1), next(n, -1);
    for (int j = n - 1; j >= 0; --j)
      if (A.parent[j] >= 0) { next[j] = head[A.parent[j]]; head[A.parent[j]] = j; }
    std::vector<int32_t> stack;
    for (int r = 0; r < n; ++r) {
      if (A.parent[r] != -1) continue;
      stack.push_back(r);
      while (!stack.empty()) {
        int v = stack.back();
        if (head[v] >= 0) {  // descend into the next unvisited child
          int c = head[v];
          head[v] = next[c];
          stack.push_back(c);
        } else {
          post.push_back(v);
          stack.pop_back();
        }
      }
    }
  }
  A.perm2.resize(n);
  A.iperm2.resize(n);
  for (int k = 0; k < n; ++k) A.perm2[k] = A.perm[post[k]];
  for (int k = 0; k < n; ++k) A.iperm2[A.perm2[k]] = k;

  // ---- internal symbolic
  std::vector<int64_t> Lp2;
  std::vector<int32_t> Li2;
  {
    std::vector<int64_t> rp;
    std::vector<int32_t> rc;
    permuted_csc(n, kp, A.iperm2, A.kp, A.ki);
    row_lists(n, A.kp, A.ki, rp, rc);
    etree_liu(n, rp, rc, A.parent2);
    row_subtrees(n, rp, rc, A.parent2, A.colcount2, &Lp2, &Li2);
  }
  // ---- fundamental supernodes (fs*), then relaxed amalgamation into the internal supernodes
  std::vector<int32_t> fsfirst, fsof(n), fsparent;
  {
    std::vector<int32_t> nchild(n, 0);
    for (int j = 0; j < n; ++j)
      if (A.parent2[j] >= 0) nchild[A.parent2[j]]++;
    for (int j = 0; j < n; ++j) {
      bool merge = j > 0 && A.parent2[j - 1] == j && A.colcount2[j - 1] == A.colcount2[j] + 1 && nchild[j] == 1;
      if (!merge) fsfirst.push_back(j);
      fsof[j] = (int)fsfirst.size() - 1;
    }
    fsfirst.push_back(n);
    const int nf = (int)fsfirst.size() - 1;
    fsparent.assign(nf, -1);
    for (int s = 0; s < nf; ++s) {
      int last = fsfirst[s + 1] - 1;
      if (A.parent2[last] >= 0) fsparent[s] = fsof[A.parent2[last]];
    }
  }
  // Relaxed amalgamation (R11: internal storage only; padded entries are exact zeros).  In
  // postorder the group ending right before supernode s is s's last child; it is merged into s
  // when the merged panel stays narrow or gains few explicit zeros.
  {
    const int nf = (int)fsfirst.size() - 1;
    std::vector<int32_t> gfirst, gtop;   // group first column, top fundamental supernode
    std::vector<double> gzeros;
    std::vector<int32_t> group_of_f(nf);
    const AmalgamationParams& P = amalgamation_params();
    for (int s = 0; s < nf; ++s) {
      const int ws = fsfirst[s + 1] - fsfirst[s];
      const int64_t ms = A.colcount2[fsfirst[s]];
      bool merged = false;
      if (!gfirst.empty() && P.enabled) {
        int g = (int)gfirst.size() - 1;
        int top = gtop[g];
        if (fsparent[top] == s && fsfirst[top + 1] == fsfirst[s]) {
          const int wg = fsfirst[s] - gfirst[g];
          const int64_t mg = wg + (A.colcount2[fsfirst[top]] - (fsfirst[top + 1] - fsfirst[top]));  // rows of group
          const int W = wg + ws;
          const double newz = gzeros[g] + (double)wg * (double)(wg + ms - mg);
          const double total = (double)W * (wg + ms) - (double)W * (W - 1) / 2.0;  // lower-trapezoid entries
          const double frac = newz / total;
          bool ok = W <= P.max_width &&
                    (W <= P.nrelax0 || (W <= P.nrelax1 && frac < P.zrelax0) || (W <= P.nrelax2 && frac < P.zrelax1) ||
                     frac < P.zrelax2);
          if (ok) {
            gtop[g] = s;
            gzeros[g] = newz;
            group_of_f[s] = g;
            merged = true;
          }
        }
      }
      if (!merged) {
        gfirst.push_back(fsfirst[s]);
        gtop.push_back(s);
        gzeros.push_back(0.0);
        group_of_f[s] = (int)gfirst.size() - 1;
      }
    }
    // final supernodes: groups split into chunks of at most MAXW columns (a chunk's rows are the
    // suffix of the group's rows starting at its first column; chunk k's parent is chunk k+1)
    constexpr int MAXW = 64;
    std::vector<int32_t> sf, stopf;  // first column, top fundamental supernode of the owning group
    for (size_t g = 0; g < gfirst.size(); ++g) {
      const int gend = fsfirst[gtop[g] + 1];
      for (int c0 = gfirst[g]; c0 < gend; c0 += MAXW) {
        sf.push_back(c0);
        stopf.push_back(gtop[g]);
      }
    }
    A.ns = (int)sf.size();
    A.sfirst = sf;
    A.sfirst.push_back(n);
    A.snode_of.resize(n);
    for (int s2 = 0; s2 < A.ns; ++s2)
      for (int j = A.sfirst[s2]; j < A.sfirst[s2 + 1]; ++j) A.snode_of[j] = s2;
    A.srowptr.assign(A.ns + 1, 0);
    A.pofs.assign(A.ns + 1, 0);
    for (int s2 = 0; s2 < A.ns; ++s2) {
      const int top = stopf[s2];
      const int w = A.sfirst[s2 + 1] - A.sfirst[s2];
      const int64_t m = (int64_t)(fsfirst[top] - A.sfirst[s2]) + A.colcount2[fsfirst[top]];
      A.srowptr[s2 + 1] = A.srowptr[s2] + m;
      A.pofs[s2 + 1] = A.pofs[s2] + m * w;
    }
    A.srows.resize(A.srowptr[A.ns]);
    for (int s2 = 0; s2 < A.ns; ++s2) {
      const int top = stopf[s2];
      int64_t o = A.srowptr[s2];
      for (int j = A.sfirst[s2]; j < fsfirst[top]; ++j) A.srows[o++] = j;
      if (A.sfirst[s2] <= fsfirst[top]) {
        std::copy(Li2.begin() + Lp2[fsfirst[top]], Li2.begin() + Lp2[fsfirst[top] + 1], A.srows.begin() + o);
      } else {  // chunk starting inside the top fundamental supernode: suffix of its structure
        const int skip = A.sfirst[s2] - fsfirst[top];
        std::copy(Li2.begin() + Lp2[fsfirst[top]] + skip, Li2.begin() + Lp2[fsfirst[top] + 1], A.srows.begin() + o);
      }
    }
    A.sparent.assign(A.ns, -1);
    for (int s2 = 0; s2 < A.ns; ++s2) {
      const int last = A.sfirst[s2 + 1] - 1;
      if (A.parent2[last] >= 0) A.sparent[s2] = A.snode_of[A.parent2[last]];
    }
  }
  const int ns = A.ns;
  Li2.clear();
  Li2.shrink_to_fit();
  // levels (children before parents; postorder => child index < parent index)
  A.slevel.assign(ns, 0);
  for (int s = 0; s < ns; ++s)
    if (A.sparent[s] >= 0) A.slevel[A.sparent[s]] = std::max(A.slevel[A.sparent[s]], A.slevel[s] + 1);
  A.nlevels = 0;
  for (int s = 0; s < ns; ++s) A.nlevels = std::max(A.nlevels, A.slevel[s] + 1);
  A.level_ptr.assign(A.nlevels + 1, 0);
  for (int s = 0; s < ns; ++s) A.level_ptr[A.slevel[s] + 1]++;
  for (int l = 0; l < A.nlevels; ++l) A.level_ptr[l + 1] += A.level_ptr[l];
  A.level_list.resize(ns);
  {
    std::vector<int32_t> nx(A.level_ptr.begin(), A.level_ptr.end() - 1);
    for (int s = 0; s < ns; ++s) A.level_list[nx[A.slevel[s]]++] = s;
  }
  // ---- multifrontal maps: children lists (ascending), relative positions of each supernode's
  //      off-diagonal rows inside its parent's rows, update-matrix and update-vector offsets
  {
    A.ch_ptr.assign(ns + 1, 0);
    for (int c = 0; c < ns; ++c)
      if (A.sparent[c] >= 0) A.ch_ptr[A.sparent[c] + 1]++;
    for (int s = 0; s < ns; ++s) A.ch_ptr[s + 1] += A.ch_ptr[s];
    A.ch_list.resize(A.ch_ptr[ns]);
    std::vector<int32_t> nx(A.ch_ptr.begin(), A.ch_ptr.end() - 1);
    for (int c = 0; c < ns; ++c)
      if (A.sparent[c] >= 0) A.ch_list[nx[A.sparent[c]]++] = c;
    A.uofs.assign(ns + 1, 0);
    A.vofs.assign(ns + 1, 0);
    A.relofs.assign(ns + 1, 0);
    for (int c = 0; c < ns; ++c) {
      const int64_t m = A.srowptr[c + 1] - A.srowptr[c], w = A.sfirst[c + 1] - A.sfirst[c];
      A.uofs[c + 1] = A.uofs[c] + (m - w) * (m - w);
      A.vofs[c + 1] = A.vofs[c] + (m - w);
      A.relofs[c + 1] = A.relofs[c] + (m - w);
    }
    A.relmap.resize(A.relofs[ns]);
    for (int c = 0; c < ns; ++c) {
      const int p = A.sparent[c];
      const int w = A.sfirst[c + 1] - A.sfirst[c];
      const int64_t r0 = A.srowptr[c];
      const int m = (int)(A.srowptr[c + 1] - r0);
      if (p < 0) {
        if (m != w) { code = CKKT_PATTERN_ERROR; return "internal: root supernode with off-diagonal rows"; }
        continue;
      }
      const int32_t* pr = &A.srows[A.srowptr[p]];
      const int mp = (int)(A.srowptr[p + 1] - A.srowptr[p]);
      int t = 0;
      for (int i = w; i < m; ++i) {
        const int row = A.srows[r0 + i];
        while (t < mp && pr[t] < row) ++t;
        if (t >= mp || pr[t] != row) { code = CKKT_PATTERN_ERROR; return "internal: row structure not nested"; }
        A.relmap[A.relofs[c] + (i - w)] = t;
      }
    }
  }
  // ---- condensation maps
  const int64_t nnzk = A.kp[n];
  A.kmap.resize(nnzk);
  for (int j = 0; j < n; ++j) {
    int s = A.snode_of[j];
    int f = A.sfirst[s];
    const int32_t* sr = &A.srows[A.srowptr[s]];
    const int ms = (int)(A.srowptr[s + 1] - A.srowptr[s]);
    int t = 0;
    for (int64_t k = A.kp[j]; k < A.kp[j + 1]; ++k) {
      while (t < ms && sr[t] < A.ki[k]) ++t;
      A.kmap[k] = (int32_t)((int64_t)(j - f) * ms + t);  // relative to the panel start pofs[s]
    }
  }
  // W terms
  {
    std::vector<int64_t> slot_of(p.w_row.size());
    A.wt_ptr.assign(nnzk + 1, 0);
    for (size_t e = 0; e < p.w_row.size(); ++e) {
      int i = A.iperm2[p.w_row[e]], j = A.iperm2[p.w_col[e]];
      slot_of[e] = find_slot(A.kp, A.ki, std::max(i, j), std::min(i, j));
      A.wt_ptr[slot_of[e] + 1]++;
    }
    for (int64_t k = 0; k < nnzk; ++k) A.wt_ptr[k + 1] += A.wt_ptr[k];
    A.wt_idx.resize(A.wt_ptr[nnzk]);
    std::vector<int64_t> nx(A.wt_ptr.begin(), A.wt_ptr.end() - 1);
    for (size_t e = 0; e < p.w_row.size(); ++e) A.wt_idx[nx[slot_of[e]]++] = (int32_t)e;
    A.w_row2.resize(p.w_row.size());
    A.w_col2.resize(p.w_row.size());
    for (size_t e = 0; e < p.w_row.size(); ++e) { A.w_row2[e] = A.iperm2[p.w_row[e]]; A.w_col2[e] = A.iperm2[p.w_col[e]]; }
  }
  A.dslot.resize(n);
  for (int j = 0; j < n; ++j) A.dslot[j] = (int32_t)A.kp[j];  // diagonal = first row of column j
  // J^T D J product terms
  {
    std::vector<int64_t> slots;
    std::vector<int32_t> ta, tb, tr;
    auto gen = [&](int m, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci, int roff) {
      for (int r = 0; r < m; ++r)
        for (int a = rp[r]; a < rp[r + 1]; ++a)
          for (int b = rp[r]; b <= a; ++b) {
            int i = A.iperm2[ci[a]], j = A.iperm2[ci[b]];
            slots.push_back(find_slot(A.kp, A.ki, std::max(i, j), std::min(i, j)));
            ta.push_back(a);
            tb.push_back(b);
            tr.push_back(r + roff);
          }
    };
    gen(p.me, p.g_rowptr, p.g_col, 0);
    gen(p.mi, p.h_rowptr, p.h_col, p.me);
    A.jt_ptr.assign(nnzk + 1, 0);
    for (int64_t s : slots) A.jt_ptr[s + 1]++;
    for (int64_t k = 0; k < nnzk; ++k) A.jt_ptr[k + 1] += A.jt_ptr[k];
    A.jt_a.resize(slots.size());
    A.jt_b.resize(slots.size());
    A.jt_r.resize(slots.size());
    std::vector<int64_t> nx(A.jt_ptr.begin(), A.jt_ptr.end() - 1);
    for (size_t t = 0; t < slots.size(); ++t) {
      int64_t o = nx[slots[t]]++;
      A.jt_a[o] = ta[t];
      A.jt_b[o] = tb[t];
      A.jt_r[o] = tr[t];
    }
  }
  // transposed J by internal column, G and H columns in internal order
  auto transpose = [&](int m, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci, std::vector<int32_t>& tp,
                       std::vector<int32_t>& te, std::vector<int32_t>& tr, std::vector<int32_t>& col2) {
    tp.assign(n + 1, 0);
    col2.resize(ci.size());
    for (size_t e = 0; e < ci.size(); ++e) { col2[e] = A.iperm2[ci[e]]; tp[col2[e] + 1]++; }
    for (int j = 0; j < n; ++j) tp[j + 1] += tp[j];
    te.resize(ci.size());
    tr.resize(ci.size());
    std::vector<int32_t> nx(tp.begin(), tp.end() - 1);
    for (int r = 0; r < m; ++r)
      for (int e = rp[r]; e < rp[r + 1]; ++e) {
        int o = nx[col2[e]]++;
        te[o] = e;
        tr[o] = r;
      }
  };
  transpose(p.me, p.g_rowptr, p.g_col, A.gt_ptr, A.gt_e, A.gt_r, A.g_col2);
  transpose(p.mi, p.h_rowptr, p.h_col, A.ht_ptr, A.ht_e, A.ht_r, A.h_col2);
  return "";
}

void export_l_pattern(const Analysis& A, std::vector<int64_t>& Lp, std::vector<int32_t>& Li) {
  const int n = A.n;
  std::vector<int32_t> iperm(n);
  for (int k = 0; k < n; ++k) iperm[A.perm[k]] = k;
  std::vector<int64_t> cp, rp;
  std::vector<int32_t> ri, rc, cc;
  permuted_csc(n, A.kpairs, iperm, cp, ri);
  row_lists(n, cp, ri, rp, rc);
  row_subtrees(n, rp, rc, A.parent, cc, &Lp, &Li);
}

}  // namespace ckkt
