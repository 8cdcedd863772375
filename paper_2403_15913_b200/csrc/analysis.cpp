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
#include <atomic>
#include <chrono>
#include <functional>
#include <thread>
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

// host threads of the analysis (CKKT_THREADS, default: the hardware concurrency, at most 64); every
// parallel step below produces exactly the arrays of the sequential algorithm
static int analysis_threads() {
  const int t = [] {
    if (const char* e = getenv("CKKT_THREADS")) return std::max(1, atoi(e));
    const unsigned h = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(h, 64u));
  }();
  return t;
}

// run f(i) for i in [0, count) on the analysis threads (dynamic assignment; f must be thread safe)
static void parallel_for(int64_t count, const std::function<void(int64_t, int)>& f) {
  const int T = (int)std::min<int64_t>(analysis_threads(), std::max<int64_t>(count, 1));
  if (T <= 1) {
    for (int64_t i = 0; i < count; ++i) f(i, 0);
    return;
  }
  std::atomic<int64_t> next(0);
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (int64_t i; (i = next.fetch_add(1)) < count;) f(i, t);
    });
  for (auto& x : th) x.join();
}

// ----------------------------------------------------------------------------
// ordering
// ----------------------------------------------------------------------------
namespace {

// Relaxed atomic accesses to the shared label / visit tags: concurrent splits work on disjoint vertex
// sets and only READ foreign vertices' labels (every tag is drawn once from one atomic counter, so a
// foreign tag never equals the reader's), so relaxed atomics suffice.
inline int32_t ald(const int32_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
inline void ast(int32_t* p, int32_t v) { __atomic_store_n(p, v, __ATOMIC_RELAXED); }

struct NDGraph {
  const std::vector<int32_t>& xadj;
  const std::vector<int32_t>& adj;
  int32_t *label, *visit;
  std::atomic<int32_t>* tags;
  int tag() const { return tags->fetch_add(1) + 1; }

  // BFS level sets of G[label == lab] from r, flat: level l = verts[lev[l] .. lev[l+1]), each sorted
  // ascending (one allocation per BFS instead of one per level)
  struct Levels {
    std::vector<int32_t> verts;
    std::vector<int64_t> lev;
    int count() const { return (int)lev.size() - 1; }
    int64_t size(int l) const { return lev[l + 1] - lev[l]; }
  };
  void bfs(int lab, int r, Levels& L) const {
    L.verts.clear();
    L.lev.assign(1, 0);
    const int ver = tag();
    visit[r] = ver;
    L.verts.push_back(r);
    int64_t b = 0;
    while (b < (int64_t)L.verts.size()) {
      const int64_t e = (int64_t)L.verts.size();
      for (int64_t q = b; q < e; ++q) {
        const int v = L.verts[q];
        for (int p = xadj[v]; p < xadj[v + 1]; ++p) {
          const int a = adj[p];
          if (ald(label + a) == lab && visit[a] != ver) {
            visit[a] = ver;
            L.verts.push_back(a);
          }
        }
      }
      std::sort(L.verts.begin() + b, L.verts.begin() + e);
      L.lev.push_back(e);
      b = e;
    }
  }

  int deg_in(int lab, int v) const {
    int d = 0;
    for (int p = xadj[v]; p < xadj[v + 1]; ++p) d += (ald(label + adj[p]) == lab);
    return d;
  }

  // connected components of G[V] (V ascending), each sorted, in order of their smallest vertex
  void components(const std::vector<int32_t>& V, std::vector<std::vector<int32_t>>& comps) const {
    comps.clear();
    if (V.empty()) return;
    const int lab = tag();
    for (int v : V) ast(label + v, lab);
    const int ver = tag();
    std::vector<int32_t> stack;
    for (int v : V) {
      if (visit[v] == ver) continue;
      std::vector<int32_t> comp;
      stack.assign(1, v);
      visit[v] = ver;
      while (!stack.empty()) {
        const int x = stack.back();
        stack.pop_back();
        comp.push_back(x);
        for (int p = xadj[x]; p < xadj[x + 1]; ++p) {
          const int a = adj[p];
          if (ald(label + a) == lab && visit[a] != ver) {
            visit[a] = ver;
            stack.push_back(a);
          }
        }
      }
      std::sort(comp.begin(), comp.end());
      comps.push_back(std::move(comp));
    }
  }

  // one nested-dissection step on the connected component C (|C| > leaf): the separator S (sorted) and
  // the components of C \ S; returns false when C is to be ordered by minimum degree instead (h < 2)
  bool split(const std::vector<int32_t>& C, std::vector<int32_t>& S, std::vector<std::vector<int32_t>>& comps) const {
    const int lab = tag();
    for (int v : C) ast(label + v, lab);
    Levels lev, lev2;
    bfs(lab, C[0], lev);
    for (;;) {  // pseudo-peripheral vertex (George-Liu)
      const int nl = lev.count();
      int x = -1, xd = 0;
      for (int64_t q = lev.lev[nl - 1]; q < lev.lev[nl]; ++q) {  // last level, ascending; strict improvement
        const int v = lev.verts[q];                             // keeps the smaller index on ties
        const int d = deg_in(lab, v);
        if (x < 0 || d < xd) { x = v; xd = d; }
      }
      bfs(lab, x, lev2);
      if (lev2.count() > lev.count()) std::swap(lev, lev2);
      else break;
    }
    const int h = lev.count() - 1;
    if (h < 2) return false;
    const int ilo = std::max(1, h / 3), ihi = std::min(h - 1, h - h / 3);
    int bi = -1;
    for (int i = ilo; i <= ihi; ++i) {
      if (bi < 0) { bi = i; continue; }
      const int64_t sz = lev.size(i), bsz = lev.size(bi);
      const int c = std::abs(2 * i - h), bc = std::abs(2 * bi - h);
      if (sz < bsz || (sz == bsz && c < bc)) bi = i;
    }
    S.assign(lev.verts.begin() + lev.lev[bi], lev.verts.begin() + lev.lev[bi + 1]);
    std::vector<int32_t> rest;
    rest.reserve(C.size() - S.size());
    std::set_difference(C.begin(), C.end(), S.begin(), S.end(), std::back_inserter(rest));
    components(rest, comps);
    return true;
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
  parallel_for((n + 4095) / 4096, [&](int64_t c, int) {
    for (int64_t j = c * 4096; j < std::min<int64_t>(n, (c + 1) * 4096); ++j)
      std::sort(ri.begin() + cp[j], ri.begin() + cp[j + 1]);
  });
}

int64_t find_slot(const std::vector<int64_t>& cp, const std::vector<int32_t>& ri, int i, int j) {
  // slot of (i, j), i >= j, in the lower CSC
  auto b = ri.begin() + cp[j], e = ri.begin() + cp[j + 1];
  auto it = std::lower_bound(b, e, i);
  if (it == e || *it != i) return -1;
  return it - ri.begin();
}

}  // namespace

// Exact minimum degree on the elimination graph of G[C]: bitset rows, ties -> smaller
// index.  loc: scratch of n entries, all -1 on entry and on exit.
static void md_order(const std::vector<int32_t>& C, const std::vector<int32_t>& xadj, const std::vector<int32_t>& adj,
                     std::vector<int32_t>& loc, std::vector<int32_t>& out) {
  const int k = (int)C.size();
  out.clear();
  if (k == 0) return;
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
  out.reserve(k);
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
      for (int w = 0; w < words; ++w) ra[w] |= rv[w];
      ra[a >> 6] &= ~(1ull << (a & 63));
      ra[v >> 6] &= ~(1ull << (v & 63));
      for (int w = 0; w < words; ++w) d += __builtin_popcountll(ra[w]);
      deg[a] = d;
    }
  }
}

std::vector<int32_t> nd_order(int n, const std::vector<int32_t>& xadj, const std::vector<int32_t>& adj, int leaf) {
  // The ordering of DESIGN.md §5, evaluated breadth first: every nested-dissection level splits all of
  // its components in parallel (they are disjoint), the leaf blocks' minimum-degree orders are computed
  // in parallel, and the output is the in-order walk of the dissection tree (the components of C \ S in
  // order of their smallest vertex, then S) — exactly the sequence of the sequential recursion.
  leaf = std::max(1, leaf);
  std::vector<int32_t> label(n, 0), visit(n, 0);
  std::atomic<int32_t> tags(0);
  NDGraph G{xadj, adj, label.data(), visit.data(), &tags};
  struct Node {
    std::vector<int32_t> C;  // vertex set (leaf: ordered later by minimum degree)
    std::vector<int32_t> S;  // separator (split nodes)
    std::vector<int> kids;   // child components in order
    bool is_leaf = false;
  };
  std::vector<Node> nodes(1);  // node 0: the whole graph, split into its components (no separator)
  {
    std::vector<int32_t> V(n);
    std::iota(V.begin(), V.end(), 0);
    std::vector<std::vector<int32_t>> comps;
    G.components(V, comps);
    for (auto& c : comps) {
      nodes[0].kids.push_back((int)nodes.size());
      nodes.emplace_back();
      nodes.back().C = std::move(c);
    }
  }
  std::vector<int> frontier(nodes[0].kids);
  std::atomic<bool> too_big(false);
  while (!frontier.empty()) {
    const int nf = (int)frontier.size();
    std::vector<std::vector<std::vector<int32_t>>> kids(nf);
    parallel_for(nf, [&](int64_t i, int) {
      Node& nd = nodes[frontier[i]];
      if ((int)nd.C.size() <= leaf || !G.split(nd.C, nd.S, kids[i])) {
        nd.is_leaf = true;
        if (nd.C.size() > 32768) too_big = true;
      }
    });
    if (too_big) return {};
    std::vector<int> next;
    for (int i = 0; i < nf; ++i) {
      const int id = frontier[i];
      if (nodes[id].is_leaf) continue;
      std::vector<int32_t>().swap(nodes[id].C);
      for (auto& c : kids[i]) {
        const int k = (int)nodes.size();
        nodes.emplace_back();
        nodes.back().C = std::move(c);
        nodes[id].kids.push_back(k);
        next.push_back(k);
      }
    }
    frontier.swap(next);
  }
  // leaf blocks: exact minimum degree, in parallel (largest first)
  std::vector<int> lv;
  for (int i = 0; i < (int)nodes.size(); ++i)
    if (nodes[i].is_leaf) lv.push_back(i);
  std::stable_sort(lv.begin(), lv.end(), [&](int x, int y) { return nodes[x].C.size() > nodes[y].C.size(); });
  std::vector<std::vector<int32_t>> ord(nodes.size());
  std::vector<std::vector<int32_t>> loc(analysis_threads());
  parallel_for((int64_t)lv.size(), [&](int64_t i, int t) {
    if (loc[t].empty()) loc[t].assign(n, -1);
    md_order(nodes[lv[i]].C, xadj, adj, loc[t], ord[lv[i]]);
  });
  // in-order walk: kids, then the separator
  std::vector<int32_t> out;
  out.reserve(n);
  std::vector<std::pair<int, int>> st{{0, 0}};
  while (!st.empty()) {
    auto& [id, k] = st.back();
    const Node& nd = nodes[id];
    if (nd.is_leaf) {
      out.insert(out.end(), ord[id].begin(), ord[id].end());
      st.pop_back();
    } else if (k < (int)nd.kids.size()) {
      const int c = nd.kids[k++];
      st.push_back({c, 0});
    } else {
      out.insert(out.end(), nd.S.begin(), nd.S.end());
      st.pop_back();
    }
  }
  if ((int)out.size() != n) return {};
  return out;
}

std::string analyze(const Pattern& p, int leaf, const int32_t* user_perm, Analysis& A, int& code) {
  code = CKKT_OK;
  const bool verbose = getenv("CKKT_VERBOSE") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!verbose) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "ckkt analyze: %-28s %8.3f s\n", what, std::chrono::duration<double>(t - t_prev).count());
    t_prev = t;
  };
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

  // ---- K pattern = W ∪ G^T G ∪ H^T H ∪ diag: adjacency lists (ascending, no self loops) built per vertex
  //      in parallel from the rows containing it; then the sorted unique lower pairs (i >= j) row by row
  {
    auto transpose_rows = [&](int m, const std::vector<int32_t>& rp, const std::vector<int32_t>& ci,
                              std::vector<int64_t>& tp, std::vector<int32_t>& tr) {
      tp.assign(n + 1, 0);
      for (int64_t q = 0; q < rp[m]; ++q) tp[ci[q] + 1]++;
      for (int i = 0; i < n; ++i) tp[i + 1] += tp[i];
      tr.resize(tp[n]);
      std::vector<int64_t> nx(tp.begin(), tp.end() - 1);
      for (int r = 0; r < m; ++r)
        for (int q = rp[r]; q < rp[r + 1]; ++q) tr[nx[ci[q]]++] = r;
    };
    std::vector<int64_t> gtp, htp, wtp;
    std::vector<int32_t> gtr, htr, wnb;
    transpose_rows(p.me, p.g_rowptr, p.g_col, gtp, gtr);
    transpose_rows(p.mi, p.h_rowptr, p.h_col, htp, htr);
    {  // W neighbours (both triangles)
      wtp.assign(n + 1, 0);
      for (size_t e = 0; e < p.w_row.size(); ++e)
        if (p.w_row[e] != p.w_col[e]) { wtp[p.w_row[e] + 1]++; wtp[p.w_col[e] + 1]++; }
      for (int i = 0; i < n; ++i) wtp[i + 1] += wtp[i];
      wnb.resize(wtp[n]);
      std::vector<int64_t> nx(wtp.begin(), wtp.end() - 1);
      for (size_t e = 0; e < p.w_row.size(); ++e)
        if (p.w_row[e] != p.w_col[e]) { wnb[nx[p.w_row[e]]++] = p.w_col[e]; wnb[nx[p.w_col[e]]++] = p.w_row[e]; }
    }
    std::vector<std::vector<int32_t>> nbs(n);
    const int64_t CH = 4096;
    parallel_for((n + CH - 1) / CH, [&](int64_t c, int) {
      std::vector<int32_t> buf;
      for (int64_t i = c * CH; i < std::min<int64_t>(n, (c + 1) * CH); ++i) {
        buf.clear();
        for (int64_t q = wtp[i]; q < wtp[i + 1]; ++q) buf.push_back(wnb[q]);
        for (int64_t q = gtp[i]; q < gtp[i + 1]; ++q) {
          const int r = gtr[q];
          for (int t = p.g_rowptr[r]; t < p.g_rowptr[r + 1]; ++t) buf.push_back(p.g_col[t]);
        }
        for (int64_t q = htp[i]; q < htp[i + 1]; ++q) {
          const int r = htr[q];
          for (int t = p.h_rowptr[r]; t < p.h_rowptr[r + 1]; ++t) buf.push_back(p.h_col[t]);
        }
        std::sort(buf.begin(), buf.end());
        buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
        buf.erase(std::remove(buf.begin(), buf.end(), (int32_t)i), buf.end());
        nbs[i] = buf;
      }
    });
    A.xadj.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) A.xadj[i + 1] = A.xadj[i] + (int32_t)nbs[i].size();
    A.adj.resize(A.xadj[n]);
    std::vector<int64_t> kofs(n + 1, 0);  // lower pairs of row i: neighbours j < i, then (i, i)
    for (int i = 0; i < n; ++i)
      kofs[i + 1] = kofs[i] + 1 + (std::lower_bound(nbs[i].begin(), nbs[i].end(), (int32_t)i) - nbs[i].begin());
    std::vector<int64_t>& kp = A.kpairs;
    kp.resize(kofs[n]);
    parallel_for((n + CH - 1) / CH, [&](int64_t c, int) {
      for (int64_t i = c * CH; i < std::min<int64_t>(n, (c + 1) * CH); ++i) {
        std::copy(nbs[i].begin(), nbs[i].end(), A.adj.begin() + A.xadj[i]);
        int64_t o = kofs[i];
        for (int32_t j : nbs[i]) {
          if (j > i) break;
          kp[o++] = i * (int64_t)n + j;
        }
        kp[o] = i * (int64_t)n + i;
        std::vector<int32_t>().swap(nbs[i]);
      }
    });
  }
  std::vector<int64_t>& kp = A.kpairs;
  lap("K pattern + adjacency");
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
  lap("ordering");

  // ---- exported symbolic: etree and column counts for perm
  {
    std::vector<int64_t> cp, rp;
    std::vector<int32_t> ri, rc;
    permuted_csc(n, kp, iperm, cp, ri);
    row_lists(n, cp, ri, rp, rc);
    etree_liu(n, rp, rc, A.parent);
    // the column counts follow from the internal symbolic below (a postorder relabels the etree and
    // the column counts without changing them)
  }

  lap("exported symbolic");
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
  {
    std::vector<int64_t> rp;
    std::vector<int32_t> rc;
    permuted_csc(n, kp, A.iperm2, A.kp, A.ki);
    row_lists(n, A.kp, A.ki, rp, rc);
    // etree of the postordered matrix = the etree of perm relabeled by the postorder
    std::vector<int32_t> ipost(n);
    for (int k = 0; k < n; ++k) ipost[post[k]] = k;
    A.parent2.resize(n);
    for (int k = 0; k < n; ++k) A.parent2[k] = A.parent[post[k]] < 0 ? -1 : ipost[A.parent[post[k]]];
    row_subtrees(n, rp, rc, A.parent2, A.colcount2, nullptr, nullptr);  // column counts only
    A.colcount.resize(n);
    for (int k = 0; k < n; ++k) A.colcount[post[k]] = A.colcount2[k];
    A.nnz_l = 0;
    A.flops = 0.0;
    for (int j = 0; j < n; ++j) { A.nnz_l += A.colcount[j]; A.flops += (double)A.colcount[j] * A.colcount[j]; }
  }
  lap("postorder + internal symbolic");
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
    const int MAXW = std::max(1, std::min(64, P.max_width));  // (amalgamation parameter; 64 by default)
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
    // Row structures of the group tops, by a postorder merge over the fundamental-supernode tree
    // (only a fundamental supernode's first column has children outside it):
    //   below(F) = rows > last(F) of K's columns in F and of below(C) for the children C of F,
    // checked against the column counts of the row-subtree pass; the L column of first(F) is then
    // first(F)..last(F) followed by below(F).  Work and memory ~ sum of the structures, not nnz(L).
    std::vector<std::vector<int32_t>> below(nf);
    {
      std::vector<char> need(nf, 0);
      for (int s2 = 0; s2 < A.ns; ++s2) need[stopf[s2]] = 1;
      std::vector<int32_t> chead(nf, -1), cnext(nf, -1);
      for (int F = nf - 1; F >= 0; --F)
        if (fsparent[F] >= 0) { cnext[F] = chead[fsparent[F]]; chead[fsparent[F]] = F; }
      std::vector<int32_t> buf, mark(n, -1);  // mark[i] == F: row i already collected for F
      for (int F = 0; F < nf; ++F) {
        const int f0 = fsfirst[F], l = fsfirst[F + 1] - 1;
        buf.clear();
        auto add = [&](int32_t i) {
          if (i > l && mark[i] != F) {
            mark[i] = F;
            buf.push_back(i);
          }
        };
        for (int j = f0; j <= l; ++j)
          for (int64_t q = A.kp[j]; q < A.kp[j + 1]; ++q) add(A.ki[q]);
        for (int C = chead[F]; C >= 0; C = cnext[C]) {
          for (int32_t i : below[C]) add(i);
          if (!need[C]) std::vector<int32_t>().swap(below[C]);
        }
        std::sort(buf.begin(), buf.end());
        if ((int64_t)buf.size() != (int64_t)A.colcount2[f0] - (l - f0 + 1)) {
          code = CKKT_INVALID_ARG;
          return "internal error: supernodal structure disagrees with the column counts";
        }
        below[F] = buf;
      }
    }
    A.srows.resize(A.srowptr[A.ns]);
    for (int s2 = 0; s2 < A.ns; ++s2) {
      const int top = stopf[s2];
      int64_t o = A.srowptr[s2];
      // columns sfirst[s2] .. last(top) (a chunk may start inside the top fundamental supernode),
      // then the structure below the top
      for (int j = A.sfirst[s2]; j < fsfirst[top + 1]; ++j) A.srows[o++] = j;
      std::copy(below[top].begin(), below[top].end(), A.srows.begin() + o);
    }
    A.sparent.assign(A.ns, -1);
    for (int s2 = 0; s2 < A.ns; ++s2) {
      const int last = A.sfirst[s2 + 1] - 1;
      if (A.parent2[last] >= 0) A.sparent[s2] = A.snode_of[A.parent2[last]];
    }
  }
  const int ns = A.ns;
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
  lap("supernodes + levels");
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
  lap("multifrontal maps");
  // ---- condensation maps
  const int64_t nnzk = A.kp[n];
  A.kmap.resize(nnzk);
  parallel_for((n + 4095) / 4096, [&](int64_t c, int) {
    for (int j = (int)(c * 4096); j < std::min<int64_t>(n, (c + 1) * 4096); ++j) {
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
  });
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
    // product terms of slot (i, j): one per row r of G (weight gamma) or H (weight d_r) containing both
    // variables, ordered by r (G rows first) — entries a >= b of row r.  Built per K column in parallel
    // by intersecting the two variables' row lists (count pass, then fill pass).
    std::vector<int64_t> vp(n + 1, 0);  // row lists of every original variable: (row id, entry index)
    std::vector<int32_t> vr, ve;
    {
      for (int64_t q = 0; q < p.g_rowptr[p.me]; ++q) vp[p.g_col[q] + 1]++;
      for (int64_t q = 0; q < p.h_rowptr[p.mi]; ++q) vp[p.h_col[q] + 1]++;
      for (int i = 0; i < n; ++i) vp[i + 1] += vp[i];
      vr.resize(vp[n]);
      ve.resize(vp[n]);
      std::vector<int64_t> nx(vp.begin(), vp.end() - 1);
      for (int r = 0; r < p.me; ++r)
        for (int q = p.g_rowptr[r]; q < p.g_rowptr[r + 1]; ++q) { const int64_t o = nx[p.g_col[q]]++; vr[o] = r; ve[o] = q; }
      for (int r = 0; r < p.mi; ++r)
        for (int q = p.h_rowptr[r]; q < p.h_rowptr[r + 1]; ++q) {
          const int64_t o = nx[p.h_col[q]]++;
          vr[o] = p.me + r;
          ve[o] = q;
        }
    }
    auto each_term = [&](int64_t k, int j, auto&& fn) {  // terms of slot k (internal row ki[k], column j)
      const int u = A.perm2[A.ki[k]], v = A.perm2[j];     // original variables
      int64_t x = vp[u], y = vp[v];
      while (x < vp[u + 1] && y < vp[v + 1]) {
        if (vr[x] < vr[y]) ++x;
        else if (vr[x] > vr[y]) ++y;
        else {
          const int ea = std::max(ve[x], ve[y]), eb = std::min(ve[x], ve[y]);
          fn(ea, eb, vr[x]);
          ++x;
          ++y;
        }
      }
    };
    A.jt_ptr.assign(nnzk + 1, 0);
    parallel_for((n + 4095) / 4096, [&](int64_t c, int) {
      for (int j = (int)(c * 4096); j < std::min<int64_t>(n, (c + 1) * 4096); ++j)
        for (int64_t k = A.kp[j]; k < A.kp[j + 1]; ++k) {
          int64_t cnt = 0;
          each_term(k, j, [&](int, int, int) { ++cnt; });
          A.jt_ptr[k + 1] = cnt;
        }
    });
    for (int64_t k = 0; k < nnzk; ++k) A.jt_ptr[k + 1] += A.jt_ptr[k];
    A.jt_a.resize(A.jt_ptr[nnzk]);
    A.jt_b.resize(A.jt_ptr[nnzk]);
    A.jt_r.resize(A.jt_ptr[nnzk]);
    parallel_for((n + 4095) / 4096, [&](int64_t c, int) {
      for (int j = (int)(c * 4096); j < std::min<int64_t>(n, (c + 1) * 4096); ++j)
        for (int64_t k = A.kp[j]; k < A.kp[j + 1]; ++k) {
          int64_t o = A.jt_ptr[k];
          each_term(k, j, [&](int ea, int eb, int r) {
            A.jt_a[o] = ea;
            A.jt_b[o] = eb;
            A.jt_r[o] = r;
            ++o;
          });
        }
    });
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
  lap("condensation maps");
  return "";
}

// ---------------------------------------------------------------------------- serialized analysis
namespace {
constexpr char kMagic[8] = {'C', 'K', 'K', 'T', 'A', 'N', '0', '1'};
constexpr uint32_t kVersion = 2;  // bump when the Analysis layout or its algorithms change

template <class F>
void for_each_array(Analysis& A, F&& f) {  // every array of the analysis, in blob order
  f(A.kpairs); f(A.perm); f(A.parent); f(A.colcount); f(A.perm2); f(A.iperm2); f(A.kp); f(A.ki);
  f(A.parent2); f(A.colcount2); f(A.sfirst); f(A.snode_of); f(A.sparent); f(A.slevel); f(A.srowptr);
  f(A.srows); f(A.pofs); f(A.level_ptr); f(A.level_list); f(A.ch_ptr); f(A.ch_list); f(A.relofs);
  f(A.uofs); f(A.vofs); f(A.relmap); f(A.kmap); f(A.wt_ptr); f(A.wt_idx); f(A.dslot); f(A.jt_ptr);
  f(A.jt_a); f(A.jt_b); f(A.jt_r); f(A.gt_ptr); f(A.gt_e); f(A.gt_r); f(A.ht_ptr); f(A.ht_e); f(A.ht_r);
  f(A.g_col2); f(A.h_col2); f(A.w_row2); f(A.w_col2);
}

struct BlobHeader {
  char magic[8];
  uint32_t version, user_perm;
  uint64_t hash;
  int32_t leaf, n, me, mi, ns, nlevels;
  int64_t nnz_l;
  double flops;
  int32_t nrelax[3], max_width;
  double zrelax[3];
};
}  // namespace

uint64_t pattern_hash(const Pattern& p) {
  uint64_t h = 1469598103934665603ull;  // FNV-1a over the dimensions and the index arrays
  auto mix = [&](const void* d, size_t bytes) {
    const unsigned char* c = static_cast<const unsigned char*>(d);
    for (size_t i = 0; i < bytes; ++i) { h ^= c[i]; h *= 1099511628211ull; }
  };
  const int32_t dims[3] = {p.n, p.me, p.mi};
  mix(dims, sizeof(dims));
  for (const std::vector<int32_t>* v : {&p.w_row, &p.w_col, &p.g_rowptr, &p.g_col, &p.h_rowptr, &p.h_col}) {
    const uint64_t len = v->size();
    mix(&len, sizeof(len));
    if (len) mix(v->data(), len * sizeof(int32_t));
  }
  return h;
}

size_t analysis_blob_size(const Analysis& A0) {
  Analysis& A = const_cast<Analysis&>(A0);  // for_each_array only reads here
  size_t total = sizeof(BlobHeader);
  for_each_array(A, [&](auto& v) { total += sizeof(uint64_t) + v.size() * sizeof(v[0]); });
  return total;
}

void save_analysis(const Analysis& A0, int leaf, bool user_perm, char* out) {
  Analysis& A = const_cast<Analysis&>(A0);  // for_each_array only reads here
  const AmalgamationParams& ap = amalgamation_params();
  BlobHeader h{};
  std::memcpy(h.magic, kMagic, 8);
  h.version = kVersion;
  h.user_perm = user_perm ? 1u : 0u;
  h.hash = pattern_hash(A.pat);
  h.leaf = leaf;
  h.n = A.n;
  h.me = A.pat.me;
  h.mi = A.pat.mi;
  h.ns = A.ns;
  h.nlevels = A.nlevels;
  h.nnz_l = A.nnz_l;
  h.flops = A.flops;
  h.nrelax[0] = ap.enabled ? ap.nrelax0 : -1;
  h.nrelax[1] = ap.nrelax1;
  h.nrelax[2] = ap.nrelax2;
  h.max_width = ap.max_width;
  h.zrelax[0] = ap.zrelax0;
  h.zrelax[1] = ap.zrelax1;
  h.zrelax[2] = ap.zrelax2;
  char* o = out;
  std::memcpy(o, &h, sizeof(h));
  o += sizeof(h);
  for_each_array(A, [&](auto& v) {
    const uint64_t len = v.size();
    std::memcpy(o, &len, sizeof(len));
    o += sizeof(len);
    if (len) std::memcpy(o, v.data(), len * sizeof(v[0]));
    o += len * sizeof(v[0]);
  });
}

std::string load_analysis(const Pattern& p, int leaf, bool user_perm, const char* blob, size_t size, Analysis& A,
                          int& code) {
  code = CKKT_INVALID_ARG;
  BlobHeader h;
  if (!blob || size < sizeof(h)) return "blob too small";
  std::memcpy(&h, blob, sizeof(h));
  const AmalgamationParams& ap = amalgamation_params();
  if (std::memcmp(h.magic, kMagic, 8) != 0 || h.version != kVersion) return "not a ckkt analysis blob of this version";
  if (h.n != p.n || h.me != p.me || h.mi != p.mi || h.leaf != leaf || h.user_perm != (user_perm ? 1u : 0u) ||
      h.hash != pattern_hash(p))
    return "blob was analysed for another pattern or ordering";
  if (h.nrelax[0] != (ap.enabled ? ap.nrelax0 : -1) || h.nrelax[1] != ap.nrelax1 || h.nrelax[2] != ap.nrelax2 ||
      h.max_width != ap.max_width || h.zrelax[0] != ap.zrelax0 || h.zrelax[1] != ap.zrelax1 || h.zrelax[2] != ap.zrelax2)
    return "blob was analysed with other amalgamation parameters";
  const char* o = blob + sizeof(h);
  const char* e = blob + size;
  bool ok = true;
  for_each_array(A, [&](auto& v) {
    uint64_t len = 0;
    if (!ok || o + sizeof(len) > e) { ok = false; return; }
    std::memcpy(&len, o, sizeof(len));
    o += sizeof(len);
    const size_t bytes = len * sizeof(v[0]);
    if (len > size || o + bytes > e) { ok = false; return; }
    v.resize(len);
    if (len) std::memcpy(v.data(), o, bytes);
    o += bytes;
  });
  if (!ok || o != e) return "truncated or corrupt analysis blob";
  A.pat = p;
  A.n = p.n;
  A.ns = h.ns;
  A.nlevels = h.nlevels;
  A.nnz_l = h.nnz_l;
  A.flops = h.flops;
  if ((int)A.perm.size() != p.n || (int)A.sfirst.size() != A.ns + 1 || (int)A.kp.size() != p.n + 1)
    return "inconsistent analysis blob";
  code = CKKT_OK;
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
