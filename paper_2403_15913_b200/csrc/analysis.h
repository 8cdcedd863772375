// Host-side symbolic analysis of the condensed KKT pattern.
// Independent of oracle/ (no shared code); the ordering follows DESIGN.md §5.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace ckkt {

struct Pattern {
  int n = 0, me = 0, mi = 0;
  std::vector<int32_t> w_row, w_col;
  std::vector<int32_t> g_rowptr, g_col, h_rowptr, h_col;
};

// Result of the analysis.  "spec" arrays are w.r.t. the exported ordering perm
// (bit-exact contract); the "internal" arrays use perm2 = perm ∘ postorder,
// which has the same fill and contiguous supernodes (reading R11).
struct Analysis {
  Pattern pat;
  int n = 0;
  // K pattern as sorted unique lower pairs (original indices): key = i * n + j, i >= j
  std::vector<int64_t> kpairs;
  // adjacency of K without self loops (original indices), lists ascending
  std::vector<int32_t> xadj, adj;
  // exported ordering and its symbolic results
  std::vector<int32_t> perm, parent, colcount;
  int64_t nnz_l = 0;
  double flops = 0.0;  // sum colcount^2
  // internal ordering
  std::vector<int32_t> perm2, iperm2;
  std::vector<int64_t> kp;      // internal lower CSC of P2 K P2^T: column pointers [n+1]
  std::vector<int32_t> ki;      // row indices
  std::vector<int32_t> parent2, colcount2;
  // supernodes (internal order): columns [sfirst[s], sfirst[s+1])
  int ns = 0;
  std::vector<int32_t> sfirst, snode_of, sparent, slevel;
  std::vector<int64_t> srowptr;  // row structure of s: srows[srowptr[s] .. srowptr[s+1])
  std::vector<int32_t> srows;
  std::vector<int64_t> pofs;     // panel offsets (column-major m_s x w_s), [ns+1]
  int nlevels = 0;
  std::vector<int32_t> level_ptr, level_list;  // supernodes grouped by level (bottom-up)
  // multifrontal structure: children of s = ch_list[ch_ptr[s] .. ch_ptr[s+1]) (ascending);
  // relmap[relofs[c] + i] = position in srows[parent(c)] of the off-diagonal row w_c + i of c;
  // update matrix U_c ((m_c-w_c)^2, column-major) at uofs[c]; update vector (m_c-w_c) at vofs[c]
  std::vector<int32_t> ch_ptr, ch_list;
  std::vector<int64_t> relofs, uofs, vofs;
  std::vector<int32_t> relmap;
  // condensation: per internal K slot k (CSC order)
  std::vector<int32_t> kmap;     // position inside the instance's panel storage
  std::vector<int64_t> wt_ptr;   // W entries summed into slot k
  std::vector<int32_t> wt_idx;
  std::vector<int32_t> dslot;    // [n] slot of the diagonal of internal column j
  std::vector<int64_t> jt_ptr;   // J^T D J product terms of slot k
  std::vector<int32_t> jt_a, jt_b, jt_r;  // entry indices a, b (into g or h values) and row r
                                          // (r < me: G row, weight gamma; else H row r-me, weight d_s)
  // transposed J (by internal column j): entries of G and H in column perm2[j]
  std::vector<int32_t> gt_ptr, gt_e, gt_r, ht_ptr, ht_e, ht_r;
  // G, H column indices mapped to internal order
  std::vector<int32_t> g_col2, h_col2;
  // W entries mapped to internal order, for the residual SpMV (row2 >= col2 not guaranteed)
  std::vector<int32_t> w_row2, w_col2;
};

// Relaxed supernode amalgamation (CHOLMOD-style thresholds): merge when the merged width is
// <= nrelax0, or <= nrelax1 with zero fraction < zrelax0, or <= nrelax2 with < zrelax1, or < zrelax2.
struct AmalgamationParams {
  bool enabled = true;
  int nrelax0 = 4, nrelax1 = 16, nrelax2 = 48;
  double zrelax0 = 0.8, zrelax1 = 0.1, zrelax2 = 0.05;
  int max_width = 64;
};
const AmalgamationParams& amalgamation_params();

// Returns "" on success, else an error message; code receives a ckkt_status value.
std::string analyze(const Pattern& p, int leaf, const int32_t* user_perm, Analysis& A, int& code);

// Serialized analysis (the symbolic analysis depends on the pattern only and can be computed
// once, offline, and reused).  The blob starts with a header (magic, version, the pattern's FNV-1a hash,
// leaf, whether a caller ordering was used, amalgamation parameters) followed by every array of the
// Analysis except the pattern itself, which load_analysis takes from the caller and checks by hash.
uint64_t pattern_hash(const Pattern& p);
size_t analysis_blob_size(const Analysis& A);
void save_analysis(const Analysis& A, int leaf, bool user_perm, char* out);  // out: analysis_blob_size bytes
// Returns "" on success; code receives CKKT_INVALID_ARG for a blob of another pattern / settings.
std::string load_analysis(const Pattern& p, int leaf, bool user_perm, const char* blob, size_t size, Analysis& A,
                          int& code);

// Exact L pattern for the exported ordering (computed on demand).
void export_l_pattern(const Analysis& A, std::vector<int64_t>& Lp, std::vector<int32_t>& Li);

// Nested-dissection ordering of DESIGN.md §5 (exposed for testing).
std::vector<int32_t> nd_order(int n, const std::vector<int32_t>& xadj, const std::vector<int32_t>& adj, int leaf);

}  // namespace ckkt
