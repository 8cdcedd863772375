// ckkt: condensed-KKT Newton-step solver — CUDA kernels (sm_100a) and the C ABI of include/ckkt.h.
//
// Per-iteration path; every step runs in the kernels below:
//   a1 k_condense        K_gamma values from W, Sigma_x, delta_x, J, D_s, gamma
//   a2 k_rhs             r~ = r1 + H^T(D_s r4 - r2) [+ gamma G^T r3]
//   a3 k_factor_*        multifrontal supernodal Cholesky (DMMA SYRK), level sched.
//   a4 k_fwd_* / k_bwd_* supernodal triangular solves, level scheduled
//   a5 CG kernels        matrix-free CG on S_gamma = G K^{-1} G^T
//   a6/a7 k_recover      dx un-permutation, ds = -r4 - H dx, dz = -r2 - D_s ds
//   a8 k_kaug_residual   rho = -r - K_aug d and componentwise backward error        (R7)
//   a9 flags             NOT_PD / minimum failing pivot
// All n-vectors on the device live in the internal elimination order (perm2).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX 3: host ranges for nsys timelines (no-ops without a tool)

#include <algorithm>
#include <array>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/ckkt.h"
#include "analysis.h"

#define CK(x)                                         \
  do {                                                \
    cudaError_t e_ = (x);                             \
    if (e_ != cudaSuccess) {                          \
      last_cuda_error = e_;                           \
      return CKKT_CUDA_ERROR;                         \
    }                                                 \
  } while (0)

static thread_local cudaError_t last_cuda_error = cudaSuccess;

// CKKT_SYNC_DEBUG=1: synchronise and check after every launch, printing the failing kernel.
static bool sync_debug() {
  static int v = getenv("CKKT_SYNC_DEBUG") ? atoi(getenv("CKKT_SYNC_DEBUG")) : 0;
  return v != 0;
}
#define DBG_SYNC(name)                                                                          \
  do {                                                                                          \
    if (sync_debug()) {                                                                         \
      cudaError_t e_ = cudaDeviceSynchronize();                                                 \
      if (e_ == cudaSuccess) e_ = cudaGetLastError();                                           \
      if (e_ != cudaSuccess) fprintf(stderr, "ckkt: kernel %s failed: %s\n", name, cudaGetErrorString(e_)); \
    }                                                                                           \
  } while (0)

// NVTX range over one ABI call (SURVEY §5 tracing: the phases show up by name in an nsys timeline)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace {

constexpr int TPB = 256;

inline unsigned nblk(int64_t n, int t = TPB) { return (unsigned)((n + t - 1) / t); }

// ------------------------------------------------------------------------------------------
// a1: condensation.  One thread per K slot of the internal lower CSC; the sum order is fixed
// by the maps (W terms, diagonal, J^T D J product terms in row order).
// ------------------------------------------------------------------------------------------
// IDX: index type of the slot pointers (int32 when every offset fits); MODE: 1 = all product terms
// are G rows (HyKKT: gamma), 2 = all are H rows (Lifted: D_s[r]), 0 = mixed (jt_r decides)
template <typename IDX, int MODE>
__global__ void k_condense(int64_t nnzk, const IDX* __restrict__ wt_ptr, const int32_t* __restrict__ wt_idx,
                           const IDX* __restrict__ jt_ptr, const int32_t* __restrict__ jt_a,
                           const int32_t* __restrict__ jt_b, const int32_t* __restrict__ jt_r,
                           const int32_t* __restrict__ kdiag, const double* __restrict__ w_val, int64_t w_nnz,
                           const double* __restrict__ g_val, int64_t g_nnz, const double* __restrict__ h_val,
                           int64_t h_nnz, const double* __restrict__ sigma, const double* __restrict__ d_s,
                           const double* __restrict__ delta, double gamma, int n, int me, int mi,
                           double* __restrict__ Kval) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (k >= nnzk) return;
  const double* w = w_val + b * w_nnz;
  const double* g = g_val + b * g_nnz;
  const double* h = h_val + b * h_nnz;
  double acc = 0.0;
#pragma unroll 4
  for (IDX t = wt_ptr[k]; t < wt_ptr[k + 1]; ++t) acc += w[wt_idx[t]];
  const int dv = kdiag[k];
  if (dv >= 0) acc += sigma[(int64_t)b * n + dv] + (delta ? delta[b] : 0.0);
#pragma unroll 4
  for (IDX t = jt_ptr[k]; t < jt_ptr[k + 1]; ++t) {
    if (MODE == 1) {
      acc += gamma * (g[jt_a[t]] * g[jt_b[t]]);
    } else {
      const int r = jt_r[t];
      if (MODE == 0 && r < me) acc += gamma * (g[jt_a[t]] * g[jt_b[t]]);
      else acc += d_s[(int64_t)b * mi + (r - me)] * (h[jt_a[t]] * h[jt_b[t]]);
    }
  }
  Kval[b * nnzk + k] = acc;
}

#include "mf_kernels.cuh"

// out[b][t] = val[b][e[t]]: a transposed copy of G or H values (one pass per refactor), so the
// column-wise products G^T v / H^T v read their values contiguously
__global__ void k_gather_t(int64_t nnz, int B, const int32_t* __restrict__ e, const double* __restrict__ val,
                           double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nnz * B) return;
  const int64_t b = t / nnz, k = t - b * nnz;
  out[t] = val[b * nnz + e[k]];
}

// out[b][k] = val[b][e[k]] with separate strides (W values in the residual's symmetric internal-row
// order), and sig[b][i] = sigma[b][perm2 i] + delta[b]: the residual then streams both contiguously
__global__ void k_gather_ws(int64_t nnz_out, int64_t nnz_in, int B, const int32_t* __restrict__ e,
                            const double* __restrict__ val, double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nnz_out * B) return;
  const int64_t b = t / nnz_out, k = t - b * nnz_out;
  out[t] = val[b * nnz_in + e[k]];
}

__global__ void k_gather_sigma(int n, const int32_t* __restrict__ perm2, const double* __restrict__ sigma,
                               const double* __restrict__ delta, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= n) return;
  out[(int64_t)b * n + i] = sigma[(int64_t)b * n + perm2[i]] + (delta ? delta[b] : 0.0);
}

// ||W||_inf per instance: max over rows of sum_j |W_ij| over the symmetric W (internal row order,
// each row summed in its fixed entry order); block maxima + atomicMax on the bit patterns of
// non-negative doubles (a maximum does not depend on the order: deterministic)
__global__ void k_w_norminf(int n, const int32_t* __restrict__ ws_ptr, const double* __restrict__ wsv,
                            int64_t ws_nnz, unsigned long long* __restrict__ out_bits) {
  __shared__ double red[TPB / 32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  double s = 0.0;
  if (i < n) {
    const double* w = wsv + b * ws_nnz;
    for (int e = ws_ptr[i]; e < ws_ptr[i + 1]; ++e) s += fabs(w[e]);
    if (s != s) s = INFINITY;
  }
  for (int o = 16; o > 0; o >>= 1) s = fmax(__shfl_down_sync(0xffffffffu, s, o), s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < TPB / 32; ++k) t = fmax(red[k], t);
    atomicMax(out_bits + b, (unsigned long long)__double_as_longlong(t));
  }
}

// fraction-to-boundary: alpha[b] = min(1, min over ds < 0 of (tau s) / (-ds)).  Grid-stride
// per instance (blockIdx.y), block minimum, then atomicMin on the bit patterns of the (non-negative)
// ratios: a minimum is order independent, so the result is bit-exact.  NaN ratios are skipped.
__global__ void k_ftb_init(int B, double* __restrict__ alpha) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) alpha[b] = 1.0;
}

__global__ void k_ftb(int64_t len, const double* __restrict__ s, const double* __restrict__ ds, double tau,
                      unsigned long long* __restrict__ alpha_bits) {
  __shared__ double red[TPB / 32];
  const int64_t b = blockIdx.y;
  double m = 1.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = ds[b * len + i];
    if (d < 0.0) {
      const double r = (tau * s[b * len + i]) / (-d);
      if (r < m) m = r;  // false for NaN
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_down_sync(0xffffffffu, m, o);
    if (t < m) m = t;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < TPB / 32; ++k)  // red[0] is this warp's own minimum
      if (red[k] < m) m = red[k];
    if (m < 1.0) atomicMin(alpha_bits + b, (unsigned long long)__double_as_longlong(m));
  }
}

__global__ void k_init_flags(int B, int* notpd, int* minpiv) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) { notpd[b] = 0; minpiv[b] = INT_MAX; }
}

__global__ void k_final_flags(int B, const int* notpd_in, const int* minpiv_in, const int32_t* perm2, int* notpd_out,
                              int* minpiv_out) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (notpd_out) notpd_out[b] = notpd_in[b];
  if (minpiv_out) minpiv_out[b] = (minpiv_in[b] == INT_MAX) ? -1 : perm2[minpiv_in[b]];
}

// ------------------------------------------------------------------------------------------
// a2: condensed rhs in internal order:  out[j] = s1*r1[perm2 j] + sum_H h (D_s r4 - r2) + gamma sum_G g r3
// (s1 = +1; r1 may be given in internal order when r1_internal != 0)
// ------------------------------------------------------------------------------------------
__global__ void k_rhs(int n, int me, int mi, const int32_t* __restrict__ perm2, const double* __restrict__ r1,
                      int r1_internal, const double* __restrict__ r2, const double* __restrict__ r3,
                      const double* __restrict__ r4, const int32_t* __restrict__ gt_ptr,
                      const int32_t* __restrict__ gt_e, const int32_t* __restrict__ gt_r,
                      const int32_t* __restrict__ ht_ptr, const int32_t* __restrict__ ht_e,
                      const int32_t* __restrict__ ht_r, const double* __restrict__ g_val, int64_t g_nnz,
                      const double* __restrict__ h_val, int64_t h_nnz, const double* __restrict__ d_s, double gamma,
                      double* __restrict__ out, const int* __restrict__ skip) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (j >= n || (skip && skip[b])) return;
  double acc = r1[(int64_t)b * n + (r1_internal ? j : perm2[j])];
  const double* h = h_val + b * h_nnz;
  for (int t = ht_ptr[j]; t < ht_ptr[j + 1]; ++t) {
    const int r = ht_r[t];
    const int64_t o = (int64_t)b * mi + r;
    acc += h[t] * (d_s[o] * r4[o] - r2[o]);
  }
  if (me > 0 && gamma != 0.0) {
    const double* g = g_val + b * g_nnz;
    double sg = 0.0;
    for (int t = gt_ptr[j]; t < gt_ptr[j + 1]; ++t) sg += g[t] * r3[(int64_t)b * me + gt_r[t]];
    acc += gamma * sg;
  }
  out[(int64_t)b * n + j] = acc;
}

// y[j] = alpha * sum_{G entries in column j} g * v[row]   (+ beta * z[j] if z)
__global__ void k_gt_spmv(int n, int me, const int32_t* __restrict__ gt_ptr, const int32_t* __restrict__ gt_e,
                          const int32_t* __restrict__ gt_r, const double* __restrict__ g_val, int64_t g_nnz,
                          const double* __restrict__ v, double alpha, const double* __restrict__ z, double beta,
                          double* __restrict__ y, const int* __restrict__ skip) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (j >= n || (skip && skip[b])) return;
  const double* g = g_val + b * g_nnz;
  double acc = 0.0;
  #pragma unroll 4
  for (int t = gt_ptr[j]; t < gt_ptr[j + 1]; ++t) acc += g[t] * v[(int64_t)b * me + gt_r[t]];
  double r = alpha * acc;
  if (z) r += beta * z[(int64_t)b * n + j];
  y[(int64_t)b * n + j] = r;
}

// y[r] = alpha * (G x)[r] + beta * z[r]
__global__ void k_g_spmv(int me, int n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col2,
                         const double* __restrict__ g_val, int64_t g_nnz, const double* __restrict__ x, double alpha,
                         const double* __restrict__ z, double beta, double* __restrict__ y,
                         const int* __restrict__ skip) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (r >= me || (skip && skip[b])) return;
  const double* g = g_val + b * g_nnz;
  double acc = 0.0;
  #pragma unroll 4
  for (int e = rowptr[r]; e < rowptr[r + 1]; ++e) acc += g[e] * x[(int64_t)b * n + col2[e]];
  double res = alpha * acc;
  if (z) res += beta * z[(int64_t)b * me + r];
  y[(int64_t)b * me + r] = res;
}

// partial dot products: part[b * nb + blockIdx.x]
__global__ void k_dot_partial(int64_t len, const double* __restrict__ a, const double* __restrict__ c,
                              double* __restrict__ part, const int* __restrict__ skip) {
  __shared__ double red[TPB / 32];
  const int b = blockIdx.y;
  double acc = 0.0;
  if (!(skip && skip[b]))
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
      acc += a[b * len + i] * c[b * len + i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < TPB / 32; ++k) t += red[k];
    part[(int64_t)b * gridDim.x + blockIdx.x] = t;
  }
}

constexpr int DOT_BLOCKS = 592;  // 4 per SM: enough loads in flight for the n-long dot products


// Fixed-order sum of a block-partials row by a whole block (TPB threads, one block per row):
// thread t adds rows t, t + TPB, ..., then a shared-memory tree.  Every thread gets the sum.
__device__ __forceinline__ double block_sum_parts(const double* __restrict__ p, int nb) {
  __shared__ double sh[TPB];
  __syncthreads();  // (sh may be reused by a previous call)
  double v = 0.0;
  for (int k = threadIdx.x; k < nb; k += TPB) v += p[k];
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = TPB / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  return sh[0];
}

// CG scalar step after q = S p:  alpha = rr / (p.q)
__global__ void k_cg_alpha(int B, const double* __restrict__ part, const double* __restrict__ rr,
                           double* __restrict__ alpha, const int* __restrict__ done, const int* __restrict__ iters,
                           const int* __restrict__ rec_enable, double* __restrict__ PQ, int krec) {
  const int b = blockIdx.x;  // one block per instance
  if (done[b]) {
    if (threadIdx.x == 0) alpha[b] = 0.0;
    return;
  }
  const double pq = block_sum_parts(part + (int64_t)b * DOT_BLOCKS, DOT_BLOCKS);
  if (threadIdx.x == 0) {
    alpha[b] = rr[b] / pq;
    if (PQ && *rec_enable && iters[b] < krec) PQ[(int64_t)iters[b] * B + b] = pq;
  }
}

__global__ void k_cg_update_xr(int me, const double* __restrict__ alpha, const double* __restrict__ p,
                               const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r,
                               const int* __restrict__ done) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= me || done[b]) return;
  const int64_t o = (int64_t)b * me + i;
  x[o] += alpha[b] * p[o];
  r[o] -= alpha[b] * q[o];
}

// rr_new from partials; convergence test ||r|| <= rtol ||b||; beta
__global__ void k_cg_beta(int B, const double* __restrict__ part, double* __restrict__ rr, const double* __restrict__ bnorm2,
                          const double* __restrict__ rtolp, double* __restrict__ beta, int* __restrict__ done,
                          int* __restrict__ iters, int* __restrict__ active) {
  const int b = blockIdx.x;  // one block per instance
  if (done[b]) {
    if (threadIdx.x == 0) beta[b] = 0.0;
    return;
  }
  const double t = block_sum_parts(part + (int64_t)b * DOT_BLOCKS, DOT_BLOCKS);
  if (threadIdx.x == 0) {
    iters[b] += 1;
    beta[b] = t / rr[b];
    rr[b] = t;
    if (sqrt(t) <= rtolp[0] * sqrt(bnorm2[b])) done[b] = 1;
    else atomicAdd(active, 1);
  }
}

__global__ void k_cg_update_p(int me, const double* __restrict__ beta, const double* __restrict__ r,
                              double* __restrict__ p, const int* __restrict__ done) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= me || done[b]) return;
  const int64_t o = (int64_t)b * me + i;
  p[o] = r[o] + beta[b] * p[o];
}

// CG init: x = 0, r = p = bvec; rr = bnorm2 = b.b (from partials); done if b == 0
__global__ void k_cg_init_scalars(int B, const double* __restrict__ part, double* __restrict__ rr,
                                  double* __restrict__ bnorm2, int* __restrict__ done, int* __restrict__ iters,
                                  const int* __restrict__ skip) {
  const int b = blockIdx.x;  // one block per instance
  const double t = block_sum_parts(part + (int64_t)b * DOT_BLOCKS, DOT_BLOCKS);
  if (threadIdx.x == 0) {
    rr[b] = t;
    bnorm2[b] = t;
    iters[b] = 0;
    done[b] = (t == 0.0) || (skip && skip[b]);
  }
}

// ---- Init-CG for the correction passes: the conjugate directions p_i of the first pass and
// q_i = S p_i are kept (up to KREC per instance); a correction pass starts from the S-orthogonal
// projection of its solution onto span{p_i}:  x0 = sum_i c_i p_i,  r0 = b - sum_i c_i q_i,
// c_i = p_i.b / p_i.q_i  (p_i.q_j = 0 for i != j by conjugacy).  Same operator, same stopping
// test ||r|| <= rtol ||b|| — only the start changes (R6).
constexpr int KREC = 32;

// store p, q and p.q of the current iteration into slot iters[b] (first pass only: *enable)
__global__ void k_cg_store(int me, int B, const double* __restrict__ p, const double* __restrict__ q,
                           const double* __restrict__ part, const int* __restrict__ iters,
                           const int* __restrict__ done, const int* __restrict__ enable, double* __restrict__ P,
                           double* __restrict__ Q, double* __restrict__ PQ) {
  if (!*enable) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (done[b]) return;
  const int k = iters[b];
  if (k >= KREC) return;
  const int64_t slot = ((int64_t)k * B + b) * me;
  if (i < me) {
    P[slot + i] = p[(int64_t)b * me + i];
    Q[slot + i] = q[(int64_t)b * me + i];
  }
}

// partial sums of p_k . b: block (x, b, k) covers a strided share of the rows of direction k
__global__ void k_rec_dots(int me, int B, const double* __restrict__ P, const double* __restrict__ bvec,
                           const int* __restrict__ nrec, const int* __restrict__ skip, double* __restrict__ part) {
  __shared__ double red[TPB / 32];
  const int b = blockIdx.y, k = blockIdx.z;
  const int nk = (skip && skip[b]) ? 0 : nrec[b];
  if (k >= nk) return;  // uniform per block
  const double* pk = P + ((int64_t)k * B + b) * me;
  const double* bb = bvec + (int64_t)b * me;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < me; i += (int64_t)gridDim.x * blockDim.x)
    acc += pk[i] * bb[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < TPB / 32; ++w) t += red[w];
    part[((int64_t)b * KREC + k) * DOT_BLOCKS + blockIdx.x] = t;
  }
}

// c_i = (p_i . b) / (p_i . q_i)
__global__ void k_rec_coef(int B, const double* __restrict__ part, const double* __restrict__ PQ,
                           const int* __restrict__ nrec, const int* __restrict__ skip, double* __restrict__ coef) {
  const int t = blockIdx.x;  // one block per (instance, direction)
  const int b = t / KREC, k = t % KREC;
  const int nk = (skip && skip[b]) ? 0 : nrec[b];
  if (k >= nk) {
    if (threadIdx.x == 0) coef[t] = 0.0;
    return;
  }
  const double v = block_sum_parts(part + (int64_t)t * DOT_BLOCKS, DOT_BLOCKS);
  if (threadIdx.x == 0) coef[t] = v / PQ[(int64_t)k * B + b];
}

// x0 = sum c_i p_i, r0 = p0 = b - sum c_i q_i
__global__ void k_rec_start(int me, int B, const double* __restrict__ P, const double* __restrict__ Q,
                            const double* __restrict__ coef, const int* __restrict__ nrec,
                            const double* __restrict__ bvec, double* __restrict__ x, double* __restrict__ r,
                            double* __restrict__ p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= me) return;
  const int nk = nrec[b];
  const int64_t o = (int64_t)b * me + i;
  double xs = 0.0, rs = bvec[o];
  for (int k = 0; k < nk; ++k) {
    const double ck = coef[b * KREC + k];
    const int64_t so = ((int64_t)k * B + b) * me + i;
    xs += ck * P[so];
    rs -= ck * Q[so];
  }
  x[o] = xs;
  r[o] = rs;
  p[o] = rs;
}

// z += alpha vn  (dx accumulation: K^{-1} G^T dy = sum_k alpha_k K^{-1} G^T p_k, the vn of each
// iteration), and (first pass) vn into its Init-CG slot
__global__ void k_cg_update_z(int n, int B, const double* __restrict__ alpha, const double* __restrict__ vn,
                              double* __restrict__ z, const int* __restrict__ done, const int* __restrict__ iters,
                              const int* __restrict__ enable, double* __restrict__ VN) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= n || done[b]) return;
  const int64_t o = (int64_t)b * n + i;
  const double v = vn[o];
  z[o] += alpha[b] * v;
  if (VN && *enable) {
    const int k = iters[b];
    if (k < KREC) VN[((int64_t)k * B + b) * n + i] = v;
  }
}

// z0 = sum_i c_i vn_i  (Init-CG start of the dx accumulation), or 0
__global__ void k_rec_start_z(int n, int B, const double* __restrict__ VN, const double* __restrict__ coef,
                              const int* __restrict__ nrec, double* __restrict__ z) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= n) return;
  const int nk = (VN && coef) ? nrec[b] : 0;
  double zs = 0.0;
  for (int k = 0; k < nk; ++k) zs += coef[b * KREC + k] * VN[((int64_t)k * B + b) * n + i];
  z[(int64_t)b * n + i] = zs;
}

// dx = -t - z
__global__ void k_dx_from_acc(int64_t len, const double* __restrict__ t, const double* __restrict__ z,
                              double* __restrict__ dx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i < len) dx[b * len + i] = -t[b * len + i] - z[b * len + i];
}

__global__ void k_rec_count(int B, const int* __restrict__ iters, int* __restrict__ nrec) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) nrec[b] = min(iters[b], KREC);
}

// CG init from r0: rr = r0.r0 (part), bnorm2 = b.b (part_b); done if converged already
__global__ void k_cg_init_scalars2(int B, const double* __restrict__ part, const double* __restrict__ part_b,
                                   double rtol, double* __restrict__ rr, double* __restrict__ bnorm2,
                                   int* __restrict__ done, int* __restrict__ iters, const int* __restrict__ skip) {
  const int b = blockIdx.x;  // one block per instance
  const double t = block_sum_parts(part + (int64_t)b * DOT_BLOCKS, DOT_BLOCKS);
  const double bb = block_sum_parts(part_b + (int64_t)b * DOT_BLOCKS, DOT_BLOCKS);
  if (threadIdx.x == 0) {
    rr[b] = t;
    bnorm2[b] = bb;
    iters[b] = 0;
    done[b] = (bb == 0.0) || (skip && skip[b]) || (sqrt(t) <= rtol * sqrt(bb));
  }
}

// end of a CG iteration inside the graph loop: continue while some instance is active and the cap
// is not reached; resets the activity counter for the next iteration
__global__ void k_cg_cond(int* active, int* loop, int maxit, cudaGraphConditionalHandle h) {
  const int it = ++(*loop);
  const unsigned go = (*active > 0 && it < maxit) ? 1u : 0u;
  *active = 0;
  cudaGraphSetConditional(h, go);
}

__global__ void k_copy_neg(int64_t len, const double* __restrict__ a, double sa, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i < len) out[b * len + i] = sa * a[b * len + i];
}

__global__ void k_zero(int64_t len, double* __restrict__ a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i < len) a[b * len + i] = 0.0;
}

// ds = -r4 - H dx ; dz = -r2 - D_s ds   (dx in internal order)
__global__ void k_recover(int mi, int n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col2,
                          const double* __restrict__ h_val, int64_t h_nnz, const double* __restrict__ dx,
                          const double* __restrict__ r2, const double* __restrict__ r4, const double* __restrict__ d_s,
                          double* __restrict__ ds, double* __restrict__ dz, const int* __restrict__ skip) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (r >= mi || (skip && skip[b])) return;
  const double* h = h_val + b * h_nnz;
  double acc = 0.0;
  for (int e = rowptr[r]; e < rowptr[r + 1]; ++e) acc += h[e] * dx[(int64_t)b * n + col2[e]];
  const int64_t o = (int64_t)b * mi + r;
  const double s = -r4[o] - acc;
  ds[o] = s;
  dz[o] = -r2[o] - d_s[o] * s;
}

// ------------------------------------------------------------------------------------------
// a8: residual of K_aug and componentwise backward error.  Row blocks x (internal), s, y, z.
//  rho = -r - K_aug d ; ratio = |rho| / (|K_aug||d| + |r|).  Writes rho (x block internal order);
//  the per-row ratio and |rho| feed block maxima in the same kernel.
// ------------------------------------------------------------------------------------------
struct ResArgs {
  int n, me, mi;
  const int32_t* perm2;
  const int32_t *ws_ptr, *ws_col;  // symmetric W (internal rows)
  const double *wsv, *sig;          // W values in that order; sigma + delta in internal order
  int64_t ws_nnz;
  const int32_t *gt_ptr, *gt_e, *gt_r, *ht_ptr, *ht_e, *ht_r;
  const int32_t *g_rowptr, *g_col2, *h_rowptr, *h_col2;
  const double *w_val, *g_val, *h_val, *sigma, *d_s, *delta;
  const double *gtv, *htv;  // transposed-order copies
  int64_t w_nnz, g_nnz, h_nnz;
  const double *r1, *r2, *r3, *r4;  // r1 original order
  const double *dx, *ds, *dy, *dz;  // dx internal
  double *rho1, *rho2, *rho3, *rho4;  // rho1 internal
  const int* skip;
};

__device__ __forceinline__ void kaug_residual_row(const ResArgs& a, int b, int64_t t, double& ratio_out, double& abs_out) {
  const int n = a.n, me = a.me, mi = a.mi;
  double res, den;
  if (t < n) {
    const int i = (int)t;
    const int oi = a.perm2[i];
    const double* w = a.wsv + b * a.ws_nnz;
    const double* dx = a.dx + (int64_t)b * n;
    double acc = 0.0, aa = 0.0;
    #pragma unroll 4
    for (int e = a.ws_ptr[i]; e < a.ws_ptr[i + 1]; ++e) {
      double v = w[e] * dx[a.ws_col[e]];
      acc += v;
      aa += fabs(v);
    }
    double dg = a.sig[(int64_t)b * n + i] * dx[i];
    acc += dg;
    aa += fabs(dg);
    if (me) {
      const double* g = a.gtv + b * a.g_nnz;
      #pragma unroll 4
      for (int e = a.gt_ptr[i]; e < a.gt_ptr[i + 1]; ++e) {
        double v = g[e] * a.dy[(int64_t)b * me + a.gt_r[e]];
        acc += v;
        aa += fabs(v);
      }
    }
    if (mi) {
      const double* h = a.htv + b * a.h_nnz;
      #pragma unroll 4
      for (int e = a.ht_ptr[i]; e < a.ht_ptr[i + 1]; ++e) {
        double v = h[e] * a.dz[(int64_t)b * mi + a.ht_r[e]];
        acc += v;
        aa += fabs(v);
      }
    }
    const double r = a.r1[(int64_t)b * n + oi];
    res = -r - acc;
    den = aa + fabs(r);
    a.rho1[(int64_t)b * n + i] = res;
  } else if (t < n + mi) {
    const int r = (int)(t - n);
    const int64_t o = (int64_t)b * mi + r;
    const double v1 = a.d_s[o] * a.ds[o], v2 = a.dz[o];
    res = -a.r2[o] - (v1 + v2);
    den = fabs(v1) + fabs(v2) + fabs(a.r2[o]);
    a.rho2[o] = res;
  } else if (t < n + mi + me) {
    const int r = (int)(t - n - mi);
    const double* g = a.g_val + b * a.g_nnz;
    const double* dx = a.dx + (int64_t)b * n;
    double acc = 0.0, aa = 0.0;
    #pragma unroll 4
    for (int e = a.g_rowptr[r]; e < a.g_rowptr[r + 1]; ++e) {
      double v = g[e] * dx[a.g_col2[e]];
      acc += v;
      aa += fabs(v);
    }
    const int64_t o = (int64_t)b * me + r;
    res = -a.r3[o] - acc;
    den = aa + fabs(a.r3[o]);
    a.rho3[o] = res;
  } else {
    const int r = (int)(t - n - mi - me);
    const double* h = a.h_val + b * a.h_nnz;
    const double* dx = a.dx + (int64_t)b * n;
    double acc = 0.0, aa = 0.0;
    #pragma unroll 4
    for (int e = a.h_rowptr[r]; e < a.h_rowptr[r + 1]; ++e) {
      double v = h[e] * dx[a.h_col2[e]];
      acc += v;
      aa += fabs(v);
    }
    const int64_t o = (int64_t)b * mi + r;
    acc += a.ds[o];
    aa += fabs(a.ds[o]);
    res = -a.r4[o] - acc;
    den = aa + fabs(a.r4[o]);
    a.rho4[o] = res;
  }
  double ratio = den > 0.0 ? fabs(res) / den : (res == 0.0 ? 0.0 : INFINITY);
  if (res != res) ratio = INFINITY;
  ratio_out = ratio;
  abs_out = fabs(res);
}

__device__ __forceinline__ double nanmax(double x, double m) { return (x > m || x != x) ? x : m; }

// rho = -r - K_aug d, one row per thread, and, fused, the maxima over rows of the componentwise
// ratio |rho_i| / (|K_aug||d| + |r|)_i and of |rho_i|: block maxima, then one atomicMax per block on
// the bit patterns (both quantities are >= 0 or +NaN, whose bit patterns order like the values;
// a maximum does not depend on the order, so the result stays deterministic)
__global__ void k_kaug_residual(ResArgs a, unsigned long long* __restrict__ omega_bits,
                                unsigned long long* __restrict__ resinf_bits) {
  __shared__ double red[2][TPB / 32];
  const int64_t rows = (int64_t)a.n + 2 * a.mi + a.me;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  double mr = 0.0, ma = 0.0;
  if (t < rows && !(a.skip && a.skip[b])) kaug_residual_row(a, b, t, mr, ma);
  for (int o = 16; o > 0; o >>= 1) {
    mr = nanmax(__shfl_down_sync(0xffffffffu, mr, o), mr);
    ma = nanmax(__shfl_down_sync(0xffffffffu, ma, o), ma);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = mr;
    red[1][threadIdx.x >> 5] = ma;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int k = 0; k < TPB / 32; ++k) {
      t0 = nanmax(red[0][k], t0);
      t1 = nanmax(red[1][k], t1);
    }
    atomicMax(omega_bits + b, (unsigned long long)__double_as_longlong(fabs(t0)));
    atomicMax(resinf_bits + b, (unsigned long long)__double_as_longlong(fabs(t1)));
  }
}

// per-instance max over rows (two-stage; max is order independent => deterministic)


// d_new = d + c for accepted instances; dest <- src where acc[b]
__global__ void k_axpy_sel(int64_t len, const double* __restrict__ d, const double* __restrict__ c,
                           double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i < len) out[b * len + i] = d[b * len + i] + c[b * len + i];
}

__global__ void k_copy_sel(int64_t len, const double* __restrict__ src, double* __restrict__ dst,
                           const int* __restrict__ acc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i < len && acc[b]) dst[b * len + i] = src[b * len + i];
}

// dx (original order) = dx_int[iperm]; NaN for NOT_PD instances
__global__ void k_unpermute(int n, const int32_t* __restrict__ perm2, const double* __restrict__ xi,
                            double* __restrict__ xo, const int* __restrict__ notpd) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (j >= n) return;
  xo[(int64_t)b * n + perm2[j]] = notpd[b] ? nan("") : xi[(int64_t)b * n + j];
}

__global__ void k_nan_fill(int64_t len, double* __restrict__ a, const int* __restrict__ notpd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i < len && notpd[b]) a[b * len + i] = nan("");
}

template <class T>
T* upload(const std::vector<T>& v, std::vector<void*>& owned, int64_t& bytes) {
  size_t sz = std::max<size_t>(1, v.size()) * sizeof(T);
  void* p = nullptr;
  if (cudaMalloc(&p, sz) != cudaSuccess) return nullptr;
  owned.push_back(p);
  bytes += sz;
  if (!v.empty()) cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return (T*)p;
}

}  // namespace

// ============================================================================================
// context
// ============================================================================================
struct ckkt_ctx {
  ckkt::Analysis A;
  ckkt_options opt{};
  bool user_perm = false;  // the ordering came from the caller (options.perm)
  int B = 1;
  bool has_device = false;
  cudaStream_t stream = nullptr;
  int64_t nnzk = 0, Lsize = 0, w_nnz = 0, g_nnz = 0, h_nnz = 0;
  int n = 0, me = 0, mi = 0;
  int max_w = 1;
  std::vector<void*> owned;
  int64_t device_bytes = 0;
  int64_t launches = 0;
  // pattern arrays on device
  SymDev S{};
  int64_t *wt_ptr = nullptr, *jt_ptr = nullptr;
  int32_t *wt_ptr32 = nullptr, *jt_ptr32 = nullptr;  // 32-bit copies when the offsets fit (less map traffic)
  int32_t *wt_idx = nullptr, *jt_a = nullptr, *jt_b = nullptr, *jt_r = nullptr, *kdiag = nullptr;
  int32_t *gt_ptr = nullptr, *gt_e = nullptr, *gt_r = nullptr, *ht_ptr = nullptr, *ht_e = nullptr, *ht_r = nullptr;
  int32_t *g_rowptr = nullptr, *g_col2 = nullptr, *h_rowptr = nullptr, *h_col2 = nullptr;
  int32_t *ws_ptr = nullptr, *ws_col = nullptr, *ws_idx = nullptr;
  int64_t ws_nnz = 0;
  double *wsv = nullptr, *sig_i = nullptr;  // residual copies (symmetric internal W order; sigma+delta internal)
  // numeric
  double *Kval = nullptr, *L = nullptr, *Ub = nullptr, *Vb = nullptr;
  int64_t Usize = 0, Vsize = 0;
  int max_m = 1;
  int ntask = 0, grid_fac = 1, grid_fwd = 1, grid_bwd = 1, grid_ftop = 1, grid_btop = 1;
  int small_panel = SMALL_PANEL_MIN;  // one-warp front threshold (doubles), chosen at setup
  int epoch_fac = 0, epoch_fwd = 0, epoch_bwd = 0;
  int* epoch_dev = nullptr;  // [2] forward / backward sweep epochs, bumped on the device
  Sched Qfac{}, Qfwd{}, Qbwd{};
  int nchunk = 0, nq = 0, nsub = 0;
  int32_t *chunk_ptr = nullptr, *queue = nullptr, *sub_ptr = nullptr, *sub_nodes = nullptr, *topq = nullptr;
  const SnMeta* qmeta = nullptr;  // metadata of the bottom queue, queue order
  const SnMeta* tmeta = nullptr;  // metadata of the tiny subtrees' nodes, sub_nodes order
  double *gtv = nullptr, *htv = nullptr;  // G / H values in transposed (column) order, refreshed at refactor
  double* gv = nullptr;  // G values (row order) copied at refactor: the captured CG graph reads only context memory
  int ntop = 0;
  const SnMeta* topmeta = nullptr;  // metadata of the top queue, top order
  int topbuf = 0;                   // doubles of the top kernels' panel buffer
  int64_t ftop_smem = 0, btop_smem = 0;
  int8_t* tinyflag = nullptr;
  std::vector<int8_t> tiny_host;
  std::vector<SnMeta> meta_h;
  // phase profiling
  bool profiling = false;
  // CG loop as a CUDA graph with a device-side WHILE condition (no host round trip per iteration)
  cudaGraph_t cg_graph = nullptr;
  cudaGraphExec_t cg_exec = nullptr;
  cudaGraphConditionalHandle cg_cond = 0;
  int* cg_loop = nullptr;  // [1] iterations executed by the graph loop
  // Init-CG: directions of the first pass (KREC slots x B x m_e), p.q, counts, coefficients
  double *rec_P = nullptr, *rec_Q = nullptr, *rec_PQ = nullptr, *rec_part = nullptr, *rec_coef = nullptr;
  double* part_b = nullptr;
  double *rec_VN = nullptr, *cg_z = nullptr;  // Init-CG vn slots; dx accumulator [B,n]
  int *rec_enable = nullptr, *rec_n = nullptr;
  bool rec_on = false;
  int64_t cg_body_launches = 0;
  bool graph_failed = false;
  bool graph_pending_loops = false;  // h_pinned_int[4B] holds the loop count of the last graph launch
  std::vector<std::array<cudaEvent_t, 2>> ev_pool;
  std::vector<int> ev_phase;
  size_t ev_used = 0;
  int prof_phase = -1;
  int64_t big_smem = 0, fac_smem = 0, sol_smem = 0, fwd_smem = 0;
  int *notpd = nullptr, *minpiv = nullptr;
  // last refactor values (caller-owned, must stay valid until the next refactor)
  const double *w_val = nullptr, *g_val = nullptr, *h_val = nullptr, *sigma = nullptr, *d_s = nullptr,
               *delta = nullptr;
  bool factored = false;
  // work vectors
  double *rg = nullptr, *tn = nullptr, *vn = nullptr;             // [B,n]
  double *cg_x = nullptr, *cg_r = nullptr, *cg_p = nullptr, *cg_q = nullptr, *bvec = nullptr;  // [B,me]
  double *dxi = nullptr, *dxi2 = nullptr, *cdx = nullptr;         // [B,n] step, trial, correction (internal)
  double *ds2 = nullptr, *dy2 = nullptr, *dz2 = nullptr;          // trial blocks
  double *cds = nullptr, *cdy = nullptr, *cdz = nullptr;          // correction blocks
  double *rho1 = nullptr, *rho2 = nullptr, *rho3 = nullptr, *rho4 = nullptr;
  double *rho1b = nullptr, *rho2b = nullptr, *rho3b = nullptr, *rho4b = nullptr;
  double *part = nullptr, *omega = nullptr, *resinf = nullptr, *wnorm_dev = nullptr;
  double* cg_rtol_dev = nullptr;  // [3]: first-pass / correction-pass / current CG tolerance
  double cg_rtol_corr = 1e-10;
  double *cg_rr = nullptr, *cg_bn = nullptr, *cg_alpha = nullptr, *cg_beta = nullptr;
  int *cg_done = nullptr, *cg_iters = nullptr, *active = nullptr, *accflag = nullptr, *skipflag = nullptr;
  int* h_pinned_int = nullptr;
  double* h_pinned_dbl = nullptr;
  // host-staging buffers for ckkt_iterate_host
  double *st_w = nullptr, *st_g = nullptr, *st_h = nullptr, *st_sig = nullptr, *st_ds = nullptr, *st_del = nullptr;
  double *st_r1 = nullptr, *st_r2 = nullptr, *st_r3 = nullptr, *st_r4 = nullptr;
  double *st_dx = nullptr, *st_ds_o = nullptr, *st_dy = nullptr, *st_dz = nullptr;
  int* st_notpd = nullptr;
  // ckkt_iterate_host: the right-hand sides are copied on a second stream while the refactorization runs
  cudaStream_t st_aux = nullptr;
  cudaEvent_t ev_vals = nullptr, ev_rhs = nullptr;
};

namespace {

void prof_begin(ckkt_ctx* c, int phase) {
  if (!c->profiling) return;
  if (c->ev_used == c->ev_pool.size()) {
    std::array<cudaEvent_t, 2> e;
    cudaEventCreate(&e[0]);
    cudaEventCreate(&e[1]);
    c->ev_pool.push_back(e);
    c->ev_phase.push_back(phase);
  }
  c->ev_phase[c->ev_used] = phase;
  cudaEventRecord(c->ev_pool[c->ev_used][0], c->stream);
}
void prof_end(ckkt_ctx* c) {
  if (!c->profiling) return;
  cudaEventRecord(c->ev_pool[c->ev_used][1], c->stream);
  ++c->ev_used;
}

ckkt_status dalloc(ckkt_ctx* c, void** p, size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (cudaMalloc(p, bytes) != cudaSuccess) return CKKT_OUT_OF_MEMORY;
  c->owned.push_back(*p);
  c->device_bytes += bytes;
  return CKKT_OK;
}

#define DALLOC(ptr, count)                                                        \
  do {                                                                            \
    ckkt_status st_ = dalloc(c, (void**)&(ptr), (size_t)(count) * sizeof(*(ptr))); \
    if (st_ != CKKT_OK) return st_;                                               \
  } while (0)

bool build_cg_graph(ckkt_ctx* c);

ckkt_status setup_device(ckkt_ctx* c) {
  ckkt::Analysis& A = c->A;
  const int B = c->B;
  const int n = c->n, me = c->me, mi = c->mi;
  CK(cudaSetDevice(c->opt.device));
  c->stream = (cudaStream_t)c->opt.stream;
  std::vector<void*>& o = c->owned;
  int64_t& by = c->device_bytes;
#define UP(dst, vec)                          \
  do {                                        \
    dst = upload(vec, o, by);                 \
    if (!dst) return CKKT_OUT_OF_MEMORY;      \
  } while (0)
  int32_t *sfirst, *srows, *level_list, *ch_ptr, *ch_list, *relmap, *kmap, *perm2, *sparent;
  int64_t *srowptr, *pofs, *relofs, *uofs, *vofs, *kp;
  UP(sfirst, A.sfirst);
  UP(srowptr, A.srowptr);
  UP(srows, A.srows);
  UP(pofs, A.pofs);
  UP(level_list, A.level_list);
  UP(ch_ptr, A.ch_ptr);
  UP(ch_list, A.ch_list);
  UP(relofs, A.relofs);
  UP(relmap, A.relmap);
  UP(uofs, A.uofs);
  UP(vofs, A.vofs);
  UP(kp, A.kp);
  UP(kmap, A.kmap);
  UP(perm2, A.perm2);
  UP(sparent, A.sparent);
  std::vector<int32_t> relw_h(A.ns, 0);
  for (int cc = 0; cc < A.ns; ++cc) {
    const int p = A.sparent[cc];
    if (p < 0) continue;
    const int wp_ = A.sfirst[p + 1] - A.sfirst[p];
    const int mc = (int)(A.srowptr[cc + 1] - A.srowptr[cc]) - (A.sfirst[cc + 1] - A.sfirst[cc]);
    int k = 0;
    while (k < mc && A.relmap[A.relofs[cc] + k] < wp_) ++k;
    relw_h[cc] = k;
  }
  int32_t* relw;
  UP(relw, relw_h);
  // packed metadata (the tiny flags of ChMeta are filled in once the tiny subtrees are known)
  c->meta_h.resize(A.ns);
  for (int s2 = 0; s2 < A.ns; ++s2) {
    SnMeta& M = c->meta_h[s2];
    M.f = A.sfirst[s2];
    M.w = A.sfirst[s2 + 1] - A.sfirst[s2];
    M.m = (int)(A.srowptr[s2 + 1] - A.srowptr[s2]);
    M.ch0 = A.ch_ptr[s2];
    M.ch1 = A.ch_ptr[s2 + 1];
    M.relw = relw_h[s2];
    M.pad0 = M.pad1 = 0;
    M.pofs = A.pofs[s2];
    M.vofs = A.vofs[s2];
    M.relofs = A.relofs[s2];
    M.r0 = A.srowptr[s2];
  }
  c->S = SymDev{nullptr, nullptr, sfirst, srowptr, srows, pofs, level_list, ch_ptr, ch_list, relofs, relmap, uofs, vofs,
                kp, kmap, perm2, sparent, relw};
  {  // tiny supernodes (m <= TINY_M, w <= TINY_W, all descendants tiny): one lane group per tiny subtree
    const int ns = A.ns;
    c->tiny_host.assign(ns, 0);
    std::vector<int8_t>& T = c->tiny_host;
    for (int s = 0; s < ns; ++s) {  // postorder: children before parents
      const int64_t m = A.srowptr[s + 1] - A.srowptr[s], w = A.sfirst[s + 1] - A.sfirst[s];
      bool t = m <= TINY_M && w <= TINY_W;
      for (int ci = A.ch_ptr[s]; t && ci < A.ch_ptr[s + 1]; ++ci) t = T[A.ch_list[ci]] != 0;
      T[s] = t;
    }
  }
  {  // factor tasks in level order (tiny supernodes excluded): big supernodes (one CTA) and bundles of
     // small ones (one warp each)
    std::vector<int32_t> tsn, tbig, tptr{0};
    c->big_smem = 0;
    int dev_sms0 = 148;
    CK(cudaDeviceGetAttribute(&dev_sms0, cudaDevAttrMultiProcessorCount, c->opt.device));
    const int64_t chunk_max = getenv("CKKT_CHUNK") ? std::max(1, atoi(getenv("CKKT_CHUNK"))) : 32;  // tuning only
    // many supernodes: more one-warp fronts keep 8 independent fronts in flight per CTA (C3: -2 ms per
    // refactor); few supernodes: the CTA path finishes the short critical path sooner (C2)
    c->small_panel = ((int64_t)A.ns * B > 200000) ? SMALL_PANEL_MAX : SMALL_PANEL_MIN;
    if (const char* e = getenv("CKKT_SMALL_PANEL")) c->small_panel = std::max(64, std::min(SMALL_PANEL_MAX, atoi(e)));
    for (int l = 0; l < A.nlevels; ++l) {
      std::vector<int32_t> small;
      for (int k = A.level_ptr[l]; k < A.level_ptr[l + 1]; ++k) {
        const int s = A.level_list[k];
        if (c->tiny_host[s]) continue;
        const int64_t m = A.srowptr[s + 1] - A.srowptr[s], w = A.sfirst[s + 1] - A.sfirst[s];
        if (m * w <= c->small_panel && w <= 32) {
          small.push_back(s);
        } else {
          tbig.push_back(1);
          tsn.push_back(s);
          tptr.push_back((int32_t)tsn.size());
          const int64_t mp = big_ldp((int)m), wp = (w + 3) & ~3;
          c->big_smem = std::max<int64_t>(c->big_smem, 8 * (mp * wp + 8));
        }
      }
      // one-warp fronts of this level in chunks of SMALL_WARPS..chunk_max (about four chunks per SM)
      const int64_t csz = std::max<int64_t>(SMALL_WARPS, std::min<int64_t>(chunk_max, (int64_t)small.size() * B /
                                                                                         (4 * (int64_t)dev_sms0)));
      for (size_t k = 0; k < small.size(); k += csz) {
        tbig.push_back(0);
        for (size_t q = k; q < std::min(small.size(), k + (size_t)csz); ++q) tsn.push_back(small[q]);
        tptr.push_back((int32_t)tsn.size());
      }
    }
    c->ntask = (int)tbig.size();
    int32_t *d_tsn, *d_tbig, *d_tptr;
    UP(d_tsn, tsn);
    UP(d_tbig, tbig);
    UP(d_tptr, tptr);
    std::vector<int32_t> zeros((size_t)B * A.ns, 0), z2(4, 0);
    int32_t *dfac, *dfwd, *dbwd, *cfac, *cfwd, *cbwd;
    UP(dfac, zeros);
    UP(dfwd, zeros);
    UP(dbwd, zeros);
    UP(cfac, z2);
    UP(cfwd, z2);
    UP(cbwd, z2);
    c->Qfac = Sched{c->ntask, d_tsn, d_tbig, d_tptr, dfac, cfac, c->small_panel};
    c->Qfwd = Sched{c->ntask, d_tsn, d_tbig, d_tptr, dfwd, cfwd, c->small_panel};
    c->Qbwd = Sched{c->ntask, d_tsn, d_tbig, d_tptr, dbwd, cbwd, c->small_panel};
    c->fac_smem = std::max<int64_t>(c->big_smem, 8 * SMALL_WARPS * c->small_panel);
    c->sol_smem = 8 * ((int64_t)SOLVE_WORKERS * (c->max_m + 64 + RED_SZ)) +
                  4 * (int64_t)SOLVE_WORKERS * c->max_m;  // + per-worker row indices (backward)
    c->fwd_smem = 8 * ((int64_t)SOLVE_WORKERS * (c->max_m + 64));
    if (c->fac_smem > 227 * 1024 || c->sol_smem > 227 * 1024) return CKKT_INVALID_ARG;
    CK(cudaFuncSetAttribute(k_factor_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->fac_smem));
    CK(cudaFuncSetAttribute(k_fwd_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->fwd_smem));
    CK(cudaFuncSetAttribute(k_bwd_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->sol_smem));
    int dev_sms = 0, occ = 0;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->opt.device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_factor_persist, MF_THREADS, c->fac_smem));
    c->grid_fac = std::max(1, std::min(occ * dev_sms, c->ntask * B));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fwd_persist, 32 * SOLVE_WARPS, c->fwd_smem));
    c->grid_fwd = std::max(1, std::min(occ * dev_sms, (A.ns * B + SOLVE_WARPS - 1) / SOLVE_WARPS));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bwd_persist, 32 * SOLVE_WARPS, c->sol_smem));
    c->grid_bwd = std::max(1, std::min(occ * dev_sms, (A.ns * B + SOLVE_WARPS - 1) / SOLVE_WARPS));
    if (getenv("CKKT_VERBOSE"))
      fprintf(stderr, "ckkt: grids factor %d fwd %d bwd %d, smem factor %lld fwd %lld bwd %lld, max_m %d\n", c->grid_fac,
              c->grid_fwd, c->grid_bwd, (long long)c->fac_smem, (long long)c->fwd_smem, (long long)c->sol_smem, c->max_m);
    {  // tiny subtrees (one thread each) and the queue of the remaining supernodes (one warp each)
      const int ns = A.ns;
      const std::vector<int8_t>& T = c->tiny_host;
      std::vector<std::vector<int32_t>> subs;
      std::vector<int32_t> stack;
      for (int s = 0; s < ns; ++s) {
        if (!T[s] || (A.sparent[s] >= 0 && T[A.sparent[s]])) continue;
        std::vector<int32_t> nodes;  // postorder of the subtree rooted at s
        std::vector<std::pair<int, int>> st{{s, A.ch_ptr[s]}};
        while (!st.empty()) {
          auto& top = st.back();
          if (top.second < A.ch_ptr[top.first + 1]) {
            const int c = A.ch_list[top.second++];
            st.push_back({c, A.ch_ptr[c]});
          } else {
            nodes.push_back(top.first);
            st.pop_back();
          }
        }
        subs.push_back(std::move(nodes));
      }
      std::stable_sort(subs.begin(), subs.end(),
                       [](const std::vector<int32_t>& a, const std::vector<int32_t>& b) { return a.size() > b.size(); });
      std::vector<int32_t> sp{0}, sn;
      for (auto& v : subs) {
        sn.insert(sn.end(), v.begin(), v.end());
        sp.push_back((int32_t)sn.size());
      }
      {
        std::vector<ChMeta> chm(A.ch_list.size());
        for (size_t k = 0; k < A.ch_list.size(); ++k) {
          const int cc = A.ch_list[k];
          chm[k].c = cc;
          chm[k].mc = (int)(A.srowptr[cc + 1] - A.srowptr[cc]) - (A.sfirst[cc + 1] - A.sfirst[cc]);
          chm[k].tiny = T[cc];
          chm[k].pad = 0;
          chm[k].vofs = A.vofs[cc];
          chm[k].relofs = A.relofs[cc];
        }
        const ChMeta* dchm = upload(chm, o, by);
        const SnMeta* dmeta = upload(c->meta_h, o, by);
        if (!dchm || !dmeta) return CKKT_OUT_OF_MEMORY;
        c->S.meta = dmeta;
        c->S.chmeta = dchm;
      }
      c->nsub = (int)subs.size();
      c->sub_ptr = upload(sp, o, by);
      c->sub_nodes = upload(sn, o, by);
      {
        std::vector<SnMeta> tm(sn.size());
        for (size_t k = 0; k < sn.size(); ++k) {
          tm[k] = c->meta_h[sn[k]];
          tm[k].pad1 = sn[k];
        }
        c->tmeta = upload(tm, o, by);
        if (!c->tmeta && !sn.empty()) return CKKT_OUT_OF_MEMORY;
      }
      c->tinyflag = upload(T, o, by);
      // top set: large supernodes (panel > TOP_PANEL doubles) and all their ancestors (one CTA each)
      std::vector<int8_t> top(ns, 0);
      int64_t top_panel = TOP_PANEL;
      if (const char* e = getenv("CKKT_TOP_PANEL")) top_panel = atoll(e);  // tuning experiments
      for (int s2 = 0; s2 < ns; ++s2) {
        const int64_t m = A.srowptr[s2 + 1] - A.srowptr[s2], w = A.sfirst[s2 + 1] - A.sfirst[s2];
        if (!T[s2] && m * w > top_panel) top[s2] = 1;
      }
      for (int s2 = 0; s2 < ns; ++s2)  // postorder: parents after children
        if (top[s2] && A.sparent[s2] >= 0) top[A.sparent[s2]] = 1;
      std::vector<int32_t> q, lp{0}, tq;
      for (int l = 0; l < A.nlevels; ++l) {
        for (int k = A.level_ptr[l]; k < A.level_ptr[l + 1]; ++k) {
          const int s2 = A.level_list[k];
          if (T[s2]) continue;
          if (top[s2]) tq.push_back(s2);
          else q.push_back(s2);
        }
        lp.push_back((int32_t)q.size());
      }
      {  // panel storage in sweep order: tiny subtrees (subtree by subtree, postorder), then the bottom
         // queue, then the top set, so every worker's supernodes occupy one contiguous span of L
        std::vector<int64_t> np(ns + 1, -1);
        int64_t off = 0;
        auto place = [&](int s2) {
          np[s2] = off;
          off += (int64_t)(A.srowptr[s2 + 1] - A.srowptr[s2]) * (A.sfirst[s2 + 1] - A.sfirst[s2]);
        };
        for (int s2 : sn) place(s2);
        for (int s2 : q) place(s2);
        for (int s2 : tq) place(s2);
        if (off != A.pofs[ns]) return CKKT_INVALID_ARG;  // every supernode placed exactly once
        np[ns] = off;
        for (int s2 = 0; s2 < ns; ++s2) c->meta_h[s2].pofs = np[s2];  // (A.pofs stays canonical: blobs)
        CK(cudaMemcpy(const_cast<int64_t*>(c->S.pofs), np.data(), sizeof(int64_t) * np.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(const_cast<SnMeta*>(c->S.meta), c->meta_h.data(), sizeof(SnMeta) * ns, cudaMemcpyHostToDevice));
        std::vector<SnMeta> tm(sn.size());
        for (size_t k = 0; k < sn.size(); ++k) {
          tm[k] = c->meta_h[sn[k]];
          tm[k].pad1 = sn[k];
        }
        if (!sn.empty())
          CK(cudaMemcpy(const_cast<SnMeta*>(c->tmeta), tm.data(), sizeof(SnMeta) * sn.size(), cudaMemcpyHostToDevice));
      }
      c->nq = (int)q.size();
      c->ntop = (int)tq.size();
      c->queue = upload(q, o, by);
      c->topq = upload(tq, o, by);
      {
        std::vector<SnMeta> tm(tq.size());
        int64_t maxp = 0;
        for (size_t k = 0; k < tq.size(); ++k) {
          tm[k] = c->meta_h[tq[k]];
          tm[k].pad0 = A.sparent[tq[k]];
          tm[k].pad1 = tq[k];
          maxp = std::max<int64_t>(maxp, (int64_t)tm[k].m * tm[k].w);
        }
        c->topmeta = upload(tm, o, by);
        if (!c->topmeta && !tq.empty()) return CKKT_OUT_OF_MEMORY;
        // panel buffer: the largest top panel (+2 for the 16-byte alignment offset), capped so that
        // two CTAs of each top kernel fit on an SM; larger panels are read from global memory
        cudaFuncAttributes fa{}, ba{};
        CK(cudaFuncGetAttributes(&fa, k_fwd_top));
        CK(cudaFuncGetAttributes(&ba, k_bwd_top));
        const int64_t per_cta = (228 * 1024) / TOP_MINB - 2048;
        const int64_t fcap = (per_cta - (int64_t)fa.sharedSizeBytes) / 8 - (c->max_m + 64);
        const int64_t bcap = (per_cta - (int64_t)ba.sharedSizeBytes) / 8 - (c->max_m + 128);
        c->topbuf = (int)std::max<int64_t>(0, std::min<int64_t>(maxp + 2, std::min(fcap, bcap)) & ~int64_t(1));
        if (const char* e = getenv("CKKT_TOPBUF"))  // experiments: cap the staging buffer (0 = panels from L2)
          c->topbuf = std::min(c->topbuf, std::max(0, atoi(e)) & ~1);
        c->ftop_smem = 8 * ((int64_t)c->topbuf + c->max_m + 64);
        c->btop_smem = 8 * ((int64_t)c->topbuf + c->max_m + 128);
        CK(cudaFuncSetAttribute(k_fwd_top, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->ftop_smem));
        CK(cudaFuncSetAttribute(k_bwd_top, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->btop_smem));
        int occ2 = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_fwd_top, TOP_THREADS, c->ftop_smem));
        c->grid_ftop = std::max(1, std::min(occ2 * dev_sms, std::max(1, c->ntop * B)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_bwd_top, TOP_THREADS, c->btop_smem));
        c->grid_btop = std::max(1, std::min(occ2 * dev_sms, std::max(1, c->ntop * B)));
        if (getenv("CKKT_VERBOSE"))
          fprintf(stderr, "ckkt: top set %d supernodes, max panel %lld, buffer %d doubles, grids %d/%d\n", c->ntop,
                  (long long)maxp, c->topbuf, c->grid_ftop, c->grid_btop);
      }
      {
        std::vector<SnMeta> qm(q.size());
        for (size_t k = 0; k < q.size(); ++k) {
          qm[k] = c->meta_h[q[k]];
          qm[k].pad0 = A.sparent[q[k]];
          qm[k].pad1 = q[k];
        }
        c->qmeta = upload(qm, o, by);
        if (!c->qmeta && !q.empty()) return CKKT_OUT_OF_MEMORY;
      }
      const int64_t warps = (int64_t)c->grid_fwd * SOLVE_WORKERS;  // bottom-set workers
      std::vector<int32_t> cp{0};
      for (int l = 0; l < A.nlevels; ++l) {
        const int64_t K = lp[l + 1] - lp[l];
        const int csz = (int)std::max<int64_t>(1, std::min<int64_t>(16, (K * B) / (4 * warps)));
        for (int64_t k = lp[l]; k < lp[l + 1]; k += csz) cp.push_back((int32_t)std::min<int64_t>(k + csz, lp[l + 1]));
      }
      c->nchunk = (int)cp.size() - 1;
      c->chunk_ptr = upload(cp, o, by);
      if (!c->chunk_ptr || !c->queue || !c->tinyflag || !c->sub_ptr || !c->sub_nodes) return CKKT_OUT_OF_MEMORY;
    }
  }
  UP(c->wt_ptr, A.wt_ptr);
  UP(c->wt_idx, A.wt_idx);
  UP(c->jt_ptr, A.jt_ptr);
  if (A.wt_ptr.back() < INT32_MAX && A.jt_ptr.back() < INT32_MAX) {
    std::vector<int32_t> w32(A.wt_ptr.begin(), A.wt_ptr.end()), j32(A.jt_ptr.begin(), A.jt_ptr.end());
    UP(c->wt_ptr32, w32);
    UP(c->jt_ptr32, j32);
  }
  UP(c->jt_a, A.jt_a);
  UP(c->jt_b, A.jt_b);
  UP(c->jt_r, A.jt_r);
  std::vector<int32_t> kdiag(c->nnzk, -1);
  for (int j = 0; j < n; ++j) kdiag[A.dslot[j]] = A.perm2[j];
  UP(c->kdiag, kdiag);
  UP(c->gt_ptr, A.gt_ptr);
  UP(c->gt_e, A.gt_e);
  UP(c->gt_r, A.gt_r);
  UP(c->ht_ptr, A.ht_ptr);
  UP(c->ht_e, A.ht_e);
  UP(c->ht_r, A.ht_r);
  UP(c->g_rowptr, A.pat.g_rowptr);
  UP(c->g_col2, A.g_col2);
  UP(c->h_rowptr, A.pat.h_rowptr);
  UP(c->h_col2, A.h_col2);
  // symmetric W rows (internal order), entries sorted by (row, col, w index)
  {
    std::vector<std::array<int32_t, 3>> ent;
    ent.reserve(2 * A.w_row2.size());
    for (size_t e = 0; e < A.w_row2.size(); ++e) {
      ent.push_back({A.w_row2[e], A.w_col2[e], (int32_t)e});
      if (A.w_row2[e] != A.w_col2[e]) ent.push_back({A.w_col2[e], A.w_row2[e], (int32_t)e});
    }
    std::sort(ent.begin(), ent.end());
    std::vector<int32_t> ptr(n + 1, 0), col(ent.size()), idx(ent.size());
    for (size_t k = 0; k < ent.size(); ++k) {
      ptr[ent[k][0] + 1]++;
      col[k] = ent[k][1];
      idx[k] = ent[k][2];
    }
    for (int i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
    UP(c->ws_ptr, ptr);
    UP(c->ws_col, col);
    UP(c->ws_idx, idx);
    c->ws_nnz = (int64_t)ent.size();
  }
#undef UP
  DALLOC(c->Kval, (size_t)B * c->nnzk);
  DALLOC(c->L, (size_t)B * c->Lsize + 4);  // +32 B: 16-byte-rounded L2 prefetches stay in bounds
  DALLOC(c->Ub, (size_t)B * c->Usize);
  DALLOC(c->Vb, (size_t)B * c->Vsize);
  DALLOC(c->epoch_dev, 2);
  CK(cudaMemset(c->epoch_dev, 0, 2 * sizeof(int)));
  DALLOC(c->gtv, (size_t)B * std::max<int64_t>(c->g_nnz, 1));
  DALLOC(c->gv, (size_t)B * std::max<int64_t>(c->g_nnz, 1));
  DALLOC(c->htv, (size_t)B * std::max<int64_t>(c->h_nnz, 1));
  DALLOC(c->wsv, (size_t)B * std::max<int64_t>(c->ws_nnz, 1));
  DALLOC(c->sig_i, (size_t)B * n);
  DALLOC(c->notpd, B);
  DALLOC(c->minpiv, B);
  const size_t Bn = (size_t)B * n, Bme = (size_t)B * std::max(me, 1), Bmi = (size_t)B * std::max(mi, 1);
  DALLOC(c->rg, Bn);
  DALLOC(c->tn, Bn);
  DALLOC(c->vn, Bn);
  DALLOC(c->cg_x, Bme);
  DALLOC(c->cg_r, Bme);
  DALLOC(c->cg_p, Bme);
  DALLOC(c->cg_q, Bme);
  DALLOC(c->bvec, Bme);
  DALLOC(c->dxi, Bn);
  DALLOC(c->dxi2, Bn);
  DALLOC(c->cdx, Bn);
  DALLOC(c->ds2, Bmi);
  DALLOC(c->dy2, Bme);
  DALLOC(c->dz2, Bmi);
  DALLOC(c->cds, Bmi);
  DALLOC(c->cdy, Bme);
  DALLOC(c->cdz, Bmi);
  DALLOC(c->rho1, Bn);
  DALLOC(c->rho2, Bmi);
  DALLOC(c->rho3, Bme);
  DALLOC(c->rho4, Bmi);
  DALLOC(c->rho1b, Bn);
  DALLOC(c->rho2b, Bmi);
  DALLOC(c->rho3b, Bme);
  DALLOC(c->rho4b, Bmi);
  DALLOC(c->part, (size_t)B * 1024);
  DALLOC(c->omega, 2 * B);
  DALLOC(c->resinf, 2 * B);
  DALLOC(c->wnorm_dev, B);
  DALLOC(c->cg_rtol_dev, 3);
  {
    c->cg_rtol_corr = c->opt.cg_rtol_corr;
    if (const char* e = getenv("CKKT_CG_RTOL_CORR")) c->cg_rtol_corr = atof(e);  // A/B experiments only
    const double h[3] = {c->opt.cg_rtol, c->cg_rtol_corr, c->opt.cg_rtol};
    CK(cudaMemcpy(c->cg_rtol_dev, h, sizeof(h), cudaMemcpyHostToDevice));
  }
  DALLOC(c->cg_rr, B);
  DALLOC(c->cg_bn, B);
  DALLOC(c->cg_alpha, B);
  DALLOC(c->cg_beta, B);
  DALLOC(c->cg_done, B);
  DALLOC(c->cg_iters, B);
  DALLOC(c->active, 1);
  DALLOC(c->cg_loop, 1);
  if (me > 0 && !getenv("CKKT_NO_INITCG")) {  // Init-CG storage (2 KREC m_e doubles per instance)
    c->rec_on = true;
    DALLOC(c->rec_P, (size_t)KREC * B * me);
    DALLOC(c->rec_Q, (size_t)KREC * B * me);
    DALLOC(c->rec_PQ, (size_t)KREC * B);
    DALLOC(c->rec_part, (size_t)B * KREC * DOT_BLOCKS);
    DALLOC(c->rec_coef, (size_t)B * KREC);
    DALLOC(c->rec_n, B);
    DALLOC(c->part_b, (size_t)B * 1024);
    DALLOC(c->rec_VN, (size_t)KREC * B * n);
  }
  if (me > 0) DALLOC(c->cg_z, (size_t)B * n);
  DALLOC(c->rec_enable, 1);
  DALLOC(c->accflag, B);
  DALLOC(c->skipflag, B);
  CK(cudaMallocHost(&c->h_pinned_int, sizeof(int) * (5 * B + 16)));
  CK(cudaMallocHost(&c->h_pinned_dbl, sizeof(double) * (8 * B + 16)));
  // device staging of ckkt_iterate_host (values, rhs, step): allocated here, never in a per-iteration call
  DALLOC(c->st_w, (size_t)B * std::max<int64_t>(c->w_nnz, 1));
  DALLOC(c->st_g, (size_t)B * std::max<int64_t>(c->g_nnz, 1));
  DALLOC(c->st_h, (size_t)B * std::max<int64_t>(c->h_nnz, 1));
  DALLOC(c->st_sig, Bn);
  DALLOC(c->st_ds, Bmi);
  DALLOC(c->st_del, B);
  DALLOC(c->st_r1, Bn);
  DALLOC(c->st_r2, Bmi);
  DALLOC(c->st_r3, Bme);
  DALLOC(c->st_r4, Bmi);
  DALLOC(c->st_dx, Bn);
  DALLOC(c->st_ds_o, Bmi);
  DALLOC(c->st_dy, Bme);
  DALLOC(c->st_dz, Bmi);
  DALLOC(c->st_notpd, B);
  CK(cudaStreamCreateWithFlags(&c->st_aux, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_vals, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_rhs, cudaEventDisableTiming));
  // the CG loop graph is captured here too (it reads only context-owned memory)
  if (me > 0 && c->stream != nullptr && !sync_debug() && !getenv("CKKT_NO_GRAPH")) {
    if (!build_cg_graph(c)) {
      c->graph_failed = true;  // the host-driven loop is used instead
      cudaGetLastError();
    }
  }
  return CKKT_OK;
}

}  // namespace

// ============================================================================================
// C ABI
// ============================================================================================
extern "C" {

void ckkt_default_options(ckkt_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->strategy = CKKT_HYKKT;
  o->gamma = 1e7;
  o->cg_rtol = 1e-10;
  o->cg_rtol_corr = 1e-6;
  o->cg_maxit = 200;
  o->ref_tol = 1e-10;  // the north-star bar on the relative KKT residual (reading R7)
  o->ref_maxit = 10;
  o->batch = 1;
  o->leaf = 64;
  o->perm = nullptr;
  o->device = 0;
  o->stream = nullptr;
}

const char* ckkt_status_str(ckkt_status s) {
  switch (s) {
    case CKKT_OK: return "ok";
    case CKKT_NOT_PD: return "not positive definite (wrong inertia)";
    case CKKT_CG_NO_CONVERGENCE: return "CG did not converge";
    case CKKT_REFINE_NOT_CONVERGED: return "refinement did not reach ref_tol";
    case CKKT_PATTERN_ERROR: return "pattern error";
    case CKKT_INVALID_ARG: return "invalid argument";
    case CKKT_CUDA_ERROR: return "CUDA error";
    case CKKT_OUT_OF_MEMORY: return "out of memory";
  }
  return "unknown";
}

void ckkt_destroy(ckkt_ctx* c) {
  if (!c) return;
  if (c->has_device) {
    cudaSetDevice(c->opt.device);
    for (auto& e : c->ev_pool) {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
    if (c->cg_exec) cudaGraphExecDestroy(c->cg_exec);
    if (c->cg_graph) cudaGraphDestroy(c->cg_graph);
    if (c->ev_vals) cudaEventDestroy(c->ev_vals);
    if (c->ev_rhs) cudaEventDestroy(c->ev_rhs);
    if (c->st_aux) cudaStreamDestroy(c->st_aux);
    for (void* p : c->owned) cudaFree(p);
    if (c->h_pinned_int) cudaFreeHost(c->h_pinned_int);
    if (c->h_pinned_dbl) cudaFreeHost(c->h_pinned_dbl);
  }
  delete c;
}

static ckkt_status setup_impl(const ckkt_pattern* p, const ckkt_options* opt, const void* blob, int64_t blob_size,
                              ckkt_ctx** out);

ckkt_status ckkt_setup(const ckkt_pattern* p, const ckkt_options* opt, ckkt_ctx** out) {
  return setup_impl(p, opt, nullptr, 0, out);
}

ckkt_status ckkt_setup_from_analysis(const ckkt_pattern* p, const ckkt_options* opt, const void* blob, int64_t size,
                                     ckkt_ctx** out) {
  if (!blob || size <= 0) return CKKT_INVALID_ARG;
  return setup_impl(p, opt, blob, size, out);
}

ckkt_status ckkt_export_analysis(const ckkt_ctx* c, void* buf, int64_t* size) {
  if (!c || !size) return CKKT_INVALID_ARG;
  const int64_t need = (int64_t)ckkt::analysis_blob_size(c->A);
  if (!buf) {
    *size = need;
    return CKKT_OK;
  }
  if (*size < need) return CKKT_INVALID_ARG;
  ckkt::save_analysis(c->A, c->opt.leaf > 0 ? c->opt.leaf : 64, c->user_perm, static_cast<char*>(buf));
  *size = need;
  return CKKT_OK;
}

static ckkt_status setup_impl(const ckkt_pattern* p, const ckkt_options* opt, const void* blob, int64_t blob_size,
                              ckkt_ctx** out) {
  NvtxRange nvtx_range("ckkt_setup");
  if (!p || !out) return CKKT_INVALID_ARG;
  *out = nullptr;
  ckkt_options o;
  if (opt) o = *opt;
  else ckkt_default_options(&o);
  if (o.batch < 1 || (o.strategy != CKKT_LIFTED && o.strategy != CKKT_HYKKT)) return CKKT_INVALID_ARG;
  // tolerances: finite and > 0 (a zero cg_rtol_corr, e.g. from a zero-initialised struct, means the
  // default); caps >= 0; gamma finite and > 0 for HyKKT
  if (o.cg_rtol_corr == 0.0) o.cg_rtol_corr = 1e-6;
  auto pos = [](double v) { return std::isfinite(v) && v > 0.0; };
  if (!pos(o.cg_rtol) || !pos(o.cg_rtol_corr) || !pos(o.ref_tol) || o.cg_maxit < 0 || o.ref_maxit < 0 ||
      (o.strategy == CKKT_HYKKT && !pos(o.gamma)))
    return CKKT_INVALID_ARG;
  if (o.strategy == CKKT_LIFTED && p->m_e != 0) return CKKT_INVALID_ARG;
  if (p->n <= 0 || p->m_e < 0 || p->m_i < 0 || p->w_nnz < 0) return CKKT_INVALID_ARG;
  if ((p->w_nnz > 0 && (!p->w_row || !p->w_col)) || (p->m_e > 0 && (!p->g_rowptr || !p->g_col)) ||
      (p->m_i > 0 && (!p->h_rowptr || !p->h_col)))
    return CKKT_INVALID_ARG;
  std::unique_ptr<ckkt_ctx> c(new ckkt_ctx());
  c->opt = o;
  c->B = o.batch;
  ckkt::Pattern pat;
  pat.n = p->n;
  pat.me = p->m_e;
  pat.mi = p->m_i;
  pat.w_row.assign(p->w_row, p->w_row + p->w_nnz);
  pat.w_col.assign(p->w_col, p->w_col + p->w_nnz);
  if (p->m_e > 0) {
    pat.g_rowptr.assign(p->g_rowptr, p->g_rowptr + p->m_e + 1);
    pat.g_col.assign(p->g_col, p->g_col + pat.g_rowptr.back());
  } else {
    pat.g_rowptr.assign(1, 0);
  }
  if (p->m_i > 0) {
    pat.h_rowptr.assign(p->h_rowptr, p->h_rowptr + p->m_i + 1);
    pat.h_col.assign(p->h_col, p->h_col + pat.h_rowptr.back());
  } else {
    pat.h_rowptr.assign(1, 0);
  }
  int code = 0;
  const int leaf = o.leaf > 0 ? o.leaf : 64;
  std::string err = blob ? ckkt::load_analysis(pat, leaf, o.perm != nullptr, static_cast<const char*>(blob),
                                               (size_t)blob_size, c->A, code)
                         : ckkt::analyze(pat, leaf, o.perm, c->A, code);
  if (!err.empty()) return (ckkt_status)code;
  if (blob && o.perm && !std::equal(c->A.perm.begin(), c->A.perm.end(), o.perm)) return CKKT_INVALID_ARG;
  c->opt.perm = nullptr;  // (the caller's array is not referenced after setup; remembered as a flag)
  c->user_perm = o.perm != nullptr;
  c->n = p->n;
  c->me = p->m_e;
  c->mi = p->m_i;
  c->nnzk = c->A.kp[c->n];
  c->Lsize = c->A.pofs[c->A.ns];
  if (c->Lsize >= ((int64_t)1 << 31)) return CKKT_OUT_OF_MEMORY;
  c->w_nnz = p->w_nnz;
  c->g_nnz = c->A.pat.g_rowptr.back();
  c->h_nnz = c->A.pat.h_rowptr.back();
  for (int s = 0; s < c->A.ns; ++s) {
    c->max_w = std::max(c->max_w, c->A.sfirst[s + 1] - c->A.sfirst[s]);
    c->max_m = std::max(c->max_m, (int)(c->A.srowptr[s + 1] - c->A.srowptr[s]));
  }
  c->Usize = c->A.uofs[c->A.ns];
  c->Vsize = c->A.vofs[c->A.ns];
  if (o.device >= 0) {
    c->has_device = true;
    ckkt_status st = setup_device(c.get());
    if (st != CKKT_OK) {
      ckkt_destroy(c.release());
      return st;
    }
  }
  *out = c.release();
  return CKKT_OK;
}

ckkt_status ckkt_get_sizes(const ckkt_ctx* c, ckkt_sizes* s) {
  if (!c || !s) return CKKT_INVALID_ARG;
  s->n = c->n;
  s->m_e = c->me;
  s->m_i = c->mi;
  s->batch = c->B;
  s->nnz_k = c->nnzk;
  s->nnz_l = c->A.nnz_l;
  s->l_storage = c->Lsize;
  s->n_supernodes = c->A.ns;
  s->n_levels = c->A.nlevels;
  s->flops_factor = c->A.flops;
  s->device_bytes = c->device_bytes;
  return CKKT_OK;
}

ckkt_status ckkt_export_symbolic(const ckkt_ctx* c, int32_t* perm, int32_t* parent, int32_t* colcount,
                                 int64_t* l_colptr, int32_t* l_rowind) {
  if (!c) return CKKT_INVALID_ARG;
  const int n = c->n;
  if (perm) std::copy(c->A.perm.begin(), c->A.perm.end(), perm);
  if (parent) std::copy(c->A.parent.begin(), c->A.parent.end(), parent);
  if (colcount) std::copy(c->A.colcount.begin(), c->A.colcount.end(), colcount);
  if (l_colptr || l_rowind) {
    std::vector<int64_t> Lp;
    std::vector<int32_t> Li;
    ckkt::export_l_pattern(c->A, Lp, Li);
    if (l_colptr) std::copy(Lp.begin(), Lp.end(), l_colptr);
    if (l_rowind) std::copy(Li.begin(), Li.end(), l_rowind);
  }
  (void)n;
  return CKKT_OK;
}

ckkt_status ckkt_export_elimination_order(const ckkt_ctx* c, int32_t* order) {
  if (!c || !order) return CKKT_INVALID_ARG;
  std::copy(c->A.perm2.begin(), c->A.perm2.end(), order);
  return CKKT_OK;
}

int64_t ckkt_launch_count(const ckkt_ctx* c) { return c ? c->launches : 0; }

ckkt_status ckkt_profile(ckkt_ctx* c, int32_t enable) {
  if (!c || !c->has_device) return CKKT_INVALID_ARG;
  c->profiling = enable != 0;
  c->ev_used = 0;
  return CKKT_OK;
}

ckkt_status ckkt_phase_times(ckkt_ctx* c, double* ms, int64_t* count) {
  if (!c || !c->has_device || !ms || !count) return CKKT_INVALID_ARG;
  for (int k = 0; k < CKKT_NPHASES; ++k) {
    ms[k] = 0.0;
    count[k] = 0;
  }
  CK(cudaStreamSynchronize(c->stream));
  for (size_t i = 0; i < c->ev_used; ++i) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, c->ev_pool[i][0], c->ev_pool[i][1]));
    ms[c->ev_phase[i]] += t;
    count[c->ev_phase[i]]++;
  }
  c->ev_used = 0;
  return CKKT_OK;
}

ckkt_status ckkt_refactor(ckkt_ctx* c, const double* w_val, const double* g_val, const double* h_val,
                          const double* sigma_x, const double* d_s, const double* delta_x, int32_t* not_pd,
                          int32_t* min_bad_pivot) {
  NvtxRange nvtx_range("ckkt_refactor");
  if (!c || !c->has_device) return CKKT_INVALID_ARG;
  if ((c->w_nnz && !w_val) || !sigma_x || (c->g_nnz && !g_val) || (c->h_nnz && !h_val) || (c->mi && !d_s))
    return CKKT_INVALID_ARG;
  CK(cudaSetDevice(c->opt.device));
  cudaStream_t st = c->stream;
  const int B = c->B;
  c->w_val = w_val;
  c->g_val = g_val;
  c->h_val = h_val;
  c->sigma = sigma_x;
  c->d_s = d_s;
  c->delta = delta_x;
  const double gamma = (c->opt.strategy == CKKT_HYKKT) ? c->opt.gamma : 0.0;
  if (c->g_nnz) {
    k_gather_t<<<(unsigned)((c->g_nnz * B + TPB - 1) / TPB), TPB, 0, st>>>(c->g_nnz, B, c->gt_e, g_val, c->gtv);
    c->launches++;
    // the CG graph (captured once) and the residual read the context's copy, never the caller's
    // buffer, so a refactor with a different g_val pointer cannot leave a stale pointer behind
    CK(cudaMemcpyAsync(c->gv, g_val, sizeof(double) * (size_t)B * c->g_nnz, cudaMemcpyDeviceToDevice, st));
  }
  if (c->h_nnz) {
    k_gather_t<<<(unsigned)((c->h_nnz * B + TPB - 1) / TPB), TPB, 0, st>>>(c->h_nnz, B, c->ht_e, h_val, c->htv);
    c->launches++;
  }
  if (c->ws_nnz) {
    k_gather_ws<<<(unsigned)((c->ws_nnz * B + TPB - 1) / TPB), TPB, 0, st>>>(c->ws_nnz, c->w_nnz, B, c->ws_idx, w_val,
                                                                          c->wsv);
    c->launches++;
  }
  k_gather_sigma<<<dim3(nblk(c->n), B), TPB, 0, st>>>(c->n, c->S.perm2, sigma_x, delta_x, c->sig_i);
  c->launches++;
  k_init_flags<<<nblk(B), TPB, 0, st>>>(B, c->notpd, c->minpiv);
  prof_begin(c, 0);
  {
    const dim3 gk(nblk(c->nnzk), B);
    const int mode = (c->mi == 0) ? 1 : (c->me == 0 ? 2 : 0);
#define CKKT_CONDENSE(IDXP, M)                                                                                      \
  k_condense<std::remove_const_t<std::remove_pointer_t<decltype(IDXP##wt)>>, M><<<gk, TPB, 0, st>>>(               \
      c->nnzk, IDXP##wt, c->wt_idx, IDXP##jt, c->jt_a, c->jt_b, c->jt_r, c->kdiag, w_val, c->w_nnz, g_val, c->g_nnz, \
      h_val, c->h_nnz, sigma_x, d_s, delta_x, gamma, c->n, c->me, c->mi, c->Kval)
    const int32_t* s32wt = c->wt_ptr32;
    const int32_t* s32jt = c->jt_ptr32;
    const int64_t* s64wt = c->wt_ptr;
    const int64_t* s64jt = c->jt_ptr;
    if (s32wt) {
      if (mode == 1) CKKT_CONDENSE(s32, 1);
      else if (mode == 2) CKKT_CONDENSE(s32, 2);
      else CKKT_CONDENSE(s32, 0);
    } else {
      if (mode == 1) CKKT_CONDENSE(s64, 1);
      else if (mode == 2) CKKT_CONDENSE(s64, 2);
      else CKKT_CONDENSE(s64, 0);
    }
#undef CKKT_CONDENSE
  }
  DBG_SYNC("k_condense");
  prof_end(c);
  c->launches += 2;
  const auto& A = c->A;
  ++c->epoch_fac;
  prof_begin(c, 1);
  if (c->nsub > 0)
    k_factor_tiny<<<(c->nsub * B * TG + FT_THREADS - 1) / FT_THREADS, FT_THREADS, 0, st>>>(
        c->S, c->tmeta, c->sub_ptr, c->nsub, B, c->L, c->Lsize, c->Ub, c->Usize, c->Kval, c->nnzk, c->notpd, c->minpiv);
  DBG_SYNC("k_factor_tiny");
  if (c->ntask > 0)
    k_factor_persist<<<c->grid_fac, MF_THREADS, c->fac_smem, st>>>(c->S, c->Qfac, A.ns, B, c->epoch_fac, c->L,
                                                                   c->Lsize, c->Ub, c->Usize, c->Kval, c->nnzk,
                                                                   c->notpd, c->minpiv, c->tinyflag);
  DBG_SYNC("k_factor_persist");
  prof_end(c);
  c->launches++;
  k_final_flags<<<nblk(B), TPB, 0, st>>>(B, c->notpd, c->minpiv, c->S.perm2, not_pd, min_bad_pivot);
  c->launches++;
  CK(cudaGetLastError());
  c->factored = true;
  return CKKT_OK;
}


// Inertia correction around the refactorization (reading R15 of DESIGN.md,
// schedule of SPEC inertia_correction).  Per instance: trial 0 uses delta = 0; on NOT_PD the first
// nonzero delta is 1e-4 * max(1, ||W||_inf) when delta_last == 0, else max(1e-20, delta_last / 3);
// every further failure multiplies it by 8; delta > 1e40 gives up (instance stays NOT_PD).  Every
// trial refactors the whole batch with the current per-instance deltas (accepted instances keep
// theirs, so their factors are recomputed bit-identically).
ckkt_status ckkt_refactor_inertia(ckkt_ctx* c, const double* w_val, const double* g_val, const double* h_val,
                                  const double* sigma_x, const double* d_s, const double* delta_last,
                                  double* delta_x, double* delta_out, int32_t* trials_out, int32_t* not_pd) {
  NvtxRange nvtx_range("ckkt_refactor_inertia");
  if (!c || !c->has_device || !delta_x) return CKKT_INVALID_ARG;
  const int B = c->B;
  cudaStream_t st = c->stream;
  std::vector<double> delta(B, 0.0), wnorm(B, -1.0);
  std::vector<int32_t> trials(B, 0), flag(B, 0), done(B, 0);
  ckkt_status rs = CKKT_OK;
  for (;;) {
    CK(cudaMemcpyAsync(delta_x, delta.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
    ckkt_status s = ckkt_refactor(c, w_val, g_val, h_val, sigma_x, d_s, delta_x, nullptr, nullptr);
    if (s != CKKT_OK) return s;
    if (wnorm[0] < 0.0) {  // once: ||W||_inf from the residual's symmetric W copy (gathered by the refactor)
      unsigned long long* nb = reinterpret_cast<unsigned long long*>(c->wnorm_dev);
      CK(cudaMemsetAsync(nb, 0, sizeof(double) * B, st));
      if (c->ws_nnz) {
        k_w_norminf<<<dim3(nblk(c->n), B), TPB, 0, st>>>(c->n, c->ws_ptr, c->wsv, c->ws_nnz, nb);
        c->launches++;
      }
      CK(cudaMemcpyAsync(wnorm.data(), nb, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(flag.data(), c->notpd, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bool again = false;
    for (int b = 0; b < B; ++b) {
      if (done[b]) continue;
      trials[b]++;
      if (!flag[b]) { done[b] = 1; continue; }
      double d;
      if (delta[b] == 0.0) {
        const double last = delta_last ? delta_last[b] : 0.0;
        d = (last == 0.0) ? 1e-4 * std::max(1.0, wnorm[b]) : std::max(1e-20, last / 3.0);
      } else {
        d = 8.0 * delta[b];
      }
      if (!(d <= 1e40)) { done[b] = 2; continue; }  // StrategyFailure: keep the last (failed) delta
      delta[b] = d;
      again = true;
    }
    if (!again) break;
  }
  for (int b = 0; b < B; ++b)
    if (done[b] == 2) rs = CKKT_NOT_PD;
  if (not_pd) CK(cudaMemcpyAsync(not_pd, c->notpd, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st));
  if (delta_out) std::copy(delta.begin(), delta.end(), delta_out);
  if (trials_out) std::copy(trials.begin(), trials.end(), trials_out);
  return rs;
}


ckkt_status ckkt_fraction_to_boundary(int32_t batch, int64_t len, const double* s, const double* ds, double tau,
                                      double* alpha, void* stream) {
  if (batch < 0 || len < 0 || !(tau > 0.0 && tau < 1.0) || (batch > 0 && (!alpha || (len > 0 && (!s || !ds)))))
    return CKKT_INVALID_ARG;
  if (batch == 0) return CKKT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  k_ftb_init<<<nblk(batch), TPB, 0, st>>>(batch, alpha);
  if (len > 0) {
    const unsigned gx = (unsigned)std::min<int64_t>(nblk(len), 4 * 148);
    k_ftb<<<dim3(gx, batch), TPB, 0, st>>>(len, s, ds, tau, reinterpret_cast<unsigned long long*>(alpha));
  }
  CK(cudaGetLastError());
  return CKKT_OK;
}

}  // extern "C"

namespace {

SweepArgs sweep_args(ckkt_ctx* c, const Sched& Q, int epoch, double* x, const int* skip, bool top) {
  SweepArgs a;
  a.queue = c->queue;
  a.qmeta = c->qmeta;
  a.chunk_ptr = c->chunk_ptr;
  a.nchunk = c->nchunk;
  a.top = c->topq;
  a.topmeta = c->topmeta;
  a.ntop = top ? c->ntop : 0;
  a.topbuf = c->topbuf;
  a.ns = c->A.ns;
  a.ctr = Q.ctr;
  a.done_all = Q.done;
  a.B = c->B;
  a.epoch = epoch;
  a.epoch_ptr = c->epoch_dev + (&Q == &c->Qbwd ? 1 : 0);
  a.L = c->L;
  a.Lsize = c->Lsize;
  a.X = x;
  a.n = c->n;
  a.Vb = c->Vb;
  a.Vsize = c->Vsize;
  a.max_m = c->max_m;
  a.skip = skip;
  return a;
}

void launch_fwd(ckkt_ctx* c, double* x, const int* skip) {
  cudaStream_t st = c->stream;
  prof_begin(c, 2);
  if (c->nsub > 0)
    k_fwd_tiny<<<(c->nsub * c->B * TG + 255) / 256, 256, 0, st>>>(c->S, c->tmeta, c->sub_ptr, c->nsub, c->B, c->L,
                                                              c->Lsize, x, c->n, c->Vb, c->Vsize, skip, c->epoch_dev);
  else
    k_epoch_bump<<<1, 1, 0, st>>>(c->epoch_dev);
  DBG_SYNC("k_fwd_tiny");
  ++c->epoch_fwd;
  if (c->nq > 0)
    k_fwd_persist<<<c->grid_fwd, 32 * SOLVE_WARPS, c->fwd_smem, st>>>(c->S,
                                                                       sweep_args(c, c->Qfwd, c->epoch_fwd, x, skip, false));
  DBG_SYNC("k_fwd_persist");
  if (c->ntop > 0) {
    k_fwd_top<<<c->grid_ftop, TOP_THREADS, c->ftop_smem, st>>>(c->S, sweep_args(c, c->Qfwd, c->epoch_fwd, x, skip, true));
    c->launches++;
  }
  DBG_SYNC("k_fwd_top");
  prof_end(c);
}

void launch_bwd(ckkt_ctx* c, double* x, const int* skip) {
  cudaStream_t st = c->stream;
  prof_begin(c, 3);
  ++c->epoch_bwd;
  if (c->ntop > 0) {
    k_bwd_top<<<c->grid_btop, TOP_THREADS, c->btop_smem, st>>>(c->S, sweep_args(c, c->Qbwd, c->epoch_bwd, x, skip, true));
    c->launches++;
  }
  DBG_SYNC("k_bwd_top");
  if (c->nq > 0)
    k_bwd_persist<<<c->grid_bwd, 32 * SOLVE_WARPS, c->sol_smem, st>>>(c->S,
                                                                       sweep_args(c, c->Qbwd, c->epoch_bwd, x, skip, false));
  DBG_SYNC("k_bwd_persist");
  if (c->nsub > 0)
    k_bwd_tiny<<<(c->nsub * c->B * TG + 255) / 256, 256, 0, st>>>(c->S, c->tmeta, c->sub_ptr, c->nsub, c->B, c->L,
                                                              c->Lsize, x, c->n, skip);
  DBG_SYNC("k_bwd_tiny");
  prof_end(c);
}

// x <- K^{-1} x  (internal order, in place), skipping instances with skip[b]
void ksolve(ckkt_ctx* c, double* x, const int* skip) {
  launch_fwd(c, x, skip);
  launch_bwd(c, x, skip);
  c->launches += 2 * ((c->nq > 0) + (c->nsub > 0));

}

void dot(ckkt_ctx* c, int64_t len, const double* a, const double* b, const int* skip) {
  k_dot_partial<<<dim3(DOT_BLOCKS, c->B), TPB, 0, c->stream>>>(len, a, b, c->part, skip);
  c->launches++;
}

// one CG iteration on S_gamma = G K_gamma^{-1} G^T; instances with
// cg_done set are skipped by every kernel
void cg_iteration(ckkt_ctx* c) {
  const int n = c->n, me = c->me, B = c->B;
  cudaStream_t st = c->stream;
  const dim3 gn(nblk(n), B), gme(nblk(std::max(me, 1)), B);
  prof_begin(c, 4);
  k_gt_spmv<<<gn, TPB, 0, st>>>(n, me, c->gt_ptr, c->gt_e, c->gt_r, c->gtv, c->g_nnz, c->cg_p, 1.0, nullptr, 0.0,
                                c->vn, c->cg_done);
  prof_end(c);
  ksolve(c, c->vn, c->cg_done);
  prof_begin(c, 4);
  k_g_spmv<<<gme, TPB, 0, st>>>(me, n, c->g_rowptr, c->g_col2, c->gv, c->g_nnz, c->vn, 1.0, nullptr, 0.0, c->cg_q,
                                c->cg_done);
  dot(c, me, c->cg_p, c->cg_q, c->cg_done);
  k_cg_alpha<<<B, TPB, 0, st>>>(B, c->part, c->cg_rr, c->cg_alpha, c->cg_done, c->cg_iters, c->rec_enable,
                                c->rec_PQ, KREC);
  if (c->rec_on) {
    k_cg_store<<<gme, TPB, 0, st>>>(me, B, c->cg_p, c->cg_q, c->part, c->cg_iters, c->cg_done, c->rec_enable,
                                    c->rec_P, c->rec_Q, c->rec_PQ);
    c->launches++;
  }
  k_cg_update_xr<<<gme, TPB, 0, st>>>(me, c->cg_alpha, c->cg_p, c->cg_q, c->cg_x, c->cg_r, c->cg_done);
  k_cg_update_z<<<gn, TPB, 0, st>>>(n, B, c->cg_alpha, c->vn, c->cg_z, c->cg_done, c->cg_iters, c->rec_enable,
                                    c->rec_VN);
  c->launches++;
  dot(c, me, c->cg_r, c->cg_r, c->cg_done);
  k_cg_beta<<<B, TPB, 0, st>>>(B, c->part, c->cg_rr, c->cg_bn, c->cg_rtol_dev + 2, c->cg_beta, c->cg_done,
                                     c->cg_iters, c->active);
  k_cg_update_p<<<gme, TPB, 0, st>>>(me, c->cg_beta, c->cg_r, c->cg_p, c->cg_done);
  c->launches += 7;
  prof_end(c);
}

// capture the CG loop once: a conditional WHILE node whose body is one iteration + k_cg_cond
bool build_cg_graph(ckkt_ctx* c) {
  cudaStream_t st = c->stream;
  if (cudaGraphCreate(&c->cg_graph, 0) != cudaSuccess) return false;
  if (cudaGraphConditionalHandleCreate(&c->cg_cond, c->cg_graph, 1, cudaGraphCondAssignDefault) != cudaSuccess)
    return false;
  cudaGraphNodeParams prm = {};
  prm.type = cudaGraphNodeTypeConditional;
  prm.conditional.handle = c->cg_cond;
  prm.conditional.type = cudaGraphCondTypeWhile;
  prm.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, c->cg_graph, nullptr, 0, &prm) != cudaSuccess) return false;
  cudaGraph_t bodyg = prm.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return false;
  const int64_t l0 = c->launches;
  cg_iteration(c);
  k_cg_cond<<<1, 1, 0, st>>>(c->active, c->cg_loop, c->opt.cg_maxit, c->cg_cond);
  c->cg_body_launches = c->launches - l0 + 1;
  c->launches = l0;
  cudaGraph_t out = nullptr;
  if (cudaStreamEndCapture(st, &out) != cudaSuccess) return false;
  if (cudaGraphInstantiate(&c->cg_exec, c->cg_graph, 0) != cudaSuccess) return false;
  return true;
}

// One unrefined pass of the strategy for right-hand side (r1 [internal if r1_internal], r2, r3, r4):
// writes dx (internal), ds, dy, dz.  Returns the total CG iterations (host copy, per instance) via c->cg_iters.
ckkt_status solve_pass(ckkt_ctx* c, const double* r1, int r1_internal, const double* r2, const double* r3,
                       const double* r4, double* dx, double* ds, double* dy, double* dz, const int* skip,
                       std::vector<int>& kcg, bool first_pass) {
  const int n = c->n, me = c->me, mi = c->mi, B = c->B;
  cudaStream_t st = c->stream;
  const double gamma = (c->opt.strategy == CKKT_HYKKT) ? c->opt.gamma : 0.0;
  const dim3 gn(nblk(n), B), gme(nblk(std::max(me, 1)), B), gmi(nblk(std::max(mi, 1)), B);
  // r_gamma (or r~) in internal order, into dx (it becomes -K^{-1}(...) after the solves)
  prof_begin(c, 4);
  k_rhs<<<gn, TPB, 0, st>>>(n, me, mi, c->S.perm2, r1, r1_internal, r2, r3, r4, c->gt_ptr, c->gt_e, c->gt_r,
                            c->ht_ptr, c->ht_e, c->ht_r, c->gtv, c->g_nnz, c->htv, c->h_nnz, c->d_s, gamma, c->rg,
                            skip);
  c->launches++;
  kcg.assign(B, 0);
  if (me > 0) {
    // t = K^{-1} r_gamma ; b = r3 - G t
    cudaMemcpyAsync(c->tn, c->rg, sizeof(double) * (size_t)B * n, cudaMemcpyDeviceToDevice, st);
    prof_end(c);
    ksolve(c, c->tn, skip);
    prof_begin(c, 4);
    k_g_spmv<<<gme, TPB, 0, st>>>(me, n, c->g_rowptr, c->g_col2, c->gv, c->g_nnz, c->tn, -1.0, r3, 1.0, c->bvec,
                                  skip);
    const bool init_cg = c->rec_on && !first_pass;
    if (c->rec_on) CK(cudaMemsetAsync(c->rec_enable, first_pass ? 1 : 0, sizeof(int), st));
    // CG stopping tolerance of this pass (slot 2, read by the captured k_cg_beta): slot 0 first pass
    // (cg_rtol), slot 1 the correction passes (cg_rtol_corr, reading R6)
    CK(cudaMemcpyAsync(c->cg_rtol_dev + 2, c->cg_rtol_dev + (first_pass ? 0 : 1), sizeof(double),
                       cudaMemcpyDeviceToDevice, st));
    if (!init_cg) {  // CG: x = 0, r = p = b
      k_zero<<<gme, TPB, 0, st>>>(me, c->cg_x);
      cudaMemcpyAsync(c->cg_r, c->bvec, sizeof(double) * (size_t)B * me, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(c->cg_p, c->bvec, sizeof(double) * (size_t)B * me, cudaMemcpyDeviceToDevice, st);
      dot(c, me, c->bvec, c->bvec, skip);
      k_cg_init_scalars<<<B, TPB, 0, st>>>(B, c->part, c->cg_rr, c->cg_bn, c->cg_done, c->cg_iters, skip);
      k_zero<<<gn, TPB, 0, st>>>(n, c->cg_z);
      c->launches += 5;
    } else {  // Init-CG: start from the projection onto the first pass's directions
      k_rec_dots<<<dim3(DOT_BLOCKS, B, KREC), TPB, 0, st>>>(me, B, c->rec_P, c->bvec, c->rec_n, skip, c->rec_part);
      k_rec_coef<<<B * KREC, TPB, 0, st>>>(B, c->rec_part, c->rec_PQ, c->rec_n, skip, c->rec_coef);
      k_rec_start<<<gme, TPB, 0, st>>>(me, B, c->rec_P, c->rec_Q, c->rec_coef, c->rec_n, c->bvec, c->cg_x, c->cg_r,
                                       c->cg_p);
      k_dot_partial<<<dim3(DOT_BLOCKS, c->B), TPB, 0, st>>>(me, c->bvec, c->bvec, c->part_b, skip);
      dot(c, me, c->cg_r, c->cg_r, skip);
      k_cg_init_scalars2<<<B, TPB, 0, st>>>(B, c->part, c->part_b, c->cg_rtol_corr, c->cg_rr, c->cg_bn,
                                                  c->cg_done, c->cg_iters, skip);
      k_rec_start_z<<<gn, TPB, 0, st>>>(n, B, c->rec_VN, c->rec_coef, c->rec_n, c->cg_z);
      c->launches += 7;
    }
    prof_end(c);
    const bool use_graph = !c->profiling && c->cg_exec != nullptr;
    if (use_graph) {
      CK(cudaMemsetAsync(c->active, 0, sizeof(int), st));
      CK(cudaMemsetAsync(c->cg_loop, 0, sizeof(int), st));
      CK(cudaGraphLaunch(c->cg_exec, st));
      CK(cudaMemcpyAsync(c->h_pinned_int + 4 * B, c->cg_loop, sizeof(int), cudaMemcpyDeviceToHost, st));
      c->graph_pending_loops = true;
    } else {
      for (int it = 0; it < c->opt.cg_maxit; ++it) {
        CK(cudaMemsetAsync(c->active, 0, sizeof(int), st));
        cg_iteration(c);
        int* h_active = c->h_pinned_int + 4 * B;
        CK(cudaMemcpyAsync(h_active, c->active, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (*h_active == 0) break;
      }
    }
    if (c->rec_on && first_pass) {
      k_rec_count<<<nblk(B), TPB, 0, st>>>(B, c->cg_iters, c->rec_n);
      c->launches++;
    }
    // dy = x ; dx = K^{-1}(-r_gamma - G^T dy) = -t - sum_k alpha_k vn_k
    prof_begin(c, 4);
    cudaMemcpyAsync(dy, c->cg_x, sizeof(double) * (size_t)B * me, cudaMemcpyDeviceToDevice, st);
    // dx = -t - K^{-1} G^T dy with K^{-1} G^T dy accumulated during CG (no extra sweep pair)
    k_dx_from_acc<<<gn, TPB, 0, st>>>(n, c->tn, c->cg_z, dx);
    c->launches++;
    prof_end(c);
    int* h_iters = c->h_pinned_int + 3 * B;
    CK(cudaMemcpyAsync(h_iters, c->cg_iters, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < B; ++b) kcg[b] = h_iters[b];
    if (c->graph_pending_loops) {  // kernels launched by the graph loop (telemetry)
      c->launches += (int64_t)c->h_pinned_int[4 * B] * c->cg_body_launches;
      c->graph_pending_loops = false;
    }
  } else {
    k_copy_neg<<<gn, TPB, 0, st>>>(n, c->rg, -1.0, dx);
    c->launches++;
    prof_end(c);
    ksolve(c, dx, skip);
  }
  if (mi > 0) {
    prof_begin(c, 4);
    k_recover<<<gmi, TPB, 0, st>>>(mi, n, c->h_rowptr, c->h_col2, c->h_val, c->h_nnz, dx, r2, r4, c->d_s, ds, dz,
                                   skip);
    c->launches++;
    prof_end(c);
  }
  CK(cudaGetLastError());
  return CKKT_OK;
}

// residual of (dx internal, ds, dy, dz) against r (r1 original order); omega/resinf [B] device at offset
void residual(ckkt_ctx* c, const double* r1, const double* r2, const double* r3, const double* r4, const double* dx,
              const double* ds, const double* dy, const double* dz, double* rho1, double* rho2, double* rho3,
              double* rho4, double* omega, double* resinf) {
  const int n = c->n, me = c->me, mi = c->mi, B = c->B;
  const int64_t rows = (int64_t)n + 2 * mi + me;
  ResArgs a;
  a.n = n; a.me = me; a.mi = mi;
  a.perm2 = c->S.perm2;
  a.ws_ptr = c->ws_ptr; a.ws_col = c->ws_col; a.wsv = c->wsv; a.sig = c->sig_i; a.ws_nnz = c->ws_nnz;
  a.gt_ptr = c->gt_ptr; a.gt_e = c->gt_e; a.gt_r = c->gt_r;
  a.ht_ptr = c->ht_ptr; a.ht_e = c->ht_e; a.ht_r = c->ht_r;
  a.g_rowptr = c->g_rowptr; a.g_col2 = c->g_col2; a.h_rowptr = c->h_rowptr; a.h_col2 = c->h_col2;
  a.w_val = c->w_val; a.g_val = c->gv; a.h_val = c->h_val; a.sigma = c->sigma; a.d_s = c->d_s; a.delta = c->delta;
  a.gtv = c->gtv; a.htv = c->htv;
  a.w_nnz = c->w_nnz; a.g_nnz = c->g_nnz; a.h_nnz = c->h_nnz;
  a.r1 = r1; a.r2 = r2; a.r3 = r3; a.r4 = r4;
  a.dx = dx; a.ds = ds; a.dy = dy; a.dz = dz;
  a.rho1 = rho1; a.rho2 = rho2; a.rho3 = rho3; a.rho4 = rho4;
  a.skip = c->notpd;
  cudaStream_t st = c->stream;
  prof_begin(c, 4);
  cudaMemsetAsync(omega, 0, sizeof(double) * B, st);
  cudaMemsetAsync(resinf, 0, sizeof(double) * B, st);
  k_kaug_residual<<<dim3(nblk(rows), B), TPB, 0, st>>>(a, reinterpret_cast<unsigned long long*>(omega),
                                                       reinterpret_cast<unsigned long long*>(resinf));
  c->launches += 1;
  prof_end(c);
}

}  // namespace

extern "C" ckkt_status ckkt_solve(ckkt_ctx* c, const double* r1, const double* r2, const double* r3, const double* r4,
                                  double* dx, double* ds, double* dy, double* dz, ckkt_info* info) {
  NvtxRange nvtx_range("ckkt_solve");
  if (!c || !c->has_device || !c->factored) return CKKT_INVALID_ARG;
  const int n = c->n, me = c->me, mi = c->mi, B = c->B;
  if (!r1 || !dx || (me && (!r3 || !dy)) || (mi && (!r2 || !r4 || !ds || !dz))) return CKKT_INVALID_ARG;
  CK(cudaSetDevice(c->opt.device));
  cudaStream_t st = c->stream;
  const dim3 gn(nblk(n), B), gme(nblk(std::max(me, 1)), B), gmi(nblk(std::max(mi, 1)), B);
  std::vector<int> kcg, kcg_total(B, 0), nref(B, 0);
  // unrefined pass: step in (dxi, ds, dy, dz)
  ckkt_status s = solve_pass(c, r1, 0, r2, r3, r4, c->dxi, ds, dy, dz, c->notpd, kcg, true);
  if (s != CKKT_OK) return s;
  for (int b = 0; b < B; ++b) kcg_total[b] = kcg[b];
  std::vector<int> kcg0 = kcg;
  residual(c, r1, r2, r3, r4, c->dxi, ds, dy, dz, c->rho1, c->rho2, c->rho3, c->rho4, c->omega, c->resinf);
  CK(cudaMemcpyAsync(c->h_pinned_dbl, c->omega, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c->h_pinned_dbl + B, c->resinf, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c->h_pinned_int, c->notpd, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<double> omega(B), omega0(B), prev(B), rinf(B);
  std::vector<int> notpd(B), done(B, 0);
  for (int b = 0; b < B; ++b) {
    omega[b] = omega0[b] = prev[b] = c->h_pinned_dbl[b];
    rinf[b] = c->h_pinned_dbl[B + b];
    notpd[b] = c->h_pinned_int[b];
    done[b] = notpd[b] || !(omega[b] > c->opt.ref_tol);
  }
  for (int it = 0; it < c->opt.ref_maxit; ++it) {
    bool any = false;
    for (int b = 0; b < B; ++b) any |= !done[b];
    if (!any) break;
    int* h_skip = c->h_pinned_int + B;  // previous H2D copies from this region completed at the last sync
    for (int b = 0; b < B; ++b) h_skip[b] = done[b];
    CK(cudaMemcpyAsync(c->skipflag, h_skip, sizeof(int) * B, cudaMemcpyHostToDevice, st));
    // correction: solve K_aug delta = rho  (i.e. right-hand side "r" = -rho)
    prof_begin(c, 4);
    k_copy_neg<<<gn, TPB, 0, st>>>(n, c->rho1, -1.0, c->rho1b);
    if (mi) {
      k_copy_neg<<<gmi, TPB, 0, st>>>(mi, c->rho2, -1.0, c->rho2b);
      k_copy_neg<<<gmi, TPB, 0, st>>>(mi, c->rho4, -1.0, c->rho4b);
    }
    if (me) k_copy_neg<<<gme, TPB, 0, st>>>(me, c->rho3, -1.0, c->rho3b);
    c->launches += 4;
    prof_end(c);
    s = solve_pass(c, c->rho1b, 1, c->rho2b, c->rho3b, c->rho4b, c->cdx, c->cds, c->cdy, c->cdz, c->skipflag, kcg,
                   false);
    if (s != CKKT_OK) return s;
    // trial = d + correction
    prof_begin(c, 4);
    k_axpy_sel<<<gn, TPB, 0, st>>>(n, c->dxi, c->cdx, c->dxi2);
    if (mi) {
      k_axpy_sel<<<gmi, TPB, 0, st>>>(mi, ds, c->cds, c->ds2);
      k_axpy_sel<<<gmi, TPB, 0, st>>>(mi, dz, c->cdz, c->dz2);
    }
    if (me) k_axpy_sel<<<gme, TPB, 0, st>>>(me, dy, c->cdy, c->dy2);
    c->launches += 4;
    prof_end(c);
    residual(c, r1, r2, r3, r4, c->dxi2, c->ds2, c->dy2, c->dz2, c->rho1b, c->rho2b, c->rho3b, c->rho4b,
             c->omega + B, c->resinf + B);
    CK(cudaMemcpyAsync(c->h_pinned_dbl + 2 * B, c->omega + B, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(c->h_pinned_dbl + 3 * B, c->resinf + B, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < B; ++b) {
      int acc = 0;
      if (!done[b]) {
        double om = c->h_pinned_dbl[2 * B + b];
        nref[b]++;
        kcg_total[b] += kcg[b];
        if (om < omega[b]) {
          acc = 1;
          omega[b] = om;
          rinf[b] = c->h_pinned_dbl[3 * B + b];
        }
        if (!(om > c->opt.ref_tol) || om > 0.5 * prev[b]) done[b] = 1;
        prev[b] = om;
      }
      c->h_pinned_int[2 * B + b] = acc;
    }
    CK(cudaMemcpyAsync(c->accflag, c->h_pinned_int + 2 * B, sizeof(int) * B, cudaMemcpyHostToDevice, st));
    prof_begin(c, 4);
    k_copy_sel<<<gn, TPB, 0, st>>>(n, c->dxi2, c->dxi, c->accflag);
    k_copy_sel<<<gn, TPB, 0, st>>>(n, c->rho1b, c->rho1, c->accflag);
    if (mi) {
      k_copy_sel<<<gmi, TPB, 0, st>>>(mi, c->ds2, ds, c->accflag);
      k_copy_sel<<<gmi, TPB, 0, st>>>(mi, c->dz2, dz, c->accflag);
      k_copy_sel<<<gmi, TPB, 0, st>>>(mi, c->rho2b, c->rho2, c->accflag);
      k_copy_sel<<<gmi, TPB, 0, st>>>(mi, c->rho4b, c->rho4, c->accflag);
    }
    if (me) {
      k_copy_sel<<<gme, TPB, 0, st>>>(me, c->dy2, dy, c->accflag);
      k_copy_sel<<<gme, TPB, 0, st>>>(me, c->rho3b, c->rho3, c->accflag);
    }
    c->launches += 8;
    prof_end(c);
  }
  prof_begin(c, 4);
  k_unpermute<<<gn, TPB, 0, st>>>(n, c->S.perm2, c->dxi, dx, c->notpd);
  if (mi) {
    k_nan_fill<<<gmi, TPB, 0, st>>>(mi, ds, c->notpd);
    k_nan_fill<<<gmi, TPB, 0, st>>>(mi, dz, c->notpd);
  }
  if (me) k_nan_fill<<<gme, TPB, 0, st>>>(me, dy, c->notpd);
  c->launches += 4;
  prof_end(c);
  CK(cudaGetLastError());
  ckkt_status worst = CKKT_OK;
  if (info) {
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < B; ++b) {
      ckkt_info& I = info[b];
      I.k_cg = kcg0[b];
      I.k_cg_total = kcg_total[b];
      I.n_ref = nref[b];
      I.rel_res = omega[b];
      I.rel_res_unrefined = omega0[b];
      I.res_inf = rinf[b];
      ckkt_status sb = CKKT_OK;
      if (notpd[b]) sb = CKKT_NOT_PD;
      else if (me && kcg0[b] >= c->opt.cg_maxit) sb = CKKT_CG_NO_CONVERGENCE;
      else if (c->opt.ref_maxit > 0 && omega[b] > c->opt.ref_tol && omega[b] > 1e-10) sb = CKKT_REFINE_NOT_CONVERGED;
      I.status = sb;
      if (sb != CKKT_OK && (worst == CKKT_OK || sb == CKKT_NOT_PD)) worst = sb;
    }
  }
  return worst;
}

extern "C" ckkt_status ckkt_iterate_host(ckkt_ctx* c, const double* w_val, const double* g_val, const double* h_val,
                                         const double* sigma_x, const double* d_s, const double* delta_x,
                                         const double* r1, const double* r2, const double* r3, const double* r4,
                                         double* dx, double* ds, double* dy, double* dz, int32_t* not_pd,
                                         ckkt_info* info) {
  NvtxRange nvtx_range("ckkt_iterate_host");
  if (!c || !c->has_device) return CKKT_INVALID_ARG;
  CK(cudaSetDevice(c->opt.device));
  const int B = c->B;
  const size_t Bn = (size_t)B * c->n, Bme = (size_t)B * c->me, Bmi = (size_t)B * c->mi;
  cudaStream_t st = c->stream;
  auto h2d = [&](double* dst, const double* src, size_t cnt, cudaStream_t sx) -> cudaError_t {
    if (!src || cnt == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, sizeof(double) * cnt, cudaMemcpyHostToDevice, sx);
  };
  // the matrix values first (the refactorization needs them), then the right-hand sides on the
  // auxiliary stream, after the values (one link), overlapping the factorization; the solve waits
  // for them.  (The previous call ended with a stream synchronisation, so the staging is free.)
  CK(h2d(c->st_w, w_val, (size_t)B * c->w_nnz, st));
  CK(h2d(c->st_g, g_val, (size_t)B * c->g_nnz, st));
  CK(h2d(c->st_h, h_val, (size_t)B * c->h_nnz, st));
  CK(h2d(c->st_sig, sigma_x, Bn, st));
  CK(h2d(c->st_ds, d_s, Bmi, st));
  CK(h2d(c->st_del, delta_x, B, st));
  CK(cudaEventRecord(c->ev_vals, st));
  CK(cudaStreamWaitEvent(c->st_aux, c->ev_vals, 0));
  CK(h2d(c->st_r1, r1, Bn, c->st_aux));
  CK(h2d(c->st_r2, r2, Bmi, c->st_aux));
  CK(h2d(c->st_r3, r3, Bme, c->st_aux));
  CK(h2d(c->st_r4, r4, Bmi, c->st_aux));
  CK(cudaEventRecord(c->ev_rhs, c->st_aux));
  ckkt_status s = ckkt_refactor(c, c->st_w, c->st_g, c->st_h, c->st_sig, c->st_ds, delta_x ? c->st_del : nullptr,
                                c->st_notpd, nullptr);
  CK(cudaStreamWaitEvent(st, c->ev_rhs, 0));
  if (s != CKKT_OK) {
    CK(cudaStreamSynchronize(st));
    return s;
  }
  std::vector<ckkt_info> tmp(B);
  s = ckkt_solve(c, c->st_r1, c->st_r2, c->st_r3, c->st_r4, c->st_dx, c->st_ds_o, c->st_dy, c->st_dz,
                 info ? info : tmp.data());
  auto d2h = [&](double* dst, const double* src, size_t cnt) -> cudaError_t {
    if (!dst || cnt == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st);
  };
  CK(d2h(dx, c->st_dx, Bn));
  CK(d2h(ds, c->st_ds_o, Bmi));
  CK(d2h(dy, c->st_dy, Bme));
  CK(d2h(dz, c->st_dz, Bmi));
  if (not_pd) CK(cudaMemcpyAsync(not_pd, c->st_notpd, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return s;
}

// ---------------------------------------------------------------------------------------------
// Debug export (not part of include/ckkt.h): copies internal arrays to host memory.
//   what: 0 = L storage (all instances), 1 = K values, 2 = perm2, 3 = sfirst, 4 = srowptr (int64),
//         5 = srows, 6 = pofs (int64), 7 = kp (int64), 8 = ki
// Returns the element count when host == NULL.
// ---------------------------------------------------------------------------------------------
// Debug timing of the kernels of one triangular solve pair on x = ones (ms, averaged over reps):
// out[0] = forward sweep, out[1] = backward sweep, out[2] = refactor.
extern "C" int ckkt_debug_time(ckkt_ctx* c, int reps, double* out) {
  if (!c || !c->has_device || !c->factored) return CKKT_INVALID_ARG;
  {
    int nw = getenv("CKKT_NOWAIT") ? 1 : 0;
    cudaMemcpyToSymbol(g_debug_nowait, &nw, sizeof(int));
  }
  cudaStream_t st = c->stream;
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  float f = 0, b = 0, t;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, st);
    launch_fwd(c, c->tn, nullptr);
    cudaEventRecord(e1, st);
    launch_bwd(c, c->tn, nullptr);
    cudaEventRecord(e2, st);
    cudaEventSynchronize(e2);
    cudaEventElapsedTime(&t, e0, e1);
    f += t;
    cudaEventElapsedTime(&t, e1, e2);
    b += t;
  }
  out[0] = f / reps;
  out[1] = b / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  return cudaGetLastError() == cudaSuccess ? 0 : CKKT_CUDA_ERROR;
}

// Debug: run one backward sweep recording per-supernode (ticket, wake, end, warp) timestamps.
extern "C" int ckkt_debug_trace_bwd(ckkt_ctx* c, unsigned long long* host_ts) {
  if (!c || !c->has_device || !c->factored) return CKKT_INVALID_ARG;
  {
    int nw = getenv("CKKT_NOWAIT") ? 1 : 0;
    cudaMemcpyToSymbol(g_debug_nowait, &nw, sizeof(int));
  }
  unsigned long long* d = nullptr;
  cudaMalloc(&d, sizeof(unsigned long long) * 4 * c->A.ns);
  cudaMemset(d, 0, sizeof(unsigned long long) * 4 * c->A.ns);
  cudaMemcpyToSymbol(g_debug_ts, &d, sizeof(d));
  unsigned long long* dph = nullptr;
  if (getenv("CKKT_TRACE_FWD")) {
    launch_fwd(c, c->tn, nullptr);
  } else if (getenv("CKKT_TRACE_FACTOR")) {
    cudaMalloc(&dph, sizeof(unsigned long long) * 8 * c->A.ns);
    cudaMemset(dph, 0, sizeof(unsigned long long) * 8 * c->A.ns);
    cudaMemcpyToSymbol(g_debug_ph, &dph, sizeof(dph));
    ckkt_refactor(c, c->w_val, c->g_val, c->h_val, c->sigma, c->d_s, c->delta, nullptr, nullptr);
  } else {
    launch_fwd(c, c->tn, nullptr);  // (the forward sweep's first launch bumps the sweep epochs)
    launch_bwd(c, c->tn, nullptr);
  }
  cudaStreamSynchronize(c->stream);
  cudaMemcpy(host_ts, d, sizeof(unsigned long long) * 4 * c->A.ns, cudaMemcpyDeviceToHost);
  if (dph) {
    FILE* fp = fopen("/tmp/ckkt_phases.bin", "wb");
    std::vector<unsigned long long> hph(8 * (size_t)c->A.ns);
    cudaMemcpy(hph.data(), dph, sizeof(unsigned long long) * hph.size(), cudaMemcpyDeviceToHost);
    fwrite(hph.data(), 8, hph.size(), fp);
    fclose(fp);
    unsigned long long* z2 = nullptr;
    cudaMemcpyToSymbol(g_debug_ph, &z2, sizeof(z2));
    cudaFree(dph);
  }
  unsigned long long* z = nullptr;
  cudaMemcpyToSymbol(g_debug_ts, &z, sizeof(z));
  cudaFree(d);
  return 0;
}

extern "C" const char* ckkt_debug_error_string() { return cudaGetErrorString(last_cuda_error); }

extern "C" int64_t ckkt_debug_get(const ckkt_ctx* c, int what, void* host) {
  if (!c) return -1;
  const auto& A = c->A;
  auto cp = [&](const void* src, size_t bytes, bool dev) -> void {
    if (!host) return;
    if (dev) cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost);
    else std::memcpy(host, src, bytes);
  };
  switch (what) {
    case 0: cp(c->L, sizeof(double) * c->B * c->Lsize, true); return (int64_t)c->B * c->Lsize;
    case 1: cp(c->Kval, sizeof(double) * c->B * c->nnzk, true); return (int64_t)c->B * c->nnzk;
    case 2: cp(A.perm2.data(), 4 * A.perm2.size(), false); return A.perm2.size();
    case 3: cp(A.sfirst.data(), 4 * A.sfirst.size(), false); return A.sfirst.size();
    case 4: cp(A.srowptr.data(), 8 * A.srowptr.size(), false); return A.srowptr.size();
    case 5: cp(A.srows.data(), 4 * A.srows.size(), false); return A.srows.size();
    case 6: cp(A.pofs.data(), 8 * A.pofs.size(), false); return A.pofs.size();
    case 7: cp(A.kp.data(), 8 * A.kp.size(), false); return A.kp.size();
    case 8: cp(A.ki.data(), 4 * A.ki.size(), false); return A.ki.size();
    case 9: cp(A.ch_ptr.data(), 4 * A.ch_ptr.size(), false); return A.ch_ptr.size();
    case 10: cp(A.ch_list.data(), 4 * A.ch_list.size(), false); return A.ch_list.size();
    case 11: cp(A.relofs.data(), 8 * A.relofs.size(), false); return A.relofs.size();
    case 12: cp(A.relmap.data(), 4 * A.relmap.size(), false); return A.relmap.size();
    case 13: cp(A.uofs.data(), 8 * A.uofs.size(), false); return A.uofs.size();
    case 14: cp(c->Ub, sizeof(double) * c->B * c->Usize, true); return (int64_t)c->B * c->Usize;
    case 15: cp(A.kmap.data(), 4 * A.kmap.size(), false); return A.kmap.size();
    case 16: cp(A.wt_ptr.data(), 8 * A.wt_ptr.size(), false); return A.wt_ptr.size();
    case 17: cp(A.wt_idx.data(), 4 * A.wt_idx.size(), false); return A.wt_idx.size();
    case 18: cp(A.jt_ptr.data(), 8 * A.jt_ptr.size(), false); return A.jt_ptr.size();
    case 19: cp(A.jt_a.data(), 4 * A.jt_a.size(), false); return A.jt_a.size();
    case 20: cp(A.jt_b.data(), 4 * A.jt_b.size(), false); return A.jt_b.size();
    case 21: cp(A.jt_r.data(), 4 * A.jt_r.size(), false); return A.jt_r.size();
    case 22: cp(A.dslot.data(), 4 * A.dslot.size(), false); return A.dslot.size();
  }
  return -1;
}
