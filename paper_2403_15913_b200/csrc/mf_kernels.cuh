// Multifrontal supernodal Cholesky and triangular-solve kernels for sm_100a (FP64).
// Included by ckkt.cu inside its anonymous namespace.
//
// Factor, front of supernode s = [panel P (m x w) | update block U_s ((m-w)^2, col-major)]:
//   P <- A(rows of s, cols of s) + panel part of the children's update matrices (extend-add)
//   P <- Cholesky of its first w columns (L11, L21); L11 <- L11^{-1} in place
//   U_s <- -L21 L21^T (FP64 DMMA tiles mma.sync.m8n8k4 for big fronts) + trailing part of the
//          children's update matrices
// Solves: forward with multifrontal update vectors u_s = v[w:m] - L21 y_s,
// backward x_s = L11^{-T}(y_s - L21^T x_R).
//
// Two granularities per level: "small" supernodes (m*w <= SMALL_PANEL) get one warp each and a
// 4 KB shared-memory panel; "big" ones one CTA with the whole panel in shared memory.
// Everything is deterministic: children are assembled in a fixed order, no value atomics.

constexpr int SMALL_PANEL = 512;   // doubles
constexpr int SMALL_WARPS = 8;     // warps per CTA for the small-supernode kernels
constexpr int BIG_THREADS = 256;

struct SymDev {
  const int32_t* sfirst;
  const int64_t* srowptr;
  const int32_t* srows;
  const int64_t* pofs;
  const int32_t* level_list;
  const int32_t* ch_ptr;
  const int32_t* ch_list;
  const int64_t* relofs;
  const int32_t* relmap;
  const int64_t* uofs;
  const int64_t* vofs;
  const int64_t* kp;
  const int32_t* kmap;
  const int32_t* perm2;
};

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ============================================================================================
// factor: small supernodes, one warp each, panel staged in shared memory (ld = m)
// ============================================================================================
__global__ void __launch_bounds__(32 * SMALL_WARPS)
    k_factor_small(SymDev S, const int32_t* __restrict__ list, int cnt, double* L, int64_t Lsize, double* Ub,
                   int64_t Usize, const double* __restrict__ Kval, int64_t nnzk, int* notpd, int* minpiv) {
  __shared__ double panel_all[SMALL_WARPS][SMALL_PANEL];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * SMALL_WARPS + wid;
  if (idx >= cnt) return;
  const int b = blockIdx.y;
  const int s = list[idx];
  double* Ps = panel_all[wid];
  const double* Kb = Kval + b * nnzk;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w;
  double* P = L + b * Lsize + S.pofs[s];
  double* U = Ub + b * Usize + S.uofs[s];
  for (int i = lane; i < m * w; i += 32) Ps[i] = 0.0;
  __syncwarp();
  for (int64_t k = S.kp[f] + lane; k < S.kp[f + w]; k += 32) Ps[S.kmap[k]] = Kb[k];
  __syncwarp();
  // panel part of the children's update matrices (columns rel[j] < w)
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = (int)(S.srowptr[c + 1] - S.srowptr[c]) - (S.sfirst[c + 1] - S.sfirst[c]);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    for (int j = 0; j < mc; ++j) {
      const int rj = rel[j];
      if (rj >= w) break;  // rel is increasing
      for (int i = j + lane; i < mc; i += 32) Ps[rel[i] + rj * m] += Uc[i + (int64_t)j * mc];
    }
    __syncwarp();
  }
  // Cholesky of the first w columns
  for (int j = 0; j < w; ++j) {
    double d = Ps[j + j * m];
    if (!(d > 0.0) || !isfinite(d)) {
      if (lane == 0) {
        notpd[b] = 1;
        atomicMin(&minpiv[b], f + j);
      }
      d = nan("");
    }
    const double piv = sqrt(d);
    __syncwarp();
    if (lane == 0) Ps[j + j * m] = piv;
    for (int i = j + 1 + lane; i < m; i += 32) Ps[i + j * m] /= piv;
    __syncwarp();
    for (int c = j + 1; c < w; ++c) {
      const double lc = Ps[c + j * m];
      for (int i = c + lane; i < m; i += 32) Ps[i + c * m] -= Ps[i + j * m] * lc;
    }
    __syncwarp();
  }
  // L11 <- L11^{-1} (rows in order; Z_ij = (delta_ij - sum_{j<=k<i} L_ik Z_kj) / L_ii), w <= 32 here
  for (int i = 0; i < w; ++i) {
    double z = 0.0;
    if (lane <= i) {
      z = (lane == i) ? 1.0 : 0.0;
      for (int k = lane; k < i; ++k) z -= Ps[i + k * m] * Ps[k + lane * m];
      z /= Ps[i + i * m];
    }
    __syncwarp();
    if (lane <= i) Ps[i + lane * m] = z;
    __syncwarp();
  }
  for (int i = lane; i < m * w; i += 32) P[i] = Ps[i];
  // U_s = -L21 L21^T (lower), then trailing part of the children
  for (int j = 0; j < mu; ++j)
    for (int i = j + lane; i < mu; i += 32) {
      double t = 0.0;
      for (int k = 0; k < w; ++k) t += Ps[w + i + k * m] * Ps[w + j + k * m];
      U[i + (int64_t)j * mu] = -t;
    }
  __syncwarp();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = (int)(S.srowptr[c + 1] - S.srowptr[c]) - (S.sfirst[c + 1] - S.sfirst[c]);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    for (int j = 0; j < mc; ++j) {
      const int rj = rel[j];
      if (rj < w) continue;
      for (int i = j + lane; i < mc; i += 32) U[(rel[i] - w) + (int64_t)(rj - w) * mu] += Uc[i + (int64_t)j * mc];
    }
    __syncwarp();
  }
}

// ============================================================================================
// factor: big supernodes, one CTA each, panel in dynamic shared memory with ld = mp (m padded
// to a multiple of 8, w padded to a multiple of 4 with zero columns) for the DMMA SYRK.
// ============================================================================================
__global__ void __launch_bounds__(BIG_THREADS)
    k_factor_big(SymDev S, const int32_t* __restrict__ list, double* L, int64_t Lsize, double* Ub, int64_t Usize,
                 const double* __restrict__ Kval, int64_t nnzk, int* notpd, int* minpiv) {
  extern __shared__ double Ps[];
  __shared__ double piv_s;
  const int s = list[blockIdx.x];
  const int b = blockIdx.y;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const double* Kb = Kval + b * nnzk;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w;
  const int mp = (m + 7) & ~7, wp = (w + 3) & ~3;
  double* P = L + b * Lsize + S.pofs[s];
  double* U = Ub + b * Usize + S.uofs[s];
  for (int i = tid; i < mp * wp; i += nt) Ps[i] = 0.0;
  __syncthreads();
  for (int64_t k = S.kp[f] + tid; k < S.kp[f + w]; k += nt) {
    const int q = S.kmap[k];
    Ps[(q % m) + (q / m) * mp] = Kb[k];
  }
  __syncthreads();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = (int)(S.srowptr[c + 1] - S.srowptr[c]) - (S.sfirst[c + 1] - S.sfirst[c]);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    // columns j of U_c with rel[j] < w: a prefix; warps over columns, lanes over rows
    int jw = 0;
    while (jw < mc && rel[jw] < w) ++jw;
    for (int j = warp; j < jw; j += nwarp) {
      const int rj = rel[j];
      for (int i = j + lane; i < mc; i += 32) Ps[rel[i] + rj * mp] += Uc[i + (int64_t)j * mc];
    }
    __syncthreads();
  }
  // Cholesky of the first w columns in shared memory
  for (int j = 0; j < w; ++j) {
    if (tid == 0) {
      double d = Ps[j + j * mp];
      if (!(d > 0.0) || !isfinite(d)) {
        notpd[b] = 1;
        atomicMin(&minpiv[b], f + j);
        d = nan("");
      }
      piv_s = sqrt(d);
      Ps[j + j * mp] = piv_s;
    }
    __syncthreads();
    const double pv = piv_s;
    for (int i = j + 1 + tid; i < m; i += nt) Ps[i + j * mp] /= pv;
    __syncthreads();
    const int nrest = w - j - 1;
    for (int e = tid; e < nrest * m; e += nt) {
      const int c = j + 1 + e / m, i = e % m;
      if (i >= c) Ps[i + c * mp] -= Ps[i + j * mp] * Ps[c + j * mp];
    }
    __syncthreads();
  }
  // U_s = -L21 L21^T: 8x8 DMMA tiles of the lower triangle, k = 0..wp step 4
  {
    const int nb = (mu + 7) >> 3;
    const int ntile = nb * (nb + 1) / 2;
    const int g = lane >> 2, t4 = lane & 3;
    for (int tI = warp; tI < ntile; tI += nwarp) {
      // tile index -> (I, J), I >= J
      int I = (int)((sqrt(8.0 * tI + 1.0) - 1.0) * 0.5);
      while ((I + 1) * (I + 2) / 2 <= tI) ++I;
      while (I * (I + 1) / 2 > tI) --I;
      const int J = tI - I * (I + 1) / 2;
      double c0 = 0.0, c1 = 0.0;
      const double* ra = Ps + w + I * 8 + g;
      const double* rb = Ps + w + J * 8 + g;
      for (int k = 0; k < wp; k += 4) dmma_8x8x4(c0, c1, ra[(k + t4) * mp], rb[(k + t4) * mp]);
      const int row = I * 8 + g, col = J * 8 + 2 * t4;
      if (row < mu) {
        if (col < mu) U[row + (int64_t)col * mu] = -c0;
        if (col + 1 < mu) U[row + (int64_t)(col + 1) * mu] = -c1;
      }
    }
  }
  // L11 <- L11^{-1} in shared memory, rows in order
  for (int i = 0; i < w; ++i) {
    double z = 0.0;
    const int j = tid;
    if (j <= i) {
      z = (j == i) ? 1.0 : 0.0;
      for (int k = j; k < i; ++k) z -= Ps[i + k * mp] * Ps[k + j * mp];
      z /= Ps[i + i * mp];
    }
    __syncthreads();
    if (j <= i) Ps[i + j * mp] = z;
    __syncthreads();
  }
  // panel -> global (column-major, ld = m)
  for (int e = tid; e < m * w; e += nt) P[e] = Ps[(e % m) + (e / m) * mp];
  __syncthreads();  // U_s tile writes of this CTA are complete before the children add into it
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = (int)(S.srowptr[c + 1] - S.srowptr[c]) - (S.sfirst[c + 1] - S.sfirst[c]);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    int jw = 0;
    while (jw < mc && rel[jw] < w) ++jw;
    for (int j = jw + warp; j < mc; j += nwarp) {
      const int rj = rel[j] - w;
      for (int i = j + lane; i < mc; i += 32) U[(rel[i] - w) + (int64_t)rj * mu] += Uc[i + (int64_t)j * mc];
    }
    __syncthreads();
  }
}

// ============================================================================================
// forward solve L y = x (in place, internal order)
// ============================================================================================
// small: one warp per supernode; v = [x_s; 0] + sum_c ext(u_c); y = Z v[0:w]; u_s = v[w:] - L21 y
__global__ void __launch_bounds__(32 * SMALL_WARPS)
    k_fwd_small(SymDev S, const int32_t* __restrict__ list, int cnt, const double* __restrict__ L, int64_t Lsize,
                double* X, int n, double* Vb, int64_t Vsize, int max_m, const int* __restrict__ skip) {
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * SMALL_WARPS + wid;
  const int b = blockIdx.y;
  if (idx >= cnt || (skip && skip[b])) return;
  const int s = list[idx];
  double* v = smem + (size_t)wid * (max_m + 32);
  double* y = v + max_m;
  double* x = X + (int64_t)b * n;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w;
  const double* P = L + b * Lsize + S.pofs[s];
  for (int i = lane; i < m; i += 32) v[i] = (i < w) ? x[f + i] : 0.0;
  __syncwarp();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = (int)(S.srowptr[c + 1] - S.srowptr[c]) - (S.sfirst[c + 1] - S.sfirst[c]);
    const double* uc = Vb + b * Vsize + S.vofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    for (int i = lane; i < mc; i += 32) v[rel[i]] += uc[i];
    __syncwarp();
  }
  if (lane < w) {  // w <= 32 for small supernodes; Z's strict upper part is zero
    double t = 0.0;
#pragma unroll 4
    for (int k = 0; k < w; ++k) t += P[lane + (int64_t)k * m] * v[k];
    y[lane] = t;
    x[f + lane] = t;
  }
  __syncwarp();
  double* us = Vb + b * Vsize + S.vofs[s];
  for (int i = lane; i < mu; i += 32) {
    double t = v[w + i];
#pragma unroll 4
    for (int k = 0; k < w; ++k) t -= P[w + i + (int64_t)k * m] * y[k];
    us[i] = t;
  }
}

// big: one CTA per supernode; threads over rows, loads of each column coalesced
__global__ void __launch_bounds__(BIG_THREADS)
    k_fwd_big(SymDev S, const int32_t* __restrict__ list, const double* __restrict__ L, int64_t Lsize, double* X,
              int n, double* Vb, int64_t Vsize, const int* __restrict__ skip) {
  extern __shared__ double sv[];
  const int s = list[blockIdx.x];
  const int b = blockIdx.y;
  if (skip && skip[b]) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* x = X + (int64_t)b * n;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w;
  double* v = sv;      // [m]
  double* y = sv + m;  // [w]
  const double* P = L + b * Lsize + S.pofs[s];
  for (int i = tid; i < m; i += nt) v[i] = (i < w) ? x[f + i] : 0.0;
  __syncthreads();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = (int)(S.srowptr[c + 1] - S.srowptr[c]) - (S.sfirst[c + 1] - S.sfirst[c]);
    const double* uc = Vb + b * Vsize + S.vofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    for (int i = tid; i < mc; i += nt) v[rel[i]] += uc[i];
    __syncthreads();
  }
  for (int i = tid; i < w; i += nt) {
    double t = 0.0;
#pragma unroll 8
    for (int k = 0; k < w; ++k) t += P[i + (int64_t)k * m] * v[k];
    y[i] = t;
    x[f + i] = t;
  }
  __syncthreads();
  double* us = Vb + b * Vsize + S.vofs[s];
  for (int i = tid; i < mu; i += nt) {
    double t = v[w + i];
#pragma unroll 8
    for (int k = 0; k < w; ++k) t -= P[w + i + (int64_t)k * m] * y[k];
    us[i] = t;
  }
}

// ============================================================================================
// backward solve L^T x = y: x_s = Z^T (y_s - L21^T x_R)
// ============================================================================================
__global__ void __launch_bounds__(32 * SMALL_WARPS)
    k_bwd_small(SymDev S, const int32_t* __restrict__ list, int cnt, const double* __restrict__ L, int64_t Lsize,
                double* X, int n, int max_m, const int* __restrict__ skip) {
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * SMALL_WARPS + wid;
  const int b = blockIdx.y;
  if (idx >= cnt || (skip && skip[b])) return;
  const int s = list[idx];
  double* xr = smem + (size_t)wid * (max_m + 32);
  double* t = xr + max_m;
  double* x = X + (int64_t)b * n;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int64_t r0 = S.srowptr[s];
  const int m = (int)(S.srowptr[s + 1] - r0);
  const double* P = L + b * Lsize + S.pofs[s];
  for (int i = w + lane; i < m; i += 32) xr[i] = x[S.srows[r0 + i]];
  __syncwarp();
  // t_c = y_c - sum_i L21(i,c) x_R(i): lanes over rows, all columns accumulated before reducing
  for (int c = 0; c < w; ++c) {
    double a = 0.0;
    for (int i = w + lane; i < m; i += 32) a += P[i + (int64_t)c * m] * xr[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == c) t[c] = x[f + c] - a;
  }
  __syncwarp();
  if (lane < w) {  // x_i = sum_k Z(k, i) t_k  (Z strictly upper part is zero)
    double a = 0.0;
#pragma unroll 4
    for (int k = 0; k < w; ++k) a += P[k + (int64_t)lane * m] * t[k];
    x[f + lane] = a;
  }
}

__global__ void __launch_bounds__(BIG_THREADS)
    k_bwd_big(SymDev S, const int32_t* __restrict__ list, const double* __restrict__ L, int64_t Lsize, double* X,
              int n, const int* __restrict__ skip) {
  extern __shared__ double sb[];
  const int s = list[blockIdx.x];
  const int b = blockIdx.y;
  if (skip && skip[b]) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  double* x = X + (int64_t)b * n;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int64_t r0 = S.srowptr[s];
  const int m = (int)(S.srowptr[s + 1] - r0);
  const double* P = L + b * Lsize + S.pofs[s];
  double* xr = sb;     // [m] (rows >= w used)
  double* t = sb + m;  // [w]
  for (int i = w + tid; i < m; i += nt) xr[i] = x[S.srows[r0 + i]];
  __syncthreads();
  for (int c = warp; c < w; c += nwarp) {  // warp per column, lanes over rows (coalesced)
    double a = 0.0;
    for (int i = w + lane; i < m; i += 32) a += P[i + (int64_t)c * m] * xr[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) t[c] = x[f + c] - a;
  }
  __syncthreads();
  for (int i = warp; i < w; i += nwarp) {  // x_i = sum_{k>=i} Z(k, i) t_k: column i of Z
    double a = 0.0;
    for (int k = i + lane; k < w; k += 32) a += P[k + (int64_t)i * m] * t[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) x[f + i] = a;
  }
}
