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
// Scheduling: one persistent launch per factorization / forward sweep / backward sweep.  Tasks are
// supernodes in topological (level) order: a "big" task is one supernode processed by the whole CTA,
// a "small" task bundles up to SMALL_WARPS small supernodes of one level, one per warp.  CTAs take
// tickets from an atomic counter; a supernode starts once its dependencies (children for factor /
// forward, parent for backward) have published the launch epoch in their done flag (release/acquire).
// Tickets are handed out in topological order, so a CTA only ever waits on work already taken by a
// running CTA: no deadlock for any grid size.  Data written by other CTAs of the same launch is read
// with ld.global.cg (L2) so that stale L1 lines are never used.
// Everything is deterministic: children are assembled in a fixed order, no value atomics.

constexpr int SMALL_PANEL = 512;   // doubles of a small supernode panel (m * w)
constexpr int SMALL_WARPS = 8;     // warps per CTA; small supernodes per task
constexpr int MF_THREADS = 32 * SMALL_WARPS;

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
  const int32_t* sparent;
};

struct Sched {
  int ntask;                      // tasks per instance
  const int32_t* task_sn;         // [ntask * SMALL_WARPS], -1 = empty slot; big task uses slot 0
  const int32_t* task_big;        // [ntask]
  int* done;                      // [B * ns] epoch flags
  int* ctr;                       // [2] ticket counters (alternating per epoch)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ int g_debug_nowait = 0;  // debug only: skip dependency waits (timing experiments)
__device__ unsigned long long* g_debug_ts = nullptr;  // debug only: [ns][4] ticket/wake/end times of sweeps

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// poll with relaxed loads, then one acquire fence (cheaper than repeated ld.acquire)
__device__ __forceinline__ void wait_epoch(const int* p, int epoch) {
  if (g_debug_nowait) return;
  int ns = 32;
  while (ld_relaxed(p) != epoch) {
    __nanosleep(ns);
    ns = ns < 2048 ? 2 * ns : 2048;
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// release-side fence: makes this thread's prior writes visible at gpu scope before the flag store
// (acq_rel is much cheaper than the sequentially-consistent fence of __threadfence())
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int off_rows(const SymDev& S, int c) {
  return (int)(S.srowptr[c + 1] - S.srowptr[c]) - (S.sfirst[c + 1] - S.sfirst[c]);
}

// ticket -> (task, instance); the shared slot broadcasts it to the CTA
__device__ __forceinline__ int next_ticket(int* ctr_slot, int* sh) {
  __syncthreads();
  if (threadIdx.x == 0) *sh = atomicAdd(ctr_slot, 1);
  __syncthreads();
  return *sh;
}

// ============================================================================================
// factor
// ============================================================================================
// small supernode, one warp, panel in shared memory (ld = m)
__device__ void factor_small(const SymDev& S, int s, int b, int lane, double* Ps, double* L, int64_t Lsize,
                             double* Ub, int64_t Usize, const double* __restrict__ Kb, int* notpd, int* minpiv) {
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w;
  double* P = L + b * Lsize + S.pofs[s];
  double* U = Ub + b * Usize + S.uofs[s];
  for (int i = lane; i < m * w; i += 32) Ps[i] = 0.0;
  __syncwarp();
  for (int64_t k = S.kp[f] + lane; k < S.kp[f + w]; k += 32) Ps[S.kmap[k]] = Kb[k];
  __syncwarp();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {  // panel part of the children
    const int c = S.ch_list[ci];
    const int mc = off_rows(S, c);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    for (int j = 0; j < mc; ++j) {
      const int rj = rel[j];
      if (rj >= w) break;  // rel is increasing
      for (int i = j + lane; i < mc; i += 32) Ps[rel[i] + rj * m] += __ldcg(Uc + i + (int64_t)j * mc);
    }
    __syncwarp();
  }
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
  for (int i = 0; i < w; ++i) {  // L11 <- L11^{-1} (w <= 32)
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
  for (int j = 0; j < mu; ++j)  // U_s = -L21 L21^T (lower)
    for (int i = j + lane; i < mu; i += 32) {
      double t = 0.0;
      for (int k = 0; k < w; ++k) t += Ps[w + i + k * m] * Ps[w + j + k * m];
      U[i + (int64_t)j * mu] = -t;
    }
  __syncwarp();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {  // trailing part of the children
    const int c = S.ch_list[ci];
    const int mc = off_rows(S, c);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    for (int j = 0; j < mc; ++j) {
      const int rj = rel[j];
      if (rj < w) continue;
      for (int i = j + lane; i < mc; i += 32)
        U[(rel[i] - w) + (int64_t)(rj - w) * mu] += __ldcg(Uc + i + (int64_t)j * mc);
    }
    __syncwarp();
  }
}

// big supernode, whole CTA, panel in shared memory with ld = mp (m padded to 8, w padded to 4)
__device__ void factor_big(const SymDev& S, int s, int b, double* Ps, double* piv_s, double* L, int64_t Lsize,
                           double* Ub, int64_t Usize, const double* __restrict__ Kb, int* notpd, int* minpiv) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w;
  const int mp = (m + 7) & ~7, wp = (w + 3) & ~3;
  double* P = L + b * Lsize + S.pofs[s];
  double* U = Ub + b * Usize + S.uofs[s];
  for (int i = tid; i < mp * wp + 8; i += nt) Ps[i] = 0.0;
  __syncthreads();
  for (int64_t k = S.kp[f] + tid; k < S.kp[f + w]; k += nt) {
    const int q = S.kmap[k];
    Ps[(q % m) + (q / m) * mp] = Kb[k];
  }
  __syncthreads();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = off_rows(S, c);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    int jw = 0;
    while (jw < mc && rel[jw] < w) ++jw;
    for (int j = warp; j < jw; j += nwarp) {
      const int rj = rel[j];
      for (int i = j + lane; i < mc; i += 32) Ps[rel[i] + rj * mp] += __ldcg(Uc + i + (int64_t)j * mc);
    }
    __syncthreads();
  }
  for (int j = 0; j < w; ++j) {
    if (tid == 0) {
      double d = Ps[j + j * mp];
      if (!(d > 0.0) || !isfinite(d)) {
        notpd[b] = 1;
        atomicMin(&minpiv[b], f + j);
        d = nan("");
      }
      *piv_s = sqrt(d);
      Ps[j + j * mp] = *piv_s;
    }
    __syncthreads();
    const double pv = *piv_s;
    for (int i = j + 1 + tid; i < m; i += nt) Ps[i + j * mp] /= pv;
    __syncthreads();
    const int nrest = w - j - 1;
    for (int e = tid; e < nrest * m; e += nt) {
      const int c = j + 1 + e / m, i = e % m;
      if (i >= c) Ps[i + c * mp] -= Ps[i + j * mp] * Ps[c + j * mp];
    }
    __syncthreads();
  }
  {  // U_s = -L21 L21^T: 8x8 DMMA tiles of the lower triangle
    const int nb = (mu + 7) >> 3;
    const int ntile = nb * (nb + 1) / 2;
    const int g = lane >> 2, t4 = lane & 3;
    for (int tI = warp; tI < ntile; tI += nwarp) {
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
  for (int i = 0; i < w; ++i) {  // L11 <- L11^{-1}
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
  for (int e = tid; e < m * w; e += nt) P[e] = Ps[(e % m) + (e / m) * mp];
  __syncthreads();  // this CTA's U_s tile writes are complete before the children add into it
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    const int mc = off_rows(S, c);
    const double* Uc = Ub + b * Usize + S.uofs[c];
    const int32_t* rel = S.relmap + S.relofs[c];
    int jw = 0;
    while (jw < mc && rel[jw] < w) ++jw;
    for (int j = jw + warp; j < mc; j += nwarp) {
      const int rj = rel[j] - w;
      for (int i = j + lane; i < mc; i += 32)
        U[(rel[i] - w) + (int64_t)rj * mu] += __ldcg(Uc + i + (int64_t)j * mc);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(MF_THREADS)
    k_factor_persist(SymDev S, Sched Q, int ns, int B, int epoch, double* L, int64_t Lsize, double* Ub,
                     int64_t Usize, const double* __restrict__ Kval, int64_t nnzk, int* notpd, int* minpiv) {
  extern __shared__ double smem[];  // max(big panel, SMALL_WARPS small panels)
  __shared__ double piv_s;
  __shared__ int tk;
  if (blockIdx.x == 0 && threadIdx.x == 0) Q.ctr[(epoch + 1) & 1] = 0;  // slot of the next launch
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int total = Q.ntask * B;
  for (;;) {
    const int t = next_ticket(&Q.ctr[epoch & 1], &tk);
    if (t >= total) break;
    const int task = t / B, b = t % B;
    int* done = Q.done + (int64_t)b * ns;
    const double* Kb = Kval + b * nnzk;
    if (Q.task_big[task]) {
      const int s = Q.task_sn[task * SMALL_WARPS];
      if (threadIdx.x == 0)
        for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) wait_epoch(done + S.ch_list[ci], epoch);
      __syncthreads();
      factor_big(S, s, b, smem, &piv_s, L, Lsize, Ub, Usize, Kb, notpd, minpiv);
      fence_acq_rel();
      __syncthreads();
      if (threadIdx.x == 0) st_release(done + s, epoch);
    } else {
      const int s = Q.task_sn[task * SMALL_WARPS + warp];
      if (s >= 0) {
        if (lane == 0)
          for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) wait_epoch(done + S.ch_list[ci], epoch);
        __syncwarp();
        factor_small(S, s, b, lane, smem + warp * SMALL_PANEL, L, Lsize, Ub, Usize, Kb, notpd, minpiv);
        fence_acq_rel();
        __syncwarp();
        if (lane == 0) st_release(done + s, epoch);
      }
    }
  }
}

// ============================================================================================
// triangular solves: one warp per supernode, each warp takes its own tickets from the supernode
// queue (level order forward, reverse level order backward).  Panel loads are issued in batches of
// up to 32 independent loads per lane (4 columns x 8 row blocks) so each warp keeps ~8 KB in flight.
// ============================================================================================
constexpr int SOLVE_WARPS = 8;

// out[i] = init[i] + sgn * sum_{k<ncols} A[i + k*ld] * xv[k],  i < nrows   (lanes over rows)
// RB row blocks of 32 per pass and CB = 32/RB columns per batch: 32 independent loads per lane in flight.
template <int RB>
__device__ __forceinline__ void warp_gemv_rb(const double* __restrict__ A, int ld, int r0, int nrows, int ncols,
                                             const double* xv, const double* init, double sgn, double* out,
                                             int lane) {
  constexpr int CB = 32 / RB;
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int i = r0 + r * 32 + lane;
    acc[r] = (init && i < nrows) ? init[i] : 0.0;
  }
  for (int k0 = 0; k0 < ncols; k0 += CB) {
    double a[CB][RB];
#pragma unroll
    for (int kk = 0; kk < CB; ++kk)
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int i = r0 + r * 32 + lane, k = k0 + kk;
        a[kk][r] = (k < ncols && i < nrows) ? A[i + (int64_t)k * ld] : 0.0;
      }
#pragma unroll
    for (int kk = 0; kk < CB; ++kk) {
      const double xk = (k0 + kk < ncols) ? sgn * xv[k0 + kk] : 0.0;
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] += a[kk][r] * xk;
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int i = r0 + r * 32 + lane;
    if (i < nrows) out[i] = acc[r];
  }
}

__device__ __forceinline__ void warp_gemv(const double* __restrict__ A, int ld, int nrows, int ncols,
                                          const double* xv, const double* init, double sgn, double* out, int lane) {
  int r0 = 0;
  for (; nrows - r0 > 96; r0 += 128) warp_gemv_rb<4>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
  const int rem = nrows - r0;
  if (rem > 64) warp_gemv_rb<4>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
  else if (rem > 32) warp_gemv_rb<2>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
  else if (rem > 0) warp_gemv_rb<1>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
}

// out[c] = init[c] + sgn * sum_{i<nrows} A[i + c*ld] * xv[i],  c < ncols   (column dot products;
// lanes over rows, RB row blocks x CB columns of loads per batch, partials reduced through shared
// memory -- no warp shuffles)
template <int RB>
__device__ __forceinline__ void warp_coldot_rb(const double* __restrict__ A, int ld, int nrows, int ncols,
                                               const double* xv, const double* init, double sgn, double* out,
                                               int lane, double* red) {
  constexpr int CB = 32 / RB;  // columns per batch (<= 32: red holds 32 x 33 doubles)
  for (int c0 = 0; c0 < ncols; c0 += CB) {
    double acc[CB];
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) acc[cc] = 0.0;
    for (int i0 = 0; i0 < nrows; i0 += 32 * RB) {
      double a[RB][CB], xr[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int i = i0 + r * 32 + lane;
        xr[r] = (i < nrows) ? xv[i] : 0.0;
#pragma unroll
        for (int cc = 0; cc < CB; ++cc)
          a[r][cc] = (i < nrows && c0 + cc < ncols) ? A[i + (int64_t)(c0 + cc) * ld] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) acc[cc] += a[r][cc] * xr[r];
    }
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) red[cc * 33 + lane] = acc[cc];
    __syncwarp();
    if (lane < CB && c0 + lane < ncols) {
      double v = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) v += red[lane * 33 + l];
      out[c0 + lane] = (init ? init[c0 + lane] : 0.0) + sgn * v;
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void warp_coldot(const double* __restrict__ A, int ld, int nrows, int ncols,
                                            const double* xv, const double* init, double sgn, double* out,
                                            int lane, double* red /* [32 * 33] shared */) {
  if (nrows > 64) warp_coldot_rb<4>(A, ld, nrows, ncols, xv, init, sgn, out, lane, red);
  else if (nrows > 32) warp_coldot_rb<2>(A, ld, nrows, ncols, xv, init, sgn, out, lane, red);
  else warp_coldot_rb<1>(A, ld, nrows, ncols, xv, init, sgn, out, lane, red);
}

__device__ __forceinline__ int warp_ticket(int* ctr_slot, int lane, volatile int* sh) {
  __syncwarp();
  if (lane == 0) *sh = atomicAdd(ctr_slot, 1);
  __syncwarp();
  return *sh;
}

// forward solve L y = x (in place, internal order):
//   v = [x_s; 0] + sum_c ext(u_c);  y = Z v[0:w];  u_s = v[w:m] - L21 y
__global__ void __launch_bounds__(32 * SOLVE_WARPS)
    k_fwd_persist(SymDev S, const int32_t* __restrict__ queue, const int32_t* __restrict__ chunk_ptr, int nchunk,
                  int ns, int* ctr, int* done_all, int B, int epoch, const double* __restrict__ L, int64_t Lsize,
                  double* X, int n, double* Vb, int64_t Vsize, int max_m, const int* __restrict__ skip,
                  const int8_t* __restrict__ tiny) {
  extern __shared__ double smem[];
  __shared__ int tk_sh[SOLVE_WARPS];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr[(epoch + 1) & 1] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* v = smem + (size_t)warp * (max_m + 64 + 32 * 33);
  double* y = v + max_m;
  const int total = nchunk * B;
  for (;;) {
    // dynamic tickets over chunks of consecutive supernodes of the topological queue (chunks are
    // long at the wide bottom levels and single supernodes near the top)
    const int t = warp_ticket(&ctr[epoch & 1], lane, &tk_sh[warp]);
    if (t >= total) break;
    const int ch = t / B, b = t % B;
    int* done = done_all + (int64_t)b * ns;
    const bool sk = skip && skip[b];
    for (int q = chunk_ptr[ch]; q < chunk_ptr[ch + 1]; ++q) {
      const int s = queue[q];
      if (!sk) {
        if (lane == 0)
          for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci)
            if (!tiny[S.ch_list[ci]]) wait_epoch(done + S.ch_list[ci], epoch);  // tiny ones: previous kernel
        __syncwarp();
        double* x = X + (int64_t)b * n;
        const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
        const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
        const int mu = m - w;
        const double* P = L + b * Lsize + S.pofs[s];
        for (int i = lane; i < m; i += 32) v[i] = (i < w) ? x[f + i] : 0.0;
        __syncwarp();
        for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
          const int c = S.ch_list[ci];
          const int mc = off_rows(S, c);
          const double* uc = Vb + b * Vsize + S.vofs[c];
          const int32_t* rel = S.relmap + S.relofs[c];
          for (int i = lane; i < mc; i += 32) v[rel[i]] += __ldcg(uc + i);
          __syncwarp();
        }
        warp_gemv(P, m, w, w, v, nullptr, 1.0, y, lane);  // y = Z v[0:w]  (Z strict upper part is zero)
        __syncwarp();
        for (int i = lane; i < w; i += 32) x[f + i] = y[i];
        warp_gemv(P + w, m, mu, w, y, v + w, -1.0, Vb + b * Vsize + S.vofs[s], lane);
        fence_acq_rel();
        __syncwarp();
      }
      if (lane == 0) st_release(done + s, epoch);
    }
  }
}

// backward solve L^T x = y: x_s = Z^T (y_s - L21^T x_R); the rows below belong to ancestors
__global__ void __launch_bounds__(32 * SOLVE_WARPS)
    k_bwd_persist(SymDev S, const int32_t* __restrict__ queue, const int32_t* __restrict__ chunk_ptr, int nchunk,
                  int ns, int* ctr, int* done_all, int B, int epoch, const double* __restrict__ L, int64_t Lsize,
                  double* X, int n, int max_m, const int* __restrict__ skip) {
  extern __shared__ double smem[];
  __shared__ int tk_sh[SOLVE_WARPS];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr[(epoch + 1) & 1] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* xr = smem + (size_t)warp * (max_m + 64 + 32 * 33);
  double* tv = xr + max_m;
  double* red = tv + 64;
  const int total = nchunk * B;
  for (;;) {
    const int t = warp_ticket(&ctr[epoch & 1], lane, &tk_sh[warp]);
    if (t >= total) break;
    const int ch = nchunk - 1 - t / B, b = t % B;  // chunks in reverse topological order
    int* done = done_all + (int64_t)b * ns;
    const bool sk = skip && skip[b];
    for (int q = chunk_ptr[ch + 1] - 1; q >= chunk_ptr[ch]; --q) {
      const int s = queue[q];
      if (!sk) {
        const int p = S.sparent[s];
        const unsigned long long t0 = gtimer();
        if (lane == 0 && p >= 0) wait_epoch(done + p, epoch);
        __syncwarp();
        const unsigned long long t1 = gtimer();
        double* x = X + (int64_t)b * n;
        const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
        const int64_t r0 = S.srowptr[s];
        const int m = (int)(S.srowptr[s + 1] - r0);
        const int mu = m - w;
        const double* P = L + b * Lsize + S.pofs[s];
        for (int i = lane; i < mu; i += 32) xr[i] = __ldcg(x + S.srows[r0 + w + i]);
        for (int i = lane; i < w; i += 32) tv[i] = x[f + i];
        __syncwarp();
        warp_coldot(P + w, m, mu, w, xr, tv, -1.0, tv, lane, red);  // t = y - L21^T x_R
        __syncwarp();
        warp_coldot(P, m, w, w, tv, nullptr, 1.0, xr, lane, red);   // x_s = Z^T t  (xr reused as output)
        __syncwarp();
        for (int i = lane; i < w; i += 32) x[f + i] = xr[i];
        fence_acq_rel();
        __syncwarp();
        if (g_debug_ts && lane == 0 && b == 0) {
          g_debug_ts[4 * s] = t0;
          g_debug_ts[4 * s + 1] = t1;
          g_debug_ts[4 * s + 2] = gtimer();
          g_debug_ts[4 * s + 3] = (unsigned long long)(blockIdx.x * SOLVE_WARPS + warp);
        }
      }
      if (lane == 0) st_release(done + s, epoch);
    }
  }
}

// ============================================================================================
// tiny supernodes (m <= TINY_M, w <= TINY_W, whole subtree tiny): one THREAD per tiny subtree,
// nodes in postorder (forward) / reverse postorder (backward).  Forward runs before the warp
// kernel, backward after it, so no flags are needed: every dependency outside the subtree was
// completed by the other launch, every dependency inside it by the same thread.
// ============================================================================================
constexpr int TINY_M = 32, TINY_W = 4;

__global__ void __launch_bounds__(256)
    k_fwd_tiny(SymDev S, const int32_t* __restrict__ sub_ptr, const int32_t* __restrict__ sub_nodes, int nsub, int B,
               const double* __restrict__ L, int64_t Lsize, double* X, int n, double* Vb, int64_t Vsize,
               const int* __restrict__ skip) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nsub * B) return;
  const int sub = t / B, b = t % B;
  if (skip && skip[b]) return;
  double* x = X + (int64_t)b * n;
  double* Vbb = Vb + b * Vsize;
  for (int q = sub_ptr[sub]; q < sub_ptr[sub + 1]; ++q) {
    const int s = sub_nodes[q];
    const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
    const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
    const double* P = L + b * Lsize + S.pofs[s];
    double v[TINY_M], y[TINY_W];
#pragma unroll
    for (int i = 0; i < TINY_M; ++i) v[i] = 0.0;
    for (int i = 0; i < w; ++i) v[i] = x[f + i];
    for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
      const int c = S.ch_list[ci];
      const int mc = off_rows(S, c);
      const double* uc = Vbb + S.vofs[c];
      const int32_t* rel = S.relmap + S.relofs[c];
      for (int i = 0; i < mc; ++i) v[rel[i]] += uc[i];
    }
#pragma unroll
    for (int k = 0; k < TINY_W; ++k) {
      double acc = 0.0;
      if (k < w)
        for (int j = 0; j <= k; ++j) acc += P[k + j * m] * v[j];
      y[k] = acc;
    }
    for (int k = 0; k < w; ++k) x[f + k] = y[k];
    double* us = Vbb + S.vofs[s];
    for (int i = w; i < m; ++i) {
      double acc = v[i];
#pragma unroll
      for (int k = 0; k < TINY_W; ++k)
        if (k < w) acc -= P[i + k * m] * y[k];
      us[i - w] = acc;
    }
  }
}

__global__ void __launch_bounds__(256)
    k_bwd_tiny(SymDev S, const int32_t* __restrict__ sub_ptr, const int32_t* __restrict__ sub_nodes, int nsub, int B,
               const double* __restrict__ L, int64_t Lsize, double* X, int n, const int* __restrict__ skip) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nsub * B) return;
  const int sub = t / B, b = t % B;
  if (skip && skip[b]) return;
  double* x = X + (int64_t)b * n;
  for (int q = sub_ptr[sub + 1] - 1; q >= sub_ptr[sub]; --q) {
    const int s = sub_nodes[q];
    const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
    const int64_t r0 = S.srowptr[s];
    const int m = (int)(S.srowptr[s + 1] - r0);
    const double* P = L + b * Lsize + S.pofs[s];
    double tv[TINY_W];
#pragma unroll
    for (int c = 0; c < TINY_W; ++c) tv[c] = (c < w) ? x[f + c] : 0.0;
    for (int i = w; i < m; ++i) {
      const double xi = x[S.srows[r0 + i]];
#pragma unroll
      for (int c = 0; c < TINY_W; ++c)
        if (c < w) tv[c] -= P[i + c * m] * xi;
    }
#pragma unroll
    for (int i = 0; i < TINY_W; ++i) {
      if (i < w) {
        double acc = 0.0;
        for (int k = i; k < w; ++k) acc += P[k + i * m] * tv[k];
        x[f + i] = acc;
      }
    }
  }
}
