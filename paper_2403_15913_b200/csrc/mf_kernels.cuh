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

#include "dense_front.cuh"

// doubles of a small (one-warp) front's panel: chosen per analysis at setup (Sched::small_panel);
// large trees profit from more one-warp fronts (8 in flight per CTA), small ones from CTA fronts
constexpr int SMALL_PANEL_MIN = 512, SMALL_PANEL_MAX = 1536;
constexpr int SMALL_WARPS = 8;     // warps per CTA; small supernodes per task
constexpr int MF_THREADS = 32 * SMALL_WARPS;

// packed per-supernode metadata (one 48-byte uniform load instead of several dependent loads)
struct __align__(16) SnMeta {
  int f, w, m, ch0;
  int ch1, relw, pad0, pad1;
  long long pofs, vofs, relofs, r0;
};
// packed per-child record, in the order of ch_list
struct __align__(16) ChMeta {
  int c, mc, tiny, pad;
  long long vofs, relofs;
};

struct SymDev {
  const SnMeta* meta;
  const ChMeta* chmeta;
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
  const int32_t* relw;  // per child: number of its off-diagonal rows inside the parent's columns
};

struct Sched {
  int ntask;                      // tasks per instance
  const int32_t* task_sn;         // fronts of task t: task_sn[task_ptr[t] .. task_ptr[t+1])
  const int32_t* task_big;        // [ntask]: 1 = one front for the whole CTA, 0 = a chunk of one-warp fronts
  const int32_t* task_ptr;        // [ntask + 1]
  int* done;                      // [B * ns] epoch flags
  int* ctr;                       // [2] ticket counters (alternating per epoch)
  int small_panel;                // doubles per warp of a small front's shared-memory panel
};

// -DCKKT_BOUNDS (tools/build_variant.sh bounds "-DCKKT_BOUNDS"): every panel / update-matrix /
// update-vector / solution access region of every supernode, and every extend-add target, is checked
// against its array before use; a violation prints and traps.  The checked build is what stands in for
// compute-sanitizer (closed on this GPU pool); release builds compile the checks away.
#ifdef CKKT_BOUNDS
#define CKB(cond)                                                                              \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("ckkt bounds: %s failed (%s:%d, block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                 \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define CKB(cond) \
  do {            \
  } while (0)
#endif

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
#ifdef CKKT_DEBUG_NO_RELEASE  // timing experiments only: drops the release ordering (results may be wrong)
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}
// debug switches live in constant memory: reading them costs no global round trip (a __device__
// variable would be re-fetched from L2 after every fence, on the critical path of each step)
__constant__ int g_debug_nowait = 0;  // debug only: skip dependency waits (timing experiments)
__constant__ unsigned long long* g_debug_ts = nullptr;  // debug only: [ns][4] ticket/wake/end times of sweeps
__constant__ unsigned long long* g_debug_ph = nullptr;  // debug only: [ns][8] phase times inside factor_big

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

#ifndef CKKT_POLL_MAX_NS
#define CKKT_POLL_MAX_NS 64
#endif
// Poll a producer's done flag until it holds `epoch`.  The poll is an ld.acquire.gpu (SASS:
// LDG.STRONG.GPU + CCTL.IVALL, no MEMBAR): the load that observes the producer's st.release
// synchronizes-with it (PTX memory model), so every later read of the producer's data — children's
// update matrices / vectors, ancestors' solution entries, also read with ld.global.cg from L2 — sees
// the producer's writes.  The successful poll is the acquire itself: no extra round trip on the
// critical path.  -DCKKT_RELAXED_POLL (timing experiments only) polls with ld.relaxed and relies on
// the control dependency, which the PTX model does not guarantee.
__device__ __forceinline__ void wait_epoch(const int* p, int epoch) {
  if (g_debug_nowait) return;
  int ns = 32;
#ifdef CKKT_RELAXED_POLL
  while (ld_relaxed(p) != epoch) {
#else
  while (ld_acquire(p) != epoch) {
#endif
    __nanosleep(ns);
    ns = ns < CKKT_POLL_MAX_NS ? 2 * ns : CKKT_POLL_MAX_NS;
  }
}

// release-side fence: makes this thread's prior writes visible at gpu scope before the flag store
// (acq_rel is much cheaper than the sequentially-consistent fence of __threadfence())
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// TMA bulk prefetch of [p, p + bytes) into L2 (fire and forget; 16-byte granularity)
__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
#ifdef CKKT_NO_PREFETCH
  return;
#endif
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  while (a < e) {
    const uint32_t sz = (uint32_t)((e - a) > (1u << 20) ? (1u << 20) : (e - a));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
    a += sz;
  }
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
// Extend-add of child c's update matrix U_c (mc x mc, lower, column-major) into the parent front:
//   part 0: columns j < relw (targets in the parent's panel, shared memory Ps with leading dim ldp)
//   part 1: columns j >= relw (targets in the parent's update block U, global, leading dim mu)
// Only the lower triangle is visited: warps take columns (4 per batch, so every lane keeps 4
// independent loads in flight), lanes take rows i >= j of those columns; rel[j] is uniform per
// column.  Targets of one child are distinct, so there are no races within a child.
template <int PART>
__device__ __forceinline__ void extend_add(const double* __restrict__ Uc, int mc, int relw,
                                           const int32_t* __restrict__ rel, int w, double* Ps, int ldp, double* U,
                                           int mu, int tid, int nt) {
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int j_lo = PART == 0 ? 0 : relw, j_hi = PART == 0 ? relw : mc;
  for (int j0 = j_lo + wid; j0 < j_hi; j0 += 4 * nw) {
    int rj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q * nw;
      rj[q] = (j < j_hi) ? __ldg(rel + j) : 0;
    }
    for (int r0 = 0; j0 + r0 < mc; r0 += 32) {  // column j0 is the longest of the batch
      double sv[4], tv[4];
      int tgt[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + q * nw, i = j + r0 + lane;
        const bool ok = j < j_hi && i < mc;
        sv[q] = ok ? __ldcg(Uc + i + (int64_t)j * mc) : 0.0;
        if (ok) {
          const int ri = __ldg(rel + i);
          CKB(ri >= rj[q] && ri < w + mu && (PART == 0 ? rj[q] < w : rj[q] >= w));
          tgt[q] = PART == 0 ? ri + rj[q] * ldp : (ri - w) + (rj[q] - w) * mu;
        } else {
          tgt[q] = -1;
        }
        if (PART == 1) tv[q] = (tgt[q] >= 0) ? U[tgt[q]] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (tgt[q] < 0) continue;
        if (PART == 0) Ps[tgt[q]] += sv[q];
        else U[tgt[q]] = tv[q] + sv[q];
      }
    }
  }
}

// U = -L21 L21^T (mu x mu, lower, column-major) from the panel in shared memory (ld ldp, L21 at row
// offset w), on 8x8 DMMA tiles (mma.sync.m8n8k4.f64); warps take tiles round robin.  Rows >= mu and
// columns >= w read as zero (guards), so the arithmetic is the same for padded and unpadded panels.
__device__ __forceinline__ void upd_tile_ij(int tI, int& I, int& J) {
  I = (int)((sqrt(8.0 * tI + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= tI) ++I;
  while (I * (I + 1) / 2 > tI) --I;
  J = tI - I * (I + 1) / 2;
}

#ifndef CKKT_UPD_TU
#define CKKT_UPD_TU 1
#endif
#ifndef CKKT_UPD_UNROLL
#define CKKT_UPD_UNROLL 2
#endif
constexpr int UPD_UNROLL = CKKT_UPD_UNROLL;
// A warp computes CKKT_UPD_TU tiles at a time (tiles tI, tI + nwarp, ...; independent DMMA chains in
// one k loop) with the k loop unrolled CKKT_UPD_UNROLL times, so the next fragments load while the
// current DMMA runs.  Each tile's k order is fixed (results do not depend on either knob).  Measured
// at C3 (factor): TU 1 / unroll 2 12.47 ms, TU 2 12.65, TU 4 12.79 (spills), unroll 4 12.69,
// unroll 8 13.26, no unroll 12.81.
__device__ __forceinline__ void front_update_dmma(const double* Ps, int ldp, int w, int mu, int lane, int warp,
                                                  int nwarp, double* U) {
  constexpr int TU = CKKT_UPD_TU;
  const int nb = (mu + 7) >> 3;
  const int ntile = nb * (nb + 1) / 2;
  const int g = lane >> 2, t4 = lane & 3;
  for (int t0 = warp; t0 < ntile; t0 += TU * nwarp) {
    int ia[TU], ib[TU];
    double c0[TU], c1[TU];
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int tI = t0 + u * nwarp;
      int I = 0, J = 0;
      if (tI < ntile) upd_tile_ij(tI, I, J);
      ia[u] = (tI < ntile) ? I * 8 + g : mu;  // rows >= mu read as zero
      ib[u] = (tI < ntile) ? J * 8 + g : mu;
      c0[u] = c1[u] = 0.0;
    }
#pragma unroll UPD_UNROLL
    for (int k = 0; k < w; k += 4) {
      const int kk = k + t4;
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const double a = (ia[u] < mu && kk < w) ? Ps[w + ia[u] + kk * ldp] : 0.0;
        const double b = (ib[u] < mu && kk < w) ? Ps[w + ib[u] + kk * ldp] : 0.0;
        dmma_8x8x4(c0[u], c1[u], a, b);
      }
    }
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int tI = t0 + u * nwarp;
      if (tI >= ntile) continue;
      const int row = ia[u], col = ib[u] - g + 2 * t4;
      if (row < mu) {
        if (col < mu) U[row + (int64_t)col * mu] = -c0[u];
        if (col + 1 < mu) U[row + (int64_t)(col + 1) * mu] = -c1[u];
      }
    }
  }
}

// small supernode, one warp, panel in shared memory (ld = m)
__device__ void factor_small(const SymDev& S, int s, int b, int tid, double* Ps, double* dsh, double* L, int64_t Lsize,
                             double* Ub, int64_t Usize, const double* __restrict__ Kb, int* notpd, int* minpiv) {
  const int nt = 32;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w, ldp = m;
  double* P = L + b * Lsize + S.pofs[s];
  double* U = Ub + b * Usize + S.uofs[s];
  CKB(S.pofs[s] + (int64_t)m * w <= Lsize && S.uofs[s] + (int64_t)mu * mu <= Usize && m * w <= SMALL_PANEL_MAX);
  for (int i = tid; i < m * w; i += nt) Ps[i] = 0.0;
  __syncwarp();
  for (int64_t k = S.kp[f] + tid; k < S.kp[f + w]; k += nt) {
    CKB(S.kmap[k] >= 0 && S.kmap[k] < m * w);
    Ps[S.kmap[k]] = Kb[k];
  }
  __syncwarp();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    CKB(S.uofs[c] + (int64_t)off_rows(S, c) * off_rows(S, c) <= Usize);
    extend_add<0>(Ub + b * Usize + S.uofs[c], off_rows(S, c), S.relw[c], S.relmap + S.relofs[c], w, Ps, ldp, U,
                  mu, tid, nt);
    __syncwarp();
  }
  dfront::dense_blocked<false>(Ps, ldp, w, m, tid, nt, dsh, notpd + b, minpiv + b, f);  // [Z; L21]
  for (int i = tid; i < m * w; i += nt) P[i] = Ps[i];
  // U_s = -L21 L21^T on 8x8 DMMA tiles of the lower triangle: the same tiles, k order and zero
  // padding (guards instead of zero-filled pads) as factor_big, so a front's update matrix is
  // bit-identical whichever path factors it (results independent of the batch size)
  front_update_dmma(Ps, ldp, w, mu, tid & 31, 0, 1, U);
  __syncwarp();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    extend_add<1>(Ub + b * Usize + S.uofs[c], off_rows(S, c), S.relw[c], S.relmap + S.relofs[c], w, Ps, ldp, U,
                  mu, tid, nt);
    __syncwarp();
  }
}

// Leading dimension of a CTA front's shared-memory panel: m rounded up to 8 doubles and then to
// 8 mod 16, so that the DMMA fragment loads (lanes g + 8 t4 ... rows g, columns t4) fall into 16
// distinct double-banks twice each — two wavefronts per 32-lane load, the minimum; a multiple of
// 16 would put all four column groups on the same 8 banks (four wavefronts).
__host__ __device__ constexpr int big_ldp(int m) {
#ifdef CKKT_NO_LDP_PAD
  return (m + 7) & ~7;
#else
  return (((m + 7) & ~7) & 15) ? ((m + 7) & ~7) : ((m + 7) & ~7) + 8;
#endif
}

// big supernode, whole CTA, panel in shared memory with ld = mp = big_ldp(m) (m padded to 8, w padded to 4)
__device__ void factor_big(const SymDev& S, int s, int b, double* Ps, double* dsh, double* L, int64_t Lsize,
                           double* Ub, int64_t Usize, const double* __restrict__ Kb, int* notpd, int* minpiv) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int f = S.sfirst[s], w = S.sfirst[s + 1] - f;
  const int m = (int)(S.srowptr[s + 1] - S.srowptr[s]);
  const int mu = m - w;
  const int mp = big_ldp(m), wp = (w + 3) & ~3, ldp = mp;
  double* P = L + b * Lsize + S.pofs[s];
  double* U = Ub + b * Usize + S.uofs[s];
  CKB(S.pofs[s] + (int64_t)m * w <= Lsize && S.uofs[s] + (int64_t)mu * mu <= Usize && w <= 64);
  unsigned long long* ph = (g_debug_ph && b == 0 && tid == 0) ? g_debug_ph + 8 * (int64_t)s : nullptr;
  if (ph) ph[0] = gtimer();
  for (int i = tid; i < mp * wp + 8; i += nt) Ps[i] = 0.0;
  __syncthreads();
  for (int64_t k = S.kp[f] + tid; k < S.kp[f + w]; k += nt) {
    const int q = S.kmap[k];
    CKB(q >= 0 && q < m * w);
    Ps[(q % m) + (q / m) * mp] = Kb[k];
  }
  __syncthreads();
  if (ph) ph[1] = gtimer();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    CKB(S.uofs[c] + (int64_t)off_rows(S, c) * off_rows(S, c) <= Usize);
    extend_add<0>(Ub + b * Usize + S.uofs[c], off_rows(S, c), S.relw[c], S.relmap + S.relofs[c], w, Ps, ldp, U,
                  mu, tid, nt);
    __syncthreads();
  }
  if (ph) ph[2] = gtimer();
  dfront::dense_blocked<true>(Ps, ldp, w, m, tid, nt, dsh, notpd + b, minpiv + b, f);  // [Z; L21]
  if (ph) ph[3] = gtimer();
  front_update_dmma(Ps, ldp, w, mu, lane, warp, nwarp, U);  // U_s = -L21 L21^T
  if (ph) ph[4] = gtimer();
  for (int e = tid; e < m * w; e += nt) P[e] = Ps[(e % m) + (e / m) * mp];
  __syncthreads();  // this CTA's U_s tile writes are complete before the children add into it
  if (ph) ph[5] = gtimer();
  for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci) {
    const int c = S.ch_list[ci];
    extend_add<1>(Ub + b * Usize + S.uofs[c], off_rows(S, c), S.relw[c], S.relmap + S.relofs[c], w, Ps, ldp, U,
                  mu, tid, nt);
    __syncthreads();
  }
  if (ph) ph[6] = gtimer();
}

#ifdef CKKT_MF_MINB  // (experiments: force more resident CTAs per SM)
#define CKKT_MF_BOUNDS __launch_bounds__(MF_THREADS, CKKT_MF_MINB)
#else
#define CKKT_MF_BOUNDS __launch_bounds__(MF_THREADS)
#endif
__global__ void CKKT_MF_BOUNDS
    k_factor_persist(SymDev S, Sched Q, int ns, int B, int epoch, double* L, int64_t Lsize, double* Ub,
                     int64_t Usize, const double* __restrict__ Kval, int64_t nnzk, int* notpd, int* minpiv,
                     const int8_t* __restrict__ tiny) {
  extern __shared__ double smem[];  // max(big panel, SMALL_WARPS small panels)
  __shared__ double dsh_all[SMALL_WARPS][64];  // reciprocal pivots (per warp; the CTA path uses row 0)
  __shared__ int tk;
  __shared__ int chunk_ctr;
  if (threadIdx.x == 0) chunk_ctr = 0;
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
      const int s = Q.task_sn[Q.task_ptr[task]];
      const unsigned long long t0 = gtimer();
      if (threadIdx.x == 0)
        for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci)
          if (!tiny[S.ch_list[ci]]) wait_epoch(done + S.ch_list[ci], epoch);
      __syncthreads();
      const unsigned long long t1 = gtimer();
      factor_big(S, s, b, smem, dsh_all[0], L, Lsize, Ub, Usize, Kb, notpd, minpiv);
      fence_acq_rel();
      __syncthreads();
      if (g_debug_ts && threadIdx.x == 0 && b == 0) {
        g_debug_ts[4 * s] = t0;
        g_debug_ts[4 * s + 1] = t1;
        g_debug_ts[4 * s + 2] = gtimer();
        g_debug_ts[4 * s + 3] = 1000000 + blockIdx.x;
      }
      if (threadIdx.x == 0) st_release(done + s, epoch);
    } else {
      // a chunk of one-warp fronts of one level (no dependencies inside it): the warps pull fronts from
      // a shared counter, so a warp that finishes early takes the next front instead of idling until the
      // slowest warp of a fixed bundle is done (the arithmetic of a front does not depend on the warp)
      const int q0 = Q.task_ptr[task], q1 = Q.task_ptr[task + 1];
      for (;;) {
        int q = 0;
        if (lane == 0) q = q0 + atomicAdd(&chunk_ctr, 1);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= q1) break;
        const int s = Q.task_sn[q];
        const unsigned long long t0 = gtimer();
        if (lane == 0)
          for (int ci = S.ch_ptr[s]; ci < S.ch_ptr[s + 1]; ++ci)
            if (!tiny[S.ch_list[ci]]) wait_epoch(done + S.ch_list[ci], epoch);
        __syncwarp();
        const unsigned long long t1 = gtimer();
        factor_small(S, s, b, lane, smem + warp * Q.small_panel, dsh_all[warp], L, Lsize, Ub, Usize, Kb, notpd, minpiv);
        fence_acq_rel();
        __syncwarp();
        if (g_debug_ts && lane == 0 && b == 0) {
          g_debug_ts[4 * s] = t0;
          g_debug_ts[4 * s + 1] = t1;
          g_debug_ts[4 * s + 2] = gtimer();
          g_debug_ts[4 * s + 3] = blockIdx.x * 8 + warp;
        }
        if (lane == 0) st_release(done + s, epoch);
      }
      __syncthreads();
      if (threadIdx.x == 0) chunk_ctr = 0;  // (next_ticket's barrier orders this before the next chunk)
    }
  }
}

// ============================================================================================
// triangular solves: one warp per supernode, each warp takes its own tickets from the supernode
// queue (level order forward, reverse level order backward).  Panel loads are issued in batches of
// up to 32 independent loads per lane (4 columns x 8 row blocks) so each warp keeps ~8 KB in flight.
// ============================================================================================
constexpr int SOLVE_WARPS = 8;
#ifndef CKKT_SOLVE_MINB
#define CKKT_SOLVE_MINB 3
#endif
constexpr int SOLVE_MINB = CKKT_SOLVE_MINB;  // resident CTAs per SM the register budget is sized for
constexpr int TOP_PANEL = 5120;  // panels above this (doubles) and their ancestors go to the top set
// Bottom-set sweeps run one supernode per WORKER of LW lanes (a warp, or a half warp: two
// independent supernode chains interleaved in one warp hide more memory latency per SM).
#ifndef CKKT_LW
#define CKKT_LW 32
#endif
constexpr int LW = CKKT_LW;
constexpr int SOLVE_WORKERS = 32 * SOLVE_WARPS / LW;  // workers per CTA
constexpr int RED_LD = LW + 1;                         // column stride of the per-worker reduction scratch
constexpr int RED_SZ = 16 * RED_LD + 32;               // doubles of it (16 columns per batch + stage 2)
static_assert(LW == 32 || LW == 16, "worker width");

__device__ __forceinline__ unsigned worker_mask() {
  return LW == 32 ? 0xFFFFFFFFu : (0xFFFFu << (threadIdx.x & 16));
}
__device__ __forceinline__ void wsync() { __syncwarp(worker_mask()); }

// out[i] = init[i] + sgn * sum_{k<ncols} A[i + k*ld] * xv[k],  i < nrows   (lanes over rows)
// RB row blocks of LW per pass and CB = 16/RB columns per batch: 16 independent loads per lane in flight.
template <int RB>
__device__ __forceinline__ void warp_gemv_rb(const double* __restrict__ A, int ld, int r0, int nrows, int ncols,
                                             const double* xv, const double* init, double sgn, double* out,
                                             int lane) {
  constexpr int CB = 16 / RB;
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int i = r0 + r * LW + lane;
    acc[r] = (init && i < nrows) ? init[i] : 0.0;
  }
  for (int k0 = 0; k0 < ncols; k0 += CB) {
    double a[CB][RB];
#pragma unroll
    for (int kk = 0; kk < CB; ++kk)
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int i = r0 + r * LW + lane, k = k0 + kk;
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
    const int i = r0 + r * LW + lane;
    if (i < nrows) out[i] = acc[r];
  }
}

__device__ __forceinline__ void warp_gemv(const double* __restrict__ A, int ld, int nrows, int ncols,
                                          const double* xv, const double* init, double sgn, double* out, int lane) {
  int r0 = 0;
  for (; nrows - r0 > 3 * LW; r0 += 4 * LW) warp_gemv_rb<4>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
  const int rem = nrows - r0;
  if (rem > 2 * LW) warp_gemv_rb<4>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
  else if (rem > LW) warp_gemv_rb<2>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
  else if (rem > 0) warp_gemv_rb<1>(A, ld, r0, nrows, ncols, xv, init, sgn, out, lane);
}

// out[c] = init[c] + sgn * sum_{i<nrows} A[i + c*ld] * xv[i],  c < ncols   (column dot products;
// lanes over rows, RB row blocks x CB columns of loads per batch; the CB per-lane partials are
// reduced by a transpose through shared memory: warp shuffles compile to the slow warp-collective
// sequence inside this persistent loop, whose convergence the compiler cannot prove)
template <int RB>
__device__ __forceinline__ void warp_coldot_rb(const double* __restrict__ A, int ld, int nrows, int ncols,
                                               const double* xv, const double* init, double sgn, double* out,
                                               int lane, double* red) {
  constexpr int CB = 16 / RB;
  for (int c0 = 0; c0 < ncols; c0 += CB) {
    double acc[CB];
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) acc[cc] = 0.0;
    for (int i0 = 0; i0 < nrows; i0 += LW * RB) {
      double a[RB][CB], xr[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int i = i0 + r * LW + lane;
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
    for (int cc = 0; cc < CB; ++cc) red[cc * RED_LD + lane] = acc[cc];
    wsync();
#ifndef CKKT_COLDOT_SERIAL
    {  // two stages with every lane busy: lane (j, h) sums segment h (CB partials) of column j, then
       // lane j < CB adds its column's H segment sums (CB + H dependent adds instead of LW)
      constexpr int H = LW / CB;
      const int j = lane % CB, h = lane / CB;
      const double* q = red + j * RED_LD + h * CB;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k = 0; k < CB; k += 2) {
        s0 += q[k];
        s1 += q[k + 1];
      }
      red[16 * RED_LD + j * H + h] = s0 + s1;
    }
    wsync();
    if (lane < CB && c0 + lane < ncols) {
      constexpr int H = LW / CB;
      double v = 0.0;
#pragma unroll
      for (int h = 0; h < H; ++h) v += red[16 * RED_LD + lane * H + h];
      out[c0 + lane] = (init ? init[c0 + lane] : 0.0) + sgn * v;
    }
#else
    if (lane < CB && c0 + lane < ncols) {
      double v = 0.0;
#pragma unroll 8
      for (int l = 0; l < LW; ++l) v += red[lane * RED_LD + l];
      out[c0 + lane] = (init ? init[c0 + lane] : 0.0) + sgn * v;
    }
#endif
    wsync();
  }
}

__device__ __forceinline__ void warp_coldot(const double* __restrict__ A, int ld, int nrows, int ncols,
                                            const double* xv, const double* init, double sgn, double* out,
                                            int lane, double* red /* [RED_SZ] shared */) {
  if (nrows > 2 * LW) warp_coldot_rb<4>(A, ld, nrows, ncols, xv, init, sgn, out, lane, red);
  else if (nrows > LW) warp_coldot_rb<2>(A, ld, nrows, ncols, xv, init, sgn, out, lane, red);
  else warp_coldot_rb<1>(A, ld, nrows, ncols, xv, init, sgn, out, lane, red);
}

__device__ __forceinline__ int warp_ticket(int* ctr_slot, int lane, volatile int* sh) {
  wsync();
  if (lane == 0) *sh = atomicAdd(ctr_slot, 1);
  wsync();
  return *sh;
}

// ---------------------------------------------------------------------------------------------
// Bottom-set sweeps: persistent kernels, one supernode per worker, workers take chunks of the
// level-ordered bottom queue from an atomic ticket counter.  The top set (large panels and their
// ancestors; ancestor-closed) runs in k_fwd_top / k_bwd_top: forward after this kernel, backward
// before it (bottom tasks never depend on top tasks in the forward sweep, and vice versa).
// ---------------------------------------------------------------------------------------------
struct SweepArgs {
  const int32_t* queue;      // bottom supernodes, level order
  const SnMeta* qmeta;       // their metadata in queue order (pad0 = parent, pad1 = supernode)
  const int32_t* chunk_ptr;  // chunks of the bottom queue
  int nchunk;
  const int32_t* top;        // top supernodes, level order
  const SnMeta* topmeta;     // their metadata in top order (pad0 = parent, pad1 = supernode)
  int ntop;
  int topbuf;                // doubles of the top kernels' shared-memory panel buffer
  int ns;                    // done-flag stride
  int* ctr;                  // [4]: worker tickets (2 epoch slots), top-kernel tickets (2 epoch slots)
  int* done_all;
  int B, epoch;              // epoch is re-read from *epoch_ptr at kernel start (device-side counter)
  const int* epoch_ptr;
  const double* L;
  int64_t Lsize;
  double* X;
  int n;
  double* Vb;
  int64_t Vsize;
  int max_m;
  const int* skip;
};

// v[rel_c] += u_c for the children c of M (extend-add of the update vectors), children in
// a fixed order (deterministic; rows inside one child are distinct so lanes never collide)
__device__ __forceinline__ void warp_gather_children(const SymDev& S, const SweepArgs& A, const SnMeta& M, int b,
                                                     int lane, double* v, ChMeta* cmeta, int* done) {
  const double* Vb = A.Vb + b * A.Vsize;
  for (int cb = M.ch0; cb < M.ch1; cb += LW) {
    const int nc = min(LW, M.ch1 - cb);
    if (lane < nc) {
      const ChMeta cm = S.chmeta[cb + lane];
      cmeta[lane] = cm;
      if (!cm.tiny) wait_epoch(done + cm.c, A.epoch);
    }
    wsync();
#ifndef CKKT_GATHER_SERIAL
    // the first 2 LW rows of GK children at a time: all their loads in flight together (one round
    // trip instead of one per child), then applied child by child in order (deterministic); rows
    // beyond 2 LW (rare) follow for each child right after its first rows
#ifndef CKKT_GK
#define CKKT_GK 4
#endif
    constexpr int GK = CKKT_GK;
    for (int k0 = 0; k0 < nc; k0 += GK) {
      double uv[GK][2];
      int rl[GK][2];
#pragma unroll
      for (int kk = 0; kk < GK; ++kk) {
        const int k = k0 + kk;
        const int mc = (k < nc) ? cmeta[k].mc : 0;
        const double* uc = Vb + ((k < nc) ? cmeta[k].vofs : 0);
        const int32_t* rel = S.relmap + ((k < nc) ? cmeta[k].relofs : 0);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = lane + r * LW;
          rl[kk][r] = (i < mc) ? __ldg(rel + i) : -1;
          uv[kk][r] = (i < mc) ? __ldcg(uc + i) : 0.0;
        }
      }
#pragma unroll
      for (int kk = 0; kk < GK; ++kk) {
        const int k = k0 + kk;
        if (k >= nc) break;
#pragma unroll
        for (int r = 0; r < 2; ++r)
          if (rl[kk][r] >= 0) {
            CKB(rl[kk][r] < M.m && cmeta[k].vofs + cmeta[k].mc <= A.Vsize);
            v[rl[kk][r]] += uv[kk][r];
          }
        const ChMeta& cm = cmeta[k];
        for (int i = 2 * LW + lane; i < cm.mc; i += LW) v[__ldg(S.relmap + cm.relofs + i)] += __ldcg(Vb + cm.vofs + i);
        wsync();
      }
    }
#else
    for (int k = 0; k < nc; ++k) {
      const ChMeta cm = cmeta[k];
      const double* uc = Vb + cm.vofs;
      const int32_t* rel = S.relmap + cm.relofs;
      CKB(cm.vofs + cm.mc <= A.Vsize);
      for (int i = lane; i < cm.mc; i += LW) {
        CKB(__ldg(rel + i) >= 0 && __ldg(rel + i) < M.m);
        v[__ldg(rel + i)] += __ldcg(uc + i);
      }
      wsync();
    }
#endif
  }
}

// forward step of supernode s by one worker (v, y: per-worker shared scratch)
__device__ __forceinline__ void fwd_warp_step(const SymDev& S, const SweepArgs& A, const SnMeta& M, int s, int b,
                                              int lane, double* v, double* y, ChMeta* cmeta, int* done,
                                              int rel_prev) {
  double* x = A.X + (int64_t)b * A.n;
  const int f = M.f, w = M.w, m = M.m, mu = m - w;
  const double* P = A.L + b * A.Lsize + M.pofs;
  CKB(M.pofs + (int64_t)m * w <= A.Lsize && M.vofs + mu <= A.Vsize && f + w <= A.n && m <= A.max_m);
  if (lane == 0) prefetch_l2(P, 8ll * m * w);  // the panel streams into L2 while the children are gathered
  const unsigned long long t0 = g_debug_ts ? gtimer() : 0ull;
  // this step's x loads are issued before the previous step's flag is published (deferred release,
  // before any wait of this step): the release fence then overlaps the loads' round trip
  constexpr int XR = 64 / LW;  // w <= 64
  double xw[XR];
#pragma unroll
  for (int r = 0; r < XR; ++r) xw[r] = (lane + r * LW < w) ? x[f + lane + r * LW] : 0.0;
  if (rel_prev >= 0 && lane == 0) st_release(done + rel_prev, A.epoch);
#pragma unroll
  for (int r = 0; r < XR; ++r)
    if (lane + r * LW < m) v[lane + r * LW] = xw[r];
  for (int i = lane + 64; i < m; i += LW) v[i] = 0.0;
  warp_gather_children(S, A, M, b, lane, v, cmeta, done);
  warp_gemv(P, m, w, w, v, nullptr, 1.0, y, lane);  // y = Z v[0:w]  (Z strict upper part is zero)
  wsync();
  for (int i = lane; i < w; i += LW) x[f + i] = y[i];
  warp_gemv(P + w, m, mu, w, y, v + w, -1.0, A.Vb + b * A.Vsize + M.vofs, lane);
  if (g_debug_ts && lane == 0 && b == 0) {
    g_debug_ts[4 * s] = t0;
    g_debug_ts[4 * s + 1] = t0;
    g_debug_ts[4 * s + 2] = gtimer();
    g_debug_ts[4 * s + 3] = 0;
  }
}

// stage the metadata of queue entries [q0, q0 + n) (n <= 16) into shared memory (and, backward,
// start the L2 prefetch of their row index lists)
__device__ __forceinline__ void warp_stage_chunk(const SymDev& S, const SweepArgs& A, int q0, int n, int b, int lane,
                                                 SnMeta* msh, bool rows) {
  const long long* src = reinterpret_cast<const long long*>(A.qmeta + q0);
  long long* dst = reinterpret_cast<long long*>(msh);
  constexpr int WPM = sizeof(SnMeta) / 8;
  for (int k = lane; k < n * WPM; k += LW) dst[k] = __ldg(src + k);
  wsync();
  if (lane == 0 && n > 0) {  // the chunk's panels are one contiguous span of L (sweep-ordered storage)
    const SnMeta& a = msh[0];
    const SnMeta& z = msh[n - 1];
    prefetch_l2(A.L + b * A.Lsize + a.pofs, 8ll * (z.pofs + (int64_t)z.m * z.w - a.pofs));
  }
  if (lane < n && rows) {
    const SnMeta& M = msh[lane];
    prefetch_l2(S.srows + M.r0 + M.w, 4ll * (M.m - M.w));
  }
}

__global__ void __launch_bounds__(32 * SOLVE_WARPS, SOLVE_MINB) k_fwd_persist(SymDev S, SweepArgs A) {
  A.epoch = *A.epoch_ptr;  // bumped by the sweep's first launch (CUDA-graph safe)
  extern __shared__ double smem[];
  __shared__ int tk_sh[SOLVE_WORKERS];
  __shared__ ChMeta cmeta_all[SOLVE_WORKERS][LW];
  __shared__ SnMeta msh_all[SOLVE_WORKERS][16];
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // slots of the next launch
    A.ctr[(A.epoch + 1) & 1] = 0;
    A.ctr[2 + ((A.epoch + 1) & 1)] = 0;
  }
  const int lane = threadIdx.x % LW, wk = threadIdx.x / LW;
  double* v = smem + (size_t)wk * (A.max_m + 64);
  double* y = v + A.max_m;
  ChMeta* cmeta = cmeta_all[wk];
  SnMeta* msh = msh_all[wk];
  for (;;) {
    const int t = warp_ticket(&A.ctr[A.epoch & 1], lane, &tk_sh[wk]);
    if (t >= A.nchunk * A.B) break;
    const int ch = t / A.B, b = t % A.B;
    int* done = A.done_all + (int64_t)b * A.ns;
    const bool sk = A.skip && A.skip[b];
    const int q0 = A.chunk_ptr[ch], n = A.chunk_ptr[ch + 1] - q0;
    if (!sk) warp_stage_chunk(S, A, q0, n, b, lane, msh, false);
    int pend = -1;  // supernode whose flag is published at the start of the next step of the chunk
    for (int j = 0; j < n; ++j) {
      const int s = sk ? A.queue[q0 + j] : msh[j].pad1;
      if (!sk) {
        fwd_warp_step(S, A, msh[j], s, b, lane, v, y, cmeta, done, pend);
        wsync();
        pend = s;
      } else if (lane == 0) {
        st_release(done + s, A.epoch);
      }
    }
    if (pend >= 0 && lane == 0) st_release(done + pend, A.epoch);
    wsync();
  }
}

// backward step of supernode s by one worker: x_s = Z^T (y_s - L21^T x_R)
__device__ __forceinline__ void bwd_warp_step(const SymDev& S, const SweepArgs& A, const SnMeta& M, int s, int b,
                                              int lane, double* xr, double* tv, double* red, int* ridx, int* done,
                                              int rel_prev) {
  const int p = M.pad0;
  double* x = A.X + (int64_t)b * A.n;
  const int f = M.f, w = M.w, m = M.m, mu = m - w;
  const double* P = A.L + b * A.Lsize + M.pofs;
  CKB(M.pofs + (int64_t)m * w <= A.Lsize && f + w <= A.n && m <= A.max_m);
  if (lane == 0) prefetch_l2(P, 8ll * m * w);  // independent of the parent: overlap with the wait
  constexpr int XR = 64 / LW;  // w <= 64
  double xw[XR];
#pragma unroll
  for (int r = 0; r < XR; ++r) xw[r] = (lane + r * LW < w) ? x[f + lane + r * LW] : 0.0;
  // the previous step's flag is published after this step's first loads are issued (see fwd)
  if (rel_prev >= 0 && lane == 0) st_release(done + rel_prev, A.epoch);
#pragma unroll
  for (int r = 0; r < XR; ++r)
    if (lane + r * LW < w) tv[lane + r * LW] = xw[r];
  for (int i = lane; i < mu; i += LW) {
    ridx[i] = __ldg(S.srows + M.r0 + w + i);
    CKB(ridx[i] >= f + w && ridx[i] < A.n);
  }
  const unsigned long long t0 = g_debug_ts ? gtimer() : 0ull;
  if (p >= 0) wait_epoch(done + p, A.epoch);  // all lanes: uniform control flow
  wsync();
  const unsigned long long t1 = g_debug_ts ? gtimer() : 0ull;
  for (int i = lane; i < mu; i += LW) xr[i] = __ldcg(x + ridx[i]);
  wsync();
  warp_coldot(P + w, m, mu, w, xr, tv, -1.0, tv, lane, red);  // t = y - L21^T x_R
  wsync();
  warp_coldot(P, m, w, w, tv, nullptr, 1.0, xr, lane, red);   // x_s = Z^T t  (xr reused as output)
  wsync();
  for (int i = lane; i < w; i += LW) x[f + i] = xr[i];
  if (g_debug_ts && lane == 0 && b == 0) {
    g_debug_ts[4 * s] = t0;
    g_debug_ts[4 * s + 1] = t1;
    g_debug_ts[4 * s + 2] = gtimer();
    g_debug_ts[4 * s + 3] = 0;
  }
}

__global__ void __launch_bounds__(32 * SOLVE_WARPS, SOLVE_MINB) k_bwd_persist(SymDev S, SweepArgs A) {
  A.epoch = *A.epoch_ptr;  // bumped by the sweep's first launch (CUDA-graph safe)
  extern __shared__ double smem[];
  __shared__ int tk_sh[SOLVE_WORKERS];
  __shared__ SnMeta msh_all[SOLVE_WORKERS][16];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.ctr[(A.epoch + 1) & 1] = 0;
    A.ctr[2 + ((A.epoch + 1) & 1)] = 0;
  }
  const int lane = threadIdx.x % LW, wk = threadIdx.x / LW;
  double* xr = smem + (size_t)wk * (A.max_m + 64 + RED_SZ);
  double* tv = xr + A.max_m;
  double* red = tv + 64;
  int* ridx = reinterpret_cast<int*>(smem + (size_t)SOLVE_WORKERS * (A.max_m + 64 + RED_SZ)) + wk * A.max_m;
  SnMeta* msh = msh_all[wk];
  // bottom queue, chunks in reverse topological order
  for (;;) {
    const int t = warp_ticket(&A.ctr[A.epoch & 1], lane, &tk_sh[wk]);
    if (t >= A.nchunk * A.B) break;
    const int ch = A.nchunk - 1 - t / A.B, b = t % A.B;
    int* done = A.done_all + (int64_t)b * A.ns;
    const bool sk = A.skip && A.skip[b];
    const int q0 = A.chunk_ptr[ch], n = A.chunk_ptr[ch + 1] - q0;
    if (!sk) warp_stage_chunk(S, A, q0, n, b, lane, msh, true);
    int pend = -1;
    for (int j = n - 1; j >= 0; --j) {
      const int s = sk ? A.queue[q0 + j] : msh[j].pad1;
      if (!sk) {
        bwd_warp_step(S, A, msh[j], s, b, lane, xr, tv, red, ridx, done, pend);
        wsync();
        pend = s;
      } else if (lane == 0) {
        st_release(done + s, A.epoch);
      }
    }
    if (pend >= 0 && lane == 0) st_release(done + pend, A.epoch);
    wsync();
  }
}

// ============================================================================================
// Top set (large panels and their ancestors): one CTA per supernode, separate persistent launches
// (forward: after the warp-mode kernel; backward: before it) sized for 2 CTAs per SM.  The panel is
// copied into shared memory by ONE bulk async copy (cp.async.bulk, completion on an mbarrier) issued
// at the start of the step, so it lands while the CTA gathers its children's update vectors
// (forward) or waits for its parent and gathers x (backward); the CTA takes its next ticket one step
// ahead and prefetches that panel into L2.  The dense work then runs out of shared memory.  Panels
// larger than the buffer are read from global memory by the same code (generic pointer).
// ============================================================================================
#ifndef CKKT_TOP_THREADS
#define CKKT_TOP_THREADS 256
#endif
#ifndef CKKT_TOP_MINB
#define CKKT_TOP_MINB 2
#endif
constexpr int TOP_THREADS = CKKT_TOP_THREADS, TOP_WARPS = TOP_THREADS / 32, TOP_MINB = CKKT_TOP_MINB;
constexpr int TOP_CPW = 64 / TOP_WARPS;  // backward: columns per warp (w <= 64)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// shared state of a top-kernel CTA
struct TopShared {
  uint64_t bar;
  int tk_next;
  SnMeta m_next;  // metadata of the reserved next ticket
  ChMeta cmeta[32];
};

// Issue the panel of (q, b) into buf (thread 0).  Returns the panel pointer the CTA computes from
// (inside buf, or the global panel when it does not fit) — every thread evaluates it identically.
__device__ __forceinline__ const double* top_panel(const SweepArgs& A, const SnMeta& M, int b, double* buf,
                                                   TopShared& sh, bool issue) {
  const double* P = A.L + b * A.Lsize + M.pofs;
  const uintptr_t a = reinterpret_cast<uintptr_t>(P);
  const int off = (int)((a & 15) >> 3);  // doubles between the 16-byte aligned start and the panel
  const int64_t bytes = ((int64_t)(M.m * M.w + off) * 8 + 15) & ~int64_t(15);
  if (bytes > (int64_t)A.topbuf * 8) return P;
  if (issue) {
    mbar_expect_tx(&sh.bar, (uint32_t)bytes);
    bulk_g2s(buf, reinterpret_cast<const void*>(a & ~uintptr_t(15)), (uint32_t)bytes, &sh.bar);
  }
  return buf + off;
}

// one thread reserves the CTA's next ticket, stages its metadata in shared memory and prefetches
// its panel into L2 (the reservation runs one step ahead; tickets stay in topological order, and a
// reserved ticket is started as soon as the current one completes, so no CTA can wait on a ticket
// that is not being worked on)
__device__ __forceinline__ void top_reserve_next(const SweepArgs& A, int* ctr, TopShared& sh, bool reverse) {
  const int tn = atomicAdd(ctr, 1);
  sh.tk_next = tn;
  if (tn >= A.ntop * A.B) return;
  const int q = reverse ? A.ntop - 1 - tn / A.B : tn / A.B, b = tn % A.B;
  const SnMeta Mn = A.topmeta[q];
  sh.m_next = Mn;
  prefetch_l2(A.L + b * A.Lsize + Mn.pofs, 8ll * Mn.m * Mn.w);
}

__global__ void __launch_bounds__(TOP_THREADS, TOP_MINB) k_fwd_top(SymDev S, SweepArgs A) {
  A.epoch = *A.epoch_ptr;  // bumped by the sweep's first launch (CUDA-graph safe)
  extern __shared__ __align__(16) double smem[];
  __shared__ TopShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* buf = smem;                       // [topbuf]
  double* v = buf + A.topbuf;               // [max_m]
  double* y = v + A.max_m;                  // [64]
  int* ctr = &A.ctr[2 + (A.epoch & 1)];
  if (blockIdx.x == 0 && tid == 0) A.ctr[2 + ((A.epoch + 1) & 1)] = 0;
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    top_reserve_next(A, ctr, sh, false);
  }
  __syncthreads();
  uint32_t parity = 0;
  int t = sh.tk_next;
  const int total = A.ntop * A.B;
  while (t < total) {
    const int b = t % A.B;
    const SnMeta M = sh.m_next;
    const int s = M.pad1, f = M.f, w = M.w, m = M.m, mu = m - w;
    int* done = A.done_all + (int64_t)b * A.ns;
    const bool sk = A.skip && A.skip[b];
    CKB(M.pofs + (int64_t)m * w <= A.Lsize && M.vofs + mu <= A.Vsize && f + w <= A.n && m <= A.max_m && w <= 64);
    const unsigned long long t0 = g_debug_ts ? gtimer() : 0ull;
    unsigned long long t1 = t0;
    const double* Pl = sk ? nullptr : top_panel(A, M, b, buf, sh, tid == 0);
    const bool in_smem = Pl != nullptr && Pl != A.L + b * A.Lsize + M.pofs;
    __syncthreads();  // everyone has read sh.tk_next (and the previous step is complete)
    if (tid == 64) top_reserve_next(A, ctr, sh, false);  // warp 2 (warp 0 polls the flags)
    if (!sk) {
      double* x = A.X + (int64_t)b * A.n;
      const double* Vb = A.Vb + b * A.Vsize;
      for (int i = tid; i < m; i += TOP_THREADS) v[i] = (i < w) ? x[f + i] : 0.0;
      // children's update vectors: all (row, value) pairs of up to 8 children are loaded before any
      // is applied (one memory round trip), then added child by child (fixed order, deterministic)
      for (int cb = M.ch0; cb < M.ch1; cb += 32) {
        const int nc = min(32, M.ch1 - cb);
        if (warp == 0 && lane < nc) {
          const ChMeta cm = S.chmeta[cb + lane];
          sh.cmeta[lane] = cm;
          if (!cm.tiny) wait_epoch(done + cm.c, A.epoch);
        }
        __syncthreads();
        for (int k0 = 0; k0 < nc; k0 += 8) {
          double uv[8];
          int rl[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            rl[k] = -1;
            if (k0 + k < nc) {
              const ChMeta& cm = sh.cmeta[k0 + k];
              if (tid < cm.mc) {
                rl[k] = __ldg(S.relmap + cm.relofs + tid);
                uv[k] = __ldcg(Vb + cm.vofs + tid);
                CKB(rl[k] >= 0 && rl[k] < m && cm.vofs + cm.mc <= A.Vsize);
              }
            }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (k0 + k < nc) {
              if (rl[k] >= 0) v[rl[k]] += uv[k];
              __syncthreads();
            }
          }
          for (int k = k0; k < min(nc, k0 + 8); ++k) {  // rows beyond the first TOP_THREADS
            const ChMeta& cm = sh.cmeta[k];
            if (cm.mc > TOP_THREADS) {
              for (int i = TOP_THREADS + tid; i < cm.mc; i += TOP_THREADS)
                v[__ldg(S.relmap + cm.relofs + i)] += __ldcg(Vb + cm.vofs + i);
              __syncthreads();
            }
          }
        }
      }
      if (g_debug_ts) t1 = gtimer();
      if (in_smem) {
        mbar_wait(&sh.bar, parity);
        parity ^= 1;
      }
      __syncthreads();
      // y = Z v[0:w]  (thread per row; Z is lower triangular)
      if (tid < w) {
        double a0 = 0.0, a1 = 0.0;
        int c = 0;
        for (; c + 1 <= tid; c += 2) {
          a0 += Pl[tid + c * m] * v[c];
          a1 += Pl[tid + (c + 1) * m] * v[c + 1];
        }
        if (c <= tid) a0 += Pl[tid + c * m] * v[c];
        y[tid] = a0 + a1;
        x[f + tid] = a0 + a1;
      }
      __syncthreads();
      // u = v[w:m] - L21 y  (thread per row)
      double* us = A.Vb + b * A.Vsize + M.vofs;
      for (int i = tid; i < mu; i += TOP_THREADS) {
        double a0 = v[w + i], a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const double* pr = Pl + w + i;
        int c = 0;
        for (; c + 3 < w; c += 4) {
          a0 -= pr[c * m] * y[c];
          a1 -= pr[(c + 1) * m] * y[c + 1];
          a2 -= pr[(c + 2) * m] * y[c + 2];
          a3 -= pr[(c + 3) * m] * y[c + 3];
        }
        for (; c < w; ++c) a0 -= pr[c * m] * y[c];
        us[i] = (a0 + a1) + (a2 + a3);
      }
    }
    __syncthreads();  // all writes of this step precede the release; buffers free for the next copy
    if (tid == 0) st_release(done + s, A.epoch);
    if (g_debug_ts && tid == 0 && b == 0) {
      g_debug_ts[4 * s] = t0;
      g_debug_ts[4 * s + 1] = t1;
      g_debug_ts[4 * s + 2] = gtimer();
      g_debug_ts[4 * s + 3] = 1;
    }
    t = sh.tk_next;
  }
}

__global__ void __launch_bounds__(TOP_THREADS, TOP_MINB) k_bwd_top(SymDev S, SweepArgs A) {
  A.epoch = *A.epoch_ptr;  // bumped by the sweep's first launch (CUDA-graph safe)
  extern __shared__ __align__(16) double smem[];
  __shared__ TopShared sh;
  __shared__ double red[TOP_WARPS][TOP_CPW * 33 + 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* buf = smem;                       // [topbuf]
  double* xr = buf + A.topbuf;              // [max_m]
  double* tv = xr + A.max_m;                // [64]
  double* xo = tv + 64;                     // [64]
  int* ctr = &A.ctr[2 + (A.epoch & 1)];
  if (blockIdx.x == 0 && tid == 0) A.ctr[2 + ((A.epoch + 1) & 1)] = 0;
  if (tid == 0) {
    mbar_init(&sh.bar, 1);
    top_reserve_next(A, ctr, sh, true);
  }
  __syncthreads();
  uint32_t parity = 0;
  int t = sh.tk_next;
  const int total = A.ntop * A.B;
  while (t < total) {
    const int b = t % A.B;
    const SnMeta M = sh.m_next;
    const int s = M.pad1, p = M.pad0, f = M.f, w = M.w, m = M.m, mu = m - w;
    int* done = A.done_all + (int64_t)b * A.ns;
    const bool sk = A.skip && A.skip[b];
    const unsigned long long t0 = g_debug_ts ? gtimer() : 0ull;
    unsigned long long t1 = t0;
    const double* Pl = sk ? nullptr : top_panel(A, M, b, buf, sh, tid == 0);
    const bool in_smem = Pl != nullptr && Pl != A.L + b * A.Lsize + M.pofs;
    __syncthreads();
    if (tid == 64) top_reserve_next(A, ctr, sh, true);
    if (!sk) {
      double* x = A.X + (int64_t)b * A.n;
      if (tid < w) tv[tid] = x[f + tid];
      int ri[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        ri[k] = (tid + k * TOP_THREADS < mu) ? __ldg(S.srows + M.r0 + w + tid + k * TOP_THREADS) : 0;
      if (tid == 0 && p >= 0) wait_epoch(done + p, A.epoch);
      __syncthreads();
      if (g_debug_ts) t1 = gtimer();
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (tid + k * TOP_THREADS < mu) xr[tid + k * TOP_THREADS] = __ldcg(x + ri[k]);
      for (int i = tid + 4 * TOP_THREADS; i < mu; i += TOP_THREADS) xr[i] = __ldcg(x + __ldg(S.srows + M.r0 + w + i));
      if (in_smem) {
        mbar_wait(&sh.bar, parity);
        parity ^= 1;
      }
      __syncthreads();
      // two column-dot passes: t = y - L21^T x_R (rows w..m), then x_s = Z^T t (rows 0..w).
      // Warp `warp` owns columns c = warp + TOP_WARPS j; lanes over rows; partials reduced through
      // shared memory in two short stages.
      for (int pass = 0; pass < 2; ++pass) {
        const double* base = pass == 0 ? Pl + w : Pl;
        const double* xv = pass == 0 ? xr : tv;
        const int nr = pass == 0 ? mu : w;
        double pp[TOP_CPW];
#pragma unroll
        for (int j = 0; j < TOP_CPW; ++j) pp[j] = 0.0;
        for (int i = lane; i < nr; i += 32) {
          const double xi = xv[i];
#pragma unroll
          for (int j = 0; j < TOP_CPW; ++j) {
            const int c = warp + TOP_WARPS * j;
            if (c < w) pp[j] += base[i + c * m] * xi;
          }
        }
        double* rw = red[warp];
#pragma unroll
        for (int j = 0; j < TOP_CPW; ++j) rw[j * 33 + lane] = pp[j];
        __syncwarp();
        {
          constexpr int H = 32 / TOP_CPW;
          const int j = lane % TOP_CPW, h = lane / TOP_CPW;
          const double* qv = rw + j * 33 + TOP_CPW * h;
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int k = 0; k < TOP_CPW; k += 2) {
            s0 += qv[k];
            s1 += qv[k + 1];
          }
          rw[TOP_CPW * 33 + j * H + h] = s0 + s1;
        }
        __syncwarp();
        if (lane < TOP_CPW) {
          constexpr int H = 32 / TOP_CPW;
          const int c = warp + TOP_WARPS * lane;
          if (c < w) {
            const double* r2 = rw + TOP_CPW * 33 + lane * H;
            double sum = 0.0;
#pragma unroll
            for (int h = 0; h < H; ++h) sum += r2[h];
            if (pass == 0) tv[c] -= sum;
            else xo[c] = sum;
          }
        }
        __syncthreads();
      }
      if (tid < w) x[f + tid] = xo[tid];
    }
    __syncthreads();
    if (tid == 0) st_release(done + s, A.epoch);
    if (g_debug_ts && tid == 0 && b == 0) {
      g_debug_ts[4 * s] = t0;
      g_debug_ts[4 * s + 1] = t1;
      g_debug_ts[4 * s + 2] = gtimer();
      g_debug_ts[4 * s + 3] = 1;
    }
    t = sh.tk_next;
  }
}

// ============================================================================================
// tiny supernodes (m <= TINY_M, w <= TINY_W, whole subtree tiny): one THREAD per tiny subtree,
// nodes in postorder (forward) / reverse postorder (backward).  Forward runs before the warp
// kernel, backward after it, so no flags are needed: every dependency outside the subtree was
// completed by the other launch, every dependency inside it by the same thread.
// ============================================================================================
#ifndef CKKT_TINY_M
#define CKKT_TINY_M 32
#endif
#ifndef CKKT_TINY_W
#define CKKT_TINY_W 6
#endif
constexpr int TINY_M = CKKT_TINY_M, TINY_W = CKKT_TINY_W;

// Sweeps of the tiny subtrees: a group of TG = 8 lanes per (subtree, instance), lanes over the
// (at most 32) rows of each node, so panel and update-vector accesses are coalesced inside a group;
// nodes in postorder (forward) / reverse postorder (backward).  tmeta = SnMeta in sub_nodes order.
#ifndef CKKT_TG
#define CKKT_TG 8
#endif
constexpr int TG = CKKT_TG;
static_assert(TINY_M <= 32 && 32 % TG == 0, "tiny sweep layout");

__global__ void __launch_bounds__(256)
    k_fwd_tiny(SymDev S, const SnMeta* __restrict__ tmeta, const int32_t* __restrict__ sub_ptr, int nsub, int B,
               const double* __restrict__ L, int64_t Lsize, double* X, int n, double* Vb, int64_t Vsize,
               const int* __restrict__ skip, int* epoch_dev) {
  __shared__ double vsh_all[256 / TG][TINY_M];
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // new sweep epochs (forward and the backward that follows)
    epoch_dev[0] += 1;
    epoch_dev[1] += 1;
  }
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / TG, g = threadIdx.x % TG;
  if (gid >= nsub * B) return;  // group-uniform
  const unsigned mask = (TG == 32 ? 0xFFFFFFFFu : ((1u << TG) - 1u)) << ((threadIdx.x & 31) & ~(TG - 1));
  const int sub = gid / B, b = gid % B;
  if (skip && skip[b]) return;
  double* v = vsh_all[threadIdx.x / TG];
  double* x = X + (int64_t)b * n;
  double* Vbb = Vb + b * Vsize;
  const int q1 = sub_ptr[sub + 1];
  if (g == 0) {  // the subtree's panels are one contiguous span of L (sweep-ordered storage)
    const SnMeta a = tmeta[sub_ptr[sub]], z = tmeta[q1 - 1];
    prefetch_l2(L + b * Lsize + a.pofs, 8ll * (z.pofs + (int64_t)z.m * z.w - a.pofs));
  }
  for (int q = sub_ptr[sub]; q < q1; ++q) {
    const SnMeta M = tmeta[q];
    const int f = M.f, w = M.w, m = M.m;
    const double* P = L + b * Lsize + M.pofs;
#pragma unroll
    for (int i = g; i < TINY_M; i += TG) v[i] = (i < w) ? x[f + i] : 0.0;
    __syncwarp(mask);
    for (int ci = M.ch0; ci < M.ch1; ++ci) {
      const ChMeta cm = S.chmeta[ci];
      const double* uc = Vbb + cm.vofs;
      const int32_t* rel = S.relmap + cm.relofs;
      for (int i = g; i < cm.mc; i += TG) v[__ldg(rel + i)] += __ldcg(uc + i);
      __syncwarp(mask);
    }
    double y[TINY_W];
#ifndef CKKT_TINY_Y_ALL
    // y = Z v[0:w]: lane k < w computes y_k, the group shares them by shuffles
    {
      static_assert(TINY_W <= TG, "one lane per column of a tiny supernode");
      double yk = 0.0;
#pragma unroll
      for (int j = 0; j < TINY_W; ++j)
        if (j <= g && g < w) yk += P[g + j * m] * v[j];
      const int lane0 = (threadIdx.x & 31) & ~(TG - 1);
#pragma unroll
      for (int k = 0; k < TINY_W; ++k) y[k] = __shfl_sync(mask, yk, lane0 + k);
    }
#else
    // y = Z v[0:w] (every lane of the group, broadcast loads); lane k < w stores y_k
#pragma unroll
    for (int k = 0; k < TINY_W; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < TINY_W; ++j)
        if (j <= k && k < w) acc += P[k + j * m] * v[j];
      y[k] = acc;
    }
#endif
#pragma unroll
    for (int k = 0; k < TINY_W; ++k)
      if (k % TG == g && k < w) x[f + k] = y[k];
    double* us = Vbb + M.vofs;
#pragma unroll
    for (int i0 = 0; i0 < TINY_M; i0 += TG) {
      const int i = i0 + g;
      if (i >= w && i < m) {
        double acc = v[i];
#pragma unroll
        for (int k = 0; k < TINY_W; ++k)
          if (k < w) acc -= P[i + k * m] * y[k];
        us[i - w] = acc;
      }
    }
    __syncwarp(mask);
  }
}

__global__ void __launch_bounds__(256)
    k_bwd_tiny(SymDev S, const SnMeta* __restrict__ tmeta, const int32_t* __restrict__ sub_ptr, int nsub, int B,
               const double* __restrict__ L, int64_t Lsize, double* X, int n, const int* __restrict__ skip) {
#ifdef CKKT_TINY_RED_SMEM
  __shared__ double red_all[256 / TG][TINY_W][TG + 1];
#endif
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / TG, g = threadIdx.x % TG;
  if (gid >= nsub * B) return;
  const unsigned mask = (TG == 32 ? 0xFFFFFFFFu : ((1u << TG) - 1u)) << ((threadIdx.x & 31) & ~(TG - 1));
  const int sub = gid / B, b = gid % B;
  if (skip && skip[b]) return;
#ifdef CKKT_TINY_RED_SMEM
  auto red = red_all[threadIdx.x / TG];
#endif
  double* x = X + (int64_t)b * n;
  const int q0 = sub_ptr[sub];
  if (g == 0) {  // contiguous span of the subtree's panels
    const SnMeta a = tmeta[q0], z = tmeta[sub_ptr[sub + 1] - 1];
    prefetch_l2(L + b * Lsize + a.pofs, 8ll * (z.pofs + (int64_t)z.m * z.w - a.pofs));
  }
  for (int q = sub_ptr[sub + 1] - 1; q >= q0; --q) {
    const SnMeta M = tmeta[q];
    const int f = M.f, w = M.w, m = M.m;
    const double* P = L + b * Lsize + M.pofs;
    // partial t_c = -sum_{rows i of this lane} L21[i, c] x_R[i]
    double part[TINY_W];
#pragma unroll
    for (int c = 0; c < TINY_W; ++c) part[c] = 0.0;
#pragma unroll
    for (int i0 = 0; i0 < TINY_M; i0 += TG) {
      const int i = i0 + g;
      if (i >= w && i < m) {
        const double xi = __ldcg(x + __ldg(S.srows + M.r0 + i));
#pragma unroll
        for (int c = 0; c < TINY_W; ++c)
          if (c < w) part[c] -= P[i + c * m] * xi;
      }
    }
    double tv[TINY_W];
#ifndef CKKT_TINY_RED_SMEM
    // butterfly over the group's TG lanes (every lane ends with every column's sum)
#pragma unroll
    for (int c = 0; c < TINY_W; ++c) {
      double v = part[c];
#pragma unroll
      for (int o = TG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
      tv[c] = ((c < w) ? x[f + c] : 0.0) + v;
    }
#else
#pragma unroll
    for (int c = 0; c < TINY_W; ++c) red[c][g] = part[c];
    __syncwarp(mask);
#pragma unroll
    for (int c = 0; c < TINY_W; ++c) {
      double acc = (c < w) ? x[f + c] : 0.0;
#pragma unroll
      for (int l = 0; l < TG; ++l) acc += red[c][l];
      tv[c] = acc;
    }
#endif
    // x_s = Z^T t: lane i < w computes row i
#pragma unroll
    for (int i = 0; i < TINY_W; ++i) {
      if (i % TG == g && i < w) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < TINY_W; ++k)
          if (k >= i && k < w) acc += P[k + i * m] * tv[k];
        x[f + i] = acc;
      }
    }
    __syncwarp(mask);
  }
}

// Factor of the tiny subtrees: a group of TG lanes per (subtree, instance), nodes in postorder,
// front panel (m <= 32 rows, w <= 4 columns, ld 32) in the group's shared memory, rows over lanes.
// Same arithmetic as the big fronts: assemble A + children's panel parts, Cholesky of
// the w columns, U_s = -L21 L21^T plus the children's trailing parts, L11 <- L11^{-1}.
#ifndef CKKT_FT_THREADS
#define CKKT_FT_THREADS 128
#endif
constexpr int FT_THREADS = CKKT_FT_THREADS;

__global__ void k_epoch_bump(int* epoch_dev) {  // sweeps without tiny subtrees
  epoch_dev[0] += 1;
  epoch_dev[1] += 1;
}
__global__ void __launch_bounds__(FT_THREADS)
    k_factor_tiny(SymDev S, const SnMeta* __restrict__ tmeta, const int32_t* __restrict__ sub_ptr, int nsub, int B,
                  double* L, int64_t Lsize, double* Ub, int64_t Usize, const double* __restrict__ Kval, int64_t nnzk,
                  int* notpd, int* minpiv) {
  constexpr int LD = 32;
  __shared__ double pan_all[FT_THREADS / TG][LD * TINY_W];
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / TG, g = threadIdx.x % TG;
  if (gid >= nsub * B) return;  // group-uniform
  const unsigned mask = (TG == 32 ? 0xFFFFFFFFu : ((1u << TG) - 1u)) << ((threadIdx.x & 31) & ~(TG - 1));
  const int sub = gid / B, b = gid % B;
  double* Pn = pan_all[threadIdx.x / TG];
  const double* Kb = Kval + b * nnzk;
  double* Ubb = Ub + b * Usize;
  const int q1 = sub_ptr[sub + 1];
  for (int q = sub_ptr[sub]; q < q1; ++q) {
    const SnMeta M = tmeta[q];
    const int f = M.f, w = M.w, m = M.m, mu = m - w;
    // (1) A's entries of the w columns (kmap is relative to the m x w panel with ld m)
    for (int e = g; e < LD * TINY_W; e += TG) Pn[e] = 0.0;
    __syncwarp(mask);
    for (int64_t k = S.kp[f] + g; k < S.kp[f + w]; k += TG) {
      const int qq = S.kmap[k];
      Pn[(qq % m) + (qq / m) * LD] = Kb[k];
    }
    __syncwarp(mask);
    // (2) children's panel parts (columns j with rel[j] < w), child by child
    for (int ci = M.ch0; ci < M.ch1; ++ci) {
      const ChMeta cm = S.chmeta[ci];
      const double* Uc = Ubb + S.uofs[cm.c];
      const int32_t* rel = S.relmap + cm.relofs;
      for (int j = 0; j < cm.mc; ++j) {
        const int rj = __ldg(rel + j);
        if (rj >= w) break;
        for (int i = j + g; i < cm.mc; i += TG) Pn[__ldg(rel + i) + rj * LD] += __ldcg(Uc + i + j * cm.mc);
      }
      __syncwarp(mask);
    }
    // (3) Cholesky of the w columns (rows over lanes)
    for (int j = 0; j < w; ++j) {
      double d = Pn[j + j * LD];
      if (!(d > 0.0) || !isfinite(d)) {
        if (g == 0) {
          notpd[b] = 1;
          atomicMin(&minpiv[b], f + j);
        }
        d = nan("");
      }
      const double rp = 1.0 / sqrt(d);
      __syncwarp(mask);
      for (int i = j + 1 + g; i < m; i += TG) Pn[i + j * LD] *= rp;
      if (g == 0) Pn[j + j * LD] = d * rp;
      __syncwarp(mask);
      for (int c2 = j + 1; c2 < w; ++c2) {
        const double lc = Pn[c2 + j * LD];
        for (int i = c2 + g; i < m; i += TG) Pn[i + c2 * LD] -= Pn[i + j * LD] * lc;
      }
      __syncwarp(mask);
    }
    // (4) U_s = -L21 L21^T (lower, column-major mu x mu), then the children's trailing parts
    double* U = Ubb + S.uofs[M.pad1];  // (tmeta: pad1 = supernode)
    for (int j = 0; j < mu; ++j)
      for (int i = j + g; i < mu; i += TG) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < TINY_W; ++k)
          if (k < w) acc += Pn[w + i + k * LD] * Pn[w + j + k * LD];
        U[i + j * mu] = -acc;
      }
    __syncwarp(mask);
    for (int ci = M.ch0; ci < M.ch1; ++ci) {
      const ChMeta cm = S.chmeta[ci];
      const double* Uc = Ubb + S.uofs[cm.c];
      const int32_t* rel = S.relmap + cm.relofs;
      for (int j = 0; j < cm.mc; ++j) {
        const int rj = __ldg(rel + j);
        if (rj < w) continue;
        for (int i = j + g; i < cm.mc; i += TG) U[(__ldg(rel + i) - w) + (rj - w) * mu] += __ldcg(Uc + i + j * cm.mc);
      }
      __syncwarp(mask);
    }
    // (5) L11 <- L11^{-1} (w <= 4): lane i < w computes row i from rows < i, one row per step
    for (int i = 0; i < w; ++i) {
      double z[TINY_W];
#pragma unroll
      for (int jj = 0; jj < TINY_W; ++jj) z[jj] = 0.0;
      if (g == 0) {
        const double rii = 1.0 / Pn[i + i * LD];
#pragma unroll
        for (int jj = 0; jj < TINY_W; ++jj) {
          if (jj <= i) {
            double acc = (jj == i) ? 1.0 : 0.0;
            for (int k = jj; k < i; ++k) acc -= Pn[i + k * LD] * Pn[k + jj * LD];
            z[jj] = acc * rii;
          }
        }
#pragma unroll
        for (int jj = 0; jj < TINY_W; ++jj)
          if (jj <= i) Pn[i + jj * LD] = z[jj];
      }
      __syncwarp(mask);
    }
    // (6) panel out (column-major m x w)
    double* Pg = L + b * Lsize + M.pofs;
    for (int e = g; e < m * w; e += TG) Pg[e] = Pn[(e % m) + (e / m) * LD];
    __syncwarp(mask);
  }
}
