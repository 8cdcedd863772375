// Blocked dense part of a multifrontal front, whole CTA, panel in shared memory (sm_100a, FP64).
// Included by mf_kernels.cuh (inside its anonymous namespace) and by tools/chol_probe.cu.
//
// Panel P (ld = ldp, rows 0..m-1, columns 0..w-1, w <= 64): on entry [A11; A21] (lower part of
// A11 significant), on exit [Z; L21] with Z = L11^{-1} (lower, strict upper part zero) and
// L21 = A21 L11^{-T}, where L11 = chol(A11)  (Z is what the GEMV-only sweeps use).
//
// Right-looking Cholesky in 16-column blocks.  Per block: one warp factors and inverts the 16 x 16
// diagonal block with the block in registers (one row per lane, one __syncwarp per column); every
// other update is an FP64 tensor-core tile product (mma.sync.m8n8k4.f64) by all warps:
//   rows below the block:   L[r, blk] = A[r, blk] Zd^T          (the TRSM, including the A21 rows)
//   trailing columns:       A[r, c]  -= L[r, blk] L[c, blk]^T   (rows >= c, A21 rows included)
// Finally Z is assembled from the inverted diagonal blocks by block forward substitution,
//   Z_ij = -Zd_i sum_{k=j}^{i-1} L_ik Z_kj,
// again on tensor-core tiles.  The serial part is 16 pivots per block instead of w dependent
// column steps over the whole width.

namespace dfront {

constexpr int NBW = 16;  // diagonal block width

__device__ __forceinline__ void mma8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 1/sqrt(d): single-precision estimate + two Newton steps (full double precision)
__device__ __forceinline__ double rsqrt_nr(double d) {
  if (!(d > 1e-30 && d < 1e30)) return 1.0 / sqrt(d);
  double r = (double)rsqrtf((float)d);
  r = r * (1.5 - 0.5 * d * r * r);
  r = r * (1.5 - 0.5 * d * r * r);
  return r;
}

// One warp: the bw x bw (bw <= 16) block at D (ld) <- its Cholesky factor's inverse (lower, zero
// upper part).  scr: per-warp shared scratch of >= 17 doubles.  Pivot failures set *notpd and the
// smallest failing global column f0 + j.
__device__ __forceinline__ void warp_chol_inv16(double* D, int ld, int bw, int lane, double* scr, int* notpd,
                                                int* minpiv, int f0) {
  double a[NBW];
#pragma unroll
  for (int c = 0; c < NBW; ++c) a[c] = (lane < bw && c <= lane) ? D[lane + c * ld] : 0.0;
  double rmine = 0.0;
#pragma unroll
  for (int j = 0; j < NBW; ++j) {
    if (j < bw) {
      if (lane == j) {
        double d = a[j];
        if (!(d > 0.0) || !isfinite(d)) {
          *notpd = 1;
          atomicMin(minpiv, f0 + j);
          d = nan("");
        }
        const double r = rsqrt_nr(d);
        rmine = r;
        a[j] = d * r;
        scr[NBW] = r;
      }
      __syncwarp();
      const double r = scr[NBW];
      if (lane > j && lane < bw) {
        a[j] *= r;
        scr[lane] = a[j];
      }
      __syncwarp();
#pragma unroll
      for (int c = j + 1; c < NBW; ++c)
        if (c <= lane && lane < bw) a[c] -= a[j] * scr[c];
      __syncwarp();
    }
  }
  // publish L (rows) with a cleared upper part, and the reciprocal pivots
#pragma unroll
  for (int c = 0; c < NBW; ++c)
    if (lane < bw && c < bw) D[lane + c * ld] = (c <= lane) ? a[c] : 0.0;
  if (lane < bw) scr[lane] = rmine;
  __syncwarp();
  // lane c: column c of Z = L^{-1} by forward substitution (z in registers)
  double z[NBW];
#pragma unroll
  for (int i = 0; i < NBW; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k)
      if (k >= lane && i < bw) s += D[i + k * ld] * z[k];  // (rows >= bw may lie outside the panel)
    const double ri = (i < bw) ? scr[i] : 0.0;
    z[i] = (i == lane) ? ri : ((i > lane) ? -ri * s : 0.0);
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NBW; ++i)
    if (lane < bw && i < bw && i >= lane) D[i + lane * ld] = z[i];
  __syncwarp();
}

// C (8 x 8 tile at rows r0.., columns c0.. of the panel) op= A B^T or A B with fragments read from
// shared memory by callers; helpers below are written out per phase for clarity.

// Dense part of a front (see the header comment).  Ps: panel, ldp, w (<= 64), m; scr >= 17
// doubles of scratch; all nt threads of the group (the CTA, or one warp with nt = 32) call it.
template <bool CTA>  // CTA: all warps of the block (__syncthreads); else one warp alone (__syncwarp)
__device__ __forceinline__ void group_sync() {
  if (CTA) __syncthreads();
  else __syncwarp();
}

template <bool CTA>
__device__ __forceinline__ void dense_blocked(double* Ps, int ldp, int w, int m, int tid, int nt, double* scr,
                                              int* notpd, int* minpiv, int f) {
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nb = (w + NBW - 1) / NBW;
  for (int kb = 0; kb < nb; ++kb) {
    const int o = NBW * kb, bw = min(NBW, w - o);
    // (a) diagonal block
    if (warp == 0) warp_chol_inv16(Ps + o + o * ldp, ldp, bw, lane, scr, notpd, minpiv, f + o);
    group_sync<CTA>();
    const int r0 = o + bw;  // first row below the block
    const int nI = (m - r0 + 7) >> 3;
    // (b) L[r, blk] = A[r, blk] Zd^T for r >= r0 (a warp owns whole 8-row tiles: in place)
    for (int I = warp; I < nI; I += nwarp) {
      const int ra = r0 + 8 * I + g;
      double c[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < NBW; k += 4) {
        const int kc = k + t4;
        const double av = (ra < m && kc < bw) ? Ps[ra + (o + kc) * ldp] : 0.0;
#pragma unroll
        for (int J = 0; J < 2; ++J) {
          const int rb = 8 * J + g;
          const double bv = (rb < bw && kc < bw) ? Ps[(o + rb) + (o + kc) * ldp] : 0.0;
          mma8x8x4(c[2 * J], c[2 * J + 1], av, bv);
        }
      }
      __syncwarp();
      if (ra < m) {
#pragma unroll
        for (int J = 0; J < 2; ++J) {
          const int col = 8 * J + 2 * t4;
          if (col < bw) Ps[ra + (o + col) * ldp] = c[2 * J];
          if (col + 1 < bw) Ps[ra + (o + col + 1) * ldp] = c[2 * J + 1];
        }
      }
    }
    group_sync<CTA>();
    // (c) trailing update of columns c >= r0 (< w), rows r >= r0: A[r, c] -= L[r, blk] L[c, blk]^T
    if (r0 < w) {
      const int nJ = (w - r0 + 7) >> 3;
      for (int tI = warp; tI < nI * nJ; tI += nwarp) {
        const int I = tI / nJ, J = tI - I * nJ;
        if (8 * I + 7 < 8 * J) continue;  // tile entirely above the diagonal
        const int ra = r0 + 8 * I + g, rb = r0 + 8 * J + g;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int k = 0; k < NBW; k += 4) {
          const int kc = k + t4;
          const double av = (ra < m && kc < bw) ? Ps[ra + (o + kc) * ldp] : 0.0;
          const double bv = (rb < w && kc < bw) ? Ps[rb + (o + kc) * ldp] : 0.0;
          mma8x8x4(c0, c1, av, bv);
        }
        const int row = r0 + 8 * I + g, col = r0 + 8 * J + 2 * t4;
        if (row < m) {
          if (col < w) Ps[row + col * ldp] -= c0;
          if (col + 1 < w) Ps[row + (col + 1) * ldp] -= c1;
        }
      }
      group_sync<CTA>();
    }
  }
  // (d) Z from the inverted diagonal blocks: Z_ij = -Zd_i sum_{k=j}^{i-1} L_ik Z_kj  (i > j)
  for (int bi = 1; bi < nb; ++bi) {
    const int oi = NBW * bi, bwi = min(NBW, w - oi);
    const int ntile = bi * 4;  // (j, 2 x 2 tiles of 8 x 8)
    // tiles of block row bi per warp: <= 2 for a CTA of 8 warps, <= 12 for one warp alone (nb <= 4)
    constexpr int MAXQ = CTA ? 2 : 12;
    double keep[MAXQ][2];
    // T_ij = sum_k L_ik Z_kj  (B = Z not transposed: b = Z[k][n])
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int tI = warp + q * nwarp;
      keep[q][0] = keep[q][1] = 0.0;
      if (tI < ntile) {
        const int j = tI >> 2, ti = (tI >> 1) & 1, tj = tI & 1;
        const int oj = NBW * j;
        const int ra = oi + 8 * ti + g;
        for (int kb2 = j; kb2 < bi; ++kb2) {
          const int okk = NBW * kb2;
#pragma unroll
          for (int k = 0; k < NBW; k += 4) {
            const int kr = okk + k + t4;  // row of Z_kj / column of L_ik
            const double av = (ra < w && kr < w) ? Ps[ra + kr * ldp] : 0.0;
            const int cb = oj + 8 * tj + g;
            const double bv = (kr < w && cb < w) ? Ps[kr + cb * ldp] : 0.0;
            mma8x8x4(keep[q][0], keep[q][1], av, bv);
          }
        }
      }
    }
    group_sync<CTA>();  // every T of block row bi computed before any L_ij is replaced
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int tI = warp + q * nwarp;
      if (tI < ntile) {
        const int j = tI >> 2, ti = (tI >> 1) & 1, tj = tI & 1;
        const int row = oi + 8 * ti + g, col = NBW * j + 8 * tj + 2 * t4;
        if (row < w) {
          Ps[row + col * ldp] = keep[q][0];
          Ps[row + (col + 1) * ldp] = keep[q][1];
        }
      }
    }
    group_sync<CTA>();
    // Z_ij = -Zd_i T_ij  (A = Zd_i lower with zero upper part, B = T not transposed)
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int tI = warp + q * nwarp;
      keep[q][0] = keep[q][1] = 0.0;
      if (tI < ntile) {
        const int j = tI >> 2, ti = (tI >> 1) & 1, tj = tI & 1;
        const int ra = oi + 8 * ti + g, cb = NBW * j + 8 * tj + g;
#pragma unroll
        for (int k = 0; k < NBW; k += 4) {
          const int kr = oi + k + t4;
          const double av = (ra < w && k + t4 < bwi) ? Ps[ra + kr * ldp] : 0.0;
          const double bv = (k + t4 < bwi) ? Ps[kr + cb * ldp] : 0.0;
          mma8x8x4(keep[q][0], keep[q][1], av, bv);
        }
      }
    }
    group_sync<CTA>();
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int tI = warp + q * nwarp;
      if (tI < ntile) {
        const int j = tI >> 2, ti = (tI >> 1) & 1, tj = tI & 1;
        const int row = oi + 8 * ti + g, col = NBW * j + 8 * tj + 2 * t4;
        if (row < w) {
          Ps[row + col * ldp] = -keep[q][0];
          Ps[row + (col + 1) * ldp] = -keep[q][1];
        }
      }
    }
    group_sync<CTA>();
  }
  // (e) clear the strict upper triangle of the w x w block (trailing-update tiles straddled it)
  for (int p = tid; p < w * w; p += nt) {
    const int i = p % w, c = p / w;
    if (i < c) Ps[i + c * ldp] = 0.0;
  }
  group_sync<CTA>();
}

}  // namespace dfront
