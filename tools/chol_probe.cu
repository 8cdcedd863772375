#include <cstdio>
#include <cstdint>
#ifndef CKKT_DBG_CHOL
#define CKKT_DBG_CHOL 0  // timing experiments only: 1 = no inversion, 2 = no pivot math, 3 = no column dots
#endif
// 1/sqrt(d) to full double precision: single-precision estimate + two Newton steps (no IEEE
// sqrt/divide subroutines on the critical path); falls back to them outside the float range.
__device__ __forceinline__ double rsqrt_fast(double d) {
  if (!(d > 1e-30 && d < 1e30)) return 1.0 / sqrt(d);
  double r = (double)rsqrtf((float)d);
  r = r * (1.5 - 0.5 * d * r * r);
  r = r * (1.5 - 0.5 * d * r * r);
  return r;
}

// One warp: A11 (w x w, w <= 64, lower part of the panel top) <- Z = L11^{-1} where L11 = chol(A11).
// Lanes own rows lane and lane + 32.  Left-looking (Crout) Cholesky fused with the row-wise
// inversion: iteration j computes column j of L (a dot product over the finished columns k < j),
// and row j of Z (row j of L is final once its pivot is known; Z[j][c] = -r_j sum_{k=c}^{j-1}
// L[j][k] Z[k][c], lanes over c).  Row j of Z replaces row j of L, which no later column needs.
// One __syncwarp per column; reciprocal pivots in dsh[].
__device__ __forceinline__ void warp_chol_inv(double* Ps, int ldp, int w, int lane, double* dsh, int* notpd_b,
                                              int* minpiv_b, int f) {
  const int i0 = lane, i1 = lane + 32;
  for (int j = 0; j < w; ++j) {
    // (a) column j of L before scaling, rows i >= j
    double s0 = 0.0, s1 = 0.0;
    const bool a0 = i0 >= j && i0 < w, a1 = i1 >= j && i1 < w;
    if (a0) s0 = Ps[i0 + j * ldp];
    if (a1) s1 = Ps[i1 + j * ldp];
#if CKKT_DBG_CHOL != 3
    for (int k = 0; k < j; ++k) {
      const double ljk = Ps[j + k * ldp];
      if (a0) s0 -= Ps[i0 + k * ldp] * ljk;
      if (a1) s1 -= Ps[i1 + k * ldp] * ljk;
    }
#endif
    // (b) pivot
    if (i0 == j || i1 == j) {
      double d = (i0 == j) ? s0 : s1;
      if (!(d > 0.0) || !isfinite(d)) {
        *notpd_b = 1;
        atomicMin(minpiv_b, f + j);
        d = nan("");
      }
#if CKKT_DBG_CHOL == 2
      dsh[j] = d;
#else
      dsh[j] = rsqrt_fast(d);
#endif
    }
    __syncwarp();
    const double rp = dsh[j];
    // (c) scale column j; row j of Z (reads row j of L and Z rows < j: disjoint from the column)
    if (a0 && i0 > j) Ps[i0 + j * ldp] = s0 * rp;
    if (a1 && i1 > j) Ps[i1 + j * ldp] = s1 * rp;
    double z0 = 0.0, z1 = 0.0;
    if (CKKT_DBG_CHOL != 1 && lane < j) {
      for (int k = lane; k < j; ++k) z0 -= Ps[j + k * ldp] * Ps[k + lane * ldp];
      z0 *= rp;
    }
    if (lane + 32 < j) {
      for (int k = lane + 32; k < j; ++k) z1 -= Ps[j + k * ldp] * Ps[k + (lane + 32) * ldp];
      z1 *= rp;
    }
    __syncwarp();
    // (d) row j of Z over row j of L
    if (lane < j) Ps[j + lane * ldp] = z0;
    if (lane + 32 < j) Ps[j + (lane + 32) * ldp] = z1;
    if (lane == (j & 31)) Ps[j + j * ldp] = rp;
  }
  __syncwarp();
}


__global__ void kc(int w, int m, long long* out, int variant) {
  extern __shared__ double sm[];
  __shared__ double dsh[64];
  __shared__ int np, mpv;
  const int ldp = ((m + 7) & ~7) | 1;
  for (int e = threadIdx.x; e < ldp * 64 + 8; e += blockDim.x) {
    const int i = e % ldp, j = e / ldp;
    sm[e] = (i == j) ? 100.0 : ((i > j && i < m) ? 1.0 / (1 + i + j) : 0.0);
  }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 32) warp_chol_inv(sm, ldp, w, threadIdx.x, dsh, &np, &mpv, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  for (int w : {1, 2, 4, 8, 16, 32}) {
    int m = 4 * w + 4, ldp = ((m + 7) & ~7) | 1;
    cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * (ldp * 64 + 8));
    long long h = 0;
    for (int r = 0; r < 3; ++r) { kc<<<1, 32, 8 * (ldp * 64 + 8)>>>(w, m, d, 0); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); }
    printf("w=%d: %lld cycles (%lld/col)\n", w, h, h / w);
  }
}
