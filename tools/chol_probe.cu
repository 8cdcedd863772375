#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include "../paper_2403_15913_b200/csrc/dense_front.cuh"
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void warp_trsm_dmma(double* Ps, int ldp, int w, int m, int warp, int nwarp, int lane) {
  const int mu = m - w, g = lane >> 2, t4 = lane & 3;
  const int nI = (mu + 7) >> 3, nJ = (w + 7) >> 3;
  for (int I = warp; I < nI; I += nwarp) {
    const int ra = w + 8 * I + g;  // A21 row of this lane's A fragment
    double c[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) c[q] = 0.0;
    for (int k = 0; k < w; k += 4) {
      const int kc = k + t4;
      const double a = (ra < m && kc < w) ? Ps[ra + kc * ldp] : 0.0;
#pragma unroll
      for (int J = 0; J < 8; ++J) {
        if (J < nJ && k < 8 * J + 8) {  // Z[j][k] = 0 for k > j
          const int rb = 8 * J + g;
          const double bv = (rb < w && kc < w) ? Ps[rb + kc * ldp] : 0.0;
          dmma_8x8x4(c[2 * J], c[2 * J + 1], a, bv);
        }
      }
    }
    __syncwarp();
    const int row = w + 8 * I + g;
    if (row < m) {
#pragma unroll
      for (int J = 0; J < 8; ++J) {
        const int col = 8 * J + 2 * t4;
        if (J < nJ) {
          if (col < w) Ps[row + col * ldp] = c[2 * J];
          if (col + 1 < w) Ps[row + (col + 1) * ldp] = c[2 * J + 1];
        }
      }
    }
  }
}
__device__ __forceinline__ void warp_chol_inv(double* Ps, int ldp, int w, int lane, double* dsh, int* notpd_b,
                                              int* minpiv_b, int f) {
  const int i0 = lane, i1 = lane + 32;
  for (int j = 0; j < w; ++j) {
    double s0 = 0.0, s1 = 0.0;
    const bool a0 = i0 >= j && i0 < w, a1 = i1 >= j && i1 < w;
    if (a0) s0 = Ps[i0 + j * ldp];
    if (a1) s1 = Ps[i1 + j * ldp];
    for (int k = 0; k < j; ++k) {
      const double ljk = Ps[j + k * ldp];
      if (a0) s0 -= Ps[i0 + k * ldp] * ljk;
      if (a1) s1 -= Ps[i1 + k * ldp] * ljk;
    }
    if (i0 == j || i1 == j) {
      double d = (i0 == j) ? s0 : s1;
      if (!(d > 0.0) || !isfinite(d)) {
        *notpd_b = 1;
        atomicMin(minpiv_b, f + j);
        d = nan("");
      }
      const double piv = sqrt(d);
      Ps[j + j * ldp] = piv;
      dsh[j] = 1.0 / piv;
    }
    __syncwarp();
    const double rp = dsh[j];
    if (a0 && i0 > j) Ps[i0 + j * ldp] = s0 * rp;
    if (a1 && i1 > j) Ps[i1 + j * ldp] = s1 * rp;
    __syncwarp();
  }
  for (int i = 0; i < w; ++i) {  // Z = L11^{-1}: row i from rows < i
    double z0 = 0.0, z1 = 0.0;
    const double ri = dsh[i];
    if (lane <= i) {
      z0 = (lane == i) ? 1.0 : 0.0;
      for (int k = lane; k < i; ++k) z0 -= Ps[i + k * ldp] * Ps[k + lane * ldp];
      z0 *= ri;
    }
    if (lane + 32 <= i) {
      z1 = (lane + 32 == i) ? 1.0 : 0.0;
      for (int k = lane + 32; k < i; ++k) z1 -= Ps[i + k * ldp] * Ps[k + (lane + 32) * ldp];
      z1 *= ri;
    }
    __syncwarp();
    if (lane <= i) Ps[i + lane * ldp] = z0;
    if (lane + 32 <= i) Ps[i + (lane + 32) * ldp] = z1;
    __syncwarp();
  }
}

__global__ void kc(int w, int m, const double* in, double* res, long long* cyc, int mode) {
  extern __shared__ double sm[];
  __shared__ double dsh[64 * 8];
  __shared__ int np, mpv;
  const int ldp = ((m + 7) & ~7) | 1;
  const int tid = threadIdx.x;
  for (int e = tid; e < ldp * 64 + 8; e += blockDim.x) sm[e] = 0.0;
  __syncthreads();
  for (int e = tid; e < m * w; e += blockDim.x) { const int i = e % m, j = e / m; if (i >= j) sm[i + j * ldp] = in[e]; }
  if (tid == 0) { np = 0; mpv = 1 << 30; }
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    if (tid < 32) warp_chol_inv(sm, ldp, w, tid, dsh, &np, &mpv, 0);
    __syncthreads();
    warp_trsm_dmma(sm, ldp, w, m, tid >> 5, blockDim.x >> 5, tid & 31);
    __syncthreads();
  } else {
    dfront::cta_dense_blocked(sm, ldp, w, m, tid, blockDim.x, dsh, &np, &mpv, 0);
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  for (int e = tid; e < m * w; e += blockDim.x) res[e] = sm[(e % m) + (e / m) * ldp];
}
int main() {
  srand(1);
  double *din, *dr; long long* dc; cudaMalloc(&din, 8 * 256 * 64); cudaMalloc(&dr, 8 * 256 * 64); cudaMalloc(&dc, 8);
  static double A[256 * 64], R0[256 * 64], R1[256 * 64];
  for (int w : {1, 3, 8, 13, 16, 17, 24, 32, 40, 55, 64}) {
    int m = w + 3 * w + 5; if (m > 256) m = 256;
    // SPD-ish panel: diagonally dominant A11 (lower), random A21
    for (int j = 0; j < w; ++j) for (int i = 0; i < m; ++i) A[i + j * m] = (i == j) ? (w + 2.0 + j) : ((double)rand() / RAND_MAX - 0.5);
    cudaMemcpy(din, A, 8 * m * w, cudaMemcpyHostToDevice);
    int ldp = ((m + 7) & ~7) | 1, smem = 8 * (ldp * 64 + 8);
    cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long c0 = 0, c1 = 0;
    for (int r = 0; r < 3; ++r) { kc<<<1, 256, smem>>>(w, m, din, dr, dc, 0); cudaMemcpy(&c0, dc, 8, cudaMemcpyDeviceToHost); }
    cudaMemcpy(R0, dr, 8 * m * w, cudaMemcpyDeviceToHost);
    for (int r = 0; r < 3; ++r) { kc<<<1, 256, smem>>>(w, m, din, dr, dc, 1); cudaMemcpy(&c1, dc, 8, cudaMemcpyDeviceToHost); }
    cudaMemcpy(R1, dr, 8 * m * w, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (int e = 0; e < m * w; ++e) { md = fmax(md, fabs(R0[e] - R1[e])); mx = fmax(mx, fabs(R0[e])); }
    printf("w=%2d m=%3d: old %7lld cycles, blocked %7lld cycles, max|diff| %.3g (max %.3g)\n", w, m, c0, c1, md, mx);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
