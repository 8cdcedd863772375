#include <cstdio>
__global__ void k(int w, long long* out, int mode) {
  __shared__ double Ps[64 * 65];
  __shared__ double dsh[64];
  const int tid = threadIdx.x, nt = blockDim.x, ldp = 65;
  for (int e = tid; e < 64 * 65; e += nt) Ps[e] = 1.0;
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j < w; ++j) {
    if (tid == 0) dsh[j] = 1.0 + Ps[j + j * ldp];
    __syncthreads();
    const double r = dsh[j];
    if (mode >= 1) {
      const int R = w - j - 1;
      int sh = 0;
      while ((1 << sh) < R) ++sh;
      for (int p = tid; p < (R << sh); p += nt) {
        const int ii = p >> sh, cc = p & ((1 << sh) - 1);
        if (cc <= ii) Ps[(j + 1 + ii) + (j + 1 + cc) * ldp] -= Ps[j + 1 + ii + j * ldp] * Ps[j + 1 + cc + j * ldp] * r;
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[mode] = t1 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[4];
  for (int w : {13, 64}) for (int nt : {32, 128, 256}) {
    for (int r = 0; r < 3; ++r) { k<<<1, nt>>>(w, d, 0); k<<<1, nt>>>(w, d, 1); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); }
    printf("w=%d nt=%d: syncs only %lld (%lld/step), with update %lld (%lld/step)\n", w, nt, h[0], h[0] / w, h[1], h[1] / w);
  }
}
