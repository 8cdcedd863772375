// latency probes: dependent DFMA chain, dependent LDS chain, __syncwarp, smem store->load
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sm[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double a = out[0], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < n; ++i) p = idx[p];
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) __syncwarp();
  long long t3 = clock64();
  double s = 0;
  for (int i = 0; i < n; ++i) { sm[(threadIdx.x + i) & 1023] = s + 1.0; s = sm[(threadIdx.x + i) & 1023]; }
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) { a = sqrt(a + 1.0); }
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) { a = 1.0 / (a + 1.0); }
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    out[1] = a + p + s;
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n; cyc[5] = (t6 - t5) / n;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 16); cudaMalloc(&c, 64); cudaMemset(o, 0, 16);
  k<<<1, 32>>>(o, c, 1000); long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("DFMA dep %lld cyc, LDS dep %lld, syncwarp %lld, STS->LDS %lld, sqrt %lld, div %lld\n", h[0], h[1], h[2], h[3], h[4], h[5]);
}
