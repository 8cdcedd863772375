#include <cstdio>
__device__ __forceinline__ double rsqrt_fast(double d) {
  if (!(d > 1e-30 && d < 1e30)) return 1.0 / sqrt(d);
  double r = (double)rsqrtf((float)d);
  r = r * (1.5 - 0.5 * d * r * r);
  r = r * (1.5 - 0.5 * d * r * r);
  return r;
}
__device__ __forceinline__ double rsqrt_nb(double d) {  // no range branch
  double r = (double)rsqrtf((float)d);
  r = r * (1.5 - 0.5 * d * r * r);
  r = r * (1.5 - 0.5 * d * r * r);
  return r;
}
template <int V>
__global__ void kc(double* g, long long* out) {
  __shared__ double sm[1024];
  __shared__ double dsh[64];
  __shared__ int np, mpv;
  const int lane = threadIdx.x;
  sm[lane] = 100.0 + lane;
  __syncwarp();
  double s0 = sm[lane];
  double dd = s0 + 1.0;  // force the load to complete
  long long t0 = clock64();
  double d = dd;
  if (lane == 0) {
    if (V == 0) {
      if (!(d > 0.0) || !isfinite(d)) { np = 1; atomicMin(&mpv, 0); d = nan(""); }
      dsh[0] = rsqrt_fast(d);
    } else if (V == 1) {
      dsh[0] = rsqrt_fast(d);
    } else if (V == 2) {
      dsh[0] = rsqrt_nb(d);
    } else if (V == 3) {
      if (!(d > 0.0)) { np = 1; d = __longlong_as_double(0x7ff8000000000000ll); }
      dsh[0] = rsqrt_nb(d);
    } else if (V == 4) {
      dsh[0] = 1.0 / sqrt(d);
    } else {
      dsh[0] = d;
    }
  }
  __syncwarp();
  double rp = dsh[0];
  long long t1 = clock64();
  g[lane] = rp;
  if (lane == 0) out[V] = t1 - t0;
}
int main() {
  long long* d; double* g; cudaMalloc(&d, 64); cudaMalloc(&g, 1024);
  long long h[6];
  for (int r = 0; r < 3; ++r) {
    kc<0><<<1, 32>>>(g, d); kc<1><<<1, 32>>>(g, d); kc<2><<<1, 32>>>(g, d); kc<3><<<1, 32>>>(g, d); kc<4><<<1, 32>>>(g, d); kc<5><<<1, 32>>>(g, d);
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
  }
  printf("full %lld | rsqrt_fast only %lld | rsqrt no range %lld | simple check + rsqrt_nb %lld | 1/sqrt %lld | none %lld\n", h[0], h[1], h[2], h[3], h[4], h[5]);
}
