// Microbenchmark: FP64 DFMA and DMMA (mma.sync m8n8k4 f64) peak throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void dfma_kernel(double* out, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = fma(acc[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_kernel(double* out, double a0, double b0) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = threadIdx.x; c[i][1] = i; }
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) for (int bps : {1, 2, 4}) {
    int grid = sms * bps;
    dfma_kernel<<<grid, threads>>>(d, 0.999, 1e-3); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) dfma_kernel<<<grid, threads>>>(d, 0.999, 1e-3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 5.0 * grid * threads * (double)ITERS * 8 * 2;
    printf("DFMA threads=%d grid=%d : %.2f TFLOP/s\n", threads, grid, fl / (ms * 1e-3) / 1e12);
    dmma_kernel<<<grid, threads>>>(d, 0.999, 1e-3); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) dmma_kernel<<<grid, threads>>>(d, 0.999, 1e-3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fm = 5.0 * grid * (threads / 32) * (double)ITERS * 8 * 512;
    printf("DMMA threads=%d grid=%d : %.2f TFLOP/s\n", threads, grid, fm / (ms * 1e-3) / 1e12);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
