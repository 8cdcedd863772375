// probe: CUDA graph conditional WHILE node with a captured body
#include <cstdio>
__global__ void body(int* c, cudaGraphConditionalHandle h) {
  int v = ++c[0];
  cudaGraphSetConditional(h, v < 10 ? 1 : 0);
}
__global__ void other(int* c) { c[1] += 1; }
int main() {
  int* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  printf("handle %s\n", cudaGetErrorString(e));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t n;
  e = cudaGraphAddNode(&n, g, nullptr, 0, &p);
  printf("add %s\n", cudaGetErrorString(e));
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  printf("cap %s\n", cudaGetErrorString(e));
  other<<<1, 1, 0, s>>>(d);
  body<<<1, 1, 0, s>>>(d, h);
  e = cudaStreamEndCapture(s, &bodyg);
  printf("endcap %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex;
  e = cudaGraphInstantiate(&ex, g, 0);
  printf("inst %s\n", cudaGetErrorString(e));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) {
    cudaMemsetAsync(d, 0, 8, s);
    cudaEventRecord(a, s);
    e = cudaGraphLaunch(ex, s);
    cudaEventRecord(b, s);
    cudaStreamSynchronize(s);
    int hh[2]; cudaMemcpy(hh, d, 8, cudaMemcpyDeviceToHost);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("launch %s counter %d other %d  %.1f us (10 iterations of 2 kernels)\n", cudaGetErrorString(e), hh[0], hh[1], ms * 1e3);
  }
}
