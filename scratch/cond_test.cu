// micro-test: WHILE conditional graph node with a body of small kernels
#include <cstdio>
#include <cuda_runtime.h>
#include <chrono>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__global__ void k_work(int* ctr, float* buf, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) buf[t] = buf[t] * 0.5f + 1.0f;
}
__global__ void k_step(int* ctr, int iters, cudaGraphConditionalHandle h) {
  int c = ++ctr[0];
  cudaGraphSetConditional(h, c < iters ? 1 : 0);
}
int main() {
  int* ctr; float* buf; int n = 1 << 16;
  CK(cudaMalloc(&ctr, 4)); CK(cudaMalloc(&buf, n * 4));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  for (int nk : {1, 5, 10}) {
    cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // capture the body
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    for (int k = 0; k < nk; k++) k_work<<<n / 256, 256, 0, st>>>(ctr, buf, n);
    k_step<<<1, 1, 0, st>>>(ctr, 1000, h);
    CK(cudaStreamEndCapture(st, &body));
    cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge, g, 0));
    for (int rep = 0; rep < 2; rep++) {
      CK(cudaMemsetAsync(ctr, 0, 4, st));
      CK(cudaStreamSynchronize(st));
      auto t0 = std::chrono::steady_clock::now();
      CK(cudaGraphLaunch(ge, st));
      CK(cudaStreamSynchronize(st));
      double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      printf("body %d kernels + step: %.2f us per iteration\n", nk, us / 1000);
    }
    // baseline: stream launches with host loop
    auto t0 = std::chrono::steady_clock::now();
    for (int it = 0; it < 1000; it++) { for (int k = 0; k < nk; k++) k_work<<<n / 256, 256, 0, st>>>(ctr, buf, n); }
    CK(cudaStreamSynchronize(st));
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    printf("  stream launches: %.2f us per iteration (%d kernels)\n", us / 1000, nk);
    t0 = std::chrono::steady_clock::now();
    for (int it = 0; it < 300; it++) { for (int k = 0; k < nk; k++) k_work<<<n / 256, 256, 0, st>>>(ctr, buf, n); CK(cudaStreamSynchronize(st)); }
    us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    printf("  stream launches + sync each: %.2f us per iteration\n", us / 300);
  }
  return 0;
}
