// nested WHILE: inner body kernel sets both the inner and the outer handle
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__global__ void k_outer_begin(int* c, cudaGraphConditionalHandle hin) { c[1] = 0; cudaGraphSetConditional(hin, 1); }
__global__ void k_inner(int* c, cudaGraphConditionalHandle hin, cudaGraphConditionalHandle hout) {
  c[1]++; c[2]++;
  cudaGraphSetConditional(hin, c[1] < 3 ? 1 : 0);
  if (c[1] >= 3) { c[0]++; cudaGraphSetConditional(hout, c[0] < 4 ? 1 : 0); }
}
__global__ void k_begin(int* c, cudaGraphConditionalHandle hout) { c[0] = 0; c[2] = 0; cudaGraphSetConditional(hout, 1); }
int main() {
  int* c; CK(cudaMalloc(&c, 16)); CK(cudaMemset(c, 0, 16));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hout, hin;
  CK(cudaGraphConditionalHandleCreate(&hout, g, 0, 0));
  // begin kernel
  CK(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_begin<<<1, 1, 0, st>>>(c, hout);
  cudaStreamCaptureStatus cs; const cudaGraphNode_t* deps; size_t nd; cudaGraph_t cg;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
  std::vector<cudaGraphNode_t> d(deps, deps + nd);
  CK(cudaStreamEndCapture(st, &g));
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = hout;
  cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t wout; CK(cudaGraphAddNode(&wout, g, d.data(), d.size(), &cp));
  cudaGraph_t bout = cp.conditional.phGraph_out[0];
  CK(cudaGraphConditionalHandleCreate(&hin, bout, 0, 0));
  CK(cudaStreamBeginCaptureToGraph(st, bout, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_outer_begin<<<1, 1, 0, st>>>(c, hin);
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
  d.assign(deps, deps + nd);
  CK(cudaStreamEndCapture(st, &bout));
  cudaGraphNodeParams ci = {}; ci.type = cudaGraphNodeTypeConditional; ci.conditional.handle = hin;
  ci.conditional.type = cudaGraphCondTypeWhile; ci.conditional.size = 1;
  cudaGraphNode_t win; CK(cudaGraphAddNode(&win, bout, d.data(), d.size(), &ci));
  cudaGraph_t bin = ci.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(st, bin, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_inner<<<1, 1, 0, st>>>(c, hin, hout);
  CK(cudaStreamEndCapture(st, &bin));
  cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge, g, 0));
  for (int r = 0; r < 2; r++) {
    CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
    int h[4]; CK(cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost));
    printf("outer iterations %d, inner total %d (expect 4, 12)\n", h[0], h[2]);
  }
  return 0;
}
