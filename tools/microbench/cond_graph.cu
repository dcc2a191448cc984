// Feasibility check: nested conditional graph nodes (WHILE containing IF and
// an inner WHILE), bodies filled by stream capture, a cooperative kernel
// inside a conditional body, handles set from device code.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void outer_begin(int* st, cudaGraphConditionalHandle hif, cudaGraphConditionalHandle hin) {
  st[0] += 1;  // outer iterations
  cudaGraphSetConditional(hif, (st[0] % 2) ? 1u : 0u);
  st[2] = 0;
  cudaGraphSetConditional(hin, 1u);
}
__global__ void inner_step(int* st, cudaGraphConditionalHandle hin) {
  st[2] += 1;
  st[3] += 1;  // total inner
  cudaGraphSetConditional(hin, st[2] < 3 ? 1u : 0u);
}
__global__ void coop_kernel(int* st) {
  cg::grid_group g = cg::this_grid();
  if (g.thread_rank() == 0) atomicAdd(&st[4], 1);
  g.sync();
  if (g.thread_rank() == 0) st[5] = st[4];
}
__global__ void if_body(int* st) { st[1] += 1; }
__global__ void outer_end(int* st, cudaGraphConditionalHandle hout) {
  cudaGraphSetConditional(hout, st[0] < 10 ? 1u : 0u);
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  int* st;
  CK(cudaMalloc(&st, 64));
  CK(cudaMemset(st, 0, 64));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hout;
  CK(cudaGraphConditionalHandleCreate(&hout, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = hout;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t nout;
  CK(cudaGraphAddNode(&nout, g, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaGraphConditionalHandle hif, hin;
  CK(cudaGraphConditionalHandleCreate(&hif, body, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hin, body, 0, 0));
  // body: outer_begin -> IF(hif){if_body} -> WHILE(hin){inner_step; coop} -> outer_end
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  outer_begin<<<1, 1, 0, s>>>(st, hif, hin);
  // conditional node appended to the capture
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps;
  size_t ndeps;
  cudaGraph_t cg_;
  CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg_, &deps, &ndeps));
  cudaGraphNodeParams pi = {};
  pi.type = cudaGraphNodeTypeConditional;
  pi.conditional.handle = hif;
  pi.conditional.type = cudaGraphCondTypeIf;
  pi.conditional.size = 1;
  cudaGraphNode_t nif;
  CK(cudaGraphAddNode(&nif, cg_, deps, ndeps, &pi));
  CK(cudaStreamUpdateCaptureDependencies(s, &nif, 1, cudaStreamSetCaptureDependencies));
  {
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamBeginCaptureToGraph(s2, pi.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    if_body<<<1, 1, 0, s2>>>(st);
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(s2, &tmp));
  }
  CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg_, &deps, &ndeps));
  cudaGraphNodeParams pw = {};
  pw.type = cudaGraphNodeTypeConditional;
  pw.conditional.handle = hin;
  pw.conditional.type = cudaGraphCondTypeWhile;
  pw.conditional.size = 1;
  cudaGraphNode_t nw;
  CK(cudaGraphAddNode(&nw, cg_, deps, ndeps, &pw));
  CK(cudaStreamUpdateCaptureDependencies(s, &nw, 1, cudaStreamSetCaptureDependencies));
  {
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamBeginCaptureToGraph(s2, pw.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    inner_step<<<1, 1, 0, s2>>>(st, hin);
    void* args[] = {&st};
    CK(cudaLaunchCooperativeKernel((void*)coop_kernel, 148, 256, args, 0, s2));
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(s2, &tmp));
  }
  outer_end<<<1, 1, 0, s>>>(st, hout);
  cudaGraph_t tmp;
  CK(cudaStreamEndCapture(s, &tmp));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, g, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaMemsetAsync(st, 0, 64, s));
    cudaEventRecord(e0, s);
    CK(cudaGraphLaunch(ex, s));
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    int h[8];
    CK(cudaMemcpy(h, st, 32, cudaMemcpyDeviceToHost));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("outer %d if %d inner_total %d coop %d/%d  %.3f ms (expect 10 5 30 30)\n", h[0], h[1], h[3], h[4], h[5], ms);
  }
  return 0;
}
