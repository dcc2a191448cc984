// Latency of graph building blocks on this B200 / driver (tuning aid):
//  (a) a chain of K dependent single-thread kernel nodes, replayed;
//  (b) a WHILE conditional node whose body is one single-thread kernel, K iterations;
//  (c) the same WHILE with a 3-kernel body;  (d) K cooperative 64-CTA kernels chained.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void tick(int* c) { c[0] += 1; }
__global__ void tick_cond(int* c, int K, cudaGraphConditionalHandle h) {
  c[1] += 1;
  cudaGraphSetConditional(h, c[1] < K ? 1u : 0u);
}
__global__ void reset(int* c, cudaGraphConditionalHandle h) { c[1] = 0; cudaGraphSetConditional(h, 1u); }
__global__ void coop(int* c) {
  cg::grid_group g = cg::this_grid();
  if (g.thread_rank() == 0) c[2] += 1;
  g.sync();
}

static float time_graph(cudaGraphExec_t ex, cudaStream_t st, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ex, st);
  cudaEventRecord(a, st);
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ex, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const int K = 64, reps = 50;
  int* c; CK(cudaMalloc(&c, 64)); CK(cudaMemset(c, 0, 64));
  cudaStream_t st, s2; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  // (a)
  {
    cudaGraph_t g; cudaGraphExec_t ex;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < K; ++i) tick<<<1, 1, 0, st>>>(c);
    CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ex, g, 0));
    printf("(a) chain of %d kernel nodes: %.2f us per node\n", K, 1e3f * time_graph(ex, st, reps) / K);
  }
  // (b), (c)
  for (int body = 1; body <= 3; body += 2) {
    cudaGraph_t g; cudaGraphExec_t ex;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    CK(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    reset<<<1, 1, 0, st>>>(c, h);
    cudaStreamCaptureStatus cs; cudaGraph_t cg_; const cudaGraphNode_t* deps; size_t nd;
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg_, &deps, &nd));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, cg_, deps, nd, &p));
    CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t bg = p.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s2, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < body - 1; ++i) tick<<<1, 1, 0, s2>>>(c);
    tick_cond<<<1, 1, 0, s2>>>(c, K, h);
    cudaGraph_t t; CK(cudaStreamEndCapture(s2, &t));
    CK(cudaStreamEndCapture(st, &t));
    CK(cudaGraphInstantiate(&ex, g, 0));
    printf("(%c) WHILE x %d, %d-kernel body: %.2f us per iteration\n", body == 1 ? 'b' : 'c', K, body,
           1e3f * time_graph(ex, st, reps) / K);
  }
  // (d)
  {
    cudaGraph_t g; cudaGraphExec_t ex;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < K; ++i) {
      void* args[] = {&c};
      CK(cudaLaunchCooperativeKernel((void*)coop, dim3(64), dim3(128), args, 0, st));
    }
    CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ex, g, 0));
    printf("(d) chain of %d cooperative 64x128 kernels: %.2f us per node\n", K, 1e3f * time_graph(ex, st, reps) / K);
  }
  return 0;
}
