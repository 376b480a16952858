// Probe: CUDA graph WHILE conditional node with a device-side cudaGraphSetConditional (development tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/graph_probe tools/graph_probe.cu && /tmp/graph_probe
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void setc(cudaGraphConditionalHandle h, int* cnt) {
  int c = ++(*cnt);
  cudaGraphSetConditional(h, c < 5 ? 1u : 0u);
}
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaGraphAddNode(&node, g, nullptr, 0, &p);
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  int* cnt; cudaMalloc(&cnt, 4); cudaMemset(cnt, 0, 4);
  cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  setc<<<1,1,0,s>>>(h, cnt);
  cudaGraph_t out; cudaStreamEndCapture(s, &out);
  cudaGraphExec_t ex; cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  printf("inst %d\n", (int)e);
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int h_cnt; cudaMemcpy(&h_cnt, cnt, 4, cudaMemcpyDeviceToHost);
  printf("cnt %d err %s\n", h_cnt, cudaGetErrorString(cudaGetLastError()));
}
