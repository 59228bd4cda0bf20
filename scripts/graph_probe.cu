// Microbenchmark: cost of a device-side WHILE conditional iteration vs straight-line
// unrolled kernels (with and without PDL) vs IF-per-layer, for a 6-kernel "layer".
#include <cstdio>
#include <cuda_runtime.h>
__global__ void work(int* flag, int iters, cudaGraphConditionalHandle h, int set, int* ctr, int check) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (check && *(volatile int*)flag) { asm volatile("griddepcontrol.launch_dependents;"); return; }
  float x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = x * 1.0001f + 0.5f;
  if (x == 12345.f) flag[1] = 1;
  asm volatile("griddepcontrol.launch_dependents;");
  if (set && threadIdx.x == 0 && blockIdx.x == 0) {
    int c = atomicAdd(ctr, 1) + 1;
    cudaGraphSetConditional(h, c < 12 ? 1u : 0u);
  }
}
static void launch(cudaStream_t s, bool pdl, int* flag, int iters, cudaGraphConditionalHandle h, int set, int* ctr, int check) {
  cudaLaunchConfig_t cfg{}; cfg.gridDim = 148; cfg.blockDim = 128; cfg.stream = s;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, work, flag, iters, h, set, ctr, check);
}
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int *flag, *ctr; cudaMalloc(&flag, 16); cudaMalloc(&ctr, 16); cudaMemset(flag, 0, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int K = 6, iters = 2000;
  for (int variant = 0; variant < 5; ++variant) {
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h = 0;
    if (variant == 0 || variant == 1) {  // WHILE loop, body = K kernels (PDL inside body when variant==1)
      cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
      cudaGraphNodeParams cp{}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
      cudaGraphNode_t w; cudaGraphAddNode(&w, g, nullptr, 0, &cp);
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
      for (int k = 0; k < K; ++k) launch(s, variant == 1 && k > 0, flag, iters, h, k == K - 1, ctr, 0);
      cudaStreamEndCapture(s, &body);
    } else {  // unrolled 12 layers; variant 3 = PDL; variant 4 = PDL + flag check (7 of 12 layers "skipped")
      cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
      for (int l = 0; l < 12; ++l) for (int k = 0; k < K; ++k) launch(s, variant >= 3 && (l + k) > 0, flag, iters, 0, 0, ctr, variant == 4 && l >= 5);
      cudaStreamEndCapture(s, &g);
    }
    cudaGraphExec_t x; cudaError_t e = cudaGraphInstantiate(&x, g, 0);
    if (e != cudaSuccess) { printf("variant %d instantiate failed %s\n", variant, cudaGetErrorString(e)); continue; }
    if (variant == 4) cudaMemset(flag, 1, 4); else cudaMemset(flag, 0, 4);
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
      cudaMemsetAsync(ctr, 0, 4, s);
      cudaEventRecord(a, s); cudaGraphLaunch(x, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    const char* names[] = {"WHILE x12 (no PDL)", "WHILE x12 (PDL in body)", "unrolled 12x6 (no PDL)", "unrolled 12x6 (PDL)", "unrolled PDL, layers 6-12 skipped by flag"};
    printf("%-45s %8.1f us total  %6.2f us/layer\n", names[variant], best * 1e3, best * 1e3 / 12);
  }
  // reference: a single kernel's duration
  cudaEventRecord(a, s); for (int r = 0; r < 20; ++r) launch(s, false, flag, iters, 0, 0, ctr, 0); cudaEventRecord(b, s); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); printf("single kernel (stream, back to back): %.2f us\n", ms * 1e3 / 20);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
