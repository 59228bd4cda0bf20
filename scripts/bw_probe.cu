// Microbenchmark: achievable HBM read bandwidth for 1-D bulk TMA streaming vs
// vectorised LDG, to size the attention kernel's pipeline. nvcc -arch=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void bulk_stream(const uint8_t* src, size_t chunk, int n_chunks, int S, unsigned long long* sink,
                            int scatter = 0, int contiguous = 0) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[16];
  const int tid = threadIdx.x;
  if (tid == 0) { for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  // chunks assigned round-robin: CTA i takes chunks i, i+G, ...
  int mine = 0; for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) ++mine;
  unsigned long long acc = 0;
  if (tid == 0) {
    for (int i = 0; i < mine + S; ++i) {
      if (i >= S) { // wait for chunk i-S
        const int s = (i - S) % S; const uint32_t ph = ((i - S) / S) & 1;
        uint32_t ok = 0; while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(su(&full[s])), "r"(ph) : "memory");
        acc += sm[(size_t)s * chunk];
      }
      if (i < mine) {
        const int s = i % S;
        size_t c = contiguous ? (size_t)blockIdx.x * mine + i : blockIdx.x + (size_t)i * gridDim.x;
        if (scatter) c = (c * 2654435761ull) % (size_t)n_chunks;  // scattered blocks (like a paged KV pool)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[s])), "r"((uint32_t)chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su(sm + (size_t)s * chunk)), "l"(src + c * chunk), "r"((uint32_t)chunk), "r"(su(&full[s])) : "memory");
      }
    }
    if (acc == 12345) *sink = acc;
  }
}
__global__ void ldg_stream(const uint4* src, size_t n, unsigned long long* sink) {
  uint32_t x = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x * 4) {
    uint4 a = __ldcs(src + i), b = (i + (size_t)gridDim.x * blockDim.x < n) ? __ldcs(src + i + (size_t)gridDim.x * blockDim.x) : make_uint4(0,0,0,0);
    uint4 c = (i + 2*(size_t)gridDim.x * blockDim.x < n) ? __ldcs(src + i + 2*(size_t)gridDim.x * blockDim.x) : make_uint4(0,0,0,0);
    uint4 d = (i + 3*(size_t)gridDim.x * blockDim.x < n) ? __ldcs(src + i + 3*(size_t)gridDim.x * blockDim.x) : make_uint4(0,0,0,0);
    x ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (x == 0xdeadbeef) *sink = x;
}
int main() {
  const size_t bytes = 1ull << 30;  // 1 GiB
  uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (size_t chunk : {16384ul, 24576ul, 49152ul}) for (int S : {2, 3, 4, 6, 8}) for (int per : {1, 2}) {
    if (chunk * S > 200 * 1024 / per) continue;
    const int n_chunks = (int)(bytes / chunk);
    const int grid = sms * per;
    bulk_stream<<<grid, 32, chunk * S>>>(buf, chunk, n_chunks, S, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) bulk_stream<<<grid, 32, chunk * S>>>(buf, chunk, n_chunks, S, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("bulk chunk=%6zu S=%d ctas/sm=%d : %.0f GB/s\n", chunk, S, per, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  // short bursts over a C2-attention-sized working set (~108 MB): fill/tail effects, scattered blocks
  for (int scat : {0, 1}) for (int contig : {0, 1}) for (int S : {3, 4}) {
    const size_t chunk = 24576; const int n_chunks = (int)(108ull * 1000 * 1000 / chunk);
    cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    bulk_stream<<<sms, 32, chunk * S>>>(buf, chunk, n_chunks, S, sink, scat, contig);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) bulk_stream<<<sms, 32, chunk * S>>>(buf + (r % 4) * (256ull << 20), chunk, n_chunks, S, sink, scat, contig);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("short 108MB scatter=%d contiguous-per-cta=%d S=%d : %.1f us/launch, %.0f GB/s\n", scat, contig, S, ms * 1e3 / 20,
           20.0 * n_chunks * chunk / (ms * 1e-3) / 1e9);
  }
  for (int tpb : {256, 512, 1024}) for (int bps : {1, 2, 4}) {
    const int grid = sms * bps;
    ldg_stream<<<grid, tpb>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) ldg_stream<<<grid, tpb>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ldg tpb=%d blocks/sm=%d : %.0f GB/s\n", tpb, bps, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
