// Is the per-SM bulk-copy serialisation per issuing thread, per CTA or per SM?
// W issuing warps per CTA (own ring of S stages each), or several CTAs per SM.
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void ingest_w(const uint8_t* src, uint32_t chunk, int per_w, int n_chunks, int S, unsigned long long* sink, int tensor) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[64];
    const int W = blockDim.x / 32, w = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S * W; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if ((threadIdx.x & 31) != 0) return;
    uint8_t* ring = sm + (size_t)w * S * chunk;
    uint64_t* fb = full + w * S;
    unsigned long long acc = 0;
    const size_t base = ((size_t)blockIdx.x * W + w) * per_w;
    for (int i = 0; i < per_w + S; ++i) {
        if (i >= S) {
            const int s = (i - S) % S;
            const uint32_t ph = ((i - S) / S) & 1;
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok) : "r"(su(&fb[s])), "r"(ph) : "memory");
            acc += ring[(size_t)s * chunk];
        }
        if (i < per_w) {
            const int s = i % S;
            const size_t c = (base + i) % (size_t)n_chunks;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&fb[s])), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su(ring + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(su(&fb[s])) : "memory");
        }
    }
    if (acc == 12345) *sink = acc;
}
int main() {
    const size_t bytes = 1ull << 30;
    uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
    uint8_t* flush; cudaMalloc(&flush, 256u << 20);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(ingest_w, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int src = 0; src < 2; ++src)
        for (uint32_t chunk : {16384u, 32768u, 65536u})
            for (int W : {1, 2, 3, 4, 6})
                for (int cps : {1, 2}) {  // CTAs per SM
                    const int S = 2;
                    if ((size_t)chunk * S * W * cps > 200 * 1024) continue;
                    for (int sms : {8, 148}) {
                        const int G = sms * cps;
                        const size_t region = src ? (16u << 20) : bytes;
                        const int n_chunks = (int)(region / chunk);
                        const int per_w = (int)std::max<size_t>(16, std::min<size_t>((src ? 48u << 20 : 6u << 20) / chunk / (W * cps), 4096));
                        float best = 1e9f;
                        for (int r = 0; r < 3; ++r) {
                            if (!src) cudaMemsetAsync(flush, r, 256u << 20);
                            else ingest_w<<<148, 32, (size_t)chunk * S>>>(buf, chunk, n_chunks / 148, n_chunks, S, sink, 0);
                            cudaEventRecord(a);
                            ingest_w<<<G, 32 * W, (size_t)chunk * S * W>>>(buf, chunk, per_w, n_chunks, S, sink, 0);
                            cudaEventRecord(b);
                            cudaEventSynchronize(b);
                            float ms; cudaEventElapsedTime(&ms, a, b);
                            best = std::min(best, ms);
                        }
                        const double gbs = (double)G * W * per_w * chunk / (best * 1e-3) / 1e9;
                        printf("%s chunk %3u KB  S=2  issuing warps %d  ctas/SM %d  SMs %3d : %7.0f GB/s total %6.1f GB/s per SM\n",
                               src ? "L2 " : "HBM", chunk / 1024, W, cps, sms, gbs, gbs / sms);
                    }
                }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
