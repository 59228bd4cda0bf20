// Per-SM ingest bandwidth of 1-D bulk copies (no consumer work): how many bytes/s can ONE CTA
// pull from HBM or from L2, as a function of the CTAs streaming at once and the bytes in flight?
// Sizes the attention ring and the GEMM CTAs' operand traffic.  nvcc -arch=sm_100a -O3
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// CTA i streams `per_cta` chunks of `chunk` bytes starting at chunk (i * per_cta) mod n_chunks
__global__ void ingest(const uint8_t* src, uint32_t chunk, int per_cta, int n_chunks, int S, unsigned long long* sink, int k = 1) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned long long acc = 0;
    for (int i = 0; i < per_cta + S; ++i) {
        if (i >= S) {
            const int s = (i - S) % S;
            const uint32_t ph = ((i - S) / S) & 1;
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok) : "r"(su(&full[s])), "r"(ph) : "memory");
            acc += sm[(size_t)s * chunk];
        }
        if (i < per_cta) {
            const int s = i % S;
            const size_t c = ((size_t)blockIdx.x * per_cta + i) % (size_t)n_chunks;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(chunk) : "memory");
            const uint32_t part = chunk / k;
            for (int j = 0; j < k; ++j)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 su(sm + (size_t)s * chunk + j * part)),
                             "l"(src + c * chunk + j * part), "r"(part), "r"(su(&full[s]))
                             : "memory");
        }
    }
    if (acc == 12345) *sink = acc;
}
int main() {
    const size_t bytes = 1ull << 30;
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    uint8_t* flush;
    cudaMalloc(&flush, 256u << 20);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int src = 0; src < 2; ++src)
        for (uint32_t chunk : {32768u, 65536u, 98304u})
            for (int k : {1, 2, 4, 8})
                for (int S : {2, 3}) {
                    if ((size_t)chunk * S > 200 * 1024) continue;
                    for (int G : {8, 74, 148}) {
                        const size_t region = src ? (16u << 20) : bytes;
                        const int n_chunks = (int)(region / chunk);
                        const int per_cta = (int)std::min<size_t>((src ? 64u << 20 : 6u << 20) / chunk, 4096);
                        float best = 1e9f;
                        for (int r = 0; r < 3; ++r) {
                            if (!src) cudaMemsetAsync(flush, r, 256u << 20);
                            else ingest<<<148, 32, (size_t)chunk * S>>>(buf, chunk, n_chunks / 148, n_chunks, S, sink, 1);
                            cudaEventRecord(a);
                            ingest<<<G, 32, (size_t)chunk * S>>>(buf, chunk, per_cta, n_chunks, S, sink, k);
                            cudaEventRecord(b);
                            cudaEventSynchronize(b);
                            float ms;
                            cudaEventElapsedTime(&ms, a, b);
                            best = ms < best ? ms : best;
                        }
                        const double gbs = (double)G * per_cta * chunk / (best * 1e-3) / 1e9;
                        printf("%s stage %3u KB as %d copies x %d stages  ctas %3d : %7.0f GB/s total %6.1f GB/s per CTA\n",
                               src ? "L2 " : "HBM", chunk / 1024, k, S, G, gbs, gbs / G);
                    }
                }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
