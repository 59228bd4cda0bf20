// Single-issuer bulk-copy throughput vs the mbarrier wait flavour, and lanes vs warps as issuers.
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>  // 0 try_wait, 1 test_wait spin, 2 try_wait hint 20 ns, 3 try_wait hint 1000ns
__device__ __forceinline__ void wait(uint32_t a, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok) {
        if (MODE == 0)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
        else if (MODE == 1)
            asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
        else if (MODE == 2)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 20; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
        else
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
    }
}
// issuers = lanes 0..I-1 of warp 0 (lanes mode) or lane 0 of warps 0..I-1
template <int MODE>
__global__ void ingest(const uint8_t* src, uint32_t chunk, int per_w, int n_chunks, int S, int I, int lanes, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[64];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S * I; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    int w;
    if (lanes) { if (threadIdx.x >= (unsigned)I) return; w = threadIdx.x; }
    else { if ((threadIdx.x & 31) != 0 || threadIdx.x / 32 >= (unsigned)I) return; w = threadIdx.x / 32; }
    uint8_t* ring = sm + (size_t)w * S * chunk;
    uint64_t* fb = full + w * S;
    unsigned long long acc = 0;
    const size_t base = ((size_t)blockIdx.x * I + w) * per_w;
    for (int i = 0; i < per_w + S; ++i) {
        if (i >= S) {
            const int s = (i - S) % S;
            wait<MODE>(su(&fb[s]), ((i - S) / S) & 1);
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
typedef void (*K)(const uint8_t*, uint32_t, int, int, int, int, int, unsigned long long*);
int main() {
    const size_t bytes = 1ull << 30;
    uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
    uint8_t* flush; cudaMalloc(&flush, 256u << 20);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    K ks[4] = {ingest<0>, ingest<1>, ingest<2>, ingest<3>};
    const char* names[4] = {"try_wait", "test_wait", "try_wait(20ns)", "try_wait(1us)"};
    for (int m = 0; m < 4; ++m) cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    struct C { int src; uint32_t chunk; int S, I, lanes; };
    const C cs[] = {{1, 32768, 2, 1, 0}, {1, 32768, 4, 1, 0}, {1, 16384, 6, 1, 0}, {1, 32768, 2, 3, 1}, {1, 16384, 2, 6, 1},
                    {0, 32768, 2, 1, 0}, {0, 32768, 4, 1, 0}, {0, 16384, 8, 1, 0}, {0, 16384, 2, 6, 1}, {0, 32768, 2, 3, 1}};
    for (const C& c : cs)
        for (int m = 0; m < 4; ++m)
            for (int sms : {8, 148}) {
                const size_t region = c.src ? (16u << 20) : bytes;
                const int n_chunks = (int)(region / c.chunk);
                const int per_w = (int)std::max<size_t>(16, std::min<size_t>((c.src ? 48u << 20 : 6u << 20) / c.chunk / c.I, 4096));
                const int threads = c.lanes ? 32 : 32 * c.I;
                float best = 1e9f;
                for (int r = 0; r < 3; ++r) {
                    if (!c.src) cudaMemsetAsync(flush, r, 256u << 20);
                    else ks[0]<<<148, 32, (size_t)c.chunk * 2>>>(buf, c.chunk, n_chunks / 148, n_chunks, 2, 1, 0, sink);
                    cudaEventRecord(a);
                    ks[m]<<<sms, threads, (size_t)c.chunk * c.S * c.I>>>(buf, c.chunk, per_w, n_chunks, c.S, c.I, c.lanes, sink);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms; cudaEventElapsedTime(&ms, a, b);
                    best = std::min(best, ms);
                }
                const double gbs = (double)sms * c.I * per_w * c.chunk / (best * 1e-3) / 1e9;
                printf("%s chunk %2u KB S=%d issuers %d (%s) %-15s SMs %3d : %7.0f GB/s total %6.1f per SM\n", c.src ? "L2 " : "HBM",
                       c.chunk / 1024, c.S, c.I, c.lanes ? "lanes" : "warps", names[m], sms, gbs, gbs / sms);
            }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
