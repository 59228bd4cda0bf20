// Probe: inside ONE cooperative persistent launch, how long does the activation
// broadcast of a batch-M GEMM phase take (every CTA bulk-copies the same 96 KB
// that the previous phase's epilogues just wrote with generic stores)?
// Each round: [write phase] fence.proxy.async, grid barrier, [read phase: producer
// lane bulk-copies nch chunks, times first/last completion in SM cycles], barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bcast_probe scripts/bcast_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_sync(unsigned* bar, unsigned k) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
        if (blockIdx.x == 0) {
            unsigned v;
            do asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            while (v < gridDim.x * k);
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1024), "r"(k) : "memory");
        } else {
            unsigned v;
            do asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1024) : "memory");
            while ((int)(v - k) < 0);
        }
    }
    __syncthreads();
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct Args {
    uint8_t* act;     // activation buffers (nbuf x 96 KB apart by `bstride`)
    size_t bstride;
    int nbuf;
    int rounds;
    int wmode;        // 0 none, 1 interleaved 16-feature slices (48 writer CTAs), 2 contiguous slices by all CTAs
    int nch;          // chunks per read
    uint32_t chunk;   // bytes per chunk
    uint64_t policy;  // L2 cache hint
    int readers;      // CTAs that read (others idle)
    unsigned* bar;
    long long* out;   // [rounds][cta][3]: issue->first, issue->last, smid
};

__global__ void __launch_bounds__(288, 1) kern(Args a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 16; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned k = 0;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    for (int r = 0; r < a.rounds; ++r) {
        uint8_t* act = a.act + (size_t)(r % a.nbuf) * a.bstride;
        // ---- write phase (like an epilogue writing the act layout [kb][64 rows][64 feats] bf16)
        if (a.wmode == 1 && blockIdx.x < 48 && threadIdx.x < 256) {
            // CTA u writes features 16u..16u+15 of 64 rows: kb = u/4, 32 B per row
            const int u = blockIdx.x, kb = u / 4, off = (u % 4) * 32;
            for (int i = threadIdx.x; i < 64 * 2; i += 256) {
                const int row = i >> 1, h = i & 1;
                *reinterpret_cast<uint4*>(act + (size_t)kb * 8192 + row * 128 + off + h * 16) =
                    make_uint4(r, u, row, h);
            }
        } else if (a.wmode == 2 && threadIdx.x < 256) {
            const uint32_t total = (uint32_t)a.nch * a.chunk;
            for (uint32_t i = (blockIdx.x * 256 + threadIdx.x) * 16; i < total; i += gridDim.x * 256 * 16)
                *reinterpret_cast<uint4*>(act + i) = make_uint4(r, i, 0, 0);
        }
        bar_sync(a.bar, ++k);
        // ---- read phase
        if (threadIdx.x == 256 && (int)blockIdx.x < a.readers) {
            const long long t0 = clock64();
            for (int c = 0; c < a.nch; ++c) {
                const uint32_t fb = su(&full[c]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(a.chunk) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                    "[%3], %4;" ::"r"(su(sm + (size_t)c * a.chunk)),
                    "l"(act + (size_t)c * a.chunk), "r"(a.chunk), "r"(fb), "l"(a.policy)
                    : "memory");
            }
            long long tf = 0;
            for (int c = 0; c < a.nch; ++c) {
                uint32_t ok = 0;
                while (!ok)
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                        : "=r"(ok)
                        : "r"(su(&full[c])), "r"((uint32_t)(r & 1))
                        : "memory");
                if (c == 0) tf = clock64();
            }
            const long long t1 = clock64();
            long long* o = a.out + ((size_t)r * gridDim.x + blockIdx.x) * 3;
            o[0] = tf - t0;
            o[1] = t1 - t0;
            o[2] = smid;
        }
        bar_sync(a.bar, ++k);
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* buf;
    const size_t big = 1ull << 30;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 1, big);
    unsigned* bar;
    cudaMalloc(&bar, 8192 * 4);
    const int rounds = 40;
    long long* out;
    cudaMalloc(&out, (size_t)rounds * sms * 3 * 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const uint64_t EF = 0x12F0000000000000ull, EL = 0x14F0000000000000ull, EN = 0x10F0000000000000ull;
    struct Case {
        const char* name;
        int wmode, nbuf, nch;
        uint32_t chunk;
        uint64_t pol;
        int readers;
    };
    std::vector<Case> cases = {
        {"clean 3x32KB evict_last", 0, 1, 3, 32768, EL, 148},
        {"clean 3x32KB evict_first", 0, 1, 3, 32768, EF, 148},
        {"interleaved-written 3x32KB EL", 1, 1, 3, 32768, EL, 148},
        {"interleaved-written 3x32KB EF", 1, 1, 3, 32768, EF, 148},
        {"interleaved-written 3x32KB EN", 1, 1, 3, 32768, EN, 148},
        {"interleaved 3 bufs 3x32KB EL", 1, 3, 3, 32768, EL, 148},
        {"contig-written 3x32KB EL", 2, 1, 3, 32768, EL, 148},
        {"interleaved-written 12x8KB EL", 1, 1, 12, 8192, EL, 148},
        {"interleaved-written 1x96KB EL", 1, 1, 1, 98304, EL, 148},
        {"interleaved-written 3x32KB, 74 readers", 1, 1, 3, 32768, EL, 74},
        {"interleaved-written 3x32KB, 16 readers", 1, 1, 3, 32768, EL, 16},
        {"clean 3x32KB, 16 readers", 0, 1, 3, 32768, EL, 16},
    };
    std::vector<long long> h((size_t)rounds * sms * 3);
    for (auto& c : cases) {
        cudaMemset(bar, 0, 8192 * 4);
        cudaMemset(out, 0, (size_t)rounds * sms * 3 * 8);
        Args a{buf, 1 << 20, c.nbuf, rounds, c.wmode, c.nch, c.chunk, c.pol, c.readers, bar, out};
        void* args[] = {&a};
        cudaLaunchCooperativeKernel((void*)kern, sms, 288, args, 200 * 1024, 0);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: %s\n", c.name, cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
        std::vector<double> first, last, lmax;
        for (int r = 5; r < rounds; ++r) {
            double mx = 0;
            for (int i = 0; i < c.readers; ++i) {
                const long long* o = &h[((size_t)r * sms + i) * 3];
                first.push_back(o[0] / 1.965e3);
                last.push_back(o[1] / 1.965e3);
                mx = std::max(mx, o[1] / 1.965e3);
            }
            lmax.push_back(mx);
        }
        std::sort(first.begin(), first.end());
        std::sort(last.begin(), last.end());
        std::sort(lmax.begin(), lmax.end());
        printf("%-42s first p50 %5.2f | last p50 %5.2f p90 %5.2f | per-round max p50 %5.2f us\n", c.name,
               first[first.size() / 2], last[last.size() / 2], last[last.size() * 9 / 10], lmax[lmax.size() / 2]);
    }
    return 0;
}
