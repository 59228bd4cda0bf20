// Probe: latency/throughput of per-CTA 1-D bulk copies when every CTA reads the
// SAME small matrix (the activation broadcast of a batch-M GEMM) vs distinct
// L2-resident regions vs distinct HBM regions.  nvcc -arch=sm_100a -o l2_probe l2_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// two copies per stage (activation chunk + weight piece) into a 10 KB-stride ring, like a batch-M
// GEMM unit; `spin` extra warps poll an mbarrier meanwhile (like waiting epilogue warps)
__global__ void probe2(const uint8_t* act, const uint8_t* wt, int nk, int spin, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[32];
    __shared__ uint64_t done;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nk; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&done)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint8_t* w = wt + (size_t)blockIdx.x * 2048;
        const unsigned long long t0 = gt();
        for (int s = 0; s < nk; ++s) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(10240)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su(sm + (size_t)s * 10240)),
                "l"(act + (size_t)s * 8192), "r"(8192), "r"(su(&full[s]))
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su(sm + (size_t)s * 10240 + 8192)),
                "l"(w + (size_t)s * 16384 * 16), "r"(2048), "r"(su(&full[s]))
                : "memory");
        }
        unsigned long long tf = 0;
        for (int s = 0; s < nk; ++s) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                    : "=r"(ok)
                    : "r"(su(&full[s])), "r"(0)
                    : "memory");
            if (s == 0) tf = gt();
        }
        const unsigned long long t1 = gt();
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&done)) : "memory");
        out[blockIdx.x * 4 + 0] = t0;
        out[blockIdx.x * 4 + 1] = tf;
        out[blockIdx.x * 4 + 2] = t1;
    } else if (spin && threadIdx.x >= 32) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(ok)
                         : "r"(su(&done)), "r"(0)
                         : "memory");
    }
}

// mode 0: all CTAs read src[0 .. nk*chunk); mode 1: CTA c reads src[c*stride ...]
__global__ void probe(const uint8_t* src, size_t stride, int mode, int nk, uint32_t chunk, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[32];
    if (threadIdx.x == 0) {
        for (int s = 0; s < nk; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint8_t* base = src + (mode ? (size_t)blockIdx.x * stride : 0);
        const unsigned long long t0 = gt();
        for (int s = 0; s < nk; ++s) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(chunk)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su(sm + (size_t)s * chunk)),
                "l"(base + (size_t)s * chunk), "r"(chunk), "r"(su(&full[s]))
                : "memory");
        }
        unsigned long long tf = 0;
        for (int s = 0; s < nk; ++s) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                    : "=r"(ok)
                    : "r"(su(&full[s])), "r"(0)
                    : "memory");
            if (s == 0) tf = gt();
        }
        const unsigned long long t1 = gt();
        out[blockIdx.x * 4 + 0] = t0;
        out[blockIdx.x * 4 + 1] = tf;
        out[blockIdx.x * 4 + 2] = t1;
    }
}

// every CTA writes a slice of the buffer with generic stores (like an epilogue producing activations)
__global__ void writer(uint8_t* buf, size_t bytes, int val) {
    for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)gridDim.x * blockDim.x * 16)
        *reinterpret_cast<uint4*>(buf + i) = make_uint4(val, val, val, val);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t big = 2ull << 30;
    uint8_t* buf;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 1, big);
    unsigned long long* out;
    cudaMalloc(&out, sms * 4 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Case {
        const char* name;
        int mode;
        size_t stride;
        int nk;
        uint32_t chunk;
        bool warm;
    };
    std::vector<Case> cases = {
        {"same 12x8KB (L2)", 0, 0, 12, 8192, true},
        {"distinct 12x8KB (L2)", 1, 96 * 1024, 12, 8192, true},
        {"distinct 12x8KB (HBM)", 1, 12 << 20, 12, 8192, false},
        {"distinct 12x2KB (HBM)", 1, 12 << 20, 12, 2048, false},
        {"distinct 12x16KB (HBM)", 1, 12 << 20, 12, 16384, false},
        {"same 12x16KB (L2)", 0, 0, 12, 16384, true},
        {"distinct 1x16KB (HBM)", 1, 12 << 20, 1, 16384, false},
        {"distinct 1x2KB (HBM)", 1, 12 << 20, 1, 2048, false},
        {"same 1x8KB (L2)", 0, 0, 1, 8192, true},
    };
    std::vector<unsigned long long> h(sms * 4);
    for (auto& c : cases) {
        for (int rep = 0; rep < 3; ++rep) {
            if (!c.warm) cudaMemset(buf + ((size_t)1 << 30), rep, (size_t)1 << 30);  // evict L2
            else probe<<<sms, 128, 200 * 1024>>>(buf, c.stride, c.mode, c.nk, c.chunk, out);  // warm L2
            probe<<<sms, 128, 200 * 1024>>>(buf + (c.warm ? 0 : ((size_t)rep << 20)), c.stride, c.mode, c.nk, c.chunk,
                                            out);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(h.data(), out, sms * 4 * 8, cudaMemcpyDeviceToHost);
        std::vector<double> first, all;
        unsigned long long t0 = ~0ull, t1 = 0;
        for (int i = 0; i < sms; ++i) {
            first.push_back((h[i * 4 + 1] - h[i * 4]) / 1e3);
            all.push_back((h[i * 4 + 2] - h[i * 4]) / 1e3);
            t0 = std::min(t0, h[i * 4]);
            t1 = std::max(t1, h[i * 4 + 2]);
        }
        std::sort(first.begin(), first.end());
        std::sort(all.begin(), all.end());
        const double bytes = (double)sms * c.nk * c.chunk;
        printf("%-26s first p50 %6.2f us | all p50 %6.2f max %6.2f us | span %6.2f us  %7.1f GB/s agg\n", c.name,
               first[sms / 2], all[sms / 2], all.back(), (t1 - t0) / 1e3, bytes / ((t1 - t0) / 1e3) / 1e3);
    }
    cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int spin : {0, 1, 2, 3}) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(buf + ((size_t)1 << 30), rep, (size_t)1 << 30);
            probe<<<sms, 128, 200 * 1024>>>(buf, 0, 0, 12, 8192, out);  // act chunk warm in L2
            const uint8_t* a0 = buf;
            const uint8_t* w0 = buf + (256 << 20) + ((size_t)rep << 22);
            int nk = 12, sp = spin & 1;
            unsigned long long* o = out;
            if (spin >= 2) {  // cooperative launch, 220 KB smem, like the persistent kernel
                void* args[] = {(void*)&a0, (void*)&w0, (void*)&nk, (void*)&sp, (void*)&o};
                cudaLaunchCooperativeKernel((void*)probe2, sms, 288, args, 220 * 1024, 0);
            } else {
                probe2<<<sms, 288, 200 * 1024>>>(a0, w0, nk, sp, o);
            }
            cudaDeviceSynchronize();
        }
        cudaMemcpy(h.data(), out, sms * 4 * 8, cudaMemcpyDeviceToHost);
        std::vector<double> first, all;
        for (int i = 0; i < sms; ++i) {
            first.push_back((h[i * 4 + 1] - h[i * 4]) / 1e3);
            all.push_back((h[i * 4 + 2] - h[i * 4]) / 1e3);
        }
        std::sort(first.begin(), first.end());
        std::sort(all.begin(), all.end());
        printf("batch-M pattern 12x(8KB L2 + 2KB HBM) spin=%d coop=%d: first p50 %.2f | all p50 %.2f max %.2f us\n", spin & 1, spin >> 1,
               first[sms / 2], all[sms / 2], all.back());
    }
    // freshly written vs clean: 3 x 32 KB same-address copies per CTA
    for (int fresh : {0, 1, 0, 1}) {
        if (fresh) writer<<<sms, 256>>>(buf, 96 * 1024, 7);
        probe<<<sms, 128, 200 * 1024>>>(buf, 0, 0, 3, 32768, out);
        cudaDeviceSynchronize();
        cudaMemcpy(h.data(), out, sms * 4 * 8, cudaMemcpyDeviceToHost);
        std::vector<double> all;
        for (int i = 0; i < sms; ++i) all.push_back((h[i * 4 + 2] - h[i * 4]) / 1e3);
        std::sort(all.begin(), all.end());
        printf("same 3x32KB (L2) %s: all p50 %.2f max %.2f us\n", fresh ? "FRESHLY WRITTEN" : "clean", all[sms / 2], all.back());
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
