// Latency of dependent fp64 / fp32 adds and of a 64-bit warp shuffle reduction on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fp64_probe scripts/fp64_probe.cu
#include <cstdio>
__global__ void k(double* out, float* outf, long long* t, int n) {
    double a = threadIdx.x * 1e-3, b = 1.0000001;
    float af = threadIdx.x * 1e-3f, bf = 1.0000001f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = a * b + 1e-9;
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) af = af * bf + 1e-9f;
    long long t2 = clock64();
    double s = a;
    for (int i = 0; i < n / 16; ++i)
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    long long t3 = clock64();
    out[threadIdx.x] = a + s;
    outf[threadIdx.x] = af;
    if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; }
}
int main() {
    double* o; float* of; long long* t;
    cudaMalloc(&o, 8 * 1024); cudaMalloc(&of, 4 * 1024); cudaMalloc(&t, 64);
    const int n = 4096;
    for (int threads : {32, 256}) {
        k<<<1, threads>>>(o, of, t, n);
        k<<<148, threads>>>(o, of, t, n);
        cudaDeviceSynchronize();
        long long h[3];
        cudaMemcpy(h, t, 24, cudaMemcpyDeviceToHost);
        printf("threads/CTA %d: DFMA chain %.1f cycles/op, FFMA chain %.1f cycles/op, fp64 warp-sum level %.1f cycles\n",
               threads, (double)h[0] / n, (double)h[1] / n, (double)h[2] / (n / 16 * 5));
    }
    return 0;
}
