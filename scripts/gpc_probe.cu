// Which SMs share a GPC: clusters are co-scheduled inside one GPC, so the %smid of the CTAs of
// each cluster of 16 (non-portable size) lists SMs of one GPC.  nvcc -arch=sm_100a -o gpc_probe gpc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(1, 1, 1) dummy() {}
__global__ void probe(int* out) {
    unsigned smid, cid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %clusterid.x;" : "=r"(cid));
    if (threadIdx.x == 0) { out[blockIdx.x * 2] = smid; out[blockIdx.x * 2 + 1] = cid; }
    // keep the CTA resident a while so clusters do not reuse SMs
    long long t0 = clock64(); while (clock64() - t0 < 2000000) {}
}
int main() {
    for (int cs : {16, 8}) {
        int* d; cudaMalloc(&d, 4096 * 8);
        cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(cs * 18); cfg.blockDim = dim3(32);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d);
        cudaDeviceSynchronize();
        int h[4096 * 2]; cudaMemcpy(h, d, cs * 18 * 8, cudaMemcpyDeviceToHost);
        printf("cluster %d: %s\n", cs, cudaGetErrorString(e));
        for (int c = 0; c < 18; ++c) { printf("  cl %2d:", c); for (int i = 0; i < cs; ++i) printf(" %3d", h[(c * cs + i) * 2]); printf("\n"); }
    }
}
