// Development aid: SM-initiated writes into page-locked host memory over
// PCIe (the IO kernel's job-record path) vs a copy-engine D2H, and the cost of
// a system-scope fence after each warp's block of writes.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sysmem_write sysmem_write.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void wr(double* dst, size_t n_per_warp, int fence_every, int warps) {
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, L = threadIdx.x & 31;
    if (w >= (unsigned)warps) return;
    double* p = dst + (size_t)w * n_per_warp;
    for (size_t i = 0; i < n_per_warp; i += 32) {
        if (i + L < n_per_warp) p[i + L] = (double)(i + L);
        if (fence_every && ((i / 32) % fence_every) == fence_every - 1) __threadfence_system();
    }
    __threadfence_system();
}

int main() {
    const size_t bytes = 20u << 20;
    double *h, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("copy engine D2H 20 MiB: %.3f ms = %.1f GB/s\n", ms, bytes / ms / 1e6);
    }
    const int warps_list[] = {592, 4096};
    const int fences[] = {0, 20, 4, 1};
    for (int warps : warps_list)
        for (int fe : fences) {
            const size_t per = bytes / 8 / warps;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                wr<<<(warps * 32 + 127) / 128, 128>>>(h, per, fe, warps);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
            }
            printf("SM stores, %4d warps x %6zu B, fence every %2d x 256 B: %.3f ms = %.1f GB/s\n", warps, per * 8,
                   fe, ms, bytes / ms / 1e6);
        }
    // same into device memory for reference
    cudaEventRecord(a);
    wr<<<(4096 * 32 + 127) / 128, 128>>>(d, bytes / 8 / 4096, 0, 4096);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("device-memory stores: %.3f ms\n", ms);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
