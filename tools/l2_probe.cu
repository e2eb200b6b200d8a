// l2_probe.cu -- development microbenchmark (not part of the product): L2-resident
// vs HBM bandwidth on this B200, to decide whether passes fused through an
// L2-resident scratch buffer can beat separate HBM passes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe tools/l2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n, int reps) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}
__global__ void read_k(const double2 *__restrict__ a, double2 *__restrict__ sink, size_t n, int reps) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            double2 v = __ldcg(a + i);
            acc += v.x + v.y;
        }
    if (acc == 12345.678) sink[0].x = acc;
}
__global__ void write_k(double2 *__restrict__ b, size_t n, int reps) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
            b[i] = make_double2(r, i);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t big = (size_t)1 << 26;   // 1 GiB of double2
    double2 *a, *b;
    cudaMalloc(&a, big * 16);
    cudaMalloc(&b, big * 16);
    cudaMemset(a, 0, big * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    size_t sizes_mb[] = {8, 16, 32, 48, 64, 96, 1024};
    for (int g = 1; g <= 4; g *= 2)
        for (size_t mb : sizes_mb) {
            size_t n = mb * (1 << 20) / 16;
            int reps = mb >= 1024 ? 2 : (int)(2048 / mb);
            int grid = sms * 4 * g, block = 256;
            for (int kind = 0; kind < 3; ++kind) {
                for (int w = 0; w < 2; ++w) {
                    if (kind == 0) copy_k<<<grid, block>>>(a, b, n / 2, 1);
                    else if (kind == 1) read_k<<<grid, block>>>(a, b, n, 1);
                    else write_k<<<grid, block>>>(b, n, 1);
                }
                cudaEventRecord(e0);
                if (kind == 0) copy_k<<<grid, block>>>(a, b, n / 2, reps);   // footprint n (half read, half write)
                else if (kind == 1) read_k<<<grid, block>>>(a, b, n, reps);
                else write_k<<<grid, block>>>(b, n, reps);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                double bytes = (double)n * 16 * reps;
                printf("%s footprint=%4zu MB grid=%d: %.0f GB/s\n", kind == 0 ? "copy " : (kind == 1 ? "read " : "write"),
                       mb, grid, bytes / (ms * 1e-3) / 1e9);
            }
        }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
