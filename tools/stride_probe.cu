// stride_probe.cu -- development microbenchmark (not part of the product): DRAM
// efficiency of the access patterns a two-pass <F1, F2> lifting needs at 2^24.
// View the n-vector as [F rows][B cols]; a tile is T adjacent columns x F rows.
//   mode 0: read the tile (runs of T*16 B, rows B*16 B apart), write it back at the
//           same positions of another buffer (the column pass)
//   mode 1: read the tile strided, write it contiguously (read side alone)
//   mode 2: read contiguously, write the tile strided (write side alone, the
//           transposed store of the row pass)
//   order 0: block b -> tile b (co-running CTAs touch adjacent columns)
//   order 1: block b -> tile (b * 1021) mod tiles (scattered)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stride_probe tools/stride_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int EPT>
__global__ void __launch_bounds__(256) tile_copy(const double2 *__restrict__ in, double2 *__restrict__ out, int logT,
                                                 int logF, int logB, int mode, int order, int tiles) {
    const int T = 1 << logT;
    int tile = blockIdx.x;
    if (order) tile = (int)(((long long)tile * 1021) % tiles);
    const long long c0 = (long long)tile * T;
    const int nel = T << logF;
    double2 v[EPT];
    for (int base = 0; base < nel; base += 256 * EPT) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            int e = base + threadIdx.x + i * 256;
            long long row = e >> logT, col = e & (T - 1);
            long long strided = (row << logB) + c0 + col;
            long long contig = ((long long)tile * nel) + e;
            if (e < nel) v[i] = __ldg(in + (mode == 2 ? contig : strided));
        }
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            int e = base + threadIdx.x + i * 256;
            long long row = e >> logT, col = e & (T - 1);
            long long strided = (row << logB) + c0 + col;
            long long contig = ((long long)tile * nel) + e;
            if (e < nel) out[mode == 1 ? contig : strided] = v[i];
        }
    }
}

int main(int argc, char **argv) {
    const int logn = argc > 1 ? atoi(argv[1]) : 24;
    const size_t n = (size_t)1 << logn;
    double2 *a, *b;
    cudaMalloc(&a, n * 16);
    cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    cudaMemset(b, 0, n * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int logFs[] = {8, 12};
    for (int logF : logFs) {
        const int logB = logn - logF;
        for (int mode = 0; mode < 3; ++mode)
            for (int order = 0; order < 2; ++order)
                for (int logT = 0; logT <= 4; ++logT) {
                    const int tiles = 1 << (logB - logT);
                    for (int w = 0; w < 2; ++w) tile_copy<16><<<tiles, 256>>>(a, b, logT, logF, logB, mode, order, tiles);
                    const int reps = 5;
                    cudaEventRecord(e0);
                    for (int r = 0; r < reps; ++r)
                        tile_copy<16><<<tiles, 256>>>(a, b, logT, logF, logB, mode, order, tiles);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    double us = ms * 1e3 / reps;
                    printf("F=2^%d B=2^%d mode=%d order=%d T=%2d run=%4dB  %8.1f us  %7.1f GB/s\n", logF, logB, mode, order,
                           1 << logT, 16 << logT, us, 32.0 * n / (us * 1e-6) / 1e9);
                }
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
