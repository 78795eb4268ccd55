// PCIe write paths for the result rows (dev microbenchmark): bulk cudaMemcpy D2H versus
// kernel stores of 384-byte rows (32 u32 ids + 32 f64 dists) into mapped pinned host
// memory, in row order, in a random row order, and in random order sorted per chunk.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void rows_out(const uint32_t* order, uint64_t nrows, uint32_t* hid, double* hd) {
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nrows) return;
    const uint64_t r = order ? order[w] : w;
    hid[r * 32 + lane] = (uint32_t)r + lane;
    hd[r * 32 + lane] = (double)r;
}

int main() {
    const uint64_t N = 1ull << 25;  // 33.5M rows = 12.9 GB
    uint32_t *hid, *dord;
    double* hd;
    cudaHostAlloc(&hid, N * 128, cudaHostAllocMapped);
    cudaHostAlloc(&hd, N * 256, cudaHostAllocMapped);
    cudaMalloc(&dord, N * 4);
    void* dbuf;
    cudaMalloc(&dbuf, N * 384);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    auto gbs = [&](double bytes) { return bytes / (ms * 1e-3) / 1e9; };
    for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        cudaMemcpyAsync(hid, dbuf, N * 128, cudaMemcpyDeviceToHost);
        cudaMemcpyAsync(hd, (char*)dbuf + N * 128, N * 256, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("memcpy D2H          %8.1f ms  %6.1f GB/s\n", ms, gbs(N * 384.0));
    }
    std::vector<uint32_t> ord(N);
    for (uint64_t i = 0; i < N; ++i) ord[i] = (uint32_t)i;
    std::mt19937_64 g(1);
    std::shuffle(ord.begin(), ord.end(), g);
    const char* names[] = {"kernel rows, in order", "kernel rows, random", "kernel rows, 8 sorted chunks"};
    for (int mode = 0; mode < 3; ++mode) {
        std::vector<uint32_t> o = ord;
        if (mode == 2)
            for (int c = 0; c < 8; ++c) std::sort(o.begin() + c * (N / 8), o.begin() + (c + 1) * (N / 8));
        cudaMemcpy(dord, o.data(), N * 4, cudaMemcpyHostToDevice);
        for (int it = 0; it < 2; ++it) {
            cudaEventRecord(a);
            rows_out<<<(unsigned)(N * 32 / 256), 256>>>(mode ? dord : nullptr, N, hid, hd);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("%-28s %8.1f ms  %6.1f GB/s\n", names[mode], ms, gbs(N * 384.0));
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
