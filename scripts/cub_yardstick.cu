// Yardstick only (never on the product path): CUB DeviceRadixSort::SortPairs on the
// frame's sort shapes, to size the headroom of the hand-written LSD sort.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cub_yardstick scripts/cub_yardstick.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

static void run(uint32_t n, int bits, const char* what) {
    std::vector<uint32_t> hk(n), hv(n);
    std::mt19937 rng(7);
    for (uint32_t i = 0; i < n; ++i) { hk[i] = rng() & ((1u << bits) - 1u); hv[i] = i; }
    uint32_t *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    cudaMemcpy(k0, hk.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, v1, n, 0, bits);
    void* tmp; cudaMalloc(&tmp, tmp_bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, n, 0, bits);
    const int reps = 20;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, n, 0, bits);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: n=%u bits=%d  %.1f us/sort  %.2f Gkeys/s\n", what, n, bits, 1000.0f * ms / reps, n / (ms / reps * 1e-3) / 1e9);
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(tmp);
}

int main() {
    run(10901796, 26, "depth keys (config 3 S)");
    run(24184701, 15, "cell keys (config 3 K)");
    run(24184701, 10, "cell keys, 10 bits");
    run(61700000, 17, "cell keys (config 4 K)");
    return 0;
}
