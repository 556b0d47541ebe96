// sort_bench.cu -- cycle timing of the block-level selection primitives (tooling only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sort_bench tools/sort_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "../paper_2505_17074_b200/csrc/select_core.cuh"

using namespace lapssd;

__global__ void __launch_bounds__(1024) bench(const uint64_t *in, uint64_t *out, int n, int B, long long *cyc, int mode) {
    extern __shared__ uint64_t sm[];
    uint64_t *a = sm, *b = sm + n, *c = sm + 2 * n;
    for (int rep = 0; rep < 3; ++rep) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = in[i];
        __syncthreads();
        long long t0 = clock64();
        const uint64_t *r;
        if (mode == 0) {
            r = block_sort(a, b, n);
        } else if (mode == 2) {
            block_sort_reg(a, n);
            r = a;
        } else {
            int bp = 1;
            while (bp < B) bp <<= 1;
            r = select_topB(a, n, B, b, c, bp);
        }
        __syncthreads();
        long long t1 = clock64();
        if (threadIdx.x == 0) cyc[rep] = t1 - t0;
        for (int i = threadIdx.x; i < (mode == 0 ? n : B); i += blockDim.x) out[i] = r[i];
        __syncthreads();
    }
}

__global__ void warp_only(const uint64_t *in, uint64_t *out, long long *cyc) {
    const int lane = threadIdx.x & 31;
    uint64_t lo = in[lane], hi = in[32 + lane];
    long long t0 = clock64();
    warp_sort64(lo, hi, lane);
    long long t1 = clock64();
    out[lane] = lo; out[32 + lane] = hi;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    const int N = 2048;
    std::vector<uint64_t> h(N);
    srand(1);
    for (int i = 0; i < N; ++i) h[i] = ((uint64_t)rand() << 40) ^ ((uint64_t)rand() << 20) ^ (uint64_t)i;
    if (getenv("REALISTIC")) {  // priority-key shaped: shared high bytes, 24-bit ids in the low bits
        for (int i = 0; i < N; ++i) {
            const uint64_t level = (uint64_t)(rand() % 3), perc = (uint64_t)(rand() % 4 == 0);
            const uint64_t est = perc ? (uint64_t)(rand() % 400000) : 0;
            h[i] = (1ull << 62) | (level << 58) | ((1 - perc) << 57) | (1ull << 56) | (est << 24) | (uint64_t)(i * 8 + 3);
        }
        printf("realistic keys\n");
    }
    uint64_t *din, *dout;
    long long *dc, hc[3];
    cudaMalloc(&din, N * 8); cudaMalloc(&dout, N * 8); cudaMalloc(&dc, 64);
    cudaMemcpy(din, h.data(), N * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    warp_only<<<1, 32>>>(din, dout, dc);
    cudaMemcpy(hc, dc, 8, cudaMemcpyDeviceToHost);
    printf("warp_sort64 (1 warp): %lld cycles\n", hc[0]);
    for (int threads : {512, 608, 1024}) {
        for (int n : {512, 2048}) {
            bench<<<1, threads, 3 * n * 8>>>(din, dout, n, 512, dc, 0);
            cudaMemcpy(hc, dc, 24, cudaMemcpyDeviceToHost);
            std::vector<uint64_t> o(n);
            cudaMemcpy(o.data(), dout, n * 8, cudaMemcpyDeviceToHost);
            bool ok = true;
            for (int i = 1; i < n; ++i) ok &= o[i - 1] <= o[i];
            printf("block_sort n=%d threads=%d: %lld / %lld / %lld cycles %s\n", n, threads, hc[0], hc[1], hc[2], ok ? "sorted" : "NOT SORTED");
        }
        for (int n : {512, 2048}) {
            bench<<<1, threads, 3 * n * 8>>>(din, dout, n, 512, dc, 2);
            if (cudaGetLastError() != cudaSuccess) printf("launch failed\n");
            cudaMemcpy(hc, dc, 24, cudaMemcpyDeviceToHost);
            std::vector<uint64_t> o(n);
            cudaMemcpy(o.data(), dout, n * 8, cudaMemcpyDeviceToHost);
            bool ok = true;
            for (int i = 1; i < n; ++i) ok &= o[i - 1] <= o[i];
            std::vector<uint64_t> ref(h.begin(), h.begin() + n);
            std::sort(ref.begin(), ref.end());
            ok &= ref == o;
            printf("block_sort_reg n=%d threads=%d: %lld / %lld / %lld cycles %s\n", n, threads, hc[0], hc[1], hc[2], ok ? "sorted" : "WRONG");
        }
        bench<<<1, threads, 3 * 2048 * 8>>>(din, dout, 2048, 512, dc, 1);
        cudaMemcpy(hc, dc, 24, cudaMemcpyDeviceToHost);
        printf("select_topB n=2048 B=512 threads=%d: %lld / %lld / %lld cycles\n", threads, hc[0], hc[1], hc[2]);
    }
    cudaError_t e = cudaGetLastError();
    printf("last launch: %s\n", cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
