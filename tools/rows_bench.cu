// rows_bench.cu -- HBM throughput of the verify access pattern (tooling, not product):
// B slots x n_chunks items, each item = two 16 KB bulk copies (chunk c of a p row and of
// a q row), items n -> CTA n % grid, ring of 6 x 32 KB stages; rows placed (0) at random
// in a 4.5 GB pool, (1) at random inside a 512 MB window, (2) contiguously.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/rows_bench tools/rows_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kCons = 8;

template <int kStages, int kChunk, int kSplit>
__global__ void __launch_bounds__((kCons + 1) * 32, 1) rows_kernel(const char *pool, const int64_t *prow, const int64_t *qrow,
                                                                 int B, int nc, int64_t row_bytes, unsigned long long *sink) {
    extern __shared__ __align__(128) uint8_t buf[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_items = B * nc, grid = gridDim.x;
    const int n_my = (int)blockIdx.x < n_items ? (n_items - 1 - (int)blockIdx.x) / grid + 1 : 0;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(kCons));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kCons) {
        if (lane == 0) {
            for (int k = 0; k < n_my; ++k) {
                const int st = k % kStages;
                if (k >= kStages) {
                    const uint32_t par = ((k / kStages) - 1) & 1;
                    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(smem_u32(&empty[st])), "r"(par) : "memory");
                }
                const int n = blockIdx.x + k * grid;
                const int b = n / nc, c = n % nc;
                const int64_t off = (int64_t)c * kChunk;
                const uint32_t bytes = (uint32_t)(off + kChunk <= row_bytes ? kChunk : ((row_bytes - off) & ~15));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(2 * bytes) : "memory");
                const uint32_t piece = (bytes / kSplit + 15) & ~15u;
                for (uint32_t o = 0; o < bytes; o += piece) {
                    const uint32_t nb = bytes - o < piece ? bytes - o : piece;
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(smem_u32(buf + (size_t)st * 2 * kChunk + o)), "l"(pool + prow[b] + off + o), "r"(nb), "r"(smem_u32(&full[st])) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(smem_u32(buf + (size_t)st * 2 * kChunk + kChunk + o)), "l"(pool + qrow[b] + off + o), "r"(nb), "r"(smem_u32(&full[st])) : "memory");
                }
            }
        }
    } else {
        uint32_t acc = 0;
        for (int k = 0; k < n_my; ++k) {
            const int st = k % kStages;
            const uint32_t par = (k / kStages) & 1;
            asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(smem_u32(&full[st])), "r"(par) : "memory");
            const uint4 *t = reinterpret_cast<const uint4 *>(buf + (size_t)st * 2 * kChunk);
            for (int v = warp * 32 + lane; v < 2 * kChunk / 16; v += kCons * 32) { uint4 x = t[v]; acc ^= x.x ^ x.w; }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
        }
        if (acc == 0x12345678u) atomicAdd(sink, 1ull);
    }
}


template <int kStages, int kChunk, int kSplit = 1>
void run(const char *pool, int64_t pool_bytes, int B, int grid, int mode, unsigned long long *sink, std::mt19937_64 &rng) {
    const int64_t V = 128256, row_bytes = V * 2;
    const int nc = (int)((row_bytes + kChunk - 1) / kChunk), L = 40;
    const size_t smem = (size_t)kStages * 2 * kChunk;
    CK(cudaFuncSetAttribute(rows_kernel<kStages, kChunk, kSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t n_rows = pool_bytes / row_bytes;
    std::vector<int64_t> hp((size_t)L * B), hq((size_t)L * B);
    for (int l = 0; l < L; ++l)
        for (int b = 0; b < B; ++b) {
            int64_t pr, qr;
            if (mode == 0) { const int64_t slab = rng() % 1024; const int r = (int)(rng() % 8); pr = slab * 17 + r; qr = slab * 17 + 9 + r; }
            else { pr = (int64_t)((l * 2 * (int64_t)B + 2 * b) % n_rows); qr = (pr + 1) % n_rows; }
            hp[(size_t)l * B + b] = pr * row_bytes;
            hq[(size_t)l * B + b] = qr * row_bytes;
        }
    int64_t *dp, *dq;
    CK(cudaMalloc(&dp, hp.size() * 8));
    CK(cudaMalloc(&dq, hq.size() * 8));
    CK(cudaMemcpy(dp, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dq, hq.data(), hq.size() * 8, cudaMemcpyHostToDevice));
    for (int l = 0; l < 4; ++l) rows_kernel<kStages, kChunk, kSplit><<<grid, (kCons + 1) * 32, smem>>>(pool, dp + l * B, dq + l * B, B, nc, row_bytes, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int l = 0; l < L; ++l) rows_kernel<kStages, kChunk, kSplit><<<grid, (kCons + 1) * 32, smem>>>(pool, dp + l * B, dq + l * B, B, nc, row_bytes, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes_total = (double)L * B * 2 * row_bytes;
    printf("%s B=%5d stages=%d chunk=%2dKB split=%d grid=%d: %7.1f us/launch  %.0f GB/s\n", mode == 0 ? "slab-random" : "contiguous ", B,
           kStages, kChunk / 1024, kSplit, grid, ms * 1e3 / L, bytes_total / (ms * 1e-3) / 1e9);
    cudaFree(dp); cudaFree(dq);
}

int main() {
    const int64_t V = 128256, row_bytes = V * 2;
    const int64_t pool_bytes = (int64_t)1024 * 17 * row_bytes;  // 4.46 GB
    char *pool;
    unsigned long long *sink;
    CK(cudaMalloc(&pool, pool_bytes));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(pool, 1, pool_bytes));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::mt19937_64 rng(1);
    for (int B : {512, 4096}) {
        run<6, 16384>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
        run<3, 32768>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
        run<3, 32768, 2>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
        run<3, 32768, 4>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
        run<2, 49152>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
        run<4, 24576>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
        run<2, 32768>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
        run<6, 16384, 2>(pool, pool_bytes, B, sms - 1, 0, sink, rng);
    }
    return 0;
}
