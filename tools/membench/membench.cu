// Micro-benchmark: streaming reads of N bytes with (a) float4 loads, (b) 4 KB bulk copies into
// shared memory (kStages per warp), to calibrate the K-pass kernels' achievable DRAM rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void rd_vec(const float4* __restrict__ a, size_t n, float* out) {
    float s = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(&a[i]);
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 12345.f) out[0] = s;
}
template <int S, int TB>
__global__ void rd_bulk(const float* __restrict__ a, size_t ntiles, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bars[8][S];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* tile = reinterpret_cast<float*>(sm) + (size_t)w * S * (TB / 4);
    const size_t G = (size_t)gridDim.x * (blockDim.x >> 5);
    const size_t gw = blockIdx.x * (blockDim.x >> 5) + w;
    if (lane == 0) for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(&bars[w][s])));
    __syncwarp();
    size_t mine = gw < ntiles ? (ntiles - gw + G - 1) / G : 0;
    auto issue = [&](size_t t) {
        int s = t % S;
        if (lane == 0) {
            unsigned b = (unsigned)__cvta_generic_to_shared(&bars[w][s]);
            unsigned d = (unsigned)__cvta_generic_to_shared(tile + s * (TB / 4));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(TB) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(d), "l"(a + (gw + t * G) * (TB / 4)), "r"(TB), "r"(b) : "memory");
        }
    };
    for (int t = 0; t < S - 1 && t < (int)mine; ++t) issue(t);
    float acc = 0.f;
    unsigned par = 0;
    for (size_t t = 0; t < mine; ++t) {
        if (t + S - 1 < mine) issue(t + S - 1);
        int s = t % S;
        unsigned b = (unsigned)__cvta_generic_to_shared(&bars[w][s]);
        unsigned done = 0;
        while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(b), "r"((par >> s) & 1u) : "memory");
        par ^= 1u << s;
        for (int q = lane; q < TB / 4; q += 32) acc += tile[s * (TB / 4) + q];
        __syncwarp();
    }
    if (acc == 12345.f) out[0] = acc;
}
int main() {
    size_t bytes = 80ull << 20;
    float *a, *out, *flush;
    cudaMalloc(&a, bytes); cudaMalloc(&out, 4); cudaMalloc(&flush, 256ull << 20);
    cudaMemset(a, 0, bytes);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaMemset(flush, r, 256ull << 20);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("%-32s %8.2f us  %8.1f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    timeit("float4 ldcs, 4 blk/SM x 512", [&] { rd_vec<<<nsm * 4, 512>>>((const float4*)a, bytes / 16, out); });
    timeit("float4 ldcs, 8 blk/SM x 256", [&] { rd_vec<<<nsm * 8, 256>>>((const float4*)a, bytes / 16, out); });
    size_t nt4 = bytes / 4096;
    auto sm3 = 8 * 3 * 4096; cudaFuncSetAttribute(rd_bulk<3, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
    timeit("bulk 4KB S=3 8w x 2 CTA/SM", [&] { rd_bulk<3, 4096><<<nsm * 2, 256, sm3>>>(a, nt4, out); });
    auto sm6 = 8 * 6 * 4096; cudaFuncSetAttribute(rd_bulk<6, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm6);
    timeit("bulk 4KB S=6 8w x 1 CTA/SM", [&] { rd_bulk<6, 4096><<<nsm * 1, 256, sm6>>>(a, nt4, out); });
    size_t nt16 = bytes / 16384;
    auto smb = 8 * 3 * 16384; cudaFuncSetAttribute(rd_bulk<3, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
    timeit("bulk 16KB S=3 8w x 1 CTA/SM", [&] { rd_bulk<3, 16384><<<nsm * 1, 256, smb>>>(a, nt16, out); });
    auto sm2 = 4 * 3 * 16384; cudaFuncSetAttribute(rd_bulk<3, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    timeit("bulk 16KB S=3 4w x 2 CTA/SM", [&] { rd_bulk<3, 16384><<<nsm * 2, 128, sm2>>>(a, nt16, out); });
    return 0;
}
