// Probe: tcgen05.mma kind::tf32 issue/completion rate for the plane K-pass tile (M = 128, N = 64,
// 4 K-steps x 3 components x 3 products = 36 MMAs per tile), operands resident (no loads):
//   variant 0: A_hi from shared memory MN-major SW128_32B (2 of 3 products), A_lo from TMEM
//   variant 1: all three products with A from TMEM
//   variant 2: all three with A from shared memory K-major (SWIZZLE_NONE)
//   variant 3: variant 0 with N = 128 (18 MMAs per 64 outputs-equivalent tile pair)
// One CTA per SM, 400 tiles each, commit + wait per tile (as the kernel); prints cycles per tile.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint64_t desc_mn32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(4096u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
template <int N> struct Id {
    static constexpr uint32_t S = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((N >> 3) << 17) | ((128u >> 4) << 24);
    static constexpr uint32_t T = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
    static constexpr uint32_t K = T;
};
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                 ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__global__ void rate(int variant, int tiles, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = raw + ((1024u - ((unsigned)__cvta_generic_to_shared(raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < (48 * 1024 + 32 * 1024) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f / (1 + i % 7);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"((unsigned)__cvta_generic_to_shared(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t a = (unsigned)__cvta_generic_to_shared(sm), b = a + 48 * 1024;
        unsigned long long t0 = clock64();
        unsigned ph = 0;
        for (int t = 0; t < tiles; ++t) {
            for (int c = 0; c < 3; ++c) {
                if (variant == 3) {
                    const uint32_t d = tm + 128u * c;
                    for (int kk = 0; kk < 4; ++kk) {
                        mma_ss(d, desc_mn32(a + 16384u * c + 1024u * kk), desc_k(b + 256u * kk, 1024), Id<128>::S, t || kk);
                        mma_ss(d, desc_mn32(a + 16384u * c + 1024u * kk), desc_k(b + 16384u + 256u * kk, 1024), Id<128>::S, 1);
                        mma_ts(d, tm + 384u + 8u * kk, desc_k(b + 256u * kk, 1024), Id<128>::T, 1);
                    }
                    continue;
                }
                const uint32_t d = tm + 64u * c;
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t bh = desc_k(b + 256u * kk, 1024), bl = desc_k(b + 8192u + 256u * kk, 1024);
                    if (variant == 0) {
                        mma_ss(d, desc_mn32(a + 16384u * c + 1024u * kk), bh, Id<64>::S, t || kk);
                        mma_ss(d, desc_mn32(a + 16384u * c + 1024u * kk), bl, Id<64>::S, 1);
                        mma_ts(d, tm + 192u + 32u * c + 8u * kk, bh, Id<64>::T, 1);
                    } else if (variant == 1) {
                        mma_ts(d, tm + 192u + 32u * c + 8u * kk, bh, Id<64>::T, t || kk);
                        mma_ts(d, tm + 288u + 32u * c + 8u * kk, bh, Id<64>::T, 1);
                        mma_ts(d, tm + 192u + 32u * c + 8u * kk, bl, Id<64>::T, 1);
                    } else {
                        const uint64_t ak = desc_k(a + 16384u * c + 256u * kk, 1024);
                        mma_ss(d, ak, bh, Id<64>::K, t || kk);
                        mma_ss(d, ak, bl, Id<64>::K, 1);
                        mma_ss(d, ak + 64, bh, Id<64>::K, 1);
                    }
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                (unsigned)__cvta_generic_to_shared(&bar)) : "memory");
            asm volatile("{\n .reg .pred P1;\n W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W;\n}\n"
                         ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(ph) : "memory");
            ph ^= 1;
        }
        out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm) : "memory");
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 8);
    unsigned long long h[148];
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 82 * 1024);
    const char* nm[4] = {"SS MN-major hi x2 + TS lo (N=64, current)", "all TS (N=64)", "all SS K-major (N=64)", "SS MN + TS, N=128"};
    for (int v = 0; v < 4; ++v) {
        rate<<<148, 128, 82 * 1024>>>(v, 400, d);
        cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
        const double cyc = s / 148 / 400;
        const double flop = 2.0 * 128 * (v == 3 ? 128 : 64) * 32 * 3 * 3;
        printf("%-45s %s: %.0f cycles per tile, %.0f flop/cycle/SM (3 products counted)\n", nm[v], cudaGetErrorString(e), cyc, flop / cyc);
    }
    return 0;
}
