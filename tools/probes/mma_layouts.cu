// Probe: tcgen05.mma kind::tf32, M = 128, N = 64, K = 8 with
//   (a) A in shared memory, MN-major SWIZZLE_128B: element (m, k) at
//       (m / 32) * LBOa + (k / 8) * 1024 + (k % 8) * 128 + (((m % 32) / 4) ^ (k % 8)) * 16 + (m % 4) * 4
//       tried with the descriptor's (LBO, SBO) = (4096, 1024) and (1024, 4096)
//   (b) A in TMEM (lane = m, column = k), a_major = 0
// B: K-major SWIZZLE_NONE core matrices [n / 8][k / 4][n % 8][k % 4] (LBO 128, SBO 1024).
// Values are small integers (exact in tf32): D must equal the CPU product exactly.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o mma_layouts mma_layouts.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint64_t desc_mn32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {   // SWIZZLE_128B_BASE32B
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
__device__ __forceinline__ uint64_t desc_kk(uint32_t saddr) {   // K-major, LBO 128, SBO 256
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
           ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint64_t desc_mn0(uint32_t saddr, uint32_t lbo, uint32_t sbo) {   // SWIZZLE_NONE
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
constexpr uint32_t kIdS = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdT = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
__device__ int aoff(int v, int m, int k) {   // byte offset of A(m, k) in variant v's buffer
    if (v == 0) return (m / 32) * 4096 + (k % 8) * 128 + ((((m % 32) / 4) ^ (k % 8)) * 16) + (m % 4) * 4;   // SW128, M-blocks at 4 KB
    if (v == 1) return (m / 32) * 4096 + (k / 4) * 512 + (k % 4) * 128 + ((((m % 32) / 8) ^ (k % 4)) * 32) + (m % 8) * 4;   // SW128_32B
    if (v == 2) return (m / 4) * 128 + (k % 8) * 16 + (m % 4) * 4;                                          // INTERLEAVE, M-cores at 128 B
    return (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4;                                       // K-major core matrices
}
__global__ void probe(const float* Ag /*[128][8]*/, const float* Bg /*[8][64]*/, float* out /*[6][128][64]*/) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = raw + ((1024u - ((unsigned)__cvta_generic_to_shared(raw) & 1023u)) & 1023u);
    float* A = reinterpret_cast<float*>(sm);            // 4 variants x 16 KB
    float* B = reinterpret_cast<float*>(sm + 65536);    // 64 x 8 (2 KB)
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 4 * 4096; i += blockDim.x) A[i] = 0.f;
    __syncthreads();
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int m = i / 8, k = i % 8;
        for (int v = 0; v < 4; ++v) A[v * 4096 + aoff(v, m, k) / 4] = Ag[i];
    }
    for (int i = tid; i < 64 * 8; i += blockDim.x) {
        const int k = i / 64, n = i % 64;
        const int d = (n / 8) * 256 + (k / 4) * 32 + (n % 8) * 4 + (k % 4);
        B[d] = Bg[i];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tm = tbase;
    // A into TMEM columns 192..199 (lane = m): warp w stores lanes 32 w.. (w < 4)
    {
        const int w = tid >> 5, lane = tid & 31;
        if (w < 4) {
            uint32_t r[8];
            for (int k = 0; k < 8; ++k) r[k] = __float_as_uint(Ag[(32 * w + lane) * 8 + k]);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
                             tm + ((uint32_t)(32 * w) << 16) + 448u),
                         "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                         : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (tid == 0) {
        const uint32_t a = (unsigned)__cvta_generic_to_shared(A), b = (unsigned)__cvta_generic_to_shared(B);
        const uint64_t d[5] = {desc_mn(a, 4096, 1024), desc_mn32(a + 16384, 4096, 512), desc_mn32(a + 16384, 512, 4096),
                               desc_mn0(a + 32768, 4096, 128), desc_kk(a + 49152)};
        for (int v = 0; v < 5; ++v)
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tm + 64u * v), "l"(d[v]), "l"(desc_k(b)), "r"(v == 4 ? kIdT : kIdS) : "memory");
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm + 320u), "r"(tm + 448u), "l"(desc_k(b)), "r"(kIdT) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(&bar)) : "memory");
    }
    {
        asm volatile("{\n .reg .pred P1;\n W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n"
                     ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const int w = tid >> 5, lane = tid & 31;
        if (w < 4) {
            for (int v = 0; v < 6; ++v)
                for (int n = 0; n < 64; ++n) {
                    uint32_t r;
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r)
                                 : "r"(tm + ((uint32_t)(32 * w) << 16) + 64u * v + n));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    out[(v * 128 + 32 * w + lane) * 64 + n] = __uint_as_float(r);
                }
        }
    }
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm) : "memory");
}
int main() {
    float hA[128 * 8], hB[8 * 64], ref[128 * 64], hout[6 * 128 * 64];
    for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7 + 3) % 11 - 5);
    for (int i = 0; i < 8 * 64; ++i) hB[i] = (float)((i * 5 + 1) % 9 - 4);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
            float s = 0;
            for (int k = 0; k < 8; ++k) s += hA[m * 8 + k] * hB[k * 64 + n];
            ref[m * 64 + n] = s;
        }
    float *dA, *dB, *dO;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dO, sizeof hout);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 72 * 1024);
    probe<<<1, 128, 72 * 1024>>>(dA, dB, dO);
    cudaError_t e = cudaMemcpy(hout, dO, sizeof hout, cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(e));
    const char* nm[6] = {"SW128 blocks@4K (LBO 4096, SBO 1024)", "SW128_32B (LBO 4096, SBO 512)",
                         "SW128_32B (LBO 512, SBO 4096)", "NONE cores@128B (LBO 4096, SBO 128)",
                         "K-major control (no transpose bit)", "TMEM A"};
    for (int v = 0; v < 6; ++v) {
        double mx = 0; int bad = 0;
        for (int i = 0; i < 128 * 64; ++i) { double d = fabs(hout[v * 8192 + i] - ref[i]); mx = d > mx ? d : mx; bad += d > 0; }
        printf("%-45s max |D - ref| = %g (%d mismatches of 8192); D[0][0..3] = %g %g %g %g ref %g %g %g %g\n", nm[v], mx, bad,
               hout[v * 8192], hout[v * 8192 + 1], hout[v * 8192 + 2], hout[v * 8192 + 3], ref[0], ref[1], ref[2], ref[3]);
    }
    return 0;
}
