// Probe: does tcgen05.mma kind::tf32 truncate or round the low 13 mantissa bits of fp32
// operands read from shared memory?  A[0][0] = 1 + 3 * 2^-12 (0.75 tf32 ulp above 1),
// B[0][0] = 1, everything else 0: D[0][0] = 1 (truncation) or 1 + 2^-10 (round to nearest).
// Also A[1][0] = 1 + 2^-11 + 2^-13 (just above half an ulp) and A[2][0] = -(1 + 3 * 2^-12).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tf32_round tf32_round.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1 << 46);
}
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
__global__ void probe(float* out) {
    __shared__ __align__(1024) float A[128 * 32];
    __shared__ __align__(1024) float B[32 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 32; i += blockDim.x) A[i] = 0.f;
    for (int i = tid; i < 32 * 32; i += blockDim.x) B[i] = 0.f;
    __syncthreads();
    auto aidx = [](int m, int k) { return ((m >> 3) * 1024 + (m & 7) * 16 + (k >> 2) * 128) / 4 + (k & 3); };
    if (tid == 0) {
        A[aidx(0, 0)] = 1.f + 3.f * exp2f(-12.f);
        A[aidx(1, 0)] = 1.f + exp2f(-11.f) + exp2f(-13.f);
        A[aidx(2, 0)] = -(1.f + 3.f * exp2f(-12.f));
        A[aidx(3, 0)] = 1.f + exp2f(-11.f);          // exactly half an ulp: RNE -> 1, RNA -> 1 + 2^-10
        B[aidx(0, 0)] = 1.f;                          // same core-matrix layout for the 32 x 32 B
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tm = tbase;
    if (tid == 0) {
        uint64_t da = desc_k((unsigned)__cvta_generic_to_shared(A)), db = desc_k((unsigned)__cvta_generic_to_shared(B));
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, 0, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(kIdesc) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(&bar)) : "memory");
    }
    if (tid < 32) {
        asm volatile("{\n .reg .pred P1;\n W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n"
                     ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        uint32_t r;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(tm));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (tid < 4) out[tid] = __uint_as_float(r);
        __syncwarp();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tm) : "memory");
    }
}
int main() {
    float* d; cudaMalloc(&d, 16);
    probe<<<1, 128>>>(d);
    float h[4];
    cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(e));
    const char* nm[4] = {"1+0.75ulp", "1+0.625ulp(>half)", "-(1+0.75ulp)", "1+0.5ulp"};
    for (int i = 0; i < 4; ++i) printf("%-20s D = %.10f  (1 + %.4f ulp)\n", nm[i], h[i], (fabsf(h[i]) - 1.f) / exp2f(-10.f));
    return 0;
}
