// Hot-path kernels of the sparse-inverse local-global iteration (sm_100a).
//
// Per L-G iteration (Alg. 4), delta form x^{k+1} = x^k + A^-1 (b - A x^k + h^2 H^T lam):
//   local        per tet: F, signed SVD, projection, force block      (eq. PD local P:L310)
//   contact_eval per contact: gaps, FB theta/E/phi, h-vector           (App. B.2)
//   gather       per vertex: u = M(s - x) + sum_i f_i + h^2 H^T lam     (delta form)
//   kpass1       y = K u            (3 RHS, column-major K, thread per row)   (P:L442 first SpMV)
//   chain_dot    (K^T y) at contact vertices (ancestor chains)
//   cr           (Theta D Theta + C) z = rho, CR in one 16-CTA cluster
//   scatter      y += K H^T z (rows on the contact vertices' chains)    (P:L956 correction)
//   kpass2       x += K^T y         (row-major K, thread per column)  (P:L442 second SpMV)
// A single scene (n_instances = 1) streams K through CUDA cores (SpMV, HBM-bound); with several
// instances sharing K the K-passes and the contact passes become dense 32x32-tile contractions
// over 3 S right-hand sides and run on the tcgen05 tensor cores (kind::tf32, 3xTF32).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"

// Programmatic dependent launch (PDL): every hot-path kernel starts by waiting for its
// stream predecessor to complete (griddepcontrol.wait: a no-op without the launch attribute)
// and then lets its own successor launch, so consecutive kernels of the frame graph overlap
// their launch and prologue with the tail of the previous grid.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
#ifdef SIM_PDL_EARLY_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

#ifndef SIM_JACOBI_SWEEPS
#define SIM_JACOBI_SWEEPS 6   // cap of the cyclic Jacobi sweeps of the local step's SVD
#endif

namespace cg = cooperative_groups;

namespace simdev {

// One-time per-device launch setup (cudaFuncSetAttribute is a per-device setting): bit d of
// `mask` records that device d is configured; the SM count is cached per device.
static std::mutex g_attr_mu;
template <class F>
static void per_device_once(unsigned long long& mask, F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (!((mask >> (dev & 63)) & 1ull)) {
        f();
        mask |= 1ull << (dev & 63);
    }
}
static int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& n = cache[dev & 63];
    if (!n) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}


// Right-hand-side vectors u, y of the K-passes: S = 1: float4 [n_f] (.w carries pass 1's column
// base); S > 1: three fp32 component planes [c][n_f][Sp], Sp = S rounded up to a multiple of 4 (the
// planes the batched K-passes stream with 16-byte copies; entries S..Sp-1 of a row are padding).
__device__ __forceinline__ float4 vec_ld(const float4* v, int S, int n_f, int row, int inst) {
    if (S == 1) return __ldg(&v[row]);
    const int Sp = plane_sp(S);
    const float* p = reinterpret_cast<const float*>(v);
    const size_t PS = (size_t)n_f * Sp, i = (size_t)row * Sp + inst;
    return make_float4(__ldg(p + i), __ldg(p + PS + i), __ldg(p + 2 * PS + i), 0.f);
}
__device__ __forceinline__ void vec_st(float4* v, int S, int n_f, int row, int inst, float a0, float a1, float a2,
                                       float w = 0.f) {
    if (S == 1) {
        v[row] = make_float4(a0, a1, a2, w);
        return;
    }
    const int Sp = plane_sp(S);
    float* p = reinterpret_cast<float*>(v);
    const size_t PS = (size_t)n_f * Sp, i = (size_t)row * Sp + inst;
    p[i] = a0;
    p[PS + i] = a1;
    p[2 * PS + i] = a2;
}
// v[row] += (a0, a1, a2), rounded once to fp32
__device__ __forceinline__ void vec_add(float4* v, int S, int n_f, int row, int inst, double a0, double a1, double a2) {
    if (S == 1) {
        const float4 yi = v[row];
        v[row] = make_float4((float)(yi.x + a0), (float)(yi.y + a1), (float)(yi.z + a2), yi.w);
        return;
    }
    const int Sp = plane_sp(S);
    float* p = reinterpret_cast<float*>(v);
    const size_t PS = (size_t)n_f * Sp, i = (size_t)row * Sp + inst;
    p[i] = (float)(p[i] + a0);
    p[PS + i] = (float)(p[PS + i] + a1);
    p[2 * PS + i] = (float)(p[2 * PS + i] + a2);
}

// ----------------------------------------------------------------------------
// predict: s = x_t + h v_t + h^2 g; pinned: x = x_t + h v_pin of that vertex-instance
// (sim_set_pin_velocity / sim_set_pins).  Frame start: default x^0 = s, lambda^0 = 0 (readings A9,
// A10); warm start x^0 = x_t + h v_t and lambda kept from the previous frame (A9w, A10w).
// ----------------------------------------------------------------------------
__global__ void k_predict(Params P, double4* __restrict__ x, double4* __restrict__ xt,
                          double4* __restrict__ v, double4* __restrict__ s, double* __restrict__ lam, int nlam,
                          double4* __restrict__ vt, int* __restrict__ bad) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;   // (vertex, instance), instance-minor
    if (!P.warm && i < nlam) lam[i] = 0.0;
    if (bad && i < P.S) bad[i] = 0;
    if (i >= P.n_v * P.S) return;
    double4 xi = x[i];
    xt[i] = xi;
    if (vt) vt[i] = v[i];   // frame-start velocity, restored if the frame turns non-finite
    double h = P.h;
    if (i < P.n_f * P.S) {
        double4 vi = v[i];
        const double4 xv = make_double4(xi.x + h * vi.x, xi.y + h * vi.y, xi.z + h * vi.z, 0.0);
        const double4 si = make_double4(xv.x + h * h * P.g[0], xv.y + h * h * P.g[1], xv.z + h * h * P.g[2], 0.0);
        s[i] = si;
        x[i] = P.warm ? xv : si;
    } else {
        const double4 vp = P.vpin[i - P.n_f * P.S];
        x[i] = make_double4(xi.x + h * vp.x, xi.y + h * vp.y, xi.z + h * vp.z, 0.0);
        v[i] = make_double4(vp.x, vp.y, vp.z, 0.0);
    }
}

__global__ void k_pin_targets(int n_f, int n_pin, int S, int inst, double h, const double4* __restrict__ x,
                              const double4* __restrict__ target, double4* __restrict__ vpin) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_pin) return;
    const double4 a = x[(size_t)(n_f + p) * S + inst], t = target[p];
    vpin[(size_t)p * S + inst] = make_double4((t.x - a.x) / h, (t.y - a.y) / h, (t.z - a.z) / h, 0.0);
}
void launch_pin_targets(cudaStream_t st, int n_f, int n_pin, int S, int inst, double h, const double4* x,
                        const double4* target, double4* vpin) {
    if (n_pin > 0) k_pin_targets<<<(n_pin + 127) / 128, 128, 0, st>>>(n_f, n_pin, S, inst, h, x, target, vpin);
}

void launch_predict(cudaStream_t st, const Params& P, double4* x, double4* xt, double4* v, double4* s,
                    double* lam, int nlam, double4* vt, int* bad) {
    int n = P.n_v * P.S > nlam ? P.n_v * P.S : nlam;
    n = n > P.S ? n : P.S;
    k_predict<<<(n + 255) / 256, 256, 0, st>>>(P, x, xt, v, s, lam, nlam, vt, bad);
}

// lambda across a contact commit (reading A10): row r of new contact c takes row r of the
// previous commit's contact carry[c] (an identical constraint), or 0
__global__ void k_carry_lambda(int C, const int32_t* __restrict__ carry, const double* __restrict__ lam_old,
                               double* __restrict__ lam) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= 3 * C) return;
    const int src = carry[j / 3];
    lam[j] = src >= 0 ? lam_old[3 * src + j % 3] : 0.0;
}
void launch_carry_lambda(cudaStream_t st, int C, const int32_t* carry, const double* lam_old, double* lam) {
    if (C > 0) k_carry_lambda<<<(3 * C + 255) / 256, 256, 0, st>>>(C, carry, lam_old, lam);
}

// ----------------------------------------------------------------------------
// failure detection: an instance whose frame produced a non-finite position or
// velocity is rolled back to its frame-start state (x_t, v_t); `rollbacks` (host-mapped)
// counts the rolled-back instance-frames for sim_synchronize to report
// ----------------------------------------------------------------------------
__global__ void k_finite_check(int n, int S, const double4* __restrict__ x, const double4* __restrict__ v,
                               int* __restrict__ bad) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * S) return;
    const double4 a = x[i], b = v[i];
    const bool ok = isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(b.x) && isfinite(b.y) && isfinite(b.z);
    if (!ok) atomicOr(&bad[i % S], 1);
}

__global__ void k_rollback(int n, int S, double4* __restrict__ x, double4* __restrict__ v,
                           const double4* __restrict__ xt, const double4* __restrict__ vt,
                           const int* __restrict__ bad, int* rollbacks) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * S) return;
    const int inst = i % S;
    if (!bad[inst]) return;
    x[i] = xt[i];
    v[i] = vt[i];
    if (i < S) atomicAdd(rollbacks, 1);   // vertex 0 of the instance
}

__global__ void k_poison(double4* x, int inst, int S) {
    if (threadIdx.x == 0 && blockIdx.x == 0) x[inst].x = __longlong_as_double(0x7ff8000000000000ll);
}
void launch_poison(cudaStream_t st, double4* x, int inst, int S) { k_poison<<<1, 32, 0, st>>>(x, inst, S); }

// dst[(inst * n_v + v) * 3 + d] = x[o2i[v] * S + inst].d  (the caller's layout, original order)
__global__ void k_pack_positions(const double4* __restrict__ x, const int32_t* __restrict__ o2i, int n_v, int S,
                                 double* __restrict__ dst) {
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;   // (instance, vertex)
    if (e >= (size_t)n_v * S) return;
    const int inst = (int)(e / n_v), vtx = (int)(e - (size_t)inst * n_v);
    const double4 a = x[(size_t)o2i[vtx] * S + inst];
    dst[3 * e] = a.x;
    dst[3 * e + 1] = a.y;
    dst[3 * e + 2] = a.z;
}
void launch_pack_positions(cudaStream_t st, const double4* x, const int32_t* o2i, int n_v, int S, double* dst) {
    const size_t n = (size_t)n_v * S;
    if (n) k_pack_positions<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, o2i, n_v, S, dst);
}

// ----------------------------------------------------------------------------
// proximity query ("simple proximity queries"): signed distance of each
// candidate vertex to analytic obstacle surfaces; nearest obstacle wins (reading A31)
// ----------------------------------------------------------------------------
__global__ void k_proximity(Params P, const double4* __restrict__ x, int inst, const int32_t* __restrict__ cand,
                            int ncand, const DObstacle* __restrict__ obs, int nobs, double margin,
                            int* __restrict__ best, double* __restrict__ gapo, double3* __restrict__ no,
                            double3* __restrict__ pto) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncand) return;
    const double4 xa = x[(size_t)cand[c] * P.S + inst];
    int bi = -1;
    double bg = 0.0, bn[3] = {0, 0, 0}, bp[3] = {0, 0, 0};
    for (int o = 0; o < nobs; ++o) {
        const DObstacle& ob = obs[o];
        double q[3], n[3], g;
        const double p[3] = {xa.x, xa.y, xa.z};
        if (ob.kind == 0) {   // plane through a with unit normal b
            g = (p[0] - ob.a[0]) * ob.b[0] + (p[1] - ob.a[1]) * ob.b[1] + (p[2] - ob.a[2]) * ob.b[2];
            for (int k = 0; k < 3; ++k) { n[k] = ob.b[k]; q[k] = p[k] - g * ob.b[k]; }
        } else {              // sphere (centre a) or capsule (segment a-b): distance to the core point
            double cpt[3] = {ob.a[0], ob.a[1], ob.a[2]};
            if (ob.kind == 2) {
                const double d[3] = {ob.b[0] - ob.a[0], ob.b[1] - ob.a[1], ob.b[2] - ob.a[2]};
                const double dd = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
                double t = dd > 0.0 ? ((p[0] - ob.a[0]) * d[0] + (p[1] - ob.a[1]) * d[1] + (p[2] - ob.a[2]) * d[2]) / dd
                                    : 0.0;
                t = fmin(fmax(t, 0.0), 1.0);
                for (int k = 0; k < 3; ++k) cpt[k] = ob.a[k] + t * d[k];
            }
            const double v[3] = {p[0] - cpt[0], p[1] - cpt[1], p[2] - cpt[2]};
            const double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            if (!(dist > 0.0)) continue;   // on the core: no defined normal
            for (int k = 0; k < 3; ++k) n[k] = v[k] / dist;
            g = dist - ob.radius;
            for (int k = 0; k < 3; ++k) q[k] = cpt[k] + ob.radius * n[k];
        }
        if (g < margin && (bi < 0 || g < bg)) {
            bi = o;
            bg = g;
            for (int k = 0; k < 3; ++k) { bn[k] = n[k]; bp[k] = q[k]; }
        }
    }
    best[c] = bi;
    gapo[c] = bg;
    no[c] = make_double3(bn[0], bn[1], bn[2]);
    pto[c] = make_double3(bp[0], bp[1], bp[2]);
}

void launch_proximity(cudaStream_t st, const Params& P, const double4* x, int inst, const int32_t* cand, int ncand,
                      const DObstacle* obs, int nobs, double margin, int* best, double* gap, double3* n, double3* pt) {
    if (ncand > 0)
        k_proximity<<<(ncand + 127) / 128, 128, 0, st>>>(P, x, inst, cand, ncand, obs, nobs, margin, best, gap, n, pt);
}

void launch_finite_guard(cudaStream_t st, int n_v, int S, double4* x, double4* v, const double4* xt,
                         const double4* vt, int* bad, int* rollbacks) {
    const int blocks = (int)(((size_t)n_v * S + 255) / 256);
    launch_pdl(k_finite_check, dim3(blocks), dim3(256), 0, st, n_v, S, x, v, bad);
    launch_pdl(k_rollback, dim3(blocks), dim3(256), 0, st, n_v, S, x, v, xt, vt, bad, rollbacks);
}

// dst[e * S + i] = src[e] for every instance i (state initialisation)
__global__ void k_replicate(const double4* __restrict__ src, double4* __restrict__ dst, int n, int S) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < (size_t)n * S) dst[i] = src[i / S];
}

void launch_replicate(cudaStream_t st, const double4* src, double4* dst, int n, int S) {
    const size_t tot = (size_t)n * S;
    if (tot == 0) return;
    k_replicate<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(src, dst, n, S);
}

// ----------------------------------------------------------------------------
// local step
// ----------------------------------------------------------------------------
// MUFU approximations with flush-to-zero semantics: the same hardware results as __fdividef /
// rsqrtf / __logf for normal inputs, without the denormal range-scaling fix-ups the non-ftz
// forms wrap around every MUFU (no denormal ever reaches them here).
__device__ __forceinline__ float rcp_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float log_ftz(float x) {   // ln x = log2(x) ln 2, as __logf
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * 0.693147180559945309f;
}

// Jacobi eigen-decomposition of a symmetric 3x3 (cyclic, Rutishauser rotations).
__device__ __forceinline__ void jacobi3(float S[3][3], float V[3][3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.f : 0.f;
#pragma unroll 1
    for (int sweep = 0; sweep < SIM_JACOBI_SWEEPS; ++sweep) {
        float off = fabsf(S[0][1]) + fabsf(S[0][2]) + fabsf(S[1][2]);
        float dia = fabsf(S[0][0]) + fabsf(S[1][1]) + fabsf(S[2][2]);
        if (off <= 1e-9f * dia) break;
#pragma unroll
        for (int pq = 0; pq < 3; ++pq) {
            const int p = pq == 2 ? 1 : 0;
            const int q = pq == 0 ? 1 : 2;
            const int r = 3 - p - q;
            float apq = S[p][q];
            if (fabsf(apq) <= 1e-30f) continue;
            // hardware-approximate reciprocal / square root (MUFU, ~1 ulp): no IEEE fix-up paths;
            // c and s come from the same t, so the rotation stays orthogonal to ~1e-7
            float theta = (S[q][q] - S[p][p]) * rcp_ftz(2.f * apq);
            float at = fabsf(theta);
            const float w = theta * theta + 1.f;
            float t = at > 1e15f ? 0.5f * rcp_ftz(at) : rcp_ftz(at + w * rsqrt_ftz(w));
            t = theta < 0.f ? -t : t;
            float c = rsqrt_ftz(t * t + 1.f);
            float s = t * c;
            S[p][p] -= t * apq;
            S[q][q] += t * apq;
            S[p][q] = S[q][p] = 0.f;
            float srp = S[r][p], srq = S[r][q];
            S[r][p] = S[p][r] = c * srp - s * srq;
            S[r][q] = S[q][r] = s * srp + c * srq;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                float vkp = V[k][p], vkq = V[k][q];
                V[k][p] = c * vkp - s * vkq;
                V[k][q] = s * vkp + c * vkq;
            }
        }
    }
}

__device__ __forceinline__ void swapcol(float V[3][3], float* e, int a, int b) {
    float t = e[a];
    e[a] = e[b];
    e[b] = t;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float u = V[k][a];
        V[k][a] = V[k][b];
        V[k][b] = u;
    }
}

// NH objective in sigma space: k/2|p-sig|^2 + mu/2(|p|^2-3) - mu lnJ + lam/2 ln^2 J
// (ln J = ln(p0 p1 p2): one hardware log2 instead of three IEEE logs)
__device__ __forceinline__ float nh_f(const float p[3], const float sg[3], float k, float mu, float lam,
                                     float lnJ) {
    float d0 = p[0] - sg[0], d1 = p[1] - sg[1], d2 = p[2] - sg[2];
    return 0.5f * k * (d0 * d0 + d1 * d1 + d2 * d2) +
           0.5f * mu * (p[0] * p[0] + p[1] * p[1] + p[2] * p[2] - 3.f) - mu * lnJ + 0.5f * lam * lnJ * lnJ;
}

// p* = argmin k/2|p - sig|^2 + psi(p)  (reading A2-A4); returns delta = p* - sig
__device__ __forceinline__ void project_sigma(int model, const float sg[3], float k, float mu, float lam,
                                              float d[3]) {
    if (model == 2) {   // ARAP: p* = 1
        d[0] = 1.f - sg[0];
        d[1] = 1.f - sg[1];
        d[2] = 1.f - sg[2];
        return;
    }
    if (model == 1) {   // linear corotated closed form
        float S = (k * (sg[0] + sg[1] + sg[2]) + 6.f * mu + 9.f * lam) / (k + 2.f * mu + 3.f * lam);
        float inv = 1.f / (k + 2.f * mu);
        // p_i - sig_i = (2mu(1 - sig_i) - lam(S - 3)) / (k + 2mu)
#pragma unroll
        for (int i = 0; i < 3; ++i) d[i] = (2.f * mu * (1.f - sg[i]) - lam * (S - 3.f)) * inv;
        return;
    }
    // Neo-Hookean: damped Newton, <= 16 iterations, from the linear-corotated minimiser (the same
    // Hessian 2 mu I + lam 1 1^T at p = 1, so it is NH's first-order solution), floored at 0.05
    float p[3];
    {
        const float Sp = (k * (sg[0] + sg[1] + sg[2]) + 6.f * mu + 9.f * lam) * rcp_ftz(k + 2.f * mu + 3.f * lam);
        const float inv = rcp_ftz(k + 2.f * mu);
#pragma unroll
        for (int i = 0; i < 3; ++i) p[i] = fmaxf(sg[i] + (2.f * mu * (1.f - sg[i]) - lam * (Sp - 3.f)) * inv, 0.05f);
    }
    float scale = fmaxf(1.f, sqrtf(sg[0] * sg[0] + sg[1] * sg[1] + sg[2] * sg[2]));
    const float gtol = 2e-6f * k * scale;
    // ln J and the objective at p are carried from the accepted line-search point
    float lnJ = log_ftz(p[0] * p[1] * p[2]);
    float f0 = nh_f(p, sg, k, mu, lam, lnJ);
#pragma unroll 1
    for (int it = 0; it < 16; ++it) {
        float iv[3] = {rcp_ftz(p[0]), rcp_ftz(p[1]), rcp_ftz(p[2])};
        float g[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) g[i] = k * (p[i] - sg[i]) + mu * p[i] - mu * iv[i] + lam * lnJ * iv[i];
        if (g[0] * g[0] + g[1] * g[1] + g[2] * g[2] <= gtol * gtol) break;   // |g| <= gtol
        float H[3][3];
        float dg = mu - lam * lnJ;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) H[i][j] = lam * iv[i] * iv[j] + (i == j ? (k + mu + dg * iv[i] * iv[i]) : 0.f);
        // Cramer solve H dd = -g
        float c00 = H[1][1] * H[2][2] - H[1][2] * H[2][1];
        float c01 = H[1][2] * H[2][0] - H[1][0] * H[2][2];
        float c02 = H[1][0] * H[2][1] - H[1][1] * H[2][0];
        float det = H[0][0] * c00 + H[0][1] * c01 + H[0][2] * c02;
        float dd[3];
        bool ok = fabsf(det) > 0.f && isfinite(det);
        if (ok) {
            float id = rcp_ftz(det);
            float c10 = H[0][2] * H[2][1] - H[0][1] * H[2][2];
            float c11 = H[0][0] * H[2][2] - H[0][2] * H[2][0];
            float c12 = H[0][1] * H[2][0] - H[0][0] * H[2][1];
            float c20 = H[0][1] * H[1][2] - H[0][2] * H[1][1];
            float c21 = H[0][2] * H[1][0] - H[0][0] * H[1][2];
            float c22 = H[0][0] * H[1][1] - H[0][1] * H[1][0];
            dd[0] = -(c00 * g[0] + c10 * g[1] + c20 * g[2]) * id;
            dd[1] = -(c01 * g[0] + c11 * g[1] + c21 * g[2]) * id;
            dd[2] = -(c02 * g[0] + c12 * g[1] + c22 * g[2]) * id;
            float slope = dd[0] * g[0] + dd[1] * g[1] + dd[2] * g[2];
            ok = slope < 0.f && isfinite(slope);
        }
        if (!ok) {
            float s = -rcp_ftz(k + mu);
            dd[0] = s * g[0];
            dd[1] = s * g[1];
            dd[2] = s * g[2];
        }
        float slope = dd[0] * g[0] + dd[1] * g[1] + dd[2] * g[2];
        float fr = 2e-6f * (k * (p[0] * p[0] + p[1] * p[1] + p[2] * p[2] + sg[0] * sg[0] + sg[1] * sg[1] +
                                 sg[2] * sg[2]) + mu * fabsf(lnJ) + lam * lnJ * lnJ + mu);
        float t = 1.f;
        bool acc = false;
#pragma unroll 1
        for (int ls = 0; ls < 40; ++ls) {
            float pn[3] = {p[0] + t * dd[0], p[1] + t * dd[1], p[2] + t * dd[2]};
            if (pn[0] > 0.f && pn[1] > 0.f && pn[2] > 0.f) {
                const float lnJn = log_ftz(pn[0] * pn[1] * pn[2]);
                const float fn = nh_f(pn, sg, k, mu, lam, lnJn);
                if (fn <= f0 + 1e-4f * t * slope + fr) {
                    acc = true;
                    lnJ = lnJn;
                    f0 = fn;
                    break;
                }
            }
            t *= 0.5f;
        }
        p[0] += t * dd[0];
        p[1] += t * dd[1];
        p[2] += t * dd[2];
        if (!acc) {   // line search exhausted: tiny step, re-evaluate at the new point
            lnJ = log_ftz(p[0] * p[1] * p[2]);
            f0 = nh_f(p, sg, k, mu, lam, lnJ);
        }
    }
    d[0] = p[0] - sg[0];
    d[1] = p[1] - sg[1];
    d[2] = p[2] - sg[2];
}

// one thread per (tet, instance), instance-minor: the instances of one tet share its rest
// data (broadcast loads) and read consecutive state entries.  f_a = h^2 w (P - F) g_a per corner
// ADMM-PD (du != nullptr; Overby et al. 2017): project F + u, u <- u + F - P = -(P - F - u),
// and the global step targets P - u_new, i.e. the force block is h^2 w (2 (P - F - u) + u) g_a.
// du is [9][n_t S] (plane per entry, instance-minor); admm_first: u = 0 (reading A33, reset per frame).
// One instantiation per material: the closed forms (corotated, ARAP) fit 64 registers (8 CTAs of
// 128 threads per SM), the NH Newton 80 (6 CTAs); measured 20 % / 7 % faster than 94 registers.
// Local step core (readings A2-A5): signed SVD F = U diag(sg) V^T (Jacobi on F^T F,
// U by Gram-Schmidt on F V, both in SO(3)) and the sigma-space projection; dlt = p* - sg, so
// P - F = U diag(dlt) V^T without cancellation.
template <int MODEL>
__device__ __forceinline__ void svd_project(const float F[3][3], float k, float mu, float lam, float U[3][3],
                                            float dlt[3], float V[3][3]) {
    // S = F^T F, eigenvectors V
    float S[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) S[i][j] = F[0][i] * F[0][j] + F[1][i] * F[1][j] + F[2][i] * F[2][j];
    jacobi3(S, V);
    float ev[3] = {S[0][0], S[1][1], S[2][2]};
    if (ev[0] < ev[1]) swapcol(V, ev, 0, 1);
    if (ev[0] < ev[2]) swapcol(V, ev, 0, 2);
    if (ev[1] < ev[2]) swapcol(V, ev, 1, 2);
    float detV = V[0][0] * (V[1][1] * V[2][2] - V[1][2] * V[2][1]) - V[0][1] * (V[1][0] * V[2][2] - V[1][2] * V[2][0]) +
                 V[0][2] * (V[1][0] * V[2][1] - V[1][1] * V[2][0]);
    if (detV < 0.f) {
        V[0][2] = -V[0][2];
        V[1][2] = -V[1][2];
        V[2][2] = -V[2][2];
    }
    // U by Gram-Schmidt on F V (U in SO(3)); signed singular values sg_i = u_i . F v_i
    float FV[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) FV[i][j] = F[i][0] * V[0][j] + F[i][1] * V[1][j] + F[i][2] * V[2][j];
    const float q0 = FV[0][0] * FV[0][0] + FV[1][0] * FV[1][0] + FV[2][0] * FV[2][0];
    float n0 = q0 > 0.f ? q0 * rsqrt_ftz(q0) : 0.f;
    if (q0 > 1e-36f) {
        const float r0 = rsqrt_ftz(q0);
        U[0][0] = FV[0][0] * r0; U[1][0] = FV[1][0] * r0; U[2][0] = FV[2][0] * r0;
    } else {
        U[0][0] = 1.f; U[1][0] = 0.f; U[2][0] = 0.f;
    }
    float dt = U[0][0] * FV[0][1] + U[1][0] * FV[1][1] + U[2][0] * FV[2][1];
    float w0 = FV[0][1] - dt * U[0][0], w1 = FV[1][1] - dt * U[1][0], w2 = FV[2][1] - dt * U[2][0];
    const float q1 = w0 * w0 + w1 * w1 + w2 * w2;
    float n1 = q1 > 0.f ? q1 * rsqrt_ftz(q1) : 0.f;
    if (n1 > 1e-30f * fmaxf(1.f, n0)) {
        const float r1 = rsqrt_ftz(q1);
        U[0][1] = w0 * r1; U[1][1] = w1 * r1; U[2][1] = w2 * r1;
    } else {   // any unit vector orthogonal to u0
        float a0 = U[0][0], a1 = U[1][0], a2 = U[2][0];
        float e0 = fabsf(a0) < 0.577f ? 1.f : 0.f, e1 = e0 == 0.f && fabsf(a1) < 0.577f ? 1.f : 0.f;
        float e2 = (e0 == 0.f && e1 == 0.f) ? 1.f : 0.f;
        float dp = a0 * e0 + a1 * e1 + a2 * e2;
        w0 = e0 - dp * a0; w1 = e1 - dp * a1; w2 = e2 - dp * a2;
        n1 = sqrtf(w0 * w0 + w1 * w1 + w2 * w2);
        U[0][1] = w0 / n1; U[1][1] = w1 / n1; U[2][1] = w2 / n1;
    }
    U[0][2] = U[1][0] * U[2][1] - U[2][0] * U[1][1];
    U[1][2] = U[2][0] * U[0][1] - U[0][0] * U[2][1];
    U[2][2] = U[0][0] * U[1][1] - U[1][0] * U[0][1];
    float sg[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) sg[j] = U[0][j] * FV[0][j] + U[1][j] * FV[1][j] + U[2][j] * FV[2][j];
    project_sigma(MODEL, sg, k, mu, lam, dlt);
}

template <int MODEL>
#ifndef SIM_LOCAL_THREADS
#define SIM_LOCAL_THREADS 128
#endif
__global__ void __launch_bounds__(SIM_LOCAL_THREADS, (MODEL == 0 ? 6 : 8) * 128 / SIM_LOCAL_THREADS) k_local(Params P, const int4* __restrict__ tet, const float* __restrict__ Bm,
                                               const float* __restrict__ hw2, const double4* __restrict__ x,
                                               float* __restrict__ fc, float* __restrict__ Pdbg,
                                               float* __restrict__ du, int admm_first) {
    pdl_enter();
    const int SI = P.S;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    if (gt >= P.n_t * SI) return;
    const int t = gt / SI, inst = gt - t * SI;
    const int nt = P.n_t;
    int4 tv = __ldg(&tet[t]);
    double4 x0 = x[tv.x * SI + inst], x1 = x[tv.y * SI + inst], x2 = x[tv.z * SI + inst], x3 = x[tv.w * SI + inst];
    // Ds columns (fp64 differences, then fp32)
    float D[3][3];
    D[0][0] = (float)(x1.x - x0.x); D[1][0] = (float)(x1.y - x0.y); D[2][0] = (float)(x1.z - x0.z);
    D[0][1] = (float)(x2.x - x0.x); D[1][1] = (float)(x2.y - x0.y); D[2][1] = (float)(x2.z - x0.z);
    D[0][2] = (float)(x3.x - x0.x); D[1][2] = (float)(x3.y - x0.y); D[2][2] = (float)(x3.z - x0.z);
    float B[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) B[e] = __ldg(&Bm[(size_t)e * nt + t]);
    float F[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) F[i][j] = D[i][0] * B[0 * 3 + j] + D[i][1] * B[1 * 3 + j] + D[i][2] * B[2 * 3 + j];
    float uo[9];
    const size_t plane = (size_t)nt * SI;
    if (du) {
#pragma unroll
        for (int e = 0; e < 9; ++e) uo[e] = admm_first ? 0.f : du[e * plane + gt];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) F[i][j] += uo[3 * i + j];   // project F + u
    }
    float U[3][3], V[3][3], dlt[3];
    svd_project<MODEL>(F, P.k, P.mu, P.lam, U, dlt, V);
    // Q = hw2 * U diag(delta) V^T  (= h^2 w (P - F); ADMM: h^2 w (2 (P - F - u) + u))
    float hw = __ldg(&hw2[t]);
    float Q[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Q[i][j] = U[i][0] * dlt[0] * V[j][0] + U[i][1] * dlt[1] * V[j][1] + U[i][2] * dlt[2] * V[j][2];
    if (du) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                du[(3 * i + j) * plane + gt] = -Q[i][j];   // u_new = u + F - P = -(P - F - u)
                Q[i][j] = 2.f * Q[i][j] + uo[3 * i + j];
            }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) Q[i][j] *= hw;
    if (Pdbg) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                Pdbg[(size_t)t * 9 + 3 * i + j] =
                    F[i][j] + (U[i][0] * dlt[0] * V[j][0] + U[i][1] * dlt[1] * V[j][1] + U[i][2] * dlt[2] * V[j][2]);
    }
    // f_a = Q g_a, g_a = row a-1 of Bm (a = 1..3), f_0 = -sum
    float f[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i) f[a][i] = Q[i][0] * B[3 * a + 0] + Q[i][1] * B[3 * a + 1] + Q[i][2] * B[3 * a + 2];
    float* o = fc + 12 * (size_t)t * SI + inst;   // [tet][corner][component][instance], no padding
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        o[i * SI] = -(f[0][i] + f[1][i] + f[2][i]);
#pragma unroll
        for (int a = 0; a < 3; ++a) o[(3 * (a + 1) + i) * SI] = f[a][i];
    }
}

// ----------------------------------------------------------------------------
// Paired local step (S > 1, S even, plain PD): one thread computes the same tet for two
// instances with Blackwell's packed FP32 (FFMA2 / FMUL2 / FADD2 on float2 pairs), halving the
// FP32 instructions of the SVD and the projection, which issue-bound the scalar kernel.  The two
// lanes run in lockstep: a lane that has converged (Jacobi sweep, Newton step, line search)
// takes a null update (rotation t = 0, step dd = 0), which leaves its values exactly as the
// scalar kernel's early exit would; per-lane MUFU (rcp, rsqrt, lg2) stay scalar.
// ----------------------------------------------------------------------------
struct v2 {
    float2 a;
    __device__ __forceinline__ v2() {}
    __device__ __forceinline__ v2(float s) : a(make_float2(s, s)) {}
    __device__ __forceinline__ v2(float x, float y) : a(make_float2(x, y)) {}
    __device__ __forceinline__ v2(float2 q) : a(q) {}
};
__device__ __forceinline__ v2 operator+(v2 p, v2 q) { return v2(__fadd2_rn(p.a, q.a)); }
__device__ __forceinline__ v2 operator-(v2 p, v2 q) { return v2(__ffma2_rn(q.a, make_float2(-1.f, -1.f), p.a)); }
__device__ __forceinline__ v2 operator*(v2 p, v2 q) { return v2(__fmul2_rn(p.a, q.a)); }
__device__ __forceinline__ v2 fma2(v2 p, v2 q, v2 r) { return v2(__ffma2_rn(p.a, q.a, r.a)); }   // p q + r
__device__ __forceinline__ v2 rcp2(v2 p) { return v2(rcp_ftz(p.a.x), rcp_ftz(p.a.y)); }
__device__ __forceinline__ v2 rsqrt2(v2 p) { return v2(rsqrt_ftz(p.a.x), rsqrt_ftz(p.a.y)); }
__device__ __forceinline__ v2 log2v(v2 p) { return v2(log_ftz(p.a.x), log_ftz(p.a.y)); }
__device__ __forceinline__ v2 abs2(v2 p) { return v2(fabsf(p.a.x), fabsf(p.a.y)); }
__device__ __forceinline__ v2 sel2(bool bx, bool by, v2 p, v2 q) { return v2(bx ? p.a.x : q.a.x, by ? p.a.y : q.a.y); }

__device__ __forceinline__ void jacobi3_2(v2 S[3][3], v2 V[3][3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) V[i][j] = v2(i == j ? 1.f : 0.f);
#pragma unroll 1
    for (int sweep = 0; sweep < SIM_JACOBI_SWEEPS; ++sweep) {
        const v2 off = abs2(S[0][1]) + abs2(S[0][2]) + abs2(S[1][2]);
        const v2 dia = abs2(S[0][0]) + abs2(S[1][1]) + abs2(S[2][2]);
        const bool cx = off.a.x <= 1e-9f * dia.a.x, cy = off.a.y <= 1e-9f * dia.a.y;   // lane converged
        if (cx && cy) break;
#pragma unroll
        for (int pq = 0; pq < 3; ++pq) {
            const int p = pq == 2 ? 1 : 0;
            const int q = pq == 0 ? 1 : 2;
            const int r = 3 - p - q;
            const v2 apq = S[p][q];
            // rotate this lane (|a_pq| > 1e-18 keeps 4 a_pq^2 a normal fp32 number)
            const bool rx = !cx && fabsf(apq.a.x) > 1e-18f, ry = !cy && fabsf(apq.a.y) > 1e-18f;
            // t = tan(phi), the smaller root of t^2 + 2 theta t - 1 = 0 with theta = d / (2 a_pq),
            // d = a_qq - a_pp, written without theta: t = sgn(d) 2 a_pq / (|d| + sqrt(d^2 + 4 a_pq^2))
            // (two MUFU operations per lane instead of three, no overflow branch)
            const v2 d = S[q][q] - S[p][p];
            const v2 a2 = apq + apq;
            const v2 rr = fma2(d, d, a2 * a2);
            v2 t = a2 * rcp2(fma2(rr, rsqrt2(rr), abs2(d)));
            t = sel2(d.a.x < 0.f, d.a.y < 0.f, v2(-t.a.x, -t.a.y), t);
            t = sel2(rx, ry, t, v2(0.f));   // null rotation (c = 1, s = 0) for a lane that skips
            const v2 c = rsqrt2(fma2(t, t, v2(1.f)));
            const v2 sn = t * c;
            const v2 nsn(-sn.a.x, -sn.a.y);
            const v2 ta = t * apq;
            S[p][p] = S[p][p] - ta;
            S[q][q] = S[q][q] + ta;
            S[p][q] = S[q][p] = sel2(rx, ry, v2(0.f), apq);
            const v2 srp = S[r][p], srq = S[r][q];
            S[r][p] = S[p][r] = fma2(nsn, srq, c * srp);
            S[r][q] = S[q][r] = fma2(sn, srp, c * srq);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const v2 vkp = V[k][p], vkq = V[k][q];
                V[k][p] = fma2(nsn, vkq, c * vkp);
                V[k][q] = fma2(sn, vkp, c * vkq);
            }
        }
    }
}

// lane-wise column swap of V and the eigenvalue list (the descending sort of the scalar kernel)
__device__ __forceinline__ void swapcol2(v2 V[3][3], v2* e, int a, int b, bool sx, bool sy) {
    const v2 ea = e[a], eb = e[b];
    e[a] = sel2(sx, sy, eb, ea);
    e[b] = sel2(sx, sy, ea, eb);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const v2 u = V[k][a], w = V[k][b];
        V[k][a] = sel2(sx, sy, w, u);
        V[k][b] = sel2(sx, sy, u, w);
    }
}

__device__ __forceinline__ v2 nh_f2(const v2 p[3], const v2 sg[3], v2 k, v2 mu, v2 lam, v2 lnJ) {
    const v2 d0 = p[0] - sg[0], d1 = p[1] - sg[1], d2 = p[2] - sg[2];
    const v2 dd = fma2(d0, d0, fma2(d1, d1, d2 * d2));
    const v2 pp = fma2(p[0], p[0], fma2(p[1], p[1], p[2] * p[2])) - v2(3.f);
    return fma2(v2(0.5f) * k, dd, fma2(v2(0.5f) * mu, pp, fma2(v2(0.5f) * lam, lnJ * lnJ, v2(0.f) - mu * lnJ)));
}

template <int MODEL>
__device__ __forceinline__ void project_sigma2(const v2 sg[3], float kf, float muf, float lamf, v2 d[3]) {
    const v2 k(kf), mu(muf), lam(lamf);
    if (MODEL == 2) {
#pragma unroll
        for (int i = 0; i < 3; ++i) d[i] = v2(1.f) - sg[i];
        return;
    }
    const v2 Sp = fma2(k, sg[0] + sg[1] + sg[2], v2(6.f * muf + 9.f * lamf)) * v2(MODEL == 1 ? 1.f / (kf + 2.f * muf + 3.f * lamf) : rcp_ftz(kf + 2.f * muf + 3.f * lamf));
    const v2 inv(MODEL == 1 ? 1.f / (kf + 2.f * muf) : rcp_ftz(kf + 2.f * muf));
    const v2 lS3 = lam * (Sp - v2(3.f));
    if (MODEL == 1) {   // linear corotated closed form
#pragma unroll
        for (int i = 0; i < 3; ++i) d[i] = (fma2(v2(2.f) * mu, v2(1.f) - sg[i], v2(0.f) - lS3)) * inv;
        return;
    }
    // Neo-Hookean: damped Newton from the linear-corotated minimiser (floored at 0.05), lockstep lanes
    v2 p[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        p[i] = sg[i] + fma2(v2(2.f) * mu, v2(1.f) - sg[i], v2(0.f) - lS3) * inv;
        p[i] = v2(fmaxf(p[i].a.x, 0.05f), fmaxf(p[i].a.y, 0.05f));
    }
    const v2 sn2 = fma2(sg[0], sg[0], fma2(sg[1], sg[1], sg[2] * sg[2]));
    const v2 scale(fmaxf(1.f, sqrtf(sn2.a.x)), fmaxf(1.f, sqrtf(sn2.a.y)));
    const v2 gtol = v2(2e-6f * kf) * scale;
    const v2 gtol2 = gtol * gtol;
    v2 lnJ = log2v(p[0] * p[1] * p[2]);
    v2 f0 = nh_f2(p, sg, k, mu, lam, lnJ);
#pragma unroll 1
    for (int it = 0; it < 16; ++it) {
        const v2 iv[3] = {rcp2(p[0]), rcp2(p[1]), rcp2(p[2])};
        v2 g[3];
        const v2 kmu = k + mu;
#pragma unroll
        for (int i = 0; i < 3; ++i) g[i] = fma2(kmu, p[i], fma2(lam * lnJ - mu, iv[i], v2(0.f) - k * sg[i]));
        const v2 gg = fma2(g[0], g[0], fma2(g[1], g[1], g[2] * g[2]));
        const bool dx = gg.a.x <= gtol2.a.x, dy = gg.a.y <= gtol2.a.y;   // lane converged (|g| <= gtol)
        if (dx && dy) break;
        v2 H[3][3];
        const v2 dg = mu - lam * lnJ;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) H[i][j] = i == j ? fma2(lam * iv[i], iv[j], fma2(dg * iv[i], iv[i], kmu)) : lam * iv[i] * iv[j];
        const v2 c00 = fma2(H[1][1], H[2][2], v2(0.f) - H[1][2] * H[2][1]);
        const v2 c01 = fma2(H[1][2], H[2][0], v2(0.f) - H[1][0] * H[2][2]);
        const v2 c02 = fma2(H[1][0], H[2][1], v2(0.f) - H[1][1] * H[2][0]);
        const v2 det = fma2(H[0][0], c00, fma2(H[0][1], c01, H[0][2] * c02));
        const v2 id = rcp2(det);
        const v2 c10 = fma2(H[0][2], H[2][1], v2(0.f) - H[0][1] * H[2][2]);
        const v2 c11 = fma2(H[0][0], H[2][2], v2(0.f) - H[0][2] * H[2][0]);
        const v2 c12 = fma2(H[0][1], H[2][0], v2(0.f) - H[0][0] * H[2][1]);
        const v2 c20 = fma2(H[0][1], H[1][2], v2(0.f) - H[0][2] * H[1][1]);
        const v2 c21 = fma2(H[0][2], H[1][0], v2(0.f) - H[0][0] * H[1][2]);
        const v2 c22 = fma2(H[0][0], H[1][1], v2(0.f) - H[0][1] * H[1][0]);
        v2 dd[3];
        dd[0] = v2(0.f) - fma2(c00, g[0], fma2(c10, g[1], c20 * g[2])) * id;
        dd[1] = v2(0.f) - fma2(c01, g[0], fma2(c11, g[1], c21 * g[2])) * id;
        dd[2] = v2(0.f) - fma2(c02, g[0], fma2(c12, g[1], c22 * g[2])) * id;
        v2 slope = fma2(dd[0], g[0], fma2(dd[1], g[1], dd[2] * g[2]));
        // Newton direction unusable (singular or not a descent direction): scaled gradient step
        const bool okx = fabsf(det.a.x) > 0.f && isfinite(det.a.x) && slope.a.x < 0.f && isfinite(slope.a.x);
        const bool oky = fabsf(det.a.y) > 0.f && isfinite(det.a.y) && slope.a.y < 0.f && isfinite(slope.a.y);
        const v2 sgd(-rcp_ftz(kf + muf));
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            dd[i] = sel2(okx, oky, dd[i], sgd * g[i]);
            dd[i] = sel2(dx, dy, v2(0.f), dd[i]);   // a converged lane stays where it is
        }
        slope = fma2(dd[0], g[0], fma2(dd[1], g[1], dd[2] * g[2]));
        const v2 fr = v2(2e-6f) * fma2(k, fma2(p[0], p[0], fma2(p[1], p[1], fma2(p[2], p[2], sn2))),
                                       fma2(mu, abs2(lnJ), fma2(lam * lnJ, lnJ, mu)));
        v2 t(1.f);
        bool ax = dx, ay = dy;                   // accepted
        bool tx = dx, ty = dy;                   // any accepted point (a converged lane keeps its state)
#pragma unroll 1
        for (int ls = 0; ls < 40; ++ls) {
            v2 pn[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) pn[i] = fma2(t, dd[i], p[i]);
            const bool vx = pn[0].a.x > 0.f && pn[1].a.x > 0.f && pn[2].a.x > 0.f;
            const bool vy = pn[0].a.y > 0.f && pn[1].a.y > 0.f && pn[2].a.y > 0.f;
            const v2 prod = pn[0] * pn[1] * pn[2];
            const v2 lnJn = v2(vx && !ax ? log_ftz(prod.a.x) : 0.f, vy && !ay ? log_ftz(prod.a.y) : 0.f);
            const v2 fn = nh_f2(pn, sg, k, mu, lam, lnJn);
            const v2 bound = fma2(v2(1e-4f) * t, slope, f0 + fr);
            const bool nx = !ax && vx && fn.a.x <= bound.a.x, ny = !ay && vy && fn.a.y <= bound.a.y;
            if (nx) { lnJ.a.x = lnJn.a.x; f0.a.x = fn.a.x; ax = true; tx = true; }
            if (ny) { lnJ.a.y = lnJn.a.y; f0.a.y = fn.a.y; ay = true; ty = true; }
            if (ax && ay) break;
            if (!ax) t.a.x *= 0.5f;
            if (!ay) t.a.y *= 0.5f;
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) p[i] = fma2(t, dd[i], p[i]);
        if (!tx) { lnJ.a.x = log_ftz(p[0].a.x * p[1].a.x * p[2].a.x); }
        if (!ty) { lnJ.a.y = log_ftz(p[0].a.y * p[1].a.y * p[2].a.y); }
        if (!tx || !ty) {
            const v2 fre = nh_f2(p, sg, k, mu, lam, lnJ);
            if (!tx) f0.a.x = fre.a.x;
            if (!ty) f0.a.y = fre.a.y;
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = p[i] - sg[i];
}

template <int MODEL>
#ifndef SIM_LOCAL2_MINB
#define SIM_LOCAL2_MINB 5
#endif
#ifndef SIM_LOCAL2_THREADS
#define SIM_LOCAL2_THREADS 32   // one warp per CTA, 20 CTAs per SM (64 / 128 / 256: 0.7 / 2.1 / 7 % slower)
#endif
__global__ void __launch_bounds__(SIM_LOCAL2_THREADS, MODEL == 0 ? SIM_LOCAL2_MINB * 128 / SIM_LOCAL2_THREADS : 6 * 128 / SIM_LOCAL2_THREADS) k_local2(Params P, const int4* __restrict__ tet,
                                                                     const float* __restrict__ Bm,
                                                                     const float* __restrict__ hw2,
                                                                     const double4* __restrict__ x, float* __restrict__ fc) {
    pdl_enter();
    const int SI = P.S, half = SI >> 1;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    if (gt >= P.n_t * half) return;
    const int t = gt / half, inst = 2 * (gt - t * half);   // instances inst, inst + 1
    const int nt = P.n_t;
    const int4 tv = __ldg(&tet[t]);
    v2 D[3][3];
    {
        const double4 a0 = x[tv.x * SI + inst], a1 = x[tv.y * SI + inst], a2 = x[tv.z * SI + inst], a3 = x[tv.w * SI + inst];
        const double4 b0 = x[tv.x * SI + inst + 1], b1 = x[tv.y * SI + inst + 1], b2 = x[tv.z * SI + inst + 1],
                      b3 = x[tv.w * SI + inst + 1];
        D[0][0] = v2((float)(a1.x - a0.x), (float)(b1.x - b0.x)); D[1][0] = v2((float)(a1.y - a0.y), (float)(b1.y - b0.y));
        D[2][0] = v2((float)(a1.z - a0.z), (float)(b1.z - b0.z));
        D[0][1] = v2((float)(a2.x - a0.x), (float)(b2.x - b0.x)); D[1][1] = v2((float)(a2.y - a0.y), (float)(b2.y - b0.y));
        D[2][1] = v2((float)(a2.z - a0.z), (float)(b2.z - b0.z));
        D[0][2] = v2((float)(a3.x - a0.x), (float)(b3.x - b0.x)); D[1][2] = v2((float)(a3.y - a0.y), (float)(b3.y - b0.y));
        D[2][2] = v2((float)(a3.z - a0.z), (float)(b3.z - b0.z));
    }
    float B[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) B[e] = __ldg(&Bm[(size_t)e * nt + t]);
    v2 F[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) F[i][j] = fma2(D[i][0], v2(B[j]), fma2(D[i][1], v2(B[3 + j]), D[i][2] * v2(B[6 + j])));
    v2 S[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) S[i][j] = fma2(F[0][i], F[0][j], fma2(F[1][i], F[1][j], F[2][i] * F[2][j]));
    v2 V[3][3];
    jacobi3_2(S, V);
    v2 ev[3] = {S[0][0], S[1][1], S[2][2]};
    swapcol2(V, ev, 0, 1, ev[0].a.x < ev[1].a.x, ev[0].a.y < ev[1].a.y);
    swapcol2(V, ev, 0, 2, ev[0].a.x < ev[2].a.x, ev[0].a.y < ev[2].a.y);
    swapcol2(V, ev, 1, 2, ev[1].a.x < ev[2].a.x, ev[1].a.y < ev[2].a.y);
    {
        const v2 detV = fma2(V[0][0], fma2(V[1][1], V[2][2], v2(0.f) - V[1][2] * V[2][1]),
                             fma2(v2(0.f) - V[0][1], fma2(V[1][0], V[2][2], v2(0.f) - V[1][2] * V[2][0]),
                                  V[0][2] * fma2(V[1][0], V[2][1], v2(0.f) - V[1][1] * V[2][0])));
        const v2 sgn(detV.a.x < 0.f ? -1.f : 1.f, detV.a.y < 0.f ? -1.f : 1.f);
        V[0][2] = V[0][2] * sgn; V[1][2] = V[1][2] * sgn; V[2][2] = V[2][2] * sgn;
    }
    v2 FV[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) FV[i][j] = fma2(F[i][0], V[0][j], fma2(F[i][1], V[1][j], F[i][2] * V[2][j]));
    // U by Gram-Schmidt on F V (lane-wise fallbacks for degenerate columns, as the scalar kernel)
    v2 U[3][3];
    const v2 q0 = fma2(FV[0][0], FV[0][0], fma2(FV[1][0], FV[1][0], FV[2][0] * FV[2][0]));
    const v2 r0 = rsqrt2(q0);
    const v2 n0 = sel2(q0.a.x > 0.f, q0.a.y > 0.f, q0 * r0, v2(0.f));
    const bool u0x = q0.a.x > 1e-36f, u0y = q0.a.y > 1e-36f;
    U[0][0] = sel2(u0x, u0y, FV[0][0] * r0, v2(1.f));
    U[1][0] = sel2(u0x, u0y, FV[1][0] * r0, v2(0.f));
    U[2][0] = sel2(u0x, u0y, FV[2][0] * r0, v2(0.f));
    const v2 dt = fma2(U[0][0], FV[0][1], fma2(U[1][0], FV[1][1], U[2][0] * FV[2][1]));
    v2 w0 = FV[0][1] - dt * U[0][0], w1 = FV[1][1] - dt * U[1][0], w2 = FV[2][1] - dt * U[2][0];
    const v2 q1 = fma2(w0, w0, fma2(w1, w1, w2 * w2));
    const v2 r1 = rsqrt2(q1);
    const v2 n1 = sel2(q1.a.x > 0.f, q1.a.y > 0.f, q1 * r1, v2(0.f));
    const bool u1x = n1.a.x > 1e-30f * fmaxf(1.f, n0.a.x), u1y = n1.a.y > 1e-30f * fmaxf(1.f, n0.a.y);
    U[0][1] = w0 * r1; U[1][1] = w1 * r1; U[2][1] = w2 * r1;
    if (!u1x || !u1y) {   // any unit vector orthogonal to u0 (rare), lane by lane
#pragma unroll
        for (int l = 0; l < 2; ++l) {
            if (l == 0 ? u1x : u1y) continue;
            const float a0 = l == 0 ? U[0][0].a.x : U[0][0].a.y, a1 = l == 0 ? U[1][0].a.x : U[1][0].a.y,
                        a2 = l == 0 ? U[2][0].a.x : U[2][0].a.y;
            const float e0 = fabsf(a0) < 0.577f ? 1.f : 0.f, e1 = e0 == 0.f && fabsf(a1) < 0.577f ? 1.f : 0.f;
            const float e2 = (e0 == 0.f && e1 == 0.f) ? 1.f : 0.f;
            const float dp = a0 * e0 + a1 * e1 + a2 * e2;
            const float z0 = e0 - dp * a0, z1 = e1 - dp * a1, z2 = e2 - dp * a2;
            const float nz = sqrtf(z0 * z0 + z1 * z1 + z2 * z2);
            if (l == 0) {
                U[0][1].a.x = z0 / nz; U[1][1].a.x = z1 / nz; U[2][1].a.x = z2 / nz;
            } else {
                U[0][1].a.y = z0 / nz; U[1][1].a.y = z1 / nz; U[2][1].a.y = z2 / nz;
            }
        }
    }
    U[0][2] = fma2(U[1][0], U[2][1], v2(0.f) - U[2][0] * U[1][1]);
    U[1][2] = fma2(U[2][0], U[0][1], v2(0.f) - U[0][0] * U[2][1]);
    U[2][2] = fma2(U[0][0], U[1][1], v2(0.f) - U[1][0] * U[0][1]);
    v2 sg[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) sg[j] = fma2(U[0][j], FV[0][j], fma2(U[1][j], FV[1][j], U[2][j] * FV[2][j]));
    v2 dlt[3];
    project_sigma2<MODEL>(sg, P.k, P.mu, P.lam, dlt);
    const v2 hw(__ldg(&hw2[t]));
    v2 Q[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Q[i][j] = hw * fma2(U[i][0] * dlt[0], V[j][0], fma2(U[i][1] * dlt[1], V[j][1], U[i][2] * dlt[2] * V[j][2]));
    float2* o = reinterpret_cast<float2*>(fc + 12 * (size_t)t * SI + inst);   // [tet][corner][xyz][instance]
    const int ss = SI >> 1;                                                    // float2 stride of one plane
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        v2 sum(0.f);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const v2 fa = fma2(Q[i][0], v2(B[3 * a]), fma2(Q[i][1], v2(B[3 * a + 1]), Q[i][2] * v2(B[3 * a + 2])));
            o[(3 * (a + 1) + i) * ss] = fa.a;
            sum = sum + fa;
        }
        o[i * ss] = make_float2(-sum.a.x, -sum.a.y);
    }
}

void launch_local(cudaStream_t st, const Params& P, const int4* tet, const float* Bm, const float* hw2,
                  const double4* x, float* fc, float* Pdbg, float* du, int admm_first) {
    if (P.S > 1 && (P.S & 1) == 0 && !du && !Pdbg && P.pair_local) {   // packed-FP32 pairs of instances
        const unsigned g2 = (unsigned)((P.n_t * (size_t)(P.S / 2) + SIM_LOCAL2_THREADS - 1) / SIM_LOCAL2_THREADS);
        if (P.model == 1)
            launch_pdl(k_local2<1>, dim3(g2), dim3(SIM_LOCAL2_THREADS), 0, st, P, tet, Bm, hw2, x, fc);
        else if (P.model == 2)
            launch_pdl(k_local2<2>, dim3(g2), dim3(SIM_LOCAL2_THREADS), 0, st, P, tet, Bm, hw2, x, fc);
        else
            launch_pdl(k_local2<0>, dim3(g2), dim3(SIM_LOCAL2_THREADS), 0, st, P, tet, Bm, hw2, x, fc);
        return;
    }
    const unsigned g = (unsigned)((P.n_t * (size_t)P.S + SIM_LOCAL_THREADS - 1) / SIM_LOCAL_THREADS);
    if (P.model == 1)
        launch_pdl(k_local<1>, dim3(g), dim3(SIM_LOCAL_THREADS), 0, st, P, tet, Bm, hw2, x, fc, Pdbg, du, admm_first);
    else if (P.model == 2)
        launch_pdl(k_local<2>, dim3(g), dim3(SIM_LOCAL_THREADS), 0, st, P, tet, Bm, hw2, x, fc, Pdbg, du, admm_first);
    else
        launch_pdl(k_local<0>, dim3(g), dim3(SIM_LOCAL_THREADS), 0, st, P, tet, Bm, hw2, x, fc, Pdbg, du, admm_first);
}

// ----------------------------------------------------------------------------
// Persistent small-scene driver (SURVEY §7 step 9, cfg1-class scenes): ONE launch runs `frames`
// frames x `iters` L-G iterations of Alg. 4 for a single contact-free instance in
// one CTA -- predict, local step (svd_project), RHS gather, y = K u and
// x += K^T y (K row- and column-major values-only, Theorem 1 addressing), integrate
// and the finite check with rollback -- with __syncthreads between the phases
// instead of kernel boundaries.  Corner forces, u and y live in shared memory; the state stays in
// global memory (double4 [n_v], L1/L2-resident at this size).  For a 45-vertex mesh the graph
// path is ~30 dependent launches per frame; here the frame is launch-free.
// ----------------------------------------------------------------------------

template <int MODEL>
__global__ void __launch_bounds__(256, 1) k_small_frames(Params P, SmallArgs A, int frames, int iters) {
    extern __shared__ double sm_small[];
    const int nv = P.n_v, nf = P.n_f, nt = P.n_t;
    double* u = sm_small;                                          // [3 nf]
    double* y = u + 3 * nf;                                        // [3 nf]
    float* fc = reinterpret_cast<float*>(y + 3 * nf);              // [12 nt]
    __shared__ int s_bad;
    const double h = P.h;
    for (int f = 0; f < frames; ++f) {
        // predict: x_t = x, s = x_t + h v + h^2 g, x^0 = s (A9) or x_t + h v (A9w); pins move
        if (threadIdx.x == 0) s_bad = 0;
        for (int i = threadIdx.x; i < nv; i += blockDim.x) {
            const double4 xi = A.x[i], vi = A.v[i];
            A.xt[i] = xi;
            A.vt[i] = vi;
            if (i < nf) {
                const double4 xv = make_double4(xi.x + h * vi.x, xi.y + h * vi.y, xi.z + h * vi.z, 0.0);
                const double4 si = make_double4(xv.x + h * h * P.g[0], xv.y + h * h * P.g[1], xv.z + h * h * P.g[2], 0.0);
                A.s[i] = si;
                A.x[i] = P.warm ? xv : si;
            } else {
                const double4 vp = P.vpin[i - nf];
                A.x[i] = make_double4(xi.x + h * vp.x, xi.y + h * vp.y, xi.z + h * vp.z, 0.0);
                A.v[i] = make_double4(vp.x, vp.y, vp.z, 0.0);
            }
        }
        __syncthreads();
        for (int k = 0; k < iters; ++k) {
            // local step: per tet, corner forces h^2 w (P - F) g_a
            for (int t = threadIdx.x; t < nt; t += blockDim.x) {
                const int4 tv = A.tet[t];
                const double4 x0 = A.x[tv.x], x1 = A.x[tv.y], x2 = A.x[tv.z], x3 = A.x[tv.w];
                float D[3][3];
                D[0][0] = (float)(x1.x - x0.x); D[1][0] = (float)(x1.y - x0.y); D[2][0] = (float)(x1.z - x0.z);
                D[0][1] = (float)(x2.x - x0.x); D[1][1] = (float)(x2.y - x0.y); D[2][1] = (float)(x2.z - x0.z);
                D[0][2] = (float)(x3.x - x0.x); D[1][2] = (float)(x3.y - x0.y); D[2][2] = (float)(x3.z - x0.z);
                float B[9];
                for (int e = 0; e < 9; ++e) B[e] = A.Bm[(size_t)e * nt + t];
                float F[3][3];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) F[i][j] = D[i][0] * B[j] + D[i][1] * B[3 + j] + D[i][2] * B[6 + j];
                float U[3][3], V[3][3], dlt[3];
                svd_project<MODEL>(F, P.k, P.mu, P.lam, U, dlt, V);
                const float hw = A.hw2[t];
                float Q[3][3];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        Q[i][j] = hw * (U[i][0] * dlt[0] * V[j][0] + U[i][1] * dlt[1] * V[j][1] + U[i][2] * dlt[2] * V[j][2]);
                float* o = fc + 12 * t;
                for (int i = 0; i < 3; ++i) {
                    float sum = 0.f;
                    for (int a = 0; a < 3; ++a) {
                        const float fa = Q[i][0] * B[3 * a] + Q[i][1] * B[3 * a + 1] + Q[i][2] * B[3 * a + 2];
                        o[3 * (a + 1) + i] = fa;
                        sum += fa;
                    }
                    o[i] = -sum;
                }
            }
            __syncthreads();
            // RHS in delta form: u_a = M_a (s_a - x_a) + sum of the incident corner forces
            for (int a = threadIdx.x; a < nf; a += blockDim.x) {
                const double4 xa = A.x[a], sa = A.s[a];
                const double m = A.M[a];
                float f0 = 0.f, f1 = 0.f, f2 = 0.f;
                for (int q = A.adjp[a]; q < A.adjp[a + 1]; ++q) {
                    const float* fq = fc + 3 * A.adj[q];
                    f0 += fq[0]; f1 += fq[1]; f2 += fq[2];
                }
                u[3 * a] = m * (sa.x - xa.x) + f0;
                u[3 * a + 1] = m * (sa.y - xa.y) + f1;
                u[3 * a + 2] = m * (sa.z - xa.z) + f2;
            }
            __syncthreads();
            // y = K u: row r spans columns [first(r), r]
            for (int r = threadIdx.x; r < nf; r += blockDim.x) {
                const int2 mr = A.meta[r];
                const float* kr = A.Krow + mr.x;
                double a0 = 0, a1 = 0, a2 = 0;
                for (int j = mr.y; j <= r; ++j) {
                    const double kv = kr[j];
                    a0 = fma(kv, u[3 * j], a0); a1 = fma(kv, u[3 * j + 1], a1); a2 = fma(kv, u[3 * j + 2], a2);
                }
                y[3 * r] = (float)a0; y[3 * r + 1] = (float)a1; y[3 * r + 2] = (float)a2;   // fp32 as the K-pass output
            }
            __syncthreads();
            // x += K^T y: column j is its ancestor chain j, parent(j), ... (Kcol order)
            const bool last = k == iters - 1;
            for (int j = threadIdx.x; j < nf; j += blockDim.x) {
                const float* kc = A.Kcol + A.colptr[j];
                double a0 = 0, a1 = 0, a2 = 0;
                int d = 0;
                for (int r = j; r >= 0; r = A.parent[r], ++d) {
                    const double kv = kc[d];
                    a0 = fma(kv, y[3 * r], a0); a1 = fma(kv, y[3 * r + 1], a1); a2 = fma(kv, y[3 * r + 2], a2);
                }
                double4 xj = A.x[j];
                xj.x += a0; xj.y += a1; xj.z += a2;
                A.x[j] = xj;
                if (last) {   // v = (x - x_t) / h
                    const double4 t0 = A.xt[j];
                    A.v[j] = make_double4((xj.x - t0.x) / h, (xj.y - t0.y) / h, (xj.z - t0.z) / h, 0.0);
                }
            }
            __syncthreads();
        }
        // failure detection: a non-finite frame is rolled back to its start (sim_synchronize reports it)
        for (int i = threadIdx.x; i < nv; i += blockDim.x) {
            const double4 a = A.x[i], b = A.v[i];
            if (!(isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(b.x) && isfinite(b.y) && isfinite(b.z)))
                s_bad = 1;
        }
        __syncthreads();
        if (s_bad) {
            for (int i = threadIdx.x; i < nv; i += blockDim.x) {
                A.x[i] = A.xt[i];
                A.v[i] = A.vt[i];
            }
            if (threadIdx.x == 0) atomicAdd(A.rollbacks, 1);
        }
        __syncthreads();
    }
}

size_t small_smem_bytes(const Params& P) { return (size_t)6 * P.n_f * sizeof(double) + (size_t)12 * P.n_t * sizeof(float); }

int launch_small_frames(cudaStream_t st, const Params& P, const SmallArgs& A, int frames, int iters) {
    const size_t sm = small_smem_bytes(P);
    cudaError_t e;
    if (P.model == 1)
        e = launch_pdl(k_small_frames<1>, dim3(1), dim3(256), sm, st, P, A, frames, iters);
    else if (P.model == 2)
        e = launch_pdl(k_small_frames<2>, dim3(1), dim3(256), sm, st, P, A, frames, iters);
    else
        e = launch_pdl(k_small_frames<0>, dim3(1), dim3(256), sm, st, P, A, frames, iters);
    return (int)e;
}

// ----------------------------------------------------------------------------
// contact evaluation (fp64): gaps at x^k (reading A22), FB indicators (App. B.2)
// ----------------------------------------------------------------------------
__global__ void k_contact_eval(Params P, const DContact* __restrict__ C, const double4* __restrict__ x,
                               const double4* __restrict__ xt, ContactState cs) {
    pdl_enter();
    int c = blockIdx.x * blockDim.x + threadIdx.x;   // global contact id
    if (c >= P.C) return;
    const DContact& ct = C[c];
    double h = P.h;
    double xc[3] = {0, 0, 0}, xtc[3] = {0, 0, 0};
    for (int q = 0; q < ct.nv; ++q) {
        const int iv = ct.vtx[q] * P.S + ct.inst;
        double4 a = x[iv], b = xt[iv];
        xc[0] += ct.w[q] * a.x; xc[1] += ct.w[q] * a.y; xc[2] += ct.w[q] * a.z;
        xtc[0] += ct.w[q] * b.x; xtc[1] += ct.w[q] * b.y; xtc[2] += ct.w[q] * b.z;
    }
    double Jx[3], Jxt[3];
    for (int k = 0; k < 3; ++k) {
        Jx[k] = ct.c[k][0] * xc[0] + ct.c[k][1] * xc[1] + ct.c[k][2] * xc[2];
        Jxt[k] = ct.c[k][0] * xtc[0] + ct.c[k][1] * xtc[1] + ct.c[k][2] * xtc[2];
    }
    double* lam = cs.lam + 3 * c;
    double th[3], E[3], hv[3];
    double phin_abs = 0.0;
    if (ct.kind == 1) {   // bilateral (reading A17): theta 1, E = e, h_b = d_b - E lam
        th[0] = 1.0; E[0] = ct.e; hv[0] = ct.dn - ct.e * lam[0];
        th[1] = th[2] = 0.0; E[1] = E[2] = 1.0; hv[1] = hv[2] = 0.0;   // padding rows (identity)
        cs.theta[3 * c] = th[0]; cs.cdiag[3 * c] = E[0] / (h * h); cs.hvec[3 * c] = hv[0];
        for (int k = 1; k < 3; ++k) { cs.theta[3 * c + k] = 0.0; cs.cdiag[3 * c + k] = 1.0; cs.hvec[3 * c + k] = 0.0; }
        for (int d = 0; d < 3; ++d) cs.hl[3 * c + d] = lam[0] * ct.c[0][d];
        cs.phi_abs[c] = 0.0;
        return;
    }
    const double pjj = P.precond ? ct.Mjj : ct.Djj;
    double rn = h * h * pjj, rf = h * pjj;
    double y = Jx[0] - ct.dn, ln = lam[0];
    if (fabs(y) <= 1e-12 * P.len_scale) y = 0.0;   // a gap within rounding of 0 is 0 (reading A15)
    double phin, thn, En;
    if (P.ncp == 1) {   // minimum map (App. B.1)
        const bool first = y <= rn * ln;
        phin = first ? y : rn * ln;
        thn = first ? 1.0 : 0.0;
        En = first ? 0.0 : rn;
    } else if (double S = sqrt(y * y + rn * rn * ln * ln); S > 0.0) {   // normal FB (A15)
        double a = y + rn * ln;
        phin = a > 0.0 ? (2.0 * y * rn * ln) / (a + S) : a - S;
        thn = 1.0 - y / S;
        En = (1.0 - rn * ln / S) * rn;
    } else {
        phin = 0.0; thn = 1.0; En = 0.0;
    }
    phin_abs = fabs(phin);
    // friction (A14, A16, A16b, A16c)
    double yd1 = (Jx[1] - Jxt[1]) / h - ct.df1, yd2 = (Jx[2] - Jxt[2]) / h - ct.df2;
    double thf, Ef;
    if (ln > 0.0 && ct.mu * ln > 0.0) {
        double s = sqrt(yd1 * yd1 + yd2 * yd2);
        double lf = sqrt(lam[1] * lam[1] + lam[2] * lam[2]);
        if (P.ncp == 1) {   // minimum map: stick 0, slip (|ydot| - r q) / (mu lam_n)
            double q = ct.mu * ln - lf;
            Ef = s <= rf * q ? 0.0 : (s - rf * q) / (ct.mu * ln);
        } else {
            // FB: q at the cone projection of lam_f (A16c: no pole at |lam_f| = 2 mu lam_n);
            // the 0/0 point (s, |lam_f|) = (0, 0) has limit 0 (A16)
            double q = ct.mu * ln - fmin(lf, ct.mu * ln);
            double R = sqrt(s * s + rf * rf * q * q);
            double num = rf * (R - rf * q);
            double den = s + ct.mu * rf * ln - R;
            Ef = den > 1e-12 * (s + ct.mu * rf * ln) ? num / den : 0.0;
        }
        thf = 1.0;
    } else {
        thf = 0.0; Ef = 1.0;
    }
    double phif1 = thf * yd1 + Ef * lam[1], phif2 = thf * yd2 + Ef * lam[2];
    th[0] = thn; th[1] = th[2] = thf;
    cs.theta[3 * c] = thn; cs.theta[3 * c + 1] = thf; cs.theta[3 * c + 2] = thf;
    cs.cdiag[3 * c] = En / (h * h); cs.cdiag[3 * c + 1] = Ef / h; cs.cdiag[3 * c + 2] = Ef / h;
    // h-vector
    cs.hvec[3 * c] = -phin + thn * Jx[0];
    cs.hvec[3 * c + 1] = -h * phif1 + thf * Jx[1];
    cs.hvec[3 * c + 2] = -h * phif2 + thf * Jx[2];
    for (int d = 0; d < 3; ++d)
        cs.hl[3 * c + d] = thn * lam[0] * ct.c[0][d] + thf * (lam[1] * ct.c[1][d] + lam[2] * ct.c[2][d]);
    cs.phi_abs[c] = phin_abs;
}

void launch_contact_eval(cudaStream_t st, const Params& P, const DContact* c, const double4* x,
                         const double4* xt, ContactState cs) {
    if (P.C == 0) return;
    k_contact_eval<<<(P.C + 127) / 128, 128, 0, st>>>(P, c, x, xt, cs);
}

// frame-end contact statistics (sim_get_stats): per contact the classification of reading A21
// (active <=> lambda_n > 0; stick <=> |ydot_f| <= r_f (mu lambda_n - |lambda_f|), P:L292-298,
// P:L1650; -1 for bilateral rows), the Coulomb-cone violation max(0, |lambda_f| - mu max(lambda_n, 0))
// and the gap y_n = J_n x - d_n, all at the state x after the last frame (x_t = its start)
__global__ void k_contact_stats(Params P, const DContact* __restrict__ C, const double4* __restrict__ x,
                                const double4* __restrict__ xt, const double* __restrict__ lamv,
                                int* __restrict__ cls, double* __restrict__ cone, double* __restrict__ gap) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P.C) return;
    const DContact& ct = C[c];
    double xc[3] = {0, 0, 0}, xtc[3] = {0, 0, 0};
    for (int q = 0; q < ct.nv; ++q) {
        const int iv = ct.vtx[q] * P.S + ct.inst;
        const double4 a = x[iv], b = xt[iv];
        xc[0] += ct.w[q] * a.x; xc[1] += ct.w[q] * a.y; xc[2] += ct.w[q] * a.z;
        xtc[0] += ct.w[q] * b.x; xtc[1] += ct.w[q] * b.y; xtc[2] += ct.w[q] * b.z;
    }
    double Jx[3], Jxt[3];
    for (int k = 0; k < 3; ++k) {
        Jx[k] = ct.c[k][0] * xc[0] + ct.c[k][1] * xc[1] + ct.c[k][2] * xc[2];
        Jxt[k] = ct.c[k][0] * xtc[0] + ct.c[k][1] * xtc[1] + ct.c[k][2] * xtc[2];
    }
    gap[c] = Jx[0] - ct.dn;
    const double* lam = lamv + 3 * c;
    if (ct.kind == 1) {
        cls[c] = -1;
        cone[c] = 0.0;
        return;
    }
    const double ln = lam[0], lf = sqrt(lam[1] * lam[1] + lam[2] * lam[2]);
    cone[c] = fmax(0.0, lf - ct.mu * fmax(ln, 0.0));
    if (!(ln > 0.0)) {
        cls[c] = 0;
        return;
    }
    const double h = P.h;
    const double yd1 = (Jx[1] - Jxt[1]) / h - ct.df1, yd2 = (Jx[2] - Jxt[2]) / h - ct.df2;
    const double rf = h * (P.precond ? ct.Mjj : ct.Djj);
    cls[c] = sqrt(yd1 * yd1 + yd2 * yd2) <= rf * (ct.mu * ln - lf) ? 1 : 2;
}

void launch_contact_stats(cudaStream_t st, const Params& P, const DContact* c, const double4* x, const double4* xt,
                          const double* lam, int* cls, double* cone, double* gap) {
    if (P.C > 0) k_contact_stats<<<(P.C + 127) / 128, 128, 0, st>>>(P, c, x, xt, lam, cls, cone, gap);
}

// ----------------------------------------------------------------------------
// gather: u_a = M_a (s_a - x_a) + sum_{(t,c) in adj(a)} f_{t,c} + h^2 (H^T lam)_a
// (colour-free: each free vertex sums its incident tets in a fixed order)
// ----------------------------------------------------------------------------
__global__ void k_gather(Params P, const int32_t* __restrict__ adjp, const int32_t* __restrict__ adj,
                         const float* __restrict__ fc, const double* __restrict__ M, const double4* __restrict__ x,
                         const double4* __restrict__ s, const int32_t* __restrict__ slotmap, Slots sl,
                         const double* __restrict__ hl, float4* __restrict__ u, double* __restrict__ resid) {
    pdl_enter();
    const int S = P.S;
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;   // (free vertex, instance), instance-minor
    if (gi >= P.n_f * S) return;
    const int a = gi / S, inst = gi - a * S;
    double4 xa = x[gi], sa = s[gi];
    double m = M[a];
    double r0 = m * (sa.x - xa.x), r1 = m * (sa.y - xa.y), r2 = m * (sa.z - xa.z);
    int p0 = adjp[a], p1 = adjp[a + 1];
    float f0 = 0.f, f1 = 0.f, f2 = 0.f;
    for (int p = p0; p < p1; ++p) {
        const float* f = fc + (size_t)__ldg(&adj[p]) * 3 * S + inst;   // (tet, corner) entry, 3 planes of S
        f0 += __ldg(f);
        f1 += __ldg(f + S);
        f2 += __ldg(f + 2 * S);
    }
    r0 += f0;
    r1 += f1;
    r2 += f2;
    if (resid) {
        resid[3 * (size_t)gi] = r0;
        resid[3 * (size_t)gi + 1] = r1;
        resid[3 * (size_t)gi + 2] = r2;
    }
    if (slotmap) {   // h^2 H^T Theta lambda at contact vertices (slot -> contacts, fixed order)
        const int b = slotmap[gi];
        if (b >= 0) {
            double hh = P.h * P.h;
            for (int p = sl.scp[b]; p < sl.scp[b + 1]; ++p) {
                int c = sl.sci[p];
                double w = sl.scw[p];
                r0 += hh * w * hl[3 * c];
                r1 += hh * w * hl[3 * c + 1];
                r2 += hh * w * hl[3 * c + 2];
            }
        }
    }
    vec_st(u, S, P.n_f, a, inst, (float)r0, (float)r1, (float)r2);
}

void launch_gather(cudaStream_t st, const Params& P, const int32_t* adjp, const int32_t* adj,
                   const float* fc, const double* M, const double4* x, const double4* s,
                   const int32_t* slotmap, Slots sl, const double* hl, float4* u, double* resid_dbg) {
    launch_pdl(k_gather, dim3((P.n_f * P.S + 255) / 256), dim3(256), 0, st, P, adjp, adj, fc, M, x, s, slotmap, sl, hl, u,
               resid_dbg);
}

// ----------------------------------------------------------------------------
// K-pass 1: y = K u.  One CTA (8 warps) per item = (<= 32 rows of one panel) x
// (<= 1024 columns); warps take interleaved 32-column chunks, lane = row.
// K is column-major: K[r][j] = Kcol[cb[j] - depth[r]], cb[j] = colptr[j] + depth[j]
// (carried in u[j].w); inside a panel depth[r0 + l] = depth[r0] - l, so the 32
// lanes read 32 consecutive words of column j.
// ----------------------------------------------------------------------------
constexpr int kWarps = 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Accumulation: fp32 FMAs over one 32-entry chunk, folded into fp64 once per
// chunk (fp32->fp64 conversion runs at 1/4 of the FP64 rate on sm_100, so a
// per-element DFMA would be conversion-bound).
//
// Memory pipeline: each warp streams its 32x32 tiles of K (and the matching
// 32 vector entries) into shared memory with cp.async (4-byte, zero-fill for
// entries outside the skyline), kStages tiles in flight per warp.
constexpr int kStages = 3;       // pass-1 tiles in flight per warp
#ifndef SIM_P2_STAGES
#define SIM_P2_STAGES 3
#endif
#ifndef SIM_P2_WARPS
#define SIM_P2_WARPS 6
#endif
constexpr int kStages2 = SIM_P2_STAGES;   // pass-2 tiles in flight per warp
constexpr int kWarps2 = SIM_P2_WARPS;     // pass-2 warps per CTA

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
// K entries are streamed once per pass: evict-first in L2 so the pass does not flush the
// state, vectors, contact data and kernel code that the latency-bound kernels reuse
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_async4_stream(void* smem, const void* gmem, bool valid, unsigned long long pol) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;\n" ::"r"(s), "l"(gmem), "r"(n),
                 "l"(pol));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct __align__(16) KTile {
    float k[32][32];    // [entry q][lane]
    float4 v[32];       // vector entry q (u_j for pass 1, y_r for pass 2); .w of u carries cb[j]
};

// ---- bulk (TMA 1-D) copy helpers ---------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
// warp-uniform wait (the whole warp leaves the loop together: the code after it is provably converged,
// so warp-uniform values stay in uniform registers)
__device__ __forceinline__ void mbar_wait_w(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!__all_sync(0xffffffffu, done)) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
// global -> shared bulk copy completing `bytes` on `bar`; evict-first in L2 when `stream`
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar, bool stream,
                                         unsigned long long pol) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    if (stream)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
            "%4;\n" ::"r"(s),
            "l"(gmem), "r"(bytes), "r"(b), "l"(pol)
            : "memory");
    else
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(s),
                     "l"(gmem), "r"(bytes), "r"(b)
                     : "memory");
}

// ---- pass 1 ----------------------------------------------------------------
// Persistent warps: warp g of G processes items g, g + G, ... (items are sorted by size,
// so the round robin balances).  An item is <= 32 rows of a panel x <= 1024 columns; its
// K tiles are contiguous in consumption order (T1, tile = [32 columns][nr rows]).  Each
// warp streams its tiles with 1-D bulk copies issued by one lane, kStages tiles in flight,
// and the issue cursor runs ahead across item boundaries so the pipeline never drains.
// Rows split over several items are combined by the last-arriving warp in fixed order.
__device__ __forceinline__ int p1_ntiles(const P1Item& it) { return (it.c1 - it.c0 + 31) >> 5; }

__global__ void __launch_bounds__(256, 2) k_kpass1(const P1Item* __restrict__ items, int nitems,
                                                   const P1Block* __restrict__ blocks,
                                                   const float* __restrict__ T1, const float4* __restrict__ u,
                                                   float4* __restrict__ y, double* __restrict__ part,
                                                   int* __restrict__ counters) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char k1smem[];
    __shared__ __align__(8) uint64_t bars[kWarps][kStages];
    KTile* tiles = reinterpret_cast<KTile*>(k1smem) + (threadIdx.x >> 5) * kStages;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x * kWarps;
    const int gw = blockIdx.x * kWarps + w;
    if (gw >= nitems) return;
    const unsigned long long pol = l2_evict_first();
    for (int s = 0; s < kStages; ++s) tiles[s].v[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane == 0)
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[w][s], 1);
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    // issue cursor
    int ik = gw, itl = 0;
    P1Item iI = items[ik];
    int ntI = p1_ntiles(iI);
    int n_issued = 0;
    auto issue_next = [&]() {
        if (ik >= nitems) return;
        const int s = n_issued % kStages;
        const int jc = iI.c0 + 32 * itl;
        const int ncol = min(32, iI.c1 - jc);
        if (lane == 0) {
            mbar_expect_tx(&bars[w][s], (unsigned)(iI.nrows * 128 + ncol * 16));
            bulk_g2s(tiles[s].k, T1 + iI.toff + (int64_t)itl * iI.nrows * 32, (unsigned)(iI.nrows * 128), &bars[w][s],
                     true, pol);
            bulk_g2s(tiles[s].v, u + jc, (unsigned)(ncol * 16), &bars[w][s], false, pol);
        }
        ++n_issued;
        if (++itl == ntI) {
            itl = 0;
            ik += G;
            if (ik < nitems) {
                iI = items[ik];
                ntI = p1_ntiles(iI);
            }
        }
    };
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) issue_next();
    // compute cursor
    int ck = gw, ctl = 0;
    P1Item cI = iI;
    cI = items[ck];
    int ntC = p1_ntiles(cI);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    unsigned par = 0;
    for (int n_done = 0; ck < nitems; ++n_done) {
        issue_next();
        const int s = n_done % kStages;
        mbar_wait(&bars[w][s], (par >> s) & 1u);
        par ^= 1u << s;
        const int nr = cI.nrows;
        const float* kk = &tiles[s].k[0][0];
        const float4* vv = tiles[s].v;
        float f0 = 0.f, f1 = 0.f, f2 = 0.f;
        if (lane < nr) {
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const float kq = kk[q * nr + lane];
                const float4 uq = vv[q];
                f0 = fmaf(kq, uq.x, f0);
                f1 = fmaf(kq, uq.y, f1);
                f2 = fmaf(kq, uq.z, f2);
            }
        }
        a0 += (double)f0;
        a1 += (double)f1;
        a2 += (double)f2;
        __syncwarp();   // stage s may be refilled by the next issue
        if (++ctl < ntC) continue;
        // ---- item complete: write y, or a partial + fixed-order reduction by the last warp
        const P1Block b = blocks[cI.block];
        if (b.nitems == 1) {
            if (lane < nr) y[cI.r0 + lane] = make_float4((float)a0, (float)a1, (float)a2, 0.f);
        } else {
            double* pp = part + (size_t)cI.part * 96 + lane;
            pp[0] = a0;
            pp[32] = a1;
            pp[64] = a2;
            __threadfence();
            __syncwarp();
            int old = 0;
            if (lane == 0) old = atomicAdd(&counters[cI.block], 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == b.nitems - 1) {
                __threadfence();
                double s0 = 0.0, s1 = 0.0, s2 = 0.0;
                for (int q = 0; q < b.nitems; ++q) {
                    const double* pq = part + (size_t)(b.part0 + q) * 96 + lane;
                    s0 += __ldcg(pq);
                    s1 += __ldcg(pq + 32);
                    s2 += __ldcg(pq + 64);
                }
                if (lane < nr) y[cI.r0 + lane] = make_float4((float)s0, (float)s1, (float)s2, 0.f);
                if (lane == 0) counters[cI.block] = 0;
            }
        }
        a0 = a1 = a2 = 0.0;
        ctl = 0;
        ck += G;
        if (ck < nitems) {
            cI = items[ck];
            ntC = p1_ntiles(cI);
        }
    }
}

constexpr size_t kKpassSmem = sizeof(KTile) * kStages * kWarps;   // >= 3 * kWarps * 32 doubles for s_red
constexpr int kP2MaxRows = 1536;                                   // cover rows whose y is staged in smem
constexpr size_t kKpass2Tiles = sizeof(KTile) * kStages2 * kWarps2;  // >= 3 * kWarps2 * 32 doubles
constexpr size_t kKpass2Smem = kKpass2Tiles + 16 * kP2MaxRows;

void launch_kpass1(cudaStream_t st, int nitems, const P1Item* it, const P1Block* bl, const float* T1,
                   const float4* u, float4* y, double* part, int* counters) {
    static unsigned long long attr = 0;
    const int nsm = sm_count();
    per_device_once(attr, [&] {
        cudaFuncSetAttribute(k_kpass1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kKpassSmem);
    });
    const int ctas = std::min((nitems + kWarps - 1) / kWarps, 2 * nsm);   // persistent: 2 CTAs per SM
    launch_pdl(k_kpass1, dim3(ctas), dim3(32 * kWarps), kKpassSmem, st, it, nitems, bl, T1, u, y, part, counters);
}

// ----------------------------------------------------------------------------
// K-pass 2: x += K^T y.  One CTA per 32-column block (lane = column).  The block's
// cover-row tiles ([32 rows][32 columns], consumption order, T2) are streamed with 1-D
// bulk copies; the y values of all cover rows are staged once in shared memory.
// No partial sums, no atomics: the CTA owns its 32 columns.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(32 * kWarps2, 2) k_kpass2(const P2Block* __restrict__ blocks,
                                                   const int32_t* __restrict__ cover, const float* __restrict__ T2,
                                                   const float4* __restrict__ y, double4* __restrict__ x,
                                                   const double4* __restrict__ xt, double4* __restrict__ v,
                                                   double inv_h, int finalize_v) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char k2smem[];
    __shared__ __align__(8) uint64_t bars[kWarps2][kStages2];
    KTile* tiles = reinterpret_cast<KTile*>(k2smem) + (threadIdx.x >> 5) * kStages2;
    double (*s_red)[kWarps2][32] = reinterpret_cast<double (*)[kWarps2][32]>(k2smem);   // aliases the tiles after the loop
    float4* s_y = reinterpret_cast<float4*>(k2smem + kKpass2Tiles);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const P2Block b = blocks[blockIdx.x];
    const int nrow = b.list1 - b.list0;
    const int nt = (nrow + 31) >> 5;
    const int mine = (nt - w + kWarps2 - 1) / kWarps2;
    const bool staged = nrow <= kP2MaxRows;
    const unsigned long long pol = l2_evict_first();
    if (lane == 0)
        for (int s = 0; s < kStages2; ++s) mbar_init(&bars[w][s], 1);
    if (staged) {
        for (int q = threadIdx.x; q < 32 * nt; q += blockDim.x)
            cp_async16(&s_y[q], &y[q < nrow ? __ldg(&cover[b.list0 + q]) : 0], q < nrow);
        cp_async_commit();
    }
    __syncwarp();
    auto issue = [&](int t) {
        const int ti = w + kWarps2 * t;
        const int s = t % kStages2;
        if (lane == 0) {
            mbar_expect_tx(&bars[w][s], 4096u);
            bulk_g2s(tiles[s].k, T2 + b.toff + (int64_t)ti * 1024, 4096u, &bars[w][s], true, pol);
        }
    };
#pragma unroll
    for (int t = 0; t < kStages2 - 1; ++t)
        if (t < mine) issue(t);
    if (staged) {
        cp_async_wait<0>();
        __syncthreads();
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    unsigned par = 0;
    for (int t = 0; t < mine; ++t) {
        if (t + kStages2 - 1 < mine) issue(t + kStages2 - 1);
        const int s = t % kStages2;
        const int ti = w + kWarps2 * t;
        const float4* yy;
        if (staged) {
            yy = s_y + 32 * ti;
        } else {   // very tall trees: gather this tile's y into the tile's vector slot
            const int kq = 32 * ti + lane;
            tiles[s].v[lane] = kq < nrow ? __ldg(&y[__ldg(&cover[b.list0 + kq])]) : make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            yy = tiles[s].v;
        }
        mbar_wait(&bars[w][s], (par >> s) & 1u);
        par ^= 1u << s;
        const float* kk = &tiles[s].k[0][0];
        float f0 = 0.f, f1 = 0.f, f2 = 0.f;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const float kq = kk[32 * q + lane];
            const float4 yq = yy[q];
            f0 = fmaf(kq, yq.x, f0);
            f1 = fmaf(kq, yq.y, f1);
            f2 = fmaf(kq, yq.z, f2);
        }
        a0 += (double)f0;
        a1 += (double)f1;
        a2 += (double)f2;
        __syncwarp();
    }
    __syncthreads();   // all warps are done with their tiles before s_red overwrites them
    s_red[0][w][lane] = a0;
    s_red[1][w][lane] = a1;
    s_red[2][w][lane] = a2;
    __syncthreads();
    const int t = threadIdx.x;
    if (t < 96) {
        double tot = 0.0;
#pragma unroll
        for (int q = 0; q < kWarps2; ++q) tot += s_red[t >> 5][q][t & 31];
        s_red[t >> 5][0][t & 31] = tot;   // each thread owns its (comp, lane) slot: no race
    }
    __syncthreads();
    if (t >= b.ncols) return;
    const int jj = b.c0 + t;
    double4 xj = x[jj];
    xj.x += s_red[0][0][t];
    xj.y += s_red[1][0][t];
    xj.z += s_red[2][0][t];
    x[jj] = xj;
    if (finalize_v) {   // v = (x - x_t) / h
        const double4 t0 = xt[jj];
        v[jj] = make_double4((xj.x - t0.x) * inv_h, (xj.y - t0.y) * inv_h, (xj.z - t0.z) * inv_h, 0.0);
    }
}

void launch_kpass2(cudaStream_t st, int nblocks, const P2Block* bl, const int32_t* cover, const float* T2,
                   const float4* y, double4* x, const double4* xt, double4* v, double inv_h, int finalize_v) {
    static unsigned long long attr = 0;
    per_device_once(attr, [&] {
        cudaFuncSetAttribute(k_kpass2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kKpass2Smem);
    });
    launch_pdl(k_kpass2, dim3(nblocks), dim3(32 * kWarps2), kKpass2Smem, st, bl, cover, T2, y, x, xt, v, inv_h, finalize_v);
}

// ----------------------------------------------------------------------------
// Batched K-passes (S > 1 instances sharing K): every K tile is read once per chunk of
// 128 instances and applied to 3 x 128 right-hand sides, so the passes become SpMM and
// turn FP32-issue-bound instead of HBM-bound.  One CTA = (unit, instance chunk); the unit's
// 32 x 32 K tiles and the matching 32 vector rows of the chunk (32 x 128 float4) are staged
// by 1-D bulk copies (2 stages).  Warp w: outputs 16 (w & 1) .. +15, instances 32 (w >> 1) +
// lane; per reduction index q it reads its 16 K values as 4 broadcast float4s and one
// float4 of the vector.  fp32 FMAs per tile, folded into fp64 once per tile (as in S = 1).
//   pass 1: out = rows of a block,    reduction over columns  (T1p, vector u, out y)
//   pass 2: out = 32 columns,         reduction over cover rows (T2, vector y, out x += .)
// Instances are the fastest grid dimension inside a unit chunk: chunk-major launch order
// keeps one chunk's vectors (n_f x 128 x 16 B) resident in L2 while its units run.
// ----------------------------------------------------------------------------
constexpr int kBInst = 128;                 // instances per CTA
constexpr int kBStages = 2;
constexpr size_t kBStageBytes = 4096 + 3 * 32 * kBInst * 4;   // K tile + 3 component planes of 32 rows
constexpr size_t kBSmem = kBStages * kBStageBytes;

template <int PASS>
__global__ void __launch_bounds__(256, 1)
    k_kpass_b(int S, int n_f, const BUnit* __restrict__ units, const float* __restrict__ T,
              const int32_t* __restrict__ cover, const float* __restrict__ vin, float* __restrict__ yout,
              double* __restrict__ part, int* __restrict__ counters, int nchunks, double4* __restrict__ x,
              const double4* __restrict__ xt, double4* __restrict__ v, double inv_h, int finalize_v) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char bsm[];
    const int Sp = plane_sp(S);
    const size_t PS = (size_t)n_f * Sp;
    __shared__ __align__(8) uint64_t full[kBStages];
    __shared__ int s_last;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int half = w & 1, ig = w >> 1;
    const BUnit U = units[blockIdx.x];
    const int chunk = blockIdx.y;
    const int i0 = chunk * kBInst;
    const int ni = min(kBInst, S - i0);
    const int li = 32 * ig + lane;           // instance within the chunk
    const unsigned long long pol = l2_evict_first();
    auto ktile = [&](int s) { return reinterpret_cast<float*>(bsm + s * kBStageBytes); };
    auto vtile = [&](int s) { return reinterpret_cast<float*>(bsm + s * kBStageBytes + 4096); };   // [3][32][kBInst]
    // zero the vector tiles once: rows / instances that are never copied must read as 0
    for (int e = threadIdx.x; e < kBStages * 3 * 32 * kBInst; e += blockDim.x)
        vtile(e / (3 * 32 * kBInst))[e % (3 * 32 * kBInst)] = 0.f;
    if (threadIdx.x == 0)
        for (int s = 0; s < kBStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // zero fill before the bulk copies
    __syncthreads();
    auto nvalid = [&](int t) {   // vector rows present in tile t
        if (PASS == 1) return max(0, min(32, n_f - (U.c0 + 32 * t)));
        return min(32, U.nlist - 32 * t);
    };
    auto issue = [&](int t) {   // warp 0 only
        const int s = t % kBStages;
        const int nv = nvalid(t);
        const unsigned rb = (unsigned)(((ni + 3) & ~3) * 4);   // one plane row of the chunk (16-byte multiple)
        if (lane == 0) mbar_expect_tx(&full[s], 4096u + 3u * (unsigned)nv * rb);
        __syncwarp();
        if (lane == 0) bulk_g2s(ktile(s), T + U.toff + (int64_t)t * 1024, 4096u, &full[s], true, pol);
        if (lane < nv) {
            const int idx = PASS == 1 ? U.c0 + 32 * t + lane : __ldg(&cover[U.list0 + 32 * t + lane]);
            for (int c = 0; c < 3; ++c)
                bulk_g2s(vtile(s) + (c * 32 + lane) * kBInst, vin + c * PS + (size_t)idx * Sp + i0, rb, &full[s], false,
                         pol);
        }
    };
    if (w == 0)
        for (int t = 0; t < kBStages && t < U.ntiles; ++t) issue(t);
    double d[16][3];
#pragma unroll
    for (int r = 0; r < 16; ++r) d[r][0] = d[r][1] = d[r][2] = 0.0;
    for (int t = 0; t < U.ntiles; ++t) {
        const int s = t % kBStages;
        mbar_wait(&full[s], (t / kBStages) & 1);
        const float* kt = ktile(s) + 16 * half;
        const float* vt = vtile(s) + li;
        float a[16][3];
#pragma unroll
        for (int r = 0; r < 16; ++r) a[r][0] = a[r][1] = a[r][2] = 0.f;
#pragma unroll 4
        for (int q = 0; q < 32; ++q) {
            const float4 vq = make_float4(vt[q * kBInst], vt[(32 + q) * kBInst], vt[(64 + q) * kBInst], 0.f);
            const float4* kq = reinterpret_cast<const float4*>(kt + 32 * q);
#pragma unroll
            for (int r4 = 0; r4 < 4; ++r4) {
                const float4 kk = kq[r4];
                const float kv[4] = {kk.x, kk.y, kk.z, kk.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    a[4 * r4 + e][0] = fmaf(kv[e], vq.x, a[4 * r4 + e][0]);
                    a[4 * r4 + e][1] = fmaf(kv[e], vq.y, a[4 * r4 + e][1]);
                    a[4 * r4 + e][2] = fmaf(kv[e], vq.z, a[4 * r4 + e][2]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            d[r][0] += (double)a[r][0];
            d[r][1] += (double)a[r][1];
            d[r][2] += (double)a[r][2];
        }
        __syncthreads();   // every warp is done with stage s
        if (w == 0 && t + kBStages < U.ntiles) issue(t + kBStages);
    }
    const bool live = li < ni;
    const int inst = i0 + li;
    if (PASS == 2) {
        if (!live) return;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int l = 16 * half + r;
            if (l < U.nr) {
                const size_t j = (size_t)(U.c0 + l) * S + inst;
                double4 xj = x[j];
                xj.x += d[r][0];
                xj.y += d[r][1];
                xj.z += d[r][2];
                x[j] = xj;
                if (finalize_v) {   // v = (x - x_t) / h
                    const double4 t0 = xt[j];
                    v[j] = make_double4((xj.x - t0.x) * inv_h, (xj.y - t0.y) * inv_h, (xj.z - t0.z) * inv_h, 0.0);
                }
            }
        }
        return;
    }
    if (U.nparts == 1) {
        if (!live) return;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int l = 16 * half + r;
            if (l < U.nr) {
                const size_t iy = (size_t)(U.r0 + l) * Sp + inst;
                yout[iy] = (float)d[r][0];
                yout[PS + iy] = (float)d[r][1];
                yout[2 * PS + iy] = (float)d[r][2];
            }
        }
        return;
    }
    // block split over several units: fp64 partials, combined in fixed order by the last unit
    const size_t pstride = (size_t)32 * S;   // one (part, component) plane: [row][instance]
    if (live) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int l = 16 * half + r;
            double* pp = part + (size_t)U.part * 3 * pstride + (size_t)l * S + inst;
            pp[0] = d[r][0];
            pp[pstride] = d[r][1];
            pp[2 * pstride] = d[r][2];
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int old = atomicAdd(&counters[U.block * nchunks + chunk], 1);
        s_last = old == U.nparts - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (live) {
        for (int r = 0; r < 16; ++r) {
            const int l = 16 * half + r;
            if (l >= U.nr) continue;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int q = 0; q < U.nparts; ++q) {
                const double* pq = part + (size_t)(U.list0 + q) * 3 * pstride + (size_t)l * S + inst;
                t0 += __ldcg(pq);
                t1 += __ldcg(pq + pstride);
                t2 += __ldcg(pq + 2 * pstride);
            }
            const size_t iy = (size_t)(U.r0 + l) * Sp + inst;
            yout[iy] = (float)t0;
            yout[PS + iy] = (float)t1;
            yout[2 * PS + iy] = (float)t2;
        }
    }
    if (threadIdx.x == 0) counters[U.block * nchunks + chunk] = 0;
}

void launch_kpass1_batched(cudaStream_t st, int S, int n_f, int nunits, const BUnit* units, const float* T1p,
                           const float* u, float* y, double* part, int* counters) {
    static unsigned long long attr = 0;
    per_device_once(attr, [&] {
        cudaFuncSetAttribute(k_kpass_b<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBSmem);
    });
    const int nch = (S + kBInst - 1) / kBInst;
    launch_pdl(k_kpass_b<1>, dim3(nunits, nch), dim3(256), kBSmem, st, S, n_f, units, T1p, (const int32_t*)nullptr, u, y,
               part, counters, nch, (double4*)nullptr, (const double4*)nullptr, (double4*)nullptr, 0.0, 0);
}

void launch_kpass2_batched(cudaStream_t st, int S, int n_f, int nunits, const BUnit* units, const int32_t* cover,
                           const float* T2, const float* y, double4* x, const double4* xt, double4* v,
                           double inv_h, int finalize_v) {
    static unsigned long long attr = 0;
    per_device_once(attr, [&] {
        cudaFuncSetAttribute(k_kpass_b<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBSmem);
    });
    const int nch = (S + kBInst - 1) / kBInst;
    launch_pdl(k_kpass_b<2>, dim3(nunits, nch), dim3(256), kBSmem, st, S, n_f, units, T2, cover, y, (float*)nullptr,
               (double*)nullptr, (int*)nullptr, nch, x, xt, v, inv_h, finalize_v);
}

// ----------------------------------------------------------------------------
// Batched K-passes on the 5th-generation tensor cores (tcgen05.mma kind::tf32, accumulators
// in TMEM).  With S instances sharing K each 32 x 32 K tile multiplies a 32 x 128 block of
// right-hand sides per component, a dense contraction: D_c[inst][out] += sum_q V_c[inst][q]
// K[q][out] is one M = 128 (instances) x N = 32 (outputs) x K = 32 (reduction) MMA per tile
// and component.  Near-fp32 accuracy from the 3xTF32 split (a = a_hi + a_lo, both rounded to
// nearest tf32, |a - a_hi - a_lo| <= 2^-22 |a|): D += V_hi K_hi + V_lo K_hi + V_hi K_lo (the
// dropped V_lo K_lo is <= 2^-22 relative); the TMEM accumulators (fp32) are folded into fp64
// registers every `drain` tiles and restarted, units combined in fp64 as in k_kpass_b.
//   operands in shared memory, SWIZZLE_NONE K-major canonical layout: core matrix = 8 rows
//   x 16 B (4 tf32 along K); LBO = 128 B between K chunks, SBO = 1024 B between 8-row groups.
//   A (vectors, 128 x 32 per component, hi and lo): written by all 512 threads from the
//   gathered rows (float4 loads, coalesced over instances, 8 per thread in flight: the whole
//   64 KB tile is requested at once); B (K tile hi / lo, 4 KB each):
//   pre-laid out on the host, one 8 KB bulk copy per tile.  Two stages: while the tensor
//   core runs tile t the threads stage tile t + 1; tcgen05.commit frees a stage.
//   thread 0 issues the 36 MMAs per tile (3 components x 4 K-steps x 3 products).
//   fold / epilogue: warp w reads TMEM lanes 32 (w % 4) .. (instances) and columns 8 (w / 4) ..
//   (outputs) of every component with tcgen05.ld.32x32b.x8.
// ----------------------------------------------------------------------------
constexpr int kTcInst = 128;
constexpr int kTcThreads = 512;                                   // 16 warps: 4 per TMEM lane quadrant
constexpr uint32_t kTcAplane = kTcInst * 32 * 4;                  // 16 KB
constexpr uint32_t kTcStage = 6 * kTcAplane + 2 * 4096;           // 104 KB
constexpr size_t kTcSmem = 2 * (size_t)kTcStage + 128;
constexpr uint32_t kIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint64_t umma_desc_k(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1 << 46);
}
__device__ __forceinline__ void umma_tf32(uint32_t dt, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
        "l"(da), "l"(db), "r"(kIdescTf32), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
// round-to-nearest to tf32 (10 explicit mantissa bits): the split v = hi + lo with both parts
// exactly representable in tf32 up to 2^-22 |v| (the tensor core ignores the low 13 bits)
__device__ __forceinline__ float tf32_rn(float v) {
    return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}

// ----------------------------------------------------------------------------
// Plane-layout batched K-passes on the tensor cores (S > 1, sim_set_kpass_mode 2, default).
// Right-hand sides are fp32 component planes v[c][row][Sp] (Sp = S rounded up to 4).  One CTA
// = one unit (simhost::build_plane_units: 64 outputs x tiles of 32 reductions) x 128 instances
// x the 3 components: per tile and component D_c[inst][out] += sum_q V_c[inst][q] K[q][out],
// tcgen05.mma kind::tf32, M = 128 (instances) x N = 64 (outputs) x K = 8, 4 K-steps per tile.
// 3xTF32: the tensor core truncates fp32 operands to tf32 (measured: tools/probes/tf32_round.cu),
// so V_hi = trunc(V) is the raw fp32 tile in shared memory and V_lo = rn_tf32(V - trunc(V)) goes
// to TMEM; K_hi / K_lo are pre-rounded on the host:
//     D += V_hi K_hi + V_hi K_lo + V_lo K_hi          (|error| <= ~2^-21 |V| |K| per product)
//   * V_hi: 16-byte cp.async straight from the planes into the MN-major SWIZZLE_128B_BASE32B
//     canonical layout (umma_desc_mn32), 3 stages; no register staging, every thread has its
//     next two tiles' copies in flight;
//   * V_lo: the 16 worker warps read their 8 rows x 32 instances of V_hi back (conflict-free,
//     one 128-B row per warp load), split, tcgen05.st into TMEM (lane = instance), 2 stages;
//   * K tiles (hi 8 KB + lo 8 KB, K-major SWIZZLE_NONE) by one bulk copy per tile;
//   * one elected thread of the extra warp issues the 36 MMAs per tile (3 components x 4
//     K-steps x 3 products) and commits to the stage's mbarrier;
//   * the TMEM accumulators (3 x 64 columns) are folded into fp32 registers every `drain`
//     tiles (warp w: lanes 32 (w % 4).., columns 16 (w / 4)..): the fp32 MMA accumulation is
//     lossy over long sums, a fold every 4 tiles bounds it.
// TMEM: D_c at columns 64 c (192), V_lo stage s at 192 + 96 s + 32 c (+ 8 per K-step).
// ----------------------------------------------------------------------------
constexpr int kPlInst = 128;
constexpr int kPlWarps = 16;
constexpr int kPlThreads = 32 * kPlWarps;
#ifndef SIM_PL_STAGES
#define SIM_PL_STAGES 3
#endif
#ifndef SIM_PL_BSTAGES
#define SIM_PL_BSTAGES 5
#endif
constexpr int kPlStages = SIM_PL_STAGES;           // V_hi stages
constexpr int kPlBStages = SIM_PL_BSTAGES;         // K tiles run further ahead (they come from HBM)
constexpr uint32_t kPlA = 3u * 16384u;            // V_hi: 3 components x 4 blocks x (32 rows x 128 B)
constexpr uint32_t kPlB = 16384u;                 // K hi (8 KB) + lo (8 KB), 64 x 32 each
constexpr uint32_t kPlBOff = kPlStages * kPlA;    // the K-tile stages follow the V_hi stages
constexpr size_t kPlSmem = (size_t)kPlStages * kPlA + (size_t)kPlBStages * kPlB + 1024;
constexpr uint32_t kPlLBO = 4096u, kPlSBO = 512u;
// D f32, A / B tf32, N = 64, M = 128; A MN-major (bit 15) for the shared-memory operand
constexpr uint32_t kIdescPlS = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescPlT = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

// MN-major tf32 operands take only the SWIZZLE_128B_BASE32B layout (layout type 1; measured:
// tools/probes/mma_layouts.cu): atom = 4 K-rows x 128 B (32 fp32 along M), 32-byte chunks XOR-permuted
// by the row (Swizzle<2,5,2>); LBO = 4 KB between 32-instance blocks, SBO = 512 B between 4-row groups
__device__ __forceinline__ uint64_t umma_desc_mn32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(kPlLBO >> 4) << 16) | ((uint64_t)(kPlSBO >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
__device__ __forceinline__ void umma_pl_ss(uint32_t dt, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
        "l"(da), "l"(db), "r"(kIdescPlS), "r"(acc)
        : "memory");
}
// warp-converged variants: the whole warp runs the issue loop (its descriptors are warp-uniform, so
// they live in uniform registers) and elect.sync picks the one lane that issues; the same lane (the
// lowest) issues every MMA and commit, as tcgen05.commit tracks the issuing thread's operations
__device__ __forceinline__ void umma_pl_ss_w(uint32_t dt, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
        "l"(da), "l"(db), "r"(kIdescPlS), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_pl_ts_w(uint32_t dt, uint32_t at, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dt),
        "r"(at), "l"(db), "r"(kIdescPlT), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit_w(uint64_t* bar) {
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                 " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void umma_pl_ts(uint32_t dt, uint32_t at, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dt),
        "r"(at), "l"(db), "r"(kIdescPlT), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void cp_async16_z(uint32_t saddr, const void* gmem, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

__device__ unsigned long long g_pl_clock[4][64][8];   // plane K-pass timeline of CTA (0, 0), first 64 tiles (SIM_PL_TIMELINE builds)
__device__ __forceinline__ void pl_stamp(int pass, int t, int k) {
#ifdef SIM_PL_TIMELINE   // build with SIM_NVCC_EXTRA=-DSIM_PL_TIMELINE for tools/pl_timeline.py
    if (blockIdx.x == 0 && blockIdx.y == 0 && t < 64) {
        unsigned long long v;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
        g_pl_clock[pass][t][k] = v;
    }
#endif
}
int debug_pl_clock(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_pl_clock, sizeof(g_pl_clock));
}
template <int PASS>
__global__ void __launch_bounds__(kPlThreads + 64, 1)
    k_kpass_pl(int S, int Sp, int n_f, const BUnit* __restrict__ units, const float* __restrict__ T,
               const int32_t* __restrict__ cover, const float* __restrict__ vin, float* __restrict__ yout,
               float* __restrict__ part, int* __restrict__ counters, int nchunks, double4* __restrict__ x,
               const double4* __restrict__ xt, double4* __restrict__ v, double inv_h, int finalize_v, int drain) {
    pdl_enter();
    extern __shared__ unsigned char pl_raw[];
    __shared__ __align__(8) uint64_t mdone[kPlStages], lofull[4], lofree[4], dfree;
    __shared__ __align__(8) uint64_t bfull[kPlBStages], bempty[kPlBStages];
    __shared__ uint32_t tmem_base_s;
    __shared__ int s_last;
    unsigned char* sm = pl_raw + ((1024u - ((unsigned)__cvta_generic_to_shared(pl_raw) & 1023u)) & 1023u);
    const uint32_t sm_a = (unsigned)__cvta_generic_to_shared(sm);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const bool mma_warp = w == kPlWarps, kload_warp = w == kPlWarps + 1;
#ifndef SIM_PL_CGROUP
#define SIM_PL_CGROUP 1
#endif
    // pass 1 launch order: groups of SIM_PL_CGROUP instance chunks run unit by unit (the chunks of a
    // group share each K tile in L2; 1 = all units of chunk 0, then chunk 1, ...)
    int unit = blockIdx.x, chunk = blockIdx.y;
    if (PASS == 1 && SIM_PL_CGROUP > 1) {
        const int G = SIM_PL_CGROUP, nu = gridDim.x, nc = gridDim.y;
        const int b = blockIdx.y * nu + blockIdx.x, full = (nc / G) * G * nu;
        if (b < full) {
            const int r = b % (G * nu);
            unit = r / G;
            chunk = (b / (G * nu)) * G + r % G;
        } else {
            const int g2 = nc - (nc / G) * G, r = b - full;
            unit = r / g2;
            chunk = (nc / G) * G + r % g2;
        }
    }
    const BUnit U = units[unit];
    const int i0 = chunk * kPlInst;
    const size_t PS = (size_t)n_f * Sp;            // plane stride
    const unsigned long long pol = l2_evict_first();
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&tmem_base_s)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 0) {
        // worker-side barriers count one elected arrival per worker warp (after __syncwarp)
        for (int s2 = 0; s2 < kPlStages; ++s2) mbar_init(&mdone[s2], 1);
        for (int k = 0; k < 4; ++k) {
            mbar_init(&lofull[k], kPlWarps);
            mbar_init(&lofree[k], 1);
        }
        for (int s2 = 0; s2 < kPlBStages; ++s2) {
            mbar_init(&bfull[s2], 1);
            mbar_init(&bempty[s2], 1);
        }
        mbar_init(&dfree, kPlWarps);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    const int nt = U.ntiles;
#ifdef SIM_PL_TIMELINE
    if (tid == 0) { pl_stamp(PASS - 1, 63, 0); if (blockIdx.x == 0 && blockIdx.y == 0) g_pl_clock[PASS - 1][62][0] = nt; }
#endif
    if (kload_warp) {
        // K tiles: one bulk copy each, kPlBStages ahead of the tensor core
        if (lane == 0) {
            for (int t = 0; t < nt; ++t) {
                const int sb = t % kPlBStages;
                if (t >= kPlBStages) mbar_wait(&bempty[sb], (unsigned)((t - kPlBStages) / kPlBStages) & 1u);
                mbar_expect_tx(&bfull[sb], kPlB);
                bulk_g2s(sm + kPlBOff + sb * kPlB, T + U.toff + (int64_t)t * 4096, kPlB, &bfull[sb], true, pol);
            }
        }
        __syncwarp();
    } else if (mma_warp) {
        {   // the whole warp runs the loop (uniform descriptors); one elected lane issues
            const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_base_s, 0);
            for (int t = 0; t < nt; ++t) {
                const int st = t % kPlStages, sb = t % kPlBStages;
                mbar_wait_w(&bfull[sb], (unsigned)(t / kPlBStages) & 1u);
                pl_stamp(PASS - 1, t, 0);
                if (t > 0 && t % drain == 0) mbar_wait_w(&dfree, (unsigned)(t / drain - 1) & 1u);
                const uint32_t abase = sm_a + st * kPlA, bbase = sm_a + kPlBOff + sb * kPlB;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    // V_lo of component c written (and this tile's V_hi copies visible to the tensor core)
                    const int sl = 3 * t + c, ks = sl & 3;   // V_lo slot of (t, c): 4 slots rotate over the 3 components
                    mbar_wait_w(&lofull[ks], (unsigned)(sl >> 2) & 1u);
                    if (c == 0) pl_stamp(PASS - 1, t, 1);
                    if (c == 2) pl_stamp(PASS - 1, t, 2);
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    const uint32_t dt = tmem + 128u * c;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t da = umma_desc_mn32(abase + 16384u * c + 1024u * kk);
                        const uint64_t db = umma_desc_k(bbase + 256u * kk);   // [K_hi ; K_lo]: N = 128
                        umma_pl_ss_w(dt, da, db, (t % drain != 0 || kk > 0) ? 1u : 0u);
                        umma_pl_ts_w(dt, tmem + 384u + 32u * ks + 8u * kk, db, 1u);      // V_lo K_hi: N = 64
                    }
                    umma_commit_w(&lofree[ks]);   // the lo slot may be rewritten
                }
                umma_commit_w(&mdone[st]);
                pl_stamp(PASS - 1, t, 3);
                umma_commit_w(&bempty[sb]);
            }
        }
        __syncwarp();
    } else {
        // ---- workers: copies, V_lo, folds ----
        // each worker warp copies exactly the V_hi rows it later reads for its V_lo (rows 8 oc .. 8 oc + 7
        // of the 32-instance block qd, 3 planes): 192 16-byte chunks per warp, 6 per lane; the warps
        // then need no CTA-wide barrier per tile (each waits for its own copies; the tensor core sees
        // every warp's through the lofull arrivals)
        const int qd = w & 3, oc = w >> 2;     // TMEM lane quadrant (= 32-instance block) / row octet
        const int ch = lane & 7;                // 16-byte chunk (4 instances) of a 128-byte row
        const int inst4 = i0 + 32 * qd + 4 * ch;
        const bool ilive4 = inst4 < Sp;
        uint32_t dsto[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int q = 8 * oc + (lane >> 3) + 4 * e;
            dsto[e] = 4096u * qd + 128u * q + 32u * ((ch >> 1) ^ (q & 3)) + 16u * (ch & 1);
        }
        // pass 2: the cover rows of a tile are read one tile before its copies are issued (the
        // dependent index load is off the copy issue path)
        int crow[2] = {0, 0};
        auto load_cover = [&](int t) {
            if (PASS == 2)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int q = 8 * oc + (lane >> 3) + 4 * e;
                    crow[e] = (t < nt && 32 * t + q < U.nlist) ? __ldg(&cover[U.list0 + 32 * t + q]) : 0;
                }
        };
        auto issue = [&](int t) {
            const int st = t % kPlStages;
            const uint32_t abase = sm_a + st * kPlA;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int q = 8 * oc + (lane >> 3) + 4 * e;
                int r;
                bool ok;
                if (PASS == 1) {
                    r = U.c0 + 32 * t + q;
                    ok = r < n_f;
                } else {
                    ok = 32 * t + q < U.nlist;
                    r = crow[e];
                }
                ok = ok && ilive4;
                const float* src = ok ? vin + (size_t)r * Sp + inst4 : vin;
                const uint32_t n = ok ? 16u : 0u;
#pragma unroll
                for (int c = 0; c < 3; ++c) cp_async16_z(abase + 16384u * c + dsto[e], ok ? src + c * PS : vin, n);
            }
            cp_async_commit();
        };
        const uint32_t lanebase = tmem + ((uint32_t)(32 * qd) << 16);
        float acc[3][16];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[c][e] = 0.f;
        auto fold = [&]() {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                uint32_t r[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15}, [%16];\n"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15])
                    : "r"(lanebase + 128u * c + 16u * oc));
                uint32_t q2[16];   // the V K_lo half of the accumulator
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15}, [%16];\n"
                    : "=r"(q2[0]), "=r"(q2[1]), "=r"(q2[2]), "=r"(q2[3]), "=r"(q2[4]), "=r"(q2[5]), "=r"(q2[6]), "=r"(q2[7]),
                      "=r"(q2[8]), "=r"(q2[9]), "=r"(q2[10]), "=r"(q2[11]), "=r"(q2[12]), "=r"(q2[13]), "=r"(q2[14]),
                      "=r"(q2[15])
                    : "r"(lanebase + 128u * c + 64u + 16u * oc));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[c][e] += __uint_as_float(r[e]) + __uint_as_float(q2[e]);
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        };
        load_cover(0);
        issue(0);
        load_cover(1);
        if (nt > 1) issue(1);
        load_cover(2);
        // per tile t: V_lo(t) as soon as its copies landed (MMA(t - 1) runs meanwhile), then the fold
        // of a closed accumulation group, then the copies of tile t + 2 into the stage MMA(t - 1) frees
        for (int t = 0; t < nt; ++t) {
            const int st = t % kPlStages;
            // this thread's copies of tile t have landed (tile t + 1's may still fly), then the warp's
            if (t + 1 < nt) cp_async_wait<1>(); else cp_async_wait<0>();
            __syncwarp();
            if (tid == 0) pl_stamp(PASS - 1, t, 4);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // cp.async data -> async proxy
            // V_lo of rows 8 oc .. 8 oc + 7 (K-step oc) for instance 32 qd + lane, one component at a
            // time into its TMEM slot once the tensor core has read the previous tile's
            const unsigned char* ab = sm + st * kPlA + 4096 * qd;
            uint32_t lo3[3][8];   // all three components first: the shared-memory loads leave the hand-off path
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int q = 8 * oc + r;
                    const float a = *reinterpret_cast<const float*>(ab + 16384 * c + 128 * q + 32 * ((lane >> 3) ^ (q & 3)) +
                                                                    4 * (lane & 7));
                    lo3[c][r] = __float_as_uint(tf32_rn(a - tf32_trunc(a)));
                }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint32_t* lo = lo3[c];
                const int sl = 3 * t + c, ks = sl & 3;
                if (sl >= 4) mbar_wait(&lofree[ks], (unsigned)((sl >> 2) - 1) & 1u);   // its previous MMA read it
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
                                 lanebase + 384u + 32u * ks + 8u * oc),
                             "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7])
                             : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&lofull[ks]);
            }
            if (tid == 0) pl_stamp(PASS - 1, t, 5);
            // the group of tiles ending at t - 1 is complete once MMA(t - 1) is: fold it, free D
            if (t > 0 && t % drain == 0) {
                mbar_wait(&mdone[(t - 1) % kPlStages], (unsigned)((t - 1) / kPlStages) & 1u);
                fold();
                __syncwarp();
                if (lane == 0) mbar_arrive(&dfree);
            }
            if (tid == 0) pl_stamp(PASS - 1, t, 6);
            if (t + 2 < nt) {
                // stage (t + 2) % kPlStages was last read by MMA(t + 2 - kPlStages); every worker has
                // passed this iteration's barrier, i.e. finished its V_lo reads of that stage
                const int tp = t + 2 - kPlStages;
                if (tp >= 0) mbar_wait(&mdone[tp % kPlStages], (unsigned)((tp / kPlStages) & 1));
                issue(t + 2);
                load_cover(t + 3);
            }
            if (tid == 0) pl_stamp(PASS - 1, t, 7);
        }
        if (nt > 0) {
            mbar_wait(&mdone[(nt - 1) % kPlStages], (unsigned)((nt - 1) / kPlStages) & 1u);
            fold();
        }
        // ---- epilogue: thread = instance i0 + 32 qd + lane, outputs 16 oc .. 16 oc + 15 ----
        const int inst = i0 + 32 * qd + lane;
        const bool live = inst < S;
        if (PASS == 2) {
            if (live) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int l = 16 * oc + e;
                    if (l < U.nr) {
                        const size_t jx = (size_t)(U.c0 + l) * S + inst;
                        double4 xj = x[jx];
                        xj.x += (double)acc[0][e];
                        xj.y += (double)acc[1][e];
                        xj.z += (double)acc[2][e];
                        x[jx] = xj;
                        if (finalize_v) {   // v = (x - x_t) / h
                            const double4 t0 = xt[jx];
                            v[jx] = make_double4((xj.x - t0.x) * inv_h, (xj.y - t0.y) * inv_h, (xj.z - t0.z) * inv_h, 0.0);
                        }
                    }
                }
            }
        } else if (U.nparts == 1) {
            if (live) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int l = 16 * oc + e;
                    if (l < U.nr) {
                        const size_t iy = (size_t)(U.r0 + l) * Sp + inst;
                        yout[iy] = acc[0][e];
                        yout[PS + iy] = acc[1][e];
                        yout[2 * PS + iy] = acc[2][e];
                    }
                }
            }
        } else {
            // a block split over several units: fp32 partials [part][3][64][Sp], summed in fp64 in
            // part order by the last unit to arrive
            const size_t pst = (size_t)64 * Sp;
            if (live) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    float* pp = part + (size_t)U.part * 3 * pst + (size_t)(16 * oc + e) * Sp + inst;
                    pp[0] = acc[0][e];
                    pp[pst] = acc[1][e];
                    pp[2 * pst] = acc[2][e];
                }
            }
            __threadfence();
            asm volatile("bar.sync 1, %0;\n" ::"r"(kPlThreads));
            if (tid == 0) {
                const int old = atomicAdd(&counters[U.block * nchunks + chunk], 1);
                s_last = old == U.nparts - 1;
            }
            asm volatile("bar.sync 1, %0;\n" ::"r"(kPlThreads));
            if (s_last) {
                __threadfence();
                if (live) {
                    for (int e = 0; e < 16; ++e) {
                        const int l = 16 * oc + e;
                        if (l >= U.nr) continue;
                        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
                        for (int q = 0; q < U.nparts; ++q) {
                            const float* pq = part + (size_t)(U.list0 + q) * 3 * pst + (size_t)l * Sp + inst;
                            t0 += (double)__ldcg(pq);
                            t1 += (double)__ldcg(pq + pst);
                            t2 += (double)__ldcg(pq + 2 * pst);
                        }
                        const size_t iy = (size_t)(U.r0 + l) * Sp + inst;
                        yout[iy] = (float)t0;
                        yout[PS + iy] = (float)t1;
                        yout[2 * PS + iy] = (float)t2;
                    }
                }
                if (tid == 0) counters[U.block * nchunks + chunk] = 0;
            }
        }
    }
    __syncthreads();
    if (w == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u) : "memory");
}

void launch_kpass1_pl(cudaStream_t st, int S, int Sp, int n_f, int nunits, const BUnit* units, const float* T,
                      const float* u, float* y, float* part, int* counters, int drain) {
    static unsigned long long attr = 0;
    per_device_once(attr, [&] {
        cudaFuncSetAttribute(k_kpass_pl<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPlSmem);
    });
    const int nch = (S + kPlInst - 1) / kPlInst;
    launch_pdl(k_kpass_pl<1>, dim3(nunits, nch), dim3(kPlThreads + 64), kPlSmem, st, S, Sp, n_f, units, T,
               (const int32_t*)nullptr, u, y, part, counters, nch, (double4*)nullptr, (const double4*)nullptr,
               (double4*)nullptr, 0.0, 0, drain);
}

void launch_kpass2_pl(cudaStream_t st, int S, int Sp, int n_f, int nunits, const BUnit* units, const int32_t* cover,
                      const float* T, const float* y, double4* x, const double4* xt, double4* v, double inv_h,
                      int finalize_v, int drain) {
    static unsigned long long attr = 0;
    per_device_once(attr, [&] {
        cudaFuncSetAttribute(k_kpass_pl<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPlSmem);
    });
    const int nch = (S + kPlInst - 1) / kPlInst;
    launch_pdl(k_kpass_pl<2>, dim3(nunits, nch), dim3(kPlThreads + 64), kPlSmem, st, S, Sp, n_f, units, T, cover, y,
               (float*)nullptr, (float*)nullptr, (int*)nullptr, nch, x, xt, v, inv_h, finalize_v, drain);
}

// ----------------------------------------------------------------------------
// TS variant: the right-hand-side operand (A, hi and lo, 3 components) goes from registers to
// TMEM with tcgen05.st instead of through shared memory, and the MMAs read A from TMEM
// (tcgen05.mma ... [d], [a_tmem], b_desc): shared memory only holds the K tiles.  TMEM: the
// accumulators in columns [0, 96), A stage s in [128 + 192 s, 320 + 192 s) as 6 planes of 32
// columns (component c hi / lo), lane = instance.  One accumulator set: it is folded into
// fp64 every `drain` tiles while the pipeline waits.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void chain_rho(int S, int inst, int s, double t0, double t1, double t2, CrContacts cc,
                                          const double4* __restrict__ x, ContactState cs);

__device__ __forceinline__ void umma_tf32_ts(uint32_t dt, uint32_t at, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dt),
        "r"(at), "l"(db), "r"(kIdescTf32), "r"(acc)
        : "memory");
}

// warp-converged issue (see umma_pl_ss_w)
__device__ __forceinline__ void umma_tf32_ts_w(uint32_t dt, uint32_t at, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dt),
        "r"(at), "l"(db), "r"(kIdescTf32), "r"(acc)
        : "memory");
}

template <int PASS>
__global__ void __launch_bounds__(kTcThreads + 32, 1)
    k_kpass_ts(int S, int n_f, const BUnit* __restrict__ units, const float* __restrict__ Ttc,
               const int32_t* __restrict__ cover, const float4* __restrict__ vin, float4* __restrict__ yout,
               double* __restrict__ part, int* __restrict__ counters, int nchunks, double4* __restrict__ x,
               const double4* __restrict__ xt, double4* __restrict__ v, double inv_h, int finalize_v, int drain,
               TsExtra ex) {
    pdl_enter();
    __shared__ __align__(128) unsigned char bsm[2][8192];
    __shared__ __align__(8) uint64_t bfull[2], mdone[2], afull[2];
    __shared__ uint32_t tmem_base_s;
    __shared__ int s_last;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const bool mma_warp = w == kTcThreads / 32;
    // grid order: pass 1 runs unit-fastest (the units in flight share right-hand-side columns of one
    // instance chunk in L2: 2.3 GB of DRAM traffic per launch at S = 1024, 5.8 GB chunk-fastest);
    // the other passes run chunk-fastest (the chunks of one unit share its K tiles in L2: pass 2
    // 2.6 -> 2.1 GB, 1.7 % faster; chain / scatter 3 % faster)
    constexpr bool kChunkFast = PASS != 1;
    const BUnit U = units[kChunkFast ? blockIdx.y : blockIdx.x];
    const int chunk = kChunkFast ? blockIdx.x : blockIdx.y;
    const int i0 = chunk * kTcInst;
    const int ni = min(kTcInst, S - i0);
    const unsigned long long pol = l2_evict_first();
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&tmem_base_s)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bfull[0], 1);
        mbar_init(&bfull[1], 1);
        mbar_init(&mdone[0], 1);
        mbar_init(&mdone[1], 1);
        mbar_init(&afull[0], kTcThreads);
        mbar_init(&afull[1], kTcThreads);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    auto acol = [&](int st, int c, int hl) { return 128u + 192u * st + 32u * (2 * c + hl); };
    auto issueB = [&](int t) {
        const int st = t & 1;
        mbar_expect_tx(&bfull[st], 8192u);
        bulk_g2s(bsm[st], Ttc + 2 * U.toff + (int64_t)t * 2048, 8192u, &bfull[st], true, pol);
    };
    if (tid == 0) {
        issueB(0);
        if (U.ntiles > 1) issueB(1);
    }
    const int q4 = w & 3, oct = w >> 2;    // TMEM lane quadrant; producer row octet / fold column octet
    const int il = 32 * q4 + lane;         // instance of this thread (TMEM lane)
    const bool ilive = il < ni;
    double dacc[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e) dacc[c][e] = 0.0;
    auto fold = [&]() {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const uint32_t ta = tmem + ((uint32_t)(32 * q4) << 16) + 32u * c + 8u * oct;
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                           "=r"(r[7])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int e = 0; e < 8; ++e) dacc[c][e] += (double)__uint_as_float(r[e]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    };
    if (mma_warp) {
        {   // the whole warp runs the loop (uniform descriptors); one elected lane issues
            const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_base_s, 0);
            for (int t = 0; t < U.ntiles; ++t) {
                const int st = t & 1;
                mbar_wait_w(&afull[st], (t >> 1) & 1);
                mbar_wait_w(&bfull[st], (t >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const uint32_t b0 = (unsigned)__cvta_generic_to_shared(bsm[st]);
                const uint32_t b1 = b0 + 4096u;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const uint32_t dt = tmem + 32u * c;
                    const uint32_t ah = tmem + acol(st, c, 0), al = tmem + acol(st, c, 1);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t dbh = umma_desc_k(b0 + 256u * kk), dbl = umma_desc_k(b1 + 256u * kk);
                        umma_tf32_ts_w(dt, ah + 8u * kk, dbh, (t % drain != 0 || kk > 0) ? 1u : 0u);
                        umma_tf32_ts_w(dt, al + 8u * kk, dbh, 1u);
                        umma_tf32_ts_w(dt, ah + 8u * kk, dbl, 1u);
                    }
                }
                umma_commit_w(&mdone[st]);
            }
        }
        __syncwarp();
    } else {
        for (int t = 0; t < U.ntiles; ++t) {
            const int st = t & 1;
            // PASS 4: contiguous reduction indices (slots); PASS 3: a chain-row list
            constexpr bool kContig = PASS == 4;
            const int nv = kContig ? max(0, min(32, n_f - (U.c0 + 32 * t))) : min(32, U.nlist - 32 * t);
            float4 r[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int q = 8 * oct + e;
                r[e] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (ilive && q < nv) {
                    if (PASS == 4) {   // wz^T, float4 [slot][S]
                        r[e] = __ldg(&vin[(size_t)(U.c0 + 32 * t + q) * S + i0 + il]);
                    } else {           // y at a chain row (planes, vec_ld)
                        r[e] = vec_ld(vin, S, ex.nf, __ldg(&cover[U.list0 + 32 * t + q]), i0 + il);
                    }
                }
            }
            if (t > 0 && t % drain == 0) {   // accumulators complete up to tile t - 1: fold, restart
                mbar_wait(&mdone[(t - 1) & 1], ((t - 1) >> 1) & 1);
                fold();
            }
            if (t >= 2) {
                mbar_wait(&mdone[st], ((t - 2) >> 1) & 1);   // the tensor core is done with A / B stage st
                if (tid == 0) issueB(t);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                uint32_t hi[8], lo[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float a = c == 0 ? r[e].x : (c == 1 ? r[e].y : r[e].z);
                    const float h = tf32_rn(a);
                    hi[e] = __float_as_uint(h);
                    lo[e] = __float_as_uint(tf32_rn(a - h));
                }
                const uint32_t lanebase = tmem + ((uint32_t)(32 * q4) << 16) + 8u * oct;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
                                 lanebase + acol(st, c, 0)),
                             "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]),
                             "r"(hi[7])
                             : "memory");
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
                                 lanebase + acol(st, c, 1)),
                             "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]),
                             "r"(lo[7])
                             : "memory");
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&afull[st]))
                         : "memory");
        }
        const int last = U.ntiles - 1;
        if (last >= 0) {
            mbar_wait(&mdone[last & 1], (last >> 1) & 1);
            fold();
        }
    }
    __syncthreads();
    if (w == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u) : "memory");
    if (mma_warp) return;
    const int li = il;
    const bool live = li < ni;
    const int inst = i0 + li;
    if (PASS == 3 && U.nparts == 1) {   // chain pass: dxt (and the Schur RHS of the slot's single contact) per slot
        if (!live) return;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int l = 8 * oct + r;
            if (l < U.nr) chain_rho(S, inst, ex.soff[inst] + U.c0 + l, dacc[0][r], dacc[1][r], dacc[2][r], ex.cc, ex.xs,
                                    ex.cs);
        }
        return;
    }
    if (PASS == 4 && U.nparts == 1) {   // scatter pass: y[row] += K H^T z on the chain rows
        if (!live) return;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int l = 8 * oct + r;
            if (l < U.nr) vec_add(yout, S, ex.nf, ex.orows[U.r0 + l], inst, dacc[0][r], dacc[1][r], dacc[2][r]);
        }
        return;
    }
    const size_t pstride = (size_t)32 * S;
    if (live) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int l = 8 * oct + r;
            double* pp = part + (size_t)U.part * 3 * pstride + (size_t)l * S + inst;
            pp[0] = dacc[0][r];
            pp[pstride] = dacc[1][r];
            pp[2 * pstride] = dacc[2][r];
        }
    }
    __threadfence();
    asm volatile("bar.sync 1, %0;\n" ::"r"(kTcThreads));   // producers only (the MMA warp has left)
    if (threadIdx.x == 0) {
        const int old = atomicAdd(&counters[U.block * nchunks + chunk], 1);
        s_last = old == U.nparts - 1;
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(kTcThreads));
    if (!s_last) return;
    __threadfence();
    const int first = U.pad;   // the block's first partial slot
    if (live) {
        for (int r = 0; r < 8; ++r) {
            const int l = 8 * oct + r;
            if (l >= U.nr) continue;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int q = 0; q < U.nparts; ++q) {
                const double* pq = part + (size_t)(first + q) * 3 * pstride + (size_t)l * S + inst;
                t0 += __ldcg(pq);
                t1 += __ldcg(pq + pstride);
                t2 += __ldcg(pq + 2 * pstride);
            }
            if (PASS == 3) {
                chain_rho(S, inst, ex.soff[inst] + U.c0 + l, t0, t1, t2, ex.cc, ex.xs, ex.cs);
            } else {
                vec_add(yout, S, ex.nf, ex.orows[U.r0 + l], inst, t0, t1, t2);
            }
        }
    }
    if (threadIdx.x == 0) counters[U.block * nchunks + chunk] = 0;
}

void launch_chain_pass_ts(cudaStream_t st, int S, int nf, int nunits, const BUnit* units, const float* Ttc,
                          const int32_t* cover, const float4* y, const int* soff, CrContacts cc, const double4* x,
                          ContactState cs, int drain, double* part, int* counters) {
    if (nunits == 0) return;
    const int nch = (S + kTcInst - 1) / kTcInst;
    TsExtra ex{nullptr, soff, cc, x, cs, nf};
    launch_pdl(k_kpass_ts<3>, dim3(nch, nunits), dim3(kTcThreads + 32), 0, st, S, 0, units, Ttc, cover, y,
               (float4*)nullptr, part, counters, nch, (double4*)nullptr, (const double4*)nullptr,
               (double4*)nullptr, 0.0, 0, drain, ex);
}

void launch_scatter_pass_ts(cudaStream_t st, int S, int nf, int ns, int nunits, const BUnit* units, const float* Ttc,
                            const int32_t* rows, const float4* wzT, float4* y, int drain, double* part,
                            int* counters) {
    if (nunits == 0) return;
    const int nch = (S + kTcInst - 1) / kTcInst;
    TsExtra ex{rows, nullptr, CrContacts{}, nullptr, ContactState{}, nf};
    launch_pdl(k_kpass_ts<4>, dim3(nch, nunits), dim3(kTcThreads + 32), 0, st, S, ns, units, Ttc,
               (const int32_t*)nullptr, wzT, y, part, counters, nch, (double4*)nullptr,
               (const double4*)nullptr, (double4*)nullptr, 0.0, 0, drain, ex);
}


// ----------------------------------------------------------------------------
// chain dot: dxt_s = (K^T y)_{a_s} = sum_k Kcol[colptr_a + k] y[chain_rows[off + k]]
// (column a of K is contiguous in Kcol; its rows are a's ancestor chain).  One CTA per
// (class slot, up to 32 instances of the class): the chain is read once for the group.
//   group of 1: 8 warps take interleaved 128-entry slices, lanes split the entries;
//   larger groups: lane = instance (coalesced y rows, instance-minor), warps split the chain.
// Thread 0 / lane l also forms the Schur RHS rho = h - theta J x~ for the slot's single
// single-vertex contact, x~ = x^k + K^T y (other contacts are handled in the CR prologue).
// ----------------------------------------------------------------------------
__device__ __forceinline__ void chain_rho(int S, int inst, int s, double t0, double t1, double t2, CrContacts cc,
                                          const double4* __restrict__ x, ContactState cs) {
    cs.dxt[3 * s] = t0;
    cs.dxt[3 * s + 1] = t1;
    cs.dxt[3 * s + 2] = t2;
    const int c = cc.c1[s];
    if (c >= 0) {
        const double4 xa = x[(size_t)cc.v0[c] * S + inst];
        const double xs0 = xa.x + t0, xs1 = xa.y + t1, xs2 = xa.z + t2;
        // the fp64 rows the h-vector's theta J x^k was formed with: its x^k terms cancel to fp64
        // rounding here (fp32 rows would leave a bias of ~6e-8 |x^k| in rho)
        const DContact& ct = cc.dc[c];
#pragma unroll
        for (int kk = 0; kk < 3; ++kk)
            cs.rho[3 * c + kk] = cs.hvec[3 * c + kk] -
                                 cs.theta[3 * c + kk] * (ct.c[kk][0] * xs0 + ct.c[kk][1] * xs1 + ct.c[kk][2] * xs2);
    }
}

__global__ void __launch_bounds__(256) k_chain_dot(int S, int n_f, InstOff off, ClassSlots csl, const float* __restrict__ Kcol,
                                                   const int64_t* __restrict__ colptr,
                                                   const int32_t* __restrict__ chain_off,
                                                   const int32_t* __restrict__ chain_rows, const float4* __restrict__ y,
                                                   CrContacts cc, const double4* __restrict__ x, ContactState cs,
                                                   const int2* __restrict__ items) {
    pdl_enter();
    __shared__ double s_red[3][kWarps][32];
    const int2 it = items[blockIdx.x];
    const int g = it.x, cl = csl.cls[g];
    const int m0 = it.y, gs = min(32, off.cmoff[cl + 1] - m0);
    const int sloc = g - off.csoff[cl];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int a = csl.vtx[g];
    const float* col = Kcol + colptr[a];
    const int o0 = chain_off[g], len = chain_off[g + 1] - o0;
    double a0 = 0, a1 = 0, a2 = 0;
    if (gs == 1) {
        const int inst = off.cmem[m0];
        for (int k0 = 128 * w; k0 < len; k0 += 128 * kWarps) {   // 4 independent gathers in flight per lane
            int rw[4];
            float kv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + 32 * u + lane;
                rw[u] = k < len ? __ldg(&chain_rows[o0 + k]) : -1;
                kv[u] = k < len ? __ldg(&col[k]) : 0.f;
            }
            float4 yy[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                yy[u] = rw[u] >= 0 ? vec_ld(y, S, n_f, rw[u], inst) : make_float4(0.f, 0.f, 0.f, 0.f);
            float f0 = 0.f, f1 = 0.f, f2 = 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                f0 = fmaf(kv[u], yy[u].x, f0);
                f1 = fmaf(kv[u], yy[u].y, f1);
                f2 = fmaf(kv[u], yy[u].z, f2);
            }
            a0 += (double)f0;
            a1 += (double)f1;
            a2 += (double)f2;
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        a2 = warp_sum(a2);
        if (lane == 0) {
            s_red[0][w][0] = a0;
            s_red[1][w][0] = a1;
            s_red[2][w][0] = a2;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
            for (int q = 0; q < kWarps; ++q) { t0 += s_red[0][q][0]; t1 += s_red[1][q][0]; t2 += s_red[2][q][0]; }
            chain_rho(S, inst, off.soff[inst] + sloc, t0, t1, t2, cc, x, cs);
        }
        return;
    }
    // lanes = instances of the group; warp w walks the whole chain of class slot it.x + w
    // (8 neighbouring slots share most of their ancestors: their y rows hit in L1)
    const int gw = g + w;
    if (gw >= off.csoff[cl + 1]) return;
    const int inst = off.cmem[m0 + min(lane, gs - 1)];
    const float* colw = Kcol + colptr[csl.vtx[gw]];
    const int ow = chain_off[gw], lw = chain_off[gw + 1] - ow;
    for (int k0 = 0; k0 < lw; k0 += 32) {
        const int n = min(32, lw - k0);
        const int rmine = lane < n ? __ldg(&chain_rows[ow + k0 + lane]) : 0;
        const float kmine = lane < n ? __ldg(&colw[k0 + lane]) : 0.f;
        float f0 = 0.f, f1 = 0.f, f2 = 0.f;
#pragma unroll 8
        for (int q = 0; q < n; ++q) {
            const int r = __shfl_sync(0xffffffffu, rmine, q);
            const float kv = __shfl_sync(0xffffffffu, kmine, q);
            const float4 yv = vec_ld(y, S, n_f, r, inst);
            f0 = fmaf(kv, yv.x, f0);
            f1 = fmaf(kv, yv.y, f1);
            f2 = fmaf(kv, yv.z, f2);
        }
        a0 += (double)f0;
        a1 += (double)f1;
        a2 += (double)f2;
    }
    if (lane < gs) chain_rho(S, inst, off.soff[inst] + (gw - off.csoff[cl]), a0, a1, a2, cc, x, cs);
}

void launch_chain_dot(cudaStream_t st, const Params& P, InstOff off, ClassSlots csl, const float* Kcol,
                      const int64_t* colptr, const int32_t* chain_off, const int32_t* chain_rows, const float4* y,
                      Slots sl, CrContacts cc, const double4* x, ContactState cs, int nitems, const int2* items) {
    if (P.NS == 0 || nitems == 0) return;
    (void)sl;
    launch_pdl(k_chain_dot, dim3(nitems), dim3(32 * kWarps), 0, st, P.S, P.n_f, off, csl, Kcol, colptr, chain_off, chain_rows,
               y, cc, x, cs, items);
}

// ----------------------------------------------------------------------------
// active contact vertices of this iteration (any incident row with theta != 0), in
// ascending slot order, and the active block G_A of the Delassus Gram.  These depend only
// on theta, so they run in a graph branch beside the RHS gather and K-pass 1.
// ----------------------------------------------------------------------------
__host__ __device__ bool cr_ga_direct(int nc, int ns, int na, int csize);
__global__ void __launch_bounds__(1024) k_active(InstOff off, CrContacts cc, Slots sl, ContactState cs,
                                                 CrActive act, int csize, const float* __restrict__ G,
                                                 float* __restrict__ GA) {
    pdl_enter();
    __shared__ int wsum[32];
    __shared__ int base;
    const int inst = blockIdx.x;
    const int sb = off.soff[inst], ns = off.soff[inst + 1] - sb, cb = off.coff[inst];
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int b0 = 0; b0 < ns; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        bool on = false;
        int only = -1;
        if (b < ns) {
            only = cc.c1[sb + b];
            if (only >= 0) {
                on = cs.theta[3 * only] != 0.0 || cs.theta[3 * only + 1] != 0.0 || cs.theta[3 * only + 2] != 0.0;
            } else {
                for (int q = sl.scp[sb + b]; q < sl.scp[sb + b + 1] && !on; ++q) {
                    const int c = sl.sci[q];
                    on = cs.theta[3 * c] != 0.0 || cs.theta[3 * c + 1] != 0.0 || cs.theta[3 * c + 2] != 0.0;
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int pos = base;
        for (int q = 0; q < wid; ++q) pos += wsum[q];
        pos += __popc(bal & ((1u << lane) - 1u));
        if (b < ns) {
            act.apos[sb + b] = on ? pos : -1;
            if (on) {
                act.aidx[sb + pos] = b;
                act.acon[sb + pos] = only >= 0 ? only - cb : -1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = base;
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += wsum[q];
            base = t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) act.na[inst] = base;
    // G_A[i][j] = G[aidx_i][aidx_j] for a lone-CTA CR whose G_A does not fit in shared memory (one
    // warp per row; k_gather_ga serves the cluster CR); the CR gathers it into shared memory otherwise
    const int na = base, nc = off.coff[inst + 1] - cb;
    if (na == 0 || csize != 1 || cr_ga_direct(nc, ns, na, csize)) return;
    const float* Gc = G + off.goff[off.cls[inst]];
    float* GAi = GA + off.gaoff[inst];
    for (int i = wid; i < na; i += blockDim.x >> 5) {
        const float* Gi = Gc + (size_t)act.aidx[sb + i] * ns;
        for (int j = lane; j < na; j += 32) GAi[(size_t)i * na + j] = Gi[act.aidx[sb + j]];
    }
}

// G_A[i][j] = G[aidx_i][aidx_j] (instance blockIdx.y, active row blockIdx.x): the cluster CR (few
// instances), whose CTAs each copy their rows of G_A from this global copy
__global__ void __launch_bounds__(256) k_gather_ga(InstOff off, const float* __restrict__ G, CrActive act,
                                                   float* __restrict__ GA) {
    pdl_enter();
    const int inst = blockIdx.y;
    const int na = act.na[inst];
    const int i = blockIdx.x;
    if (i >= na) return;
    const int sb = off.soff[inst], ns = off.soff[inst + 1] - sb;
    const float* Gi = G + off.goff[off.cls[inst]] + (size_t)act.aidx[sb + i] * ns;
    float* GAi = GA + off.gaoff[inst] + (size_t)i * na;
    for (int j = threadIdx.x; j < na; j += blockDim.x) GAi[j] = Gi[act.aidx[sb + j]];
}

void launch_active(cudaStream_t st, const Params& P, InstOff off, CrContacts cc, Slots sl, ContactState cs,
                   CrActive act, const float* G, float* GA) {
    if (P.NS == 0) return;
    const int csize = cr_cluster_size(P.S);
    if (csize > 1) return;   // the cluster CR builds the active list and G_A itself
    k_active<<<P.S, 1024, 0, st>>>(off, cc, sl, cs, act, csize, G, GA);
}

// per-contact-set: chain rows of every class slot (walk panel runs), per-class row flags;
// warp w also writes slotmap for instance slot w
__global__ void k_chain_rows(Params P, ClassSlots csl, Slots sl, const int32_t* __restrict__ chain_off,
                             const int32_t* __restrict__ parent, const int32_t* __restrict__ ptop,
                             int32_t* __restrict__ chain_rows, uint8_t* __restrict__ flag,
                             int32_t* __restrict__ slotmap) {
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s < P.NS && lane == 0) slotmap[(size_t)sl.vtx[s] * P.S + sl.inst[s]] = s;
    if (s >= P.CS) return;
    uint8_t* fl = flag + (size_t)csl.cls[s] * P.n_f;
    int pos = chain_off[s];
    for (int i = csl.vtx[s]; i >= 0;) {
        const int top = ptop[i];
        const int len = top - i + 1;
        for (int o = lane; o < len; o += 32) {
            chain_rows[pos + o] = i + o;
            fl[i + o] = 1;
        }
        pos += len;
        i = parent[top];
    }
}

void launch_chain_rows(cudaStream_t st, const Params& P, ClassSlots csl, Slots sl, const int32_t* chain_off,
                       const int32_t* parent, const int32_t* ptop, int32_t* chain_rows, uint8_t* flag,
                       int32_t* slotmap) {
    const int n = std::max(P.NS, P.CS);
    if (n == 0) return;
    k_chain_rows<<<(n + 7) / 8, 256, 0, st>>>(P, csl, sl, chain_off, parent, ptop, chain_rows, flag, slotmap);
}

// rows on any chain of class blockIdx.y, with the class-local slot range in their subtree
// [first(i), i] and an offset into the compact copy Zc of K[i][a_s], s in [s0, s1)
__global__ void k_ulist(int n_f, InstOff off, const uint8_t* __restrict__ flag, ClassSlots csl,
                        const int2* __restrict__ meta, int* __restrict__ ucount, int4* __restrict__ ulist) {
    const int c = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_f || !flag[(size_t)c * n_f + i]) return;
    const int sb = off.csoff[c], ns = off.csoff[c + 1] - sb;
    const int32_t* v = csl.vtx + sb;
    const int f = meta[i].y;
    int lo = 0, hi = ns;
    while (lo < hi) { int m = (lo + hi) >> 1; if (v[m] < f) lo = m + 1; else hi = m; }
    const int s0 = lo;
    hi = ns;
    while (lo < hi) { int m = (lo + hi) >> 1; if (v[m] <= i) lo = m + 1; else hi = m; }
    // list order and offsets are arbitrary but each row's values stay contiguous
    const int idx = atomicAdd(&ucount[2 * c], 1);
    const int o = atomicAdd(&ucount[2 * c + 1], lo - s0);
    ulist[off.uoff[c] + idx] = make_int4(i, s0, lo, (int)(off.zoff[c] + o));
}

// Zc[off + s - s0] = K[i][a_s]  (one warp per listed row)
__global__ void k_zfill(InstOff off, const int* __restrict__ ucount, const int4* __restrict__ ulist, ClassSlots csl,
                        const float* __restrict__ Krow, const int2* __restrict__ meta, float* __restrict__ Zc) {
    const int c = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int cnt = ucount[2 * c];
    const int4* ul = ulist + off.uoff[c];
    const int32_t* v = csl.vtx + off.csoff[c];
    for (int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += nw) {
        const int4 u = ul[e];
        const float* row = Krow + meta[u.x].x;
        for (int s = u.y + lane; s < u.z; s += 32) Zc[u.w + s - u.y] = row[v[s]];
    }
}

void launch_ulist(cudaStream_t st, const Params& P, InstOff off, const uint8_t* flag, ClassSlots csl,
                  const int2* meta, int* ucount, int4* ulist, const float* Krow, float* Zc) {
    if (P.CS == 0) return;
    k_ulist<<<dim3((P.n_f + 255) / 256, P.NCL), 256, 0, st>>>(P.n_f, off, flag, csl, meta, ucount, ulist);
    const int gx = P.NCL >= 148 ? 4 : (148 * 4 + P.NCL - 1) / P.NCL;
    k_zfill<<<dim3(gx, P.NCL), 256, 0, st>>>(off, ucount, ulist, csl, Krow, meta, Zc);
}

// ----------------------------------------------------------------------------
// scatter (P:L956 correction, delta form): y_i += sum_{s0 <= s < s1} K[i][a_s] wz_s
// for the rows i on the class's chains.  Item = (class, 32 members):
//   group of 1: warp per row, lanes split the slot range (4 loads in flight per lane);
//   larger groups: warp per row, lane = instance (coalesced y), slots in sequence.
// ----------------------------------------------------------------------------
__global__ void k_scatter(int S, int n_f, InstOff off, const int* __restrict__ ucount, const int4* __restrict__ ulist,
                          const float* __restrict__ Zc, const double* __restrict__ wz,
                          const float4* __restrict__ wzT, float4* __restrict__ y, const int2* __restrict__ items) {
    pdl_enter();
    const int2 it = items[blockIdx.y];
    const int c = it.x, m0 = it.y, gs = min(32, off.cmoff[c + 1] - m0);
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int cnt = ucount[2 * c];
    const int4* ul = ulist + off.uoff[c];
    if (gs == 1) {
        const int inst = off.cmem[m0];
        const double* wzi = wz + 3 * (size_t)off.soff[inst];
        for (int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += nw) {
            const int4 u = ul[e];
            const float* zr = Zc + u.w - u.y;   // zr[s] = K[i][a_s]
            double a0 = 0, a1 = 0, a2 = 0;
            for (int s0 = u.y; s0 < u.z; s0 += 128) {
                double kv[4], w0[4], w1[4], w2[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int sq = s0 + 32 * q + lane;
                    const bool ok = sq < u.z;
                    const int iq = ok ? sq : u.y;
                    kv[q] = ok ? (double)__ldg(&zr[sq]) : 0.0;
                    w0[q] = __ldg(&wzi[3 * iq]);
                    w1[q] = __ldg(&wzi[3 * iq + 1]);
                    w2[q] = __ldg(&wzi[3 * iq + 2]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a0 = fma(kv[q], w0[q], a0);
                    a1 = fma(kv[q], w1[q], a1);
                    a2 = fma(kv[q], w2[q], a2);
                }
            }
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            a2 = warp_sum(a2);
            if (lane == 0) vec_add(y, S, n_f, u.x, inst, a0, a1, a2);
        }
        return;
    }
    // lanes = instances: wz^T rows (instance-minor float4) read coalesced; fp32 FMAs over 32-slot
    // chunks folded into fp64 (as the K-passes)
    const bool live = lane < gs;
    const int inst = off.cmem[m0 + min(lane, gs - 1)];
    for (int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += nw) {
        const int4 u = ul[e];
        const float* zr = Zc + u.w - u.y;
        double a0 = 0, a1 = 0, a2 = 0;
        for (int s0 = u.y; s0 < u.z; s0 += 32) {
            const int n = min(32, u.z - s0);
            const float zmine = lane < n ? __ldg(&zr[s0 + lane]) : 0.f;
            float f0 = 0.f, f1 = 0.f, f2 = 0.f;
#pragma unroll 8
            for (int q = 0; q < n; ++q) {
                const float kv = __shfl_sync(0xffffffffu, zmine, q);
                const float4 wv = __ldg(&wzT[(size_t)(s0 + q) * S + inst]);
                f0 = fmaf(kv, wv.x, f0);
                f1 = fmaf(kv, wv.y, f1);
                f2 = fmaf(kv, wv.z, f2);
            }
            a0 += (double)f0;
            a1 += (double)f1;
            a2 += (double)f2;
        }
        if (live) vec_add(y, S, n_f, u.x, inst, a0, a1, a2);
    }
}

void launch_scatter(cudaStream_t st, const Params& P, int max_rows, InstOff off, const int* ucount,
                    const int4* ulist, const float* Zc, const double* wz, const float4* wzT, float4* y, int nitems,
                    const int2* items) {
    if (P.NS == 0 || nitems == 0) return;
    int gx = (max_rows + 7) / 8;
    if (nitems > 1) gx = std::min(gx, std::max(1, (148 * 8 + nitems - 1) / nitems));
    launch_pdl(k_scatter, dim3(gx, nitems), dim3(256), 0, st, P.S, P.n_f, off, ucount, ulist, Zc, wz, wzT, y, items);
}

// ----------------------------------------------------------------------------
// Delassus Gram G = K[:,Vc]^T K[:,Vc] (P:L858 via the sparse inverse):
// G_st = sum over common ancestors i of K[i][a_s] K[i][a_t] = sum over depths
// d <= depth(lca(a_s, a_t)) of Z[d][s] Z[d][t], Z[d][s] = Kcol[colptr_s + depth_s - d].
// 32x32 tiles of slot pairs, depth staged in chunks of 32 levels.
// ----------------------------------------------------------------------------

// four LCA walks advanced together (their dependent ptop / parent loads overlap instead of running
// one after the other); each walk is lca_depth's
__device__ void lca_depth4(const int (&a_)[4], const int (&b_)[4], const bool (&on)[4], int (&out)[4],
                           const int32_t* parent, const int32_t* ptop, const int32_t* depth) {
    int i[4], b[4];
    bool live[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int lo = min(a_[q], b_[q]), hi = max(a_[q], b_[q]);
        i[q] = lo;
        b[q] = hi;
        live[q] = on[q];
        out[q] = -1;
    }
    while (live[0] || live[1] || live[2] || live[3]) {
        int top[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) top[q] = live[q] ? __ldg(&ptop[i[q]]) : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!live[q]) continue;
            if (top[q] >= b[q]) {
                out[q] = __ldg(&depth[i[q] > b[q] ? i[q] : b[q]]);
                live[q] = false;
            } else {
                i[q] = __ldg(&parent[top[q]]);
                if (i[q] < 0) live[q] = false;
            }
        }
    }
}

__device__ int lca_depth(int a, int b, const int32_t* parent, const int32_t* ptop, const int32_t* depth) {
    // a <= b in postorder: lca = first ancestor run of a whose top >= b, at row max(i, b)
    if (a > b) { int t = a; a = b; b = t; }
    for (int i = a; i >= 0;) {
        int top = ptop[i];
        if (top >= b) return depth[i > b ? i : b];
        i = parent[top];
    }
    return -1;
}

__global__ void __launch_bounds__(256) k_delassus(InstOff off, const int32_t* __restrict__ vtx_all,
                                                  const float* __restrict__ Kcol, const int64_t* __restrict__ colptr,
                                                  const int32_t* __restrict__ depth, const int32_t* __restrict__ parent,
                                                  const int32_t* __restrict__ ptop, float* __restrict__ Gall) {
    // class blockIdx.y; tile (bs, bt) with bt >= bs from a linear triangular index
    const int cl = blockIdx.y;
    const int sb = off.csoff[cl], ns = off.csoff[cl + 1] - sb;
    const int32_t* slot_vtx = vtx_all + sb;
    float* G = Gall + off.goff[cl];
    const int tiles = (ns + 31) / 32;
    if ((int)blockIdx.x >= tiles * (tiles + 1) / 2) return;
    int idx = blockIdx.x, bs = 0;
    while (idx >= tiles - bs) { idx -= tiles - bs; ++bs; }
    const int bt = bs + idx;
    constexpr int NST = 3;   // chunks of 32 depth levels in flight (cp.async straight into shared memory)
    __shared__ float Zs[NST][32][33], Zt[NST][32][33];
    __shared__ double Ds[32][33], Dt[32][33];   // the chunk being consumed, converted to fp64 once
    __shared__ int ds_[32], dt_[32];
    __shared__ int64_t cs_[32], ct_[32];
    __shared__ int smax;
    const int tid = threadIdx.x;
    if (tid < 32) {
        const int s = bs * 32 + tid;
        if (s < ns) { const int a = slot_vtx[s]; ds_[tid] = depth[a]; cs_[tid] = colptr[a]; }
        else { ds_[tid] = -1; cs_[tid] = 0; }
    } else if (tid < 64) {
        const int t = bt * 32 + tid - 32;
        if (t < ns) { const int a = slot_vtx[t]; dt_[tid - 32] = depth[a]; ct_[tid - 32] = colptr[a]; }
        else { dt_[tid - 32] = -1; ct_[tid - 32] = 0; }
    }
    if (tid == 0) smax = -1;
    __syncthreads();
    // thread owns pairs (ls, lt0 + 8 q), q = 0..3 (the fp64 reads of Dt hit distinct banks)
    const int ls = tid >> 3, lt0 = tid & 7;
    const int s = bs * 32 + ls;
    int dl[4];
    int maxd = -1;
    {
        int av[4], bv[4];
        bool on[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = bt * 32 + lt0 + 8 * q;
            on[q] = s < ns && t < ns;
            av[q] = on[q] ? slot_vtx[s] : 0;
            bv[q] = on[q] ? slot_vtx[t] : 0;
        }
        lca_depth4(av, bv, on, dl, parent, ptop, depth);
#pragma unroll
        for (int q = 0; q < 4; ++q) maxd = max(maxd, dl[q]);
    }
    atomicMax(&smax, maxd);
    __syncthreads();
    const int D = smax;
    // staging: each thread copies 4 (slot, depth) entries of each block per 32-level chunk, NST - 1
    // chunks ahead (latency-bound otherwise: ~2 CTAs per SM for an 800-slot Gram)
    const int nch = D >= 0 ? D / 32 + 1 : 0;
    auto issue = [&](int c) {
        if (c < nch) {
            const int d0 = 32 * c, st = c % NST;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = tid + 256 * u;
                const int sl = e >> 5, dd = e & 31, d = d0 + dd;
                const bool vs = ds_[sl] >= d, vt = dt_[sl] >= d;
                cp_async4(&Zs[st][dd][sl], vs ? &Kcol[cs_[sl] + ds_[sl] - d] : Kcol, vs);
                cp_async4(&Zt[st][dd][sl], vt ? &Kcol[ct_[sl] + dt_[sl] - d] : Kcol, vt);
            }
        }
        cp_async_commit();   // possibly empty: keeps one group per chunk slot
    };
    // fp64 accumulation: G_ab sums up to etree-height products; an fp32 running sum loses ~1e-5
    // relative on cancelling pairs, and fp32 sums of 32-term chunks folded into fp64 still flip an
    // A21 classification on the soft-soft pile -- D = J G J^T drives the CR
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < NST - 1; ++c) issue(c);
    for (int c = 0; c < nch; ++c) {
        cp_async_wait<NST - 2>();   // chunk c landed (this thread's copies)
        __syncthreads();            // ... everyone's; and chunk c - 1 is consumed everywhere
        issue(c + NST - 1);         // into the stage chunk c - 1 used
        const int st = c % NST, d0 = 32 * c;
        // fp32 -> fp64 once per staged element (the products are exact in fp64 either way; converting
        // in the FMA loop cost 5 conversions per 4 DFMA and bound the kernel)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + 256 * u;
            const int dd = e >> 5, sl = e & 31;
            Ds[dd][sl] = (double)Zs[st][dd][sl];
            Dt[dd][sl] = (double)Zt[st][dd][sl];
        }
        __syncthreads();
#pragma unroll 8
        for (int dd = 0; dd < 32; ++dd) {
            const int d = d0 + dd;
            const double zs = Ds[dd][ls];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (d <= dl[q]) acc[q] = fma(zs, Dt[dd][lt0 + 8 * q], acc[q]);
        }
    }
    for (int q = 0; q < 4; ++q) {
        const int t = bt * 32 + lt0 + 8 * q;
        if (s < ns && t < ns) {
            G[(size_t)s * ns + t] = (float)acc[q];
            G[(size_t)t * ns + s] = (float)acc[q];
        }
    }
}

void launch_delassus(cudaStream_t st, const Params& P, InstOff off, ClassSlots csl, const float* Kcol,
                     const int64_t* colptr, const int32_t* depth, const int32_t* parent, const int32_t* ptop,
                     float* G) {
    if (P.CS == 0) return;
    const int tiles = (P.ns_max + 31) / 32;
    const int ntri = tiles * (tiles + 1) / 2;
    k_delassus<<<dim3(ntri, P.NCL), 256, 0, st>>>(off, csl.vtx, Kcol, colptr, depth, parent, ptop, G);
}

// ----------------------------------------------------------------------------
// Gram reuse across commits ("reuse strategy ... to exploit shared contact data between
// consecutive time steps"): G[a][b] depends only on the vertex pair, so the
// entries of vertex pairs present in the previous contact set are copied and only the rows of
// new contact vertices are computed -- with the same fp32 accumulation order as k_delassus,
// so the result is bitwise the full recomputation.
//   rmap[class slot] = slot of the same vertex in the previous block of the class, or -1
// ----------------------------------------------------------------------------
__global__ void k_gram_copy(InstOff off, const int* __restrict__ rmap, const int64_t* __restrict__ pgoff,
                            const int* __restrict__ pns, const float* __restrict__ Gprev, float* __restrict__ G) {
    const int cl = blockIdx.y;
    const int sb = off.csoff[cl], ns = off.csoff[cl + 1] - sb;
    const int nso = pns[cl];
    float* Gc = G + off.goff[cl];
    const float* Go = Gprev + pgoff[cl];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ns * ns; e += gridDim.x * blockDim.x) {
        const int sa = e / ns, tb = e - sa * ns;
        const int ma = rmap[sb + sa], mb = rmap[sb + tb];
        if (ma >= 0 && mb >= 0) Gc[e] = Go[(size_t)ma * nso + mb];
    }
}

// rows (and columns) of the new slots: one warp per (new slot, 32 partner slots), lane = partner
__global__ void k_gram_rows(InstOff off, const int32_t* __restrict__ vtx_all, const int* __restrict__ rmap,
                            const int2* __restrict__ newslots, int nnew, const float* __restrict__ Kcol,
                            const int64_t* __restrict__ colptr, const int32_t* __restrict__ depth,
                            const int32_t* __restrict__ parent, const int32_t* __restrict__ ptop, float* __restrict__ G) {
    const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int ni = wg / 32, chunk = wg % 32;   // up to 32 chunks of 32 partners per new slot
    if (ni >= nnew) return;
    const int2 ns_ = newslots[ni];             // {class, class-local slot}
    const int cl = ns_.x, s = ns_.y;
    const int sb = off.csoff[cl], ns = off.csoff[cl + 1] - sb;
    float* Gc = G + off.goff[cl];
    const int a = vtx_all[sb + s];
    const float* ca = Kcol + colptr[a] + depth[a];   // K at depth d: ca[-d]
    for (int t = 32 * chunk + lane; t < ns; t += 32 * 32) {
        // pairs with an older partner of lower index are owned by this row; two new slots: the
        // lower one writes (keeps one writer per entry)
        if (rmap[sb + t] < 0 && t < s) continue;
        const int b = vtx_all[sb + t];
        const int dl = lca_depth(a, b, parent, ptop, depth);
        const float* cb = Kcol + colptr[b] + depth[b];
        double acc = 0.0;   // the same order and precision as k_delassus (bitwise equal entries)
        for (int d = 0; d <= dl; ++d) acc = fma((double)__ldg(ca - d), (double)__ldg(cb - d), acc);
        Gc[(size_t)s * ns + t] = (float)acc;
        Gc[(size_t)t * ns + s] = (float)acc;
    }
}

void launch_gram_reuse(cudaStream_t st, const Params& P, InstOff off, const int32_t* vtx_all, const int* rmap,
                       const int64_t* pgoff, const int* pns, const float* Gprev, const int2* newslots, int nnew,
                       const float* Kcol, const int64_t* colptr, const int32_t* depth, const int32_t* parent,
                       const int32_t* ptop, float* G) {
    if (P.CS == 0) return;
    const int gx = std::max(1, std::min(64, (P.ns_max * P.ns_max + 255) / 256));
    k_gram_copy<<<dim3(gx, P.NCL), 256, 0, st>>>(off, rmap, pgoff, pns, Gprev, G);
    if (nnew > 0) {
        const int warps = nnew * 32;
        k_gram_rows<<<(warps + 7) / 8, 256, 0, st>>>(off, vtx_all, rmap, newslots, nnew, Kcol, colptr, depth, parent,
                                                     ptop, G);
    }
}

// ----------------------------------------------------------------------------
// K = L^-1 on the device: column j of K is the solution of L k = e_j,
// nonzero on the ancestor chain of j only (Theorem 1; Fig. 4 "ancestor"
// traversal).  One warp per column walks the chain: k_l = w_l / L_ll, then the
// lanes scatter w_i -= L_il k_l over column l of L (all rows i are ancestors of l, so on the
// chain, at position depth(j) - depth(i)).  The per-element update order is the host's
// (simhost::sparse_inverse_values) and products are not contracted into FMAs, so the fp64
// values and their fp32 storage are bitwise the host's.
// ----------------------------------------------------------------------------
constexpr int kInvWarps = 8;

__global__ void __launch_bounds__(32 * kInvWarps) k_inverse_cols(int n, int hmax, const int64_t* __restrict__ Lp,
                                                                 const int32_t* __restrict__ Li,
                                                                 const double* __restrict__ Lx,
                                                                 const int32_t* __restrict__ parent,
                                                                 const int32_t* __restrict__ depth,
                                                                 const int32_t* __restrict__ first,
                                                                 const int64_t* __restrict__ colptr,
                                                                 const int64_t* __restrict__ rowptr, double drop_tol,
                                                                 float* __restrict__ Kcol, float* __restrict__ Krow) {
    extern __shared__ double wsh[];
    const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* w = wsh + (size_t)wl * hmax;
    for (int j = blockIdx.x * kInvWarps + wl; j < n; j += gridDim.x * kInvWarps) {
        const int D = depth[j];
        for (int q = lane; q <= D; q += 32) w[q] = q == 0 ? 1.0 : 0.0;
        __syncwarp();
        double kjj = 0.0;
        int q = 0;
        for (int l = j; l != -1; l = parent[l], ++q) {
            const double kl = __ddiv_rn(w[q], Lx[Lp[l]]);
            if (q == 0) kjj = kl;
            for (int64_t p = Lp[l] + 1 + lane; p < Lp[l + 1]; p += 32) {
                const int i = Li[p];
                const int pos = D - depth[i];
                w[pos] = __dsub_rn(w[pos], __dmul_rn(Lx[p], kl));
            }
            if (lane == 0) {
                double kv = kl;
                if (drop_tol > 0 && fabs(kv) < drop_tol * fabs(kjj)) kv = 0.0;
                const float kf = (float)kv;
                Kcol[colptr[j] + q] = kf;
                Krow[rowptr[l] + (j - first[l])] = kf;
            }
            __syncwarp();
        }
    }
}

int launch_inverse_columns(cudaStream_t st, int n, int hmax, const int64_t* Lp, const int32_t* Li, const double* Lx,
                           const int32_t* parent, const int32_t* depth, const int32_t* first, const int64_t* colptr,
                           const int64_t* rowptr, double drop_tol, float* Kcol, float* Krow) {
    const size_t smem = (size_t)kInvWarps * hmax * sizeof(double);
    if (smem > 227 * 1024) return (int)cudaErrorInvalidValue;   // etree too tall for the per-warp chain buffer
    cudaError_t e = cudaFuncSetAttribute(k_inverse_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = std::min((n + kInvWarps - 1) / kInvWarps, nsm * 8);
    k_inverse_cols<<<blocks, 32 * kInvWarps, smem, st>>>(n, hmax, Lp, Li, Lx, parent, depth, first, colptr, rowptr,
                                                          drop_tol, Kcol, Krow);
    return (int)cudaGetLastError();
}

// D_jj = sum_{a,b in j} w_a w_b G_ab (unit directions; reading A18)
__global__ void k_djj(int C, InstOff off, DContact* Cs, const float* __restrict__ G) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    DContact& ct = Cs[c];
    const int sb = off.soff[ct.inst], ns = off.soff[ct.inst + 1] - sb;
    const float* Gi = G + off.goff[off.cls[ct.inst]];
    double d = 0.0;
    for (int p = 0; p < ct.nv; ++p)
        for (int q = 0; q < ct.nv; ++q)
            d += ct.w[p] * ct.w[q] * (double)Gi[(size_t)(ct.slot[p] - sb) * ns + (ct.slot[q] - sb)];
    ct.Djj = d;
}

void launch_djj(cudaStream_t st, const Params& P, InstOff off, DContact* c, const float* G) {
    if (P.C == 0) return;
    k_djj<<<(P.C + 127) / 128, 128, 0, st>>>(P.C, off, c, G);
}

// ----------------------------------------------------------------------------
// CR (Saad Alg. 6.20) on S = Theta D Theta + C, z0 = 0, exactly N_CR matvecs
// (reading A19), in ONE cluster of kCluster CTAs.
//
// * Theta-sparsity: rows with theta = 0 contribute nothing to Theta D Theta, so the D
//   product runs over the active contact vertices only (k_active / k_gather_ga build the
//   active block G_A of G in a graph branch; exact, not an approximation).
// * Every CTA runs the O(m) recurrences redundantly (dot products come out identical
//   everywhere without communication).  Thread t owns rows t + 512 k: z, p, Ap, Ar are
//   registers, r (read by the W gather) is in shared memory.  q = G_A W is split by rows
//   of G_A and exchanged with st.async + mbarrier transaction counts (no cluster barrier).
// * One block reduction per iteration: after Ar = S r the three dots r.Ar, Ar.Ar, Ar.Ap
//   give beta and |Ap_new|^2 = Ar.Ar + 2 beta Ar.Ap + beta^2 |Ap|^2 (algebraically the
//   oracle's direct form).
// * fp64 in the D product: G = A_v^-1 is a smoothing kernel, so G W cancels heavily for
//   the oscillatory Krylov vectors (fp32 W or fp32 sums cost ~3e-3).
// ----------------------------------------------------------------------------
constexpr int kRptMax = 6;   // rows per thread: m = 3 nc <= kRpt * kCrThreads (kernel templated on kRpt)

// shared-memory layout of one CR CTA; W and q are sized by the active count na, the
// contact directions c9 are staged only when they fit next to this CTA's rows of G_A
struct CrLayout {
    int m, nc, ns;
    size_t r, th, cd, s0, aidx, apos, acon, red, mbar, W, q, qp, c9, gA, total;
    // parts > 1: the solo matvec splits the columns of G_A over `parts` thread groups (partial sums in qp)
    __host__ __device__ CrLayout(int nc_, int ns_, int na, bool with_c9, int parts = 1)
        : m(3 * nc_), nc(nc_), ns(ns_) {
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~size_t(15); return at; };
        r = take(8 * (size_t)m);
        th = take(4 * (size_t)m); cd = take(4 * (size_t)m);
        s0 = take(4 * (size_t)nc);
        aidx = take(4 * (size_t)ns); apos = take(4 * (size_t)ns); acon = take(4 * (size_t)ns);
        red = take(8 * 2 * 3 * (kCrThreads / 32));   // double-buffered 3 doubles per warp
        mbar = take(32);                              // two exchange mbarriers (one per q buffer)
        W = take(8 * 3 * (size_t)na); q = take(8 * 2 * 3 * (size_t)na);
        qp = parts > 1 ? take(8 * 3 * (size_t)na * parts) : 0;
        c9 = with_c9 ? take(4 * 9 * (size_t)nc) : 0;
        gA = o;
        total = o;
    }
};

// CR shape of one instance: the G_A row stride in shared memory and the column groups of the
// one-CTA-per-instance matvec
__host__ __device__ inline int cr_lda(int na, int csize) { return csize == 1 ? (na | 1) : na; }
__host__ __device__ inline int cr_parts_max(int na, int csize) {
    return csize == 1 ? max(1, min(4, kCrThreads / max(32, (na + 31) & ~31))) : 1;
}
// column groups of the one-CTA matvec: as many as keep the threads busy, unless their partial-sum
// buffer (qp) is what keeps G_A out of shared memory -- G_A resident beats the extra parallelism
__host__ __device__ inline int cr_parts(int nc, int ns, int na, int csize) {
    const int P = cr_parts_max(na, csize);
    if (P == 1) return 1;
    const size_t ga = (size_t)na * cr_lda(na, csize) * sizeof(float);
    const size_t t1 = CrLayout(nc, ns, na, false, 1).total;   // + the partial sums of P groups:
    const size_t qp = ((size_t)8 * 3 * na * P + 15) & ~(size_t)15;
    return (t1 + qp + ga > kCrMaxSmem && t1 + ga <= kCrMaxSmem) ? 1 : P;
}
// a lone CTA holds the whole instance and its G_A fits next to the minimal layout: it gathers
// G_A from the class Gram itself (k_active skips the global copy)
__host__ __device__ bool cr_ga_direct(int nc, int ns, int na, int csize) {
    if (csize != 1) return false;
    return CrLayout(nc, ns, na, false, cr_parts(nc, ns, na, csize)).total + (size_t)na * cr_lda(na, csize) * sizeof(float) <=
           kCrMaxSmem;
}

// The active slots of one instance in slot order (the list k_active builds), computed by one CTA
// into its shared memory: apos[b] = position or -1, aidx[pos] = b, acon[pos] = local id of the
// slot's single single-vertex contact or -1.  Returns na (every thread).
// scratch: >= 33 ints of shared memory (the CTA's reduction buffer; no static shared memory:
// k_cr takes the whole 227 KB dynamically)
__device__ int cr_active_block(int ns, int sb, int cb, const CrContacts& cc, const Slots& sl,
                               const ContactState& cs, int* aidx, int* apos, int* acon, int* scratch) {
    int* wsum = scratch;
    int& sbase = scratch[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) sbase = 0;
    __syncthreads();
    for (int b0 = 0; b0 < ns; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        bool on = false;
        int only = -1;
        if (b < ns) {
            only = cc.c1[sb + b];
            if (only >= 0) {
                on = cs.theta[3 * only] != 0.0 || cs.theta[3 * only + 1] != 0.0 || cs.theta[3 * only + 2] != 0.0;
            } else {
                for (int q = sl.scp[sb + b]; q < sl.scp[sb + b + 1] && !on; ++q) {
                    const int c = sl.sci[q];
                    on = cs.theta[3 * c] != 0.0 || cs.theta[3 * c + 1] != 0.0 || cs.theta[3 * c + 2] != 0.0;
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int pos = sbase;
        for (int q = 0; q < wid; ++q) pos += wsum[q];
        pos += __popc(bal & ((1u << lane) - 1u));
        if (b < ns) {
            apos[b] = on ? pos : -1;
            if (on) {
                aidx[pos] = b;
                acon[pos] = only >= 0 ? only - cb : -1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = sbase;
            for (int q = 0; q < nw; ++q) t += wsum[q];
            sbase = t;
        }
        __syncthreads();
    }
    return sbase;
}

__device__ unsigned long long g_cr_clock[32];   // phase timestamps (ns) of the last CR call, instance 0 rank 0
__device__ __forceinline__ void cr_stamp(int i) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_cr_clock[i] = t;
    }
}

// one instance's view (local contact ids 0..nc-1, local slot ids 0..ns-1)
struct CrInst {
    const DContact* C;       // + cb   (slot[] global: subtract sb; vtx: state index vtx * S + inst)
    const int32_t* scp;      // + sb   (values: global positions into sci)
    const int32_t* sci;      // global (values: global contact ids: subtract cb)
    const float* scw;
    int cb, sb, S, inst;
};

struct CrCtx {
    double *r, *W, *q, *qp, *red;
    float *gA, *th, *cd, *c9;
    int *s0, *aidx, *apos, *acon;
    int na, ns, i0, i1, gA_smem, csize;
    int lda, parts;        // solo path: G_A row stride in shared memory (odd), column groups
    unsigned mbar;         // shared-window address of the 2 exchange mbarriers
    unsigned par0, par1;   // phase parity of each barrier
    int stamp;             // >= 0: fine-grained phase stamps of this apply at g_cr_clock[stamp..]
    const float* GAg;      // G_A in global memory (fallback when this CTA's rows do not fit)
};

// single-barrier block sum of 3 doubles (red is double-buffered by the caller)
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* red) {
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { red[3 * w] = a; red[3 * w + 1] = b; red[3 * w + 2] = c; }
    __syncthreads();
    a = b = c = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { a += red[3 * q]; b += red[3 * q + 1]; c += red[3 * q + 2]; }
}

// Per-thread row metadata of the contact-row map C^T (fixed for one CR solve: Theta and the active
// slots do not change inside it), hoisted out of the CR iterations into registers: ip = the active
// position of the row's single contact vertex (-2: theta = 0, -1: multi-vertex contact, mapped
// through its vertex list).
template <int kRpt>
struct CrRows {
    int ip[kRpt];
};

template <int kRpt>
__device__ __forceinline__ void cr_rows_init(const CrCtx& X, int m, CrRows<kRpt>& R) {
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        const int j = min(threadIdx.x + kCrThreads * k, m - 1);
        const int c = j / 3;
        R.ip[k] = -2;
        if (X.th[j] != 0.f) {
            const int sl0 = X.s0[c];
            R.ip[k] = sl0 >= 0 ? X.apos[sl0] : -1;
        }
    }
}

// Ar = S r for this thread's rows (registers); r is read from shared memory
template <int kRpt, int kSolo>
__device__ __forceinline__ void cr_apply(CrCtx& X, int m, const CrInst& I, int buf, double (&Ar)[kRpt],
                                         const CrRows<kRpt>& R) {
    const int na = X.na;
    double* qb = X.q + (size_t)buf * 3 * X.na;   // SoA: q0 | q1 | q2
    const unsigned bar = X.mbar + 8u * (unsigned)buf;
    constexpr bool solo = kSolo != 0;   // (X.csize == 1) one CTA per instance: q stays local, no cluster exchange
    //   // one CTA per instance: q stays local, no cluster exchange
    if (!solo && threadIdx.x == 0 && na > 0)   // this phase expects 24 bytes per row of G_A from the peers
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(24 * na) : "memory");
    for (int i = threadIdx.x; i < na; i += blockDim.x) {
        double w0 = 0.0, w1 = 0.0, w2 = 0.0;
        const int c1 = X.acon[i];
        if (c1 >= 0) {   // the single single-vertex contact on this slot (weight 1)
            const float* cc = X.c9 + 9 * c1;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double tv = (double)X.th[3 * c1 + k] * X.r[3 * c1 + k];
                w0 = fma(tv, (double)cc[3 * k], w0);
                w1 = fma(tv, (double)cc[3 * k + 1], w1);
                w2 = fma(tv, (double)cc[3 * k + 2], w2);
            }
        } else {
            const int b = X.aidx[i];
            for (int p = __ldg(&I.scp[b]); p < __ldg(&I.scp[b + 1]); ++p) {
                const int c = __ldg(&I.sci[p]) - I.cb;
                const double wt = __ldg(&I.scw[p]);
                const float* cc = X.c9 + 9 * c;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double tv = wt * (double)X.th[3 * c + k] * X.r[3 * c + k];
                    w0 = fma(tv, (double)cc[3 * k], w0);
                    w1 = fma(tv, (double)cc[3 * k + 1], w1);
                    w2 = fma(tv, (double)cc[3 * k + 2], w2);
                }
            }
        }
        X.W[i] = w0;
        X.W[na + i] = w1;
        X.W[2 * na + i] = w2;
    }
    __syncthreads();
    if (X.stamp >= 0) cr_stamp(X.stamp);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (solo) {
        // one row of G_A per thread, the columns split over `parts` groups of threads whose partial sums
        // are added in part order (deterministic); no warp reductions.  G_A in shared memory: row i at
        // stride lda (odd: the 32 rows a warp reads sit in 32 banks; W is a broadcast).  G_A in global
        // memory (too large for shared memory): G_A is symmetric (G_A[b][i] = G_A[i][b], both written
        // from one sum), so thread i reads column i -- a warp's 32 rows are 128 contiguous bytes of row
        // b, coalesced -- and the result is bitwise that of the shared-memory path
        const int nap = (na + 31) & ~31, P = X.parts, cs = (na + P - 1) / P;
        if (X.gA_smem) {
            for (int t = threadIdx.x; t < nap * P; t += blockDim.x) {
                const int part = t / nap, i = t - part * nap;
                if (i >= na) continue;
                const float* g = X.gA + (size_t)i * X.lda;
                const int b1 = min(na, (part + 1) * cs);
                int b = part * cs;
                double d0 = 0.0, d1 = 0.0, d2 = 0.0;
                for (; b + 4 <= b1; b += 4) {
                    float gv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) gv[u] = g[b + u];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double gd = (double)gv[u];
                        d0 = fma(gd, X.W[b + u], d0);
                        d1 = fma(gd, X.W[na + b + u], d1);
                        d2 = fma(gd, X.W[2 * na + b + u], d2);
                    }
                }
                for (; b < b1; ++b) {
                    const double gd = (double)g[b];
                    d0 = fma(gd, X.W[b], d0);
                    d1 = fma(gd, X.W[na + b], d1);
                    d2 = fma(gd, X.W[2 * na + b], d2);
                }
                double* o = P > 1 ? X.qp + (size_t)part * 3 * na : qb;
                o[i] = d0;
                o[na + i] = d1;
                o[2 * na + i] = d2;
            }
        } else {
            for (int t = threadIdx.x; t < nap * P; t += blockDim.x) {
                const int part = t / nap, i = t - part * nap;
                if (i >= na) continue;
                const float* g = X.GAg + i;   // column i
                const int b1 = min(na, (part + 1) * cs);
                double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll 4
                for (int b = part * cs; b < b1; ++b) {
                    const double gd = (double)__ldcg(g + (size_t)b * na);
                    d0 = fma(gd, X.W[b], d0);
                    d1 = fma(gd, X.W[na + b], d1);
                    d2 = fma(gd, X.W[2 * na + b], d2);
                }
                double* o = P > 1 ? X.qp + (size_t)part * 3 * na : qb;
                o[i] = d0;
                o[na + i] = d1;
                o[2 * na + i] = d2;
            }
        }
        if (P > 1) {
            __syncthreads();
            for (int e = threadIdx.x; e < 3 * na; e += blockDim.x) {
                double acc = X.qp[e];
                for (int q = 1; q < P; ++q) acc += X.qp[(size_t)q * 3 * na + e];
                qb[e] = acc;
            }
        }
    }
    for (int i = X.i0 + wid; !solo && i < X.i1; i += nw) {
        const float* g = X.gA_smem ? X.gA + (size_t)(i - X.i0) * na : X.GAg + (size_t)i * na;
        double d0 = 0, d1 = 0, d2 = 0;
        for (int b0 = 0; b0 < na; b0 += 128) {
            double gv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int bb = b0 + 32 * u + lane;
                gv[u] = bb < na ? (double)(X.gA_smem ? g[bb] : __ldcg(&g[bb])) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int bb = min(b0 + 32 * u + lane, na - 1);
                d0 = fma(gv[u], X.W[bb], d0);
                d1 = fma(gv[u], X.W[na + bb], d1);
                d2 = fma(gv[u], X.W[2 * na + bb], d2);
            }
        }
        d0 = warp_sum(d0);
        d1 = warp_sum(d1);
        d2 = warp_sum(d2);
        if (lane < X.csize) {
            // asynchronous stores of q_i into CTA `lane` of the cluster, completing 24 tx bytes on its mbarrier
            const unsigned l0 = (unsigned)__cvta_generic_to_shared(qb + i);
            const unsigned l1 = (unsigned)__cvta_generic_to_shared(qb + na + i);
            const unsigned l2 = (unsigned)__cvta_generic_to_shared(qb + 2 * na + i);
            unsigned r0, r1, r2, rb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r0) : "r"(l0), "r"(lane));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r1) : "r"(l1), "r"(lane));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r2) : "r"(l2), "r"(lane));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(bar), "r"(lane));
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(r0),
                         "d"(d0), "r"(rb)
                         : "memory");
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(r1),
                         "d"(d1), "r"(rb)
                         : "memory");
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(r2),
                         "d"(d2), "r"(rb)
                         : "memory");
        }
    }
    if (X.stamp >= 0) cr_stamp(X.stamp + 1);
    if (!solo && threadIdx.x == 0 && na > 0) {   // wait until all na rows have landed here (acquire)
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                " selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(bar), "r"(buf ? X.par1 : X.par0)
                : "memory");
        }
    }
    if (!solo) {
        if (buf) X.par1 ^= 1u; else X.par0 ^= 1u;
    }
    __syncthreads();
    if (X.stamp >= 0) cr_stamp(X.stamp + 2);
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        const int j = min(threadIdx.x + kCrThreads * k, m - 1);   // rows >= m are padding (never used)
        const double th = (double)X.th[j];
        double acc = 0.0;
        const int ip = R.ip[k];
        const int c = j / 3, kk = j - 3 * c;
        const float* cc = X.c9 + 9 * c + 3 * kk;
        if (ip >= 0) {
            acc = (double)cc[0] * qb[ip] + (double)cc[1] * qb[na + ip] + (double)cc[2] * qb[2 * na + ip];
        } else if (ip == -1) {
            const DContact& ct = I.C[c];
            for (int p = 0; p < ct.nv; ++p) {
                const int iq = X.apos[ct.slot[p] - I.sb];
                acc += ct.w[p] * ((double)cc[0] * qb[iq] + (double)cc[1] * qb[na + iq] +
                                  (double)cc[2] * qb[2 * na + iq]);
            }
        }
        Ar[k] = th * acc + (double)X.cd[j] * X.r[j];
    }
}

// One cluster of csize CTAs per instance (csize = 16 for a single scene, fewer when many
// instances fill the GPU).  Launched with a runtime cluster dimension (cudaLaunchKernelEx).
// kSolo: compiled separately for one CTA per instance (csize == 1) and for clusters, so that neither
// path's registers weigh on the other's allocation
template <int kRpt, int kSolo>
__global__ void __launch_bounds__(kCrThreads, 1)
    k_cr(Params P, InstOff off, const DContact* __restrict__ C, CrContacts cc, Slots sl, const float* __restrict__ G,
         float* GA, const double4* __restrict__ x, ContactState cs, CrActive act) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smraw[];
    cg::cluster_group cl = cg::this_cluster();
    const int csize = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const int inst = blockIdx.x / csize;
    const int cb = off.coff[inst], nc = off.coff[inst + 1] - cb;
    const int sb = off.soff[inst], ns = off.soff[inst + 1] - sb;
    if (nc == 0) {   // uniform over the cluster
        if (threadIdx.x == 0 && rank == 0) cs.cr_res[inst] = 0.0;
        return;
    }
    const int m = 3 * nc;
    const double h = P.h;
    const int S = P.S;
    cr_stamp(0);
    // cluster CR (few instances): every CTA builds the active list itself (no k_active /
    // k_gather_ga launches on the single-scene critical path); one CTA per instance: k_active's list
    int na;
    if (csize > 1) {
        const CrLayout L0(nc, ns, 0, false);   // the active-list offsets do not depend on na
        na = cr_active_block(ns, sb, cb, cc, sl, cs, (int*)(smraw + L0.aidx), (int*)(smraw + L0.apos),
                             (int*)(smraw + L0.acon), (int*)(smraw + L0.red));
    } else {
        na = act.na[inst];
    }
    cr_stamp(22);   // active list built
    const int per = (na + csize - 1) / csize;
    const int i0 = min(na, rank * per), i1 = min(na, i0 + per);
    constexpr bool solo = kSolo != 0;   // == (csize == 1), chosen by the launcher
    const int lda = cr_lda(na, csize);
    const int parts = cr_parts(nc, ns, na, csize);
    const size_t needA = (size_t)(i1 - i0) * lda * sizeof(float);
    // prefer G_A rows in shared memory; stage c9 too when both fit
    const bool c9s = CrLayout(nc, ns, na, true, parts).total + needA <= kCrMaxSmem ||
                     CrLayout(nc, ns, na, false, parts).total + needA > kCrMaxSmem;
    const CrLayout L(nc, ns, na, c9s, parts);
    CrInst I{C + cb, sl.scp + sb, sl.sci, sl.scw, cb, sb, S, inst};
    double* th_g = cs.theta + 3 * cb;
    double* cd_g = cs.cdiag + 3 * cb;
    double* rho_g = cs.rho + 3 * cb;
    double* hv_g = cs.hvec + 3 * cb;
    double* lam_g = cs.lam + 3 * cb;
    const double* dxt_g = cs.dxt + 3 * sb;
    double* wz_g = cs.wz + 3 * sb;
    CrCtx X;
    X.r = (double*)(smraw + L.r);
    X.th = (float*)(smraw + L.th);
    X.cd = (float*)(smraw + L.cd);
    X.c9 = c9s ? (float*)(smraw + L.c9) : const_cast<float*>(cc.c9 + 9 * (size_t)cb);
    X.s0 = (int*)(smraw + L.s0);
    X.W = (double*)(smraw + L.W);
    X.q = (double*)(smraw + L.q);
    X.qp = (double*)(smraw + L.qp);
    X.lda = lda;
    X.parts = parts;
    X.aidx = (int*)(smraw + L.aidx);
    X.apos = (int*)(smraw + L.apos);
    X.acon = (int*)(smraw + L.acon);
    X.red = (double*)(smraw + L.red);
    X.gA = (float*)(smraw + L.gA);
    X.mbar = (unsigned)__cvta_generic_to_shared(smraw + L.mbar);
    X.par0 = X.par1 = 0u;
    X.stamp = -1;
    X.ns = ns;
    X.csize = csize;
    X.GAg = GA + off.gaoff[inst];
    // everything the prologue needs is precomputed (chain dot, k_active): plain loads only
    if (c9s)
        for (int e = threadIdx.x; e < 9 * nc; e += blockDim.x) cp_async4(&X.c9[e], &cc.c9[9 * cb + e], true);
    for (int b = threadIdx.x; b < ns && solo; b += blockDim.x) {
        cp_async4(&X.apos[b], &act.apos[sb + b], true);
        if (b < na) {   // k_active writes aidx/acon for the na active slots only
            cp_async4(&X.aidx[b], &act.aidx[sb + b], true);
            cp_async4(&X.acon[b], &act.acon[sb + b], true);
        }
    }
    cp_async_commit();
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
        const int s0g = cc.s0[cb + c];
        X.s0[c] = s0g >= 0 ? s0g - sb : -1;
    }
    X.na = na;
    X.i0 = i0;
    X.i1 = i1;
    X.gA_smem = L.total + needA <= kCrMaxSmem;
    if (X.gA_smem) {   // asynchronous 4-byte copies, all in flight (waited for with the rest below)
        if (solo) {       // G_A[i][j] = G[aidx_i][aidx_j] straight from the class Gram (cr_ga_direct)
            cp_async_wait<0>();
            __syncthreads();   // aidx staged
            const float* Gc = G + off.goff[off.cls[inst]];
            for (int rw = threadIdx.x >> 5; rw < na; rw += blockDim.x >> 5) {
                const float* Gi = Gc + (size_t)X.aidx[rw] * ns;
                for (int c = threadIdx.x & 31; c < na; c += 32)
                    cp_async4(&X.gA[(size_t)rw * lda + c], &Gi[X.aidx[c]], true);
            }
        } else {          // this CTA's rows of G_A from the class Gram (active list built above)
            const float* Gc = G + off.goff[off.cls[inst]];
            const int rows = X.i1 - X.i0;
            for (int rw = threadIdx.x >> 5; rw < rows; rw += blockDim.x >> 5) {
                const float* Gi = Gc + (size_t)X.aidx[X.i0 + rw] * ns;
                for (int c = threadIdx.x & 31; c < na; c += 32)
                    cp_async4(&X.gA[(size_t)rw * lda + c], &Gi[X.aidx[c]], true);
            }
        }
        cp_async_commit();
    } else if (!solo) {   // rows too large for shared memory: this CTA's rows of G_A into its global copy
        const float* Gc = G + off.goff[off.cls[inst]];
        for (int i = X.i0 + (threadIdx.x >> 5); i < X.i1; i += blockDim.x >> 5) {
            const float* Gi = Gc + (size_t)X.aidx[i] * ns;
            for (int c = threadIdx.x & 31; c < na; c += 32) GA[off.gaoff[inst] + (size_t)i * na + c] = Gi[X.aidx[c]];
        }
        __syncthreads();   // visible to this CTA's matvec (L2 loads)
    }
    cr_stamp(23);   // G_A copies issued
    double z[kRpt], p[kRpt], Ap[kRpt], Ar[kRpt];
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        z[k] = p[k] = Ap[k] = Ar[k] = 0.0;
        const int j = threadIdx.x + kCrThreads * k;
        if (j < m) {
            const int c = j / 3;
            const double th = th_g[j];
            double rho = rho_g[j];
            // v0 and s0 loaded together, then c1: two dependent loads instead of three
            const int v0 = __ldg(&cc.v0[cb + c]);
            const int s0i = __ldg(&cc.s0[cb + c]);
            const int c1v = __ldg(&cc.c1[s0i >= 0 ? s0i : 0]);
            const bool viaSlot = v0 >= 0 && s0i >= 0 && c1v == cb + c;
            if (!viaSlot) {   // rho of contacts the chain dot did not cover
                const int kk = j - 3 * c;
                const DContact& ct = I.C[c];
                double xs0 = 0.0, xs1 = 0.0, xs2 = 0.0;
                for (int q = 0; q < ct.nv; ++q) {
                    const double4 xa = x[(size_t)ct.vtx[q] * S + inst];
                    const int slq = ct.slot[q] - sb;
                    xs0 += ct.w[q] * (xa.x + dxt_g[3 * slq]);
                    xs1 += ct.w[q] * (xa.y + dxt_g[3 * slq + 1]);
                    xs2 += ct.w[q] * (xa.z + dxt_g[3 * slq + 2]);
                }
                rho = hv_g[j] - th * (ct.c[kk][0] * xs0 + ct.c[kk][1] * xs1 + ct.c[kk][2] * xs2);
            }
            X.th[j] = (float)th;
            X.cd[j] = (float)cd_g[j];
            X.r[j] = rho;
            p[k] = rho;
        }
    }
    cr_stamp(24);   // rho / vectors staged (this thread)
    cp_async_wait<0>();
    cr_stamp(25);   // this thread's copies landed
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(X.mbar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(X.mbar + 8u));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cl.sync();   // smem staged everywhere; every CTA's exchange mbarriers initialised
    CrRows<kRpt> R;
    cr_rows_init<kRpt>(X, m, R);
    cr_stamp(1);
    if (threadIdx.x == 0 && blockIdx.x == 0) {   // debug: na, G_A placement (1 = shared memory), csize
        g_cr_clock[31] = g_cr_clock[0] + 1000ull * na;
        g_cr_clock[30] = g_cr_clock[0] + 1000ull * (X.gA_smem ? 1 : 0) + 10000ull * csize;
    }
    double rr = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int k = 0; k < kRpt; ++k) rr = fma(p[k], p[k], rr);
    int rb = 0;   // reduction buffer
    block_sum3(rr, t1, t2, X.red + rb * 3 * (kCrThreads / 32));
    rb ^= 1;
    cr_stamp(2);
    if (rr > 0.0 && P.cr_iters > 0) {
        int buf = 0;
        cr_apply<kRpt, kSolo>(X, m, I, buf, Ar, R);
        buf ^= 1;
        double rAr = 0.0, ApAp = 0.0, dummy = 0.0;
#pragma unroll
        for (int k = 0; k < kRpt; ++k) {
            const int j = threadIdx.x + kCrThreads * k;
            Ap[k] = Ar[k];
            if (j < m) {
                rAr = fma(X.r[j], Ar[k], rAr);
                ApAp = fma(Ap[k], Ap[k], ApAp);
            }
        }
        block_sum3(rAr, ApAp, dummy, X.red + rb * 3 * (kCrThreads / 32));
        rb ^= 1;
        for (int it = 0; it < P.cr_iters; ++it) {
            if (ApAp <= 1e-300 || fabs(rAr) <= 1e-300) break;
            const double alpha = rAr / ApAp;
#pragma unroll
            for (int k = 0; k < kRpt; ++k) {
                const int j = threadIdx.x + kCrThreads * k;
                if (j < m) {
                    z[k] += alpha * p[k];
                    X.r[j] -= alpha * Ap[k];
                }
            }
            __syncthreads();
            if (it == P.cr_iters - 1) break;
            X.stamp = it == 3 ? 13 : -1;
            if (it == 3) cr_stamp(12);
            cr_apply<kRpt, kSolo>(X, m, I, buf, Ar, R);
            buf ^= 1;
            if (it == 3) cr_stamp(16);
            double s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int k = 0; k < kRpt; ++k) {
                const int j = threadIdx.x + kCrThreads * k;
                if (j < m) {
                    s1 = fma(X.r[j], Ar[k], s1);
                    s2 = fma(Ar[k], Ar[k], s2);
                    s3 = fma(Ar[k], Ap[k], s3);
                }
            }
            block_sum3(s1, s2, s3, X.red + rb * 3 * (kCrThreads / 32));
            rb ^= 1;
            const double beta = s1 / rAr;
            rAr = s1;
            // |Ap_new|^2 = |Ar + beta Ap|^2 by its expansion (no extra reduction) unless the expansion
            // cancels: then the direct sum (a uniform branch; the expansion loses all digits when
            // Ar ~ -beta Ap and would turn alpha into noise)
            const double apx = s2 + 2.0 * beta * s3 + beta * beta * ApAp;
            const double aps = s2 + beta * beta * ApAp;
#pragma unroll
            for (int k = 0; k < kRpt; ++k) {
                const int j = threadIdx.x + kCrThreads * k;   // entries past m stay 0
                p[k] = j < m ? X.r[j] + beta * p[k] : 0.0;
                Ap[k] = Ar[k] + beta * Ap[k];
            }
            if (apx > 1e-3 * aps) {
                ApAp = apx;
            } else {
                double d = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
                for (int k = 0; k < kRpt; ++k)
                    if (threadIdx.x + kCrThreads * k < m) d = fma(Ap[k], Ap[k], d);
                block_sum3(d, e1, e2, X.red + rb * 3 * (kCrThreads / 32));
                rb ^= 1;
                ApAp = d;
            }
            if (it == 3) cr_stamp(17);
            if (it < 9 && it != 3) cr_stamp(3 + it);
        }
    }
    cr_stamp(20);
    double res = 0.0, u1 = 0.0, u2 = 0.0;
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        const int j = threadIdx.x + kCrThreads * k;
        if (j < m) res = fma(X.r[j], X.r[j], res);
    }
    block_sum3(res, u1, u2, X.red + rb * 3 * (kCrThreads / 32));
    cr_stamp(27);
    // epilogue split over the cluster (every CTA holds the identical z):
    // lambda += z / h^2 (reading A11) for this CTA's rows; z to shared memory (reuse r)
    const int rper = (m + csize - 1) / csize;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        const int j = threadIdx.x + kCrThreads * k;
        if (j < m) {
            X.r[j] = z[k];
            if (j / rper == rank) lam_g[j] += z[k] / (h * h);
        }
    }
    __syncthreads();
    cr_stamp(28);
    // wz_b = sum w theta z c  (for y += K H^T z), this CTA's slots
    const int sper = (ns + csize - 1) / csize;
    for (int b = rank * sper + threadIdx.x; b < min(ns, (rank + 1) * sper); b += blockDim.x) {
        double w0 = 0, w1 = 0, w2 = 0;
        const int onlyg = __ldg(&cc.c1[sb + b]);
        const int qa = onlyg >= 0 ? 0 : I.scp[b], qb = onlyg >= 0 ? 1 : I.scp[b + 1];
        for (int q = qa; q < qb; ++q) {
            const int c = onlyg >= 0 ? onlyg - cb : sl.sci[q] - cb;
            const double wt = onlyg >= 0 ? 1.0 : (double)sl.scw[q];
            const float* c9 = X.c9 + 9 * c;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double tv = wt * (double)X.th[3 * c + k] * X.r[3 * c + k];
                w0 += tv * (double)c9[3 * k];
                w1 += tv * (double)c9[3 * k + 1];
                w2 += tv * (double)c9[3 * k + 2];
            }
        }
        wz_g[3 * b] = w0;
        wz_g[3 * b + 1] = w1;
        wz_g[3 * b + 2] = w2;
        if (cs.wzT) cs.wzT[(size_t)b * S + inst] = make_float4((float)w0, (float)w1, (float)w2, 0.f);
    }
    if (threadIdx.x == 0 && rank == 0) cs.cr_res[inst] = sqrt(res);
    cr_stamp(21);
    // no trailing cluster barrier: after its last exchange wait no CTA touches a peer's shared memory
}

// ----------------------------------------------------------------------------
// Grid CR: the constraint solve for contact sets too large for one cluster's shared memory
// (one scene, any number of contacts, e.g. a multi-object pile).  Same algorithm as k_cr
// (Saad's CR from z = 0, exactly N_CR matvecs, stop only on breakdown; reading A19), with
// the vectors in global memory and one kernel per phase:
//   gcr_slot   W_b = sum_{(c, w) on slot b} w sum_k theta_ck v_ck c_ck       (J^T Theta v)
//   gcr_gram   q_a = sum_b G[a][b] W_b over a's Delassus group                (A^-1 on V_c)
//   gcr_row    (S v)_j = theta_j c_j . sum_q w_q q_{slot q} + C_j v_j, partial dots
//   gcr_update every CTA reduces the partials in a fixed order, then the CR vector updates
// The Delassus Gram is stored per group = etree component (a tree of the forest): K is
// block-diagonal over the components, so G[a][b] = 0 across them (Theorem 1).
// ----------------------------------------------------------------------------
constexpr int kGcrThreads = 256;


__device__ __forceinline__ void block_sum3_gcr(double& a, double& b, double& c, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    a = warp_sum(a); b = warp_sum(b); c = warp_sum(c);
    if (lane == 0) { red[w] = a; red[nw + w] = b; red[2 * nw + w] = c; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0, s1 = 0, s2 = 0;
        for (int q = 0; q < nw; ++q) { s0 += red[q]; s1 += red[nw + q]; s2 += red[2 * nw + q]; }
        red[3 * nw] = s0; red[3 * nw + 1] = s1; red[3 * nw + 2] = s2;
    }
    __syncthreads();
    a = red[3 * nw]; b = red[3 * nw + 1]; c = red[3 * nw + 2];
}

// r = rho (rho of multi-vertex contacts here; single-vertex ones come from the chain dot), z = 0
__global__ void k_gcr_init(Params P, GcrData g, const DContact* __restrict__ C, CrContacts cc,
                           const double4* __restrict__ x, ContactState cs) {
    pdl_enter();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P.C) return;
    const int v0 = cc.v0[c];
    const bool viaSlot = v0 >= 0 && cc.c1[cc.s0[c]] == c;
    double xs0 = 0.0, xs1 = 0.0, xs2 = 0.0;
    const DContact& ct = C[c];
    if (!viaSlot)
        for (int q = 0; q < ct.nv; ++q) {
            const double4 xa = x[(size_t)ct.vtx[q] * P.S + ct.inst];
            const int s = ct.slot[q];
            xs0 += ct.w[q] * (xa.x + cs.dxt[3 * s]);
            xs1 += ct.w[q] * (xa.y + cs.dxt[3 * s + 1]);
            xs2 += ct.w[q] * (xa.z + cs.dxt[3 * s + 2]);
        }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int j = 3 * c + k;
        const double rho = viaSlot ? cs.rho[j]
                                   : cs.hvec[j] - cs.theta[j] * (ct.c[k][0] * xs0 + ct.c[k][1] * xs1 + ct.c[k][2] * xs2);
        cs.rho[j] = rho;
        g.r[j] = rho;
        g.z[j] = 0.0;
    }
}

// W_b = sum over the contacts on slot b of w * sum_k theta_k v_k c_k  (fixed contact order)
__global__ void k_gcr_slot(int NS, Slots sl, CrContacts cc, const double* __restrict__ theta,
                           const double* __restrict__ v, double* __restrict__ W) {
    pdl_enter();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= NS) return;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    for (int p = sl.scp[b]; p < sl.scp[b + 1]; ++p) {
        const int c = sl.sci[p];
        const double wt = (double)sl.scw[p];
        const float* c9 = cc.c9 + 9 * (size_t)c;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double tv = wt * theta[3 * c + k] * v[3 * c + k];
            w0 = fma(tv, (double)c9[3 * k], w0);
            w1 = fma(tv, (double)c9[3 * k + 1], w1);
            w2 = fma(tv, (double)c9[3 * k + 2], w2);
        }
    }
    W[3 * b] = w0;
    W[3 * b + 1] = w1;
    W[3 * b + 2] = w2;
}

// q_a = sum_{b in group(a)} G[a][b] W_b.  One CTA per (group, 32 consecutive rows): the
// group's W is staged in shared memory (fp64 SoA); warp w owns rows w, w+8, w+16, w+24 and
// streams the 4 G rows together (4 independent loads in flight per lane and step).
// Groups wider than kGramSmemSlots fall back to one warp per row reading W from L1/L2.
constexpr int kGramSmemSlots = 2000;   // 47 KB of fp64 W (static shared memory)

__global__ void __launch_bounds__(256) k_gcr_gram(int NS, GcrData g, const int2* __restrict__ items) {
    pdl_enter();
    __shared__ double Ws[3 * kGramSmemSlots];
    const int2 it = items[blockIdx.x];   // {first row (global slot), rows}
    const int a0 = it.x, nrows = it.y;
    const int b0 = g.gs0[a0], n = g.gn[a0];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool smem = n <= kGramSmemSlots;
    if (smem) {
        for (int b = threadIdx.x; b < n; b += blockDim.x) {
            Ws[b] = g.W[3 * (size_t)(b0 + b)];
            Ws[kGramSmemSlots + b] = g.W[3 * (size_t)(b0 + b) + 1];
            Ws[2 * kGramSmemSlots + b] = g.W[3 * (size_t)(b0 + b) + 2];
        }
        __syncthreads();
        const float* rows[4];
        double acc[4][3];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int r = min(w + 8 * k, nrows - 1);
            rows[k] = g.G + g.rowoff[a0 + r];
            acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
        }
        for (int b = lane; b < n; b += 32) {
            float gv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) gv[k] = __ldcs(&rows[k][b]);
            const double w0 = Ws[b], w1 = Ws[kGramSmemSlots + b], w2 = Ws[2 * kGramSmemSlots + b];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                acc[k][0] = fma((double)gv[k], w0, acc[k][0]);
                acc[k][1] = fma((double)gv[k], w1, acc[k][1]);
                acc[k][2] = fma((double)gv[k], w2, acc[k][2]);
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double d0 = warp_sum(acc[k][0]), d1 = warp_sum(acc[k][1]), d2 = warp_sum(acc[k][2]);
            const int r = w + 8 * k;
            if (lane == 0 && r < nrows) {
                g.q[3 * (size_t)(a0 + r)] = d0;
                g.q[3 * (size_t)(a0 + r) + 1] = d1;
                g.q[3 * (size_t)(a0 + r) + 2] = d2;
            }
        }
        return;
    }
    for (int r = w; r < nrows; r += 8) {
        const float* row = g.G + g.rowoff[a0 + r];
        const double* W = g.W + 3 * (size_t)b0;
        double d0 = 0.0, d1 = 0.0, d2 = 0.0;
        for (int b = lane; b < n; b += 32) {
            const double gv = (double)__ldg(&row[b]);
            d0 = fma(gv, W[3 * b], d0);
            d1 = fma(gv, W[3 * b + 1], d1);
            d2 = fma(gv, W[3 * b + 2], d2);
        }
        d0 = warp_sum(d0);
        d1 = warp_sum(d1);
        d2 = warp_sum(d2);
        if (lane == 0) {
            g.q[3 * (size_t)(a0 + r)] = d0;
            g.q[3 * (size_t)(a0 + r) + 1] = d1;
            g.q[3 * (size_t)(a0 + r) + 2] = d2;
        }
    }
}

// Ar_j = theta_j c_j . sum_q w_q q_{slot q} + C_j r_j; per-CTA partials of r.Ar, Ar.Ar, Ar.Ap
__global__ void __launch_bounds__(kGcrThreads) k_gcr_row(Params P, GcrData g, const DContact* __restrict__ C,
                                                       ContactState cs, int first) {
    pdl_enter();
    __shared__ double red[3 * (kGcrThreads / 32) + 3];
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (c < P.C) {
        const DContact& ct = C[c];
        double q0 = 0.0, q1 = 0.0, q2 = 0.0;
        for (int p = 0; p < ct.nv; ++p) {
            const int s = ct.slot[p];
            q0 += ct.w[p] * g.q[3 * s];
            q1 += ct.w[p] * g.q[3 * s + 1];
            q2 += ct.w[p] * g.q[3 * s + 2];
        }
        const float* c9 = g.c9 + 9 * (size_t)c;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int j = 3 * c + k;
            const double th = cs.theta[j];
            const double acc = th != 0.0 ? (double)c9[3 * k] * q0 + (double)c9[3 * k + 1] * q1 +
                                               (double)c9[3 * k + 2] * q2
                                         : 0.0;
            const double rj = g.r[j];
            const double ar = th * acc + cs.cdiag[j] * rj;
            g.Ar[j] = ar;
            s1 = fma(rj, ar, s1);
            s2 = fma(ar, ar, s2);
            if (!first) s3 = fma(ar, g.Ap[j], s3);
        }
    }
    block_sum3_gcr(s1, s2, s3, red);
    if (threadIdx.x == 0) {
        g.part[3 * blockIdx.x] = s1;
        g.part[3 * blockIdx.x + 1] = s2;
        g.part[3 * blockIdx.x + 2] = s3;
    }
}

// CR iteration `it`, first half: r.Ar from the row partials (same fixed order in every CTA), beta,
// p = r + beta p, Ap = Ar + beta Ap, and this CTA's partial |Ap|^2 (part[3 b + 2]; the row
// kernel's s3 slot, unused since |Ap|^2 is reduced directly).  Scalars ping-pong between
// sc[.. + (it & 1)] (read) and sc[.. + ((it + 1) & 1)] (written by CTA 0); launched on the row blocks.
__global__ void __launch_bounds__(kGcrThreads) k_gcr_update(GcrData g, int m, int it) {
    pdl_enter();
    __shared__ double sh[2];
    __shared__ double red[3 * (kGcrThreads / 32) + 3];
    const int rp = it & 1, wp = rp ^ 1;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double s1 = 0.0;
        for (int b = lane; b < g.nblk; b += 32) s1 += g.part[3 * b];
        s1 = warp_sum(s1);
        if (lane == 0) {
            const double stop = it == 0 ? 0.0 : g.sc[4 + rp];
            const double beta = (it == 0 || stop != 0.0) ? 0.0 : s1 / g.sc[rp];
            sh[0] = beta;
            sh[1] = stop;
            if (blockIdx.x == 0) {
                g.sc[wp] = s1;
                g.sc[4 + wp] = stop;
            }
        }
    }
    __syncthreads();
    const double beta = sh[0];
    double d = 0.0, e1 = 0.0, e2 = 0.0;
    if (sh[1] == 0.0) {
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
            double p, Ap;
            if (it == 0) {
                p = g.r[j];
                Ap = g.Ar[j];
            } else {
                p = g.r[j] + beta * g.p[j];
                Ap = g.Ar[j] + beta * g.Ap[j];
            }
            g.p[j] = p;
            g.Ap[j] = Ap;
            d = fma(Ap, Ap, d);
        }
    }
    block_sum3_gcr(d, e1, e2, red);
    if (threadIdx.x == 0) g.part[3 * blockIdx.x + 2] = d;
}

// second half: |Ap|^2 from the partials (fixed order), breakdown test (reading A19), alpha = r.Ar /
// |Ap|^2, z += alpha p, r -= alpha Ap.  Every CTA takes the same decision from the same sums.
__global__ void __launch_bounds__(kGcrThreads) k_gcr_step(GcrData g, int m, int it) {
    pdl_enter();
    __shared__ double sh[2];
    const int wp = (it & 1) ^ 1;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double ApAp = 0.0;
        for (int b = lane; b < g.nblk; b += 32) ApAp += g.part[3 * b + 2];
        ApAp = warp_sum(ApAp);
        if (lane == 0) {
            const double rAr = g.sc[wp];
            double stop = g.sc[4 + wp];
            if (stop == 0.0 && (ApAp <= 1e-300 || fabs(rAr) <= 1e-300)) stop = 1.0;
            sh[0] = stop != 0.0 ? 0.0 : rAr / ApAp;
            sh[1] = stop;
            if (blockIdx.x == 0) g.sc[2 + wp] = ApAp;
        }
    }
    __syncthreads();
    if (sh[1] != 0.0) {   // broken down (now or earlier): keep the iterate
        if (blockIdx.x == 0 && threadIdx.x == 0) g.sc[4 + wp] = 1.0;
        return;
    }
    const double alpha = sh[0];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        g.z[j] += alpha * g.p[j];
        g.r[j] -= alpha * g.Ap[j];
    }
}

// lambda += z / h^2 (reading A11); |r| -> cr_res by the last CTA to finish (partials summed
// in CTA order, so the value is deterministic)
__global__ void __launch_bounds__(kGcrThreads) k_gcr_final(GcrData g, int m, double h, double* lam, double* cr_res) {
    pdl_enter();
    __shared__ double red[3 * (kGcrThreads / 32) + 3];
    __shared__ bool last;
    double rr = 0.0, d1 = 0.0, d2 = 0.0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        lam[j] += g.z[j] / (h * h);
        rr = fma(g.r[j], g.r[j], rr);
    }
    block_sum3_gcr(rr, d1, d2, red);
    if (threadIdx.x == 0) {
        g.part[3 * blockIdx.x] = rr;
        __threadfence();
        last = atomicAdd(g.cnt, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double t = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(&g.part[3 * b]);
        cr_res[0] = sqrt(t);
        *g.cnt = 0;
    }
}

// D_jj = sum_{p,q} w_p w_q G[slot p][slot q] over pairs in the same Delassus group (reading A18)
__global__ void k_djj_grid(int C, DContact* Cs, GcrData g) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    DContact& ct = Cs[c];
    double d = 0.0;
    for (int p = 0; p < ct.nv; ++p)
        for (int q = 0; q < ct.nv; ++q) {
            const int sp = ct.slot[p], sq = ct.slot[q];
            if (g.gs0[sp] != g.gs0[sq]) continue;
            d += ct.w[p] * ct.w[q] * (double)g.G[g.rowoff[sp] + (sq - g.gs0[sq])];
        }
    ct.Djj = d;
}

void launch_djj_grid(cudaStream_t st, const Params& P, DContact* c, GcrData g) {
    if (P.C == 0) return;
    k_djj_grid<<<(P.C + 127) / 128, 128, 0, st>>>(P.C, c, g);
}

int gcr_row_blocks(int C) { return (C + kGcrThreads - 1) / kGcrThreads; }

int launch_gcr(cudaStream_t st, const Params& P, GcrData g, const DContact* c, CrContacts cc, Slots sl,
               const double4* x, ContactState cs) {
    if (P.C == 0) return 0;
    const int m = 3 * P.C, NS = P.NS;
    const int nb = gcr_row_blocks(P.C);
    const int ub = std::min(148, (m + kGcrThreads - 1) / kGcrThreads);
    g.nblk = nb;
    launch_pdl(k_gcr_init, dim3(nb), dim3(kGcrThreads), 0, st, P, g, c, cc, x, cs);
    for (int it = 0; it < P.cr_iters; ++it) {
        launch_pdl(k_gcr_slot, dim3((NS + 255) / 256), dim3(256), 0, st, NS, sl, cc, (const double*)cs.theta,
                   (const double*)g.r, g.W);
        launch_pdl(k_gcr_gram, dim3(g.n_gram_items), dim3(256), 0, st, NS, g, g.gram_items);
        launch_pdl(k_gcr_row, dim3(nb), dim3(kGcrThreads), 0, st, P, g, c, cs, (int)(it == 0));
        launch_pdl(k_gcr_update, dim3(nb), dim3(kGcrThreads), 0, st, g, m, it);
        launch_pdl(k_gcr_step, dim3(ub), dim3(kGcrThreads), 0, st, g, m, it);
    }
    launch_pdl(k_gcr_final, dim3(ub), dim3(kGcrThreads), 0, st, g, m, P.h, cs.lam, cs.cr_res);
    launch_pdl(k_gcr_slot, dim3((NS + 255) / 256), dim3(256), 0, st, NS, sl, cc, (const double*)cs.theta,
               (const double*)g.z, cs.wz);
    return (int)cudaGetLastError();
}

int gcr_kernels_per_iteration(int cr_iters) { return 3 + 5 * cr_iters; }

int read_cr_clock(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_cr_clock, sizeof(unsigned long long) * 32);
}

size_t cr_smem_bytes(int nc, int ns) { return CrLayout(nc, ns, ns, false).total; }

int cr_cluster_size(int S) {
    int c = kCluster;
    while (c > 1 && c * S > 148) c >>= 1;   // enough CTAs per instance to fill the GPU, no more
    return c;
}

int launch_cr(cudaStream_t st, const Params& P, InstOff off, const DContact* c, CrContacts cc, Slots sl,
              const float* G, const float* GA, const double4* x, ContactState cs, CrActive act) {
    if (P.C == 0) return 0;
    static unsigned long long attr = 0;
    cudaError_t err = cudaSuccess;
    per_device_once(attr, [&] {
        void* fns[2 * kRptMax] = {(void*)k_cr<1, 0>, (void*)k_cr<2, 0>, (void*)k_cr<3, 0>, (void*)k_cr<4, 0>,
                                  (void*)k_cr<5, 0>, (void*)k_cr<6, 0>, (void*)k_cr<1, 1>, (void*)k_cr<2, 1>,
                                  (void*)k_cr<3, 1>, (void*)k_cr<4, 1>, (void*)k_cr<5, 1>, (void*)k_cr<6, 1>};
        for (void* f : fns) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) { err = e; return; }
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCrMaxSmem);
            if (e != cudaSuccess) { err = e; return; }
        }
    });
    if (err != cudaSuccess) return (int)err;
    const int csize = cr_cluster_size(P.S);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.S * csize, 1, 1);
    cfg.blockDim = dim3(kCrThreads, 1, 1);
    cfg.dynamicSmemBytes = kCrMaxSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    const int rpt = (3 * P.nc_max + kCrThreads - 1) / kCrThreads;
    cudaError_t e;
#define SIM_CR_LAUNCH(R)                                                                                   \
    (csize == 1 ? cudaLaunchKernelEx(&cfg, k_cr<R, 1>, P, off, c, cc, sl, G, const_cast<float*>(GA), x, cs, act) \
                : cudaLaunchKernelEx(&cfg, k_cr<R, 0>, P, off, c, cc, sl, G, const_cast<float*>(GA), x, cs, act))
    switch (rpt) {
        case 0:
        case 1: e = SIM_CR_LAUNCH(1); break;
        case 2: e = SIM_CR_LAUNCH(2); break;
        case 3: e = SIM_CR_LAUNCH(3); break;
        case 4: e = SIM_CR_LAUNCH(4); break;
        case 5: e = SIM_CR_LAUNCH(5); break;
        default: e = SIM_CR_LAUNCH(6); break;
    }
#undef SIM_CR_LAUNCH
    return (int)e;
}

}  // namespace simdev
