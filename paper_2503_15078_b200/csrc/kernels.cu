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
// No tensor cores: every step is sparse / memory- or latency-bound.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace simdev {

// ----------------------------------------------------------------------------
// predict: s = x_t + h v_t + h^2 g; x^0 = s; pinned: x = x_t + h v_pin
// ----------------------------------------------------------------------------
__global__ void k_predict(Params P, double4* __restrict__ x, double4* __restrict__ xt,
                          double4* __restrict__ v, double4* __restrict__ s, double* __restrict__ lam, int nlam) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nlam) lam[i] = 0.0;   // lambda^0 = 0 (reading A10)
    if (i >= P.n_v) return;
    double4 xi = x[i];
    xt[i] = xi;
    double h = P.h;
    if (i < P.n_f) {
        double4 vi = v[i];
        double4 si = make_double4(xi.x + h * vi.x + h * h * P.g[0], xi.y + h * vi.y + h * h * P.g[1],
                                  xi.z + h * vi.z + h * h * P.g[2], 0.0);
        s[i] = si;
        x[i] = si;
    } else {
        x[i] = make_double4(xi.x + h * P.vpin[0], xi.y + h * P.vpin[1], xi.z + h * P.vpin[2], 0.0);
        v[i] = make_double4(P.vpin[0], P.vpin[1], P.vpin[2], 0.0);
    }
}

void launch_predict(cudaStream_t st, const Params& P, double4* x, double4* xt, double4* v, double4* s,
                    double* lam, int nlam) {
    int n = P.n_v > nlam ? P.n_v : nlam;
    k_predict<<<(n + 255) / 256, 256, 0, st>>>(P, x, xt, v, s, lam, nlam);
}

// ----------------------------------------------------------------------------
// local step
// ----------------------------------------------------------------------------
// Jacobi eigen-decomposition of a symmetric 3x3 (cyclic, Rutishauser rotations).
__device__ __forceinline__ void jacobi3(float S[3][3], float V[3][3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.f : 0.f;
#pragma unroll 1
    for (int sweep = 0; sweep < 6; ++sweep) {
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
            float theta = (S[q][q] - S[p][p]) / (2.f * apq);
            float at = fabsf(theta);
            float t = at > 1e15f ? 0.5f / at : 1.f / (at + sqrtf(theta * theta + 1.f));
            t = theta < 0.f ? -t : t;
            float c = rsqrtf(t * t + 1.f);
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
__device__ __forceinline__ float nh_f(const float p[3], const float sg[3], float k, float mu, float lam) {
    float lnJ = logf(p[0]) + logf(p[1]) + logf(p[2]);
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
    // Neo-Hookean: damped Newton from p0 = max(sig, 0.05), <= 16 iterations
    float p[3] = {fmaxf(sg[0], 0.05f), fmaxf(sg[1], 0.05f), fmaxf(sg[2], 0.05f)};
    float scale = fmaxf(1.f, sqrtf(sg[0] * sg[0] + sg[1] * sg[1] + sg[2] * sg[2]));
#pragma unroll 1
    for (int it = 0; it < 16; ++it) {
        float lnJ = logf(p[0]) + logf(p[1]) + logf(p[2]);
        float iv[3] = {1.f / p[0], 1.f / p[1], 1.f / p[2]};
        float g[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) g[i] = k * (p[i] - sg[i]) + mu * p[i] - mu * iv[i] + lam * lnJ * iv[i];
        float gn = sqrtf(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
        if (gn <= 2e-6f * k * scale) break;
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
            float id = 1.f / det;
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
            float s = -1.f / (k + mu);
            dd[0] = s * g[0];
            dd[1] = s * g[1];
            dd[2] = s * g[2];
        }
        float slope = dd[0] * g[0] + dd[1] * g[1] + dd[2] * g[2];
        float f0 = nh_f(p, sg, k, mu, lam);
        float fr = 2e-6f * (k * (p[0] * p[0] + p[1] * p[1] + p[2] * p[2] + sg[0] * sg[0] + sg[1] * sg[1] +
                                 sg[2] * sg[2]) + mu * fabsf(lnJ) + lam * lnJ * lnJ + mu);
        float t = 1.f;
#pragma unroll 1
        for (int ls = 0; ls < 40; ++ls) {
            float pn[3] = {p[0] + t * dd[0], p[1] + t * dd[1], p[2] + t * dd[2]};
            if (pn[0] > 0.f && pn[1] > 0.f && pn[2] > 0.f) {
                float fn = nh_f(pn, sg, k, mu, lam);
                if (fn <= f0 + 1e-4f * t * slope + fr) break;
            }
            t *= 0.5f;
        }
        p[0] += t * dd[0];
        p[1] += t * dd[1];
        p[2] += t * dd[2];
    }
    d[0] = p[0] - sg[0];
    d[1] = p[1] - sg[1];
    d[2] = p[2] - sg[2];
}

// one thread per tet: f_a = h^2 w (P - F) g_a, written per corner
__global__ void __launch_bounds__(128) k_local(Params P, const int4* __restrict__ tet, const float* __restrict__ Bm,
                                               const float* __restrict__ hw2, const double4* __restrict__ x,
                                               float4* __restrict__ fc, float* __restrict__ Pdbg) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.n_t) return;
    const int nt = P.n_t;
    int4 tv = __ldg(&tet[t]);
    double4 x0 = x[tv.x], x1 = x[tv.y], x2 = x[tv.z], x3 = x[tv.w];
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
    // S = F^T F, eigenvectors V
    float S[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) S[i][j] = F[0][i] * F[0][j] + F[1][i] * F[1][j] + F[2][i] * F[2][j];
    float V[3][3];
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
    float U[3][3];
    float n0 = sqrtf(FV[0][0] * FV[0][0] + FV[1][0] * FV[1][0] + FV[2][0] * FV[2][0]);
    if (n0 > 1e-30f) {
        U[0][0] = FV[0][0] / n0; U[1][0] = FV[1][0] / n0; U[2][0] = FV[2][0] / n0;
    } else {
        U[0][0] = 1.f; U[1][0] = 0.f; U[2][0] = 0.f;
    }
    float dt = U[0][0] * FV[0][1] + U[1][0] * FV[1][1] + U[2][0] * FV[2][1];
    float w0 = FV[0][1] - dt * U[0][0], w1 = FV[1][1] - dt * U[1][0], w2 = FV[2][1] - dt * U[2][0];
    float n1 = sqrtf(w0 * w0 + w1 * w1 + w2 * w2);
    if (n1 > 1e-30f * fmaxf(1.f, n0)) {
        U[0][1] = w0 / n1; U[1][1] = w1 / n1; U[2][1] = w2 / n1;
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
    float dlt[3];
    project_sigma(P.model, sg, P.k, P.mu, P.lam, dlt);
    // Q = hw2 * U diag(delta) V^T  (= h^2 w (P - F))
    float hw = __ldg(&hw2[t]);
    float Q[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Q[i][j] = hw * (U[i][0] * dlt[0] * V[j][0] + U[i][1] * dlt[1] * V[j][1] + U[i][2] * dlt[2] * V[j][2]);
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
    float4* o = fc + 4 * (size_t)t;
    o[0] = make_float4(-(f[0][0] + f[1][0] + f[2][0]), -(f[0][1] + f[1][1] + f[2][1]), -(f[0][2] + f[1][2] + f[2][2]), 0.f);
    o[1] = make_float4(f[0][0], f[0][1], f[0][2], 0.f);
    o[2] = make_float4(f[1][0], f[1][1], f[1][2], 0.f);
    o[3] = make_float4(f[2][0], f[2][1], f[2][2], 0.f);
}

void launch_local(cudaStream_t st, const Params& P, const int4* tet, const float* Bm, const float* hw2,
                  const double4* x, float4* fc, float* Pdbg) {
    k_local<<<(P.n_t + 127) / 128, 128, 0, st>>>(P, tet, Bm, hw2, x, fc, Pdbg);
}

// ----------------------------------------------------------------------------
// contact evaluation (fp64): gaps at x^k (reading A22), FB indicators (App. B.2)
// ----------------------------------------------------------------------------
__global__ void k_contact_eval(Params P, const DContact* __restrict__ C, const double4* __restrict__ x,
                               const double4* __restrict__ xt, ContactState cs) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P.nc) return;
    const DContact& ct = C[c];
    double h = P.h;
    double xc[3] = {0, 0, 0}, xtc[3] = {0, 0, 0};
    for (int q = 0; q < ct.nv; ++q) {
        double4 a = x[ct.vtx[q]], b = xt[ct.vtx[q]];
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
    double rn = h * h * ct.Djj, rf = h * ct.Djj;
    // normal FB (A15)
    double y = Jx[0] - ct.dn, ln = lam[0];
    double S = sqrt(y * y + rn * rn * ln * ln);
    double phin, thn, En;
    if (S > 0.0) {
        double a = y + rn * ln;
        phin = a > 0.0 ? (2.0 * y * rn * ln) / (a + S) : a - S;
        thn = 1.0 - y / S;
        En = (1.0 - rn * ln / S) * rn;
    } else {
        phin = 0.0; thn = 1.0; En = 0.0;
    }
    phin_abs = fabs(phin);
    // friction (A14, A16, A16b)
    double yd1 = (Jx[1] - Jxt[1]) / h - ct.df1, yd2 = (Jx[2] - Jxt[2]) / h - ct.df2;
    double thf, Ef;
    if (ln > 0.0 && ct.mu * ln > 0.0) {
        double s = sqrt(yd1 * yd1 + yd2 * yd2);
        double lf = sqrt(lam[1] * lam[1] + lam[2] * lam[2]);
        double q = ct.mu * ln - lf;
        double R = sqrt(s * s + rf * rf * q * q);
        double num = rf * (R - rf * q);
        double den = s + ct.mu * rf * ln - R;
        double fl = 1e-6 * (s + ct.mu * rf * ln);
        den = den > fl ? den : fl;
        Ef = den > 0.0 ? num / den : 0.0;
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
    if (P.nc == 0) return;
    k_contact_eval<<<(P.nc + 127) / 128, 128, 0, st>>>(P, c, x, xt, cs);
}

// ----------------------------------------------------------------------------
// gather: u_a = M_a (s_a - x_a) + sum_{(t,c) in adj(a)} f_{t,c} + h^2 (H^T lam)_a
// (colour-free: each free vertex sums its incident tets in a fixed order)
// ----------------------------------------------------------------------------
__global__ void k_gather(Params P, const int32_t* __restrict__ adjp, const int32_t* __restrict__ adj,
                         const float4* __restrict__ fc, const double* __restrict__ M, const double4* __restrict__ x,
                         const double4* __restrict__ s, const int32_t* __restrict__ vcp,
                         const int32_t* __restrict__ vci, const float* __restrict__ vcw,
                         const double* __restrict__ hl, const int32_t* __restrict__ cb, float4* __restrict__ u,
                         double* __restrict__ resid) {
    int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= P.n_f) return;
    double4 xa = x[a], sa = s[a];
    double m = M[a];
    double r0 = m * (sa.x - xa.x), r1 = m * (sa.y - xa.y), r2 = m * (sa.z - xa.z);
    int p0 = adjp[a], p1 = adjp[a + 1];
    float f0 = 0.f, f1 = 0.f, f2 = 0.f;
    for (int p = p0; p < p1; ++p) {
        float4 f = __ldg(&fc[adj[p]]);
        f0 += f.x;
        f1 += f.y;
        f2 += f.z;
    }
    r0 += f0;
    r1 += f1;
    r2 += f2;
    if (resid) {
        resid[3 * (size_t)a] = r0;
        resid[3 * (size_t)a + 1] = r1;
        resid[3 * (size_t)a + 2] = r2;
    }
    if (vcp) {
        double hh = P.h * P.h;
        for (int p = vcp[a]; p < vcp[a + 1]; ++p) {
            int c = vci[p];
            double w = vcw[p];
            r0 += hh * w * hl[3 * c];
            r1 += hh * w * hl[3 * c + 1];
            r2 += hh * w * hl[3 * c + 2];
        }
    }
    u[a] = make_float4((float)r0, (float)r1, (float)r2, __int_as_float(cb[a]));
}

void launch_gather(cudaStream_t st, const Params& P, const int32_t* adjp, const int32_t* adj,
                   const float4* fc, const double* M, const double4* x, const double4* s,
                   const int32_t* vcp, const int32_t* vci, const float* vcw, const double* hl,
                   const int32_t* cb, float4* u, double* resid_dbg) {
    k_gather<<<(P.n_f + 255) / 256, 256, 0, st>>>(P, adjp, adj, fc, M, x, s, vcp, vci, vcw, hl, cb, u, resid_dbg);
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
constexpr int kStages2 = 3;      // pass-2 tiles in flight per warp
constexpr int kWarps2 = 6;       // pass-2 warps per CTA

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
    static bool attr = false;
    static int nsm = 148;
    if (!attr) {
        cudaFuncSetAttribute(k_kpass1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kKpassSmem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        attr = true;
    }
    const int ctas = std::min((nitems + kWarps - 1) / kWarps, 2 * nsm);   // persistent: 2 CTAs per SM
    k_kpass1<<<ctas, 32 * kWarps, kKpassSmem, st>>>(it, nitems, bl, T1, u, y, part, counters);
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
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_kpass2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kKpass2Smem);
        attr = true;
    }
    k_kpass2<<<nblocks, 32 * kWarps2, kKpass2Smem, st>>>(bl, cover, T2, y, x, xt, v, inv_h, finalize_v);
}

// ----------------------------------------------------------------------------
// chain dot: dxt_s = (K^T y)_{a_s} = sum_{k} Kcol[colptr_a + k] y[chain_rows[off_s + k]]
// (column a of K is contiguous in Kcol; its rows are a's ancestor chain)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_chain_dot(int ns, const int32_t* __restrict__ slot_vtx,
                                                   const float* __restrict__ Kcol, const int64_t* __restrict__ colptr,
                                                   const int32_t* __restrict__ chain_off,
                                                   const int32_t* __restrict__ chain_rows, const float4* __restrict__ y,
                                                   double* __restrict__ dxt, CrContacts cc,
                                                   const double4* __restrict__ x, ContactState cs) {
    // one CTA per contact vertex; its 8 warps take interleaved 128-entry slices of the chain
    __shared__ double s_red[3][kWarps];
    const int s = blockIdx.x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int a = slot_vtx[s];
    const float* col = Kcol + colptr[a];
    const int o0 = chain_off[s], len = chain_off[s + 1] - o0;
    double a0 = 0, a1 = 0, a2 = 0;
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
        for (int u = 0; u < 4; ++u) yy[u] = rw[u] >= 0 ? __ldg(&y[rw[u]]) : make_float4(0.f, 0.f, 0.f, 0.f);
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
        s_red[0][w] = a0;
        s_red[1][w] = a1;
        s_red[2][w] = a2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int q = 0; q < kWarps; ++q) { t0 += s_red[0][q]; t1 += s_red[1][q]; t2 += s_red[2][q]; }
        dxt[3 * s] = t0;
        dxt[3 * s + 1] = t1;
        dxt[3 * s + 2] = t2;
        // Schur RHS rho = h - theta J x~, x~ = x^k + K^T y, for the single contact on this slot
        // (other contacts are handled in the CR prologue)
        const int c = cc.c1[s];
        if (c >= 0) {
            const double4 xa = x[cc.v0[c]];
            const double xs0 = xa.x + t0, xs1 = xa.y + t1, xs2 = xa.z + t2;
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                const float* c3 = cc.c9 + 9 * c + 3 * kk;
                cs.rho[3 * c + kk] = cs.hvec[3 * c + kk] - cs.theta[3 * c + kk] * ((double)c3[0] * xs0 +
                                                                                   (double)c3[1] * xs1 +
                                                                                   (double)c3[2] * xs2);
            }
        }
    }
}

void launch_chain_dot(cudaStream_t st, int ns, const int32_t* slot_vtx, const float* Kcol,
                      const int64_t* colptr, const int32_t* chain_off, const int32_t* chain_rows,
                      const float4* y, double* dxt, CrContacts cc, const double4* x, ContactState cs) {
    if (ns == 0) return;
    k_chain_dot<<<ns, 32 * kWarps, 0, st>>>(ns, slot_vtx, Kcol, colptr, chain_off, chain_rows, y, dxt, cc, x, cs);
}

// ----------------------------------------------------------------------------
// active contact vertices of this iteration (any incident row with theta != 0), in
// ascending slot order, and the active block G_A of the Delassus Gram.  These depend only
// on theta, so they run in a graph branch beside the RHS gather and K-pass 1.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_active(int ns, CrContacts cc, const int32_t* __restrict__ scp,
                                                 const int32_t* __restrict__ sci, ContactState cs, CrActive act) {
    __shared__ int wsum[32];
    __shared__ int base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int b0 = 0; b0 < ns; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        bool on = false;
        int only = -1;
        if (b < ns) {
            only = cc.c1[b];
            if (only >= 0) {
                on = cs.theta[3 * only] != 0.0 || cs.theta[3 * only + 1] != 0.0 || cs.theta[3 * only + 2] != 0.0;
            } else {
                for (int q = scp[b]; q < scp[b + 1] && !on; ++q) {
                    const int c = sci[q];
                    on = cs.theta[3 * c] != 0.0 || cs.theta[3 * c + 1] != 0.0 || cs.theta[3 * c + 2] != 0.0;
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int q = 0; q < wid; ++q) off += wsum[q];
        off += __popc(bal & ((1u << lane) - 1u));
        if (b < ns) {
            act.apos[b] = on ? off : -1;
            if (on) {
                act.aidx[off] = b;
                act.acon[off] = only;
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
    if (threadIdx.x == 0) act.na[0] = base;
}

__global__ void __launch_bounds__(256) k_gather_ga(int ns, const double* __restrict__ G, CrActive act,
                                                   double* __restrict__ GA) {
    const int na = act.na[0];
    const int i = blockIdx.x;
    if (i >= na) return;
    const size_t row = (size_t)act.aidx[i] * ns;
    for (int j = threadIdx.x; j < na; j += blockDim.x) GA[(size_t)i * na + j] = G[row + act.aidx[j]];
}

void launch_active(cudaStream_t st, int ns, CrContacts cc, const int32_t* scp, const int32_t* sci, ContactState cs,
                   CrActive act, const double* G, double* GA) {
    if (ns == 0) return;
    k_active<<<1, 1024, 0, st>>>(ns, cc, scp, sci, cs, act);
    k_gather_ga<<<ns, 256, 0, st>>>(ns, G, act, GA);
}

// per-contact-set: chain rows of every slot (walk panel runs) + row flags
__global__ void k_chain_rows(int ns, const int32_t* __restrict__ slot_vtx, const int32_t* __restrict__ chain_off,
                             const int32_t* __restrict__ parent, const int32_t* __restrict__ ptop,
                             int32_t* __restrict__ chain_rows, uint8_t* __restrict__ flag) {
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    int pos = chain_off[s];
    for (int i = slot_vtx[s]; i >= 0;) {
        const int top = ptop[i];
        const int len = top - i + 1;
        for (int o = lane; o < len; o += 32) {
            chain_rows[pos + o] = i + o;
            flag[i + o] = 1;
        }
        pos += len;
        i = parent[top];
    }
}

void launch_chain_rows(cudaStream_t st, int ns, const int32_t* slot_vtx, const int32_t* chain_off,
                       const int32_t* parent, const int32_t* ptop, int32_t* chain_rows, uint8_t* flag) {
    if (ns == 0) return;
    k_chain_rows<<<(ns + 7) / 8, 256, 0, st>>>(ns, slot_vtx, chain_off, parent, ptop, chain_rows, flag);
}

// rows on any chain, with the slot range in their subtree [first(i), i] and an
// offset into the compact copy Zc of K[i][a_s], s in [s0, s1)
__global__ void k_ulist(int n_f, int ns, const uint8_t* __restrict__ flag, const int32_t* __restrict__ slot_vtx,
                        const int2* __restrict__ meta, int* __restrict__ ucount, int4* __restrict__ ulist) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_f || !flag[i]) return;
    const int f = meta[i].y;
    int lo = 0, hi = ns;
    while (lo < hi) { int m = (lo + hi) >> 1; if (slot_vtx[m] < f) lo = m + 1; else hi = m; }
    const int s0 = lo;
    hi = ns;
    while (lo < hi) { int m = (lo + hi) >> 1; if (slot_vtx[m] <= i) lo = m + 1; else hi = m; }
    // list order and offsets are arbitrary but each row's values stay contiguous
    const int idx = atomicAdd(&ucount[0], 1);
    const int off = atomicAdd(&ucount[1], lo - s0);
    ulist[idx] = make_int4(i, s0, lo, off);
}

// Zc[off + s - s0] = K[i][a_s]  (one warp per listed row)
__global__ void k_zfill(const int* __restrict__ ucount, const int4* __restrict__ ulist,
                        const int32_t* __restrict__ slot_vtx, const float* __restrict__ Krow,
                        const int2* __restrict__ meta, float* __restrict__ Zc) {
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int cnt = ucount[0];
    for (int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += nw) {
        const int4 u = ulist[e];
        const float* row = Krow + meta[u.x].x;
        for (int s = u.y + lane; s < u.z; s += 32) Zc[u.w + s - u.y] = row[slot_vtx[s]];
    }
}

void launch_ulist(cudaStream_t st, int n_f, int ns, const uint8_t* flag, const int32_t* slot_vtx,
                  const int2* meta, int* ucount, int4* ulist, const float* Krow, float* Zc) {
    if (ns == 0) return;
    k_ulist<<<(n_f + 255) / 256, 256, 0, st>>>(n_f, ns, flag, slot_vtx, meta, ucount, ulist);
    k_zfill<<<148 * 4, 256, 0, st>>>(ucount, ulist, slot_vtx, Krow, meta, Zc);
}

// ----------------------------------------------------------------------------
// scatter (P:L956 correction, delta form): y_i += sum_{s0 <= s < s1} K[i][a_s] wz_s
// for the rows i on the contact vertices' chains (warp per row, grid-stride)
// ----------------------------------------------------------------------------
__global__ void k_scatter(const int* __restrict__ ucount, const int4* __restrict__ ulist,
                          const float* __restrict__ Zc, const double* __restrict__ wz, float4* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int cnt = ucount[0];
    for (int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < cnt; e += nw) {
        const int4 u = ulist[e];
        const float* zr = Zc + u.w - u.y;   // zr[s] = K[i][a_s]
        double a0 = 0, a1 = 0, a2 = 0;
        for (int s0 = u.y; s0 < u.z; s0 += 128) {   // 4 independent loads in flight per lane
            double kv[4], w0[4], w1[4], w2[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int sq = s0 + 32 * q + lane;
                const bool ok = sq < u.z;
                const int iq = ok ? sq : u.y;
                kv[q] = ok ? (double)__ldg(&zr[sq]) : 0.0;
                w0[q] = __ldg(&wz[3 * iq]);
                w1[q] = __ldg(&wz[3 * iq + 1]);
                w2[q] = __ldg(&wz[3 * iq + 2]);
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
        if (lane == 0) {
            const float4 yi = y[u.x];
            y[u.x] = make_float4((float)(yi.x + a0), (float)(yi.y + a1), (float)(yi.z + a2), yi.w);
        }
    }
}

void launch_scatter(cudaStream_t st, int max_rows, const int* ucount, const int4* ulist, const float* Zc,
                    const double* wz, float4* y) {
    k_scatter<<<(max_rows + 7) / 8, 256, 0, st>>>(ucount, ulist, Zc, wz, y);
}

// ----------------------------------------------------------------------------
// Delassus Gram G = K[:,Vc]^T K[:,Vc] (P:L858 via the sparse inverse):
// G_st = sum over common ancestors i of K[i][a_s] K[i][a_t] = sum over depths
// d <= depth(lca(a_s, a_t)) of Z[d][s] Z[d][t], Z[d][s] = Kcol[colptr_s + depth_s - d].
// 32x32 tiles of slot pairs, depth staged in chunks of 32 levels.
// ----------------------------------------------------------------------------

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

__global__ void __launch_bounds__(256) k_delassus(int ns, const int32_t* __restrict__ slot_vtx,
                                                  const float* __restrict__ Kcol, const int64_t* __restrict__ colptr,
                                                  const int32_t* __restrict__ depth, const int32_t* __restrict__ parent,
                                                  const int32_t* __restrict__ ptop, double* __restrict__ G) {
    // tile (bs, bt) with bt >= bs from a linear triangular index
    const int tiles = (ns + 31) / 32;
    int idx = blockIdx.x, bs = 0;
    while (idx >= tiles - bs) { idx -= tiles - bs; ++bs; }
    const int bt = bs + idx;
    __shared__ float Zs[2][32][33], Zt[2][32][33];
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
    // thread owns pairs (ls, lt0..lt0+3)
    const int ls = tid >> 3, lt0 = (tid & 7) * 4;
    const int s = bs * 32 + ls;
    int dl[4];
    int maxd = -1;
    for (int q = 0; q < 4; ++q) {
        const int t = bt * 32 + lt0 + q;
        dl[q] = (s < ns && t < ns) ? lca_depth(slot_vtx[s], slot_vtx[t], parent, ptop, depth) : -1;
        maxd = max(maxd, dl[q]);
    }
    atomicMax(&smax, maxd);
    __syncthreads();
    const int D = smax;
    // staging: each thread loads 4 (slot, depth) entries of each block per 32-level chunk
    float rs[4], rt[4];
    auto fetch = [&](int d0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + 256 * u;
            const int sl = e >> 5, dd = e & 31, d = d0 + dd;
            rs[u] = (ds_[sl] >= d) ? __ldg(&Kcol[cs_[sl] + ds_[sl] - d]) : 0.f;
            rt[u] = (dt_[sl] >= d) ? __ldg(&Kcol[ct_[sl] + dt_[sl] - d]) : 0.f;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + 256 * u;
            Zs[buf][e & 31][e >> 5] = rs[u];
            Zt[buf][e & 31][e >> 5] = rt[u];
        }
    };
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (D >= 0) fetch(0);
    int buf = 0;
    for (int d0 = 0; d0 <= D; d0 += 32) {
        stash(buf);
        __syncthreads();
        if (d0 + 32 <= D) fetch(d0 + 32);   // next chunk in flight while this one is consumed
#pragma unroll 8
        for (int dd = 0; dd < 32; ++dd) {
            const int d = d0 + dd;
            const float zs = Zs[buf][dd][ls];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (d <= dl[q]) acc[q] = fmaf(zs, Zt[buf][dd][lt0 + q], acc[q]);
        }
        buf ^= 1;
    }
    for (int q = 0; q < 4; ++q) {
        const int t = bt * 32 + lt0 + q;
        if (s < ns && t < ns) {
            G[(size_t)s * ns + t] = (double)acc[q];
            G[(size_t)t * ns + s] = (double)acc[q];
        }
    }
}

void launch_delassus(cudaStream_t st, int ns, const int32_t* slot_vtx, const float* Kcol,
                     const int64_t* colptr, const int32_t* depth, const int32_t* parent,
                     const int32_t* ptop, double* G) {
    if (ns == 0) return;
    int tiles = (ns + 31) / 32;
    int ntri = tiles * (tiles + 1) / 2;
    k_delassus<<<ntri, 256, 0, st>>>(ns, slot_vtx, Kcol, colptr, depth, parent, ptop, G);
}

// D_jj = sum_{a,b in j} w_a w_b G_ab (unit directions; reading A18)
__global__ void k_djj(int nc, int ns, DContact* C, const double* __restrict__ G) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    DContact& ct = C[c];
    double d = 0.0;
    for (int p = 0; p < ct.nv; ++p)
        for (int q = 0; q < ct.nv; ++q) d += ct.w[p] * ct.w[q] * G[(size_t)ct.slot[p] * ns + ct.slot[q]];
    ct.Djj = d;
}

void launch_djj(cudaStream_t st, int nc, int ns, DContact* c, const double* G) {
    if (nc == 0) return;
    k_djj<<<(nc + 127) / 128, 128, 0, st>>>(nc, ns, c, G);
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

struct CrLayout {
    int m, nc, ns;
    size_t r, th, cd, c9, s0, W, q, aidx, apos, acon, red, mbar, gA, total;
    __host__ __device__ CrLayout(int nc_, int ns_) : m(3 * nc_), nc(nc_), ns(ns_) {
        size_t o = 0;
        auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~size_t(15); return at; };
        r = take(8 * (size_t)m);
        th = take(4 * (size_t)m); cd = take(4 * (size_t)m);
        c9 = take(4 * 9 * (size_t)nc); s0 = take(4 * (size_t)nc);
        W = take(8 * 3 * (size_t)ns); q = take(8 * 2 * 3 * (size_t)ns);
        aidx = take(4 * (size_t)ns); apos = take(4 * (size_t)ns); acon = take(4 * (size_t)ns);
        red = take(8 * 2 * 3 * (kCrThreads / 32));   // double-buffered 3 doubles per warp
        mbar = take(32);                              // two exchange mbarriers (one per q buffer)
        gA = o;
        total = o;
    }
};

__device__ unsigned long long g_cr_clock[32];   // phase timestamps (ns) of the last CR call, rank 0
__device__ __forceinline__ void cr_stamp(int i) {
    if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_cr_clock[i] = t;
    }
}

struct CrCtx {
    double *r, *W, *q, *red, *gA;
    float *th, *cd, *c9;
    int *s0, *aidx, *apos, *acon;
    int na, ns, i0, i1, gA_smem;
    unsigned mbar;         // shared-window address of the 2 exchange mbarriers
    unsigned par0, par1;   // phase parity of each barrier
    int stamp;             // >= 0: fine-grained phase stamps of this apply at g_cr_clock[stamp..]
    const double* GAg;     // G_A in global memory (fallback when this CTA's rows do not fit)
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

// Ar = S r for this thread's rows (registers); r is read from shared memory
template <int kRpt>
__device__ __forceinline__ void cr_apply(cg::cluster_group& cl, CrCtx& X, int m, const DContact* __restrict__ C,
                                         const int32_t* __restrict__ scp, const int32_t* __restrict__ sci,
                                         const float* __restrict__ scw, int buf, double (&Ar)[kRpt]) {
    const int na = X.na;
    double* qb = X.q + (size_t)buf * 3 * X.ns;   // SoA: q0 | q1 | q2
    const unsigned bar = X.mbar + 8u * (unsigned)buf;
    if (threadIdx.x == 0 && na > 0)   // this phase expects 24 bytes per row of G_A from the peers
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
            for (int p = __ldg(&scp[b]); p < __ldg(&scp[b + 1]); ++p) {
                const int c = __ldg(&sci[p]);
                const double wt = __ldg(&scw[p]);
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
    for (int i = X.i0 + wid; i < X.i1; i += nw) {
        const double* g = X.gA_smem ? X.gA + (size_t)(i - X.i0) * na : X.GAg + (size_t)i * na;
        double d0 = 0, d1 = 0, d2 = 0;
        for (int b0 = 0; b0 < na; b0 += 128) {
            double gv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int bb = b0 + 32 * u + lane;
                gv[u] = bb < na ? (X.gA_smem ? g[bb] : __ldcg(&g[bb])) : 0.0;
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
        if (lane < kCluster) {
            // asynchronous stores of q_i into CTA `lane`, completing 24 tx bytes on its mbarrier
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
    if (threadIdx.x == 0 && na > 0) {   // wait until all na rows have landed here (acquire)
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
    if (buf) X.par1 ^= 1u; else X.par0 ^= 1u;
    __syncthreads();
    if (X.stamp >= 0) cr_stamp(X.stamp + 2);
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        const int j = min(threadIdx.x + kCrThreads * k, m - 1);   // rows >= m are padding (never used)
        const int c = j / 3, kk = j - 3 * c;
        const double th = (double)X.th[j];
        double acc = 0.0;
        if (th != 0.0) {
            const float* cc = X.c9 + 9 * c + 3 * kk;
            const int sl0 = X.s0[c];
            if (sl0 >= 0) {
                const int ip = X.apos[sl0];
                acc = (double)cc[0] * qb[ip] + (double)cc[1] * qb[na + ip] + (double)cc[2] * qb[2 * na + ip];
            } else {
                const DContact& ct = C[c];
                for (int p = 0; p < ct.nv; ++p) {
                    const int ip = X.apos[ct.slot[p]];
                    acc += ct.w[p] * ((double)cc[0] * qb[ip] + (double)cc[1] * qb[na + ip] +
                                      (double)cc[2] * qb[2 * na + ip]);
                }
            }
        }
        Ar[k] = th * acc + (double)X.cd[j] * X.r[j];
    }
}

template <int kRpt>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kCrThreads, 1)
    k_cr(Params P, const DContact* __restrict__ C, CrContacts cc, const int32_t* __restrict__ scp,
         const int32_t* __restrict__ sci, const float* __restrict__ scw, const double* __restrict__ GA,
         const double4* __restrict__ x, ContactState cs, CrActive act, int gA_cap) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const CrLayout L(P.nc, P.ns);
    cg::cluster_group cl = cg::this_cluster();
    const int nc = P.nc, ns = P.ns, m = 3 * nc;
    const double h = P.h;
    cr_stamp(0);
    CrCtx X;
    X.r = (double*)(smraw + L.r);
    X.th = (float*)(smraw + L.th);
    X.cd = (float*)(smraw + L.cd);
    X.c9 = (float*)(smraw + L.c9);
    X.s0 = (int*)(smraw + L.s0);
    X.W = (double*)(smraw + L.W);
    X.q = (double*)(smraw + L.q);
    X.aidx = (int*)(smraw + L.aidx);
    X.apos = (int*)(smraw + L.apos);
    X.acon = (int*)(smraw + L.acon);
    X.red = (double*)(smraw + L.red);
    X.gA = (double*)(smraw + L.gA);
    X.mbar = (unsigned)__cvta_generic_to_shared(smraw + L.mbar);
    X.par0 = X.par1 = 0u;
    X.stamp = -1;
    X.ns = ns;
    X.GAg = GA;
    // everything the prologue needs is precomputed (chain dot, k_active): plain loads only
    for (int e = threadIdx.x; e < 9 * nc; e += blockDim.x) cp_async4(&X.c9[e], &cc.c9[e], true);
    for (int c = threadIdx.x; c < nc; c += blockDim.x) cp_async4(&X.s0[c], &cc.s0[c], true);
    for (int b = threadIdx.x; b < ns; b += blockDim.x) {
        cp_async4(&X.aidx[b], &act.aidx[b], true);
        cp_async4(&X.apos[b], &act.apos[b], true);
        cp_async4(&X.acon[b], &act.acon[b], true);
    }
    cp_async_commit();
    const int na = act.na[0];
    X.na = na;
    {
        const int per = (na + kCluster - 1) / kCluster;
        X.i0 = min(na, (int)cl.block_rank() * per);
        X.i1 = min(na, X.i0 + per);
        X.gA_smem = (size_t)(X.i1 - X.i0) * na <= (size_t)gA_cap;
        if (X.gA_smem)
            for (int e = threadIdx.x; e < (X.i1 - X.i0) * na; e += blockDim.x)
                X.gA[e] = __ldcg(&GA[(size_t)X.i0 * na + e]);
    }
    double z[kRpt], p[kRpt], Ap[kRpt], Ar[kRpt];
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        z[k] = p[k] = Ap[k] = Ar[k] = 0.0;
        const int j = threadIdx.x + kCrThreads * k;
        if (j < m) {
            const int c = j / 3;
            const double th = cs.theta[j];
            double rho = cs.rho[j];
            const int v0 = __ldg(&cc.v0[c]);
            const bool viaSlot = v0 >= 0 && __ldg(&cc.c1[__ldg(&cc.s0[c])]) == c;
            if (!viaSlot) {   // rho of contacts the chain dot did not cover
                const int kk = j - 3 * c;
                const DContact& ct = C[c];
                double xs0 = 0.0, xs1 = 0.0, xs2 = 0.0;
                for (int q = 0; q < ct.nv; ++q) {
                    const double4 xa = x[ct.vtx[q]];
                    const int sl = ct.slot[q];
                    xs0 += ct.w[q] * (xa.x + cs.dxt[3 * sl]);
                    xs1 += ct.w[q] * (xa.y + cs.dxt[3 * sl + 1]);
                    xs2 += ct.w[q] * (xa.z + cs.dxt[3 * sl + 2]);
                }
                rho = cs.hvec[j] - th * (ct.c[kk][0] * xs0 + ct.c[kk][1] * xs1 + ct.c[kk][2] * xs2);
            }
            X.th[j] = (float)th;
            X.cd[j] = (float)cs.cdiag[j];
            X.r[j] = rho;
            p[k] = rho;
        }
    }
    cp_async_wait<0>();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(X.mbar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(X.mbar + 8u));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cl.sync();   // smem staged everywhere; every CTA's exchange mbarriers initialised
    cr_stamp(1);
    if (threadIdx.x == 0 && cl.block_rank() == 0) g_cr_clock[31] = g_cr_clock[0] + 1000ull * na;   // na (debug)
    double rr = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int k = 0; k < kRpt; ++k) rr = fma(p[k], p[k], rr);
    int rb = 0;   // reduction buffer
    block_sum3(rr, t1, t2, X.red + rb * 3 * (kCrThreads / 32));
    rb ^= 1;
    cr_stamp(2);
    if (rr > 0.0 && P.cr_iters > 0) {
        int buf = 0;
        cr_apply<kRpt>(cl, X, m, C, scp, sci, scw, buf, Ar);
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
            cr_apply<kRpt>(cl, X, m, C, scp, sci, scw, buf, Ar);
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
            ApAp = s2 + 2.0 * beta * s3 + beta * beta * ApAp;
#pragma unroll
            for (int k = 0; k < kRpt; ++k) {
                const int j = min(threadIdx.x + kCrThreads * k, m - 1);
                p[k] = X.r[j] + beta * p[k];
                Ap[k] = Ar[k] + beta * Ap[k];
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
    const int rank = cl.block_rank();
    const int rper = (m + kCluster - 1) / kCluster;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
        const int j = threadIdx.x + kCrThreads * k;
        if (j < m) {
            X.r[j] = z[k];
            if (j / rper == rank) cs.lam[j] += z[k] / (h * h);
        }
    }
    __syncthreads();
    cr_stamp(28);
    // wz_b = sum w theta z c  (for y += K H^T z), this CTA's slots
    const int sper = (ns + kCluster - 1) / kCluster;
    for (int b = rank * sper + threadIdx.x; b < min(ns, (rank + 1) * sper); b += blockDim.x) {
        double w0 = 0, w1 = 0, w2 = 0;
        const int only = __ldg(&cc.c1[b]);
        const int qa = only >= 0 ? 0 : scp[b], qb = only >= 0 ? 1 : scp[b + 1];
        for (int q = qa; q < qb; ++q) {
            const int c = only >= 0 ? only : sci[q];
            const double wt = only >= 0 ? 1.0 : (double)scw[q];
            const float* c9 = X.c9 + 9 * c;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double tv = wt * (double)X.th[3 * c + k] * X.r[3 * c + k];
                w0 += tv * (double)c9[3 * k];
                w1 += tv * (double)c9[3 * k + 1];
                w2 += tv * (double)c9[3 * k + 2];
            }
        }
        cs.wz[3 * b] = w0;
        cs.wz[3 * b + 1] = w1;
        cs.wz[3 * b + 2] = w2;
    }
    if (threadIdx.x == 0 && rank == 0) cs.cr_res[0] = sqrt(res);
    cr_stamp(21);
    // no trailing cluster barrier: after its last exchange wait no CTA touches a peer's shared memory
}

int read_cr_clock(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_cr_clock, sizeof(unsigned long long) * 32);
}

size_t cr_smem_bytes(int nc, int ns) { return CrLayout(nc, ns).total; }

int launch_cr(cudaStream_t st, const Params& P, const DContact* c, CrContacts cc, const int32_t* scp,
              const int32_t* sci, const float* scw, const double* GA, const double4* x, ContactState cs,
              CrActive act) {
    if (P.nc == 0) return 0;
    static bool attr = false;
    if (!attr) {
        void* fns[kRptMax] = {(void*)k_cr<1>, (void*)k_cr<2>, (void*)k_cr<3>, (void*)k_cr<4>, (void*)k_cr<5>, (void*)k_cr<6>};
        for (void* f : fns) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return (int)e;
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCrMaxSmem);
            if (e != cudaSuccess) return (int)e;
        }
        attr = true;
    }
    const size_t base = cr_smem_bytes(P.nc, P.ns);
    const int cap = (int)((kCrMaxSmem - base) / sizeof(double));
    const int rpt = (3 * P.nc + kCrThreads - 1) / kCrThreads;
#define CRL(R) k_cr<R><<<kCluster, kCrThreads, kCrMaxSmem, st>>>(P, c, cc, scp, sci, scw, GA, x, cs, act, cap)
    switch (rpt) {
        case 1: CRL(1); break;
        case 2: CRL(2); break;
        case 3: CRL(3); break;
        case 4: CRL(4); break;
        case 5: CRL(5); break;
        default: CRL(6); break;
    }
#undef CRL
    return (int)cudaGetLastError();
}

}  // namespace simdev
