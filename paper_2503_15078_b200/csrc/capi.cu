// C ABI (include/sim.h) and the iteration driver: one CUDA Graph per frame.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sim.h"
#include "host.hpp"
#include "kernels.cuh"

using namespace simdev;

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            return fail(e_ == cudaErrorMemoryAllocation ? SIM_E_OOM : SIM_E_CUDA, "%s: %s (%s:%d)", #call, \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                          \
        }                                                                                     \
    } while (0)

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t alloc(size_t cnt) {
        release();
        n = cnt;
        if (cnt == 0) return cudaSuccess;
        return cudaMalloc(&p, cnt * sizeof(T));
    }
    cudaError_t upload(const T* h, size_t cnt, cudaStream_t st) {
        if (cnt == 0) return cudaSuccess;
        return cudaMemcpyAsync(p, h, cnt * sizeof(T), cudaMemcpyHostToDevice, st);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct sim_handle {
    bool host_only = false;
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;            // fork branch inside the frame graph
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    bool own_stream = false;
    int state = 0;   // 0 created, 1 built
    // host copies
    int n_v = 0, n_t = 0, n_f = 0;
    std::vector<double> X;
    std::vector<int32_t> T;
    std::vector<uint8_t> fixed;
    sim_material mat{};
    double h = 0, mu_l = 0, lam_l = 0, kproj = 0;
    simhost::RestData rd;
    std::vector<int32_t> int2orig, orig2int;
    simhost::Inverse K;
    simhost::WorkLists wl;
    std::vector<float> T1h, T2h;
    int64_t nnzL = 0;
    double build_seconds = 0;
    double vpin[3] = {0, 0, 0};
    // device: state
    DBuf<double4> x, xt, v, s;
    DBuf<double> M;
    DBuf<int4> tet;
    DBuf<float> Bm, hw2;
    DBuf<float4> fc, u, y;
    DBuf<int32_t> adjp, adj;
    // device: K
    DBuf<float> Krow, Kcol, T1, T2;   // K row/column-major + the two passes' tile streams
    DBuf<int64_t> colptr;
    DBuf<int32_t> cb, depth, parent, ptop, cover;
    DBuf<int2> meta;                 // {rowptr[i] - first[i], first[i]}
    DBuf<P1Item> p1;
    DBuf<P1Block> p1b;
    DBuf<P2Block> p2b;
    DBuf<double> part1;
    DBuf<int> counters;
    // contacts
    int nc = 0, ns = 0, row_lo = 0;
    std::vector<DContact> hc;
    std::vector<int32_t> slot_vtx_h;
    DBuf<DContact> dc;
    DBuf<float> cc9;
    DBuf<int32_t> cs0, cv0, cc1;
    DBuf<int32_t> slot_vtx, scp, sci, vcp, vci;
    DBuf<float> scw, vcw;
    DBuf<double> G, GA;   // Delassus Gram and the CR's active-block scratch
    DBuf<double> lam, theta, cdiag, hvec, hl, dxt, wz, phi_abs, cr_res, rho;
    DBuf<int> act_na, act_idx, act_pos, act_con;   // CR active set (k_active)
    DBuf<int32_t> chain_off, chain_rows;
    DBuf<uint8_t> flag;
    DBuf<int> ucount;
    DBuf<int4> ulist;
    DBuf<float> Zc;
    int contact_gen = 0;
    // graph
    cudaGraphExec_t gexec = nullptr;
    int g_iters = -1, g_nc = -1, g_ns = -1, g_prof = -1, g_gen = -1;
    // in-graph kernel timing (event record nodes between kernels)
    int profiling = 0;
    std::vector<cudaEvent_t> pev;
    std::vector<int> pkind;   // kind of the kernel that follows event i
    int kernels_per_frame = 0;
    int64_t frames_done = 0;
    int64_t h2d_contact_bytes = 0;   // bytes uploaded by the last sim_set_contacts
    // pinned staging for asynchronous sim_set_contacts uploads (reused once the last copy is done)
    unsigned char* stage = nullptr;
    size_t stage_cap = 0, stage_used = 0;
    cudaEvent_t stage_free = nullptr;
    double set_contacts_host_us = 0;
};

// copy n elements of src into the pinned staging area and enqueue the H2D copy to dst
template <class T>
static cudaError_t stage_upload(sim_handle* H, T* dst, const T* src, size_t n) {
    if (n == 0) return cudaSuccess;
    const size_t bytes = n * sizeof(T);
    const size_t at = (H->stage_used + 15) & ~size_t(15);
    if (at + bytes > H->stage_cap) return cudaErrorMemoryAllocation;   // caller sized the area
    memcpy(H->stage + at, src, bytes);
    H->stage_used = at + bytes;
    return cudaMemcpyAsync(dst, H->stage + at, bytes, cudaMemcpyHostToDevice, H->stream);
}

// ---------------------------------------------------------------------------
static int validate_create(const sim_mesh* m, const sim_material* mat, double h) {
    if (!m || !mat) return fail(SIM_E_INVALID, "null mesh or material");
    if (m->n_vertices <= 0 || m->n_tets <= 0 || !m->rest_positions || !m->tets)
        return fail(SIM_E_INVALID, "empty mesh or null arrays");
    if (!(h > 0) || !std::isfinite(h)) return fail(SIM_E_INVALID, "h must be > 0");
    if (mat->model < 0 || mat->model > 2) return fail(SIM_E_INVALID, "unknown material model %d", mat->model);
    if (!(mat->density > 0) || !(mat->youngs > 0) || !std::isfinite(mat->youngs))
        return fail(SIM_E_INVALID, "density and youngs must be > 0");
    if (!(mat->poisson >= 0 && mat->poisson < 0.5)) return fail(SIM_E_INVALID, "poisson must be in [0, 0.5)");
    if (mat->proj_stiffness < 0) return fail(SIM_E_INVALID, "proj_stiffness must be >= 0");
    for (int d = 0; d < 3; ++d)
        if (!std::isfinite(mat->gravity[d])) return fail(SIM_E_INVALID, "gravity not finite");
    for (int64_t i = 0; i < 3LL * m->n_vertices; ++i)
        if (!std::isfinite(m->rest_positions[i])) return fail(SIM_E_INVALID, "rest position %lld not finite", (long long)i);
    for (int64_t i = 0; i < 4LL * m->n_tets; ++i)
        if (m->tets[i] < 0 || m->tets[i] >= m->n_vertices) return fail(SIM_E_INVALID, "tet index out of range");
    return SIM_OK;
}

static int create_common(const sim_mesh* m, const sim_material* mat, double h, sim_handle** out, bool host_only) {
    if (!out) return fail(SIM_E_INVALID, "null out");
    *out = nullptr;
    int rc = validate_create(m, mat, h);
    if (rc) return rc;
    sim_handle* H = new (std::nothrow) sim_handle();
    if (!H) return fail(SIM_E_OOM, "host allocation");
    H->host_only = host_only;
    H->n_v = m->n_vertices;
    H->n_t = m->n_tets;
    H->X.assign(m->rest_positions, m->rest_positions + 3 * (size_t)H->n_v);
    H->T.assign(m->tets, m->tets + 4 * (size_t)H->n_t);
    H->fixed.assign(H->n_v, 0);
    if (m->fixed)
        for (int i = 0; i < H->n_v; ++i) H->fixed[i] = m->fixed[i] ? 1 : 0;
    H->mat = *mat;
    if (H->mat.cr_iterations <= 0) H->mat.cr_iterations = 10;
    H->h = h;
    H->mu_l = mat->youngs / (2.0 * (1.0 + mat->poisson));
    H->lam_l = mat->youngs * mat->poisson / ((1.0 + mat->poisson) * (1.0 - 2.0 * mat->poisson));
    H->kproj = mat->proj_stiffness > 0 ? mat->proj_stiffness : 2.0 * H->mu_l;
    int bad = -1;
    std::string msg = simhost::rest_data(H->n_v, H->n_t, H->X.data(), H->T.data(), mat->density, H->kproj, H->rd, bad);
    if (!msg.empty()) {
        delete H;
        return fail(SIM_E_DEGENERATE, "%s", msg.c_str());
    }
    int nf = 0;
    for (int i = 0; i < H->n_v; ++i) nf += !H->fixed[i];
    if (nf == 0) {
        delete H;
        return fail(SIM_E_INVALID, "all vertices pinned");
    }
    if (!host_only) {
        cudaError_t e = cudaGetDevice(&H->device);
        if (e == cudaSuccess) {
            int ndev = 0;
            e = cudaGetDeviceCount(&ndev);
            if (e == cudaSuccess && ndev == 0) e = cudaErrorNoDevice;
        }
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&H->aux, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&H->fork_ev, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&H->join_ev, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            delete H;
            return fail(SIM_E_CUDA, "no usable CUDA device: %s", cudaGetErrorString(e));
        }
        H->own_stream = true;
    }
    *out = H;
    return SIM_OK;
}

extern "C" int sim_create(const sim_mesh* m, const sim_material* mat, double h, sim_handle** out) {
    return create_common(m, mat, h, out, false);
}
extern "C" int sim_create_host(const sim_mesh* m, const sim_material* mat, double h, sim_handle** out) {
    return create_common(m, mat, h, out, true);
}

extern "C" const char* sim_last_error(void) { return g_err.c_str(); }

extern "C" void sim_destroy(sim_handle* H) {
    if (!H) return;
    if (!H->host_only) {
        if (H->stream) cudaStreamSynchronize(H->stream);
        if (H->gexec) cudaGraphExecDestroy(H->gexec);
        H->x.release(); H->xt.release(); H->v.release(); H->s.release(); H->M.release();
        H->tet.release(); H->Bm.release(); H->hw2.release(); H->fc.release(); H->u.release(); H->y.release();
        H->adjp.release(); H->adj.release(); H->Krow.release(); H->Kcol.release(); H->T1.release(); H->T2.release(); H->meta.release();
        H->colptr.release(); H->cb.release(); H->cover.release(); H->depth.release(); H->parent.release();
        H->ptop.release(); H->p1.release(); H->p1b.release(); H->p2b.release();
        H->part1.release(); H->counters.release();
        H->chain_off.release(); H->chain_rows.release(); H->flag.release(); H->ucount.release(); H->ulist.release(); H->Zc.release();
        H->dc.release(); H->cc9.release(); H->cs0.release(); H->cv0.release(); H->cc1.release(); H->slot_vtx.release(); H->scp.release(); H->sci.release(); H->vcp.release();
        H->vci.release(); H->scw.release(); H->vcw.release(); H->G.release(); H->GA.release(); H->lam.release();
        H->theta.release(); H->cdiag.release(); H->hvec.release(); H->hl.release(); H->dxt.release();
        H->wz.release(); H->phi_abs.release(); H->cr_res.release(); H->rho.release();
        H->act_na.release(); H->act_idx.release(); H->act_pos.release(); H->act_con.release();
        for (auto e : H->pev) cudaEventDestroy(e);
        if (H->stage_free) cudaEventDestroy(H->stage_free);
        if (H->fork_ev) cudaEventDestroy(H->fork_ev);
        if (H->join_ev) cudaEventDestroy(H->join_ev);
        if (H->aux) cudaStreamDestroy(H->aux);
        if (H->stage) cudaFreeHost(H->stage);
        if (H->own_stream && H->stream) cudaStreamDestroy(H->stream);
    }
    delete H;
}

extern "C" int sim_set_stream(sim_handle* H, void* st) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->host_only) return fail(SIM_E_STATE, "host-only handle");
    CK(cudaStreamSynchronize(H->stream));
    if (H->own_stream) cudaStreamDestroy(H->stream);
    H->stream = (cudaStream_t)st;
    H->own_stream = false;
    if (H->gexec) {
        cudaGraphExecDestroy(H->gexec);
        H->gexec = nullptr;
    }
    return SIM_OK;
}

// ---------------------------------------------------------------------------
// sim_build_sparse_inverse
// ---------------------------------------------------------------------------
static int upload_all(sim_handle* H) {
    cudaStream_t st = H->stream;
    const int nv = H->n_v, nt = H->n_t, nf = H->n_f;
    // state: rest, v = 0
    std::vector<double4> xs(nv), zero(nv, make_double4(0, 0, 0, 0));
    for (int i = 0; i < nv; ++i) {
        int o = H->int2orig[i];
        xs[i] = make_double4(H->X[3 * o], H->X[3 * o + 1], H->X[3 * o + 2], 0.0);
    }
    CK(H->x.alloc(nv)); CK(H->xt.alloc(nv)); CK(H->v.alloc(nv)); CK(H->s.alloc(nv));
    CK(H->x.upload(xs.data(), nv, st));
    CK(H->xt.upload(xs.data(), nv, st));
    CK(H->v.upload(zero.data(), nv, st));
    CK(H->s.upload(xs.data(), nv, st));
    std::vector<double> M(nf);
    for (int i = 0; i < nf; ++i) M[i] = H->rd.mass[H->int2orig[i]];
    CK(H->M.alloc(nf));
    CK(H->M.upload(M.data(), nf, st));
    // tets (original order), SoA Bm, h^2 w
    std::vector<int4> tv(nt);
    std::vector<float> Bm((size_t)9 * nt), hw(nt);
    for (int t = 0; t < nt; ++t) {
        const int32_t* q = &H->T[4 * (size_t)t];
        tv[t] = make_int4(H->orig2int[q[0]], H->orig2int[q[1]], H->orig2int[q[2]], H->orig2int[q[3]]);
        for (int e = 0; e < 9; ++e) Bm[(size_t)e * nt + t] = (float)H->rd.Bm[9 * (size_t)t + e];
        hw[t] = (float)(H->h * H->h * H->rd.w[t]);
    }
    CK(H->tet.alloc(nt)); CK(H->tet.upload(tv.data(), nt, st));
    CK(H->Bm.alloc((size_t)9 * nt)); CK(H->Bm.upload(Bm.data(), (size_t)9 * nt, st));
    CK(H->hw2.alloc(nt)); CK(H->hw2.upload(hw.data(), nt, st));
    CK(H->fc.alloc((size_t)4 * nt));
    CK(H->u.alloc(nf)); CK(H->y.alloc(nf));
    // vertex -> (tet, corner) adjacency for free vertices, ascending tet order
    std::vector<int32_t> adjp(nf + 1, 0), adj;
    for (int t = 0; t < nt; ++t)
        for (int c = 0; c < 4; ++c) {
            int a = tv[t].x;
            if (c == 1) a = tv[t].y;
            if (c == 2) a = tv[t].z;
            if (c == 3) a = tv[t].w;
            if (a < nf) adjp[a + 1]++;
        }
    for (int i = 0; i < nf; ++i) adjp[i + 1] += adjp[i];
    adj.resize(adjp[nf]);
    std::vector<int32_t> fill(adjp.begin(), adjp.end() - 1);
    for (int t = 0; t < nt; ++t) {
        int q[4] = {tv[t].x, tv[t].y, tv[t].z, tv[t].w};
        for (int c = 0; c < 4; ++c)
            if (q[c] < nf) adj[fill[q[c]]++] = 4 * t + c;
    }
    CK(H->adjp.alloc(nf + 1)); CK(H->adjp.upload(adjp.data(), nf + 1, st));
    CK(H->adj.alloc(adj.size())); CK(H->adj.upload(adj.data(), adj.size(), st));
    // K
    const simhost::Inverse& K = H->K;
    CK(H->Krow.alloc(K.nnz)); CK(H->Krow.upload(K.Krow.data(), K.nnz, st));
    CK(H->Kcol.alloc(K.nnz)); CK(H->Kcol.upload(K.Kcol.data(), K.nnz, st));
    CK(H->T1.alloc(H->T1h.size())); CK(H->T1.upload(H->T1h.data(), H->T1h.size(), st));
    CK(H->T2.alloc(H->T2h.size())); CK(H->T2.upload(H->T2h.data(), H->T2h.size(), st));
    std::vector<int32_t> cb(nf);
    std::vector<int2> meta(nf);
    for (int j = 0; j < nf; ++j) {
        cb[j] = (int32_t)(K.colptr[j] + K.depth[j]);
        meta[j] = make_int2((int32_t)(K.rowptr[j] - K.first[j]), K.first[j]);
    }
    CK(H->colptr.alloc(nf + 1)); CK(H->colptr.upload(K.colptr.data(), nf + 1, st));
    CK(H->cb.alloc(nf)); CK(H->cb.upload(cb.data(), nf, st));
    CK(H->meta.alloc(nf)); CK(H->meta.upload(meta.data(), nf, st));
    CK(H->depth.alloc(nf)); CK(H->depth.upload(K.depth.data(), nf, st));
    CK(H->parent.alloc(nf)); CK(H->parent.upload(K.parent.data(), nf, st));
    CK(H->ptop.alloc(nf)); CK(H->ptop.upload(K.ptop.data(), nf, st));
    const simhost::WorkLists& W = H->wl;
    CK(H->p1.alloc(W.p1.size())); CK(H->p1.upload(W.p1.data(), W.p1.size(), st));
    CK(H->p1b.alloc(W.p1b.size())); CK(H->p1b.upload(W.p1b.data(), W.p1b.size(), st));
    CK(H->p2b.alloc(W.p2b.size())); CK(H->p2b.upload(W.p2b.data(), W.p2b.size(), st));
    CK(H->cover.alloc(W.cover.size())); CK(H->cover.upload(W.cover.data(), W.cover.size(), st));
    CK(H->part1.alloc((size_t)std::max(1, W.p1_parts) * 32 * 3));
    size_t ncnt = W.p1b.size();
    CK(H->counters.alloc(ncnt));
    CK(cudaMemsetAsync(H->counters.p, 0, ncnt * sizeof(int), st));
    // contact buffers at capacity (pointers stay fixed for graph reuse)
    CK(H->dc.alloc(kMaxContacts));
    CK(H->cc9.alloc(9 * kMaxContacts)); CK(H->cs0.alloc(kMaxContacts)); CK(H->cv0.alloc(kMaxContacts));
    CK(H->cc1.alloc(kMaxSlots));
    CK(H->slot_vtx.alloc(kMaxSlots));
    CK(H->scp.alloc(kMaxSlots + 1));
    CK(H->sci.alloc(4 * kMaxContacts));
    CK(H->scw.alloc(4 * kMaxContacts));
    CK(H->vcp.alloc(nf + 1));
    CK(H->vci.alloc(4 * kMaxContacts));
    CK(H->vcw.alloc(4 * kMaxContacts));
    CK(H->G.alloc((size_t)kMaxSlots * kMaxSlots));
    CK(H->GA.alloc((size_t)kMaxSlots * kMaxSlots));
    CK(H->lam.alloc(3 * kMaxContacts)); CK(H->theta.alloc(3 * kMaxContacts)); CK(H->cdiag.alloc(3 * kMaxContacts));
    CK(H->hvec.alloc(3 * kMaxContacts)); CK(H->hl.alloc(3 * kMaxContacts)); CK(H->dxt.alloc(3 * kMaxSlots));
    CK(H->wz.alloc(3 * kMaxSlots)); CK(H->phi_abs.alloc(kMaxContacts)); CK(H->cr_res.alloc(1));
    CK(H->rho.alloc(3 * kMaxContacts)); CK(H->act_na.alloc(1)); CK(H->act_idx.alloc(kMaxSlots));
    CK(H->act_pos.alloc(kMaxSlots)); CK(H->act_con.alloc(kMaxSlots));
    CK(H->chain_off.alloc(kMaxSlots + 1)); CK(H->flag.alloc(nf)); CK(H->ucount.alloc(2)); CK(H->ulist.alloc(nf));
    CK(cudaMemsetAsync(H->ucount.p, 0, 2 * sizeof(int), st));
    CK(cudaMemsetAsync(H->lam.p, 0, 3 * kMaxContacts * sizeof(double), st));
    CK(cudaMemsetAsync(H->vcp.p, 0, (nf + 1) * sizeof(int32_t), st));
    CK(cudaMemsetAsync(H->cr_res.p, 0, sizeof(double), st));
    CK(cudaStreamSynchronize(st));
    return SIM_OK;
}

extern "C" int sim_build_sparse_inverse(sim_handle* H, double drop_tol) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 0) return fail(SIM_E_STATE, "sparse inverse already built");
    if (!(drop_tol >= 0) || !std::isfinite(drop_tol)) return fail(SIM_E_INVALID, "drop tolerance must be >= 0");
    auto t0 = std::chrono::steady_clock::now();
    const int nv = H->n_v;
    std::vector<int32_t> vid(nv, -1), freev;
    for (int i = 0; i < nv; ++i)
        if (!H->fixed[i]) {
            vid[i] = (int)freev.size();
            freev.push_back(i);
        }
    const int nf = (int)freev.size();
    simhost::Csr A = simhost::assemble_Av(nv, H->n_t, H->T.data(), H->rd, H->h, vid, nf);
    std::vector<double> coords(3 * (size_t)nf);
    for (int k = 0; k < nf; ++k)
        for (int d = 0; d < 3; ++d) coords[3 * k + d] = H->X[3 * (size_t)freev[k] + d];
    std::vector<int32_t> nd = simhost::nested_dissection(A, coords);
    simhost::Csr C = simhost::permute_sym(A, nd);
    std::vector<int32_t> par = simhost::etree(C);
    std::vector<int32_t> post = simhost::postorder(par);
    std::vector<int32_t> perm(nf);   // perm[new] = free-local old index
    for (int k = 0; k < nf; ++k) perm[k] = nd[post[k]];
    C = simhost::permute_sym(A, perm);
    par = simhost::etree(C);
    simhost::Factor F;
    if (!simhost::cholesky(C, par, F))
        return fail(SIM_E_NOT_SPD, "non-positive pivot at column %d", F.bad_col);
    H->nnzL = (int64_t)F.Lp[nf];
    int nthr = (int)std::max(1u, std::thread::hardware_concurrency());
    simhost::sparse_inverse(F, drop_tol, H->K, nthr);
    if (H->K.nnz >= (int64_t)INT32_MAX)
        return fail(SIM_E_LIMIT, "nnz(K) = %lld exceeds the int32 offset limit", (long long)H->K.nnz);
    simhost::build_worklists(H->K, H->wl, 1024);
    simhost::build_tiles(H->K, H->wl, H->T1h, H->T2h);
    H->n_f = nf;
    H->int2orig.assign(nv, -1);
    H->orig2int.assign(nv, -1);
    for (int k = 0; k < nf; ++k) H->int2orig[k] = freev[perm[k]];
    int q = nf;
    for (int i = 0; i < nv; ++i)
        if (H->fixed[i]) H->int2orig[q++] = i;
    for (int k = 0; k < nv; ++k) H->orig2int[H->int2orig[k]] = k;
    H->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!H->host_only) {
        int rc = upload_all(H);
        if (rc) return rc;
    }
    H->state = 1;
    return SIM_OK;
}

// ---------------------------------------------------------------------------
// contacts
// ---------------------------------------------------------------------------
static void gram_schmidt(const double n[3], double t1[3], double t2[3]) {
    int a = 0;
    for (int d = 1; d < 3; ++d)
        if (std::fabs(n[d]) < std::fabs(n[a])) a = d;
    double e[3] = {0, 0, 0};
    e[a] = 1.0;
    double dp = n[a];
    double w[3] = {e[0] - dp * n[0], e[1] - dp * n[1], e[2] - dp * n[2]};
    double l = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    for (int d = 0; d < 3; ++d) t1[d] = w[d] / l;
    t2[0] = n[1] * t1[2] - n[2] * t1[1];
    t2[1] = n[2] * t1[0] - n[0] * t1[2];
    t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

extern "C" int sim_set_contacts(sim_handle* H, const sim_contact* cs, int32_t n) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1) return fail(SIM_E_STATE, "build the sparse inverse first");
    if (H->host_only) return fail(SIM_E_STATE, "host-only handle");
    if (n < 0 || (n > 0 && !cs)) return fail(SIM_E_INVALID, "bad contact array");
    if (n > kMaxContacts) return fail(SIM_E_LIMIT, "at most %d contacts per handle", kMaxContacts);
    auto th0 = std::chrono::steady_clock::now();
    std::vector<DContact> hc(n);
    std::vector<int32_t> verts;
    for (int c = 0; c < n; ++c) {
        const sim_contact& s = cs[c];
        if (s.kind != 0 && s.kind != 1) return fail(SIM_E_INVALID, "contact %d: kind must be 0 or 1", c);
        if (s.n_verts < 1 || s.n_verts > 4) return fail(SIM_E_INVALID, "contact %d: 1..4 vertices", c);
        double nn = std::sqrt(s.normal[0] * s.normal[0] + s.normal[1] * s.normal[1] + s.normal[2] * s.normal[2]);
        if (!(std::fabs(nn - 1.0) < 1e-6)) return fail(SIM_E_INVALID, "contact %d: normal not unit", c);
        if (!(s.mu >= 0) || !std::isfinite(s.mu)) return fail(SIM_E_INVALID, "contact %d: mu must be >= 0", c);
        if (!(s.compliance >= 0)) return fail(SIM_E_INVALID, "contact %d: compliance must be >= 0", c);
        if (!std::isfinite(s.offset)) return fail(SIM_E_INVALID, "contact %d: offset not finite", c);
        DContact& d = hc[c];
        memset(&d, 0, sizeof d);
        d.kind = s.kind;
        d.nv = s.n_verts;
        for (int q = 0; q < s.n_verts; ++q) {
            if (s.verts[q] < 0 || s.verts[q] >= H->n_v) return fail(SIM_E_INVALID, "contact %d: vertex out of range", c);
            if (H->fixed[s.verts[q]]) return fail(SIM_E_INVALID, "contact %d: vertex %d is pinned", c, s.verts[q]);
            if (!std::isfinite(s.weights[q])) return fail(SIM_E_INVALID, "contact %d: weight not finite", c);
            d.vtx[q] = H->orig2int[s.verts[q]];
            d.w[q] = s.weights[q];
            verts.push_back(d.vtx[q]);
        }
        double t1[3], t2[3];
        bool zt = true;
        for (int k = 0; k < 3; ++k) zt = zt && s.tangent1[k] == 0.0 && s.tangent2[k] == 0.0;
        if (zt) {
            gram_schmidt(s.normal, t1, t2);
        } else {
            for (int k = 0; k < 3; ++k) { t1[k] = s.tangent1[k]; t2[k] = s.tangent2[k]; }
        }
        for (int k = 0; k < 3; ++k) {
            d.c[0][k] = s.normal[k] / nn;
            d.c[1][k] = s.kind == 1 ? 0.0 : t1[k];
            d.c[2][k] = s.kind == 1 ? 0.0 : t2[k];
        }
        d.dn = s.offset;
        d.df1 = s.kind == 1 ? 0.0 : t1[0] * s.obstacle_velocity[0] + t1[1] * s.obstacle_velocity[1] + t1[2] * s.obstacle_velocity[2];
        d.df2 = s.kind == 1 ? 0.0 : t2[0] * s.obstacle_velocity[0] + t2[1] * s.obstacle_velocity[1] + t2[2] * s.obstacle_velocity[2];
        d.mu = s.mu;
        d.e = s.compliance;
    }
    std::sort(verts.begin(), verts.end());
    verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
    if ((int)verts.size() > kMaxSlots) return fail(SIM_E_LIMIT, "at most %d contact vertices", kMaxSlots);
    if (cr_smem_bytes(n, (int)verts.size()) > kCrMaxSmem)
        return fail(SIM_E_LIMIT, "%d contacts on %d vertices exceed the CR cluster's shared memory (%zu > %zu B)", n,
                    (int)verts.size(), cr_smem_bytes(n, (int)verts.size()), kCrMaxSmem);
    const int ns = (int)verts.size();
    std::vector<int32_t> slot_of(H->n_f, -1);
    for (int s = 0; s < ns; ++s) slot_of[verts[s]] = s;
    // slot -> (contact, weight) and vertex -> (contact, weight) lists
    std::vector<std::vector<std::pair<int, float>>> sl(ns);
    for (int c = 0; c < n; ++c)
        for (int q = 0; q < hc[c].nv; ++q) {
            hc[c].slot[q] = slot_of[hc[c].vtx[q]];
            sl[hc[c].slot[q]].push_back({c, (float)hc[c].w[q]});
        }
    std::vector<int32_t> scp(ns + 1, 0), sci;
    std::vector<float> scw;
    for (int s = 0; s < ns; ++s) {
        for (auto& e : sl[s]) { sci.push_back(e.first); scw.push_back(e.second); }
        scp[s + 1] = (int)sci.size();
    }
    std::vector<int32_t> vcp(H->n_f + 1, 0);
    for (int s = 0; s < ns; ++s) vcp[verts[s] + 1] = scp[s + 1] - scp[s];
    for (int i = 0; i < H->n_f; ++i) vcp[i + 1] += vcp[i];
    cudaStream_t st = H->stream;
    // asynchronous uploads through pinned staging: wait only for the previous call's copies
    {
        const size_t need = n * sizeof(DContact) + 64 * (size_t)n + 32 * (size_t)ns + 16 * sci.size() +
                            4 * ((size_t)H->n_f + 1) + 1024;
        if (!H->stage_free) CK(cudaEventCreateWithFlags(&H->stage_free, cudaEventDisableTiming));
        CK(cudaEventSynchronize(H->stage_free));
        if (need > H->stage_cap) {
            if (H->stage) CK(cudaFreeHost(H->stage));
            H->stage = nullptr;
            H->stage_cap = 0;
            CK(cudaMallocHost((void**)&H->stage, 2 * need));
            H->stage_cap = 2 * need;
        }
        H->stage_used = 0;
    }
    CK(stage_upload(H, H->dc.p, hc.data(), n));
    {
        std::vector<float> c9(9 * (size_t)n);
        std::vector<int32_t> s0(n), v0(n);
        for (int q = 0; q < n; ++q) {
            for (int a = 0; a < 3; ++a)
                for (int d = 0; d < 3; ++d) c9[9 * q + 3 * a + d] = (float)hc[q].c[a][d];
            const bool single = hc[q].nv == 1 && hc[q].w[0] == 1.0;
            s0[q] = single ? hc[q].slot[0] : -1;
            v0[q] = single ? hc[q].vtx[0] : -1;
        }
        CK(stage_upload(H, H->cc9.p, c9.data(), c9.size()));
        CK(stage_upload(H, H->cs0.p, s0.data(), n));
        CK(stage_upload(H, H->cv0.p, v0.data(), n));
        std::vector<int32_t> c1(ns, -1);
        for (int s = 0; s < ns; ++s)
            if (scp[s + 1] - scp[s] == 1 && s0[sci[scp[s]]] == s) c1[s] = sci[scp[s]];
        CK(stage_upload(H, H->cc1.p, c1.data(), ns));
    }
    CK(stage_upload(H, H->slot_vtx.p, verts.data(), ns));
    CK(stage_upload(H, H->scp.p, scp.data(), ns + 1));
    CK(stage_upload(H, H->sci.p, sci.data(), sci.size()));
    CK(stage_upload(H, H->scw.p, scw.data(), scw.size()));
    CK(stage_upload(H, H->vcp.p, vcp.data(), (size_t)H->n_f + 1));
    CK(stage_upload(H, H->vci.p, sci.data(), sci.size()));   // slots are sorted by vertex: same order
    CK(stage_upload(H, H->vcw.p, scw.data(), scw.size()));
    H->h2d_contact_bytes = (int64_t)(n * sizeof(DContact) + ns * sizeof(int32_t) + (ns + 1) * sizeof(int32_t) +
                                     2 * sci.size() * (sizeof(int32_t) + sizeof(float)) +
                                     (H->n_f + 1) * sizeof(int32_t));
    // ancestor chains of the contact vertices (for chain_dot / scatter)
    std::vector<int32_t> coff(ns + 1, 0);
    for (int s = 0; s < ns; ++s) coff[s + 1] = coff[s] + H->K.depth[verts[s]] + 1;
    if ((size_t)coff[ns] > H->chain_rows.n) {
        CK(cudaStreamSynchronize(st));
        CK(H->chain_rows.alloc(std::max<size_t>(coff[ns], 2 * H->chain_rows.n)));
        CK(H->Zc.alloc(H->chain_rows.n));
        H->contact_gen++;
    }
    CK(stage_upload(H, H->chain_off.p, coff.data(), ns + 1));
    CK(cudaEventRecord(H->stage_free, st));
    CK(cudaMemsetAsync(H->flag.p, 0, H->n_f, st));
    CK(cudaMemsetAsync(H->ucount.p, 0, 2 * sizeof(int), st));
    launch_chain_rows(st, ns, H->slot_vtx.p, H->chain_off.p, H->parent.p, H->ptop.p, H->chain_rows.p, H->flag.p);
    launch_ulist(st, H->n_f, ns, H->flag.p, H->slot_vtx.p, H->meta.p, H->ucount.p, H->ulist.p, H->Krow.p, H->Zc.p);
    H->h2d_contact_bytes += (ns + 1) * sizeof(int32_t);
    // Delassus Gram and D_jj on the device
    launch_delassus(st, ns, H->slot_vtx.p, H->Kcol.p, H->colptr.p, H->depth.p, H->parent.p, H->ptop.p, H->G.p);
    launch_djj(st, n, ns, H->dc.p, H->G.p);
    CK(cudaGetLastError());
    H->nc = n;
    H->ns = ns;
    H->row_lo = ns ? verts[0] : H->n_f;
    H->hc = hc;
    H->slot_vtx_h = verts;
    H->set_contacts_host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count();
    return SIM_OK;   // asynchronous: the copies and kernels are ordered on the handle's stream
}

// ---------------------------------------------------------------------------
// frame driver
// ---------------------------------------------------------------------------
static Params make_params(const sim_handle* H) {
    Params P;
    P.n_v = H->n_v;
    P.n_f = H->n_f;
    P.n_t = H->n_t;
    P.h = H->h;
    for (int d = 0; d < 3; ++d) { P.g[d] = H->mat.gravity[d]; P.vpin[d] = H->vpin[d]; }
    P.model = H->mat.model;
    P.k = (float)H->kproj;
    P.mu = (float)H->mu_l;
    P.lam = (float)H->lam_l;
    P.nc = H->nc;
    P.ns = H->ns;
    P.cr_iters = H->mat.cr_iterations;
    return P;
}

static ContactState cstate(sim_handle* H) {
    return ContactState{H->lam.p, H->theta.p, H->cdiag.p, H->hvec.p, H->hl.p, H->dxt.p, H->wz.p, H->phi_abs.p, H->cr_res.p, H->rho.p};
}

// enqueue one frame (predict + iters x L-G); returns kernel count or negative
enum { KK_PREDICT, KK_CONTACT, KK_LOCAL, KK_GATHER, KK_KPASS1, KK_CHAIN, KK_CR, KK_SCATTER, KK_KPASS2, KK_ACTIVE, KK_N };

static int enqueue_frame(sim_handle* H, int iters) {
    cudaStream_t st = H->stream;
    Params P = make_params(H);
    ContactState cs = cstate(H);
    const CrContacts ccr{H->cc9.p, H->cs0.p, H->cv0.p, H->cc1.p};
    const CrActive act{H->act_na.p, H->act_idx.p, H->act_pos.p, H->act_con.p};
    int nk = 0;
    size_t ev = 0;
    H->pkind.clear();
    auto mark = [&](int kind) -> int {
        if (!H->profiling) return 0;
        while (H->pev.size() <= ev) {
            cudaEvent_t e;
            cudaError_t r = cudaEventCreate(&e);
            if (r != cudaSuccess) return (int)r;
            H->pev.push_back(e);
        }
        H->pkind.push_back(kind);
        return (int)cudaEventRecordWithFlags(H->pev[ev++], st, cudaEventRecordExternal);
    };
#define MARK(k) do { int r_ = mark(k); if (r_) return -r_; } while (0)
#define CKR(call) do { cudaError_t r_ = (call); if (r_ != cudaSuccess) return -(int)r_; } while (0)
    MARK(KK_PREDICT);
    launch_predict(st, P, H->x.p, H->xt.p, H->v.p, H->s.p, H->lam.p, 3 * H->nc); nk++;
    const bool con = H->nc > 0;
    for (int k = 0; k < iters; ++k) {
        // contact evaluation and the local step only read x^k: run them as two graph
        // branches (serial when profiling, so the per-kernel events stay meaningful)
        const bool fork = con && !H->profiling;
        if (fork) {
            CKR(cudaEventRecord(H->fork_ev, st));
            CKR(cudaStreamWaitEvent(H->aux, H->fork_ev, 0));
            launch_contact_eval(H->aux, P, H->dc.p, H->x.p, H->xt.p, cs); nk++;
            launch_active(H->aux, H->ns, ccr, H->scp.p, H->sci.p, cs, act, H->G.p, H->GA.p); nk += 2;
            CKR(cudaEventRecord(H->join_ev, H->aux));
        } else if (con) {
            MARK(KK_CONTACT); launch_contact_eval(st, P, H->dc.p, H->x.p, H->xt.p, cs); nk++;
            MARK(KK_ACTIVE); launch_active(st, H->ns, ccr, H->scp.p, H->sci.p, cs, act, H->G.p, H->GA.p); nk += 2;
        }
        MARK(KK_LOCAL);
        launch_local(st, P, H->tet.p, H->Bm.p, H->hw2.p, H->x.p, H->fc.p, nullptr); nk++;
        if (fork) CKR(cudaStreamWaitEvent(st, H->join_ev, 0));
        MARK(KK_GATHER);
        launch_gather(st, P, H->adjp.p, H->adj.p, H->fc.p, H->M.p, H->x.p, H->s.p, con ? H->vcp.p : nullptr,
                      H->vci.p, H->vcw.p, H->hl.p, H->cb.p, H->u.p, nullptr); nk++;
        MARK(KK_KPASS1);
        launch_kpass1(st, (int)H->wl.p1.size(), H->p1.p, H->p1b.p, H->T1.p, H->u.p, H->y.p, H->part1.p,
                      H->counters.p); nk++;
        if (con) {
            MARK(KK_CHAIN);
            launch_chain_dot(st, H->ns, H->slot_vtx.p, H->Kcol.p, H->colptr.p, H->chain_off.p, H->chain_rows.p,
                             H->y.p, H->dxt.p, ccr, H->x.p, cs); nk++;
            MARK(KK_CR);
            int e = launch_cr(st, P, H->dc.p, ccr, H->scp.p, H->sci.p, H->scw.p, H->GA.p, H->x.p, cs, act); nk++;
            if (e) return -e;
            MARK(KK_SCATTER);
            launch_scatter(st, H->n_f, H->ucount.p, H->ulist.p, H->Zc.p, H->wz.p, H->y.p); nk++;
        }
        MARK(KK_KPASS2);
        launch_kpass2(st, (int)H->wl.p2b.size(), H->p2b.p, H->cover.p, H->T2.p, H->y.p, H->x.p, H->xt.p, H->v.p,
                      1.0 / H->h, k == iters - 1); nk++;
    }
    MARK(KK_N);
#undef MARK
#undef CKR
    return nk;
}

extern "C" int sim_set_profiling(sim_handle* H, int on) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    H->profiling = on ? 1 : 0;
    return SIM_OK;
}

// per-kind device time (ms) of the most recent replayed frame: out[kind] += ...
extern "C" int sim_get_kernel_times(sim_handle* H, double* out, int32_t cap) {
    if (!H || !out) return fail(SIM_E_INVALID, "null argument");
    if (cap < KK_N) return fail(SIM_E_INVALID, "capacity must be >= %d", KK_N);
    for (int k = 0; k < KK_N; ++k) out[k] = 0.0;
    if (!H->profiling || H->g_prof != 1 || H->pkind.size() < 2) return fail(SIM_E_STATE, "profiling off");
    CK(cudaStreamSynchronize(H->stream));
    for (size_t i = 0; i + 1 < H->pkind.size(); ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, H->pev[i], H->pev[i + 1]));
        out[H->pkind[i]] += ms;
    }
    return SIM_OK;
}

extern "C" int sim_step(sim_handle* H, int32_t frames, int32_t iters) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->host_only) return fail(SIM_E_STATE, "host-only handle");
    if (H->state != 1) return fail(SIM_E_STATE, "build the sparse inverse first");
    if (frames < 0 || iters < 1) return fail(SIM_E_INVALID, "frames >= 0 and iterations >= 1");
    if (frames == 0) return SIM_OK;
    if (!H->gexec || H->g_iters != iters || H->g_nc != H->nc || H->g_ns != H->ns || H->g_prof != H->profiling ||
        H->g_gen != H->contact_gen) {
        if (H->gexec) {
            cudaGraphExecDestroy(H->gexec);
            H->gexec = nullptr;
        }
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(H->stream, cudaStreamCaptureModeThreadLocal));
        int nk = enqueue_frame(H, iters);
        cudaError_t ce = cudaStreamEndCapture(H->stream, &g);
        if (nk < 0) return fail(SIM_E_CUDA, "launch failed in capture: %s", cudaGetErrorString((cudaError_t)(-nk)));
        if (ce != cudaSuccess) return fail(SIM_E_CUDA, "capture: %s", cudaGetErrorString(ce));
        cudaError_t ie = cudaGraphInstantiate(&H->gexec, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) return fail(SIM_E_CUDA, "instantiate: %s", cudaGetErrorString(ie));
        H->g_iters = iters;
        H->g_nc = H->nc;
        H->g_ns = H->ns;
        H->g_prof = H->profiling;
        H->g_gen = H->contact_gen;
        H->kernels_per_frame = nk;
    }
    for (int f = 0; f < frames; ++f) CK(cudaGraphLaunch(H->gexec, H->stream));
    H->frames_done += frames;
    return SIM_OK;
}

extern "C" int sim_synchronize(sim_handle* H) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->host_only) return SIM_OK;
    CK(cudaStreamSynchronize(H->stream));
    return SIM_OK;
}

extern "C" int sim_set_pin_velocity(sim_handle* H, const double v[3]) {
    if (!H || !v) return fail(SIM_E_INVALID, "null argument");
    for (int d = 0; d < 3; ++d)
        if (!std::isfinite(v[d])) return fail(SIM_E_INVALID, "pin velocity not finite");
    for (int d = 0; d < 3; ++d) H->vpin[d] = v[d];
    if (H->gexec) {   // vpin is a captured kernel argument
        cudaGraphExecDestroy(H->gexec);
        H->gexec = nullptr;
    }
    return SIM_OK;
}

extern "C" int sim_get_state(sim_handle* H, double* x, double* v) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    std::vector<double4> hx(H->n_v), hv(H->n_v);
    CK(cudaStreamSynchronize(H->stream));
    CK(cudaMemcpy(hx.data(), H->x.p, H->n_v * sizeof(double4), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hv.data(), H->v.p, H->n_v * sizeof(double4), cudaMemcpyDeviceToHost));
    for (int i = 0; i < H->n_v; ++i) {
        int o = H->int2orig[i];
        if (x) { x[3 * o] = hx[i].x; x[3 * o + 1] = hx[i].y; x[3 * o + 2] = hx[i].z; }
        if (v) { v[3 * o] = hv[i].x; v[3 * o + 1] = hv[i].y; v[3 * o + 2] = hv[i].z; }
    }
    return SIM_OK;
}

extern "C" int sim_set_state(sim_handle* H, const double* x, const double* v) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    std::vector<double4> hx(H->n_v), hv(H->n_v);
    CK(cudaStreamSynchronize(H->stream));
    CK(cudaMemcpy(hx.data(), H->x.p, H->n_v * sizeof(double4), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hv.data(), H->v.p, H->n_v * sizeof(double4), cudaMemcpyDeviceToHost));
    for (int i = 0; i < H->n_v; ++i) {
        int o = H->int2orig[i];
        if (x) {
            for (int d = 0; d < 3; ++d)
                if (!std::isfinite(x[3 * o + d])) return fail(SIM_E_INVALID, "x not finite");
            hx[i] = make_double4(x[3 * o], x[3 * o + 1], x[3 * o + 2], 0.0);
        }
        if (v) {
            for (int d = 0; d < 3; ++d)
                if (!std::isfinite(v[3 * o + d])) return fail(SIM_E_INVALID, "v not finite");
            hv[i] = make_double4(v[3 * o], v[3 * o + 1], v[3 * o + 2], 0.0);
        }
    }
    CK(cudaMemcpy(H->x.p, hx.data(), H->n_v * sizeof(double4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(H->v.p, hv.data(), H->n_v * sizeof(double4), cudaMemcpyHostToDevice));
    return SIM_OK;
}

extern "C" int sim_get_lambda(sim_handle* H, double* lam, int32_t cap) {
    if (!H || !lam) return fail(SIM_E_INVALID, "null argument");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    int rows = 0;
    for (int c = 0; c < H->nc; ++c) rows += H->hc[c].kind == 1 ? 1 : 3;
    if (cap < rows) return fail(SIM_E_INVALID, "capacity %d < %d rows", cap, rows);
    std::vector<double> l(3 * (size_t)H->nc);
    CK(cudaStreamSynchronize(H->stream));
    if (H->nc) CK(cudaMemcpy(l.data(), H->lam.p, l.size() * sizeof(double), cudaMemcpyDeviceToHost));
    int r = 0;
    for (int c = 0; c < H->nc; ++c) {
        lam[r++] = l[3 * c];
        if (H->hc[c].kind != 1) {
            lam[r++] = l[3 * c + 1];
            lam[r++] = l[3 * c + 2];
        }
    }
    return SIM_OK;
}

extern "C" int sim_get_stats(sim_handle* H, sim_stats* o) {
    if (!H || !o) return fail(SIM_E_INVALID, "null argument");
    memset(o, 0, sizeof *o);
    o->n_vertices = H->n_v;
    o->n_free = H->n_f;
    o->n_tets = H->n_t;
    o->nnz_K = H->K.nnz;
    o->nnz_L = H->nnzL;
    o->etree_height = H->K.height;
    o->n_panels = H->K.panel_start.empty() ? 0 : (int)H->K.panel_start.size() - 1;
    o->n_contacts = H->nc;
    o->n_contact_vertices = H->ns;
    o->frames_done = H->frames_done;
    o->kernels_per_frame = H->kernels_per_frame;
    o->build_seconds = H->build_seconds;
    o->h2d_contact_bytes = H->h2d_contact_bytes;
    o->last_cr_residual = -1;
    if (!H->host_only && H->state == 1 && H->nc > 0) {
        CK(cudaStreamSynchronize(H->stream));
        double r;
        CK(cudaMemcpy(&r, H->cr_res.p, sizeof r, cudaMemcpyDeviceToHost));
        o->last_cr_residual = r;
        std::vector<double> ph(H->nc), l(3 * (size_t)H->nc);
        CK(cudaMemcpy(ph.data(), H->phi_abs.p, H->nc * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(l.data(), H->lam.p, l.size() * sizeof(double), cudaMemcpyDeviceToHost));
        double mx = 0;
        int act = 0;
        for (int c = 0; c < H->nc; ++c) {
            mx = std::max(mx, ph[c]);
            act += (H->hc[c].kind == 0 && l[3 * c] > 0);
        }
        o->max_abs_phi_n = mx;
        o->n_active = act;
    }
    return SIM_OK;
}

// ---------------------------------------------------------------------------
// test hooks
// ---------------------------------------------------------------------------
extern "C" int sim_debug_get_inverse(sim_handle* H, int32_t* perm, int32_t* parent, int64_t* rowptr, float* vals) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1) return fail(SIM_E_STATE, "build first");
    int nf = H->n_f;
    if (perm) for (int k = 0; k < nf; ++k) perm[k] = H->int2orig[k];
    if (parent) std::copy(H->K.parent.begin(), H->K.parent.end(), parent);
    if (rowptr) std::copy(H->K.rowptr.begin(), H->K.rowptr.end(), rowptr);
    if (vals) std::copy(H->K.Krow.begin(), H->K.Krow.end(), vals);
    return SIM_OK;
}

extern "C" int sim_debug_apply_inverse(sim_handle* H, const double* b, double* xo) {
    if (!H || !b || !xo) return fail(SIM_E_INVALID, "null argument");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    const int nf = H->n_f;
    std::vector<float4> hu(nf);
    for (int k = 0; k < nf; ++k) {
        int o = H->int2orig[k];
        int32_t cbk = (int32_t)(H->K.colptr[k] + H->K.depth[k]);
        float cbf;
        memcpy(&cbf, &cbk, sizeof cbf);
        hu[k] = make_float4((float)b[3 * o], (float)b[3 * o + 1], (float)b[3 * o + 2], cbf);
    }
    DBuf<double4> dx;
    CK(dx.alloc(nf));
    cudaStream_t st = H->stream;
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(H->u.p, hu.data(), nf * sizeof(float4), cudaMemcpyHostToDevice));
    CK(cudaMemset(dx.p, 0, nf * sizeof(double4)));
    launch_kpass1(st, (int)H->wl.p1.size(), H->p1.p, H->p1b.p, H->T1.p, H->u.p, H->y.p, H->part1.p, H->counters.p);
    launch_kpass2(st, (int)H->wl.p2b.size(), H->p2b.p, H->cover.p, H->T2.p, H->y.p, dx.p, nullptr, nullptr, 1.0, 0);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    std::vector<double4> hx(nf);
    CK(cudaMemcpy(hx.data(), dx.p, nf * sizeof(double4), cudaMemcpyDeviceToHost));
    dx.release();
    for (int i = 0; i < 3 * H->n_v; ++i) xo[i] = 0.0;
    for (int k = 0; k < nf; ++k) {
        int o = H->int2orig[k];
        xo[3 * o] = hx[k].x;
        xo[3 * o + 1] = hx[k].y;
        xo[3 * o + 2] = hx[k].z;
    }
    return SIM_OK;
}

extern "C" int sim_debug_local(sim_handle* H, const double* x, const double* s, float* Pout, double* resid) {
    if (!H || !x || !s) return fail(SIM_E_INVALID, "null argument");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    const int nv = H->n_v, nf = H->n_f, nt = H->n_t;
    std::vector<double4> hx(nv), hs(nv);
    for (int i = 0; i < nv; ++i) {
        int o = H->int2orig[i];
        hx[i] = make_double4(x[3 * o], x[3 * o + 1], x[3 * o + 2], 0.0);
        hs[i] = make_double4(s[3 * o], s[3 * o + 1], s[3 * o + 2], 0.0);
    }
    cudaStream_t st = H->stream;
    CK(cudaStreamSynchronize(st));
    DBuf<double4> dx, ds;
    DBuf<float> dP;
    DBuf<double> dr;
    CK(dx.alloc(nv)); CK(ds.alloc(nv)); CK(dP.alloc((size_t)9 * nt)); CK(dr.alloc(3 * (size_t)nf));
    CK(cudaMemcpy(dx.p, hx.data(), nv * sizeof(double4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ds.p, hs.data(), nv * sizeof(double4), cudaMemcpyHostToDevice));
    Params P = make_params(H);
    launch_local(st, P, H->tet.p, H->Bm.p, H->hw2.p, dx.p, H->fc.p, dP.p);
    launch_gather(st, P, H->adjp.p, H->adj.p, H->fc.p, H->M.p, dx.p, ds.p, nullptr, nullptr, nullptr, nullptr,
                  H->cb.p, H->u.p, dr.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    if (Pout) CK(cudaMemcpy(Pout, dP.p, (size_t)9 * nt * sizeof(float), cudaMemcpyDeviceToHost));
    if (resid) {
        std::vector<double> hr(3 * (size_t)nf);
        CK(cudaMemcpy(hr.data(), dr.p, hr.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 3 * nv; ++i) resid[i] = 0.0;
        for (int k = 0; k < nf; ++k) {
            int o = H->int2orig[k];
            for (int d = 0; d < 3; ++d) resid[3 * o + d] = hr[3 * k + d];
        }
    }
    dx.release(); ds.release(); dP.release(); dr.release();
    return SIM_OK;
}

extern "C" int sim_debug_get_delassus(sim_handle* H, int32_t* cv, float* G, int32_t cap) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    if (cap < H->ns) return fail(SIM_E_INVALID, "capacity %d < %d contact vertices", cap, H->ns);
    CK(cudaStreamSynchronize(H->stream));
    if (cv) for (int s = 0; s < H->ns; ++s) cv[s] = H->int2orig[H->slot_vtx_h[s]];
    if (G && H->ns) {
        std::vector<double> g((size_t)H->ns * H->ns);
        CK(cudaMemcpy(g.data(), H->G.p, g.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (size_t q = 0; q < g.size(); ++q) G[q] = (float)g[q];
    }
    return SIM_OK;
}

// contact scratch of the last evaluated L-G iteration: per row (3 per contact)
// theta, C diagonal, h-vector; per slot dxt = (K^T y) at the slot vertex; slot vertices
extern "C" int sim_debug_contact_state(sim_handle* H, double* theta, double* cdiag, double* hvec, double* dxt,
                                       int32_t* slot_vertex, double* djj) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    CK(cudaStreamSynchronize(H->stream));
    size_t m = 3 * (size_t)H->nc;
    if (theta && m) CK(cudaMemcpy(theta, H->theta.p, m * sizeof(double), cudaMemcpyDeviceToHost));
    if (cdiag && m) CK(cudaMemcpy(cdiag, H->cdiag.p, m * sizeof(double), cudaMemcpyDeviceToHost));
    if (hvec && m) CK(cudaMemcpy(hvec, H->hvec.p, m * sizeof(double), cudaMemcpyDeviceToHost));
    if (dxt && H->ns) CK(cudaMemcpy(dxt, H->dxt.p, 3 * (size_t)H->ns * sizeof(double), cudaMemcpyDeviceToHost));
    if (slot_vertex) for (int s = 0; s < H->ns; ++s) slot_vertex[s] = H->int2orig[H->slot_vtx_h[s]];
    if (djj && H->nc) {
        std::vector<DContact> hc(H->nc);
        CK(cudaMemcpy(hc.data(), H->dc.p, H->nc * sizeof(DContact), cudaMemcpyDeviceToHost));
        for (int c = 0; c < H->nc; ++c) djj[c] = hc[c].Djj;
    }
    return SIM_OK;
}

// phase timestamps (ns, %globaltimer) of the most recent CR call: [0] start,
// [1] after rho, [2] after active set + G_A gather, [3 + it] after CR iteration it,
// [20] loop end, [21] epilogue end.  out must hold 32 values.
extern "C" int sim_debug_cr_timeline(sim_handle* H, double* out) {
    if (!H || !out) return fail(SIM_E_INVALID, "null argument");
    if (H->host_only) return fail(SIM_E_STATE, "no device");
    CK(cudaStreamSynchronize(H->stream));
    unsigned long long t[32];
    CK((cudaError_t)read_cr_clock(t));
    for (int i = 0; i < 32; ++i) out[i] = (double)(t[i] - t[0]) * 1e-3;   // us since start
    return SIM_OK;
}
