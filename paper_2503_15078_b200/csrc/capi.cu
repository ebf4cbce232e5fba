// C ABI (include/sim.h) and the iteration driver: one CUDA Graph per frame.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>
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

// device allocator (sim_set_allocator): process-wide; every buffer remembers the allocator it
// was allocated with and is returned to it
struct SimAllocator {
    void* (*alloc)(size_t, void*) = nullptr;
    void (*free_)(void*, void*) = nullptr;
    void* ctx = nullptr;
};
static std::mutex g_alloc_mu;
static SimAllocator g_alloc;

static cudaError_t dev_alloc(void** p, size_t bytes, SimAllocator& used) {
    {
        std::lock_guard<std::mutex> lk(g_alloc_mu);
        used = g_alloc;
    }
    if (!used.alloc) return cudaMalloc(p, bytes);
    *p = used.alloc(bytes, used.ctx);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
}
static void dev_free(void* p, const SimAllocator& used) {
    if (!used.free_) {
        cudaFree(p);   // implicitly waits for the device work that may still read p
        return;
    }
    cudaDeviceSynchronize();   // a caching allocator may hand p out again right away
    used.free_(p, used.ctx);
}

template <class T>
struct DPtr {   // a view into a device arena
    T* p = nullptr;
};

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    SimAllocator al;
    cudaError_t alloc(size_t cnt) {
        release();
        n = cnt;
        if (cnt == 0) return cudaSuccess;
        void* q = nullptr;
        cudaError_t e = dev_alloc(&q, cnt * sizeof(T), al);
        if (e != cudaSuccess) {
            n = 0;
            return e;
        }
        p = (T*)q;
        return cudaSuccess;
    }
    cudaError_t upload(const T* h, size_t cnt, cudaStream_t st) {
        if (cnt == 0) return cudaSuccess;
        return cudaMemcpyAsync(p, h, cnt * sizeof(T), cudaMemcpyHostToDevice, st);
    }
    // grow to at least cnt elements (contents not preserved); sets grew when reallocated
    cudaError_t ensure(size_t cnt, bool& grew) {
        if (cnt <= n && p) return cudaSuccess;
        grew = true;
        return alloc(std::max<size_t>(cnt + cnt / 4, 16));
    }
    void release() {
        if (p) dev_free(p, al);
        p = nullptr;
        n = 0;
    }
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
};

// one instance's contact set, host side, in instance-local numbering (validated)
struct InstContacts {
    std::vector<DContact> hc;        // slot[] local, vtx internal
    std::vector<int32_t> verts;      // slot -> internal vertex (ascending)
    std::vector<int32_t> scp, sci;   // slot -> local contacts
    std::vector<float> scw;
    std::vector<float> c9;
    std::vector<int32_t> s0, v0, c1; // local slot / vertex / local contact
    int64_t chain_total = 0;         // sum over slots of (depth + 1)
    bool large = false;              // beyond the cluster CR's limits: needs the grid CR (one scene)
    // lambda carried across commits (reading A10): carry[c] = local index of the identical
    // constraint in the instance's device-committed set (whose lambda is on the device), or -1
    std::vector<int32_t> carry;
    bool dev = false;                // this set is the device-committed one
};

// identity of a constraint for the lambda carry: kind, vertices, weights, row directions
static bool same_constraint(const DContact& a, const DContact& b) {
    if (a.kind != b.kind || a.nv != b.nv) return false;
    for (int q = 0; q < a.nv; ++q)
        if (a.vtx[q] != b.vtx[q] || a.w[q] != b.w[q]) return false;
    return memcmp(a.c, b.c, sizeof a.c) == 0;
}
static uint64_t constraint_hash(const DContact& a) {
    uint64_t h = 1469598103934665603ull ^ (uint64_t)(a.kind * 8 + a.nv);
    for (int q = 0; q < a.nv; ++q) h = (h ^ (uint64_t)(uint32_t)a.vtx[q]) * 1099511628211ull;
    return h;
}
// nw.carry from the instance's previous set `old`: each new contact takes the first unused
// identical constraint of `old` (old.dev: its index; otherwise old's own carry, so that several
// sim_set_contacts calls between two steps compose)
static void compute_carry(const InstContacts& old, InstContacts& nw) {
    const int n = (int)nw.hc.size(), no = (int)old.hc.size();
    nw.carry.assign(n, -1);
    if (no == 0 || n == 0) return;
    {   // common case (a detector re-emitting the same set): contact c is old contact c
        int c = 0;
        while (c < std::min(n, no) && same_constraint(old.hc[c], nw.hc[c])) ++c;
        if (c == n) {
            for (int k = 0; k < n; ++k) nw.carry[k] = old.dev ? k : (k < (int)old.carry.size() ? old.carry[k] : -1);
            return;
        }
    }
    std::unordered_map<uint64_t, std::vector<int>> pool;
    for (int c = no - 1; c >= 0; --c) pool[constraint_hash(old.hc[c])].push_back(c);   // popped from the back
    for (int c = 0; c < n; ++c) {
        auto it = pool.find(constraint_hash(nw.hc[c]));
        if (it == pool.end()) continue;
        std::vector<int>& v = it->second;
        for (int k = (int)v.size() - 1; k >= 0; --k)
            if (same_constraint(old.hc[v[k]], nw.hc[c])) {
                const int o = v[k];
                v.erase(v.begin() + k);
                nw.carry[c] = old.dev ? o : (o < (int)old.carry.size() ? old.carry[o] : -1);
                break;
            }
    }
}

struct sim_handle {
    bool host_only = false;
    int device = -1;
    int S = 1;                             // instances sharing mesh, material and K
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
    double len_scale = 0;   // max(rest bbox diagonal, max |rest coordinate|) (gap snapping, reading A15)
    simhost::RestData rd;
    std::vector<int32_t> int2orig, orig2int;
    simhost::Inverse K;
    simhost::WorkLists wl;
    std::vector<float> T1h, T2h;
    std::vector<simhost::BUnit> bu1, bu2;   // batched K-pass units (S > 1)
    std::vector<float> T1ph;
    int bparts = 0, bblocks1 = 0;
    simhost::PlaneUnits pu;                 // plane-layout tensor-core K-pass units (S > 1)
    int64_t nnzL = 0;
    int64_t nnz_kept = 0;            // nonzeros of K after the drop tolerance
    double build_seconds = 0;
    DBuf<double4> vpin;              // [n_v - n_f][S] pinned-vertex velocities (moving Dirichlet targets)
    DBuf<double4> pin_tgt;           // sim_set_pins staging on the device
    double4* pin_stage = nullptr;    // pinned host staging of sim_set_pins
    cudaEvent_t pin_free = nullptr;
    // device: state, [entity][S]
    DBuf<double4> x, xt, v, s;
    DBuf<double4> vt;                // frame-start velocity (rollback on a non-finite frame)
    DBuf<int> bad;                   // [S] per-instance failure flags of the current frame
    DBuf<int> rollbacks;             // device counter of rolled-back instance-frames (read by sim_synchronize)
    int64_t rollbacks_total = 0;
    double build_phase[5] = {0, 0, 0, 0, 0};   // assemble, ordering, Cholesky, K = L^-1, work lists + tiles
    bool inverse_on_device = false;
    int poison_inst = -1;            // sim_debug_poison: instance whose next frame gets a NaN
    // asynchronous position read-back (sim_get_positions_async): double-buffered device staging
    // in the caller's layout, copied to the host on a copy stream while the next frames compute
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t pos_ready[2] = {nullptr, nullptr}, pos_copied[2] = {nullptr, nullptr};
    DBuf<double> pos_stage[2];
    DBuf<int32_t> o2i;               // original vertex -> internal index (device)
    int pos_slot = 0, pos_last = -1;
    DBuf<double> M;
    DBuf<int4> tet;
    DBuf<float> Bm, hw2;
    DBuf<float> fc;          // corner forces [tet][corner][xyz][instance]
    DBuf<float4> u, y;
    DBuf<int32_t> adjp, adj;
    // device: K
    DBuf<float> Krow, Kcol, T1, T2, T1p;   // K row/column-major + the passes' tile streams
    DBuf<float> Tpl1, Tpl2;                // plane-layout tensor-core tile streams (S > 1)
    DBuf<simhost::BUnit> pu1d, pu2d;
    DBuf<int32_t> pcover;
    DBuf<float> ppart;                     // fp32 partials of split pass-1 blocks
    DBuf<int> pcounters;
    int kpass_mode = 2;                    // S > 1: 2 (or 0) tcgen05 plane kernels, 1 CUDA-core FP32
    int tc_drain = 4;                      // tensor-core K-pass: tiles per fp32 TMEM accumulation
    DBuf<int64_t> colptr;
    DBuf<int32_t> depth, parent, ptop, cover;
    DBuf<int2> meta;                 // {rowptr[i] - first[i], first[i]}
    DBuf<P1Item> p1;
    DBuf<P1Block> p1b;
    DBuf<P2Block> p2b;
    DBuf<simhost::BUnit> bu1d, bu2d;
    DBuf<double> part1;
    DBuf<int> counters;
    // contacts: host per instance, device packed over instances
    std::vector<InstContacts> ic;
    bool dirty = false;
    int C = 0, NS = 0, nc_max = 0, ns_max = 0, urows_max = 0;
    std::vector<int> coff_h, soff_h;
    // uploaded contact data: one device arena with the staging layout (one H2D copy per commit)
    DBuf<unsigned char> arena;
    // the H2D upload of a commit lands in arena_up on up_stream (overlapping the frames still
    // running on the handle's stream); the stream then takes it with one D2D copy into arena
    DBuf<unsigned char> arena_up;
    cudaStream_t up_stream = nullptr;
    cudaEvent_t up_done = nullptr, up_free = nullptr;
    std::vector<size_t> arena_layout;
    DPtr<DContact> dc;
    DPtr<float> cc9;
    DPtr<int32_t> cs0, cv0, cc1;
    DPtr<int32_t> slot_vtx, slot_inst, scp, sci;
    DPtr<float> scw;
    DPtr<int> coff, soff, uoff, cls, csoff, cmoff, cmem;
    DPtr<int64_t> goff, zoff, gaoff;
    DPtr<int32_t> cvtx, ccls;        // class slots
    DPtr<int2> it_cd, it_sc;         // grouped chain-dot / scatter work items
    DPtr<int32_t> chain_off;
    int NCL = 0, CS = 0, cm_max = 0, n_it_cd = 0, n_it_sc = 0;
    std::vector<int64_t> gaoff_h;
    DBuf<float> G, GA;   // Delassus Gram blocks and the CR's active blocks (fp32-exact values)
    // Gram reuse across commits (sim_set_schur_reuse): the previous commit's class blocks
    bool schur_reuse = false, have_prev = false;
    bool dev_pending = false;        // host half of a contact commit done, device half not yet
    // contact passes on the tensor cores (S > 1, one slot-set class): work lists + tiles
    bool tc_contact = false;
    std::vector<int32_t> tc_verts;   // the class vertex set the tiles were built for
    DBuf<simhost::BUnit> tcu_c, tcu_s;
    DBuf<double> tc_cpart, tc_spart;   // chain / scatter-pass partial sums (units split when few instances
    DBuf<int> tc_ccnt, tc_scnt;        // leave SMs idle) and their per-unit arrival counters
    DBuf<int32_t> tc_cover, tc_rows;
    DBuf<float> tc_Tc, tc_Ts;
    int tc_nuc = 0, tc_nus = 0, tc_ns = 0;
    bool pend_reuse = false;
    int pend_nnew = 0;
    std::vector<std::vector<int32_t>> prev_cls_verts;
    std::vector<int64_t> prev_goff;
    std::vector<int> prev_cls_of_inst;
    int64_t prev_gsize = 0;
    DBuf<float> Gprev;
    int64_t gram_rows_computed = 0, gram_rows_reused = 0;   // statistics of the last commit
    DPtr<int> rmap, pns;
    DPtr<int64_t> pgoff;
    DPtr<int2> newslots;
    DBuf<double> lam, theta, cdiag, hvec, hl, dxt, wz, phi_abs, cr_res, rho;
    DBuf<double> lam_prev;           // the previous commit's lambda while it is carried (reading A10)
    std::vector<int> coff_dev;       // contact offsets of the device-committed set (lambda's layout)
    int C_dev = 0;
    DPtr<int32_t> carry;             // [C] (arena): previous-commit contact of each contact, or -1
    DBuf<int> act_na, act_idx, act_pos, act_con;   // CR active set (k_active)
    DBuf<float4> wzT;
    DBuf<int32_t> chain_rows, slotmap;
    DBuf<uint8_t> flag;
    DBuf<int> ucount;
    DBuf<int4> ulist;
    DBuf<float> Zc;
    int contact_gen = 0;
    // graph
    cudaGraphExec_t gexec = nullptr;
    std::vector<int64_t> gkey;   // what the captured graph was built for
    int g_prof = -1;
    // in-graph kernel timing (event record nodes between kernels)
    int profiling = 0;
    std::vector<cudaEvent_t> pev;
    std::vector<int> pkind;   // kind of the kernel that follows event i
    int kernels_per_frame = 0;
    int64_t frames_done = 0;
    int64_t h2d_contact_bytes = 0;   // bytes uploaded by the last contact commit
    // pinned staging for asynchronous contact uploads (reused once the last copy is done)
    unsigned char* stage = nullptr;
    size_t stage_cap = 0;
    cudaEvent_t stage_free = nullptr;
    double set_contacts_host_us = 0;
    // grid CR (large contact sets of one scene): Delassus groups = etree components
    int cr_mode = 0;                 // 0 auto, 1 cluster CR only, 2 grid CR always
    int ncp = 0, precond = 0;        // NCP function / complementarity preconditioner (sim_set_ncp)
    int admm = 0;                    // ADMM-PD local-global (sim_set_admm)
    int warm = 0;                    // frame start (sim_set_warm_start): readings A9/A10 or A9w/A10w
    int persistent = 0;              // sim_set_persistent: 0 auto (small contact-free scenes), 1 off
    int local_mode = 0;              // sim_set_local_mode: 0 packed-FP32 instance pairs when S is even, 1 scalar
    bool last_persistent = false;    // the last sim_step ran the persistent small-scene kernel
    DBuf<float> du;                  // ADMM dual, [9][n_t S]
    bool grid = false;               // the committed contact set uses the grid CR
    int NG = 0, ng_max = 0;
    std::vector<int32_t> comp_root;  // [n_f] root of each free vertex's etree component
    DPtr<int> gcsoff, gs0, gn;       // group slot offsets [NG+1]; per slot: group start, size
    DPtr<int64_t> ggoff, growoff;    // group G offsets [NG+1]; per slot: its G row
    DBuf<double> g_r, g_p, g_Ap, g_z, g_Ar, g_W, g_q, g_part, g_sc;
    DBuf<int> g_cnt;
    DPtr<int2> g_items;              // Gram matvec items (arena)
    int n_g_items = 0;
};

// ---------------------------------------------------------------------------
static int validate_create(const sim_mesh* m, const sim_material* mat, double h) {
    if (!m || !mat) return fail(SIM_E_INVALID, "null mesh or material");
    if (m->n_vertices <= 0 || m->n_tets <= 0 || !m->rest_positions || !m->tets)
        return fail(SIM_E_INVALID, "empty mesh or null arrays");
    if (m->n_instances < 0 || m->n_instances > 65535) return fail(SIM_E_INVALID, "n_instances must be in [0, 65535]");
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
    if ((int64_t)m->n_tets * 4 * std::max(1, m->n_instances) >= (int64_t)INT32_MAX)
        return fail(SIM_E_LIMIT, "n_tets x 4 x n_instances exceeds the int32 index range");
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
    H->S = std::max(1, m->n_instances);
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
    {
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300}, amax = 0.0;
        for (int i = 0; i < H->n_v; ++i)
            for (int d = 0; d < 3; ++d) {
                const double c = H->X[3 * (size_t)i + d];
                lo[d] = std::min(lo[d], c);
                hi[d] = std::max(hi[d], c);
                amax = std::max(amax, std::fabs(c));
            }
        const double dg = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                    (hi[2] - lo[2]) * (hi[2] - lo[2]));
        H->len_scale = std::max(dg, amax);
    }
    H->mu_l = mat->youngs / (2.0 * (1.0 + mat->poisson));
    H->lam_l = mat->youngs * mat->poisson / ((1.0 + mat->poisson) * (1.0 - 2.0 * mat->poisson));
    H->kproj = mat->proj_stiffness > 0 ? mat->proj_stiffness : 2.0 * H->mu_l;
    H->ic.resize(H->S);
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

extern "C" int sim_set_allocator(void* (*alloc)(size_t, void*), void (*free_)(void*, void*), void* ctx) {
    if ((alloc == nullptr) != (free_ == nullptr)) return fail(SIM_E_INVALID, "alloc and free must both be set or both NULL");
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_alloc.alloc = alloc;
    g_alloc.free_ = free_;
    g_alloc.ctx = alloc ? ctx : nullptr;
    return SIM_OK;
}

extern "C" void sim_destroy(sim_handle* H) {
    if (!H) return;
    if (!H->host_only) {
        if (H->stream) cudaStreamSynchronize(H->stream);
        if (H->gexec) cudaGraphExecDestroy(H->gexec);
        for (auto e : H->pev) cudaEventDestroy(e);
        if (H->stage_free) cudaEventDestroy(H->stage_free);
        if (H->up_stream) cudaStreamSynchronize(H->up_stream);
        if (H->up_done) cudaEventDestroy(H->up_done);
        if (H->up_free) cudaEventDestroy(H->up_free);
        if (H->up_stream) cudaStreamDestroy(H->up_stream);
        if (H->fork_ev) cudaEventDestroy(H->fork_ev);
        if (H->copy_stream) cudaStreamSynchronize(H->copy_stream);
        for (int k = 0; k < 2; ++k) {
            if (H->pos_ready[k]) cudaEventDestroy(H->pos_ready[k]);
            if (H->pos_copied[k]) cudaEventDestroy(H->pos_copied[k]);
        }
        if (H->copy_stream) cudaStreamDestroy(H->copy_stream);
        if (H->join_ev) cudaEventDestroy(H->join_ev);
        if (H->aux) cudaStreamDestroy(H->aux);
        if (H->stage) cudaFreeHost(H->stage);
        if (H->pin_free) cudaEventSynchronize(H->pin_free);
        if (H->pin_stage) cudaFreeHost(H->pin_stage);
        if (H->pin_free) cudaEventDestroy(H->pin_free);
        if (H->own_stream && H->stream) cudaStreamDestroy(H->stream);
    }
    delete H;   // device buffers are released by their destructors
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
    const int nv = H->n_v, nt = H->n_t, nf = H->n_f, S = H->S;
    // state: rest, v = 0, replicated over the instances ([vertex][instance])
    std::vector<double4> xs(nv);
    for (int i = 0; i < nv; ++i) {
        int o = H->int2orig[i];
        xs[i] = make_double4(H->X[3 * o], H->X[3 * o + 1], H->X[3 * o + 2], 0.0);
    }
    const size_t nvS = (size_t)nv * S;
    CK(H->x.alloc(nvS)); CK(H->xt.alloc(nvS)); CK(H->v.alloc(nvS)); CK(H->s.alloc(nvS));
    CK(H->vt.alloc(nvS)); CK(H->bad.alloc(S));
    CK(H->vpin.alloc((size_t)(nv - nf) * S));
    if (nv > nf) CK(cudaMemsetAsync(H->vpin.p, 0, (size_t)(nv - nf) * S * sizeof(double4), st));
    CK(cudaMemsetAsync(H->bad.p, 0, S * sizeof(int), st));
    CK(H->rollbacks.alloc(1));
    CK(cudaMemsetAsync(H->rollbacks.p, 0, sizeof(int), st));
    {
        DBuf<double4> x1;
        CK(x1.alloc(nv));
        CK(x1.upload(xs.data(), nv, st));
        launch_replicate(st, x1.p, H->x.p, nv, S);
        launch_replicate(st, x1.p, H->xt.p, nv, S);
        launch_replicate(st, x1.p, H->s.p, nv, S);
        CK(cudaMemsetAsync(H->v.p, 0, nvS * sizeof(double4), st));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
    }
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
    CK(H->fc.alloc((size_t)12 * nt * S));
    // u, y: float4 [n_f] at S = 1, three fp32 planes [3][n_f][Sp] at S > 1 (vec_ld in kernels.cu)
    const size_t nvec4 = S == 1 ? (size_t)nf : ((size_t)3 * nf * plane_sp(S) + 3) / 4;
    CK(H->u.alloc(nvec4)); CK(H->y.alloc(nvec4));
    CK(cudaMemsetAsync(H->u.p, 0, nvec4 * sizeof(float4), st));
    CK(cudaMemsetAsync(H->y.p, 0, nvec4 * sizeof(float4), st));
    // vertex -> (tet, corner) adjacency for free vertices, ascending tet order
    std::vector<int32_t> adjp(nf + 1, 0), adj;
    for (int t = 0; t < nt; ++t) {
        int q[4] = {tv[t].x, tv[t].y, tv[t].z, tv[t].w};
        for (int c = 0; c < 4; ++c)
            if (q[c] < nf) adjp[q[c] + 1]++;
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
    CK(H->T2.alloc(H->T2h.size())); CK(H->T2.upload(H->T2h.data(), H->T2h.size(), st));
    std::vector<int2> meta(nf);
    for (int j = 0; j < nf; ++j) meta[j] = make_int2((int32_t)(K.rowptr[j] - K.first[j]), K.first[j]);
    CK(H->colptr.alloc(nf + 1)); CK(H->colptr.upload(K.colptr.data(), nf + 1, st));
    CK(H->meta.alloc(nf)); CK(H->meta.upload(meta.data(), nf, st));
    CK(H->depth.alloc(nf)); CK(H->depth.upload(K.depth.data(), nf, st));
    CK(H->parent.alloc(nf)); CK(H->parent.upload(K.parent.data(), nf, st));
    CK(H->ptop.alloc(nf)); CK(H->ptop.upload(K.ptop.data(), nf, st));
    const simhost::WorkLists& W = H->wl;
    CK(H->p2b.alloc(W.p2b.size())); CK(H->p2b.upload(W.p2b.data(), W.p2b.size(), st));
    CK(H->cover.alloc(W.cover.size())); CK(H->cover.upload(W.cover.data(), W.cover.size(), st));
    if (S == 1) {
        CK(H->T1.alloc(H->T1h.size())); CK(H->T1.upload(H->T1h.data(), H->T1h.size(), st));
        CK(H->p1.alloc(W.p1.size())); CK(H->p1.upload(W.p1.data(), W.p1.size(), st));
        CK(H->p1b.alloc(W.p1b.size())); CK(H->p1b.upload(W.p1b.data(), W.p1b.size(), st));
        CK(H->part1.alloc((size_t)std::max(1, W.p1_parts) * 32 * 3));
        size_t ncnt = W.p1b.size();
        CK(H->counters.alloc(ncnt));
        CK(cudaMemsetAsync(H->counters.p, 0, ncnt * sizeof(int), st));
    } else {
        CK(H->T1p.alloc(H->T1ph.size())); CK(H->T1p.upload(H->T1ph.data(), H->T1ph.size(), st));
        {
            const simhost::PlaneUnits& PU = H->pu;
            CK(H->Tpl1.alloc(PU.T1.size())); CK(H->Tpl1.upload(PU.T1.data(), PU.T1.size(), st));
            CK(H->Tpl2.alloc(PU.T2.size())); CK(H->Tpl2.upload(PU.T2.data(), PU.T2.size(), st));
            CK(H->pu1d.alloc(PU.u1.size())); CK(H->pu1d.upload(PU.u1.data(), PU.u1.size(), st));
            CK(H->pu2d.alloc(PU.u2.size())); CK(H->pu2d.upload(PU.u2.data(), PU.u2.size(), st));
            CK(H->pcover.alloc(PU.cover.size())); CK(H->pcover.upload(PU.cover.data(), PU.cover.size(), st));
            CK(H->ppart.alloc((size_t)std::max(1, PU.nparts1) * 3 * 64 * plane_sp(S)));
            const size_t npc = (size_t)std::max(1, PU.nblocks1) * ((S + 127) / 128);
            CK(H->pcounters.alloc(npc));
            CK(cudaMemsetAsync(H->pcounters.p, 0, npc * sizeof(int), st));
            CK(cudaStreamSynchronize(st));
        }
        CK(H->bu1d.alloc(H->bu1.size())); CK(H->bu1d.upload(H->bu1.data(), H->bu1.size(), st));
        CK(H->bu2d.alloc(H->bu2.size())); CK(H->bu2d.upload(H->bu2.data(), H->bu2.size(), st));
        CK(H->part1.alloc((size_t)std::max(1, H->bparts) * 3 * 32 * S));
        const int nch = (S + 127) / 128;
        size_t ncnt = (size_t)H->bblocks1 * nch;
        CK(H->counters.alloc(ncnt));
        CK(cudaMemsetAsync(H->counters.p, 0, ncnt * sizeof(int), st));
    }
    // per-instance contact scalars
    CK(H->cr_res.alloc(S)); CK(H->act_na.alloc(S)); CK(H->ucount.alloc(2 * (size_t)S));
    CK(cudaMemsetAsync(H->cr_res.p, 0, S * sizeof(double), st));
    CK(H->flag.alloc((size_t)S * nf));
    CK(H->slotmap.alloc((size_t)nf * S));
    CK(cudaMemsetAsync(H->slotmap.p, 0xff, (size_t)nf * S * sizeof(int32_t), st));
    H->coff_h.assign(S + 1, 0);
    H->soff_h.assign(S + 1, 0);
    CK(cudaStreamSynchronize(st));
    return SIM_OK;
}

static int device_inverse(sim_handle* H, const simhost::Factor& F, double drop_tol) {
    const simhost::Inverse& K = H->K;
    const int n = F.n;
    const int64_t nnzL = F.Lp[n];
    cudaStream_t st = H->stream;
    DBuf<int64_t> Lp, colptr, rowptr;
    DBuf<int32_t> Li, parent, depth, first;
    DBuf<double> Lx;
    DBuf<float> Kc, Kr;
    CK(Lp.alloc(n + 1)); CK(Lp.upload(F.Lp.data(), n + 1, st));
    CK(Li.alloc(nnzL)); CK(Li.upload(F.Li.data(), nnzL, st));
    CK(Lx.alloc(nnzL)); CK(Lx.upload(F.Lx.data(), nnzL, st));
    CK(parent.alloc(n)); CK(parent.upload(F.parent.data(), n, st));
    CK(depth.alloc(n)); CK(depth.upload(K.depth.data(), n, st));
    CK(first.alloc(n)); CK(first.upload(K.first.data(), n, st));
    CK(colptr.alloc(n + 1)); CK(colptr.upload(K.colptr.data(), n + 1, st));
    CK(rowptr.alloc(n + 1)); CK(rowptr.upload(K.rowptr.data(), n + 1, st));
    CK(Kc.alloc(K.nnz)); CK(Kr.alloc(K.nnz));
    const int e = launch_inverse_columns(st, n, K.height, Lp.p, Li.p, Lx.p, parent.p, depth.p, first.p, colptr.p,
                                         rowptr.p, drop_tol, Kc.p, Kr.p);
    if (e) return fail(SIM_E_CUDA, "device inverse: %s", cudaGetErrorString((cudaError_t)e));
    CK(cudaMemcpyAsync(H->K.Kcol.data(), Kc.p, K.nnz * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(H->K.Krow.data(), Kr.p, K.nnz * sizeof(float), cudaMemcpyDeviceToHost, st));
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
    if ((int64_t)nf * H->S >= (int64_t)INT32_MAX / 4)
        return fail(SIM_E_LIMIT, "n_free x n_instances exceeds the int32 index range");
    // phase timings of the precompute (sim_stats.build_phase_seconds)
    auto tp = std::chrono::steady_clock::now();
    auto lap = [&](int k) {
        const auto now = std::chrono::steady_clock::now();
        H->build_phase[k] = std::chrono::duration<double>(now - tp).count();
        tp = now;
    };
    simhost::Csr A = simhost::assemble_Av(nv, H->n_t, H->T.data(), H->rd, H->h, vid, nf);
    lap(0);
    std::vector<double> coords(3 * (size_t)nf);
    for (int k = 0; k < nf; ++k)
        for (int d = 0; d < 3; ++d) coords[3 * k + d] = H->X[3 * (size_t)freev[k] + d];
    std::vector<int32_t> nd = simhost::nested_dissection(A, coords);
    lap(1);
    simhost::Csr C = simhost::permute_sym(A, nd);
    std::vector<int32_t> par = simhost::etree(C);
    std::vector<int32_t> post = simhost::postorder(par);
    std::vector<int32_t> perm(nf);   // perm[new] = free-local old index
    for (int k = 0; k < nf; ++k) perm[k] = nd[post[k]];
    C = simhost::permute_sym(A, perm);
    par = simhost::etree(C);
    simhost::Factor F;
    const bool chol_ok = simhost::cholesky(C, par, F);
    lap(2);
    if (!chol_ok)
        return fail(SIM_E_NOT_SPD, "non-positive pivot at column %d", F.bad_col);
    H->nnzL = (int64_t)F.Lp[nf];
    int nthr = (int)std::max(1u, std::thread::hardware_concurrency());
    if (H->host_only) {
        simhost::sparse_inverse(F, drop_tol, H->K, nthr);
        H->inverse_on_device = false;
    } else {   // K = L^-1 on the device (bitwise the host result), values read back for the tile layouts
        simhost::sparse_inverse_structure(F, H->K);
        int rc = device_inverse(H, F, drop_tol);
        if (rc) return rc;
        H->inverse_on_device = true;
    }
    lap(3);
    if (H->K.nnz >= (int64_t)INT32_MAX)
        return fail(SIM_E_LIMIT, "nnz(K) = %lld exceeds the int32 offset limit", (long long)H->K.nnz);
    simhost::trim_dropped(H->K);   // kept skyline (drop tolerance, reading A25)
    H->nnz_kept = 0;
    for (float q : H->K.Krow) H->nnz_kept += q != 0.f;
    {   // pass-1 items: <= 32 rows x p1cols columns (SIM_P1_ITEM_COLS overrides, multiple of 32)
        int p1cols = 512;   // 1024: 9 % slower pass 1 on cfg3 (the largest items set the tail), 256 / 128 slower too
        if (const char* e = getenv("SIM_P1_ITEM_COLS")) p1cols = std::max(32, atoi(e) / 32 * 32);
        simhost::build_worklists(H->K, H->wl, p1cols);
    }
    simhost::build_tiles(H->K, H->wl, H->T1h, H->T2h);
    if (H->S > 1) {
        H->bparts = simhost::build_batched(H->K, H->wl, 64, H->bu1, H->T1ph, H->bu2, H->bblocks1);
        int ut = 96;   // tiles per plane unit (SIM_PL_UNIT_TILES overrides; 48 / 64 / 128 / 192: pass 1 7 / 2 / 3 / 8 % slower)
        if (const char* e = getenv("SIM_PL_UNIT_TILES")) ut = std::max(4, atoi(e));
        simhost::build_plane_units(H->K, ut, H->pu);
    }
    lap(4);
    H->n_f = nf;
    H->int2orig.assign(nv, -1);
    H->orig2int.assign(nv, -1);
    for (int k = 0; k < nf; ++k) H->int2orig[k] = freev[perm[k]];
    int q = nf;
    for (int i = 0; i < nv; ++i)
        if (H->fixed[i]) H->int2orig[q++] = i;
    for (int k = 0; k < nv; ++k) H->orig2int[H->int2orig[k]] = k;
    // etree components (trees of the forest: one per connected object); parent[i] > i in postorder
    H->comp_root.assign(nf, -1);
    for (int i = nf - 1; i >= 0; --i) H->comp_root[i] = H->K.parent[i] < 0 ? i : H->comp_root[H->K.parent[i]];
    H->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!H->host_only) {
        int rc = upload_all(H);
        if (rc) return rc;
    }
    H->state = 1;
    return SIM_OK;
}

// ---------------------------------------------------------------------------
// contacts: validated per instance on the host, committed to the device for all
// instances at once (packed arrays + batched Delassus) before the next step
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

// validate one instance's contacts and build its local arrays; returns SIM_OK or an error
// code with the message in `err` (thread-safe: no globals touched)
static int build_inst(const sim_handle* H, const sim_contact* cs, int n, InstContacts& I, std::string& err) {
    char buf[256];
    auto bad = [&](int code, const char* fmt, int c, int v = 0) {
        snprintf(buf, sizeof buf, fmt, c, v);
        err = buf;
        return code;
    };
    if (n < 0 || (n > 0 && !cs)) { err = "bad contact array"; return SIM_E_INVALID; }
    I = InstContacts();
    I.hc.resize(n);
    std::vector<int32_t> verts;
    for (int c = 0; c < n; ++c) {
        const sim_contact& s = cs[c];
        if (s.kind != 0 && s.kind != 1) return bad(SIM_E_INVALID, "contact %d: kind must be 0 or 1", c);
        if (s.n_verts < 1 || s.n_verts > 4) return bad(SIM_E_INVALID, "contact %d: 1..4 vertices", c);
        double nn = std::sqrt(s.normal[0] * s.normal[0] + s.normal[1] * s.normal[1] + s.normal[2] * s.normal[2]);
        if (!(std::fabs(nn - 1.0) < 1e-6)) return bad(SIM_E_INVALID, "contact %d: normal not unit", c);
        if (!(s.mu >= 0) || !std::isfinite(s.mu)) return bad(SIM_E_INVALID, "contact %d: mu must be >= 0", c);
        if (!(s.compliance >= 0)) return bad(SIM_E_INVALID, "contact %d: compliance must be >= 0", c);
        if (!std::isfinite(s.offset)) return bad(SIM_E_INVALID, "contact %d: offset not finite", c);
        DContact& d = I.hc[c];
        memset(&d, 0, sizeof d);
        d.kind = s.kind;
        d.nv = s.n_verts;
        for (int q = 0; q < s.n_verts; ++q) {
            if (s.verts[q] < 0 || s.verts[q] >= H->n_v) return bad(SIM_E_INVALID, "contact %d: vertex out of range", c);
            if (H->fixed[s.verts[q]]) return bad(SIM_E_INVALID, "contact %d: vertex %d is pinned", c, s.verts[q]);
            if (!std::isfinite(s.weights[q])) return bad(SIM_E_INVALID, "contact %d: weight not finite", c);
            d.vtx[q] = H->orig2int[s.verts[q]];
            d.w[q] = s.weights[q];
            d.Mjj += s.weights[q] * s.weights[q] / H->rd.mass[s.verts[q]];   // [J M^-1 J^T]_jj, unit c
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
    const int ns = (int)verts.size();
    I.large = n > kMaxContacts || ns > kMaxSlots || cr_smem_bytes(n, ns) > kCrMaxSmem;
    if (I.large && (H->S > 1 || H->cr_mode == 1)) {
        snprintf(buf, sizeof buf,
                 "%d contacts on %d vertices exceed the cluster CR (<= %d contacts, <= %d vertices, %zu B shared "
                 "memory); larger sets need n_instances == 1 and the grid CR", n, ns, kMaxContacts, kMaxSlots,
                 kCrMaxSmem);
        err = buf;
        return SIM_E_LIMIT;
    }
    if ((int64_t)n * 3 >= (int64_t)INT32_MAX / 4) return bad(SIM_E_LIMIT, "too many contacts (%d)", n);
    // slot -> (contact, weight) lists in contact order
    std::vector<int> cnt(ns + 1, 0);
    auto slot_of = [&](int v) { return (int)(std::lower_bound(verts.begin(), verts.end(), v) - verts.begin()); };
    for (int c = 0; c < n; ++c)
        for (int q = 0; q < I.hc[c].nv; ++q) {
            I.hc[c].slot[q] = slot_of(I.hc[c].vtx[q]);
            cnt[I.hc[c].slot[q] + 1]++;
        }
    I.scp.assign(ns + 1, 0);
    for (int s = 0; s < ns; ++s) I.scp[s + 1] = I.scp[s] + cnt[s + 1];
    I.sci.resize(I.scp[ns]);
    I.scw.resize(I.scp[ns]);
    std::vector<int> fillp(I.scp.begin(), I.scp.end() - 1);
    for (int c = 0; c < n; ++c)
        for (int q = 0; q < I.hc[c].nv; ++q) {
            const int s = I.hc[c].slot[q];
            I.sci[fillp[s]] = c;
            I.scw[fillp[s]++] = (float)I.hc[c].w[q];
        }
    I.c9.resize(9 * (size_t)n);
    I.s0.resize(n);
    I.v0.resize(n);
    for (int q = 0; q < n; ++q) {
        for (int a = 0; a < 3; ++a)
            for (int d = 0; d < 3; ++d) I.c9[9 * q + 3 * a + d] = (float)I.hc[q].c[a][d];
        const bool single = I.hc[q].nv == 1 && I.hc[q].w[0] == 1.0;
        I.s0[q] = single ? I.hc[q].slot[0] : -1;
        I.v0[q] = single ? I.hc[q].vtx[0] : -1;
    }
    I.c1.assign(ns, -1);
    for (int s = 0; s < ns; ++s)
        if (I.scp[s + 1] - I.scp[s] == 1 && I.s0[I.sci[I.scp[s]]] == s) I.c1[s] = I.sci[I.scp[s]];
    I.verts = std::move(verts);
    I.chain_total = 0;
    for (int s = 0; s < ns; ++s) I.chain_total += H->K.depth[I.verts[s]] + 1;
    return SIM_OK;
}

static int check_contact_call(sim_handle* H) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1) return fail(SIM_E_STATE, "build the sparse inverse first");
    if (H->host_only) return fail(SIM_E_STATE, "host-only handle");
    return SIM_OK;
}

static int commit_host(sim_handle* H);

extern "C" int sim_set_contacts(sim_handle* H, int32_t instance, const sim_contact* cs, int32_t n) {
    int rc = check_contact_call(H);
    if (rc) return rc;
    if (instance < 0 || instance >= H->S) return fail(SIM_E_INVALID, "instance %d out of range [0, %d)", instance, H->S);
    auto th0 = std::chrono::steady_clock::now();
    InstContacts I;
    std::string err;
    rc = build_inst(H, cs, n, I, err);
    if (rc) return fail(rc, "%s", err.c_str());
    compute_carry(H->ic[instance], I);
    H->ic[instance] = std::move(I);
    H->dirty = true;
    H->set_contacts_host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count();
    // every instance's set is now known: pack and start the upload right away (it overlaps the
    // frames already enqueued); the device half runs at the next step
    if (H->S == 1) return commit_host(H);
    return SIM_OK;
}

static Params make_params(const sim_handle* H);

extern "C" int sim_detect_contacts(sim_handle* H, int32_t inst, const sim_obstacle* obs, int32_t nobs,
                                   const int32_t* cand, int32_t ncand, double margin, int32_t* n_found) {
    int rc = check_contact_call(H);
    if (rc) return rc;
    if (inst < 0 || inst >= H->S) return fail(SIM_E_INVALID, "instance %d out of range [0, %d)", inst, H->S);
    if (nobs < 0 || ncand < 0 || (nobs > 0 && !obs) || (ncand > 0 && !cand))
        return fail(SIM_E_INVALID, "bad obstacle or candidate arrays");
    if (!(margin >= 0) || !std::isfinite(margin)) return fail(SIM_E_INVALID, "margin must be >= 0");
    std::vector<DObstacle> dob(nobs);
    for (int o = 0; o < nobs; ++o) {
        const sim_obstacle& q = obs[o];
        if (q.kind < 0 || q.kind > 2) return fail(SIM_E_INVALID, "obstacle %d: kind must be 0, 1 or 2", o);
        if (!(q.radius >= 0) || !(q.mu >= 0)) return fail(SIM_E_INVALID, "obstacle %d: radius and mu must be >= 0", o);
        if (q.kind == 0) {
            const double nn = std::sqrt(q.b[0] * q.b[0] + q.b[1] * q.b[1] + q.b[2] * q.b[2]);
            if (!(std::fabs(nn - 1.0) < 1e-6)) return fail(SIM_E_INVALID, "obstacle %d: plane normal not unit", o);
        }
        DObstacle& d = dob[o];
        d.kind = q.kind;
        d.pad = 0;
        for (int k = 0; k < 3; ++k) { d.a[k] = q.a[k]; d.b[k] = q.b[k]; d.v[k] = q.velocity[k]; }
        d.radius = q.radius;
        d.mu = q.mu;
    }
    std::vector<int32_t> ci;   // internal ids of the free candidates, candidate order
    std::vector<int32_t> co;
    for (int c = 0; c < ncand; ++c) {
        if (cand[c] < 0 || cand[c] >= H->n_v) return fail(SIM_E_INVALID, "candidate %d out of range", c);
        if (H->fixed[cand[c]]) continue;
        ci.push_back(H->orig2int[cand[c]]);
        co.push_back(cand[c]);
    }
    const int nc = (int)ci.size();
    DBuf<DObstacle> dobs;
    DBuf<int32_t> dci;
    DBuf<int> dbest;
    DBuf<double> dgap;
    DBuf<double3> dn, dp;
    CK(dobs.alloc(std::max(nobs, 1))); CK(dci.alloc(std::max(nc, 1))); CK(dbest.alloc(std::max(nc, 1)));
    CK(dgap.alloc(std::max(nc, 1))); CK(dn.alloc(std::max(nc, 1))); CK(dp.alloc(std::max(nc, 1)));
    cudaStream_t st = H->stream;
    CK(dobs.upload(dob.data(), nobs, st));
    CK(dci.upload(ci.data(), nc, st));
    launch_proximity(st, make_params(H), H->x.p, inst, dci.p, nc, dobs.p, nobs, margin, dbest.p, dgap.p, dn.p, dp.p);
    CK(cudaGetLastError());
    std::vector<int> best(nc);
    std::vector<double3> hn(nc), hp(nc);
    CK(cudaStreamSynchronize(st));
    if (nc) {
        CK(cudaMemcpy(best.data(), dbest.p, nc * sizeof(int), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hn.data(), dn.p, nc * sizeof(double3), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hp.data(), dp.p, nc * sizeof(double3), cudaMemcpyDeviceToHost));
    }
    std::vector<sim_contact> cs;
    for (int c = 0; c < nc; ++c) {
        if (best[c] < 0) continue;
        const DObstacle& o = dob[best[c]];
        sim_contact k;
        memset(&k, 0, sizeof k);
        k.kind = 0;
        k.n_verts = 1;
        k.verts[0] = co[c];
        k.weights[0] = 1.0;
        const double n[3] = {hn[c].x, hn[c].y, hn[c].z}, p[3] = {hp[c].x, hp[c].y, hp[c].z};
        for (int d = 0; d < 3; ++d) { k.normal[d] = n[d]; k.obstacle_velocity[d] = o.v[d]; }
        k.offset = n[0] * p[0] + n[1] * p[1] + n[2] * p[2];
        k.mu = o.mu;
        cs.push_back(k);
    }
    rc = sim_set_contacts(H, inst, cs.data(), (int32_t)cs.size());
    if (rc) return rc;
    if (n_found) *n_found = (int32_t)cs.size();
    return SIM_OK;
}

extern "C" int sim_get_contacts(sim_handle* H, int32_t inst, sim_contact* out, int32_t cap, int32_t* n) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (inst < 0 || inst >= H->S) return fail(SIM_E_INVALID, "instance %d out of range [0, %d)", inst, H->S);
    const InstContacts& I = H->ic[inst];
    const int nc = (int)I.hc.size();
    if (n) *n = nc;
    if (!out) return SIM_OK;
    if (cap < nc) return fail(SIM_E_INVALID, "capacity %d < %d contacts", cap, nc);
    for (int c = 0; c < nc; ++c) {
        const DContact& d = I.hc[c];
        sim_contact& k = out[c];
        memset(&k, 0, sizeof k);
        k.kind = d.kind;
        k.n_verts = d.nv;
        for (int q = 0; q < d.nv; ++q) { k.verts[q] = H->int2orig[d.vtx[q]]; k.weights[q] = d.w[q]; }
        for (int e = 0; e < 3; ++e) {
            k.normal[e] = d.c[0][e];
            k.tangent1[e] = d.c[1][e];
            k.tangent2[e] = d.c[2][e];
        }
        k.offset = d.dn;
        k.mu = d.mu;
        k.compliance = d.e;
        // obstacle velocity is stored as its tangential projections d_f = t . v only
        for (int e = 0; e < 3; ++e) k.obstacle_velocity[e] = d.df1 * d.c[1][e] + d.df2 * d.c[2][e];
    }
    return SIM_OK;
}

extern "C" int sim_set_contacts_batch(sim_handle* H, int32_t first, int32_t count, const int32_t* counts,
                                      const sim_contact* cs) {
    int rc = check_contact_call(H);
    if (rc) return rc;
    if (first < 0 || count < 0 || first + count > H->S) return fail(SIM_E_INVALID, "instance range out of bounds");
    if (count > 0 && !counts) return fail(SIM_E_INVALID, "null counts");
    auto th0 = std::chrono::steady_clock::now();
    std::vector<int64_t> at(count + 1, 0);
    for (int i = 0; i < count; ++i) {
        if (counts[i] < 0) return fail(SIM_E_INVALID, "negative count for instance %d", first + i);
        at[i + 1] = at[i] + counts[i];
    }
    if (at[count] > 0 && !cs) return fail(SIM_E_INVALID, "null contacts");
    std::vector<InstContacts> tmp(count);
    std::vector<int> codes(count, SIM_OK);
    std::vector<std::string> errs(count);
#pragma omp parallel for schedule(dynamic, 4)
    for (int i = 0; i < count; ++i) {
        codes[i] = build_inst(H, cs + at[i], counts[i], tmp[i], errs[i]);
        if (codes[i] == SIM_OK) compute_carry(H->ic[first + i], tmp[i]);
    }
    for (int i = 0; i < count; ++i)
        if (codes[i]) return fail(codes[i], "instance %d: %s", first + i, errs[i].c_str());
    for (int i = 0; i < count; ++i) H->ic[first + i] = std::move(tmp[i]);
    H->dirty = true;
    H->set_contacts_host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count();
    if (count == H->S) return commit_host(H);   // all instances set: pack + upload now (see sim_set_contacts)
    return SIM_OK;
}

static InstOff inst_off(sim_handle* H) {
    return InstOff{H->coff.p, H->soff.p, H->gaoff.p, H->cls.p, H->csoff.p, H->goff.p, H->uoff.p, H->zoff.p,
                   H->cmoff.p, H->cmem.p};
}
static ClassSlots class_slots(sim_handle* H) { return ClassSlots{H->cvtx.p, H->ccls.p}; }
static Slots slots(sim_handle* H) { return Slots{H->slot_vtx.p, H->slot_inst.p, H->scp.p, H->sci.p, H->scw.p}; }
static CrContacts cr_contacts(sim_handle* H) { return CrContacts{H->cc9.p, H->dc.p, H->cs0.p, H->cv0.p, H->cc1.p}; }

static GcrData gcr_data(sim_handle* H) {
    GcrData g;
    g.c9 = H->cc9.p;
    g.G = H->G.p;
    g.rowoff = H->growoff.p;
    g.gs0 = H->gs0.p;
    g.gn = H->gn.p;
    g.r = H->g_r.p; g.p = H->g_p.p; g.Ap = H->g_Ap.p; g.z = H->g_z.p; g.Ar = H->g_Ar.p;
    g.W = H->g_W.p; g.q = H->g_q.p; g.part = H->g_part.p; g.sc = H->g_sc.p;
    g.cnt = H->g_cnt.p;
    g.gram_items = H->g_items.p;
    g.n_gram_items = H->n_g_items;
    g.nblk = 0;
    return g;
}

static Params make_params(const sim_handle* H) {
    Params P;
    P.n_v = H->n_v;
    P.n_f = H->n_f;
    P.n_t = H->n_t;
    P.S = H->S;
    P.h = H->h;
    for (int d = 0; d < 3; ++d) P.g[d] = H->mat.gravity[d];
    P.vpin = H->vpin.p;
    P.model = H->mat.model;
    P.k = (float)H->kproj;
    P.mu = (float)H->mu_l;
    P.lam = (float)H->lam_l;
    P.C = H->C;
    P.NS = H->NS;
    P.nc_max = H->nc_max;
    P.ns_max = H->ns_max;
    P.NCL = H->NCL;
    P.CS = H->CS;
    P.cm_max = H->cm_max;
    P.cr_iters = H->mat.cr_iterations;
    P.ncp = H->ncp;
    P.len_scale = H->len_scale;
    P.warm = H->warm;
    P.precond = H->precond;
    P.pair_local = H->local_mode == 0 ? 1 : 0;
    return P;
}

// pack every instance's contacts, upload them asynchronously and build the per-contact-set
// device data (chains, row lists, Delassus Gram, D_jj) for all instances in batched launches
static int commit_device(sim_handle* H);

// host half of a contact commit: classes, layouts, packing into pinned staging and one
// asynchronous H2D copy of the whole arena (enqueued on the handle's stream)
static int commit_host(sim_handle* H) {
    if (!H->dirty) return SIM_OK;
    const int S = H->S, nf = H->n_f;
    cudaStream_t st = H->stream;
    // slot-set classes: instances with equal contact-vertex sets (hash, then exact compare)
    std::vector<int> cls(S), rep;                 // class of instance, representative of class
    {
        std::unordered_map<uint64_t, std::vector<int>> byhash;
        for (int i = 0; i < S; ++i) {
            const std::vector<int32_t>& v = H->ic[i].verts;
            uint64_t hsh = 1469598103934665603ull ^ v.size();
            for (int32_t q : v) hsh = (hsh ^ (uint64_t)(uint32_t)q) * 1099511628211ull;
            std::vector<int>& cand = byhash[hsh];
            int found = -1;
            for (int k : cand)
                if (H->ic[rep[k]].verts == v) { found = k; break; }
            if (found < 0) {
                found = (int)rep.size();
                rep.push_back(i);
                cand.push_back(found);
            }
            cls[i] = found;
        }
    }
    const int NCL = (int)rep.size();
    // grid CR: one scene whose contact set exceeds the cluster CR (or forced); the Delassus Gram
    // is stored per etree component holding contact slots (zero across components, Theorem 1)
    const bool grid = S == 1 && !H->ic[0].hc.empty() && (H->cr_mode == 2 || H->ic[0].large);
    std::vector<int> gcs(1, 0);
    std::vector<int64_t> ggo(1, 0);
    int ngmax = 0;
    if (grid) {
        const std::vector<int32_t>& v = H->ic[0].verts;
        for (size_t q = 1; q < v.size(); ++q)
            if (H->comp_root[v[q]] != H->comp_root[v[q - 1]]) gcs.push_back((int)q);
        gcs.push_back((int)v.size());
        for (size_t g = 0; g + 1 < gcs.size(); ++g) {
            const int n = gcs[g + 1] - gcs[g];
            ggo.push_back(ggo.back() + (int64_t)n * n);
            ngmax = std::max(ngmax, n);
        }
    }
    const int NG = (int)gcs.size() - 1;
    // Gram reuse: every class maps to the previous class of its representative instance
    // (not while the previous commit's device half is pending: G does not hold that commit's
    // blocks yet, while prev_* already describes them)
    bool reuse = H->schur_reuse && !grid && H->have_prev && !H->dev_pending && (int)H->prev_cls_of_inst.size() == S;
    std::vector<int> rmap_h, pns_h(NCL, 0);
    std::vector<int64_t> pgoff_h(NCL, 0);
    std::vector<int2> news_h;
    if (reuse) {
        for (int k = 0; k < NCL && reuse; ++k) {
            const int ko = H->prev_cls_of_inst[rep[k]];
            if (ko < 0 || ko >= (int)H->prev_cls_verts.size()) { reuse = false; break; }
            const std::vector<int32_t>& vo = H->prev_cls_verts[ko];
            const std::vector<int32_t>& vn = H->ic[rep[k]].verts;
            size_t q = 0;
            for (size_t sidx = 0; sidx < vn.size(); ++sidx) {   // both lists ascending
                while (q < vo.size() && vo[q] < vn[sidx]) ++q;
                const int m = (q < vo.size() && vo[q] == vn[sidx]) ? (int)q : -1;
                rmap_h.push_back(m);
                if (m < 0) news_h.push_back(make_int2(k, (int)sidx));
            }
            pgoff_h[k] = H->prev_goff[ko];
            pns_h[k] = (int)vo.size();
        }
        if (!reuse) { rmap_h.clear(); news_h.clear(); }
    }
    if (reuse) {   // keep the previous blocks: G may be reallocated below
        bool g2 = false;
        CK(H->Gprev.ensure(std::max<int64_t>(H->prev_gsize, 1), g2));
        if (H->prev_gsize) CK(cudaMemcpyAsync(H->Gprev.p, H->G.p, H->prev_gsize * sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
    std::vector<int> cmoff(NCL + 1, 0), cmem(S);
    for (int i = 0; i < S; ++i) cmoff[cls[i] + 1]++;
    for (int k = 0; k < NCL; ++k) cmoff[k + 1] += cmoff[k];
    {
        std::vector<int> fillm(cmoff.begin(), cmoff.end() - 1);
        for (int i = 0; i < S; ++i) cmem[fillm[cls[i]]++] = i;
    }
    std::vector<int> coff(S + 1, 0), soff(S + 1, 0), csoff(NCL + 1, 0), uoff(NCL + 1, 0);
    std::vector<int64_t> gaoff(S + 1, 0), goff(NCL + 1, 0), zoff(NCL + 1, 0);
    int ncm = 0, nsm = 0, um = 0, cmm = 0;
    for (int i = 0; i < S; ++i) {
        const InstContacts& I = H->ic[i];
        const int n = (int)I.hc.size(), ns = (int)I.verts.size();
        coff[i + 1] = coff[i] + n;
        soff[i + 1] = soff[i] + ns;
        gaoff[i + 1] = gaoff[i] + (grid ? 0 : (int64_t)ns * ns);
        ncm = std::max(ncm, n);
        nsm = std::max(nsm, ns);
    }
    for (int k = 0; k < NCL; ++k) {
        const InstContacts& I = H->ic[rep[k]];
        const int ns = (int)I.verts.size();
        csoff[k + 1] = csoff[k] + ns;
        goff[k + 1] = goff[k] + (grid ? ggo.back() : (int64_t)ns * ns);
        zoff[k + 1] = zoff[k] + I.chain_total;
        const int urows = (int)std::min<int64_t>(nf, I.chain_total);
        uoff[k + 1] = uoff[k] + urows;
        um = std::max(um, urows);
        cmm = std::max(cmm, cmoff[k + 1] - cmoff[k]);
    }
    if (zoff[NCL] >= (int64_t)INT32_MAX) return fail(SIM_E_LIMIT, "total ancestor-chain entries exceed int32");
    const int Ct = coff[S], NSt = soff[S], CSt = csoff[NCL];
    // work items of the grouped kernels: chain dot (class slot, 32 members), scatter (class, 32 members);
    // member-chunk-major so one chunk's vectors stay in L2
    std::vector<int2> it_cd, it_sc;
    for (int m = 0; m < cmm; m += 32)
        for (int k = 0; k < NCL; ++k) {
            const int m0 = cmoff[k] + m;
            if (m0 >= cmoff[k + 1] || csoff[k + 1] == csoff[k]) continue;
            it_sc.push_back(make_int2(k, m0));
            const int gs = std::min(32, cmoff[k + 1] - m0);
            const int stride = gs == 1 ? 1 : 8;   // grouped chain dot: one warp per class slot, 8 per CTA
            for (int g = csoff[k]; g < csoff[k + 1]; g += stride) it_cd.push_back(make_int2(g, m0));
        }
    bool grew = false;
    const size_t cC = std::max(Ct, 1), cS = std::max(NSt, 1), cCS = std::max(CSt, 1);
    CK(H->G.ensure(std::max<int64_t>(goff[NCL], 1), grew));
    CK(H->GA.ensure(std::max<int64_t>(gaoff[S], 1), grew));
    CK(H->theta.ensure(3 * cC, grew)); CK(H->cdiag.ensure(3 * cC, grew));
    CK(H->hvec.ensure(3 * cC, grew)); CK(H->hl.ensure(3 * cC, grew)); CK(H->rho.ensure(3 * cC, grew));
    CK(H->phi_abs.ensure(cC, grew)); CK(H->dxt.ensure(3 * cS, grew)); CK(H->wz.ensure(3 * cS, grew));
    CK(H->act_idx.ensure(cS, grew)); CK(H->act_pos.ensure(cS, grew)); CK(H->act_con.ensure(cS, grew));
    if (S > 1) CK(H->wzT.ensure((size_t)std::max(nsm, 1) * S, grew));
    if (grid) {
        const size_t nb = (size_t)gcr_row_blocks(Ct);
        CK(H->g_r.ensure(3 * cC, grew)); CK(H->g_p.ensure(3 * cC, grew)); CK(H->g_Ap.ensure(3 * cC, grew));
        CK(H->g_z.ensure(3 * cC, grew)); CK(H->g_Ar.ensure(3 * cC, grew)); CK(H->g_W.ensure(3 * cS, grew));
        CK(H->g_q.ensure(3 * cS, grew)); CK(H->g_part.ensure(3 * std::max<size_t>(nb, 148), grew));
        CK(H->g_sc.ensure(8, grew));
        if (!H->g_cnt.p) {
            CK(H->g_cnt.alloc(1));
            CK(cudaMemset(H->g_cnt.p, 0, sizeof(int)));
        }
    }
    CK(H->chain_rows.ensure(std::max<int64_t>(zoff[NCL], 1), grew));
    CK(H->Zc.ensure(std::max<int64_t>(zoff[NCL], 1), grew)); CK(H->ulist.ensure(std::max(uoff[NCL], 1), grew));
    (void)cC; (void)cS; (void)cCS;
    // per-instance positions of the slot -> contact lists
    std::vector<int64_t> poff(S + 1, 0);
    for (int i = 0; i < S; ++i) poff[i + 1] = poff[i] + (int64_t)H->ic[i].sci.size();
    const int64_t NP = poff[S];
    // staging layout: every array packed straight into pinned memory (instances in parallel)
    struct Seg { size_t at, bytes; };
    size_t cur = 0;
    auto seg = [&](size_t bytes) { Seg s{cur, bytes}; cur = (cur + bytes + 255) & ~size_t(255); return s; };
    const size_t S1 = (size_t)S + 1, C1 = (size_t)NCL + 1;
    const Seg g_dc = seg(sizeof(DContact) * (size_t)Ct), g_c9 = seg(36 * (size_t)Ct), g_s0 = seg(4 * (size_t)Ct),
              g_v0 = seg(4 * (size_t)Ct), g_c1 = seg(4 * (size_t)NSt), g_sv = seg(4 * (size_t)NSt),
              g_si = seg(4 * (size_t)NSt), g_scp = seg(4 * ((size_t)NSt + 1)), g_sci = seg(4 * (size_t)NP),
              g_scw = seg(4 * (size_t)NP), g_ch = seg(4 * ((size_t)CSt + 1)), g_cv = seg(4 * (size_t)CSt),
              g_cc = seg(4 * (size_t)CSt), g_co = seg(4 * S1), g_so = seg(4 * S1), g_ga = seg(8 * S1),
              g_cl = seg(4 * (size_t)S), g_cso = seg(4 * C1), g_go = seg(8 * C1), g_uo = seg(4 * C1),
              g_zo = seg(8 * C1), g_cmo = seg(4 * C1), g_cm = seg(4 * (size_t)S), g_icd = seg(8 * it_cd.size()),
              g_isc = seg(8 * it_sc.size()), g_car = seg(4 * (size_t)Ct);
    const size_t NSg = grid ? (size_t)NSt : 0;
    const Seg g_rm = seg(4 * rmap_h.size()), g_pg = seg(8 * pgoff_h.size()), g_pn = seg(4 * pns_h.size()),
              g_nw = seg(8 * news_h.size());
    std::vector<int2> gitems;   // Gram matvec items: 32 consecutive rows of one group
    for (int g = 0; grid && g < NG; ++g)
        for (int q = gcs[g]; q < gcs[g + 1]; q += 32) gitems.push_back(make_int2(q, std::min(32, gcs[g + 1] - q)));
    const Seg g_gcs = seg(4 * gcs.size()), g_ggo = seg(8 * ggo.size()), g_grw = seg(8 * NSg), g_gs0 = seg(4 * NSg),
              g_gn = seg(4 * NSg), g_git = seg(8 * gitems.size());
    const size_t need = cur + 256;
    CK(H->arena.ensure(need, grew));
    {   // captured pointers change when the arena moves or any segment offset moves
        const std::vector<size_t> lay = {g_dc.at, g_c9.at, g_s0.at, g_v0.at, g_c1.at, g_sv.at, g_si.at, g_scp.at,
                                         g_sci.at, g_scw.at, g_ch.at, g_cv.at, g_cc.at, g_co.at, g_so.at, g_ga.at,
                                         g_cl.at, g_cso.at, g_go.at, g_uo.at, g_zo.at, g_cmo.at, g_cm.at, g_icd.at,
                                         g_isc.at, g_gcs.at, g_ggo.at, g_grw.at, g_gs0.at, g_gn.at, g_git.at,
                                         g_rm.at, g_pg.at, g_pn.at, g_nw.at, g_car.at};
        if (grew || lay != H->arena_layout) H->contact_gen++;
        H->arena_layout = lay;
    }
    {
        unsigned char* A = H->arena.p;
        H->dc.p = (DContact*)(A + g_dc.at); H->cc9.p = (float*)(A + g_c9.at); H->cs0.p = (int32_t*)(A + g_s0.at);
        H->cv0.p = (int32_t*)(A + g_v0.at); H->cc1.p = (int32_t*)(A + g_c1.at);
        H->slot_vtx.p = (int32_t*)(A + g_sv.at); H->slot_inst.p = (int32_t*)(A + g_si.at);
        H->scp.p = (int32_t*)(A + g_scp.at); H->sci.p = (int32_t*)(A + g_sci.at); H->scw.p = (float*)(A + g_scw.at);
        H->chain_off.p = (int32_t*)(A + g_ch.at); H->cvtx.p = (int32_t*)(A + g_cv.at);
        H->ccls.p = (int32_t*)(A + g_cc.at); H->coff.p = (int*)(A + g_co.at); H->soff.p = (int*)(A + g_so.at);
        H->gaoff.p = (int64_t*)(A + g_ga.at); H->cls.p = (int*)(A + g_cl.at); H->csoff.p = (int*)(A + g_cso.at);
        H->goff.p = (int64_t*)(A + g_go.at); H->uoff.p = (int*)(A + g_uo.at); H->zoff.p = (int64_t*)(A + g_zo.at);
        H->cmoff.p = (int*)(A + g_cmo.at); H->cmem.p = (int*)(A + g_cm.at); H->it_cd.p = (int2*)(A + g_icd.at);
        H->it_sc.p = (int2*)(A + g_isc.at);
        H->gcsoff.p = (int*)(A + g_gcs.at); H->ggoff.p = (int64_t*)(A + g_ggo.at);
        H->growoff.p = (int64_t*)(A + g_grw.at); H->gs0.p = (int*)(A + g_gs0.at); H->gn.p = (int*)(A + g_gn.at);
        H->g_items.p = (int2*)(A + g_git.at);
        H->rmap.p = (int*)(A + g_rm.at); H->pgoff.p = (int64_t*)(A + g_pg.at); H->pns.p = (int*)(A + g_pn.at);
        H->newslots.p = (int2*)(A + g_nw.at);
        H->carry.p = (int32_t*)(A + g_car.at);
    }
    if (!H->stage_free) CK(cudaEventCreateWithFlags(&H->stage_free, cudaEventDisableTiming));
    CK(cudaEventSynchronize(H->stage_free));   // the previous commit's copies are done
    if (need > H->stage_cap) {
        if (H->stage) CK(cudaFreeHost(H->stage));
        H->stage = nullptr;
        H->stage_cap = 0;
        CK(cudaMallocHost((void**)&H->stage, need + need / 4));
        H->stage_cap = need + need / 4;
    }
    unsigned char* B = H->stage;
    DContact* dc = (DContact*)(B + g_dc.at);
    float* c9 = (float*)(B + g_c9.at);
    int32_t *s0 = (int32_t*)(B + g_s0.at), *v0 = (int32_t*)(B + g_v0.at), *c1 = (int32_t*)(B + g_c1.at);
    int32_t *svtx = (int32_t*)(B + g_sv.at), *sinst = (int32_t*)(B + g_si.at), *scp = (int32_t*)(B + g_scp.at);
    int32_t* sci = (int32_t*)(B + g_sci.at);
    float* scw = (float*)(B + g_scw.at);
    int32_t* car = (int32_t*)(B + g_car.at);
    const bool have_dev = (int)H->coff_dev.size() == S + 1;
#pragma omp parallel for schedule(dynamic, 8)
    for (int i = 0; i < S; ++i) {
        const InstContacts& I = H->ic[i];
        const int cb = coff[i], sb = soff[i], n = (int)I.hc.size(), ns = (int)I.verts.size();
        const int pb = (int)poff[i];
        // lambda carry into the device layout of the last device commit (reading A10)
        for (int c = 0; c < n; ++c) {
            int src = -1;
            if (have_dev) {
                const int lc = I.dev ? c : (c < (int)I.carry.size() ? I.carry[c] : -1);
                if (lc >= 0 && lc < H->coff_dev[i + 1] - H->coff_dev[i]) src = H->coff_dev[i] + lc;
            }
            car[cb + c] = src;
        }
        for (int c = 0; c < n; ++c) {
            DContact d = I.hc[c];
            d.inst = i;
            for (int q = 0; q < d.nv; ++q) d.slot[q] += sb;
            dc[cb + c] = d;
            s0[cb + c] = I.s0[c] >= 0 ? I.s0[c] + sb : -1;
            v0[cb + c] = I.v0[c];
        }
        memcpy(c9 + 9 * (size_t)cb, I.c9.data(), 36 * (size_t)n);
        for (int s = 0; s < ns; ++s) {
            const int g = sb + s;
            c1[g] = I.c1[s] >= 0 ? I.c1[s] + cb : -1;
            svtx[g] = I.verts[s];
            sinst[g] = i;
            scp[g] = pb + I.scp[s];
        }
        for (size_t p = 0; p < I.sci.size(); ++p) {
            sci[pb + p] = I.sci[p] + cb;
            scw[pb + p] = I.scw[p];
        }
    }
    scp[NSt] = (int32_t)NP;
    {
        int32_t *choff = (int32_t*)(B + g_ch.at), *cv = (int32_t*)(B + g_cv.at), *cc = (int32_t*)(B + g_cc.at);
        const int32_t* depth = H->K.depth.data();
        int64_t ch = 0;
        for (int k = 0; k < NCL; ++k) {
            const std::vector<int32_t>& v = H->ic[rep[k]].verts;
            for (size_t s = 0; s < v.size(); ++s) {
                const int g = csoff[k] + (int)s;
                cv[g] = v[s];
                cc[g] = k;
                choff[g] = (int32_t)ch;
                ch += depth[v[s]] + 1;
            }
        }
        choff[CSt] = (int32_t)ch;
    }
    memcpy(B + g_co.at, coff.data(), 4 * S1);
    memcpy(B + g_so.at, soff.data(), 4 * S1);
    memcpy(B + g_ga.at, gaoff.data(), 8 * S1);
    memcpy(B + g_cl.at, cls.data(), 4 * (size_t)S);
    memcpy(B + g_cso.at, csoff.data(), 4 * C1);
    memcpy(B + g_go.at, goff.data(), 8 * C1);
    memcpy(B + g_uo.at, uoff.data(), 4 * C1);
    memcpy(B + g_zo.at, zoff.data(), 8 * C1);
    memcpy(B + g_cmo.at, cmoff.data(), 4 * C1);
    memcpy(B + g_cm.at, cmem.data(), 4 * (size_t)S);
    if (!it_cd.empty()) memcpy(B + g_icd.at, it_cd.data(), 8 * it_cd.size());
    if (!it_sc.empty()) memcpy(B + g_isc.at, it_sc.data(), 8 * it_sc.size());
    memcpy(B + g_gcs.at, gcs.data(), 4 * gcs.size());
    if (!gitems.empty()) memcpy(B + g_git.at, gitems.data(), 8 * gitems.size());
    if (!rmap_h.empty()) memcpy(B + g_rm.at, rmap_h.data(), 4 * rmap_h.size());
    if (!pgoff_h.empty()) memcpy(B + g_pg.at, pgoff_h.data(), 8 * pgoff_h.size());
    if (!pns_h.empty()) memcpy(B + g_pn.at, pns_h.data(), 4 * pns_h.size());
    if (!news_h.empty()) memcpy(B + g_nw.at, news_h.data(), 8 * news_h.size());
    H->n_g_items = (int)gitems.size();
    memcpy(B + g_ggo.at, ggo.data(), 8 * ggo.size());
    if (grid) {
        int64_t* rw = (int64_t*)(B + g_grw.at);
        int *s0g = (int*)(B + g_gs0.at), *sng = (int*)(B + g_gn.at);
        for (int g = 0; g < NG; ++g)
            for (int q = gcs[g]; q < gcs[g + 1]; ++q) {
                const int n = gcs[g + 1] - gcs[g];
                rw[q] = ggo[g] + (int64_t)(q - gcs[g]) * n;
                s0g[q] = gcs[g];
                sng[q] = n;
            }
    }
    H->h2d_contact_bytes = (int64_t)cur;
    // the whole layout in one H2D copy on the upload stream, then one D2D copy in stream order
    if (!H->up_stream) {
        CK(cudaStreamCreateWithFlags(&H->up_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&H->up_done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&H->up_free, cudaEventDisableTiming));
    }
    {
        bool grew_up = false;
        CK(H->arena_up.ensure(need, grew_up));
    }
    CK(cudaStreamWaitEvent(H->up_stream, H->up_free, 0));   // the previous commit's D2D has read arena_up
    CK(cudaMemcpyAsync(H->arena_up.p, B, cur, cudaMemcpyHostToDevice, H->up_stream));
    CK(cudaEventRecord(H->stage_free, H->up_stream));       // pinned staging reusable
    CK(cudaEventRecord(H->up_done, H->up_stream));
    CK(cudaStreamWaitEvent(st, H->up_done, 0));
    CK(cudaMemcpyAsync(H->arena.p, H->arena_up.p, cur, cudaMemcpyDeviceToDevice, st));
    CK(cudaEventRecord(H->up_free, st));
    H->NCL = NCL;
    H->CS = CSt;
    H->cm_max = cmm;
    H->n_it_cd = (int)it_cd.size();
    H->n_it_sc = (int)it_sc.size();
    H->gaoff_h = gaoff;
    H->C = Ct;
    H->NS = NSt;
    H->nc_max = ncm;
    H->ns_max = nsm;
    H->urows_max = um;
    H->coff_h = coff;
    H->soff_h = soff;
    H->grid = grid;
    H->NG = NG;
    H->ng_max = ngmax;
    // chain dot and scatter on the tensor cores: S > 1 instances all in one slot-set class
    H->tc_contact = S > 1 && NCL == 1 && Ct > 0 && H->kpass_mode != 1 && H->kpass_mode != 3;
    if (H->tc_contact && H->ic[rep[0]].verts != H->tc_verts) {   // tiles depend on K and the vertex set only
        simhost::ContactPasses cp;
        simhost::build_contact_passes(H->K, H->ic[rep[0]].verts, cp);
        // split the units over tile ranges until about two CTAs per SM are in flight (fp64 partials,
        // added in part order by the last part of each unit)
        auto split = [&](std::vector<simhost::BUnit>& units, bool cover_list, DBuf<double>& part,
                         DBuf<int>& cnt) -> cudaError_t {
            const int nch = (S + 127) / 128, nu = (int)units.size();
            int per_sm = 2;   // target CTAs in flight per SM (SIM_TS_CTAS_PER_SM overrides)
            if (const char* e = getenv("SIM_TS_CTAS_PER_SM")) per_sm = std::max(1, atoi(e));
            const int want = nu ? std::max(1, (per_sm * 148 + nu * nch - 1) / (nu * nch)) : 1;
            std::vector<simhost::BUnit> su;
            int nslot = 0;
            for (int b = 0; b < nu; ++b) {
                const simhost::BUnit u = units[b];
                const int p = std::max(1, std::min(want, u.ntiles));
                for (int k = 0; k < p; ++k) {
                    const int t0 = u.ntiles * k / p, t1 = u.ntiles * (k + 1) / p;
                    simhost::BUnit v = u;
                    if (cover_list) {   // chain pass: tiles walk the unit's cover-row list
                        v.list0 = u.list0 + 32 * t0;
                        v.nlist = std::min(u.nlist - 32 * t0, 32 * (t1 - t0));
                    } else {            // scatter pass: tiles walk consecutive slots
                        v.c0 = u.c0 + 32 * t0;
                    }
                    v.ntiles = t1 - t0;
                    v.toff = u.toff + (int64_t)t0 * 1024;
                    v.block = b;
                    v.nparts = p;
                    v.part = p > 1 ? nslot + k : 0;
                    v.pad = nslot;
                    su.push_back(v);
                }
                if (p > 1) nslot += p;
            }
            units.swap(su);
            cudaError_t e = part.alloc(std::max<size_t>((size_t)nslot * 3 * 32 * S, 1));
            if (e == cudaSuccess) e = cnt.alloc((size_t)std::max(1, nu) * nch);
            if (e == cudaSuccess) e = cudaMemsetAsync(cnt.p, 0, sizeof(int) * (size_t)std::max(1, nu) * nch, st);
            return e;
        };
        CK(split(cp.uc, true, H->tc_cpart, H->tc_ccnt));
        CK(split(cp.us, false, H->tc_spart, H->tc_scnt));
        std::vector<float> tc, ts;
        simhost::tc_tiles(cp.Tc, tc);
        simhost::tc_tiles(cp.Ts, ts);
        CK(H->tcu_c.alloc(std::max<size_t>(cp.uc.size(), 1))); CK(H->tcu_c.upload(cp.uc.data(), cp.uc.size(), st));
        CK(H->tcu_s.alloc(std::max<size_t>(cp.us.size(), 1))); CK(H->tcu_s.upload(cp.us.data(), cp.us.size(), st));
        CK(H->tc_cover.alloc(std::max<size_t>(cp.cover.size(), 1)));
        CK(H->tc_cover.upload(cp.cover.data(), cp.cover.size(), st));
        CK(H->tc_rows.alloc(std::max<size_t>(cp.rows.size(), 1))); CK(H->tc_rows.upload(cp.rows.data(), cp.rows.size(), st));
        CK(H->tc_Tc.alloc(std::max<size_t>(tc.size(), 1))); CK(H->tc_Tc.upload(tc.data(), tc.size(), st));
        CK(H->tc_Ts.alloc(std::max<size_t>(ts.size(), 1))); CK(H->tc_Ts.upload(ts.data(), ts.size(), st));
        CK(cudaStreamSynchronize(st));   // the host vectors die here
        H->tc_nuc = (int)cp.uc.size();
        H->tc_nus = (int)cp.us.size();
        H->tc_ns = (int)H->ic[rep[0]].verts.size();
        H->tc_verts = H->ic[rep[0]].verts;
        H->contact_gen++;   // captured pointers changed
    }
    H->pend_reuse = reuse;
    H->pend_nnew = (int)news_h.size();
    H->gram_rows_computed = reuse ? (int64_t)news_h.size() : CSt;
    H->gram_rows_reused = reuse ? (int64_t)CSt - (int64_t)news_h.size() : 0;
    // remember this commit's blocks for the next one
    H->have_prev = !grid;
    H->prev_cls_verts.assign(NCL, {});
    for (int k = 0; k < NCL; ++k) H->prev_cls_verts[k] = H->ic[rep[k]].verts;
    H->prev_goff.assign(goff.begin(), goff.end() - 1);
    H->prev_cls_of_inst = cls;
    H->prev_gsize = goff[NCL];
    H->dirty = false;
    H->dev_pending = true;
    return SIM_OK;
}

// device half: the per-contact-set kernels (chain rows, row lists, Delassus Gram, D_jj)
static int commit_device(sim_handle* H) {
    if (!H->dev_pending) return SIM_OK;
    cudaStream_t st = H->stream;
    const int S = H->S, nf = H->n_f, NCL = H->NCL, NG = H->NG, ngmax = H->ng_max;
    const bool grid = H->grid, reuse = H->pend_reuse;
    CK(cudaMemsetAsync(H->flag.p, 0, (size_t)NCL * nf, st));
    CK(cudaMemsetAsync(H->slotmap.p, 0xff, (size_t)nf * S * sizeof(int32_t), st));
    CK(cudaMemsetAsync(H->ucount.p, 0, 2 * (size_t)NCL * sizeof(int), st));
    CK(cudaMemsetAsync(H->cr_res.p, 0, S * sizeof(double), st));
    {   // lambda of the previous commit -> lam_prev, then carried into the new layout (reading A10)
        bool g1 = false, g2 = false;
        const size_t nold = 3 * (size_t)H->C_dev;
        if (nold) {
            CK(H->lam_prev.ensure(nold, g1));
            CK(cudaMemcpyAsync(H->lam_prev.p, H->lam.p, nold * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
        if (3 * (size_t)std::max(H->C, 1) > H->lam.n || !H->lam.p) {
            CK(cudaStreamSynchronize(st));   // the frames in flight and the copy above are done with lam
            CK(H->lam.ensure(3 * (size_t)std::max(H->C, 1), g2));
            H->contact_gen++;                // lam is a captured kernel argument
        }
        launch_carry_lambda(st, H->C, H->carry.p, nold ? H->lam_prev.p : nullptr, H->lam.p);
        H->coff_dev = H->coff_h;
        H->C_dev = H->C;
        for (InstContacts& I : H->ic) { I.dev = true; I.carry.clear(); }
    }
    Params P = make_params(H);
    const InstOff off = inst_off(H);
    const Slots sl = slots(H);
    const ClassSlots csl = class_slots(H);
    launch_chain_rows(st, P, csl, sl, H->chain_off.p, H->parent.p, H->ptop.p, H->chain_rows.p, H->flag.p,
                      H->slotmap.p);
    launch_ulist(st, P, off, H->flag.p, csl, H->meta.p, H->ucount.p, H->ulist.p, H->Krow.p, H->Zc.p);
    if (grid) {   // per-component Gram blocks: the class-slot kernel run over the groups
        Params Pg = P;
        Pg.NCL = NG;
        Pg.ns_max = ngmax;
        InstOff og = off;
        og.csoff = H->gcsoff.p;
        og.goff = H->ggoff.p;
        launch_delassus(st, Pg, og, csl, H->Kcol.p, H->colptr.p, H->depth.p, H->parent.p, H->ptop.p, H->G.p);
        launch_djj_grid(st, P, H->dc.p, gcr_data(H));
    } else {
        if (reuse)
            launch_gram_reuse(st, P, off, csl.vtx, H->rmap.p, H->pgoff.p, H->pns.p, H->Gprev.p, H->newslots.p,
                              H->pend_nnew, H->Kcol.p, H->colptr.p, H->depth.p, H->parent.p, H->ptop.p, H->G.p);
        else
            launch_delassus(st, P, off, csl, H->Kcol.p, H->colptr.p, H->depth.p, H->parent.p, H->ptop.p, H->G.p);
        launch_djj(st, P, off, H->dc.p, H->G.p);
    }
    CK(cudaGetLastError());
    H->dev_pending = false;
    return SIM_OK;   // asynchronous: the copies and kernels are ordered on the handle's stream
}

static int commit_contacts(sim_handle* H) {
    int rc = commit_host(H);
    if (rc) return rc;
    return commit_device(H);
}

// ---------------------------------------------------------------------------
// frame driver
// ---------------------------------------------------------------------------
static ContactState cstate(sim_handle* H) {
    return ContactState{H->lam.p, H->theta.p, H->cdiag.p, H->hvec.p, H->hl.p, H->dxt.p, H->wz.p, H->phi_abs.p,
                        H->cr_res.p, H->rho.p, H->S > 1 ? H->wzT.p : nullptr};
}

static void enqueue_kpass1(sim_handle* H, cudaStream_t st) {
    if (H->S == 1)
        launch_kpass1(st, (int)H->wl.p1.size(), H->p1.p, H->p1b.p, H->T1.p, H->u.p, H->y.p, H->part1.p,
                      H->counters.p);
    else if (H->kpass_mode != 1)
        launch_kpass1_pl(st, H->S, plane_sp(H->S), H->n_f, (int)H->pu.u1.size(), H->pu1d.p, H->Tpl1.p,
                         (const float*)H->u.p, (float*)H->y.p, H->ppart.p, H->pcounters.p, H->tc_drain);
    else
        launch_kpass1_batched(st, H->S, H->n_f, (int)H->bu1.size(), H->bu1d.p, H->T1p.p, (const float*)H->u.p,
                              (float*)H->y.p, H->part1.p, H->counters.p);
}
static void enqueue_kpass2(sim_handle* H, cudaStream_t st, double4* x, const double4* xt, double4* v, double inv_h,
                           int fin) {
    if (H->S == 1)
        launch_kpass2(st, (int)H->wl.p2b.size(), H->p2b.p, H->cover.p, H->T2.p, H->y.p, x, xt, v, inv_h, fin);
    else if (H->kpass_mode != 1)
        launch_kpass2_pl(st, H->S, plane_sp(H->S), H->n_f, (int)H->pu.u2.size(), H->pu2d.p, H->pcover.p, H->Tpl2.p,
                         (const float*)H->y.p, x, xt, v, inv_h, fin, H->tc_drain);
    else
        launch_kpass2_batched(st, H->S, H->n_f, (int)H->bu2.size(), H->bu2d.p, H->cover.p, H->T2.p,
                              (const float*)H->y.p, x, xt, v, inv_h, fin);
}

// enqueue one frame (predict + iters x L-G); returns kernel count or negative
enum { KK_PREDICT, KK_CONTACT, KK_LOCAL, KK_GATHER, KK_KPASS1, KK_CHAIN, KK_CR, KK_SCATTER, KK_KPASS2, KK_ACTIVE, KK_N };

static int enqueue_frame(sim_handle* H, int iters) {
    cudaStream_t st = H->stream;
    Params P = make_params(H);
    ContactState cs = cstate(H);
    const CrContacts ccr = cr_contacts(H);
    const CrActive act{H->act_na.p, H->act_idx.p, H->act_pos.p, H->act_con.p};
    const InstOff off = inst_off(H);
    const Slots sl = slots(H);
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
    launch_predict(st, P, H->x.p, H->xt.p, H->v.p, H->s.p, H->lam.p, 3 * H->C, H->vt.p, H->bad.p); nk++;
    if (H->poison_inst >= 0) launch_poison(st, H->x.p, H->poison_inst, H->S);   // test hook (not captured)
    const bool con = H->C > 0;
    for (int k = 0; k < iters; ++k) {
        // contact evaluation (+ active set) and the local step only read x^k: two graph
        // branches (serial when profiling, so the per-kernel events stay meaningful)
        const bool fork = con && !H->profiling;
        if (fork) {
            CKR(cudaEventRecord(H->fork_ev, st));
            CKR(cudaStreamWaitEvent(H->aux, H->fork_ev, 0));
            launch_contact_eval(H->aux, P, H->dc.p, H->x.p, H->xt.p, cs); nk++;
            if (!H->grid) { launch_active(H->aux, P, off, ccr, sl, cs, act, H->G.p, H->GA.p); nk += cr_cluster_size(P.S) > 1 ? 0 : 1; }
            CKR(cudaEventRecord(H->join_ev, H->aux));
        } else if (con) {
            MARK(KK_CONTACT); launch_contact_eval(st, P, H->dc.p, H->x.p, H->xt.p, cs); nk++;
            if (!H->grid) { MARK(KK_ACTIVE); launch_active(st, P, off, ccr, sl, cs, act, H->G.p, H->GA.p); nk += cr_cluster_size(P.S) > 1 ? 0 : 1; }
        }
        MARK(KK_LOCAL);
        launch_local(st, P, H->tet.p, H->Bm.p, H->hw2.p, H->x.p, H->fc.p, nullptr, H->admm ? H->du.p : nullptr,
                     k == 0); nk++;
        if (fork) CKR(cudaStreamWaitEvent(st, H->join_ev, 0));
        MARK(KK_GATHER);
        launch_gather(st, P, H->adjp.p, H->adj.p, H->fc.p, H->M.p, H->x.p, H->s.p, con ? H->slotmap.p : nullptr, sl,
                      H->hl.p, H->u.p, nullptr); nk++;
        MARK(KK_KPASS1);
        enqueue_kpass1(H, st); nk++;
        if (con) {
            MARK(KK_CHAIN);
            if (H->tc_contact)
                launch_chain_pass_ts(st, H->S, H->n_f, H->tc_nuc, H->tcu_c.p, H->tc_Tc.p, H->tc_cover.p, H->y.p, H->soff.p,
                                     ccr, H->x.p, cs, 1, H->tc_cpart.p, H->tc_ccnt.p);   // fold every tile: the Schur RHS is sensitive
            else
                launch_chain_dot(st, P, off, class_slots(H), H->Kcol.p, H->colptr.p, H->chain_off.p,
                                 H->chain_rows.p, H->y.p, sl, ccr, H->x.p, cs, H->n_it_cd, H->it_cd.p);
            nk++;
            MARK(KK_CR);
            if (H->grid) {
                int e = launch_gcr(st, P, gcr_data(H), H->dc.p, ccr, sl, H->x.p, cs);
                if (e) return -e;
                nk += gcr_kernels_per_iteration(P.cr_iters);
            } else {
                int e = launch_cr(st, P, off, H->dc.p, ccr, sl, H->G.p, H->GA.p, H->x.p, cs, act); nk++;
                if (e) return -e;
            }
            MARK(KK_SCATTER);
            if (H->tc_contact)
                launch_scatter_pass_ts(st, H->S, H->n_f, H->tc_ns, H->tc_nus, H->tcu_s.p, H->tc_Ts.p, H->tc_rows.p, H->wzT.p,
                                       H->y.p, 1, H->tc_spart.p, H->tc_scnt.p);
            else
                launch_scatter(st, P, H->urows_max, off, H->ucount.p, H->ulist.p, H->Zc.p, H->wz.p, H->wzT.p, H->y.p,
                               H->n_it_sc, H->it_sc.p);
            nk++;
        }
        MARK(KK_KPASS2);
        enqueue_kpass2(H, st, H->x.p, H->xt.p, H->v.p, 1.0 / H->h, k == iters - 1); nk++;
    }
    launch_finite_guard(st, H->n_v, H->S, H->x.p, H->v.p, H->xt.p, H->vt.p, H->bad.p, H->rollbacks.p); nk += 2;
    MARK(KK_N);
#undef MARK
#undef CKR
    return nk;
}

extern "C" int sim_set_ncp(sim_handle* H, int32_t ncp_function, int32_t preconditioner) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (ncp_function < 0 || ncp_function > 1) return fail(SIM_E_INVALID, "NCP function must be 0 (FB) or 1 (min-map)");
    if (preconditioner < 0 || preconditioner > 1)
        return fail(SIM_E_INVALID, "preconditioner must be 0 (Delassus) or 1 (mass inverse)");
    H->ncp = ncp_function;
    H->precond = preconditioner;
    return SIM_OK;   // Params are captured: the graph key includes both
}

extern "C" int sim_set_admm(sim_handle* H, int32_t on) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (on != 0 && on != 1) return fail(SIM_E_INVALID, "ADMM flag must be 0 or 1");
    if (on && H->state == 1 && !H->host_only && !H->du.p) CK(H->du.alloc((size_t)9 * H->n_t * H->S));
    if (on && H->state != 1) return fail(SIM_E_STATE, "build the sparse inverse first");
    H->admm = on;
    return SIM_OK;
}

static int check_instance(sim_handle* H, int inst);

extern "C" int sim_debug_poison(sim_handle* H, int32_t inst) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    H->poison_inst = inst;
    return SIM_OK;
}

extern "C" int sim_set_warm_start(sim_handle* H, int32_t on) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (on != 0 && on != 1) return fail(SIM_E_INVALID, "flag must be 0 or 1");
    H->warm = on;
    return SIM_OK;
}

extern "C" int sim_set_local_mode(sim_handle* H, int32_t mode) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (mode != 0 && mode != 1) return fail(SIM_E_INVALID, "mode must be 0 (paired) or 1 (scalar)");
    H->local_mode = mode;
    return SIM_OK;
}

extern "C" int sim_set_persistent(sim_handle* H, int32_t mode) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (mode != 0 && mode != 1) return fail(SIM_E_INVALID, "mode must be 0 (auto) or 1 (graph only)");
    H->persistent = mode;
    return SIM_OK;
}

// the persistent small-scene kernel applies: one instance, no contacts, plain PD, small enough for
// one CTA (its shared-memory vectors stay under 48 KB)
static bool small_path(const sim_handle* H) {
    if (H->persistent != 0 || H->S != 1 || H->C != 0 || H->admm || H->profiling || H->poison_inst >= 0) return false;
    const Params P = make_params(const_cast<sim_handle*>(H));
    return H->n_f + H->n_t <= 1024 && small_smem_bytes(P) <= 48 * 1024;
}

extern "C" int sim_set_schur_reuse(sim_handle* H, int32_t on) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (on != 0 && on != 1) return fail(SIM_E_INVALID, "flag must be 0 or 1");
    H->schur_reuse = on != 0;
    return SIM_OK;
}

extern "C" int sim_set_kpass_mode(sim_handle* H, int32_t mode) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    // mode 0 | 1; mode >= 16: tensor cores with (mode >> 4) tiles per fp32 TMEM accumulation (tuning)
    if (mode >= 16) {
        H->kpass_mode = 2;
        H->tc_drain = std::max(2, mode >> 4);
        return SIM_OK;
    }
    if (mode < 0 || mode > 3)
        return fail(SIM_E_INVALID, "K-pass mode must be 0 or 2 (tensor cores), 1 (CUDA-core FP32) or 3 (tensor-core K-passes, "
                    "CUDA-core contact passes)");
    H->kpass_mode = mode;
    return SIM_OK;
}

extern "C" int sim_set_cr_mode(sim_handle* H, int32_t mode) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (mode < 0 || mode > 2) return fail(SIM_E_INVALID, "CR mode must be 0 (auto), 1 (cluster) or 2 (grid)");
    if (mode == 1)
        for (const InstContacts& I : H->ic)
            if (I.large) return fail(SIM_E_LIMIT, "the current contact set needs the grid CR");
    if (mode == 2 && H->S > 1) return fail(SIM_E_LIMIT, "the grid CR needs n_instances == 1");
    H->cr_mode = mode;
    H->dirty = true;   // recommit (and recapture) with the new solver
    return SIM_OK;
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
    int rc = commit_contacts(H);
    if (rc) return rc;
    if (H->poison_inst >= 0) {   // sim_debug_poison: this one frame runs uncaptured with a NaN injected
        const int nk = enqueue_frame(H, iters);
        H->poison_inst = -1;
        if (nk < 0) return fail(SIM_E_CUDA, "launch failed: %s", cudaGetErrorString((cudaError_t)(-nk)));
        H->frames_done += 1;
        if (--frames == 0) return SIM_OK;
    }
    if (small_path(H)) {   // persistent small-scene driver: all frames in one launch
        const Params P = make_params(H);
        SmallArgs A{H->tet.p, H->Bm.p, H->hw2.p, H->M.p, H->adjp.p, H->adj.p, H->Krow.p, H->meta.p, H->Kcol.p,
                    H->colptr.p, H->parent.p, H->x.p, H->xt.p, H->v.p, H->s.p, H->vt.p, H->rollbacks.p};
        const int e = launch_small_frames(H->stream, P, A, frames, iters);
        if (e) return fail(SIM_E_CUDA, "launch failed: %s", cudaGetErrorString((cudaError_t)e));
        H->frames_done += frames;
        H->kernels_per_frame = 1;
        H->last_persistent = true;
        return SIM_OK;
    }
    H->last_persistent = false;
    const std::vector<int64_t> key = {iters, H->C, H->NS, H->nc_max, H->ns_max, H->urows_max, H->profiling,
                                      H->contact_gen, H->NCL, H->CS, H->n_it_cd, H->n_it_sc, H->grid, H->NG,
                                      H->ncp, H->precond, H->admm, H->kpass_mode, H->tc_drain, H->cr_mode, H->warm, H->local_mode,
                                      H->tc_contact};
    if (!H->gexec || key != H->gkey) {
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
        H->gkey = key;
        H->g_prof = H->profiling;
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
    if (H->rollbacks.p) {
        int n = 0;
        CK(cudaMemcpy(&n, H->rollbacks.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (n > 0) {
            CK(cudaMemset(H->rollbacks.p, 0, sizeof(int)));
            H->rollbacks_total += n;
            return fail(SIM_E_NONFINITE, "%d instance-frame(s) became non-finite and were rolled back to their "
                        "frame-start state", n);
        }
    }
    return SIM_OK;
}

extern "C" int sim_set_pin_velocity(sim_handle* H, const double v[3]) {
    if (!H || !v) return fail(SIM_E_INVALID, "null argument");
    for (int d = 0; d < 3; ++d)
        if (!std::isfinite(v[d])) return fail(SIM_E_INVALID, "pin velocity not finite");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "build the sparse inverse first");
    const size_t n = (size_t)(H->n_v - H->n_f) * H->S;
    if (n == 0) return SIM_OK;
    std::vector<double4> hv(n, make_double4(v[0], v[1], v[2], 0.0));
    CK(cudaStreamSynchronize(H->stream));
    CK(cudaMemcpy(H->vpin.p, hv.data(), n * sizeof(double4), cudaMemcpyHostToDevice));
    return SIM_OK;
}

extern "C" int sim_set_pins(sim_handle* H, int32_t inst, const double* xyz, int32_t n_pinned) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "build the sparse inverse first");
    if (inst < 0 || inst >= H->S) return fail(SIM_E_INVALID, "instance %d out of range [0, %d)", inst, H->S);
    const int np = H->n_v - H->n_f;
    if (n_pinned != np) return fail(SIM_E_INVALID, "%d targets given, the mesh has %d pinned vertices", n_pinned, np);
    if (np == 0) return SIM_OK;
    if (!xyz) return fail(SIM_E_INVALID, "null targets");
    for (int64_t i = 0; i < 3LL * np; ++i)
        if (!std::isfinite(xyz[i])) return fail(SIM_E_INVALID, "target %lld not finite", (long long)(i / 3));
    cudaStream_t st = H->stream;
    if (!H->pin_stage) {
        CK(H->pin_tgt.alloc(np));
        CK(cudaMallocHost((void**)&H->pin_stage, np * sizeof(double4)));
        CK(cudaEventCreateWithFlags(&H->pin_free, cudaEventDisableTiming));
        CK(cudaEventRecord(H->pin_free, st));
    }
    CK(cudaEventSynchronize(H->pin_free));   // the previous call's copy has left the staging buffer
    // compact order = ascending original id of the pinned vertices = internal ids n_f .. n_v - 1
    for (int p = 0; p < np; ++p) H->pin_stage[p] = make_double4(xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2], 0.0);
    CK(cudaMemcpyAsync(H->pin_tgt.p, H->pin_stage, np * sizeof(double4), cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(H->pin_free, st));
    launch_pin_targets(st, H->n_f, np, H->S, inst, H->h, H->x.p, H->pin_tgt.p, H->vpin.p);
    CK(cudaGetLastError());
    return SIM_OK;
}

static int check_instance(sim_handle* H, int inst) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    if (inst < 0 || inst >= H->S) return fail(SIM_E_INVALID, "instance %d out of range [0, %d)", inst, H->S);
    return SIM_OK;
}

// x [n_instances][n_vertices][3] (original vertex order) into a caller-pinned host buffer,
// asynchronously: a packing kernel on the handle's stream fills one of two device staging
// buffers, the copy stream moves it to the host while the following frames run
extern "C" int sim_get_positions_async(sim_handle* H, double* host_dst) {
    int rc = check_instance(H, 0);
    if (rc) return rc;
    if (!host_dst) return fail(SIM_E_INVALID, "null argument");
    const size_t n = (size_t)H->n_v * H->S * 3;
    if (!H->copy_stream) {
        CK(cudaStreamCreateWithFlags(&H->copy_stream, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            CK(cudaEventCreateWithFlags(&H->pos_ready[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&H->pos_copied[k], cudaEventDisableTiming));
            CK(cudaEventRecord(H->pos_copied[k], H->copy_stream));
            CK(H->pos_stage[k].alloc(n));
        }
        CK(H->o2i.alloc(H->n_v));
        CK(cudaMemcpy(H->o2i.p, H->orig2int.data(), H->n_v * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    const int k = H->pos_slot;
    CK(cudaStreamWaitEvent(H->stream, H->pos_copied[k], 0));   // staging k no longer being read
    launch_pack_positions(H->stream, H->x.p, H->o2i.p, H->n_v, H->S, H->pos_stage[k].p);
    CK(cudaGetLastError());
    CK(cudaEventRecord(H->pos_ready[k], H->stream));
    CK(cudaStreamWaitEvent(H->copy_stream, H->pos_ready[k], 0));
    CK(cudaMemcpyAsync(host_dst, H->pos_stage[k].p, n * sizeof(double), cudaMemcpyDeviceToHost, H->copy_stream));
    CK(cudaEventRecord(H->pos_copied[k], H->copy_stream));
    H->pos_last = k;
    H->pos_slot ^= 1;
    return SIM_OK;
}

extern "C" int sim_wait_positions(sim_handle* H, int32_t block_host) {
    if (!H) return fail(SIM_E_INVALID, "null handle");
    if (H->pos_last < 0) return SIM_OK;
    if (block_host) CK(cudaEventSynchronize(H->pos_copied[H->pos_last]));
    else CK(cudaStreamWaitEvent(H->stream, H->pos_copied[H->pos_last], 0));
    return SIM_OK;
}

// one instance's column of a [vertex][instance] double4 array
static cudaError_t copy_column_d2h(sim_handle* H, const double4* src, int inst, double4* dst) {
    return cudaMemcpy2D(dst, sizeof(double4), src + inst, sizeof(double4) * H->S, sizeof(double4), H->n_v,
                        cudaMemcpyDeviceToHost);
}
static cudaError_t copy_column_h2d(sim_handle* H, const double4* src, int inst, double4* dst) {
    return cudaMemcpy2D(dst + inst, sizeof(double4) * H->S, src, sizeof(double4), sizeof(double4), H->n_v,
                        cudaMemcpyHostToDevice);
}

extern "C" int sim_get_state(sim_handle* H, int32_t inst, double* x, double* v) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    std::vector<double4> hx(H->n_v), hv(H->n_v);
    CK(cudaStreamSynchronize(H->stream));
    if (x) CK(copy_column_d2h(H, H->x.p, inst, hx.data()));
    if (v) CK(copy_column_d2h(H, H->v.p, inst, hv.data()));
    for (int i = 0; i < H->n_v; ++i) {
        int o = H->int2orig[i];
        if (x) { x[3 * o] = hx[i].x; x[3 * o + 1] = hx[i].y; x[3 * o + 2] = hx[i].z; }
        if (v) { v[3 * o] = hv[i].x; v[3 * o + 1] = hv[i].y; v[3 * o + 2] = hv[i].z; }
    }
    return SIM_OK;
}

// positions of all instances: x [n_instances][n_vertices][3] (original vertex order)
extern "C" int sim_get_positions(sim_handle* H, double* x) {
    int rc = check_instance(H, 0);
    if (rc) return rc;
    if (!x) return fail(SIM_E_INVALID, "null argument");
    const size_t n = (size_t)H->n_v * H->S;
    std::vector<double4> hx(n);
    CK(cudaStreamSynchronize(H->stream));
    CK(cudaMemcpy(hx.data(), H->x.p, n * sizeof(double4), cudaMemcpyDeviceToHost));
    const int S = H->S, nv = H->n_v;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < S; ++i)
        for (int k = 0; k < nv; ++k) {
            const double4 a = hx[(size_t)k * S + i];
            double* o = x + ((size_t)i * nv + H->int2orig[k]) * 3;
            o[0] = a.x; o[1] = a.y; o[2] = a.z;
        }
    return SIM_OK;
}

// states of all instances: x, v [n_instances][n_vertices][3] (either may be NULL)
extern "C" int sim_set_states(sim_handle* H, const double* x, const double* v) {
    int rc = check_instance(H, 0);
    if (rc) return rc;
    const int S = H->S, nv = H->n_v;
    const size_t n3 = 3 * (size_t)nv * S;
    for (size_t i = 0; i < n3; ++i) {
        if (x && !std::isfinite(x[i])) return fail(SIM_E_INVALID, "x not finite");
        if (v && !std::isfinite(v[i])) return fail(SIM_E_INVALID, "v not finite");
    }
    CK(cudaStreamSynchronize(H->stream));
    std::vector<double4> h((size_t)nv * S);
    for (int pass = 0; pass < 2; ++pass) {
        const double* src = pass == 0 ? x : v;
        if (!src) continue;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < S; ++i)
            for (int k = 0; k < nv; ++k) {
                const double* a = src + ((size_t)i * nv + H->int2orig[k]) * 3;
                h[(size_t)k * S + i] = make_double4(a[0], a[1], a[2], 0.0);
            }
        CK(cudaMemcpy(pass == 0 ? H->x.p : H->v.p, h.data(), h.size() * sizeof(double4), cudaMemcpyHostToDevice));
    }
    // a new initial state starts from lambda = 0 (the multipliers are part of the state, A10)
    if (H->C_dev > 0) CK(cudaMemset(H->lam.p, 0, 3 * (size_t)H->C_dev * sizeof(double)));
    return SIM_OK;
}

extern "C" int sim_set_state(sim_handle* H, int32_t inst, const double* x, const double* v) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    for (int i = 0; i < 3 * H->n_v; ++i) {
        if (x && !std::isfinite(x[i])) return fail(SIM_E_INVALID, "x not finite");
        if (v && !std::isfinite(v[i])) return fail(SIM_E_INVALID, "v not finite");
    }
    std::vector<double4> hx(H->n_v), hv(H->n_v);
    for (int i = 0; i < H->n_v; ++i) {
        int o = H->int2orig[i];
        if (x) hx[i] = make_double4(x[3 * o], x[3 * o + 1], x[3 * o + 2], 0.0);
        if (v) hv[i] = make_double4(v[3 * o], v[3 * o + 1], v[3 * o + 2], 0.0);
    }
    CK(cudaStreamSynchronize(H->stream));
    if (x) CK(copy_column_h2d(H, hx.data(), inst, H->x.p));
    if (v) CK(copy_column_h2d(H, hv.data(), inst, H->v.p));
    if ((int)H->coff_dev.size() == H->S + 1) {   // this instance's multipliers restart from 0 (A10)
        const int c0 = H->coff_dev[inst], c1 = H->coff_dev[inst + 1];
        if (c1 > c0) CK(cudaMemset(H->lam.p + 3 * (size_t)c0, 0, 3 * (size_t)(c1 - c0) * sizeof(double)));
    }
    return SIM_OK;
}

// rows of an instance's device-committed contact set (1 per bilateral, 3 per unilateral contact)
static int lambda_rows(const InstContacts& I) {
    int rows = 0;
    for (const DContact& d : I.hc) rows += d.kind == 1 ? 1 : 3;
    return rows;
}

extern "C" int sim_get_lambda(sim_handle* H, int32_t inst, double* lam, int32_t cap, int32_t* n_rows) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    rc = commit_contacts(H);   // a pending commit carries lambda into the current set's layout
    if (rc) return rc;
    const InstContacts& I = H->ic[inst];
    const int nc = (int)I.hc.size();
    const int rows = lambda_rows(I);
    if (n_rows) *n_rows = rows;
    if (!lam) return SIM_OK;
    if (cap < rows) return fail(SIM_E_INVALID, "capacity %d < %d rows", cap, rows);
    std::vector<double> l(3 * (size_t)nc);
    CK(cudaStreamSynchronize(H->stream));
    if (nc) CK(cudaMemcpy(l.data(), H->lam.p + 3 * (size_t)H->coff_h[inst], l.size() * sizeof(double),
                          cudaMemcpyDeviceToHost));
    int r = 0;
    for (int c = 0; c < nc; ++c) {
        lam[r++] = l[3 * c];
        if (I.hc[c].kind != 1) {
            lam[r++] = l[3 * c + 1];
            lam[r++] = l[3 * c + 2];
        }
    }
    return SIM_OK;
}

extern "C" int sim_set_lambda(sim_handle* H, int32_t inst, const double* lam, int32_t n) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    rc = commit_contacts(H);
    if (rc) return rc;
    const InstContacts& I = H->ic[inst];
    const int nc = (int)I.hc.size();
    if (n != lambda_rows(I)) return fail(SIM_E_INVALID, "%d rows given, the contact set has %d", n, lambda_rows(I));
    if (n > 0 && !lam) return fail(SIM_E_INVALID, "null lambda");
    for (int j = 0; j < n; ++j)
        if (!std::isfinite(lam[j])) return fail(SIM_E_INVALID, "lambda row %d not finite", j);
    std::vector<double> l(3 * (size_t)nc, 0.0);
    int r = 0;
    for (int c = 0; c < nc; ++c) {
        l[3 * c] = lam[r++];
        if (I.hc[c].kind != 1) {
            l[3 * c + 1] = lam[r++];
            l[3 * c + 2] = lam[r++];
        }
    }
    CK(cudaStreamSynchronize(H->stream));
    if (nc) CK(cudaMemcpy(H->lam.p + 3 * (size_t)H->coff_h[inst], l.data(), l.size() * sizeof(double),
                          cudaMemcpyHostToDevice));
    return SIM_OK;
}

extern "C" int sim_get_stats(sim_handle* H, int32_t inst, sim_stats* o) {
    if (!H || !o) return fail(SIM_E_INVALID, "null argument");
    if (inst < -1 || inst >= H->S) return fail(SIM_E_INVALID, "instance %d out of range [-1, %d)", inst, H->S);
    memset(o, 0, sizeof *o);
    o->instance = inst;
    o->n_vertices = H->n_v;
    o->n_free = H->n_f;
    o->n_tets = H->n_t;
    o->nnz_K = H->K.nnz;
    {
        o->nnz_K_kept = H->nnz_kept;
        o->kpass_bytes = H->S == 1 ? (int64_t)(H->T1h.size() + H->T2h.size()) * 4
                                   : (int64_t)(H->pu.T1.size() + H->pu.T2.size()) * 4;
    }
    o->nnz_L = H->nnzL;
    o->etree_height = H->K.height;
    o->n_panels = H->K.panel_start.empty() ? 0 : (int)H->K.panel_start.size() - 1;
    o->n_instances = H->S;
    const int i0 = inst < 0 ? 0 : inst, i1 = inst < 0 ? H->S : inst + 1;
    int nc = 0, ns = 0;
    for (int i = i0; i < i1; ++i) { nc += (int)H->ic[i].hc.size(); ns += (int)H->ic[i].verts.size(); }
    o->n_contacts = nc;
    o->n_contact_vertices = ns;
    o->frames_done = H->frames_done;
    o->kernels_per_frame = H->kernels_per_frame;
    o->build_seconds = H->build_seconds;
    o->h2d_contact_bytes = H->h2d_contact_bytes;
    o->nonfinite_rollbacks = H->rollbacks_total;
    o->gram_rows_computed = H->gram_rows_computed;
    o->gram_rows_reused = H->gram_rows_reused;
    for (int k = 0; k < 5; ++k) o->build_phase_seconds[k] = H->build_phase[k];
    if (!H->host_only && H->rollbacks.p) {
        int n = 0;
        CK(cudaStreamSynchronize(H->stream));
        CK(cudaMemcpy(&n, H->rollbacks.p, sizeof(int), cudaMemcpyDeviceToHost));
        o->nonfinite_rollbacks += n;
    }
    o->last_cr_residual = -1;
    if (!H->host_only && H->state == 1 && H->C > 0 && !H->dirty && !H->dev_pending && H->frames_done > 0) {
        cudaStream_t st = H->stream;
        DBuf<int> dcls;
        DBuf<double> dcone, dgap;
        CK(dcls.alloc(H->C)); CK(dcone.alloc(H->C)); CK(dgap.alloc(H->C));
        launch_contact_stats(st, make_params(H), H->dc.p, H->x.p, H->xt.p, H->lam.p, dcls.p, dcone.p, dgap.p);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        const int c0 = H->coff_h[i0], c1 = H->coff_h[i1], n = c1 - c0;
        std::vector<double> r(H->S), ph(n), cone(n), gap(n);
        std::vector<int> cl(n);
        CK(cudaMemcpy(r.data(), H->cr_res.p, H->S * sizeof(double), cudaMemcpyDeviceToHost));
        if (n) {
            CK(cudaMemcpy(ph.data(), H->phi_abs.p + c0, n * sizeof(double), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(cl.data(), dcls.p + c0, n * sizeof(int), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(cone.data(), dcone.p + c0, n * sizeof(double), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(gap.data(), dgap.p + c0, n * sizeof(double), cudaMemcpyDeviceToHost));
        }
        o->last_cr_residual = *std::max_element(r.begin() + i0, r.begin() + i1);
        for (int k = 0; k < n; ++k) {
            o->max_abs_phi_n = std::max(o->max_abs_phi_n, ph[k]);
            if (cl[k] < 0) continue;
            o->n_active += cl[k] > 0;
            o->n_stick += cl[k] == 1;
            o->n_slip += cl[k] == 2;
            o->max_cone_violation = std::max(o->max_cone_violation, cone[k]);
            o->max_penetration = std::max(o->max_penetration, -gap[k]);
        }
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

// b, x_out: [n_instances][n_vertices][3]
extern "C" int sim_debug_apply_inverse(sim_handle* H, const double* b, double* xo) {
    if (!H || !b || !xo) return fail(SIM_E_INVALID, "null argument");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    const int nf = H->n_f, nv = H->n_v, S = H->S;
    const int Sp = plane_sp(S);
    std::vector<float4> hu(S == 1 ? (size_t)nf : ((size_t)3 * nf * Sp + 3) / 4, make_float4(0.f, 0.f, 0.f, 0.f));
    float* hp = reinterpret_cast<float*>(hu.data());   // S > 1: planes [3][nf][Sp]
    for (int i = 0; i < S; ++i)
        for (int k = 0; k < nf; ++k) {
            const double* bb = b + ((size_t)i * nv + H->int2orig[k]) * 3;
            if (S == 1) {
                hu[k] = make_float4((float)bb[0], (float)bb[1], (float)bb[2], 0.f);
            } else {
                for (int c = 0; c < 3; ++c) hp[(size_t)c * nf * Sp + (size_t)k * Sp + i] = (float)bb[c];
            }
        }
    DBuf<double4> dx;
    CK(dx.alloc((size_t)nf * S));
    cudaStream_t st = H->stream;
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(H->u.p, hu.data(), hu.size() * sizeof(float4), cudaMemcpyHostToDevice));
    CK(cudaMemset(dx.p, 0, (size_t)nf * S * sizeof(double4)));
    enqueue_kpass1(H, st);
    enqueue_kpass2(H, st, dx.p, nullptr, nullptr, 1.0, 0);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    std::vector<double4> hx((size_t)nf * S);
    CK(cudaMemcpy(hx.data(), dx.p, hx.size() * sizeof(double4), cudaMemcpyDeviceToHost));
    for (size_t q = 0; q < 3 * (size_t)nv * S; ++q) xo[q] = 0.0;
    for (int i = 0; i < S; ++i)
        for (int k = 0; k < nf; ++k) {
            double* o = xo + ((size_t)i * nv + H->int2orig[k]) * 3;
            const double4 a = hx[(size_t)k * S + i];
            o[0] = a.x; o[1] = a.y; o[2] = a.z;
        }
    return SIM_OK;
}

extern "C" int sim_debug_local(sim_handle* H, const double* x, const double* s, float* Pout, double* resid) {
    if (!H || !x || !s) return fail(SIM_E_INVALID, "null argument");
    if (H->state != 1 || H->host_only) return fail(SIM_E_STATE, "no device state");
    if (H->S != 1) return fail(SIM_E_STATE, "sim_debug_local needs a single-instance handle");
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
    launch_gather(st, P, H->adjp.p, H->adj.p, H->fc.p, H->M.p, dx.p, ds.p, nullptr, slots(H), nullptr, H->u.p, dr.p);
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
    return SIM_OK;
}

extern "C" int sim_debug_get_delassus(sim_handle* H, int32_t inst, int32_t* cv, float* G, int32_t cap) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    rc = commit_contacts(H);
    if (rc) return rc;
    const InstContacts& I = H->ic[inst];
    const int ns = (int)I.verts.size();
    if (cap < ns) return fail(SIM_E_INVALID, "capacity %d < %d contact vertices", cap, ns);
    CK(cudaStreamSynchronize(H->stream));
    if (cv) for (int s = 0; s < ns; ++s) cv[s] = H->int2orig[I.verts[s]];
    if (G && ns && H->grid) {
        std::vector<int> gcs(H->NG + 1);
        std::vector<int64_t> ggo(H->NG + 1);
        CK(cudaMemcpy(gcs.data(), H->gcsoff.p, gcs.size() * sizeof(int), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ggo.data(), H->ggoff.p, ggo.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
        std::fill(G, G + (size_t)ns * ns, 0.f);
        for (int g = 0; g < H->NG; ++g) {
            const int n = gcs[g + 1] - gcs[g];
            std::vector<float> blk((size_t)n * n);
            CK(cudaMemcpy(blk.data(), H->G.p + ggo[g], blk.size() * sizeof(float), cudaMemcpyDeviceToHost));
            for (int a = 0; a < n; ++a)
                for (int b = 0; b < n; ++b) G[(size_t)(gcs[g] + a) * ns + gcs[g] + b] = blk[(size_t)a * n + b];
        }
    } else if (G && ns) {
        int cl = 0;
        int64_t go = 0;
        CK(cudaMemcpy(&cl, H->cls.p + inst, sizeof(int), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&go, H->goff.p + cl, sizeof(int64_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(G, H->G.p + go, (size_t)ns * ns * sizeof(float), cudaMemcpyDeviceToHost));
    }
    return SIM_OK;
}

// contact scratch of the last evaluated L-G iteration: per row (3 per contact)
// theta, C diagonal, h-vector; per slot dxt = (K^T y) at the slot vertex; slot vertices
extern "C" int sim_debug_contact_state(sim_handle* H, int32_t inst, double* theta, double* cdiag, double* hvec,
                                       double* dxt, int32_t* slot_vertex, double* djj) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    if (H->dirty || H->dev_pending) return fail(SIM_E_STATE, "contacts changed since the last step");
    CK(cudaStreamSynchronize(H->stream));
    const InstContacts& I = H->ic[inst];
    const int nc = (int)I.hc.size(), ns = (int)I.verts.size();
    const size_t cb = H->coff_h[inst], sb = H->soff_h[inst];
    size_t m = 3 * (size_t)nc;
    if (theta && m) CK(cudaMemcpy(theta, H->theta.p + 3 * cb, m * sizeof(double), cudaMemcpyDeviceToHost));
    if (cdiag && m) CK(cudaMemcpy(cdiag, H->cdiag.p + 3 * cb, m * sizeof(double), cudaMemcpyDeviceToHost));
    if (hvec && m) CK(cudaMemcpy(hvec, H->hvec.p + 3 * cb, m * sizeof(double), cudaMemcpyDeviceToHost));
    if (dxt && ns) CK(cudaMemcpy(dxt, H->dxt.p + 3 * sb, 3 * (size_t)ns * sizeof(double), cudaMemcpyDeviceToHost));
    if (slot_vertex) for (int s = 0; s < ns; ++s) slot_vertex[s] = H->int2orig[I.verts[s]];
    if (djj && nc) {
        std::vector<DContact> hc(nc);
        CK(cudaMemcpy(hc.data(), H->dc.p + cb, nc * sizeof(DContact), cudaMemcpyDeviceToHost));
        for (int c = 0; c < nc; ++c) djj[c] = hc[c].Djj;
    }
    return SIM_OK;
}

// Schur right-hand side rho = h - Theta J x~ of the most recent L-G iteration ([3 * n_contacts], rows
// n, t1, t2 per contact; bilateral contacts pad rows 1-2 with 0): the input of that iteration's CR
extern "C" int sim_debug_contact_rho(sim_handle* H, int32_t inst, double* rho) {
    int rc = check_instance(H, inst);
    if (rc) return rc;
    if (!rho) return fail(SIM_E_INVALID, "null argument");
    if (H->dirty || H->dev_pending) return fail(SIM_E_STATE, "contacts changed since the last step");
    CK(cudaStreamSynchronize(H->stream));
    const InstContacts& I = H->ic[inst];
    const size_t m = 3 * I.hc.size();
    if (m) CK(cudaMemcpy(rho, H->rho.p + 3 * (size_t)H->coff_h[inst], m * sizeof(double), cudaMemcpyDeviceToHost));
    return SIM_OK;
}

// phase timestamps (ns, %globaltimer) of the most recent CR call (instance 0): [0] start,
// [1] staged, [2] first reduction, [3 + it] after CR iteration it, [20] loop end,
// [21] epilogue end.  out must hold 32 values.
extern "C" int sim_debug_cr_timeline(sim_handle* H, double* out) {
    if (!H || !out) return fail(SIM_E_INVALID, "null argument");
    if (H->host_only) return fail(SIM_E_STATE, "no device");
    CK(cudaStreamSynchronize(H->stream));
    unsigned long long t[32];
    CK((cudaError_t)read_cr_clock(t));
    for (int i = 0; i < 32; ++i) out[i] = (double)(t[i] - t[0]) * 1e-3;   // us since start
    return SIM_OK;
}

namespace simdev { int debug_pl_clock(unsigned long long* out); }
// plane K-pass timeline of CTA (0, 0): [pass][tile][8] %globaltimer stamps (all zero unless built with
// -DSIM_PL_TIMELINE; tools/pl_timeline.py)
extern "C" int sim_debug_pl_timeline(unsigned long long* out) { return simdev::debug_pl_clock(out); }
