// Device data structures and kernel declarations (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "host.hpp"

namespace simdev {

using simhost::P1Block;
using simhost::P1Item;
using simhost::P2Block;
using simhost::BUnit;

// row stride of the fp32 component planes u, y hold for S > 1 (see vec_ld in kernels.cu)
__host__ __device__ inline int plane_sp(int S) { return S == 1 ? 1 : (S + 3) & ~3; }

constexpr int kMaxContacts = 1024;   // per instance: the CR keeps fp64 vectors of 3*kMaxContacts rows in SMEM
constexpr int kMaxSlots = 1024;      // distinct contact vertices per instance
#ifndef SIM_CR_CLUSTER
#define SIM_CR_CLUSTER 16
#endif
constexpr int kCluster = SIM_CR_CLUSTER;   // max CTAs per instance in the CR cluster (non-portable size)
constexpr int kCrThreads = 512;
constexpr size_t kCrMaxSmem = 232448;  // 227 KB opt-in shared memory per CTA (sm_100)
int read_cr_clock(unsigned long long* out);   // phase timestamps of the last CR call (debug)

// one contact on the device.  Contacts, slots (distinct contact vertices) and the
// per-contact scratch of all instances are packed back to back (instance i owns
// contacts [coff[i], coff[i+1]) and slots [soff[i], soff[i+1])); slot ids are global.
struct DContact {
    int32_t kind, nv, inst, pad;
    int32_t vtx[4];     // internal vertex ids (state index = vtx * S + inst)
    int32_t slot[4];    // global slot ids
    double w[4];
    double c[3][3];     // rows: n, t1, t2 (bilateral: n, 0, 0)
    double dn, df1, df2, mu, e;
    double Djj;         // D_jj (Delassus diagonal, same for the 3 unit rows)
    double Mjj;         // [J M^-1 J^T]_jj (mass-inverse preconditioner of the ablation)
};

struct Params {
    int n_v, n_f, n_t;
    int S;                // instances; per-vertex / per-tet state is [entity][S] (instance-minor)
    double h;
    double g[3];
    const double4* vpin;  // [n_v - n_f][S]: velocity of each pinned vertex-instance (moving Dirichlet targets)
    int model;
    float k, mu, lam;     // projection stiffness and Lame parameters
    int C, NS;            // contacts, contact slots over all instances
    int nc_max, ns_max;   // per-instance maxima
    int NCL, CS;          // slot-set classes, class slots
    int cm_max;           // largest class (members)
    int cr_iters;
    int warm;             // frame start: 0 x^0 = s, lambda^0 = 0 (A9, A10); 1 x^0 = x_t + h v_t, lambda kept (A9w, A10w)
    double len_scale;     // max(rest bbox diagonal, max |rest coordinate|): gaps within 1e-12 of it are 0 (A15)
    int ncp;              // 0 Fischer-Burmeister (App. B.2, the paper's choice), 1 minimum map (App. B.1)
    int precond;          // 0 Delassus diagonal, 1 mass inverse
    int pair_local;       // S > 1, S even: the packed-FP32 paired local step (k_local2)
};

// Offsets of the packed contact data.  Instances whose contact-vertex sets are equal form
// a slot-set class: the ancestor chains, the chain-row list, the compact K copy Zc and the
// Delassus Gram G depend only on K and that vertex set, so they are built once per class.
struct InstOff {
    const int* coff;        // [S+1] contacts per instance
    const int* soff;        // [S+1] slots per instance (slot s of instance i <-> class slot s)
    const int64_t* gaoff;   // [S+1] active blocks G_A per instance (ns_i^2 floats)
    const int* cls;         // [S] class of each instance
    const int* csoff;       // [NCL+1] class slots
    const int64_t* goff;    // [NCL+1] Delassus Gram block per class (ns^2 floats)
    const int* uoff;        // [NCL+1] chain-row list capacity per class
    const int64_t* zoff;    // [NCL+1] chain entries / Zc per class
    const int* cmoff;       // [NCL+1] class members in cmem
    const int* cmem;        // [S] instances grouped by class (ascending within a class)
};
// class slots (global class-slot ids): vertex and class
struct ClassSlots {
    const int32_t* vtx;     // [CS] internal vertex (ascending within a class)
    const int32_t* cls;     // [CS]
};

// per-iteration contact scratch (device, packed over instances)
struct ContactState {
    double* lam;      // [3 C]
    double* theta;    // [3 C]
    double* cdiag;    // [3 C]
    double* hvec;     // [3 C]
    double* hl;       // [C][3]  sum_rows theta lam c   (H^T lambda per contact)
    double* dxt;      // [NS][3]  (K^T y) at slot vertices
    double* wz;       // [NS][3]  sum_rows w theta z c per slot
    double* phi_abs;  // [C] |phi_n| (stats)
    double* cr_res;   // [S]
    double* rho;      // [3 C] Schur RHS h - Theta J x~ (from the chain dot)
    float4* wzT;      // [ns_max][S] wz, class-slot-major / instance-minor (grouped scatter; S > 1)
};

// active contact vertices of the current iteration (theta != 0 on an incident row)
struct CrActive {
    int* na;     // [S]
    int* aidx;   // [NS] (instance section) active position -> local slot
    int* apos;   // [NS] global slot -> active position or -1
    int* acon;   // [NS] active position -> local id of its single single-vertex contact or -1
};

// compact per-contact arrays for the CR: rows' directions, single-vertex slot / vertex (-1 otherwise)
struct CrContacts {
    const float* c9;   // [C][3][3] rows n, t1, t2
    const DContact* dc;   // the fp64 rows (the Schur RHS uses the directions h-vector used)
    const int* s0;     // [C] global slot of a single-vertex weight-1 contact, else -1
    const int* v0;     // [C] its internal vertex, else -1
    const int* c1;     // [NS] the only contact (global id) on a slot if it is single-vertex weight-1, else -1
};

// slot data (global slot ids)
struct Slots {
    const int32_t* vtx;    // [NS] internal vertex (ascending within an instance)
    const int32_t* inst;   // [NS]
    const int32_t* scp;    // [NS+1] slot -> contacts CSR (global positions)
    const int32_t* sci;    // global contact ids
    const float* scw;      // weights
};

// --- frame kernels -----------------------------------------------------------
void launch_replicate(cudaStream_t st, const double4* src, double4* dst, int n, int S);
// vt (nullable): frame-start velocity copy; bad (nullable): per-instance failure flags, zeroed here
void launch_predict(cudaStream_t st, const Params& P, double4* x, double4* xt, double4* v, double4* s,
                    double* lam, int nlam, double4* vt = nullptr, int* bad = nullptr);
// sim_set_pins: vpin[p][inst] = (target[p] - x[n_f + p][inst]) / h for the n_pin pinned vertices of one instance
void launch_pin_targets(cudaStream_t st, int n_f, int n_pin, int S, int inst, double h, const double4* x,
                        const double4* target, double4* vpin);
// lam[3c + r] = carry[c] >= 0 ? lam_old[3 carry[c] + r] : 0 for the C contacts of a new commit
void launch_carry_lambda(cudaStream_t st, int C, const int32_t* carry, const double* lam_old, double* lam);
void launch_poison(cudaStream_t st, double4* x, int inst, int S);
void launch_pack_positions(cudaStream_t st, const double4* x, const int32_t* o2i, int n_v, int S, double* dst);   // test hook: x[vertex 0] of inst = NaN
// end of frame: instances with a non-finite x or v get x = x_t, v = v_t; *rollbacks += count
void launch_finite_guard(cudaStream_t st, int n_v, int S, double4* x, double4* v, const double4* xt,
                         const double4* vt, int* bad, int* rollbacks);
// du: ADMM-PD dual [9][n_t S] or nullptr (plain PD); admm_first: treat u as 0 (first iteration of a frame)
void launch_local(cudaStream_t st, const Params& P, const int4* tet, const float* Bm, const float* hw2,
                  const double4* x, float* fc, float* Pdbg, float* du = nullptr, int admm_first = 0);
void launch_contact_eval(cudaStream_t st, const Params& P, const DContact* c, const double4* x,
                         const double4* xt, ContactState cs);
// frame-end statistics per contact: A21 class (-1 bilateral, 0 inactive, 1 stick, 2 slip), cone
// violation max(0, |lambda_f| - mu max(lambda_n, 0)), gap y_n
void launch_contact_stats(cudaStream_t st, const Params& P, const DContact* c, const double4* x, const double4* xt,
                          const double* lam, int* cls, double* cone, double* gap);
// slotmap[a * S + i] = global slot of vertex a in instance i, or -1
void launch_gather(cudaStream_t st, const Params& P, const int32_t* adjp, const int32_t* adj,
                   const float* fc, const double* M, const double4* x, const double4* s,
                   const int32_t* slotmap, Slots sl, const double* hl, float4* u, double* resid_dbg);
// K-passes over the tile streams T1 / T2 (see simhost::build_tiles); S = 1
void launch_kpass1(cudaStream_t st, int nitems, const P1Item* it, const P1Block* bl, const float* T1,
                   const float4* u, float4* y, double* part, int* counters);
void launch_kpass2(cudaStream_t st, int nblocks, const P2Block* bl, const int32_t* cover, const float* T2,
                   const float4* y, double4* x, const double4* xt, double4* v, double inv_h, int finalize_v);
// batched K-passes (S > 1): K tiles shared by all instances (SpMM over 3 S right-hand sides)
void launch_kpass1_batched(cudaStream_t st, int S, int n_f, int nunits, const BUnit* units, const float* T1p,
                           const float* u, float* y, double* part, int* counters);
void launch_kpass2_batched(cudaStream_t st, int S, int n_f, int nunits, const BUnit* units, const int32_t* cover,
                           const float* T2, const float* y, double4* x, const double4* xt, double4* v,
                           double inv_h, int finalize_v);
// plane-layout K-passes on the tensor cores (tcgen05 kind::tf32, 3xTF32; S > 1): u, y as fp32
// component planes [3][n_f][Sp], units and tile streams of simhost::build_plane_units; split pass-1
// blocks use fp32 partials part[nparts][3][64][Sp] and counters[nblocks][chunks] (zero between launches)
void launch_kpass1_pl(cudaStream_t st, int S, int Sp, int n_f, int nunits, const BUnit* units, const float* T,
                      const float* u, float* y, float* part, int* counters, int drain);
void launch_kpass2_pl(cudaStream_t st, int S, int Sp, int n_f, int nunits, const BUnit* units, const int32_t* cover,
                      const float* T, const float* y, double4* x, const double4* xt, double4* v, double inv_h,
                      int finalize_v, int drain);   // drain: tiles accumulated in TMEM (fp32) per register fold
// extra arguments of the contact passes on the tensor cores
struct TsExtra {
    const int32_t* orows;   // scatter pass: output rows
    const int* soff;        // chain pass: first slot of each instance
    CrContacts cc;
    const double4* xs;
    ContactState cs;
    int nf;                 // free vertices (plane stride of y)
};
// contact passes of the single slot-set class (S > 1) on the tensor cores (simhost::ContactPasses)
// units split over several parts (nparts > 1; pad = the block's first partial slot) sum fp64
// partials in `part` ([slot][3][32][S]); the last part of a block (counters, zero on entry and
// reset on exit) adds them in part order and evaluates the slots' Schur right-hand sides
void launch_chain_pass_ts(cudaStream_t st, int S, int nf, int nunits, const BUnit* units, const float* Ttc,
                          const int32_t* cover, const float4* y, const int* soff, CrContacts cc, const double4* x,
                          ContactState cs, int drain, double* part, int* counters);
void launch_scatter_pass_ts(cudaStream_t st, int S, int nf, int ns, int nunits, const BUnit* units, const float* Ttc,
                            const int32_t* rows, const float4* wzT, float4* y, int drain, double* part,
                            int* counters);   // split units: as launch_chain_pass_ts
// grouped: one work item per (class slot, 32 class members); items int2 {class slot, member0}
void launch_chain_dot(cudaStream_t st, const Params& P, InstOff off, ClassSlots csl, const float* Kcol,
                      const int64_t* colptr, const int32_t* chain_off, const int32_t* chain_rows, const float4* y,
                      Slots sl, CrContacts cc, const double4* x, ContactState cs, int nitems, const int2* items);

void launch_active(cudaStream_t st, const Params& P, InstOff off, CrContacts cc, Slots sl, ContactState cs,
                   CrActive act, const float* G, float* GA);
// G: the class Delassus Grams; a CTA that owns a whole instance gathers its G_A rows from G straight
// into shared memory (cr_ga_direct), else it reads the G_A copy k_active wrote to GA
int launch_cr(cudaStream_t st, const Params& P, InstOff off, const DContact* c, CrContacts cc, Slots sl,
              const float* G, const float* GA, const double4* x, ContactState cs, CrActive act);
// y_i += sum_{slots s in subtree(i)} K[i][a_s] wz_s over the rows of each instance's ulist
// (int4 {row, s0, s1, zoff}); max_rows bounds the per-instance list length
// grouped: items int2 {class, member0} (32 members per item)
void launch_scatter(cudaStream_t st, const Params& P, int max_rows, InstOff off, const int* ucount,
                    const int4* ulist, const float* Zc, const double* wz, const float4* wzT, float4* y, int nitems,
                    const int2* items);

// --- persistent small-scene driver (S = 1, no contacts, no ADMM) -------------------------
struct SmallArgs {
    const int4* tet; const float* Bm; const float* hw2; const double* M;
    const int32_t* adjp; const int32_t* adj;
    const float* Krow; const int2* meta;     // meta[r] = {rowptr[r] - first[r], first[r]}
    const float* Kcol; const int64_t* colptr; const int32_t* parent;
    double4 *x, *xt, *v, *s, *vt;
    int* rollbacks;
};
size_t small_smem_bytes(const Params& P);
// frames x iters L-G iterations in one single-CTA launch (returns a cudaError_t)
int launch_small_frames(cudaStream_t st, const Params& P, const SmallArgs& A, int frames, int iters);

// --- proximity query ------------------------------------------------------------------
struct DObstacle {   // device copy of sim_obstacle
    int kind, pad;
    double a[3], b[3], radius, mu, v[3];
};
// per candidate c (internal vertex cand[c] of instance inst): best[c] = index of the nearest
// obstacle within margin or -1, with its outward normal n[c] and closest surface point p[c]
void launch_proximity(cudaStream_t st, const Params& P, const double4* x, int inst, const int32_t* cand, int ncand,
                      const DObstacle* obs, int nobs, double margin, int* best, double* gap, double3* n, double3* pt);

// --- per-contact-set kernels (all instances at once) ----------------------------
void launch_delassus(cudaStream_t st, const Params& P, InstOff off, ClassSlots csl, const float* Kcol,
                     const int64_t* colptr, const int32_t* depth, const int32_t* parent, const int32_t* ptop,
                     float* G);
void launch_djj(cudaStream_t st, const Params& P, InstOff off, DContact* c, const float* G);
// K = L^-1 column by column on the device (bitwise the host's simhost::sparse_inverse_values);
// L in CSC with the diagonal first in each column; hmax = etree height; returns a cudaError_t
int launch_inverse_columns(cudaStream_t st, int n, int hmax, const int64_t* Lp, const int32_t* Li, const double* Lx,
                           const int32_t* parent, const int32_t* depth, const int32_t* first, const int64_t* colptr,
                           const int64_t* rowptr, double drop_tol, float* Kcol, float* Krow);
// Gram reuse: copy entries of vertex pairs from the previous blocks (rmap, pgoff, pns), compute
// the rows of the new slots (newslots: {class, class-local slot}); bitwise = launch_delassus
void launch_gram_reuse(cudaStream_t st, const Params& P, InstOff off, const int32_t* vtx_all, const int* rmap,
                       const int64_t* pgoff, const int* pns, const float* Gprev, const int2* newslots, int nnew,
                       const float* Kcol, const int64_t* colptr, const int32_t* depth, const int32_t* parent,
                       const int32_t* ptop, float* G);
// ancestor-chain rows of every class slot (chain order = Kcol order); flags rows per class
// (flag[c * n_f + row]); slotmap[vtx * S + inst] = instance slot
void launch_chain_rows(cudaStream_t st, const Params& P, ClassSlots csl, Slots sl, const int32_t* chain_off,
                       const int32_t* parent, const int32_t* ptop, int32_t* chain_rows, uint8_t* flag,
                       int32_t* slotmap);
// ucount[2 c] = rows listed for class c, ucount[2 c + 1] = its values in Zc (zeroed by the caller)
void launch_ulist(cudaStream_t st, const Params& P, InstOff off, const uint8_t* flag, ClassSlots csl,
                  const int2* meta, int* ucount, int4* ulist, const float* Krow, float* Zc);

// --- grid CR (one scene, contact sets beyond the cluster CR's shared memory) ------
// Delassus groups = etree components holding contact slots; slot a's Gram row is
// G[rowoff[a] .. + gn[a]) over the group's slots gs0[a] .. gs0[a] + gn[a] - 1.
struct GcrData {
    const float* c9;          // [C][3][3] row directions
    const float* G;           // group blocks, gn^2 floats each
    const int64_t* rowoff;    // [NS]
    const int* gs0;           // [NS] first slot of the slot's group
    const int* gn;            // [NS] slots in the group
    double *r, *p, *Ap, *z, *Ar;   // [3 C]
    double *W, *q;                 // [NS][3]
    double* part;                  // [row blocks][3] partial dot products
    double* sc;                    // [6] ping-pong CR scalars rAr, ApAp, stop
    int* cnt;                      // [1] arrival counter of the final reduction (zero between launches)
    const int2* gram_items;        // Gram matvec items {first slot row, rows <= 32} within one group
    int n_gram_items;
    int nblk;
};
int gcr_row_blocks(int C);
int gcr_kernels_per_iteration(int cr_iters);
int launch_gcr(cudaStream_t st, const Params& P, GcrData g, const DContact* c, CrContacts cc, Slots sl,
               const double4* x, ContactState cs);
void launch_djj_grid(cudaStream_t st, const Params& P, DContact* c, GcrData g);

size_t cr_smem_bytes(int nc, int ns);   // the CR CTA's shared-memory footprint for (nc, ns) without G_A
int cr_cluster_size(int S);             // CTAs per instance in the CR launch

}  // namespace simdev
