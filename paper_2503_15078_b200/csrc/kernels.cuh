// Device data structures and kernel declarations (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "host.hpp"

namespace simdev {

using simhost::P1Block;
using simhost::P1Item;
using simhost::P2Block;

constexpr int kMaxContacts = 1024;   // CR cluster keeps fp64 vectors of 3*kMaxContacts rows in SMEM
constexpr int kMaxSlots = 1024;      // distinct contact vertices
constexpr int kCluster = 16;         // CTAs in the CR cluster (non-portable size)
constexpr int kCrThreads = 512;
constexpr size_t kCrMaxSmem = 232448;  // 227 KB opt-in shared memory per CTA (sm_100)
size_t cr_smem_bytes(int nc, int ns);
int read_cr_clock(unsigned long long* out);   // phase timestamps of the last CR call (debug)  // the CR cluster's shared-memory footprint for (nc, ns)

// one contact on the device (internal vertex ids, slot ids into the sorted contact-vertex list)
struct DContact {
    int32_t kind, nv;
    int32_t vtx[4];
    int32_t slot[4];
    double w[4];
    double c[3][3];     // rows: n, t1, t2 (bilateral: n, 0, 0)
    double dn, df1, df2, mu, e;
    double Djj;         // D_jj (Delassus diagonal, same for the 3 unit rows)
};

struct Params {
    int n_v, n_f, n_t;
    double h;
    double g[3];
    double vpin[3];
    int model;
    float k, mu, lam;     // projection stiffness and Lame parameters
    int nc, ns;           // contacts, contact slots
    int cr_iters;
};

// per-iteration contact scratch (device)
struct ContactState {
    double* lam;      // [3 nc]
    double* theta;    // [3 nc]
    double* cdiag;    // [3 nc]
    double* hvec;     // [3 nc]
    double* hl;       // [nc][3]  sum_rows theta lam c   (H^T lambda per contact)
    double* dxt;      // [ns][3]  (K^T y) at slot vertices
    double* wz;       // [ns][3]  sum_rows w theta z c per slot
    double* phi_abs;  // [nc] |phi_n| (stats)
    double* cr_res;   // [1]
    double* rho;      // [3 nc] Schur RHS h - Theta J x~ (from the chain dot)
};

// active contact vertices of the current iteration (theta != 0 on an incident row)
struct CrActive {
    int* na;     // [1]
    int* aidx;   // [ns] active position -> slot
    int* apos;   // [ns] slot -> active position or -1
    int* acon;   // [ns] active position -> its single single-vertex contact or -1
};

// --- frame kernels -----------------------------------------------------------
void launch_predict(cudaStream_t st, const Params& P, double4* x, double4* xt, double4* v, double4* s,
                    double* lam, int nlam);
void launch_local(cudaStream_t st, const Params& P, const int4* tet, const float* Bm, const float* hw2,
                  const double4* x, float4* fc, float* Pdbg);
void launch_contact_eval(cudaStream_t st, const Params& P, const DContact* c, const double4* x,
                         const double4* xt, ContactState cs);
void launch_gather(cudaStream_t st, const Params& P, const int32_t* adjp, const int32_t* adj,
                   const float4* fc, const double* M, const double4* x, const double4* s,
                   const int32_t* vcp, const int32_t* vci, const float* vcw, const double* hl,
                   const int32_t* cb, float4* u, double* resid_dbg);
// K-passes over the tile streams T1 / T2 (see simhost::build_tiles)
void launch_kpass1(cudaStream_t st, int nitems, const P1Item* it, const P1Block* bl, const float* T1,
                   const float4* u, float4* y, double* part, int* counters);
void launch_kpass2(cudaStream_t st, int nblocks, const P2Block* bl, const int32_t* cover, const float* T2,
                   const float4* y, double4* x, const double4* xt, double4* v, double inv_h, int finalize_v);
// compact per-contact arrays for the CR: rows' directions, single-vertex slot / vertex (-1 otherwise)
struct CrContacts {
    const float* c9;   // [nc][3][3] rows n, t1, t2
    const int* s0;     // [nc] slot of a single-vertex weight-1 contact, else -1
    const int* v0;     // [nc] its vertex, else -1
    const int* c1;     // [ns] the only contact on a slot if it is single-vertex weight-1, else -1
};
void launch_chain_dot(cudaStream_t st, int ns, const int32_t* slot_vtx, const float* Kcol,
                      const int64_t* colptr, const int32_t* chain_off, const int32_t* chain_rows,
                      const float4* y, double* dxt, CrContacts cc, const double4* x, ContactState cs);

void launch_active(cudaStream_t st, int ns, CrContacts cc, const int32_t* scp, const int32_t* sci, ContactState cs,
                   CrActive act, const double* G, double* GA);
int launch_cr(cudaStream_t st, const Params& P, const DContact* c, CrContacts cc, const int32_t* scp,
              const int32_t* sci, const float* scw, const double* GA, const double4* x, ContactState cs,
              CrActive act);
// y_i += sum_{slots s in subtree(i)} K[i][a_s] wz_s over the rows of ulist (int4 {row, s0, s1, -})
void launch_scatter(cudaStream_t st, int max_rows, const int* ucount, const int4* ulist, const float* Zc,
                    const double* wz, float4* y);

// --- per-contact-set kernels ----------------------------------------------------
void launch_delassus(cudaStream_t st, int ns, const int32_t* slot_vtx, const float* Kcol,
                     const int64_t* colptr, const int32_t* depth, const int32_t* parent,
                     const int32_t* ptop, double* G);
void launch_djj(cudaStream_t st, int nc, int ns, DContact* c, const double* G);
// ancestor-chain rows of every slot (chain order = Kcol order) and the rows on
// any chain with their slot ranges [s0, s1) = slots in [first(i), i]
void launch_chain_rows(cudaStream_t st, int ns, const int32_t* slot_vtx, const int32_t* chain_off,
                       const int32_t* parent, const int32_t* ptop, int32_t* chain_rows, uint8_t* flag);
// ucount[0] = rows listed, ucount[1] = values in the compact copy Zc (both zeroed by the caller)
void launch_ulist(cudaStream_t st, int n_f, int ns, const uint8_t* flag, const int32_t* slot_vtx,
                  const int2* meta, int* ucount, int4* ulist, const float* Krow, float* Zc);

}  // namespace simdev
