// Device data structures and kernel declarations (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "host.hpp"

namespace simdev {

using simhost::P1Block;
using simhost::P1Item;
using simhost::P2Block;
using simhost::P2Item;
using simhost::Run;

constexpr int kMaxContacts = 1024;   // CR cluster keeps fp64 vectors of 3*kMaxContacts rows in SMEM
constexpr int kMaxSlots = 1024;      // distinct contact vertices
constexpr int kCluster = 16;         // CTAs in the CR cluster (non-portable size)
constexpr int kCrThreads = 512;

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
                   float4* u, double* resid_dbg);
void launch_kpass1(cudaStream_t st, int nitems, const P1Item* it, const P1Block* bl, const float* Kcol,
                   const int64_t* cb, const int32_t* depth, const float4* u, float4* y, double* part,
                   int* counters);
void launch_kpass2(cudaStream_t st, int nitems, const P2Item* it, const P2Block* bl, const Run* runs,
                   const float* Krow, const float4* y, double* part, int* counters, double4* x,
                   const double4* xt, double4* v, double inv_h, int finalize_v);
void launch_chain_dot(cudaStream_t st, int ns, const int32_t* slot_vtx, const float* Kcol,
                      const int64_t* colptr, const int32_t* parent, const int32_t* ptop, const float4* y,
                      double* dxt);
int launch_cr(cudaStream_t st, const Params& P, const DContact* c, const int32_t* slot_vtx,
              const int32_t* scp, const int32_t* sci, const float* scw, const float* G, const double4* x,
              ContactState cs);
void launch_scatter(cudaStream_t st, int n_f, int ns, int row_lo, const int32_t* slot_vtx, const float* Krow,
                    const int64_t* rowptr, const int32_t* first, const double* wz, float4* y);

// --- per-contact-set kernels ----------------------------------------------------
void launch_delassus(cudaStream_t st, int ns, const int32_t* slot_vtx, const float* Kcol,
                     const int64_t* colptr, const int32_t* depth, const int32_t* parent,
                     const int32_t* ptop, float* G);
void launch_djj(cudaStream_t st, int nc, int ns, DContact* c, const float* G);

}  // namespace simdev
