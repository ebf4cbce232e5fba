// Host-side precompute of the sparse inverse (C++17, fp64).
//
//   A_v = M + h^2 sum_i w_i g_a g_b^T            (eq. PD global)
//   ordering: geometric nested dissection        ("e.g. nested dissection")
//   etree + postorder; up-looking Cholesky       (Alg. 2 line 1)
//   K = L^-1 column by column over the ancestor chain of each column
//                                                (Thm 1, Fig. 4)
//
// In etree postorder every row i of K is the contiguous column range
// [first(i), i] (first(i) = i - |subtree(i)| + 1) and every column j is the
// ancestor chain of j, so K is stored values-only twice: row-major (for the
// transposed pass) and column-major (for the forward pass).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace simhost {

struct Csr {
    int n = 0;
    std::vector<int64_t> ptr;
    std::vector<int32_t> col;
    std::vector<double> val;
};

struct RestData {
    std::vector<double> Bm;     // [n_t][9] row-major Dm^-1
    std::vector<double> vol;    // [n_t]
    std::vector<double> w;      // [n_t] w_i = k vol_i
    std::vector<double> mass;   // [n_v] lumped
};

// returns "" on success, else message; bad_tet set on degenerate tet
std::string rest_data(int n_v, int n_t, const double* X, const int32_t* T, double density,
                      double k_proj, RestData& out, int& bad_tet);

// A_v restricted to the vertex subset `vid` (vid[v] = row index or -1), full symmetric CSR
Csr assemble_Av(int n_v, int n_t, const int32_t* T, const RestData& rd, double h,
                const std::vector<int32_t>& vid, int n_rows);

// geometric nested dissection: returns order[k] = row index eliminated k-th
std::vector<int32_t> nested_dissection(const Csr& A, const std::vector<double>& coords /*[n][3]*/);

struct Factor {
    int n = 0;
    std::vector<int32_t> parent;     // etree (postordered: parent[i] > i or -1)
    std::vector<int64_t> Lp;         // CSC of L, diagonal first in each column
    std::vector<int32_t> Li;
    std::vector<double> Lx;
    int bad_col = -1;
};

// symmetric permutation C = P A P^T with perm[new] = old
Csr permute_sym(const Csr& A, const std::vector<int32_t>& perm);
std::vector<int32_t> etree(const Csr& A);
std::vector<int32_t> postorder(const std::vector<int32_t>& parent);
// up-looking Cholesky; returns false on non-positive pivot (f.bad_col)
bool cholesky(const Csr& A, const std::vector<int32_t>& parent, Factor& f);

struct Inverse {
    int n = 0;
    std::vector<int32_t> parent, depth, first, ptop, panel_of;
    // kept skyline after the drop tolerance (reading A25): firstk[r] = the smallest column j of row r
    // with K[r][j] != 0 after dropping (= first[r] at tol 0).  The K-pass work lists and tile
    // streams cover [firstk(r), r] only, so dropped leading entries cost no bytes
    std::vector<int32_t> firstk;
    std::vector<int64_t> rowptr, colptr;   // row-major and column-major offsets
    std::vector<float> Krow, Kcol;         // fp32 values
    std::vector<int32_t> panel_start;      // [n_panels+1]
    int height = 0;
    int64_t nnz = 0;
};

// firstk from the stored values (after sparse_inverse / the device inverse)
void trim_dropped(Inverse& K);
// K = L^-1 (fp64 compute, fp32 store); drop |K_ij| < tol |K_jj| (tol > 0)
void sparse_inverse(const Factor& f, double drop_tol, Inverse& K, int n_threads);
// the two halves: index structure (depth, first, row/column offsets, panels; values zeroed) and
// the values column by column (the device variant is simdev::launch_inverse_columns)
void sparse_inverse_structure(const Factor& f, Inverse& K);
void sparse_inverse_values(const Factor& f, double drop_tol, Inverse& K, int n_threads);

// ---------------- K-pass work lists (one CTA per item) ----------------------
// pass 1 (y = K u, column-major K): item = (<= 32 rows of one panel) x (<= 1024 columns)
struct P1Item { int32_t r0, nrows, c0, c1, block, part; int64_t toff; };   // toff: tile stream offset (floats)
struct P1Block { int32_t r0, nrows, nitems, part0; };
// pass 2 (x += K^T y, row-major K): one item per 32-column block, its cover rows
// (rows i >= c0 with first(i) <= c0 + 31) in cover[list0, list1)
struct P2Block { int32_t c0, ncols, list0, list1; int64_t toff; };

struct WorkLists {
    std::vector<P1Item> p1;
    std::vector<P1Block> p1b;
    std::vector<P2Block> p2b;
    std::vector<int32_t> cover;
    int p1_parts = 0;
};

void build_worklists(const Inverse& K, WorkLists& wl, int p1_chunk_cols);

// K re-laid out as tile streams in the exact order each pass consumes them, so a pass
// streams contiguous 4 KB tiles with bulk (TMA) copies:
//   pass 1 item (rows r0..r0+nr-1, columns c0..c1-1): tiles of 32 columns, tile[q][l] =
//     K[r0 + l][jc + q]  (nr x 32 floats, zero outside the skyline)
//   pass 2 block (32 columns c0..): tiles of 32 cover rows, tile[q][l] = K[row_q][c0 + l]
//     (32 x 32 floats, zero outside [first(row), row])
// Fills wl.p1[*].toff / wl.p2b[*].toff.
void build_tiles(const Inverse& K, WorkLists& wl, std::vector<float>& T1, std::vector<float>& T2);

// ---------------- batched K-passes (S instances share K) --------------------
// A unit is one CTA's share of a pass for one chunk of instances:
//   pass 1: rows r0..r0+nr-1 of one block x tiles [c0 + 32 t, +32), t < ntiles; tiles of the
//           padded stream T1p, tile[q][l] = K[r0 + l][c0 + 32 t + q] (32 x 32, zero-padded);
//           a block split over nparts units writes partials part..; list0 = the block's first part
//   pass 2: columns c0..c0+nr-1, cover rows cover[list0 .. list0 + nlist), T2 tiles at toff
struct BUnit { int32_t r0, nr, c0, ntiles, list0, nlist, block, part, nparts, pad; int64_t toff; };

// unit_tiles: max tiles per pass-1 unit (bounds the longest CTA); returns the number of partials
int build_batched(const Inverse& K, const WorkLists& wl, int unit_tiles, std::vector<BUnit>& u1,
                  std::vector<float>& T1p, std::vector<BUnit>& u2, int& nblocks1);

// ---------------- plane-layout tensor-core K-passes (S > 1), 64 outputs per unit -------------
// Right-hand sides in fp32 component planes; one CTA = one unit x 128 instances x 3 components,
// tcgen05 M = 128 (instances) x N = 64 (outputs) x K = 32 (tile reductions).
//   pass 1 (y = K u): blocks of <= 64 consecutive rows r0..r0+nr-1, columns [first(r0), r0 + nr)
//       in tiles of 32 from c0 (the block's first column), split into units of <= unit_tiles
//       tiles; tile[q][l] = K[r0 + l][c0 + 32 t + q]; a split block writes fp64 partials (part,
//       list0 = the block's first part, block = counter index)
//   pass 2 (x += K^T y): blocks of <= 64 consecutive columns c0..c0+nr-1, their sorted cover rows
//       (rows i >= c0 with first(i) <= c0 + nr - 1) in cover[list0 .. list0 + nlist);
//       tile[q][l] = K[cover[list0 + 32 t + q]][c0 + l]
// Tile stream: per tile 4096 floats = the tf32 hi tile (round to nearest) then the lo tile
// (v - hi, rounded), each in the tcgen05 SWIZZLE_NONE K-major core-matrix layout
// [l / 8][q / 4][l % 8][q % 4] (64 x 32); toff in floats.
struct PlaneUnits {
    std::vector<BUnit> u1, u2;
    std::vector<int32_t> cover;     // pass-2 cover rows
    std::vector<float> T1, T2;      // tile streams (hi/lo)
    int nparts1 = 0, nblocks1 = 0;
    int64_t tiles1 = 0, tiles2 = 0;
};
void build_plane_units(const Inverse& K, int unit_tiles, PlaneUnits& pu);

// ---------------- contact passes of a slot-set class on the tensor cores (S > 1) -------------
// With Z[s][r] = K[r][a_s] (r on the ancestor chain of the contact vertex a_s):
//   chain pass   dxt[s] = sum_r Z[s][r] y[r]   -- units like pass 2: 32 slots (c0, nr), their
//                sorted chain-row union in cover[list0 .. list0 + nlist), tiles tile[q][l] = Z[c0+l][cover q]
//   scatter pass y[r] += sum_s Z[s][r] wz[s]    -- units like pass 1: 32 chain rows rows[r0 .. r0 + nr),
//                slots c0 .. c0 + 32 ntiles, tiles tile[q][l] = Z[c0 + 32 t + q][rows[r0 + l]]
// Tile streams are in the plain tile[q][l] order (tc_tiles re-lays them out).
struct ContactPasses {
    std::vector<BUnit> uc, us;
    std::vector<int32_t> cover, rows;
    std::vector<float> Tc, Ts;
};
void build_contact_passes(const Inverse& K, const std::vector<int32_t>& slot_vtx, ContactPasses& cp);

// Tensor-core copy of a tile stream (1024-float tiles, tile[q * 32 + l], q = reduction index,
// l = output): per tile 2048 floats = the tf32 "hi" tile then the "lo" tile (v - hi), both
// rounded to nearest tf32, each in the tcgen05 SWIZZLE_NONE K-major core-matrix layout
// [l / 8][q / 4][l % 8][q % 4].
void tc_tiles(const std::vector<float>& T, std::vector<float>& Ttc);

}  // namespace simhost
