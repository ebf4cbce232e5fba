// Host precompute of the sparse inverse; see host.hpp for the citations.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace simhost {

std::string rest_data(int n_v, int n_t, const double* X, const int32_t* T, double density,
                      double k_proj, RestData& out, int& bad_tet) {
    out.Bm.assign((size_t)n_t * 9, 0.0);
    out.vol.assign(n_t, 0.0);
    out.w.assign(n_t, 0.0);
    out.mass.assign(n_v, 0.0);
    bad_tet = -1;
    for (int t = 0; t < n_t; ++t) {
        const int32_t* v = T + 4 * (size_t)t;
        double D[3][3];
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) D[r][c] = X[3 * (size_t)v[c + 1] + r] - X[3 * (size_t)v[0] + r];
        double det = D[0][0] * (D[1][1] * D[2][2] - D[1][2] * D[2][1]) -
                     D[0][1] * (D[1][0] * D[2][2] - D[1][2] * D[2][0]) +
                     D[0][2] * (D[1][0] * D[2][1] - D[1][1] * D[2][0]);
        if (!(std::fabs(det) > 0.0) || !std::isfinite(det)) {
            bad_tet = t;
            return "degenerate tetrahedron " + std::to_string(t);
        }
        double inv = 1.0 / det;
        double* B = &out.Bm[9 * (size_t)t];
        B[0] = (D[1][1] * D[2][2] - D[1][2] * D[2][1]) * inv;
        B[1] = (D[0][2] * D[2][1] - D[0][1] * D[2][2]) * inv;
        B[2] = (D[0][1] * D[1][2] - D[0][2] * D[1][1]) * inv;
        B[3] = (D[1][2] * D[2][0] - D[1][0] * D[2][2]) * inv;
        B[4] = (D[0][0] * D[2][2] - D[0][2] * D[2][0]) * inv;
        B[5] = (D[0][2] * D[1][0] - D[0][0] * D[1][2]) * inv;
        B[6] = (D[1][0] * D[2][1] - D[1][1] * D[2][0]) * inv;
        B[7] = (D[0][1] * D[2][0] - D[0][0] * D[2][1]) * inv;
        B[8] = (D[0][0] * D[1][1] - D[0][1] * D[1][0]) * inv;
        double vol = std::fabs(det) / 6.0;
        out.vol[t] = vol;
        out.w[t] = k_proj * vol;
        for (int a = 0; a < 4; ++a) out.mass[v[a]] += density * vol / 4.0;
    }
    return "";
}

// shape gradient g_a (a = 0..3) of tet t: F = sum_a x_a g_a^T
static inline void shape_grad(const double* B, double g[4][3]) {
    for (int a = 1; a < 4; ++a)
        for (int d = 0; d < 3; ++d) g[a][d] = B[3 * (a - 1) + d];
    for (int d = 0; d < 3; ++d) g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
}

Csr assemble_Av(int n_v, int n_t, const int32_t* T, const RestData& rd, double h,
                const std::vector<int32_t>& vid, int n) {
    // triplets -> CSR with summation
    std::vector<std::vector<std::pair<int32_t, double>>> rows(n);
    for (int t = 0; t < n_t; ++t) {
        double g[4][3];
        shape_grad(&rd.Bm[9 * (size_t)t], g);
        double s = h * h * rd.w[t];
        for (int a = 0; a < 4; ++a) {
            int ra = vid[T[4 * (size_t)t + a]];
            if (ra < 0) continue;
            for (int b = 0; b < 4; ++b) {
                int rb = vid[T[4 * (size_t)t + b]];
                if (rb < 0) continue;
                double v = s * (g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2]);
                rows[ra].push_back({rb, v});
            }
        }
    }
    for (int v = 0; v < n_v; ++v)
        if (vid[v] >= 0) rows[vid[v]].push_back({vid[v], rd.mass[v]});
    Csr A;
    A.n = n;
    A.ptr.assign(n + 1, 0);
    for (int r = 0; r < n; ++r) {
        auto& R = rows[r];
        std::sort(R.begin(), R.end(), [](auto& x, auto& y) { return x.first < y.first; });
        int32_t last = -1;
        for (auto& e : R) {
            if (e.first == last) {
                A.val.back() += e.second;
            } else {
                A.col.push_back(e.first);
                A.val.push_back(e.second);
                last = e.first;
            }
        }
        A.ptr[r + 1] = (int64_t)A.col.size();
    }
    return A;
}

// ---------------------------------------------------------------------------
// geometric nested dissection with one-sided vertex separators
// ---------------------------------------------------------------------------
namespace {
struct ND {
    const Csr& A;
    const std::vector<double>& X;
    std::vector<int32_t> order;
    std::vector<int32_t> side;   // scratch: 0 none, 1 left, 2 right
    ND(const Csr& A_, const std::vector<double>& X_) : A(A_), X(X_), side(A_.n, 0) {}

    void run(std::vector<int32_t> v) {
        if (v.size() <= 48) {
            std::sort(v.begin(), v.end());
            order.insert(order.end(), v.begin(), v.end());
            return;
        }
        // disconnected pieces (separate objects, or parts a cut isolated) need no separator:
        // dissect each on its own, so every object gets its own etree
        {
            for (int32_t i : v) side[i] = 4;
            std::vector<std::vector<int32_t>> comps;
            for (int32_t s0 : v) {
                if (side[s0] != 4) continue;
                std::vector<int32_t> cmp{s0};
                side[s0] = 5;
                for (size_t q = 0; q < cmp.size(); ++q) {
                    const int32_t i = cmp[q];
                    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p)
                        if (side[A.col[p]] == 4) { side[A.col[p]] = 5; cmp.push_back(A.col[p]); }
                }
                comps.push_back(std::move(cmp));
            }
            for (int32_t i : v) side[i] = 0;
            if (comps.size() > 1) {
                for (auto& cmp : comps) run(std::move(cmp));
                return;
            }
        }
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (int32_t i : v)
            for (int d = 0; d < 3; ++d) {
                lo[d] = std::min(lo[d], X[3 * (size_t)i + d]);
                hi[d] = std::max(hi[d], X[3 * (size_t)i + d]);
            }
        int ax = 0;
        for (int d = 1; d < 3; ++d)
            if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
        if (!(hi[ax] - lo[ax] > 0)) {
            std::sort(v.begin(), v.end());
            order.insert(order.end(), v.begin(), v.end());
            return;
        }
        // split at the median coordinate (ties kept together by value)
        std::vector<double> c(v.size());
        for (size_t k = 0; k < v.size(); ++k) c[k] = X[3 * (size_t)v[k] + ax];
        std::vector<double> cs = c;
        std::nth_element(cs.begin(), cs.begin() + cs.size() / 2, cs.end());
        double med = cs[cs.size() / 2];
        std::vector<int32_t> L, R;
        for (size_t k = 0; k < v.size(); ++k) (c[k] < med ? L : R).push_back(v[k]);
        if (L.empty() || R.empty()) {
            L.clear();
            R.clear();
            for (size_t k = 0; k < v.size(); ++k) (c[k] <= med ? L : R).push_back(v[k]);
        }
        if (L.empty() || R.empty()) {
            std::sort(v.begin(), v.end());
            order.insert(order.end(), v.begin(), v.end());
            return;
        }
        for (int32_t i : L) side[i] = 1;
        for (int32_t i : R) side[i] = 2;
        // one-sided separators: boundary of L (touching R) and of R (touching L)
        std::vector<int32_t> SL, SR;
        for (int32_t i : L) {
            for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p)
                if (side[A.col[p]] == 2) { SL.push_back(i); break; }
        }
        for (int32_t i : R) {
            for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p)
                if (side[A.col[p]] == 1) { SR.push_back(i); break; }
        }
        bool useL = SL.size() <= SR.size();
        const std::vector<int32_t>& S = useL ? SL : SR;
        for (int32_t i : S) side[i] = 3;
        std::vector<int32_t> L2, R2;
        for (int32_t i : L) if (side[i] != 3) L2.push_back(i);
        for (int32_t i : R) if (side[i] != 3) R2.push_back(i);
        for (int32_t i : v) side[i] = 0;
        std::vector<int32_t> Sv(S.begin(), S.end());
        run(std::move(L2));
        run(std::move(R2));
        std::sort(Sv.begin(), Sv.end());
        order.insert(order.end(), Sv.begin(), Sv.end());
    }
};
}  // namespace

std::vector<int32_t> nested_dissection(const Csr& A, const std::vector<double>& coords) {
    ND nd(A, coords);
    std::vector<int32_t> all(A.n);
    std::iota(all.begin(), all.end(), 0);
    nd.run(std::move(all));
    return nd.order;
}

Csr permute_sym(const Csr& A, const std::vector<int32_t>& perm) {
    int n = A.n;
    std::vector<int32_t> inv(n);
    for (int k = 0; k < n; ++k) inv[perm[k]] = k;
    Csr C;
    C.n = n;
    C.ptr.assign(n + 1, 0);
    for (int k = 0; k < n; ++k) C.ptr[k + 1] = C.ptr[k] + (A.ptr[perm[k] + 1] - A.ptr[perm[k]]);
    C.col.resize(C.ptr[n]);
    C.val.resize(C.ptr[n]);
    for (int k = 0; k < n; ++k) {
        int o = perm[k];
        std::vector<std::pair<int32_t, double>> r;
        for (int64_t p = A.ptr[o]; p < A.ptr[o + 1]; ++p) r.push_back({inv[A.col[p]], A.val[p]});
        std::sort(r.begin(), r.end(), [](auto& x, auto& y) { return x.first < y.first; });
        for (size_t q = 0; q < r.size(); ++q) {
            C.col[C.ptr[k] + q] = r[q].first;
            C.val[C.ptr[k] + q] = r[q].second;
        }
    }
    return C;
}

// Liu's elimination tree with path compression (symmetric CSR, uses j < i entries)
std::vector<int32_t> etree(const Csr& A) {
    int n = A.n;
    std::vector<int32_t> parent(n, -1), anc(n, -1);
    for (int i = 0; i < n; ++i) {
        for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
            int j = A.col[p];
            while (j != -1 && j < i) {
                int jn = anc[j];
                anc[j] = i;
                if (jn == -1) { parent[j] = i; break; }
                j = jn;
            }
        }
    }
    return parent;
}

std::vector<int32_t> postorder(const std::vector<int32_t>& parent) {
    int n = (int)parent.size();
    std::vector<int32_t> head(n, -1), next(n, -1), post;
    post.reserve(n);
    for (int j = n - 1; j >= 0; --j) {
        if (parent[j] == -1) continue;
        next[j] = head[parent[j]];
        head[parent[j]] = j;
    }
    std::vector<int32_t> stack;
    for (int r = 0; r < n; ++r) {
        if (parent[r] != -1) continue;
        stack.push_back(r);
        while (!stack.empty()) {
            int p = stack.back();
            int c = head[p];
            if (c == -1) {
                stack.pop_back();
                post.push_back(p);
            } else {
                head[p] = next[c];
                stack.push_back(c);
            }
        }
    }
    return post;   // post[k] = node visited k-th
}

// up-looking Cholesky (row k of L from a sparse triangular solve over ereach(k))
// Up-looking Cholesky.  Rows of different elimination trees never interact (the etree of a
// block-diagonal A is a forest, and in postorder every tree is a contiguous index range), so
// the trees are factorised in parallel, each by the same sequential row loop.
bool cholesky(const Csr& A, const std::vector<int32_t>& parent, Factor& f) {
    const int n = A.n;
    f.n = n;
    f.parent = parent;
    // tree ranges [lo, root] (postorder: a subtree occupies root - size + 1 .. root)
    std::vector<int32_t> size(n, 1);
    for (int i = 0; i < n; ++i)
        if (parent[i] >= 0) size[parent[i]] += size[i];
    std::vector<std::pair<int32_t, int32_t>> trees;
    for (int i = 0; i < n; ++i)
        if (parent[i] < 0) trees.push_back({i - size[i] + 1, i});
    const int nt = (int)trees.size();
    std::vector<int32_t> cnt(n, 1);
    // pass 1: column counts
#pragma omp parallel
    {
        std::vector<int32_t> mark(n, -1), pattern;
#pragma omp for schedule(dynamic, 1)
        for (int t = 0; t < nt; ++t)
            for (int k = trees[t].first; k <= trees[t].second; ++k) {
                pattern.clear();
                mark[k] = k;
                for (int64_t p = A.ptr[k]; p < A.ptr[k + 1]; ++p) {
                    int j = A.col[p];
                    if (j >= k) continue;
                    while (j != -1 && mark[j] != k) {
                        pattern.push_back(j);
                        mark[j] = k;
                        j = parent[j];
                    }
                }
                for (int j : pattern) cnt[j]++;
            }
    }
    f.Lp.assign(n + 1, 0);
    for (int j = 0; j < n; ++j) f.Lp[j + 1] = f.Lp[j] + cnt[j];
    f.Li.assign(f.Lp[n], 0);
    f.Lx.assign(f.Lp[n], 0.0);
    std::vector<int64_t> fill(n);
    for (int j = 0; j < n; ++j) fill[j] = f.Lp[j] + 1;   // slot 0 of each column = diagonal
    std::vector<int> bad(nt, -1);
#pragma omp parallel
    {
        std::vector<int32_t> mark(n, -1), pattern;
        std::vector<double> x(n, 0.0);
#pragma omp for schedule(dynamic, 1)
        for (int t = 0; t < nt; ++t)
            for (int k = trees[t].first; k <= trees[t].second; ++k) {
                pattern.clear();
                mark[k] = k;
                for (int64_t p = A.ptr[k]; p < A.ptr[k + 1]; ++p) {
                    int j = A.col[p];
                    if (j >= k) continue;
                    while (j != -1 && mark[j] != k) {
                        pattern.push_back(j);
                        mark[j] = k;
                        j = parent[j];
                    }
                }
                std::sort(pattern.begin(), pattern.end());
                double d = 0.0;
                for (int64_t p = A.ptr[k]; p < A.ptr[k + 1]; ++p) {
                    int j = A.col[p];
                    if (j < k) x[j] = A.val[p];
                    else if (j == k) d = A.val[p];
                }
                for (int j : pattern) {
                    double lkj = x[j] / f.Lx[f.Lp[j]];
                    x[j] = 0.0;
                    for (int64_t p = f.Lp[j] + 1; p < fill[j]; ++p) x[f.Li[p]] -= f.Lx[p] * lkj;
                    d -= lkj * lkj;
                    f.Li[fill[j]] = k;
                    f.Lx[fill[j]] = lkj;
                    fill[j]++;
                }
                if (!(d > 0.0) || !std::isfinite(d)) {
                    bad[t] = k;
                    break;
                }
                f.Li[f.Lp[k]] = k;
                f.Lx[f.Lp[k]] = std::sqrt(d);
            }
    }
    for (int t = 0; t < nt; ++t)
        if (bad[t] >= 0) {
            f.bad_col = bad[t];
            return false;
        }
    return true;
}

void sparse_inverse(const Factor& f, double drop_tol, Inverse& K, int n_threads) {
    sparse_inverse_structure(f, K);
    sparse_inverse_values(f, drop_tol, K, n_threads);
}

void sparse_inverse_structure(const Factor& f, Inverse& K) {
    int n = f.n;
    K.n = n;
    K.parent = f.parent;
    K.depth.assign(n, 0);
    for (int i = n - 1; i >= 0; --i) K.depth[i] = f.parent[i] < 0 ? 0 : K.depth[f.parent[i]] + 1;
    std::vector<int32_t> size(n, 1), nchild(n, 0);
    for (int i = 0; i < n; ++i)
        if (f.parent[i] >= 0) { size[f.parent[i]] += size[i]; nchild[f.parent[i]]++; }
    K.first.resize(n);
    K.height = 0;
    for (int i = 0; i < n; ++i) {
        K.first[i] = i - size[i] + 1;
        K.height = std::max(K.height, K.depth[i] + 1);
    }
    K.rowptr.assign(n + 1, 0);
    K.colptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        K.rowptr[i + 1] = K.rowptr[i] + size[i];
        K.colptr[i + 1] = K.colptr[i] + K.depth[i] + 1;
    }
    K.nnz = K.rowptr[n];
    // panels: row i+1 continues row i's panel iff parent[i] == i+1 and i+1 has one child
    K.panel_of.assign(n, 0);
    K.panel_start.clear();
    for (int i = 0; i < n; ++i) {
        bool cont = i > 0 && f.parent[i - 1] == i && nchild[i] == 1;
        if (!cont) K.panel_start.push_back(i);
        K.panel_of[i] = (int)K.panel_start.size() - 1;
    }
    K.panel_start.push_back(n);
    K.ptop.resize(n);
    for (size_t p = 0; p + 1 < K.panel_start.size(); ++p)
        for (int i = K.panel_start[p]; i < K.panel_start[p + 1]; ++i) K.ptop[i] = K.panel_start[p + 1] - 1;
    K.Krow.assign(K.nnz, 0.f);
    K.Kcol.assign(K.nnz, 0.f);
}

void sparse_inverse_values(const Factor& f, double drop_tol, Inverse& K, int n_threads) {
    const int n = f.n;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel
    {
        std::vector<double> w(n, 0.0);
        std::vector<int32_t> chain;
#pragma omp for schedule(dynamic, 16)
        for (int j = 0; j < n; ++j) {
            chain.clear();
            for (int l = j; l != -1; l = f.parent[l]) chain.push_back(l);
            w[j] = 1.0;
            double kjj = 0.0;
            for (size_t q = 0; q < chain.size(); ++q) {
                int l = chain[q];
                double kl = w[l] / f.Lx[f.Lp[l]];
                w[l] = 0.0;
                for (int64_t p = f.Lp[l] + 1; p < f.Lp[l + 1]; ++p) w[f.Li[p]] -= f.Lx[p] * kl;
                if (q == 0) kjj = kl;
                if (drop_tol > 0 && std::fabs(kl) < drop_tol * std::fabs(kjj)) kl = 0.0;
                float kf = (float)kl;
                K.Kcol[K.colptr[j] + (int64_t)q] = kf;
                K.Krow[K.rowptr[l] + (j - K.first[l])] = kf;
            }
        }
    }
}

void trim_dropped(Inverse& K) {
    K.firstk.assign(K.n, 0);
#pragma omp parallel for schedule(dynamic, 64)
    for (int r = 0; r < K.n; ++r) {
        const float* row = K.Krow.data() + K.rowptr[r];
        int j = K.first[r];
        while (j < r && row[j - K.first[r]] == 0.f) ++j;
        K.firstk[r] = j;
    }
}

void build_worklists(const Inverse& K, WorkLists& wl, int p1_chunk_cols) {
    int n = K.n;
    wl = WorkLists();
    // ---- pass 1: per panel, 32-row blocks, column chunks of the block's range [f, r0 + nr)
    int npan = (int)K.panel_start.size() - 1;
    for (int p = 0; p < npan; ++p) {
        int rs = K.panel_start[p], re = K.panel_start[p + 1];
        for (int r0 = rs; r0 < re; r0 += 32) {
            int nr = std::min(32, re - r0);
            int cend = r0 + nr;
            int f = cend - 1;   // the block's kept columns [min firstk, r0 + nr)
            for (int l = 0; l < nr; ++l) f = std::min(f, (int)K.firstk[r0 + l]);
            P1Block b{r0, nr, 0, wl.p1_parts};
            int bi = (int)wl.p1b.size();
            for (int c0 = f; c0 < cend; c0 += p1_chunk_cols) {
                int c1 = std::min(cend, c0 + p1_chunk_cols);
                wl.p1.push_back(P1Item{r0, nr, c0, c1, bi, wl.p1_parts + b.nitems, 0});
                b.nitems++;
            }
            wl.p1_parts += b.nitems;
            wl.p1b.push_back(b);
        }
    }
    // heavy items first (longest-processing-time order); partial slots are fixed per item
    std::stable_sort(wl.p1.begin(), wl.p1.end(), [](const P1Item& a, const P1Item& b) {
        return (int64_t)a.nrows * (a.c1 - a.c0) > (int64_t)b.nrows * (b.c1 - b.c0);
    });
    // ---- pass 2: 32-column blocks with their sorted cover rows
    std::vector<int32_t> mark(n, -1);
    std::vector<int32_t> cov;
    std::vector<std::pair<int64_t, P2Block>> blocks;
    for (int c0 = 0; c0 < n; c0 += 32) {
        int nc = std::min(32, n - c0);
        int bi = c0 / 32;
        cov.clear();
        for (int j = c0; j < c0 + nc; ++j)
            for (int i = j; i != -1 && mark[i] != bi; i = K.parent[i]) {
                mark[i] = bi;
                if (K.firstk[i] <= c0 + nc - 1) cov.push_back(i);   // rows with a kept entry in the block
            }
        std::sort(cov.begin(), cov.end());
        P2Block b{c0, nc, (int)wl.cover.size(), (int)(wl.cover.size() + cov.size()), 0};
        wl.cover.insert(wl.cover.end(), cov.begin(), cov.end());
        blocks.push_back({(int64_t)cov.size(), b});
    }
    std::stable_sort(blocks.begin(), blocks.end(), [](auto& a, auto& b) { return a.first > b.first; });
    for (auto& b : blocks) wl.p2b.push_back(b.second);
}

void build_tiles(const Inverse& K, WorkLists& wl, std::vector<float>& T1, std::vector<float>& T2) {
    auto kval = [&](int r, int j) -> float {   // K[r][j], 0 outside the skyline
        if (j < K.first[r] || j > r) return 0.f;
        return K.Krow[K.rowptr[r] + (j - K.first[r])];
    };
    int64_t n1 = 0;
    for (auto& it : wl.p1) n1 += (int64_t)it.nrows * 32 * ((it.c1 - it.c0 + 31) / 32);
    T1.assign(n1, 0.f);
    int64_t o = 0;
    for (auto& it : wl.p1) {
        it.toff = o;
        for (int jc = it.c0; jc < it.c1; jc += 32) {
            for (int q = 0; q < 32; ++q) {
                const int j = jc + q;
                if (j >= it.c1) continue;
                for (int l = 0; l < it.nrows; ++l) T1[o + (int64_t)q * it.nrows + l] = kval(it.r0 + l, j);
            }
            o += (int64_t)it.nrows * 32;
        }
    }
    int64_t n2 = 0;
    for (auto& b : wl.p2b) n2 += 1024LL * ((b.list1 - b.list0 + 31) / 32);
    T2.assign(n2, 0.f);
    o = 0;
    for (auto& b : wl.p2b) {
        b.toff = o;
        for (int k0 = b.list0; k0 < b.list1; k0 += 32) {
            for (int q = 0; q < 32 && k0 + q < b.list1; ++q) {
                const int r = wl.cover[k0 + q];
                for (int l = 0; l < b.ncols; ++l) T2[o + 32 * q + l] = kval(r, b.c0 + l);
            }
            o += 1024;
        }
    }
}

int build_batched(const Inverse& K, const WorkLists& wl, int unit_tiles, std::vector<BUnit>& u1,
                  std::vector<float>& T1p, std::vector<BUnit>& u2, int& nblocks1) {
    auto kval = [&](int r, int j) -> float {
        if (j < K.first[r] || j > r) return 0.f;
        return K.Krow[K.rowptr[r] + (j - K.first[r])];
    };
    u1.clear();
    u2.clear();
    int64_t ntot = 0;
    auto block_c0 = [&](const P1Block& b) {   // the block's kept columns start
        int c0 = b.r0 + b.nrows - 1;
        for (int l = 0; l < b.nrows; ++l) c0 = std::min(c0, (int)K.firstk[b.r0 + l]);
        return c0;
    };
    for (auto& b : wl.p1b) {
        const int c0 = block_c0(b), c1 = b.r0 + b.nrows;   // columns [c0, c1)
        ntot += (c1 - c0 + 31) / 32;
    }
    T1p.assign(ntot * 1024, 0.f);
    int64_t o = 0;
    int nparts = 0;
    nblocks1 = (int)wl.p1b.size();
    for (int bi = 0; bi < (int)wl.p1b.size(); ++bi) {
        const P1Block& b = wl.p1b[bi];
        const int c0 = block_c0(b), c1 = b.r0 + b.nrows;
        const int nt = (c1 - c0 + 31) / 32;
        const int nu = (nt + unit_tiles - 1) / unit_tiles;
        const int part0 = nu > 1 ? nparts : -1;
        for (int u = 0; u < nu; ++u) {
            BUnit U{};
            U.r0 = b.r0;
            U.nr = b.nrows;
            U.c0 = c0 + 32 * unit_tiles * u;
            U.ntiles = std::min(unit_tiles, nt - unit_tiles * u);
            U.list0 = part0;
            U.block = bi;
            U.part = nu > 1 ? nparts++ : -1;
            U.nparts = nu;
            U.toff = o + (int64_t)1024 * unit_tiles * u;
            u1.push_back(U);
        }
        for (int t = 0; t < nt; ++t)
            for (int q = 0; q < 32; ++q) {
                const int j = c0 + 32 * t + q;
                if (j >= c1) break;
                for (int l = 0; l < b.nrows; ++l) T1p[o + 1024LL * t + 32 * q + l] = kval(b.r0 + l, j);
            }
        o += 1024LL * nt;
    }
    // longest units first (the tail of each instance chunk is then short)
    std::stable_sort(u1.begin(), u1.end(), [](const BUnit& a, const BUnit& b) { return a.ntiles > b.ntiles; });
    for (auto& b : wl.p2b) {
        BUnit U{};
        U.r0 = b.c0;
        U.nr = b.ncols;
        U.c0 = b.c0;
        U.nlist = b.list1 - b.list0;
        U.ntiles = (U.nlist + 31) / 32;
        U.list0 = b.list0;
        U.block = -1;
        U.part = -1;
        U.nparts = 1;
        U.toff = b.toff;
        u2.push_back(U);
    }
    std::stable_sort(u2.begin(), u2.end(), [](const BUnit& a, const BUnit& b) { return a.ntiles > b.ntiles; });
    return nparts;
}

void tc_tiles(const std::vector<float>& T, std::vector<float>& Ttc) {
    const size_t nt = T.size() / 1024;
    Ttc.assign(2048 * nt, 0.f);
#pragma omp parallel for schedule(static)
    for (long long t = 0; t < (long long)nt; ++t) {
        const float* src = T.data() + 1024 * (size_t)t;
        float* hi = Ttc.data() + 2048 * (size_t)t;
        float* lo = hi + 1024;
        for (int q = 0; q < 32; ++q)
            for (int l = 0; l < 32; ++l) {
                const float v = src[q * 32 + l];
                auto rn = [](float a) {   // round to nearest tf32
                    uint32_t b;
                    std::memcpy(&b, &a, 4);
                    b = (b + 0x1000u) & 0xFFFFE000u;
                    float r;
                    std::memcpy(&r, &b, 4);
                    return r;
                };
                const float h = rn(v);
                const int d = (l / 8) * 256 + (q / 4) * 32 + (l % 8) * 4 + (q % 4);
                hi[d] = h;
                lo[d] = rn(v - h);
            }
    }
}

void build_contact_passes(const Inverse& K, const std::vector<int32_t>& sv, ContactPasses& cp) {
    cp = ContactPasses();
    const int ns = (int)sv.size();
    auto is_anc = [&](int r, int a) { return K.first[r] <= a && a <= r; };   // r ancestor-or-self of a
    auto kval = [&](int r, int a) { return K.Krow[K.rowptr[r] + (a - K.first[r])]; };
    // chain pass: blocks of 32 slots
    std::vector<int32_t> mark(K.n, -1), rows;
    for (int c0 = 0; c0 < ns; c0 += 32) {
        const int nb = std::min(32, ns - c0);
        rows.clear();
        for (int s = c0; s < c0 + nb; ++s)
            for (int r = sv[s]; r >= 0; r = K.parent[r])
                if (mark[r] != c0) { mark[r] = c0; rows.push_back(r); }
        std::sort(rows.begin(), rows.end());
        BUnit u{};
        u.c0 = c0;
        u.nr = nb;
        u.list0 = (int32_t)cp.cover.size();
        u.nlist = (int32_t)rows.size();
        u.ntiles = (u.nlist + 31) / 32;
        u.part = 0;
        u.nparts = 1;
        u.toff = (int64_t)cp.Tc.size();
        cp.cover.insert(cp.cover.end(), rows.begin(), rows.end());
        for (int t = 0; t < u.ntiles; ++t) {
            const size_t base = cp.Tc.size();
            cp.Tc.resize(base + 1024, 0.f);
            for (int q = 0; q < 32 && 32 * t + q < u.nlist; ++q) {
                const int r = rows[32 * t + q];
                for (int l = 0; l < nb; ++l)
                    if (is_anc(r, sv[c0 + l])) cp.Tc[base + 32 * q + l] = kval(r, sv[c0 + l]);
            }
        }
        cp.uc.push_back(u);
    }
    // scatter pass: the union of all chains, blocks of 32 rows; each row reaches the slots whose
    // vertex lies in its subtree [first(r), r], a contiguous slot range (slots ascending)
    std::fill(mark.begin(), mark.end(), -1);
    for (int s = 0; s < ns; ++s)
        for (int r = sv[s]; r >= 0 && mark[r] < 0; r = K.parent[r]) { mark[r] = 1; cp.rows.push_back(r); }
    std::sort(cp.rows.begin(), cp.rows.end());
    const int nu = (int)cp.rows.size();
    for (int r0 = 0; r0 < nu; r0 += 32) {
        const int nb = std::min(32, nu - r0);
        int lo = ns, hi = 0;
        for (int l = 0; l < nb; ++l) {
            const int r = cp.rows[r0 + l];
            const int a = (int)(std::lower_bound(sv.begin(), sv.end(), K.first[r]) - sv.begin());
            const int b = (int)(std::upper_bound(sv.begin(), sv.end(), r) - sv.begin());
            if (a < b) { lo = std::min(lo, a); hi = std::max(hi, b); }
        }
        if (lo >= hi) continue;
        BUnit u{};
        u.r0 = r0;
        u.nr = nb;
        u.c0 = lo;
        u.ntiles = (hi - lo + 31) / 32;
        u.part = 0;
        u.nparts = 1;
        u.toff = (int64_t)cp.Ts.size();
        for (int t = 0; t < u.ntiles; ++t) {
            const size_t base = cp.Ts.size();
            cp.Ts.resize(base + 1024, 0.f);
            for (int q = 0; q < 32 && lo + 32 * t + q < ns; ++q) {
                const int a = sv[lo + 32 * t + q];
                for (int l = 0; l < nb; ++l) {
                    const int r = cp.rows[r0 + l];
                    if (is_anc(r, a)) cp.Ts[base + 32 * q + l] = kval(r, a);
                }
            }
        }
        cp.us.push_back(u);
    }
}

// ---- plane-layout tensor-core K-passes: 64-output units (see host.hpp) ----
static void put_tile64(float* dst, const float* src /*[32 q][64 l]*/) {
    auto rn = [](float a) {   // round to nearest tf32
        uint32_t b;
        std::memcpy(&b, &a, 4);
        b = (b + 0x1000u) & 0xFFFFE000u;
        float r;
        std::memcpy(&r, &b, 4);
        return r;
    };
    float* hi = dst;
    float* lo = dst + 2048;
    for (int q = 0; q < 32; ++q)
        for (int l = 0; l < 64; ++l) {
            const float v = src[q * 64 + l];
            const float h = rn(v);
            const int d = (l / 8) * 256 + (q / 4) * 32 + (l % 8) * 4 + (q % 4);
            hi[d] = h;
            lo[d] = rn(v - h);
        }
}

void build_plane_units(const Inverse& K, int unit_tiles, PlaneUnits& pu) {
    pu = PlaneUnits();
    const int n = K.n;
    auto kval = [&](int r, int j) -> float {
        if (j < K.first[r] || j > r) return 0.f;
        return K.Krow[K.rowptr[r] + (j - K.first[r])];
    };
    // pass 1: 64-row blocks
    struct B1 { int r0, nr, c0, nt; };
    std::vector<B1> blocks;
    int64_t nt1 = 0;
    for (int r0 = 0; r0 < n; r0 += 64) {
        const int nr = std::min(64, n - r0);
        int c0 = r0;
        for (int l = 0; l < nr; ++l) c0 = std::min(c0, (int)K.firstk[r0 + l]);
        const int nt = (r0 + nr - c0 + 31) / 32;
        blocks.push_back({r0, nr, c0, nt});
        nt1 += nt;
    }
    pu.tiles1 = nt1;
    pu.T1.assign((size_t)nt1 * 4096, 0.f);
    std::vector<int64_t> boff(blocks.size());
    {
        int64_t o = 0;
        for (size_t b = 0; b < blocks.size(); ++b) { boff[b] = o; o += (int64_t)blocks[b].nt * 4096; }
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (long long b = 0; b < (long long)blocks.size(); ++b) {
        const B1& B = blocks[b];
        std::vector<float> tile(32 * 64);
        for (int t = 0; t < B.nt; ++t) {
            std::fill(tile.begin(), tile.end(), 0.f);
            for (int q = 0; q < 32; ++q) {
                const int j = B.c0 + 32 * t + q;
                if (j >= B.r0 + B.nr) break;
                for (int l = 0; l < B.nr; ++l) tile[q * 64 + l] = kval(B.r0 + l, j);
            }
            put_tile64(pu.T1.data() + boff[b] + (int64_t)t * 4096, tile.data());
        }
    }
    pu.nblocks1 = (int)blocks.size();
    for (int b = 0; b < (int)blocks.size(); ++b) {
        const B1& B = blocks[b];
        const int nu = (B.nt + unit_tiles - 1) / unit_tiles;
        const int part0 = nu > 1 ? pu.nparts1 : -1;
        for (int u = 0; u < nu; ++u) {
            BUnit U{};
            U.r0 = B.r0;
            U.nr = B.nr;
            U.c0 = B.c0 + 32 * unit_tiles * u;
            U.ntiles = std::min(unit_tiles, B.nt - unit_tiles * u);
            U.list0 = part0;
            U.block = b;
            U.part = nu > 1 ? pu.nparts1++ : -1;
            U.nparts = nu;
            U.toff = boff[b] + (int64_t)4096 * unit_tiles * u;
            pu.u1.push_back(U);
        }
    }
    std::stable_sort(pu.u1.begin(), pu.u1.end(), [](const BUnit& a, const BUnit& b) { return a.ntiles > b.ntiles; });
    // pass 2: 64-column blocks and their cover rows
    std::vector<int32_t> mark(n, -1), cov;
    int64_t nt2 = 0;
    for (int c0 = 0; c0 < n; c0 += 64) {
        const int nc = std::min(64, n - c0);
        const int bi = c0 / 64;
        cov.clear();
        for (int j = c0; j < c0 + nc; ++j)
            for (int i = j; i != -1 && mark[i] != bi; i = K.parent[i]) {
                mark[i] = bi;
                if (K.firstk[i] <= c0 + nc - 1) cov.push_back(i);
            }
        std::sort(cov.begin(), cov.end());
        BUnit U{};
        U.r0 = c0;
        U.c0 = c0;
        U.nr = nc;
        U.list0 = (int32_t)pu.cover.size();
        U.nlist = (int32_t)cov.size();
        U.ntiles = (U.nlist + 31) / 32;
        U.block = -1;
        U.part = -1;
        U.nparts = 1;
        U.toff = nt2 * 4096;
        nt2 += U.ntiles;
        pu.cover.insert(pu.cover.end(), cov.begin(), cov.end());
        pu.u2.push_back(U);
    }
    pu.tiles2 = nt2;
    pu.T2.assign((size_t)nt2 * 4096, 0.f);
#pragma omp parallel for schedule(dynamic, 4)
    for (long long b = 0; b < (long long)pu.u2.size(); ++b) {
        const BUnit& U = pu.u2[b];
        std::vector<float> tile(32 * 64);
        for (int t = 0; t < U.ntiles; ++t) {
            std::fill(tile.begin(), tile.end(), 0.f);
            for (int q = 0; q < 32 && 32 * t + q < U.nlist; ++q) {
                const int r = pu.cover[U.list0 + 32 * t + q];
                for (int l = 0; l < U.nr; ++l) tile[q * 64 + l] = kval(r, U.c0 + l);
            }
            put_tile64(pu.T2.data() + U.toff + (int64_t)t * 4096, tile.data());
        }
    }
    std::stable_sort(pu.u2.begin(), pu.u2.end(), [](const BUnit& a, const BUnit& b) { return a.ntiles > b.ntiles; });
}

}  // namespace simhost
