/*
 * sim.h -- C ABI of the B200-native sparse-inverse local-global solver with
 * non-smooth frictional contact (arXiv 2503.15078, "Fast But Accurate").
 *
 * Citations: P:L<n> = line n of the paper's LaTeX source.
 *
 * The four calls of the paper's problem statement (Alg. 4):
 *   sim_create               mesh, material, time step h
 *   sim_build_sparse_inverse K = L^-1 of A = M + h^2 sum w G^T G    (Thm 1, Alg. 2)
 *   sim_set_contacts         J rows, Delassus D = J K^T K J^T, r
 *   sim_step                 frames x (predict; iterations x L-G)
 * plus state/pin accessors, statistics and test hooks (sim_debug_*).
 *
 * Conventions
 *  - Every function returns SIM_OK (0) or a negative SIM_E_* code; the
 *    message of the last error on the calling thread is sim_last_error().
 *  - All input pointers are borrowed for the duration of the call and deep-
 *    copied; the library never retains caller pointers.  Output buffers are
 *    caller-owned.  Host pointers unless stated otherwise.
 *  - A handle owns all of its device memory and binds the CUDA device that is
 *    current at sim_create.  A handle is not thread-safe.
 *  - Call order: create -> build_sparse_inverse -> (set_contacts)* -> step.
 *    Violations return SIM_E_STATE.  Every call except sim_step gives the
 *    strong guarantee (no state change on error).
 *  - Vertex indices in all calls are the caller's original indices; the
 *    library's internal (elimination-tree postorder) numbering is hidden.
 *  - Results are deterministic for a given device and configuration (fixed
 *    reduction orders, no floating-point atomics).
 *  - Instances: one handle may hold n_instances independent scenes that share
 *    the mesh topology, rest shape, material, h and therefore K (BASELINE
 *    config 5).  Each instance has its own state and contact set;
 *    every sim_step advances all of them.  The K-passes then read each K tile
 *    once for all instances (3 x n_instances right-hand sides).
 */
#ifndef SIM_H_
#define SIM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIM_OK            0
#define SIM_E_INVALID    -1  /* null/size/NaN input, mu < 0, nu not in [0,0.5), bad normal   */
#define SIM_E_DEGENERATE -2  /* zero-volume tetrahedron (index in the message)               */
#define SIM_E_NOT_SPD    -3  /* non-positive Cholesky pivot (column in the message)          */
#define SIM_E_STATE      -4  /* call made out of order                                       */
#define SIM_E_CUDA       -5  /* CUDA runtime failure or no usable device                     */
#define SIM_E_OOM        -6  /* host or device allocation failed                             */
#define SIM_E_NONFINITE  -7  /* non-finite state detected; state rolled back to frame start  */
#define SIM_E_LIMIT      -8  /* a size exceeds a documented implementation limit             */

typedef struct sim_handle sim_handle;

/* Tetrahedral mesh.  rest_positions [n_vertices][3] in metres;
 * tets [n_tets][4] (orientation not required); fixed [n_vertices] Dirichlet
 * mask (nonzero = pinned) or NULL.  n_instances: scenes sharing this mesh
 * (0 or 1 = one scene; at most 65535). */
typedef struct {
    int32_t n_vertices;
    int32_t n_tets;
    const double  *rest_positions;
    const int32_t *tets;
    const uint8_t *fixed;
    int32_t n_instances;
} sim_mesh;

/* Material models of the local step (eq. PD local). */
enum { SIM_NEOHOOKEAN = 0, SIM_COROTATED = 1, SIM_ARAP = 2 };

/* density kg/m^3, youngs Pa, poisson in [0,0.5) (Table 3 columns).
 * proj_stiffness k of w_i = k vol_i; 0 selects k = 2 mu_Lame.
 * gravity m/s^2 (f_ext = M g).  cr_iterations: CR budget, 0 -> 10. */
typedef struct {
    int32_t model;
    double  density, youngs, poisson;
    double  proj_stiffness;
    double  gravity[3];
    int32_t cr_iterations;
} sim_material;

/* One contact pair (App. A).
 * kind 0: unilateral normal row + two Coulomb friction rows (t1, t2);
 * kind 1: one bilateral row along `normal` with compliance.
 * verts/weights: up to 4 vertices, (J x)_row = c . sum_a w_a x_a.
 * normal must be unit length; tangents all-zero -> Gram-Schmidt frame
 * (e = least-aligned axis, t1 = normalize(e - (n.e) n), t2 = n x t1).
 * offset: d_n = n . p_obstacle (+ min separation) or d_b.
 * obstacle_velocity: d_f = t . v_obstacle.  Contacts may not touch
 * pinned vertices. */
typedef struct {
    int32_t kind;
    int32_t n_verts;
    int32_t verts[4];
    double  weights[4];
    double  normal[3];
    double  tangent1[3];
    double  tangent2[3];
    double  offset;
    double  obstacle_velocity[3];
    double  mu;
    double  compliance;
} sim_contact;

/* Analytic obstacle for the GPU proximity query (sim_detect_contacts; the paper's
 * "simple proximity queries").  kind 0 plane: point a, unit normal b (the
 * solid side is -b); kind 1 sphere: centre a, radius; kind 2 capsule: segment a-b, radius.
 * mu: Coulomb coefficient of its contacts; velocity: rigid obstacle velocity (d_f). */
typedef struct {
    int32_t kind;
    int32_t pad;
    double  a[3];
    double  b[3];
    double  radius;
    double  mu;
    double  velocity[3];
} sim_obstacle;

typedef struct {
    int64_t n_vertices, n_free, n_tets;
    int64_t nnz_K;             /* nnz of the vertex-level K = L^-1 (stored twice: row- and column-major) */
    int64_t nnz_L;
    int32_t etree_height;
    int32_t n_panels;          /* fundamental supernodes (rows sharing their first column)               */
    int32_t n_contacts, n_contact_vertices;   /* summed over instances */
    int64_t frames_done;
    double  last_cr_residual;  /* max over the instance(s) of |r| of the last CR solve (fp64), -1 if none */
    double  max_abs_phi_n;     /* max |phi_n| (NCP function) over unilateral contacts at the last iterate */
    int32_t n_active, n_stick, n_slip;   /* frame-end classification (reading A21: lambda_n > 0; stick:
                                            |ydot_f| <= r_f (mu lambda_n - |lambda_f|); slip otherwise)     */
    int32_t kernels_per_frame; /* kernel launches in one captured frame                                  */
    double  build_seconds;     /* host time of sim_build_sparse_inverse                                  */
    int64_t h2d_contact_bytes; /* host->device bytes of the last contact commit                          */
    int32_t n_instances;
    int64_t nonfinite_rollbacks; /* instance-frames rolled back to x_t, v_t (non-finite x or v), total    */
    int64_t gram_rows_computed;  /* last contact commit: Delassus Gram rows computed ...                  */
    int64_t gram_rows_reused;    /* ... and rows copied from the previous commit (sim_set_schur_reuse)    */
    double  build_phase_seconds[5]; /* precompute: assemble A_v, ordering, Cholesky, K = L^-1, tile layouts  */
    double  max_cone_violation; /* max over unilateral contacts of max(0, |lambda_f| - mu max(lambda_n, 0)) */
    double  max_penetration;    /* max over unilateral contacts of max(0, -(J_n x - d_n)) at the frame end  */
    int32_t instance;           /* the instance these per-instance fields describe, -1 = all            */
    int64_t kpass_bytes;        /* K values one K-pass pair streams per L-G iteration (both tile streams of the
                                   handle's path, fp32; S > 1: the tensor-core hi + lo streams)         */
    int64_t nnz_K_kept;         /* entries of K left nonzero after the drop tolerance (= nnz_K at tol 0) */
} sim_stats;

/* Validate the mesh and material, compute rest data (Dm^-1, volumes, lumped
 * mass, w_i = k vol_i).  h > 0 is the time step (s).  No device work yet
 * except binding the current device. */
int sim_create(const sim_mesh *mesh, const sim_material *mat, double h, sim_handle **out);

/* Assemble A_v over free vertices (A = A_v (x) I_3), order it (geometric
 * nested dissection + elimination-tree postorder), factor A_v = L L^T in fp64,
 * compute K = L^-1 column by column over ancestor chains (Thm 1), store K in
 * fp32 twice (row-major and column-major values-only panels), build the
 * K-pass work lists and upload everything.  drop_tolerance: entries with
 * |K_ij| < tol |K_jj| are dropped (0 = exact Theorem-1 pattern; reading A25): each row's stored
 * range starts at its first kept column, so the K-pass streams shrink by the dropped leading
 * entries (sim_stats.kpass_bytes); the result approximates A^-1 (no 1e-5 parity claim). */
int sim_build_sparse_inverse(sim_handle *h, double drop_tolerance);

/* Replace the contact set of one instance (n may be 0).  Validates and builds
 * the rows on the host; the next sim_step (or debug accessor) uploads the
 * contact sets of all instances in one batch and computes on the device
 * G = K[:,Vc]^T K[:,Vc] per instance, the Delassus diagonal and the
 * preconditioner r_n = h^2 D_jj, r_f = h D_jj (eq. schur-complement P:L858,
 * eq. complementarity preconditioner P:L919-925).  The constraint solve (CR,
 * P:L1047-1049) runs in one thread-block cluster per instance when the set
 * has n <= 1024 contacts on <= 1024 distinct vertices and its fp64 working set
 * 184 n + 72 n_vertices bytes fits 227 KB (about 900 single-vertex contacts).
 * Larger sets (any size, e.g. a multi-object pile with soft-soft contact rows)
 * use the grid CR, which needs n_instances == 1 (SIM_E_LIMIT otherwise); its
 * Gram G is stored per etree component (G is zero across components). */
int sim_set_contacts(sim_handle *h, int32_t instance, const sim_contact *contacts, int32_t n);
/* Multipliers across sim_set_contacts (warm start, reading A10w): a contact that is the same constraint as
 * one of the instance's previous set -- same kind, vertices, weights and row directions
 * (n, t1, t2); offset, mu, compliance and obstacle velocity may change -- keeps that
 * contact's lambda rows (the first unused match in the previous order); other contacts start
 * from lambda = 0. */
/* The same for instances first .. first+count-1 at once: counts[count],
 * contacts concatenated in instance order.  All-or-nothing on error. */
int sim_set_contacts_batch(sim_handle *h, int32_t first, int32_t count, const int32_t *counts,
                           const sim_contact *contacts);

/* Proximity query on the device: for every candidate vertex (original
 * ids, n_cand of them, e.g. the surface; pinned vertices are skipped) of `instance`, the
 * signed distance to each obstacle surface at the current positions; the nearest obstacle
 * wins (one contact per vertex, reading A31) and a unilateral contact is created when the
 * distance is below `margin` (metres): normal = outward surface normal at the closest point
 * p, offset d_n = n . p (so y = n . x - d_n is the signed distance), Gram-Schmidt tangents,
 * the obstacle's mu and velocity.  The contacts replace the instance's set in candidate
 * order (as sim_set_contacts); *n_found (may be NULL) receives their count.  Candidates and
 * obstacles are borrowed for the call.  SIM_E_INVALID on bad kinds, non-unit plane normals,
 * negative radii / margin, candidate ids out of range; SIM_E_LIMIT as sim_set_contacts. */
/* The instance's current contact set as stored (original vertex ids, the normalised normal,
 * the tangents in use, offset, mu, compliance; obstacle_velocity is returned as its tangential
 * part d_f1 t1 + d_f2 t2, the only part the method uses).  *n (may be NULL) receives the
 * count; out may be NULL to query it; SIM_E_INVALID if cap < count. */
int sim_get_contacts(sim_handle *h, int32_t instance, sim_contact *out, int32_t capacity, int32_t *n);

int sim_detect_contacts(sim_handle *h, int32_t instance, const sim_obstacle *obstacles, int32_t n_obstacles,
                        const int32_t *candidates, int32_t n_candidates, double margin, int32_t *n_found);

/* Advance `frames` frames of `iterations` local-global iterations each
 * (Alg. 4).  Per frame: s = x_t + h v_t + h^2 g; the iterate starts at x^0 = s with
 * lambda^0 = 0 (readings A9, A10), or -- sim_set_warm_start(h, 1) -- at x^0 = x_t + h v_t with the
 * previous frame's lambda (A9w, A10w: Alg. 4 never resets lambda; see sim_set_contacts for the
 * carry across a new contact set).  Pinned vertices move by h * their pin velocity per frame.
 * Enqueued on the handle's stream; returns after enqueueing (use sim_synchronize or any
 * blocking accessor). */
int sim_step(sim_handle *h, int32_t frames, int32_t iterations);

/* Block until all work enqueued on the handle's stream is done; checks the
 * device-side failure counter: every frame ends with a check of x and v, and an
 * instance whose frame produced a non-finite value is rolled back to its
 * frame-start state (x_t, v_t) on the device.  Returns SIM_E_NONFINITE (once,
 * with the count in sim_last_error) if any instance-frame was rolled back since
 * the previous call; the running total is sim_stats.nonfinite_rollbacks. */
int sim_synchronize(sim_handle *h);

/* Pinned vertices (the mesh's `fixed` mask) are Dirichlet conditions eliminated from the
 * system (reading A7) that move as "moving positional constraints": each
 * pinned vertex-instance has a velocity, and every frame moves it by h * velocity (its frame-end
 * position is the Dirichlet target of that frame; its v is that velocity).
 * sim_set_pin_velocity: the same velocity v[3] (m/s) for every pinned vertex of every instance.
 * sim_set_pins: per-vertex targets for one instance: pinned_xyz [n_pinned][3] (metres), the
 * positions the pinned vertices take at the end of the NEXT frame, ordered by ascending
 * original vertex index; n_pinned must equal the mesh's pinned-vertex count.  The call sets
 * each pinned vertex's velocity to (target - current position) / h, on the handle's stream after
 * the frames already enqueued, so later frames without a new call continue at that velocity.
 * Both: SIM_E_INVALID on null / non-finite input or a wrong count, SIM_E_STATE before the build;
 * borrowed for the call. */
int sim_set_pin_velocity(sim_handle *h, const double v[3]);
int sim_set_pins(sim_handle *h, int32_t instance, const double *pinned_xyz, int32_t n_pinned);

/* x, v: [n_vertices][3] of one instance in original vertex order (caller
 * buffers; either may be NULL). */
int sim_get_state(sim_handle *h, int32_t instance, double *x, double *v);
int sim_set_state(sim_handle *h, int32_t instance, const double *x, const double *v);
/* Both setters start the affected instances' multipliers from 0 (lambda is part of the state,
 * reading A10); sim_set_lambda sets them explicitly. */
/* Positions of all instances: x [n_instances][n_vertices][3]. */
int sim_get_positions(sim_handle *h, double *x);
/* The same positions, asynchronously: enqueued on the handle's stream after the frames
 * already enqueued, packed on the device into one of two staging buffers and copied to
 * host_dst (caller-owned; pinned memory for real overlap) on a separate copy stream, so the
 * transfer overlaps the next frames.  host_dst must stay valid until sim_wait_positions.
 * Two calls may be in flight (the third waits for the first copy on the device). */
int sim_get_positions_async(sim_handle *h, double *host_dst);
/* Completion of the last sim_get_positions_async: block_host != 0 blocks the calling
 * thread; 0 makes the handle's stream wait (device-side join, for event timing). */
int sim_wait_positions(sim_handle *h, int32_t block_host);
/* States of all instances: x, v [n_instances][n_vertices][3] (either may be NULL). */
int sim_set_states(sim_handle *h, const double *x, const double *v);

/* lambda: [rows] = (lambda_n, lambda_f1, lambda_f2) per unilateral contact,
 * (lambda_b) per bilateral contact of one instance, in the order given to
 * sim_set_contacts: the multipliers the next frame starts from (the most recent step's, carried
 * into the current contact set).  *n_rows (may be NULL) receives the row count; lambda may be
 * NULL to query it; SIM_E_INVALID if capacity < rows. */
int sim_get_lambda(sim_handle *h, int32_t instance, double *lambda, int32_t capacity, int32_t *n_rows);
/* Set the multipliers the next frame of one instance starts from (same row layout; n must be
 * the instance's row count).  Borrowed for the call.  SIM_E_INVALID on a wrong count or a
 * non-finite value. */
int sim_set_lambda(sim_handle *h, int32_t instance, const double *lambda, int32_t n);

/* Statistics.  instance = -1: the whole handle (contact counts and classification summed, residual,
 * |phi|, cone violation and penetration maximised over all instances); 0 <= instance < n_instances:
 * the contact fields of that instance only (the mesh / build / timing fields are the handle's).
 * The frame-end fields describe the state after the last sim_step (lambda and x of its last
 * iteration); they are 0 (last_cr_residual -1) while no frame has run on the current contact
 * set.  Synchronises the handle's stream.  SIM_E_INVALID on a bad instance. */
int sim_get_stats(sim_handle *h, int32_t instance, sim_stats *out);

/* Use a caller-provided cudaStream_t (e.g. torch.cuda.current_stream()). */
int sim_set_stream(sim_handle *h, void *cuda_stream);

/* Kernel timing: when on, the captured frame graph records an event between
 * consecutive kernels; sim_get_kernel_times then returns, per kernel kind
 * (0 predict, 1 contact_eval, 2 local, 3 gather, 4 kpass1, 5 chain_dot, 6 cr,
 * 7 scatter, 8 kpass2, 9 active-set + G_A gather), the summed device ms of
 * the most recent frame.  out must hold >= 10 doubles. */
int sim_set_profiling(sim_handle *h, int on);

/* Constraint-solver selection (same CR algorithm and result up to rounding
 * order): 0 = automatic (cluster CR when the set fits, grid CR otherwise),
 * 1 = cluster CR only (SIM_E_LIMIT if the current set does not fit),
 * 2 = grid CR always (n_instances == 1 only).  Takes effect at the next step. */
int sim_set_cr_mode(sim_handle *h, int32_t mode);

/* NCP function and complementarity preconditioner (the paper's ablation,
 * Fig. 11, P:L883-916 / P:L1200-1214).  ncp_function: 0 = Fischer-Burmeister
 * (App. B.2, the paper's choice), 1 = minimum map (App. B.1).
 * preconditioner: 0 = Delassus diagonal r_n = h^2 D_jj, r_f = h D_jj
 * (eq. complementarity preconditioner), 1 = mass inverse
 * r = h^2 / h [J M^-1 J^T]_jj with the lumped M.  Defaults 0, 0;
 * SIM_E_INVALID on other values.  Takes effect at the next step. */
int sim_set_ncp(sim_handle *h, int32_t ncp_function, int32_t preconditioner);

/* Local-global variant: 0 = projective dynamics (Alg. 1/4; default),
 * 1 = ADMM-PD (Overby et al. 2017, which the paper's implementation is based on,
 * P:L1052 / P:L1340): per-tet dual u (9 floats per tet and instance, allocated
 * here, reset to 0 at every frame), local step on F + u, u <- u + F - p, global
 * step on p - u.  Its fixed point is the implicit-Euler solution (plain PD's
 * is the Moreau-envelope one).  Needs a built handle (SIM_E_STATE otherwise);
 * SIM_E_OOM if the dual cannot be allocated.  Takes effect at the next step. */
int sim_set_admm(sim_handle *h, int32_t on);

/* Frame start: 0 (default) x^0 = s and lambda^0 = 0 every frame (readings A9,
 * A10); 1 x^0 = x_t + h v_t and lambda^0 = the previous frame's lambda (A9w, A10w) -- the reading
 * that reproduces the 0.001 stick/slide resolution of Fig. 11, at the price of a
 * frame map that amplifies rounding near stick.  SIM_E_INVALID on other values.  Takes effect at
 * the next step. */
int sim_set_warm_start(sim_handle *h, int32_t on);

/* Batched K-passes (n_instances > 1): 2 (default; 0 is an alias) = tcgen05 tensor cores: the
 * right-hand sides in fp32 component planes, one CTA per 64-output unit x 128 instances x 3
 * components, kind::tf32 with a 3xTF32 split (V_hi = the raw fp32 tile in shared memory, MN-major;
 * V_lo in TMEM; K_hi / K_lo pre-rounded), TMEM accumulators folded every 4 tiles;
 * 1 = CUDA-core FP32 FMAs; 3 = the tensor-core K-passes with the contact chain / scatter passes on
 * the CUDA cores (accuracy studies).  Takes effect at the next contact commit.  Results agree
 * with FP32 to ~2e-6 relative.  n_instances == 1 always
 * uses the HBM-streaming SpMV kernels.  (mode >> 4) >= 2 sets the fold interval (tuning). */
int sim_set_kpass_mode(sim_handle *h, int32_t mode);

/* Delassus reuse across contact commits (the "reuse strategy ... to exploit shared contact data
 * between consecutive time steps" the paper implements, P:L863 / P:L1016): G[a][b] depends only
 * on the vertex pair, so entries of pairs already in the previous commit of the instance's
 * class are copied and only the rows of new contact vertices are computed (same fp32
 * accumulation order: bitwise the full recomputation).  Off by default (reading A23: the bench
 * recomputes D at every commit).  Cluster-CR scenes only; the grid CR always recomputes. */
int sim_set_schur_reuse(sim_handle *h, int32_t on);

/* Small-scene frame driver: 0 (default) = auto -- a handle with one instance, no contacts and plain
 * PD whose n_free + n_tets <= 1024 runs sim_step's frames x iterations in ONE persistent single-CTA
 * kernel (predict, local step, RHS, both K-passes, integrate and the finite check per frame, with
 * block barriers instead of kernel boundaries: the cfg1 cantilever is launch-latency bound on the
 * graph path); 1 = always the per-frame CUDA graph.  Same method and readings; results agree with
 * the graph path to fp32 rounding (different accumulation order).  SIM_E_INVALID on other values. */
int sim_set_persistent(sim_handle *h, int32_t mode);

/* Local step with n_instances > 1: 0 (default) = when n_instances is even, one thread computes a tet
 * for two instances with packed FP32 (FFMA2 / FMUL2 / FADD2) in lockstep; 1 = one thread per
 * tet-instance (scalar FP32).  Same formulas; results agree to fp32 rounding (FMA contraction order).
 * ADMM-PD always uses the scalar kernel.  SIM_E_INVALID on other values. */
int sim_set_local_mode(sim_handle *h, int32_t mode);
int sim_get_kernel_times(sim_handle *h, double *out, int32_t capacity);

void sim_destroy(sim_handle *h);         /* NULL-safe */

/* Device memory (process-wide, e.g. PyTorch's caching allocator): every device buffer a handle
 * allocates after this call comes from alloc(bytes, ctx) (device memory of the handle's device;
 * NULL -> SIM_E_OOM from the calling API) and goes back through free_(ptr, ctx), called after
 * cudaDeviceSynchronize so that no enqueued work still reads the buffer.  A buffer is always
 * returned to the allocator it came from.  alloc = free_ = NULL restores cudaMalloc / cudaFree.
 * SIM_E_INVALID if exactly one of alloc, free_ is NULL.  Thread-safe. */
int sim_set_allocator(void *(*alloc)(size_t bytes, void *ctx), void (*free_)(void *ptr, void *ctx), void *ctx);
const char *sim_last_error(void);

/* ---------------------------------------------------------------------------
 * Test hooks.  They run exactly the product kernels on caller data.
 * ------------------------------------------------------------------------- */
/* Host-side K (fp64 before fp32 rounding is NOT kept; these are the stored
 * fp32 values): perm[n_free] maps internal free index -> original vertex;
 * parent[n_free]; rowptr[n_free+1] (int64); vals[nnz_K] row-major.  Any
 * pointer may be NULL.  Works without a GPU (host precompute only, see
 * sim_create_host). */
int sim_debug_get_inverse(sim_handle *h, int32_t *perm, int32_t *parent, int64_t *rowptr, float *vals);
/* Create a handle that only runs the host precompute (no device). */
int sim_create_host(const sim_mesh *mesh, const sim_material *mat, double h, sim_handle **out);
/* x_out = A^-1 b on the device via the two K-passes (y = K P b, x = P^T K^T y),
 * b and x_out [n_instances][n_vertices][3] (the batched passes when
 * n_instances > 1); rows of pinned vertices are ignored / zero.  b is rounded
 * to fp32 (the K-pass input precision) before the product. */
int sim_debug_apply_inverse(sim_handle *h, const double *b, double *x_out);
/* (single-instance handles) One local step at positions x [n_vertices][3] with prediction s
 * [n_vertices][3]: returns the per-tet projection P [n_tets][9] (row-major
 * 3x3; NULL to skip) and the global-step residual r = b - A x
 * = M(s - x) + h^2 sum_i w_i G_i^T (P_i - F_i)  [n_vertices][3] (0 on pinned
 * rows; NULL to skip).  Does not modify the simulation state. */
int sim_debug_local(sim_handle *h, const double *x, const double *s, float *P, double *resid);
/* G = K[:,Vc]^T K[:,Vc] for an instance's current contact set: returns the
 * contact vertex list (original ids) and G (row-major, n_cv x n_cv). */
int sim_debug_get_delassus(sim_handle *h, int32_t instance, int32_t *cv, float *G, int32_t capacity);

/* Contact scratch of the most recent L-G iteration (after sim_step):
 * theta, C diagonal and h-vector per row ([3 * n_contacts], rows n, t1, t2;
 * bilateral contacts pad rows 1-2 with theta 0, C 1), dxt = (A^-1 r) at each
 * contact vertex ([n_cv][3]), the contact vertices (original ids, [n_cv]) and
 * D_jj per contact ([n_contacts]).  Any pointer may be NULL. */
int sim_debug_contact_state(sim_handle *h, int32_t instance, double *theta, double *cdiag, double *hvec,
                            double *dxt, int32_t *slot_vertex, double *djj);
/* Schur right-hand side rho = h - Theta J x~ (the CR's input) of the most recent L-G iteration,
 * [3 * n_contacts] (rows n, t1, t2; bilateral contacts pad rows 1-2 with 0).  Test hook. */
int sim_debug_contact_rho(sim_handle *h, int32_t instance, double *rho);
/* Phase timestamps (us since the CR kernel started) of the most recent CR
 * solve: [1] rho built, [2] active set + G_A gathered, [3 + it] after CR
 * iteration it, [20] loop end, [21] epilogue end.  out must hold 32 doubles. */
int sim_debug_cr_timeline(sim_handle *h, double *out);
/* Per-tile timeline of the plane K-passes (CTA (0, 0) of the last pass-1 / pass-2 launch, first 64
 * tiles; out[4][64][8] %globaltimer ns: MMA warp [K tile landed, V_lo(c=0) seen, V_lo(c=2) seen,
 * committed], workers [copies landed, V_lo written, fold done, next copies issued]; out[p][63][0] =
 * CTA start, out[p][62][0] = tile count).  Caller-owned buffer of 2048 values; all zero unless the
 * library was built with -DSIM_PL_TIMELINE (tools/pl_timeline.py).  Returns a cudaError_t code. */
int sim_debug_pl_timeline(unsigned long long *out);
/* Failure-injection hook: the next frame (run outside the captured graph) writes a NaN into
 * vertex 0 of `instance` right after the prediction step, so the end-of-frame check must roll
 * that instance back to its frame-start state and sim_synchronize must report
 * SIM_E_NONFINITE.  SIM_E_INVALID / SIM_E_STATE as the other per-instance accessors. */
int sim_debug_poison(sim_handle *h, int32_t instance);

#ifdef __cplusplus
}
#endif
#endif /* SIM_H_ */
