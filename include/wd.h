/*
 * wd.h -- C ABI of the B200-native (sm_100a, fp64) mass-consistent wind
 * downscaling library (Mandel, Farguell, Kochanski, Mallia, Hilburn,
 * arXiv 2101.08453; "P:n" = /root/reference/PAPER.md line n).
 *
 * The library solves, on a terrain-following grid of isoparametric 8-node
 * hexahedra, the generalised Poisson problem (Eq. (4))
 *        -div A^{-1} grad lambda = div u0,  lambda = 0 on dOmega \ Gamma,
 * in its variational form (Eq. (5)) with 2x2x2 Gauss quadrature on
 * the left and one-point quadrature on the right, by a multigrid
 * V-cycle (Eq. (6)-(7)), and recovers u = u0 + A^{-1} grad lambda
 * at element centres (Eq. (3)).  A = diag(a1^2,a2^2,a3^2).
 *
 * Conventions for every array argument (all IEEE fp64, C-contiguous):
 *   node arrays   [n3][n2][n1]       i fastest, node (i,j,k), n1 = nx + 1 ...
 *                 (X, Y, Z, f, lambda, lambda0)
 *   element arrays [3][n3-1][n2-1][n1-1]  SoA components u, v, w (u0, u)
 *   Gamma (the terrain, natural boundary) is the k = 0 node plane; the
 *   Dirichlet set D is i in {0, n1-1}, j in {0, n2-1}, k = n3-1.
 * Pointers may be device pointers (cudaMalloc / torch CUDA tensors) or host
 * pointers; host arrays are staged through device memory inside the call
 * and the call then synchronises `stream` before returning.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 * stream-ordered on it, except wd_assemble (synchronous) and wd_solve (which
 * synchronises once per V-cycle to test convergence, or once per solve with
 * wd_options.device_loop).
 *
 * Ownership: the caller owns every array passed in or out; the context owns
 * only internal copies and workspaces, allocated by wd_assemble and freed by
 * wd_destroy (wd_device_bytes reports their size).  A context is not
 * thread-safe; use one per host thread / stream.
 *
 * Errors: every int-returning call returns WD_OK (0) or a WD_E_* code and
 * never aborts; wd_last_error() returns a thread-local message for the last
 * non-zero return of the calling thread.
 */
#ifndef WD_H
#define WD_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
    WD_OK = 0,
    WD_E_INVAL = 1,     /* n1,n2 < 3; n3 < 2; NULL pointer; a_d <= 0 or non-finite; tol not in (0,1) */
    WD_E_MESH = 2,      /* Z not increasing in k, or detJ <= 0 at a Gauss point (message names element) */
    WD_E_NOCONV = 3,    /* max_cycles reached; lambda valid, report filled */
    WD_E_DIVERGED = 4,  /* relative residual grew 10x over 3 consecutive cycles */
    WD_E_NONFINITE = 5, /* residual norm became NaN/Inf */
    WD_E_CUDA = 6,      /* CUDA runtime failure */
    WD_E_NCCL = 7,      /* communicator failure (multi-GPU) */
    WD_E_OOM = 8,       /* device allocation failed */
    WD_E_INTERNAL = 9   /* planner/Galerkin invariant violated */
};

/* Semicoarsening rule of P:192-202 (readings C1/C1b of DESIGN.md):
 *  COUPLING_CUR   ratio (h3/h1)(a3/a1), vertical test with the current-level h1 (default)
 *  COUPLING_PAPER ratio (h3/h1)(a3/a1), vertical test with the coarsened h1 (P:196-199 literal)
 *  VERBATIM       ratio h3/(h1 a3) exactly as printed, coarsened h1
 *  FULL           base method: 2x2x2 coarsening at every level */
enum { WD_RULE_COUPLING_CUR = 0, WD_RULE_COUPLING_PAPER = 1, WD_RULE_VERBATIM = 2, WD_RULE_FULL = 3 };

/* Schedule of the 4-colour smoother.  Both compute the same
 * iterate bit for bit (same operations in the same order per node):
 *  FUSED   one launch per sweep: all four colour phases pipelined over k in
 *          shared-memory tiles filled by TMA (k_gs_fused2.cu; k_gs_fused.cu for
 *          levels of >= 2^31 entries); on slab levels one 2-row halo exchange
 *          of lambda per sweep (default)
 *  PHASED  four launches per sweep, one per colour (k_mg.cu gs_phase_kernel);
 *          on slab levels halo rows exchanged after colours 1 and 3
 * and a different smoother (north_star "vertical-column line
 * relaxation parallel over (i,j)"):
 *  LINE    the same colour groups and order, each free column solved exactly
 *          (tridiagonal in k, Thomas algorithm) given the latest values of the
 *          other columns; four launches per sweep (k_mg.cu line_phase_kernel) */
enum { WD_SMOOTH_FUSED = 0, WD_SMOOTH_PHASED = 1, WD_SMOOTH_LINE = 2 };

typedef struct wd_ctx wd_ctx;

typedef struct {
    int pre_smooth;          /* GS sweeps before the coarse correction (default 2; "four smoothing steps") */
    int post_smooth;         /* GS sweeps after it (default 2) */
    int max_cycles;          /* wd_solve cycle cap (default 100) */
    int coarsest_max_free;   /* direct coarsest solve at <= this many free unknowns (default 4096) */
    int coarse_iters;        /* GS sweeps on the coarsest level when it is larger (default 50) */
    int coarsen_rule;        /* WD_RULE_* (default WD_RULE_COUPLING_CUR) */
    int use_graph;           /* capture the V-cycle as a CUDA graph (default 1) */
    long long gather_below_nodes; /* slab decomposition: replicate ("gather") coarse levels with
                                     fewer nodes than this (default 2,000,000) */
    int rank, nranks;        /* slab decomposition in node rows j:
                                nranks = 1: one GPU, whole grid (default; with rank = 0 and
                                  a one-rank nccl_comm the NCCL code path runs, no neighbours);
                                nranks > 1, rank >= 0: this process is `rank` of nranks (one
                                  GPU per process, NCCL over NVLink, nccl_comm required); the
                                  node/element arrays passed to every call are this rank's
                                  rows [max(j_begin-2,0), min(j_end+2,n2)) (2 halo rows);
                                nranks > 1, rank = -1: virtual ranks -- the whole grid on this
                                  GPU split into nranks slabs with the same halo exchanges done
                                  as device copies (arrays are the whole grid) */
    void* nccl_comm;         /* ncclComm_t of the nranks processes (wd_nccl_comm_init) */
    int j_begin, j_end;      /* owned node rows [j_begin, j_end) of this rank; must equal
                                wd_partition_rows(n2, nranks, rank) */
    int profile;             /* 1: CUDA events around level-0 smoothing and each V-cycle (default 0) */
    int smoother;            /* WD_SMOOTH_* (default WD_SMOOTH_FUSED) */
    int line_from_level;     /* per-level smoother (SURVEY 8(f) f1 "per-level decisions"):
                                vertical line relaxation (the WD_SMOOTH_LINE sweep) on the
                                levels >= this one, `smoother` below it; -1 = `smoother` on
                                every level (default -1) */
    int device_loop;         /* 1: wd_solve runs its cycle loop on the device -- one CUDA graph
                                whose conditional WHILE node repeats the cycle while a kernel's
                                convergence test says so, no host round trip per cycle -- when
                                the context is eligible (one GPU, fused smoother, graphs on,
                                profile off); same iterates, history and cycle count as the
                                host-driven loop.  Default 0 (host loop): measured no faster
                                (scripts/device_loop_timing.py, profiles/r2_device_loop.jsonl) */
    int overlap_halo;        /* slabs (nranks > 1): each fused sweep on a distributed level runs
                                the tile rows holding the first / last 2 owned rows first and
                                exchanges those rows on a second stream while the interior tiles
                                run (boundary-first); results identical to 0.  Default 0: with
                                virtual ranks on one GPU it measured slower (the boundary launch
                                runs one tile row per CTA on part of the SMs); untested on
                                several GPUs (profiles/r2_virtual_ranks.jsonl) */
} wd_options;

typedef struct {
    int status;              /* WD_OK / WD_E_NOCONV / WD_E_DIVERGED / WD_E_NONFINITE */
    int cycles;              /* V-cycles performed */
    int converged;           /* rel_res_final <= tol */
    int nlevels;             /* hierarchy depth (incl. the fine level) */
    double rel_res0;         /* ||f - K lambda0|| / ||f|| over free nodes (abs if ||f|| = 0) */
    double rel_res_final;
    double rate;             /* (rel_N / rel_1)^(1/(N-1)); rel_1/rel_0 if N = 1 */
    double rel_res_hist[256];/* [c] = relative residual after cycle c, [0] = initial */
    int dims[32][3];         /* node dims (n1,n2,n3) per level */
    int coarse_direct;       /* 1 dense direct coarsest solve, 0 GS fallback */
    int coarse_free;         /* free unknowns on the coarsest level */
} wd_report;

/* Fill opt with the defaults above. */
void wd_default_options(wd_options* opt);

/* Setup once per mesh (P:107-111 assembly, P:151-158 + P:192-202 hierarchy).
 * X, Y, Z: node coordinates [n3][n2][n1] (in NCCL mode [n3][slab rows][n1],
 * n2 still being the grid's row count); a1, a2, a3 > 0: penalty constants of
 * A = diag(a1^2, a2^2, a3^2).  Validates the mesh (WD_E_MESH names
 * the lowest failing element), assembles the 27-point operator (stored as 14
 * symmetric coefficients per node), plans the coarsening, forms the Galerkin
 * coarse operators and factors the coarsest level.  opt may be NULL
 * (defaults).  Synchronous; the caller may free X, Y, Z on return.
 * On success *out receives a new context. */
int wd_assemble(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                double a1, double a2, double a3, const wd_options* opt, void* stream,
                wd_ctx** out);

/* RHS of Eq. (5) by one-point quadrature:
 * f_p = sum_{e ni p} -8 detJ_e(0) grad N_p(0) . u0_e, f = 0 on D.
 * u0: element array; f: node array (written). */
int wd_rhs(wd_ctx* ctx, const double* u0, double* f, void* stream);

/* One multigrid V-cycle on lambda (in/out node array) for K lambda = f
 * (Eq. (7)): pre-smoothing, f_c = P^T (f - K lambda), recursive
 * coarse solve from 0, lambda += P lambda_c, post-smoothing.  lambda entries
 * on D are treated as 0 and returned as 0.  rel_res_out (nullable, host)
 * receives ||f - K lambda||/||f|| after the cycle (synchronises). */
int wd_vcycle(wd_ctx* ctx, double* lambda, const double* f, double* rel_res_out, void* stream);

/* Iterate V-cycles from lambda0 (NULL = zero start; entries on D ignored)
 * until ||f - K lambda||/||f|| <= rel_tol (in (0,1)), max_cycles, divergence
 * or a non-finite residual.  f = 0 returns lambda = 0 after 0 cycles.
 * lambda (out) may alias lambda0.  rep (nullable, host) is filled.
 * The test is made after every cycle.  With the fused smoother (and at least
 * one pre-smoothing sweep on a multi-level hierarchy) the residual of iterate
 * c is returned by the first sweep of cycle c+1, which reads that iterate
 * unchanged; if the test passes the sweep's output is discarded, so the
 * result and the cycle count are those of "cycle, then test" (the residual
 * agrees with a separate residual pass to rounding, about 1e-13 of ||f||).
 * Returns WD_OK, WD_E_NOCONV, WD_E_DIVERGED or WD_E_NONFINITE (lambda is the
 * last iterate in every case). */
int wd_solve(wd_ctx* ctx, const double* f, const double* lambda0, double rel_tol,
             double* lambda, wd_report* rep, void* stream);

/* Wind recovery, Eq. (3) with grad lambda at element centres:
 * u_e = u0_e + A^{-1} J_e(0)^{-T} sum_a lambda_a grad_xi N_a(0).
 * lambda: node array; u0, u: element arrays (u may alias u0). */
int wd_recover_wind(wd_ctx* ctx, const double* lambda, const double* u0, double* u,
                    void* stream);

/* Free the context and all its device memory (NULL is a no-op).  The NCCL
 * communicator passed in the options is not destroyed. */
void wd_destroy(wd_ctx* ctx);

/* ---- slab decomposition helpers ----
 * Owned node rows [*j_begin, *j_end) of `rank` among nranks: an even split
 * floor(n2 r / R) .. floor(n2 (r+1) / R).  Every rank must own >= 4 rows. */
void wd_partition_rows(int n2, int nranks, int rank, int* j_begin, int* j_end);
/* Host-only inspection of the slab decomposition (SURVEY 8(e)
 * requirement (1); no device work, callable without a GPU): the hierarchy
 * wd_assemble builds for these global node dims, penalty constants, options
 * and planner inputs (h1 = sqrt(dx dy), h3[n3-1] = layer thicknesses of the
 * minimum-terrain column, reading C2), seen from `rank` of `nranks`.
 *   *nlevels, *gather (first replicated level, -1: none);
 *   lev[8 l + 0..2]  global node dims of level l (l < max_levels);
 *   lev[8 l + 3]     1 if level l is distributed (slab rows), 0 if replicated;
 *   lev[8 l + 4..5]  global rows [a, b) this rank holds (owned + halo rows);
 *   lev[8 l + 6..7]  global rows [a, b) it owns (distributed) or computes
 *                    before the gather (replicated);
 *   msgs[5 m + 0..4] the messages of one w-row halo exchange (the ncclSend /
 *                    ncclRecv pairs the V-cycle issues; virtual ranks copy the
 *                    same rows) on every distributed level: level, peer,
 *                    1 send / 0 receive, first global row, rows;  *nmsgs.
 * Returns WD_OK; WD_E_INVAL for bad dims/ranks (also when a rank would own
 * fewer than 4 rows) or when an output array is too short. */
int wd_plan_decomposition(int n1, int n2, int n3, double a1, double a2, double a3, double h1,
                          const double* h3, const wd_options* opt, int nranks, int rank, int w,
                          int* nlevels, int* gather, int* lev, int max_levels, int* msgs,
                          int max_msgs, int* nmsgs);
/* ncclGetUniqueId (libnccl.so.2 is loaded at run time) into id[128]; rank 0
 * calls it and broadcasts the bytes to the other ranks. */
int wd_nccl_unique_id(char id[128]);
/* ncclCommInitRank; *comm receives the ncclComm_t for wd_options.nccl_comm. */
int wd_nccl_comm_init(const char id[128], int nranks, int rank, void** comm);
/* First replicated (gathered) level of a decomposed context, -1 if none. */
int wd_gather_level(const wd_ctx* ctx);

/* Thread-local message of the last failing call ("" if none). */
const char* wd_last_error(void);

/* ---- inspection entry points (used by the parity tests; same conventions) ---- */

/* Bytes of device memory owned by the context. */
long long wd_device_bytes(const wd_ctx* ctx);
/* Number of levels; node dims of level l (dims[3] = n1, n2, n3). */
int wd_num_levels(const wd_ctx* ctx);
int wd_level_dims(const wd_ctx* ctx, int level, int dims[3]);
/* Plan of the transition level -> level+1: *horizontal, kept node layers. */
int wd_level_plan(const wd_ctx* ctx, int level, int* horizontal, int* kept, int* nkept);
/* Full 27-point stencil of level l as [n3][n2][n1][27] (o = (dx+1)+3(dy+1)+9(dz+1)),
 * both directions of each symmetric coupling (device or host output). */
int wd_get_stencil(wd_ctx* ctx, int level, double* K27, void* stream);
/* y = K_l x on free nodes, 0 on D (node arrays of level l). */
int wd_apply(wd_ctx* ctx, int level, const double* x, double* y, void* stream);
/* `sweeps` 4-colour bottom-up Gauss-Seidel sweeps on level l. */
int wd_smooth(wd_ctx* ctx, int level, double* x, const double* f, int sweeps, void* stream);
/* fc = P^T r from level l to level l+1 (r treated as 0 on D). */
int wd_restrict(wd_ctx* ctx, int level, const double* r, double* fc, void* stream);
/* x += P xc from level l+1 to level l on free nodes. */
int wd_prolong(wd_ctx* ctx, int level, const double* xc, double* x, void* stream);
/* Coarsest-level solve x = K_L^{-1} f (or the GS fallback), node arrays of the last level. */
int wd_coarse_solve(wd_ctx* ctx, const double* f, double* x, void* stream);
/* ||f - K x||_2 over free nodes of level 0 and its ratio to ||f||_2 (host outputs). */
int wd_residual_norm(wd_ctx* ctx, const double* x, const double* f, double* abs_out,
                     double* rel_out, void* stream);

/* Device-side profile gathered while opt.profile = 1 (CUDA events, also inside
 * the captured V-cycle graph), accumulated over wd_solve/wd_vcycle calls:
 *   out[0] ms in plain level-0 sweeps        out[1] their number
 *   out[2] ms in V-cycles                    out[3] V-cycles
 *   out[4] ms in residual-norm passes        out[5] residual-norm passes
 *   out[6] ms in level-0 sweeps that also return the residual of their input
 *          (the first sweep of a cycle in wd_solve)   out[7] their number
 *   out[8] ms in the level-0 residual r = f - K lambda before the restriction
 *          (one per V-cycle)                 out[9] their number
 *   out[10], out[11]: plain / residual-returning level-0 sweeps executed in
 *          wd_solve's split cycles, timed or not (wd_solve times the sweeps
 *          of every 4th cycle only; these counts weight the sampled times)
 * A sweep is one launch of the fused smoother (four launches with
 * WD_SMOOTH_PHASED).  Returns the number of values written (<= n, <= 12). */
int wd_profile_read(const wd_ctx* ctx, double* out, int n);
/* Reset the accumulated profile. */
void wd_profile_reset(wd_ctx* ctx);
/* Cumulative number of kernel launches executed by this library in this
 * process (a CUDA-graph replay counts its kernel nodes). */
long long wd_launch_count(void);
/* ---- steps either side of the solver ---------------- */

/* Terrain-following mesh from a terrain array ("terrain-following
 * grid"; the domain-top reading C13 of DESIGN.md):
 *   X(i,j,k) = x0 + i dx,  Y(i,j,k) = y0 + j dy,
 *   Z(i,j,k) = zs(i,j) + zeta[k] (H - zs(i,j)) / zeta[n3-1].
 * zs: terrain [n2][n1] (device or host); zeta: n3 level heights, HOST array,
 * zeta[0] = 0, strictly increasing; H: the flat domain top; X, Y, Z: node
 * arrays [n3][n2][n1] (written; device or host).  Every cell of the result is
 * valid (detJ > 0) when H > zs everywhere.  Synchronous.  Errors: WD_E_INVAL
 * (NULL, n < 2, dx/dy <= 0, non-finite, zeta not increasing from 0),
 * WD_E_MESH (H <= zs at some column; the message names the first one). */
int wd_build_mesh(const double* zs, int n1, int n2, double x0, double y0, double dx, double dy,
                  const double* zeta, int n3, double H, double* X, double* Y, double* Z,
                  void* stream);

/* Interpolation of a coarse (WRF-like) wind to the element centres of a mesh
 * (the fire grid's initial wind u0 comes from the
 * atmospheric model).  uc: [3][nzc][nyc][nxc] (u, v, w) on the horizontal grid
 * (xc0 + a DXc, yc0 + b DYc) at heights above ground hc[0..nzc-1] (HOST
 * array, strictly increasing); X, Y, Z: node arrays [n3][n2][n1]; u0: element
 * array [3][n3-1][n2-1][n1-1] (written).  Per element: centre = mean of its 8
 * nodes, height above ground = centre Z - mean of its column's 4 bottom-node
 * Z; value = trilinear interpolant in (x, y, height), each coordinate clamped
 * to the coarse grid.  Synchronous.  Errors: WD_E_INVAL. */
int wd_interp_wind(const double* uc, int nxc, int nyc, int nzc, double xc0, double yc0,
                   double DXc, double DYc, const double* hc, const double* X, const double* Y,
                   const double* Z, int n1, int n2, int n3, double* u0, void* stream);

/* Mass-consistency diagnostics of a wind u (element array) on the context's
 * mesh (Eq. (1) "div u = 0"; reading C12): the one-point weak divergence
 * D1(u)_mu = sum_e 8 detJ_e(0) grad mu(0) . u_e over the free nodes mu;
 * out[0] = its l2 norm, out[1] = its max abs (host array).  For the
 * recovered wind D1(u) = (K1 - K) lambda + (K lambda - f) (C12): not zero,
 * but the projection lowers it below D1(u0) = -f.  Synchronous. */
int wd_mass_consistency(wd_ctx* ctx, const double* u, double out[2], void* stream);

/* One model time step with the persistent hierarchy: f = RHS(u0),
 * lambda = solve (warm-started from the caller's lambda when warm != 0, from
 * zero otherwise) to rel_tol, u = u0 + A^-1 grad lambda.  lambda is in/out
 * (node array), u out (element array); rep nullable.  Returns wd_solve's
 * status (the wind is recovered also for WD_E_NOCONV). */
int wd_downscale_step(wd_ctx* ctx, const double* u0, double* lambda, int warm, double rel_tol,
                      double* u, wd_report* rep, void* stream);

/* Time one internal kernel (or step) on the context's own buffers with CUDA
 * events: which = 0 GS sweep (the context's smoother), 1 residual apply,
 * 2 restrict (level -> level+1), 3 prolong, 4 V-cycle (level 0), 5 residual
 * norm (level 0), 6 Galerkin (level -> level+1), 7 level-0 assembly, 8 GS
 * sweep as 4 colour-phase launches, 9 fused GS sweep that also returns the
 * residual of its input (the first sweep of a cycle in wd_solve).  One untimed
 * warm-up, then *ms_out = mean over `reps`.  Overwrites internal vectors
 * (and, for 6/7, recomputes identical operators). */
int wd_bench_kernel(wd_ctx* ctx, int which, int level, int reps, double* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* WD_H */
