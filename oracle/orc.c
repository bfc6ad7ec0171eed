/*
 * oracle/orc.c -- TEST INFRASTRUCTURE ONLY (plain, slow, obviously correct).
 *
 * A CPU reference of the mass-consistent wind downscaling hot path of
 * Mandel et al., arXiv 2101.08453 ("P:n" = /root/reference/PAPER.md line n).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA path in paper_2101_08453_b200/.
 *
 * Conventions (natural layout, the paper's grid):
 *   node (i,j,k), i fastest:  p = (k*n2 + j)*n1 + i,  n1 = nx+1 ...
 *   element (i,j,k) has local nodes a = da + 2 db + 4 dc at (i+da, j+db, k+dc)
 *   K is stored FULL: 27 couplings per node, K[p*27 + o],
 *   o = (dx+1) + 3 (dy+1) + 9 (dz+1)   (coupling of p to p + (dx,dy,dz)).
 *   Dirichlet set D ("lambda = 0 on dOmega \ Gamma"): lateral node
 *   planes and the top plane; bottom (Gamma) nodes are free.  Dirichlet is
 *   realised by masking: D rows are never used, lambda_D = 0, r_D = 0
 *   (reading C11).
 *
 * Floating point: IEEE fp64, compiled with -ffp-contract=off (no FMA
 * contraction) so every line below is evaluated as written.
 *
 * Parity status of each function: see DESIGN.md "Oracle pins".  Every
 * function here is pinned by tests/test_oracle_*.py.  The V-cycle and its
 * convergence factor are pinned against a dense recursive V-cycle on 3-4
 * level hierarchies (tests/test_oracle_vcycle_dense.py); at large sizes the
 * factor rests on the same code plus the paper's anchors (P:169-172,
 * P:200-202).
 *
 * The scatter loops run owner-partitioned under OpenMP (own_rows): each
 * thread performs the serial loop in the serial order and adds only into the
 * target rows it owns, so the result is bitwise that of one thread
 * (tests/test_oracle_threads.py).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long long i64;

#define ORC_MAXLEV 32
#define ORC_MAXNZ 256

/* ------------------------------------------------------------------ */
/* small helpers                                                        */
/* ------------------------------------------------------------------ */

static inline i64 nid(int n1, int n2, int i, int j, int k) {
    return ((i64)k * n2 + j) * n1 + i;
}

static inline int is_dir(int n1, int n2, int n3, int i, int j, int k) {
    return i == 0 || i == n1 - 1 || j == 0 || j == n2 - 1 || k == n3 - 1;
}

static inline int o27(int dx, int dy, int dz) { return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1); }

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the parallel regions (tests compare 1 thread with many). */
void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Owner partition of the scatter loops (element assembly, RHS, Galerkin,
 * restriction): inside a parallel region, thread t owns the target rows
 * [*r0, *r1) of n.  Each thread runs the SERIAL loop in its serial order and
 * adds only into the rows it owns, so every target entry receives the same
 * terms in the same order as in the one-thread loop: the result is bitwise
 * that of the serial code (tests/test_oracle_threads.py checks it). */
static void own_rows(int n, int* r0, int* r1) {
#ifdef _OPENMP
    const int t = omp_get_thread_num(), T = omp_get_num_threads();
#else
    const int t = 0, T = 1;
#endif
    *r0 = (int)((i64)n * t / T);
    *r1 = (int)((i64)n * (t + 1) / T);
}

/* ------------------------------------------------------------------ */
/* isoparametric trilinear hexahedron                       */
/* ------------------------------------------------------------------ */

/* Reference-space gradients of the 8 trilinear shape functions
 * N_a(xi) = prod_d (1 + s_d xi_d)/2, s = 2(da,db,dc) - 1.  G[a*3+d]. */
void orc_shape_grad(const double xi[3], double G[24]) {
    for (int a = 0; a < 8; a++) {
        double s0 = 2.0 * (a & 1) - 1.0;
        double s1 = 2.0 * ((a >> 1) & 1) - 1.0;
        double s2 = 2.0 * ((a >> 2) & 1) - 1.0;
        double n0 = 0.5 * (1.0 + s0 * xi[0]);
        double n1 = 0.5 * (1.0 + s1 * xi[1]);
        double n2 = 0.5 * (1.0 + s2 * xi[2]);
        G[a * 3 + 0] = 0.5 * s0 * n1 * n2;
        G[a * 3 + 1] = 0.5 * s1 * n0 * n2;
        G[a * 3 + 2] = 0.5 * s2 * n0 * n1;
    }
}

/* Jacobian J[m][d] = dx_m/dxi_d = sum_a x_{a,m} dN_a/dxi_d; returns det J.
 * Also returns the physical gradients B[a][m] = (J^{-T} grad_xi N_a)_m. */
static double phys_grad(const double xe[24], const double G[24], double B[24]) {
    double J[3][3];
    for (int m = 0; m < 3; m++)
        for (int d = 0; d < 3; d++) {
            double s = 0.0;
            for (int a = 0; a < 8; a++) s += xe[a * 3 + m] * G[a * 3 + d];
            J[m][d] = s;
        }
    double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
               - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
               + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    /* inverse by cofactors: Jinv[d][m] */
    double Ji[3][3];
    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    /* grad_x N = J^{-T} grad_xi N  ->  B[a][m] = sum_d Ji[d][m] G[a][d] */
    for (int a = 0; a < 8; a++)
        for (int m = 0; m < 3; m++) {
            double s = 0.0;
            for (int d = 0; d < 3; d++) s += Ji[d][m] * G[a * 3 + d];
            B[a * 3 + m] = s;
        }
    return det;
}

/* Element stiffness, P:109-110 ("tensor-product Gauss quadrature with two
 * nodes in each dimension") applied to the LHS of Eq. (5):
 *   Ke_ab = sum_g w_g detJ(g) (grad N_a)^T diag(c) (grad N_b),  w_g = 1,
 *   g in {-1/sqrt3, +1/sqrt3}^3, c = (a1^-2, a2^-2, a3^-2) = A^{-1}.
 * Only the upper triangle is integrated; the lower one is its mirror, so Ke is
 * exactly symmetric.  Returns 0, or -(g+1) for the first Gauss point with
 * detJ <= 0. */
int orc_element_stiffness(const double xe[24], const double c[3], double Ke[64]) {
    const double gp = 1.0 / sqrt(3.0);
    double G[24], B[24];
    for (int t = 0; t < 64; t++) Ke[t] = 0.0;
    for (int g = 0; g < 8; g++) {
        double xi[3] = {(g & 1) ? gp : -gp, (g & 2) ? gp : -gp, (g & 4) ? gp : -gp};
        orc_shape_grad(xi, G);
        double det = phys_grad(xe, G, B);
        if (!(det > 0.0)) return -(g + 1);
        for (int a = 0; a < 8; a++)
            for (int b = a; b < 8; b++) {
                double s = 0.0;
                for (int m = 0; m < 3; m++) s += c[m] * B[a * 3 + m] * B[b * 3 + m];
                Ke[a * 8 + b] += det * s;
            }
    }
    for (int a = 0; a < 8; a++)
        for (int b = 0; b < a; b++) Ke[a * 8 + b] = Ke[b * 8 + a];
    return 0;
}

/* One-point (centre) element stiffness K1e_ab = 8 detJ(0) gradN_a(0).C gradN_b(0)
 * (used only by the C12 divergence identity). */
int orc_element_stiffness_onepoint(const double xe[24], const double c[3], double Ke[64]) {
    const double xi[3] = {0.0, 0.0, 0.0};
    double G[24], B[24];
    orc_shape_grad(xi, G);
    double det = phys_grad(xe, G, B);
    if (!(det > 0.0)) return -1;
    for (int a = 0; a < 8; a++)
        for (int b = a; b < 8; b++) {
            double s = 0.0;
            for (int m = 0; m < 3; m++) s += c[m] * B[a * 3 + m] * B[b * 3 + m];
            Ke[a * 8 + b] = 8.0 * det * s;
        }
    for (int a = 0; a < 8; a++)
        for (int b = 0; b < a; b++) Ke[a * 8 + b] = Ke[b * 8 + a];
    return 0;
}

/* Element RHS, P:110-111 ("one-node quadrature at the center of the element")
 * applied to the RHS of Eq. (5), -int grad mu . u0:
 *   fe_a = -8 detJ(0) gradN_a(0) . u0_e   (reference-cube volume 8). */
int orc_element_rhs(const double xe[24], const double u0[3], double fe[8]) {
    const double xi[3] = {0.0, 0.0, 0.0};
    double G[24], B[24];
    orc_shape_grad(xi, G);
    double det = phys_grad(xe, G, B);
    if (!(det > 0.0)) return -1;
    for (int a = 0; a < 8; a++) {
        double s = 0.0;
        for (int m = 0; m < 3; m++) s += B[a * 3 + m] * u0[m];
        fe[a] = -8.0 * det * s;
    }
    return 0;
}

/* grad lambda at the element centre ("the same code for the
 * derivatives ... at the center of each element"). */
int orc_element_grad_centre(const double xe[24], const double lam[8], double g[3]) {
    const double xi[3] = {0.0, 0.0, 0.0};
    double G[24], B[24];
    orc_shape_grad(xi, G);
    double det = phys_grad(xe, G, B);
    for (int m = 0; m < 3; m++) {
        double s = 0.0;
        for (int a = 0; a < 8; a++) s += lam[a] * B[a * 3 + m];
        g[m] = s;
    }
    return det > 0.0 ? 0 : -1;
}

static void gather_xe(const double* X, const double* Y, const double* Z, int n1, int n2,
                      int i, int j, int k, double xe[24]) {
    for (int a = 0; a < 8; a++) {
        i64 p = nid(n1, n2, i + (a & 1), j + ((a >> 1) & 1), k + ((a >> 2) & 1));
        xe[a * 3 + 0] = X[p];
        xe[a * 3 + 1] = Y[p];
        xe[a * 3 + 2] = Z[p];
    }
}

static i64 enode(int n1, int n2, int i, int j, int k, int a) {
    return nid(n1, n2, i + (a & 1), j + ((a >> 1) & 1), k + ((a >> 2) & 1));
}

/* Mesh validation: Z strictly increasing along every vertical
 * edge and detJ > 0 at the 8 Gauss points.  Returns -1 if valid, else the
 * lowest linear element index e = (k*ny + j)*nx + i that fails; *what = 0
 * for a Z-monotonicity failure, g+1 for Gauss point g. */
i64 orc_validate_mesh(const double* X, const double* Y, const double* Z, int n1, int n2,
                      int n3, int* what) {
    int nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    double xe[24], Ke[64];
    const double c[3] = {1.0, 1.0, 1.0};
    for (int k = 0; k < nz; k++)
        for (int j = 0; j < ny; j++)
            for (int i = 0; i < nx; i++) {
                i64 e = ((i64)k * ny + j) * nx + i;
                for (int a = 0; a < 4; a++) {
                    i64 pb = enode(n1, n2, i, j, k, a);
                    i64 pt = enode(n1, n2, i, j, k, a + 4);
                    if (!(Z[pt] > Z[pb])) { if (what) *what = 0; return e; }
                }
                gather_xe(X, Y, Z, n1, n2, i, j, k, xe);
                int rc = orc_element_stiffness(xe, c, Ke);
                if (rc < 0) { if (what) *what = -rc; return e; }
            }
    return -1;
}

/* ------------------------------------------------------------------ */
/* steps either side of the path                       */
/* ------------------------------------------------------------------ */

/* Terrain-following mesh ("terrain-following grid"; the domain top
 * reading C13 of DESIGN.md; SPEC build_mesh):
 *   X(i,j,k) = x0 + i dx,  Y(i,j,k) = y0 + j dy,
 *   Z(i,j,k) = zs(i,j) + zeta_k (H - zs(i,j)) / zeta_{n3-1},
 * zs: terrain [n2][n1], zeta: n3 level heights (zeta_0 = 0, increasing), H:
 * flat domain top.  Returns 0, or 1 + (j n1 + i) of the first column with
 * H <= zs (no valid cell there). */
i64 orc_build_mesh(const double* zs, int n1, int n2, double x0, double y0, double dx, double dy,
                   const double* zeta, int n3, double H, double* X, double* Y, double* Z) {
    for (i64 c = 0; c < (i64)n1 * n2; c++)
        if (!(H > zs[c])) return 1 + c;
    const double T = zeta[n3 - 1];
    for (int k = 0; k < n3; k++)
        for (int j = 0; j < n2; j++)
            for (int i = 0; i < n1; i++) {
                const i64 p = nid(n1, n2, i, j, k);
                const double z = zs[(i64)j * n1 + i];
                X[p] = x0 + i * dx;
                Y[p] = y0 + j * dy;
                Z[p] = z + zeta[k] * (H - z) / T;
            }
    return 0;
}

/* Coarse (WRF-like) wind to element centres (the fire
 * grid's initial wind u0 "downscaled" from the atmospheric model's):
 * uc [3][nzc][nyc][nxc] given on the horizontal grid (xc0 + a DXc, yc0 + b DYc)
 * at heights above ground hc[0..nzc-1] (increasing).  For every element:
 * centre (xe, ye, ze) = mean of its 8 nodes, height above ground
 * he = ze - (mean of the 4 bottom nodes' Z); the value is the trilinear
 * interpolant (bilinear in x, y; linear in he between the bracketing hc),
 * with all three coordinates clamped to the coarse grid's extent. */
static void bracket(double t, int n, int* i0, double* w) {
    /* t in index units; clamp to [0, n-1]; i0 in [0, n-2], weight of i0+1 */
    if (t <= 0.0) { *i0 = 0; *w = 0.0; return; }
    if (t >= n - 1) { *i0 = n - 2; *w = 1.0; return; }
    int a = (int)floor(t);
    if (a > n - 2) a = n - 2;
    *i0 = a;
    *w = t - a;
}

int orc_interp_wind(const double* uc, int nxc, int nyc, int nzc, double xc0, double yc0,
                    double DXc, double DYc, const double* hc, const double* X, const double* Y,
                    const double* Z, int n1, int n2, int n3, double* u0) {
    if (nxc < 2 || nyc < 2 || nzc < 2) return -1;
    const int nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    const i64 ne = (i64)nx * ny * nz;
#pragma omp parallel for schedule(static)
    for (int k = 0; k < nz; k++)
        for (int j = 0; j < ny; j++)
            for (int i = 0; i < nx; i++) {
                double xe = 0, ye = 0, ze = 0, zb = 0;
                for (int c = 0; c < 2; c++)
                    for (int b = 0; b < 2; b++)
                        for (int a = 0; a < 2; a++) {
                            const i64 p = nid(n1, n2, i + a, j + b, k + c);
                            xe += X[p]; ye += Y[p]; ze += Z[p];
                        }
                for (int b = 0; b < 2; b++)
                    for (int a = 0; a < 2; a++) zb += Z[nid(n1, n2, i + a, j + b, 0)];
                xe /= 8.0; ye /= 8.0; ze /= 8.0; zb /= 4.0;
                const double he = ze - zb;
                int ia, ib, ic;
                double wa, wb, wc;
                bracket((xe - xc0) / DXc, nxc, &ia, &wa);
                bracket((ye - yc0) / DYc, nyc, &ib, &wb);
                /* vertical: find the bracketing pair of heights */
                if (he <= hc[0]) { ic = 0; wc = 0.0; }
                else if (he >= hc[nzc - 1]) { ic = nzc - 2; wc = 1.0; }
                else {
                    ic = 0;
                    while (ic < nzc - 2 && he >= hc[ic + 1]) ic++;
                    wc = (he - hc[ic]) / (hc[ic + 1] - hc[ic]);
                }
                const i64 e = ((i64)k * ny + j) * nx + i;
                for (int m = 0; m < 3; m++) {
                    double v = 0.0;
                    for (int c = 0; c < 2; c++)
                        for (int b = 0; b < 2; b++)
                            for (int a = 0; a < 2; a++) {
                                const double w = (a ? wa : 1 - wa) * (b ? wb : 1 - wb) * (c ? wc : 1 - wc);
                                v += w * uc[(((i64)m * nzc + ic + c) * nyc + ib + b) * nxc + ia + a];
                            }
                    u0[m * ne + e] = v;
                }
            }
    return 0;
}

/* ------------------------------------------------------------------ */
/* global assembly (Eq. (5) discretised)                     */
/* ------------------------------------------------------------------ */

/* K = sum_e Ke scattered into the full 27-point nodal stencil, element loop in
 * natural order.  Natural couplings to Dirichlet nodes are kept (masking,
 * C11).  Returns 0 or -1 on a non-positive Jacobian. */
int orc_assemble(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                 const double c[3], double* K) {
    i64 N = (i64)n1 * n2 * n3;
    memset(K, 0, sizeof(double) * 27 * N);
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        int J0, J1;
        own_rows(n2, &J0, &J1);   /* node rows owned by this thread */
        double xe[24], Ke[64];
        for (int k = 0; k < n3 - 1 && !bad; k++)
            for (int j = (J0 > 0 ? J0 - 1 : 0); j < n2 - 1 && j < J1; j++)
                for (int i = 0; i < n1 - 1; i++) {
                    gather_xe(X, Y, Z, n1, n2, i, j, k, xe);
                    if (orc_element_stiffness(xe, c, Ke) < 0) { bad = 1; break; }
                    for (int a = 0; a < 8; a++) {
                        const int ja = j + ((a >> 1) & 1);
                        if (ja < J0 || ja >= J1) continue;
                        i64 p = enode(n1, n2, i, j, k, a);
                        for (int b = 0; b < 8; b++) {
                            int o = o27(((b & 1) - (a & 1)), (((b >> 1) & 1) - ((a >> 1) & 1)),
                                        (((b >> 2) & 1) - ((a >> 2) & 1)));
                            K[p * 27 + o] += Ke[a * 8 + b];
                        }
                    }
                }
    }
    return bad ? -1 : 0;
}

/* One-point stiffness K1 (C12 identity only). */
int orc_assemble_onepoint(const double* X, const double* Y, const double* Z, int n1, int n2,
                          int n3, const double c[3], double* K) {
    i64 N = (i64)n1 * n2 * n3;
    memset(K, 0, sizeof(double) * 27 * N);
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        int J0, J1;
        own_rows(n2, &J0, &J1);   /* node rows owned by this thread */
        double xe[24], Ke[64];
        for (int k = 0; k < n3 - 1 && !bad; k++)
            for (int j = (J0 > 0 ? J0 - 1 : 0); j < n2 - 1 && j < J1; j++)
                for (int i = 0; i < n1 - 1; i++) {
                    gather_xe(X, Y, Z, n1, n2, i, j, k, xe);
                    if (orc_element_stiffness_onepoint(xe, c, Ke) < 0) { bad = 1; break; }
                    for (int a = 0; a < 8; a++) {
                        const int ja = j + ((a >> 1) & 1);
                        if (ja < J0 || ja >= J1) continue;
                        i64 p = enode(n1, n2, i, j, k, a);
                        for (int b = 0; b < 8; b++) {
                            int o = o27(((b & 1) - (a & 1)), (((b >> 1) & 1) - ((a >> 1) & 1)),
                                        (((b >> 2) & 1) - ((a >> 2) & 1)));
                            K[p * 27 + o] += Ke[a * 8 + b];
                        }
                    }
                }
    }
    return bad ? -1 : 0;
}

/* RHS f = sum_e fe (element loop, natural order); f_D = 0.
 * u0 layout [3][nz][ny][nx]. */
int orc_rhs(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
            const double* u0, double* f) {
    int nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    i64 N = (i64)n1 * n2 * n3, E = (i64)nx * ny * nz;
    memset(f, 0, sizeof(double) * N);
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        int J0, J1;
        own_rows(n2, &J0, &J1);   /* node rows owned by this thread */
        double xe[24], fe[8], ue[3];
        for (int k = 0; k < nz && !bad; k++)
            for (int j = (J0 > 0 ? J0 - 1 : 0); j < ny && j < J1; j++)
                for (int i = 0; i < nx; i++) {
                    i64 e = ((i64)k * ny + j) * nx + i;
                    gather_xe(X, Y, Z, n1, n2, i, j, k, xe);
                    ue[0] = u0[e];
                    ue[1] = u0[E + e];
                    ue[2] = u0[2 * E + e];
                    if (orc_element_rhs(xe, ue, fe) < 0) { bad = 1; break; }
                    for (int a = 0; a < 8; a++) {
                        const int ja = j + ((a >> 1) & 1);
                        if (ja >= J0 && ja < J1) f[enode(n1, n2, i, j, k, a)] += fe[a];
                    }
                }
    }
    if (bad) return -1;
    for (int k = 0; k < n3; k++)
        for (int j = 0; j < n2; j++)
            for (int i = 0; i < n1; i++)
                if (is_dir(n1, n2, n3, i, j, k)) f[nid(n1, n2, i, j, k)] = 0.0;
    return 0;
}

/* One-point weak divergence D1(v)_mu = sum_e 8 detJ_e(0) grad mu(0) . v_e over
 * free nodes mu (0 on D); f = -D1(u0).  (C12 identity.) */
int orc_d1(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
           const double* v, double* out) {
    int nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    i64 N = (i64)n1 * n2 * n3, E = (i64)nx * ny * nz;
    memset(out, 0, sizeof(double) * N);
    double G[24];
    const double xi[3] = {0.0, 0.0, 0.0};
    orc_shape_grad(xi, G);
#pragma omp parallel
    {
        int J0, J1;
        own_rows(n2, &J0, &J1);   /* node rows owned by this thread */
        double xe[24], B[24];
        for (int k = 0; k < nz; k++)
            for (int j = (J0 > 0 ? J0 - 1 : 0); j < ny && j < J1; j++)
                for (int i = 0; i < nx; i++) {
                    i64 e = ((i64)k * ny + j) * nx + i;
                    gather_xe(X, Y, Z, n1, n2, i, j, k, xe);
                    double det = phys_grad(xe, G, B);
                    for (int a = 0; a < 8; a++) {
                        const int ja = j + ((a >> 1) & 1);
                        if (ja < J0 || ja >= J1) continue;
                        double s = B[a * 3 + 0] * v[e] + B[a * 3 + 1] * v[E + e] + B[a * 3 + 2] * v[2 * E + e];
                        out[enode(n1, n2, i, j, k, a)] += 8.0 * det * s;
                    }
                }
    }
    for (int k = 0; k < n3; k++)
        for (int j = 0; j < n2; j++)
            for (int i = 0; i < n1; i++)
                if (is_dir(n1, n2, n3, i, j, k)) out[nid(n1, n2, i, j, k)] = 0.0;
    return 0;
}

/* Wind recovery, Eq. (3) u = u0 + A^{-1} grad lambda, with grad lambda at the
 * element centre. */
int orc_recover(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                const double c[3], const double* lam, const double* u0, double* u) {
    int nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    i64 E = (i64)nx * ny * nz;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int k = 0; k < nz; k++) {
        double xe[24], le[8], g[3];
        for (int j = 0; j < ny; j++)
            for (int i = 0; i < nx; i++) {
                i64 e = ((i64)k * ny + j) * nx + i;
                gather_xe(X, Y, Z, n1, n2, i, j, k, xe);
                for (int a = 0; a < 8; a++) le[a] = lam[enode(n1, n2, i, j, k, a)];
                if (orc_element_grad_centre(xe, le, g) < 0) bad = 1;
                for (int m = 0; m < 3; m++) u[m * E + e] = u0[m * E + e] + c[m] * g[m];
            }
    }
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------ */
/* stencil operator on a level ("K u = f")                    */
/* ------------------------------------------------------------------ */

static double row_dot(const double* K, const double* x, int n1, int n2, int n3, int i, int j,
                      int k, int skip_diag) {
    i64 p = nid(n1, n2, i, j, k);
    double s = 0.0;
    for (int dz = -1; dz <= 1; dz++) {
        int kk = k + dz;
        if (kk < 0 || kk >= n3) continue;
        for (int dy = -1; dy <= 1; dy++) {
            int jj = j + dy;
            if (jj < 0 || jj >= n2) continue;
            for (int dx = -1; dx <= 1; dx++) {
                int ii = i + dx;
                if (ii < 0 || ii >= n1) continue;
                if (skip_diag && dx == 0 && dy == 0 && dz == 0) continue;
                s += K[p * 27 + o27(dx, dy, dz)] * x[nid(n1, n2, ii, jj, kk)];
            }
        }
    }
    return s;
}

/* y = K x on free rows, y_D = 0 (x_D assumed 0). */
void orc_apply(const double* K, int n1, int n2, int n3, const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (int k = 0; k < n3; k++)
        for (int j = 0; j < n2; j++)
            for (int i = 0; i < n1; i++) {
                i64 p = nid(n1, n2, i, j, k);
                y[p] = is_dir(n1, n2, n3, i, j, k) ? 0.0 : row_dot(K, x, n1, n2, n3, i, j, k, 0);
            }
}

/* r = f - K x on free rows, r_D = 0; returns ||r||_2 (natural-order sum). */
double orc_residual(const double* K, int n1, int n2, int n3, const double* x, const double* f,
                    double* r) {
    i64 N = (i64)n1 * n2 * n3;
#pragma omp parallel for schedule(static)
    for (int k = 0; k < n3; k++)
        for (int j = 0; j < n2; j++)
            for (int i = 0; i < n1; i++) {
                i64 p = nid(n1, n2, i, j, k);
                r[p] = is_dir(n1, n2, n3, i, j, k) ? 0.0 : f[p] - row_dot(K, x, n1, n2, n3, i, j, k, 0);
            }
    double s = 0.0;
    for (i64 p = 0; p < N; p++) s += r[p] * r[p];
    return sqrt(s);
}

double orc_norm2(const double* v, i64 n) {
    double s = 0.0;
    for (i64 p = 0; p < n; p++) s += v[p] * v[p];
    return sqrt(s);
}

/* Smoother: "vertical sweeps of Gauss-Seidel from the bottom up to
 * the top, with red-black ordering horizontally into 4 groups".  Groups are
 * (i mod 2, j mod 2) = (0,0),(1,0),(0,1),(1,1) in this order (reading C7);
 * in every free column of a group, k = 0 .. n3-2 bottom-up, point update with
 * the latest values:  x_p <- (f_p - sum_{q != p} K_pq x_q) / K_pp.
 * Columns of one group are independent (stencil reach 1), so the loop over
 * them may run in parallel without changing the result. */
void orc_gs_sweep(const double* K, int n1, int n2, int n3, double* x, const double* f) {
    static const int colour[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
    for (int c = 0; c < 4; c++) {
        int ci = colour[c][0], cj = colour[c][1];
#pragma omp parallel for schedule(static)
        for (int j = 1; j < n2 - 1; j++) {
            if ((j & 1) != cj) continue;
            for (int i = 1; i < n1 - 1; i++) {
                if ((i & 1) != ci) continue;
                for (int k = 0; k < n3 - 1; k++) {
                    i64 p = nid(n1, n2, i, j, k);
                    double s = row_dot(K, x, n1, n2, n3, i, j, k, 1);
                    x[p] = (f[p] - s) / K[p * 27 + 13];
                }
            }
        }
    }
}

/* Vertical line relaxation (BASELINE north_star "vertical-
 * column line relaxation parallel over (i,j)"): the colour groups and group
 * order of the point smoother above (reading C7), but each free
 * column c of a group is solved exactly for its free unknowns k = 0..n3-2
 * given the latest values of every other column:
 *     T_c x_c = f_c - sum_{q not in column c} K_cq x_q,
 * T_c the column's own block, tridiagonal in k (couplings dz = -1, 0, +1;
 * the top neighbour is Dirichlet, x = 0).  T_c is a principal submatrix of
 * the SPD K_FF, so the Thomas algorithm (no pivoting) is stable.  Written out
 * as the textbook recurrences:
 *     c'_0 = c_0 / b_0,  d'_0 = r_0 / b_0,
 *     m_k = b_k - a_k c'_{k-1},  c'_k = c_k / m_k,  d'_k = (r_k - a_k d'_{k-1}) / m_k,
 *     x_{top} = d'_{top},  x_k = d'_k - c'_k x_{k+1}. */
void orc_line_sweep(const double* K, int n1, int n2, int n3, double* x, const double* f) {
    static const int colour[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
    const int m = n3 - 1;   /* free unknowns per column */
    for (int c = 0; c < 4; c++) {
        int ci = colour[c][0], cj = colour[c][1];
#pragma omp parallel for schedule(static)
        for (int j = 1; j < n2 - 1; j++) {
            if ((j & 1) != cj) continue;
            double* cp = (double*)malloc(sizeof(double) * (size_t)m);
            double* dp = (double*)malloc(sizeof(double) * (size_t)m);
            for (int i = 1; i < n1 - 1; i++) {
                if ((i & 1) != ci) continue;
                for (int k = 0; k < m; k++) {
                    i64 p = nid(n1, n2, i, j, k);
                    /* r_k = f_k - (off-column part of row p) */
                    double s = 0.0;
                    for (int dz = -1; dz <= 1; dz++) {
                        int kk = k + dz;
                        if (kk < 0 || kk >= n3) continue;
                        for (int dy = -1; dy <= 1; dy++)
                            for (int dx = -1; dx <= 1; dx++) {
                                if (dx == 0 && dy == 0) continue;
                                s += K[p * 27 + o27(dx, dy, dz)] * x[nid(n1, n2, i + dx, j + dy, kk)];
                            }
                    }
                    double r = f[p] - s;
                    double a = k > 0 ? K[p * 27 + o27(0, 0, -1)] : 0.0;
                    double b = K[p * 27 + o27(0, 0, 0)];
                    double cc = k < m - 1 ? K[p * 27 + o27(0, 0, 1)] : 0.0;
                    if (k == 0) {
                        cp[0] = cc / b;
                        dp[0] = r / b;
                    } else {
                        double mk = b - a * cp[k - 1];
                        cp[k] = cc / mk;
                        dp[k] = (r - a * dp[k - 1]) / mk;
                    }
                }
                x[nid(n1, n2, i, j, m - 1)] = dp[m - 1];
                for (int k = m - 2; k >= 0; k--)
                    x[nid(n1, n2, i, j, k)] = dp[k] - cp[k] * x[nid(n1, n2, i, j, k + 1)];
            }
            free(cp);
            free(dp);
        }
    }
}

/* ------------------------------------------------------------------ */
/* coarsening plan, readings C1-C5 of DESIGN.md             */
/* ------------------------------------------------------------------ */

enum { ORC_RULE_COUPLING_CUR = 0, ORC_RULE_COUPLING_PAPER = 1, ORC_RULE_VERBATIM = 2,
       ORC_RULE_FULL = 3 };

/* Ratio of the paper's tests "h3/(h1 a3) > 1/3" and "< 3", with
 * a1 = a2 normalised to 1 by dividing a3 by ah = sqrt(a1 a2) (C2).
 * VERBATIM: rho = h3 / (h1 a3')    (the formula as printed)
 * COUPLING: rho = (h3/h1) a3'      (the same test expressed through the
 *           coupling strength of Eq. (4), whose vertical coefficient is
 *           a3^-2 -- reading C1). */
static double plan_rho(double h3, double h1, double a3n, int rule) {
    if (rule == ORC_RULE_VERBATIM) return h3 / (h1 * a3n);
    return (h3 / h1) * a3n;
}

/* One planning step.  Inputs: horizontal spacing h1 of the level, layer
 * thicknesses h3[0..nz-1], node counts n1, n2.  Outputs: *hflag (coarsen i
 * and j by 2), kept[] node-layer indices (kept[0] = 0, last = nz), *nkept,
 * and the next level's h1/h3.  Returns 1 if anything coarsens, else 0.
 *   horizontal: rho(h3[0], h1) > 1/3, needs n1, n2 >= 4
 *   vertical:   from the ground up, from kept layer k: if k+1 < nz and
 *               rho(h3[k], h1v) < 3 then drop node layer k+1
 *   h1v = h1' (= 2 h1 when coarsened horizontally) for COUPLING_PAPER and
 *   VERBATIM ("replace h1 and h2 by their new values"), and the current h1
 *   for COUPLING_CUR (reading C1b).  FULL: always coarsen both. */
int orc_plan_level(double h1, const double* h3, int nz, double a1, double a2, double a3,
                   int rule, int n1, int n2, int* hflag, int* kept, int* nkept,
                   double* h1_new, double* h3_new) {
    double a3n = a3 / sqrt(a1 * a2);
    int hz;
    if (rule == ORC_RULE_FULL) hz = 1;
    else hz = plan_rho(h3[0], h1, a3n, rule) > 1.0 / 3.0;
    if (n1 < 4 || n2 < 4) hz = 0;
    double h1p = hz ? 2.0 * h1 : h1;
    double h1v = (rule == ORC_RULE_COUPLING_CUR) ? h1 : h1p;
    int nk = 0, k = 0;
    kept[nk++] = 0;
    while (k < nz) {
        int merge;
        if (rule == ORC_RULE_FULL) merge = (k + 1 < nz);
        else merge = (k + 1 < nz) && (plan_rho(h3[k], h1v, a3n, rule) < 3.0);
        k = merge ? k + 2 : k + 1;
        kept[nk++] = k;
    }
    *nkept = nk;
    for (int t = 0; t + 1 < nk; t++) {
        double s = 0.0;
        for (int kk = kept[t]; kk < kept[t + 1]; kk++) s += h3[kk];
        h3_new[t] = s;
    }
    *hflag = hz;
    *h1_new = h1p;
    return hz || (nk - 1 < nz);
}

/* 1-D maps of the index-space trilinear prolongation (C4, C5):
 * coarse node c sits at fine index pos[c]; fine index t has the lower parent
 * lo[t] (pos[lo] <= t) and co[t] = 1 if coincident (weight 1), else weights
 * 1/2, 1/2 on lo[t] and lo[t]+1. */
static int horiz_kept(int n, int* pos) {
    int m = 0;
    for (int t = 0; t < n; t += 2) pos[m++] = t;
    if (pos[m - 1] != n - 1) pos[m++] = n - 1;
    return m;
}

static void build_map1d(int n, const int* pos, int m, int* lo, int* co) {
    int c = 0;
    for (int t = 0; t < n; t++) {
        while (c + 1 < m && pos[c + 1] <= t) c++;
        lo[t] = c;
        co[t] = (pos[c] == t);
    }
}

typedef struct {
    int n1, n2, n3;
    double* K;           /* 27 * N */
    double *x, *f, *r;   /* level vectors */
    /* transition to the next level */
    int hflag;
    int nkept;
    int kept[ORC_MAXNZ];
    int *lo[3], *co[3];  /* fine-index maps per direction (size n_d) */
    int smoother;        /* -1: the hierarchy's smoother; else 0 point GS, 1 line relaxation */
} orc_level;

typedef struct {
    int nlev;
    orc_level L[ORC_MAXLEV];
    int pre, post;
    int rule;
    int cmax;
    int coarse_direct;    /* 1: dense Cholesky; 0: fallback GS sweeps (C8) */
    int coarse_iters;
    int smoother;         /* 0: point GS, 1: vertical line relaxation (f1) */
    int nf;               /* free unknowns on the coarsest level */
    i64* fidx;            /* free node index list (natural order) */
    double* chol;         /* nf x nf lower factor */
    double h1;
    double h3[ORC_MAXNZ];
} orc_mg;

static i64 level_N(const orc_level* l) { return (i64)l->n1 * l->n2 * l->n3; }
static i64 level_free(int n1, int n2, int n3) { return (i64)(n1 - 2) * (n2 - 2) * (n3 - 1); }

/* one sweep of the hierarchy's smoother on level l */
static void mg_smooth(const orc_mg* mg, const orc_level* l, double* x, const double* f) {
    const int sm = l->smoother >= 0 ? l->smoother : mg->smoother;
    if (sm == 1) orc_line_sweep(l->K, l->n1, l->n2, l->n3, x, f);
    else orc_gs_sweep(l->K, l->n1, l->n2, l->n3, x, f);
}

/* select the smoother (0 point GS, 1 vertical line relaxation) */
void orc_mg_set_smoother(orc_mg* mg, int smoother) { mg->smoother = smoother; }
/* per-level override (SURVEY 8(f) f1 "per-level decisions"); -1 = the global choice */
void orc_mg_set_level_smoother(orc_mg* mg, int l, int smoother) {
    if (l >= 0 && l < mg->nlev) mg->L[l].smoother = smoother;
}

/* parents of fine index t along direction d of level l: returns count (1|2) */
static inline int parents(const orc_level* l, int d, int t, int* pc, double* pw) {
    int c = l->lo[d][t];
    if (l->co[d][t]) { pc[0] = c; pw[0] = 1.0; return 1; }
    pc[0] = c; pw[0] = 0.5; pc[1] = c + 1; pw[1] = 0.5;
    return 2;
}

/* Galerkin coarse operator, Eq. (7) "K_c = P^T K P", restricted to
 * coarse free rows (C11).  Scatter over fine free p and its 27 neighbours q:
 *   Kc[P][Q-P] += w_P(p) K_pq w_Q(q). */
static int galerkin(const orc_level* f, orc_level* c) {
    int n1 = f->n1, n2 = f->n2, n3 = f->n3;
    int m1 = c->n1, m2 = c->n2, m3 = c->n3;
    memset(c->K, 0, sizeof(double) * 27 * level_N(c));
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
    int C0, C1;
    own_rows(m2, &C0, &C1);   /* coarse rows owned by this thread */
    for (int k = 0; k < n3 - 1 && !bad; k++)
        for (int j = 1; j < n2 - 1 && !bad; j++) {
            {   /* skip fine rows with no parent row owned here */
                int pj[2];
                double wj[2];
                int np = parents(f, 1, j, pj, wj), any = 0;
                for (int t = 0; t < np; t++) any |= pj[t] >= C0 && pj[t] < C1;
                if (!any) continue;
            }
            for (int i = 1; i < n1 - 1 && !bad; i++) {
                i64 p = nid(n1, n2, i, j, k);
                int pci[2], pcj[2], pck[2];
                double pwi[2], pwj[2], pwk[2];
                int npi = parents(f, 0, i, pci, pwi);
                int npj = parents(f, 1, j, pcj, pwj);
                int npk = parents(f, 2, k, pck, pwk);
                for (int dz = -1; dz <= 1; dz++)
                    for (int dy = -1; dy <= 1; dy++)
                        for (int dx = -1; dx <= 1; dx++) {
                            int qi = i + dx, qj = j + dy, qk = k + dz;
                            if (qk < 0 || qk >= n3) continue;
                            double kpq = f->K[p * 27 + o27(dx, dy, dz)];
                            int qci[2], qcj[2], qck[2];
                            double qwi[2], qwj[2], qwk[2];
                            int nqi = parents(f, 0, qi, qci, qwi);
                            int nqj = parents(f, 1, qj, qcj, qwj);
                            int nqk = parents(f, 2, qk, qck, qwk);
                            for (int a3 = 0; a3 < npk; a3++)
                                for (int a2 = 0; a2 < npj; a2++)
                                    for (int a1 = 0; a1 < npi; a1++) {
                                        int Pi = pci[a1], Pj = pcj[a2], Pk = pck[a3];
                                        if (Pj < C0 || Pj >= C1) continue;
                                        if (is_dir(m1, m2, m3, Pi, Pj, Pk)) continue;
                                        double wP = pwi[a1] * pwj[a2] * pwk[a3];
                                        i64 P = nid(m1, m2, Pi, Pj, Pk);
                                        for (int b3 = 0; b3 < nqk; b3++)
                                            for (int b2 = 0; b2 < nqj; b2++)
                                                for (int b1 = 0; b1 < nqi; b1++) {
                                                    int ex = qci[b1] - Pi, ey = qcj[b2] - Pj, ez = qck[b3] - Pk;
                                                    if (ex < -1 || ex > 1 || ey < -1 || ey > 1 || ez < -1 || ez > 1) {
                                                        bad = 1;
                                                        continue;
                                                    }
                                                    double wQ = qwi[b1] * qwj[b2] * qwk[b3];
                                                    c->K[P * 27 + o27(ex, ey, ez)] += wP * kpq * wQ;
                                                }
                                    }
                        }
            }
        }
    }
    return bad ? -1 : 0;
}

/* f_c = P^T r (Eq. (7) "f_c = P^T (f - K u)"), scatter over fine free p into
 * coarse free P; coarse D entries stay 0. */
static void restrict_(const orc_level* f, const orc_level* c, const double* r, double* fc) {
    int n1 = f->n1, n2 = f->n2, n3 = f->n3;
    memset(fc, 0, sizeof(double) * level_N(c));
#pragma omp parallel
    {
    int C0, C1;
    own_rows(c->n2, &C0, &C1);   /* coarse rows owned by this thread */
    for (int k = 0; k < n3 - 1; k++)
        for (int j = 1; j < n2 - 1; j++) {
            {   /* skip fine rows with no parent row owned here */
                int pj[2];
                double wj[2];
                int np = parents(f, 1, j, pj, wj), any = 0;
                for (int t = 0; t < np; t++) any |= pj[t] >= C0 && pj[t] < C1;
                if (!any) continue;
            }
            for (int i = 1; i < n1 - 1; i++) {
                double rp = r[nid(n1, n2, i, j, k)];
                int pci[2], pcj[2], pck[2];
                double pwi[2], pwj[2], pwk[2];
                int npi = parents(f, 0, i, pci, pwi);
                int npj = parents(f, 1, j, pcj, pwj);
                int npk = parents(f, 2, k, pck, pwk);
                for (int a3 = 0; a3 < npk; a3++)
                    for (int a2 = 0; a2 < npj; a2++)
                        for (int a1 = 0; a1 < npi; a1++) {
                            if (pcj[a2] < C0 || pcj[a2] >= C1) continue;
                            if (is_dir(c->n1, c->n2, c->n3, pci[a1], pcj[a2], pck[a3])) continue;
                            fc[nid(c->n1, c->n2, pci[a1], pcj[a2], pck[a3])] +=
                                pwi[a1] * pwj[a2] * pwk[a3] * rp;
                        }
            }
        }
    }
}

/* x += P x_c (Eq. (7) "u <- u + P u_c") on fine free nodes; x_c,D = 0. */
static void prolong_(const orc_level* f, const orc_level* c, const double* xc, double* x) {
    int n1 = f->n1, n2 = f->n2, n3 = f->n3;
#pragma omp parallel for schedule(static)
    for (int k = 0; k < n3 - 1; k++)
        for (int j = 1; j < n2 - 1; j++)
            for (int i = 1; i < n1 - 1; i++) {
                int pci[2], pcj[2], pck[2];
                double pwi[2], pwj[2], pwk[2];
                int npi = parents(f, 0, i, pci, pwi);
                int npj = parents(f, 1, j, pcj, pwj);
                int npk = parents(f, 2, k, pck, pwk);
                double s = 0.0;
                for (int a3 = 0; a3 < npk; a3++)
                    for (int a2 = 0; a2 < npj; a2++)
                        for (int a1 = 0; a1 < npi; a1++)
                            s += pwi[a1] * pwj[a2] * pwk[a3] *
                                 xc[nid(c->n1, c->n2, pci[a1], pcj[a2], pck[a3])];
                x[nid(n1, n2, i, j, k)] += s;
            }
}

/* Coarsest-level direct solve ("solved by a direct method"): dense
 * Cholesky K_FF = L L^T of the free block (natural order of free nodes),
 * built from the lower triangle of the stencil matrix. */
static int coarse_factor(orc_mg* mg) {
    orc_level* l = &mg->L[mg->nlev - 1];
    int n1 = l->n1, n2 = l->n2, n3 = l->n3;
    i64 nf = level_free(n1, n2, n3);
    mg->nf = (int)nf;
    mg->fidx = (i64*)malloc(sizeof(i64) * (nf > 0 ? nf : 1));
    i64* rowof = (i64*)malloc(sizeof(i64) * level_N(l));
    i64 t = 0;
    for (i64 p = 0; p < level_N(l); p++) rowof[p] = -1;
    for (int k = 0; k < n3 - 1; k++)
        for (int j = 1; j < n2 - 1; j++)
            for (int i = 1; i < n1 - 1; i++) {
                i64 p = nid(n1, n2, i, j, k);
                rowof[p] = t;
                mg->fidx[t++] = p;
            }
    double* A = (double*)calloc((size_t)(nf > 0 ? nf * nf : 1), sizeof(double));
    for (i64 r = 0; r < nf; r++) {
        i64 p = mg->fidx[r];
        int k = (int)(p / ((i64)n1 * n2)), j = (int)((p / n1) % n2), i = (int)(p % n1);
        for (int dz = -1; dz <= 1; dz++)
            for (int dy = -1; dy <= 1; dy++)
                for (int dx = -1; dx <= 1; dx++) {
                    int ii = i + dx, jj = j + dy, kk = k + dz;
                    if (kk < 0 || kk >= n3 || is_dir(n1, n2, n3, ii, jj, kk)) continue;
                    i64 q = rowof[nid(n1, n2, ii, jj, kk)];
                    A[r * nf + q] = l->K[p * 27 + o27(dx, dy, dz)];
                }
    }
    free(rowof);
    /* Cholesky (lower), column by column */
    for (i64 jc = 0; jc < nf; jc++) {
        double s = A[jc * nf + jc];
        for (i64 kc = 0; kc < jc; kc++) s -= A[jc * nf + kc] * A[jc * nf + kc];
        if (!(s > 0.0)) { free(A); return -1; }
        double d = sqrt(s);
        A[jc * nf + jc] = d;
        for (i64 ic = jc + 1; ic < nf; ic++) {
            double v = A[ic * nf + jc];
            for (i64 kc = 0; kc < jc; kc++) v -= A[ic * nf + kc] * A[jc * nf + kc];
            A[ic * nf + jc] = v / d;
        }
    }
    mg->chol = A;
    return 0;
}

static void coarse_solve(const orc_mg* mg, const double* f, double* x) {
    i64 nf = mg->nf;
    const double* A = mg->chol;
    double* y = (double*)malloc(sizeof(double) * (nf > 0 ? nf : 1));
    for (i64 r = 0; r < nf; r++) {
        double s = f[mg->fidx[r]];
        for (i64 c = 0; c < r; c++) s -= A[r * nf + c] * y[c];
        y[r] = s / A[r * nf + r];
    }
    for (i64 r = nf - 1; r >= 0; r--) {
        double s = y[r];
        for (i64 c = r + 1; c < nf; c++) s -= A[c * nf + r] * y[c];
        y[r] = s / A[r * nf + r];
    }
    for (i64 r = 0; r < nf; r++) x[mg->fidx[r]] = y[r];
    free(y);
}

static void alloc_level(orc_level* l, int n1, int n2, int n3) {
    l->n1 = n1; l->n2 = n2; l->n3 = n3;
    i64 N = level_N(l);
    l->K = (double*)calloc((size_t)(27 * N), sizeof(double));
    l->x = (double*)calloc((size_t)N, sizeof(double));
    l->f = (double*)calloc((size_t)N, sizeof(double));
    l->r = (double*)calloc((size_t)N, sizeof(double));
    for (int d = 0; d < 3; d++) { l->lo[d] = NULL; l->co[d] = NULL; }
    l->smoother = -1;
}

void orc_mg_free(orc_mg* mg) {
    if (!mg) return;
    for (int l = 0; l < mg->nlev; l++) {
        free(mg->L[l].K); free(mg->L[l].x); free(mg->L[l].f); free(mg->L[l].r);
        for (int d = 0; d < 3; d++) { free(mg->L[l].lo[d]); free(mg->L[l].co[d]); }
    }
    free(mg->fidx);
    free(mg->chol);
    free(mg);
}

/* Planner inputs (C2): h1 = sqrt(dx dy) at the grid origin; h3[k] = layer
 * thicknesses at the column (i*,j*) of minimum Z(i,j,0), ties -> smallest
 * linear index. */
void orc_planner_inputs(const double* X, const double* Y, const double* Z, int n1, int n2,
                        int n3, double* h1, double* h3) {
    double dx = X[nid(n1, n2, 1, 0, 0)] - X[0];
    double dy = Y[nid(n1, n2, 0, 1, 0)] - Y[0];
    *h1 = sqrt(dx * dy);
    i64 best = 0;
    for (i64 p = 1; p < (i64)n1 * n2; p++)
        if (Z[p] < Z[best]) best = p;
    int i = (int)(best % n1), j = (int)(best / n1);
    for (int k = 0; k < n3 - 1; k++) h3[k] = Z[nid(n1, n2, i, j, k + 1)] - Z[nid(n1, n2, i, j, k)];
}

/* Build the hierarchy: level-0 assembly, repeated planning + Galerkin until
 * the free count is <= cmax or nothing coarsens,
 * coarsest dense factorisation (or the GS fallback, C8).
 * *err: 0 ok, 1 mesh (non-positive Jacobian), 2 Galerkin reach > 1,
 *       3 Cholesky failure, 4 bad arguments. */
orc_mg* orc_mg_setup(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                     double a1, double a2, double a3, int rule, int cmax, int pre, int post,
                     int* err) {
    *err = 0;
    if (n1 < 3 || n2 < 3 || n3 < 2 || n3 - 1 > ORC_MAXNZ - 1) { *err = 4; return NULL; }
    orc_mg* mg = (orc_mg*)calloc(1, sizeof(orc_mg));
    mg->pre = pre; mg->post = post; mg->rule = rule; mg->cmax = cmax;
    mg->coarse_iters = 50;
    mg->smoother = 0;
    double c[3] = {1.0 / (a1 * a1), 1.0 / (a2 * a2), 1.0 / (a3 * a3)};
    alloc_level(&mg->L[0], n1, n2, n3);
    mg->nlev = 1;
    if (orc_assemble(X, Y, Z, n1, n2, n3, c, mg->L[0].K) < 0) { *err = 1; orc_mg_free(mg); return NULL; }
    double h1, h3[ORC_MAXNZ];
    orc_planner_inputs(X, Y, Z, n1, n2, n3, &h1, h3);
    mg->h1 = h1;
    memcpy(mg->h3, h3, sizeof(double) * (n3 - 1));
    while (mg->nlev < ORC_MAXLEV) {
        orc_level* f = &mg->L[mg->nlev - 1];
        if (level_free(f->n1, f->n2, f->n3) <= cmax) break;
        int hflag, nk;
        double h1n, h3n[ORC_MAXNZ];
        if (!orc_plan_level(h1, h3, f->n3 - 1, a1, a2, a3, rule, f->n1, f->n2, &hflag, f->kept,
                            &nk, &h1n, h3n))
            break;
        f->hflag = hflag;
        f->nkept = nk;
        int m1, m2;
        static int posbuf[2][1 << 16];
        for (int d = 0; d < 3; d++) {
            int n = d == 0 ? f->n1 : (d == 1 ? f->n2 : f->n3);
            f->lo[d] = (int*)malloc(sizeof(int) * n);
            f->co[d] = (int*)malloc(sizeof(int) * n);
        }
        if (hflag) {
            m1 = horiz_kept(f->n1, posbuf[0]);
            m2 = horiz_kept(f->n2, posbuf[1]);
        } else {
            m1 = f->n1; m2 = f->n2;
            for (int t = 0; t < m1; t++) posbuf[0][t] = t;
            for (int t = 0; t < m2; t++) posbuf[1][t] = t;
        }
        build_map1d(f->n1, posbuf[0], m1, f->lo[0], f->co[0]);
        build_map1d(f->n2, posbuf[1], m2, f->lo[1], f->co[1]);
        build_map1d(f->n3, f->kept, nk, f->lo[2], f->co[2]);
        orc_level* cl = &mg->L[mg->nlev];
        alloc_level(cl, m1, m2, nk);
        mg->nlev++;
        if (galerkin(f, cl) < 0) { *err = 2; orc_mg_free(mg); return NULL; }
        h1 = h1n;
        memcpy(h3, h3n, sizeof(double) * (nk - 1));
    }
    orc_level* lc = &mg->L[mg->nlev - 1];
    if (level_free(lc->n1, lc->n2, lc->n3) <= cmax) {
        mg->coarse_direct = 1;
        if (coarse_factor(mg) < 0) { *err = 3; orc_mg_free(mg); return NULL; }
    } else {
        mg->coarse_direct = 0;
        mg->nf = (int)level_free(lc->n1, lc->n2, lc->n3);
    }
    return mg;
}

int orc_mg_nlevels(const orc_mg* mg) { return mg->nlev; }
int orc_mg_coarse_direct(const orc_mg* mg) { return mg->coarse_direct; }
void orc_mg_level_dims(const orc_mg* mg, int l, int dims[3]) {
    dims[0] = mg->L[l].n1; dims[1] = mg->L[l].n2; dims[2] = mg->L[l].n3;
}
double* orc_mg_K(orc_mg* mg, int l) { return mg->L[l].K; }
int orc_mg_plan(const orc_mg* mg, int l, int* hflag, int* kept) {
    *hflag = mg->L[l].hflag;
    for (int t = 0; t < mg->L[l].nkept; t++) kept[t] = mg->L[l].kept[t];
    return mg->L[l].nkept;
}
void orc_mg_gs(orc_mg* mg, int l, double* x, const double* f) {
    mg_smooth(mg, &mg->L[l], x, f);
}
void orc_mg_apply(orc_mg* mg, int l, const double* x, double* y) {
    orc_apply(mg->L[l].K, mg->L[l].n1, mg->L[l].n2, mg->L[l].n3, x, y);
}
void orc_mg_restrict(orc_mg* mg, int l, const double* r, double* fc) {
    restrict_(&mg->L[l], &mg->L[l + 1], r, fc);
}
void orc_mg_prolong(orc_mg* mg, int l, const double* xc, double* x) {
    prolong_(&mg->L[l], &mg->L[l + 1], xc, x);
}
void orc_mg_coarse_solve(orc_mg* mg, const double* f, double* x) {
    orc_level* l = &mg->L[mg->nlev - 1];
    if (mg->coarse_direct) {
        memset(x, 0, sizeof(double) * level_N(l));
        coarse_solve(mg, f, x);
    } else {
        memset(x, 0, sizeof(double) * level_N(l));
        for (int s = 0; s < mg->coarse_iters; s++) mg_smooth(mg, l, x, f);
    }
}

/* V-cycle, P:128-149 and Eq. (7): pre-smoothing; f_c = P^T(f - K x);
 * solve the coarse problem recursively from x_c = 0 (or directly at the
 * coarsest); x += P x_c; post-smoothing. */
static void vcycle_rec(orc_mg* mg, int l, double* x, const double* f) {
    orc_level* L = &mg->L[l];
    if (l == mg->nlev - 1) { orc_mg_coarse_solve(mg, f, x); return; }
    for (int s = 0; s < mg->pre; s++) mg_smooth(mg, L, x, f);
    orc_residual(L->K, L->n1, L->n2, L->n3, x, f, L->r);
    orc_level* C = &mg->L[l + 1];
    restrict_(L, C, L->r, C->f);
    memset(C->x, 0, sizeof(double) * level_N(C));
    vcycle_rec(mg, l + 1, C->x, C->f);
    prolong_(L, C, C->x, x);
    for (int s = 0; s < mg->post; s++) mg_smooth(mg, L, x, f);
}

void orc_mg_vcycle(orc_mg* mg, double* x, const double* f) { vcycle_rec(mg, 0, x, f); }

/* Solve loop (S:354 interface; reading C9/C10): from lambda0 (D entries
 * zeroed) or 0; rel = ||f - K x||_2 / ||f||_2 over F (abs if ||f|| = 0);
 * stop at rel <= tol, max_cycles, divergence (rel_c > 10 rel_{c-3}) or a
 * non-finite residual.  Returns 0 converged, 1 not converged, 2 diverged,
 * 3 non-finite.  hist[c] = rel after cycle c (hist[0] = initial). */
int orc_mg_solve(orc_mg* mg, const double* f, const double* lam0, double tol, int max_cycles,
                 double* x, double* hist, int* cycles, double* rate) {
    orc_level* L = &mg->L[0];
    int n1 = L->n1, n2 = L->n2, n3 = L->n3;
    i64 N = level_N(L);
    for (int k = 0; k < n3; k++)
        for (int j = 0; j < n2; j++)
            for (int i = 0; i < n1; i++) {
                i64 p = nid(n1, n2, i, j, k);
                x[p] = (lam0 && !is_dir(n1, n2, n3, i, j, k)) ? lam0[p] : 0.0;
            }
    double fn = orc_norm2(f, N);
    *cycles = 0;
    *rate = 0.0;
    if (fn == 0.0) {
        memset(x, 0, sizeof(double) * N);
        hist[0] = 0.0;
        return 0;
    }
    double rel = orc_residual(L->K, n1, n2, n3, x, f, L->r) / fn;
    hist[0] = rel;
    int status = 1;
    if (rel <= tol) status = 0;
    int c = 0;
    while (status == 1 && c < max_cycles) {
        orc_mg_vcycle(mg, x, f);
        c++;
        rel = orc_residual(L->K, n1, n2, n3, x, f, L->r) / fn;
        hist[c] = rel;
        if (!isfinite(rel)) { status = 3; break; }
        if (rel <= tol) { status = 0; break; }
        if (c >= 3 && rel > 10.0 * hist[c - 3]) { status = 2; break; }
    }
    *cycles = c;
    if (c >= 2) *rate = pow(hist[c] / hist[1], 1.0 / (c - 1));
    else if (c == 1) *rate = hist[1] / hist[0];
    return status;
}

/* Standalone Galerkin on a given plan (for tests): Kf full 27-storage on
 * (n1,n2,n3); hflag/kept as orc_plan_level; Kc sized for the coarse dims. */
int orc_galerkin_plan(const double* Kf, int n1, int n2, int n3, int hflag, const int* kept,
                      int nkept, double* Kc, int cdims[3]) {
    orc_level f, c;
    memset(&f, 0, sizeof f);
    memset(&c, 0, sizeof c);
    f.n1 = n1; f.n2 = n2; f.n3 = n3;
    f.K = (double*)Kf;
    static int posbuf[2][1 << 16];
    int m1, m2;
    if (hflag) { m1 = horiz_kept(n1, posbuf[0]); m2 = horiz_kept(n2, posbuf[1]); }
    else {
        m1 = n1; m2 = n2;
        for (int t = 0; t < m1; t++) posbuf[0][t] = t;
        for (int t = 0; t < m2; t++) posbuf[1][t] = t;
    }
    for (int d = 0; d < 3; d++) {
        int n = d == 0 ? n1 : (d == 1 ? n2 : n3);
        f.lo[d] = (int*)malloc(sizeof(int) * n);
        f.co[d] = (int*)malloc(sizeof(int) * n);
    }
    build_map1d(n1, posbuf[0], m1, f.lo[0], f.co[0]);
    build_map1d(n2, posbuf[1], m2, f.lo[1], f.co[1]);
    build_map1d(n3, kept, nkept, f.lo[2], f.co[2]);
    cdims[0] = m1; cdims[1] = m2; cdims[2] = nkept;
    int rc = 0;
    if (Kc) {
        c.n1 = m1; c.n2 = m2; c.n3 = nkept;
        c.K = Kc;
        rc = galerkin(&f, &c);
    }
    for (int d = 0; d < 3; d++) { free(f.lo[d]); free(f.co[d]); }
    return rc;
}
