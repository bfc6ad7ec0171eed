// wd_internal.cuh -- shared definitions of the sm_100a kernels and the C ABI.
//
// Internal data layout in HBM ("i-split" layout):
//   node (i,j,k) of a level lives at  off = k*plane + j*P + (i&1)*H + (i>>1)
//   H = half-row pitch (ceil(n1/2) rounded up to 16 doubles = 128 B),
//   P = 2H, plane = n2*P.  Within a row, even-i nodes come first and odd-i
//   nodes second, so every colour phase of the 4-colour smoother
//   ((i mod 2, j mod 2)) reads and writes stride-1 half rows.
// Operator storage: 14 symmetric coefficients per node, SoA planes of NT
// doubles each (coef[s*NT + off]):  s = 0 diagonal; s = 1..13 the "forward"
// couplings K(p, p+d_s),  d_s in {(1,0,0), (-1,1,0), (0,1,0), (1,1,0),
// (dx,dy,1) for dy, dx in -1..1}.  The backward coupling K(p, p-d_s) is read
// from the node p-d_s, so the stored operator is symmetric by construction.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace wd {

// kernels launched by this library (defined in wd_api.cu); launchers add the
// number of kernels they enqueue
extern std::atomic<long long> g_launches;
// development knob: thread mapping of apply_kernel (env WD_APPLY_VARIANT)
extern int g_apply_variant;
extern int g_tma_debug;
// race stress tests (env WD_TEST_JITTER: max ns of a random per-warp sleep per
// pipeline step in the fused sweep and the TMA residual; WD_TEST_GS_GRID: cap
// on their persistent CTA count); 0 = off
extern int g_test_jitter, g_test_gs_grid;
extern int g_fuse_prolong;   // env WD_FUSE_PROLONG=1: fold the prolongation into the sweep
extern int g_galerkin_generic;   // env WD_GALERKIN_GENERIC=1: disable the unrolled path (tests)

typedef long long i64;

// Row-outer layout [j][k][half][pos]: one node row of all levels (n3 * P
// doubles) is contiguous, so a slab halo row is a single block to copy/send.
//
// Slab decomposition: a level may hold only the node rows
// [jg0, jg0 + n2) of a grid with n2g rows (its own rows plus halo rows).
// Kernels update only the owned local rows [own0, own1); the Dirichlet set is
// decided on global rows (jg = j + jg0 in {0, n2g - 1}).  Without
// decomposition jg0 = 0, n2g = n2, own0 = 0, own1 = n2.
struct LevDev {
    int n1, n2, n3;
    int H, P;      // half-row pitch, row pitch (2H)
    i64 sk, sj;    // strides of k (= P) and of j (= n3 P)
    i64 NT;        // entries per array (= n2 sj)
    int jg0, n2g;  // global row of local row 0, global row count
    int own0, own1;  // owned local rows
};

// node row j (local) is owned and not a lateral Dirichlet row
__host__ __device__ __forceinline__ bool row_free(const LevDev& L, int j) {
    const int g = j + L.jg0;
    return j >= L.own0 && j < L.own1 && g >= 1 && g <= L.n2g - 2;
}
__host__ __device__ __forceinline__ bool row_dirichlet(const LevDev& L, int j) {
    const int g = j + L.jg0;
    return g == 0 || g == L.n2g - 1;
}

// a natural-layout array of the ABI: node (i, j_loc, k) at
// (k * n2a + j_loc + jofs) * n1 + i   (element arrays: rows n2a, columns n1).
struct Nat {
    const double* p;
    int n2a, jofs;
};

__host__ __device__ __forceinline__ i64 loff(const LevDev& L, int i, int j, int k) {
    return (i64)j * L.sj + (i64)k * L.sk + (i64)((i & 1) * L.H + (i >> 1));
}

// forward offsets of the 14 slots (slot 0 = diagonal)
__host__ __device__ __forceinline__ int slot_dx(int s) {
    return s == 0 ? 0 : s == 1 ? 1 : s <= 4 ? (s - 3) : ((s - 5) % 3) - 1;
}
__host__ __device__ __forceinline__ int slot_dy(int s) {
    return s <= 1 ? 0 : s <= 4 ? 1 : ((s - 5) / 3) - 1;
}
__host__ __device__ __forceinline__ int slot_dz(int s) { return s <= 4 ? 0 : 1; }

// slot of offset (dx,dy,dz); returns +s for forward/zero offsets, -s for backward
__host__ __device__ __forceinline__ int slot_of(int dx, int dy, int dz) {
    if (dz == 1) return 5 + (dx + 1) + 3 * (dy + 1);
    if (dz == -1) return -(5 + (-dx + 1) + 3 * (-dy + 1));
    if (dy == 1) return 3 + dx;
    if (dy == -1) return -(3 - dx);
    if (dx == 1) return 1;
    if (dx == -1) return -1;
    return 0;
}

// ----------------------------------------------------------------- launchers
// (all stream-ordered on `st`; defined in the .cu files)

// k_fe.cu: finite elements
// tile rows [ty0, ty1) of the assembly grid (ty1 < 0: all); assemble_rows_needed(t):
// node rows [0, .) the tile rows < t+1 read (for chunked host copies)
void launch_assemble(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                     const double c[3], const LevDev& L, double* coef,
                     unsigned long long* bad, cudaStream_t st, int ty0 = 0, int ty1 = -1);
int assemble_tile_rows(int n2);
int assemble_rows_needed(int t);
void launch_rhs(const double* X, const double* Y, const double* Z, const LevDev& L, Nat u0, Nat f,
                cudaStream_t st);
void launch_recover(const double* X, const double* Y, const double* Z, const LevDev& L,
                    const double c[3], Nat lam, Nat u0, Nat u, cudaStream_t st);

// k_mg.cu: multigrid on the stencil
void launch_nat2int(const LevDev& L, Nat src, double* dst, bool zero_dirichlet, cudaStream_t st);
void launch_int2nat(const LevDev& L, const double* src, Nat dst, cudaStream_t st);
void launch_gs_sweep(const LevDev& L, const double* coef, double* lam, const double* f,
                     cudaStream_t st);
void launch_gs_phase(const LevDev& L, const double* coef, double* lam, const double* f, int c,
                     cudaStream_t st);
// colour phase c of vertical line relaxation; cpb/dpb: two
// level-sized scratch arrays for the Thomas recurrences
void launch_line_phase(const LevDev& L, const double* coef, double* lam, const double* f,
                       double* cpb, double* dpb, int c, cudaStream_t st);
void launch_sum_ordered(const double* v, int n, double* out, cudaStream_t st);
// y = K x (f == NULL) or y = f - K x; optional block partials of sum y^2;
// variant < 0: the process default (env WD_APPLY_VARIANT); 4: one plane per
// CTA layer (small levels)
int launch_apply(const LevDev& L, const double* coef, const double* x, const double* f,
                 double* y, double* partial, cudaStream_t st, int variant = -1);
constexpr long long APPLY_SMALL_COLS = 100LL * 100LL;   // measured crossover ~100^2 (189^2: 14.5 -> 20.1 us)
void launch_reduce_sum(const double* partial, int n, double* out, cudaStream_t st);
void launch_norm2_partial(const LevDev& L, const double* v, double* partial, int* nblk,
                          cudaStream_t st);
struct MapDev {
    // per direction d: lo[d][t], co[d][t] over fine indices; pos[d][c] over coarse
    const int* lo[3];
    const int* co[3];
    const int* pos[3];
};
// zident: the z map of the transition is the identity (fast paths, bitwise equal)
void launch_restrict(const LevDev& F, const LevDev& Cl, const MapDev& M, const double* r,
                     double* fc, int zident, cudaStream_t st);
// x += w P xc; w = 1 is Eq. (7) (w != 1 only for the divergence-guard test)
void launch_prolong(const LevDev& F, const LevDev& Cl, const MapDev& M, const double* xc,
                    double* x, int zident, cudaStream_t st, double w = 1.0);
// zident: the z map of this transition is the identity (no layer merged);
// regular interior columns then take an unrolled path (bitwise equal)
// zeros at the coefficient entries neither the assembly nor (galerkin) the
// Galerkin product writes: half-row padding, and Dirichlet nodes when galerkin
void launch_zero_unwritten(const LevDev& L, double* coef, bool galerkin, cudaStream_t st);
void launch_galerkin(const LevDev& F, const LevDev& Cl, const MapDev& M, const double* coefF,
                     double* coefC, int zident, cudaStream_t st);
void launch_export27(const LevDev& L, const double* coef, double* K27, cudaStream_t st);
void launch_zero_dirichlet(const LevDev& L, double* v, cudaStream_t st);
void launch_argmin_bottom(const double* Z, int n, double* pval, long long* pidx, int nblk,
                          cudaStream_t st);

// k_gs_fused.cu: one whole 4-colour sweep per launch, lin -> lout (ping-pong)
// partial != NULL: also the residual of lin, ||f - K lin||^2 as per-CTA
// partials (returns their number)
int launch_gs_fused(const LevDev& L, const double* coef, const double* lin, double* lout,
                    const double* f, cudaStream_t st, double* partial = nullptr);
// per-device kernel attributes; returns the device's SM count
int gs_fused_prepare();
// k_gs_fused2.cu: the same sweep (bitwise) with a TMA-filled lambda ring and
// 32-bit coupling offsets (needs NT < 2^31)
extern int g_gs_v2;   // env WD_GS_V2=0: use k_gs_fused.cu
int make_ring_map(const LevDev& L, const double* v, void* map, int tj);   // box rows tj + 3
int gs_fused2_prepare();
// the prolongation folded into a sweep: lin + w P xc is the sweep's input
// (identity-z transitions with horizontal coarsening only; k_gs_fused2.cu)
struct ProlongIn {
    const double* xc;
    LevDev C;
    MapDev M;
    double w;
};
// ring_map / ring_map_res / ring_map_small: make_ring_map(.., tj = 8 / 6 / 4) of
// lin (the plain / PRO sweeps tile 64 x 8, the residual variant (partial) 64 x 6,
// the plain sweep on small levels 64 x 4); tr0, tr1: only the tile rows
// [tr0, tr1) (plain / PRO sweeps on 64 x 8 tiles; tr1 < 0: all)
int launch_gs_fused2(const LevDev& L, const double* coef, const void* ring_map,
                     const void* ring_map_res, const void* ring_map_small, double* lout,
                     const double* f, cudaStream_t st, double* partial = nullptr,
                     const ProlongIn* pro = nullptr, int tr0 = 0, int tr1 = -1);
void gs_fused2_tile_rows(const LevDev& L, int w, int* b0, int* b1, int* nty);

// k_io.cu: steps either side of the path
void launch_build_mesh(const double* zs, int n1, int n2, int n3, double x0, double y0, double dx,
                       double dy, const double* zeta, double H, double* X, double* Y, double* Z,
                       unsigned long long* bad, cudaStream_t st);
void launch_interp_wind(const double* uc, int nxc, int nyc, int nzc, double xc0, double yc0,
                        double DXc, double DYc, const double* hc, const double* X,
                        const double* Y, const double* Z, int n1, int n2, int n3, double* u0,
                        cudaStream_t st);
void launch_free_norms(const LevDev& L, const double* v, double* partial, int nb, double* out,
                       cudaStream_t st);

// k_apply_tma.cu: TMA-staged residual / apply
int make_coef_maps(const LevDev& L, const double* coef, void* mapA, void* mapB);
int make_vec_map(const LevDev& L, const double* v, void* map, bool halo);
void apply_tma_prepare();
int launch_apply_tma(const LevDev& L, const void* mapA, const void* mapB, const void* mapX,
                     const void* mapF, double* y, double* partial, cudaStream_t st);

// k_coarse.cu: coarsest-level direct solve
void launch_dense_build(const LevDev& L, const double* coef, double* A, int nf, cudaStream_t st);
void coarse_prepare(int nf);
int gj_invert(double* A, int n, double* scratch, cudaStream_t st);
void launch_coarse_gemv(const LevDev& L, const double* Ainv, int nf, const double* f,
                        double* x, cudaStream_t st);

}  // namespace wd
