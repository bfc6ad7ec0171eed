// k_mg.cu -- multigrid kernels on the 14-coefficient stencil (Sec. 3).
//
//   gs_phase_kernel  : one colour phase of the smoother, "vertical sweeps of
//                      Gauss-Seidel from the bottom up to the top, with
//                      red-black ordering horizontally into 4 groups"
//                      (P:174-176).  One thread per column of the colour,
//                      sequential in k, lambda of the 9 columns kept in a
//                      3-level register window.
//   apply_kernel     : y = K x  or  r = f - K x with deterministic block
//                      partial sums of r^2 (Eq. (7) residual, convergence test).
//   restrict_kernel  : f_c = P^T r  (Eq. (7), gather form, fixed order).
//   prolong_kernel   : x += P x_c   (Eq. (7)).
//   galerkin_kernel  : K_c = P^T K P (Eq. (7)) on the 14 forward slots.
// P is the index-space trilinear interpolation of P:176-181 (weights 1 and
// 1/2 per direction, tensor product), described by per-direction maps.
#include "wd_internal.cuh"

namespace wd {

namespace {

constexpr int GS_BLK = 128;
constexpr int AP_ROWS = 4;
constexpr int AP_BLK = 64 * AP_ROWS;

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// column offsets (same level) of the 9 columns (ox,oy) around (i,j), i of parity ci:
// c = (ox+1) + 3(oy+1)
__device__ __forceinline__ void column_offsets(const LevDev& L, int ci, i64 (&co)[9]) {
    const i64 xm = ci ? -(i64)L.H : (i64)L.H - 1;   // i-1 lives in the other half
    const i64 xp = ci ? 1 - (i64)L.H : (i64)L.H;    // i+1
#pragma unroll
    for (int oy = -1; oy <= 1; oy++) {
        co[0 + 3 * (oy + 1)] = (i64)oy * L.sj + xm;
        co[1 + 3 * (oy + 1)] = (i64)oy * L.sj;
        co[2 + 3 * (oy + 1)] = (i64)oy * L.sj + xp;
    }
}

__device__ __forceinline__ int cidx(int ox, int oy) { return (ox + 1) + 3 * (oy + 1); }

// sum_{q != p} K_pq x_q for node p at level k of column `o` (offset of level 0),
// with x of the 9 columns at levels k-1, k, k+1 in xm, x0, xp.
__device__ __forceinline__ double offdiag(const LevDev& L, const double* __restrict__ K,
                                          i64 base, const i64 (&co)[9], const double (&xm)[9],
                                          const double (&x0)[9], const double (&xp)[9],
                                          bool has_below) {
    const i64 NT = L.NT;
    double s = 0.0;
    // forward couplings K(p, p + d_s) stored at p
#pragma unroll
    for (int sl = 1; sl < 14; sl++) {
        const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
        const double kv = ldg(K + sl * NT + base);
        s = fma(kv, dz ? xp[cidx(dx, dy)] : x0[cidx(dx, dy)], s);
    }
    // backward couplings K(p, p - d_s) stored at p - d_s
#pragma unroll
    for (int sl = 1; sl < 14; sl++) {
        const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
        if (dz) {
            if (has_below) {
                const double kv = ldg(K + sl * NT + base - L.sk + co[cidx(-dx, -dy)]);
                s = fma(kv, xm[cidx(-dx, -dy)], s);
            }
        } else {
            const double kv = ldg(K + sl * NT + base + co[cidx(-dx, -dy)]);
            s = fma(kv, x0[cidx(-dx, -dy)], s);
        }
    }
    return s;
}

__global__ void __launch_bounds__(GS_BLK)
gs_phase_kernel(LevDev L, const double* __restrict__ K, double* lam,
                const double* __restrict__ f, int ci, int cj) {
    const int a = blockIdx.x * GS_BLK + threadIdx.x;
    const int i = 2 * a + ci;
    // owned local rows whose global row has parity cj
    const int j = L.own0 + ((cj - (L.own0 + L.jg0)) & 1) + 2 * (int)blockIdx.y;
    if (i < 1 || i > L.n1 - 2 || !row_free(L, j)) return;
    i64 co[9];
    column_offsets(L, ci, co);
    const i64 own = loff(L, i, j, 0);
    double xm[9], x0[9], xp[9];
#pragma unroll
    for (int c = 0; c < 9; c++) {
        xm[c] = 0.0;
        x0[c] = c == 4 ? lam[own] : ldg(lam + own + co[c]);
        xp[c] = c == 4 ? lam[own + L.sk] : ldg(lam + own + L.sk + co[c]);
    }
    const int kt = L.n3 - 2;   // top free level
    for (int k = 0; k <= kt; k++) {
        const i64 base = own + (i64)k * L.sk;
        const double s = offdiag(L, K, base, co, xm, x0, xp, k > 0);
        const double v = (ldg(f + base) - s) / ldg(K + base);
        lam[base] = v;
        x0[4] = v;
#pragma unroll
        for (int c = 0; c < 9; c++) {
            xm[c] = x0[c];
            x0[c] = xp[c];
        }
        if (k + 2 <= L.n3 - 1) {
            const i64 nb = base + 2 * L.sk;
#pragma unroll
            for (int c = 0; c < 9; c++) xp[c] = c == 4 ? lam[nb] : ldg(lam + nb + co[c]);
        }
    }
}

// One colour phase of vertical line relaxation: every free
// column of the colour is solved exactly for its planes 0..n3-2 given the
// current values of the 8 neighbouring columns (columns of one colour are not
// neighbours, so the phase is order-independent):  T x = f - (off-column
// part of K x), T tridiagonal with a_k = K(k, k-1) (slot 9 stored at k-1),
// b_k = K(k, k), c_k = K(k, k+1) (slot 9 at k; the top plane is Dirichlet).
// Thomas algorithm: forward elimination bottom-up, back substitution top-down
// into lam.  c'_k, d'_k are kept in shared memory ([k][thread], conflict
// free) when the column fits (SMEM_T), else in the two scratch arrays cpb,
// dpb at the node's own offset (HBM).
template <bool SMEM_T>
__global__ void __launch_bounds__(GS_BLK)
line_phase_kernel(LevDev L, const double* __restrict__ K, double* lam,
                  const double* __restrict__ f, double* __restrict__ cpb, double* __restrict__ dpb,
                  int ci, int cj) {
    extern __shared__ double tsc[];   // SMEM_T: c' at [k][t], d' at [m + k][t]
    const int a = blockIdx.x * GS_BLK + threadIdx.x;
    const int i = 2 * a + ci;
    const int j = L.own0 + ((cj - (L.own0 + L.jg0)) & 1) + 2 * (int)blockIdx.y;
    if (i < 1 || i > L.n1 - 2 || !row_free(L, j)) return;
    i64 co[9];
    column_offsets(L, ci, co);
    const i64 own = loff(L, i, j, 0);
    const i64 NT = L.NT;
    double xm[9], x0[9], xp[9];
#pragma unroll
    for (int c = 0; c < 9; c++) {
        xm[c] = 0.0;
        x0[c] = c == 4 ? 0.0 : ldg(lam + own + co[c]);
        xp[c] = c == 4 ? 0.0 : ldg(lam + own + L.sk + co[c]);
    }
    const int m = L.n3 - 1;   // free planes
    double cprev = 0.0, dprev = 0.0;
    for (int k = 0; k < m; k++) {
        const i64 base = own + (i64)k * L.sk;
        double s = 0.0;
        // forward couplings except the own column's (slot 9 = (0,0,1))
#pragma unroll
        for (int sl = 1; sl < 14; sl++) {
            const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
            if (dx == 0 && dy == 0) continue;
            s = fma(ldg(K + sl * NT + base), dz ? xp[cidx(dx, dy)] : x0[cidx(dx, dy)], s);
        }
        // backward couplings except the own column's
#pragma unroll
        for (int sl = 1; sl < 14; sl++) {
            const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
            if (dx == 0 && dy == 0) continue;
            if (dz) {
                if (k > 0) s = fma(ldg(K + sl * NT + base - L.sk + co[cidx(-dx, -dy)]), xm[cidx(-dx, -dy)], s);
            } else {
                s = fma(ldg(K + sl * NT + base + co[cidx(-dx, -dy)]), x0[cidx(-dx, -dy)], s);
            }
        }
        const double r = ldg(f + base) - s;
        const double b = ldg(K + base);
        const double cc = k < m - 1 ? ldg(K + 9 * NT + base) : 0.0;
        double cp, dp;
        if (k == 0) {
            cp = cc / b;
            dp = r / b;
        } else {
            const double ak = ldg(K + 9 * NT + base - L.sk);
            const double mk = b - ak * cprev;
            cp = cc / mk;
            dp = (r - ak * dprev) / mk;
        }
        if (SMEM_T) {
            tsc[k * GS_BLK + threadIdx.x] = cp;
            tsc[(m + k) * GS_BLK + threadIdx.x] = dp;
        } else {
            cpb[base] = cp;
            dpb[base] = dp;
        }
        cprev = cp;
        dprev = dp;
#pragma unroll
        for (int c = 0; c < 9; c++) {
            xm[c] = x0[c];
            x0[c] = xp[c];
        }
        if (k + 2 <= L.n3 - 1) {
            const i64 nb = base + 2 * L.sk;
#pragma unroll
            for (int c = 0; c < 9; c++) xp[c] = c == 4 ? 0.0 : ldg(lam + nb + co[c]);
        }
    }
    // back substitution, top-down
    double xn = dprev;
    lam[own + (i64)(m - 1) * L.sk] = xn;
    for (int k = m - 2; k >= 0; k--) {
        const i64 base = own + (i64)k * L.sk;
        if (SMEM_T)
            xn = tsc[(m + k) * GS_BLK + threadIdx.x] - tsc[k * GS_BLK + threadIdx.x] * xn;
        else
            xn = dpb[base] - cpb[base] * xn;
        lam[base] = xn;
    }
}

// deterministic block reduction (warp shuffle tree + fixed-order smem)
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double ws[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int w = tid >> 5, l = tid & 31;
    if (l == 0) ws[w] = v;
    __syncthreads();
    double r = 0.0;
    if (tid == 0) {
        const int nw = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
        for (int t = 0; t < nw; t++) r += ws[t];
    }
    __syncthreads();
    return r;
}

// CTA = 32 half-row positions x 2 parities x AP_ROWS rows: the backward
// couplings of a node (stored at the neighbour) are mostly loaded by another
// thread of the same CTA in the same or the previous k step (L1/L2 reuse).
__global__ void __launch_bounds__(AP_BLK)
apply_kernel(LevDev L, const double* __restrict__ K, const double* __restrict__ x,
             const double* __restrict__ f, double* __restrict__ y, double* __restrict__ partial,
             int variant) {
    int a, ci, j;
    if (variant == 0) {          // 128 along the half row, parity in blockIdx.z
        a = blockIdx.x * 128 + threadIdx.x; ci = blockIdx.z; j = blockIdx.y;
    } else if (variant == 1) {   // 128 along the half row, parity interleaved in blockIdx.x
        a = (blockIdx.x >> 1) * 128 + threadIdx.x; ci = blockIdx.x & 1; j = blockIdx.y;
    } else if (variant == 4) {   // as 1, one plane per CTA layer (blockIdx.z; small levels)
        a = (blockIdx.x >> 1) * 128 + threadIdx.x; ci = blockIdx.x & 1; j = blockIdx.y;
    } else if (variant == 2) {   // 32 x 2 parities x AP_ROWS rows
        a = blockIdx.x * 32 + threadIdx.x; ci = threadIdx.y; j = blockIdx.y * AP_ROWS + threadIdx.z;
    } else {                     // 128 x 2 parities, one row
        a = blockIdx.x * 128 + threadIdx.x; ci = threadIdx.y; j = blockIdx.y;
    }
    const int i = 2 * a + ci;
    double acc = 0.0;
    if (i >= 1 && i <= L.n1 - 2 && row_free(L, j)) {
        i64 co[9];
        column_offsets(L, ci, co);
        const i64 own = loff(L, i, j, 0);
        const int kz0 = variant == 4 ? (int)blockIdx.z : 0;
        const int kz1 = variant == 4 ? kz0 + 1 : L.n3 - 1;
        const i64 o0 = own + (i64)kz0 * L.sk;
        double xm[9], x0[9], xp[9];
#pragma unroll
        for (int c = 0; c < 9; c++) {
            xm[c] = kz0 > 0 ? ldg(x + o0 - L.sk + co[c]) : 0.0;
            x0[c] = ldg(x + o0 + co[c]);
            xp[c] = ldg(x + o0 + L.sk + co[c]);
        }
        for (int k = kz0; k < kz1; k++) {
            const i64 base = own + (i64)k * L.sk;
            double s = offdiag(L, K, base, co, xm, x0, xp, k > 0);
            s = fma(ldg(K + base), x0[4], s);
            const double v = f ? ldg(f + base) - s : s;
            y[base] = v;
            acc = fma(v, v, acc);
#pragma unroll
            for (int c = 0; c < 9; c++) {
                xm[c] = x0[c];
                x0[c] = xp[c];
            }
            if (k + 2 <= L.n3 - 1) {
                const i64 nb = base + 2 * L.sk;
#pragma unroll
                for (int c = 0; c < 9; c++) xp[c] = ldg(x + nb + co[c]);
            }
        }
    }
    if (partial) {
        const double s = block_sum(acc);
        if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0)
            partial[((i64)(variant == 4 ? blockIdx.z : 0) * gridDim.y + blockIdx.y) * gridDim.x +
                    blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(1024) reduce_kernel(const double* __restrict__ p, int n,
                                                      double* out) {
    double v = 0.0;
    for (int t = threadIdx.x; t < n; t += 1024) v += p[t];
    v = block_sum(v);
    if (threadIdx.x == 0) *out = v;
}

__global__ void __launch_bounds__(256) norm2_partial_kernel(const double* __restrict__ v, i64 n,
                                                             double* partial) {
    double acc = 0.0;
    const i64 stride = (i64)gridDim.x * 256;
    for (i64 t = (i64)blockIdx.x * 256 + threadIdx.x; t < n; t += stride) {
        const double a = v[t];
        acc = fma(a, a, acc);
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// natural [k][j][i] (ABI arrays, described by Nat) <-> internal i-split layout
__global__ void nat2int_kernel(LevDev L, Nat src, double* __restrict__ dst, int zero_dir) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, k = blockIdx.z;
    if (i >= L.n1) return;
    double v = src.p[((i64)k * src.n2a + j + src.jofs) * L.n1 + i];
    if (zero_dir && (i == 0 || i == L.n1 - 1 || row_dirichlet(L, j) || k == L.n3 - 1)) v = 0.0;
    dst[loff(L, i, j, k)] = v;
}

// internal -> natural, owned rows only
__global__ void int2nat_kernel(LevDev L, const double* __restrict__ src, Nat dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = L.own0 + (int)blockIdx.y, k = blockIdx.z;
    if (i >= L.n1 || j >= L.own1) return;
    const_cast<double*>(dst.p)[((i64)k * dst.n2a + j + dst.jofs) * L.n1 + i] = src[loff(L, i, j, k)];
}

__global__ void zero_dirichlet_kernel(LevDev L, double* v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, k = blockIdx.z;
    if (i >= L.n1) return;
    if (i == 0 || i == L.n1 - 1 || row_dirichlet(L, j) || k == L.n3 - 1) v[loff(L, i, j, k)] = 0.0;
}

// is coarse index c regular along a direction (kept fine indices of c-1..c+2 at spacing 2)?
__device__ __forceinline__ bool regular1d(const int* __restrict__ pos, int nc, int c) {
    if (c < 1 || c + 2 > nc - 1) return false;
    const int p = pos[c];
    return pos[c - 1] == p - 2 && pos[c + 1] == p + 2 && pos[c + 2] == p + 4;
}

// 1-D support of coarse index c along one direction: fine indices and weights
__device__ __forceinline__ int support1d(const int* __restrict__ pos, const int* __restrict__ co,
                                         int n, int c, int (&t)[3], double (&w)[3]) {
    const int p = pos[c];
    int m = 0;
    if (p - 1 >= 0 && !co[p - 1]) { t[m] = p - 1; w[m] = 0.5; m++; }
    t[m] = p; w[m] = 1.0; m++;
    if (p + 1 < n && !co[p + 1]) { t[m] = p + 1; w[m] = 0.5; m++; }
    return m;
}

// ZID: the transition's z map is the identity; the merging instance keeps
// the z supports of every coarse plane in shared memory (once per CTA), the
// identity one no shared memory (its L1 serves the 3 x 3 neighbourhoods)
template <bool ZID>
__global__ void __launch_bounds__(128)
restrict_kernel(LevDev F, LevDev C, MapDev M, const double* __restrict__ r,
                double* __restrict__ fc) {
    constexpr bool zident = ZID;
    const int I = blockIdx.x * 128 + threadIdx.x;
    const int J = blockIdx.y;
    constexpr int ZMAX = ZID ? 1 : 128;
    __shared__ int zt[ZMAX][3];
    __shared__ double zw[ZMAX][3];
    __shared__ int zm[ZMAX];
    const bool ztab = !ZID && C.n3 - 1 <= ZMAX;
    if (ztab) {
        for (int Kc = threadIdx.x; Kc <= C.n3 - 2; Kc += 128) {
            int t[3];
            double w[3];
            zm[Kc] = support1d(M.pos[2], M.co[2], F.n3, Kc, t, w);
            for (int c = 0; c < 3; c++) {
                zt[Kc][c] = t[c];
                zw[Kc][c] = w[c];
            }
        }
        __syncthreads();
    }
    if (I < 1 || I > C.n1 - 2 || !row_free(C, J)) return;
    // coarse planes of this thread: all, or (small levels, gridDim.z > 1) one
    const int kz0 = gridDim.z > 1 ? (int)blockIdx.z : 0;
    const int kz1 = gridDim.z > 1 ? min(kz0 + 1, C.n3 - 1) : C.n3 - 1;
    if (ztab && regular1d(M.pos[0], C.n1, I) && regular1d(M.pos[1], C.n2, J)) {
        // regular x and y supports {-1, 0, 1}, weights (1/2, 1, 1/2), z from the
        // table: the generic loop below with x and y unrolled (bitwise equal)
        const double w[3] = {0.5, 1.0, 0.5};
        const int fi = M.pos[0][I], fj = M.pos[1][J];
        for (int Kc = kz0; Kc < kz1; Kc++) {
            const int mz = zm[Kc];
            double s = 0.0;
            for (int c = 0; c < mz; c++) {
                const int kz = zt[Kc][c];
                const double wzc = zw[Kc][c];
#pragma unroll
                for (int b = 0; b < 3; b++) {
                    double sr = 0.0;
#pragma unroll
                    for (int a = 0; a < 3; a++) sr = fma(w[a], ldg(r + loff(F, fi + a - 1, fj + b - 1, kz)), sr);
                    s = fma(wzc * w[b], sr, s);
                }
            }
            fc[loff(C, I, J, Kc)] = s;
        }
        return;
    }
    if (zident && regular1d(M.pos[0], C.n1, I) && regular1d(M.pos[1], C.n2, J)) {
        // regular supports {-1, 0, 1} x {-1, 0, 1}, weights (1/2, 1, 1/2), identity in z:
        // the generic loop below with compile-time weights (same order, bitwise equal)
        const double w[3] = {0.5, 1.0, 0.5};
        const int fi = M.pos[0][I], fj = M.pos[1][J];
#pragma unroll 5   // several planes' 9 loads in flight
        for (int Kc = kz0; Kc < kz1; Kc++) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < 3; b++) {
                double sr = 0.0;
#pragma unroll
                for (int a = 0; a < 3; a++) sr = fma(w[a], ldg(r + loff(F, fi + a - 1, fj + b - 1, Kc)), sr);
                s = fma(1.0 * w[b], sr, s);
            }
            fc[loff(C, I, J, Kc)] = s;
        }
        return;
    }
    int tx[3], ty[3];
    double wx[3], wy[3];
    const int mx = support1d(M.pos[0], M.co[0], F.n1, I, tx, wx);
    const int my = support1d(M.pos[1], M.co[1], F.n2, J, ty, wy);
#pragma unroll 4
    for (int Kc = kz0; Kc < kz1; Kc++) {
        int tz[3];
        double wz[3];
        const int mz = support1d(M.pos[2], M.co[2], F.n3, Kc, tz, wz);
        double s = 0.0;
        for (int c = 0; c < mz; c++)
            for (int b = 0; b < my; b++) {
                double sr = 0.0;
                for (int a = 0; a < mx; a++) sr = fma(wx[a], ldg(r + loff(F, tx[a], ty[b], tz[c])), sr);
                s = fma(wz[c] * wy[b], sr, s);
            }
        fc[loff(C, I, J, Kc)] = s;
    }
}

// ZTAB: the merging instance, which tables every fine plane's z parent and
// count in shared memory; the identity-z instance keeps zident a run-time
// flag (as a compile-time constant the compiler batches the plane loop's
// loads at 120 registers: level-0 prolongation 0.67 -> 1.56 ms)
template <bool ZTAB>
__global__ void __launch_bounds__(128)
prolong_kernel(LevDev F, LevDev C, MapDev M, const double* __restrict__ xc,
               double* __restrict__ x, int zident, double w) {
    const int i = blockIdx.x * 128 + threadIdx.x;
    const int j = blockIdx.y;
    constexpr int ZMAX = ZTAB ? 256 : 1;
    __shared__ int zl[ZMAX], zn[ZMAX];
    const bool ztab = ZTAB && !zident && F.n3 - 1 <= ZMAX;
    if (ztab) {
        for (int k = threadIdx.x; k <= F.n3 - 2; k += 128) {
            zl[k] = M.lo[2][k];
            zn[k] = M.co[2][k] ? 1 : 2;
        }
        __syncthreads();
    }
    if (i < 1 || i > F.n1 - 2 || !row_free(F, j)) return;
    // fine planes of this thread: all, or (small levels, gridDim.z > 1) one
    const int kz0 = gridDim.z > 1 ? (int)blockIdx.z : 0;
    const int kz1 = gridDim.z > 1 ? min(kz0 + 1, F.n3 - 1) : F.n3 - 1;
    const int ix = M.lo[0][i], iy = M.lo[1][j];
    const int nx = M.co[0][i] ? 1 : 2, ny = M.co[1][j] ? 1 : 2;
    const double wx = nx == 1 ? 1.0 : 0.5, wy = ny == 1 ? 1.0 : 0.5;
    if (zident) {
        // identity in z (no layer merged): the loop below with iz = k and one z
        // term, branch-free in x (even and odd i share a warp; adding -0.0 is
        // the identity, so the sums are those of the generic loop bit for bit)
        const double* c0 = xc + loff(C, ix, iy, 0);
        const double* c1 = xc + loff(C, ix + nx - 1, iy, 0);
        const double* c2 = xc + loff(C, ix, iy + ny - 1, 0);
        const double* c3 = xc + loff(C, ix + nx - 1, iy + ny - 1, 0);
        double* xo = x + loff(F, i, j, 0);
        const bool two = nx == 2;
// one plane per iteration (unroll 16): batching 2, 4 or 8 planes' loads
// ahead of the stores, and a memory-order (row block) variant, all measured
// slower at Paper-scale level 0 (0.73 / 0.93 / 1.26 / 0.79 ms against 0.66)
#pragma unroll 16
        for (int k = kz0; k < kz1; k++) {
            const i64 kc = (i64)k * C.sk;
            double sr = 0.0 + ldg(c0 + kc);
            sr += two ? ldg(c1 + kc) : -0.0;
            double s = fma(wy * 1.0, wx * sr, 0.0);
            if (ny == 2) {
                double sr2 = 0.0 + ldg(c2 + kc);
                sr2 += two ? ldg(c3 + kc) : -0.0;
                s = fma(wy * 1.0, wx * sr2, s);
            }
            // x + w s: with w = 1 (Eq. (7)) the product is exact, so this is
            // x + s bit for bit; w != 1 only for the divergence-guard test
            xo[(i64)k * F.sk] = fma(w, s, xo[(i64)k * F.sk]);
        }
        return;
    }
    if (ztab) {
        // the generic loop below with x branch-free (as the identity-z path)
        // and z from the table (bitwise equal)
        const double* c0 = xc + loff(C, ix, iy, 0);
        const double* c1 = xc + loff(C, ix + nx - 1, iy, 0);
        const double* c2 = xc + loff(C, ix, iy + ny - 1, 0);
        const double* c3 = xc + loff(C, ix + nx - 1, iy + ny - 1, 0);
        double* xo = x + loff(F, i, j, 0);
        const bool two = nx == 2;
#pragma unroll 4
        for (int k = kz0; k < kz1; k++) {
            const int iz = zl[k], nz = zn[k];
            const double wz = nz == 1 ? 1.0 : 0.5;
            double s = 0.0;
            for (int c = 0; c < nz; c++) {
                const i64 kc = (i64)(iz + c) * C.sk;
                double sr = 0.0 + ldg(c0 + kc);
                sr += two ? ldg(c1 + kc) : -0.0;
                s = fma(wy * wz, wx * sr, s);
                if (ny == 2) {
                    double sr2 = 0.0 + ldg(c2 + kc);
                    sr2 += two ? ldg(c3 + kc) : -0.0;
                    s = fma(wy * wz, wx * sr2, s);
                }
            }
            xo[(i64)k * F.sk] = fma(w, s, xo[(i64)k * F.sk]);
        }
        return;
    }
#pragma unroll 4
    for (int k = kz0; k < kz1; k++) {
        const int iz = M.lo[2][k];
        const int nz = M.co[2][k] ? 1 : 2;
        const double wz = nz == 1 ? 1.0 : 0.5;
        double s = 0.0;
        for (int c = 0; c < nz; c++)
            for (int b = 0; b < ny; b++) {
                double sr = 0.0;
                for (int a = 0; a < nx; a++) sr += ldg(xc + loff(C, ix + a, iy + b, iz + c));
                s = fma(wy * wz, wx * sr, s);
            }
        const i64 o = loff(F, i, j, k);
        x[o] = fma(w, s, x[o]);
    }
}

// K(p, p + d) from 14-slot storage (d in {-1,0,1}^3, both ends inside the grid)
__device__ __forceinline__ double kget(const LevDev& L, const double* __restrict__ K, int i, int j,
                                       int k, int dx, int dy, int dz) {
    const int s = slot_of(dx, dy, dz);
    if (s >= 0) return ldg(K + s * L.NT + loff(L, i, j, k));
    return ldg(K + (-s) * L.NT + loff(L, i + dx, j + dy, k + dz));
}

// 1-D pair lists of the Galerkin product for a regular coarse index (coarse
// neighbours at fine distance 2 on both sides, so the support of I is the
// fine offsets -1, 0, 1 with weights 1/2, 1, 1/2 around pos(I)): for coarse
// offset D the pairs (u, v) = (offset of a node of supp(I), offset of a node
// of supp(I+D)), both relative to pos(I), with |v - u| <= 1, and the product
// of their weights, in the order support1d/galerkin_kernel enumerate them
// (u major, both ascending).
struct Pair1 { int u, v; double w; };

template <int D>
__device__ __forceinline__ constexpr int npairs() { return D == 0 ? 7 : 3; }
template <int D>
__device__ __forceinline__ Pair1 pair(int n) {
    // compile-time tables (the loops below are fully unrolled)
    constexpr Pair1 P0[7] = {{-1, -1, 0.25}, {-1, 0, 0.5}, {0, -1, 0.5}, {0, 0, 1.0},
                             {0, 1, 0.5}, {1, 0, 0.5}, {1, 1, 0.25}};
    constexpr Pair1 PP[3] = {{0, 1, 0.5}, {1, 1, 0.25}, {1, 2, 0.5}};
    constexpr Pair1 PM[3] = {{-1, -2, 0.5}, {-1, -1, 0.25}, {0, -1, 0.5}};
    return D == 0 ? P0[n] : D > 0 ? PP[n] : PM[n];
}

// K_c(I, I + (DX, DY, DZ)) for a coarse node whose x and y supports are
// regular and whose z map is the identity: the same products and sums in the
// same order as the generic loop of galerkin_kernel (bitwise equal), with
// every index a compile-time offset.
template <int DX, int DY, int DZ>
__device__ __forceinline__ double galerkin_regular(const LevDev& F, const double* __restrict__ K,
                                                   int fi, int fj, int k) {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < npairs<DY>(); b++) {
        const Pair1 py = pair<DY>(b);
        double sr = 0.0;
#pragma unroll
        for (int a = 0; a < npairs<DX>(); a++) {
            const Pair1 px = pair<DX>(a);
            sr = fma(px.w, kget(F, K, fi + px.u, fj + py.u, k, px.v - px.u, py.v - py.u, DZ), sr);
        }
        s = fma(1.0 * py.w, sr, s);
    }
    return s;
}

// z pair list of the Galerkin product for coarse plane Kc and offset DZ (the
// generic loop's construction: u major, v minor, |q - p| <= 1)
__device__ __forceinline__ int zpairs(const MapDev& M, int fn3, int Kc, int DZ, int (&lt)[9],
                                      int (&ld)[9], double (&lw)[9]) {
    int pt[3], qt[3];
    double pw[3], qw[3];
    const int pm = support1d(M.pos[2], M.co[2], fn3, Kc, pt, pw);
    const int qm = support1d(M.pos[2], M.co[2], fn3, Kc + DZ, qt, qw);
    int n = 0;
    for (int u = 0; u < pm; u++)
        for (int v = 0; v < qm; v++) {
            const int dd = qt[v] - pt[u];
            if (dd >= -1 && dd <= 1) {
                lt[n] = pt[u];
                ld[n] = dd;
                lw[n] = pw[u] * qw[v];
                n++;
            }
        }
    return n;
}

// K_c(I, I + (DX, DY, DZ)) for a coarse node with regular x and y supports on a
// transition that merges layers (z map not the identity): x and y unrolled
// with compile-time offsets, z pairs from zpairs() (computed once per CTA --
// the coarse plane is blockIdx.z -- and read from shared memory), each pair's
// z offset dispatched to a compile-time body; the generic loop's products and
// sums in its order (bitwise equal)
template <int DX, int DY, int DZ>
__device__ __forceinline__ double galerkin_zpair(const LevDev& F, const double* __restrict__ K,
                                                 int fi, int fj, int k, double wz, double s) {
#pragma unroll
    for (int b = 0; b < npairs<DY>(); b++) {
        const Pair1 py = pair<DY>(b);
        double sr = 0.0;
#pragma unroll
        for (int a = 0; a < npairs<DX>(); a++) {
            const Pair1 px = pair<DX>(a);
            sr = fma(px.w, kget(F, K, fi + px.u, fj + py.u, k, px.v - px.u, py.v - py.u, DZ), sr);
        }
        s = fma(wz * py.w, sr, s);
    }
    return s;
}

struct ZPairs {
    int t[9], d[9];
    double w[9];
    int n;
};

template <int DX, int DY>
__device__ __forceinline__ double galerkin_xyreg(const LevDev& F, const double* __restrict__ K,
                                                 int fi, int fj, const ZPairs& zp) {
    double s = 0.0;
    for (int c = 0; c < zp.n; c++) {
        const int k = zp.t[c], dz = zp.d[c];
        const double wz = zp.w[c];
        if (dz < 0) s = galerkin_zpair<DX, DY, -1>(F, K, fi, fj, k, wz, s);
        else if (dz == 0) s = galerkin_zpair<DX, DY, 0>(F, K, fi, fj, k, wz, s);
        else s = galerkin_zpair<DX, DY, 1>(F, K, fi, fj, k, wz, s);
    }
    return s;
}

// (128, 8): <= 64 registers, 8 CTAs per SM: Paper-scale Galerkin products 12.8 -> 12.2 ms
// (a 48- or 40-register cap spilled: 13.9 / 16.2 ms)
// ZID: the transition's z map is the identity (an instance per case, so that
// the merging case's shared z-pair lists do not weigh on the other)
template <bool ZID>
__global__ void __launch_bounds__(128, 8)
galerkin_kernel(LevDev F, LevDev C, MapDev M, const double* __restrict__ KF,
                double* __restrict__ KC, int fast) {
    const int I = blockIdx.x * 128 + threadIdx.x;
    const int J = blockIdx.y, Kc = blockIdx.z;
    __shared__ ZPairs zp[ZID ? 1 : 2];   // z pairs of coarse plane Kc for DZ = 0, 1 (merging)
    if (!ZID && fast) {
        if (threadIdx.x < 2 && Kc + (int)threadIdx.x <= C.n3 - 1) {
            ZPairs& z = zp[threadIdx.x];
            z.n = zpairs(M, F.n3, Kc, threadIdx.x, z.t, z.d, z.w);
        }
        __syncthreads();
    }
    if (I < 1 || I > C.n1 - 2 || !row_free(C, J) || Kc > C.n3 - 2) return;
    const bool xyreg = fast && regular1d(M.pos[0], C.n1, I) && regular1d(M.pos[1], C.n2, J);
    if (!ZID && xyreg) {
        const int fi = M.pos[0][I], fj = M.pos[1][J];
        const ZPairs& z0 = zp[0];
        const ZPairs& z1 = zp[ZID ? 0 : 1];
        double* o = KC + loff(C, I, J, Kc);
        o[0 * C.NT] = galerkin_xyreg<0, 0>(F, KF, fi, fj, z0);
        o[1 * C.NT] = galerkin_xyreg<1, 0>(F, KF, fi, fj, z0);
        o[2 * C.NT] = galerkin_xyreg<-1, 1>(F, KF, fi, fj, z0);
        o[3 * C.NT] = galerkin_xyreg<0, 1>(F, KF, fi, fj, z0);
        o[4 * C.NT] = galerkin_xyreg<1, 1>(F, KF, fi, fj, z0);
        o[5 * C.NT] = galerkin_xyreg<-1, -1>(F, KF, fi, fj, z1);
        o[6 * C.NT] = galerkin_xyreg<0, -1>(F, KF, fi, fj, z1);
        o[7 * C.NT] = galerkin_xyreg<1, -1>(F, KF, fi, fj, z1);
        o[8 * C.NT] = galerkin_xyreg<-1, 0>(F, KF, fi, fj, z1);
        o[9 * C.NT] = galerkin_xyreg<0, 0>(F, KF, fi, fj, z1);
        o[10 * C.NT] = galerkin_xyreg<1, 0>(F, KF, fi, fj, z1);
        o[11 * C.NT] = galerkin_xyreg<-1, 1>(F, KF, fi, fj, z1);
        o[12 * C.NT] = galerkin_xyreg<0, 1>(F, KF, fi, fj, z1);
        o[13 * C.NT] = galerkin_xyreg<1, 1>(F, KF, fi, fj, z1);
        return;
    }
    if (xyreg) {   // identity z
        const int fi = M.pos[0][I], fj = M.pos[1][J];
        const i64 out = loff(C, I, J, Kc);
        double* o = KC + out;
        o[0 * C.NT] = galerkin_regular<0, 0, 0>(F, KF, fi, fj, Kc);
        o[1 * C.NT] = galerkin_regular<1, 0, 0>(F, KF, fi, fj, Kc);
        o[2 * C.NT] = galerkin_regular<-1, 1, 0>(F, KF, fi, fj, Kc);
        o[3 * C.NT] = galerkin_regular<0, 1, 0>(F, KF, fi, fj, Kc);
        o[4 * C.NT] = galerkin_regular<1, 1, 0>(F, KF, fi, fj, Kc);
        o[5 * C.NT] = galerkin_regular<-1, -1, 1>(F, KF, fi, fj, Kc);
        o[6 * C.NT] = galerkin_regular<0, -1, 1>(F, KF, fi, fj, Kc);
        o[7 * C.NT] = galerkin_regular<1, -1, 1>(F, KF, fi, fj, Kc);
        o[8 * C.NT] = galerkin_regular<-1, 0, 1>(F, KF, fi, fj, Kc);
        o[9 * C.NT] = galerkin_regular<0, 0, 1>(F, KF, fi, fj, Kc);
        o[10 * C.NT] = galerkin_regular<1, 0, 1>(F, KF, fi, fj, Kc);
        o[11 * C.NT] = galerkin_regular<-1, 1, 1>(F, KF, fi, fj, Kc);
        o[12 * C.NT] = galerkin_regular<0, 1, 1>(F, KF, fi, fj, Kc);
        o[13 * C.NT] = galerkin_regular<1, 1, 1>(F, KF, fi, fj, Kc);
        return;
    }
    int pt[3][3];
    double pw[3][3];
    int pm[3];
    pm[0] = support1d(M.pos[0], M.co[0], F.n1, I, pt[0], pw[0]);
    pm[1] = support1d(M.pos[1], M.co[1], F.n2, J, pt[1], pw[1]);
    pm[2] = support1d(M.pos[2], M.co[2], F.n3, Kc, pt[2], pw[2]);
    const int nd[3] = {F.n1, F.n2, F.n3};
    const int Pc[3] = {I, J, Kc};
    const i64 out = loff(C, I, J, Kc);
    for (int sl = 0; sl < 14; sl++) {
        const int d[3] = {slot_dx(sl), slot_dy(sl), slot_dz(sl)};
        // per-direction pair lists (p_t, q_t - p_t, w_P w_Q) with |q_t - p_t| <= 1
        int lt[3][9], ld[3][9];
        double lw[3][9];
        int ln[3];
#pragma unroll
        for (int e = 0; e < 3; e++) {
            int qt[3];
            double qw[3];
            const int qm = support1d(M.pos[e], M.co[e], nd[e], Pc[e] + d[e], qt, qw);
            int n = 0;
            for (int u = 0; u < pm[e]; u++)
                for (int v = 0; v < qm; v++) {
                    const int dd = qt[v] - pt[e][u];
                    if (dd >= -1 && dd <= 1) {
                        lt[e][n] = pt[e][u];
                        ld[e][n] = dd;
                        lw[e][n] = pw[e][u] * qw[v];
                        n++;
                    }
                }
            ln[e] = n;
        }
        double s = 0.0;
        for (int c = 0; c < ln[2]; c++)
            for (int b = 0; b < ln[1]; b++) {
                double sr = 0.0;
                for (int a = 0; a < ln[0]; a++)
                    sr = fma(lw[0][a], kget(F, KF, lt[0][a], lt[1][b], lt[2][c], ld[0][a], ld[1][b],
                                            ld[2][c]), sr);
                s = fma(lw[2][c] * lw[1][b], sr, s);
            }
        KC[sl * C.NT + out] = s;
    }
}

__global__ void export27_kernel(LevDev L, const double* __restrict__ K, double* __restrict__ K27) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, k = blockIdx.z;
    if (i >= L.n1) return;
    const i64 p = ((i64)k * L.n2 + j) * L.n1 + i;
    for (int o = 0; o < 27; o++) {
        const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
        const int ii = i + dx, jj = j + dy, kk = k + dz;
        double v = 0.0;
        if (ii >= 0 && ii < L.n1 && jj >= 0 && jj < L.n2 && kk >= 0 && kk < L.n3)
            v = kget(L, K, i, j, k, dx, dy, dz);
        K27[p * 27 + o] = v;
    }
}

// argmin over the bottom plane (ties -> smallest index), two passes
__global__ void argmin_kernel(const double* __restrict__ z, long long n,
                              const long long* __restrict__ idx_in, double* pval,
                              long long* pidx) {
    __shared__ double sv[256];
    __shared__ long long si[256];
    double best = 1.0 / 0.0;
    long long bi = 0x7fffffffffffffffll;
    const long long stride = (long long)gridDim.x * 256;
    for (long long t = (long long)blockIdx.x * 256 + threadIdx.x; t < n; t += stride) {
        const double v = z[t];
        const long long id = idx_in ? idx_in[t] : t;
        if (v < best || (v == best && id < bi)) { best = v; bi = id; }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const double v = sv[threadIdx.x + o];
            const long long id = si[threadIdx.x + o];
            if (v < sv[threadIdx.x] || (v == sv[threadIdx.x] && id < si[threadIdx.x])) {
                sv[threadIdx.x] = v;
                si[threadIdx.x] = id;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pval[blockIdx.x] = sv[0];
        pidx[blockIdx.x] = si[0];
    }
}

dim3 node_grid(const LevDev& L) { return dim3((L.n1 + 127) / 128, L.n2, L.n3); }

}  // namespace

void launch_nat2int(const LevDev& L, Nat src, double* dst, bool zero_dirichlet, cudaStream_t st) {
    g_launches += 1;
    nat2int_kernel<<<node_grid(L), 128, 0, st>>>(L, src, dst, zero_dirichlet ? 1 : 0);
}

void launch_int2nat(const LevDev& L, const double* src, Nat dst, cudaStream_t st) {
    g_launches += 1;
    int2nat_kernel<<<node_grid(L), 128, 0, st>>>(L, src, dst);
}

void launch_zero_dirichlet(const LevDev& L, double* v, cudaStream_t st) {
    g_launches += 1;
    zero_dirichlet_kernel<<<node_grid(L), 128, 0, st>>>(L, v);
}

// colour phase c of the smoother: (i mod 2, j mod 2) = (0,0),(1,0),(0,1),(1,1) (reading C7)
void launch_gs_phase(const LevDev& L, const double* coef, double* lam, const double* f, int c,
                     cudaStream_t st) {
    static const int colour[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
    const int half = (L.n1 + 1) / 2;
    dim3 grid((half + GS_BLK - 1) / GS_BLK, (L.own1 - L.own0 + 2) / 2);
    g_launches += 1;
    gs_phase_kernel<<<grid, GS_BLK, 0, st>>>(L, coef, lam, f, colour[c][0], colour[c][1]);
}

void launch_line_phase(const LevDev& L, const double* coef, double* lam, const double* f,
                       double* cpb, double* dpb, int c, cudaStream_t st) {
    static const int colour[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
    const int half = (L.n1 + 1) / 2;
    dim3 grid((half + GS_BLK - 1) / GS_BLK, (L.own1 - L.own0 + 2) / 2);
    g_launches += 1;
    // the Thomas scratch of a column in shared memory when it fits (n3 <= 33:
    // <= 64 KB per 128-thread block), else in HBM
    const int m = L.n3 - 1;
    const size_t smem = sizeof(double) * 2 * (size_t)m * GS_BLK;
    if (m <= 32) {
        static int attr_set[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= 0 && dev < 64 && !attr_set[dev]) {
            cudaFuncSetAttribute(line_phase_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 64 * 1024 + 1024);
            attr_set[dev] = 1;
        }
        line_phase_kernel<true><<<grid, GS_BLK, smem, st>>>(L, coef, lam, f, cpb, dpb, colour[c][0],
                                                            colour[c][1]);
    } else {
        line_phase_kernel<false><<<grid, GS_BLK, 0, st>>>(L, coef, lam, f, cpb, dpb, colour[c][0],
                                                          colour[c][1]);
    }
}

void launch_gs_sweep(const LevDev& L, const double* coef, double* lam, const double* f,
                     cudaStream_t st) {
    for (int c = 0; c < 4; c++) launch_gs_phase(L, coef, lam, f, c, st);
}

__global__ void sum_ordered_kernel(const double* __restrict__ v, int n, double* out) {
    double s = 0.0;
    for (int t = 0; t < n; t++) s += v[t];
    *out = s;
}

// out = v[0] + v[1] + ... + v[n-1] in this order (rank-ordered partial sums)
void launch_sum_ordered(const double* v, int n, double* out, cudaStream_t st) {
    g_launches += 1;
    sum_ordered_kernel<<<1, 1, 0, st>>>(v, n, out);
}

int launch_apply(const LevDev& L, const double* coef, const double* x, const double* f, double* y,
                 double* partial, cudaStream_t st, int variant) {
    const int half = (L.n1 + 1) / 2;
    const int v = variant >= 0 ? variant : g_apply_variant;
    dim3 grid, blk;
    if (v == 0) { grid = dim3((half + 127) / 128, L.n2, 2); blk = dim3(128); }
    else if (v == 1) { grid = dim3(2 * ((half + 127) / 128), L.n2, 1); blk = dim3(128); }
    else if (v == 2) { grid = dim3((half + 31) / 32, (L.n2 + AP_ROWS - 1) / AP_ROWS, 1); blk = dim3(32, 2, AP_ROWS); }
    else if (v == 4) { grid = dim3(2 * ((half + 127) / 128), L.n2, L.n3 - 1); blk = dim3(128); }
    else { grid = dim3((half + 127) / 128, L.n2, 1); blk = dim3(128, 2); }
    g_launches += 1;
    apply_kernel<<<grid, blk, 0, st>>>(L, coef, x, f, y, partial, v);
    return (int)(grid.x * grid.y * grid.z);
}

void launch_reduce_sum(const double* partial, int n, double* out, cudaStream_t st) {
    g_launches += 1;
    reduce_kernel<<<1, 1024, 0, st>>>(partial, n, out);
}

void launch_norm2_partial(const LevDev& L, const double* v, double* partial, int* nblk,
                          cudaStream_t st) {
    const int nb = 1184;   // 8 x 148 SMs
    g_launches += 1;
    norm2_partial_kernel<<<nb, 256, 0, st>>>(v, L.NT, partial);
    *nblk = nb;
}

#ifndef WD_SMALL_COLS
#define WD_SMALL_COLS (300LL * 300LL)
#endif
constexpr long long SMALL_COLS = WD_SMALL_COLS;

void launch_restrict(const LevDev& F, const LevDev& Cl, const MapDev& M, const double* r,
                     double* fc, int zident, cudaStream_t st) {
    // small levels: one coarse plane per CTA layer (the per-thread plane loop
    // is latency-bound there)
    const bool split = (long long)Cl.n1 * Cl.n2 <= SMALL_COLS;
    dim3 grid((Cl.n1 + 127) / 128, Cl.n2, split ? Cl.n3 - 1 : 1);
    g_launches += 1;
    if (zident) restrict_kernel<true><<<grid, 128, 0, st>>>(F, Cl, M, r, fc);
    else restrict_kernel<false><<<grid, 128, 0, st>>>(F, Cl, M, r, fc);
}

void launch_prolong(const LevDev& F, const LevDev& Cl, const MapDev& M, const double* xc,
                    double* x, int zident, cudaStream_t st, double w) {
    const bool split = (long long)F.n1 * F.n2 <= SMALL_COLS;
    dim3 grid((F.n1 + 127) / 128, F.n2, split ? F.n3 - 1 : 1);
    g_launches += 1;
    if (zident) prolong_kernel<false><<<grid, 128, 0, st>>>(F, Cl, M, xc, x, 1, w);
    else prolong_kernel<true><<<grid, 128, 0, st>>>(F, Cl, M, xc, x, 0, w);
}

// The 14 coefficient arrays are allocated without a zero fill; this writes
// zeros where neither writer does: the padding positions of every half row,
// and (galerkin) the Dirichlet nodes, which the Galerkin product skips (the
// assembly writes every real node).  Either writer fills the rest.
__global__ void zero_unwritten_kernel(LevDev L, double* __restrict__ coef, int galerkin) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;   // position in the row block's plane
    const int j = blockIdx.y, k = blockIdx.z;
    if (e >= L.P) return;
    const int half = e >= L.H, pos = e - half * L.H;
    const int i = 2 * pos + half;
    const bool pad = i >= L.n1;
    const bool dir = i == 0 || i == L.n1 - 1 || row_dirichlet(L, j) || k == L.n3 - 1;
    if (!pad && !(galerkin && dir)) return;
    const i64 o = (i64)j * L.sj + (i64)k * L.sk + e;
#pragma unroll
    for (int s = 0; s < 14; s++) coef[s * L.NT + o] = 0.0;
}

void launch_zero_unwritten(const LevDev& L, double* coef, bool galerkin, cudaStream_t st) {
    dim3 grid((L.P + 127) / 128, L.n2, L.n3);
    g_launches += 1;
    zero_unwritten_kernel<<<grid, 128, 0, st>>>(L, coef, galerkin ? 1 : 0);
}

void launch_galerkin(const LevDev& F, const LevDev& Cl, const MapDev& M, const double* coefF,
                     double* coefC, int zident, cudaStream_t st) {
    dim3 grid((Cl.n1 + 127) / 128, Cl.n2, Cl.n3);
    g_launches += 1;
    if (zident) galerkin_kernel<true><<<grid, 128, 0, st>>>(F, Cl, M, coefF, coefC, !g_galerkin_generic);
    else galerkin_kernel<false><<<grid, 128, 0, st>>>(F, Cl, M, coefF, coefC, !g_galerkin_generic);
}

void launch_export27(const LevDev& L, const double* coef, double* K27, cudaStream_t st) {
    g_launches += 1;
    export27_kernel<<<node_grid(L), 128, 0, st>>>(L, coef, K27);
}

void launch_argmin_bottom(const double* Z, int n, double* pval, long long* pidx, int nblk,
                          cudaStream_t st) {
    g_launches += 2;
    argmin_kernel<<<nblk, 256, 0, st>>>(Z, n, nullptr, pval, pidx);
    argmin_kernel<<<1, 256, 0, st>>>(pval, nblk, pidx, pval + nblk, pidx + nblk);
}

}  // namespace wd
