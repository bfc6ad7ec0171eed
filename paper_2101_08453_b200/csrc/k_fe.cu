// k_fe.cu -- finite-element kernels for sm_100a, fp64 (Sec. 2).
//
//   assemble_kernel : element stiffness by 2x2x2 Gauss quadrature
//                     gathered into the 14-coefficient symmetric nodal stencil,
//                     fused with mesh validation (detJ > 0, Z increasing).
//   rhs_kernel      : one-point RHS f = -int grad mu . u0.
//   recover_kernel  : u = u0 + A^{-1} grad lambda at element centres
//                     (Eq. (3)).
// The RHS and recovery kernels share one centre-derivative routine
// (centre_jacobian), as P:112-114 prescribes.
//
// Tiling: a CTA owns a (TX-1) x (TY-1) tile of node columns and computes the
// TX x TY element columns around it (1-element halo recomputed), streaming
// upward in k.  Element results go to shared memory; each node thread gathers
// its couplings from the 4 element columns in a fixed order (deterministic,
// no atomics).  Partial sums of the node level k+1 (contributions of the
// element level k) stay in registers until element level k+1 completes them.
#include "wd_internal.cuh"

namespace wd {

namespace {

constexpr int TX = 32, TY = 8, NTH = TX * TY;   // element columns per CTA
constexpr double GP = 0.57735026918962576451;  // 1/sqrt(3)

__host__ __device__ constexpr double sgn(int a, int d) { return ((a >> d) & 1) ? 1.0 : -1.0; }

// dN_a/dxi_d at reference point xi (compile-time constant when xi is)
__host__ __device__ constexpr double dN(int a, int d, double x0, double x1, double x2) {
    return d == 0 ? 0.5 * sgn(a, 0) * 0.5 * (1.0 + sgn(a, 1) * x1) * 0.5 * (1.0 + sgn(a, 2) * x2)
         : d == 1 ? 0.5 * sgn(a, 1) * 0.5 * (1.0 + sgn(a, 0) * x0) * 0.5 * (1.0 + sgn(a, 2) * x2)
                  : 0.5 * sgn(a, 2) * 0.5 * (1.0 + sgn(a, 0) * x0) * 0.5 * (1.0 + sgn(a, 1) * x1);
}

__host__ __device__ constexpr int ut(int a, int b) { return a * (15 - a) / 2 + b; }  // a <= b

// J[m][d] = sum_a x[a][m] dN_a/dxi_d ; returns det and Ji = J^{-1} (Ji[d][m])
__device__ __forceinline__ double jac_inv(const double (&x)[8][3], double x0, double x1,
                                          double x2, double (&Ji)[3][3]) {
    double J[3][3];
#pragma unroll
    for (int m = 0; m < 3; m++)
#pragma unroll
        for (int d = 0; d < 3; d++) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < 8; a++) s = fma(x[a][m], dN(a, d, x0, x1, x2), s);
            J[m][d] = s;
        }
    double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    double id = 1.0 / det;
    Ji[0][0] = c00 * id;
    Ji[1][0] = c01 * id;
    Ji[2][0] = c02 * id;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
    return det;
}

// Centre geometry shared by the RHS and the recovery.
__device__ __forceinline__ double centre_jacobian(const double (&x)[8][3], double (&Ji)[3][3]) {
    return jac_inv(x, 0.0, 0.0, 0.0, Ji);
}

// Upper triangle of the element stiffness,
//   Ke_ab = sum_g detJ_g grad N_a . diag(c) grad N_b
//         = sum_g sum_{d,e} dN_a/dxi_d (detJ_g Ji c Ji^T)_{de} dN_b/dxi_e,
// accumulated Gauss point by Gauss point (weights 1).  Returns the first
// failing Gauss point + 1, or 0.
__device__ __forceinline__ int element_stiffness(const double (&x)[8][3], double c0, double c1,
                                                 double c2, double (&K)[36]) {
    int badg = 0;
#pragma unroll
    for (int t = 0; t < 36; t++) K[t] = 0.0;
#pragma unroll
    for (int g = 0; g < 8; g++) {
        const double x0 = (g & 1) ? GP : -GP;
        const double x1 = (g & 2) ? GP : -GP;
        const double x2 = (g & 4) ? GP : -GP;
        double Ji[3][3];
        double det = jac_inv(x, x0, x1, x2, Ji);
        if (!(det > 0.0) && badg == 0) badg = g + 1;
        // M = det * Ji diag(c) Ji^T  (symmetric 3x3)
        double M[3][3];
#pragma unroll
        for (int d = 0; d < 3; d++)
#pragma unroll
            for (int e = d; e < 3; e++) {
                double s = c0 * Ji[d][0] * Ji[e][0];
                s = fma(c1 * Ji[d][1], Ji[e][1], s);
                s = fma(c2 * Ji[d][2], Ji[e][2], s);
                M[d][e] = det * s;
                M[e][d] = M[d][e];
            }
        // v_b = M grad_xi N_b (9 FMA per node), then K_ab += grad_xi N_a . v_b
        // (3 FMA per pair): 72 + 108 instead of 36 x 9 FMA per Gauss point
#pragma unroll
        for (int b = 0; b < 8; b++) {
            double v[3];
#pragma unroll
            for (int d = 0; d < 3; d++) {
                double t = M[d][0] * dN(b, 0, x0, x1, x2);
                t = fma(M[d][1], dN(b, 1, x0, x1, x2), t);
                v[d] = fma(M[d][2], dN(b, 2, x0, x1, x2), t);
            }
#pragma unroll
            for (int a = 0; a <= b; a++) {
                double s = K[ut(a, b)];
#pragma unroll
                for (int d = 0; d < 3; d++) s = fma(dN(a, d, x0, x1, x2), v[d], s);
                K[ut(a, b)] = s;
            }
        }
    }
    return badg;
}

__device__ __forceinline__ void load_plane(const double* __restrict__ X,
                                           const double* __restrict__ Y,
                                           const double* __restrict__ Z, int n1, int n2, int i,
                                           int j, int k, double (&x)[8][3], int top) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
        i64 p = ((i64)k * n2 + (j + (q >> 1))) * n1 + (i + (q & 1));
        x[q + 4 * top][0] = __ldg(X + p);
        x[q + 4 * top][1] = __ldg(Y + p);
        x[q + 4 * top][2] = __ldg(Z + p);
    }
}

// node-side gather of the element-level couplings: node is local index
// a = (1-ex) + 2(1-ey) + 4 dc in the element column (ex, ey) of its 2x2.
template <int DC>
__device__ __forceinline__ void gather_couplings(const double* ke, int t, double (&acc)[14]) {
#pragma unroll
    for (int ey = 0; ey < 2; ey++)
#pragma unroll
        for (int ex = 0; ex < 2; ex++) {
            const int te = t + ex + ey * TX;
            const int a = (1 - ex) + 2 * (1 - ey) + 4 * DC;
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const int s = slot_of((b & 1) - (a & 1), ((b >> 1) & 1) - ((a >> 1) & 1),
                                      ((b >> 2) & 1) - DC);
                if (s >= 0) {
                    const int u = a <= b ? ut(a, b) : ut(b, a);
                    acc[s] += ke[u * NTH + te];
                }
            }
        }
}

__global__ void __launch_bounds__(NTH, 1)
assemble_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                const double* __restrict__ Z, int n1, int n2, int n3, double c0, double c1,
                double c2, LevDev L, double* __restrict__ coef, unsigned long long* bad,
                int ty0) {
    extern __shared__ double ke[];   // [36][NTH]
    const int t = threadIdx.x;
    const int tx = t % TX, ty = t / TX;
    const int i0 = blockIdx.x * (TX - 1), j0 = (blockIdx.y + ty0) * (TY - 1);
    const int ei = i0 - 1 + tx, ej = j0 - 1 + ty;
    const bool ev = ei >= 0 && ei < n1 - 1 && ej >= 0 && ej < n2 - 1;
    const int ni = i0 + tx, nj = j0 + ty;
    const bool nv = tx < TX - 1 && ty < TY - 1 && ni < n1 && nj < n2;
    const int nx = n1 - 1, ny = n2 - 1;

    double x[8][3];
    if (ev) load_plane(X, Y, Z, n1, n2, ei, ej, 0, x, 0);
    double acc[14];
#pragma unroll
    for (int s = 0; s < 14; s++) acc[s] = 0.0;
    for (int ek = 0; ek < n3 - 1; ek++) {
        double K[36];
        if (ev) {
            load_plane(X, Y, Z, n1, n2, ei, ej, ek + 1, x, 1);
            int badg = element_stiffness(x, c0, c1, c2, K);
            int zbad = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) zbad |= !(x[q + 4][2] > x[q][2]);
            if (zbad || badg) {
                unsigned long long e = ((unsigned long long)ek * ny + ej) * nx + ei;
                atomicMin(bad, e * 16ull + (zbad ? 0ull : (unsigned long long)badg));
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                x[q][0] = x[q + 4][0];
                x[q][1] = x[q + 4][1];
                x[q][2] = x[q + 4][2];
            }
        } else {
#pragma unroll
            for (int u = 0; u < 36; u++) K[u] = 0.0;
        }
#pragma unroll
        for (int u = 0; u < 36; u++) ke[u * NTH + t] = K[u];
        __syncthreads();
        if (nv) {
            gather_couplings<0>(ke, t, acc);   // node level ek as a bottom node
            const i64 o = loff(L, ni, nj, ek);
#pragma unroll
            for (int s = 0; s < 14; s++) coef[s * L.NT + o] = acc[s];
#pragma unroll
            for (int s = 0; s < 14; s++) acc[s] = 0.0;
            gather_couplings<1>(ke, t, acc);   // node level ek+1 as a top node
        }
        __syncthreads();
    }
    if (nv) {
        const i64 o = loff(L, ni, nj, n3 - 1);
#pragma unroll
        for (int s = 0; s < 14; s++) coef[s * L.NT + o] = acc[s];
    }
}

// ------------------------------------------------------------------ RHS
// f_p = sum_{e ni p} fe_a(p),  fe_a = -8 detJ(0) gradN_a(0).u0_e
//     = -detJ(0) sum_d s_ad (Ji(0) u0_e)_d = -(s_a . h_e),  h_e = detJ(0) Ji(0) u0_e
// (dN_a/dxi_d(0) = s_ad/8).  Per element only the 3-vector h_e is needed: a
// node at local corner (da, db) of the four elements of one element layer
// gets from them -(S - T) as their bottom node and -(S + T) as their top node,
// S = sum_e (s_x hx + s_y hy), T = sum_e hz, s_x = 2 da - 1, s_y = 2 db - 1.
// A CTA computes TX x TY element columns (1-element halo recomputed) upward in
// k; h goes through a double-buffered shared plane, so one barrier per layer.
// Coordinates: the level's local rows; u0 / f: ABI arrays (Nat); f is written
// on the owned rows only, 0 on the Dirichlet set.
constexpr int RTX = 32, RTY = 8, RNTH = RTX * RTY;   // 256 threads: 3 CTAs per SM at 79 registers (RTY = 16: 1 CTA, 3.12 -> 2.46 ms at Paper-scale)
__global__ void __launch_bounds__(RNTH)
rhs_kernel(const double* __restrict__ X, const double* __restrict__ Y,
           const double* __restrict__ Z, LevDev L, Nat u0, Nat f) {
    __shared__ double hs[2][3][RNTH];
    const int n1 = L.n1, n2 = L.n2, n3 = L.n3;
    const int t = threadIdx.x;
    const int tx = t % RTX, ty = t / RTX;
    const int i0 = blockIdx.x * (RTX - 1), j0 = blockIdx.y * (RTY - 1);
    const int ei = i0 - 1 + tx, ej = j0 - 1 + ty;
    const int nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    const bool ev = ei >= 0 && ei < nx && ej >= 0 && ej < ny;
    const int ni = i0 + tx, nj = j0 + ty;
    const bool nv = tx < RTX - 1 && ty < RTY - 1 && ni < n1 && nj >= L.own0 && nj < L.own1;
    const bool ndir = ni == 0 || ni == n1 - 1 || row_dirichlet(L, nj);
    const i64 EC = (i64)nz * u0.n2a * nx;   // one component of the element array
    double* fo = const_cast<double*>(f.p);
    double x[8][3];
    if (ev) load_plane(X, Y, Z, n1, n2, ei, ej, 0, x, 0);
    double top = 0.0;   // contribution to node level ek from element level ek-1
    for (int ek = 0; ek < nz; ek++) {
        double h0 = 0.0, h1 = 0.0, h2 = 0.0;
        if (ev) {
            load_plane(X, Y, Z, n1, n2, ei, ej, ek + 1, x, 1);
            const i64 e = ((i64)ek * u0.n2a + ej + u0.jofs) * nx + ei;
            const double u = __ldg(u0.p + e), w1 = __ldg(u0.p + EC + e), w2 = __ldg(u0.p + 2 * EC + e);
            double Ji[3][3];
            const double det = centre_jacobian(x, Ji);
            h0 = det * (Ji[0][0] * u + Ji[0][1] * w1 + Ji[0][2] * w2);
            h1 = det * (Ji[1][0] * u + Ji[1][1] * w1 + Ji[1][2] * w2);
            h2 = det * (Ji[2][0] * u + Ji[2][1] * w1 + Ji[2][2] * w2);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                x[q][0] = x[q + 4][0];
                x[q][1] = x[q + 4][1];
                x[q][2] = x[q + 4][2];
            }
        }
        double* hb = &hs[ek & 1][0][0];
        hb[t] = h0;
        hb[RNTH + t] = h1;
        hb[2 * RNTH + t] = h2;
        __syncthreads();
        if (nv) {
            // elements (ex, ey) of the node's 2 x 2: threads t + ex + ey RTX;
            // the node is their corner (1 - ex, 1 - ey): s_x = 1 - 2 ex, s_y = 1 - 2 ey
            const int t00 = t, t10 = t + 1, t01 = t + RTX, t11 = t + RTX + 1;
            const double S = (hb[t00] - hb[t10] + hb[t01] - hb[t11]) +
                             (hb[RNTH + t00] + hb[RNTH + t10] - hb[RNTH + t01] - hb[RNTH + t11]);
            const double T = (hb[2 * RNTH + t00] + hb[2 * RNTH + t10]) +
                             (hb[2 * RNTH + t01] + hb[2 * RNTH + t11]);
            fo[((i64)ek * f.n2a + nj + f.jofs) * n1 + ni] = ndir ? 0.0 : top - (S - T);
            top = -(S + T);
        }
    }
    if (nv) fo[((i64)nz * f.n2a + nj + f.jofs) * n1 + ni] = 0.0;   // top plane is Dirichlet
}

// ------------------------------------------------------------------ recovery
// u_e = u0_e + c .* (Ji(0)^T g),  g_d = sum_a lambda_a s_ad / 8
// Owned element rows: local rows [own0, own1) that are element rows of the grid.
__global__ void __launch_bounds__(256)
recover_kernel(const double* __restrict__ X, const double* __restrict__ Y,
               const double* __restrict__ Z, LevDev L, double c0, double c1, double c2,
               Nat lam, Nat u0, Nat u) {
    const int n1 = L.n1, n2 = L.n2, n3 = L.n3;
    const int ei = blockIdx.x * blockDim.x + threadIdx.x;
    const int ej = L.own0 + (int)blockIdx.y;
    const int nx = n1 - 1, nz = n3 - 1;
    if (ei >= nx || ej >= L.own1 || ej + L.jg0 > L.n2g - 2) return;
    const i64 EC = (i64)nz * u0.n2a * nx, EU = (i64)nz * u.n2a * nx;
    double* uo = const_cast<double*>(u.p);
    auto lat = [&](int k, int j, int i) {
        return __ldg(lam.p + ((i64)k * lam.n2a + j + lam.jofs) * n1 + i);
    };
    double x[8][3], l[8];
    load_plane(X, Y, Z, n1, n2, ei, ej, 0, x, 0);
#pragma unroll
    for (int q = 0; q < 4; q++) l[q] = lat(0, ej + (q >> 1), ei + (q & 1));
    for (int ek = 0; ek < nz; ek++) {
        load_plane(X, Y, Z, n1, n2, ei, ej, ek + 1, x, 1);
#pragma unroll
        for (int q = 0; q < 4; q++) l[q + 4] = lat(ek + 1, ej + (q >> 1), ei + (q & 1));
        double Ji[3][3];
        centre_jacobian(x, Ji);
        double g[3];
#pragma unroll
        for (int d = 0; d < 3; d++) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < 8; a++) s = fma(l[a], sgn(a, d), s);
            g[d] = 0.125 * s;
        }
        const i64 e = ((i64)ek * u0.n2a + ej + u0.jofs) * nx + ei;
        const i64 eo = ((i64)ek * u.n2a + ej + u.jofs) * nx + ei;
        const double gx = Ji[0][0] * g[0] + Ji[1][0] * g[1] + Ji[2][0] * g[2];
        const double gy = Ji[0][1] * g[0] + Ji[1][1] * g[1] + Ji[2][1] * g[2];
        const double gz = Ji[0][2] * g[0] + Ji[1][2] * g[1] + Ji[2][2] * g[2];
        const double a0 = __ldg(u0.p + e), a1 = __ldg(u0.p + EC + e), a2 = __ldg(u0.p + 2 * EC + e);
        uo[eo] = fma(c0, gx, a0);
        uo[EU + eo] = fma(c1, gy, a1);
        uo[2 * EU + eo] = fma(c2, gz, a2);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            x[q][0] = x[q + 4][0];
            x[q][1] = x[q + 4][1];
            x[q][2] = x[q + 4][2];
            l[q] = l[q + 4];
        }
    }
}

}  // namespace

void launch_assemble(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                     const double c[3], const LevDev& L, double* coef, unsigned long long* bad,
                     cudaStream_t st, int ty0, int ty1) {
    const size_t smem = sizeof(double) * 36 * NTH;
    cudaFuncSetAttribute(assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int nty = (n2 + TY - 2) / (TY - 1);
    if (ty1 < 0 || ty1 > nty) ty1 = nty;
    if (ty1 <= ty0) return;
    dim3 grid((n1 + TX - 2) / (TX - 1), ty1 - ty0);
    g_launches += 1;
    assemble_kernel<<<grid, NTH, smem, st>>>(X, Y, Z, n1, n2, n3, c[0], c[1], c[2], L, coef, bad, ty0);
}

int assemble_tile_rows(int n2) { return (n2 + TY - 2) / (TY - 1); }
int assemble_rows_needed(int t) { return t * (TY - 1) + TY; }   // node rows [0, .) tile row t reads

void launch_rhs(const double* X, const double* Y, const double* Z, const LevDev& L, Nat u0, Nat f,
                cudaStream_t st) {
    dim3 grid((L.n1 + RTX - 2) / (RTX - 1), (L.n2 + RTY - 2) / (RTY - 1));
    g_launches += 1;
    rhs_kernel<<<grid, RNTH, 0, st>>>(X, Y, Z, L, u0, f);
}

void launch_recover(const double* X, const double* Y, const double* Z, const LevDev& L,
                    const double c[3], Nat lam, Nat u0, Nat u, cudaStream_t st) {
    if (L.own1 <= L.own0) return;
    dim3 grid((L.n1 - 1 + 127) / 128, L.own1 - L.own0);
    g_launches += 1;
    recover_kernel<<<grid, 128, 0, st>>>(X, Y, Z, L, c[0], c[1], c[2], lam, u0, u);
}

}  // namespace wd
