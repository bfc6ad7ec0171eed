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
//         = sum_g sum_{d,e} dN_a/dxi_d (detJ_g Ji c Ji^T)_{de} dN_b/dxi_e
// (2x2x2 Gauss, weights 1), sum-factorised: the same integral on
// the same Gauss points with the products regrouped (equal to the Gauss-point
// by Gauss-point accumulation up to rounding).  Returns the first failing
// Gauss point + 1, or 0.
// On the 2x2x2 Gauss points xi_d = +-G every shape derivative factorises,
//   dN_a/dxi_d(g) = (s_ad / 2) prod_{f != d} L(s_af xi_f),  L(t) = (1 + t) / 2,
// with L(+-G) in {p, m}.  Hence K_ab = sum_g sum_{d,e} dN_a/dxi_d M_de dN_b/dxi_e
// (M = detJ Ji c Ji^T per Gauss point) needs, per direction pair, only a few
// one-dimensional contractions of M over the Gauss points:
//   d = e:   T_d[sa][sb] = sum over the two other directions of
//            (sum over xi_d of M_dd) w(sa, .) w(sb, .),
//   d != e:  U_de = M_de contracted with one L factor per direction,
// where w(sigma, i) = L(s_a xi_i) L(s_b xi_i) depends only on the sign class
// sigma of (s_a, s_b): ++ -> L(+)^2, -- -> L(-)^2, mixed -> p m.  Per element:
// 8 x (Jacobian + inverse + M + 10 accumulations) + ~0.6 k FMA for T, U and
// the 36 entries, against 8 x (72 + 108) FMA for v_b = M grad N_b and
// K_ab += grad N_a . v_b.
namespace sf {
constexpr double P = 0.5 * (1.0 + GP), Mn = 0.5 * (1.0 - GP);
// L(s xi), xi = i ? +G : -G, s = +1 (sp = 1) or -1 (sp = 0)
__host__ __device__ constexpr double Ls(int sp, int i) { return (sp == i) ? P : Mn; }
// w(sigma, i): sigma 0 = (+,+), 1 = (-,-), 2 = mixed
__host__ __device__ constexpr double Wc(int sg, int i) {
    return sg == 0 ? Ls(1, i) * Ls(1, i) : sg == 1 ? Ls(0, i) * Ls(0, i) : P * Mn;
}
__host__ __device__ constexpr int bit(int a, int d) { return (a >> d) & 1; }
__host__ __device__ constexpr int cls(int a, int b, int d) {
    return bit(a, d) == bit(b, d) ? (bit(a, d) ? 0 : 1) : 2;
}
__host__ __device__ constexpr double sg(int a, int d) { return bit(a, d) ? 1.0 : -1.0; }
}  // namespace sf

__device__ __forceinline__ int element_stiffness_sf(const double (&x)[8][3], double c0, double c1,
                                                    double c2, double (&K)[36]) {
    using namespace sf;
    int badg = 0;
    // accumulators over the Gauss points
    double S0[2][2], S1[2][2], S2[2][2];   // sum over xi_d of M_dd, indexed by the other two
    double V01[2][2][2], V02[2][2][2];     // [beta(xi0)][i1][i2]
    double V12[3][2][2];                   // [sigma(xi0)][i1][i2]
#pragma unroll
    for (int u = 0; u < 2; u++)
#pragma unroll
        for (int v = 0; v < 2; v++) {
            S0[u][v] = S1[u][v] = S2[u][v] = 0.0;
#pragma unroll
            for (int q = 0; q < 2; q++) V01[q][u][v] = V02[q][u][v] = 0.0;
#pragma unroll
            for (int q = 0; q < 3; q++) V12[q][u][v] = 0.0;
        }
#pragma unroll
    for (int g = 0; g < 8; g++) {
        const int i0 = g & 1, i1 = (g >> 1) & 1, i2 = (g >> 2) & 1;
        const double x0 = i0 ? GP : -GP, x1 = i1 ? GP : -GP, x2 = i2 ? GP : -GP;
        double Ji[3][3];
        const double det = jac_inv(x, x0, x1, x2, Ji);
        if (!(det > 0.0) && badg == 0) badg = g + 1;
        double M[3][3];
#pragma unroll
        for (int d = 0; d < 3; d++)
#pragma unroll
            for (int e = d; e < 3; e++) {
                double t = c0 * Ji[d][0] * Ji[e][0];
                t = fma(c1 * Ji[d][1], Ji[e][1], t);
                t = fma(c2 * Ji[d][2], Ji[e][2], t);
                M[d][e] = det * t;
            }
        S0[i1][i2] += M[0][0];
        S1[i0][i2] += M[1][1];
        S2[i0][i1] += M[2][2];
#pragma unroll
        for (int q = 0; q < 2; q++) {
            V01[q][i1][i2] = fma(M[0][1], Ls(q, i0), V01[q][i1][i2]);
            V02[q][i1][i2] = fma(M[0][2], Ls(q, i0), V02[q][i1][i2]);
        }
#pragma unroll
        for (int q = 0; q < 3; q++) V12[q][i1][i2] = fma(M[1][2], Wc(q, i0), V12[q][i1][i2]);
    }
    // one-dimensional contractions over the remaining directions
    double T0[3][3], T1[3][3], T2[3][3];   // [sigma of the lower other dir][sigma of the upper]
#pragma unroll
    for (int p = 0; p < 3; p++)
#pragma unroll
        for (int q = 0; q < 3; q++) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
            for (int u = 0; u < 2; u++)
#pragma unroll
                for (int v = 0; v < 2; v++) {
                    const double w = Wc(p, u) * Wc(q, v);
                    t0 = fma(S0[u][v], w, t0);
                    t1 = fma(S1[u][v], w, t1);
                    t2 = fma(S2[u][v], w, t2);
                }
            T0[p][q] = t0;
            T1[p][q] = t1;
            T2[p][q] = t2;
        }
    double U01[2][2][3], U02[2][2][3], U12[3][2][2];
#pragma unroll
    for (int b0 = 0; b0 < 2; b0++)
#pragma unroll
        for (int a1 = 0; a1 < 2; a1++)
#pragma unroll
            for (int q = 0; q < 3; q++) {
                double u01 = 0.0, u02 = 0.0;
#pragma unroll
                for (int u = 0; u < 2; u++)
#pragma unroll
                    for (int v = 0; v < 2; v++) {
                        // U01[b0][a1][s2]: L(a1, i1) w(s2, i2);  U02[b0][a2][s1]: w(s1, i1) L(a2, i2)
                        u01 = fma(V01[b0][u][v], Ls(a1, u) * Wc(q, v), u01);
                        u02 = fma(V02[b0][u][v], Wc(q, u) * Ls(a1, v), u02);
                    }
                U01[b0][a1][q] = u01;
                U02[b0][a1][q] = u02;
            }
#pragma unroll
    for (int q = 0; q < 3; q++)
#pragma unroll
        for (int b1 = 0; b1 < 2; b1++)
#pragma unroll
            for (int a2 = 0; a2 < 2; a2++) {
                double u12 = 0.0;
#pragma unroll
                for (int u = 0; u < 2; u++)
#pragma unroll
                    for (int v = 0; v < 2; v++)
                        u12 = fma(V12[q][u][v], Ls(b1, u) * Ls(a2, v), u12);
                U12[q][b1][a2] = u12;
            }
    // the 36 upper-triangle entries
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = a; b < 8; b++) {
            const int s0 = cls(a, b, 0), s1 = cls(a, b, 1), s2 = cls(a, b, 2);
            double k = 0.25 * sg(a, 0) * sg(b, 0) * T0[s1][s2];
            k = fma(0.25 * sg(a, 1) * sg(b, 1), T1[s0][s2], k);
            k = fma(0.25 * sg(a, 2) * sg(b, 2), T2[s0][s1], k);
            // (0,1): (s_a0 s_b1/4) U01[b0 of b][a1 of a][s2] + (s_a1 s_b0/4) U01[b0 of a][a1 of b][s2]
            k = fma(0.25 * sg(a, 0) * sg(b, 1), U01[bit(b, 0)][bit(a, 1)][s2], k);
            k = fma(0.25 * sg(a, 1) * sg(b, 0), U01[bit(a, 0)][bit(b, 1)][s2], k);
            // (0,2): (s_a0 s_b2/4) U02[bit b0][bit a2][s1] + (s_a2 s_b0/4) U02[bit a0][bit b2][s1]
            k = fma(0.25 * sg(a, 0) * sg(b, 2), U02[bit(b, 0)][bit(a, 2)][s1], k);
            k = fma(0.25 * sg(a, 2) * sg(b, 0), U02[bit(a, 0)][bit(b, 2)][s1], k);
            // (1,2): (s_a1 s_b2/4) U12[s0][bit b1][bit a2] + (s_a2 s_b1/4) U12[s0][bit a1][bit b2]
            k = fma(0.25 * sg(a, 1) * sg(b, 2), U12[s0][bit(b, 1)][bit(a, 2)], k);
            k = fma(0.25 * sg(a, 2) * sg(b, 1), U12[s0][bit(a, 1)][bit(b, 2)], k);
            K[ut(a, b)] = k;
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
            int badg = element_stiffness_sf(x, c0, c1, c2, K);
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
