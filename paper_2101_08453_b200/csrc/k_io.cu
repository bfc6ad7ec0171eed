// k_io.cu -- the steps either side of the solver:
//
//   build_mesh_kernel   terrain-following mesh from a terrain array (P:37-38,
//                       reading C13 of DESIGN.md):
//                         X = x0 + i dx, Y = y0 + j dy,
//                         Z = zs + zeta_k (H - zs) / zeta_{n3-1};
//   interp_wind_kernel  coarse (WRF-like) wind to element centres:
//                       trilinear in (x, y, height above ground), clamped;
//   free_norms_kernel   l2 / max-abs block partials of a natural-layout node
//                       vector over the owned free nodes (mass-consistency
//                       diagnostics of Eq. (1), reading C12).
// All are single-pass HBM streams (one thread per column / element / node).
#include "wd_internal.cuh"

namespace wd {

namespace {

__global__ void __launch_bounds__(128)
build_mesh_kernel(const double* __restrict__ zs, int n1, int n2, int n3, double x0, double y0,
                  double dx, double dy, const double* __restrict__ zeta, double H, double* X,
                  double* Y, double* Z, unsigned long long* bad) {
    const int i = blockIdx.x * 128 + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= n1) return;
    const i64 col = (i64)j * n1 + i;
    const double z = zs[col];
    if (!(H > z)) atomicMin(bad, (unsigned long long)col);
    const double T = zeta[n3 - 1];
    const double x = x0 + i * dx, y = y0 + j * dy;
    const i64 plane = (i64)n1 * n2;
    for (int k = 0; k < n3; k++) {
        const i64 p = (i64)k * plane + col;
        X[p] = x;
        Y[p] = y;
        Z[p] = z + zeta[k] * (H - z) / T;
    }
}

// index-space bracket of t in [0, n-1]: lower index i0 in [0, n-2], weight of i0+1
__device__ __forceinline__ void bracket(double t, int n, int& i0, double& w) {
    if (t <= 0.0) { i0 = 0; w = 0.0; return; }
    if (t >= n - 1) { i0 = n - 2; w = 1.0; return; }
    int a = (int)floor(t);
    if (a > n - 2) a = n - 2;
    i0 = a;
    w = t - a;
}

__global__ void __launch_bounds__(128)
interp_wind_kernel(const double* __restrict__ uc, int nxc, int nyc, int nzc, double xc0,
                   double yc0, double DXc, double DYc, const double* __restrict__ hc,
                   const double* __restrict__ X, const double* __restrict__ Y,
                   const double* __restrict__ Z, int n1, int n2, int n3, double* __restrict__ u0) {
    const int i = blockIdx.x * 128 + threadIdx.x;
    const int j = blockIdx.y, k = blockIdx.z;
    const int nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    if (i >= nx) return;
    const i64 plane = (i64)n1 * n2;
    double xe = 0, ye = 0, ze = 0, zb = 0;
    for (int c = 0; c < 2; c++)
        for (int b = 0; b < 2; b++)
            for (int a = 0; a < 2; a++) {
                const i64 p = (i64)(k + c) * plane + (i64)(j + b) * n1 + i + a;
                xe += X[p];
                ye += Y[p];
                ze += Z[p];
            }
    for (int b = 0; b < 2; b++)
        for (int a = 0; a < 2; a++) zb += Z[(i64)(j + b) * n1 + i + a];
    xe /= 8.0;
    ye /= 8.0;
    ze /= 8.0;
    zb /= 4.0;
    const double he = ze - zb;
    int ia, ib, ic;
    double wa, wb, wc;
    bracket((xe - xc0) / DXc, nxc, ia, wa);
    bracket((ye - yc0) / DYc, nyc, ib, wb);
    if (he <= hc[0]) { ic = 0; wc = 0.0; }
    else if (he >= hc[nzc - 1]) { ic = nzc - 2; wc = 1.0; }
    else {
        ic = 0;
        while (ic < nzc - 2 && he >= hc[ic + 1]) ic++;
        wc = (he - hc[ic]) / (hc[ic + 1] - hc[ic]);
    }
    const i64 ne = (i64)nx * ny * nz;
    const i64 e = ((i64)k * ny + j) * nx + i;
    for (int m = 0; m < 3; m++) {
        double v = 0.0;
        for (int c = 0; c < 2; c++)
            for (int b = 0; b < 2; b++)
                for (int a = 0; a < 2; a++) {
                    const double w = (a ? wa : 1 - wa) * (b ? wb : 1 - wb) * (c ? wc : 1 - wc);
                    v = fma(w, uc[(((i64)m * nzc + ic + c) * nyc + ib + b) * nxc + ia + a], v);
                }
        u0[m * ne + e] = v;
    }
}

// per-block (sum of squares, max abs) over owned free nodes of a natural-layout
// node vector v (rows of the part: v[(k n2 + j) n1 + i], j local)
__global__ void __launch_bounds__(256)
free_norms_kernel(LevDev L, const double* __restrict__ v, double* partial) {
    __shared__ double s2[256], sm[256];
    const int t = threadIdx.x;
    const i64 nrow = (i64)(L.own1 - L.own0);
    const i64 n = (i64)(L.n1 - 2) * nrow * (L.n3 - 1);
    double a2 = 0.0, am = 0.0;
    for (i64 q = (i64)blockIdx.x * 256 + t; q < n; q += (i64)gridDim.x * 256) {
        const int i = 1 + (int)(q % (L.n1 - 2));
        const i64 r = q / (L.n1 - 2);
        const int j = L.own0 + (int)(r % nrow);
        const int k = (int)(r / nrow);
        if (!row_free(L, j)) continue;
        const double x = v[((i64)k * L.n2 + j) * L.n1 + i];
        a2 = fma(x, x, a2);
        am = fmax(am, fabs(x));
    }
    s2[t] = a2;
    sm[t] = am;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (t < o) {
            s2[t] += s2[t + o];
            sm[t] = fmax(sm[t], sm[t + o]);
        }
        __syncthreads();
    }
    if (t == 0) {
        partial[2 * blockIdx.x] = s2[0];
        partial[2 * blockIdx.x + 1] = sm[0];
    }
}

__global__ void norms_final_kernel(const double* partial, int nb, double* out) {
    double s = 0.0, m = 0.0;
    for (int b = 0; b < nb; b++) {
        s += partial[2 * b];
        m = fmax(m, partial[2 * b + 1]);
    }
    out[0] = s;
    out[1] = m;
}

}  // namespace

void launch_build_mesh(const double* zs, int n1, int n2, int n3, double x0, double y0, double dx,
                       double dy, const double* zeta, double H, double* X, double* Y, double* Z,
                       unsigned long long* bad, cudaStream_t st) {
    g_launches += 1;
    build_mesh_kernel<<<dim3((n1 + 127) / 128, n2), 128, 0, st>>>(zs, n1, n2, n3, x0, y0, dx, dy,
                                                                  zeta, H, X, Y, Z, bad);
}

void launch_interp_wind(const double* uc, int nxc, int nyc, int nzc, double xc0, double yc0,
                        double DXc, double DYc, const double* hc, const double* X,
                        const double* Y, const double* Z, int n1, int n2, int n3, double* u0,
                        cudaStream_t st) {
    g_launches += 1;
    interp_wind_kernel<<<dim3((n1 - 1 + 127) / 128, n2 - 1, n3 - 1), 128, 0, st>>>(
        uc, nxc, nyc, nzc, xc0, yc0, DXc, DYc, hc, X, Y, Z, n1, n2, n3, u0);
}

// out[0] = sum of squares, out[1] = max abs over owned free nodes (deterministic)
void launch_free_norms(const LevDev& L, const double* v, double* partial, int nb, double* out,
                       cudaStream_t st) {
    g_launches += 2;
    free_norms_kernel<<<nb, 256, 0, st>>>(L, v, partial);
    norms_final_kernel<<<1, 1, 0, st>>>(partial, nb, out);
}

}  // namespace wd
