// k_coarse.cu -- coarsest-level direct solve ("the
// coarsest grid problem is solved by a direct method").
//
// Setup: the free block of the coarsest stencil is expanded into a dense SPD
// matrix (natural order of free nodes) and inverted in place on the device by
// blocked Gauss-Jordan elimination without pivoting (SPD), 32x32 blocks,
// three launches per block step.  Per V-cycle: one GEMV with the explicit
// inverse (<= 4096^2 doubles, L2 resident), fused with the gather of the
// free right-hand side and the scatter of the solution.
#include "wd_internal.cuh"

namespace wd {

namespace {

constexpr int BS = 32;

__device__ __forceinline__ void free_rc(const LevDev& L, int r, int& i, int& j, int& k) {
    const int fx = L.n1 - 2, fy = L.n2 - 2;
    i = r % fx + 1;
    j = (r / fx) % fy + 1;
    k = r / (fx * fy);
}

__device__ __forceinline__ int free_row(const LevDev& L, int i, int j, int k) {
    return (k * (L.n2 - 2) + (j - 1)) * (L.n1 - 2) + (i - 1);
}

__global__ void dense_build_kernel(LevDev L, const double* __restrict__ K, double* A, int nf) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nf) return;
    int i, j, k;
    free_rc(L, r, i, j, k);
    for (int dz = -1; dz <= 1; dz++)
        for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++) {
                const int ii = i + dx, jj = j + dy, kk = k + dz;
                if (ii < 1 || ii > L.n1 - 2 || jj < 1 || jj > L.n2 - 2 || kk < 0 || kk > L.n3 - 2)
                    continue;
                const int s = slot_of(dx, dy, dz);
                const double v = s >= 0 ? K[s * L.NT + loff(L, i, j, k)]
                                        : K[(-s) * L.NT + loff(L, ii, jj, kk)];
                A[(i64)r * nf + free_row(L, ii, jj, kk)] = v;
            }
}

// (1) + (2) the diagonal block's inverse Dinv (scalar Gauss-Jordan in shared
//     memory, double-buffered: one barrier and one division per pivot) fused
//     with the row panel A_Kj <- Dinv A_Kj (j outside block K): every CTA
//     inverts the diagonal block itself (identical operations, so identical
//     Dinv) instead of waiting for a separate launch, and the CTA of block K
//     writes Dinv for the column panel
__global__ void gj_rowdiag_kernel(double* A, int n, int k0, int nb, double* Dinv) {
    const int kb = k0 / BS;
    __shared__ double D2[2][BS][BS + 1], S[BS][BS + 1];
    const int r = threadIdx.y, c = threadIdx.x;
    D2[0][r][c] = (r < nb && c < nb) ? A[(i64)(k0 + r) * n + k0 + c] : (r == c ? 1.0 : 0.0);
    const int j = blockIdx.x * BS + c;
    if ((int)blockIdx.x != kb) S[r][c] = (r < nb && j < n) ? A[(i64)(k0 + r) * n + j] : 0.0;
    __syncthreads();
    int b = 0;
    for (int t = 0; t < BS; t++) {
        const double (&Q)[BS][BS + 1] = D2[b];
        const double piv = Q[t][t];
        const double ip = 1.0 / piv;
        const double drt = Q[r][t], dtc = Q[t][c], drc = Q[r][c];
        double v;
        if (r == t && c == t) v = ip;
        else if (r == t) v = dtc * ip;
        else if (c == t) v = -drt * ip;
        else v = drc - drt * (dtc * ip);
        D2[b ^ 1][r][c] = v;
        b ^= 1;
        __syncthreads();
    }
    const double (&D)[BS][BS + 1] = D2[b];
    if ((int)blockIdx.x == kb) {
        Dinv[r * BS + c] = D[r][c];
        return;
    }
    if (r < nb && j < n) {
        double s = 0.0;
        for (int t = 0; t < nb; t++) s = fma(D[r][t], S[t][c], s);
        A[(i64)(k0 + r) * n + j] = s;
    }
}

// (3) trailing update: A_ij -= A_iK A_Kj(new), i, j outside block K.
//     64 x 64 output tiles, 256 threads with 4 x 4 outputs each (register
//     tiling), the K-panel (<= 32 wide) staged in shared memory
constexpr int TT = 64;
__global__ void __launch_bounds__(256)
gj_trail_kernel(double* A, int n, int k0, int nb) {
    __shared__ double Ac[TT][BS + 1], Ar[BS][TT + 1];
    const int tid = threadIdx.x;
    const int i0 = blockIdx.y * TT, j0 = blockIdx.x * TT;
    for (int e = tid; e < TT * BS; e += 256) {
        const int rr = e / BS, cc = e % BS;
        const int i = i0 + rr;
        Ac[rr][cc] = (i < n && cc < nb && (i < k0 || i >= k0 + nb)) ? A[(i64)i * n + k0 + cc] : 0.0;
        const int r2 = e / TT, c2 = e % TT;
        const int j = j0 + c2;
        Ar[r2][c2] = (r2 < nb && j < n) ? A[(i64)(k0 + r2) * n + j] : 0.0;
    }
    __syncthreads();
    const int ty = tid / 16, tx = tid % 16;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0.0;
    for (int t = 0; t < nb; t++) {
        double x[4], y[4];
#pragma unroll
        for (int a = 0; a < 4; a++) x[a] = Ac[ty + 16 * a][t];
#pragma unroll
        for (int b = 0; b < 4; b++) y[b] = Ar[t][tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) acc[a][b] = fma(x[a], y[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int i = i0 + ty + 16 * a;
        if (i >= n || (i >= k0 && i < k0 + nb)) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int j = j0 + tx + 16 * b;
            if (j >= n || (j >= k0 && j < k0 + nb)) continue;
            A[(i64)i * n + j] -= acc[a][b];
        }
    }
}

// (4) column panel: A_iK <- -A_iK Dinv (i outside K), A_KK <- Dinv
__global__ void gj_col_kernel(double* A, int n, int k0, int nb, const double* __restrict__ Dinv) {
    const int kb = k0 / BS;
    __shared__ double D[BS][BS + 1], S[BS][BS + 1];
    const int r = threadIdx.y, c = threadIdx.x;
    const int i = blockIdx.x * BS + r;
    D[r][c] = Dinv[r * BS + c];
    if ((int)blockIdx.x == kb) {
        if (r < nb && c < nb) A[(i64)(k0 + r) * n + k0 + c] = D[r][c];
        return;
    }
    S[r][c] = (i < n && c < nb) ? A[(i64)i * n + k0 + c] : 0.0;
    __syncthreads();
    if (i < n && c < nb) {
        double s = 0.0;
        for (int t = 0; t < nb; t++) s = fma(S[r][t], D[t][c], s);
        A[(i64)i * n + k0 + c] = -s;
    }
}

// x[free r] = sum_c Ainv[r][c] f[free c]
__global__ void __launch_bounds__(256)
coarse_gemv_kernel(LevDev L, const double* __restrict__ Ainv, int nf,
                   const double* __restrict__ f, double* __restrict__ x) {
    extern __shared__ double b[];
    for (int c = threadIdx.x; c < nf; c += 256) {
        int i, j, k;
        free_rc(L, c, i, j, k);
        b[c] = f[loff(L, i, j, k)];
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int rr = 0; rr < 4; rr++) {
        const int r = (blockIdx.x * 8 + w) * 4 + rr;
        if (r >= nf) break;
        const double* row = Ainv + (i64)r * nf;
        double s = 0.0;
        for (int c = l; c < nf; c += 32) s = fma(row[c], b[c], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (l == 0) {
            int i, j, k;
            free_rc(L, r, i, j, k);
            x[loff(L, i, j, k)] = s;
        }
    }
}

}  // namespace

void launch_dense_build(const LevDev& L, const double* coef, double* A, int nf, cudaStream_t st) {
    cudaMemsetAsync(A, 0, sizeof(double) * (size_t)nf * nf, st);
    g_launches += 1;
    dense_build_kernel<<<(nf + 127) / 128, 128, 0, st>>>(L, coef, A, nf);
}

void coarse_prepare(int nf) {
    const size_t smem = sizeof(double) * (size_t)nf;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(coarse_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
}

int gj_invert(double* A, int n, double* Dinv, cudaStream_t st) {
    const int nbk = (n + BS - 1) / BS;
    dim3 blk(BS, BS);
    for (int kb = 0; kb < nbk; kb++) {
        const int k0 = kb * BS, nb = (n - k0) < BS ? (n - k0) : BS;
        g_launches += 3;
        gj_rowdiag_kernel<<<nbk, blk, 0, st>>>(A, n, k0, nb, Dinv);
        const int ntt = (n + TT - 1) / TT;
        gj_trail_kernel<<<dim3(ntt, ntt), 256, 0, st>>>(A, n, k0, nb);
        gj_col_kernel<<<nbk, blk, 0, st>>>(A, n, k0, nb, Dinv);
    }
    return 0;
}

void launch_coarse_gemv(const LevDev& L, const double* Ainv, int nf, const double* f, double* x,
                        cudaStream_t st) {
    const int rows_per_blk = 32;
    const size_t smem = sizeof(double) * (size_t)nf;
    g_launches += 1;
    coarse_gemv_kernel<<<(nf + rows_per_blk - 1) / rows_per_blk, 256, smem, st>>>(L, Ainv, nf, f, x);
}

}  // namespace wd
