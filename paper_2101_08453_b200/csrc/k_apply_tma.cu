// k_apply_tma.cu -- residual / 27-point operator apply with TMA-staged (i,j)
// tiles and vertical streaming over k (sm_100a).
//
//   r = f - K x   (Eq. (7) residual; the convergence test of S:198)  or  y = K x
//
// A persistent CTA walks over tiles of 32 half-row positions x 2 parities x
// 4 rows (256 node columns, one thread each) and, inside a tile, upward over
// the levels k.  For every level one elected thread issues
// cp.async.bulk.tensor loads (TMA) into shared-memory rings, D = 2 levels
// ahead of the consumers, completing on mbarriers:
//   A-ring: coefficient slots 0..4 (diagonal + the dz = 0 forward couplings)
//           for rows j0-1 .. j0+3, positions a0-2 .. a0+33, plus f of the tile;
//   B-ring: slots 5..13 (the dz = 1 couplings) for rows j0-1 .. j0+4;
//   X-ring: x for rows j0-1 .. j0+4.
// Every stored coupling is then read from HBM once per tile (halo rows and
// columns are shared with the neighbouring tiles through L2) and the
// backward couplings K(p, p-d) = K_d[p-d] (symmetric 14-coefficient storage)
// come from shared memory.  Out-of-grid box elements are zero-filled by TMA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "wd_internal.cuh"

#include <cstdlib>

namespace wd {

int g_tma_debug = 0;   // development knob (env WD_TMA_DEBUG): bit mask of disabled TMA rings

namespace {

constexpr int TI = 32;           // half-row positions per tile
constexpr int TJ = 4;            // rows per tile
constexpr int BP = TI + 4;       // box positions: 2 before (16-byte aligned start), 2 after
constexpr int NTHR = TI * 2 * TJ;
constexpr int D = 2;             // prefetch depth (levels)
constexpr int RA = D + 1, RB = D + 2, RX = D + 4;
constexpr int A_ROWS = TJ + 1, B_ROWS = TJ + 2, X_ROWS = TJ + 2;
constexpr int pad128(int n) { return (n + 15) / 16 * 16; }   // doubles -> 128 B multiple
// TMA destinations must be 128-byte aligned: every buffer is padded
constexpr unsigned A_BYTES = 5 * A_ROWS * 2 * BP * 8, F_BYTES = TJ * 2 * TI * 8,
                   B_BYTES = 9 * B_ROWS * 2 * BP * 8, X_BYTES = X_ROWS * 2 * BP * 8;
constexpr int A_ELEMS = pad128(5 * A_ROWS * 2 * BP);
constexpr int F_ELEMS = pad128(TJ * 2 * TI);
constexpr int B_ELEMS = pad128(9 * B_ROWS * 2 * BP);
constexpr int X_ELEMS = pad128(X_ROWS * 2 * BP);
constexpr size_t SMEM = (size_t)8 * (RA * (A_ELEMS + F_ELEMS) + RB * B_ELEMS + RX * X_ELEMS) +
                        2 * 8 * (RA + RB + RX) + 8 * 8 + 256;

__device__ __forceinline__ uint32_t sa(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}

__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(sa(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma5(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                     int c4, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(sa(bar))
        : "memory");
}

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                     uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sa(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(bar))
        : "memory");
}

struct Tiles {
    int ntx, nty, ntiles, nk;   // tiles along positions / rows; levels per tile (n3-1)
};

// issue the loads of level k of tile t (A+f and B units) and of x-unit kk
__device__ __forceinline__ void load_AB(const CUtensorMap* mA, const CUtensorMap* mB,
                                        const CUtensorMap* mF, double* a, double* fbuf, double* b,
                                        uint64_t* barA, uint64_t* barB, int a0, int j0, int k,
                                        bool with_f, int dbg) {
    const bool ea = !(dbg & 1), eb = !(dbg & 2), ef = with_f && !(dbg & 8);
    mbar_expect(barA, (ea ? A_BYTES : 0) + (ef ? F_BYTES : 0));
    const int c0 = a0 > 0 ? a0 - 2 : 0, c2 = j0 > 0 ? j0 - 1 : 0;   // halo box origin (>= 0, even)
    if (ea) tma5(a, mA, c0, 0, c2, k, 0, barA);
    if (ef) tma4(fbuf, mF, a0, 0, j0, k, barA);
    mbar_expect(barB, eb ? B_BYTES : 0);
    if (eb) tma5(b, mB, c0, 0, c2, k, 5, barB);
}

__device__ __forceinline__ void load_X(const CUtensorMap* mX, double* x, uint64_t* bar, int a0,
                                       int j0, int k, int dbg) {
    mbar_expect(bar, (dbg & 4) ? 0 : X_BYTES);
    if (!(dbg & 4)) tma4(x, mX, a0 > 0 ? a0 - 2 : 0, 0, j0 > 0 ? j0 - 1 : 0, k, bar);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}

// Warp-specialised: warps 0..7 compute (one node column each), warp 8 is the
// TMA producer.  full[] barriers complete when a unit's bytes have landed;
// empty[] barriers (8 arrivals, one per consumer warp) release a slot.
__global__ void __launch_bounds__(NTHR + 32, 1)
apply_tma_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                 const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mF,
                 LevDev L, Tiles T, int with_f, int dbg, int jitter, double* __restrict__ y,
                 double* __restrict__ partial) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((128 - (sa(smem_raw) & 127)) & 127);
    double* sA = reinterpret_cast<double*>(smem);
    double* sF = sA + RA * A_ELEMS;
    double* sB = sF + RA * F_ELEMS;
    double* sX = sB + RB * B_ELEMS;
    uint64_t* fA = reinterpret_cast<uint64_t*>(sX + RX * X_ELEMS);
    uint64_t* fB = fA + RA;
    uint64_t* fX = fB + RB;
    uint64_t* eA = fX + RX;
    uint64_t* eB = eA + RA;
    uint64_t* eX = eB + RB;
    double* ws = reinterpret_cast<double*>(eX + RX);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int NCW = NTHR / 32;   // consumer warps
    if (tid == 0) {
        for (int t = 0; t < RA; t++) { mbar_init(&fA[t], 1); mbar_init(&eA[t], NCW); }
        for (int t = 0; t < RB; t++) { mbar_init(&fB[t], 1); mbar_init(&eB[t], NCW); }
        for (int t = 0; t < RX; t++) { mbar_init(&fX[t], 1); mbar_init(&eX[t], NCW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int nk = T.nk;                  // levels per tile: 0 .. n3-2
    const int my_tiles = (T.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int nsteps = my_tiles * nk;
    auto tile_of = [&](int it, int& a0, int& j0) {
        const int t = (int)blockIdx.x + it * (int)gridDim.x;
        a0 = (t % T.ntx) * TI;
        j0 = L.own0 + (t / T.ntx) * TJ;   // tiles cover the owned local rows
    };

    if (warp == NCW) {
        // ---------------- producer: units in consumption order, gated by empty[]
        if (lane == 0) {
            for (int s = 0; s < nsteps; s++) {
                const int it = s / nk, k = s % nk;
                int a0, j0;
                tile_of(it, a0, j0);
                mbar_wait(&eA[s % RA], ((s / RA) & 1) ^ 1);
                mbar_wait(&eB[s % RB], ((s / RB) & 1) ^ 1);
                load_AB(&mA, &mB, &mF, sA + (s % RA) * A_ELEMS, sF + (s % RA) * F_ELEMS,
                        sB + (s % RB) * B_ELEMS, &fA[s % RA], &fB[s % RB], a0, j0, k, with_f != 0,
                        dbg);
                const int xu = it * (nk + 1) + k;
                for (int u = (k == 0 ? xu : xu + 1); u <= xu + 1; u++) {
                    mbar_wait(&eX[u % RX], ((u / RX) & 1) ^ 1);
                    load_X(&mX, sX + (u % RX) * X_ELEMS, &fX[u % RX], a0, j0, u - it * (nk + 1), dbg);
                }
            }
        }
        __syncthreads();
        return;
    }

    // ---------------- consumers
    const int tx = lane, ci = warp & 1, tz = warp >> 1;
    const int hp = 1 - ci;
    double acc = 0.0;
    double xm[9], x0[9], xp[9];

    for (int s = 0; s < nsteps; s++) {
        if (jitter) {   // race stress test (tests only, env WD_TEST_JITTER)
            unsigned h = (unsigned)(blockIdx.x * 977u + warp * 131u + s * 7919u);
            h ^= h >> 13;
            h *= 0x5bd1e995u;
            h ^= h >> 15;
            __nanosleep(h % (unsigned)jitter);
        }
        const int it = s / nk, k = s % nk;
        int a0, j0;
        tile_of(it, a0, j0);
        const int xu = it * (nk + 1) + k;         // X unit of level k
        mbar_wait(&fA[s % RA], (s / RA) & 1);
        mbar_wait(&fB[s % RB], (s / RB) & 1);
        mbar_wait(&fX[(xu + 1) % RX], ((xu + 1) / RX) & 1);
        if (k == 0) mbar_wait(&fX[xu % RX], (xu / RX) & 1);
        const double* A = sA + (s % RA) * A_ELEMS;
        const double* Fb = sF + (s % RA) * F_ELEMS;
        const double* B = sB + (s % RB) * B_ELEMS;
        const double* Bm = sB + ((s + RB - 1) % RB) * B_ELEMS;   // level k-1 (same tile if k > 0)
        // The halo boxes start two positions / one row before the tile, except
        // at the grid edge (a0 = 0 / j0 = 0) where they start at the tile: the
        // missing halo there only concerns the Dirichlet column i = 0 / row
        // j = 0 (never computed).
        const int p = tx + (a0 > 0 ? 2 : 0);      // own position in a box row
        const int rr = tz + (j0 > 0 ? 1 : 0);     // own row in a box
        const int pm = p - 1 + ci, pp = p + ci;   // positions of i-1 and i+1 (half hp)
        const int i = 2 * (a0 + tx) + ci, j = j0 + tz;
        const bool valid = i >= 1 && i <= L.n1 - 2 && row_free(L, j);
        // x window (box rows rr-1..rr+1 = j-1..j+1)
        auto xat = [&](const double* X, int r, int c) -> double {
            const int ox = c % 3 - 1;
            const int h = ox ? hp : ci;
            const int q = ox < 0 ? pm : (ox > 0 ? pp : p);
            return X[((r) * 2 + h) * BP + q];
        };
        const double* Xk1 = sX + ((xu + 1) % RX) * X_ELEMS;
        if (k == 0) {
            const double* Xk = sX + (xu % RX) * X_ELEMS;
#pragma unroll
            for (int c = 0; c < 9; c++) {
                xm[c] = 0.0;
                x0[c] = valid ? xat(Xk, rr - 1 + c / 3, c) : 0.0;
            }
        }
#pragma unroll
        for (int c = 0; c < 9; c++) xp[c] = valid ? xat(Xk1, rr - 1 + c / 3, c) : 0.0;

        if (valid) {
            // element (slot, box row, half, position)
            auto a_at = [&](int sl, int r, int h, int q) { return A[((sl * A_ROWS + r) * 2 + h) * BP + q]; };
            auto b_at = [&](const double* Bx, int sl, int r, int h, int q) {
                return Bx[(((sl - 5) * B_ROWS + r) * 2 + h) * BP + q];
            };
            // four independent partial sums (ILP), combined in a fixed order
            double s0 = a_at(0, rr, ci, p) * x0[4], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int sl = 1; sl < 14; sl++) {
                const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
                const int cf = (dx + 1) + 3 * (dy + 1);     // forward neighbour column
                const int cb = (-dx + 1) + 3 * (-dy + 1);   // backward neighbour column
                const int hb = dx ? hp : ci;
                const int qb = dx > 0 ? pm : (dx < 0 ? pp : p);   // position of i - dx
                if (!dz) {
                    s0 = fma(a_at(sl, rr, ci, p), x0[cf], s0);
                    s1 = fma(a_at(sl, rr - dy, hb, qb), x0[cb], s1);
                } else {
                    s2 = fma(b_at(B, sl, rr, ci, p), xp[cf], s2);
                    if (k > 0) s3 = fma(b_at(Bm, sl, rr - dy, hb, qb), xm[cb], s3);
                }
            }
            const double s_ = (s0 + s1) + (s2 + s3);
            const double v = with_f ? Fb[(tz * 2 + ci) * TI + tx] - s_ : s_;
            y[loff(L, i, j, k)] = v;
            acc = fma(v, v, acc);
        }
#pragma unroll
        for (int c = 0; c < 9; c++) {
            xm[c] = x0[c];
            x0[c] = xp[c];
        }
        // release this step's slots (B of level k-1 now, B of level k after
        // the next level, or now at the tile's last level)
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&eA[s % RA]);
            mbar_arrive(&eX[(xu + 1) % RX]);
            if (k == 0) mbar_arrive(&eX[xu % RX]);
            if (k > 0) mbar_arrive(&eB[(s + RB - 1) % RB]);
            if (k == nk - 1) mbar_arrive(&eB[s % RB]);
        }
    }
    __syncthreads();
    if (partial) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (lane == 0) ws[warp] = acc;
        asm volatile("bar.sync 1, %0;" ::"n"(NTHR));   // consumer warps only
        if (tid == 0) {
            double r = 0.0;
            for (int w = 0; w < NCW; w++) r += ws[w];
            partial[blockIdx.x] = r;
        }
    }
}

// L2 promotion of the residual's TMA boxes (env WD_APPLY_L2PROMO 0..3 = none,
// 64, 128, 256 B; default 256 B)
CUtensorMapL2promotion apply_promo() {
    static const CUtensorMapL2promotion promo[4] = {
        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    int pr = 3;
    if (const char* e = getenv("WD_APPLY_L2PROMO")) pr = atoi(e) & 3;
    return promo[pr];
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int grid_size() {
    static int g = 0;
    if (!g) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g = sms;
    }
    return g;
}

}  // namespace

// coefficient maps: [14][n3][n2][2][H] as a 5-D tensor (pos, half, row, level, slot)
int make_coef_maps(const LevDev& L, const double* coef, void* mapA, void* mapB) {
    auto enc = encode_fn();
    if (!enc) return -1;
    cuuint64_t dims[5] = {(cuuint64_t)L.H, 2, (cuuint64_t)L.n2, (cuuint64_t)L.n3, 14};
    cuuint64_t str[4] = {(cuuint64_t)L.H * 8, (cuuint64_t)L.sj * 8, (cuuint64_t)L.sk * 8,
                         (cuuint64_t)L.NT * 8};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    cuuint32_t boxA[5] = {BP, 2, A_ROWS, 1, 5};
    cuuint32_t boxB[5] = {BP, 2, B_ROWS, 1, 9};
    CUresult r1 = enc((CUtensorMap*)mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)coef, dims,
                      str, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      apply_promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc((CUtensorMap*)mapB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)coef, dims,
                      str, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      apply_promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return (r1 == CUDA_SUCCESS && r2 == CUDA_SUCCESS) ? 0 : -1;
}

// vector maps: [n3][n2][2][H] (pos, half, row, level); halo box (x) or tile box (f).
// TMA box starts must be 16-byte aligned in the innermost dimension (an odd
// double offset raised "illegal instruction" on B200): the halo boxes start 2
// positions before the tile (clamped to 0 at the grid edge).
int make_vec_map(const LevDev& L, const double* v, void* map, bool halo) {
    auto enc = encode_fn();
    if (!enc) return -1;
    cuuint64_t dims[4] = {(cuuint64_t)L.H, 2, (cuuint64_t)L.n2, (cuuint64_t)L.n3};
    cuuint64_t str[3] = {(cuuint64_t)L.H * 8, (cuuint64_t)L.sj * 8, (cuuint64_t)L.sk * 8};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint32_t boxX[4] = {BP, 2, X_ROWS, 1};
    cuuint32_t boxF[4] = {TI, 2, TJ, 1};
    CUresult r = enc((CUtensorMap*)map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)v, dims, str,
                     halo ? boxX : boxF, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, apply_promo(),
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -1;
}

void apply_tma_prepare() {
    cudaFuncSetAttribute(apply_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
}

// r = f - K x (mapF != NULL) or y = K x; partial (nullable) gets one value per CTA.
// Returns the number of partials written.
int launch_apply_tma(const LevDev& L, const void* mapA, const void* mapB, const void* mapX,
                     const void* mapF, double* y, double* partial, cudaStream_t st) {
    Tiles T;
    T.ntx = ((L.n1 + 1) / 2 + TI - 1) / TI;
    T.nty = (L.own1 - L.own0 + TJ - 1) / TJ;
    T.ntiles = T.ntx * T.nty;
    T.nk = L.n3 - 1;
    int g = grid_size();
    if (g > T.ntiles) g = T.ntiles;
    const CUtensorMap* F = (const CUtensorMap*)(mapF ? mapF : mapX);
    g_launches += 1;
    if (g_test_gs_grid > 0 && g > g_test_gs_grid) g = g_test_gs_grid;
    apply_tma_kernel<<<g, NTHR + 32, SMEM, st>>>(
        *(const CUtensorMap*)mapA, *(const CUtensorMap*)mapB, *(const CUtensorMap*)mapX, *F, L, T,
        mapF ? 1 : 0, g_tma_debug, g_test_jitter, y, partial);
    return g;
}

}  // namespace wd
