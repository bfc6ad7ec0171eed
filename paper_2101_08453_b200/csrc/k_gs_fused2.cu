// k_gs_fused2.cu -- the one-pass four-colour sweep of k_gs_fused.cu with a
// leaner instruction stream (same schedule, same floating-point operations in
// the same order, hence bitwise equal to it and to the phased schedule).
//
// Smoother: "vertical sweeps of Gauss-Seidel from the bottom up to
// the top, with red-black ordering horizontally into 4 groups", colours
// (i mod 2, j mod 2) = (0,0),(1,0),(0,1),(1,1) (reading C7).  The schedule
// (64 x 8 tiles with a recomputed halo, colour c at virtual plane s - 2c at
// step s, persistent CTAs with the k-pipeline running across tiles, lambda in
// a 12-plane shared-memory ring, the 27 couplings of the next node in
// registers one step ahead) is described in k_gs_fused.cu.
//
// Measured there (ncu source counters, Paper-scale level 0): ~440 warp
// instructions per node update, 52 % of them integer address arithmetic, the
// SM issue slots half busy and 35 % of the warp samples waiting at the
// per-step barrier -- the step is as long as the slowest warp's instruction
// stream plus the exposed coupling-load latency.  This version cuts the
// instruction stream:
//   * the lambda ring is filled by the tensor-memory accelerator: one
//     cp.async.bulk.tensor per plane (box 36 positions x 2 halves x 11 rows,
//     out-of-grid entries zero-filled), issued by one thread LA planes ahead,
//     completing on one mbarrier per ring slot -- instead of ~50 instructions
//     per thread and step of per-pair cp.async address arithmetic;
//   * coupling addresses: the 28 per-slot base pointers (slot plane, row and
//     plane shift of the backward neighbour) are kernel parameters, so a load
//     is one 32-bit node offset (+ the thread's x shift) scaled onto a base
//     instead of a 64-bit multiply-add chain per load;
//   * ring addressing: plane slots advance incrementally (no modulo per step).
// The residual variant runs 64 x 6 tiles, the plain sweep on small levels 64 x 4
// (Geo<TJ_RES>, Geo<TJ_SMALL>; see TJ_SWEEP below).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "wd_internal.cuh"

#include <algorithm>
#include <cstdlib>
#include <atomic>

namespace wd {

namespace {

constexpr int HI = 32;              // positions per parity per tile row (TI = 64 columns)
constexpr int TI = 2 * HI;
constexpr int SW = HI + 4;          // ring positions per parity per row (columns I0-4 .. I0+TI+3)
constexpr int RW = 2 * SW;          // ring doubles per row
constexpr int RING = 12;            // planes in the ring (>= LA + 8: colour 3 reads plane s-7)
constexpr int RING_PRO = 13, LA_PRO = 5;   // PRO: one more plane in flight (see below)
constexpr int LAG = 2;              // plane lag between consecutive colours
constexpr int LA = 4;               // lambda planes loaded ahead
constexpr int SHADOW = 8;
// PRO (fused prolongation): coarse region under a tile (<= CXM x CYM per
// plane, two planes), the ring-column / ring-row parent tables and the coarse
// origin of two tiles
constexpr int CXM = 40, CYM = 8, CPL = CXM * CYM;
static_assert(RING >= LA + 8, "ring too short");

}  // namespace

// geometry of a tile of TI x TJ columns (TJ even)
template <int TJ_>
struct Geo {
    static constexpr int TJ = TJ_;
    static constexpr int SH = TJ + 3;          // ring rows J0-1 .. J0+TJ+1
    static constexpr int PLD = RW * SH;        // doubles of one TMA box (one plane of the ring)
    static constexpr int PL = (PLD + 15) / 16 * 16;   // ring plane pitch (128-byte aligned)
    static constexpr unsigned BOX_BYTES = PLD * 8;
    // colour regions: rows per colour (B) and halo columns beyond the 32 aligned ones
    static constexpr int B0 = TJ / 2 + 1, B1 = TJ / 2 + 1, B2 = TJ / 2, B3 = TJ / 2;
    static constexpr int W0 = B0, W1 = W0 + B1, W2 = W1 + B2, W3 = W2 + B3;   // warp ranges
    static constexpr int NHALO = 3 * B0 + 2 * B1 + B2;       // 29 halo columns at TJ = 8
    static constexpr int PRODUCER = 32 * (W3 + 1);           // first thread of the TMA warp
    static constexpr int THREADS = 32 * (W3 + 2);   // colour warps, 1 halo warp, 1 TMA producer warp
    static constexpr size_t SMEM = sizeof(double) * PL * RING + 8 * RING + 128;
    static constexpr size_t SMEM_RES = SMEM + sizeof(double) * PL * SHADOW;
    static constexpr int PTAB = RW + SH + 2;   // ints per tile: xtab, ytab, (cI0, cJ0)
    static constexpr size_t SMEM_PRO = sizeof(double) * PL * RING_PRO + 8 * RING_PRO + 128 +
                                       sizeof(double) * 2 * CPL + sizeof(int) * 2 * PTAB + 64;
    static_assert(TJ % 2 == 0 && NHALO <= 32, "tile rows even; halo columns must fit one warp");
};
// The plain and PRO sweeps run 64 x 8 tiles (18 colour warps); the residual
// variant 64 x 6 tiles (14 colour warps, 16 in all): its 8-plane shadow makes
// it register- and L1-tighter, and at Paper-scale level 0 it measured 5.34 ms
// on 64 x 6 against 6.08 ms on 64 x 8 (the plain sweep: 4.67 against 4.54)
constexpr int TJ_SWEEP = 8, TJ_RES = 6, TJ_SMALL = 4;

namespace {

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
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(sa(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// bounded wait: a copy that never lands (a fault) traps instead of hanging
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    unsigned n = 0;
    while (!mbar_try(b, parity))
        if (++n > (1u << 26)) __trap();
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                     uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sa(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(bar))
        : "memory");
}

// Fused prolongation (PRO variant: the first post-smoothing sweep of a level
// whose transition to the next level is horizontal with an identity z map).
// The sweep's input is lambda + w P lambda_c (Eq. (7) "u <- u + P u_c",
// P:176-181), formed in the ring: during step s every thread corrects its
// share of the ring plane s + 2 (landed: the producer waited for it at the end
// of step s - 1, one plane further ahead than the plain sweep, hence the
// 13-plane ring and 5 planes in flight) from the coarse values under the tile,
// staged the step before by cp.async, with exactly prolong_kernel's
// operations -- bitwise equal to the prolongation pass followed by the sweep.
struct ProArgs {
    const double* xc;         // coarse lambda (i-split layout of level C)
    LevDev C;                 // the coarse level
    const int* lox;           // fine index -> lower parent, coincident flag (x, y)
    const int* cox;
    const int* loy;
    const int* coy;
    double w;                 // correction weight (1 = Eq. (7))
};

// base pointers of the coupling loads: slot s of node p is kf[s][o(p)];
// the backward coupling K(p, p - d_s) = K_s[p - d_s] is kb[s][o(p) + x shift]
// (kb[s] already holds the row / plane shift of -d_s)
struct KBase {
    const double* kf[14];
    const double* kb[14];
};

// MODE 0: plain sweep; 1 (RES): also ||f - K lin||^2; 2 (PRO): input lin + w P xc
template <int MODE, int TJ_>
__global__ void __launch_bounds__(Geo<TJ_>::THREADS, 1)
gs_fused2_kernel(const __grid_constant__ CUtensorMap mL, const __grid_constant__ KBase KB,
                 LevDev L, double* __restrict__ lout, const double* __restrict__ f, int jt0,
                 int ntx, int ntiles, int jitter, double* __restrict__ partial,
                 const __grid_constant__ ProArgs PA) {
    constexpr bool RES = MODE == 1, PRO = MODE == 2;
    using Gm = Geo<TJ_>;
    constexpr int TJ = Gm::TJ, SH = Gm::SH, PLD = Gm::PLD, PL = Gm::PL, PTAB = Gm::PTAB;
    constexpr int B0 = Gm::B0, B1 = Gm::B1, W0 = Gm::W0, W1 = Gm::W1, W2 = Gm::W2, W3 = Gm::W3;
    constexpr int NHALO = Gm::NHALO, PRODUCER = Gm::PRODUCER, THREADS = Gm::THREADS;
    constexpr unsigned BOX_BYTES = Gm::BOX_BYTES;
    constexpr int RING = PRO ? RING_PRO : ::wd::RING;
    constexpr int LA = PRO ? LA_PRO : ::wd::LA;
    static_assert(RING >= LA + 8, "ring too short");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw + ((128 - (sa(smem_raw) & 127)) & 127));
    double* shadow = ring + PL * RING;
    double* csm = ring + PL * RING;                             // PRO: [2][CPL]
    int* ptab = reinterpret_cast<int*>(csm + 2 * CPL);          // PRO: [2][PTAB]
    constexpr int EXTRA = RES ? PL * SHADOW : PRO ? 2 * CPL + PTAB + 8 : 0;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + PL * RING + EXTRA);
    for (int t = threadIdx.x; t < PL * RING + (RES ? PL * SHADOW : PRO ? 2 * CPL : 0); t += THREADS)
        ring[t] = 0.0;
    if (threadIdx.x == 0) {
        for (int t = 0; t < RING; t++) mbar_init(&full[t], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int c, di, dj;
    bool inreg = true;
    if (w < W0) { c = 0; dj = 2 * w; di = 2 * lane; }
    else if (w < W1) { c = 1; dj = 2 * (w - W0); di = 1 + 2 * lane; }
    else if (w < W2) { c = 2; dj = 1 + 2 * (w - W1); di = 2 * lane; }
    else if (w < W3) { c = 3; dj = 1 + 2 * (w - W2); di = 1 + 2 * lane; }
    else if (w > W3) { c = 0; dj = 0; di = -10; inreg = false; }   // the TMA producer warp
    else if (lane < 3 * B0) {
        c = 0; dj = 2 * (lane / 3);
        const int e = lane % 3;
        di = e == 0 ? -2 : TI + 2 * e - 2;
    } else if (lane < 3 * B0 + 2 * B1) {
        const int q = lane - 3 * B0;
        c = 1; dj = 2 * (q / 2); di = (q % 2) == 0 ? -1 : TI + 1;
    } else if (lane < NHALO) {
        const int q = lane - 3 * B0 - 2 * B1;
        c = 2; dj = 1 + 2 * q; di = TI;
    } else { c = 0; dj = 0; di = -10; inreg = false; }
    const int ci = c & 1;
    const int li = di + 4, lj = dj + 1;
    const int so = lj * RW + (li & 1) * SW + (li >> 1);
    const int sxm = ci ? -SW : SW - 1, sxp = ci ? 1 - SW : SW;
    const int gxm = ci ? -L.H : L.H - 1, gxp = ci ? 1 - L.H : L.H;
    const int sk = (int)L.sk;
    const int n3 = L.n3, nz = L.n3 - 1;
    const int ntk = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int G = ntk * n3;

    auto origin = [&](int k, int& I0, int& J0) {
        const int tau = (int)blockIdx.x + k * (int)gridDim.x;
        const int ty = tau / ntx;
        I0 = (tau - ty * ntx) * TI;
        J0 = jt0 + ty * TJ;
    };
    bool act = false, wrt = false;
    int own = 0;   // offset of the thread's column at plane 0 (< NT < 2^31)
    auto set_tile = [&](int k) {
        int I0, J0;
        origin(k, I0, J0);
        const int i = I0 + di, j = J0 + dj;
        const int jg = j + L.jg0;
        act = inreg && i >= 1 && i <= L.n1 - 2 && j >= 1 && j <= L.n2 - 2 && jg >= 1 &&
              jg <= L.n2g - 2;
        wrt = act && di >= 0 && di < TI && dj < TJ && j >= L.own0 && j < L.own1;
        own = act ? (int)loff(L, i, j, 0) : 0;
    };
    // TMA producer state (thread 0): the virtual plane gl = kl * n3 + zl
    int kl = 0, zl = 0, lI0 = 0, lJ0 = 0, lslot = 0;
    auto issue = [&]() {
        if (zl == 0) origin(kl, lI0, lJ0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(&full[lslot], BOX_BYTES);
        tma4(ring + lslot * PL, &mL, (lI0 >> 1) - 2, 0, zl, lJ0 - 1, &full[lslot]);
        if (++lslot == RING) lslot = 0;
        if (++zl == n3) { zl = 0; ++kl; }
    };
    // ---- PRO helpers (every thread takes a share)
    // tables of tile tk (in buffer tk & 1): ring column r -> (coarse x index
    // relative to the tile's coarse origin << 1 | two parents), -1 if the
    // column is not free; ring row rj likewise for y; then (cI0, cJ0)
    auto build_tables = [&](int tk) {
        int I0, J0;
        origin(tk, I0, J0);
        int* t = ptab + (tk & 1) * PTAB;
        const int cI0 = __ldg(PA.lox + max(I0 - 4, 0)), cJ0 = __ldg(PA.loy + max(J0 - 1, 0));
        for (int r = threadIdx.x; r < PTAB; r += THREADS) {
            int v = -1;
            if (r < RW) {   // column: half = r / SW, pos = r % SW
                const int i = I0 - 4 + 2 * (r % SW) + r / SW;
                if (i >= 1 && i <= L.n1 - 2)
                    v = ((__ldg(PA.lox + i) - cI0) << 1) | (__ldg(PA.cox + i) ? 0 : 1);
            } else if (r < RW + SH) {
                const int j = J0 - 1 + (r - RW);
                if (j >= 0 && j < L.n2 && row_free(L, j))
                    v = ((__ldg(PA.loy + j) - cJ0) << 1) | (__ldg(PA.coy + j) ? 0 : 1);
            } else {
                v = r == RW + SH ? cI0 : cJ0;
            }
            t[r] = v;
        }
    };
    // coarse values of plane q (tile q / n3, plane z) -> csm[q & 1] (cp.async;
    // the tile's tables must be built and visible)
    auto stage_coarse = [&](int q) {
        const int tk = q / n3, z = q - tk * n3;
        const int* t = ptab + (tk & 1) * PTAB;
        const int cI0 = t[RW + SH], cJ0 = t[RW + SH + 1];
        double* dst = csm + (q & 1) * CPL;
        for (int e = threadIdx.x; e < CPL; e += THREADS) {
            const int I = cI0 + e % CXM, J = cJ0 + e / CXM;
            if (I < PA.C.n1 && J < PA.C.n2 && z < PA.C.n3) {
                const unsigned sd = (unsigned)__cvta_generic_to_shared(dst + e);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sd),
                             "l"(PA.xc + loff(PA.C, I, J, z)) : "memory");
            } else {
                dst[e] = 0.0;
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // ring plane q += w P (coarse plane q) on its free nodes (prolong_kernel's
    // identity-z operations, bitwise equal)
    auto correct_plane = [&](int q) {
        const int tk = q / n3, z = q - tk * n3;
        if (z >= nz) return;
        const int* t = ptab + (tk & 1) * PTAB;
        const double* cs = csm + (q & 1) * CPL;
        double* rp = ring + (q % RING) * PL;
        for (int e = threadIdx.x; e < PLD; e += THREADS) {
            const int rj = e / RW, r = e - rj * RW;
            const int xt = t[r], yt = t[RW + rj];
            if (xt < 0 || yt < 0) continue;
            const bool two = xt & 1, ny2 = yt & 1;
            const double wx = two ? 0.5 : 1.0, wy = ny2 ? 0.5 : 1.0;
            const double* c0 = cs + (yt >> 1) * CXM + (xt >> 1);
            const double a0 = c0[0], a1 = c0[1], a2 = c0[CXM], a3 = c0[CXM + 1], x = rp[e];
            double sr = 0.0 + a0;
            sr += two ? a1 : -0.0;
            double sv = fma(wy * 1.0, wx * sr, 0.0);
            if (ny2) {
                double sr2 = 0.0 + a2;
                sr2 += two ? a3 : -0.0;
                sv = fma(wy * 1.0, wx * sr2, sv);
            }
            rp[e] = fma(PA.w, sv, x);
        }
    };
    __syncthreads();   // ring zeroed, barriers initialised
    // One thread issues the plane loads and waits for their mbarriers; the
    // CTA barrier that follows its wait orders the landed plane before every
    // other thread's reads (the waiting thread acquires the TMA writes, the
    // barrier carries them on), so the 608 threads do not poll the mbarriers.
    if (threadIdx.x == PRODUCER) {
        for (int p = 0; p < LA && p < G; p++) issue();
        for (int p = 0; p < (PRO ? 3 : 2) && p < G; p++) mbar_wait(&full[p], 0);
    }
    if (PRO && G > 0) {   // planes 0 and 1 corrected, plane 2's coarse values staged
        build_tables(0);
        if (n3 <= 3 && ntk > 1) build_tables(1);   // tile 1 starts within planes 0..3
        __syncthreads();
        for (int p = 0; p < 3 && p < G; p++) {
            stage_coarse(p);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncthreads();
            if (p < 2) correct_plane(p);
        }
    }
    __syncthreads();

    double kf[13], kb[13], fv = 0.0, kd = 1.0;
    auto load_k = [&](int z) {
        const int o = own + z * sk;
        const int om = o + gxm, op = o + gxp;
#pragma unroll
        for (int sl = 1; sl < 14; sl++) kf[sl - 1] = __ldg(KB.kf[sl] + o);
#pragma unroll
        for (int sl = 1; sl < 14; sl++) {
            const int dx = slot_dx(sl), dz = slot_dz(sl);
            const int ob = dx > 0 ? om : dx < 0 ? op : o;   // x of the backward neighbour i - dx
            if (dz) kb[sl - 1] = z > 0 ? __ldg(KB.kb[sl] + ob) : 0.0;
            else kb[sl - 1] = __ldg(KB.kb[sl] + ob);
        }
        fv = __ldg(f + o);
        kd = __ldg(KB.kf[0] + o);
    };
    int kn = 0, zn = 0;
    if (G > 0) set_tile(0);
    if (c == 0 && act && G > 0) load_k(0);

    // ring slot of the thread's current virtual plane g (advanced with g)
    int rg = 0;
    double rr = 0.0;
    const int nsteps = G + LAG * 3;
    for (int s = 0; s < nsteps; s++) {
        if (threadIdx.x == PRODUCER && s + LA < G) issue();
        if (jitter) {
            // race stress test (tests only, env WD_TEST_JITTER): every warp
            // sleeps a pseudo-random 0..jitter ns before its step, so the warps
            // and CTAs reach their reads and writes in shuffled orders; the
            // result must not change (bitwise)
            unsigned h = (unsigned)(blockIdx.x * 977u + (threadIdx.x >> 5) * 131u + s * 7919u);
            h ^= h >> 13;
            h *= 0x5bd1e995u;
            h ^= h >> 15;
            __nanosleep(h % (unsigned)jitter);
        }
        const int g = s - LAG * c;
        if (g >= 0 && g < G) {
            const int z = zn;
            const int rp = rg + 1 == RING ? 0 : rg + 1, rq = rg == 0 ? RING - 1 : rg - 1;
            double* r0 = ring + rg * PL + so;
            if (RES && inreg) shadow[(g & (SHADOW - 1)) * PL + so] = *r0;
            if (z < nz && act) {
                const double* r1 = ring + rp * PL + so;
                const double* rm = ring + rq * PL + so;
                auto sc = [&](int dx, int dy) { return dy * RW + (dx < 0 ? sxm : dx > 0 ? sxp : 0); };
                double acc = 0.0;
#pragma unroll
                for (int sl = 1; sl < 14; sl++) {
                    const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
                    acc = fma(kf[sl - 1], (dz ? r1 : r0)[sc(dx, dy)], acc);
                }
#pragma unroll
                for (int sl = 1; sl < 14; sl++) {
                    const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
                    if (dz) {
                        if (z > 0) acc = fma(kb[sl - 1], rm[sc(-dx, -dy)], acc);
                    } else {
                        acc = fma(kb[sl - 1], r0[sc(-dx, -dy)], acc);
                    }
                }
                const double v = (fv - acc) / kd;
                if (RES && wrt) {
                    const bool codd = c & 1, chi = c >= 2;
                    const double* s1 = shadow + ((g + 1) & (SHADOW - 1)) * PL + so;
                    const double* s0 = shadow + (g & (SHADOW - 1)) * PL + so;
                    const double* sm = shadow + ((g + SHADOW - 1) & (SHADOW - 1)) * PL + so;
                    auto oldv = [&](int dx, int dy, int dz) {
                        const bool sh = (dx == 0 && dy == 0) ? dz < 0 : ((dy & 1) ? chi : codd);
                        const double* rpp = dz > 0 ? r1 : dz < 0 ? rm : r0;
                        const double* sp = dz > 0 ? s1 : dz < 0 ? sm : s0;
                        return (sh ? sp : rpp)[sc(dx, dy)];
                    };
                    double q = kd * r0[0];
#pragma unroll
                    for (int sl = 1; sl < 14; sl++) {
                        const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
                        q = fma(kf[sl - 1], oldv(dx, dy, dz), q);
                    }
#pragma unroll
                    for (int sl = 1; sl < 14; sl++) {
                        const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
                        if (dz) {
                            if (z > 0) q = fma(kb[sl - 1], oldv(-dx, -dy, -dz), q);
                        } else {
                            q = fma(kb[sl - 1], oldv(-dx, -dy, 0), q);
                        }
                    }
                    const double rv = fv - q;
                    rr = fma(rv, rv, rr);
                }
                *r0 = v;
                if (wrt) lout[own + z * sk] = v;
            }
            rg = rp;
            if (++zn == n3) {
                zn = 0;
                if (++kn < ntk) set_tile(kn);
            }
            if (PRO) {   // this thread's share of plane s + 2, staging of plane s + 3
                if (s + 2 < G) correct_plane(s + 2);
                if (s + 3 < G) stage_coarse(s + 3);
            }
            if (g + 1 < G && zn < nz && act) load_k(zn);
        } else {
            if (PRO) {
                if (s + 2 < G) correct_plane(s + 2);
                if (s + 3 < G) stage_coarse(s + 3);
            }
            if (g == -1 && act && G > 0) load_k(0);
        }
        if (PRO) {
            // the tables of the tile whose first plane is staged at step s + 1
            const int q = s + 4;
            if (q < G && q % n3 == 0) build_tables(q / n3);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        // the newest plane read at step s + 1 is s + 2 (colour 0's plane above);
        // PRO corrects plane s + 3 during step s + 1, so it waits one plane ahead
        const int qw = s + (PRO ? 3 : 2);
        if (threadIdx.x == PRODUCER && qw < G) mbar_wait(&full[qw % RING], (qw / RING) & 1);
        __syncthreads();
    }
    if (RES) {
        __shared__ double wsum[THREADS / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rr += __shfl_down_sync(0xffffffffu, rr, o);
        if (lane == 0) wsum[w] = rr;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < THREADS / 32; q++) t += wsum[q];
            partial[blockIdx.x] = t;
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn2() {
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

}  // namespace

// lambda of a level as the 4-D tensor (position, half, plane, row) with the
// ring box of one plane: 36 positions x 2 halves x 1 plane x 11 rows; the
// position extent is the grid's (ceil(n1/2)), so the padding of a half row
// and everything outside the grid read as zeros
int make_ring_map(const LevDev& L, const double* v, void* map, int tj) {
    auto enc = encode_fn2();
    if (!enc) return -1;
    cuuint64_t dims[4] = {(cuuint64_t)((L.n1 + 1) / 2), 2, (cuuint64_t)L.n3, (cuuint64_t)L.n2};
    cuuint64_t str[3] = {(cuuint64_t)L.H * 8, (cuuint64_t)L.sk * 8, (cuuint64_t)L.sj * 8};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint32_t box[4] = {SW, 2, 1, (cuuint32_t)(tj + 3)};   // Geo<tj>::SH
    static const CUtensorMapL2promotion promo[4] = {
        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    int pr = 0;
    if (const char* e = getenv("WD_RING_L2PROMO")) pr = atoi(e) & 3;
    CUresult r = enc((CUtensorMap*)map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)v, dims, str,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo[pr],
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -1;
}

int gs_fused2_prepare() {
    static std::atomic<int> nsm_dev[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int nsm = nsm_dev[dev].load(std::memory_order_acquire);
    if (nsm > 0) return nsm;
    cudaFuncSetAttribute(gs_fused2_kernel<0, TJ_SWEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Geo<TJ_SWEEP>::SMEM);
    cudaFuncSetAttribute(gs_fused2_kernel<1, TJ_RES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Geo<TJ_RES>::SMEM_RES);
    cudaFuncSetAttribute(gs_fused2_kernel<0, TJ_SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Geo<TJ_SMALL>::SMEM);
    cudaFuncSetAttribute(gs_fused2_kernel<1, TJ_SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Geo<TJ_SMALL>::SMEM_RES);
    cudaFuncSetAttribute(gs_fused2_kernel<2, TJ_SWEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Geo<TJ_SWEEP>::SMEM_PRO);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
    nsm_dev[dev].store(nsm, std::memory_order_release);
    return nsm;
}

// one sweep lin -> lout (k_gs_fused.cu launch_gs_fused); ring_map /
// ring_map_res: the make_ring_map tensor maps of lin (plain / residual tiles)
// tile rows of a plain sweep: [0, b0) hold the first w owned rows, [b1, nty)
// the last w (the rows a slab's neighbours need after the sweep); b0 >= b1
// means the boundary tiles cover everything
void gs_fused2_tile_rows(const LevDev& L, int w, int* b0, int* b1, int* nty) {
    const int jt0 = L.own0 - ((L.own0 + L.jg0) & 1);
    *nty = (L.own1 - jt0 + TJ_SWEEP - 1) / TJ_SWEEP;
    *b0 = std::min((L.own0 + w - 1 - jt0) / TJ_SWEEP + 1, *nty);
    *b1 = std::max((L.own1 - w - jt0) / TJ_SWEEP, 0);
}

int launch_gs_fused2(const LevDev& L, const double* coef, const void* ring_map,
                     const void* ring_map_res, const void* ring_map_small, double* lout,
                     const double* f, cudaStream_t st, double* partial, const ProlongIn* pro,
                     int tr0, int tr1) {
    const int nsm = gs_fused2_prepare();
    KBase KB;
    for (int s = 0; s < 14; s++) {
        const int dy = slot_dy(s), dz = slot_dz(s);
        KB.kf[s] = coef + (i64)s * L.NT;
        // backward neighbour p - d_s: row j - dy, plane z - dz (x shift per thread)
        KB.kb[s] = coef + (i64)s * L.NT - (i64)dy * L.sj - (i64)dz * L.sk;
    }
    // small levels (n1 < 200): the plain sweep on 64 x 4 tiles (more, shorter
    // tiles for the few CTAs such a level keeps busy: Small's V-cycle -17 %,
    // Paper-scale 189^2 / 95^2 / 48^2 sweeps 31 / 26 / 18 -> 26 / 22 / 15 us on
    // 64 x 6 and less on 64 x 4; from 251^2 up the 64 x 8 tiles are faster).
    // Any tiling gives the same node updates (bitwise)
    const bool small = !pro && tr1 < 0 && L.n1 < 200;
    const int tj = small ? TJ_SMALL : partial ? TJ_RES : TJ_SWEEP;
    int jt0 = L.own0 - ((L.own0 + L.jg0) & 1);
    const int ntx = (L.n1 + TI - 1) / TI;
    int nty = (L.own1 - jt0 + tj - 1) / tj;
    if (tr1 >= 0 && !partial) {   // tile rows [tr0, tr1) of the plain / PRO sweep
        jt0 += tr0 * tj;
        nty = std::max(std::min(tr1, nty) - tr0, 0);
        if (nty == 0) return 0;
    }
    g_launches += 1;
    // persistent CTAs; tests may cap their number (env WD_TEST_GS_GRID) so that
    // other tiles share a CTA's cross-tile pipeline
    int grid = std::min(ntx * nty, nsm);
    if (g_test_gs_grid > 0) grid = std::min(grid, g_test_gs_grid);
    ProArgs PA{};
    if (pro) {
        PA.xc = pro->xc;
        PA.C = pro->C;
        PA.lox = pro->M.lo[0];
        PA.cox = pro->M.co[0];
        PA.loy = pro->M.lo[1];
        PA.coy = pro->M.co[1];
        PA.w = pro->w;
    }
    if (small && partial) {
        using G = Geo<TJ_SMALL>;
        gs_fused2_kernel<1, TJ_SMALL><<<grid, G::THREADS, G::SMEM_RES, st>>>(
            *(const CUtensorMap*)ring_map_small, KB, L, lout, f, jt0, ntx, ntx * nty, g_test_jitter,
            partial, PA);
    } else if (small) {
        using G = Geo<TJ_SMALL>;
        gs_fused2_kernel<0, TJ_SMALL><<<grid, G::THREADS, G::SMEM, st>>>(
            *(const CUtensorMap*)ring_map_small, KB, L, lout, f, jt0, ntx, ntx * nty, g_test_jitter,
            nullptr, PA);
    } else if (partial) {
        using G = Geo<TJ_RES>;
        gs_fused2_kernel<1, TJ_RES><<<grid, G::THREADS, G::SMEM_RES, st>>>(
            *(const CUtensorMap*)ring_map_res, KB, L, lout, f, jt0, ntx, ntx * nty, g_test_jitter,
            partial, PA);
    } else {
        using G = Geo<TJ_SWEEP>;
        const CUtensorMap& m = *(const CUtensorMap*)ring_map;
        if (pro)
            gs_fused2_kernel<2, TJ_SWEEP><<<grid, G::THREADS, G::SMEM_PRO, st>>>(
                m, KB, L, lout, f, jt0, ntx, ntx * nty, g_test_jitter, nullptr, PA);
        else
            gs_fused2_kernel<0, TJ_SWEEP><<<grid, G::THREADS, G::SMEM, st>>>(
                m, KB, L, lout, f, jt0, ntx, ntx * nty, g_test_jitter, nullptr, PA);
    }
    return grid;
}

}  // namespace wd
