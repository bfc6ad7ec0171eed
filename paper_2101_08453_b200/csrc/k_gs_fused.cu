// k_gs_fused.cu -- one whole smoothing sweep (all four colour phases) in one pass.
//
// The smoother is P:174-176: "vertical sweeps of Gauss-Seidel from the bottom
// up to the top, with red-black ordering horizontally into 4 groups", colours
// (i mod 2, j mod 2) = (0,0),(1,0),(0,1),(1,1) in this order (reading C7).
// gs_phase_kernel (k_mg.cu) runs one launch per colour; every launch reads the
// 27 couplings of its quarter of the nodes, so the stored operator (14 slots)
// crosses HBM about twice per sweep (SURVEY 8(d) "practical" 264 B/node).
//
// This kernel computes the same iterate (same dependency graph, same
// floating-point operations in the same order, hence bitwise equal) with a
// schedule that touches the operator once per sweep from HBM:
//
//   * a CTA owns a tile of 64 x 8 node columns and redundantly recomputes
//     colour c on a halo of (3-c) columns in i and 1 row in j for c <= 1
//     (phase 3 needs phase 2 at i+-1; phase 2 needs phase 1 at (i+-1, j+-1);
//     phase 1 needs phase 0 at i+-1), so it never waits for another CTA
//     (605 columns computed for 512 owned: 1.18x);
//   * one warp per (colour, row) covers 32 aligned half-row positions (full
//     32 B sectors in the i-split layout); one extra warp takes the 29 halo
//     columns;
//   * the four phases run concurrently in a k-pipeline with a lag of two
//     planes: at step s colour c updates plane z = s - 2c.  Colour c at plane
//     z needs the NEW values of colours c' < c at planes z-1..z+1 (updated at
//     steps <= s-1) and the OLD values of colours c' > c at z-1..z+1 (updated
//     at steps >= s+1), so one barrier per step orders everything;
//   * persistent CTAs (one per SM) walk their tiles back to back and the
//     k-pipeline runs on across them: with virtual plane g = k n3 + z (k-th
//     tile of the CTA), colour c handles g = s - 2c at step s, so the next
//     tile's first planes are updated while the previous tile's last colours
//     finish (no per-tile fill/drain or prologue);
//   * lambda of the tile (+ halo) lives in a 12-plane shared-memory ring
//     (76 KB: the kernel depends on the L1 left beside it -- the same kernel
//     with 2x the shared memory reserved takes 2x as long),
//     filled with cp.async four planes ahead; the old iterate is read from one
//     buffer and the new one written to another (ping-pong), so halo reads
//     never see a neighbour CTA's new values;
//   * the 27 couplings, f and the diagonal of a thread's next node are loaded
//     into registers one step ahead (before the barrier); the second use of
//     every stored coefficient (by the node at the other end of the coupling,
//     at most 7 steps later) and the halo recomputation hit L2, so HBM sees
//     the operator about once per sweep (ncu, Paper-scale level 0: 19.7 GB
//     read per sweep against 18.3 GB algorithmic; the four phase launches
//     read ~34 GB).
//
// Residual variant (RES = true, used for the first sweep of a V-cycle inside
// wd_solve): the sweep also returns ||f - K lin||^2 over its owned free nodes,
// i.e. the convergence test of the previous cycle's iterate, from the
// couplings it already holds in registers; old values of neighbours already
// updated come from an 8-plane shadow where each thread saves its node's old
// value when it overwrites it -- no separate residual pass over the operator.
#include "wd_internal.cuh"

#include <algorithm>
#include <atomic>

namespace wd {


namespace {

constexpr int HI = 32;              // positions per parity per tile row (TI = 64 columns)
constexpr int TI = 2 * HI;
constexpr int TJ = 8;               // tile rows
constexpr int SW = HI + 4;          // ring positions per parity per row (columns I0-3 .. I0+TI+3)
constexpr int RW = 2 * SW;          // ring doubles per row
constexpr int SH = TJ + 3;          // ring rows J0-1 .. J0+TJ+1
constexpr int PL = RW * SH;         // ring doubles per plane
constexpr int RING = 12;            // planes in the ring (>= LA + 8: colour 3 reads plane s-7)
constexpr int LAG = 2;              // plane lag between consecutive colours
constexpr int LA = 4;               // lambda planes loaded ahead
// colour regions: rows per colour (B) and halo columns beyond the 32 aligned ones
constexpr int B0 = TJ / 2 + 1, B1 = TJ / 2 + 1, B2 = TJ / 2, B3 = TJ / 2;
constexpr int W0 = B0, W1 = W0 + B1, W2 = W1 + B2, W3 = W2 + B3;   // warp ranges
constexpr int NHALO = 3 * B0 + 2 * B1 + B2;                          // 29 halo columns
constexpr int THREADS = 32 * (W3 + 1);                               // 19 warps
constexpr size_t SMEM = sizeof(double) * PL * RING;
// residual variant: a node of colour c' is overwritten at step z + 2c' and its
// old value read by higher colours up to plane z + 1 at step z + 1 + 6
constexpr int SHADOW = 8;
constexpr size_t SMEM_RES = SMEM + sizeof(double) * PL * SHADOW;
static_assert(NHALO <= 32, "halo columns must fit one warp");

__device__ __forceinline__ void cp_async8(double* s, const double* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(double* s, const double* g) {   // bypasses L1
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <bool RES>
__global__ void __launch_bounds__(THREADS, 1)
gs_fused_kernel(LevDev L, const double* __restrict__ K, const double* __restrict__ lin,
                     double* __restrict__ lout, const double* __restrict__ f, int jt0, int ntx,
                     int ntiles, double* __restrict__ partial) {
    extern __shared__ double ring[];
    // RES: the old values of the last SHADOW planes, saved by each thread when
    // it overwrites its node in the ring
    double* shadow = ring + PL * RING;
    for (int t = threadIdx.x; t < PL * (RING + (RES ? SHADOW : 0)); t += THREADS) ring[t] = 0.0;

    // this thread's colour c and the in-tile offsets (di, dj) of its column:
    // one warp per (colour, row) over the 32 aligned positions, the last warp
    // takes the 29 halo columns (colour 0: -2, TI, TI+2; 1: -1, TI+1; 2: TI)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int c, di, dj;
    bool inreg = true;
    if (w < W0) { c = 0; dj = 2 * w; di = 2 * lane; }
    else if (w < W1) { c = 1; dj = 2 * (w - W0); di = 1 + 2 * lane; }
    else if (w < W2) { c = 2; dj = 1 + 2 * (w - W1); di = 2 * lane; }
    else if (w < W3) { c = 3; dj = 1 + 2 * (w - W2); di = 1 + 2 * lane; }
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
    const int gsj = (int)L.sj;
    auto sc = [&](int dx, int dy) { return dy * RW + (dx < 0 ? sxm : dx > 0 ? sxp : 0); };
    auto co = [&](int dx, int dy) { return dy * gsj + (dx < 0 ? gxm : dx > 0 ? gxp : 0); };
    const i64 NT = L.NT;
    const int n3 = L.n3, nz = L.n3 - 1;
    const int ntk = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int G = ntk * n3;

    // tile k of this CTA -> origin (I0, J0)
    auto origin = [&](int k, int& I0, int& J0) {
        const int tau = (int)blockIdx.x + k * (int)gridDim.x;
        const int ty = tau / ntx;
        I0 = (tau - ty * ntx) * TI;
        J0 = jt0 + ty * TJ;
    };
    // this thread's column in tile k: active / writes / offset of plane 0
    bool act = false, wrt = false;
    i64 own = 0;
    auto set_tile = [&](int k) {
        int I0, J0;
        origin(k, I0, J0);
        const int i = I0 + di, j = J0 + dj;
        // computed: a free node whose rows j-1, j+1 are present in this part
        // (on a slab the halo rows next to the owned ones are recomputed as
        // tile halo; their inputs come from the 2-row exchange before the sweep)
        const int jg = j + L.jg0;
        act = inreg && i >= 1 && i <= L.n1 - 2 && j >= 1 && j <= L.n2 - 2 && jg >= 1 &&
              jg <= L.n2g - 2;
        // written: owned rows of the tile's own region only
        wrt = act && di >= 0 && di < TI && dj < TJ && j >= L.own0 && j < L.own1;
        own = act ? loff(L, i, j, 0) : 0;
    };
    // lambda load stream: virtual plane gl = (kl, zl).  Each thread fills the
    // ring entries e = threadIdx.x + q THREADS (q < NE) of every plane; their
    // offsets relative to the tile origin are fixed, so per plane only the
    // tile base and the plane stride change.
    // Entries go in pairs (2e, 2e+1: adjacent positions of one half row, 16 B
    // aligned in HBM and in the ring) copied with one 16-byte cp.async.cg that
    // bypasses L1 (the kernel lives on L1 hits of the couplings); a pair
    // straddling the grid edge is copied or zeroed entry by entry.
    constexpr int NE = (PL / 2 + THREADS - 1) / THREADS;   // pairs per thread
    constexpr int NEL = 2 * NE;
    static_assert(RW % 2 == 0 && SW % 2 == 0, "pairs must not straddle half rows");
    i64 eoff[NEL];
    int eri[NEL], erj[NEL];
#pragma unroll
    for (int q = 0; q < NEL; q++) {
        const int e = 2 * ((int)threadIdx.x + (q >> 1) * THREADS) + (q & 1);
        const int rj = e / RW, r = e - rj * RW;
        const int half = r >= SW, pos = r - half * SW;
        erj[q] = e < PL ? rj : -1000000;   // never valid beyond the ring
        eri[q] = 2 * pos + half;
        // loff(i, j, 0) - loff(I0 - 4, J0 - 1, 0) for i = I0 - 4 + ri (I0 even), j = J0 - 1 + rj
        eoff[q] = (i64)rj * L.sj + (i64)half * L.H + pos;
    }
    int kl = 0, zl = 0;
    i64 lbase = 0;        // loff(I0 - 4 (even part), J0 - 1, zl) of the loading tile
    unsigned lvalid = 0;  // bit q: entry q lies inside the grid (NEL <= 32)
    auto load_tile = [&](int k) {
        int I0, J0;
        origin(k, I0, J0);
        lbase = (i64)(J0 - 1) * L.sj + (I0 >> 1) - 2;
        lvalid = 0;
#pragma unroll
        for (int q = 0; q < NEL; q++) {
            const int i = I0 - 4 + eri[q], j = J0 - 1 + erj[q];
            if (eri[q] >= 1 && i >= 0 && i < L.n1 && j >= 0 && j < L.n2) lvalid |= 1u << q;
        }
    };
    if (G > 0) load_tile(0);
    auto load_next = [&]() {
        double* dst = ring + ((kl * n3 + zl) % RING) * PL;
        const i64 pb = lbase + (i64)zl * L.sk;
#pragma unroll
        for (int q = 0; q < NE; q++) {
            const int e = 2 * ((int)threadIdx.x + q * THREADS);
            const unsigned b = (lvalid >> (2 * q)) & 3u;
            if (b == 3u) cp_async16(dst + e, lin + pb + eoff[2 * q]);
            else if (e < PL) {
                if (b & 1u) cp_async8(dst + e, lin + pb + eoff[2 * q]);
                else dst[e] = 0.0;
                if (b & 2u) cp_async8(dst + e + 1, lin + pb + eoff[2 * q + 1]);
                else dst[e + 1] = 0.0;
            }
        }
        if (++zl == n3) {
            zl = 0;
            if (++kl < ntk) load_tile(kl);
        }
    };
    __syncthreads();   // ring zeroed before the first copies land
    for (int p = 0; p < LA; p++) {
        if (p < G) load_next();
        cp_async_commit();
    }
    cp_async_wait<LA - 2>();
    __syncthreads();

    double kf[13], kb[13], fv = 0.0, kd = 1.0;
    auto load_k = [&](int z) {
        const i64 base = own + (i64)z * L.sk;
#pragma unroll
        for (int sl = 1; sl < 14; sl++) kf[sl - 1] = __ldg(K + sl * NT + base);
#pragma unroll
        for (int sl = 1; sl < 14; sl++) {
            const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
            if (dz) kb[sl - 1] = z > 0 ? __ldg(K + sl * NT + base - L.sk + co(-dx, -dy)) : 0.0;
            else kb[sl - 1] = __ldg(K + sl * NT + base + co(-dx, -dy));
        }
        fv = __ldg(f + base);
        kd = __ldg(K + base);
    };
    // the thread's next node: plane zn of its kn-th tile (virtual plane s - 2c)
    int kn = 0, zn = 0;
    if (G > 0) set_tile(0);
    if (c == 0 && act && G > 0) load_k(0);

    double rr = 0.0;   // RES: this thread's sum of squared residuals
    const int nsteps = G + LAG * 3;
    for (int s = 0; s < nsteps; s++) {
        if (s + LA < G) load_next();
        cp_async_commit();
        const int g = s - LAG * c;
        if (g >= 0 && g < G) {
            const int z = zn;
            // RES: every mapped column saves its old value (also Dirichlet and
            // outside-grid columns, which are never updated) before the update
            if (RES && inreg) shadow[(g & (SHADOW - 1)) * PL + so] = ring[(g % RING) * PL + so];
            if (z < nz && act) {
                const double* r1 = ring + ((g + 1) % RING) * PL + so;
                const double* r0 = ring + (g % RING) * PL + so;
                const double* rm = ring + ((g + RING - 1) % RING) * PL + so;
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
                    // residual of the old iterate at this node.  Neighbours of a
                    // lower colour (c' < c, any plane) and the node below in the
                    // column are already overwritten in the ring: their old values
                    // are in the shadow.  c' = c ^ (dx odd) ^ 2 (dy odd), so
                    // c' < c iff c is odd (dx odd, dy even) or c >= 2 (dy odd).
                    const bool codd = c & 1, chi = c >= 2;
                    const double* s1 = shadow + ((g + 1) & (SHADOW - 1)) * PL + so;
                    const double* s0 = shadow + (g & (SHADOW - 1)) * PL + so;
                    const double* sm = shadow + ((g + SHADOW - 1) & (SHADOW - 1)) * PL + so;
                    auto oldv = [&](int dx, int dy, int dz) {
                        const bool sh = (dx == 0 && dy == 0) ? dz < 0 : ((dy & 1) ? chi : codd);
                        const double* rp = dz > 0 ? r1 : dz < 0 ? rm : r0;
                        const double* sp = dz > 0 ? s1 : dz < 0 ? sm : s0;
                        return (sh ? sp : rp)[sc(dx, dy)];
                    };
                    double q = kd * r0[0];   // own old value (overwritten below)
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
                ring[(g % RING) * PL + so] = v;
                if (wrt) lout[own + (i64)z * L.sk] = v;
            }
            if (++zn == n3) {
                zn = 0;
                if (++kn < ntk) set_tile(kn);
            }
            if (g + 1 < G && zn < nz && act) load_k(zn);
        } else if (g == -1 && act && G > 0) {
            load_k(0);   // colours c > 0: first node, one step ahead
        }
        cp_async_wait<LA - 2>();
        __syncthreads();
    }
    cp_async_wait<0>();
    if (RES) {   // fixed-order block sum (deterministic): warp tree, then warps in order
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

}  // namespace

// Per-device setup (the dynamic shared-memory limit is a per-device function
// attribute): done once per device, from wd_assemble and on first use; the
// SM count is cached per device.  Setting an attribute twice is harmless, so
// concurrent first calls need no lock.
int gs_fused_prepare() {
    static std::atomic<int> nsm_dev[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int nsm = nsm_dev[dev].load(std::memory_order_acquire);
    if (nsm > 0) return nsm;
    cudaFuncSetAttribute(gs_fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    cudaFuncSetAttribute(gs_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_RES);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
    nsm_dev[dev].store(nsm, std::memory_order_release);
    return nsm;
}

// one sweep: lin (old iterate, unchanged) -> lout (new iterate on the owned
// free nodes; D entries of lout must already be 0).  partial != NULL: also
// ||f - K lin||^2 over the owned free nodes as one partial per CTA; returns
// the number of CTAs (partials)
int launch_gs_fused(const LevDev& L, const double* coef, const double* lin, double* lout,
                    const double* f, cudaStream_t st, double* partial) {
    const int nsm = gs_fused_prepare();
    // tiles of TJ rows from the even global row at or below the first owned row
    const int jt0 = L.own0 - ((L.own0 + L.jg0) & 1);
    const int ntx = (L.n1 + TI - 1) / TI, nty = (L.own1 - jt0 + TJ - 1) / TJ;
    g_launches += 1;
    const int grid = std::min(ntx * nty, nsm);   // persistent: one CTA per SM
    if (partial)
        gs_fused_kernel<true><<<grid, THREADS, SMEM_RES, st>>>(L, coef, lin, lout, f, jt0, ntx,
                                                               ntx * nty, partial);
    else
        gs_fused_kernel<false><<<grid, THREADS, SMEM, st>>>(L, coef, lin, lout, f, jt0, ntx,
                                                            ntx * nty, nullptr);
    return grid;
}

}  // namespace wd
