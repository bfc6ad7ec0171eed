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
//   * lambda of the tile (+ halo) lives in a 16-plane shared-memory ring,
//     filled with cp.async five planes ahead; the old iterate is read from one
//     buffer and the new one written to another (ping-pong), so halo reads
//     never see a neighbour CTA's new values;
//   * the 27 couplings, f and the diagonal of a thread's next node are loaded
//     into registers one step ahead (before the barrier); the second use of
//     every stored coefficient (by the node at the other end of the coupling,
//     at most 7 steps later) and the halo recomputation hit L2, so HBM sees
//     the operator about once per sweep (ncu, Paper-scale level 0: 19.7 GB
//     read per sweep against 18.3 GB algorithmic; the four phase launches
//     read ~34 GB).
#include "wd_internal.cuh"

namespace wd {

namespace {

constexpr int HI = 32;              // positions per parity per tile row (TI = 64 columns)
constexpr int TI = 2 * HI;
constexpr int TJ = 8;               // tile rows
constexpr int SW = HI + 4;          // ring positions per parity per row (columns I0-3 .. I0+TI+3)
constexpr int RW = 2 * SW;          // ring doubles per row
constexpr int SH = TJ + 3;          // ring rows J0-1 .. J0+TJ+1
constexpr int PL = RW * SH;         // ring doubles per plane
constexpr int RING = 16;            // planes in the ring (power of 2, >= LA + 8)
constexpr int LAG = 2;              // plane lag between consecutive colours
constexpr int LA = 5;               // lambda planes loaded ahead
// colour regions: rows per colour (B) and halo columns beyond the 32 aligned ones
constexpr int B0 = TJ / 2 + 1, B1 = TJ / 2 + 1, B2 = TJ / 2, B3 = TJ / 2;
constexpr int W0 = B0, W1 = W0 + B1, W2 = W1 + B2, W3 = W2 + B3;   // warp ranges
constexpr int NHALO = 3 * B0 + 2 * B1 + B2;                          // 29 halo columns
constexpr int THREADS = 32 * (W3 + 1);                               // 19 warps
constexpr size_t SMEM = sizeof(double) * PL * RING;
static_assert(NHALO <= 32, "halo columns must fit one warp");

__device__ __forceinline__ void cp_async8(double* s, const double* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// issue the copies of plane p (old iterate) of the tile's lambda region
// (columns I0-3..I0+TI+3, rows J0-1..J0+TJ+1) into its ring slot
__device__ __forceinline__ void load_plane(const LevDev& L, const double* __restrict__ lin,
                                           double* ring, int I0, int J0, int p) {
    double* dst = ring + (p & (RING - 1)) * PL;
    for (int t = threadIdx.x; t < PL; t += THREADS) {
        const int lj = t / RW, r = t - lj * RW;
        const int half = r >= SW, pos = r - half * SW;
        const int li = 2 * pos + half;
        const int i = I0 - 4 + li, j = J0 - 1 + lj;
        if (li >= 1 && i >= 0 && i < L.n1 && j >= 0 && j < L.n2)
            cp_async8(dst + t, lin + loff(L, i, j, p));
    }
}

__global__ void __launch_bounds__(THREADS, 1)
gs_fused_kernel(LevDev L, const double* __restrict__ K, const double* __restrict__ lin,
                double* __restrict__ lout, const double* __restrict__ f, int jt0) {
    extern __shared__ double ring[];
    const int I0 = blockIdx.x * TI;
    const int J0 = jt0 + blockIdx.y * TJ;   // local row of an even global row
    // zero the ring (columns/rows outside the grid stay 0 = never-used values)
    for (int t = threadIdx.x; t < PL * RING; t += THREADS) ring[t] = 0.0;
    __syncthreads();

    // this thread's colour c and column (i, j)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int c, i, j;
    bool inreg = true;
    if (w < W0) { c = 0; j = J0 + 2 * w; i = I0 + 2 * lane; }
    else if (w < W1) { c = 1; j = J0 + 2 * (w - W0); i = I0 + 1 + 2 * lane; }
    else if (w < W2) { c = 2; j = J0 + 1 + 2 * (w - W1); i = I0 + 2 * lane; }
    else if (w < W3) { c = 3; j = J0 + 1 + 2 * (w - W2); i = I0 + 1 + 2 * lane; }
    else if (lane < 3 * B0) {           // colour 0 halo: I0-2, I0+TI, I0+TI+2
        c = 0; j = J0 + 2 * (lane / 3);
        const int e = lane % 3;
        i = e == 0 ? I0 - 2 : I0 + TI + 2 * e - 2;
    } else if (lane < 3 * B0 + 2 * B1) {   // colour 1 halo: I0-1, I0+TI+1
        const int q = lane - 3 * B0;
        c = 1; j = J0 + 2 * (q / 2);
        i = (q % 2) == 0 ? I0 - 1 : I0 + TI + 1;
    } else if (lane < NHALO) {          // colour 2 halo: I0+TI
        const int q = lane - 3 * B0 - 2 * B1;
        c = 2; j = J0 + 1 + 2 * q; i = I0 + TI;
    } else { c = 0; j = J0; i = -10; inreg = false; }
    const int ci = c & 1;
    const bool active = inreg && i >= 1 && i <= L.n1 - 2 && j >= 0 && j < L.n2 && row_free(L, j);
    const bool writes = active && i >= I0 && i < I0 + TI && j >= J0 && j < J0 + TJ;
    const int li = i - I0 + 4, lj = j - J0 + 1;
    const int so = lj * RW + (li & 1) * SW + (li >> 1);
    // offsets of the neighbour column (dx,dy), dx,dy in -1..1, in the ring
    // (smem) and in the i-split layout (global): the column i-1 / i+1 lives
    // in the other parity half
    const int sxm = ci ? -SW : SW - 1, sxp = ci ? 1 - SW : SW;
    const int gxm = ci ? -L.H : L.H - 1, gxp = ci ? 1 - L.H : L.H;
    const int gsj = (int)L.sj;
    auto sc = [&](int dx, int dy) { return dy * RW + (dx < 0 ? sxm : dx > 0 ? sxp : 0); };
    auto co = [&](int dx, int dy) { return dy * gsj + (dx < 0 ? gxm : dx > 0 ? gxp : 0); };
    const i64 own = active ? loff(L, i, j, 0) : 0;
    const i64 NT = L.NT;
    const int nz = L.n3 - 1;   // free planes 0..nz-1 (top plane n3-1 is Dirichlet)

    // lambda planes stream in LA planes ahead, one cp.async group per plane
    for (int p = 0; p < LA; p++) {
        if (p <= L.n3 - 1) load_plane(L, lin, ring, I0, J0, p);
        cp_async_commit();
    }
    cp_async_wait<LA - 2>();   // planes 0, 1
    __syncthreads();

    // couplings (forward kf stored here, backward kb stored at the neighbours),
    // f and the diagonal of the node this thread updates next
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
    if (active && c == 0) load_k(0);

    const int nsteps = nz + LAG * 3;
    for (int s = 0; s < nsteps; s++) {
        if (s + LA <= L.n3 - 1) load_plane(L, lin, ring, I0, J0, s + LA);
        cp_async_commit();
        const int z = s - LAG * c;
        if (active && z >= 0 && z < nz) {
            const double* r1 = ring + ((z + 1) & (RING - 1)) * PL + so;
            const double* r0 = ring + (z & (RING - 1)) * PL + so;
            const double* rm = ring + ((z - 1) & (RING - 1)) * PL + so;
            double acc = 0.0;
            // forward couplings K(p, p + d_s) stored at p  (same order as gs_phase_kernel)
#pragma unroll
            for (int sl = 1; sl < 14; sl++) {
                const int dx = slot_dx(sl), dy = slot_dy(sl), dz = slot_dz(sl);
                acc = fma(kf[sl - 1], (dz ? r1 : r0)[sc(dx, dy)], acc);
            }
            // backward couplings K(p, p - d_s) stored at p - d_s
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
            ring[(z & (RING - 1)) * PL + so] = v;
            if (writes) lout[own + (i64)z * L.sk] = v;
        }
        // next plane's couplings, issued before the barrier that precedes their use
        if (active && z + 1 >= 0 && z + 1 < nz) load_k(z + 1);
        cp_async_wait<LA - 2>();   // planes <= s + 2 (needed by step s + 1)
        __syncthreads();
    }
    cp_async_wait<0>();
}

}  // namespace

// one sweep: lin (old iterate, unchanged) -> lout (new iterate on the owned
// free nodes; D entries of lout must already be 0)
void launch_gs_fused(const LevDev& L, const double* coef, const double* lin, double* lout,
                     const double* f, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gs_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        attr = true;
    }
    // tiles of TJ rows from the even global row at or below the first owned row
    const int jt0 = L.own0 - ((L.own0 + L.jg0) & 1);
    dim3 grid((L.n1 + TI - 1) / TI, (L.own1 - jt0 + TJ - 1) / TJ);
    g_launches += 1;
    gs_fused_kernel<<<grid, THREADS, SMEM, st>>>(L, coef, lin, lout, f, jt0);
}

}  // namespace wd
