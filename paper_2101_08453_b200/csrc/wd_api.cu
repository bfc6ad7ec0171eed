// wd_api.cu -- the C ABI (include/wd.h): context, host planner, V-cycle
// driver and solve loop on top of the sm_100a kernels.
//
// Host-side work is control only: argument checks, the coarsening plan
// (PAPER.md P:192-202 applied to a handful of spacings), launch sequencing,
// CUDA-graph capture of the V-cycle and the convergence test on one scalar
// per cycle.  Every array operation of the path runs in the kernels of
// k_fe.cu, k_mg.cu and k_coarse.cu.
#include "../../include/wd.h"
#include "wd_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

using namespace wd;

namespace {

thread_local char g_err[1024] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            int code_ = (e_ == cudaErrorMemoryAllocation) ? WD_E_OOM : WD_E_CUDA;              \
            return fail(code_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                             \
        }                                                                                      \
    } while (0)

#define CKL()                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = cudaGetLastError();                                                   \
        if (e_ != cudaSuccess)                                                                 \
            return fail(WD_E_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                   \
    } while (0)

constexpr int MAXLEV = 32;
constexpr int MAXNZ = 512;

LevDev make_level(int n1, int n2, int n3) {
    LevDev L;
    L.n1 = n1;
    L.n2 = n2;
    L.n3 = n3;
    int half = (n1 + 1) / 2;
    L.H = std::max((half + 15) / 16 * 16, 48);   // >= the TMA box width (34)
    L.P = 2 * L.H;
    L.sk = L.P;
    L.sj = (i64)n3 * L.P;
    L.NT = (i64)n2 * L.sj;
    return L;
}

i64 level_free(const LevDev& L) { return (i64)(L.n1 - 2) * (L.n2 - 2) * (L.n3 - 1); }

struct Level {
    LevDev L;
    double* coef = nullptr;   // 14 * NT
    double* lam = nullptr;
    double* f = nullptr;
    double* r = nullptr;
    double* raw[4] = {nullptr, nullptr, nullptr, nullptr};   // allocations (with front guard)
    // transition to level + 1
    int hflag = 0;
    int nkept = 0;
    int kept[MAXNZ];
    int* dmap = nullptr;      // device: lo/co/pos for 3 directions
    MapDev M;
    // TMA tensor maps (CUtensorMap, 128 B each): coefficient slots 0-4 and 5-13,
    // x = lam (halo box) and f (tile box) of this level
    alignas(64) unsigned char tmA[128], tmB[128], tmX[128], tmF[128];
};

// residual r = f - K lam (f_on) or r = K lam on level `lv`; optional per-CTA partials
int apply_level(Level& lv, bool f_on, double* partial, cudaStream_t st) {
    if (g_apply_variant >= 0)
        return launch_apply_tma(lv.L, lv.tmA, lv.tmB, lv.tmX, f_on ? lv.tmF : nullptr, lv.r,
                                partial, st);
    return launch_apply(lv.L, lv.coef, lv.lam, f_on ? lv.f : nullptr, lv.r, partial, st);
}

}  // namespace

struct wd_ctx {
    int n1, n2, n3;
    double a[3], c[3];
    wd_options opt;
    double *X = nullptr, *Y = nullptr, *Z = nullptr;
    int nlev = 0;
    Level lev[MAXLEV];
    int coarse_direct = 0;
    int nf = 0;
    double* Ainv = nullptr;
    double* Dinv = nullptr;
    double* partial = nullptr;
    int npartial = 0;
    double* dscal = nullptr;    // device scalars
    double* hscal = nullptr;    // pinned host scalars
    cudaStream_t cap = nullptr; // capture stream
    cudaGraphExec_t vgraph = nullptr;
    long long bytes = 0;
    std::vector<std::pair<void*, size_t>> pool;   // staging buffers for host pointers
    std::vector<int> pool_busy;
    long long graph_kernels = 0;                  // kernel nodes of the V-cycle graph
    // profiling (opt.profile): events around level-0 sweeps, the V-cycle, the residual
    cudaEvent_t ev_gs[32] = {};
    cudaEvent_t ev_cyc[2] = {};
    cudaEvent_t ev_res[2] = {};
    double prof[6] = {0, 0, 0, 0, 0, 0};
};

namespace wd {
std::atomic<long long> g_launches{0};
int g_apply_variant = 1;
}

namespace {

// Device allocations come from the device's default stream-ordered memory pool
// with an unlimited release threshold, so a context built after another one
// was destroyed reuses the retained memory instead of remapping it.
void ensure_pool() {
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[dev] = true;
}

int dalloc(wd_ctx* ctx, void** p, size_t bytes) {
    ensure_pool();
    const size_t b = bytes > 0 ? bytes : 8;
    cudaError_t e = cudaMallocAsync(p, b, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? WD_E_OOM : WD_E_CUDA,
                    "cudaMallocAsync(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
    if (ctx) ctx->bytes += (long long)bytes;
    e = cudaMemsetAsync(*p, 0, b, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) return fail(WD_E_CUDA, "cudaMemset failed: %s", cudaGetErrorString(e));
    return WD_OK;
}

void dfree(void* p) {
    if (p) cudaFreeAsync(p, 0);
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Staging of host arrays through device memory (pooled per context).
struct Stage {
    wd_ctx* ctx = nullptr;
    int slot = -1;
    void* own = nullptr;
    double* d = nullptr;
    const void* host = nullptr;
    size_t bytes = 0;
    bool out = false;
    bool staged = false;
};

int stage_acquire(wd_ctx* ctx, Stage& s, size_t bytes) {
    if (ctx) {
        for (size_t t = 0; t < ctx->pool.size(); t++)
            if (!ctx->pool_busy[t] && ctx->pool[t].second >= bytes) {
                ctx->pool_busy[t] = 1;
                s.slot = (int)t;
                s.d = (double*)ctx->pool[t].first;
                return WD_OK;
            }
        void* p;
        int rc = dalloc(nullptr, &p, bytes);
        if (rc) return rc;
        ctx->pool.push_back({p, bytes});
        ctx->pool_busy.push_back(1);
        s.slot = (int)ctx->pool.size() - 1;
        s.d = (double*)p;
        return WD_OK;
    }
    int rc = dalloc(nullptr, &s.own, bytes);
    s.d = (double*)s.own;
    return rc;
}

int stage_in(wd_ctx* ctx, Stage& s, const double* p, size_t n, cudaStream_t st) {
    s.ctx = ctx;
    s.bytes = n * sizeof(double);
    if (is_device_ptr(p)) {
        s.d = const_cast<double*>(p);
        return WD_OK;
    }
    s.staged = true;
    int rc = stage_acquire(ctx, s, s.bytes);
    if (rc) return rc;
    CK(cudaMemcpyAsync(s.d, p, s.bytes, cudaMemcpyHostToDevice, st));
    return WD_OK;
}

int stage_out(wd_ctx* ctx, Stage& s, double* p, size_t n) {
    s.ctx = ctx;
    s.bytes = n * sizeof(double);
    s.out = true;
    s.host = p;
    if (is_device_ptr(p)) {
        s.d = p;
        return WD_OK;
    }
    s.staged = true;
    return stage_acquire(ctx, s, s.bytes);
}

// finish: copy staged outputs back, synchronise if anything was staged, release
int stage_finish(cudaStream_t st, std::initializer_list<Stage*> list) {
    bool any = false;
    for (Stage* s : list) {
        if (s->staged && s->out)
            CK(cudaMemcpyAsync(const_cast<void*>(s->host), s->d, s->bytes, cudaMemcpyDeviceToHost, st));
        any |= s->staged;
    }
    if (any) CK(cudaStreamSynchronize(st));
    for (Stage* s : list) {
        if (!s->staged) continue;
        if (s->ctx && s->slot >= 0) s->ctx->pool_busy[s->slot] = 0;
        if (s->own) dfree(s->own);
        s->staged = false;
    }
    return WD_OK;
}

// ------------------------------------------------------------------ planner
// Ratio of the paper's tests with a1 = a2 normalised to 1 by
// dividing a3 by sqrt(a1 a2) (reading C2).  VERBATIM: h3/(h1 a3) as printed;
// COUPLING (reading C1): (h3/h1) a3, the same test through the coupling
// strength of Eq. (4) whose vertical coefficient is a3^-2.
double plan_rho(double h3, double h1, double a3n, int rule) {
    if (rule == WD_RULE_VERBATIM) return h3 / (h1 * a3n);
    return (h3 / h1) * a3n;
}

// One planning step: horizontal iff rho(h3[0], h1) > 1/3 (needs
// n1, n2 >= 4); then from the ground up, from kept layer k: drop layer k+1 if
// k+1 < nz and rho(h3[k], h1v) < 3, with h1v the current h1 (COUPLING_CUR,
// reading C1b) or the coarsened one (COUPLING_PAPER, VERBATIM).
bool plan_level(double h1, const double* h3, int nz, const double a[3], int rule, int n1, int n2,
                int* hflag, int* kept, int* nkept, double* h1n, double* h3n) {
    const double a3n = a[2] / std::sqrt(a[0] * a[1]);
    int hz = rule == WD_RULE_FULL ? 1 : (plan_rho(h3[0], h1, a3n, rule) > 1.0 / 3.0);
    if (n1 < 4 || n2 < 4) hz = 0;
    const double h1p = hz ? 2.0 * h1 : h1;
    const double h1v = rule == WD_RULE_COUPLING_CUR ? h1 : h1p;
    int nk = 0, k = 0;
    kept[nk++] = 0;
    while (k < nz) {
        bool merge = (k + 1 < nz) &&
                     (rule == WD_RULE_FULL || plan_rho(h3[k], h1v, a3n, rule) < 3.0);
        k = merge ? k + 2 : k + 1;
        kept[nk++] = k;
    }
    *nkept = nk;
    for (int t = 0; t + 1 < nk; t++) {
        double s = 0.0;
        for (int q = kept[t]; q < kept[t + 1]; q++) s += h3[q];
        h3n[t] = s;
    }
    *hflag = hz;
    *h1n = h1p;
    return hz || (nk - 1 < nz);
}

// per-direction maps of the index-space prolongation (C4, C5)
void map1d(int n, const int* pos, int m, int* lo, int* co) {
    int c = 0;
    for (int t = 0; t < n; t++) {
        while (c + 1 < m && pos[c + 1] <= t) c++;
        lo[t] = c;
        co[t] = pos[c] == t;
    }
}

int horiz_kept(int n, int* pos) {
    int m = 0;
    for (int t = 0; t < n; t += 2) pos[m++] = t;
    if (pos[m - 1] != n - 1) pos[m++] = n - 1;
    return m;
}

int alloc_level(wd_ctx* ctx, Level& lv, int n1, int n2, int n3) {
    lv.L = make_level(n1, n2, n3);
    const size_t nt = (size_t)lv.L.NT;
    int rc;
    const size_t g = 0;   // front guard (doubles) before each array
    double** arr[4] = {&lv.coef, &lv.lam, &lv.f, &lv.r};
    const size_t len[4] = {14 * nt, nt, nt, nt};
    for (int t = 0; t < 4; t++) {
        if ((rc = dalloc(ctx, (void**)&lv.raw[t], sizeof(double) * (len[t] + g)))) return rc;
        *arr[t] = lv.raw[t] + g;
    }
    if (make_coef_maps(lv.L, lv.coef, lv.tmA, lv.tmB) || make_vec_map(lv.L, lv.lam, lv.tmX, true) ||
        make_vec_map(lv.L, lv.f, lv.tmF, false))
        return fail(WD_E_CUDA, "cuTensorMapEncodeTiled failed for level dims (%d,%d,%d)", n1, n2, n3);
    return WD_OK;
}

// ------------------------------------------------------------------ V-cycle
int coarse_solve(wd_ctx* ctx, cudaStream_t st) {
    Level& lc = ctx->lev[ctx->nlev - 1];
    if (ctx->coarse_direct) {
        if (ctx->nf > 0) launch_coarse_gemv(lc.L, ctx->Ainv, ctx->nf, lc.f, lc.lam, st);
    } else {
        CK(cudaMemsetAsync(lc.lam, 0, sizeof(double) * lc.L.NT, st));
        for (int s = 0; s < ctx->opt.coarse_iters; s++) launch_gs_sweep(lc.L, lc.coef, lc.lam, lc.f, st);
    }
    CKL();
    return WD_OK;
}

int vcycle_level(wd_ctx* ctx, int l, cudaStream_t st) {
    if (l == ctx->nlev - 1) return coarse_solve(ctx, st);
    Level& F = ctx->lev[l];
    Level& C = ctx->lev[l + 1];
    const bool prof = ctx->opt.profile && l == 0;
    int ns = 0;
    for (int s = 0; s < ctx->opt.pre_smooth; s++, ns++) {
        if (prof && ns < 16) CK(cudaEventRecordWithFlags(ctx->ev_gs[2 * ns], st, cudaEventRecordExternal));
        launch_gs_sweep(F.L, F.coef, F.lam, F.f, st);
        if (prof && ns < 16) CK(cudaEventRecordWithFlags(ctx->ev_gs[2 * ns + 1], st, cudaEventRecordExternal));
    }
    apply_level(F, true, nullptr, st);
    launch_restrict(F.L, C.L, F.M, F.r, C.f, st);
    CK(cudaMemsetAsync(C.lam, 0, sizeof(double) * C.L.NT, st));
    CKL();
    int rc = vcycle_level(ctx, l + 1, st);
    if (rc) return rc;
    launch_prolong(F.L, C.L, F.M, C.lam, F.lam, st);
    for (int s = 0; s < ctx->opt.post_smooth; s++, ns++) {
        if (prof && ns < 16) CK(cudaEventRecordWithFlags(ctx->ev_gs[2 * ns], st, cudaEventRecordExternal));
        launch_gs_sweep(F.L, F.coef, F.lam, F.f, st);
        if (prof && ns < 16) CK(cudaEventRecordWithFlags(ctx->ev_gs[2 * ns + 1], st, cudaEventRecordExternal));
    }
    CKL();
    return WD_OK;
}

// after a synchronisation: add the elapsed times of the last V-cycle / residual
void profile_accumulate(wd_ctx* ctx, bool cycle, bool resid) {
    if (!ctx->opt.profile) return;
    float ms;
    if (cycle) {
        const int ns = std::min(ctx->opt.pre_smooth + ctx->opt.post_smooth, 16);
        if (ctx->nlev > 1)
            for (int s = 0; s < ns; s++)
                if (cudaEventElapsedTime(&ms, ctx->ev_gs[2 * s], ctx->ev_gs[2 * s + 1]) == cudaSuccess) {
                    ctx->prof[0] += ms;
                    ctx->prof[1] += 1;
                }
        if (cudaEventElapsedTime(&ms, ctx->ev_cyc[0], ctx->ev_cyc[1]) == cudaSuccess) {
            ctx->prof[2] += ms;
            ctx->prof[3] += 1;
        }
    }
    if (resid && cudaEventElapsedTime(&ms, ctx->ev_res[0], ctx->ev_res[1]) == cudaSuccess) {
        ctx->prof[4] += ms;
        ctx->prof[5] += 1;
    }
    cudaGetLastError();
}

// one V-cycle on the internal level-0 vectors, optionally through a CUDA graph
int run_vcycle(wd_ctx* ctx, cudaStream_t st) {
    if (ctx->opt.profile) CK(cudaEventRecord(ctx->ev_cyc[0], st));
    if (!ctx->opt.use_graph) {
        int rc = vcycle_level(ctx, 0, st);
        if (rc) return rc;
    } else {
        if (!ctx->vgraph) {
            const long long before = g_launches.load();
            CK(cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal));
            int rc = vcycle_level(ctx, 0, ctx->cap);
            cudaGraph_t g;
            cudaError_t e = cudaStreamEndCapture(ctx->cap, &g);
            ctx->graph_kernels = g_launches.load() - before;
            g_launches -= ctx->graph_kernels;   // captured, not executed
            if (rc) return rc;
            if (e != cudaSuccess) return fail(WD_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
            e = cudaGraphInstantiate(&ctx->vgraph, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) return fail(WD_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
        }
        CK(cudaGraphLaunch(ctx->vgraph, st));
        g_launches += ctx->graph_kernels;
    }
    if (ctx->opt.profile) CK(cudaEventRecord(ctx->ev_cyc[1], st));
    return WD_OK;
}

// ||f - K lam||^2 of level 0 into dscal[slot] (device), stream-ordered
int residual_sq(wd_ctx* ctx, int slot, cudaStream_t st) {
    Level& F = ctx->lev[0];
    if (ctx->opt.profile) CK(cudaEventRecord(ctx->ev_res[0], st));
    int nb = apply_level(F, true, ctx->partial, st);
    launch_reduce_sum(ctx->partial, nb, ctx->dscal + slot, st);
    if (ctx->opt.profile) CK(cudaEventRecord(ctx->ev_res[1], st));
    CKL();
    return WD_OK;
}

int norm_sq(wd_ctx* ctx, const LevDev& L, const double* v, int slot, cudaStream_t st) {
    int nb;
    launch_norm2_partial(L, v, ctx->partial, &nb, st);
    launch_reduce_sum(ctx->partial, nb, ctx->dscal + slot, st);
    CKL();
    return WD_OK;
}

int fetch_scalars(wd_ctx* ctx, int n, cudaStream_t st) {
    CK(cudaMemcpyAsync(ctx->hscal, ctx->dscal, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return WD_OK;
}

int check_level(const wd_ctx* ctx, int level) {
    if (!ctx) return fail(WD_E_INVAL, "NULL context");
    if (level < 0 || level >= ctx->nlev) return fail(WD_E_INVAL, "level %d out of range", level);
    return WD_OK;
}

size_t nodes_of(const LevDev& L) { return (size_t)L.n1 * L.n2 * L.n3; }

}  // namespace

extern "C" {

void wd_default_options(wd_options* o) {
    memset(o, 0, sizeof *o);
    o->pre_smooth = 2;
    o->post_smooth = 2;
    o->max_cycles = 100;
    o->coarsest_max_free = 4096;
    o->coarse_iters = 50;
    o->coarsen_rule = WD_RULE_COUPLING_CUR;
    o->use_graph = 1;
    o->rank = 0;
    o->nranks = 1;
}

const char* wd_last_error(void) { return g_err; }

void wd_destroy(wd_ctx* ctx) {
    if (!ctx) return;
    cudaDeviceSynchronize();   // no work of the context may still be in flight
    cudaGetLastError();
    if (ctx->vgraph) cudaGraphExecDestroy(ctx->vgraph);
    if (ctx->cap) cudaStreamDestroy(ctx->cap);
    for (auto e : ctx->ev_gs) if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_cyc) if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_res) if (e) cudaEventDestroy(e);
    for (int l = 0; l < ctx->nlev; l++) {
        Level& lv = ctx->lev[l];
        for (double* p : lv.raw) dfree(p);
        dfree(lv.dmap);
    }
    dfree(ctx->X);
    dfree(ctx->Y);
    dfree(ctx->Z);
    dfree(ctx->Ainv);
    dfree(ctx->Dinv);
    dfree(ctx->partial);
    dfree(ctx->dscal);
    if (ctx->hscal) cudaFreeHost(ctx->hscal);
    for (auto& p : ctx->pool) dfree(p.first);
    delete ctx;
}

long long wd_device_bytes(const wd_ctx* ctx) { return ctx ? ctx->bytes : 0; }

static int assemble_impl(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                         double a1, double a2, double a3, const wd_options* opt,
                         cudaStream_t st, wd_ctx* ctx) {
    int rc;
    ctx->n1 = n1;
    ctx->n2 = n2;
    ctx->n3 = n3;
    ctx->a[0] = a1;
    ctx->a[1] = a2;
    ctx->a[2] = a3;
    for (int d = 0; d < 3; d++) ctx->c[d] = 1.0 / (ctx->a[d] * ctx->a[d]);
    if (opt) ctx->opt = *opt;
    else wd_default_options(&ctx->opt);
    const size_t N = (size_t)n1 * n2 * n3;
    // internal copies of the coordinates (natural layout)
    Stage sx, sy, sz;
    if ((rc = stage_in(nullptr, sx, X, N, st)) || (rc = stage_in(nullptr, sy, Y, N, st)) ||
        (rc = stage_in(nullptr, sz, Z, N, st)))
        return rc;
    if ((rc = dalloc(ctx, (void**)&ctx->X, sizeof(double) * N))) return rc;
    if ((rc = dalloc(ctx, (void**)&ctx->Y, sizeof(double) * N))) return rc;
    if ((rc = dalloc(ctx, (void**)&ctx->Z, sizeof(double) * N))) return rc;
    CK(cudaMemcpyAsync(ctx->X, sx.d, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->Y, sy.d, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->Z, sz.d, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    if ((rc = stage_finish(st, {&sx, &sy, &sz}))) return rc;

    if ((rc = dalloc(ctx, (void**)&ctx->dscal, sizeof(double) * 4096))) return rc;
    CK(cudaMallocHost((void**)&ctx->hscal, sizeof(double) * 64));
    CK(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
    apply_tma_prepare();
    if (ctx->opt.profile) {
        for (auto& e : ctx->ev_gs) CK(cudaEventCreate(&e));
        for (auto& e : ctx->ev_cyc) CK(cudaEventCreate(&e));
        for (auto& e : ctx->ev_res) CK(cudaEventCreate(&e));
    }

    // level 0: assembly fused with validation
    Level& L0 = ctx->lev[0];
    if ((rc = alloc_level(ctx, L0, n1, n2, n3))) return rc;
    ctx->nlev = 1;
    unsigned long long* dbad = (unsigned long long*)ctx->dscal;
    CK(cudaMemsetAsync(dbad, 0xff, sizeof(unsigned long long), st));
    launch_assemble(ctx->X, ctx->Y, ctx->Z, n1, n2, n3, ctx->c, L0.L, L0.coef, dbad, st);
    CKL();
    unsigned long long hbad;
    CK(cudaMemcpyAsync(&hbad, dbad, sizeof hbad, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hbad != ~0ull) {
        const unsigned long long e = hbad / 16, what = hbad % 16;
        const int nx = n1 - 1, ny = n2 - 1;
        const int ei = (int)(e % nx), ej = (int)((e / nx) % ny), ek = (int)(e / ((unsigned long long)nx * ny));
        if (what == 0)
            return fail(WD_E_MESH, "element (%d,%d,%d): Z not increasing in k", ei, ej, ek);
        return fail(WD_E_MESH, "element (%d,%d,%d): detJ <= 0 at Gauss point %d", ei, ej, ek,
                    (int)what - 1);
    }

    // planner inputs (reading C2): h1 = sqrt(dx dy); h3 at the column of minimum Z(i,j,0)
    double h[2], org[2];
    CK(cudaMemcpy(&org[0], ctx->X, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&h[0], ctx->X + 1, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&org[1], ctx->Y, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&h[1], ctx->Y + n1, sizeof(double), cudaMemcpyDeviceToHost));
    double h1 = std::sqrt((h[0] - org[0]) * (h[1] - org[1]));
    {
        const int nblk = 256;
        double* pval = ctx->dscal + 16;
        long long* pidx = (long long*)(ctx->dscal + 16 + 2 * (nblk + 1));
        launch_argmin_bottom(ctx->Z, n1 * n2, pval, pidx, nblk, st);
        CKL();
        long long best;
        CK(cudaMemcpyAsync(&best, pidx + nblk, sizeof best, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<double> zc(n3);
        for (int k = 0; k < n3; k++)
            CK(cudaMemcpy(&zc[k], ctx->Z + (size_t)k * n1 * n2 + best, sizeof(double),
                          cudaMemcpyDeviceToHost));
        double h3[MAXNZ], h3n[MAXNZ], h1n;
        for (int k = 0; k + 1 < n3; k++) h3[k] = zc[k + 1] - zc[k];
        // hierarchy
        while (ctx->nlev < MAXLEV) {
            Level& F = ctx->lev[ctx->nlev - 1];
            if (level_free(F.L) <= ctx->opt.coarsest_max_free) break;
            int hflag;
            if (!plan_level(h1, h3, F.L.n3 - 1, ctx->a, ctx->opt.coarsen_rule, F.L.n1, F.L.n2,
                            &hflag, F.kept, &F.nkept, &h1n, h3n))
                break;
            F.hflag = hflag;
            std::vector<int> px(F.L.n1), py(F.L.n2);
            int m1, m2;
            if (hflag) {
                m1 = horiz_kept(F.L.n1, px.data());
                m2 = horiz_kept(F.L.n2, py.data());
            } else {
                m1 = F.L.n1;
                m2 = F.L.n2;
                for (int t = 0; t < m1; t++) px[t] = t;
                for (int t = 0; t < m2; t++) py[t] = t;
            }
            const int nd[3] = {F.L.n1, F.L.n2, F.L.n3};
            const int md[3] = {m1, m2, F.nkept};
            const int* pos[3] = {px.data(), py.data(), F.kept};
            size_t tot = 0;
            for (int d = 0; d < 3; d++) tot += 2 * nd[d] + md[d];
            std::vector<int> hmap(tot);
            size_t offs[3][3], o = 0;
            for (int d = 0; d < 3; d++) {
                offs[d][0] = o;
                offs[d][1] = o + nd[d];
                offs[d][2] = o + 2 * nd[d];
                map1d(nd[d], pos[d], md[d], &hmap[o], &hmap[o + nd[d]]);
                for (int c = 0; c < md[d]; c++) hmap[o + 2 * nd[d] + c] = pos[d][c];
                o += 2 * nd[d] + md[d];
            }
            if ((rc = dalloc(ctx, (void**)&F.dmap, sizeof(int) * tot))) return rc;
            CK(cudaMemcpy(F.dmap, hmap.data(), sizeof(int) * tot, cudaMemcpyHostToDevice));
            for (int d = 0; d < 3; d++) {
                F.M.lo[d] = F.dmap + offs[d][0];
                F.M.co[d] = F.dmap + offs[d][1];
                F.M.pos[d] = F.dmap + offs[d][2];
            }
            Level& C = ctx->lev[ctx->nlev];
            if ((rc = alloc_level(ctx, C, m1, m2, F.nkept))) return rc;
            ctx->nlev++;
            launch_galerkin(F.L, C.L, F.M, F.coef, C.coef, nullptr, st);
            CKL();
            h1 = h1n;
            for (int t = 0; t + 1 < F.nkept; t++) h3[t] = h3n[t];
        }
    }
    // coarsest level (reading C8)
    Level& Lc = ctx->lev[ctx->nlev - 1];
    const i64 nf = level_free(Lc.L);
    ctx->nf = (int)nf;
    ctx->coarse_direct = nf <= ctx->opt.coarsest_max_free;
    if (ctx->coarse_direct && nf > 0) {
        if ((rc = dalloc(ctx, (void**)&ctx->Ainv, sizeof(double) * (size_t)nf * nf))) return rc;
        if ((rc = dalloc(ctx, (void**)&ctx->Dinv, sizeof(double) * 32 * 32))) return rc;
        coarse_prepare((int)nf);
        launch_dense_build(Lc.L, Lc.coef, ctx->Ainv, (int)nf, st);
        gj_invert(ctx->Ainv, (int)nf, ctx->Dinv, st);
        CKL();
    }
    // partial-sum scratch: enough for the apply grid of level 0 and the norm kernel
    {
        const LevDev& L = L0.L;
        ctx->npartial = ((L.n1 + 1) / 2 + 127) / 128 * L.n2 * 2 + 2048;
        if ((rc = dalloc(ctx, (void**)&ctx->partial, sizeof(double) * ctx->npartial))) return rc;
    }
    CK(cudaStreamSynchronize(st));
    CKL();
    return WD_OK;
}

int wd_assemble(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                double a1, double a2, double a3, const wd_options* opt, void* stream,
                wd_ctx** out) {
    if (!out) return fail(WD_E_INVAL, "out is NULL");
    *out = nullptr;
    if (const char* v = getenv("WD_APPLY_VARIANT")) g_apply_variant = atoi(v);
    if (const char* v = getenv("WD_TMA_DEBUG")) g_tma_debug = atoi(v);
    if (!X || !Y || !Z) return fail(WD_E_INVAL, "NULL coordinate array");
    if (n1 < 3 || n2 < 3 || n3 < 2) return fail(WD_E_INVAL, "dims (%d,%d,%d): need n1,n2 >= 3, n3 >= 2", n1, n2, n3);
    if (n3 - 1 >= MAXNZ) return fail(WD_E_INVAL, "n3 = %d exceeds %d", n3, MAXNZ);
    if (!(a1 > 0 && a2 > 0 && a3 > 0) || !std::isfinite(a1) || !std::isfinite(a2) || !std::isfinite(a3))
        return fail(WD_E_INVAL, "penalty constants must be positive and finite");
    if (opt && (opt->pre_smooth < 0 || opt->post_smooth < 0 || opt->max_cycles < 0 ||
                opt->coarsen_rule < 0 || opt->coarsen_rule > 3 || opt->coarse_iters < 0))
        return fail(WD_E_INVAL, "invalid options");
    if (opt && opt->coarsest_max_free > 8192)
        return fail(WD_E_INVAL, "coarsest_max_free %d > 8192 (dense inverse)", opt->coarsest_max_free);
    wd_ctx* ctx = new wd_ctx();
    int rc = assemble_impl(X, Y, Z, n1, n2, n3, a1, a2, a3, opt, (cudaStream_t)stream, ctx);
    if (rc) {
        char keep[1024];
        memcpy(keep, g_err, sizeof keep);
        cudaStreamSynchronize((cudaStream_t)stream);
        cudaGetLastError();
        wd_destroy(ctx);
        memcpy(g_err, keep, sizeof keep);
        return rc;
    }
    *out = ctx;
    return WD_OK;
}

int wd_rhs(wd_ctx* ctx, const double* u0, double* f, void* stream) {
    if (!ctx || !u0 || !f) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t E = (size_t)(ctx->n1 - 1) * (ctx->n2 - 1) * (ctx->n3 - 1);
    const size_t N = (size_t)ctx->n1 * ctx->n2 * ctx->n3;
    Stage su, sf;
    int rc;
    if ((rc = stage_in(ctx, su, u0, 3 * E, st)) || (rc = stage_out(ctx, sf, f, N))) return rc;
    launch_rhs(ctx->X, ctx->Y, ctx->Z, ctx->n1, ctx->n2, ctx->n3, su.d, sf.d, st);
    CKL();
    return stage_finish(st, {&su, &sf});
}

int wd_recover_wind(wd_ctx* ctx, const double* lambda, const double* u0, double* u, void* stream) {
    if (!ctx || !lambda || !u0 || !u) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t E = (size_t)(ctx->n1 - 1) * (ctx->n2 - 1) * (ctx->n3 - 1);
    const size_t N = (size_t)ctx->n1 * ctx->n2 * ctx->n3;
    Stage sl, su0, su;
    int rc;
    if ((rc = stage_in(ctx, sl, lambda, N, st)) || (rc = stage_in(ctx, su0, u0, 3 * E, st)) ||
        (rc = stage_out(ctx, su, u, 3 * E)))
        return rc;
    launch_recover(ctx->X, ctx->Y, ctx->Z, ctx->n1, ctx->n2, ctx->n3, ctx->c, sl.d, su0.d, su.d, st);
    CKL();
    return stage_finish(st, {&sl, &su0, &su});
}

int wd_vcycle(wd_ctx* ctx, double* lambda, const double* f, double* rel_res_out, void* stream) {
    if (!ctx || !lambda || !f) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Level& F = ctx->lev[0];
    const size_t N = nodes_of(F.L);
    Stage sl, sf, so;
    int rc;
    if ((rc = stage_in(ctx, sl, lambda, N, st)) || (rc = stage_in(ctx, sf, f, N, st))) return rc;
    launch_nat2int(F.L, sf.d, F.f, true, st);
    launch_nat2int(F.L, sl.d, F.lam, true, st);
    CKL();
    if ((rc = run_vcycle(ctx, st))) return rc;
    if (rel_res_out) {
        if ((rc = residual_sq(ctx, 0, st)) || (rc = norm_sq(ctx, F.L, F.f, 1, st)) ||
            (rc = fetch_scalars(ctx, 2, st)))
            return rc;
        const double a = std::sqrt(ctx->hscal[0]), fn = std::sqrt(ctx->hscal[1]);
        *rel_res_out = fn > 0 ? a / fn : a;
        profile_accumulate(ctx, true, true);
    }
    // write back (lambda may be host or device)
    so = sl;
    so.out = true;
    so.host = lambda;
    launch_int2nat(F.L, F.lam, so.d, st);
    CKL();
    rc = stage_finish(st, {&so, &sf});
    return rc;
}

int wd_solve(wd_ctx* ctx, const double* f, const double* lambda0, double rel_tol, double* lambda,
             wd_report* rep, void* stream) {
    if (!ctx || !f || !lambda) return fail(WD_E_INVAL, "NULL argument");
    if (!(rel_tol > 0.0 && rel_tol < 1.0)) return fail(WD_E_INVAL, "rel_tol must be in (0,1)");
    cudaStream_t st = (cudaStream_t)stream;
    Level& F = ctx->lev[0];
    const size_t N = nodes_of(F.L);
    Stage sf, s0, sl;
    int rc;
    if ((rc = stage_in(ctx, sf, f, N, st))) return rc;
    if (lambda0 && (rc = stage_in(ctx, s0, lambda0, N, st))) return rc;
    if ((rc = stage_out(ctx, sl, lambda, N))) return rc;
    launch_nat2int(F.L, sf.d, F.f, true, st);
    if (lambda0) launch_nat2int(F.L, s0.d, F.lam, true, st);
    else CK(cudaMemsetAsync(F.lam, 0, sizeof(double) * F.L.NT, st));
    CKL();
    wd_report R;
    memset(&R, 0, sizeof R);
    R.nlevels = ctx->nlev;
    for (int l = 0; l < ctx->nlev && l < 32; l++) {
        R.dims[l][0] = ctx->lev[l].L.n1;
        R.dims[l][1] = ctx->lev[l].L.n2;
        R.dims[l][2] = ctx->lev[l].L.n3;
    }
    R.coarse_direct = ctx->coarse_direct;
    R.coarse_free = ctx->nf;
    if ((rc = norm_sq(ctx, F.L, F.f, 1, st)) || (rc = residual_sq(ctx, 0, st)) ||
        (rc = fetch_scalars(ctx, 2, st)))
        return rc;
    profile_accumulate(ctx, false, true);
    const double fn = std::sqrt(ctx->hscal[1]);
    int status = WD_E_NOCONV;
    int c = 0;
    if (fn == 0.0) {
        CK(cudaMemsetAsync(F.lam, 0, sizeof(double) * F.L.NT, st));
        R.rel_res_hist[0] = 0.0;
        status = WD_OK;
    } else {
        double rel = std::sqrt(ctx->hscal[0]) / fn;
        R.rel_res_hist[0] = rel;
        R.rel_res0 = rel;
        if (!std::isfinite(rel)) status = WD_E_NONFINITE;
        else if (rel <= rel_tol) status = WD_OK;
        while (status == WD_E_NOCONV && c < ctx->opt.max_cycles) {
            if ((rc = run_vcycle(ctx, st)) || (rc = residual_sq(ctx, 0, st)) ||
                (rc = fetch_scalars(ctx, 1, st)))
                return rc;
            c++;
            profile_accumulate(ctx, true, true);
            rel = std::sqrt(ctx->hscal[0]) / fn;
            if (c < 256) R.rel_res_hist[c] = rel;
            if (!std::isfinite(rel)) { status = WD_E_NONFINITE; break; }
            if (rel <= rel_tol) { status = WD_OK; break; }
            if (c >= 3 && c < 256 && rel > 10.0 * R.rel_res_hist[c - 3]) { status = WD_E_DIVERGED; break; }
        }
    }
    R.cycles = c;
    R.status = status;
    R.converged = status == WD_OK;
    const int ch = c < 255 ? c : 255;
    R.rel_res_final = R.rel_res_hist[ch];
    if (c >= 2) R.rate = std::pow(R.rel_res_hist[ch] / R.rel_res_hist[1], 1.0 / (ch - 1));
    else if (c == 1) R.rate = R.rel_res_hist[1] / R.rel_res_hist[0];
    launch_int2nat(F.L, F.lam, sl.d, st);
    CKL();
    if ((rc = stage_finish(st, {&sf, &s0, &sl}))) return rc;
    if (rep) *rep = R;
    if (status == WD_E_NOCONV) return fail(WD_E_NOCONV, "not converged after %d cycles (rel %.3e)", c, R.rel_res_final);
    if (status == WD_E_DIVERGED) return fail(WD_E_DIVERGED, "diverged at cycle %d", c);
    if (status == WD_E_NONFINITE) return fail(WD_E_NONFINITE, "non-finite residual at cycle %d", c);
    return WD_OK;
}

// ------------------------------------------------------------------ profiling
int wd_profile_read(const wd_ctx* ctx, double* out, int n) {
    if (!ctx || !out) return 0;
    int m = n < 6 ? n : 6;
    for (int t = 0; t < m; t++) out[t] = ctx->prof[t];
    return m;
}

void wd_profile_reset(wd_ctx* ctx) {
    if (ctx)
        for (double& v : ctx->prof) v = 0.0;
}

long long wd_launch_count(void) { return g_launches.load(); }

int wd_bench_kernel(wd_ctx* ctx, int which, int level, int reps, double* ms_out) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    if (reps < 1 || !ms_out) return fail(WD_E_INVAL, "reps < 1 or NULL output");
    if ((which == 2 || which == 3 || which == 6) && level >= ctx->nlev - 1)
        return fail(WD_E_INVAL, "no coarser level");
    cudaStream_t st = ctx->cap;
    Level& F = ctx->lev[level];
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto body = [&]() -> int {
        switch (which) {
            case 0: launch_gs_sweep(F.L, F.coef, F.lam, F.f, st); break;
            case 1: apply_level(F, true, nullptr, st); break;
            case 2: launch_restrict(F.L, ctx->lev[level + 1].L, F.M, F.r, ctx->lev[level + 1].f, st); break;
            case 3: launch_prolong(F.L, ctx->lev[level + 1].L, F.M, ctx->lev[level + 1].lam, F.lam, st); break;
            case 4: return run_vcycle(ctx, st);
            case 5: return residual_sq(ctx, 0, st);
            case 6: launch_galerkin(F.L, ctx->lev[level + 1].L, F.M, F.coef, ctx->lev[level + 1].coef, nullptr, st); break;
            case 7: {
                unsigned long long* dbad = (unsigned long long*)(ctx->dscal + 8);
                launch_assemble(ctx->X, ctx->Y, ctx->Z, ctx->n1, ctx->n2, ctx->n3, ctx->c,
                                ctx->lev[0].L, ctx->lev[0].coef, dbad, st);
                break;
            }
            default: return fail(WD_E_INVAL, "unknown kernel %d", which);
        }
        return WD_OK;
    };
    if ((rc = body())) return rc;   // warm-up
    CK(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; r++)
        if ((rc = body())) return rc;
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CKL();
    return WD_OK;
}

// ------------------------------------------------------------------ inspection
int wd_num_levels(const wd_ctx* ctx) { return ctx ? ctx->nlev : 0; }

int wd_level_dims(const wd_ctx* ctx, int level, int dims[3]) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    dims[0] = ctx->lev[level].L.n1;
    dims[1] = ctx->lev[level].L.n2;
    dims[2] = ctx->lev[level].L.n3;
    return WD_OK;
}

int wd_level_plan(const wd_ctx* ctx, int level, int* horizontal, int* kept, int* nkept) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    if (level >= ctx->nlev - 1) return fail(WD_E_INVAL, "level %d is the coarsest", level);
    *horizontal = ctx->lev[level].hflag;
    *nkept = ctx->lev[level].nkept;
    for (int t = 0; t < ctx->lev[level].nkept; t++) kept[t] = ctx->lev[level].kept[t];
    return WD_OK;
}

int wd_get_stencil(wd_ctx* ctx, int level, double* K27, void* stream) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Level& lv = ctx->lev[level];
    Stage so;
    if ((rc = stage_out(ctx, so, K27, 27 * nodes_of(lv.L)))) return rc;
    launch_export27(lv.L, lv.coef, so.d, st);
    CKL();
    return stage_finish(st, {&so});
}

int wd_apply(wd_ctx* ctx, int level, const double* x, double* y, void* stream) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Level& lv = ctx->lev[level];
    const size_t N = nodes_of(lv.L);
    Stage sx, sy;
    if ((rc = stage_in(ctx, sx, x, N, st)) || (rc = stage_out(ctx, sy, y, N))) return rc;
    launch_nat2int(lv.L, sx.d, lv.lam, true, st);
    CK(cudaMemsetAsync(lv.r, 0, sizeof(double) * lv.L.NT, st));
    apply_level(lv, false, nullptr, st);
    launch_int2nat(lv.L, lv.r, sy.d, st);
    CKL();
    return stage_finish(st, {&sx, &sy});
}

int wd_smooth(wd_ctx* ctx, int level, double* x, const double* f, int sweeps, void* stream) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Level& lv = ctx->lev[level];
    const size_t N = nodes_of(lv.L);
    Stage sx, sf;
    if ((rc = stage_in(ctx, sx, x, N, st)) || (rc = stage_in(ctx, sf, f, N, st))) return rc;
    launch_nat2int(lv.L, sx.d, lv.lam, true, st);
    launch_nat2int(lv.L, sf.d, lv.f, true, st);
    for (int s = 0; s < sweeps; s++) launch_gs_sweep(lv.L, lv.coef, lv.lam, lv.f, st);
    sx.out = true;
    sx.host = x;
    launch_int2nat(lv.L, lv.lam, sx.d, st);
    CKL();
    return stage_finish(st, {&sx, &sf});
}

int wd_restrict(wd_ctx* ctx, int level, const double* r, double* fc, void* stream) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    if (level >= ctx->nlev - 1) return fail(WD_E_INVAL, "no coarser level");
    cudaStream_t st = (cudaStream_t)stream;
    Level& F = ctx->lev[level];
    Level& C = ctx->lev[level + 1];
    Stage sr, sc;
    if ((rc = stage_in(ctx, sr, r, nodes_of(F.L), st)) || (rc = stage_out(ctx, sc, fc, nodes_of(C.L))))
        return rc;
    launch_nat2int(F.L, sr.d, F.r, true, st);
    CK(cudaMemsetAsync(C.f, 0, sizeof(double) * C.L.NT, st));
    launch_restrict(F.L, C.L, F.M, F.r, C.f, st);
    launch_int2nat(C.L, C.f, sc.d, st);
    CKL();
    return stage_finish(st, {&sr, &sc});
}

int wd_prolong(wd_ctx* ctx, int level, const double* xc, double* x, void* stream) {
    int rc = check_level(ctx, level);
    if (rc) return rc;
    if (level >= ctx->nlev - 1) return fail(WD_E_INVAL, "no coarser level");
    cudaStream_t st = (cudaStream_t)stream;
    Level& F = ctx->lev[level];
    Level& C = ctx->lev[level + 1];
    Stage sc, sx;
    if ((rc = stage_in(ctx, sc, xc, nodes_of(C.L), st)) || (rc = stage_in(ctx, sx, x, nodes_of(F.L), st)))
        return rc;
    launch_nat2int(C.L, sc.d, C.lam, true, st);
    launch_nat2int(F.L, sx.d, F.lam, true, st);
    launch_prolong(F.L, C.L, F.M, C.lam, F.lam, st);
    sx.out = true;
    sx.host = x;
    launch_int2nat(F.L, F.lam, sx.d, st);
    CKL();
    return stage_finish(st, {&sc, &sx});
}

int wd_coarse_solve(wd_ctx* ctx, const double* f, double* x, void* stream) {
    if (!ctx || !f || !x) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Level& lc = ctx->lev[ctx->nlev - 1];
    const size_t N = nodes_of(lc.L);
    Stage sf, sx;
    int rc;
    if ((rc = stage_in(ctx, sf, f, N, st)) || (rc = stage_out(ctx, sx, x, N))) return rc;
    launch_nat2int(lc.L, sf.d, lc.f, true, st);
    CK(cudaMemsetAsync(lc.lam, 0, sizeof(double) * lc.L.NT, st));
    if ((rc = coarse_solve(ctx, st))) return rc;
    launch_int2nat(lc.L, lc.lam, sx.d, st);
    CKL();
    return stage_finish(st, {&sf, &sx});
}

int wd_residual_norm(wd_ctx* ctx, const double* x, const double* f, double* abs_out,
                     double* rel_out, void* stream) {
    if (!ctx || !x || !f) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Level& F = ctx->lev[0];
    const size_t N = nodes_of(F.L);
    Stage sx, sf;
    int rc;
    if ((rc = stage_in(ctx, sx, x, N, st)) || (rc = stage_in(ctx, sf, f, N, st))) return rc;
    launch_nat2int(F.L, sx.d, F.lam, true, st);
    launch_nat2int(F.L, sf.d, F.f, true, st);
    CKL();
    if ((rc = residual_sq(ctx, 0, st)) || (rc = norm_sq(ctx, F.L, F.f, 1, st)) ||
        (rc = fetch_scalars(ctx, 2, st)))
        return rc;
    const double a = std::sqrt(ctx->hscal[0]), fn = std::sqrt(ctx->hscal[1]);
    if (abs_out) *abs_out = a;
    if (rel_out) *rel_out = fn > 0 ? a / fn : a;
    return stage_finish(st, {&sx, &sf});
}

}  // extern "C"
