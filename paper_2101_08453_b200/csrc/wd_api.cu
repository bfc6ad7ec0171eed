// wd_api.cu -- the C ABI (include/wd.h): context, host planner, slab
// decomposition and transport, V-cycle driver and solve loop on top of the
// sm_100a kernels.
//
// Host-side work is control only: argument checks, the coarsening plan
// (PAPER.md P:192-202 applied to a handful of spacings), the row partition,
// launch sequencing, halo exchanges, CUDA-graph capture of the V-cycle and the
// convergence test on one scalar per cycle.  Every array operation of the path
// runs in the kernels of k_fe.cu, k_mg.cu, k_apply_tma.cu and k_coarse.cu.
//
// Decomposition (requirement (1) of P:39-40): the grid is split
// into slabs of node rows j.  A context holds one "part" per slab it drives:
//   * single GPU:      1 part, the whole grid, no transport;
//   * NCCL (one process per GPU): 1 part (this rank's slab), halo rows are
//     exchanged with ncclSend/ncclRecv, coarse levels gathered by ncclBroadcast;
//   * virtual ranks:   R parts of one grid on one GPU, the same exchanges as
//     device-to-device copies (tests the decomposition logic bit for bit).
// Every part keeps 2 halo rows on each side.  Levels below the gather level
// are distributed; from the gather level on every part holds the whole
// (small) level and computes it redundantly (identical results).
#include "../../include/wd.h"
#include "wd_internal.cuh"

#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <vector>

using namespace wd;

namespace {

thread_local char g_err[1024] = "";

// NVTX range for the lifetime of a scope (ABI calls, solve cycles, and the
// V-cycle phases per level when they are enqueued -- with the CUDA graph that
// is once, at capture; WD_USE_GRAPH-free runs show them on every cycle)
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    Nvtx(const char* fmt, int a) {
        char b[64];
        snprintf(b, sizeof b, fmt, a);
        nvtxRangePushA(b);
    }
    ~Nvtx() { end(); }
    void end() {   // close the range early (once)
        if (on) nvtxRangePop();
        on = false;
    }
    bool on = true;
};

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

// development: WD_SETUP_TIMING=1 prints the setup phases (stream-synchronised)
struct PhaseTimer {
    bool on = false;
    double t0 = 0;
    cudaStream_t st = nullptr;
    static double now() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
    }
    void start(cudaStream_t s) {
        on = getenv("WD_SETUP_TIMING") != nullptr;
        st = s;
        if (on) { cudaStreamSynchronize(st); t0 = now(); }
    }
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const double t = now();
        fprintf(stderr, "[wd setup] %-28s %8.2f ms\n", what, t - t0);
        t0 = t;
    }
};

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

#define RC(x)                \
    do {                     \
        int rc_ = (x);       \
        if (rc_) return rc_; \
    } while (0)

constexpr int MAXLEV = 32;
constexpr int MAXNZ = 512;
constexpr int HALO = 2;          // halo rows of every slab, each side
constexpr int MIN_OWNED = 4;     // fewer owned rows on any rank -> gather

LevDev make_level(int n1, int n2, int n3, int jg0, int n2g, int own0, int own1) {
    LevDev L;
    L.n1 = n1;
    L.n2 = n2;
    L.n3 = n3;
    int half = (n1 + 1) / 2;
    L.H = std::max((half + 15) / 16 * 16, 48);   // >= the TMA box width (36)
    L.P = 2 * L.H;
    L.sk = L.P;
    L.sj = (i64)n3 * L.P;
    L.NT = (i64)n2 * L.sj;
    L.jg0 = jg0;
    L.n2g = n2g;
    L.own0 = own0;
    L.own1 = own1;
    return L;
}

i64 free_count(int n1, int n2, int n3) { return (i64)(n1 - 2) * (n2 - 2) * (n3 - 1); }

struct Level {
    LevDev L;
    bool dist = false;        // distributed (slab) level; else replicated / single
    int cown0 = 0, cown1 = 0; // rows this part computes when restricting / forming K_c into
                              // this level (= owned rows; a slice of the gather level)
    double* coef = nullptr;   // 14 * NT
    double* lam = nullptr;
    double* f = nullptr;
    double* r = nullptr;
    double* lam2 = nullptr;   // second iterate buffer of the fused smoother (ping-pong)
    double* raw[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    // transition to level + 1
    int hflag = 0;
    int nkept = 0;
    int kept[MAXNZ];
    int* dmap = nullptr;      // device: lo/co/pos for 3 directions (y local to the part)
    MapDev M;
    alignas(64) unsigned char tmA[128], tmB[128], tmX[128], tmF[128];
    alignas(64) unsigned char tmR[2][128];   // ring maps of raw[1] and raw[4] (k_gs_fused2.cu)
    alignas(64) unsigned char tmRr[2][128];  // the same for the residual variant's tiles
    alignas(64) unsigned char tmRs[2][128];  // and for the small levels' plain tiles
};

struct Part {
    int rank = 0;
    int jlo = 0, jhi = 0;     // level-0 local rows = global rows [jlo, jhi)
    int own0g = 0, own1g = 0; // owned global rows at level 0
    double *X = nullptr, *Y = nullptr, *Z = nullptr;   // local coordinates (natural layout)
    double* Ainv = nullptr;
    double* Dinv = nullptr;
    double* partial = nullptr;
    int npartial = 0;
    Level lev[MAXLEV];
};

// ------------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*ErrStr)(ncclResult_t);
};

Nccl& nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return n;
#define SYM(f, name) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, name))
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(Bcast, "ncclBroadcast");
    SYM(AllGather, "ncclAllGather");
    SYM(AllReduce, "ncclAllReduce");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(ErrStr, "ncclGetErrorString");
#undef SYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.Send && n.Recv && n.Bcast && n.AllGather &&
           n.AllReduce && n.GroupStart && n.GroupEnd;
    return n;
}

#define NK(call)                                                                               \
    do {                                                                                       \
        ncclResult_t r_ = (call);                                                              \
        if (r_ != ncclSuccess)                                                                 \
            return fail(WD_E_NCCL, "%s failed: %s", #call,                                     \
                        nccl().ErrStr ? nccl().ErrStr(r_) : "nccl error");                     \
    } while (0)

enum { MODE_SINGLE = 0, MODE_NCCL = 1, MODE_VIRTUAL = 2 };

}  // namespace

// wd_solve's cycle-loop state when the loop runs on the device (see
// build_device_loop): the host loop's locals, the report's history and the
// number of times each conditional body ran
struct LoopDev {
    double fn, tol, rel0, rel1, rel_last;
    double ring4[4];
    double hist[256];
    int max_cycles, c, have, first_done, status;
    int n_first_res, n_first, n_res;
};

struct wd_ctx {
    int n1, n2, n3;            // global node dims
    // test / experiment knobs (env, read at wd_assemble): gs_v2, jitter,
    // gs_grid, fuse_prolong, apply_variant -- kept per context
    // and installed by KnobScope at every entry point that launches work, so
    // contexts assembled under different settings keep them (graphs are
    // captured lazily, at the first cycle)
    int knob[5] = {1, 0, 0, 0, 1};
    double a[3], c[3];
    wd_options opt;
    int mode = MODE_SINGLE;
    int nranks = 1, rank = 0;  // this process's rank (NCCL mode)
    ncclComm_t comm = nullptr;
    std::vector<int> own0g, own1g;   // owned level-0 rows of every rank
    // per level, per rank: global rows the rank owns (distributed levels) or
    // contributes before the gather (the gather level)
    std::vector<std::vector<std::pair<int, int>>> rrows;
    std::vector<Part> parts;
    int nlev = 0;
    int gather = MAXLEV;       // first replicated level (multi-rank), MAXLEV if none
    int levdims[MAXLEV][3];    // global node dims per level
    int coarse_direct = 0;
    int nf = 0;
    double* dscal = nullptr;   // device scalars
    double* hscal = nullptr;   // pinned host scalars
    cudaStream_t cap = nullptr;
    // slabs: the halo exchange after a sweep's boundary tiles runs on `side`
    // while the interior tiles run (boundary-first overlap); halo_fresh[l]:
    // level l's iterate already has its 2 halo rows current (host-side state
    // of the launch sequence; reset at every entry point and capture)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool halo_fresh[MAXLEV] = {};
    // host-pointer pipelining (copy-in / compute + copy-out streams, chunk events)
    cudaStream_t pin_s = nullptr, pout_s = nullptr;
    cudaEvent_t pev[17] = {};
    cudaGraphExec_t vgraph = nullptr;
    // wd_solve with the fused smoother: the V-cycle split after its first
    // level-0 sweep; that sweep also returns the residual of its input
    // (k_gs_fused.cu RES), so the convergence test needs no residual pass
    // [1]: the profiling variant, with event records around the level-0
    // sweeps (used on every PROF_EVERY-th cycle when opt.profile is on; the
    // event nodes cost ~6 us each, 23 % of a Small solve if on every cycle)
    cudaGraphExec_t g_first_res[2] = {}, g_first[2] = {}, g_rest[2] = {};
    long long k_first_res[2] = {}, k_first[2] = {}, k_rest[2] = {};
    bool cyc_evented = false;   // the current split cycle uses the profiling variant
    bool prof_on = true;        // vcycle_level may record its profiling events
    // the whole cycle loop as one graph (conditional WHILE node), its kernel
    // counts per body and the device / pinned host copies of its state
    cudaGraphExec_t g_loop = nullptr;
    long long kl_first_res = 0, kl_first = 0, kl_rest = 0, kl_res = 0;
    LoopDev* loopd = nullptr;
    LoopDev* looph = nullptr;
    bool loop_broken = false;   // building the loop graph failed once: host loop
    long long bytes = 0;
    std::vector<std::pair<void*, size_t>> pool;   // staging buffers for host pointers
    std::vector<int> pool_busy;
    long long graph_kernels = 0;
    cudaEvent_t ev_gs[32] = {};
    cudaEvent_t ev_cyc[2] = {};
    // wd_solve's split cycles: the start of cycle c on ev_cs[c & 1] (so that
    // its events can be read one cycle later, while the GPU already runs the
    // next one -- waiting for them at once would idle the GPU every cycle)
    cudaEvent_t ev_cs[2] = {};
    int cyc_par = 0;
    bool pend_rest = false;    // the last split cycle's rest not yet read
    bool pend_rest_sweeps = false;   // ... including its sweep / residual events
    int pend_par = 0;
    bool pend_first = false;   // the last split cycle's first sweep not yet read
    bool pend_first_res = false;
    bool first_res = false;    // the last cycle's first sweep was the residual variant
    cudaEvent_t ev_res[2] = {};
    cudaEvent_t ev_ap[2] = {};   // the level-0 residual before the restriction
    double prof[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    // weight w of the coarse-grid correction lam += w P lam_c: 1 (Eq. (7));
    // env WD_TEST_CORRECTION_WEIGHT sets another value, only so that the tests
    // can drive a cycle to divergence and exercise the WD_E_DIVERGED guard
    double corr_w = 1.0;
};

namespace wd {
std::atomic<long long> g_launches{0};
int g_gs_v2 = 1;
int g_test_jitter = 0, g_test_gs_grid = 0;
int g_fuse_prolong = 0;
int g_apply_variant = 1;
int g_galerkin_generic = 0;
}

namespace {

// ------------------------------------------------------------------ memory
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

// Device allocations come from the stream-ordered pool of the device with an
// unlimited release threshold: a context built after another one was destroyed
// reuses the retained memory instead of remapping it.
// zero = false: the caller overwrites every entry that is ever read (big
// arrays whose zero-fill would cost a pass over HBM)
int dalloc(wd_ctx* ctx, void** p, size_t bytes, bool zero = true) {
    ensure_pool();
    const size_t b = bytes > 0 ? bytes : 8;
    cudaError_t e = cudaMallocAsync(p, b, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? WD_E_OOM : WD_E_CUDA,
                    "cudaMallocAsync(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
    if (ctx) ctx->bytes += (long long)bytes;
    if (zero) e = cudaMemsetAsync(*p, 0, b, 0);
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
// A Stage still holding a buffer when it goes out of scope (an early error
// return before stage_finish) gives the buffer back; nothing is copied out.
struct Stage {
    wd_ctx* ctx = nullptr;
    int slot = -1;
    void* own = nullptr;
    double* d = nullptr;
    const void* host = nullptr;
    size_t bytes = 0;
    bool out = false;
    bool staged = false;
    Stage() = default;
    Stage(const Stage&) = delete;
    Stage& operator=(const Stage&) = delete;
    ~Stage();
};

void stage_release(Stage& s);
Stage::~Stage() { stage_release(*this); }

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
        RC(dalloc(nullptr, &p, bytes));
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
    RC(stage_acquire(ctx, s, s.bytes));
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

// copy staged outputs back, synchronise if anything was staged, release
int stage_finish(cudaStream_t st, std::initializer_list<Stage*> list) {
    bool any = false;
    for (Stage* s : list) {
        if (s->staged && s->out)
            CK(cudaMemcpyAsync(const_cast<void*>(s->host), s->d, s->bytes, cudaMemcpyDeviceToHost, st));
        any |= s->staged;
    }
    if (any) CK(cudaStreamSynchronize(st));
    for (Stage* s : list) stage_release(*s);
    return WD_OK;
}

void stage_release(Stage& s) {
    if (!s.staged) return;
    if (s.ctx && s.slot >= 0) s.ctx->pool_busy[s.slot] = 0;
    if (s.own) dfree(s.own);
    s.own = nullptr;
    s.slot = -1;
    s.staged = false;
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

// rows [a, b) of a fine level -> coarse rows J with pos[J] in [a, b)
void coarse_range(const std::vector<int>& pos, int a, int b, int& c0, int& c1) {
    c0 = (int)(std::lower_bound(pos.begin(), pos.end(), a) - pos.begin());
    c1 = (int)(std::lower_bound(pos.begin(), pos.end(), b) - pos.begin());
}

// ------------------------------------------------------------------ host plan
// The hierarchy and its slab layout, computed on the host from the global
// dims, the options, the row partition and the planner inputs (h1, h3) --
// no device work.  wd_assemble builds exactly this plan (then assembles and
// forms the Galerkin operators on it); wd_plan_decomposition returns it for
// inspection, so the multi-rank layout and the exchange / gather schedule can
// be checked without GPUs (tests/test_dist_plan.py).
struct PartLevel {
    LevDev L;
    bool dist = false;
    int cown0 = 0, cown1 = 0;
};
struct HierPlan {
    int nlev = 0;
    int gather = MAXLEV;
    int dims[MAXLEV][3];
    int hflag[MAXLEV], nkept[MAXLEV];
    int kept[MAXLEV][MAXNZ];
    std::vector<int> px[MAXLEV], py[MAXLEV];   // kept fine positions of transition l -> l+1
    std::vector<std::vector<std::pair<int, int>>> rrows;   // [level][rank] rows owned / computed
    std::vector<std::vector<PartLevel>> part;              // [part][level]
    std::vector<int> own0g, own1g;                         // level-0 owned rows per rank
};

// parts: the ranks whose layout is wanted (all R in virtual mode, this rank
// with NCCL, {0} on one GPU)
int plan_hierarchy(int n1, int n2, int n3, const double a[3], const wd_options& o, int nranks,
                   const std::vector<int>& parts, double h1, const double* h3_in, HierPlan& H) {
    const bool multi = nranks > 1;
    H.own0g.resize(nranks);
    H.own1g.resize(nranks);
    for (int r = 0; r < nranks; r++) wd_partition_rows(n2, nranks, r, &H.own0g[r], &H.own1g[r]);
    for (int r = 0; r < nranks; r++)   // slabs need >= MIN_OWNED rows; one GPU takes any grid
        if (multi && H.own1g[r] - H.own0g[r] < MIN_OWNED)
            return fail(WD_E_INVAL, "rank %d owns %d rows (< %d)", r, H.own1g[r] - H.own0g[r], MIN_OWNED);
    H.part.assign(parts.size(), std::vector<PartLevel>(MAXLEV));
    for (size_t p = 0; p < parts.size(); p++) {
        const int r = parts[p];
        const int jlo = multi ? std::max(H.own0g[r] - HALO, 0) : 0;
        const int jhi = multi ? std::min(H.own1g[r] + HALO, n2) : n2;
        PartLevel& L0 = H.part[p][0];
        L0.L = make_level(n1, jhi - jlo, n3, jlo, n2, H.own0g[r] - jlo, H.own1g[r] - jlo);
        L0.dist = multi;
        L0.cown0 = L0.L.own0;
        L0.cown1 = L0.L.own1;
    }
    H.nlev = 1;
    H.gather = MAXLEV;
    H.dims[0][0] = n1;
    H.dims[0][1] = n2;
    H.dims[0][2] = n3;
    H.rrows.assign(1, std::vector<std::pair<int, int>>(nranks));
    for (int r = 0; r < nranks; r++) H.rrows[0][r] = {H.own0g[r], H.own1g[r]};
    double h3[MAXNZ], h3n[MAXNZ], h1n;
    for (int k = 0; k + 1 < n3; k++) h3[k] = h3_in[k];
    while (H.nlev < MAXLEV) {
        const int l = H.nlev - 1;
        const int fn1 = H.dims[l][0], fn2 = H.dims[l][1], fn3 = H.dims[l][2];
        if (free_count(fn1, fn2, fn3) <= o.coarsest_max_free) break;
        int hflag, nk;
        if (!plan_level(h1, h3, fn3 - 1, a, o.coarsen_rule, fn1, fn2, &hflag, H.kept[l], &nk, &h1n, h3n))
            break;
        std::vector<int>& px = H.px[l];
        std::vector<int>& py = H.py[l];
        px.assign(fn1, 0);
        py.assign(fn2, 0);
        int m1, m2;
        if (hflag) {
            m1 = horiz_kept(fn1, px.data());
            m2 = horiz_kept(fn2, py.data());
        } else {
            m1 = fn1;
            m2 = fn2;
            for (int t = 0; t < m1; t++) px[t] = t;
            for (int t = 0; t < m2; t++) py[t] = t;
        }
        px.resize(m1);
        py.resize(m2);
        H.hflag[l] = hflag;
        H.nkept[l] = nk;
        const int cl = l + 1;
        H.dims[cl][0] = m1;
        H.dims[cl][1] = m2;
        H.dims[cl][2] = nk;
        // gather decision (multi-rank): replicate the coarse level when it is
        // small or when a rank would own fewer than MIN_OWNED rows of it
        bool coarse_dist = false;
        H.rrows.resize(cl + 1);
        H.rrows[cl].resize(nranks);
        for (int r = 0; r < nranks; r++) {
            int c0 = 0, c1 = m2;
            if (l < H.gather) coarse_range(py, H.rrows[l][r].first, H.rrows[l][r].second, c0, c1);
            H.rrows[cl][r] = {c0, c1};
        }
        if (multi && H.gather == MAXLEV) {
            coarse_dist = (long long)m1 * m2 * nk >= o.gather_below_nodes;
            for (int r = 0; r < nranks; r++)
                if (H.rrows[cl][r].second - H.rrows[cl][r].first < MIN_OWNED) coarse_dist = false;
            if (!coarse_dist) H.gather = cl;
        }
        for (size_t p = 0; p < parts.size(); p++) {
            const PartLevel& F = H.part[p][l];
            PartLevel& C = H.part[p][cl];
            // coarse rows this part owns / computes
            int c0, c1;
            coarse_range(py, F.L.jg0 + F.L.own0, F.L.jg0 + F.L.own1, c0, c1);
            if (!F.dist) { c0 = 0; c1 = m2; }   // replicated fine level: everything
            if (coarse_dist) {
                const int jlo_c = std::max(c0 - HALO, 0), jhi_c = std::min(c1 + HALO, m2);
                C.L = make_level(m1, jhi_c - jlo_c, nk, jlo_c, m2, c0 - jlo_c, c1 - jlo_c);
                C.dist = true;
                C.cown0 = C.L.own0;
                C.cown1 = C.L.own1;
            } else {
                C.L = make_level(m1, m2, nk, 0, m2, 0, m2);
                C.dist = false;
                C.cown0 = c0;   // slice this part computes before the gather
                C.cown1 = c1;
            }
        }
        H.nlev++;
        h1 = h1n;
        for (int t = 0; t + 1 < nk; t++) h3[t] = h3n[t];
    }
    return WD_OK;
}

// The messages of a w-row halo exchange of distributed level l for rank r
// (the ncclSend/ncclRecv pairs of exchange(); virtual ranks copy the same
// rows): {peer, send(1)/recv(0), first global row, rows}.
struct HaloMsg { int peer, send, row0, rows; };
std::vector<HaloMsg> halo_msgs(const PartLevel& P, int rank, int nranks, int w) {
    std::vector<HaloMsg> m;
    if (!P.dist) return m;
    const int g0 = P.L.jg0 + P.L.own0, g1 = P.L.jg0 + P.L.own1;
    if (rank > 0) {
        m.push_back({rank - 1, 1, g0, w});
        m.push_back({rank - 1, 0, g0 - w, w});
    }
    if (rank < nranks - 1) {
        m.push_back({rank + 1, 1, g1 - w, w});
        m.push_back({rank + 1, 0, g1, w});
    }
    return m;
}

// galerkin: the coefficients will come from the Galerkin product (free nodes
// only) rather than the assembly (every node); either way the entries the
// writer leaves alone are zeroed here instead of zero-filling all 14 arrays
int alloc_level(wd_ctx* ctx, Level& lv, bool galerkin) {
    const size_t nt = (size_t)lv.L.NT;
    double** arr[5] = {&lv.coef, &lv.lam, &lv.f, &lv.r, &lv.lam2};
    const size_t len[5] = {14 * nt, nt, nt, nt, nt};
    for (int t = 0; t < 5; t++) {
        // the vectors zero-filled (D entries of the ping-pong buffer stay 0:
        // the fused sweep writes free nodes only)
        RC(dalloc(ctx, (void**)&lv.raw[t], sizeof(double) * len[t], t != 0));
        *arr[t] = lv.raw[t];
    }
    launch_zero_unwritten(lv.L, lv.coef, galerkin, 0);
    CK(cudaStreamSynchronize(0));
    if (make_coef_maps(lv.L, lv.coef, lv.tmA, lv.tmB) || make_vec_map(lv.L, lv.lam, lv.tmX, true) ||
        make_vec_map(lv.L, lv.f, lv.tmF, false) || make_ring_map(lv.L, lv.raw[1], lv.tmR[0], 8) ||
        make_ring_map(lv.L, lv.raw[4], lv.tmR[1], 8) ||
        make_ring_map(lv.L, lv.raw[1], lv.tmRr[0], 6) ||
        make_ring_map(lv.L, lv.raw[4], lv.tmRr[1], 6) ||
        make_ring_map(lv.L, lv.raw[1], lv.tmRs[0], 4) ||
        make_ring_map(lv.L, lv.raw[4], lv.tmRs[1], 4))
        return fail(WD_E_CUDA, "cuTensorMapEncodeTiled failed for level dims (%d,%d,%d)", lv.L.n1,
                    lv.L.n2, lv.L.n3);
    return WD_OK;
}

// one fused sweep lam -> lam2 of a level (k_gs_fused2.cu unless disabled or
// the level is too large for 32-bit offsets); partial: also ||f - K lam||^2
bool v2_level(const Level& F) {
    return g_gs_v2 && F.L.NT < (1ll << 31) && (F.lam == F.raw[1] || F.lam == F.raw[4]);
}
int gs_sweep_level(Level& F, cudaStream_t st, double* partial = nullptr,
                   const ProlongIn* pro = nullptr, int tr0 = 0, int tr1 = -1) {
    if (v2_level(F))
    {
        const int b = F.lam == F.raw[1] ? 0 : 1;
        return launch_gs_fused2(F.L, F.coef, F.tmR[b], F.tmRr[b], F.tmRs[b], F.lam2, F.f, st,
                                partial, pro, tr0, tr1);
    }
    return launch_gs_fused(F.L, F.coef, F.lam, F.lam2, F.f, st, partial);
}

// residual r = f - K lam (f_on) or r = K lam on level `lv`; optional per-CTA partials
int apply_level(Level& lv, bool f_on, double* partial, cudaStream_t st) {
    // small levels: the plane-parallel operator kernel (the TMA kernel's
    // persistent tiles are latency-bound there).  Decided on the level's global
    // size, so that every slab and one part take the same kernel (the two sum
    // the stencil in different orders)
    if (g_apply_variant >= 0 && (long long)lv.L.n1 * lv.L.n2g <= APPLY_SMALL_COLS)
        return launch_apply(lv.L, lv.coef, lv.lam, f_on ? lv.f : nullptr, lv.r, partial, st, 4);
    if (g_apply_variant >= 0)
        return launch_apply_tma(lv.L, lv.tmA, lv.tmB, lv.tmX, f_on ? lv.tmF : nullptr, lv.r,
                                partial, st);
    return launch_apply(lv.L, lv.coef, lv.lam, f_on ? lv.f : nullptr, lv.r, partial, st);
}

// level with the compute rows [cown0, cown1) (restriction / Galerkin target)
LevDev target(const Level& lv) {
    LevDev L = lv.L;
    L.own0 = lv.cown0;
    L.own1 = lv.cown1;
    return L;
}

// ------------------------------------------------------------------ transport
enum { ARR_LAM = 0, ARR_R = 1, ARR_COEF = 2, ARR_F = 3, ARR_LAM2 = 4 };

double* arr_of(Level& lv, int which) {
    return which == ARR_LAM ? lv.lam : which == ARR_LAM2 ? lv.lam2 : which == ARR_R ? lv.r
         : which == ARR_F ? lv.f : lv.coef;
}

// Halo exchange of w rows each side on a distributed level: a part's first w
// owned rows go to the upper halo of the rank below, its last w owned rows to
// the lower halo of the rank above (all levels of a row are contiguous).
int exchange(wd_ctx* ctx, int l, int which, int w, cudaStream_t st) {
    if (ctx->mode == MODE_SINGLE || !ctx->parts[0].lev[l].dist) return WD_OK;
    const int np = which == ARR_COEF ? 14 : 1;
    auto pl_of = [](Level& lv) {
        PartLevel q;
        q.L = lv.L;
        q.dist = lv.dist;
        return q;
    };
    if (ctx->mode == MODE_VIRTUAL) {
        // every send of part p lands in the same global rows of its peer part
        const int R = (int)ctx->parts.size();
        for (int p = 0; p < R; p++) {
            Level& me = ctx->parts[p].lev[l];
            for (const HaloMsg& m : halo_msgs(pl_of(me), p, R, w)) {
                if (!m.send) continue;
                Level& to = ctx->parts[m.peer].lev[l];
                for (int pl = 0; pl < np; pl++)
                    CK(cudaMemcpyAsync(arr_of(to, which) + (i64)pl * to.L.NT + (i64)(m.row0 - to.L.jg0) * to.L.sj,
                                       arr_of(me, which) + (i64)pl * me.L.NT + (i64)(m.row0 - me.L.jg0) * me.L.sj,
                                       sizeof(double) * m.rows * me.L.sj, cudaMemcpyDeviceToDevice, st));
            }
        }
        return WD_OK;
    }
    // NCCL: one process per GPU, this rank's single part
    Nccl& N = nccl();
    Level& me = ctx->parts[0].lev[l];
    const LevDev& L = me.L;
    const std::vector<HaloMsg> msgs = halo_msgs(pl_of(me), ctx->rank, ctx->nranks, w);
    NK(N.GroupStart());
    for (int pl = 0; pl < np; pl++) {
        double* a = arr_of(me, which) + (i64)pl * L.NT;
        for (const HaloMsg& m : msgs) {
            double* buf = a + (i64)(m.row0 - L.jg0) * L.sj;
            const size_t cnt = (size_t)m.rows * L.sj;
            if (m.send) NK(N.Send(buf, cnt, ncclDouble, m.peer, ctx->comm, st));
            else NK(N.Recv(buf, cnt, ncclDouble, m.peer, ctx->comm, st));
        }
    }
    NK(N.GroupEnd());
    return WD_OK;
}

// Gather level: every rank computed the rows [cown0, cown1) of the (full)
// level; give every rank all rows.
int gather_rows(wd_ctx* ctx, int l, int which, cudaStream_t st) {
    if (ctx->mode == MODE_SINGLE) return WD_OK;
    const int np = which == ARR_COEF ? 14 : 1;
    if (ctx->mode == MODE_VIRTUAL) {
        const int R = (int)ctx->parts.size();
        for (int p = 0; p < R; p++) {
            Level& src = ctx->parts[p].lev[l];
            const size_t n = (size_t)(src.cown1 - src.cown0) * src.L.sj;
            if (!n) continue;
            for (int q = 0; q < R; q++) {
                if (q == p) continue;
                Level& dst = ctx->parts[q].lev[l];
                for (int pl = 0; pl < np; pl++)
                    CK(cudaMemcpyAsync(arr_of(dst, which) + (i64)pl * dst.L.NT + (i64)src.cown0 * src.L.sj,
                                       arr_of(src, which) + (i64)pl * src.L.NT + (i64)src.cown0 * src.L.sj,
                                       sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            }
        }
        return WD_OK;
    }
    Nccl& N = nccl();
    Level& me = ctx->parts[0].lev[l];
    NK(N.GroupStart());
    for (int r = 0; r < ctx->nranks; r++) {
        const int a = ctx->rrows[l][r].first, b = ctx->rrows[l][r].second;   // rank r's rows
        const size_t n = (size_t)(b - a) * me.L.sj;
        if (!n) continue;
        for (int pl = 0; pl < np; pl++) {
            double* buf = arr_of(me, which) + (i64)pl * me.L.NT + (i64)a * me.L.sj;
            NK(N.Bcast(buf, buf, n, ncclDouble, r, ctx->comm, st));
        }
    }
    NK(N.GroupEnd());
    return WD_OK;
}

// sum of one device scalar per rank, in rank order (identical on every rank
// and in every mode): in = per-part scalars (virtual) or this rank's scalar
int sum_ranks(wd_ctx* ctx, const double* in, double* out, cudaStream_t st) {
    if (ctx->mode == MODE_SINGLE) {
        if (in != out) CK(cudaMemcpyAsync(out, in, sizeof(double), cudaMemcpyDeviceToDevice, st));
        return WD_OK;
    }
    double* tmp = ctx->dscal + 256;   // nranks values
    if (ctx->mode == MODE_VIRTUAL) {
        CK(cudaMemcpyAsync(tmp, in, sizeof(double) * ctx->parts.size(), cudaMemcpyDeviceToDevice, st));
    } else {
        NK(nccl().AllGather(in, tmp, 1, ncclDouble, ctx->comm, st));
    }
    launch_sum_ordered(tmp, ctx->nranks, out, st);
    CKL();
    return WD_OK;
}

// ------------------------------------------------------------------ V-cycle
// Canonical roles of the level buffers: the iterate in raw[1] (every kernel
// and TMA map refers to it) and the fused sweep's second buffer raw[4].  The
// sweeps swap the host-side pointers as they are enqueued or captured; every
// ABI call that runs sweeps restores the canonical roles on exit, error paths
// included, so a failed capture or an early return cannot leave a level
// pointing at the wrong buffer for the next call.
struct RoleGuard {
    wd_ctx* ctx;
    explicit RoleGuard(wd_ctx* c) : ctx(c) {}
    ~RoleGuard() {
        if (!ctx) return;
        for (Part& P : ctx->parts)
            for (int l = 0; l < ctx->nlev; l++) {
                P.lev[l].lam = P.lev[l].raw[1];
                P.lev[l].lam2 = P.lev[l].raw[4];
            }
    }
};

// installs a context's knobs (wd_ctx::knob) in the launchers' globals
// (and marks every level's halo rows as not known to be current: the caller
// may have changed the arrays)
struct KnobScope {
    explicit KnobScope(wd_ctx* c) {
        if (!c) return;
        for (bool& b : c->halo_fresh) b = false;
        g_gs_v2 = c->knob[0];
        g_test_jitter = c->knob[1];
        g_test_gs_grid = c->knob[2];
        g_fuse_prolong = c->knob[3];
        g_apply_variant = c->knob[4];
    }
};

int smooth(wd_ctx* ctx, int l, bool prof, int ns, cudaStream_t st,
           const ProlongIn* pro = nullptr);
int smooth_end(wd_ctx* ctx, int l, cudaStream_t st);

int coarse_solve(wd_ctx* ctx, cudaStream_t st) {
    const int l = ctx->nlev - 1;
    if (ctx->coarse_direct) {
        for (Part& P : ctx->parts) {
            Level& lc = P.lev[l];
            if (ctx->nf > 0) launch_coarse_gemv(lc.L, P.Ainv, ctx->nf, lc.f, lc.lam, st);
        }
    } else {   // reading C8: GS sweeps from 0 (with halo exchanges on a slab level)
        for (Part& P : ctx->parts) CK(cudaMemsetAsync(P.lev[l].lam, 0, sizeof(double) * P.lev[l].L.NT, st));
        for (int s = 0; s < ctx->opt.coarse_iters; s++) RC(smooth(ctx, l, false, 0, st));
        RC(smooth_end(ctx, l, st));
    }
    CKL();
    return WD_OK;
}

// does level l use the fused one-pass sweep (k_gs_fused.cu)?
bool line_level(const wd_ctx* ctx, int l) {
    return ctx->opt.smoother == WD_SMOOTH_LINE ||
           (ctx->opt.line_from_level >= 0 && l >= ctx->opt.line_from_level);
}
bool fused_level(const wd_ctx* ctx, int l) {
    return ctx->opt.smoother == WD_SMOOTH_FUSED && !line_level(ctx, l);
}

// one smoothing sweep on level l.
//  * fused: lam -> lam2 in one launch, then the two buffers swap roles (the
//    caller restores the canonical buffer with smooth_end); on slabs the two
//    halo rows of the input iterate are exchanged first (the sweep recomputes
//    the nearest halo row as tile halo and writes owned rows only);
//  * phased / line relaxation: 4 colour phases in place; on slabs the boundary
//    rows are exchanged after phase 1 (even rows final) and phase 3 (odd rows
//    final)
// boundary-first: may level l's sweeps run their boundary tile rows first and
// exchange the new boundary rows while the interior tiles run?  Slabs
// (virtual or NCCL ranks) on a distributed level with the TMA fused sweep
bool overlap_level(const wd_ctx* ctx, int l) {
    if (!ctx->opt.overlap_halo || ctx->mode == MODE_SINGLE || !ctx->side) return false;
    if (!ctx->parts[0].lev[l].dist || !fused_level(ctx, l)) return false;
    for (const Part& P : ctx->parts)
        if (!v2_level(P.lev[l])) return false;
    return true;
}

int smooth(wd_ctx* ctx, int l, bool prof, int ns, cudaStream_t st, const ProlongIn* pro) {
    if (prof && ns < 16) CK(cudaEventRecordWithFlags(ctx->ev_gs[2 * ns], st, cudaEventRecordExternal));
    const bool fresh = ctx->halo_fresh[l];
    ctx->halo_fresh[l] = false;
    if (fused_level(ctx, l) && overlap_level(ctx, l) && !pro) {
        // the input's halo rows, unless the previous sweep's overlapped exchange
        // already brought them; then the tile rows holding the first / last 2
        // owned rows, the exchange of those rows of the output on the side
        // stream, the interior tile rows meanwhile (any tiling gives the same
        // node updates: the tiles recompute their halos)
        if (!fresh) RC(exchange(ctx, l, ARR_LAM, 2, st));
        std::vector<int> b0(ctx->parts.size()), b1(ctx->parts.size()), nty(ctx->parts.size());
        for (size_t p = 0; p < ctx->parts.size(); p++) {
            Level& F = ctx->parts[p].lev[l];
            gs_fused2_tile_rows(F.L, 2, &b0[p], &b1[p], &nty[p]);
            if (b0[p] >= b1[p]) {   // no interior: all tile rows now
                gs_sweep_level(F, st);
            } else {
                gs_sweep_level(F, st, nullptr, nullptr, 0, b0[p]);
                gs_sweep_level(F, st, nullptr, nullptr, b1[p], nty[p]);
            }
        }
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        RC(exchange(ctx, l, ARR_LAM2, 2, ctx->side));
        for (size_t p = 0; p < ctx->parts.size(); p++)
            if (b0[p] < b1[p]) gs_sweep_level(ctx->parts[p].lev[l], st, nullptr, nullptr, b0[p], b1[p]);
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
        CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
        for (Part& P : ctx->parts) std::swap(P.lev[l].lam, P.lev[l].lam2);
        ctx->halo_fresh[l] = true;
    } else if (fused_level(ctx, l)) {
        if (!fresh) RC(exchange(ctx, l, ARR_LAM, 2, st));
        for (Part& P : ctx->parts) {
            Level& F = P.lev[l];
            gs_sweep_level(F, st, nullptr, pro);
            std::swap(F.lam, F.lam2);
        }
    } else {
        for (int c = 0; c < 4; c++) {
            for (Part& P : ctx->parts) {
                Level& F = P.lev[l];
                if (line_level(ctx, l)) launch_line_phase(F.L, F.coef, F.lam, F.f, F.lam2, F.r, c, st);
                else launch_gs_phase(F.L, F.coef, F.lam, F.f, c, st);
            }
            if (c == 1 || c == 3) RC(exchange(ctx, l, ARR_LAM, 1, st));
        }
    }
    if (prof && ns < 16) CK(cudaEventRecordWithFlags(ctx->ev_gs[2 * ns + 1], st, cudaEventRecordExternal));
    return WD_OK;
}

// after a group of sweeps: the iterate back in the canonical buffer raw[1]
// (the TMA maps and every other kernel refer to it); on slabs the fused
// sweeps leave the halo rows stale, so one row is exchanged for the residual
int smooth_end(wd_ctx* ctx, int l, cudaStream_t st) {
    for (Part& P : ctx->parts) {
        Level& F = P.lev[l];
        if (F.lam != F.raw[1]) {
            CK(cudaMemcpyAsync(F.raw[1], F.lam, sizeof(double) * F.L.NT, cudaMemcpyDeviceToDevice, st));
            F.lam2 = F.lam;
            F.lam = F.raw[1];
        }
    }
    if (fused_level(ctx, l) && !ctx->halo_fresh[l]) RC(exchange(ctx, l, ARR_LAM, 1, st));
    return WD_OK;
}

// the first level-0 sweep of a V-cycle with the fused kernel's residual
// output: ||f - K lam||^2 of the iterate entering the sweep (all ranks) into
// dscal[0]; the sweep itself is the one smooth() performs
int smooth_first_res(wd_ctx* ctx, bool prof, cudaStream_t st) {
    if (prof) CK(cudaEventRecordWithFlags(ctx->ev_gs[0], st, cudaEventRecordExternal));
    RC(exchange(ctx, 0, ARR_LAM, 2, st));
    ctx->halo_fresh[0] = false;
    double* per = ctx->dscal + 128;   // per-part sums
    for (size_t p = 0; p < ctx->parts.size(); p++) {
        Part& P = ctx->parts[p];
        Level& F = P.lev[0];
        const int nb = gs_sweep_level(F, st, P.partial);
        std::swap(F.lam, F.lam2);
        launch_reduce_sum(P.partial, nb, per + p, st);
    }
    RC(sum_ranks(ctx, per, ctx->dscal, st));
    if (prof) CK(cudaEventRecordWithFlags(ctx->ev_gs[1], st, cudaEventRecordExternal));
    CKL();
    return WD_OK;
}

// can wd_solve take its convergence test from the first sweep of each cycle?
bool lagged_residual(const wd_ctx* ctx) {
    return fused_level(ctx, 0) && ctx->nlev > 1 && ctx->opt.pre_smooth >= 1;
}

// first = 1: the first level-0 pre-smoothing sweep has already run
// (smooth_first_res or smooth), continue the cycle from there
// can the prolongation of transition l -> l+1 be folded into level l's first
// post-smoothing sweep (k_gs_fused2.cu PRO)?  One part, the fused TMA sweep on
// level l, a horizontal transition with an identity z map (the coarse region
// under a tile is then <= 40 x 8).  Off by default (env WD_FUSE_PROLONG=1 turns
// it on): bitwise equal, but measured slower -- Paper-scale V-cycle 32.3 ms
// folded against 30.8 ms with the separate pass: the sweep's per-step critical
// path grows by more than the 0.6-ms pass it saves
bool fuse_prolong(const wd_ctx* ctx, int l) {
    if (!g_fuse_prolong || ctx->parts.size() != 1 || ctx->mode != MODE_SINGLE) return false;
    if (!fused_level(ctx, l) || ctx->opt.post_smooth < 1) return false;
    const Level& F = ctx->parts[0].lev[l];
    return v2_level(F) && F.hflag && F.nkept == F.L.n3;
}

int vcycle_level(wd_ctx* ctx, int l, cudaStream_t st, int first = 0) {
    Nvtx nv("level %d", l);
    if (l == ctx->nlev - 1) {
        Nvtx nc("coarsest solve");
        return coarse_solve(ctx, st);
    }
    const bool prof = ctx->opt.profile && ctx->prof_on && l == 0 && ctx->parts.size() == 1;
    int ns = first;
    {
        Nvtx n_("pre-smoothing");
        for (int s = first; s < ctx->opt.pre_smooth; s++, ns++) RC(smooth(ctx, l, prof, ns, st));
        RC(smooth_end(ctx, l, st));
    }
    Nvtx n_res("residual + restriction");
    if (prof) CK(cudaEventRecordWithFlags(ctx->ev_ap[0], st, cudaEventRecordExternal));
    for (Part& P : ctx->parts) apply_level(P.lev[l], true, nullptr, st);
    if (prof) CK(cudaEventRecordWithFlags(ctx->ev_ap[1], st, cudaEventRecordExternal));
    RC(exchange(ctx, l, ARR_R, 1, st));
    for (Part& P : ctx->parts) {
        Level& F = P.lev[l];
        Level& C = P.lev[l + 1];
        launch_restrict(F.L, target(C), F.M, F.r, C.f, F.nkept == F.L.n3, st);
    }
    if (l + 1 == ctx->gather) RC(gather_rows(ctx, l + 1, ARR_F, st));
    else if (fused_level(ctx, l + 1)) RC(exchange(ctx, l + 1, ARR_F, 1, st));   // halo row of f_c
    for (Part& P : ctx->parts) CK(cudaMemsetAsync(P.lev[l + 1].lam, 0, sizeof(double) * P.lev[l + 1].L.NT, st));
    ctx->halo_fresh[l + 1] = false;
    CKL();
    n_res.end();
    RC(vcycle_level(ctx, l + 1, st));
    const bool fpro = fuse_prolong(ctx, l);
    ProlongIn pro{};
    if (fpro) {   // folded into the first post-smoothing sweep
        Level& F = ctx->parts[0].lev[l];
        Level& C = ctx->parts[0].lev[l + 1];
        pro.xc = C.lam;
        pro.C = C.L;
        pro.M = F.M;
        pro.w = ctx->corr_w;
    } else {
        Nvtx n_pro("prolongation");
        ctx->halo_fresh[l] = false;
        for (Part& P : ctx->parts) {
            Level& F = P.lev[l];
            Level& C = P.lev[l + 1];
            launch_prolong(F.L, C.L, F.M, C.lam, F.lam, F.nkept == F.L.n3, st, ctx->corr_w);
        }
        RC(exchange(ctx, l, ARR_LAM, 1, st));
    }
    Nvtx n_post(fpro ? "post-smoothing (+ prolongation)" : "post-smoothing");
    for (int s = 0; s < ctx->opt.post_smooth; s++, ns++)
        RC(smooth(ctx, l, prof, ns, st, (fpro && s == 0) ? &pro : nullptr));
    RC(smooth_end(ctx, l, st));
    CKL();
    return WD_OK;
}

void profile_accumulate(wd_ctx* ctx, bool cycle, bool resid) {
    if (!ctx->opt.profile) return;
    // the split V-cycle of wd_solve reaches here before any stream sync: wait
    // for the events (profile mode only)
    if (cycle) cudaEventSynchronize(ctx->ev_cyc[1]);
    if (resid) cudaEventSynchronize(ctx->ev_res[1]);
    float ms;
    if (cycle) {
        const int ns = std::min(ctx->opt.pre_smooth + ctx->opt.post_smooth, 16);
        if (ctx->nlev > 1 && ctx->parts.size() == 1)
            // level-0 sweeps of the plain kernel (the residual variant is not counted)
            for (int s = 0; s < ns; s++)
                if (cudaEventElapsedTime(&ms, ctx->ev_gs[2 * s], ctx->ev_gs[2 * s + 1]) == cudaSuccess) {
                    // the residual variant (first sweep of a cycle in wd_solve) apart
                    const int slot = (s == 0 && ctx->first_res) ? 6 : 0;
                    ctx->prof[slot] += ms;
                    ctx->prof[slot + 1] += 1;
                }
        if (cudaEventElapsedTime(&ms, ctx->ev_cyc[0], ctx->ev_cyc[1]) == cudaSuccess) {
            ctx->prof[2] += ms;
            ctx->prof[3] += 1;
        }
        if (ctx->nlev > 1 && ctx->parts.size() == 1 &&
            cudaEventElapsedTime(&ms, ctx->ev_ap[0], ctx->ev_ap[1]) == cudaSuccess) {
            ctx->prof[8] += ms;
            ctx->prof[9] += 1;
        }
    }
    if (resid && cudaEventElapsedTime(&ms, ctx->ev_res[0], ctx->ev_res[1]) == cudaSuccess) {
        ctx->prof[4] += ms;
        ctx->prof[5] += 1;
    }
    cudaGetLastError();
}

// profile mode: the level-0 sweeps of every PROF_EVERY-th split cycle are
// timed (event records in the graphs); the cycle times of all cycles
constexpr int PROF_EVERY = 4;

// wd_solve's split cycles (profile mode): the first level-0 sweep of a cycle
// (events ev_gs[0..1]) and the rest of it (the other level-0 sweeps, the
// residual before the restriction, the cycle) are read separately, each just
// before the events are recorded again -- after the GPU has been given the
// next work, so the reads never leave it idle
void profile_first(wd_ctx* ctx) {
    if (!ctx->opt.profile || !ctx->pend_first) return;
    ctx->pend_first = false;
    float ms;
    if (ctx->nlev > 1 && ctx->parts.size() == 1 && cudaEventSynchronize(ctx->ev_gs[1]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, ctx->ev_gs[0], ctx->ev_gs[1]) == cudaSuccess) {
        const int slot = ctx->pend_first_res ? 6 : 0;
        ctx->prof[slot] += ms;
        ctx->prof[slot + 1] += 1;
    }
    cudaGetLastError();
}

void profile_rest(wd_ctx* ctx) {
    if (!ctx->opt.profile || !ctx->pend_rest) return;
    ctx->pend_rest = false;
    cudaEventSynchronize(ctx->ev_cyc[1]);
    float ms;
    const int ns = std::min(ctx->opt.pre_smooth + ctx->opt.post_smooth, 16);
    if (ctx->pend_rest_sweeps && ctx->nlev > 1 && ctx->parts.size() == 1) {
        for (int sw = 1; sw < ns; sw++)
            if (cudaEventElapsedTime(&ms, ctx->ev_gs[2 * sw], ctx->ev_gs[2 * sw + 1]) == cudaSuccess) {
                ctx->prof[0] += ms;
                ctx->prof[1] += 1;
            }
        if (cudaEventElapsedTime(&ms, ctx->ev_ap[0], ctx->ev_ap[1]) == cudaSuccess) {
            ctx->prof[8] += ms;
            ctx->prof[9] += 1;
        }
    }
    if (cudaEventElapsedTime(&ms, ctx->ev_cs[ctx->pend_par], ctx->ev_cyc[1]) == cudaSuccess) {
        ctx->prof[2] += ms;
        ctx->prof[3] += 1;
    }
    cudaGetLastError();
}

int run_vcycle(wd_ctx* ctx, cudaStream_t st) {
    ctx->first_res = false;
    if (ctx->opt.profile) CK(cudaEventRecord(ctx->ev_cyc[0], st));
    if (!ctx->opt.use_graph) {
        RC(vcycle_level(ctx, 0, st));
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

// capture fn(stream) into an executable graph (kernels counted, not executed)
template <class Fn>
int capture_graph(wd_ctx* ctx, cudaGraphExec_t* out, long long* nk, Fn fn) {
    const long long before = g_launches.load();
    CK(cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal));
    const int rc = fn(ctx->cap);
    cudaGraph_t g;
    cudaError_t e = cudaStreamEndCapture(ctx->cap, &g);
    *nk = g_launches.load() - before;
    g_launches -= *nk;
    if (rc) return rc;
    if (e != cudaSuccess) return fail(WD_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(WD_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
    return WD_OK;
}

// the split V-cycle of wd_solve: which = 0 first sweep + residual of its
// input, 1 first sweep only, 2 the rest of the cycle.  The host-side buffer
// roles follow the stream order (the first sweep swaps lam/lam2 of level 0;
// the rest of the cycle ends with the iterate back in the canonical buffer).
int run_split(wd_ctx* ctx, int which, cudaStream_t st) {
    const int set = ctx->opt.profile && ctx->cyc_evented ? 1 : 0;
    const bool prof = set == 1 && ctx->parts.size() == 1;
    struct ProfOn {   // vcycle_level records events only in the profiling variant
        wd_ctx* c;
        ProfOn(wd_ctx* x, bool on) : c(x) { c->prof_on = on; }
        ~ProfOn() { c->prof_on = true; }
    } prof_on_(ctx, set == 1);
    if (which < 2 && ctx->opt.profile) CK(cudaEventRecord(ctx->ev_cs[ctx->cyc_par], st));
    auto body = [&](cudaStream_t s) -> int {
        if (which == 0) return smooth_first_res(ctx, prof, s);
        if (which == 1) return smooth(ctx, 0, prof, 0, s);
        return vcycle_level(ctx, 0, s, 1);
    };
    if (!ctx->opt.use_graph) {
        RC(body(st));
    } else {
        if (!ctx->g_first_res[set]) {
            if (which == 2) return fail(WD_E_INVAL, "split V-cycle: rest before first sweep");
            // capture all three from the canonical state: the two first-sweep
            // variants each swap the level-0 buffers, the rest swaps them back
            cudaGraphExec_t g1 = nullptr, g0 = nullptr, g2 = nullptr;
            long long k1 = 0, k0 = 0, k2 = 0;
            int rc = capture_graph(ctx, &g1, &k1,
                                   [&](cudaStream_t s) { return smooth(ctx, 0, prof, 0, s); });
            for (Part& P : ctx->parts) std::swap(P.lev[0].lam, P.lev[0].lam2);
            if (!rc)
                rc = capture_graph(ctx, &g0, &k0,
                                   [&](cudaStream_t s) { return smooth_first_res(ctx, prof, s); });
            if (!rc)
                rc = capture_graph(ctx, &g2, &k2,
                                   [&](cudaStream_t s) { return vcycle_level(ctx, 0, s, 1); });
            if (rc) {
                for (cudaGraphExec_t g : {g1, g0, g2})
                    if (g) cudaGraphExecDestroy(g);
                return rc;
            }
            ctx->g_first[set] = g1, ctx->g_first_res[set] = g0, ctx->g_rest[set] = g2;
            ctx->k_first[set] = k1, ctx->k_first_res[set] = k0, ctx->k_rest[set] = k2;
            // host roles now canonical; replay the first sweep's swap below
        }
        cudaGraphExec_t g = which == 0 ? ctx->g_first_res[set] : which == 1 ? ctx->g_first[set]
                                                               : ctx->g_rest[set];
        CK(cudaGraphLaunch(g, st));
        g_launches += which == 0 ? ctx->k_first_res[set] : which == 1 ? ctx->k_first[set]
                                                             : ctx->k_rest[set];
        // keep the host-side roles in step with the replayed graph
        if (which < 2)
            for (Part& P : ctx->parts) std::swap(P.lev[0].lam, P.lev[0].lam2);
        else
            for (Part& P : ctx->parts) {
                Level& F = P.lev[0];
                if (F.lam != F.raw[1]) std::swap(F.lam, F.lam2);
            }
    }
    if (which == 2 && ctx->opt.profile) CK(cudaEventRecord(ctx->ev_cyc[1], st));
    return WD_OK;
}

// ||f - K lam||^2 over free nodes of level 0, all ranks, into dscal[slot]
int residual_sq(wd_ctx* ctx, int slot, cudaStream_t st) {
    if (ctx->opt.profile) CK(cudaEventRecord(ctx->ev_res[0], st));
    double* per = ctx->dscal + 128;   // per-part sums
    for (size_t p = 0; p < ctx->parts.size(); p++) {
        Part& P = ctx->parts[p];
        int nb = apply_level(P.lev[0], true, P.partial, st);
        launch_reduce_sum(P.partial, nb, per + p, st);
    }
    RC(sum_ranks(ctx, per, ctx->dscal + slot, st));
    if (ctx->opt.profile) CK(cudaEventRecord(ctx->ev_res[1], st));
    CKL();
    return WD_OK;
}

// sum of squares of the owned rows of an internal level-0 vector (all ranks)
int norm_sq(wd_ctx* ctx, int which, int slot, cudaStream_t st) {
    double* per = ctx->dscal + 128;
    for (size_t p = 0; p < ctx->parts.size(); p++) {
        Part& P = ctx->parts[p];
        Level& lv = P.lev[0];
        LevDev L = lv.L;
        // owned rows only: view the owned block as a flat array
        const double* v = arr_of(lv, which) + (i64)L.own0 * L.sj;
        LevDev Lv = L;
        Lv.NT = (i64)(L.own1 - L.own0) * L.sj;
        int nb;
        launch_norm2_partial(Lv, v, P.partial, &nb, st);
        launch_reduce_sum(P.partial, nb, per + p, st);
    }
    RC(sum_ranks(ctx, per, ctx->dscal + slot, st));
    CKL();
    return WD_OK;
}

// ------------------------------------------------------------ device loop
// wd_solve's cycle loop as one CUDA graph.  The host loop below it runs, per
// cycle: test -> [first sweep] -> rest of the cycle -> [residual pass | first
// sweep of the next cycle returning the residual of this cycle's iterate];
// the bracketed steps are taken or skipped on the outcome of the test and of
// the rate prediction.  Here the same steps are bodies of conditional nodes
// whose conditions two one-thread kernels set from the device scalars, with
// the host loop's decisions in its order and arithmetic, so iterates,
// history and cycle count are the host loop's bit for bit
// (tests/test_gpu_device_loop.py):
//
//   top:  WHILE(hw) { test -> IF(hr) R }
//   R:    IF(h1) first -> rest of the cycle -> post -> IF(hp) residual
//                                                     ELSE first_res
//
// (a warm start's first residual-returning sweep is launched by the host
// before the graph).  Conditional bodies may hold kernels, memsets and
// copies only (no events), so the loop is used when profiling is off.
struct LoopHandles {
    cudaGraphConditionalHandle hw, hr, h1, hp;
};

// the test of iterate c: rel = ||f - K lam_c|| / ||f|| (dscal[0] = ||r||^2)
__global__ void loop_test_kernel(LoopDev* L, const double* __restrict__ dscal, LoopHandles h) {
    const int c = L->c;
    const double rel = sqrt(dscal[0]) / L->fn;
    if (c < 256) L->hist[c] = rel;
    if (c == 0) L->rel0 = rel;
    if (c == 1) L->rel1 = rel;
    L->ring4[c & 3] = rel;
    L->rel_last = rel;
    int st;
    if (!isfinite(rel)) st = WD_E_NONFINITE;
    else if (rel <= L->tol) st = WD_OK;
    else if (c >= 3 && rel > 10.0 * L->ring4[(c - 3) & 3]) st = WD_E_DIVERGED;
    else if (c >= L->max_cycles) st = WD_E_NOCONV;
    else st = -1;
    L->status = st;
    const bool go = st == -1;
    const bool first = go && !L->first_done;   // the cycle's first sweep still to run
    if (first) L->n_first++;
    cudaGraphSetConditional(h.hw, go ? 1u : 0u);
    cudaGraphSetConditional(h.hr, go ? 1u : 0u);
    cudaGraphSetConditional(h.h1, first ? 1u : 0u);
}

// after the cycle: a separate residual pass when the last two factors
// predict convergence, or at the cycle cap; else the next cycle's first
// sweep, which returns the residual of this cycle's iterate
__global__ void loop_post_kernel(LoopDev* L, LoopHandles h) {
    const int c = ++L->c;
    const double rel = L->rel_last;
    const double prev = c >= 2 ? L->ring4[(c - 2) & 3] : 0.0;
    const bool predicted = prev > 0.0 && rel * (rel / prev) <= L->tol;
    const bool res = predicted || c >= L->max_cycles;
    L->first_done = res ? 0 : 1;
    if (res) L->n_res++;
    else L->n_first_res++;
    cudaGraphSetConditional(h.hp, res ? 1u : 0u);   // else: the first sweep
}

// append a conditional node (handle h, one body) to the graph `st` is
// capturing, after its current dependencies; capture continues after it
int capture_conditional(cudaStream_t st, cudaGraphConditionalHandle h,
                        cudaGraphConditionalNodeType type, cudaGraph_t* body,
                        cudaGraph_t* else_body = nullptr) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
    if (cs != cudaStreamCaptureStatusActive) return fail(WD_E_CUDA, "device loop: stream not capturing");
    cudaGraphNodeParams p = {cudaGraphNodeTypeConditional};
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = else_body ? 2 : 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, deps, nd, &p));
    *body = p.conditional.phGraph_out[0];
    if (else_body) *else_body = p.conditional.phGraph_out[1];
    CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    return WD_OK;
}

// capture fn(stream) into the existing graph g; *nk = kernels it launched
template <class Fn>
int capture_into(wd_ctx* ctx, cudaGraph_t g, long long* nk, Fn fn) {
    const long long before = g_launches.load();
    CK(cudaStreamBeginCaptureToGraph(ctx->cap, g, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    const int rc = fn(ctx->cap);
    cudaGraph_t out = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->cap, &out);
    const long long d = g_launches.load() - before;
    if (nk) *nk = d;
    g_launches -= d;   // captured, not executed
    if (rc) return rc;
    if (e != cudaSuccess) return fail(WD_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
    return WD_OK;
}

// build ctx->g_loop (one part, lagged residual, graphs on); buffer roles
// canonical on entry and on return
int build_device_loop(wd_ctx* ctx) {
    if (!ctx->loopd) RC(dalloc(ctx, (void**)&ctx->loopd, sizeof(LoopDev)));
    if (!ctx->looph) CK(cudaMallocHost((void**)&ctx->looph, sizeof(LoopDev)));
    LoopDev* L = ctx->loopd;
    const double* dscal = ctx->dscal;
    cudaGraph_t top = nullptr;
    CK(cudaGraphCreate(&top, 0));
    struct Drop {
        cudaGraph_t g;
        ~Drop() { if (g) cudaGraphDestroy(g); }
    } drop{top};
    LoopHandles h;
    CK(cudaGraphConditionalHandleCreate(&h.hw, top, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {cudaGraphNodeTypeConditional};
    p.conditional.handle = h.hw;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, top, nullptr, 0, &p));
    cudaGraph_t W = p.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&h.hr, W, 0, 0));
    cudaGraph_t R = nullptr, S1 = nullptr, SR = nullptr, S0 = nullptr;
    // R's handles live in R, which exists once its node does: create the
    // node first (empty body), then the handles, then capture the bodies
    RC(capture_into(ctx, W, nullptr, [&](cudaStream_t s) -> int {
        return capture_conditional(s, h.hr, cudaGraphCondTypeIf, &R);
    }));
    CK(cudaGraphConditionalHandleCreate(&h.h1, R, 0, 0));
    CK(cudaGraphConditionalHandleCreate(&h.hp, R, 0, 0));
    // W = test -> IF(hr) R: the test kernel goes in front of the IF node
    {
        cudaKernelNodeParams kp;
        memset(&kp, 0, sizeof kp);
        void* args[] = {(void*)&L, (void*)&dscal, (void*)&h};
        kp.func = (void*)loop_test_kernel;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args;
        cudaGraphNode_t tn, rn;
        size_t nn = 1;
        CK(cudaGraphGetNodes(W, &rn, &nn));
        CK(cudaGraphAddKernelNode(&tn, W, nullptr, 0, &kp));
        CK(cudaGraphAddDependencies(W, &tn, &rn, 1));
    }
    // R: captured with the roles a first sweep leaves (swapped); the rest of
    // the cycle ends canonical
    for (Part& P : ctx->parts) std::swap(P.lev[0].lam, P.lev[0].lam2);
    RC(capture_into(ctx, R, &ctx->kl_rest, [&](cudaStream_t s) -> int {
        RC(capture_conditional(s, h.h1, cudaGraphCondTypeIf, &S1));
        RC(vcycle_level(ctx, 0, s, 1));
        loop_post_kernel<<<1, 1, 0, s>>>(L, h);
        return capture_conditional(s, h.hp, cudaGraphCondTypeIf, &SR, &S0);
    }));
    for (Part& P : ctx->parts) {
        Level& F = P.lev[0];
        if (F.lam != F.raw[1]) std::swap(F.lam, F.lam2);
    }
    // S1 runs from the canonical roles, before the rest of the cycle
    RC(capture_into(ctx, S1, &ctx->kl_first,
                    [&](cudaStream_t s) { return smooth(ctx, 0, false, 0, s); }));
    for (Part& P : ctx->parts) std::swap(P.lev[0].lam, P.lev[0].lam2);
    // SR and S0 run after the rest of the cycle, from the canonical roles
    RC(capture_into(ctx, SR, &ctx->kl_res, [&](cudaStream_t s) { return residual_sq(ctx, 0, s); }));
    RC(capture_into(ctx, S0, &ctx->kl_first_res,
                    [&](cudaStream_t s) { return smooth_first_res(ctx, false, s); }));
    for (Part& P : ctx->parts) std::swap(P.lev[0].lam, P.lev[0].lam2);
    const cudaError_t e = cudaGraphInstantiate(&ctx->g_loop, top, 0);
    if (e != cudaSuccess) {
        ctx->g_loop = nullptr;
        return fail(WD_E_CUDA, "device loop instantiate: %s", cudaGetErrorString(e));
    }
    return WD_OK;
}

// may wd_solve run its loop on the device?  Builds the graph on first use; a
// failed build leaves the host loop in charge for this context
bool use_device_loop(wd_ctx* ctx, bool lag) {
    if (!lag || !ctx->opt.device_loop || ctx->opt.profile || !ctx->opt.use_graph) return false;
    if (ctx->parts.size() != 1 || ctx->mode != MODE_SINGLE || ctx->loop_broken) return false;
    if (!ctx->g_loop && build_device_loop(ctx) != WD_OK) {
        ctx->loop_broken = true;
        cudaGetLastError();
        for (Part& P : ctx->parts) {   // roles back to canonical
            P.lev[0].lam = P.lev[0].raw[1];
            P.lev[0].lam2 = P.lev[0].raw[4];
        }
        return false;
    }
    return true;
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

int check_single(const wd_ctx* ctx) {
    if (ctx->mode != MODE_SINGLE) return fail(WD_E_INVAL, "inspection calls need a single-GPU context");
    return WD_OK;
}

size_t nodes_of(const LevDev& L) { return (size_t)L.n1 * L.n2 * L.n3; }

// ABI node / element arrays of part P: virtual ranks index the global array,
// a NCCL rank its slab (rows jlo .. jhi-1), a single GPU the whole grid
Nat nat_nodes(const wd_ctx* ctx, const Part& P, const double* p) {
    Nat a;
    a.p = p;
    if (ctx->mode == MODE_VIRTUAL) { a.n2a = ctx->n2; a.jofs = P.jlo; }
    else { a.n2a = P.jhi - P.jlo; a.jofs = 0; }
    return a;
}
Nat nat_elems(const wd_ctx* ctx, const Part& P, const double* p) {
    Nat a;
    a.p = p;
    if (ctx->mode == MODE_VIRTUAL) { a.n2a = ctx->n2 - 1; a.jofs = P.jlo; }
    else { a.n2a = P.jhi - P.jlo - 1; a.jofs = 0; }
    return a;
}
// element count / node count of the ABI arrays this context expects
size_t abi_nodes(const wd_ctx* ctx) {
    const Part& P = ctx->parts[0];
    const int rows = ctx->mode == MODE_NCCL ? P.jhi - P.jlo : ctx->n2;
    return (size_t)ctx->n1 * rows * ctx->n3;
}
size_t abi_elems(const wd_ctx* ctx) {
    const Part& P = ctx->parts[0];
    const int rows = ctx->mode == MODE_NCCL ? P.jhi - P.jlo : ctx->n2;
    return (size_t)3 * (ctx->n1 - 1) * (rows - 1) * (ctx->n3 - 1);
}

// internal level-0 vector of every part -> ABI array (owned rows; a NCCL rank
// also writes its halo rows, which are current after a V-cycle)
void out_nodes(wd_ctx* ctx, const double* dst, cudaStream_t st) {
    for (Part& P : ctx->parts) {
        LevDev L = P.lev[0].L;
        if (ctx->mode == MODE_NCCL) { L.own0 = 0; L.own1 = L.n2; }
        launch_int2nat(L, P.lev[0].lam, nat_nodes(ctx, P, dst), st);
    }
}

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
    o->gather_below_nodes = 2000000;
    o->rank = 0;
    o->nranks = 1;
    o->smoother = WD_SMOOTH_FUSED;
    o->line_from_level = -1;
    o->device_loop = 0;
    o->overlap_halo = 0;
}

const char* wd_last_error(void) { return g_err; }

void wd_destroy(wd_ctx* ctx) {
    if (!ctx) return;
    cudaDeviceSynchronize();   // no work of the context may still be in flight
    cudaGetLastError();
    if (ctx->vgraph) cudaGraphExecDestroy(ctx->vgraph);
    for (int v = 0; v < 2; v++)
        for (cudaGraphExec_t g : {ctx->g_first_res[v], ctx->g_first[v], ctx->g_rest[v]})
            if (g) cudaGraphExecDestroy(g);
    if (ctx->g_loop) cudaGraphExecDestroy(ctx->g_loop);
    dfree(ctx->loopd);
    if (ctx->looph) cudaFreeHost(ctx->looph);
    if (ctx->cap) cudaStreamDestroy(ctx->cap);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->pin_s) cudaStreamDestroy(ctx->pin_s);
    if (ctx->pout_s) cudaStreamDestroy(ctx->pout_s);
    for (auto e : ctx->pev) if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_gs) if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_cyc) if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_cs) if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_res) if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_ap) if (e) cudaEventDestroy(e);
    for (Part& P : ctx->parts) {
        for (int l = 0; l < ctx->nlev; l++) {
            for (double* p : P.lev[l].raw) dfree(p);
            dfree(P.lev[l].dmap);
        }
        dfree(P.X);
        dfree(P.Y);
        dfree(P.Z);
        dfree(P.Ainv);
        dfree(P.Dinv);
        dfree(P.partial);
    }
    dfree(ctx->dscal);
    if (ctx->hscal) cudaFreeHost(ctx->hscal);
    for (auto& p : ctx->pool) dfree(p.first);
    if (ctx->comm && nccl().CommDestroy) nccl().CommDestroy(ctx->comm);
    delete ctx;
}

long long wd_device_bytes(const wd_ctx* ctx) { return ctx ? ctx->bytes : 0; }

int wd_nccl_unique_id(char id[128]) {
    Nccl& N = nccl();
    if (!N.ok) return fail(WD_E_NCCL, "libnccl.so.2 not available");
    ncclUniqueId u;
    NK(N.GetUniqueId(&u));
    memcpy(id, u.internal, 128);
    return WD_OK;
}

int wd_nccl_comm_init(const char id[128], int nranks, int rank, void** comm) {
    Nccl& N = nccl();
    if (!N.ok) return fail(WD_E_NCCL, "libnccl.so.2 not available");
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclComm_t c;
    NK(N.CommInitRank(&c, nranks, u, rank));
    *comm = c;
    return WD_OK;
}

void wd_partition_rows(int n2, int nranks, int rank, int* j_begin, int* j_end) {
    *j_begin = (int)((long long)n2 * rank / nranks);
    *j_end = (int)((long long)n2 * (rank + 1) / nranks);
}

int wd_plan_decomposition(int n1, int n2, int n3, double a1, double a2, double a3, double h1,
                          const double* h3, const wd_options* opt, int nranks, int rank, int w,
                          int* nlevels, int* gather, int* lev, int max_levels, int* msgs,
                          int max_msgs, int* nmsgs) {
    if (!h3 || !nlevels || !gather || !lev || !msgs || !nmsgs) return fail(WD_E_INVAL, "NULL argument");
    if (n1 < 3 || n2 < 3 || n3 < 2 || n3 - 1 >= MAXNZ) return fail(WD_E_INVAL, "bad dims");
    if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks || w < 1 || w > HALO)
        return fail(WD_E_INVAL, "bad nranks / rank / w");
    wd_options o;
    if (opt) o = *opt;
    else wd_default_options(&o);
    const double a[3] = {a1, a2, a3};
    HierPlan H;
    RC(plan_hierarchy(n1, n2, n3, a, o, nranks, std::vector<int>{rank}, h1, h3, H));
    if (H.nlev > max_levels) return fail(WD_E_INVAL, "max_levels %d < %d levels", max_levels, H.nlev);
    *nlevels = H.nlev;
    *gather = H.gather < MAXLEV ? H.gather : -1;
    int nm = 0;
    for (int l = 0; l < H.nlev; l++) {
        const PartLevel& P = H.part[0][l];
        int* v = lev + 8 * l;
        for (int d = 0; d < 3; d++) v[d] = H.dims[l][d];
        v[3] = P.dist ? 1 : 0;
        v[4] = P.L.jg0;
        v[5] = P.L.jg0 + P.L.n2;
        v[6] = P.dist ? P.L.jg0 + P.L.own0 : P.cown0;
        v[7] = P.dist ? P.L.jg0 + P.L.own1 : P.cown1;
        for (const HaloMsg& m : halo_msgs(P, rank, nranks, w)) {
            if (nm >= max_msgs) return fail(WD_E_INVAL, "max_msgs %d too small", max_msgs);
            int* q = msgs + 5 * nm++;
            q[0] = l;
            q[1] = m.peer;
            q[2] = m.send;
            q[3] = m.row0;
            q[4] = m.rows;
        }
    }
    *nmsgs = nm;
    return WD_OK;
}

int ensure_pipe(wd_ctx* ctx);

static int assemble_impl(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                         double a1, double a2, double a3, const wd_options* opt, cudaStream_t st,
                         wd_ctx* ctx) {
    ctx->n1 = n1;
    ctx->n2 = n2;
    ctx->n3 = n3;
    ctx->a[0] = a1;
    ctx->a[1] = a2;
    ctx->a[2] = a3;
    for (int d = 0; d < 3; d++) ctx->c[d] = 1.0 / (ctx->a[d] * ctx->a[d]);
    if (opt) ctx->opt = *opt;
    else wd_default_options(&ctx->opt);
    const wd_options& o = ctx->opt;
    PhaseTimer PT;
    PT.start(st);
    // ---- decomposition
    ctx->nranks = o.nranks > 1 ? o.nranks : 1;
    // one rank with a communicator runs the NCCL path (no neighbours: the
    // exchanges are empty groups, rank sums go through ncclAllGather)
    if (ctx->nranks == 1 && !(o.rank == 0 && o.nccl_comm)) ctx->mode = MODE_SINGLE;
    else if (o.rank < 0) ctx->mode = MODE_VIRTUAL;
    else ctx->mode = MODE_NCCL;
    if (ctx->nranks > 64) return fail(WD_E_INVAL, "nranks %d > 64", ctx->nranks);
    ctx->own0g.resize(ctx->nranks);
    ctx->own1g.resize(ctx->nranks);
    if (ctx->mode == MODE_NCCL) {
        if (!o.nccl_comm) return fail(WD_E_INVAL, "NCCL mode needs opt.nccl_comm (wd_nccl_comm_init)");
        if (!nccl().ok) return fail(WD_E_NCCL, "libnccl.so.2 not available");
        ctx->comm = (ncclComm_t)o.nccl_comm;
        ctx->rank = o.rank;
    }
    for (int r = 0; r < ctx->nranks; r++) wd_partition_rows(n2, ctx->nranks, r, &ctx->own0g[r], &ctx->own1g[r]);
    if (ctx->mode == MODE_NCCL && (o.j_begin != ctx->own0g[o.rank] || o.j_end != ctx->own1g[o.rank]))
        return fail(WD_E_INVAL, "rank %d: rows [%d,%d) differ from wd_partition_rows [%d,%d)", o.rank,
                    o.j_begin, o.j_end, ctx->own0g[o.rank], ctx->own1g[o.rank]);
    for (int r = 0; r < ctx->nranks; r++)
        if (ctx->nranks > 1 && ctx->own1g[r] - ctx->own0g[r] < MIN_OWNED)
            return fail(WD_E_INVAL, "rank %d owns %d rows (< %d)", r, ctx->own1g[r] - ctx->own0g[r], MIN_OWNED);
    const int nparts = ctx->mode == MODE_VIRTUAL ? ctx->nranks : 1;
    ctx->parts.resize(nparts);
    for (int p = 0; p < nparts; p++) {
        Part& P = ctx->parts[p];
        P.rank = ctx->mode == MODE_NCCL ? ctx->rank : p;
        P.own0g = ctx->own0g[P.rank];
        P.own1g = ctx->own1g[P.rank];
        P.jlo = ctx->nranks > 1 ? std::max(P.own0g - HALO, 0) : 0;
        P.jhi = ctx->nranks > 1 ? std::min(P.own1g + HALO, n2) : n2;
    }

    PT.mark("decomposition");
    // ---- coordinates: internal copies of the part's rows (natural layout).
    // Host arrays on one GPU: copied straight into the internal copies in
    // chunks of node rows on a copy stream; the level-0 assembly below starts
    // on each chunk's tile rows as soon as their rows have arrived.
    const bool piped = ctx->mode == MODE_SINGLE && !is_device_ptr(X) && !is_device_ptr(Y) &&
                       !is_device_ptr(Z);
    constexpr int NCH = 8;
    int chunk_rows[NCH + 1] = {0};
    if (piped) {
        RC(ensure_pipe(ctx));
        Part& P = ctx->parts[0];
        const size_t n = (size_t)n1 * n2 * n3, plane = (size_t)n1 * n2;
        double** dst[3] = {&P.X, &P.Y, &P.Z};
        const double* src[3] = {X, Y, Z};
        for (int d = 0; d < 3; d++) RC(dalloc(ctx, (void**)dst[d], sizeof(double) * n, false));
        CK(cudaEventRecord(ctx->pev[16], st));
        CK(cudaStreamWaitEvent(ctx->pin_s, ctx->pev[16], 0));
        for (int c = 0; c < NCH; c++) {
            const int r0 = (int)((long long)n2 * c / NCH), r1 = (int)((long long)n2 * (c + 1) / NCH);
            chunk_rows[c + 1] = r1;
            for (int d = 0; d < 3; d++)
                CK(cudaMemcpy2DAsync(*dst[d] + (size_t)r0 * n1, sizeof(double) * plane,
                                     src[d] + (size_t)r0 * n1, sizeof(double) * plane,
                                     sizeof(double) * (size_t)(r1 - r0) * n1, n3,
                                     cudaMemcpyHostToDevice, ctx->pin_s));
            CK(cudaEventRecord(ctx->pev[c], ctx->pin_s));
        }
    } else {
        const size_t N = abi_nodes(ctx);
        Stage sx, sy, sz;
        RC(stage_in(nullptr, sx, X, N, st));
        RC(stage_in(nullptr, sy, Y, N, st));
        RC(stage_in(nullptr, sz, Z, N, st));
        const int rows_in = ctx->mode == MODE_NCCL ? ctx->parts[0].jhi - ctx->parts[0].jlo : n2;
        for (Part& P : ctx->parts) {
            const int rows = P.jhi - P.jlo;
            const size_t n = (size_t)n1 * rows * n3;
            const int jofs = ctx->mode == MODE_NCCL ? 0 : P.jlo;
            double** dst[3] = {&P.X, &P.Y, &P.Z};
            const double* src[3] = {sx.d, sy.d, sz.d};
            for (int d = 0; d < 3; d++) {
                RC(dalloc(ctx, (void**)dst[d], sizeof(double) * n, false));   // copied over
                CK(cudaMemcpy2DAsync(*dst[d], sizeof(double) * n1 * rows,
                                     src[d] + (size_t)jofs * n1, sizeof(double) * n1 * rows_in,
                                     sizeof(double) * n1 * rows, n3, cudaMemcpyDeviceToDevice, st));
            }
        }
        RC(stage_finish(st, {&sx, &sy, &sz}));
    }
    RC(dalloc(ctx, (void**)&ctx->dscal, sizeof(double) * 4096));
    CK(cudaMallocHost((void**)&ctx->hscal, sizeof(double) * 64));
    CK(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
    if (ctx->mode != MODE_SINGLE) {
        CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    }
    apply_tma_prepare();
    gs_fused_prepare();
    gs_fused2_prepare();
    if (o.profile) {
        for (auto& e : ctx->ev_gs) CK(cudaEventCreate(&e));
        for (auto& e : ctx->ev_cyc) CK(cudaEventCreate(&e));
        for (auto& e : ctx->ev_cs) CK(cudaEventCreate(&e));
        for (auto& e : ctx->ev_res) CK(cudaEventCreate(&e));
        for (auto& e : ctx->ev_ap) CK(cudaEventCreate(&e));
    }

    PT.mark("coordinates + ctx");
    // ---- level 0: assembly fused with validation
    const bool multi = ctx->nranks > 1;
    unsigned long long* dbad = (unsigned long long*)(ctx->dscal + 8);
    unsigned long long worst = ~0ull;
    int wei = 0, wej = 0, wek = 0;
    for (Part& P : ctx->parts) {
        Level& L0 = P.lev[0];
        const int rows = P.jhi - P.jlo;
        L0.L = make_level(n1, rows, n3, P.jlo, n2, P.own0g - P.jlo, P.own1g - P.jlo);
        L0.dist = multi;
        L0.cown0 = L0.L.own0;
        L0.cown1 = L0.L.own1;
        RC(alloc_level(ctx, L0, false));
        CK(cudaMemsetAsync(dbad, 0xff, sizeof(unsigned long long), st));
        if (piped) {
            // tile rows whose node rows have all arrived, chunk by chunk
            CK(cudaEventRecord(ctx->pev[15], st));
            CK(cudaStreamWaitEvent(ctx->pout_s, ctx->pev[15], 0));
            const int nty = assemble_tile_rows(rows);
            int t0 = 0;
            for (int c = 0; c < NCH; c++) {
                int t1 = t0;
                while (t1 < nty && (assemble_rows_needed(t1) <= chunk_rows[c + 1] || c == NCH - 1)) t1++;
                CK(cudaStreamWaitEvent(ctx->pout_s, ctx->pev[c], 0));
                launch_assemble(P.X, P.Y, P.Z, n1, rows, n3, ctx->c, L0.L, L0.coef, dbad, ctx->pout_s,
                                t0, t1);
                t0 = t1;
            }
            CK(cudaEventRecord(ctx->pev[14], ctx->pout_s));
            CK(cudaStreamWaitEvent(st, ctx->pev[14], 0));
        } else {
            launch_assemble(P.X, P.Y, P.Z, n1, rows, n3, ctx->c, L0.L, L0.coef, dbad, st);
        }
        CKL();
        unsigned long long hb;
        CK(cudaMemcpyAsync(&hb, dbad, sizeof hb, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hb != ~0ull) {
            const unsigned long long e = hb / 16;
            const int nx = n1 - 1, nyl = rows - 1;
            const int ei = (int)(e % nx), ej = (int)((e / nx) % nyl) + P.jlo,
                      ek = (int)(e / ((unsigned long long)nx * nyl));
            const unsigned long long g = (((unsigned long long)ek * (n2 - 1) + ej) * nx + ei) * 16 + hb % 16;
            if (g < worst) { worst = g; wei = ei; wej = ej; wek = ek; }
        }
        int cnt = (((n1 + 1) / 2 + 31) / 32) * ((rows + 3) / 4) + 4096;
        P.npartial = cnt;
        RC(dalloc(ctx, (void**)&P.partial, sizeof(double) * cnt));
    }
    ctx->nlev = 1;
    ctx->levdims[0][0] = n1;
    ctx->levdims[0][1] = n2;
    ctx->levdims[0][2] = n3;
    ctx->rrows.assign(1, std::vector<std::pair<int, int>>(ctx->nranks));
    for (int r = 0; r < ctx->nranks; r++) ctx->rrows[0][r] = {ctx->own0g[r], ctx->own1g[r]};
    if (ctx->mode == MODE_NCCL) {   // agree on the lowest failing element
        unsigned long long* d = (unsigned long long*)(ctx->dscal + 16);
        CK(cudaMemcpyAsync(d, &worst, sizeof worst, cudaMemcpyHostToDevice, st));
        NK(nccl().AllReduce(d, d, 1, ncclUint64, ncclMin, ctx->comm, st));
        unsigned long long g;
        CK(cudaMemcpyAsync(&g, d, sizeof g, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (g != worst) {
            worst = g;
            const unsigned long long e = g / 16;
            wei = (int)(e % (n1 - 1));
            wej = (int)((e / (n1 - 1)) % (n2 - 1));
            wek = (int)(e / ((unsigned long long)(n1 - 1) * (n2 - 1)));
        }
    }
    if (worst != ~0ull) {
        const unsigned long long what = worst % 16;
        if (what == 0) return fail(WD_E_MESH, "element (%d,%d,%d): Z not increasing in k", wei, wej, wek);
        return fail(WD_E_MESH, "element (%d,%d,%d): detJ <= 0 at Gauss point %d", wei, wej, wek,
                    (int)what - 1);
    }
    RC(exchange(ctx, 0, ARR_COEF, HALO, st));   // rows at the slab edges come from the neighbours

    PT.mark("level-0 assembly");
    // ---- planner inputs (reading C2): h1 = sqrt(dx dy); h3 at the column of minimum Z(i,j,0)
    double h1;
    double h3[MAXNZ];
    {
        Part& P0 = ctx->parts[0];
        double v[4];
        CK(cudaMemcpy(&v[0], P0.X, sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&v[1], P0.X + 1, sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&v[2], P0.Y, sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&v[3], P0.Y + n1, sizeof(double), cudaMemcpyDeviceToHost));
        h1 = std::sqrt((v[1] - v[0]) * (v[3] - v[2]));
        if (ctx->mode == MODE_NCCL) {   // every rank plans with rank 0's (global origin) h1
            double* dh = ctx->dscal + 2040;
            CK(cudaMemcpyAsync(dh, &h1, sizeof h1, cudaMemcpyHostToDevice, st));
            NK(nccl().Bcast(dh, dh, 1, ncclDouble, 0, ctx->comm, st));
            CK(cudaMemcpyAsync(&h1, dh, sizeof h1, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
        // every part: argmin over its owned bottom rows -> (value, global index)
        const int nblk = 256;
        double* pval = ctx->dscal + 1024;
        long long* pidx = (long long*)(ctx->dscal + 1024 + 2 * (nblk + 1));
        double best = 0.0;
        long long bidx = -1;
        int bpart = 0;
        std::vector<double> cand_v;
        std::vector<long long> cand_i;
        for (size_t p = 0; p < ctx->parts.size(); p++) {
            Part& P = ctx->parts[p];
            const int o0 = P.lev[0].L.own0, o1 = P.lev[0].L.own1;
            launch_argmin_bottom(P.Z + (size_t)o0 * n1, (o1 - o0) * n1, pval, pidx, nblk, st);
            CKL();
            double hv;
            long long hi;
            CK(cudaMemcpyAsync(&hv, pval + nblk, sizeof hv, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(&hi, pidx + nblk, sizeof hi, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const long long gi = hi + (long long)P.own0g * n1;   // global bottom index
            if (bidx < 0 || hv < best || (hv == best && gi < bidx)) { best = hv; bidx = gi; bpart = (int)p; }
        }
        std::vector<double> zc(n3);
        if (ctx->mode == MODE_NCCL) {
            // agree on (value, index): all-gather both, pick the minimum
            double* dv = ctx->dscal + 2048;
            double mine[2] = {best, (double)bidx};
            CK(cudaMemcpyAsync(dv, mine, sizeof mine, cudaMemcpyHostToDevice, st));
            NK(nccl().AllGather(dv, dv + 2, 2, ncclDouble, ctx->comm, st));
            std::vector<double> all(2 * ctx->nranks);
            CK(cudaMemcpyAsync(all.data(), dv + 2, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            int win = 0;
            for (int r = 1; r < ctx->nranks; r++)
                if (all[2 * r] < all[2 * win] || (all[2 * r] == all[2 * win] && all[2 * r + 1] < all[2 * win + 1]))
                    win = r;
            bidx = (long long)all[2 * win + 1];
            // the winner broadcasts its column
            double* col = ctx->dscal + 2560;
            if (win == ctx->rank) {
                Part& P = ctx->parts[0];
                const long long li = bidx - (long long)P.jlo * n1;
                for (int k = 0; k < n3; k++)
                    CK(cudaMemcpyAsync(col + k, P.Z + (size_t)k * n1 * (P.jhi - P.jlo) + li, sizeof(double),
                                       cudaMemcpyDeviceToDevice, st));
            }
            NK(nccl().Bcast(col, col, n3, ncclDouble, win, ctx->comm, st));
            CK(cudaMemcpyAsync(zc.data(), col, sizeof(double) * n3, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {
            Part& P = ctx->parts[bpart];
            const long long li = bidx - (long long)P.jlo * n1;
            for (int k = 0; k < n3; k++)
                CK(cudaMemcpy(&zc[k], P.Z + (size_t)k * n1 * (P.jhi - P.jlo) + li, sizeof(double),
                              cudaMemcpyDeviceToHost));
        }
        for (int k = 0; k + 1 < n3; k++) h3[k] = zc[k + 1] - zc[k];
    }

    PT.mark("planner inputs");
    // ---- hierarchy: the host plan, then per
    // transition the coarse level's storage, its maps and the Galerkin product
    HierPlan H;
    {
        std::vector<int> prank;
        for (Part& P : ctx->parts) prank.push_back(P.rank);
        RC(plan_hierarchy(n1, n2, n3, ctx->a, o, ctx->nranks, prank, h1, h3, H));
        for (size_t p = 0; p < ctx->parts.size(); p++) {   // level 0 as laid out above
            const LevDev &a = ctx->parts[p].lev[0].L, &b = H.part[p][0].L;
            if (a.n2 != b.n2 || a.jg0 != b.jg0 || a.own0 != b.own0 || a.own1 != b.own1)
                return fail(WD_E_INTERNAL, "level-0 layout differs from the host plan");
        }
    }
    ctx->gather = H.gather;
    ctx->rrows = H.rrows;
    for (int l = 0; l + 1 < H.nlev; l++) {
        const int cl = l + 1;
        const int fn1 = H.dims[l][0], fn2 = H.dims[l][1], fn3 = H.dims[l][2];
        const int m1 = H.dims[cl][0], m2 = H.dims[cl][1], nk = H.dims[cl][2];
        const int* kept = H.kept[l];
        const std::vector<int>& px = H.px[l];
        const std::vector<int>& py = H.py[l];
        for (int d = 0; d < 3; d++) ctx->levdims[cl][d] = H.dims[cl][d];
        for (size_t p = 0; p < ctx->parts.size(); p++) {
            Part& P = ctx->parts[p];
            Level& F = P.lev[l];
            F.hflag = H.hflag[l];
            F.nkept = nk;
            for (int t = 0; t < nk; t++) F.kept[t] = kept[t];
            Level& C = P.lev[cl];
            const PartLevel& pc = H.part[p][cl];
            C.L = pc.L;
            C.dist = pc.dist;
            C.cown0 = pc.cown0;
            C.cown1 = pc.cown1;
            const int jlo_c = C.L.jg0;
            RC(alloc_level(ctx, C, true));
            // maps: x and z global; y local to the part (fine rows F.jg0.., coarse rows jlo_c..)
            const int fr = F.L.n2, cr = C.L.n2;
            std::vector<int> glo(fn2), gco(fn2), xlo(fn1), xco(fn1), zlo(fn3), zco(fn3);
            map1d(fn1, px.data(), m1, xlo.data(), xco.data());
            map1d(fn2, py.data(), m2, glo.data(), gco.data());
            map1d(fn3, kept, nk, zlo.data(), zco.data());
            std::vector<int> hmap;
            size_t offs[3][3];
            auto put = [&](int d, const int* lo, const int* co, int n, const int* pos, int m) {
                offs[d][0] = hmap.size();
                hmap.insert(hmap.end(), lo, lo + n);
                offs[d][1] = hmap.size();
                hmap.insert(hmap.end(), co, co + n);
                offs[d][2] = hmap.size();
                hmap.insert(hmap.end(), pos, pos + m);
            };
            std::vector<int> ylo(fr), yco(fr), ypos(cr);
            for (int t = 0; t < fr; t++) {
                const int g = t + F.L.jg0;
                ylo[t] = glo[g] - jlo_c;
                yco[t] = gco[g];
            }
            for (int cc = 0; cc < cr; cc++) ypos[cc] = py[cc + jlo_c] - F.L.jg0;
            put(0, xlo.data(), xco.data(), fn1, px.data(), m1);
            put(1, ylo.data(), yco.data(), fr, ypos.data(), cr);
            put(2, zlo.data(), zco.data(), fn3, kept, nk);
            RC(dalloc(ctx, (void**)&F.dmap, sizeof(int) * hmap.size()));
            CK(cudaMemcpy(F.dmap, hmap.data(), sizeof(int) * hmap.size(), cudaMemcpyHostToDevice));
            for (int d = 0; d < 3; d++) {
                F.M.lo[d] = F.dmap + offs[d][0];
                F.M.co[d] = F.dmap + offs[d][1];
                F.M.pos[d] = F.dmap + offs[d][2];
            }
            launch_galerkin(F.L, target(C), F.M, F.coef, C.coef, nk == fn3, st);
            CKL();
        }
        ctx->nlev++;
        if (H.part[0][cl].dist) RC(exchange(ctx, cl, ARR_COEF, HALO, st));
        else if (cl == ctx->gather) RC(gather_rows(ctx, cl, ARR_COEF, st));
    }
    PT.mark("hierarchy (plan+Galerkin)");
    // ---- coarsest level (reading C8): replicated or single
    {
        const int l = ctx->nlev - 1;
        const int* d = ctx->levdims[l];
        const i64 nf = free_count(d[0], d[1], d[2]);
        ctx->nf = (int)nf;
        ctx->coarse_direct = nf <= o.coarsest_max_free;
        if (ctx->parts[0].lev[l].dist && ctx->coarse_direct)
            return fail(WD_E_INTERNAL, "coarsest level is distributed (raise gather_below_nodes)");
        if (ctx->coarse_direct && nf > 0) {
            coarse_prepare((int)nf);
            for (Part& P : ctx->parts) {
                RC(dalloc(ctx, (void**)&P.Ainv, sizeof(double) * (size_t)nf * nf));
                RC(dalloc(ctx, (void**)&P.Dinv, sizeof(double) * 32 * 32));
                launch_dense_build(P.lev[l].L, P.lev[l].coef, P.Ainv, (int)nf, st);
                gj_invert(P.Ainv, (int)nf, P.Dinv, st);
                CKL();
            }
        }
    }
    PT.mark("coarsest inverse");
    CK(cudaStreamSynchronize(st));
    CKL();
    return WD_OK;
}

int wd_assemble(const double* X, const double* Y, const double* Z, int n1, int n2, int n3,
                double a1, double a2, double a3, const wd_options* opt, void* stream,
                wd_ctx** out) {
    Nvtx nvtx_("wd_assemble");
    if (!out) return fail(WD_E_INVAL, "out is NULL");
    *out = nullptr;
    if (const char* v = getenv("WD_APPLY_VARIANT")) g_apply_variant = atoi(v);
    if (const char* v = getenv("WD_TMA_DEBUG")) g_tma_debug = atoi(v);
    g_galerkin_generic = getenv("WD_GALERKIN_GENERIC") ? atoi(getenv("WD_GALERKIN_GENERIC")) : 0;
    g_gs_v2 = getenv("WD_GS_V2") ? atoi(getenv("WD_GS_V2")) : 1;
    g_test_jitter = getenv("WD_TEST_JITTER") ? atoi(getenv("WD_TEST_JITTER")) : 0;
    g_fuse_prolong = getenv("WD_FUSE_PROLONG") ? atoi(getenv("WD_FUSE_PROLONG")) : 0;
    g_test_gs_grid = getenv("WD_TEST_GS_GRID") ? atoi(getenv("WD_TEST_GS_GRID")) : 0;
    if (!X || !Y || !Z) return fail(WD_E_INVAL, "NULL coordinate array");
    if (n1 < 3 || n2 < 3 || n3 < 2) return fail(WD_E_INVAL, "dims (%d,%d,%d): need n1,n2 >= 3, n3 >= 2", n1, n2, n3);
    if (n3 - 1 >= MAXNZ) return fail(WD_E_INVAL, "n3 = %d exceeds %d", n3, MAXNZ);
    if (!(a1 > 0 && a2 > 0 && a3 > 0) || !std::isfinite(a1) || !std::isfinite(a2) || !std::isfinite(a3))
        return fail(WD_E_INVAL, "penalty constants must be positive and finite");
    if (opt && (opt->pre_smooth < 0 || opt->post_smooth < 0 || opt->max_cycles < 0 ||
                opt->coarsen_rule < 0 || opt->coarsen_rule > 3 || opt->coarse_iters < 0 ||
                opt->smoother < 0 || opt->smoother > 2))
        return fail(WD_E_INVAL, "invalid options");
    if (opt && opt->coarsest_max_free > 8192)
        return fail(WD_E_INVAL, "coarsest_max_free %d > 8192 (dense inverse)", opt->coarsest_max_free);
    wd_ctx* ctx = new wd_ctx();
    const int kn[5] = {g_gs_v2, g_test_jitter, g_test_gs_grid, g_fuse_prolong, g_apply_variant};
    memcpy(ctx->knob, kn, sizeof kn);
    if (const char* v = getenv("WD_TEST_CORRECTION_WEIGHT")) ctx->corr_w = atof(v);
    int rc = assemble_impl(X, Y, Z, n1, n2, n3, a1, a2, a3, opt, (cudaStream_t)stream, ctx);
    if (rc) {
        char keep[1024];
        memcpy(keep, g_err, sizeof keep);
        cudaStreamSynchronize((cudaStream_t)stream);
        cudaGetLastError();
        ctx->comm = nullptr;   // owned by the caller
        wd_destroy(ctx);
        memcpy(g_err, keep, sizeof keep);
        return rc;
    }
    if (ctx->mode == MODE_NCCL) ctx->comm = (ncclComm_t)ctx->opt.nccl_comm;
    *out = ctx;
    return WD_OK;
}

int wd_rhs(wd_ctx* ctx, const double* u0, double* f, void* stream) {
    KnobScope knobs_(ctx);
    Nvtx nvtx_("wd_rhs");
    if (!ctx || !u0 || !f) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Stage su, sf;
    RC(stage_in(ctx, su, u0, abi_elems(ctx), st));
    RC(stage_out(ctx, sf, f, abi_nodes(ctx)));
    for (Part& P : ctx->parts)
        launch_rhs(P.X, P.Y, P.Z, P.lev[0].L, nat_elems(ctx, P, su.d), nat_nodes(ctx, P, sf.d), st);
    CKL();
    return stage_finish(st, {&su, &sf});
}

int ensure_pipe(wd_ctx* ctx) {
    if (!ctx->pin_s) {
        CK(cudaStreamCreateWithFlags(&ctx->pin_s, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->pout_s, cudaStreamNonBlocking));
        for (auto& e : ctx->pev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return WD_OK;
}

// Host-pointer recovery on one GPU, pipelined over chunks of element rows:
// the copy-in of chunk c+1 (lambda node rows, u0 element rows) runs on one
// stream while chunk c is recovered and copied out on another, so the PCIe
// directions overlap (H2D and D2H use separate copy engines).
static int recover_pipelined(wd_ctx* ctx, const double* lambda, const double* u0, double* u,
                             cudaStream_t st) {
    constexpr int NCH = 8;
    RC(ensure_pipe(ctx));
    Part& P = ctx->parts[0];
    const LevDev& L0 = P.lev[0].L;
    const int n1 = ctx->n1, n2 = ctx->n2, n3 = ctx->n3, nx = n1 - 1, ny = n2 - 1, nz = n3 - 1;
    const bool hl = !is_device_ptr(lambda), hu0 = !is_device_ptr(u0), hu = !is_device_ptr(u);
    Stage sl, su0, su;
    sl.ctx = su0.ctx = su.ctx = ctx;
    double *dl = const_cast<double*>(lambda), *du0 = const_cast<double*>(u0), *du = u;
    if (hl) { sl.staged = true; RC(stage_acquire(ctx, sl, sizeof(double) * abi_nodes(ctx))); dl = sl.d; }
    if (hu0) { su0.staged = true; RC(stage_acquire(ctx, su0, sizeof(double) * abi_elems(ctx))); du0 = su0.d; }
    if (hu) { su.staged = true; RC(stage_acquire(ctx, su, sizeof(double) * abi_elems(ctx))); du = su.d; }
    cudaEvent_t* ev = ctx->pev;
    CK(cudaEventRecord(ev[16], st));   // after the caller's prior work
    CK(cudaStreamWaitEvent(ctx->pin_s, ev[16], 0));
    CK(cudaStreamWaitEvent(ctx->pout_s, ev[16], 0));
    const size_t nplane = (size_t)n1 * n2, eplane = (size_t)nx * ny;
    int copied = -1;   // last node row of lambda copied in
    for (int c = 0; c < NCH; c++) {
        const int r0 = (int)((long long)ny * c / NCH), r1 = (int)((long long)ny * (c + 1) / NCH);
        if (r1 <= r0) continue;
        // recovering element rows r0 .. r1-1 reads node rows r0 .. r1; each node
        // row is copied once: a chunk copies the rows after the last one copied
        // up to r1; row r0 came with an earlier chunk on the same copy stream
        if (hl) {
            const int a = copied + 1;
            copied = r1;
            const size_t off = (size_t)a * n1, w = (size_t)(r1 + 1 - a) * n1;
            CK(cudaMemcpy2DAsync(dl + off, sizeof(double) * nplane, lambda + off, sizeof(double) * nplane,
                                 sizeof(double) * w, n3, cudaMemcpyHostToDevice, ctx->pin_s));
        }
        if (hu0) {  // element rows r0 .. r1-1 of every (component, plane)
            const size_t off = (size_t)r0 * nx, w = (size_t)(r1 - r0) * nx;
            CK(cudaMemcpy2DAsync(du0 + off, sizeof(double) * eplane, u0 + off, sizeof(double) * eplane,
                                 sizeof(double) * w, (size_t)3 * nz, cudaMemcpyHostToDevice, ctx->pin_s));
        }
        CK(cudaEventRecord(ev[c], ctx->pin_s));
        CK(cudaStreamWaitEvent(ctx->pout_s, ev[c], 0));
        LevDev L = L0;
        L.own0 = r0;
        L.own1 = r1;
        launch_recover(P.X, P.Y, P.Z, L, ctx->c, nat_nodes(ctx, P, dl), nat_elems(ctx, P, du0),
                       nat_elems(ctx, P, du), ctx->pout_s);
        if (hu) {
            const size_t off = (size_t)r0 * nx, w = (size_t)(r1 - r0) * nx;
            CK(cudaMemcpy2DAsync(u + off, sizeof(double) * eplane, du + off, sizeof(double) * eplane,
                                 sizeof(double) * w, (size_t)3 * nz, cudaMemcpyDeviceToHost, ctx->pout_s));
        }
    }
    CKL();
    CK(cudaEventRecord(ev[8], ctx->pout_s));
    CK(cudaEventRecord(ev[9], ctx->pin_s));
    CK(cudaStreamWaitEvent(st, ev[8], 0));
    CK(cudaStreamWaitEvent(st, ev[9], 0));
    CK(cudaStreamSynchronize(st));   // host outputs complete on return
    for (Stage* x : {&sl, &su0, &su}) stage_release(*x);
    return WD_OK;
}

int wd_recover_wind(wd_ctx* ctx, const double* lambda, const double* u0, double* u, void* stream) {
    KnobScope knobs_(ctx);
    Nvtx nvtx_("wd_recover_wind");
    if (!ctx || !lambda || !u0 || !u) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (ctx->mode == MODE_SINGLE && (!is_device_ptr(lambda) || !is_device_ptr(u0) || !is_device_ptr(u)))
        return recover_pipelined(ctx, lambda, u0, u, st);
    Stage sl, su0, su;
    RC(stage_in(ctx, sl, lambda, abi_nodes(ctx), st));
    RC(stage_in(ctx, su0, u0, abi_elems(ctx), st));
    RC(stage_out(ctx, su, u, abi_elems(ctx)));
    for (Part& P : ctx->parts)
        launch_recover(P.X, P.Y, P.Z, P.lev[0].L, ctx->c, nat_nodes(ctx, P, sl.d),
                       nat_elems(ctx, P, su0.d), nat_elems(ctx, P, su.d), st);
    CKL();
    return stage_finish(st, {&sl, &su0, &su});
}

// ------------------------------------------------------------------ f4: either side of the path
int wd_build_mesh(const double* zs, int n1, int n2, double x0, double y0, double dx, double dy,
                  const double* zeta, int n3, double H, double* X, double* Y, double* Z,
                  void* stream) {
    if (!zs || !zeta || !X || !Y || !Z) return fail(WD_E_INVAL, "NULL argument");
    if (n1 < 2 || n2 < 2 || n3 < 2) return fail(WD_E_INVAL, "need n1, n2, n3 >= 2");
    if (!(dx > 0 && dy > 0) || !std::isfinite(dx) || !std::isfinite(dy) || !std::isfinite(x0) ||
        !std::isfinite(y0) || !std::isfinite(H))
        return fail(WD_E_INVAL, "dx, dy must be positive and finite; x0, y0, H finite");
    if (zeta[0] != 0.0) return fail(WD_E_INVAL, "zeta[0] must be 0");
    for (int k = 1; k < n3; k++)
        if (!(zeta[k] > zeta[k - 1]) || !std::isfinite(zeta[k]))
            return fail(WD_E_INVAL, "zeta must be finite and strictly increasing (k = %d)", k);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)n1 * n2 * n3;
    Stage sz, sx, sy, szz;
    RC(stage_in(nullptr, sz, zs, (size_t)n1 * n2, st));
    RC(stage_out(nullptr, sx, X, N));
    RC(stage_out(nullptr, sy, Y, N));
    RC(stage_out(nullptr, szz, Z, N));
    double* dzeta = nullptr;
    RC(dalloc(nullptr, (void**)&dzeta, sizeof(double) * n3 + sizeof(unsigned long long)));
    unsigned long long* dbad = (unsigned long long*)(dzeta + n3);
    CK(cudaMemcpyAsync(dzeta, zeta, sizeof(double) * n3, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(dbad, 0xff, sizeof(unsigned long long), st));
    launch_build_mesh(sz.d, n1, n2, n3, x0, y0, dx, dy, dzeta, H, sx.d, sy.d, szz.d, dbad, st);
    CKL();
    unsigned long long bad = ~0ull;
    CK(cudaMemcpyAsync(&bad, dbad, sizeof bad, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    dfree(dzeta);
    const int rc = stage_finish(st, {&sz, &sx, &sy, &szz});
    if (rc) return rc;
    if (bad != ~0ull)
        return fail(WD_E_MESH, "domain top H = %g is not above the terrain at column (i=%llu, j=%llu)",
                    H, bad % (unsigned long long)n1, bad / (unsigned long long)n1);
    return WD_OK;
}

int wd_interp_wind(const double* uc, int nxc, int nyc, int nzc, double xc0, double yc0,
                   double DXc, double DYc, const double* hc, const double* X, const double* Y,
                   const double* Z, int n1, int n2, int n3, double* u0, void* stream) {
    if (!uc || !hc || !X || !Y || !Z || !u0) return fail(WD_E_INVAL, "NULL argument");
    if (nxc < 2 || nyc < 2 || nzc < 2) return fail(WD_E_INVAL, "coarse grid needs >= 2 points per direction");
    if (n1 < 2 || n2 < 2 || n3 < 2) return fail(WD_E_INVAL, "need n1, n2, n3 >= 2");
    if (!(DXc > 0 && DYc > 0)) return fail(WD_E_INVAL, "coarse spacings must be positive");
    for (int k = 1; k < nzc; k++)
        if (!(hc[k] > hc[k - 1])) return fail(WD_E_INVAL, "hc must be strictly increasing (k = %d)", k);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t N = (size_t)n1 * n2 * n3, E = (size_t)3 * (n1 - 1) * (n2 - 1) * (n3 - 1);
    Stage su, sx, sy, sz, so;
    RC(stage_in(nullptr, su, uc, (size_t)3 * nxc * nyc * nzc, st));
    RC(stage_in(nullptr, sx, X, N, st));
    RC(stage_in(nullptr, sy, Y, N, st));
    RC(stage_in(nullptr, sz, Z, N, st));
    RC(stage_out(nullptr, so, u0, E));
    double* dhc = nullptr;
    RC(dalloc(nullptr, (void**)&dhc, sizeof(double) * nzc));
    CK(cudaMemcpyAsync(dhc, hc, sizeof(double) * nzc, cudaMemcpyHostToDevice, st));
    launch_interp_wind(su.d, nxc, nyc, nzc, xc0, yc0, DXc, DYc, dhc, sx.d, sy.d, sz.d, n1, n2, n3,
                       so.d, st);
    CKL();
    CK(cudaStreamSynchronize(st));   // dhc is freed below
    dfree(dhc);
    return stage_finish(st, {&su, &sx, &sy, &sz, &so});
}

int wd_mass_consistency(wd_ctx* ctx, const double* u, double out[2], void* stream) {
    KnobScope knobs_(ctx);
    if (!ctx || !u || !out) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Stage su;
    RC(stage_in(ctx, su, u, abi_elems(ctx), st));
    const int nb = 1184;
    const int np = (int)ctx->parts.size();
    double* per = ctx->dscal + 3000;   // 2 per part
    for (int p = 0; p < np; p++) {
        Part& P = ctx->parts[p];
        Level& F = P.lev[0];
        // D1(u) = -(RHS kernel applied to u) (reading C12), natural layout in the r buffer
        Nat d;
        d.p = F.r;
        d.n2a = F.L.n2;
        d.jofs = 0;
        launch_rhs(P.X, P.Y, P.Z, F.L, nat_elems(ctx, P, su.d), d, st);
        launch_free_norms(F.L, F.r, P.partial, nb, per + 2 * p, st);
    }
    CKL();
    std::vector<double> h;
    if (ctx->mode == MODE_NCCL) {
        double* all = ctx->dscal + 3200;
        NK(nccl().AllGather(per, all, 2, ncclDouble, ctx->comm, st));
        h.resize(2 * ctx->nranks);
        CK(cudaMemcpyAsync(h.data(), all, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
    } else {
        h.resize(2 * np);
        CK(cudaMemcpyAsync(h.data(), per, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    double s2 = 0.0, mx = 0.0;
    for (size_t r = 0; r < h.size() / 2; r++) {   // rank order
        s2 += h[2 * r];
        mx = std::max(mx, h[2 * r + 1]);
    }
    out[0] = std::sqrt(s2);
    out[1] = mx;
    return stage_finish(st, {&su});
}

int wd_downscale_step(wd_ctx* ctx, const double* u0, double* lambda, int warm, double rel_tol,
                      double* u, wd_report* rep, void* stream) {
    KnobScope knobs_(ctx);
    Nvtx nvtx_("wd_downscale_step");
    if (!ctx || !u0 || !lambda || !u) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    // host arrays cross PCIe once: u0 up, (lambda up when warm), lambda and u down
    Stage sf, su0, sl, su;
    sf.ctx = ctx;
    sf.bytes = sizeof(double) * abi_nodes(ctx);
    sf.staged = true;   // a pooled device scratch for f (released by stage_finish)
    RC(stage_acquire(ctx, sf, sf.bytes));
    RC(stage_in(ctx, su0, u0, abi_elems(ctx), st));
    if (warm) RC(stage_in(ctx, sl, lambda, abi_nodes(ctx), st));
    else RC(stage_out(ctx, sl, lambda, abi_nodes(ctx)));
    sl.out = true;
    sl.host = lambda;
    RC(stage_out(ctx, su, u, abi_elems(ctx)));
    int rc = wd_rhs(ctx, su0.d, sf.d, stream);
    int rs = rc ? rc : wd_solve(ctx, sf.d, warm ? sl.d : nullptr, rel_tol, sl.d, rep, stream);
    if (rs == WD_OK || rs == WD_E_NOCONV) rc = wd_recover_wind(ctx, sl.d, su0.d, su.d, stream);
    const int rf = stage_finish(st, {&sf, &su0, &sl, &su});
    if (rs) return rs;
    return rc ? rc : rf;
}

int wd_vcycle(wd_ctx* ctx, double* lambda, const double* f, double* rel_res_out, void* stream) {
    KnobScope knobs_(ctx);
    Nvtx nvtx_("wd_vcycle");
    if (!ctx || !lambda || !f) return fail(WD_E_INVAL, "NULL argument");
    RoleGuard roles(ctx);
    cudaStream_t st = (cudaStream_t)stream;
    Stage sl, sf;
    RC(stage_in(ctx, sl, lambda, abi_nodes(ctx), st));
    RC(stage_in(ctx, sf, f, abi_nodes(ctx), st));
    for (Part& P : ctx->parts) {
        launch_nat2int(P.lev[0].L, nat_nodes(ctx, P, sf.d), P.lev[0].f, true, st);
        launch_nat2int(P.lev[0].L, nat_nodes(ctx, P, sl.d), P.lev[0].lam, true, st);
    }
    CKL();
    // the caller's halo rows need not be current (outputs cover owned rows)
    RC(exchange(ctx, 0, ARR_F, 2, st));
    RC(exchange(ctx, 0, ARR_LAM, 2, st));
    RC(run_vcycle(ctx, st));
    if (rel_res_out) {
        RC(residual_sq(ctx, 0, st));
        RC(norm_sq(ctx, ARR_F, 1, st));
        RC(fetch_scalars(ctx, 2, st));
        const double a = std::sqrt(ctx->hscal[0]), fn = std::sqrt(ctx->hscal[1]);
        *rel_res_out = fn > 0 ? a / fn : a;
        profile_accumulate(ctx, true, true);
    }
    sl.out = true;
    sl.host = lambda;
    out_nodes(ctx, sl.d, st);
    CKL();
    return stage_finish(st, {&sl, &sf});
}

int wd_solve(wd_ctx* ctx, const double* f, const double* lambda0, double rel_tol, double* lambda,
             wd_report* rep, void* stream) {
    KnobScope knobs_(ctx);
    Nvtx nvtx_("wd_solve");
    if (!ctx || !f || !lambda) return fail(WD_E_INVAL, "NULL argument");
    RoleGuard roles(ctx);
    if (!(rel_tol > 0.0 && rel_tol < 1.0)) return fail(WD_E_INVAL, "rel_tol must be in (0,1)");
    cudaStream_t st = (cudaStream_t)stream;
    ctx->pend_first = ctx->pend_rest = false;
    Stage sf, s0, sl;
    RC(stage_in(ctx, sf, f, abi_nodes(ctx), st));
    if (lambda0) RC(stage_in(ctx, s0, lambda0, abi_nodes(ctx), st));
    RC(stage_out(ctx, sl, lambda, abi_nodes(ctx)));
    for (Part& P : ctx->parts) {
        Level& F = P.lev[0];
        launch_nat2int(F.L, nat_nodes(ctx, P, sf.d), F.f, true, st);
        if (lambda0) launch_nat2int(F.L, nat_nodes(ctx, P, s0.d), F.lam, true, st);
        else CK(cudaMemsetAsync(F.lam, 0, sizeof(double) * F.L.NT, st));
    }
    CKL();
    // the caller's halo rows need not be current (outputs cover owned rows)
    RC(exchange(ctx, 0, ARR_F, 2, st));
    RC(exchange(ctx, 0, ARR_LAM, 2, st));
    wd_report R;
    memset(&R, 0, sizeof R);
    R.nlevels = ctx->nlev;
    for (int l = 0; l < ctx->nlev && l < 32; l++)
        for (int d = 0; d < 3; d++) R.dims[l][d] = ctx->levdims[l][d];
    R.coarse_direct = ctx->coarse_direct;
    R.coarse_free = ctx->nf;
    RC(norm_sq(ctx, ARR_F, 1, st));
    // convergence test of iterate c: ||f - K lam_c|| / ||f||.  With the fused
    // smoother it is normally taken from the first sweep of cycle c+1, which
    // reads lam_c unchanged (ping-pong) and returns its residual (RES variant);
    // when the test passes, lam_c is still in the canonical buffer and the
    // sweep's output is dropped.  A separate residual pass is used for the
    // warm start when the split is not available, at the cycle cap, and after
    // a cycle predicted (from the last two factors) to reach rel_tol.  Either
    // way the test sees the same quantity after every cycle, so the cycle
    // count is the one of "cycle, then test".
    const bool lag = lagged_residual(ctx);
    bool have = true;   // hscal[0] holds ||r||^2 of the current iterate
    if (lambda0 && !lag) {
        RC(residual_sq(ctx, 0, st));
        RC(fetch_scalars(ctx, 2, st));
        profile_accumulate(ctx, false, true);
    } else if (lambda0) {
        RC(fetch_scalars(ctx, 2, st));
        have = false;
    } else {
        // zero start: f - K 0 = f exactly, no residual pass needed
        RC(fetch_scalars(ctx, 2, st));
        ctx->hscal[0] = ctx->hscal[1];
    }
    const double fn = std::sqrt(ctx->hscal[1]);
    int status = WD_E_NOCONV;
    int c = 0;
    // the last four residuals, the one after cycle 1 and the last one are kept
    // here (rel_res_hist only reports the first 256 cycles)
    double ring4[4] = {0.0, 0.0, 0.0, 0.0}, rel1 = 0.0, rel_last = 0.0;
    if (fn == 0.0) {
        for (Part& P : ctx->parts) CK(cudaMemsetAsync(P.lev[0].lam, 0, sizeof(double) * P.lev[0].L.NT, st));
        R.rel_res_hist[0] = 0.0;
        status = WD_OK;
    } else if (use_device_loop(ctx, lag)) {
        LoopDev* H = ctx->looph;
        memset(H, 0, sizeof *H);
        H->fn = fn;
        H->tol = rel_tol;
        H->max_cycles = ctx->opt.max_cycles;
        H->first_done = have ? 0 : 1;
        H->status = -1;
        CK(cudaMemcpyAsync(ctx->loopd, H, sizeof *H, cudaMemcpyHostToDevice, st));
        if (have)   // zero start: the residual of lam = 0 is f
            CK(cudaMemcpyAsync(ctx->dscal, ctx->dscal + 1, sizeof(double), cudaMemcpyDeviceToDevice, st));
        else        // warm start: cycle 1's first sweep returns the residual of lam0
            RC(run_split(ctx, 0, st));
        CK(cudaGraphLaunch(ctx->g_loop, st));
        CK(cudaMemcpyAsync(H, ctx->loopd, sizeof *H, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        c = H->c;
        status = H->status;
        memcpy(R.rel_res_hist, H->hist, sizeof(double) * std::min(c + 1, 256));
        R.rel_res0 = H->rel0;
        rel1 = H->rel1;
        rel_last = H->rel_last;
        // the iterate is in the canonical buffer whichever way the loop ended
        for (Part& P : ctx->parts) {
            P.lev[0].lam = P.lev[0].raw[1];
            P.lev[0].lam2 = P.lev[0].raw[4];
        }
        // kernels executed: one test per test (c + 1), per cycle the post
        // kernel and the rest of the cycle, plus the bodies the conditions
        // selected (a warm start's first sweep counted by run_split)
        g_launches += (long long)(c + 1) + (long long)c * (1 + ctx->kl_rest) +
                      H->n_first_res * ctx->kl_first_res + H->n_first * ctx->kl_first +
                      H->n_res * ctx->kl_res;
    } else {
        for (;;) {
            Nvtx n_cyc("cycle %d", c + 1);
            bool first_done = false;
            if (!have) {   // first sweep of cycle c+1, returning the residual of lam_c
                profile_first(ctx);    // the previous cycle's, before its events are reused
                ctx->cyc_par ^= 1;
                ctx->cyc_evented = c % PROF_EVERY == 0;
                RC(run_split(ctx, 0, st));
                ctx->prof[11] += 1;
                RC(fetch_scalars(ctx, 1, st));
                profile_rest(ctx);     // the previous cycle has finished
                ctx->pend_first = ctx->cyc_evented;
                ctx->pend_first_res = true;
                first_done = true;
            }
            const double rel = std::sqrt(ctx->hscal[0]) / fn;
            if (c < 256) R.rel_res_hist[c] = rel;
            if (c == 0) R.rel_res0 = rel;
            if (c == 1) rel1 = rel;
            ring4[c & 3] = rel;
            rel_last = rel;
            if (!std::isfinite(rel)) status = WD_E_NONFINITE;
            else if (rel <= rel_tol) status = WD_OK;
            else if (c >= 3 && rel > 10.0 * ring4[(c - 3) & 3]) status = WD_E_DIVERGED;
            else if (c >= ctx->opt.max_cycles) status = WD_E_NOCONV;
            else status = -1;   // continue
            if (status != -1) {
                if (first_done)   // drop the sweep: lam_c is the result
                    for (Part& P : ctx->parts) std::swap(P.lev[0].lam, P.lev[0].lam2);
                break;
            }
            if (!lag) {
                RC(run_vcycle(ctx, st));
                RC(residual_sq(ctx, 0, st));
                RC(fetch_scalars(ctx, 1, st));
                c++;
                profile_accumulate(ctx, true, true);
                continue;
            }
            if (!first_done) {
                profile_first(ctx);
                ctx->cyc_par ^= 1;
                ctx->cyc_evented = c % PROF_EVERY == 0;
                RC(run_split(ctx, 1, st));
                ctx->prof[10] += 1;
                ctx->pend_first = ctx->cyc_evented;
                ctx->pend_first_res = false;
            }
            ctx->first_res = first_done;
            profile_rest(ctx);   // (already read: a no-op)
            RC(run_split(ctx, 2, st));
            ctx->prof[10] += std::max(ctx->opt.pre_smooth + ctx->opt.post_smooth - 1, 0);
            ctx->pend_rest = ctx->opt.profile;
            ctx->pend_rest_sweeps = ctx->cyc_evented;
            ctx->pend_par = ctx->cyc_par;
            c++;
            const double prev = c >= 2 ? ring4[(c - 2) & 3] : 0.0;
            const bool predicted = prev > 0.0 && rel * (rel / prev) <= rel_tol;
            if (predicted || c >= ctx->opt.max_cycles) {
                RC(residual_sq(ctx, 0, st));
                RC(fetch_scalars(ctx, 1, st));
                profile_first(ctx);
                profile_rest(ctx);
                profile_accumulate(ctx, false, true);
                have = true;
            } else {
                have = false;
            }
        }
    }
    if (ctx->opt.profile && (ctx->pend_first || ctx->pend_rest)) {
        CK(cudaStreamSynchronize(st));
        profile_first(ctx);
        profile_rest(ctx);
    }
    R.cycles = c;
    R.status = status;
    R.converged = status == WD_OK;
    if (fn != 0.0) R.rel_res_final = rel_last;
    if (c >= 2) R.rate = std::pow(rel_last / rel1, 1.0 / (c - 1));
    else if (c == 1) R.rate = rel_last / R.rel_res0;
    out_nodes(ctx, sl.d, st);
    CKL();
    RC(stage_finish(st, {&sf, &s0, &sl}));
    if (rep) *rep = R;
    if (status == WD_E_NOCONV) return fail(WD_E_NOCONV, "not converged after %d cycles (rel %.3e)", c, R.rel_res_final);
    if (status == WD_E_DIVERGED) return fail(WD_E_DIVERGED, "diverged at cycle %d", c);
    if (status == WD_E_NONFINITE) return fail(WD_E_NONFINITE, "non-finite residual at cycle %d", c);
    return WD_OK;
}

// ------------------------------------------------------------------ profiling
int wd_profile_read(const wd_ctx* ctx, double* out, int n) {
    if (!ctx || !out) return 0;
    int m = n < 12 ? n : 12;
    for (int t = 0; t < m; t++) out[t] = ctx->prof[t];
    return m;
}

void wd_profile_reset(wd_ctx* ctx) {
    if (ctx)
        for (double& v : ctx->prof) v = 0.0;
}

long long wd_launch_count(void) { return g_launches.load(); }

int wd_bench_kernel(wd_ctx* ctx, int which, int level, int reps, double* ms_out) {
    KnobScope knobs_(ctx);
    RC(check_level(ctx, level));
    RC(check_single(ctx));
    RoleGuard roles(ctx);
    if (reps < 1 || !ms_out) return fail(WD_E_INVAL, "reps < 1 or NULL output");
    if ((which == 2 || which == 3 || which == 6) && level >= ctx->nlev - 1)
        return fail(WD_E_INVAL, "no coarser level");
    cudaStream_t st = ctx->cap;
    Part& P = ctx->parts[0];
    Level& F = P.lev[level];
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto body = [&]() -> int {
        switch (which) {
            case 0:   // two sweeps (the V-cycle's pairs: no copy-back), reported per sweep
                RC(smooth(ctx, level, false, 0, st));
                RC(smooth(ctx, level, false, 0, st));
                return smooth_end(ctx, level, st);
            case 8: launch_gs_sweep(F.L, F.coef, F.lam, F.f, st); break;
            case 9:   // two fused sweeps of the residual variant, reported per sweep
                for (int t = 0; t < 2; t++) {
                    gs_sweep_level(F, st, P.partial);
                    std::swap(F.lam, F.lam2);
                }
                return smooth_end(ctx, level, st);
            case 1: apply_level(F, true, nullptr, st); break;
            case 2: launch_restrict(F.L, target(P.lev[level + 1]), F.M, F.r, P.lev[level + 1].f, F.nkept == F.L.n3, st); break;
            case 3: launch_prolong(F.L, P.lev[level + 1].L, F.M, P.lev[level + 1].lam, F.lam, F.nkept == F.L.n3, st); break;
            case 4: return run_vcycle(ctx, st);
            case 5: return residual_sq(ctx, 0, st);
            case 6: launch_galerkin(F.L, target(P.lev[level + 1]), F.M, F.coef, P.lev[level + 1].coef, F.nkept == F.L.n3, st); break;
            case 7: {
                unsigned long long* dbad = (unsigned long long*)(ctx->dscal + 8);
                launch_assemble(P.X, P.Y, P.Z, ctx->n1, ctx->n2, ctx->n3, ctx->c, P.lev[0].L,
                                P.lev[0].coef, dbad, st);
                break;
            }
            default: return fail(WD_E_INVAL, "unknown kernel %d", which);
        }
        return WD_OK;
    };
    RC(body());   // warm-up
    CK(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; r++) RC(body());
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / reps / (which == 0 || which == 9 ? 2 : 1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CKL();
    return WD_OK;
}

// ------------------------------------------------------------------ inspection
int wd_num_levels(const wd_ctx* ctx) { return ctx ? ctx->nlev : 0; }

int wd_level_dims(const wd_ctx* ctx, int level, int dims[3]) {
    RC(check_level(ctx, level));
    for (int d = 0; d < 3; d++) dims[d] = ctx->levdims[level][d];
    return WD_OK;
}

int wd_level_plan(const wd_ctx* ctx, int level, int* horizontal, int* kept, int* nkept) {
    RC(check_level(ctx, level));
    if (level >= ctx->nlev - 1) return fail(WD_E_INVAL, "level %d is the coarsest", level);
    const Level& lv = ctx->parts[0].lev[level];
    *horizontal = lv.hflag;
    *nkept = lv.nkept;
    for (int t = 0; t < lv.nkept; t++) kept[t] = lv.kept[t];
    return WD_OK;
}

int wd_gather_level(const wd_ctx* ctx) { return ctx ? (ctx->gather < MAXLEV ? ctx->gather : -1) : -1; }

int wd_get_stencil(wd_ctx* ctx, int level, double* K27, void* stream) {
    KnobScope knobs_(ctx);
    RC(check_level(ctx, level));
    RC(check_single(ctx));
    cudaStream_t st = (cudaStream_t)stream;
    Level& lv = ctx->parts[0].lev[level];
    Stage so;
    RC(stage_out(ctx, so, K27, 27 * nodes_of(lv.L)));
    launch_export27(lv.L, lv.coef, so.d, st);
    CKL();
    return stage_finish(st, {&so});
}

static Nat whole(const LevDev& L, const double* p) {
    Nat a;
    a.p = p;
    a.n2a = L.n2;
    a.jofs = 0;
    return a;
}

int wd_apply(wd_ctx* ctx, int level, const double* x, double* y, void* stream) {
    KnobScope knobs_(ctx);
    RC(check_level(ctx, level));
    RC(check_single(ctx));
    cudaStream_t st = (cudaStream_t)stream;
    Level& lv = ctx->parts[0].lev[level];
    const size_t N = nodes_of(lv.L);
    Stage sx, sy;
    RC(stage_in(ctx, sx, x, N, st));
    RC(stage_out(ctx, sy, y, N));
    launch_nat2int(lv.L, whole(lv.L, sx.d), lv.lam, true, st);
    CK(cudaMemsetAsync(lv.r, 0, sizeof(double) * lv.L.NT, st));
    apply_level(lv, false, nullptr, st);
    launch_int2nat(lv.L, lv.r, whole(lv.L, sy.d), st);
    CKL();
    return stage_finish(st, {&sx, &sy});
}

int wd_smooth(wd_ctx* ctx, int level, double* x, const double* f, int sweeps, void* stream) {
    KnobScope knobs_(ctx);
    RC(check_level(ctx, level));
    RC(check_single(ctx));
    RoleGuard roles(ctx);
    cudaStream_t st = (cudaStream_t)stream;
    Level& lv = ctx->parts[0].lev[level];
    const size_t N = nodes_of(lv.L);
    Stage sx, sf;
    RC(stage_in(ctx, sx, x, N, st));
    RC(stage_in(ctx, sf, f, N, st));
    launch_nat2int(lv.L, whole(lv.L, sx.d), lv.lam, true, st);
    launch_nat2int(lv.L, whole(lv.L, sf.d), lv.f, true, st);
    for (int s = 0; s < sweeps; s++) RC(smooth(ctx, level, false, 0, st));
    RC(smooth_end(ctx, level, st));
    sx.out = true;
    sx.host = x;
    launch_int2nat(lv.L, lv.lam, whole(lv.L, sx.d), st);
    CKL();
    return stage_finish(st, {&sx, &sf});
}

int wd_restrict(wd_ctx* ctx, int level, const double* r, double* fc, void* stream) {
    KnobScope knobs_(ctx);
    RC(check_level(ctx, level));
    RC(check_single(ctx));
    if (level >= ctx->nlev - 1) return fail(WD_E_INVAL, "no coarser level");
    cudaStream_t st = (cudaStream_t)stream;
    Level& F = ctx->parts[0].lev[level];
    Level& C = ctx->parts[0].lev[level + 1];
    Stage sr, sc;
    RC(stage_in(ctx, sr, r, nodes_of(F.L), st));
    RC(stage_out(ctx, sc, fc, nodes_of(C.L)));
    launch_nat2int(F.L, whole(F.L, sr.d), F.r, true, st);
    CK(cudaMemsetAsync(C.f, 0, sizeof(double) * C.L.NT, st));
    launch_restrict(F.L, target(C), F.M, F.r, C.f, F.nkept == F.L.n3, st);
    launch_int2nat(C.L, C.f, whole(C.L, sc.d), st);
    CKL();
    return stage_finish(st, {&sr, &sc});
}

int wd_prolong(wd_ctx* ctx, int level, const double* xc, double* x, void* stream) {
    KnobScope knobs_(ctx);
    RC(check_level(ctx, level));
    RC(check_single(ctx));
    if (level >= ctx->nlev - 1) return fail(WD_E_INVAL, "no coarser level");
    cudaStream_t st = (cudaStream_t)stream;
    Level& F = ctx->parts[0].lev[level];
    Level& C = ctx->parts[0].lev[level + 1];
    Stage sc, sx;
    RC(stage_in(ctx, sc, xc, nodes_of(C.L), st));
    RC(stage_in(ctx, sx, x, nodes_of(F.L), st));
    launch_nat2int(C.L, whole(C.L, sc.d), C.lam, true, st);
    launch_nat2int(F.L, whole(F.L, sx.d), F.lam, true, st);
    launch_prolong(F.L, C.L, F.M, C.lam, F.lam, F.nkept == F.L.n3, st);
    sx.out = true;
    sx.host = x;
    launch_int2nat(F.L, F.lam, whole(F.L, sx.d), st);
    CKL();
    return stage_finish(st, {&sc, &sx});
}

int wd_coarse_solve(wd_ctx* ctx, const double* f, double* x, void* stream) {
    KnobScope knobs_(ctx);
    if (!ctx || !f || !x) return fail(WD_E_INVAL, "NULL argument");
    RC(check_single(ctx));
    RoleGuard roles(ctx);
    cudaStream_t st = (cudaStream_t)stream;
    Level& lc = ctx->parts[0].lev[ctx->nlev - 1];
    const size_t N = nodes_of(lc.L);
    Stage sf, sx;
    RC(stage_in(ctx, sf, f, N, st));
    RC(stage_out(ctx, sx, x, N));
    launch_nat2int(lc.L, whole(lc.L, sf.d), lc.f, true, st);
    CK(cudaMemsetAsync(lc.lam, 0, sizeof(double) * lc.L.NT, st));
    RC(coarse_solve(ctx, st));
    launch_int2nat(lc.L, lc.lam, whole(lc.L, sx.d), st);
    CKL();
    return stage_finish(st, {&sf, &sx});
}

int wd_residual_norm(wd_ctx* ctx, const double* x, const double* f, double* abs_out,
                     double* rel_out, void* stream) {
    KnobScope knobs_(ctx);
    if (!ctx || !x || !f) return fail(WD_E_INVAL, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    Stage sx, sf;
    RC(stage_in(ctx, sx, x, abi_nodes(ctx), st));
    RC(stage_in(ctx, sf, f, abi_nodes(ctx), st));
    for (Part& P : ctx->parts) {
        launch_nat2int(P.lev[0].L, nat_nodes(ctx, P, sx.d), P.lev[0].lam, true, st);
        launch_nat2int(P.lev[0].L, nat_nodes(ctx, P, sf.d), P.lev[0].f, true, st);
    }
    CKL();
    RC(residual_sq(ctx, 0, st));
    RC(norm_sq(ctx, ARR_F, 1, st));
    RC(fetch_scalars(ctx, 2, st));
    const double a = std::sqrt(ctx->hscal[0]), fn = std::sqrt(ctx->hscal[1]);
    if (abs_out) *abs_out = a;
    if (rel_out) *rel_out = fn > 0 ? a / fn : a;
    return stage_finish(st, {&sx, &sf});
}

}  // extern "C"
