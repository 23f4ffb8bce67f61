// parareal.cu — C ABI (include/parareal.h) and host runtime of the B200 hot
// path: nu tables, CUDA-graph batches of stencil steps, the Parareal driver
// (Alg.1) and its NCCL point-to-point pipeline.
//
// Nothing here includes or calls the CPU oracle (oracle/); this file and
// kernels.cuh are the whole product path.
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/parareal.h"
#include "kernels.cuh"
#include "fused.cuh"
#include "comb.cuh"
#include "onestep.cuh"
#include "z2.cuh"

namespace prk {
// two z planes per consumer iteration: 6-slot intermediate ring; K_A input ring 9 slots, K_B 8
using FusedZ2 = WithZ2<FusedCfgP<16, 8, 6, 2, 2, 2, 2, 0, 9>>;
}  // namespace prk

using namespace prk;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

static pr_status fail(pr_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(e_ == cudaErrorMemoryAllocation ? PR_ENOMEM : PR_ECUDA,            \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                        \
    } while (0)
#define CKS(expr)                          \
    do {                                   \
        pr_status s_ = (expr);             \
        if (s_ != PR_OK) return s_;        \
    } while (0)
#define CKL()                                                                              \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess)                                                             \
            return fail(PR_ECUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                               \
    } while (0)

// ------------------------------------------------------------------ grid
namespace {

struct LaunchCfg {
    int tiles_x = 0, tiles_y = 0, cz = 0, chunks_z = 0, blocks = 0, occ = 0, threads = 0;
    size_t smem = 0;
};

struct NuTable {
    double *d = nullptr;
    size_t cap = 0;          // doubles
    int64_t lo = 0, hi = 0;  // global step range covered
    double dt = 0.0;
    bool valid = false;
};

constexpr int FINE_BATCH = 16;    // RK4 steps per CUDA graph (64 kernels)
constexpr int COARSE_PAIRS = 16;  // Euler step pairs per CUDA graph (32 kernels)

// In-process rank group (pr_local_group): W grids of one process (on one device or
// several) linked as ranks 0..W-1 of the time-slice pipeline without NCCL.  The
// hand-off data path is the peer path's (the correction kernel stores u^{k+1} into the
// successor's receive buffer); ordering goes through CUDA events whose records the
// ranks' host threads announce to each other here, so no stream or kernel ever waits
// on a value another rank has not yet been told to produce.
struct LocalRank {
    unsigned long long started = 0;  // base + 1 of the call in progress (0: none yet)
    unsigned long long data = 0;     // last hand-off published: base + k + 1
    unsigned long long freed = 0;    // last receive-buffer release published: base + k + 1
    double *mail[2] = {nullptr, nullptr};  // this rank's two receive buffers (k even / odd)
    std::vector<cudaEvent_t> ev_data, ev_free;  // recorded on the rank's stream per iteration
    int dev = 0;
};
struct LocalGroup {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<LocalRank> r;
    ~LocalGroup() {
        for (LocalRank &x : r) {
            cudaSetDevice(x.dev);
            for (cudaEvent_t e : x.ev_data) cudaEventDestroy(e);
            for (cudaEvent_t e : x.ev_free) cudaEventDestroy(e);
        }
    }
};

}  // namespace

struct pr_grid {
    int dev = 0;
    int variant = 0;                    // stencil tile variant (PR_TILE env, tuning)
    bool f1 = false;                    // F as ONE kernel per RK4 step (variant 24, NEXT-1)
    bool wparam = false;                // fused F launched directly, weights as parameters
    bool pdl = false;                   // fused F with programmatic dependent launch (PR_PDL=1)
    bool f2 = false;                    // fused two-kernel RK4 step (tile-aligned n)
    int fvariant = 14;                  // fused F variant (PR_FTILE; default set per n below)
    bool c2 = false;                    // persistent TMA-fed G kernel (n % 32 == 0; PR_C2=0 disables)
    int cvariant = 0;                   // its variant (PR_CTILE 0..2)
    LaunchCfg lcp;                      // its launch config
    LaunchCfg lf[2];                    // launch configs of fused_persist_kernel<K_A>, <K_B>
    pr_problem prob{};
    int n = 0;
    int64_t N = 0;
    size_t bytes = 0;
    int sms = 0;
    cudaStream_t cap_stream = nullptr;  // private stream used only for graph capture
    double *acc = nullptr, *ya = nullptr, *yb = nullptr, *ctmp = nullptr;
    double *d_sine = nullptr;
    long long *d_pos = nullptr;             // [0] fine cursor, [1] coarse cursor
    unsigned long long *d_red = nullptr;    // reduction slots
    unsigned long long *h_red = nullptr;    // pinned mirror
    int red_cap = 0;
    NuTable tab_f, tab_c;
    double *h_stage = nullptr;              // pinned staging for nu tables
    size_t h_stage_cap = 0;
    cudaEvent_t stage_ev = nullptr;         // last table upload
    LaunchCfg lc[5];
    // cached CUDA graphs keyed by (kind, state buffer); each remembers the exact step
    // size and nu-table pointer it was captured with
    struct CachedGraph {
        cudaGraphExec_t exec;
        double dt;
        const double *tab;
    };
    std::map<std::pair<int, const void *>, CachedGraph> graphs;
    // host-pointer staging
    double *stage_a = nullptr, *stage_b = nullptr;
    // Parareal state
    int par_s = 0;
    std::vector<double *> pool;
    // NCCL
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> evs, dep_evs;
    double timings[5] = {0, 0, 0, 0, 0};
    std::vector<double> monitors;           // iterate-change monitor of the last pr_parareal
    int iters = 0;                          // iterations it ran
    double *h_flag = nullptr;               // pinned: received stop flag
    pr_status launch_err = PR_OK;           // sticky error of an enqueue helper (TMA map encode)
    // peer hand-off (PR_FLAG_PEER_HANDOFF): flag words [0] data sequence (written by the
    // predecessor), [1] free sequence (written by the successor); IPC mappings of the
    // successor's two receive buffers and flag words and of the predecessor's flag words
    unsigned int *d_flags = nullptr;
    unsigned char *d_ipc = nullptr;         // all-gather staging of the IPC handles
    double *peer_mail[2] = {nullptr, nullptr};
    unsigned int *succ_flags = nullptr, *pred_flags = nullptr;
    std::vector<void *> ipc_open;
    long long pool_gen = 0, mapped_gen = -1;
    unsigned int seq_base = 0;              // advances by K + 2 per peer-mode pr_parareal
    // spatially coarsened G (NEXT-4): a child grid on the n/2 mesh and one field there
    pr_grid *half = nullptr;
    double *half_u = nullptr;
    // concurrent F over a slice group (NEXT-2, small n): one child grid (own RK4 scratch,
    // nu table, graphs) and one stream per slice; fork / join events
    std::vector<pr_grid *> slice_grids;
    std::vector<cudaStream_t> slice_streams;
    std::vector<cudaEvent_t> slice_events;  // [0] fork, [1 + l] join of slice l
    // in-process rank group (pr_local_group): shared state, this grid's rank, and the
    // grid's own compute stream (the caller's stream is joined by events)
    std::shared_ptr<LocalGroup> lgroup;
    cudaStream_t work_stream = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // peer hand-off ordering on the consumer side: CU_STREAM_WAIT_VALUE_FLUSH if the
    // device can flush remote writes (-1: not queried yet)
    int can_flush = -1;
};

// cuStreamWaitValue32 through the runtime's driver entry point: the stream's
// front end waits on a 32-bit word (no kernel spins).
static PFN_cuStreamWaitValue32_v11070 stream_wait_fn() {
    static PFN_cuStreamWaitValue32_v11070 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
    }();
    return fn;
}

// ------------------------------------------------------------------ TMA tensor maps
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// 3-D map of an n^3 fp64 field (x fastest), box bx x by x 1 (one z plane of a tile)
static bool tma_encode3(CUtensorMap *m, const double *p, int n, int bx, int by) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tma_encoder();
    if (!enc || !p) return false;
    const cuuint64_t dims[3] = {cuuint64_t(n), cuuint64_t(n), cuuint64_t(n)};
    const cuuint64_t strides[2] = {cuuint64_t(n) * 8, cuuint64_t(n) * n * 8};
    const cuuint32_t box[3] = {cuuint32_t(bx), cuuint32_t(by), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// z-chunk count that fills whole waves of resident CTAs with little halo re-read
static int pick_chunks(int n, int tiles, int slots, int halo) {
    int best_chunks = 1;
    double best = -1.0;
    const int min_cz = std::min(n, 8);
    for (int ch = 1; ch <= n / min_cz; ++ch) {
        const int cz = (n + ch - 1) / ch;
        const int che = (n + cz - 1) / cz;
        const long items = long(tiles) * che;
        const long waves = (items + slots - 1) / slots;
        const double eff = double(items) / double(waves * slots);
        const double over = 1.0 + 0.5 * double(2 * halo) / double(cz);
        const double score = eff / over;
        if (score > best + 1e-9) { best = score; best_chunks = che; }
    }
    if (const char *env = getenv("PR_CHUNKS_Z")) {
        int v = atoi(env);
        if (v >= 1 && v <= n) best_chunks = v;
    }
    return best_chunks;
}

template <int KIND, class C>
static pr_status setup_kind_cfg(pr_grid *g) {
    const size_t smem = Layout<KIND, C>::SMEM_BYTES;
    CK(cudaFuncSetAttribute(stencil_kernel<KIND, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil_kernel<KIND, C>, C::NTHREADS,
                                                     smem));
    if (occ < 1) return fail(PR_ECUDA, "stencil kernel %d cannot be resident", KIND);
    LaunchCfg &c = g->lc[KIND];
    const int n = g->n;
    c.occ = occ;
    c.threads = C::NTHREADS;
    c.smem = smem;
    c.tiles_x = (n + TX - 1) / TX;
    c.tiles_y = (n + C::TY - 1) / C::TY;
    const int tiles = c.tiles_x * c.tiles_y;
    const int slots = g->sms * occ;
    const int best_chunks = pick_chunks(n, tiles, slots, Traits<KIND>::R);
    c.cz = (n + best_chunks - 1) / best_chunks;
    c.chunks_z = (n + c.cz - 1) / c.cz;
    c.blocks = tiles * c.chunks_z;
    return PR_OK;
}

template <int KIND>
static pr_status setup_kind(pr_grid *g) {
    switch (g->variant) {
#ifdef PRK_VARIANTS
    case 1: return setup_kind_cfg<KIND, Tile1>(g);
    case 2: return setup_kind_cfg<KIND, Tile2>(g);
    case 3: return setup_kind_cfg<KIND, Tile3>(g);
#endif
    case 0: return setup_kind_cfg<KIND, Tile0>(g);
    default: return fail(PR_EINVAL, "four-stage tile variant %d is not built (PRK_VARIANTS)", g->variant);
    }
}

// the kernel of a fused-F config: separate stage-B warps (fused.cuh) or stage B in the
// stage-A lanes (comb.cuh)
template <int KB, class C>
static constexpr auto fused_kernel_of() {
    if constexpr (std::is_same_v<C, OneCfg>) return &onestep_kernel<KB, C>;
    else if constexpr (C::COMB) return &fused_comb_kernel<KB, C>;
    else if constexpr (C::Z2) return &fused_z2_kernel<KB, C>;
    else return &fused_persist_kernel<KB, C>;
}

template <int KB, class C>
static pr_status setup_fused_persist(pr_grid *g) {
    const size_t smem = C::template smem_bytes<KB>();
    constexpr auto kern = fused_kernel_of<KB, C>();
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, smem));
    if (occ < 1) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        return fail(PR_ECUDA,
                    "persistent fused kernel %d cannot be resident (%d threads, %d regs, %zu B smem, "
                    "max threads %d)",
                    KB, C::NT, fa.numRegs, smem, fa.maxThreadsPerBlock);
    }
    LaunchCfg &c = g->lf[KB];
    const int n = g->n;
    c.occ = occ;
    c.threads = C::NT;
    c.smem = smem;
    c.tiles_x = n / C::TXO;
    c.tiles_y = n / C::TYO;
    const int slots = g->sms * occ;
    const int ch = pick_chunks(n, c.tiles_x * c.tiles_y, slots, std::is_same_v<C, OneCfg> ? 8 : 4);
    c.cz = (n + ch - 1) / ch;
    if constexpr (!std::is_same_v<C, OneCfg>) {
        if constexpr (C::Z2) c.cz = (c.cz + 1) & ~1;  // two planes per iteration: even chunks
    }
    c.chunks_z = (n + c.cz - 1) / c.cz;
    const int items = c.tiles_x * c.tiles_y * c.chunks_z;
    c.blocks = std::min(items, slots);  // persistent: one CTA per resident slot
    return PR_OK;
}

template <class C>
static pr_status setup_coarse_persist(pr_grid *g) {
    const size_t smem = C::smem_bytes();
    CK(cudaFuncSetAttribute(coarse_persist_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, coarse_persist_kernel<C>, C::NT, smem));
    if (occ < 1) return fail(PR_ECUDA, "persistent coarse kernel cannot be resident");
    LaunchCfg &c = g->lcp;
    const int n = g->n;
    c.occ = occ;
    c.threads = C::NT;
    c.smem = smem;
    c.tiles_x = n / C::TXO;
    c.tiles_y = n / C::TYO;
    const int slots = g->sms * occ;
    const int ch = pick_chunks(n, c.tiles_x * c.tiles_y, slots, 1);
    c.cz = (n + ch - 1) / ch;
    c.chunks_z = (n + c.cz - 1) / c.cz;
    c.blocks = std::min(c.tiles_x * c.tiles_y * c.chunks_z, slots);
    return PR_OK;
}

static pr_status setup_coarse(pr_grid *g) {
    switch (g->cvariant) {
#ifdef PRK_VARIANTS
    case 1: return setup_coarse_persist<CoarseP1>(g);
    case 2: return setup_coarse_persist<CoarseP2>(g);
#endif
    case 0: return setup_coarse_persist<CoarseP0>(g);
    default: return fail(PR_EINVAL, "coarse variant %d is not built (PRK_VARIANTS)", g->cvariant);
    }
}

template <class C>
static void launch_coarse_persist(pr_grid *g, const StencilArgs &a0, cudaStream_t st) {
    StencilArgs a = a0;
    const LaunchCfg &c = g->lcp;
    a.tiles_x = c.tiles_x;
    a.tiles_y = c.tiles_y;
    a.cz = c.cz;
    a.chunks_z = c.chunks_z;
    TmaMaps tm;
    memset(&tm, 0, sizeof tm);
    if constexpr (C::FILL == 2) {
        if (!tma_encode3(&tm.y, a.y, g->n, C::IWS, C::IH)) {
            g->launch_err = fail(PR_ECUDA, "cuTensorMapEncodeTiled failed (coarse kernel)");
            return;
        }
    }
    coarse_persist_kernel<C><<<c.blocks, c.threads, c.smem, st>>>(a, tm);
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Fused F variants (PR_FTILE): the tile configuration of each of the two kernels
// (K_A: stages 1+2, K_B: stages 3+4; they are independent launches over the whole
// grid, so their tilings may differ).  X(id, config of K_A, config of K_B)
#define PRK_FVARIANTS(X) \
    X(14, FusedP4, FusedP4) X(22, Comb16, Comb16) X(23, FusedTM, FusedTM) X(24, OneCfg, OneCfg) \
    X(25, FusedZ2, FusedZ2)
#ifdef PRK_VARIANTS
// tuning history and timing diagnostics (26-28 give garbage results by design)
#define PRK_FVARIANTS_OLD(X)                                                                    \
    X(10, FusedP0, FusedP0) X(11, FusedP1, FusedP1) X(12, FusedP2, FusedP2) X(13, FusedP3, FusedP3) \
    X(15, FusedP5, FusedP5) X(16, FusedP6, FusedP6) X(17, FusedP7, FusedP7) X(18, FusedP8, FusedP8) \
    X(19, FusedP9, FusedP9) X(20, FusedT32, FusedP4) X(21, FusedT32, FusedT32B)                    \
    X(26, FusedD1, FusedD1) X(27, FusedD2, FusedD2) X(28, FusedD3, FusedD3) X(31, FusedQ16, FusedQ16) \
    X(32, FusedQ8, FusedQ8) X(29, FusedPF, FusedPF) X(33, FusedZD6, FusedP5) X(34, FusedZD8, FusedP5) \
    X(35, FusedSW, FusedSW) X(36, FusedNoPIN, FusedNoPIN) X(37, FusedOFF32, FusedOFF32) X(38, FusedTM2, FusedTM2) X(39, FusedTM3, FusedTM3) \
    X(40, FusedTM, FusedP4) X(41, FusedP4, FusedTM) X(42, FusedTMQ16, FusedTM) X(43, FusedTMACC, FusedTMACC) X(44, FusedTMPF4, FusedTMPF4) \
    X(45, FusedTMPF8, FusedTMPF8)
#else
#define PRK_FVARIANTS_OLD(X)
#endif
template <int KB, class CA, class CB> using PickCfg = std::conditional_t<KB == K_A, CA, CB>;

// output tile heights of a fused variant's two kernels (0, 0: not built)
static void fused_tiles(int v, int *tya, int *tyb) {
    *tya = *tyb = 0;
    switch (v) {
#define X(id, A, B) case id: *tya = A::TYO; *tyb = B::TYO; break;
        PRK_FVARIANTS(X) PRK_FVARIANTS_OLD(X)
#undef X
    default: break;
    }
}

// variants that also exist with the weights as launch parameters (WithWP)
#define PRK_FVARIANTS_WP(X) X(14, FusedP4, FusedP4) X(23, FusedTM, FusedTM) X(25, FusedZ2, FusedZ2)
static bool fused_has_wp(int v) {
    switch (v) {
#define X(id, A, B) case id: return true;
        PRK_FVARIANTS_WP(X)
#undef X
    default: return false;
    }
}

template <int KB>
static pr_status setup_fused(pr_grid *g) {
    if (g->wparam) {
        switch (g->fvariant) {
#define X(id, A, B) case id: return setup_fused_persist<KB, WithWP<PickCfg<KB, A, B>>>(g);
            PRK_FVARIANTS_WP(X)
#undef X
        default: break;
        }
    }
    switch (g->fvariant) {
#define X(id, A, B) case id: return setup_fused_persist<KB, PickCfg<KB, A, B>>(g);
        PRK_FVARIANTS(X) PRK_FVARIANTS_OLD(X)
#undef X
    default: return fail(PR_EINVAL, "fused variant %d is not built (PRK_VARIANTS)", g->fvariant);
    }
}

template <int KB, class C>
static void launch_persist(pr_grid *g, const StencilArgs &a, const LaunchCfg &c, cudaStream_t st) {
    TmaMaps tm;
    memset(&tm, 0, sizeof tm);
    if constexpr (C::FILL == 2) {
        bool ok = tma_encode3(&tm.y, a.y, g->n, C::IWS, C::IH);
        if (KB == K_B) {
            ok = ok && tma_encode3(&tm.u, a.p0, g->n, C::EWS, C::EH);
            ok = ok && tma_encode3(&tm.c, a.p1, g->n, C::TXO, C::TYO);
        }
        if (!ok) {
            g->launch_err = fail(PR_ECUDA, "cuTensorMapEncodeTiled failed (fused kernel %d)", KB);
            return;
        }
    }
    constexpr auto kern = fused_kernel_of<KB, C>();
    if (g->pdl) {  // programmatic dependent launch (the kernel waits with griddepcontrol.wait)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.blocks);
        cfg.blockDim = dim3(c.threads);
        cfg.dynamicSmemBytes = c.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, a, tm) != cudaSuccess)
            g->launch_err = fail(PR_ECUDA, "cudaLaunchKernelEx failed (fused kernel %d)", KB);
        return;
    }
    kern<<<c.blocks, c.threads, c.smem, st>>>(a, tm);
}

template <int KB>
static void launch_fused(pr_grid *g, const StencilArgs &a0, cudaStream_t st) {
    StencilArgs a = a0;
    const LaunchCfg &c = g->lf[KB];
    a.tiles_x = c.tiles_x;
    a.tiles_y = c.tiles_y;
    a.cz = c.cz;
    a.chunks_z = c.chunks_z;
    bool done = false;
    if (g->wparam) {
        switch (g->fvariant) {
#define X(id, A, B) case id: launch_persist<KB, WithWP<PickCfg<KB, A, B>>>(g, a, c, st); done = true; break;
            PRK_FVARIANTS_WP(X)
#undef X
        default: break;
        }
    }
    if (!done) {
        switch (g->fvariant) {
#define X(id, A, B) case id: launch_persist<KB, PickCfg<KB, A, B>>(g, a, c, st); break;
            PRK_FVARIANTS(X) PRK_FVARIANTS_OLD(X)
#undef X
        default: break;
        }
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

static StencilArgs base_args(const pr_grid *g, int kind) {
    StencilArgs a{};
    const LaunchCfg &c = g->lc[kind];
    a.n = g->n;
    a.tiles_x = c.tiles_x;
    a.tiles_y = c.tiles_y;
    a.cz = c.cz;
    a.chunks_z = c.chunks_z;
    a.inv_dx = double(g->n);  // dx = 1/n
    for (int d = 0; d < 3; ++d) a.c[d] = g->prob.c[d];
    return a;
}

template <int KIND>
static void launch_stencil(pr_grid *g, const StencilArgs &a0, cudaStream_t st) {
    StencilArgs a = a0;  // tile decomposition of this kind (occupancy differs per kind)
    const LaunchCfg &c = g->lc[KIND];
    a.tiles_x = c.tiles_x;
    a.tiles_y = c.tiles_y;
    a.cz = c.cz;
    a.chunks_z = c.chunks_z;
    switch (g->variant) {
#ifdef PRK_VARIANTS
    case 1: stencil_kernel<KIND, Tile1><<<c.blocks, c.threads, c.smem, st>>>(a); break;
    case 2: stencil_kernel<KIND, Tile2><<<c.blocks, c.threads, c.smem, st>>>(a); break;
    case 3: stencil_kernel<KIND, Tile3><<<c.blocks, c.threads, c.smem, st>>>(a); break;
#endif
    default: stencil_kernel<KIND, Tile0><<<c.blocks, c.threads, c.smem, st>>>(a); break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// One classical RK4 step as four fused stage passes.
static void enqueue_fine_step(pr_grid *g, const double *u_src, double *u_dst, int j_local,
                              double dt, cudaStream_t st) {
    StencilArgs a = base_args(g, K_S1);
    a.nu_tab = g->tab_f.d;
    a.nu_pos = g->d_pos + 0;
    a.j_local = j_local;
    a.dt = dt;
    // S1: k1 = L(u); acc = u + dt/6 k1; Ya = u + dt/2 k1
    a.y = u_src; a.p0 = nullptr; a.p1 = nullptr; a.o0 = g->acc; a.o1 = g->ya;
    launch_stencil<K_S1>(g, a, st);
    // S2: k2 = L(Ya); acc += dt/3 k2; Yb = u + dt/2 k2
    a.y = g->ya; a.p0 = u_src; a.p1 = g->acc; a.o0 = g->acc; a.o1 = g->yb;
    launch_stencil<K_S2>(g, a, st);
    // S3: k3 = L(Yb); acc += dt/3 k3; Ya = u + dt k3
    a.y = g->yb; a.p0 = u_src; a.p1 = g->acc; a.o0 = g->acc; a.o1 = g->ya;
    launch_stencil<K_S3>(g, a, st);
    // S4: k4 = L(Ya); u = acc + dt/6 k4
    a.y = g->ya; a.p0 = g->acc; a.p1 = nullptr; a.o0 = u_dst; a.o1 = nullptr;
    launch_stencil<K_S4>(g, a, st);
}

static inline double nu_of(const pr_problem &p, double t);

// nu of RK4 stage s (0..3) of global fine step j: the expressions of the device table
// (ensure_table; readings C1, C6)
static double nu_stage(const pr_grid *g, int64_t j, int s, double dt) {
    const pr_problem &p = g->prob;
    if (p.nu_mode == PR_NU_STEP_START || s == 0) return nu_of(p, double(j) * dt);
    if (s == 3) return nu_of(p, (double(j) + 1.0) * dt);
    return nu_of(p, (double(j) + 0.5) * dt);
}

// One classical RK4 step as two fused kernels (fused.cuh): state u_src ->
// new state in acc_dst (u_src is only read; Yb lives in g->ya).  jglob: the global
// step index, used when the weights travel as launch parameters (g->wparam).
static void enqueue_fine_step2(pr_grid *g, const double *u_src, double *acc_dst, int j_local,
                               double dt, cudaStream_t st, int64_t jglob = -1) {
    StencilArgs a = base_args(g, K_S1);
    a.nu_tab = g->tab_f.d;
    a.nu_pos = g->d_pos + 0;
    a.j_local = j_local;
    a.dt = dt;
    if (g->wparam) {  // stage weights of this step on the host (fine_weights13: same bits)
        fine_weights13(nu_stage(g, jglob, 0, dt), a.inv_dx, a.c, a.wA);
        fine_weights13(nu_stage(g, jglob, 1, dt), a.inv_dx, a.c, a.wB);
    }
    if (g->f1) {  // the whole step in one kernel: u_src -> acc_dst (NEXT-1)
        a.y = u_src; a.p0 = nullptr; a.p1 = nullptr; a.o0 = acc_dst; a.o1 = nullptr;
        launch_fused<K_A>(g, a, st);
        return;
    }
    // K_A: k1 = L(u), Ya (shared), k2 = L(Ya); acc = u + dt/6 k1 + dt/3 k2; Yb = u + dt/2 k2
    a.y = u_src; a.p0 = nullptr; a.p1 = nullptr; a.o0 = acc_dst; a.o1 = g->ya;
    launch_fused<K_A>(g, a, st);
    // K_B: k3 = L(Yb), Ya' = u + dt k3 (shared), k4 = L(Ya'); u_new = acc + dt/3 k3 + dt/6 k4
    a.y = g->ya; a.p0 = u_src; a.p1 = acc_dst; a.o0 = acc_dst; a.o1 = nullptr;
    if (g->wparam) {
        fine_weights13(nu_stage(g, jglob, 2, dt), a.inv_dx, a.c, a.wA);
        fine_weights13(nu_stage(g, jglob, 3, dt), a.inv_dx, a.c, a.wB);
    }
    launch_fused<K_B>(g, a, st);
}

// One forward-Euler step (Alg.2).
static void enqueue_coarse_step(pr_grid *g, const double *src, double *dst, int j_local,
                                double dt, cudaStream_t st) {
    StencilArgs a = base_args(g, K_COARSE);
    a.nu_tab = g->tab_c.d;
    a.nu_pos = g->d_pos + 1;
    a.j_local = j_local;
    a.dt = dt;
    a.y = src;
    a.o0 = dst;
    if (g->c2) {
        switch (g->cvariant) {
#ifdef PRK_VARIANTS
        case 1: launch_coarse_persist<CoarseP1>(g, a, st); break;
        case 2: launch_coarse_persist<CoarseP2>(g, a, st); break;
#endif
        default: launch_coarse_persist<CoarseP0>(g, a, st); break;
        }
    } else {
        launch_stencil<K_COARSE>(g, a, st);
    }
}

static pr_status set_pos(pr_grid *g, int which, long long v, cudaStream_t st) {
    set_pos_kernel<<<1, 1, 0, st>>>(g->d_pos + which, v);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    return PR_OK;
}

// nu(t) = nu0 + nu0/2 sin(omega t)
static inline double nu_of(const pr_problem &p, double t) {
    return p.nu0 + (p.nu0 / 2.0) * std::sin(p.omega * t);
}

static void clear_graphs(pr_grid *g, int kind) {
    for (auto it = g->graphs.begin(); it != g->graphs.end();) {
        if (kind < 0 || it->first.first == kind) {
            cudaGraphExecDestroy(it->second.exec);
            it = g->graphs.erase(it);
        } else {
            ++it;
        }
    }
}

// Make the device nu table of `fine` (0/1) cover global steps [lo, hi) of size dt.
static pr_status ensure_table(pr_grid *g, int fine, double dt, int64_t lo, int64_t hi,
                              cudaStream_t st) {
    NuTable &T = fine ? g->tab_f : g->tab_c;
    if (T.valid && T.dt == dt && lo >= T.lo && hi <= T.hi) return PR_OK;
    const int per = fine ? 4 : 1;
    const size_t need = size_t(std::max<int64_t>(hi - lo, 1)) * per;
    if (need > T.cap) {
        CK(cudaStreamSynchronize(st));
        if (T.d) CK(cudaFree(T.d));
        T.d = nullptr;
        const size_t cap = std::max(need, T.cap * 2);
        CK(cudaMalloc(&T.d, cap * sizeof(double)));
        T.cap = cap;
        if (fine) {  // graphs captured the old table pointer (four-pass and fused)
            clear_graphs(g, 0);
            clear_graphs(g, 2);
        } else {
            clear_graphs(g, 1);
        }
    }
    if (need > g->h_stage_cap) {
        CK(cudaEventSynchronize(g->stage_ev));
        if (g->h_stage) CK(cudaFreeHost(g->h_stage));
        g->h_stage = nullptr;
        CK(cudaMallocHost(&g->h_stage, need * sizeof(double)));
        g->h_stage_cap = need;
    }
    CK(cudaEventSynchronize(g->stage_ev));  // previous upload has consumed the staging buffer
    const pr_problem &p = g->prob;
    for (int64_t j = lo; j < hi; ++j) {
        double *r = g->h_stage + size_t(j - lo) * per;
        if (!fine) {
            r[0] = nu_of(p, double(j) * dt);  // nu at the step start (C2)
        } else if (p.nu_mode == PR_NU_STEP_START) {
            r[0] = r[1] = r[2] = r[3] = nu_of(p, double(j) * dt);
        } else {  // stage times t_j, t_j + dt/2, t_j + dt/2, t_j + dt (C1, C6)
            r[0] = nu_of(p, double(j) * dt);
            r[1] = r[2] = nu_of(p, (double(j) + 0.5) * dt);
            r[3] = nu_of(p, (double(j) + 1.0) * dt);
        }
    }
    CK(cudaMemcpyAsync(T.d, g->h_stage, size_t(hi - lo) * per * sizeof(double),
                       cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(g->stage_ev, st));
    T.lo = lo;
    T.hi = hi;
    T.dt = dt;
    T.valid = true;
    return PR_OK;
}

// Cached CUDA graph: FINE_BATCH RK4 steps in place on `u` (kind 0), or
// COARSE_PAIRS Euler step pairs u -> tmp -> u (kind 1); the last node
// advances the nu cursor.  The step size is baked in, so the key includes it
// through the table (re-captured when the table pointer changes).
static pr_status get_graph(pr_grid *g, int kind, double *u, double dt, cudaGraphExec_t *out) {
    auto key = std::make_pair(kind, (const void *)u);
    const double *tab = kind == 1 ? g->tab_c.d : g->tab_f.d;
    auto it = g->graphs.find(key);
    if (it != g->graphs.end() && it->second.dt == dt && it->second.tab == tab) {
        *out = it->second.exec;
        return PR_OK;
    }
    if (it != g->graphs.end()) {
        cudaGraphExecDestroy(it->second.exec);
        g->graphs.erase(it);
    }
    cudaGraph_t graph;
    const long long before = g_launches.load();
    CK(cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeThreadLocal));
    if (kind == 0) {
        for (int b = 0; b < FINE_BATCH; ++b) enqueue_fine_step(g, u, u, b, dt, g->cap_stream);
        advance_pos_kernel<<<1, 1, 0, g->cap_stream>>>(g->d_pos + 0, FINE_BATCH);
    } else if (kind == 2) {  // fused path: state ping-pongs u -> acc -> u
        for (int b = 0; b < FINE_BATCH; b += 2) {
            enqueue_fine_step2(g, u, g->acc, b, dt, g->cap_stream);
            enqueue_fine_step2(g, g->acc, u, b + 1, dt, g->cap_stream);
        }
        advance_pos_kernel<<<1, 1, 0, g->cap_stream>>>(g->d_pos + 0, FINE_BATCH);
    } else {
        for (int b = 0; b < COARSE_PAIRS; ++b) {
            enqueue_coarse_step(g, u, g->ctmp, 2 * b, dt, g->cap_stream);
            enqueue_coarse_step(g, g->ctmp, u, 2 * b + 1, dt, g->cap_stream);
        }
        advance_pos_kernel<<<1, 1, 0, g->cap_stream>>>(g->d_pos + 1, 2 * COARSE_PAIRS);
    }
    cudaError_t ce = cudaStreamEndCapture(g->cap_stream, &graph);
    g_launches.store(before);  // capture does not launch
    if (ce != cudaSuccess)
        return fail(PR_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
    cudaGraphExec_t exec;
    ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess)
        return fail(PR_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
    if (g->graphs.size() > 64) clear_graphs(g, -1);  // bound the cache (every kind)
    g->graphs[key] = pr_grid::CachedGraph{exec, dt, tab};
    *out = exec;
    return PR_OK;
}

// Fused path: the state ping-pongs between u_out and g->acc; the step parity
// is arranged so the last step lands in u_out.
static pr_status run_fine2(pr_grid *g, const double *uin, double *uout, int64_t nsteps,
                           long long base, double dt, cudaStream_t st, int64_t step0) {
    if (g->wparam) {  // direct launches, weights as parameters: ping-pong uout <-> acc
        const double *src = uin;
        for (int64_t k = 0; k < nsteps; ++k) {
            // the last step must land in uout: parity of the remaining steps decides
            double *dst = ((nsteps - k) % 2 == 1) ? uout : g->acc;
            if (dst == src) dst = (dst == uout) ? g->acc : uout;
            enqueue_fine_step2(g, src, dst, 0, dt, st, step0 + k);
            src = dst;
        }
        if (src != uout) CK(cudaMemcpyAsync(uout, src, g->bytes, cudaMemcpyDeviceToDevice, st));
        CKL();
        if (g->launch_err != PR_OK) {
            const pr_status e = g->launch_err;
            g->launch_err = PR_OK;
            return e;
        }
        return PR_OK;
    }
    int64_t done = 0;
    int jl = 0;
    const double *state = uout;
    if (uin != uout) {
        double *dst = (nsteps % 2) ? uout : g->acc;
        enqueue_fine_step2(g, uin, dst, jl++, dt, st);
        state = dst;
        done = 1;
        if (state == g->acc) {
            enqueue_fine_step2(g, g->acc, uout, jl++, dt, st);
            state = uout;
            done = 2;
        }
        CKL();
        CKS(set_pos(g, 0, base + done, st));
        jl = 0;
    }
    if (nsteps - done >= FINE_BATCH) {
        cudaGraphExec_t ge;
        CKS(get_graph(g, 2, uout, dt, &ge));
        while (nsteps - done >= FINE_BATCH) {
            CK(cudaGraphLaunch(ge, st));
            g_launches.fetch_add((g->f1 ? 1 : 2) * FINE_BATCH + 1, std::memory_order_relaxed);
            done += FINE_BATCH;
        }
    }
    while (nsteps - done >= 2) {
        enqueue_fine_step2(g, uout, g->acc, jl++, dt, st);
        enqueue_fine_step2(g, g->acc, uout, jl++, dt, st);
        done += 2;
    }
    if (done < nsteps) {  // in place with an odd count: last step into acc, copy back
        enqueue_fine_step2(g, uout, g->acc, jl++, dt, st);
        CK(cudaMemcpyAsync(uout, g->acc, g->bytes, cudaMemcpyDeviceToDevice, st));
        ++done;
    }
    (void)state;
    CKL();
    if (g->launch_err != PR_OK) {
        const pr_status e = g->launch_err;
        g->launch_err = PR_OK;
        return e;
    }
    return PR_OK;
}

static pr_status run_fine(pr_grid *g, const double *uin, double *uout, int64_t step0,
                          int64_t nsteps, double dt, cudaStream_t st) {
    if (nsteps == 0) {
        if (uin != uout) CK(cudaMemcpyAsync(uout, uin, g->bytes, cudaMemcpyDeviceToDevice, st));
        return PR_OK;
    }
    CKS(ensure_table(g, 1, dt, step0, step0 + nsteps, st));
    if (g->f2) {
        const long long b0 = step0 - g->tab_f.lo;
        CKS(set_pos(g, 0, b0, st));
        return run_fine2(g, uin, uout, nsteps, b0, dt, st, step0);
    }
    const long long base = step0 - g->tab_f.lo;
    int64_t done = 0;
    CKS(set_pos(g, 0, base, st));
    if (uin != uout) {  // first step reads u_in, writes u_out; later steps in place
        enqueue_fine_step(g, uin, uout, 0, dt, st);
        CKL();
        done = 1;
        CKS(set_pos(g, 0, base + 1, st));
    }
    if (nsteps - done >= FINE_BATCH) {
        cudaGraphExec_t ge;
        CKS(get_graph(g, 0, uout, dt, &ge));
        while (nsteps - done >= FINE_BATCH) {
            CK(cudaGraphLaunch(ge, st));
            g_launches.fetch_add(4 * FINE_BATCH + 1, std::memory_order_relaxed);
            done += FINE_BATCH;
        }
    }
    for (int b = 0; done < nsteps; ++b, ++done) enqueue_fine_step(g, uout, uout, b, dt, st);
    CKL();
    return PR_OK;
}

static pr_status run_coarse(pr_grid *g, const double *uin, double *uout, int64_t step0,
                            int64_t nsteps, double dt, cudaStream_t st) {
    if (nsteps == 0) {
        if (uin != uout) CK(cudaMemcpyAsync(uout, uin, g->bytes, cudaMemcpyDeviceToDevice, st));
        return PR_OK;
    }
    CKS(ensure_table(g, 0, dt, step0, step0 + nsteps, st));
    const long long base = step0 - g->tab_c.lo;
    int64_t done = 0;
    CKS(set_pos(g, 1, base, st));
    int jl = 0;
    if (uin != uout) {
        if (nsteps % 2) {  // odd: u_in -> u_out, then pairs on u_out
            enqueue_coarse_step(g, uin, uout, jl++, dt, st);
            done = 1;
        } else {           // even: u_in -> tmp -> u_out, then pairs on u_out
            enqueue_coarse_step(g, uin, g->ctmp, jl++, dt, st);
            enqueue_coarse_step(g, g->ctmp, uout, jl++, dt, st);
            done = 2;
        }
        CKL();
        CKS(set_pos(g, 1, base + done, st));
        jl = 0;
    }
    const int64_t pairs = (nsteps - done) / 2;
    int64_t p = 0;
    if (pairs >= COARSE_PAIRS) {
        cudaGraphExec_t ge;
        CKS(get_graph(g, 1, uout, dt, &ge));
        for (; p + COARSE_PAIRS <= pairs; p += COARSE_PAIRS) {
            CK(cudaGraphLaunch(ge, st));
            g_launches.fetch_add(2 * COARSE_PAIRS + 1, std::memory_order_relaxed);
            done += 2 * COARSE_PAIRS;
        }
    }
    for (; p < pairs; ++p) {
        enqueue_coarse_step(g, uout, g->ctmp, jl++, dt, st);
        enqueue_coarse_step(g, g->ctmp, uout, jl++, dt, st);
        done += 2;
    }
    if (done < nsteps) {  // in place with an odd count: last step via tmp + copy
        enqueue_coarse_step(g, uout, g->ctmp, jl++, dt, st);
        CK(cudaMemcpyAsync(uout, g->ctmp, g->bytes, cudaMemcpyDeviceToDevice, st));
        ++done;
    }
    CKL();
    if (g->launch_err != PR_OK) {
        const pr_status e = g->launch_err;
        g->launch_err = PR_OK;
        return e;
    }
    return PR_OK;
}

static int red_blocks(const pr_grid *g) { return g->sms * 4; }

static pr_status ensure_red(pr_grid *g, int slots) {
    if (slots <= g->red_cap) return PR_OK;
    if (g->d_red) CK(cudaFree(g->d_red));
    if (g->h_red) CK(cudaFreeHost(g->h_red));
    g->d_red = nullptr;
    g->h_red = nullptr;
    CK(cudaMalloc(&g->d_red, slots * sizeof(unsigned long long)));
    CK(cudaMallocHost(&g->h_red, slots * sizeof(unsigned long long)));
    g->red_cap = slots;
    return PR_OK;
}

static double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}

static bool is_host_ptr(const void *p) {
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

static pr_status ensure_stage(pr_grid *g) {
    if (!g->stage_a) CK(cudaMalloc(&g->stage_a, g->bytes));
    if (!g->stage_b) CK(cudaMalloc(&g->stage_b, g->bytes));
    return PR_OK;
}

static bool overlaps(const void *a, const void *b, size_t bytes) {
    const char *x = static_cast<const char *>(a), *y = static_cast<const char *>(b);
    return x < y + bytes && y < x + bytes;
}

static pr_status check_grid(pr_grid *g) {
    if (!g) return fail(PR_EINVAL, "grid is NULL");
    CK(cudaSetDevice(g->dev));
    return PR_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

const char *pr_last_error(void) { return g_err.c_str(); }
const char *pr_version(void) { return "parareal-b200 0.1 (sm_100a)"; }
int64_t pr_kernel_launches(void) { return g_launches.load(); }

pr_status pr_create_grid(const pr_problem *problem, int32_t cuda_device, pr_grid **out) {
    if (!problem || !out) return fail(PR_EINVAL, "null argument");
    *out = nullptr;
    const int n = problem->n;
    if (n < 4 || n > 2048 || n % 2) return fail(PR_EINVAL, "n must be even and in [4, 2048], got %d", n);
    if (!(problem->nu0 >= 0.0) || !(problem->T > 0.0) || !std::isfinite(problem->omega))
        return fail(PR_EINVAL, "need nu0 >= 0, T > 0, finite omega");
    for (int d = 0; d < 3; ++d)
        if (!std::isfinite(problem->c[d])) return fail(PR_EINVAL, "non-finite velocity");
    if (problem->nu_mode != PR_NU_STAGE && problem->nu_mode != PR_NU_STEP_START)
        return fail(PR_EINVAL, "bad nu_mode %d", problem->nu_mode);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (cuda_device < 0 || cuda_device >= ndev)
        return fail(PR_EINVAL, "cuda_device %d out of range (%d devices)", cuda_device, ndev);
    CK(cudaSetDevice(cuda_device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, cuda_device));
    if (prop.major != 10)
        return fail(PR_ECUDA, "this library is built for sm_100a (B200); device is sm_%d%d",
                    prop.major, prop.minor);
    pr_grid *g = new pr_grid();
    g->dev = cuda_device;
    g->prob = *problem;
    g->n = n;
    g->N = int64_t(n) * n * n;
    g->bytes = size_t(g->N) * sizeof(double);
    g->sms = prop.multiProcessorCount;
    if (const char *tv = getenv("PR_TILE")) g->variant = atoi(tv);
    auto bail = [&](pr_status s) { pr_destroy_grid(g); return s; };
#define GK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return bail(fail(e_ == cudaErrorMemoryAllocation ? PR_ENOMEM : PR_ECUDA,         \
                             "%s failed: %s", #call, cudaGetErrorString(e_)));              \
    } while (0)
    GK(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
    GK(cudaEventCreateWithFlags(&g->stage_ev, cudaEventDisableTiming));
    GK(cudaMalloc(&g->acc, g->bytes));
    GK(cudaMalloc(&g->ya, g->bytes));
    GK(cudaMalloc(&g->yb, g->bytes));
    GK(cudaMalloc(&g->ctmp, g->bytes));
    GK(cudaMalloc(&g->d_pos, 2 * sizeof(long long)));
    GK(cudaMemset(g->d_pos, 0, 2 * sizeof(long long)));
    GK(cudaMalloc(&g->d_sine, n * sizeof(double)));
    {
        std::vector<double> s(n);
        const double dx = 1.0 / n;
        for (int i = 0; i < n; ++i) s[i] = std::sin(2.0 * M_PI * (i * dx));
        GK(cudaMemcpy(g->d_sine, s.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    }
    pr_status s;
    if ((s = setup_kind<K_COARSE>(g)) != PR_OK) return bail(s);
    if ((s = setup_kind<K_S1>(g)) != PR_OK) return bail(s);
    if ((s = setup_kind<K_S2>(g)) != PR_OK) return bail(s);
    if ((s = setup_kind<K_S3>(g)) != PR_OK) return bail(s);
    if ((s = setup_kind<K_S4>(g)) != PR_OK) return bail(s);
    {
        const char *fe = getenv("PR_F2");
        // default: the TMEM stage-A -> stage-B hand-off (23) from 256^3 up, where it is 2-4 %
        // faster than the shared-memory hand-off (14; bench 2019 vs 2061 ms per solve), 14
        // below (3 % faster at 128^3); both give the same bits (test_fused_variants_bitwise)
        g->fvariant = n >= 256 ? 23 : 14;
        if (const char *fv = getenv("PR_FTILE")) g->fvariant = atoi(fv);
        int tya = 0, tyb = 0;
        fused_tiles(g->fvariant, &tya, &tyb);
        if (!tya) return bail(fail(PR_EINVAL, "fused variant %d is not built (PRK_VARIANTS)", g->fvariant));
        g->f2 = (n % FusedP4::TXO == 0) && (n % tya == 0) && (n % tyb == 0) && !(fe && fe[0] == '0');
        g->f1 = g->f2 && g->fvariant == 24;
        // PR_WPARAM=1: fused kernels launched directly with the stage weights as launch
        // parameters (uniform registers instead of 26 per thread) instead of CUDA-graph
        // batches reading the nu table.  Measured neutral at 256^3 / 512^3 and 9 % slower
        // at 128^3 (launch gaps), so the graphs stay the default.
        const char *we = getenv("PR_WPARAM");
        const char *pe = getenv("PR_PDL");
        g->pdl = g->f2 && pe && pe[0] == '1';
        g->wparam = g->f2 && !g->f1 && fused_has_wp(g->fvariant) &&
                    (we ? we[0] == '1' : g->fvariant == 25);  // z2 pays its registers with WP
    }
    if (g->f2) {
        if ((s = setup_fused<K_A>(g)) != PR_OK) return bail(s);
        if (!g->f1 && (s = setup_fused<K_B>(g)) != PR_OK) return bail(s);
    }
    {
        const char *ce = getenv("PR_C2");
        if (const char *cv = getenv("PR_CTILE")) g->cvariant = atoi(cv);
        g->c2 = (n % CoarseP0::TXO == 0) && (n % CoarseP0::TYO == 0) && !(ce && ce[0] == '0');
    }
    if (g->c2 && (s = setup_coarse(g)) != PR_OK) return bail(s);
    if ((s = ensure_red(g, 8)) != PR_OK) return bail(s);
    GK(cudaMallocHost(&g->h_flag, 2 * sizeof(double)));
    // generous initial table capacities (graphs capture the pointers)
    GK(cudaMalloc(&g->tab_f.d, (size_t(1) << 20) * sizeof(double)));
    g->tab_f.cap = size_t(1) << 20;
    GK(cudaMalloc(&g->tab_c.d, (size_t(1) << 18) * sizeof(double)));
    g->tab_c.cap = size_t(1) << 18;
#undef GK
    *out = g;
    return PR_OK;
}

pr_status pr_destroy_grid(pr_grid *g) {
    if (!g) return PR_OK;
    cudaSetDevice(g->dev);
    cudaDeviceSynchronize();
    for (auto &kv : g->graphs) cudaGraphExecDestroy(kv.second.exec);
    g->graphs.clear();
    for (void *p : g->ipc_open) cudaIpcCloseMemHandle(p);
    cudaFree(g->d_flags); cudaFree(g->d_ipc);
    if (g->half) pr_destroy_grid(g->half);
    cudaFree(g->half_u);
    for (pr_grid *c : g->slice_grids) pr_destroy_grid(c);
    cudaSetDevice(g->dev);
    for (cudaStream_t t : g->slice_streams) cudaStreamDestroy(t);
    for (cudaEvent_t e : g->slice_events) cudaEventDestroy(e);
    if (g->comm) ncclCommDestroy(g->comm);
    g->lgroup.reset();  // the last member's release destroys the group's events
    cudaSetDevice(g->dev);
    if (g->work_stream) cudaStreamDestroy(g->work_stream);
    if (g->fork_ev) cudaEventDestroy(g->fork_ev);
    if (g->join_ev) cudaEventDestroy(g->join_ev);
    for (double *p : g->pool) cudaFree(p);
    cudaFree(g->acc); cudaFree(g->ya); cudaFree(g->yb); cudaFree(g->ctmp);
    cudaFree(g->d_pos); cudaFree(g->d_red); cudaFree(g->d_sine);
    cudaFree(g->tab_f.d); cudaFree(g->tab_c.d);
    cudaFree(g->stage_a); cudaFree(g->stage_b);
    if (g->h_red) cudaFreeHost(g->h_red);
    if (g->h_stage) cudaFreeHost(g->h_stage);
    if (g->h_flag) cudaFreeHost(g->h_flag);
    for (cudaEvent_t e : g->evs) cudaEventDestroy(e);
    for (cudaEvent_t e : g->dep_evs) cudaEventDestroy(e);
    if (g->stage_ev) cudaEventDestroy(g->stage_ev);
    if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
    if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
    delete g;
    return PR_OK;
}

// G_c = prolong o (Alg.2 on the n/2 mesh) o restrict  (NEXT-4, C24-C26).
// The n/2 mesh is a child grid with its own nu table, tiles and graphs.
static pr_status ensure_half(pr_grid *g) {
    if (g->half) return PR_OK;
    pr_problem hp = g->prob;
    hp.n = g->n / 2;
    CKS(pr_create_grid(&hp, g->dev, &g->half));
    const size_t m = size_t(g->n / 2);
    CK(cudaMalloc(&g->half_u, m * m * m * sizeof(double)));
    return PR_OK;
}

static pr_status run_coarse_mesh(pr_grid *g, const double *uin, double *uout, int64_t step0,
                                 int64_t nsteps, double dt, cudaStream_t st) {
    if (g->n % 4) return fail(PR_EINVAL, "coarse-mesh G needs n %% 4 == 0 (n = %d)", g->n);
    CKS(ensure_half(g));
    const int blocks = g->sms * 8;
    restrict_kernel<<<blocks, 256, 0, st>>>(uin, g->half_u, g->n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    CKS(run_coarse(g->half, g->half_u, g->half_u, step0, nsteps, dt, st));
    prolong_kernel<<<blocks, 256, 0, st>>>(g->half_u, uout, g->n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    return PR_OK;
}

static pr_status propagate(pr_grid *g, int fine, const double *u_in, double *u_out, int64_t step0,
                           int64_t nsteps, double dt, void *stream) {
    CKS(check_grid(g));
    if (!u_in || !u_out) return fail(PR_EINVAL, "null field pointer");
    if (nsteps < 0 || step0 < 0) return fail(PR_EINVAL, "need step0 >= 0 and n_steps >= 0");
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(PR_EINVAL, "need dt > 0");
    if (u_in != u_out && overlaps(u_in, u_out, g->bytes))
        return fail(PR_EINVAL, "u_in and u_out overlap without being identical");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool hin = is_host_ptr(u_in), hout = is_host_ptr(u_out);
    const double *din = u_in;
    double *dout = u_out;
    if (hin || hout) {
        CKS(ensure_stage(g));
        if (hin) {
            CK(cudaMemcpyAsync(g->stage_a, u_in, g->bytes, cudaMemcpyHostToDevice, st));
            din = g->stage_a;
        }
        if (hout) dout = (hin && u_in == u_out) ? g->stage_a : g->stage_b;
    }
    CKS(fine == 1   ? run_fine(g, din, dout, step0, nsteps, dt, st)
        : fine == 2 ? run_coarse_mesh(g, din, dout, step0, nsteps, dt, st)
                    : run_coarse(g, din, dout, step0, nsteps, dt, st));
    if (hout) {
        CK(cudaMemcpyAsync(u_out, dout, g->bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    } else if (hin) {
        CK(cudaStreamSynchronize(st));
    }
    return PR_OK;
}

pr_status pr_fine(pr_grid *g, const double *u_in, double *u_out, int64_t step0, int64_t n_steps,
                  double dt, void *stream) {
    return propagate(g, 1, u_in, u_out, step0, n_steps, dt, stream);
}

pr_status pr_coarse(pr_grid *g, const double *u_in, double *u_out, int64_t step0,
                    int64_t n_steps, double dt, void *stream) {
    return propagate(g, 0, u_in, u_out, step0, n_steps, dt, stream);
}

pr_status pr_coarse_mesh(pr_grid *g, const double *u_in, double *u_out, int64_t step0,
                         int64_t n_steps, double dt, void *stream) {
    return propagate(g, 2, u_in, u_out, step0, n_steps, dt, stream);
}

static pr_status launch_maxabs(pr_grid *g, const double *u, const double *ref,
                               unsigned long long *d_diff, unsigned long long *d_ref,
                               cudaStream_t st) {
    maxabs_kernel<<<red_blocks(g), RED_THREADS, 0, st>>>(
        reinterpret_cast<const double2 *>(u), reinterpret_cast<const double2 *>(ref), d_diff,
        d_ref, g->N / 2);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    return PR_OK;
}

pr_status pr_defect(pr_grid *g, const double *u, const double *u_ref, double *d_host,
                    void *stream) {
    CKS(check_grid(g));
    if (!u || !u_ref || !d_host) return fail(PR_EINVAL, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const double *du = u, *dr = u_ref;
    if (is_host_ptr(u) || is_host_ptr(u_ref)) {
        CKS(ensure_stage(g));
        if (is_host_ptr(u)) {
            CK(cudaMemcpyAsync(g->stage_a, u, g->bytes, cudaMemcpyHostToDevice, st));
            du = g->stage_a;
        }
        if (is_host_ptr(u_ref)) {
            CK(cudaMemcpyAsync(g->stage_b, u_ref, g->bytes, cudaMemcpyHostToDevice, st));
            dr = g->stage_b;
        }
    }
    CK(cudaMemsetAsync(g->d_red, 0, 2 * sizeof(unsigned long long), st));
    CKS(launch_maxabs(g, du, dr, g->d_red, g->d_red + 1, st));
    CK(cudaMemcpyAsync(g->h_red, g->d_red, 2 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const double m = bits_to_double(g->h_red[0]), M = bits_to_double(g->h_red[1]);
    if (M == 0.0) return fail(PR_EDOMAIN, "max|u_ref| = 0: defect undefined (Eq.(defect))");
    *d_host = m / M;
    return PR_OK;
}

pr_status pr_fill_sine(pr_grid *g, double *u, void *stream) {
    CKS(check_grid(g));
    if (!u) return fail(PR_EINVAL, "null field pointer");
    fill_sine_kernel<<<g->sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(g->d_sine, u, g->n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    return PR_OK;
}

static pr_status launch_correct(pr_grid *g, const double *f, const double *gn, const double *go,
                                double *uo, const double *ref, unsigned long long *dmax,
                                cudaStream_t st, const double *prev = nullptr,
                                unsigned long long *cmax = nullptr,
                                unsigned long long *nmax = nullptr, double *peer = nullptr) {
    correct_kernel<<<red_blocks(g), RED_THREADS, 0, st>>>(
        reinterpret_cast<const double2 *>(f), reinterpret_cast<const double2 *>(gn),
        reinterpret_cast<const double2 *>(go), reinterpret_cast<double2 *>(uo),
        reinterpret_cast<const double2 *>(ref), dmax, reinterpret_cast<const double2 *>(prev),
        cmax, nmax, g->N / 2, reinterpret_cast<double2 *>(peer));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    return PR_OK;
}

pr_status pr_correct(pr_grid *g, const double *f, const double *g_new, const double *g_old,
                     double *u_out, const double *u_ref, double *d_host, void *stream) {
    CKS(check_grid(g));
    if (!f || !g_new || !g_old || !u_out) return fail(PR_EINVAL, "null field pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool want = u_ref && d_host;
    if (want) {
        CK(cudaMemsetAsync(g->d_red, 0, 2 * sizeof(unsigned long long), st));
        CKS(launch_maxabs(g, nullptr, u_ref, g->d_red, g->d_red + 1, st));
    }
    CKS(launch_correct(g, f, g_new, g_old, u_out, want ? u_ref : nullptr, g->d_red, st));
    if (want) {
        CK(cudaMemcpyAsync(g->h_red, g->d_red, 2 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double M = bits_to_double(g->h_red[1]);
        if (M == 0.0) return fail(PR_EDOMAIN, "max|u_ref| = 0");
        *d_host = bits_to_double(g->h_red[0]) / M;
    }
    return PR_OK;
}

pr_status pr_stability_ratio(const pr_problem *p, double dt, int32_t fine, double *ratio) {
    if (!p || !ratio || p->n < 1 || !(dt > 0.0)) return fail(PR_EINVAL, "bad argument");
    const double inv = double(p->n), numax = 1.5 * p->nu0;
    if (fine) {
        *ratio = dt * (16.0 * numax * inv * inv) / 2.785;
    } else {
        double s = 6.0 * numax * inv * inv;
        for (int d = 0; d < 3; ++d) s += std::fabs(p->c[d]) * inv;
        *ratio = dt * s;
    }
    return PR_OK;
}

// ------------------------------------------------------------------ Parareal
pr_status pr_plan(int32_t Np, int32_t K, int32_t W, int32_t r, pr_op *ops, int32_t cap,
                  int32_t *count) {
    if (!count) return fail(PR_EINVAL, "count is NULL");
    if (Np < 1 || K < 0 || W < 1 || r < 0 || r >= W || Np % W)
        return fail(PR_EINVAL, "bad plan sizes (N_p=%d K=%d W=%d r=%d)", Np, K, W, r);
    const int s = Np / W, j0 = r * s;
    int c = 0;
    auto emit = [&](int op, int k, int slice, int peer) {
        if (ops && c < cap) ops[c] = pr_op{op, k, slice, peer};
        ++c;
    };
    for (int m = 0; m < j0; ++m) emit(PR_OP_G_PREFIX, -1, m, -1);
    for (int l = 0; l < s; ++l) emit(PR_OP_G_INIT, -1, j0 + l, -1);
    if (r == W - 1) emit(PR_OP_DEFECT0, -1, Np - 1, -1);
    for (int k = 0; k < K; ++k) {
        for (int l = 0; l < s; ++l) emit(PR_OP_F, k, j0 + l, -1);
        for (int l = 0; l < s; ++l) {
            const int j = j0 + l;
            if (l == 0 && j > 0) emit(PR_OP_RECV, k, j, r - 1);
            emit(PR_OP_G, k, j, -1);
            emit(PR_OP_CORRECT, k, j, -1);
            if (l == s - 1 && r < W - 1) emit(PR_OP_SEND, k, j, r + 1);
        }
        emit(PR_OP_END_ITER, k, -1, -1);
    }
    *count = c;
    return PR_OK;
}

pr_status pr_nccl_unique_id(void *id_out) {
    if (!id_out) return fail(PR_EINVAL, "null id");
    static_assert(sizeof(ncclUniqueId) == PR_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(PR_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
    std::memcpy(id_out, &id, sizeof id);
    return PR_OK;
}

pr_status pr_comm_init(pr_grid *g, int32_t world, int32_t rank, const void *id) {
    CKS(check_grid(g));
    if (!id || world < 1 || rank < 0 || rank >= world)
        return fail(PR_EINVAL, "bad world/rank (%d/%d)", world, rank);
    if (g->comm) {
        ncclCommDestroy(g->comm);
        g->comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclResult_t r = ncclCommInitRank(&g->comm, world, uid, rank);
    if (r != ncclSuccess) {
        g->comm = nullptr;
        return fail(PR_ENCCL, "rank %d: ncclCommInitRank: %s", rank, ncclGetErrorString(r));
    }
    if (!g->comm_stream) CK(cudaStreamCreateWithFlags(&g->comm_stream, cudaStreamNonBlocking));
    // Connect the pipeline's links now, while every rank is inside this collective call:
    // NCCL sets up a point-to-point connection at its first use, and that handshake
    // blocks the host until the peer joins, so a predecessor that never reaches
    // pr_parareal would hang the successor inside ncclRecv instead of failing it.
    if (world > 1) {
        if (!g->d_red) CK(cudaMalloc(&g->d_red, 8 * sizeof(unsigned long long)));
        ncclGroupStart();
        if (rank + 1 < world) ncclSend(g->d_red, 1, ncclUint64, rank + 1, g->comm, g->comm_stream);
        if (rank > 0) ncclRecv(g->d_red + 1, 1, ncclUint64, rank - 1, g->comm, g->comm_stream);
        r = ncclGroupEnd();
        if (r != ncclSuccess)
            return fail(PR_ENCCL, "rank %d: connecting the pipeline links: %s", rank, ncclGetErrorString(r));
        CK(cudaStreamSynchronize(g->comm_stream));
    }
    g->lgroup.reset();  // a communicator replaces an in-process rank group
    g->world = world;
    g->rank = rank;
    g->mapped_gen = -1;  // peer mappings belong to the previous communicator
    return PR_OK;
}

pr_status pr_local_group(pr_grid **grids, int32_t world) {
    if (!grids || world < 1) return fail(PR_EINVAL, "need grids and world >= 1");
    for (int i = 0; i < world; ++i) {
        if (!grids[i]) return fail(PR_EINVAL, "grid %d is NULL", i);
        for (int j = 0; j < i; ++j)
            if (grids[j] == grids[i]) return fail(PR_EINVAL, "grid %d appears twice", i);
    }
    auto grp = std::make_shared<LocalGroup>();
    grp->r.resize(size_t(world));
    for (int i = 0; i < world; ++i) grp->r[i].dev = grids[i]->dev;
    // rank r's correction kernel stores into rank r+1's memory: peer access across devices
    for (int i = 0; i + 1 < world; ++i) {
        const int a = grids[i]->dev, b = grids[i + 1]->dev;
        if (a == b) continue;
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, a, b));
        if (!ok) return fail(PR_EINVAL, "device %d cannot access device %d (peer access)", a, b);
        CK(cudaSetDevice(a));
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CK(e);
    }
    for (int i = 0; i < world; ++i) {
        pr_grid *g = grids[i];
        CK(cudaSetDevice(g->dev));
        if (g->comm) {
            ncclCommDestroy(g->comm);
            g->comm = nullptr;
        }
        if (!g->work_stream) CK(cudaStreamCreateWithFlags(&g->work_stream, cudaStreamNonBlocking));
        if (!g->fork_ev) CK(cudaEventCreateWithFlags(&g->fork_ev, cudaEventDisableTiming));
        if (!g->join_ev) CK(cudaEventCreateWithFlags(&g->join_ev, cudaEventDisableTiming));
        g->lgroup = grp;
        g->world = world;
        g->rank = i;
        g->seq_base = 0;
    }
    return PR_OK;
}

static pr_status ensure_events(pr_grid *g, size_t count) {
    while (g->evs.size() < count) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        g->evs.push_back(e);
    }
    return PR_OK;
}

// Seconds a rank waits for its predecessor's hand-off before it gives up with
// PR_ENCCL (PR_NCCL_TIMEOUT_S; <= 0 waits forever).  Default 900 s: far above the
// longest solve of BASELINE's configurations, finite so a stuck peer fails the call.
static double handoff_timeout_s() {
    const char *tenv = getenv("PR_NCCL_TIMEOUT_S");
    return tenv ? atof(tenv) : 900.0;
}

// Wait for `st` (and the comm stream), polling NCCL for asynchronous errors.
static pr_status wait_all(pr_grid *g, cudaStream_t st, int k_hint, bool with_comm = true) {
    const double timeout = handoff_timeout_s();
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t ss[2] = {st, g->comm ? g->comm_stream : st};
    for (int i = 0; i < (with_comm ? 2 : 1); ++i) {
        for (;;) {
            cudaError_t e = cudaStreamQuery(ss[i]);
            if (e == cudaSuccess) break;
            if (e != cudaErrorNotReady)
                return fail(PR_ECUDA, "rank %d: stream error: %s", g->rank, cudaGetErrorString(e));
            if (g->lgroup && timeout > 0) {  // in-process group: a peer that never delivers
                const double el = std::chrono::duration<double>(
                                      std::chrono::steady_clock::now() - t0).count();
                if (el > timeout)
                    return fail(PR_ENCCL, "rank %d, iteration %d: stream not done after %.1f s",
                                g->rank, k_hint, el);
            }
            if (g->comm) {
                ncclResult_t ae = ncclSuccess;
                ncclCommGetAsyncError(g->comm, &ae);
                if (ae != ncclSuccess && ae != ncclInProgress) {
                    ncclCommAbort(g->comm);
                    g->comm = nullptr;
                    return fail(PR_ENCCL, "rank %d, iteration %d: NCCL async error: %s", g->rank,
                                k_hint, ncclGetErrorString(ae));
                }
                if (timeout > 0) {
                    const double el = std::chrono::duration<double>(
                                          std::chrono::steady_clock::now() - t0).count();
                    if (el > timeout) {
                        ncclCommAbort(g->comm);
                        g->comm = nullptr;
                        return fail(PR_ENCCL, "rank %d, iteration %d: timed out after %.1f s",
                                    g->rank, k_hint, el);
                    }
                }
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    return PR_OK;
}

#define NCK(call, k)                                                                     \
    do {                                                                                 \
        ncclResult_t r_ = (call);                                                        \
        if (r_ != ncclSuccess)                                                           \
            return fail(PR_ENCCL, "rank %d, iteration %d: %s: %s", g->rank, (k), #call,  \
                        ncclGetErrorString(r_));                                         \
    } while (0)

// Peer hand-off setup, collective over the communicator, once per buffer pool:
// every rank exports (CUDA IPC) the two pool fields that alternate as its
// receive buffer and its flag words; the handles travel by one ncclAllGather;
// rank r maps its successor's buffers and flags and its predecessor's flags.
static pr_status peer_setup(pr_grid *g, double *mail_even, double *mail_odd) {
    if (g->mapped_gen == g->pool_gen) return PR_OK;
    for (void *p : g->ipc_open) cudaIpcCloseMemHandle(p);
    g->ipc_open.clear();
    g->peer_mail[0] = g->peer_mail[1] = nullptr;
    g->succ_flags = g->pred_flags = nullptr;
    g->mapped_gen = -1;
    if (!stream_wait_fn()) return fail(PR_ECUDA, "cuStreamWaitValue32 entry point not found");
    const int W = g->world, r = g->rank;
    constexpr size_t HREC = 3 * sizeof(cudaIpcMemHandle_t), REC = HREC + 8;  // + seq_base
    // flag words are zeroed once and never reset: sequence numbers only grow
    // (seq_base advances on every peer-mode call, on every rank alike), so a late
    // store from a peer's previous call can never satisfy a newer wait
    if (!g->d_flags) {
        CK(cudaMalloc(&g->d_flags, 256));
        CK(cudaMemset(g->d_flags, 0, 256));
    }
    if (g->d_ipc) CK(cudaFree(g->d_ipc));
    g->d_ipc = nullptr;
    CK(cudaMalloc(&g->d_ipc, REC * size_t(W)));
    cudaIpcMemHandle_t h[3];
    CK(cudaIpcGetMemHandle(&h[0], mail_even));
    CK(cudaIpcGetMemHandle(&h[1], mail_odd));
    CK(cudaIpcGetMemHandle(&h[2], g->d_flags));
    unsigned char rec[REC] = {};
    std::memcpy(rec, h, HREC);
    std::memcpy(rec + HREC, &g->seq_base, sizeof g->seq_base);
    CK(cudaMemcpy(g->d_ipc + REC * size_t(r), rec, REC, cudaMemcpyHostToDevice));
    NCK(ncclAllGather(g->d_ipc + REC * size_t(r), g->d_ipc, REC, ncclUint8, g->comm, g->comm_stream), -1);
    CK(cudaStreamSynchronize(g->comm_stream));
    std::vector<unsigned char> all(REC * size_t(W));
    CK(cudaMemcpy(all.data(), g->d_ipc, all.size(), cudaMemcpyDeviceToHost));
    auto open = [&](int rank, int idx, void **out) -> pr_status {
        cudaIpcMemHandle_t hh;
        std::memcpy(&hh, all.data() + REC * size_t(rank) + idx * sizeof hh, sizeof hh);
        CK(cudaIpcOpenMemHandle(out, hh, cudaIpcMemLazyEnablePeerAccess));
        g->ipc_open.push_back(*out);
        return PR_OK;
    };
    void *p = nullptr;
    if (r < W - 1) {
        CKS(open(r + 1, 0, &p)); g->peer_mail[0] = static_cast<double *>(p);
        CKS(open(r + 1, 1, &p)); g->peer_mail[1] = static_cast<double *>(p);
        CKS(open(r + 1, 2, &p)); g->succ_flags = static_cast<unsigned int *>(p);
    }
    if (r > 0) {
        CKS(open(r - 1, 2, &p));
        g->pred_flags = static_cast<unsigned int *>(p);
    }
    // common sequence base: the largest any rank has used (grids with different call
    // histories meet in one communicator); every stale flag value is below it
    for (int q = 0; q < W; ++q) {
        unsigned int b = 0;
        std::memcpy(&b, all.data() + REC * size_t(q) + HREC, sizeof b);
        g->seq_base = std::max(g->seq_base, b);
    }
    g->mapped_gen = g->pool_gen;
    return PR_OK;
}

// The consumer side of a peer hand-off: the stream front end waits until the word the
// peer publishes (st.release.sys after its data stores) reaches v.  The data arrived
// over NVLink before the word, but a front-end wait is not an acquire: with
// CU_STREAM_WAIT_VALUE_FLUSH (where the device supports it) the wait also flushes the
// remote writes that preceded the word, and a one-thread ld.acquire.sys of the word +
// fence.acq_rel.sys kernel orders every later kernel of the stream after them (the
// value is already there, so it never spins).  cuda.h: CU_STREAM_WAIT_VALUE_FLUSH.
static pr_status stream_wait_geq(pr_grid *g, cudaStream_t st, const unsigned int *addr, unsigned int v,
                                 bool acquire) {
    if (g->can_flush < 0) {
        int f = 0;
        if (cudaDeviceGetAttribute(&f, cudaDevAttrCanFlushRemoteWrites, g->dev) != cudaSuccess) {
            cudaGetLastError();
            f = 0;
        }
        g->can_flush = f ? 1 : 0;
    }
    const unsigned int flags = CU_STREAM_WAIT_VALUE_GEQ | (g->can_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
    CUresult e = stream_wait_fn()(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr),
                                  v, flags);
    if (e != CUDA_SUCCESS) return fail(PR_ECUDA, "cuStreamWaitValue32 failed (%d)", int(e));
    if (acquire) {
        acquire_kernel<<<1, 1, 0, st>>>(addr);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        CKL();
    }
    return PR_OK;
}

}  // extern "C"

// ---- in-process rank group (pr_local_group): host-side announcements
// Block until pred() holds for the group state, or fail with PR_ENCCL after the
// hand-off timeout (a stuck or failed peer rank).
template <class Pred>
static pr_status local_wait(pr_grid *g, int k, int peer, const char *what, Pred pred) {
    LocalGroup &G = *g->lgroup;
    const double tmo = handoff_timeout_s();
    std::unique_lock<std::mutex> lk(G.mu);
    const auto t0 = std::chrono::steady_clock::now();
    while (!pred(G)) {
        if (tmo > 0) {
            const auto until = t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                                        std::chrono::duration<double>(tmo));
            if (G.cv.wait_until(lk, until) == std::cv_status::timeout && !pred(G))
                return fail(PR_ENCCL, "rank %d, iteration %d: timed out after %.1f s waiting for rank %d (%s)",
                            g->rank, k, tmo, peer, what);
        } else {
            G.cv.wait(lk);
        }
    }
    return PR_OK;
}

// record `ev` on st, then publish `field = v` of this rank under the group lock
static pr_status local_publish(pr_grid *g, cudaEvent_t ev, cudaStream_t st,
                               unsigned long long LocalRank::*field, unsigned long long v) {
    if (ev) CK(cudaEventRecord(ev, st));
    LocalGroup &G = *g->lgroup;
    {
        std::lock_guard<std::mutex> lk(G.mu);
        G.r[g->rank].*field = v;
    }
    G.cv.notify_all();
    return PR_OK;
}

extern "C" {

static pr_status post(pr_grid *g, double *stop_dst, double stop, unsigned int *flag, unsigned int seq,
                      cudaStream_t st) {
    post_kernel<<<1, 1, 0, st>>>(stop_dst, stop, flag, seq);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CKL();
    return PR_OK;
}

// Concurrent F over the s slices of a group: F of different slices of one iteration are
// independent (each starts from the previous iteration's value), so each slice runs on its
// own stream with its own child grid (4 fields of scratch each); the launches overlap their
// pipeline fill / drain and, for small n, fill an otherwise idle GPU.  Measured: 3.4x at 32^3,
// 1.1x at 128^3, 1.03x at 256^3.  Used while the children's scratch stays <= 16 GiB.
static bool conc_wanted(const pr_grid *g, int s) {
    const char *e = getenv("PR_CONC");
    if (e) return s > 1 && e[0] == '1';
    return s > 1 && double(s) * 4.0 * double(g->bytes) <= 16.0 * (1 << 30);
}

static pr_status ensure_slice_grids(pr_grid *g, int s) {
    while (int(g->slice_grids.size()) < s) {
        pr_grid *c = nullptr;
        CKS(pr_create_grid(&g->prob, g->dev, &c));
        g->slice_grids.push_back(c);
    }
    CK(cudaSetDevice(g->dev));
    while (int(g->slice_streams.size()) < s) {
        cudaStream_t t;
        CK(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
        g->slice_streams.push_back(t);
    }
    while (int(g->slice_events.size()) < s + 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        g->slice_events.push_back(e);
    }
    return PR_OK;
}

pr_status pr_parareal(pr_grid *g, const pr_parareal_cfg *cfg, const double *u0, double *u_T,
                      const double *u_ref, double *defects_host, void *stream) {
    CKS(check_grid(g));
    if (!cfg || !u0) return fail(PR_EINVAL, "null argument");
    const int Np = cfg->n_slices, nc = cfg->n_coarse_per_slice, nf = cfg->n_fine_per_slice,
              K = cfg->K;
    const bool g_is_f = (cfg->flags & PR_FLAG_G_IS_F) != 0;
    const bool g_half = !g_is_f && (cfg->flags & PR_FLAG_G_HALF_MESH) != 0;
    if (g_half && g->n % 4) return fail(PR_EINVAL, "PR_FLAG_G_HALF_MESH needs n %% 4 == 0");
    const double tol = cfg->tol;
    const bool ctrl = tol > 0.0;  // convergence-controlled stopping (C23)
    if (Np < 1 || nc < 1 || nf < 1 || K < 0 || !(tol == tol))
        return fail(PR_EINVAL, "need n_slices, N_c, N_f >= 1, K >= 0 and a number for tol");
    const bool local = g->lgroup != nullptr;  // in-process rank group (pr_local_group)
    const int W = (g->comm || local) ? g->world : 1, r = (g->comm || local) ? g->rank : 0;
    if (g->world > 1 && !g->comm && !local) return fail(PR_ESTATE, "world > 1 but no communicator");
    if (Np % W) return fail(PR_EINVAL, "n_slices (%d) must be a multiple of world (%d)", Np, W);
    const bool last = (r == W - 1);
    if (last && !u_T) return fail(PR_EINVAL, "u_T is NULL on the last rank");
    const int s = Np / W, j0 = r * s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaStream_t user_st = st;
    if (local) {  // each rank of a group runs on its grid's own stream, joined to the caller's
        CK(cudaEventRecord(g->fork_ev, user_st));
        st = g->work_stream;
        CK(cudaStreamWaitEvent(st, g->fork_ev, 0));
    }
    const double T = g->prob.T;
    const double Dt = T / double(int64_t(Np) * nc);  // coarse step
    const double dt = T / double(int64_t(Np) * nf);  // fine step

    std::vector<pr_op> plan;
    int32_t cnt = 0;
    CKS(pr_plan(Np, K, W, r, nullptr, 0, &cnt));
    plan.resize(cnt);
    CKS(pr_plan(Np, K, W, r, plan.data(), cnt, &cnt));

    // buffers: start[s], f[s], out[s], gold[s], gnew, recv, u0d; each field has
    // two trailing doubles (the hand-off message carries a stop flag at [N])
    const size_t nbuf = size_t(4 * s + 3);
    if (g->par_s != s || g->pool.size() != nbuf) {
        CK(cudaDeviceSynchronize());
        for (double *p : g->pool) CK(cudaFree(p));
        g->pool.clear();
        for (size_t i = 0; i < nbuf; ++i) {
            double *p = nullptr;
            CK(cudaMalloc(&p, g->bytes + 2 * sizeof(double)));
            g->pool.push_back(p);
        }
        g->par_s = s;
        ++g->pool_gen;
    }
    std::vector<double *> start(s), f(s), out(s), gold(s);
    for (int l = 0; l < s; ++l) {
        start[l] = g->pool[l];
        f[l] = g->pool[s + l];
        out[l] = g->pool[2 * s + l];
        gold[l] = g->pool[3 * s + l];
    }
    double *gnew = g->pool[4 * s], *recvb = g->pool[4 * s + 1], *u0d = g->pool[4 * s + 2];
    // peer hand-off: the receive buffer alternates between pool[4s+1] (even k) and
    // pool[0] (odd k: start[0] swaps with recvb at the end of every iteration)
    const bool lh = local && W > 1;  // in-process hand-off (events announced through the group)
    const bool peer = (cfg->flags & PR_FLAG_PEER_HANDOFF) && W > 1 && !local;
    unsigned int base = 0;
    if (peer) {
        CKS(peer_setup(g, g->pool[4 * s + 1], g->pool[0]));
        base = g->seq_base;
        g->seq_base += unsigned(K) + 2;
    }
    LocalGroup *LG = lh ? g->lgroup.get() : nullptr;
    if (lh) {
        base = g->seq_base;
        g->seq_base += unsigned(K) + 2;
        {  // this call's receive buffers (idle until its first receive) and event slots
            std::lock_guard<std::mutex> lk(LG->mu);
            LocalRank &me = LG->r[r];
            while (me.ev_data.size() < size_t(std::max(K, 1))) {
                cudaEvent_t a, b;
                CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
                me.ev_data.push_back(a);
                me.ev_free.push_back(b);
            }
            me.mail[0] = g->pool[4 * s + 1];
            me.mail[1] = g->pool[0];
            me.freed = base;
            me.started = base + 1ull;
        }
        LG->cv.notify_all();
    }
    const bool want_def = last && u_ref && defects_host;
    const double *refd = u_ref;
    if (want_def && is_host_ptr(u_ref)) {
        CKS(ensure_stage(g));
        CK(cudaMemcpyAsync(g->stage_b, u_ref, g->bytes, cudaMemcpyHostToDevice, st));
        refd = g->stage_b;
    }
    // reduction slots: [0..K] defect maxima, [K+1] max|u_ref|,
    // [K+2+2k] max change in iteration k, [K+3+2k] max |u^{k+1}|, [3K+2] spare
    CKS(ensure_red(g, 3 * K + 4));
    unsigned long long *red_chg = g->d_red + K + 2;
    // events: 0 start, 1 init done, then per iteration 4: F done, recv done (compute), iter done, send done
    CKS(ensure_events(g, size_t(2 + 4 * K + 2)));
    cudaEvent_t ev_start = g->evs[0], ev_init = g->evs[1];
    auto evF = [&](int k) { return g->evs[2 + 4 * k]; };
    auto evW = [&](int k) { return g->evs[3 + 4 * k]; };
    auto evI = [&](int k) { return g->evs[4 + 4 * k]; };
    auto evS = [&](int k) { return g->evs[5 + 4 * k]; };
    std::vector<cudaEvent_t> &dep = g->dep_evs;
    while (dep.size() < size_t(2 * K + 2)) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        dep.push_back(e);
    }
    auto recv_ev = [&](int k) { return dep[2 * k]; };
    auto corr_ev = [&](int k) { return dep[2 * k + 1]; };
    cudaEvent_t fdone_ev = dep[2 * K];

    CK(cudaEventRecord(ev_start, st));
    if (is_host_ptr(u0))
        CK(cudaMemcpyAsync(u0d, u0, g->bytes, cudaMemcpyHostToDevice, st));
    else
        CK(cudaMemcpyAsync(u0d, u0, g->bytes, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(g->d_red, 0, size_t(3 * K + 4) * sizeof(unsigned long long), st));
    // nu tables for everything this rank will run (one upload each)
    if (g_is_f) {
        CKS(ensure_table(g, 1, dt, 0, int64_t(j0 + s) * nf, st));
    } else {
        CKS(ensure_table(g, 1, dt, int64_t(j0) * nf, int64_t(j0 + s) * nf, st));
        if (g_half) {  // G_c runs on the n/2 child grid: its table, once, for all slices
            CKS(ensure_half(g));
            CKS(ensure_table(g->half, 0, Dt, 0, int64_t(j0 + s) * nc, st));
        } else {
            CKS(ensure_table(g, 0, Dt, 0, int64_t(j0 + s) * nc, st));
        }
    }
    // slots: d_red[k] = max|u^k_{N_p} - u_ref| (k = 0..K), d_red[K+1] = max|u_ref|
    if (want_def) CKS(launch_maxabs(g, nullptr, refd, nullptr, g->d_red + K + 1, st));

    auto G = [&](const double *in, double *o, int m) -> pr_status {
        if (g_is_f) return run_fine(g, in, o, int64_t(m) * nf, nf, dt, st);
        if (g_half) return run_coarse_mesh(g, in, o, int64_t(m) * nc, nc, Dt, st);
        return run_coarse(g, in, o, int64_t(m) * nc, nc, Dt, st);
    };
    auto Fp = [&](const double *in, double *o, int m) -> pr_status {
        return run_fine(g, in, o, int64_t(m) * nf, nf, dt, st);
    };
    const bool conc = conc_wanted(g, s);
    if (conc) CKS(ensure_slice_grids(g, s));
    const size_t msg = size_t(g->N) + (ctrl ? 1 : 0);  // hand-off length (doubles)

    // peer mode: this rank's receive buffers are idle until its first receive
    if (peer && r > 0) CKS(post(g, nullptr, 0.0, g->pred_flags + 1, base, st));
    const double *v = u0d;
    bool sent_pending = false, init_marked = false, pred_stopped = (r == 0), stopped = false;
    bool recvd = false;
    int last_send_k = -1, iters = 0;
    float ms_fine = 0, ms_wait = 0, ms_gc = 0;
    g->monitors.assign(size_t(K), std::nan(""));
    for (const pr_op &op : plan) {
        if (stopped) break;
        const int l = op.slice - j0;
        if (op.k >= 0 && !init_marked) {
            CK(cudaEventRecord(ev_init, st));
            init_marked = true;
        }
        switch (op.op) {
        case PR_OP_G_PREFIX:
            CKS(G(v, start[0], op.slice));
            v = start[0];
            break;
        case PR_OP_G_INIT:
            if (op.slice == 0) {
                start[0] = u0d;  // rank 0 keeps u0 as its start value
            } else if (start[l] != v) {
                CK(cudaMemcpyAsync(start[l], v, g->bytes, cudaMemcpyDeviceToDevice, st));
            }
            CKS(G(start[l], gold[l], op.slice));
            v = gold[l];
            break;
        case PR_OP_DEFECT0:  // d^0: coarse initial guess at T vs u_ref (C11)
            if (want_def) CKS(launch_maxabs(g, gold[s - 1], refd, g->d_red + 0, nullptr, st));
            break;
        case PR_OP_F:
            if (conc) {  // fork at the first slice, join after the last
                if (l == 0) CK(cudaEventRecord(g->slice_events[0], st));
                cudaStream_t fs = g->slice_streams[l];
                CK(cudaStreamWaitEvent(fs, g->slice_events[0], 0));
                CKS(run_fine(g->slice_grids[l], start[l], f[l], int64_t(op.slice) * nf, nf, dt, fs));
                CK(cudaEventRecord(g->slice_events[1 + l], fs));
                if (l == s - 1)
                    for (int ll = 0; ll < s; ++ll) CK(cudaStreamWaitEvent(st, g->slice_events[1 + ll], 0));
            } else {
                CKS(Fp(start[l], f[l], op.slice));
            }
            // peer mode: start[0] (next iteration's receive buffer of the same parity) is free
            if (peer && r > 0 && (conc ? l == s - 1 : l == 0))
                CKS(post(g, nullptr, 0.0, g->pred_flags + 1, base + unsigned(op.k) + 1, st));
            if (lh && r > 0 && (conc ? l == s - 1 : l == 0))
                CKS(local_publish(g, LG->r[r].ev_free[op.k], st, &LocalRank::freed,
                                  base + unsigned(op.k) + 1ull));
            if (l == s - 1) {
                CK(cudaEventRecord(evF(op.k), st));
                CK(cudaEventRecord(fdone_ev, st));
            }
            break;
        case PR_OP_RECV:
            recvd = false;
            if (pred_stopped) break;  // the predecessor sent its last message earlier
            if (peer) {  // the predecessor's correction stored straight into recvb
                CKS(stream_wait_geq(g, st, g->d_flags + 0, base + unsigned(op.k) + 1, true));
                if (ctrl) CK(cudaMemcpyAsync(g->h_flag, recvb + g->N, sizeof(double),
                                             cudaMemcpyDeviceToHost, st));
                recvd = true;
                break;
            }
            if (lh) {  // same data path; order after the predecessor's announced event
                const unsigned long long want = base + unsigned(op.k) + 1ull;
                CKS(local_wait(g, op.k, r - 1, "its hand-off",
                               [&](LocalGroup &G_) { return G_.r[r - 1].data >= want; }));
                cudaEvent_t ev;
                {
                    std::lock_guard<std::mutex> lk(LG->mu);
                    ev = LG->r[r - 1].ev_data[op.k];
                }
                CK(cudaStreamWaitEvent(st, ev, 0));
                if (ctrl) CK(cudaMemcpyAsync(g->h_flag, recvb + g->N, sizeof(double),
                                             cudaMemcpyDeviceToHost, st));
                recvd = true;
                break;
            }
            // the receive buffer was last read by F of iteration k-1, but the receive is posted
            // only after THIS iteration's F: NCCL's receive kernel holds an SM while it waits for
            // the data, and one of F's persistent CTAs (one per SM, statically assigned work)
            // would then wait for that SM -- posting it after iteration k-1 instead made the
            // 4-GPU NCCL solve 18 % slower (profiles/r02_gpu_multi_w4_nccl_recv.log)
            CK(cudaStreamWaitEvent(g->comm_stream, fdone_ev, 0));
            NCK(ncclRecv(recvb, msg, ncclDouble, op.peer, g->comm, g->comm_stream), op.k);
            CK(cudaEventRecord(recv_ev(op.k), g->comm_stream));
            CK(cudaStreamWaitEvent(st, recv_ev(op.k), 0));
            if (ctrl) CK(cudaMemcpyAsync(g->h_flag, recvb + g->N, sizeof(double),
                                         cudaMemcpyDeviceToHost, st));
            recvd = true;
            break;
        case PR_OP_G: {
            const double *in;
            if (op.slice == 0) in = u0d;
            else if (l == 0) in = recvd ? recvb : start[0];  // stopped predecessor: last value
            else in = out[l - 1];
            if (l == 0) CK(cudaEventRecord(evW(op.k), st));
            CKS(G(in, gnew, op.slice));
            break;
        }
        case PR_OP_CORRECT: {
            if (l == s - 1 && sent_pending) {  // out[s-1] still being sent from iteration k-1
                CK(cudaStreamWaitEvent(st, evS(last_send_k), 0));
                sent_pending = false;
            }
            const bool fuse = want_def && op.slice == Np - 1;
            // previous iterate of this slice's end value: the coarse guess in
            // iteration 0, else start[l+1] (l < s-1) or out[s-1] itself
            const double *prev = op.k == 0 ? gold[l] : (l < s - 1 ? start[l + 1] : out[s - 1]);
            // peer mode, hand-off slice: the same pass stores into the successor's
            // receive buffer once the successor has released it
            double *pmail = nullptr;
            if (peer && l == s - 1 && r < W - 1) {
                CKS(stream_wait_geq(g, st, g->d_flags + 1, base + unsigned(op.k), false));
                pmail = g->peer_mail[op.k & 1];
            }
            if (lh && l == s - 1 && r < W - 1) {  // the successor has released the buffer
                const int k = op.k;
                if (k == 0) {
                    CKS(local_wait(g, k, r + 1, "the start of its call",
                                   [&](LocalGroup &G_) { return G_.r[r + 1].started >= base + 1ull; }));
                } else {
                    CKS(local_wait(g, k, r + 1, "its receive buffer",
                                   [&](LocalGroup &G_) { return G_.r[r + 1].freed >= base + unsigned(k); }));
                }
                cudaEvent_t ev = nullptr;
                {
                    std::lock_guard<std::mutex> lk(LG->mu);
                    if (k > 0) ev = LG->r[r + 1].ev_free[k - 1];
                    pmail = LG->r[r + 1].mail[k & 1];
                }
                if (ev) CK(cudaStreamWaitEvent(st, ev, 0));
            }
            CKS(launch_correct(g, f[l], gnew, gold[l], out[l], fuse ? refd : nullptr,
                               g->d_red + op.k + 1, st, prev, red_chg + 2 * op.k,
                               red_chg + 2 * op.k + 1, pmail));
            std::swap(gold[l], gnew);
            if (l == s - 1) {  // end of this rank's iteration: the stop decision
                iters = op.k + 1;
                bool stop_now = (op.k == K - 1);
                if (ctrl) {
                    CK(cudaMemcpyAsync(g->h_red, red_chg + 2 * op.k, 2 * sizeof(unsigned long long),
                                       cudaMemcpyDeviceToHost, st));
                    CKS(wait_all(g, st, op.k, false));
                    const double dm = bits_to_double(g->h_red[0]), um = bits_to_double(g->h_red[1]);
                    const double ch = um > 0.0 ? dm / um : dm;
                    g->monitors[op.k] = ch;
                    if (recvd && g->h_flag[0] != 0.0) pred_stopped = true;
                    if (pred_stopped && ch <= tol) stop_now = true;
                    if (r < W - 1 && !peer && !lh) {  // the flag rides on this iteration's message
                        set_flag_kernel<<<1, 1, 0, st>>>(out[s - 1] + g->N, stop_now ? 1.0 : 0.0);
                        g_launches.fetch_add(1, std::memory_order_relaxed);
                        CKL();
                    }
                }
                if (peer && r < W - 1)  // publish: stop flag, then the data sequence word
                    CKS(post(g, ctrl ? pmail + g->N : nullptr, stop_now ? 1.0 : 0.0,
                             g->succ_flags + 0, base + unsigned(op.k) + 1, st));
                if (lh && r < W - 1) {  // stop flag into the message tail, then announce
                    if (ctrl) {
                        set_flag_kernel<<<1, 1, 0, st>>>(pmail + g->N, stop_now ? 1.0 : 0.0);
                        g_launches.fetch_add(1, std::memory_order_relaxed);
                        CKL();
                    }
                    CKS(local_publish(g, LG->r[r].ev_data[op.k], st, &LocalRank::data,
                                      base + unsigned(op.k) + 1ull));
                }
                if (stop_now) stopped = true;
            }
            break;
        }
        case PR_OP_SEND:
            if (peer || lh) break;  // stored by the correction kernel, then published
            CK(cudaEventRecord(corr_ev(op.k), st));
            CK(cudaStreamWaitEvent(g->comm_stream, corr_ev(op.k), 0));
            NCK(ncclSend(out[s - 1], msg, ncclDouble, op.peer, g->comm, g->comm_stream), op.k);
            CK(cudaEventRecord(evS(op.k), g->comm_stream));
            sent_pending = true;
            last_send_k = op.k;
            break;
        case PR_OP_END_ITER:
            CK(cudaEventRecord(evI(op.k), st));
            // start[l] <- the input slice l used in this iteration (buffer rotation)
            for (int ll = s - 1; ll >= 1; --ll) std::swap(start[ll], out[ll - 1]);
            if (j0 > 0 && recvd) std::swap(start[0], recvb);
            break;
        default:
            return fail(PR_EINVAL, "bad plan op %d", op.op);
        }
        // a rank that stops still sends its last message (and records its iteration end)
        if (stopped && op.op == PR_OP_CORRECT && op.slice == j0 + s - 1) {
            if (r < W - 1 && !peer && !lh) {
                CK(cudaEventRecord(corr_ev(op.k), st));
                CK(cudaStreamWaitEvent(g->comm_stream, corr_ev(op.k), 0));
                NCK(ncclSend(out[s - 1], msg, ncclDouble, r + 1, g->comm, g->comm_stream), op.k);
                CK(cudaEventRecord(evS(op.k), g->comm_stream));
            }
            CK(cudaEventRecord(evI(op.k), st));
        }
    }
    if (!init_marked) CK(cudaEventRecord(ev_init, st));
    g->iters = iters;
    if (last) {
        const double *res = iters > 0 ? out[s - 1] : gold[s - 1];
        // after END_ITER the final output of the last slice is still out[s-1]
        CK(cudaMemcpyAsync(u_T, res, g->bytes,
                           is_host_ptr(u_T) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaMemcpyAsync(g->h_red, g->d_red, size_t(3 * K + 4) * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
    cudaEvent_t ev_end = g->evs[2 + 4 * K];
    CK(cudaEventRecord(ev_end, st));
    if (local) {
        CK(cudaEventRecord(g->join_ev, st));
        CK(cudaStreamWaitEvent(user_st, g->join_ev, 0));
    }
    CKS(wait_all(g, st, K - 1));
    if (want_def) {
        const double M = bits_to_double(g->h_red[K + 1]);
        if (M == 0.0) return fail(PR_EDOMAIN, "max|u_ref| = 0: defect undefined");
        for (int k = 0; k <= K; ++k)
            defects_host[k] = k <= iters ? bits_to_double(g->h_red[k]) / M : std::nan("");
    }
    if (!ctrl) {
        for (int k = 0; k < iters; ++k) {
            const double dm = bits_to_double(g->h_red[K + 2 + 2 * k]);
            const double um = bits_to_double(g->h_red[K + 3 + 2 * k]);
            g->monitors[k] = um > 0.0 ? dm / um : dm;
        }
    }
    // timings
    float tot = 0, init = 0;
    cudaEventElapsedTime(&tot, ev_start, ev_end);
    cudaEventElapsedTime(&init, ev_start, ev_init);
    for (int k = 0; k < iters; ++k) {
        float a = 0, b = 0, cc = 0;
        cudaEvent_t prev = k == 0 ? ev_init : evI(k - 1);
        cudaEventElapsedTime(&a, prev, evF(k));
        cudaEventElapsedTime(&b, evF(k), evW(k));
        cudaEventElapsedTime(&cc, evW(k), evI(k));
        ms_fine += a;
        ms_wait += b;
        ms_gc += cc;
    }
    g->timings[0] = tot;
    g->timings[1] = init;
    g->timings[2] = ms_fine;
    g->timings[3] = ms_wait;
    g->timings[4] = ms_gc;
    return PR_OK;
}

pr_status pr_last_monitors(pr_grid *g, double *changes, int32_t cap, int32_t *iterations) {
    if (!g || !iterations || (cap > 0 && !changes)) return fail(PR_EINVAL, "bad argument");
    *iterations = g->iters;
    for (int k = 0; k < std::min<int>(cap, int(g->monitors.size())); ++k) changes[k] = g->monitors[k];
    return PR_OK;
}

pr_status pr_grid_info(const pr_grid *g, pr_grid_info_t *info) {
    if (!g || !info) return fail(PR_EINVAL, "null argument");
    info->fine_kernels_per_step = g->f1 ? 1 : g->f2 ? 2 : 4;
    info->fine_bytes_per_point = g->f1 ? 16 : g->f2 ? 56 : 128;
    info->coarse_bytes_per_point = 16;
    info->sms = g->sms;
    info->fine_variant = g->f2 ? g->fvariant : 0;
    return PR_OK;
}

pr_status pr_last_timings(pr_grid *g, double *out, int32_t cap) {
    if (!g || !out || cap < 5) return fail(PR_EINVAL, "bad argument");
    for (int i = 0; i < 5; ++i) out[i] = g->timings[i];
    return PR_OK;
}

}  // extern "C"
