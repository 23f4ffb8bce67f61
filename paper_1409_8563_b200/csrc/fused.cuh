// fused.cuh — one classical RK4 step as TWO kernels, each fusing
// two stages with an overlapped (redundantly computed) halo ring.  DESIGN.md §5.
//
//   fused_persist_kernel<K_A>:  k1 = L(u) on the tile + 2-point ring, Ya = u + dt/2 k1
//                       kept in shared memory; k2 = L(Ya) on the tile;
//                       acc = u + dt/6 k1 + dt/3 k2,  Yb = u + dt/2 k2.
//                       HBM: read u, write acc, Yb               (24 B/point)
//   fused_persist_kernel<K_B>:  k3 = L(Yb) on tile + ring, Ya' = u + dt k3 in shared
//                       memory; k4 = L(Ya') on the tile;
//                       u_new = acc + dt/3 k3 + dt/6 k4  (written over acc).
//                       HBM: read Yb, u, acc, write u_new        (32 B/point)
// One RK4 step moves 56 B/point instead of 128 B/point for four stage passes,
// with exactly the same floating-point operation sequence per point as the
// four-stage kernels (the two paths agree bitwise).
//
// Geometry: output tile 32 x TYO (x, y); stage A runs on the extended region
// 36 x (TYO+4); its input is read on 40 x (TYO+8).  One persistent CTA per SM
// walks work items (tile x z chunk).  Warp specialisation:
//   * producer warps stream the input planes (and K_B's u/acc planes) into a
//     DEPTH-slot shared ring: one TMA tensor copy per array and plane for tiles
//     away from the periodic seams (FILL = 2), 16-byte cp.async with the wrap
//     folded into a per-lane copy plan otherwise; arrivals by
//     cp.async.mbarrier.arrive.noinc plus the TMA transaction bytes; stage-A
//     warps release slots through an mbarrier;
//   * stage-A warps keep z neighbours in register queues (two adjacent x points
//     and RPT consecutive rows per thread), and write each intermediate plane
//     (Ya or Ya') plus the per-tile-point data stage B needs into a ZD-slot
//     shared ring;
//   * stage-B warps consume that ring (mbarrier full/empty hand-off, so both
//     stages run concurrently, stage A up to ZD-2 planes ahead) and store the
//     outputs to HBM coalesced along x.
#pragma once
#include <type_traits>

#include <cuda.h>  // CUtensorMap (header only; the encoder comes from the runtime)

#include "kernels.cuh"

namespace prk {

enum Kind2 { K_A = 0, K_B = 1 };

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// the same with the barrier's 32-bit shared-window address precomputed by the caller
// (smem_u32 of a barrier array inside a loop costs an S2R + LEA per use)
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// non-blocking probe of the phase with the given parity (1 = completed); acquire on success.
// Issued well ahead of its use, its latency overlaps independent work (try_wait costs ~90
// cycles even on a completed phase, B300_MICROARCH.md "mbarrier")
__device__ __forceinline__ uint32_t mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok;
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
// a barrier array in shared memory by its 32-bit address
struct SBars {
    uint32_t base;
    __device__ __forceinline__ uint32_t operator[](int i) const { return base + 8u * uint32_t(i); }
};
// a value the compiler cannot rematerialise: kept in a register instead of being rebuilt
// (S2R SR_CgaCtaId + LEA for a shared-window address) in every loop iteration
__device__ __forceinline__ uint32_t pin_u32(uint32_t v) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
// the dynamic shared-memory base with its window address pinned the same way (the generic
// pointer is rebuilt from the shared address, so loads through it stay LDS)
template <class C> __device__ __forceinline__ double *smem_base(double *sm) {
    if constexpr (C::PIN) {
        return reinterpret_cast<double *>(__cvta_shared_to_generic(pin_u32(smem_u32(sm))));
    } else {
        return sm;
    }
}
template <class C> __device__ __forceinline__ SBars sbars(const uint64_t *bar) {
    return SBars{C::PIN ? pin_u32(smem_u32(bar)) : smem_u32(bar)};
}
// arrive on the mbarrier once all of this thread's prior cp.async copies land
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// add `bytes` of expected transactions to the barrier's current phase (no arrival)
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) { mbar_expect_tx(smem_u32(bar), bytes); }
// 3-D tensor tile global -> shared on the TMA unit (no L1 data-pipe wavefronts);
// its bytes complete on the barrier.  map: address of a __grid_constant__ param.
__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap *map, int x, int y, int z,
                                          uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap *map, int x, int y, int z,
                                          uint64_t *bar) {
    tma_load3(dst, map, x, y, z, smem_u32(bar));
}
// prefetch a 3-D tensor tile into L2 (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch3(const CUtensorMap *map, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(z)
                 : "memory");
}
// Tensor maps of the TMA fills (FusedCfgP::FILL == 2), 3-D (x, y, z) over the
// n^3 fields, boxes one z plane deep: the padded smem pitch is the box width.
struct TmaMaps {
    CUtensorMap y;  // stencil input, box {IWS, IH, 1} at (x0 - 4, y0 - 4, z)
    CUtensorMap u;  // K_B aux u,     box {EWS, EH, 1} at (x0 - 2, y0 - 2, z)
    CUtensorMap c;  // K_B aux acc,   box {TXO, TYO, 1} at (x0, y0, z)
};
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---- Tensor memory (TMEM) as a warp-to-warp staging buffer (FusedCfgP::TM = 1).
// 128 lanes x 512 columns of 32 bits per SM; warp w reaches lanes 32 (w % 4) .. +31 with
// tcgen05.ld / tcgen05.st (thread i <-> lane 32 (w % 4) + i), a datapath separate from
// shared memory.  A stage-A warp and the stage-B warp of the same lane quadrant hand
// per-point values over through it instead of through the shared intermediate ring.
__device__ __forceinline__ void tm_alloc(uint32_t *dst_smem, uint32_t ncols) {  // one warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_dealloc(uint32_t taddr, uint32_t ncols) {  // the allocating warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tm_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 8 columns (two rows of a lane's two x points) from / to this thread's lane
__device__ __forceinline__ void tm_st8(uint32_t taddr, double2 a, double2 b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(__double2loint(a.x)), "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)),
                 "r"(__double2hiint(a.y)), "r"(__double2loint(b.x)), "r"(__double2hiint(b.x)),
                 "r"(__double2loint(b.y)), "r"(__double2hiint(b.y))
                 : "memory");
}
struct TmRaw8 { uint32_t r[8]; };
__device__ __forceinline__ void tm_ld8(uint32_t taddr, TmRaw8 &v) {  // tm_wait_ld() before use
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]),
                   "=r"(v.r[6]), "=r"(v.r[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ double2 tm_row(const TmRaw8 &v, int r) {  // row r of the two
    double2 d;
    d.x = __hiloint2double(int(v.r[4 * r + 1]), int(v.r[4 * r + 0]));
    d.y = __hiloint2double(int(v.r[4 * r + 3]), int(v.r[4 * r + 2]));
    return d;
}

// folded 13-point operator, C3 (same order as stencil_kernel)
struct Weights {
    double wm1[3], wp1[3], wm2[3], wp2[3], w0;
    __device__ __forceinline__ void load(const double *w) {  // fine_weights13 layout
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            wm1[d] = w[d]; wp1[d] = w[3 + d]; wm2[d] = w[6 + d]; wp2[d] = w[9 + d];
        }
        w0 = w[12];
    }
    __device__ __forceinline__ void set(double nu, double inv_dx, const double *c) {
        double w[13];
        fine_weights13(nu, inv_dx, c, w);
        load(w);
    }
};

template <int P> using Ph = std::integral_constant<int, P>;

// Run body(Ph<j % 5>{}, j) for j = 0 .. NJ-1: the loop is unrolled by five so
// that z queues indexed with (P + o) % 5 rotate by renaming, not by moves.
template <class Body>
__device__ __forceinline__ void rotating_loop(int NJ, Body &&body) {
    int j = 0;
#pragma unroll 1
    for (; j + 5 <= NJ; j += 5) {
        body(Ph<0>{}, j);
        body(Ph<1>{}, j + 1);
        body(Ph<2>{}, j + 2);
        body(Ph<3>{}, j + 3);
        body(Ph<4>{}, j + 4);
    }
    if (j < NJ) body(Ph<0>{}, j++);
    if (j < NJ) body(Ph<1>{}, j++);
    if (j < NJ) body(Ph<2>{}, j++);
    if (j < NJ) body(Ph<3>{}, j++);
}

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void sts2(double *p, double2 v) { *reinterpret_cast<double2 *>(p) = v; }

// the folded operator on explicit neighbours, same operation order as stencil_kernel:
// one FMA chain, centre first, then x, y and z neighbours (-1, +1, -2, +2) -- 13 FP64
// instructions per point (three partial sums cost 15; measured 2.3 % faster per RK4 step
// in the bench)
__device__ __forceinline__ double apply13(const Weights &W, double c, double xm2, double xm1,
                                          double xp1, double xp2, double ym2, double ym1,
                                          double yp1, double yp2, double zm2, double zm1,
                                          double zp1, double zp2) {
    double s = W.w0 * c;
    s = fma(W.wm1[0], xm1, s);
    s = fma(W.wp1[0], xp1, s);
    s = fma(W.wm2[0], xm2, s);
    s = fma(W.wp2[0], xp2, s);
    s = fma(W.wm1[1], ym1, s);
    s = fma(W.wp1[1], yp1, s);
    s = fma(W.wm2[1], ym2, s);
    s = fma(W.wp2[1], yp2, s);
    s = fma(W.wm1[2], zm1, s);
    s = fma(W.wp1[2], zp1, s);
    s = fma(W.wm2[2], zm2, s);
    s = fma(W.wp2[2], zp2, s);
    return s;
}

// both points of a lane pair: L = (x-2, x-1), Cc = (x, x+1), R = (x+2, x+3)
template <int P>
__device__ __forceinline__ double2 apply_pair(const Weights &W, double2 L, double2 R, double2 ym2,
                                              double2 ym1, double2 yp1, double2 yp2,
                                              const double2 *q) {
    const double2 Cc = q[(P + 2) % 5];
    const double2 zm2 = q[P % 5], zm1 = q[(P + 1) % 5], zp1 = q[(P + 3) % 5], zp2 = q[(P + 4) % 5];
    double2 k;
    k.x = apply13(W, Cc.x, L.x, L.y, Cc.y, R.x, ym2.x, ym1.x, yp1.x, yp2.x, zm2.x, zm1.x, zp1.x, zp2.x);
    k.y = apply13(W, Cc.y, L.y, Cc.x, R.x, R.y, ym2.y, ym1.y, yp1.y, yp2.y, zm2.y, zm1.y, zp1.y, zp2.y);
    return k;
}

// ---------------------------------------------------------------------------
// Persistent variant: one CTA per SM walks work items (tile x z chunk)
// blockIdx.x, blockIdx.x + gridDim.x, ...  All ring counters run on across
// items, so the producer warp streams the next item's first planes while the
// compute warps finish the current one (no per-item pipeline fill).  Aux planes
// (K_B) share the slot index of the input element they ride with.
template <int TYO_, int DEPTH_, int ZD_, int RPTA_, int RPTB_, int PW_ = 1, int FILL_ = 0,
          int UIN_ = 0, int DEPTHA_ = DEPTH_, int TM_ = 0, int DIAG_ = 0>
struct FusedCfgP {
    // DIAG (timing diagnostics only, results are garbage): 1 = consumers never wait for the
    // input ring after its first fill (compute-only upper bound); 2 = in addition stage A
    // and stage B never wait for each other; 3 = every tile by TMA
    static constexpr int DIAG = DIAG_;
    static constexpr bool COMB = false;  // comb.cuh configs: stage B in the stage-A lanes
    static constexpr bool WP = false;    // weights from the nu table (graph replays)
    static constexpr bool Z2 = false;    // z2.cuh: two z planes per consumer iteration
    static constexpr bool PF = false;    // stage A loads the next plane's operands one iteration ahead
    static constexpr bool SW = false;    // split-phase ring waits: probe early, block only on failure
    // shared-window addresses of the barriers and rings pinned in registers (pin_u32):
    // 2-3 % faster than letting the compiler rebuild them per iteration (variant 36 = off)
    static constexpr bool PIN = true;
    static constexpr bool OFF32 = false;  // stage-B stores by 32-bit element offsets (n^3 < 2^32)
    // ACCG (with TM): K_B's stage B reads acc from global memory itself (LDG, the producer only
    // prefetches the tile into L2), stage A hands k3 instead of t0 = acc + dt/3 k3 through TMEM
    static constexpr bool ACCG = false;
    // PFL2 > 0: the producer also prefetches the input plane PFL2 planes ahead into L2
    // (cp.async.bulk.prefetch.tensor), so the ring's TMA fills hit L2
    static constexpr int PFL2 = 0;
    static constexpr int TXO = 32, TYO = TYO_, DEPTH = DEPTH_, ZD = ZD_, MINB = 1, XP = 2,
                         PROD = 1, PW = PW_;  // PW producer warps
    // FILL 0: every plane by 16-byte cp.async; 2: planes of tiles away from the
    // periodic seams by one TMA tensor copy per array (box = padded slot rows)
    static constexpr int FILL = FILL_;
    // UIN: K_A's stage B reads u (for Yb = u + dt/2 k2) from the input ring instead of a
    // copy stage A leaves in the intermediate ring; input slots are then released by both
    // stages (one fewer shared store per point, slots held two planes longer)
    static constexpr int UIN = UIN_;
    static constexpr int RPTA = RPTA_, RPT = RPTB_;
    static constexpr int EW = TXO + 4, EH = TYO + 4, IW = TXO + 8, IH = TYO + 8;
    static constexpr int HX = 4, HY = 4, HZ = 4;  // input halo (two radius-2 stages)
    static constexpr int IWS = IW + 2, EWS = EW + 6;  // padded pitches: no bank conflicts for the lane maps
    static constexpr int GA = EH / RPTA, GB = TYO / RPT;
    static constexpr int A_ITEMS = (EW / 2) * GA, B_ITEMS = (TXO / 2) * GB;
    static constexpr int WA = (A_ITEMS + 31) / 32, WB = (B_ITEMS + 31) / 32;
    static constexpr int NTA = 32 * WA, NTB = 32 * WB, NTP = 32 * PW, NT = NTA + NTB + NTP;
    // TM: the per-point values stage B needs from stage A (its intermediate-plane z column,
    // t0 and, in K_A, u) go through tensor memory.  Thread layout [stage-A tile lanes |
    // stage B | stage-A ring lanes | producers], so that stage-A tile lane i and stage-B
    // lane i sit in warps of the same TMEM lane quadrant.
    static constexpr int TM = TM_;
    static constexpr int NTC = (TXO / 2) * (TYO / RPTA_);  // stage-A lanes on the tile
    static constexpr int B_BASE = TM ? NTC : NTA;           // first stage-B thread
    static constexpr int R_LANES = A_ITEMS - NTC;           // stage-A lanes on the halo ring
    static constexpr int TM_PLANE = 24;                     // TMEM columns per plane
    static constexpr int TM_COLS = TM_PLANE * ZD_ <= 32 ? 32 : TM_PLANE * ZD_ <= 64 ? 64 :
                                   TM_PLANE * ZD_ <= 128 ? 128 : TM_PLANE * ZD_ <= 256 ? 256 : 512;
    // register cap: the whole register file for one CTA of NT threads (multiple of 8),
    // or PRK_FUSED_MAXR when the build defines it (tuning)
#ifdef PRK_FUSED_MAXR
    static constexpr int MAXR = PRK_FUSED_MAXR;
#else
    static constexpr int MAXR = (65536 / NT) / 8 * 8 > 255 ? 255 : (65536 / NT) / 8 * 8;
#endif
    static constexpr int AD = DEPTH;  // aux slots follow the input slots
    // Z_ELEMS padded to 16 doubles: every slot and its T part stay 128-byte aligned (TMA)
    static constexpr int Y_ELEMS = IH * IWS, Z_ELEMS = (EH * EWS + 15) / 16 * 16, T_ELEMS = TYO * TXO;
    static constexpr int AUX_ELEMS = Z_ELEMS + T_ELEMS;
    static constexpr int Y_CHUNKS = IH * (IW / 2), U_CHUNKS = EH * (EW / 2), C_CHUNKS = TYO * (TXO / 2);
    static_assert(TYO % RPT == 0 && EH % RPTA == 0, "rows must split into row groups");
    static_assert(Y_ELEMS % 16 == 0 && Z_ELEMS % 16 == 0, "slots must stay 128-byte aligned");
    static_assert(DEPTH >= 5 && ZD >= 3, "rings too shallow");
    static_assert(!TM_ || (RPTA_ == RPTB_ && NTC % 128 == 0 && NTC == 32 * WB && !UIN_),
                  "TMEM hand-off: stage-A tile lanes map 1:1 onto stage-B lanes, four warps each");
    // input ring depth per kernel: K_A has shared memory to spare (no aux ring)
    template <int KB> static constexpr int DEPTH_K = KB == K_A ? DEPTHA_ : DEPTH;
    template <int KB> static constexpr int NTV = (KB == K_A && !UIN) ? 2 : 1;
    template <int KB> static constexpr int IN_CONSUMERS = (KB == K_A && UIN) ? NTA + NTB : NTA;
    template <int KB> static constexpr int ZS_ELEMS = Z_ELEMS + (TM ? 0 : NTV<KB> * T_ELEMS);
    template <int KB> static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t(DEPTH_K<KB>) * Y_ELEMS + (KB == K_B ? size_t(AD) * AUX_ELEMS : 0) +
                                 size_t(ZD) * ZS_ELEMS<KB>);
    }
};
using FusedP4 = FusedCfgP<16, 9, 4, 2, 2, 2, 2>;  // 32x16 tile, TMA tensor fills (default, PR_FTILE=14)
// 32x32 output tile, four rows per lane in both stages (12 warps): stage A's halo ring
// recomputes 27 % instead of 41 %, and each lane reads 2 instead of 2.5 shared values per point
// power-of-two ring depths: ring positions as masked counters (K_A 16 input slots, K_B 8)
using FusedQ16 = FusedCfgP<16, 8, 4, 2, 2, 2, 2, 0, 16>;
using FusedQ8 = FusedCfgP<16, 8, 4, 2, 2, 2, 2, 0, 8>;
using FusedT32 = FusedCfgP<32, 7, 4, 4, 4, 2, 2, 0, 7>;
using FusedT32B = FusedCfgP<32, 5, 3, 4, 4, 2, 2, 0, 5>;  // K_B at 32x32: shallower rings to fit
// 32x16 tile with the stage A -> stage B per-point hand-off through tensor memory
using FusedTM = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 9, 1>;
// the same with stage A's TMEM stores issued before its shared ones (PR_FTILE=38), or stage
// B's three TMEM loads of an iteration behind one wait (39; spills), PRK_VARIANTS
using FusedTM2 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 9, 2>;
using FusedTM3 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 9, 3>;
// TMEM hand-off with a 16-slot K_A input ring (K_A has the shared memory to spare once the
// per-point values leave the Z ring; PR_FTILE=42 with FusedTM for K_B, PRK_VARIANTS)
using FusedTMQ16 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 16, 1>;
template <class C> struct WithACCG : C {
    static_assert(C::TM == 1, "ACCG hands k3 through tensor memory");
    static constexpr bool ACCG = true;
};
using FusedTMACC = WithACCG<FusedTM>;  // PR_FTILE=43 (PRK_VARIANTS)
template <class C, int D> struct WithPFL2 : C { static constexpr int PFL2 = D; };
using FusedTMPF4 = WithPFL2<FusedTM, 4>;  // PR_FTILE=44 (PRK_VARIANTS)
using FusedTMPF8 = WithPFL2<FusedTM, 8>;  // PR_FTILE=45
// timing diagnostics (garbage results): no input waits / no waits at all (PR_FTILE 26 / 27)
using FusedD1 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 9, 0, 1>;
using FusedD2 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 9, 0, 2>;
using FusedD3 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 9, 0, 3>;  // every tile by TMA (PR_FTILE 28)
// the same kernel with the two stages' weights passed as launch parameters (direct launches):
// they sit in uniform registers / the constant bank instead of 26 registers per thread
template <class C> struct WithWP : C { static constexpr bool WP = true; };
// stage A software-pipelined: the next plane's shared-memory operands are loaded before
// this plane's stencil, so their latency hides under its FMA chains (more live registers)
template <class C> struct WithPF : C { static constexpr bool PF = true; };
// split-phase ring waits: each consumer probes (mbarrier.test_wait) the barrier it needs
// next one step ahead and blocks (try_wait) only if the probe failed
template <class C> struct WithSW : C { static constexpr bool SW = true; };
using FusedSW = WithSW<FusedP4>;
template <class C> struct NoPIN : C { static constexpr bool PIN = false; };
using FusedNoPIN = NoPIN<FusedP4>;
template <class C> struct WithOFF32 : C { static constexpr bool OFF32 = true; };
using FusedOFF32 = WithOFF32<FusedP4>;
using FusedPF = WithPF<FusedP4>;  // PR_FTILE=29 (PRK_VARIANTS): 12 % slower, spills at 168 registers
#ifdef PRK_VARIANTS  // tuning history (profiles/r01_kernel_bench_variants.txt)
// deeper intermediate (Z) rings: stage A may run further ahead of stage B (K_A ZD 6 / 8, K_B 5)
using FusedZD6 = FusedCfgP<16, 9, 6, 2, 2, 2, 2>;
using FusedZD8 = FusedCfgP<16, 9, 8, 2, 2, 2, 2>;
using FusedP0 = FusedCfgP<16, 7, 4, 2, 2, 1>;   // one producer warp
using FusedP1 = FusedCfgP<16, 9, 4, 2, 2, 1>;
using FusedP2 = FusedCfgP<16, 8, 5, 2, 2, 2>;   // 5-slot intermediate ring
using FusedP3 = FusedCfgP<16, 9, 4, 2, 2, 2>;     // two producer warps, cp.async only
using FusedP5 = FusedCfgP<16, 9, 5, 2, 2, 2, 2>;  // + 5-slot intermediate ring
using FusedP6 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 1>;  // + K_A stage B reads u from the input ring
using FusedP7 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 0, 12>;  // 12-slot input ring in K_A
using FusedP8 = FusedCfgP<16, 9, 4, 4, 4, 2, 2>;  // four rows per lane (7 warps: <= 256 threads at ~190 regs)
using FusedP9 = FusedCfgP<16, 9, 4, 2, 2, 2, 2, 1, 13>;  // UIN + 13-slot input ring in K_A
#endif

struct WorkItem {
    int x0, y0, z_begin, nz;
};
// periodic wrap of an index known to lie in [-n, 2n) (fused path: n >= 32, halo <= 4)
__device__ __forceinline__ int wrap1(int i, int n) {
    i += (i < 0) ? n : 0;
    return i - ((i >= n) ? n : 0);
}
__device__ __forceinline__ WorkItem decode_item(const StencilArgs &a, int item, int txo, int tyo) {
    WorkItem w;
    int b = item;
    const int tix = b % a.tiles_x; b /= a.tiles_x;
    const int tiy = b % a.tiles_y; b /= a.tiles_y;
    w.x0 = tix * txo;
    w.y0 = tiy * tyo;
    w.z_begin = b * a.cz;
    w.nz = min(a.cz, a.n - w.z_begin);
    PRK_CHECK(w.x0 + txo <= a.n && w.y0 + tyo <= a.n && w.nz >= 1 && w.z_begin + w.nz <= a.n);
    return w;
}

// ring position: slot index and the fill round it belongs to
struct RingPos {
    int slot = 0, round = 0;
    __device__ __forceinline__ void step(int depth) {
        if (++slot == depth) { slot = 0; ++round; }
    }
};
__device__ __forceinline__ RingPos ring_at(RingPos p, int k, int depth) {
    for (int i = 0; i < k; ++i) p.step(depth);
    return p;
}

// ring position of a D-slot ring as a running counter: for power-of-two D the slot
// and round are a mask and a shift of it (fewer integer instructions per pipeline
// step than the incremental slot/round pair, which other depths keep)
template <int D, bool P2 = (D & (D - 1)) == 0> struct RingP;
template <int D> struct RingP<D, true> {
    unsigned c = 0;
    __device__ __forceinline__ int slot() const { return int(c & unsigned(D - 1)); }
    __device__ __forceinline__ int round() const { return int(c / unsigned(D)); }
    __device__ __forceinline__ void step() { ++c; }
    __device__ __forceinline__ RingP at(int k) const { RingP r; r.c = c + unsigned(k); return r; }
};
template <int D> struct RingP<D, false> {
    int s = 0, r = 0;
    __device__ __forceinline__ int slot() const { return s; }
    __device__ __forceinline__ int round() const { return r; }
    __device__ __forceinline__ void step() { if (++s == D) { s = 0; ++r; } }
    __device__ __forceinline__ RingP at(int k) const {
        RingP q = *this;
        for (int i = 0; i < k; ++i) q.step();
        return q;
    }
};

// Chunk c (16 bytes) of a rows x (mid + 2 hc)-chunk tile plane -> (row, chunk column),
// ordered so that eight consecutive producer lanes fetch one aligned 128-byte
// global line: first the mid chunks of every row (the tile's own x range, 256-byte
// aligned), then the hc halo chunks on each side.  Fewer L1 wavefronts per LDGSTS.
__device__ __forceinline__ void line_order(int c, int rows, int mid, int hc, int &r, int &cc) {
    if (c < rows * mid) {
        r = c / mid;
        cc = hc + c % mid;
    } else {
        const int e = c - rows * mid, k = e % (2 * hc);
        r = e / (2 * hc);
        cc = k < hc ? k : mid + k;
    }
}

template <int KB, class C>
__device__ __forceinline__ void producer_p(const StencilArgs &a, const TmaMaps *tm, double *sm,
                                           int items, uint64_t *in_full, uint64_t *in_empty) {
    const SBars in_full_s = sbars<C>(in_full);
    const SBars in_empty_s = sbars<C>(in_empty);
    constexpr int DEPTH = C::template DEPTH_K<KB>, EW = C::EWS, IW = C::IWS, TXO = C::TXO;
    constexpr int NP = C::NTP;
    constexpr int NY = (C::Y_CHUNKS + NP - 1) / NP, NU = (C::U_CHUNKS + NP - 1) / NP,
                  NC = (C::C_CHUNKS + NP - 1) / NP;
    double *yring = sm;
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    // 0 .. NP-1 (NTA + NTB is a multiple of 32, so the % keeps the range visible)
    const int lane = (threadIdx.x - (C::NTA + C::NTB)) % NP;
    const uint32_t yring_s = C::PIN ? pin_u32(smem_u32(yring)) : smem_u32(yring);
    const uint32_t aring_s = yring_s + uint32_t(sizeof(double) * DEPTH * C::Y_ELEMS);
    RingP<DEPTH> pos;
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int E = w.nz + 2 * C::HZ, NJ = w.nz + 4;
        int ysrc[NY], ydst[NY];
#pragma unroll
        for (int k = 0; k < NY; ++k) {
            const int c = lane + NP * k;
            ysrc[k] = -1;
            ydst[k] = 0;
            if (c < C::Y_CHUNKS) {
                int r, cc;
                line_order(c, C::IH, TXO / 2, C::HX / 2, r, cc);
                ysrc[k] = wrap1(w.y0 - C::HY + r, n) * n + wrap1(w.x0 - C::HX + 2 * cc, n);
                ydst[k] = 8 * (r * IW + 2 * cc);
                PRK_CHECK(ysrc[k] >= 0 && ysrc[k] + 2 <= n * n && ydst[k] + 16 <= 8 * C::Y_ELEMS);
            }
        }
        int usrc[KB == K_B ? NU : 1], udst[KB == K_B ? NU : 1];
        int csrc[KB == K_B ? NC : 1], cdst[KB == K_B ? NC : 1];
        if constexpr (KB == K_B) {
#pragma unroll
            for (int k = 0; k < NU; ++k) {
                const int c = lane + NP * k;
                usrc[k] = -1;
                udst[k] = 0;
                if (c < C::U_CHUNKS) {
                    int r, cc;
                    line_order(c, C::EH, TXO / 2, 1, r, cc);
                    usrc[k] = wrap1(w.y0 - 2 + r, n) * n + wrap1(w.x0 - 2 + 2 * cc, n);
                    udst[k] = 8 * (r * EW + 2 * cc);
                    PRK_CHECK(usrc[k] >= 0 && usrc[k] + 2 <= n * n && udst[k] + 16 <= 8 * C::Z_ELEMS);
                }
            }
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                const int c = lane + NP * k;
                csrc[k] = -1;
                cdst[k] = 0;
                if (c < C::C_CHUNKS) {
                    const int r = c / (TXO / 2), cc = c % (TXO / 2);
                    csrc[k] = (w.y0 + r) * n + w.x0 + 2 * cc;
                    cdst[k] = 8 * (C::Z_ELEMS + r * TXO + 2 * cc);
                    PRK_CHECK(csrc[k] + 2 <= n * n && cdst[k] + 16 <= 8 * C::AUX_ELEMS);
                }
            }
        }
        // TMA fills for tiles whose boxes stay inside the field (no periodic seam)
        // (DIAG 3, timing only: every tile by TMA, zero-filled instead of wrapped at the seams)
        const bool tma = C::FILL == 2 && ((w.x0 >= C::HX && w.x0 - C::HX + IW <= n &&
                                           w.y0 >= C::HY && w.y0 - C::HY + C::IH <= n &&
                                           (KB == K_A || w.x0 - 2 + EW <= n)) || C::DIAG == 3);
        int zin = wrap1(w.z_begin - C::HZ, n);
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
            if constexpr (C::DIAG == 1 || C::DIAG == 2) {
                if (pos.round() > 0) break;  // only the first fill
            }
            if (pos.round() > 0) mbar_wait(in_empty_s[pos.slot()], (pos.round() - 1) & 1);
            if constexpr (C::FILL == 2) {
                if (tma) {
                    if (lane == 0) {
                        const uint32_t bar = in_full_s[pos.slot()];
                        const int j = e - 4;
                        const bool ua = KB == K_B && j >= 0 && j < NJ;
                        const bool ca = ua && j >= 2 && j < w.nz + 2 && !C::ACCG;
                        mbar_expect_tx(bar, 8u * (C::IH * IW + (ua ? C::EH * EW : 0) +
                                                  (ca ? C::T_ELEMS : 0)));
                        tma_load3(yring_s + uint32_t(pos.slot()) * (C::Y_ELEMS * 8), &tm->y,
                                  w.x0 - C::HX, w.y0 - C::HY, zin, bar);
                        if constexpr (C::PFL2 > 0) {  // within this item's planes only
                            if (e + C::PFL2 < E) {
                                int zp = zin + C::PFL2;
                                if (zp >= n) zp -= n;
                                tma_prefetch3(&tm->y, w.x0 - C::HX, w.y0 - C::HY, zp);
                            }
                        }
                        if (ua) {
                            const int zaux = zin >= 2 ? zin - 2 : zin - 2 + n;
                            const uint32_t dst = aring_s + uint32_t(pos.slot()) * (C::AUX_ELEMS * 8);
                            tma_load3(dst, &tm->u, w.x0 - 2, w.y0 - 2, zaux, bar);
                            if (ca) tma_load3(dst + 8 * C::Z_ELEMS, &tm->c, w.x0, w.y0, zaux, bar);
                            if (C::ACCG && j >= 2 && j < w.nz + 2) tma_prefetch3(&tm->c, w.x0, w.y0, zaux);
                        }
                    }
                    cp_async_mbar_arrive(in_full_s[pos.slot()]);
                    zin = (zin + 1 == n) ? 0 : zin + 1;
                    pos.step();
                    continue;
                }
            }
            {
                const double *src = a.y + size_t(zin) * nn;
                const uint32_t dst = yring_s + uint32_t(pos.slot()) * (C::Y_ELEMS * 8);
#pragma unroll
                for (int k = 0; k < NY; ++k)
                    if (ysrc[k] >= 0) cp_async16s(dst + ydst[k], src + ysrc[k]);
            }
            if constexpr (KB == K_B) {
                const int j = e - 4;  // aux j rides with input element j+4
                if (j >= 0 && j < NJ) {
                    int zaux = zin - 2;
                    if (zaux < 0) zaux += n;
                    const size_t pl = size_t(zaux) * nn;
                    const uint32_t dst = aring_s + uint32_t(pos.slot()) * (C::AUX_ELEMS * 8);
#pragma unroll
                    for (int k = 0; k < NU; ++k)
                        if (usrc[k] >= 0) cp_async16s(dst + udst[k], a.p0 + pl + usrc[k]);
                    if (!C::ACCG && j >= 2 && j < w.nz + 2) {
#pragma unroll
                        for (int k = 0; k < NC; ++k)
                            if (csrc[k] >= 0) cp_async16s(dst + cdst[k], a.p1 + pl + csrc[k]);
                    }
                }
            }
            cp_async_mbar_arrive(in_full_s[pos.slot()]);
            zin = (zin + 1 == n) ? 0 : zin + 1;
            pos.step();
        }
    }
    cp_async_wait<0>();
}

template <int KB, class C>
__device__ __forceinline__ void stage_a_p(const StencilArgs &a, double *sm, int items,
                                          uint64_t *full, uint64_t *empty, uint64_t *in_full,
                                          uint64_t *in_empty, uint32_t tmem) {
    const SBars full_s = sbars<C>(full);
    const SBars empty_s = sbars<C>(empty);
    const SBars in_full_s = sbars<C>(in_full);
    const SBars in_empty_s = sbars<C>(in_empty);
    constexpr int RPT = C::RPTA, DEPTH = C::template DEPTH_K<KB>, EW = C::EWS, IW = C::IWS, TXO = C::TXO,
                  ZD = C::ZD;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    double *yring = smem_base<C>(sm);
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    double *zring = aring + (KB == K_B ? size_t(C::AD) * C::AUX_ELEMS : 0);
    // stage-A lane index: TM puts the tile lanes first (threads 0 .. NTC-1) and the ring
    // lanes after the stage-B threads
    const int t = (!C::TM || threadIdx.x < C::NTC) ? int(threadIdx.x)
                                                    : C::NTC + int(threadIdx.x) - (C::B_BASE + C::NTB);
    const bool tile_lane = C::TM && t < C::NTC;  // writes its per-point values to TMEM
    // TMEM address of this warp's lane quadrant
    const uint32_t tq_addr = tmem + (uint32_t(32 * ((threadIdx.x >> 5) & 3)) << 16);

    Weights W;
    if constexpr (C::WP) {
        W.load(a.wA);
    } else {
        const long long row = (*a.nu_pos + a.j_local) * 4;
        W.set(a.nu_tab[row + (KB == K_A ? 0 : 2)], a.inv_dx, a.c);
    }
    const double dt = a.dt;

    const bool valid = t < C::A_ITEMS;
    int l = valid ? t % (C::EW / 2) : 0, g = valid ? t / (C::EW / 2) : 0;
    if constexpr (C::TM) {  // tile lanes as stage B's lanes, then the ring (comb.cuh's map)
        if (t < C::NTC) {
            l = t % (TXO / 2) + 1;
            g = t / (TXO / 2) + 1;
        } else {
            const int u = t - C::NTC, top = C::EW / 2;
            if (!valid) { l = 0; g = 0; }
            else if (u < top) { l = u; g = 0; }
            else if (u < 2 * top) { l = u - top; g = C::EH / RPT - 1; }
            else { const int v = u - 2 * top; l = (v & 1) ? top - 1 : 0; g = 1 + (v >> 1); }
        }
    }
    const int r0 = g * RPT;
    const int sY = (r0 + 2) * IW + 2 * l + 2;
    const int sZ = r0 * EW + 2 * l;
    // every shared access of this lane: x/y neighbours of its RPT rows, its Z-ring rows
    PRK_CHECK(sY - 2 * IW - 2 >= 0 && sY + (RPT + 1) * IW + 4 <= C::Y_ELEMS);
    PRK_CHECK(sZ >= 0 && sZ + (RPT - 1) * EW + 2 <= C::Z_ELEMS);
    const bool tcol = l >= 1 && l <= TXO / 2;
    const int tp0 = (r0 - 2) * TXO + 2 * l - 2;

    RingP<DEPTH> base;  // input element 0 of the current item
    RingP<ZD> zpos;     // next Z plane
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;
        double2 q[RPT][5];
        RingP<DEPTH> p0 = base;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if ((C::DIAG != 1 && C::DIAG != 2) || p0.round() == 0) mbar_wait(in_full_s[p0.slot()], p0.round() & 1);
            const double *ys = yring + size_t(p0.slot()) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][e] = lds2(ys + r * IW);
            p0.step();
        }
        // elements 0 and 1 were only needed for the queue
        mbar_arrive(in_empty_s[base.slot()]);
        mbar_arrive(in_empty_s[base.at(1).slot()]);
        RingP<DEPTH> p2 = base.at(2), p4 = p0;  // elements j+2, j+4
        // the shared-memory operands of one plane: the new z-queue entry (element j+4), the
        // y (+-2 rows) and x neighbours on element j+2, K_B's u and acc (aux j)
        struct LdA {
            double2 qn[RPT], ym[2], yp[2], L[RPT], R[RPT], ub[KB == K_B ? RPT : 1], ac[KB == K_B ? RPT : 1];
        };
        auto load = [&](LdA &d, RingP<DEPTH> e4, RingP<DEPTH> e2, bool ready = false) {
            if (!ready && ((C::DIAG != 1 && C::DIAG != 2) || e4.round() == 0))
                mbar_wait(in_full_s[e4.slot()], e4.round() & 1);  // element j+4 (+ aux j) landed
            const double *yq = yring + size_t(e4.slot()) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) d.qn[r] = lds2(yq + r * IW);
            const double *ys = yring + size_t(e2.slot()) * C::Y_ELEMS + sY;
            d.ym[0] = lds2(ys - 2 * IW);
            d.ym[1] = lds2(ys - IW);
            d.yp[0] = lds2(ys + RPT * IW);
            d.yp[1] = lds2(ys + (RPT + 1) * IW);
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                d.L[r] = lds2(ys + r * IW - 2);
                d.R[r] = lds2(ys + r * IW + 2);
            }
        };
        // K_B: u on the ring and the acc values of this lane's tile points (lanes without a
        // tile point read entry 0); aux j rides with element j+4 (waited for in load)
        auto load_aux = [&](LdA &d, RingP<DEPTH> e4) {
            if constexpr (KB == K_B) {
                const double *au = aring + size_t(e4.slot()) * C::AUX_ELEMS;  // aux j
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    d.ub[r] = lds2(au + sZ + r * EW);
                    const int er = r0 + r;
                    const bool need = tcol && er >= 2 && er < C::TYO + 2;
                    if constexpr (!C::ACCG) d.ac[r] = lds2(au + C::Z_ELEMS + (need ? tp0 + r * TXO : 0));
                }
            }
        };
        [[maybe_unused]] LdA nx;  // PF: the next plane's operands, loaded one iteration ahead
        if constexpr (C::PF) load(nx, p4, p2);
        uint32_t in_ok = 0;  // SW: element j+4 already probed complete
        rotating_loop(NJ, [&](auto ph, int j) {
            constexpr int P = decltype(ph)::value;
            LdA cur;
            if constexpr (C::PF) {
                cur = nx;
                if (j + 1 < NJ) load(nx, p4.at(1), p2.at(1));
            } else {
                load(cur, p4, p2, C::SW && in_ok);
            }
            load_aux(cur, p4);
            [[maybe_unused]] uint32_t z_ok = 0;
            if constexpr (C::SW) {  // probes for the next element and this plane's Z slot
                // branch-free, so that the stencil below shares their basic block: the probe of
                // element j+5 may look at the next item's first slot (harmless, masked), the
                // round-0 probe of a Z slot (parity 1 on a fresh barrier) passes at once
                const RingP<DEPTH> e5 = p4.at(1);
                in_ok = mbar_test(in_full_s[e5.slot()], e5.round() & 1) & uint32_t(j + 1 < NJ);
                z_ok = mbar_test(empty_s[zpos.slot()], uint32_t(zpos.round() - 1) & 1);
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = cur.qn[r];
            double2 col[RPT + 4];
#pragma unroll
            for (int r = 0; r < RPT + 4; ++r)
                col[r] = r < 2 ? cur.ym[r] : r < RPT + 2 ? q[r - 2][(P + 2) % 5] : cur.yp[r - RPT - 2];
            [[maybe_unused]] const bool outp = j >= 2 && j < w.nz + 2;
            const double2 *ubv = cur.ub, *acv = cur.ac;
            double2 k[RPT];
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                k[r] = apply_pair<P>(W, cur.L[r], cur.R[r], col[r], col[r + 1], col[r + 3], col[r + 4], q[r]);
            if (C::DIAG != 2 && zpos.round() > 0 && !(C::SW && z_ok))
                mbar_wait(empty_s[zpos.slot()], (zpos.round() - 1) & 1);
            double *zs = zring + size_t(zpos.slot()) * ZS;
            if constexpr (C::TM) {
                if (tile_lane) {  // intermediate centre, t0 (and u) of this plane -> TMEM
                    tm_fence_after();
                    double2 zz[RPT], t0v[RPT];
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        const double2 yc = q[r][(P + 2) % 5];
                        if (KB == K_A) {
                            zz[r].x = yc.x + (dt / 2.0) * k[r].x;
                            zz[r].y = yc.y + (dt / 2.0) * k[r].y;
                            t0v[r].x = yc.x + (dt / 6.0) * k[r].x;
                            t0v[r].y = yc.y + (dt / 6.0) * k[r].y;
                        } else {
                            const double2 ub = ubv[KB == K_B ? r : 0];
                            zz[r].x = ub.x + dt * k[r].x;
                            zz[r].y = ub.y + dt * k[r].y;
                            if constexpr (C::ACCG) {  // k3 itself: stage B adds acc
                                t0v[r] = k[r];
                            } else {
                                const double2 ac = acv[KB == K_B ? r : 0];
                                t0v[r].x = ac.x + (dt / 3.0) * k[r].x;
                                t0v[r].y = ac.y + (dt / 3.0) * k[r].y;
                            }
                        }
                        if constexpr (C::TM != 2) sts2(zs + sZ + r * EW, zz[r]);  // x/y neighbours for stage B
                    }
                    const uint32_t col = tq_addr + uint32_t(zpos.slot() * C::TM_PLANE);
                    tm_st8(col, zz[0], zz[1]);
                    tm_st8(col + 8, t0v[0], t0v[1]);
                    if (KB == K_A) tm_st8(col + 16, q[0][(P + 2) % 5], q[1][(P + 2) % 5]);
                    if constexpr (C::TM == 2) {  // the shared stores under the TMEM stores' latency
#pragma unroll
                        for (int r = 0; r < RPT; ++r) sts2(zs + sZ + r * EW, zz[r]);
                    }
                    tm_wait_st();
                    tm_fence_before();
                } else if (valid) {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        double2 z;
                        if (KB == K_A) {
                            const double2 yc = q[r][(P + 2) % 5];
                            z.x = yc.x + (dt / 2.0) * k[r].x;
                            z.y = yc.y + (dt / 2.0) * k[r].y;
                        } else {
                            const double2 ub = ubv[KB == K_B ? r : 0];
                            z.x = ub.x + dt * k[r].x;
                            z.y = ub.y + dt * k[r].y;
                        }
                        sts2(zs + sZ + r * EW, z);
                    }
                }
            } else if (valid) {
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double2 yc = q[r][(P + 2) % 5];
                    double2 z;
                    if (KB == K_A) {
                        z.x = yc.x + (dt / 2.0) * k[r].x;
                        z.y = yc.y + (dt / 2.0) * k[r].y;
                    } else {
                        const double2 ub = ubv[KB == K_B ? r : 0];
                        z.x = ub.x + dt * k[r].x;
                        z.y = ub.y + dt * k[r].y;
                    }
                    sts2(zs + sZ + r * EW, z);
                    const int er = r0 + r;
                    if (outp && tcol && er >= 2 && er < C::TYO + 2) {
                        const int tp = tp0 + r * TXO;
                        PRK_CHECK(tp >= 0 && tp + 2 <= C::T_ELEMS);
                        if (KB == K_A) {
                            double2 t0;
                            t0.x = yc.x + (dt / 6.0) * k[r].x;
                            t0.y = yc.y + (dt / 6.0) * k[r].y;
                            sts2(zs + C::Z_ELEMS + tp, t0);
                            if constexpr (!C::UIN) sts2(zs + C::Z_ELEMS + C::T_ELEMS + tp, yc);
                        } else {
                            const double2 ac = acv[KB == K_B ? r : 0];
                            double2 t0;
                            t0.x = ac.x + (dt / 3.0) * k[r].x;
                            t0.y = ac.y + (dt / 3.0) * k[r].y;
                            sts2(zs + C::Z_ELEMS + tp, t0);
                        }
                    }
                }
            }
            mbar_arrive(full_s[zpos.slot()]);
            mbar_arrive(in_empty_s[p2.slot()]);  // element j+2 done (aux j lives in slot j+4)
            p2.step();
            p4.step();
            zpos.step();
        });
        // the item's last two input elements were only used by the queue
        mbar_arrive(in_empty_s[p2.slot()]);
        mbar_arrive(in_empty_s[p2.at(1).slot()]);
        base = p2.at(2);
    }
}

template <int KB, class C>
__device__ __forceinline__ void stage_b_p(const StencilArgs &a, double *sm, int items,
                                          uint64_t *full, uint64_t *empty, uint64_t *in_empty,
                                          uint32_t tmem) {
    const SBars full_s = sbars<C>(full);
    const SBars empty_s = sbars<C>(empty);
    const SBars in_empty_s = sbars<C>(in_empty);
    constexpr bool UIN = KB == K_A && C::UIN;
    constexpr int RPT = C::RPT, EW = C::EWS, TXO = C::TXO, ZD = C::ZD, DEPTH = C::template DEPTH_K<KB>;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    sm = smem_base<C>(sm);
    double *zring = sm + size_t(DEPTH) * C::Y_ELEMS + (KB == K_B ? size_t(C::AD) * C::AUX_ELEMS : 0);
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int tb = threadIdx.x - C::B_BASE;
    const bool valid = tb < C::B_ITEMS;
    const uint32_t tq_addr = tmem + (uint32_t(32 * ((threadIdx.x >> 5) & 3)) << 16);
    const int m = valid ? tb % (TXO / 2) : 0, g = valid ? tb / (TXO / 2) : 0;
    const int r0 = g * RPT;
    const int sZ = (r0 + 2) * EW + 2 * m + 2;
    const int sT = r0 * TXO + 2 * m;
    PRK_CHECK(sZ - 2 * EW - 2 >= 0 && sZ + (RPT + 1) * EW + 4 <= C::Z_ELEMS);
    PRK_CHECK(sT >= 0 && sT + (RPT - 1) * TXO + 2 <= C::T_ELEMS);
    const double *yring = sm;
    const int sU = (r0 + C::HY) * C::IWS + 2 * m + C::HX;  // tile point in an input slot

    Weights W;
    if constexpr (C::WP) {
        W.load(a.wB);
    } else {
        const long long row = (*a.nu_pos + a.j_local) * 4;
        W.set(a.nu_tab[row + (KB == K_A ? 1 : 3)], a.inv_dx, a.c);
    }
    const double dt = a.dt;

    RingP<ZD> zq_pos;     // Z plane j of the current item
    RingP<DEPTH> in_pos;  // UIN: input element j of the current item
    [[maybe_unused]] uint32_t full_ok = 0;  // SW: Z plane j already probed complete
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;
        // OFF32: one 32-bit element offset for both outputs (n^3 < 2^32), each store address a
        // single IMAD.WIDE off the kernel-parameter base instead of 64-bit pointer pairs
        [[maybe_unused]] uint32_t off = uint32_t(w.z_begin) * uint32_t(nn) + uint32_t(w.y0 + r0) * uint32_t(n) +
                                        uint32_t(w.x0 + 2 * m);
        double *o0 = a.o0 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * m;
        double *o1 = KB == K_A ? a.o1 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * m
                               : nullptr;
        double2 q[RPT][5];
        RingP<ZD> zc_pos = zq_pos;  // Z plane j-2 (valid from j = 2)
        rotating_loop(NJ, [&](auto ph, int j) {
            constexpr int P = decltype(ph)::value;
            [[maybe_unused]] double2 accv[KB == K_B && C::ACCG ? RPT : 1];
            if constexpr (KB == K_B && C::ACCG) {  // acc of this iteration's output points (j >= 4)
                if (j >= 4 && valid) {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) accv[r] = *reinterpret_cast<const double2 *>(o0 + size_t(r) * n);
                }
            }
            if (C::DIAG != 2 && !(C::SW && full_ok)) mbar_wait(full_s[zq_pos.slot()], zq_pos.round() & 1);
            TmRaw8 tt0, tt1;  // TM: t0 and u of the output point (plane j-2)
            if constexpr (C::TM) {
                tm_fence_after();
                TmRaw8 tz;
                tm_ld8(tq_addr + uint32_t(zq_pos.slot() * C::TM_PLANE), tz);  // own centre, plane j
                if (C::TM == 3 && j >= 4) {  // TM 3: plane j-2's per-point values in the same wait
                    const uint32_t cc = tq_addr + uint32_t(zc_pos.slot() * C::TM_PLANE);
                    tm_ld8(cc + 8, tt0);
                    if (KB == K_A) tm_ld8(cc + 16, tt1);
                }
                tm_wait_ld();
#pragma unroll
                for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = tm_row(tz, r);
            } else {
                const double *zq = zring + size_t(zq_pos.slot()) * ZS + sZ;
#pragma unroll
                for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = lds2(zq + r * EW);
            }
            if constexpr (C::SW) {  // probe plane j+1 (possibly the next item's first plane)
                const RingP<ZD> zn = zq_pos.at(1);
                full_ok = mbar_test(full_s[zn.slot()], zn.round() & 1);
            }
            if (j >= 4 && valid) {
                const double *zs = zring + size_t(zc_pos.slot()) * ZS;
                const double *zc = zs + sZ;
                double2 col[RPT + 4];
#pragma unroll
                for (int r = 0; r < RPT + 4; ++r)
                    col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : lds2(zc + (r - 2) * EW);
                double2 kBs[RPT];
#pragma unroll
                for (int r = 0; r < RPT; ++r)
                    kBs[r] = apply_pair<P>(W, lds2(zc + r * EW - 2), lds2(zc + r * EW + 2), col[r], col[r + 1],
                                           col[r + 3], col[r + 4], q[r]);
                if constexpr (C::TM == 1 || C::TM == 2) {
                    const uint32_t cc = tq_addr + uint32_t(zc_pos.slot() * C::TM_PLANE);
                    tm_ld8(cc + 8, tt0);
                    if (KB == K_A) tm_ld8(cc + 16, tt1);
                    tm_wait_ld();
                }
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double2 kB = kBs[r];
                    const size_t gofs = size_t(r) * n;
                    if (KB == K_A) {
                        const double2 t0 = C::TM ? tm_row(tt0, r) : lds2(zs + C::Z_ELEMS + sT + r * TXO);
                        // u at the output point: input element j (plane z_begin + j - 4)
                        const double2 t1 =
                            C::TM ? tm_row(tt1, r)
                            : UIN ? lds2(yring + size_t(in_pos.slot()) * C::Y_ELEMS + sU + r * C::IWS)
                                  : lds2(zs + C::Z_ELEMS + C::T_ELEMS + sT + r * TXO);
                        double2 v0, v1;
                        v0.x = t0.x + (dt / 3.0) * kB.x;  v0.y = t0.y + (dt / 3.0) * kB.y;
                        v1.x = t1.x + (dt / 2.0) * kB.x;  v1.y = t1.y + (dt / 2.0) * kB.y;
                        if constexpr (C::OFF32) {
                            const uint32_t e = off + uint32_t(r) * uint32_t(n);
                            *reinterpret_cast<double2 *>(a.o0 + e) = v0;
                            *reinterpret_cast<double2 *>(a.o1 + e) = v1;
                        } else {
                            *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                            *reinterpret_cast<double2 *>(o1 + gofs) = v1;
                        }
                    } else {
                        double2 t0 = C::TM ? tm_row(tt0, r) : lds2(zs + C::Z_ELEMS + sT + r * TXO);
                        if constexpr (KB == K_B && C::ACCG) {  // t0 = acc + dt/3 k3, as stage A would
                            const double2 k3 = t0;
                            t0.x = accv[r].x + (dt / 3.0) * k3.x;
                            t0.y = accv[r].y + (dt / 3.0) * k3.y;
                        }
                        double2 v0;
                        v0.x = t0.x + (dt / 6.0) * kB.x;  v0.y = t0.y + (dt / 6.0) * kB.y;
                        if constexpr (C::OFF32) {
                            *reinterpret_cast<double2 *>(a.o0 + (off + uint32_t(r) * uint32_t(n))) = v0;
                        } else {
                            *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                        }
                    }
                }
            }
            if (j >= 4) {
                if constexpr (C::OFF32) {
                    off += uint32_t(nn);
                } else {
                    o0 += nn;
                    if (KB == K_A) o1 += nn;
                }
            }
            if (j >= 2) {
                if constexpr (C::TM) tm_fence_before();
                mbar_arrive(empty_s[zc_pos.slot()]);
                zc_pos.step();
            }
            zq_pos.step();
            if constexpr (UIN) {  // input element j: read above (j >= 4) or never (j < 4)
                mbar_arrive(in_empty_s[in_pos.slot()]);
                in_pos.step();
            }
        });
        // release the item's last two Z planes (never a centre)
        mbar_arrive(empty_s[zc_pos.slot()]);
        zc_pos.step();
        mbar_arrive(empty_s[zc_pos.slot()]);
        if constexpr (UIN) {  // input elements nz+4 .. nz+7 (z halo only)
#pragma unroll 1
            for (int e = 0; e < 4; ++e) {
                mbar_arrive(in_empty_s[in_pos.slot()]);
                in_pos.step();
            }
        }
    }
}

// ---------------------------------------------------------------------------
// G (one forward-Euler step, Alg.2) in the same persistent,
// warp-specialised form: producer warps stream input planes with a (2, 1, 1)
// halo (TMA tensor copies for tiles away from the seams, cp.async otherwise)
// into a DEPTH-slot ring; consumer lanes own two adjacent x points and RPT
// rows, keep z neighbours in a 3-deep register queue and write
// u' = u + Dt L_G(u) straight to HBM.  Same per-point operation order as
// stencil_kernel<K_COARSE> (bitwise identical results).
template <int TYO_, int DEPTH_, int RPT_, int PW_, int FILL_>
struct CoarseCfgP {
    static constexpr int DIAG = 0;
    static constexpr bool PIN = false;
    static constexpr bool ACCG = false;
    static constexpr int PFL2 = 0;
    static constexpr int TXO = 32, TYO = TYO_, DEPTH = DEPTH_, RPT = RPT_, PW = PW_, FILL = FILL_;
    static constexpr int HX = 2, HY = 1, HZ = 1;  // radius-1 stencil; x halo pair-aligned
    static constexpr int IW = TXO + 2 * HX, IH = TYO + 2 * HY, IWS = IW;
    static constexpr int Y_ELEMS = (IH * IWS + 15) / 16 * 16;  // 128-byte aligned slots (TMA)
    static constexpr int Y_CHUNKS = IH * (IW / 2);
    static constexpr int GC = TYO / RPT, C_ITEMS = (TXO / 2) * GC;
    static constexpr int NTA = (C_ITEMS + 31) / 32 * 32, NTB = 0, NTP = 32 * PW, NT = NTA + NTP;
    static constexpr int MAXR = (65536 / NT) / 8 * 8 > 255 ? 255 : (65536 / NT) / 8 * 8;
    // unused by the K_A producer path (aux planes belong to the RK4 K_B kernel)
    static constexpr int EW = IW, EH = IH, EWS = IWS, Z_ELEMS = 0, T_ELEMS = 0, AUX_ELEMS = 0,
                         U_CHUNKS = 0, C_CHUNKS = 0, AD = 0, ZD = 1, RPTA = RPT;
    static_assert(TYO % RPT == 0 && C_ITEMS % 32 == 0, "full consumer warps");
    template <int KB> static constexpr int DEPTH_K = DEPTH;
    static size_t smem_bytes() { return sizeof(double) * size_t(DEPTH) * Y_ELEMS; }
};
using CoarseP0 = CoarseCfgP<16, 8, 2, 2, 2>;   // default
#ifdef PRK_VARIANTS
using CoarseP1 = CoarseCfgP<16, 8, 1, 2, 2>;   // one row per lane (8 consumer warps)
using CoarseP2 = CoarseCfgP<16, 10, 2, 1, 2>;
#endif

template <class Body>
__device__ __forceinline__ void rotating_loop3(int NJ, Body &&body) {
    int j = 0;
#pragma unroll 1
    for (; j + 3 <= NJ; j += 3) {
        body(Ph<0>{}, j);
        body(Ph<1>{}, j + 1);
        body(Ph<2>{}, j + 2);
    }
    if (j < NJ) body(Ph<0>{}, j++);
    if (j < NJ) body(Ph<1>{}, j++);
}

template <class C>
__device__ __forceinline__ void stage_c_p(const StencilArgs &a, double *sm, int items,
                                          uint64_t *in_full, uint64_t *in_empty) {
    const SBars in_full_s = sbars<C>(in_full);
    const SBars in_empty_s = sbars<C>(in_empty);
    constexpr int RPT = C::RPT, IW = C::IWS, TXO = C::TXO, DEPTH = C::DEPTH;
    const double *yring = sm;
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int t = threadIdx.x;
    const int m = t % (TXO / 2), g = t / (TXO / 2);
    const int r0 = g * RPT;
    const int sY = (r0 + C::HY) * IW + 2 * m + C::HX;
    PRK_CHECK(sY - IW - 2 >= 0 && sY + RPT * IW + 4 <= C::Y_ELEMS);

    // folded weights of Alg.2 (same expressions as stencil_kernel<K_COARSE>)
    const double nu = a.nu_tab[*a.nu_pos + a.j_local];
    const double al = nu * a.inv_dx * a.inv_dx;
    double w0 = -6.0 * al, wm1[3], wp1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double b1 = a.c[d] * a.inv_dx;
        if (a.c[d] > 0) {
            wm1[d] = al + b1; wp1[d] = al; w0 -= b1;
        } else {
            wm1[d] = al; wp1[d] = al - b1; w0 += b1;
        }
    }
    const double dt = a.dt;

    RingP<DEPTH> base;  // input element 0 of the current item
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        double *o0 = a.o0 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * m;
        double2 q[RPT][3];
        RingP<DEPTH> p0 = base;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            mbar_wait(in_full_s[p0.slot()], p0.round() & 1);
            const double *ys = yring + size_t(p0.slot()) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][e] = lds2(ys + r * IW);
            p0.step();
        }
        mbar_arrive(in_empty_s[base.slot()]);      // element 0: queue only
        RingP<DEPTH> pc = base.at(1), pq = p0;  // elements j+1 (centre), j+2
        rotating_loop3(w.nz, [&](auto ph, int j) {
            constexpr int P = decltype(ph)::value;  // q[.][P] = z-1, [P+1] = z, [P+2] = z+1
            mbar_wait(in_full_s[pq.slot()], pq.round() & 1);
            const double *yq = yring + size_t(pq.slot()) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][(P + 2) % 3] = lds2(yq + r * IW);
            const double *ys = yring + size_t(pc.slot()) * C::Y_ELEMS + sY;
            double2 col[RPT + 2];
#pragma unroll
            for (int r = 0; r < RPT + 2; ++r)
                col[r] = (r >= 1 && r <= RPT) ? q[r - 1][(P + 1) % 3] : lds2(ys + (r - 1) * IW);
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double2 L = lds2(ys + r * IW - 2), R = lds2(ys + r * IW + 2);
                const double2 c = q[r][(P + 1) % 3], zm = q[r][P % 3], zp = q[r][(P + 2) % 3];
                double2 v;
                {
                    double ax = wm1[0] * L.y;
                    ax = fma(wp1[0], c.y, ax);
                    double ay = wm1[1] * col[r].x;
                    ay = fma(wp1[1], col[r + 2].x, ay);
                    double az = wm1[2] * zm.x;
                    az = fma(wp1[2], zp.x, az);
                    const double Lv = fma(w0, c.x, ax) + (ay + az);
                    v.x = c.x + dt * Lv;
                }
                {
                    double ax = wm1[0] * c.x;
                    ax = fma(wp1[0], R.x, ax);
                    double ay = wm1[1] * col[r].y;
                    ay = fma(wp1[1], col[r + 2].y, ay);
                    double az = wm1[2] * zm.y;
                    az = fma(wp1[2], zp.y, az);
                    const double Lv = fma(w0, c.y, ax) + (ay + az);
                    v.y = c.y + dt * Lv;
                }
                *reinterpret_cast<double2 *>(o0 + size_t(r) * n) = v;
            }
            o0 += nn;
            mbar_arrive(in_empty_s[pc.slot()]);  // the centre plane is no longer read from smem
            pc.step();
            pq.step();
        });
        mbar_arrive(in_empty_s[pc.slot()]);  // the item's last element (queue only)
        base = pc.at(1);
    }
}

template <class C>
__global__ void __maxnreg__(C::MAXR)
coarse_persist_kernel(const StencilArgs a, const __grid_constant__ TmaMaps tm) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t in_full[C::DEPTH], in_empty[C::DEPTH];
    const int items = a.tiles_x * a.tiles_y * a.chunks_z;
    if constexpr (C::FILL == 2) {
        if (smem_u32(sm) & 127) __trap();
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::DEPTH; ++s) {
            mbar_init(&in_full[s], C::NTP);
            mbar_init(&in_empty[s], C::NTA);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x < C::NTA)
        stage_c_p<C>(a, sm, items, in_full, in_empty);
    else
        producer_p<K_A, C>(a, &tm, sm, items, in_full, in_empty);
}

template <int KB, class C>
__global__ void __maxnreg__(C::MAXR)
fused_persist_kernel(const StencilArgs a, const __grid_constant__ TmaMaps tm) {
    extern __shared__ __align__(128) double sm[];
    constexpr int DEPTH = C::template DEPTH_K<KB>;
    __shared__ __align__(8) uint64_t full[C::ZD], empty[C::ZD], in_full[DEPTH], in_empty[DEPTH];
    const int items = a.tiles_x * a.tiles_y * a.chunks_z;
    if constexpr (C::FILL == 2) {
        if (smem_u32(sm) & 127) __trap();  // TMA destinations need 128-byte alignment
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::ZD; ++s) {
            mbar_init(&full[s], C::NTA);
            mbar_init(&empty[s], C::NTB);
        }
        for (int s = 0; s < DEPTH; ++s) {
            mbar_init(&in_full[s], C::NTP);
            mbar_init(&in_empty[s], C::template IN_CONSUMERS<KB>);
        }
        fence_mbar_init();
    }
    uint32_t tmem = 0;
    if constexpr (C::TM) {  // warp 0 allocates the TMEM hand-off ring
        __shared__ uint32_t tmem_base;
        if (threadIdx.x < 32) tm_alloc(&tmem_base, C::TM_COLS);
        tm_fence_before();
        __syncthreads();
        tm_fence_after();
        tmem = tmem_base;
    } else {
        __syncthreads();
    }
    // Programmatic dependent launch (PR_PDL): let the next kernel of the stream be launched
    // now (its CTAs take an SM as soon as one of ours exits), and wait here until the
    // previous kernel has completed and its writes are visible -- everything above (barrier
    // and TMEM set-up) overlaps the previous kernel's tail.  No-ops without the attribute.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tid = threadIdx.x;
    const bool is_a = C::TM ? (tid < C::NTC || (tid >= C::B_BASE + C::NTB && tid < C::NTA + C::NTB))
                            : tid < C::NTA;
    const bool is_b = tid >= C::B_BASE && tid < C::B_BASE + C::NTB;
    if (is_a)
        stage_a_p<KB, C>(a, sm, items, full, empty, in_full, in_empty, tmem);
    else if (is_b)
        stage_b_p<KB, C>(a, sm, items, full, empty, in_empty, tmem);
    else
        producer_p<KB, C>(a, &tm, sm, items, in_full, in_empty);
    if constexpr (C::TM) {
        tm_fence_before();
        __syncthreads();
        if (threadIdx.x < 32) {
            tm_fence_after();
            tm_dealloc(tmem, C::TM_COLS);
        }
    }
}

}  // namespace prk
