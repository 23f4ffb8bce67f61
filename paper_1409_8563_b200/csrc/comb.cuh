// comb.cuh — the two-kernel RK4 step (fused.cuh: K_A = stages 1+2, K_B = stages
// 3+4, 56 B/point) with the second stage of each kernel done by the SAME lanes
// that compute the first stage on the tile points.  DESIGN.md §5.
//
// In fused_persist_kernel a stage-A warp group writes the intermediate plane
// (Ya / Ya') plus the per-tile-point values stage B needs (t0 and, in K_A, u)
// into a shared ring, and a separate stage-B group reads them back: per 32x16
// tile plane that hand-off costs ~40 % of the kernel's shared-memory wavefronts,
// which bound it (ncu: L1 data pipe ~75 %, FP64 pipe ~37 %).  Here a lane owns
// the same two x points and two rows in both stages:
//   * its own intermediate values go into a register z-queue (no ring reads
//     for the stencil centre column), only the x/y neighbours come from the
//     shared intermediate ring, which every lane still writes;
//   * t0 (= u + dt/6 k1, or acc + dt/3 k3) waits three planes in registers;
//   * K_A's u at the output point is the oldest entry of the input z-queue.
// The extended ring of stage A (2 points around the tile) is computed by two
// "ring" warps that do stage A only.  Per tile plane: stage B of output plane m
// runs in iteration j = m + 5 (its intermediate planes m..m+4 are all done),
// then stage A of plane j; the intermediate ring (ZD slots) is ordered by
// mbarrier pairs (full: every compute lane wrote the plane; empty: every
// combined lane read its neighbours in it), so warps drift up to ZD-4 planes
// apart instead of running in lockstep.  Producer warps and the
// input ring are those of fused.cuh (TMA tensor fills, cp.async on seams).
// Same per-point floating-point operation sequence as the four-pass kernels:
// the results are bitwise identical.
#pragma once
#include "fused.cuh"

namespace prk {

template <int TYO_, int DEPTH_, int PW_ = 2, int FILL_ = 2, int ZD_ = 4>
struct CombCfg {
    static constexpr bool COMB = true, Z2 = false, WP = false;
    static constexpr int DIAG = 0;
    static constexpr bool PIN = true;
    static constexpr bool ACCG = false;
    static constexpr int PFL2 = 0;
    static constexpr int TXO = 32, TYO = TYO_, DEPTH = DEPTH_, ZD = ZD_, PW = PW_, FILL = FILL_;
    static constexpr int RPT = 2, RPTA = 2, XP = 2;
    static constexpr int EW = TXO + 4, EH = TYO + 4, IW = TXO + 8, IH = TYO + 8;
    static constexpr int HX = 4, HY = 4, HZ = 4;
    static constexpr int IWS = IW + 2, EWS = EW + 6;  // padded pitches (fused.cuh)
    static constexpr int GT = TYO / RPT;                       // row groups of the tile
    static constexpr int C_LANES = (TXO / 2) * GT;             // combined lanes (tile)
    static constexpr int R_LANES = (EW / 2) * (EH / RPT) - C_LANES;  // ring lanes (stage A only)
    static constexpr int NTC = (C_LANES + 31) / 32 * 32, NTR = (R_LANES + 31) / 32 * 32;
    static constexpr int NTA = NTC + NTR, NTB = 0, NTP = 32 * PW, NT = NTA + NTP;
    static constexpr int MAXR = (65536 / NT) / 8 * 8 > 255 ? 255 : (65536 / NT) / 8 * 8;
    static constexpr int Y_ELEMS = IH * IWS, Z_ELEMS = (EH * EWS + 15) / 16 * 16, T_ELEMS = TYO * TXO;
    static constexpr int AUX_ELEMS = Z_ELEMS + T_ELEMS, AD = DEPTH;
    static constexpr int Y_CHUNKS = IH * (IW / 2), U_CHUNKS = EH * (EW / 2), C_CHUNKS = TYO * (TXO / 2);
    static_assert(C_LANES % 32 == 0, "combined lanes fill whole warps");
    static_assert(Y_ELEMS % 16 == 0 && Z_ELEMS % 16 == 0, "slots must stay 128-byte aligned");
    static_assert(DEPTH >= 5 && ZD >= 4, "rings too shallow");
    template <int KB> static constexpr int DEPTH_K = DEPTH;
    template <int KB> static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t(DEPTH) * Y_ELEMS + (KB == K_B ? size_t(AD) * AUX_ELEMS : 0) +
                                 size_t(ZD) * Z_ELEMS);
    }
};
using Comb16 = CombCfg<16, 9, 2, 2, 6>;  // 32x16 tile: 4 combined + 2 ring + 2 producer warps

template <int KB, class C>
__device__ __forceinline__ void comb_consumer(const StencilArgs &a, double *sm, int items,
                                              uint64_t *in_full, uint64_t *in_empty, uint64_t *zfull,
                                              uint64_t *zempty) {
    constexpr int RPT = C::RPT, DEPTH = C::DEPTH, EW = C::EWS, IW = C::IWS, TXO = C::TXO, ZD = C::ZD;
    // barrier and ring addresses pinned in registers (fused.cuh, FusedCfgP::PIN)
    const SBars zfull_s = sbars<C>(zfull), zempty_s = sbars<C>(zempty);
    const SBars in_full_s = sbars<C>(in_full), in_empty_s = sbars<C>(in_empty);
    double *yring = smem_base<C>(sm);
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    double *zring = aring + (KB == K_B ? size_t(C::AD) * C::AUX_ELEMS : 0);
    const int t = threadIdx.x;
    const int n = a.n;
    const size_t nn = size_t(n) * n;

    // lane -> (extended column pair l, extended row group g); combined lanes first
    const bool comb = t < C::NTC;
    int l = 0, g = 0;
    bool valid = true;
    if (comb) {
        l = t % (TXO / 2) + 1;
        g = t / (TXO / 2) + 1;
    } else {
        const int u = t - C::NTC;
        valid = u < C::R_LANES;
        const int top = C::EW / 2;  // lanes of extended row group 0 and of the last one
        if (!valid) {
            l = 0; g = 0;
        } else if (u < top) {
            l = u; g = 0;
        } else if (u < 2 * top) {
            l = u - top; g = C::EH / RPT - 1;
        } else {
            const int v = u - 2 * top;
            l = (v & 1) ? C::EW / 2 - 1 : 0;
            g = 1 + (v >> 1);
        }
    }
    const int r0 = g * RPT;  // first extended row of this lane
    const int sY = (r0 + 2) * IW + 2 * l + 2;   // its centre in an input slot
    const int sZ = r0 * EW + 2 * l;             // its point in an intermediate slot
    PRK_CHECK(sY - 2 * IW - 2 >= 0 && sY + (RPT + 1) * IW + 4 <= C::Y_ELEMS);
    PRK_CHECK(sZ - 2 * EW - 2 >= 0 || !comb);
    PRK_CHECK(sZ + (RPT - 1) * EW + 2 <= C::Z_ELEMS);
    const int tp0 = (r0 - 2) * TXO + 2 * l - 2;  // tile point of a combined lane (aux acc)

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights WA, WB;
    WA.set(a.nu_tab[row + (KB == K_A ? 0 : 2)], a.inv_dx, a.c);
    WB.set(a.nu_tab[row + (KB == K_A ? 1 : 3)], a.inv_dx, a.c);
    const double dt = a.dt;

    RingPos base;  // input element 0 of the current item
    RingPos zw;    // intermediate ring: position of the plane stage A writes next
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;  // >= 5
        double *o0 = a.o0 + size_t(w.z_begin) * nn + size_t(w.y0 + r0 - 2) * n + w.x0 + 2 * l - 2;
        double *o1 = KB == K_A ? a.o1 + size_t(w.z_begin) * nn + size_t(w.y0 + r0 - 2) * n + w.x0 + 2 * l - 2
                               : nullptr;
        double2 qa[RPT][5];  // input z-queue: element e at index e % 5 (e = j .. j+4 in iteration j)
        double2 qb[RPT][5];  // own intermediate values: plane p at index p % 5
        double2 tq[RPT][5];  // own t0 values: plane p at index p % 5
        RingPos p0 = base;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            mbar_wait(in_full_s[p0.slot], p0.round & 1);
            const double *ys = yring + size_t(p0.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) qa[r][e] = lds2(ys + r * IW);
            p0.step(DEPTH);
        }
        mbar_arrive(in_empty_s[base.slot]);
        mbar_arrive(in_empty_s[ring_at(base, 1, DEPTH).slot]);
        RingPos p2 = ring_at(base, 2, DEPTH), p4 = p0;  // elements j+2, j+4
        RingPos zr = zw;  // intermediate ring: plane j-3 (stage B's centre in iteration j >= 5)

        // ---- the pieces of one iteration j (phase P = j % 5)
        // stage A loads: element j+4 into the z-queue, x/y neighbours of element j+2, aux j
        struct ALd { double2 col[RPT + 4], xl[RPT], xr[RPT], ub[RPT], ac[RPT]; };
        auto a_load = [&](auto ph, ALd &L) {
            constexpr int P = decltype(ph)::value;
            const double *yq = yring + size_t(p4.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) qa[r][(P + 4) % 5] = lds2(yq + r * IW);
            const double *ys = yring + size_t(p2.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT + 4; ++r)
                L.col[r] = (r >= 2 && r < RPT + 2) ? qa[r - 2][(P + 2) % 5] : lds2(ys + (r - 2) * IW);
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                L.xl[r] = lds2(ys + r * IW - 2);
                L.xr[r] = lds2(ys + r * IW + 2);
            }
            if constexpr (KB == K_B) {
                const double *au = aring + size_t(p4.slot) * C::AUX_ELEMS;  // aux j
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    L.ub[r] = lds2(au + sZ + r * EW);
                    L.ac[r] = lds2(au + C::Z_ELEMS + (comb ? tp0 + r * TXO : 0));
                }
            }
        };
        // stage A compute (registers only)
        struct K2 { double2 k[RPT]; };
        auto a_compute = [&](auto ph, const ALd &L, K2 &K) {
            constexpr int P = decltype(ph)::value;
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                K.k[r] = apply_pair<P>(WA, L.xl[r], L.xr[r], L.col[r], L.col[r + 1], L.col[r + 3], L.col[r + 4],
                                       qa[r]);
        };
        // stage A results: the intermediate plane j (ring and own queue) and t0
        auto a_store = [&](auto ph, const ALd &L, const K2 &K) {
            constexpr int P = decltype(ph)::value;
            mbar_arrive(in_empty_s[p2.slot]);  // element j+2 done (aux j lives in slot j+4)
            if (zw.round > 0) mbar_wait(zempty_s[zw.slot], (zw.round - 1) & 1);
            double *zd = zring + size_t(zw.slot) * C::Z_ELEMS + sZ;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double2 yc = qa[r][(P + 2) % 5];
                double2 z, t0;
                if (KB == K_A) {
                    z.x = yc.x + (dt / 2.0) * K.k[r].x;
                    z.y = yc.y + (dt / 2.0) * K.k[r].y;
                    t0.x = yc.x + (dt / 6.0) * K.k[r].x;
                    t0.y = yc.y + (dt / 6.0) * K.k[r].y;
                } else {
                    z.x = L.ub[r].x + dt * K.k[r].x;
                    z.y = L.ub[r].y + dt * K.k[r].y;
                    t0.x = L.ac[r].x + (dt / 3.0) * K.k[r].x;
                    t0.y = L.ac[r].y + (dt / 3.0) * K.k[r].y;
                }
                if (valid) sts2(zd + r * EW, z);
                qb[r][P] = z;  // plane j replaces plane j-5
                tq[r][P] = t0;
            }
            mbar_arrive(zfull_s[zw.slot]);
            zw.step(ZD);
            p2.step(DEPTH);
            p4.step(DEPTH);
        };
        // stage B loads: x/y neighbours of intermediate plane j-3 (centre of output j-5)
        struct BLd { double2 col[RPT + 4], xl[RPT], xr[RPT], t1[RPT]; };
        auto b_load = [&](auto ph, BLd &L) {
            constexpr int P = decltype(ph)::value;
            const double *zp = zring + size_t(zr.slot) * C::Z_ELEMS + sZ;
#pragma unroll
            for (int r = 0; r < RPT + 4; ++r)
                L.col[r] = (r >= 2 && r < RPT + 2) ? qb[r - 2][(P + 2) % 5] : lds2(zp + (r - 2) * EW);
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                L.xl[r] = lds2(zp + r * EW - 2);
                L.xr[r] = lds2(zp + r * EW + 2);
                L.t1[r] = qa[r][(P + 4) % 5];  // u at the output point (element j-1), before a_load
            }
        };
        // stage B compute (registers only)
        auto b_compute = [&](auto ph, const BLd &L, K2 &K) {
            constexpr int P = decltype(ph)::value;
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                K.k[r] = apply_pair<P>(WB, L.xl[r], L.xr[r], L.col[r], L.col[r + 1], L.col[r + 3], L.col[r + 4],
                                       qb[r]);
        };
        // stage B results: output plane j-5 to HBM
        auto b_store = [&](auto ph, const BLd &L, const K2 &K) {
            constexpr int P = decltype(ph)::value;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double2 kB = K.k[r];
                const size_t gofs = size_t(r) * n;
                const double2 t0 = tq[r][(P + 2) % 5];
                if (KB == K_A) {
                    const double2 t1 = L.t1[r];
                    double2 v0, v1;
                    v0.x = t0.x + (dt / 3.0) * kB.x;  v0.y = t0.y + (dt / 3.0) * kB.y;
                    v1.x = t1.x + (dt / 2.0) * kB.x;  v1.y = t1.y + (dt / 2.0) * kB.y;
                    *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                    *reinterpret_cast<double2 *>(o1 + gofs) = v1;
                } else {
                    double2 v0;
                    v0.x = t0.x + (dt / 6.0) * kB.x;  v0.y = t0.y + (dt / 6.0) * kB.y;
                    *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                }
            }
            o0 += nn;
            if (KB == K_A) o1 += nn;
            mbar_arrive(zempty_s[zr.slot]);  // plane j-3 read
            zr.step(ZD);
        };
        // release a plane stage B never reads (0, 1, NJ-2, NJ-1) -- only once every lane has
        // written it: an early release could complete the slot's empty phase twice before
        // a slow writer waits on it (its parity wait would then never return)
        auto release_unread = [&]() {
            mbar_wait(zfull_s[zr.slot], zr.round & 1);
            mbar_arrive(zempty_s[zr.slot]);
            zr.step(ZD);
        };
        auto stage_a = [&](auto ph) {
            mbar_wait(in_full_s[p4.slot], p4.round & 1);  // element j+4 (+ aux j) landed
            ALd L;
            K2 K;
            a_load(ph, L);
            a_compute(ph, L, K);
            a_store(ph, L, K);
        };
        auto stage_b = [&](auto ph) {
            mbar_wait(zfull_s[zr.slot], zr.round & 1);
            BLd L;
            K2 K;
            b_load(ph, L);
            b_compute(ph, L, K);
            b_store(ph, L, K);
        };

        if (comb) {
            // j = 0 .. 4: stage A only; intermediate planes 0 and 1 are never a centre
            stage_a(Ph<0>{});
            stage_a(Ph<1>{});
            stage_a(Ph<2>{});
            release_unread();
            stage_a(Ph<3>{});
            release_unread();
            stage_a(Ph<4>{});
            // j = 5 .. NJ-1: both stages; every wait first, then both stages' loads, so the
            // two dependency chains of the iteration overlap
            rotating_loop(NJ - 5, [&](auto ph, int) {
                mbar_wait(zfull_s[zr.slot], zr.round & 1);
                mbar_wait(in_full_s[p4.slot], p4.round & 1);
                BLd LB;
                ALd LA;
                K2 KB_, KA_;
                b_load(ph, LB);
                a_load(ph, LA);
                b_compute(ph, LB, KB_);
                a_compute(ph, LA, KA_);
                b_store(ph, LB, KB_);
                a_store(ph, LA, KA_);
            });
            // j = NJ: stage B of the last output plane
            switch (NJ % 5) {
            case 0: stage_b(Ph<0>{}); break;
            case 1: stage_b(Ph<1>{}); break;
            case 2: stage_b(Ph<2>{}); break;
            case 3: stage_b(Ph<3>{}); break;
            default: stage_b(Ph<4>{}); break;
            }
            // the item's last two intermediate planes are never a centre
            release_unread();
            release_unread();
        } else {  // ring lanes: stage A on the extended ring only
            rotating_loop(NJ, [&](auto ph, int) { stage_a(ph); });
        }
        // the item's last two input elements were only used by the queue
        mbar_arrive(in_empty_s[p2.slot]);
        mbar_arrive(in_empty_s[ring_at(p2, 1, DEPTH).slot]);
        base = ring_at(p2, 2, DEPTH);
    }
}

template <int KB, class C>
__global__ void __maxnreg__(C::MAXR)
fused_comb_kernel(const StencilArgs a, const __grid_constant__ TmaMaps tm) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t in_full[C::DEPTH], in_empty[C::DEPTH], zfull[C::ZD], zempty[C::ZD];
    const int items = a.tiles_x * a.tiles_y * a.chunks_z;
    if constexpr (C::FILL == 2) {
        if (smem_u32(sm) & 127) __trap();  // TMA destinations need 128-byte alignment
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::DEPTH; ++s) {
            mbar_init(&in_full[s], C::NTP);
            mbar_init(&in_empty[s], C::NTA);
        }
        for (int s = 0; s < C::ZD; ++s) {
            mbar_init(&zfull[s], C::NTA);   // every compute thread wrote its part of the plane
            mbar_init(&zempty[s], C::NTC);  // every combined thread read its neighbours in it
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x < C::NTA)
        comb_consumer<KB, C>(a, sm, items, in_full, in_empty, zfull, zempty);
    else
        producer_p<KB, C>(a, &tm, sm, items, in_full, in_empty);
}

}  // namespace prk
