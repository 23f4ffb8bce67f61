// fused.cuh — one classical RK4 step as TWO kernels, each fusing
// two stages with an overlapped (redundantly computed) halo ring.  DESIGN.md §5.
//
//   fused_kernel<K_A>:  k1 = L(u) on the tile + 2-point ring, Ya = u + dt/2 k1 kept
//                       in shared memory; k2 = L(Ya) on the tile;
//                       acc = u + dt/6 k1 + dt/3 k2,  Yb = u + dt/2 k2.
//                       HBM: read u, write acc, Yb               (24 B/point)
//   fused_kernel<K_B>:  k3 = L(Yb) on tile + ring, Ya' = u + dt k3 in shared memory;
//                       k4 = L(Ya') on the tile;
//                       u_new = acc + dt/3 k3 + dt/6 k4  (written over acc).
//                       HBM: read Yb, u, acc, write u_new        (32 B/point)
// One RK4 step moves 56 B/point instead of 128 B/point for four stage passes,
// with exactly the same floating-point operation sequence per point as the
// four-stage kernels (the two paths agree bitwise).
//
// Geometry: output tile 32 x TYO (x, y); stage A runs on the extended region
// 36 x (TYO+4); its input is read on 40 x (TYO+8).  A CTA marches a z chunk.
// Warp specialisation:
//   * a producer warp (default variant) streams the input planes (and K_B's
//     u/acc planes) into a DEPTH-slot shared ring with 16-byte cp.async copies
//     (periodic wrap folded into a per-lane copy plan) and signals each plane
//     with cp.async.mbarrier.arrive.noinc; stage-A warps release slots through
//     an mbarrier (older variants: stage-A warps issue the copies themselves
//     and synchronise with a named barrier);
//   * stage-A warps keep z neighbours in register queues (two adjacent x points
//     and RPT consecutive rows per thread), and write each intermediate plane
//     (Ya or Ya') plus the per-tile-point data stage B needs into a ZD-slot
//     shared ring;
//   * stage-B warps consume that ring (mbarrier full/empty hand-off, so both
//     stages run concurrently, stage A up to ZD-2 planes ahead) and store the
//     outputs to HBM coalesced along x.
#pragma once
#include <type_traits>

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
// arrive on the mbarrier once all of this thread's prior cp.async copies land
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int TYO_, int DEPTH_, int ZD_, int MINB_, int RPTA_ = 4> struct FusedCfg {
    static constexpr int TXO = 32, TYO = TYO_, DEPTH = DEPTH_, ZD = ZD_, MINB = MINB_, XP = 1,
                         PROD = 0;
    static constexpr int RPT = 4, RPTA = RPTA_;        // rows per thread: stage B, stage A
    static constexpr int EW = TXO + 4, EH = TYO + 4;   // stage-A (extended) region
    static constexpr int IW = TXO + 8, IH = TYO + 8;   // input region
    // shared-memory row strides (doubles), padded so that row groups of the
    // edge-column warps fall into different banks; multiples of 2 (16 B rows)
    static constexpr int IWS = IW + 2, EWS = EW + 2;
    static constexpr int GA = EH / RPTA, GB = TYO / RPT;  // row groups
    static constexpr int EDGE_ITEMS = 4 * GA;            // ext columns 32..35
    static constexpr int EA = (EDGE_ITEMS + 31) / 32;
    static constexpr int WA = GA + EA, WB = GB;
    static constexpr int NTA = 32 * WA, NTB = 32 * WB, NT = NTA + NTB;
    static constexpr int AD = DEPTH - 2;                 // aux ring (K_B)
    static constexpr int Y_ELEMS = IH * IWS;
    static constexpr int Z_ELEMS = EH * EWS;
    static constexpr int T_ELEMS = TYO * TXO;
    static constexpr int AUX_ELEMS = Z_ELEMS + T_ELEMS;  // u on the ext region, acc on the tile
    static constexpr int Y_CHUNKS = IH * (IW / 2);
    static constexpr int U_CHUNKS = EH * (EW / 2);
    static constexpr int C_CHUNKS = TYO * (TXO / 2);
    static constexpr int NCY = (Y_CHUNKS + NTA - 1) / NTA;
    static constexpr int NCU = (U_CHUNKS + NTA - 1) / NTA;
    static constexpr int NCC = (C_CHUNKS + NTA - 1) / NTA;
    static_assert(TYO % RPT == 0 && EH % RPTA == 0, "rows must split into RPT groups");
    static_assert(DEPTH >= 6 && ZD >= 3, "rings too shallow");
    template <int KB> static constexpr int NTV = KB == K_A ? 2 : 1;
    template <int KB> static constexpr int ZS_ELEMS = Z_ELEMS + NTV<KB> * T_ELEMS;
    template <int KB> static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t(DEPTH) * Y_ELEMS + (KB == K_B ? size_t(AD) * AUX_ELEMS : 0) +
                                 size_t(ZD) * ZS_ELEMS<KB>);
    }
};
using Fused0 = FusedCfg<16, 6, 4, 1, 4>;
using Fused1 = FusedCfg<16, 6, 4, 1, 2>;   // twice the stage-A warps
using Fused2 = FusedCfg<32, 6, 3, 1, 4>;   // larger tile, less halo work

// folded 13-point operator, C3 (same order as stencil_kernel)
struct Weights {
    double wm1[3], wp1[3], wm2[3], wp2[3], w0;
    __device__ __forceinline__ void set(double nu, double inv_dx, const double *c) {
        const double al = nu * inv_dx * inv_dx / 12.0;
        w0 = -90.0 * al;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double be = c[d] * inv_dx / 12.0;
            wp2[d] = -al + be; wp1[d] = 16.0 * al - 8.0 * be;
            wm1[d] = 16.0 * al + 8.0 * be; wm2[d] = -al - be;
        }
    }
    // xr: pointer to the centre in the current plane (x neighbours at +-1, +-2);
    // ym2..yp2: y neighbours; q: z queue (q[2] = centre)
    __device__ __forceinline__ double apply(const double *xr, double ym2, double ym1, double yp1,
                                            double yp2, const double *q) const {
        double ax = wm1[0] * xr[-1];
        ax = fma(wp1[0], xr[1], ax);
        ax = fma(wm2[0], xr[-2], ax);
        ax = fma(wp2[0], xr[2], ax);
        double ay = wm1[1] * ym1;
        ay = fma(wp1[1], yp1, ay);
        ay = fma(wm2[1], ym2, ay);
        ay = fma(wp2[1], yp2, ay);
        double az = wm1[2] * q[1];
        az = fma(wp1[2], q[3], az);
        az = fma(wm2[2], q[0], az);
        az = fma(wp2[2], q[4], az);
        return fma(w0, q[2], ax) + (ay + az);
    }
    // same, z queue given as a circular buffer whose oldest entry sits at P
    template <int P>
    __device__ __forceinline__ double apply_rot(const double *xr, double ym2, double ym1, double yp1,
                                                double yp2, const double *q) const {
        double ax = wm1[0] * xr[-1];
        ax = fma(wp1[0], xr[1], ax);
        ax = fma(wm2[0], xr[-2], ax);
        ax = fma(wp2[0], xr[2], ax);
        double ay = wm1[1] * ym1;
        ay = fma(wp1[1], yp1, ay);
        ay = fma(wm2[1], ym2, ay);
        ay = fma(wp2[1], yp2, ay);
        double az = wm1[2] * q[(P + 1) % 5];
        az = fma(wp1[2], q[(P + 3) % 5], az);
        az = fma(wm2[2], q[P % 5], az);
        az = fma(wp2[2], q[(P + 4) % 5], az);
        return fma(w0, q[(P + 2) % 5], ax) + (ay + az);
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

template <int KB, class C>
__device__ __forceinline__ void stage_a_warps(const StencilArgs &a, double *sm, uint64_t *full,
                                              uint64_t *empty, int x0, int y0, int z_begin,
                                              int nz) {
    constexpr int RPT = C::RPTA, DEPTH = C::DEPTH, EW = C::EWS, IW = C::IWS, TXO = C::TXO,
                  ZD = C::ZD, AD = C::AD;
    constexpr int NTV = C::template NTV<KB>, ZS = C::template ZS_ELEMS<KB>;
    double *yring = sm;
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    double *zring = aring + (KB == K_B ? size_t(AD) * C::AUX_ELEMS : 0);
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int E = nz + 8, NJ = nz + 4;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;

    // copy plans (periodic wrap in x and y folded in), computed once
    int ysrc[C::NCY], ydst[C::NCY];
#pragma unroll
    for (int k = 0; k < C::NCY; ++k) {
        const int c = t + k * C::NTA;
        ysrc[k] = -1;
        ydst[k] = 0;
        if (c < C::Y_CHUNKS) {
            const int r = c / (C::IW / 2), cc = c % (C::IW / 2);
            ysrc[k] = wrapi(y0 - 4 + r, n) * n + wrapi(x0 - 4 + 2 * cc, n);
            ydst[k] = 8 * (r * IW + 2 * cc);  // bytes
        }
    }
    int usrc[KB == K_B ? C::NCU : 1], udst[KB == K_B ? C::NCU : 1];
    int csrc[KB == K_B ? C::NCC : 1], cdst[KB == K_B ? C::NCC : 1];
    if constexpr (KB == K_B) {
#pragma unroll
        for (int k = 0; k < C::NCU; ++k) {
            const int c = t + k * C::NTA;
            usrc[k] = -1;
            udst[k] = 0;
            if (c < C::U_CHUNKS) {
                const int r = c / (C::EW / 2), cc = c % (C::EW / 2);
                usrc[k] = wrapi(y0 - 2 + r, n) * n + wrapi(x0 - 2 + 2 * cc, n);
                udst[k] = 8 * (r * EW + 2 * cc);
            }
        }
#pragma unroll
        for (int k = 0; k < C::NCC; ++k) {
            const int c = t + k * C::NTA;
            csrc[k] = -1;
            cdst[k] = 0;
            if (c < C::C_CHUNKS) {
                const int r = c / (TXO / 2), cc = c % (TXO / 2);
                csrc[k] = (y0 + r) * n + x0 + 2 * cc;
                cdst[k] = 8 * (C::Z_ELEMS + r * TXO + 2 * cc);
            }
        }
    }
    // input element e = plane z_begin-4+e; aux j (K_B) = u on the ext region and
    // acc on the tile at stage-A plane j (physical z_begin-2+j), issued with
    // input element j+4 so both are waited for together.
    // issue state: plane of the next input element and its ring slot, and of
    // the next aux element (kept incrementally: no runtime modulo by n)
    int zin = wrapi(z_begin - 4, n), sin_ = 0, saux = 0;
    const uint32_t yring_s = smem_u32(yring), aring_s = smem_u32(aring);
    auto issue = [&](int e) {
        {
            const double *src = a.y + size_t(zin) * nn;
            const uint32_t dst = yring_s + uint32_t(sin_) * (C::Y_ELEMS * 8);
#pragma unroll
            for (int k = 0; k < C::NCY; ++k)
                if (ysrc[k] >= 0) cp_async16s(dst + ydst[k], src + ysrc[k]);
        }
        if constexpr (KB == K_B) {
            const int j = e - 4;
            if (j >= 0 && j < NJ) {
                // aux j is at physical plane z_begin-2+j = plane of input element j+2
                int zaux = zin - 2;
                if (zaux < 0) zaux += n;
                const size_t pl = size_t(zaux) * nn;
                const uint32_t dst = aring_s + uint32_t(saux) * (C::AUX_ELEMS * 8);
                saux = (saux + 1 == AD) ? 0 : saux + 1;
#pragma unroll
                for (int k = 0; k < C::NCU; ++k)
                    if (usrc[k] >= 0) cp_async16s(dst + udst[k], a.p0 + pl + usrc[k]);
                if (j >= 2 && j < nz + 2) {
#pragma unroll
                    for (int k = 0; k < C::NCC; ++k)
                        if (csrc[k] >= 0) cp_async16s(dst + cdst[k], a.p1 + pl + csrc[k]);
                }
            }
        }
        zin = (zin + 1 == n) ? 0 : zin + 1;
        sin_ = (sin_ + 1 == DEPTH) ? 0 : sin_ + 1;
    };
#pragma unroll 1
    for (int e = 0; e < DEPTH; ++e) {
        if (e < E) issue(e);
        cp_async_commit();
    }
    int e_next = DEPTH;

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights W;
    W.set(a.nu_tab[row + (KB == K_A ? 0 : 2)], a.inv_dx, a.c);
    const double dt = a.dt;

    // item: main warps own ext columns 0..31 of row group `warp`; edge warps own
    // ext columns 32..35 of row group idx/4.
    bool valid = true;
    int c, g;
    if (warp < C::GA) {
        c = lane;
        g = warp;
    } else {
        const int idx = (warp - C::GA) * 32 + lane;
        valid = idx < C::EDGE_ITEMS;
        c = 32 + (idx & 3);
        g = valid ? idx >> 2 : 0;
    }
    const int r0 = g * RPT;                  // first ext row
    const int sY = (r0 + 2) * IW + c + 2;    // centre of the first row in an input plane
    const int sZ = r0 * EW + c;              // same point in a Z / aux-u plane

    double q[RPT][5];
    cp_async_wait<DEPTH - 4>();
    named_bar_sync(1, C::NTA);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const double *ys = yring + size_t(e) * C::Y_ELEMS + sY;
#pragma unroll
        for (int r = 0; r < RPT; ++r) q[r][e] = ys[r * IW];
    }

    int s4 = 4 % DEPTH, s2 = 2, szs = 0, sau = 0;  // slots of elements j+4, j+2; Z slot; aux slot
    rotating_loop(NJ, [&](auto ph, int j) {
        constexpr int P = decltype(ph)::value;  // q[r][(P + o) % 5] = plane j-2+o ... (z-2 .. z+2)
        if (j + 4 >= DEPTH + 2) cp_async_wait<DEPTH - 4>();
        else cp_async_wait<DEPTH - 5>();
        named_bar_sync(1, C::NTA);  // element j+4 (+ aux j) visible; slots of j-1 released
        while (e_next < E && e_next - DEPTH <= j + 1) issue(e_next++);
        cp_async_commit();

        const double *yq = yring + size_t(s4) * C::Y_ELEMS + sY;
#pragma unroll
        for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = yq[r * IW];
        const double *ys = yring + size_t(s2) * C::Y_ELEMS + sY;
        double col[RPT + 4];
#pragma unroll
        for (int r = 0; r < RPT + 4; ++r)
            col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : ys[(r - 2) * IW];
        double k[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r)
            k[r] = W.template apply_rot<P>(ys + r * IW, col[r], col[r + 1], col[r + 3], col[r + 4], q[r]);

        const int zslot = szs;
        if (j >= ZD) mbar_wait(&empty[zslot], ((j / ZD) & 1) ^ 1);
        double *zs = zring + size_t(zslot) * ZS;
        const double *au = aring + size_t(sau) * C::AUX_ELEMS;
        const bool outp = j >= 2 && j < nz + 2;
        if (valid) {
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double yc = q[r][(P + 2) % 5];
                if (KB == K_A) zs[sZ + r * EW] = yc + (dt / 2.0) * k[r];            // Ya
                else zs[sZ + r * EW] = au[sZ + r * EW] + dt * k[r];                  // Ya'
                const int er = r0 + r;
                if (outp && c >= 2 && c < TXO + 2 && er >= 2 && er < C::TYO + 2) {
                    const int tp = (er - 2) * TXO + (c - 2);
                    if (KB == K_A) {
                        zs[C::Z_ELEMS + tp] = yc + (dt / 6.0) * k[r];               // u + dt/6 k1
                        zs[C::Z_ELEMS + C::T_ELEMS + tp] = yc;                       // u
                    } else {
                        zs[C::Z_ELEMS + tp] = au[C::Z_ELEMS + tp] + (dt / 3.0) * k[r];  // acc + dt/3 k3
                    }
                }
            }
        }
        mbar_arrive(&full[zslot]);
        s4 = (s4 + 1 == DEPTH) ? 0 : s4 + 1;
        s2 = (s2 + 1 == DEPTH) ? 0 : s2 + 1;
        szs = (szs + 1 == ZD) ? 0 : szs + 1;
        sau = (sau + 1 == AD) ? 0 : sau + 1;
    });
    cp_async_wait<0>();
    (void)NTV;
}

template <int KB, class C>
__device__ __forceinline__ void stage_b_warps(const StencilArgs &a, double *sm, uint64_t *full,
                                              uint64_t *empty, int x0, int y0, int z_begin,
                                              int nz) {
    constexpr int RPT = C::RPT, EW = C::EWS, TXO = C::TXO, ZD = C::ZD, DEPTH = C::DEPTH,
                  AD = C::AD;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    double *zring = sm + size_t(DEPTH) * C::Y_ELEMS + (KB == K_B ? size_t(AD) * C::AUX_ELEMS : 0);
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int NJ = nz + 4;
    const int tb = threadIdx.x - C::NTA;
    const int c = tb % 32, g = tb / 32;
    const int r0 = g * RPT;                       // first tile row
    const int sZ = (r0 + 2) * EW + c + 2;         // centre of the first row in a Z plane
    const int sT = r0 * TXO + c;

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights W;
    W.set(a.nu_tab[row + (KB == K_A ? 1 : 3)], a.inv_dx, a.c);
    const double dt = a.dt;
    double *o0 = a.o0 + size_t(z_begin) * nn + size_t(y0 + r0) * n + x0 + c;
    double *o1 = KB == K_A ? a.o1 + size_t(z_begin) * nn + size_t(y0 + r0) * n + x0 + c : nullptr;

    double q[RPT][5];
    int szs = 0, szc = ZD - 2;  // Z slots of planes j and j-2
    rotating_loop(NJ, [&](auto ph, int j) {
        constexpr int P = decltype(ph)::value;  // q[r][(P + o) % 5] = Z plane j-4+o
        const int zslot = szs;
        mbar_wait(&full[zslot], (j / ZD) & 1);
        const double *zq = zring + size_t(zslot) * ZS + sZ;
#pragma unroll
        for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = zq[r * EW];
        if (j >= 4) {  // output plane j-4, centred on Z plane j-2
            const double *zs = zring + size_t(szc) * ZS;
            const double *zc = zs + sZ;
            double col[RPT + 4];
#pragma unroll
            for (int r = 0; r < RPT + 4; ++r)
                col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : zc[(r - 2) * EW];
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double kB = W.template apply_rot<P>(zc + r * EW, col[r], col[r + 1], col[r + 3],
                                                          col[r + 4], q[r]);
                const size_t gofs = size_t(r) * n;
                if (KB == K_A) {
                    o0[gofs] = zs[C::Z_ELEMS + sT + r * TXO] + (dt / 3.0) * kB;                 // acc
                    o1[gofs] = zs[C::Z_ELEMS + C::T_ELEMS + sT + r * TXO] + (dt / 2.0) * kB;    // Yb
                } else {
                    o0[gofs] = zs[C::Z_ELEMS + sT + r * TXO] + (dt / 6.0) * kB;                 // u_new
                }
            }
            o0 += nn;
            if (KB == K_A) o1 += nn;
        }
        if (j >= 2) mbar_arrive(&empty[szc]);
        szs = (szs + 1 == ZD) ? 0 : szs + 1;
        szc = (szc + 1 == ZD) ? 0 : szc + 1;
    });
}


// ---------------------------------------------------------------------------
// x-pair variant: every lane owns two adjacent x points (16-byte shared loads
// and stores).  The 36 extended columns are exactly 18 lane pairs, so there are
// no edge warps; the floating-point sequence per point is unchanged.
template <int TYO_, int DEPTH_, int ZD_, int MINB_, int RPTA_, int RPTB_, int PROD_ = 0>
struct FusedCfgX {
    static constexpr int TXO = 32, TYO = TYO_, DEPTH = DEPTH_, ZD = ZD_, MINB = MINB_, XP = 2;
    static constexpr int RPTA = RPTA_, RPT = RPTB_;
    // PROD = 1: a dedicated producer warp streams every input/aux plane
    // (cp.async + cp.async.mbarrier.arrive.noinc); stage-A warps only compute
    static constexpr int PROD = PROD_;
    static constexpr int EW = TXO + 4, EH = TYO + 4, IW = TXO + 8, IH = TYO + 8;
    static constexpr int IWS = IW + 2, EWS = EW + 2;   // even strides: pairs stay 16-byte aligned
    static constexpr int GA = EH / RPTA, GB = TYO / RPT;
    static constexpr int A_ITEMS = (EW / 2) * GA, B_ITEMS = (TXO / 2) * GB;
    static constexpr int WA = (A_ITEMS + 31) / 32, WB = (B_ITEMS + 31) / 32;
    static constexpr int NTA = 32 * WA, NTB = 32 * WB, NTP = PROD ? 32 : 0, NT = NTA + NTB + NTP;
    static constexpr int AD = DEPTH - 2;
    static constexpr int Y_ELEMS = IH * IWS, Z_ELEMS = EH * EWS, T_ELEMS = TYO * TXO;
    static constexpr int AUX_ELEMS = Z_ELEMS + T_ELEMS;
    static constexpr int Y_CHUNKS = IH * (IW / 2), U_CHUNKS = EH * (EW / 2), C_CHUNKS = TYO * (TXO / 2);
    static constexpr int NCY = (Y_CHUNKS + NTA - 1) / NTA;
    static constexpr int NCU = (U_CHUNKS + NTA - 1) / NTA;
    static constexpr int NCC = (C_CHUNKS + NTA - 1) / NTA;
    static_assert(TYO % RPT == 0 && EH % RPTA == 0, "rows must split into row groups");
    static_assert(DEPTH >= 5 && ZD >= 3, "rings too shallow");
    template <int KB> static constexpr int NTV = KB == K_A ? 2 : 1;
    template <int KB> static constexpr int ZS_ELEMS = Z_ELEMS + NTV<KB> * T_ELEMS;
    template <int KB> static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t(DEPTH) * Y_ELEMS + (KB == K_B ? size_t(AD) * AUX_ELEMS : 0) +
                                 size_t(ZD) * ZS_ELEMS<KB>);
    }
};
using Fused3 = FusedCfgX<16, 6, 4, 1, 2, 2>;
using Fused4 = FusedCfgX<16, 6, 4, 1, 4, 4>;
using Fused5 = FusedCfgX<32, 5, 3, 1, 4, 4>;
using Fused6 = FusedCfgX<16, 6, 4, 1, 1, 2>;   // 12 stage-A warps : 4 stage-B warps
using Fused7 = FusedCfgX<32, 6, 3, 1, 2, 4>;   // 32-row tile, 11 : 4
using Fused8 = FusedCfgX<16, 6, 4, 1, 2, 2, 1>;   // Fused3 + producer warp
using Fused9 = FusedCfgX<16, 7, 4, 1, 2, 2, 1>;   // same, deeper input ring

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void sts2(double *p, double2 v) { *reinterpret_cast<double2 *>(p) = v; }

// the folded operator on explicit neighbours, same operation order as Weights::apply
__device__ __forceinline__ double apply13(const Weights &W, double c, double xm2, double xm1,
                                          double xp1, double xp2, double ym2, double ym1,
                                          double yp1, double yp2, double zm2, double zm1,
                                          double zp1, double zp2) {
    double ax = W.wm1[0] * xm1;
    ax = fma(W.wp1[0], xp1, ax);
    ax = fma(W.wm2[0], xm2, ax);
    ax = fma(W.wp2[0], xp2, ax);
    double ay = W.wm1[1] * ym1;
    ay = fma(W.wp1[1], yp1, ay);
    ay = fma(W.wm2[1], ym2, ay);
    ay = fma(W.wp2[1], yp2, ay);
    double az = W.wm1[2] * zm1;
    az = fma(W.wp1[2], zp1, az);
    az = fma(W.wm2[2], zm2, az);
    az = fma(W.wp2[2], zp2, az);
    return fma(W.w0, c, ax) + (ay + az);
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

template <int KB, class C>
__device__ __forceinline__ void stage_a_xp(const StencilArgs &a, double *sm, uint64_t *full,
                                           uint64_t *empty, int x0, int y0, int z_begin, int nz,
                                           uint64_t *in_full, uint64_t *in_empty) {
    constexpr int RPT = C::RPTA, DEPTH = C::DEPTH, EW = C::EWS, IW = C::IWS, TXO = C::TXO,
                  ZD = C::ZD, AD = C::AD;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    double *yring = sm;
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    double *zring = aring + (KB == K_B ? size_t(AD) * C::AUX_ELEMS : 0);
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int E = nz + 8, NJ = nz + 4;
    const int t = threadIdx.x;

    constexpr bool PROD = C::PROD != 0;
    int ysrc[PROD ? 1 : C::NCY], ydst[PROD ? 1 : C::NCY];
    if constexpr (!PROD) {
#pragma unroll
    for (int k = 0; k < C::NCY; ++k) {
        const int c = t + k * C::NTA;
        ysrc[k] = -1;
        ydst[k] = 0;
        if (c < C::Y_CHUNKS) {
            const int r = c / (C::IW / 2), cc = c % (C::IW / 2);
            ysrc[k] = wrapi(y0 - 4 + r, n) * n + wrapi(x0 - 4 + 2 * cc, n);
            ydst[k] = 8 * (r * IW + 2 * cc);
        }
    }
    }
    int usrc[KB == K_B && !PROD ? C::NCU : 1], udst[KB == K_B && !PROD ? C::NCU : 1];
    int csrc[KB == K_B && !PROD ? C::NCC : 1], cdst[KB == K_B && !PROD ? C::NCC : 1];
    if constexpr (KB == K_B && !PROD) {
#pragma unroll
        for (int k = 0; k < C::NCU; ++k) {
            const int c = t + k * C::NTA;
            usrc[k] = -1;
            udst[k] = 0;
            if (c < C::U_CHUNKS) {
                const int r = c / (C::EW / 2), cc = c % (C::EW / 2);
                usrc[k] = wrapi(y0 - 2 + r, n) * n + wrapi(x0 - 2 + 2 * cc, n);
                udst[k] = 8 * (r * EW + 2 * cc);
            }
        }
#pragma unroll
        for (int k = 0; k < C::NCC; ++k) {
            const int c = t + k * C::NTA;
            csrc[k] = -1;
            cdst[k] = 0;
            if (c < C::C_CHUNKS) {
                const int r = c / (TXO / 2), cc = c % (TXO / 2);
                csrc[k] = (y0 + r) * n + x0 + 2 * cc;
                cdst[k] = 8 * (C::Z_ELEMS + r * TXO + 2 * cc);
            }
        }
    }
    int zin = wrapi(z_begin - 4, n), sin_ = 0, saux = 0;
    const uint32_t yring_s = smem_u32(yring), aring_s = smem_u32(aring);
    auto issue = [&](int e) {
        if constexpr (!PROD) {
            const double *src = a.y + size_t(zin) * nn;
            const uint32_t dst = yring_s + uint32_t(sin_) * (C::Y_ELEMS * 8);
#pragma unroll
            for (int k = 0; k < C::NCY; ++k)
                if (ysrc[k] >= 0) cp_async16s(dst + ydst[k], src + ysrc[k]);
        }
        if constexpr (KB == K_B && !PROD) {
            const int j = e - 4;
            if (j >= 0 && j < NJ) {
                int zaux = zin - 2;
                if (zaux < 0) zaux += n;
                const size_t pl = size_t(zaux) * nn;
                const uint32_t dst = aring_s + uint32_t(saux) * (C::AUX_ELEMS * 8);
                saux = (saux + 1 == AD) ? 0 : saux + 1;
#pragma unroll
                for (int k = 0; k < C::NCU; ++k)
                    if (usrc[k] >= 0) cp_async16s(dst + udst[k], a.p0 + pl + usrc[k]);
                if (j >= 2 && j < nz + 2) {
#pragma unroll
                    for (int k = 0; k < C::NCC; ++k)
                        if (csrc[k] >= 0) cp_async16s(dst + cdst[k], a.p1 + pl + csrc[k]);
                }
            }
        }
        zin = (zin + 1 == n) ? 0 : zin + 1;
        sin_ = (sin_ + 1 == DEPTH) ? 0 : sin_ + 1;
    };
    int e_next = DEPTH;
    if constexpr (!PROD) {
#pragma unroll 1
        for (int e = 0; e < DEPTH; ++e) {
            if (e < E) issue(e);
            cp_async_commit();
        }
    }

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights W;
    W.set(a.nu_tab[row + (KB == K_A ? 0 : 2)], a.inv_dx, a.c);
    const double dt = a.dt;

    const bool valid = t < C::A_ITEMS;
    const int l = valid ? t % (C::EW / 2) : 0, g = valid ? t / (C::EW / 2) : 0;
    const int r0 = g * RPT;                     // first ext row
    const int sY = (r0 + 2) * IW + 2 * l + 2;   // pair start, first row, input plane
    const int sZ = r0 * EW + 2 * l;             // same points in a Z / aux-u plane
    const bool tcol = l >= 1 && l <= TXO / 2;   // both points inside the tile
    const int tp0 = (r0 - 2) * TXO + 2 * l - 2; // tile offset of row r0 (valid when inside)

    double2 q[RPT][5];
    if constexpr (PROD) {
        for (int e = 0; e < 4; ++e) mbar_wait(&in_full[e], 0);
    } else {
        cp_async_wait<DEPTH - 4>();
        named_bar_sync(1, C::NTA);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const double *ys = yring + size_t(e) * C::Y_ELEMS + sY;
#pragma unroll
        for (int r = 0; r < RPT; ++r) q[r][e] = lds2(ys + r * IW);
    }
    if constexpr (PROD) {  // elements 0 and 1 were only needed for the queue
        mbar_arrive(&in_empty[0]);
        mbar_arrive(&in_empty[1]);
    }

    int s4 = 4 % DEPTH, s2 = 2, szs = 0, sau = 0;
    rotating_loop(NJ, [&](auto ph, int j) {
        constexpr int P = decltype(ph)::value;
        if constexpr (PROD) {
            mbar_wait(&in_full[s4], ((j + 4) / DEPTH) & 1);  // element j+4 (+ aux j) landed
        } else {
            if (j + 4 >= DEPTH + 2) cp_async_wait<DEPTH - 4>();
            else cp_async_wait<DEPTH - 5>();
            named_bar_sync(1, C::NTA);
            while (e_next < E && e_next - DEPTH <= j + 1) issue(e_next++);
            cp_async_commit();
        }

        const double *yq = yring + size_t(s4) * C::Y_ELEMS + sY;
#pragma unroll
        for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = lds2(yq + r * IW);
        const double *ys = yring + size_t(s2) * C::Y_ELEMS + sY;
        double2 col[RPT + 4];
#pragma unroll
        for (int r = 0; r < RPT + 4; ++r)
            col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : lds2(ys + (r - 2) * IW);
        double2 k[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r)
            k[r] = apply_pair<P>(W, lds2(ys + r * IW - 2), lds2(ys + r * IW + 2), col[r], col[r + 1],
                                 col[r + 3], col[r + 4], q[r]);

        const int zslot = szs;
        if (j >= ZD) mbar_wait(&empty[zslot], ((j / ZD) & 1) ^ 1);
        double *zs = zring + size_t(zslot) * ZS;
        const double *au = aring + size_t(sau) * C::AUX_ELEMS;
        const bool outp = j >= 2 && j < nz + 2;
        if (valid) {
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double2 yc = q[r][(P + 2) % 5];
                double2 z;
                if (KB == K_A) {
                    z.x = yc.x + (dt / 2.0) * k[r].x;                         // Ya
                    z.y = yc.y + (dt / 2.0) * k[r].y;
                } else {
                    const double2 ub = lds2(au + sZ + r * EW);
                    z.x = ub.x + dt * k[r].x;                                 // Ya'
                    z.y = ub.y + dt * k[r].y;
                }
                sts2(zs + sZ + r * EW, z);
                const int er = r0 + r;
                if (outp && tcol && er >= 2 && er < C::TYO + 2) {
                    const int tp = tp0 + r * TXO;
                    if (KB == K_A) {
                        double2 t0;
                        t0.x = yc.x + (dt / 6.0) * k[r].x;                    // u + dt/6 k1
                        t0.y = yc.y + (dt / 6.0) * k[r].y;
                        sts2(zs + C::Z_ELEMS + tp, t0);
                        sts2(zs + C::Z_ELEMS + C::T_ELEMS + tp, yc);          // u
                    } else {
                        const double2 ac = lds2(au + C::Z_ELEMS + tp);
                        double2 t0;
                        t0.x = ac.x + (dt / 3.0) * k[r].x;                    // acc + dt/3 k3
                        t0.y = ac.y + (dt / 3.0) * k[r].y;
                        sts2(zs + C::Z_ELEMS + tp, t0);
                    }
                }
            }
        }
        mbar_arrive(&full[zslot]);
        if constexpr (PROD) mbar_arrive(&in_empty[s2]);  // element j+2 and aux j are done
        s4 = (s4 + 1 == DEPTH) ? 0 : s4 + 1;
        s2 = (s2 + 1 == DEPTH) ? 0 : s2 + 1;
        szs = (szs + 1 == ZD) ? 0 : szs + 1;
        sau = (sau + 1 == AD) ? 0 : sau + 1;
    });
    if constexpr (!PROD) cp_async_wait<0>();
    (void)e_next;
    (void)E;
}

// Producer warp (C::PROD): streams input element e (plane z_begin-4+e) and, for
// K_B, aux element e-4 into the rings; element e may reuse its slot once the
// stage-A warps released element e-DEPTH (in_empty), and completion is signalled
// per lane with cp.async.mbarrier.arrive.noinc on in_full (32 arrivals).
template <int KB, class C>
__device__ __forceinline__ void producer_xp(const StencilArgs &a, double *sm, int x0, int y0,
                                            int z_begin, int nz, uint64_t *in_full,
                                            uint64_t *in_empty) {
    constexpr int DEPTH = C::DEPTH, EW = C::EWS, IW = C::IWS, TXO = C::TXO, AD = C::AD;
    constexpr int NY = (C::Y_CHUNKS + 31) / 32, NU = (C::U_CHUNKS + 31) / 32,
                  NC = (C::C_CHUNKS + 31) / 32;
    double *yring = sm;
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int E = nz + 8, NJ = nz + 4;
    const int lane = threadIdx.x % 32;
    int ysrc[NY], ydst[NY];
#pragma unroll
    for (int k = 0; k < NY; ++k) {
        const int c = lane + 32 * k;
        ysrc[k] = -1;
        ydst[k] = 0;
        if (c < C::Y_CHUNKS) {
            const int r = c / (C::IW / 2), cc = c % (C::IW / 2);
            ysrc[k] = wrapi(y0 - 4 + r, n) * n + wrapi(x0 - 4 + 2 * cc, n);
            ydst[k] = 8 * (r * IW + 2 * cc);
        }
    }
    int usrc[KB == K_B ? NU : 1], udst[KB == K_B ? NU : 1];
    int csrc[KB == K_B ? NC : 1], cdst[KB == K_B ? NC : 1];
    if constexpr (KB == K_B) {
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            const int c = lane + 32 * k;
            usrc[k] = -1;
            udst[k] = 0;
            if (c < C::U_CHUNKS) {
                const int r = c / (C::EW / 2), cc = c % (C::EW / 2);
                usrc[k] = wrapi(y0 - 2 + r, n) * n + wrapi(x0 - 2 + 2 * cc, n);
                udst[k] = 8 * (r * EW + 2 * cc);
            }
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const int c = lane + 32 * k;
            csrc[k] = -1;
            cdst[k] = 0;
            if (c < C::C_CHUNKS) {
                const int r = c / (TXO / 2), cc = c % (TXO / 2);
                csrc[k] = (y0 + r) * n + x0 + 2 * cc;
                cdst[k] = 8 * (C::Z_ELEMS + r * TXO + 2 * cc);
            }
        }
    }
    const uint32_t yring_s = smem_u32(yring), aring_s = smem_u32(aring);
    int zin = wrapi(z_begin - 4, n), sin_ = 0, saux = 0;
#pragma unroll 1
    for (int e = 0; e < E; ++e) {
        if (e >= DEPTH) mbar_wait(&in_empty[sin_], ((e / DEPTH) - 1) & 1);
        {
            const double *src = a.y + size_t(zin) * nn;
            const uint32_t dst = yring_s + uint32_t(sin_) * (C::Y_ELEMS * 8);
#pragma unroll
            for (int k = 0; k < NY; ++k)
                if (ysrc[k] >= 0) cp_async16s(dst + ydst[k], src + ysrc[k]);
        }
        if constexpr (KB == K_B) {
            const int j = e - 4;
            if (j >= 0 && j < NJ) {
                int zaux = zin - 2;
                if (zaux < 0) zaux += n;
                const size_t pl = size_t(zaux) * nn;
                const uint32_t dst = aring_s + uint32_t(saux) * (C::AUX_ELEMS * 8);
                saux = (saux + 1 == AD) ? 0 : saux + 1;
#pragma unroll
                for (int k = 0; k < NU; ++k)
                    if (usrc[k] >= 0) cp_async16s(dst + udst[k], a.p0 + pl + usrc[k]);
                if (j >= 2 && j < nz + 2) {
#pragma unroll
                    for (int k = 0; k < NC; ++k)
                        if (csrc[k] >= 0) cp_async16s(dst + cdst[k], a.p1 + pl + csrc[k]);
                }
            }
        }
        cp_async_mbar_arrive(&in_full[sin_]);
        zin = (zin + 1 == n) ? 0 : zin + 1;
        sin_ = (sin_ + 1 == DEPTH) ? 0 : sin_ + 1;
    }
    cp_async_wait<0>();
}

template <int KB, class C>
__device__ __forceinline__ void stage_b_xp(const StencilArgs &a, double *sm, uint64_t *full,
                                           uint64_t *empty, int x0, int y0, int z_begin, int nz) {
    constexpr int RPT = C::RPT, EW = C::EWS, TXO = C::TXO, ZD = C::ZD, DEPTH = C::DEPTH,
                  AD = C::AD;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    double *zring = sm + size_t(DEPTH) * C::Y_ELEMS + (KB == K_B ? size_t(AD) * C::AUX_ELEMS : 0);
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int NJ = nz + 4;
    const int tb = threadIdx.x - C::NTA;
    const bool valid = tb < C::B_ITEMS;
    const int m = valid ? tb % (TXO / 2) : 0, g = valid ? tb / (TXO / 2) : 0;
    const int r0 = g * RPT;                        // first tile row
    const int sZ = (r0 + 2) * EW + 2 * m + 2;      // pair start, first row, Z plane
    const int sT = r0 * TXO + 2 * m;

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights W;
    W.set(a.nu_tab[row + (KB == K_A ? 1 : 3)], a.inv_dx, a.c);
    const double dt = a.dt;
    double *o0 = a.o0 + size_t(z_begin) * nn + size_t(y0 + r0) * n + x0 + 2 * m;
    double *o1 = KB == K_A ? a.o1 + size_t(z_begin) * nn + size_t(y0 + r0) * n + x0 + 2 * m : nullptr;

    double2 q[RPT][5];
    int szs = 0, szc = ZD - 2;
    rotating_loop(NJ, [&](auto ph, int j) {
        constexpr int P = decltype(ph)::value;
        const int zslot = szs;
        mbar_wait(&full[zslot], (j / ZD) & 1);
        const double *zq = zring + size_t(zslot) * ZS + sZ;
#pragma unroll
        for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = lds2(zq + r * EW);
        if (j >= 4 && valid) {
            const double *zs = zring + size_t(szc) * ZS;
            const double *zc = zs + sZ;
            double2 col[RPT + 4];
#pragma unroll
            for (int r = 0; r < RPT + 4; ++r)
                col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : lds2(zc + (r - 2) * EW);
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double2 kB = apply_pair<P>(W, lds2(zc + r * EW - 2), lds2(zc + r * EW + 2),
                                                 col[r], col[r + 1], col[r + 3], col[r + 4], q[r]);
                const size_t gofs = size_t(r) * n;
                if (KB == K_A) {
                    const double2 t0 = lds2(zs + C::Z_ELEMS + sT + r * TXO);
                    const double2 t1 = lds2(zs + C::Z_ELEMS + C::T_ELEMS + sT + r * TXO);
                    double2 v0, v1;
                    v0.x = t0.x + (dt / 3.0) * kB.x;  v0.y = t0.y + (dt / 3.0) * kB.y;   // acc
                    v1.x = t1.x + (dt / 2.0) * kB.x;  v1.y = t1.y + (dt / 2.0) * kB.y;   // Yb
                    *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                    *reinterpret_cast<double2 *>(o1 + gofs) = v1;
                } else {
                    const double2 t0 = lds2(zs + C::Z_ELEMS + sT + r * TXO);
                    double2 v0;
                    v0.x = t0.x + (dt / 6.0) * kB.x;  v0.y = t0.y + (dt / 6.0) * kB.y;   // u_new
                    *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                }
            }
        }
        if (j >= 4) {
            o0 += nn;
            if (KB == K_A) o1 += nn;
        }
        if (j >= 2) mbar_arrive(&empty[szc]);
        szs = (szs + 1 == ZD) ? 0 : szs + 1;
        szc = (szc + 1 == ZD) ? 0 : szc + 1;
    });
}

template <int KB, class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
fused_kernel(const StencilArgs a) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t full[C::ZD], empty[C::ZD];
    constexpr int NIN = (C::XP == 2 && C::PROD) ? C::DEPTH : 1;
    __shared__ __align__(8) uint64_t in_full[NIN], in_empty[NIN];
    int b = blockIdx.x;
    const int tix = b % a.tiles_x; b /= a.tiles_x;
    const int tiy = b % a.tiles_y; b /= a.tiles_y;
    const int x0 = tix * C::TXO, y0 = tiy * C::TYO;
    const int z_begin = b * a.cz;
    const int nz = min(a.cz, a.n - z_begin);
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::ZD; ++s) {
            mbar_init(&full[s], C::NTA);
            mbar_init(&empty[s], C::NTB);
        }
        if constexpr (C::XP == 2 && C::PROD) {
            for (int s = 0; s < C::DEPTH; ++s) {
                mbar_init(&in_full[s], 32);
                mbar_init(&in_empty[s], C::NTA);
            }
        }
        fence_mbar_init();
    }
    __syncthreads();
    if constexpr (C::XP == 2) {
        if (threadIdx.x < C::NTA)
            stage_a_xp<KB, C>(a, sm, full, empty, x0, y0, z_begin, nz, in_full, in_empty);
        else if (threadIdx.x < C::NTA + C::NTB)
            stage_b_xp<KB, C>(a, sm, full, empty, x0, y0, z_begin, nz);
        else if constexpr (C::PROD)
            producer_xp<KB, C>(a, sm, x0, y0, z_begin, nz, in_full, in_empty);
    } else {
        if (threadIdx.x < C::NTA)
            stage_a_warps<KB, C>(a, sm, full, empty, x0, y0, z_begin, nz);
        else
            stage_b_warps<KB, C>(a, sm, full, empty, x0, y0, z_begin, nz);
    }
}


// ---------------------------------------------------------------------------
// Persistent variant: one CTA per SM walks work items (tile x z chunk)
// blockIdx.x, blockIdx.x + gridDim.x, ...  All ring counters run on across
// items, so the producer warp streams the next item's first planes while the
// compute warps finish the current one (no per-item pipeline fill).  Aux planes
// (K_B) share the slot index of the input element they ride with.
template <int TYO_, int DEPTH_, int ZD_, int RPTA_, int RPTB_, int PW_ = 1> struct FusedCfgP {
    static constexpr int TXO = 32, TYO = TYO_, DEPTH = DEPTH_, ZD = ZD_, MINB = 1, XP = 2,
                         PROD = 1, PW = PW_;  // PW producer warps
    static constexpr int RPTA = RPTA_, RPT = RPTB_;
    static constexpr int EW = TXO + 4, EH = TYO + 4, IW = TXO + 8, IH = TYO + 8;
    static constexpr int IWS = IW + 2, EWS = EW + 2;
    static constexpr int GA = EH / RPTA, GB = TYO / RPT;
    static constexpr int A_ITEMS = (EW / 2) * GA, B_ITEMS = (TXO / 2) * GB;
    static constexpr int WA = (A_ITEMS + 31) / 32, WB = (B_ITEMS + 31) / 32;
    static constexpr int NTA = 32 * WA, NTB = 32 * WB, NTP = 32 * PW, NT = NTA + NTB + NTP;
    static constexpr int AD = DEPTH;  // aux slots follow the input slots
    static constexpr int Y_ELEMS = IH * IWS, Z_ELEMS = EH * EWS, T_ELEMS = TYO * TXO;
    static constexpr int AUX_ELEMS = Z_ELEMS + T_ELEMS;
    static constexpr int Y_CHUNKS = IH * (IW / 2), U_CHUNKS = EH * (EW / 2), C_CHUNKS = TYO * (TXO / 2);
    static_assert(TYO % RPT == 0 && EH % RPTA == 0, "rows must split into row groups");
    static_assert(DEPTH >= 5 && ZD >= 3, "rings too shallow");
    template <int KB> static constexpr int NTV = KB == K_A ? 2 : 1;
    template <int KB> static constexpr int ZS_ELEMS = Z_ELEMS + NTV<KB> * T_ELEMS;
    template <int KB> static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t(DEPTH) * Y_ELEMS + (KB == K_B ? size_t(AD) * AUX_ELEMS : 0) +
                                 size_t(ZD) * ZS_ELEMS<KB>);
    }
};
using FusedP0 = FusedCfgP<16, 7, 4, 2, 2>;
using FusedP1 = FusedCfgP<16, 9, 4, 2, 2>;   // deeper input ring
using FusedP2 = FusedCfgP<16, 9, 6, 2, 2>;   // deeper input and intermediate rings
using FusedP3 = FusedCfgP<16, 9, 4, 2, 2, 2>;   // two producer warps (default, PR_FTILE=13)
using FusedP4 = FusedCfgP<16, 9, 4, 2, 2, 3>;   // three producer warps
using FusedP5 = FusedCfgP<16, 9, 6, 2, 2, 2>;   // two producers, 6-slot intermediate ring
using FusedP6 = FusedCfgP<16, 8, 5, 2, 2, 2>;   // two producers, 8 / 5 slots

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

template <int KB, class C>
__device__ __forceinline__ void producer_p(const StencilArgs &a, double *sm, int items,
                                           uint64_t *in_full, uint64_t *in_empty) {
    constexpr int DEPTH = C::DEPTH, EW = C::EWS, IW = C::IWS, TXO = C::TXO;
    constexpr int NP = C::NTP;
    constexpr int NY = (C::Y_CHUNKS + NP - 1) / NP, NU = (C::U_CHUNKS + NP - 1) / NP,
                  NC = (C::C_CHUNKS + NP - 1) / NP;
    double *yring = sm;
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    // 0 .. NP-1 (NTA + NTB is a multiple of 32, so the % keeps the range visible)
    const int lane = (threadIdx.x - (C::NTA + C::NTB)) % NP;
    const uint32_t yring_s = smem_u32(yring), aring_s = smem_u32(aring);
    RingPos pos;
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int E = w.nz + 8, NJ = w.nz + 4;
        int ysrc[NY], ydst[NY];
#pragma unroll
        for (int k = 0; k < NY; ++k) {
            const int c = lane + NP * k;
            ysrc[k] = -1;
            ydst[k] = 0;
            if (c < C::Y_CHUNKS) {
                const int r = c / (C::IW / 2), cc = c % (C::IW / 2);
                ysrc[k] = wrap1(w.y0 - 4 + r, n) * n + wrap1(w.x0 - 4 + 2 * cc, n);
                ydst[k] = 8 * (r * IW + 2 * cc);
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
                    const int r = c / (C::EW / 2), cc = c % (C::EW / 2);
                    usrc[k] = wrap1(w.y0 - 2 + r, n) * n + wrap1(w.x0 - 2 + 2 * cc, n);
                    udst[k] = 8 * (r * EW + 2 * cc);
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
                }
            }
        }
        int zin = wrap1(w.z_begin - 4, n);
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
            if (pos.round > 0) mbar_wait(&in_empty[pos.slot], (pos.round - 1) & 1);
            {
                const double *src = a.y + size_t(zin) * nn;
                const uint32_t dst = yring_s + uint32_t(pos.slot) * (C::Y_ELEMS * 8);
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
                    const uint32_t dst = aring_s + uint32_t(pos.slot) * (C::AUX_ELEMS * 8);
#pragma unroll
                    for (int k = 0; k < NU; ++k)
                        if (usrc[k] >= 0) cp_async16s(dst + udst[k], a.p0 + pl + usrc[k]);
                    if (j >= 2 && j < w.nz + 2) {
#pragma unroll
                        for (int k = 0; k < NC; ++k)
                            if (csrc[k] >= 0) cp_async16s(dst + cdst[k], a.p1 + pl + csrc[k]);
                    }
                }
            }
            cp_async_mbar_arrive(&in_full[pos.slot]);
            zin = (zin + 1 == n) ? 0 : zin + 1;
            pos.step(DEPTH);
        }
    }
    cp_async_wait<0>();
}

template <int KB, class C>
__device__ __forceinline__ void stage_a_p(const StencilArgs &a, double *sm, int items,
                                          uint64_t *full, uint64_t *empty, uint64_t *in_full,
                                          uint64_t *in_empty) {
    constexpr int RPT = C::RPTA, DEPTH = C::DEPTH, EW = C::EWS, IW = C::IWS, TXO = C::TXO,
                  ZD = C::ZD;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    double *yring = sm;
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    double *zring = aring + (KB == K_B ? size_t(C::AD) * C::AUX_ELEMS : 0);
    const int t = threadIdx.x;

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights W;
    W.set(a.nu_tab[row + (KB == K_A ? 0 : 2)], a.inv_dx, a.c);
    const double dt = a.dt;

    const bool valid = t < C::A_ITEMS;
    const int l = valid ? t % (C::EW / 2) : 0, g = valid ? t / (C::EW / 2) : 0;
    const int r0 = g * RPT;
    const int sY = (r0 + 2) * IW + 2 * l + 2;
    const int sZ = r0 * EW + 2 * l;
    const bool tcol = l >= 1 && l <= TXO / 2;
    const int tp0 = (r0 - 2) * TXO + 2 * l - 2;

    RingPos base, zpos;  // input element 0 of the current item; next Z plane
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;
        double2 q[RPT][5];
        RingPos p0 = base;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            mbar_wait(&in_full[p0.slot], p0.round & 1);
            const double *ys = yring + size_t(p0.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][e] = lds2(ys + r * IW);
            p0.step(DEPTH);
        }
        // elements 0 and 1 were only needed for the queue
        mbar_arrive(&in_empty[base.slot]);
        mbar_arrive(&in_empty[ring_at(base, 1, DEPTH).slot]);
        RingPos p2 = ring_at(base, 2, DEPTH), p4 = p0;  // elements j+2, j+4
        rotating_loop(NJ, [&](auto ph, int j) {
            constexpr int P = decltype(ph)::value;
            mbar_wait(&in_full[p4.slot], p4.round & 1);  // element j+4 (+ aux j) landed
            const double *yq = yring + size_t(p4.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = lds2(yq + r * IW);
            const double *ys = yring + size_t(p2.slot) * C::Y_ELEMS + sY;
            double2 col[RPT + 4];
#pragma unroll
            for (int r = 0; r < RPT + 4; ++r)
                col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : lds2(ys + (r - 2) * IW);
            double2 k[RPT];
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                k[r] = apply_pair<P>(W, lds2(ys + r * IW - 2), lds2(ys + r * IW + 2), col[r],
                                     col[r + 1], col[r + 3], col[r + 4], q[r]);
            if (zpos.round > 0) mbar_wait(&empty[zpos.slot], (zpos.round - 1) & 1);
            double *zs = zring + size_t(zpos.slot) * ZS;
            const double *au = aring + size_t(p4.slot) * C::AUX_ELEMS;  // aux j
            const bool outp = j >= 2 && j < w.nz + 2;
            if (valid) {
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double2 yc = q[r][(P + 2) % 5];
                    double2 z;
                    if (KB == K_A) {
                        z.x = yc.x + (dt / 2.0) * k[r].x;
                        z.y = yc.y + (dt / 2.0) * k[r].y;
                    } else {
                        const double2 ub = lds2(au + sZ + r * EW);
                        z.x = ub.x + dt * k[r].x;
                        z.y = ub.y + dt * k[r].y;
                    }
                    sts2(zs + sZ + r * EW, z);
                    const int er = r0 + r;
                    if (outp && tcol && er >= 2 && er < C::TYO + 2) {
                        const int tp = tp0 + r * TXO;
                        if (KB == K_A) {
                            double2 t0;
                            t0.x = yc.x + (dt / 6.0) * k[r].x;
                            t0.y = yc.y + (dt / 6.0) * k[r].y;
                            sts2(zs + C::Z_ELEMS + tp, t0);
                            sts2(zs + C::Z_ELEMS + C::T_ELEMS + tp, yc);
                        } else {
                            const double2 ac = lds2(au + C::Z_ELEMS + tp);
                            double2 t0;
                            t0.x = ac.x + (dt / 3.0) * k[r].x;
                            t0.y = ac.y + (dt / 3.0) * k[r].y;
                            sts2(zs + C::Z_ELEMS + tp, t0);
                        }
                    }
                }
            }
            mbar_arrive(&full[zpos.slot]);
            mbar_arrive(&in_empty[p2.slot]);  // element j+2 done (aux j lives in slot j+4)
            p2.step(DEPTH);
            p4.step(DEPTH);
            zpos.step(ZD);
        });
        // the item's last two input elements were only used by the queue
        mbar_arrive(&in_empty[p2.slot]);
        mbar_arrive(&in_empty[ring_at(p2, 1, DEPTH).slot]);
        base = ring_at(p2, 2, DEPTH);
    }
}

template <int KB, class C>
__device__ __forceinline__ void stage_b_p(const StencilArgs &a, double *sm, int items,
                                          uint64_t *full, uint64_t *empty) {
    constexpr int RPT = C::RPT, EW = C::EWS, TXO = C::TXO, ZD = C::ZD, DEPTH = C::DEPTH;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    double *zring = sm + size_t(DEPTH) * C::Y_ELEMS + (KB == K_B ? size_t(C::AD) * C::AUX_ELEMS : 0);
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int tb = threadIdx.x - C::NTA;
    const bool valid = tb < C::B_ITEMS;
    const int m = valid ? tb % (TXO / 2) : 0, g = valid ? tb / (TXO / 2) : 0;
    const int r0 = g * RPT;
    const int sZ = (r0 + 2) * EW + 2 * m + 2;
    const int sT = r0 * TXO + 2 * m;

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights W;
    W.set(a.nu_tab[row + (KB == K_A ? 1 : 3)], a.inv_dx, a.c);
    const double dt = a.dt;

    RingPos zq_pos;  // Z plane j of the current item
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;
        double *o0 = a.o0 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * m;
        double *o1 = KB == K_A ? a.o1 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * m
                               : nullptr;
        double2 q[RPT][5];
        RingPos zc_pos = zq_pos;  // Z plane j-2 (valid from j = 2)
        rotating_loop(NJ, [&](auto ph, int j) {
            constexpr int P = decltype(ph)::value;
            mbar_wait(&full[zq_pos.slot], zq_pos.round & 1);
            const double *zq = zring + size_t(zq_pos.slot) * ZS + sZ;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = lds2(zq + r * EW);
            if (j >= 4 && valid) {
                const double *zs = zring + size_t(zc_pos.slot) * ZS;
                const double *zc = zs + sZ;
                double2 col[RPT + 4];
#pragma unroll
                for (int r = 0; r < RPT + 4; ++r)
                    col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : lds2(zc + (r - 2) * EW);
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double2 kB = apply_pair<P>(W, lds2(zc + r * EW - 2), lds2(zc + r * EW + 2),
                                                     col[r], col[r + 1], col[r + 3], col[r + 4], q[r]);
                    const size_t gofs = size_t(r) * n;
                    if (KB == K_A) {
                        const double2 t0 = lds2(zs + C::Z_ELEMS + sT + r * TXO);
                        const double2 t1 = lds2(zs + C::Z_ELEMS + C::T_ELEMS + sT + r * TXO);
                        double2 v0, v1;
                        v0.x = t0.x + (dt / 3.0) * kB.x;  v0.y = t0.y + (dt / 3.0) * kB.y;
                        v1.x = t1.x + (dt / 2.0) * kB.x;  v1.y = t1.y + (dt / 2.0) * kB.y;
                        *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                        *reinterpret_cast<double2 *>(o1 + gofs) = v1;
                    } else {
                        const double2 t0 = lds2(zs + C::Z_ELEMS + sT + r * TXO);
                        double2 v0;
                        v0.x = t0.x + (dt / 6.0) * kB.x;  v0.y = t0.y + (dt / 6.0) * kB.y;
                        *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                    }
                }
            }
            if (j >= 4) {
                o0 += nn;
                if (KB == K_A) o1 += nn;
            }
            if (j >= 2) {
                mbar_arrive(&empty[zc_pos.slot]);
                zc_pos.step(ZD);
            }
            zq_pos.step(ZD);
        });
        // release the item's last two Z planes (never a centre)
        mbar_arrive(&empty[zc_pos.slot]);
        zc_pos.step(ZD);
        mbar_arrive(&empty[zc_pos.slot]);
    }
}

template <int KB, class C>
__global__ void __launch_bounds__(C::NT, 1)
fused_persist_kernel(const StencilArgs a) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t full[C::ZD], empty[C::ZD], in_full[C::DEPTH], in_empty[C::DEPTH];
    const int items = a.tiles_x * a.tiles_y * a.chunks_z;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::ZD; ++s) {
            mbar_init(&full[s], C::NTA);
            mbar_init(&empty[s], C::NTB);
        }
        for (int s = 0; s < C::DEPTH; ++s) {
            mbar_init(&in_full[s], C::NTP);
            mbar_init(&in_empty[s], C::NTA);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x < C::NTA)
        stage_a_p<KB, C>(a, sm, items, full, empty, in_full, in_empty);
    else if (threadIdx.x < C::NTA + C::NTB)
        stage_b_p<KB, C>(a, sm, items, full, empty);
    else
        producer_p<KB, C>(a, sm, items, in_full, in_empty);
}

}  // namespace prk
