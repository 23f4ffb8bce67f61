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
// then stage A of plane j; one named barrier over the compute warps per
// iteration orders the intermediate ring (4 slots).  Producer warps and the
// input ring are those of fused.cuh (TMA tensor fills, cp.async on seams).
// Same per-point floating-point operation sequence as the four-pass kernels:
// the results are bitwise identical.
#pragma once
#include "fused.cuh"

namespace prk {

template <int TYO_, int DEPTH_, int PW_ = 2, int FILL_ = 2, int ZD_ = 4>
struct CombCfg {
    static constexpr bool COMB = true;
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
using Comb16 = CombCfg<16, 9>;  // 32x16 tile: 4 combined + 2 ring + 2 producer warps

__device__ __forceinline__ void bar_compute(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int KB, class C>
__device__ __forceinline__ void comb_consumer(const StencilArgs &a, double *sm, int items,
                                              uint64_t *in_full, uint64_t *in_empty) {
    constexpr int RPT = C::RPT, DEPTH = C::DEPTH, EW = C::EWS, IW = C::IWS, TXO = C::TXO, ZD = C::ZD;
    double *yring = sm;
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
    constexpr int NC = C::NTA;

    RingPos base;  // input element 0 of the current item
    int zj = 0;    // intermediate ring slot of plane j (runs on across items)
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;
        double *o0 = a.o0 + size_t(w.z_begin) * nn + size_t(w.y0 + r0 - 2) * n + w.x0 + 2 * l - 2;
        double *o1 = KB == K_A ? a.o1 + size_t(w.z_begin) * nn + size_t(w.y0 + r0 - 2) * n + w.x0 + 2 * l - 2
                               : nullptr;
        double2 qa[RPT][5];  // input z-queue
        double2 qb[RPT][5];  // own intermediate values, planes j-5 .. j-1
        double2 tl[3][RPT];  // t0 of planes j-3, j-2, j-1
        RingPos p0 = base;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            mbar_wait(&in_full[p0.slot], p0.round & 1);
            const double *ys = yring + size_t(p0.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) qa[r][e] = lds2(ys + r * IW);
            p0.step(DEPTH);
        }
        mbar_arrive(&in_empty[base.slot]);
        mbar_arrive(&in_empty[ring_at(base, 1, DEPTH).slot]);
        RingPos p2 = ring_at(base, 2, DEPTH), p4 = p0;  // elements j+2, j+4
        // iteration j: stage B of output plane j-5 (j >= 5), then stage A of plane j (j < NJ)
        rotating_loop(NJ + 1, [&](auto ph, int j) {
            constexpr int P = decltype(ph)::value;  // qa[.][(P+k)%5] = element j+k-1 before the load
            if (comb && j >= 5) {
                // x/y neighbours of intermediate plane j-3 (the centre of output j-5)
                const int zc = zj >= 3 ? zj - 3 : zj - 3 + ZD;
                const double *zp = zring + size_t(zc) * C::Z_ELEMS + sZ;
                double2 col[RPT + 4];
#pragma unroll
                for (int r = 0; r < RPT + 4; ++r)
                    col[r] = (r >= 2 && r < RPT + 2) ? qb[r - 2][(P + 2) % 5] : lds2(zp + (r - 2) * EW);
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double2 kB = apply_pair<P>(WB, lds2(zp + r * EW - 2), lds2(zp + r * EW + 2), col[r],
                                                     col[r + 1], col[r + 3], col[r + 4], qb[r]);
                    const size_t gofs = size_t(r) * n;
                    const double2 t0 = tl[0][r];
                    if (KB == K_A) {
                        const double2 t1 = qa[r][(P + 4) % 5];  // u at the output point (element j-1)
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
            }
            if (j < NJ) {
                mbar_wait(&in_full[p4.slot], p4.round & 1);  // element j+4 (+ aux j) landed
                const double *yq = yring + size_t(p4.slot) * C::Y_ELEMS + sY;
#pragma unroll
                for (int r = 0; r < RPT; ++r) qa[r][(P + 4) % 5] = lds2(yq + r * IW);
                const double *ys = yring + size_t(p2.slot) * C::Y_ELEMS + sY;
                double2 col[RPT + 4];
#pragma unroll
                for (int r = 0; r < RPT + 4; ++r)
                    col[r] = (r >= 2 && r < RPT + 2) ? qa[r - 2][(P + 2) % 5] : lds2(ys + (r - 2) * IW);
                const double *au = aring + size_t(p4.slot) * C::AUX_ELEMS;  // aux j
                double2 ubv[KB == K_B ? RPT : 1], acv[KB == K_B ? RPT : 1];
                if constexpr (KB == K_B) {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        ubv[r] = lds2(au + sZ + r * EW);
                        acv[r] = lds2(au + C::Z_ELEMS + (comb ? tp0 + r * TXO : 0));
                    }
                } else {
                    (void)au;
                }
                double2 k[RPT];
#pragma unroll
                for (int r = 0; r < RPT; ++r)
                    k[r] = apply_pair<P>(WA, lds2(ys + r * IW - 2), lds2(ys + r * IW + 2), col[r], col[r + 1],
                                         col[r + 3], col[r + 4], qa[r]);
                double *zd = zring + size_t(zj) * C::Z_ELEMS + sZ;
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double2 yc = qa[r][(P + 2) % 5];
                    double2 z, t0;
                    if (KB == K_A) {
                        z.x = yc.x + (dt / 2.0) * k[r].x;
                        z.y = yc.y + (dt / 2.0) * k[r].y;
                        t0.x = yc.x + (dt / 6.0) * k[r].x;
                        t0.y = yc.y + (dt / 6.0) * k[r].y;
                    } else {
                        const double2 ub = ubv[KB == K_B ? r : 0], ac = acv[KB == K_B ? r : 0];
                        z.x = ub.x + dt * k[r].x;
                        z.y = ub.y + dt * k[r].y;
                        t0.x = ac.x + (dt / 3.0) * k[r].x;
                        t0.y = ac.y + (dt / 3.0) * k[r].y;
                    }
                    if (valid) sts2(zd + r * EW, z);
                    if (comb) {
                        qb[r][P] = z;  // plane j replaces plane j-5
                        tl[0][r] = tl[1][r];
                        tl[1][r] = tl[2][r];
                        tl[2][r] = t0;
                    }
                }
                mbar_arrive(&in_empty[p2.slot]);  // element j+2 done (aux j lives in slot j+4)
                p2.step(DEPTH);
                p4.step(DEPTH);
            }
            zj = (zj + 1 == ZD) ? 0 : zj + 1;
            bar_compute(NC);
        });
        // the item's last two input elements were only used by the queue
        mbar_arrive(&in_empty[p2.slot]);
        mbar_arrive(&in_empty[ring_at(p2, 1, DEPTH).slot]);
        base = ring_at(p2, 2, DEPTH);
    }
}

template <int KB, class C>
__global__ void __maxnreg__(C::MAXR)
fused_comb_kernel(const StencilArgs a, const __grid_constant__ TmaMaps tm) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t in_full[C::DEPTH], in_empty[C::DEPTH];
    const int items = a.tiles_x * a.tiles_y * a.chunks_z;
    if constexpr (C::FILL == 2) {
        if (smem_u32(sm) & 127) __trap();  // TMA destinations need 128-byte alignment
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
        comb_consumer<KB, C>(a, sm, items, in_full, in_empty);
    else
        producer_p<KB, C>(a, &tm, sm, items, in_full, in_empty);
}

}  // namespace prk
