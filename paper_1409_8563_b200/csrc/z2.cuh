// z2.cuh — the two-kernel RK4 step of fused.cuh with every consumer warp working on
// TWO z planes per pipeline iteration (FusedCfgP + WithZ2): twice the independent
// DFMA chains between two waits, and half the barrier hand-offs per plane.  Round 2's
// profiles show the one-plane kernels latency-bound (issue ~45 %, no pipe saturated,
// time following the SM clock); this variant tests that reading.  The z queues grow
// from 5 to 6 entries (element / plane p at index p % 6, the loop unrolled by three
// iterations so they rotate by renaming), the intermediate ring from 4 to 6 slots, and
// the stencil weights come from the launch parameters (WithWP) to pay for the extra
// registers.  Same per-point operation sequence: bitwise identical results.
#pragma once
#include "fused.cuh"

namespace prk {

template <class C> struct WithZ2 : C { static constexpr bool Z2 = true; };

// the folded operator on a lane pair with z neighbours from a 6-entry queue, zm2 at index Z0
template <int Z0>
__device__ __forceinline__ double2 apply_pair6(const Weights &W, double2 L, double2 R, double2 ym2, double2 ym1,
                                               double2 yp1, double2 yp2, const double2 *q) {
    const double2 Cc = q[(Z0 + 2) % 6];
    const double2 zm2 = q[Z0 % 6], zm1 = q[(Z0 + 1) % 6], zp1 = q[(Z0 + 3) % 6], zp2 = q[(Z0 + 4) % 6];
    double2 k;
    k.x = apply13(W, Cc.x, L.x, L.y, Cc.y, R.x, ym2.x, ym1.x, yp1.x, yp2.x, zm2.x, zm1.x, zp1.x, zp2.x);
    k.y = apply13(W, Cc.y, L.y, Cc.x, R.x, R.y, ym2.y, ym1.y, yp1.y, yp2.y, zm2.y, zm1.y, zp1.y, zp2.y);
    return k;
}

// body(Ph<jj % 3>, jj) for jj = 0 .. NI-1, unrolled by three
template <class Body>
__device__ __forceinline__ void rotating_loop_by3(int NI, Body &&body) {
    int jj = 0;
#pragma unroll 1
    for (; jj + 3 <= NI; jj += 3) {
        body(Ph<0>{}, jj);
        body(Ph<1>{}, jj + 1);
        body(Ph<2>{}, jj + 2);
    }
    if (jj < NI) body(Ph<0>{}, jj++);
    if (jj < NI) body(Ph<1>{}, jj++);
}

template <int KB, class C>
__device__ __forceinline__ void stage_a_z2(const StencilArgs &a, double *sm, int items, uint64_t *full,
                                           uint64_t *empty, uint64_t *in_full, uint64_t *in_empty) {
    constexpr int RPT = C::RPTA, DEPTH = C::template DEPTH_K<KB>, EW = C::EWS, IW = C::IWS, TXO = C::TXO,
                  ZD = C::ZD;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    // barrier and ring addresses pinned in registers (fused.cuh, FusedCfgP::PIN)
    const SBars full_s = sbars<C>(full), empty_s = sbars<C>(empty);
    const SBars in_full_s = sbars<C>(in_full), in_empty_s = sbars<C>(in_empty);
    double *yring = smem_base<C>(sm);
    double *aring = yring + size_t(DEPTH) * C::Y_ELEMS;
    double *zring = aring + (KB == K_B ? size_t(C::AD) * C::AUX_ELEMS : 0);
    const int t = threadIdx.x;
    Weights W;
    if constexpr (C::WP) {
        W.load(a.wA);
    } else {
        const long long row = (*a.nu_pos + a.j_local) * 4;
        W.set(a.nu_tab[row + (KB == K_A ? 0 : 2)], a.inv_dx, a.c);
    }
    const double dt = a.dt;
    const bool valid = t < C::A_ITEMS;
    const int l = valid ? t % (C::EW / 2) : 0, g = valid ? t / (C::EW / 2) : 0;
    const int r0 = g * RPT;
    const int sY = (r0 + 2) * IW + 2 * l + 2;
    const int sZ = r0 * EW + 2 * l;
    const bool tcol = l >= 1 && l <= TXO / 2;
    const int tp0 = (r0 - 2) * TXO + 2 * l - 2;
    bool tile_row[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) tile_row[r] = tcol && r0 + r >= 2 && r0 + r < C::TYO + 2;

    RingPos base, zpos;
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;  // even (the z chunks are even)
        double2 q[RPT][6];        // input element e at index e % 6
        RingPos p0 = base;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            mbar_wait(in_full_s[p0.slot], p0.round & 1);
            const double *ys = yring + size_t(p0.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][e] = lds2(ys + r * IW);
            p0.step(DEPTH);
        }
        mbar_arrive(in_empty_s[base.slot]);
        mbar_arrive(in_empty_s[ring_at(base, 1, DEPTH).slot]);
        RingPos p2 = ring_at(base, 2, DEPTH), p4 = p0;  // elements j+2, j+4 (j = 2 jj)
        rotating_loop_by3(NJ / 2, [&](auto ph, int jj) {
            constexpr int B = 2 * decltype(ph)::value;  // index of element j
            const int j = 2 * jj;
            RingPos p3 = p2, p5 = p4;
            p3.step(DEPTH);
            p5.step(DEPTH);
            mbar_wait(in_full_s[p4.slot], p4.round & 1);
            mbar_wait(in_full_s[p5.slot], p5.round & 1);
            const double *yq4 = yring + size_t(p4.slot) * C::Y_ELEMS + sY;
            const double *yq5 = yring + size_t(p5.slot) * C::Y_ELEMS + sY;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                q[r][(B + 4) % 6] = lds2(yq4 + r * IW);
                q[r][(B + 5) % 6] = lds2(yq5 + r * IW);
            }
            const double *ys[2] = {yring + size_t(p2.slot) * C::Y_ELEMS + sY,
                                   yring + size_t(p3.slot) * C::Y_ELEMS + sY};
            const double *au[2] = {aring + size_t(p4.slot) * C::AUX_ELEMS,   // aux j
                                   aring + size_t(p5.slot) * C::AUX_ELEMS};  // aux j+1
            double2 k[2][RPT], ubv[2][KB == K_B ? RPT : 1], acv[2][KB == K_B ? RPT : 1];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if constexpr (KB == K_B) {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        ubv[h][r] = lds2(au[h] + sZ + r * EW);
                        acv[h][r] = lds2(au[h] + C::Z_ELEMS + (tile_row[r] ? tp0 + r * TXO : 0));
                    }
                }
                double2 col[RPT + 4];
#pragma unroll
                for (int r = 0; r < RPT + 4; ++r)
                    col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(B + h + 2) % 6] : lds2(ys[h] + (r - 2) * IW);
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    if (h == 0)
                        k[h][r] = apply_pair6<B>(W, lds2(ys[h] + r * IW - 2), lds2(ys[h] + r * IW + 2), col[r],
                                                 col[r + 1], col[r + 3], col[r + 4], q[r]);
                    else
                        k[h][r] = apply_pair6<B + 1>(W, lds2(ys[h] + r * IW - 2), lds2(ys[h] + r * IW + 2),
                                                     col[r], col[r + 1], col[r + 3], col[r + 4], q[r]);
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (zpos.round > 0) mbar_wait(empty_s[zpos.slot], (zpos.round - 1) & 1);
                double *zs = zring + size_t(zpos.slot) * ZS;
                const bool outp = j + h >= 2 && j + h < w.nz + 2;
                if (valid) {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        const double2 yc = q[r][(B + h + 2) % 6];
                        double2 z;
                        if (KB == K_A) {
                            z.x = yc.x + (dt / 2.0) * k[h][r].x;
                            z.y = yc.y + (dt / 2.0) * k[h][r].y;
                        } else {
                            const double2 ub = ubv[h][KB == K_B ? r : 0];
                            z.x = ub.x + dt * k[h][r].x;
                            z.y = ub.y + dt * k[h][r].y;
                        }
                        sts2(zs + sZ + r * EW, z);
                        if (outp && tile_row[r]) {
                            const int tp = tp0 + r * TXO;
                            if (KB == K_A) {
                                double2 t0;
                                t0.x = yc.x + (dt / 6.0) * k[h][r].x;
                                t0.y = yc.y + (dt / 6.0) * k[h][r].y;
                                sts2(zs + C::Z_ELEMS + tp, t0);
                                sts2(zs + C::Z_ELEMS + C::T_ELEMS + tp, yc);
                            } else {
                                const double2 ac = acv[h][KB == K_B ? r : 0];
                                double2 t0;
                                t0.x = ac.x + (dt / 3.0) * k[h][r].x;
                                t0.y = ac.y + (dt / 3.0) * k[h][r].y;
                                sts2(zs + C::Z_ELEMS + tp, t0);
                            }
                        }
                    }
                }
                mbar_arrive(full_s[zpos.slot]);
                zpos.step(ZD);
            }
            mbar_arrive(in_empty_s[p2.slot]);  // elements j+2, j+3 done
            mbar_arrive(in_empty_s[p3.slot]);
            p2.step(DEPTH);
            p2.step(DEPTH);
            p4.step(DEPTH);
            p4.step(DEPTH);
        });
        mbar_arrive(in_empty_s[p2.slot]);
        mbar_arrive(in_empty_s[ring_at(p2, 1, DEPTH).slot]);
        base = ring_at(p2, 2, DEPTH);
    }
}

template <int KB, class C>
__device__ __forceinline__ void stage_b_z2(const StencilArgs &a, double *sm, int items, uint64_t *full,
                                           uint64_t *empty) {
    constexpr int RPT = C::RPT, EW = C::EWS, TXO = C::TXO, ZD = C::ZD, DEPTH = C::template DEPTH_K<KB>;
    constexpr int ZS = C::template ZS_ELEMS<KB>;
    const SBars full_s = sbars<C>(full), empty_s = sbars<C>(empty);
    sm = smem_base<C>(sm);
    double *zring = sm + size_t(DEPTH) * C::Y_ELEMS + (KB == K_B ? size_t(C::AD) * C::AUX_ELEMS : 0);
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int tb = threadIdx.x - C::NTA;
    const bool valid = tb < C::B_ITEMS;
    const int m = valid ? tb % (TXO / 2) : 0, g = valid ? tb / (TXO / 2) : 0;
    const int r0 = g * RPT;
    const int sZ = (r0 + 2) * EW + 2 * m + 2;
    const int sT = r0 * TXO + 2 * m;
    Weights W;
    if constexpr (C::WP) {
        W.load(a.wB);
    } else {
        const long long row = (*a.nu_pos + a.j_local) * 4;
        W.set(a.nu_tab[row + (KB == K_A ? 1 : 3)], a.inv_dx, a.c);
    }
    const double dt = a.dt;

    RingPos zq_pos;  // plane j of the current iteration (queue loads)
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 4;
        double *o0 = a.o0 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * m;
        double *o1 = KB == K_A ? a.o1 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * m
                               : nullptr;
        double2 q[RPT][6];        // intermediate plane p at index p % 6
        RingPos zc_pos = zq_pos;  // plane j-2 (the first centre), valid from jj = 2
        rotating_loop_by3(NJ / 2, [&](auto ph, int jj) {
            constexpr int B = 2 * decltype(ph)::value;  // index of plane j
            RingPos zq1 = zq_pos;
            zq1.step(ZD);
            mbar_wait(full_s[zq_pos.slot], zq_pos.round & 1);
            mbar_wait(full_s[zq1.slot], zq1.round & 1);
            const double *zq[2] = {zring + size_t(zq_pos.slot) * ZS + sZ, zring + size_t(zq1.slot) * ZS + sZ};
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                q[r][B % 6] = lds2(zq[0] + r * EW);
                q[r][(B + 1) % 6] = lds2(zq[1] + r * EW);
            }
            if (jj >= 2 && valid) {  // outputs centred on planes j-2 and j-1
                RingPos zc1 = zc_pos;
                zc1.step(ZD);
                const double *zs[2] = {zring + size_t(zc_pos.slot) * ZS, zring + size_t(zc1.slot) * ZS};
                double2 kB[2][RPT];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double *zc = zs[h] + sZ;
                    double2 col[RPT + 4];
#pragma unroll
                    for (int r = 0; r < RPT + 4; ++r)
                        col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(B + 4 + h) % 6] : lds2(zc + (r - 2) * EW);
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        if (h == 0)
                            kB[h][r] = apply_pair6<B + 2>(W, lds2(zc + r * EW - 2), lds2(zc + r * EW + 2), col[r],
                                                          col[r + 1], col[r + 3], col[r + 4], q[r]);
                        else
                            kB[h][r] = apply_pair6<B + 3>(W, lds2(zc + r * EW - 2), lds2(zc + r * EW + 2), col[r],
                                                          col[r + 1], col[r + 3], col[r + 4], q[r]);
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        const size_t gofs = size_t(r) * n;
                        const double2 t0 = lds2(zs[h] + C::Z_ELEMS + sT + r * TXO);
                        if (KB == K_A) {
                            const double2 t1 = lds2(zs[h] + C::Z_ELEMS + C::T_ELEMS + sT + r * TXO);
                            double2 v0, v1;
                            v0.x = t0.x + (dt / 3.0) * kB[h][r].x;  v0.y = t0.y + (dt / 3.0) * kB[h][r].y;
                            v1.x = t1.x + (dt / 2.0) * kB[h][r].x;  v1.y = t1.y + (dt / 2.0) * kB[h][r].y;
                            *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                            *reinterpret_cast<double2 *>(o1 + gofs) = v1;
                        } else {
                            double2 v0;
                            v0.x = t0.x + (dt / 6.0) * kB[h][r].x;  v0.y = t0.y + (dt / 6.0) * kB[h][r].y;
                            *reinterpret_cast<double2 *>(o0 + gofs) = v0;
                        }
                    }
                    o0 += nn;
                    if (KB == K_A) o1 += nn;
                }
            }
            if (jj >= 1) {  // planes j-2 and j-1 are no longer read
                mbar_arrive(empty_s[zc_pos.slot]);
                zc_pos.step(ZD);
                mbar_arrive(empty_s[zc_pos.slot]);
                zc_pos.step(ZD);
            }
            zq_pos.step(ZD);
            zq_pos.step(ZD);
        });
        // the item's last two planes (never a centre)
        mbar_arrive(empty_s[zc_pos.slot]);
        zc_pos.step(ZD);
        mbar_arrive(empty_s[zc_pos.slot]);
    }
}

template <int KB, class C>
__global__ void __maxnreg__(C::MAXR) fused_z2_kernel(const StencilArgs a, const __grid_constant__ TmaMaps tm) {
    extern __shared__ __align__(128) double sm[];
    constexpr int DEPTH = C::template DEPTH_K<KB>;
    __shared__ __align__(8) uint64_t full[C::ZD], empty[C::ZD], in_full[DEPTH], in_empty[DEPTH];
    const int items = a.tiles_x * a.tiles_y * a.chunks_z;
    if constexpr (C::FILL == 2) {
        if (smem_u32(sm) & 127) __trap();
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::ZD; ++s) {
            mbar_init(&full[s], C::NTA);
            mbar_init(&empty[s], C::NTB);
        }
        for (int s = 0; s < DEPTH; ++s) {
            mbar_init(&in_full[s], C::NTP);
            mbar_init(&in_empty[s], C::NTA);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x < C::NTA)
        stage_a_z2<KB, C>(a, sm, items, full, empty, in_full, in_empty);
    else if (threadIdx.x < C::NTA + C::NTB)
        stage_b_z2<KB, C>(a, sm, items, full, empty);
    else
        producer_p<KB, C>(a, &tm, sm, items, in_full, in_empty);
}

}  // namespace prk
