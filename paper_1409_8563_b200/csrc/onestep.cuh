// onestep.cuh — one classical RK4 step in ONE kernel:
// 16 B/point of HBM traffic (read u, write u_new) instead of 56 (two kernels).
//
// Four warp groups, one per RK4 stage, chained along z by shared-memory rings:
//   group 1: k1 = L(u)  on the tile + a 6-point ring; Ya = u + dt/2 k1, acc = u + dt/6 k1
//   group 2: k2 = L(Ya) on the tile + 4;              Yb = u + dt/2 k2, acc += dt/3 k2
//   group 3: k3 = L(Yb) on the tile + 2;              Ya'= u + dt k3,   acc += dt/3 k3
//   group 4: k4 = L(Ya') on the tile;                 u_new = acc + dt/6 k4  -> HBM
// Stage s runs on the output tile grown by 2 (4 - s) points per side, so the input
// is read with a halo of 8 (the "halo 8" of a fused step).  Each group keeps its z
// neighbours in a register queue (the fused kernels' scheme) and reads x/y
// neighbours from the ring of the previous group; u at a group's points and the
// running acc at the tile points ride in the same ring slot.  One producer warp
// fills the input ring with wrap-aware 16-byte cp.async copies.  Same per-point
// operation sequence as the four-pass kernels: bitwise identical results.
//
// Why it is not the default (measured): with B200's 64K registers
// per SM, four register-queued groups fit only on a 16 x 8 tile, where the rings
// recompute 2.5x the stencils of the two-kernel step (which recomputes 1.3x).
#pragma once
#include "fused.cuh"

namespace prk {

namespace one {  // geometry of the one-kernel step: output tile 16 x 8, stage s on tile + 2(4-s)
constexpr int TXO = 16, TYO = 8;
__host__ __device__ constexpr int h(int s) { return 2 * (4 - s); }  // halo of stage s (0: the input)
__host__ __device__ constexpr int W(int s) { return TXO + 2 * h(s); }
__host__ __device__ constexpr int H(int s) { return TYO + 2 * h(s); }
__host__ __device__ constexpr int P(int s) { return W(s) + 2; }  // padded pitch
__host__ __device__ constexpr int lanes(int s) { return (W(s) / 2) * (H(s) / 2); }
__host__ __device__ constexpr int warps(int s) { return (lanes(s) + 31) / 32; }
__host__ __device__ constexpr int base(int s) { return s <= 1 ? 0 : base(s - 1) + 32 * warps(s - 1); }  // first thread
__host__ __device__ constexpr int pad16(int e) { return (e + 15) / 16 * 16; }
// ring s (1..3) slot: Y part on R_s, U part on R_{s+1} (s < 3), A part (acc) on the tile
__host__ __device__ constexpr int UO(int s) { return pad16(H(s) * P(s)); }
__host__ __device__ constexpr int AO(int s) { return UO(s) + (s < 3 ? pad16(H(s + 1) * P(s + 1)) : 0); }
__host__ __device__ constexpr int RS(int s) { return AO(s) + TYO * TXO; }
}  // namespace one

struct OneCfg {
    static constexpr bool COMB = false;
    static constexpr int TXO = one::TXO, TYO = one::TYO, DEPTH = 12, ZD = 4, FILL = 0;
    __host__ __device__ static constexpr int h(int s) { return one::h(s); }
    __host__ __device__ static constexpr int W(int s) { return one::W(s); }
    __host__ __device__ static constexpr int H(int s) { return one::H(s); }
    __host__ __device__ static constexpr int P(int s) { return one::P(s); }
    __host__ __device__ static constexpr int lanes(int s) { return one::lanes(s); }
    __host__ __device__ static constexpr int warps(int s) { return one::warps(s); }
    __host__ __device__ static constexpr int base(int s) { return one::base(s); }
    __host__ __device__ static constexpr int UO(int s) { return one::UO(s); }
    __host__ __device__ static constexpr int AO(int s) { return one::AO(s); }
    __host__ __device__ static constexpr int RS(int s) { return one::RS(s); }
    static constexpr int NTP = 32, NT = one::base(5) + NTP;
    static constexpr int MAXR = (65536 / NT) / 8 * 8 > 255 ? 255 : (65536 / NT) / 8 * 8;
    static constexpr int IN_ELEMS = one::pad16(one::H(0) * one::P(0));
    __host__ __device__ static constexpr int RING_BASE(int s) {  // doubles from the start of dynamic smem
        return s <= 1 ? DEPTH_ * IN_ELEMS_ : RING_BASE(s - 1) + 4 * one::RS(s - 1);
    }
    static constexpr int DEPTH_ = 12, IN_ELEMS_ = one::pad16(one::H(0) * one::P(0));
    template <int KB> static constexpr size_t smem_bytes() { return sizeof(double) * size_t(RING_BASE(4)); }
    static constexpr int IN_CHUNKS = one::H(0) * (one::W(0) / 2);
    static_assert(NT <= 1024, "too many threads");
};

// producer: the input plane (output tile + halo 8, periodic wrap folded into the plan)
template <class C>
__device__ __forceinline__ void one_producer(const StencilArgs &a, double *sm, int items, uint64_t *in_full,
                                             uint64_t *in_empty) {
    constexpr int NP = C::NTP, NY = (C::IN_CHUNKS + NP - 1) / NP;
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int lane = threadIdx.x - C::base(5);
    const uint32_t ring_s = smem_u32(sm);
    RingPos pos;
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, C::TXO, C::TYO);
        int src[NY], dst[NY];
#pragma unroll
        for (int k = 0; k < NY; ++k) {
            const int c = lane + NP * k;
            src[k] = -1;
            dst[k] = 0;
            if (c < C::IN_CHUNKS) {
                const int r = c / (C::W(0) / 2), cc = c % (C::W(0) / 2);
                src[k] = wrapi(w.y0 - C::h(0) + r, n) * n + wrapi(w.x0 - C::h(0) + 2 * cc, n);
                dst[k] = 8 * (r * C::P(0) + 2 * cc);
            }
        }
        const int E = w.nz + 2 * C::h(0);
        int zin = wrapi(w.z_begin - C::h(0), n);
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
            if (pos.round > 0) mbar_wait(&in_empty[pos.slot], (pos.round - 1) & 1);
            const double *s = a.y + size_t(zin) * nn;
            const uint32_t d = ring_s + uint32_t(pos.slot) * (C::IN_ELEMS * 8);
#pragma unroll
            for (int k = 0; k < NY; ++k)
                if (src[k] >= 0) cp_async16s(d + dst[k], s + src[k]);
            cp_async_mbar_arrive(&in_full[pos.slot]);
            zin = (zin + 1 == n) ? 0 : zin + 1;
            pos.step(C::DEPTH);
        }
    }
    cp_async_wait<0>();
}

// group S (1..4).  Group 1 reads the input ring; group S >= 2 reads ring S-1; groups
// 1..3 write ring S, group 4 writes u_new to HBM.
template <int S, class C>
__device__ __forceinline__ void one_group(const StencilArgs &a, double *sm, int items, uint64_t *in_full,
                                          uint64_t *in_empty, uint64_t *full, uint64_t *empty) {
    constexpr int PI = C::P(S - 1), PO = C::P(S), TXO = C::TXO, ZD = C::ZD, RPT = 2;
    constexpr int IN_RS = S == 1 ? C::IN_ELEMS : C::RS(S - 1);  // slot size of the input ring
    constexpr int IN_DEPTH = S == 1 ? C::DEPTH : ZD;
    double *in_ring = sm + (S == 1 ? 0 : C::RING_BASE(S - 1));
    double *out_ring = sm + (S < 4 ? C::RING_BASE(S) : 0);
    uint64_t *ifull = S == 1 ? in_full : full + (S - 2) * ZD;     // barriers of the input ring
    uint64_t *iempty = S == 1 ? in_empty : empty + (S - 2) * ZD;
    uint64_t *ofull = full + (S - 1) * ZD, *oempty = empty + (S - 1) * ZD;  // of ring S (S < 4)
    const int n = a.n;
    const size_t nn = size_t(n) * n;
    const int t = threadIdx.x - C::base(S);
    const bool valid = t < C::lanes(S);
    const int l = valid ? t % (C::W(S) / 2) : 0, g = valid ? t / (C::W(S) / 2) : 0;
    const int r0 = 2 * g;
    const int sIn = (r0 + 2) * PI + 2 * l + 2;  // own centre in the input ring
    const int sOut = r0 * PO + 2 * l;          // own point in ring S
    // own point inside the next region (U part of ring S) and inside the tile (A parts)
    const bool in_next = S < 3 && l >= 1 && l < C::W(S) / 2 - 1 && g >= 1 && g < C::H(S) / 2 - 1;
    const int sUn = S < 3 ? (r0 - 2) * C::P(S + 1) + 2 * l - 2 : 0;
    const bool in_tile = l >= C::h(S) / 2 && l < C::h(S) / 2 + TXO / 2 && g >= C::h(S) / 2 &&
                         g < C::h(S) / 2 + C::TYO / 2;
    const int sA = (r0 - C::h(S)) * TXO + 2 * l - C::h(S);

    const long long row = (*a.nu_pos + a.j_local) * 4;
    Weights W;
    W.set(a.nu_tab[row + (S - 1)], a.inv_dx, a.c);
    const double dt = a.dt;

    RingPos ipos;  // input ring: plane 0 of the current item
    RingPos opos;  // ring S: next plane to write
#pragma unroll 1
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const WorkItem w = decode_item(a, item, TXO, C::TYO);
        const int NJ = w.nz + 2 * C::h(S - 1);  // planes of the input ring in this item
        double *o0 = nullptr;
        if (S == 4) o0 = a.o0 + size_t(w.z_begin) * nn + size_t(w.y0 + r0) * n + w.x0 + 2 * l;
        double2 q[RPT][5];
        RingPos qpos = ipos;                 // input plane j (queue)
        RingPos cpos = ipos;                 // input plane j-2 (centre)
        rotating_loop(NJ, [&](auto ph, int j) {
            constexpr int P = decltype(ph)::value;
            mbar_wait(&ifull[qpos.slot], qpos.round & 1);
            const double *iq = in_ring + size_t(qpos.slot) * IN_RS + sIn;
#pragma unroll
            for (int r = 0; r < RPT; ++r) q[r][(P + 4) % 5] = lds2(iq + r * PI);
            if (j >= 4) {  // own plane j-4 (centre: input plane j-2)
                const double *ic = in_ring + size_t(cpos.slot) * IN_RS;
                const double *ys = ic + sIn;
                double2 k[RPT];
                if (valid) {
                    double2 col[RPT + 4];
#pragma unroll
                    for (int r = 0; r < RPT + 4; ++r)
                        col[r] = (r >= 2 && r < RPT + 2) ? q[r - 2][(P + 2) % 5] : lds2(ys + (r - 2) * PI);
#pragma unroll
                    for (int r = 0; r < RPT; ++r)
                        k[r] = apply_pair<P>(W, lds2(ys + r * PI - 2), lds2(ys + r * PI + 2), col[r], col[r + 1],
                                             col[r + 3], col[r + 4], q[r]);
                }
                if constexpr (S < 4) {
                    if (opos.round > 0) mbar_wait(&oempty[opos.slot], (opos.round - 1) & 1);
                }
                if (valid) {
                    double *od = S < 4 ? out_ring + size_t(opos.slot) * C::RS(S) : nullptr;
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        // u at the own point: the input centre (group 1) or the U part of the input slot
                        const double2 u = S == 1 ? q[r][(P + 2) % 5] : lds2(ic + C::UO(S - 1) + sOut + r * PO);
                        double2 acc;  // the running RK4 sum at tile points
                        if (S > 1 && in_tile) acc = lds2(ic + C::AO(S - 1) + sA + r * TXO);
                        if (S == 1) {
                            double2 y;
                            y.x = u.x + (dt / 2.0) * k[r].x;  y.y = u.y + (dt / 2.0) * k[r].y;
                            sts2(od + sOut + r * PO, y);
                            if (in_tile) {
                                double2 c;
                                c.x = u.x + (dt / 6.0) * k[r].x;  c.y = u.y + (dt / 6.0) * k[r].y;
                                sts2(od + C::AO(S) + sA + r * TXO, c);
                            }
                        } else if (S == 2 || S == 3) {
                            double2 y;
                            const double f = S == 2 ? dt / 2.0 : dt;
                            y.x = u.x + f * k[r].x;  y.y = u.y + f * k[r].y;
                            sts2(od + sOut + r * PO, y);
                            if (in_tile) {
                                double2 c;
                                c.x = acc.x + (dt / 3.0) * k[r].x;  c.y = acc.y + (dt / 3.0) * k[r].y;
                                sts2(od + C::AO(S) + sA + r * TXO, c);
                            }
                        } else {
                            double2 v;
                            v.x = acc.x + (dt / 6.0) * k[r].x;  v.y = acc.y + (dt / 6.0) * k[r].y;
                            *reinterpret_cast<double2 *>(o0 + size_t(r) * n) = v;
                        }
                        if (S < 3 && in_next) sts2(od + C::UO(S) + sUn + r * C::P(S + 1), u);
                    }
                }
                if constexpr (S < 4) {
                    mbar_arrive(&ofull[opos.slot]);
                    opos.step(ZD);
                } else {
                    o0 += nn;
                }
            }
            if (j >= 2) {  // input plane j-2 is no longer read
                mbar_arrive(&iempty[cpos.slot]);
                cpos.step(IN_DEPTH);
            }
            qpos.step(IN_DEPTH);
        });
        // the item's last two input planes were only queue entries
        mbar_arrive(&iempty[cpos.slot]);
        cpos.step(IN_DEPTH);
        mbar_arrive(&iempty[cpos.slot]);
        cpos.step(IN_DEPTH);
        ipos = cpos;
    }
}

template <int KB, class C>
__global__ void __maxnreg__(C::MAXR) onestep_kernel(const StencilArgs a, const __grid_constant__ TmaMaps tm) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t in_full[C::DEPTH], in_empty[C::DEPTH], full[3 * C::ZD], empty[3 * C::ZD];
    const int items = a.tiles_x * a.tiles_y * a.chunks_z;
    (void)tm;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::DEPTH; ++s) {
            mbar_init(&in_full[s], C::NTP);
            mbar_init(&in_empty[s], 32 * C::warps(1));
        }
        for (int s = 1; s <= 3; ++s)
            for (int k = 0; k < C::ZD; ++k) {
                mbar_init(&full[(s - 1) * C::ZD + k], 32 * C::warps(s));
                mbar_init(&empty[(s - 1) * C::ZD + k], 32 * C::warps(s + 1));
            }
        fence_mbar_init();
    }
    __syncthreads();
    const int tid = threadIdx.x;
    if (tid < C::base(2))
        one_group<1, C>(a, sm, items, in_full, in_empty, full, empty);
    else if (tid < C::base(3))
        one_group<2, C>(a, sm, items, in_full, in_empty, full, empty);
    else if (tid < C::base(4))
        one_group<3, C>(a, sm, items, in_full, in_empty, full, empty);
    else if (tid < C::base(5))
        one_group<4, C>(a, sm, items, in_full, in_empty, full, empty);
    else
        one_producer<C>(a, sm, items, in_full, in_empty);
}

}  // namespace prk
