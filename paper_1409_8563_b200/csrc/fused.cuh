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
// One RK4 step moves 56 B/point instead of 128 B/point for four stage passes.
//
// Geometry: output tile TXO x TYO (x, y); stage A runs on the extended region
// (TXO+4) x (TYO+4); its input is read on (TXO+8) x (TYO+8).  A CTA marches a
// z chunk; stage A lags the input stream by 2 planes and stage B lags stage A
// by 2 planes.  The stencil input is streamed into a DEPTH-slot shared ring
// with 16-byte cp.async copies (periodic wrap folded into a per-thread plan),
// Ya lives in a 3-plane shared ring, z neighbours in per-thread register
// queues, each thread handles RPT = 4 consecutive rows (shared y neighbours).
#pragma once
#include "kernels.cuh"

namespace prk {

enum Kind2 { K_A = 0, K_B = 1 };

template <int TYO_, int DEPTH_, int MINB_ = 1> struct FusedCfg {
    static constexpr int TXO = 32, TYO = TYO_, DEPTH = DEPTH_, RPT = 4, MINB = MINB_;
    static constexpr int EW = TXO + 4, EH = TYO + 4;   // stage-A (extended) region
    static constexpr int IW = TXO + 8, IH = TYO + 8;   // input region
    static constexpr int A_ITEMS = EW * (EH / RPT);
    static constexpr int B_ITEMS = TXO * (TYO / RPT);
    static constexpr int NT = ((A_ITEMS + 31) / 32) * 32;
    static constexpr int Y_ELEMS = IH * IW;
    static constexpr int Z_ELEMS = EH * EW;
    static constexpr int T_ELEMS = TYO * TXO;
    static constexpr int Y_CHUNKS = IH * (IW / 2);
    static constexpr int NCY = (Y_CHUNKS + NT - 1) / NT;
    static_assert(TYO % RPT == 0 && EH % RPT == 0, "rows must split into RPT groups");
    static_assert(DEPTH >= 6, "ring too shallow");
    template <int KB> static constexpr int NTV = KB == K_A ? 2 : 1;
    template <int KB> static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t(DEPTH) * Y_ELEMS + 3 * Z_ELEMS + 3 * NTV<KB> * T_ELEMS);
    }
};
using Fused0 = FusedCfg<16, 6, 1>;
using Fused1 = FusedCfg<16, 6, 2>;   // register-capped for 2 CTAs/SM
using Fused2 = FusedCfg<8, 6, 2>;    // smaller tile

template <int KB, class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
fused_kernel(const StencilArgs a) {
    constexpr int RPT = C::RPT, DEPTH = C::DEPTH, EW = C::EW, IW = C::IW, TXO = C::TXO;
    constexpr int NTV = C::template NTV<KB>;
    extern __shared__ __align__(128) double sm[];
    double *yring = sm;                                  // DEPTH x input planes
    double *zring = yring + size_t(DEPTH) * C::Y_ELEMS;  // 3 x intermediate planes
    double *tring = zring + 3 * C::Z_ELEMS;              // 3 x NTV tile planes

    const int n = a.n;
    const size_t nn = size_t(n) * n;
    int b = blockIdx.x;
    const int tix = b % a.tiles_x; b /= a.tiles_x;
    const int tiy = b % a.tiles_y; b /= a.tiles_y;
    const int x0 = tix * TXO, y0 = tiy * C::TYO;
    const int z_begin = b * a.cz;
    const int nz = min(a.cz, n - z_begin);
    const int E = nz + 8;    // input planes z_begin-4 .. z_begin+nz+3
    const int NJ = nz + 4;   // stage-A planes z_begin-2 .. z_begin+nz+1
    const int t = threadIdx.x;

    // copy plan of one input plane (periodic wrap in x and y folded in)
    int ysrc[C::NCY], ydst[C::NCY];
#pragma unroll
    for (int k = 0; k < C::NCY; ++k) {
        const int c = t + k * C::NT;
        ysrc[k] = -1;
        ydst[k] = 0;
        if (c < C::Y_CHUNKS) {
            const int r = c / (IW / 2), cc = c % (IW / 2);
            ysrc[k] = wrapi(y0 - 4 + r, n) * n + wrapi(x0 - 4 + 2 * cc, n);
            ydst[k] = r * IW + 2 * cc;
        }
    }
    auto issue = [&](int e) {
        const double *src = a.y + size_t(wrapi(z_begin - 4 + e, n)) * nn;
        double *dst = yring + size_t(e % DEPTH) * C::Y_ELEMS;
#pragma unroll
        for (int k = 0; k < C::NCY; ++k)
            if (ysrc[k] >= 0) cp_async16(dst + ydst[k], src + ysrc[k]);
    };
#pragma unroll 1
    for (int e = 0; e < DEPTH; ++e) {
        if (e < E) issue(e);
        cp_async_commit();
    }
    int e_next = DEPTH;

    // nu of the two stages of this kernel: (1, 2) for K_A, (3, 4) for K_B
    const long long row = (*a.nu_pos + a.j_local) * 4;
    const double nuA = a.nu_tab[row + (KB == K_A ? 0 : 2)];
    const double nuB = a.nu_tab[row + (KB == K_A ? 1 : 3)];
    // folded weights (C3): L = w0 y + sum_a [wp2 y+2 + wp1 y+1 + wm1 y-1 + wm2 y-2]
    double wp2[3], wp1[3], wm1[3], wm2[3];
    const double alA = nuA * a.inv_dx * a.inv_dx / 12.0, alB = nuB * a.inv_dx * a.inv_dx / 12.0;
    const double w0A = -90.0 * alA, w0B = -90.0 * alB;
    double be[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) be[d] = a.c[d] * a.inv_dx / 12.0;
    // the advection part is the same in both stages, the diffusion part scales with nu
    const double dt = a.dt;

    // stage-A item: column cA of the extended region, rows rA0 .. rA0+3
    const bool actA = t < C::A_ITEMS;
    const int cA = t % EW, rA0 = (t / EW) * RPT;
    // stage-B item: column cB of the tile, rows rB0 .. rB0+3
    const bool actB = t < C::B_ITEMS;
    const int cB = t % TXO, rB0 = (t / TXO) * RPT;

    // K_B: the base field u on the extended points and acc on the tile points
    // are read from global memory one iteration ahead into registers.
    int uoffA[RPT];
    const int uxA = wrapi(x0 - 2 + cA, n);
#pragma unroll
    for (int r = 0; r < RPT; ++r) uoffA[r] = wrapi(y0 - 2 + rA0 + r, n) * n + uxA;
    double ubase[RPT], accp[RPT];
    auto prefetch_u = [&](int j) {  // base for stage-A plane j (physical z_begin-2+j)
        const double *src = a.p0 + size_t(wrapi(z_begin - 2 + j, n)) * nn;
#pragma unroll
        for (int r = 0; r < RPT; ++r) ubase[r] = src[uoffA[r]];
    };
    auto prefetch_acc = [&](int i) {  // acc of output plane i
        const double *src = a.p1 + size_t(z_begin + i) * nn + size_t(y0 + rB0) * n + x0 + cB;
#pragma unroll
        for (int r = 0; r < RPT; ++r) accp[r] = src[size_t(r) * n];
    };
    if (KB == K_B) {
        if (actA) prefetch_u(0);
    }

    double qa[RPT][5], qb[RPT][5];
    // initial stage-A queue: input elements 0..3
    cp_async_wait<DEPTH - 4>();
    __syncthreads();
    const int sA = (rA0 + 2) * IW + cA + 2;  // centre of the first row, input plane
    const int sB = (rB0 + 2) * EW + cB + 2;  // centre of the first row, Ya plane
    if (actA) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double *ys = yring + size_t(e) * C::Y_ELEMS + sA;
#pragma unroll
            for (int r = 0; r < RPT; ++r) qa[r][e] = ys[r * IW];
        }
    }
    double *o0 = a.o0 + size_t(z_begin) * nn + size_t(y0 + rB0) * n + x0 + cB;
    double *o1 = KB == K_A ? a.o1 + size_t(z_begin) * nn + size_t(y0 + rB0) * n + x0 + cB : nullptr;

#pragma unroll 1
    for (int j = 0; j < NJ; ++j) {
        if (j + 4 >= DEPTH + 2) cp_async_wait<DEPTH - 4>();
        else cp_async_wait<DEPTH - 5>();
        __syncthreads();  // input element j+4 visible; iteration j-1 finished with its slots
        while (e_next < E && e_next - DEPTH <= j + 1) issue(e_next++);
        cp_async_commit();

        const int zslot = j % 3;
        if (actA) {  // ---- stage A on the extended region, plane j
            const double *yq = yring + size_t((j + 4) % DEPTH) * C::Y_ELEMS + sA;
#pragma unroll
            for (int r = 0; r < RPT; ++r) qa[r][4] = yq[r * IW];
            const double *ys = yring + size_t((j + 2) % DEPTH) * C::Y_ELEMS + sA;
            double col[RPT + 4];
#pragma unroll
            for (int r = 0; r < RPT + 4; ++r)
                col[r] = (r >= 2 && r < RPT + 2) ? qa[r - 2][2] : ys[(r - 2) * IW];
            double *zs = zring + size_t(zslot) * C::Z_ELEMS + rA0 * EW + cA;
            const bool outp = j >= 2 && j < nz + 2;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const double *yr = ys + r * IW;
                const double yc = qa[r][2];
                double ax = (16.0 * alA + 8.0 * be[0]) * yr[-1];
                ax = fma(16.0 * alA - 8.0 * be[0], yr[1], ax);
                ax = fma(-alA - be[0], yr[-2], ax);
                ax = fma(-alA + be[0], yr[2], ax);
                double ay = (16.0 * alA + 8.0 * be[1]) * col[r + 1];
                ay = fma(16.0 * alA - 8.0 * be[1], col[r + 3], ay);
                ay = fma(-alA - be[1], col[r], ay);
                ay = fma(-alA + be[1], col[r + 4], ay);
                double az = (16.0 * alA + 8.0 * be[2]) * qa[r][1];
                az = fma(16.0 * alA - 8.0 * be[2], qa[r][3], az);
                az = fma(-alA - be[2], qa[r][0], az);
                az = fma(-alA + be[2], qa[r][4], az);
                const double kA = fma(w0A, yc, ax) + (ay + az);
                const double base = KB == K_A ? yc : ubase[r];
                zs[r * EW] = base + (KB == K_A ? dt / 2.0 : dt) * kA;  // Ya or Ya'
                const int er = rA0 + r;
                if (outp && cA >= 2 && cA < TXO + 2 && er >= 2 && er < C::TYO + 2) {
                    double *ts = tring + size_t(zslot) * NTV * C::T_ELEMS + (er - 2) * TXO + (cA - 2);
                    if (KB == K_A) {
                        ts[0] = yc + (dt / 6.0) * kA;   // u + dt/6 k1
                        ts[C::T_ELEMS] = yc;            // u
                    } else {
                        ts[0] = kA;                     // k3
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int o = 0; o < 4; ++o) qa[r][o] = qa[r][o + 1];
        }
        if (KB == K_B && actA && j + 1 < NJ) prefetch_u(j + 1);
        __syncthreads();  // Ya plane j visible
        if (actB) {  // ---- stage B on the tile, output plane j-4
            const double *zq = zring + size_t(zslot) * C::Z_ELEMS + sB;
#pragma unroll
            for (int r = 0; r < RPT; ++r) qb[r][4] = zq[r * EW];
            if (j >= 4) {
                const int i = j - 4;
                const int cslot = (j - 2) % 3;
                const double *zs = zring + size_t(cslot) * C::Z_ELEMS + sB;
                const double *ts = tring + size_t(cslot) * NTV * C::T_ELEMS + rB0 * TXO + cB;
                double col[RPT + 4];
#pragma unroll
                for (int r = 0; r < RPT + 4; ++r)
                    col[r] = (r >= 2 && r < RPT + 2) ? qb[r - 2][2] : zs[(r - 2) * EW];
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double *zr = zs + r * EW;
                    const double zc = qb[r][2];
                    double ax = (16.0 * alB + 8.0 * be[0]) * zr[-1];
                    ax = fma(16.0 * alB - 8.0 * be[0], zr[1], ax);
                    ax = fma(-alB - be[0], zr[-2], ax);
                    ax = fma(-alB + be[0], zr[2], ax);
                    double ay = (16.0 * alB + 8.0 * be[1]) * col[r + 1];
                    ay = fma(16.0 * alB - 8.0 * be[1], col[r + 3], ay);
                    ay = fma(-alB - be[1], col[r], ay);
                    ay = fma(-alB + be[1], col[r + 4], ay);
                    double az = (16.0 * alB + 8.0 * be[2]) * qb[r][1];
                    az = fma(16.0 * alB - 8.0 * be[2], qb[r][3], az);
                    az = fma(-alB - be[2], qb[r][0], az);
                    az = fma(-alB + be[2], qb[r][4], az);
                    const double kB = fma(w0B, zc, ax) + (ay + az);
                    const size_t g = size_t(r) * n;
                    if (KB == K_A) {
                        o0[g] = ts[r * TXO] + (dt / 3.0) * kB;                 // acc
                        o1[g] = ts[C::T_ELEMS + r * TXO] + (dt / 2.0) * kB;    // Yb
                    } else {
                        o0[g] = accp[r] + (dt / 3.0) * ts[r * TXO] + (dt / 6.0) * kB;  // u_new
                    }
                }
                o0 += nn;
                if (KB == K_A) o1 += nn;
                (void)i;
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int o = 0; o < 4; ++o) qb[r][o] = qb[r][o + 1];
            if (KB == K_B && j + 1 >= 4 && j + 1 - 4 < nz) prefetch_acc(j + 1 - 4);
        }
    }
    cp_async_wait<0>();
}

}  // namespace prk
