// vd_fast.cuh -- TMA-fed z-streaming kernels of the acoustic_iso engine.
//
// ref: AcousticVdEngine::update_velocity / update_pressure
// (propagator_impl.hpp:214-273), staggered_derivative_at (stencil.hpp:103-111).
//
// Both kernels are persistent (one CTA per resident slot) and pull
// (x-y tile, z-chunk) items from a work queue ordered chunk-major, so the
// items in flight are neighbouring tiles at the same depth and their halos
// meet in L2.  A tile is 32 x 32 points; a thread owns 4 consecutive x points
// (one float4) of one row.
//  * k_vdv (velocity): p planes with their x-y halo arrive by TMA into a ring
//    of NS = 2R + lead slots that holds the whole z window; every neighbour
//    of the staggered forward derivative is a shared-memory load.
//  * k_vdp (pressure): vz tiles stream through a ring the same way (z
//    window); vx with its x halo and vy with its y halo arrive per plane in a
//    two-stage ring.
//  * point-wise streams (dt/rho, v in k_vdv; dt*bulk, p in k_vdp) arrive by
//    TMA in a stage ring a few planes ahead and are written back with 16-byte
//    stores; CPML memory (the damping-layer runs) moves as float4 loads issued
//    at the top of a plane.
//  * thread 0 issues the TMA loads after the per-plane barrier.
// Arithmetic: the reference's association order, every operation rounded
// separately (__fadd_rn / __fmul_rn): bit-identical to the CPU reference.
#pragma once

#include "fast_common.cuh"

namespace mmb {
namespace vdk {

using fast::comp;
using fast::lds4;
using fast::pad32;
using fast::smem_u32;

__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
// lane pairs (FADD2 / FFMA2 with an opaque -0, fast_common.cuh): each lane
// rounded like the scalar operation
using fast::F2;
using fast::f2;
using fast::half2;
using fast::unf2;
// t + w * (a - b), both lanes (staggered_derivative_at's term)
__device__ __forceinline__ F2 dterm2(F2 t, float w, F2 a, F2 b) {
    return fast::acc2<2>(t, w, fast::fs2<2>(a, b));
}
// x + c * y lane-wise
__device__ __forceinline__ F2 axpy2(F2 x, F2 c, F2 y) {
    return fast::fa2<2>(x, fast::fmul2<2>(c, y));
}
__device__ __forceinline__ void unpack(const F2 (&v)[2], float (&d)[4]) {
    unf2(v[0], d[0], d[1]);
    unf2(v[1], d[2], d[3]);
}

template <int R>
struct VdCfg {
    static constexpr int TXT = 8;          // threads per row, 4 x-points each
    static constexpr int TX = 4 * TXT;     // 32
#ifndef MM_VD_TY
#define MM_VD_TY 32
#endif
    static constexpr int TY = MM_VD_TY;    // rows (one per thread row)
    static constexpr int NT = TXT * TY;    // 256
    static constexpr int MINB = TY >= 32 ? 2 : 4;  // CTAs per SM the registers allow
    static constexpr int HX = R <= 4 ? 4 : 8;  // x halo (float4 granules)
    static constexpr int BX = TX + 2 * HX;
    static constexpr int BY = TY + 2 * R;
    static constexpr int TILE = pad32(TX * TY);
    // velocity: p halo planes, ring = z window 2R + lead
    static constexpr int PPLANE = pad32(BX * BY);
#ifndef MM_VD_LEADV
#define MM_VD_LEADV 1
#endif
#ifndef MM_VD_NQV
#define MM_VD_NQV 3
#endif
#ifndef MM_VD_LEADP
#define MM_VD_LEADP 2
#endif
#ifndef MM_VD_NQP
#define MM_VD_NQP 3
#endif
    static constexpr int NSV = 2 * R + MM_VD_LEADV;
    static constexpr int NQV = R <= 4 ? MM_VD_NQV : 2;  // dt/rho + v stages
    // pressure: vz tiles (z window 2R + lead), vx / vy halo boxes + dtb + p (NQ stages)
    static constexpr int NSP = 2 * R + MM_VD_LEADP;
    static constexpr int NQP = MM_VD_NQP;
    static constexpr int VXB = pad32(BX * TY), VYB = pad32(TX * BY);
    static constexpr size_t SMEM_V =
        sizeof(float) * (size_t)(NSV * PPLANE + NQV * 4 * TILE) + 8 * (NSV + NQV) + 16;
    static constexpr size_t SMEM_P = sizeof(float) * (size_t)(NSP * TILE + NQP * (VXB + VYB + 2 * TILE)) +
                                     8 * (NSP + NQP) + 16;
};

struct VdTables {
    const float* ta[3];
    const float* tb[3];
    const float* tik[3];
};

struct VdFastParams {
    Layout lay;
    int nd[3];
    float* p;
    float* v[3];
    const float* ir;   // dt / rho
    const float* dtb;  // dt * ((rho * vp) * vp)
    float w[3][kMaxR];
    VdTables tab;
    CpmlRun run[3][2];  // psi of this pass
    const int4* items;  // (tile_x, tile_y, z_begin, z_end)
    fast::WorkQueue wq;
};

// CPML memory of one axis for one thread's 4 points: the run array element
// of point 0 at the item's first plane, the per-plane step, and which of the
// 4 points lie in the run.
struct RunPtr {
    float* p;  // nullptr: no point of the thread in this run
    long long step;
    bool on[4];
    bool all;
};

// One thread's 4 points: masks, CPML tables and run pointers of the item.
struct PointSet {
    int xg, y;
    bool ok[4], all, any;
    float xa[4], xb[4], xk[4], ya, yb, yk;
    RunPtr rx[2], ry;
};

__device__ __forceinline__ void run_ptr(RunPtr& rp, const CpmlRun& r, int ax, int xg, int y,
                                        int zb, const bool (&ok)[4]) {
    rp.p = nullptr;
    rp.step = 0;
    rp.all = true;
    bool any = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int c = ax == 0 ? xg + e : y;
        rp.on[e] = ok[e] && c >= r.lo && c < r.hi;
        any = any || rp.on[e];
        rp.all = rp.all && rp.on[e];
    }
    if (any) {
        rp.p = r.psi + run_off(r, ax, xg, y, zb);
        rp.step = r.s2;
    }
}

template <int R>
__device__ __forceinline__ void point_set(PointSet& S, const VdFastParams& P, int x0, int y0,
                                          int tx, int ty, int zb) {
    const Layout& L = P.lay;
    S.xg = x0 + 4 * tx;
    S.y = y0 + ty;
    const bool yok = S.y < L.n[1];
    S.all = yok;
    S.any = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        S.ok[e] = yok && S.xg + e < L.n[0];
        S.all = S.all && S.ok[e];
        S.any = S.any || S.ok[e];
        const int xc = min(S.xg + e, L.n[0] - 1);
        S.xa[e] = __ldg(P.tab.ta[0] + xc);
        S.xb[e] = __ldg(P.tab.tb[0] + xc);
        S.xk[e] = __ldg(P.tab.tik[0] + xc);
    }
    const int yc = min(S.y, L.n[1] - 1);
    S.ya = __ldg(P.tab.ta[1] + yc);
    S.yb = __ldg(P.tab.tb[1] + yc);
    S.yk = __ldg(P.tab.tik[1] + yc);
    run_ptr(S.rx[0], P.run[0][0], 0, S.xg, S.y, zb, S.ok);
    run_ptr(S.rx[1], P.run[0][1], 0, S.xg, S.y, zb, S.ok);
    run_ptr(S.ry, P.run[1][0], 1, S.xg, S.y, zb, S.ok);
    if (!S.ry.p) run_ptr(S.ry, P.run[1][1], 1, S.xg, S.y, zb, S.ok);
}

// CPML (propagator_impl.hpp:231-238 / :260-267): psi = b psi + a d;
// d = d ik + psi, on the points of each damping-layer run.  Points outside
// every run of an axis have a = 0, b = ik = 1 there: their psi stays +0 and d
// is unchanged for the update (v and p never hold -0), so they are skipped
// (see vd_engine.cu).  The old psi values are loaded at the top of a plane
// (psi_load) so their latency hides behind the stencil; psi_apply finishes.
struct PsiState {
    float ox[4], oy[4], oz[4];
    float* pz;  // z-run element of point 0 at this plane (nullptr: none)
};

__device__ __forceinline__ void ld_run(float (&old)[4], const float* ps, const bool (&on)[4],
                                       bool all) {
    if (all) {
        const float4 v = *reinterpret_cast<const float4*>(ps);
        old[0] = v.x, old[1] = v.y, old[2] = v.z, old[3] = v.w;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (on[e]) old[e] = ps[e];
    }
}
__device__ __forceinline__ void st_run(float* ps, const float (&nw)[4], const bool (&on)[4],
                                       bool all) {
    if (all) {
        *reinterpret_cast<float4*>(ps) = make_float4(nw[0], nw[1], nw[2], nw[3]);
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (on[e]) ps[e] = nw[e];
    }
}

__device__ __forceinline__ void psi_load(PsiState& st, const VdFastParams& P, const PointSet& S,
                                         int o, int k) {
#pragma unroll
    for (int e = 0; e < 4; ++e) st.ox[e] = st.oy[e] = st.oz[e] = 0.0f;
#pragma unroll
    for (int sd = 0; sd < 2; ++sd)
        if (S.rx[sd].p) ld_run(st.ox, S.rx[sd].p + o * S.rx[sd].step, S.rx[sd].on, S.rx[sd].all);
    if (S.ry.p) ld_run(st.oy, S.ry.p + o * S.ry.step, S.ry.on, S.ry.all);
    st.pz = nullptr;
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
        const CpmlRun& r = P.run[2][sd];
        if (S.any && k >= r.lo && k < r.hi) st.pz = r.psi + run_off(r, 2, S.xg, S.y, k);
    }
    if (st.pz) ld_run(st.oz, st.pz, S.ok, S.all);
}

__device__ __forceinline__ void psi_step(float (&d)[4], float (&nw)[4], const float (&old)[4],
                                         const bool (&on)[4], const float (&a)[4],
                                         const float (&b)[4], const float (&ik)[4]) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        nw[e] = fa(fm(b[e], old[e]), fm(a[e], d[e]));
        if (on[e]) d[e] = fa(fm(d[e], ik[e]), nw[e]);
    }
}

__device__ __forceinline__ void psi_apply(float (&d)[3][4], const PsiState& st,
                                          const VdFastParams& P, const PointSet& S, int o,
                                          int k) {
    float nw[4];
    if (S.rx[0].p || S.rx[1].p) {
        bool on[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) on[e] = S.rx[0].on[e] || S.rx[1].on[e];
        psi_step(d[0], nw, st.ox, on, S.xa, S.xb, S.xk);
#pragma unroll
        for (int sd = 0; sd < 2; ++sd)
            if (S.rx[sd].p) st_run(S.rx[sd].p + o * S.rx[sd].step, nw, S.rx[sd].on, S.rx[sd].all);
    }
    if (S.ry.p) {
        const float a[4] = {S.ya, S.ya, S.ya, S.ya}, b[4] = {S.yb, S.yb, S.yb, S.yb},
                    ik[4] = {S.yk, S.yk, S.yk, S.yk};
        psi_step(d[1], nw, st.oy, S.ry.on, a, b, ik);
        st_run(S.ry.p + o * S.ry.step, nw, S.ry.on, S.ry.all);
    }
    if (st.pz) {
        const float za = __ldg(P.tab.ta[2] + k), zb = __ldg(P.tab.tb[2] + k),
                    zk = __ldg(P.tab.tik[2] + k);
        const float a[4] = {za, za, za, za}, b[4] = {zb, zb, zb, zb}, ik[4] = {zk, zk, zk, zk};
        psi_step(d[2], nw, st.oz, S.ok, a, b, ik);
        st_run(st.pz, nw, S.ok, S.all);
    }
}

__device__ __forceinline__ void st4v(float* p, const float (&v)[4], const PointSet& S) {
    fast::st4(p, v, S.ok, S.all);
}

// ----------------------------------------------------------------- velocity
// maps: p (BX x BY halo box), dt/rho and vx, vy, vz (TX x TY tiles)
struct VdvMaps {
    CUtensorMap p, ir, vx, vy, vz;
};

template <int R>
__global__ void __launch_bounds__(VdCfg<R>::NT, VdCfg<R>::MINB)
    k_vdv(const __grid_constant__ VdvMaps M, const VdFastParams P) {
    using C = VdCfg<R>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NSV * C::PPLANE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + C::NQV * 4 * C::TILE);
    const uint32_t bar0 = smem_u32(bars), barQ = smem_u32(bars + C::NSV);
    const int tid = threadIdx.x;
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const Layout L = P.lay;
    if (tid == 0) {
        fast::prefetch_tmap(&M.p);
        fast::prefetch_tmap(&M.ir);
        fast::prefetch_tmap(&M.vx);
        fast::prefetch_tmap(&M.vy);
        fast::prefetch_tmap(&M.vz);
        for (int s = 0; s < C::NSV + C::NQV; ++s) fast::mbar_init(bar0 + 8 * s, 1);
        fast::fence_barrier_init();
    }
    __syncthreads();
    uint32_t ph = 0, phQ = 0;  // parity bit per slot / stage
    unsigned qn = 0;           // stages consumed so far
    __shared__ int s_item;
    const int soff = (R + ty) * C::BX + C::HX + 4 * tx;
    const int toff = ty * C::TX + 4 * tx;

    for (;;) {
        const int item = fast::wq_next(P.wq, &s_item);
        if (item >= P.wq.nitems) break;
        const int4 it = P.items[item];
        const int x0 = it.x * C::TX, y0 = it.y * C::TY, zb = it.z, ze = it.w;
        const int nout = ze - zb;
        const int nring = nout + 2 * R - 1;  // planes zb-R+1 .. ze+R-1
        auto issue = [&](int j) {
            const int s = j % C::NSV;
            const uint32_t bar = bar0 + 8 * s;
            fast::mbar_expect_tx(bar, 4u * C::BX * C::BY);
            fast::tma_load_3d(smem_u32(ring + s * C::PPLANE), &M.p, L.L + x0 - C::HX,
                              y0 - R + L.r, zb - R + 1 + j + L.r, bar);
        };
        const unsigned qbase = qn;
        auto issue_q = [&](int o) {
            const int st = (qbase + o) % C::NQV;
            const uint32_t bar = barQ + 8 * st;
            float* dst = qring + st * 4 * C::TILE;
            const int zz = zb + o + L.r, xx = L.L + x0, yy = y0 + L.r;
            fast::mbar_expect_tx(bar, 4u * 4 * C::TX * C::TY);
            fast::tma_load_3d(smem_u32(dst), &M.ir, xx, yy, zz, bar);
            fast::tma_load_3d(smem_u32(dst + C::TILE), &M.vx, xx, yy, zz, bar);
            fast::tma_load_3d(smem_u32(dst + 2 * C::TILE), &M.vy, xx, yy, zz, bar);
            fast::tma_load_3d(smem_u32(dst + 3 * C::TILE), &M.vz, xx, yy, zz, bar);
        };
        if (tid == 0) {
            for (int j = 0; j < min(C::NSV, nring); ++j) issue(j);
            for (int o = 0; o < min(C::NQV, nout); ++o) issue_q(o);
        }
        PointSet S;
        point_set<R>(S, P, x0, y0, tx, ty, zb);
        const long long o0 = L.off(S.xg, S.y, zb);
        for (int j = 0; j < 2 * R - 1; ++j) {
            fast::mbar_wait(bar0 + 8 * (j % C::NSV), (ph >> (j % C::NSV)) & 1u);
            ph ^= 1u << (j % C::NSV);
        }
        for (int o = 0; o < nout; ++o) {
            const int k = zb + o;
            PsiState ps;
            psi_load(ps, P, S, o, k);
            const int jn = o + 2 * R - 1;  // newest plane of the window
            fast::mbar_wait(bar0 + 8 * (jn % C::NSV), (ph >> (jn % C::NSV)) & 1u);
            ph ^= 1u << (jn % C::NSV);
            const int c = (o + R - 1) % C::NSV;  // slot of plane k
            const float* Sc = ring + c * C::PPLANE + soff;
            float d[3][4];
            // x: t += c_m (p[x+m] - p[x+1-m])
            {
                float xs[4 + 2 * C::HX];
#pragma unroll
                for (int h = 0; h < (4 + 2 * C::HX) / 4; ++h) {
                    const float4 v = lds4(Sc - C::HX + 4 * h);
#pragma unroll
                    for (int e = 0; e < 4; ++e) xs[4 * h + e] = comp(v, e);
                }
                F2 t[2] = {fast::f2zero(), fast::f2zero()};
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        t[h] = dterm2(t[h], P.w[0][m - 1],
                                      f2(xs[C::HX + 2 * h + m], xs[C::HX + 2 * h + 1 + m]),
                                      f2(xs[C::HX + 2 * h + 1 - m], xs[C::HX + 2 * h + 2 - m]));
                unpack(t, d[0]);
            }
            // y: rows y+m and y+1-m
            {
                F2 t[2] = {fast::f2zero(), fast::f2zero()};
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float4 u = lds4(Sc + m * C::BX), dn = lds4(Sc + (1 - m) * C::BX);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        t[h] = dterm2(t[h], P.w[1][m - 1], half2(u, h), half2(dn, h));
                }
                unpack(t, d[1]);
            }
            // z: planes k+m <-> ring plane o+R-1+m, k+1-m <-> o+R-m
            {
                F2 t[2] = {fast::f2zero(), fast::f2zero()};
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float4 u = lds4(ring + ((o + R - 1 + m) % C::NSV) * C::PPLANE + soff);
                    const float4 dn = lds4(ring + ((o + R - m) % C::NSV) * C::PPLANE + soff);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        t[h] = dterm2(t[h], P.w[2][m - 1], half2(u, h), half2(dn, h));
                }
                unpack(t, d[2]);
            }
            const int st = qn % C::NQV;
            fast::mbar_wait(barQ + 8 * st, (phQ >> st) & 1u);
            phQ ^= 1u << st;
            ++qn;
            if (S.any) {
                psi_apply(d, ps, P, S, o, k);
                const float* Q = qring + st * 4 * C::TILE + toff;
                const float4 ir = lds4(Q);
                const long long oo = o0 + (long long)o * L.plane;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const float4 v = lds4(Q + (a + 1) * C::TILE);
                    float out[4];
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        unf2(axpy2(half2(v, h), half2(ir, h), f2(d[a][2 * h], d[a][2 * h + 1])),
                             out[2 * h], out[2 * h + 1]);
                    st4v(P.v[a] + oo, out, S);
                }
            }
            __syncthreads();  // plane o (the window's oldest) and stage o are free
            if (tid == 0) {
                if (o + C::NSV < nring) issue(o + C::NSV);
                if (o + C::NQV < nout) issue_q(o + C::NQV);
            }
        }
    }
    fast::wq_done(P.wq);
}

// ----------------------------------------------------------------- pressure
// maps: vx (BX x TY, x halo), vy (TX x BY, y halo), vz, dtb, p (TX x TY tiles)
struct VdpMaps {
    CUtensorMap vx, vy, vz, dtb, p;
};

template <int R>
__global__ void __launch_bounds__(VdCfg<R>::NT, VdCfg<R>::MINB)
    k_vdp(const __grid_constant__ VdpMaps M, const VdFastParams P) {
    using C = VdCfg<R>;
    constexpr int QST = C::VXB + C::VYB + 2 * C::TILE;  // floats per stage
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NSP * C::TILE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + C::NQP * QST);
    const uint32_t barZ = smem_u32(bars), barQ = smem_u32(bars + C::NSP);
    const int tid = threadIdx.x;
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const Layout L = P.lay;
    if (tid == 0) {
        fast::prefetch_tmap(&M.vx);
        fast::prefetch_tmap(&M.vy);
        fast::prefetch_tmap(&M.vz);
        fast::prefetch_tmap(&M.dtb);
        fast::prefetch_tmap(&M.p);
        for (int s = 0; s < C::NSP + C::NQP; ++s) fast::mbar_init(barZ + 8 * s, 1);
        fast::fence_barrier_init();
    }
    __syncthreads();
    uint32_t phZ = 0, phQ = 0;
    unsigned qn = 0;
    __shared__ int s_item;
    const int toff = ty * C::TX + 4 * tx;
    const int xoff = ty * C::BX + C::HX + 4 * tx;  // in a vx box
    const int yoff = (R + ty) * C::TX + 4 * tx;    // in a vy box

    for (;;) {
        const int item = fast::wq_next(P.wq, &s_item);
        if (item >= P.wq.nitems) break;
        const int4 it = P.items[item];
        const int x0 = it.x * C::TX, y0 = it.y * C::TY, zb = it.z, ze = it.w;
        const int nout = ze - zb;
        const int nring = nout + 2 * R - 1;  // vz planes zb-R .. ze+R-2
        auto issue_z = [&](int j) {
            const int s = j % C::NSP;
            const uint32_t bar = barZ + 8 * s;
            fast::mbar_expect_tx(bar, 4u * C::TX * C::TY);
            fast::tma_load_3d(smem_u32(ring + s * C::TILE), &M.vz, L.L + x0, y0 + L.r,
                              zb - R + j + L.r, bar);
        };
        const unsigned qbase = qn;
        auto issue_q = [&](int o) {
            const int st = (qbase + o) % C::NQP;
            const uint32_t bar = barQ + 8 * st;
            float* dst = qring + st * QST;
            const int zz = zb + o + L.r;
            fast::mbar_expect_tx(bar, 4u * (C::BX * C::TY + C::TX * C::BY + 2 * C::TX * C::TY));
            fast::tma_load_3d(smem_u32(dst), &M.vx, L.L + x0 - C::HX, y0 + L.r, zz, bar);
            fast::tma_load_3d(smem_u32(dst + C::VXB), &M.vy, L.L + x0, y0 - R + L.r, zz, bar);
            fast::tma_load_3d(smem_u32(dst + C::VXB + C::VYB), &M.dtb, L.L + x0, y0 + L.r, zz,
                              bar);
            fast::tma_load_3d(smem_u32(dst + C::VXB + C::VYB + C::TILE), &M.p, L.L + x0,
                              y0 + L.r, zz, bar);
        };
        if (tid == 0) {
            for (int j = 0; j < min(C::NSP, nring); ++j) issue_z(j);
            for (int o = 0; o < min(C::NQP, nout); ++o) issue_q(o);
        }
        PointSet S;
        point_set<R>(S, P, x0, y0, tx, ty, zb);
        const long long o0 = L.off(S.xg, S.y, zb);
        for (int j = 0; j < 2 * R - 1; ++j) {
            fast::mbar_wait(barZ + 8 * (j % C::NSP), (phZ >> (j % C::NSP)) & 1u);
            phZ ^= 1u << (j % C::NSP);
        }
        for (int o = 0; o < nout; ++o) {
            const int k = zb + o;
            PsiState ps;
            psi_load(ps, P, S, o, k);
            const int jn = o + 2 * R - 1;
            fast::mbar_wait(barZ + 8 * (jn % C::NSP), (phZ >> (jn % C::NSP)) & 1u);
            phZ ^= 1u << (jn % C::NSP);
            const int st = qn % C::NQP;
            fast::mbar_wait(barQ + 8 * st, (phQ >> st) & 1u);
            phQ ^= 1u << st;
            ++qn;
            const float* Q = qring + st * QST;
            float d[3][4];
            // x: t += c_m (vx[x+m-1] - vx[x-m])
            {
                float xs[4 + 2 * C::HX];
#pragma unroll
                for (int h = 0; h < (4 + 2 * C::HX) / 4; ++h) {
                    const float4 v = lds4(Q + xoff - C::HX + 4 * h);
#pragma unroll
                    for (int e = 0; e < 4; ++e) xs[4 * h + e] = comp(v, e);
                }
                F2 t[2] = {fast::f2zero(), fast::f2zero()};
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        t[h] = dterm2(t[h], P.w[0][m - 1],
                                      f2(xs[C::HX + 2 * h + m - 1], xs[C::HX + 2 * h + m]),
                                      f2(xs[C::HX + 2 * h - m], xs[C::HX + 2 * h + 1 - m]));
                unpack(t, d[0]);
            }
            // y: rows y+m-1 and y-m
            {
                F2 t[2] = {fast::f2zero(), fast::f2zero()};
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float4 u = lds4(Q + C::VXB + yoff + (m - 1) * C::TX);
                    const float4 dn = lds4(Q + C::VXB + yoff - m * C::TX);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        t[h] = dterm2(t[h], P.w[1][m - 1], half2(u, h), half2(dn, h));
                }
                unpack(t, d[1]);
            }
            // z: planes k+m-1 <-> ring plane o+R+m-1, k-m <-> o+R-m
            {
                F2 t[2] = {fast::f2zero(), fast::f2zero()};
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float4 u = lds4(ring + ((o + R + m - 1) % C::NSP) * C::TILE + toff);
                    const float4 dn = lds4(ring + ((o + R - m) % C::NSP) * C::TILE + toff);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        t[h] = dterm2(t[h], P.w[2][m - 1], half2(u, h), half2(dn, h));
                }
                unpack(t, d[2]);
            }
            if (S.any) {
                psi_apply(d, ps, P, S, o, k);
                const float4 dt = lds4(Q + C::VXB + C::VYB + toff);
                const float4 pc = lds4(Q + C::VXB + C::VYB + C::TILE + toff);
                float out[4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const F2 sum = fast::fa2<2>(
                        fast::fa2<2>(f2(d[0][2 * h], d[0][2 * h + 1]), f2(d[1][2 * h], d[1][2 * h + 1])),
                        f2(d[2][2 * h], d[2][2 * h + 1]));
                    unf2(axpy2(half2(pc, h), half2(dt, h), sum), out[2 * h], out[2 * h + 1]);
                }
                st4v(P.p + o0 + (long long)o * L.plane, out, S);
            }
            __syncthreads();  // vz plane o and stage o are free
            if (tid == 0) {
                if (o + C::NSP < nring) issue_z(o + C::NSP);
                if (o + C::NQP < nout) issue_q(o + C::NQP);
            }
        }
    }
    fast::wq_done(P.wq);
}

}  // namespace vdk
}  // namespace mmb
