// fast_boundary.cuh -- damping-slab (CPML) update kernels, MM_MODE_FAST.
//
// ref: update_damping_pass2 (propagator_impl.hpp:125-152) and
//      update_damping_pass1 (propagator_impl.hpp:106-123).
//
// k_bnd: the interior kernel's warp-specialised 2.5D TMA pipeline over the six
// slab boxes (grid.cpp:34-41), cut into 32 x 16 tiles (two x-points per
// consumer thread, 8 consumer warps + 1 producer warp, two CTAs per SM).
// Besides the p_cur ring and the p_prev / c tiles, the producer streams the
// CPML memory each tile needs:
//   psi_x box (x halo), zeta_x      -- X-slab tiles
//   psi_y box(es) (y halo), zeta_y  -- X/Y-slab tiles near a y damping run
//   psi_z tile with the p_cur plane (z window through a register queue),
//   zeta_z                          -- planes in a z damping run
// The run arrays are the reference's per-slab zero-halo boxes, so TMA's
// out-of-bounds zero fill IS the reference's zero halo (cpml.hpp:77-99).
// New zeta values go out with plain global stores.
//
// k_pass1: psi = b psi + a D1(p_cur) over the damping runs, 4 x-points per
// thread, a z register queue for the runs along z.
#pragma once

#include "fast_common.cuh"

namespace mmb {
namespace fast {

template <int R>
struct BndCfg {
    static constexpr int PX = 2;         // x-points per consumer thread (float2)
    static constexpr int TXT = 16;
    static constexpr int TX = PX * TXT;  // 32
    // 7 consumer warps + 1 producer: 8 warps (a 4-warp register granule
    // multiple), 128 registers, two CTAs per SM.  14 rows also tile the
    // 27-row Y slabs (2 x 14) with little waste.
    static constexpr int TR = 14;
    static constexpr int TY = TR;        // one row per thread
    static constexpr int NC = TXT * TR;  // 224 consumer threads
    static constexpr int NCW = NC / 32;
    static constexpr int NT = NC + 32;   // + producer warp
    static constexpr int HX = R <= 4 ? 4 : 8;
    static constexpr int BX = TX + 2 * HX;
    static constexpr int BY = TY + 2 * R;
    static constexpr int QW = 2 * R + 1;
    static constexpr int D = 3;
    static constexpr int NS = R + 1 + D;
    static constexpr int NQ = 3;
    static constexpr int QLEAD = NQ - 1;
    // *_N: floats a TMA box delivers; unsuffixed: 128-byte-padded region size
    static constexpr int PPLANE_N = BX * BY, PPLANE = pad32(PPLANE_N);  // p_cur halo plane
    static constexpr int ZT_N = TX * TY, ZT = pad32(ZT_N);              // psi_z tile
    static constexpr int TILE_N = TX * TY, TILE = pad32(TILE_N);
    static constexpr int PSX_N = BX * TY, PSX = pad32(PSX_N);  // psi_x box (x halo)
    static constexpr int PSY_N = TX * BY, PSY = pad32(PSY_N);  // psi_y box (y halo)
    // stage layout: pp | cv | psx | zx | psy_lo | psy_hi | zy | zz
    static constexpr int O_PP = 0, O_CV = TILE, O_PSX = 2 * TILE, O_ZX = O_PSX + PSX,
                         O_PSY0 = O_ZX + TILE, O_PSY1 = O_PSY0 + PSY, O_ZY = O_PSY1 + PSY,
                         O_ZZ = O_ZY + TILE, QSTAGE = O_ZZ + TILE;
    static constexpr int RSLOT = PPLANE + ZT;
    static constexpr int NBAR = 2 * NS + 2 * NQ + 4;
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(NS * RSLOT + NQ * QSTAGE) + 8 * NBAR + 64;
};

struct BndMaps {
    CUtensorMap pc, pp, cv;
    CUtensorMap psi[3][2];
    CUtensorMap zeta[3][2];
};

struct BndBox {
    int lo[3], hi[3];
    int kind;  // 0 = X slab, 1 = Y slab, 2 = Z slab
    int side;  // 0 = low slab, 1 = high slab
    int x_base;
};

struct BndParams {
    Layout lay;
    BndBox box[6];
    int nbox;
    CpmlRun run[3][2];  // lo/hi/org (local), zeta pointers and strides
    const float* ta[3];
    const float* tb[3];
    const float* tik[3];
    float c2[3][kMaxR], c1[3][kMaxR];
    float* pn;
    const int4* segs;   // items (box | tile_x << 3, tile_y, z_begin, z_end)
    WorkQueue wq;
};

__device__ __forceinline__ bool in_run(const CpmlRun& r, int l) { return l >= r.lo && l < r.hi; }
__device__ __forceinline__ bool near_run(const CpmlRun& r, int a, int b) {
    return r.hi > r.lo && a < r.hi && b > r.lo;  // [a, b) meets the run
}
__device__ __forceinline__ float2 lds2(const float* p) {
    return *reinterpret_cast<const float2*>(p);
}
__device__ __forceinline__ float c2of(const float2& v, int e) { return e == 0 ? v.x : v.y; }
__device__ __forceinline__ void mbar_arrive_b(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Per-tile CPML configuration, computed identically by producer and consumers.
template <int R>
struct TileCfg {
    int x0, y0, zb, ze, nring, nout;
    int xside, zyside;
    bool fx, fy0, fy1;
    BndBox B;
    __device__ TileCfg(const BndParams& P, const int4& sg) {
        using C = BndCfg<R>;
        B = P.box[sg.x & 7];
        x0 = B.x_base + (sg.x >> 3) * C::TX;
        y0 = B.lo[1] + sg.y * C::TY;
        zb = sg.z;
        ze = sg.w;
        nring = ze - zb + 2 * R;
        nout = ze - zb;
        xside = B.kind == 0 ? B.side : -1;
        fx = xside >= 0 && P.run[0][xside].hi > P.run[0][xside].lo;
        const bool usey = B.kind <= 1;  // dpsi_y only in X and Y slabs
        fy0 = usey && near_run(P.run[1][0], y0 - R, y0 + C::TY + R);
        fy1 = usey && near_run(P.run[1][1], y0 - R, y0 + C::TY + R);
        zyside = near_run(P.run[1][0], y0, y0 + C::TY)   ? 0
                 : near_run(P.run[1][1], y0, y0 + C::TY) ? 1
                                                         : -1;
    }
};

__device__ __forceinline__ int zrun_of(const BndParams& P, int z) {
    return in_run(P.run[2][0], z) ? 0 : in_run(P.run[2][1], z) ? 1 : -1;
}

template <int R, int ORD>
// Register cap for two CTAs of 8 warps per SM (see k_inner).
__global__ void __maxnreg__(128)
    k_bnd(const __grid_constant__ BndMaps M, const BndParams P) {
    using C = BndCfg<R>;
    constexpr int PX = C::PX;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NS * C::RSLOT;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + C::NQ * C::QSTAGE);
    int4* items = reinterpret_cast<int4*>(bars + C::NBAR);
    const uint32_t fullP = smem_u32(bars), emptyP = fullP + 8 * C::NS;
    const uint32_t fullQ = emptyP + 8 * C::NS, emptyQ = fullQ + 8 * C::NQ;
    const uint32_t fullI = emptyQ + 8 * C::NQ, emptyI = fullI + 16;
    const int tid = threadIdx.x;
    const int warp = tid / 32, lane = tid % 32;
    const Layout L = P.lay;

    if (tid == 0) {
        for (int s = 0; s < C::NS; ++s) {
            mbar_init(fullP + 8 * s, 1);
            mbar_init(emptyP + 8 * s, C::NCW);
        }
        for (int s = 0; s < C::NQ; ++s) {
            mbar_init(fullQ + 8 * s, 1);
            mbar_init(emptyQ + 8 * s, C::NCW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(fullI + 8 * s, 1);
            mbar_init(emptyI + 8 * s, C::NCW);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == C::NCW) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            unsigned np = 0, nq = 0, ni = 0;
            for (;;) {
                const int item = atomicAdd(P.wq.ctr, 1);
                const int4 sg = item < P.wq.nitems ? P.segs[item] : make_int4(0, 0, 0, -1);
                {
                    const int s = ni & 1;
                    mbar_wait(emptyI + 8 * s, ((ni >> 1) & 1) ^ 1);
                    items[s] = sg;
                    mbar_arrive_b(fullI + 8 * s);
                    ++ni;
                }
                if (sg.w < 0) break;
                const TileCfg<R> T(P, sg);
                const uint32_t qfixed =
                    4u * (2 * C::TILE_N + (T.fx ? C::PSX_N + C::TILE_N : 0) +
                          (T.fy0 ? C::PSY_N : 0) + (T.fy1 ? C::PSY_N : 0) +
                          (T.zyside >= 0 ? C::TILE_N : 0));
                auto issue_q = [&](int o) {
                    const int z = T.zb + o;
                    const int s = nq % C::NQ;
                    mbar_wait(emptyQ + 8 * s, ((nq / C::NQ) & 1) ^ 1);
                    const uint32_t bar = fullQ + 8 * s;
                    float* dst = qring + s * C::QSTAGE;
                    const int zr = zrun_of(P, z);
                    mbar_expect_tx(bar, qfixed + (zr >= 0 ? 4u * C::TILE_N : 0u));
                    tma_load_3d(smem_u32(dst + C::O_PP), &M.pp, L.L + T.x0, T.y0 + L.r, z + L.r,
                                bar);
                    tma_load_3d(smem_u32(dst + C::O_CV), &M.cv, L.L + T.x0, T.y0 + L.r, z + L.r,
                                bar);
                    if (T.fx) {
                        const int org = P.run[0][T.xside].org;  // multiple of 4
                        tma_load_3d(smem_u32(dst + C::O_PSX), &M.psi[0][T.xside],
                                    T.x0 - org - C::HX, T.y0, z, bar);
                        tma_load_3d(smem_u32(dst + C::O_ZX), &M.zeta[0][T.xside], T.x0 - org,
                                    T.y0, z, bar);
                    }
                    if (T.fy0)
                        tma_load_3d(smem_u32(dst + C::O_PSY0), &M.psi[1][0], T.x0,
                                    T.y0 - R - P.run[1][0].org, z, bar);
                    if (T.fy1)
                        tma_load_3d(smem_u32(dst + C::O_PSY1), &M.psi[1][1], T.x0,
                                    T.y0 - R - P.run[1][1].org, z, bar);
                    if (T.zyside >= 0)
                        tma_load_3d(smem_u32(dst + C::O_ZY), &M.zeta[1][T.zyside], T.x0,
                                    T.y0 - P.run[1][T.zyside].org, z, bar);
                    if (zr >= 0)
                        tma_load_3d(smem_u32(dst + C::O_ZZ), &M.zeta[2][zr], T.x0, T.y0,
                                    z - P.run[2][zr].org, bar);
                    ++nq;
                };
                int oq = 0;
                for (int j = 0; j < T.nring; ++j) {
                    const int z = T.zb - R + j;
                    const int zr = zrun_of(P, z);
                    const int s = np % C::NS;
                    mbar_wait(emptyP + 8 * s, ((np / C::NS) & 1) ^ 1);
                    const uint32_t bar = fullP + 8 * s;
                    float* dst = ring + s * C::RSLOT;
                    mbar_expect_tx(bar, 4u * (C::PPLANE_N + (zr >= 0 ? C::ZT_N : 0)));
                    tma_load_3d(smem_u32(dst), &M.pc, L.L + T.x0 - C::HX, T.y0 - R + L.r, z + L.r,
                                bar);
                    if (zr >= 0)
                        tma_load_3d(smem_u32(dst + C::PPLANE), &M.psi[2][zr], T.x0, T.y0,
                                    z - P.run[2][zr].org, bar);
                    ++np;
                    for (; oq < T.nout && oq <= j - 2 * R + C::QLEAD; ++oq) issue_q(oq);
                }
                for (; oq < T.nout; ++oq) issue_q(oq);
            }
            __threadfence();
            if (atomicAdd(P.wq.ctr + 1, 1) == (int)gridDim.x - 1) {
                atomicExch(P.wq.ctr, 0);
                atomicExch(P.wq.ctr + 1, 0);
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const int soff = (R + ty) * C::BX + C::HX + PX * tx;  // in the p_cur plane
    const int toff = ty * C::TX + PX * tx;                 // in a tile
    unsigned np = 0, nq = 0, ni = 0;

    for (;;) {
        int4 sg;
        {
            const int s = ni & 1;
            mbar_wait(fullI + 8 * s, (ni >> 1) & 1);
            sg = items[s];
            __syncwarp();
            if (lane == 0) mbar_arrive_b(emptyI + 8 * s);
            ++ni;
        }
        if (sg.w < 0) break;
        const TileCfg<R> T(P, sg);
        const bool fx = T.fx, fy0 = T.fy0, fy1 = T.fy1;
        const int xside = T.xside, zyside = T.zyside;

        // --- per-thread constants for this item
        const int xg = T.x0 + PX * tx;
        const int y = T.y0 + ty;
        bool pok[PX];  // point inside the box
        float axa[PX], axb[PX], axk[PX];
#pragma unroll
        for (int e = 0; e < PX; ++e) {
            const int x = xg + e;
            pok[e] = x >= T.B.lo[0] && x < T.B.hi[0] && y >= T.B.lo[1] && y < T.B.hi[1];
            const int xc = min(max(x, 0), L.n[0] - 1);
            axa[e] = __ldg(P.ta[0] + xc);
            axb[e] = __ldg(P.tb[0] + xc);
            axk[e] = __ldg(P.tik[0] + xc);
        }
        const int yc = min(max(y, 0), L.n[1] - 1);
        const float aya = __ldg(P.ta[1] + yc), ayb = __ldg(P.tb[1] + yc),
                    ayk = __ldg(P.tik[1] + yc);
        const bool y_in_zy = zyside >= 0 && in_run(P.run[1][zyside], y);
        float* dst_base = P.pn + L.off(xg, y, T.zb);
        float* zx_base =
            fx ? P.run[0][xside].zeta + run_off(P.run[0][xside], 0, xg, y, T.zb) : nullptr;
        float* zy_base =
            y_in_zy ? P.run[1][zyside].zeta + run_off(P.run[1][zyside], 1, xg, y, T.zb) : nullptr;
        const long long zx_step = fx ? P.run[0][xside].s2 : 0;
        const long long zy_step = y_in_zy ? P.run[1][zyside].s2 : 0;

        // register queues of p_cur and psi_z along z: q[k] holds plane j-2R+k
        float2 q[C::QW];
        float2 qz[C::QW];
#pragma unroll 1
        for (int j = 0; j < T.nring; ++j) {
            const int s = np % C::NS;
            mbar_wait(fullP + 8 * s, (np / C::NS) & 1);
#pragma unroll
            for (int k = 0; k < C::QW - 1; ++k) {
                q[k] = q[k + 1];
                qz[k] = qz[k + 1];
            }
            {
                const float* S = ring + s * C::RSLOT;
                q[C::QW - 1] = lds2(S + soff);
                qz[C::QW - 1] = zrun_of(P, T.zb - R + j) >= 0 ? lds2(S + C::PPLANE + toff)
                                                              : make_float2(0.f, 0.f);
            }
            const int cs = (np + C::NS - R) % C::NS;  // slot of plane j - R
            if (j >= 2 * R) {
                const int o = j - 2 * R;
                const int z = T.zb + o;
                const float* S = ring + cs * C::RSLOT + soff;
                const int st = nq % C::NQ;
                mbar_wait(fullQ + 8 * st, (nq / C::NQ) & 1);
                const float* Q = qring + st * C::QSTAGE;
                const int zr = zrun_of(P, z);
                const float aza = __ldg(P.ta[2] + z), azb = __ldg(P.tb[2] + z),
                            azk = __ldg(P.tik[2] + z);
                // x neighbours of p: columns c-HX .. c+PX-1+HX
                float xs[PX + 2 * C::HX];
#pragma unroll
                for (int h = 0; h < C::HX / 2; ++h) {
                    const float2 lft = lds2(S - C::HX + 2 * h);
                    const float2 rgt = lds2(S + PX + 2 * h);
                    xs[2 * h] = lft.x;
                    xs[2 * h + 1] = lft.y;
                    xs[C::HX + PX + 2 * h] = rgt.x;
                    xs[C::HX + PX + 2 * h + 1] = rgt.y;
                }
                xs[C::HX] = q[R].x;
                xs[C::HX + 1] = q[R].y;
                float2 yu[R], yd[R];
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    yu[m - 1] = lds2(S + m * C::BX);
                    yd[m - 1] = lds2(S - m * C::BX);
                }
                const float2 pp = lds2(Q + C::O_PP + toff);
                const float2 cv = lds2(Q + C::O_CV + toff);
                // CPML inputs: dpsi per axis for both points
                float dpx[PX] = {0.f, 0.f}, dpy[PX] = {0.f, 0.f}, dpz[PX] = {0.f, 0.f};
                if (fx) {
                    const float* px = Q + C::O_PSX + ty * C::BX + C::HX + PX * tx;
                    float ps[PX + 2 * C::HX];
#pragma unroll
                    for (int h = 0; h < (PX + 2 * C::HX) / 2; ++h) {
                        const float2 v = lds2(px - C::HX + 2 * h);
                        ps[2 * h] = v.x;
                        ps[2 * h + 1] = v.y;
                    }
#pragma unroll
                    for (int e = 0; e < PX; ++e)
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            dpx[e] = acc<ORD>(dpx[e], P.c1[0][m - 1],
                                              fs<ORD>(ps[C::HX + e + m], ps[C::HX + e - m]));
                }
                if (fy0 || fy1) {
                    const float* p0y = Q + C::O_PSY0 + (R + ty) * C::TX + PX * tx;
                    const float* p1y = Q + C::O_PSY1 + (R + ty) * C::TX + PX * tx;
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        float2 up = make_float2(0.f, 0.f), dn = up;
                        if (fy0) {
                            const float2 a = lds2(p0y + m * C::TX), b = lds2(p0y - m * C::TX);
                            up.x += a.x;
                            up.y += a.y;
                            dn.x += b.x;
                            dn.y += b.y;
                        }
                        if (fy1) {
                            const float2 a = lds2(p1y + m * C::TX), b = lds2(p1y - m * C::TX);
                            up.x += a.x;
                            up.y += a.y;
                            dn.x += b.x;
                            dn.y += b.y;
                        }
                        dpy[0] = acc<ORD>(dpy[0], P.c1[1][m - 1], fs<ORD>(up.x, dn.x));
                        dpy[1] = acc<ORD>(dpy[1], P.c1[1][m - 1], fs<ORD>(up.y, dn.y));
                    }
                }
                float2 zx = make_float2(0.f, 0.f), zy = zx, zz = zx;
                if (fx) zx = lds2(Q + C::O_ZX + toff);
                if (y_in_zy) zy = lds2(Q + C::O_ZY + toff);
                if (zr >= 0) zz = lds2(Q + C::O_ZZ + toff);
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyQ + 8 * st);  // stage fully read
                ++nq;
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    dpz[0] = acc<ORD>(dpz[0], P.c1[2][m - 1], fs<ORD>(qz[R + m].x, qz[R - m].x));
                    dpz[1] = acc<ORD>(dpz[1], P.c1[2][m - 1], fs<ORD>(qz[R + m].y, qz[R - m].y));
                }
                float out[PX], nzx[PX], nzy[PX], nzz[PX];
#pragma unroll
                for (int e = 0; e < PX; ++e) {
                    const float p0 = xs[C::HX + e];
                    const float two_p0 = 2.0f * p0;
                    float d2x = 0.f, d2y = 0.f, d2z = 0.f;
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        d2x = d2_term<ORD>(d2x, P.c2[0][m - 1], xs[C::HX + e + m],
                                           xs[C::HX + e - m], two_p0);
                        d2y = d2_term<ORD>(d2y, P.c2[1][m - 1], c2of(yu[m - 1], e),
                                           c2of(yd[m - 1], e), two_p0);
                        d2z = d2_term<ORD>(d2z, P.c2[2][m - 1], c2of(q[R + m], e),
                                           c2of(q[R - m], e), two_p0);
                    }
                    // reference: drive = d2p*ik + dpsi; zeta = b*zeta + a*drive;
                    // term = drive + zeta; lap = (term_x + term_y) + term_z
                    const float drx = acc<ORD>(dpx[e], d2x, axk[e]);
                    const float dry = acc<ORD>(dpy[e], d2y, ayk);
                    const float drz = acc<ORD>(dpz[e], d2z, azk);
                    nzx[e] = fx ? acc<ORD>(fm<ORD>(axa[e], drx), axb[e], c2of(zx, e)) : 0.f;
                    nzy[e] = y_in_zy ? acc<ORD>(fm<ORD>(aya, dry), ayb, c2of(zy, e)) : 0.f;
                    nzz[e] = zr >= 0 ? acc<ORD>(fm<ORD>(aza, drz), azb, c2of(zz, e)) : 0.f;
                    const float lap = fa<ORD>(fa<ORD>(fa<ORD>(drx, nzx[e]), fa<ORD>(dry, nzy[e])),
                                              fa<ORD>(drz, nzz[e]));
                    out[e] = acc<ORD>(fs<ORD>(two_p0, c2of(pp, e)), c2of(cv, e), lap);
                }
                // stores: p_next for points inside the box, zeta where a run holds them
                float* dst = dst_base + (long long)o * L.plane;
                float* dzz = zr >= 0 ? P.run[2][zr].zeta + run_off(P.run[2][zr], 2, xg, y, z)
                                     : nullptr;
#pragma unroll
                for (int e = 0; e < PX; ++e) {
                    if (!pok[e]) continue;
                    dst[e] = out[e];
                    if (fx) zx_base[(long long)o * zx_step + e] = nzx[e];
                    if (y_in_zy) zy_base[(long long)o * zy_step + e] = nzy[e];
                    if (zr >= 0) dzz[e] = nzz[e];
                }
            }
            if (j >= R) {  // plane j - R has had its last use
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyP + 8 * cs);
            }
            ++np;
        }
#pragma unroll 1
        for (int k = R; k >= 1; --k) {  // planes that never became centres
            __syncwarp();
            if (lane == 0) mbar_arrive_b(emptyP + 8 * ((np + C::NS - k) % C::NS));
        }
    }
}

// ---------------------------------------------------------------- pass 1
// One block = one damping run x an x-y tile of 32 x 32 points x a z-chunk.
// Four x-points per thread (float4); p_cur through L1, z runs through a
// register queue along z; loads of the next planes are unrolled for ILP.
struct RunDesc {
    int ax, side;
    int lo[3], hi[3];  // box of points the run covers (local coordinates)
    int x_base;        // multiple of 4 (absolute x; run org is a multiple of 4)
};

template <int R, int ORD>
__global__ void __launch_bounds__(256)
    k_pass1(const StepParams p, const RunDesc* runs, const int4* items, int nitems) {
    const int it = blockIdx.x;
    if (it >= nitems) return;
    const int4 itm = items[it];  // (run | tile_x << 4, tile_y, z_begin, z_end)
    const RunDesc rd = runs[itm.x & 15];
    const int ax = rd.ax;
    const CpmlRun run = p.run[ax][rd.side];
    const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;
    const int x = rd.x_base + (itm.x >> 4) * 32 + 4 * tx;
    const int y = rd.lo[1] + itm.y * 32 + ty;
    if (y >= rd.hi[1] || x >= rd.hi[0]) return;
    const int zb = itm.z, ze = itm.w;
    const Layout& L = p.lay;
    bool ok[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) ok[e] = x + e >= rd.lo[0] && x + e < rd.hi[0];
    const bool all = ok[0] && ok[1] && ok[2] && ok[3];
    float c1[R];
#pragma unroll
    for (int m = 0; m < R; ++m) c1[m] = p.c1[ax][m];
    float av[4] = {0.f, 0.f, 0.f, 0.f}, bv[4] = {1.f, 1.f, 1.f, 1.f};
    if (ax == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (ok[e]) {
                av[e] = __ldg(p.ta[0] + x + e);
                bv[e] = __ldg(p.tb[0] + x + e);
            }
    } else if (ax == 1) {
        const float a = __ldg(p.ta[1] + y), b = __ldg(p.tb[1] + y);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            av[e] = a;
            bv[e] = b;
        }
    }
    auto update = [&](float* ps, const float (&dp)[4], const float (&a)[4], const float (&b)[4]) {
        if (all) {
            float4 v = *reinterpret_cast<float4*>(ps);
            // reference: psi = b * psi + a * dp
            v.x = acc<ORD>(fm<ORD>(a[0], dp[0]), b[0], v.x);
            v.y = acc<ORD>(fm<ORD>(a[1], dp[1]), b[1], v.y);
            v.z = acc<ORD>(fm<ORD>(a[2], dp[2]), b[2], v.z);
            v.w = acc<ORD>(fm<ORD>(a[3], dp[3]), b[3], v.w);
            *reinterpret_cast<float4*>(ps) = v;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (ok[e]) ps[e] = acc<ORD>(fm<ORD>(a[e], dp[e]), b[e], ps[e]);
        }
    };
    if (ax == 2) {
        float4 qq[2 * R + 1];  // p_cur along z: planes z-R .. z+R
        const float* base = p.pc + L.off(x, y, zb);
#pragma unroll
        for (int k = 0; k < 2 * R; ++k)
            qq[k + 1] = __ldg(reinterpret_cast<const float4*>(base + (long long)(k - R) * L.plane));
#pragma unroll 2
        for (int z = zb; z < ze; ++z) {
#pragma unroll
            for (int k = 0; k < 2 * R; ++k) qq[k] = qq[k + 1];
            qq[2 * R] = __ldg(
                reinterpret_cast<const float4*>(base + (long long)(z - zb + R) * L.plane));
            float dp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 1; m <= R; ++m) {
                dp[0] = acc<ORD>(dp[0], c1[m - 1], fs<ORD>(qq[R + m].x, qq[R - m].x));
                dp[1] = acc<ORD>(dp[1], c1[m - 1], fs<ORD>(qq[R + m].y, qq[R - m].y));
                dp[2] = acc<ORD>(dp[2], c1[m - 1], fs<ORD>(qq[R + m].z, qq[R - m].z));
                dp[3] = acc<ORD>(dp[3], c1[m - 1], fs<ORD>(qq[R + m].w, qq[R - m].w));
            }
            const float az = __ldg(p.ta[2] + z), bz = __ldg(p.tb[2] + z);
            const float a4[4] = {az, az, az, az}, b4[4] = {bz, bz, bz, bz};
            update(run.psi + run_off(run, 2, x, y, z), dp, a4, b4);
        }
        return;
    }
#pragma unroll 4
    for (int z = zb; z < ze; ++z) {
        const float* c = p.pc + L.off(x, y, z);
        float dp[4] = {0.f, 0.f, 0.f, 0.f};
        if (ax == 0) {
            constexpr int H = 4 * ((R + 3) / 4);
            float v[4 + 2 * H];
#pragma unroll
            for (int h = 0; h < (4 + 2 * H) / 4; ++h) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(c - H + 4 * h));
                v[4 * h] = t.x;
                v[4 * h + 1] = t.y;
                v[4 * h + 2] = t.z;
                v[4 * h + 3] = t.w;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int m = 1; m <= R; ++m)
                    dp[e] = acc<ORD>(dp[e], c1[m - 1], fs<ORD>(v[H + e + m], v[H + e - m]));
            update(run.psi + run_off(run, 0, x, y, z), dp, av, bv);
        } else {
#pragma unroll
            for (int m = 1; m <= R; ++m) {
                const float4 u = __ldg(reinterpret_cast<const float4*>(c + m * L.P));
                const float4 d = __ldg(reinterpret_cast<const float4*>(c - m * L.P));
                dp[0] = acc<ORD>(dp[0], c1[m - 1], fs<ORD>(u.x, d.x));
                dp[1] = acc<ORD>(dp[1], c1[m - 1], fs<ORD>(u.y, d.y));
                dp[2] = acc<ORD>(dp[2], c1[m - 1], fs<ORD>(u.z, d.z));
                dp[3] = acc<ORD>(dp[3], c1[m - 1], fs<ORD>(u.w, d.w));
            }
            update(run.psi + run_off(run, 1, x, y, z), dp, av, bv);
        }
    }
}

}  // namespace fast
}  // namespace mmb
