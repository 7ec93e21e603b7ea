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
    // p_cur ring: the 2R+1-plane z window plus producer lead; a power of two
    // so that slot arithmetic is a mask
    static constexpr int NS = R <= 4 ? 16 : 32;
    // *_N: floats a TMA box delivers; unsuffixed: 128-byte-padded region size
    static constexpr int PPLANE_N = BX * BY, PPLANE = pad32(PPLANE_N);  // p_cur halo plane
    static constexpr int TILE_N = TX * TY, TILE = pad32(TILE_N);
    static constexpr int PSX_N = BX * TY, PSX = pad32(PSX_N);  // psi_x box (x halo)
    static constexpr int PSY_N = TX * BY, PSY = pad32(PSY_N);  // psi_y box (y halo)
    static constexpr int RSLOT = PPLANE;
    // Per-plane stages (pp | cv | the CPML regions the tile needs, see QLay)
    // are carved out of a QB-float circular buffer, so light tiles (Z slabs:
    // 4 tiles) run many stages ahead and heavy ones (X slabs: up to 9) fewer.
    static constexpr int NQD = 8;  // stage barriers: at most NQD stages in flight
    static constexpr int NBAR = 2 * NS + 2 * NQD + 4;
    static constexpr int BUDGET = 112 * 1024;  // bytes per CTA: two CTAs per SM
    static constexpr int QB_RAW = (BUDGET - 4 * NS * RSLOT - 8 * NBAR - 4 * NQD - 64) / 4;
    static constexpr int QB = QB_RAW > 32 ? QB_RAW / 32 * 32 : 32;
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(NS * RSLOT + QB) + 8 * NBAR + 4 * NQD + 64;
};

struct BndMaps {
    CUtensorMap pc, pp, cv;
    CUtensorMap psi[3][2];
    CUtensorMap zeta[3][2];
    CUtensorMap dpz[2];  // dpsi_z of the z runs (written by k_p1)
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
    int dz_lo[2], dz_hi[2];  // planes [lo-R, hi+R) of each z run holding dpsi_z
};

__device__ __forceinline__ bool in_run(const CpmlRun& r, int l) { return l >= r.lo && l < r.hi; }
__device__ __forceinline__ bool near_run(const CpmlRun& r, int a, int b) {
    return r.hi > r.lo && a < r.hi && b > r.lo;  // [a, b) meets the run
}
__device__ __forceinline__ float2 lds2(const float* p) {
    return *reinterpret_cast<const float2*>(p);
}
__device__ __forceinline__ float c2of(const float2& v, int e) { return e == 0 ? v.x : v.y; }

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
// z run whose dpsi_z planes hold z (the ranges never overlap: see kernels_fast.cu)
__device__ __forceinline__ int zext_of(const BndParams& P, int z) {
    return z >= P.dz_lo[0] && z < P.dz_hi[0] ? 0 : z >= P.dz_lo[1] && z < P.dz_hi[1] ? 1 : -1;
}

// Stage layout of a tile: pp | cv | psi_x box | zeta_x | psi_y lo | psi_y hi |
// zeta_y (each only if the tile needs it), then per plane zeta_z | dpsi_z.
struct QLay {
    int o_psx, o_zx, o_psy0, o_psy1, o_zy, fixed;
    uint32_t bytes;  // TMA bytes of the fixed part
};
template <int R>
__device__ __forceinline__ QLay qlay(const TileCfg<R>& T) {
    using C = BndCfg<R>;
    QLay q;
    int o = 2 * C::TILE, b = 2 * C::TILE_N;
    q.o_psx = o;
    if (T.fx) o += C::PSX, b += C::PSX_N;
    q.o_zx = o;
    if (T.fx) o += C::TILE, b += C::TILE_N;
    q.o_psy0 = o;
    if (T.fy0) o += C::PSY, b += C::PSY_N;
    q.o_psy1 = o;
    if (T.fy1) o += C::PSY, b += C::PSY_N;
    q.o_zy = o;
    if (T.zyside >= 0) o += C::TILE, b += C::TILE_N;
    q.fixed = o;
    q.bytes = 4u * b;
    return q;
}
// Circular stage allocation (identical on both sides): a stage never wraps.
__device__ __forceinline__ uint32_t q_alloc(uint32_t& V, int size, int qb) {
    uint32_t v = V;
    const uint32_t r = v % qb;
    if (r + size > (uint32_t)qb) v += qb - r;
    V = v + size;
    return v;
}

#ifndef MM_BND_MAXREG
#define MM_BND_MAXREG 128
#endif
template <int R, int ORD>
// Register cap for two CTAs of 8 warps per SM (see k_inner).
__global__ void __maxnreg__(MM_BND_MAXREG)
    k_bnd(const __grid_constant__ BndMaps M, const BndParams P) {
    using C = BndCfg<R>;
    constexpr int PX = C::PX;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NS * C::RSLOT;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + C::QB);
    int4* items = reinterpret_cast<int4*>(bars + C::NBAR);
    uint32_t* qv = reinterpret_cast<uint32_t*>(items + 2);  // producer: stage starts
    const uint32_t fullP = smem_u32(bars), emptyP = fullP + 8 * C::NS;
    const uint32_t fullQ = emptyP + 8 * C::NS, emptyQ = fullQ + 8 * C::NQD;
    const uint32_t fullI = emptyQ + 8 * C::NQD, emptyI = fullI + 16;
    const int tid = threadIdx.x;
    const int warp = tid / 32, lane = tid % 32;
    const Layout L = P.lay;

    if (tid == 0) {
        for (int s = 0; s < C::NS; ++s) {
            mbar_init(fullP + 8 * s, 1);
            mbar_init(emptyP + 8 * s, C::NCW);
        }
        for (int s = 0; s < C::NQD; ++s) {
            mbar_init(fullQ + 8 * s, 1);
            mbar_init(emptyQ + 8 * s, C::NCW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(fullI + 8 * s, 1);
            mbar_init(emptyI + 8 * s, C::NCW + 1);  // consumer warps + stage lane
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == C::NCW) {
        // ------------------------------------------------------------ producers
        // lane 0: work items + the p_cur ring; lane 1: the per-plane stages.
        // Two lanes keep two independent TMA issue streams in flight.
        if (lane == 0) {
            unsigned np = 0, ni = 0;
            for (;;) {
                const int item = atomicAdd(P.wq.ctr, 1);
                const int4 sg = item < P.wq.nitems ? P.segs[item] : make_int4(0, 0, 0, -1);
                {
                    const int s = ni & 1;
                    mbar_wait_sleep(emptyI + 8 * s, ((ni >> 1) & 1) ^ 1);
                    items[s] = sg;
                    mbar_arrive_b(fullI + 8 * s);
                    ++ni;
                }
                if (sg.w < 0) break;
                const TileCfg<R> T(P, sg);
                for (int j = 0; j < T.nring; ++j) {
                    const int s = np & (C::NS - 1);
                    mbar_wait_sleep(emptyP + 8 * s, ((np / C::NS) & 1) ^ 1);
                    const uint32_t bar = fullP + 8 * s;
#ifdef MM_BND_NOP  // experiment: no p_cur traffic
                    mbar_arrive_b(bar);
                    ++np;
                    continue;
#endif
                    mbar_expect_tx(bar, 4u * C::PPLANE_N);
                    tma_load_3d(smem_u32(ring + s * C::RSLOT), &M.pc, L.L + T.x0 - C::HX,
                                T.y0 - R + L.r, T.zb - R + j + L.r, bar);
                    ++np;
                }
            }
            __threadfence();
            if (atomicAdd(P.wq.ctr + 1, 1) == (int)gridDim.x - 1) {
                atomicExch(P.wq.ctr, 0);
                atomicExch(P.wq.ctr + 1, 0);
            }
        } else if (lane == 1) {
            unsigned nq = 0, qtail = 0, ni = 0;
            uint32_t V = 0;
            for (;;) {
                int4 sg;
                {
                    const int s = ni & 1;
                    mbar_wait(fullI + 8 * s, (ni >> 1) & 1);
                    sg = items[s];
                    mbar_arrive_b(emptyI + 8 * s);
                    ++ni;
                }
                if (sg.w < 0) break;
                const TileCfg<R> T(P, sg);
                const QLay ql = qlay<R>(T);
                for (int oq = 0; oq < T.nout; ++oq) {
                    const int z = T.zb + oq;
                    const int zr = zrun_of(P, z);
                    const int ze = zext_of(P, z);
                    const int size = ql.fixed + (zr >= 0 ? C::TILE : 0) + (ze >= 0 ? C::TILE : 0);
                    const uint32_t vn = q_alloc(V, size, C::QB);
                    // free: stage nq - NQD (barrier reuse) and every stage whose space
                    // the new one overlaps (stages are released in order)
                    while (qtail < nq &&
                           (nq - qtail >= (unsigned)C::NQD || qv[qtail % C::NQD] + C::QB < vn + size)) {
                        mbar_wait_sleep(emptyQ + 8 * (qtail % C::NQD), (qtail / C::NQD) & 1);
                        ++qtail;
                    }
                    qv[nq % C::NQD] = vn;
                    const uint32_t bar = fullQ + 8 * (nq % C::NQD);
                    float* dst = qring + vn % C::QB;
#ifdef MM_BND_NOQ  // experiment: no stage traffic
                    mbar_arrive_b(bar);
                    ++nq;
                    continue;
#endif
                    mbar_expect_tx(bar, ql.bytes + (zr >= 0 ? 4u * C::TILE_N : 0u) +
                                            (ze >= 0 ? 4u * C::TILE_N : 0u));
                    tma_load_3d(smem_u32(dst), &M.pp, L.L + T.x0, T.y0 + L.r, z + L.r, bar);
                    tma_load_3d(smem_u32(dst + C::TILE), &M.cv, L.L + T.x0, T.y0 + L.r, z + L.r,
                                bar);
                    if (T.fx) {
                        const int org = P.run[0][T.xside].org;  // multiple of 4
                        tma_load_3d(smem_u32(dst + ql.o_psx), &M.psi[0][T.xside],
                                    T.x0 - org - C::HX, T.y0, z, bar);
                        tma_load_3d(smem_u32(dst + ql.o_zx), &M.zeta[0][T.xside], T.x0 - org,
                                    T.y0, z, bar);
                    }
                    if (T.fy0)
                        tma_load_3d(smem_u32(dst + ql.o_psy0), &M.psi[1][0], T.x0,
                                    T.y0 - R - P.run[1][0].org, z, bar);
                    if (T.fy1)
                        tma_load_3d(smem_u32(dst + ql.o_psy1), &M.psi[1][1], T.x0,
                                    T.y0 - R - P.run[1][1].org, z, bar);
                    if (T.zyside >= 0)
                        tma_load_3d(smem_u32(dst + ql.o_zy), &M.zeta[1][T.zyside], T.x0,
                                    T.y0 - P.run[1][T.zyside].org, z, bar);
                    if (zr >= 0)
                        tma_load_3d(smem_u32(dst + ql.fixed), &M.zeta[2][zr], T.x0, T.y0,
                                    z - P.run[2][zr].org, bar);
                    if (ze >= 0)
                        tma_load_3d(smem_u32(dst + ql.fixed + (zr >= 0 ? C::TILE : 0)),
                                    &M.dpz[ze], T.x0, T.y0, z - P.dz_lo[ze], bar);
                    ++nq;
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const int soff = (R + ty) * C::BX + C::HX + PX * tx;  // in the p_cur plane
    const int toff = ty * C::TX + PX * tx;                 // in a tile
    unsigned np = 0, nq = 0, ni = 0;
    uint32_t V = 0;  // stage allocator, in step with the producer's

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
        const QLay ql = qlay<R>(T);
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

        // The whole z window (planes j-2R .. j) stays resident in the ring:
        // z neighbours of p_cur and psi_z are read from shared memory.
#pragma unroll 1
        for (int j = 0; j < T.nring; ++j) {
            const int s = np % C::NS;
#ifndef MM_BND_NOWAIT
            mbar_wait(fullP + 8 * s, (np / C::NS) & 1);
#endif
            if (j >= 2 * R) {
                const int o = j - 2 * R;
                const int z = T.zb + o;
                const int cs = (np - R) & (C::NS - 1);  // slot of plane j - R
                auto slot_of = [&](int m) {             // slot of plane j - R + m
                    return (cs + m) & (C::NS - 1);
                };
                const float* S = ring + cs * C::RSLOT + soff;
                float2 zu[R], zd[R];
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    zu[m - 1] = lds2(ring + slot_of(m) * C::RSLOT + soff);
                    zd[m - 1] = lds2(ring + slot_of(-m) * C::RSLOT + soff);
                }
                const int zr = zrun_of(P, z);
                const int zex = zext_of(P, z);
                const int st = nq % C::NQD;
                const float* Q =
                    qring + q_alloc(V, ql.fixed + (zr >= 0 ? C::TILE : 0) + (zex >= 0 ? C::TILE : 0),
                                    C::QB) % C::QB;
#ifndef MM_BND_NOWAIT
                mbar_wait(fullQ + 8 * st, (nq / C::NQD) & 1);
#endif
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
                {
                    const float2 c = lds2(S);
                    xs[C::HX] = c.x;
                    xs[C::HX + 1] = c.y;
                }
                float2 yu[R], yd[R];
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    yu[m - 1] = lds2(S + m * C::BX);
                    yd[m - 1] = lds2(S - m * C::BX);
                }
                const float2 pp = lds2(Q + toff);
                const float2 cv = lds2(Q + C::TILE + toff);
                // CPML inputs: dpsi per axis for both points
                float dpx[PX] = {0.f, 0.f}, dpy[PX] = {0.f, 0.f}, dpz[PX] = {0.f, 0.f};
                if (fx) {
                    const float* px = Q + ql.o_psx + ty * C::BX + C::HX + PX * tx;
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
                    const float* p0y = Q + ql.o_psy0 + (R + ty) * C::TX + PX * tx;
                    const float* p1y = Q + ql.o_psy1 + (R + ty) * C::TX + PX * tx;
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
                if (fx) zx = lds2(Q + ql.o_zx + toff);
                if (y_in_zy) zy = lds2(Q + ql.o_zy + toff);
                if (zr >= 0) zz = lds2(Q + ql.fixed + toff);
                // dpsi_z (k_p1); +0 where no psi_z reaches the window
                if (zex >= 0) {
                    const float2 v = lds2(Q + ql.fixed + (zr >= 0 ? C::TILE : 0) + toff);
                    dpz[0] = v.x;
                    dpz[1] = v.y;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyQ + 8 * st);  // stage fully read
                ++nq;
                float out[PX], nzx[PX], nzy[PX], nzz[PX];
#pragma unroll
                for (int e = 0; e < PX; ++e) {
                    const float p0 = xs[C::HX + e];
#ifdef MM_BND_NOFP  // experiment: the data pipeline without the arithmetic
                    nzx[e] = c2of(zx, e);
                    nzy[e] = c2of(zy, e);
                    nzz[e] = c2of(zz, e);
                    out[e] = p0 + xs[e] + xs[C::HX + e + 4] + c2of(yu[R - 1], e) +
                             c2of(yd[R - 1], e) + c2of(zu[R - 1], e) + c2of(zd[R - 1], e) +
                             dpx[e] + dpy[e] + dpz[e] + c2of(pp, e) + c2of(cv, e) + axk[e] + ayk + azk;
                    continue;
#endif
                    const float two_p0 = 2.0f * p0;
                    float d2x = 0.f, d2y = 0.f, d2z = 0.f;
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        d2x = d2_term<ORD>(d2x, P.c2[0][m - 1], xs[C::HX + e + m],
                                           xs[C::HX + e - m], two_p0);
                        d2y = d2_term<ORD>(d2y, P.c2[1][m - 1], c2of(yu[m - 1], e),
                                           c2of(yd[m - 1], e), two_p0);
                        d2z = d2_term<ORD>(d2z, P.c2[2][m - 1], c2of(zu[m - 1], e),
                                           c2of(zd[m - 1], e), two_p0);
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
#ifdef MM_BND_NOST
                    if (out[e] == 12345.f) dst[e] = out[e];
                    continue;
#endif
                    dst[e] = out[e];
                    if (fx) zx_base[(long long)o * zx_step + e] = nzx[e];
                    if (y_in_zy) zy_base[(long long)o * zy_step + e] = nzy[e];
                    if (zr >= 0) dzz[e] = nzz[e];
                }
                // plane j - 2R has had its last use
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyP + 8 * slot_of(-R));
            }
            ++np;
        }
#pragma unroll 1
        for (int k = 2 * R; k >= 1; --k) {  // the item's last 2R planes
            __syncwarp();
            if (lane == 0) mbar_arrive_b(emptyP + 8 * ((np - k) & (C::NS - 1)));
        }
    }
}

}  // namespace fast
}  // namespace mmb
