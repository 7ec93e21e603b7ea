// fast_boundary.cuh -- damping-slab (CPML pass 2) update kernel, MM_MODE_FAST.
//
// ref: update_damping_pass2 (propagator_impl.hpp:125-152), second_derivative_at
//      / central_derivative_at (stencil.hpp:86-99).
//
// k_bnd: 2.5D streaming along z over the six slab boxes (grid.cpp:34-41), cut
// into 32 x 28 x-y tiles; a consumer thread owns 4 consecutive x points (one
// float4) of one row, seven consumer warps + one producer warp per CTA, two
// CTAs per SM.
//  * producer lane 0: work items + the p_cur ring (TMA, one 40 x 36 halo
//    plane per z); the ring holds the whole 2R+1-plane z window plus lead, so
//    every neighbour of p_cur is a shared-memory load.
//  * producer lane 1: the CPML boxes with a halo the tile needs -- psi_x box
//    (X slabs), psi_y boxes (tiles within R of a y damping run) -- carved out
//    of a circular stage buffer.  The run arrays are the reference's per-slab
//    zero-halo boxes, so TMA's out-of-bounds zero fill IS the reference's zero
//    halo (cpml.hpp:77-99).
//  * the point-wise streams (p_prev, c, zeta_x/y/z, dpsi_z from k_p1) have no
//    reuse; lane 1 stages them by TMA too, per plane, in the same circular
//    stage buffer as the psi boxes (16-byte LDG into registers left the
//    lockstep consumers waiting on the loads: 12 % slower).
//  * new p and zeta go out with 16-byte stores.
#pragma once

#include "fast_common.cuh"

namespace mmb {
namespace fast {

#ifndef MM_BND_NS
#define MM_BND_NS 12
#endif

template <int R>
struct BndCfg {
    static constexpr int PX = 4;         // x points per consumer thread (float4)
    static constexpr int TXT = 8;        // threads per row
    static constexpr int TX = PX * TXT;  // 32
    // 7 consumer warps x 4 rows: 28 rows also tile the 27-row Y slabs.
#ifndef MM_BND_TY
#define MM_BND_TY 28
#endif
    static constexpr int TY = MM_BND_TY;
    static constexpr int NC = TXT * TY;  // 224 consumer threads
    static constexpr int NCW = NC / 32;
    static constexpr int NT = NC + 32;   // + producer warp
    static constexpr int HX = R <= 4 ? 4 : 8;
    static constexpr int BX = TX + 2 * HX;
    static constexpr int BY = TY + 2 * R;
    // *_N: floats a TMA box delivers; unsuffixed: 128-byte-padded region size
    static constexpr int PPLANE_N = BX * BY, PPLANE = pad32(PPLANE_N);  // p_cur halo plane
    static constexpr int PSX_N = BX * TY, PSX = pad32(PSX_N);           // psi_x box
    static constexpr int PSY_N = TX * BY, PSY = pad32(PSY_N);           // psi_y box
    static constexpr int TILE_N = TX * TY, TILE = pad32(TILE_N);        // p_prev, c tiles
    // p_cur ring: the 2R+1-plane z window plus producer lead
    static constexpr int NS = MM_BND_NS > 2 * R + 1 ? MM_BND_NS : 2 * R + 2;
#ifndef MM_BND_NQD
#define MM_BND_NQD 8
#endif
    static constexpr int NQD = MM_BND_NQD;  // stage barriers: at most NQD stages in flight
    static constexpr int NBAR = 2 * NS + 2 * NQD + 4;
    // bytes per CTA: two CTAs per SM up to R = 4; one (with the registers of
    // two) for wider stencils, whose z window needs a deeper ring
#ifndef MM_BND_CTAS4
#define MM_BND_CTAS4 2
#endif
    static constexpr int CTAS = R <= 4 ? MM_BND_CTAS4 : 1;
    static constexpr int BUDGET = CTAS == 2 ? 112 * 1024 : 220 * 1024;
    static constexpr int MAXREG = CTAS == 2 ? 65536 / (2 * NT) / 8 * 8 : 255;
    static constexpr int QB_RAW = (BUDGET - 4 * NS * PPLANE - 8 * NBAR - 4 * NQD - 64) / 4;
    static constexpr int QMAX = 7 * TILE + PSX + 2 * PSY;
    static constexpr int QB = QB_RAW > QMAX ? QB_RAW / 32 * 32 : QMAX;
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(NS * PPLANE + QB) + 8 * NBAR + 4 * NQD + 64;
};

struct BndMaps {
    CUtensorMap pc;          // p_cur, 40 x 36 halo box
    CUtensorMap pp, cv;      // p_prev, c: 32 x 28 tiles
    CUtensorMap psi[2][2];   // psi_x (x-halo box), psi_y (y-halo box) per side
    CUtensorMap zeta[3][2];  // 32 x 28 tiles of the zeta runs
    CUtensorMap dpz[2];      // 32 x 28 tiles of dpsi_z (k_p1)
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
    const float* pp;
    const float* cv;
    float* pn;
    const int4* segs;  // items (box | tile_x << 3, tile_y, z_begin, z_end)
    WorkQueue wq;
    // dpsi_z of the z runs (k_p1): planes [dz_lo, dz_hi) = [lo-R, hi+R), run strides
    const float* dpz[2];
    int dz_lo[2], dz_hi[2];
};


// Per-tile CPML configuration, computed identically by producer and consumers.
template <int R>
struct TileCfg {
    int x0, y0, zb, ze, nring, nout;
    int xside;
    bool fx, fy0, fy1;
    // stage: pp | cv | psi_x box | psi_y boxes | zeta_x | zeta_y (per run) --
    // the regions the tile needs -- then per plane zeta_z | dpsi_z
    int qsize;
    uint32_t qbytes;
    int o_psx, o_psy0, o_psy1, o_zx, o_zy0, o_zy1;
    bool fzy0, fzy1;  // tile rows in y run 0 / 1
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
        // an X slab spans every y and sees both y runs; a Y slab box holds its
        // own run only (the other is zero halo even within R of it)
        fy0 = usey && (B.kind == 0 || B.side == 0) &&
              near_run(P.run[1][0], y0 - R, y0 + C::TY + R);
        fy1 = usey && (B.kind == 0 || B.side == 1) &&
              near_run(P.run[1][1], y0 - R, y0 + C::TY + R);
        int o = 2 * C::TILE, b = 2 * C::TILE_N;
        o_psx = o;
        if (fx) o += C::PSX, b += C::PSX_N;
        o_psy0 = o;
        if (fy0) o += C::PSY, b += C::PSY_N;
        o_psy1 = o;
        if (fy1) o += C::PSY, b += C::PSY_N;
        o_zx = o;
        if (fx) o += C::TILE, b += C::TILE_N;
        fzy0 = usey && near_run(P.run[1][0], y0, y0 + C::TY);
        fzy1 = usey && near_run(P.run[1][1], y0, y0 + C::TY);
        o_zy0 = o;
        if (fzy0) o += C::TILE, b += C::TILE_N;
        o_zy1 = o;
        if (fzy1) o += C::TILE, b += C::TILE_N;
        qsize = o;
        qbytes = 4u * b;
    }
};

__device__ __forceinline__ int zrun_of(const BndParams& P, int z) {
    return in_run(P.run[2][0], z) ? 0 : in_run(P.run[2][1], z) ? 1 : -1;
}
// z run whose dpsi_z planes hold z (the ranges never overlap: see kernels_fast.cu)
__device__ __forceinline__ int zext_of(const BndParams& P, int z) {
    return z >= P.dz_lo[0] && z < P.dz_hi[0] ? 0 : z >= P.dz_lo[1] && z < P.dz_hi[1] ? 1 : -1;
}
// ... as seen from box B: a Z slab box holds its own z layer only, so the other
// run's dpsi_z (within R of it when the inner z extent is < R) is zero halo there
__device__ __forceinline__ int zext_in(const BndParams& P, int z, const BndBox& B) {
    const int e = zext_of(P, z);
    return B.kind == 2 && e != B.side ? -1 : e;
}
// Circular stage allocation (identical on both sides): a stage never wraps.
__device__ __forceinline__ uint32_t q_alloc(uint32_t& V, int size, int qb) {
    uint32_t v = V;
    const uint32_t r = v % qb;
    if (r + size > (uint32_t)qb) v += qb - r;
    V = v + size;
    return v;
}

template <int R, int ORD>
// Register cap for two CTAs of 8 warps per SM (see k_inner).
__global__ void __maxnreg__(BndCfg<R>::MAXREG)
    k_bnd(const __grid_constant__ BndMaps M, const BndParams P) {
    using C = BndCfg<R>;
    MM_TRACE_BEGIN
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NS * C::PPLANE;
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
        // lane 0: work items + the p_cur ring; lane 1: the psi boxes.
        if (lane == 0) {
            unsigned np = 0, ni = 0;
            unsigned s = 0, ph = 0;  // ring slot of plane np, its pass parity
            for (;;) {
                const int item = atomicAdd(P.wq.ctr, 1);
                const int4 sg = item < P.wq.nitems ? P.segs[item] : make_int4(0, 0, 0, -1);
                {
                    const int si = ni & 1;
                    mbar_wait_sleep(emptyI + 8 * si, ((ni >> 1) & 1) ^ 1);
                    items[si] = sg;
                    mbar_arrive_b(fullI + 8 * si);
                    ++ni;
                }
                if (sg.w < 0) {
                    // the queue is empty: a programmatically launched successor
                    // (the step epilogue) may start while the last items drain
                    grid_dep_launch();
                    break;
                }
                const TileCfg<R> T(P, sg);
                for (int j = 0; j < T.nring; ++j) {
                    mbar_wait_sleep(emptyP + 8 * s, ph ^ 1);
                    const uint32_t bar = fullP + 8 * s;
                    mbar_expect_tx(bar, 4u * C::PPLANE_N);
                    tma_load_3d(smem_u32(ring + s * C::PPLANE), &M.pc, L.L + T.x0 - C::HX,
                                T.y0 - R + L.r, T.zb - R + j + L.r, bar);
                    ++np;
                    if (++s == C::NS) s = 0, ph ^= 1;
                }
            }
            __threadfence();
            if (atomicAdd(P.wq.ctr + 1, 1) == (int)gridDim.x - 1) {
                atomicExch(P.wq.ctr, 0);
                atomicExch(P.wq.ctr + 1, 0);
            }
        } else if (lane == 1) {
            // the stages carry pass-1 results (psi, dpsi_z): with a programmatic
            // launch after k_p1 they wait for it; the p_cur ring (lane 0) does not
            grid_dep_wait();
            unsigned nq = 0, qtail = 0, ni = 0;
            uint32_t V = 0;
            for (;;) {
                int4 sg;
                {
                    const int si = ni & 1;
                    mbar_wait(fullI + 8 * si, (ni >> 1) & 1);
                    sg = items[si];
                    mbar_arrive_b(emptyI + 8 * si);
                    ++ni;
                }
                if (sg.w < 0) break;
                const TileCfg<R> T(P, sg);
                for (int oq = 0; oq < T.nout; ++oq) {
                    const int z = T.zb + oq;
                    const int zr = zrun_of(P, z), ze = zext_in(P, z, T.B);
                    const int size = T.qsize + (zr >= 0 ? C::TILE : 0) + (ze >= 0 ? C::TILE : 0);
                    const uint32_t vn = q_alloc(V, size, C::QB);
                    // free: stage nq - NQD (barrier reuse) and every stage whose space
                    // the new one overlaps (stages are released in order)
                    while (qtail < nq && (nq - qtail >= (unsigned)C::NQD ||
                                          qv[qtail % C::NQD] + C::QB < vn + size)) {
                        mbar_wait_sleep(emptyQ + 8 * (qtail % C::NQD), (qtail / C::NQD) & 1);
                        ++qtail;
                    }
                    qv[nq % C::NQD] = vn;
                    const uint32_t bar = fullQ + 8 * (nq % C::NQD);
                    float* dst = qring + vn % C::QB;
                    mbar_expect_tx(bar, T.qbytes + (zr >= 0 ? 4u * C::TILE_N : 0u) +
                                            (ze >= 0 ? 4u * C::TILE_N : 0u));
                    tma_load_3d(smem_u32(dst), &M.pp, L.L + T.x0, T.y0 + L.r, z + L.r, bar);
                    tma_load_3d(smem_u32(dst + C::TILE), &M.cv, L.L + T.x0, T.y0 + L.r, z + L.r, bar);
                    if (T.fx)
                        tma_load_3d(smem_u32(dst + T.o_psx), &M.psi[0][T.xside],
                                    T.x0 - P.run[0][T.xside].org - C::HX, T.y0, z, bar);
                    if (T.fy0)
                        tma_load_3d(smem_u32(dst + T.o_psy0), &M.psi[1][0], T.x0,
                                    T.y0 - R - P.run[1][0].org, z, bar);
                    if (T.fy1)
                        tma_load_3d(smem_u32(dst + T.o_psy1), &M.psi[1][1], T.x0,
                                    T.y0 - R - P.run[1][1].org, z, bar);
                    if (T.fx)
                        tma_load_3d(smem_u32(dst + T.o_zx), &M.zeta[0][T.xside],
                                    T.x0 - P.run[0][T.xside].org, T.y0, z, bar);
                    if (T.fzy0)
                        tma_load_3d(smem_u32(dst + T.o_zy0), &M.zeta[1][0], T.x0,
                                    T.y0 - P.run[1][0].org, z, bar);
                    if (T.fzy1)
                        tma_load_3d(smem_u32(dst + T.o_zy1), &M.zeta[1][1], T.x0,
                                    T.y0 - P.run[1][1].org, z, bar);
                    if (zr >= 0)
                        tma_load_3d(smem_u32(dst + T.qsize), &M.zeta[2][zr], T.x0, T.y0,
                                    z - P.run[2][zr].org, bar);
                    if (ze >= 0)
                        tma_load_3d(smem_u32(dst + T.qsize + (zr >= 0 ? C::TILE : 0)), &M.dpz[ze],
                                    T.x0, T.y0, z - P.dz_lo[ze], bar);
                    ++nq;
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const int soff = (R + ty) * C::BX + C::HX + 4 * tx;  // in a p_cur plane
    unsigned ni = 0, nq = 0;
    unsigned s = 0, ph = 0;  // ring slot / parity of the next plane to arrive
    int qo = 0;              // stage offset in the circular buffer (the producer's V % QB)

    for (;;) {
        int4 sg;
        {
            const int si = ni & 1;
            mbar_wait(fullI + 8 * si, (ni >> 1) & 1);
            sg = items[si];
            __syncwarp();
            if (lane == 0) mbar_arrive_b(emptyI + 8 * si);
            ++ni;
        }
        if (sg.w < 0) break;
        const TileCfg<R> T(P, sg);
        const bool fx = T.fx, fy0 = T.fy0, fy1 = T.fy1;
        const int xside = T.xside;

        // --- per-thread constants for this item
        const int xg = T.x0 + 4 * tx;
        const int y = T.y0 + ty;
        bool pok[4];  // point inside the box
        const bool yok = y >= T.B.lo[1] && y < T.B.hi[1];
        float axa[4], axb[4], axk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int x = xg + e;
            pok[e] = yok && x >= T.B.lo[0] && x < T.B.hi[0];
            const int xc = min(max(x, 0), L.n[0] - 1);
            axa[e] = __ldg(P.ta[0] + xc);
            axb[e] = __ldg(P.tb[0] + xc);
            axk[e] = __ldg(P.tik[0] + xc);
        }
        const bool pall = pok[0] && pok[1] && pok[2] && pok[3];
        const bool pany = yok && (pok[0] || pok[1] || pok[2] || pok[3]);
        const int yc = min(max(y, 0), L.n[1] - 1);
        const float aya = __ldg(P.ta[1] + yc), ayb = __ldg(P.tb[1] + yc),
                    ayk = __ldg(P.tik[1] + yc);
        // zeta_y: the y run holding this row (a tile may meet both runs)
        // (only where the tile's stage carries that run's zeta_y: Z-slab tiles
        // never do, although rows past their box may fall in a y run)
        const int zyside = in_run(P.run[1][0], y) ? 0 : in_run(P.run[1][1], y) ? 1 : -1;
        const bool y_in_zy = zyside == 0 ? T.fzy0 : zyside == 1 ? T.fzy1 : false;
        // streams: element (xg, y, z) at base + (z - zb) * step
        const long long foff = L.off(xg, y, T.zb);
        float* pn_p = P.pn + foff;
        float* zx_p = fx ? P.run[0][xside].zeta + run_off(P.run[0][xside], 0, xg, y, T.zb) : nullptr;
        float* zy_p =
            y_in_zy ? P.run[1][zyside].zeta + run_off(P.run[1][zyside], 1, xg, y, T.zb) : nullptr;
        const long long zx_step = fx ? P.run[0][xside].s2 : 0;
        const long long zy_step = y_in_zy ? P.run[1][zyside].s2 : 0;
        const int psx_off = ty * C::BX + C::HX + 4 * tx;    // in the psi_x box
        const int toff = ty * C::TX + 4 * tx;               // in a tile
        const int psy_off = (R + ty) * C::TX + 4 * tx;      // in a psi_y box
        // zeta_z of the two z runs at plane zb (same x/y strides)
        auto zz_at_zb = [&](int sd) {
            return P.run[2][sd].hi > P.run[2][sd].lo
                       ? P.run[2][sd].zeta + run_off(P.run[2][sd], 2, xg, y, T.zb)
                       : nullptr;
        };
        float* const zzb0 = zz_at_zb(0);
        float* const zzb1 = zz_at_zb(1);
        const long long zz_step = P.run[2][0].hi > P.run[2][0].lo ? P.run[2][0].s2 : P.run[2][1].s2;
        // z window: shared-memory offsets of this thread's points in planes
        // j-2R .. j, rotated by one slot per plane (no modular slot arithmetic)
        int wo[2 * R + 1];
        int rel = (int)s;  // slot of the oldest window plane (next to release)

#pragma unroll 1
        for (int j = 0; j < T.nring; ++j) {
#pragma unroll
            for (int k = 0; k < 2 * R; ++k) wo[k] = wo[k + 1];
            wo[2 * R] = (int)s * C::PPLANE + soff;
            if (j >= 2 * R) {
                const int o = j - 2 * R;
                const int z = T.zb + o;
                const long long fo = (long long)o * L.plane;
                const int zr = zrun_of(P, z);
                const int zex = zext_in(P, z, T.B);
                float* zz_p = (zr == 0 ? zzb0 : zzb1) + o * zz_step;
                const float aza = __ldg(P.ta[2] + z), azb = __ldg(P.tb[2] + z),
                            azk = __ldg(P.tik[2] + z);

                mbar_wait(fullP + 8 * s, ph);
                // centre plane j - R, window planes j - 2R .. j
                const float* S = ring + wo[R];
                float xs[4 + 2 * C::HX];
#pragma unroll
                for (int h = 0; h < (4 + 2 * C::HX) / 4; ++h) {
                    const float4 v = lds4(S - C::HX + 4 * h);
                    xs[4 * h] = v.x;
                    xs[4 * h + 1] = v.y;
                    xs[4 * h + 2] = v.z;
                    xs[4 * h + 3] = v.w;
                }
                // lane pairs (FADD2, fast_common.cuh): pair h = points 2h, 2h + 1
                auto px = [&](const float* v, int h, int m) {
                    return f2(v[C::HX + 2 * h + m], v[C::HX + 2 * h + 1 + m]);
                };
                F2 two_p0[2], d2x[2], d2y[2], d2z[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const F2 c = px(xs, h, 0);
                    two_p0[h] = fa2<ORD>(c, c);  // T(2) * c (exact)
                    d2x[h] = d2y[h] = d2z[h] = f2zero();
                }
                // second derivatives, one axis at a time (stencil.hpp:86-91)
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        d2x[h] = d2_term2<ORD>(d2x[h], P.c2[0][m - 1], px(xs, h, m), px(xs, h, -m),
                                               two_p0[h]);
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    F2 u[2], d[2];
                    lds4x2(S + m * C::BX, u[0], u[1]);
                    lds4x2(S - m * C::BX, d[0], d[1]);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        d2y[h] = d2_term2<ORD>(d2y[h], P.c2[1][m - 1], u[h], d[h], two_p0[h]);
                }
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    F2 u[2], d[2];
                    lds4x2(ring + wo[R + m], u[0], u[1]);
                    lds4x2(ring + wo[R - m], d[0], d[1]);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        d2z[h] = d2_term2<ORD>(d2z[h], P.c2[2][m - 1], u[h], d[h], two_p0[h]);
                }
                // dpsi_x, dpsi_y from the psi boxes (central_derivative_at)
                F2 dpx[2] = {f2zero(), f2zero()}, dpy[2] = {f2zero(), f2zero()};
                F2 pp[2], cv[2], zx[2] = {f2zero(), f2zero()}, zy[2] = {f2zero(), f2zero()},
                                 zz[2] = {f2zero(), f2zero()}, dz[2] = {f2zero(), f2zero()};
                {
                    const int st = nq % C::NQD;
                    const int qsz = T.qsize + (zr >= 0 ? C::TILE : 0) + (zex >= 0 ? C::TILE : 0);
                    if (qo + qsz > C::QB) qo = 0;  // a stage never wraps (q_alloc)
                    const float* Q = qring + qo;
                    mbar_wait(fullQ + 8 * st, (nq / C::NQD) & 1);
                    qo += qsz;
                    lds4x2(Q + toff, pp[0], pp[1]);
                    lds4x2(Q + C::TILE + toff, cv[0], cv[1]);
                    if (fx) lds4x2(Q + T.o_zx + toff, zx[0], zx[1]);
                    if (y_in_zy) lds4x2(Q + (zyside == 0 ? T.o_zy0 : T.o_zy1) + toff, zy[0], zy[1]);
                    if (zr >= 0) lds4x2(Q + T.qsize + toff, zz[0], zz[1]);
                    // dpsi_z (k_p1); +0 where no psi_z reaches the window
                    if (zex >= 0) lds4x2(Q + T.qsize + (zr >= 0 ? C::TILE : 0) + toff, dz[0], dz[1]);
                    if (fx) {
                        float ps[4 + 2 * C::HX];
#pragma unroll
                        for (int h = 0; h < (4 + 2 * C::HX) / 4; ++h) {
                            const float4 v = lds4(Q + T.o_psx + psx_off - C::HX + 4 * h);
                            ps[4 * h] = v.x;
                            ps[4 * h + 1] = v.y;
                            ps[4 * h + 2] = v.z;
                            ps[4 * h + 3] = v.w;
                        }
#pragma unroll
                        for (int m = 1; m <= R; ++m)
#pragma unroll
                            for (int h = 0; h < 2; ++h)
                                dpx[h] = acc2<ORD>(dpx[h], P.c1[0][m - 1],
                                                   fs2<ORD>(px(ps, h, m), px(ps, h, -m)));
                    }
                    if (fy0 || fy1) {
                        const float* q0 = Q + T.o_psy0 + psy_off;
                        const float* q1 = Q + T.o_psy1 + psy_off;
#pragma unroll
                        for (int m = 1; m <= R; ++m) {
                            float4 up = make_float4(0.f, 0.f, 0.f, 0.f), dn = up;
                            // the two y runs never share a point: one of each pair is 0
                            if (fy0) {
                                up = lds4(q0 + m * C::TX);
                                dn = lds4(q0 - m * C::TX);
                            }
                            if (fy1) {
                                const float4 a = lds4(q1 + m * C::TX), b = lds4(q1 - m * C::TX);
                                up.x += a.x, up.y += a.y, up.z += a.z, up.w += a.w;
                                dn.x += b.x, dn.y += b.y, dn.z += b.z, dn.w += b.w;
                            }
                            const F2 u[2] = {f2(up.x, up.y), f2(up.z, up.w)};
                            const F2 d[2] = {f2(dn.x, dn.y), f2(dn.z, dn.w)};
#pragma unroll
                            for (int h = 0; h < 2; ++h)
                                dpy[h] = acc2<ORD>(dpy[h], P.c1[1][m - 1], fs2<ORD>(u[h], d[h]));
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive_b(emptyQ + 8 * st);  // stage fully read
                    ++nq;
                }
                // plane j - 2R has had its last use
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyP + 8 * rel);
                if (++rel == C::NS) rel = 0;

                // reference: drive = d2p*ik + dpsi; zeta = b*zeta + a*drive;
                // term = drive + zeta; lap = (term_x + term_y) + term_z
                F2 drx[2], dry[2], drz[2];
                F2 nzx[2] = {f2zero(), f2zero()}, nzy[2] = {f2zero(), f2zero()},
                   nzz[2] = {f2zero(), f2zero()};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    drx[h] = fa2<ORD>(fm2v<ORD>(axk[2 * h], axk[2 * h + 1], d2x[h]), dpx[h]);
                    dry[h] = fa2<ORD>(fm2<ORD>(ayk, d2y[h]), dpy[h]);
                    drz[h] = fa2<ORD>(fm2<ORD>(azk, d2z[h]), dz[h]);
                }
                // zeta updates only where a run holds the row / plane (uniform
                // branches: no FP spent on the other tiles' terms)
                if (fx) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        nzx[h] = fa2<ORD>(fm2v<ORD>(axa[2 * h], axa[2 * h + 1], drx[h]),
                                          fm2v<ORD>(axb[2 * h], axb[2 * h + 1], zx[h]));
                }
                if (y_in_zy) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        nzy[h] = fa2<ORD>(fm2<ORD>(aya, dry[h]), fm2<ORD>(ayb, zy[h]));
                }
                if (zr >= 0) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        nzz[h] = fa2<ORD>(fm2<ORD>(aza, drz[h]), fm2<ORD>(azb, zz[h]));
                }
                float out[4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const F2 lap = fa2<ORD>(fa2<ORD>(fa2<ORD>(drx[h], nzx[h]), fa2<ORD>(dry[h], nzy[h])),
                                            fa2<ORD>(drz[h], nzz[h]));
                    float c0, c1;
                    unf2(cv[h], c0, c1);
                    unf2(fa2<ORD>(fs2<ORD>(two_p0[h], pp[h]), fm2v<ORD>(c0, c1, lap)), out[2 * h],
                         out[2 * h + 1]);
                }
                float vzx[4], vzy[4], vzz[4];
                unf2(nzx[0], vzx[0], vzx[1]);
                unf2(nzx[1], vzx[2], vzx[3]);
                unf2(nzy[0], vzy[0], vzy[1]);
                unf2(nzy[1], vzy[2], vzy[3]);
                unf2(nzz[0], vzz[0], vzz[1]);
                unf2(nzz[1], vzz[2], vzz[3]);
                // stores: p_next inside the box, zeta where a run holds the point
                if (pany) {
                    st4(pn_p + fo, out, pok, pall);
                    if (fx) st4(zx_p + o * zx_step, vzx, pok, pall);
                    if (y_in_zy) st4(zy_p + o * zy_step, vzy, pok, pall);
                    if (zr >= 0) st4(zz_p, vzz, pok, pall);
                }
            } else {
                mbar_wait(fullP + 8 * s, ph);
            }
            if (++s == C::NS) s = 0, ph ^= 1;
        }
        // the item's last 2R planes
#pragma unroll 1
        for (int k = 0; k < 2 * R; ++k) {
            __syncwarp();
            if (lane == 0) mbar_arrive_b(emptyP + 8 * rel);
            if (++rel == C::NS) rel = 0;
        }
    }
    MM_TRACE_END(3)
}

}  // namespace fast
}  // namespace mmb
