// fast_cpml.cuh -- the fused one-pass CPML kernel (k_cpml), MM_MODE_FAST.
//
// ref: update_damping_pass1 (propagator_impl.hpp:106-123) and
//      update_damping_pass2 (propagator_impl.hpp:125-152) of every damping
//      slab; second_derivative_at / central_derivative_at (stencil.hpp:86-99).
//
// One launch does both CPML passes: per (x, y) tile and z chunk it streams
// p_cur planes along z (the slowest device axis) and, per output plane k,
//   1. psi_x(k), psi_y(k) = b psi + a D1(p_cur(k)) for the tile's points in
//      an x / y damping run -> global (in place) and a shared exchange plane;
//   2. psi_z(k+R) = b psi + a D1_z(p_cur) -> a per-thread register window of
//      2R+1 planes (and, for the chunk's own planes, global);
//   3. one __syncthreads;
//   4. dpsi_x / dpsi_y from the exchange planes, dpsi_z from the window,
//      zeta, the Laplacian and p_next.
// psi goes through HBM once per step (read + write); the two-pass path read
// it again in pass 2 and wrote + read dpsi_z.
//
// Why this is exact without a halo of neighbour tiles' psi: the tiles are
// cut so that every x run lies inside one tile's x range and every y run plus
// the R rows past it inside one tile's rows (kernels_fast.cu builds them and
// falls back to the two-pass kernels when a layout does not allow it), so
// dpsi_x and dpsi_y only read psi the tile itself produced (the zero halo of
// the reference's per-slab boxes, cpml.hpp:77-99, is the zero padding of the
// exchange planes).  Along z a chunk recomputes the psi_z planes within R of
// its ends from the OLD psi_z and stores only its own planes, in place: the
// host never puts a chunk boundary of one launch within R of a z run
// ((lo - R, hi + R) is forbidden), so no chunk reads a psi_z plane another
// chunk of the same launch writes.  Every value is formed with the
// reference's operation order and separate roundings (ORD 2), hence
// bit-identical to the CPU reference.
//
// Per-point masks (the A9 rule of SURVEY.md §8a): dpsi_x only in X slabs,
// dpsi_y in X and Y slabs, dpsi_z in every slab; p_next is stored at the
// tile's owned slab points only (k_inner writes the inner box).
//
// Hardware mapping: one CTA per SM, 8 consumer warps + 1 producer warp; a
// 32 x 32 tile, each consumer thread four consecutive x points (float4) of
// one row: 128-bit shared loads, 16-byte global stores, and the arithmetic
// on lane pairs (FADD2, see fast_common.cuh).  Producer lane 0 pulls work
// items, hands them to the consumers (and to lane 1) through a 4-slot item
// ring and streams p_cur planes with their 4-column / R-row halo into a ring
// of NS slots (the 3R+1-plane window psi_z needs plus lead); lane 1 streams,
// per output plane, one stage of 32 x 32 boxes -- p_prev, c and the tile's
// psi / zeta run boxes, only the ones the item needs (TMA's out-of-bounds
// zero fill is the runs' zero halo).  Each lane waits only on the empty
// barriers of its own slots, so the ring runs as far ahead as its depth
// allows (one lane serving both fell back to the stages' one-plane lead).  Consumers synchronise once per plane on a named barrier (the
// exchange planes) and release ring slots and stages with one mbarrier
// arrive each.  The z neighbours of the ring are addressed through a
// per-thread array of slot offsets shifted once per plane (no index
// arithmetic per tap); the z loop is instantiated for items with and without
// the psi_z window.
#pragma once

#include "fast_common.cuh"

namespace mmb {
namespace fast {

// Experiment builds (build.py --variant ... -D MM_CPML_EXP_NOFP): consumers
// only wait, synchronise and release -- the data pipeline's own rate.
#ifdef MM_CPML_EXP_NOFP
constexpr bool kCpmlExpNoFp = true;
#else
constexpr bool kCpmlExpNoFp = false;
#endif

#ifndef MM_CPML_PX
#define MM_CPML_PX 4
#endif

// Producer waits: a plain mbarrier.try_wait loop (the instruction suspends
// the thread in hardware) or a nanosleep back-off between polls.
#ifndef MM_CPML_PROD_SLEEP
#define MM_CPML_PROD_SLEEP 1
#endif
__device__ __forceinline__ void prod_wait(uint32_t bar, uint32_t parity) {
#if MM_CPML_PROD_SLEEP
    mbar_wait_sleep(bar, parity);
#else
    mbar_wait(bar, parity);
#endif
}

template <int R>
struct CpmlCfg {
    static_assert(R <= 4, "k_cpml: the 3R+1-plane window of wider stencils does not fit");
    static constexpr int PX = MM_CPML_PX;    // x points per thread (2: float2, 4: float4)
    static constexpr int NH = PX / 2;        // lane pairs per thread
    static constexpr int TXT = 32 / PX;      // threads per row
    static constexpr int TX = PX * TXT;      // 32
    static constexpr int TY = 32;
    static constexpr int NC = TXT * TY;      // consumer threads
    static constexpr int NT = NC + 32;       // + one producer warp
    static constexpr int HX = 4;             // x halo (16-byte TMA granule)
    static constexpr int BX = TX + 2 * HX;   // 40
    static constexpr int BY = TY + 2 * R;
    static constexpr int PLANE = pad32(BX * BY);
    static constexpr int NS = 3 * R + 5;     // p_cur ring slots (3R+1 window + lead)
    static constexpr int TILE = TX * TY;     // one 32 x 32 stage box
    static constexpr int NBOX = 8;           // stage boxes: pp cv psi_x zeta_x psi_y zeta_y zeta_z psi_z
    static constexpr int SSIZE = NBOX * TILE;
    static constexpr int NI = 4;             // work-item slots (producer -> consumers)
    static constexpr int PXW = TX + 2 * HX;  // psi_x exchange row (zero pads)
    static constexpr int PXN = TY * PXW;
    static constexpr int PYN = (TY + 2 * R) * TX;
    static constexpr int BUDGET = 227 * 1024 - 256;
    static constexpr int NQ = 3;             // stages (p_prev, c, CPML boxes of one plane)
    static constexpr int NBAR = 2 * NS + 2 * NQ + 4 * NI;
    static constexpr size_t SMEM =
        4 * (size_t)(NS * PLANE + 2 * PXN + 2 * PYN + NQ * SSIZE) + 8 * NBAR + 16 * NI + 64;
    static_assert(SMEM <= BUDGET, "k_cpml shared memory");
};

// A tile of the slab region: TX x TY points from (x0, y0); it owns (stores)
// x in [ox0, x1), rows [oy0, y1); xside / yside the x / y damping run whose
// points lie in it (-1: none).
struct CTile {
    int x0, x1, y0, y1;
    int xside, yside;
    int ox0, oy0;
};

struct CpmlMaps {
    CUtensorMap pc;          // p_cur, (TX + 2HX) x (TY + 2R) halo box
    CUtensorMap pp, cv;      // TX x TY tiles
    CUtensorMap psi[3][2];   // TX x TY boxes of the runs
    CUtensorMap zeta[3][2];
};

struct CpmlParams {
    Layout lay;
    int ilo[3], ihi[3];     // local inner box (grid.cpp:24-45)
    const CTile* tiles;
    const int4* items;      // (tile, z_begin, z_end, -)
    WorkQueue wq;
    CpmlRun run[3][2];      // psi / zeta of every run, updated in place
    const float* ta[3];
    const float* tb[3];
    const float* tik[3];
    float c2[3][kMaxR], c1[3][kMaxR];
    float* pn;
};

__device__ __forceinline__ void sts4(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
// PX consecutive floats (PX = 2 or 4) as lane pairs / plain values
template <int PX>
__device__ __forceinline__ void ldsp(const float* p, F2 (&v)[PX / 2]) {
    if constexpr (PX == 4) {
        lds4x2(p, v[0], v[1]);
    } else {
        const float2 a = *reinterpret_cast<const float2*>(p);
        v[0] = f2(a.x, a.y);
    }
}
// the x neighbours x - 4 .. x + PX + 3 of a thread's points
template <int PX>
__device__ __forceinline__ void ldrow(const float* S, float (&xs)[PX + 8]) {
    if constexpr (PX == 4) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const float4 a = *reinterpret_cast<const float4*>(S - 4 + 4 * i);
            xs[4 * i] = a.x;
            xs[4 * i + 1] = a.y;
            xs[4 * i + 2] = a.z;
            xs[4 * i + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const float2 a = *reinterpret_cast<const float2*>(S - 4 + 2 * i);
            xs[2 * i] = a.x;
            xs[2 * i + 1] = a.y;
        }
    }
}
template <int PX>
__device__ __forceinline__ void stsv(float* p, const float (&v)[PX]) {
    if constexpr (PX == 4)
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
}
template <int PX>
__device__ __forceinline__ void stgv(float* p, const float (&v)[PX], const bool (&ok)[PX], bool all) {
    if (all) {
        stsv<PX>(p, v);
    } else {
#pragma unroll
        for (int e = 0; e < PX; ++e)
            if (ok[e]) p[e] = v[e];
    }
}
template <int PX>
__device__ __forceinline__ void ldgp(const float* p, const bool (&ok)[PX], bool all, F2 (&v)[PX / 2]) {
    float a[PX];
    if (all) {
        if constexpr (PX == 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(p));
            a[0] = t.x, a[1] = t.y, a[2] = t.z, a[3] = t.w;
        } else {
            const float2 t = __ldg(reinterpret_cast<const float2*>(p));
            a[0] = t.x, a[1] = t.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < PX; ++e) a[e] = ok[e] ? __ldg(p + e) : 0.0f;
    }
#pragma unroll
    for (int h = 0; h < PX / 2; ++h) v[h] = f2(a[2 * h], a[2 * h + 1]);
}
__device__ __forceinline__ void unpack4(const float4& v, float* o) {
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
}

__device__ __forceinline__ int zrun_at(const CpmlParams& P, int z) {
    return in_run(P.run[2][0], z) ? 0 : in_run(P.run[2][1], z) ? 1 : -1;
}

// Stage box offsets (floats) inside one stage.
enum { QO_PP = 0, QO_CV = 1, QO_PSX = 2, QO_ZX = 3, QO_PSY = 4, QO_ZY = 5, QO_ZZ = 6, QO_PSZ = 7 };

// Barriers / rings of one CTA (shared-memory addresses).
struct CpmlSync {
    uint32_t fullP, emptyP;  // per ring slot
    uint32_t fullQ, emptyQ;  // per stage
    uint32_t fullI, emptyI;  // per work-item slot (consumers)
    uint32_t fullS, emptyS;  // per work-item slot (stage producer lane)
};

// Producer lane 0: the p_cur ring planes of one work item (tile T, output
// planes [zb, ze)), each gated by the empty barrier of its slot, as far ahead
// of the consumers as the ring allows.
template <int R, bool ZACT>
__device__ __forceinline__ void cpml_produce_ring(const CpmlMaps& M, const CpmlParams& P,
                                                  const CTile& T, int zb, int ze, float* ring,
                                                  const CpmlSync& B, uint32_t& peP, int& pslot) {
    using C = CpmlCfg<R>;
    constexpr int LAG = ZACT ? 2 * R : R;
    const Layout& L = P.lay;
    const int nring = ze - zb + 2 * LAG;
    const int zr0 = zb - LAG;
    const int tmx = L.L + T.x0 - C::HX, tmy = T.y0 - R + L.r;
#pragma unroll 1
    for (int j = 0; j < nring; ++j) {
        const int slot = pslot;
        pslot = pslot + 1 == C::NS ? 0 : pslot + 1;
        prod_wait(B.emptyP + 8 * slot, ((peP >> slot) & 1u) ^ 1u);
        peP ^= 1u << slot;
        const uint32_t bar = B.fullP + 8 * slot;
        mbar_expect_tx(bar, 4u * C::BX * C::BY);
        tma_load_3d(smem_u32(ring + slot * C::PLANE), &M.pc, tmx, tmy, zr0 + j + L.r, bar);
    }
}

// Producer lane 1: the stage of every output plane (p_prev, c and the
// tile's CPML boxes of that plane), each gated by the empty barrier of its
// stage.
template <int R, bool ZACT>
__device__ __forceinline__ void cpml_produce_stages(const CpmlMaps& M, const CpmlParams& P,
                                                    const CTile& T, int zb, int ze, float* qbuf,
                                                    const CpmlSync& B, uint32_t& peQ,
                                                    int& pstage) {
    using C = CpmlCfg<R>;
    const Layout& L = P.lay;
    const bool fx = T.xside >= 0, fy = T.yside >= 0;
    const CpmlRun& RX = P.run[0][fx ? T.xside : 0];
    const CpmlRun& RY = P.run[1][fy ? T.yside : 0];
    const int tmx = L.L + T.x0, tmy = T.y0 + L.r;
#pragma unroll 1
    for (int z = zb; z < ze; ++z) {
        const int st = pstage;
        pstage = pstage + 1 == C::NQ ? 0 : pstage + 1;
        prod_wait(B.emptyQ + 8 * st, ((peQ >> st) & 1u) ^ 1u);
        peQ ^= 1u << st;
        const uint32_t bar = B.fullQ + 8 * st;
        float* dst = qbuf + st * C::SSIZE;
        const int zr = ZACT ? zrun_at(P, z) : -1;
        const int zp = ZACT ? zrun_at(P, z + R) : -1;
        const uint32_t nb = 2 + (fx ? 2 : 0) + (fy ? 2 : 0) + (zr >= 0 ? 1 : 0) + (zp >= 0 ? 1 : 0);
        mbar_expect_tx(bar, nb * 4u * C::TILE);
        tma_load_3d(smem_u32(dst + QO_PP * C::TILE), &M.pp, tmx, tmy, z + L.r, bar);
        tma_load_3d(smem_u32(dst + QO_CV * C::TILE), &M.cv, tmx, tmy, z + L.r, bar);
        if (fx) {
            tma_load_3d(smem_u32(dst + QO_PSX * C::TILE), &M.psi[0][T.xside], T.x0 - RX.org, T.y0,
                        z, bar);
            tma_load_3d(smem_u32(dst + QO_ZX * C::TILE), &M.zeta[0][T.xside], T.x0 - RX.org, T.y0,
                        z, bar);
        }
        if (fy) {
            tma_load_3d(smem_u32(dst + QO_PSY * C::TILE), &M.psi[1][T.yside], T.x0, T.y0 - RY.org,
                        z, bar);
            tma_load_3d(smem_u32(dst + QO_ZY * C::TILE), &M.zeta[1][T.yside], T.x0, T.y0 - RY.org,
                        z, bar);
        }
        if (zr >= 0)
            tma_load_3d(smem_u32(dst + QO_ZZ * C::TILE), &M.zeta[2][zr], T.x0, T.y0,
                        z - P.run[2][zr].org, bar);
        if (zp >= 0)
            tma_load_3d(smem_u32(dst + QO_PSZ * C::TILE), &M.psi[2][zp], T.x0, T.y0,
                        z + R - P.run[2][zp].org, bar);
    }
}

template <int NC>
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
}

// Consumers: one work item (tile T, output planes [zb, ze)).  ZACT: a z run
// lies within R of the item's planes (psi_z window, output lags the newest
// plane by 2R).
template <int R, int ORD, bool ZACT>
__device__ __forceinline__ void cpml_consume(const CpmlParams& P, const CTile& T, int zb, int ze,
                                             const float* ring, const float* qbuf, float* PXb,
                                             float* PYb, const CpmlSync& B, uint32_t& phP,
                                             uint32_t& phQ, int& cslot, int& cstage) {
    using C = CpmlCfg<R>;
    constexpr int PX = C::PX, NH = C::NH;
    constexpr int LAG = ZACT ? 2 * R : R;  // output plane k <-> newest ring plane k + LAG
    constexpr int Q = LAG + R + 1;         // ring planes a thread reads in one iteration
    const int tid = threadIdx.x;
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const Layout& L = P.lay;
    const int nout = ze - zb;
    const int nring = nout + 2 * LAG;
    const int zr0 = zb - LAG;  // z of ring plane 0
    const bool fx = T.xside >= 0, fy = T.yside >= 0;
    const CpmlRun& RX = P.run[0][fx ? T.xside : 0];
    const CpmlRun& RY = P.run[1][fy ? T.yside : 0];

    // ---- per-thread constants of this item
    const int xg = T.x0 + PX * tx;
    const int y = T.y0 + ty;
    const bool yok = y >= T.oy0 && y < T.y1;
    bool pok[PX], inX[PX], rx[PX];
    float axa[PX], axb[PX], axk[PX];
#pragma unroll
    for (int e = 0; e < PX; ++e) {
        const int x = xg + e;
        pok[e] = yok && x >= T.ox0 && x < T.x1;
        inX[e] = x < P.ilo[0] || x >= P.ihi[0];
        rx[e] = fx && in_run(RX, x);
        const int xc = min(x, L.n[0] - 1);
        axk[e] = __ldg(P.tik[0] + xc);
        axa[e] = fx ? __ldg(P.ta[0] + xc) : 0.0f;
        axb[e] = fx ? __ldg(P.tb[0] + xc) : 1.0f;
    }
    const bool rowY = y < P.ilo[1] || y >= P.ihi[1];
    const bool ry = fy && in_run(RY, y);
    const int yc = min(max(y, 0), L.n[1] - 1);
    const float aya = __ldg(P.ta[1] + yc), ayb = __ldg(P.tb[1] + yc), ayk = __ldg(P.tik[1] + yc);
    bool allp = true;
    bool okx[PX], oky[PX];
    bool allx = true, ally = true;
#pragma unroll
    for (int e = 0; e < PX; ++e) {
        okx[e] = pok[e] && rx[e];
        oky[e] = pok[e] && ry;
        allp = allp && pok[e];
        allx = allx && okx[e];
        ally = ally && oky[e];
    }
    // running global pointers (advanced by one plane per output)
    float* pn_p = P.pn + L.off(xg, y, zb);
    float* psx_p = fx ? RX.psi + run_off(RX, 0, xg, y, zb) : nullptr;
    float* zx_p = fx ? RX.zeta + run_off(RX, 0, xg, y, zb) : nullptr;
    float* psy_p = fy ? RY.psi + run_off(RY, 1, xg, y, zb) : nullptr;
    float* zy_p = fy ? RY.zeta + run_off(RY, 1, xg, y, zb) : nullptr;
    const long long sxz = fx ? RX.s2 : 0, syz = fy ? RY.s2 : 0;
    const int soff = (R + ty) * C::BX + C::HX + PX * tx;  // centre in a p_cur plane
    const int toff = ty * C::TX + PX * tx;                 // in a stage box
    const int pxo = ty * C::PXW + C::HX + PX * tx;         // in a psi_x exchange plane
    const int pyo = (R + ty) * C::TX + PX * tx;            // in a psi_y exchange plane
    const float* ringT = ring + soff;

    // slot offsets (floats) of the last Q ring planes, oldest first
    int so[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) so[i] = 0;
    // psi_z planes k-R .. k+R of output plane k, as two lane pairs
    constexpr int W = ZACT ? 2 * R + 1 : 1;
    F2 pw[NH][W];
#pragma unroll
    for (int i = 0; i < W; ++i)
#pragma unroll
        for (int h = 0; h < NH; ++h) pw[h][i] = f2zero();
    // lane pair h of the x-neighbour values v[0..PX+7] (x - 4 .. x + PX + 3)
    auto pairx = [](const float* v, int h, int m) { return f2(v[4 + 2 * h + m], v[5 + 2 * h + m]); };
    auto mask4 = [](F2 (&v)[NH], const bool (&ok)[PX]) {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            float a, b;
            unf2(v[h], a, b);
            v[h] = f2(ok[2 * h] ? a : 0.0f, ok[2 * h + 1] ? b : 0.0f);
        }
    };
    auto to4 = [](const F2 (&v)[NH], float (&o)[PX]) {
#pragma unroll
        for (int h = 0; h < NH; ++h) unf2(v[h], o[2 * h], o[2 * h + 1]);
    };

    int rel = 0;             // ring planes of this item released so far
    int rslot = cslot;       // ring slot of plane `rel`
    int pst_prev = -1;       // stage of the previous output (released after the next barrier)
#pragma unroll 1
    for (int j = 0; j < nring; ++j) {
        const int slot = cslot;
        cslot = cslot + 1 == C::NS ? 0 : cslot + 1;
        mbar_wait(B.fullP + 8 * slot, (phP >> slot) & 1u);
        phP ^= 1u << slot;
#pragma unroll
        for (int i = 0; i < Q - 1; ++i) so[i] = so[i + 1];
        so[Q - 1] = slot * C::PLANE;
        const int zj = zr0 + j;
        const bool outp = j >= 2 * LAG;
        const int o = j - 2 * LAG;  // output plane index (valid if outp)
        const int k = zb + o;
        const int st = cstage;
        const float* Q0 = qbuf + st * C::SSIZE + toff;
        if (outp) {
            mbar_wait(B.fullQ + 8 * st, (phQ >> st) & 1u);
            phQ ^= 1u << st;
            cstage = cstage + 1 == C::NQ ? 0 : cstage + 1;
        }

        // ---- psi_z(zj - R) into the window (update_damping_pass1, z axis)
        if constexpr (ZACT && !kCpmlExpNoFp) {
            if (j >= 2 * R) {
                const int pz = zj - R;
                F2 nv[NH] = {};
                const int zr = zrun_at(P, pz);
                if (zr >= 0) {
                    const CpmlRun& RZ = P.run[2][zr];
                    // ring planes pz +- m: so[Q-1-R +- m]
                    F2 dp[NH] = {};
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        F2 u[NH], d[NH];
                        ldsp<PX>(ringT + so[Q - 1 - R + m], u);
                        ldsp<PX>(ringT + so[Q - 1 - R - m], d);
#pragma unroll
                        for (int h = 0; h < NH; ++h)
                            dp[h] = acc2<ORD>(dp[h], P.c1[2][m - 1], fs2<ORD>(u[h], d[h]));
                    }
                    // old psi_z: from the stage of output plane pz - R, or (the
                    // chunk's first 2R planes) straight from the run
                    const long long ro = run_off(RZ, 2, xg, y, pz);
                    F2 old[NH];
                    if (outp) {
                        ldsp<PX>(Q0 + QO_PSZ * C::TILE, old);
                    } else {
                        ldgp<PX>(RZ.psi + ro, pok, allp, old);
                    }
                    const float az = __ldg(P.ta[2] + pz), bz = __ldg(P.tb[2] + pz);
                    // reference: psi = b * psi + a * dp  (propagator_impl.hpp:118-120)
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        nv[h] = fa2<ORD>(fm2<ORD>(az, dp[h]), fm2<ORD>(bz, old[h]));
                    if (pz >= zb && pz < ze) {
                        float v4[PX];
                        to4(nv, v4);
                        stgv<PX>(RZ.psi + ro, v4, pok, allp);
                    }
                }
#pragma unroll
                for (int i = 0; i < 2 * R; ++i)
#pragma unroll
                    for (int h = 0; h < NH; ++h) pw[h][i] = pw[h][i + 1];
#pragma unroll
                for (int h = 0; h < NH; ++h) pw[h][2 * R] = nv[h];
            }
        }

        // ---- output plane k, before the exchange
        F2 two_p0[NH], d2x[NH], d2y[NH], d2z[NH];
        const int xb = j & 1;  // exchange buffer of this iteration
        if (outp && !kCpmlExpNoFp) {
            const float* S = ringT + so[Q - 1 - LAG];  // plane k
            float xs[PX + 2 * C::HX];
            ldrow<PX>(S, xs);
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const F2 c = pairx(xs, h, 0);
                two_p0[h] = fa2<ORD>(c, c);  // T(2) * c (exact)
                d2x[h] = d2y[h] = d2z[h] = f2zero();
            }
#pragma unroll
            for (int m = 1; m <= R; ++m)
#pragma unroll
                for (int h = 0; h < NH; ++h)
                    d2x[h] = d2_term2<ORD>(d2x[h], P.c2[0][m - 1], pairx(xs, h, m),
                                           pairx(xs, h, -m), two_p0[h]);
            F2 d1y[NH] = {};
#pragma unroll
            for (int m = 1; m <= R; ++m) {
                F2 u[NH], d[NH];
                ldsp<PX>(S + m * C::BX, u);
                ldsp<PX>(S - m * C::BX, d);
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    d2y[h] = d2_term2<ORD>(d2y[h], P.c2[1][m - 1], u[h], d[h], two_p0[h]);
                    if (fy) d1y[h] = acc2<ORD>(d1y[h], P.c1[1][m - 1], fs2<ORD>(u[h], d[h]));
                }
            }
#pragma unroll
            for (int m = 1; m <= R; ++m) {
                F2 u[NH], d[NH];
                ldsp<PX>(ringT + so[Q - 1 - LAG + m], u);
                ldsp<PX>(ringT + so[Q - 1 - LAG - m], d);
#pragma unroll
                for (int h = 0; h < NH; ++h)
                    d2z[h] = d2_term2<ORD>(d2z[h], P.c2[2][m - 1], u[h], d[h], two_p0[h]);
            }
            if (fx) {  // psi_x(k) of the tile's x run (pass 1)
                F2 old[NH], dp[NH] = {}, nv[NH];
                ldsp<PX>(Q0 + QO_PSX * C::TILE, old);
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        dp[h] = acc2<ORD>(dp[h], P.c1[0][m - 1],
                                          fs2<ORD>(pairx(xs, h, m), pairx(xs, h, -m)));
#pragma unroll
                for (int h = 0; h < NH; ++h)
                    nv[h] = fa2<ORD>(fm2v<ORD>(axa[2 * h], axa[2 * h + 1], dp[h]),
                                     fm2v<ORD>(axb[2 * h], axb[2 * h + 1], old[h]));
                mask4(nv, rx);
                float v4[PX];
                to4(nv, v4);
                stsv<PX>(PXb + xb * C::PXN + pxo, v4);
                stgv<PX>(psx_p, v4, okx, allx);
            }
            if (fy) {  // psi_y(k) of the tile's y run (pass 1)
                F2 old[NH], nv[NH];
                ldsp<PX>(Q0 + QO_PSY * C::TILE, old);
#pragma unroll
                for (int h = 0; h < NH; ++h)
                    nv[h] = ry ? fa2<ORD>(fm2<ORD>(aya, d1y[h]), fm2<ORD>(ayb, old[h])) : f2zero();
                float v4[PX];
                to4(nv, v4);
                stsv<PX>(PYb + xb * C::PYN + pyo, v4);
                stgv<PX>(psy_p, v4, oky, ally);
            }
        }

        consumer_sync<C::NC>();  // exchange planes complete; iteration j-1 done everywhere
        {
            // ring planes no later iteration reads: index < j + 1 - (LAG + R);
            // the stage of the previous output
            const int upto = j + 1 - LAG - R;
            for (; rel < upto; ++rel) {
                if (tid == 0) mbar_arrive_b(B.emptyP + 8 * rslot);
                rslot = rslot + 1 == C::NS ? 0 : rslot + 1;
            }
            if (pst_prev >= 0 && tid == 0) mbar_arrive_b(B.emptyQ + 8 * pst_prev);
            pst_prev = outp ? st : -1;
        }

        if (outp && !kCpmlExpNoFp) {
            // ---- pass 2 at (x, y, k)
            const bool planeZ = k < P.ilo[2] || k >= P.ihi[2];
            const int zr = ZACT ? zrun_at(P, k) : -1;
            F2 dpx[NH] = {}, dpy[NH] = {}, dpz[NH] = {};
            if (fx) {
                float ps[PX + 2 * C::HX];
                ldrow<PX>(PXb + xb * C::PXN + pxo, ps);
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        dpx[h] = acc2<ORD>(dpx[h], P.c1[0][m - 1],
                                           fs2<ORD>(pairx(ps, h, m), pairx(ps, h, -m)));
                mask4(dpx, inX);
            }
            if (fy) {
                const float* Yp = PYb + xb * C::PYN + pyo;
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    F2 u[NH], d[NH];
                    ldsp<PX>(Yp + m * C::TX, u);
                    ldsp<PX>(Yp - m * C::TX, d);
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        dpy[h] = acc2<ORD>(dpy[h], P.c1[1][m - 1], fs2<ORD>(u[h], d[h]));
                }
                if (!rowY) mask4(dpy, inX);
            }
            if constexpr (ZACT) {
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        dpz[h] = acc2<ORD>(dpz[h], P.c1[2][m - 1],
                                           fs2<ORD>(pw[h][R + m], pw[h][R - m]));
            }
            F2 pp[NH], cv[NH], zx[NH] = {}, zy[NH] = {}, zz[NH] = {};
            ldsp<PX>(Q0 + QO_PP * C::TILE, pp);
            ldsp<PX>(Q0 + QO_CV * C::TILE, cv);
            if (fx) ldsp<PX>(Q0 + QO_ZX * C::TILE, zx);
            if (fy) ldsp<PX>(Q0 + QO_ZY * C::TILE, zy);
            if (zr >= 0) ldsp<PX>(Q0 + QO_ZZ * C::TILE, zz);
            const float aza = __ldg(P.ta[2] + k), azb = __ldg(P.tb[2] + k),
                        azk = __ldg(P.tik[2] + k);
            // reference: drive = d2p*ik + dpsi; zeta = b*zeta + a*drive;
            // term = drive + zeta; lap = (term_x + term_y) + term_z
            F2 out[NH], drx[NH], dry[NH], drz[NH], nzx[NH], nzy[NH], nzz[NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                drx[h] = fa2<ORD>(fm2v<ORD>(axk[2 * h], axk[2 * h + 1], d2x[h]), dpx[h]);
                dry[h] = fa2<ORD>(fm2<ORD>(ayk, d2y[h]), dpy[h]);
                drz[h] = fa2<ORD>(fm2<ORD>(azk, d2z[h]), dpz[h]);
                nzx[h] = fx ? fa2<ORD>(fm2v<ORD>(axa[2 * h], axa[2 * h + 1], drx[h]),
                                       fm2v<ORD>(axb[2 * h], axb[2 * h + 1], zx[h]))
                            : f2zero();
                nzy[h] = ry ? fa2<ORD>(fm2<ORD>(aya, dry[h]), fm2<ORD>(ayb, zy[h])) : f2zero();
                nzz[h] = zr >= 0 ? fa2<ORD>(fm2<ORD>(aza, drz[h]), fm2<ORD>(azb, zz[h])) : f2zero();
            }
            if (fx) mask4(nzx, rx);
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const F2 lap = fa2<ORD>(fa2<ORD>(fa2<ORD>(drx[h], nzx[h]), fa2<ORD>(dry[h], nzy[h])),
                                        fa2<ORD>(drz[h], nzz[h]));
                float c0, c1;
                unf2(cv[h], c0, c1);
                out[h] = fa2<ORD>(fs2<ORD>(two_p0[h], pp[h]), fm2v<ORD>(c0, c1, lap));
            }
            bool pst[PX];  // p_next store: owned slab points (k_inner does the inner box)
            bool pall = true;
#pragma unroll
            for (int e = 0; e < PX; ++e) {
                pst[e] = pok[e] && (inX[e] || rowY || planeZ);
                pall = pall && pst[e];
            }
            float v4[PX];
            to4(out, v4);
            stgv<PX>(pn_p, v4, pst, pall);
            if (fx) {
                to4(nzx, v4);
                stgv<PX>(zx_p, v4, okx, allx);
            }
            if (fy) {
                to4(nzy, v4);
                stgv<PX>(zy_p, v4, oky, ally);
            }
            if (zr >= 0) {
                const CpmlRun& RZ = P.run[2][zr];
                to4(nzz, v4);
                stgv<PX>(RZ.zeta + run_off(RZ, 2, xg, y, k), v4, pok, allp);
            }
            pn_p += L.plane;
            psx_p += sxz;
            zx_p += sxz;
            psy_p += syz;
            zy_p += syz;
        }
    }
    // the item's last reads are done once every consumer passes this barrier:
    // release its remaining ring planes and its last stage
    consumer_sync<C::NC>();
    if (tid == 0) {
        for (; rel < nring; ++rel) {
            mbar_arrive_b(B.emptyP + 8 * rslot);
            rslot = rslot + 1 == C::NS ? 0 : rslot + 1;
        }
        if (pst_prev >= 0) mbar_arrive_b(B.emptyQ + 8 * pst_prev);
    }
}

template <int R, int ORD>
__global__ void __launch_bounds__(CpmlCfg<R>::NT, 1)
    k_cpml(const __grid_constant__ CpmlMaps M, const CpmlParams P) {
    using C = CpmlCfg<R>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qbuf = ring + C::NS * C::PLANE;  // stages
    float* PXb = qbuf + C::NQ * C::SSIZE;   // 2 psi_x exchange planes
    float* PYb = PXb + 2 * C::PXN;          // 2 psi_y exchange planes
    int4* items = reinterpret_cast<int4*>(PYb + 2 * C::PYN);
    uint64_t* bars = reinterpret_cast<uint64_t*>(items + C::NI);
    CpmlSync B;
    B.fullP = smem_u32(bars);
    B.emptyP = B.fullP + 8 * C::NS;
    B.fullQ = B.emptyP + 8 * C::NS;
    B.emptyQ = B.fullQ + 8 * C::NQ;
    B.fullI = B.emptyQ + 8 * C::NQ;
    B.emptyI = B.fullI + 8 * C::NI;
    B.fullS = B.emptyI + 8 * C::NI;
    B.emptyS = B.fullS + 8 * C::NI;
    const int tid = threadIdx.x;

    if (tid == 0) {
        prefetch_tmap(&M.pc);
        prefetch_tmap(&M.pp);
        prefetch_tmap(&M.cv);
        for (int s = 0; s < C::NBAR; ++s) mbar_init(B.fullP + 8 * s, 1);
        fence_barrier_init();
    }
    // zero pads of the exchange planes (never written afterwards)
    for (int i = tid; i < 2 * C::PXN; i += C::NT) {
        const int c = i % C::PXW;
        if (c < C::HX || c >= C::HX + C::TX) PXb[i] = 0.0f;
    }
    for (int i = tid; i < 2 * C::PYN; i += C::NT) {
        const int r = (i % C::PYN) / C::TX;
        if (r < R || r >= R + C::TY) PYb[i] = 0.0f;
    }
    __syncthreads();

    auto zact_of = [&](int zb, int ze) {
        // psi_z is needed where a z run lies within R of the chunk's planes
        return near_run(P.run[2][0], zb - R, ze + R) || near_run(P.run[2][1], zb - R, ze + R);
    };
    if (tid >= C::NC) {
        // ---- producer warp: lane 0 pulls items and streams the p_cur ring,
        // lane 1 streams the stages; each waits only on its own slots
        const int lane = tid - C::NC;
        if (lane == 0) {
            uint32_t peP = 0, peI = 0;
            int pslot = 0;
            for (int n = 0;; ++n) {
                const int item = atomicAdd(P.wq.ctr, 1);
                const int si = n % C::NI;
                const uint32_t par = ((peI >> si) & 1u) ^ 1u;
                prod_wait(B.emptyI + 8 * si, par);
                prod_wait(B.emptyS + 8 * si, par);
                peI ^= 1u << si;
                int4 sg = make_int4(-1, 0, 0, 0);
                if (item < P.wq.nitems) sg = P.items[item];
                items[si] = sg;
                mbar_arrive_b(B.fullI + 8 * si);  // (release: the item is visible)
                mbar_arrive_b(B.fullS + 8 * si);
                if (sg.x < 0) break;
                const CTile T = P.tiles[sg.x];
                if (zact_of(sg.y, sg.z))
                    cpml_produce_ring<R, true>(M, P, T, sg.y, sg.z, ring, B, peP, pslot);
                else
                    cpml_produce_ring<R, false>(M, P, T, sg.y, sg.z, ring, B, peP, pslot);
            }
        } else if (lane == 1) {
            uint32_t peQ = 0, phS = 0;
            int pstage = 0;
            for (int n = 0;; ++n) {
                const int si = n % C::NI;
                prod_wait(B.fullS + 8 * si, (phS >> si) & 1u);
                phS ^= 1u << si;
                const int4 sg = items[si];
                mbar_arrive_b(B.emptyS + 8 * si);
                if (sg.x < 0) break;
                const CTile T = P.tiles[sg.x];
                if (zact_of(sg.y, sg.z))
                    cpml_produce_stages<R, true>(M, P, T, sg.y, sg.z, qbuf, B, peQ, pstage);
                else
                    cpml_produce_stages<R, false>(M, P, T, sg.y, sg.z, qbuf, B, peQ, pstage);
            }
        }
        return;
    }
    // ---- consumers
    uint32_t phP = 0, phQ = 0, phI = 0;
    int cslot = 0, cstage = 0;
    for (int n = 0;; ++n) {
        const int si = n % C::NI;
        mbar_wait(B.fullI + 8 * si, (phI >> si) & 1u);
        phI ^= 1u << si;
        const int4 sg = items[si];
        consumer_sync<C::NC>();  // every consumer has read the item
        if (tid == 0) mbar_arrive_b(B.emptyI + 8 * si);
        if (sg.x < 0) break;
        const CTile T = P.tiles[sg.x];
        if (zact_of(sg.y, sg.z))
            cpml_consume<R, ORD, true>(P, T, sg.y, sg.z, ring, qbuf, PXb, PYb, B, phP, phQ, cslot,
                                       cstage);
        else
            cpml_consume<R, ORD, false>(P, T, sg.y, sg.z, ring, qbuf, PXb, PYb, B, phP, phQ, cslot,
                                        cstage);
    }
    // last CTA out resets the work counter (WorkQueue: ctr[1] counts CTAs done)
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(P.wq.ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(P.wq.ctr, 0);
            atomicExch(P.wq.ctr + 1, 0);
        }
    }
}

}  // namespace fast
}  // namespace mmb
