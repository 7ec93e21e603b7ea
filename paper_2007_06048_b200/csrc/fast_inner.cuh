// fast_inner.cuh -- the interior (inner-box) update kernel, MM_MODE_FAST.
//
// ref: AcousticCdEngine::update_plain (propagator_impl.hpp:89-104),
//      laplacian_at (stencil.hpp:70-82).
//
// 2.5D streaming along z (the slowest device axis).  Two CTAs per SM (8
// warps each) pull (tile, z-chunk) items from a work queue ordered so that the
// items in flight are neighbouring tiles at the same z (halos meet in L2).
//  * p_cur planes (64 x 16 tile + halo) arrive by TMA (cp.async.bulk.tensor,
//    mbarrier complete_tx) into a ring of QW = 2R+1 shared slots; ring slot
//    == register-queue slot == plane index mod QW, so every shared address is
//    a compile-time offset (the z loop is unrolled by QW).
//  * p_prev and (dt2 vp) vp tiles arrive by TMA into an NQ-stage ring.
//  * z neighbours: per-thread register queue of QW planes (4 x-points,
//    float4); x/y neighbours: 128-bit shared loads; output: 128-bit stores.
//  * one elected thread issues the TMA loads after the per-plane barrier.
// (A warp-specialised producer/consumer variant with empty barriers was
// measured slower on B200: 212 vs 300 Gpts/s at 512^3.)
#pragma once

#include "fast_common.cuh"

namespace mmb {
namespace fast {

template <int R>
struct InnerCfg {
    static constexpr int TXT = 16;               // thread columns, 4 x-points each
    static constexpr int TX = 4 * TXT;           // 64
#ifndef MM_INNER_TR
#define MM_INNER_TR 16
#endif
    static constexpr int TR = R <= 4 ? MM_INNER_TR : 16;  // thread rows (one row each)
    static constexpr int MINB = TR == 32 ? 1 : 2;           // CTAs per SM
    static constexpr int TY = TR;
    static constexpr int NT = TXT * TR;          // 512 (16 warps) or 256 threads
    static constexpr int HX = R <= 4 ? 4 : 8;    // x halo in shared memory (float4 granules)
    static constexpr int BX = TX + 2 * HX;
    static constexpr int BY = TY + 2 * R;
    static constexpr int QW = 2 * R + 1;         // register queue depth == ring slots
    static constexpr int NQ = R <= 4 ? 5 : 3;    // p_prev / c stages
    static constexpr int PLANE = pad32(BX * BY);  // floats per ring slot (128B-aligned)
    static constexpr int TILE = pad32(TX * TY);   // floats per p_prev / c tile
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(QW * PLANE + NQ * 2 * TILE) + 8 * (QW + NQ) + 16;
};

struct InnerParams {
    Layout lay;
    int lo[3], hi[3];   // x-y box of the tiles (inner box), local coordinates
    int x_base;         // x of tile column 0 (multiple of 4)
    const int4* segs;   // work items (tile_x, tile_y, z_begin, z_end)
    WorkQueue wq;
    float* pn;
    float cx[kMaxR], cy[kMaxR], cz[kMaxR];
    float center;       // -2 (sum cx + sum cy + sum cz), ORD 0 only
    // Z slabs (the inner x-y box at planes outside [zi_lo, zi_hi)) are updated
    // here too, with the CPML pass-2 formula along z (update_damping_pass2,
    // propagator_impl.hpp:125-152): dpsi_z from k_p1, zeta_z in the z runs.
    int zi_lo, zi_hi;
    int zsplit;  // first local plane of the high z layer (a Z slab sees its own run only)
    const float* tik_x;
    const float* tik_y;
    const float* ta_z;
    const float* tb_z;
    const float* tik_z;
    CpmlRun zrun[2];
    const float* dpz[2];
    int dz_lo[2], dz_hi[2];
};

template <int R, int ORD>
__global__ void __launch_bounds__(InnerCfg<R>::NT, InnerCfg<R>::MINB)
    k_inner(const __grid_constant__ CUtensorMap tm_pc, const __grid_constant__ CUtensorMap tm_pp,
            const __grid_constant__ CUtensorMap tm_cv, const InnerParams P) {
    using C = InnerCfg<R>;
    MM_TRACE_BEGIN
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::QW * C::PLANE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + C::NQ * 2 * C::TILE);
    const uint32_t barP = smem_u32(bars), barQ = smem_u32(bars + C::QW);
    const int tid = threadIdx.x;
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const Layout L = P.lay;

    if (tid == 0) {
        prefetch_tmap(&tm_pc);
        prefetch_tmap(&tm_pp);
        prefetch_tmap(&tm_cv);
        for (int s = 0; s < C::QW + C::NQ; ++s) mbar_init(barP + 8 * s, 1);
        fence_barrier_init();
    }
    __syncthreads();

    uint32_t phP = 0;  // parity bit per ring slot
    uint32_t phQ = 0;  // parity bit per p_prev/c stage
    unsigned qissue = 0, qcons = 0;
    __shared__ int s_item;
    const int soff = (R + ty) * C::BX + C::HX + 4 * tx;  // in a p_cur plane
    const int toff = ty * C::TX + 4 * tx;                 // in a p_prev / c tile

    for (;;) {
        const int item = wq_next(P.wq, &s_item);
        if (item >= P.wq.nitems) break;
        const int4 sg = P.segs[item];
        const int x0 = P.x_base + sg.x * C::TX;
        const int y0 = P.lo[1] + sg.y * C::TY;
        const int zb = sg.z, ze = sg.w;
        const int nring = ze - zb + 2 * R;  // planes zb-R .. ze+R-1
        const int nout = ze - zb;
        const int tmx_halo = L.L + x0 - C::HX, tmy_halo = y0 - R + L.r;
        const int tmx = L.L + x0, tmy = y0 + L.r;
        auto issue_p = [&](int j, int slot) {  // ring plane j <-> z = zb - R + j
            const uint32_t bar = barP + 8 * slot;
            mbar_expect_tx(bar, C::BX * C::BY * 4);
            tma_load_3d(smem_u32(ring + slot * C::PLANE), &tm_pc, tmx_halo, tmy_halo,
                        zb - R + j + L.r, bar);
        };
        auto issue_q = [&](int o) {  // output plane o <-> z = zb + o
            const int st = qissue % C::NQ;
            const uint32_t bar = barQ + 8 * st;
            float* dst = qring + st * 2 * C::TILE;
            mbar_expect_tx(bar, 2 * C::TX * C::TY * 4);
            tma_load_3d(smem_u32(dst), &tm_pp, tmx, tmy, zb + o + L.r, bar);
            tma_load_3d(smem_u32(dst + C::TILE), &tm_cv, tmx, tmy, zb + o + L.r, bar);
            ++qissue;
        };
        if (tid == 0) {
            for (int j = 0; j < min(C::QW, nring); ++j) issue_p(j, j);
            for (int o = 0; o < min(C::NQ, nout); ++o) issue_q(o);
        }

        // output masks for this item
        const int xg = x0 + 4 * tx;
        const int y = y0 + ty;
        bool xok[4];
        bool xall = true;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            xok[e] = xg + e >= P.lo[0] && xg + e < P.hi[0];
            xall = xall && xok[e];
        }
        const bool yok = y >= P.lo[1] && y < P.hi[1];
        float* dst_base = P.pn + L.off(xg, y, zb);

        float4 q[C::QW];  // q[plane % QW]
        for (int jb = 0; jb < nring; jb += C::QW) {
#pragma unroll
            for (int u = 0; u < C::QW; ++u) {
                const int j = jb + u;
                if (j >= nring) break;
                mbar_wait(barP + 8 * u, (phP >> u) & 1u);
                phP ^= 1u << u;
                q[u] = lds4(ring + u * C::PLANE + soff);
                const int CU = (u + C::QW - R) % C::QW;  // slot of the centre plane j - R
                if (j >= 2 * R) {
                    const int o = j - 2 * R;
                    const float* S = ring + CU * C::PLANE + soff;
                    const int st = qcons % C::NQ;
                    mbar_wait(barQ + 8 * st, (phQ >> st) & 1u);
                    phQ ^= 1u << st;
                    const float* Qp = qring + st * 2 * C::TILE + toff;
                    float xs[4 + 2 * C::HX];
#pragma unroll
                    for (int h = 0; h < C::HX / 4; ++h) {
                        const float4 lft = lds4(S - C::HX + 4 * h);
                        const float4 rgt = lds4(S + 4 + 4 * h);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            xs[4 * h + e] = comp(lft, e);
                            xs[C::HX + 4 + 4 * h + e] = comp(rgt, e);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) xs[C::HX + e] = comp(q[CU], e);
                    float4 yu[R], yd[R];
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        yu[m - 1] = lds4(S + m * C::BX);
                        yd[m - 1] = lds4(S - m * C::BX);
                    }
                    const float4 pp = lds4(Qp);
                    const float4 cv = lds4(Qp + C::TILE);
                    float out[4];
#ifndef MM_INNER_SCALAR
                    if constexpr (ORD == 2) {
                        // lane pairs (x, x+1) = points (0,1) and (2,3): FADD2 /
                        // FFMA2 with every lane rounded like the scalar code
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int e = 2 * h;
                            const F2 two_p0 = fm2<ORD>(2.0f, f2(xs[C::HX + e], xs[C::HX + e + 1]));
                            F2 tx_ = f2zero(), ty_ = f2zero(), tz_ = f2zero();
#pragma unroll
                            for (int m = 1; m <= R; ++m) {
                                tx_ = d2_term2<ORD>(tx_, P.cx[m - 1],
                                                    f2(xs[C::HX + e + m], xs[C::HX + e + 1 + m]),
                                                    f2(xs[C::HX + e - m], xs[C::HX + e + 1 - m]),
                                                    two_p0);
                                ty_ = d2_term2<ORD>(ty_, P.cy[m - 1], half2(yu[m - 1], h),
                                                    half2(yd[m - 1], h), two_p0);
                                tz_ = d2_term2<ORD>(tz_, P.cz[m - 1], half2(q[(CU + m) % C::QW], h),
                                                    half2(q[(CU + C::QW - m) % C::QW], h), two_p0);
                            }
                            const F2 lap = fa2<ORD>(fa2<ORD>(tx_, ty_), tz_);
                            const F2 o2 = fa2<ORD>(fs2<ORD>(two_p0, half2(pp, h)),
                                                   fmul2<ORD>(half2(cv, h), lap));
                            unf2(o2, out[e], out[e + 1]);
                        }
                    } else
#endif
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float p0 = xs[C::HX + e];
                        const float two_p0 = 2.0f * p0;
                        float lap;
                        if (ORD >= 1) {
                            float tx_ = 0.0f, ty_ = 0.0f, tz_ = 0.0f;
#pragma unroll
                            for (int m = 1; m <= R; ++m) {
                                tx_ = d2_term<ORD>(tx_, P.cx[m - 1], xs[C::HX + e + m],
                                                 xs[C::HX + e - m], two_p0);
                                ty_ = d2_term<ORD>(ty_, P.cy[m - 1], comp(yu[m - 1], e),
                                                 comp(yd[m - 1], e), two_p0);
                                tz_ = d2_term<ORD>(tz_, P.cz[m - 1],
                                                 comp(q[(CU + m) % C::QW], e),
                                                 comp(q[(CU + C::QW - m) % C::QW], e), two_p0);
                            }
                            lap = fa<ORD>(fa<ORD>(tx_, ty_), tz_);
                        } else {
                            float t = P.center * p0;
#pragma unroll
                            for (int m = 1; m <= R; ++m) {
                                t = d2_term<0>(t, P.cx[m - 1], xs[C::HX + e + m],
                                               xs[C::HX + e - m], 0.0f);
                                t = d2_term<0>(t, P.cy[m - 1], comp(yu[m - 1], e),
                                               comp(yd[m - 1], e), 0.0f);
                                t = d2_term<0>(t, P.cz[m - 1], comp(q[(CU + m) % C::QW], e),
                                               comp(q[(CU + C::QW - m) % C::QW], e), 0.0f);
                            }
                            lap = t;
                        }
                        out[e] = ORD == 2 ? __fadd_rn(__fsub_rn(two_p0, comp(pp, e)), __fmul_rn(comp(cv, e), lap))
                                        : fmaf(comp(cv, e), lap, two_p0 - comp(pp, e));
                    }
                    if (yok) {
                        float* dst = dst_base + (long long)o * L.plane;
                        if (xall) {
                            *reinterpret_cast<float4*>(dst) =
                                make_float4(out[0], out[1], out[2], out[3]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (xok[e]) dst[e] = out[e];
                        }
                    }
                    ++qcons;
                }
                __syncthreads();  // all threads are done with plane j-R and stage o
                if (tid == 0) {
                    if (j >= R && j - R + C::QW < nring) issue_p(j - R + C::QW, CU);
                    if (j >= 2 * R && j - 2 * R + C::NQ < nout) issue_q(j - 2 * R + C::NQ);
                }
            }
        }
        // qissue is only advanced by thread 0; every thread's copy is reset here
        qissue = qcons;
    }
    wq_done(P.wq);
    MM_TRACE_END(2)
}

// ---------------------------------------------------------------- z columns
// k_zslab streams whole z columns of the inner x-y box: planes inside
// [zi_lo, zi_hi) get the plain update, the Z-slab planes outside it the pass-2
// formula along z (update_damping_pass2, propagator_impl.hpp:125-152; dpsi_x,
// dpsi_y, zeta_x, zeta_y are masked to 0 there).  It serves the inner box at
// r > 4 (k_inner's register queue would unroll the z loop 2R+1 = 17 deep and
// overflow the instruction cache) and, optionally, the Z slabs at r <= 4.
// Same 64 x 16 tiles as k_inner; the z window is read from a ring of
// NS = 2R+1+lead shared slots through a per-thread array of slot offsets
// rotated once per plane (no register queue, no unrolled loop, no modular
// slot arithmetic).  8 consumer warps + 1 producer warp: lane 0 pulls work
// items (4-slot item ring) and streams the p_cur ring, lane 1 the p_prev / c
// stages, each gated by its own empty barriers, so the consumers never issue
// TMA and the ring runs as far ahead as its depth allows.  dpsi_z (k_p1) and
// zeta_z come from global memory one plane ahead.  Arithmetic on lane pairs
// (FADD2), reference order (bit-exact for ORD 2).
template <int R>
struct ZSlabCfg {
    using I = InnerCfg<R>;
    static constexpr int NS = 2 * R + 1 + (R <= 4 ? 3 : 2);
    static constexpr int NQ = R <= 4 ? 4 : 3;
    static constexpr int NC = I::NT;       // consumer threads
    static constexpr int NT = NC + 32;     // + producer warp
    static constexpr int NI = 4;           // work-item slots
    static constexpr int NBAR = 2 * NS + 2 * NQ + 4 * NI;
    static constexpr size_t SMEM = sizeof(float) * (size_t)(NS * I::PLANE + NQ * 2 * I::TILE) +
                                   8 * NBAR + 16 * NI + 64;
};

template <int R, int ORD>
__global__ void __launch_bounds__(ZSlabCfg<R>::NT, 1)
    k_zslab(const __grid_constant__ CUtensorMap tm_pc, const __grid_constant__ CUtensorMap tm_pp,
            const __grid_constant__ CUtensorMap tm_cv, const InnerParams P) {
    using C = InnerCfg<R>;
    using Z = ZSlabCfg<R>;
    constexpr int OC = ORD >= 1 ? ORD : 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + Z::NS * C::PLANE;
    int4* items = reinterpret_cast<int4*>(qring + Z::NQ * 2 * C::TILE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(items + Z::NI);
    const uint32_t fullP = smem_u32(bars), emptyP = fullP + 8 * Z::NS;
    const uint32_t fullQ = emptyP + 8 * Z::NS, emptyQ = fullQ + 8 * Z::NQ;
    const uint32_t fullI = emptyQ + 8 * Z::NQ, emptyI = fullI + 8 * Z::NI;
    const uint32_t fullS = emptyI + 8 * Z::NI, emptyS = fullS + 8 * Z::NI;
    const int tid = threadIdx.x;
    const Layout L = P.lay;

    if (tid == 0) {
        prefetch_tmap(&tm_pc);
        prefetch_tmap(&tm_pp);
        prefetch_tmap(&tm_cv);
        for (int s = 0; s < Z::NBAR; ++s) mbar_init(fullP + 8 * s, 1);
        fence_barrier_init();
    }
    __syncthreads();

    if (tid >= Z::NC) {
        // ---- producer warp
        const int lane = tid - Z::NC;
        if (lane == 0) {  // items + the p_cur ring
            uint32_t peP = 0, peI = 0;
            int slot = 0;
            for (int n = 0;; ++n) {
                const int item = atomicAdd(P.wq.ctr, 1);
                const int si = n % Z::NI;
                const uint32_t par = ((peI >> si) & 1u) ^ 1u;
                mbar_wait_sleep(emptyI + 8 * si, par);
                mbar_wait_sleep(emptyS + 8 * si, par);
                peI ^= 1u << si;
                const int4 sg = item < P.wq.nitems ? P.segs[item] : make_int4(-1, 0, 0, 0);
                items[si] = sg;
                mbar_arrive_b(fullI + 8 * si);
                mbar_arrive_b(fullS + 8 * si);
                if (sg.x < 0) break;
                const int x0 = P.x_base + sg.x * C::TX, y0 = P.lo[1] + sg.y * C::TY;
                const int nring = sg.w - sg.z + 2 * R;
                for (int j = 0; j < nring; ++j) {
                    mbar_wait_sleep(emptyP + 8 * slot, ((peP >> slot) & 1u) ^ 1u);
                    peP ^= 1u << slot;
                    const uint32_t bar = fullP + 8 * slot;
                    mbar_expect_tx(bar, C::BX * C::BY * 4);
                    tma_load_3d(smem_u32(ring + slot * C::PLANE), &tm_pc, L.L + x0 - C::HX,
                                y0 - R + L.r, sg.z - R + j + L.r, bar);
                    slot = slot + 1 == Z::NS ? 0 : slot + 1;
                }
            }
        } else if (lane == 1) {  // p_prev / c stages
            uint32_t peQ = 0, phS = 0;
            int st = 0;
            for (int n = 0;; ++n) {
                const int si = n % Z::NI;
                mbar_wait_sleep(fullS + 8 * si, (phS >> si) & 1u);
                phS ^= 1u << si;
                const int4 sg = items[si];
                mbar_arrive_b(emptyS + 8 * si);
                if (sg.x < 0) break;
                const int tmx = L.L + P.x_base + sg.x * C::TX, tmy = P.lo[1] + sg.y * C::TY + L.r;
                for (int z = sg.z; z < sg.w; ++z) {
                    mbar_wait_sleep(emptyQ + 8 * st, ((peQ >> st) & 1u) ^ 1u);
                    peQ ^= 1u << st;
                    const uint32_t bar = fullQ + 8 * st;
                    float* dst = qring + st * 2 * C::TILE;
                    mbar_expect_tx(bar, 2 * C::TX * C::TY * 4);
                    tma_load_3d(smem_u32(dst), &tm_pp, tmx, tmy, z + L.r, bar);
                    tma_load_3d(smem_u32(dst + C::TILE), &tm_cv, tmx, tmy, z + L.r, bar);
                    st = st + 1 == Z::NQ ? 0 : st + 1;
                }
            }
        }
        return;
    }

    // ---- consumers
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const int soff = (R + ty) * C::BX + C::HX + 4 * tx;
    const int toff = ty * C::TX + 4 * tx;
    uint32_t phP = 0, phQ = 0, phI = 0;
    int cslot = 0, cst = 0;
    auto csync = [] { asm volatile("bar.sync 1, %0;" ::"n"(Z::NC) : "memory"); };

    for (int n = 0;; ++n) {
        const int si = n % Z::NI;
        mbar_wait(fullI + 8 * si, (phI >> si) & 1u);
        phI ^= 1u << si;
        const int4 sg = items[si];
        csync();  // every consumer has read the item
        if (tid == 0) mbar_arrive_b(emptyI + 8 * si);
        if (sg.x < 0) break;
        const int x0 = P.x_base + sg.x * C::TX;
        const int y0 = P.lo[1] + sg.y * C::TY;
        const int zb = sg.z, ze = sg.w;
        const int nring = ze - zb + 2 * R;
        const int nout = ze - zb;

        const int xg = x0 + 4 * tx;
        const int y = y0 + ty;
        const bool yok = y >= P.lo[1] && y < P.hi[1];
        bool pok[4];
        bool pall = yok;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            pok[e] = yok && xg + e >= P.lo[0] && xg + e < P.hi[0];
            pall = pall && pok[e];
        }
        float ikx[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) ikx[e] = __ldg(P.tik_x + min(xg + e, L.n[0] - 1));
        const float iky = __ldg(P.tik_y + min(max(y, 0), L.n[1] - 1));
        float* dst_base = P.pn + L.off(xg, y, zb);

        // point-wise CPML streams of output plane o (zeta_z, dpsi_z, z tables),
        // loaded one plane ahead so their latency hides behind a plane's work
        auto zrun_at = [&](int z) {
            return in_run(P.zrun[0], z) ? 0 : in_run(P.zrun[1], z) ? 1 : -1;
        };
        auto load_cpml = [&](int o, float4& zz, float4& dz, float& aza, float& azb, float& azk) {
            const int z = zb + o;
            if (z >= P.zi_lo && z < P.zi_hi) return;  // inner plane: plain update
            const int zr = zrun_at(z);
            int ze2 = z >= P.dz_lo[0] && z < P.dz_hi[0]   ? 0
                      : z >= P.dz_lo[1] && z < P.dz_hi[1] ? 1
                                                          : -1;
            if (ze2 != (z >= P.zsplit ? 1 : 0)) ze2 = -1;  // the other layer is halo
            zz = make_float4(0.f, 0.f, 0.f, 0.f);
            dz = zz;
            if (yok) {
                if (zr >= 0) zz = ld4(P.zrun[zr].zeta + run_off(P.zrun[zr], 2, xg, y, z), pok, pall);
                if (ze2 >= 0)
                    dz = ld4(P.dpz[ze2] + xg + (long long)y * P.zrun[ze2].s1 +
                                 (long long)(z - P.dz_lo[ze2]) * P.zrun[ze2].s2,
                             pok, pall);
            }
            aza = __ldg(P.ta_z + z);
            azb = __ldg(P.tb_z + z);
            azk = __ldg(P.tik_z + z);
        };
        float4 nx_zz = make_float4(0.f, 0.f, 0.f, 0.f), nx_dz = nx_zz;
        float nx_a = 0.f, nx_b = 1.f, nx_k = 1.f;
        if (nout > 0) load_cpml(0, nx_zz, nx_dz, nx_a, nx_b, nx_k);

        // slot offsets (floats) of planes j-2R .. j, oldest first
        int so[2 * R + 1];
#pragma unroll
        for (int i = 0; i <= 2 * R; ++i) so[i] = 0;
        int rslot = cslot;  // oldest ring slot not yet released
        const float* ringT = ring + soff;
        auto px = [](const float* v, int h, int m) {
            return f2(v[C::HX + 2 * h + m], v[C::HX + 2 * h + 1 + m]);
        };
#pragma unroll 1
        for (int j = 0; j < nring; ++j) {
            const int slot = cslot;
            cslot = cslot + 1 == Z::NS ? 0 : cslot + 1;
            mbar_wait(fullP + 8 * slot, (phP >> slot) & 1u);
            phP ^= 1u << slot;
#pragma unroll
            for (int i = 0; i < 2 * R; ++i) so[i] = so[i + 1];
            so[2 * R] = slot * C::PLANE;
            int st = -1;
            if (j >= 2 * R) {
                const int o = j - 2 * R;
                const int z = zb + o;
                const int zr = zrun_at(z);
                float* zz_p = zr >= 0 ? P.zrun[zr].zeta + run_off(P.zrun[zr], 2, xg, y, z) : nullptr;
                const float4 zz4 = nx_zz, dz4 = nx_dz;
                const float aza = nx_a, azb = nx_b, azk = nx_k;
                if (o + 1 < nout) load_cpml(o + 1, nx_zz, nx_dz, nx_a, nx_b, nx_k);
                st = cst;
                cst = cst + 1 == Z::NQ ? 0 : cst + 1;
                mbar_wait(fullQ + 8 * st, (phQ >> st) & 1u);
                phQ ^= 1u << st;
                const float* Qp = qring + st * 2 * C::TILE + toff;
                const float* S = ringT + so[R];  // centre plane j - R
                float xs[4 + 2 * C::HX];
#pragma unroll
                for (int h = 0; h < (4 + 2 * C::HX) / 4; ++h) {
                    const float4 v = lds4(S - C::HX + 4 * h);
                    xs[4 * h] = v.x;
                    xs[4 * h + 1] = v.y;
                    xs[4 * h + 2] = v.z;
                    xs[4 * h + 3] = v.w;
                }
                F2 two_p0[2], d2x[2], d2y[2], d2z[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const F2 c = px(xs, h, 0);
                    two_p0[h] = fa2<OC>(c, c);  // T(2) * c (exact)
                    d2x[h] = d2y[h] = d2z[h] = f2zero();
                }
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        d2x[h] = d2_term2<OC>(d2x[h], P.cx[m - 1], px(xs, h, m), px(xs, h, -m),
                                              two_p0[h]);
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    F2 u[2], d[2];
                    lds4x2(S + m * C::BX, u[0], u[1]);
                    lds4x2(S - m * C::BX, d[0], d[1]);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        d2y[h] = d2_term2<OC>(d2y[h], P.cy[m - 1], u[h], d[h], two_p0[h]);
                }
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    F2 u[2], d[2];
                    lds4x2(ringT + so[R + m], u[0], u[1]);
                    lds4x2(ringT + so[R - m], d[0], d[1]);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        d2z[h] = d2_term2<OC>(d2z[h], P.cz[m - 1], u[h], d[h], two_p0[h]);
                }
                F2 pp[2], cv[2];
                lds4x2(Qp, pp[0], pp[1]);
                lds4x2(Qp + C::TILE, cv[0], cv[1]);
                float out[4];
                if (z >= P.zi_lo && z < P.zi_hi) {  // inner plane (update_plain)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const F2 lap = fa2<OC>(fa2<OC>(d2x[h], d2y[h]), d2z[h]);
                        float c0, c1;
                        unf2(cv[h], c0, c1);
                        unf2(fa2<OC>(fs2<OC>(two_p0[h], pp[h]), fm2v<OC>(c0, c1, lap)),
                             out[2 * h], out[2 * h + 1]);
                    }
                    if (yok) st4(dst_base + (long long)o * L.plane, out, pok, pall);
                } else {
                    const F2 zz[2] = {f2(zz4.x, zz4.y), f2(zz4.z, zz4.w)};
                    const F2 dz[2] = {f2(dz4.x, dz4.y), f2(dz4.z, dz4.w)};
                    float nzz[4];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        // drive = d2p * ik + dpsi (dpsi_x, dpsi_y and zeta_x/y are 0 here)
                        const F2 drx = fa2<OC>(fm2v<OC>(ikx[2 * h], ikx[2 * h + 1], d2x[h]), f2zero());
                        const F2 dry = fa2<OC>(fm2<OC>(iky, d2y[h]), f2zero());
                        const F2 drz = fa2<OC>(fm2<OC>(azk, d2z[h]), dz[h]);
                        const F2 nz =
                            zr >= 0 ? fa2<OC>(fm2<OC>(aza, drz), fm2<OC>(azb, zz[h])) : f2zero();
                        unf2(nz, nzz[2 * h], nzz[2 * h + 1]);
                        const F2 lap = fa2<OC>(fa2<OC>(fa2<OC>(drx, f2zero()), fa2<OC>(dry, f2zero())),
                                               fa2<OC>(drz, nz));
                        float c0, c1;
                        unf2(cv[h], c0, c1);
                        unf2(fa2<OC>(fs2<OC>(two_p0[h], pp[h]), fm2v<OC>(c0, c1, lap)),
                             out[2 * h], out[2 * h + 1]);
                    }
                    if (yok) {
                        st4(dst_base + (long long)o * L.plane, out, pok, pall);
                        if (zr >= 0) st4(zz_p, nzz, pok, pall);
                    }
                }
            }
            csync();  // all consumers are done with plane j - 2R and stage st
            if (tid == 0) {
                if (j >= 2 * R) {
                    mbar_arrive_b(emptyP + 8 * rslot);
                    rslot = rslot + 1 == Z::NS ? 0 : rslot + 1;
                }
                if (st >= 0) mbar_arrive_b(emptyQ + 8 * st);
            }
        }
        // the item's last 2R ring planes
        if (tid == 0)
            for (int k = 0; k < min(2 * R, nring); ++k) {
                mbar_arrive_b(emptyP + 8 * rslot);
                rslot = rslot + 1 == Z::NS ? 0 : rslot + 1;
            }
    }
    // last CTA out resets the work counter
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(P.wq.ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(P.wq.ctr, 0);
            atomicExch(P.wq.ctr + 1, 0);
        }
    }
}


// ------------------------------------------------------------ wide stencils
// k_innerw: the inner box for R > 4 (update_plain, propagator_impl.hpp:89-104).
// k_inner's register queue needs its z loop unrolled 2R+1 deep so that every
// queue index is static (19 k instructions at R = 8: instruction-cache bound);
// the column kernel k_zslab keeps the z window in shared memory instead (38
// LDS.128 per thread-plane at R = 8: shared-memory-bandwidth bound).  Here the
// z window stays in registers: the z loop is unrolled U (4) planes deep and the
// queue shifted by moves once per U planes (2R float4 moves), so the loop
// body stays short; the x/y neighbours come
// from the centre plane's halo in shared memory, which therefore stays
// resident only from its arrival until it is the centre (R + 1 planes plus
// TMA lead) instead of the whole 2R+1 window.  One CTA of 12 warps per SM
// (64 x 24 tiles), registers up to 168 per thread.
template <int R>
struct InnerWCfg {
    static constexpr int TXT = 16;               // thread columns, 4 x-points each
    static constexpr int TX = 4 * TXT;           // 64
#ifndef MM_INNERW_TY
#define MM_INNERW_TY 24
#endif
    static constexpr int TY = MM_INNERW_TY;      // thread rows
    static constexpr int NT = TXT * TY;          // 384 threads
    static constexpr int HX = 8;                 // x halo in shared memory (2 float4)
    static constexpr int BX = TX + 2 * HX;
    static constexpr int BY = TY + 2 * R;
#ifndef MM_INNERW_U
#define MM_INNERW_U 4
#endif
    static constexpr int U = MM_INNERW_U;        // planes per register-queue shift
#ifndef MM_INNERW_LEAD
#define MM_INNERW_LEAD 3
#endif
    static constexpr int LEAD = MM_INNERW_LEAD;  // planes the TMA ring runs ahead
    static constexpr int NS = R + 1 + LEAD;      // ring slots: centre .. newest + lead
    static constexpr int NQ = 4;                 // p_prev / c stages
    static constexpr int PLANE = pad32(BX * BY);
    static constexpr int TILE = pad32(TX * TY);
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(NS * PLANE + NQ * 2 * TILE) + 8 * (NS + NQ) + 16;
};

template <int R, int ORD>
__global__ void __launch_bounds__(InnerWCfg<R>::NT, 1)
    k_innerw(const __grid_constant__ CUtensorMap tm_pc, const __grid_constant__ CUtensorMap tm_pp,
             const __grid_constant__ CUtensorMap tm_cv, const InnerParams P) {
    using C = InnerWCfg<R>;
    static_assert(C::NS <= 32 && C::NQ <= 32, "parity bit masks");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NS * C::PLANE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + C::NQ * 2 * C::TILE);
    const uint32_t barP = smem_u32(bars), barQ = smem_u32(bars + C::NS);
    const int tid = threadIdx.x;
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const Layout L = P.lay;

    if (tid == 0) {
        prefetch_tmap(&tm_pc);
        prefetch_tmap(&tm_pp);
        prefetch_tmap(&tm_cv);
        for (int s = 0; s < C::NS + C::NQ; ++s) mbar_init(barP + 8 * s, 1);
        fence_barrier_init();
    }
    __syncthreads();

    uint32_t phP = 0, phQ = 0;  // parity bit per ring slot / stage
    unsigned qissue = 0, qcons = 0;
    __shared__ int s_item;
    const int soff = (R + ty) * C::BX + C::HX + 4 * tx;  // in a p_cur plane
    const int toff = ty * C::TX + 4 * tx;                 // in a p_prev / c tile

    for (;;) {
        const int item = wq_next(P.wq, &s_item);
        if (item >= P.wq.nitems) break;
        const int4 sg = P.segs[item];
        const int x0 = P.x_base + sg.x * C::TX;
        const int y0 = P.lo[1] + sg.y * C::TY;
        const int zb = sg.z, ze = sg.w;
        const int nring = ze - zb + 2 * R;  // planes zb-R .. ze+R-1; plane j in slot j % NS
        const int nout = ze - zb;
        auto issue_p = [&](int j, int slot) {
            const uint32_t bar = barP + 8 * slot;
            mbar_expect_tx(bar, C::BX * C::BY * 4);
            tma_load_3d(smem_u32(ring + slot * C::PLANE), &tm_pc, L.L + x0 - C::HX, y0 - R + L.r,
                        zb - R + j + L.r, bar);
        };
        auto issue_q = [&](int o) {
            const int st = qissue % C::NQ;
            const uint32_t bar = barQ + 8 * st;
            float* dst = qring + st * 2 * C::TILE;
            mbar_expect_tx(bar, 2 * C::TX * C::TY * 4);
            tma_load_3d(smem_u32(dst), &tm_pp, L.L + x0, y0 + L.r, zb + o + L.r, bar);
            tma_load_3d(smem_u32(dst + C::TILE), &tm_cv, L.L + x0, y0 + L.r, zb + o + L.r, bar);
            ++qissue;
        };
        if (tid == 0) {
            for (int j = 0; j < min(C::NS, nring); ++j) issue_p(j, j);
            for (int o = 0; o < min(C::NQ, nout); ++o) issue_q(o);
        }

        const int xg = x0 + 4 * tx;
        const int y = y0 + ty;
        bool xok[4];
        bool xall = true;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            xok[e] = xg + e >= P.lo[0] && xg + e < P.hi[0];
            xall = xall && xok[e];
        }
        const bool yok = y >= P.lo[1] && y < P.hi[1];
        float* dst = P.pn + L.off(xg, y, zb);

        // register queue: q[k] = this thread's points in plane jb - 2R + k for
        // a block of U planes jb .. jb + U - 1 (static indices inside the
        // block), shifted by U after it: 2R float4 moves per U planes
        constexpr int U = C::U;
        float4 q[2 * R + U];
        int sj = 0;  // slot of plane j
        int sc = 0;  // slot of plane j - R (the centre once j >= 2R)
#pragma unroll 1
        for (int jb = 0; jb < nring; jb += U) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = jb + u;
                if (j >= nring) break;
                mbar_wait(barP + 8 * sj, (phP >> sj) & 1u);
                phP ^= 1u << sj;
                q[2 * R + u] = lds4(ring + sj * C::PLANE + soff);
                if (j >= 2 * R) {
                    const float* S = ring + sc * C::PLANE + soff;
                    const int st = qcons % C::NQ;
                    const float4 p0 = q[R + u];
                    float xs[4 + 2 * C::HX];  // x - HX .. x + 3 + HX
#pragma unroll
                    for (int h = 0; h < C::HX / 4; ++h) {
                        const float4 lft = lds4(S - C::HX + 4 * h);
                        const float4 rgt = lds4(S + 4 + 4 * h);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            xs[4 * h + e] = comp(lft, e);
                            xs[C::HX + 4 + 4 * h + e] = comp(rgt, e);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) xs[C::HX + e] = comp(p0, e);
                    F2 two_p0[2], tx_[2], ty_[2], tz_[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        two_p0[h] = fm2<ORD>(2.0f, half2(p0, h));
                        tx_[h] = ty_[h] = tz_[h] = f2zero();
                    }
                    // laplacian_at (stencil.hpp:70-82), every lane in the reference order
#pragma unroll
                    for (int m = 1; m <= R; ++m)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tx_[h] = d2_term2<ORD>(
                                tx_[h], P.cx[m - 1],
                                f2(xs[C::HX + 2 * h + m], xs[C::HX + 2 * h + 1 + m]),
                                f2(xs[C::HX + 2 * h - m], xs[C::HX + 2 * h + 1 - m]), two_p0[h]);
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        const float4 up = lds4(S + m * C::BX), dn = lds4(S - m * C::BX);
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            ty_[h] = d2_term2<ORD>(ty_[h], P.cy[m - 1], half2(up, h), half2(dn, h),
                                                   two_p0[h]);
                    }
#pragma unroll
                    for (int m = 1; m <= R; ++m)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tz_[h] = d2_term2<ORD>(tz_[h], P.cz[m - 1], half2(q[R + u + m], h),
                                                   half2(q[R + u - m], h), two_p0[h]);
                    mbar_wait(barQ + 8 * st, (phQ >> st) & 1u);
                    phQ ^= 1u << st;
                    const float* Qp = qring + st * 2 * C::TILE + toff;
                    const float4 pp = lds4(Qp), cv = lds4(Qp + C::TILE);
                    float out[4];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const F2 lap = fa2<ORD>(fa2<ORD>(tx_[h], ty_[h]), tz_[h]);
                        const F2 o2 = fa2<ORD>(fs2<ORD>(two_p0[h], half2(pp, h)),
                                               fmul2<ORD>(half2(cv, h), lap));
                        unf2(o2, out[2 * h], out[2 * h + 1]);
                    }
                    ++qcons;
                    if (yok) {
                        float* d = dst + (long long)(j - 2 * R) * L.plane;
                        if (xall) {
                            *reinterpret_cast<float4*>(d) =
                                make_float4(out[0], out[1], out[2], out[3]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (xok[e]) d[e] = out[e];
                        }
                    }
                }
                __syncthreads();  // plane j - R (slot sc) and stage st have had their last use
                if (tid == 0) {
                    if (j >= R && j - R + C::NS < nring) issue_p(j - R + C::NS, sc);
                    if (j >= 2 * R && j - 2 * R + C::NQ < nout) issue_q(j - 2 * R + C::NQ);
                }
                if (j >= R && ++sc == C::NS) sc = 0;
                if (++sj == C::NS) sj = 0;
            }
#pragma unroll
            for (int k = 0; k < 2 * R; ++k) q[k] = q[k + U];
        }
        qissue = qcons;
    }
    wq_done(P.wq);
}

}  // namespace fast
}  // namespace mmb
