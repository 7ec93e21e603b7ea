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
}

// ---------------------------------------------------------------- z columns
// k_zslab streams whole z columns of the inner x-y box: planes inside
// [zi_lo, zi_hi) get the plain update, the Z-slab planes outside it the pass-2
// formula along z (update_damping_pass2, propagator_impl.hpp:125-152; dpsi_x,
// dpsi_y, zeta_x, zeta_y are masked to 0 there).  Same 64 x 16 tiles and TMA
// pipeline as k_inner.  The z window is read from a ring of
// NS = 2R+1+lead shared slots (no register queue, so the loop is not unrolled
// and the code stays small), dpsi_z (k_p1) and zeta_z come straight from
// global memory.
template <int R>
struct ZSlabCfg {
    using I = InnerCfg<R>;
    static constexpr int NS = 2 * R + 1 + (R <= 4 ? 3 : 2);
    static constexpr int NQ = R <= 4 ? 4 : 2;
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(NS * I::PLANE + NQ * 2 * I::TILE) + 8 * (NS + NQ) + 16;
};

template <int R, int ORD>
__global__ void __launch_bounds__(InnerCfg<R>::NT, 1)
    k_zslab(const __grid_constant__ CUtensorMap tm_pc, const __grid_constant__ CUtensorMap tm_pp,
            const __grid_constant__ CUtensorMap tm_cv, const InnerParams P) {
    using C = InnerCfg<R>;
    using Z = ZSlabCfg<R>;
    constexpr int OC = ORD >= 1 ? ORD : 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + Z::NS * C::PLANE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + Z::NQ * 2 * C::TILE);
    const uint32_t barP = smem_u32(bars), barQ = smem_u32(bars + Z::NS);
    const int tid = threadIdx.x;
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const Layout L = P.lay;

    if (tid == 0) {
        prefetch_tmap(&tm_pc);
        prefetch_tmap(&tm_pp);
        prefetch_tmap(&tm_cv);
        for (int s = 0; s < Z::NS + Z::NQ; ++s) mbar_init(barP + 8 * s, 1);
        fence_barrier_init();
    }
    __syncthreads();

    uint32_t phP = 0, phQ = 0;
    unsigned qissue = 0, qcons = 0;
    __shared__ int s_item;
    const int soff = (R + ty) * C::BX + C::HX + 4 * tx;
    const int toff = ty * C::TX + 4 * tx;

    for (;;) {
        const int item = wq_next(P.wq, &s_item);
        if (item >= P.wq.nitems) break;
        const int4 sg = P.segs[item];
        const int x0 = P.x_base + sg.x * C::TX;
        const int y0 = P.lo[1] + sg.y * C::TY;
        const int zb = sg.z, ze = sg.w;
        const int nring = ze - zb + 2 * R;
        const int nout = ze - zb;
        const int tmx_halo = L.L + x0 - C::HX, tmy_halo = y0 - R + L.r;
        const int tmx = L.L + x0, tmy = y0 + L.r;
        auto issue_p = [&](int j, int slot) {
            const uint32_t bar = barP + 8 * slot;
            mbar_expect_tx(bar, C::BX * C::BY * 4);
            tma_load_3d(smem_u32(ring + slot * C::PLANE), &tm_pc, tmx_halo, tmy_halo,
                        zb - R + j + L.r, bar);
        };
        auto issue_q = [&](int o) {
            const int st = qissue % Z::NQ;
            const uint32_t bar = barQ + 8 * st;
            float* dst = qring + st * 2 * C::TILE;
            mbar_expect_tx(bar, 2 * C::TX * C::TY * 4);
            tma_load_3d(smem_u32(dst), &tm_pp, tmx, tmy, zb + o + L.r, bar);
            tma_load_3d(smem_u32(dst + C::TILE), &tm_cv, tmx, tmy, zb + o + L.r, bar);
            ++qissue;
        };
        if (tid == 0) {
            for (int j = 0; j < min(Z::NS, nring); ++j) issue_p(j, j);
            for (int o = 0; o < min(Z::NQ, nout); ++o) issue_q(o);
        }

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
        float4 nx_zz, nx_dz;
        float nx_a, nx_b, nx_k;
        if (nout > 0) load_cpml(0, nx_zz, nx_dz, nx_a, nx_b, nx_k);

        int slot = 0;  // ring slot of plane j (j mod NS)
#pragma unroll 1
        for (int j = 0; j < nring; ++j) {
            mbar_wait(barP + 8 * slot, (phP >> slot) & 1u);
            phP ^= 1u << slot;
            if (j >= 2 * R) {
                const int o = j - 2 * R;
                const int z = zb + o;
                const int zr = zrun_at(z);
                float* zz_p = zr >= 0 ? P.zrun[zr].zeta + run_off(P.zrun[zr], 2, xg, y, z) : nullptr;
                const float4 zz = nx_zz, dz = nx_dz;
                const float aza = nx_a, azb = nx_b, azk = nx_k;
                if (o + 1 < nout) load_cpml(o + 1, nx_zz, nx_dz, nx_a, nx_b, nx_k);
                int cu = slot - R;  // slot of the centre plane j - R
                if (cu < 0) cu += Z::NS;
                auto slot_of = [&](int m) {
                    int t = cu + m;
                    if (t >= Z::NS) t -= Z::NS;
                    if (t < 0) t += Z::NS;
                    return t;
                };
                const float* S = ring + cu * C::PLANE + soff;
                const int st = qcons % Z::NQ;
                mbar_wait(barQ + 8 * st, (phQ >> st) & 1u);
                phQ ^= 1u << st;
                const float* Qp = qring + st * 2 * C::TILE + toff;
                float xs[4 + 2 * C::HX];
#pragma unroll
                for (int h = 0; h < (4 + 2 * C::HX) / 4; ++h) {
                    const float4 v = lds4(S - C::HX + 4 * h);
                    xs[4 * h] = v.x;
                    xs[4 * h + 1] = v.y;
                    xs[4 * h + 2] = v.z;
                    xs[4 * h + 3] = v.w;
                }
                float two_p0[4], d2x[4] = {0.f, 0.f, 0.f, 0.f}, d2y[4] = {0.f, 0.f, 0.f, 0.f},
                                 d2z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int e = 0; e < 4; ++e) two_p0[e] = 2.0f * xs[C::HX + e];
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        d2x[e] = d2_term<OC>(d2x[e], P.cx[m - 1], xs[C::HX + e + m],
                                             xs[C::HX + e - m], two_p0[e]);
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float4 u = lds4(S + m * C::BX), d = lds4(S - m * C::BX);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        d2y[e] = d2_term<OC>(d2y[e], P.cy[m - 1], comp(u, e), comp(d, e), two_p0[e]);
                }
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float4 u = lds4(ring + slot_of(m) * C::PLANE + soff);
                    const float4 d = lds4(ring + slot_of(-m) * C::PLANE + soff);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        d2z[e] = d2_term<OC>(d2z[e], P.cz[m - 1], comp(u, e), comp(d, e), two_p0[e]);
                }
                const float4 pp = lds4(Qp);
                const float4 cv = lds4(Qp + C::TILE);
                float out[4], nzz[4];
                if (z >= P.zi_lo && z < P.zi_hi) {  // inner plane (update_plain)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        out[e] = acc<OC>(fs<OC>(two_p0[e], comp(pp, e)), comp(cv, e),
                                         fa<OC>(fa<OC>(d2x[e], d2y[e]), d2z[e]));
                    if (yok) st4(dst_base + (long long)o * L.plane, out, pok, pall);
                } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float drx = acc<OC>(0.0f, d2x[e], ikx[e]);
                    const float dry = acc<OC>(0.0f, d2y[e], iky);
                    const float drz = acc<OC>(comp(dz, e), d2z[e], azk);
                    nzz[e] = zr >= 0 ? acc<OC>(fm<OC>(aza, drz), azb, comp(zz, e)) : 0.0f;
                    const float lap = fa<OC>(fa<OC>(fa<OC>(drx, 0.0f), fa<OC>(dry, 0.0f)),
                                             fa<OC>(drz, nzz[e]));
                    out[e] = acc<OC>(fs<OC>(two_p0[e], comp(pp, e)), comp(cv, e), lap);
                }
                if (yok) {
                    st4(dst_base + (long long)o * L.plane, out, pok, pall);
                    if (zr >= 0) st4(zz_p, nzz, pok, pall);
                }
                }
                ++qcons;
            }
            __syncthreads();  // all threads are done with plane j-2R and stage o
            if (tid == 0 && j >= 2 * R) {
                const int jf = j - 2 * R + Z::NS;  // refill plane j-2R's slot
                if (jf < nring) {
                    int fs_ = slot - 2 * R;
                    if (fs_ < 0) fs_ += Z::NS;
                    issue_p(jf, fs_);
                }
                if (j - 2 * R + Z::NQ < nout) issue_q(j - 2 * R + Z::NQ);
            }
            if (++slot == Z::NS) slot = 0;
        }
        qissue = qcons;
    }
    wq_done(P.wq);
}

}  // namespace fast
}  // namespace mmb
