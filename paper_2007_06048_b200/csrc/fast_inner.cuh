// fast_inner.cuh -- the interior (inner-box) update kernel, MM_MODE_FAST.
//
// ref: AcousticCdEngine::update_plain (propagator_impl.hpp:89-104),
//      laplacian_at (stencil.hpp:70-82).
//
// 2.5D streaming along z (the slowest device axis).  One CTA per SM (16
// warps) pulls (tile, z-chunk) items from a work queue ordered so that the
// items in flight are neighbouring tiles at the same z (halos meet in L2).
//  * p_cur planes (64 x 32 tile + halo) arrive by TMA (cp.async.bulk.tensor,
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
    static constexpr int TR = R <= 4 ? 32 : 16;  // thread rows (one row each)
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
    int lo[3], hi[3];   // inner box, local coordinates
    int x_base;         // x of tile column 0 (multiple of 4)
    const int4* segs;   // work items (tile_x, tile_y, z_begin, z_end)
    WorkQueue wq;
    float* pn;
    float cx[kMaxR], cy[kMaxR], cz[kMaxR];
    float center;       // -2 (sum cx + sum cy + sum cz), ORD 0 only
};

template <int R, int ORD>
__global__ void __launch_bounds__(InnerCfg<R>::NT, 1)
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

}  // namespace fast
}  // namespace mmb
