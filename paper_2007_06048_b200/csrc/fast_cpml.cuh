// fast_cpml.cuh -- the fused single-pass CPML kernel (k_cpml), MM_MODE_FAST.
//
// ref: update_damping_pass1 (propagator_impl.hpp:106-123) and
//      update_damping_pass2 (propagator_impl.hpp:125-152) of every damping
//      slab, plus update_plain (:89-104) for the inner points that share the
//      slab tiles; second_derivative_at / central_derivative_at
//      (stencil.hpp:86-99).
//
// One launch does both CPML passes: per (x, y) tile and z chunk it streams
// p_cur planes along z (the slowest device axis) and, per output plane k,
//   1. psi_x(k), psi_y(k) = b psi + a D1(p_cur(k)) for the tile's points in
//      an x / y damping run -> global (in place) and a shared exchange plane;
//   2. psi_z(k+R) = b psi + a D1_z(p_cur) -> a per-thread register window of
//      2R+1 planes (and, for owned planes, global);
//   3. one __syncthreads;
//   4. dpsi_x / dpsi_y from the exchange planes, dpsi_z from the window,
//      zeta, the Laplacian and p_next.
// No pass-1 state goes through HBM twice: psi is read and written once per
// point (the two-pass path read it again and wrote + read dpsi_z).
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
// dpsi_y in X and Y slabs, dpsi_z in every slab; inner points that fall in a
// slab tile get the plain Laplacian (the CPML formula with every CPML term
// masked to +0 and inv_kappa 1 -- identical bits, since a second-derivative
// sum is never -0).
//
// Hardware mapping: 512 threads (16 warps), one CTA per SM (221 KB shared
// memory); a 32 x 32 tile, each thread two consecutive x points (float2) of
// one row.  Thread 0 issues every TMA load: p_cur planes with their 4-column
// / R-row halo into a 16-slot ring (the 3R+1-plane window psi_z needs plus
// lead) and, per output plane, one stage of 32 x 32 boxes (p_prev, c, and the
// tile's psi / zeta run boxes; TMA's out-of-bounds zero fill is the runs'
// zero halo) into a 3-slot stage ring.  Stores are 8-byte STG per thread
// (128-byte rows per half warp).
#pragma once

#include "fast_common.cuh"

namespace mmb {
namespace fast {

template <int R>
struct CpmlCfg {
    static_assert(R <= 4, "k_cpml: the 3R+1-plane window of wider stencils does not fit");
    static constexpr int TXT = 16;           // threads per row, 2 x points each
    static constexpr int TX = 2 * TXT;       // 32
    static constexpr int TY = 32;
    static constexpr int NT = TXT * TY;      // 512
    static constexpr int HX = 4;             // x halo (16-byte TMA granule)
    static constexpr int BX = TX + 2 * HX;   // 40
    static constexpr int BY = TY + 2 * R;
    static constexpr int PLANE = pad32(BX * BY);
    static constexpr int NS = 16;            // p_cur ring slots
    static constexpr int TILE = TX * TY;     // one 32 x 32 stage box
    static constexpr int NQ = 3;             // stage slots
    static constexpr int NBOX = 8;           // pp, cv, psi_x, zeta_x, psi_y, zeta_y, zeta_z, psi_z
    static constexpr int QSLOT = NBOX * TILE;
    static constexpr int PXW = TX + 2 * HX;  // psi_x exchange row (zero pads)
    static constexpr int PXN = TY * PXW;
    static constexpr int PYN = (TY + 2 * R) * TX;
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(NS * PLANE + NQ * QSLOT + 2 * PXN + 2 * PYN) + 8 * (NS + NQ) + 16;
    static_assert(2 * R + R + 1 + 2 <= NS, "ring too shallow");
};

// Stage box order (offset = index * TILE).
enum { QB_PP = 0, QB_CV, QB_PSX, QB_ZX, QB_PSY, QB_ZY, QB_ZZ, QB_PSZ };

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
    CUtensorMap psi[3][2];   // TX x TY boxes of the runs (z: the read buffer)
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

__device__ __forceinline__ float2 lds2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void sts2(float* p, float a, float b) {
    *reinterpret_cast<float2*>(p) = make_float2(a, b);
}
__device__ __forceinline__ void stg2(float* p, const float (&v)[2], const bool (&ok)[2]) {
    if (ok[0] && ok[1])
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    else if (ok[0])
        p[0] = v[0];
    else if (ok[1])
        p[1] = v[1];
}
__device__ __forceinline__ float2 ldg2m(const float* p, const bool (&ok)[2]) {
    if (ok[0] && ok[1]) return __ldg(reinterpret_cast<const float2*>(p));
    float2 v = make_float2(0.f, 0.f);
    if (ok[0]) v.x = __ldg(p);
    if (ok[1]) v.y = __ldg(p + 1);
    return v;
}
__device__ __forceinline__ float c2of(const float2& v, int e) { return e == 0 ? v.x : v.y; }

__device__ __forceinline__ int zrun_at(const CpmlParams& P, int z) {
    return in_run(P.run[2][0], z) ? 0 : in_run(P.run[2][1], z) ? 1 : -1;
}

template <int R, int ORD>
__global__ void __launch_bounds__(CpmlCfg<R>::NT, 1)
    k_cpml(const __grid_constant__ CpmlMaps M, const CpmlParams P) {
    using C = CpmlCfg<R>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NS * C::PLANE;
    float* PXb = qring + C::NQ * C::QSLOT;  // 2 psi_x exchange planes
    float* PYb = PXb + 2 * C::PXN;          // 2 psi_y exchange planes
    uint64_t* bars = reinterpret_cast<uint64_t*>(PYb + 2 * C::PYN);
    const uint32_t barP = smem_u32(bars), barQ = smem_u32(bars + C::NS);
    const int tid = threadIdx.x;
    const int tx = tid % C::TXT, ty = tid / C::TXT;
    const Layout L = P.lay;

    if (tid == 0) {
        prefetch_tmap(&M.pc);
        prefetch_tmap(&M.pp);
        prefetch_tmap(&M.cv);
        for (int s = 0; s < C::NS + C::NQ; ++s) mbar_init(barP + 8 * s, 1);
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

    uint32_t phP = 0, phQ = 0;  // parity bit per ring / stage slot
    __shared__ int s_item;
    const int soff = (R + ty) * C::BX + C::HX + 2 * tx;  // centre in a p_cur plane
    const int toff = ty * C::TX + 2 * tx;                 // in a stage box
    const int pxo = ty * C::PXW + C::HX + 2 * tx;         // in a psi_x exchange plane
    const int pyo = (R + ty) * C::TX + 2 * tx;            // in a psi_y exchange plane

    for (;;) {
        const int item = wq_next(P.wq, &s_item);
        if (item >= P.wq.nitems) break;
        const int4 sg = P.items[item];
        const CTile T = P.tiles[sg.x];
        const int zb = sg.y, ze = sg.z;
        // psi_z is needed where a z run lies within R of the chunk's planes
        bool zact = false;
#pragma unroll
        for (int sd = 0; sd < 2; ++sd)
            zact = zact || near_run(P.run[2][sd], zb - R, ze + R);
        const int lag = zact ? 2 * R : R;  // output plane k <-> ring plane k + lag
        const int nring = ze - zb + 2 * lag;
        const int nout = ze - zb;
        const int zr0 = zb - lag;  // z of ring plane 0
        const bool fx = T.xside >= 0, fy = T.yside >= 0;
        const CpmlRun& RX = P.run[0][fx ? T.xside : 0];
        const CpmlRun& RY = P.run[1][fy ? T.yside : 0];

        auto issue_p = [&](int j) {
            const int slot = j % C::NS;
            const uint32_t bar = barP + 8 * slot;
            mbar_expect_tx(bar, 4u * C::BX * C::BY);
            tma_load_3d(smem_u32(ring + slot * C::PLANE), &M.pc, L.L + T.x0 - C::HX,
                        T.y0 - R + L.r, zr0 + j + L.r, bar);
        };
        auto issue_q = [&](int o) {
            const int st = o % C::NQ;
            const uint32_t bar = barQ + 8 * st;
            float* dst = qring + st * C::QSLOT;
            const int z = zb + o;
            const int zr = zrun_at(P, z);
            const int zp = zact ? zrun_at(P, z + R) : -1;
            uint32_t nb = 2 + (fx ? 2 : 0) + (fy ? 2 : 0) + (zr >= 0 ? 1 : 0) + (zp >= 0 ? 1 : 0);
            mbar_expect_tx(bar, nb * 4u * C::TILE);
            const int tmx = L.L + T.x0, tmy = T.y0 + L.r;
            tma_load_3d(smem_u32(dst + QB_PP * C::TILE), &M.pp, tmx, tmy, z + L.r, bar);
            tma_load_3d(smem_u32(dst + QB_CV * C::TILE), &M.cv, tmx, tmy, z + L.r, bar);
            if (fx) {
                tma_load_3d(smem_u32(dst + QB_PSX * C::TILE), &M.psi[0][T.xside], T.x0 - RX.org,
                            T.y0, z, bar);
                tma_load_3d(smem_u32(dst + QB_ZX * C::TILE), &M.zeta[0][T.xside], T.x0 - RX.org,
                            T.y0, z, bar);
            }
            if (fy) {
                tma_load_3d(smem_u32(dst + QB_PSY * C::TILE), &M.psi[1][T.yside], T.x0,
                            T.y0 - RY.org, z, bar);
                tma_load_3d(smem_u32(dst + QB_ZY * C::TILE), &M.zeta[1][T.yside], T.x0,
                            T.y0 - RY.org, z, bar);
            }
            if (zr >= 0)
                tma_load_3d(smem_u32(dst + QB_ZZ * C::TILE), &M.zeta[2][zr], T.x0, T.y0,
                            z - P.run[2][zr].org, bar);
            if (zp >= 0)
                tma_load_3d(smem_u32(dst + QB_PSZ * C::TILE), &M.psi[2][zp], T.x0, T.y0,
                            z + R - P.run[2][zp].org, bar);
        };
        if (tid == 0) {
            for (int j = 0; j < min(C::NS, nring); ++j) issue_p(j);
            for (int o = 0; o < min(C::NQ, nout); ++o) issue_q(o);
        }

        // ---- per-thread constants of this item
        const int xg = T.x0 + 2 * tx;
        const int y = T.y0 + ty;
        const bool yok = y >= T.oy0 && y < T.y1;
        bool pok[2], inX[2], rx[2];
        float axa[2] = {0.f, 0.f}, axb[2] = {1.f, 1.f}, axk[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int x = xg + e;
            pok[e] = yok && x >= T.ox0 && x < T.x1;
            inX[e] = x < P.ilo[0] || x >= P.ihi[0];
            rx[e] = fx && in_run(RX, x);
            const int xc = min(x, L.n[0] - 1);
            axk[e] = __ldg(P.tik[0] + xc);
            if (fx) {
                axa[e] = __ldg(P.ta[0] + xc);
                axb[e] = __ldg(P.tb[0] + xc);
            }
        }
        const bool rowY = y < P.ilo[1] || y >= P.ihi[1];
        const bool ry = fy && in_run(RY, y);
        const int yc = min(y, L.n[1] - 1);
        const float aya = __ldg(P.ta[1] + yc), ayb = __ldg(P.tb[1] + yc), ayk = __ldg(P.tik[1] + yc);
        float* const pn_b = P.pn + L.off(xg, y, zb);
        float* const psx_b = fx ? RX.psi + run_off(RX, 0, xg, y, zb) : nullptr;
        float* const zx_b = fx ? RX.zeta + run_off(RX, 0, xg, y, zb) : nullptr;
        float* const psy_b = fy ? RY.psi + run_off(RY, 1, xg, y, zb) : nullptr;
        float* const zy_b = fy ? RY.zeta + run_off(RY, 1, xg, y, zb) : nullptr;
        const long long sxz = fx ? RX.s2 : 0, syz = fy ? RY.s2 : 0;
        bool okx[2], oky[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            okx[e] = pok[e] && rx[e];
            oky[e] = pok[e] && ry;
        }

        float2 psw[2 * R + 1];  // psi_z planes k-R .. k+R of output plane k
#pragma unroll
        for (int i = 0; i <= 2 * R; ++i) psw[i] = make_float2(0.f, 0.f);

        int rel = 0;  // ring planes released (refilled) so far
#pragma unroll 1
        for (int j = 0; j < nring; ++j) {
            const int slot = j % C::NS;
            mbar_wait(barP + 8 * slot, (phP >> slot) & 1u);
            phP ^= 1u << slot;
            const int zj = zr0 + j;
            const bool outp = j >= 2 * lag;
            const int o = j - 2 * lag;  // output plane index (valid if outp)
            const int k = zb + o;
            const int st = (outp ? o : 0) % C::NQ;
            const float* Q = qring + st * C::QSLOT + toff;
            if (outp) {
                mbar_wait(barQ + 8 * st, (phQ >> st) & 1u);
                phQ ^= 1u << st;
            }

            // ---- psi_z(zj - R) into the window (update_damping_pass1, z axis)
            if (zact && j >= 2 * R) {
                const int pz = zj - R;
                float2 nv = make_float2(0.f, 0.f);
                const int zr = zrun_at(P, pz);
                if (zr >= 0) {
                    const CpmlRun& RZ = P.run[2][zr];
                    const int cs = (j - R) % C::NS;
                    float dp[2] = {0.f, 0.f};
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        const float2 u = lds2(ring + ((cs + m) % C::NS) * C::PLANE + soff);
                        const float2 d = lds2(ring + ((cs + C::NS - m) % C::NS) * C::PLANE + soff);
                        dp[0] = acc<ORD>(dp[0], P.c1[2][m - 1], fs<ORD>(u.x, d.x));
                        dp[1] = acc<ORD>(dp[1], P.c1[2][m - 1], fs<ORD>(u.y, d.y));
                    }
                    // old psi_z: from the stage of output plane pz - R, or (the
                    // chunk's first 2R planes) straight from the read buffer
                    const long long ro = run_off(RZ, 2, xg, y, pz);
                    float2 old;
                    if (outp)
                        old = lds2(Q + QB_PSZ * C::TILE);
                    else
                        old = ldg2m(RZ.psi + ro, pok);
                    const float az = __ldg(P.ta[2] + pz), bz = __ldg(P.tb[2] + pz);
                    // reference: psi = b * psi + a * dp  (propagator_impl.hpp:118-120)
                    nv.x = acc<ORD>(fm<ORD>(az, dp[0]), bz, old.x);
                    nv.y = acc<ORD>(fm<ORD>(az, dp[1]), bz, old.y);
                    if (pz >= zb && pz < ze) {
                        const float v[2] = {nv.x, nv.y};
                        stg2(RZ.psi + ro, v, pok);
                    }
                }
#pragma unroll
                for (int i = 0; i < 2 * R; ++i) psw[i] = psw[i + 1];
                psw[2 * R] = nv;
            }

            // ---- output plane k, before the exchange
            float two_p0[2], d2x[2] = {0.f, 0.f}, d2y[2] = {0.f, 0.f}, d2z[2] = {0.f, 0.f};
            const int xb = j & 1;  // exchange buffer of this iteration
            if (outp) {
                const int cs = (j - lag) % C::NS;  // ring slot of plane k
                const float* S = ring + cs * C::PLANE + soff;
                float xs[2 + 2 * C::HX];
#pragma unroll
                for (int h = 0; h < (2 + 2 * C::HX) / 2; ++h) {
                    const float2 v = lds2(S - C::HX + 2 * h);
                    xs[2 * h] = v.x;
                    xs[2 * h + 1] = v.y;
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) two_p0[e] = 2.0f * xs[C::HX + e];
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        d2x[e] = d2_term<ORD>(d2x[e], P.c2[0][m - 1], xs[C::HX + e + m],
                                              xs[C::HX + e - m], two_p0[e]);
                float d1y[2] = {0.f, 0.f};
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float2 u = lds2(S + m * C::BX), d = lds2(S - m * C::BX);
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        d2y[e] = d2_term<ORD>(d2y[e], P.c2[1][m - 1], c2of(u, e), c2of(d, e),
                                              two_p0[e]);
                        if (fy) d1y[e] = acc<ORD>(d1y[e], P.c1[1][m - 1], fs<ORD>(c2of(u, e), c2of(d, e)));
                    }
                }
#pragma unroll
                for (int m = 1; m <= R; ++m) {
                    const float2 u = lds2(ring + ((cs + m) % C::NS) * C::PLANE + soff);
                    const float2 d = lds2(ring + ((cs + C::NS - m) % C::NS) * C::PLANE + soff);
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        d2z[e] = d2_term<ORD>(d2z[e], P.c2[2][m - 1], c2of(u, e), c2of(d, e),
                                              two_p0[e]);
                }
                const long long fo = (long long)o;
                if (fx) {  // psi_x(k) of the tile's x run (pass 1)
                    const float2 old = lds2(Q + QB_PSX * C::TILE);
                    float nv[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        float dp = 0.f;
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            dp = acc<ORD>(dp, P.c1[0][m - 1], fs<ORD>(xs[C::HX + e + m], xs[C::HX + e - m]));
                        nv[e] = rx[e] ? acc<ORD>(fm<ORD>(axa[e], dp), axb[e], c2of(old, e)) : 0.0f;
                    }
                    sts2(PXb + xb * C::PXN + pxo, nv[0], nv[1]);
                    stg2(psx_b + fo * sxz, nv, okx);
                }
                if (fy) {  // psi_y(k) of the tile's y run (pass 1)
                    const float2 old = lds2(Q + QB_PSY * C::TILE);
                    float nv[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        nv[e] = ry ? acc<ORD>(fm<ORD>(aya, d1y[e]), ayb, c2of(old, e)) : 0.0f;
                    sts2(PYb + xb * C::PYN + pyo, nv[0], nv[1]);
                    stg2(psy_b + fo * syz, nv, oky);
                }
            }

            __syncthreads();  // exchange planes complete; iteration j-1 done everywhere
            if (tid == 0) {
                // ring planes no later iteration reads: index < j + 1 - lag - R
                const int upto = j + 1 - lag - R;
                for (; rel < upto; ++rel)
                    if (rel + C::NS < nring) issue_p(rel + C::NS);
                // the stage of output o - 1 is free
                if (outp && o >= 1 && o - 1 + C::NQ < nout) issue_q(o - 1 + C::NQ);
            }

            if (outp) {
                // ---- pass 2 at (x, y, k)
                const bool planeZ = k < P.ilo[2] || k >= P.ihi[2];
                const int zr = zrun_at(P, k);
                float dpx[2] = {0.f, 0.f}, dpy[2] = {0.f, 0.f}, dpz[2] = {0.f, 0.f};
                if (fx) {
                    float ps[2 + 2 * C::HX];
                    const float* X = PXb + xb * C::PXN + pxo;
#pragma unroll
                    for (int h = 0; h < (2 + 2 * C::HX) / 2; ++h) {
                        const float2 v = lds2(X - C::HX + 2 * h);
                        ps[2 * h] = v.x;
                        ps[2 * h + 1] = v.y;
                    }
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            dpx[e] = acc<ORD>(dpx[e], P.c1[0][m - 1],
                                              fs<ORD>(ps[C::HX + e + m], ps[C::HX + e - m]));
                        if (!inX[e]) dpx[e] = 0.0f;
                    }
                }
                if (fy) {
                    const float* Yp = PYb + xb * C::PYN + pyo;
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        const float2 u = lds2(Yp + m * C::TX), d = lds2(Yp - m * C::TX);
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            dpy[e] = acc<ORD>(dpy[e], P.c1[1][m - 1], fs<ORD>(c2of(u, e), c2of(d, e)));
                    }
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (!(inX[e] || rowY)) dpy[e] = 0.0f;
                }
                if (zact) {
#pragma unroll
                    for (int m = 1; m <= R; ++m)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            dpz[e] = acc<ORD>(dpz[e], P.c1[2][m - 1],
                                              fs<ORD>(c2of(psw[R + m], e), c2of(psw[R - m], e)));
                }
                const float2 pp = lds2(Q + QB_PP * C::TILE);
                const float2 cv = lds2(Q + QB_CV * C::TILE);
                float2 zx = make_float2(0.f, 0.f), zy = zx, zz = zx;
                if (fx) zx = lds2(Q + QB_ZX * C::TILE);
                if (fy) zy = lds2(Q + QB_ZY * C::TILE);
                if (zr >= 0) zz = lds2(Q + QB_ZZ * C::TILE);
                const float aza = __ldg(P.ta[2] + k), azb = __ldg(P.tb[2] + k),
                            azk = __ldg(P.tik[2] + k);
                float out[2], nzx[2], nzy[2], nzz[2];
                bool pst[2];  // p_next store: owned slab points (k_inner does the inner box)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const bool cp = inX[e] || rowY || planeZ;
                    pst[e] = pok[e] && cp;
                    if (!cp) dpz[e] = 0.0f;
                    // reference: drive = d2p*ik + dpsi; zeta = b*zeta + a*drive;
                    // term = drive + zeta; lap = (term_x + term_y) + term_z
                    const float drx = acc<ORD>(dpx[e], d2x[e], cp ? axk[e] : 1.0f);
                    const float dry = acc<ORD>(dpy[e], d2y[e], cp ? ayk : 1.0f);
                    const float drz = acc<ORD>(dpz[e], d2z[e], cp ? azk : 1.0f);
                    nzx[e] = rx[e] ? acc<ORD>(fm<ORD>(axa[e], drx), axb[e], c2of(zx, e)) : 0.0f;
                    nzy[e] = ry ? acc<ORD>(fm<ORD>(aya, dry), ayb, c2of(zy, e)) : 0.0f;
                    nzz[e] = zr >= 0 ? acc<ORD>(fm<ORD>(aza, drz), azb, c2of(zz, e)) : 0.0f;
                    const float lap = fa<ORD>(fa<ORD>(fa<ORD>(drx, nzx[e]), fa<ORD>(dry, nzy[e])),
                                              fa<ORD>(drz, nzz[e]));
                    out[e] = acc<ORD>(fs<ORD>(two_p0[e], c2of(pp, e)), c2of(cv, e), lap);
                }
                const long long fo = (long long)o;
                stg2(pn_b + fo * L.plane, out, pst);
                if (fx) stg2(zx_b + fo * sxz, nzx, okx);
                if (fy) stg2(zy_b + fo * syz, nzy, oky);
                if (zr >= 0) {
                    const CpmlRun& RZ = P.run[2][zr];
                    stg2(RZ.zeta + run_off(RZ, 2, xg, y, k), nzz, pok);
                }
            }
        }
    }
    wq_done(P.wq);
}

}  // namespace fast
}  // namespace mmb
