// fast_pass1.cuh -- CPML pass 1, MM_MODE_FAST.
//
// ref: update_damping_pass1 (propagator_impl.hpp:106-123):
//        psi_a = b_a * psi_a + a_a * D1_a(p_cur)   over every damping run.
//
// k_p1: a persistent, warp-specialised TMA stream.  One work item is a run x a
// 32 x 16 x-y tile x a z chunk.  Producer lane 0 streams, per plane, the
// p_cur box the axis' first derivative needs (x halo for x runs, y halo for y
// runs, a 2R+1-plane ring for z runs), lane 1 the psi tiles, into shared
// memory; four consumer warps (one float4 of x points per thread) compute the new psi
// and store it with coalesced 16-byte global stores.  Bytes in flight are held
// by TMA, not registers, so the kernel streams at HBM rate.
#pragma once

#include "fast_common.cuh"

namespace mmb {
namespace fast {

#ifndef MM_P1_LEAD
#define MM_P1_LEAD 4
#endif
#ifndef MM_P1_NQ
#define MM_P1_NQ 8
#endif

// Z = true: the z-run items (2R+1-plane window, dpsi_z emission); Z = false:
// the x- and y-run items, which need no window and run many more CTAs per SM.
#ifndef MM_P1Z_TY
#define MM_P1Z_TY 16
#endif
#ifndef MM_P1X_TY
#define MM_P1X_TY 16
#endif

// z runs: x points per consumer thread.  2 (twice the warps per tile, half the
// serial work per warp and plane) measured slower: z items alone 27.7 vs 25.1
// us at 240^3, 66 vs 58 at 512^3 -- the items' chains are not bound by the
// work of one warp.
#ifndef MM_P1Z_PX
#define MM_P1Z_PX 4
#endif

template <int R, bool Z>
struct P1Cfg {
    static constexpr int TX = 32, TY = Z ? MM_P1Z_TY : MM_P1X_TY;
    static constexpr int PX = Z ? MM_P1Z_PX : 4;  // x points per consumer thread
    static constexpr int NC = (TX / PX) * TY;  // consumer threads
    static constexpr int NCW = NC / 32;
    static constexpr int NT = NC + 32;        // + producer warp
    static constexpr int HX = R <= 4 ? 4 : 8;  // x halo (16-byte aligned TMA starts)
    static constexpr int BXX = TX + 2 * HX;    // x-run p box width
    static constexpr int BYY = TY + 2 * R;     // y-run p box height
    static constexpr int PXN = BXX * TY, PYN = TX * BYY, PZN = TX * TY;
    static constexpr int PSLOT = pad32(PXN > PYN ? PXN : PYN);
    static constexpr int PSI_N = TX * TY, PSI = pad32(PSI_N);
    static constexpr int D = Z ? MM_P1_LEAD : 6;  // producer lead beyond the z window
    static constexpr int NS = (Z ? 2 * R + 1 : 1) + D;  // p slots
    static constexpr int NQ = Z ? MM_P1_NQ : 8;   // psi stages
    static constexpr int QLEAD = NQ - 1;
    static constexpr int NBAR = 2 * NS + 2 * NQ + 4;
    static constexpr size_t SMEM =
        sizeof(float) * (size_t)(NS * PSLOT + NQ * PSI) + 8 * NBAR + 64;
};

struct P1Maps {
    CUtensorMap px, py, pz;  // p_cur: x-run box, y-run box, plain tile
    CUtensorMap psi[3][2];
};

// One damping run as a box of points (local coordinates).
struct RunDesc {
    int ax, side;
    int lo[3], hi[3];
    int x_base;  // multiple of 4 (the run array origin for axis 0)
};

struct P1Params {
    Layout lay;
    RunDesc rd[6];
    CpmlRun run[3][2];
    const float* ta[3];
    const float* tb[3];
    float c1[3][kMaxR];
    const int4* items;  // (run | tile_x << 3, tile_y, z_begin, z_end)
    WorkQueue wq;
    // dpsi_z = D1_z(new psi_z) of each z run over its planes lo-R .. hi+R-1,
    // same x/y strides as the run's psi array (plane index z - (lo - R)).
    float* dpz[2];
};

template <int R, bool Z>
struct P1Tile {
    int ax, side, x0, y0, zb, ze, w, nring, nout;
    __device__ P1Tile(const P1Params& P, const int4& sg) {
        const RunDesc& d = P.rd[sg.x & 7];
        ax = d.ax;
        side = d.side;
        x0 = d.x_base + (sg.x >> 3) * P1Cfg<R, Z>::TX;
        y0 = d.lo[1] + sg.y * P1Cfg<R, Z>::TY;
        zb = sg.z;
        ze = sg.w;
        w = Z && ax == 2 ? R : 0;  // z window half-width
        nout = ze - zb;
        nring = nout + 2 * w;
    }
};

// Producer lanes: 1 = lane 0 streams items, the p_cur ring and the psi stages
// (a stage issued as the ring reaches it); 2 = lane 1 streams the psi stages.
#ifndef MM_P1_LANES
#define MM_P1_LANES 2
#endif
constexpr bool kSplitLanes = MM_P1_LANES == 2;

template <int R, int ORD, bool Z>
__global__ void __launch_bounds__(P1Cfg<R, Z>::NT)
    k_p1(const __grid_constant__ P1Maps M, const P1Params P) {
    using C = P1Cfg<R, Z>;
    MM_TRACE_BEGIN
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>(smem_raw);
    float* qring = ring + C::NS * C::PSLOT;
    uint64_t* bars = reinterpret_cast<uint64_t*>(qring + C::NQ * C::PSI);
    int4* items = reinterpret_cast<int4*>(bars + C::NBAR);
    const uint32_t fullP = smem_u32(bars), emptyP = fullP + 8 * C::NS;
    const uint32_t fullQ = emptyP + 8 * C::NS, emptyQ = fullQ + 8 * C::NQ;
    const uint32_t fullI = emptyQ + 8 * C::NQ, emptyI = fullI + 16;
    const int tid = threadIdx.x;
    const int warp = tid / 32, lane = tid % 32;
    const Layout L = P.lay;

    // the boundary kernel may be scheduled as soon as SMs free up (it waits
    // for this grid's results itself)
    grid_dep_launch();
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
            mbar_init(emptyI + 8 * s, C::NCW + (kSplitLanes ? 1 : 0));  // + the stage lane
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
                const int4 sg = item < P.wq.nitems ? P.items[item] : make_int4(0, 0, 0, -1);
                {
                    const int s = ni & 1;
                    mbar_wait_sleep(emptyI + 8 * s, ((ni >> 1) & 1) ^ 1);
                    items[s] = sg;
                    mbar_arrive_b(fullI + 8 * s);
                    ++ni;
                }
                if (sg.w < 0) break;
                const P1Tile<R, Z> T(P, sg);
                const CpmlRun& run = P.run[T.ax][T.side];
                const CUtensorMap* pmap = T.ax == 0 ? &M.px : T.ax == 1 ? &M.py : &M.pz;
                const uint32_t pbytes = 4u * (T.ax == 0 ? C::PXN : T.ax == 1 ? C::PYN : C::PZN);
                const int px = L.L + T.x0 - (T.ax == 0 ? C::HX : 0);
                const int py = T.y0 + L.r - (T.ax == 1 ? R : 0);
                // psi tile origin in the run array (run_off's coordinates)
                const int qx = T.x0 - (T.ax == 0 ? run.org : 0);
                const int qy = T.y0 - (T.ax == 1 ? run.org : 0);
                const int qz = T.ax == 2 ? run.org : 0;
                auto issue_q = [&](int o) {
                    const int s = nq % C::NQ;
                    mbar_wait_sleep(emptyQ + 8 * s, ((nq / C::NQ) & 1) ^ 1);
                    const uint32_t bar = fullQ + 8 * s;
                    mbar_expect_tx(bar, 4u * C::PSI_N);
                    tma_load_3d(smem_u32(qring + s * C::PSI), &M.psi[T.ax][T.side], qx, qy,
                                T.zb + o - qz, bar);
                    ++nq;
                };
                int oq = 0;
                for (int j = 0; j < T.nring; ++j) {
                    const int z = T.zb - T.w + j;
                    const int s = np % C::NS;
                    mbar_wait_sleep(emptyP + 8 * s, ((np / C::NS) & 1) ^ 1);
                    const uint32_t bar = fullP + 8 * s;
                    mbar_expect_tx(bar, pbytes);
                    tma_load_3d(smem_u32(ring + s * C::PSLOT), pmap, px, py, z + L.r, bar);
                    ++np;
                    if (!kSplitLanes)
                        for (; oq < T.nout && oq <= j - 2 * T.w + C::QLEAD; ++oq) issue_q(oq);
                }
                if (!kSplitLanes)
                    for (; oq < T.nout; ++oq) issue_q(oq);
            }
            __threadfence();
            if (atomicAdd(P.wq.ctr + 1, 1) == (int)gridDim.x - 1) {
                atomicExch(P.wq.ctr, 0);
                atomicExch(P.wq.ctr + 1, 0);
            }
        } else if (kSplitLanes && lane == 1) {
            // the psi stages, as far ahead as the stage ring allows (not gated
            // by the p_cur ring's progress)
            unsigned nq = 0, ni = 0;
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
                const P1Tile<R, Z> T(P, sg);
                const CpmlRun& run = P.run[T.ax][T.side];
                const int qx = T.x0 - (T.ax == 0 ? run.org : 0);
                const int qy = T.y0 - (T.ax == 1 ? run.org : 0);
                const int qz = T.ax == 2 ? run.org : 0;
                for (int o = 0; o < T.nout; ++o) {
                    const int s = nq % C::NQ;
                    mbar_wait_sleep(emptyQ + 8 * s, ((nq / C::NQ) & 1) ^ 1);
                    const uint32_t bar = fullQ + 8 * s;
                    mbar_expect_tx(bar, 4u * C::PSI_N);
                    tma_load_3d(smem_u32(qring + s * C::PSI), &M.psi[T.ax][T.side], qx, qy,
                                T.zb + o - qz, bar);
                    ++nq;
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int tx = tid % (C::TX / C::PX), ty = tid / (C::TX / C::PX);
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
        const P1Tile<R, Z> T(P, sg);
        const int ax = T.ax;
        const RunDesc& d = P.rd[sg.x & 7];
        const CpmlRun& run = P.run[ax][T.side];
        const int x = T.x0 + C::PX * tx, y = T.y0 + ty;
        bool ok[C::PX];
        bool all = true, any = false;
#pragma unroll
        for (int e = 0; e < C::PX; ++e) {
            ok[e] = x + e >= d.lo[0] && x + e < d.hi[0] && y >= d.lo[1] && y < d.hi[1];
            all = all && ok[e];
            any = any || ok[e];
        }
        float c1[R];
#pragma unroll
        for (int m = 0; m < R; ++m) c1[m] = P.c1[ax][m];
        // damping coefficients: per x (x runs), per y (y runs), per z (z runs)
        float av[C::PX], bv[C::PX];
        if (ax == 0) {
#pragma unroll
            for (int e = 0; e < C::PX; ++e) {
                const int xc = min(max(x + e, 0), L.n[0] - 1);
                av[e] = __ldg(P.ta[0] + xc);
                bv[e] = __ldg(P.tb[0] + xc);
            }
        } else {
            const int yc = min(max(y, 0), L.n[1] - 1);
            const float a = ax == 1 ? __ldg(P.ta[1] + yc) : 0.f;
            const float b = ax == 1 ? __ldg(P.tb[1] + yc) : 0.f;
#pragma unroll
            for (int e = 0; e < C::PX; ++e) {
                av[e] = a;
                bv[e] = b;
            }
        }
        float* dst = run.psi + run_off(run, ax, x, y, T.zb);
        const long long zstep = run.s2;
        // offset of this thread's 4 points in a p slot
        const int poff = ax == 0 ? ty * C::BXX + C::HX + C::PX * tx
                         : ax == 1 ? (ty + R) * C::TX + C::PX * tx
                                   : ty * C::TX + C::PX * tx;
        const int qoff = ty * C::TX + C::PX * tx;
        if constexpr (Z) {
            // z runs (an item covers the whole run, zb = lo, ze = hi).  The
            // new psi_z of this thread's points rides a register queue
            // zq[k] = plane o-1-2R+k (zeros outside the run), from which dpsi_z
            // at plane o-1-R is emitted while plane o is computed; the
            // p_cur z window is addressed through rotating slot offsets.
            constexpr int NPR = C::PX / 2;  // lane pairs per thread
            F2 zq[2 * R + 1][NPR];
#pragma unroll
            for (int k = 0; k <= 2 * R; ++k)
#pragma unroll
                for (int h = 0; h < NPR; ++h) zq[k][h] = f2zero();
            // PX points from / to shared or global memory as lane pairs
            auto ldp = [](const float* q, F2 (&v)[NPR]) {
#pragma unroll
                for (int h = 0; h < NPR; ++h) v[h].r = reinterpret_cast<const unsigned long long*>(q)[h];
            };
            auto stp = [&](float* q, const F2 (&v)[NPR]) {
                if (all) {
                    if constexpr (NPR == 2) {
                        *reinterpret_cast<float4*>(q) = f4(v[0], v[1]);
                    } else {
#pragma unroll
                        for (int h = 0; h < NPR; ++h)
                            reinterpret_cast<unsigned long long*>(q)[h] = v[h].r;
                    }
                } else if (any) {
#pragma unroll
                    for (int h = 0; h < NPR; ++h) {
                        float a0, a1;
                        unf2(v[h], a0, a1);
                        if (ok[2 * h]) q[2 * h] = a0;
                        if (ok[2 * h + 1]) q[2 * h + 1] = a1;
                    }
                }
            };
            float* dz_p = P.dpz[T.side] + x + (long long)y * run.s1;  // plane od = -R
            auto emit_dpz = [&]() {  // dpsi_z at queue centre (plane od)
                F2 dz[NPR];
#pragma unroll
                for (int h = 0; h < NPR; ++h) dz[h] = f2zero();  // lane pairs (x, x+1), ...
#pragma unroll
                for (int m = 1; m <= R; ++m)
#pragma unroll
                    for (int h = 0; h < NPR; ++h)
                        dz[h] = d1_term2<ORD>(dz[h], c1[m - 1], zq[R + m][h], zq[R - m][h]);
                stp(dz_p, dz);
                dz_p += run.s2;
            };
            int wo[2 * R + 1];     // p_cur slot offsets of planes j-2R .. j
            int rel = (int)(np % C::NS);  // slot of the oldest window plane
            int sl = rel;                 // slot of plane j
            unsigned ph = (np / C::NS) & 1;
#pragma unroll 1
            for (int j = 0; j < T.nring; ++j) {
#pragma unroll
                for (int k = 0; k < 2 * R; ++k) wo[k] = wo[k + 1];
                wo[2 * R] = sl * C::PSLOT + poff;
                mbar_wait(fullP + 8 * sl, ph);
                if (j >= 2 * R) {
                    const int o = j - 2 * R;
                    const int z = T.zb + o;
                    // dpsi_z of plane o-1-R first: its window ends at plane o-1, so
                    // it is independent of this plane's psi (more ILP per plane)
                    if (o > 0) emit_dpz();
                    const float az = __ldg(P.ta[2] + z), bz = __ldg(P.tb[2] + z);
                    F2 dp[NPR];
#pragma unroll
                    for (int h = 0; h < NPR; ++h) dp[h] = f2zero();
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        F2 u[NPR], dn[NPR];
                        ldp(ring + wo[R + m], u);
                        ldp(ring + wo[R - m], dn);
#pragma unroll
                        for (int h = 0; h < NPR; ++h)
                            dp[h] = d1_term2<ORD>(dp[h], c1[m - 1], u[h], dn[h]);
                    }
                    const int st = nq % C::NQ;
                    mbar_wait(fullQ + 8 * st, (nq / C::NQ) & 1);
                    F2 v[NPR];
                    ldp(qring + st * C::PSI + qoff, v);
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive_b(emptyQ + 8 * st);
                        mbar_arrive_b(emptyP + 8 * rel);  // plane j - 2R has had its last use
                    }
                    ++nq;
                    if (++rel == C::NS) rel = 0;
                    // reference: psi = b * psi + a * dp  (propagator_impl.hpp:118-120)
#pragma unroll
                    for (int h = 0; h < NPR; ++h) v[h] = acc2<ORD>(fm2<ORD>(az, dp[h]), bz, v[h]);
                    stp(dst + (long long)o * zstep, v);
#pragma unroll
                    for (int k = 0; k < 2 * R; ++k)
#pragma unroll
                        for (int h = 0; h < NPR; ++h) zq[k][h] = zq[k + 1][h];
#pragma unroll
                    for (int h = 0; h < NPR; ++h) zq[2 * R][h] = v[h];
                }
                ++np;
                if (++sl == C::NS) sl = 0, ph ^= 1;
            }
            // the last plane's dpsi_z, then the planes whose window reaches
            // past the run (psi_z = 0 there)
            emit_dpz();
#pragma unroll 1
            for (int t = 0; t < 2 * R; ++t) {
#pragma unroll
                for (int k = 0; k < 2 * R; ++k)
#pragma unroll
                    for (int h = 0; h < NPR; ++h) zq[k][h] = zq[k + 1][h];
#pragma unroll
                for (int h = 0; h < NPR; ++h) zq[2 * R][h] = f2zero();
                emit_dpz();
            }
#pragma unroll 1
            for (int k = 0; k < 2 * R; ++k) {  // the item's last 2R planes
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyP + 8 * rel);
                if (++rel == C::NS) rel = 0;
            }
        } else {
        auto store4 = [&](float* q, const float4& v) {
            if (all) {
                *reinterpret_cast<float4*>(q) = v;
            } else if (any) {
                if (ok[0]) q[0] = v.x;
                if (ok[1]) q[1] = v.y;
                if (ok[2]) q[2] = v.z;
                if (ok[3]) q[3] = v.w;
            }
        };
#pragma unroll 1
        for (int j = 0; j < T.nring; ++j) {
            const int s = np % C::NS;
            mbar_wait(fullP + 8 * s, (np / C::NS) & 1);
            if (j >= 2 * T.w) {
                const int o = j - 2 * T.w;
                const int z = T.zb + o;
                if (ax == 2) {
                    const float a = __ldg(P.ta[2] + z), b = __ldg(P.tb[2] + z);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        av[e] = a;
                        bv[e] = b;
                    }
                }
                const int cs = (np + C::NS - T.w) % C::NS;  // slot of plane j - w
                auto slot_of = [&](int m) {                 // slot of plane j - w + m
                    const int t = cs + m;
                    return t < 0 ? t + C::NS : t >= C::NS ? t - C::NS : t;
                };
                F2 dp[2] = {f2zero(), f2zero()};  // lane pairs (x, x+1), (x+2, x+3)
                const float* S = ring + cs * C::PSLOT + poff;
                if (ax == 0) {
                    constexpr int H = C::HX;
                    float v[4 + 2 * H];
#pragma unroll
                    for (int h = 0; h < (4 + 2 * H) / 4; ++h) {
                        const float4 t = lds4(S - H + 4 * h);
                        v[4 * h] = t.x;
                        v[4 * h + 1] = t.y;
                        v[4 * h + 2] = t.z;
                        v[4 * h + 3] = t.w;
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int m = 1; m <= R; ++m)
                            dp[h] = d1_term2<ORD>(dp[h], c1[m - 1],
                                                  f2(v[H + 2 * h + m], v[H + 2 * h + 1 + m]),
                                                  f2(v[H + 2 * h - m], v[H + 2 * h + 1 - m]));
                } else {
#pragma unroll
                    for (int m = 1; m <= R; ++m) {
                        const float4 u4 = ax == 1 ? lds4(S + m * C::TX)
                                                  : lds4(ring + slot_of(m) * C::PSLOT + poff);
                        const float4 d4 = ax == 1 ? lds4(S - m * C::TX)
                                                  : lds4(ring + slot_of(-m) * C::PSLOT + poff);
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            dp[h] = d1_term2<ORD>(dp[h], c1[m - 1], half2(u4, h), half2(d4, h));
                    }
                }
                const int st = nq % C::NQ;
                mbar_wait(fullQ + 8 * st, (nq / C::NQ) & 1);
                float4 v = lds4(qring + st * C::PSI + qoff);
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyQ + 8 * st);
                ++nq;
                // reference: psi = b * psi + a * dp  (propagator_impl.hpp:118-120)
                v = f4(acc2v<ORD>(fm2v<ORD>(av[0], av[1], dp[0]), bv[0], bv[1], half2(v, 0)),
                       acc2v<ORD>(fm2v<ORD>(av[2], av[3], dp[1]), bv[2], bv[3], half2(v, 1)));
                store4(dst + (long long)o * zstep, v);
                // plane j - 2w has had its last use
                __syncwarp();
                if (lane == 0) mbar_arrive_b(emptyP + 8 * slot_of(-T.w));
            }
            ++np;
        }
#pragma unroll 1
        for (int k = 2 * T.w; k >= 1; --k) {  // the item's last 2w planes
            __syncwarp();
            if (lane == 0) mbar_arrive_b(emptyP + 8 * ((np + C::NS - k) % C::NS));
        }
        }  // if constexpr (Z)
    }
    MM_TRACE_END(Z ? 0 : 1)
}

}  // namespace fast
}  // namespace mmb
