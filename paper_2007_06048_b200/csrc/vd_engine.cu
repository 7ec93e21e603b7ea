// vd_engine.cu -- the acoustic_iso (variable-density) engine on the GPU.
//
// AcousticVdEngine<float> (ref: propagator.hpp:147-176,
// propagator_impl.hpp:175-295).  First-order pressure-velocity system on a
// staggered grid:
//   velocity:  dp_ax = D+_ax p            (staggered_derivative_at Forward)
//              v_ax += (dt / rho) * dp_ax
//   pressure:  dv_ax = D-_ax v_ax          (Backward)
//              p    += (dt * ((rho vp) vp)) * ((dv_x + dv_y) + dv_z)
// and, in the damping boxes, the CPML recursion on every derivative term
//   psi = b psi + a d;  d = d ik + psi.
//
// Device layout: the engine-wide one (mm_internal.hpp, x fastest, z slowest).
// Two kernels per step (vd_fast.cuh): k_vdv (velocity) and k_vdp (pressure),
// TMA-fed 2.5D sweeps along z.  Bytes per point and step (compulsory):
// velocity p, dt/rho, v (r+w) = 32 B; pressure v, dtb, p (r+w) = 24 B --
// 56 B against the reference cost model's fused 40 B (bench.cpp:97), see
// DESIGN.md.  The one-thread-per-point kernels below (k_vd_velocity /
// k_vd_pressure) are the plain restatement, kept for A/B checks
// (MM_VD_SIMPLE=1); both families are bit-identical.
//
// CPML memory lives only where it can be non-zero: one array per axis, per
// damping layer along that axis and per pass (the "runs" of mm_internal.hpp).
// The reference keeps psi over whole damping boxes (FoDampRegion<T, 6>); on
// the rest of a box a = 0 and b = ik = 1, so its psi stays +0 and
// d * 1 + (+0) leaves every update unchanged (v and p never hold -0): the
// results are bit-identical for finite data.
//
// Arithmetic: explicit round-to-nearest intrinsics in the reference's
// association order, built with -fmad=false (no contraction).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/minimod_b200.h"
#include "mm_fast.hpp"
#include "mm_internal.hpp"
#include "vd_fast.cuh"

namespace mmb {
namespace vd {

__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }

struct VdParams {
    Layout lay;
    int nd[3];  // inner box = [nd, n - nd) per axis (grid.cpp:24-45)
    float* p;
    float* v[3];
    const float* ir;   // dt / rho
    const float* dtb;  // dt * ((rho * vp) * vp)
    float w[3][kMaxR];  // staggered taps per axis (1/h folded)
    const float* ta[3];
    const float* tb[3];
    const float* tik[3];
    CpmlRun run[3][2];  // psi of the pass being launched, [axis][layer]
    int zc;             // z planes per block
};

constexpr int BX = 32, BY = 8;

// CPML on one derivative term (propagator_impl.hpp:231-238 / :260-267).
__device__ __forceinline__ float cpml_term(float d, const CpmlRun& r0, const CpmlRun& r1, int ax,
                                           int c, int i, int j, int k, float a, float b,
                                           float ik) {
    float* ps = nullptr;
    if (c >= r0.lo && c < r0.hi)
        ps = r0.psi + run_off(r0, ax, i, j, k);
    else if (c >= r1.lo && c < r1.hi)
        ps = r1.psi + run_off(r1, ax, i, j, k);
    const float old = ps ? *ps : 0.0f;
    const float psi = fa(fm(b, old), fm(a, d));
    if (ps) *ps = psi;
    return fa(fm(d, ik), psi);
}

// update_velocity (propagator_impl.hpp:214-244) on every interior point.
template <int R>
__global__ void __launch_bounds__(BX* BY) k_vd_velocity(const VdParams P) {
    const Layout L = P.lay;
    const int i = blockIdx.x * BX + threadIdx.x;
    const int j = blockIdx.y * BY + threadIdx.y;
    if (i >= L.n[0] || j >= L.n[1]) return;
    const int k0 = blockIdx.z * P.zc, k1 = min(k0 + P.zc, L.n[2]);
    const long long pl = L.plane, sy = L.P;
    const float* __restrict__ p = P.p;
    long long o = L.off(i, j, k0);
    // z window of p: q[t] = p(k - R + 1 + t), t = 0 .. 2R-1
    float q[2 * R];
#pragma unroll
    for (int t = 0; t < 2 * R - 1; ++t) q[t] = __ldg(p + o + (t - R + 1) * pl);
    const bool xy_in = i >= P.nd[0] && i < L.n[0] - P.nd[0] && j >= P.nd[1] &&
                       j < L.n[1] - P.nd[1];
    const float ax_a = __ldg(P.ta[0] + i), ax_b = __ldg(P.tb[0] + i), ax_k = __ldg(P.tik[0] + i);
    const float ay_a = __ldg(P.ta[1] + j), ay_b = __ldg(P.tb[1] + j), ay_k = __ldg(P.tik[1] + j);
    for (int k = k0; k < k1; ++k, o += pl) {
        q[2 * R - 1] = __ldg(p + o + R * pl);
        float d[3] = {0.0f, 0.0f, 0.0f};
        // staggered_derivative_at Forward: t += c_m (f[m s] - f[(1-m) s])
#pragma unroll
        for (int m = 1; m <= R; ++m)
            d[0] = fa(d[0], fm(P.w[0][m - 1], fs(__ldg(p + o + m), __ldg(p + o + 1 - m))));
#pragma unroll
        for (int m = 1; m <= R; ++m)
            d[1] = fa(d[1], fm(P.w[1][m - 1],
                               fs(__ldg(p + o + m * sy), __ldg(p + o + (1 - m) * sy))));
#pragma unroll
        for (int m = 1; m <= R; ++m) d[2] = fa(d[2], fm(P.w[2][m - 1], fs(q[R - 1 + m], q[R - m])));
        if (!(xy_in && k >= P.nd[2] && k < L.n[2] - P.nd[2])) {
            d[0] = cpml_term(d[0], P.run[0][0], P.run[0][1], 0, i, i, j, k, ax_a, ax_b, ax_k);
            d[1] = cpml_term(d[1], P.run[1][0], P.run[1][1], 1, j, i, j, k, ay_a, ay_b, ay_k);
            d[2] = cpml_term(d[2], P.run[2][0], P.run[2][1], 2, k, i, j, k, __ldg(P.ta[2] + k),
                             __ldg(P.tb[2] + k), __ldg(P.tik[2] + k));
        }
        const float ir = __ldg(P.ir + o);
#pragma unroll
        for (int a = 0; a < 3; ++a) P.v[a][o] = fa(P.v[a][o], fm(ir, d[a]));
#pragma unroll
        for (int t = 0; t < 2 * R - 1; ++t) q[t] = q[t + 1];
    }
}

// update_pressure (propagator_impl.hpp:246-273) on every interior point.
template <int R>
__global__ void __launch_bounds__(BX* BY) k_vd_pressure(const VdParams P) {
    const Layout L = P.lay;
    const int i = blockIdx.x * BX + threadIdx.x;
    const int j = blockIdx.y * BY + threadIdx.y;
    if (i >= L.n[0] || j >= L.n[1]) return;
    const int k0 = blockIdx.z * P.zc, k1 = min(k0 + P.zc, L.n[2]);
    const long long pl = L.plane, sy = L.P;
    const float* __restrict__ vx = P.v[0];
    const float* __restrict__ vy = P.v[1];
    const float* __restrict__ vz = P.v[2];
    long long o = L.off(i, j, k0);
    // z window of vz: q[t] = vz(k - R + t), t = 0 .. 2R-1
    float q[2 * R];
#pragma unroll
    for (int t = 0; t < 2 * R - 1; ++t) q[t] = __ldg(vz + o + (t - R) * pl);
    const bool xy_in = i >= P.nd[0] && i < L.n[0] - P.nd[0] && j >= P.nd[1] &&
                       j < L.n[1] - P.nd[1];
    const float ax_a = __ldg(P.ta[0] + i), ax_b = __ldg(P.tb[0] + i), ax_k = __ldg(P.tik[0] + i);
    const float ay_a = __ldg(P.ta[1] + j), ay_b = __ldg(P.tb[1] + j), ay_k = __ldg(P.tik[1] + j);
    for (int k = k0; k < k1; ++k, o += pl) {
        q[2 * R - 1] = __ldg(vz + o + (R - 1) * pl);
        float d[3] = {0.0f, 0.0f, 0.0f};
        // staggered_derivative_at Backward: t += c_m (f[(m-1) s] - f[-m s])
#pragma unroll
        for (int m = 1; m <= R; ++m)
            d[0] = fa(d[0], fm(P.w[0][m - 1], fs(__ldg(vx + o + m - 1), __ldg(vx + o - m))));
#pragma unroll
        for (int m = 1; m <= R; ++m)
            d[1] = fa(d[1], fm(P.w[1][m - 1],
                               fs(__ldg(vy + o + (m - 1) * sy), __ldg(vy + o - m * sy))));
#pragma unroll
        for (int m = 1; m <= R; ++m) d[2] = fa(d[2], fm(P.w[2][m - 1], fs(q[R + m - 1], q[R - m])));
        if (!(xy_in && k >= P.nd[2] && k < L.n[2] - P.nd[2])) {
            d[0] = cpml_term(d[0], P.run[0][0], P.run[0][1], 0, i, i, j, k, ax_a, ax_b, ax_k);
            d[1] = cpml_term(d[1], P.run[1][0], P.run[1][1], 1, j, i, j, k, ay_a, ay_b, ay_k);
            d[2] = cpml_term(d[2], P.run[2][0], P.run[2][1], 2, k, i, j, k, __ldg(P.ta[2] + k),
                             __ldg(P.tb[2] + k), __ldg(P.tik[2] + k));
        }
        P.p[o] = fa(P.p[o], fm(__ldg(P.dtb + o), fa(fa(d[0], d[1]), d[2])));
#pragma unroll
        for (int t = 0; t < 2 * R - 1; ++t) q[t] = q[t + 1];
    }
}

template <int R>
void launch_pass(bool velocity, const VdParams& P, cudaStream_t s) {
    const Layout& L = P.lay;
    dim3 blk(BX, BY);
    dim3 grd((L.n[0] + BX - 1) / BX, (L.n[1] + BY - 1) / BY, (L.n[2] + P.zc - 1) / P.zc);
    if (velocity)
        k_vd_velocity<R><<<grd, blk, 0, s>>>(P);
    else
        k_vd_pressure<R><<<grd, blk, 0, s>>>(P);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch(bool velocity, const VdParams& P, cudaStream_t s) {
    switch (P.lay.r) {
#define MM_VD_CASE(RR)                       \
    case RR:                                 \
        launch_pass<RR>(velocity, P, s);     \
        break;
        MM_VD_CASE(1)
        MM_VD_CASE(2)
        MM_VD_CASE(3)
        MM_VD_CASE(4)
        MM_VD_CASE(5)
        MM_VD_CASE(6)
        MM_VD_CASE(7)
        MM_VD_CASE(8)
#undef MM_VD_CASE
        default:
            raise(ST_CONFIG, "stencil radius must be in [1, 8]");
    }
}

// TMA plan: tensor maps, work items and queues of k_vdv / k_vdp.
template <int R>
struct FastVd {
    using C = vdk::VdCfg<R>;
    vdk::VdvMaps mv;
    vdk::VdpMaps mp;
    DevBuf<int4> items;
    DevBuf<int> ctr;  // [0..1] velocity queue, [2..3] pressure queue
    int nitems = 0, grid_v = 0, grid_p = 0;

    FastVd(const Layout& L, float* p, float* const v[3], const float* ir, const float* dtb,
           int device, cudaStream_t s) {
        mv.p = tma_field_map(L, p, C::BX, C::BY);
        mv.ir = tma_field_map(L, ir, C::TX, C::TY);
        mv.vx = tma_field_map(L, v[0], C::TX, C::TY);
        mv.vy = tma_field_map(L, v[1], C::TX, C::TY);
        mv.vz = tma_field_map(L, v[2], C::TX, C::TY);
        mp.vx = tma_field_map(L, v[0], C::BX, C::TY);
        mp.vy = tma_field_map(L, v[1], C::TX, C::BY);
        mp.vz = mv.vz;
        mp.dtb = tma_field_map(L, dtb, C::TX, C::TY);
        mp.p = tma_field_map(L, p, C::TX, C::TY);
        MM_CUDA(cudaFuncSetAttribute(vdk::k_vdv<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)C::SMEM_V));
        MM_CUDA(cudaFuncSetAttribute(vdk::k_vdp<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)C::SMEM_P));
        int sms = 0, ov = 0, op = 0;
        MM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ov, vdk::k_vdv<R>, C::NT, C::SMEM_V));
        MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&op, vdk::k_vdp<R>, C::NT, C::SMEM_P));
        if (ov < 1 || op < 1) raise(ST_CUDA, "acoustic_iso kernels do not fit on an SM");
        // (tile, z-chunk) items, chunk-major, short enough that the tiles in
        // flight stay at nearby depths (their halo planes meet in L2): about
        // 20 planes per item and at least ~6 items per resident CTA.
        // Measured: 1000^3 59 -> 93 Gpts/s going from 500- to 20-plane items,
        // 512^3 76 -> 89 (73 -> 16 planes); 240^3 best at 8-12 planes.
        const int tx = (L.n[0] + C::TX - 1) / C::TX, ty = (L.n[1] + C::TY - 1) / C::TY;
        const int slots = sms * std::max(ov, op);
        int nch = std::max((L.n[2] + 19) / 20, (6 * slots + tx * ty - 1) / (tx * ty));
        nch = std::max(1, std::min(nch, std::max(1, L.n[2] / 8)));
        if (tuning("vd_zchunks") > 0) nch = (int)tuning("vd_zchunks");
        std::vector<int4> it;
        for (int c = 0; c < nch; ++c) {
            const int zb = (int)((long long)L.n[2] * c / nch), ze = (int)((long long)L.n[2] * (c + 1) / nch);
            if (ze <= zb) continue;
            for (int y = 0; y < ty; ++y)
                for (int x = 0; x < tx; ++x) it.push_back(make_int4(x, y, zb, ze));
        }
        nitems = (int)it.size();
        items.upload(it.data(), it.size(), s);
        ctr.alloc_zero(4, s);
        grid_v = std::min(nitems, sms * ov);
        grid_p = std::min(nitems, sms * op);
        // tuning "vd_ctas" (diagnostics): cap the CTA count (long item sequences per CTA)
        if (const long long cap = tuning("vd_ctas"); cap > 0) {
            grid_v = std::min(grid_v, (int)cap);
            grid_p = std::min(grid_p, (int)cap);
        }
    }

    void launch(bool velocity, vdk::VdFastParams P, cudaStream_t s) {
        P.items = items.ptr;
        P.wq.nitems = nitems;
        if (velocity) {
            P.wq.ctr = ctr.ptr;
            vdk::k_vdv<R><<<grid_v, C::NT, C::SMEM_V, s>>>(mv, P);
        } else {
            P.wq.ctr = ctr.ptr + 2;
            vdk::k_vdp<R><<<grid_p, C::NT, C::SMEM_P, s>>>(mp, P);
        }
        note_launches(1);
        MM_CUDA(cudaGetLastError());
    }
};

struct FastVdAny {
    virtual ~FastVdAny() = default;
    virtual void launch(bool velocity, const vdk::VdFastParams& P, cudaStream_t s) = 0;
};
template <int R>
struct FastVdR : FastVdAny {
    FastVd<R> f;
    FastVdR(const Layout& L, float* p, float* const v[3], const float* ir, const float* dtb,
            int dev, cudaStream_t s)
        : f(L, p, v, ir, dtb, dev, s) {}
    void launch(bool velocity, const vdk::VdFastParams& P, cudaStream_t s) override {
        f.launch(velocity, P, s);
    }
};

std::unique_ptr<FastVdAny> make_fast_vd(const Layout& L, float* p, float* const v[3],
                                        const float* ir, const float* dtb, int dev,
                                        cudaStream_t s) {
    switch (L.r) {
#define MM_VD_FAST(RR) \
    case RR:           \
        return std::make_unique<FastVdR<RR>>(L, p, v, ir, dtb, dev, s);
        MM_VD_FAST(1)
        MM_VD_FAST(2)
        MM_VD_FAST(3)
        MM_VD_FAST(4)
        MM_VD_FAST(5)
        MM_VD_FAST(6)
        MM_VD_FAST(7)
        MM_VD_FAST(8)
#undef MM_VD_FAST
        default:
            return nullptr;
    }
}

}  // namespace vd
}  // namespace mmb

using namespace mmb;

struct mm_vd_engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    Layout lay;
    HostGrid hg;
    int nd[3];
    bool free_surface = false;
    float dt = 0;
    Profile prof;
    float w[3][kMaxR] = {};
    DevBuf<float> p, v[3], ir, dtb;
    DevBuf<float> ta[3], tb[3], tik[3];
    CpmlRun vrun[3][2] = {}, prun[3][2] = {};
    DevBuf<float> vpsi[3][2], ppsi[3][2];
    std::vector<int> rec_ijk;
    DevBuf<long long> rec_offs;
    DevBuf<float> traces;
    int nrec = 0, cap = 0;
    DevBuf<int> counters;  // [0] step counter, [1] first bad step, [2] epilogue ticket
    TraceCopier tcopy;
    DevBuf<float> amps;
    long long steps = 0;
    int zc = 32;
    std::unique_ptr<vd::FastVdAny> fast;  // null: the plain kernels (MM_VD_SIMPLE)

    vd::VdParams params(bool velocity) const {
        vd::VdParams s;
        std::memset(&s, 0, sizeof s);
        s.lay = lay;
        s.p = p.ptr;
        s.ir = ir.ptr;
        s.dtb = dtb.ptr;
        s.zc = zc;
        for (int a = 0; a < 3; ++a) {
            s.nd[a] = nd[a];
            s.v[a] = v[a].ptr;
            s.ta[a] = ta[a].ptr;
            s.tb[a] = tb[a].ptr;
            s.tik[a] = tik[a].ptr;
            for (int m = 0; m < kMaxR; ++m) s.w[a][m] = w[a][m];
            for (int side = 0; side < 2; ++side)
                s.run[a][side] = velocity ? vrun[a][side] : prun[a][side];
        }
        return s;
    }

    // psi arrays of both passes: one per axis and damping layer, allocated
    // only where some a != 0 (elsewhere psi stays +0; see the file comment)
    void setup_cpml() {
        for (int ax = 0; ax < 3; ++ax) {
            const int n = lay.n[ax];
            ta[ax].upload(prof.a[ax].data(), n, stream);
            tb[ax].upload(prof.b[ax].data(), n, stream);
            tik[ax].upload(prof.ik[ax].data(), n, stream);
            const int lo_[2] = {0, n - nd[ax]}, hi_[2] = {nd[ax], n};
            for (int side = 0; side < 2; ++side) {
                CpmlRun r{0, 0, 0, nullptr, nullptr, 0, 0};
                bool active = false;
                for (int l = lo_[side]; l < hi_[side]; ++l) active |= prof.a[ax][l] != 0.0f;
                vrun[ax][side] = prun[ax][side] = r;
                if (hi_[side] <= lo_[side] || !active) continue;
                const long long wdt = hi_[side] - lo_[side];
                const long long nx4 = (lay.n[0] + 3) / 4 * 4;
                r.lo = lo_[side];
                r.hi = hi_[side];
                // rows start 16-byte aligned so the fast kernels move psi as float4
                r.org = ax == 0 ? (r.lo & ~3) : r.lo;
                size_t count;
                if (ax == 0) {
                    r.s1 = (r.hi - r.org + 3) / 4 * 4;
                    r.s2 = r.s1 * lay.n[1];
                    count = (size_t)r.s2 * lay.n[2];
                } else if (ax == 1) {
                    r.s1 = nx4;
                    r.s2 = nx4 * wdt;
                    count = (size_t)r.s2 * lay.n[2];
                } else {
                    r.s1 = nx4;
                    r.s2 = nx4 * lay.n[1];
                    count = (size_t)r.s2 * wdt;
                }
                vpsi[ax][side].alloc_zero(count, stream);
                ppsi[ax][side].alloc_zero(count, stream);
                vrun[ax][side] = prun[ax][side] = r;
                vrun[ax][side].psi = vpsi[ax][side].ptr;
                prun[ax][side].psi = ppsi[ax][side].ptr;
            }
        }
    }

    long long src_off(const int* src) const {
        for (int a = 0; a < 3; ++a)
            if (src[a] < 0 || src[a] >= lay.n[a])
                raise(ST_CONFIG, "source location outside grid interior");
        return lay.off(src[0], src[1], src[2]);
    }

    vdk::VdFastParams fast_params(bool velocity) const {
        vdk::VdFastParams f;
        std::memset(&f, 0, sizeof f);
        const vd::VdParams s = params(velocity);
        f.lay = s.lay;
        f.p = s.p;
        f.ir = s.ir;
        f.dtb = s.dtb;
        for (int a = 0; a < 3; ++a) {
            f.nd[a] = s.nd[a];
            f.v[a] = s.v[a];
            f.tab.ta[a] = s.ta[a];
            f.tab.tb[a] = s.tb[a];
            f.tab.tik[a] = s.tik[a];
            for (int m = 0; m < kMaxR; ++m) f.w[a][m] = s.w[a][m];
            f.run[a][0] = s.run[a][0];
            f.run[a][1] = s.run[a][1];
        }
        return f;
    }
    void velocity() {
        if (fast)
            fast->launch(true, fast_params(true), stream);
        else
            vd::launch(true, params(true), stream);
    }
    void pressure() {
        if (fast)
            fast->launch(false, fast_params(false), stream);
        else
            vd::launch(false, params(false), stream);
    }
    void inject(float amp, const int* src, const float* amp_dev, const int* step_dev) {
        launch_inject(p.ptr, dtb.ptr, src_off(src), amp, amp_dev, step_dev, stream);
    }
    // velocity, pressure, then k_epilogue: injection, free surface and -- from
    // mm_vd_run -- the receiver sample and the step counter in one launch
    void full_step(float amp, const int* src, const float* amp_dev, int* step_dev,
                   const RecParams* rec = nullptr) {
        const long long so = src ? src_off(src) : -1LL;
        velocity();
        pressure();
        Epilogue ep;
        std::memset(&ep, 0, sizeof ep);
        ep.p = p.ptr;
        ep.cv = dtb.ptr;
        ep.src_off = so;
        ep.amp = amp;
        ep.amp_dev = amp_dev;
        ep.step_dev = step_dev;
        ep.count = step_dev != nullptr;
        ep.fs = free_surface;
        ep.lay = lay;
        if (rec) ep.rec = *rec;
        ep.done = counters.ptr + 2;
        launch_epilogue(ep, stream);
        ++steps;
    }

    void to_host(const float* dev, float* host) {
        DevBuf<float> stage;
        stage.alloc(hg.volume());
        launch_to_host_layout(dev, stage.ptr, lay, stream);
        MM_CUDA(cudaMemcpyAsync(host, stage.ptr, hg.volume() * sizeof(float),
                                cudaMemcpyDeviceToHost, stream));
        MM_CUDA(cudaStreamSynchronize(stream));
    }
    void from_host(const float* host, float* dev) {
        DevBuf<float> stage;
        stage.upload(host, hg.volume(), stream);
        launch_to_device_layout(stage.ptr, dev, lay, stream);
        MM_CUDA(cudaStreamSynchronize(stream));
    }

    ~mm_vd_engine() {
        if (stream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
            cudaStreamDestroy(stream);
        }
    }
};

namespace {

void use(mm_vd_engine* e) {
    need(e, "engine");
    MM_CUDA(cudaSetDevice(e->device));
}

void check_rho(const float* rho, const HostGrid& g) {
    for (int i = 0; i < g.n[0]; ++i)
        for (int j = 0; j < g.n[1]; ++j)
            for (int k = 0; k < g.n[2]; ++k) {
                const float v = rho[g.off(i, j, k)];
                if (!std::isfinite(v) || v <= 0.0f)
                    raise(ST_VALIDATION, "rho must be finite and > 0 everywhere");
            }
}

}  // namespace

extern "C" {

int mm_staggered_first_derivative_coeffs(int radius, double h, double* c) {
    MM_API_BEGIN
    need(c, "c");
    const Coeffs s = staggered_first_derivative(radius, h);
    for (int m = 0; m < radius; ++m) c[m] = s.c[m];
    MM_API_END
}

int mm_integrate_wavelet(const float* w, int n, double dt, float* out) {
    MM_API_BEGIN
    if (n < 0) raise(ST_INVAL, "negative sample count");
    if (n == 0) return MM_OK;
    need(w, "w");
    need(out, "out");
    const std::vector<float> r = integrate_wavelet(std::vector<float>(w, w + n), dt);
    std::memcpy(out, r.data(), sizeof(float) * n);
    MM_API_END
}

int mm_vd_create(const mm_grid* grid, const float* vp, const float* rho,
                 const mm_engine_options* opts, float dt, double vmax, int device,
                 mm_vd_engine** out) {
    MM_API_BEGIN
    need(grid, "grid");
    need(vp, "vp");
    need(opts, "options");
    need(out, "out");
    *out = nullptr;
    // propagator_impl.hpp:186-187
    if (!rho) raise(ST_VALIDATION, "acoustic_iso requires a density volume (rho)");
    static const char* axn[3] = {"x", "y", "z"};
    for (int a = 0; a < 3; ++a) {
        if (grid->n[a] < 1)
            raise(ST_CONFIG, std::string("grid size must be >= 1 along ") + axn[a] + ", got " +
                               std::to_string(grid->n[a]));
        if (!(grid->d[a] > 0.0))
            raise(ST_CONFIG, std::string("grid spacing must be > 0 along ") + axn[a]);
    }
    if (grid->radius < 1 || grid->radius > kMaxR)
        raise(ST_CONFIG, "stencil radius must be in [1, 8], got " + std::to_string(grid->radius));
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        raise(ST_CUDA, "no CUDA device available: the acoustic_iso engine runs on the GPU only");
    }
    if (device < 0 || device >= ndev) raise(ST_INVAL, "device ordinal out of range");
    MM_CUDA(cudaSetDevice(device));

    auto e = std::make_unique<mm_vd_engine>();
    e->device = device;
    MM_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    const int r = grid->radius;
    e->lay = Layout::make(grid->n, r);
    e->hg = HostGrid{{grid->n[0], grid->n[1], grid->n[2]}, r};
    e->free_surface = opts->free_surface != 0;
    e->dt = dt;
    for (int a = 0; a < 3; ++a) {
        e->nd[a] = opts->ndamping[a];
        if (opts->ndamping[a] < 0) raise(ST_CONFIG, "ndamping must be >= 0");
        if (2 * opts->ndamping[a] >= grid->n[a])
            raise(ST_CONFIG, std::string("damping layers too thick along ") + axn[a] + ": 2*" +
                               std::to_string(opts->ndamping[a]) +
                               " >= " + std::to_string(grid->n[a]));
    }
    // staggered weights (propagator_impl.hpp:197-198)
    for (int ax = 0; ax < 3; ++ax) {
        const Coeffs c = staggered_first_derivative(r, grid->d[ax]);
        for (int m = 0; m < r; ++m) e->w[ax][m] = static_cast<float>(c.c[m]);
    }
    // profile (propagator_impl.hpp:199-200) with the engine's float dt
    e->prof = build_profile(grid->n, grid->d, opts->ndamping, opts->fmax, vmax,
                            static_cast<double>(dt), opts->r_target, e->free_surface);
    // vp copy, tapered (:201); rho as given
    const HostGrid& g = e->hg;
    std::vector<float> vpc(vp, vp + g.volume());
    const int zero[3] = {0, 0, 0};
    if (opts->taper) taper_material(vpc.data(), g, opts->ntaper, zero, grid->n);
    // per-point coefficients, computed as the reference does each step:
    // inv_rho = dt / rho (:224), dt * bulk with bulk = (rho * vp) * vp (:269-270)
    std::vector<float> irh(g.volume(), 0.0f), dtbh(g.volume(), 0.0f);
    for (int i = 0; i < g.n[0]; ++i)
        for (int j = 0; j < g.n[1]; ++j)
            for (int k = 0; k < g.n[2]; ++k) {
                const size_t o = g.off(i, j, k);
                irh[o] = dt / rho[o];
                const float bulk = rho[o] * vpc[o] * vpc[o];
                dtbh[o] = dt * bulk;
            }
    const Layout& L = e->lay;
    e->p.alloc_zero(L.total, e->stream);
    for (int a = 0; a < 3; ++a) e->v[a].alloc_zero(L.total, e->stream);
    e->ir.alloc_zero(L.total, e->stream);
    e->dtb.alloc_zero(L.total, e->stream);
    e->from_host(irh.data(), e->ir.ptr);
    e->from_host(dtbh.data(), e->dtb.ptr);
    e->setup_cpml();
    e->counters.alloc_zero(3, e->stream);  // + the epilogue's block ticket
    if (tuning("vd_zc") > 0) e->zc = (int)tuning("vd_zc");
    if (!tuning("vd_simple")) {
        float* const vv[3] = {e->v[0].ptr, e->v[1].ptr, e->v[2].ptr};
        e->fast = vd::make_fast_vd(e->lay, e->p.ptr, vv, e->ir.ptr, e->dtb.ptr, device, e->stream);
    }
    MM_CUDA(cudaStreamSynchronize(e->stream));
    *out = e.release();
    MM_API_END
}

int mm_vd_destroy(mm_vd_engine* e) {
    MM_API_BEGIN
    if (!e) return MM_OK;
    cudaSetDevice(e->device);
    delete e;
    MM_API_END
}

int mm_vd_step(mm_vd_engine* e, float amp, const int* src) {
    MM_API_BEGIN
    use(e);
    e->full_step(amp, src, nullptr, nullptr);
    MM_API_END
}

int mm_vd_update_velocity(mm_vd_engine* e) {
    MM_API_BEGIN
    use(e);
    e->velocity();
    MM_API_END
}

int mm_vd_update_pressure(mm_vd_engine* e) {
    MM_API_BEGIN
    use(e);
    e->pressure();
    MM_API_END
}

int mm_vd_inject_source(mm_vd_engine* e, float amp, const int* src) {
    MM_API_BEGIN
    use(e);
    need(src, "src");
    e->inject(amp, src, nullptr, nullptr);
    MM_API_END
}

int mm_vd_apply_free_surface(mm_vd_engine* e) {
    MM_API_BEGIN
    use(e);
    if (e->free_surface) launch_free_surface(e->p.ptr, e->lay, e->stream);
    MM_API_END
}

int mm_vd_synchronize(mm_vd_engine* e) {
    MM_API_BEGIN
    use(e);
    MM_CUDA(cudaStreamSynchronize(e->stream));
    e->tcopy.sync();
    MM_API_END
}

int mm_vd_field_size(mm_vd_engine* e, size_t* count) {
    MM_API_BEGIN
    need(e, "engine");
    need(count, "count");
    *count = e->hg.volume();
    MM_API_END
}

int mm_vd_get_dt(mm_vd_engine* e, float* dt) {
    MM_API_BEGIN
    need(e, "engine");
    need(dt, "dt");
    *dt = e->dt;
    MM_API_END
}

int mm_vd_steps_taken(mm_vd_engine* e, long long* steps) {
    MM_API_BEGIN
    need(e, "engine");
    need(steps, "steps");
    *steps = e->steps;
    MM_API_END
}

int mm_vd_get_pressure(mm_vd_engine* e, float* host) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    e->to_host(e->p.ptr, host);
    MM_API_END
}

int mm_vd_get_velocity(mm_vd_engine* e, int axis, float* host) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    if (axis < 0 || axis > 2) raise(ST_INVAL, "axis must be 0, 1 or 2");
    e->to_host(e->v[axis].ptr, host);
    MM_API_END
}

int mm_vd_set_pressure(mm_vd_engine* e, const float* host) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    e->from_host(host, e->p.ptr);
    MM_API_END
}

int mm_vd_set_velocity(mm_vd_engine* e, int axis, const float* host) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    if (axis < 0 || axis > 2) raise(ST_INVAL, "axis must be 0, 1 or 2");
    e->from_host(host, e->v[axis].ptr);
    MM_API_END
}

int mm_vd_set_receivers(mm_vd_engine* e, const int* ijk, int nreceivers, int capacity) {
    MM_API_BEGIN
    use(e);
    if (nreceivers < 0 || capacity < 0) raise(ST_INVAL, "negative receiver count or capacity");
    if (nreceivers > 0) need(ijk, "ijk");
    std::vector<long long> offs(nreceivers);
    for (int r = 0; r < nreceivers; ++r) {
        const int* c = ijk + 3 * r;
        for (int a = 0; a < 3; ++a)
            if (c[a] < 0 || c[a] >= e->lay.n[a]) raise(ST_CONFIG, "receiver outside grid interior");
        offs[r] = e->lay.off(c[0], c[1], c[2]);
    }
    e->rec_ijk.assign(ijk, ijk + 3 * (size_t)nreceivers);
    e->nrec = nreceivers;
    e->cap = capacity;
    e->rec_offs.upload(offs.data(), offs.size(), e->stream);
    e->traces.alloc_zero((size_t)nreceivers * capacity, e->stream);
    MM_CUDA(cudaStreamSynchronize(e->stream));
    MM_API_END
}

int mm_vd_record(mm_vd_engine* e, int step) {
    MM_API_BEGIN
    use(e);
    if (step < 0 || step >= e->cap) raise(ST_INVAL, "record step outside the trace capacity");
    RecParams rp{e->p.ptr, e->rec_offs.ptr, e->traces.ptr, e->nrec, step, nullptr};
    launch_record(rp, nullptr, e->stream);
    MM_API_END
}

int mm_vd_get_traces(mm_vd_engine* e, float* host, int nsteps) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    if (nsteps < 0 || nsteps > e->cap) raise(ST_INVAL, "nsteps exceeds the trace capacity");
    std::vector<float> dev((size_t)e->nrec * nsteps);
    if (!dev.empty())
        MM_CUDA(cudaMemcpyAsync(dev.data(), e->traces.ptr, dev.size() * sizeof(float),
                                cudaMemcpyDeviceToHost, e->stream));
    MM_CUDA(cudaStreamSynchronize(e->stream));
    for (int s = 0; s < nsteps; ++s)
        for (int r = 0; r < e->nrec; ++r)
            host[(size_t)r * nsteps + s] = dev[(size_t)s * e->nrec + r];
    MM_API_END
}

int mm_vd_copy_trace_step(mm_vd_engine* e, int step, float* host, int async) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    if (step < 0 || step >= e->cap) raise(ST_INVAL, "step outside the trace capacity");
    if (e->nrec == 0) return MM_OK;
    if (async) {
        // off the compute stream: the copy overlaps the next step
        e->tcopy.copy(host, e->traces.ptr + (size_t)step * e->nrec, sizeof(float) * e->nrec,
                      e->stream);
        return MM_OK;
    }
    MM_CUDA(cudaMemcpyAsync(host, e->traces.ptr + (size_t)step * e->nrec,
                            sizeof(float) * e->nrec, cudaMemcpyDeviceToHost, e->stream));
    MM_CUDA(cudaStreamSynchronize(e->stream));
    MM_API_END
}

int mm_vd_run(mm_vd_engine* e, const float* amps, int nsteps, const int* src, int record,
              int first_sample, float* device_ms) {
    MM_API_BEGIN
    use(e);
    if (nsteps < 0) raise(ST_INVAL, "nsteps must be >= 0");
    if (nsteps == 0) return MM_OK;
    need(amps, "amps");
    if (record && (first_sample < 0 || first_sample + nsteps > e->cap))
        raise(ST_INVAL, "recorded steps exceed the trace capacity");
    if (src) (void)e->src_off(src);
    e->amps.upload(amps, nsteps, e->stream);
    const int init[2] = {0, INT_MAX};
    MM_CUDA(cudaMemcpyAsync(e->counters.ptr, init, sizeof init, cudaMemcpyHostToDevice,
                            e->stream));
    int* step_dev = e->counters.ptr;
    int* bad = e->counters.ptr + 1;
    cudaEvent_t t0, t1;
    MM_CUDA(cudaEventCreate(&t0));
    MM_CUDA(cudaEventCreate(&t1));
    MM_CUDA(cudaEventRecord(t0, e->stream));
    auto one_step = [&] {
        const RecParams rp{nullptr, e->rec_offs.ptr,
                           e->traces.ptr + (size_t)first_sample * e->nrec, e->nrec, 0, bad};
        e->full_step(0.0f, src, e->amps.ptr, step_dev, record && e->nrec > 0 ? &rp : nullptr);
    };
    // The fields update in place, so one step is captured as a CUDA graph and
    // replayed; per-step values come through the device step counter.
    int s = 0;
    const bool use_graph = nsteps >= 4 && tuning("step_graph") != 0;
    if (use_graph) {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        const long long l0 = launches_so_far();
        MM_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        one_step();
        MM_CUDA(cudaStreamEndCapture(e->stream, &g));
        const long long per_graph = launches_so_far() - l0;
        MM_CUDA(cudaGraphInstantiate(&ge, g, 0));
        for (int k = 0; k < nsteps; ++k) MM_CUDA(cudaGraphLaunch(ge, e->stream));
        e->steps += nsteps - 1;  // capture advanced the host counter once
        s = nsteps;
        MM_CUDA(cudaGraphExecDestroy(ge));
        MM_CUDA(cudaGraphDestroy(g));
        note_launches(per_graph * (nsteps - 1));
    }
    for (; s < nsteps; ++s) one_step();
    MM_CUDA(cudaEventRecord(t1, e->stream));
    MM_CUDA(cudaEventSynchronize(t1));
    float ms = 0;
    MM_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (device_ms) *device_ms = ms;
    int bad_h = INT_MAX;
    MM_CUDA(cudaMemcpy(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (bad_h != INT_MAX)
        throw Error(ST_INSTABILITY,
                    "non-finite wavefield sample detected at time step " +
                        std::to_string(first_sample + bad_h),
                    first_sample + bad_h);
    MM_API_END
}

int mm_vd_stream(mm_vd_engine* e, void** stream) {
    MM_API_BEGIN
    need(e, "engine");
    need(stream, "stream");
    *stream = (void*)e->stream;
    MM_API_END
}

int mm_run_vd(const mm_sim_config* c, const float* vp_model, const float* rho_model, int device,
              float* traces, mm_run_report* rep) {
    MM_API_BEGIN
    need(c, "cfg");
    need(vp_model, "vp_model");
    const auto wall0 = std::chrono::steady_clock::now();
    if (c->nsteps < 1) raise(ST_CONFIG, "nsteps must be >= 1");
    for (int a = 0; a < 3; ++a) {
        if (c->ngrid[a] < 1) raise(ST_CONFIG, "grid size must be >= 1");
        if (!(c->dgrid[a] > 0.0)) raise(ST_CONFIG, "grid spacing must be > 0");
    }
    if (c->stencil_radius < 1) raise(ST_CONFIG, "stencil radius must be >= 1");
    if (!rho_model) raise(ST_VALIDATION, "acoustic_iso requires a density volume (rho)");
    const HostGrid g{{c->ngrid[0], c->ngrid[1], c->ngrid[2]}, c->stencil_radius};
    // the EarthModel (model.cpp:15-43): validated, ghosts replicated
    std::vector<float> vp(vp_model, vp_model + g.volume());
    std::vector<float> rho(rho_model, rho_model + g.volume());
    float vmin = 0, vmax = 0;
    validate_vp(vp.data(), g, &vmin, &vmax);
    check_rho(rho.data(), g);
    fill_ghosts_replicate(vp.data(), g);
    fill_ghosts_replicate(rho.data(), g);
    // driver.cpp:88-96, :122-128
    const double dt = cfl_dt(vmax, c->ngrid, c->dgrid, c->stencil_radius, c->cfl);
    const std::vector<float> wi = integrate_wavelet(ricker(c->fmax, dt, c->nsteps), dt);
    int src[3] = {c->ngrid[0] / 2, c->ngrid[1] / 2, c->ngrid[2] / 2};
    if (c->has_source_loc)
        for (int a = 0; a < 3; ++a) src[a] = c->source_loc[a];
    for (int a = 0; a < 3; ++a)
        if (src[a] < 0 || src[a] >= c->ngrid[a])
            raise(ST_CONFIG, "source location outside grid interior");
    const int inc0 = c->receiver_increment[0], inc1 = c->receiver_increment[1];
    if (inc0 < 1 || inc1 < 1) raise(ST_CONFIG, "receiver increment must be >= 1");
    std::vector<int> rec;
    for (int i = 0; i < c->ngrid[0]; i += inc0)
        for (int j = 0; j < c->ngrid[1]; j += inc1) {
            rec.push_back(i);
            rec.push_back(j);
            rec.push_back(c->ndamping[2]);
        }
    const int nrec = (int)rec.size() / 3;
    mm_grid grid;
    for (int a = 0; a < 3; ++a) {
        grid.n[a] = c->ngrid[a];
        grid.d[a] = c->dgrid[a];
    }
    grid.radius = c->stencil_radius;
    mm_engine_options o;
    for (int a = 0; a < 3; ++a) {
        o.ndamping[a] = c->ndamping[a];
        o.ntaper[a] = c->ntaper[a];
    }
    o.fmax = c->fmax;
    o.r_target = c->r_target;
    o.free_surface = c->free_surface;
    o.taper = c->taper;
    mm_vd_engine* e = nullptr;
    int rc = mm_vd_create(&grid, vp.data(), rho.data(), &o, static_cast<float>(dt), vmax, device,
                          &e);
    if (rc) return rc;
    std::unique_ptr<mm_vd_engine, int (*)(mm_vd_engine*)> guard(e, mm_vd_destroy);
    rc = mm_vd_set_receivers(e, rec.data(), nrec, c->nsteps);
    if (rc) return rc;
    float ms = 0;
    rc = mm_vd_run(e, wi.data(), c->nsteps, src, 1, 0, &ms);
    if (rc) return rc;
    if (traces) {
        rc = mm_vd_get_traces(e, traces, c->nsteps);
        if (rc) return rc;
    }
    if (rep) {
        rep->dt = dt;
        rep->kernel_seconds = ms * 1e-3;
        rep->steps_run = c->nsteps;
        rep->nreceivers = nrec;
        rep->modeling_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    }
    MM_API_END
}

}  // extern "C"
