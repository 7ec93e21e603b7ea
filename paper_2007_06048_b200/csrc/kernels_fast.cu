// kernels_fast.cu -- MM_MODE_FAST step: plan (tensor maps, work lists) + launches.
//
// One step = k_cpml (both CPML passes over the six damping slabs, one launch,
// fast_cpml.cuh) on the step's stream || k_inner (the inner box, update_plain,
// fast_inner.cuh) on a side stream -> the epilogue (engine.cu).  Each kernel
// is persistent over the whole GPU and pulls (tile, z-chunk) work items.
// Layouts k_cpml cannot serve (radius > 4, damping layers wider than its
// 32-point tiles, grids whose layers lie within a tile of each other) run the
// two-pass path: k_p1 (pass 1: psi, and dpsi_z of the z runs, fast_pass1.cuh)
// -> k_bnd (pass 2 over the X and Y slabs, fast_boundary.cuh) with k_inner
// (and the Z slabs); and where those cannot either (z runs closer than 2R),
// the strict kernels.  The sub-phase API (pass1 / update / update_ranges)
// always runs the two-pass kernels, which keep the reference's pass
// boundaries (psi is updated by pass 1, not by the boundary update).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "fast_boundary.cuh"
#include "fast_cpml.cuh"
#include "fast_inner.cuh"
#include "fast_pass1.cuh"
#include "mm_fast.hpp"

namespace mmb {

namespace {

using namespace fast;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    if (!fn) raise(ST_CUDA, "cuTensorMapEncodeTiled is unavailable");
    return fn;
}

// 3D fp32 tensor map, x fastest; OOB elements read as zero.
CUtensorMap make_map(const void* base, long long dx, long long dy, long long dz,
                     long long row_floats, long long plane_floats, int bx, int by) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    if (!base) return m;  // absent run: never dereferenced
    const cuuint64_t dims[3] = {(cuuint64_t)dx, (cuuint64_t)dy, (cuuint64_t)dz};
    const cuuint64_t strides[2] = {(cuuint64_t)row_floats * 4, (cuuint64_t)plane_floats * 4};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    // L2 promotion: 128B by default (boxes start 16B- but not always
    // 256B-aligned; 256B promotion would fetch unused bytes).  Tuning
    // "l2_promo" 0..3 selects none/64B/128B/256B for experiments.
    const long long v = tuning("l2_promo");
    const CUtensorMapL2promotion promo = v == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                         : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                         : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                  : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base),
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(ST_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

CUtensorMap field_map(const Layout& L, const float* base, int bx, int by) {
    return make_map(base, L.P, L.ey, L.ez, L.P, L.plane, bx, by);
}

// Tensor map over one CPML run array (see CpmlRun in mm_internal.hpp).
CUtensorMap run_map(const Layout& L, const CpmlRun& r, int ax, const float* base, int bx, int by) {
    if (r.hi <= r.lo || !base) return make_map(nullptr, 0, 0, 0, 0, 0, 0, 0);
    const long long w = r.hi - r.lo;
    if (ax == 0) return make_map(base, r.s1, L.n[1], L.n[2], r.s1, r.s2, bx, by);
    if (ax == 1) return make_map(base, r.s1, w, L.n[2], r.s1, r.s2, bx, by);
    return make_map(base, r.s1, L.n[1], w, r.s1, r.s2, bx, by);
}

}  // namespace

CUtensorMap tma_field_map(const Layout& L, const float* base, int bx, int by) {
    return field_map(L, base, bx, by);
}

namespace {

template <typename T>
struct DArr {
    T* ptr = nullptr;
    size_t n = 0;
    DArr() = default;
    DArr(const DArr&) = delete;
    DArr& operator=(const DArr&) = delete;
    DArr(DArr&& o) noexcept : ptr(o.ptr), n(o.n) { o.ptr = nullptr; }
    ~DArr() {
        if (ptr) cudaFree(ptr);
    }
    void set(const std::vector<T>& v, cudaStream_t s) {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        n = v.size();
        if (n == 0) return;
        MM_CUDA(cudaMalloc(&ptr, n * sizeof(T)));
        MM_CUDA(cudaMemcpyAsync(ptr, v.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
        MM_CUDA(cudaStreamSynchronize(s));
    }
    void alloc_zero(size_t count, cudaStream_t s) {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        n = count;
        if (n == 0) return;
        MM_CUDA(cudaMalloc(&ptr, n * sizeof(T)));
        MM_CUDA(cudaMemsetAsync(ptr, 0, n * sizeof(T), s));
        MM_CUDA(cudaStreamSynchronize(s));
    }
};

struct Box {
    int lo[3], hi[3];
};

// Dynamic shared memory limit of a kernel, and the L1 / shared-memory split
// the step kernels run with (tuning smem_carveout, experiment: -1 leaves the
// driver's choice).  Per-CTA globaltimer traces (MM_TRACE builds,
// mm_trace_dump) show the four persistent kernels of a step running one after
// another, not side by side: a grid's CTAs are dispatched in order within a
// priority, and each kernel's resident CTAs leave no room for the next one's;
// a common carveout only reorders them.
template <typename F>
void set_smem(F* fn, int bytes) {
    MM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const long long co = tuning("smem_carveout");
    if (co >= 0)
        MM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)co));
}

// Launch with programmatic dependent launch allowed (PDL): the kernel may start
// while the previous kernel in the stream drains; it orders its dependent
// reads itself (griddepcontrol.wait).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                bool pdl, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? at : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    MM_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Work items for the persistent kernels: each (tile, z-chunk) is one item.
// Items are ordered chunk-major (all tiles of chunk 0, then chunk 1, ...) and
// handed out dynamically (WorkQueue), so the items in flight at any moment are
// neighbouring tiles at the same z and their halo planes meet in L2.  The
// chunk length is chosen so that every CTA gets about per_cta / target
// items (at least one), `target` planes long.
struct Item {
    int tag, ty, zlo, zhi;
};
void wave_items(const std::vector<Item>& tiles, int ctas, double target,
                std::vector<int4>& out, bool even = false, int whole_le = 0) {
    out.clear();
    if (tiles.empty()) return;
    // tiles of at most whole_le planes: one item each, first in the queue
    // (long items first; no z-window warm-up per chunk for short tiles)
    if (whole_le > 0) {
        std::vector<Item> rest;
        for (const auto& t : tiles)
            if (t.zhi - t.zlo <= whole_le)
                out.push_back(make_int4(t.tag, t.ty, t.zlo, t.zhi));
            else
                rest.push_back(t);
        std::vector<int4> more;
        wave_items(rest, ctas, target, more, even, 0);
        out.insert(out.end(), more.begin(), more.end());
        return;
    }
    long long tp = 0;
    int zmax = 0;
    for (const auto& t : tiles) {
        tp += t.zhi - t.zlo;
        zmax = std::max(zmax, t.zhi - t.zlo);
    }
    const double per_cta = (double)tp / std::max(1, ctas);
    const int waves = std::max(1, (int)std::lround(per_cta / target));
    const int zc = std::max(4, (int)((tp + (long long)ctas * waves - 1) / ((long long)ctas * waves)));
    if (!even) {
        for (int k = 0; (long long)k * zc < zmax; ++k)
            for (const auto& t : tiles) {
                const int zb = t.zlo + k * zc;
                if (zb >= t.zhi) continue;
                out.push_back(make_int4(t.tag, t.ty, zb, std::min(t.zhi, zb + zc)));
            }
        return;
    }
    // the same number of chunks per tile, of equal length (no short last
    // chunk paying a whole z-window warm-up for a few planes)
    const int kmax = (zmax + zc - 1) / zc;
    for (int k = 0; k < kmax; ++k)
        for (const auto& t : tiles) {
            const int len = t.zhi - t.zlo, nc = (len + zc - 1) / zc;
            if (k >= nc) continue;
            out.push_back(make_int4(t.tag, t.ty, t.zlo + (int)((long long)len * k / nc),
                                    t.zlo + (int)((long long)len * (k + 1) / nc)));
        }
}

template <int R>
class FastPlanR final : public FastPlan {
    using IC = InnerCfg<R>;
    using BC = BndCfg<R>;
    using P1C = P1Cfg<R, true>;    // z runs (dpsi_z window)
    using P1X = P1Cfg<R, false>;   // x and y runs
    static constexpr bool kBnd = BC::SMEM <= 227 * 1024;  // TMA boundary kernel fits
    static constexpr bool kZs = ZSlabCfg<R>::SMEM <= 227 * 1024;  // optional Z-slab kernel
    using IW = InnerWCfg<R>;
    static constexpr bool kW = R > 4 && IW::SMEM <= 227 * 1024;  // wide-stencil inner kernel
    static constexpr bool kP1 = P1C::SMEM <= 200 * 1024;
    static constexpr int RC = R <= 4 ? R : 4;  // (k_cpml is instantiated for R <= 4 only)
    using CC = CpmlCfg<RC>;
    static constexpr bool kCpml = R <= 4 && CC::SMEM <= 227 * 1024;

public:
    FastPlanR(const Layout& lay, int device, float* const bufs[3], const float* cv, int order)
        : lay_(lay), device_(device), order_(order) {
        for (int b = 0; b < 3; ++b) {
            bufs_[b] = bufs[b];
            in_halo_[b] = field_map(lay, bufs[b], IC::BX, IC::BY);
            in_tile_[b] = field_map(lay, bufs[b], IC::TX, IC::TY);
            bd_halo_[b] = field_map(lay, bufs[b], BC::BX, BC::BY);
            bd_tile_[b] = field_map(lay, bufs[b], BC::TX, BC::TY);
            p1x_[b] = field_map(lay, bufs[b], P1X::BXX, P1X::TY);
            p1y_[b] = field_map(lay, bufs[b], P1X::TX, P1X::BYY);
            p1z_[b] = field_map(lay, bufs[b], P1C::TX, P1C::TY);
            if constexpr (kCpml) {
                cm_pc_[b] = field_map(lay, bufs[b], CC::BX, CC::BY);
                cm_tile_[b] = field_map(lay, bufs[b], CC::TX, CC::TY);
            }
        }
        cv_in_ = field_map(lay, cv, IC::TX, IC::TY);
        if constexpr (kW) {
            for (int b = 0; b < 3; ++b) {
                inw_halo_[b] = field_map(lay, bufs[b], IW::BX, IW::BY);
                inw_tile_[b] = field_map(lay, bufs[b], IW::TX, IW::TY);
            }
            cv_inw_ = field_map(lay, cv, IW::TX, IW::TY);
        }
        cv_bd_ = field_map(lay, cv, BC::TX, BC::TY);
        if constexpr (kCpml) cm_cv_ = field_map(lay, cv, CC::TX, CC::TY);
        // z-chunk targets (planes per work item) of the persistent kernels
        inner_zt_ = (double)std::max(1LL, tuning("inner_zt"));
        bnd_zt_ = (double)std::max(1LL, tuning("bnd_zt"));
        p1_zt_ = (double)std::max(1LL, tuning("p1_zt"));
        cpml_zt_ = (int)tuning("cpml_zt");
        cpml_on_ = kCpml && tuning("cpml_fused") != 0;
        // Z slabs: 0 = k_bnd tiles, 1 = k_zslab over the Z slabs after k_inner,
        // 2 = k_zslab over whole z columns of the inner box (instead of k_inner)
        const long long zm = tuning("zslabs");
        if (zm >= 0) zmode_ = (int)std::min(2LL, zm);
        if (!kZs) zmode_ = 0;
        if (zmode_ != 0) cpml_on_ = false;  // (k_cpml does the Z slabs itself)
        overlap_ = tuning("overlap") != 0;
        inner_late_ = (int)tuning("inner_late");
        dbg_ = tuning("debug_sync") == 1;
        bnd_kinds_ = (int)tuning("bnd_kinds");
        bnd_cap_ = tuning("bnd_ctas") > 0 ? (int)tuning("bnd_ctas") : 1 << 30;
        p1_axes_ = (int)tuning("p1_axes");
        // pass 1's x/y runs at the step stream's priority (tuning main_prio 2),
        // above the interior kernel's side stream (lowest): when both have CTAs
        // pending, the CPML chain's go first (without priorities the interior
        // kernel won that race in some engines: 145-159 us/step at 240^3)
        int prio_lo = 0, prio_hi = 0;
        MM_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        MM_CUDA(cudaStreamCreateWithPriority(&p1_side_, cudaStreamNonBlocking,
                                             tuning("main_prio") >= 2 ? prio_hi : prio_lo));
        {  // auto: on for grids whose steps replay as CUDA graphs (step_graph)
            const long long pd = tuning("pdl");
            pdl_ = pd < 0 ? (double)lay.n[0] * lay.n[1] * lay.n[2] < 6.0e6 : pd != 0;
        }
        MM_CUDA(cudaEventCreateWithFlags(&p1_fork_, cudaEventDisableTiming));
        MM_CUDA(cudaEventCreateWithFlags(&p1_join_, cudaEventDisableTiming));
        if (overlap_) {
            int lo = 0, hi = 0;
            MM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            MM_CUDA(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, lo));
            MM_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
            MM_CUDA(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming));
        }
        // R > 4: k_inner's z loop unrolled by 2R+1 overflows the instruction
        // cache; k_innerw (register queue rotated by moves) serves the inner box
        // (tuning wide_inner: 0 = the column kernel k_zslab over the inner box
        // and the Z slabs, 1 = k_inner, 2 = k_innerw)
        if constexpr (R > 4) {
            const long long wi = tuning("wide_inner");
            wide_ = kW && (wi < 0 || wi == 2);
            col_inner_ = kZs && !wide_ && wi != 1;
        }
        if (col_inner_ && zm < 0) zmode_ = 2;
        cudaDeviceProp prop;
        MM_CUDA(cudaGetDeviceProperties(&prop, device));
        sms_ = prop.multiProcessorCount;
        for (auto fn : {k_inner<R, 1>, k_inner<R, 2>})
            set_smem(fn, (int)IC::SMEM);
        if constexpr (kW)
            for (auto fn : {k_innerw<R, 1>, k_innerw<R, 2>})
                set_smem(fn, (int)IW::SMEM);
        if constexpr (kCpml) {
            for (auto fn : {k_cpml<RC, 1>, k_cpml<RC, 2>})
                set_smem(fn, (int)CC::SMEM);
            int per = 0;
            MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cpml<RC, 2>, CC::NT,
                                                                  CC::SMEM));
            cpml_per_sm_ = std::max(1, per);
        }
        if constexpr (kZs)
            for (auto fn : {k_zslab<R, 1>, k_zslab<R, 2>})
                set_smem(fn, (int)ZSlabCfg<R>::SMEM);
        int per_sm = 0;
        MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inner<R, 2>, IC::NT,
                                                              IC::SMEM));
        inner_per_sm_ = std::max(1, per_sm);
        inner_cap_ = tuning("inner_ctas") > 0 ? (int)tuning("inner_ctas") : 1 << 30;
        if constexpr (kBnd) {
            set_smem(k_bnd<R, 1>, (int)BC::SMEM);
            set_smem(k_bnd<R, 2>, (int)BC::SMEM);
            MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bnd<R, 2>, BC::NT,
                                                                  BC::SMEM));
            bnd_per_sm_ = std::max(1, per_sm);
        }
        if constexpr (kP1) {
            for (auto fn : {k_p1<R, 1, true>, k_p1<R, 2, true>})
                set_smem(fn, (int)P1C::SMEM);
            for (auto fn : {k_p1<R, 1, false>, k_p1<R, 2, false>})
                set_smem(fn, (int)P1X::SMEM);
            MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_p1<R, 2, true>,
                                                                  P1C::NT, P1C::SMEM));
            p1_per_sm_ = std::max(1, per_sm);
            MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_p1<R, 2, false>,
                                                                  P1X::NT, P1X::SMEM));
            p1x_per_sm_ = std::max(1, per_sm);
        }
    }
    ~FastPlanR() override {
        if (fork_) cudaEventDestroy(fork_);
        if (join_) cudaEventDestroy(join_);
        if (side_) cudaStreamDestroy(side_);
        if (p1_fork_) cudaEventDestroy(p1_fork_);
        if (p1_join_) cudaEventDestroy(p1_join_);
        if (p1_side_) cudaStreamDestroy(p1_side_);
    }

    void pass1(const StepParams& p, cudaStream_t s) override { launch_pass1(p, 0, lay_.n[2], s); }

    void update(const StepParams& p, int region, int z_lo, int z_hi, cudaStream_t s) override {
        const bool fc = fast_cpml(p);
        if (region == 0 || region == 1)
            launch_inner(p, z_lo, z_hi, region == 0 && fc && zmode_ != 0 ? kFull : kInnerOnly, s);
        if (region == 0 || region == 2) {
            if (fc) {
                launch_boundary(p, z_lo, z_hi, s);  // X and Y slabs
                if (region == 2 && zmode_ != 0) launch_inner(p, z_lo, z_hi, kZSlabs, s);
            } else {
                strict_update(p, 2, z_lo, z_hi, s);
            }
        }
    }

    // p_next on the union of several plane ranges (the z-slab schedule's edge
    // planes) with one launch per kernel
    void update_ranges(const StepParams& p, const int* ranges, int n, cudaStream_t s) override {
        ZRanges zr;
        for (int i = 0; i < n; ++i)
            if (ranges[2 * i + 1] > ranges[2 * i]) zr.emplace_back(ranges[2 * i], ranges[2 * i + 1]);
        if (zr.empty()) return;
        const bool fc = fast_cpml(p);
        if (!fc) {
            for (const auto& r : zr) update(p, 0, r.first, r.second, s);
            return;
        }
        launch_inner(p, zr, zmode_ != 0 ? kFull : kInnerOnly, s);
        launch_boundary(p, zr, s);
    }

    void fork_point(cudaStream_t s) override {
        if (overlap_) MM_CUDA(cudaEventRecord(fork_, s));
    }
    bool interior_side(const StepParams& p, int z_lo, int z_hi) override {
        if (!fast_cpml(p) || zmode_ != 0 || !overlap_) return false;
        // the interior needs p_cur only: from the step's start (fork_point),
        // at the side stream's low priority
        MM_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
        const int ti = timer.begin("inner", side_);
        launch_inner(p, z_lo, z_hi, kInnerOnly, side_);
        timer.end(ti, side_);
        MM_CUDA(cudaEventRecord(join_, side_));
        return true;
    }
    void finish_overlap(const StepParams& p, int z_lo, int z_hi, cudaStream_t s,
                        bool side) override {
        if (!side) {
            update(p, 0, z_lo, z_hi, s);
            return;
        }
        const int tb = timer.begin("boundary", s);
        launch_boundary(p, z_lo, z_hi, s);
        timer.end(tb, s);
        MM_CUDA(cudaStreamWaitEvent(s, join_, 0));
    }

    void step(const StepParams& p, long long src_off, float amp, const float* amp_dev,
              const int* step_dev, cudaStream_t s) override {
        if (use_cpml(p)) {
            // k_cpml (both CPML passes, all slabs) on the step's stream; the
            // interior kernel, which needs no CPML state, beside it on the side
            // stream (a second branch of a captured graph), joined before the
            // epilogue.  k_cpml is issued first: both kernels are persistent and
            // one k_cpml CTA fills an SM, so the interior CTAs take the SMs its
            // tail frees.
            if (overlap_) MM_CUDA(cudaEventRecord(fork_, s));
            const int tc = timer.begin("cpml", s);
            launch_cpml(p, ZRanges{{0, lay_.n[2]}}, s);
            timer.end(tc, s);
            if (overlap_) {
                MM_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
                const int ti = timer.begin("inner", side_);
                launch_inner(p, 0, lay_.n[2], kInnerOnly, side_);
                timer.end(ti, side_);
                MM_CUDA(cudaEventRecord(join_, side_));
            }
            dbg(s, "cpml", overlap_ ? side_ : nullptr);
            if (overlap_) {
                MM_CUDA(cudaStreamWaitEvent(s, join_, 0));
            } else {
                const int ti = timer.begin("inner", s);
                launch_inner(p, 0, lay_.n[2], kInnerOnly, s);
                timer.end(ti, s);
            }
            if (src_off >= 0) launch_inject(p.pn, p.cv, src_off, amp, amp_dev, step_dev, s);
            return;
        }
        const bool fc = fast_cpml(p);
        const int imode = fc && zmode_ != 0 ? kFull : kInnerOnly;
        // (the Z-slab planes read dpsi_z from pass 1: no overlap then)
        const bool ov = overlap_ && imode == kInnerOnly;
        auto fork_inner = [&] {
            // the interior kernel needs no CPML state: it runs on a second
            // stream beside pass 1 -> boundary and takes SMs as their tails free
            // them (a second branch of the captured graph)
            MM_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
            const int ti = timer.begin("inner", side_);
            launch_inner(p, 0, lay_.n[2], imode, side_);
            timer.end(ti, side_);
            MM_CUDA(cudaEventRecord(join_, side_));
        };
        if (ov) MM_CUDA(cudaEventRecord(fork_, s));  // the step's start
        if (ov && inner_late_ == 0) fork_inner();
        dbg(s, "inner(side)", ov ? side_ : nullptr);
        const int t1 = timer.begin("pass1", s);
        launch_pass1(p, 0, lay_.n[2], s);
        timer.end(t1, s);
        dbg(s, "pass1", p1_side_);
        // issued after pass 1 (default), the interior kernel still depends only
        // on the step's start, but pass 1's launches reach the hardware first and
        // take their SMs before the interior kernel fills the rest: issued first,
        // the interior kernel won that race in most engines and left pass 1 (the
        // critical path) the leftovers -- 159 instead of 145 us/step at 240^3
        if (ov && inner_late_ == 1) fork_inner();
        const int t2 = timer.begin("boundary", s);
        if (fc)
            launch_boundary(p, 0, lay_.n[2], s, t2 < 0);  // (timer events break the PDL pair)
        else
            strict_update(p, 2, 0, lay_.n[2], s);
        timer.end(t2, s);
        dbg(s, "boundary", nullptr);
        if (ov && inner_late_ == 2) fork_inner();
        if (ov) {
            MM_CUDA(cudaStreamWaitEvent(s, join_, 0));
        } else {
            const int ti = timer.begin("inner", s);
            launch_inner(p, 0, lay_.n[2], imode, s);
            timer.end(ti, s);
        }
        dbg(s, "inner", nullptr);
        if (src_off >= 0) launch_inject(p.pn, p.cv, src_off, amp, amp_dev, step_dev, s);
    }

    const char* cpml_path(const StepParams& p) override {
        if (use_cpml(p)) return "cpml";
        return fast_cpml(p) ? "two-pass" : "strict";
    }

    // tuning "debug_sync" == 1: synchronize after each kernel of the step and
    // name the one that faulted (diagnostics only)
    void dbg(cudaStream_t s, const char* what, cudaStream_t s2) {
        if (!dbg_) return;
        cudaError_t e = s2 ? cudaStreamSynchronize(s2) : cudaSuccess;
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess)
            raise(ST_CUDA, std::string("fault after ") + what + ": " + cudaGetErrorString(e));
    }

private:
    int buf_index(const float* ptr) const {
        for (int b = 0; b < 3; ++b)
            if (bufs_[b] == ptr) return b;
        raise(ST_INVAL, "unknown pressure buffer");
    }

    // inner box + the six slab boxes of the local grid (grid.cpp:34-41)
    void regions(const StepParams& p, Box& inner, std::vector<std::pair<int, Box>>& slabs) const {
        int ilo[3], ihi[3];
        for (int a = 0; a < 3; ++a) {
            ilo[a] = std::max(p.nd[a] - p.goff[a], 0);
            ihi[a] = std::min(p.gn[a] - p.nd[a] - p.goff[a], lay_.n[a]);
            ihi[a] = std::max(ihi[a], ilo[a]);
        }
        const int n0 = lay_.n[0], n1 = lay_.n[1], n2 = lay_.n[2];
        inner = Box{{ilo[0], ilo[1], ilo[2]}, {ihi[0], ihi[1], ihi[2]}};
        // first = 2 * kind + side (kind 0/1/2 = X/Y/Z slab, side 0/1 = low/high)
        const std::pair<int, Box> cand[6] = {
            {0, Box{{0, 0, 0}, {ilo[0], n1, n2}}},
            {1, Box{{ihi[0], 0, 0}, {n0, n1, n2}}},
            {2, Box{{ilo[0], 0, 0}, {ihi[0], ilo[1], n2}}},
            {3, Box{{ilo[0], ihi[1], 0}, {ihi[0], n1, n2}}},
            {4, Box{{ilo[0], ilo[1], 0}, {ihi[0], ihi[1], ilo[2]}}},
            {5, Box{{ilo[0], ilo[1], ihi[2]}, {ihi[0], ihi[1], n2}}},
        };
        slabs.clear();
        for (const auto& b : cand)
            if (b.second.hi[0] > b.second.lo[0] && b.second.hi[1] > b.second.lo[1] &&
                b.second.hi[2] > b.second.lo[2])
                slabs.push_back(b);
    }

    struct Work {
        DArr<int4> segs;
        DArr<int> ctr;  // WorkQueue counters
        int nitems = 0;
        int ctas = 0;
        bool empty = true;
        Box box{};
        int x_base = 0;
        BndBox bboxes[6];
        int nbox = 0;
    };

    // inner-kernel domains: the inner box, inner box + Z slabs (one z column),
    // Z slabs only
    enum InnerMode { kInnerOnly = 0, kFull = 1, kZSlabs = 2 };

    using ZRanges = std::vector<std::pair<int, int>>;  // [z_lo, z_hi) plane ranges
    static std::vector<int> wkey(const ZRanges& zr, int mode) {
        std::vector<int> k{mode};
        for (const auto& r : zr) k.push_back(r.first), k.push_back(r.second);
        return k;
    }

    void finish_work(Work& w, const std::vector<Item>& tiles, int ctas, double target,
                     bool even = false, int whole_le = 0, int tail_pct = 0) {
        std::vector<int4> items;
        wave_items(tiles, ctas, target, items, even, whole_le);
        // (tuning bnd_tail) the last tail_pct % of the queue in half-length
        // items: CTAs that finish early take the small ones
        if (tail_pct > 0) {
            const size_t keep = items.size() - items.size() * (size_t)tail_pct / 100;
            std::vector<int4> out(items.begin(), items.begin() + keep);
            for (size_t i = keep; i < items.size(); ++i) {
                const int4 t = items[i];
                const int len = t.w - t.z;
                if (len >= 8) {
                    const int mid = t.z + len / 2;
                    out.push_back(make_int4(t.x, t.y, t.z, mid));
                    out.push_back(make_int4(t.x, t.y, mid, t.w));
                } else {
                    out.push_back(t);
                }
            }
            items.swap(out);
        }
        w.nitems = (int)items.size();
        w.ctas = std::max(1, std::min(ctas, w.nitems));
        w.segs.set(items, stream_setup_);
        w.ctr.set(std::vector<int>{0, 0}, stream_setup_);
    }

    Work& inner_work(const StepParams& p, const ZRanges& ranges, int mode) {
        const auto key = wkey(ranges, mode);
        auto it = inner_cache_.find(key);
        if (it != inner_cache_.end()) return it->second;
        Work& w = inner_cache_[key];
        Box inner;
        std::vector<std::pair<int, Box>> slabs;
        regions(p, inner, slabs);
        w.box = inner;  // x-y box of the tiles; z = the inner z range
        if (inner.hi[0] <= inner.lo[0] || inner.hi[1] <= inner.lo[1]) return w;
        // z ranges of this launch
        std::vector<std::pair<int, int>> zr;
        for (const auto& rg : ranges) {
            auto add = [&](int a, int b) {
                a = std::max(a, rg.first);
                b = std::min(b, rg.second);
                if (b > a) zr.emplace_back(a, b);
            };
            if (mode == kInnerOnly) add(inner.lo[2], inner.hi[2]);
            if (mode == kFull) add(0, lay_.n[2]);
            if (mode == kZSlabs) {
                add(0, inner.lo[2]);
                add(inner.hi[2], lay_.n[2]);
            }
        }
        if (zr.empty()) return w;
        w.empty = false;
        w.x_base = inner.lo[0] & ~3;
        const bool wk = mode == kInnerOnly && wide_;  // k_innerw: 64 x 24 tiles, 1 CTA/SM
        const int ttx = wk ? IW::TX : IC::TX, tty = wk ? IW::TY : IC::TY;
        const int tiles_x = (inner.hi[0] - w.x_base + ttx - 1) / ttx;
        const int tiles_y = (inner.hi[1] - inner.lo[1] + tty - 1) / tty;
        std::vector<Item> tiles;
        for (const auto& r : zr)
            for (int ty = 0; ty < tiles_y; ++ty)
                for (int tx = 0; tx < tiles_x; ++tx) tiles.push_back(Item{tx, ty, r.first, r.second});
        // the target scales with the z-window warm-up (2R planes per item):
        // k_innerw at r = 8 with 96-plane items 1318 -> 1292 us/step at 512^3,
        // r = 2 with 24-plane items 676-682 -> 665-669
        finish_work(w, tiles, sms_ * (wk ? 1 : inner_per_sm_), inner_zt_ * R / 4.0,
                    (tuning("even_chunks") & 1) != 0);
        return w;
    }

    // X and Y slabs (the Z slabs go with the inner kernel)
    Work& bnd_work(const StepParams& p, const ZRanges& ranges) {
        const auto key = wkey(ranges, 0);
        auto it = bnd_cache_.find(key);
        if (it != bnd_cache_.end()) return it->second;
        Work& w = bnd_cache_[key];
        Box inner;
        std::vector<std::pair<int, Box>> slabs;
        regions(p, inner, slabs);
        std::vector<Item> items;  // one per tile
        w.nbox = 0;
        const int kinds = bnd_kinds_;  // (profiling: slab kinds to update)
        for (const auto& s : slabs) {
            if ((s.first / 2 == 2 && zmode_ != 0) || !((kinds >> (s.first / 2)) & 1)) continue;
            const Box& b = s.second;
            ZRanges zs;  // the box's planes within the launch's ranges
            for (const auto& rg : ranges) {
                const int zl = std::max(b.lo[2], rg.first), zh = std::min(b.hi[2], rg.second);
                if (zh > zl) zs.emplace_back(zl, zh);
            }
            if (zs.empty()) continue;
            BndBox& bb = w.bboxes[w.nbox];
            for (int a = 0; a < 3; ++a) {
                bb.lo[a] = b.lo[a];
                bb.hi[a] = b.hi[a];
            }
            bb.kind = s.first / 2;
            bb.side = s.first % 2;
            bb.x_base = b.lo[0] & ~3;
            const int tiles_x = (b.hi[0] - bb.x_base + BC::TX - 1) / BC::TX;
            const int tiles_y = (b.hi[1] - b.lo[1] + BC::TY - 1) / BC::TY;
            for (const auto& z : zs)
                for (int ty = 0; ty < tiles_y; ++ty)
                    for (int tx = 0; tx < tiles_x; ++tx)
                        items.push_back(Item{w.nbox | (tx << 3), ty, z.first, z.second});
            ++w.nbox;
        }
        if (items.empty()) return w;
        w.empty = false;
        // short tiles (the Z slabs) as whole items on big grids: 512^3 729.8 ->
        // 722.3 us, r=8 1340 -> 1318, 1000^3 3910 -> 3878; at 240^3 (too few items
        // per CTA to balance 27-plane items) 141.2 -> 141.8, so auto = off there
        long long bw = tuning("bnd_whole");
        if (bw < 0) bw = (double)lay_.n[0] * lay_.n[1] * lay_.n[2] > 3.0e7 ? 64 : 0;
        // (the target scales with the z warm-up like the interior's: r = 8 with
        // 24-plane items 1293 -> 1263 us/step at 512^3, 229 -> 223 at 240^3;
        // r = 2 with 6-plane items 131.0 -> 129.0 at 240^3)
        finish_work(w, items, sms_ * bnd_per_sm_, bnd_zt_ * R / 4.0,
                    (tuning("even_chunks") & 2) != 0, (int)bw, (int)tuning("bnd_tail"));
        return w;
    }

    // k_zslab runs one CTA per SM
    int zs_ctas(const Work& w) const { return std::max(1, std::min(w.nitems, sms_)); }

    void launch_inner(const StepParams& p, int z_lo, int z_hi, int mode, cudaStream_t s) {
        launch_inner(p, ZRanges{{z_lo, z_hi}}, mode, s);
    }
    void launch_inner(const StepParams& p, const ZRanges& zr, int mode, cudaStream_t s) {
        if (mode == kFull && zmode_ == 1) {  // inner box and Z slabs separately
            launch_inner(p, zr, kInnerOnly, s);
            launch_inner(p, zr, kZSlabs, s);
            return;
        }
        Work& w = inner_work(p, zr, mode);
        if (w.empty) return;
        InnerParams ip;
        std::memset(&ip, 0, sizeof ip);
        ip.lay = lay_;
        for (int a = 0; a < 3; ++a) {
            ip.lo[a] = w.box.lo[a];
            ip.hi[a] = w.box.hi[a];
        }
        ip.x_base = w.x_base;
        ip.segs = w.segs.ptr;
        ip.wq = WorkQueue{w.ctr.ptr, w.nitems};
        ip.pn = p.pn;
        float sum = 0.0f;
        for (int m = 0; m < R; ++m) {
            ip.cx[m] = p.c2[0][m];
            ip.cy[m] = p.c2[1][m];
            ip.cz[m] = p.c2[2][m];
            sum += p.c2[0][m] + p.c2[1][m] + p.c2[2][m];
        }
        ip.center = -2.0f * sum;
        ip.zi_lo = w.box.lo[2];
        ip.zi_hi = w.box.hi[2];
        ip.zsplit = p.gn[2] - p.nd[2] - p.goff[2];
        ip.tik_x = p.tik[0];
        ip.tik_y = p.tik[1];
        ip.ta_z = p.ta[2];
        ip.tb_z = p.tb[2];
        ip.tik_z = p.tik[2];
        for (int sd = 0; sd < 2; ++sd) {
            ip.zrun[sd] = p.run[2][sd];
            ip.dpz[sd] = dpz_[sd].ptr;
            ip.dz_lo[sd] = dz_lo_[sd];
            ip.dz_hi[sd] = dz_hi_[sd];
        }
        const int bc = buf_index(p.pc), bp = buf_index(p.pp);
        const CUtensorMap &a = in_halo_[bc], &b = in_tile_[bp];
        if (mode == kInnerOnly && wide_) {
            if constexpr (kW) {
                const int g = std::min(w.ctas, inner_cap_);
                if (order_ == 2)
                    k_innerw<R, 2><<<g, IW::NT, IW::SMEM, s>>>(inw_halo_[bc], inw_tile_[bp],
                                                                cv_inw_, ip);
                else
                    k_innerw<R, 1><<<g, IW::NT, IW::SMEM, s>>>(inw_halo_[bc], inw_tile_[bp],
                                                                cv_inw_, ip);
            }
        } else if (mode != kInnerOnly || col_inner_) {  // column kernel (MM_ZSLABS = 1, 2; R > 4)
            if constexpr (kZs) {
                constexpr size_t zsm = ZSlabCfg<R>::SMEM;
                if (order_ == 2)
                    k_zslab<R, 2><<<zs_ctas(w), ZSlabCfg<R>::NT, zsm, s>>>(a, b, cv_in_, ip);
                else
                    k_zslab<R, 1><<<zs_ctas(w), ZSlabCfg<R>::NT, zsm, s>>>(a, b, cv_in_, ip);
            }
        } else if (order_ == 2) {
            k_inner<R, 2><<<std::min(w.ctas, inner_cap_), IC::NT, IC::SMEM, s>>>(a, b, cv_in_, ip);
        } else {
            k_inner<R, 1><<<std::min(w.ctas, inner_cap_), IC::NT, IC::SMEM, s>>>(a, b, cv_in_, ip);
        }
        note_launches(1);
        MM_CUDA(cudaGetLastError());
    }

    // dpsi_z planes [lo-R, hi+R) of each z run (k_p1 writes, k_bnd reads).  When
    // the two ranges would overlap (z extent < 2 (nd + R)), a plane's dpsi_z mixes
    // both runs and the strict kernels do pass 1 and the slabs instead.
    bool ensure_dpz(const StepParams& p) {
        if (dpz_valid_) return !zmix_;
        const CpmlRun& r0 = p.run[2][0];
        const CpmlRun& r1 = p.run[2][1];
        const bool h0 = r0.hi > r0.lo, h1 = r1.hi > r1.lo;
        zmix_ = h0 && h1 && r0.hi + R > r1.lo - R;
        for (int sd = 0; sd < 2; ++sd) {
            const CpmlRun& r = p.run[2][sd];
            dz_lo_[sd] = 0;
            dz_hi_[sd] = 0;
            if (r.hi <= r.lo || zmix_) continue;
            dz_lo_[sd] = r.lo - R;
            dz_hi_[sd] = r.hi + R;
            const long long planes = r.hi - r.lo + 2 * R;
            dpz_[sd].alloc_zero((size_t)(r.s2 * planes), stream_setup_);
            maps_.dpz[sd] = make_map(dpz_[sd].ptr, r.s1, lay_.n[1], planes, r.s1, r.s2, BC::TX,
                                     BC::TY);
        }
        dpz_valid_ = true;
        return !zmix_;
    }

    void refresh_run_maps(const StepParams& p) {
        bool same = true;
        for (int a = 0; a < 3; ++a)
            for (int sd = 0; sd < 2; ++sd)
                same = same && p.run[a][sd].psi == runs_[a][sd].psi &&
                       p.run[a][sd].zeta == runs_[a][sd].zeta;
        if (same && runs_valid_) return;
        for (int a = 0; a < 3; ++a)
            for (int sd = 0; sd < 2; ++sd) {
                const CpmlRun& r = p.run[a][sd];
                runs_[a][sd] = r;
                if (a == 0) maps_.psi[0][sd] = run_map(lay_, r, a, r.psi, BC::BX, BC::TY);  // x halo
                if (a == 1) maps_.psi[1][sd] = run_map(lay_, r, a, r.psi, BC::TX, BC::BY);  // y halo
                maps_.zeta[a][sd] = run_map(lay_, r, a, r.zeta, BC::TX, BC::TY);
                p1maps_.psi[a][sd] = a == 2 ? run_map(lay_, r, a, r.psi, P1C::TX, P1C::TY)
                                            : run_map(lay_, r, a, r.psi, P1X::TX, P1X::TY);
                if constexpr (kCpml) {
                    cmaps_.psi[a][sd] = run_map(lay_, r, a, r.psi, CC::TX, CC::TY);
                    cmaps_.zeta[a][sd] = run_map(lay_, r, a, r.zeta, CC::TX, CC::TY);
                }
            }
        // the fused kernel's tiles follow the runs' extents
        cgeo_.built = false;
        cpml_cache_.clear();
        runs_valid_ = true;
    }

    // fast CPML: k_p1 + k_bnd + the inner kernel's Z-slab planes
    bool fast_cpml(const StepParams& p) {
        if constexpr (!(kBnd && kP1))
            return false;
        else
            return ensure_dpz(p);
    }

    // after_p1: k_p1 is the kernel right before on `s` (the step): k_bnd may
    // then launch programmatically (PDL) -- its p_cur ring streams before
    // griddepcontrol.wait, which is safe only behind a kernel that does not
    // write p_cur.  Any other predecessor (the epilogue, an injection, the
    // interior kernel of the plane-range schedule) gets a plain launch.
    void launch_boundary(const StepParams& p, int z_lo, int z_hi, cudaStream_t s,
                         bool after_p1 = false) {
        launch_boundary(p, ZRanges{{z_lo, z_hi}}, s, after_p1);
    }
    void launch_boundary(const StepParams& p, const ZRanges& zr, cudaStream_t s,
                         bool after_p1 = false) {
        if constexpr (kBnd && kP1) {
            Work& w = bnd_work(p, zr);
            if (w.empty) return;
            refresh_run_maps(p);
            maps_.pc = bd_halo_[buf_index(p.pc)];
            maps_.pp = bd_tile_[buf_index(p.pp)];
            maps_.cv = cv_bd_;
            BndParams bp_;
            std::memset(&bp_, 0, sizeof bp_);
            bp_.lay = lay_;
            for (int i = 0; i < w.nbox; ++i) bp_.box[i] = w.bboxes[i];
            bp_.nbox = w.nbox;
            for (int a = 0; a < 3; ++a) {
                bp_.run[a][0] = p.run[a][0];
                bp_.run[a][1] = p.run[a][1];
                bp_.ta[a] = p.ta[a];
                bp_.tb[a] = p.tb[a];
                bp_.tik[a] = p.tik[a];
                for (int m = 0; m < kMaxR; ++m) {
                    bp_.c2[a][m] = p.c2[a][m];
                    bp_.c1[a][m] = p.c1[a][m];
                }
            }
            for (int sd = 0; sd < 2; ++sd) {
                bp_.dpz[sd] = dpz_[sd].ptr;
                bp_.dz_lo[sd] = dz_lo_[sd];
                bp_.dz_hi[sd] = dz_hi_[sd];
            }
            bp_.pp = p.pp;
            bp_.cv = p.cv;
            bp_.pn = p.pn;
            bp_.segs = w.segs.ptr;
            bp_.wq = WorkQueue{w.ctr.ptr, w.nitems};
            // tuning "bnd_ctas" (diagnostics): cap the CTA count (more items per CTA)
            const int ctas = std::min(w.ctas, bnd_cap_);
            const bool pdl = pdl_ && after_p1;
            if (order_ == 2)
                launch_pdl(k_bnd<R, 2>, ctas, BC::NT, BC::SMEM, s, pdl, maps_, bp_);
            else
                launch_pdl(k_bnd<R, 1>, ctas, BC::NT, BC::SMEM, s, pdl, maps_, bp_);
            note_launches(1);
            MM_CUDA(cudaGetLastError());
        }
    }

    void launch_pass1(const StepParams& p, int z_lo, int z_hi, cudaStream_t s) {
        if constexpr (!(kBnd && kP1)) {
            strict_pass1(p, z_lo, z_hi, s);
            return;
        } else {
            if (!fast_cpml(p)) {
                strict_pass1(p, z_lo, z_hi, s);
                return;
            }
            const auto key = std::make_pair(z_lo, z_hi);
            auto it = pass1_cache_.find(key);
            if (it == pass1_cache_.end()) {
                Pass1Work& e = pass1_cache_[key];
                std::vector<Item> tiles;
                std::vector<int4> zitems;
                const int axes = p1_axes_;  // (profiling: run axes to update)
                for (int ax = 0; ax < 3; ++ax)
                    for (int side = 0; side < 2; ++side) {
                        const CpmlRun& r = p.run[ax][side];
                        if (r.hi <= r.lo || !((axes >> ax) & 1)) continue;
                        RunDesc d{ax, side, {0, 0, 0}, {lay_.n[0], lay_.n[1], lay_.n[2]}, 0};
                        d.lo[ax] = r.lo;
                        d.hi[ax] = r.hi;
                        d.lo[2] = std::max(d.lo[2], z_lo);
                        d.hi[2] = std::min(d.hi[2], z_hi);
                        if (d.hi[2] <= d.lo[2]) continue;
                        d.x_base = d.lo[0] & ~3;  // = r.org for axis 0
                        const int ri = e.nrd++;
                        e.rd[ri] = d;
                        const int TXa = ax == 2 ? P1C::TX : P1X::TX, TYa = ax == 2 ? P1C::TY : P1X::TY;
                        const int tx = (d.hi[0] - d.x_base + TXa - 1) / TXa;
                        const int ty = (d.hi[1] - d.lo[1] + TYa - 1) / TYa;
                        // z runs: one item spans the whole run (the dpsi_z window)
                        if (ax == 2 && (d.lo[2] != r.lo || d.hi[2] != r.hi))
                            raise(ST_INVAL, "pass 1 z range must not cut a z damping run");
                        for (int b = 0; b < ty; ++b)
                            for (int a = 0; a < tx; ++a) {
                                if (ax == 2)
                                    zitems.push_back(make_int4(ri | (a << 3), b, d.lo[2], d.hi[2]));
                                else
                                    tiles.push_back(Item{ri | (a << 3), b, d.lo[2], d.hi[2]});
                            }
                    }
                // two launches: the x/y runs (many small CTAs) and the z runs
                std::vector<int4> items;
                wave_items(tiles, sms_ * p1x_per_sm_, p1_zt_, items, (tuning("even_chunks") & 4) != 0);
                e.nx = (int)items.size();
                // (tuning p1x_ctas: x/y CTAs per SM; 0 = as many as fit)
                const long long pxs = tuning("p1x_ctas");
                const int xper = pxs > 0 ? (int)std::min<long long>(pxs, p1x_per_sm_) : p1x_per_sm_;
                e.ctas_x = std::max(1, std::min(sms_ * xper, e.nx));
                e.nz = (int)zitems.size();
                e.ctas_z = std::max(1, std::min(sms_ * p1_per_sm_, e.nz));
                items.insert(items.end(), zitems.begin(), zitems.end());
                e.nitems = (int)items.size();
                e.items.set(items, stream_setup_);
                e.ctr.set(std::vector<int>{0, 0, 0, 0}, stream_setup_);
                it = pass1_cache_.find(key);
            }
            auto& e = it->second;
            if (e.nitems == 0) return;
            refresh_run_maps(p);
            const int bc = buf_index(p.pc);
            p1maps_.px = p1x_[bc];
            p1maps_.py = p1y_[bc];
            p1maps_.pz = p1z_[bc];
            P1Params pp;
            std::memset(&pp, 0, sizeof pp);
            pp.lay = lay_;
            for (int i = 0; i < e.nrd; ++i) pp.rd[i] = e.rd[i];
            for (int a = 0; a < 3; ++a) {
                pp.run[a][0] = p.run[a][0];
                pp.run[a][1] = p.run[a][1];
                pp.ta[a] = p.ta[a];
                pp.tb[a] = p.tb[a];
                for (int m = 0; m < kMaxR; ++m) pp.c1[a][m] = p.c1[a][m];
            }
            pp.dpz[0] = dpz_[0].ptr;
            pp.dpz[1] = dpz_[1].ptr;
            // the two launches run concurrently (z on a second stream, joined
            // before returning): the long z items share the SMs with x/y work
            // (z on the step's stream, so the boundary kernel can follow it with
            // a programmatic dependency; x/y on a second stream, joined first)
            const bool two = e.nz > 0 && e.nx > 0 && p1_side_;
            cudaStream_t sz = s, sx = s;
            if (two) {
                MM_CUDA(cudaEventRecord(p1_fork_, s));
                MM_CUDA(cudaStreamWaitEvent(p1_side_, p1_fork_, 0));
                sx = p1_side_;
            }
            if (e.nz > 0) {  // z runs first: their items are the long ones
                pp.items = e.items.ptr + e.nx;
                pp.wq = WorkQueue{e.ctr.ptr + 2, e.nz};
                if (order_ == 2)
                    k_p1<R, 2, true><<<e.ctas_z, P1C::NT, P1C::SMEM, sz>>>(p1maps_, pp);
                else
                    k_p1<R, 1, true><<<e.ctas_z, P1C::NT, P1C::SMEM, sz>>>(p1maps_, pp);
                note_launches(1);
                MM_CUDA(cudaGetLastError());
            }
            if (e.nx > 0) {
                pp.items = e.items.ptr;
                pp.wq = WorkQueue{e.ctr.ptr, e.nx};
                if (order_ == 2)
                    k_p1<R, 2, false><<<e.ctas_x, P1X::NT, P1X::SMEM, sx>>>(p1maps_, pp);
                else
                    k_p1<R, 1, false><<<e.ctas_x, P1X::NT, P1X::SMEM, sx>>>(p1maps_, pp);
                note_launches(1);
                MM_CUDA(cudaGetLastError());
            }
            if (two) {
                MM_CUDA(cudaEventRecord(p1_join_, p1_side_));
                MM_CUDA(cudaStreamWaitEvent(s, p1_join_, 0));
            }
        }
    }

    // ---------------------------------------------------------------- k_cpml
    // 1-D tile partition of [0, n) along x (margin 0; the tile of a run starts
    // at its 16-byte-aligned origin) or y (margin R) for the fused kernel:
    // each part = physical tile start t0, owned range [lo, hi), damping run
    // side (-1: none).  Rules (fast_cpml.cuh): a run lies inside its tile, the
    // rows within `margin` of it are owned by that tile only, and no other
    // tile of the partition holds a run.  false: the two-pass path serves it.
    struct Part {
        int t0, lo, hi, side;
    };
    static bool cpml_parts(int n, const CpmlRun& L, const CpmlRun& H, int margin, bool xaxis,
                           std::vector<Part>& out) {
        constexpr int T = CC::TX;  // == CC::TY
        out.clear();
        const bool hl = L.hi > L.lo, hh = H.hi > H.lo;
        if (hl && (L.lo != 0 || L.org != 0)) return false;
        const int c1 = hl ? std::min(T, n) : 0;
        int t0h = n, own_h = n;
        if (hh) {
            t0h = xaxis ? H.org : std::max(n - T, 0);
            own_h = xaxis ? H.org : std::max(t0h, c1);
            if (H.hi > t0h + T) return false;         // the run fits in its tile
            if (own_h > H.lo - margin) return false;  // run + margin owned by its tile
        }
        const int c1e = std::min(c1, own_h);
        if (hl && L.hi + margin > c1e) return false;
        if (hl) out.push_back(Part{0, 0, c1e, 0});
        for (int m = c1e; m < own_h; m += T) out.push_back(Part{m, m, std::min(m + T, own_h), -1});
        if (hh) out.push_back(Part{t0h, own_h, n, 1});
        return true;
    }

    // Tiles of the fused kernel (built once per CPML run geometry).
    struct CpmlGeo {
        bool built = false, ok = false;
        std::vector<CTile> tiles;
        std::vector<char> full;  // 1: every plane; 0: the Z-slab planes only
        DArr<CTile> dtiles;
        std::vector<std::pair<int, int>> forb;  // forbidden chunk boundaries (a, b), open
        Box inner{};
    };
    CpmlGeo& cpml_geo(const StepParams& p) {
        CpmlGeo& g = cgeo_;
        if (g.built) return g;
        g.built = true;
        g.ok = false;
        if constexpr (kCpml) {
            // x and y are whole in every engine the fused kernel serves (the
            // multi-GPU path cuts z only)
            if (p.goff[0] != 0 || p.goff[1] != 0 || lay_.n[0] != p.gn[0] || lay_.n[1] != p.gn[1])
                return g;
            std::vector<Part> xp, yp;
            if (!cpml_parts(lay_.n[0], p.run[0][0], p.run[0][1], 0, true, xp)) return g;
            if (!cpml_parts(lay_.n[1], p.run[1][0], p.run[1][1], R, false, yp)) return g;
            const CpmlRun &z0 = p.run[2][0], &z1 = p.run[2][1];
            const bool h0 = z0.hi > z0.lo, h1 = z1.hi > z1.lo;
            // a Z slab sees its own z run only: the other run must lie R away
            if (h0 && h1 && z1.lo - z0.hi < R) return g;
            std::vector<std::pair<int, Box>> slabs;
            regions(p, g.inner, slabs);
            const Box& I = g.inner;
            g.forb.clear();
            for (const CpmlRun* r : {&z0, &z1})
                if (r->hi > r->lo) g.forb.emplace_back(r->lo - R, r->hi + R);
            g.tiles.clear();
            g.full.clear();
            for (const Part& a : xp)
                for (const Part& b : yp) {
                    if (a.hi <= a.lo || b.hi <= b.lo) continue;
                    const bool xyslab = a.lo < I.lo[0] || a.hi > I.hi[0] || b.lo < I.lo[1] ||
                                        b.hi > I.hi[1] || I.hi[0] <= I.lo[0] || I.hi[1] <= I.lo[1];
                    const bool zslab = I.lo[2] > 0 || I.hi[2] < lay_.n[2];
                    if (!xyslab && !zslab) continue;
                    g.tiles.push_back(CTile{a.t0, a.hi, b.t0, b.hi, a.side, b.side, a.lo, b.lo});
                    g.full.push_back(xyslab ? 1 : 0);
                }
            g.dtiles.set(g.tiles, stream_setup_);
            g.ok = true;
        }
        return g;
    }

    bool use_cpml(const StepParams& p) {
        if (!cpml_on_) return false;
        refresh_run_maps(p);  // (rebuilds the tiles when the runs changed)
        return cpml_geo(p).ok;
    }

    // [a, b) cut into chunks of about `target` planes, no boundary inside a
    // forbidden zone (within R of a z run: chunks update psi_z in place); a
    // boundary that falls in a zone moves down to the zone's start when the
    // chunk stays non-empty, else up to its end
    static void chunk_planes(int a, int b, int target, const std::vector<std::pair<int, int>>& forb,
                             std::vector<std::pair<int, int>>& out) {
        int zb = a;
        while (zb < b) {
            int ze = std::min(b, zb + std::max(1, target));
            for (bool moved = true; moved;) {
                moved = false;
                for (const auto& f : forb)
                    if (ze > f.first && ze < f.second && ze < b) {
                        ze = f.first > zb ? f.first : std::min(b, f.second);
                        moved = true;
                    }
            }
            out.emplace_back(zb, ze);
            zb = ze;
        }
    }

    struct CpmlWork {
        DArr<int4> items;
        DArr<int> ctr;
        int nitems = 0, ctas = 0;
    };
    CpmlWork& cpml_work(const StepParams& p, const ZRanges& ranges) {
        const auto key = wkey(ranges, 0);
        auto it = cpml_cache_.find(key);
        if (it != cpml_cache_.end()) return it->second;
        CpmlWork& w = cpml_cache_[key];
        CpmlGeo& g = cpml_geo(p);
        const int nz = lay_.n[2];
        // the planes of every tile within this launch's ranges
        std::vector<std::pair<int, std::pair<int, int>>> segs;  // (tile, [a, b))
        long long planes = 0;
        for (size_t t = 0; t < g.tiles.size(); ++t) {
            std::vector<std::pair<int, int>> zs;
            if (g.full[t])
                zs.emplace_back(0, nz);
            else {
                zs.emplace_back(0, g.inner.lo[2]);
                zs.emplace_back(g.inner.hi[2], nz);
            }
            for (const auto& z : zs)
                for (const auto& rg : ranges) {
                    const int a = std::max(z.first, rg.first), b = std::min(z.second, rg.second);
                    if (b > a) {
                        segs.push_back({(int)t, {a, b}});
                        planes += b - a;
                    }
                }
        }
        const int slots = sms_ * cpml_per_sm_;
        // about two items per CTA, at least 12 planes each (items pay a 2R- or
        // 4R-plane warm-up of the z window)
        int target = cpml_zt_ > 0 ? cpml_zt_
                                  : (int)std::max<long long>(12, (planes + 2LL * slots - 1) / (2LL * slots));
        // order: items near a z run first (they also update psi_z and carry a
        // 4R-plane warm-up, the longest items), then chunk-major -- the items
        // in flight are neighbouring tiles at nearby depths, whose p_cur halo
        // planes meet in L2
        auto near_z = [&](int zb, int ze) {
            for (const auto& f : g.forb)
                if (zb < f.second && ze > f.first) return true;
            return false;
        };
        std::vector<std::pair<long long, int4>> items;  // (sort key, item)
        for (const auto& sg : segs) {
            std::vector<std::pair<int, int>> ch;
            chunk_planes(sg.second.first, sg.second.second, target, g.forb, ch);
            for (const auto& c : ch) {
                const long long key = (near_z(c.first, c.second) ? 0LL : 1LL << 40) +
                                      ((long long)c.first << 20) + sg.first;
                items.push_back({key, make_int4(sg.first, c.first, c.second, 0)});
            }
        }
        std::stable_sort(items.begin(), items.end(),
                         [](const auto& a, const auto& b) { return a.first < b.first; });
        std::vector<int4> v;
        for (const auto& i : items) v.push_back(i.second);
        w.nitems = (int)v.size();
        w.ctas = std::max(1, std::min(slots, w.nitems));
        w.items.set(v, stream_setup_);
        w.ctr.set(std::vector<int>{0, 0}, stream_setup_);
        return w;
    }

    void launch_cpml(const StepParams& p, const ZRanges& zr, cudaStream_t s) {
        if constexpr (kCpml) {
            refresh_run_maps(p);
            CpmlGeo& g = cpml_geo(p);
            if (!g.ok) raise(ST_INVAL, "k_cpml cannot serve this layout");
            CpmlWork& w = cpml_work(p, zr);
            if (w.nitems == 0) return;
            CpmlMaps M = cmaps_;
            M.pc = cm_pc_[buf_index(p.pc)];
            M.pp = cm_tile_[buf_index(p.pp)];
            M.cv = cm_cv_;
            CpmlParams P;
            std::memset(&P, 0, sizeof P);
            P.lay = lay_;
            for (int a = 0; a < 3; ++a) {
                P.ilo[a] = g.inner.lo[a];
                P.ihi[a] = g.inner.hi[a];
                P.run[a][0] = p.run[a][0];
                P.run[a][1] = p.run[a][1];
                P.ta[a] = p.ta[a];
                P.tb[a] = p.tb[a];
                P.tik[a] = p.tik[a];
                for (int m = 0; m < kMaxR; ++m) {
                    P.c2[a][m] = p.c2[a][m];
                    P.c1[a][m] = p.c1[a][m];
                }
            }
            P.tiles = g.dtiles.ptr;
            P.items = w.items.ptr;
            P.wq = WorkQueue{w.ctr.ptr, w.nitems};
            P.pn = p.pn;
            if (order_ == 2)
                k_cpml<RC, 2><<<w.ctas, CC::NT, CC::SMEM, s>>>(M, P);
            else
                k_cpml<RC, 1><<<w.ctas, CC::NT, CC::SMEM, s>>>(M, P);
            note_launches(1);
            MM_CUDA(cudaGetLastError());
        }
    }

    struct Pass1Work {
        RunDesc rd[6];
        int nrd = 0;
        DArr<int4> items;  // x/y-run items, then z-run items
        DArr<int> ctr;     // two WorkQueue counter pairs
        int nitems = 0, nx = 0, nz = 0;
        int ctas_x = 0, ctas_z = 0;
    };

    Layout lay_;
    int device_;
    int order_ = 2;
    int sms_ = 148, inner_per_sm_ = 1, bnd_per_sm_ = 1, cpml_per_sm_ = 1;
    int inner_cap_ = 1 << 30;
    bool cpml_on_ = false, dbg_ = false;
    int cpml_zt_ = 0, inner_late_ = 0, bnd_kinds_ = 7, bnd_cap_ = 1 << 30, p1_axes_ = 7;
    CUtensorMap cm_pc_[3], cm_tile_[3], cm_cv_;
    CpmlMaps cmaps_{};
    CpmlGeo cgeo_;
    std::map<std::vector<int>, CpmlWork> cpml_cache_;
    double inner_zt_ = 48.0, bnd_zt_ = 48.0;
    int zmode_ = 0;
    bool wide_ = false;  // R > 4: k_innerw serves the inner box
    bool pdl_ = true;
    bool overlap_ = false;
    cudaStream_t side_ = nullptr;
    cudaEvent_t fork_ = nullptr, join_ = nullptr;
    cudaStream_t p1_side_ = nullptr;
    cudaEvent_t p1_fork_ = nullptr, p1_join_ = nullptr;
    bool col_inner_ = false;
    const float* bufs_[3];
    CUtensorMap in_halo_[3], in_tile_[3], bd_halo_[3], bd_tile_[3], cv_in_, cv_bd_;
    CUtensorMap inw_halo_[3], inw_tile_[3], cv_inw_;  // k_innerw (R > 4)
    BndMaps maps_;
    P1Maps p1maps_;
    DArr<float> dpz_[2];
    int dz_lo_[2] = {0, 0}, dz_hi_[2] = {0, 0};
    bool dpz_valid_ = false, zmix_ = false;
    CUtensorMap p1x_[3], p1y_[3], p1z_[3];
    int p1_per_sm_ = 1, p1x_per_sm_ = 1;
    double p1_zt_ = 16.0;
    CpmlRun runs_[3][2] = {};
    bool runs_valid_ = false;
    cudaStream_t stream_setup_ = nullptr;
    std::map<std::vector<int>, Work> inner_cache_, bnd_cache_;
    std::map<std::pair<int, int>, Pass1Work> pass1_cache_;
};

}  // namespace

std::unique_ptr<FastPlan> make_fast_plan(const Layout& lay, int device, float* const bufs[3],
                                         const float* cv, int order) {
    switch (lay.r) {
        case 2: return std::make_unique<FastPlanR<2>>(lay, device, bufs, cv, order);
        case 4: return std::make_unique<FastPlanR<4>>(lay, device, bufs, cv, order);
        case 8: return std::make_unique<FastPlanR<8>>(lay, device, bufs, cv, order);
        default: return nullptr;  // other radii run the strict kernels
    }
}

}  // namespace mmb

#ifdef MM_TRACE
// (diagnostics) the per-CTA trace ring of the fast kernels: n records of
// (kernel id, SM, start ns, end ns); the ring restarts after the read
extern "C" int mm_trace_dump(unsigned long long* out, int cap, int* n) {
    unsigned int cnt = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&cnt, mmb::fast::g_mm_trace_n, sizeof cnt);
    const int m = (int)(cnt < 65536u ? cnt : 65536u);
    const int k = m < cap ? m : cap;
    if (k > 0)
        cudaMemcpyFromSymbol(out, mmb::fast::g_mm_trace, sizeof(unsigned long long) * 4 * (size_t)k);
    *n = k;
    const unsigned int zero = 0;
    cudaMemcpyToSymbol(mmb::fast::g_mm_trace_n, &zero, sizeof zero);
    return 0;
}
#endif
