// kernels_fast.cu -- MM_MODE_FAST step: plan (tensor maps, work lists) + launches.
//
// One step = k_p1 (CPML pass 1: psi, and dpsi_z of the z runs) -> k_bnd (pass 2
// over the X and Y slabs) -> k_inner (the inner x-y box over every z: plain
// update inside, pass 2 along z in the Z slabs) -> source injection, each
// kernel persistent over the whole GPU, pulling (tile, z-chunk) work items.
// Kernels: fast_pass1.cuh (k_p1), fast_boundary.cuh (k_bnd), fast_inner.cuh (k_inner).
// When the fast CPML kernels cannot serve a layout (radius 8, or z runs closer
// than 2R), pass 1 and the slabs run the strict kernels and k_inner the inner box.
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
    // 256B-aligned; 256B promotion would fetch unused bytes).  MM_L2PROMO=0..3
    // selects none/64B/128B/256B for experiments.
    static const CUtensorMapL2promotion promo = [] {
        const char* e = std::getenv("MM_L2PROMO");
        const int v = e ? std::atoi(e) : 2;
        return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
               : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
               : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                        : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    }();
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
                std::vector<int4>& out) {
    out.clear();
    if (tiles.empty()) return;
    long long tp = 0;
    int zmax = 0;
    for (const auto& t : tiles) {
        tp += t.zhi - t.zlo;
        zmax = std::max(zmax, t.zhi - t.zlo);
    }
    const double per_cta = (double)tp / std::max(1, ctas);
    const int waves = std::max(1, (int)std::lround(per_cta / target));
    const int zc = std::max(4, (int)((tp + (long long)ctas * waves - 1) / ((long long)ctas * waves)));
    for (int k = 0; (long long)k * zc < zmax; ++k)
        for (const auto& t : tiles) {
            const int zb = t.zlo + k * zc;
            if (zb >= t.zhi) continue;
            out.push_back(make_int4(t.tag, t.ty, zb, std::min(t.zhi, zb + zc)));
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
    static constexpr bool kP1 = P1C::SMEM <= 200 * 1024;

public:
    FastPlanR(const Layout& lay, int device, float* const bufs[3], const float* cv)
        : lay_(lay), device_(device) {
        for (int b = 0; b < 3; ++b) {
            bufs_[b] = bufs[b];
            in_halo_[b] = field_map(lay, bufs[b], IC::BX, IC::BY);
            in_tile_[b] = field_map(lay, bufs[b], IC::TX, IC::TY);
            bd_halo_[b] = field_map(lay, bufs[b], BC::BX, BC::BY);
            bd_tile_[b] = field_map(lay, bufs[b], BC::TX, BC::TY);
            p1x_[b] = field_map(lay, bufs[b], P1C::BXX, P1C::TY);
            p1y_[b] = field_map(lay, bufs[b], P1C::TX, P1C::BYY);
            p1z_[b] = field_map(lay, bufs[b], P1C::TX, P1C::TY);
        }
        cv_in_ = field_map(lay, cv, IC::TX, IC::TY);
        cv_bd_ = field_map(lay, cv, BC::TX, BC::TY);
        const char* ord = std::getenv("MM_FAST_ORDER");
        // MM_FAST_ORDER: 2 (default) bit-exact reference order, 1 FMA, 0 factored
        order_ = ord ? std::max(0, std::min(2, std::atoi(ord))) : 2;
        // z-chunk targets (planes per work item) of the two persistent kernels
        auto envf = [](const char* k, double d) {
            const char* v = std::getenv(k);
            return v ? std::max(1.0, std::atof(v)) : d;
        };
        inner_zt_ = envf("MM_INNER_ZT", 48.0);
        bnd_zt_ = envf("MM_BND_ZT", 12.0);
        p1_zt_ = envf("MM_P1_ZT", 16.0);
        // Z slabs: 0 = k_bnd tiles, 1 = k_zslab over the Z slabs after k_inner,
        // 2 = k_zslab over whole z columns of the inner box (instead of k_inner)
        if (const char* zm = std::getenv("MM_ZSLABS")) zmode_ = std::max(0, std::min(2, std::atoi(zm)));
        if (!kZs) zmode_ = 0;
        { const char* ov = std::getenv("MM_OVERLAP"); overlap_ = !ov || ov[0] != '0'; }
        // side streams at the lowest priority: pass 1's z runs (on the step's
        // stream, the critical path) are scheduled first
        int prio_lo = 0, prio_hi = 0;
        MM_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        MM_CUDA(cudaStreamCreateWithPriority(&p1_side_, cudaStreamNonBlocking,
                                             main_stream_priority() >= 2 ? prio_hi : prio_lo));
        { const char* e = std::getenv("MM_PDL"); pdl_ = !e || e[0] != '0'; }
        MM_CUDA(cudaEventCreateWithFlags(&p1_fork_, cudaEventDisableTiming));
        MM_CUDA(cudaEventCreateWithFlags(&p1_join_, cudaEventDisableTiming));
        if (overlap_) {
            int lo = 0, hi = 0;
            MM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            MM_CUDA(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, lo));
            MM_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
            MM_CUDA(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming));
        }
        // R > 4: the interior kernel's z loop unrolled by 2R+1 overflows the
        // instruction cache; the column kernel (smem z window) serves the inner
        // box and the Z slabs instead
        col_inner_ = kZs && R > 4;
        if (col_inner_ && !std::getenv("MM_ZSLABS")) zmode_ = 2;
        cudaDeviceProp prop;
        MM_CUDA(cudaGetDeviceProperties(&prop, device));
        sms_ = prop.multiProcessorCount;
        for (auto fn : {k_inner<R, 0>, k_inner<R, 1>, k_inner<R, 2>})
            MM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)IC::SMEM));
        if constexpr (kZs)
            for (auto fn : {k_zslab<R, 0>, k_zslab<R, 1>, k_zslab<R, 2>})
                MM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)ZSlabCfg<R>::SMEM));
        int per_sm = 0;
        MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inner<R, 2>, IC::NT,
                                                              IC::SMEM));
        inner_per_sm_ = std::max(1, per_sm);
        if constexpr (kBnd) {
            MM_CUDA(cudaFuncSetAttribute(k_bnd<R, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)BC::SMEM));
            MM_CUDA(cudaFuncSetAttribute(k_bnd<R, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)BC::SMEM));
            MM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bnd<R, 2>, BC::NT,
                                                                  BC::SMEM));
            bnd_per_sm_ = std::max(1, per_sm);
        }
        if constexpr (kP1) {
            for (auto fn : {k_p1<R, 1, true>, k_p1<R, 2, true>})
                MM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)P1C::SMEM));
            for (auto fn : {k_p1<R, 1, false>, k_p1<R, 2, false>})
                MM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)P1X::SMEM));
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

    void step(const StepParams& p, long long src_off, float amp, const float* amp_dev,
              const int* step_dev, cudaStream_t s) override {
        const bool fc = fast_cpml(p);
        const int imode = fc && zmode_ != 0 ? kFull : kInnerOnly;
        // (the Z-slab planes read dpsi_z from pass 1: no overlap then)
        const bool ov = overlap_ && imode == kInnerOnly;
        static const int inner_late = [] {
            const char* e = std::getenv("MM_INNER_LATE");
            return e ? std::atoi(e) : 0;
        }();
        auto fork_inner = [&] {
            // the interior kernel needs no CPML state: it runs on a second
            // stream beside pass 1 -> boundary and takes SMs as their tails free
            // them (a second branch of the captured graph)
            MM_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
            launch_inner(p, 0, lay_.n[2], imode, side_);
            MM_CUDA(cudaEventRecord(join_, side_));
        };
        if (ov) MM_CUDA(cudaEventRecord(fork_, s));  // the step's start
        if (ov && inner_late == 0) fork_inner();
        dbg(s, "inner(side)", ov ? side_ : nullptr);
        launch_pass1(p, 0, lay_.n[2], s);
        dbg(s, "pass1", p1_side_);
        if (ov && inner_late == 1) fork_inner();  // (issue order only: still from the start)
        if (fc)
            launch_boundary(p, 0, lay_.n[2], s);
        else
            strict_update(p, 2, 0, lay_.n[2], s);
        dbg(s, "boundary", nullptr);
        if (ov && inner_late == 2) fork_inner();
        if (ov)
            MM_CUDA(cudaStreamWaitEvent(s, join_, 0));
        else
            launch_inner(p, 0, lay_.n[2], imode, s);
        dbg(s, "inner", nullptr);
        if (src_off >= 0) launch_inject(p.pn, p.cv, src_off, amp, amp_dev, step_dev, s);
    }
    // MM_DEBUG_SYNC=kernels: synchronize after each kernel of the step and name
    // the one that faulted (diagnostics only)
    void dbg(cudaStream_t s, const char* what, cudaStream_t s2) {
        static const bool on = [] {
            const char* e = std::getenv("MM_DEBUG_SYNC");
            return e && std::strcmp(e, "kernels") == 0;
        }();
        if (!on) return;
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

    void finish_work(Work& w, const std::vector<Item>& tiles, int ctas, double target) {
        std::vector<int4> items;
        wave_items(tiles, ctas, target, items);
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
        const int tiles_x = (inner.hi[0] - w.x_base + IC::TX - 1) / IC::TX;
        const int tiles_y = (inner.hi[1] - inner.lo[1] + IC::TY - 1) / IC::TY;
        std::vector<Item> tiles;
        for (const auto& r : zr)
            for (int ty = 0; ty < tiles_y; ++ty)
                for (int tx = 0; tx < tiles_x; ++tx) tiles.push_back(Item{tx, ty, r.first, r.second});
        finish_work(w, tiles, sms_ * inner_per_sm_, inner_zt_);
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
        // MM_BND_KINDS (profiling only): bit mask of the slab kinds to update
        static const int kinds = [] {
            const char* e = std::getenv("MM_BND_KINDS");
            return e ? std::atoi(e) : 7;
        }();
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
        finish_work(w, items, sms_ * bnd_per_sm_, bnd_zt_);
        return w;
    }

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
        if (mode != kInnerOnly || col_inner_) {  // column kernel (MM_ZSLABS = 1, 2; R > 4)
            if constexpr (kZs) {
                constexpr size_t zsm = ZSlabCfg<R>::SMEM;
                if (order_ == 2)
                    k_zslab<R, 2><<<w.ctas, IC::NT, zsm, s>>>(a, b, cv_in_, ip);
                else if (order_ == 1)
                    k_zslab<R, 1><<<w.ctas, IC::NT, zsm, s>>>(a, b, cv_in_, ip);
                else
                    k_zslab<R, 0><<<w.ctas, IC::NT, zsm, s>>>(a, b, cv_in_, ip);
            }
        } else if (order_ == 2) {
            k_inner<R, 2><<<w.ctas, IC::NT, IC::SMEM, s>>>(a, b, cv_in_, ip);
        } else if (order_ == 1) {
            k_inner<R, 1><<<w.ctas, IC::NT, IC::SMEM, s>>>(a, b, cv_in_, ip);
        } else {
            k_inner<R, 0><<<w.ctas, IC::NT, IC::SMEM, s>>>(a, b, cv_in_, ip);
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
                p1maps_.psi[a][sd] = run_map(lay_, r, a, r.psi, P1C::TX, P1C::TY);
            }
        runs_valid_ = true;
    }

    // fast CPML: k_p1 + k_bnd + the inner kernel's Z-slab planes
    bool fast_cpml(const StepParams& p) {
        if constexpr (!(kBnd && kP1))
            return false;
        else
            return ensure_dpz(p);
    }

    void launch_boundary(const StepParams& p, int z_lo, int z_hi, cudaStream_t s) {
        launch_boundary(p, ZRanges{{z_lo, z_hi}}, s);
    }
    void launch_boundary(const StepParams& p, const ZRanges& zr, cudaStream_t s) {
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
            // MM_BND_CTAS (diagnostics): cap the CTA count (more items per CTA)
            static const int cap = [] {
                const char* e = std::getenv("MM_BND_CTAS");
                return e ? std::max(1, std::atoi(e)) : 1 << 30;
            }();
            const int ctas = std::min(w.ctas, cap);
            if (order_ == 2)
                launch_pdl(k_bnd<R, 2>, ctas, BC::NT, BC::SMEM, s, pdl_, maps_, bp_);
            else
                launch_pdl(k_bnd<R, 1>, ctas, BC::NT, BC::SMEM, s, pdl_, maps_, bp_);
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
                // MM_P1_AXES (profiling only): bit mask of the run axes to update
                static const int axes = [] {
                    const char* e = std::getenv("MM_P1_AXES");
                    return e ? std::atoi(e) : 7;
                }();
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
                        const int tx = (d.hi[0] - d.x_base + P1C::TX - 1) / P1C::TX;
                        const int ty = (d.hi[1] - d.lo[1] + P1C::TY - 1) / P1C::TY;
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
                wave_items(tiles, sms_ * p1x_per_sm_, p1_zt_, items);
                e.nx = (int)items.size();
                e.ctas_x = std::max(1, std::min(sms_ * p1x_per_sm_, e.nx));
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
    int sms_ = 148, inner_per_sm_ = 1, bnd_per_sm_ = 1;
    int order_ = 2;
    double inner_zt_ = 48.0, bnd_zt_ = 48.0;
    int zmode_ = 0;
    bool pdl_ = true;
    bool overlap_ = false;
    cudaStream_t side_ = nullptr;
    cudaEvent_t fork_ = nullptr, join_ = nullptr;
    cudaStream_t p1_side_ = nullptr;
    cudaEvent_t p1_fork_ = nullptr, p1_join_ = nullptr;
    bool col_inner_ = false;
    const float* bufs_[3];
    CUtensorMap in_halo_[3], in_tile_[3], bd_halo_[3], bd_tile_[3], cv_in_, cv_bd_;
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
                                         const float* cv) {
    switch (lay.r) {
        case 2: return std::make_unique<FastPlanR<2>>(lay, device, bufs, cv);
        case 4: return std::make_unique<FastPlanR<4>>(lay, device, bufs, cv);
        case 8: return std::make_unique<FastPlanR<8>>(lay, device, bufs, cv);
        default: return nullptr;  // other radii run the strict kernels
    }
}

}  // namespace mmb
