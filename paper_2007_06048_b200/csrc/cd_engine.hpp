// cd_engine.hpp -- the acoustic_iso_cd engine object behind the C ABI
// (engine.cu) and the multi-GPU z-slab group (group.cu).
//
// Mirrors minimod::AcousticCdEngine<float> (propagator.hpp:93-140,
// propagator_impl.hpp:53-173): the constructor (mm_cd_create) does the same
// setup on the host (weights, CPML profile with the float-rounded dt,
// material taper, region partition), uploads the fields in the device layout
// of mm_internal.hpp and from then on every step runs on the GPU.  The three
// pressure buffers rotate by index exactly as the reference swaps
// p_prev/p_cur/p_next, so ghost contents (zero, free-surface mirror or halo
// planes) behave identically.
#pragma once

#include <cstring>
#include <memory>
#include <vector>

#include "../../include/minimod_b200.h"
#include "mm_fast.hpp"
#include "mm_internal.hpp"

// (internal header of the library: its two translation units work in mmb)
using namespace mmb;

struct mm_cd_engine {
    int device = 0;
    int mode = MM_MODE_FAST;
    cudaStream_t stream = nullptr;
    Layout lay;
    HostGrid hg;
    int goff[3], gn[3], nd[3];
    double d[3];
    bool free_surface = false;
    float dt = 0, dt2 = 0;
    Profile prof;
    float c2[3][kMaxR] = {};
    float c1[3][kMaxR] = {};
    DevBuf<float> p[3];
    int ip = 0, ic = 1, in = 2;  // prev / cur / next buffer indices
    DevBuf<float> cv, vp;
    // CPML
    DevBuf<float> ta[3], tb[3], tik[3];
    CpmlRun run[3][2] = {};
    DevBuf<float> psi[3][2], zeta[3][2];
    // receivers / driver
    std::vector<int> rec_ijk;
    DevBuf<long long> rec_offs;
    DevBuf<float> traces;
    int nrec = 0, cap = 0;
    DevBuf<int> counters;  // [0] step counter, [1] first bad step, [2] epilogue ticket
    TraceCopier tcopy;
    DevBuf<float> amps;
    long long steps = 0;
    std::unique_ptr<FastPlan> fast;
    // Host-driven steps (mm_cd_step) in fast mode: the step's kernels (pass 1,
    // boundary and interior over two streams) are captured once per buffer
    // rotation state as a CUDA graph and replayed -- one launch instead of
    // seven plus the cross-stream events; the injection (host amplitude) and
    // the free surface follow it on the stream.  Keyed by `ic`, recaptured when
    // (ip, in) differ from the capture or the CPML runs are rebuilt.
    struct StepGraph {
        cudaGraphExec_t exec = nullptr;
        int ip = -1, in = -1;
        long long launches = 0;
    } step_graph[3];
    bool fast_warm = false;  // one eager fast step ran (lazy work lists / dpsi_z built)
    void drop_step_graphs() {
        for (auto& g : step_graph) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            g = StepGraph{};
        }
    }
    // Per-step graphs (and mm_cd_run's rotation-period graph) only where
    // issuing the step's kernels one by one would bound the loop:
    // eager issue costs ~65 us of host time per step, a replay ~20 us, but at
    // 240^3 the eager step runs ~4 % faster on the device (147 vs 153 us,
    // tools/e2e_probe.py), so grids past ~6 M points (a ~90 us step) issue
    // eagerly.  MM_STEP_GRAPH=0/1 forces either.
    // ("step_graph" tuning forces either; kernel timing and debug
    // synchronisation need the eager path)
    bool step_graphs_enabled() const {
        if (fast && fast->timer.on) return false;
        if (tuning("debug_sync")) return false;
        const long long forced = tuning("step_graph");
        if (forced >= 0) return forced == 1;
        return (double)lay.n[0] * lay.n[1] * lay.n[2] < 6.0e6;
    }
    void graph_fast_step(const StepParams& sp) {
        StepGraph& g = step_graph[ic];
        if (g.exec && (g.ip != ip || g.in != in)) {
            cudaGraphExecDestroy(g.exec);
            g = StepGraph{};
        }
        if (!g.exec) {
            cudaGraph_t graph = nullptr;
            const long long l0 = launches_so_far();
            MM_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
            try {
                fast->step(sp, -1LL, 0.0f, nullptr, nullptr, stream);
            } catch (...) {
                cudaStreamEndCapture(stream, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            MM_CUDA(cudaStreamEndCapture(stream, &graph));
            g.launches = launches_so_far() - l0;
            const cudaError_t err = cudaGraphInstantiate(&g.exec, graph, 0);
            cudaGraphDestroy(graph);
            MM_CUDA(err);
            g.ip = ip;
            g.in = in;
            note_launches(-g.launches);  // counted per replay
        }
        MM_CUDA(cudaGraphLaunch(g.exec, stream));
        note_launches(g.launches);
    }

    StepParams params() const {
        StepParams s;
        std::memset(&s, 0, sizeof s);
        s.lay = lay;
        for (int a = 0; a < 3; ++a) {
            s.goff[a] = goff[a];
            s.gn[a] = gn[a];
            s.nd[a] = nd[a];
            s.ta[a] = ta[a].ptr;
            s.tb[a] = tb[a].ptr;
            s.tik[a] = tik[a].ptr;
            s.run[a][0] = run[a][0];
            s.run[a][1] = run[a][1];
            for (int m = 0; m < kMaxR; ++m) {
                s.c2[a][m] = c2[a][m];
                s.c1[a][m] = c1[a][m];
            }
        }
        s.pc = p[ic].ptr;
        s.pp = p[ip].ptr;
        s.pn = p[in].ptr;
        s.cv = cv.ptr;
        return s;
    }

    // Local tables + the CPML memory runs (one per damping layer and axis,
    // allocated only where some a != 0) from prof.
    void setup_cpml() {
        drop_step_graphs();  // captured with the previous runs' pointers
        fast_warm = false;
        const long long nx4 = (lay.n[0] + 3) / 4 * 4;
        for (int ax = 0; ax < 3; ++ax) {
            const int n = lay.n[ax];
            std::vector<float> a(n), b(n), k(n);
            for (int l = 0; l < n; ++l) {
                const int g = l + goff[ax];
                a[l] = prof.a[ax][g];
                b[l] = prof.b[ax][g];
                k[l] = prof.ik[ax][g];
            }
            ta[ax].upload(a.data(), n, stream);
            tb[ax].upload(b.data(), n, stream);
            tik[ax].upload(k.data(), n, stream);
            // global layers [0, nd) and [gn - nd, gn), clipped to the local box
            const int glo[2] = {0, gn[ax] - nd[ax]}, ghi[2] = {nd[ax], gn[ax]};
            for (int side = 0; side < 2; ++side) {
                CpmlRun& r = run[ax][side];
                r = CpmlRun{0, 0, 0, nullptr, nullptr, 0, 0};
                psi[ax][side].reset();
                zeta[ax][side].reset();
                const int lo = std::max(glo[side] - goff[ax], 0);
                const int hi = std::min(ghi[side] - goff[ax], n);
                bool active = false;
                for (int l = lo; l < hi; ++l) active |= a[l] != 0.0f;
                if (hi <= lo || !active) continue;
                const long long w = hi - lo;
                r.lo = lo;
                r.hi = hi;
                r.org = ax == 0 ? (lo & ~3) : lo;
                size_t count;
                if (ax == 0) {
                    // rows start 16-byte aligned in x and are at least as wide as
                    // the fast kernel's TMA boxes; padding columns stay zero (they
                    // are part of the zero halo)
                    r.s1 = std::max<long long>((hi - r.org + 3) / 4 * 4, 64);
                    r.s2 = r.s1 * lay.n[1];
                    count = (size_t)r.s2 * lay.n[2];
                } else if (ax == 1) {
                    r.s1 = nx4;
                    r.s2 = nx4 * w;
                    count = (size_t)r.s2 * lay.n[2];
                } else {
                    r.s1 = nx4;
                    r.s2 = nx4 * lay.n[1];
                    count = (size_t)r.s2 * w;
                }
                psi[ax][side].alloc_zero(count, stream);
                zeta[ax][side].alloc_zero(count, stream);
                r.psi = psi[ax][side].ptr;
                r.zeta = zeta[ax][side].ptr;
            }
        }
    }

    void rotate() {
        const int t = ip;
        ip = ic;
        ic = in;
        in = t;
    }

    long long src_off(const int* src) const {
        for (int a = 0; a < 3; ++a)
            if (src[a] < 0 || src[a] >= lay.n[a])
                raise(ST_CONFIG, "source location outside grid interior");
        return lay.off(src[0], src[1], src[2]);
    }

    void pass1() {
        const StepParams s = params();
        if (mode == MM_MODE_STRICT || !fast)
            strict_pass1(s, 0, lay.n[2], stream);
        else
            fast->pass1(s, stream);
    }
    void update(int region, int z_lo, int z_hi) {
        const StepParams s = params();
        if (mode == MM_MODE_STRICT || !fast)
            strict_update(s, region, z_lo, z_hi, stream);
        else
            fast->update(s, region, z_lo, z_hi, stream);
    }
    void update_ranges(const int* r, int n) {
        const StepParams s = params();
        if (mode == MM_MODE_STRICT || !fast) {
            for (int i = 0; i < n; ++i) strict_update(s, 0, r[2 * i], r[2 * i + 1], stream);
        } else {
            fast->update_ranges(s, r, n, stream);
        }
    }
    // The deferred epilogue of the last host-driven step (see full_step):
    // launched by the next API call on this engine (use() in engine.cu).
    Epilogue pending_ep;
    bool ep_pending = false;
    void flush_epilogue() {
        if (!ep_pending) return;
        ep_pending = false;
        launch_epilogue(pending_ep, stream);
    }

    // One step: the update kernels, then k_epilogue (injection, free surface
    // and -- from mm_cd_run -- the receiver sample and the step counter).
    void full_step(float amp, const int* src, const float* amp_dev, int* step_dev,
                   const RecParams* rec = nullptr, long long check_off = -1) {
        const StepParams sp = params();
        const long long so = src ? src_off(src) : -1LL;
        const bool fst = mode != MM_MODE_STRICT && fast;
        if (fst) {
            if (!amp_dev && !step_dev && fast_warm && step_graphs_enabled()) {
                graph_fast_step(sp);
            } else {
                fast->step(sp, -1LL, 0.0f, nullptr, nullptr, stream);
                fast_warm = true;
            }
        } else {
            pass1();
            update(0, 0, lay.n[2]);
        }
        const int te = fst ? fast->timer.begin("epilogue", stream) : -1;
        Epilogue ep;
        std::memset(&ep, 0, sizeof ep);
        ep.p = sp.pn;
        ep.cv = sp.cv;
        ep.src_off = so;
        ep.amp = amp;
        ep.amp_dev = amp_dev;
        ep.step_dev = step_dev;
        ep.count = step_dev != nullptr;
        ep.fs = free_surface && goff[2] == 0;
        ep.lay = lay;
        if (rec) ep.rec = *rec;
        ep.check_off = check_off;
        ep.done = counters.ptr + 2;
        ep.pdl = fst && tuning("epi_pdl") != 0;
        // a host-driven step's epilogue waits for the next API call: when that
        // is mm_cd_record (the reference's step-then-record loop) the receiver
        // sample rides in the epilogue instead of a second launch
        if (te < 0 && !amp_dev && !step_dev && !rec && check_off < 0 &&
            tuning("defer_epilogue") != 0) {
            pending_ep = ep;
            ep_pending = true;
        } else {
            launch_epilogue(ep, stream);
        }
        if (te >= 0) fast->timer.end(te, stream);
        rotate();
        ++steps;
        debug_sync(fst ? "fast" : "strict");
    }
    // tuning "debug_sync" != 0: synchronize after every step and name the
    // engine whose step faulted (diagnostics only)
    void debug_sync(const char* what) {
        if (!tuning("debug_sync")) return;
        const cudaError_t e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess)
            raise(ST_CUDA, std::string("fault in ") + what + " step " + std::to_string(steps) +
                               ": " + cudaGetErrorString(e));
    }

    // host <-> device layout transposes go through one engine-lifetime
    // staging buffer (allocated on first use), so pressure() costs a transpose
    // and a copy, not an allocation
    DevBuf<float> stage;
    void to_host(const float* dev, float* host) {
        if (stage.count < hg.volume()) stage.alloc(hg.volume());
        launch_to_host_layout(dev, stage.ptr, lay, stream);
        MM_CUDA(cudaMemcpyAsync(host, stage.ptr, hg.volume() * sizeof(float),
                                cudaMemcpyDeviceToHost, stream));
        MM_CUDA(cudaStreamSynchronize(stream));
    }
    void from_host(const float* host, float* dev) {
        stage.upload(host, hg.volume(), stream);
        launch_to_device_layout(stage.ptr, dev, lay, stream);
        MM_CUDA(cudaStreamSynchronize(stream));
    }

    ~mm_cd_engine() {
        if (stream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
        }
        drop_step_graphs();
        fast.reset();
        if (stream) cudaStreamDestroy(stream);
    }
};

