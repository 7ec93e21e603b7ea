// engine.cu -- the AcousticCdEngine drop-in behind the C ABI (include/minimod_b200.h).
//
// Mirrors minimod::AcousticCdEngine<float> (propagator.hpp:93-140,
// propagator_impl.hpp:53-173): the constructor does the same setup on the
// host (weights, CPML profile with the float-rounded dt, material taper,
// region partition), uploads the fields in the device layout of
// mm_internal.hpp and from then on every step runs on the GPU.  The three
// pressure buffers rotate by index exactly as the reference swaps
// p_prev/p_cur/p_next, so ghost contents (zero, free-surface mirror or halo
// planes) behave identically.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/minimod_b200.h"
#include "cd_engine.hpp"
#include "mm_fast.hpp"
#include "mm_internal.hpp"

namespace mmb {

namespace {
thread_local std::string g_err;
thread_local int g_step = 0;
std::atomic<long long> g_launches{0};

// Tuning parameters: name, product default, meaning.  Changed only through
// mm_set_tuning (no environment reads in the library).
struct Tunable {
    const char* name;
    long long def;
};
const Tunable kTunables[] = {
    {"step_graph", -1},  // host-driven steps as CUDA graphs: -1 auto (grids < 6 M points), 0 off, 1 on
    {"cpml_fused", 0},   // fast mode: one-pass CPML kernel k_cpml where the layout allows it (0: k_p1 + k_bnd)
    {"cpml_zt", 0},      // k_cpml planes per work item (0: automatic)
    {"overlap", 1},      // interior kernel on a side stream beside the CPML kernels
    {"pdl", -1},         // programmatic launch of k_bnd after k_p1: -1 auto (grids < 6 M points), 0 off, 1 on
                         // (on big grids its early CTAs race the interior kernel for SMs while
                         // pass 1 drains: 145-158 us/step at 240^3 by engine, 145 without)
    {"epi_pdl", 0},      // (experiment) programmatic launch of the step epilogue behind the boundary kernel
    {"inner_late", 1},   // issue the interior kernel before pass 1 (0), after it (1) or after the boundary (2)
    {"main_prio", 2},    // pass 1 -> boundary streams above the interior kernel's: 0 none, 1 the step's
                         // stream, 2 both pass-1 streams (the CPML chain wins every race for SMs)
    {"debug_sync", 0},   // (diagnostics) synchronize after every kernel (1) or every step (2)
    {"l2_promo", 2},     // TMA L2 promotion: 0 none, 1 64 B, 2 128 B, 3 256 B
    {"inner_zt", 48},    // k_inner planes per work item (target)
    {"inner_ctas", 0},   // cap on the interior kernel's CTAs beside the CPML kernels (0: every slot)
    {"bnd_zt", 12},      // k_bnd planes per work item (target)
    {"bnd_tail", 15},    // the last % of the boundary queue in half-length items: CTAs that finish
                         // early take the small ones (240^3: 141-144.5 -> 136.1 us/step; a per-CTA
                         // globaltimer trace showed k_bnd CTAs ending from 56 to 80+ us)
    {"smem_carveout", -1},   // (experiment) L1 / shared split (percent shared) of every step kernel;
                             // -1 driver default (100: same step time, pass 1's kernels reordered)
    {"p1x_ctas", 0},     // (experiment) pass-1 x/y CTAs per SM (0: as many as fit; 2-3 let the z
                         // and x/y launches start together, but x/y then runs longer: no gain)
    {"bnd_whole", -1},   // k_bnd tiles of at most this many planes (the Z slabs) as one item, queued
                         // first: -1 auto (64 on grids over 30 M points, else 0)
    {"p1_zt", 16},       // k_p1 planes per work item (target)
    {"field_stagger", 1024},  // pressure / c field k starts k x this many floats into its allocation
                            // (240^3: the fast step mode in 6 of 7 engines vs 2-3 of 7 unstaggered)
    {"defer_epilogue", 1},  // host-driven steps: epilogue launched by the next call (fuses record)
    {"even_chunks", 5},  // equal-length z chunks per tile (bit mask: 1 interior, 2 boundary, 4 pass-1 x/y;
                         // 240^3: 143.6 with 5, 145.0 with 0, boundary chunks 146.5)
    {"zslabs", -1},      // Z slabs: -1 auto, 0 k_bnd tiles, 1 k_zslab after k_inner, 2 k_zslab columns
    {"wide_inner", -1},  // r > 4 interior: -1 auto (2), 0 column kernel k_zslab, 1 unrolled k_inner, 2 k_innerw
    {"bnd_kinds", 7},    // (profiling) slab kinds k_bnd updates (bit mask X/Y/Z)
    {"bnd_ctas", 0},     // (diagnostics) cap on k_bnd CTAs (0: none)
    {"p1_axes", 7},      // (profiling) run axes k_p1 updates (bit mask)
    {"vd_zchunks", 0},   // acoustic_iso: z chunks per tile column (0: automatic)
    {"vd_ctas", 0},      // acoustic_iso (diagnostics): cap on CTAs (0: none)
    {"vd_zc", 0},        // acoustic_iso: simple-kernel z chunk (0: default)
    {"vd_simple", 0},    // acoustic_iso: one-thread-per-point kernels instead of the TMA kernels
};
std::mutex g_tun_mu;
std::map<std::string, long long> g_tun;

const Tunable* find_tunable(const char* name) {
    if (!name) return nullptr;
    for (const auto& t : kTunables)
        if (std::strcmp(t.name, name) == 0) return &t;
    return nullptr;
}
}  // namespace

long long tuning(const char* name) {
    const Tunable* t = find_tunable(name);
    if (!t) raise(ST_INVAL, std::string("unknown tuning parameter ") + (name ? name : "(null)"));
    std::lock_guard<std::mutex> lk(g_tun_mu);
    const auto it = g_tun.find(t->name);
    return it == g_tun.end() ? t->def : it->second;
}

// ---- KernelTimer
cudaEvent_t KernelTimer::get() {
    if (!pool_.empty()) {
        cudaEvent_t e = pool_.back();
        pool_.pop_back();
        return e;
    }
    cudaEvent_t e;
    MM_CUDA(cudaEventCreate(&e));
    return e;
}
int KernelTimer::begin(const char* name, cudaStream_t s) {
    if (!on) return -1;
    Rec r{name, get(), get()};
    MM_CUDA(cudaEventRecord(r.a, s));
    pending_.push_back(r);
    return (int)pending_.size() - 1;
}
void KernelTimer::end(int idx, cudaStream_t s) {
    if (idx < 0) return;
    MM_CUDA(cudaEventRecord(pending_[idx].b, s));
}
void KernelTimer::collect() {
    for (auto& r : pending_) {
        MM_CUDA(cudaEventSynchronize(r.b));
        float ms = 0;
        MM_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        auto& a = acc[r.name];
        a.first += ms;
        a.second += 1;
        pool_.push_back(r.a);
        pool_.push_back(r.b);
    }
    pending_.clear();
}
void KernelTimer::reset() {
    collect();
    acc.clear();
}
KernelTimer::~KernelTimer() {
    for (auto& r : pending_) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : pool_) cudaEventDestroy(e);
}

void note_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launches_so_far() { return g_launches.load(); }

int set_api_error(int code, const std::string& msg, int step) {
    g_err = msg;
    g_step = step;
    return code;
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw Error(ST_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what +
                               " (" + file + ":" + std::to_string(line) + ")");
}

Layout Layout::make(const int n[3], int r) {
    Layout l;
    for (int a = 0; a < 3; ++a) l.n[a] = n[a];
    l.r = r;
    l.L = (r + 3) / 4 * 4;
    l.P = (l.L + n[0] + r + 31) / 32 * 32;
    l.ey = n[1] + 2 * r;
    l.ez = n[2] + 2 * r;
    l.plane = (long long)l.ey * l.P;
    l.total = l.plane * l.ez;
    return l;
}

}  // namespace mmb

using namespace mmb;

namespace {

void use(mm_cd_engine* e, bool flush = true) {
    need(e, "engine");
    MM_CUDA(cudaSetDevice(e->device));
    if (flush) e->flush_epilogue();  // a host-driven step's deferred epilogue
}

}  // namespace

extern "C" {

const char* mm_last_error(void) { return g_err.c_str(); }

int mm_set_tuning(const char* name, long long value) {
    MM_API_BEGIN
    const Tunable* t = find_tunable(name);
    if (!t) raise(ST_INVAL, std::string("unknown tuning parameter ") + (name ? name : "(null)"));
    std::lock_guard<std::mutex> lk(g_tun_mu);
    g_tun[t->name] = value;
    MM_API_END
}

int mm_reset_tuning(void) {
    MM_API_BEGIN
    std::lock_guard<std::mutex> lk(g_tun_mu);
    g_tun.clear();
    MM_API_END
}

int mm_get_tuning(const char* name, long long* value) {
    MM_API_BEGIN
    need(value, "value");
    *value = tuning(name);
    MM_API_END
}
int mm_last_instability_step(void) { return g_step; }
const char* mm_version(void) { return "minimod-b200 0.1 (sm_100a)"; }
long long mm_kernel_launch_count(void) { return g_launches.load(); }

int mm_device_count(int* count) {
    MM_API_BEGIN
    need(count, "count");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *count = c;
    MM_API_END
}

int mm_second_derivative_coeffs(int radius, double h, double* c, double* center) {
    MM_API_BEGIN
    need(c, "c");
    const Coeffs k = second_derivative(radius, h);
    for (int m = 0; m < radius; ++m) c[m] = k.c[m];
    if (center) *center = k.center;
    MM_API_END
}

int mm_central_first_derivative_coeffs(int radius, double h, double* c) {
    MM_API_BEGIN
    need(c, "c");
    const Coeffs k = central_first_derivative(radius, h);
    for (int m = 0; m < radius; ++m) c[m] = k.c[m];
    MM_API_END
}

int mm_cfl_dt(double vmax, const mm_grid* grid, double cfl, double* dt) {
    MM_API_BEGIN
    need(grid, "grid");
    need(dt, "dt");
    *dt = cfl_dt(vmax, grid->n, grid->d, grid->radius, cfl);
    MM_API_END
}

int mm_ricker(double fmax, double dt, int nsteps, float* out) {
    MM_API_BEGIN
    const std::vector<float> w = ricker(fmax, dt, nsteps);
    if (nsteps > 0) {
        need(out, "out");
        std::memcpy(out, w.data(), sizeof(float) * w.size());
    }
    MM_API_END
}

int mm_build_profile(const int n[3], const double h[3], const int nd[3], double fmax, double vmax,
                     double dt, double r_target, int free_surface, float* a, float* b,
                     float* inv_kappa, double* d0) {
    MM_API_BEGIN
    need(n, "n");
    need(h, "h");
    need(nd, "ndamping");
    const Profile p = build_profile(n, h, nd, fmax, vmax, dt, r_target, free_surface != 0);
    size_t o = 0;
    for (int ax = 0; ax < 3; ++ax) {
        if (a) std::memcpy(a + o, p.a[ax].data(), sizeof(float) * n[ax]);
        if (b) std::memcpy(b + o, p.b[ax].data(), sizeof(float) * n[ax]);
        if (inv_kappa) std::memcpy(inv_kappa + o, p.ik[ax].data(), sizeof(float) * n[ax]);
        if (d0) d0[ax] = p.d0[ax];
        o += n[ax];
    }
    MM_API_END
}

int mm_taper_material(float* f, const int n[3], int radius, const int ntaper[3],
                      const int offset[3], const int global_n[3]) {
    MM_API_BEGIN
    need(f, "f");
    const HostGrid g{{n[0], n[1], n[2]}, radius};
    taper_material(f, g, ntaper, offset, global_n);
    MM_API_END
}

int mm_layered_model(const int n[3], int radius, float* vp, float* vmin, float* vmax) {
    MM_API_BEGIN
    need(vp, "vp");
    const HostGrid g{{n[0], n[1], n[2]}, radius};
    std::fill(vp, vp + g.volume(), 0.0f);
    const int half = n[2] / 2;
    for (int i = 0; i < n[0]; ++i)
        for (int j = 0; j < n[1]; ++j)
            for (int k = 0; k < n[2]; ++k) vp[g.off(i, j, k)] = k < half ? 1500.0f : 4500.0f;
    validate_vp(vp, g, vmin, vmax);
    fill_ghosts_replicate(vp, g);
    MM_API_END
}

int mm_validate_model(const int n[3], int radius, float* vp, float* vmin, float* vmax) {
    MM_API_BEGIN
    need(vp, "vp");
    const HostGrid g{{n[0], n[1], n[2]}, radius};
    validate_vp(vp, g, vmin, vmax);
    fill_ghosts_replicate(vp, g);
    MM_API_END
}

int mm_cd_create(const mm_grid* local, const int offset[3], const int global_n[3],
                 const float* vp_local, const mm_engine_options* opts, float dt,
                 double vmax_global, int device, int mode, mm_cd_engine** out) {
    MM_API_BEGIN
    need(local, "grid");
    need(offset, "offset");
    need(global_n, "global_n");
    need(vp_local, "vp_local");
    need(opts, "options");
    need(out, "out");
    *out = nullptr;
    // make_grid validation (grid.cpp:5-22)
    static const char* axn[3] = {"x", "y", "z"};
    for (int a = 0; a < 3; ++a) {
        if (local->n[a] < 1)
            raise(ST_CONFIG, std::string("grid size must be >= 1 along ") + axn[a] + ", got " +
                               std::to_string(local->n[a]));
        if (!(local->d[a] > 0.0))
            raise(ST_CONFIG, std::string("grid spacing must be > 0 along ") + axn[a]);
    }
    if (local->radius < 1 || local->radius > kMaxR)
        raise(ST_CONFIG, "stencil radius must be in [1, 8], got " + std::to_string(local->radius));
    if (mode != MM_MODE_FAST && mode != MM_MODE_STRICT && mode != MM_MODE_FAST_FMA)
        raise(ST_INVAL, "unknown mode");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        raise(ST_CUDA, "no CUDA device available: the acoustic_iso_cd engine runs on the GPU only");
    }
    if (device < 0 || device >= ndev) raise(ST_INVAL, "device ordinal out of range");
    MM_CUDA(cudaSetDevice(device));

    auto e = std::make_unique<mm_cd_engine>();
    e->device = device;
    e->mode = mode;
    // tuning "main_prio": the step's stream (pass 1 -> boundary, the critical
    // path) at the greatest priority, above the interior kernel's side stream
    if (tuning("main_prio") > 0) {
        int lo = 0, hi = 0;
        MM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        MM_CUDA(cudaStreamCreateWithPriority(&e->stream, cudaStreamNonBlocking, hi));
    } else {
        MM_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    }
    e->lay = Layout::make(local->n, local->radius);
    e->hg = HostGrid{{local->n[0], local->n[1], local->n[2]}, local->radius};
    for (int a = 0; a < 3; ++a) {
        e->goff[a] = offset[a];
        e->gn[a] = global_n[a];
        e->nd[a] = opts->ndamping[a];
        e->d[a] = local->d[a];
        if (offset[a] < 0 || offset[a] + local->n[a] > global_n[a])
            raise(ST_CONFIG, "local box does not fit inside the global grid");
    }
    e->free_surface = opts->free_surface != 0;
    e->dt = dt;
    e->dt2 = dt * dt;
    const int r = local->radius;
    // weights (propagator_impl.hpp:67-70)
    for (int ax = 0; ax < 3; ++ax) {
        const Coeffs w2 = second_derivative(r, local->d[ax]);
        const Coeffs w1 = central_first_derivative(r, local->d[ax]);
        for (int m = 0; m < r; ++m) {
            e->c2[ax][m] = static_cast<float>(w2.c[m]);
            e->c1[ax][m] = static_cast<float>(w1.c[m]);
        }
    }
    // CPML profile with the float-rounded dt (propagator_impl.hpp:71-72)
    e->prof = build_profile(global_n, local->d, opts->ndamping, opts->fmax, vmax_global,
                            static_cast<double>(dt), opts->r_target, e->free_surface);
    // taper on the engine's own vp copy (propagator_impl.hpp:73)
    std::vector<float> vp(vp_local, vp_local + e->hg.volume());
    if (opts->taper) taper_material(vp.data(), e->hg, opts->ntaper, offset, global_n);
    // region partition checks (grid.cpp:24-33)
    for (int a = 0; a < 3; ++a) {
        if (opts->ndamping[a] < 0) raise(ST_CONFIG, "ndamping must be >= 0");
        if (2 * opts->ndamping[a] >= global_n[a])
            raise(ST_CONFIG, std::string("damping layers too thick along ") + axn[a] + ": 2*" +
                               std::to_string(opts->ndamping[a]) +
                               " >= " + std::to_string(global_n[a]));
    }
    // device fields
    const Layout& L = e->lay;
    // tuning field_stagger: field k starts k x stagger floats into its
    // allocation (multiples of 32: rows stay 128-byte aligned), so the same
    // point of p_prev, p_cur, p_next and c -- streamed side by side by every
    // kernel -- does not sit at the same offset of identically aligned
    // allocations (the step was 141 or 144.5 us at 240^3 by engine: unstaggered
    // 2-3 of 7 engines fast, staggered by 1024 floats 6 of 7)
    const size_t stag = (size_t)std::max(0LL, tuning("field_stagger")) / 32 * 32;
    for (int b = 0; b < 3; ++b) e->p[b].alloc_zero(L.total, e->stream, stag * (size_t)b);
    e->vp.alloc_zero(L.total, e->stream, stag * 3);
    e->cv.alloc_zero(L.total, e->stream, stag * 4);
    e->from_host(vp.data(), e->vp.ptr);
    launch_velocity_coeff(e->vp.ptr, e->cv.ptr, e->dt2, L.total, e->stream);
    e->setup_cpml();
    e->counters.alloc_zero(3, e->stream);  // + the epilogue's block ticket
    if (mode != MM_MODE_STRICT) {
        float* const bufs[3] = {e->p[0].ptr, e->p[1].ptr, e->p[2].ptr};
        // MM_MODE_FAST: reference order, every operation rounded (bit-exact);
        // MM_MODE_FAST_FMA: reference order with FMA contraction
        e->fast = make_fast_plan(e->lay, device, bufs, e->cv.ptr, mode == MM_MODE_FAST ? 2 : 1);
    }
    MM_CUDA(cudaStreamSynchronize(e->stream));
    *out = e.release();
    MM_API_END
}

int mm_cd_destroy(mm_cd_engine* e) {
    MM_API_BEGIN
    if (!e) return MM_OK;
    cudaSetDevice(e->device);
    delete e;
    MM_API_END
}

int mm_cd_step(mm_cd_engine* e, float amp, const int* src) {
    MM_API_BEGIN
    use(e);
    e->full_step(amp, src, nullptr, nullptr);
    MM_API_END
}

int mm_cd_update_boundary_psi(mm_cd_engine* e) {
    MM_API_BEGIN
    use(e);
    e->pass1();
    MM_API_END
}

int mm_cd_update_inner(mm_cd_engine* e) {
    MM_API_BEGIN
    use(e);
    e->update(1, 0, e->lay.n[2]);
    MM_API_END
}

int mm_cd_update_boundary(mm_cd_engine* e) {
    MM_API_BEGIN
    use(e);
    e->update(2, 0, e->lay.n[2]);
    MM_API_END
}

int mm_cd_update_planes(mm_cd_engine* e, int z_lo, int z_hi) {
    MM_API_BEGIN
    use(e);
    if (z_lo < 0 || z_hi > e->lay.n[2] || z_lo > z_hi) raise(ST_INVAL, "plane range out of bounds");
    e->update(0, z_lo, z_hi);
    MM_API_END
}

int mm_cd_update_plane_ranges(mm_cd_engine* e, const int* ranges, int n) {
    MM_API_BEGIN
    use(e);
    if (n < 0 || (n > 0 && !ranges)) raise(ST_INVAL, "plane ranges");
    for (int i = 0; i < n; ++i)
        if (ranges[2 * i] < 0 || ranges[2 * i + 1] > e->lay.n[2] || ranges[2 * i] > ranges[2 * i + 1])
            raise(ST_INVAL, "plane range out of bounds");
    e->update_ranges(ranges, n);
    MM_API_END
}

int mm_cd_inject_source(mm_cd_engine* e, float amp, const int* src) {
    MM_API_BEGIN
    use(e);
    if (src) launch_inject(e->p[e->in].ptr, e->cv.ptr, e->src_off(src), amp, nullptr, nullptr,
                           e->stream);
    MM_API_END
}

int mm_cd_apply_free_surface(mm_cd_engine* e) {
    MM_API_BEGIN
    use(e);
    if (e->free_surface && e->goff[2] == 0) launch_free_surface(e->p[e->in].ptr, e->lay, e->stream);
    MM_API_END
}

int mm_cd_rotate(mm_cd_engine* e) {
    MM_API_BEGIN
    use(e);
    e->rotate();
    ++e->steps;
    MM_API_END
}

int mm_cd_synchronize(mm_cd_engine* e) {
    MM_API_BEGIN
    use(e);
    MM_CUDA(cudaStreamSynchronize(e->stream));
    e->tcopy.sync();
    MM_API_END
}

int mm_cd_field_size(mm_cd_engine* e, size_t* count) {
    MM_API_BEGIN
    need(e, "engine");
    need(count, "count");
    *count = e->hg.volume();
    MM_API_END
}

int mm_cd_get_dt(mm_cd_engine* e, float* dt) {
    MM_API_BEGIN
    need(e, "engine");
    need(dt, "dt");
    *dt = e->dt;
    MM_API_END
}

int mm_cd_get_mode(mm_cd_engine* e, int* mode) {
    MM_API_BEGIN
    need(e, "engine");
    need(mode, "mode");
    *mode = e->mode;
    MM_API_END
}

int mm_cd_steps_taken(mm_cd_engine* e, long long* steps) {
    MM_API_BEGIN
    need(e, "engine");
    need(steps, "steps");
    *steps = e->steps;
    MM_API_END
}

int mm_cd_get_pressure(mm_cd_engine* e, float* host) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    e->to_host(e->p[e->ic].ptr, host);
    MM_API_END
}

int mm_cd_get_pressure_prev(mm_cd_engine* e, float* host) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    e->to_host(e->p[e->ip].ptr, host);
    MM_API_END
}

int mm_cd_get_velocity(mm_cd_engine* e, float* host) {
    MM_API_BEGIN
    use(e);
    need(host, "host");
    e->to_host(e->vp.ptr, host);
    MM_API_END
}

int mm_cd_set_state(mm_cd_engine* e, const float* p_prev, const float* p_cur) {
    MM_API_BEGIN
    use(e);
    need(p_prev, "p_prev");
    need(p_cur, "p_cur");
    e->from_host(p_prev, e->p[e->ip].ptr);
    e->from_host(p_cur, e->p[e->ic].ptr);
    MM_API_END
}

int mm_cd_get_profile(mm_cd_engine* e, int axis, float* a, float* b, float* inv_kappa) {
    MM_API_BEGIN
    need(e, "engine");
    if (axis < 0 || axis > 2) raise(ST_INVAL, "axis must be 0, 1 or 2");
    const size_t n = e->prof.a[axis].size();
    if (a) std::memcpy(a, e->prof.a[axis].data(), n * sizeof(float));
    if (b) std::memcpy(b, e->prof.b[axis].data(), n * sizeof(float));
    if (inv_kappa) std::memcpy(inv_kappa, e->prof.ik[axis].data(), n * sizeof(float));
    MM_API_END
}

int mm_cd_set_profile(mm_cd_engine* e, int axis, const float* a, const float* b,
                      const float* inv_kappa) {
    MM_API_BEGIN
    use(e);
    if (axis < 0 || axis > 2) raise(ST_INVAL, "axis must be 0, 1 or 2");
    if (e->steps > 0)
        raise(ST_INVAL, "the CPML profile can only be replaced before the first step");
    const int n = e->gn[axis], nd = e->nd[axis];
    if (a)
        for (int g = nd; g < n - nd; ++g)
            if (a[g] != 0.0f)
                raise(ST_INVAL, "CPML coefficient a must be zero outside the damping layers");
    if (a) std::memcpy(e->prof.a[axis].data(), a, n * sizeof(float));
    if (b) std::memcpy(e->prof.b[axis].data(), b, n * sizeof(float));
    if (inv_kappa) std::memcpy(e->prof.ik[axis].data(), inv_kappa, n * sizeof(float));
    MM_CUDA(cudaStreamSynchronize(e->stream));
    e->setup_cpml();
    MM_CUDA(cudaStreamSynchronize(e->stream));
    MM_API_END
}

int mm_cd_get_d0(mm_cd_engine* e, double d0[3]) {
    MM_API_BEGIN
    need(e, "engine");
    need(d0, "d0");
    for (int a = 0; a < 3; ++a) d0[a] = e->prof.d0[a];
    MM_API_END
}

int mm_cd_set_receivers(mm_cd_engine* e, const int* ijk, int nreceivers, int capacity) {
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

int mm_cd_record(mm_cd_engine* e, int step) {
    MM_API_BEGIN
    use(e, false);
    if (step < 0 || step >= e->cap) raise(ST_INVAL, "record step outside the trace capacity");
    RecParams rp{e->p[e->ic].ptr, e->rec_offs.ptr, e->traces.ptr, e->nrec, step, nullptr};
    if (e->ep_pending && e->pending_ep.p == rp.p) {
        // right after a host-driven step: the sample rides in its epilogue
        // (the values it reads are the ones the epilogue leaves: injection and
        // free surface applied)
        e->pending_ep.rec = rp;
        e->flush_epilogue();
    } else {
        e->flush_epilogue();
        launch_record(rp, nullptr, e->stream);
    }
    MM_API_END
}

int mm_cd_get_traces(mm_cd_engine* e, float* host, int nsteps) {
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

int mm_cd_copy_trace_step(mm_cd_engine* e, int step, float* host, int async) {
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

int mm_cd_run(mm_cd_engine* e, const float* amps, int nsteps, const int* src, int record,
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
    // events, graph and exec are released on every exit path; a throw while
    // capturing ends the capture so the engine stream stays usable
    struct Res {
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        ~Res() {
            if (ge) cudaGraphExecDestroy(ge);
            if (g) cudaGraphDestroy(g);
            if (t0) cudaEventDestroy(t0);
            if (t1) cudaEventDestroy(t1);
        }
    } res;
    MM_CUDA(cudaEventCreate(&res.t0));
    MM_CUDA(cudaEventCreate(&res.t1));
    MM_CUDA(cudaEventRecord(res.t0, e->stream));
    // per-step finiteness check (ref: driver.cpp:68-71,108): receiver 0 when
    // recording; without recording the same check on receiver 0 (or the source)
    const bool rec_on = record && e->nrec > 0;
    long long check = -1;
    if (!rec_on) {
        if (e->nrec > 0)
            check = e->lay.off(e->rec_ijk[0], e->rec_ijk[1], e->rec_ijk[2]);
        else if (src)
            check = e->src_off(src);
    }
    auto one_step = [&] {
        const RecParams rp{nullptr, e->rec_offs.ptr,
                           e->traces.ptr + (size_t)first_sample * e->nrec, rec_on ? e->nrec : 0, 0,
                           bad};
        e->full_step(0.0f, src, e->amps.ptr, step_dev, &rp, check);
    };
    // The first step runs eagerly (it also builds the lazily created work
    // lists); then the buffer rotation's period of three steps is captured
    // once as a CUDA graph and replayed -- every per-step value (wavelet
    // sample, trace column) is read through the device step counter.
    int s = 0;
    if (nsteps > 0) {
        one_step();
        ++s;
    }
    // (large grids issue eagerly: the host stays ahead, and the eager step is
    // the faster one on the device -- see step_graphs_enabled)
    const bool use_graph = nsteps - s >= 6 && e->step_graphs_enabled();
    if (use_graph) {
        const long long l0 = g_launches.load();
        MM_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        try {
            for (int k = 0; k < 3; ++k) one_step();  // rotation period: host state returns
        } catch (...) {
            cudaStreamEndCapture(e->stream, &res.g);
            throw;
        }
        MM_CUDA(cudaStreamEndCapture(e->stream, &res.g));
        const long long per_graph = g_launches.load() - l0;  // kernels in the graph
        MM_CUDA(cudaGraphInstantiate(&res.ge, res.g, 0));
        const int reps = (nsteps - s) / 3;
        for (int k = 0; k < reps; ++k) MM_CUDA(cudaGraphLaunch(res.ge, e->stream));
        e->steps += 3LL * reps - 3;  // capture advanced the host counter by 3
        s += 3 * reps;
        note_launches(per_graph * (reps - 1));  // kernels executed by the replays
    }
    for (; s < nsteps; ++s) one_step();
    MM_CUDA(cudaEventRecord(res.t1, e->stream));
    MM_CUDA(cudaEventSynchronize(res.t1));
    float ms = 0;
    MM_CUDA(cudaEventElapsedTime(&ms, res.t0, res.t1));
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

int mm_cd_cpml_path(mm_cd_engine* e, char* buf, int cap) {
    MM_API_BEGIN
    use(e);
    need(buf, "buf");
    if (cap < 1) raise(ST_INVAL, "cap must be >= 1");
    const char* v = (e->mode == MM_MODE_STRICT || !e->fast) ? "strict" : e->fast->cpml_path(e->params());
    std::strncpy(buf, v, cap - 1);
    buf[cap - 1] = 0;
    MM_API_END
}

int mm_cd_kernel_timing(mm_cd_engine* e, int on) {
    MM_API_BEGIN
    use(e);
    if (!e->fast) raise(ST_INVAL, "kernel timing needs a fast-mode engine");
    MM_CUDA(cudaStreamSynchronize(e->stream));
    e->fast->timer.reset();
    e->fast->timer.on = on != 0;
    MM_API_END
}

int mm_cd_kernel_times(mm_cd_engine* e, int cap, char (*names)[32], double* total_ms,
                       long long* launches, int* n) {
    MM_API_BEGIN
    use(e);
    need(n, "n");
    *n = 0;
    if (!e->fast) return MM_OK;
    e->fast->timer.collect();
    int i = 0;
    for (const auto& kv : e->fast->timer.acc) {
        if (i < cap) {
            if (names) {
                std::strncpy(names[i], kv.first.c_str(), 31);
                names[i][31] = 0;
            }
            if (total_ms) total_ms[i] = kv.second.first;
            if (launches) launches[i] = kv.second.second;
        }
        ++i;
    }
    *n = i;
    MM_API_END
}

int mm_cd_stream(mm_cd_engine* e, void** stream) {
    MM_API_BEGIN
    need(e, "engine");
    need(stream, "stream");
    *stream = (void*)e->stream;
    MM_API_END
}

static void halo_range(mm_cd_engine* e, int buf, int side, int which, void** ptr, size_t* bytes) {
    need(ptr, "dev_ptr");
    need(bytes, "bytes");
    if (side < 0 || side > 1 || which < 0 || which > 1) raise(ST_INVAL, "side/which must be 0 or 1");
    const Layout& L = e->lay;
    const int nz = L.n[2], r = L.r;
    if (nz < r) raise(ST_INVAL, "slab thinner than the stencil radius");
    // plane index in [0, ez): ghost low [0,r), owned low [r,2r),
    // owned high [nz, nz+r), ghost high [nz+r, nz+2r)
    long long first;
    if (side == 0)
        first = which == 0 ? r : 0;
    else
        first = which == 0 ? nz : nz + r;
    *ptr = (void*)(e->p[buf].ptr + first * L.plane);
    *bytes = (size_t)r * L.plane * sizeof(float);
}

int mm_cd_halo_planes(mm_cd_engine* e, int side, int which, void** dev_ptr, size_t* bytes) {
    MM_API_BEGIN
    need(e, "engine");
    halo_range(e, e->ic, side, which, dev_ptr, bytes);
    MM_API_END
}

int mm_cd_next_halo_planes(mm_cd_engine* e, int side, int which, void** dev_ptr, size_t* bytes) {
    MM_API_BEGIN
    need(e, "engine");
    halo_range(e, e->in, side, which, dev_ptr, bytes);
    MM_API_END
}

int mm_sim_config_default(mm_sim_config* c) {
    MM_API_BEGIN
    need(c, "cfg");
    std::memset(c, 0, sizeof *c);
    for (int a = 0; a < 3; ++a) {
        c->ngrid[a] = 100;
        c->dgrid[a] = 20.0;
        c->ndamping[a] = 27;
        c->ntaper[a] = 3;
    }
    c->nsteps = 1000;
    c->fmax = 25.0;
    c->cfl = 0.8;
    c->taper = 1;
    c->free_surface = 0;
    c->r_target = 1e-3;
    c->has_source_loc = 0;
    c->receiver_increment[0] = c->receiver_increment[1] = 1;
    c->stencil_radius = 4;
    MM_API_END
}

int mm_run(const mm_sim_config* c, const float* vp_model, int device, int mode, float* traces,
           mm_run_report* rep) {
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
    const HostGrid g{{c->ngrid[0], c->ngrid[1], c->ngrid[2]}, c->stencil_radius};
    std::vector<float> vp(vp_model, vp_model + g.volume());
    float vmin = 0, vmax = 0;
    validate_vp(vp.data(), g, &vmin, &vmax);
    fill_ghosts_replicate(vp.data(), g);
    // driver.cpp:88-96
    const double dt = cfl_dt(vmax, c->ngrid, c->dgrid, c->stencil_radius, c->cfl);
    const std::vector<float> w = ricker(c->fmax, dt, c->nsteps);
    int src[3] = {c->ngrid[0] / 2, c->ngrid[1] / 2, c->ngrid[2] / 2};
    if (c->has_source_loc)
        for (int a = 0; a < 3; ++a) src[a] = c->source_loc[a];
    for (int a = 0; a < 3; ++a)
        if (src[a] < 0 || src[a] >= c->ngrid[a])
            raise(ST_CONFIG, "source location outside grid interior");
    // default receiver carpet (source.cpp:40-50)
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
    const int zero[3] = {0, 0, 0};
    mm_cd_engine* e = nullptr;
    int rc = mm_cd_create(&grid, zero, c->ngrid, vp.data(), &o, static_cast<float>(dt), vmax,
                          device, mode, &e);
    if (rc) return rc;
    std::unique_ptr<mm_cd_engine, int (*)(mm_cd_engine*)> guard(e, mm_cd_destroy);
    rc = mm_cd_set_receivers(e, rec.data(), nrec, c->nsteps);
    if (rc) return rc;
    float ms = 0;
    rc = mm_cd_run(e, w.data(), c->nsteps, src, 1, 0, &ms);
    if (rc) return rc;
    if (traces) {
        rc = mm_cd_get_traces(e, traces, c->nsteps);
        if (rc) return rc;
    }
    // driver.cpp:120 check_finite(p(src), nsteps)
    float ps = 0;
    MM_CUDA(cudaMemcpy(&ps, e->p[e->ic].ptr + e->lay.off(src[0], src[1], src[2]), sizeof(float),
                       cudaMemcpyDeviceToHost));
    if (!std::isfinite(ps))
        throw Error(ST_INSTABILITY,
                    "non-finite wavefield sample detected at time step " +
                        std::to_string(c->nsteps),
                    c->nsteps);
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
