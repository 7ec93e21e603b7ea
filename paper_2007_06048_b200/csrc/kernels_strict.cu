// kernels_strict.cu -- bit-exact (MM_MODE_STRICT) step kernels + plumbing kernels.
//
// One thread per grid point, reference association order, every operation an
// explicitly rounded __fadd_rn/__fsub_rn/__fmul_rn (never contracted to FMA),
// so results equal the CPU reference bit for bit:
//   k_strict_update  = update_plain (propagator_impl.hpp:89-104, stencil.hpp:70-82)
//                      + update_damping_pass2 (propagator_impl.hpp:125-152)
//   k_strict_pass1   = update_damping_pass1 (propagator_impl.hpp:106-123)
// The CPML memory lives in compact per-axis arrays over the active (a != 0)
// layer indices; the per-slab zero-halo semantics of the reference's
// BoxArray (cpml.hpp:77-99) are reproduced by the slab mask below (see
// DESIGN.md "CPML masking rule").
#include <algorithm>
#include <climits>

#include "mm_internal.hpp"

namespace mmb {

namespace {

__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

// second_derivative_at (stencil.hpp:86-91): t += c_m * ((p[+m] + p[-m]) - 2 p0)
template <int R>
__device__ __forceinline__ float d2_strict(const float* q, long long s, const float* c,
                                           float two_p0) {
    float t = 0.0f;
#pragma unroll
    for (int m = 1; m <= R; ++m)
        t = fadd(t, fmul(c[m - 1], fsub(fadd(__ldg(q + m * s), __ldg(q - m * s)), two_p0)));
    return t;
}

// The CPML run of axis `ax` containing local coordinate l, or nullptr.
__device__ __forceinline__ const CpmlRun* run_at(const StepParams& p, int ax, int l) {
    if (l >= p.run[ax][0].lo && l < p.run[ax][0].hi) return &p.run[ax][0];
    if (l >= p.run[ax][1].lo && l < p.run[ax][1].hi) return &p.run[ax][1];
    return nullptr;
}

// psi_ax at local (i,j,k) shifted by `sh` along ax; zero outside the damping
// runs and outside the local box (the reference's zero halo).  With `only`,
// `own` is the one run the point's slab box holds along ax (nullptr: none
// active): a slab of axis ax spans just its own layer, so the opposite layer
// is halo there even when it lies within R (inner extent < R), while slabs of
// an earlier axis span the whole of ax and see both layers.
__device__ __forceinline__ float psi_at(const StepParams& p, int ax, int i, int j, int k, int sh,
                                        bool only, const CpmlRun* own) {
    int loc[3] = {i, j, k};
    loc[ax] += sh;
    const CpmlRun* r = run_at(p, ax, loc[ax]);
    if (!r || (only && r != own)) return 0.0f;
    return __ldg(r->psi + run_off(*r, ax, loc[0], loc[1], loc[2]));
}

template <int R>
__global__ void k_strict_update(StepParams p, int region, int z_lo) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = z_lo + blockIdx.z;
    if (i >= p.lay.n[0] || j >= p.lay.n[1]) return;
    const int g[3] = {i + p.goff[0], j + p.goff[1], k + p.goff[2]};
    bool in[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) in[a] = g[a] >= p.nd[a] && g[a] < p.gn[a] - p.nd[a];
    const bool inner = in[0] && in[1] && in[2];
    if ((region == 1 && !inner) || (region == 2 && inner)) return;

    const long long o = p.lay.off(i, j, k);
    const float* q = p.pc + o;
    const long long s[3] = {1, p.lay.P, p.lay.plane};
    const float two_p0 = fmul(2.0f, q[0]);
    float lap;
    if (inner) {
        const float tx = d2_strict<R>(q, s[0], p.c2[0], two_p0);
        const float ty = d2_strict<R>(q, s[1], p.c2[1], two_p0);
        const float tz = d2_strict<R>(q, s[2], p.c2[2], two_p0);
        lap = fadd(fadd(tx, ty), tz);
    } else {
        // slab membership (grid.cpp:34-41): X slabs span all y,z; Y slabs the
        // inner x range; Z slabs the inner x,y range.  dpsi_ax reads psi only
        // inside the point's own slab box, which is what these masks encode.
        const bool use[3] = {!in[0], !in[0] || !in[1], true};
        const int sa = !in[0] ? 0 : !in[1] ? 1 : 2;  // the axis of the point's slab
        const int loc[3] = {i, j, k};
        float term[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const float d2p = d2_strict<R>(q, s[ax], p.c2[ax], two_p0);
            const int l = loc[ax];
            const float a = __ldg(p.ta[ax] + l), b = __ldg(p.tb[ax] + l),
                        ik = __ldg(p.tik[ax] + l);
            float dpsi = 0.0f;
            if (use[ax]) {
                const bool only = ax == sa;
                const CpmlRun* own = only ? run_at(p, ax, l) : nullptr;
#pragma unroll
                for (int m = 1; m <= R; ++m)
                    dpsi = fadd(dpsi,
                                fmul(p.c1[ax][m - 1], fsub(psi_at(p, ax, i, j, k, m, only, own),
                                                           psi_at(p, ax, i, j, k, -m, only, own))));
            }
            const float drive = fadd(fmul(d2p, ik), dpsi);
            const CpmlRun* run = run_at(p, ax, l);
            float z;
            if (run) {
                float* zp = run->zeta + run_off(*run, ax, i, j, k);
                z = fadd(fmul(b, *zp), fmul(a, drive));
                *zp = z;
            } else {
                z = fadd(fmul(b, 0.0f), fmul(a, drive));
            }
            term[ax] = fadd(drive, z);
        }
        lap = fadd(fadd(term[0], term[1]), term[2]);
    }
    p.pn[o] = fadd(fsub(two_p0, p.pp[o]), fmul(p.cv[o], lap));
}

// Pass 1 over the compact storage of one axis: psi = b psi + a D1(p_cur).
template <int R>
__global__ void k_strict_pass1(StepParams p, int ax, int side, int z_lo) {
    const CpmlRun& run = p.run[ax][side];
    int loc[3] = {(int)(blockIdx.x * blockDim.x + threadIdx.x),
                  (int)(blockIdx.y * blockDim.y + threadIdx.y), z_lo + (int)blockIdx.z};
    loc[ax] += run.lo;
    const int hi[3] = {ax == 0 ? run.hi : p.lay.n[0], ax == 1 ? run.hi : p.lay.n[1],
                       ax == 2 ? run.hi : p.lay.n[2]};
    if (loc[0] >= hi[0] || loc[1] >= hi[1] || loc[2] >= hi[2]) return;
    const long long s[3] = {1, p.lay.P, p.lay.plane};
    const float* q = p.pc + p.lay.off(loc[0], loc[1], loc[2]);
    float dp = 0.0f;
#pragma unroll
    for (int m = 1; m <= R; ++m)
        dp = fadd(dp, fmul(p.c1[ax][m - 1], fsub(__ldg(q + m * s[ax]), __ldg(q - m * s[ax]))));
    const int l = loc[ax];
    const float a = __ldg(p.ta[ax] + l), b = __ldg(p.tb[ax] + l);
    float* ps = run.psi + run_off(run, ax, loc[0], loc[1], loc[2]);
    *ps = fadd(fmul(b, *ps), fmul(a, dp));
}

template <int R>
void strict_pass1_r(const StepParams& p, int z_lo, int z_hi, cudaStream_t st) {
    for (int ax = 0; ax < 3; ++ax)
        for (int side = 0; side < 2; ++side) {
            const CpmlRun& run = p.run[ax][side];
            if (run.hi <= run.lo) continue;
            int lo[3] = {0, 0, z_lo}, hi[3] = {p.lay.n[0], p.lay.n[1], z_hi};
            lo[ax] = ax == 2 ? std::max(run.lo, z_lo) : run.lo;
            hi[ax] = ax == 2 ? std::min(run.hi, z_hi) : run.hi;
            if (hi[0] <= lo[0] || hi[1] <= lo[1] || hi[2] <= lo[2]) continue;
            dim3 blk(32, 8, 1);
            dim3 grd((hi[0] - lo[0] + 31) / 32, (hi[1] - lo[1] + 7) / 8, hi[2] - lo[2]);
            // kernel coordinates: offset along ax is relative to run.lo
            k_strict_pass1<R><<<grd, blk, 0, st>>>(p, ax, side, ax == 2 ? lo[2] - run.lo + 0 : lo[2]);
            note_launches(1);
        }
}

template <int R>
void strict_update_r(const StepParams& p, int region, int z_lo, int z_hi, cudaStream_t st) {
    if (z_hi <= z_lo) return;
    dim3 blk(32, 8, 1);
    dim3 grd((p.lay.n[0] + 31) / 32, (p.lay.n[1] + 7) / 8, z_hi - z_lo);
    k_strict_update<R><<<grd, blk, 0, st>>>(p, region, z_lo);
    note_launches(1);
}

__global__ void k_inject(float* pn, const float* cv, long long off, float amp,
                         const float* amp_dev, const int* step_dev) {
    // ref: propagator_impl.hpp:166-169  p_next[src] += ((dt2 vp) vp) amp
    const float a = amp_dev ? amp_dev[*step_dev] : amp;
    pn[off] = __fadd_rn(pn[off], __fmul_rn(cv[off], a));
}

__global__ void k_free_surface(float* p, Layout lay) {
    // ref: cpml.hpp:103-111, over i,j in [-r, n+r)
    const int i = blockIdx.x * blockDim.x + threadIdx.x - lay.r;
    const int j = blockIdx.y * blockDim.y + threadIdx.y - lay.r;
    if (i >= lay.n[0] + lay.r || j >= lay.n[1] + lay.r) return;
    p[lay.off(i, j, 0)] = 0.0f;
    for (int m = 1; m <= lay.r; ++m) p[lay.off(i, j, -m)] = -p[lay.off(i, j, m)];
}

__global__ void k_record(RecParams rp, const int* step_dev) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rp.nrec) return;
    const int step = step_dev ? *step_dev : rp.step;
    const float v = rp.p[rp.offs[r]];
    rp.traces[(long long)step * rp.nrec + r] = v;
    // ref: driver.cpp:68-71,108 check_finite(rec.at(0, n), n + 1)
    if (r == 0 && !isfinite(v) && rp.bad_step) atomicMin(rp.bad_step, step + 1);
}

__global__ void k_step_counter(int* step_dev) { *step_dev += 1; }

// k_inject + k_free_surface + k_record + k_step_counter in one launch, with
// the results of running them in that order.  Every thread reads the
// pre-injection field; values that the injection or the surface change are
// formed in registers (the injected source sample, 0 on the surface plane,
// the odd mirror), and the one write of p_next[src] -- the only location
// another thread could read -- is made by the last block to finish, after
// all reads.  That block also advances the step counter.
__global__ void k_epilogue(Epilogue e) {
    // Everything the update kernels do not write is read before
    // griddepcontrol.wait (a no-op without a programmatic launch): the step
    // counter and wavelet sample, c at the source, the receiver offsets.
    const int step = e.step_dev ? *e.step_dev : e.rec.step;
    const Layout& L = e.lay;
    const bool has_src = e.src_off >= 0;
    const float a = has_src ? (e.amp_dev ? e.amp_dev[step] : e.amp) : 0.0f;
    const float cs = has_src ? e.cv[e.src_off] : 0.0f;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int ex = L.n[0] + 2 * L.r;
    const long long nfs = e.fs ? (long long)ex * L.ey : 0;
    const bool is_rec = t >= nfs && t - nfs < e.rec.nrec;
    const long long roff = is_rec ? e.rec.offs[t - nfs] : 0;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float inj = 0.0f;
    if (has_src) inj = __fadd_rn(e.p[e.src_off], __fmul_rn(cs, a));  // propagator_impl.hpp:166-169
    auto value = [&](long long o) { return has_src && o == e.src_off ? inj : e.p[o]; };
    if (t < nfs) {  // cpml.hpp:103-111
        const int i = (int)(t % ex) - L.r, j = (int)(t / ex) - L.r;
        e.p[L.off(i, j, 0)] = 0.0f;
        for (int m = 1; m <= L.r; ++m) e.p[L.off(i, j, -m)] = -value(L.off(i, j, m));
    } else if (is_rec) {
        const int r = (int)(t - nfs);
        const long long o = roff;
        const bool on_surface = e.fs && o / L.plane == L.r;  // local z = 0
        const float v = on_surface ? 0.0f : value(o);
        e.rec.traces[(long long)step * e.rec.nrec + r] = v;
        // ref: driver.cpp:68-71,108 check_finite(rec.at(0, n), n + 1)
        if (r == 0 && !isfinite(v) && e.rec.bad_step) atomicMin(e.rec.bad_step, step + 1);
    } else if (t == nfs + e.rec.nrec && e.check_off >= 0 && e.rec.bad_step) {
        // per-step finiteness check of one more point: receiver 0 or the source
        // without recording (mm_cd_run), a slab's centre (dist.cpp:222-224)
        const bool on_surface = e.fs && e.check_off / L.plane == L.r;
        const float v = on_surface ? 0.0f : value(e.check_off);
        if (!isfinite(v)) atomicMin(e.rec.bad_step, step + 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(e.done, 1) == gridDim.x - 1) {
            __threadfence();
            if (has_src && !(e.fs && e.src_off / L.plane == L.r)) e.p[e.src_off] = inj;
            if (e.count) *e.step_dev = step + 1;
            *e.done = 0;
        }
    }
}

// Host layout (i slowest, k fastest, ghosted) <-> device layout (k slowest,
// i fastest, ghosted + padded), tiled 32x32 transposes over (i, k) per j.
__global__ void k_to_device(const float* __restrict__ h, float* __restrict__ d, Layout lay) {
    __shared__ float tile[32][33];
    const int ex = lay.n[0] + 2 * lay.r, ey = lay.ey, ez = lay.ez;
    const int j = blockIdx.z;
    const int k0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    for (int t = threadIdx.y; t < 32; t += blockDim.y) {
        const int i = i0 + t, k = k0 + threadIdx.x;
        if (i < ex && k < ez) tile[t][threadIdx.x] = h[((long long)i * ey + j) * ez + k];
    }
    __syncthreads();
    for (int t = threadIdx.y; t < 32; t += blockDim.y) {
        const int k = k0 + t, i = i0 + threadIdx.x;
        if (i < ex && k < ez)
            d[((long long)k * ey + j) * lay.P + (i - lay.r + lay.L)] = tile[threadIdx.x][t];
    }
}

__global__ void k_to_host(const float* __restrict__ d, float* __restrict__ h, Layout lay) {
    __shared__ float tile[32][33];
    const int ex = lay.n[0] + 2 * lay.r, ey = lay.ey, ez = lay.ez;
    const int j = blockIdx.z;
    const int k0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    for (int t = threadIdx.y; t < 32; t += blockDim.y) {
        const int k = k0 + t, i = i0 + threadIdx.x;
        if (i < ex && k < ez)
            tile[t][threadIdx.x] = d[((long long)k * ey + j) * lay.P + (i - lay.r + lay.L)];
    }
    __syncthreads();
    for (int t = threadIdx.y; t < 32; t += blockDim.y) {
        const int i = i0 + t, k = k0 + threadIdx.x;
        if (i < ex && k < ez) h[((long long)i * ey + j) * ez + k] = tile[threadIdx.x][t];
    }
}

__global__ void k_velocity_coeff(const float* vp, float* cv, float dt2, long long total) {
    // (dt2 * vp) * vp: bit-identical to the reference's dt2_*vp*vp
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x)
        cv[x] = __fmul_rn(__fmul_rn(dt2, vp[x]), vp[x]);
}

}  // namespace

#define MM_RADIUS_SWITCH(R_, CALL)                                   \
    switch (R_) {                                                    \
        case 1: CALL(1); break;                                      \
        case 2: CALL(2); break;                                      \
        case 3: CALL(3); break;                                      \
        case 4: CALL(4); break;                                      \
        case 5: CALL(5); break;                                      \
        case 6: CALL(6); break;                                      \
        case 7: CALL(7); break;                                      \
        case 8: CALL(8); break;                                      \
        default: raise(ST_CONFIG, "stencil radius must be in [1, 8]"); \
    }

void strict_pass1(const StepParams& p, int z_lo, int z_hi, cudaStream_t s) {
#define CALL(R) strict_pass1_r<R>(p, z_lo, z_hi, s)
    MM_RADIUS_SWITCH(p.lay.r, CALL)
#undef CALL
    MM_CUDA(cudaGetLastError());
}

void strict_update(const StepParams& p, int region, int z_lo, int z_hi, cudaStream_t s) {
#define CALL(R) strict_update_r<R>(p, region, z_lo, z_hi, s)
    MM_RADIUS_SWITCH(p.lay.r, CALL)
#undef CALL
    MM_CUDA(cudaGetLastError());
}

void launch_inject(float* pn, const float* cv, long long off, float amp, const float* amp_dev,
                   const int* step_dev, cudaStream_t s) {
    k_inject<<<1, 1, 0, s>>>(pn, cv, off, amp, amp_dev, step_dev);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch_free_surface(float* p, const Layout& lay, cudaStream_t s) {
    dim3 blk(32, 8);
    dim3 grd((lay.n[0] + 2 * lay.r + 31) / 32, (lay.n[1] + 2 * lay.r + 7) / 8);
    k_free_surface<<<grd, blk, 0, s>>>(p, lay);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch_record(const RecParams& rp, const int* step_dev, cudaStream_t s) {
    if (rp.nrec == 0) return;
    k_record<<<(rp.nrec + 255) / 256, 256, 0, s>>>(rp, step_dev);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch_step_counter(int* step_dev, cudaStream_t s) {
    k_step_counter<<<1, 1, 0, s>>>(step_dev);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch_epilogue(const Epilogue& ep, cudaStream_t s) {
    const long long nfs = ep.fs ? (long long)(ep.lay.n[0] + 2 * ep.lay.r) * ep.lay.ey : 0;
    const long long work = nfs + ep.rec.nrec + (ep.check_off >= 0 ? 1 : 0);
    if (work == 0 && ep.src_off < 0 && !ep.count) return;
    const int blocks = (int)std::max<long long>((work + 255) / 256, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = ep.pdl ? at : nullptr;
    cfg.numAttrs = ep.pdl ? 1 : 0;
    MM_CUDA(cudaLaunchKernelEx(&cfg, k_epilogue, ep));
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch_to_device_layout(const float* h, float* d, const Layout& lay, cudaStream_t s) {
    const int ex = lay.n[0] + 2 * lay.r;
    dim3 blk(32, 8);
    dim3 grd((lay.ez + 31) / 32, (ex + 31) / 32, lay.ey);
    k_to_device<<<grd, blk, 0, s>>>(h, d, lay);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch_to_host_layout(const float* d, float* h, const Layout& lay, cudaStream_t s) {
    const int ex = lay.n[0] + 2 * lay.r;
    dim3 blk(32, 8);
    dim3 grd((lay.ez + 31) / 32, (ex + 31) / 32, lay.ey);
    k_to_host<<<grd, blk, 0, s>>>(d, h, lay);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

void launch_velocity_coeff(const float* vp, float* cv, float dt2, long long total,
                           cudaStream_t s) {
    k_velocity_coeff<<<1184, 256, 0, s>>>(vp, cv, dt2, total);
    note_launches(1);
    MM_CUDA(cudaGetLastError());
}

}  // namespace mmb
