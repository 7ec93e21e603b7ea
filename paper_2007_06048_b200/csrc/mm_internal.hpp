// mm_internal.hpp -- shared internals of the B200 acoustic_iso_cd library.
//
// Device layout: x fastest, z slowest,
// the reverse of the reference's z-fastest host layout (grid.hpp:61-65), so
// that z-slabs, halo planes and the receiver plane are contiguous and the
// 2.5D kernels stream along the slowest axis.
//   dev_off(i,j,k) = ((k + r) * ey + (j + r)) * P + (i + L)
//   L = round_up(r, 4)     left x pad: interior x = 0 is 16-byte aligned
//   P = round_up(L + nx + r, 32)   row pitch (128-byte rows)
//   ey = ny + 2r, ez = nz + 2r
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace mmb {

// ---------------------------------------------------------------- errors
enum Status { ST_OK = 0, ST_CONFIG = 1, ST_VALIDATION = 2, ST_INSTABILITY = 3, ST_INVAL = 4, ST_CUDA = 5,
              ST_NCCL = 6 };

struct Error : std::runtime_error {
    int code;
    int step;
    Error(int c, const std::string& m, int s = 0) : std::runtime_error(m), code(c), step(s) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define MM_CUDA(x) ::mmb::cuda_check((x), #x, __FILE__, __LINE__)

// Counts kernel launches issued through the library (evidence for bench.py).
void note_launches(long long n);
long long launches_so_far();

// Process-wide tuning parameters (mm_set_tuning in the C ABI; engine.cu).
// The library never reads the environment: every parameter has a product
// default, and tests / experiments change one explicitly before creating an
// engine (most are read when an engine or its fast plan is created).
long long tuning(const char* name);

// C-ABI error plumbing (engine.cu): records the thread-local message/step
// behind mm_last_error() and returns the status code.
int set_api_error(int code, const std::string& msg, int step = 0);
inline void need(const void* p, const char* what) {
    if (!p) raise(ST_INVAL, std::string(what) + " must not be NULL");
}
#define MM_API_BEGIN try {
#define MM_API_END                                                       \
    }                                                                    \
    catch (const ::mmb::Error& ex) {                                     \
        return ::mmb::set_api_error(ex.code, ex.what(), ex.step);        \
    }                                                                    \
    catch (const std::bad_alloc&) {                                      \
        return ::mmb::set_api_error(MM_EINVAL, "host allocation failed"); \
    }                                                                    \
    catch (const std::exception& ex) {                                   \
        return ::mmb::set_api_error(MM_EINVAL, ex.what());               \
    }                                                                    \
    return MM_OK;

// ---------------------------------------------------------------- numerics
// All of these restate the reference bit for bit (see host_numerics.cpp).
struct Coeffs {
    std::vector<double> c;  // taps m = 1..radius (c[m-1])
    double center = 0.0;
};
Coeffs second_derivative(int radius, double h);      // ref: stencil.cpp:50-74
Coeffs central_first_derivative(int radius, double h);  // ref: stencil.cpp:99-117
Coeffs staggered_first_derivative(int radius, double h);  // ref: stencil.cpp:76-97
std::vector<float> integrate_wavelet(const std::vector<float>& w, double dt);  // source.cpp:30-38
double cfl_dt(double vmax, const int n[3], const double d[3], int radius, double cfl);
std::vector<float> ricker(double fmax, double dt, int nsteps);

struct Profile {  // ref: cpml.hpp:13-26 (float tables over the global axis)
    std::vector<float> a[3], b[3], ik[3];
    double d0[3] = {0, 0, 0};
};
Profile build_profile(const int n[3], const double h[3], const int nd[3], double fmax,
                      double vmax, double dt, double r_target, bool free_surface);

// Host reference-layout helpers (ghosted, z fastest).
struct HostGrid {
    int n[3];
    int r;
    size_t ext(int a) const { return (size_t)n[a] + 2 * r; }
    size_t volume() const { return ext(0) * ext(1) * ext(2); }
    size_t off(int i, int j, int k) const {
        return ((size_t)(i + r) * ext(1) + (size_t)(j + r)) * ext(2) + (size_t)(k + r);
    }
};
void fill_ghosts_replicate(float* f, const HostGrid& g);
void taper_material(float* f, const HostGrid& g, const int ntaper[3], const int offset[3],
                    const int global_n[3]);
void validate_vp(const float* vp, const HostGrid& g, float* vmin, float* vmax);

// ---------------------------------------------------------------- device
// Owning device allocation (engine-lifetime buffers).
template <typename T>
struct DevBuf {
    T* ptr = nullptr;
    T* base = nullptr;  // the allocation (ptr = base + a stagger of `pad` elements)
    size_t count = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void reset() {
        if (base) cudaFree(base);
        ptr = base = nullptr;
        count = 0;
    }
    void alloc(size_t n, size_t pad = 0) {
        reset();
        if (n == 0) return;
        MM_CUDA(cudaMalloc(&base, (n + pad) * sizeof(T)));
        ptr = base + pad;
        count = n;
    }
    void alloc_zero(size_t n, cudaStream_t s, size_t pad = 0) {
        alloc(n, pad);
        if (n) MM_CUDA(cudaMemsetAsync(ptr, 0, n * sizeof(T), s));
    }
    void upload(const T* host, size_t n, cudaStream_t s) {
        if (count < n) alloc(n);
        if (n) MM_CUDA(cudaMemcpyAsync(ptr, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
};

// Asynchronous device->host copies of recorded receiver samples on their own
// stream, ordered after the recording kernel by an event, so the copy engine
// overlaps the next step's kernels instead of stalling the compute stream.
struct TraceCopier {
    cudaStream_t cs = nullptr;
    cudaEvent_t ev = nullptr;
    void copy(void* dst, const void* src, size_t bytes, cudaStream_t after) {
        if (!cs) {
            MM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            MM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        MM_CUDA(cudaEventRecord(ev, after));
        MM_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        MM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, cs));
    }
    void sync() {
        if (cs) MM_CUDA(cudaStreamSynchronize(cs));
    }
    ~TraceCopier() {
        if (cs) {
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
        }
        if (ev) cudaEventDestroy(ev);
    }
};

// Per-kernel CUDA-event timing of the launches of a step (bench evidence:
// the dominant kernel's duration inside the real, concurrent step).  Off by
// default; begin/end record events on the launching stream.
struct KernelTimer {
    bool on = false;
    int begin(const char* name, cudaStream_t s);  // -1 when off
    void end(int idx, cudaStream_t s);
    // waits for the recorded events and adds their durations to `acc`
    void collect();
    void reset();
    std::map<std::string, std::pair<double, long long>> acc;  // name -> (total ms, launches)
    ~KernelTimer();

private:
    struct Rec {
        std::string name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> pending_;
    std::vector<cudaEvent_t> pool_;
    cudaEvent_t get();
};

struct Layout {
    int n[3];
    int r, L, P, ey, ez;
    long long plane;  // ey * P
    long long total;  // plane * ez
    static Layout make(const int n[3], int r);
    __host__ __device__ long long off(int i, int j, int k) const {
        return ((long long)(k + r) * ey + (j + r)) * (long long)P + (i + L);
    }
};

constexpr int kMaxR = 8;

// CPML memory of one damping layer ("run") of one axis: the local index range
// [lo, hi) along that axis, full extent along the other two.  Reads outside
// the run return 0 -- the zero halo of the reference's per-slab BoxArray
// (cpml.hpp:77-99).  Element (i,j,k), c = (axis coordinate) - lo:
//   axis 0: c + j*s1 + k*s2      (s1 = W = round_up(hi-lo, 4), s2 = W*ny)
//   axis 1: i + c*s1 + k*s2      (s1 = nx4, s2 = nx4*(hi-lo))
//   axis 2: i + j*s1 + c*s2      (s1 = nx4, s2 = nx4*ny)
// nx4 = round_up(nx, 4).  A run is allocated only if some a != 0 in it.
struct CpmlRun {
    int lo, hi;  // hi <= lo: absent
    int org;     // array origin along the axis: lo, rounded down to 4 for axis 0
                 // (TMA box starts must be 16-byte aligned in the fastest dim)
    float* psi;
    float* zeta;
    long long s1, s2;
};

__host__ __device__ inline long long run_off(const CpmlRun& r, int ax, int i, int j, int k) {
    if (ax == 0) return (i - r.org) + j * r.s1 + k * r.s2;
    if (ax == 1) return i + (j - r.org) * r.s1 + k * r.s2;
    return i + j * r.s1 + (k - r.org) * r.s2;
}

// Everything a step kernel needs, passed by value.
struct StepParams {
    Layout lay;
    int goff[3];  // local -> global index offset
    int gn[3];    // global interior size
    int nd[3];    // ndamping (region partition, grid.cpp:24-45)
    const float* pc;  // p_cur
    const float* pp;  // p_prev
    float* pn;        // p_next
    const float* cv;  // (dt2 * vp) * vp, device layout
    float c2[3][kMaxR];  // second-derivative taps per axis (float, 1/h^2 folded)
    float c1[3][kMaxR];  // central first-derivative taps per axis
    // CPML: local tables (length n[ax]) and the per-layer memory runs
    const float* ta[3];
    const float* tb[3];
    const float* tik[3];
    CpmlRun run[3][2];  // [axis][0 = low layer, 1 = high layer]
};

// Receiver sampling, device trace layout [step][receiver].
struct RecParams {
    const float* p;
    const long long* offs;  // device offsets of receivers
    float* traces;
    int nrec;
    int step;
    int* bad_step;  // first 1-based step with non-finite receiver 0 (INT_MAX if none)
};

// The end of a step in one launch: source injection, free surface, receiver
// sampling of the new field and the device step counter (k_epilogue).
struct Epilogue {
    float* p;              // p_next (p_cur after the rotation)
    const float* cv;
    long long src_off;     // < 0: no source
    float amp;
    const float* amp_dev;  // non-null: amplitude amp_dev[*step_dev]
    int* step_dev;         // device step counter (or null: rec.step)
    bool count;            // advance *step_dev once every block has read it
    bool fs;               // free surface at local z = 0
    Layout lay;
    RecParams rec;         // nrec = 0: no sampling (rec.p is ignored: p)
    long long check_off;   // >= 0: finiteness check of this point into rec.bad_step
    int* done;             // block ticket (zero between launches)
    bool pdl;              // programmatic launch: may start while the kernel before drains
};

// ---- launchers (kernels_strict.cu)
void strict_pass1(const StepParams& p, int z_lo, int z_hi, cudaStream_t s);
// region: 0 = every point, 1 = inner box only, 2 = damping slabs only
void strict_update(const StepParams& p, int region, int z_lo, int z_hi, cudaStream_t s);
void launch_inject(float* pn, const float* cv, long long off, float amp, const float* amp_dev,
                   const int* step_dev, cudaStream_t s);
void launch_free_surface(float* p, const Layout& lay, cudaStream_t s);
void launch_record(const RecParams& rp, const int* step_dev, cudaStream_t s);
void launch_step_counter(int* step_dev, cudaStream_t s);
void launch_epilogue(const Epilogue& ep, cudaStream_t s);
void launch_to_device_layout(const float* host_layout, float* dev_layout, const Layout& lay,
                             cudaStream_t s);
void launch_to_host_layout(const float* dev_layout, float* host_layout, const Layout& lay,
                           cudaStream_t s);
void launch_velocity_coeff(const float* vp_dev_layout, float* cv, float dt2, long long total,
                           cudaStream_t s);

}  // namespace mmb
