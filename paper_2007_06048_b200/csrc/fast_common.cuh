// fast_common.cuh -- PTX helpers (mbarrier, TMA) shared by the fast kernels.
#pragma once

#include <cuda.h>

#include "mm_internal.hpp"

namespace mmb {
namespace fast {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MM_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra MM_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
#ifndef MM_PROD_SLEEP_NS
#define MM_PROD_SLEEP_NS 64
#endif
// Producer-side wait: back off with nanosleep between polls so a spinning
// producer lane does not take issue slots from the consumer warps.
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// Non-blocking probe of a phase (mbarrier.test_wait).
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
#ifdef MM_PROD_SPIN
    mbar_wait(bar, parity);
#else
    while (!mbar_try(bar, parity)) __nanosleep(MM_PROD_SLEEP_NS);
#endif
}
__device__ __forceinline__ void mbar_arrive_b(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// 3D tiled TMA load global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            int z, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}
// (diagnostics, build with -DMM_TRACE) per-CTA start / end globaltimer
#ifdef MM_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// records (kid, sm, t0, t1) into a device ring read by mm_trace_dump
__device__ unsigned long long g_mm_trace[4 * 65536];
__device__ unsigned int g_mm_trace_n;
#define MM_TRACE_BEGIN const unsigned long long mm_t0 = gtimer();
#define MM_TRACE_END(kid)                                                              \
    if (threadIdx.x == 0) {                                                           \
        unsigned sm;                                                                  \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));                               \
        const unsigned i = atomicAdd(&g_mm_trace_n, 1u) % 65536u;                      \
        g_mm_trace[4 * i] = (unsigned long long)(kid);                                \
        g_mm_trace[4 * i + 1] = sm;                                                   \
        g_mm_trace[4 * i + 2] = mm_t0;                                                \
        g_mm_trace[4 * i + 3] = gtimer();                                             \
    }
#else
#define MM_TRACE_BEGIN
#define MM_TRACE_END(kid)
#endif
// Programmatic dependent launch: wait for the preceding grid's memory / let
// the dependent grid launch.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Dynamic work queue shared by the persistent kernels.  Items are ordered so
// that the ~gridDim.x items in flight at any moment are spatial neighbours at
// the same z (their halos meet in L2).  ctr[0] = next item, ctr[1] = CTAs
// done; the last CTA resets both, so every launch / graph replay starts at 0.
struct WorkQueue {
    int* ctr;
    int nitems;
};
__device__ __forceinline__ int wq_next(const WorkQueue& q, int* s_slot) {
    if (threadIdx.x == 0) *s_slot = atomicAdd(q.ctr, 1);
    __syncthreads();
    const int v = *s_slot;
    __syncthreads();
    return v;
}
__device__ __forceinline__ void wq_done(const WorkQueue& q) {
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(q.ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(q.ctr, 0);
            atomicExch(q.ctr + 1, 0);
        }
    }
}

// Shared-memory region sizes rounded up to 128 bytes (32 floats): TMA
// destinations must be 128-byte aligned.
__host__ __device__ constexpr int pad32(int n) { return (n + 31) / 32 * 32; }

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float comp(const float4& v, int e) {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

// CPML run membership and 4-point (float4) global access helpers
__device__ __forceinline__ bool in_run(const CpmlRun& r, int l) { return l >= r.lo && l < r.hi; }
__device__ __forceinline__ bool near_run(const CpmlRun& r, int a, int b) {
    return r.hi > r.lo && a < r.hi && b > r.lo;  // [a, b) meets the run
}
__device__ __forceinline__ float4 ldg4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}
// 16-byte load of 4 points, element-wise (zeros elsewhere) at a box edge
__device__ __forceinline__ float4 ld4(const float* p, const bool (&ok)[4], bool all) {
    if (all) return ldg4(p);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok[0]) v.x = __ldg(p);
    if (ok[1]) v.y = __ldg(p + 1);
    if (ok[2]) v.z = __ldg(p + 2);
    if (ok[3]) v.w = __ldg(p + 3);
    return v;
}
__device__ __forceinline__ void st4(float* p, const float (&v)[4], const bool (&ok)[4], bool all) {
    if (all) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (ok[e]) p[e] = v[e];
    }
}

// Arithmetic of the fast kernels, by association order ORD:
//  ORD 2 (default): the reference's order with every operation separately
//         rounded (no FMA contraction) -- bit-identical to the CPU reference
//  ORD 1: reference order with FMA contraction
//  ORD 0: factored stencil, t = fma(c_m, p+ + p-, t), centre added once
template <int ORD>
__device__ __forceinline__ float fa(float a, float b) {
    return ORD == 2 ? __fadd_rn(a, b) : a + b;
}
template <int ORD>
__device__ __forceinline__ float fs(float a, float b) {
    return ORD == 2 ? __fsub_rn(a, b) : a - b;
}
template <int ORD>
__device__ __forceinline__ float fm(float a, float b) {
    return ORD == 2 ? __fmul_rn(a, b) : a * b;
}
// t + c * x  (reference: `t += c * x`)
template <int ORD>
__device__ __forceinline__ float acc(float t, float c, float x) {
    return ORD == 2 ? __fadd_rn(t, __fmul_rn(c, x)) : fmaf(c, x, t);
}

// Per-axis second-derivative term (second_derivative_at, stencil.hpp:86-91):
//   t += c_m * ((p[+m] + p[-m]) - 2 p0)
template <int ORD>
__device__ __forceinline__ float d2_term(float t, float c, float pp, float pm, float two_p0) {
    if (ORD == 0) return fmaf(c, pp + pm, t);
    return acc<ORD>(t, c, fs<ORD>(fa<ORD>(pp, pm), two_p0));
}

// ---- packed pairs of fp32 (Blackwell's f32x2 ALU: FADD2 / FFMA2)
// add.rn.f32x2 / sub.rn.f32x2 round each lane like add.rn.f32, so ORD 2 stays
// bit-identical.  A packed product in ORD 2 is fma.rn.f32x2(c, x, -0): the
// exact product plus -0, rounded once == mul.rn (+0 + -0 = +0, subnormals
// kept).  The -0 comes from constant memory so ptxas cannot see it: with a
// literal -0 it rewrites the FMA as a multiply and then contracts that
// multiply with the following add into one FFMA2 (checked in SASS), which
// changes the rounding; so does mul.rn.f32x2 followed by add.rn.f32x2.
static __constant__ unsigned long long kNegZero2 = 0x8000000080000000ull;
struct F2 {
    unsigned long long r;
};
__device__ __forceinline__ F2 f2(float a, float b) {
    F2 p;
    asm("mov.b64 %0, {%1, %2};" : "=l"(p.r) : "f"(a), "f"(b));
    return p;
}
__device__ __forceinline__ void unf2(F2 p, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(p.r));
}
__device__ __forceinline__ float f2lo(F2 p) {
    float a, b;
    unf2(p, a, b);
    return a;
}
__device__ __forceinline__ float f2hi(F2 p) {
    float a, b;
    unf2(p, a, b);
    return b;
}
__device__ __forceinline__ F2 f2zero() { return f2(0.0f, 0.0f); }
template <int ORD>
__device__ __forceinline__ F2 fa2(F2 a, F2 b) {
    F2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.r) : "l"(a.r), "l"(b.r));
    return d;
}
template <int ORD>
__device__ __forceinline__ F2 fs2(F2 a, F2 b) {
    F2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.r) : "l"(a.r), "l"(b.r));
    return d;
}
// (c0, c1) * x lane-wise, each lane rounded once
template <int ORD>
__device__ __forceinline__ F2 fm2v(float c0, float c1, F2 x) {
    F2 d;
    if constexpr (ORD == 2) {
#ifdef MM_F2_SCALAR_MUL  // A/B build variant: two FMULs and a pack
        float a, b;
        unf2(x, a, b);
        return f2(__fmul_rn(c0, a), __fmul_rn(c1, b));
#endif
        asm("fma.rn.f32x2 %0, %1, %2, %3;"
            : "=l"(d.r)
            : "l"(f2(c0, c1).r), "l"(x.r), "l"(kNegZero2));
    } else {
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.r) : "l"(f2(c0, c1).r), "l"(x.r));
    }
    return d;
}
template <int ORD>
__device__ __forceinline__ F2 fm2(float c, F2 x) {
    return fm2v<ORD>(c, c, x);
}
// a * b lane-wise
template <int ORD>
__device__ __forceinline__ F2 fmul2(F2 a, F2 b) {
    float a0, a1;
    unf2(a, a0, a1);
    return fm2v<ORD>(a0, a1, b);
}
// lanes (x, y) or (z, w) of a float4
__device__ __forceinline__ F2 half2(const float4& v, int h) {
    return h == 0 ? f2(v.x, v.y) : f2(v.z, v.w);
}
// t + c * x  (reference `t += c * x`)
template <int ORD>
__device__ __forceinline__ F2 acc2(F2 t, float c, F2 x) {
    if constexpr (ORD == 2) {
        return fa2<ORD>(t, fm2<ORD>(c, x));
    } else {
        F2 d;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.r) : "l"(x.r), "l"(f2(c, c).r), "l"(t.r));
        return d;
    }
}
// t + (c0, c1) * x lane-wise
template <int ORD>
__device__ __forceinline__ F2 acc2v(F2 t, float c0, float c1, F2 x) {
    if constexpr (ORD == 2) {
        return fa2<ORD>(t, fm2v<ORD>(c0, c1, x));
    } else {
        F2 d;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.r) : "l"(x.r), "l"(f2(c0, c1).r), "l"(t.r));
        return d;
    }
}
// central_derivative_at term, both lanes: t += c * (pp - pm)
template <int ORD>
__device__ __forceinline__ F2 d1_term2(F2 t, float c, F2 pp, F2 pm) {
    return acc2<ORD>(t, c, fs2<ORD>(pp, pm));
}
__device__ __forceinline__ float4 f4(F2 a, F2 b) {
    float4 v;
    unf2(a, v.x, v.y);
    unf2(b, v.z, v.w);
    return v;
}
// second_derivative_at term, both lanes: t += c * ((pp + pm) - 2 p0)
template <int ORD>
__device__ __forceinline__ F2 d2_term2(F2 t, float c, F2 pp, F2 pm, F2 two_p0) {
    return acc2<ORD>(t, c, fs2<ORD>(fa2<ORD>(pp, pm), two_p0));
}
__device__ __forceinline__ void lds4x2(const float* p, F2& a, F2& b) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    a = f2(v.x, v.y);
    b = f2(v.z, v.w);
}

}  // namespace fast
}  // namespace mmb
