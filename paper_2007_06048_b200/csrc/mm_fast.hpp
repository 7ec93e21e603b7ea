// mm_fast.hpp -- the MM_MODE_FAST step (TMA-fed 2.5D kernels), see kernels_fast.cu.
#pragma once

#include <cuda.h>

#include <memory>

#include "mm_internal.hpp"

namespace mmb {

// 3D fp32 TMA tensor map (x fastest, box bx x by x 1, out-of-bounds reads
// zero) over a device-layout field; shared with the acoustic_iso engine.
CUtensorMap tma_field_map(const Layout& L, const float* base, int bx, int by);

class FastPlan {
public:
    virtual ~FastPlan() = default;
    // CPML pass 1 over the compact psi storage (all local planes).
    virtual void pass1(const StepParams& p, cudaStream_t s) = 0;
    // Pass 2 + inner update on local planes [z_lo, z_hi); region as strict_update.
    virtual void update(const StepParams& p, int region, int z_lo, int z_hi, cudaStream_t s) = 0;
    // Pass 2 + inner update on the union of n plane ranges [r[2i], r[2i+1]).
    virtual void update_ranges(const StepParams& p, const int* ranges, int n, cudaStream_t s) = 0;
    // The z-slab schedule's interior part (group.cu), in three calls: the
    // step's start on s (before pass 1); the interior kernel of planes
    // [z_lo, z_hi) on the side stream from that point (true) -- or false when
    // this layout has no side-stream interior; then the boundary kernel of
    // those planes on s and the join (or, after false, the whole update).
    virtual void fork_point(cudaStream_t s) = 0;
    virtual bool interior_side(const StepParams& p, int z_lo, int z_hi) = 0;
    virtual void finish_overlap(const StepParams& p, int z_lo, int z_hi, cudaStream_t s,
                                bool side) = 0;
    // One whole step (pass 1, update, source injection); src_off < 0: no source.
    virtual void step(const StepParams& p, long long src_off, float amp, const float* amp_dev,
                      const int* step_dev, cudaStream_t s) = 0;
    // The kernel the step uses for the damping slabs: "cpml" (fused one-pass
    // k_cpml), "two-pass" (k_p1 + k_bnd) or "strict".
    virtual const char* cpml_path(const StepParams& p) = 0;
    KernelTimer timer;  // per-kernel events around the step's launches (off by default)
};

// nullptr when the fast kernels cannot serve this layout (the engine then
// runs the strict kernels, which are exact for every radius).
// order: 2 = reference order, every operation rounded (bit-exact); 1 = FMA.
std::unique_ptr<FastPlan> make_fast_plan(const Layout& lay, int device, float* const bufs[3],
                                         const float* cv, int order);

}  // namespace mmb
