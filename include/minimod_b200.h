/*
 * minimod_b200.h -- C ABI of the B200-native acoustic_iso_cd propagator.
 *
 * Drop-in boundary for the reference's minimod::AcousticCdEngine<float>
 * (/root/reference/proj/core/include/minimod/propagator.hpp:93-140,
 * implemented at propagator_impl.hpp:53-173) and its callers run()
 * (driver.cpp:83-144) and run_distributed_rank() (dist.cpp:144-267).
 * Plain pointers and sizes only; no CUDA or torch types cross this boundary
 * (streams are passed as void*).
 *
 * Conventions
 *  - Every function returns an mm_status; on failure mm_last_error() holds a
 *    thread-local message.  Status codes mirror the reference exceptions
 *    (errors.hpp:10-30): ConfigError -> MM_ECONFIG, ValidationError ->
 *    MM_EVALIDATION, InstabilityError -> MM_EINSTABILITY (step in
 *    mm_last_instability_step()), std::invalid_argument -> MM_EINVAL.
 *  - Host field arrays use the reference layout: ghosted, z fastest,
 *    offset(i,j,k) = ((i+r)*(ny+2r) + (j+r))*(nz+2r) + (k+r)
 *    (grid.hpp:61-65); (nx+2r)*(ny+2r)*(nz+2r) floats.
 *  - Host pointers are caller-owned and only touched during the call.  The
 *    engine owns all device memory.  One host thread drives one engine at a
 *    time; calls are not reentrant (same rule as the reference).
 *  - Engine calls are asynchronous on the engine's CUDA stream except those
 *    that return host data (get_*) and mm_cd_synchronize.
 */
#ifndef MINIMOD_B200_H
#define MINIMOD_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mm_status {
    MM_OK = 0,
    MM_ECONFIG = 1,      /* minimod::ConfigError */
    MM_EVALIDATION = 2,  /* minimod::ValidationError */
    MM_EINSTABILITY = 3, /* minimod::InstabilityError */
    MM_EINVAL = 4,       /* std::invalid_argument / contract violation */
    MM_ECUDA = 5,        /* CUDA runtime failure */
    MM_ENCCL = 6         /* collective failure (multi-GPU plumbing) */
} mm_status;

/* Kernel families / arithmetic of the device step (chosen at create time).
 *  MM_MODE_FAST:     the TMA / register-queue kernels (default), reference
 *                    association order with every operation separately
 *                    rounded: bit-identical to the CPU reference.
 *  MM_MODE_STRICT:   one thread per point, same arithmetic; bit-identical.
 *  MM_MODE_FAST_FMA: the fast kernels with FMA contraction of the reference
 *                    order (not bit-identical; ~1e-5 relative). */
typedef enum mm_mode { MM_MODE_FAST = 0, MM_MODE_STRICT = 1, MM_MODE_FAST_FMA = 2 } mm_mode;

/* ref: grid.hpp:49-73 Grid3D (n, d, radius; stagger is not used by CD). */
typedef struct mm_grid {
    int n[3];
    double d[3];
    int radius;
} mm_grid;

/* ref: propagator.hpp:23-30 EngineOptions (defaults: ndamping 0, fmax 25,
 * r_target 1e-3, free_surface 0, taper 0, ntaper 3). */
typedef struct mm_engine_options {
    int ndamping[3];
    double fmax;
    double r_target;
    int free_surface;
    int taper;
    int ntaper[3];
} mm_engine_options;

typedef struct mm_cd_engine mm_cd_engine;

const char* mm_last_error(void);
int mm_last_instability_step(void);
const char* mm_version(void);
/* Number of CUDA devices visible (0 on a CPU-only host). */
int mm_device_count(int* count);
/* Kernel launches issued by this process so far (all engines). */
long long mm_kernel_launch_count(void);
/* Process-wide tuning parameters (work-item sizes, CUDA-graph use, kernel
 * families, diagnostics; the list and defaults are in csrc/engine.cu
 * kTunables).  The library never reads the environment; most parameters are
 * read when an engine is created.  Unknown names: MM_EINVAL. */
int mm_set_tuning(const char* name, long long value);
int mm_get_tuning(const char* name, long long* value);
int mm_reset_tuning(void);

/* ------------------------------------------------------------------------
 * Host numerics (C++; bit-identical to the reference)
 * --------------------------------------------------------------------- */

/* ref: stencil.cpp:50-74 second_derivative_coeffs -> c[radius] (1/h^2 folded
 * in) and the center weight. */
int mm_second_derivative_coeffs(int radius, double h, double* c, double* center);
/* ref: stencil.cpp:99-117 central_first_derivative_coeffs -> c[radius]. */
int mm_central_first_derivative_coeffs(int radius, double h, double* c);
/* ref: driver.cpp:19-29 cfl_dt. */
int mm_cfl_dt(double vmax, const mm_grid* grid, double cfl, double* dt);
/* ref: source.cpp:11-28 ricker. */
int mm_ricker(double fmax, double dt, int nsteps, float* out);
/* ref: cpml.hpp:34-72 build_profile<float>.  a/b/inv_kappa are the three
 * axes concatenated (n[0]+n[1]+n[2] floats each); d0[3] optional. */
int mm_build_profile(const int n[3], const double h[3], const int ndamping[3], double fmax,
                     double vmax, double dt, double r_target, int free_surface, float* a,
                     float* b, float* inv_kappa, double* d0);
/* ref: propagator.hpp:36-62 taper_material (then fill_ghosts_replicate), in
 * place on a ghosted z-fastest field. */
int mm_taper_material(float* f, const int n[3], int radius, const int ntaper[3],
                      const int offset[3], const int global_n[3]);
/* ref: model.cpp:63-77 default_layered_model (vp only) + validate_model. */
int mm_layered_model(const int n[3], int radius, float* vp, float* vmin, float* vmax);
/* ref: model.cpp:15-43 validate_model for vp: checks finite and > 0,
 * computes vmin/vmax, replicates ghosts in place. */
int mm_validate_model(const int n[3], int radius, float* vp, float* vmin, float* vmax);

/* ------------------------------------------------------------------------
 * Engine (ref: AcousticCdEngine<float>)
 * --------------------------------------------------------------------- */

/* ref: propagator.hpp:96-98 ctor.  vp_local: ghosted z-fastest local field
 * (copied).  offset/global_n place the local box in the global grid (0 and
 * local n for single-device use).  device: CUDA ordinal; mode: mm_mode. */
int mm_cd_create(const mm_grid* local, const int offset[3], const int global_n[3],
                 const float* vp_local, const mm_engine_options* opts, float dt,
                 double vmax_global, int device, int mode, mm_cd_engine** out);
int mm_cd_destroy(mm_cd_engine* e);

/* ref: propagator.hpp:103-104 step(amp, src).  src_local: 3 ints in local
 * interior coordinates, or NULL when this engine does not own the source.
 * The step's last kernel (source injection, free surface) is launched by the
 * next call on this engine -- mm_cd_record then samples inside it -- so work
 * a host enqueues on the engine stream itself must follow a call such as
 * mm_cd_stream or mm_cd_synchronize (tuning "defer_epilogue" = 0: launched at
 * once). */
int mm_cd_step(mm_cd_engine* e, float amp, const int* src_local);

/* Sub-phases of one step, in the reference order (propagator_impl.hpp:
 * 154-173).  Calling them in this order equals mm_cd_step. */
int mm_cd_update_boundary_psi(mm_cd_engine* e); /* pass 1, :106-123 */
int mm_cd_update_inner(mm_cd_engine* e);        /* update_plain, :89-104 */
int mm_cd_update_boundary(mm_cd_engine* e);     /* pass 2, :125-152 */
int mm_cd_inject_source(mm_cd_engine* e, float amp, const int* src_local); /* :166-169 */
int mm_cd_apply_free_surface(mm_cd_engine* e);  /* :170, cpml.hpp:103-111 */
int mm_cd_rotate(mm_cd_engine* e);              /* :171-172 */

int mm_cd_synchronize(mm_cd_engine* e);
/* Number of floats in one ghosted local field (host layout). */
int mm_cd_field_size(mm_cd_engine* e, size_t* count);
int mm_cd_get_dt(mm_cd_engine* e, float* dt);
int mm_cd_get_mode(mm_cd_engine* e, int* mode);
int mm_cd_steps_taken(mm_cd_engine* e, long long* steps);

/* ref: propagator.hpp:106-110 pressure()/pressure_prev() (device -> host,
 * reference layout, ghosts included). */
int mm_cd_get_pressure(mm_cd_engine* e, float* host);
int mm_cd_get_pressure_prev(mm_cd_engine* e, float* host);
/* Tapered vp copy the engine steps with (ref: propagator_impl.hpp:60,73). */
int mm_cd_get_velocity(mm_cd_engine* e, float* host);
/* ref: propagator.hpp:116-120 set_state(p_prev, p_cur). */
int mm_cd_set_state(mm_cd_engine* e, const float* p_prev, const float* p_cur);

/* ref: propagator.hpp:112-114 profile().  Tables over the GLOBAL axis
 * length global_n[axis].  set_profile replaces the tables; it is accepted
 * before the first step only, and a must be zero outside the damping
 * layers (the CPML memory lives only there). */
int mm_cd_get_profile(mm_cd_engine* e, int axis, float* a, float* b, float* inv_kappa);
int mm_cd_set_profile(mm_cd_engine* e, int axis, const float* a, const float* b,
                      const float* inv_kappa);
int mm_cd_get_d0(mm_cd_engine* e, double d0[3]);

/* Receiver hooks (ref: source.cpp:40-66 default_receivers/record,
 * source.hpp:44-52 ShotRecord).  ijk: n receivers x 3 local interior
 * coordinates.  capacity: number of time samples the device trace buffer
 * holds.  mm_cd_record(step) samples p_cur into column `step`.
 * mm_cd_get_traces copies out in ShotRecord layout traces[r*nsteps + s]. */
int mm_cd_set_receivers(mm_cd_engine* e, const int* ijk, int nreceivers, int capacity);
int mm_cd_record(mm_cd_engine* e, int step);
int mm_cd_get_traces(mm_cd_engine* e, float* host, int nsteps);
/* Copy one recorded time sample (all receivers, nreceivers floats, receiver
 * order) to host memory.  async != 0: enqueue on the engine's copy stream,
 * ordered after the work enqueued so far, and return -- the copy overlaps the
 * following steps (host should be pinned; read it after mm_cd_synchronize,
 * which also waits for the copy stream). */
int mm_cd_copy_trace_step(mm_cd_engine* e, int step, float* host, int async);

/* Device-resident time loop: nsteps steps with source amplitudes amps[]
 * (device copy), recording every step into columns [first_sample, ...) when
 * record != 0, one receiver-0 finiteness check per step (ref: driver.cpp:
 * 102-112,68-71).  CUDA-graph captured.  *device_ms (optional) = device
 * time of the loop (CUDA events).  Returns MM_EINSTABILITY with the first
 * failing step (1-based, as the reference) if receiver 0 went non-finite. */
int mm_cd_run(mm_cd_engine* e, const float* amps, int nsteps, const int* src_local, int record,
              int first_sample, float* device_ms);

/* ------------------------------------------------------------------------
 * Multi-GPU plumbing (z-slabs; ref: dist.cpp:92-115 exchange_halos).
 * The halo transport itself (NCCL send/recv) is issued by the host runtime
 * on the engine's stream; these expose the contiguous plane ranges.
 * --------------------------------------------------------------------- */
/* Which kernels update the damping slabs in a full step: "cpml" (the fused
 * one-pass kernel), "two-pass" (CPML pass 1 then pass 2) or "strict". */
int mm_cd_cpml_path(mm_cd_engine* e, char* buf, int cap);
/* Per-kernel device timing of fast-mode steps (benchmark evidence): on != 0
 * brackets every kernel a step launches with CUDA events on the stream it is
 * launched on (steps then issue eagerly, no CUDA graphs).  Enabling or
 * disabling clears the totals. */
int mm_cd_kernel_timing(mm_cd_engine* e, int on);
/* Totals since timing was enabled, one entry per kernel name: names[i]
 * (NUL-terminated), total_ms[i], launches[i] for i < min(cap, *n); *n = the
 * number of kernel names.  Any output array may be NULL. */
int mm_cd_kernel_times(mm_cd_engine* e, int cap, char (*names)[32], double* total_ms,
                       long long* launches, int* n);

/* CUDA stream (cudaStream_t) the engine launches on (launches a deferred
 * step epilogue first, see mm_cd_step). */
int mm_cd_stream(mm_cd_engine* e, void** stream);
/* Device pointer + byte size of the r z-planes of p_cur on one side:
 * side 0 = low z, 1 = high z; which 0 = owned edge planes (send),
 * 1 = ghost planes (receive).  The device layout is z slowest, so each
 * range is one contiguous block. */
int mm_cd_halo_planes(mm_cd_engine* e, int side, int which, void** dev_ptr, size_t* bytes);
/* Same for p_next (the field the current step is writing). */
int mm_cd_next_halo_planes(mm_cd_engine* e, int side, int which, void** dev_ptr, size_t* bytes);
/* Restricted step pieces for overlap: compute p_next on local planes
 * [z_lo, z_hi) only (both CPML passes and the inner update). */
int mm_cd_update_planes(mm_cd_engine* e, int z_lo, int z_hi);
/* Same on the union of n plane ranges [ranges[2i], ranges[2i+1]) (e.g. the
 * edge planes next to both cuts), with one launch per kernel. */
int mm_cd_update_plane_ranges(mm_cd_engine* e, const int* ranges, int n);

/* ------------------------------------------------------------------------
 * Multi-GPU z-slab group (ref: run_distributed_rank, dist.cpp:144-267, with
 * Cartesian dims {1, 1, P}; exchange_halos, dist.cpp:92-115).  One process
 * (rank) per GPU; the host runtime shares one NCCL unique id between the
 * ranks (e.g. a torch.distributed broadcast) and every rank creates its
 * group with it.  NCCL is loaded at run time (libnccl.so.2).
 * --------------------------------------------------------------------- */
typedef struct mm_cd_group mm_cd_group;

/* ncclGetUniqueId: 128 bytes for mm_cd_group_create (made by rank 0). */
int mm_nccl_get_unique_id(unsigned char id[128]);
/* ref: dist.cpp:119-132 validate_cuts for z cuts[world+1] (0 = cuts[0] <
 * ... < cuts[world] = nz): interior cuts at least ndamping_z + radius from
 * both faces, slabs at least radius planes thick.  MM_ECONFIG otherwise. */
int mm_zslab_validate_cuts(const int* cuts, int world, int nz, int ndamping_z, int radius);
/* One rank's slab [cuts[rank], cuts[rank+1]) of the global grid: its engine
 * (vp_local: the ghosted z-fastest slice of the global model, the
 * reference's vp_local, dist.cpp:171-180), the halo plan and the NCCL
 * communicator (ncclCommInitRank: a collective over all ranks).  nccl_id
 * NULL: no communicator (world == 1, or in-process ranks for
 * mm_cd_group_step_local). */
int mm_cd_group_create(const mm_grid* global, const int* cuts, int world, int rank,
                       const unsigned char nccl_id[128], const float* vp_local,
                       const mm_engine_options* opts, float dt, double vmax, int device, int mode,
                       mm_cd_group** out);
int mm_cd_group_destroy(mm_cd_group* g);
/* The rank's slab engine (owned by the group): receivers, pressure, traces,
 * stream.  Its local z = global z - z0. */
int mm_cd_group_engine(mm_cd_group* g, mm_cd_engine** e);
int mm_cd_group_slab(mm_cd_group* g, int* z0, int* nz);
/* One step on every rank (ref: exchange_halos + eng.step, dist.cpp:212-215):
 * CPML pass 1 -> the r planes next to each cut -> NCCL send/recv of those
 * planes into the neighbours' ghost planes on a communication stream,
 * overlapped with the interior planes -> join -> source (global coordinates;
 * the owning rank injects), free surface (rank 0), rotation.  Asynchronous
 * on the engine stream. */
int mm_cd_group_step(mm_cd_group* g, float amp, const int* src_global);
/* Test hook: one step of the ranks 0 .. n-1 of one decomposition created in
 * this process on one device without an NCCL id: the same schedule, with
 * device-to-device copies of the edge planes in place of NCCL and the ranks'
 * phases interleaved from this thread by stream events (no kernel waits on
 * another). */
int mm_cd_group_step_local(mm_cd_group** groups, int n, float amp, const int* src_global);
/* nsteps group steps with device amplitudes, receiver recording into columns
 * [first_sample, ...) when record != 0 (the rank's own receivers), and the
 * reference's per-rank finiteness check of the slab centre every step
 * (dist.cpp:222-224): MM_EINSTABILITY with the first failing step.
 * *device_ms: device time of this rank's loop. */
int mm_cd_group_run(mm_cd_group* g, const float* amps, int nsteps, const int* src_global,
                    int record, int first_sample, float* device_ms);

/* ------------------------------------------------------------------------
 * Driver (ref: driver.cpp:83-144 run(), acoustic_iso_cd only)
 * --------------------------------------------------------------------- */
typedef struct mm_sim_config {
    int ngrid[3];
    double dgrid[3];
    int nsteps;
    double fmax;
    double cfl;
    int ndamping[3];
    int ntaper[3];
    int taper;
    int free_surface;
    double r_target;
    int has_source_loc;
    int source_loc[3];
    int receiver_increment[2];
    int stencil_radius;
} mm_sim_config;

typedef struct mm_run_report {
    double dt;
    double kernel_seconds;   /* device time of the step loop */
    double modeling_seconds; /* wall time of the whole run */
    int steps_run;
    int nreceivers;
} mm_run_report;

/* Fills *cfg with the reference SimConfig defaults (driver.hpp:21-47). */
int mm_sim_config_default(mm_sim_config* cfg);
/* vp_model: ghosted z-fastest model (validated/replicated here).  traces:
 * nreceivers*nsteps floats (NULL to skip the copy-out); nreceivers of the
 * default carpet = ceil(nx/inc0)*ceil(ny/inc1). */
int mm_run(const mm_sim_config* cfg, const float* vp_model, int device, int mode, float* traces,
           mm_run_report* report);

/* ------------------------------------------------------------------------
 * acoustic_iso: the variable-density first-order engine, SURVEY.md §8(f)
 * row 4 (ref: AcousticVdEngine<float>, propagator.hpp:147-176, implemented at
 * propagator_impl.hpp:175-295; driven by run(), driver.cpp:122-128).
 * Same conventions as the acoustic_iso_cd engine above: host fields in the
 * reference layout, every call asynchronous on the engine stream except the
 * ones returning host data.  Arithmetic is the reference's association order
 * (bit-identical results); there is one kernel family.
 * --------------------------------------------------------------------- */
typedef struct mm_vd_engine mm_vd_engine;

/* ref: stencil.cpp:76-97 staggered_first_derivative_coeffs -> c[radius]. */
int mm_staggered_first_derivative_coeffs(int radius, double h, double* c);
/* ref: source.cpp:30-38 integrate_wavelet: out[s] = float(sum_{t<=s} w[t]*dt). */
int mm_integrate_wavelet(const float* w, int n, double dt, float* out);

/* ref: propagator_impl.hpp:175-212 ctor.  vp, rho: ghosted z-fastest model
 * volumes (validated and ghost-replicated, as EarthModel holds them; copied).
 * rho == NULL is the reference's "acoustic_iso requires a density volume"
 * ValidationError.  vmax: the model's vmax (feeds the CPML profile). */
int mm_vd_create(const mm_grid* grid, const float* vp, const float* rho,
                 const mm_engine_options* opts, float dt, double vmax, int device,
                 mm_vd_engine** out);
int mm_vd_destroy(mm_vd_engine* e);
/* ref: propagator.hpp:154-155 step(amp, src); amp is the time-integrated
 * wavelet sample; src: 3 interior coordinates or NULL. */
int mm_vd_step(mm_vd_engine* e, float amp, const int* src);
/* Sub-phases of one step in the reference order (propagator_impl.hpp:275-295). */
int mm_vd_update_velocity(mm_vd_engine* e);  /* update_velocity, :214-244 */
int mm_vd_update_pressure(mm_vd_engine* e);  /* update_pressure, :246-273 */
int mm_vd_inject_source(mm_vd_engine* e, float amp, const int* src); /* :287-291 */
int mm_vd_apply_free_surface(mm_vd_engine* e);                       /* :292 */
int mm_vd_synchronize(mm_vd_engine* e);
int mm_vd_field_size(mm_vd_engine* e, size_t* count);
int mm_vd_get_dt(mm_vd_engine* e, float* dt);
int mm_vd_steps_taken(mm_vd_engine* e, long long* steps);
/* ref: propagator.hpp:157-158 pressure() / velocity(axis): copies out
 * (reference layout, ghosts included); set_* replace the device state (the
 * reference hands out mutable references). */
int mm_vd_get_pressure(mm_vd_engine* e, float* host);
int mm_vd_get_velocity(mm_vd_engine* e, int axis, float* host);
int mm_vd_set_pressure(mm_vd_engine* e, const float* host);
int mm_vd_set_velocity(mm_vd_engine* e, int axis, const float* host);
/* Receivers and the device-resident loop: as mm_cd_set_receivers /
 * mm_cd_record / mm_cd_get_traces / mm_cd_copy_trace_step / mm_cd_run. */
int mm_vd_set_receivers(mm_vd_engine* e, const int* ijk, int nreceivers, int capacity);
int mm_vd_record(mm_vd_engine* e, int step);
int mm_vd_get_traces(mm_vd_engine* e, float* host, int nsteps);
int mm_vd_copy_trace_step(mm_vd_engine* e, int step, float* host, int async);
int mm_vd_run(mm_vd_engine* e, const float* amps, int nsteps, const int* src, int record,
              int first_sample, float* device_ms);
int mm_vd_stream(mm_vd_engine* e, void** stream);
/* ref: driver.cpp:83-144 run() with Propagator::AcousticIso: integrated
 * Ricker source, default receiver carpet, per-step receiver-0 finiteness
 * check.  vp_model, rho_model: ghosted z-fastest (validated / replicated
 * here). */
int mm_run_vd(const mm_sim_config* cfg, const float* vp_model, const float* rho_model,
              int device, float* traces, mm_run_report* report);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* MINIMOD_B200_H */
