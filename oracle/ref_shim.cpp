// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY.  oracle/build_ref.sh compiles this file together
// with the reference's own translation units from /root/reference/proj/core
// (no reference source is copied into this repo) into
// oracle/_ref/libminimod_ref.so.  It is used to pin the C restatement
// (oracle/minimod_oracle.c) and as the "reference" CPU baseline in bench.py.
// The shim only marshals arguments; every number comes from the reference's
// AcousticCdEngine<float> (propagator_impl.hpp:53-173), AcousticVdEngine<float>
// (propagator_impl.hpp:175-295) and run() (driver.cpp:83-144).
#include <cstring>
#include <exception>
#include <string>

#include "minimod/driver.hpp"
#include "minimod/model.hpp"
#include "minimod/source.hpp"
#include "minimod/propagator.hpp"

using namespace minimod;

namespace {
thread_local std::string g_err;
int catch_all() {
    try {
        throw;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 2;
    } catch (const InstabilityError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_second_derivative_coeffs(int radius, double h, double* c, double* center) {
    try {
        const StencilCoeffs s = second_derivative_coeffs(radius, h);
        for (int m = 0; m < radius; ++m) c[m] = s.c[m];
        *center = s.center;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

int ref_central_first_derivative_coeffs(int radius, double h, double* c) {
    try {
        const StencilCoeffs s = central_first_derivative_coeffs(radius, h);
        for (int m = 0; m < radius; ++m) c[m] = s.c[m];
        return 0;
    } catch (...) {
        return catch_all();
    }
}

int ref_ricker(double fmax, double dt, int nsteps, float* out) {
    try {
        const Wavelet w = ricker(fmax, dt, nsteps);
        std::memcpy(out, w.samples.data(), sizeof(float) * nsteps);
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// vp: ghosted z-fastest model of size n (validated + ghost-replicated here
// through validate_model, model.cpp:15-43).
static EarthModel make_model(const int n[3], const double d[3], int radius, const float* vp) {
    EarthModel m;
    m.grid = make_grid({n[0], n[1], n[2]}, {d[0], d[1], d[2]}, radius);
    m.vp = Field(m.grid, "vp");
    std::memcpy(m.vp.data.data(), vp, sizeof(float) * m.vp.data.size());
    validate_model(m);
    return m;
}

int ref_cfl_dt(const int n[3], const double d[3], int radius, const float* vp, double cfl,
               double* dt, float* vmin, float* vmax) {
    try {
        const EarthModel m = make_model(n, d, radius, vp);
        *dt = cfl_dt(m, m.grid, cfl);
        if (vmin) *vmin = m.vmin;
        if (vmax) *vmax = m.vmax;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

int ref_layered_model(const int n[3], const double d[3], int radius, float* vp, float* vmin,
                      float* vmax) {
    try {
        const EarthModel m =
            default_layered_model(make_grid({n[0], n[1], n[2]}, {d[0], d[1], d[2]}, radius));
        std::memcpy(vp, m.vp.data.data(), sizeof(float) * m.vp.data.size());
        *vmin = m.vmin;
        *vmax = m.vmax;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// minimod::run() on a given vp model (traces[r*nsteps+s]); nthreads > 1
// selects Target::Parallel.
int ref_run(const int n[3], const double d[3], int radius, int nsteps, double fmax, double cfl,
            const int ndamping[3], const int ntaper[3], int taper, int free_surface,
            double r_target, const int* src_loc, const float* vp, int nthreads, float* traces,
            double* dt_out, double* kernel_seconds, double* modeling_seconds) {
    try {
        const EarthModel m = make_model(n, d, radius, vp);
        SimConfig c;
        c.ngrid = {n[0], n[1], n[2]};
        c.dgrid = {d[0], d[1], d[2]};
        c.stencil_radius = radius;
        c.nsteps = nsteps;
        c.fmax = fmax;
        c.cfl = cfl;
        c.ndamping = {ndamping[0], ndamping[1], ndamping[2]};
        c.ntaper = {ntaper[0], ntaper[1], ntaper[2]};
        c.taper = taper != 0;
        c.free_surface = free_surface != 0;
        c.r_target = r_target;
        if (src_loc) c.source_loc = std::array<int, 3>{src_loc[0], src_loc[1], src_loc[2]};
        c.target = nthreads > 1 ? Target::Parallel : Target::Seq;
        c.nthreads = nthreads > 1 ? nthreads : 1;
        const auto [rec, rep] = run(c, m);
        if (traces) std::memcpy(traces, rec.traces.data(), sizeof(float) * rec.traces.size());
        if (dt_out) *dt_out = rep.dt;
        if (kernel_seconds) *kernel_seconds = rep.kernel_seconds;
        if (modeling_seconds) *modeling_seconds = rep.modeling_seconds;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

static EarthModel make_vd_model(const int n[3], const double d[3], int radius, const float* vp,
                                const float* rho);

struct ref_engine {
    AcousticCdEngine<float>* eng;
    int nthreads;
};

int ref_engine_create(const int n_local[3], const double d[3], int radius, const int offset[3],
                      const int global_n[3], const float* vp_local, const int ndamping[3],
                      double fmax, double r_target, int free_surface, int taper,
                      const int ntaper[3], float dt, double vmax_global, int nthreads,
                      ref_engine** out) {
    try {
        const Grid3D g = make_grid({n_local[0], n_local[1], n_local[2]}, {d[0], d[1], d[2]},
                                   radius);
        Field vp(g, "vp");
        std::memcpy(vp.data.data(), vp_local, sizeof(float) * vp.data.size());
        EngineOptions o;
        o.ndamping = {ndamping[0], ndamping[1], ndamping[2]};
        o.fmax = fmax;
        o.r_target = r_target;
        o.free_surface = free_surface != 0;
        o.taper = taper != 0;
        o.ntaper = {ntaper[0], ntaper[1], ntaper[2]};
        auto* e = new ref_engine;
        e->eng = new AcousticCdEngine<float>(g, {offset[0], offset[1], offset[2]},
                                             {global_n[0], global_n[1], global_n[2]}, vp, o, dt,
                                             vmax_global);
        e->nthreads = nthreads < 1 ? 1 : nthreads;
        *out = e;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

void ref_engine_destroy(ref_engine* e) {
    if (!e) return;
    delete e->eng;
    delete e;
}

int ref_engine_step(ref_engine* e, float amp, const int* src) {
    try {
        std::optional<std::array<int, 3>> s;
        if (src) s = std::array<int, 3>{src[0], src[1], src[2]};
        e->eng->step(amp, s, TaskRunner(e->nthreads));
        return 0;
    } catch (...) {
        return catch_all();
    }
}

float* ref_engine_pressure(ref_engine* e) { return e->eng->pressure().data.data(); }
float* ref_engine_pressure_prev(ref_engine* e) { return e->eng->pressure_prev().data.data(); }

float* ref_engine_profile(ref_engine* e, int which, int axis) {
    auto& A = e->eng->profile().axis[axis];
    return which == 0 ? A.a.data() : which == 1 ? A.b.data() : A.inv_kappa.data();
}
double ref_engine_d0(ref_engine* e, int axis) { return e->eng->profile().d0[axis]; }

int ref_engine_set_state(ref_engine* e, const float* p_prev, const float* p_cur) {
    try {
        Field a(e->eng->grid(), "p_prev"), b(e->eng->grid(), "p_cur");
        std::memcpy(a.data.data(), p_prev, sizeof(float) * a.data.size());
        std::memcpy(b.data.data(), p_cur, sizeof(float) * b.data.size());
        e->eng->set_state(a, b);
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// Tapered copy of a ghosted vp field (propagator.hpp:36-62), in place.
int ref_taper_material(float* f, const int n[3], int radius, const int ntaper[3],
                       const int offset[3], const int global_n[3]) {
    try {
        const Grid3D g = make_grid({n[0], n[1], n[2]}, {1.0, 1.0, 1.0}, radius);
        Field fld(g, "vp");
        std::memcpy(fld.data.data(), f, sizeof(float) * fld.data.size());
        detail::taper_material(fld, {ntaper[0], ntaper[1], ntaper[2]},
                               {offset[0], offset[1], offset[2]},
                               {global_n[0], global_n[1], global_n[2]});
        std::memcpy(f, fld.data.data(), sizeof(float) * fld.data.size());
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// ---- on-disk formats and the report (driver.cpp:150-215, source.cpp:68-95,
//      model.cpp:80-190): used to pin the repo's writers / parsers byte-wise.
int ref_save_record(const float* traces, int nrec, int nsteps, double dt, const int source_loc[3],
                    const int receiver_increment[2], int nshots, const char* path) {
    try {
        AcquisitionGeometry g;
        g.source_loc = {source_loc[0], source_loc[1], source_loc[2]};
        g.receiver_increment = {receiver_increment[0], receiver_increment[1]};
        g.nshots = nshots;
        g.receivers.assign(static_cast<std::size_t>(nrec), std::array<int, 3>{0, 0, 0});
        ShotRecord r = make_record(g, nsteps, dt);
        std::memcpy(r.traces.data(), traces, sizeof(float) * r.traces.size());
        save_record(r, path);
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// vp: ghosted z-fastest field of a grid with stencil radius `radius`
int ref_save_model(const int n[3], const double d[3], int radius, const float* vp,
                   const char* manifest) {
    try {
        const EarthModel m = make_model(n, d, radius, vp);
        save_model(m, manifest);
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// n, d of the manifest; vp (optional) receives the ghosted field of radius 4
// (make_grid's default), vmin / vmax as validate_model computed them
int ref_load_model(const char* manifest, int n[3], double d[3], float* vp, float* vmin,
                   float* vmax) {
    try {
        const EarthModel m = load_model(manifest);
        for (int a = 0; a < 3; ++a) {
            n[a] = m.grid.n[a];
            d[a] = m.grid.d[a];
        }
        if (vp) std::memcpy(vp, m.vp.data.data(), sizeof(float) * m.vp.data.size());
        *vmin = m.vmin;
        *vmax = m.vmax;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// save_model of a model with a density volume (rho.f32 next to vp.f32)
int ref_save_model_rho(const int n[3], const double d[3], int radius, const float* vp,
                       const float* rho, const char* manifest) {
    try {
        const EarthModel m = make_vd_model(n, d, radius, vp, rho);
        save_model(m, manifest);
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// rho of a loaded manifest (ghosted, radius 4); *has = 0 when it lists none
int ref_load_model_rho(const char* manifest, float* rho, int* has) {
    try {
        const EarthModel m = load_model(manifest);
        *has = m.rho.has_value() ? 1 : 0;
        if (m.rho && rho) std::memcpy(rho, m.rho->data.data(), sizeof(float) * m.rho->data.size());
        return 0;
    } catch (...) {
        return catch_all();
    }
}

int ref_render_report(const int ngrid[3], const double dgrid[3], int nsteps, double fmax,
                      double cfl, int radius, const int ndamping[3], const int ntaper[3],
                      const int* source_loc, const int receiver_increment[2],
                      const int source_increment[3], int nshots, double time_rec, int nthreads,
                      float vmin, float vmax, double kernel_s, double modeling_s, char* out,
                      int cap) {
    try {
        SimConfig c;
        c.ngrid = {ngrid[0], ngrid[1], ngrid[2]};
        c.dgrid = {dgrid[0], dgrid[1], dgrid[2]};
        c.nsteps = nsteps;
        c.fmax = fmax;
        c.cfl = cfl;
        c.stencil_radius = radius;
        c.ndamping = {ndamping[0], ndamping[1], ndamping[2]};
        c.ntaper = {ntaper[0], ntaper[1], ntaper[2]};
        if (source_loc) c.source_loc = std::array<int, 3>{source_loc[0], source_loc[1], source_loc[2]};
        c.receiver_increment = {receiver_increment[0], receiver_increment[1]};
        c.source_increment = {source_increment[0], source_increment[1], source_increment[2]};
        c.nshots = nshots;
        c.time_rec = time_rec;
        c.target = nthreads > 1 ? Target::Parallel : Target::Seq;
        c.nthreads = nthreads > 1 ? nthreads : 1;
        EarthModel m;
        m.vmin = vmin;
        m.vmax = vmax;
        RunReport rep;
        rep.kernel_seconds = kernel_s;
        rep.modeling_seconds = modeling_s;
        const std::string s = render_parameter_block(c, m) + render_timing(rep);
        if ((int)s.size() + 1 > cap) throw std::invalid_argument("report buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// ---------------------------------------------------------------- acoustic_iso
// The variable-density engine AcousticVdEngine<float> (propagator_impl.hpp:
// 175-295), its weights (stencil.cpp:76-97) and source (source.cpp:30-38), and
// run() with Propagator::AcousticIso (driver.cpp:122-128).

int ref_staggered_first_derivative_coeffs(int radius, double h, double* c) {
    try {
        const StencilCoeffs s = staggered_first_derivative_coeffs(radius, h);
        for (int m = 0; m < radius; ++m) c[m] = s.c[m];
        return 0;
    } catch (...) {
        return catch_all();
    }
}

int ref_integrate_wavelet(const float* w, int n, double dt, float* out) {
    try {
        Wavelet in;
        in.dt = dt;
        in.samples.assign(w, w + n);
        const Wavelet o = integrate_wavelet(in);
        std::memcpy(out, o.samples.data(), sizeof(float) * n);
        return 0;
    } catch (...) {
        return catch_all();
    }
}

// vp, rho: ghosted z-fastest (validated + ghost-replicated by validate_model);
// rho may be NULL (the engine then rejects the model).
static EarthModel make_vd_model(const int n[3], const double d[3], int radius, const float* vp,
                                const float* rho) {
    EarthModel m;
    m.grid = make_grid({n[0], n[1], n[2]}, {d[0], d[1], d[2]}, radius);
    m.vp = Field(m.grid, "vp");
    std::memcpy(m.vp.data.data(), vp, sizeof(float) * m.vp.data.size());
    if (rho) {
        m.rho = Field(m.grid, "rho");
        std::memcpy(m.rho->data.data(), rho, sizeof(float) * m.rho->data.size());
    }
    validate_model(m);
    return m;
}

struct ref_vd {
    AcousticVdEngine<float>* eng;
    int nthreads;
};

int ref_vd_create(const int n[3], const double d[3], int radius, const float* vp,
                  const float* rho, const int ndamping[3], double fmax, double r_target,
                  int free_surface, int taper, const int ntaper[3], float dt, int nthreads,
                  ref_vd** out) {
    try {
        const EarthModel m = make_vd_model(n, d, radius, vp, rho);
        EngineOptions o;
        o.ndamping = {ndamping[0], ndamping[1], ndamping[2]};
        o.fmax = fmax;
        o.r_target = r_target;
        o.free_surface = free_surface != 0;
        o.taper = taper != 0;
        o.ntaper = {ntaper[0], ntaper[1], ntaper[2]};
        auto* e = new ref_vd;
        e->eng = nullptr;
        e->nthreads = nthreads < 1 ? 1 : nthreads;
        try {
            e->eng = new AcousticVdEngine<float>(m.grid, m, o, dt);
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

void ref_vd_destroy(ref_vd* e) {
    if (!e) return;
    delete e->eng;
    delete e;
}

int ref_vd_step(ref_vd* e, float amp, const int* src) {
    try {
        std::optional<std::array<int, 3>> s;
        if (src) s = std::array<int, 3>{src[0], src[1], src[2]};
        e->eng->step(amp, s, TaskRunner(e->nthreads));
        return 0;
    } catch (...) {
        return catch_all();
    }
}

float* ref_vd_pressure(ref_vd* e) { return e->eng->pressure().data.data(); }
float* ref_vd_velocity(ref_vd* e, int axis) { return e->eng->velocity(axis).data.data(); }

// run() with Propagator::AcousticIso (traces[r*nsteps+s]).
int ref_run_vd(const int n[3], const double d[3], int radius, int nsteps, double fmax,
               double cfl, const int ndamping[3], const int ntaper[3], int taper,
               int free_surface, double r_target, const int* src_loc, const float* vp,
               const float* rho, int nthreads, float* traces, double* dt_out,
               double* kernel_seconds, double* modeling_seconds) {
    try {
        const EarthModel m = make_vd_model(n, d, radius, vp, rho);
        SimConfig c;
        c.propagator = Propagator::AcousticIso;
        c.ngrid = {n[0], n[1], n[2]};
        c.dgrid = {d[0], d[1], d[2]};
        c.stencil_radius = radius;
        c.nsteps = nsteps;
        c.fmax = fmax;
        c.cfl = cfl;
        c.ndamping = {ndamping[0], ndamping[1], ndamping[2]};
        c.ntaper = {ntaper[0], ntaper[1], ntaper[2]};
        c.taper = taper != 0;
        c.free_surface = free_surface != 0;
        c.r_target = r_target;
        if (src_loc) c.source_loc = std::array<int, 3>{src_loc[0], src_loc[1], src_loc[2]};
        c.target = nthreads > 1 ? Target::Parallel : Target::Seq;
        c.nthreads = nthreads > 1 ? nthreads : 1;
        const auto [rec, rep] = run(c, m);
        if (traces) std::memcpy(traces, rec.traces.data(), sizeof(float) * rec.traces.size());
        if (dt_out) *dt_out = rep.dt;
        if (kernel_seconds) *kernel_seconds = rep.kernel_seconds;
        if (modeling_seconds) *modeling_seconds = rep.modeling_seconds;
        return 0;
    } catch (...) {
        return catch_all();
    }
}

}  // extern "C"
