// minimod_b200.hpp -- header-only C++ drop-in over the C ABI (minimod_b200.h).
//
// AcousticVdEngine (acoustic_iso) follows at the end.  AcousticCdEngine has
// the same shape as the reference's minimod::AcousticCdEngine<float>
// (propagator.hpp:93-140): construct from a ghosted z-fastest vp field,
// step(amp, src), pressure(), pressure_prev(), set_state(), profile().  Status
// codes are rethrown as the reference's exception types (errors.hpp:10-30).
// pressure()/pressure_prev() return host mirrors synchronised on demand; a
// caller that records receivers every step should use set_receivers()/run()
// (device-side recording) instead of reading the whole field per step.
#pragma once

#include <array>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "minimod_b200.h"

namespace minimod_b200 {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InstabilityError : std::runtime_error {
    InstabilityError(const std::string& m, int s) : std::runtime_error(m), step_(s) {}
    int step() const { return step_; }

private:
    int step_;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == MM_OK) return;
    const std::string msg = mm_last_error();
    switch (rc) {
        case MM_ECONFIG: throw ConfigError(msg);
        case MM_EVALIDATION: throw ValidationError(msg);
        case MM_EINSTABILITY: throw InstabilityError(msg, mm_last_instability_step());
        case MM_EINVAL: throw std::invalid_argument(msg);
        default: throw DeviceError(msg);
    }
}

struct EngineOptions {  // ref: propagator.hpp:23-30
    std::array<int, 3> ndamping{0, 0, 0};
    double fmax = 25.0;
    double r_target = 1e-3;
    bool free_surface = false;
    bool taper = false;
    std::array<int, 3> ntaper{3, 3, 3};
};

struct Grid {  // ref: grid.hpp:49-73
    std::array<int, 3> n{0, 0, 0};
    std::array<double, 3> d{0, 0, 0};
    int radius = 4;
    size_t volume() const {
        return (size_t)(n[0] + 2 * radius) * (n[1] + 2 * radius) * (n[2] + 2 * radius);
    }
};

struct AxisCpml {
    std::vector<float> a, b, inv_kappa;
};

class AcousticCdEngine {
public:
    AcousticCdEngine(const Grid& g, std::array<int, 3> offset, std::array<int, 3> global_n,
                     const std::vector<float>& vp_local, const EngineOptions& o, float dt,
                     double vmax_global, int device = 0, int mode = MM_MODE_FAST)
        : grid_(g), global_n_(global_n) {
        if (vp_local.size() != g.volume())
            throw std::invalid_argument("vp_local size does not match the ghosted grid");
        mm_grid cg{{g.n[0], g.n[1], g.n[2]}, {g.d[0], g.d[1], g.d[2]}, g.radius};
        mm_engine_options co{{o.ndamping[0], o.ndamping[1], o.ndamping[2]},
                             o.fmax,
                             o.r_target,
                             o.free_surface ? 1 : 0,
                             o.taper ? 1 : 0,
                             {o.ntaper[0], o.ntaper[1], o.ntaper[2]}};
        check(mm_cd_create(&cg, offset.data(), global_n.data(), vp_local.data(), &co, dt,
                           vmax_global, device, mode, &h_));
    }
    ~AcousticCdEngine() {
        if (h_) mm_cd_destroy(h_);
    }
    AcousticCdEngine(const AcousticCdEngine&) = delete;
    AcousticCdEngine& operator=(const AcousticCdEngine&) = delete;

    // ref: propagator.hpp:103-104 (the TaskRunner argument has no GPU meaning)
    void step(float amp, std::optional<std::array<int, 3>> src) {
        check(mm_cd_step(h_, amp, src ? src->data() : nullptr));
    }

    std::vector<float> pressure() const { return fetch(mm_cd_get_pressure); }
    std::vector<float> pressure_prev() const { return fetch(mm_cd_get_pressure_prev); }
    void set_state(const std::vector<float>& p_prev, const std::vector<float>& p_cur) {
        check(mm_cd_set_state(h_, p_prev.data(), p_cur.data()));
    }
    const Grid& grid() const { return grid_; }
    float dt() const {
        float v = 0;
        check(mm_cd_get_dt(h_, &v));
        return v;
    }
    std::array<AxisCpml, 3> profile() const {
        std::array<AxisCpml, 3> p;
        for (int ax = 0; ax < 3; ++ax) {
            p[ax].a.resize(global_n_[ax]);
            p[ax].b.resize(global_n_[ax]);
            p[ax].inv_kappa.resize(global_n_[ax]);
            check(mm_cd_get_profile(h_, ax, p[ax].a.data(), p[ax].b.data(),
                                    p[ax].inv_kappa.data()));
        }
        return p;
    }
    void set_profile(const std::array<AxisCpml, 3>& p) {
        for (int ax = 0; ax < 3; ++ax)
            check(mm_cd_set_profile(h_, ax, p[ax].a.data(), p[ax].b.data(),
                                    p[ax].inv_kappa.data()));
    }
    mm_cd_engine* handle() { return h_; }

private:
    template <typename F>
    std::vector<float> fetch(F fn) const {
        std::vector<float> out(grid_.volume());
        check(fn(h_, out.data()));
        return out;
    }
    Grid grid_;
    std::array<int, 3> global_n_;
    mm_cd_engine* h_ = nullptr;
};

// ref: propagator.hpp:147-176 AcousticVdEngine<float> (acoustic_iso).  vp and
// rho are the model's ghosted z-fastest volumes; rho == nullptr reproduces the
// reference's ValidationError.  pressure()/velocity() return host copies; the
// reference's mutable references map to set_pressure()/set_velocity().
class AcousticVdEngine {
public:
    AcousticVdEngine(const Grid& g, const std::vector<float>& vp, const std::vector<float>* rho,
                     const EngineOptions& o, float dt, double vmax, int device = 0)
        : grid_(g) {
        if (vp.size() != g.volume() || (rho && rho->size() != g.volume()))
            throw std::invalid_argument("model volumes do not match the ghosted grid");
        mm_grid cg{{g.n[0], g.n[1], g.n[2]}, {g.d[0], g.d[1], g.d[2]}, g.radius};
        mm_engine_options co{{o.ndamping[0], o.ndamping[1], o.ndamping[2]},
                             o.fmax,
                             o.r_target,
                             o.free_surface ? 1 : 0,
                             o.taper ? 1 : 0,
                             {o.ntaper[0], o.ntaper[1], o.ntaper[2]}};
        check(mm_vd_create(&cg, vp.data(), rho ? rho->data() : nullptr, &co, dt, vmax, device,
                           &h_));
    }
    ~AcousticVdEngine() {
        if (h_) mm_vd_destroy(h_);
    }
    AcousticVdEngine(const AcousticVdEngine&) = delete;
    AcousticVdEngine& operator=(const AcousticVdEngine&) = delete;

    // ref: propagator.hpp:154-155 (amp: the time-integrated wavelet sample)
    void step(float amp, std::optional<std::array<int, 3>> src) {
        check(mm_vd_step(h_, amp, src ? src->data() : nullptr));
    }
    std::vector<float> pressure() const {
        std::vector<float> out(grid_.volume());
        check(mm_vd_get_pressure(h_, out.data()));
        return out;
    }
    std::vector<float> velocity(int axis) const {
        std::vector<float> out(grid_.volume());
        check(mm_vd_get_velocity(h_, axis, out.data()));
        return out;
    }
    void set_pressure(const std::vector<float>& p) { check(mm_vd_set_pressure(h_, p.data())); }
    void set_velocity(int axis, const std::vector<float>& v) {
        check(mm_vd_set_velocity(h_, axis, v.data()));
    }
    const Grid& grid() const { return grid_; }
    float dt() const {
        float v = 0;
        check(mm_vd_get_dt(h_, &v));
        return v;
    }
    mm_vd_engine* handle() { return h_; }

private:
    Grid grid_;
    mm_vd_engine* h_ = nullptr;
};

}  // namespace minimod_b200
