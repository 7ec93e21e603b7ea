// dropin_driver.cpp -- the INTEGRATION.md binding compiled and run as a C++
// host: one SimConfig through the reference's own run() (driver.cpp:83-144,
// compiled unmodified from /root/reference by oracle/build_dropin.sh) and
// through the drop-in path a maintainer would put in driver.cpp:116-121
// (minimod_b200::AcousticCdEngine over the C ABI, device-side receivers),
// plus the one-call device loop mm_run().  Prints one JSON line and exits 0
// when every trace matrix is bit-identical to the reference's.
//
// TEST INFRASTRUCTURE: links the reference objects only to compare against
// them (tests/test_gpu_dropin.py runs it on the GPU box).
//
// usage: dropin_driver [n] [nsteps] [free_surface 0|1]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "minimod/driver.hpp"
#include "minimod/model.hpp"
#include "minimod/source.hpp"
#include "minimod_b200.hpp"

namespace {

struct Cmp {
    bool equal = true;
    double rel_l2 = 0.0, max_abs = 0.0;
};

Cmp compare(const std::vector<float>& got, const std::vector<float>& want) {
    Cmp c;
    if (got.size() != want.size()) {
        c.equal = false;
        c.rel_l2 = c.max_abs = INFINITY;
        return c;
    }
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < got.size(); ++i) {
        const double d = (double)got[i] - (double)want[i];
        num += d * d;
        den += (double)want[i] * want[i];
        c.max_abs = std::fmax(c.max_abs, std::fabs(d));
        if (got[i] != want[i]) c.equal = false;
    }
    c.rel_l2 = std::sqrt(num) / std::fmax(std::sqrt(den), 1e-300);
    return c;
}

}  // namespace

int main(int argc, char** argv) {
    using namespace minimod;
    const int n = argc > 1 ? std::atoi(argv[1]) : 64;
    const int nsteps = argc > 2 ? std::atoi(argv[2]) : 200;
    const bool fs = argc > 3 && std::atoi(argv[3]) != 0;

    SimConfig config;
    config.ngrid = {n, n, n};
    config.nsteps = nsteps;
    config.ndamping = {std::min(27, n / 4), std::min(27, n / 4), std::min(27, n / 4)};
    config.free_surface = fs;
    config.target = Target::Parallel;
    config.nthreads = 8;
    const Grid3D grid = make_grid(config.ngrid, config.dgrid, config.stencil_radius);
    const EarthModel model = default_layered_model(grid);

    // ---- the reference's own run()
    auto [ref, ref_rep] = run(config, model);

    // ---- the drop-in ("C++ binding a maintainer would add"):
    // the setup of driver.cpp:88-115, then the engine behind the C ABI
    const double dt = cfl_dt(model, grid, config.cfl);
    const Wavelet w = ricker(config.fmax, dt, config.nsteps);
    const AcquisitionGeometry geometry = build_geometry(config, grid);
    EngineOptions opts;
    opts.ndamping = config.ndamping;
    opts.fmax = config.fmax;
    opts.r_target = config.r_target;
    opts.free_surface = config.free_surface;
    opts.taper = config.taper;
    opts.ntaper = config.ntaper;
    std::vector<float> traces((size_t)geometry.nreceivers() * nsteps);
    const auto t0 = std::chrono::steady_clock::now();
    {
        minimod_b200::Grid g{grid.n, grid.d, grid.radius};
        minimod_b200::EngineOptions o{opts.ndamping, opts.fmax, opts.r_target,
                                      opts.free_surface, opts.taper, opts.ntaper};
        minimod_b200::AcousticCdEngine eng(g, {0, 0, 0}, grid.n, model.vp.data, o,
                                           static_cast<float>(dt), model.vmax);
        std::vector<int> ijk;
        for (const auto& r : geometry.receivers) ijk.insert(ijk.end(), r.begin(), r.end());
        minimod_b200::check(
            mm_cd_set_receivers(eng.handle(), ijk.data(), geometry.nreceivers(), nsteps));
        const std::array<int, 3> src = geometry.source_loc;
        for (int s = 0; s < nsteps; ++s) {
            eng.step(w.samples[s], src);                         // was eng.step(w, src, runner)
            minimod_b200::check(mm_cd_record(eng.handle(), s));  // was record(eng.pressure(), ..)
        }
        minimod_b200::check(mm_cd_get_traces(eng.handle(), traces.data(), nsteps));
    }
    const double t_dropin =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    // ---- the one-call device loop
    mm_sim_config cfg;
    minimod_b200::check(mm_sim_config_default(&cfg));
    for (int a = 0; a < 3; ++a) {
        cfg.ngrid[a] = n;
        cfg.ndamping[a] = config.ndamping[a];
    }
    cfg.nsteps = nsteps;
    cfg.free_surface = fs ? 1 : 0;
    std::vector<float> traces_run(traces.size());
    mm_run_report rep{};
    minimod_b200::check(
        mm_run(&cfg, model.vp.data.data(), 0, MM_MODE_FAST, traces_run.data(), &rep));

    const Cmp a = compare(traces, ref.traces), b = compare(traces_run, ref.traces);
    const bool ok = a.equal && b.equal && rep.dt == ref_rep.dt;
    std::printf(
        "{\"n\": %d, \"nsteps\": %d, \"free_surface\": %d, \"nreceivers\": %d, "
        "\"dropin\": {\"bitwise\": %s, \"rel_l2\": %.3e, \"max_abs\": %.3e, \"seconds\": %.3f}, "
        "\"mm_run\": {\"bitwise\": %s, \"rel_l2\": %.3e, \"max_abs\": %.3e, \"kernel_s\": %.4f}, "
        "\"reference\": {\"kernel_s\": %.3f, \"dt\": %.10g}, \"ok\": %s}\n",
        n, nsteps, fs ? 1 : 0, geometry.nreceivers(), a.equal ? "true" : "false", a.rel_l2,
        a.max_abs, t_dropin, b.equal ? "true" : "false", b.rel_l2, b.max_abs,
        rep.kernel_seconds, ref_rep.kernel_seconds, ref_rep.dt, ok ? "true" : "false");
    return ok ? 0 : 1;
}
