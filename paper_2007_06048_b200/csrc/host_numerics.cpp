// host_numerics.cpp -- setup-time numerics of the acoustic_iso_cd path.
//
// Each routine reproduces the reference's arithmetic bit for bit (same
// precision per operation, same association order), which the parity tests
// check against the reference build (tests/test_host_numerics.py):
//   second_derivative / central_first_derivative  ref: stencil.cpp:9-31,50-74,99-117
//   staggered_first_derivative                    ref: stencil.cpp:76-97
//   integrate_wavelet                             ref: source.cpp:30-38
//   cfl_dt                                        ref: driver.cpp:19-29
//   ricker                                        ref: source.cpp:11-28
//   build_profile                                 ref: cpml.hpp:34-72
//   taper_material                                ref: propagator.hpp:36-62
//   fill_ghosts_replicate / validate_vp           ref: grid.hpp:96-108, model.cpp:15-43
// This file is compiled with -ffp-contract=off so no FMA is formed.
#include <algorithm>
#include <cmath>
#include <limits>

#include "mm_internal.hpp"

namespace mmb {

namespace {

void require_stencil(int radius, double h) {
    if (radius < 1 || radius > 8)
        raise(ST_CONFIG, "stencil radius must be in [1, 8], got " + std::to_string(radius));
    if (!(h > 0.0)) raise(ST_CONFIG, "stencil spacing must be > 0");
}

// Taylor-matching system for symmetric (odd = false) or antisymmetric
// (odd = true) taps on unit spacing: row k demands that the taps reproduce
// the 2k-th (resp. (2k-1)-th) derivative of x^q exactly.  Nodes sit at x = m
// (collocated) or x = m - 1/2 (staggered).
std::vector<double> taylor_solve(int radius, bool odd, bool staggered = false) {
    const int n = radius;
    std::vector<long double> A(static_cast<size_t>(n) * n), rhs(n, 0.0L);
    rhs[0] = 1.0L;
    for (int k = 1; k <= n; ++k) {
        const int q = odd ? 2 * k - 1 : 2 * k;
        long double qfact = 1;
        for (int f = 2; f <= q; ++f) qfact *= f;
        for (int m = 1; m <= n; ++m)
            A[(k - 1) * n + (m - 1)] =
                2.0L * powl(staggered ? static_cast<long double>(m) - 0.5L
                                      : static_cast<long double>(m),
                            q) /
                qfact;
    }
    // Forward elimination, partial pivoting on double-rounded magnitudes.
    for (int col = 0; col < n; ++col) {
        int best = col;
        for (int row = col + 1; row < n; ++row) {
            const double cand = std::fabs(static_cast<double>(A[row * n + col]));
            if (cand > std::fabs(static_cast<double>(A[best * n + col]))) best = row;
        }
        if (best != col) {
            for (int c = 0; c < n; ++c) std::swap(A[col * n + c], A[best * n + c]);
            std::swap(rhs[col], rhs[best]);
        }
        for (int row = col + 1; row < n; ++row) {
            const long double f = A[row * n + col] / A[col * n + col];
            for (int c = col; c < n; ++c) A[row * n + c] -= f * A[col * n + c];
            rhs[row] -= f * rhs[col];
        }
    }
    std::vector<double> x(n, 0.0);
    for (int row = n - 1; row >= 0; --row) {
        long double acc = rhs[row];
        for (int c = row + 1; c < n; ++c) acc -= A[row * n + c] * x[c];
        x[row] = static_cast<double>(acc / A[row * n + row]);
    }
    return x;
}

}  // namespace

Coeffs second_derivative(int radius, double h) {
    require_stencil(radius, h);
    Coeffs out;
    out.c = taylor_solve(radius, false);
    double sum = 0.0;
    for (double& v : out.c) {
        v /= h * h;
        sum += v;
    }
    out.center = -2.0 * sum;
    return out;
}

Coeffs central_first_derivative(int radius, double h) {
    require_stencil(radius, h);
    Coeffs out;
    out.c = taylor_solve(radius, true);
    for (double& v : out.c) v /= h;
    return out;
}

Coeffs staggered_first_derivative(int radius, double h) {
    require_stencil(radius, h);
    Coeffs out;
    out.c = taylor_solve(radius, true, true);
    for (double& v : out.c) v /= h;
    return out;
}

std::vector<float> integrate_wavelet(const std::vector<float>& w, double dt) {
    std::vector<float> out(w.size());
    double acc = 0.0;
    for (size_t s = 0; s < w.size(); ++s) {
        acc += static_cast<double>(w[s]) * dt;
        out[s] = static_cast<float>(acc);
    }
    return out;
}

double cfl_dt(double vmax, const int n[3], const double d[3], int radius, double cfl) {
    (void)n;
    if (!(cfl > 0.0 && cfl <= 1.0)) raise(ST_CONFIG, "cfl must be in (0, 1]");
    double sum = 0.0;
    for (int ax = 0; ax < 3; ++ax) {
        const Coeffs s = second_derivative(radius, d[ax]);
        double row = std::fabs(s.center);
        for (double v : s.c) row += 2.0 * std::fabs(v);
        sum += row;
    }
    return cfl * 2.0 / (vmax * std::sqrt(sum));
}

std::vector<float> ricker(double fmax, double dt, int nsteps) {
    if (!(fmax > 0.0)) raise(ST_CONFIG, "fmax must be > 0");
    if (!(dt > 0.0)) raise(ST_CONFIG, "dt must be > 0");
    if (dt > 1.0 / (2.0 * fmax)) raise(ST_CONFIG, "dt too coarse to sample fmax: dt > 1/(2 fmax)");
    const double peak = fmax / 2.5;
    const double delay = 1.5 / peak;
    std::vector<float> w(static_cast<size_t>(std::max(nsteps, 0)));
    for (int s = 0; s < nsteps; ++s) {
        const double tau = M_PI * peak * (s * dt - delay);
        const double t2 = tau * tau;
        w[s] = static_cast<float>((1.0 - 2.0 * t2) * std::exp(-t2));
    }
    return w;
}

Profile build_profile(const int n[3], const double h[3], const int nd[3], double fmax,
                      double vmax, double dt, double r_target, bool free_surface) {
    if (!(r_target > 0.0 && r_target < 1.0))
        raise(ST_CONFIG, "CPML reflection target must be in (0, 1)");
    Profile p;
    const double amax = M_PI * fmax;
    for (int ax = 0; ax < 3; ++ax) {
        p.a[ax].assign(n[ax], 0.0f);
        p.b[ax].assign(n[ax], 1.0f);
        p.ik[ax].assign(n[ax], 1.0f);
        if (nd[ax] < 1) continue;
        const double width = nd[ax] * h[ax];
        p.d0[ax] = -3.0 * vmax * std::log(r_target) / (2.0 * width);
        for (int layer = 0; layer < nd[ax]; ++layer) {
            const double depth = static_cast<double>(nd[ax] - layer) / nd[ax];
            const double damp = p.d0[ax] * depth * depth;
            const double shift = amax * (1.0 - depth);
            const double decay = std::exp(-(damp + shift) * dt);
            const float bf = static_cast<float>(decay);
            const float af = damp > 0.0 ? static_cast<float>(damp * (decay - 1.0) / (damp + shift))
                                        : 0.0f;
            const int hi = n[ax] - 1 - layer;
            if (!(ax == 2 && free_surface)) {
                p.a[ax][layer] = af;
                p.b[ax][layer] = bf;
            }
            p.a[ax][hi] = af;
            p.b[ax][hi] = bf;
        }
    }
    return p;
}

void fill_ghosts_replicate(float* f, const HostGrid& g) {
    const int r = g.r;
    auto clamp = [](int v, int n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); };
    for (int i = -r; i < g.n[0] + r; ++i)
        for (int j = -r; j < g.n[1] + r; ++j) {
            const bool ij_in = i >= 0 && i < g.n[0] && j >= 0 && j < g.n[1];
            for (int k = -r; k < g.n[2] + r; ++k) {
                if (ij_in && k >= 0 && k < g.n[2]) {
                    k = g.n[2] - 1;  // jump over the interior run
                    continue;
                }
                f[g.off(i, j, k)] = f[g.off(clamp(i, g.n[0]), clamp(j, g.n[1]), clamp(k, g.n[2]))];
            }
        }
}

void taper_material(float* f, const HostGrid& g, const int ntaper[3], const int offset[3],
                    const int global_n[3]) {
    for (int ax = 0; ax < 3; ++ax) {
        const int nt = ntaper[ax];
        if (nt < 1) continue;
        for (int i = 0; i < g.n[0]; ++i)
            for (int j = 0; j < g.n[1]; ++j)
                for (int k = 0; k < g.n[2]; ++k) {
                    const int loc[3] = {i, j, k};
                    const int gidx = loc[ax] + offset[ax];
                    const int depth = std::min(gidx, global_n[ax] - 1 - gidx);
                    if (depth >= nt) continue;
                    int src[3] = {i, j, k};
                    src[ax] = (gidx < nt ? nt : global_n[ax] - 1 - nt) - offset[ax];
                    if (src[ax] < 0 || src[ax] >= g.n[ax]) continue;
                    const double beta =
                        0.5 * (1.0 - std::cos(M_PI * (depth + 1) / static_cast<double>(nt + 1)));
                    const float here = f[g.off(i, j, k)];
                    const float anchor = f[g.off(src[0], src[1], src[2])];
                    const float diff = here - anchor;  // float subtraction, as the reference
                    f[g.off(i, j, k)] =
                        static_cast<float>(static_cast<double>(anchor) + beta * diff);
                }
    }
    fill_ghosts_replicate(f, g);
}

void validate_vp(const float* vp, const HostGrid& g, float* vmin, float* vmax) {
    float lo = std::numeric_limits<float>::max();
    float hi = std::numeric_limits<float>::lowest();
    for (int i = 0; i < g.n[0]; ++i)
        for (int j = 0; j < g.n[1]; ++j)
            for (int k = 0; k < g.n[2]; ++k) {
                const float v = vp[g.off(i, j, k)];
                if (!std::isfinite(v) || v <= 0.0f)
                    raise(ST_VALIDATION, "vp must be finite and > 0 everywhere");
                lo = std::min(lo, v);
                hi = std::max(hi, v);
            }
    if (vmin) *vmin = lo;
    if (vmax) *vmax = hi;
}

}  // namespace mmb
