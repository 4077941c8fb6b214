// Host-side problem setup and schedule arithmetic.  Compiled WITHOUT -march
// and with -ffp-contract=off so the initial condition and dt round exactly as
// the reference's no-FMA x86-64 build.
#include <cmath>
#include <cstring>
#include <string>

#include "sg_internal.hpp"

namespace sg {

namespace {
constexpr double kPi = 3.14159265358979323846;  // std::numbers::pi
}

Equation equation_for(int problem) {
    Equation e;
    e.problem = problem;
    if (problem == SG_HEAT) {  // StencilShape::heat, geometry.cpp:8-14
        e.nvars = 1;
        e.halo = 1;
        e.substeps = 1;
    } else {  // StencilShape::euler, geometry.cpp:16-24
        e.nvars = 4;
        e.halo = 2;
        e.substeps = 2;
    }
    return e;
}

int max_levels(int b, int n) {  // geometry.cpp:59-66
    if (n < 1) fail(SG_EINVAL, "max_levels: halo must be >= 1");
    if (b % (2 * n) != 0) fail(SG_EINVAL, "max_levels: block size must be divisible by 2n");
    if (b < 4 * n) fail(SG_EINVAL, "max_levels: block size must be at least 4n");
    return b / (2 * n) - 1;
}

long schedule_octahedra(long steps, int k, int substeps, long* flat) {
    // geometry.cpp:169-184: nearest flat level, half-up; flat = k(m+1) (:132)
    if (steps < 1) fail(SG_EINVAL, "build_schedule: requested steps must be >= 1");
    const long levels = steps * substeps;
    long m = static_cast<long>(std::floor(static_cast<double>(levels - k) / k + 0.5));
    if (m < 0) m = 0;
    const long f = static_cast<long>(k) * (m + 1);
    if (f / substeps < 1) fail(SG_EINVAL, "build_schedule: nearest achievable step count is 0");
    if (flat) *flat = f;
    return m;
}

const char* kind_name(int k) {
    switch (k) {
        case K_UP: return "UpPyramid";
        case K_YB: return "YBridge";
        case K_XB: return "XBridge";
        case K_OCT: return "Octahedron";
        case K_DOWN: return "DownPyramid";
    }
    return "?";
}

int kind_levels(int kind, int kk) { return kind == K_OCT ? 2 * kk : kk; }

Rect kind_rect(int kind, int b, int n, int kk, int r) {
    // phase_region, geometry.cpp:93-115
    Rect t;
    switch (kind) {
        case K_UP: t = {n * r, b - n * r, n * r, b - n * r}; break;
        case K_YB: t = {n * r, b - n * r, b - n * r, b + n * r}; break;
        case K_XB: t = {b / 2 - n * r, b / 2 + n * r, b / 2 + n * r, 3 * b / 2 - n * r}; break;
        case K_DOWN: t = {b / 2 - n * r, b / 2 + n * r, b / 2 - n * r, b / 2 + n * r}; break;
        case K_OCT:
            if (r <= kk) {
                t = {b / 2 - n * r, b / 2 + n * r, b / 2 - n * r, b / 2 + n * r};
            } else {
                const int w = b - 2 * n * (r - kk);
                t = {b / 2 - w / 2, b / 2 + w / 2, b / 2 - w / 2, b / 2 + w / 2};
            }
            break;
    }
    return t;
}

void validate(const sg_config& c) {
    // SolverConfig::validate, config.cpp:31-62
    if (c.problem != SG_HEAT && c.problem != SG_EULER) fail(SG_EINVAL, "unknown problem");
    const Equation eq = equation_for(c.problem);
    max_levels(c.block, eq.halo);
    const int ny = c.ny > 0 ? c.ny : c.nx;
    if (c.nx <= 0 || c.nx % c.block != 0)
        fail(SG_EINVAL, "config: nx must be a positive multiple of block");
    if (ny <= 0 || ny % c.block != 0)
        fail(SG_EINVAL, "config: ny must be a positive multiple of block");
    int px = c.px, py = c.py;
    if (px <= 0 && py <= 0) {
        px = c.ranks;
        py = 1;
    }
    if (px <= 0) px = 1;
    if (py <= 0) py = 1;
    if (c.ranks <= 0 || (c.nx / c.block) % px != 0)
        fail(SG_EINVAL, "config: ranks must evenly divide the block-column count");
    if ((ny / c.block) % py != 0)
        fail(SG_EINVAL, "config: py must evenly divide the block-row count");
    if (px * py != c.ranks) fail(SG_EINVAL, "config: px*py must equal ranks");
    if (c.steps <= 0) fail(SG_EINVAL, "config: steps must be positive");
    if (c.share < 0.0 || c.share > 1.0) fail(SG_EINVAL, "config: share must be in [0, 1]");
    if (c.pool_a_workers <= 0 || c.pool_b_workers <= 0)
        fail(SG_EINVAL, "config: pool workers must be positive");
    if (c.pool_a_cost <= 0.0 || c.pool_b_cost <= 0.0)
        fail(SG_EINVAL, "config: pool cost must be positive");
    if (c.cell_cost < 0.0) fail(SG_EINVAL, "config: cell cost must be non-negative");
    if (c.problem == SG_HEAT) {
        if (c.heat_fourier <= 0.0 || c.heat_fourier > 0.25)
            fail(SG_EINVAL, "config: heat stability requires fourier number in (0, 0.25]");
        if (c.heat_alpha <= 0.0) fail(SG_EINVAL, "config: heat alpha must be positive");
    } else {
        if (c.cfl <= 0.0 || c.cfl > 1.0) fail(SG_EINVAL, "config: cfl must be in (0, 1]");
        if (c.gamma <= 1.0) fail(SG_EINVAL, "config: gamma must exceed 1");
    }
    if (c.snapshot_every <= 0) fail(SG_EINVAL, "config: snapshot cadence must be positive");
    // LinkModel::validate, transport.hpp:27-30
    if (c.link_latency < 0.0 || !(c.link_bandwidth > 0.0))
        fail(SG_EINVAL, "LinkModel: latency >= 0 and bandwidth > 0 required");
    if (c.mode != SG_WALL)
        fail(SG_EINVAL, "config: only mode=wall is supported on the GPU (the virtual network "
                        "model is out of scope)");
}

namespace {

// VortexSpec::standard, physics.cpp:28-39: {alpha, mach, R, sigma, beta, L}
struct Vortex {
    double alpha, mach, radius, sigma, beta, half_extent;
};
Vortex vortex_standard(double gamma) {
    Vortex s;
    s.alpha = kPi / 4.0;
    s.mach = std::sqrt(2.0 / gamma);
    s.radius = 1.0;
    s.sigma = 1.0;
    s.beta = s.mach * (5.0 * std::sqrt(2.0) / (4.0 * kPi)) * std::exp(0.5);
    s.half_extent = 5.0;
    return s;
}

// vortex_state, physics.cpp:158-174
void vortex_state(double x, double y, const Vortex& s, double gamma, double* q) {
    const double f = -0.5 / (s.sigma * s.sigma) *
                     ((x / s.radius) * (x / s.radius) + (y / s.radius) * (y / s.radius));
    const double omega = s.beta * std::exp(f);
    const double du = -(y / s.radius) * omega;
    const double dv = (x / s.radius) * omega;
    const double dt_pert = -0.5 * (gamma - 1.0) * omega * omega;
    const double base = 1.0 + dt_pert;
    if (!(base > 0.0)) fail(SG_ENONPHYS, "vortex perturbation drives 1 + dT <= 0");
    const double rho = std::pow(base, 1.0 / (gamma - 1.0));
    const double u = s.mach * std::cos(s.alpha) + du;
    const double v = s.mach * std::sin(s.alpha) + dv;
    const double p = (1.0 / gamma) * std::pow(base, gamma / (gamma - 1.0));
    const double e = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v);
    q[0] = rho;
    q[1] = rho * u;
    q[2] = rho * v;
    q[3] = e;
}

double pressure_host(const double* q, double gamma) {  // physics.cpp:52-61
    const double rho = q[0];
    if (!(rho > 0.0)) fail(SG_ENONPHYS, "non-physical state: rho <= 0");
    const double p = (gamma - 1.0) * (q[3] - 0.5 * (q[1] * q[1] + q[2] * q[2]) / rho);
    if (!(p > 0.0)) fail(SG_ENONPHYS, "non-physical state: p <= 0");
    return p;
}

}  // namespace

Setup make_setup(const sg_config& c) {
    validate(c);
    Setup s;
    s.eq = equation_for(c.problem);
    s.nx = c.nx;
    s.ny = c.ny > 0 ? c.ny : c.nx;
    const int nx = s.nx, ny = s.ny;
    const std::size_t plane = static_cast<std::size_t>(nx) * ny;
    s.initial.assign(plane * s.eq.nvars, 0.0);
    if (c.problem == SG_HEAT) {
        // engine.cpp:31-42; heat_analytic physics.cpp:47-50 at node positions
        s.dx = 1.0 / nx;
        s.dy = 1.0 / ny;
        s.dt = c.heat_fourier * s.dx * s.dx / c.heat_alpha;
        std::vector<double> sx(nx), sy(ny);
        for (int x = 0; x < nx; ++x) sx[x] = std::sin(2.0 * kPi * (0.0 + (x + 0.0) * s.dx));
        for (int y = 0; y < ny; ++y) sy[y] = std::sin(2.0 * kPi * (0.0 + (y + 0.0) * s.dy));
        const double decay = std::exp(-8.0 * kPi * kPi * c.heat_alpha * 0.0);
        for (int y = 0; y < ny; ++y) {
            double* row = &s.initial[static_cast<std::size_t>(y) * nx];
            for (int x = 0; x < nx; ++x) row[x] = sx[x] * sy[y] * decay;
        }
        s.heat_fx = c.heat_alpha * s.dt / (s.dx * s.dx);
        s.heat_fy = c.heat_alpha * s.dt / (s.dy * s.dy);
    } else {
        // engine.cpp:43-68; vortex_init physics.cpp:176-191 (cell centred)
        const Vortex v = vortex_standard(c.gamma);
        const double L = v.half_extent;
        s.dx = 2.0 * L / nx;
        s.dy = 2.0 * L / ny;
        for (int j = 0; j < ny; ++j) {
            const double y = -L + (j + 0.5) * s.dy;
            for (int i = 0; i < nx; ++i) {
                const double x = -L + (i + 0.5) * s.dx;
                double q[4];
                vortex_state(x, y, v, c.gamma, q);
                for (int k = 0; k < 4; ++k) s.initial[k * plane + static_cast<std::size_t>(j) * nx + i] = q[k];
            }
        }
        double radius = 0.0;
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                double q[4];
                for (int k = 0; k < 4; ++k) q[k] = s.initial[k * plane + static_cast<std::size_t>(y) * nx + x];
                const double p = pressure_host(q, c.gamma);
                const double cs = std::sqrt(c.gamma * p / q[0]);
                const double rx = std::abs(q[1] / q[0]) + cs;
                const double ry = std::abs(q[2] / q[0]) + cs;
                const double r = rx / s.dx + ry / s.dy;
                radius = (radius < r) ? r : radius;  // std::max
            }
        s.dt = c.cfl / radius;
        s.gamma = c.gamma;
        s.cx_pred = 0.5 * s.dt / s.dx;
        s.cy_pred = 0.5 * s.dt / s.dy;
        s.cx_corr = s.dt / s.dx;
        s.cy_corr = s.dt / s.dy;
    }
    return s;
}

}  // namespace sg
