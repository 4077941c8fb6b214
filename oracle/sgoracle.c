/* Test infrastructure only -- NOT product code.  See sgoracle.h.
 * CPU restatement of the reference hot path; each function cites the
 * reference file:line (relative to /root/reference/proj) it restates.
 * Built with -ffp-contract=off so every a*b+c rounds twice, as the reference's
 * no-march x86-64 build does. */
#include "sgoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846; /* std::numbers::pi */

int sgo_max_levels(int b, int n) { /* geometry.cpp:59-66 */
    if (n < 1 || b % (2 * n) != 0 || b < 4 * n) return -1;
    return b / (2 * n) - 1;
}

long sgo_schedule(long requested_steps, int b, int n, int substeps, long* flat_level) {
    /* geometry.cpp:169-184: m = floor((levels - k)/k + 0.5), clamped at 0 */
    int k = sgo_max_levels(b, n);
    if (k < 0 || requested_steps < 1) return -1;
    long levels = requested_steps * substeps;
    long m = (long)floor((double)(levels - k) / k + 0.5);
    if (m < 0) m = 0;
    long flat = (long)k * (m + 1); /* geometry.cpp:132 */
    if (flat / substeps < 1) return -1;
    if (flat_level) *flat_level = flat;
    return m;
}

/* ---------------------------------------------------------------- setup -- */

static void vortex_spec(double gamma, double* s /* alpha mach R sigma beta L */) {
    /* physics.cpp:28-39 VortexSpec::standard */
    s[0] = kPi / 4.0;
    s[1] = sqrt(2.0 / gamma);
    s[2] = 1.0;
    s[3] = 1.0;
    s[4] = s[1] * (5.0 * sqrt(2.0) / (4.0 * kPi)) * exp(0.5);
    s[5] = 5.0;
}

static int vortex_state(double x, double y, const double* s, double gamma, double* q) {
    /* physics.cpp:158-174 */
    const double R = s[2], sigma = s[3];
    const double f = -0.5 / (sigma * sigma) * ((x / R) * (x / R) + (y / R) * (y / R));
    const double omega = s[4] * exp(f);
    const double du = -(y / R) * omega;
    const double dv = (x / R) * omega;
    const double dt_pert = -0.5 * (gamma - 1.0) * omega * omega;
    const double base = 1.0 + dt_pert;
    if (!(base > 0.0)) return SGO_ENONPHYS;
    const double rho = pow(base, 1.0 / (gamma - 1.0));
    const double u = s[1] * cos(s[0]) + du;
    const double v = s[1] * sin(s[0]) + dv;
    const double p = (1.0 / gamma) * pow(base, gamma / (gamma - 1.0));
    const double e = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v);
    q[0] = rho;
    q[1] = rho * u;
    q[2] = rho * v;
    q[3] = e;
    return SGO_OK;
}

int sgo_pressure(const double* q, double gamma, double* pout) {
    /* physics.cpp:52-61 */
    const double rho = q[0];
    if (!(rho > 0.0)) return SGO_ENONPHYS;
    const double p = (gamma - 1.0) * (q[3] - 0.5 * (q[1] * q[1] + q[2] * q[2]) / rho);
    if (!(p > 0.0)) return SGO_ENONPHYS;
    *pout = p;
    return SGO_OK;
}

int sgo_setup(int problem, int nx, int ny, double heat_alpha, double heat_fourier,
              double gamma, double cfl, double* initial, double* out3) {
    /* engine.cpp:27-70 */
    if (problem == SGO_HEAT) {
        const double dx = 1.0 / nx, dy = 1.0 / ny;
        const double dt = heat_fourier * dx * dx / heat_alpha;
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                /* xpos/ypos engine.hpp:25-26; heat_analytic physics.cpp:47-50 */
                const double px = 0.0 + (x + 0.0) * dx, py = 0.0 + (y + 0.0) * dy;
                initial[(long)y * nx + x] = sin(2.0 * kPi * px) * sin(2.0 * kPi * py) *
                                            exp(-8.0 * kPi * kPi * heat_alpha * 0.0);
            }
        out3[0] = dt;
        out3[1] = dx;
        out3[2] = dy;
        return SGO_OK;
    }
    double s[6];
    vortex_spec(gamma, s);
    const double L = s[5];
    const double dx = 2.0 * L / nx, dy = 2.0 * L / ny;
    const long plane = (long)nx * ny;
    for (int j = 0; j < ny; ++j) { /* vortex_init physics.cpp:176-191 */
        const double y = -L + (j + 0.5) * dy;
        for (int i = 0; i < nx; ++i) {
            const double x = -L + (i + 0.5) * dx;
            double q[4];
            if (vortex_state(x, y, s, gamma, q)) return SGO_ENONPHYS;
            for (int v = 0; v < 4; ++v) initial[v * plane + (long)j * nx + i] = q[v];
        }
    }
    double radius = 0.0; /* engine.cpp:56-66 */
    for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) {
            double q[4], p;
            for (int v = 0; v < 4; ++v) q[v] = initial[v * plane + (long)y * nx + x];
            if (sgo_pressure(q, gamma, &p)) return SGO_ENONPHYS;
            const double c = sqrt(gamma * p / q[0]);
            const double rx = fabs(q[1] / q[0]) + c;
            const double ry = fabs(q[2] / q[0]) + c;
            const double r = rx / dx + ry / dy;
            radius = (radius < r) ? r : radius; /* std::max */
        }
    out3[0] = cfl / radius;
    out3[1] = dx;
    out3[2] = dy;
    return SGO_OK;
}

/* -------------------------------------------------------------- kernels -- */

typedef struct {
    const double* d;
    int nvars, nx, ny, wrapx;
} view_t;

static inline double at(const view_t* g, int v, int x, int y) {
    /* field.hpp:18-24 (y wraps); x wraps too for the periodic single-loop solver */
    y %= g->ny;
    if (y < 0) y += g->ny;
    if (g->wrapx) {
        x %= g->nx;
        if (x < 0) x += g->nx;
    }
    return g->d[((long)v * g->ny + y) * g->nx + x];
}

static inline double heat_point(const view_t* in, int x, int y, const double* hp) {
    /* physics.hpp:57-63 */
    const double fx = hp[0] * hp[3] / (hp[1] * hp[1]);
    const double fy = hp[0] * hp[3] / (hp[2] * hp[2]);
    const double c = at(in, 0, x, y);
    return c + fx * (at(in, 0, x + 1, y) - 2.0 * c + at(in, 0, x - 1, y)) +
           fy * (at(in, 0, x, y + 1) - 2.0 * c + at(in, 0, x, y - 1));
}

static void minmod(const double* qm1, const double* q0, const double* qp1, const double* qp2,
                   double pm1, double p0, double pp1, double pp2, double* ql, double* qr) {
    /* physics.cpp:75-92 */
    const double ratio = (pp1 - p0) / (p0 - pm1);
    if (isfinite(ratio) && ratio > 0.0) {
        const double w = 0.5 * ((1.0 < ratio) ? 1.0 : ratio); /* std::min(ratio, 1.0) */
        for (int v = 0; v < 4; ++v) ql[v] = q0[v] + w * (qp1[v] - q0[v]);
    } else {
        for (int v = 0; v < 4; ++v) ql[v] = q0[v];
    }
    const double inv = (pp1 - p0) / (pp2 - pp1);
    if (isfinite(inv) && inv > 0.0) {
        const double w = 0.5 * ((1.0 < inv) ? 1.0 : inv);
        for (int v = 0; v < 4; ++v) qr[v] = qp1[v] + w * (q0[v] - qp1[v]);
    } else {
        for (int v = 0; v < 4; ++v) qr[v] = qp1[v];
    }
}

void sgo_minmod(const double* q, const double* p, double* ql, double* qr) {
    minmod(q, q + 4, q + 8, q + 12, p[0], p[1], p[2], p[3], ql, qr);
}

static void flux(const double* q, int axis, double gamma, double p, double* f) {
    /* euler_flux_x / euler_flux_y, physics.cpp:63-73 */
    if (axis == 0) {
        const double u = q[1] / q[0];
        f[0] = q[1];
        f[1] = q[1] * u + p;
        f[2] = q[2] * u;
        f[3] = (q[3] + p) * u;
    } else {
        const double v = q[2] / q[0];
        f[0] = q[2];
        f[1] = q[1] * v;
        f[2] = q[2] * v + p;
        f[3] = (q[3] + p) * v;
    }
}

static int iflux(const double* ql, const double* qr, int axis, double gamma, double* f) {
    /* interface_flux, physics.cpp:94-107 */
    double pl, pr;
    if (sgo_pressure(ql, gamma, &pl) || sgo_pressure(qr, gamma, &pr)) return SGO_ENONPHYS;
    const double unl = (axis == 0 ? ql[1] : ql[2]) / ql[0];
    const double unr = (axis == 0 ? qr[1] : qr[2]) / qr[0];
    const double a = fabs(unl) + sqrt(gamma * pl / ql[0]);
    const double b = fabs(unr) + sqrt(gamma * pr / qr[0]);
    const double rsp = (a < b) ? b : a; /* std::max */
    double fl[4], fr[4];
    flux(ql, axis, gamma, pl, fl);
    flux(qr, axis, gamma, pr, fr);
    for (int v = 0; v < 4; ++v) f[v] = 0.5 * (fl[v] + fr[v] + rsp * (ql[v] - qr[v]));
    return SGO_OK;
}

int sgo_interface_flux(const double* ql, const double* qr, int axis, double gamma, double* f) {
    return iflux(ql, qr, axis, gamma, f);
}

static int rflux(const view_t* g, int x, int y, int axis, double gamma, double* f) {
    /* reconstructed_flux_x/y, physics.cpp:109-129 */
    double q[4][4], p[4];
    for (int i = 0; i < 4; ++i) {
        const int xx = axis == 0 ? x - 1 + i : x, yy = axis == 0 ? y : y - 1 + i;
        for (int v = 0; v < 4; ++v) q[i][v] = at(g, v, xx, yy);
        if (sgo_pressure(q[i], gamma, &p[i])) return SGO_ENONPHYS;
    }
    double ql[4], qr[4];
    minmod(q[0], q[1], q[2], q[3], p[0], p[1], p[2], p[3], ql, qr);
    return iflux(ql, qr, axis, gamma, f);
}

static int euler_point(const view_t* base, const view_t* src, int x, int y, int stage,
                       const double* ep, double* out) {
    /* euler_predictor_point / euler_corrector_point, physics.cpp:131-156 */
    double fe[4], fw[4], gn[4], gs[4];
    int err = rflux(src, x, y, 0, ep[0], fe) | rflux(src, x - 1, y, 0, ep[0], fw) |
              rflux(src, x, y, 1, ep[0], gn) | rflux(src, x, y - 1, 1, ep[0], gs);
    const double cx = stage == 0 ? 0.5 * ep[3] / ep[1] : ep[3] / ep[1];
    const double cy = stage == 0 ? 0.5 * ep[3] / ep[2] : ep[3] / ep[2];
    for (int v = 0; v < 4; ++v)
        out[v] = at(base, v, x, y) - cx * (fe[v] - fw[v]) - cy * (gn[v] - gs[v]);
    return err;
}

/* One sub-step over a rectangle whose cells may wrap in both axes (wrapx) or
 * only in y (the reference GridView contract). */
static int rect_step(int problem, int stage, const view_t* r1, const view_t* r2, double* out,
                     int x0, int x1, int y0, int y1, const double* params) {
    const int nx = r1->nx, ny = r1->ny, nvars = r1->nvars;
    int err = 0;
    for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) {
            int wy = y % ny;
            if (wy < 0) wy += ny;
            int wx = x;
            if (r1->wrapx) {
                wx = x % nx;
                if (wx < 0) wx += nx;
            }
            if (problem == SGO_HEAT) {
                out[(long)wy * nx + wx] = heat_point(r1, x, y, params);
            } else {
                double q[4];
                /* physics.cpp:234-237: corrector base = read2 (Q^n), fluxes from read1 */
                err |= euler_point(stage == 0 ? r1 : r2, r1, x, y, stage, params, q);
                for (int v = 0; v < nvars; ++v) out[((long)v * ny + wy) * nx + wx] = q[v];
            }
        }
    return err ? SGO_ENONPHYS : SGO_OK;
}

int sgo_substep(int problem, int stage, const double* read1, const double* read2, double* out,
                int nvars, int nx, int ny, const int* rects, int nrects, const double* params) {
    /* run_substep_serial, physics.cpp:345-350 */
    view_t r1 = {read1, nvars, nx, ny, 0}, r2 = {read2, nvars, nx, ny, 0};
    int err = 0;
    for (int i = 0; i < nrects; ++i)
        err |= rect_step(problem, stage, &r1, &r2, out, rects[4 * i], rects[4 * i + 1],
                         rects[4 * i + 2], rects[4 * i + 3], params);
    return err;
}

int sgo_standard_solve(int problem, int nx, int ny, long levels, const double* params,
                       const double* initial, double* out, int threads) {
    /* test_engine.cpp:43-91: ring of S+1 planes; level l reads l-1 (and l-2
     * for the corrector, stage = (l-1) % S, engine.cpp:383-387) */
    const int S = problem == SGO_HEAT ? 1 : 2, nvars = problem == SGO_HEAT ? 1 : 4;
    const long plane = (long)nvars * nx * ny;
    double* ring = (double*)malloc(sizeof(double) * plane * (S + 1));
    if (!ring) return SGO_EINVAL;
    memcpy(ring, initial, sizeof(double) * plane);
    int err = 0;
    for (long l = 1; l <= levels; ++l) {
        const int stage = (int)((l - 1) % S);
        view_t r1 = {ring + ((l - 1) % (S + 1)) * plane, nvars, nx, ny, 1};
        view_t r2 = {ring + ((l >= 2 ? l - 2 : l - 1) % (S + 1)) * plane, nvars, nx, ny, 1};
        double* o = ring + (l % (S + 1)) * plane;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1) reduction(| : err)
        for (int y = 0; y < ny; ++y) err |= rect_step(problem, stage, &r1, &r2, o, 0, nx, y, y + 1, params);
    }
    memcpy(out, ring + (levels % (S + 1)) * plane, sizeof(double) * plane);
    free(ring);
    return err ? SGO_ENONPHYS : SGO_OK;
}

/* Phase templates, geometry.cpp:83-120, per block with origin (0,0). */
enum { UP, YB, XB, OD, OU, DN };
static void region(int ph, int b, int n, int k, int l, int* r) {
    switch (ph) {
        case UP: r[0] = n * l; r[1] = b - n * l; r[2] = n * l; r[3] = b - n * l; break;
        case YB: r[0] = n * l; r[1] = b - n * l; r[2] = b - n * l; r[3] = b + n * l; break;
        case XB: r[0] = b / 2 - n * l; r[1] = b / 2 + n * l; r[2] = b / 2 + n * l; r[3] = 3 * b / 2 - n * l; break;
        case OD:
        case DN: r[0] = b / 2 - n * l; r[1] = b / 2 + n * l; r[2] = b / 2 - n * l; r[3] = b / 2 + n * l; break;
        default: {
            const int w = b - 2 * n * (l - k);
            r[0] = b / 2 - w / 2; r[1] = b / 2 + w / 2; r[2] = b / 2 - w / 2; r[3] = b / 2 + w / 2;
        }
    }
}

int sgo_swept_solve(int problem, int nx, int ny, int b, long m, long out_level, const double* params,
                    const double* initial, double* out) {
    const int n = problem == SGO_HEAT ? 1 : 2, S = problem == SGO_HEAT ? 1 : 2;
    const int nvars = problem == SGO_HEAT ? 1 : 4, k = sgo_max_levels(b, n);
    if (k < 0 || nx % b || ny % b) return SGO_EINVAL;
    const int cap = 2 * k + S; /* engine.cpp:174 */
    const long plane = (long)nvars * nx * ny;
    double* ring = (double*)malloc(sizeof(double) * plane * cap);
    if (!ring) return SGO_EINVAL;
    memcpy(ring, initial, sizeof(double) * plane);
    int off = 0, err = 0; /* frame offset: physical = template + origin - off */
    /* build_schedule_cycles order, geometry.cpp:153-165; each Communicate
     * toggles the frame between block centres and block corners. */
    long total = 3 + 3 * m + 1, seq = 0;
    for (long step = 0; step < total; ++step) {
        int ph, cnt = k, lo = 1;
        long base = 0;
        if (step == 0) ph = UP;
        else if (step == 1) ph = YB;
        else if (step == 2) { off = b / 2; ph = XB; }
        else if (step == total - 1) { ph = DN; base = m * k; }
        else {
            const long j = (step - 3) / 3 + 1;
            const int w = (int)((step - 3) % 3);
            if (w == 0) { ph = OD; base = (j - 1) * k; cnt = 2 * k; }
            else if (w == 1) { ph = YB; base = j * k; }
            else { off = off ? 0 : b / 2; ph = XB; base = j * k; }
        }
        for (int l = lo; l <= cnt; ++l) {
            int r[4];
            region(l > k && ph == OD ? OU : ph, b, n, k, l, r);
            const long abs_level = base + l;
            const int stage = (int)((abs_level - 1) % S);
            view_t r1 = {ring + ((abs_level - 1) % cap) * plane, nvars, nx, ny, 1};
            view_t r2 = {ring + ((abs_level >= 2 ? abs_level - 2 : abs_level - 1) % cap) * plane, nvars, nx, ny, 1};
            double* o = ring + (abs_level % cap) * plane;
            for (int bj = 0; bj < ny / b; ++bj)
                for (int bi = 0; bi < nx / b; ++bi)
                    err |= rect_step(problem, stage, &r1, &r2, o, r[0] + bi * b - off, r[1] + bi * b - off,
                                     r[2] + bj * b - off, r[3] + bj * b - off, params);
        }
        ++seq;
    }
    memcpy(out, ring + (out_level % cap) * plane, sizeof(double) * plane);
    free(ring);
    return err ? SGO_ENONPHYS : SGO_OK;
}

unsigned long long sgo_fnv1a(const double* d, long n) {
    unsigned long long h = 1469598103934665603ull;
    const unsigned char* p = (const unsigned char*)d;
    for (long i = 0; i < n * (long)sizeof(double); ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}
