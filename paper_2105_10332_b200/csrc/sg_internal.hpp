// Internal host-side types of the B200 swept solver (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sweptgpu.h"

namespace sg {

// Error carrying the C-ABI status code; thrown by host code, caught at the ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

// ------------------------------------------------------------- problem --
// Equation plugin metadata: StencilShape::heat/euler (geometry.cpp:8-24),
// nvars_for (physics.cpp:26).
struct Equation {
    int problem = SG_HEAT;
    int nvars = 1;
    int halo = 1;      // n
    int substeps = 1;  // S
};
Equation equation_for(int problem);

// make_setup (engine.cpp:27-70): spacing, dt and the initial condition,
// computed on the host with glibc exactly as the reference does.
struct Setup {
    Equation eq;
    int nx = 0, ny = 0;
    double dx = 0, dy = 0, dt = 0;
    // Kernel coefficients precomputed with the reference's association
    // order (physics.hpp:58-59, physics.cpp:136-137,150-151).
    double heat_fx = 0, heat_fy = 0;          // (alpha*dt)/(dx*dx)
    double gamma = 1.4;
    double cx_pred = 0, cy_pred = 0;          // (0.5*dt)/dx
    double cx_corr = 0, cy_corr = 0;          // dt/dx
    std::vector<double> initial;              // [var][y][x]
};

void validate(const sg_config& c);
Setup make_setup(const sg_config& c);

// ------------------------------------------------------------ schedule --
int max_levels(int b, int n);                                     // geometry.cpp:59-66
long schedule_octahedra(long steps, int k, int substeps, long* flat);  // geometry.cpp:169-184

// Phase kinds of the GPU plan.  UP/YB/XB/DOWN = the reference phases of the
// same names; OCT = OctahedronDown + OctahedronUp fused into one launch
// (geometry.cpp:159-160).
enum Kind { K_UP = 0, K_YB = 1, K_XB = 2, K_OCT = 3, K_DOWN = 4, K_NKINDS = 5 };
const char* kind_name(int k);

struct Rect {
    int x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    int w() const { return x1 - x0; }
    int h() const { return y1 - y0; }
    long area() const { return (long)w() * h(); }
    bool empty() const { return x1 <= x0 || y1 <= y0; }
};

// Per-block template of kind `k` at relative level r (1-based), origin (0,0):
// phase_region, geometry.cpp:83-120.
Rect kind_rect(int kind, int b, int n, int kk, int r);
int kind_levels(int kind, int kk);

}  // namespace sg
