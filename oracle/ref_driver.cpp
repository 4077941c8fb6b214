// Test infrastructure only (see oracle/Makefile).  A thin extern "C" driver
// over the UNMODIFIED reference library compiled from /root/reference/proj/src,
// so pytest (ctypes) and bench.py's reference arm can call the reference's own
// public API:
//   run(const SolverConfig&) -> RunResult          proj/include/sweptgrid/engine.hpp:61
//   make_setup(const SolverConfig&)                proj/src/engine.cpp:27-70
//   build_schedule / build_schedule_cycles         proj/src/geometry.cpp:122-184
//   run_substep_serial / run_substep_omp           proj/src/physics.cpp:345-369
//   pressure / minmod_reconstruct / interface_flux proj/src/physics.cpp:52-107
// No reference source is copied here; this file only calls it.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sweptgrid/config.hpp"
#include "sweptgrid/engine.hpp"
#include "sweptgrid/geometry.hpp"
#include "sweptgrid/physics.hpp"

using namespace sweptgrid;

namespace {
void put(char* dst, long cap, const std::string& s) {
    if (!dst || cap <= 0) return;
    std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
    std::memcpy(dst, s.data(), n);
    dst[n] = '\0';
}
// 1 invalid_argument, 2 NonPhysicalState, 3 TransportError, 4 runtime, 5 logic/other
int classify(std::exception_ptr e, char* err, long errlen) {
    try {
        std::rethrow_exception(e);
    } catch (const std::invalid_argument& x) {
        put(err, errlen, x.what());
        return 1;
    } catch (const NonPhysicalState& x) {
        put(err, errlen, x.what());
        return 2;
    } catch (const TransportError& x) {
        put(err, errlen, x.what());
        return 3;
    } catch (const std::logic_error& x) {
        put(err, errlen, x.what());
        return 5;
    } catch (const std::runtime_error& x) {
        put(err, errlen, x.what());
        return 4;
    } catch (const std::exception& x) {
        put(err, errlen, x.what());
        return 5;
    }
    return 5;
}
}  // namespace

extern "C" {

int ref_run(const char* cfg_json, double* out, long out_len, char* rec_json, long rec_len,
            char* err, long errlen) {
    try {
        const SolverConfig cfg = SolverConfig::from_json(nlohmann::json::parse(cfg_json));
        RunResult r = run(cfg);
        if (out) {
            if (static_cast<long>(r.final_field.data.size()) > out_len) {
                put(err, errlen, "ref_run: output buffer too small");
                return 5;
            }
            std::memcpy(out, r.final_field.data.data(), r.final_field.data.size() * sizeof(double));
        }
        nlohmann::json j = r.record.to_json();
        j["final_level"] = r.final_field.level;
        put(rec_json, rec_len, j.dump(2));
        return 0;
    } catch (...) {
        return classify(std::current_exception(), err, errlen);
    }
}

int ref_setup(const char* cfg_json, double* initial, long len, double* dt_dx_dy, char* err,
              long errlen) {
    try {
        const SolverConfig cfg = SolverConfig::from_json(nlohmann::json::parse(cfg_json));
        ProblemSetup s = make_setup(cfg);
        if (initial) {
            if (static_cast<long>(s.initial.data.size()) > len) return 5;
            std::memcpy(initial, s.initial.data.data(), s.initial.data.size() * sizeof(double));
        }
        dt_dx_dy[0] = s.dt;
        dt_dx_dy[1] = s.dx;
        dt_dx_dy[2] = s.dy;
        return 0;
    } catch (...) {
        return classify(std::current_exception(), err, errlen);
    }
}

// Plan rows: phase, level, abs_level, x0, x1, y0, y1, shift_sign, frontier.
// meta: octahedra, flat_level, k, substeps.  Returns the entry count or -1.
long ref_schedule(long steps_or_m, int by_cycles, int b, int n, int substeps, long* rows,
                  long max_rows, long* meta, char* err, long errlen) {
    try {
        const StencilShape st = (n == 1 && substeps == 1)   ? StencilShape::heat()
                                : (n == 2 && substeps == 2) ? StencilShape::euler()
                                                            : StencilShape::generic(n, substeps);
        const BlockGeometry g(b, n);
        PhasePlan p = by_cycles ? build_schedule_cycles(steps_or_m, g, st)
                                : build_schedule(steps_or_m, g, st);
        meta[0] = p.octahedra;
        meta[1] = p.flat_level;
        meta[2] = p.k;
        meta[3] = p.substeps;
        long i = 0;
        for (const auto& e : p.entries) {
            if (i >= max_rows) break;
            long* r = rows + 9 * i;
            r[0] = static_cast<long>(e.phase);
            r[1] = e.level;
            r[2] = e.abs_level;
            r[3] = e.region.x0;
            r[4] = e.region.x1;
            r[5] = e.region.y0;
            r[6] = e.region.y1;
            r[7] = e.shift_sign;
            r[8] = e.frontier;
            ++i;
        }
        return static_cast<long>(p.entries.size());
    } catch (...) {
        classify(std::current_exception(), err, errlen);
        return -1;
    }
}

// rects: nrects x {x0, x1, y0, y1}; params: heat{alpha,dx,dy,dt} euler{gamma,dx,dy,dt,cfl}
int ref_substep(int problem, int stage, const double* read1, const double* read2, double* out,
                int nvars, int nx, int ny, const int* rects, int nrects, const double* hp,
                const double* ep, int threads, char* err, long errlen) {
    try {
        SubstepArgs a;
        a.problem = problem == 0 ? Problem::Heat : Problem::Euler;
        a.stage = stage;
        a.read1 = {read1, nvars, nx, ny};
        a.read2 = {read2, nvars, nx, ny};
        a.out = {out, nvars, nx, ny};
        a.heat = {hp[0], hp[1], hp[2], hp[3]};
        a.euler = {ep[0], ep[1], ep[2], ep[3], ep[4]};
        std::vector<CellBlock> blocks;
        for (int i = 0; i < nrects; ++i)
            blocks.push_back({{rects[4 * i], rects[4 * i + 1], rects[4 * i + 2], rects[4 * i + 3]}, 1});
        if (threads <= 0)
            run_substep_serial(a, blocks);
        else
            run_substep_omp(a, blocks, threads);
        return 0;
    } catch (...) {
        return classify(std::current_exception(), err, errlen);
    }
}

int ref_pressure(const double* q, double gamma, double* p, char* err, long errlen) {
    try {
        *p = pressure({q[0], q[1], q[2], q[3]}, gamma);
        return 0;
    } catch (...) {
        return classify(std::current_exception(), err, errlen);
    }
}

int ref_interface_flux(const double* ql, const double* qr, int axis, double gamma, double* f,
                       char* err, long errlen) {
    try {
        Vec4 r = interface_flux({ql[0], ql[1], ql[2], ql[3]}, {qr[0], qr[1], qr[2], qr[3]},
                                axis, gamma);
        for (int v = 0; v < 4; ++v) f[v] = r[v];
        return 0;
    } catch (...) {
        return classify(std::current_exception(), err, errlen);
    }
}

void ref_minmod(const double* q4x4, const double* p4, double* ql, double* qr) {
    Vec4 a{q4x4[0], q4x4[1], q4x4[2], q4x4[3]}, b{q4x4[4], q4x4[5], q4x4[6], q4x4[7]},
        c{q4x4[8], q4x4[9], q4x4[10], q4x4[11]}, d{q4x4[12], q4x4[13], q4x4[14], q4x4[15]};
    Vec4 l, r;
    minmod_reconstruct(a, b, c, d, p4[0], p4[1], p4[2], p4[3], l, r);
    for (int v = 0; v < 4; ++v) {
        ql[v] = l[v];
        qr[v] = r[v];
    }
}

int ref_vortex_state(double x, double y, double gamma, double* q, char* err, long errlen) {
    try {
        Vec4 r = vortex_state(x, y, VortexSpec::standard(gamma), gamma);
        for (int v = 0; v < 4; ++v) q[v] = r[v];
        return 0;
    } catch (...) {
        return classify(std::current_exception(), err, errlen);
    }
}

}  // extern "C"
