// extern "C" boundary (include/sweptgpu.h).  Exceptions never cross it: every
// entry point maps sg::Error / CUDA failures to an sg_status and a message.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "engine.hpp"
#include "sg_internal.hpp"

namespace sg {
cudaError_t launch_substep(int problem, int stage, const double* r1, const double* r2, double* out, int nx,
                           int ny, const int* d_rects, const long* d_prefix, int nrects, long total,
                           const double* c, int* d_err, cudaStream_t s);
}

struct sg_solver {
    sg::Solver* s;
};

namespace {

void put(char* err, size_t len, const char* msg) {
    if (!err || len == 0) return;
    std::snprintf(err, len, "%s", msg);
}

template <class F>
int guard(char* err, size_t errlen, F&& f) {
    try {
        f();
        return SG_OK;
    } catch (const sg::Error& e) {
        put(err, errlen, e.what());
        return e.code;
    } catch (const std::exception& e) {
        put(err, errlen, e.what());
        return SG_ELOGIC;
    } catch (...) {
        put(err, errlen, "unknown error");
        return SG_ELOGIC;
    }
}

}  // namespace

extern "C" {

void sg_config_default(sg_config* c) {
    // SolverConfig defaults, config.hpp:29-48
    std::memset(c, 0, sizeof *c);
    c->problem = SG_HEAT;
    c->nx = 64;
    c->ny = 0;
    c->block = 8;
    c->share = 1.0;
    c->steps = 10;
    c->ranks = 1;
    c->engine = SG_SWEPT;
    c->mode = SG_WALL;
    c->link_latency = 0.0;
    c->link_bandwidth = __builtin_inf();
    c->pool_a_workers = 1;
    c->pool_a_cost = 1.0;
    c->pool_b_workers = 1;
    c->pool_b_cost = 1.0;
    c->cell_cost = 5.0e-8;
    c->heat_alpha = 1.0;
    c->heat_fourier = 0.2;
    c->gamma = 1.4;
    c->cfl = 0.4;
    c->snapshot_path = nullptr;
    c->snapshot_every = 1;
    c->px = 0;
    c->py = 0;
    c->devices = 0;
}

int sg_validate(const sg_config* cfg, char* err, size_t errlen) {
    return guard(err, errlen, [&] { sg::validate(*cfg); });
}

int sg_solver_create(const sg_config* cfg, sg_solver** out, char* err, size_t errlen) {
    *out = nullptr;
    return guard(err, errlen, [&] {
        auto* h = new sg_solver{nullptr};
        try {
            h->s = new sg::Solver(*cfg);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int sg_dist_create(const sg_config* cfg, int rank, int world, sg_solver** out, char* err, size_t errlen) {
    *out = nullptr;
    return guard(err, errlen, [&] {
        auto* h = new sg_solver{nullptr};
        try {
            h->s = new sg::Solver(*cfg, rank, world);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

long sg_dist_blob(sg_solver* s, void* buf, long cap, char* err, size_t errlen) {
    long n = -1;
    const int rc = guard(err, errlen, [&] {
        const auto b = s->s->ipc_blob();
        n = static_cast<long>(b.size());
        if (buf && cap >= n) std::memcpy(buf, b.data(), b.size());
    });
    return rc == SG_OK ? n : -rc;
}

int sg_dist_connect(sg_solver* s, const void* blobs, long per_rank, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        s->s->connect(static_cast<const unsigned char*>(blobs), static_cast<std::size_t>(per_rank));
    });
}

int sg_solver_reset(sg_solver* s, char* err, size_t errlen) {
    return guard(err, errlen, [&] { s->s->reset(); });
}

int sg_solver_solve(sg_solver* s, double* secs, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        const double t = s->s->solve();
        if (secs) *secs = t;
    });
}

int sg_solver_fetch(sg_solver* s, sg_result* out, char* err, size_t errlen) {
    return guard(err, errlen, [&] { s->s->fetch(out); });
}

int sg_solver_kernel_stats(sg_solver* s, int which, double* seconds, long* launches, double* alg_bytes,
                           double* updates) {
    s->s->kernel_stats(which, seconds, launches, alg_bytes, updates);
    return SG_OK;
}

int sg_solver_upload(sg_solver* s, const double* host, char* err, size_t errlen) {
    return guard(err, errlen, [&] { s->s->upload(host); });
}

int sg_solver_download(sg_solver* s, double* host, char* err, size_t errlen) {
    return guard(err, errlen, [&] { s->s->download(host); });
}

int sg_solver_initial(sg_solver* s, double* host, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        const auto& v = s->s->setup().initial;
        std::memcpy(host, v.data(), v.size() * sizeof(double));
    });
}

int sg_solver_set_profile(sg_solver* s, int on) {
    s->s->profile = on != 0;
    if (on >= 2) s->s->set_prof_kind(on - 2);  // 2 + phase kind: time that kind's launches
    return SG_OK;
}

void sg_solver_destroy(sg_solver* s) {
    if (!s) return;
    delete s->s;
    delete s;
}

int sg_run(const sg_config* cfg, sg_result* out, char* err, size_t errlen) {
    std::memset(out, 0, sizeof *out);
    return guard(err, errlen, [&] {
        sg::Solver solver(*cfg);
        solver.set_graph(false);  // one solve: no graph capture inside wall_seconds
        const auto t0 = std::chrono::steady_clock::now();
        solver.reset();
        solver.solve();
        solver.fetch(out);
        out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

void sg_free_result(sg_result* r) {
    if (!r) return;
    std::free(r->final_field);
    std::free(r->part_messages);
    std::free(r->part_bytes);
    r->final_field = nullptr;
    r->part_messages = nullptr;
    r->part_bytes = nullptr;
    r->nparts = 0;
}

double sg_measure_fp64_peak(void) { return sg::measure_fp64_peak(); }

long sg_div_selftest(long n, unsigned long long seed, double* xy_bad) { return sg::div_selftest(n, seed, xy_bad); }

int sg_max_levels(int block, int halo) {
    try {
        return sg::max_levels(block, halo);
    } catch (...) {
        return -1;
    }
}

long sg_schedule(long steps, int block, int halo, int substeps, long* flat) {
    try {
        return sg::schedule_octahedra(steps, sg::max_levels(block, halo), substeps, flat);
    } catch (...) {
        return -1;
    }
}

int sg_substep(int problem, int stage, const double* d_read1, const double* d_read2, double* d_out, int nvars,
               int nx, int ny, const int* rects, int nrects, const double* params, void* stream, char* err,
               size_t errlen) {
    return guard(err, errlen, [&] {
        if (problem != SG_HEAT && problem != SG_EULER) sg::fail(SG_EINVAL, "unknown problem");
        if (nvars != (problem == SG_HEAT ? 1 : 4)) sg::fail(SG_EINVAL, "nvars does not match the problem");
        if (stage < 0 || stage > (problem == SG_HEAT ? 0 : 1)) sg::fail(SG_EINVAL, "bad stage");
        const int n = problem == SG_HEAT ? 1 : 2;
        std::vector<long> prefix(nrects + 1, 0);
        for (int i = 0; i < nrects; ++i) {
            const int* r = rects + 4 * i;
            if (r[1] < r[0] || r[3] < r[2]) sg::fail(SG_EINVAL, "substep: malformed rect");
            if (r[0] - n < 0 || r[1] + n > nx) sg::fail(SG_EINVAL, "substep: stencil leaves the plane in x");
            prefix[i + 1] = prefix[i] + static_cast<long>(r[1] - r[0]) * (r[3] - r[2]);
        }
        double c[4];
        if (problem == SG_HEAT) {  // params {alpha, dx, dy, dt}; physics.hpp:58-59
            c[0] = params[0] * params[3] / (params[1] * params[1]);
            c[1] = params[0] * params[3] / (params[2] * params[2]);
            c[2] = c[3] = 0.0;
        } else {  // params {gamma, dx, dy, dt}; physics.cpp:136-137, 150-151
            c[0] = params[0];
            c[1] = stage == 0 ? 0.5 * params[3] / params[1] : params[3] / params[1];
            c[2] = stage == 0 ? 0.5 * params[3] / params[2] : params[3] / params[2];
            c[3] = 0.0;
        }
        auto s = static_cast<cudaStream_t>(stream);
        auto ck = [](cudaError_t e) {
            if (e != cudaSuccess) sg::fail(SG_ECUDA, cudaGetErrorString(e));
        };
        // scratch freed on every path (a failing check throws through guard())
        struct DevBuf {
            void* p = nullptr;
            ~DevBuf() {
                if (p) cudaFree(p);
            }
        } rb, pb, eb;
        ck(cudaMalloc(&rb.p, sizeof(int) * 4 * std::max(nrects, 1)));
        ck(cudaMalloc(&pb.p, sizeof(long) * (nrects + 1)));
        ck(cudaMalloc(&eb.p, sizeof(int)));
        int* d_rects = static_cast<int*>(rb.p);
        long* d_prefix = static_cast<long*>(pb.p);
        int* d_err = static_cast<int*>(eb.p);
        ck(cudaMemsetAsync(d_err, 0, sizeof(int), s));
        if (nrects) ck(cudaMemcpyAsync(d_rects, rects, sizeof(int) * 4 * nrects, cudaMemcpyHostToDevice, s));
        ck(cudaMemcpyAsync(d_prefix, prefix.data(), sizeof(long) * (nrects + 1), cudaMemcpyHostToDevice, s));
        ck(sg::launch_substep(problem, stage, d_read1, d_read2, d_out, nx, ny, d_rects, d_prefix, nrects,
                              prefix[nrects], c, d_err, s));
        int e = 0;
        ck(cudaMemcpyAsync(&e, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
        ck(cudaStreamSynchronize(s));
        if (e) sg::fail(SG_ENONPHYS, "non-physical state: rho <= 0 or p <= 0");
    });
}

uint64_t sg_fnv1a64(const void* data, size_t bytes) {
    std::uint64_t h = 1469598103934665603ull;
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

const char* sg_version(void) {
    return "sweptgpu 0.1 (sm_100a, fp64, -fmad=false; ABI " "1" ")";
}

int sg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return n;
}

// Plan introspection for tests (host only, no GPU needed):
// returns the plan description text length; fills stats[16]:
// {k, m, flat, launches, classes, nslots, ghost, max_epad,
//  oct_imports, oct_exports, oct_updates, yb_imports, yb_exports, yb_updates,
//  oct_smem_bytes, replay_cycles}
int sg_plan_info(int problem, int block, long steps, long* stats, char* text, size_t textlen, char* err,
                 size_t errlen) {
    return guard(err, errlen, [&] {
        const sg::Equation eq = sg::equation_for(problem);
        const int k = sg::max_levels(block, eq.halo);
        long flat = 0;
        const long m = sg::schedule_octahedra(steps, k, eq.substeps, &flat);
        const long final_level = (flat / eq.substeps) * eq.substeps;
        const sg::SweptPlan p = sg::compile_swept_plan(block, eq, m, final_level);
        long sb[16] = {p.k, p.m, p.flat, (long)p.launches.size(), (long)p.classes.size(), p.nslots, p.ghost,
                       p.max_epad, p.imports_per_kind[sg::K_OCT], (long)p.kinds[sg::K_OCT].exp_cells.size(),
                       p.updates_per_kind[sg::K_OCT], p.imports_per_kind[sg::K_YB],
                       (long)p.kinds[sg::K_YB].exp_cells.size(), p.updates_per_kind[sg::K_YB],
                       (long)p.kinds[sg::K_OCT].smem_doubles * 8, p.replay_cycles};
        std::memcpy(stats, sb, sizeof sb);
        put(text, textlen, sg::describe_plan(p).c_str());
    });
}

}  // extern "C"
