// sweptgrid_gpu.hpp -- the reference-side binding of the B200 solver.
//
// Drop this header next to the reference's sources (it includes the
// reference's own headers, proj/include/sweptgrid/{engine,physics,transport}.hpp)
// and link libsweptgpu.so: run_gpu() has the signature and the exception
// behaviour of sweptgrid::run (proj/include/sweptgrid/engine.hpp:61,
// proj/src/engine.cpp:493-568), so a caller swaps `run(cfg)` for
// `run_gpu(cfg)` (e.g. proj/tools/sweptgrid_main.cpp:115) and keeps
// RunRecord::to_json() (engine.cpp:461-491), per-rank ledger included.
// Compiled against the reference headers by tests/test_capi.py.
#ifndef SWEPTGRID_GPU_HPP
#define SWEPTGRID_GPU_HPP

#include <algorithm>
#include <stdexcept>
#include <string>

#include "sweptgpu.h"
#include "sweptgrid/engine.hpp"
#include "sweptgrid/physics.hpp"
#include "sweptgrid/transport.hpp"

namespace sweptgrid {

inline RunResult run_gpu(const SolverConfig& c) {
    sg_config g;
    sg_config_default(&g);
    g.problem = c.problem == Problem::Heat ? SG_HEAT : SG_EULER;
    g.nx = c.nx;
    g.block = c.block;
    g.share = c.share;
    g.steps = c.steps;
    g.ranks = c.ranks;  // partitions (x-strips like the reference); spread over the visible GPUs
    g.engine = c.engine == EngineKind::Swept ? SG_SWEPT : SG_STANDARD;
    g.mode = c.mode == TransportMode::Wall ? SG_WALL : SG_VIRTUAL;  // virtual: SG_EINVAL (out of scope)
    g.link_latency = c.link.latency;
    g.link_bandwidth = c.link.bandwidth;
    g.pool_a_workers = c.pool_a.workers;
    g.pool_a_cost = c.pool_a.cost;
    g.pool_b_workers = c.pool_b.workers;
    g.pool_b_cost = c.pool_b.cost;
    g.cell_cost = c.cell_cost;
    g.heat_alpha = c.heat_alpha;
    g.heat_fourier = c.heat_fourier;
    g.gamma = c.gamma;
    g.cfl = c.cfl;
    g.snapshot_path = c.snapshot_path.empty() ? nullptr : c.snapshot_path.c_str();  // SWPT2D, snapshot.cpp
    g.snapshot_every = c.snapshot_every;
    sg_result r;
    char err[1024];
    switch (sg_run(&g, &r, err, sizeof err)) {
        case SG_OK: break;
        case SG_EINVAL: throw std::invalid_argument(err);
        case SG_ENONPHYS: throw NonPhysicalState(err);
        case SG_ETRANSPORT: throw TransportError(err);
        case SG_ELOGIC: throw std::logic_error(err);
        default: throw std::runtime_error(err);  // SG_EIO (snapshot I/O), SG_ECUDA
    }
    RunResult out;
    out.final_field = FieldState(r.nvars, r.nx, r.ny, r.final_level);
    std::copy(r.final_field, r.final_field + out.final_field.data.size(), out.final_field.data.begin());
    RunRecord& rec = out.record;
    rec.engine = c.engine == EngineKind::Swept ? "swept" : "standard";
    rec.problem = problem_name(c.problem);
    rec.mode = "wall";
    rec.nx = r.nx;
    rec.block = r.block;
    rec.ranks = r.ranks;
    rec.steps_requested = r.steps_requested;
    rec.actual_steps = r.actual_steps;
    rec.total_levels = r.total_levels;
    rec.octahedra = r.octahedra;
    rec.communicates = r.communicates;
    rec.dt = r.dt;
    rec.setup_seconds = r.setup_seconds;
    rec.wall_seconds = r.wall_seconds;
    rec.modeled_seconds = 0.0;
    rec.messages = r.messages;
    rec.bytes = r.bytes;
    rec.cell_updates = r.cell_updates;
    rec.snapshot_frames = r.snapshot_frames;
    rec.ledger.ranks.resize(static_cast<std::size_t>(r.nparts));  // CostLedger::PerRank, transport.hpp:35-44
    for (int q = 0; q < r.nparts; ++q) {
        rec.ledger.ranks[q].messages = r.part_messages[q];
        rec.ledger.ranks[q].bytes_sent = r.part_bytes[q];
    }
    sg_free_result(&r);
    return out;
}

}  // namespace sweptgrid

#endif
