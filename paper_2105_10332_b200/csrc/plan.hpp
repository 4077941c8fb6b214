// Swept plan compiler: turns the reference phase schedule
// (build_schedule_cycles, geometry.cpp:122-167) into GPU launches plus the
// gather/scatter tables the phase kernels execute.
//
// Every phase instance (one per block per launch) is translation invariant, so
// the compiler replays the schedule on a small periodic tile of R x R blocks
// (the same replay the reference's CoverageOracle does, tests/oracle.hpp),
// records for one representative instance which foreign cells it reads and
// who produced them, and from that derives:
//   * per phase KIND: the shared-memory layout of one instance (a bounding
//     rectangle per relative level) and the export list -- the cells other
//     instances read, in record order (the "edges" of the swept rule);
//   * per launch CLASS: the import list -- (producer launch distance,
//     producer instance offset, record index) -> smem slot.
// The replay also proves the schedule: every read cell was produced earlier
// by a different launch, or by the same instance at a lower level.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "sg_internal.hpp"

namespace sg {

struct PlanLevel {   // one relative level r of a kind, r in [rmin, nlev]
    Rect bbox;       // cells resident in smem at this level (instance coords)
    int off = 0;     // smem offset (doubles) of var 0; var v at off + v*vstride
    int vstride = 0; // bbox rows * pitch
    int pitch = 0;   // row pitch in doubles (>= bbox width; uniform b+1 for heat)
    Rect comp;       // computed cells (empty for r <= 0)
};

struct KindLayout {
    int kind = 0;
    int nlev = 0;                 // computed levels 1..nlev
    int rmin = 0;                 // lowest resident relative level (0 or -1)
    std::vector<PlanLevel> lev;   // index r - rmin
    int smem_doubles = 0;         // per instance, all vars
    // export list: record index i -> (r, x, y) and its smem offset (var 0)
    std::vector<std::array<int, 3>> exp_cells;
    std::vector<int> exp_off, exp_vstride;
    // the scatter's table: {smem offset, record index}; inside every aligned
    // group of 32 (one warp instruction) the entries are permuted so the smem
    // reads hit distinct bank pairs (global coalescing is unchanged)
    std::vector<std::array<int, 2>> exp_pairs;
    int epad = 0;                 // record length, padded to a multiple of 4
    // storage reuse: levels > split receive no imports and are laid out over
    // the storage of levels < split-S+1; exports of levels <= split (the
    // first nexp_early record entries) are flushed before those levels run.
    int split = 0, nexp_early = 0;
    // warp lane map (heat kernel): per computed level r (1..nlev) and lane
    // 0..31: {smem offset of the lane's first source cell at r-1, smem offset
    // of its first destination cell, rows, x | y << 16 of the first cell};
    // rows = 0 for idle lanes.  pitch[r-1] = {bbox width at r-1, at r}.
    std::vector<std::array<int, 4>> lanes;
    std::vector<std::array<int, 2>> pitch;
    const PlanLevel& at(int r) const { return lev[r - rmin]; }
};

struct Segment {          // one producer of a launch class
    int delta = 0;        // producer = launch index - delta  (0 => initial plane)
    int di = 0, dj = 0;   // producer instance = consumer instance + (di, dj)
    int pkind = 0;        // producer kind (record length)
};
struct Import {           // one imported cell
    int seg = 0;
    int src = 0;          // record index in the producer (or packed rel. xy for the initial plane)
    int dst = 0;          // smem offset of var 0
    int vstride = 0;
    int r = 0, qx = 0, qy = 0;  // consumer relative level / coords
};
struct InitImport {       // a level-0 cell read straight from the initial plane
    int rx = 0, ry = 0;   // relative to the consumer origin
    int dst = 0, vstride = 0;
    int r = 0;
};
struct ClassTab {
    int kind = 0;
    std::vector<Segment> segs;
    std::vector<Import> imports;       // sorted by (seg, src); column kernels: (part, seg, src)
    int nimp_b = 0;                    // column kernels: imports of levels > gather_split (part B)
    std::vector<InitImport> inits;
};

struct Launch {
    int kind = 0;
    long lo = 0, hi = 0;   // absolute levels computed
    int frame = 0;         // 0: block-aligned (A), 1: shifted by b/2 (B)
    int cls = 0;
    int stage0 = 0;        // stage of relative level 1: (lo-1) % S
    int r_out = 0;         // relative level written to the output plane, 0 = none
    int slot = -1;         // record slot written (-1: no exports)
};

struct SweptPlan {
    int b = 0, n = 0, k = 0, S = 1, nvars = 1;
    long m = 0, flat = 0, final_level = 0;
    std::vector<Launch> launches;
    std::vector<ClassTab> classes;
    KindLayout kinds[K_NKINDS];
    int nslots = 0;        // record ring size (max delta + 1)
    int ghost = 0;         // ghost ring width in instances (max |di|,|dj|)
    int max_epad = 0;
    long replay_cycles = 0;
    // column-register heat kernels (colgeom.hpp): block size, 0 = generic
    // table-driven kernels; overexport = exported cells nobody reads
    int colB = 0;
    long overexport = 0;
    // statistics (per instance, cells): imports / exports / updates per kind
    long imports_per_kind[K_NKINDS] = {0, 0, 0, 0, 0};
    long updates_per_kind[K_NKINDS] = {0, 0, 0, 0, 0};
};

// Warp lane map of a w x h rectangle: lanes take (column, row-chunk) items;
// the row split divides h exactly when it can (uniform trip counts).
void lane_split(int w, int h, int* splits, int* rps);

// Reorder the entries of every aligned group of 32 so that, within each half
// warp, the 8-byte shared-memory addresses key(e) fall on distinct bank pairs
// where possible.
template <class T, class Key>
void spread_banks(std::vector<T>& v, std::size_t begin, std::size_t end, Key key);

// m = octahedra; final_level = the level the run must output; instances =
// block instances per launch over all partitions (0: unknown).  Heat runs with
// b in {8, 12, 16, 24, 32} use the register-tile kernels (colgeom.hpp) unless
// SG_HEAT_KERNEL=generic is set, or the grid is so small (< 2048 instances)
// that the per-instance latency of the generic kernels wins (SG_HEAT_KERNEL=
// column forces them).  (The engine recompiles with instances = 1, i.e.
// generic, when a partition's record ring would exceed the column kernels'
// 32-bit gather offsets; partition_instances is unused.)
SweptPlan compile_swept_plan(int b, const Equation& eq, long m, long final_level, long instances = 0,
                             long partition_instances = 0);

std::string describe_plan(const SweptPlan& p);

}  // namespace sg
