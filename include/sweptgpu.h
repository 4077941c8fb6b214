/*
 * sweptgpu.h -- C-ABI drop-in boundary of the B200-native 2D swept-rule solver.
 *
 * The reference (CPU C++20 "sweptgrid", /root/reference/proj) exposes its hot
 * path through
 *     RunResult sweptgrid::run(const SolverConfig&)          engine.hpp:61
 * with the equation plugin
 *     run_substep_serial/omp(const SubstepArgs&, span<const CellBlock>)
 *                                                            physics.hpp:132-134
 * Every entry point below replaces one of those; the mapping is cited per
 * declaration.  Plain C types only: no torch / CUDA types in the signatures
 * (the stream argument of sg_substep is an opaque pointer).
 *
 * Errors mirror the reference's exception types as return codes:
 *   SG_EINVAL    std::invalid_argument   (config.cpp:31-62, geometry.cpp:43-66)
 *   SG_ENONPHYS  NonPhysicalState        (physics.hpp:18-20, physics.cpp:52-61)
 *   SG_ETRANSPORT TransportError         (transport.hpp:62-64)
 *   SG_EIO       std::runtime_error I/O  (snapshot.cpp:59-112, config.cpp:129)
 *   SG_ELOGIC    std::logic_error        (engine.cpp:295,565)
 *   SG_ECUDA     a CUDA runtime failure (no reference analogue)
 * and the message is copied into the caller's `err` buffer.
 */
#ifndef SWEPTGPU_H
#define SWEPTGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 1

enum sg_status {
    SG_OK = 0,
    SG_EINVAL = 1,
    SG_ENONPHYS = 2,
    SG_ETRANSPORT = 3,
    SG_EIO = 4,
    SG_ELOGIC = 5,
    SG_ECUDA = 6
};

enum sg_problem { SG_HEAT = 0, SG_EULER = 1 };        /* physics.hpp:14 Problem */
enum sg_engine { SG_SWEPT = 0, SG_STANDARD = 1 };     /* config.hpp:13-15 EngineKind */
enum sg_mode { SG_WALL = 0, SG_VIRTUAL = 1 };         /* transport.hpp TransportMode */

/* SolverConfig (config.hpp:28-56) plus the GPU partition knobs.  Obtain the
 * reference defaults (config.hpp:29-48) from sg_config_default(). */
typedef struct sg_config {
    int problem;            /* SG_HEAT | SG_EULER                  config.hpp:29 */
    int nx;                 /*                                     config.hpp:30 */
    int ny;                 /* 0 => nx (the reference is square-only, config.hpp:50) */
    int block;              /*                                     config.hpp:31 */
    double share;           /* validated, no effect (no CPU/GPU split) config.hpp:32 */
    long steps;             /*                                     config.hpp:33 */
    int ranks;              /* partitions (GPUs), px*py           config.hpp:34 */
    int engine;             /* SG_SWEPT | SG_STANDARD              config.hpp:35 */
    int mode;               /* SG_WALL only; SG_VIRTUAL => SG_EINVAL (simulated
                               network is out of scope)            config.hpp:36 */
    double link_latency;    /* validated, no effect                config.hpp:37 */
    double link_bandwidth;
    int pool_a_workers;     /* validated, no effect                config.hpp:38-39 */
    double pool_a_cost;
    int pool_b_workers;
    double pool_b_cost;
    double cell_cost;       /* validated, no effect                config.hpp:40 */
    double heat_alpha;      /*                                     config.hpp:42 */
    double heat_fourier;    /*                                     config.hpp:43 */
    double gamma;           /*                                     config.hpp:44 */
    double cfl;             /*                                     config.hpp:45 */
    const char* snapshot_path; /* NULL/"" = none                   config.hpp:47 */
    long snapshot_every;    /*                                     config.hpp:48 */
    /* GPU extensions */
    int px, py;             /* partition grid; 0,0 => auto from ranks (ranks x 1,
                               the reference's x-only decomposition) */
    int devices;            /* CUDA devices to spread partitions over; 0 => all
                               visible, capped at ranks (partitions > devices
                               are emulated round-robin on the same GPU) */
} sg_config;

/* RunRecord (engine.hpp:35-59) + RunResult (engine.hpp:61-64). */
typedef struct sg_result {
    int engine, problem, mode;
    int nx, ny, block, ranks, px, py, nvars;
    long steps_requested;
    long actual_steps;     /* swept: flat/S (geometry.hpp:90) */
    long total_levels;     /* completed sub-step levels */
    long octahedra;        /* swept only */
    long communicates;     /* swept only */
    long final_level;      /* level of final_field: actual_steps * S */
    double dt, dx, dy;
    double setup_seconds;  /* host: validate + initial condition + plan */
    double wall_seconds;   /* H2D + solve + D2H, wall clock (reference: solver loop) */
    double solve_seconds;  /* device time of the solve alone (CUDA events) */
    double modeled_seconds;/* always 0 (virtual clock out of scope) */
    long messages;         /* partition-boundary exchanges (ledger analogue) */
    long long bytes;       /* bytes pushed across partition boundaries */
    long long cell_updates;/* sum of computed cells over all levels, engine.cpp:519-528 */
    long snapshot_frames;
    long kernel_launches;  /* our kernels launched by the solve */
    double* final_field;   /* library-owned [var][y][x] fp64; sg_free_result */
    /* per-partition ledger (the reference's per-rank CostLedger,
     * transport.hpp:35-60, RunRecord::to_json per_rank, engine.cpp:482-489):
     * messages / bytes each partition pushed into other partitions (P2P
     * stores over NVLink between GPUs), exact counts of the launch plan.
     * Library-owned arrays of nparts entries, freed by sg_free_result. */
    int nparts;
    long* part_messages;
    long long* part_bytes;
} sg_result;

/* ---------------------------------------------------------------- solver -- */

/* Fill `cfg` with the reference defaults (config.hpp:29-48). */
void sg_config_default(sg_config* cfg);

/* SolverConfig::validate (config.cpp:31-62) + the GPU partition constraints. */
int sg_validate(const sg_config* cfg, char* err, size_t errlen);

/* sweptgrid::run (engine.cpp:493-568): synchronous, host in, host out. */
int sg_run(const sg_config* cfg, sg_result* out, char* err, size_t errlen);
void sg_free_result(sg_result* r);

/* Split form of sg_run for callers that keep state resident on the GPU
 * (benchmarks, drivers that reuse buffers):
 *   create   = make_setup + plan + device allocation (engine.cpp:27-70, 493-545)
 *   reset    = load the initial condition (engine.cpp:199-209 / 336-345)
 *              from the device-resident copy made at create
 *   solve    = the timed solver loop; returns device seconds
 *   fetch    = gather the final field to host (FrameCollector analogue)   */
typedef struct sg_solver sg_solver;
int sg_solver_create(const sg_config* cfg, sg_solver** out, char* err, size_t errlen);
int sg_solver_reset(sg_solver* s, char* err, size_t errlen);
int sg_solver_solve(sg_solver* s, double* device_seconds, char* err, size_t errlen);
int sg_solver_fetch(sg_solver* s, sg_result* out, char* err, size_t errlen);
/* Profiling hook: kernel time of the dominant kernel class over the last
 * solve (CUDA events around each of its launches), summed, and its count. */
int sg_solver_kernel_stats(sg_solver* s, int which, double* seconds, long* launches,
                           double* alg_bytes, double* updates);
/* Host-buffer I/O of the resident solver (the e2e path): upload replaces the
 * level-0 field with `host` ([var][ny][nx] fp64, pinned or pageable) and
 * download writes the final field into `host`; both synchronous.  A
 * distributed solver (sg_dist_create) reads / writes only its own partition
 * [var][ny/py][nx/px]. */
int sg_solver_upload(sg_solver* s, const double* host, char* err, size_t errlen);
int sg_solver_download(sg_solver* s, double* host, char* err, size_t errlen);
/* The initial condition make_setup computed (engine.cpp:27-70), [var][ny][nx]. */
int sg_solver_initial(sg_solver* s, double* host, char* err, size_t errlen);
/* Enable (1) / disable (0) per-launch CUDA events around the dominant kernel;
 * 2 + k times the launches of swept phase kind k instead (0 UpPyramid,
 * 1 YBridge, 2 XBridge, 3 Octahedron, 4 DownPyramid). */
int sg_solver_set_profile(sg_solver* s, int on);
void sg_solver_destroy(sg_solver* s);

/* ------------------------------------------- one process per GPU (NVLink) --
 * The distributed form of sg_solver_create for runs launched one process per
 * GPU (torchrun): rank r owns partition r of the px*py grid (world == px*py)
 * on its current CUDA device.  Its buffers are exported as CUDA IPC handles
 * (sg_dist_blob); the caller all-gathers the blobs in rank order by any means
 * (torch.distributed does it in the Python layer) and hands them to
 * sg_dist_connect, after which kernels store partition-edge cells straight
 * into the peers' memory over NVLink and dependent launches are ordered by
 * device-side epoch flags (no host round trip).  This replaces the
 * reference's Transport::exchange (transport.hpp:78-79).  reset / solve /
 * upload / download / fetch then act on the local partition (fetch fills only
 * this rank's part of final_field). */
int sg_dist_create(const sg_config* cfg, int rank, int world, sg_solver** out, char* err, size_t errlen);
/* Writes this rank's IPC blob into buf (if cap suffices); returns its size. */
long sg_dist_blob(sg_solver* s, void* buf, long cap, char* err, size_t errlen);
int sg_dist_connect(sg_solver* s, const void* blobs, long per_rank, char* err, size_t errlen);

/* Swept plan introspection (host only, no GPU): compiles the phase plan of
 * build_schedule (geometry.cpp:169-184) for (problem, block, steps) and
 * returns 16 statistics {k, m, flat, launches, classes, record slots, ghost,
 * max record, Oct imports, Oct exports, Oct updates, YB imports, YB exports,
 * YB updates, Oct smem bytes, replay cycles} plus a text description. */
int sg_plan_info(int problem, int block, long steps, long* stats, char* text, size_t textlen,
                 char* err, size_t errlen);

/* ----------------------------------------------------- equation plugin -- */

/* Measured FP64 throughput of the current device without FMA (DADD + DMUL,
 * the solver's arithmetic), in flop/s; -1 without a device.  Diagnostic for
 * the FP64 roofline; no reference counterpart. */
double sg_measure_fp64_peak(void);

/* Self-test of the shared-reciprocal IEEE division the Euler kernels use
 * (physics.cuh div_dn): bitwise mismatches against x / y over n operand pairs
 * (random bit patterns incl. zeros, subnormals, infinities, NaNs, and
 * physical magnitudes); the first mismatching pair goes to xy_bad[0..1].
 * -1 without a device.  Diagnostic; no reference counterpart. */
long sg_div_selftest(long n, unsigned long long seed, double* xy_bad);

/* Plan arithmetic, geometry.cpp:59-66 and 169-184.  Returns k / m or -1. */
int sg_max_levels(int block, int halo);
long sg_schedule(long requested_steps, int block, int halo, int substeps, long* flat_level);

/* One sub-step over rectangles on DEVICE buffers, the GPU replacement of
 * run_substep_serial/omp (physics.hpp:110-134, physics.cpp:345-369):
 * layout [var][y][x] fp64, y wraps, x must stay in range (GridView contract,
 * field.hpp:12-24).  rects: nrects x {x0,x1,y0,y1} (host array).
 * params: heat {alpha,dx,dy,dt} | euler {gamma,dx,dy,dt}.  `stream` is a
 * cudaStream_t (NULL = legacy default).  Non-physical states -> SG_ENONPHYS. */
int sg_substep(int problem, int stage, const double* d_read1, const double* d_read2,
               double* d_out, int nvars, int nx, int ny, const int* rects, int nrects,
               const double* params, void* stream, char* err, size_t errlen);

/* FNV-1a-64 of a host buffer: the final-field fingerprint of the reference's
 * parity probes.  Lets callers compare a solve with a
 * reference run byte for byte without moving the field. */
uint64_t sg_fnv1a64(const void* data, size_t bytes);

/* Library version / build info string (static storage). */
const char* sg_version(void);
/* Number of CUDA devices visible, or -1 with no driver. */
int sg_device_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SWEPTGPU_H */
