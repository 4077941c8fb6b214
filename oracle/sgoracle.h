/* Test infrastructure only -- NOT product code.
 *
 * CPU restatement (plain C, no FMA: built with -ffp-contract=off) of the
 * reference swept-rule solver's hot path, used by tests/ and bench.py's
 * cpu_baseline leg as the parity checker.  Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).
 *
 * Parity pinned: tests/test_oracle.py checks this restatement bit-for-bit
 * against (a) the reference library itself built from its own sources
 * (oracle/_ref, when present) and (b) the committed golden fixtures in
 * tests/golden/ (FNV-1a-64 hashes of reference outputs).
 */
#ifndef SGORACLE_H
#define SGORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum { SGO_HEAT = 0, SGO_EULER = 1 };
enum { SGO_OK = 0, SGO_EINVAL = 1, SGO_ENONPHYS = 2 };

/* geometry.cpp:59-66 */
int sgo_max_levels(int b, int n);
/* geometry.cpp:169-184 (m rounding) and :132 (flat = k(m+1)); returns m or -1 */
long sgo_schedule(long requested_steps, int b, int n, int substeps, long* flat_level);

/* engine.cpp:27-70: initial condition (nvars*ny*nx, [var][y][x]) and dt/dx/dy */
int sgo_setup(int problem, int nx, int ny, double heat_alpha, double heat_fourier,
              double gamma, double cfl, double* initial, double* dt_dx_dy);

/* physics.hpp:57-63 / physics.cpp:131-156 applied on rectangles; the grid wraps
 * in y (field.hpp:18-21); x must be in range.  rects: n x {x0,x1,y0,y1}.
 * params: heat {alpha,dx,dy,dt}; euler {gamma,dx,dy,dt}. */
int sgo_substep(int problem, int stage, const double* read1, const double* read2, double* out,
                int nvars, int nx, int ny, const int* rects, int nrects, const double* params);

/* Single-loop periodic solver (test_engine.cpp:43-91 reference_solve):
 * advances `initial` by `levels` sub-step levels, writes the last level to out.
 * threads>1 parallelises rows (bitwise identical: cells are independent). */
int sgo_standard_solve(int problem, int nx, int ny, long levels, const double* params,
                       const double* initial, double* out, int threads);

/* Swept executor restated in physical coordinates: runs the reference phase
 * plan (geometry.cpp:122-167) with the frame offsets that replace the shift
 * (engine.cpp:240-291), both axes periodic, on a ring of 2k+S planes; writes
 * level `out_level` to out.  Used to pin the frame recipe of SURVEY.md §8a. */
int sgo_swept_solve(int problem, int nx, int ny, int b, long octahedra, long out_level,
                    const double* params, const double* initial, double* out);

/* physics.cpp:52-107 known-answer helpers */
int sgo_pressure(const double* q, double gamma, double* p);
void sgo_minmod(const double* q4x4, const double* p4, double* ql, double* qr);
int sgo_interface_flux(const double* ql, const double* qr, int axis, double gamma, double* f);

unsigned long long sgo_fnv1a(const double* d, long n);

#ifdef __cplusplus
}
#endif
#endif
