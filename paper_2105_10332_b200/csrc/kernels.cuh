// Kernel argument structures shared by kernels.cu and engine.cpp.
#pragma once

#include <cstdint>

namespace sg {

constexpr int kMaxLevels = 64;   // relative levels per kind (2k + 2 <= 64; level masks are 64-bit)
constexpr int kMaxSegs = 24;
constexpr int kMaxParts = 64;

struct DevLevel {
    int bx0, by0, bw, bh;   // resident bounding box
    int off, vstride;       // smem offset of var 0 / per-var stride
    int cx0, cx1, cy0, cy1; // computed rect (empty for r <= 0)
};

struct DevSeg {
    int slot;   // record slot of the producer launch
    int di, dj;
    int epad;   // producer record length
};

// Uniform per-level parameters of the heat phase kernel, kept in the kernel's
// parameter block (constant-cache broadcast, no dependent global loads).
struct HeatLevel {
    int cx0, cy0, cy1, w, items, rps;
    int poff, pbw, doff, cbw;   // src(x,y) = poff + y*pbw + x; dst(x,y) = doff + y*cbw + x
    float inv_w;
    int pad;
};

// One swept phase launch (all partitions resident on one device).
struct SweptArgs {
    // kind layout
    int nlev, rmin, smem_doubles, nexp, epad;
    int split, nexp_early;   // flush exports [0, nexp_early) after level `split`
    int ps_doubles, fx_doubles;  // euler scratch (pressure plane, per-axis flux arrays)
    const DevLevel* lev;     // [nlev - rmin + 1]
    const int* exp_off;      // [nexp]
    const int* exp_vs;       // [nexp]
    const int2* exp_pairs;   // [nexp] {smem off, record idx}, bank-spread within 32-groups
    const int4* lanes;       // [nlev][32] warp lane map (heat)
    const int2* pitch;       // [nlev] {bbox width at r-1, at r}
    // class tables
    const int4* imports;     // {seg, src, dst, vstride}
    const int2* imports2;    // {seg << 20 | src, dst}  (same entries, compact)
    const int2* imp_off;     // column kernels: {offset from the instance's slot-0 record, smem slot}
    int nimp_b;              // column kernels: the last nimp_b entries are gather part B
    double* gm_scratch;      // phases too large for shared memory: per-CTA (Euler) / per-warp (heat)
    long gm_stride;          // level storage in global memory, gm_stride doubles each (null: shared)
    int gm_ctas;             // persistent grid of the GM kernels
    double* oct_scratch;     // column kernels, b24 / b32: [dev part][bj][bi][row][lane] level-k state between
                             // the two halves of a split Octahedron (null: one launch)
    const int* imp_dense;    // column kernels, steady classes: [import slot] -> offset from the slot-0 record
    int dense;               // 1: imp_dense covers every import slot (no initial-plane cells)
    int lo_parity;           // column kernels: launch index parity (odd: CTAs walk the instances backwards)
    int nimp;
    const int4* inits;       // {rx, ry, dst, vstride}
    int ninit;
    DevSeg segs[kMaxSegs];
    int nsegs;
    // launch
    int frame, stage0, r_out, my_slot;
    int kind;                        // phase kind (sg::Kind)
    int colB;                        // heat: column-register kernels for block colB (0 = generic)
    unsigned long long out_mask;     // bit r: relative level r is the output level
    unsigned long long snap_mask;    // bit r: relative level r is a snapshot level
    // geometry
    int b, nx, ny, pw, ph, pbx, pby, px, py, ghost, extw, nslots;
    int ndev_parts;
    int dev_parts[kMaxParts];        // partitions handled by this launch
    int dev_pij[kMaxParts];          // their (pi | pj << 16)
    double* const* rec;              // [part * nslots + slot]
    const double* const* init_planes;// [part] [var][ph][pw]
    double* const* out_planes;       // [part] [var][ph][pw]
    double c0, c1, c2, c3;           // heat: fx, fy | euler: gamma, cx, cy (per stage)
    double c4, c5;
    int* err;
    // snapshots: every computed cell of a level l with l % snap_every == 0 also
    // goes to frame slot l % frame_ring of the owning partition
    double* const* frames;           // [part] -> frame_ring planes [var][ph][pw]
    int snap_every, frame_ring;
    long lo;                         // absolute level of relative level 1
    HeatLevel hl[kMaxLevels];        // heat kernel: levels 1..nlev
};

// One standard sub-step (all partitions on one device); planes carry a
// ghost frame of width n: pitch = pw + 2n, rows = ph + 2n.
struct StdArgs {
    int nvars, n, pw, ph, px, py, pitch, rows;
    int stage;
    int ndev_parts;
    int dev_parts[kMaxParts];
    const double* const* read1;   // [part] level-1 plane (ghosted)
    const double* const* read2;   // [part] level-2 plane (corrector base)
    double* const* out;           // [part] level plane (ghosted, pushes into neighbours)
    double c0, c1, c2, c3;
    int* err;
};

// FP64 flop/s of the current device without FMA (kernels.cu), -1 on error
double measure_fp64_peak();
// div_dn / recip_dn (physics.cuh) against IEEE division on n operand pairs:
// number of bitwise mismatches (first one in xy_bad[0..1]), -1 on error
long div_selftest(long n, unsigned long long seed, double* xy_bad);

}  // namespace sg
