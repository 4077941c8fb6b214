// sm_100a kernels of the swept solver.
//
//  swept_heat_col_kernel (heat, b = 8/12/16/24/32; the bench path) /
//  swept_heat_kernel (heat on tiny grids, SG_HEAT_KERNEL=generic) /
//  swept_euler_kernel: one launch = one swept phase
//      (UpPyramid, YBridge, XBridge, Octahedron = OctahedronDown+OctahedronUp,
//      DownPyramid) for every block instance of the partitions on this GPU:
//        1. gather: imported edge cells (records of earlier phases, or the
//           initial plane) -> shared memory (cp.async, straight to place);
//        2. advance all levels of the phase on chip (register tiles for the
//           column kernel, shared memory for the others);
//        3. scatter: the cells later phases read (this instance's record)
//           -> HBM, plus the copies partition-edge instances push into the
//           neighbouring partitions' ghost records (NVLink P2P stores when
//           the neighbour is another GPU);
//        4. cells at the output level -> the owning partition's output plane.
//  std_heat_kernel / std_euler_kernel: the standard decomposition, one
//      sub-step over the whole partition with boundary cells pushed into the
//      neighbours' ghost frames (StandardRank::exchange_ghosts + compute,
//      engine.cpp:351-408 of the reference).  std_step_kernel<PROB> is the
//      point-wise fallback for odd partition widths.
//  substep_rects_kernel<PROB>: run_substep on rectangles (physics.cpp:345-369).
//  dist_barrier_kernel: cross-process launch ordering (one process per GPU).
//  fp64_peak_kernel: DADD+DMUL microbenchmark for the FP64 roofline.
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>
#include <utility>

#include "devutil.cuh"
#include "kernels.cuh"
#include "physics.cuh"

namespace sg {

namespace {

// Heat phase kernel: one WARP per block instance, WPC instances per CTA, no
// CTA-wide barriers (the warp is the instance's only owner).
//  1. gather: cp.async lands every imported edge cell (a record entry of an
//     earlier phase) at its final place in the instance's level storage;
//  2. levels 1..nlev on chip: lane l takes the (column, row-chunk) item the
//     plan's lane map gives it and walks down the chunk, four rows per trip,
//     centre/south kept in registers (3 LDS + 1 STS per update);
//  3. scatter: the record entries (cells later phases read) go to HBM in
//     record order, plus ghost copies from partition-edge instances.  Levels
//     above `split` (an Octahedron's shrinking half, which gets no imports)
//     reuse the storage of the dead lower levels, so the lower levels'
//     exports are flushed first.
// GM: the phase's level storage lives in a per-warp global-memory scratch
// (A.gm_scratch, L1/L2-cached) instead of shared memory -- blocks whose
// phases exceed the 227 KB of shared memory (heat b > 48); a persistent grid
// walks the instances.  Correct, not fast.
template <int WPC, bool GM = false>
__global__ void __launch_bounds__(WPC * 32) swept_heat_kernel(const __grid_constant__ SweptArgs A) {
    extern __shared__ double sm[];
    __shared__ const double* segbase[WPC][kMaxSegs];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ninst = A.pbx * A.pby;
    for (int inst = blockIdx.x * WPC + warp; inst < ninst; inst += GM ? gridDim.x * WPC : ninst) {
    const int part = A.dev_parts[blockIdx.y];
    const int pi = part % A.px, pj = part / A.px;
    const int bi = inst % A.pbx, bj = inst / A.pbx;
    const int half = A.frame * (A.b / 2);
    double* S = GM ? A.gm_scratch + (((long)blockIdx.y * gridDim.x + blockIdx.x) * WPC + warp) * A.gm_stride
                   : sm + warp * A.smem_doubles;
    const double** sb = segbase[warp];

    // ---- 1. gather
    if (lane < A.nsegs) {
        const DevSeg sg = A.segs[lane];
        const long ext = (long)(bj + sg.dj + A.ghost) * A.extw + (bi + sg.di + A.ghost);
        sb[lane] = A.rec[part * A.nslots + sg.slot] + ext * sg.epad;
    }
    __syncwarp();
    if (GM) {
        for (int i = lane; i < A.nimp; i += 32) {
            const int2 e = ldg_keep(&A.imports2[i]);
            S[e.y] = sb[e.x >> 20][e.x & 0xFFFFF];
        }
    } else {
        const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(S));
        int i = lane;
        for (; i + 96 < A.nimp; i += 128) {
            const int2 e0 = ldg_keep(&A.imports2[i]), e1 = ldg_keep(&A.imports2[i + 32]);
            const int2 e2 = ldg_keep(&A.imports2[i + 64]), e3 = ldg_keep(&A.imports2[i + 96]);
            const double* g0 = sb[e0.x >> 20] + (e0.x & 0xFFFFF);
            const double* g1 = sb[e1.x >> 20] + (e1.x & 0xFFFFF);
            const double* g2 = sb[e2.x >> 20] + (e2.x & 0xFFFFF);
            const double* g3 = sb[e3.x >> 20] + (e3.x & 0xFFFFF);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * e0.y), "l"(g0) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * e1.y), "l"(g1) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * e2.y), "l"(g2) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * e3.y), "l"(g3) : "memory");
        }
        for (; i < A.nimp; i += 32) {
            const int2 e = ldg_keep(&A.imports2[i]);
            const double* g = sb[e.x >> 20] + (e.x & 0xFFFFF);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * e.y), "l"(g) : "memory");
        }
    }
    for (int i = lane; i < A.ninit; i += 32) {
        const int4 im = __ldg(&A.inits[i]);
        const int gx = wrapi(pi * A.pw + bi * A.b - half + im.x, A.nx);
        const int gy = wrapi(pj * A.ph + bj * A.b - half + im.y, A.ny);
        const int opi = gx / A.pw, opj = gy / A.ph;
        S[im.z] = A.init_planes[opj * A.px + opi][(long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw)];
    }
    cp_async_wait_all();
    __syncwarp();

    const int gh = A.ghost;
    double* dst = A.rec[part * A.nslots + A.my_slot] + ((long)(bj + gh) * A.extw + (bi + gh)) * A.epad;
    const bool edge = bi < gh || bi >= A.pbx - gh || bj < gh || bj >= A.pby - gh;
    auto flush = [&](int e0, int e1) {  // record entries [e0, e1) -> HBM (+ ghosts)
        int e = e0 + lane;
        for (; e + 96 < e1; e += 128) {
            const int2 p0 = ldg_keep(&A.exp_pairs[e]), p1 = ldg_keep(&A.exp_pairs[e + 32]);
            const int2 p2 = ldg_keep(&A.exp_pairs[e + 64]), p3 = ldg_keep(&A.exp_pairs[e + 96]);
            const double v0 = S[p0.x], v1 = S[p1.x], v2 = S[p2.x], v3 = S[p3.x];
            dst[p0.y] = v0;
            dst[p1.y] = v1;
            dst[p2.y] = v2;
            dst[p3.y] = v3;
        }
        for (; e < e1; e += 32) {
            const int2 p = ldg_keep(&A.exp_pairs[e]);
            dst[p.y] = S[p.x];
        }
        if (edge)
            for (int e2 = e0 + lane; e2 < e1; e2 += 32) {
                const int2 p = ldg_keep(&A.exp_pairs[e2]);
                const double v = S[p.x];
                for (int ej = -1; ej <= 1; ++ej)
                    for (int ei = -1; ei <= 1; ++ei) {
                        if (ei == 0 && ej == 0) continue;
                        const int tbi = bi - ei * A.pbx, tbj = bj - ej * A.pby;
                        if (tbi < -gh || tbi >= A.pbx + gh || tbj < -gh || tbj >= A.pby + gh) continue;
                        const int tp = wrapi(pj + ej, A.py) * A.px + wrapi(pi + ei, A.px);
                        A.rec[tp * A.nslots + A.my_slot][((long)(tbj + gh) * A.extw + (tbi + gh)) * A.epad + p.y] = v;
                    }
            }
    };

    // ---- 2. levels (per-level parameters come from the parameter block)
    const double fx = A.c0, fy = A.c1;
    for (int r = 1; r <= A.nlev; ++r) {
        const HeatLevel& L = A.hl[r - 1];
        const int bp = L.pbw, bc = L.cbw;
        // rows [y0, y0 + n) of column x: walk down, four rows per trip
        auto walk = [&](int x, int y0, int n) {
            const double* P = S + L.poff + y0 * bp + x;
            double* D = S + L.doff + y0 * bc + x;
            double south = P[-bp], c = P[0];
            int m = n;
            for (; m >= 4; m -= 4) {
                const double n1 = P[bp], n2 = P[2 * bp], n3 = P[3 * bp], n4 = P[4 * bp];
                const double v1 = heat_update(c, P[1], P[-1], n1, south, fx, fy);
                const double v2 = heat_update(n1, P[bp + 1], P[bp - 1], n2, c, fx, fy);
                const double v3 = heat_update(n2, P[2 * bp + 1], P[2 * bp - 1], n3, n1, fx, fy);
                const double v4 = heat_update(n3, P[3 * bp + 1], P[3 * bp - 1], n4, n2, fx, fy);
                D[0] = v1;
                D[bc] = v2;
                D[2 * bc] = v3;
                D[3 * bc] = v4;
                south = n3;
                c = n4;
                P += 4 * bp;
                D += 4 * bc;
            }
            if (m >= 2) {
                const double n1 = P[bp], n2 = P[2 * bp];
                const double v1 = heat_update(c, P[1], P[-1], n1, south, fx, fy);
                const double v2 = heat_update(n1, P[bp + 1], P[bp - 1], n2, c, fx, fy);
                D[0] = v1;
                D[bc] = v2;
                south = n1;
                c = n2;
                P += 2 * bp;
                D += 2 * bc;
                m -= 2;
            }
            if (m) D[0] = heat_update(c, P[1], P[-1], P[bp], south, fx, fy);
            const long lev = A.lo + r - 1;
            const bool snap = A.snap_every > 0 && lev % A.snap_every == 0;
            if (r == A.r_out || snap) {
                const double* Dv = S + L.doff + y0 * bc + x;
                const long pl = (long)A.pw * A.ph;
                for (int y = y0; y < y0 + n; ++y, Dv += bc) {
                    const int gx = wrapi(pi * A.pw + bi * A.b - half + x, A.nx);
                    const int gy = wrapi(pj * A.ph + bj * A.b - half + y, A.ny);
                    const int opi = gx / A.pw, opj = gy / A.ph;
                    const long o = (long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw);
                    if (r == A.r_out) A.out_planes[opj * A.px + opi][o] = *Dv;
                    if (snap) A.frames[opj * A.px + opi][(lev % A.frame_ring) * pl + o] = *Dv;
                }
            }
        };
        if (L.items > 0) {
            if (lane < L.items) {
                // item -> (column, row chunk); exact (items < 2^5, w <= 2^5)
                const int ch = __float2int_rz((lane + 0.5f) * L.inv_w);
                const int x = L.cx0 + (lane - ch * L.w);
                const int y0 = L.cy0 + ch * L.rps;
                const int n = min(L.rps, L.cy1 - y0);
                if (n > 0) walk(x, y0, n);
            }
        } else {
            // rectangles wider than a warp (block > 34): lanes stride the columns
            for (int x = L.cx0 + lane; x < L.cx0 + L.w; x += 32) walk(x, L.cy0, L.cy1 - L.cy0);
        }
        __syncwarp();
        if (r == A.split && A.nexp_early > 0) {
            flush(0, A.nexp_early);
            __syncwarp();
        }
    }
    // ---- 3. scatter the rest of the record
    if (A.nexp > A.nexp_early) flush(A.nexp_early, A.nexp);
    __syncwarp();  // (GM: the next instance reuses the scratch)
    }
}

// Euler phase kernel: one CTA (128 threads) per block instance.  Gather as
// the heat kernel (4 variables per record entry), then every level of the
// phase runs through euler_rect on shared memory (pressures, shared x/y
// interface fluxes, update), then the record is scattered.
// GM: level storage and flux scratch in a per-CTA global-memory scratch
// (Euler b > 32), a persistent grid walking the instances (see the heat
// kernel above).
template <int MINB, int NT = 128, bool FUSED = false, bool GM = false>
__global__ void __launch_bounds__(NT, MINB) swept_euler_kernel(const __grid_constant__ SweptArgs A) {
    extern __shared__ double Ssm[];
    __shared__ const double* sb[kMaxSegs];
    const int tid = threadIdx.x, T = NT;
    const int ninst = A.pbx * A.pby;
    for (int inst = blockIdx.x; inst < ninst; inst += GM ? gridDim.x : ninst) {
    double* S = GM ? A.gm_scratch + ((long)blockIdx.y * gridDim.x + blockIdx.x) * A.gm_stride : Ssm;
    const int part = A.dev_parts[blockIdx.y];
    const int pi = part % A.px, pj = part / A.px;
    const int bi = inst % A.pbx, bj = inst / A.pbx;
    const int half = A.frame * (A.b / 2);
    double* ps = S + A.smem_doubles;
    double* fxs = ps + A.ps_doubles;
    double* fys = fxs + A.fx_doubles;
    int err = 0;

    if (tid < A.nsegs) {
        const DevSeg sg = A.segs[tid];
        const long ext = (long)(bj + sg.dj + A.ghost) * A.extw + (bi + sg.di + A.ghost);
        sb[tid] = A.rec[part * A.nslots + sg.slot] + ext * 4 * sg.epad;
    }
    __syncthreads();
    if (GM) {
        for (int i = tid; i < A.nimp; i += T) {
            const int4 e = __ldg(&A.imports[i]);
            const int ep = A.segs[e.x].epad;
            const double* g = sb[e.x] + e.y;
#pragma unroll
            for (int v = 0; v < 4; ++v) S[e.z + v * e.w] = g[v * ep];
        }
    } else {
        const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(S));
        for (int i = tid; i < A.nimp; i += T) {
            const int4 e = __ldg(&A.imports[i]);
            const int ep = A.segs[e.x].epad;
            const double* g = sb[e.x] + e.y;
#pragma unroll
            for (int v = 0; v < 4; ++v)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * (e.z + v * e.w)),
                             "l"(g + v * ep)
                             : "memory");
        }
    }
    for (int i = tid; i < A.ninit; i += T) {
        const int4 im = __ldg(&A.inits[i]);
        const int gx = wrapi(pi * A.pw + bi * A.b - half + im.x, A.nx);
        const int gy = wrapi(pj * A.ph + bj * A.b - half + im.y, A.ny);
        const int opi = gx / A.pw, opj = gy / A.ph;
        const double* src = A.init_planes[opj * A.px + opi] + (long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw);
        const long pl = (long)A.pw * A.ph;
#pragma unroll
        for (int v = 0; v < 4; ++v) S[im.z + v * im.w] = src[v * pl];
    }
    cp_async_wait_all();
    __syncthreads();

    const int gh = A.ghost;
    double* dst = A.rec[part * A.nslots + A.my_slot] + ((long)(bj + gh) * A.extw + (bi + gh)) * 4 * A.epad;
    const bool edge = bi < gh || bi >= A.pbx - gh || bj < gh || bj >= A.pby - gh;
    auto flush = [&](int e0, int e1) {
        for (int e = e0 + tid; e < e1; e += T) {
            const int so = __ldg(&A.exp_off[e]), vs = __ldg(&A.exp_vs[e]);
            double val[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) val[v] = S[so + v * vs];
#pragma unroll
            for (int v = 0; v < 4; ++v) dst[v * A.epad + e] = val[v];
            if (edge)
                for (int ej = -1; ej <= 1; ++ej)
                    for (int ei = -1; ei <= 1; ++ei) {
                        if (ei == 0 && ej == 0) continue;
                        const int tbi = bi - ei * A.pbx, tbj = bj - ej * A.pby;
                        if (tbi < -gh || tbi >= A.pbx + gh || tbj < -gh || tbj >= A.pby + gh) continue;
                        const int tp = wrapi(pj + ej, A.py) * A.px + wrapi(pi + ei, A.px);
                        double* d = A.rec[tp * A.nslots + A.my_slot] + ((long)(tbj + gh) * A.extw + (tbi + gh)) * 4 * A.epad + e;
#pragma unroll
                        for (int v = 0; v < 4; ++v) d[v * A.epad] = val[v];
                    }
        }
    };

    for (int r = 1; r <= A.nlev; ++r) {
        const int stage = (A.stage0 + r - 1) & 1;
        const DevLevel Lc = A.lev[r - A.rmin];
        const DevLevel Lp = A.lev[r - 1 - A.rmin];
        const DevLevel Lb = stage == 1 ? A.lev[r - 2 - A.rmin] : Lp;
        auto Q = [&](int x, int y, int v) { return S[Lp.off + v * Lp.vstride + (y - Lp.by0) * Lp.bw + (x - Lp.bx0)]; };
        auto B = [&](int x, int y, int v) { return S[Lb.off + v * Lb.vstride + (y - Lb.by0) * Lb.bw + (x - Lb.bx0)]; };
        const bool out = r == A.r_out;
        const long lev = A.lo + r - 1;
        const bool snap = A.snap_every > 0 && lev % A.snap_every == 0;
        auto O = [&](int x, int y, const double o[4]) {
            double* d = S + Lc.off + (y - Lc.by0) * Lc.bw + (x - Lc.bx0);
#pragma unroll
            for (int v = 0; v < 4; ++v) d[v * Lc.vstride] = o[v];
            if (out || snap) {
                const int gx = wrapi(pi * A.pw + bi * A.b - half + x, A.nx);
                const int gy = wrapi(pj * A.ph + bj * A.b - half + y, A.ny);
                const int opi = gx / A.pw, opj = gy / A.ph;
                const long pl = (long)A.pw * A.ph;
                const long oo = (long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw);
                if (out) {
                    double* g = A.out_planes[opj * A.px + opi] + oo;
#pragma unroll
                    for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
                }
                if (snap) {
                    double* g = A.frames[opj * A.px + opi] + (lev % A.frame_ring) * 4 * pl + oo;
#pragma unroll
                    for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
                }
            }
        };
        euler_rect<FUSED>(tid, T, Lc.cx0, Lc.cx1, Lc.cy0, Lc.cy1, Q, B, O, ps, fxs, fys, A.c0, stage == 0 ? A.c1 : A.c3,
                   stage == 0 ? A.c2 : A.c4, err);
        if (r == A.split && A.nexp_early > 0) {
            flush(0, A.nexp_early);
            __syncthreads();
        }
    }
    if (A.nexp > A.nexp_early) flush(A.nexp_early, A.nexp);
    if (err) *A.err = 1;
    __syncthreads();  // (GM: the next instance reuses the scratch)
    }
}

// Standard Euler step on a TX x TY output tile per CTA: the cross-shaped
// radius-2 neighbourhood of the tile is staged in shared memory, then
// euler_rect (shared interface fluxes); boundary cells are pushed into the
// neighbouring partitions' ghost frames.
template <int TX, int TY, int MINB>
__global__ void __launch_bounds__(256, MINB) std_euler_kernel(const __grid_constant__ StdArgs A) {
    constexpr int QW = TX + 4, QH = TY + 4;
    __shared__ double q[4][QH][QW];
    __shared__ double ps[QH * QW];
    __shared__ double fxs[4 * TY * (TX + 1)];
    __shared__ double fys[4 * (TY + 1) * TX];
    const int tid = threadIdx.x, T = 256;
    const int part = A.dev_parts[blockIdx.z];
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int x1 = min(x0 + TX, A.pw), y1 = min(y0 + TY, A.ph);
    const int P = A.pitch;
    const long pl = (long)A.pitch * A.rows;
    const double* r1 = A.read1[part];
    // stage the tile + radius-2 frame (corners included; they are never used)
    for (int i = tid; i < QW * QH; i += T) {
        const int yy = i / QW, xx = i - yy * QW;
        const int x = x0 - 2 + xx, y = y0 - 2 + yy;
        if (x < -2 || x >= A.pw + 2 || y < -2 || y >= A.ph + 2) continue;
        const double* g = r1 + (long)(y + 2) * P + (x + 2);
#pragma unroll
        for (int v = 0; v < 4; ++v) q[v][yy][xx] = __ldg(g + v * pl);
    }
    __syncthreads();
    const int pi = part % A.px, pj = part / A.px;
    const double* r2 = A.read2[part];
    const bool corr = A.stage == 1;
    auto Q = [&](int x, int y, int v) { return q[v][y - y0 + 2][x - x0 + 2]; };
    auto B = [&](int x, int y, int v) {
        return corr ? __ldg(r2 + v * pl + (long)(y + 2) * P + (x + 2)) : q[v][y - y0 + 2][x - x0 + 2];
    };
    auto O = [&](int x, int y, const double o[4]) {
        const long idx = (long)(y + 2) * P + (x + 2);
#pragma unroll
        for (int v = 0; v < 4; ++v) A.out[part][idx + v * pl] = o[v];
        if (x < 2) {
            double* g = A.out[pj * A.px + (pi + A.px - 1) % A.px] + (long)(y + 2) * P + (x + A.pw + 2);
            for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
        }
        if (x >= A.pw - 2) {
            double* g = A.out[pj * A.px + (pi + 1) % A.px] + (long)(y + 2) * P + (x - A.pw + 2);
            for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
        }
        if (y < 2) {
            double* g = A.out[((pj + A.py - 1) % A.py) * A.px + pi] + (long)(y + A.ph + 2) * P + (x + 2);
            for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
        }
        if (y >= A.ph - 2) {
            double* g = A.out[((pj + 1) % A.py) * A.px + pi] + (long)(y - A.ph + 2) * P + (x + 2);
            for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
        }
    };
    int err = 0;
    euler_rect<true>(tid, T, x0, x1, y0, y1, Q, B, O, ps, fxs, fys, A.c0, A.c1, A.c2, err);
    if (err) *A.err = 1;
}

// Standard Euler step, column marching (no shared memory, no barriers): a
// warp owns 31 consecutive columns (lane L = column x0 - 1 + L) of a strip of
// ROWS rows and walks down it.  Per row j:
//   * y-interface j+1/2 (euler_row_fast's shared fluxes, physics.cpp:270-321):
//     the lane keeps its column's rows j-1..j+2 (and their pressures) in a
//     register window, one new row loaded per step; the flux of j-1/2 is the
//     previous step's j+1/2;
//   * x-interface x+1/2 from the cells x-1..x+2 of row j (the neighbours'
//     cells come from L1; their pressures are recomputed -- cheaper than the
//     divergent edge handling shuffles would need); the flux of x-1/2 is lane
//     L-1's, by shuffle (lane 0 only supplies it);
//   * out = base - cx*(fe - fw) - cy*(gn - gs) (physics.cpp:131-156), plus the
//     pushes of partition-edge cells into the neighbours' ghost frames.
// Non-physical states seen on a path an output cell needs raise the error flag.
template <int ROWS, int MINB = 4>
__global__ void __launch_bounds__(128, MINB) std_euler_col_kernel(const __grid_constant__ StdArgs A) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x0 = (blockIdx.x * 4 + warp) * 31;
    const int x = x0 - 1 + lane;
    if (x0 >= A.pw) return;  // whole warp past the partition
    const bool active = x < A.pw;         // computes a needed x-flux
    const bool outl = active && lane > 0;  // owns an output cell
    const int xc = active ? x : A.pw - 1;  // loads stay inside the ghosted plane
    const int ybeg = blockIdx.y * ROWS, yend = min(ybeg + ROWS, A.ph);
    const int part = A.dev_parts[blockIdx.z];
    const int P = A.pitch;
    const long pl = (long)A.pitch * A.rows;
    const double* r1 = A.read1[part];
    const double* bse = A.stage == 1 ? A.read2[part] : r1;
    double* out = A.out[part];
    const int pi = part % A.px, pj = part / A.px;
    const double gamma = A.c0, cx = A.c1, cy = A.c2;
    auto at = [&](int xx, int yy) { return (long)(yy + 2) * P + (xx + 2); };
    int errx = 0, erry = 0;
    // window: rows j-1, j, j+1, j+2 of column xc (w[0..3]) and their pressures
    double w[4][4], pw_[4], gs[4];
    auto load = [&](int yy, double q[4]) {
        const double* g = r1 + at(xc, yy);
#pragma unroll
        for (int v = 0; v < 4; ++v) q[v] = __ldg(g + v * pl);
    };
    // prologue: rows ybeg-2 .. ybeg+1 -> flux of ybeg-1/2
    {
        double t[4][4], tp[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            load(ybeg - 2 + k, t[k]);
            tp[k] = pressure_d(t[k], gamma, erry);
        }
        iface_flux_d<1>(t, tp, gamma, gs, erry);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
#pragma unroll
            for (int v = 0; v < 4; ++v) w[k][v] = t[k + 1][v];
            pw_[k] = tp[k + 1];
        }
    }
    // (issuing the next row's loads one step ahead was measured: +4 % at
    // 4096^2, -15 % at 960^2 from the lost occupancy at 162 registers; a 5th
    // or 6th resident CTA needs spills and is slower)
    auto load_x = [&](int yy, double q[3][4]) {
        const double* g = r1 + at(xc, yy);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            q[0][v] = __ldg(g - 1 + v * pl);
            q[1][v] = __ldg(g + 1 + v * pl);
            q[2][v] = __ldg(g + 2 + v * pl);
        }
    };
    for (int y = ybeg; y < yend; ++y) {
        // new row y+2 enters the window (rows y-1 .. y+2); x-stencil of row y
        double xs[3][4];
        load(y + 2, w[3]);
        load_x(y, xs);
        pw_[3] = pressure_d(w[3], gamma, erry);
        double gn[4];
        iface_flux_d<1>(w, pw_, gamma, gn, erry);
        // x-interface x+1/2 of row y: cells x-1, x, x+1, x+2
        double fe[4];
        {
            double q[4][4], p[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                q[0][v] = xs[0][v];
                q[1][v] = w[1][v];
                q[2][v] = xs[1][v];
                q[3][v] = xs[2][v];
            }
            p[0] = pressure_d(q[0], gamma, errx);
            p[1] = pw_[1];
            p[2] = pressure_d(q[2], gamma, errx);
            p[3] = pressure_d(q[3], gamma, errx);
            iface_flux_d<0>(q, p, gamma, fe, errx);
        }
        double o[4];
        const long idx = at(xc, y);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const double fw = __shfl_up_sync(0xffffffffu, fe[v], 1);
            o[v] = __ldg(bse + idx + v * pl) - cx * (fe[v] - fw) - cy * (gn[v] - gs[v]);
        }
        if (outl) {
#pragma unroll
            for (int v = 0; v < 4; ++v) out[idx + v * pl] = o[v];
            // partition-edge cells -> the neighbours' ghost frames (cross stencil: no corners)
            if (x < 2) {
                double* g = A.out[pj * A.px + (pi + A.px - 1) % A.px] + at(x + A.pw, y);
#pragma unroll
                for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
            }
            if (x >= A.pw - 2) {
                double* g = A.out[pj * A.px + (pi + 1) % A.px] + at(x - A.pw, y);
#pragma unroll
                for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
            }
            if (y < 2) {
                double* g = A.out[((pj + A.py - 1) % A.py) * A.px + pi] + at(x, y + A.ph);
#pragma unroll
                for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
            }
            if (y >= A.ph - 2) {
                double* g = A.out[((pj + 1) % A.py) * A.px + pi] + at(x, y - A.ph);
#pragma unroll
                for (int v = 0; v < 4; ++v) g[v * pl] = o[v];
            }
        }
        // slide
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            gs[v] = gn[v];
            w[0][v] = w[1][v];
            w[1][v] = w[2][v];
            w[2][v] = w[3][v];
        }
        pw_[0] = pw_[1];
        pw_[1] = pw_[2];
        pw_[2] = pw_[3];
    }
    if ((active && errx) || (outl && erry)) *A.err = 1;
}

// Standard heat step, column marching: a thread owns two adjacent columns of
// a 256 x ROWS tile and walks down them four rows per trip with 16-byte
// loads/stores; centre/south stay in registers and the E/W neighbours of the
// pair come from the L1-resident neighbouring pairs, so each plane value
// crosses HBM once.  Partition-edge cells are pushed into the neighbours'
// ghost frames by the same kernel (the fused halo export).  Requires pw even.
template <int ROWS>
__global__ void __launch_bounds__(128) std_heat_kernel(const __grid_constant__ StdArgs A) {
    const int x = 2 * (blockIdx.x * 128 + threadIdx.x);
    const int ybeg = blockIdx.y * ROWS;
    if (x >= A.pw) return;
    const int part = A.dev_parts[blockIdx.z];
    const int P = A.pitch;
    const int yend = min(ybeg + ROWS, A.ph);
    const double* r = A.read1[part] + (long)(ybeg + 1) * P + (x + 1);
    double* o = A.out[part] + (long)(ybeg + 1) * P + (x + 1);
    const int pi = part % A.px, pj = part / A.px;
    const double fx = A.c0, fy = A.c1;
    // ghost frame pitch is pw + 2 (odd offset +1): rows are 8-byte aligned only,
    // so the pair is loaded as two 8-byte loads the compiler merges where legal
    auto ld2 = [](const double* p) { return make_double2(__ldg(p), __ldg(p + 1)); };
    double2 south = ld2(r - P), c = ld2(r);
    int y = ybeg;
    auto row = [&](double2 cc, double2 nn, double2 ss, const double* rr, double* oo, int yy) {
        const double w = __ldg(rr - 1), e = __ldg(rr + 2);
        const double v0 = heat_update(cc.x, cc.y, w, nn.x, ss.x, fx, fy);
        const double v1 = heat_update(cc.y, e, cc.x, nn.y, ss.y, fx, fy);
        oo[0] = v0;
        oo[1] = v1;
        if (x == 0) A.out[pj * A.px + (pi + A.px - 1) % A.px][(long)(yy + 1) * P + (A.pw + 1)] = v0;
        if (x + 2 == A.pw) A.out[pj * A.px + (pi + 1) % A.px][(long)(yy + 1) * P] = v1;
        if (yy == 0) {
            double* g = A.out[((pj + A.py - 1) % A.py) * A.px + pi] + (long)(A.ph + 1) * P + (x + 1);
            g[0] = v0;
            g[1] = v1;
        }
        if (yy == A.ph - 1) {
            double* g = A.out[((pj + 1) % A.py) * A.px + pi] + (x + 1);
            g[0] = v0;
            g[1] = v1;
        }
    };
    for (; y + 4 <= yend; y += 4) {
        const double2 n1 = ld2(r + P), n2 = ld2(r + 2 * P), n3 = ld2(r + 3 * P), n4 = ld2(r + 4 * P);
        row(c, n1, south, r, o, y);
        row(n1, n2, c, r + P, o + P, y + 1);
        row(n2, n3, n1, r + 2 * P, o + 2 * P, y + 2);
        row(n3, n4, n2, r + 3 * P, o + 3 * P, y + 3);
        south = n3;
        c = n4;
        r += 4 * P;
        o += 4 * P;
    }
    for (; y < yend; ++y) {
        const double2 nn = ld2(r + P);
        row(c, nn, south, r, o, y);
        south = c;
        c = nn;
        r += P;
        o += P;
    }
}

template <int PROB>
__global__ void __launch_bounds__(256) std_step_kernel(const __grid_constant__ StdArgs A) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= A.pw || y >= A.ph) return;
    const int part = A.dev_parts[blockIdx.z];
    const int n = A.n, P = A.pitch;
    const long pl = (long)A.pitch * A.rows;
    const long idx = (long)(y + n) * P + (x + n);
    const double* r1 = A.read1[part] + idx;
    double outv[PROB == 0 ? 1 : 4];
    int err = 0;
    if (PROB == 0) {
        outv[0] = heat_update(__ldg(r1), __ldg(r1 + 1), __ldg(r1 - 1), __ldg(r1 + P), __ldg(r1 - P), A.c0, A.c1);
    } else {
        const double* b = (A.stage == 0 ? A.read1[part] : A.read2[part]) + idx;
        double q0[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) q0[v] = __ldg(b + v * pl);
        // c0 = gamma, (c1, c2) = (cx, cy) of this stage, set by the host
        euler_update_d([&](int dx, int dy, int v) { return __ldg(r1 + v * pl + (long)dy * P + dx); }, q0, A.c1,
                       A.c2, A.c0, outv, err);
    }
    constexpr int NV = PROB == 0 ? 1 : 4;
    const int pi = part % A.px, pj = part / A.px;
#pragma unroll
    for (int v = 0; v < NV; ++v) A.out[part][idx + v * pl] = outv[v];
    // push boundary cells into the neighbours' ghost frames (cross stencil: no corners)
    if (x < n) {
        double* o = A.out[pj * A.px + (pi + A.px - 1) % A.px] + (long)(y + n) * P + (x + A.pw + n);
        for (int v = 0; v < NV; ++v) o[v * pl] = outv[v];
    }
    if (x >= A.pw - n) {
        double* o = A.out[pj * A.px + (pi + 1) % A.px] + (long)(y + n) * P + (x - A.pw + n);
        for (int v = 0; v < NV; ++v) o[v * pl] = outv[v];
    }
    if (y < n) {
        double* o = A.out[((pj + A.py - 1) % A.py) * A.px + pi] + (long)(y + A.ph + n) * P + (x + n);
        for (int v = 0; v < NV; ++v) o[v * pl] = outv[v];
    }
    if (y >= A.ph - n) {
        double* o = A.out[((pj + 1) % A.py) * A.px + pi] + (long)(y - A.ph + n) * P + (x + n);
        for (int v = 0; v < NV; ++v) o[v * pl] = outv[v];
    }
    if (err) *A.err = 1;
}

// run_substep over rectangles (x in range, y wraps: GridView, field.hpp:12-24)
template <int PROB>
__global__ void substep_rects_kernel(int stage, const double* __restrict__ r1, const double* __restrict__ r2,
                                     double* __restrict__ out, int nx, int ny, const int* rects,
                                     const long* prefix, int nrects, double c0, double c1, double c2,
                                     double c3, int* errflag) {
    const long total = prefix[nrects];
    const long pl = (long)nx * ny;
    for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < total; c += (long)gridDim.x * blockDim.x) {
        // rectangle of cell c: the last ri with prefix[ri] <= c (binary search)
        int lo = 0, hi = nrects - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= c) lo = mid;
            else hi = mid - 1;
        }
        const int ri = lo;
        const int x0 = rects[4 * ri], w = rects[4 * ri + 1] - x0, y0 = rects[4 * ri + 2];
        const long rem = c - prefix[ri];
        const int x = x0 + (int)(rem % w), y = y0 + (int)(rem / w);
        auto row = [&](int yy) { return (long)wrapi(yy, ny) * nx; };
        int err = 0;
        if (PROB == 0) {
            const double cc = r1[row(y) + x];
            out[row(y) + x] =
                heat_update(cc, r1[row(y) + x + 1], r1[row(y) + x - 1], r1[row(y + 1) + x], r1[row(y - 1) + x], c0, c1);
        } else {
            const double* b = stage == 0 ? r1 : r2;
            double q0[4], o[4];
            for (int v = 0; v < 4; ++v) q0[v] = b[v * pl + row(y) + x];
            euler_update_d([&](int dx, int dy, int v) { return r1[v * pl + row(y + dy) + x + dx]; }, q0,
                           c1, c2, c0, o, err);
            for (int v = 0; v < 4; ++v) out[v * pl + row(y) + x] = o[v];
        }
        if (err) *errflag = 1;
    }
}

// Cross-process barrier between dependent launches of a distributed run (one
// process per GPU): publish this rank's epoch into every peer's flag array
// (system-scope release after the previous kernel's P2P stores), then wait
// until every peer has published the same epoch into ours.  Bounded: after
// 60 s without progress it raises bit 1 of the error flag (TransportError)
// instead of hanging the GPU.
__global__ void dist_barrier_kernel(unsigned long long* const* peer_flags, unsigned long long* my_flags, int world,
                                    int rank, unsigned long long* counter, int* err) {
    if (threadIdx.x != 0) return;
    // the epoch lives on the device (every rank passes the same sequence of
    // barriers), so a solve's launches can be replayed from a CUDA graph
    const unsigned long long epoch = *counter + 1;
    *counter = epoch;
    __threadfence_system();
    for (int q = 0; q < world; ++q) {
        unsigned long long* f = peer_flags[q] + rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
    }
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int q = 0; q < world; ++q) {
        while (true) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + q) : "memory");
            if (v >= epoch) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 60ull * 1000000000ull) {
                atomicOr(err, 2);
                return;
            }
            __nanosleep(200);
        }
    }
    __threadfence_system();
}

// FP64 pipe peak without FMA (the solver's arithmetic, -fmad=false): 8
// independent DADD/DMUL chains per thread, 2 ops per chain step.
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = x[k] * a + b;  // DMUL + DADD (no contraction)
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5) out[0] = s;  // keep the chains alive
}

}  // namespace

double measure_fp64_peak() {
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = nsm * 8, iters = 4096;
    fp64_peak_kernel<<<blocks, 256>>>(out, 64, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        fp64_peak_kernel<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return -1.0;
    return 2.0 * 8.0 * iters * blocks * 256.0 / (best * 1e-3);
}

// div_dn / div_nb / sqrt_nb self-test: operands are random bit patterns (every exponent,
// zeros, subnormals, infinities, NaNs included) plus, every fourth pair,
// "physical" operands (the magnitudes the Euler fluxes divide); a mismatch is
// any pair where div_dn(x, y, recip_dn(y)) and x / y differ in bits (two NaNs
// count as equal).
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long& s) {
    unsigned long long z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__global__ void div_selftest_kernel(long n, unsigned long long seed, unsigned long long* bad,
                                    double* first_bad) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        unsigned long long st = seed ^ (0x632be59bd9b4e019ull * (unsigned long long)(i + 1));
        const unsigned long long a = splitmix64(st), b = splitmix64(st);
        double x = __longlong_as_double((long long)a), y = __longlong_as_double((long long)b);
        if ((i & 3) == 3) {  // physical magnitudes: x in +-[1e-3, 1e3], y in [1e-2, 1e2]
            x = (a & 1 ? -1.0 : 1.0) * exp10(-3.0 + 6.0 * ((a >> 11) * 0x1.0p-53));
            y = exp10(-2.0 + 4.0 * ((b >> 11) * 0x1.0p-53));
        }
        if ((i & 255) == 7) y = 0.0;
        if ((i & 255) == 9) x = 0.0;
        const double q1 = x / y, q2 = div_dn(x, y, recip_dn(y));
        bool ok = true;
        double q3 = div_nb(x, y, recip_dn(y), ok);
        if (!ok) q3 = x / y;
        // sqrt: the same operands as |x| (and x itself: negative / NaN cases)
        const double sa = (i & 1) ? fabs(x) : x;
        const double s1 = sqrt(sa);
        bool oks = true;
        double s2 = sqrt_nb(sa, oks);
        if (!oks) s2 = sqrt(sa);
        auto eq = [](double u, double w) {
            return __double_as_longlong(u) == __double_as_longlong(w) || (isnan(u) && isnan(w));
        };
        const bool same = eq(q1, q2) && eq(q1, q3) && eq(s1, s2);
        if (!same) {
            if (atomicAdd(bad, 1ull) == 0ull) {
                first_bad[0] = x;
                first_bad[1] = y;
            }
        }
    }
}

long div_selftest(long n, unsigned long long seed, double* xy_bad) {
    unsigned long long* bad = nullptr;
    double* fb = nullptr;
    if (cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (cudaMalloc(&fb, 2 * sizeof(double)) != cudaSuccess) return -1;
    cudaMemset(bad, 0, sizeof(unsigned long long));
    div_selftest_kernel<<<148 * 16, 256>>>(n, seed, bad, fb);
    unsigned long long h = 0;
    double hb[2] = {0, 0};
    const bool ok = cudaMemcpy(&h, bad, sizeof h, cudaMemcpyDeviceToHost) == cudaSuccess &&
                    cudaMemcpy(hb, fb, sizeof hb, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(bad);
    cudaFree(fb);
    if (!ok) return -1;
    if (xy_bad) {
        xy_bad[0] = hb[0];
        xy_bad[1] = hb[1];
    }
    return static_cast<long>(h);
}

cudaError_t launch_dist_barrier(unsigned long long* const* peer_flags, unsigned long long* my_flags, int world,
                                int rank, unsigned long long* counter, int* err, cudaStream_t s) {
    dist_barrier_kernel<<<1, 32, 0, s>>>(peer_flags, my_flags, world, rank, counter, err);
    return cudaGetLastError();
}

cudaError_t launch_heat_col8(const SweptArgs& a, cudaStream_t s);
cudaError_t launch_heat_col12(const SweptArgs& a, cudaStream_t s);
cudaError_t launch_heat_col16(const SweptArgs& a, cudaStream_t s);
cudaError_t launch_heat_col24(const SweptArgs& a, cudaStream_t s);
cudaError_t launch_heat_col32(const SweptArgs& a, cudaStream_t s);

cudaError_t launch_swept(int problem, const SweptArgs& a, cudaStream_t s) {
    const int ninst = a.pbx * a.pby;
    if (problem == 0 && a.colB == 16) return launch_heat_col16(a, s);
    if (problem == 0 && a.colB == 8) return launch_heat_col8(a, s);
    if (problem == 0 && a.colB == 32) return launch_heat_col32(a, s);
    if (problem == 0 && a.colB == 12) return launch_heat_col12(a, s);
    if (problem == 0 && a.colB == 24) return launch_heat_col24(a, s);
    if (problem == 0 && a.gm_scratch) {
        dim3 grid(a.gm_ctas, a.ndev_parts);
        swept_heat_kernel<4, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (problem == 1 && a.gm_scratch) {
        dim3 grid(a.gm_ctas, a.ndev_parts);
        swept_euler_kernel<4, 128, true, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (problem == 0) {
        const size_t per_inst = static_cast<size_t>(a.smem_doubles) * sizeof(double);
        auto go = [&](auto kern, int wpc) {
            const size_t smem = wpc * per_inst;
            if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            dim3 grid((ninst + wpc - 1) / wpc, a.ndev_parts);
            kern<<<grid, wpc * 32, smem, s>>>(a);
            return cudaGetLastError();
        };
        if (4 * per_inst <= 64 * 1024) return go(swept_heat_kernel<4>, 4);
        if (2 * per_inst <= 100 * 1024) return go(swept_heat_kernel<2>, 2);
        return go(swept_heat_kernel<1>, 1);
    }
    {
        const size_t smem = static_cast<size_t>(a.smem_doubles + a.ps_doubles + 2 * a.fx_doubles) * sizeof(double);
        // 6-7 resident CTAs: occupancy hides the FP64 dependency chains and
        // the per-level barriers (1.09e10 at 72 registers vs 8.5e9 at 112,
        // Euler 960^2 b16); 6 (<= 80 registers) since the branch-free flux
        // code: 1.20e10 vs 1.16e10 (7 CTAs, more spills)
        static const int minb = [] { const char* v = std::getenv("SG_EULER_MINB"); return v ? std::atoi(v) : 6; }();
        // x- and y-interface fluxes in one balanced loop (+3 % at 960^2; 160-
        // and 192-thread CTAs measured slower: 1.14e10 / 1.05e10 vs 1.23e10)
        dim3 grid(ninst, a.ndev_parts);
        auto go = [&](auto kern) {
            if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kern<<<grid, 128, smem, s>>>(a);
            return cudaGetLastError();
        };
        if (minb == 5) return go(swept_euler_kernel<5, 128, true>);
        if (minb == 7) return go(swept_euler_kernel<7, 128, true>);
        return go(swept_euler_kernel<6, 128, true>);
    }
}

cudaError_t launch_std(int problem, const StdArgs& a, cudaStream_t s) {
    if (problem == 0 && a.pw % 2 == 0) {
        constexpr int ROWS = 32;
        dim3 grid((a.pw / 2 + 127) / 128, (a.ph + ROWS - 1) / ROWS, a.ndev_parts);
        std_heat_kernel<ROWS><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (problem == 1 && !std::getenv("SG_EULER_TILE")) {
        // column marching: 124 columns x ROWS rows per 4-warp CTA; ROWS as
        // large as keeps ~16 warps per SM busy (each strip re-reads 3 rows)
        const long warps = (a.pw + 123) / 124 * 4L * a.ndev_parts;
        const long want_rows = a.ph * warps / (148L * 16);
        dim3 grid((a.pw + 123) / 124, 1, a.ndev_parts);
        auto go = [&](auto kern, int rows) {
            grid.y = (a.ph + rows - 1) / rows;
            kern<<<grid, 128, 0, s>>>(a);
            return cudaGetLastError();
        };
        // large grids (>= 16-row strips, plenty of warps): 5 resident CTAs
        // at 96 registers (some spills) beat 4 at 128 (4096^2: 2.18e10 vs
        // 2.08e10); the 960^2 grid keeps 4 (1.81e10 vs 1.76e10)
        static const int minb = [] { const char* v = std::getenv("SG_EULER_STD_MINB"); return v ? std::atoi(v) : 0; }();
        if (minb == 5 || (minb == 0 && want_rows >= 16)) {
            if (want_rows >= 64) return go(std_euler_col_kernel<64, 5>, 64);
            if (want_rows >= 32) return go(std_euler_col_kernel<32, 5>, 32);
            if (want_rows >= 16) return go(std_euler_col_kernel<16, 5>, 16);
            return go(std_euler_col_kernel<8, 5>, 8);
        }
        if (want_rows >= 64) return go(std_euler_col_kernel<64>, 64);
        if (want_rows >= 32) return go(std_euler_col_kernel<32>, 32);
        if (want_rows >= 16) return go(std_euler_col_kernel<16>, 16);
        return go(std_euler_col_kernel<8>, 8);
    }
    if (problem == 1) {
        // 32 x 7: the fused flux step has 7*33 + 8*32 = 487 items = two rounds of 256
        constexpr int TX = 32, TY = 7;
        dim3 grid((a.pw + TX - 1) / TX, (a.ph + TY - 1) / TY, a.ndev_parts);
        // 4 resident CTAs (64 registers, no spills): 1.58e10 vs 1.01e10 at 96
        std_euler_kernel<TX, TY, 4><<<grid, 256, 0, s>>>(a);
        return cudaGetLastError();
    }
    dim3 block(32, 8);
    dim3 grid((a.pw + 31) / 32, (a.ph + 7) / 8, a.ndev_parts);
    if (problem == 0) std_step_kernel<0><<<grid, block, 0, s>>>(a);
    else std_step_kernel<1><<<grid, block, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_substep(int problem, int stage, const double* r1, const double* r2, double* out, int nx,
                           int ny, const int* d_rects, const long* d_prefix, int nrects, long total,
                           const double* c, int* d_err, cudaStream_t s) {
    if (total <= 0) return cudaSuccess;
    const int threads = 256;
    const int grid = static_cast<int>(std::min<long>((total + threads - 1) / threads, 148L * 16));
    if (problem == 0)
        substep_rects_kernel<0><<<grid, threads, 0, s>>>(stage, r1, r2, out, nx, ny, d_rects, d_prefix, nrects,
                                                         c[0], c[1], c[2], c[3], d_err);
    else
        substep_rects_kernel<1><<<grid, threads, 0, s>>>(stage, r1, r2, out, nx, ny, d_rects, d_prefix, nrects,
                                                         c[0], c[1], c[2], c[3], d_err);
    return cudaGetLastError();
}

}  // namespace sg
