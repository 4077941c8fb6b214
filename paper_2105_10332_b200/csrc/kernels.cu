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

#include "colgeom.hpp"
#include "kernels.cuh"
#include "physics.cuh"

namespace sg {

namespace {

__device__ __forceinline__ int wrapi(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}

// Table loads that should stay in L1: the gathers' cp.async.ca traffic would
// otherwise evict the small per-launch tables from the L1 left over by shared
// memory.
__device__ __forceinline__ int4 ldg_keep(const int4* p) {
    int4 v;
    asm("ld.global.nc.L1::evict_last.v4.s32 {%0, %1, %2, %3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p));
    return v;
}
__device__ __forceinline__ int2 ldg_keep(const int2* p) {
    int2 v;
    asm("ld.global.nc.L1::evict_last.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned ldg_keep(const unsigned* p) {
    unsigned v;
    asm("ld.global.nc.L1::evict_last.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ldg_keep(const int* p) {
    int v;
    asm("ld.global.nc.L1::evict_last.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

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
template <int WPC>
__global__ void __launch_bounds__(WPC * 32) swept_heat_kernel(const __grid_constant__ SweptArgs A) {
    extern __shared__ double sm[];
    __shared__ const double* segbase[WPC][kMaxSegs];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ninst = A.pbx * A.pby;
    const int inst = blockIdx.x * WPC + warp;
    if (inst >= ninst) return;
    const int part = A.dev_parts[blockIdx.y];
    const int pi = part % A.px, pj = part / A.px;
    const int bi = inst % A.pbx, bj = inst / A.pbx;
    const int half = A.frame * (A.b / 2);
    double* S = sm + warp * A.smem_doubles;
    const double** sb = segbase[warp];

    // ---- 1. gather
    if (lane < A.nsegs) {
        const DevSeg sg = A.segs[lane];
        const long ext = (long)(bj + sg.dj + A.ghost) * A.extw + (bi + sg.di + A.ghost);
        sb[lane] = A.rec[part * A.nslots + sg.slot] + ext * sg.epad;
    }
    __syncwarp();
    {
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
        int x = 0, y0 = 0, n = 0;
        if (lane < L.items) {
            // item -> (column, row chunk); exact (items < 2^5, w <= 2^5)
            const int ch = __float2int_rz((lane + 0.5f) * L.inv_w);
            x = L.cx0 + (lane - ch * L.w);
            y0 = L.cy0 + ch * L.rps;
            n = min(L.rps, L.cy1 - y0);
        }
        if (n > 0) {
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
        }
        __syncwarp();
        if (r == A.split && A.nexp_early > 0) {
            flush(0, A.nexp_early);
            __syncwarp();
        }
    }
    // ---- 3. scatter the rest of the record
    if (A.nexp > A.nexp_early) flush(A.nexp_early, A.nexp);
}

// Predicated shared load / global store (one instruction, no branch).
__device__ __forceinline__ void lds_if(double& v, unsigned saddr, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f64 %0, [%1];\n\t}"
                 : "+d"(v)
                 : "r"(saddr), "r"(static_cast<int>(p)));
}
__device__ __forceinline__ void stg_if(double* g, double v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}" ::"l"(g), "d"(v),
                 "r"(static_cast<int>(p)));
}

// Compile-time loop: f(std::integral_constant<int, I>) for I = 0..N-1.
template <class F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
    sfor_impl(f, std::make_integer_sequence<int, N>{});
}

// Writes cells stash[i], i in [i0, i1), of one lane's line (a column when
// (dx, dy) = (0, 1), a row when (1, 0)) to the owning partitions' output plane
// and/or snapshot frame; cell i sits at (x0 + i*dx, y0 + i*dy) relative to the
// partition origin (both may wrap).
__device__ __noinline__ void put_cells(const SweptArgs& A, const double* stash, int i0, int i1, int pi, int pj, int x0,
                                       int y0, int dx, int dy, long lev, bool out, bool snap) {
    const long pl = (long)A.pw * A.ph;
    for (int i = i0; i < i1; ++i) {
        const int gx = wrapi(pi * A.pw + x0 + i * dx, A.nx);
        const int gy = wrapi(pj * A.ph + y0 + i * dy, A.ny);
        const int opi = gx / A.pw, opj = gy / A.ph;
        const long o = (long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw);
        if (out) A.out_planes[opj * A.px + opi][o] = stash[i];
        if (snap) A.frames[opj * A.px + opi][(lev % A.frame_ring) * pl + o] = stash[i];
    }
}

// Heat phase kernel, register-tile form (block B in {8, 16, 32}, geometry in
// colgeom.hpp).  L = B/CPL lanes own one phase instance (32/L instances per
// warp, WPC warps per CTA).  At each level the instance's B x B window lives
// in the lanes' registers, in one of two layouts (col::mode):
//   COL: lane l holds columns c = CPL*l + q, v[q][i] = row ylo + i;
//   ROW: lane l holds rows ylo + CPL*l + q, v[q][x] = column x.
// The bridges switch layout once (a transpose through shared memory) so that
// every level iterates over the shorter side of its rectangle.  Per level r
// (geometry compile-time, levels and cells fully unrolled):
//   1. imports: cells of level r-1 this instance did not compute come from
//      shared memory, where the gather landed them (predicated LDS);
//   2. update R_r in place: neighbours along a lane's lines and between its
//      own CPL lines are registers; across lanes they come from lanes +-1 by
//      warp shuffle, one 64-bit shuffle each way per CPL lines (heat_point,
//      physics.hpp:57-63; no FMA);
//   3. exports: the cells of R_r that other instances read go from registers
//      into this instance's record (predicated stores).
// Lanes outside R_r compute too (SIMT); their cells are never read before an
// import overwrites them.
template <int B, int KIND, int CPL, int WPC>
__global__ void __launch_bounds__(WPC * 32) swept_heat_col_kernel(const __grid_constant__ SweptArgs A) {
    constexpr int L = B / CPL;      // lanes per instance
    constexpr int IPW = 32 / L;     // instances per warp
    constexpr int IPC = WPC * IPW;  // instances per CTA
    constexpr int NL = col::nlev(KIND, B);
    constexpr int YLO = col::ylo(KIND, B);
    constexpr int NIMP = col::imp_total(KIND, B);  // import slots; the transpose tile follows
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // b = 12 / 24: the last 32 - IPW*L lanes of a warp are dead (they run the
    // code, shuffles included, but never write anything)
    const bool dead = lane >= IPW * L;
    const int sub = dead ? 0 : lane / L, l = lane % L;
    const int slot_in_cta = warp * IPW + sub;
    const int ninst = A.pbx * A.pby;
    // odd launches walk the instances backwards: their first CTAs read the
    // records the previous launch wrote last (still in L2)
    const int cta = (A.lo_parity & 1) ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const int inst = cta * IPC + slot_in_cta;
    const bool live = !dead && inst < ninst;
    const int part = A.dev_parts[blockIdx.y];
    const int pi = part % A.px, pj = part / A.px;
    const int bi = live ? inst % A.pbx : 0, bj = live ? inst / A.pbx : 0;
    const int half = A.frame * (B / 2);
    const int gh = A.ghost;
    double* S = sm + slot_in_cta * A.smem_doubles;

    // ---- gather the imports: {offset from this instance's slot-0 record, smem slot}
    if (live) {
        const double* ibase = A.rec[part * A.nslots] + ((long)(bj + gh) * A.extw + (bi + gh)) * A.epad;
        // part A (levels <= gather_split), one cp.async group, then part B
        const int na = A.nimp - A.nimp_b;
        int i = l;
        for (; i + 3 * L < na; i += 4 * L) {
            const int2 e0 = ldg_keep(&A.imp_off[i]), e1 = ldg_keep(&A.imp_off[i + L]);
            const int2 e2 = ldg_keep(&A.imp_off[i + 2 * L]), e3 = ldg_keep(&A.imp_off[i + 3 * L]);
            cp_async8(S + e0.y, ibase + e0.x);
            cp_async8(S + e1.y, ibase + e1.x);
            cp_async8(S + e2.y, ibase + e2.x);
            cp_async8(S + e3.y, ibase + e3.x);
        }
        for (; i < na; i += L) {
            const int2 e = ldg_keep(&A.imp_off[i]);
            cp_async8(S + e.y, ibase + e.x);
        }
        cp_async_commit();
        i = na + l;
        for (; i + 3 * L < A.nimp; i += 4 * L) {
            const int2 e0 = ldg_keep(&A.imp_off[i]), e1 = ldg_keep(&A.imp_off[i + L]);
            const int2 e2 = ldg_keep(&A.imp_off[i + 2 * L]), e3 = ldg_keep(&A.imp_off[i + 3 * L]);
            cp_async8(S + e0.y, ibase + e0.x);
            cp_async8(S + e1.y, ibase + e1.x);
            cp_async8(S + e2.y, ibase + e2.x);
            cp_async8(S + e3.y, ibase + e3.x);
        }
        for (; i < A.nimp; i += L) {
            const int2 e = ldg_keep(&A.imp_off[i]);
            cp_async8(S + e.y, ibase + e.x);
        }
        for (int j = l; j < A.ninit; j += L) {
            const int4 im = __ldg(&A.inits[j]);
            const int gx = wrapi(pi * A.pw + bi * B - half + im.x, A.nx);
            const int gy = wrapi(pj * A.ph + bj * B - half + im.y, A.ny);
            const int opi = gx / A.pw, opj = gy / A.ph;
            S[im.z] = A.init_planes[opj * A.px + opi][(long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw)];
        }
    }
    cp_async_commit();
    cp_async_wait_group<1>();  // part A (part B may still be in flight)
    __syncwarp();

    double* dst = A.rec[part * A.nslots + A.my_slot] + ((long)(bj + gh) * A.extw + (bi + gh)) * A.epad;
    const double fx = A.c0, fy = A.c1;
    const unsigned s_imp = static_cast<unsigned>(__cvta_generic_to_shared(S));
    double* tile = S + NIMP;
    // output stash (only allocated by launches that write the output level or snapshots)
    double* stash = sm + IPC * A.smem_doubles + (slot_in_cta * L + l) * CPL * B;
    double v[CPL][B];
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int i = 0; i < B; ++i) v[q][i] = 0.0;

    sfor<NL>([&](auto RI) {
        constexpr int r = decltype(RI)::value + 1;
        constexpr int MODE = col::mode(KIND, B, r);
        constexpr col::CRect q0 = col::rect(KIND, B, r);
        if constexpr (r == col::gather_split(KIND, B) + 1) {
            cp_async_wait_all();  // part B
            __syncwarp();
        }
        // ---------------- 1. imports of level r-1
        if constexpr (MODE == col::COL) {
            bool ip[CPL][4];
            unsigned ia[CPL][4];
            sfor<4>([&](auto TI) {
                constexpr int t = decltype(TI)::value;
                constexpr col::RowSet ts = col::Geo<KIND, B>::t.imp_tset[r][t];
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int c = CPL * l + q;
                    ip[q][t] = ts.count() > 0 && ts.has(c);
                    ia[q][t] = s_imp + 8u * static_cast<unsigned>(ts.count() > 0 ? ts.rank(c) : 0);
                }
            });
            sfor<B>([&](auto YI) {
                constexpr int j = decltype(YI)::value;
                constexpr int t = col::Geo<KIND, B>::t.imp_type[r][j];
                constexpr int base = col::Geo<KIND, B>::t.imp_base[r][j];
                if constexpr (t >= 0) {
#pragma unroll
                    for (int q = 0; q < CPL; ++q) lds_if(v[q][j], ia[q][t] + 8u * base, ip[q][t]);
                }
            });
        } else {
            int myt[CPL], mybase[CPL];
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int i = CPL * l + q;
                myt[q] = -1;
                mybase[q] = 0;
                sfor<col::kMaxRuns>([&](auto UI) {
                    constexpr col::Run ru = col::Geo<KIND, B>::t.imp_runs[r][decltype(UI)::value];
                    if constexpr (ru.t >= 0)
                        if (i >= ru.i0 && i < ru.i1) {
                            myt[q] = ru.t;
                            mybase[q] = ru.base + (i - ru.i0) * ru.cnt;
                        }
                });
            }
            sfor<4>([&](auto TI) {
                constexpr int t = decltype(TI)::value;
                constexpr col::RowSet ts = col::Geo<KIND, B>::t.imp_tset[r][t];
                if constexpr (ts.count() > 0) {
                    sfor<B>([&](auto XI) {
                        constexpr int x = decltype(XI)::value;
                        constexpr col::RowSet tx = col::Geo<KIND, B>::t.imp_tset[r][t];
                        constexpr int rk = tx.rank(x);
                        if constexpr (tx.has(x)) {
#pragma unroll
                            for (int q = 0; q < CPL; ++q)
                                lds_if(v[q][x], s_imp + 8u * static_cast<unsigned>(mybase[q] + rk), myt[q] == t);
                        }
                    });
                }
            });
        }
        // ---------------- 2. update R_r in place
        if constexpr (MODE == col::COL) {
            double prev[CPL];  // old values of the row below
#pragma unroll
            for (int q = 0; q < CPL; ++q) prev[q] = v[q][q0.y0 - 1 - YLO];
            sfor<B>([&](auto YI) {
                constexpr int j = decltype(YI)::value;
                constexpr col::CRect qr = col::rect(KIND, B, r);
                if constexpr (YLO + j >= qr.y0 && YLO + j < qr.y1) {
                    double cur[CPL];
#pragma unroll
                    for (int q = 0; q < CPL; ++q) cur[q] = v[q][j];
                    const double east = __shfl_down_sync(0xffffffffu, cur[0], 1);
                    const double west = __shfl_up_sync(0xffffffffu, cur[CPL - 1], 1);
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const double e = q + 1 < CPL ? cur[q + 1 < CPL ? q + 1 : 0] : east;
                        const double w = q > 0 ? cur[q > 0 ? q - 1 : 0] : west;
                        v[q][j] = heat_update(cur[q], e, w, v[q][j + 1], prev[q], fx, fy);
                        prev[q] = cur[q];
                    }
                }
            });
        } else {
            double prev[CPL];  // old values of the column to the west
#pragma unroll
            for (int q = 0; q < CPL; ++q) prev[q] = v[q][q0.x0 - 1];
            sfor<B>([&](auto XI) {
                constexpr int x = decltype(XI)::value;
                constexpr col::CRect qr = col::rect(KIND, B, r);
                if constexpr (x >= qr.x0 && x < qr.x1) {
                    double cur[CPL];
#pragma unroll
                    for (int q = 0; q < CPL; ++q) cur[q] = v[q][x];
                    const double north = __shfl_down_sync(0xffffffffu, cur[0], 1);
                    const double south = __shfl_up_sync(0xffffffffu, cur[CPL - 1], 1);
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const double n = q + 1 < CPL ? cur[q + 1 < CPL ? q + 1 : 0] : north;
                        const double sv = q > 0 ? cur[q > 0 ? q - 1 : 0] : south;
                        v[q][x] = heat_update(cur[q], v[q][x + 1], prev[q], n, sv, fx, fy);
                        prev[q] = cur[q];
                    }
                }
            });
        }
        // ---------------- 3. exports of level r (grouped layout, colgeom.hpp ExpLev)
        if constexpr (col::grouped_exports(B)) if (live) {
            constexpr col::ExpLev E = col::Geo<KIND, B>::t.exp.lev[r];
            if constexpr (E.count() > 0) {
                if constexpr (MODE == col::COL) {
                    bool pb[CPL], pm[CPL];
                    double* gh_[CPL];
                    double* gc[CPL];
                    double* gm[CPL];
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = CPL * l + q;
                        pb[q] = E.band(c);
                        pm[q] = E.mid(c) && c >= E.x0 && c < E.x1;
                        const int rb = pb[q] ? E.rank_band(c) : 0;
                        gh_[q] = dst + (E.g1 + rb - E.yh0 * E.bw());  // hole rows: + y * bw
                        gc[q] = dst + (E.g3 + rb);                     // full rows, band: + f * bw
                        gm[q] = dst + (E.g2 + (pm[q] ? c - E.mp : 0)); // full rows, middle: + f * mw
                    }
                    sfor<B>([&](auto YI) {
                        constexpr int j = decltype(YI)::value;
                        constexpr col::ExpLev Ej = col::Geo<KIND, B>::t.exp.lev[r];
                        constexpr int y = YLO + j;
                        constexpr int f = Ej.full_index(y);
                        if constexpr (Ej.hole_row(y)) {
#pragma unroll
                            for (int q = 0; q < CPL; ++q) stg_if(gh_[q] + y * Ej.bw(), v[q][j], pb[q]);
                        } else if constexpr (f >= 0) {
                            if constexpr (Ej.bw() > 0) {
#pragma unroll
                                for (int q = 0; q < CPL; ++q) stg_if(gc[q] + f * Ej.bw(), v[q][j], pb[q]);
                            }
#pragma unroll
                            for (int q = 0; q < CPL; ++q) stg_if(gm[q] + f * Ej.mw(), v[q][j], pm[q]);
                        }
                    });
                } else {
                    bool pbr[CPL], pmr[CPL];
                    double* gb[CPL];
                    double* gm[CPL];
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int y = YLO + CPL * l + q;  // the lane's window row
                        const bool hole = E.hole_row(y);
                        const int f = E.full_index(y);
                        pbr[q] = hole || f >= 0;
                        pmr[q] = f >= 0;
                        gb[q] = dst + (hole ? E.g1 + (y - E.yh0) * E.bw() : E.g3 + (f >= 0 ? f : 0) * E.bw());
                        gm[q] = dst + (E.g2 + (f >= 0 ? f : 0) * E.mw() - E.mp);
                    }
                    sfor<B>([&](auto XI) {
                        constexpr int x = decltype(XI)::value;
                        constexpr col::ExpLev Ex = col::Geo<KIND, B>::t.exp.lev[r];
                        if constexpr (Ex.band(x)) {
                            constexpr int rk = Ex.rank_band(x);
#pragma unroll
                            for (int q = 0; q < CPL; ++q) stg_if(gb[q] + rk, v[q][x], pbr[q]);
                        } else if constexpr (Ex.mid(x) && x >= Ex.x0 && x < Ex.x1) {
#pragma unroll
                            for (int q = 0; q < CPL; ++q) stg_if(gm[q] + x, v[q][x], pmr[q]);
                        }
                    });
                }
            }
        }
        // b = 32: row-major record (colgeom.hpp grouped_exports)
        if constexpr (!col::grouped_exports(B)) if (live) {
            if constexpr (MODE == col::COL) {
                bool ep[CPL][2];
                double* eg[CPL][2];
                sfor<2>([&](auto TI) {
                    constexpr int t = decltype(TI)::value;
                    constexpr col::RowSet ts = col::Geo<KIND, B>::t.exp_tset[r][t];
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = CPL * l + q;
                        ep[q][t] = ts.count() > 0 && ts.has(c);
                        eg[q][t] = dst + (ts.count() > 0 ? ts.rank(c) : 0);
                    }
                });
                sfor<B>([&](auto YI) {
                    constexpr int j = decltype(YI)::value;
                    constexpr int t = col::Geo<KIND, B>::t.exp_type[r][j];
                    constexpr int base = col::Geo<KIND, B>::t.exp_base[r][j];
                    static_assert(t < 2, "export row types");
                    if constexpr (t >= 0) {
#pragma unroll
                        for (int q = 0; q < CPL; ++q) stg_if(eg[q][t] + base, v[q][j], ep[q][t]);
                    }
                });
            } else {
                int myt[CPL];
                double* eb[CPL];
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int i = CPL * l + q;
                    myt[q] = -1;
                    int mybase = 0;
                    sfor<col::kMaxRuns>([&](auto UI) {
                        constexpr col::Run ru = col::Geo<KIND, B>::t.exp_runs[r][decltype(UI)::value];
                        if constexpr (ru.t >= 0)
                            if (i >= ru.i0 && i < ru.i1) {
                                myt[q] = ru.t;
                                mybase = ru.base + (i - ru.i0) * ru.cnt;
                            }
                    });
                    eb[q] = dst + mybase;
                }
                sfor<2>([&](auto TI) {
                    constexpr int t = decltype(TI)::value;
                    constexpr col::RowSet ts = col::Geo<KIND, B>::t.exp_tset[r][t];
                    if constexpr (ts.count() > 0) {
                        sfor<B>([&](auto XI) {
                            constexpr int x = decltype(XI)::value;
                            constexpr col::RowSet tx = col::Geo<KIND, B>::t.exp_tset[r][t];
                            constexpr int rk = tx.rank(x);
                            if constexpr (tx.has(x)) {
#pragma unroll
                                for (int q = 0; q < CPL; ++q) stg_if(eb[q] + rk, v[q][x], myt[q] == t);
                            }
                        });
                    }
                });
            }
        }
        // ---------------- output level / snapshot (rare): through the lane's
        // shared-memory stash to a non-inlined writer
        if ((((A.out_mask | A.snap_mask) >> r) & 1ull) && !dead) {
#pragma unroll
            for (int q = 0; q < CPL; ++q)
#pragma unroll
                for (int i = 0; i < B; ++i) stash[q * B + i] = v[q][i];
            const long lev = A.lo + r - 1;
            const bool o = (A.out_mask >> r) & 1ull, sn = (A.snap_mask >> r) & 1ull;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int m = CPL * l + q;  // the lane's column (COL) or window row (ROW)
                if constexpr (MODE == col::COL) {
                    if (live && m >= q0.x0 && m < q0.x1)
                        put_cells(A, stash + q * B, q0.y0 - YLO, q0.y1 - YLO, pi, pj, bi * B - half + m,
                                  bj * B - half + YLO, 0, 1, lev, o, sn);
                } else {
                    if (live && YLO + m >= q0.y0 && YLO + m < q0.y1)
                        put_cells(A, stash + q * B, q0.x0, q0.x1, pi, pj, bi * B - half, bj * B - half + YLO + m, 1,
                                  0, lev, o, sn);
                }
            }
        }
        // ---------------- layout switch after this level: transpose R_r
        if constexpr (r < NL && col::mode(KIND, B, r + 1) != MODE) {
            constexpr int w = q0.x1 - q0.x0;
            static_assert(w * (q0.y1 - q0.y0) <= col::tile_doubles(KIND, B), "transpose tile");
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int m = CPL * l + q;
                if constexpr (MODE == col::COL) {
                    if (!dead && m >= q0.x0 && m < q0.x1) {
                        double* t0 = tile + (m - q0.x0);
                        sfor<B>([&](auto YI) {
                            constexpr int j = decltype(YI)::value;
                            constexpr col::CRect qr = col::rect(KIND, B, r);
                            if constexpr (YLO + j >= qr.y0 && YLO + j < qr.y1) t0[(YLO + j - qr.y0) * w] = v[q][j];
                        });
                    }
                } else {
                    if (!dead && YLO + m >= q0.y0 && YLO + m < q0.y1) {
                        double* t0 = tile + (YLO + m - q0.y0) * w;
                        sfor<B>([&](auto XI) {
                            constexpr int x = decltype(XI)::value;
                            constexpr col::CRect qr = col::rect(KIND, B, r);
                            if constexpr (x >= qr.x0 && x < qr.x1) t0[x - qr.x0] = v[q][x];
                        });
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int m = CPL * l + q;
                if constexpr (MODE == col::COL) {  // now ROW: m = window row
                    if (YLO + m >= q0.y0 && YLO + m < q0.y1) {
                        const double* t0 = tile + (YLO + m - q0.y0) * w;
                        sfor<B>([&](auto XI) {
                            constexpr int x = decltype(XI)::value;
                            constexpr col::CRect qr = col::rect(KIND, B, r);
                            if constexpr (x >= qr.x0 && x < qr.x1) v[q][x] = t0[x - qr.x0];
                        });
                    }
                } else {  // now COL: m = column
                    if (m >= q0.x0 && m < q0.x1) {
                        const double* t0 = tile + (m - q0.x0);
                        sfor<B>([&](auto YI) {
                            constexpr int j = decltype(YI)::value;
                            constexpr col::CRect qr = col::rect(KIND, B, r);
                            if constexpr (YLO + j >= qr.y0 && YLO + j < qr.y1) v[q][j] = t0[(YLO + j - qr.y0) * w];
                        });
                    }
                }
            }
            __syncwarp();
        }
    });

    // ---- partition-edge instances: copy the record into the neighbours' ghost rings
    const bool edge = bi < gh || bi >= A.pbx - gh || bj < gh || bj >= A.pby - gh;
    if (edge && live && A.nexp > 0) {
        asm volatile("" ::: "memory");
        if constexpr (L == 32) __syncwarp();
        else __syncwarp(((1u << L) - 1u) << (sub * L));
        for (int e = l; e < A.nexp; e += L) {
            const double val = __ldcg(dst + e);
            for (int ej = -1; ej <= 1; ++ej)
                for (int ei = -1; ei <= 1; ++ei) {
                    if (ei == 0 && ej == 0) continue;
                    const int tbi = bi - ei * A.pbx, tbj = bj - ej * A.pby;
                    if (tbi < -gh || tbi >= A.pbx + gh || tbj < -gh || tbj >= A.pby + gh) continue;
                    const int tp = wrapi(pj + ej, A.py) * A.px + wrapi(pi + ei, A.px);
                    A.rec[tp * A.nslots + A.my_slot][((long)(tbj + gh) * A.extw + (tbi + gh)) * A.epad + e] = val;
                }
        }
    }
}

// Euler phase kernel: one CTA (128 threads) per block instance.  Gather as
// the heat kernel (4 variables per record entry), then every level of the
// phase runs through euler_rect on shared memory (pressures, shared x/y
// interface fluxes, update), then the record is scattered.
template <int MINB>
__global__ void __launch_bounds__(128, MINB) swept_euler_kernel(const __grid_constant__ SweptArgs A) {
    extern __shared__ double S[];
    __shared__ const double* sb[kMaxSegs];
    const int tid = threadIdx.x, T = 128;
    const int inst = blockIdx.x;
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
    {
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
        euler_rect(tid, T, Lc.cx0, Lc.cx1, Lc.cy0, Lc.cy1, Q, B, O, ps, fxs, fys, A.c0, stage == 0 ? A.c1 : A.c3,
                   stage == 0 ? A.c2 : A.c4, err);
        if (r == A.split && A.nexp_early > 0) {
            flush(0, A.nexp_early);
            __syncthreads();
        }
    }
    if (A.nexp > A.nexp_early) flush(A.nexp_early, A.nexp);
    if (err) *A.err = 1;
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
        int ri = 0;
        while (prefix[ri + 1] <= c) ++ri;
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
                                    int rank, unsigned long long epoch, int* err) {
    if (threadIdx.x != 0) return;
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

cudaError_t launch_dist_barrier(unsigned long long* const* peer_flags, unsigned long long* my_flags, int world,
                                int rank, unsigned long long epoch, int* err, cudaStream_t s) {
    dist_barrier_kernel<<<1, 32, 0, s>>>(peer_flags, my_flags, world, rank, epoch, err);
    return cudaGetLastError();
}

template <int B, int CPL, int WPC>
cudaError_t launch_heat_col_t(const SweptArgs& a, cudaStream_t s) {
    constexpr int IPC = WPC * (32 / (B / CPL));  // instances per CTA
    const int ninst = a.pbx * a.pby;
    const bool stash = (a.out_mask | a.snap_mask) != 0ull;
    const size_t smem = static_cast<size_t>(IPC) * (a.smem_doubles + (stash ? B * B : 0)) * sizeof(double);
    dim3 grid((ninst + IPC - 1) / IPC, a.ndev_parts);
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, WPC * 32, smem, s>>>(a);
        return cudaGetLastError();
    };
    switch (a.kind) {
        case col::UP: return go(swept_heat_col_kernel<B, col::UP, CPL, WPC>);
        case col::YB: return go(swept_heat_col_kernel<B, col::YB, CPL, WPC>);
        case col::XB: return go(swept_heat_col_kernel<B, col::XB, CPL, WPC>);
        case col::OCT: return go(swept_heat_col_kernel<B, col::OCT, CPL, WPC>);
        default: return go(swept_heat_col_kernel<B, col::DOWN, CPL, WPC>);
    }
}
// One column (row) per lane: two per lane halves the shuffles but doubles the
// live registers (Oct b16: 182 vs 106), and the lost occupancy costs more
// (Oct launch 0.82 vs 0.62 ms, profiles/r01_summary.md).
template <int B>
cudaError_t launch_heat_col(const SweptArgs& a, cudaStream_t s) {
    // 4 warps per CTA on big grids; single-warp CTAs when there are too few
    // instances to fill the 148 SMs otherwise (the paper's 320^2..1120^2 grids)
    if constexpr (B == 16)
        if (a.pbx * a.pby * a.ndev_parts < 2 * 4 * 148 * 8) return launch_heat_col_t<B, 1, 1>(a, s);
    // b16: 2-warp CTAs (finer-grained residency: 18 instead of 16 warps per
    // SM at ~100 registers; 3.69e11 vs 3.65e11 (4 warps) and 3.61e11 (8))
    if constexpr (B == 16) return launch_heat_col_t<B, 1, 2>(a, s);
    return launch_heat_col_t<B, 1, 4>(a, s);
}

cudaError_t launch_swept(int problem, const SweptArgs& a, cudaStream_t s) {
    const int ninst = a.pbx * a.pby;
    if (problem == 0 && a.colB == 16) return launch_heat_col<16>(a, s);
    if (problem == 0 && a.colB == 8) return launch_heat_col<8>(a, s);
    if (problem == 0 && a.colB == 32) return launch_heat_col<32>(a, s);
    if (problem == 0 && a.colB == 12) return launch_heat_col<12>(a, s);
    if (problem == 0 && a.colB == 24) return launch_heat_col<24>(a, s);
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
        // 7 resident CTAs (<= 72 registers): occupancy hides the FP64
        // dependency chains and the per-level barriers (1.09e10 vs 8.5e9
        // updates/s at 112 registers, Euler 960^2 b16)
        auto kern = swept_euler_kernel<7>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        dim3 grid(ninst, a.ndev_parts);
        kern<<<grid, 128, smem, s>>>(a);
        return cudaGetLastError();
    }
}

cudaError_t launch_std(int problem, const StdArgs& a, cudaStream_t s) {
    if (problem == 0 && a.pw % 2 == 0) {
        constexpr int ROWS = 32;
        dim3 grid((a.pw / 2 + 127) / 128, (a.ph + ROWS - 1) / ROWS, a.ndev_parts);
        std_heat_kernel<ROWS><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
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
