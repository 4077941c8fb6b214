// sm_100a kernels of the swept solver.
//
//  swept_phase_kernel<PROB>  one launch = one swept phase (UpPyramid, YBridge,
//      XBridge, Octahedron = OctahedronDown+OctahedronUp, DownPyramid) for every
//      block instance of the partitions on this GPU.  A CTA owns G instances:
//        1. gather: imported edge cells (records of earlier phases, or the
//           initial plane) -> shared memory, coalesced along the records;
//        2. advance all levels of the phase on chip (the pyramid / bridge /
//           octahedron), one __syncthreads per level;
//        3. scatter: the cells later phases read (this instance's record)
//           -> HBM, plus the copies partition-edge instances push into the
//           neighbouring partitions' ghost records (NVLink P2P stores when
//           the neighbour is another GPU);
//        4. cells at the output level -> the owning partition's output plane.
//  std_step_kernel<PROB>     the standard decomposition: one sub-step over the
//      whole partition, boundary cells pushed into the neighbours' ghost
//      frames (replaces StandardRank::exchange_ghosts + compute,
//      engine.cpp:351-408).
//  substep_rects_kernel<PROB>  run_substep on rectangles (physics.cpp:551-575).
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "physics.cuh"

namespace sg {

namespace {

__device__ __forceinline__ int wrapi(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}

template <int PROB>
__global__ void __launch_bounds__(128) swept_phase_kernel(const __grid_constant__ SweptArgs A, int G) {
    extern __shared__ double sm[];
    constexpr int NV = PROB == 0 ? 1 : 4;
    const int T = blockDim.x, tid = threadIdx.x;
    const int ninst = A.pbx * A.pby;
    const int batches = (ninst + G - 1) / G;
    const int part = A.dev_parts[blockIdx.x / batches];
    const int inst0 = (blockIdx.x % batches) * G;
    const int pi = part % A.px, pj = part / A.px;
    const int SD = A.smem_doubles;
    const int half = A.frame * (A.b / 2);
    int err = 0;

    // ---- 1. gather -------------------------------------------------------
    for (int e = tid; e < G * A.nimp; e += T) {
        const int g = e / A.nimp, i = e - g * A.nimp;
        const int inst = inst0 + g;
        if (inst >= ninst) continue;
        const int bi = inst % A.pbx, bj = inst / A.pbx;
        const int4 im = __ldg(&A.imports[i]);
        const DevSeg s = A.segs[im.x];
        const long ext = (long)(bj + s.dj + A.ghost) * A.extw + (bi + s.di + A.ghost);
        const double* src = A.rec[part * A.nslots + s.slot] + ext * NV * s.epad + im.y;
        double* dst = sm + g * SD + im.z;
#pragma unroll
        for (int v = 0; v < NV; ++v) dst[v * im.w] = src[v * s.epad];
    }
    for (int e = tid; e < G * A.ninit; e += T) {
        const int g = e / A.ninit, i = e - g * A.ninit;
        const int inst = inst0 + g;
        if (inst >= ninst) continue;
        const int bi = inst % A.pbx, bj = inst / A.pbx;
        const int4 im = __ldg(&A.inits[i]);
        const int gx = wrapi(pi * A.pw + bi * A.b - half + im.x, A.nx);
        const int gy = wrapi(pj * A.ph + bj * A.b - half + im.y, A.ny);
        const int opi = gx / A.pw, opj = gy / A.ph;
        const double* src = A.init_planes[opj * A.px + opi] + (long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw);
        double* dst = sm + g * SD + im.z;
        const long pl = (long)A.pw * A.ph;
#pragma unroll
        for (int v = 0; v < NV; ++v) dst[v * im.w] = src[v * pl];
    }
    __syncthreads();

    // ---- 2. advance the phase on chip ------------------------------------
    for (int r = 1; r <= A.nlev; ++r) {
        const DevLevel Lc = A.lev[r - A.rmin];
        const DevLevel Lp = A.lev[r - 1 - A.rmin];
        const int cw = Lc.cx1 - Lc.cx0, ch = Lc.cy1 - Lc.cy0, cells = cw * ch;
        int stage = 0;
        DevLevel Lpp = Lp;
        if (PROB == 1) {
            stage = (A.stage0 + r - 1) & 1;
            if (stage == 1) Lpp = A.lev[r - 2 - A.rmin];
        }
        for (int c = tid; c < G * cells; c += T) {
            const int g = c / cells, rem = c - g * cells;
            const int yy = rem / cw, xx = rem - yy * cw;
            const int x = Lc.cx0 + xx, y = Lc.cy0 + yy;
            if (inst0 + g >= ninst) continue;
            double* base = sm + g * SD;
            const double* sp = base + Lp.off + (y - Lp.by0) * Lp.bw + (x - Lp.bx0);
            double* dp = base + Lc.off + (y - Lc.by0) * Lc.bw + (x - Lc.bx0);
            double outv[NV];
            if (PROB == 0) {
                outv[0] = heat_update(sp[0], sp[1], sp[-1], sp[Lp.bw], sp[-Lp.bw], A.c0, A.c1);
            } else {
                double q0[4];
                const double* bp =
                    stage == 0 ? sp : base + Lpp.off + (y - Lpp.by0) * Lpp.bw + (x - Lpp.bx0);
                const int bvs = stage == 0 ? Lp.vstride : Lpp.vstride;
#pragma unroll
                for (int v = 0; v < 4; ++v) q0[v] = bp[v * bvs];
                const double cx = stage == 0 ? A.c1 : A.c3;
                const double cy = stage == 0 ? A.c2 : A.c4;
                const int pbw = Lp.bw, pvs = Lp.vstride;
                euler_update_d([&](int dx, int dy, int v) { return sp[v * pvs + dy * pbw + dx]; }, q0, cx,
                               cy, A.c0, outv, err);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) dp[v * Lc.vstride] = outv[v];
            if (r == A.r_out) {
                const int inst = inst0 + g;
                const int bi = inst % A.pbx, bj = inst / A.pbx;
                const int gx = wrapi(pi * A.pw + bi * A.b - half + x, A.nx);
                const int gy = wrapi(pj * A.ph + bj * A.b - half + y, A.ny);
                const int opi = gx / A.pw, opj = gy / A.ph;
                double* o = A.out_planes[opj * A.px + opi] + (long)(gy - opj * A.ph) * A.pw + (gx - opi * A.pw);
                const long pl = (long)A.pw * A.ph;
#pragma unroll
                for (int v = 0; v < NV; ++v) o[v * pl] = outv[v];
            }
        }
        __syncthreads();
    }

    // ---- 3. scatter the record (+ ghost pushes at partition edges) ------
    if (A.nexp > 0) {
        for (int e = tid; e < G * A.nexp; e += T) {
            const int g = e / A.nexp, i = e - g * A.nexp;
            const int inst = inst0 + g;
            if (inst >= ninst) continue;
            const int bi = inst % A.pbx, bj = inst / A.pbx;
            const int so = __ldg(&A.exp_off[i]), vs = __ldg(&A.exp_vs[i]);
            double val[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) val[v] = sm[g * SD + so + v * vs];
            {
                const long ext = (long)(bj + A.ghost) * A.extw + (bi + A.ghost);
                double* d = A.rec[part * A.nslots + A.my_slot] + ext * NV * A.epad + i;
#pragma unroll
                for (int v = 0; v < NV; ++v) d[v * A.epad] = val[v];
            }
            const int gh = A.ghost;
            if (bi < gh || bi >= A.pbx - gh || bj < gh || bj >= A.pby - gh) {
                for (int ej = -1; ej <= 1; ++ej)
                    for (int ei = -1; ei <= 1; ++ei) {
                        if (ei == 0 && ej == 0) continue;
                        const int tbi = bi - ei * A.pbx, tbj = bj - ej * A.pby;
                        if (tbi < -gh || tbi >= A.pbx + gh || tbj < -gh || tbj >= A.pby + gh) continue;
                        const int tp = wrapi(pj + ej, A.py) * A.px + wrapi(pi + ei, A.px);
                        const long ext = (long)(tbj + gh) * A.extw + (tbi + gh);
                        double* d = A.rec[tp * A.nslots + A.my_slot] + ext * NV * A.epad + i;
#pragma unroll
                        for (int v = 0; v < NV; ++v) d[v * A.epad] = val[v];
                    }
            }
        }
    }
    if (err) *A.err = 1;
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

}  // namespace

cudaError_t launch_swept(int problem, const SweptArgs& a, int G, int threads, cudaStream_t s) {
    const int ninst = a.pbx * a.pby;
    const int grid = a.ndev_parts * ((ninst + G - 1) / G);
    const size_t smem = static_cast<size_t>(G) * a.smem_doubles * sizeof(double);
    if (problem == 0) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(swept_phase_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        swept_phase_kernel<0><<<grid, threads, smem, s>>>(a, G);
    } else {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(swept_phase_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        swept_phase_kernel<1><<<grid, threads, smem, s>>>(a, G);
    }
    return cudaGetLastError();
}

cudaError_t launch_std(int problem, const StdArgs& a, cudaStream_t s) {
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
