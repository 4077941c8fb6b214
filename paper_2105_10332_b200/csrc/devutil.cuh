// Device helpers shared by the kernel translation units (kernels.cu and the
// per-block column-kernel units kernels_col<B>.cu).
#pragma once

#include <cuda_runtime.h>

#include <type_traits>
#include <utility>

#include "kernels.cuh"

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
// smem byte address + compile-time offset (folded into the LDGSTS immediate)
template <int IMM>
__device__ __forceinline__ void cp_async8_imm(unsigned saddr, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0+%2], [%1], 8;\n" ::"r"(saddr), "l"(gmem), "n"(IMM) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

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

// ... with a compile-time byte offset folded into the instruction
template <int IMM>
__device__ __forceinline__ void lds_if_imm(double& v, unsigned saddr, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f64 %0, [%1+%3];\n\t}"
                 : "+d"(v)
                 : "r"(saddr), "r"(static_cast<int>(p)), "n"(IMM));
}
template <int IMM>
__device__ __forceinline__ void stg_if_imm(const double* g, double v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0+%3], %1;\n\t}" ::"l"(g), "d"(v),
                 "r"(static_cast<int>(p)), "n"(IMM));
}

template <int IMM>
__device__ __forceinline__ void sts_imm(unsigned saddr, double v) {
    asm volatile("st.shared.f64 [%0+%2], %1;" ::"r"(saddr), "d"(v), "n"(IMM) : "memory");
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

}  // namespace
}  // namespace sg
