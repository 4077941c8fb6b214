// Register-tile heat phase kernel (swept_heat_col_kernel) and its launcher,
// instantiated once per block size in kernels_col<B>.cu so the five block
// sizes compile in parallel.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "colgeom.hpp"
#include "devutil.cuh"
#include "physics.cuh"

namespace sg {
namespace {

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
// FLAGS bit 0 (FAST): a steady-state launch -- no output / snapshot stash
// (its non-inlined writer call costs the unrolled level code ~20-60
// registers) and no initial-plane imports.  Bit 1 (DENSE): the gather table
// is indexed by shared-memory slot (imp_dense), so every shared address and
// table index is a compile-time immediate off one per-lane base.  Launches
// with an output or snapshot level or initial-plane cells use FLAGS = 0.
template <int B, int KIND, int CPL, int WPC, int FLAGS>
__global__ void __launch_bounds__(WPC * 32) swept_heat_col_kernel(const __grid_constant__ SweptArgs A) {
    constexpr int L = B / CPL;      // lanes per instance
    constexpr int IPW = 32 / L;     // instances per warp
    constexpr int IPC = WPC * IPW;  // instances per CTA
    constexpr int NL = col::nlev(KIND, B);
    constexpr int YLO = col::ylo(KIND, B);
    constexpr int NIMP = col::imp_total(KIND, B);  // import slots; the transpose tile follows
    constexpr bool FAST = FLAGS & 1;               // no output / snapshot stash, no initial-plane imports
    constexpr bool DENSE = FLAGS & 2;              // dense gather (implies FAST)
    constexpr bool REGS = FLAGS & 4;               // dense gather through registers (implies DENSE)
    // HALF (FLAGS bits 4-5): 0 = all levels; 1 / 2 = the Octahedron's levels
    // 1..k / k+1..2k as two launches, the level-k state through oct_scratch
    constexpr int HALF = (FLAGS >> 4) & 3;
    constexpr int KO = B / 2 - 1;
    constexpr int RLO = HALF == 2 ? KO + 1 : 1, RHI = HALF == 1 ? KO : NL;
    static_assert(HALF == 0 || (KIND == col::OCT && DENSE && !REGS && CPL == 1), "split Octahedron");
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // b = 12 / 24: the last 32 - IPW*L lanes of a warp are dead (they run the
    // code, shuffles included, but never write anything)
    const bool dead = lane >= IPW * L;
    const int sub = dead ? 0 : lane / L, l = lane % L;
    const int slot_in_cta = warp * IPW + sub;
    // grid (ceil(pbx / IPC), pby, partitions); odd launches walk the
    // instances backwards: their first CTAs read the records the previous
    // launch wrote last (still in L2)
    const bool rev = A.lo_parity & 1;
    const int cbx = rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const int cby = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y;
    const int ibx = cbx * IPC + slot_in_cta;
    const bool live = !dead && ibx < A.pbx;
    const int part = A.dev_parts[blockIdx.z];
    const int pi = A.dev_pij[blockIdx.z] & 0xffff, pj = A.dev_pij[blockIdx.z] >> 16;
    const int bi = live ? ibx : 0, bj = cby;
    const int half = A.frame * (B / 2);
    const int gh = A.ghost;
    double* S = sm + slot_in_cta * A.smem_doubles;
    // the second half of a split Octahedron holds only slots [NK, NIMP): its
    // shared addresses are offset by -NK slots (unsigned arithmetic)
    constexpr unsigned SOFF = HALF == 2 ? 8u * col::imp_base(KIND, B, KO + 1, YLO) : 0u;

    // ---- gather the imports
    // REGS: part A through registers (LDG, then STS: an LDGSTS writes shared
    // memory one 32-byte sector per wavefront, an STS.64 of a warp 128 bytes),
    // part B stays in registers until level gather_split + 1
    constexpr int NA_ = col::imp_base(KIND, B, col::gather_split(KIND, B) + 1, YLO);
    constexpr int KA = (NA_ + L - 1) / L, KB = (NIMP - NA_ + L - 1) / L;
    double gbuf[REGS ? (KB > 0 ? KB : 1) : 1];
    const unsigned s0r = static_cast<unsigned>(__cvta_generic_to_shared(S)) + 8u * l;
    if constexpr (REGS) if (!dead) {
        const double* ibase = A.rec[part * A.nslots] + ((long)(bj + gh) * A.extw + (bi + gh)) * A.epad;
        const int* tab = A.imp_dense + l;
        double ga[KA > 0 ? KA : 1];
        sfor<KA>([&](auto KI) {
            constexpr int i0 = decltype(KI)::value * L;
            if constexpr (i0 + L <= NA_) ga[decltype(KI)::value] = __ldg(ibase + ldg_keep(tab + i0));
            else if (i0 + l < NA_) ga[decltype(KI)::value] = __ldg(ibase + ldg_keep(tab + i0));
        });
        sfor<KB>([&](auto KI) {
            constexpr int i0 = NA_ + decltype(KI)::value * L;
            if constexpr (i0 + L <= NIMP) gbuf[decltype(KI)::value] = __ldg(ibase + ldg_keep(tab + i0));
            else if (i0 + l < NIMP) gbuf[decltype(KI)::value] = __ldg(ibase + ldg_keep(tab + i0));
        });
        sfor<KA>([&](auto KI) {
            constexpr int i0 = decltype(KI)::value * L;
            if constexpr (i0 + L <= NA_) sts_imm<8 * i0>(s0r, ga[decltype(KI)::value]);
            else if (i0 + l < NA_) sts_imm<8 * i0>(s0r, ga[decltype(KI)::value]);
        });
    }
    if constexpr (DENSE && !REGS) {
        // dense: slot i <- ibase[imp_dense[i]], lane l takes slots l, l + L, ...
        // part A = slots [0, NA) (levels <= gather_split), then part B; a split
        // Octahedron's halves gather the slots of their own levels only
        constexpr int NK = col::imp_base(KIND, B, KO + 1, YLO);
        constexpr int NS = col::imp_base(KIND, B, col::gather_split(KIND, B) + 1, YLO);
        constexpr int GA0 = HALF == 2 ? NK : 0;
        constexpr int NA = HALF == 2 ? NIMP : HALF == 1 ? (NS < NK ? NS : NK) : NS;
        constexpr int NEND = HALF == 1 ? NK : NIMP;
        if (live) {
            const double* ibase = A.rec[part * A.nslots] + ((long)(bj + gh) * A.extw + (bi + gh)) * A.epad;
            const int* tab = A.imp_dense + l;
            const unsigned s0 = static_cast<unsigned>(__cvta_generic_to_shared(S)) - SOFF + 8u * l;
            auto part_copy = [&](auto LO, auto HI) {
                constexpr int lo = decltype(LO)::value, hi = decltype(HI)::value;
                sfor<(hi - lo + L - 1) / L>([&](auto KI) {
                    constexpr int i0 = lo + decltype(KI)::value * L;  // slot of lane 0
                    if constexpr (i0 + L <= hi) {
                        cp_async8_imm<8 * i0>(s0, ibase + ldg_keep(tab + i0));
                    } else {
                        if (i0 + l < hi) cp_async8_imm<8 * i0>(s0, ibase + ldg_keep(tab + i0));
                    }
                });
            };
            part_copy(std::integral_constant<int, GA0>{}, std::integral_constant<int, NA>{});
            cp_async_commit();
            part_copy(std::integral_constant<int, NA>{}, std::integral_constant<int, NEND>{});
        }
    }
    // ---- table gather: {offset from this instance's slot-0 record, smem slot}
    if (!DENSE && live) {
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
        if (!FAST) for (int j = l; j < A.ninit; j += L) {
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
    const unsigned s_imp = static_cast<unsigned>(__cvta_generic_to_shared(S)) - SOFF;
    unsigned sc[CPL];  // shared address of slot c (c = the lane's column), for COL-mode imports
    double* pc[CPL];   // record address of index c, for COL-mode exports
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
        sc[q] = s_imp + 8u * (CPL * l + q);
        pc[q] = dst + (CPL * l + q);
    }
    double* tile = S + NIMP;
    // output stash (only allocated by launches that write the output level or snapshots)
    double* stash = sm + IPC * A.smem_doubles + (slot_in_cta * L + l) * CPL * B;
    double v[CPL][B];
    // the split Octahedron's level-k state: [dev part][bj][bi][row][lane]
    double* scr = HALF ? A.oct_scratch + ((((long)blockIdx.z * A.pby + bj) * A.pbx + bi) * B) * B + l : nullptr;
    if constexpr (HALF == 2) {
#pragma unroll
        for (int i = 0; i < B; ++i) v[0][i] = scr[i * B];
    } else {
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int i = 0; i < B; ++i) v[q][i] = 0.0;
    }

    sfor<NL>([&](auto RI) {
        constexpr int r = decltype(RI)::value + 1;
        if constexpr (r >= RLO && r <= RHI) {
        constexpr int MODE = col::mode(KIND, B, r);
        constexpr col::CRect q0 = col::rect(KIND, B, r);
        if constexpr (r == col::gather_split(KIND, B) + 1) {
            if constexpr (REGS) {
                if (!dead) sfor<KB>([&](auto KI) {
                    constexpr int i0 = NA_ + decltype(KI)::value * L;
                    if constexpr (i0 + L <= NIMP) sts_imm<8 * i0>(s0r, gbuf[decltype(KI)::value]);
                    else if (i0 + l < NIMP) sts_imm<8 * i0>(s0r, gbuf[decltype(KI)::value]);
                });
            } else {
                cp_async_wait_all();  // part B
            }
            __syncwarp();
        }
        // ---------------- 1. imports of level r-1
        if constexpr (MODE == col::COL) {
            // row type t: columns [a, b) minus [hp, hq); the cell of column c
            // sits at slot base(row) + c - a - (c >= hq ? hq - hp : 0), so the
            // address is the lane's column address sc (minus the hole width
            // right of a hole) plus a compile-time offset per row
            bool ip[CPL][4];
            unsigned ia[CPL][4];
            sfor<4>([&](auto TI) {
                constexpr int t = decltype(TI)::value;
                constexpr col::RowSet ts = col::Geo<KIND, B>::t.imp_tset[r][t];
                if constexpr (ts.count() > 0) {
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = CPL * l + q;
                        ip[q][t] = static_cast<unsigned>(c - ts.a) < static_cast<unsigned>(ts.b - ts.a);
                        if constexpr (ts.hq > ts.hp) {
                            ip[q][t] = ip[q][t] && !(static_cast<unsigned>(c - ts.hp) < static_cast<unsigned>(ts.hq - ts.hp));
                            ia[q][t] = sc[q] - (c >= ts.hq ? 8u * (ts.hq - ts.hp) : 0u);
                        } else {
                            ia[q][t] = sc[q];
                        }
                    }
                }
            });
            sfor<B>([&](auto YI) {
                constexpr int j = decltype(YI)::value;
                constexpr int t = col::Geo<KIND, B>::t.imp_type[r][j];
                constexpr int base = col::Geo<KIND, B>::t.imp_base[r][j];
                if constexpr (t >= 0) {
                    constexpr int a0 = col::Geo<KIND, B>::t.imp_tset[r][t].a;
#pragma unroll
                    for (int q = 0; q < CPL; ++q) lds_if_imm<8 * (base - a0)>(v[q][j], ia[q][t], ip[q][t]);
                }
            });
        } else {
            // lane = window row y: the level's imports are column-major
            // (colgeom imp_col), the transpose of the COL-mode case above
            static_assert(col::imp_cols_ok(KIND, B), "imp_col / imp_row disagree");
            bool ip[CPL][4];
            unsigned ia[CPL][4];
            sfor<4>([&](auto TI) {
                constexpr int t = decltype(TI)::value;
                constexpr col::RowSet ts = col::Geo<KIND, B>::t.impc_tset[r][t];
                if constexpr (ts.count() > 0) {
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int y = YLO + CPL * l + q;
                        ip[q][t] = static_cast<unsigned>(y - ts.a) < static_cast<unsigned>(ts.b - ts.a);
                        if constexpr (ts.hq > ts.hp) {
                            ip[q][t] = ip[q][t] && !(static_cast<unsigned>(y - ts.hp) < static_cast<unsigned>(ts.hq - ts.hp));
                            ia[q][t] = sc[q] - (y >= ts.hq ? 8u * (ts.hq - ts.hp) : 0u);
                        } else {
                            ia[q][t] = sc[q];
                        }
                    }
                }
            });
            sfor<B>([&](auto XI) {
                constexpr int x = decltype(XI)::value;
                constexpr int t = col::Geo<KIND, B>::t.impc_type[r][x];
                constexpr int base = col::Geo<KIND, B>::t.impc_base[r][x];
                if constexpr (t >= 0) {
                    constexpr int a0 = col::Geo<KIND, B>::t.impc_tset[r][t].a;
#pragma unroll
                    for (int q = 0; q < CPL; ++q) lds_if_imm<8 * (base - a0 + YLO)>(v[q][x], ia[q][t], ip[q][t]);
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
                    // rank_band(c) = c - x0 - (c >= mq ? mw : 0): one adjusted
                    // pointer pa per level, every row's offset compile-time
                    bool pb[CPL], pm[CPL];
                    double* pa[CPL];
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int c = CPL * l + q;
                        const bool in = static_cast<unsigned>(c - E.x0) < static_cast<unsigned>(E.x1 - E.x0);
                        const bool mid = static_cast<unsigned>(c - E.mp) < static_cast<unsigned>(E.mq - E.mp);
                        pb[q] = in && !mid;
                        pm[q] = in && mid;
                        if constexpr (E.mw() > 0) pa[q] = pc[q] - (c >= E.mq ? E.mw() : 0);
                        else pa[q] = pc[q];
                    }
                    sfor<B>([&](auto YI) {
                        constexpr int j = decltype(YI)::value;
                        constexpr col::ExpLev Ej = col::Geo<KIND, B>::t.exp.lev[r];
                        constexpr int y = YLO + j;
                        constexpr int f = Ej.full_index(y);
                        if constexpr (Ej.hole_row(y)) {
#pragma unroll
                            for (int q = 0; q < CPL; ++q)
                                stg_if_imm<8 * (Ej.g1 + (y - Ej.yh0) * Ej.bw() - Ej.x0)>(pa[q], v[q][j], pb[q]);
                        } else if constexpr (f >= 0) {
                            if constexpr (Ej.bw() > 0) {
#pragma unroll
                                for (int q = 0; q < CPL; ++q)
                                    stg_if_imm<8 * (Ej.g3 + f * Ej.bw() - Ej.x0)>(pa[q], v[q][j], pb[q]);
                            }
                            if constexpr (Ej.mw() > 0) {
#pragma unroll
                                for (int q = 0; q < CPL; ++q)
                                    stg_if_imm<8 * (Ej.g2 + f * Ej.mw() - Ej.mp)>(pc[q], v[q][j], pm[q]);
                            }
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
                    if constexpr (ts.count() > 0) {
#pragma unroll
                        for (int q = 0; q < CPL; ++q) {
                            const int c = CPL * l + q;
                            ep[q][t] = static_cast<unsigned>(c - ts.a) < static_cast<unsigned>(ts.b - ts.a);
                            if constexpr (ts.hq > ts.hp) {
                                ep[q][t] = ep[q][t] &&
                                           !(static_cast<unsigned>(c - ts.hp) < static_cast<unsigned>(ts.hq - ts.hp));
                                eg[q][t] = pc[q] - (c >= ts.hq ? ts.hq - ts.hp : 0);
                            } else {
                                eg[q][t] = pc[q];
                            }
                        }
                    }
                });
                sfor<B>([&](auto YI) {
                    constexpr int j = decltype(YI)::value;
                    constexpr int t = col::Geo<KIND, B>::t.exp_type[r][j];
                    constexpr int base = col::Geo<KIND, B>::t.exp_base[r][j];
                    static_assert(t < 2, "export row types");
                    if constexpr (t >= 0) {
                        constexpr int a0 = col::Geo<KIND, B>::t.exp_tset[r][t].a;
#pragma unroll
                        for (int q = 0; q < CPL; ++q) stg_if_imm<8 * (base - a0)>(eg[q][t], v[q][j], ep[q][t]);
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
        if (!FAST && (((A.out_mask | A.snap_mask) >> r) & 1ull) && !dead) {
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
            // tile rows of odd stride ws: the lanes of a row-mode access hit
            // distinct banks
            constexpr int ws = (q0.x1 - q0.x0) | 1;
            static_assert(ws * (q0.y1 - q0.y0) <= col::tile_doubles(KIND, B), "transpose tile");
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int m = CPL * l + q;
                if constexpr (MODE == col::COL) {
                    if (!dead && m >= q0.x0 && m < q0.x1) {
                        double* t0 = tile + (m - q0.x0);
                        sfor<B>([&](auto YI) {
                            constexpr int j = decltype(YI)::value;
                            constexpr col::CRect qr = col::rect(KIND, B, r);
                            if constexpr (YLO + j >= qr.y0 && YLO + j < qr.y1) t0[(YLO + j - qr.y0) * ws] = v[q][j];
                        });
                    }
                } else {
                    if (!dead && YLO + m >= q0.y0 && YLO + m < q0.y1) {
                        double* t0 = tile + (YLO + m - q0.y0) * ws;
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
                        const double* t0 = tile + (YLO + m - q0.y0) * ws;
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
                            if constexpr (YLO + j >= qr.y0 && YLO + j < qr.y1) v[q][j] = t0[(YLO + j - qr.y0) * ws];
                        });
                    }
                }
            }
            __syncwarp();
        }
        }  // level range (split Octahedron)
    });
    if constexpr (HALF == 1) {
        if (live) {
#pragma unroll
            for (int i = 0; i < B; ++i) scr[i * B] = v[0][i];
        }
        return;  // the second half pushes the partition-edge records
    }

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

// Function attributes (dynamic shared-memory limit, carveout) set only when
// they change: the launcher runs once per phase launch, and outside CUDA
// graphs (one process per GPU) every host call is on the launch path.
inline void set_attrs(const void* fn, size_t smem, int carve) {
    struct Attr {
        const void* fn;
        int dev;
        size_t smem;
        int carve;
    };
    static thread_local std::vector<Attr> seen;
    int dev = 0;
    cudaGetDevice(&dev);  // attributes are per device context
    for (Attr& e : seen)
        if (e.fn == fn && e.dev == dev) {
            if (smem > e.smem && smem > 48 * 1024) {
                cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                e.smem = smem;
            }
            if (carve != e.carve) {
                cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
                e.carve = carve;
            }
            return;
        }
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    seen.push_back({fn, dev, smem > 48 * 1024 ? smem : 48 * 1024, carve});
}

inline int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// Resident CTAs per SM the shared-memory carveout is sized for (0: driver
// default).  The gathers land through L1 (cp.async.ca, the gather tables):
// with the register-lean steady-state kernels the driver would otherwise
// pack up to ~28 warps per SM and leave L1 a few KB (b16 YBridge 0.36 vs
// 0.29 ms, Octahedron 0.73 vs 0.55 ms; profiles/r02b_summary.md).
template <int B, int WPC>
constexpr int target_ctas(int kind) {
    if constexpr (B == 16) return WPC <= 2 ? 9 : 18 / WPC;  // 18 warps per SM
    // 4-warp CTAs (measured carveout sweeps, 4128^2): the bridges want more
    // warps than the Octahedron (b8 8, b12 10, b24 7, b32 4 CTAs: +2..4 %)
    // (b24: the first half of the split Octahedron, 4 CTAs: 0.295 vs 0.315 ms)
    if (kind == col::OCT) return B < 16 ? 18 / WPC : B == 24 ? 4 : 0;
    return B == 8 ? 8 : B == 12 ? 10 : B == 24 ? 7 : 4;
}

template <int B, int CPL, int WPC>
cudaError_t launch_heat_col_t(const SweptArgs& a, cudaStream_t s) {
    constexpr int IPC = WPC * (32 / (B / CPL));  // instances per CTA
    const bool stash = (a.out_mask | a.snap_mask) != 0ull;
    const size_t smem = static_cast<size_t>(IPC) * (a.smem_doubles + (stash ? B * B : 0)) * sizeof(double);
    dim3 grid((a.pbx + IPC - 1) / IPC, a.pby, a.ndev_parts);
    // variant: 3 = steady state with the dense gather, 1 = steady state with
    // the table gather, 0 = general (output / snapshot stash, initial-plane
    // imports).  SG_FAST_KINDS / SG_DENSE_KINDS (bit per kind) restrict them.
    static const int fast_kinds = env_int("SG_FAST_KINDS", 31);
    static const int dense_kinds = env_int("SG_DENSE_KINDS", 31);
    const bool steady = !stash && a.ninit == 0 && ((fast_kinds >> a.kind) & 1);
    // b32: the Octahedron's part A through registers (b32 1.25 vs 1.34 ms;
    // at b16 the LDGSTS path is faster: 0.56 vs 0.67 ms)
    static const int reg_kinds = env_int("SG_REG_KINDS", B == 32 ? (1 << col::OCT) : 0);
    const int flags = !steady ? 0
                      : (a.dense && ((dense_kinds >> a.kind) & 1)) ? (((reg_kinds >> a.kind) & 1) ? 7 : 3)
                                                                   : 1;
    const bool bridge = a.kind == col::YB || a.kind == col::XB;
    int carve = -1;
    if (const int t = target_ctas<B, WPC>(a.kind); t > 0 && flags != 0)
        carve = std::min(100, static_cast<int>((100 * t * (smem + 1024) + 228 * 1024 - 1) / (228 * 1024)));
    static const int carve_oct = env_int("SG_CARVE_OCT", -2), carve_br = env_int("SG_CARVE_BR", -2);
    if (a.kind == col::OCT && carve_oct != -2) carve = carve_oct;
    if (bridge && carve_br != -2) carve = carve_br;
    auto go = [&](auto kern) {
        set_attrs(reinterpret_cast<const void*>(kern), smem,
                  carve >= 0 ? carve : static_cast<int>(cudaSharedmemCarveoutDefault));
        kern<<<grid, WPC * 32, smem, s>>>(a);
        return cudaGetLastError();
    };
    auto pick = [&](auto K) {
        constexpr int kd = decltype(K)::value;
        if constexpr (B >= 24 && kd == col::OCT && CPL == 1) {
            if (a.oct_scratch && (flags == 3 || flags == 7)) {
                const cudaError_t e = go(swept_heat_col_kernel<B, kd, CPL, WPC, 3 | 16>);
                if (e != cudaSuccess) return e;
                // second half: shared memory for its own imports only
                constexpr int NK = col::imp_base(col::OCT, B, B / 2, 0), NI = col::imp_total(col::OCT, B);
                static_assert(col::tile_doubles(col::OCT, B) == 0, "no transpose tile in the Octahedron");
                SweptArgs a2 = a;
                a2.smem_doubles = NI - NK;
                const size_t smem2 = static_cast<size_t>(IPC) * a2.smem_doubles * sizeof(double);
                auto kern2 = swept_heat_col_kernel<B, kd, CPL, WPC, 3 | 32>;
                set_attrs(reinterpret_cast<const void*>(kern2), smem2,
                          static_cast<int>(cudaSharedmemCarveoutDefault));
                kern2<<<grid, WPC * 32, smem2, s>>>(a2);
                return cudaGetLastError();
            }
        }
        if (flags == 7) return go(swept_heat_col_kernel<B, kd, CPL, WPC, 7>);
        if (flags == 3) return go(swept_heat_col_kernel<B, kd, CPL, WPC, 3>);
        if (flags == 1) return go(swept_heat_col_kernel<B, kd, CPL, WPC, 1>);
        return go(swept_heat_col_kernel<B, kd, CPL, WPC, 0>);
    };
    switch (a.kind) {
        case col::UP: return pick(std::integral_constant<int, col::UP>{});
        case col::YB: return pick(std::integral_constant<int, col::YB>{});
        case col::XB: return pick(std::integral_constant<int, col::XB>{});
        case col::OCT: return pick(std::integral_constant<int, col::OCT>{});
        default: return pick(std::integral_constant<int, col::DOWN>{});
    }
}
// One column (row) per lane: two per lane halves the shuffles but doubles the
// shared memory and registers per warp, and each memory instruction spans
// four instances' records (steady-state b16 Octahedron 0.88 vs 0.55 ms,
// DESIGN.md §4).
template <int B>
cudaError_t launch_heat_col(const SweptArgs& a, cudaStream_t s) {
    // 4 warps per CTA on big grids; single-warp CTAs when there are too few
    // instances to fill the 148 SMs otherwise (the paper's 320^2..1120^2 grids)
    if constexpr (B == 16)
        if (a.pbx * a.pby * a.ndev_parts < 2 * 4 * 148 * 8) return launch_heat_col_t<B, 1, 1>(a, s);
    // b16: 2-warp CTAs (finer-grained residency; 4- and 8-warp CTAs measured
    // 0.58 / 0.63 vs 0.56 ms for the steady-state Octahedron)
    if constexpr (B == 16) {
        return launch_heat_col_t<B, 1, 2>(a, s);
    }
    return launch_heat_col_t<B, 1, 4>(a, s);
}

}  // namespace
}  // namespace sg
