// Closed-form geometry of the column-register heat phase kernels, shared by
// the plan compiler (host) and the kernels (device) so both agree on where
// every imported cell lands in shared memory and where every exported cell
// sits in an instance's record.
//
// Column mode (heat, n = 1, S = 1, block B in {8, 12, 16, 24, 32}): B lanes own one
// phase instance, lane c = instance column c, and each lane holds its
// column's cells of the current level in registers, rows [ylo, ylo + B).
// Every kind's cells (computed and read) fit that B x B window:
//   UpPyramid / Octahedron / DownPyramid rows [0, B), YBridge / XBridge rows
//   [B/2, 3B/2); columns [0, B) for all (phase_region, geometry.cpp:93-115).
//
// Level r of a kind reads level r-1 on the cross Read(R_r) = R_r grown by one
// in x (rows of R_r) and one in y (columns of R_r).  What the instance did not
// compute itself at r-1 (R_{r-1}) is imported:
//     imports(r) = Read(R_r) \ R_{r-1}            (R_0 = empty)
// and a cell of R_r is exported iff another instance reads it at r+1, i.e.
// unless it and its four neighbours all lie in R_{r+1}:
//     exports(r) = R_r \ interior(R_{r+1})        (R_{nlev+1} = empty)
// Both sets are, row by row, a column interval minus a column hole; they are
// enumerated level by level, row by row, column by column.  The plan compiler
// checks them against its schedule replay (plan.cpp) before using them.
#pragma once

#if defined(__CUDACC__)
#define SG_HD __host__ __device__
#else
#define SG_HD
#endif

namespace sg {
namespace col {

// Kind ids (= sg::Kind, checked by a static_assert in plan.cpp)
constexpr int UP = 0, YB = 1, XB = 2, OCT = 3, DOWN = 4;

struct CRect {
    int x0, x1, y0, y1;
};

SG_HD constexpr int nlev(int kind, int B) { return kind == OCT ? 2 * (B / 2 - 1) : B / 2 - 1; }
SG_HD constexpr int ylo(int kind, int B) { return (kind == YB || kind == XB) ? B / 2 : 0; }

// phase_region (geometry.cpp:93-115) for n = 1, k = B/2 - 1; empty outside 1..nlev
SG_HD constexpr CRect rect(int kind, int B, int r) {
    const int k = B / 2 - 1;
    if (r < 1 || r > nlev(kind, B)) return CRect{0, 0, 0, 0};
    switch (kind) {
        case UP: return CRect{r, B - r, r, B - r};
        case YB: return CRect{r, B - r, B - r, B + r};
        case XB: return CRect{B / 2 - r, B / 2 + r, B / 2 + r, 3 * B / 2 - r};
        case DOWN: return CRect{B / 2 - r, B / 2 + r, B / 2 - r, B / 2 + r};
        default: {
            if (r <= k) return CRect{B / 2 - r, B / 2 + r, B / 2 - r, B / 2 + r};
            const int w = B - 2 * (r - k);
            return CRect{B / 2 - w / 2, B / 2 + w / 2, B / 2 - w / 2, B / 2 + w / 2};
        }
    }
}
SG_HD constexpr bool empty(CRect q) { return q.x1 <= q.x0 || q.y1 <= q.y0; }

// one row of a cell set: columns [a, b) minus [hp, hq)
struct RowSet {
    int a, b, hp, hq;
    SG_HD constexpr int count() const { return b > a ? (b - a) - (hq - hp) : 0; }
    SG_HD constexpr bool has(int x) const { return x >= a && x < b && !(x >= hp && x < hq); }
    // rank of column x among the row's columns
    SG_HD constexpr int rank(int x) const { return x - a - (x >= hq ? hq - hp : 0); }
};

SG_HD constexpr RowSet make_row(int a, int b, int hp, int hq) {
    if (b <= a) return RowSet{0, 0, 0, 0};
    if (hp < a) hp = a;
    if (hq > b) hq = b;
    if (hq <= hp) hp = hq = b;  // no hole
    return RowSet{a, b, hp, hq};
}

// imported columns of row y at level r-1 (read by level r)
SG_HD constexpr RowSet imp_row(int kind, int B, int r, int y) {
    const CRect q = rect(kind, B, r);
    if (empty(q)) return RowSet{0, 0, 0, 0};
    int a = 0, b = 0;
    if (y >= q.y0 && y < q.y1) {
        a = q.x0 - 1;
        b = q.x1 + 1;
    } else if (y == q.y0 - 1 || y == q.y1) {
        a = q.x0;
        b = q.x1;
    } else {
        return RowSet{0, 0, 0, 0};
    }
    const CRect p = rect(kind, B, r - 1);
    if (!empty(p) && y >= p.y0 && y < p.y1) return make_row(a, b, p.x0, p.x1);
    return make_row(a, b, b, b);
}

// exported columns of row y at level r
SG_HD constexpr RowSet exp_row(int kind, int B, int r, int y) {
    if (kind == DOWN) return RowSet{0, 0, 0, 0};  // the last phase: output only
    const CRect q = rect(kind, B, r);
    if (empty(q) || y < q.y0 || y >= q.y1) return RowSet{0, 0, 0, 0};
    const CRect nq = rect(kind, B, r + 1);
    if (!empty(nq) && y >= nq.y0 + 1 && y < nq.y1 - 1) return make_row(q.x0, q.x1, nq.x0 + 1, nq.x1 - 1);
    return make_row(q.x0, q.x1, q.x1, q.x1);
}

// slot of (r, row y) = level base + row base; rows y in [ylo, ylo + B)
SG_HD constexpr int imp_base(int kind, int B, int r, int y) {
    int s = 0;
    for (int rr = 1; rr < r; ++rr)
        for (int yy = ylo(kind, B); yy < ylo(kind, B) + B; ++yy) s += imp_row(kind, B, rr, yy).count();
    for (int yy = ylo(kind, B); yy < y; ++yy) s += imp_row(kind, B, r, yy).count();
    return s;
}
SG_HD constexpr int exp_base_rm(int kind, int B, int r, int y) {
    int s = 0;
    for (int rr = 1; rr < r; ++rr)
        for (int yy = ylo(kind, B); yy < ylo(kind, B) + B; ++yy) s += exp_row(kind, B, rr, yy).count();
    for (int yy = ylo(kind, B); yy < y; ++yy) s += exp_row(kind, B, r, yy).count();
    return s;
}
SG_HD constexpr int imp_total(int kind, int B) { return imp_base(kind, B, nlev(kind, B) + 1, ylo(kind, B)); }

// row-major slot of an imported cell at level r-1 (column x, row y), -1 if
// not an import (COL-mode levels; imp_slot below picks per level)
SG_HD constexpr int imp_slot_rm(int kind, int B, int r, int x, int y) {
    if (y < ylo(kind, B) || y >= ylo(kind, B) + B) return -1;
    const RowSet s = imp_row(kind, B, r, y);
    return s.has(x) ? imp_base(kind, B, r, y) + s.rank(x) : -1;
}
// Record layout of the exports, grouped by who reads them (so that the
// cells one consumer launch reads from a record are contiguous and whole
// 128-byte lines serve it; with a plain level/row order the lines a launch
// touches are shared with cells other launches read, 1.7x the read bytes):
//   G1: the band cells (left/right columns) of the rows with a hole -- read
//       by the horizontal neighbours,
//   G3: the band cells of the full rows (the corners),
//   G2: the middle cells of the full rows -- read by the vertical neighbours,
// in the order [G1][G3][G2]; within a group by level, row, column.  A level's
// band is [x0, x1) minus the middle [mp, mq) (the hole of its hole rows; a
// level without hole rows has no band).
struct ExpLev {
    int x0, x1, mp, mq;  // R_r columns; middle columns
    int yh0, nh;         // hole rows [yh0, yh0 + nh)
    int ytop, ntop;      // full rows: a top run ...
    int ybot, nbot;      // ... and a bottom run
    int g1, g3, g2;      // first record index of the level in each group
    SG_HD constexpr int bw() const { return (mp - x0) + (x1 - mq); }
    SG_HD constexpr int mw() const { return mq - mp; }
    SG_HD constexpr int nf() const { return ntop + nbot; }
    SG_HD constexpr int count() const { return nh * bw() + nf() * (bw() + mw()); }
    SG_HD constexpr bool band(int x) const { return x >= x0 && x < x1 && !(x >= mp && x < mq); }
    SG_HD constexpr bool mid(int x) const { return x >= mp && x < mq; }
    SG_HD constexpr int rank_band(int x) const { return x - x0 - (x >= mq ? mq - mp : 0); }
    SG_HD constexpr bool hole_row(int y) const { return y >= yh0 && y < yh0 + nh; }
    SG_HD constexpr int full_index(int y) const {  // -1: not a full row
        return (y >= ytop && y < ytop + ntop) ? y - ytop : (y >= ybot && y < ybot + nbot) ? ntop + (y - ybot) : -1;
    }
    SG_HD constexpr int slot(int x, int y) const {
        if (hole_row(y)) return band(x) ? g1 + (y - yh0) * bw() + rank_band(x) : -1;
        const int f = full_index(y);
        if (f < 0 || x < x0 || x >= x1) return -1;
        return band(x) ? g3 + f * bw() + rank_band(x) : g2 + f * mw() + (x - mp);
    }
};
constexpr int kMaxLevCap = 32;
struct ExpLayout {
    ExpLev lev[kMaxLevCap];
    int total;
};
SG_HD constexpr ExpLayout exp_layout(int kind, int B) {
    ExpLayout L{};
    const int nl = nlev(kind, B);
    int t1 = 0, t3 = 0, t2 = 0;
    for (int r = 1; r <= nl; ++r) {
        ExpLev c{};
        const CRect q = rect(kind, B, r);
        c.x0 = q.x0;
        c.x1 = q.x1;
        c.mp = q.x0;
        c.mq = q.x1;
        bool holes = false;
        for (int y = ylo(kind, B); y < ylo(kind, B) + B; ++y) {
            const RowSet s = exp_row(kind, B, r, y);
            if (s.count() == 0) continue;
            if (s.hq > s.hp) {  // a hole row
                if (c.nh == 0) c.yh0 = y;
                ++c.nh;
                c.mp = s.hp;
                c.mq = s.hq;
                holes = true;
            } else if (c.nh == 0 && c.nbot == 0 && (c.ntop == 0 || y == c.ytop + c.ntop)) {
                if (c.ntop == 0) c.ytop = y;
                ++c.ntop;
            } else {
                if (c.nbot == 0) c.ybot = y;
                ++c.nbot;
            }
        }
        if (!holes) {
            c.mp = q.x0;
            c.mq = q.x1;
        }
        c.g1 = t1;
        t1 += c.nh * c.bw();
        c.g3 = t3;
        t3 += c.nf() * c.bw();
        c.g2 = t2;
        t2 += c.nf() * c.mw();
        L.lev[r] = c;
    }
    for (int r = 1; r <= nl; ++r) {
        L.lev[r].g3 += t1;
        L.lev[r].g2 += t1 + t3;
    }
    L.total = t1 + t3 + t2;
    return L;
}
// b = 32 keeps the plain level/row/column order: its records are large
// enough that the lines each launch reads are already 90 % useful (1.11x vs
// 1.10x grouped) and the grouped store code costs the 30-level Octahedron
// ~50 registers (2 instead of 3 resident CTAs)
SG_HD constexpr bool grouped_exports(int B) { return B < 32; }
SG_HD constexpr int exp_total(int kind, int B) {
    return grouped_exports(B) ? exp_layout(kind, B).total : exp_base_rm(kind, B, nlev(kind, B) + 1, ylo(kind, B));
}
// record index of an exported cell at level r, -1 if not exported
SG_HD constexpr int exp_slot(int kind, int B, int r, int x, int y) {
    const RowSet s = exp_row(kind, B, r, y);
    if (!s.has(x)) return -1;
    return grouped_exports(B) ? exp_layout(kind, B).lev[r].slot(x, y) : exp_base_rm(kind, B, r, y) + s.rank(x);
}

// Row types of a level: the distinct RowSets among its rows, in row order
// (at most 4 for imports, 2 for exports), so the kernels evaluate each lane
// predicate / rank once per level and address rows with immediates.
SG_HD constexpr bool same(RowSet p, RowSet q) { return p.a == q.a && p.b == q.b && p.hp == q.hp && p.hq == q.hq; }
template <bool IMP>
SG_HD constexpr RowSet row_of(int kind, int B, int r, int y) {
    return IMP ? imp_row(kind, B, r, y) : exp_row(kind, B, r, y);
}
// type index of row y (-1: the row is empty)
template <bool IMP>
SG_HD constexpr int type_of(int kind, int B, int r, int y) {
    const RowSet s = row_of<IMP>(kind, B, r, y);
    if (s.count() == 0) return -1;
    int t = 0;
    for (int yy = ylo(kind, B); yy < y; ++yy) {
        const RowSet q = row_of<IMP>(kind, B, r, yy);
        if (q.count() == 0) continue;
        bool seen = false;
        for (int zz = ylo(kind, B); zz < yy; ++zz)
            if (row_of<IMP>(kind, B, r, zz).count() > 0 && same(row_of<IMP>(kind, B, r, zz), q)) seen = true;
        if (seen) continue;
        if (same(q, s)) return t;
        ++t;
    }
    return t;
}
// the t-th distinct row set of level r (count() == 0 if none)
template <bool IMP>
SG_HD constexpr RowSet type_set(int kind, int B, int r, int t) {
    for (int y = ylo(kind, B); y < ylo(kind, B) + B; ++y)
        if (type_of<IMP>(kind, B, r, y) == t) return row_of<IMP>(kind, B, r, y);
    return RowSet{0, 0, 0, 0};
}

// Lane mode per level: COL (lane = column, registers = rows) or ROW (lane =
// row, registers = columns), whichever iterates fewer registers: the bridges
// start wide-and-short and end narrow-and-tall (YBridge) or the reverse
// (XBridge), so each switches once; the pyramids and the octahedron stay COL.
constexpr int COL = 0, ROW = 1;
SG_HD constexpr int mode(int kind, int B, int r) {
    const CRect q = rect(kind, B, r);
    if (empty(q)) return COL;
    return (q.x1 - q.x0) < (q.y1 - q.y0) ? ROW : COL;
}
// Imported rows of column x at level r-1 (the transpose of imp_row): ROW-mode
// levels (lane = window row) store their imports column-major, so that a
// warp's per-column shared load reads consecutive slots (no bank conflicts)
// exactly as a COL-mode level's per-row load does.
SG_HD constexpr RowSet imp_col(int kind, int B, int r, int x) {
    const CRect q = rect(kind, B, r);
    if (empty(q)) return RowSet{0, 0, 0, 0};
    int a = 0, b = 0;
    if (x >= q.x0 && x < q.x1) {
        a = q.y0 - 1;
        b = q.y1 + 1;
    } else if (x == q.x0 - 1 || x == q.x1) {
        a = q.y0;
        b = q.y1;
    } else {
        return RowSet{0, 0, 0, 0};
    }
    const CRect p = rect(kind, B, r - 1);
    if (!empty(p) && x >= p.x0 && x < p.x1) return make_row(a, b, p.y0, p.y1);
    return make_row(a, b, b, b);
}
// first slot of column x's imports at a ROW-mode level r (after the level base)
SG_HD constexpr int imp_cbase(int kind, int B, int r, int x) {
    int s = imp_base(kind, B, r, ylo(kind, B));
    for (int xx = 0; xx < x; ++xx) s += imp_col(kind, B, r, xx).count();
    return s;
}
// slot of an imported cell at level r-1 (column x, row y), -1 if not an
// import: row-major at COL-mode levels, column-major at ROW-mode levels
SG_HD constexpr int imp_slot(int kind, int B, int r, int x, int y) {
    if (y < ylo(kind, B) || y >= ylo(kind, B) + B || x < 0 || x >= B) return -1;
    if (mode(kind, B, r) == COL) return imp_slot_rm(kind, B, r, x, y);
    const RowSet c = imp_col(kind, B, r, x);
    return c.has(y) ? imp_cbase(kind, B, r, x) + c.rank(y) : -1;
}

// both enumerations cover the same cells (checked at compile time by the kernels)
SG_HD constexpr bool imp_cols_ok(int kind, int B) {
    for (int r = 1; r <= nlev(kind, B); ++r) {
        int nr = 0, nc = 0;
        for (int i = 0; i < B; ++i) {
            nr += imp_row(kind, B, r, ylo(kind, B) + i).count();
            nc += imp_col(kind, B, r, i).count();
            const RowSet c = imp_col(kind, B, r, i);
            for (int y = c.a; y < c.b; ++y)
                if (c.has(y) && (y < ylo(kind, B) || y >= ylo(kind, B) + B || !imp_row(kind, B, r, y).has(i)))
                    return false;
        }
        if (nr != nc) return false;
    }
    return true;
}

// transpose tile (cells of R_r at a mode switch after level r), doubles
SG_HD constexpr int tile_doubles(int kind, int B) {
    int m = 0;
    for (int r = 1; r < nlev(kind, B); ++r)
        if (mode(kind, B, r) != mode(kind, B, r + 1)) {
            const CRect q = rect(kind, B, r);
            const int a = ((q.x1 - q.x0) | 1) * (q.y1 - q.y0);  // odd row stride: no bank conflicts
            m = a > m ? a : m;
        }
    return m;
}

// All of the above for one (kind, B), evaluated once per kernel instantiation
// (the kernels index these tables in constant expressions; recomputing the
// loops above at every use made the device build slow).
constexpr int kMaxB = 32;
constexpr int kMaxNL = 2 * (kMaxB / 2 - 1);
// a run of consecutive window rows i in [i0, i1) of the same row type t whose
// first slot is base and which hold cnt cells each (ROW-mode lane lookup)
struct Run {
    int i0, i1, t, base, cnt;
};
constexpr int kMaxRuns = 6;
struct Tables {
    RowSet imp[kMaxNL + 1][kMaxB], expr[kMaxNL + 1][kMaxB];
    Run imp_runs[kMaxNL + 1][kMaxRuns], exp_runs[kMaxNL + 1][kMaxRuns];
    int imp_base[kMaxNL + 2][kMaxB], exp_base[kMaxNL + 2][kMaxB];
    int imp_type[kMaxNL + 1][kMaxB], exp_type[kMaxNL + 1][kMaxB];
    RowSet imp_tset[kMaxNL + 1][4], exp_tset[kMaxNL + 1][2];
    // ROW-mode levels: imported rows per column, their types and first slots
    RowSet impc[kMaxNL + 1][kMaxB];
    int impc_type[kMaxNL + 1][kMaxB], impc_base[kMaxNL + 1][kMaxB];
    RowSet impc_tset[kMaxNL + 1][4];
    ExpLayout exp;  // grouped layout (b < 32); the exp_* row tables: row-major (b = 32)
};
template <int NT>
SG_HD constexpr void fill_types(const RowSet (&rows)[kMaxNL + 1][kMaxB], int nl, int B, int (&type)[kMaxNL + 1][kMaxB],
                                RowSet (&tset)[kMaxNL + 1][NT]) {
    for (int r = 1; r <= nl; ++r) {
        RowSet seen[kMaxB] = {};
        int n = 0;
        for (int i = 0; i < B; ++i) {
            const RowSet s = rows[r][i];
            type[r][i] = -1;
            if (s.count() == 0) continue;
            int t = -1;
            for (int u = 0; u < n; ++u)
                if (same(seen[u], s)) t = u;
            if (t < 0) {
                t = n;
                seen[n++] = s;
            }
            type[r][i] = t;
        }
        for (int u = 0; u < NT; ++u) tset[r][u] = u < n ? seen[u] : RowSet{0, 0, 0, 0};
    }
}
SG_HD constexpr void fill_runs(const int (&type)[kMaxNL + 1][kMaxB], const int (&base)[kMaxNL + 2][kMaxB],
                               const RowSet (&rows)[kMaxNL + 1][kMaxB], int nl, int B,
                               Run (&runs)[kMaxNL + 1][kMaxRuns]) {
    for (int r = 1; r <= nl; ++r) {
        int n = 0;
        for (int u = 0; u < kMaxRuns; ++u) runs[r][u] = Run{0, 0, -1, 0, 0};
        for (int i = 0; i < B; ++i) {
            if (type[r][i] < 0) continue;
            if (n > 0 && runs[r][n - 1].i1 == i && runs[r][n - 1].t == type[r][i]) {
                runs[r][n - 1].i1 = i + 1;
                continue;
            }
            if (n == kMaxRuns) return;  // (never for the supported kinds; checked by static_assert in the kernel)
            runs[r][n++] = Run{i, i + 1, type[r][i], base[r][i], rows[r][i].count()};
        }
    }
}
SG_HD constexpr Tables make_tables(int kind, int B) {
    Tables t{};
    const int nl = nlev(kind, B), y0 = ylo(kind, B);
    int si = 0, se = 0;
    for (int r = 1; r <= nl + 1; ++r)
        for (int i = 0; i < B; ++i) {
            t.imp_base[r][i] = si;
            t.exp_base[r][i] = se;
            if (r <= nl) {
                t.imp[r][i] = imp_row(kind, B, r, y0 + i);
                t.expr[r][i] = exp_row(kind, B, r, y0 + i);
                si += t.imp[r][i].count();
                se += t.expr[r][i].count();
            }
        }
    fill_types<4>(t.imp, nl, B, t.imp_type, t.imp_tset);
    for (int r = 1; r <= nl; ++r) {
        int sc = t.imp_base[r][0];
        for (int x = 0; x < B; ++x) {
            t.impc[r][x] = imp_col(kind, B, r, x);
            t.impc_base[r][x] = sc;
            sc += t.impc[r][x].count();
        }
    }
    fill_types<4>(t.impc, nl, B, t.impc_type, t.impc_tset);
    fill_types<2>(t.expr, nl, B, t.exp_type, t.exp_tset);
    fill_runs(t.imp_type, t.imp_base, t.imp, nl, B, t.imp_runs);
    fill_runs(t.exp_type, t.exp_base, t.expr, nl, B, t.exp_runs);
    t.exp = exp_layout(kind, B);
    return t;
}
template <int KIND, int B>
struct Geo {
    static constexpr Tables t = make_tables(KIND, B);
};

// Two-part gather: imports read by levels <= gather_split (part A) are waited
// for before level 1, the rest (part B) only before level split+1, so part
// B's HBM latency overlaps the first levels' compute.
SG_HD constexpr int last_imp_level(int kind, int B) {
    int last = 0;
    for (int r = 1; r <= nlev(kind, B); ++r)
        for (int y = ylo(kind, B); y < ylo(kind, B) + B; ++y)
            if (imp_row(kind, B, r, y).count() > 0) last = r;
    return last;
}
SG_HD constexpr int gather_split(int kind, int B) { return (last_imp_level(kind, B) + 1) / 2; }

SG_HD constexpr bool supported(int B) { return B == 8 || B == 12 || B == 16 || B == 24 || B == 32; }

}  // namespace col
}  // namespace sg
