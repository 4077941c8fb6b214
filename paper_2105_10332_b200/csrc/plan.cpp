// Swept plan compiler -- see plan.hpp.
#include "plan.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <map>
#include <sstream>
#include <tuple>
#include <unordered_map>

#include "colgeom.hpp"

namespace sg {

static_assert(col::UP == K_UP && col::YB == K_YB && col::XB == K_XB && col::OCT == K_OCT && col::DOWN == K_DOWN,
              "colgeom kind ids");

namespace {

constexpr int R = 5;       // replay tile: R x R blocks, periodic
constexpr int REP = 2;     // representative instance (REP, REP)
constexpr long MAXR = 9;   // replay at most this many octahedron cycles

struct RLaunch {
    int kind;
    long lo, hi;
    int frame;
    long cycle;
};

// build_schedule_cycles (geometry.cpp:122-167) as GPU launches, with the
// frame recipe of SURVEY.md §8a: every Communicate toggles the frame.
std::vector<RLaunch> launch_sequence(long m, int k) {
    std::vector<RLaunch> s;
    s.push_back({K_UP, 1, k, 0, 0});
    s.push_back({K_YB, 1, k, 0, 0});
    s.push_back({K_XB, 1, k, 1, 0});
    for (long j = 1; j <= m; ++j) {
        const int F = (j % 2 == 1) ? 1 : 0;
        s.push_back({K_OCT, (j - 1) * k + 1, (j + 1) * k, F, j});
        s.push_back({K_YB, j * k + 1, (j + 1) * k, F, j});
        s.push_back({K_XB, j * k + 1, (j + 1) * k, 1 - F, j});
    }
    s.push_back({K_DOWN, m * k + 1, (m + 1) * k, ((m + 1) % 2 == 1) ? 1 : 0, m + 1});
    return s;
}

// One imported cell of a replayed instance, in relative terms.
struct RImport {
    int r, qx, qy;             // consumer relative level and coords
    int delta;                 // 0 => initial plane
    int di, dj, pkind;         // producer offset / kind
    int pr, px, py;            // producer relative level / coords
    bool operator<(const RImport& o) const {
        return std::tie(delta, di, dj, pr, py, px, r, qy, qx) <
               std::tie(o.delta, o.di, o.dj, o.pr, o.py, o.px, o.r, o.qy, o.qx);
    }
    bool operator==(const RImport& o) const {
        return std::tie(r, qx, qy, delta, di, dj, pkind, pr, px, py) ==
               std::tie(o.r, o.qx, o.qy, o.delta, o.di, o.dj, o.pkind, o.pr, o.px, o.py);
    }
};

// 8-byte shared accesses of one warp instruction: wavefronts = per half warp
// the max number of distinct addresses sharing a bank pair
int wavefronts(const std::vector<long>& addr) {
    int wf = 0;
    for (int h = 0; h < 2; ++h) {
        std::map<long, std::vector<long>> bank;
        for (std::size_t l = h * 16; l < std::min<std::size_t>(addr.size(), h * 16 + 16); ++l)
            if (addr[l] >= 0) {
                auto& v = bank[((addr[l] % 16) + 16) % 16];
                if (std::find(v.begin(), v.end(), addr[l]) == v.end()) v.push_back(addr[l]);
            }
        int mx = 0;
        for (auto& kv : bank) mx = std::max<int>(mx, static_cast<int>(kv.second.size()));
        wf += mx;
    }
    return wf;
}

}  // namespace

void lane_split(int w, int h, int* splits_out, int* rps_out) {
    const int cap = w >= 32 ? 1 : std::max(1, std::min(h, 32 / std::max(1, w)));
    int splits = 1;
    for (int d = cap; d >= 1; --d)
        if (h % d == 0) {
            splits = d;
            break;
        }
    if (2 * splits < cap) splits = cap;  // no good divisor: accept a ragged last chunk
    const int rps = (h + splits - 1) / splits;
    *splits_out = (h + rps - 1) / rps;
    *rps_out = rps;
}

template <class T, class Key>
void spread_banks(std::vector<T>& v, std::size_t begin, std::size_t end, Key key) {
    for (std::size_t g = begin; g < end; g += 32) {
        const std::size_t ge = std::min(end, g + 32);
        std::vector<T> in(v.begin() + g, v.begin() + ge), out;
        std::vector<bool> used(in.size(), false);
        for (int half = 0; half < 2 && out.size() < in.size(); ++half) {
            bool taken[16] = {false};
            const std::size_t target = std::min(in.size(), out.size() + 16);
            for (std::size_t i = 0; i < in.size() && out.size() < target; ++i)  // one per bank pair first
                if (!used[i] && !taken[((key(in[i]) % 16) + 16) % 16]) {
                    taken[((key(in[i]) % 16) + 16) % 16] = true;
                    used[i] = true;
                    out.push_back(in[i]);
                }
            for (std::size_t i = 0; i < in.size() && out.size() < target; ++i)
                if (!used[i]) {
                    used[i] = true;
                    out.push_back(in[i]);
                }
        }
        std::copy(out.begin(), out.end(), v.begin() + g);
    }
}

SweptPlan compile_swept_plan(int b, const Equation& eq, long m, long final_level, long instances,
                             long partition_instances) {
    SweptPlan P;
    P.b = b;
    P.n = eq.halo;
    P.S = eq.substeps;
    P.nvars = eq.nvars;
    P.k = max_levels(b, eq.halo);
    P.m = m;
    P.flat = static_cast<long>(P.k) * (m + 1);
    P.final_level = final_level;
    const int n = P.n, k = P.k, S = P.S;
    {
        const char* env = std::getenv("SG_HEAT_KERNEL");
        const bool forced = env && std::strcmp(env, "column") == 0;
        // (a record ring too large for the column kernels' 32-bit gather
        // offsets is caught by the engine, which then recompiles generic)
        (void)partition_instances;
        const bool generic =
            (env && std::strcmp(env, "generic") == 0) || (!forced && instances > 0 && instances < 2048);
        if (eq.problem == SG_HEAT && n == 1 && S == 1 && col::supported(b) && !generic) P.colB = b;
    }
    if (final_level < 1 || final_level > P.flat) fail(SG_ELOGIC, "plan: final level outside the schedule");

    const long mr = (m <= MAXR) ? m : (8 + (m % 2));
    P.replay_cycles = mr;
    const std::vector<RLaunch> rseq = launch_sequence(mr, k);
    const long rflat = static_cast<long>(k) * (mr + 1);

    // ---------------------------------------------------------- replay --
    const int W = R * b;
    const int WIN = 2 * k + S + 2;
    const int RR = R * R;
    std::vector<int> owner(static_cast<std::size_t>(WIN) * W * W, -1);
    std::vector<long> slot_level(WIN, -1);
    auto wrap = [W](int v) { return ((v % W) + W) % W; };
    auto wrapc = [W, b](int v) { return ((v + b) % W + W) % W - b; };
    auto wrapd = [](int d) { return ((d + 2) % R + R) % R - 2; };
    auto slot_of = [&](long lev) { return static_cast<int>(lev % WIN); };
    auto at = [&](long lev, int x, int y) -> int& {
        return owner[(static_cast<std::size_t>(slot_of(lev)) * W + y) * W + x];
    };
    // level 0 = the initial plane
    slot_level[0] = 0;
    std::fill(owner.begin(), owner.begin() + static_cast<std::size_t>(W) * W, -2);

    std::vector<std::vector<RImport>> rep_imports(rseq.size());
    for (std::size_t L = 0; L < rseq.size(); ++L) {
        const RLaunch& la = rseq[L];
        const int nlev = kind_levels(la.kind, k);
        for (int r = 1; r <= nlev; ++r) {
            const long lev = la.lo + r - 1;
            const int s = slot_of(lev);
            if (slot_level[s] != lev) {
                if (slot_level[s] > lev) fail(SG_ELOGIC, "plan: replay window overflow");
                std::fill(owner.begin() + static_cast<std::size_t>(s) * W * W,
                          owner.begin() + static_cast<std::size_t>(s + 1) * W * W, -1);
                slot_level[s] = lev;
            }
        }
        std::vector<RImport> rep_sig;
        for (int inst = 0; inst < RR; ++inst) {
            const int bi = inst % R, bj = inst / R;
            const int ox = bi * b - la.frame * (b / 2), oy = bj * b - la.frame * (b / 2);
            const int me = static_cast<int>(L) * RR + inst;
            std::map<std::tuple<int, int, int>, RImport> imps;
            for (int r = 1; r <= nlev; ++r) {
                const long lev = la.lo + r - 1;
                const int stage = static_cast<int>((lev - 1) % S);
                const Rect rc = kind_rect(la.kind, b, n, k, r);
                for (int y = rc.y0; y < rc.y1; ++y)
                    for (int x = rc.x0; x < rc.x1; ++x) {
                        int& mine = at(lev, wrap(ox + x), wrap(oy + y));
                        if (mine != -1) fail(SG_ELOGIC, "plan: cell computed twice");
                        // cross stencil at level-1 (StencilShape reads, geometry.cpp:8-24)
                        auto visit = [&](long rl, int qx, int qy) {
                            if (slot_level[slot_of(rl)] != rl)
                                fail(SG_ELOGIC, "plan: read of a level outside the window");
                            const int o = at(rl, wrap(ox + qx), wrap(oy + qy));
                            if (o == -1) fail(SG_ELOGIC, "plan: read before write");
                            if (o == me) return;
                            if (o >= 0 && o / RR == static_cast<int>(L))
                                fail(SG_ELOGIC, "plan: reads a concurrent instance");
                            const int rr = static_cast<int>(rl - la.lo + 1);
                            RImport im{rr, qx, qy, 0, 0, 0, 0, 0, 0, 0};
                            if (o == -2) {
                                im.delta = 0;
                                im.pr = 0;
                                im.px = qx;
                                im.py = qy;
                            } else {
                                const int pl = o / RR, pi = o % RR;
                                const RLaunch& pla = rseq[pl];
                                const int pbi = pi % R, pbj = pi / R;
                                const int pox = pbi * b - pla.frame * (b / 2),
                                          poy = pbj * b - pla.frame * (b / 2);
                                im.delta = static_cast<int>(L) - pl;
                                im.di = wrapd(pbi - bi);
                                im.dj = wrapd(pbj - bj);
                                im.pkind = pla.kind;
                                im.pr = static_cast<int>(rl - pla.lo + 1);
                                im.px = wrapc(wrap(ox + qx) - pox);
                                im.py = wrapc(wrap(oy + qy) - poy);
                            }
                            imps.emplace(std::make_tuple(rr, qy, qx), im);
                        };
                        for (int d = -n; d <= n; ++d) {
                            visit(lev - 1, x + d, y);
                            if (d != 0) visit(lev - 1, x, y + d);
                        }
                        if (stage == 1) visit(lev - 2, x, y);  // corrector base Q^n
                        mine = me;
                    }
            }
            std::vector<RImport> sig;
            sig.reserve(imps.size());
            for (auto& kv : imps) sig.push_back(kv.second);
            std::sort(sig.begin(), sig.end());
            if (inst == 0) rep_sig = sig;
            else if (!(sig == rep_sig))
                fail(SG_ELOGIC, "plan: phase instances are not translation invariant");
            if (bi == REP && bj == REP) rep_imports[L] = sig;
        }
    }
    // every cell of every level up to the flat level was produced exactly once
    for (long lev = std::max(1L, rflat - (WIN - 3)); lev <= rflat; ++lev) {
        if (slot_level[slot_of(lev)] != lev) fail(SG_ELOGIC, "plan: level missing from replay");
        for (int y = 0; y < W; ++y)
            for (int x = 0; x < W; ++x)
                if (at(lev, x, y) < 0) fail(SG_ELOGIC, "plan: schedule leaves a hole");
    }

    // --------------------------------------------- real -> replay launches --
    const std::vector<RLaunch> seq = launch_sequence(m, k);
    auto map_cycle = [&](long j) -> long {
        if (m <= MAXR) return j;
        if (j <= 3) return j;
        if (j >= m - 2) return j - (m - mr);
        return (j % 2 == 0) ? 4 : 5;
    };
    auto replay_index = [&](std::size_t i) -> std::size_t {
        const RLaunch& la = seq[i];
        if (la.kind == K_DOWN) return rseq.size() - 1;
        if (la.cycle == 0) return i;
        const long jr = map_cycle(la.cycle);
        return 3 + static_cast<std::size_t>(jr - 1) * 3 + (i - 3) % 3;
    };
    if (m > MAXR) {  // steady state must repeat with period 2 (one shift pair)
        for (int j : {4, 5})
            for (int w = 0; w < 3; ++w) {
                const std::size_t a = 3 + (j - 1) * 3 + w, c = 3 + (j + 1) * 3 + w;
                if (!(rep_imports[a] == rep_imports[c]))
                    fail(SG_ELOGIC, "plan: swept steady state is not periodic");
            }
    }

    // ----------------------------------------------------- kind layouts --
    // Export sets: every cell some other instance imports, per producer kind,
    // tagged with the consumer groups that read it (for record ordering).
    std::map<std::array<int, 3>, unsigned long long> exp_mask[K_NKINDS];
    std::map<std::tuple<int, int, int>, int> group_id;
    for (std::size_t L = 0; L < rseq.size(); ++L)
        for (const RImport& im : rep_imports[L]) {
            if (im.delta == 0) continue;
            auto key = std::make_tuple(rseq[L].kind, -im.di, -im.dj);
            auto g = group_id.emplace(key, static_cast<int>(group_id.size())).first->second;
            exp_mask[im.pkind][{im.pr, im.px, im.py}] |= 1ull << (g % 64);
        }
    for (int kd = 0; kd < K_NKINDS; ++kd) {
        KindLayout& K = P.kinds[kd];
        K.kind = kd;
        K.nlev = kind_levels(kd, k);
        // resident cells per relative level
        std::map<int, Rect> box;
        auto grow = [&](int r, int x, int y) {
            auto it = box.find(r);
            if (it == box.end()) box[r] = Rect{x, x + 1, y, y + 1};
            else {
                Rect& q = it->second;
                q.x0 = std::min(q.x0, x);
                q.x1 = std::max(q.x1, x + 1);
                q.y0 = std::min(q.y0, y);
                q.y1 = std::max(q.y1, y + 1);
            }
        };
        for (int r = 1; r <= K.nlev; ++r) {
            const Rect c = kind_rect(kd, b, n, k, r);
            grow(r, c.x0, c.y0);
            grow(r, c.x1 - 1, c.y1 - 1);
        }
        for (std::size_t L = 0; L < rseq.size(); ++L)
            if (rseq[L].kind == kd)
                for (const RImport& im : rep_imports[L]) grow(im.r, im.qx, im.qy);
        K.rmin = box.empty() ? 1 : std::min(1, box.begin()->first);
        int mil = K.rmin;  // highest level that receives imports
        for (std::size_t L = 0; L < rseq.size(); ++L)
            if (rseq[L].kind == kd)
                for (const RImport& im : rep_imports[L]) mil = std::max(mil, im.r);
        int off = 0;
        for (int r = K.rmin; r <= K.nlev; ++r) {
            PlanLevel pl;
            auto it = box.find(r);
            if (it != box.end()) pl.bbox = it->second;
            pl.off = off;
            pl.pitch = pl.bbox.w();
            if (eq.problem == SG_HEAT && !pl.bbox.empty()) {
                // row pitch >= width that makes the lane maps touching this level
                // (its own writes, level r+1's reads) free of bank conflicts
                std::vector<std::vector<std::pair<int, int>>> maps;  // lane -> (x, y)
                for (int rr : {r, r + 1}) {
                    if (rr < 1 || rr > K.nlev) continue;
                    const Rect cr = kind_rect(kd, b, n, k, rr);
                    int sp, rp;
                    lane_split(cr.w(), cr.h(), &sp, &rp);
                    std::vector<std::pair<int, int>> m;
                    for (int l = 0; l < 32; ++l)
                        if (cr.w() <= 32 && l < cr.w() * sp && cr.y0 + (l / cr.w()) * rp < cr.y1)
                            m.push_back({cr.x0 + l % cr.w(), cr.y0 + (l / cr.w()) * rp});
                        else
                            m.push_back({-1 << 20, 0});
                    maps.push_back(m);
                }
                int best = -1, bestp = pl.bbox.w();
                for (int cand = pl.bbox.w(); cand < pl.bbox.w() + 16; ++cand) {
                    int cost = 0;
                    for (const auto& m : maps) {
                        std::vector<long> a;
                        for (const auto& xy : m)
                            a.push_back(xy.first < -1000 ? -1 : (long)(xy.second - pl.bbox.y0) * cand + (xy.first - pl.bbox.x0));
                        cost += wavefronts(a);
                    }
                    if (best < 0 || cost < best) {
                        best = cost;
                        bestp = cand;
                    }
                }
                pl.pitch = bestp;
            }
            pl.vstride = pl.bbox.h() * pl.pitch;
            if (r >= 1) pl.comp = kind_rect(kd, b, n, k, r);
            off += pl.vstride * P.nvars;
            K.lev.push_back(pl);
        }
        K.smem_doubles = off;
        K.split = K.nlev;
        if (mil >= 1 && mil < K.nlev) {
            // levels above `mil` overwrite the dead storage of levels < mil-S+1
            const int keep = mil - S + 1;
            const int limit = (keep >= K.rmin) ? K.at(keep).off : 0;
            int upper = 0;
            for (int r = mil + 1; r <= K.nlev; ++r) upper += K.at(r).vstride * P.nvars;
            if (upper <= limit) {
                int o = 0;
                for (int r = mil + 1; r <= K.nlev; ++r) {
                    K.lev[r - K.rmin].off = o;
                    o += K.lev[r - K.rmin].vstride * P.nvars;
                }
                K.smem_doubles = K.at(mil).off + K.at(mil).vstride * P.nvars;
                K.split = mil;
            }
        }
        // export list ordered by consumer group set, then level, row, column
        std::vector<std::tuple<int, unsigned long long, int, int, int>> cells;
        for (auto& kv : exp_mask[kd])
            cells.emplace_back(kv.first[0] > K.split ? 1 : 0, kv.second, kv.first[0], kv.first[2], kv.first[1]);
        std::sort(cells.begin(), cells.end());
        for (auto& c : cells) {
            const int r = std::get<2>(c), y = std::get<3>(c), x = std::get<4>(c);
            if (r <= K.split) ++K.nexp_early;
            if (r < K.rmin || r > K.nlev) fail(SG_ELOGIC, "plan: export outside kind levels");
            const PlanLevel& pl = K.at(r);
            K.exp_cells.push_back({r, x, y});
            K.exp_off.push_back(pl.off + (y - pl.bbox.y0) * pl.pitch + (x - pl.bbox.x0));
            K.exp_vstride.push_back(pl.vstride);
        }
        K.epad = static_cast<int>((K.exp_cells.size() + 3) / 4 * 4);
        for (std::size_t i = 0; i < K.exp_off.size(); ++i) K.exp_pairs.push_back({K.exp_off[i], static_cast<int>(i)});
        spread_banks(K.exp_pairs, 0, K.nexp_early, [](const std::array<int, 2>& e) { return e[0]; });
        spread_banks(K.exp_pairs, K.nexp_early, K.exp_pairs.size(), [](const std::array<int, 2>& e) { return e[0]; });
        // warp lane map: (column, row-chunk) items of each computed rectangle;
        // the row split divides the height exactly when it can, so every
        // active lane runs the same trip count (no divergent row loops)
        for (int r = 1; r <= K.nlev; ++r) {
            const PlanLevel& Lc = K.at(r);
            const PlanLevel& Lp = K.at(r - 1);
            const int w = Lc.comp.w(), h = Lc.comp.h();
            K.pitch.push_back({Lp.pitch, Lc.pitch});
            int splits, rps;
            lane_split(w, h, &splits, &rps);
            for (int l = 0; l < 32; ++l) {
                std::array<int, 4> e{0, 0, 0, 0};
                if (w <= 32 && l < w * splits) {
                    const int xi = l % w, ch = l / w;
                    const int x = Lc.comp.x0 + xi, y0 = Lc.comp.y0 + ch * rps;
                    const int rows = std::max(0, std::min(rps, Lc.comp.y1 - y0));
                    if (rows > 0) {
                        e[0] = Lp.off + (y0 - Lp.bbox.y0) * Lp.pitch + (x - Lp.bbox.x0);
                        e[1] = Lc.off + (y0 - Lc.bbox.y0) * Lc.pitch + (x - Lc.bbox.x0);
                        e[2] = rows;
                        e[3] = (x & 0xFFFF) | ((y0 & 0xFFFF) << 16);
                    }
                }
                K.lanes.push_back(e);
            }
        }
        P.max_epad = std::max(P.max_epad, K.epad);
        long upd = 0;
        for (int r = 1; r <= K.nlev; ++r) upd += kind_rect(kd, b, n, k, r).area();
        P.updates_per_kind[kd] = upd;
    }
    if (P.colB) {
        // column-register kernels: closed-form export order and import slots
        // (colgeom.hpp); the replayed export set must be covered
        P.max_epad = 0;
        for (int kd = 0; kd < K_NKINDS; ++kd) {
            KindLayout& K = P.kinds[kd];
            std::set<std::array<int, 3>> formula;
            K.exp_cells.clear();
            K.exp_off.clear();
            K.exp_vstride.clear();
            K.exp_pairs.clear();
            std::vector<std::array<int, 3>> by_slot(static_cast<std::size_t>(col::exp_total(kd, b)), {-1, 0, 0});
            for (int r = 1; r <= K.nlev; ++r)
                for (int y = col::ylo(kd, b); y < col::ylo(kd, b) + b; ++y)
                    for (int x = 0; x < b; ++x)
                        if (col::exp_row(kd, b, r, y).has(x)) {
                            const int sl = col::exp_slot(kd, b, r, x, y);
                            if (sl < 0 || sl >= static_cast<int>(by_slot.size()) || by_slot[sl][0] >= 0)
                                fail(SG_ELOGIC, "plan: column export layout is not a bijection");
                            by_slot[sl] = {r, x, y};
                            formula.insert({r, x, y});
                        }
            for (const auto& c : by_slot) {
                if (c[0] < 0) fail(SG_ELOGIC, "plan: column export layout has a gap");
                K.exp_cells.push_back(c);
                K.exp_off.push_back(0);
                K.exp_vstride.push_back(0);
                K.exp_pairs.push_back({0, static_cast<int>(K.exp_pairs.size())});
            }
            if (static_cast<int>(K.exp_cells.size()) != col::exp_total(kd, b))
                fail(SG_ELOGIC, "plan: column export count");
            for (auto& kv : exp_mask[kd])
                if (!formula.count(kv.first)) fail(SG_ELOGIC, "plan: column exports miss a replayed read");
            P.overexport += static_cast<long>(formula.size() - exp_mask[kd].size());
            K.epad = static_cast<int>((K.exp_cells.size() + 3) / 4 * 4);
            K.smem_doubles = std::max(1, col::imp_total(kd, b) + col::tile_doubles(kd, b));
            // per-instance stride = 8 mod 16 doubles: a warp's next instance
            // starts half a bank row later, so a row load with <= 8 lanes per
            // instance is one wavefront (b8 +5 %, b16 +0.6 %)
            if (const char* e = std::getenv("SG_SMEM_PAD"); !(e && e[0] == '0'))
                K.smem_doubles = (K.smem_doubles + 7) / 16 * 16 + 8;
            K.split = K.nlev;
            K.nexp_early = 0;
            P.max_epad = std::max(P.max_epad, K.epad);
        }
    }
    std::map<std::array<int, 3>, int> exp_index[K_NKINDS];
    for (int kd = 0; kd < K_NKINDS; ++kd)
        for (std::size_t i = 0; i < P.kinds[kd].exp_cells.size(); ++i) {
            const auto& c = P.kinds[kd].exp_cells[i];
            exp_index[kd][{c[0], c[1], c[2]}] = static_cast<int>(i);
        }

    // ----------------------------------------------------- class tables --
    std::map<std::size_t, int> class_of_replay;
    auto build_class = [&](std::size_t L) {
        ClassTab T;
        T.kind = rseq[L].kind;
        const KindLayout& K = P.kinds[T.kind];
        std::map<std::tuple<int, int, int, int>, int> seg_id;
        for (const RImport& im : rep_imports[L]) {
            const PlanLevel& pl = K.at(im.r);
            int dst = pl.off + (im.qy - pl.bbox.y0) * pl.pitch + (im.qx - pl.bbox.x0);
            if (P.colB) {  // level im.r is read by level im.r + 1
                dst = col::imp_slot(T.kind, b, im.r + 1, im.qx, im.qy);
                if (dst < 0) fail(SG_ELOGIC, "plan: import outside the column layout");
            }
            if (im.delta == 0) {
                InitImport ii;
                ii.rx = im.qx;
                ii.ry = im.qy;
                ii.dst = dst;
                ii.vstride = pl.vstride;
                ii.r = im.r;
                T.inits.push_back(ii);
                continue;
            }
            auto key = std::make_tuple(im.delta, im.di, im.dj, im.pkind);
            auto it = seg_id.find(key);
            if (it == seg_id.end()) {
                it = seg_id.emplace(key, static_cast<int>(T.segs.size())).first;
                T.segs.push_back({im.delta, im.di, im.dj, im.pkind});
            }
            Import x;
            x.seg = it->second;
            x.src = exp_index[im.pkind].at({im.pr, im.px, im.py});
            x.dst = dst;
            x.vstride = pl.vstride;
            x.r = im.r;
            x.qx = im.qx;
            x.qy = im.qy;
            T.imports.push_back(x);
        }
        std::sort(T.imports.begin(), T.imports.end(), [](const Import& a, const Import& c) {
            return std::tie(a.seg, a.src) < std::tie(c.seg, c.src);
        });
        if (P.colB) {
            // column kernels: part A (levels <= gather_split) before part B,
            // each in (seg, src) order
            const int split = col::gather_split(T.kind, b);
            std::stable_sort(T.imports.begin(), T.imports.end(), [split](const Import& a, const Import& c) {
                return (a.r + 1 > split) < (c.r + 1 > split);
            });
            for (const Import& x : T.imports) T.nimp_b += x.r + 1 > split ? 1 : 0;
        } else {
            spread_banks(T.imports, 0, T.imports.size(), [](const Import& e) { return e.dst; });
        }
        if (P.colB) {
            std::vector<int> seen(static_cast<std::size_t>(K.smem_doubles), 0);
            for (const Import& x : T.imports) seen.at(static_cast<std::size_t>(x.dst))++;
            for (const InitImport& x : T.inits) seen.at(static_cast<std::size_t>(x.dst))++;
            for (int v : seen)
                if (v > 1) fail(SG_ELOGIC, "plan: two imports share a column slot");
        }
        return T;
    };
    int maxdelta = 0, ghost = 0;
    for (std::size_t i = 0; i < seq.size(); ++i) {
        const std::size_t ri = replay_index(i);
        auto it = class_of_replay.find(ri);
        if (it == class_of_replay.end()) {
            ClassTab T = build_class(ri);
            int found = -1;
            for (std::size_t c = 0; c < P.classes.size(); ++c) {
                const ClassTab& U = P.classes[c];
                if (U.kind != T.kind || U.segs.size() != T.segs.size() ||
                    U.imports.size() != T.imports.size() || U.inits.size() != T.inits.size())
                    continue;
                bool same = true;
                for (std::size_t s = 0; same && s < T.segs.size(); ++s)
                    same = U.segs[s].delta == T.segs[s].delta && U.segs[s].di == T.segs[s].di &&
                           U.segs[s].dj == T.segs[s].dj && U.segs[s].pkind == T.segs[s].pkind;
                for (std::size_t s = 0; same && s < T.imports.size(); ++s)
                    same = U.imports[s].seg == T.imports[s].seg && U.imports[s].src == T.imports[s].src &&
                           U.imports[s].dst == T.imports[s].dst;
                for (std::size_t s = 0; same && s < T.inits.size(); ++s)
                    same = U.inits[s].rx == T.inits[s].rx && U.inits[s].ry == T.inits[s].ry &&
                           U.inits[s].dst == T.inits[s].dst;
                if (same) found = static_cast<int>(c);
            }
            if (found < 0) {
                for (const Segment& s : T.segs) {
                    maxdelta = std::max(maxdelta, s.delta);
                    ghost = std::max(ghost, std::max(std::abs(s.di), std::abs(s.dj)));
                }
                found = static_cast<int>(P.classes.size());
                P.classes.push_back(std::move(T));
            }
            it = class_of_replay.emplace(ri, found).first;
        }
        const RLaunch& la = seq[i];
        Launch x;
        x.kind = la.kind;
        x.lo = la.lo;
        x.hi = la.hi;
        x.frame = la.frame;
        x.cls = it->second;
        x.stage0 = static_cast<int>((la.lo - 1) % S);
        x.r_out = (final_level >= la.lo && final_level <= la.hi) ? static_cast<int>(final_level - la.lo + 1) : 0;
        P.launches.push_back(x);
    }
    P.nslots = maxdelta + 1;
    P.ghost = ghost;
    for (std::size_t i = 0; i < P.launches.size(); ++i)
        if (P.kinds[P.launches[i].kind].epad > 0) P.launches[i].slot = static_cast<int>(i % P.nslots);
    for (const ClassTab& T : P.classes)
        P.imports_per_kind[T.kind] =
            std::max<long>(P.imports_per_kind[T.kind], static_cast<long>(T.imports.size() + T.inits.size()));
    return P;
}

std::string describe_plan(const SweptPlan& p) {
    std::ostringstream os;
    os << "swept plan b=" << p.b << " n=" << p.n << " k=" << p.k << " S=" << p.S << " m=" << p.m
       << " flat=" << p.flat << " final=" << p.final_level << " launches=" << p.launches.size()
       << " classes=" << p.classes.size() << " slots=" << p.nslots << " ghost=" << p.ghost
       << " replay_cycles=" << p.replay_cycles << " heat_kernel=" << (p.colB ? "column" : "generic")
       << " overexport=" << p.overexport << "\n";
    for (int kd = 0; kd < K_NKINDS; ++kd) {
        const KindLayout& K = p.kinds[kd];
        os << "  " << kind_name(kd) << ": levels " << K.rmin << ".." << K.nlev << " smem "
           << K.smem_doubles * 8 << " B, exports " << K.exp_cells.size() << " (pad " << K.epad
           << "), updates " << p.updates_per_kind[kd] << ", max imports " << p.imports_per_kind[kd]
           << "\n";
    }
    for (std::size_t c = 0; c < p.classes.size(); ++c) {
        const ClassTab& T = p.classes[c];
        os << "  class " << c << " " << kind_name(T.kind) << ": imports " << T.imports.size()
           << " init " << T.inits.size() << " segs";
        for (const Segment& s : T.segs)
            os << " [d" << s.delta << " " << s.di << "," << s.dj << " " << kind_name(s.pkind) << "]";
        {  // contiguous record runs per producer (what one bulk copy each could move)
            std::map<int, std::vector<int>> by;
            for (const Import& x : T.imports) by[x.seg].push_back(x.src);
            long runs = 0, cells16 = 0;
            for (auto& kv : by) {
                std::sort(kv.second.begin(), kv.second.end());
                for (std::size_t i = 0; i < kv.second.size();) {
                    std::size_t j = i;
                    while (j + 1 < kv.second.size() && kv.second[j + 1] == kv.second[j] + 1) ++j;
                    ++runs;
                    cells16 += ((kv.second[j] + 2) & ~1) - (kv.second[i] & ~1);
                    i = j + 1;
                }
            }
            os << " runs " << runs << " cells16 " << cells16;
        }
        os << "\n";
    }
    return os.str();
}

}  // namespace sg
