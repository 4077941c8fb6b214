// GPU engine -- see engine.hpp.
#include "engine.hpp"
#include "colgeom.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

namespace sg {

cudaError_t launch_swept(int problem, const SweptArgs& a, cudaStream_t s);
cudaError_t launch_std(int problem, const StdArgs& a, cudaStream_t s);

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dev_alloc(DeviceCtx& d, std::size_t count) {
    void* p = nullptr;
    ck(cudaSetDevice(d.dev), "cudaSetDevice");
    ck(cudaMalloc(&p, std::max<std::size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    d.allocs.push_back(p);
    return static_cast<T*>(p);
}

template <class T>
T* dev_upload(DeviceCtx& d, const std::vector<T>& v) {
    T* p = dev_alloc<T>(d, v.size());
    if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return p;
}

}  // namespace

Solver::Solver(const sg_config& cfg, int rank, int world) : cfg_(cfg), rank_(rank), world_(world) {
    const auto t0 = std::chrono::steady_clock::now();
    setup_ = make_setup(cfg_);
    if (cfg_.snapshot_path && cfg_.snapshot_path[0]) {
        snap_path_ = cfg_.snapshot_path;
        snap_every_ = cfg_.snapshot_every;
    }
    cfg_.snapshot_path = nullptr;  // the caller's string may not outlive us
    const Equation& eq = setup_.eq;
    px_ = cfg_.px;
    py_ = cfg_.py;
    if (px_ <= 0 && py_ <= 0) {
        px_ = cfg_.ranks;
        py_ = 1;
    }
    if (px_ <= 0) px_ = 1;
    if (py_ <= 0) py_ = 1;
    nparts_ = px_ * py_;
    if (nparts_ > kMaxParts) fail(SG_EINVAL, "config: too many partitions");
    pw_ = setup_.nx / px_;
    ph_ = setup_.ny / py_;

    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (ndev < 1) fail(SG_ECUDA, "no CUDA device visible (the GPU solver has no CPU fallback)");
    // SG_DEVICE_ALIAS=1 (tests only): every logical device is the current
    // physical one, so the one-process multi-device path (per-device streams,
    // cross-device event waits) runs on a single-GPU box
    const bool alias = [] {
        const char* v = std::getenv("SG_DEVICE_ALIAS");
        return v && v[0] == '1';
    }();
    int use = cfg_.devices > 0 ? (alias ? cfg_.devices : std::min(cfg_.devices, ndev)) : ndev;
    use = std::min(use, nparts_);
    int dev0 = 0;
    ck(cudaGetDevice(&dev0), "cudaGetDevice");
    if (!dist() && !alias) dev0 = 0;  // one process, many GPUs: devices 0 .. use-1
    if (dist()) {  // one process per GPU: this rank owns partition `rank` on its current device
        if (world_ != nparts_) fail(SG_EINVAL, "distributed run: world size must equal px*py");
        if (rank_ < 0 || rank_ >= world_) fail(SG_EINVAL, "distributed run: bad rank");
        use = 1;
    }
    devs_.resize(use);
    for (int d = 0; d < use; ++d) {
        const int phys = alias ? dev0 : dev0 + d;
        devs_[d].dev = phys;
        ck(cudaSetDevice(phys), "cudaSetDevice");
        ck(cudaStreamCreateWithFlags(&devs_[d].stream, cudaStreamNonBlocking), "stream");
        {  // every launch of device d goes to a stream of device d
            int sdev = -1;
            ck(cudaStreamGetDevice(devs_[d].stream, &sdev), "cudaStreamGetDevice");
            if (sdev != phys) fail(SG_ELOGIC, "stream created on the wrong device");
        }
        ck(cudaEventCreate(&devs_[d].ev_start), "event");
        ck(cudaEventCreate(&devs_[d].ev_stop), "event");
        ck(cudaEventCreateWithFlags(&devs_[d].ev_sync, cudaEventDisableTiming), "event");
        devs_[d].d_err = dev_alloc<int>(devs_[d], 1);
        for (int e = 0; e < use; ++e) {
            const int pe = alias ? dev0 : dev0 + e;
            if (pe != phys) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, phys, pe);
                if (can) {
                    cudaError_t r = cudaDeviceEnablePeerAccess(pe, 0);
                    if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled)
                        ck(r, "cudaDeviceEnablePeerAccess");
                    cudaGetLastError();
                }
            }
        }
    }
    parts_.resize(nparts_);
    for (int p = 0; p < nparts_; ++p) {
        parts_[p].id = p;
        parts_[p].pi = p % px_;
        parts_[p].pj = p / px_;
        // contiguous blocks of partitions per device; remote partitions (other
        // ranks of a distributed run) have dev = -1 and IPC-mapped buffers
        if (dist()) {
            parts_[p].dev = p == rank_ ? 0 : -1;
        } else {
            parts_[p].dev = static_cast<int>(static_cast<long>(p) * use / nparts_);
        }
        if (parts_[p].dev >= 0) devs_[parts_[p].dev].parts.push_back(p);
    }
    if (dist()) {
        DeviceCtx& d = devs_[0];
        // [kMaxParts] epochs signalled by the ranks + this rank's epoch counter
        flags_ = dev_alloc<unsigned long long>(d, kMaxParts + 1);
        ck(cudaMemset(flags_, 0, (kMaxParts + 1) * sizeof(unsigned long long)), "flags");
    }

    if (cfg_.engine == SG_SWEPT) {
        const int k = max_levels(cfg_.block, eq.halo);
        long flat = 0;
        const long m = schedule_octahedra(cfg_.steps, k, eq.substeps, &flat);
        actual_steps_ = flat / eq.substeps;
        total_levels_ = flat;
        final_level_ = actual_steps_ * eq.substeps;  // engine.cpp:518
        const long instances = static_cast<long>(setup_.nx / cfg_.block) * (setup_.ny / cfg_.block);
        plan_ = compile_swept_plan(cfg_.block, eq, m, final_level_, instances);
        if (plan_.colB) {
            // the column kernels address every producer record as a 32-bit
            // offset from the consumer's slot-0 record (imp_off): a partition's
            // whole record ring -- its real slot count, ghost ring and record
            // stride -- must fit, else the generic table-driven kernels run
            const long ring = static_cast<long>(pw_ / cfg_.block + 2 * plan_.ghost) *
                              (ph_ / cfg_.block + 2 * plan_.ghost) * plan_.max_epad * plan_.nslots;
            if (ring >= 0x7fffffffL) plan_ = compile_swept_plan(cfg_.block, eq, m, final_level_, 1);
        }
        for (const Launch& l : plan_.launches)
            cell_updates_ += static_cast<long long>(plan_.updates_per_kind[l.kind]) *
                             (setup_.nx / cfg_.block) * (setup_.ny / cfg_.block);
        build_swept();
        if (!dist()) finalize_swept();
    } else {
        actual_steps_ = cfg_.steps;
        total_levels_ = cfg_.steps * eq.substeps;
        final_level_ = total_levels_;
        cell_updates_ = total_levels_ * static_cast<long long>(setup_.nx) * setup_.ny;
        build_standard();
        if (!dist()) finalize_standard();
    }
    for (auto& d : devs_) {
        ck(cudaSetDevice(d.dev), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "setup sync");
    }
    if (const char* v = std::getenv("SG_NO_GRAPH"); v && v[0] == '1') use_graph_ = false;
    setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

Solver::~Solver() {
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    for (double* h : drain_.host) cudaFreeHost(h);
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        if (d.copy) {
            cudaStreamSynchronize(d.copy);
            cudaStreamDestroy(d.copy);
        }
        if (d.ev_ready) cudaEventDestroy(d.ev_ready);
        for (auto e : d.ev_copied) cudaEventDestroy(e);
    }
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        cudaStreamSynchronize(d.stream);
        for (void* p : d.allocs) cudaFree(p);
        for (void* p : ipc_open_) cudaIpcCloseMemHandle(p);
        ipc_open_.clear();
        for (auto e : d.prof_ev) cudaEventDestroy(e);
        for (auto e : d.launch_ev) cudaEventDestroy(e);
        if (d.side) cudaStreamDestroy(d.side);
        cudaEventDestroy(d.ev_start);
        cudaEventDestroy(d.ev_stop);
        cudaEventDestroy(d.ev_sync);
        cudaStreamDestroy(d.stream);
    }
}

void Solver::build_swept() {
    const SweptPlan& P = plan_;
    const int nv = setup_.eq.nvars;
    const int b = cfg_.block;
    const int pbx = pw_ / b, pby = ph_ / b;
    const int g = P.ghost, extw = pbx + 2 * g, exth = pby + 2 * g;
    const std::size_t rec_len = static_cast<std::size_t>(extw) * exth * nv * P.max_epad;
    rec_len_ = rec_len;
    const std::size_t plane = static_cast<std::size_t>(pw_) * ph_;

    // one instance's phase must fit on chip (levels + Euler flux scratch)
    int inst_smem = 0;
    for (int kd = 0; kd < K_NKINDS; ++kd) inst_smem = std::max(inst_smem, P.kinds[kd].smem_doubles * 8);
    // phases that do not fit on chip (heat b > 48, Euler b > 32) keep their
    // level storage in HBM (the GM kernels, kernels.cu); allocated in finalize
    // Euler: also when fewer than 3 instances would fit an SM's shared memory
    // -- the GM kernels then run 4 CTAs per SM with the levels in L1/L2 and
    // win (960^2: b32 1.03e10 vs 6.8e9 in shared memory; b24 0.98e10 vs 1.01e10)
    // Heat: when fewer than 2 instances fit (4160^2 b52: 1.21e11 in GM mode vs
    // 6.7e10 in shared memory; b40 1.15e11 vs 1.18e11)
    gm_phases_ = inst_smem > 220 * 1024 || (setup_.eq.problem != SG_HEAT && inst_smem > 76 * 1024) ||
                 (setup_.eq.problem == SG_HEAT && inst_smem > 114 * 1024) || std::getenv("SG_FORCE_GM");

    if (!snap_path_.empty()) {
        // level l is complete after the last launch computing it; frames are
        // drained right then, so the ring needs the widest window of levels
        // that are touched but not yet complete
        const long flat = P.flat;
        std::vector<long> last(flat + 1, -1);
        for (std::size_t i = 0; i < P.launches.size(); ++i)
            for (long l = P.launches[i].lo; l <= P.launches[i].hi; ++l) last[l] = static_cast<long>(i);
        done_after_.assign(P.launches.size(), {});
        for (long l = 1; l <= flat; ++l) done_after_[last[l]].push_back(l);
        long lowest = 1, highest = 0, width = 1;
        for (std::size_t i = 0; i < P.launches.size(); ++i) {
            highest = std::max(highest, P.launches[i].hi);
            width = std::max(width, highest - lowest + 1);
            for (long l : done_after_[i]) lowest = std::max(lowest, l + 1);
        }
        // + spare slots: a completed frame's D2H (copy stream) overlaps the
        // next launches instead of blocking the first one that reuses its slot
        frame_ring_ = static_cast<int>(width) + (dist() ? 0 : 2);
    }
    for (auto& pb : parts_) {
        if (pb.dev < 0) continue;
        DeviceCtx& d = devs_[pb.dev];
        if (frame_ring_ > 0) pb.frames = dev_alloc<double>(d, static_cast<std::size_t>(frame_ring_) * plane * nv);
        pb.init = dev_alloc<double>(d, plane * nv);
        pb.out = dev_alloc<double>(d, plane * nv);
        // one allocation per partition, slot s at s * rec_len (the column
        // kernels address every producer record from the instance's slot-0 base)
        pb.rec.resize(P.nslots);
        double* all = dev_alloc<double>(d, std::max<std::size_t>(rec_len * P.nslots, 1));
        for (int s = 0; s < P.nslots; ++s) pb.rec[s] = all + rec_len * s;
        // level-0 piece of this partition (engine.cpp:199-209 load_initial)
        std::vector<double> piece(plane * nv);
        for (int v = 0; v < nv; ++v)
            for (int y = 0; y < ph_; ++y)
                std::memcpy(&piece[(static_cast<std::size_t>(v) * ph_ + y) * pw_],
                            &setup_.initial[(static_cast<std::size_t>(v) * setup_.ny + pb.pj * ph_ + y) * setup_.nx +
                                            pb.pi * pw_],
                            sizeof(double) * pw_);
        ck(cudaMemcpy(pb.init, piece.data(), piece.size() * sizeof(double), cudaMemcpyHostToDevice), "init H2D");
    }
    // ledger: record pushes across partition boundaries (P2P / NVLink stores),
    // per partition: the instances whose record lands in another partition's
    // ghost ring, and the distinct partitions one launch pushes into
    part_messages_.assign(nparts_, 0);
    part_bytes_.assign(nparts_, 0);
    for (const auto& pb : parts_) {
        long pushes = 0;
        std::vector<char> peer(nparts_, 0);
        for (int bj = 0; bj < pby; ++bj)
            for (int bi = 0; bi < pbx; ++bi)
                for (int ej = -1; ej <= 1; ++ej)
                    for (int ei = -1; ei <= 1; ++ei) {
                        if (!ei && !ej) continue;
                        const int tbi = bi - ei * pbx, tbj = bj - ej * pby;
                        if (tbi < -g || tbi >= pbx + g || tbj < -g || tbj >= pby + g) continue;
                        const int tp = ((pb.pj + ej + py_) % py_) * px_ + (pb.pi + ei + px_) % px_;
                        if (tp != pb.id) {
                            ++pushes;
                            peer[tp] = 1;
                        }
                    }
        long npeers = 0;
        for (char c : peer) npeers += c;
        for (const Launch& l : P.launches) {
            if (P.kinds[l.kind].epad == 0) continue;
            part_bytes_[pb.id] += static_cast<long long>(pushes) * P.kinds[l.kind].exp_cells.size() * nv * 8;
            part_messages_[pb.id] += npeers;
        }
    }
    for (int q = 0; q < nparts_; ++q) {
        bytes_ += part_bytes_[q];
        messages_ += part_messages_[q];
    }
}

void Solver::finalize_swept() {
    const SweptPlan& P = plan_;
    const int b = cfg_.block;
    const int pbx = pw_ / b, pby = ph_ / b;
    const int g = P.ghost, extw = pbx + 2 * g;
    for (auto& d : devs_) {
        ck(cudaSetDevice(d.dev), "cudaSetDevice");
        for (int kd = 0; kd < K_NKINDS; ++kd) {
            const KindLayout& K = P.kinds[kd];
            if (K.nlev > kMaxLevels - 2) fail(SG_EINVAL, "swept: too many levels per phase");
            std::vector<DevLevel> lv;
            for (const PlanLevel& pl : K.lev)
                lv.push_back({pl.bbox.x0, pl.bbox.y0, pl.pitch, pl.bbox.h(), pl.off, pl.vstride, pl.comp.x0,
                              pl.comp.x1, pl.comp.y0, pl.comp.y1});
            d.d_lev[kd] = dev_upload(d, lv);
            d.d_exp_off[kd] = dev_upload(d, K.exp_off);
            d.d_exp_vs[kd] = dev_upload(d, K.exp_vstride);
            std::vector<int2> ep;
            for (const auto& e : K.exp_pairs) ep.push_back(make_int2(e[0], e[1]));
            d.d_exp_pairs[kd] = dev_upload(d, ep);
            std::vector<int4> ln;
            std::vector<int2> pt;
            for (const auto& e : K.lanes) ln.push_back(make_int4(e[0], e[1], e[2], e[3]));
            for (const auto& e : K.pitch) pt.push_back(make_int2(e[0], e[1]));
            d.d_lanes[kd] = dev_upload(d, ln);
            d.d_pitch[kd] = dev_upload(d, pt);
        }
        for (const ClassTab& T : P.classes) {
            std::vector<int4> im, in;
            std::vector<int2> im2;
            for (const Import& x : T.imports) {
                if (x.src >= (1 << 20) || x.seg >= (1 << 11)) fail(SG_ELOGIC, "swept: import table overflow");
                im.push_back(make_int4(x.seg, x.src, x.dst, x.vstride));
                im2.push_back(make_int2((x.seg << 20) | x.src, x.dst));
            }
            d.d_imp2.push_back(dev_upload(d, im2));
            for (const InitImport& x : T.inits) in.push_back(make_int4(x.rx, x.ry, x.dst, x.vstride));
            d.d_imp.push_back(dev_upload(d, im));
            d.d_init.push_back(dev_upload(d, in));
        }
        // b24 / b32: the Octahedron runs as two launches (levels 1..k, k+1..2k) so
        // each kernel's straight-line code is half as long (instruction
        // fetch bound it); the level-k state goes through HBM
        if (gm_phases_ && !d.parts.empty()) {
            // per-CTA (Euler: level planes + pressure / flux scratch) or per-warp
            // (heat, 4 warps per CTA) storage for a persistent grid of <= 4
            // CTAs per SM, capped at ~8 GB
            const bool heat = setup_.eq.problem == SG_HEAT;
            long per = 0;
            for (int kd = 0; kd < K_NKINDS; ++kd) {
                const KindLayout& K = P.kinds[kd];
                long need = K.smem_doubles;
                if (!heat) {
                    long ps = 1, fx = 1;
                    for (int r = 1; r <= K.nlev; ++r) {
                        const Rect c = K.at(r).comp;
                        ps = std::max<long>(ps, (c.w() + 4) * (c.h() + 4));
                        fx = std::max<long>(fx, 4L * std::max(c.h() * (c.w() + 1), (c.h() + 1) * c.w()));
                    }
                    need += ((ps + 1) & ~1L) + 2 * ((fx + 1) & ~1L);
                }
                per = std::max(per, need);
            }
            d.gm_stride = (per + 31) / 32 * 32;
            const long slots_per_cta = heat ? 4 : 1;
            const long ninst = static_cast<long>(pbx) * pby;
            long ctas = std::min<long>((ninst + slots_per_cta - 1) / slots_per_cta, 148L * 4);
            const long cap = (8L << 30) / (8L * d.gm_stride * slots_per_cta * static_cast<long>(d.parts.size()));
            ctas = std::max<long>(1, std::min(ctas, cap));
            d.gm_ctas = static_cast<int>(ctas);
            d.gm_scratch = dev_alloc<double>(d, static_cast<std::size_t>(ctas * slots_per_cta * d.gm_stride) *
                                                    d.parts.size());
        }
        if (P.colB >= 24 && !std::getenv("SG_NO_OCT_SPLIT") && !d.parts.empty())
            d.oct_scratch =
                dev_alloc<double>(d, d.parts.size() * static_cast<std::size_t>(pbx) * pby * P.colB * P.colB);
        std::vector<double*> rt(static_cast<std::size_t>(nparts_) * P.nslots);
        std::vector<const double*> it(nparts_);
        std::vector<double*> ot(nparts_);
        for (const auto& pb : parts_) {
            for (int s = 0; s < P.nslots; ++s) rt[pb.id * P.nslots + s] = pb.rec[s];
            it[pb.id] = pb.init;
            ot[pb.id] = pb.out;
        }
        d.d_rec_tab = dev_upload(d, rt);
        d.d_init_tab = dev_upload(d, it);
        d.d_out_tab = dev_upload(d, ot);
        std::vector<double*> ft(nparts_, nullptr);
        for (const auto& pb : parts_) ft[pb.id] = pb.frames;
        d.d_frames_tab = dev_upload(d, ft);

        for (std::size_t li = 0; li < P.launches.size(); ++li) {
            const Launch& L = P.launches[li];
            const KindLayout& K = P.kinds[L.kind];
            const ClassTab& T = P.classes[L.cls];
            SweptArgs a;
            std::memset(&a, 0, sizeof a);
            a.nlev = K.nlev;
            a.rmin = K.rmin;
            a.smem_doubles = K.smem_doubles;
            a.nexp = static_cast<int>(K.exp_cells.size());
            a.split = K.split;
            {
                int ps = 0, fx = 0;
                for (int kd = 0; kd < K_NKINDS; ++kd)
                    for (int r = 1; r <= P.kinds[kd].nlev; ++r) {
                        const Rect c = P.kinds[kd].at(r).comp;
                        ps = std::max(ps, (c.w() + 4) * (c.h() + 4));
                        fx = std::max(fx, 4 * std::max(c.h() * (c.w() + 1), (c.h() + 1) * c.w()));
                    }
                a.ps_doubles = (ps + 1) & ~1;
                a.fx_doubles = (fx + 1) & ~1;
            }
            a.nexp_early = K.nexp_early;
            a.epad = P.max_epad;  // uniform record stride per instance (all kinds)
            a.lev = d.d_lev[L.kind];
            a.exp_off = d.d_exp_off[L.kind];
            a.exp_vs = d.d_exp_vs[L.kind];
            a.exp_pairs = d.d_exp_pairs[L.kind];
            a.lanes = d.d_lanes[L.kind];
            a.pitch = d.d_pitch[L.kind];
            a.imports = d.d_imp[L.cls];
            a.imports2 = d.d_imp2[L.cls];
            if (P.colB) {
                // imports as signed offsets from the consumer instance's slot-0
                // record base: producer slot * rec_len + (dj*extw + di)*stride + src
                const int rot = static_cast<int>(li % P.nslots);
                auto key = std::make_pair(L.cls, rot);
                auto it = d.imp_off.find(key);
                if (it == d.imp_off.end()) {
                    std::vector<int2> tab;
                    for (const Import& x : T.imports) {
                        const Segment& sg = T.segs[x.seg];
                        const long pslot = ((static_cast<long>(li) - sg.delta) % P.nslots + P.nslots) % P.nslots;
                        const long off = pslot * static_cast<long>(rec_len_) +
                                         (static_cast<long>(sg.dj) * extw + sg.di) * P.max_epad + x.src;
                        if (off > INT32_MAX || off < INT32_MIN) fail(SG_ELOGIC, "swept: record offset overflow");
                        tab.push_back(make_int2(static_cast<int>(off), x.dst));
                    }
                    std::vector<int>& th = d.imp_off_host[key];
                    for (const int2& e : tab) th.push_back(e.x);
                    it = d.imp_off.emplace(key, dev_upload(d, tab)).first;
                }
                a.imp_off = it->second;
                // steady classes: every import slot [0, imp_total) is filled by
                // exactly one import (no initial-plane cells) -> a table
                // indexed by slot, so the kernel's shared-memory addresses are
                // compile-time (colkernel.cuh, dense gather)
                auto jt = d.imp_dense.find(key);
                if (jt == d.imp_dense.end()) {
                    int* dt = nullptr;
                    const int ntot = col::imp_total(L.kind, P.colB);
                    const int split = col::gather_split(L.kind, P.colB);
                    const int na = col::imp_base(L.kind, P.colB, split + 1, col::ylo(L.kind, P.colB));
                    if (T.inits.empty() && static_cast<int>(T.imports.size()) == ntot) {
                        std::vector<int> tab(static_cast<std::size_t>(ntot), INT32_MIN);
                        bool ok = true;
                        for (std::size_t q = 0; q < T.imports.size(); ++q) {
                            const Import& x = T.imports[q];
                            if (x.dst < 0 || x.dst >= ntot || tab[x.dst] != INT32_MIN ||
                                (x.dst < na) != (x.r + 1 <= split)) {
                                ok = false;
                                break;
                            }
                            tab[x.dst] = d.imp_off_host[key][q];
                        }
                        if (ok) dt = dev_upload(d, tab);
                    }
                    jt = d.imp_dense.emplace(key, dt).first;
                }
                a.imp_dense = jt->second;
                a.dense = jt->second != nullptr && !std::getenv("SG_NO_DENSE") ? 1 : 0;
            }
            a.nimp = static_cast<int>(T.imports.size());
            a.nimp_b = T.nimp_b;
            a.oct_scratch = d.oct_scratch;
            a.gm_scratch = d.gm_scratch;
            a.gm_stride = d.gm_stride;
            a.gm_ctas = d.gm_ctas;
            a.lo_parity = std::getenv("SG_NO_SERPENTINE") ? 0 : static_cast<int>(li & 1);
            a.inits = d.d_init[L.cls];
            a.ninit = static_cast<int>(T.inits.size());
            if (T.segs.size() > static_cast<std::size_t>(kMaxSegs)) fail(SG_ELOGIC, "swept: too many segments");
            for (std::size_t s = 0; s < T.segs.size(); ++s) {
                const long pl = static_cast<long>(li) - T.segs[s].delta;
                if (pl < 0 || P.launches[pl].slot < 0) fail(SG_ELOGIC, "swept: import from a launch without record");
                a.segs[s] = {P.launches[pl].slot, T.segs[s].di, T.segs[s].dj, P.max_epad};
            }
            a.nsegs = static_cast<int>(T.segs.size());
            a.frame = L.frame;
            a.stage0 = L.stage0;
            a.r_out = L.r_out;
            a.my_slot = L.slot < 0 ? 0 : L.slot;
            a.kind = L.kind;
            a.colB = P.colB;
            a.b = b;
            a.nx = setup_.nx;
            a.ny = setup_.ny;
            a.pw = pw_;
            a.ph = ph_;
            a.pbx = pbx;
            a.pby = pby;
            a.px = px_;
            a.py = py_;
            a.ghost = g;
            a.extw = extw;
            a.nslots = P.nslots;
            a.ndev_parts = static_cast<int>(d.parts.size());
            for (std::size_t q = 0; q < d.parts.size(); ++q) {
                a.dev_parts[q] = d.parts[q];
                a.dev_pij[q] = (d.parts[q] % px_) | ((d.parts[q] / px_) << 16);
            }
            a.rec = d.d_rec_tab;
            a.init_planes = d.d_init_tab;
            a.out_planes = d.d_out_tab;
            if (setup_.eq.problem == SG_HEAT) {
                a.c0 = setup_.heat_fx;
                a.c1 = setup_.heat_fy;
            } else {
                a.c0 = setup_.gamma;
                a.c1 = setup_.cx_pred;
                a.c2 = setup_.cy_pred;
                a.c3 = setup_.cx_corr;
                a.c4 = setup_.cy_corr;
            }
            a.err = d.d_err;
            a.frames = d.d_frames_tab;
            a.snap_every = frame_ring_ > 0 ? static_cast<int>(snap_every_) : 0;
            a.frame_ring = std::max(1, frame_ring_);
            a.lo = L.lo;
            a.out_mask = L.r_out > 0 ? 1ull << L.r_out : 0ull;
            a.snap_mask = 0;
            if (a.snap_every > 0)
                for (int r = 1; r <= K.nlev; ++r)
                    if ((L.lo + r - 1) % a.snap_every == 0) a.snap_mask |= 1ull << r;
            for (int r = 1; r <= K.nlev; ++r) {  // heat lane map: (column, row-chunk) items of a warp
                const PlanLevel& Lc = K.at(r);
                const PlanLevel& Lp = K.at(r - 1);
                const int w = Lc.comp.w(), h = Lc.comp.h();
                int splits, rps;
                lane_split(w, h, &splits, &rps);
                HeatLevel hl;
                hl.cx0 = Lc.comp.x0;
                hl.cy0 = Lc.comp.y0;
                hl.cy1 = Lc.comp.y1;
                hl.w = w;
                hl.items = w <= 32 ? w * splits : 0;
                hl.rps = rps;
                hl.poff = Lp.off - Lp.bbox.y0 * Lp.pitch - Lp.bbox.x0;
                hl.pbw = Lp.pitch;
                hl.doff = Lc.off - Lc.bbox.y0 * Lc.pitch - Lc.bbox.x0;
                hl.cbw = Lc.pitch;
                hl.inv_w = w > 0 ? 1.0f / static_cast<float>(w) : 0.0f;
                hl.pad = 0;
                a.hl[r - 1] = hl;
            }
            d.swept_args.push_back(a);
        }
    }
    prof_kind_ = P.m > 0 ? K_OCT : K_UP;
}

void Solver::build_standard() {
    const Equation& eq = setup_.eq;
    const int n = eq.halo, nv = eq.nvars, S = eq.substeps;
    const int pitch = pw_ + 2 * n, rows = ph_ + 2 * n;
    const std::size_t gplane = static_cast<std::size_t>(pitch) * rows;
    for (auto& pb : parts_) {
        if (pb.dev < 0) continue;
        DeviceCtx& d = devs_[pb.dev];
        pb.ring.resize(S + 1);
        for (int s = 0; s <= S; ++s) pb.ring[s] = dev_alloc<double>(d, gplane * nv);
        pb.init_ghosted = dev_alloc<double>(d, gplane * nv);
        // ghosted level-0 piece, ghosts from the periodic neighbours (cross only)
        std::vector<double> piece(gplane * nv, 0.0);
        for (int v = 0; v < nv; ++v)
            for (int y = -n; y < ph_ + n; ++y)
                for (int x = -n; x < pw_ + n; ++x) {
                    const bool inx = x >= 0 && x < pw_, iny = y >= 0 && y < ph_;
                    if (!inx && !iny) continue;  // corners are never read
                    const int gx = ((pb.pi * pw_ + x) % setup_.nx + setup_.nx) % setup_.nx;
                    const int gy = ((pb.pj * ph_ + y) % setup_.ny + setup_.ny) % setup_.ny;
                    piece[(static_cast<std::size_t>(v) * rows + (y + n)) * pitch + (x + n)] =
                        setup_.initial[(static_cast<std::size_t>(v) * setup_.ny + gy) * setup_.nx + gx];
                }
        ck(cudaMemcpy(pb.init_ghosted, piece.data(), piece.size() * sizeof(double), cudaMemcpyHostToDevice),
           "init H2D");
    }
    // ledger: per level, each partition pushes its n-wide face strips into
    // the face neighbours that are other partitions
    part_messages_.assign(nparts_, 0);
    part_bytes_.assign(nparts_, 0);
    for (int q = 0; q < nparts_; ++q) {
        if (px_ > 1) {
            part_messages_[q] += 2 * final_level_;
            part_bytes_[q] += 2LL * ph_ * n * nv * 8 * final_level_;
        }
        if (py_ > 1) {
            part_messages_[q] += 2 * final_level_;
            part_bytes_[q] += 2LL * pw_ * n * nv * 8 * final_level_;
        }
        messages_ += part_messages_[q];
        bytes_ += part_bytes_[q];
    }
    prof_kind_ = 100;  // std step
}

void Solver::finalize_standard() {
    const int S = setup_.eq.substeps;
    for (auto& d : devs_) {
        ck(cudaSetDevice(d.dev), "cudaSetDevice");
        for (int phase = 0; phase <= S; ++phase) {
            // level L with L % (S+1) == phase
            std::vector<const double*> r1(nparts_), r2(nparts_);
            std::vector<double*> o(nparts_);
            for (const auto& pb : parts_) {
                r1[pb.id] = pb.ring[(phase + S) % (S + 1)];
                r2[pb.id] = pb.ring[(phase + S - 1 + (S + 1)) % (S + 1)];
                o[pb.id] = pb.ring[phase];
            }
            d.d_std_r1.push_back(dev_upload(d, r1));
            d.d_std_r2.push_back(dev_upload(d, r2));
            d.d_std_out.push_back(dev_upload(d, o));
        }
    }
}

void Solver::reset() {
    for (auto& d : devs_) {
        ck(cudaSetDevice(d.dev), "cudaSetDevice");
        ck(cudaMemsetAsync(d.d_err, 0, sizeof(int), d.stream), "memset");
    }
    if (cfg_.engine == SG_STANDARD) {
        const Equation& eq = setup_.eq;
        const std::size_t gplane =
            static_cast<std::size_t>(pw_ + 2 * eq.halo) * (ph_ + 2 * eq.halo) * eq.nvars;
        for (auto& pb : parts_) {
            if (pb.dev < 0) continue;
            DeviceCtx& d = devs_[pb.dev];
            ck(cudaSetDevice(d.dev), "cudaSetDevice");
            ck(cudaMemcpyAsync(pb.ring[0], pb.init_ghosted, gplane * sizeof(double), cudaMemcpyDeviceToDevice,
                               d.stream),
               "reset");
        }
    }
}

double Solver::solve() {
    const bool multi = devs_.size() > 1;
    const int prob = setup_.eq.problem;
    launches_ = 0;
    prof_seconds_ = 0.0;
    prof_launches_ = 0;
    prof_bytes_ = 0.0;
    prof_updates_ = 0.0;
    DeviceCtx& d0 = devs_[0];
    std::size_t prof_i = 0;
    auto prof_begin = [&](bool on) -> cudaEvent_t {
        if (!on) return nullptr;
        if (prof_i + 2 > d0.prof_ev.size()) {
            cudaEvent_t a, c;
            cudaSetDevice(d0.dev);
            ck(cudaEventCreate(&a), "event");
            ck(cudaEventCreate(&c), "event");
            d0.prof_ev.push_back(a);
            d0.prof_ev.push_back(c);
        }
        cudaEvent_t e = d0.prof_ev[prof_i];
        ck(cudaEventRecord(e, d0.stream), "event");
        return e;
    };
    auto prof_end = [&](bool on) {
        if (!on) return;
        ck(cudaEventRecord(d0.prof_ev[prof_i + 1], d0.stream), "event");
        prof_i += 2;
    };
    // barrier between dependent launches on different GPUs
    if (dist() && !connected_) fail(SG_ETRANSPORT, "distributed solver used before connect()");
    auto cross_sync = [&]() {
        if (dist()) {
            dist_barrier(devs_[0]);
            return;
        }
        if (!multi) return;
        for (auto& d : devs_) {
            cudaSetDevice(d.dev);
            ck(cudaEventRecord(d.ev_sync, d.stream), "event");
        }
        for (auto& d : devs_)
            for (auto& e : devs_)
                if (&d != &e) ck(cudaStreamWaitEvent(d.stream, e.ev_sync, 0), "wait");
    };
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        ck(cudaEventRecord(d.ev_start, d.stream), "event");
    }
    if (dist()) dist_barrier(devs_[0]);  // no rank starts writing into a peer still in its previous solve
    std::unique_ptr<SnapshotWriter> writer;
    const bool snap = !snap_path_.empty();
    if (snap && (!dist() || rank_ == 0)) {  // FrameSink, engine.cpp:75-117 of the reference
        SnapshotMeta m;
        m.problem = setup_.eq.problem == SG_HEAT ? "heat" : "euler";
        m.nx = setup_.nx;
        m.ny = setup_.ny;
        m.nvars = setup_.eq.nvars;
        m.block = cfg_.block;
        m.dt = setup_.dt;
        m.dx = setup_.dx;
        m.dy = setup_.dy;
        m.alpha = cfg_.heat_alpha;
        m.gamma = cfg_.gamma;
        writer = std::make_unique<SnapshotWriter>(snap_path_, m);
        writer->append_frame(0, setup_.initial.data());  // level 0 % every == 0
    }
    // Single device, no profiling / snapshots: an XBridge launch that does not
    // depend on the YBridge launched just before it (the XBridge reads only the
    // previous cycle's YBridge) runs on a second stream, so the
    // two bridges of a cycle overlap (their launch tails and gather ramps).
    // Cross-stream edges come from the plan: producer launches (segments),
    // earlier readers of the record slot a launch overwrites, and its previous
    // writer.
    const bool concurrent = cfg_.engine == SG_SWEPT && !multi && !dist() && !snap && !profile &&
                            !gm_phases_ &&  // (the GM kernels share one level-storage scratch)
                            !std::getenv("SG_SERIAL_BRIDGES");
    std::vector<int> on_side;
    if (concurrent) {
        DeviceCtx& d = d0;
        if (!d.side) ck(cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking), "stream");
        while (d.launch_ev.size() < plan_.launches.size()) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            d.launch_ev.push_back(e);
        }
        on_side.assign(plan_.launches.size(), 0);
    }
    auto deps_of = [&](std::size_t li) {
        std::vector<long> deps;
        const long n = plan_.nslots;
        const long L = static_cast<long>(li);
        for (const Segment& sg : plan_.classes[plan_.launches[li].cls].segs) deps.push_back(L - sg.delta);
        if (plan_.launches[li].slot >= 0) {
            deps.push_back(L - n);  // previous writer of this slot
            for (long q = std::max(0L, L - n + 1); q < L; ++q)  // its readers
                for (const Segment& sg : plan_.classes[plan_.launches[q].cls].segs)
                    if (q - sg.delta == L - n) deps.push_back(q);
        }
        return deps;
    };
    // snapshot levels: one process -> overlapped drain (D2H on the copy
    // streams, launches that reuse a frame slot wait for its copy); one
    // process per GPU -> rank 0 gathers every partition's frame through the
    // IPC-mapped buffers after the launch barrier, then all ranks pass one
    // more barrier so no peer overwrites a frame slot still being read
    auto snap_before = [&](long lo, long hi, int ring) {
        if (!snap || dist()) return;
        for (long l = lo; l <= hi; ++l)
            if (l % snap_every_ == 0) drain_wait_slot(static_cast<int>(l % ring));
    };
    auto snap_after = [&](const std::vector<long>& done, int ring) {
        if (!snap) return;
        bool any = false;
        for (long l : done)
            if (l % snap_every_ == 0) {
                any = true;
                if (!dist()) drain_start(*writer, l, static_cast<int>(l % ring));
                else if (writer) snapshot_frame(*writer, l, static_cast<int>(l % ring));
            }
        if (any && dist()) dist_barrier(devs_[0]);
    };
    auto enqueue = [&]() {
        if (cfg_.engine == SG_SWEPT) {
            cudaEvent_t fork = nullptr;
            if (concurrent) {  // bring the side stream into the capture / stream order
                fork = d0.launch_ev[0];
                ck(cudaEventRecord(fork, d0.stream), "event");
                ck(cudaStreamWaitEvent(d0.side, fork, 0), "wait");
            }
            long last_side = -1;
            for (std::size_t li = 0; li < plan_.launches.size(); ++li) {
                const bool pr = profile && plan_.launches[li].kind == prof_kind_;
                if (concurrent) {
                    const std::vector<long> deps = deps_of(li);
                    const bool side = li > 0 && plan_.launches[li].kind == K_XB &&
                                      plan_.launches[li - 1].kind == K_YB &&
                                      std::find(deps.begin(), deps.end(), static_cast<long>(li) - 1) == deps.end();
                    on_side[li] = side;
                    cudaStream_t st = side ? d0.side : d0.stream;
                    for (long q : deps)
                        if (q >= 0 && on_side[q] != static_cast<int>(side)) ck(cudaStreamWaitEvent(st, d0.launch_ev[q], 0), "wait");
                    ck(launch_swept(prob, d0.swept_args[li], st), "swept launch");
                    ck(cudaEventRecord(d0.launch_ev[li], st), "event");
                    ++launches_;
                    if (side) last_side = static_cast<long>(li);
                    continue;
                }
                snap_before(plan_.launches[li].lo, plan_.launches[li].hi, frame_ring_);
                for (auto& d : devs_) {
                    if (multi) cudaSetDevice(d.dev);
                    if (&d == &d0) prof_begin(pr);
                    ck(launch_swept(prob, d.swept_args[li], d.stream), "swept launch");
                    if (&d == &d0) prof_end(pr);
                    ++launches_;
                }
                if (pr) {
                    ++prof_launches_;
                    const Launch& L = plan_.launches[li];
                    const ClassTab& T = plan_.classes[L.cls];
                    const double inst = static_cast<double>(pw_ / cfg_.block) * (ph_ / cfg_.block) *
                                        devs_[0].parts.size();
                    prof_bytes_ += inst * (T.imports.size() + T.inits.size() + plan_.kinds[L.kind].exp_cells.size()) *
                                   setup_.eq.nvars * 8.0;
                    prof_updates_ += inst * plan_.updates_per_kind[L.kind];
                }
                cross_sync();
                if (snap) snap_after(done_after_[li], frame_ring_);
            }
            if (concurrent) {  // join: the main stream waits for the side stream's last launch
                if (last_side >= 0) ck(cudaStreamWaitEvent(d0.stream, d0.launch_ev[last_side], 0), "wait");
                else {
                    ck(cudaEventRecord(fork, d0.side), "event");
                    ck(cudaStreamWaitEvent(d0.stream, fork, 0), "wait");
                }
            }
        } else {
            const Equation& eq = setup_.eq;
            const int S = eq.substeps;
            for (long l = 1; l <= final_level_; ++l) {
                const int phase = static_cast<int>(l % (S + 1));
                const int stage = static_cast<int>((l - 1) % S);
                const bool pr = profile;
                snap_before(l, l, S + 1);
                for (auto& d : devs_) {
                    if (multi) cudaSetDevice(d.dev);
                    StdArgs a;
                    std::memset(&a, 0, sizeof a);
                    a.nvars = eq.nvars;
                    a.n = eq.halo;
                    a.pw = pw_;
                    a.ph = ph_;
                    a.px = px_;
                    a.py = py_;
                    a.pitch = pw_ + 2 * eq.halo;
                    a.rows = ph_ + 2 * eq.halo;
                    a.stage = stage;
                    a.ndev_parts = static_cast<int>(d.parts.size());
                    for (std::size_t q = 0; q < d.parts.size(); ++q) a.dev_parts[q] = d.parts[q];
                    a.read1 = d.d_std_r1[phase];
                    a.read2 = l >= 2 ? d.d_std_r2[phase] : d.d_std_r1[phase];
                    a.out = d.d_std_out[phase];
                    if (eq.problem == SG_HEAT) {
                        a.c0 = setup_.heat_fx;
                        a.c1 = setup_.heat_fy;
                    } else {
                        a.c0 = setup_.gamma;
                        a.c1 = stage == 0 ? setup_.cx_pred : setup_.cx_corr;
                        a.c2 = stage == 0 ? setup_.cy_pred : setup_.cy_corr;
                    }
                    a.err = d.d_err;
                    if (&d == &d0) prof_begin(pr);
                    ck(launch_std(eq.problem, a, d.stream), "std launch");
                    if (&d == &d0) prof_end(pr);
                    ++launches_;
                }
                if (pr) {
                    ++prof_launches_;
                    const double cells = static_cast<double>(pw_) * ph_ * devs_[0].parts.size();
                    // heat: read 8 + write 8; euler: predictor 64, corrector 96
                    const double bpu = eq.problem == SG_HEAT ? 16.0 : (stage == 0 ? 64.0 : 96.0);
                    prof_bytes_ += cells * bpu;
                    prof_updates_ += cells;
                }
                cross_sync();
                if (snap) snap_after({l}, S + 1);
            }
        }
    };
    // Solves on one device per process without snapshots/profiling are
    // replayed from a CUDA graph captured on the first solve: every launch of
    // the solve (up to ~4300 phase launches at 10k steps, twice that with the
    // barriers of one process per GPU) goes to the GPU in one call.
    const bool graphable = !multi && !snap && !profile && use_graph_;
    if (graphable) {
        DeviceCtx& d = devs_[0];
        if (!graph_exec_) {
            cudaGraph_t g = nullptr;
            ck(cudaStreamBeginCapture(d.stream, cudaStreamCaptureModeThreadLocal), "capture");
            enqueue();
            ck(cudaStreamEndCapture(d.stream, &g), "capture");
            ck(cudaGraphInstantiate(&graph_exec_, g, 0), "graph instantiate");
            cudaGraphDestroy(g);
            graph_launches_ = launches_;
        }
        launches_ = graph_launches_;
        ck(cudaGraphLaunch(graph_exec_, d.stream), "graph launch");
    } else {
        enqueue();
    }
    double worst = 0.0;
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        ck(cudaEventRecord(d.ev_stop, d.stream), "event");
    }
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        ck(cudaEventSynchronize(d.ev_stop), "solve");
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, d.ev_start, d.ev_stop), "elapsed");
        worst = std::max(worst, ms * 1e-3);
    }
    for (std::size_t i = 0; i + 1 < prof_i; i += 2) {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, d0.prof_ev[i], d0.prof_ev[i + 1]), "elapsed");
        prof_seconds_ += ms * 1e-3;
    }
    last_solve_ = worst;
    if (writer) {
        while (!drain_.queue.empty()) drain_pop(*writer);
        writer->flush();
        snapshot_frames_ = writer->frames();
    }
    check_error();
    return worst;
}

void Solver::snapshot_frame(SnapshotWriter& w, long level, int slot) {
    // gather one complete level from every partition (FrameCollector,
    // snapshot.cpp:122-153) and append it
    const Equation& eq = setup_.eq;
    const int nv = eq.nvars;
    const std::size_t nx = setup_.nx, ny = setup_.ny, plane = static_cast<std::size_t>(pw_) * ph_;
    std::vector<double> full(nv * nx * ny), piece;
    for (auto& pb : parts_) {
        if (pb.dev < 0 && !dist()) continue;
        DeviceCtx& d = devs_[pb.dev < 0 ? 0 : pb.dev];  // remote partitions: IPC-mapped buffers
        cudaSetDevice(d.dev);
        ck(cudaStreamSynchronize(d.stream), "snapshot sync");
        if (cfg_.engine == SG_SWEPT) {
            piece.resize(plane * nv);
            ck(cudaMemcpy(piece.data(), pb.frames + static_cast<std::size_t>(slot) * plane * nv,
                          piece.size() * sizeof(double), cudaMemcpyDeviceToHost),
               "snapshot D2H");
            for (int v = 0; v < nv; ++v)
                for (int y = 0; y < ph_; ++y)
                    std::memcpy(&full[(v * ny + pb.pj * ph_ + y) * nx + pb.pi * pw_],
                                &piece[(static_cast<std::size_t>(v) * ph_ + y) * pw_], sizeof(double) * pw_);
        } else {
            const int n = eq.halo, pitch = pw_ + 2 * n, rows = ph_ + 2 * n;
            piece.resize(static_cast<std::size_t>(pitch) * rows * nv);
            ck(cudaMemcpy(piece.data(), pb.ring[slot], piece.size() * sizeof(double), cudaMemcpyDeviceToHost),
               "snapshot D2H");
            for (int v = 0; v < nv; ++v)
                for (int y = 0; y < ph_; ++y)
                    std::memcpy(&full[(v * ny + pb.pj * ph_ + y) * nx + pb.pi * pw_],
                                &piece[(static_cast<std::size_t>(v) * rows + y + n) * pitch + n], sizeof(double) * pw_);
        }
    }
    w.append_frame(level, full.data());
}

int Solver::nslots_frames() const {
    return cfg_.engine == SG_SWEPT ? frame_ring_ : setup_.eq.substeps + 1;
}

void Solver::drain_start(SnapshotWriter& w, long level, int slot) {
    FrameDrain& D = drain_;
    const Equation& eq = setup_.eq;
    const int nv = eq.nvars;
    const std::size_t nx = setup_.nx, ny = setup_.ny, plane = static_cast<std::size_t>(pw_) * ph_;
    if (D.host.empty()) {
        const std::size_t bytes = sizeof(double) * nv * nx * ny;
        const int K = bytes <= (512ull << 20) ? 3 : bytes <= (2048ull << 20) ? 2 : 1;
        D.host.assign(K, nullptr);
        for (auto& h : D.host) ck(cudaMallocHost(&h, bytes), "cudaMallocHost");
        D.level.assign(K, -1);
        D.slot_host.assign(nslots_frames(), -1);
        for (auto& d : devs_) {
            ck(cudaSetDevice(d.dev), "cudaSetDevice");
            ck(cudaStreamCreateWithFlags(&d.copy, cudaStreamNonBlocking), "stream");
            ck(cudaEventCreateWithFlags(&d.ev_ready, cudaEventDisableTiming), "event");
            d.ev_copied.resize(K);
            for (auto& e : d.ev_copied) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        }
    }
    const int k = D.next;
    D.next = (k + 1) % static_cast<int>(D.host.size());
    while (D.level[k] >= 0) drain_pop(w);  // round robin: frame k is the oldest pending
    double* host = D.host[k];
    for (auto& d : devs_) {
        ck(cudaSetDevice(d.dev), "cudaSetDevice");
        ck(cudaEventRecord(d.ev_ready, d.stream), "event");
        ck(cudaStreamWaitEvent(d.copy, d.ev_ready, 0), "wait");
        for (int p : d.parts) {
            const PartBuffers& pb = parts_[p];
            for (int v = 0; v < nv; ++v) {
                double* dst = host + (static_cast<std::size_t>(v) * ny + static_cast<std::size_t>(pb.pj) * ph_) * nx +
                              static_cast<std::size_t>(pb.pi) * pw_;
                if (cfg_.engine == SG_SWEPT) {
                    const double* src = pb.frames + (static_cast<std::size_t>(slot) * nv + v) * plane;
                    ck(cudaMemcpy2DAsync(dst, nx * sizeof(double), src, pw_ * sizeof(double), pw_ * sizeof(double),
                                         ph_, cudaMemcpyDeviceToHost, d.copy),
                       "snapshot D2H");
                } else {
                    const int n = eq.halo, pitch = pw_ + 2 * n, rows = ph_ + 2 * n;
                    const double* src = pb.ring[slot] + static_cast<std::size_t>(v) * pitch * rows +
                                        static_cast<std::size_t>(n) * pitch + n;
                    ck(cudaMemcpy2DAsync(dst, nx * sizeof(double), src, pitch * sizeof(double), pw_ * sizeof(double),
                                         ph_, cudaMemcpyDeviceToHost, d.copy),
                       "snapshot D2H");
                }
            }
        }
        ck(cudaEventRecord(d.ev_copied[k], d.copy), "event");
    }
    D.level[k] = level;
    D.slot_host[slot] = k;
    D.queue.push_back({level, k});
}

void Solver::drain_wait_slot(int slot) {
    FrameDrain& D = drain_;
    if (D.slot_host.empty() || D.slot_host[slot] < 0) return;
    const int k = D.slot_host[slot];
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        for (auto& e : devs_) ck(cudaStreamWaitEvent(d.stream, e.ev_copied[k], 0), "wait");
    }
    D.slot_host[slot] = -1;
}

void Solver::drain_pop(SnapshotWriter& w) {
    FrameDrain& D = drain_;
    const auto [level, k] = D.queue.front();
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        ck(cudaEventSynchronize(d.ev_copied[k]), "snapshot D2H");
    }
    w.append_frame(level, D.host[k]);
    D.level[k] = -1;
    D.queue.erase(D.queue.begin());
}

void Solver::check_error() {
    for (auto& d : devs_) {
        int e = 0;
        cudaSetDevice(d.dev);
        ck(cudaMemcpy(&e, d.d_err, sizeof(int), cudaMemcpyDeviceToHost), "err D2H");
        if (e & 2) fail(SG_ETRANSPORT, "distributed barrier timed out waiting for a peer GPU");
        if (e) fail(SG_ENONPHYS, "non-physical state: rho <= 0 or p <= 0");
    }
}

// ---------------------------------------------------------- distributed --
namespace {
struct IpcBlob {
    int rank, nbuf;
    cudaIpcMemHandle_t h[40];
};
}  // namespace

std::vector<unsigned char> Solver::ipc_blob() const {
    if (!dist()) fail(SG_ELOGIC, "ipc_blob: not a distributed solver");
    IpcBlob b;
    std::memset(&b, 0, sizeof b);
    b.rank = rank_;
    const PartBuffers& pb = parts_[rank_];
    std::vector<void*> bufs;
    if (cfg_.engine == SG_SWEPT) {
        bufs.push_back(pb.rec[0]);  // all slots: one allocation
        bufs.push_back(pb.init);
        bufs.push_back(pb.out);
        if (pb.frames) bufs.push_back(pb.frames);  // snapshot frame ring (peers write edge cells)
    } else {
        for (double* r : pb.ring) bufs.push_back(r);
        bufs.push_back(pb.init_ghosted);
    }
    bufs.push_back(flags_);
    if (bufs.size() > 40) fail(SG_ELOGIC, "ipc_blob: too many buffers");
    b.nbuf = static_cast<int>(bufs.size());
    cudaSetDevice(devs_[0].dev);
    for (std::size_t i = 0; i < bufs.size(); ++i) ck(cudaIpcGetMemHandle(&b.h[i], bufs[i]), "cudaIpcGetMemHandle");
    std::vector<unsigned char> out(sizeof b);
    std::memcpy(out.data(), &b, sizeof b);
    return out;
}

void Solver::connect(const unsigned char* blobs, std::size_t per_rank) {
    if (!dist()) fail(SG_ELOGIC, "connect: not a distributed solver");
    if (per_rank != sizeof(IpcBlob)) fail(SG_ETRANSPORT, "connect: peer blob size mismatch");
    cudaSetDevice(devs_[0].dev);
    peer_flags_.assign(world_, nullptr);
    peer_flags_[rank_] = flags_;
    for (int q = 0; q < world_; ++q) {
        IpcBlob b;
        std::memcpy(&b, blobs + q * per_rank, sizeof b);
        if (b.rank != q) fail(SG_ETRANSPORT, "connect: blobs out of rank order");
        if (q == rank_) continue;
        std::vector<void*> p(b.nbuf, nullptr);
        for (int i = 0; i < b.nbuf; ++i) {
            ck(cudaIpcOpenMemHandle(&p[i], b.h[i], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            ipc_open_.push_back(p[i]);
        }
        PartBuffers& pb = parts_[q];
        int i = 0;
        if (cfg_.engine == SG_SWEPT) {
            pb.rec.resize(plan_.nslots);
            double* all = static_cast<double*>(p[i++]);
            for (int s2 = 0; s2 < plan_.nslots; ++s2) pb.rec[s2] = all + rec_len_ * s2;
            pb.init = static_cast<double*>(p[i++]);
            pb.out = static_cast<double*>(p[i++]);
            if (frame_ring_ > 0) pb.frames = static_cast<double*>(p[i++]);
        } else {
            pb.ring.resize(setup_.eq.substeps + 1);
            for (auto& r : pb.ring) r = static_cast<double*>(p[i++]);
            pb.init_ghosted = static_cast<double*>(p[i++]);
        }
        peer_flags_[q] = static_cast<unsigned long long*>(p[i++]);
        if (i != b.nbuf) fail(SG_ETRANSPORT, "connect: peer buffer list mismatch");
    }
    d_peer_flags_ = dev_upload(devs_[0], peer_flags_);
    if (cfg_.engine == SG_SWEPT) finalize_swept();
    else finalize_standard();
    ck(cudaDeviceSynchronize(), "connect sync");
    connected_ = true;
}

cudaError_t launch_dist_barrier(unsigned long long* const* peer_flags, unsigned long long* my_flags, int world,
                                int rank, unsigned long long* counter, int* err, cudaStream_t s);

void Solver::dist_barrier(DeviceCtx& d) {
    ++epoch_;
    ck(launch_dist_barrier(d_peer_flags_, flags_, world_, rank_, flags_ + kMaxParts, d.d_err, d.stream),
       "dist barrier");
    ++launches_;
}

void Solver::fetch(sg_result* r) {
    const Equation& eq = setup_.eq;
    const int nv = eq.nvars;
    const std::size_t nx = setup_.nx, ny = setup_.ny;
    double* field = static_cast<double*>(std::malloc(sizeof(double) * nv * nx * ny));
    if (!field) fail(SG_ELOGIC, "out of host memory");
    std::vector<double> piece;
    if (dist()) std::memset(field, 0, sizeof(double) * nv * nx * ny);
    for (auto& pb : parts_) {
        if (pb.dev < 0) continue;
        DeviceCtx& d = devs_[pb.dev];
        cudaSetDevice(d.dev);
        if (cfg_.engine == SG_SWEPT) {
            piece.resize(static_cast<std::size_t>(pw_) * ph_ * nv);
            ck(cudaMemcpy(piece.data(), pb.out, piece.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
            for (int v = 0; v < nv; ++v)
                for (int y = 0; y < ph_; ++y)
                    std::memcpy(&field[(v * ny + pb.pj * ph_ + y) * nx + pb.pi * pw_],
                                &piece[(static_cast<std::size_t>(v) * ph_ + y) * pw_], sizeof(double) * pw_);
        } else {
            const int n = eq.halo, pitch = pw_ + 2 * n, rows = ph_ + 2 * n;
            piece.resize(static_cast<std::size_t>(pitch) * rows * nv);
            const double* src = pb.ring[final_level_ % (eq.substeps + 1)];
            ck(cudaMemcpy(piece.data(), src, piece.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
            for (int v = 0; v < nv; ++v)
                for (int y = 0; y < ph_; ++y)
                    std::memcpy(&field[(v * ny + pb.pj * ph_ + y) * nx + pb.pi * pw_],
                                &piece[(static_cast<std::size_t>(v) * rows + y + n) * pitch + n], sizeof(double) * pw_);
        }
    }
    std::memset(r, 0, sizeof *r);
    r->engine = cfg_.engine;
    r->problem = cfg_.problem;
    r->mode = cfg_.mode;
    r->nx = setup_.nx;
    r->ny = setup_.ny;
    r->block = cfg_.block;
    r->ranks = cfg_.ranks;
    r->px = px_;
    r->py = py_;
    r->nvars = nv;
    r->steps_requested = cfg_.steps;
    r->actual_steps = actual_steps_;
    r->total_levels = total_levels_;
    if (cfg_.engine == SG_SWEPT) {
        r->octahedra = plan_.m;
        r->communicates = plan_.m + 1;
    }
    r->final_level = final_level_;
    r->dt = setup_.dt;
    r->dx = setup_.dx;
    r->dy = setup_.dy;
    r->setup_seconds = setup_seconds;
    r->solve_seconds = last_solve_;
    r->messages = messages_;
    r->bytes = bytes_;
    r->cell_updates = cell_updates_;
    r->kernel_launches = launches_;
    r->snapshot_frames = snapshot_frames_;
    r->final_field = field;
    r->nparts = nparts_;
    r->part_messages = static_cast<long*>(std::malloc(sizeof(long) * nparts_));
    r->part_bytes = static_cast<long long*>(std::malloc(sizeof(long long) * nparts_));
    for (int q = 0; q < nparts_; ++q) {
        r->part_messages[q] = q < static_cast<int>(part_messages_.size()) ? part_messages_[q] : 0;
        r->part_bytes[q] = q < static_cast<int>(part_bytes_.size()) ? part_bytes_[q] : 0;
    }
}

void Solver::upload(const double* host) {
    // Level 0 from a host field [var][ny][nx] (pinned host memory is DMA'd
    // directly).  Distributed runs pass only this rank's piece [var][ph][pw].
    const Equation& eq = setup_.eq;
    const std::size_t nx = dist() ? pw_ : setup_.nx, ny = dist() ? ph_ : setup_.ny;
    const int ox = dist() ? 0 : 1, oy = dist() ? 0 : 1;  // piece origin multiplier
    for (auto& pb : parts_) {
        if (pb.dev < 0) continue;
        DeviceCtx& d = devs_[pb.dev];
        cudaSetDevice(d.dev);
        for (int v = 0; v < eq.nvars; ++v) {
            const double* src = host + (v * ny + static_cast<std::size_t>(oy * pb.pj) * ph_) * nx + ox * pb.pi * pw_;
            if (cfg_.engine == SG_SWEPT) {
                ck(cudaMemcpy2DAsync(pb.init + static_cast<std::size_t>(v) * ph_ * pw_, pw_ * sizeof(double), src,
                                     nx * sizeof(double), pw_ * sizeof(double), ph_, cudaMemcpyHostToDevice,
                                     d.stream),
                   "upload");
            } else {
                const int n = eq.halo, pitch = pw_ + 2 * n, rows = ph_ + 2 * n;
                double* dst = pb.init_ghosted + static_cast<std::size_t>(v) * pitch * rows;
                if (dist()) fail(SG_EINVAL, "upload: the distributed standard engine takes its ghosts from peers; "
                                            "upload is supported for the swept engine only");
                auto copy = [&](int gx0, int gy0, int w, int h, int lx, int ly) {
                    // global window (wrapped start) -> local ghosted coords (lx, ly) in [-n, pw+n)
                    const int sx = ((gx0 % (int)nx) + (int)nx) % (int)nx, sy = ((gy0 % (int)ny) + (int)ny) % (int)ny;
                    ck(cudaMemcpy2DAsync(dst + static_cast<std::size_t>(ly + n) * pitch + (lx + n), pitch * sizeof(double),
                                         host + (v * ny + sy) * nx + sx, nx * sizeof(double), w * sizeof(double), h,
                                         cudaMemcpyHostToDevice, d.stream),
                       "upload");
                };
                const int gx = pb.pi * pw_, gy = pb.pj * ph_;
                copy(gx, gy, pw_, ph_, 0, 0);
                copy(gx - n, gy, n, ph_, -n, 0);
                copy(gx + pw_, gy, n, ph_, pw_, 0);
                copy(gx, gy - n, pw_, n, 0, -n);
                copy(gx, gy + ph_, pw_, n, 0, ph_);
            }
        }
    }
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        ck(cudaStreamSynchronize(d.stream), "upload sync");
    }
}

void Solver::download(double* host) {
    const Equation& eq = setup_.eq;
    const std::size_t nx = dist() ? pw_ : setup_.nx, ny = dist() ? ph_ : setup_.ny;
    const int ox = dist() ? 0 : 1, oy = dist() ? 0 : 1;
    for (auto& pb : parts_) {
        if (pb.dev < 0) continue;
        DeviceCtx& d = devs_[pb.dev];
        cudaSetDevice(d.dev);
        for (int v = 0; v < eq.nvars; ++v) {
            double* dst = host + (v * ny + static_cast<std::size_t>(oy * pb.pj) * ph_) * nx + ox * pb.pi * pw_;
            if (cfg_.engine == SG_SWEPT) {
                ck(cudaMemcpy2DAsync(dst, nx * sizeof(double), pb.out + static_cast<std::size_t>(v) * ph_ * pw_,
                                     pw_ * sizeof(double), pw_ * sizeof(double), ph_, cudaMemcpyDeviceToHost, d.stream),
                   "download");
            } else {
                const int n = eq.halo, pitch = pw_ + 2 * n, rows = ph_ + 2 * n;
                const double* src = pb.ring[final_level_ % (eq.substeps + 1)] +
                                    static_cast<std::size_t>(v) * pitch * rows + static_cast<std::size_t>(n) * pitch + n;
                ck(cudaMemcpy2DAsync(dst, nx * sizeof(double), src, pitch * sizeof(double), pw_ * sizeof(double), ph_,
                                     cudaMemcpyDeviceToHost, d.stream),
                   "download");
            }
        }
    }
    for (auto& d : devs_) {
        cudaSetDevice(d.dev);
        ck(cudaStreamSynchronize(d.stream), "download sync");
    }
}

void Solver::kernel_stats(int which, double* seconds, long* launches, double* alg_bytes, double* updates) const {
    (void)which;
    if (seconds) *seconds = prof_seconds_;
    if (launches) *launches = prof_launches_;
    if (alg_bytes) *alg_bytes = prof_bytes_;
    if (updates) *updates = prof_updates_;
}

}  // namespace sg
