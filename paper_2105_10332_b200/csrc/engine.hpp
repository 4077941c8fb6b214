// GPU engine: partitions, device buffers and the solve loops for the swept
// and standard engines (the B200 replacement of SweptRank / StandardRank,
// engine.cpp:169-425 of the reference).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "kernels.cuh"
#include "plan.hpp"
#include "snapshot.hpp"
#include "sg_internal.hpp"

namespace sg {

struct PartBuffers {
    int id = 0, pi = 0, pj = 0, dev = 0;
    // swept
    double* init = nullptr;             // [var][ph][pw] level-0 piece
    double* out = nullptr;              // [var][ph][pw] output level piece
    std::vector<double*> rec;           // [nslots] records, ghost-extended instance grid
    // standard
    std::vector<double*> ring;          // [S+1] ghosted planes
    double* init_ghosted = nullptr;     // resident ghosted copy of level 0
    // snapshots (swept): ring of frame planes [slot][var][ph][pw]
    double* frames = nullptr;
};

struct DeviceCtx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr, ev_sync = nullptr;
    int* d_err = nullptr;
    std::vector<int> parts;
    // device-resident tables
    std::vector<void*> allocs;
    DevLevel* d_lev[K_NKINDS] = {};
    int* d_exp_off[K_NKINDS] = {};
    int* d_exp_vs[K_NKINDS] = {};
    int2* d_exp_pairs[K_NKINDS] = {};
    int4* d_lanes[K_NKINDS] = {};
    int2* d_pitch[K_NKINDS] = {};
    std::vector<int4*> d_imp, d_init;
    std::vector<int2*> d_imp2;
    std::map<std::pair<int, int>, int2*> imp_off;  // (class, slot rotation) -> column gather table
    std::map<std::pair<int, int>, std::vector<int>> imp_off_host;  // host copy of imp_off's offsets
    std::map<std::pair<int, int>, int*> imp_dense; // (class, slot rotation) -> dense gather table (or null)
    double** d_rec_tab = nullptr;
    double* oct_scratch = nullptr;  // b32 split Octahedron: level-k state of every instance
    double* gm_scratch = nullptr;   // phases too large for shared memory: level storage in HBM
    long gm_stride = 0;
    int gm_ctas = 0;
    double** d_frames_tab = nullptr;
    const double** d_init_tab = nullptr;
    double** d_out_tab = nullptr;
    std::vector<const double**> d_std_r1, d_std_r2;
    std::vector<double**> d_std_out;
    // per-launch arguments (swept) -- built once at create
    std::vector<SweptArgs> swept_args;
    std::vector<cudaEvent_t> prof_ev;   // kernel profiling pairs
    // concurrent bridges (single device): a second stream and one event per launch
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> launch_ev;
    // snapshot drain: D2H copies of completed frames on their own stream
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_ready = nullptr;            // compute stream: frame level complete
    std::vector<cudaEvent_t> ev_copied;        // per pinned host frame: copies done
};

// Snapshot frames in flight (one process): pinned host frames filled by
// cudaMemcpy2DAsync on each device's copy stream while the solve goes on;
// written to the SWPT2D file in level order once their copies completed.
struct FrameDrain {
    std::vector<double*> host;                 // pinned full frames [var][ny][nx]
    std::vector<long> level;                   // level held by host frame k (-1: free)
    std::vector<int> slot_host;                // device frame slot -> host frame copying it (-1: none)
    std::vector<std::pair<long, int>> queue;   // (level, host frame) in append order
    int next = 0;
};

class Solver {
  public:
    // rank/world >= 0: distributed run, one process per GPU owning partition `rank`
    explicit Solver(const sg_config& cfg, int rank = -1, int world = 0);
    ~Solver();
    void reset();
    double solve();  // device seconds (max over devices)
    void fetch(sg_result* r);
    void upload(const double* host);    // replace level 0 from a host field
    void download(double* host);        // final field into a host buffer
    void kernel_stats(int which, double* seconds, long* launches, double* alg_bytes, double* updates) const;
    void set_prof_kind(int k) { prof_kind_ = k; }

    const Setup& setup() const { return setup_; }
    double setup_seconds = 0.0;
    bool profile = false;
    // a one-shot solve (sg_run) enqueues its launches directly: capturing and
    // instantiating a CUDA graph costs more than it saves on a single replay
    void set_graph(bool on) { use_graph_ = use_graph_ && on; }
    bool use_graph_ = true;   // SG_NO_GRAPH=1 disables CUDA graph replay
    bool gm_phases_ = false;  // swept phases with their level storage in HBM (blocks too large for smem)

    // distributed (one process per GPU): export this rank's buffers as CUDA
    // IPC handles, then map every other rank's and build the kernel tables
    std::vector<unsigned char> ipc_blob() const;
    void connect(const unsigned char* blobs, std::size_t per_rank);
    bool dist() const { return rank_ >= 0; }

  private:
    void build_swept();
    void build_standard();
    void finalize_swept();
    void finalize_standard();
    void dist_barrier(DeviceCtx& d);
    void check_error();

    sg_config cfg_;
    Setup setup_;
    SweptPlan plan_;
    int px_ = 1, py_ = 1, pw_ = 0, ph_ = 0, nparts_ = 1;
    long final_level_ = 0, total_levels_ = 0, actual_steps_ = 0;
    long long cell_updates_ = 0;
    long messages_ = 0;
    long long bytes_ = 0;
    std::vector<long> part_messages_;       // per partition (ledger per rank)
    std::vector<long long> part_bytes_;
    long launches_ = 0;
    std::vector<PartBuffers> parts_;
    std::vector<DeviceCtx> devs_;
    double last_solve_ = 0.0;
    int rank_ = -1, world_ = 0;
    bool connected_ = false;
    unsigned long long* flags_ = nullptr;            // [kMaxParts] epochs signalled by each rank
    std::vector<unsigned long long*> peer_flags_;     // every rank's flag array (IPC-mapped)
    unsigned long long** d_peer_flags_ = nullptr;
    unsigned long long epoch_ = 0;
    std::vector<void*> ipc_open_;
    cudaGraphExec_t graph_exec_ = nullptr;
    long graph_launches_ = 0;
    // snapshots (SWPT2D, snapshot.cpp of the reference)
    std::string snap_path_;
    long snap_every_ = 1;
    int frame_ring_ = 0;
    std::size_t rec_len_ = 0;     // doubles per record slot (all slots contiguous)
    std::vector<std::vector<long>> done_after_;  // swept: levels completed by launch i
    long snapshot_frames_ = 0;
    void snapshot_frame(SnapshotWriter& w, long level, int slot_or_ring);  // D2H + assemble + append
    // one process: start the D2H of level `level` (device frame `slot`) after
    // the work enqueued so far; wait for host frames / device slots as needed
    void drain_start(SnapshotWriter& w, long level, int slot);
    void drain_wait_slot(int slot);            // compute streams wait until `slot` was copied out
    void drain_pop(SnapshotWriter& w);         // oldest pending frame -> file
    FrameDrain drain_;
    int nslots_frames() const;
    // profiling of the dominant kernel class
    int prof_kind_ = -1;
    double prof_seconds_ = 0.0;
    long prof_launches_ = 0;
    double prof_bytes_ = 0.0, prof_updates_ = 0.0;
};

}  // namespace sg
