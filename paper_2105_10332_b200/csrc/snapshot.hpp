// SWPT2D v1 snapshot stream (reference format, proj/src/snapshot.cpp:11-84):
// magic "SWPT2D\0\0", u32 version 1, u64 header length, JSON header
// {block, dt, dx, dy, nvars, nx, ny, params{alpha, gamma}, problem}, then
// frames of (u64 level, f64[var][y][x]) in increasing level order.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

namespace sg {

struct SnapshotMeta {
    std::string problem;
    int nx = 0, ny = 0, nvars = 0, block = 0;
    double dt = 0, dx = 0, dy = 0, alpha = 1.0, gamma = 1.4;
};

class SnapshotWriter {
  public:
    SnapshotWriter(const std::string& path, const SnapshotMeta& meta);
    ~SnapshotWriter();
    void append_frame(long level, const double* data);
    void flush();
    long frames() const { return frames_; }

  private:
    std::FILE* f_ = nullptr;
    SnapshotMeta meta_;
    long frames_ = 0, last_ = -1;
    std::size_t plane_ = 0;
};

}  // namespace sg
