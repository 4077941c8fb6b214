// SWPT2D v1 writer -- see snapshot.hpp.  The JSON header is produced by the
// same library the reference uses (nlohmann/json 3.11.3, default std::map
// object => keys sorted, same number formatting), so files are byte-identical
// to the reference's for identical fields.
#include "snapshot.hpp"

#include <json.hpp>

#include "sg_internal.hpp"

namespace sg {

namespace {
constexpr char kMagic[8] = {'S', 'W', 'P', 'T', '2', 'D', '\0', '\0'};
constexpr std::uint32_t kVersion = 1;
}  // namespace

SnapshotWriter::SnapshotWriter(const std::string& path, const SnapshotMeta& m) : meta_(m) {
    f_ = std::fopen(path.c_str(), "wb");
    if (!f_) fail(SG_EIO, "snapshot: cannot open " + path);
    nlohmann::json j;  // SnapshotMeta::to_json, snapshot.cpp:29-41
    j["problem"] = m.problem;
    j["nx"] = m.nx;
    j["ny"] = m.ny;
    j["nvars"] = m.nvars;
    j["block"] = m.block;
    j["dt"] = m.dt;
    j["dx"] = m.dx;
    j["dy"] = m.dy;
    j["params"] = {{"alpha", m.alpha}, {"gamma", m.gamma}};  // engine.cpp:89
    const std::string header = j.dump();
    const std::uint64_t hlen = header.size();
    std::fwrite(kMagic, 1, sizeof kMagic, f_);
    std::fwrite(&kVersion, sizeof kVersion, 1, f_);
    std::fwrite(&hlen, sizeof hlen, 1, f_);
    std::fwrite(header.data(), 1, header.size(), f_);
    plane_ = static_cast<std::size_t>(m.nvars) * m.nx * m.ny;
}

SnapshotWriter::~SnapshotWriter() {
    if (f_) std::fclose(f_);
}

void SnapshotWriter::append_frame(long level, const double* data) {
    if (level <= last_) fail(SG_EIO, "snapshot: frames must be appended in level order");
    last_ = level;
    const std::uint64_t lv = static_cast<std::uint64_t>(level);
    std::fwrite(&lv, sizeof lv, 1, f_);
    if (std::fwrite(data, sizeof(double), plane_, f_) != plane_) fail(SG_EIO, "snapshot: write failed");
    ++frames_;
}

void SnapshotWriter::flush() {
    if (std::fflush(f_) != 0) fail(SG_EIO, "snapshot: write failed");
}

}  // namespace sg
