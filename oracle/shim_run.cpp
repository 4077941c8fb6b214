// Test/bench infrastructure only: the reference-side drop-in, exercised.
//   shim_run '<SolverConfig JSON>'
// Parses the config with the reference's own SolverConfig::from_json
// (proj/src/config.cpp:79-125), runs it through sweptgrid::run_gpu
// (include/sweptgrid_gpu.hpp -> libsweptgpu.so, the B200 solver) and prints
// the reference's RunRecord::to_json (proj/src/engine.cpp:461-491) plus the
// FNV-1a-64 of the final field -- the same line ref_run prints for the CPU
// reference, so a test can compare the two byte for byte.
#include <cstdint>
#include <cstdio>
#include <iostream>

#include "sweptgrid/config.hpp"
#include "sweptgrid_gpu.hpp"

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: shim_run '<config json>'\n");
        return 2;
    }
    try {
        const auto cfg = sweptgrid::SolverConfig::from_json(nlohmann::json::parse(argv[1]));
        const sweptgrid::RunResult r = sweptgrid::run_gpu(cfg);
        nlohmann::json j = r.record.to_json();
        j["final_level"] = r.final_field.level;
        std::uint64_t h = 1469598103934665603ull;
        const auto* p = reinterpret_cast<const unsigned char*>(r.final_field.data.data());
        for (std::size_t i = 0; i < r.final_field.data.size() * sizeof(double); ++i) {
            h ^= p[i];
            h *= 1099511628211ull;
        }
        char hex[32];
        std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(h));
        j["fnv1a64"] = hex;
        std::cout << j.dump() << std::endl;
        return 0;
    } catch (const std::exception& e) {
        std::cout << "{\"error\": " << nlohmann::json(std::string(e.what())).dump() << "}" << std::endl;
        return 1;
    }
}
