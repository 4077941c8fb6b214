// Test/bench infrastructure only.  CLI over the unmodified reference library:
//   ref_run '<SolverConfig JSON>' [reps]
// Runs sweptgrid::run (proj/src/engine.cpp:493) `reps` times and prints one
// JSON object: the last RunRecord plus the median wall_seconds, the rate
// cell_updates / wall_seconds (the reference's own unit, engine.cpp:519-528)
// and an FNV-1a-64 hash of the final field bytes.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <vector>

#include "sweptgrid/config.hpp"
#include "sweptgrid/engine.hpp"

using namespace sweptgrid;

static std::uint64_t fnv1a(const std::vector<double>& d) {
    std::uint64_t h = 1469598103934665603ull;
    const unsigned char* p = reinterpret_cast<const unsigned char*>(d.data());
    for (std::size_t i = 0; i < d.size() * sizeof(double); ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_run '<config json>' [reps]\n");
        return 2;
    }
    const int reps = argc > 2 ? std::atoi(argv[2]) : 1;
    try {
        const SolverConfig cfg = SolverConfig::from_json(nlohmann::json::parse(argv[1]));
        std::vector<double> walls;
        RunResult r;
        for (int i = 0; i < reps; ++i) {
            r = run(cfg);
            walls.push_back(r.record.wall_seconds);
        }
        std::sort(walls.begin(), walls.end());
        nlohmann::json j = r.record.to_json();
        j.erase("per_rank");
        j["final_level"] = r.final_field.level;
        j["median_wall_seconds"] = walls[walls.size() / 2];
        j["cell_updates_per_s"] = static_cast<double>(r.record.cell_updates) / walls[walls.size() / 2];
        char hex[32];
        std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(fnv1a(r.final_field.data)));
        j["fnv1a64"] = hex;
        std::cout << j.dump() << std::endl;
        return 0;
    } catch (const std::exception& e) {
        std::cout << "{\"error\": " << nlohmann::json(std::string(e.what())).dump() << "}" << std::endl;
        return 1;
    }
}
