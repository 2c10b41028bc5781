// acotsp_gpu — minimal C++ driver over include/aco_gpu.hpp: the reference's
// `acotsp solve` path (tools/acotsp.cpp:110-136) on the B200 engine.  Also the
// C++ compile/link check of the drop-in header (tests/test_cpp_wrapper.py).
//
//   acotsp_gpu <instance.tsp | synth:N> [iters] [roulette|nn|data-parallel]
//              [accumulate|scatter-gather|scatter-gather-tiled|symmetric-reduction]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "aco_gpu.hpp"

namespace {

aco::gpu::InstanceSpec synthetic(int n) {
    // splitmix64 seeded with 42, coords in [0, 10000]
    aco::gpu::InstanceSpec s;
    s.name = "synth" + std::to_string(n);
    s.dimension = n;
    uint64_t st = 42;
    auto next = [&st] {
        uint64_t z = (st += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    for (int i = 0; i < n; ++i) {
        s.xs.push_back(static_cast<double>(next() % 10001u));
        s.ys.push_back(static_cast<double>(next() % 10001u));
    }
    return s;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <instance.tsp|synth:N> [iters] [selection] [deposit]\n",
                     argv[0]);
        return 1;
    }
    try {
        const std::string src = argv[1];
        const aco::gpu::InstanceSpec spec = src.rfind("synth:", 0) == 0
                                                ? synthetic(std::atoi(src.c_str() + 6))
                                                : aco::gpu::load_instance(src);
        aco::gpu::RunConfig cfg;
        cfg.params.iterations = argc > 2 ? std::atoi(argv[2]) : 10;
        cfg.selection = aco::gpu::Selection::roulette_full;
        if (argc > 3) {
            const std::string s = argv[3];
            cfg.selection = s == "nn" ? aco::gpu::Selection::roulette_nn
                          : s == "data-parallel" ? aco::gpu::Selection::data_parallel_tiled
                                                 : aco::gpu::Selection::roulette_full;
        }
        if (argc > 4) {
            const std::string d = argv[4];
            cfg.deposit = d == "scatter-gather" ? aco::gpu::Deposit::scatter_gather
                        : d == "scatter-gather-tiled" ? aco::gpu::Deposit::scatter_gather_tiled
                        : d == "symmetric-reduction" ? aco::gpu::Deposit::symmetric_reduction
                                                     : aco::gpu::Deposit::accumulate;
        }
        aco::gpu::Engine engine(aco::gpu::build_problem(spec), cfg);
        const aco::gpu::RunReport rep = engine.run();
        for (const auto& r : rep.per_iteration)
            std::printf("iter %d best %lld mean %.17g construct_ms %.3f update_ms %.3f\n",
                        r.iteration, static_cast<long long>(r.best_length), r.mean_length,
                        r.construct_ms, r.update_ms);
        std::printf("best %lld\n", static_cast<long long>(rep.best_length));
        return 0;
    } catch (const aco::gpu::Error& e) {
        std::fprintf(stderr, "error (%d): %s\n", e.status(), e.what());
        // CLI exit codes of the reference (acotsp.cpp:44-55): I/O-class -> 2, other -> 1
        const int c = e.errc();
        return (c == 11 || (c >= 0 && c <= 3)) ? 2 : 1;
    }
}
