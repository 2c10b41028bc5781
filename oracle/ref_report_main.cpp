// TEST INFRASTRUCTURE ONLY: writes the reference's own RunReport JSON
// (report_to_json(...).dump(2), report.hpp:32-67) and bench CSV rows
// (report.hpp:72-86) for the synth198 golden runs into tests/golden/.
// Built and run by tests/golden/make_golden.py (needs /root/reference and the
// image's vendored nlohmann/json.hpp).
#include <cstdint>
#include <fstream>
#include <iostream>
#include <string>

#include "aco/engine.hpp"
#include "aco/report.hpp"

int main(int argc, char** argv) {
    // args: out_prefix deposit iterations ; coords on stdin "n\nx y\n..."
    if (argc < 4) return 1;
    const std::string prefix = argv[1];
    const int deposit = std::atoi(argv[2]), iterations = std::atoi(argv[3]);
    int n = 0;
    std::cin >> n;
    aco::InstanceSpec spec;
    spec.name = "synth198";
    spec.dimension = n;
    spec.edge_weight_type = aco::EdgeWeightType::euc_2d;
    spec.coords.resize(n);
    for (int i = 0; i < n; ++i) std::cin >> spec.coords[i].first >> spec.coords[i].second;
    aco::RunConfig cfg;
    cfg.params.iterations = iterations;
    cfg.selection.variant = aco::Selection::roulette_full;
    cfg.deposit.variant = static_cast<aco::Deposit>(deposit);
    cfg.workers = 1;
    aco::Engine engine(aco::build_problem(spec), cfg);
    aco::RunReport rep = engine.run();
    rep.instance_name = spec.name;
    std::ofstream(prefix + ".json") << aco::report_to_json(rep).dump(2) << '\n';
    std::ofstream csv(prefix + ".csv");
    csv << aco::bench_csv_header() << '\n';
    for (const auto& r : rep.per_iteration)
        aco::write_bench_csv_row(csv, spec.name, n, cfg.selection.variant, cfg.deposit.variant,
                                 cfg.deposit.tile_size, 0, r);
    return 0;
}
