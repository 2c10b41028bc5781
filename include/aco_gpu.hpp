// aco_gpu.hpp — header-only C++ wrapper over the C ABI (aco_gpu.h) that keeps
// the reference's aco:: API shape (proj/include/aco/engine.hpp:22-204), so a
// caller of aco::Engine / aco::run swaps in aco::gpu::Engine / aco::gpu::run.
//
//   reference (CPU)                         this header (B200)
//   aco::Parameters        model.hpp:29     aco::gpu::Parameters
//   aco::RunConfig         engine.hpp:22    aco::gpu::RunConfig
//   aco::IterationRecord   engine.hpp:31    aco::gpu::IterationRecord
//   aco::RunReport         engine.hpp:40    aco::gpu::RunReport
//   aco::Engine            engine.hpp:55    aco::gpu::Engine
//   aco::run               engine.hpp:198   aco::gpu::run
//   aco::Error{Errc}       errors.hpp:31    aco::gpu::Error{status}
//
// Link with libaco_gpu.so (paper_1101_2678_b200/).  Errors arrive as status
// codes and are rethrown here as aco::gpu::Error (code = 1 + aco::Errc for the
// reference's error classes, ACO_E_* for device/NCCL failures).
#pragma once

#include <cstdint>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "aco_gpu.h"

namespace aco::gpu {

class Error : public std::runtime_error {
public:
    Error(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
    int status() const noexcept { return status_; }
    // index into aco::Errc (errors.hpp:8-27) when 1 <= status <= 13
    int errc() const noexcept { return status_ >= 1 && status_ <= 13 ? status_ - 1 : -1; }

private:
    int status_;
};

inline void check(aco_status s, const aco_gpu_ctx* ctx = nullptr) {
    if (s != ACO_OK)
        throw Error(s, std::string(aco_errc_name(s)) + ": " +
                           (ctx ? aco_gpu_last_error(ctx) : aco_last_error()));
}

enum class Selection { roulette_full = ACO_SEL_ROULETTE, roulette_nn = ACO_SEL_NN,
                       data_parallel_tiled = ACO_SEL_DATA_PARALLEL };
enum class Deposit { accumulate = ACO_DEP_ACCUMULATE, scatter_gather = ACO_DEP_SCATTER_GATHER,
                     scatter_gather_tiled = ACO_DEP_SCATTER_GATHER_TILED,
                     symmetric_reduction = ACO_DEP_SYMMETRIC_REDUCTION };

struct InstanceSpec {  // tsplib.hpp:27
    std::string name;
    int dimension = 0;
    int edge_weight_type = ACO_EUC_2D;
    std::vector<double> xs, ys;
};

inline InstanceSpec parse_instance(const std::string& text) {  // tsplib.hpp:76
    InstanceSpec s;
    int32_t dim = 0, ewt = 0;
    check(aco_parse_instance(text.c_str(), &dim, &ewt, nullptr, nullptr, 0, nullptr, 0));
    s.dimension = dim;
    s.edge_weight_type = ewt;
    s.xs.resize(dim);
    s.ys.resize(dim);
    char name[4096] = {0};
    check(aco_parse_instance(text.c_str(), &dim, &ewt, s.xs.data(), s.ys.data(), dim, name,
                             sizeof(name)));
    s.name = name;
    return s;
}

inline InstanceSpec load_instance(const std::string& path) {  // tsplib.hpp:281
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(ACO_E_IO_ERROR, "io_error: cannot open file: " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return parse_instance(ss.str());
}

struct ProblemInstance {  // model.hpp:23
    int n = 0;
    std::vector<int32_t> dist;  // n x n row-major
};

inline ProblemInstance build_problem(const InstanceSpec& spec) {  // model.hpp:125
    ProblemInstance p;
    p.n = spec.dimension;
    p.dist.resize(static_cast<size_t>(p.n) * p.n);
    check(aco_build_distances(p.n, spec.xs.data(), spec.ys.data(), spec.edge_weight_type,
                              p.dist.data()));
    return p;
}

struct Parameters {  // model.hpp:29
    double alpha = 1.0, beta = 2.0, rho = 0.5;
    int m = 0, nn = 30, iterations = 100;
    uint64_t seed = 1;
    int tile_size = 64;
};

struct RunConfig {  // engine.hpp:22 (+ device placement / sharding)
    Parameters params;
    Selection selection = Selection::roulette_nn;
    Deposit deposit = Deposit::accumulate;
    bool random_start = false;
    std::string instance_path;
    int device = 0;
    int stream = ACO_STREAM_AUTO;
    int rank = 0, world = 1;
    const uint8_t* nccl_id = nullptr;
};

struct AccessLedger { double global_loads = 0, global_stores = 0, shared_loads = 0, atomic_ops = 0; };

struct IterationRecord {  // engine.hpp:31
    int iteration = 0;
    int64_t best_length = 0;
    double mean_length = 0.0;
    double construct_ms = 0.0;
    double update_ms = 0.0;
    AccessLedger deposit_ledger;
};

struct RunReport {  // engine.hpp:40
    std::string instance_name;
    int n = 0, m = 0;
    uint64_t seed = 0;
    RunConfig config;
    std::vector<int32_t> best_tour;
    int64_t best_length = 0;
    std::vector<IterationRecord> per_iteration;
};

class Engine {  // engine.hpp:55
public:
    Engine(ProblemInstance problem, RunConfig config)
        : problem_(std::move(problem)), config_(std::move(config)) {
        if (config_.params.iterations < 1)
            throw Error(ACO_E_CONFIG_ERROR, "config_error: iterations must be >= 1");
        aco_gpu_params p{};
        p.n = problem_.n;
        p.m = config_.params.m;
        p.nn = config_.params.nn;
        p.theta = config_.params.tile_size;
        p.selection = static_cast<int32_t>(config_.selection);
        p.deposit = static_cast<int32_t>(config_.deposit);
        p.random_start = config_.random_start ? 1 : 0;
        p.stream = config_.stream;
        p.alpha = config_.params.alpha;
        p.beta = config_.params.beta;
        p.rho = config_.params.rho;
        p.seed = config_.params.seed;
        p.device = config_.device;
        p.rank = config_.rank;
        p.world = config_.world;
        if (config_.nccl_id)
            for (int i = 0; i < 128; ++i) p.nccl_id[i] = config_.nccl_id[i];
        check(aco_gpu_create(&p, problem_.dist.data(), &ctx_));
        int32_t m = 0, a0 = 0, a1 = 0, st = 0, it = 0;
        double tau0 = 0;
        aco_gpu_get_info(ctx_, &m, &a0, &a1, &tau0, &st, &it);
        m_ = m;
        local_ants_ = a1 - a0;
        config_.params.m = m;
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() { aco_gpu_destroy(ctx_); }

    const ProblemInstance& problem() const noexcept { return problem_; }
    const RunConfig& config() const noexcept { return config_; }

    std::vector<double> pheromone() const {  // engine.hpp:82 (copied out of HBM)
        std::vector<double> t(static_cast<size_t>(problem_.n) * problem_.n);
        check(aco_gpu_get_pheromone(ctx_, t.data()), ctx_);
        return t;
    }
    std::vector<double> choice() const {  // engine.hpp:83
        std::vector<double> c(static_cast<size_t>(problem_.n) * problem_.n);
        check(aco_gpu_get_choice(ctx_, c.data()), ctx_);
        return c;
    }
    // engine.hpp:84: this rank's ants, rows of n+1 cities, and their lengths
    void ants(std::vector<int32_t>& tours, std::vector<int64_t>& lengths) const {
        tours.resize(static_cast<size_t>(local_ants_) * (problem_.n + 1));
        lengths.resize(local_ants_);
        check(aco_gpu_get_tours(ctx_, tours.data(), lengths.data()), ctx_);
    }
    int64_t best_length() const {  // engine.hpp:85
        int64_t len = 0;
        check(aco_gpu_get_best(ctx_, nullptr, &len), ctx_);
        return len;
    }
    std::vector<int32_t> best_tour() const {  // engine.hpp:86
        std::vector<int32_t> t(problem_.n + 1);
        int64_t len = 0;
        check(aco_gpu_get_best(ctx_, t.data(), &len), ctx_);
        return t;
    }

    IterationRecord run_iteration() {  // engine.hpp:88
        aco_gpu_iter_record r{};
        check(aco_gpu_iterate(ctx_, &r, nullptr, nullptr), ctx_);
        IterationRecord out;
        out.iteration = r.iteration;
        out.best_length = r.best_length;
        out.mean_length = r.mean_length;
        out.construct_ms = r.construct_ms;
        out.update_ms = r.update_ms;
        out.deposit_ledger = {r.ledger[0], r.ledger[1], r.ledger[2], r.ledger[3]};
        return out;
    }

    RunReport run() {  // engine.hpp:159
        RunReport rep;
        rep.n = problem_.n;
        rep.m = m_;
        rep.seed = config_.params.seed;
        rep.config = config_;
        for (int it = 0; it < config_.params.iterations; ++it)
            rep.per_iteration.push_back(run_iteration());
        rep.best_length = best_length();
        rep.best_tour = best_tour();
        return rep;
    }

    aco_gpu_ctx* handle() noexcept { return ctx_; }

private:
    ProblemInstance problem_;
    RunConfig config_;
    aco_gpu_ctx* ctx_ = nullptr;
    int m_ = 0;
    int local_ants_ = 0;
};

inline RunReport run(const RunConfig& config) {  // engine.hpp:198
    const InstanceSpec spec = load_instance(config.instance_path);
    Engine engine(build_problem(spec), config);
    RunReport rep = engine.run();
    rep.instance_name = spec.name;
    return rep;
}

} // namespace aco::gpu
