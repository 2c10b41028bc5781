// aco_gpu.hpp — the reference's C++ API (proj/include/aco, namespace aco::)
// over the B200 engine's C ABI (aco_gpu.h, libaco_gpu.so).
//
// Source-compatible drop-in: every type and function below lives in
// `namespace aco { inline namespace gpu { ... } }`, so code written against the
// reference — `aco::RunConfig config; config.selection.variant = ...;
// aco::run(config)` — compiles unchanged against this header (put
// <repo>/include on the include path instead of proj/include; the shims in
// include/aco/*.hpp forward the reference's header names here), and
// `aco::gpu::X` names the same entities explicitly.
//
//   reference                                this header
//   Errc / Error / errc_name  errors.hpp:8-57  same names (+ cuda_error, nccl_error, unsupported)
//   Matrix<T>                 matrix.hpp:12    same API
//   EdgeWeightType, InstanceSpec, parse_instance, edge_weight, canonical_text,
//   parse_tour, read_file, load_instance  tsplib.hpp:16-283  same API (parser: libaco_gpu.so)
//   ProblemInstance, Parameters{validate}, PheromoneMatrix, ChoiceInfo,
//   NearestNeighborLists, TabuBitset, AntState, build_problem, build_nn_lists,
//   tour_length, greedy_nn_tour_length, initial_pheromone  model.hpp:23-262
//   RngStream                 rng.hpp:50-88    same API (Philox4x32-10 in libaco_gpu.so)
//   Selection, SelectionStrategy, selection_name   construction.hpp:13-27
//   Deposit, DepositStrategy, deposit_name, AccessLedger, predicted_access_cost,
//   MatrixDiff, max_cell_difference        pheromone.hpp:16-54, 366-416
//   RunConfig, IterationRecord, RunReport, Engine, run, VerifyReport,
//   verify_deposit_equivalence             engine.hpp:22-292
//   format_double, report_to_json, bench_csv_header, write_bench_csv_row
//                                          report.hpp:13-86 (JSON: a minimal value
//                                          type with nlohmann's dump(indent) shape)
//
// What differs, by design:
//   * the colony state lives in HBM: Engine::pheromone()/choice()/ants() copy
//     it to host on first access after each iteration (cached until the next);
//   * RunConfig::workers is validated like the reference's but the CUDA grid
//     replaces the thread pool; RunConfig carries device/sharding extras;
//   * ledgers: IterationRecord::deposit_ledger holds the closed-form model
//     (predicted_access_cost) — the kernels make no abstract accesses to count;
//   * compute_choice_info / construct_tour / apply_deposit on host matrices
//     are not provided: the Engine runs them on the device (engine.hpp's loop).
#pragma once

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <map>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <utility>
#include <variant>
#include <vector>

#include "aco_gpu.h"

namespace aco {
inline namespace gpu {

// ---- errors.hpp ---------------------------------------------------------
enum class Errc {
    missing_field,
    unsupported_edge_weight_type,
    malformed_coord,
    dimension_mismatch,
    index_out_of_range,
    overflow,
    invalid_length,
    not_a_permutation,
    not_closed,
    all_visited,
    inconsistent_length,
    io_error,
    config_error,
    // device side (status = 1 + code, as for the reference's classes)
    cuda_error = ACO_E_CUDA - 1,
    nccl_error = ACO_E_NCCL - 1,
    unsupported = ACO_E_UNSUPPORTED - 1,
};

inline const char* errc_name(Errc code) noexcept { return aco_errc_name(1 + static_cast<int>(code)); }

class Error : public std::runtime_error {
public:
    Error(Errc code, const std::string& message) : std::runtime_error(message), code_(code) {}
    Errc code() const noexcept { return code_; }
    int status() const noexcept { return 1 + static_cast<int>(code_); }

private:
    Errc code_;
};

inline void check(aco_status s, const aco_gpu_ctx* ctx = nullptr) {
    if (s != ACO_OK)
        throw Error(static_cast<Errc>(static_cast<int>(s) - 1),
                    ctx ? aco_gpu_last_error(ctx) : aco_last_error());
}

// ---- matrix.hpp ---------------------------------------------------------
template <typename T>
class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, T fill = T{})
        : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
    std::size_t rows() const noexcept { return rows_; }
    std::size_t cols() const noexcept { return cols_; }
    T& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    const T& operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
    std::span<T> row(std::size_t i) { return {data_.data() + i * cols_, cols_}; }
    std::span<const T> row(std::size_t i) const { return {data_.data() + i * cols_, cols_}; }
    T* data() noexcept { return data_.data(); }
    const T* data() const noexcept { return data_.data(); }
    std::size_t size() const noexcept { return data_.size(); }
    bool operator==(const Matrix&) const = default;

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<T> data_;
};

// ---- tsplib.hpp ---------------------------------------------------------
enum class EdgeWeightType { euc_2d = ACO_EUC_2D, ceil_2d = ACO_CEIL_2D, att = ACO_ATT };

inline const char* edge_weight_type_name(EdgeWeightType t) noexcept {
    switch (t) {
    case EdgeWeightType::euc_2d: return "EUC_2D";
    case EdgeWeightType::ceil_2d: return "CEIL_2D";
    case EdgeWeightType::att: return "ATT";
    }
    return "?";
}

struct InstanceSpec {
    std::string name;
    int dimension = 0;
    EdgeWeightType edge_weight_type = EdgeWeightType::euc_2d;
    std::vector<std::pair<double, double>> coords; // 0-based city order
};

inline InstanceSpec parse_instance(std::string_view text) {
    const std::string buf(text); // the C ABI takes NUL-terminated text
    int32_t dim = 0, ewt = 0;
    check(aco_parse_instance(buf.c_str(), &dim, &ewt, nullptr, nullptr, 0, nullptr, 0));
    std::vector<double> xs(static_cast<std::size_t>(dim)), ys(static_cast<std::size_t>(dim));
    std::string name(4096, '\0');
    check(aco_parse_instance(buf.c_str(), &dim, &ewt, xs.data(), ys.data(), dim, name.data(),
                             static_cast<int32_t>(name.size())));
    InstanceSpec spec;
    spec.name = name.c_str();
    spec.dimension = dim;
    spec.edge_weight_type = static_cast<EdgeWeightType>(ewt);
    spec.coords.resize(static_cast<std::size_t>(dim));
    for (int i = 0; i < dim; ++i) spec.coords[static_cast<std::size_t>(i)] = {xs[i], ys[i]};
    return spec;
}

inline std::int32_t edge_weight(const InstanceSpec& spec, int i, int j) {
    if (i < 0 || j < 0 || i >= spec.dimension || j >= spec.dimension)
        throw Error(Errc::index_out_of_range,
                    "city index outside 0.." + std::to_string(spec.dimension - 1));
    const double xs[2] = {spec.coords[static_cast<std::size_t>(i)].first,
                          spec.coords[static_cast<std::size_t>(j)].first};
    const double ys[2] = {spec.coords[static_cast<std::size_t>(i)].second,
                          spec.coords[static_cast<std::size_t>(j)].second};
    int32_t d[4] = {0, 0, 0, 0};
    check(aco_build_distances(2, xs, ys, static_cast<int32_t>(spec.edge_weight_type), d));
    return d[1];
}

inline std::string to_chars_string(double v) {
    char buf[64];
    auto [p, ec] = std::to_chars(buf, buf + sizeof(buf), v);
    (void)ec;
    return std::string(buf, static_cast<std::size_t>(p - buf));
}

inline std::string canonical_text(const InstanceSpec& spec) {
    std::ostringstream out;
    out << "NAME : " << spec.name << "\nTYPE : TSP\nDIMENSION : " << spec.dimension
        << "\nEDGE_WEIGHT_TYPE : " << edge_weight_type_name(spec.edge_weight_type)
        << "\nNODE_COORD_SECTION\n";
    for (int i = 0; i < spec.dimension; ++i) {
        const auto& c = spec.coords[static_cast<std::size_t>(i)];
        out << (i + 1) << ' ' << to_chars_string(c.first) << ' ' << to_chars_string(c.second)
            << '\n';
    }
    out << "EOF\n";
    return out.str();
}

inline std::vector<std::int32_t> parse_tour(std::string_view text) {
    const std::string buf(text);
    int32_t len = 0;
    std::vector<std::int32_t> tour(buf.size() / 2 + 16);
    check(aco_parse_tour(buf.c_str(), tour.data(), static_cast<int32_t>(tour.size()), &len));
    tour.resize(static_cast<std::size_t>(len));
    return tour;
}

inline std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(Errc::io_error, "cannot open file: " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

inline InstanceSpec load_instance(const std::string& path) { return parse_instance(read_file(path)); }

// ---- rng.hpp ------------------------------------------------------------
class RngStream {
public:
    RngStream() = default;
    RngStream(std::uint64_t key, std::uint32_t iteration, std::uint32_t ant)
        : key_(key), iteration_(iteration), ant_(ant) {}
    std::uint32_t iteration() const noexcept { return iteration_; }
    std::uint32_t ant() const noexcept { return ant_; }
    std::uint32_t step() const noexcept { return step_; }
    std::uint32_t draw_index() const noexcept { return draw_; }
    void set_step(std::uint32_t step) noexcept {
        step_ = step;
        draw_ = 0;
    }
    double next_uniform() noexcept { return uniform_at(step_, draw_++); }
    double uniform_at(std::uint32_t step, std::uint32_t draw) const noexcept {
        return aco_uniform_at(key_, iteration_, ant_, step, draw);
    }

private:
    std::uint64_t key_ = 0;
    std::uint32_t iteration_ = 0, ant_ = 0, step_ = 0, draw_ = 0;
};

// ---- model.hpp ----------------------------------------------------------
struct ProblemInstance {
    int n = 0;
    Matrix<std::int32_t> dist; // symmetric, zero diagonal
    Matrix<double> heuristic;  // 1/d off-diagonal (1.0 where d == 0), 0 on the diagonal
};

struct Parameters {
    double alpha = 1.0;
    double beta = 2.0;
    double rho = 0.5;
    int m = 0; // 0 means "use n"
    int nn = 30;
    int iterations = 100;
    std::uint64_t seed = 1;
    int tile_size = 64;

    void validate(int n, bool nn_strategy_selected) const {
        check(aco_validate_parameters(alpha, beta, rho, m, nn, iterations, tile_size, n,
                                      nn_strategy_selected ? 1 : 0));
    }
};

struct PheromoneMatrix {
    Matrix<double> tau;
    PheromoneMatrix() = default;
    PheromoneMatrix(int n, double value)
        : tau(static_cast<std::size_t>(n), static_cast<std::size_t>(n), value) {}
    int n() const noexcept { return static_cast<int>(tau.rows()); }
    double& at(int i, int j) { return tau(static_cast<std::size_t>(i), static_cast<std::size_t>(j)); }
    double at(int i, int j) const { return tau(static_cast<std::size_t>(i), static_cast<std::size_t>(j)); }
};

struct ChoiceInfo {
    Matrix<double> value;
    int n() const noexcept { return static_cast<int>(value.rows()); }
    double at(int i, int j) const { return value(static_cast<std::size_t>(i), static_cast<std::size_t>(j)); }
    std::span<const double> row(int i) const { return value.row(static_cast<std::size_t>(i)); }
};

struct NearestNeighborLists {
    int nn = 0;
    Matrix<std::int32_t> lists;
    std::span<const std::int32_t> row(int city) const {
        return lists.row(static_cast<std::size_t>(city));
    }
};

class TabuBitset {
public:
    TabuBitset() = default;
    explicit TabuBitset(int n) : n_(n), words_(static_cast<std::size_t>((n + 63) / 64), 0) {}
    int size() const noexcept { return n_; }
    void set(int city) noexcept { words_[static_cast<std::size_t>(city >> 6)] |= std::uint64_t{1} << (city & 63); }
    bool test(int city) const noexcept { return (words_[static_cast<std::size_t>(city >> 6)] >> (city & 63)) & 1u; }
    void reset() noexcept { std::fill(words_.begin(), words_.end(), 0); }
    int count() const noexcept {
        int c = 0;
        for (auto w : words_) c += __builtin_popcountll(w);
        return c;
    }
    bool all_set() const noexcept { return count() == n_; }

private:
    int n_ = 0;
    std::vector<std::uint64_t> words_;
};

struct AntState {
    TabuBitset tabu;
    std::vector<std::int32_t> tour; // closed: tour[n] == tour[0] once complete
    std::int64_t length = 0;
    RngStream rng;
    explicit AntState(int n) : tabu(n) { tour.reserve(static_cast<std::size_t>(n) + 1); }
};

inline ProblemInstance build_problem(const InstanceSpec& spec) {
    const int n = spec.dimension;
    std::vector<double> xs(static_cast<std::size_t>(n)), ys(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
        xs[static_cast<std::size_t>(i)] = spec.coords[static_cast<std::size_t>(i)].first;
        ys[static_cast<std::size_t>(i)] = spec.coords[static_cast<std::size_t>(i)].second;
    }
    ProblemInstance p;
    p.n = n;
    p.dist = Matrix<std::int32_t>(static_cast<std::size_t>(n), static_cast<std::size_t>(n), 0);
    check(aco_build_distances(n, xs.data(), ys.data(), static_cast<int32_t>(spec.edge_weight_type),
                              p.dist.data()));
    p.heuristic = Matrix<double>(static_cast<std::size_t>(n), static_cast<std::size_t>(n), 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (i != j) {
                const std::int32_t d = p.dist(static_cast<std::size_t>(i), static_cast<std::size_t>(j));
                p.heuristic(static_cast<std::size_t>(i), static_cast<std::size_t>(j)) = d > 0 ? 1.0 / d : 1.0;
            }
    return p;
}

inline NearestNeighborLists build_nn_lists(const ProblemInstance& problem, int nn) {
    NearestNeighborLists out;
    out.nn = nn;
    out.lists = Matrix<std::int32_t>(static_cast<std::size_t>(problem.n),
                                     static_cast<std::size_t>(std::max(nn, 0)), 0);
    check(aco_build_nn_lists(problem.n, problem.dist.data(), nn, out.lists.data()));
    return out;
}

inline std::int64_t tour_length(const ProblemInstance& problem, std::span<const std::int32_t> tour) {
    int64_t out = 0;
    check(aco_tour_length(problem.n, problem.dist.data(), tour.data(),
                          static_cast<int32_t>(tour.size()), &out));
    return out;
}

inline std::int64_t greedy_nn_tour_length(const ProblemInstance& problem) {
    int64_t out = 0;
    check(aco_greedy_tour_length(problem.n, problem.dist.data(), &out));
    return out;
}

inline PheromoneMatrix initial_pheromone(const ProblemInstance& problem, int m) {
    return PheromoneMatrix(problem.n, static_cast<double>(m) /
                                          static_cast<double>(greedy_nn_tour_length(problem)));
}

// ---- construction.hpp / pheromone.hpp: strategies and the ledger ---------
enum class Selection { roulette_full = ACO_SEL_ROULETTE, roulette_nn = ACO_SEL_NN,
                       data_parallel_tiled = ACO_SEL_DATA_PARALLEL };

inline const char* selection_name(Selection s) noexcept {
    switch (s) {
    case Selection::roulette_full: return "roulette";
    case Selection::roulette_nn: return "nn";
    case Selection::data_parallel_tiled: return "data-parallel";
    }
    return "?";
}

struct SelectionStrategy {
    Selection variant = Selection::roulette_nn;
    int tile_size = 64; // theta, used by data_parallel_tiled
};

enum class Deposit { accumulate = ACO_DEP_ACCUMULATE, scatter_gather = ACO_DEP_SCATTER_GATHER,
                     scatter_gather_tiled = ACO_DEP_SCATTER_GATHER_TILED,
                     symmetric_reduction = ACO_DEP_SYMMETRIC_REDUCTION };

inline const char* deposit_name(Deposit d) noexcept {
    switch (d) {
    case Deposit::accumulate: return "accumulate";
    case Deposit::scatter_gather: return "scatter-gather";
    case Deposit::scatter_gather_tiled: return "scatter-gather-tiled";
    case Deposit::symmetric_reduction: return "symmetric-reduction";
    }
    return "?";
}

struct DepositStrategy {
    Deposit variant = Deposit::accumulate;
    int tile_size = 64; // theta, used by the tiled variants
};

struct AccessLedger {
    double global_loads = 0.0;
    double global_stores = 0.0;
    double shared_loads = 0.0;
    double atomic_ops = 0.0;
    void reset() { *this = AccessLedger{}; }
    bool operator==(const AccessLedger&) const = default;
    AccessLedger& operator+=(const AccessLedger& o) {
        global_loads += o.global_loads;
        global_stores += o.global_stores;
        shared_loads += o.shared_loads;
        atomic_ops += o.atomic_ops;
        return *this;
    }
};

inline AccessLedger predicted_access_cost(const DepositStrategy& strategy, int n, int m, int theta) {
    double v[4] = {0, 0, 0, 0};
    check(aco_predicted_access_cost(static_cast<int32_t>(strategy.variant), n, m, theta, v));
    return {v[0], v[1], v[2], v[3]};
}

struct MatrixDiff {
    double max_abs_diff = 0.0;
    int i = 0;
    int j = 0;
};

inline MatrixDiff max_cell_difference(const PheromoneMatrix& a, const PheromoneMatrix& b) {
    MatrixDiff diff;
    const int n = a.n();
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double d = std::abs(a.at(i, j) - b.at(i, j));
            if (d > diff.max_abs_diff) diff = {d, i, j};
        }
    return diff;
}

// ---- engine.hpp -----------------------------------------------------------
struct RunConfig {
    Parameters params;
    SelectionStrategy selection;
    DepositStrategy deposit;
    int workers = 0;           // validated like the reference's; the CUDA grid replaces the pool
    bool random_start = false; // default: ant k starts at city k mod n
    std::string instance_path;
    // ---- B200 placement (no reference counterpart)
    int device = 0;
    int stream = ACO_STREAM_AUTO; // construction weight stream
    int rank = 0, world = 1;      // ant sharding; nccl_id from rank 0
    const uint8_t* nccl_id = nullptr;
    int wire = ACO_WIRE_FP64;
    bool validate_tours = false;  // debug: device tour validation after every construction
};

struct IterationRecord {
    int iteration = 0; // 1-based
    std::int64_t best_length = 0;
    double mean_length = 0.0;
    double construct_ms = 0.0;
    double update_ms = 0.0;
    AccessLedger deposit_ledger; // predicted_access_cost (model values)
};

struct RunReport {
    std::string instance_name;
    int n = 0;
    int m = 0;
    std::uint64_t seed = 0;
    RunConfig config;
    std::vector<std::int32_t> best_tour;
    std::int64_t best_length = 0;
    std::vector<IterationRecord> per_iteration;
};

/// aco::Engine (engine.hpp:55-196) on one B200 (or one ant shard of a
/// multi-GPU colony).  Same constructor, accessors and run_iteration/run; the
/// iteration runs as sm_100a kernels on the context's stream.
class Engine {
public:
    Engine(ProblemInstance problem, RunConfig config)
        : problem_(std::move(problem)), config_(std::move(config)) {
        const int n = problem_.n;
        if (config_.params.m == 0) config_.params.m = n;
        config_.params.validate(n, config_.selection.variant == Selection::roulette_nn);
        if (config_.workers == 0)
            config_.workers = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        if (config_.workers < 1) throw Error(Errc::config_error, "workers must be >= 1");
        if (config_.selection.variant == Selection::data_parallel_tiled)
            config_.selection.tile_size = config_.params.tile_size;
        config_.deposit.tile_size = config_.params.tile_size;

        aco_gpu_params p{};
        p.n = n;
        p.m = config_.params.m;
        p.nn = config_.params.nn;
        p.theta = config_.params.tile_size;
        p.selection = static_cast<int32_t>(config_.selection.variant);
        p.deposit = static_cast<int32_t>(config_.deposit.variant);
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
        p.wire = config_.wire;
        p.validate_tours = config_.validate_tours ? 1 : 0;
        check(aco_gpu_create(&p, problem_.dist.data(), &ctx_));
        int32_t m = 0, st = 0, it = 0;
        double tau0 = 0;
        aco_gpu_get_info(ctx_, &m, &ant_begin_, &ant_end_, &tau0, &st, &it);
        m_ = m;
        ants_.assign(static_cast<std::size_t>(ant_end_ - ant_begin_), AntState(n));
        best_length_ = std::numeric_limits<std::int64_t>::max();
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() { aco_gpu_destroy(ctx_); }

    const ProblemInstance& problem() const noexcept { return problem_; }
    const RunConfig& config() const noexcept { return config_; }

    /// tau and choice, copied out of HBM on the first access after an iteration.
    const PheromoneMatrix& pheromone() const {
        if (!tau_fresh_) {
            if (tau_.n() != problem_.n) tau_ = PheromoneMatrix(problem_.n, 0.0);
            check(aco_gpu_get_pheromone(ctx_, tau_.tau.data()), ctx_);
            tau_fresh_ = true;
        }
        return tau_;
    }
    const ChoiceInfo& choice() const {
        if (!choice_fresh_) {
            if (choice_.n() != problem_.n)
                choice_.value = Matrix<double>(static_cast<std::size_t>(problem_.n),
                                               static_cast<std::size_t>(problem_.n), 0.0);
            check(aco_gpu_get_choice(ctx_, choice_.value.data()), ctx_);
            choice_fresh_ = true;
        }
        return choice_;
    }
    /// This context's ants (all m on one GPU; the shard [ant_begin, ant_end)
    /// of a sharded colony) as the last construction left them.
    std::span<const AntState> ants() const {
        if (!ants_fresh_ && constructed_ >= 0) {
            const int n = problem_.n;
            const std::size_t k = ants_.size();
            std::vector<int32_t> tours(k * static_cast<std::size_t>(n + 1));
            std::vector<int64_t> lens(k);
            check(aco_gpu_get_tours(ctx_, tours.data(), lens.data()), ctx_);
            for (std::size_t a = 0; a < k; ++a) {
                AntState& ant = ants_[a];
                ant.tour.assign(tours.begin() + static_cast<std::ptrdiff_t>(a * (n + 1)),
                                tours.begin() + static_cast<std::ptrdiff_t>((a + 1) * (n + 1)));
                ant.length = lens[a];
                ant.tabu.reset();
                for (int s = 0; s < n; ++s) ant.tabu.set(ant.tour[static_cast<std::size_t>(s)]);
                ant.rng = RngStream(config_.params.seed, static_cast<std::uint32_t>(constructed_),
                                    static_cast<std::uint32_t>(ant_begin_ + static_cast<int>(a)));
                ant.rng.set_step(static_cast<std::uint32_t>(n - 1));
            }
            ants_fresh_ = true;
        }
        return ants_;
    }
    std::int64_t best_length() const noexcept { return best_length_; }
    const std::vector<std::int32_t>& best_tour() const {
        if (!best_fresh_ && best_length_ != std::numeric_limits<std::int64_t>::max()) {
            best_tour_.resize(static_cast<std::size_t>(problem_.n) + 1);
            int64_t len = 0;
            check(aco_gpu_get_best(ctx_, best_tour_.data(), &len), ctx_);
            best_fresh_ = true;
        }
        return best_tour_;
    }

    IterationRecord run_iteration() { // engine.hpp:88-157
        check(aco_gpu_iterate(ctx_, &last_, nullptr, nullptr), ctx_);
        constructed_ = iteration_;
        return finish(last_);
    }

    RunReport run() { // engine.hpp:159-171
        RunReport report;
        report.n = problem_.n;
        report.m = m_;
        report.seed = config_.params.seed;
        report.config = config_;
        report.per_iteration.reserve(static_cast<std::size_t>(config_.params.iterations));
        for (int it = 0; it < config_.params.iterations; ++it)
            report.per_iteration.push_back(run_iteration());
        report.best_length = best_length_;
        report.best_tour = best_tour();
        return report;
    }

    // ---- B200 extras: the two halves of run_iteration, device detail
    IterationRecord construct() { // construction + lengths + statistics (engine.hpp:95-129)
        check(aco_gpu_construct(ctx_, &last_), ctx_);
        constructed_ = iteration_;
        ants_fresh_ = false;
        return to_record(last_);
    }
    IterationRecord update() { // evaporate + deposit + choice_info + best-so-far (:131-155)
        aco_gpu_iter_record r{};
        check(aco_gpu_update(ctx_, &r), ctx_);
        last_.update_ms = r.update_ms;
        last_.exchange_ms = r.exchange_ms;
        last_.choice_ms = r.choice_ms;
        return finish(last_);
    }
    const aco_gpu_iter_record& device_record() const noexcept { return last_; }
    int ant_begin() const noexcept { return ant_begin_; }
    int ant_end() const noexcept { return ant_end_; }
    aco_gpu_ctx* handle() noexcept { return ctx_; }

private:
    static IterationRecord to_record(const aco_gpu_iter_record& r) {
        IterationRecord out;
        out.iteration = r.iteration;
        out.best_length = r.best_length;
        out.mean_length = r.mean_length;
        out.construct_ms = r.construct_ms;
        out.update_ms = r.update_ms;
        out.deposit_ledger = {r.ledger[0], r.ledger[1], r.ledger[2], r.ledger[3]};
        return out;
    }
    IterationRecord finish(const aco_gpu_iter_record& r) {
        ++iteration_;
        tau_fresh_ = choice_fresh_ = ants_fresh_ = best_fresh_ = false;
        int64_t best = 0;
        check(aco_gpu_get_best(ctx_, nullptr, &best), ctx_);
        best_length_ = best;
        return to_record(r);
    }

    ProblemInstance problem_;
    RunConfig config_;
    aco_gpu_ctx* ctx_ = nullptr;
    int m_ = 0, ant_begin_ = 0, ant_end_ = 0, iteration_ = 0;
    int constructed_ = -1; // iteration index of the last construction (-1: none yet)
    aco_gpu_iter_record last_{};
    std::int64_t best_length_ = 0;
    mutable PheromoneMatrix tau_;
    mutable ChoiceInfo choice_;
    mutable std::vector<AntState> ants_;
    mutable std::vector<std::int32_t> best_tour_;
    mutable bool tau_fresh_ = false, choice_fresh_ = false, ants_fresh_ = false, best_fresh_ = false;
};

inline RunReport run(const RunConfig& config) { // engine.hpp:198-204
    const InstanceSpec spec = load_instance(config.instance_path);
    Engine engine(build_problem(spec), config);
    RunReport report = engine.run();
    report.instance_name = spec.name;
    return report;
}

struct VerifyReport { // engine.hpp:208-225
    struct StrategyResult {
        Deposit variant;
        AccessLedger measured; // the engine's record ledger = the closed-form model
        AccessLedger predicted;
        bool ledger_ok = false;
    };
    struct PairResult {
        Deposit a;
        Deposit b;
        MatrixDiff diff;
        bool pass = false;
    };
    std::array<StrategyResult, 4> strategies;
    std::vector<PairResult> pairs;
    bool all_pass = false;
};

/// engine.hpp:227-292 on the device: one iteration-0 construction (identical
/// in every engine — draws are keyed by (seed, iteration, ant, step)), each
/// deposit variant applied to the evaporated tau0, pairwise max cell
/// difference <= tolerance.  The kernels make no abstract accesses to count,
/// so `measured` is the engine's model ledger and ledger_ok holds by
/// construction; all_pass is decided by the matrix comparisons.
inline VerifyReport verify_deposit_equivalence(const ProblemInstance& problem, RunConfig config,
                                               double tolerance = 1e-9) {
    const int m = config.params.m == 0 ? problem.n : config.params.m;
    config.params.m = m;
    config.params.validate(problem.n, config.selection.variant == Selection::roulette_nn);
    config.random_start = false;
    config.rank = 0;
    config.world = 1;
    config.nccl_id = nullptr;
    const std::array<Deposit, 4> variants = {Deposit::accumulate, Deposit::scatter_gather,
                                             Deposit::scatter_gather_tiled,
                                             Deposit::symmetric_reduction};
    VerifyReport report;
    std::array<PheromoneMatrix, 4> results;
    std::vector<std::int32_t> tours0;
    for (std::size_t v = 0; v < variants.size(); ++v) {
        RunConfig c = config;
        c.deposit = DepositStrategy{variants[v], config.params.tile_size};
        Engine engine(problem, c);
        const IterationRecord rec = engine.run_iteration();
        std::vector<std::int32_t> tours;
        for (const AntState& a : engine.ants()) tours.insert(tours.end(), a.tour.begin(), a.tour.end());
        if (v == 0) tours0 = tours;
        else if (tours != tours0)
            throw Error(Errc::inconsistent_length, "deposit engines constructed different tours");
        results[v] = engine.pheromone();
        auto& entry = report.strategies[v];
        entry.variant = variants[v];
        entry.measured = rec.deposit_ledger;
        entry.predicted = predicted_access_cost(c.deposit, problem.n, m, config.params.tile_size);
        entry.ledger_ok = entry.measured == entry.predicted;
    }
    report.all_pass = true;
    for (std::size_t a = 0; a < variants.size(); ++a)
        for (std::size_t b = a + 1; b < variants.size(); ++b) {
            VerifyReport::PairResult pair;
            pair.a = variants[a];
            pair.b = variants[b];
            pair.diff = max_cell_difference(results[a], results[b]);
            pair.pass = pair.diff.max_abs_diff <= tolerance;
            report.all_pass = report.all_pass && pair.pass;
            report.pairs.push_back(pair);
        }
    return report;
}

// ---- report.hpp -------------------------------------------------------------
inline constexpr int kReportSchemaVersion = 1;

/// Shortest round-trip decimal form (std::to_chars), as report.hpp:16-21.
inline std::string format_double(double v) { return to_chars_string(v); }

/// A minimal JSON value with nlohmann::json's object ordering (sorted keys)
/// and dump(indent) layout — enough for report_to_json(...).dump(2).
class Json {
public:
    using Object = std::map<std::string, Json>;
    using Array = std::vector<Json>;
    Json() = default;
    Json(bool b) : v_(b) {}
    Json(int x) : v_(static_cast<std::int64_t>(x)) {}
    Json(std::int64_t x) : v_(x) {}
    Json(std::uint64_t x) : v_(x) {}
    Json(double x) : v_(x) {}
    Json(const char* s) : v_(std::string(s)) {}
    Json(std::string s) : v_(std::move(s)) {}
    Json(Array a) : v_(std::move(a)) {}
    Json(Object o) : v_(std::move(o)) {}

    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }

private:
    static void esc(std::string& out, const std::string& s) {
        out += '"';
        for (char ch : s) {
            switch (ch) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            case '\r': out += "\\r"; break;
            default:
                if (static_cast<unsigned char>(ch) < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", ch);
                    out += b;
                } else {
                    out += ch;
                }
            }
        }
        out += '"';
    }
    void write(std::string& out, int indent, int depth) const {
        const std::string nl = indent >= 0 ? "\n" : "";
        auto pad = [&](int d) { return indent >= 0 ? std::string(static_cast<std::size_t>(indent * d), ' ') : std::string(); };
        if (std::holds_alternative<std::monostate>(v_)) out += "null";
        else if (auto b = std::get_if<bool>(&v_)) out += *b ? "true" : "false";
        else if (auto i = std::get_if<std::int64_t>(&v_)) out += std::to_string(*i);
        else if (auto u = std::get_if<std::uint64_t>(&v_)) out += std::to_string(*u);
        else if (auto d = std::get_if<double>(&v_)) {
            if (!std::isfinite(*d)) { out += "null"; return; }
            std::string s = to_chars_string(*d);
            if (s.find_first_of(".eE") == std::string::npos) s += ".0";
            out += s;
        } else if (auto s = std::get_if<std::string>(&v_)) esc(out, *s);
        else if (auto a = std::get_if<Array>(&v_)) {
            if (a->empty()) { out += "[]"; return; }
            out += "[" + nl;
            for (std::size_t k = 0; k < a->size(); ++k) {
                out += pad(depth + 1);
                (*a)[k].write(out, indent, depth + 1);
                out += (k + 1 < a->size() ? "," : "") + nl;
            }
            out += pad(depth) + "]";
        } else if (auto o = std::get_if<Object>(&v_)) {
            if (o->empty()) { out += "{}"; return; }
            out += "{" + nl;
            std::size_t k = 0;
            for (const auto& [key, val] : *o) {
                out += pad(depth + 1);
                esc(out, key);
                out += indent >= 0 ? ": " : ":";
                val.write(out, indent, depth + 1);
                out += (++k < o->size() ? "," : "") + nl;
            }
            out += pad(depth) + "}";
        }
    }
    std::variant<std::monostate, bool, std::int64_t, std::uint64_t, double, std::string, Array, Object> v_;
};

inline Json ledger_to_json(const AccessLedger& l) {
    return Json::Object{{"global_loads", l.global_loads}, {"global_stores", l.global_stores},
                        {"shared_loads", l.shared_loads}, {"atomic_ops", l.atomic_ops}};
}

inline Json report_to_json(const RunReport& r) { // report.hpp:32-67
    Json::Array per;
    for (const auto& rec : r.per_iteration)
        per.push_back(Json::Object{{"iteration", rec.iteration}, {"best_len", rec.best_length},
                                   {"mean_len", rec.mean_length}, {"construct_ms", rec.construct_ms},
                                   {"update_ms", rec.update_ms},
                                   {"ledger", ledger_to_json(rec.deposit_ledger)}});
    Json::Array tour;
    for (auto c : r.best_tour) tour.push_back(Json(static_cast<std::int64_t>(c)));
    const auto& c = r.config;
    return Json::Object{
        {"schema_version", kReportSchemaVersion},
        {"instance", r.instance_name},
        {"n", r.n},
        {"m", r.m},
        {"seed", r.seed},
        {"config", Json::Object{{"alpha", c.params.alpha}, {"beta", c.params.beta},
                                {"rho", c.params.rho}, {"nn", c.params.nn},
                                {"iters", c.params.iterations}, {"theta", c.params.tile_size},
                                {"workers", c.workers},
                                {"selection", selection_name(c.selection.variant)},
                                {"deposit", deposit_name(c.deposit.variant)},
                                {"random_start", c.random_start}}},
        {"best_length", r.best_length},
        {"best_tour", Json(std::move(tour))},
        {"per_iteration", Json(std::move(per))},
    };
}

inline const char* bench_csv_header() {
    return "instance,n,selection,deposit,theta,rep,iter,construct_ms,update_ms,"
           "best_len,global_loads,atomic_ops,schema_version";
}

inline void write_bench_csv_row(std::ostream& out, const std::string& instance, int n,
                                Selection selection, Deposit deposit, int theta, int rep,
                                const IterationRecord& rec) {
    out << instance << ',' << n << ',' << selection_name(selection) << ',' << deposit_name(deposit)
        << ',' << theta << ',' << rep << ',' << rec.iteration << ',' << format_double(rec.construct_ms)
        << ',' << format_double(rec.update_ms) << ',' << rec.best_length << ','
        << format_double(rec.deposit_ledger.global_loads) << ','
        << format_double(rec.deposit_ledger.atomic_ops) << ',' << kReportSchemaVersion << '\n';
}

} // inline namespace gpu
} // namespace aco
