// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI harness around the UNMODIFIED reference headers
// (/root/reference/proj/include/aco/*.hpp), compiled with the reference's own
// flags (g++ -std=c++20 -O3 -DNDEBUG, no -march; CMakeLists.txt:1-22) by
// oracle/Makefile into oracle/_ref/libaco_ref.so.  Only tests/, smoke() and
// bench.py's reference / cpu_baseline legs may load it, and only as the
// checker or the timed CPU baseline.
//
// Every entry point returns 0 on success or 1 + (int)aco::Errc on an
// aco::Error (errors.hpp:8-27), 100 on any other exception; the message is
// kept in ref_last_error().

#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <memory>
#include <string>
#include <vector>

#include "aco/engine.hpp"
#ifdef ACO_REF_WITH_JSON
#include "aco/report.hpp" // needs nlohmann/json.hpp (vendored in the image's cudnn_frontend)
#endif

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const aco::Error& e) {
        g_err = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 100;
    }
}

aco::InstanceSpec make_spec(int n, const double* xs, const double* ys, int ewt) {
    aco::InstanceSpec s;
    s.name = "harness";
    s.dimension = n;
    s.edge_weight_type = static_cast<aco::EdgeWeightType>(ewt);
    s.coords.resize(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) s.coords[static_cast<std::size_t>(i)] = {xs[i], ys[i]};
    return s;
}

struct RefEngine {
    std::unique_ptr<aco::Engine> engine;
    double last_choice_ms = 0.0;
};

aco::ProblemInstance problem_from_dist(int n, const int32_t* dist) {
    aco::ProblemInstance p;
    p.n = n;
    p.dist = aco::Matrix<std::int32_t>(n, n, 0);
    p.heuristic = aco::Matrix<double>(n, n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (i == j) continue;
            const int32_t d = dist[(size_t)i * n + j];
            p.dist(i, j) = d;
            p.heuristic(i, j) = d > 0 ? 1.0 / d : 1.0;
        }
    return p;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- rng.hpp -------------------------------------------------------------
void ref_philox_block(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t key,
                      uint32_t out[4]) {
    const aco::philox::Block b = aco::philox::permute({{c0, c1, c2, c3}}, key);
    std::memcpy(out, b.v, sizeof(b.v));
}

double ref_uniform_at(uint64_t seed, uint32_t iteration, uint32_t ant, uint32_t step,
                      uint32_t draw) {
    return aco::RngStream(seed, iteration, ant).uniform_at(step, draw);
}

// ---- tsplib.hpp ----------------------------------------------------------
// Parses TSPLIB text; writes dimension/ewt, then (if xs != nullptr and cap >=
// dimension) the coords.
int ref_parse_instance(const char* text, int* dimension, int* ewt, double* xs, double* ys,
                       int cap) {
    return guarded([&] {
        const aco::InstanceSpec s = aco::parse_instance(text);
        *dimension = s.dimension;
        *ewt = static_cast<int>(s.edge_weight_type);
        if (xs && cap >= s.dimension)
            for (int i = 0; i < s.dimension; ++i) {
                xs[i] = s.coords[(size_t)i].first;
                ys[i] = s.coords[(size_t)i].second;
            }
    });
}

int ref_parse_tour(const char* text, int32_t* out, int cap, int* len) {
    return guarded([&] {
        const auto t = aco::parse_tour(text);
        *len = static_cast<int>(t.size());
        for (int i = 0; i < (int)t.size() && i < cap; ++i) out[i] = t[(size_t)i];
    });
}

// ---- model.hpp -----------------------------------------------------------
int ref_build_problem(int n, const double* xs, const double* ys, int ewt, int32_t* dist,
                      double* heuristic) {
    return guarded([&] {
        const aco::ProblemInstance p = aco::build_problem(make_spec(n, xs, ys, ewt));
        std::memcpy(dist, p.dist.data(), sizeof(int32_t) * (size_t)n * n);
        if (heuristic) std::memcpy(heuristic, p.heuristic.data(), sizeof(double) * (size_t)n * n);
    });
}

int ref_compute_choice_info(int n, const int32_t* dist, const double* tau, double alpha,
                            double beta, double* choice) {
    return guarded([&] {
        const aco::ProblemInstance p = problem_from_dist(n, dist);
        aco::PheromoneMatrix t(n, 0.0);
        std::memcpy(t.tau.data(), tau, sizeof(double) * (size_t)n * n);
        const aco::ChoiceInfo c = aco::compute_choice_info(t, p, alpha, beta);
        std::memcpy(choice, c.value.data(), sizeof(double) * (size_t)n * n);
    });
}

int ref_build_nn_lists(int n, const int32_t* dist, int nn, int32_t* out) {
    return guarded([&] {
        const aco::NearestNeighborLists l = aco::build_nn_lists(problem_from_dist(n, dist), nn);
        std::memcpy(out, l.lists.data(), sizeof(int32_t) * (size_t)n * nn);
    });
}

int ref_tour_length(int n, const int32_t* dist, const int32_t* tour, int len, int64_t* out) {
    return guarded([&] {
        *out = aco::tour_length(problem_from_dist(n, dist),
                                std::span<const int32_t>(tour, (size_t)len));
    });
}

int ref_initial_pheromone(int n, const int32_t* dist, int m, double* tau0) {
    return guarded([&] {
        const aco::PheromoneMatrix t = aco::initial_pheromone(problem_from_dist(n, dist), m);
        *tau0 = t.at(0, 0);
    });
}

// ---- construction.hpp ----------------------------------------------------
// Constructs the tours of ants [k0, k1) of `iteration` from a given choice
// matrix (selection 0 roulette, 1 nn, 2 data-parallel), exactly as the engine
// loop does (engine.hpp:98-114).  tours: (k1-k0) x (n+1), lengths: (k1-k0).
int ref_construct(int n, const int32_t* dist, const double* choice, const int32_t* nn_lists,
                  int nn, int selection, int theta, uint64_t seed, uint32_t iteration,
                  int random_start, int k0, int k1, int32_t* tours, int64_t* lengths) {
    return guarded([&] {
        const aco::ProblemInstance p = problem_from_dist(n, dist);
        aco::ChoiceInfo c;
        c.value = aco::Matrix<double>(n, n, 0.0);
        std::memcpy(c.value.data(), choice, sizeof(double) * (size_t)n * n);
        aco::NearestNeighborLists lists;
        if (selection == 1) {
            lists.nn = nn;
            lists.lists = aco::Matrix<int32_t>(n, nn, 0);
            std::memcpy(lists.lists.data(), nn_lists, sizeof(int32_t) * (size_t)n * nn);
        }
        aco::SelectionStrategy sel;
        sel.variant = static_cast<aco::Selection>(selection);
        sel.tile_size = theta;
        aco::AntState ant(n);
        for (int k = k0; k < k1; ++k) {
            ant.rng = aco::RngStream(seed, iteration, (uint32_t)k);
            int start;
            if (random_start) {
                start = static_cast<int>(ant.rng.uniform_at(0, 0) * n);
                if (start >= n) start = n - 1;
            } else {
                start = k % n;
            }
            aco::construct_tour(p, c, selection == 1 ? &lists : nullptr, sel, ant, start);
            std::memcpy(tours + (size_t)(k - k0) * (n + 1), ant.tour.data(),
                        sizeof(int32_t) * (size_t)(n + 1));
            lengths[k - k0] = ant.length;
        }
    });
}

// ---- pheromone.hpp -------------------------------------------------------
// evaporate + TourBuffer::make + apply_deposit, i.e. the update window of
// engine.hpp:134-138, on a caller-supplied tau (in place).
int ref_update(int n, const int32_t* dist, int m, const int32_t* tours, const int64_t* lengths,
               double rho, int deposit, int theta, int workers, double* tau,
               double* ledger4) {
    return guarded([&] {
        const aco::ProblemInstance p = problem_from_dist(n, dist);
        aco::PheromoneMatrix t(n, 0.0);
        std::memcpy(t.tau.data(), tau, sizeof(double) * (size_t)n * n);
        std::vector<std::vector<int32_t>> tv((size_t)m);
        for (int k = 0; k < m; ++k)
            tv[(size_t)k].assign(tours + (size_t)k * (n + 1), tours + (size_t)(k + 1) * (n + 1));
        std::unique_ptr<aco::ThreadPool> pool;
        if (workers != 1) pool = std::make_unique<aco::ThreadPool>(
                              workers == 0 ? aco::ThreadPool::hardware_workers() : workers);
        aco::AccessLedger ev, led;
        aco::evaporate(t, rho, ev, pool.get());
        const aco::TourBuffer buf = aco::TourBuffer::make(
            p, tv, std::span<const int64_t>(lengths, (size_t)m), theta);
        aco::apply_deposit({static_cast<aco::Deposit>(deposit), theta}, t, buf, led, pool.get());
        std::memcpy(tau, t.tau.data(), sizeof(double) * (size_t)n * n);
        if (ledger4) {
            ledger4[0] = led.global_loads;
            ledger4[1] = led.global_stores;
            ledger4[2] = led.shared_loads;
            ledger4[3] = led.atomic_ops;
        }
    });
}

void ref_predicted_access_cost(int deposit, int n, int m, int theta, double* ledger4) {
    const aco::AccessLedger l =
        aco::predicted_access_cost({static_cast<aco::Deposit>(deposit), theta}, n, m, theta);
    ledger4[0] = l.global_loads;
    ledger4[1] = l.global_stores;
    ledger4[2] = l.shared_loads;
    ledger4[3] = l.atomic_ops;
}

// ---- engine.hpp ----------------------------------------------------------
int ref_engine_create(int n, const double* xs, const double* ys, int ewt, double alpha,
                      double beta, double rho, int m, int nn, uint64_t seed, int theta,
                      int selection, int deposit, int workers, int random_start,
                      void** out) {
    return guarded([&] {
        aco::RunConfig cfg;
        cfg.params.alpha = alpha;
        cfg.params.beta = beta;
        cfg.params.rho = rho;
        cfg.params.m = m;
        cfg.params.nn = nn;
        cfg.params.seed = seed;
        cfg.params.tile_size = theta;
        cfg.selection.variant = static_cast<aco::Selection>(selection);
        cfg.selection.tile_size = theta;
        cfg.deposit.variant = static_cast<aco::Deposit>(deposit);
        cfg.deposit.tile_size = theta;
        cfg.workers = workers;
        cfg.random_start = random_start != 0;
        auto* e = new RefEngine;
        try {
            e->engine = std::make_unique<aco::Engine>(
                aco::build_problem(make_spec(n, xs, ys, ewt)), cfg);
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    });
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_engine_m(void* h) { return static_cast<RefEngine*>(h)->engine->config().params.m; }

int ref_engine_workers(void* h) { return static_cast<RefEngine*>(h)->engine->config().workers; }

// rec6 = {best_length, mean_length, construct_ms, update_ms, choice_ms(wall of
// the whole call minus the two windows), ledger_atomic_ops}
int ref_engine_iterate(void* h, double* rec6) {
    return guarded([&] {
        auto* e = static_cast<RefEngine*>(h);
        const auto t0 = std::chrono::steady_clock::now();
        const aco::IterationRecord r = e->engine->run_iteration();
        const double wall =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                .count();
        rec6[0] = static_cast<double>(r.best_length);
        rec6[1] = r.mean_length;
        rec6[2] = r.construct_ms;
        rec6[3] = r.update_ms;
        rec6[4] = wall - r.construct_ms - r.update_ms;
        rec6[5] = r.deposit_ledger.atomic_ops;
    });
}

void ref_engine_tau(void* h, double* out) {
    const auto& t = static_cast<RefEngine*>(h)->engine->pheromone();
    std::memcpy(out, t.tau.data(), sizeof(double) * t.tau.size());
}

void ref_engine_choice(void* h, double* out) {
    const auto& c = static_cast<RefEngine*>(h)->engine->choice();
    std::memcpy(out, c.value.data(), sizeof(double) * c.value.size());
}

void ref_engine_tours(void* h, int32_t* tours, int64_t* lengths) {
    auto* e = static_cast<RefEngine*>(h);
    const int n = e->engine->problem().n;
    const auto ants = e->engine->ants();
    for (size_t k = 0; k < ants.size(); ++k) {
        if (tours && ants[k].tour.size() == (size_t)n + 1)
            std::memcpy(tours + k * (n + 1), ants[k].tour.data(), sizeof(int32_t) * (n + 1));
        if (lengths) lengths[k] = ants[k].length;
    }
}

int64_t ref_engine_best(void* h, int32_t* tour) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& b = e->engine->best_tour();
    if (tour) std::memcpy(tour, b.data(), sizeof(int32_t) * b.size());
    return e->engine->best_length();
}

// verify_deposit_equivalence (engine.hpp:227-295): returns all_pass and the
// worst pairwise max_abs_diff.
int ref_verify_deposit_equivalence(int n, const double* xs, const double* ys, int ewt,
                                   int m, int selection, int nn, int theta, uint64_t seed,
                                   double tolerance, int* all_pass, double* worst) {
    return guarded([&] {
        aco::RunConfig cfg;
        cfg.params.m = m;
        cfg.params.nn = nn;
        cfg.params.seed = seed;
        cfg.params.tile_size = theta;
        cfg.selection.variant = static_cast<aco::Selection>(selection);
        const auto rep = aco::verify_deposit_equivalence(
            aco::build_problem(make_spec(n, xs, ys, ewt)), cfg, tolerance);
        *all_pass = rep.all_pass ? 1 : 0;
        double w = 0.0;
        for (const auto& p : rep.pairs) w = std::max(w, p.diff.max_abs_diff);
        *worst = w;
    });
}

#ifdef ACO_REF_WITH_JSON
void ref_format_double(double v, char* out) {
    const std::string s = aco::format_double(v);
    std::memcpy(out, s.c_str(), s.size() + 1);
}

#endif

} // extern "C"
