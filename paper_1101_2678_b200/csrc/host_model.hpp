// Host-side model pieces shared by the C ABI (see host_model.cpp).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace acob200 {

// Same order as aco::Errc (errors.hpp:8-27); status = 1 + code.
enum class Errc {
    missing_field, unsupported_edge_weight_type, malformed_coord, dimension_mismatch,
    index_out_of_range, overflow, invalid_length, not_a_permutation, not_closed, all_visited,
    inconsistent_length, io_error, config_error
};

struct ModelError : std::runtime_error {
    ModelError(Errc c, const std::string& msg) : std::runtime_error(msg), code(c) {}
    Errc code;
};

struct Instance {
    std::string name;
    int dimension = 0;
    int edge_weight_type = 0; // 0 EUC_2D, 1 CEIL_2D, 2 ATT
    std::vector<double> xs, ys;
};

struct Config {
    int n = 0, m = 0, nn = 30, theta = 64, selection = 0, deposit = 0, iterations = 1;
    double alpha = 1.0, beta = 2.0, rho = 0.5;
};

void parse_instance(std::string_view text, Instance& out);
std::vector<int32_t> parse_tour(std::string_view text);
int32_t edge_weight(int ewt, double xi, double yi, double xj, double yj);
int64_t build_distances(int n, const double* xs, const double* ys, int ewt, int32_t* dist);
void build_nn_lists(int n, const int32_t* dist, int nn, int32_t* out);
int64_t greedy_tour_length(int n, const int32_t* dist);
int64_t tour_length(int n, const int32_t* dist, const int32_t* tour, int len);
void validate(const Config& c);
std::vector<double> eta_beta_table(int64_t max_d, double beta);

// The tables of the host libm's pow (glibc __pow_log_data / __exp_data), read
// out of the loaded libm.so so the device can replay pow(tau, alpha) exactly
// (libm_pow.cuh).  Layout as the FMA build of glibc 2.28+ reads them.
struct LibmPowTables {
    // __pow_log_data: ln2hi, ln2lo, A[0..6], tab[128] = {invc, pad, logc, logctail}
    double ln2hi, ln2lo, A[7];
    double ltab[128 * 4];
    // __exp_data: InvLn2N, Shift, NegLn2hiN, NegLn2loN, C2..C5, tab[2*128] = {tail, sbits}
    double invln2N, shift, negln2hiN, negln2loN, C[4];
    uint64_t etab[256];
};
// false (with the reason) when the loaded libm does not carry them
bool read_libm_pow_tables(LibmPowTables& out, std::string& why);
// the host libm's own pow (what compute_choice_info calls, model.hpp:167)
double host_pow(double x, double y);
void predicted_access_cost(int deposit, int n, int m, int theta, double out[4]);

} // namespace acob200
