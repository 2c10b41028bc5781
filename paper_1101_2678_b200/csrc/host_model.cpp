// Host-side model of the B200 Ant System engine: TSPLIB parsing, integer
// edge weights, nearest-neighbour lists, the greedy tour that seeds tau0, the
// eta^beta table, parameter validation and the closed-form access ledger.
//
// These run once per instance on the host (they are not on the iteration
// hot path) and restate the reference's semantics so an aco:: caller sees
// the same values and the same error codes:
//   parse_instance      tsplib.hpp:76-186      edge_weight   tsplib.hpp:190-210
//   parse_tour          tsplib.hpp:238-270     build_problem model.hpp:125-152
//   build_nn_lists      model.hpp:177-202      tour_length   model.hpp:205-226
//   greedy tour / tau0  model.hpp:230-262      validate      model.hpp:39-53
//   predicted_access_cost pheromone.hpp:366-397
// Compiled with -ffp-contract=off and no -march so sqrt/pow/divisions round
// exactly like the reference build (CMakeLists.txt:1-22).
#include "host_model.hpp"

#include <dlfcn.h>
#include <link.h>

#include <cstring>
#include <fstream>
#include <iterator>

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <string_view>
#include <vector>

namespace acob200 {

namespace {

bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

std::string_view strip(std::string_view s) {
    size_t a = 0, b = s.size();
    while (a < b && is_blank(s[a])) ++a;
    while (b > a && is_blank(s[b - 1])) --b;
    return s.substr(a, b - a);
}

std::vector<std::string_view> tokens(std::string_view s) {
    std::vector<std::string_view> out;
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && is_blank(s[i])) ++i;
        size_t j = i;
        while (j < s.size() && !is_blank(s[j])) ++j;
        if (j > i) out.emplace_back(s.substr(i, j - i));
        i = j;
    }
    return out;
}

template <class T>
bool full_number(std::string_view s, T& v) {
    const char* e = s.data() + s.size();
    auto r = std::from_chars(s.data(), e, v);
    return r.ec == std::errc{} && r.ptr == e;
}

// Line cursor over a text buffer; every line comes back stripped.
struct Lines {
    std::string_view text;
    size_t pos = 0;
    bool next(std::string_view& line) {
        if (pos >= text.size()) return false;
        size_t nl = text.find('\n', pos);
        if (nl == std::string_view::npos) nl = text.size();
        line = strip(text.substr(pos, nl - pos));
        pos = nl + 1;
        return true;
    }
};

int tsplib_nint(double x) { return static_cast<int>(x + 0.5); }

} // namespace

void parse_instance(std::string_view text, Instance& spec) {
    spec = Instance{};
    bool got_name = false, got_dim = false, got_ewt = false, got_coords = false;
    Lines lines{text};
    std::string_view line;
    while (lines.next(line)) {
        if (line.empty()) continue;
        if (line == "EOF") break;
        if (line == "NODE_COORD_SECTION") {
            if (!got_dim) throw ModelError(Errc::missing_field,
                                           "DIMENSION must precede NODE_COORD_SECTION");
            const int n = spec.dimension;
            spec.xs.assign(n, 0.0);
            spec.ys.assign(n, 0.0);
            std::vector<char> seen(n, 0);
            int have = 0;
            while (have < n) {
                if (!lines.next(line) || line == "EOF")
                    throw ModelError(Errc::dimension_mismatch,
                                     "NODE_COORD_SECTION ended after " + std::to_string(have) +
                                         " of " + std::to_string(n) + " coords");
                if (line.empty()) continue;
                const auto tok = tokens(line);
                if (tok.size() != 3)
                    throw ModelError(Errc::malformed_coord,
                                     "coord line needs <id> <x> <y>: '" + std::string(line) + "'");
                long id = 0;
                double x = 0, y = 0;
                if (!full_number(tok[0], id) || !full_number(tok[1], x) || !full_number(tok[2], y))
                    throw ModelError(Errc::malformed_coord,
                                     "non-numeric coord line: '" + std::string(line) + "'");
                if (id < 1 || id > n)
                    throw ModelError(Errc::malformed_coord, "node id " + std::to_string(id) +
                                                                " outside 1.." + std::to_string(n));
                if (seen[id - 1])
                    throw ModelError(Errc::malformed_coord, "duplicate node id " + std::to_string(id));
                seen[id - 1] = 1;
                spec.xs[id - 1] = x;
                spec.ys[id - 1] = y;
                ++have;
            }
            // Trailing coordinate-shaped lines mean DIMENSION undercounts.
            while (lines.next(line)) {
                if (line.empty()) continue;
                if (line == "EOF") break;
                if (tokens(line).size() == 3)
                    throw ModelError(Errc::dimension_mismatch,
                                     "more coord lines than DIMENSION=" + std::to_string(n));
                break;
            }
            got_coords = true;
            break;
        }
        if (line == "EDGE_WEIGHT_SECTION")
            throw ModelError(Errc::unsupported_edge_weight_type,
                             "explicit edge weight matrices are not supported");
        const size_t colon = line.find(':');
        if (colon == std::string_view::npos) continue;
        const std::string_view key = strip(line.substr(0, colon));
        const std::string_view val = strip(line.substr(colon + 1));
        if (key == "NAME") {
            spec.name = std::string(val);
            got_name = true;
        } else if (key == "DIMENSION") {
            long d = 0;
            if (!full_number(val, d))
                throw ModelError(Errc::missing_field,
                                 "DIMENSION value is not an integer: '" + std::string(val) + "'");
            if (d < 2)
                throw ModelError(Errc::dimension_mismatch,
                                 "DIMENSION must be at least 2, got " + std::to_string(d));
            spec.dimension = static_cast<int>(d);
            got_dim = true;
        } else if (key == "EDGE_WEIGHT_TYPE") {
            if (val == "EUC_2D") spec.edge_weight_type = 0;
            else if (val == "CEIL_2D") spec.edge_weight_type = 1;
            else if (val == "ATT") spec.edge_weight_type = 2;
            else
                throw ModelError(Errc::unsupported_edge_weight_type,
                                 "unsupported EDGE_WEIGHT_TYPE '" + std::string(val) + "'");
            got_ewt = true;
        }
    }
    if (!got_name) throw ModelError(Errc::missing_field, "missing NAME header");
    if (!got_dim) throw ModelError(Errc::missing_field, "missing DIMENSION header");
    if (!got_ewt) throw ModelError(Errc::missing_field, "missing EDGE_WEIGHT_TYPE header");
    if (!got_coords) throw ModelError(Errc::missing_field, "missing NODE_COORD_SECTION");
}

std::vector<int32_t> parse_tour(std::string_view text) {
    std::vector<int32_t> tour;
    bool in_section = false;
    size_t pos = 0;
    while (pos <= text.size()) {
        size_t nl = text.find('\n', pos);
        if (nl == std::string_view::npos) nl = text.size();
        const std::string_view line = strip(text.substr(pos, nl - pos));
        pos = nl + 1;
        if (line.empty()) {
            if (pos > text.size()) break;
            continue;
        }
        if (!in_section) {
            in_section = (line == "TOUR_SECTION");
            if (pos > text.size()) break;
            continue;
        }
        if (line == "-1" || line == "EOF") break;
        for (auto tok : tokens(line)) {
            long id = 0;
            if (!full_number(tok, id))
                throw ModelError(Errc::malformed_coord,
                                 "non-numeric tour entry: '" + std::string(tok) + "'");
            if (id == -1) return tour;
            tour.push_back(static_cast<int32_t>(id - 1));
        }
        if (pos > text.size()) break;
    }
    if (!in_section) throw ModelError(Errc::missing_field, "missing TOUR_SECTION");
    return tour;
}

int32_t edge_weight(int ewt, double xi, double yi, double xj, double yj) {
    const double dx = xi - xj;
    const double dy = yi - yj;
    const double sq = dx * dx + dy * dy; // two roundings, never contracted
    if (ewt == 0) return tsplib_nint(std::sqrt(sq));
    if (ewt == 1) return static_cast<int32_t>(std::ceil(std::sqrt(sq)));
    const double r = std::sqrt(sq / 10.0); // ATT pseudo-Euclidean
    const int t = tsplib_nint(r);
    return (t < r) ? t + 1 : t;
}

int64_t build_distances(int n, const double* xs, const double* ys, int ewt, int32_t* dist) {
    int64_t max_d = 0;
    for (int i = 0; i < n; ++i) {
        int32_t* row = dist + static_cast<size_t>(i) * n;
        row[i] = 0;
        for (int j = i + 1; j < n; ++j) {
            const int32_t d = edge_weight(ewt, xs[i], ys[i], xs[j], ys[j]);
            if (d < 0) throw ModelError(Errc::overflow, "negative distance computed");
            row[j] = d;
            dist[static_cast<size_t>(j) * n + i] = d;
            max_d = std::max<int64_t>(max_d, d);
        }
    }
    if (max_d > 0 && static_cast<int64_t>(n) > std::numeric_limits<int64_t>::max() / max_d)
        throw ModelError(Errc::overflow, "tour lengths would overflow 64-bit range");
    return max_d;
}

void build_nn_lists(int n, const int32_t* dist, int nn, int32_t* out) {
    if (!(nn >= 1 && nn < n))
        throw ModelError(Errc::invalid_length, "nn list length must satisfy 1 <= nn < n");
    std::vector<int32_t> cand(static_cast<size_t>(n) - 1);
    for (int i = 0; i < n; ++i) {
        const int32_t* row = dist + static_cast<size_t>(i) * n;
        size_t k = 0;
        for (int j = 0; j < n; ++j)
            if (j != i) cand[k++] = j;
        // (distance, index) is a strict total order, so the first nn of a
        // partial sort equal the first nn of the full order.
        std::partial_sort(cand.begin(), cand.begin() + nn, cand.end(),
                          [row](int32_t a, int32_t b) {
                              return row[a] != row[b] ? row[a] < row[b] : a < b;
                          });
        std::copy(cand.begin(), cand.begin() + nn, out + static_cast<size_t>(i) * nn);
    }
}

int64_t greedy_tour_length(int n, const int32_t* dist) {
    std::vector<char> seen(n, 0);
    int cur = 0;
    seen[0] = 1;
    int64_t total = 0;
    for (int step = 1; step < n; ++step) {
        const int32_t* row = dist + static_cast<size_t>(cur) * n;
        int best = -1;
        int32_t best_d = std::numeric_limits<int32_t>::max();
        for (int j = 0; j < n; ++j)
            if (!seen[j] && row[j] < best_d) {
                best_d = row[j];
                best = j;
            }
        total += best_d;
        seen[best] = 1;
        cur = best;
    }
    return total + dist[static_cast<size_t>(cur) * n];
}

int64_t tour_length(int n, const int32_t* dist, const int32_t* tour, int len) {
    if (len != n + 1)
        throw ModelError(Errc::not_closed,
                         "closed tour must have n+1 entries, got " + std::to_string(len));
    if (tour[0] != tour[len - 1]) throw ModelError(Errc::not_closed, "tour does not return to its start");
    std::vector<char> seen(n, 0);
    for (int k = 0; k < n; ++k) {
        const int32_t c = tour[k];
        if (c < 0 || c >= n || seen[c])
            throw ModelError(Errc::not_a_permutation,
                             "tour is not a permutation of 0.." + std::to_string(n - 1));
        seen[c] = 1;
    }
    int64_t total = 0;
    for (int k = 0; k < n; ++k) total += dist[static_cast<size_t>(tour[k]) * n + tour[k + 1]];
    return total;
}

void validate(const Config& c) {
    if (!(c.rho > 0.0 && c.rho <= 1.0)) throw ModelError(Errc::config_error, "rho must be in (0,1]");
    if (c.alpha < 0.0 || c.beta < 0.0)
        throw ModelError(Errc::config_error, "alpha and beta must be >= 0");
    if (c.m < 0) throw ModelError(Errc::config_error, "ant count must be >= 1");
    if (c.iterations < 1) throw ModelError(Errc::config_error, "iterations must be >= 1");
    if (c.theta < 1) throw ModelError(Errc::config_error, "tile size must be >= 1");
    if (c.selection < 0 || c.selection > 2)
        throw ModelError(Errc::config_error, "unknown selection strategy");
    if (c.deposit < 0 || c.deposit > 3) throw ModelError(Errc::config_error, "unknown deposit strategy");
    if (c.selection == 1 && !(c.nn >= 1 && c.nn < c.n))
        throw ModelError(Errc::config_error,
                         "nn must satisfy 1 <= nn < n (n=" + std::to_string(c.n) + ")");
}

std::vector<double> eta_beta_table(int64_t max_d, double beta) {
    // eta = 1/d for d > 0, 1.0 for coincident distinct cities
    // (model.hpp:140-145); choice uses pow(eta, beta) (model.hpp:167).
    std::vector<double> lut(static_cast<size_t>(max_d) + 1);
    for (int64_t d = 0; d <= max_d; ++d) {
        const double eta = d > 0 ? 1.0 / static_cast<double>(d) : 1.0;
        lut[static_cast<size_t>(d)] = std::pow(eta, beta);
    }
    return lut;
}

void predicted_access_cost(int deposit, int n, int m, int theta, double out[4]) {
    auto share = [](int64_t inspections, int th) {
        return 2.0 * static_cast<double>(inspections) / static_cast<double>(th);
    };
    out[0] = out[1] = out[2] = out[3] = 0.0;
    const int64_t cells = static_cast<int64_t>(n) * n;
    switch (deposit) {
    case 0:
        out[3] = 2.0 * static_cast<double>(m) * static_cast<double>(n);
        break;
    case 1: {
        const int64_t insp = cells * m * n;
        out[0] = share(insp, 1);
        out[1] = static_cast<double>(cells);
        break;
    }
    case 2: {
        const int64_t insp = cells * m * n;
        out[0] = share(insp, theta);
        out[2] = share(insp, 1) - out[0];
        out[1] = static_cast<double>(cells);
        break;
    }
    default: {
        const int64_t insp = ((cells + 1) / 2) * m * n;
        out[0] = share(insp, theta);
        out[2] = share(insp, 1) - out[0];
        out[1] = static_cast<double>(cells);
        break;
    }
    }
}

double host_pow(double x, double y) { return std::pow(x, y); }

namespace {

int find_libm(struct dl_phdr_info* info, size_t, void* data) {
    const char* name = info->dlpi_name;
    if (name && std::strstr(name, "libm.so")) {
        *static_cast<std::string*>(data) = name;
        return 1;
    }
    return 0;
}

double rd(const std::string& img, size_t off) {
    double v;
    std::memcpy(&v, img.data() + off, sizeof(v));
    return v;
}

uint64_t ru(const std::string& img, size_t off) {
    uint64_t v;
    std::memcpy(&v, img.data() + off, sizeof(v));
    return v;
}

// first offset >= from where the 16 bytes (a, b) occur, or npos
size_t find_pair(const std::string& img, double a, double b, size_t from) {
    char pat[16];
    std::memcpy(pat, &a, 8);
    std::memcpy(pat + 8, &b, 8);
    return img.find(std::string(pat, 16), from);
}

} // namespace

bool read_libm_pow_tables(LibmPowTables& T, std::string& why) {
    std::string path;
    host_pow(2.0, 0.5); // make sure libm is mapped
    dl_iterate_phdr(find_libm, &path);
    if (path.empty()) {
        why = "libm.so is not loaded";
        return false;
    }
    std::ifstream f(path, std::ios::binary);
    const std::string img((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (img.empty()) {
        why = "cannot read " + path;
        return false;
    }
    // __pow_log_data: {ln2hi, ln2lo} then A[0] = -0.5, then the table whose
    // first entry is invc = 0x1.6ap+0 with a zero pad (glibc pow_log_data.c);
    // __log_data shares the (ln2hi, ln2lo) prefix, hence the extra checks.
    const double ln2hi = 0x1.62e42fefa3800p-1, ln2lo = 0x1.ef35793c76730p-45;
    size_t lo = std::string::npos;
    for (size_t at = find_pair(img, ln2hi, ln2lo, 0); at != std::string::npos;
         at = find_pair(img, ln2hi, ln2lo, at + 1)) {
        if (at + 72 + 128 * 32 <= img.size() && rd(img, at + 16) == -0.5 &&
            rd(img, at + 72) == 0x1.6ap+0 && ru(img, at + 80) == 0) {
            lo = at;
            break;
        }
    }
    // __exp_data: {InvLn2N = 0x1.71547652b82fep0 * 128, Shift = 0x1.8p52};
    // its 2^(i/128) table starts {tail 0, sbits(1.0)} a fixed distance later
    const size_t ex = find_pair(img, 0x1.71547652b82fep7, 0x1.8p52, 0);
    size_t et = std::string::npos;
    if (ex != std::string::npos)
        for (size_t off = ex + 64; off + 16 <= img.size() && off < ex + 512; off += 8)
            if (ru(img, off) == 0 && ru(img, off + 8) == 0x3ff0000000000000ull) {
                et = off;
                break;
            }
    if (lo == std::string::npos || et == std::string::npos || et + 256 * 8 > img.size()) {
        why = "pow tables not found in " + path;
        return false;
    }
    T.ln2hi = rd(img, lo);
    T.ln2lo = rd(img, lo + 8);
    for (int k = 0; k < 7; ++k) T.A[k] = rd(img, lo + 16 + 8 * k);
    for (int k = 0; k < 128 * 4; ++k) T.ltab[k] = rd(img, lo + 72 + 8 * k);
    T.invln2N = rd(img, ex);
    T.shift = rd(img, ex + 8);
    T.negln2hiN = rd(img, ex + 16);
    T.negln2loN = rd(img, ex + 24);
    for (int k = 0; k < 4; ++k) T.C[k] = rd(img, ex + 32 + 8 * k);
    for (int k = 0; k < 256; ++k) T.etab[k] = ru(img, et + 8 * k);
    return true;
}

} // namespace acob200
