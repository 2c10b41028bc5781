/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference Ant System hot
 * path (see aco_oracle.h for the rules and how parity is pinned).
 *
 * Build: oracle/Makefile, gcc -O2 -std=c11 -ffp-contract=off (no -march, like
 * the reference's CMakeLists.txt:1-22, so no FMA contraction and the same
 * libm pow the reference calls at model.hpp:167).
 */
#include "aco_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Errc order, errors.hpp:8-27 (code returned = index + 1). */
enum { E_OVERFLOW = 6, E_INVALID_LENGTH = 7, E_NOT_PERM = 8, E_NOT_CLOSED = 9,
       E_ALL_VISITED = 10 };

/* ---- Philox4x32-10: rng.hpp:12-43 ------------------------------------- */
void orc_philox(const uint32_t ctr[4], uint64_t key, uint32_t out[4]) {
    uint32_t v0 = ctr[0], v1 = ctr[1], v2 = ctr[2], v3 = ctr[3];
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int r = 0; r < 10; ++r) {                       /* rng.hpp:37-41 */
        uint64_t p0 = (uint64_t)0xD2511F53u * v0;         /* rng.hpp:22 */
        uint64_t p1 = (uint64_t)0xCD9E8D57u * v2;         /* rng.hpp:23 */
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ v1 ^ k0;     /* rng.hpp:28 */
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ v3 ^ k1;     /* rng.hpp:30 */
        v1 = (uint32_t)p1;
        v3 = (uint32_t)p0;
        v0 = n0;
        v2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = v0; out[1] = v1; out[2] = v2; out[3] = v3;
}

/* RngStream::uniform_at, rng.hpp:74-80: counter {draw, step, ant, iteration}. */
double orc_uniform_at(uint64_t seed, uint32_t iteration, uint32_t ant, uint32_t step,
                      uint32_t draw) {
    uint32_t c[4] = {draw, step, ant, iteration}, o[4];
    orc_philox(c, seed, o);
    uint64_t bits = ((uint64_t)o[1] << 32) | o[0];
    return (double)(bits >> 11) * 0x1.0p-53;
}

/* ---- synthetic instance generator, SURVEY.md App. B ------------------- */
static uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void orc_synth_coords(int n, uint64_t state, double* xs, double* ys) {
    for (int i = 0; i < n; ++i) {
        xs[i] = (double)(splitmix64(&state) % 10001u);
        ys[i] = (double)(splitmix64(&state) % 10001u);
    }
}

/* ---- edge weights, tsplib.hpp:69-70, 190-210 --------------------------- */
static int nint_(double x) { return (int)(x + 0.5); }

static int32_t edge_weight(int ewt, double xi, double yi, double xj, double yj) {
    const double dx = xi - xj, dy = yi - yj;
    switch (ewt) {
    case 0: return nint_(sqrt(dx * dx + dy * dy));                 /* :200 */
    case 1: return (int32_t)ceil(sqrt(dx * dx + dy * dy));         /* :202 */
    default: {                                                     /* :204-206 */
        const double r = sqrt((dx * dx + dy * dy) / 10.0);
        const int t = nint_(r);
        return (t < r) ? t + 1 : t;
    }
    }
}

/* build_problem, model.hpp:125-152 (dist part; eta is folded into the
 * choice restatement below). */
int orc_build_dist(int n, const double* xs, const double* ys, int ewt, int32_t* dist) {
    int64_t max_d = 0;
    for (int i = 0; i < n; ++i) dist[(size_t)i * n + i] = 0;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            const int32_t d = edge_weight(ewt, xs[i], ys[i], xs[j], ys[j]);
            if (d < 0) return E_OVERFLOW;                          /* :136-137 */
            dist[(size_t)i * n + j] = d;
            dist[(size_t)j * n + i] = d;
            if (d > max_d) max_d = d;
        }
    if (max_d > 0 && (int64_t)n > INT64_MAX / max_d) return E_OVERFLOW; /* :148-150 */
    return 0;
}

/* greedy_nn_tour_length, model.hpp:230-255 */
int64_t orc_greedy_nn_tour_length(int n, const int32_t* dist) {
    char* visited = calloc((size_t)n, 1);
    int cur = 0;
    int64_t total = 0;
    visited[0] = 1;
    for (int step = 1; step < n; ++step) {
        int best = -1;
        int32_t best_d = INT32_MAX;
        for (int j = 0; j < n; ++j) {
            if (visited[j]) continue;
            const int32_t d = dist[(size_t)cur * n + j];
            if (d < best_d) { best_d = d; best = j; }
        }
        total += best_d;
        visited[best] = 1;
        cur = best;
    }
    total += dist[(size_t)cur * n];
    free(visited);
    return total;
}

/* initial_pheromone, model.hpp:258-262 */
double orc_tau0(int n, const int32_t* dist, int m) {
    return (double)m / (double)orc_greedy_nn_tour_length(n, dist);
}

/* build_nn_lists, model.hpp:177-202: nn nearest distinct cities, ascending
 * distance, ties by lower index.  partial_sort with a strict total order
 * yields exactly the first nn elements of the fully sorted order. */
static const int32_t* g_nn_row;
static int cmp_nn(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    if (g_nn_row[x] != g_nn_row[y]) return g_nn_row[x] < g_nn_row[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

int orc_build_nn_lists(int n, const int32_t* dist, int nn, int32_t* out) {
    if (!(nn >= 1 && nn < n)) return E_INVALID_LENGTH;             /* :179-181 */
    int32_t* order = malloc(sizeof(int32_t) * (size_t)(n - 1));
    for (int i = 0; i < n; ++i) {
        int k = 0;
        for (int j = 0; j < n; ++j)
            if (j != i) order[k++] = j;
        g_nn_row = dist + (size_t)i * n;
        qsort(order, (size_t)(n - 1), sizeof(int32_t), cmp_nn);
        memcpy(out + (size_t)i * nn, order, sizeof(int32_t) * (size_t)nn);
    }
    free(order);
    return 0;
}

/* compute_choice_info, model.hpp:154-173, with heuristic(i,j) = 1/d (1.0 for
 * d == 0 off-diagonal, 0 on the diagonal), model.hpp:142-145. */
void orc_choice_info(int n, const int32_t* dist, const double* tau, double alpha, double beta,
                     double* choice) {
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            const int32_t d = dist[(size_t)i * n + j];
            const double eta = (i == j) ? 0.0 : (d > 0 ? 1.0 / d : 1.0);
            choice[(size_t)i * n + j] = pow(tau[(size_t)i * n + j], alpha) * pow(eta, beta);
        }
        choice[(size_t)i * n + i] = 0.0;                           /* :169 */
    }
}

/* tour_length, model.hpp:205-226 (validation + int64 sum). Returns -1 on an
 * invalid tour. */
int64_t orc_tour_length(int n, const int32_t* dist, const int32_t* tour) {
    if (tour[0] != tour[n]) return -1;
    char* seen = calloc((size_t)n, 1);
    for (int k = 0; k < n; ++k) {
        const int32_t c = tour[k];
        if (c < 0 || c >= n || seen[c]) { free(seen); return -1; }
        seen[c] = 1;
    }
    free(seen);
    int64_t total = 0;
    for (int k = 0; k < n; ++k) total += dist[(size_t)tour[k] * n + tour[k + 1]];
    return total;
}

/* ---- selection, construction.hpp ---------------------------------------- */
#define TEST(tabu, j) (((tabu)[(j) >> 6] >> ((j) & 63)) & 1u)

static int lowest_unvisited(const uint64_t* tabu, int n) {          /* :31-35 */
    for (int j = 0; j < n; ++j)
        if (!TEST(tabu, j)) return j;
    return -1;
}

/* select_next_roulette, construction.hpp:42-68 */
static int sel_roulette(const double* w, int n, const uint64_t* tabu, double u, int64_t* st) {
    double total = 0.0;
    for (int j = 0; j < n; ++j)
        if (!TEST(tabu, j)) total += w[j];
    if (total <= 0.0) { st[2]++; return lowest_unvisited(tabu, n); }
    const double target = u * total;
    double acc = 0.0;
    int last_positive = -1;
    for (int j = 0; j < n; ++j) {
        if (TEST(tabu, j)) continue;
        if (w[j] > 0.0) last_positive = j;
        acc += w[j];
        if (acc > target) return j;
    }
    st[1]++;
    if (last_positive >= 0) return last_positive;
    return lowest_unvisited(tabu, n);
}

/* select_next_nn, construction.hpp:73-121. *used_draw tells the caller
 * whether the step consumed its draw (the argmax fallback does not). */
static int sel_nn(const double* w, int n, const int32_t* nb, int nn, const uint64_t* tabu,
                  double u, int64_t* st) {
    double total = 0.0;
    int any = 0;
    for (int q = 0; q < nn; ++q)
        if (!TEST(tabu, nb[q])) { any = 1; total += w[nb[q]]; }
    if (any) {
        if (total <= 0.0) {
            st[2]++;
            for (int q = 0; q < nn; ++q)
                if (!TEST(tabu, nb[q])) return nb[q];
        }
        const double target = u * total;
        double acc = 0.0;
        int last_positive = -1;
        for (int q = 0; q < nn; ++q) {
            const int j = nb[q];
            if (TEST(tabu, j)) continue;
            if (w[j] > 0.0) last_positive = j;
            acc += w[j];
            if (acc > target) return j;
        }
        st[1]++;
        if (last_positive >= 0) return last_positive;
        for (int q = 0; q < nn; ++q)
            if (!TEST(tabu, nb[q])) return nb[q];
    }
    st[0]++;
    int best = -1;
    double best_w = -1.0;
    for (int j = 0; j < n; ++j) {
        if (TEST(tabu, j)) continue;
        if (w[j] > best_w) { best_w = w[j]; best = j; }
    }
    return best;
}

/* select_next_data_parallel, construction.hpp:129-162.  One draw per city
 * (draw index = city), consumed whether or not the city is visited. */
static int sel_data_parallel(const double* w, int n, const uint64_t* tabu, int theta,
                             uint64_t seed, uint32_t it, uint32_t ant, uint32_t step,
                             int64_t* st) {
    int best_city = -1;
    double best_score = 0.0;
    for (int t0 = 0; t0 < n; t0 += theta) {
        const int t1 = t0 + theta < n ? t0 + theta : n;
        int tile_city = -1;
        double tile_score = 0.0;
        for (int j = t0; j < t1; ++j) {
            const double u = orc_uniform_at(seed, it, ant, step, (uint32_t)j);
            if (TEST(tabu, j)) continue;
            const double score = w[j] * u;
            if (tile_city < 0 || score > tile_score) { tile_score = score; tile_city = j; }
        }
        if (tile_city >= 0 && (best_city < 0 || tile_score > best_score)) {
            best_score = tile_score;
            best_city = tile_city;
        }
    }
    if (best_city < 0) return -1;
    if (best_score <= 0.0) { st[2]++; return lowest_unvisited(tabu, n); }
    return best_city;
}

/* construct_tour, construction.hpp:181-201, driven like engine.hpp:98-114.
 * stats (may be NULL): [0] nn argmax fallbacks, [1] walk-fell-short
 * (last_positive) branches, [2] zero-total branches. */
int orc_construct(int n, const int32_t* dist, const double* choice, const int32_t* nn_lists,
                  int nn, int selection, int theta, uint64_t seed, uint32_t iteration,
                  int random_start, int k0, int k1, int32_t* tours, int64_t* lengths,
                  int64_t* stats) {
    const int words = (n + 63) / 64;
    uint64_t* tabu = malloc(sizeof(uint64_t) * (size_t)words);
    int64_t st_local[3] = {0, 0, 0};
    int64_t* st = stats ? stats : st_local;
    int rc = 0;
    for (int k = k0; k < k1 && rc == 0; ++k) {
        int32_t* tour = tours + (size_t)(k - k0) * (n + 1);
        int start;
        if (random_start) {                                         /* engine.hpp:105-108 */
            start = (int)(orc_uniform_at(seed, iteration, (uint32_t)k, 0, 0) * n);
            if (start >= n) start = n - 1;
        } else {
            start = k % n;
        }
        memset(tabu, 0, sizeof(uint64_t) * (size_t)words);
        tour[0] = start;
        tabu[start >> 6] |= 1ull << (start & 63);
        int cur = start;
        for (int step = 1; step < n; ++step) {
            const double* w = choice + (size_t)cur * n;
            int next;
            if (selection == 0) {
                next = sel_roulette(w, n, tabu,
                                    orc_uniform_at(seed, iteration, (uint32_t)k, (uint32_t)step, 0),
                                    st);
            } else if (selection == 1) {
                next = sel_nn(w, n, nn_lists + (size_t)cur * nn, nn, tabu,
                              orc_uniform_at(seed, iteration, (uint32_t)k, (uint32_t)step, 0),
                              st);
            } else {
                next = sel_data_parallel(w, n, tabu, theta, seed, iteration, (uint32_t)k,
                                         (uint32_t)step, st);
            }
            if (next < 0) { rc = E_ALL_VISITED; break; }
            tour[step] = next;
            tabu[next >> 6] |= 1ull << (next & 63);
            cur = next;
        }
        tour[n] = start;
        lengths[k - k0] = orc_tour_length(n, dist, tour);
    }
    free(tabu);
    return rc;
}

/* ---- update: pheromone.hpp ---------------------------------------------- */
/* evaporate (pheromone.hpp:174-189) followed by
 *  - deposit 0: deposit_accumulate (pheromone.hpp:195-208), serial ant-major,
 *    edge-minor, both orientations, straight into the evaporated tau;
 *  - deposit 1: the gather family (pheromone.hpp:133-148, 213-341), restated
 *    in O(m n): cell (i,j) receives acc = sum over ants k ascending (and,
 *    within a tour, steps ascending) of w_k for every traversal of edge {i,j},
 *    summed from 0.0, then tau(i,j) += acc once.  Within one tour the edge
 *    {i,j} is crossed at most once for n >= 3 (twice for n == 2, where both
 *    crossings are added in step order), so walking the ants in ascending k
 *    and adding w_k into a per-cell accumulator reproduces gather_cell's
 *    summation order exactly.  w_k = 1.0 / (double)C_k (pheromone.hpp:123-128).
 */
void orc_update(int n, int m, const int32_t* tours, const int64_t* lengths, double rho,
                int deposit, double* tau) {
    const double keep = 1.0 - rho;                                  /* :179 */
    const size_t cells = (size_t)n * n;
    for (size_t c = 0; c < cells; ++c) tau[c] *= keep;              /* :183 */
    if (deposit == 0) {
        for (int k = 0; k < m; ++k) {
            const int32_t* row = tours + (size_t)k * (n + 1);
            const double w = 1.0 / (double)lengths[k];
            for (int s = 0; s < n; ++s) {
                tau[(size_t)row[s] * n + row[s + 1]] += w;          /* :202 */
                tau[(size_t)row[s + 1] * n + row[s]] += w;          /* :203 */
            }
        }
        return;
    }
    double* acc = calloc(cells, sizeof(double));
    for (int k = 0; k < m; ++k) {
        const int32_t* row = tours + (size_t)k * (n + 1);
        const double w = 1.0 / (double)lengths[k];
        for (int s = 0; s < n; ++s) {
            const int32_t a = row[s], b = row[s + 1];
            acc[(size_t)a * n + b] += w;
            if (a != b) acc[(size_t)b * n + a] += w;
        }
    }
    for (size_t c = 0; c < cells; ++c) tau[c] += acc[c];            /* :220 */
    free(acc);
}

/* The host libm's pow over arrays (the function model.hpp:167 calls), for
 * the device libm_pow parity test. */
void orc_pow(int n, const double* x, const double* y, double* out) {
    for (int i = 0; i < n; ++i) out[i] = pow(x[i], y[i]);
}
