/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the reference
 * Ant System hot path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker.  The product
 * library (paper_1101_2678_b200/libaco_gpu.so) never links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Parity of this restatement is PINNED against
 * (a) the reference headers compiled unmodified into oracle/_ref/libaco_ref.so
 * (tests/test_oracle_vs_ref.py), (b) the Random123 Philox known-answer
 * vectors, (c) the SURVEY.md App. B golden traces (tests/golden/), and
 * (d) att48.opt.tour = 10628 (tests/golden/att48.*).
 */
#ifndef ACO_ORACLE_H
#define ACO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

void orc_philox(const uint32_t ctr[4], uint64_t key, uint32_t out[4]);
double orc_uniform_at(uint64_t seed, uint32_t iteration, uint32_t ant, uint32_t step,
                      uint32_t draw);

void orc_synth_coords(int n, uint64_t seed_state, double* xs, double* ys);
/* ewt: 0 EUC_2D, 1 CEIL_2D, 2 ATT.  Returns 0 or an Errc+1 code. */
int orc_build_dist(int n, const double* xs, const double* ys, int ewt, int32_t* dist);
int64_t orc_greedy_nn_tour_length(int n, const int32_t* dist);
double orc_tau0(int n, const int32_t* dist, int m);
int orc_build_nn_lists(int n, const int32_t* dist, int nn, int32_t* out);
void orc_choice_info(int n, const int32_t* dist, const double* tau, double alpha, double beta,
                     double* choice);
void orc_pow(int n, const double* x, const double* y, double* out);
int64_t orc_tour_length(int n, const int32_t* dist, const int32_t* tour);

/* selection: 0 roulette_full, 1 roulette_nn, 2 data_parallel_tiled */
int orc_construct(int n, const int32_t* dist, const double* choice, const int32_t* nn_lists,
                  int nn, int selection, int theta, uint64_t seed, uint32_t iteration,
                  int random_start, int k0, int k1, int32_t* tours, int64_t* lengths,
                  int64_t* stats);

/* deposit: 0 accumulate (serial scatter), 1 gather (O(m n) restatement of the
 * scatter-gather / tiled / symmetric family, bit-identical to all three). */
void orc_update(int n, int m, const int32_t* tours, const int64_t* lengths, double rho,
                int deposit, double* tau);

#ifdef __cplusplus
}
#endif
#endif
