/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's Brouwer-Zimmermann path
 * (/root/reference/proj, C++20), used only as a parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg. Pinned against the
 * compiled reference (oracle/_ref, see Makefile) through tests/golden/.
 *
 * Matrices: k rows x W u64 words, W = ceil(n/64), bit i of a row in word
 * i/64 at position i%64 (LSB-first; the same bit order as the reference's
 * u32 words, f2core.hpp:9-12), padding bits zero.
 */
#ifndef MDORACLE_H
#define MDORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* util.hpp:12-24 */
uint64_t mdo_splitmix64_next(uint64_t* state);
/* std::mt19937_64 restated (input generator convention) */
void mdo_gen_matrix(uint32_t n, uint32_t k, uint64_t seed, int identity, uint64_t* rows_out);

/* f2core.cpp:79-82 */
uint32_t mdo_rank(const uint64_t* rows, uint32_t k, uint32_t n);
/* f2core.cpp:92-97: writes the rref rows (zero rows dropped); returns the rank */
uint32_t mdo_row_basis(const uint64_t* rows, uint32_t k, uint32_t n, uint64_t* out);

/* gamma.cpp:32-94. gammas_out: up to ceil(n/k) * k * W words; ranks_out /
 * perm_out sized ceil(n/k) and n. Returns m (number of Gammas) or 0 on error. */
uint32_t mdo_best_gamma(const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials, uint64_t seed,
                        uint64_t* gammas_out, uint32_t* ranks_out, uint32_t* perm_out,
                        uint32_t* k_last_out);
uint32_t mdo_compute_gamma(const uint64_t* G, uint32_t k, uint32_t n, uint64_t* gammas_out,
                           uint32_t* ranks_out, uint32_t* perm_out, uint32_t* k_last_out);

/* gamma.cpp:96-106 */
uint32_t mdo_lower_bound(uint32_t m, uint32_t g, uint32_t k, uint32_t k_last);
uint32_t mdo_singleton_upper(uint32_t n, uint32_t k);

/* engines.cpp:221-243 (round_stack): min weight over all c-subsets of the k
 * rows. Returns UINT32_MAX for an invalid c. */
uint32_t mdo_round(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t c, uint64_t* combos);
/* Same enumeration, all weights into hist[0..n]; returns the minimum. */
uint32_t mdo_round_hist(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t c, uint64_t* hist);
/* engines.cpp:480-506 (serial Gray brute force over all 2^k - 1 codewords) */
uint32_t mdo_brute(const uint64_t* rows, uint32_t k, uint32_t n);

/* One executed round / one completed level of the BZ loop. */
typedef struct { uint32_t c, j, w, U_after; } mdo_round_rec;
typedef struct { uint32_t c, L_after, U_after; } mdo_level_rec;

typedef struct {
    uint32_t d;        /* U at termination (or at the cap) */
    uint32_t capped;   /* 1 when the level cap stopped the loop */
    uint32_t m, k, n, k_last, g_final;
    uint32_t n_rounds, n_levels;
    uint64_t combinations;
} mdo_result;

/* engines.cpp:617-648 + 447-476: row_basis -> best_gamma_over_permutations ->
 * singleton upper bound -> level loop with round_stack. level_cap 0 = none.
 * rounds/levels: caller arrays of capacity cap_rounds / cap_levels. */
int mdo_min_weight(const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials, uint64_t seed,
                   uint32_t level_cap, mdo_result* res, mdo_round_rec* rounds, uint32_t cap_rounds,
                   mdo_level_rec* levels, uint32_t cap_levels, uint32_t* perm_out,
                   uint64_t* gamma_hash_out);

/* FNV-1a 64 over rows' u64 words, little-endian bytes (harness convention) */
uint64_t mdo_hash_rows(const uint64_t* rows, uint32_t k, uint32_t n);

#ifdef __cplusplus
}
#endif
#endif
