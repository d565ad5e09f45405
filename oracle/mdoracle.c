/* TEST INFRASTRUCTURE — NOT PRODUCT CODE. See mdoracle.h.
 *
 * Plain-C restatement of the reference's CPU path, function by function, each
 * citing the reference file:line (relative to /root/reference/proj) it follows.
 * Parity of this restatement is pinned by tests/test_oracle.py against the
 * golden vectors in tests/golden/ that oracle/make_golden.py produced by
 * running the compiled reference (oracle/_ref) on the same inputs.
 */
#include "mdoracle.h"

#include <stdlib.h>
#include <string.h>

#define WORDS(n) (((n) + 63u) / 64u)

static int getbit(const uint64_t* row, uint32_t i) { return (int)((row[i >> 6] >> (i & 63)) & 1u); }
static void setbit(uint64_t* row, uint32_t i, int v) {
    uint64_t m = 1ull << (i & 63);
    if (v) row[i >> 6] |= m; else row[i >> 6] &= ~m;
}
static uint32_t popc64(uint64_t x) { return (uint32_t)__builtin_popcountll(x); }

/* util.hpp:12-24 — SplitMix64 */
uint64_t mdo_splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* std::mt19937_64 (the published MT19937-64 algorithm), the BASELINE.json
 * input generator; SURVEY.md §8d fixes one draw per bit, bit = draw & 1,
 * row-major over A (k x (n-k)) and G = (I_k | A); identity=0 fills all of G. */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}
static uint64_t mt64_next(mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

void mdo_gen_matrix(uint32_t n, uint32_t k, uint64_t seed, int identity, uint64_t* rows) {
    uint32_t W = WORDS(n);
    mt64 s;
    mt64_seed(&s, seed);
    memset(rows, 0, sizeof(uint64_t) * k * W);
    uint32_t off = identity ? k : 0;
    for (uint32_t r = 0; r < k; ++r) {
        if (identity) setbit(rows + r * W, r, 1);
        for (uint32_t c = off; c < n; ++c)
            if (mt64_next(&s) & 1) setbit(rows + r * W, c, 1);
    }
}

/* f2core.cpp:63-75 — rref_in_place: pivot = first row >= rank with a 1 in col */
static uint32_t rref_in_place(uint64_t* w, uint32_t k, uint32_t n) {
    uint32_t W = WORDS(n), rank = 0;
    for (uint32_t col = 0; col < n && rank < k; ++col) {
        uint32_t p = rank;
        while (p < k && !getbit(w + p * W, col)) ++p;
        if (p == k) continue;
        if (p != rank)
            for (uint32_t i = 0; i < W; ++i) {
                uint64_t t = w[rank * W + i]; w[rank * W + i] = w[p * W + i]; w[p * W + i] = t;
            }
        for (uint32_t r = 0; r < k; ++r)
            if (r != rank && getbit(w + r * W, col))
                for (uint32_t i = 0; i < W; ++i) w[r * W + i] ^= w[rank * W + i];
        ++rank;
    }
    return rank;
}

/* f2core.cpp:79-82 */
uint32_t mdo_rank(const uint64_t* rows, uint32_t k, uint32_t n) {
    uint32_t W = WORDS(n);
    uint64_t* w = malloc(sizeof(uint64_t) * k * W);
    memcpy(w, rows, sizeof(uint64_t) * k * W);
    uint32_t r = rref_in_place(w, k, n);
    free(w);
    return r;
}

/* f2core.cpp:84-97 (rref_of + row_basis; 0 on the zero matrix, which throws there) */
uint32_t mdo_row_basis(const uint64_t* rows, uint32_t k, uint32_t n, uint64_t* out) {
    uint32_t W = WORDS(n);
    uint64_t* w = malloc(sizeof(uint64_t) * k * W);
    memcpy(w, rows, sizeof(uint64_t) * k * W);
    uint32_t r = rref_in_place(w, k, n);
    memcpy(out, w, sizeof(uint64_t) * r * W);
    free(w);
    return r;
}

/* f2core.cpp:9-16 — BitMatrix::swap_cols */
static void swap_cols(uint64_t* m, uint32_t k, uint32_t W, uint32_t a, uint32_t b) {
    if (a == b) return;
    for (uint32_t r = 0; r < k; ++r) {
        int va = getbit(m + r * W, a), vb = getbit(m + r * W, b);
        setbit(m + r * W, a, vb);
        setbit(m + r * W, b, va);
    }
}

/* gamma.cpp:32-75 — compute_gamma_matrices */
uint32_t mdo_compute_gamma(const uint64_t* G, uint32_t k, uint32_t n, uint64_t* gammas,
                           uint32_t* ranks, uint32_t* perm, uint32_t* k_last) {
    if (k == 0 || k > n) return 0;
    if (mdo_rank(G, k, n) != k) return 0;
    uint32_t W = WORDS(n);
    size_t gsz = (size_t)k * W;
    uint64_t* w = malloc(sizeof(uint64_t) * gsz);
    memcpy(w, G, sizeof(uint64_t) * gsz);
    for (uint32_t j = 0; j < n; ++j) perm[j] = j;
    uint32_t m = 0;
    for (uint32_t offset = 0; offset < n; offset += k) {
        uint32_t br = 0;
        for (; br < k; ++br) {
            uint32_t target = offset + br;
            if (target >= n) break;
            uint32_t pc = n, pr = k;
            for (uint32_t c = target; c < n && pc == n; ++c)
                for (uint32_t r = br; r < k; ++r)
                    if (getbit(w + r * W, c)) { pc = c; pr = r; break; }
            if (pc == n) break;
            if (pc != target) {
                swap_cols(w, k, W, target, pc);
                uint32_t t = perm[target]; perm[target] = perm[pc]; perm[pc] = t;
                for (uint32_t s = 0; s < m; ++s) swap_cols(gammas + s * gsz, k, W, target, pc);
            }
            if (pr != br)
                for (uint32_t i = 0; i < W; ++i) {
                    uint64_t t = w[br * W + i]; w[br * W + i] = w[pr * W + i]; w[pr * W + i] = t;
                }
            for (uint32_t r = 0; r < k; ++r)
                if (r != br && getbit(w + r * W, target))
                    for (uint32_t i = 0; i < W; ++i) w[r * W + i] ^= w[br * W + i];
        }
        if (br == 0) break;
        memcpy(gammas + m * gsz, w, sizeof(uint64_t) * gsz);
        ranks[m++] = br;
        if (br < k) break;
    }
    free(w);
    *k_last = m ? ranks[m - 1] : 0;
    return m;
}

/* gamma.cpp:16-22 — permute_columns: output column j = input column perm[j] */
static void permute_columns(const uint64_t* G, uint32_t k, uint32_t n, const uint32_t* perm,
                            uint64_t* out) {
    uint32_t W = WORDS(n);
    memset(out, 0, sizeof(uint64_t) * k * W);
    for (uint32_t j = 0; j < n; ++j)
        for (uint32_t r = 0; r < k; ++r)
            if (getbit(G + r * W, perm[j])) setbit(out + r * W, j, 1);
}

/* gamma.cpp:77-94 — best_gamma_over_permutations (util.hpp:28-33 shuffle) */
uint32_t mdo_best_gamma(const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials, uint64_t seed,
                        uint64_t* gammas, uint32_t* ranks, uint32_t* perm, uint32_t* k_last) {
    if (trials < 1) return 0;
    uint32_t W = WORDS(n);
    uint32_t mmax = (n + k - 1) / k;
    size_t gsz = (size_t)k * W;
    uint32_t m = mdo_compute_gamma(G, k, n, gammas, ranks, perm, k_last);
    if (!m) return 0;
    uint64_t* cg = malloc(sizeof(uint64_t) * gsz * mmax);
    uint32_t* cr = malloc(sizeof(uint32_t) * mmax);
    uint32_t* cp = malloc(sizeof(uint32_t) * n);
    uint32_t* pm = malloc(sizeof(uint32_t) * n);
    uint64_t* Gp = malloc(sizeof(uint64_t) * gsz);
    uint64_t st = seed;
    for (uint32_t t = 0; t < trials; ++t) {
        for (uint32_t j = 0; j < n; ++j) pm[j] = j;
        for (size_t i = n; i > 1; --i) {
            size_t j = (size_t)(mdo_splitmix64_next(&st) % i);
            uint32_t x = pm[i - 1]; pm[i - 1] = pm[j]; pm[j] = x;
        }
        permute_columns(G, k, n, pm, Gp);
        uint32_t ckl = 0;
        uint32_t cm = mdo_compute_gamma(Gp, k, n, cg, cr, cp, &ckl);
        for (uint32_t j = 0; j < n; ++j) cp[j] = pm[cp[j]];
        if (cm > m || (cm == m && ckl > *k_last)) {
            m = cm;
            *k_last = ckl;
            memcpy(gammas, cg, sizeof(uint64_t) * gsz * cm);
            memcpy(ranks, cr, sizeof(uint32_t) * cm);
            memcpy(perm, cp, sizeof(uint32_t) * n);
        }
    }
    free(cg); free(cr); free(cp); free(pm); free(Gp);
    return m;
}

/* gamma.cpp:96-100 */
uint32_t mdo_lower_bound(uint32_t m, uint32_t g, uint32_t k, uint32_t k_last) {
    int64_t partial = (int64_t)g + 1 - (int64_t)k + (int64_t)k_last;
    if (partial < 0) partial = 0;
    return (m - 1) * (g + 1) + (uint32_t)partial;
}

/* gamma.cpp:102-106 (0 where the reference throws) */
uint32_t mdo_singleton_upper(uint32_t n, uint32_t k) {
    if (k < 1 || n < k) return 0;
    return n - k + 1;
}

/* engines.cpp:221-243 — round_stack: the prefix (first c-1 elements) walks
 * lex order over {0..k-2} (advance_prefix, engines.cpp:39-49) with a stack of
 * partial sums; the last element e runs over prefix.back()+1 .. k-1 fused into
 * the weight evaluation. hist (optional) collects every weight. */
static uint32_t round_walk(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t c, uint64_t* combos,
                           uint64_t* hist) {
    if (c < 1 || c > k) return UINT32_MAX;
    uint32_t W = WORDS(n);
    uint32_t best = UINT32_MAX;
    uint64_t cnt = 0;
    if (c == 1) { /* engines.cpp:22-30 scan_rows */
        for (uint32_t r = 0; r < k; ++r) {
            uint32_t w = 0;
            for (uint32_t i = 0; i < W; ++i) w += popc64(rows[r * W + i]);
            if (hist) hist[w]++;
            if (w < best) best = w;
            ++cnt;
        }
        if (combos) *combos = cnt;
        return best;
    }
    uint32_t p = c - 1;
    uint32_t* prefix = malloc(sizeof(uint32_t) * p);
    uint64_t* stack = malloc(sizeof(uint64_t) * p * W);
    for (uint32_t i = 0; i < p; ++i) prefix[i] = i;
    uint32_t changed = 0;
    for (;;) {
        for (uint32_t i = changed; i < p; ++i) /* AdditionStack::rebuild_from, engines.cpp:160-171 */
            for (uint32_t x = 0; x < W; ++x)
                stack[i * W + x] = (i ? stack[(i - 1) * W + x] : 0) ^ rows[prefix[i] * W + x];
        const uint64_t* top = stack + (p - 1) * W;
        for (uint32_t e = prefix[p - 1] + 1; e < k; ++e) {
            uint32_t w = 0;
            for (uint32_t x = 0; x < W; ++x) w += popc64(top[x] ^ rows[e * W + x]);
            if (hist) hist[w]++;
            if (w < best) best = w;
            ++cnt;
        }
        /* advance_prefix over {0..k-2} */
        uint32_t i = p;
        int adv = 0;
        while (i-- > 0) {
            if (prefix[i] < (k - 2) - (p - 1 - i)) {
                ++prefix[i];
                for (uint32_t j = i + 1; j < p; ++j) prefix[j] = prefix[j - 1] + 1;
                changed = i;
                adv = 1;
                break;
            }
        }
        if (!adv) break;
    }
    free(prefix);
    free(stack);
    if (combos) *combos = cnt;
    return best;
}

uint32_t mdo_round(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t c, uint64_t* combos) {
    return round_walk(rows, k, n, c, combos, NULL);
}

uint32_t mdo_round_hist(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t c, uint64_t* hist) {
    memset(hist, 0, sizeof(uint64_t) * (n + 1));
    return round_walk(rows, k, n, c, NULL, hist);
}

/* engines.cpp:489-505 — serial Gray-code brute force (gray_diff = ctz) */
uint32_t mdo_brute(const uint64_t* rows, uint32_t k, uint32_t n) {
    if (k == 0 || k > 40) return UINT32_MAX;
    uint32_t W = WORDS(n);
    uint64_t acc[64] = {0};
    if (W > 64) return UINT32_MAX;
    uint32_t best = UINT32_MAX;
    uint64_t total = (1ull << k) - 1;
    for (uint64_t i = 1; i <= total; ++i) {
        uint32_t b = (uint32_t)__builtin_ctzll(i);
        uint32_t w = 0;
        for (uint32_t x = 0; x < W; ++x) { acc[x] ^= rows[b * W + x]; w += popc64(acc[x]); }
        if (w < best) best = w;
    }
    return best;
}

uint64_t mdo_hash_rows(const uint64_t* rows, uint32_t k, uint32_t n) {
    uint32_t W = WORDS(n);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < (size_t)k * W; ++i)
        for (int b = 0; b < 8; ++b) {
            h ^= (rows[i] >> (8 * b)) & 0xff;
            h *= 1099511628211ull;
        }
    return h;
}

/* engines.cpp:617-648 (min_weight) + 447-476 (run_bz_loop) with the level cap
 * of the harness (a round at level g > cap is never run). */
int mdo_min_weight(const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials, uint64_t seed,
                   uint32_t level_cap, mdo_result* res, mdo_round_rec* rounds, uint32_t cap_rounds,
                   mdo_level_rec* levels, uint32_t cap_levels, uint32_t* perm_out,
                   uint64_t* gamma_hash_out) {
    memset(res, 0, sizeof *res);
    uint32_t W = WORDS(n);
    uint64_t* B = malloc(sizeof(uint64_t) * k * W);
    uint32_t kb = mdo_row_basis(G, k, n, B);
    if (kb == 0) { free(B); return -1; }
    uint32_t mmax = (n + kb - 1) / kb;
    size_t gsz = (size_t)kb * W;
    uint64_t* gam = malloc(sizeof(uint64_t) * gsz * mmax);
    uint32_t* ranks = malloc(sizeof(uint32_t) * mmax);
    uint32_t* perm = malloc(sizeof(uint32_t) * n);
    uint32_t k_last = 0;
    uint32_t m = mdo_best_gamma(B, kb, n, trials, seed, gam, ranks, perm, &k_last);
    if (!m) { free(B); free(gam); free(ranks); free(perm); return -1; }
    if (perm_out) memcpy(perm_out, perm, sizeof(uint32_t) * n);
    if (gamma_hash_out)
        for (uint32_t j = 0; j < m; ++j) gamma_hash_out[j] = mdo_hash_rows(gam + j * gsz, kb, n);

    uint32_t U = mdo_singleton_upper(n, kb);
    uint32_t L = 1;
    int done = U <= L;
    uint32_t nr = 0, nl = 0;
    for (uint32_t g = 1; !done && g <= kb; ++g) {
        if (level_cap && g > level_cap) { res->capped = 1; break; }
        for (uint32_t j = 0; j < m; ++j) {
            if (U <= L) { done = 1; break; }
            uint64_t combos = 0;
            uint32_t w = mdo_round(gam + j * gsz, kb, n, g, &combos);
            res->combinations += combos;
            res->g_final = g;
            if (w < U) U = w;
            if (nr < cap_rounds) {
                rounds[nr].c = g; rounds[nr].j = j; rounds[nr].w = w; rounds[nr].U_after = U;
            }
            ++nr;
        }
        if (done) break;
        uint32_t lb = mdo_lower_bound(m, g, kb, k_last);
        if (lb > L) L = lb;
        if (nl < cap_levels) { levels[nl].c = g; levels[nl].L_after = L; levels[nl].U_after = U; }
        ++nl;
        if (L >= U) done = 1;
    }
    res->d = U;
    res->m = m;
    res->k = kb;
    res->n = n;
    res->k_last = k_last;
    res->n_rounds = nr;
    res->n_levels = nl;
    free(B); free(gam); free(ranks); free(perm);
    return 0;
}
