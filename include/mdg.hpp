// mdg — C++ host API of the B200 Brouwer–Zimmermann engine.
//
// Mirrors the reference's md:: interface for this path (same names, argument
// meaning and exception types) so reference callers switch by namespace:
//   BitMatrix / row_basis / rank_of           f2core.hpp:57-105
//   GammaSet / compute_gamma_matrices /
//   best_gamma_over_permutations /
//   lower_bound / singleton_upper             gamma.hpp:14-53
//   RoundStats / RoundRunner / run_bz_loop    engines.hpp:26-48,151-152
//   EngineConfig / min_weight                 engines.hpp:60-71,164-166
//   parse_matrix / serialize_matrix           io.hpp:13-29
// Storage differs (u64 words, one contiguous buffer per matrix) — the bit
// order does not.
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace mdg {

// ------------------------------------------------------------- F2 matrices
class BitMatrix {
public:
    BitMatrix() = default;
    BitMatrix(uint32_t rows, uint32_t cols)
        : rows_(rows), cols_(cols), W_((cols + 63) / 64), data_(size_t(rows) * W_, 0) {}

    uint32_t rows() const { return rows_; }
    uint32_t cols() const { return cols_; }
    uint32_t words() const { return W_; }
    uint64_t* row(uint32_t r) { return data_.data() + size_t(r) * W_; }
    const uint64_t* row(uint32_t r) const { return data_.data() + size_t(r) * W_; }
    uint64_t* data() { return data_.data(); }
    const uint64_t* data() const { return data_.data(); }

    bool get(uint32_t r, uint32_t c) const { return (row(r)[c >> 6] >> (c & 63)) & 1u; }
    void set(uint32_t r, uint32_t c, bool v) {
        uint64_t m = uint64_t{1} << (c & 63);
        if (v) row(r)[c >> 6] |= m; else row(r)[c >> 6] &= ~m;
    }
    void swap_rows(uint32_t a, uint32_t b);
    void swap_cols(uint32_t a, uint32_t b);
    void xor_row(uint32_t dst, uint32_t src) {
        uint64_t* d = row(dst);
        const uint64_t* s = row(src);
        for (uint32_t i = 0; i < W_; ++i) d[i] ^= s[i];
    }
    uint32_t row_weight(uint32_t r) const;

    bool operator==(const BitMatrix& o) const {
        return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_;
    }

private:
    uint32_t rows_ = 0, cols_ = 0, W_ = 0;
    std::vector<uint64_t> data_;
};

uint32_t rank_of(const BitMatrix& m);
BitMatrix rref_of(const BitMatrix& m);
BitMatrix row_basis(const BitMatrix& m); // throws std::invalid_argument on the zero matrix
uint64_t hash_rows(const BitMatrix& m);  // FNV-1a 64 over the u64 words, little-endian bytes

// ----------------------------------------------------------------- PRNG
class SplitMix64 { // util.hpp:12-24
public:
    explicit SplitMix64(uint64_t seed) : state_(seed) {}
    void discard(uint64_t draws) { state_ += draws * 0x9E3779B97F4A7C15ull; } // skip ahead
    uint64_t next() {
        uint64_t z = (state_ += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
private:
    uint64_t state_;
};

// ---------------------------------------------------------------- Gammas
struct GammaSet {
    std::vector<BitMatrix> gammas;   // each k x n
    std::vector<uint32_t> ranks;     // k for j < m-1, k_last for the last
    uint32_t k_last = 0;
    std::vector<uint32_t> column_perm; // stored column j = original column column_perm[j]

    uint32_t m() const { return static_cast<uint32_t>(gammas.size()); }
    uint32_t k() const { return gammas.empty() ? 0 : gammas[0].rows(); }
    uint32_t n() const { return gammas.empty() ? 0 : gammas[0].cols(); }
};

struct Bounds {
    uint32_t lower = 1;
    uint32_t upper = 0;
};

GammaSet compute_gamma_matrices(const BitMatrix& G);
GammaSet best_gamma_over_permutations(const BitMatrix& G, uint32_t trials, uint64_t seed);
// True when gs has the largest (m, k_last) any column order of a k x n matrix allows
// (then best_gamma_over_permutations returns the identity's set for every trial count).
bool gamma_set_is_maximal(const GammaSet& gs, uint32_t n, uint32_t k);
// The column order of trial t of best_gamma_over_permutations(G, trials, seed) (n columns):
// identity shuffled by Fisher-Yates with the generator advanced past the t earlier trials.
std::vector<uint32_t> trial_permutation(uint32_t n, uint64_t seed, uint64_t t);
// compute_gamma_matrices on G's columns in the order `perm`, column_perm composed with perm
// (one candidate of the permutation search, gamma.cpp:85-91).
GammaSet gamma_for_permutation(const BitMatrix& G, const std::vector<uint32_t>& perm);
// fn(i) for i in [0, n) on the library's host thread pool (the calling thread joins in)
void parallel_for(uint32_t n, const std::function<void(uint32_t)>& fn);
uint32_t lower_bound(uint32_t m, uint32_t g, uint32_t k, uint32_t k_last);
uint32_t singleton_upper(uint32_t n, uint32_t k);
BitMatrix permute_columns(const BitMatrix& m, const std::vector<uint32_t>& perm);

// ------------------------------------------------------------ level loop
struct RoundStats {
    uint32_t g = 0;
    uint32_t gamma_index = 0;
    uint32_t stop_at = 0;          // set by the loop: current L (early-exit hint)
    uint32_t upper = 0;            // set by the loop: current U (bound for pruned rounds)
    bool bounded = false;          // set by the runner: w is only a lower bound (>= U)
    uint64_t additions = 0;
    uint64_t combinations = 0;     // C(k, g): the reference's counter
    uint64_t evaluated = 0;        // codewords the device actually evaluated
    double device_ms = 0;
};

struct RoundRec { uint32_t c, j, w, U_after, bounded; };
struct LevelRec { uint32_t c, L_after, U_after; };

struct WorkStats {
    uint64_t row_additions = 0;
    uint64_t combinations = 0;
    uint64_t evaluated = 0;
    double device_ms = 0;
    uint32_t g_final = 0;
    std::vector<RoundStats> per_g;
    std::vector<RoundRec> rounds;
    std::vector<LevelRec> levels;
};

struct EngineResult {
    uint32_t d = 0;
    bool capped = false;
    WorkStats stats;
    // first executed round whose minimum equals the final U (witness source)
    int32_t witness_round = -1;
};

using RoundRunner = std::function<uint32_t(uint32_t gamma_index, uint32_t g, RoundStats&)>;
EngineResult run_bz_loop(const GammaSet& gs, Bounds bounds, const RoundRunner& round,
                         uint32_t level_cap = 0);

// ----------------------------------------------------------------- I/O
class ParseError : public std::invalid_argument {
public:
    ParseError(uint32_t line, uint32_t column, const std::string& message);
    uint32_t line;
    uint32_t column;
};
BitMatrix parse_matrix(const std::string& text);
BitMatrix parse_matrix_file(const std::string& path);
std::string serialize_matrix(const BitMatrix& M);
BitMatrix gen_matrix(uint32_t n, uint32_t k, uint64_t seed, bool identity);

// -------------------------------------------------------------- binomials
uint64_t binomial(uint32_t p, int64_t q); // throws std::overflow_error past 64 bits
void rd_unrank(uint32_t c, uint64_t rank, uint32_t* idx);
uint64_t rd_rank(uint32_t c, const uint32_t* idx);

} // namespace mdg
