// Device engine of the B200 Brouwer–Zimmermann round (host-facing C++).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "mdg.hpp"

namespace mdg {

class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// tab: prefix-sum tiles (prefix table x suffix table); rd: the same tiles with each tile's
// prefixes a revolving-door rank range walked one row swap at a time. Identical results.
enum class Kernel : int { tab = 0, rd = 1 };

// Limits of the device path (checked up front, std::invalid_argument).
constexpr uint32_t kMaxK = 1024;        // rows of a Gamma
constexpr uint32_t kMaxC = 64;          // level
constexpr uint32_t kMaxWords32 = 32;    // 32-bit words of a compacted row (n' <= 1024)

// Round keys (64-bit, min-reduced over blocks and ranks): the weight in bits 52..63 (weights
// are <= 2048); bit 51 set (kPosFlag): the task (< 2^32) in bits 19..50 and the winner's
// position in that tile in bits 0..18 (smem-side index << 11 | register-side index, the
// smallest of the tile's minimum); bit 51 clear: the task in bits 0..50 and the witness is
// searched again (tab_find). The minimum key is the lowest task, then position, of the
// round minimum either way.
constexpr int kKeyShift = 52;
constexpr unsigned long long kPosFlag = 1ull << 51;
constexpr int kPosBits = 19;

// GPU permutation search key layout (see permutation_search)
constexpr int kSearchMShift = 51;
constexpr int kSearchKShift = 41;

struct RoundResult {
    uint32_t w = UINT32_MAX;
    bool stopped = false;
    bool bounded = false;  // nothing below the cutoff: w == cutoff is only a lower bound
    uint64_t key = ~uint64_t{0};
    uint64_t combinations = 0;
    uint64_t evaluated = 0;
    uint64_t task_lo = 0, task_hi = 0;
    double ms = 0;
    // tile plan the round ran on (bit 0 set: valid; bit 1 pruning on; bit 2 revolving-door
    // plan); 0 = the engine's current setting. Engine::witness decodes the key with it.
    uint32_t plan_tag = 0;
};

// Pivot split of a level-c round (the "tab" kernel's enumeration): a sorted
// c-subset S = P ∪ Q with |P| = p, |Q| = s, e = max(P) < min(Q). For pivot e
// the prefixes are (p-1)-subsets of [0, e) plus e, NX(e) = C(e, p-1), and the
// suffixes are s-subsets of (e, k), NY(e) = C(k-1-e, s) — a prefix of one
// suffix table in reverse-colex order. Tiles are TX prefixes x YC suffixes.
struct TabPlan {
    uint32_t k = 0, c = 0, p = 0, s = 0, emin = 0, emax = 0;
    uint32_t TX = 0, YC = 0;
    std::vector<uint64_t> prefix; // tiles before pivot emin + i; size npiv + 1
    std::vector<uint8_t> tr;      // per pivot: 1 = transposed tiles (suffixes in smem)
    bool rd = false;              // prefixes in revolving-door order (Kernel::rd)
    uint64_t tiles() const { return prefix.empty() ? 0 : prefix.back(); }
};

// In-process exchange group (engine.cu): `world` engines in one process reduce each split
// round's key through stream-ordered events and a min kernel instead of NCCL.
struct ExchangeGroup;
// timeout_s < 0: MDG_GROUP_TIMEOUT seconds if set, else none (0 = none)
std::shared_ptr<ExchangeGroup> make_exchange_group(uint32_t world, double timeout_s = -1.0);
void abort_exchange_group(ExchangeGroup& g, const std::string& reason);

class Engine {
public:
    explicit Engine(int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // ranks == nullptr: raw matrices (no identity elision)
    void load(uint32_t m, uint32_t k, uint32_t n, const uint64_t* rows, const uint32_t* ranks);
    uint32_t m() const { return m_; }
    uint32_t k() const { return k_; }
    uint32_t n() const { return n_; }

    void set_kernel(Kernel kern);
    void set_pruning(bool on);
    Kernel kernel() const { return kernel_; }

    uint64_t tasks(uint32_t j, uint32_t c);
    // rank's contiguous task range of round (j, c) split `world` ways by codewords (tab_split)
    std::pair<uint64_t, uint64_t> split_range(uint32_t j, uint32_t c, uint32_t rank, uint32_t world);
    // cutoff: only weights < cutoff matter (0 = the exact round minimum). With a
    // cutoff the result is min(true minimum, cutoff) and `bounded` is set when no
    // codeword lies below it — what run_bz_loop's U = min(U, w) needs.
    // shared_bound: a split round of a multi-process run -- publish / poll the ranks' common
    // round key (shared_bound_create / _open), if one is mapped
    RoundResult round(uint32_t j, uint32_t c, uint32_t stop_at, uint64_t task_lo = 0,
                      uint64_t task_hi = UINT64_MAX, uint32_t cutoff = 0, bool shared_bound = false);
    // rank / world: this rank's contiguous share of the histogram kernel's tiles (about 1/world
    // of the codewords); with an NCCL communicator attached the counts are summed across the
    // ranks in stream, otherwise `hist` is this rank's partial histogram
    RoundResult round_hist(uint32_t j, uint32_t c, uint64_t* hist, uint32_t rank = 0, uint32_t world = 1);
    bool has_comm() const;
    // Cross-process shared bound: rank 0 creates a ring of round-key words
    // and hands its CUDA IPC handle to the other ranks (one process per GPU), which map it.
    // In every split round each tile result is also atomicMin_system-ed into the round's word
    // and every tile fetch polls it: one rank's find prunes and stops the others. The round's
    // result stays the reduction of the ranks' own keys. advance(): after a split round's
    // reduction (host-loop callers; the chained NCCL loop does it in stream).
    void shared_bound_create(uint8_t handle[64]);
    void shared_bound_open(const uint8_t handle[64]);
    void shared_bound_close();
    void shared_bound_advance();
    bool has_shared_bound() const;

    // The whole level loop with rounds chained on the stream (either kernel):
    // a device-side state carries U / L / done, a finalize kernel per round
    // applies run_bz_loop's updates, and the host only synchronizes after
    // enough enqueued work (or at the end) to look at `done`. world > 1 adds an
    // in-stream NCCL allreduce(min) of every round's key (nccl_init first).
    struct ChainRound {
        uint32_t c, j, w, U_after, bounded, L_after, level_end;
        uint64_t key, evaluated;
        double ms;
        uint32_t plan_tag; // the tile plan this round ran on (a fused level's rounds use larger tiles)
    };
    struct ChainResult {
        uint32_t U = 0, L = 0;
        bool done = false, capped = false;
        uint32_t plan_tag = 0;          // RoundResult::plan_tag of every round of the loop
        std::vector<ChainRound> rounds; // executed rounds, in loop order
    };
    // Gray-code brute force over all 2^k - 1 nonzero codewords of a k-row basis
    // (brute_force_gray, engines.cpp:480-558): d and the rows of one weight-d codeword.
    struct BruteResult {
        uint32_t d = 0;
        uint64_t evaluated = 0;
        double ms = 0;
        std::vector<uint32_t> idx;
    };
    BruteResult brute_force(uint32_t k, uint32_t n, const uint64_t* rows);

    // split_min: with world > 1 only rounds of >= split_min codewords are divided across
    // the ranks (and reduced); smaller rounds run whole on every rank.
    ChainResult chain_loop(uint32_t U0, uint32_t L0, uint32_t level_cap, bool exact,
                           uint32_t k_last, uint32_t rank = 0, uint32_t world = 1,
                           bool allreduce = false, uint64_t split_min = 1);
    std::vector<uint32_t> witness(uint32_t j, uint32_t c, const RoundResult& rr);

    // In-process multi-engine runs: attach this engine as member `rank` of an exchange group
    // (null: detach); chain_loop then reduces split rounds through the group, not NCCL.
    void group_attach(std::shared_ptr<ExchangeGroup> g, uint32_t rank);
    // Resident-SM count the tile plans assume (default: this device's). Multi-rank runs agree
    // on one value so every rank cuts a split round into the same tiles.
    void set_plan_sms(int sms);
    int plan_sms() const { return plan_sms_; }

    // NCCL (loaded at runtime) for the multi-GPU reduction
    void nccl_init(const uint8_t id[128], uint32_t rank, uint32_t world);
    void nccl_reduce_min(uint64_t* keys, uint32_t count);
    static void nccl_unique_id(uint8_t id[128]);

    int device() const { return device_; }
    int sm_count() const { return sms_; }

    // GPU permutation search (gsearch.cu): best (m, k_last, earliest trial) of `trials`
    // SplitMix64 / Fisher-Yates column orders of the k x n matrix `rows` (row-major u64),
    // packed as m << 51 | k_last << 41 | (2^41 - 1 - trial): m <= n <= 4096 needs 13 bits,
    // k_last <= k <= 512 needs 10.
    uint64_t permutation_search(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t trials,
                                uint64_t seed);
    struct CUstream_st* stream() const; // the engine's CUDA stream
    void* scratch(size_t bytes);         // a persistent device buffer (grows; never freed early)
    void count_launch();

    // counters (kernel launches, host<->device bytes) and a CUDA-event timer
    // on the engine's stream (host gaps between launches included)
    struct Counters { uint64_t launches = 0, h2d = 0, d2h = 0; };
    Counters counters() const;
    void reset_counters();
    void timer_start();
    double timer_stop_ms();

    struct Impl;

private:
    void check_round(uint32_t j, uint32_t c) const;
    int device_ = 0, sms_ = 0, plan_sms_ = 0;
    bool pdl_ = true; // programmatic dependent launch between chained rounds (MDG_PDL=0: off)
    double fuse_max_ = 4e9; // chained levels up to this many codewords run as one launch (MDG_FUSE_MAX)
    uint32_t m_ = 0, k_ = 0, n_ = 0;
    Kernel kernel_ = Kernel::tab;
    std::unique_ptr<Impl> impl_;
};

// tiles_per_block: the smallest tile count per resident block the plan aims for (0: the
// default, 2 -- or MDG_TILES_PER_BLOCK; exact-weight rounds take 8: their tiles run ~3x longer)
TabPlan make_tab_plan(uint32_t k, uint32_t c, uint32_t nw32, uint32_t resident_blocks, bool rd = false,
                      uint32_t tiles_per_block = 0);
uint32_t tab_yc(uint32_t nw32);
uint32_t tab_tx();
// kernel template width for a row of nw32 words (rows are zero-padded up to it)
uint32_t template_width(uint32_t nw32);
// codewords in tiles [0, t) of a plan, and rank's codeword-balanced contiguous tile range
uint64_t tab_codewords_before(const TabPlan& plan, uint64_t t);
std::pair<uint64_t, uint64_t> tab_split(const TabPlan& plan, uint32_t rank, uint32_t world);
// reconstruct the combination of tile `tile`, local prefix x / suffix y
void tab_decode(const TabPlan& plan, uint64_t tile, uint32_t x_local, uint32_t y_local,
                uint32_t* idx);

} // namespace mdg
