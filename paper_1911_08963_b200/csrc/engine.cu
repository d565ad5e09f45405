// Device side of the B200 Brouwer–Zimmermann round: one (c, Gamma_j) round =
// the minimum Hamming weight over all C(k, c) XOR-sums of c rows of Gamma_j
// (reference: round_* in proj/src/engines.cpp:175-443; level loop :447-476).
//
// Data layout in HBM / shared memory:
//   * Gamma_j is stored "compacted": its identity block (columns
//     [j*k, j*k + rank_j), rows [0, rank_j), gamma.cpp:44-71) is dropped, so a
//     row is NW = ceil((n - rank_j)/32) u32 words, and the weight of a sum
//     over row set S is |S ∩ [0, rank_j)| + popcount of the compacted sum.
//     For full-rank blocks that count is the constant c.
//   * suffix table (per Gamma, per suffix size s, built once and reused by
//     every level): all s-subsets Q of [0,k) in reverse-colex order, XOR-sum
//     (+ identity count) per entry, YS words per entry — the reference's
//     "saved additions" table (engines.cpp:96-151) turned into a GPU operand.
//
// Kernels (all integer; no tensor cores):
//   tab_round<NW,HID>  persistent grid over tiles (prefix chunk x suffix chunk, or
//                      transposed); smem items built per tile, each lane holds R
//                      register items; stage 1 bounds the weight from below (OR-folds
//                      of the words of X ^ Y, or one AND of two codewords' folds per
//                      pair: 3 LOP3 + 1 POPC for two codewords), the plan choosing per
//                      tile bound T; exact weights only where the bound can still win;
//                      warp __reduce_min_sync; global 64-bit atomicMin of
//                      (weight << 52 | tile | position); tile fetches poll the bound for early
//                      exit; in a chained loop the last block closes the round.
//                      With a revolving-door plan (Kernel::rd) the prefixes are a
//                      contiguous revolving-door rank range walked with one
//                      (row out ^ row in) XOR per step.
//   tab_level<NW,HID>  all rounds of a small level in one launch.
//   tab_find           re-evaluates the winning tile to name the witness (keys without
//                      the position: revolving-door plans, rounds of >= 2^32 tiles).
//   tab_hist           the full weight histogram of a round (per-warp smem bins).
//   tables_build       prefix / suffix tables; span_build / span_round: brute force.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <condition_variable>
#include <mutex>
#include <sstream>

#include "engine.hpp"

namespace mdg {

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw CudaError(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x);      \
    } while (0)

namespace {

constexpr int kWarps = 8;           // warps per block (tab kernels)
constexpr int kThreads = kWarps * 32;
constexpr int kTX = 256;            // prefixes per tile (= threads that build them)
constexpr int kFindX = 4;           // smem-side items per block of the witness search
constexpr int kFoldDrop = 16;       // fold-option flag: stage 1 leaves out the last word
constexpr int kFoldHalf = 32;       // fold-option flag: stage 1 folds the first ceil(NW/2) words
constexpr int kFold3 = 128;         // fold-option flag: one group over the first 3 words (NW >= 7)
constexpr int kFoldPair = 64;       // fold-option flag: two register items share one POPC
                                    // (popc of the AND of their folds bounds both weights)
constexpr int kPlanT = 128;         // stage-1 choice per tile bound T < kPlanT (above: exact)

// Stage-1 option of a round per tile bound T (host-sampled expected cost, the cheapest):
// code = G | kFoldDrop | kFoldHalf | kFold3 | kFoldPair, 0 = exact weights.
struct FoldPlan {
    uint8_t code[kPlanT];
};
constexpr uint32_t kBT = kMaxC + 1; // binomial table row stride

__host__ __device__ constexpr int r_for(int nw) { return nw <= 4 ? 8 : (nw <= 8 ? 4 : (nw <= 16 ? 2 : 1)); }
__host__ __device__ constexpr int stride_for(int words) {
    return words <= 2 ? 2 : ((words + 3) / 4) * 4;
}

// -------------------------------------------------------------- helpers
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t BT(const uint64_t* __restrict__ T, uint32_t x, uint32_t t) {
    return __ldg(T + size_t(x) * kBT + t);
}

// largest x in [i-1, hi-1] with C(x, i) <= r (colex unrank step)
__device__ __forceinline__ uint32_t colex_top(const uint64_t* __restrict__ T, uint64_t r,
                                              uint32_t i, uint32_t hi) {
    uint32_t lo = i - 1, h = hi - 1;
    while (lo < h) {
        uint32_t mid = (lo + h + 1) >> 1;
        if (BT(T, mid, i) <= r) lo = mid; else h = mid - 1;
    }
    return lo;
}

template <int NW>
__device__ __forceinline__ void load_row(const uint32_t* __restrict__ rows, uint32_t r,
                                         uint32_t (&v)[NW]) {
#pragma unroll
    for (int w = 0; w < NW; ++w) v[w] = __ldg(rows + size_t(r) * NW + w);
}

template <int NW>
__device__ __forceinline__ void xor_row(const uint32_t* __restrict__ rows, uint32_t r,
                                        uint32_t (&v)[NW]) {
#pragma unroll
    for (int w = 0; w < NW; ++w) v[w] ^= __ldg(rows + size_t(r) * NW + w);
}

// vector load of S consecutive u32 (S = 2 or a multiple of 4), 8/16-byte aligned
template <int S>
__device__ __forceinline__ void vload(const uint32_t* p, uint32_t (&v)[S]) {
    if constexpr (S == 2) {
        uint2 t = *reinterpret_cast<const uint2*>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
#pragma unroll
        for (int i = 0; i < S / 4; ++i) {
            uint4 t = *reinterpret_cast<const uint4*>(p + 4 * i);
            v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
        }
    }
}
template <int S>
__device__ __forceinline__ void vload_global(const uint32_t* __restrict__ p, uint32_t (&v)[S]) {
    if constexpr (S == 2) {
        uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
        v[0] = t.x; v[1] = t.y;
    } else {
#pragma unroll
        for (int i = 0; i < S / 4; ++i) {
            uint4 t = __ldg(reinterpret_cast<const uint4*>(p + 4 * i));
            v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
        }
    }
}

// Sum of the popcounts of N words with a carry-save adder chain (Harley–Seal):
// each CSA folds two more words into the running "ones" word with 2 LOP3
// (0x96 sum, 0xE8 majority) and emits one carry word of weight 2, reduced
// the same way. POPC count per codeword drops from N to 2 (N=3), 3 (N=4..5,7),
// 4 (N=6,8), 5 (N=16) — the XU pipe (16 POPC/clk/SM) is the binding unit,
// LOP3 runs 4x faster on the ALU pipe.
template <int N>
__device__ __forceinline__ uint32_t popsum(const uint32_t (&v)[N]) {
    if constexpr (N == 0) {
        return 0u;
    } else if constexpr (N == 1) {
        return __popc(v[0]);
    } else if constexpr (N == 2) {
        return __popc(v[0]) + __popc(v[1]);
    } else {
        constexpr int M = (N - 1) / 2;
        uint32_t carries[M];
        uint32_t ones = v[0];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const uint32_t b = v[1 + 2 * i], c = v[2 + 2 * i];
            const uint32_t t = ones ^ b ^ c;
            carries[i] = (ones & b) | (ones & c) | (b & c);
            ones = t;
        }
        uint32_t w = __popc(ones);
        if constexpr ((N - 1) % 2 == 1) w += __popc(v[N - 1]);
        return w + 2u * popsum<M>(carries);
    }
}

// acc + scale * (sum of the popcounts of N words): the same carry-save chain as popsum, the
// popcounts combined by multiply-adds whose multipliers are opaque registers (s[0] = scale,
// s[1] = 2 scale, ...) so ptxas issues them as IMAD on the FMA pipe instead of IADD3 / LEA on
// the ALU pipe -- the histogram kernel is ALU-bound on its LOP3s (ncu: 85 % busy)
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
template <int N>
__device__ __forceinline__ uint32_t popsum_mad(const uint32_t (&v)[N], uint32_t acc, const uint32_t* s) {
    if constexpr (N == 0) {
        return acc;
    } else if constexpr (N == 1) {
        return mad_u32(__popc(v[0]), s[0], acc);
    } else if constexpr (N == 2) {
        return mad_u32(__popc(v[1]), s[0], mad_u32(__popc(v[0]), s[0], acc));
    } else {
        constexpr int M = (N - 1) / 2;
        uint32_t carries[M];
        uint32_t ones = v[0];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const uint32_t b = v[1 + 2 * i], c = v[2 + 2 * i];
            const uint32_t t = ones ^ b ^ c;
            carries[i] = (ones & b) | (ones & c) | (b & c);
            ones = t;
        }
        acc = mad_u32(__popc(ones), s[0], acc);
        if constexpr ((N - 1) % 2 == 1) acc = mad_u32(__popc(v[N - 1]), s[0], acc);
        return popsum_mad<M>(carries, acc, s + 1);
    }
}

// weight of X ^ Y over words [B, E)
template <int B, int E, int S, int NW>
__device__ __forceinline__ uint32_t xor_weight(const uint32_t (&X)[S], const uint32_t (&Y)[NW]) {
    if constexpr (E <= B) {
        return 0u;
    } else {
        uint32_t a[E - B];
#pragma unroll
        for (int i = 0; i < E - B; ++i) a[i] = X[B + i] ^ Y[B + i];
        return popsum<E - B>(a);
    }
}

// OR of the NW words of X ^ Y: popc(fold) <= popc(X ^ Y) (every set bit of the
// fold is a set bit of some word) — a one-POPC lower bound on the weight.
// f | (x ^ y) as ONE 3-input LOP3 (LUT 0xF6): keeps the per-word XORs out of
// registers (the compiler would otherwise share them with the exact stage).
__device__ __forceinline__ uint32_t or_xor(uint32_t f, uint32_t x, uint32_t y) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xF6;" : "=r"(r) : "r"(f), "r"(x), "r"(y));
    return r;
}

template <int S, int NW>
__device__ __forceinline__ uint32_t xor_fold(const uint32_t (&X)[S], const uint32_t (&Y)[NW]) {
    uint32_t f = X[0] ^ Y[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) f = or_xor(f, X[i], Y[i]);
    return f;
}

// ------------------------------------------------------ suffix table build
// entry y: Q' = colex_unrank(y, s) ⊆ [0,k), Q = {k-1-q'}; XOR of rows(Q)
// (+ |Q ∩ [0, id_rows)| in word NW when HID).
// reverse = false builds the prefix table instead: Q = Q' itself (plain colex
// order, so the (p-1)-subsets of [0, e) are its first C(e, p-1) entries).
template <int NW, bool HID>
__global__ void ytab_build(const uint32_t* __restrict__ rows, const uint64_t* __restrict__ T,
                           uint32_t k, uint32_t s, uint32_t id_rows, uint64_t count,
                           uint32_t* __restrict__ out, bool reverse) {
    constexpr int YS = stride_for(NW + (HID ? 1 : 0));
    uint64_t y = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (y >= count) return;
    uint32_t acc[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) acc[w] = 0;
    uint32_t id = 0;
    uint64_t r = y;
    uint32_t hi = k;
    for (uint32_t i = s; i >= 1; --i) {
        uint32_t x = colex_top(T, r, i, hi);
        r -= BT(T, x, i);
        hi = x;
        uint32_t q = reverse ? k - 1 - x : x;
        xor_row<NW>(rows, q, acc);
        id += q < id_rows;
    }
    uint32_t* o = out + y * YS;
#pragma unroll
    for (int w = 0; w < YS; ++w) o[w] = w < NW ? acc[w] : (HID && w == NW ? id : 0u);
}

// Several tables in one launch (the tables of the first levels of a chained loop: one
// latency-bound launch instead of one per table and Gamma). Thread gi builds entry
// gi - begin of the job whose range holds gi, exactly as ytab_build.
constexpr int kMaxTableJobs = 48;
struct TableJob {
    const uint32_t* rows;
    uint32_t* out;
    uint64_t begin;
    uint32_t s, id_rows, reverse, pad;
};
struct TableJobs {
    uint32_t n, k;
    uint64_t total;
    TableJob job[kMaxTableJobs];
};

// Each thread builds kTabRun consecutive entries: it unranks the first (a binary search per
// element, dependent loads of the binomial table) and steps through the rest by the colex
// successor -- the lowest element that can grow grows by one and the ones below it reset to
// 0, 1, ... -- XORing only the rows that leave and enter (about two per entry instead of s).
constexpr uint32_t kTabRun = 8;
constexpr uint32_t kTabMaxS = 8; // longer subsets: every entry unranked

template <int NW, bool HID>
__global__ void tables_build(const __grid_constant__ TableJobs J, const uint64_t* __restrict__ T) {
    constexpr int YS = stride_for(NW + (HID ? 1 : 0));
    const uint64_t g0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kTabRun;
    if (g0 >= J.total) return;
    uint32_t acc[NW];
    uint32_t id = 0, jb = 0, c[kTabMaxS];
    uint64_t job_end = 0, y = 0;
    for (uint64_t gi = g0; gi < g0 + kTabRun && gi < J.total; ++gi, ++y) {
        const bool fresh = gi == g0 || gi == job_end;
        if (fresh) { // locate the job and unrank its entry
            jb = 0;
            for (uint32_t i = 1; i < J.n; ++i)
                if (J.job[i].begin <= gi) jb = i;
            job_end = jb + 1 < J.n ? J.job[jb + 1].begin : J.total;
            y = gi - J.job[jb].begin;
        }
        const TableJob& jo = J.job[jb];
        if (fresh || jo.s > kTabMaxS) {
#pragma unroll
            for (int w = 0; w < NW; ++w) acc[w] = 0;
            id = 0;
            uint64_t r = y;
            uint32_t hi = J.k;
            for (uint32_t i = jo.s; i >= 1; --i) {
                uint32_t x = colex_top(T, r, i, hi);
                r -= BT(T, x, i);
                hi = x;
                if (i <= kTabMaxS) c[i - 1] = x;
                uint32_t q = jo.reverse ? J.k - 1 - x : x;
                xor_row<NW>(jo.rows, q, acc);
                id += q < jo.id_rows;
            }
        } else { // colex successor of c[0..s) (ascending)
            uint32_t j = 0;
            while (j + 1 < jo.s && c[j] + 1 == c[j + 1]) ++j;
            for (uint32_t t = 0; t <= j; ++t) {
                const uint32_t nv = t < j ? t : c[j] + 1;
                if (nv == c[t]) continue;
                const uint32_t qo = jo.reverse ? J.k - 1 - c[t] : c[t];
                const uint32_t qn = jo.reverse ? J.k - 1 - nv : nv;
                xor_row<NW>(jo.rows, qo, acc);
                xor_row<NW>(jo.rows, qn, acc);
                id += (qn < jo.id_rows) - (qo < jo.id_rows);
                c[t] = nv;
            }
        }
        uint32_t* o = jo.out + y * YS;
#pragma unroll
        for (int w = 0; w < YS; ++w) o[w] = w < NW ? acc[w] : (HID && w == NW ? id : 0u);
    }
}

// Device-side state of the level loop (run_bz_loop, engines.cpp:447-476) when
// rounds are chained on the stream: round kernels read U / L / done at start,
// a one-thread finalize kernel applies U = min(U, w), the per-level L update,
// the fast path (U <= L) and termination (L >= U) exactly as the host loop.
struct ChainState {
    uint32_t U, L, done, exact;
    uint32_t run, pad;     // run: the chain_loop call's id, stamped into every record it closes
    unsigned long long t0; // %globaltimer at the loop's start (chain_stamp)
    uint32_t* progress;    // mapped pinned host words {levels closed, done} (null: none), see chain_loop
};
struct ChainRec {
    uint32_t c, j, w, U_after, bounded, ran, L_after, level_end;
    unsigned long long key, evaluated, t_ns; // t_ns: %globaltimer when the round closed
    unsigned long long run;                  // ChainState::run of the loop that closed the round
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}


// Close a chained round (run_bz_loop's per-round step, engines.cpp:456-472): the fast
// path (U <= L ends the loop, the round is not run), U = min(U, w) with the bounded-round
// rule, and after the last Gamma of a level L = max(L, lower_bound) and L >= U -> done.
__device__ __forceinline__ void finalize_round(ChainState* st, const unsigned long long* slot,
                                               ChainRec* rec, uint32_t c, uint32_t j,
                                               uint32_t last_of_level, uint32_t lb) {
    ChainRec r{};
    r.c = c;
    r.j = j;
    r.run = st->run;
    r.t_ns = globaltimer_ns();
    auto publish = [&](uint32_t levels_closed) { // host-visible progress (zero-copy, no sync)
        if (!st->progress) return;
        volatile uint32_t* p = st->progress;
        // posted writes, no fence: the host only polls them opportunistically (a system-scope
        // fence here cost ~2 % of the eight-code bench: it sits between a level and the next)
        if (st->done) p[1] = st->run; // tagged with the loop's id: a straggler of an earlier loop cannot end this one
        if (levels_closed) p[0] = levels_closed;
    };
    if (st->done || st->U <= st->L) { // fast path: the round is not run, the loop ends
        st->done = 1;
        r.ran = 0;
        *rec = r;
        publish(last_of_level ? c : 0u);
        return;
    }
    const uint32_t cutoff = st->exact ? 0u : st->U;
    unsigned long long key = *reinterpret_cast<volatile const unsigned long long*>(slot);
    uint32_t w = key == ~0ull ? 0xFFFFFFFFu : uint32_t(key >> kKeyShift);
    if (cutoff && (key == ~0ull || w >= cutoff)) {
        w = cutoff;
        key = ~0ull;
        r.bounded = 1;
    }
    r.ran = 1;
    r.w = w;
    r.key = key;
    r.evaluated = *reinterpret_cast<volatile const unsigned long long*>(slot + 1);
    if (w < st->U) st->U = w;
    r.U_after = st->U;
    if (last_of_level) {
        if (lb > st->L) st->L = lb;
        r.L_after = st->L;
        r.level_end = 1;
        if (st->L >= st->U) st->done = 1;
    }
    *rec = r;
    if (last_of_level) publish(c);
}

// In-process exchange group (ExchangeGroup): min of every member's round key, read
// after the stream waited on the members' round events (peer loads for members on other
// devices), written to this member's slot -- the group's allreduce(min) of one u64.
constexpr int kMaxGroup = 16;
struct GroupKeys {
    const unsigned long long* key[kMaxGroup];
    uint32_t n;
};
__global__ void group_min(GroupKeys g, unsigned long long* slot) {
    if (threadIdx.x == 0) {
        unsigned long long m = ~0ull;
        for (uint32_t i = 0; i < g.n; ++i) {
            const unsigned long long v = *reinterpret_cast<volatile const unsigned long long*>(g.key[i]);
            m = v < m ? v : m;
        }
        *slot = m;
    }
}

// chain start time stamp (device clock), read back with the records
__global__ void chain_stamp(unsigned long long* t) {
    if (threadIdx.x == 0) *t = globaltimer_ns();
}

struct TabArgs {
    const ChainState* st;          // non-null: cutoff / stop_at / skip from the chain state
    ChainState* fin_st;            // non-null: the last block closes the round (fused finalize)
    ChainRec* fin_rec;
    unsigned long long* blocks_done;
    uint32_t fin_c, fin_j, fin_last, fin_lb;
    const uint32_t* rows;
    const uint32_t* ytab;
    const uint32_t* xtab;          // optional prefix table (colex (p-1)-subset sums)
    const uint64_t* binom;
    const uint64_t* prefix;
    const uint8_t* tr;             // per pivot: 1 = transposed tiles (null: none)
    uint32_t k, p, s, emin, npiv, id_rows, add_const, stop_at, tx;
    uint32_t cutoff;               // only weights < cutoff matter (0 = exact round)
    FoldPlan fold;                 // stage-1 options (host-sampled), cheapest first
    uint32_t pos_key;              // 1: round keys carry the winner's position (kPosFlag layout)
    uint32_t rd;                   // 1: prefixes in revolving-door order; the round kernels walk
                                   //    them with one (row out ^ row in) XOR per step
    uint64_t tile_lo, tile_hi;
    unsigned long long* best_key;
    unsigned long long* shared_key; // split rounds of an exchange group: the members' common
                                    // key word (peer memory for members on other devices):
                                    // every tile result goes there too, every tile fetch polls
                                    // it -- one rank's find prunes and stops the others
    unsigned long long* evaluated;
    unsigned long long* counter;   // dynamic tile scheduler (next tile - tile_lo)
    unsigned long long* find_out;  // tab_find only
    uint32_t find_target;          // tab_find only
    uint32_t nbins;                // tab_hist only
    unsigned long long* hist;      // tab_hist only
};

// A tile of pivot e is an (smem side) x (register side) block of codewords. Normal
// orientation: smem side = prefixes (row e ^ (p-1)-subset sums), register side = suffixes
// from the suffix table. Transposed (tr = 1, pivots whose suffix range is shorter than a
// register tile): smem side = suffixes, register side = prefixes -- no masked lanes.
// x0/nx: smem-side start/count (<= TX); y0/nyv: register-side start/count (<= YC).
struct TileInfo {
    uint32_t e, nx, nyv, stop, tr;
    uint64_t x0, y0, tile;
    int32_t T;                     // pruning bound on the compacted weight (inclusive)
    int32_t G;                     // stage-1 fold groups for T (0 = exact weights)
};

// decode tile -> (pivot, prefix chunk, suffix chunk); thread 0 only
template <int YC>
__device__ __forceinline__ void decode_tile(const TabArgs& a, uint64_t tile, TileInfo& ti) {
    uint32_t lo = 0, hi = a.npiv - 1; // largest i with prefix[i] <= tile
    while (lo < hi) {
        uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(a.prefix + mid) <= tile) lo = mid; else hi = mid - 1;
    }
    uint32_t e = a.emin + lo;
    uint64_t local = tile - __ldg(a.prefix + lo);
    uint64_t NY = BT(a.binom, a.k - 1 - e, a.s);
    uint64_t NX = BT(a.binom, e, a.p - 1);
    const uint32_t tr = a.tr ? __ldg(a.tr + lo) : 0u;
    const uint64_t A = tr ? NY : NX, B = tr ? NX : NY; // smem side, register side
    uint64_t ntb = (B + YC - 1) / YC;
    uint64_t ta = local / ntb, tb = local - ta * ntb;
    ti.e = e;
    ti.tr = tr;
    ti.tile = tile;
    ti.x0 = ta * a.tx;
    ti.nx = uint32_t(umin64(uint64_t(a.tx), A - ti.x0));
    ti.y0 = tb * YC;
    ti.nyv = uint32_t(umin64(uint64_t(YC), B - ti.y0));
}

// decode_tile by a whole warp (all 32 lanes call it; lane 0 writes ti): the pivot search
// reads 32 prefix entries per step instead of a dependent binary search, and the two
// binomials load in parallel -- the short rounds of a level loop are latency-bound.
template <int YC>
__device__ __forceinline__ void decode_tile_warp(const TabArgs& a, uint64_t tile, TileInfo& ti) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t base = 0, lo = 0;
    uint64_t pv = 0, pre = 0;
    for (;;) {
        const uint32_t i = base + lane;
        const bool in = i < a.npiv;
        pv = in ? __ldg(a.prefix + i) : ~0ull;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, in && pv <= tile);
        if (m != 0xFFFFFFFFu || base + 32 >= a.npiv) {
            if (m) { // monotone prefix sums: the set lanes are a prefix of the warp
                lo = base + __popc(m) - 1;
                pre = __shfl_sync(0xFFFFFFFFu, pv, __popc(m) - 1);
            } else { // the pivot is the last entry of the previous chunk (base > 0)
                lo = base - 1;
                pre = __ldg(a.prefix + lo);
            }
            break;
        }
        base += 32;
    }
    const uint32_t e = a.emin + lo;
    const uint64_t b = lane == 0 ? BT(a.binom, a.k - 1 - e, a.s)
                     : lane == 1 ? BT(a.binom, e, a.p - 1)
                     : lane == 2 ? uint64_t(a.tr ? __ldg(a.tr + lo) : 0u) : 0;
    const uint64_t NY = __shfl_sync(0xFFFFFFFFu, b, 0), NX = __shfl_sync(0xFFFFFFFFu, b, 1);
    const uint32_t tr = uint32_t(__shfl_sync(0xFFFFFFFFu, b, 2));
    if (lane == 0) {
        const uint64_t A = tr ? NY : NX, B = tr ? NX : NY; // smem side, register side
        const uint64_t local = tile - pre;
        const uint64_t ntb = (B + YC - 1) / YC;
        const uint64_t ta = local / ntb, tb = local - ta * ntb;
        ti.e = e;
        ti.tr = tr;
        ti.tile = tile;
        ti.x0 = ta * a.tx;
        ti.nx = uint32_t(umin64(uint64_t(a.tx), A - ti.x0));
        ti.y0 = tb * YC;
        ti.nyv = uint32_t(umin64(uint64_t(YC), B - ti.y0));
    }
}

// Programmatic dependent launch (chained rounds): the prologue of round N+1 (tile decode,
// prefix build, suffix loads -- immutable tables only) overlaps round N's tail; the
// chain state is read after griddepcontrol.wait. No-ops without the launch attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// prefix sum for pivot e, colex rank x among (p-1)-subsets of [0, e)
template <int NW, bool HID>
__device__ __forceinline__ void build_prefix(const TabArgs& a, uint32_t e, uint64_t x,
                                             uint32_t* dst) {
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    uint32_t acc[NW];
    load_row<NW>(a.rows, e, acc);
    uint32_t id = e < a.id_rows;
    if (a.xtab) { // row e + entry x of the prefix table: no unranking
        uint32_t v[XS];
        vload_global<XS>(a.xtab + x * XS, v);
#pragma unroll
        for (int w = 0; w < NW; ++w) acc[w] ^= v[w];
        if (HID) id += v[NW];
#pragma unroll
        for (int w = 0; w < XS; ++w) dst[w] = w < NW ? acc[w] : (HID && w == NW ? id : 0u);
        return;
    }
    uint64_t r = x;
    uint32_t hi = e;
    for (uint32_t i = a.p - 1; i >= 1; --i) {
        uint32_t q = colex_top(a.binom, r, i, hi);
        r -= BT(a.binom, q, i);
        hi = q;
        xor_row<NW>(a.rows, q, acc);
        id += q < a.id_rows;
    }
#pragma unroll
    for (int w = 0; w < XS; ++w) dst[w] = w < NW ? acc[w] : (HID && w == NW ? id : 0u);
}

// XOR-sum of the rows of the rank-th t-subset of [0, e) in revolving-door order (Knuth
// 7.2.1.3 Algorithm R; the t-subsets of [0, e) are the first C(e, t) ranks of the order for
// any larger ground set, host.cpp rd_unrank) into acc; returns its identity-row count.
template <int NW>
__device__ __forceinline__ uint32_t rd_subset_sum(const TabArgs& a, uint32_t e, uint32_t t,
                                                  uint64_t rank, uint32_t (&acc)[NW]) {
    uint32_t id = 0;
    uint64_t r = rank;
    for (uint32_t i = t; i >= 1; --i) {
        // smallest x >= i-1 with C(x+1, i) > r
        uint32_t lo = i - 1, hi = e - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (BT(a.binom, mid + 1, i) > r) hi = mid; else lo = mid + 1;
        }
        xor_row<NW>(a.rows, lo, acc);
        id += lo < a.id_rows;
        r = BT(a.binom, lo + 1, i) - 1 - r;
    }
    return id;
}

// smem-side item t of the tile: a prefix (normal) or a suffix-table entry (transposed).
// Revolving-door plans (a.rd): prefix x = x0 + t is row e plus the x-th (p-1)-subset of
// [0, e) in revolving-door order; with `walk` (the round kernels) item t > 0 holds instead
// the difference to prefix x - 1 -- the XOR of the row leaving and the row entering -- and
// its identity-count change, so the kernel advances each codeword with one XOR per step.
template <int NW, bool HID>
__device__ __forceinline__ void build_smem_item(const TabArgs& a, const TileInfo& ti, uint32_t t,
                                                uint32_t* dst, bool walk = false) {
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    if (a.rd) {
        const uint64_t x = ti.x0 + t;
        uint32_t acc[NW];
        uint32_t id;
        if (walk && t > 0) {
            uint32_t prev[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) acc[w] = prev[w] = 0;
            id = rd_subset_sum<NW>(a, ti.e, a.p - 1, x, acc);
            id -= rd_subset_sum<NW>(a, ti.e, a.p - 1, x - 1, prev); // signed change, mod 2^32
#pragma unroll
            for (int w = 0; w < NW; ++w) acc[w] ^= prev[w];
        } else {
            load_row<NW>(a.rows, ti.e, acc);
            id = (ti.e < a.id_rows) + rd_subset_sum<NW>(a, ti.e, a.p - 1, x, acc);
        }
#pragma unroll
        for (int w = 0; w < XS; ++w) dst[w] = w < NW ? acc[w] : (HID && w == NW ? id : 0u);
        return;
    }
    if (!ti.tr) {
        build_prefix<NW, HID>(a, ti.e, ti.x0 + t, dst);
        return;
    }
    uint32_t v[XS];
    vload_global<XS>(a.ytab + (ti.x0 + t) * XS, v);
#pragma unroll
    for (int w = 0; w < XS; ++w) dst[w] = v[w];
}

// register side of the tile: R entries per thread (lane-interleaved); lanes past nyv
// duplicate entry y0 and are flagged invalid
template <int NW, bool HID>
__device__ __forceinline__ void load_suffixes(const TabArgs& a, const TileInfo& ti,
                                              uint32_t (&Y)[r_for(NW)][NW],
                                              uint32_t (&idY)[r_for(NW)],
                                              bool (&valid)[r_for(NW)]) {
    constexpr int R = r_for(NW);
    constexpr int YS = stride_for(NW + (HID ? 1 : 0));
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (ti.tr) { // prefixes: row e ^ prefix-table entry (the plan only transposes with a table)
        uint32_t row[NW];
        load_row<NW>(a.rows, ti.e, row);
        const uint32_t id_e = ti.e < a.id_rows;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t yl = r * kThreads + warp * 32 + lane;
            valid[r] = yl < ti.nyv;
            uint64_t x = ti.y0 + (valid[r] ? yl : 0u);
            uint32_t v[YS];
            vload_global<YS>(a.xtab + x * YS, v);
#pragma unroll
            for (int w = 0; w < NW; ++w) Y[r][w] = row[w] ^ v[w];
            idY[r] = HID ? id_e + v[NW] : 0u;
        }
        return;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        uint32_t yl = r * kThreads + warp * 32 + lane;
        valid[r] = yl < ti.nyv;
        uint64_t y = ti.y0 + (valid[r] ? yl : 0u); // invalid lanes duplicate entry y0
        uint32_t v[YS];
        vload_global<YS>(a.ytab + y * YS, v);
#pragma unroll
        for (int w = 0; w < NW; ++w) Y[r][w] = v[w];
        idY[r] = HID ? v[NW] : 0u;
    }
}

// OR-folds of the words of X ^ Y in G contiguous groups: sum_g popc(fold_g) is a
// lower bound on the weight (G POPCs); larger G = tighter bound for sparse codewords.
// Only the first NWF words take part (NWF = NW, or NW - 1 when the last word holds a few
// bits only: its fold would cost a LOP3 per codeword for almost no bound).
template <int G, int S, int NW, int NWF = NW>
__device__ __forceinline__ uint32_t fold_bound(const uint32_t (&X)[S], const uint32_t (&Y)[NW],
                                               uint32_t lb = 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int b = g * NWF / G, e = (g + 1) * NWF / G;
        if (b < e) {
            uint32_t f = X[b] ^ Y[b];
#pragma unroll
            for (int i = b + 1; i < e; ++i) f = or_xor(f, X[i], Y[i]);
            lb += __popc(f);
        }
    }
    return lb;
}

template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return r;
}

// Pair bound: popc(fold(X ^ Ya) & fold(X ^ Yb)) is at most each of the two fold bounds, so
// it bounds both weights from below with one POPC for two codewords. With dense folds (a bit
// set w.p. 3/4 for two words) the AND keeps 9/16 of the bits: a weaker bound that still
// rejects nearly every pair at the deep levels' small T, and the XU pipe stops binding.
// For a two-word fold it takes 3 LOP3 instead of 5: per bit the AND of the two folds is 1
// iff the smem item's bit pair x = (x0, x1) is neither a's nor b's. With
// d = x ^ a and c = a ^ b: c = 00 -> d0 | d1; c = 10 -> d1 (x0 is free); c = 01 -> d0;
// c = 11 -> d0 ^ d1 (x in {a, ~a}). So with per-pair constants K0 = ~(c0 & ~c1),
// K1 = ~(c1 & ~c0), KX = c0 & c1 (register side, built once per tile):
//   u = (x0 ^ a0) & K0, v = (x1 ^ a1) & K1, bound bits = KX ? u ^ v : u | v.
struct Pair2 { uint32_t k0, k1, kx; };
__device__ __forceinline__ Pair2 pair2_consts(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
    const uint32_t c0 = a0 ^ b0, c1 = a1 ^ b1;
    Pair2 k{~(c0 & ~c1), ~(c1 & ~c0), c0 & c1};
    // opaque to the compiler: under register pressure it would rebuild them from the
    // register items inside the smem loop (2 LOP3 each) instead of keeping them
    asm volatile("" : "+r"(k.k0), "+r"(k.k1), "+r"(k.kx));
    return k;
}
__device__ __forceinline__ uint32_t pair2_bits(uint32_t x0, uint32_t x1, uint32_t a0, uint32_t a1,
                                               const Pair2& k) {
    const uint32_t u = lop3<0x28>(x0, a0, k.k0); // (x0 ^ a0) & k0
    const uint32_t v = lop3<0x28>(x1, a1, k.k1); // (x1 ^ a1) & k1
    return lop3<0x7C>(u, v, k.kx);               // kx ? u ^ v : u | v
}

// The tile searches track the lane's best as weight * 256 + (smem index of its first
// occurrence): one shift-add and the same min per exactly weighed group. The kernel then
// names the register item (warp_round_key) and the round key carries the position, so no
// witness re-search is needed. (A factor of 257 would make it an IMAD on the FMA pipe, but
// measured 9 % slower on the pruned level-7 round.) kNone: nothing at or below the bound.
constexpr uint32_t kNone = 0xFFFFFFFFu;
#ifndef MDG_PACKX
#define MDG_PACKX 256
#endif
constexpr uint32_t kPackX = MDG_PACKX;
__device__ __forceinline__ uint32_t pack_best(uint32_t w, uint32_t xi) { return w * kPackX + xi; }
__device__ __forceinline__ uint32_t best_weight(uint32_t b) { return b == kNone ? kNone : b / kPackX; }

// Exact weights of register items [r0, r0 + n) against smem item xi; lowers best and T.
template <int NW, bool HID, int XS, int R>
__device__ __forceinline__ void group_exact(const uint32_t (&X)[XS], const uint32_t (&Y)[R][NW],
                                            const uint32_t (&idY)[R], int r0, int n, uint32_t xi,
                                            uint32_t& best, int32_t& T) {
    uint32_t m = kNone;
#pragma unroll
    for (int r = 0; r < n; ++r) {
        uint32_t w = xor_weight<0, NW, XS, NW>(X, Y[r0 + r]);
        if (HID) w += X[NW] + idY[r0 + r];
        m = min(m, w);
    }
    best = min(best, pack_best(m, xi));
    T = min(T, int32_t(m));
}

// Pair bounds of smem item X against the register items (one per two items, pair2_bits).
template <int NW, bool HID, int XS, int R>
__device__ __forceinline__ void pair_bounds(const uint32_t (&X)[XS], const uint32_t (&Y)[R][NW],
                                            const uint32_t (&idY)[R], const Pair2 (&K2)[R / 2],
                                            uint32_t (&lp)[R / 2]) {
#pragma unroll
    for (int b = 0; b < R / 2; ++b) {
        const uint32_t id = HID ? min(idY[2 * b], idY[2 * b + 1]) : 0u;
        lp[b] = id + __popc(pair2_bits(X[0], X[1], Y[2 * b][0], Y[2 * b][1], K2[b]));
    }
}

// A smem item whose pair bounds were not all rejected by a vote: per vote group of GP items
// the pair bounds again, then the single-item folds (vote groups of GR), then exact weights.
template <int NW, bool HID, int G, int NWF, int XS, int R, int GP, int GR>
__device__ __forceinline__ void pair_fall_through(const uint32_t (&X)[XS], const uint32_t (&Y)[R][NW],
                                                  const uint32_t (&idY)[R], const uint32_t (&lp)[R / 2],
                                                  uint32_t xi, uint32_t& best, int32_t& T) {
#pragma unroll
    for (int g0 = 0; g0 < R; g0 += GP) {
        uint32_t gmin = lp[g0 / 2];
#pragma unroll
        for (int b = 1; b < GP / 2; ++b) gmin = min(gmin, lp[g0 / 2 + b]);
        const int32_t Tx = HID ? T - int32_t(X[NW]) : T;
        if (__any_sync(0xFFFFFFFFu, int32_t(gmin) <= Tx)) {
#pragma unroll
            for (int h0 = g0; h0 < g0 + GP; h0 += GR) {
                uint32_t hmin = 0xFFFFFFFFu;
#pragma unroll
                for (int r = 0; r < GR; ++r)
                    hmin = min(hmin, fold_bound<G, XS, NW, NWF>(X, Y[h0 + r], HID ? idY[h0 + r] : 0u));
                const int32_t Th = HID ? T - int32_t(X[NW]) : T; // T may have dropped
                if (__any_sync(0xFFFFFFFFu, int32_t(hmin) <= Th))
                    group_exact<NW, HID>(X, Y, idY, h0, GR, xi, best, T);
            }
        }
    }
}

// The bound-pruned walk with G fold groups over the first NWF words (see tile_min).
// PAIR (one fold group of two words): a pre-filter of one bound per two register items
// (pair2_bits); two smem items share one warp vote over all their pair bounds (half the
// vote / min / loop overhead per codeword), and an item the vote cannot reject falls
// through to pair_fall_through.
template <int NW, bool HID, int G, int NWF = NW, bool PAIR = false>
__device__ __forceinline__ uint32_t tile_min_pruned(const uint32_t* xs, uint32_t x_begin, uint32_t nx,
                                                    const uint32_t (&Y)[r_for(NW)][NW],
                                                    const uint32_t (&idY)[r_for(NW)], int32_t T) {
    constexpr int R = r_for(NW);
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
#ifndef MDG_VOTE_GROUP
#define MDG_VOTE_GROUP 4
#endif
#ifndef MDG_PAIR_VOTE_GROUP
#define MDG_PAIR_VOTE_GROUP 8
#endif
    constexpr int GR = R >= MDG_VOTE_GROUP ? MDG_VOTE_GROUP : R;           // single-bound vote
    constexpr int GP = R >= MDG_PAIR_VOTE_GROUP ? MDG_PAIR_VOTE_GROUP : R; // pair-bound vote
    static_assert(!PAIR || (GP % 2 == 0 && GP % GR == 0), "pair vote groups");
    static_assert(!PAIR || (G == 1 && NWF == 2), "pair bounds: one two-word fold group");
    uint32_t best = 0xFFFFFFFFu;
    uint32_t xi = x_begin;
    if constexpr (PAIR) {
        Pair2 K2[R / 2];
#pragma unroll
        for (int b = 0; b < R / 2; ++b) K2[b] = pair2_consts(Y[2 * b][0], Y[2 * b][1], Y[2 * b + 1][0], Y[2 * b + 1][1]);
#ifndef MDG_PAIR_X2
#define MDG_PAIR_X2 1
#endif
        if (MDG_PAIR_X2) {
            for (; xi + 1 < nx; xi += 2) {
                uint32_t X0[XS], X1[XS], l0[R / 2], l1[R / 2];
                vload<XS>(xs + xi * XS, X0);
                vload<XS>(xs + (xi + 1) * XS, X1);
                pair_bounds<NW, HID>(X0, Y, idY, K2, l0);
                pair_bounds<NW, HID>(X1, Y, idY, K2, l1);
                uint32_t m0 = l0[0], m1 = l1[0];
#pragma unroll
                for (int b = 1; b < R / 2; ++b) m0 = min(m0, l0[b]), m1 = min(m1, l1[b]);
                const int32_t T0 = HID ? T - int32_t(X0[NW]) : T, T1 = HID ? T - int32_t(X1[NW]) : T;
                if (__any_sync(0xFFFFFFFFu, int32_t(m0) <= T0 || int32_t(m1) <= T1)) {
                    pair_fall_through<NW, HID, G, NWF, XS, R, GP, GR>(X0, Y, idY, l0, xi, best, T);
                    pair_fall_through<NW, HID, G, NWF, XS, R, GP, GR>(X1, Y, idY, l1, xi + 1, best, T);
                }
            }
        }
        for (; xi < nx; ++xi) {
            uint32_t X[XS], l[R / 2];
            vload<XS>(xs + xi * XS, X);
            pair_bounds<NW, HID>(X, Y, idY, K2, l);
            pair_fall_through<NW, HID, G, NWF, XS, R, GP, GR>(X, Y, idY, l, xi, best, T);
        }
        return best;
    }
    // the single-bound vote groups of one smem item (T may drop between groups)
    auto item_groups = [&](const uint32_t (&X)[XS], const uint32_t (&lb)[R], uint32_t x) {
        // partial identity block: the register item's count starts the popcount sum (one
        // IADD3 with the fold POPCs) and the smem item's comes off the bound once per row
        const int32_t Tx = HID ? T - int32_t(X[NW]) : T;
#pragma unroll
        for (int g0 = 0; g0 < R; g0 += GR) {
            uint32_t gmin = lb[g0];
#pragma unroll
            for (int r = 1; r < GR; ++r) gmin = min(gmin, lb[g0 + r]);
            if (__any_sync(0xFFFFFFFFu, int32_t(gmin) <= Tx)) group_exact<NW, HID>(X, Y, idY, g0, GR, x, best, T);
        }
    };
#ifndef MDG_SINGLE_X2
#define MDG_SINGLE_X2 1
#endif
    if (MDG_SINGLE_X2 && R <= 4) { // R = 8 (NW <= 4): 16 bounds per vote fall through more
                                   // and the second item's registers cost more than the vote
                                   // saves (config 4 Gamma_0 level 7: 541 -> 563 ms; Gamma_1,
                                   // R = 4: 739 -> 707 ms)
        // two smem items share one warp vote over all their bounds (as the pair path): half
        // the vote / branch / loop instructions per codeword; a pair the vote cannot reject
        // takes the per-item groups (T only decreases, so the shared vote is conservative)
        for (; xi + 1 < nx; xi += 2) {
            uint32_t X0[XS], X1[XS], l0[R], l1[R];
            vload<XS>(xs + xi * XS, X0);
            vload<XS>(xs + (xi + 1) * XS, X1);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                l0[r] = fold_bound<G, XS, NW, NWF>(X0, Y[r], HID ? idY[r] : 0u);
                l1[r] = fold_bound<G, XS, NW, NWF>(X1, Y[r], HID ? idY[r] : 0u);
            }
            uint32_t m0 = l0[0], m1 = l1[0];
#pragma unroll
            for (int r = 1; r < R; ++r) m0 = min(m0, l0[r]), m1 = min(m1, l1[r]);
            const int32_t T0 = HID ? T - int32_t(X0[NW]) : T, T1 = HID ? T - int32_t(X1[NW]) : T;
            if (__any_sync(0xFFFFFFFFu, int32_t(m0) <= T0 || int32_t(m1) <= T1)) {
                item_groups(X0, l0, xi);
                item_groups(X1, l1, xi + 1);
            }
        }
    }
    for (; xi < nx; ++xi) {
        uint32_t X[XS], lb[R];
        vload<XS>(xs + xi * XS, X);
#pragma unroll
        for (int r = 0; r < R; ++r) lb[r] = fold_bound<G, XS, NW, NWF>(X, Y[r], HID ? idY[r] : 0u);
        item_groups(X, lb, xi);
    }
    return best;
}

template <int NW, bool HID>
__device__ __forceinline__ uint32_t tile_min_exact(const uint32_t* xs, uint32_t x_begin, uint32_t nx,
                                                   const uint32_t (&Y)[r_for(NW)][NW],
                                                   const uint32_t (&idY)[r_for(NW)]) {
    constexpr int R = r_for(NW);
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    uint32_t best = kNone;
    for (uint32_t xi = x_begin; xi < nx; ++xi) {
        uint32_t X[XS];
        vload<XS>(xs + xi * XS, X);
        uint32_t m = kNone;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t w = xor_weight<0, NW, XS, NW>(X, Y[r]);
            if (HID) w += X[NW] + idY[r];
            m = min(m, w);
        }
        best = min(best, pack_best(m, xi));
    }
    return best;
}

// the stage-1 variant for fold code G (without the pair flag); exact if none
template <int NW, bool HID>
__device__ __forceinline__ uint32_t tile_min_folds(const uint32_t* xs, uint32_t x_begin, uint32_t nx,
                                                   const uint32_t (&Y)[r_for(NW)][NW],
                                                   const uint32_t (&idY)[r_for(NW)], int32_t T, int G) {
    constexpr int ND = NW >= 2 ? NW - 1 : NW, NH = (NW + 1) / 2; // drop / half fold widths
    if (G == 1) return tile_min_pruned<NW, HID, 1, NW>(xs, x_begin, nx, Y, idY, T);
    if constexpr (NW >= 3) {
        if (G == 2) return tile_min_pruned<NW, HID, 2, NW>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (NW >= 5) {
        if (G == 4) return tile_min_pruned<NW, HID, 4, NW>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (NW >= 2) {
        if (G == (1 | kFoldDrop)) return tile_min_pruned<NW, HID, 1, ND>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (ND >= 3 && NW >= 2) {
        if (G == (2 | kFoldDrop)) return tile_min_pruned<NW, HID, 2, ND>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (ND >= 5 && NW >= 2) {
        if (G == (4 | kFoldDrop)) return tile_min_pruned<NW, HID, 4, ND>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (NW >= 3) {
        if (G == (1 | kFoldHalf)) return tile_min_pruned<NW, HID, 1, NH>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (NH >= 3 && NW >= 3) {
        if (G == (2 | kFoldHalf)) return tile_min_pruned<NW, HID, 2, NH>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (NH >= 5 && NW >= 3) {
        if (G == (4 | kFoldHalf)) return tile_min_pruned<NW, HID, 4, NH>(xs, x_begin, nx, Y, idY, T);
    }
    if constexpr (NW >= 7) {
        if (G == (1 | kFold3)) return tile_min_pruned<NW, HID, 1, 3>(xs, x_begin, nx, Y, idY, T);
    }
    return tile_min_exact<NW, HID>(xs, x_begin, nx, Y, idY);
}

// Minimum of (compacted weight + identity count) over prefixes xs[x_begin, nx) x the
// lane's R suffixes, considering only values <= T (T < 0: none). Values above T may be
// reported as "none" (0xFFFFFFFF) or exactly — never as anything smaller than the
// truth. G (warp-uniform): 0 = exact weights for every codeword; 1, 2, 4 = stage-1
// lower bound from that many OR-fold groups (| kFoldPair: one bound per two register
// items), exact weight only for warp groups of 4 suffixes in which some lane can still
// reach T (a real warp-uniform branch: a per-codeword vote gets if-converted and the
// predicated POPCs would still occupy the XU pipe). T must be warp-uniform on entry.
template <int NW, bool HID>
__device__ __forceinline__ uint32_t tile_min(const uint32_t* xs, uint32_t x_begin, uint32_t nx,
                                             const uint32_t (&Y)[r_for(NW)][NW],
                                             const uint32_t (&idY)[r_for(NW)], int32_t T,
                                             int G) {
    if (T < 0) return 0xFFFFFFFFu; // every codeword here is above the bound
    // pair codes exist for a single two-word fold group only: all of NW = 2, the first two
    // words of NW = 3 (drop) or 4 (half) -- the host plans no other
    if constexpr (NW >= 2 && NW <= 4 && r_for(NW) >= 2) {
        if (G & kFoldPair) return tile_min_pruned<NW, HID, 1, 2, true>(xs, x_begin, nx, Y, idY, T);
    }
    return tile_min_folds<NW, HID>(xs, x_begin, nx, Y, idY, T, G & ~kFoldPair);
}

// ------------------------------------------------ revolving-door walk (Kernel::rd)
// Stage-1 bound of an accumulated codeword: OR-folds of G word groups of A (first NWF words).
template <int G, int NW, int NWF = NW>
__device__ __forceinline__ uint32_t fold_or_bound(const uint32_t (&A)[NW], uint32_t lb) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int b = g * NWF / G, e = (g + 1) * NWF / G;
        if (b < e) {
            uint32_t f = A[b];
#pragma unroll
            for (int i = b + 1; i < e; ++i) f |= A[i];
            lb += __popc(f);
        }
    }
    return lb;
}

template <int NW>
__device__ __forceinline__ uint32_t popc_words(const uint32_t (&A)[NW]) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) w += __popc(A[i]);
    return w;
}

// The revolving-door walk of a tile: register item r starts as its suffix sum and takes
// smem item 0 (the first prefix) and then, step by step, each (row out ^ row in) difference
// -- consecutive prefixes in revolving-door order differ by one row swap -- so every step
// is one XOR per word on codewords held in registers (north_star's formulation). Bound
// pruning as tile_min (G: 0 = exact; 1/2/4 groups, | kFoldDrop). A and idA are consumed.
template <int NW, bool HID, int G, int NWF = NW, bool PAIR = false>
__device__ __forceinline__ uint32_t walk_min(const uint32_t* xs, uint32_t nx,
                                             uint32_t (&A)[r_for(NW)][NW], uint32_t (&idA)[r_for(NW)],
                                             int32_t T) {
    constexpr int R = r_for(NW);
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    constexpr int GR = R >= MDG_VOTE_GROUP ? MDG_VOTE_GROUP : R;
    uint32_t best = 0xFFFFFFFFu;
    for (uint32_t xi = 0; xi < nx; ++xi) {
        uint32_t X[XS];
        vload<XS>(xs + xi * XS, X);
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int w = 0; w < NW; ++w) A[r][w] ^= X[w];
            if (HID) idA[r] += X[NW];
        }
        if (G == 0) {
            uint32_t m = kNone;
#pragma unroll
            for (int r = 0; r < R; ++r) m = min(m, popc_words<NW>(A[r]) + (HID ? idA[r] : 0u));
            best = min(best, pack_best(m, xi));
            continue;
        }
        if constexpr (PAIR) { // one bound per two codewords: popc(fold_a & fold_b), 2 LOP3 per pair
            static_assert(G == 1 && NWF == 2 && R % 2 == 0, "walk pair bound: one two-word fold");
            uint32_t pmin = kNone;
#pragma unroll
            for (int b = 0; b < R / 2; ++b) {
                const uint32_t fa = A[2 * b][0] | A[2 * b][1];
                uint32_t g;
                asm("lop3.b32 %0, %1, %2, %3, 0xA8;" : "=r"(g) : "r"(A[2 * b + 1][0]), "r"(A[2 * b + 1][1]), "r"(fa));
                pmin = min(pmin, __popc(g) + (HID ? min(idA[2 * b], idA[2 * b + 1]) : 0u));
            }
            if (!__any_sync(0xFFFFFFFFu, int32_t(pmin) <= T)) continue;
        }
        uint32_t lb[R];
#pragma unroll
        for (int r = 0; r < R; ++r) lb[r] = fold_or_bound<(G > 0 ? G : 1), NW, NWF>(A[r], HID ? idA[r] : 0u);
#pragma unroll
        for (int g0 = 0; g0 < R; g0 += GR) {
            uint32_t gmin = lb[g0];
#pragma unroll
            for (int r = 1; r < GR; ++r) gmin = min(gmin, lb[g0 + r]);
            if (__any_sync(0xFFFFFFFFu, int32_t(gmin) <= T)) {
                uint32_t m = kNone;
#pragma unroll
                for (int r = 0; r < GR; ++r)
                    m = min(m, popc_words<NW>(A[g0 + r]) + (HID ? idA[g0 + r] : 0u));
                best = min(best, pack_best(m, xi));
                T = min(T, int32_t(m));
            }
        }
    }
    return best;
}

template <int NW, bool HID>
__device__ __forceinline__ uint32_t tile_min_walk(const uint32_t* xs, uint32_t nx,
                                                  uint32_t (&A)[r_for(NW)][NW],
                                                  uint32_t (&idA)[r_for(NW)], int32_t T, int G) {
    if (T < 0) return 0xFFFFFFFFu;
    if constexpr (NW >= 2 && NW <= 4) // pair codes: one two-word fold group (see tile_min)
        if ((G & kFoldPair) && (G & 15) == 1) return walk_min<NW, HID, 1, 2, true>(xs, nx, A, idA, T);
    G &= ~kFoldPair;
    constexpr int ND = NW >= 2 ? NW - 1 : NW, NH = (NW + 1) / 2;
    if constexpr (NW >= 2) {
        if (G == (1 | kFoldDrop)) return walk_min<NW, HID, 1, ND>(xs, nx, A, idA, T);
    }
    if constexpr (ND >= 3 && NW >= 2) {
        if (G == (2 | kFoldDrop)) return walk_min<NW, HID, 2, ND>(xs, nx, A, idA, T);
    }
    if constexpr (ND >= 5 && NW >= 2) {
        if (G == (4 | kFoldDrop)) return walk_min<NW, HID, 4, ND>(xs, nx, A, idA, T);
    }
    if constexpr (NW >= 3) {
        if (G == (1 | kFoldHalf)) return walk_min<NW, HID, 1, NH>(xs, nx, A, idA, T);
    }
    if constexpr (NH >= 3 && NW >= 3) {
        if (G == (2 | kFoldHalf)) return walk_min<NW, HID, 2, NH>(xs, nx, A, idA, T);
    }
    if constexpr (NH >= 5 && NW >= 3) {
        if (G == (4 | kFoldHalf)) return walk_min<NW, HID, 4, NH>(xs, nx, A, idA, T);
    }
    if constexpr (NW >= 7) {
        if (G == (1 | kFold3)) return walk_min<NW, HID, 1, 3>(xs, nx, A, idA, T);
    }
    if (G == 1) return walk_min<NW, HID, 1>(xs, nx, A, idA, T);
    if constexpr (NW >= 3) {
        if (G == 2) return walk_min<NW, HID, 2>(xs, nx, A, idA, T);
    }
    if constexpr (NW >= 5) {
        if (G == 4) return walk_min<NW, HID, 4>(xs, nx, A, idA, T);
    }
    return walk_min<NW, HID, 0>(xs, nx, A, idA, T);
}

// fold groups for bound T: the smallest G whose stage-1 bound still rejects almost every
// codeword at T (lim[] from the host's density estimate; -1 = unusable), else 0 (exact)
// Cheapest first: fewer groups (POPCs) first, and at equal G the fold without the last
// (nearly empty) word (limd, kFoldDrop: one LOP3 less per codeword).
__device__ __forceinline__ int pick_groups(int32_t T, const int32_t (&lim)[4]) {
    if (T <= lim[3]) return 1 | kFoldPair; // pair bound over words 0-1 (NW 2..4, see tile_min)
    if (T <= lim[0]) return 1;
    if (T <= lim[1]) return 2;
    if (T <= lim[2]) return 4;
    return 0;
}
__device__ __forceinline__ int pick_fold(int32_t T, const FoldPlan& fp) {
    return (T >= 0 && T < kPlanT) ? int(fp.code[T]) : 0;
}

// The warp's contribution to a round key from the lanes' packed bests (pack_best): with
// pos_key the smallest (smem index, register index) of the warp's minimum --
// the lane re-evaluates its R register items at its best smem index and takes the first
// valid one of that weight (duplicated lanes past the tile's edge are not positions; the
// item they duplicate is evaluated by its own lane) -- packed as (weight << 19 | xi << 11 |
// yl), reduced over the warp. Returns the warp's key (kKeyShift / kPosFlag layout, engine.hpp)
// or ~0 if it has nothing below the cutoff.
template <int NW, bool HID>
__device__ __forceinline__ unsigned long long warp_round_key(uint32_t bc, const uint32_t* xs,
                                                             const uint32_t (&Y)[r_for(NW)][NW],
                                                             const uint32_t (&idY)[r_for(NW)],
                                                             uint32_t nyv, uint32_t add,
                                                             uint32_t cutoff, uint32_t pos_key, uint64_t tile) {
    constexpr int R = r_for(NW);
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    uint32_t comb = kNone;
    if (bc != kNone) {
        const uint32_t w = best_weight(bc), xi = bc - w * kPackX;
        if (pos_key) {
            uint32_t X[XS];
            vload<XS>(xs + xi * XS, X);
            uint32_t yl = kNone;
#pragma unroll
            for (int r = R - 1; r >= 0; --r) {
                uint32_t wr = xor_weight<0, NW, XS, NW>(X, Y[r]);
                if (HID) wr += X[NW] + idY[r];
                const uint32_t y = uint32_t(r) * kThreads + threadIdx.x; // valid below nyv
                if (y < nyv && wr == w) yl = y;
            }
            if (yl != kNone) comb = ((w + add) << kPosBits) | (xi << 11) | yl;
        } else {
            comb = w + add;
        }
    }
    comb = __reduce_min_sync(0xFFFFFFFFu, comb);
    if (comb == kNone) return ~0ull;
    const uint32_t w = pos_key ? comb >> kPosBits : comb;
    if (cutoff != 0 && w >= cutoff) return ~0ull;
    return pos_key ? (static_cast<unsigned long long>(w) << kKeyShift) | kPosFlag | (tile << kPosBits) |
                         (comb & ((1u << kPosBits) - 1))
                   : (static_cast<unsigned long long>(w) << kKeyShift) | tile;
}

#ifndef MDG_MINBLK_SMALL
#define MDG_MINBLK_SMALL 5
#endif
template <int NW, bool HID>
__global__ void __launch_bounds__(kThreads, NW <= 2 ? MDG_MINBLK_SMALL : 4) tab_round(TabArgs a) {
    constexpr int R = r_for(NW);
    constexpr int YC = R * kThreads;
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    __shared__ __align__(16) uint32_t xs[kTX * XS];
    __shared__ TileInfo ti;
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long seen = ~0ull; // lane 0's view of the global best key
    unsigned long long done_local = 0;
    uint32_t cutoff = a.cutoff, stop_at = a.stop_at;
    // First tile: static (blockIdx.x; the launch clamps the grid to the tile count), and
    // its operands come from immutable tables only, so under PDL this prologue overlaps
    // the previous round. Later tiles: dynamic scheduler (atomic counter).
    if (threadIdx.x < 32) decode_tile_warp<YC>(a, a.tile_lo + blockIdx.x, ti);
    __syncthreads();
    if (threadIdx.x < ti.nx) build_smem_item<NW, HID>(a, ti, threadIdx.x, xs + threadIdx.x * XS, true);
    uint32_t Y[R][NW], idY[R];
    bool valid[R];
    load_suffixes<NW, HID>(a, ti, Y, idY, valid);
    bool skip = false;
    if (a.st) { // chained round: the loop state decides (same values in every block)
        griddep_wait();
        const ChainState cs = *a.st;
        skip = cs.done || cs.U <= cs.L;
        cutoff = cs.exact ? 0u : cs.U;
        stop_at = cs.L;
    }
    griddep_launch_dependents();
    const bool dynamic = a.tile_lo + gridDim.x < a.tile_hi;
    uint32_t gw = 0xFFFFFFFFu; // thread 0: the global best weight at the last tile fetch

    for (bool first = true; !skip; first = false) {
        if (!first) {
            if (!dynamic) break;
            if (threadIdx.x < 32) {
                uint32_t stop = 0;
                uint64_t t = 0;
                if (lane == 0) {
                    // the next tile (dynamic scheduler: uniform tiles, no static tail) and the
                    // global best, fetched together; early exit once the best meets stop_at
                    // -- a tile claimed then is simply not evaluated
                    t = a.tile_lo + gridDim.x + atomicAdd(a.counter, 1ull);
                    unsigned long long g = *reinterpret_cast<volatile unsigned long long*>(a.best_key);
                    if (a.shared_key) {
                        const unsigned long long sg = *reinterpret_cast<volatile unsigned long long*>(a.shared_key);
                        g = sg < g ? sg : g;
                    }
                    gw = uint32_t(g >> kKeyShift);
                    stop = gw <= stop_at || t >= a.tile_hi;
                }
                stop = __shfl_sync(0xFFFFFFFFu, stop, 0);
                t = __shfl_sync(0xFFFFFFFFu, t, 0);
                if (!stop) decode_tile_warp<YC>(a, t, ti);
                if (lane == 0) ti.stop = stop;
            }
            __syncthreads();
            if (ti.stop) break;
            if (threadIdx.x < ti.nx) build_smem_item<NW, HID>(a, ti, threadIdx.x, xs + threadIdx.x * XS, true);
            load_suffixes<NW, HID>(a, ti, Y, idY, valid);
        }
        if (threadIdx.x == 0) {
            done_local += uint64_t(ti.nx) * ti.nyv;
            // weights that still matter: <= min(cutoff - 1, best found so far)
            int64_t lim = cutoff ? int64_t(cutoff) - 1 : int64_t(0x7FFFFFFF);
            if (int64_t(gw) < lim) lim = gw;
            lim -= a.add_const;
            ti.T = lim < -1 ? -1 : (lim > 0x7FFFFFFF ? 0x7FFFFFFF : int32_t(lim));
            ti.G = pick_fold(ti.T, a.fold);
        }
        __syncthreads();
        const uint64_t tile = ti.tile;

        const uint32_t bc = a.rd ? tile_min_walk<NW, HID>(xs, ti.nx, Y, idY, ti.T, ti.G)
                                 : tile_min<NW, HID>(xs, 0, ti.nx, Y, idY, ti.T, ti.G);
        const unsigned long long key =
            warp_round_key<NW, HID>(bc, xs, Y, idY, ti.nyv, a.add_const, cutoff, a.pos_key, tile);
        if (lane == 0 && key != ~0ull) {
            if (key < seen) {
                unsigned long long old = atomicMin(a.best_key, key);
                if (a.shared_key) {
                    const unsigned long long so = atomicMin_system(a.shared_key, key);
                    old = so < old ? so : old;
                }
                seen = old < key ? old : key;
            }
        }
        __syncthreads(); // xs / ti reused by the next tile
    }
    if (threadIdx.x == 0) {
        if (done_local) atomicAdd(a.evaluated, done_local);
        if (a.fin_rec) { // fused finalize: the last block to finish closes the round
            __threadfence();
            if (atomicAdd(a.blocks_done, 1ull) == gridDim.x - 1) {
                __threadfence();
                finalize_round(a.fin_st, a.best_key, a.fin_rec, a.fin_c, a.fin_j, a.fin_last, a.fin_lb);
            }
        }
    }
}

// ------------------------------------------------------- fused level
// All m rounds of one level in one launch (chained loop, single rank, Gammas of one row
// width): the tile space is the m rounds' tiles back to back (round-major), one shared
// dynamic scheduler, one finalize (the last block closes the rounds in order, exactly as
// run_bz_loop would). Round j prunes with min(U, best of rounds i < j) - 1 and its own best:
// every round i < j has true minimum >= its best, so round j's result is exact whenever it
// lies below U_before_j = min(U, w_0 .. w_{j-1}), and >= U_before_j otherwise -- the
// sequential finalize then reproduces each bounded w_j and the (L, U) trace bit for bit.
// A tile is skipped once some round i <= j has a best <= L (the reference would stop there:
// that round's minimum is exactly L and the rounds after it hit the fast path).
constexpr int kMaxFuse = 16;
struct LevelRound {
    const uint32_t* rows;
    const uint32_t* ytab;
    const uint32_t* xtab;
    unsigned long long* slot; // {best key, evaluated, -, -, -}
    ChainRec* rec;
    FoldPlan fold;
    uint32_t id_rows, add_const;
};
struct LevelDesc {
    uint32_t m;
    uint64_t T; // tiles per round (one plan for all rounds)
    LevelRound r[kMaxFuse];
};

template <int NW, bool HID>
__global__ void __launch_bounds__(kThreads, NW <= 2 ? MDG_MINBLK_SMALL : 4)
tab_level(TabArgs a, const __grid_constant__ LevelDesc L) {
    constexpr int R = r_for(NW);
    constexpr int YC = R * kThreads;
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    __shared__ __align__(16) uint32_t xs[kTX * XS];
    __shared__ TileInfo ti;
    __shared__ TabArgs sa; // a with the current tile's round fields
    __shared__ uint32_t cur_j, skip_tile;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t total = uint64_t(L.m) * L.T;
    auto set_round = [&](uint32_t j) { // thread 0
        const LevelRound& r = L.r[j];
        sa.rows = r.rows;
        sa.ytab = r.ytab;
        sa.xtab = r.xtab;
        sa.id_rows = r.id_rows;
        sa.add_const = r.add_const;
        sa.fold = r.fold;
        cur_j = j;
    };
    if (threadIdx.x == 0) {
        sa = a;
        set_round(uint32_t(uint64_t(blockIdx.x) / L.T));
    }
    __syncthreads();
    if (threadIdx.x < 32) decode_tile_warp<YC>(sa, uint64_t(blockIdx.x) % L.T, ti);
    __syncthreads();
    if (threadIdx.x < ti.nx) build_smem_item<NW, HID>(sa, ti, threadIdx.x, xs + threadIdx.x * XS, true);
    uint32_t Y[R][NW], idY[R];
    bool valid[R];
    load_suffixes<NW, HID>(sa, ti, Y, idY, valid);
    griddep_wait();
    const ChainState cs = *a.st;
    const bool skip = cs.done || cs.U <= cs.L;
    const uint32_t cutoff = cs.exact ? 0u : cs.U, stop_at = cs.L;
    const bool exact = cs.exact != 0;
    griddep_launch_dependents();
    const bool dynamic = uint64_t(gridDim.x) < total;

    for (bool first = true; !skip; first = false) {
        if (!first) {
            if (!dynamic) break;
            if (threadIdx.x < 32) {
                uint32_t stop = 0;
                uint64_t t = 0;
                if (lane == 0) {
                    t = gridDim.x + atomicAdd(a.counter, 1ull);
                    stop = t >= total;
                    if (!stop && uint32_t(t / L.T) != cur_j) set_round(uint32_t(t / L.T));
                }
                stop = __shfl_sync(0xFFFFFFFFu, stop, 0);
                t = __shfl_sync(0xFFFFFFFFu, t, 0);
                __syncwarp();
                if (!stop) decode_tile_warp<YC>(sa, t % L.T, ti);
                if (lane == 0) ti.stop = stop;
            }
            __syncthreads();
            if (ti.stop) break;
        }
        if (threadIdx.x == 0) {
            // bests of rounds 0..j: own best (ties still evaluated) and, bounded, the earlier
            // rounds' (strictly below them); skip once any is <= L
            const uint32_t j = cur_j;
            uint32_t own = uint32_t(*reinterpret_cast<volatile unsigned long long*>(L.r[j].slot) >> kKeyShift);
            uint32_t prev = 0xFFFFFFFFu, lowest = own;
            for (uint32_t i = 0; i < j; ++i) {
                const uint32_t b = uint32_t(*reinterpret_cast<volatile unsigned long long*>(L.r[i].slot) >> kKeyShift);
                prev = min(prev, b);
            }
            lowest = min(lowest, prev);
            skip_tile = lowest <= stop_at;
            int64_t lim = cutoff ? int64_t(cutoff) - 1 : int64_t(0x7FFFFFFF);
            if (int64_t(own) < lim) lim = own;
            if (!exact && prev != 0xFFFFFFFFu && int64_t(prev) - 1 < lim) lim = int64_t(prev) - 1;
            lim -= sa.add_const;
            ti.T = lim < -1 ? -1 : (lim > 0x7FFFFFFF ? 0x7FFFFFFF : int32_t(lim));
            ti.G = pick_fold(ti.T, sa.fold);
            if (!skip_tile) atomicAdd(L.r[j].slot + 1, uint64_t(ti.nx) * ti.nyv);
        }
        __syncthreads();
        if (!skip_tile) {
            if (!first) {
                if (threadIdx.x < ti.nx) build_smem_item<NW, HID>(sa, ti, threadIdx.x, xs + threadIdx.x * XS, true);
                load_suffixes<NW, HID>(sa, ti, Y, idY, valid);
                __syncthreads();
            }
            const uint64_t tile = ti.tile;
            const uint32_t add = sa.add_const;
            unsigned long long* best_key = L.r[cur_j].slot;
            const uint32_t bc = a.rd ? tile_min_walk<NW, HID>(xs, ti.nx, Y, idY, ti.T, ti.G)
                                     : tile_min<NW, HID>(xs, 0, ti.nx, Y, idY, ti.T, ti.G);
            const unsigned long long key =
                warp_round_key<NW, HID>(bc, xs, Y, idY, ti.nyv, add, cutoff, a.pos_key, tile);
            if (lane == 0 && key != ~0ull) atomicMin(best_key, key);
        }
        __syncthreads(); // xs / ti / sa reused by the next tile
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.blocks_done, 1ull) == gridDim.x - 1) {
            __threadfence();
            for (uint32_t j = 0; j < L.m; ++j)
                finalize_round(a.fin_st, L.r[j].slot, L.r[j].rec, a.fin_c, j, j + 1 == L.m ? 1u : 0u,
                               a.fin_lb);
        }
    }
}

// One thread: close a chained round (engines.cpp:456-472 semantics).
__global__ void chain_finalize(ChainState* st, const unsigned long long* slot, ChainRec* rec,
                               uint32_t c, uint32_t j, uint32_t last_of_level, uint32_t lb) {
    if (threadIdx.x == 0) finalize_round(st, slot, rec, c, j, last_of_level, lb);
}

// witness: the smallest (x_local, y_local) of the tile whose weight == target
template <int NW, bool HID>
__global__ void __launch_bounds__(kThreads) tab_find(TabArgs a) {
    // block b scans smem-side items [b * kFindX, (b + 1) * kFindX) of the tile (one block
    // per slice: the whole tile in a few microseconds instead of one block's serial scan)
    constexpr int R = r_for(NW);
    constexpr int YC = R * kThreads;
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    __shared__ __align__(16) uint32_t xs[kFindX * XS];
    __shared__ TileInfo ti;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) decode_tile<YC>(a, a.tile_lo, ti);
    __syncthreads();
    const uint32_t xb = blockIdx.x * kFindX;
    if (xb >= ti.nx) return;
    const uint32_t xe = min(ti.nx, xb + kFindX);
    if (threadIdx.x < xe - xb) build_smem_item<NW, HID>(a, ti, xb + threadIdx.x, xs + threadIdx.x * XS);
    uint32_t Y[R][NW], idY[R];
    bool valid[R];
    load_suffixes<NW, HID>(a, ti, Y, idY, valid);
    __syncthreads();
    unsigned long long cand = ~0ull;
    for (uint32_t xi = xb; xi < xe; ++xi) {
        uint32_t X[XS];
        vload<XS>(xs + (xi - xb) * XS, X);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t w = xor_weight<0, NW, XS, NW>(X, Y[r]);
            if (HID) w += X[NW] + idY[r];
            w += a.add_const;
            uint32_t yl = r * kThreads + warp * 32 + lane;
            if (valid[r] && w == a.find_target) {
                unsigned long long c = (static_cast<unsigned long long>(xi) << 32) | yl;
                cand = c < cand ? c : cand;
            }
        }
    }
    if (cand != ~0ull) atomicMin(a.find_out, cand);
}

// full weight histogram (config 5): per-warp privatized u32 bins in smem. The lanes past
// the tile's edge count into a per-warp scratch copy of the bins (no divergent branch and no
// select per codeword); the bin address is a 32-bit shared-window offset accumulated by IMADs
// from the popcounts (popsum_mad: the FMA pipe is idle, the ALU pipe carries the LOP3s); the
// smem bins are flushed into the u64 global histogram before any could wrap (a block counts
// at most 2^32 - 1 codewords between flushes).
//
// Chain basis. popsum's carry-save chain folds words (ones, v[2i+1], v[2i+2]) into a new ones
// word S_{i+1} = v[0] ^ ... ^ v[2i+2] and a carry. XOR is linear, so when both sides of the tile
// store S_{i+1} in place of word 2i+2 (to_chain_basis, once per item per tile), X' ^ Y' yields
// the chain's ones words directly and each carry is ONE LOP3 of (ones before, v[2i+1], ones
// after): maj(a, b, t ^ a ^ b), LUT 0xD4 -- one LOP3 per chain step instead of two (NW = 8:
// 13 LOP3 per codeword instead of 16, 27 instead of 30 instructions).
#ifndef MDG_HIST_CHAIN
#define MDG_HIST_CHAIN 1
#endif
template <int N>
__device__ __forceinline__ void to_chain_basis(uint32_t* v) {
#pragma unroll
    for (int i = 0; i < (N - 1) / 2; ++i) v[2 + 2 * i] ^= v[2 * i] ^ v[1 + 2 * i];
}
template <int N>
__device__ __forceinline__ uint32_t popsum_chain_mad(const uint32_t (&v)[N], uint32_t acc, const uint32_t* s) {
    if constexpr (N < 3) {
        return popsum_mad<N>(v, acc, s);
    } else {
        constexpr int M = (N - 1) / 2;
        uint32_t carries[M];
#pragma unroll
        for (int i = 0; i < M; ++i) carries[i] = lop3<0xD4>(v[2 * i], v[1 + 2 * i], v[2 + 2 * i]);
        acc = mad_u32(__popc(v[2 * M]), s[0], acc);
        if constexpr ((N - 1) % 2 == 1) acc = mad_u32(__popc(v[N - 1]), s[0], acc);
        return popsum_mad<M>(carries, acc, s + 1);
    }
}

template <int NW, bool HID>
#ifdef MDG_HIST_MINBLK // tuning builds only: a minimum of resident blocks (5 / 6 measured slower)
__global__ void __launch_bounds__(kThreads, MDG_HIST_MINBLK) tab_hist(TabArgs a) {
#else
__global__ void __launch_bounds__(kThreads) tab_hist(TabArgs a) {
#endif
    constexpr int R = r_for(NW);
    constexpr int YC = R * kThreads;
    constexpr int XS = stride_for(NW + (HID ? 1 : 0));
    extern __shared__ __align__(16) uint32_t dyn[];
    uint32_t* xs = dyn;
    const uint32_t bs = a.nbins;      // per-warp bins, then a per-warp scratch copy
    uint32_t* bins = dyn + a.tx * XS; // kWarps x 2 x bs
    __shared__ TileInfo ti;
    __shared__ uint32_t flush_now;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = threadIdx.x; i < kWarps * 2 * bs; i += kThreads) bins[i] = 0;
    const uint32_t sreal = uint32_t(__cvta_generic_to_shared(bins + warp * 2 * bs));
    const uint32_t sjunk = sreal + 4u * bs;
    uint32_t sc[6] = {4u, 8u, 16u, 32u, 64u, 128u}; // popsum_mad multipliers (bytes per bin << i)
    asm volatile("" : "+r"(sc[0]), "+r"(sc[1]), "+r"(sc[2]), "+r"(sc[3]), "+r"(sc[4]), "+r"(sc[5]));
    unsigned long long done_local = 0, since_flush = 0; // thread 0
    auto flush = [&]() { // all threads; real bins -> global, zeroed
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < bs; b += kThreads) {
            unsigned long long sum = 0;
            for (int w = 0; w < kWarps; ++w) {
                sum += bins[w * 2 * bs + b];
                bins[w * 2 * bs + b] = 0;
            }
            if (sum) atomicAdd(a.hist + b, sum);
        }
        __syncthreads();
    };
    for (;;) {
        if (threadIdx.x < 32) {
            uint32_t stop = 0;
            uint64_t t = 0;
            if (lane == 0) {
                t = a.tile_lo + atomicAdd(a.counter, 1ull);
                stop = t >= a.tile_hi;
            }
            stop = __shfl_sync(0xFFFFFFFFu, stop, 0);
            t = __shfl_sync(0xFFFFFFFFu, t, 0);
            if (!stop) decode_tile_warp<YC>(a, t, ti);
            if (lane == 0) {
                ti.stop = stop;
                flush_now = 0;
                if (!stop) {
                    const uint64_t cw = uint64_t(ti.nx) * ti.nyv;
                    done_local += cw;
                    if (since_flush + cw > 0xFFFFFFFFull) {
                        flush_now = 1;
                        since_flush = 0;
                    }
                    since_flush += cw;
                }
            }
        }
        __syncthreads();
        if (ti.stop) break;
        if (flush_now) flush();
        if (threadIdx.x < ti.nx) {
            build_smem_item<NW, HID>(a, ti, threadIdx.x, xs + threadIdx.x * XS);
            if (MDG_HIST_CHAIN) to_chain_basis<NW>(xs + threadIdx.x * XS);
        }
        uint32_t Y[R][NW], idY[R];
        bool valid[R];
        load_suffixes<NW, HID>(a, ti, Y, idY, valid);
        if (MDG_HIST_CHAIN) {
#pragma unroll
            for (int r = 0; r < R; ++r) to_chain_basis<NW>(Y[r]);
        }
        uint32_t base[R]; // the item's bin row: real bins + weight offset, or the scratch copy
#pragma unroll
        for (int r = 0; r < R; ++r) base[r] = (valid[r] ? sreal : sjunk) + 4u * (a.add_const + (HID ? idY[r] : 0u));
        __syncthreads();
        const uint32_t nx = ti.nx;
        for (uint32_t xi = 0; xi < nx; ++xi) {
            uint32_t X[XS];
            vload<XS>(xs + xi * XS, X);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                uint32_t v[NW];
#pragma unroll
                for (int w = 0; w < NW; ++w) v[w] = X[w] ^ Y[r][w];
                const uint32_t b0 = HID ? mad_u32(X[NW], sc[0], base[r]) : base[r];
                asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(
                    MDG_HIST_CHAIN ? popsum_chain_mad<NW>(v, b0, sc) : popsum_mad<NW>(v, b0, sc)));
            }
        }
        __syncthreads();
    }
    flush();
    if (threadIdx.x == 0 && done_local) atomicAdd(a.evaluated, done_local);
}



// ------------------------------------------------------------ brute force
// All 2^k - 1 nonzero codewords of a k-row basis (the reference's
// brute_force_gray, engines.cpp:480-558, restated as a product of two spans):
// rows split into A = [0, a) and B = [a, k); TA[i] = XOR of the A rows at the
// set bits of gray(i) (2^a entries, binary reflected Gray order,
// enumeration.hpp:19), TB likewise over B; codeword (x, y) = TA[x] ^ TB[y],
// the pair (0, 0) excluded. Tiles are TX x-entries (smem) x YC y-entries
// (registers), bound-pruned by the running minimum.
template <int NW>
__global__ void span_build(const uint32_t* __restrict__ rows, uint32_t first, uint64_t count,
                           uint32_t* __restrict__ out) {
    constexpr int S = stride_for(NW);
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint64_t g = i ^ (i >> 1);
    uint32_t acc[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) acc[w] = 0;
    while (g) {
        uint32_t b = uint32_t(__ffsll(static_cast<long long>(g)) - 1);
        g &= g - 1;
        xor_row<NW>(rows, first + b, acc);
    }
#pragma unroll
    for (int w = 0; w < S; ++w) out[i * S + w] = w < NW ? acc[w] : 0u;
}

struct SpanArgs {
    int32_t fold_lim[4];           // G = 1, 2, 4; [3]: pair bound over words 0-1 (NW 2..4)
    const uint32_t* ta;
    const uint32_t* tb;
    uint64_t na, nb, nty;
    uint32_t tx;
    uint64_t tile_lo, tile_hi;
    unsigned long long* best_key;
    unsigned long long* evaluated;
    unsigned long long* counter;
    unsigned long long* find_out;
    uint32_t find_target;
};


template <int NW, bool FIND>
__global__ void __launch_bounds__(kThreads, 4) span_round(SpanArgs a) {
    constexpr int R = r_for(NW);
    constexpr int YC = R * kThreads;
    constexpr int S = stride_for(NW);
    __shared__ __align__(16) uint32_t xs[kTX * S];
    __shared__ uint64_t s_x0, s_y0, s_tile;
    __shared__ uint32_t s_nx, s_nyv, s_stop;
    __shared__ int32_t s_T;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long seen = ~0ull, done_local = 0;
    for (uint32_t it = 0;; ++it) {
        if (threadIdx.x == 0) {
            uint64_t t;
            if (FIND) {
                t = a.tile_lo;
                s_stop = it > 0;
            } else {
                t = a.tile_lo + atomicAdd(a.counter, 1ull);
                s_stop = t >= a.tile_hi;
            }
            if (!s_stop) {
                uint64_t xt = t / a.nty, yt = t - xt * a.nty;
                s_tile = t;
                s_x0 = xt * a.tx;
                s_nx = uint32_t(umin64(a.tx, a.na - s_x0));
                s_y0 = yt * YC;
                s_nyv = uint32_t(umin64(uint64_t(YC), a.nb - s_y0));
                unsigned long long g = *reinterpret_cast<volatile unsigned long long*>(a.best_key);
                uint32_t gw = uint32_t(g >> kKeyShift);
                s_T = gw >= 0x7FFFFFFFu ? 0x7FFFFFFF : int32_t(gw);
                done_local += uint64_t(s_nx) * s_nyv;
            }
        }
        __syncthreads();
        if (s_stop) break;
        const uint32_t nx = s_nx, nyv = s_nyv;
        const uint64_t x0 = s_x0, y0 = s_y0;
        if (threadIdx.x < nx) {
            uint32_t v[S];
            vload_global<S>(a.ta + (x0 + threadIdx.x) * S, v);
#pragma unroll
            for (int w = 0; w < S; ++w) xs[threadIdx.x * S + w] = v[w];
        }
        uint32_t Y[R][NW], idY[R];
        bool valid[R];
        uint64_t yi[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t yl = r * kThreads + warp * 32 + lane;
            valid[r] = yl < nyv;
            yi[r] = y0 + (valid[r] ? yl : 0u);
            uint32_t v[S];
            vload_global<S>(a.tb + yi[r] * S, v);
#pragma unroll
            for (int w = 0; w < NW; ++w) Y[r][w] = v[w];
            idY[r] = 0;
        }
        __syncthreads();
        if (FIND) {
            unsigned long long cand = ~0ull;
            for (uint32_t xi = 0; xi < nx; ++xi) {
                uint32_t X[S];
                vload<S>(xs + xi * S, X);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    uint32_t w = xor_weight<0, NW, S, NW>(X, Y[r]);
                    bool zero_pair = x0 + xi == 0 && yi[r] == 0;
                    if (valid[r] && !zero_pair && w == a.find_target) {
                        unsigned long long c = (static_cast<unsigned long long>(xi) << 32) |
                                               (r * kThreads + warp * 32 + lane);
                        cand = c < cand ? c : cand;
                    }
                }
            }
            if (cand != ~0ull) atomicMin(a.find_out, cand);
        } else {
            uint32_t best = 0xFFFFFFFFu;
            uint32_t xb = 0;
            if (x0 == 0) { // row x = 0 is the zero vector: codewords from B alone, minus (0,0)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    uint32_t w = 0;
#pragma unroll
                    for (int i = 0; i < NW; ++i) w += __popc(Y[r][i]);
                    if (yi[r] != 0) best = min(best, w);
                }
                xb = 1;
            }
            // the bound must be warp-uniform: tile_min branches on it around warp votes
            const uint32_t wbest = __reduce_min_sync(0xFFFFFFFFu, best);
            const int32_t T = wbest == 0xFFFFFFFFu ? s_T : min(s_T, int32_t(wbest));
            best = min(best, best_weight(tile_min<NW, false>(xs, xb, nx, Y, idY, T, pick_groups(T, a.fold_lim))));
            best = __reduce_min_sync(0xFFFFFFFFu, best);
            if (lane == 0 && best != 0xFFFFFFFFu) {
                unsigned long long key = (static_cast<unsigned long long>(best) << kKeyShift) | s_tile;
                if (key < seen) {
                    unsigned long long old = atomicMin(a.best_key, key);
                    seen = old < key ? old : key;
                }
            }
        }
        __syncthreads();
    }
    if (!FIND && threadIdx.x == 0 && done_local) atomicAdd(a.evaluated, done_local);
}

template <int NW, bool HID>
struct SpanLaunch { // HID unused: dispatch shape only
    static void run(const uint32_t* rows, uint32_t a_rows, uint32_t b_rows, uint32_t* ta, uint32_t* tb,
                    SpanArgs sa, int mode, cudaStream_t st, int sms) {
        if (mode == 0) {
            uint64_t na = uint64_t(1) << a_rows, nb = uint64_t(1) << b_rows;
            span_build<NW><<<uint32_t((na + 255) / 256), 256, 0, st>>>(rows, 0, na, ta);
            span_build<NW><<<uint32_t((nb + 255) / 256), 256, 0, st>>>(rows, a_rows, nb, tb);
        } else if (mode == 1) {
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, span_round<NW, false>, kThreads, 0);
            if (occ < 1) occ = 1;
            uint64_t tiles = sa.tile_hi - sa.tile_lo;
            uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>(tiles, uint64_t(sms) * occ));
            span_round<NW, false><<<uint32_t(g), kThreads, 0, st>>>(sa);
        } else {
            span_round<NW, true><<<1, kThreads, 0, st>>>(sa);
        }
    }
};

// ------------------------------------------------------------ dispatch
template <template <int, bool> class F, typename... Args>
void dispatch_nw_hid(uint32_t nw, bool hid, Args&&... args) {
#define MDG_CASE(N)                                                              \
    case N:                                                                      \
        if (hid) F<N, true>::run(args...); else F<N, false>::run(args...);       \
        break;
    switch (nw) {
#ifdef MDG_DEV_FEW_WIDTHS // tuning builds only (tools/build_variant.sh): compiles in a minute
        MDG_CASE(2) MDG_CASE(4) MDG_CASE(7) MDG_CASE(8)
#else
        MDG_CASE(1) MDG_CASE(2) MDG_CASE(3) MDG_CASE(4) MDG_CASE(5) MDG_CASE(6) MDG_CASE(7)
        MDG_CASE(8) MDG_CASE(10) MDG_CASE(12) MDG_CASE(14) MDG_CASE(16) MDG_CASE(20)
        MDG_CASE(24) MDG_CASE(28) MDG_CASE(32)
#endif
        default: throw std::invalid_argument("row width beyond the device limit");
    }
#undef MDG_CASE
}

template <int NW, bool HID>
struct YtabLaunch {
    static void run(const uint32_t* rows, const uint64_t* T, uint32_t k, uint32_t s,
                    uint32_t id_rows, uint64_t count, uint32_t* out, bool reverse, cudaStream_t st) {
        uint64_t blocks = (count + 255) / 256;
        ytab_build<NW, HID><<<dim3(uint32_t(blocks)), 256, 0, st>>>(rows, T, k, s, id_rows, count, out,
                                                                   reverse);
    }
};

template <int NW, bool HID>
struct TablesLaunch {
    static void run(const TableJobs& J, const uint64_t* T, cudaStream_t st) {
        uint64_t blocks = (J.total + 256 * kTabRun - 1) / (256 * kTabRun);
        tables_build<NW, HID><<<dim3(uint32_t(blocks)), 256, 0, st>>>(J, T);
    }
};

template <int NW, bool HID>
struct LevelLaunch {
    static void run(const TabArgs& a, const LevelDesc& L, uint64_t total, bool pdl, cudaStream_t st,
                    int sms) {
        // per instantiation (the kernel's resources never change); several host threads
        // (the batch front door) may race to fill it: atomic, and every writer stores the same value
        static std::atomic<int> cached{-1};
        int occ = cached.load(std::memory_order_relaxed);
        if (occ < 0) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tab_level<NW, HID>, kThreads, 0);
            cached.store(occ, std::memory_order_relaxed);
        }
        const uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>(total, uint64_t(sms) * std::max(occ, 1)));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(uint32_t(g));
        cfg.blockDim = dim3(kThreads);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, tab_level<NW, HID>, a, L);
    }
};

template <int NW, bool HID>
struct TabOcc {
    static void run(int* occ) {
        static std::atomic<int> cached{-1}; // per instantiation, as LevelLaunch
        int o = cached.load(std::memory_order_relaxed);
        if (o < 0) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tab_round<NW, HID>, kThreads, 0);
            cached.store(o, std::memory_order_relaxed);
        }
        *occ = o;
    }
};

template <int NW, bool HID>
struct HistOcc { // resident tab_hist blocks per SM at `dyn` bytes of dynamic smem
    static void run(size_t dyn, int* occ) {
        auto fn = tab_hist<NW, HID>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, kThreads, dyn);
    }
};

template <int NW, bool HID>
struct TabLaunch {
    // grid: number of tiles for mode 0/2 (clamped to the resident-block count)
    static void run(const TabArgs& a, uint64_t grid, cudaStream_t st, int mode, size_t dyn, int sms) {
        if (mode == 0 || mode == 3) { // 3: programmatic dependent launch after a chained round
            int occ = 0;
            TabOcc<NW, HID>::run(&occ);
            if (occ < 1) occ = 1;
            uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>(grid, uint64_t(sms) * occ));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(uint32_t(g));
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = 0;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = mode == 3 ? 1 : 0;
            cudaLaunchKernelEx(&cfg, tab_round<NW, HID>, a);
        }
        else if (mode == 1) tab_find<NW, HID><<<(kTX + kFindX - 1) / kFindX, kThreads, 0, st>>>(a);
        else {
            auto fn = tab_hist<NW, HID>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, dyn);
            if (occ < 1) occ = 1;
            uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>(grid, uint64_t(sms) * occ));
            fn<<<uint32_t(g), kThreads, dyn, st>>>(a);
        }
    }
};

__global__ void init_slots(unsigned long long* s, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        s[8 * i + 0] = ~0ull; // best key
        s[8 * i + 1] = 0;     // evaluated
        s[8 * i + 2] = 0;     // tile counter
        s[8 * i + 3] = ~0ull; // witness search result
        s[8 * i + 4] = 0;     // blocks done (fused finalize)
        s[8 * i + 5] = s[8 * i + 6] = s[8 * i + 7] = 0;
    }
}

} // namespace

// ================================================================ host side
uint32_t template_width(uint32_t nw32) {
    if (nw32 <= 8) return std::max<uint32_t>(nw32, 1);
    if (nw32 <= 16) return (nw32 + 1) & ~1u;
    if (nw32 <= 32) return (nw32 + 3) & ~3u;
    throw std::invalid_argument("row width exceeds the device limit (n - rank <= 1024)");
}


uint32_t tab_yc(uint32_t nw32) { return uint32_t(r_for(int(nw32))) * kThreads; }
uint32_t tab_tx() { return kTX; }

static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// RoundResult::plan_tag: bit 0 valid, bit 1 pruning on, bit 2 revolving-door plan, bits 4..8 the
// number of rounds m of the fused level the round ran in (0: a launch of its own) -- a fused
// level plans its tiles for 1/m of the resident blocks per round
static uint32_t plan_tag(bool rd, bool prune, uint32_t fused_m = 0) {
    return 1u | (prune ? 2u : 0u) | (rd ? 4u : 0u) | ((fused_m & 31u) << 4);
}

// saturating Pascal table C(x, t), x <= kMaxK, t <= kMaxC (host and device copies)
static const std::vector<uint64_t>& binom_table() {
    static const std::vector<uint64_t> T = [] {
        std::vector<uint64_t> t(size_t(kMaxK + 1) * kBT, 0);
        for (uint32_t x = 0; x <= kMaxK; ++x) {
            t[size_t(x) * kBT] = 1;
            for (uint32_t q = 1; q <= kMaxC && q <= x; ++q) {
                uint64_t a = t[size_t(x - 1) * kBT + q - 1], b = t[size_t(x - 1) * kBT + q];
                uint64_t sum = a + b;
                t[size_t(x) * kBT + q] = (sum < a || a == ~0ull || b == ~0ull) ? ~0ull : sum;
            }
        }
        return t;
    }();
    return T;
}

static inline uint64_t hb(uint32_t x, uint32_t t) {
    if (t > x) return 0;
    if (x <= kMaxK && t <= kMaxC) return binom_table()[size_t(x) * kBT + t];
    return binomial(x, t);
}

// the prefix table ((p-1)-subset sums) exists when it is non-empty and <= 4M entries
static bool xtab_ok(uint32_t k, uint32_t pm1) { return pm1 >= 1 && hb(k, pm1) <= (uint64_t{1} << 22); }

// MDG_TRANSPOSE=0 disables transposed tiles (A/B switch)
static bool transpose_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MDG_TRANSPOSE");
        return e ? std::atoi(e) != 0 : true;
    }();
    return on;
}

// Orientation of pivot e's tiles: transposed (suffixes in smem, prefixes in registers)
// when that masks fewer register lanes; needs the prefix table.
static bool pivot_transposed(uint64_t NX, uint64_t NY, uint32_t YC, bool can) {
    if (!can) return false;
    const uint64_t waste_n = NX * (ceil_div(NY, YC) * YC - NY);
    const uint64_t waste_t = NY * (ceil_div(NX, YC) * YC - NX);
    return waste_t < waste_n;
}

// per-tile overhead of the cost model, in prefix rows (MDG_TILE_OVERHEAD)
static uint64_t tile_overhead() {
    static const uint64_t v = [] {
        const char* e = std::getenv("MDG_TILE_OVERHEAD");
        return e ? uint64_t(std::max(0, std::atoi(e))) : uint64_t(4);
    }();
    return v;
}

// total cost in codeword-slots: masked register lanes + a per-tile overhead
static uint64_t plan_cost(uint32_t k, uint32_t c, uint32_t s, uint32_t TX, uint32_t YC,
                          uint64_t* tiles_out, bool allow_tr = true) {
    uint32_t p = c - s;
    const bool can = allow_tr && transpose_enabled() && xtab_ok(k, p - 1);
    uint64_t cost = 0, tiles = 0;
    for (uint32_t e = p - 1; e + s <= k - 1; ++e) {
        uint64_t NX = hb(e, p - 1), NY = hb(k - 1 - e, s);
        if (pivot_transposed(NX, NY, YC, can)) std::swap(NX, NY);
        uint64_t ntx = ceil_div(NX, TX), nty = ceil_div(NY, YC);
        tiles += ntx * nty;
        cost += NX * nty * YC + ntx * nty * uint64_t(YC) * tile_overhead();
    }
    if (tiles_out) *tiles_out = tiles;
    return cost;
}

// Suffix size s minimizes the tile cost (suffix table <= 4M entries); the
// prefix chunk TX is the largest of 256/128/64/32/16 that still yields >= 8
// tiles per resident block, so the dynamic scheduler's tail stays short.
TabPlan make_tab_plan(uint32_t k, uint32_t c, uint32_t nw32, uint32_t resident_blocks, bool rd,
                      uint32_t tiles_per_block) {
    TabPlan pl;
    pl.k = k;
    pl.c = c;
    pl.rd = rd; // revolving-door prefix walk: the prefixes stay on the smem side (no transposition)
    pl.YC = tab_yc(nw32);
    uint32_t best_s = 0;
    if (c >= 2) {
        uint64_t best_cost = ~uint64_t{0};
        for (uint32_t s = 1; s <= c - 1; ++s) {
            if (hb(k, s) > (uint64_t{1} << 22) && s > 1) break;
            uint64_t cost = plan_cost(k, c, s, kTX, pl.YC, nullptr, !rd);
            if (cost < best_cost) { best_cost = cost; best_s = s; }
        }
    }
    if (const char* e = std::getenv("MDG_FORCE_S")) { // development: fixed suffix size
        const int fs = std::atoi(e);
        if (fs >= 1 && uint32_t(fs) < c) best_s = uint32_t(fs);
    }
    pl.s = best_s;
    pl.p = c - best_s;
    pl.emin = pl.p - 1;
    pl.emax = k - 1 - pl.s;
    // tuning knobs (defaults measured on B200): tiles per resident block, smallest chunk
    static const uint32_t kTilesPerBlock = [] {
        const char* e = std::getenv("MDG_TILES_PER_BLOCK");
        return e ? uint32_t(std::max(1, std::atoi(e))) : 2u;
    }();
    static const uint32_t kMinTX = [] {
        const char* e = std::getenv("MDG_MIN_TX");
        return e ? uint32_t(std::max(1, std::min(256, std::atoi(e)))) : 16u;
    }();
    pl.TX = kMinTX;
    for (uint32_t tx = kTX; tx >= kMinTX; tx /= 2) {
        uint64_t tiles = 0;
        plan_cost(k, c, pl.s, tx, pl.YC, &tiles, !rd);
        const uint32_t tpb = tiles_per_block ? tiles_per_block : kTilesPerBlock;
        if (tiles >= uint64_t(resident_blocks) * tpb || tx <= kMinTX) { pl.TX = tx; break; }
    }
    const bool can = !rd && transpose_enabled() && xtab_ok(k, pl.p - 1);
    pl.prefix.assign(1, 0);
    pl.tr.clear();
    for (uint32_t e = pl.emin; e <= pl.emax; ++e) {
        uint64_t NX = hb(e, pl.p - 1), NY = hb(k - 1 - e, pl.s);
        const bool tr = pivot_transposed(NX, NY, pl.YC, can);
        pl.tr.push_back(tr ? 1 : 0);
        if (tr) std::swap(NX, NY);
        pl.prefix.push_back(pl.prefix.back() + ceil_div(NX, pl.TX) * ceil_div(NY, pl.YC));
    }
    if (std::getenv("MDG_PLAN_DEBUG")) {
        size_t ntr = 0;
        for (uint8_t t : pl.tr) ntr += t;
        std::fprintf(stderr, "[mdg plan] k=%u c=%u nw=%u s=%u TX=%u YC=%u tiles=%llu transposed_pivots=%zu/%zu\n",
                     k, c, nw32, pl.s, pl.TX, pl.YC, (unsigned long long)pl.tiles(), ntr, pl.tr.size());
    }
    return pl;
}

// Codewords in tiles [0, t) of a plan: the tiles of pivot e cut its A x B grid (smem side x
// register side) into TX x YC blocks, row-major, the last row and column partial.
uint64_t tab_codewords_before(const TabPlan& pl, uint64_t t) {
    uint64_t cw = 0;
    const size_t npiv = pl.prefix.size() - 1;
    for (size_t i = 0; i < npiv && t > pl.prefix[i]; ++i) {
        const uint32_t e = pl.emin + uint32_t(i);
        const uint64_t NX = hb(e, pl.p - 1), NY = hb(pl.k - 1 - e, pl.s);
        const bool tr = i < pl.tr.size() && pl.tr[i];
        const uint64_t A = tr ? NY : NX, B = tr ? NX : NY;
        if (t >= pl.prefix[i + 1]) {
            cw += A * B;
            continue;
        }
        const uint64_t local = t - pl.prefix[i], ntb = ceil_div(B, pl.YC);
        const uint64_t ta = local / ntb, tb = local % ntb;
        cw += std::min<uint64_t>(ta * pl.TX, A) * B;
        cw += std::min<uint64_t>(pl.TX, A - ta * pl.TX) * std::min<uint64_t>(tb * pl.YC, B);
    }
    return cw;
}

// Rank r's contiguous tile range of a split round: boundaries at the tiles where the
// cumulative codeword count crosses r/world of the round (tiles are not equal-sized: the last
// pivots' tiles are partial), so every rank gets ~1/world of the codewords, not of the tiles.
// Deterministic: every rank computes the same boundaries from the same plan.
std::pair<uint64_t, uint64_t> tab_split(const TabPlan& pl, uint32_t rank, uint32_t world) {
    const uint64_t T = pl.tiles();
    if (world <= 1) return {0, T};
    const uint64_t total = tab_codewords_before(pl, T);
    auto bound = [&](uint32_t r) -> uint64_t {
        if (r == 0) return 0;
        if (r >= world) return T;
        const uint64_t target = uint64_t((unsigned __int128)total * r / world);
        uint64_t lo = 0, hi = T; // smallest t with codewords_before(t) >= target
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (tab_codewords_before(pl, mid) >= target) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    return {bound(rank), bound(rank + 1)};
}

// host colex unrank: t-subset of [0, hi) with colex rank r, ascending
static void colex_unrank_host(uint64_t r, uint32_t t, uint32_t hi, uint32_t* out) {
    for (uint32_t i = t; i >= 1; --i) {
        uint32_t x = hi - 1;
        while (hb(x, i) > r) --x;
        out[i - 1] = x;
        r -= hb(x, i);
        hi = x;
    }
}

void tab_decode(const TabPlan& pl, uint64_t tile, uint32_t x_local, uint32_t y_local, uint32_t* idx) {
    uint32_t i = uint32_t(std::upper_bound(pl.prefix.begin(), pl.prefix.end(), tile) - pl.prefix.begin()) - 1;
    uint32_t e = pl.emin + i;
    uint64_t local = tile - pl.prefix[i];
    const bool tr = !pl.tr.empty() && pl.tr[i];
    uint64_t B = tr ? hb(e, pl.p - 1) : hb(pl.k - 1 - e, pl.s); // register side
    uint64_t ntb = ceil_div(B, pl.YC);
    uint64_t ta = local / ntb, tb = local % ntb;
    uint64_t sm = ta * pl.TX + x_local, rg = tb * pl.YC + y_local; // smem / register index
    uint64_t x = tr ? rg : sm, y = tr ? sm : rg;                   // prefix / suffix index
    std::vector<uint32_t> out;
    std::vector<uint32_t> tmp(pl.c + 1);
    if (pl.p > 1 && pl.rd) rd_unrank(pl.p - 1, x, tmp.data()); // revolving-door prefix order
    else if (pl.p > 1) colex_unrank_host(x, pl.p - 1, e, tmp.data());
    for (uint32_t q = 0; q + 1 < pl.p; ++q) out.push_back(tmp[q]);
    out.push_back(e);
    if (pl.s) {
        colex_unrank_host(y, pl.s, pl.k, tmp.data());
        for (uint32_t q = 0; q < pl.s; ++q) out.push_back(pl.k - 1 - tmp[q]);
    }
    std::sort(out.begin(), out.end());
    std::copy(out.begin(), out.end(), idx);
}

// ------------------------------------------------------------ NCCL (dlopen)
namespace {
typedef struct { char internal[128]; } ncclUniqueId_t;
typedef void* ncclComm_t;
struct NcclApi {
    void* h = nullptr;
    int (*GetUniqueId)(ncclUniqueId_t*) = nullptr;
    int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId_t, int) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.h, "ncclCommInitRank"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.h, "ncclAllReduce"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    });
    if (!api.h || !api.AllReduce) throw std::runtime_error("NCCL (libnccl.so.2) not available");
    return api;
}
constexpr int kNcclUint64 = 5; // ncclUint64
constexpr int kNcclMin = 3;    // ncclMin
constexpr int kNcclSum = 0;    // ncclSum
} // namespace

// ------------------------------------------------------------ exchange group
// SURVEY.md §8e's per-round reduction without NCCL, for `world` engines in ONE process
// (one host thread each; on one device or on peer-accessible devices). Each split round:
// the member records an event after its round kernel and publishes (slot, event); a host
// barrier waits for all members; each member's stream then waits on the others' events
// and a one-thread kernel takes the min of all members' keys (group_min). No kernel waits
// on another kernel -- the dependency is stream-ordered. One barrier per round also orders
// event reuse: a member re-records its event only after every member passed the barrier
// of the next split round, i.e. after they enqueued their waits on the previous record.
// Members whose enqueue decisions diverge (a bug: the loop is deterministic) time out.
struct ExchangeGroup {
    explicit ExchangeGroup(uint32_t world, double timeout_s)
        : world(world), timeout_s(timeout_s), slots(world, nullptr), events(world, nullptr),
          tags(world, 0), loops(world, 0), left(world, 0) {}
    const uint32_t world;
    const double timeout_s; // <= 0: wait as long as the other members run (a split round may take hours)
    std::mutex mu;
    std::condition_variable cv;
    uint64_t generation = 0;
    uint32_t arrived = 0;
    bool aborted = false;
    std::string why;
    std::vector<unsigned long long*> slots;
    std::vector<cudaEvent_t> events;
    // what each barrier handed out, by generation parity: a member woken late from barrier g
    // must not read `slots` / `events` -- a fast member may already have published round g + 1
    // there. Barrier g + 1 needs the late member, so snapshot g stays valid until it has read it.
    std::vector<unsigned long long*> snap_slots[2];
    std::vector<cudaEvent_t> snap_events[2];
    std::vector<uint64_t> tags;  // (c << 32 | j) of the split round each member arrived with
    std::vector<uint64_t> loops; // level loops each member has entered
    std::vector<uint64_t> left;  // the last loop each member has left
    std::vector<int> devices;
    // shared round keys (tile results of every member, polled at every tile fetch): a ring on
    // rank 0's device, entry i % kRing for the i-th split round; rank 0 resets an entry after
    // the round's exchange (every member's round kernel is then done with it), and stream order
    // puts that reset before any member's round i + kRing (it follows rank 0's round-(i+1) event)
    static constexpr uint32_t kRing = 64;
    unsigned long long* ring = nullptr;
    int ring_device = -1;
    bool ring_ok = true; // false: some member pair has no native peer atomics (no shared key)
    ~ExchangeGroup() {
        if (ring) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(ring_device);
            cudaFree(ring);
            cudaSetDevice(cur);
        }
    }
    void fail(const std::string& reason) { // with mu held
        if (!aborted) why = reason;
        aborted = true;
        cv.notify_all();
    }
    // a member starts / ends a level loop: a member still waiting for the others at a split
    // round of loop L while one of them has left loop L has diverged (it enqueued a split round
    // the other never will) -- fail at once instead of waiting forever
    void enter(uint32_t rank) {
        std::lock_guard<std::mutex> lk(mu);
        ++loops[rank];
    }
    void leave(uint32_t rank) {
        std::lock_guard<std::mutex> lk(mu);
        left[rank] = loops[rank];
        cv.notify_all();
    }

    // publish (slot, ev) of `rank` for split round (c, j), wait for every member of this round;
    // copies out all. Members must arrive with the same (c, j): their enqueue sequences are
    // identical by construction, so a mismatch is a bug -- fail loudly.
    void exchange(uint32_t rank, uint32_t c, uint32_t j, unsigned long long* slot, cudaEvent_t ev,
                  std::vector<unsigned long long*>& all_slots, std::vector<cudaEvent_t>& all_events) {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) throw std::runtime_error("exchange group aborted: " + why);
        slots[rank] = slot;
        events[rank] = ev;
        tags[rank] = (uint64_t(c) << 32) | j;
        const uint64_t gen = generation, loop = loops[rank];
        auto departed = [&] {
            for (uint32_t r = 0; r < world; ++r)
                if (r != rank && left[r] == loop && loops[r] == loop) return true;
            return false;
        };
        if (++arrived == world) {
            arrived = 0;
            snap_slots[gen & 1] = slots;
            snap_events[gen & 1] = events;
            ++generation;
            for (uint32_t r = 0; r < world; ++r)
                if (tags[r] != tags[rank])
                    fail("members diverged: rank " + std::to_string(r) + " is at another split round");
            cv.notify_all();
        } else {
            auto ready = [&] { return generation != gen || aborted || departed(); };
            if (timeout_s > 0) {
                if (!cv.wait_for(lk, std::chrono::duration<double>(timeout_s), ready))
                    fail("member " + std::to_string(rank) + " timed out at a split round");
            } else {
                cv.wait(lk, ready);
            }
            if (generation == gen && !aborted)
                fail("members diverged: a member left the level loop while rank " + std::to_string(rank) +
                     " waits at a split round");
        }
        if (aborted) throw std::runtime_error("exchange group aborted: " + why);
        all_slots = snap_slots[gen & 1];
        all_events = snap_events[gen & 1];
    }
    void abort(const std::string& reason) {
        std::lock_guard<std::mutex> lk(mu);
        fail(reason);
    }
};

std::shared_ptr<ExchangeGroup> make_exchange_group(uint32_t world, double timeout_s) {
    if (world < 1 || world > uint32_t(kMaxGroup))
        throw std::invalid_argument("exchange group: 1 <= world <= 16");
    if (timeout_s < 0) { // default: MDG_GROUP_TIMEOUT seconds, else no timeout
        const char* e = std::getenv("MDG_GROUP_TIMEOUT");
        timeout_s = e ? std::atof(e) : 0.0;
    }
    return std::make_shared<ExchangeGroup>(world, timeout_s);
}
void abort_exchange_group(ExchangeGroup& g, const std::string& reason) { g.abort(reason); }

// ------------------------------------------------------------ Engine impl
// Bump allocator over large cudaMalloc'd chunks: Gamma rows and suffix tables
// are carved from it and released all at once by reset() on the next load, so
// the steady state makes no cudaMalloc / cudaFree calls (cudaFree synchronizes
// the device and costs far more than a small round).
class DevArena {
public:
    ~DevArena() {
        for (auto& c : chunks_) cudaFree(c.base);
    }
    void* alloc(size_t bytes) {
        bytes = (bytes + 255) & ~size_t(255);
        for (; cur_ < chunks_.size(); ++cur_) {
            Chunk& c = chunks_[cur_];
            if (c.used + bytes <= c.size) {
                void* p = static_cast<char*>(c.base) + c.used;
                c.used += bytes;
                return p;
            }
        }
        Chunk c;
        c.size = std::max<size_t>(bytes, size_t(64) << 20);
        CK(cudaMalloc(&c.base, c.size));
        c.used = bytes;
        chunks_.push_back(c);
        cur_ = chunks_.size() - 1;
        return c.base;
    }
    void reset() {
        for (auto& c : chunks_) c.used = 0;
        cur_ = 0;
    }

private:
    struct Chunk {
        void* base = nullptr;
        size_t size = 0, used = 0;
    };
    std::vector<Chunk> chunks_;
    size_t cur_ = 0;
};

// Stage-1 limits for G = 1, 2, 4 fold groups over the template's NW words: with
// codeword bit density rho_c, a fold bit over m words is set with probability
// 1 - (1 - rho_c)^m, so popc(folds) ~ mean E_G, variance V_G; pruning with G groups
// is worth it while the bound T <= E_G - 4 sqrt(V_G) (then almost no codeword passes).
// G must leave some group with two or more words (G=2 needs NW >= 3, G=4 needs NW >= 5).
static void fold_limits(uint32_t bits, uint32_t nw, double rho_c, int32_t (&lim)[4]) {
    const int Gs[3] = {1, 2, 4};
    for (int gi = 0; gi < 3; ++gi) {
        const int G = Gs[gi];
        if ((G == 2 && nw < 3) || (G == 4 && nw < 5)) { lim[gi] = -1; continue; }
        double mean = 0, var = 0;
        for (int g = 0; g < G; ++g) {
            const uint32_t b = uint32_t(g) * nw / G, e = uint32_t(g + 1) * nw / G;
            for (uint32_t p = 0; p < 32; ++p) {
                uint32_t m = 0;
                for (uint32_t w = b; w < e; ++w)
                    if (w * 32 + p < bits) ++m;
                const double q = 1.0 - std::pow(1.0 - rho_c, double(m));
                mean += q;
                var += q * (1.0 - q);
            }
        }
        lim[gi] = int32_t(std::floor(mean - 4.0 * std::sqrt(var)));
    }
    // a larger G only helps if it raises the limit
    if (lim[1] <= lim[0]) lim[1] = -1;
    if (lim[2] <= std::max(lim[0], lim[1])) lim[2] = -1;
    // pair pre-filter over words 0-1 (tile_min's pair variant; NW 2..4): a bit of the AND of
    // two codewords' folds is set w.p. q^2; used while T is 3.5 sd below its mean (a vote
    // that falls through takes the single folds, then exact weights)
    lim[3] = -1;
    if (nw >= 2 && nw <= 4) {
        double mean = 0, var = 0;
        for (uint32_t p = 0; p < 32; ++p) {
            const uint32_t m = (p < bits ? 1u : 0u) + (32 + p < bits ? 1u : 0u);
            const double q = 1.0 - std::pow(1.0 - rho_c, double(m)), q2 = q * q;
            mean += q2;
            var += q2 * (1.0 - q2);
        }
        lim[3] = int32_t(std::floor(mean - 3.5 * std::sqrt(var)));
    }
}

// density of an XOR of c rows of density rho (independent bits)
static double level_density(double rho, uint32_t c) {
    return 0.5 * (1.0 - std::pow(1.0 - 2.0 * rho, double(c)));
}

struct GammaDev {
    double rho = 0.5;          // bit density of the compacted rows
    std::vector<uint32_t> host_rows; // compacted rows on the host (stage-1 sampling)
    uint32_t* rows = nullptr;  // k x nw (compacted, zero-padded to the template width)
    uint32_t nw = 0;
    uint32_t id_rows = 0;      // identity rows [0, id_rows)
    uint32_t n_compact = 0;
    bool hid = false;          // partial identity block: per-entry identity counts
};

struct PlanEntry {
    TabPlan plan;
    uint64_t* d_prefix = nullptr;
    uint8_t* d_tr = nullptr; // per-pivot orientation (null: all normal)
};

// per-round scratch slots {best key, evaluated, counter, find, blocks done}: a ring of kSlots
// (MDG_SLOTS shrinks it so tests wrap it often), re-initialized by one kernel per wrap
constexpr int kSlots = 4096;
static int ring_slots() {
    static const int n = [] {
        const char* e = std::getenv("MDG_SLOTS");
        return e ? std::max(2 * (kMaxFuse + 2), std::min(kSlots, std::atoi(e))) : kSlots;
    }();
    return n;
}

struct Engine::Impl {
    cudaStream_t stream = nullptr;
    void* stage = nullptr;     // pinned host staging for uploads (grows)
    size_t stage_cap = 0;
    uint32_t* staging(size_t bytes) {
        if (stage_cap < bytes) {
            if (stage) cudaFreeHost(stage);
            stage = nullptr;
            CK(cudaHostAlloc(&stage, bytes, cudaHostAllocDefault));
            stage_cap = bytes;
        }
        return static_cast<uint32_t*>(stage);
    }
    bool rd = false;           // revolving-door prefix walk (Kernel::rd) instead of prefix sums
    void* scratch = nullptr;   // Engine::scratch (GPU permutation search)
    size_t scratch_cap = 0;
    bool prune = true; // stage-1 bound pruning (mdg_set_pruning)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, tev0 = nullptr, tev1 = nullptr;
    Engine::Counters cnt;
    uint64_t* binom = nullptr;
    unsigned long long* slots = nullptr;
    unsigned long long* host_slot = nullptr; // pinned, 4 words
    int nslots = ring_slots();
    int next_slot = kSlots;                  // >= nslots: forces an init on first use
    uint32_t chain_runs = 0;                 // chain_loop calls so far (ChainState::run)
    // Cross-process shared bound (one process per GPU): a ring of round-key words in rank 0's
    // device memory, mapped into the other ranks through a CUDA IPC handle. Entry i % kXRing
    // serves the i-th split round; the owner resets it after that round's reduction.
    static constexpr uint32_t kXRing = 64;
    unsigned long long* xring = nullptr;
    bool xowner = false;
    uint64_t xround = 0; // split rounds so far (the same on every rank)
    unsigned long long* xword() const {
        static const bool off = std::getenv("MDG_NO_SHARED_BOUND") != nullptr;
        return (xring && !off) ? xring + xround % kXRing : nullptr;
    }
    void xadvance() { // after a split round's reduction (every rank has finished the round)
        if (!xring) return;
        if (xowner) CK(cudaMemsetAsync(xring + xround % kXRing, 0xFF, sizeof(unsigned long long), stream));
        ++xround;
    }
    unsigned long long* hist_dev = nullptr;
    size_t hist_cap = 0;
    std::vector<GammaDev> gammas;
    std::map<std::tuple<uint32_t, uint32_t, bool>, uint32_t*> tables; // (j, size, reverse) -> table
    std::map<std::tuple<uint32_t, uint32_t, uint32_t, bool, bool, bool, uint32_t>, PlanEntry> plans; // (k, c, nw, hid, rd, prune, tiles per block)
    std::map<std::pair<uint32_t, bool>, int> occ;                     // (nw, hid)
    std::map<std::pair<uint32_t, uint32_t>, FoldPlan> fold_cache; // (j, c)
    ncclComm_t comm = nullptr;
    std::shared_ptr<ExchangeGroup> group; // in-process exchange (group_attach)
    uint32_t group_rank = 0;
    uint64_t group_round = 0;              // split rounds exchanged so far (same on every member)
    cudaEvent_t group_ev = nullptr;
    uint64_t* red_dev = nullptr;
    size_t red_cap = 0;
    DevArena arena;                  // Gamma rows + suffix tables (reset per load)
    DevArena plan_arena;             // plan prefix arrays (kept: plans are cached)
    ChainState* d_state = nullptr;
    ChainState* h_state = nullptr;   // pinned
    uint32_t* h_progress = nullptr;  // pinned + mapped: {levels closed, done} written by finalize_round
    ChainRec* d_recs = nullptr;
    size_t recs_cap = 0;
    std::vector<cudaEvent_t> evpool;
    cudaEvent_t event(size_t i) {
        while (evpool.size() <= i) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            evpool.push_back(e);
        }
        return evpool[i];
    }

    // The ring is re-initialized (in stream order) when it wraps, so a slot must be USED by a
    // launch enqueued before the next re-initialization: a launch that needs several slots
    // reserves them first, so the wrap cannot fall between its take_slot calls. (Taken one by
    // one, a fused level's first slots could predate the re-initialization that its launch
    // then followed: they were written after it and stayed dirty for the ring's next cycle --
    // a stale lighter key then won that later round's atomicMin.)
    void reserve_slots(int n) {
        if (next_slot + n > nslots) {
            init_slots<<<(nslots + 255) / 256, 256, 0, stream>>>(slots, nslots);
            CK(cudaGetLastError());
            cnt.launches += 1;
            next_slot = 0;
        }
    }
    unsigned long long* take_slot() {
        reserve_slots(1);
        return slots + 8 * size_t(next_slot++);
    }
    void read_slot(unsigned long long* slot) {
        CK(cudaMemcpyAsync(host_slot, slot, 32, cudaMemcpyDeviceToHost, stream));
        cnt.d2h += 32;
    }
    int resident(uint32_t nw, bool hid, int sms) {
        auto key = std::make_pair(nw, hid);
        auto it = occ.find(key);
        if (it != occ.end()) return it->second * sms;
        int o = 0;
        dispatch_nw_hid<TabOcc>(nw, hid, &o);
        if (o < 1) o = 1;
        occ[key] = o;
        return o * sms;
    }
    const PlanEntry& plan(uint32_t k, uint32_t c, const GammaDev& g, int sms) {
        return plan(k, c, g, sms, rd, prune);
    }
    // the tile plan of an explicit variant (a round's witness is decoded with the plan it ran on)
    // fused_m > 1: the plan of one round of a fused level of m rounds. The level's tile space is
    // its m rounds' tiles back to back, so each round needs only 1/m of the tiles that keep the
    // resident blocks busy: larger tiles, fewer tile prologues (config 3, eight Gammas of 32 rows:
    // TX 16 -> 128 at level 9)
    const PlanEntry& plan(uint32_t k, uint32_t c, const GammaDev& g, int sms, bool rd, bool prune,
                          uint32_t tpb = 0, int resident_override = 0, uint32_t fused_m = 0) {
        if (fused_m < 2) fused_m = 0;
        auto key = std::make_tuple(k, c, g.nw, g.hid, rd, prune, tpb | (fused_m << 24));
        auto it = plans.find(key);
        if (it != plans.end()) return it->second;
        PlanEntry pe;
        int res = resident_override ? resident_override : resident(g.nw, g.hid, sms);
        if (fused_m) {
            // tiles per resident block over the whole level (the plan aims for 2 per round): 2 for
            // two or three rounds, 4 from four rounds on -- measured (profiles/r02j_fused_tiles.txt):
            // the eight-code config-2 step (m = 2) 2.02 -> 1.99 ms at 2 (2.02 at 4), config 3
            // (m = 8, exact weights, tiles of very different lengths) 0.65 -> 0.62 ms at 4 (0.74 at 2)
            static const int kFusedTiles = [] {
                const char* e = std::getenv("MDG_FUSED_TILES");
                return e ? std::max(1, std::atoi(e)) : 0;
            }();
            const int tiles = kFusedTiles ? kFusedTiles : (fused_m >= 4 ? 4 : 2);
            res = std::max(1, res * tiles / (2 * int(fused_m)));
        }
        pe.plan = make_tab_plan(k, c, g.nw, uint32_t(res), rd, tpb ? tpb : (prune ? 0u : 8u));
        const size_t pb = pe.plan.prefix.size() * 8, tb = pe.plan.tr.size();
        pe.d_prefix = static_cast<uint64_t*>(plan_arena.alloc(pb + tb));
        CK(cudaMemcpyAsync(pe.d_prefix, pe.plan.prefix.data(), pb, cudaMemcpyHostToDevice, stream));
        bool any_tr = false;
        for (uint8_t t : pe.plan.tr) any_tr = any_tr || t;
        if (any_tr) {
            pe.d_tr = reinterpret_cast<uint8_t*>(pe.d_prefix) + pb;
            CK(cudaMemcpyAsync(pe.d_tr, pe.plan.tr.data(), tb, cudaMemcpyHostToDevice, stream));
        }
        CK(cudaStreamSynchronize(stream));
        cnt.h2d += pb + (any_tr ? tb : 0);
        return plans.emplace(key, pe).first->second;
    }
};

Engine::Engine(int device) : device_(device), impl_(new Impl) {
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw std::invalid_argument("mdg: no such CUDA device");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    sms_ = prop.multiProcessorCount;
    plan_sms_ = sms_;
    if (const char* e = std::getenv("MDG_PDL")) pdl_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MDG_FUSE_MAX")) fuse_max_ = std::atof(e);
    CK(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&impl_->ev0));
    CK(cudaEventCreate(&impl_->ev1));
    CK(cudaEventCreate(&impl_->tev0));
    CK(cudaEventCreate(&impl_->tev1));
    const auto& T = binom_table();
    CK(cudaMalloc(&impl_->binom, T.size() * 8));
    CK(cudaMemcpy(impl_->binom, T.data(), T.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&impl_->slots, size_t(kSlots) * 64));
    CK(cudaHostAlloc(&impl_->host_slot, 32, cudaHostAllocDefault));
    CK(cudaMalloc(&impl_->d_state, sizeof(ChainState)));
    CK(cudaHostAlloc(&impl_->h_state, sizeof(ChainState), cudaHostAllocDefault));
    CK(cudaHostAlloc(&impl_->h_progress, 64, cudaHostAllocMapped));
}

Engine::~Engine() {
    if (!impl_) return;
    cudaSetDevice(device_);
    if (impl_->stream) cudaStreamSynchronize(impl_->stream);
    if (impl_->comm) {
        try { nccl().CommDestroy(impl_->comm); } catch (...) {}
    }
    if (impl_->group_ev) cudaEventDestroy(impl_->group_ev);
    if (impl_->xring) {
        if (impl_->xowner) cudaFree(impl_->xring); else cudaIpcCloseMemHandle(impl_->xring);
    }
    cudaFree(impl_->red_dev);
    cudaFree(impl_->scratch);
    cudaFree(impl_->d_state);
    cudaFree(impl_->d_recs);
    cudaFreeHost(impl_->h_state);
    cudaFreeHost(impl_->h_progress);
    if (impl_->stage) cudaFreeHost(impl_->stage);
    for (auto e : impl_->evpool) cudaEventDestroy(e);
    cudaFree(impl_->hist_dev);
    cudaFree(impl_->binom);
    cudaFree(impl_->slots);
    cudaFreeHost(impl_->host_slot);
    cudaEventDestroy(impl_->ev0);
    cudaEventDestroy(impl_->ev1);
    cudaEventDestroy(impl_->tev0);
    cudaEventDestroy(impl_->tev1);
    cudaStreamDestroy(impl_->stream);
}

void Engine::load(uint32_t m, uint32_t k, uint32_t n, const uint64_t* rows, const uint32_t* ranks) {
    if (m < 1 || k < 1 || n < 1) throw std::invalid_argument("mdg_load: empty matrix set");
    if (k > kMaxK) throw std::invalid_argument("mdg_load: k exceeds the device limit of 1024 rows");
    CK(cudaSetDevice(device_));
    CK(cudaStreamSynchronize(impl_->stream));
    const uint32_t W = (n + 63) / 64;
    std::vector<GammaDev> next;
    std::vector<std::vector<uint32_t>> host(m);
    for (uint32_t j = 0; j < m; ++j) {
        const uint64_t* G = rows + size_t(j) * k * W;
        uint32_t rk = ranks ? ranks[j] : 0;
        uint32_t off = j * k;
        if (ranks) {
            if (rk > k || off + rk > n) throw std::invalid_argument("mdg_load: rank out of range");
            // the identity block the kernels elide must really be there (gamma.cpp:44-71)
            for (uint32_t r = 0; r < k; ++r)
                for (uint32_t t = 0; t < rk; ++t) {
                    uint32_t col = off + t;
                    bool bit = (G[size_t(r) * W + col / 64] >> (col % 64)) & 1u;
                    if (bit != (r == t))
                        throw std::invalid_argument("mdg_load: Gamma " + std::to_string(j) +
                                                    " lacks its identity block");
                }
        }
        // A partial Gamma's rows [rk, k) usually still own a unit column of the previous
        // block's identity (the last block's row operations add pivot rows, whose earlier
        // identity bits are the pivots' own: gamma.cpp:57-62), so every row owns exactly one
        // weight-1 column. Then |S| counts all of them and the Gamma is compacted like a
        // full-rank one (no per-entry identity counts; config 4's Gamma_1: 7 words + counts
        // -> 4 words). Otherwise only the identity block is elided (per-entry counts, HID).
        std::vector<uint32_t> extra; // unit column owned by row rk + i
        if (ranks && rk > 0 && rk < k && !getenv("MDG_NO_UNIT_ELISION")) {
            std::vector<int32_t> owner(n, -1); // row of a weight-1 column, -2 heavier, -1 empty
            for (uint32_t r = 0; r < k; ++r) {
                const uint64_t* row = G + size_t(r) * W;
                for (uint32_t col = 0; col < n; ++col)
                    if ((row[col / 64] >> (col % 64)) & 1u) owner[col] = owner[col] == -1 ? int32_t(r) : -2;
            }
            extra.assign(k - rk, UINT32_MAX);
            for (uint32_t col = 0; col < n; ++col) {
                if (col >= off && col < off + rk) continue;
                const int32_t r = owner[col];
                if (r >= int32_t(rk) && extra[r - rk] == UINT32_MAX) extra[r - rk] = col;
            }
            for (uint32_t x : extra)
                if (x == UINT32_MAX) { extra.clear(); break; }
        }
        const bool all_unit = !extra.empty();
        std::vector<uint8_t> elide(n, 0);
        if (ranks)
            for (uint32_t t = 0; t < rk; ++t) elide[off + t] = 1;
        for (uint32_t col : extra) elide[col] = 1;
        GammaDev gd;
        gd.id_rows = all_unit ? k : rk;
        gd.n_compact = n - rk - uint32_t(extra.size());
        gd.nw = template_width(std::max<uint32_t>(1, (gd.n_compact + 31) / 32)); // zero-padded
        gd.hid = rk > 0 && rk < k && !all_unit;
        auto& hr = host[j];
        hr.assign(size_t(k) * gd.nw, 0);
        if (all_unit) { // compacted row = the non-elided columns in order (bit by bit: k x n)
            for (uint32_t r = 0; r < k; ++r) {
                const uint64_t* row = G + size_t(r) * W;
                uint32_t* dst = hr.data() + size_t(r) * gd.nw;
                for (uint32_t col = 0, p = 0; col < n; ++col) {
                    if (elide[col]) continue;
                    if ((row[col / 64] >> (col % 64)) & 1u) dst[p / 32] |= 1u << (p % 32);
                    ++p;
                }
            }
        }
        // compacted row = bits [0, off) then bits [off + rk, n): two word-level bit-range copies
        auto get64 = [&](const uint64_t* row, uint32_t pos) -> uint64_t { // 64 bits from pos (0-padded)
            const uint32_t w = pos / 64, sh = pos % 64;
            uint64_t v = w < W ? row[w] >> sh : 0;
            if (sh && w + 1 < W) v |= row[w + 1] << (64 - sh);
            return v;
        };
        const uint32_t cut = ranks ? rk : 0, head = ranks ? off : n;
        for (uint32_t r = 0; r < k && !all_unit; ++r) {
            const uint64_t* row = G + size_t(r) * W;
            uint32_t* dst = hr.data() + size_t(r) * gd.nw;
            auto put = [&](uint32_t from, uint32_t len, uint32_t to) { // bits [from, from+len) -> to
                for (uint32_t done = 0; done < len;) {
                    const uint32_t take = std::min<uint32_t>(32, len - done);
                    uint32_t v = uint32_t(get64(row, from + done));
                    if (take < 32) v &= (1u << take) - 1u;
                    const uint32_t p = to + done, w = p / 32, sh = p % 32;
                    dst[w] |= v << sh;
                    if (sh && sh + take > 32) dst[w + 1] |= v >> (32 - sh);
                    done += take;
                }
            };
            put(0, std::min(head, n), 0);
            if (ranks && off + cut < n) put(off + cut, n - off - cut, off);
        }
        uint64_t ones = 0;
        for (uint32_t x : hr) ones += uint32_t(__builtin_popcount(x));
        gd.rho = gd.n_compact ? double(ones) / (double(k) * gd.n_compact) : 0.5;
        gd.host_rows = hr;
        next.push_back(gd);
    }
    impl_->gammas.clear();
    impl_->tables.clear();
    impl_->fold_cache.clear();
    impl_->arena.reset(); // the stream is idle (synchronized above)
    // all Gammas in one device block, one copy from a pinned staging buffer
    size_t total = 0;
    for (uint32_t j = 0; j < m; ++j) total += (host[j].size() + 63) / 64 * 64; // 256-B aligned
    uint32_t* block = static_cast<uint32_t*>(impl_->arena.alloc(total * 4));
    uint32_t* stage = impl_->staging(total * 4);
    size_t o = 0;
    for (uint32_t j = 0; j < m; ++j) {
        std::memcpy(stage + o, host[j].data(), host[j].size() * 4);
        next[j].rows = block + o;
        o += (host[j].size() + 63) / 64 * 64;
    }
    CK(cudaMemcpyAsync(block, stage, total * 4, cudaMemcpyHostToDevice, impl_->stream));
    impl_->cnt.h2d += total * 4;
    CK(cudaStreamSynchronize(impl_->stream));
    impl_->gammas = std::move(next);
    m_ = m;
    k_ = k;
    n_ = n;
}

void Engine::check_round(uint32_t j, uint32_t c) const {
    if (j >= m_) throw std::invalid_argument("round: gamma index out of range");
    if (c < 1 || c > k_) throw std::invalid_argument("round: need 1 <= g <= k");
    if (c > kMaxC) throw std::invalid_argument("round: level beyond the device limit of 64");
    binomial(k_, c); // throws std::overflow_error when C(k, c) exceeds 64 bits
}

static uint32_t* ensure_table(Engine::Impl& im, uint32_t j, uint32_t k, uint32_t s, bool reverse) {
    auto key = std::make_tuple(j, s, reverse);
    auto it = im.tables.find(key);
    if (it != im.tables.end()) return it->second;
    const GammaDev& g = im.gammas[j];
    uint32_t YS = uint32_t(stride_for(int(g.nw) + (g.hid ? 1 : 0)));
    uint64_t count = hb(k, s);
    uint32_t* t = static_cast<uint32_t*>(im.arena.alloc(size_t(count) * YS * 4));
    dispatch_nw_hid<YtabLaunch>(g.nw, g.hid, g.rows, im.binom, k, s, g.id_rows, count, t, reverse,
                                im.stream);
    CK(cudaGetLastError());
    im.cnt.launches += 1;
    im.tables[key] = t;
    return t;
}

// Build, in as few launches as possible, every suffix / prefix table the rounds of
// levels [c_lo, c_hi] will ask for (ensure_ytab / ensure_xtab then find them cached).
struct TableNeed { uint32_t j, s; bool reverse; };

static std::vector<TableNeed> table_needs(Engine::Impl& im, uint32_t m, uint32_t k, uint32_t c_lo,
                                          uint32_t c_hi, int sms) {
    std::vector<TableNeed> need;
    auto want = [&](uint32_t j, uint32_t s, bool rev) {
        if (s == 0 || im.tables.count(std::make_tuple(j, s, rev))) return;
        for (const TableNeed& q : need)
            if (q.j == j && q.s == s && q.reverse == rev) return;
        need.push_back({j, s, rev});
    };
    for (uint32_t c = c_lo; c <= c_hi; ++c)
        for (uint32_t j = 0; j < m; ++j) {
            const PlanEntry& pe = im.plan(k, c, im.gammas[j], sms);
            want(j, pe.plan.s, true);
            if (!pe.plan.rd && xtab_ok(k, pe.plan.p - 1)) want(j, pe.plan.p - 1, false);
        }
    return need;
}

static uint64_t table_bytes(const Engine::Impl& im, uint32_t k, const std::vector<TableNeed>& need) {
    uint64_t b = 0;
    for (const TableNeed& q : need) {
        const GammaDev& g = im.gammas[q.j];
        b += hb(k, q.s) * uint64_t(stride_for(int(g.nw) + (g.hid ? 1 : 0))) * 4;
    }
    return b;
}

static void prebuild_tables(Engine::Impl& im, uint32_t m, uint32_t k, uint32_t c_lo, uint32_t c_hi,
                            int sms) {
    const std::vector<TableNeed> need = table_needs(im, m, k, c_lo, c_hi, sms);
    // one launch per (row width, identity flag) group, <= kMaxTableJobs tables each
    std::vector<bool> done(need.size(), false);
    for (size_t a = 0; a < need.size(); ++a) {
        if (done[a]) continue;
        const GammaDev& ga = im.gammas[need[a].j];
        TableJobs J{};
        J.k = k;
        for (size_t b = a; b < need.size() && J.n < uint32_t(kMaxTableJobs); ++b) {
            const GammaDev& g = im.gammas[need[b].j];
            if (done[b] || g.nw != ga.nw || g.hid != ga.hid) continue;
            const uint32_t YS = uint32_t(stride_for(int(g.nw) + (g.hid ? 1 : 0)));
            const uint64_t count = hb(k, need[b].s);
            uint32_t* t = static_cast<uint32_t*>(im.arena.alloc(size_t(count) * YS * 4));
            im.tables[std::make_tuple(need[b].j, need[b].s, need[b].reverse)] = t;
            TableJob& jo = J.job[J.n++];
            jo.rows = g.rows;
            jo.out = t;
            jo.begin = J.total;
            jo.s = need[b].s;
            jo.id_rows = g.id_rows;
            jo.reverse = need[b].reverse ? 1u : 0u;
            J.total += count;
            done[b] = true;
        }
        dispatch_nw_hid<TablesLaunch>(ga.nw, ga.hid, J, im.binom, im.stream);
        CK(cudaGetLastError());
        im.cnt.launches += 1;
    }
}

// suffix table (reverse colex s-subsets)
static uint32_t* ensure_ytab(Engine::Impl& im, uint32_t j, uint32_t k, uint32_t s) {
    return ensure_table(im, j, k, s, true);
}

// prefix table (colex (p-1)-subsets) when it is small enough, else nullptr (unrank per tile)
static const uint32_t* ensure_xtab(Engine::Impl& im, uint32_t j, uint32_t k, uint32_t pm1) {
    if (pm1 == 0 || hb(k, pm1) > (uint64_t{1} << 22)) return nullptr;
    return ensure_table(im, j, k, pm1, false);
}


// sd inflation of the normal tail used for overdispersed stage-1 bounds
#ifndef MDG_SD_SCALE
#define MDG_SD_SCALE 1.15
#endif
constexpr double kSdScale = MDG_SD_SCALE;

// Stage-1 choice per tile bound T, from the round's own codewords: 128 uniform random
// c-subsets of Gamma_j's compacted rows (SplitMix64 seeded by (j, c)) give mean and sd of
// each option's lower bound lb_G (sum of popc over G fold groups + identity count) and of
// its pair bound (the AND of two codewords' folds, the second sharing half the rows as
// two codewords of a tile share the prefix). Per T the option with the smallest expected
// pipe time per codeword wins (see the cost model below); exact weights when none beats
// them. Sampling captures the column structure a density model misses (the partial
// Gamma's rows are e_r plus subsets of the pivot columns: dense in half the columns).
static FoldPlan compute_fold_plan(const Engine::Impl& im, uint32_t j, uint32_t k, uint32_t c);

static FoldPlan sampled_fold_plan(Engine::Impl& im, uint32_t j, uint32_t k, uint32_t c) {
    auto key = std::make_pair(j, c);
    auto it = im.fold_cache.find(key);
    if (it != im.fold_cache.end()) return it->second;
    FoldPlan fp = compute_fold_plan(im, j, k, c);
    im.fold_cache[key] = fp;
    return fp;
}

// the fold plans of all Gammas of levels [c, c_hi] not yet cached, sampled in parallel on
// the host pool (one job)
static void prefetch_fold_plans(Engine::Impl& im, uint32_t m, uint32_t k, uint32_t c, uint32_t c_hi) {
    std::vector<std::pair<uint32_t, uint32_t>> todo;
    for (uint32_t g = c; g <= std::min(c_hi, std::min(k, uint32_t(kMaxC))); ++g)
        for (uint32_t j = 0; j < m; ++j)
            if (!im.fold_cache.count(std::make_pair(j, g))) todo.push_back({j, g});
    if (todo.size() < 2) return;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<FoldPlan> out(todo.size());
    parallel_for(uint32_t(todo.size()),
                 [&](uint32_t i) { out[i] = compute_fold_plan(im, todo[i].first, k, todo[i].second); });
    for (size_t i = 0; i < todo.size(); ++i) im.fold_cache[todo[i]] = out[i];
    if (std::getenv("MDG_PLAN_DEBUG"))
        std::fprintf(stderr, "[mdg fold] %zu plans (levels %u..%u) in %.1f us\n", todo.size(), c, c_hi,
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
}

// POPCs of popsum<n> (Harley-Seal chain)
static int popsum_popcs(int n) {
    if (n <= 2) return n < 0 ? 0 : n;
    const int m = (n - 1) / 2;
    return 1 + ((n - 1) % 2) + popsum_popcs(m);
}

static FoldPlan compute_fold_plan(const Engine::Impl& im, uint32_t j, uint32_t k, uint32_t c) {
    FoldPlan fp;
    std::memset(fp.code, 0, sizeof fp.code);
    const GammaDev& g = im.gammas[j];
    if (const char* f = std::getenv("MDG_FORCE_FOLD")) { // tests / A-B: one code for every T
        std::memset(fp.code, std::atoi(f), sizeof fp.code);
        return fp;
    }
    if (hb(k, c) < (uint64_t{1} << 20)) return fp; // a small round: exact weights cost nothing
    const uint32_t nw = g.nw;
    const int R = r_for(int(nw));
    const int GP = std::min(R, 8); // register items per pair-filter vote (MDG_PAIR_VOTE_GROUP)
    static const bool no_pair = std::getenv("MDG_NO_PAIR") != nullptr; // A/B switch
    // fold widths: all words, all but the last, the first half (the kernel's variants)
    struct Opt { uint32_t fw; int G; int code; double sum = 0, sq = 0, psum = 0, psq = 0; };
    std::vector<Opt> opts;
    const uint32_t widths[3] = {nw, nw >= 2 ? nw - 1 : 0, nw >= 3 ? (nw + 1) / 2 : 0};
    const int flags[3] = {0, kFoldDrop, kFoldHalf};
    for (int v = 0; v < 3; ++v) {
        const uint32_t fw = widths[v];
        if (fw == 0 || (v == 2 && fw >= widths[1])) continue;
        for (int G : {1, 2, 4})
            if ((G == 1) || (G == 2 && fw >= 3) || (G == 4 && fw >= 5)) opts.push_back({fw, G, G | flags[v]});
    }
    if (nw >= 7) opts.push_back({3, 1, 1 | kFold3}); // one group over the first three words
    constexpr int kSamples = 128;
    SplitMix64 rng(0x9E3779B97F4A7C15ull ^ (uint64_t(j) << 32) ^ c);
    std::vector<uint32_t> acc(nw), acc2(nw), pick;
    std::vector<uint8_t> used(k);
    auto draw = [&](uint32_t keep, std::vector<uint32_t>& out) -> uint32_t { // c distinct rows
        for (uint32_t i = 0; i < keep; ++i) used[pick[i]] = 1;
        pick.resize(keep);
        while (pick.size() < c) {
            uint32_t r;
            do { r = uint32_t(((rng.next() >> 32) * k) >> 32); } while (used[r]); // no division
            used[r] = 1;
            pick.push_back(r);
        }
        std::fill(out.begin(), out.end(), 0u);
        uint32_t id = 0;
        for (uint32_t r : pick) {
            used[r] = 0;
            id += r < g.id_rows;
            for (uint32_t w = 0; w < nw; ++w) out[w] ^= g.host_rows[size_t(r) * nw + w];
        }
        return id;
    };
    const auto tp0 = std::chrono::steady_clock::now();
    const bool pairs = R >= 2 && !no_pair && std::any_of(opts.begin(), opts.end(), [](const Opt& o) {
        return o.G == 1 && o.fw == 2; // pair2_bits: one two-word fold group
    });
    for (int t = 0; t < kSamples; ++t) {
        pick.clear();
        const uint32_t id = draw(0, acc);
        // a second codeword of the tile for the pair bound: shares rows, as two codewords of a
        // tile share the prefix
        const uint32_t id2 = pairs ? draw(c / 2, acc2) : id;
        for (Opt& o : opts) {
            uint32_t lb = g.hid ? id : 0, lp = g.hid ? std::min(id, id2) : 0;
            for (int q = 0; q < o.G; ++q) {
                uint32_t f = 0, f2 = 0;
                for (uint32_t w = uint32_t(q) * o.fw / o.G; w < uint32_t(q + 1) * o.fw / o.G; ++w)
                    f |= acc[w], f2 |= acc2[w];
                lb += uint32_t(__builtin_popcount(f));
                if (pairs) lp += uint32_t(__builtin_popcount(f & f2));
            }
            o.sum += lb;
            o.sq += double(lb) * lb;
            o.psum += lp;
            o.psq += double(lp) * lp;
        }
    }
    // Expected pipe time per codeword in ALU-op units, max(ALU ops, 4 x POPCs) (the XU pipe
    // issues POPC at a quarter of the LOP3 rate; the two pipes overlap). Exact weight: NW
    // XORs, the carry-save chain, one add per POPC, the min; stage 1: one LOP3 per folded
    // word, an IADD3 per two groups, ~1.4 ops of vote-group min / compare / vote / smem
    // load per item (~0.9 with pairs); a vote that falls through costs its items the next
    // stage. P(fall through) = 1 - (1 - p)^(bounds per vote), p = P(lb <= T).
    auto csa = [](auto&& self, int n) -> int { return n <= 2 ? 0 : (n - 1) / 2 + self(self, (n - 1) / 2); };
    const int pe = popsum_popcs(int(nw));
    const double exact = std::max(double(nw) + 2.0 * csa(csa, int(nw)) + pe + 2.0, 4.0 * pe);
    // P(lb <= T): lb is a popcount of nearly independent bits, so a binomial with the sampled
    // mean and variance (N = mean / q, q = 1 - var / mean) models its tail; overdispersed
    // samples (var >= mean: structured columns) fall back to an inflated normal tail
    // CDF of the bound at T = 0 .. kPlanT-1 in one pass (pmf recurrence, log domain)
    // (a partial Gamma's bound adds the identity count of the row set -- hypergeometric, not
    // a popcount -- so it takes the normal tail too)
    const bool normal = g.hid;
    auto tail = [normal](double mean, double var, std::array<double, kPlanT>& cdf) {
        const double q = var > 0 ? 1.0 - var / mean : 0.0;
        if (var <= 0) {
            for (int T = 0; T < kPlanT; ++T) cdf[T] = T >= mean ? 1.0 : 0.0;
        } else if (normal || !(q > 0.05)) {
            const double sd = kSdScale * std::sqrt(var);
            for (int T = 0; T < kPlanT; ++T) cdf[T] = 0.5 * std::erfc(-(T + 0.5 - mean) / (sd * std::sqrt(2.0)));
        } else {
            const int N = std::min(4094, std::max(1, int(std::lround(mean / q))));
            const double qq = std::min(1.0 - 1e-9, mean / N);
            static const std::vector<double> logi = [] { // log(i); N <= 4094 >= any bound
                std::vector<double> v(4096, 0.0);
                for (size_t i = 1; i < v.size(); ++i) v[i] = std::log(double(i));
                return v;
            }();
            // pmf(T+1) = pmf(T) (N - T) / (T + 1) * q / (1 - q): in logs while pmf is below
            // the double range, then by multiplication (one exp per option)
            double lp = N * std::log1p(-qq), acc = 0, pm = 0; // log pmf(0)
            const double odds = qq / (1.0 - qq), lodds = std::log(odds);
            int T = 0;
            for (; T < kPlanT && T <= N && acc < 1.0; ++T) {
                if (pm == 0 && lp > -700) pm = std::exp(lp);
                acc += pm;
                cdf[T] = std::min(1.0, acc);
                if (T < N) {
                    if (pm == 0) lp += logi[N - T] - logi[T + 1] + lodds;
                    else pm *= double(N - T) / double(T + 1) * odds;
                }
            }
            for (; T < kPlanT; ++T) cdf[T] = std::min(1.0, acc);
        }
    };
    // 1 - (1 - p)^bounds for bounds = 32 x a power of two (vote groups of 1..8 items), by
    // repeated squaring: the plan is on the host's critical path between levels
    auto fall = [](double p, int bounds) {
        double q = 1.0 - std::min(p, 1.0);
        for (int b = 1; b < bounds; b *= 2) q *= q;
        return 1.0 - q;
    };
    const int GR = std::min(R, 4);
    // A vote group that falls through costs far more than its exact weights' pipe time: the
    // branch, the dependent carry-save -> POPC -> add -> min chain and the warp-wide wait showed
    // 7-9 x the stage-1 time per codeword on config 4's NW = 4 rounds (two-word fold at T = 12..15
    // against the three-word fold, profiles/r02f_fold_calibration.txt), 3 x the modelled `exact`.
    static const double kFallPenalty = [] {
        const char* e = std::getenv("MDG_FALL_PENALTY");
        return e ? std::max(0.1, std::atof(e)) : 3.0;
    }();
    int last = -2;
    std::string dbg;
    const auto tp1 = std::chrono::steady_clock::now();
    const size_t no = opts.size();
    std::vector<std::array<double, kPlanT>> c1(no), c2(no);
    for (size_t i = 0; i < no; ++i) {
        const Opt& o = opts[i];
        const double m1 = o.sum / kSamples, m2 = o.psum / kSamples;
        tail(m1, std::max(0.0, o.sq / kSamples - m1 * m1), c1[i]);
        tail(m2, std::max(0.0, o.psq / kSamples - m2 * m2), c2[i]);
    }
    for (int T = 0; T < kPlanT; ++T) {
        double best = exact;
        int code = 0;
        for (size_t i = 0; i < no; ++i) {
            const Opt& o = opts[i];
            const double adds = (o.G + 1) / 2;
            const double f1 = fall(c1[i][T], 32 * GR);
            const double single = std::max(o.fw + adds + 1.4, 4.0 * o.G) + f1 * kFallPenalty * exact;
            if (single < best) best = single, code = o.code;
            if (!pairs || o.G != 1 || o.fw != 2) continue; // pair2_bits: one 2-word group
            const double f2 = fall(c2[i][T], 32 * (GP / 2));
            // a fall-through group takes the single bounds (folds already computed: POPCs only)
            // 3 LOP3 per pair (pair2_bits)
            const double pair = std::max(1.5 + 0.5 * adds + 0.9, 2.0 * o.G) +
                                f2 * (std::max(adds + 1.4, 4.0 * o.G) + f1 * kFallPenalty * exact);
            if (pair < best) best = pair, code = o.code | kFoldPair;
        }
        fp.code[T] = uint8_t(code);
        if (code != last) {
            char b[64];
            std::snprintf(b, sizeof b, " T>=%d:%s%d%s%s", T, code ? "G" : "exact", code & 15,
                          (code & kFoldDrop) ? "d" : (code & kFoldHalf) ? "h" : (code & kFold3) ? "3" : "",
                          (code & kFoldPair) ? "p" : "");
            dbg += b;
            last = code;
        }
    }
    if (std::getenv("MDG_PLAN_DEBUG")) {
        const auto tp2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[mdg fold] j=%u c=%u nw=%u (sampling %.1f us, choice %.1f us):%s\n", j, c, nw,
                     std::chrono::duration<double, std::micro>(tp1 - tp0).count(),
                     std::chrono::duration<double, std::micro>(tp2 - tp1).count(), dbg.c_str());
    }
    return fp;
}

static TabArgs tab_args(Engine::Impl& im, const GammaDev& g, const PlanEntry& pe, uint32_t* yt,
                        uint32_t k, uint32_t c, bool want_fold = true) {
    TabArgs a{};
    a.rows = g.rows; a.ytab = yt; a.binom = im.binom; a.prefix = pe.d_prefix; a.tr = pe.d_tr;
    a.k = k; a.p = pe.plan.p; a.s = pe.plan.s; a.emin = pe.plan.emin;
    a.npiv = uint32_t(pe.plan.prefix.size() - 1);
    a.id_rows = g.id_rows; a.add_const = (g.id_rows == k) ? c : 0; a.tx = pe.plan.TX;
    if (want_fold) // (the histogram kernel weighs everything: no stage-1 plan to sample)
        a.fold = sampled_fold_plan(im, uint32_t(&g - im.gammas.data()), k, c);
    if (!im.prune || !want_fold) // exact weights only
        std::memset(a.fold.code, 0, sizeof a.fold.code);
    a.rd = pe.plan.rd ? 1u : 0u;
    static const bool no_pos = std::getenv("MDG_NO_POS_KEY") != nullptr; // tests: the tab_find path
    a.pos_key = (!no_pos && !pe.plan.rd && pe.plan.tiles() <= 0xFFFFFFFFull) ? 1u : 0u; // see kPosFlag
    a.xtab = pe.plan.rd ? nullptr : ensure_xtab(im, uint32_t(&g - im.gammas.data()), k, pe.plan.p - 1);
    return a;
}

std::pair<uint64_t, uint64_t> Engine::split_range(uint32_t j, uint32_t c, uint32_t rank, uint32_t world) {
    check_round(j, c);
    return tab_split(impl_->plan(k_, c, impl_->gammas[j], plan_sms_).plan, rank, world);
}

uint64_t Engine::tasks(uint32_t j, uint32_t c) {
    check_round(j, c);
    return impl_->plan(k_, c, impl_->gammas[j], plan_sms_).plan.tiles();
}

RoundResult Engine::round(uint32_t j, uint32_t c, uint32_t stop_at, uint64_t task_lo, uint64_t task_hi,
                          uint32_t cutoff, bool shared_bound) {
    check_round(j, c);
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    const GammaDev& g = im.gammas[j];
    RoundResult rr;
    rr.combinations = binomial(k_, c);
    const PlanEntry& pe = im.plan(k_, c, g, plan_sms_);
    uint64_t lo = std::min(task_lo, pe.plan.tiles()), hi = std::min(task_hi, pe.plan.tiles());
    rr.task_lo = lo;
    rr.task_hi = hi;
    rr.plan_tag = plan_tag(im.rd, im.prune);
    uint32_t* yt = ensure_ytab(im, j, k_, pe.plan.s);
    unsigned long long* slot = im.take_slot();
    TabArgs a = tab_args(im, g, pe, yt, k_, c);
    a.stop_at = stop_at;
    a.cutoff = cutoff;
    a.tile_lo = lo; a.tile_hi = hi;
    a.best_key = slot; a.evaluated = slot + 1; a.counter = slot + 2;
    if (shared_bound) a.shared_key = im.xword(); // a split round of a multi-process run
    CK(cudaEventRecord(im.ev0, im.stream));
    if (hi > lo) {
        dispatch_nw_hid<TabLaunch>(g.nw, g.hid, a, hi - lo, im.stream, 0, size_t(0), sms_);
        CK(cudaGetLastError());
        im.cnt.launches += 1;
    }
    CK(cudaEventRecord(im.ev1, im.stream));
    im.read_slot(slot);
    CK(cudaStreamSynchronize(im.stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, im.ev0, im.ev1));
    rr.ms = ms;
    rr.key = im.host_slot[0];
    rr.evaluated = im.host_slot[1];
    rr.w = rr.key == ~0ull ? UINT32_MAX : uint32_t(rr.key >> kKeyShift);
    if (cutoff && rr.w >= cutoff) { // rd reports full minima; tab never reports >= cutoff
        rr.w = cutoff;
        rr.key = ~0ull;
        rr.bounded = true;
    }
    rr.stopped = !rr.bounded && rr.w != UINT32_MAX && rr.w <= stop_at;
    return rr;
}

RoundResult Engine::round_hist(uint32_t j, uint32_t c, uint64_t* hist, uint32_t rank, uint32_t world) {
    check_round(j, c);
    if (world < 1 || rank >= world) throw std::invalid_argument("round_hist: bad rank / world");
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    const GammaDev& g = im.gammas[j];
    const uint32_t nbins = n_ + 1;
    if (im.hist_cap < nbins) {
        cudaFree(im.hist_dev);
        CK(cudaMalloc(&im.hist_dev, nbins * 8));
        im.hist_cap = nbins;
    }
    RoundResult rr;
    rr.combinations = binomial(k_, c);
    // its own tile plan: every codeword is weighed (no pruning), so the plan aims for 4 tiles
    // per resident tab_hist block (its occupancy is set by the smem bins) -- the pruned
    // rounds' plan leaves most SMs idle on a config-5 sized round
    const int XSh = stride_for(int(g.nw) + (g.hid ? 1 : 0));
    int hocc = 0;
    dispatch_nw_hid<HistOcc>(g.nw, g.hid, size_t(kTX) * XSh * 4 + size_t(kWarps) * 2 * nbins * 4, &hocc);
    static const uint32_t kHistTpb = [] { // tiles per resident block (MDG_HIST_TPB, tuning)
        const char* e = std::getenv("MDG_HIST_TPB");
        return e ? uint32_t(std::max(1, std::atoi(e))) : 4u;
    }();
    // (plan_sms_: the SM count the ranks agreed on, so every rank cuts the same tiles)
    const PlanEntry& pe = im.plan(k_, c, g, plan_sms_, im.rd, false, kHistTpb, std::max(1, hocc) * plan_sms_);
    uint32_t* yt = ensure_ytab(im, j, k_, pe.plan.s);
    unsigned long long* slot = im.take_slot();
    CK(cudaMemsetAsync(im.hist_dev, 0, nbins * 8, im.stream));
    TabArgs a = tab_args(im, g, pe, yt, k_, c, /*want_fold=*/false);
    // multi-rank: rank r counts a contiguous tile range holding about
    // 1/world of the codewords; the counts are summed across ranks (NCCL, below, or the caller)
    const auto range = world > 1 ? tab_split(pe.plan, rank, world) : std::make_pair(uint64_t(0), pe.plan.tiles());
    a.tile_lo = range.first; a.tile_hi = range.second;
    a.evaluated = slot + 1; a.counter = slot + 2;
    a.nbins = nbins;
    a.hist = im.hist_dev;
    int XS = stride_for(int(g.nw) + (g.hid ? 1 : 0));
    size_t dyn = size_t(pe.plan.TX) * XS * 4 + size_t(kWarps) * 2 * nbins * 4; // bins + scratch per warp
    CK(cudaEventRecord(im.ev0, im.stream));
    if (a.tile_hi > a.tile_lo) {
        dispatch_nw_hid<TabLaunch>(g.nw, g.hid, a, a.tile_hi - a.tile_lo, im.stream, 2, dyn, sms_);
        CK(cudaGetLastError());
        im.cnt.launches += 1;
    }
    if (world > 1 && im.comm) { // every rank receives the whole histogram
        int rc = nccl().AllReduce(im.hist_dev, im.hist_dev, nbins, kNcclUint64, kNcclSum, im.comm, im.stream);
        if (rc != 0) throw std::runtime_error(std::string("ncclAllReduce: ") + nccl().GetErrorString(rc));
    }
    CK(cudaEventRecord(im.ev1, im.stream));
    CK(cudaMemcpyAsync(hist, im.hist_dev, nbins * 8, cudaMemcpyDeviceToHost, im.stream));
    im.cnt.d2h += nbins * 8;
    im.read_slot(slot);
    CK(cudaStreamSynchronize(im.stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, im.ev0, im.ev1));
    rr.ms = ms;
    rr.evaluated = im.host_slot[1];
    rr.task_lo = a.tile_lo;
    rr.task_hi = a.tile_hi;
    for (uint32_t w = 0; w < nbins; ++w)
        if (hist[w]) { rr.w = w; break; }
    rr.key = rr.w == UINT32_MAX ? ~0ull : (uint64_t(rr.w) << kKeyShift);
    return rr;
}

std::vector<uint32_t> Engine::witness(uint32_t j, uint32_t c, const RoundResult& rr) {
    check_round(j, c);
    if (rr.key == ~0ull) throw std::invalid_argument("witness: the round evaluated nothing");
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    const GammaDev& g = im.gammas[j];
    const bool pos = (rr.key & kPosFlag) != 0;
    const uint64_t task = pos ? (rr.key >> kPosBits) & 0xFFFFFFFFull : rr.key & (kPosFlag - 1);
    const uint32_t target = uint32_t(rr.key >> kKeyShift);
    std::vector<uint32_t> idx(c);
    // decode with the tile plan the round ran on (tagged by Engine::round / chain_loop), not
    // whatever kernel / pruning setting is current: the plans differ
    const bool tagged = (rr.plan_tag & 1u) != 0;
    const PlanEntry& pe = im.plan(k_, c, g, plan_sms_, tagged ? (rr.plan_tag & 4u) != 0 : im.rd,
                                  tagged ? (rr.plan_tag & 2u) != 0 : im.prune, 0, 0,
                                  tagged ? (rr.plan_tag >> 4) & 31u : 0u);
    if (task >= pe.plan.tiles()) throw std::invalid_argument("witness: key names no task of this round");
    if (pos) { // the kernel named the position: smem-side index << 11 | register-side index
        const uint32_t p = uint32_t(rr.key & ((1u << kPosBits) - 1));
        tab_decode(pe.plan, task, p >> 11, p & 0x7FFu, idx.data());
    } else {
        unsigned long long* slot = im.take_slot();
        uint32_t* yt = ensure_ytab(im, j, k_, pe.plan.s);
        TabArgs a = tab_args(im, g, pe, yt, k_, c);
        a.tile_lo = task; a.tile_hi = task + 1;
        a.find_out = slot + 3;
        a.find_target = target;
        dispatch_nw_hid<TabLaunch>(g.nw, g.hid, a, uint64_t(1), im.stream, 1, size_t(0), sms_);
        CK(cudaGetLastError());
        im.cnt.launches += 1;
        im.read_slot(slot);
        CK(cudaStreamSynchronize(im.stream));
        uint64_t f = im.host_slot[3];
        if (f == ~0ull) {
            char buf[160];
            std::snprintf(buf, sizeof buf, " (key 0x%llx, plan tag %u, task %llu of %llu, weight %u, slot %d)",
                          (unsigned long long)rr.key, rr.plan_tag, (unsigned long long)task,
                          (unsigned long long)pe.plan.tiles(), target, im.next_slot);
            throw std::logic_error(std::string("witness: winning tile holds no codeword of the round minimum") + buf);
        }
        tab_decode(pe.plan, task, uint32_t(f >> 32), uint32_t(f & 0xFFFFFFFFu), idx.data());
    }
    // the decoded rows must have the key's weight (compacted XOR + identity rows), else the
    // key was decoded against the wrong plan or Gamma: fail loudly instead of a wrong witness
    std::vector<uint32_t> acc(g.nw, 0);
    uint32_t wt = 0;
    for (uint32_t i = 0; i < c; ++i) {
        if (idx[i] >= k_ || (i && idx[i] <= idx[i - 1]))
            throw std::logic_error("witness: decoded combination is not a sorted c-subset");
        for (uint32_t w = 0; w < g.nw; ++w) acc[w] ^= g.host_rows[size_t(idx[i]) * g.nw + w];
        if (idx[i] < g.id_rows) ++wt;
    }
    for (uint32_t w = 0; w < g.nw; ++w) wt += uint32_t(__builtin_popcount(acc[w]));
    if (wt != target)
        throw std::logic_error("witness: decoded combination has weight " + std::to_string(wt) +
                               ", the round key says " + std::to_string(target) +
                               " (key from a different plan or Gamma set?)");
    return idx;
}

Engine::ChainResult Engine::chain_loop(uint32_t U0, uint32_t L0, uint32_t level_cap, bool exact,
                                       uint32_t k_last, uint32_t rank, uint32_t world,
                                       bool allreduce, uint64_t split_min) {
    allreduce = allreduce || world > 1;
    if (allreduce && !impl_->comm && !impl_->group)
        throw std::invalid_argument("chain_loop: no NCCL communicator or exchange group attached");
    if (impl_->group && (impl_->group->world != world || impl_->group_rank != rank))
        throw std::invalid_argument("chain_loop: rank / world differ from the attached exchange group");
    struct GroupLoop { // enter / leave the group's level loop (see ExchangeGroup::enter)
        ExchangeGroup* g;
        uint32_t r;
        GroupLoop(ExchangeGroup* g, uint32_t r) : g(g), r(r) { if (g) g->enter(r); }
        ~GroupLoop() { if (g) g->leave(r); }
    } group_loop(allreduce && !impl_->comm ? impl_->group.get() : nullptr, rank);
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    // host work per check: ~2e8 codewords (~0.1 ms of device time) between looks at `done`
    constexpr double kCheckWork = 2e8;
    ChainState init{U0, L0 < 1 ? 1u : L0, 0u, exact ? 1u : 0u, 0u, 0u, 0ull, nullptr};
    init.done = init.U <= init.L ? 1u : 0u;
    init.run = ++im.chain_runs;
    // Stop enqueuing at termination (single-rank loops). Small levels never add up to the
    // codeword count that triggers a look at `done`, so the host used to enqueue every level up
    // to k and the device skipped those past termination one launch at a time (config 1: 40
    // launches for 4 levels). finalize_round now publishes {levels closed, done} into mapped
    // host memory and the host stops enqueuing as soon as it sees `done` -- a volatile read per
    // level, no synchronization, no waiting (config 1: 0.30 -> 0.21 ms). MDG_LEVELS_AHEAD = a > 0
    // also keeps at most a levels enqueued beyond the last closed one (measured: config 1
    // no further gain for config 1, config 3 + 8 % and the eight-code bench - 2.5 %: the wait delays
    // enqueues the GPU could have had; off by default). Multi-rank loops keep the deterministic
    // enqueue sequence (every rank must enqueue the same collectives), so they use neither.
    static const uint32_t kAhead = [] {
        const char* e = std::getenv("MDG_LEVELS_AHEAD");
        return e ? uint32_t(std::max(0, std::atoi(e))) : 0u;
    }();
    volatile uint32_t* prog = nullptr;
    bool stopped_on_progress = false;
    if (!allreduce) {
        im.h_progress[0] = 0; // the stream is idle of earlier loops' writers (each loop ends synchronized)
        im.h_progress[1] = 0;
        uint32_t* dp = nullptr;
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), im.h_progress, 0));
        init.progress = dp;
        prog = im.h_progress;
    }
    *im.h_state = init;
    CK(cudaMemcpyAsync(im.d_state, im.h_state, sizeof(ChainState), cudaMemcpyHostToDevice, im.stream));
    im.cnt.h2d += sizeof(ChainState);
    const size_t max_rounds = size_t(k_) * m_;
    if (im.recs_cap < max_rounds) {
        cudaFree(im.d_recs);
        CK(cudaMalloc(&im.d_recs, max_rounds * sizeof(ChainRec)));
        im.recs_cap = max_rounds;
    }
    ChainResult res;
    size_t nrec = 0;
    double pending = 0;
    chain_stamp<<<1, 32, 0, im.stream>>>(&im.d_state->t0);
    CK(cudaGetLastError());
    im.cnt.launches += 1;
    // Tables: those of the first levels in one launch up front (while the levels add up to
    // <= 2e10 codewords and their tables to <= 32 MB), then each later level's tables for
    // all Gammas in one launch before its rounds.
    uint32_t built_to = 0;
    if (!init.done) {
        double work = 0;
        for (uint32_t c = 1; c <= k_ && c <= kMaxC && (!level_cap || c <= level_cap); ++c) {
            work += double(m_) * double(hb(k_, c));
            if (c > 1 && (work > 2e10 ||
                          table_bytes(im, k_, table_needs(im, m_, k_, 1, c, plan_sms_)) > (uint64_t{32} << 20)))
                break;
            built_to = c;
        }
        if (built_to >= 1) prebuild_tables(im, m_, k_, 1, built_to, plan_sms_);
    }
    uint32_t g = 1;
    bool done = init.done != 0;
    std::vector<uint32_t> rec_tag; // per enqueued round: the plan it runs on (plan_tag)
    static const bool fuse_tiles = std::getenv("MDG_NO_FUSED_TILES") == nullptr; // A/B switch
    uint64_t after_round = ~0ull; // launch count right after the last round launch
    bool synced = false;          // a host copy was enqueued since that launch
    // NVTX: one range per level's host enqueue (header-only NVTX3: no-ops unless a profiler
    // such as nsys / ncu --nvtx is attached)
    struct NvtxLevel {
        bool open = false;
        void start(uint32_t c) {
            char name[32];
            std::snprintf(name, sizeof name, "mdg level %u", c);
            nvtxRangePushA(name);
            open = true;
        }
        ~NvtxLevel() { if (open) nvtxRangePop(); }
    };
    while (!done && g <= k_) {
        if (level_cap && g > level_cap) break;
        if (prog) { // stop on `done`; optionally at most kAhead levels beyond the last closed one
            const auto t_wait = std::chrono::steady_clock::now();
            while (kAhead > 0 && prog[1] != init.run && g > prog[0] + kAhead) {
                if (std::chrono::steady_clock::now() - t_wait > std::chrono::milliseconds(2)) {
                    CK(cudaStreamSynchronize(im.stream)); // a long level: block instead of spinning
                    break;
                }
            }
            if (prog[1] == init.run) { // closed on the device: nothing more to enqueue
                done = true;
                stopped_on_progress = true;
                break;
            }
        }
        NvtxLevel nvtx_level;
        nvtx_level.start(g);
        bool too_big = g > kMaxC;
        if (!too_big) {
            try { binomial(k_, g); } catch (const std::overflow_error&) { too_big = true; }
        }
        if (too_big) { // the host loop would raise here only if it gets here
            CK(cudaMemcpyAsync(im.h_state, im.d_state, sizeof(ChainState), cudaMemcpyDeviceToHost, im.stream));
            CK(cudaStreamSynchronize(im.stream));
            synced = true;
            if (im.h_state->done) { done = true; break; }
            check_round(0, g); // throws the reference's error for this level
        }
        const uint32_t lb = lower_bound(m_, g, k_, k_last);
        if (g > built_to) {
            prebuild_tables(im, m_, k_, g, g, plan_sms_);
            built_to = g;
        }
        // this level's plans (only the first sampled level waits for them) and the next
        // level's, computed while the GPU runs the levels already enqueued
        if (hb(k_, g) >= (uint64_t{1} << 20))
            prefetch_fold_plans(im, m_, k_, g, level_cap ? std::min(level_cap, g + 1) : g + 1);
        // small levels of Gammas of one row width: all m rounds in one launch (tab_level);
        // multi-rank, only a level none of whose rounds is split (every rank runs it whole)
        const bool level_split = allreduce && double(binomial(k_, g)) >= double(split_min);
        bool fuse_level = !level_split && m_ >= 2 && m_ <= uint32_t(kMaxFuse) && fuse_max_ > 0 &&
                          double(m_) * double(binomial(k_, g)) <= fuse_max_;
        for (uint32_t j = 1; fuse_level && j < m_; ++j)
            fuse_level = im.gammas[j].nw == im.gammas[0].nw && im.gammas[j].hid == im.gammas[0].hid;
        if (fuse_level) {
            const GammaDev& g0 = im.gammas[0];
            const uint32_t fm = fuse_tiles ? m_ : 0u;
            const PlanEntry& pe = im.plan(k_, g, g0, plan_sms_, im.rd, im.prune, 0, 0, fm);
            for (uint32_t j = 0; j < m_; ++j) rec_tag.push_back(plan_tag(im.rd, im.prune, fm));
#ifndef MDG_NO_SLOT_RESERVE // (test builds only: reproduces the round-2 ring hazard)
            im.reserve_slots(int(m_) + 1); // the m rounds' slots + the scheduler's: one ring cycle
#endif
            LevelDesc L{};
            L.m = m_;
            L.T = pe.plan.tiles();
            TabArgs a{};
            for (uint32_t j = 0; j < m_; ++j) {
                const GammaDev& gd = im.gammas[j];
                uint32_t* yt = ensure_ytab(im, j, k_, pe.plan.s);
                TabArgs aj = tab_args(im, gd, pe, yt, k_, g);
                if (j == 0) a = aj;
                LevelRound& r = L.r[j];
                r.rows = aj.rows;
                r.ytab = aj.ytab;
                r.xtab = aj.xtab;
                r.slot = im.take_slot();
                r.rec = im.d_recs + nrec + j;
                r.fold = aj.fold;
                r.id_rows = aj.id_rows;
                r.add_const = aj.add_const;
            }
            unsigned long long* ls = im.take_slot(); // shared counter + blocks done

            a.st = im.d_state;
            a.counter = ls + 2;
            a.blocks_done = ls + 4;
            a.fin_st = im.d_state;
            a.fin_c = g;
            a.fin_lb = lb;
            const bool pdl = pdl_ && im.cnt.launches == after_round && !synced;
            const uint64_t total = uint64_t(m_) * L.T;
            dispatch_nw_hid<LevelLaunch>(g0.nw, g0.hid, a, L, total, pdl, im.stream, sms_);
            CK(cudaGetLastError());
            im.cnt.launches += 1;
            after_round = im.cnt.launches;
            synced = false;
            nrec += m_;
            pending += double(m_) * double(binomial(k_, g));
        }
        for (uint32_t j = 0; j < m_ && !fuse_level; ++j) {
            const GammaDev& gd = im.gammas[j];
            const PlanEntry& pe = im.plan(k_, g, gd, plan_sms_);
            uint32_t* yt = ensure_ytab(im, j, k_, pe.plan.s);
            unsigned long long* slot = im.take_slot();
            TabArgs a = tab_args(im, gd, pe, yt, k_, g);
            const uint64_t T = pe.plan.tiles();
            // a round below split_min codewords runs whole on every rank: the same result
            // everywhere with no exchange (the split would cost more in reduction latency)
            const bool split = allreduce && double(binomial(k_, g)) >= double(split_min);
            a.st = im.d_state;
            const auto range = split ? tab_split(pe.plan, rank, world) : std::make_pair(uint64_t(0), T);
            a.tile_lo = range.first;
            a.tile_hi = range.second;
            a.best_key = slot; a.evaluated = slot + 1; a.counter = slot + 2;
            if (split && !im.comm && im.group && im.group->ring && im.group->ring_ok) // group: shared key
                a.shared_key = im.group->ring + im.group_round % ExchangeGroup::kRing;
            if (split && im.comm) a.shared_key = im.xword(); // processes: the IPC-mapped word, if any
            const bool fuse = !split && a.tile_hi > a.tile_lo;
            if (fuse) { // the round kernel's last block closes the round: one launch per round
                a.fin_st = im.d_state;
                a.fin_rec = im.d_recs + nrec;
                a.blocks_done = slot + 4;
                a.fin_c = g;
                a.fin_j = j;
                a.fin_last = j + 1 == m_ ? 1u : 0u;
                a.fin_lb = lb;
            }
            if (a.tile_hi > a.tile_lo) {
                // PDL only when the previous stream operation is this chain's previous round
                // kernel (a table build or slot reset in between must complete first)
                const int mode = fuse && pdl_ && im.cnt.launches == after_round && !synced ? 3 : 0;
                dispatch_nw_hid<TabLaunch>(gd.nw, gd.hid, a, a.tile_hi - a.tile_lo, im.stream, mode, size_t(0), sms_);
                CK(cudaGetLastError());
                im.cnt.launches += 1;
                after_round = im.cnt.launches;
                synced = false;
            }
            if (split && im.comm) {
                int rc = nccl().AllReduce(slot, slot, 1, kNcclUint64, kNcclMin, im.comm, im.stream);
                if (rc != 0) throw std::runtime_error(std::string("ncclAllReduce: ") + nccl().GetErrorString(rc));
                im.xadvance(); // the owner frees the shared word (stream order: after the reduction)
            } else if (split) { // in-process exchange group
                CK(cudaEventRecord(im.group_ev, im.stream));
                std::vector<unsigned long long*> all;
                std::vector<cudaEvent_t> evs;
                im.group->exchange(rank, g, j, slot, im.group_ev, all, evs);
                GroupKeys gk{};
                gk.n = world;
                for (uint32_t r = 0; r < world; ++r) {
                    gk.key[r] = all[r];
                    if (r != rank) CK(cudaStreamWaitEvent(im.stream, evs[r], 0));
                }
                group_min<<<1, 32, 0, im.stream>>>(gk, slot);
                CK(cudaGetLastError());
                im.cnt.launches += 1;
                if (im.group->ring) { // rank 0 frees the shared word for round + kRing
                    if (rank == 0)
                        CK(cudaMemsetAsync(im.group->ring + im.group_round % ExchangeGroup::kRing, 0xFF,
                                           sizeof(unsigned long long), im.stream));
                    ++im.group_round;
                }
                synced = true; // the next round must not overlap the exchange (no PDL)
            }
            if (!fuse) {
                chain_finalize<<<1, 32, 0, im.stream>>>(im.d_state, slot, im.d_recs + nrec, g, j,
                                                        j + 1 == m_ ? 1u : 0u, lb);
                CK(cudaGetLastError());
                im.cnt.launches += 1;
            }
            ++nrec;
            rec_tag.push_back(plan_tag(im.rd, im.prune));
            pending += double(binomial(k_, g)) / (split ? world : 1);
        }
        ++g;
        if (pending >= kCheckWork || g > k_ || (level_cap && g > level_cap)) {
            CK(cudaMemcpyAsync(im.h_state, im.d_state, sizeof(ChainState), cudaMemcpyDeviceToHost, im.stream));
            CK(cudaStreamSynchronize(im.stream));
            im.cnt.d2h += sizeof(ChainState);
            synced = true;
            done = im.h_state->done != 0;
            pending = 0;
        }
    }
    CK(cudaMemcpyAsync(im.h_state, im.d_state, sizeof(ChainState), cudaMemcpyDeviceToHost, im.stream));
    std::vector<ChainRec> recs(nrec);
    if (nrec)
        CK(cudaMemcpyAsync(recs.data(), im.d_recs, nrec * sizeof(ChainRec), cudaMemcpyDeviceToHost, im.stream));
    CK(cudaStreamSynchronize(im.stream));
    const unsigned long long t_start = im.h_state->t0;
    im.cnt.d2h += sizeof(ChainState) + nrec * sizeof(ChainRec);
    res.U = im.h_state->U;
    res.L = im.h_state->L;
    res.plan_tag = plan_tag(im.rd, im.prune);
    res.done = im.h_state->done != 0;
    if (stopped_on_progress && !res.done)
        throw std::logic_error("chain_loop: the progress word reported termination but the loop state is not done");
    // run_bz_loop: capped when the loop reaches level cap + 1 (<= k) without being done
    res.capped = !res.done && level_cap && level_cap < k_ && g > level_cap;
    // per-round device time: between consecutive round closes (device clock;
    // includes the finalize launch, ~2 us)
    unsigned long long prev = t_start;
    for (size_t i = 0; i < nrec; ++i) {
        const ChainRec& r = recs[i];
        // every enqueued round must have been closed by THIS loop (its last block / finalize
        // launch): a record left over from an earlier loop would be a silent wrong trace
        if (r.run != init.run)
            throw std::logic_error("chain_loop: round record " + std::to_string(i) + " was not closed on the device (run " +
                                   std::to_string(r.run) + ", expected " + std::to_string(init.run) + "; c " +
                                   std::to_string(r.c) + ", j " + std::to_string(r.j) + ")");
        const double ms = r.t_ns > prev ? double(r.t_ns - prev) * 1e-6 : 0.0;
        prev = r.t_ns;
        if (!r.ran) continue;
        res.rounds.push_back({r.c, r.j, r.w, r.U_after, r.bounded, r.L_after, r.level_end, r.key,
                              r.evaluated, ms, rec_tag[i]});
    }
    return res;
}

Engine::BruteResult Engine::brute_force(uint32_t k, uint32_t n, const uint64_t* rows) {
    if (k < 1 || k > 62) throw std::invalid_argument("brute force: need 1 <= k <= 62");
    load(1, k, n, rows, nullptr); // raw basis rows, no identity elision
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    const GammaDev& g = im.gammas[0];
    const uint32_t a_rows = k / 2, b_rows = k - a_rows;
    const uint64_t na = uint64_t(1) << a_rows, nb = uint64_t(1) << b_rows;
    const uint32_t S = uint32_t(stride_for(int(g.nw)));
    uint32_t* ta = static_cast<uint32_t*>(im.arena.alloc(size_t(na) * S * 4));
    uint32_t* tb = static_cast<uint32_t*>(im.arena.alloc(size_t(nb) * S * 4));
    SpanArgs sa{};
    dispatch_nw_hid<SpanLaunch>(g.nw, false, g.rows, a_rows, b_rows, ta, tb, sa, 0, im.stream, sms_);
    CK(cudaGetLastError());
    im.cnt.launches += 2;
    const uint32_t YC = tab_yc(g.nw);
    const uint64_t nty = ceil_div(nb, YC);
    uint32_t tx = kTX;
    int resident = im.resident(g.nw, false, sms_);
    while (tx > 16 && ceil_div(na, tx) * nty < uint64_t(resident) * 16) tx /= 2;
    const uint64_t tiles = ceil_div(na, tx) * nty;
    unsigned long long* slot = im.take_slot();
    sa.ta = ta; sa.tb = tb; sa.na = na; sa.nb = nb; sa.nty = nty; sa.tx = tx;
    fold_limits(g.n_compact, g.nw, level_density(g.rho, k / 2), sa.fold_lim);
    sa.tile_lo = 0; sa.tile_hi = tiles;
    sa.best_key = slot; sa.evaluated = slot + 1; sa.counter = slot + 2; sa.find_out = slot + 3;
    CK(cudaEventRecord(im.ev0, im.stream));
    dispatch_nw_hid<SpanLaunch>(g.nw, false, g.rows, a_rows, b_rows, ta, tb, sa, 1, im.stream, sms_);
    CK(cudaGetLastError());
    im.cnt.launches += 1;
    CK(cudaEventRecord(im.ev1, im.stream));
    im.read_slot(slot);
    CK(cudaStreamSynchronize(im.stream));
    BruteResult br;
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, im.ev0, im.ev1));
    br.ms = ms;
    br.evaluated = im.host_slot[1] - 1; // tiles count the excluded zero pair (0, 0)
    const uint64_t key = im.host_slot[0];
    if (key == ~0ull) throw std::logic_error("brute force: no nonzero codeword evaluated");
    br.d = uint32_t(key >> kKeyShift);
    // witness: smallest (x, y) of the winning tile with that weight
    unsigned long long* fslot = im.take_slot();
    sa.tile_lo = key & ((uint64_t{1} << kKeyShift) - 1);
    sa.tile_hi = sa.tile_lo + 1;
    sa.best_key = fslot; sa.evaluated = fslot + 1; sa.counter = fslot + 2; // (unused by the search)
    sa.find_out = fslot + 3;
    sa.find_target = br.d;
    dispatch_nw_hid<SpanLaunch>(g.nw, false, g.rows, a_rows, b_rows, ta, tb, sa, 2, im.stream, sms_);
    CK(cudaGetLastError());
    im.cnt.launches += 1;
    im.read_slot(fslot);
    CK(cudaStreamSynchronize(im.stream));
    const uint64_t f = im.host_slot[3];
    if (f == ~0ull) throw std::logic_error("brute force: winning tile holds no codeword of weight d");
    const uint64_t xt = sa.tile_lo / nty, yt = sa.tile_lo % nty;
    const uint64_t x = xt * tx + (f >> 32), y = yt * YC + (f & 0xFFFFFFFFu);
    const uint64_t gx = x ^ (x >> 1), gy = y ^ (y >> 1);
    for (uint32_t b = 0; b < a_rows; ++b)
        if ((gx >> b) & 1u) br.idx.push_back(b);
    for (uint32_t b = 0; b < b_rows; ++b)
        if ((gy >> b) & 1u) br.idx.push_back(a_rows + b);
    return br;
}

Engine::Counters Engine::counters() const { return impl_->cnt; }
void Engine::set_pruning(bool on) { impl_->prune = on; }
void Engine::set_kernel(Kernel kern) {
    kernel_ = kern;
    impl_->rd = kern == Kernel::rd;
}
struct CUstream_st* Engine::stream() const { return impl_->stream; }
bool Engine::has_comm() const { return impl_->comm != nullptr; }

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "mdg_shared_bound handles are 64 bytes");
void Engine::shared_bound_create(uint8_t handle[64]) {
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    shared_bound_close();
    CK(cudaMalloc(&im.xring, Impl::kXRing * sizeof(unsigned long long)));
    CK(cudaMemset(im.xring, 0xFF, Impl::kXRing * sizeof(unsigned long long)));
    im.xowner = true;
    im.xround = 0;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, im.xring));
    std::memcpy(handle, &h, sizeof h);
}
void Engine::shared_bound_open(const uint8_t handle[64]) {
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    shared_bound_close();
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    im.xring = static_cast<unsigned long long*>(p);
    im.xowner = false;
    im.xround = 0;
}
void Engine::shared_bound_close() {
    Impl& im = *impl_;
    if (!im.xring) return;
    CK(cudaSetDevice(device_));
    CK(cudaStreamSynchronize(im.stream));
    if (im.xowner) CK(cudaFree(im.xring)); else CK(cudaIpcCloseMemHandle(im.xring));
    im.xring = nullptr;
    im.xowner = false;
    im.xround = 0;
}
void Engine::shared_bound_advance() { impl_->xadvance(); }
bool Engine::has_shared_bound() const { return impl_->xring != nullptr; }
void* Engine::scratch(size_t bytes) {
    Impl& im = *impl_;
    if (im.scratch_cap < bytes) {
        CK(cudaStreamSynchronize(im.stream));
        cudaFree(im.scratch);
        im.scratch = nullptr;
        CK(cudaMalloc(&im.scratch, bytes));
        im.scratch_cap = bytes;
    }
    return im.scratch;
}
void Engine::count_launch() { impl_->cnt.launches += 1; }
void Engine::reset_counters() { impl_->cnt = Counters{}; }
void Engine::timer_start() {
    CK(cudaSetDevice(device_));
    CK(cudaEventRecord(impl_->tev0, impl_->stream));
}
double Engine::timer_stop_ms() {
    CK(cudaSetDevice(device_));
    CK(cudaEventRecord(impl_->tev1, impl_->stream));
    CK(cudaEventSynchronize(impl_->tev1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, impl_->tev0, impl_->tev1));
    return ms;
}

void Engine::set_plan_sms(int sms) {
    if (sms < 1) throw std::invalid_argument("set_plan_sms: need >= 1");
    if (sms == plan_sms_) return;
    CK(cudaSetDevice(device_));
    CK(cudaStreamSynchronize(impl_->stream));
    plan_sms_ = sms;
    impl_->plans.clear(); // tile plans depend on it (their arena memory is simply kept)
}

void Engine::group_attach(std::shared_ptr<ExchangeGroup> g, uint32_t rank) {
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    if (!g) { // detach
        im.group.reset();
        im.group_rank = 0;
        return;
    }
    if (rank >= g->world) throw std::invalid_argument("group_attach: rank >= world");
    if (!im.group_ev) CK(cudaEventCreateWithFlags(&im.group_ev, cudaEventDisableTiming));
    // members on other devices read this engine's round slots (and it theirs): peer access
    {
        std::lock_guard<std::mutex> lk(g->mu);
        for (int d : g->devices) {
            if (d == device_) continue;
            int can = 0;
            CK(cudaDeviceCanAccessPeer(&can, device_, d));
            if (!can) throw std::invalid_argument("group_attach: devices " + std::to_string(device_) + " and " +
                                                  std::to_string(d) + " have no peer access");
            int atomics = 0; // the shared round key needs native peer atomics (NVLink)
            CK(cudaDeviceGetP2PAttribute(&atomics, cudaDevP2PAttrNativeAtomicSupported, device_, d));
            if (!atomics) g->ring_ok = false;
            for (auto [from, to] : {std::make_pair(device_, d), std::make_pair(d, device_)}) {
                CK(cudaSetDevice(from));
                cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else CK(e);
            }
            CK(cudaSetDevice(device_));
        }
        g->devices.push_back(device_);
        if (rank == 0 && !g->ring && !std::getenv("MDG_NO_SHARED_BOUND")) {
            CK(cudaMalloc(&g->ring, ExchangeGroup::kRing * sizeof(unsigned long long)));
            CK(cudaMemsetAsync(g->ring, 0xFF, ExchangeGroup::kRing * sizeof(unsigned long long), im.stream));
            CK(cudaStreamSynchronize(im.stream)); // before any member's (non-blocking) stream uses it
            g->ring_device = device_;
        }
    }
    im.group = std::move(g);
    im.group_rank = rank;
    im.group_round = 0;
}

void Engine::nccl_unique_id(uint8_t id[128]) {
    ncclUniqueId_t u;
    int rc = nccl().GetUniqueId(&u);
    if (rc != 0) throw std::runtime_error("ncclGetUniqueId failed");
    std::memcpy(id, u.internal, 128);
}

void Engine::nccl_init(const uint8_t id[128], uint32_t rank, uint32_t world) {
    CK(cudaSetDevice(device_));
    ncclUniqueId_t u;
    std::memcpy(u.internal, id, 128);
    int rc = nccl().CommInitRank(&impl_->comm, int(world), u, int(rank));
    if (rc != 0) throw std::runtime_error(std::string("ncclCommInitRank: ") + nccl().GetErrorString(rc));
    // every rank must cut a split round into the same tiles: the tile plans depend on the
    // resident-block count, so the ranks agree on the smallest SM count (identical on a B200
    // box; a mixed or partitioned node would otherwise split rounds inconsistently)
    uint64_t sms = uint64_t(sms_);
    nccl_reduce_min(&sms, 1);
    set_plan_sms(int(sms));
}

void Engine::nccl_reduce_min(uint64_t* keys, uint32_t count) {
    if (!impl_->comm) throw std::logic_error("nccl_reduce_min: communicator not initialised");
    CK(cudaSetDevice(device_));
    Impl& im = *impl_;
    if (im.red_cap < count) {
        cudaFree(im.red_dev);
        CK(cudaMalloc(&im.red_dev, size_t(count) * 8));
        im.red_cap = count;
    }
    CK(cudaMemcpyAsync(im.red_dev, keys, size_t(count) * 8, cudaMemcpyHostToDevice, im.stream));
    int rc = nccl().AllReduce(im.red_dev, im.red_dev, count, kNcclUint64, kNcclMin, im.comm, im.stream);
    im.cnt.h2d += size_t(count) * 8;
    im.cnt.d2h += size_t(count) * 8;
    if (rc != 0) throw std::runtime_error(std::string("ncclAllReduce: ") + nccl().GetErrorString(rc));
    CK(cudaMemcpyAsync(keys, im.red_dev, size_t(count) * 8, cudaMemcpyDeviceToHost, im.stream));
    CK(cudaStreamSynchronize(im.stream));
}

} // namespace mdg
