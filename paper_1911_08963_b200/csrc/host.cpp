// Host side of the B200 Brouwer–Zimmermann engine: F2 matrices, the Gamma
// systematization + permutation search, the bounds and the level loop.
// Everything here must reproduce the reference bit for bit (Gamma matrices,
// column_perm, per-round/per-level trace); tests/test_host.py pins it against
// the golden vectors made from the compiled reference.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <exception>
#include <thread>
#include <fstream>
#include <limits>
#include <random>
#include <sstream>

#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>

#include "mdg.hpp"

namespace mdg {

namespace {
// Small persistent host thread pool for independent candidate systematizations
// (thread creation would cost as much as the work). MDG_HOST_THREADS caps it.
class HostPool {
public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    unsigned size() const { return unsigned(workers_.size()) + 1; }
    // runs fn(i) for i in [0, n) on the pool and the calling thread; rethrows the first
    // error. Several callers (e.g. the batch front door's workers) may run jobs at once:
    // idle pool threads take items from any open job.
    void run(uint32_t n, const std::function<void(uint32_t)>& fn) {
        if (n == 0) return;
        auto job = std::make_shared<Job>();
        job->fn = &fn;
        job->n = n;
        {
            std::lock_guard<std::mutex> lk(m_);
            jobs_.push_back(job);
        }
        cv_.notify_all();
        job->drain();
        {
            std::unique_lock<std::mutex> lk(job->m);
            job->cv.wait(lk, [&] { return job->done.load() == job->n; });
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            jobs_.erase(std::remove(jobs_.begin(), jobs_.end(), job), jobs_.end());
        }
        if (job->err) std::rethrow_exception(job->err);
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

private:
    struct Job {
        const std::function<void(uint32_t)>* fn = nullptr;
        uint32_t n = 0;
        std::atomic<uint32_t> next{0}, done{0};
        std::mutex m;
        std::condition_variable cv;
        std::exception_ptr err;
        bool open() const { return next.load() < n; }
        void drain() {
            for (uint32_t i; (i = next.fetch_add(1)) < n;) {
                try {
                    (*fn)(i);
                } catch (...) {
                    std::lock_guard<std::mutex> lk(m);
                    if (!err) err = std::current_exception();
                }
                if (done.fetch_add(1) + 1 == n) {
                    std::lock_guard<std::mutex> lk(m);
                    cv.notify_all();
                }
            }
        }
    };
    HostPool() {
        unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        if (const char* e = std::getenv("MDG_HOST_THREADS")) hw = unsigned(std::max(1, std::atoi(e)));
        hw = std::min(hw, 16u);
        for (unsigned i = 1; i < hw; ++i) workers_.emplace_back([this] { loop(); });
    }
    void loop() {
        for (;;) {
            std::shared_ptr<Job> job;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] {
                    if (stop_) return true;
                    for (const auto& j : jobs_)
                        if (j->open()) return true;
                    return false;
                });
                if (stop_) return;
                for (const auto& j : jobs_)
                    if (j->open()) { job = j; break; }
            }
            if (job) job->drain();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_;
    std::vector<std::shared_ptr<Job>> jobs_;
    bool stop_ = false;
};
} // namespace

// ------------------------------------------------------------- BitMatrix
void BitMatrix::swap_rows(uint32_t a, uint32_t b) {
    if (a == b) return;
    uint64_t* x = row(a);
    uint64_t* y = row(b);
    for (uint32_t i = 0; i < W_; ++i) std::swap(x[i], y[i]);
}

// f2core.cpp:9-16 (column swap; the bits move, nothing else)
void BitMatrix::swap_cols(uint32_t a, uint32_t b) {
    if (a == b) return;
    const uint32_t wa = a >> 6, wb = b >> 6, sa = a & 63, sb = b & 63;
    for (uint32_t r = 0; r < rows_; ++r) { // branch-free: flip both bits where they differ
        uint64_t* p = row(r);
        const uint64_t d = ((p[wa] >> sa) ^ (p[wb] >> sb)) & 1u;
        p[wa] ^= d << sa;
        p[wb] ^= d << sb;
    }
}

uint32_t BitMatrix::row_weight(uint32_t r) const {
    uint32_t w = 0;
    const uint64_t* p = row(r);
    for (uint32_t i = 0; i < W_; ++i) w += static_cast<uint32_t>(__builtin_popcountll(p[i]));
    return w;
}

namespace {
// f2core.cpp:63-75: pivot = first row at or below `rank` with a 1 in `col`
uint32_t rref_in_place(BitMatrix& w) {
    uint32_t rank = 0;
    for (uint32_t col = 0; col < w.cols() && rank < w.rows(); ++col) {
        uint32_t pivot = rank;
        while (pivot < w.rows() && !w.get(pivot, col)) ++pivot;
        if (pivot == w.rows()) continue;
        w.swap_rows(rank, pivot);
        for (uint32_t r = 0; r < w.rows(); ++r)
            if (r != rank && w.get(r, col)) w.xor_row(r, rank);
        ++rank;
    }
    return rank;
}
} // namespace

uint32_t rank_of(const BitMatrix& m) {
    BitMatrix w = m;
    return rref_in_place(w);
}

BitMatrix rref_of(const BitMatrix& m) {
    BitMatrix w = m;
    uint32_t rank = rref_in_place(w);
    BitMatrix out(rank, m.cols());
    std::copy(w.data(), w.data() + size_t(rank) * w.words(), out.data());
    return out;
}

BitMatrix row_basis(const BitMatrix& m) {
    BitMatrix b = rref_of(m);
    if (b.rows() == 0) throw std::invalid_argument("row_basis: zero matrix spans the zero code");
    return b;
}

uint64_t hash_rows(const BitMatrix& m) {
    uint64_t h = 1469598103934665603ull;
    const uint64_t* p = m.data();
    for (size_t i = 0, e = size_t(m.rows()) * m.words(); i < e; ++i)
        for (int b = 0; b < 8; ++b) {
            h ^= (p[i] >> (8 * b)) & 0xff;
            h *= 1099511628211ull;
        }
    return h;
}

// ---------------------------------------------------------------- Gammas
// gamma.cpp:16-22 — output column j = input column perm[j]
BitMatrix permute_columns(const BitMatrix& m, const std::vector<uint32_t>& perm) {
    BitMatrix out(m.rows(), m.cols());
    for (uint32_t r = 0; r < m.rows(); ++r) {
        const uint64_t* src = m.row(r);
        uint64_t* dst = out.row(r);
        for (uint32_t j = 0; j < m.cols(); ++j)
            dst[j >> 6] |= ((src[perm[j] >> 6] >> (perm[j] & 63)) & 1u) << (j & 63);
    }
    return out;
}

// gamma.cpp:32-75 — progressive block diagonalization. Per block, the pivot is
// the first workable column at or after the target and, in it, the first row
// at or below the block rank; column swaps are mirrored into column_perm and
// into every earlier snapshot.
static GammaSet gamma_blocks(const BitMatrix& G) {
    const uint32_t k = G.rows();
    const uint32_t n = G.cols();
    GammaSet gs;
    gs.column_perm.resize(n);
    for (uint32_t i = 0; i < n; ++i) gs.column_perm[i] = i;
    BitMatrix w = G;
    for (uint32_t offset = 0; offset < n; offset += k) {
        uint32_t br = 0;
        for (; br < k; ++br) {
            const uint32_t target = offset + br;
            if (target >= n) break;
            uint32_t pc = n, pr = k;
            for (uint32_t c = target; c < n && pc == n; ++c) {
                const uint32_t wi = c >> 6;
                const uint64_t bit = uint64_t{1} << (c & 63);
                for (uint32_t r = br; r < k; ++r)
                    if (w.row(r)[wi] & bit) { pc = c; pr = r; break; }
            }
            if (pc == n) break;
            if (pc != target) {
                w.swap_cols(target, pc);
                std::swap(gs.column_perm[target], gs.column_perm[pc]);
                for (auto& snap : gs.gammas) snap.swap_cols(target, pc);
            }
            if (pr != br) w.swap_rows(br, pr);
            const uint32_t wi = target >> 6;
            const uint64_t bit = uint64_t{1} << (target & 63);
            for (uint32_t r = 0; r < k; ++r)
                if (r != br && (w.row(r)[wi] & bit)) w.xor_row(r, br);
        }
        if (br == 0) break;
        gs.gammas.push_back(w);
        gs.ranks.push_back(br);
        if (br < k) break;
    }
    gs.k_last = gs.ranks.back();
    return gs;
}

GammaSet compute_gamma_matrices(const BitMatrix& G) {
    const uint32_t k = G.rows();
    const uint32_t n = G.cols();
    if (k == 0 || k > n) throw std::invalid_argument("compute_gamma_matrices: need 1 <= k <= n");
    // gamma.cpp checks rank_of(G) == k first; the first block's elimination searches every
    // column for its pivots, so its rank is rank(G) -- the same check without a second pass
    GammaSet gs = gamma_blocks(G);
    if (gs.ranks.empty() || gs.ranks[0] != k)
        throw std::invalid_argument("compute_gamma_matrices: rank-deficient generator matrix");
    return gs;
}

// gamma.cpp:77-94 — identity plus `trials` Fisher–Yates shuffles
// (util.hpp:28-33, j = next() % i), keeping the lexicographic max of
// (m, k_last) with the earliest winner on ties. The permutations are drawn in
// the reference's order; the candidates (independent of each other; a column
// permutation keeps the rank, so the reference's per-candidate rank check is
// the identity's) are systematized on host threads, then chosen in order.
std::vector<uint32_t> trial_permutation(uint32_t n, uint64_t seed, uint64_t t) {
    SplitMix64 rng(seed);
    rng.discard(t * uint64_t(n ? n - 1 : 0));
    std::vector<uint32_t> perm(n);
    for (uint32_t i = 0; i < n; ++i) perm[i] = i;
    for (size_t i = perm.size(); i > 1; --i) {
        size_t j = static_cast<size_t>(rng.next() % i);
        std::swap(perm[i - 1], perm[j]);
    }
    return perm;
}

void parallel_for(uint32_t n, const std::function<void(uint32_t)>& fn) {
    if (n >= 2 && HostPool::get().size() > 1) HostPool::get().run(n, fn);
    else
        for (uint32_t i = 0; i < n; ++i) fn(i);
}

GammaSet gamma_for_permutation(const BitMatrix& G, const std::vector<uint32_t>& perm) {
    GammaSet g = gamma_blocks(permute_columns(G, perm));
    for (uint32_t j = 0; j < g.column_perm.size(); ++j) g.column_perm[j] = perm[g.column_perm[j]];
    return g;
}

// The largest (m, k_last) any column order can give: blocks take k columns each, so
// m <= ceil(n / k) and then k_last <= min(k, n - (m - 1) k). A candidate replaces the
// current best only when strictly larger (gamma.cpp:88-91), so once the identity order
// reaches this maximum no trial can change the result -- the trials are skipped.
bool gamma_set_is_maximal(const GammaSet& gs, uint32_t n, uint32_t k) {
    const uint32_t m_max = (n + k - 1) / k;
    const uint32_t kl_max = std::min(k, n - (m_max - 1) * k);
    return gs.m() == m_max && gs.k_last == kl_max;
}

// (m, k_last) of compute_gamma_matrices on the columns of G in the order `order`, without
// the systematization (gsearch.cu's kernel, on the host): block j's pivots are the greedy
// independent columns from position j*k on (row operations keep column dependencies), a
// pick at position pc swaps with `target` like gamma.cpp's column swap, and what the
// forward-only scan skips is dependent and stays so. cols: n column vectors, KW words each.
//
// The basis is kept fully reduced (each basis vector is zero at every other pivot), so a
// column reduces by XORing the basis vectors of the pivot bits it has set -- read off once,
// no data-dependent branch per basis vector -- and a new pivot is cleared from the others
// with masked XORs. Same independence test as an echelon basis, several times faster.
template <uint32_t KW>
static std::pair<uint32_t, uint32_t> block_shape_w(const uint64_t* cols, uint32_t n, uint32_t k,
                                                   std::vector<uint32_t>& order) {
    thread_local std::vector<uint64_t> basis; // by pivot bit: KW words each
    thread_local std::vector<uint32_t> pivs;  // pivots in insertion order
    basis.resize(size_t(64) * KW * KW);
    pivs.resize(k);
    uint32_t m = 0, k_last = 0;
    for (uint32_t o = 0; o < n; o += k) {
        uint64_t pmask[KW] = {};
        uint32_t cnt = 0, target = o, s = o;
        while (cnt < k && target < n) {
            bool found = false;
            for (; s < n; ++s) {
                uint64_t v[KW];
                const uint64_t* src = cols + size_t(order[s]) * KW;
                for (uint32_t w = 0; w < KW; ++w) v[w] = src[w];
                for (uint32_t w = 0; w < KW; ++w)
                    for (uint64_t mb = src[w] & pmask[w]; mb; mb &= mb - 1) {
                        const uint64_t* b = basis.data() + (size_t(w) * 64 + uint32_t(__builtin_ctzll(mb))) * KW;
                        for (uint32_t x = 0; x < KW; ++x) v[x] ^= b[x];
                    }
                uint32_t lowest = UINT32_MAX;
                for (uint32_t w = 0; w < KW; ++w)
                    if (v[w]) { lowest = w * 64 + uint32_t(__builtin_ctzll(v[w])); break; }
                if (lowest != UINT32_MAX) {
                    const uint32_t lw = lowest >> 6, lb = lowest & 63;
                    for (uint32_t i = 0; i < cnt; ++i) { // clear the new pivot from the others
                        uint64_t* b = basis.data() + size_t(pivs[i]) * KW;
                        const uint64_t sel = uint64_t{0} - ((b[lw] >> lb) & 1u);
                        for (uint32_t x = 0; x < KW; ++x) b[x] ^= v[x] & sel;
                    }
                    for (uint32_t x = 0; x < KW; ++x) basis[size_t(lowest) * KW + x] = v[x];
                    pmask[lw] |= uint64_t{1} << lb;
                    pivs[cnt] = lowest;
                    std::swap(order[target], order[s]);
                    ++cnt;
                    ++target;
                    ++s;
                    found = true;
                    break;
                }
            }
            if (!found) break;
        }
        if (cnt == 0) break;
        ++m;
        k_last = cnt;
        if (cnt < k) break;
    }
    return {m, k_last};
}

// column-vector stride for k rows: a template width (the layout block_shape expects)
static uint32_t shape_words(uint32_t k) {
    const uint32_t kw = (k + 63) / 64;
    return kw <= 4 ? kw : kw <= 8 ? 8 : kw <= 16 ? 16 : kw <= 32 ? 32 : (kw + 63) / 64 * 64;
}

// `order` is left in the column order compute_gamma_matrices ends with on it (its pivot
// column swaps, applied in the same sequence)
static std::pair<uint32_t, uint32_t> block_shape(const std::vector<uint64_t>& cols, uint32_t KW, uint32_t n,
                                                 uint32_t k, std::vector<uint32_t>& order) {
    switch (KW) {
        case 1: return block_shape_w<1>(cols.data(), n, k, order);
        case 2: return block_shape_w<2>(cols.data(), n, k, order);
        case 3: return block_shape_w<3>(cols.data(), n, k, order);
        case 4: return block_shape_w<4>(cols.data(), n, k, order);
        case 8: return block_shape_w<8>(cols.data(), n, k, order);
        case 16: return block_shape_w<16>(cols.data(), n, k, order);
        case 32: return block_shape_w<32>(cols.data(), n, k, order);
        default: break;
    }
    // very tall matrices: plain loop over KW words
    std::vector<uint64_t> basis(size_t(k) * KW), v(KW);
    std::vector<uint32_t> piv(k);
    uint32_t m = 0, k_last = 0;
    for (uint32_t o = 0; o < n; o += k) {
        uint32_t cnt = 0, target = o, s = o;
        while (cnt < k && target < n) {
            bool found = false;
            for (; s < n; ++s) {
                std::copy(cols.begin() + size_t(order[s]) * KW, cols.begin() + size_t(order[s] + 1) * KW, v.begin());
                for (uint32_t i = 0; i < cnt; ++i)
                    if ((v[piv[i] >> 6] >> (piv[i] & 63)) & 1u)
                        for (uint32_t w = 0; w < KW; ++w) v[w] ^= basis[size_t(i) * KW + w];
                uint32_t lowest = UINT32_MAX;
                for (uint32_t w = 0; w < KW && lowest == UINT32_MAX; ++w)
                    if (v[w]) lowest = w * 64 + uint32_t(__builtin_ctzll(v[w]));
                if (lowest != UINT32_MAX) {
                    std::copy(v.begin(), v.end(), basis.begin() + size_t(cnt) * KW);
                    piv[cnt] = lowest;
                    std::swap(order[target], order[s]);
                    ++cnt;
                    ++target;
                    ++s;
                    found = true;
                    break;
                }
            }
            if (!found) break;
        }
        if (cnt == 0) break;
        ++m;
        k_last = cnt;
        if (cnt < k) break;
    }
    return {m, k_last};
}

GammaSet best_gamma_over_permutations(const BitMatrix& G, uint32_t trials, uint64_t seed) {
    if (trials < 1) throw std::invalid_argument("best_gamma_over_permutations: trials must be >= 1");
    const uint32_t n = G.cols();
    const uint32_t k = G.rows();
    const uint32_t KW = shape_words(k);
    std::vector<uint64_t> cols(size_t(n) * KW, 0);
    for (uint32_t r = 0; r < k; ++r) {
        const uint64_t* row = G.row(r);
        for (uint32_t w = 0; w < G.words(); ++w)
            for (uint64_t bits = row[w]; bits; bits &= bits - 1) {
                const uint32_t c = w * 64 + uint32_t(__builtin_ctzll(bits));
                if (c < n) cols[size_t(c) * KW + (r >> 6)] |= uint64_t{1} << (r & 63);
            }
    }
    // the identity order's (m, k_last) by the block scan too: only the winner is systematized
    std::vector<uint32_t> ident(n);
    for (uint32_t i = 0; i < n; ++i) ident[i] = i;
    const std::pair<uint32_t, uint32_t> id_mk = block_shape(cols, KW, n, k, ident);
    const uint32_t m_max = (n + k - 1) / k;
    if (id_mk.first == 0 || (id_mk.first == m_max && id_mk.second == std::min(k, n - (m_max - 1) * k))) {
        GammaSet best = compute_gamma_matrices(G); // (throws the reference's errors)
        if (best.m() != id_mk.first || best.k_last != id_mk.second)
            throw std::logic_error("best_gamma_over_permutations: block scan disagrees with the systematization");
        return best; // maximal: no trial can replace it (gamma_set_is_maximal)
    }
    // Each candidate needs only its (m, k_last) to be compared (gamma.cpp:88-91): computed on
    // the column vectors by the greedy block scan (block_shape); the winner alone is
    // systematized in full, as the GPU search does. The winner is the earliest trial with the
    // largest (m, k_last) (strict improvement, in trial order); once a trial reaches the
    // largest value any order can have -- (ceil(n/k), min(k, n - (m-1)k)) -- no later trial can
    // win, so the trials are scanned in growing chunks (the first on the calling thread: the
    // pool's wake-up costs more than a few scans) and the scan stops at the first chunk that
    // holds a maximal trial. Same winner as scanning all of them; config 2's codes reach the
    // maximum within the first trials (145 -> ~20 us per code).
    const std::pair<uint32_t, uint32_t> mk_max{m_max, std::min(k, n - (m_max - 1) * k)};
    SplitMix64 rng(seed);
    std::vector<std::vector<uint32_t>> perms;
    perms.reserve(trials);
    std::vector<std::pair<uint32_t, uint32_t>> mk;
    mk.reserve(trials);
    int64_t win = -1;
    uint32_t bm = id_mk.first, bk = id_mk.second;
    const bool pool = uint64_t(k) * n >= 1024 && HostPool::get().size() > 1;
    for (uint32_t t0 = 0, chunk = 2; t0 < trials && !(bm == mk_max.first && bk == mk_max.second);
         t0 += chunk, chunk = std::min<uint32_t>(chunk * 2, 256)) {
        const uint32_t t1 = std::min(trials, t0 + chunk);
        for (uint32_t t = t0; t < t1; ++t) { // Fisher-Yates draws in trial order (one stream)
            std::vector<uint32_t> perm(n);
            for (uint32_t i = 0; i < n; ++i) perm[i] = i;
            for (size_t i = perm.size(); i > 1; --i) {
                size_t j = static_cast<size_t>(rng.next() % i);
                std::swap(perm[i - 1], perm[j]);
            }
            perms.push_back(std::move(perm));
            mk.emplace_back(0, 0);
        }
        std::function<void(uint32_t)> work = [&](uint32_t i) { // perms[t] -> its final order
            mk[t0 + i] = block_shape(cols, KW, n, k, perms[t0 + i]);
        };
        if (pool && t1 - t0 >= 8)
            HostPool::get().run(t1 - t0, work);
        else
            for (uint32_t i = 0; i < t1 - t0; ++i) work(i);
        for (uint32_t t = t0; t < t1; ++t)
            if (mk[t].first > bm || (mk[t].first == bm && mk[t].second > bk)) {
                bm = mk[t].first;
                bk = mk[t].second;
                win = t;
            }
    }
    // the winner is systematized on its FINAL column order (block_shape applied the pivot swaps):
    // every block's pivots are then in place, so gamma_blocks does no column swaps (each one
    // costs a pass over all rows of the matrix and of every earlier snapshot) -- the same Gamma
    // set and column_perm as systematizing the trial order itself
    GammaSet cand = win < 0 ? compute_gamma_matrices(G) : gamma_for_permutation(G, perms[size_t(win)]);
    if (cand.m() != bm || cand.k_last != bk)
        throw std::logic_error("best_gamma_over_permutations: block scan disagrees with the systematization");
    return cand;
}

// The BZ lower bound after level g (gamma.cpp:96-100): each of the m - 1 full information sets
// contributes g + 1, the last one g + 1 less the k - k_last rows it lacks (never below 0).
uint32_t lower_bound(uint32_t m, uint32_t g, uint32_t k, uint32_t k_last) {
    const int64_t last = int64_t(g) + 1 - (int64_t(k) - int64_t(k_last));
    return (m - 1) * (g + 1) + static_cast<uint32_t>(std::max<int64_t>(last, 0));
}

// The Singleton bound n - k + 1 as the loop's first upper bound (gamma.cpp:102-106).
uint32_t singleton_upper(uint32_t n, uint32_t k) {
    if (k == 0 || k > n) throw std::invalid_argument("singleton_upper: need n >= k >= 1");
    return n - k + 1;
}

// ------------------------------------------------------------ level loop
// engines.cpp:447-476, verbatim semantics: U from the bounds, L = max(1, lower);
// for g = 1..k, for each Gamma: the fast path ends the run as soon as U <= L
// (no L update for that level); otherwise run the round and U = min(U, w).
// After a full level L = max(L, lower_bound(m, g, k, k_last)); stop at L >= U.
// Added: the level cap (a round at level g > cap is never run; capped=true)
// and the trace. rs.stop_at carries the current L to the runner: a round may
// stop once it has found a weight <= L, because at that point U > L and
// d >= L, so its minimum is exactly L. rs.upper carries
// U: a runner may return min(w, U) and set rs.bounded when no codeword lies
// below U — U = min(U, w) and hence d and every (L, U) are unchanged.
EngineResult run_bz_loop(const GammaSet& gs, Bounds bounds, const RoundRunner& round,
                         uint32_t level_cap) {
    const uint32_t k = gs.k();
    const uint32_t m = gs.m();
    uint32_t U = bounds.upper;
    uint32_t L = bounds.lower < 1 ? 1 : bounds.lower;
    EngineResult res;
    bool done = U <= L;
    for (uint32_t g = 1; !done && g <= k; ++g) {
        if (level_cap && g > level_cap) {
            res.capped = true;
            break;
        }
        for (uint32_t j = 0; j < m; ++j) {
            if (U <= L) {
                done = true;
                break;
            }
            RoundStats rs;
            rs.g = g;
            rs.gamma_index = j;
            rs.stop_at = L;
            rs.upper = U;
            uint32_t w = round(j, g, rs);
            if (rs.bounded && w < U)
                throw std::logic_error("run_bz_loop: a bounded round reported a weight below U");
            res.stats.row_additions += rs.additions;
            res.stats.combinations += rs.combinations;
            res.stats.evaluated += rs.evaluated;
            res.stats.device_ms += rs.device_ms;
            res.stats.per_g.push_back(rs);
            res.stats.g_final = g;
            if (w < U) {
                U = w;
                res.witness_round = static_cast<int32_t>(res.stats.rounds.size());
            } else if (w == U && !rs.bounded && res.witness_round < 0) {
                res.witness_round = static_cast<int32_t>(res.stats.rounds.size());
            }
            res.stats.rounds.push_back({g, j, w, U, rs.bounded ? 1u : 0u});
        }
        if (done) break;
        uint32_t nl = lower_bound(m, g, k, gs.k_last);
        if (nl > L) L = nl;
        res.stats.levels.push_back({g, L, U});
        if (L >= U) done = true;
    }
    res.d = U;
    return res;
}

// ----------------------------------------------------------------- I/O
ParseError::ParseError(uint32_t line_no, uint32_t column_no, const std::string& message)
    : std::invalid_argument("line " + std::to_string(line_no) + ", column " +
                            std::to_string(column_no) + ": " + message),
      line(line_no),
      column(column_no) {}

namespace {
// One pass over the text of a matrix file: yields the payload lines (whitespace-trimmed,
// neither empty nor a '#' comment) with their 1-based line numbers. A last line without a
// newline counts when it has characters, as with std::getline.
class PayloadLines {
public:
    explicit PayloadLines(const std::string& text) : text_(text) {}
    uint32_t lines_read() const { return line_no_; }
    bool next(std::string& out) {
        while (pos_ < text_.size()) {
            size_t end = text_.find('\n', pos_);
            if (end == std::string::npos) end = text_.size();
            ++line_no_;
            size_t b = pos_, e = end;
            pos_ = end + 1;
            auto pad = [](char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; };
            while (b < e && pad(text_[b])) ++b;
            while (e > b && pad(text_[e - 1])) --e;
            if (b == e || text_[b] == '#') continue;
            out.assign(text_, b, e - b);
            return true;
        }
        return false;
    }

private:
    const std::string& text_;
    size_t pos_ = 0;
    uint32_t line_no_ = 0;
};
} // namespace

// The reference's text format (io.cpp:33-73): a header "n k", then k rows of exactly n symbols
// 0 / 1; blank lines and '#' comment lines anywhere; every error names its line and column
// (same messages and positions as the reference's ParseError).
BitMatrix parse_matrix(const std::string& text) {
    PayloadLines src(text);
    std::string item;
    if (!src.next(item)) throw ParseError(src.lines_read() + 1, 1, "missing header line");
    uint64_t n = 0, k = 0;
    {
        std::istringstream header(item);
        std::string extra;
        if (!(header >> n >> k)) throw ParseError(src.lines_read(), 1, "header must be two integers: n k");
        if (header >> extra) throw ParseError(src.lines_read(), 1, "header must be exactly: n k");
    }
    if (n == 0 || k == 0) throw ParseError(src.lines_read(), 1, "n and k must be >= 1");
    constexpr uint64_t kMaxDim = uint64_t{1} << 20;
    if (n > kMaxDim || k > kMaxDim) throw ParseError(src.lines_read(), 1, "unreasonable dimensions");
    BitMatrix M(static_cast<uint32_t>(k), static_cast<uint32_t>(n));
    for (uint32_t r = 0; r < k; ++r) {
        if (!src.next(item))
            throw ParseError(src.lines_read() + 1, 1,
                             "expected " + std::to_string(k) + " rows, got " + std::to_string(r));
        if (item.size() != n)
            throw ParseError(src.lines_read(), static_cast<uint32_t>(item.size()) + 1,
                             "row must have exactly " + std::to_string(n) + " symbols");
        uint64_t* words = M.row(r);
        for (uint32_t col = 0; col < n; ++col) {
            const char ch = item[col];
            if (ch == '1') words[col >> 6] |= uint64_t{1} << (col & 63);
            else if (ch != '0') throw ParseError(src.lines_read(), col + 1, "symbols must be 0 or 1");
        }
    }
    return M;
}

BitMatrix parse_matrix_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::invalid_argument("cannot open file: " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    return parse_matrix(ss.str());
}

// io.cpp:81-88: "n k" and one line of n symbols per row
std::string serialize_matrix(const BitMatrix& M) {
    const uint32_t k = M.rows(), n = M.cols();
    std::string out = std::to_string(n) + ' ' + std::to_string(k) + '\n';
    const size_t body = out.size();
    out.resize(body + size_t(k) * (size_t(n) + 1), '0');
    for (uint32_t r = 0; r < k; ++r) {
        char* line = &out[body + size_t(r) * (size_t(n) + 1)];
        const uint64_t* words = M.row(r);
        for (uint32_t col = 0; col < n; ++col)
            if ((words[col >> 6] >> (col & 63)) & 1u) line[col] = '1';
        line[n] = '\n';
    }
    return out;
}

// SURVEY.md §8d input convention (BASELINE.json configs): mt19937_64(seed),
// one draw per bit, bit = draw & 1, row-major over A; G = (I_k | A).
BitMatrix gen_matrix(uint32_t n, uint32_t k, uint64_t seed, bool identity) {
    if (k < 1 || n < 1 || (identity && k > n)) throw std::invalid_argument("gen_matrix: bad shape");
    std::mt19937_64 eng(seed);
    BitMatrix G(k, n);
    const uint32_t off = identity ? k : 0;
    for (uint32_t r = 0; r < k; ++r) {
        if (identity) G.set(r, r, true);
        for (uint32_t c = off; c < n; ++c)
            if (eng() & 1) G.set(r, c, true);
    }
    return G;
}

// ------------------------------------------------------------ binomials
// C(p, q) exactly (enumeration.cpp:9-20: 0 outside 0 <= q <= p, std::overflow_error past 64
// bits). With t = min(q, p - q) the running value after i factors is C(p - t + i, i): always an
// integer, never above the result, so it overflows iff the result does.
uint64_t binomial(uint32_t p, int64_t q) {
    if (q < 0 || q > static_cast<int64_t>(p)) return 0;
    const uint32_t t = static_cast<uint32_t>(std::min<int64_t>(q, static_cast<int64_t>(p) - q));
    unsigned __int128 v = 1;
    for (uint32_t i = 1, top = p - t + 1; i <= t; ++i, ++top) {
        v = v * top / i;
        if (v >> 64) throw std::overflow_error("binomial: value exceeds 64 bits");
    }
    return static_cast<uint64_t>(v);
}

// Revolving-door order R(n,t) = R(n-1,t) ++ reverse(R(n-1,t-1)) (n-1 appended)
// — Knuth TAOCP 7.2.1.3. No reference counterpart (its only Gray machinery is
// the binary reflected code, enumeration.hpp:19-20). idx ascending.
//   rank(c_1 < ... < c_t) = sum_i (-1)^(t-i) (C(c_i + 1, i) - 1)
//   unrank: for t down to 1, c_t = min{x : C(x+1, t) > r}, r <- C(x+1,t) - 1 - r
void rd_unrank(uint32_t c, uint64_t rank, uint32_t* idx) {
    uint64_t r = rank;
    for (uint32_t t = c; t >= 1; --t) {
        uint32_t x = t - 1;
        while (binomial(x + 1, t) <= r) ++x;
        idx[t - 1] = x;
        r = binomial(x + 1, t) - 1 - r;
    }
}

uint64_t rd_rank(uint32_t c, const uint32_t* idx) {
    int64_t s = 0;
    for (uint32_t i = 1; i <= c; ++i) {
        int64_t term = static_cast<int64_t>(binomial(idx[i - 1] + 1, i)) - 1;
        s += ((c - i) % 2 == 0) ? term : -term;
    }
    return static_cast<uint64_t>(s);
}

} // namespace mdg
