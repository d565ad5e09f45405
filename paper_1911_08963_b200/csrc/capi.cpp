// C ABI of the B200 Brouwer–Zimmermann engine (include/mdg.h) and the GPU
// front door min_weight (reference: engines.cpp:617-648 + cli.cpp:69-112).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "engine.hpp"
#include "mdg.h"
#include "mdg.hpp"

using namespace mdg;

struct mdg_ctx {
    std::unique_ptr<Engine> eng;
    std::vector<std::unique_ptr<Engine>> extra; // mdg_min_weight_batch's further streams
};

struct mdg_gset {
    GammaSet gs;
};

struct mdg_group {
    std::shared_ptr<ExchangeGroup> g;
};

struct mdg_run {
    EngineResult er;
    uint32_t n = 0, k = 0, m = 0, k_last = 0;
    uint32_t level_cap = 0, trials = 0, devices = 1, workers = 1;
    uint64_t seed = 0;
    std::string algorithm = "gpu", kernel = "tab";
    std::vector<uint32_t> perm;
    std::vector<uint64_t> gamma_hash;
    std::vector<uint64_t> witness;      // W words, original column order
    std::vector<uint32_t> witness_idx;  // row indices into Gamma witness_gamma
    int32_t witness_gamma = -1;
    uint32_t witness_level = 0;
    bool witness_ok = false;
    bool witness_from_trace = true;
    bool exact_rounds = false;
    double wall = 0, gamma_s = 0, loop_s = 0;
    Engine::Counters cnt;
};

namespace {

thread_local std::string g_err;

// NVTX range for the current scope (header-only NVTX3: a no-op unless a profiler is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return MDG_OK;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return MDG_EOVERFLOW;
    } catch (const CudaError& e) {
        g_err = e.what();
        return MDG_ECUDA;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return MDG_EINVAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MDG_EINTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return MDG_EINTERNAL;
    }
}

BitMatrix from_rows(const uint64_t* rows, uint32_t k, uint32_t n) {
    if (!rows) throw std::invalid_argument("null matrix");
    if (k < 1 || n < 1) throw std::invalid_argument("empty matrix");
    BitMatrix M(k, n);
    std::memcpy(M.data(), rows, size_t(k) * M.words() * 8);
    // padding bits must be zero (f2core.hpp:9-12)
    if (n % 64)
        for (uint32_t r = 0; r < k; ++r) M.row(r)[M.words() - 1] &= (uint64_t{1} << (n % 64)) - 1;
    return M;
}

uint32_t weight_of(const std::vector<uint64_t>& v) {
    uint32_t w = 0;
    for (uint64_t x : v) w += static_cast<uint32_t>(__builtin_popcountll(x));
    return w;
}

// XOR of Gamma_j rows idx, mapped back to the original column order with
// column_perm (the semantics of unpermute_columns, gamma.cpp:24-30).
std::vector<uint64_t> codeword(const GammaSet& gs, uint32_t j, const std::vector<uint32_t>& idx) {
    const BitMatrix& Gm = gs.gammas[j];
    std::vector<uint64_t> acc(Gm.words(), 0);
    for (uint32_t r : idx)
        for (uint32_t i = 0; i < Gm.words(); ++i) acc[i] ^= Gm.row(r)[i];
    std::vector<uint64_t> out(Gm.words(), 0);
    for (uint32_t c = 0; c < Gm.cols(); ++c)
        if ((acc[c >> 6] >> (c & 63)) & 1u) {
            uint32_t o = gs.column_perm[c];
            out[o >> 6] |= uint64_t{1} << (o & 63);
        }
    return out;
}

// w (original column order) lies in the code: permuted into the stored
// column order it does not raise the rank of Gamma_0 (same row space).
bool in_code(const GammaSet& gs, const std::vector<uint64_t>& w) {
    const BitMatrix& G0 = gs.gammas[0];
    BitMatrix S(G0.rows() + 1, G0.cols());
    std::memcpy(S.data(), G0.data(), size_t(G0.rows()) * G0.words() * 8);
    for (uint32_t c = 0; c < G0.cols(); ++c) {
        uint32_t o = gs.column_perm[c];
        if ((w[o >> 6] >> (o & 63)) & 1u) S.set(G0.rows(), c, true);
    }
    return rank_of(S) == G0.rows();
}

struct RoundLog {
    uint32_t j, c;
    RoundResult rr;
};

void upload(Engine& eng, const GammaSet& gs) {
    const uint32_t m = gs.m(), k = gs.k(), W = gs.gammas[0].words();
    std::vector<uint64_t> all(size_t(m) * k * W);
    for (uint32_t j = 0; j < m; ++j)
        std::memcpy(all.data() + size_t(j) * k * W, gs.gammas[j].data(), size_t(k) * W * 8);
    eng.load(m, k, gs.n(), all.data(), gs.ranks.data());
}

// best_gamma_over_permutations (gamma.cpp:77-94) with the trials on the GPU: the device
// returns the best trial's (m, k_last) and index; the host keeps the identity unless that
// is a strict improvement, exactly the reference's rule, and rebuilds the winner.
GammaSet best_gamma_gpu(Engine& eng, const BitMatrix& B, uint32_t trials, uint64_t seed) {
    if (trials < 1) throw std::invalid_argument("best_gamma_over_permutations: trials must be >= 1");
    GammaSet best = compute_gamma_matrices(B);
    if (gamma_set_is_maximal(best, B.cols(), B.rows())) return best;
    const uint64_t key = eng.permutation_search(B.data(), B.rows(), B.cols(), trials, seed);
    const uint32_t m = uint32_t(key >> kSearchMShift);
    const uint32_t kl = uint32_t((key >> kSearchKShift) & ((1u << (kSearchMShift - kSearchKShift)) - 1));
    const uint64_t t = ((uint64_t{1} << kSearchKShift) - 1) - (key & ((uint64_t{1} << kSearchKShift) - 1));
    if (m > best.m() || (m == best.m() && kl > best.k_last)) {
        GammaSet cand = gamma_for_permutation(B, trial_permutation(B.cols(), seed, t));
        if (cand.m() != m || cand.k_last != kl)
            throw std::logic_error("gpu permutation search: trial " + std::to_string(t) +
                                   " does not reproduce on the host");
        return cand;
    }
    return best;
}

// The level loop on the device over the Gamma set already loaded into eng
// (run_bz_loop, engines.cpp:447-476, with the GPU RoundRunner), then the
// witness. world > 1: every rank evaluates its contiguous task range of each
// round and the per-round keys are min-reduced across ranks.
void run_device_loop(Engine& eng, const GammaSet& gs, const mdg_config& cfg, uint32_t rank,
                     uint32_t world, mdg_reduce_fn reduce, void* user, mdg_run& out) {
    const uint32_t m = gs.m(), k = gs.k(), n = gs.n();
    if (eng.m() != m || eng.k() != k || eng.n() != n)
        throw std::invalid_argument("device holds a different Gamma set");
    eng.set_kernel(cfg.kernel == MDG_KERNEL_RD ? Kernel::rd : Kernel::tab);
    Engine::Counters c0 = eng.counters();
    std::vector<RoundLog> log;
    const uint64_t split_min = cfg.split_min ? cfg.split_min : uint64_t(200000000);
    auto do_round = [&](uint32_t j, uint32_t g, uint32_t stop_at, uint32_t cutoff) {
        RoundResult rr;
        // a round below split_min codewords runs whole on every rank: no exchange (and the
        // in-process group has no host-side reducer: its host-loop rounds -- the witness
        // search only -- run whole too)
        if (world <= 1 || double(binomial(k, g)) < double(split_min) || reduce == &mdg_group_reduce_min) {
            rr = eng.round(j, g, stop_at, 0, UINT64_MAX, cutoff);
        } else {
            const auto [lo, hi] = eng.split_range(j, g, rank, world);
            rr = eng.round(j, g, stop_at, lo, hi, cutoff, /*shared_bound=*/true);
            uint64_t key = rr.key;
            int rc = reduce(user, &key, 1);
            if (rc != 0) throw std::runtime_error("mdg: cross-rank reduction failed");
            eng.shared_bound_advance(); // every rank has finished the round: the owner frees its word
            rr.key = key;
            rr.bounded = false;
            rr.w = key == ~0ull ? UINT32_MAX : uint32_t(key >> kKeyShift);
            if (cutoff && (key == ~0ull || rr.w >= cutoff)) {
                rr.w = cutoff;
                rr.key = ~0ull;
                rr.bounded = true;
            }
        }
        return rr;
    };
    RoundRunner runner = [&](uint32_t j, uint32_t g, RoundStats& rs) -> uint32_t {
        RoundResult rr = do_round(j, g, rs.stop_at, cfg.exact_rounds ? 0u : rs.upper);
        rs.bounded = rr.bounded;
        rs.combinations = rr.combinations;
        rs.evaluated = rr.evaluated;
        rs.additions = rr.evaluated; // one row XOR per evaluated codeword
        rs.device_ms = rr.ms;
        log.push_back({j, g, rr});
        return rr.w;
    };
    Bounds bounds;
    bounds.lower = 1;
    bounds.upper = singleton_upper(n, k);
    // NCCL or the in-process exchange group: the reduction is enqueued on the stream
    const bool device_reduce = reduce == &mdg_nccl_reduce_min || reduce == &mdg_group_reduce_min;
    eng.timer_start();
    if (world == 1 || device_reduce) {
        // device-chained level loop: same semantics as run_bz_loop, no host sync per round;
        // with the NCCL reducer the per-round allreduce(min) is enqueued in-stream
        Engine::ChainResult cr = eng.chain_loop(bounds.upper, bounds.lower, cfg.level_cap,
                                                cfg.exact_rounds != 0, gs.k_last, rank, world,
                                                device_reduce, split_min);
        EngineResult& er = out.er;
        uint32_t U = bounds.upper;
        for (const auto& r : cr.rounds) {
            RoundStats rs;
            rs.g = r.c;
            rs.gamma_index = r.j;
            rs.bounded = r.bounded != 0;
            rs.combinations = binomial(k, r.c);
            rs.evaluated = r.evaluated;
            rs.additions = r.evaluated;
            rs.device_ms = r.ms;
            er.stats.row_additions += rs.additions;
            er.stats.combinations += rs.combinations;
            er.stats.evaluated += rs.evaluated;
            er.stats.device_ms += rs.device_ms;
            er.stats.per_g.push_back(rs);
            er.stats.g_final = r.c;
            if (r.w < U) {
                U = r.w;
                er.witness_round = int32_t(er.stats.rounds.size());
            } else if (r.w == U && !rs.bounded && er.witness_round < 0) {
                er.witness_round = int32_t(er.stats.rounds.size());
            }
            if (U != r.U_after) throw std::logic_error("chain_loop: device U disagrees with the trace");
            er.stats.rounds.push_back({r.c, r.j, r.w, r.U_after, r.bounded});
            if (r.level_end) er.stats.levels.push_back({r.c, r.L_after, r.U_after});
            RoundResult rr;
            rr.w = r.w;
            rr.key = r.key;
            rr.bounded = r.bounded != 0;
            rr.evaluated = r.evaluated;
            rr.combinations = rs.combinations;
            rr.ms = r.ms;
            rr.plan_tag = r.plan_tag;
            log.push_back({r.j, r.c, rr});
        }
        er.d = cr.U;
        er.capped = cr.capped;
    } else {
        out.er = run_bz_loop(gs, bounds, runner, cfg.level_cap);
    }
    out.loop_s = eng.timer_stop_ms() * 1e-3;
    const uint32_t d = out.er.d;

    static const bool timing = std::getenv("MDG_TIMING") != nullptr;
    auto tw0 = std::chrono::steady_clock::now();
    if (cfg.want_witness) {
        const RoundLog* src = nullptr;
        if (out.er.witness_round >= 0) src = &log[size_t(out.er.witness_round)];
        RoundLog extra;
        if (!src) {
            // U never came from a round (it is the Singleton bound, or a run
            // with no rounds): search the levels for a codeword of weight U.
            out.witness_from_trace = false;
            for (uint32_t g = 1; g <= k && !src; ++g)
                for (uint32_t j = 0; j < m && !src; ++j) {
                    RoundResult rr = do_round(j, g, d, d + 1);
                    if (!rr.bounded && rr.w <= d) {
                        extra = {j, g, rr};
                        src = &extra;
                    }
                }
        }
        if (src) {
            out.witness_idx = eng.witness(src->j, src->c, src->rr);
            out.witness_gamma = int32_t(src->j);
            out.witness_level = src->c;
            out.witness = codeword(gs, src->j, out.witness_idx);
            auto tw1 = std::chrono::steady_clock::now();
            out.witness_ok = weight_of(out.witness) == d && in_code(gs, out.witness) && src->rr.w == d;
            if (timing)
                std::fprintf(stderr, "[mdg timing] witness search %.1f us (from trace: %d), check %.1f us\n",
                             std::chrono::duration<double>(tw1 - tw0).count() * 1e6,
                             int(out.witness_from_trace),
                             std::chrono::duration<double>(std::chrono::steady_clock::now() - tw1).count() * 1e6);
        }
    }
    Engine::Counters c1 = eng.counters();
    out.cnt.launches = c1.launches - c0.launches;
    out.cnt.h2d = c1.h2d - c0.h2d;
    out.cnt.d2h = c1.d2h - c0.d2h;
    out.n = n;
    out.k = k;
    out.m = m;
    out.k_last = gs.k_last;
    out.perm = gs.column_perm;
    out.gamma_hash.clear();
    for (uint32_t j = 0; j < m; ++j) out.gamma_hash.push_back(hash_rows(gs.gammas[j]));
    out.level_cap = cfg.level_cap;
    out.trials = cfg.trials;
    out.seed = cfg.seed;
    out.devices = world;
    out.workers = cfg.workers ? cfg.workers : 1;
    out.kernel = cfg.kernel == MDG_KERNEL_RD ? "rd" : "tab";
    out.exact_rounds = cfg.exact_rounds != 0;
}

// min_weight on the device(s): row_basis -> Gamma search -> Singleton U ->
// level loop -> witness (engines.cpp:617-648).
std::unique_ptr<mdg_run> min_weight_device(Engine& eng, const BitMatrix& G, const mdg_config& cfg,
                                           uint32_t rank, uint32_t world, mdg_reduce_fn reduce,
                                           void* user) {
    auto t0 = std::chrono::steady_clock::now();
    auto run = std::make_unique<mdg_run>();
    Engine::Counters c0 = eng.counters();
    std::optional<GammaSet> gsearch;
    {
        NvtxRange r("mdg gamma search");
        gsearch.emplace(cfg.gamma_search == MDG_GAMMA_GPU
                            ? best_gamma_gpu(eng, row_basis(G), cfg.trials, cfg.seed)
                            : best_gamma_over_permutations(row_basis(G), cfg.trials, cfg.seed));
    }
    const GammaSet& gs = *gsearch;
    auto t1 = std::chrono::steady_clock::now();
    run->gamma_s = std::chrono::duration<double>(t1 - t0).count();
    {
        NvtxRange r("mdg upload");
        upload(eng, gs);
    }
    {
        NvtxRange r("mdg level loop + witness");
        run_device_loop(eng, gs, cfg, rank, world, reduce, user, *run);
    }
    Engine::Counters c1 = eng.counters();
    run->cnt.launches = c1.launches - c0.launches;
    run->cnt.h2d = c1.h2d - c0.h2d;
    run->cnt.d2h = c1.d2h - c0.d2h;
    run->wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return run;
}

std::string json_of(const mdg_run& r) {
    std::ostringstream o;
    const auto& st = r.er.stats;
    o << "{\"d\":" << r.er.d << ",\"n\":" << r.n << ",\"k\":" << r.k << ",\"algorithm\":\""
      << r.algorithm << "\",\"m\":" << r.m << ",\"k_last\":" << r.k_last
      << ",\"g_final\":" << st.g_final << ",\"row_additions\":" << st.row_additions
      << ",\"combinations\":" << st.combinations << ",\"wall_seconds\":" << r.wall
      << ",\"seed\":" << r.seed << ",\"workers\":" << r.workers;
    // new keys: witness, trace, level cap, devices, throughput
    o << ",\"capped\":" << (r.er.capped ? "true" : "false") << ",\"level_cap\":" << r.level_cap
      << ",\"exact_rounds\":" << (r.exact_rounds ? "true" : "false")
      << ",\"devices\":" << r.devices << ",\"kernel\":\"" << r.kernel << "\""
      << ",\"combinations_evaluated\":" << st.evaluated
      << ",\"device_seconds\":" << st.device_ms * 1e-3 << ",\"loop_seconds\":" << r.loop_s
      << ",\"gamma_seconds\":" << r.gamma_s << ",\"gpu_launches\":" << r.cnt.launches
      << ",\"codewords_per_s\":" << (st.device_ms > 0 ? double(st.evaluated) / (st.device_ms * 1e-3) : 0.0);
    o << ",\"witness\":";
    if (r.witness.empty()) {
        o << "null";
    } else {
        o << "\"";
        for (uint32_t c = 0; c < r.n; ++c) o << (((r.witness[c >> 6] >> (c & 63)) & 1u) ? '1' : '0');
        o << "\"";
    }
    o << ",\"witness_ok\":" << (r.witness_ok ? "true" : "false") << ",\"trace\":[";
    for (size_t i = 0; i < st.rounds.size(); ++i) {
        const auto& x = st.rounds[i];
        o << (i ? "," : "") << "[" << x.c << "," << x.j << "," << x.w << "," << x.U_after << ","
          << x.bounded << "]";
    }
    o << "],\"levels\":[";
    for (size_t i = 0; i < st.levels.size(); ++i) {
        const auto& x = st.levels[i];
        o << (i ? "," : "") << "[" << x.c << "," << x.L_after << "," << x.U_after << "]";
    }
    o << "]}";
    return o.str();
}

long copy_out(const std::string& s, char* buf, size_t cap) {
    if (!buf || s.size() + 1 > cap) {
        g_err = "buffer too small (need " + std::to_string(s.size() + 1) + " bytes)";
        return -static_cast<long>(s.size() + 1);
    }
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<long>(s.size());
}

} // namespace

std::string mdg_json_of(const mdg_run& r) { return json_of(r); }

extern "C" {

const char* mdg_last_error(void) { return g_err.c_str(); }
const char* mdg_version(void) { return "mdg 0.1 (sm_100a)"; }

int mdg_open(int device, mdg_ctx** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null out");
        auto c = std::make_unique<mdg_ctx>();
        c->eng = std::make_unique<Engine>(device);
        *out = c.release();
    });
}

void mdg_close(mdg_ctx* ctx) { delete ctx; }

int mdg_load_gammas(mdg_ctx* ctx, uint32_t m, uint32_t k, uint32_t n, const uint64_t* rows,
                    const uint32_t* ranks) {
    return guard([&] {
        if (!ctx || !rows) throw std::invalid_argument("null argument");
        ctx->eng->load(m, k, n, rows, ranks);
    });
}

static void fill_out(const RoundResult& rr, mdg_round_out* out) {
    out->min_weight = rr.w;
    out->stopped_early = rr.stopped ? 1u : 0u;
    out->bounded = rr.bounded ? 1u : 0u;
    out->plan_tag = rr.plan_tag;
    out->argmin_key = rr.key;
    out->combinations = rr.combinations;
    out->evaluated = rr.evaluated;
    out->task_lo = rr.task_lo;
    out->task_hi = rr.task_hi;
    out->device_ms = rr.ms;
}

static RoundResult to_rr(const mdg_round_out* out) {
    RoundResult rr;
    rr.w = out->min_weight;
    rr.key = out->argmin_key;
    rr.plan_tag = out->plan_tag;
    rr.combinations = out->combinations;
    rr.evaluated = out->evaluated;
    return rr;
}

int mdg_round(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t stop_at, mdg_round_out* out) {
    return guard([&] {
        if (!ctx || !out) throw std::invalid_argument("null argument");
        fill_out(ctx->eng->round(j, c, stop_at), out);
    });
}

int mdg_round_tasks(mdg_ctx* ctx, uint32_t j, uint32_t c, uint64_t* n_tasks) {
    return guard([&] {
        if (!ctx || !n_tasks) throw std::invalid_argument("null argument");
        *n_tasks = ctx->eng->tasks(j, c);
    });
}

int mdg_round_split(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t rank, uint32_t world,
                    uint64_t* task_lo, uint64_t* task_hi) {
    return guard([&] {
        if (!ctx || !task_lo || !task_hi) throw std::invalid_argument("null argument");
        if (world < 1 || rank >= world) throw std::invalid_argument("bad rank / world");
        const auto r = ctx->eng->split_range(j, c, rank, world);
        *task_lo = r.first;
        *task_hi = r.second;
    });
}

int mdg_plan_split(uint32_t k, uint32_t c, uint32_t nw32, uint32_t resident_blocks, uint32_t rank,
                   uint32_t world, uint64_t* task_lo, uint64_t* task_hi, uint64_t* codewords) {
    return guard([&] {
        if (!task_lo || !task_hi || !codewords) throw std::invalid_argument("null argument");
        if (world < 1 || rank >= world) throw std::invalid_argument("bad rank / world");
        if (c < 1 || c > k || k > kMaxK || c > kMaxC) throw std::invalid_argument("need 1 <= c <= k <= 1024, c <= 64");
        binomial(k, c);
        const TabPlan pl = make_tab_plan(k, c, template_width(std::max(1u, nw32)), std::max(1u, resident_blocks));
        const auto r = tab_split(pl, rank, world);
        *task_lo = r.first;
        *task_hi = r.second;
        *codewords = tab_codewords_before(pl, r.second) - tab_codewords_before(pl, r.first);
    });
}

int mdg_round_range(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t stop_at, uint64_t task_lo,
                    uint64_t task_hi, mdg_round_out* out) {
    return guard([&] {
        if (!ctx || !out) throw std::invalid_argument("null argument");
        if (task_lo > task_hi) throw std::invalid_argument("task range reversed");
        fill_out(ctx->eng->round(j, c, stop_at, task_lo, task_hi), out);
    });
}

int mdg_round_bounded(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t stop_at, uint32_t cutoff,
                      uint64_t task_lo, uint64_t task_hi, mdg_round_out* out) {
    return guard([&] {
        if (!ctx || !out) throw std::invalid_argument("null argument");
        if (task_lo > task_hi) throw std::invalid_argument("task range reversed");
        fill_out(ctx->eng->round(j, c, stop_at, task_lo, task_hi, cutoff), out);
    });
}

int mdg_round_hist(mdg_ctx* ctx, uint32_t j, uint32_t c, uint64_t* hist, mdg_round_out* out) {
    return guard([&] {
        if (!ctx || !hist || !out) throw std::invalid_argument("null argument");
        fill_out(ctx->eng->round_hist(j, c, hist), out);
    });
}

int mdg_shared_bound_create(mdg_ctx* ctx, uint8_t handle[64]) {
    return guard([&] {
        if (!ctx || !handle) throw std::invalid_argument("null argument");
        ctx->eng->shared_bound_create(handle);
    });
}

int mdg_shared_bound_open(mdg_ctx* ctx, const uint8_t handle[64]) {
    return guard([&] {
        if (!ctx || !handle) throw std::invalid_argument("null argument");
        ctx->eng->shared_bound_open(handle);
    });
}

int mdg_shared_bound_close(mdg_ctx* ctx) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null ctx");
        ctx->eng->shared_bound_close();
    });
}

int mdg_round_hist_dist(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t rank, uint32_t world,
                        uint64_t* hist, mdg_round_out* out, int* reduced) {
    return guard([&] {
        if (!ctx || !hist || !out) throw std::invalid_argument("null argument");
        if (world < 1 || rank >= world) throw std::invalid_argument("bad rank / world");
        fill_out(ctx->eng->round_hist(j, c, hist, rank, world), out);
        if (reduced) *reduced = (world > 1 && ctx->eng->has_comm()) ? 1 : 0;
    });
}

int mdg_round_witness(mdg_ctx* ctx, uint32_t j, uint32_t c, const mdg_round_out* out, uint32_t* idx) {
    return guard([&] {
        if (!ctx || !out || !idx) throw std::invalid_argument("null argument");
        auto v = ctx->eng->witness(j, c, to_rr(out));
        std::memcpy(idx, v.data(), v.size() * 4);
    });
}

int mdg_set_kernel(mdg_ctx* ctx, int kernel) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null argument");
        if (kernel != MDG_KERNEL_TAB && kernel != MDG_KERNEL_RD)
            throw std::invalid_argument("unknown kernel");
        ctx->eng->set_kernel(kernel == MDG_KERNEL_RD ? Kernel::rd : Kernel::tab);
    });
}

int mdg_set_pruning(mdg_ctx* ctx, int on) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null argument");
        ctx->eng->set_pruning(on != 0);
    });
}

// ------------------------------------------------------------- gamma sets
int mdg_gset_build(const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials, uint64_t seed,
                   mdg_gset** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null out");
        auto g = std::make_unique<mdg_gset>();
        g->gs = best_gamma_over_permutations(row_basis(from_rows(G, k, n)), trials, seed);
        *out = g.release();
    });
}

int mdg_gset_build_gpu(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials,
                       uint64_t seed, mdg_gset** out) {
    return guard([&] {
        if (!ctx || !out || !G) throw std::invalid_argument("null argument");
        auto g = std::make_unique<mdg_gset>();
        g->gs = best_gamma_gpu(*ctx->eng, row_basis(from_rows(G, k, n)), trials, seed);
        *out = g.release();
    });
}

int mdg_gset_compute(const uint64_t* G, uint32_t k, uint32_t n, mdg_gset** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null out");
        auto g = std::make_unique<mdg_gset>();
        g->gs = compute_gamma_matrices(from_rows(G, k, n));
        *out = g.release();
    });
}

void mdg_gset_free(mdg_gset* gs) { delete gs; }

int mdg_gset_info(const mdg_gset* g, uint32_t* m, uint32_t* k, uint32_t* n, uint32_t* k_last) {
    return guard([&] {
        if (!g) throw std::invalid_argument("null gset");
        if (m) *m = g->gs.m();
        if (k) *k = g->gs.k();
        if (n) *n = g->gs.n();
        if (k_last) *k_last = g->gs.k_last;
    });
}

int mdg_gset_gamma(const mdg_gset* g, uint32_t j, uint64_t* rows) {
    return guard([&] {
        if (!g || !rows) throw std::invalid_argument("null argument");
        if (j >= g->gs.m()) throw std::invalid_argument("gamma index out of range");
        const BitMatrix& M = g->gs.gammas[j];
        std::memcpy(rows, M.data(), size_t(M.rows()) * M.words() * 8);
    });
}

int mdg_gset_ranks(const mdg_gset* g, uint32_t* ranks) {
    return guard([&] {
        if (!g || !ranks) throw std::invalid_argument("null argument");
        std::memcpy(ranks, g->gs.ranks.data(), g->gs.ranks.size() * 4);
    });
}

int mdg_gset_perm(const mdg_gset* g, uint32_t* perm) {
    return guard([&] {
        if (!g || !perm) throw std::invalid_argument("null argument");
        std::memcpy(perm, g->gs.column_perm.data(), g->gs.column_perm.size() * 4);
    });
}

uint64_t mdg_gset_hash(const mdg_gset* g, uint32_t j) {
    if (!g || j >= g->gs.m()) return 0;
    return hash_rows(g->gs.gammas[j]);
}

int mdg_load_gset(mdg_ctx* ctx, const mdg_gset* g) {
    return guard([&] {
        if (!ctx || !g) throw std::invalid_argument("null argument");
        const GammaSet& gs = g->gs;
        uint32_t W = gs.gammas[0].words();
        std::vector<uint64_t> all(size_t(gs.m()) * gs.k() * W);
        for (uint32_t j = 0; j < gs.m(); ++j)
            std::memcpy(all.data() + size_t(j) * gs.k() * W, gs.gammas[j].data(), size_t(gs.k()) * W * 8);
        ctx->eng->load(gs.m(), gs.k(), gs.n(), all.data(), gs.ranks.data());
    });
}

uint32_t mdg_lower_bound(uint32_t m, uint32_t g, uint32_t k, uint32_t k_last) {
    return lower_bound(m, g, k, k_last);
}

uint32_t mdg_singleton_upper(uint32_t n, uint32_t k) {
    if (k < 1 || n < k) {
        g_err = "singleton_upper: need n >= k >= 1";
        return 0;
    }
    return singleton_upper(n, k);
}

// ---------------------------------------------------------------- loops
int mdg_bz_loop_cb(const mdg_gset* g, uint32_t lower, uint32_t upper, uint32_t level_cap,
                   mdg_round_fn fn, void* user, mdg_run** out) {
    return guard([&] {
        if (!g || !fn || !out) throw std::invalid_argument("null argument");
        auto t0 = std::chrono::steady_clock::now();
        auto run = std::make_unique<mdg_run>();
        RoundRunner runner = [&](uint32_t j, uint32_t c, RoundStats& rs) -> uint32_t {
            uint32_t w = UINT32_MAX;
            int rc = fn(user, j, c, rs.stop_at, &w);
            if (rc != 0) throw std::runtime_error("round callback failed with status " + std::to_string(rc));
            rs.combinations = binomial(g->gs.k(), c);
            return w;
        };
        Bounds b;
        b.lower = lower;
        b.upper = upper;
        run->er = run_bz_loop(g->gs, b, runner, level_cap);
        run->n = g->gs.n();
        run->k = g->gs.k();
        run->m = g->gs.m();
        run->k_last = g->gs.k_last;
        run->perm = g->gs.column_perm;
        run->level_cap = level_cap;
        run->algorithm = "callback";
        run->kernel = "callback";
        for (uint32_t j = 0; j < run->m; ++j) run->gamma_hash.push_back(hash_rows(g->gs.gammas[j]));
        run->wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = run.release();
    });
}

void mdg_config_default(mdg_config* cfg) {
    if (!cfg) return;
    cfg->trials = 10;
    cfg->seed = 0;
    cfg->level_cap = 0;
    cfg->kernel = MDG_KERNEL_TAB;
    cfg->want_witness = 1;
    cfg->exact_rounds = 0;
    cfg->gamma_search = MDG_GAMMA_HOST;
    cfg->split_min = 0;
    cfg->workers = 1;
}

int mdg_min_weight(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n, const mdg_config* cfg,
                   mdg_run** out) {
    return mdg_min_weight_dist(ctx, G, k, n, cfg, 0, 1, nullptr, nullptr, out);
}

int mdg_min_weight_dist(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n,
                        const mdg_config* cfg, uint32_t rank, uint32_t world,
                        mdg_reduce_fn reduce_min, void* user, mdg_run** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null out");
        if (world < 1 || rank >= world) throw std::invalid_argument("bad rank / world");
        if (world > 1 && !reduce_min) throw std::invalid_argument("multi-rank run needs a reducer");
        mdg_config c;
        mdg_config_default(&c);
        if (cfg) c = *cfg;
        if (c.trials < 1) throw std::invalid_argument("best_gamma_over_permutations: trials must be >= 1");
        std::unique_ptr<mdg_ctx> own;
        if (!ctx) {
            own = std::make_unique<mdg_ctx>();
            own->eng = std::make_unique<Engine>(0);
            ctx = own.get();
        }
        BitMatrix M = from_rows(G, k, n);
        *out = min_weight_device(*ctx->eng, M, c, rank, world, reduce_min, user).release();
    });
}

namespace {
// Workers of the batch front doors, kept between calls (spawning three threads per call cost
// ~0.1 ms of a 2 ms eight-code step). run(S, fn) runs fn(0) on the caller and fn(1..S-1) on pool
// threads and returns when all are done; a second batch call arriving meanwhile spawns its own
// threads instead of waiting.
class BatchPool {
public:
    static BatchPool& get() {
        static BatchPool p;
        return p;
    }
    void run(uint32_t S, const std::function<void(uint32_t)>& fn) {
        if (S <= 1) {
            fn(0);
            return;
        }
        std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
        if (!busy.owns_lock()) { // pool in use by another caller: plain threads
            std::vector<std::thread> th;
            for (uint32_t w = 1; w < S; ++w) th.emplace_back(fn, w);
            fn(0);
            for (auto& t : th) t.join();
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            while (workers_.size() + 1 < S) workers_.emplace_back([this, id = uint32_t(workers_.size() + 1)] { loop(id); });
            fn_ = &fn;
            want_ = S;
            pending_ = S - 1;
            ++epoch_;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    BatchPool() = default;
    ~BatchPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    void loop(uint32_t id) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(uint32_t)>* fn = nullptr;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || (epoch_ != seen && id < want_); });
                if (stop_) return;
                seen = epoch_;
                fn = fn_;
            }
            (*fn)(id);
            {
                std::lock_guard<std::mutex> lk(m_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::mutex busy_, m_;
    std::condition_variable cv_, done_;
    std::vector<std::thread> workers_;
    const std::function<void(uint32_t)>* fn_ = nullptr;
    uint32_t want_ = 0, pending_ = 0;
    uint64_t epoch_ = 0;
    bool stop_ = false;
};
} // namespace

int mdg_min_weight_batch(mdg_ctx* ctx, uint32_t count, const uint64_t* const* G, const uint32_t* k,
                         const uint32_t* n, const mdg_config* cfg, uint32_t streams,
                         mdg_run** out) {
    return guard([&] {
        if (!ctx || !out || (count && (!G || !k || !n))) throw std::invalid_argument("null argument");
        std::vector<mdg_config> cf(count);
        for (uint32_t i = 0; i < count; ++i) {
            if (!G[i]) throw std::invalid_argument("null matrix");
            out[i] = nullptr;
            mdg_config_default(&cf[i]);
            if (cfg) cf[i] = cfg[i];
            if (cf[i].trials < 1)
                throw std::invalid_argument("best_gamma_over_permutations: trials must be >= 1");
        }
        const uint32_t S = std::max(1u, std::min(streams ? streams : 4u, std::max(count, 1u)));
        const int dev = ctx->eng->device();
        while (ctx->extra.size() + 1 < S) ctx->extra.push_back(std::make_unique<Engine>(dev));
        std::vector<std::unique_ptr<mdg_run>> runs(count);
        std::vector<std::exception_ptr> errs(S);
        static const bool timing = std::getenv("MDG_TIMING") != nullptr;
        const auto t_batch = std::chrono::steady_clock::now();
        std::atomic<uint32_t> next{0};
        const std::function<void(uint32_t)> worker = [&](uint32_t w) {
            Engine& eng = w == 0 ? *ctx->eng : *ctx->extra[w - 1];
            try {
                for (uint32_t i; (i = next.fetch_add(1)) < count;) {
                    const auto ts = std::chrono::steady_clock::now();
                    BitMatrix M = from_rows(G[i], k[i], n[i]);
                    runs[i] = min_weight_device(eng, M, cf[i], 0, 1, nullptr, nullptr);
                    if (timing) {
                        auto us = [&](std::chrono::steady_clock::time_point x) {
                            return std::chrono::duration<double>(x - t_batch).count() * 1e6;
                        };
                        const double end = us(std::chrono::steady_clock::now());
                        std::fprintf(stderr, "[mdg batch] code %u worker %u start %.0f gamma %.0f loop %.0f end %.0f us\n",
                                     i, w, us(ts), runs[i]->gamma_s * 1e6, runs[i]->loop_s * 1e6, end);
                    }
                }
            } catch (...) {
                errs[w] = std::current_exception();
                next.store(count); // stop handing out codes
            }
        };
        BatchPool::get().run(S, worker);
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        for (uint32_t i = 0; i < count; ++i) out[i] = runs[i].release();
    });
}

int mdg_bz_loop_device_batch(mdg_ctx* const* ctxs, const mdg_gset* const* gs, uint32_t count,
                             const mdg_config* cfg, uint32_t streams, mdg_run** out) {
    return guard([&] {
        if (count && (!ctxs || !gs || !out)) throw std::invalid_argument("null argument");
        for (uint32_t i = 0; i < count; ++i) {
            if (!ctxs[i] || !gs[i]) throw std::invalid_argument("null context or Gamma set");
            for (uint32_t q = 0; q < i; ++q)
                if (ctxs[q] == ctxs[i]) throw std::invalid_argument("one context per code: contexts must be distinct");
            out[i] = nullptr;
        }
        mdg_config c;
        mdg_config_default(&c);
        if (cfg) c = *cfg;
        const uint32_t S = std::max(1u, std::min(streams ? streams : 4u, std::max(count, 1u)));
        std::vector<std::unique_ptr<mdg_run>> runs(count);
        std::vector<std::exception_ptr> errs(S);
        std::atomic<uint32_t> next{0};
        const std::function<void(uint32_t)> worker = [&](uint32_t w) {
            try {
                for (uint32_t i; (i = next.fetch_add(1)) < count;) {
                    auto t0 = std::chrono::steady_clock::now();
                    auto run = std::make_unique<mdg_run>();
                    run_device_loop(*ctxs[i]->eng, gs[i]->gs, c, 0, 1, nullptr, nullptr, *run);
                    run->wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                    runs[i] = std::move(run);
                }
            } catch (...) {
                errs[w] = std::current_exception();
                next.store(count);
            }
        };
        BatchPool::get().run(S, worker);
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        for (uint32_t i = 0; i < count; ++i) out[i] = runs[i].release();
    });
}

int mdg_bz_loop_device(mdg_ctx* ctx, const mdg_gset* g, const mdg_config* cfg, mdg_run** out) {
    return mdg_bz_loop_device_dist(ctx, g, cfg, 0, 1, nullptr, nullptr, out);
}

int mdg_bz_loop_device_dist(mdg_ctx* ctx, const mdg_gset* g, const mdg_config* cfg, uint32_t rank,
                            uint32_t world, mdg_reduce_fn reduce_min, void* user, mdg_run** out) {
    return guard([&] {
        if (!ctx || !g || !out) throw std::invalid_argument("null argument");
        if (world < 1 || rank >= world) throw std::invalid_argument("bad rank / world");
        if (world > 1 && !reduce_min) throw std::invalid_argument("multi-rank run needs a reducer");
        mdg_config c;
        mdg_config_default(&c);
        if (cfg) c = *cfg;
        auto t0 = std::chrono::steady_clock::now();
        auto run = std::make_unique<mdg_run>();
        run_device_loop(*ctx->eng, g->gs, c, rank, world, reduce_min, user, *run);
        run->wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = run.release();
    });
}

int mdg_timer_start(mdg_ctx* ctx) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null ctx");
        ctx->eng->timer_start();
    });
}

int mdg_timer_stop(mdg_ctx* ctx, double* ms) {
    return guard([&] {
        if (!ctx || !ms) throw std::invalid_argument("null argument");
        *ms = ctx->eng->timer_stop_ms();
    });
}

int mdg_ctx_counters(mdg_ctx* ctx, uint64_t* launches, uint64_t* h2d, uint64_t* d2h) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null ctx");
        Engine::Counters c = ctx->eng->counters();
        if (launches) *launches = c.launches;
        if (h2d) *h2d = c.h2d;
        if (d2h) *d2h = c.d2h;
    });
}

int mdg_device_info(mdg_ctx* ctx, int* sms, int* device) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null ctx");
        if (sms) *sms = ctx->eng->sm_count();
        if (device) *device = ctx->eng->device();
    });
}

int mdg_brute_force(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n, uint32_t brute_cap,
                    mdg_run** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null out");
        if (brute_cap < 1 || brute_cap > 63)
            throw std::invalid_argument("config: brute_cap must be in 1..63");
        auto t0 = std::chrono::steady_clock::now();
        std::unique_ptr<mdg_ctx> own;
        if (!ctx) {
            own = std::make_unique<mdg_ctx>();
            own->eng = std::make_unique<Engine>(0);
            ctx = own.get();
        }
        BitMatrix B = row_basis(from_rows(G, k, n));
        if (B.rows() > brute_cap)
            throw std::invalid_argument("brute force: k = " + std::to_string(B.rows()) + " exceeds cap " +
                                        std::to_string(brute_cap) + "; use a Brouwer-Zimmermann engine");
        Engine& eng = *ctx->eng;
        Engine::Counters c0 = eng.counters();
        Engine::BruteResult br = eng.brute_force(B.rows(), n, B.data());
        auto run = std::make_unique<mdg_run>();
        run->algorithm = "brute";
        run->kernel = "span";
        run->er.d = br.d;
        const uint64_t total = (uint64_t{1} << B.rows()) - 1;
        run->er.stats.combinations = total;
        run->er.stats.row_additions = total; // serial Gray walk: one XOR per codeword
        run->er.stats.evaluated = br.evaluated;
        run->er.stats.device_ms = br.ms;
        run->n = n;
        run->k = B.rows();
        run->m = 0;
        run->k_last = 0;
        std::vector<uint64_t> w(B.words(), 0);
        for (uint32_t r : br.idx)
            for (uint32_t i = 0; i < B.words(); ++i) w[i] ^= B.row(r)[i];
        BitMatrix S(B.rows() + 1, n);
        std::memcpy(S.data(), B.data(), size_t(B.rows()) * B.words() * 8);
        std::memcpy(S.row(B.rows()), w.data(), B.words() * 8);
        run->witness = w;
        run->witness_idx = br.idx;
        run->witness_ok = weight_of(w) == br.d && !br.idx.empty() && rank_of(S) == B.rows();
        run->perm.resize(n);
        for (uint32_t i = 0; i < n; ++i) run->perm[i] = i;
        Engine::Counters c1 = eng.counters();
        run->cnt.launches = c1.launches - c0.launches;
        run->cnt.h2d = c1.h2d - c0.h2d;
        run->cnt.d2h = c1.d2h - c0.d2h;
        run->loop_s = br.ms * 1e-3;
        run->wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = run.release();
    });
}

int mdg_group_create(uint32_t world, mdg_group** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null out");
        auto g = std::make_unique<mdg_group>();
        g->g = make_exchange_group(world);
        *out = g.release();
    });
}

void mdg_group_free(mdg_group* g) { delete g; }

int mdg_group_attach(mdg_ctx* ctx, mdg_group* g, uint32_t rank) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null ctx");
        ctx->eng->group_attach(g ? g->g : nullptr, rank);
    });
}

int mdg_group_reduce_min(void*, uint64_t*, uint32_t) {
    g_err = "mdg_group_reduce_min is a marker for the device-side group exchange, not a host reducer";
    return MDG_EINVAL;
}

int mdg_min_weight_multi(mdg_ctx* const* ctxs, uint32_t world, const uint64_t* G, uint32_t k,
                         uint32_t n, const mdg_config* cfg, mdg_run** out) {
    return guard([&] {
        if (!ctxs || !G || !out) throw std::invalid_argument("null argument");
        if (world < 1) throw std::invalid_argument("bad rank / world");
        for (uint32_t r = 0; r < world; ++r) {
            if (!ctxs[r]) throw std::invalid_argument("null ctx");
            for (uint32_t q = 0; q < r; ++q)
                if (ctxs[q] == ctxs[r]) throw std::invalid_argument("a context appears twice");
            out[r] = nullptr;
        }
        mdg_config c;
        mdg_config_default(&c);
        if (cfg) c = *cfg;
        if (c.trials < 1) throw std::invalid_argument("best_gamma_over_permutations: trials must be >= 1");
        const BitMatrix M = from_rows(G, k, n);
        auto group = make_exchange_group(world);
        int plan_sms = ctxs[0]->eng->sm_count();
        for (uint32_t r = 0; r < world; ++r) plan_sms = std::min(plan_sms, ctxs[r]->eng->sm_count());
        std::vector<int> old_sms(world);
        for (uint32_t r = 0; r < world; ++r) { // one tile cut of every split round on all ranks
            ctxs[r]->eng->group_attach(group, r);
            old_sms[r] = ctxs[r]->eng->plan_sms();
            ctxs[r]->eng->set_plan_sms(plan_sms);
        }
        std::vector<std::unique_ptr<mdg_run>> runs(world);
        std::vector<std::exception_ptr> errs(world);
        auto member = [&](uint32_t r) {
            try {
                runs[r] = min_weight_device(*ctxs[r]->eng, M, c, r, world, &mdg_group_reduce_min, nullptr);
            } catch (const std::exception& e) {
                errs[r] = std::current_exception();
                abort_exchange_group(*group, "rank " + std::to_string(r) + ": " + e.what());
            } catch (...) {
                errs[r] = std::current_exception();
                abort_exchange_group(*group, "rank " + std::to_string(r) + " failed");
            }
        };
        std::vector<std::thread> th;
        for (uint32_t r = 1; r < world; ++r) th.emplace_back(member, r);
        member(0);
        for (auto& t : th) t.join();
        for (uint32_t r = 0; r < world; ++r) {
            ctxs[r]->eng->group_attach(nullptr, 0);
            ctxs[r]->eng->set_plan_sms(old_sms[r]);
        }
        // the first real failure is the cause; the others' "aborted" errors follow from it
        for (uint32_t r = 0; r < world; ++r)
            if (errs[r]) {
                try {
                    std::rethrow_exception(errs[r]);
                } catch (const std::runtime_error& e) {
                    if (std::string(e.what()).find("exchange group aborted") != std::string::npos) continue;
                    throw;
                }
            }
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        for (uint32_t r = 0; r < world; ++r) out[r] = runs[r].release();
    });
}

int mdg_nccl_unique_id(uint8_t id[128]) {
    return guard([&] { Engine::nccl_unique_id(id); });
}

int mdg_nccl_init(mdg_ctx* ctx, const uint8_t id[128], uint32_t rank, uint32_t world) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null ctx");
        ctx->eng->nccl_init(id, rank, world);
    });
}

int mdg_nccl_reduce_min(void* ctx, uint64_t* keys, uint32_t count) {
    return guard([&] {
        if (!ctx) throw std::invalid_argument("null ctx");
        static_cast<mdg_ctx*>(ctx)->eng->nccl_reduce_min(keys, count);
    });
}

// ----------------------------------------------------------- run results
int mdg_run_info_get(const mdg_run* r, mdg_run_info* info) {
    return guard([&] {
        if (!r || !info) throw std::invalid_argument("null argument");
        std::memset(info, 0, sizeof *info);
        const auto& st = r->er.stats;
        info->d = r->er.d;
        info->capped = r->er.capped ? 1 : 0;
        info->n = r->n;
        info->k = r->k;
        info->m = r->m;
        info->k_last = r->k_last;
        info->g_final = st.g_final;
        info->n_rounds = uint32_t(st.rounds.size());
        info->n_levels = uint32_t(st.levels.size());
        info->witness_ok = r->witness_ok ? 1 : 0;
        info->combinations = st.combinations;
        info->evaluated = st.evaluated;
        info->row_additions = st.row_additions;
        info->wall_seconds = r->wall;
        info->device_seconds = st.device_ms * 1e-3;
        info->gamma_seconds = r->gamma_s;
        info->loop_seconds = r->loop_s;
        info->launches = r->cnt.launches;
        info->h2d_bytes = r->cnt.h2d;
        info->d2h_bytes = r->cnt.d2h;
    });
}

int mdg_run_rounds(const mdg_run* r, mdg_round_rec* out) {
    return guard([&] {
        if (!r || !out) throw std::invalid_argument("null argument");
        for (size_t i = 0; i < r->er.stats.rounds.size(); ++i) {
            const auto& x = r->er.stats.rounds[i];
            out[i] = {x.c, x.j, x.w, x.U_after, x.bounded};
        }
    });
}

int mdg_run_levels(const mdg_run* r, mdg_level_rec* out) {
    return guard([&] {
        if (!r || !out) throw std::invalid_argument("null argument");
        for (size_t i = 0; i < r->er.stats.levels.size(); ++i) {
            const auto& x = r->er.stats.levels[i];
            out[i] = {x.c, x.L_after, x.U_after, 0};
        }
    });
}

int mdg_run_witness(const mdg_run* r, uint64_t* row) {
    return guard([&] {
        if (!r || !row) throw std::invalid_argument("null argument");
        if (r->witness.empty()) throw std::invalid_argument("run has no witness");
        std::memcpy(row, r->witness.data(), r->witness.size() * 8);
    });
}

int mdg_run_round_perf(const mdg_run* r, uint64_t* evaluated, double* device_ms) {
    return guard([&] {
        if (!r) throw std::invalid_argument("null run");
        const auto& pg = r->er.stats.per_g;
        for (size_t i = 0; i < pg.size(); ++i) {
            if (evaluated) evaluated[i] = pg[i].evaluated;
            if (device_ms) device_ms[i] = pg[i].device_ms;
        }
    });
}

int mdg_run_perm(const mdg_run* r, uint32_t* perm) {
    return guard([&] {
        if (!r || !perm) throw std::invalid_argument("null argument");
        std::memcpy(perm, r->perm.data(), r->perm.size() * 4);
    });
}

uint64_t mdg_run_gamma_hash(const mdg_run* r, uint32_t j) {
    if (!r || j >= r->gamma_hash.size()) return 0;
    return r->gamma_hash[j];
}

long mdg_run_json(const mdg_run* r, char* buf, size_t cap) {
    if (!r) {
        g_err = "null run";
        return MDG_EINVAL;
    }
    return copy_out(json_of(*r), buf, cap);
}

void mdg_run_free(mdg_run* r) { delete r; }

// -------------------------------------------------------------- misc I/O
int mdg_parse_matrix(const char* text, uint32_t* k, uint32_t* n, uint64_t* rows_out) {
    return guard([&] {
        if (!text) throw std::invalid_argument("null text");
        BitMatrix M = parse_matrix(text);
        if (k) *k = M.rows();
        if (n) *n = M.cols();
        if (rows_out) std::memcpy(rows_out, M.data(), size_t(M.rows()) * M.words() * 8);
    });
}

long mdg_serialize_matrix(const uint64_t* rows, uint32_t k, uint32_t n, char* buf, size_t cap) {
    std::string s;
    int rc = guard([&] { s = serialize_matrix(from_rows(rows, k, n)); });
    if (rc) return rc;
    return copy_out(s, buf, cap);
}

int mdg_gen_matrix(uint32_t n, uint32_t k, uint64_t seed, int identity, uint64_t* rows) {
    return guard([&] {
        if (!rows) throw std::invalid_argument("null out");
        BitMatrix M = gen_matrix(n, k, seed, identity != 0);
        std::memcpy(rows, M.data(), size_t(k) * M.words() * 8);
    });
}

uint32_t mdg_rank(const uint64_t* rows, uint32_t k, uint32_t n) {
    uint32_t r = 0;
    guard([&] { r = rank_of(from_rows(rows, k, n)); });
    return r;
}

uint64_t mdg_hash_rows(const uint64_t* rows, uint32_t k, uint32_t n) {
    uint64_t h = 0;
    guard([&] { h = hash_rows(from_rows(rows, k, n)); });
    return h;
}

int mdg_binomial(uint32_t p, uint32_t q, uint64_t* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null out");
        *out = binomial(p, q);
    });
}

int mdg_rd_unrank(uint32_t c, uint64_t rank, uint32_t* idx) {
    return guard([&] {
        if (!idx || c < 1) throw std::invalid_argument("bad argument");
        rd_unrank(c, rank, idx);
    });
}

uint64_t mdg_rd_rank(uint32_t c, const uint32_t* idx) {
    uint64_t r = 0;
    guard([&] { r = rd_rank(c, idx); });
    return r;
}

} // extern "C"
