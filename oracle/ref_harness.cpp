// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Harness around the UNMODIFIED reference library (compiled from the sources
// under /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It
// adds only what the reference lacks for parity checking:
//   * a recording RoundRunner plugged into the reference's own level loop
//     `md::run_bz_loop` (proj/src/engines.cpp:447-476) to capture the per-round
//     minima; the per-level (L, U) trace is replayed from those minima with the
//     reference's `md::lower_bound` (proj/src/gamma.cpp:96-100);
//   * a level cap, implemented as a sentinel exception thrown from the runner
//     (run_bz_loop has no cap parameter, engines.cpp:454);
//   * the config input generator of SURVEY.md §8d with std::mt19937_64;
//   * the config-5 weight histogram over reference primitives
//     (CombinationCursor enumeration.cpp:52-63, combine_rows f2core.cpp:45-57,
//     weight f2core.cpp:26-32), cross-checked against round_stack.
// Only tests/, bench.py's reference arm and oracle/make_golden.py run it.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "mindist/engines.hpp"
#include "mindist/enumeration.hpp"
#include "mindist/f2core.hpp"
#include "mindist/gamma.hpp"
#include "mindist/io.hpp"
#include "mindist/parallel.hpp"
#include "mindist/util.hpp"

using namespace md;

namespace {

struct LevelCapReached {};

// FNV-1a 64 over the row's bits packed LSB-first into u64 words, each word
// serialized little-endian (the convention shared with the product's hashes).
uint64_t hash_matrix(const BitMatrix& m) {
    uint64_t h = 1469598103934665603ull;
    for (uint32_t r = 0; r < m.rows(); ++r) {
        const BitVector& v = m.row(r);
        uint32_t w32 = v.word_count();
        for (uint32_t i = 0; i < (w32 + 1) / 2; ++i) {
            uint64_t lo = v.words()[2 * i];
            uint64_t hi = (2 * i + 1 < w32) ? v.words()[2 * i + 1] : 0;
            uint64_t w = lo | (hi << 32);
            for (int b = 0; b < 8; ++b) {
                h ^= (w >> (8 * b)) & 0xff;
                h *= 1099511628211ull;
            }
        }
    }
    return h;
}

std::string row_hex(const BitVector& v) {
    // bits LSB-first in u64 words, words printed as 16 hex digits each, word 0 first
    std::string out;
    char buf[17];
    uint32_t w32 = v.word_count();
    for (uint32_t i = 0; i < (w32 + 1) / 2; ++i) {
        uint64_t lo = v.words()[2 * i];
        uint64_t hi = (2 * i + 1 < w32) ? v.words()[2 * i + 1] : 0;
        std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)(lo | (hi << 32)));
        out += buf;
    }
    return out;
}

struct RoundRec { uint32_t c, j, w; };

struct TraceOut {
    GammaSet gs;
    std::vector<RoundRec> rounds;
    uint32_t d = 0;
    bool capped = false;
    uint64_t combinations = 0;
    uint64_t row_additions = 0;
    double seconds = 0;
};

// Reference engines behind the recording runner. engine: saved | stack | scheduled
TraceOut trace_run(const BitMatrix& G, uint32_t trials, uint64_t seed, const std::string& engine,
                   uint32_t s, uint32_t workers, uint32_t level_cap) {
    TraceOut out;
    auto t0 = std::chrono::steady_clock::now();
    BitMatrix B = row_basis(G);
    out.gs = best_gamma_over_permutations(B, trials, seed);
    const GammaSet& gs = out.gs;
    Bounds bounds;
    bounds.lower = 1;
    bounds.upper = singleton_upper(B.cols(), B.rows());

    EngineConfig ecfg;
    ecfg.s = s;
    ecfg.workers = workers;
    ecfg.memory_cap_bytes = uint64_t{64} << 30;
    std::vector<SavedAdditions> tables;
    if (engine == "saved") {
        tables.reserve(gs.m());
        for (const auto& g : gs.gammas) tables.emplace_back(g, s, ecfg.memory_cap_bytes);
    }
    ScheduleConfig scfg;
    scfg.mode = ScheduleMode::dynamic;
    scfg.workers = workers;
    scfg.prefix_param = 3;

    RoundRunner runner = [&](uint32_t j, uint32_t g, RoundStats& rs) -> uint32_t {
        if (level_cap && g > level_cap) throw LevelCapReached{};
        uint32_t w;
        if (engine == "saved")
            w = workers > 1 ? round_saved_parallel(tables[j], g, workers, rs)
                            : round_saved(tables[j], g, rs);
        else if (engine == "stack")
            w = round_stack(gs.gammas[j], g, rs);
        else if (engine == "scheduled")
            w = scheduled_round(gs.gammas[j], g, scfg, rs);
        else
            throw std::invalid_argument("unknown engine " + engine);
        out.rounds.push_back({g, j, w});
        out.combinations += rs.combinations;
        out.row_additions += rs.additions;
        return w;
    };
    try {
        EngineResult er = run_bz_loop(gs, bounds, runner);
        out.d = er.d;
    } catch (const LevelCapReached&) {
        out.capped = true;
    }
    out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

std::string trace_json(const BitMatrix& G, const TraceOut& t, uint32_t trials, uint64_t seed,
                       const std::string& engine, uint32_t workers, uint32_t level_cap,
                       bool with_rows) {
    const GammaSet& gs = t.gs;
    uint32_t k = gs.k(), m = gs.m();
    // Replay run_bz_loop (engines.cpp:447-476) over the recorded minima to
    // obtain the per-level (L, U) trace; assert it consumes exactly them.
    uint32_t U = singleton_upper(gs.n(), k);
    uint32_t L = 1;
    bool done = U <= L;
    size_t ri = 0;
    std::ostringstream rounds, levels;
    uint32_t g_final = 0;
    bool first_r = true, first_l = true;
    for (uint32_t g = 1; !done && g <= k; ++g) {
        bool level_complete = true;
        for (uint32_t j = 0; j < m; ++j) {
            if (U <= L) { done = true; break; }
            if (ri >= t.rounds.size()) { level_complete = false; break; }
            const RoundRec& r = t.rounds[ri++];
            if (r.c != g || r.j != j) throw std::logic_error("trace replay mismatch");
            if (r.w < U) U = r.w;
            g_final = g;
            rounds << (first_r ? "" : ",") << "[" << r.c << "," << r.j << "," << r.w << "," << U << "]";
            first_r = false;
        }
        if (done || !level_complete) break;
        uint32_t nl = lower_bound(m, g, k, gs.k_last);
        if (nl > L) L = nl;
        levels << (first_l ? "" : ",") << "[" << g << "," << L << "," << U << "]";
        first_l = false;
        if (L >= U) done = true;
    }
    if (ri != t.rounds.size()) throw std::logic_error("trace replay left rounds unconsumed");
    if (!t.capped && U != t.d) throw std::logic_error("trace replay disagrees with run_bz_loop");

    std::ostringstream o;
    o << "{\"n\":" << G.cols() << ",\"k\":" << gs.k() << ",\"trials\":" << trials
      << ",\"seed\":" << seed << ",\"engine\":\"" << engine << "\",\"workers\":" << workers
      << ",\"level_cap\":" << level_cap << ",\"capped\":" << (t.capped ? "true" : "false")
      << ",\"d\":";
    if (t.capped) o << "null"; else o << t.d;
    o << ",\"U_final\":" << U << ",\"L_final\":" << L << ",\"m\":" << m << ",\"k_last\":" << gs.k_last
      << ",\"g_final\":" << g_final << ",\"ranks\":[";
    for (uint32_t j = 0; j < m; ++j) o << (j ? "," : "") << gs.ranks[j];
    o << "],\"column_perm\":[";
    for (size_t j = 0; j < gs.column_perm.size(); ++j) o << (j ? "," : "") << gs.column_perm[j];
    o << "],\"gamma_hash\":[";
    for (uint32_t j = 0; j < m; ++j) {
        char buf[32];
        std::snprintf(buf, sizeof buf, "\"%016llx\"", (unsigned long long)hash_matrix(gs.gammas[j]));
        o << (j ? "," : "") << buf;
    }
    o << "]";
    if (with_rows) {
        o << ",\"gammas\":[";
        for (uint32_t j = 0; j < m; ++j) {
            o << (j ? "," : "") << "[";
            for (uint32_t r = 0; r < k; ++r)
                o << (r ? "," : "") << "\"" << row_hex(gs.gammas[j].row(r)) << "\"";
            o << "]";
        }
        o << "]";
    }
    o << ",\"rounds\":[" << rounds.str() << "],\"levels\":[" << levels.str() << "]"
      << ",\"combinations\":" << t.combinations << ",\"row_additions\":" << t.row_additions
      << ",\"wall_seconds\":" << t.seconds << "}";
    return o.str();
}

// SURVEY.md §8d input convention: std::mt19937_64(seed); fill A (k x (n-k),
// or the whole k x n matrix when identity=false) row-major with bit = draw & 1.
BitMatrix gen_matrix(uint32_t n, uint32_t k, uint64_t seed, bool identity) {
    std::mt19937_64 eng(seed);
    BitMatrix G(k, n);
    uint32_t off = identity ? k : 0;
    if (identity)
        for (uint32_t r = 0; r < k; ++r) G.set(r, r, true);
    for (uint32_t r = 0; r < k; ++r)
        for (uint32_t c = off; c < n; ++c)
            if (eng() & 1) G.set(r, c, true);
    return G;
}

std::string hist_json(const BitMatrix& M, uint32_t cmax) {
    std::ostringstream o;
    o << "{\"n\":" << M.cols() << ",\"k\":" << M.rows() << ",\"levels\":[";
    for (uint32_t c = 1; c <= cmax; ++c) {
        std::vector<uint64_t> hist(M.cols() + 1, 0);
        uint32_t best = UINT32_MAX;
        uint64_t count = 0;
        auto cur = CombinationCursor::first(M.rows(), c, CombOrder::lex);
        do {
            uint32_t w = weight(combine_rows(M, cur.current()));
            hist[w] += 1;
            if (w < best) best = w;
            ++count;
        } while (cur.next());
        RoundStats rs;
        uint32_t stack_min = round_stack(M, c, rs);
        if (stack_min != best || rs.combinations != count)
            throw std::logic_error("histogram restatement disagrees with round_stack");
        o << (c > 1 ? "," : "") << "{\"c\":" << c << ",\"min\":" << best << ",\"count\":" << count
          << ",\"hist\":[";
        for (size_t w = 0; w < hist.size(); ++w) o << (w ? "," : "") << hist[w];
        o << "]}";
    }
    o << "]}";
    return o.str();
}

std::string arg(int argc, char** argv, const char* name, const char* dflt) {
    for (int i = 1; i + 1 < argc; ++i)
        if (std::strcmp(argv[i], name) == 0) return argv[i + 1];
    return dflt;
}

} // namespace

// ------------------------------------------------------------------ C ABI
// Used from Python by tests/ and bench.py --impl reference (ctypes).
extern "C" {

// Full trace run over a matrix given in the reference text format.
// Returns the number of bytes written (excluding NUL), or -1 on error
// (message in out). engine: "saved" | "stack" | "scheduled".
long mdref_trace(const char* matrix_text, uint32_t trials, uint64_t seed, const char* engine,
                 uint32_t s, uint32_t workers, uint32_t level_cap, int with_rows, char* out,
                 size_t cap) {
    try {
        std::istringstream in(matrix_text);
        BitMatrix G = parse_matrix(in);
        TraceOut t = trace_run(G, trials, seed, engine, s, workers, level_cap);
        std::string js = trace_json(G, t, trials, seed, engine, workers, level_cap, with_rows != 0);
        if (js.size() + 1 > cap) return -2;
        std::memcpy(out, js.c_str(), js.size() + 1);
        return static_cast<long>(js.size());
    } catch (const std::exception& e) {
        std::snprintf(out, cap, "%s", e.what());
        return -1;
    }
}

// One reference round over an arbitrary k x n matrix (rows LSB-first u64
// words, W = ceil(n/64) per row). engine: "stack" | "saved" | "saved_parallel"
// | "scheduled". Returns the minimum; *combos gets RoundStats.combinations.
long mdref_round(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t c, const char* engine,
                 uint32_t s, uint32_t workers, uint64_t* combos) {
    try {
        BitMatrix M(k, n);
        uint32_t W = (n + 63) / 64;
        for (uint32_t r = 0; r < k; ++r)
            for (uint32_t b = 0; b < n; ++b)
                if ((rows[r * W + b / 64] >> (b % 64)) & 1) M.set(r, b, true);
        RoundStats rs;
        uint32_t w;
        std::string e(engine);
        if (e == "stack") {
            w = round_stack(M, c, rs);
        } else if (e == "saved" || e == "saved_parallel") {
            SavedAdditions sa(M, s, uint64_t{64} << 30);
            w = e == "saved" ? round_saved(sa, c, rs) : round_saved_parallel(sa, c, workers, rs);
        } else if (e == "scheduled") {
            ScheduleConfig scfg;
            scfg.mode = ScheduleMode::dynamic;
            scfg.workers = workers;
            scfg.prefix_param = 3;
            w = scheduled_round(M, c, scfg, rs);
        } else {
            return -1;
        }
        if (combos) *combos = rs.combinations;
        return static_cast<long>(w);
    } catch (const std::exception&) {
        return -1;
    }
}

// Generate a config matrix and serialize it in the reference
// text format (io.cpp:81-88). Returns bytes written or -1.
long mdref_gen(uint32_t n, uint32_t k, uint64_t seed, int identity, char* out, size_t cap) {
    std::string s = serialize_matrix(gen_matrix(n, k, seed, identity != 0));
    if (s.size() + 1 > cap) return -1;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<long>(s.size());
}

// random_full_rank_matrix (gamma.cpp:108-121) seeded as in the reference's
// tests (test_engines.cpp:30-33): SplitMix64(seed), then the matrix.
long mdref_random_full_rank(uint32_t n, uint32_t k, uint64_t seed, char* out, size_t cap) {
    try {
        SplitMix64 rng(seed);
        std::string s = serialize_matrix(random_full_rank_matrix(n, k, rng));
        if (s.size() + 1 > cap) return -1;
        std::memcpy(out, s.c_str(), s.size() + 1);
        return static_cast<long>(s.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// seeded_code of acceptance_main.cpp:44-53 (criterion 1's 200 random codes).
long mdref_seeded_code(uint64_t seed, uint32_t n_lo, uint32_t n_span, uint32_t k_cap, char* out,
                       size_t cap) {
    try {
        SplitMix64 rng(seed);
        uint32_t n = n_lo + static_cast<uint32_t>(rng.next() % n_span);
        uint32_t k_max = std::min(k_cap, n - 1);
        uint32_t k = 4 + static_cast<uint32_t>(rng.next() % (k_max - 3));
        std::string s = serialize_matrix(random_full_rank_matrix(n, k, rng));
        if (s.size() + 1 > cap) return -1;
        std::memcpy(out, s.c_str(), s.size() + 1);
        return static_cast<long>(s.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// min_weight (engines.cpp:617-648) with a named algorithm; returns d or -1.
long mdref_min_weight(const char* matrix_text, const char* algorithm, uint32_t trials,
                      uint64_t seed, uint32_t workers) {
    try {
        std::istringstream in(matrix_text);
        BitMatrix G = parse_matrix(in);
        EngineConfig cfg;
        cfg.algorithm = algorithm_from_name(algorithm);
        cfg.permutation_trials = trials;
        cfg.seed = seed;
        cfg.workers = workers;
        return static_cast<long>(min_weight(G, cfg).d);
    } catch (const std::exception&) {
        return -1;
    }
}

} // extern "C"

// -------------------------------------------------------------------- CLI
// mdref gen --n N --k K --seed S [--plain]         -> matrix text
// mdref trace FILE --trials T --seed S --engine E --s S --workers W --cap C [--rows]
// mdref hist FILE --cmax C
int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: mdref gen|trace|hist ...\n";
        return 2;
    }
    try {
        std::string cmd = argv[1];
        if (cmd == "gen") {
            uint32_t n = std::stoul(arg(argc, argv, "--n", "0"));
            uint32_t k = std::stoul(arg(argc, argv, "--k", "0"));
            uint64_t seed = std::stoull(arg(argc, argv, "--seed", "0"));
            bool plain = false;
            for (int i = 2; i < argc; ++i) plain |= std::strcmp(argv[i], "--plain") == 0;
            std::cout << serialize_matrix(gen_matrix(n, k, seed, !plain));
            return 0;
        }
        if (argc < 3) return 2;
        BitMatrix G = parse_matrix_file(argv[2]);
        if (cmd == "trace") {
            uint32_t trials = std::stoul(arg(argc, argv, "--trials", "10"));
            uint64_t seed = std::stoull(arg(argc, argv, "--seed", "0"));
            std::string engine = arg(argc, argv, "--engine", "saved");
            uint32_t s = std::stoul(arg(argc, argv, "--s", "5"));
            uint32_t workers = std::stoul(arg(argc, argv, "--workers", "1"));
            uint32_t cap = std::stoul(arg(argc, argv, "--cap", "0"));
            bool rows = false;
            for (int i = 3; i < argc; ++i) rows |= std::strcmp(argv[i], "--rows") == 0;
            TraceOut t = trace_run(G, trials, seed, engine, s, workers, cap);
            std::cout << trace_json(G, t, trials, seed, engine, workers, cap, rows) << "\n";
            return 0;
        }
        if (cmd == "hist") {
            uint32_t cmax = std::stoul(arg(argc, argv, "--cmax", "5"));
            std::cout << hist_json(G, cmax) << "\n";
            return 0;
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 2;
}
