// TEST BINARY — the reference-side binding of INTEGRATION.md §1 compiled literally against the
// UNMODIFIED reference library (oracle/_ref/v3/*.o, built from /root/reference/proj/src by
// oracle/Makefile) and the product's C ABI (paper_1911_08963_b200/lib/libmdg.so).
//
// The GPU RoundRunner and bz_gpu below are the maintainer's patch of INTEGRATION.md §1; the
// only part of that patch not reproduced is the registry edit (a new Algorithm::gpu enum value
// and its `case` in min_weight's dispatch, engines.cpp:635-642), which needs the reference's
// sources to change. main() does what that dispatch would: min_weight's own steps
// (engines.cpp:617-648 -- row_basis, best_gamma_over_permutations, singleton_upper) and then
// bz_gpu, i.e. the REFERENCE's run_bz_loop (engines.cpp:447-476) driving mdg_round on the GPU.
//
// usage: bz_gpu FILE --seed S [--trials T] [--cap C]  -> one JSON line:
//   {"d":..,"g_final":..,"m":..,"k_last":..,"rounds":[[c,j,w,U_after],...],"combinations":..}
// (--cap C: the runner throws past level C, as oracle/ref_harness.cpp does)
#include <cstdint>
#include <cstring>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mdg.h"
#include "mindist/engines.hpp"
#include "mindist/f2core.hpp"
#include "mindist/gamma.hpp"
#include "mindist/io.hpp"

namespace md {

// ---- the GPU engine behind RoundRunner (engines.hpp:151) ----
RoundRunner gpu_round_runner(mdg_ctx* ctx) {
    return [ctx](uint32_t j, uint32_t g, RoundStats& rs) -> uint32_t {
        mdg_round_out out;
        int rc = mdg_round(ctx, j, g, /*stop_at=*/0, &out); // exact round minimum
        if (rc == MDG_EINVAL || rc == MDG_EOVERFLOW) throw std::invalid_argument(mdg_last_error());
        if (rc != MDG_OK) throw std::runtime_error(mdg_last_error());
        rs.combinations = out.combinations; // C(k, g), as every reference round
        rs.additions = out.evaluated;
        return out.min_weight;
    };
}

// upload: m Gammas, k rows of W = ceil(n/64) u64 words (LSB-first = BitVector's bit order)
mdg_ctx* gpu_open_with(const GammaSet& gs) {
    mdg_ctx* ctx = nullptr;
    if (mdg_open(/*device=*/0, &ctx) != MDG_OK) throw std::runtime_error(mdg_last_error());
    const uint32_t m = gs.m(), k = gs.k(), n = gs.n(), W = (n + 63) / 64;
    std::vector<uint64_t> rows(size_t(m) * k * W, 0);
    for (uint32_t j = 0; j < m; ++j)
        for (uint32_t r = 0; r < k; ++r)
            for (uint32_t i = 0; i < gs.gammas[j].row(r).word_count(); ++i)
                rows[(size_t(j) * k + r) * W + i / 2] |=
                    uint64_t(gs.gammas[j].row(r).words()[i]) << (32 * (i % 2));
    if (mdg_load_gammas(ctx, m, k, n, rows.data(), gs.ranks.data()) != MDG_OK) {
        std::string e = mdg_last_error();
        mdg_close(ctx);
        throw std::invalid_argument(e);
    }
    return ctx;
}

EngineResult bz_gpu(const GammaSet& gs, Bounds bounds, const EngineConfig& config) {
    config.validate();
    mdg_ctx* ctx = gpu_open_with(gs);
    try {
        EngineResult er = run_bz_loop(gs, bounds, gpu_round_runner(ctx));
        mdg_close(ctx);
        return er;
    } catch (...) {
        mdg_close(ctx);
        throw;
    }
}
// min_weight's dispatch switch (engines.cpp:635-642) would gain:
//     case Algorithm::gpu: er = bz_gpu(gs, bounds, config); break;

} // namespace md

namespace {
struct CapReached {};

std::string arg(int argc, char** argv, const char* name, const char* dflt) {
    for (int i = 1; i + 1 < argc; ++i)
        if (std::strcmp(argv[i], name) == 0) return argv[i + 1];
    return dflt;
}
} // namespace

int main(int argc, char** argv) {
    using namespace md;
    if (argc < 2) {
        std::cerr << "usage: bz_gpu FILE --seed S [--trials T] [--cap C]\n";
        return 2;
    }
    try {
        BitMatrix G = parse_matrix_file(argv[1]);
        EngineConfig cfg;
        cfg.seed = std::stoull(arg(argc, argv, "--seed", "0"));
        cfg.permutation_trials = std::stoul(arg(argc, argv, "--trials", "10"));
        const uint32_t cap = std::stoul(arg(argc, argv, "--cap", "0"));
        // min_weight (engines.cpp:617-648) up to its dispatch
        BitMatrix B = row_basis(G);
        GammaSet gs = best_gamma_over_permutations(B, cfg.permutation_trials, cfg.seed);
        Bounds bounds;
        bounds.lower = 1;
        bounds.upper = singleton_upper(B.cols(), B.rows());
        // bz_gpu with a recording wrapper around the same GPU runner (the trace is not part of
        // EngineResult); the plain bz_gpu result must agree with it
        mdg_ctx* ctx = gpu_open_with(gs);
        RoundRunner gpu = gpu_round_runner(ctx);
        std::ostringstream rounds;
        uint32_t U = bounds.upper;
        bool first = true, capped = false;
        RoundRunner recording = [&](uint32_t j, uint32_t g, RoundStats& rs) -> uint32_t {
            if (cap && g > cap) throw CapReached{};
            uint32_t w = gpu(j, g, rs);
            if (w < U) U = w;
            rounds << (first ? "" : ",") << "[" << g << "," << j << "," << w << "," << U << "]";
            first = false;
            return w;
        };
        EngineResult er;
        try {
            er = run_bz_loop(gs, bounds, recording);
        } catch (const CapReached&) {
            capped = true;
        }
        mdg_close(ctx);
        if (!capped) {
            EngineResult plain = bz_gpu(gs, bounds, cfg);
            if (plain.d != er.d || plain.stats.g_final != er.stats.g_final ||
                plain.stats.combinations != er.stats.combinations)
                throw std::logic_error("bz_gpu disagrees with the recorded run");
        }
        std::cout << "{\"d\":" << (capped ? U : er.d) << ",\"capped\":" << (capped ? "true" : "false")
                  << ",\"g_final\":" << (capped ? cap : er.stats.g_final) << ",\"m\":" << gs.m()
                  << ",\"k_last\":" << gs.k_last << ",\"rounds\":[" << rounds.str()
                  << "],\"combinations\":" << er.stats.combinations << "}\n";
        return 0;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return 1;
    }
}
