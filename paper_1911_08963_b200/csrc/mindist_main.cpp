// `mindist` command line for the GPU engine — the reference's `mindist
// mindist <file> --algorithm ... --seed S --trials T` (cli.cpp:69-112,
// 257-278) with `--algorithm gpu`, emitting the reference's JSON record
// (cli.cpp:223-238) plus the new keys (witness, trace, levels, capped, ...).
// Exit codes as the reference: 0 ok, 1 internal error, 2 invalid input or
// config (cli.cpp:198-219).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

#include "mdg.h"
#include "mdg.hpp"

namespace {

int usage() {
    std::cerr << "usage:\n"
                 "  mindist mindist FILE [FILE ...] [--algorithm gpu|brute] [--kernel tab|rd] [--trials T]\n"
                 "                       [--seed S] [--level-cap C] [--device D] [--devices D0,D1,..]\n"
                 "                       [--split-min N] [--exact-rounds]\n"
                 "                       [--gamma-search host|gpu] [--pretty]\n"
                 "    accepted for the reference's command line (cli.cpp:264-277), validated as there\n"
                 "    and not used by the GPU engine: --algorithm basic|optimized|stack|saved|\n"
                 "    saved_unrolled (run the GPU engine: same d and trace), --s 1..8, --unroll 1..3,\n"
                 "    --workers W>=1 (else MINDIST_WORKERS; echoed as \"workers\"), --schedule serial|dynamic|dynamic_2cm|static_cyclic|static_snake,\n"
                 "    --prefix P, --order lex|left_lex\n"
                 "    several FILEs: one record per file, the codes run as one batch\n"
                 "  mindist gen --n N --k K --seed S [--plain]\n";
    return 2;
}

int exit_code(int rc) {
    if (rc == MDG_OK) return 0;
    std::cerr << (rc == MDG_EINVAL || rc == MDG_EOVERFLOW ? "error: " : "internal error: ")
              << mdg_last_error() << "\n";
    return (rc == MDG_EINVAL || rc == MDG_EOVERFLOW) ? 2 : 1;
}

bool parse_u64(const char* s, uint64_t& out) {
    char* end = nullptr;
    errno = 0;
    unsigned long long v = std::strtoull(s, &end, 10);
    if (errno || !end || *end || s[0] == '-') return false;
    out = v;
    return true;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    std::string cmd = argv[1];
    if (cmd == "gen") {
        uint64_t n = 0, k = 0, seed = 0;
        bool plain = false;
        for (int i = 2; i < argc; ++i) {
            std::string a = argv[i];
            if (a == "--plain") { plain = true; continue; }
            if (i + 1 >= argc) return usage();
            uint64_t* dst = a == "--n" ? &n : a == "--k" ? &k : a == "--seed" ? &seed : nullptr;
            if (!dst || !parse_u64(argv[++i], *dst)) return usage();
        }
        try {
            mdg::BitMatrix M = mdg::gen_matrix(uint32_t(n), uint32_t(k), seed, !plain);
            std::cout << "# mt19937_64 seed " << seed << (plain ? " (plain)" : " (I|A)") << "\n"
                      << mdg::serialize_matrix(M);
        } catch (const std::exception& e) {
            std::cerr << "error: " << e.what() << "\n";
            return 2;
        }
        return 0;
    }
    if (cmd != "mindist" || argc < 3) return usage();
    std::vector<std::string> paths; // the reference takes one FILE; several run as one batch
    mdg_config cfg;
    mdg_config_default(&cfg);
    bool pretty = false;
    int device = 0;
    std::vector<int> devices; // --devices: one process, several contexts (mdg_min_weight_multi)
    bool seed_given = false;
    bool brute = false;
    bool workers_given = false;
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) != 0) { paths.push_back(a); continue; }
        if (a == "--pretty") { pretty = true; continue; }
        if (a == "--exact-rounds") { cfg.exact_rounds = 1; continue; }
        if (i + 1 >= argc) return usage();
        std::string v = argv[++i];
        uint64_t x = 0;
        if (a == "--algorithm") {
            if (v == "brute") {
                brute = true;
            } else if (v != "gpu" && v != "basic" && v != "optimized" && v != "stack" && v != "saved" &&
                       v != "saved_unrolled") { // engines.cpp:65-73 names: all run the GPU engine
                std::cerr << "error: unknown algorithm: " << v << "\n";
                return 2;
            }
        } else if (a == "--s" || a == "--unroll" || a == "--workers" || a == "--prefix") {
            // CPU-engine settings (EngineConfig::validate, engines.cpp:83-92): checked, unused
            if (!parse_u64(v.c_str(), x)) {
                std::cerr << "error: bad option " << a << " " << v << "\n";
                return 2;
            }
            if (a == "--s" && (x < 1 || x > 8)) { std::cerr << "error: config: s must be in 1..8\n"; return 2; }
            if (a == "--unroll" && (x < 1 || x > 3)) { std::cerr << "error: config: unroll must be in 1..3\n"; return 2; }
            if (a == "--workers" && x < 1) { std::cerr << "error: config: workers must be >= 1\n"; return 2; }
            if (a == "--workers") {
                cfg.workers = uint32_t(x);
                workers_given = true;
            }
        } else if (a == "--schedule") { // parallel.cpp:46-53
            if (v != "serial" && v != "dynamic" && v != "dynamic_2cm" && v != "static_cyclic" &&
                v != "static_snake") {
                std::cerr << "error: unknown schedule: " << v << "\n";
                return 2;
            }
        } else if (a == "--order") { // cli.cpp:86-87
            if (v != "lex" && v != "left_lex") {
                std::cerr << "error: order must be lex or left_lex\n";
                return 2;
            }
        } else if (a == "--gamma-search") {
            if (v == "host") cfg.gamma_search = MDG_GAMMA_HOST;
            else if (v == "gpu") cfg.gamma_search = MDG_GAMMA_GPU;
            else { std::cerr << "error: unknown gamma search: " << v << "\n"; return 2; }
        } else if (a == "--kernel") {
            if (v == "tab") cfg.kernel = MDG_KERNEL_TAB;
            else if (v == "rd") cfg.kernel = MDG_KERNEL_RD;
            else { std::cerr << "error: unknown kernel: " << v << "\n"; return 2; }
        } else if (a == "--trials" && parse_u64(v.c_str(), x)) {
            cfg.trials = uint32_t(x);
        } else if (a == "--seed" && parse_u64(v.c_str(), x)) {
            cfg.seed = x;
            seed_given = true;
        } else if (a == "--level-cap" && parse_u64(v.c_str(), x)) {
            cfg.level_cap = uint32_t(x);
        } else if (a == "--device" && parse_u64(v.c_str(), x)) {
            device = int(x);
        } else if (a == "--devices") { // comma-separated CUDA devices (repeats allowed)
            size_t p0 = 0;
            while (p0 <= v.size()) {
                const size_t p1 = std::min(v.find(',', p0), v.size());
                if (!parse_u64(v.substr(p0, p1 - p0).c_str(), x)) {
                    std::cerr << "error: bad option --devices " << v << "\n";
                    return 2;
                }
                devices.push_back(int(x));
                p0 = p1 + 1;
            }
        } else if (a == "--split-min" && parse_u64(v.c_str(), x)) {
            cfg.split_min = x;
        } else {
            std::cerr << "error: bad option " << a << " " << v << "\n";
            return 2;
        }
    }
    // cli.cpp:78-80: --workers, else MINDIST_WORKERS (default 1); MINDIST_MEMORY_CAP_BYTES
    // (default 2 GiB) caps the CPU engines' saved tables -- parsed and validated as there (a
    // malformed value is an invalid argument, exit 2); the GPU engine's tables live in HBM
    // and are not bound by it
    for (const char* env : {"MINDIST_WORKERS", "MINDIST_MEMORY_CAP_BYTES"}) {
        const char* v = std::getenv(env);
        uint64_t x = 0;
        if (!v || !*v) continue;
        if (!parse_u64(v, x)) {
            std::cerr << "error: " << env << ": not an unsigned integer: " << v << "\n";
            return 2;
        }
        if (!workers_given && std::strcmp(env, "MINDIST_WORKERS") == 0) {
            if (x < 1) { std::cerr << "error: config: workers must be >= 1\n"; return 2; }
            cfg.workers = uint32_t(x);
        }
    }
    if (!seed_given) { // cli.cpp:46-53 draws and logs a seed
        cfg.seed = (uint64_t(std::rand()) << 32) ^ uint64_t(std::rand()) ^ uint64_t(time(nullptr));
        std::cerr << "seed: " << cfg.seed << "\n";
    }
    if (paths.empty()) return usage();
    std::vector<mdg::BitMatrix> Gs(paths.size());
    for (size_t f = 0; f < paths.size(); ++f) {
        try {
            Gs[f] = mdg::parse_matrix_file(paths[f]);
        } catch (const std::invalid_argument& e) {
            std::cerr << "error: " << (paths.size() > 1 ? paths[f] + ": " : "") << e.what() << "\n";
            return 2;
        }
    }
    if (devices.size() > 1 && (brute || paths.size() > 1)) {
        std::cerr << "error: --devices splits the rounds of ONE code (no --algorithm brute, one FILE)\n";
        return 2;
    }
    mdg_ctx* ctx = nullptr;
    int rc = mdg_open(devices.empty() ? device : devices[0], &ctx);
    if (rc) return exit_code(rc);
    std::vector<mdg_run*> runs(paths.size(), nullptr);
    if (devices.size() > 1) { // rounds split across the contexts; rank 0's record is printed
        std::vector<mdg_ctx*> ctxs{ctx};
        for (size_t i = 1; i < devices.size() && rc == 0; ++i) {
            mdg_ctx* c = nullptr;
            rc = mdg_open(devices[i], &c);
            if (rc == 0) ctxs.push_back(c);
        }
        std::vector<mdg_run*> all(ctxs.size(), nullptr);
        if (rc == 0)
            rc = mdg_min_weight_multi(ctxs.data(), uint32_t(ctxs.size()), Gs[0].data(), Gs[0].rows(),
                                      Gs[0].cols(), &cfg, all.data());
        for (size_t i = 1; i < all.size(); ++i)
            if (all[i]) mdg_run_free(all[i]);
        for (size_t i = 1; i < ctxs.size(); ++i) mdg_close(ctxs[i]);
        runs[0] = all[0];
    } else if (brute) {
        for (size_t f = 0; f < paths.size() && rc == 0; ++f)
            rc = mdg_brute_force(ctx, Gs[f].data(), Gs[f].rows(), Gs[f].cols(), 40, &runs[f]);
    } else if (paths.size() == 1) {
        rc = mdg_min_weight(ctx, Gs[0].data(), Gs[0].rows(), Gs[0].cols(), &cfg, &runs[0]);
    } else { // several files: codes in flight on their own streams (mdg_min_weight_batch)
        std::vector<const uint64_t*> ptr;
        std::vector<uint32_t> ks, ns;
        std::vector<mdg_config> cfgs(paths.size(), cfg);
        for (const auto& G : Gs) {
            ptr.push_back(G.data());
            ks.push_back(G.rows());
            ns.push_back(G.cols());
        }
        rc = mdg_min_weight_batch(ctx, uint32_t(paths.size()), ptr.data(), ks.data(), ns.data(),
                                  cfgs.data(), 0, runs.data());
    }
    if (rc) {
        for (mdg_run* r : runs)
            if (r) mdg_run_free(r);
        mdg_close(ctx);
        return exit_code(rc);
    }
    std::vector<char> buf(1 << 20);
    for (size_t f = 0; f < paths.size(); ++f) {
        mdg_run* run = runs[f];
        long len = mdg_run_json(run, buf.data(), buf.size());
        if (len < 0) {
            buf.resize(size_t(-len) + 16);
            len = mdg_run_json(run, buf.data(), buf.size());
        }
        if (pretty) { // result_to_text (cli.cpp:240-255), then the new keys that matter
            mdg_run_info info;
            mdg_run_info_get(run, &info);
            if (paths.size() > 1) std::cout << "file:          " << paths[f] << "\n";
            std::cout << "d:             " << info.d << "\n"
                      << "n:             " << info.n << "\n"
                      << "k:             " << info.k << "\n"
                      << "algorithm:     " << (brute ? "brute" : "gpu") << "\n"
                      << "m:             " << info.m << "\n"
                      << "k_last:        " << info.k_last << "\n"
                      << "g_final:       " << info.g_final << "\n"
                      << "row_additions: " << info.row_additions << "\n"
                      << "combinations:  " << info.combinations << "\n"
                      << "wall_seconds:  " << info.wall_seconds << "\n"
                      << "seed:          " << cfg.seed << "\n"
                      << "workers:       " << cfg.workers << "\n";
            if (info.capped) std::cout << "capped:        true (d is the upper bound at the level cap)\n";
        } else {
            std::cout << buf.data() << "\n";
        }
        mdg_run_free(run);
    }
    mdg_close(ctx);
    return 0;
}
