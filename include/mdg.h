/*
 * mdg — B200-native Brouwer–Zimmermann minimum-distance engine: C ABI.
 *
 * The reference (arXiv 1911.08963, /root/reference/proj) is a C++20 library
 * with no FFI; its seam for this path is the round runner
 *   using RoundRunner = std::function<uint32_t(uint32_t gamma_index, uint32_t g, RoundStats&)>;
 *   EngineResult run_bz_loop(const GammaSet&, Bounds, const RoundRunner&);
 * (proj/include/mindist/engines.hpp:151-152, proj/src/engines.cpp:447-476)
 * and its front door  md::min_weight(const BitMatrix&, const EngineConfig&)
 * (engines.hpp:164-166, engines.cpp:617-648). Each entry point below names the
 * reference interface it replaces. Plain pointers and sizes only.
 *
 * Bit layout of every matrix crossing this boundary: row-major, W = ceil(n/64)
 * u64 words per row, bit i of a row in word i/64 at bit position i%64
 * (LSB-first — the same bit order as the reference's u32 words,
 * f2core.hpp:9-12), padding bits zero.
 *
 * Status codes: 0 OK; MDG_EINVAL (-2) bad argument / input (the reference's
 * std::invalid_argument family, CLI exit 2); MDG_EOVERFLOW (-3) 64-bit
 * overflow (std::overflow_error, exit 2); MDG_ECUDA (-4) device failure and
 * MDG_EINTERNAL (-1) anything else (std::exception, exit 1). The message of
 * the last failure on the calling thread: mdg_last_error().
 */
#ifndef MDG_H
#define MDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDG_OK 0
#define MDG_EINTERNAL (-1)
#define MDG_EINVAL (-2)
#define MDG_EOVERFLOW (-3)
#define MDG_ECUDA (-4)

/* Round kernel selector. MDG_KERNEL_TAB: pivot-split Cartesian enumeration
 * (saved suffix table in HBM x prefix chunk in shared memory; the default).
 * MDG_KERNEL_RD: the same tiles with each tile's prefixes a contiguous rank
 * range of the revolving-door order, walked with one (row out ^ row in) XOR
 * per step on the codewords held in registers. Identical results. */
#define MDG_KERNEL_TAB 0
#define MDG_KERNEL_RD 1

const char* mdg_last_error(void);
const char* mdg_version(void);

/* ---------------------------------------------------------------- device */
typedef struct mdg_ctx mdg_ctx;

/* Open a device context (one CUDA stream, device buffers). Replaces the
 * reference's per-engine state (SavedAdditions tables, engines.hpp:94-125). */
int mdg_open(int device, mdg_ctx** out);
void mdg_close(mdg_ctx* ctx);

/* Upload m Gamma matrices (m*k rows of W words). ranks[j] = rank of block j
 * (GammaSet::ranks, gamma.hpp:14-24): Gamma j carries the identity on rows
 * [0, ranks[j]) in columns [j*k, j*k + ranks[j]), which the kernels elide
 * (weight = |S ∩ [0,ranks[j])| + weight of the other columns). ranks == NULL
 * loads raw matrices with no identity structure (config 5). */
int mdg_load_gammas(mdg_ctx* ctx, uint32_t m, uint32_t k, uint32_t n, const uint64_t* rows,
                    const uint32_t* ranks);

typedef struct {
    uint32_t min_weight;      /* UINT32_MAX when nothing was evaluated */
    uint32_t stopped_early;   /* 1 when the early-exit bound fired */
    uint32_t bounded;         /* 1: no codeword below the cutoff; min_weight == cutoff is a bound */
    uint32_t plan_tag;        /* opaque: the tile plan the round ran on (mdg_round_witness decodes with it) */
    uint64_t argmin_key;      /* opaque (weight << 52 | position of the winner); input of mdg_round_witness */
    uint64_t combinations;    /* C(k,c): the reference's RoundStats.combinations */
    uint64_t evaluated;       /* codewords actually evaluated on this device */
    uint64_t task_lo, task_hi;/* task range this call covered (partition units) */
    double device_ms;         /* CUDA-event time of the round's kernels */
} mdg_round_out;

/* One (c, Gamma_j) round: min weight of all XOR-sums of c rows of Gamma_j.
 * Replaces round_saved / round_stack / round_saved_parallel
 * (engines.hpp:140-146, engines.cpp:175-443) behind RoundRunner
 * (engines.hpp:151). stop_at: stop as soon as a weight <= stop_at is found
 * (pass L_prev of the level loop; 0 = enumerate everything). */
int mdg_round(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t stop_at, mdg_round_out* out);

/* Number of partition tasks of round (j, c) and the same round restricted to
 * tasks [task_lo, task_hi) — the unit the multi-GPU path splits across ranks
 * (parallel.cpp:72-88 prefix tasks / engines.cpp:508-557 contiguous blocks). */
int mdg_round_tasks(mdg_ctx* ctx, uint32_t j, uint32_t c, uint64_t* n_tasks);
/* Rank `rank`'s range of a round split `world` ways, as the multi-rank loops cut it: contiguous
 * tasks holding about 1/world of the codewords each (tasks differ in size: a task count split
 * would give the first ranks most of the work; engines.cpp:508-557 splits by combinations). */
int mdg_round_split(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t rank, uint32_t world,
                    uint64_t* task_lo, uint64_t* task_hi);
/* The same split on the host alone (no device): the tile plan of a level-c round of k rows of
 * nw32 compacted 32-bit words for `resident_blocks` resident blocks; *codewords = the range's
 * codeword count. For planning and tests. */
int mdg_plan_split(uint32_t k, uint32_t c, uint32_t nw32, uint32_t resident_blocks, uint32_t rank,
                   uint32_t world, uint64_t* task_lo, uint64_t* task_hi, uint64_t* codewords);
int mdg_round_range(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t stop_at, uint64_t task_lo,
                    uint64_t task_hi, mdg_round_out* out);

/* Bound-pruned round: only weights < cutoff matter (pass the level loop's U).
 * Returns min(true minimum, cutoff); bounded = 1 when no codeword lies below
 * the cutoff. run_bz_loop's U = min(U, w) — hence d and every (L, U) — is the
 * same as with the exact round, while the kernel skips the rest of a codeword's
 * weight as soon as a partial weight exceeds the bound. cutoff 0 = exact. */
int mdg_round_bounded(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t stop_at, uint32_t cutoff,
                      uint64_t task_lo, uint64_t task_hi, mdg_round_out* out);

/* Full weight histogram of round (j, c) (no early exit): hist[0..n] (config 5;
 * no reference counterpart). Returns the min in out. */
int mdg_round_hist(mdg_ctx* ctx, uint32_t j, uint32_t c, uint64_t* hist, mdg_round_out* out);
/* The same histogram at N > 1: rank `rank` counts its contiguous share
 * of the histogram kernel's tiles (about 1/world of the codewords; out->task_lo/hi, out->evaluated
 * are this rank's). With an NCCL communicator attached (mdg_nccl_init) the n + 1 counts are summed
 * across the ranks in stream (ncclAllReduce(sum)): every rank receives the whole histogram and
 * *reduced = 1. Without one hist holds the rank's partial counts (*reduced = 0) for the caller to
 * sum (contexts of one process add them on the host). out->min_weight = first nonzero bin of
 * what hist holds. The reference analog is the merge of worker-local results at join
 * (engines.cpp:432-441). reduced may be NULL. */
int mdg_round_hist_dist(mdg_ctx* ctx, uint32_t j, uint32_t c, uint32_t rank, uint32_t world,
                        uint64_t* hist, mdg_round_out* out, int* reduced);

/* Combination (c sorted row indices) achieving out->min_weight in the task
 * named by out->argmin_key — the witness of that round. */
int mdg_round_witness(mdg_ctx* ctx, uint32_t j, uint32_t c, const mdg_round_out* out,
                      uint32_t* idx);

/* Kernel selection and launch geometry (0 = keep the current value). */
int mdg_set_kernel(mdg_ctx* ctx, int kernel);
/* Bound pruning of the tab kernel (on by default): off computes every
 * codeword's exact weight (results are identical; for roofline measurements
 * of the unpruned kernel). The two settings use different tile plans; the
 * round's plan_tag records which, so mdg_round_witness decodes correctly after
 * a switch, and it re-weighs the decoded rows (MDG_EINTERNAL on a mismatch). */
int mdg_set_pruning(mdg_ctx* ctx, int on);

/* ----------------------------------------------------------- host objects */
typedef struct mdg_gset mdg_gset;   /* GammaSet (gamma.hpp:14-24) */

/* best_gamma_over_permutations(row_basis(G), trials, seed) (gamma.cpp:77-94,
 * f2core.cpp:92-97): rank-deficient G is row-reduced first, as min_weight
 * does (engines.cpp:619). */
int mdg_gset_build(const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials, uint64_t seed,
                   mdg_gset** out);
/* The same search with the trials on the GPU: one warp per
 * trial derives its column order (SplitMix64 skipped ahead to draw t*(n-1)) and
 * the (m, k_last) of compute_gamma_matrices on it; the best trial's Gammas are
 * rebuilt on the host. Identical result to mdg_gset_build for every (trials, seed);
 * meant for trial counts far above the reference default of 10 (a larger k_last
 * lifts L sooner). Needs k <= 512, n <= 4096. */
int mdg_gset_build_gpu(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n, uint32_t trials,
                       uint64_t seed, mdg_gset** out);
/* compute_gamma_matrices on a full-rank G (gamma.cpp:32-75). */
int mdg_gset_compute(const uint64_t* G, uint32_t k, uint32_t n, mdg_gset** out);
void mdg_gset_free(mdg_gset* gs);
/* m, k (effective), n, k_last */
int mdg_gset_info(const mdg_gset* gs, uint32_t* m, uint32_t* k, uint32_t* n, uint32_t* k_last);
/* rows of Gamma j (k*W words), ranks (m), column_perm (n), FNV-1a hash of Gamma j */
int mdg_gset_gamma(const mdg_gset* gs, uint32_t j, uint64_t* rows);
int mdg_gset_ranks(const mdg_gset* gs, uint32_t* ranks);
int mdg_gset_perm(const mdg_gset* gs, uint32_t* perm);
uint64_t mdg_gset_hash(const mdg_gset* gs, uint32_t j);
int mdg_load_gset(mdg_ctx* ctx, const mdg_gset* gs);

/* gamma.cpp:96-100 and :102-106 */
uint32_t mdg_lower_bound(uint32_t m, uint32_t g, uint32_t k, uint32_t k_last);
uint32_t mdg_singleton_upper(uint32_t n, uint32_t k);

/* -------------------------------------------------------------- the loop */
typedef struct { uint32_t c, j, w, U_after, bounded; } mdg_round_rec;
typedef struct { uint32_t c, L_after, U_after, pad; } mdg_level_rec;

/* RoundRunner as a C callback (engines.hpp:151): return 0 and set *w, or a
 * status. stop_at is the loop's current lower bound (early-exit hint). */
typedef int (*mdg_round_fn)(void* user, uint32_t j, uint32_t c, uint32_t stop_at, uint32_t* w);

typedef struct mdg_run mdg_run;     /* result of one BZ run */

/* Cross-rank reduction: replace keys[0..count) by their elementwise minimum over ranks. */
typedef int (*mdg_reduce_fn)(void* user, uint64_t* keys, uint32_t count); /* in-place min */

/* run_bz_loop (engines.cpp:447-476) with the reference's exact semantics,
 * a level cap (0 = none) and the round trace, driving a caller-supplied
 * round. Used for host-logic tests and custom engines. */
int mdg_bz_loop_cb(const mdg_gset* gs, uint32_t lower, uint32_t upper, uint32_t level_cap,
                   mdg_round_fn fn, void* user, mdg_run** out);

/* Front door: min_weight(G, cfg) with the GPU engine (engines.cpp:617-648):
 * row_basis -> Gamma search -> Singleton U -> level loop on the device ->
 * witness. ctx == NULL opens a context on device 0 for the call. */
typedef struct {
    uint32_t trials;      /* permutation_trials, default 10 (engines.hpp:64) */
    uint64_t seed;        /* EngineConfig.seed */
    uint32_t level_cap;   /* 0 = run to termination */
    int kernel;           /* MDG_KERNEL_TAB | MDG_KERNEL_RD */
    int want_witness;     /* 1 = reconstruct and verify a minimum-weight codeword */
    int exact_rounds;     /* 1 = every round's exact minimum (per-round trace parity with the
                             reference's rounds); 0 = rounds bounded by U (same d and (L, U)
                             trace, faster) */
    int gamma_search;     /* MDG_GAMMA_HOST: the permutation trials on host threads;
                             MDG_GAMMA_GPU: on the device (mdg_gset_build_gpu) -- the same
                             Gamma set for the same trials and seed, faster for many trials */
    uint64_t split_min;   /* multi-rank runs: rounds of >= split_min codewords are split across
                             the ranks and their keys reduced; smaller rounds run whole on every
                             rank (identical results, no exchange). 0 = 2e8; 1 = split all */
    uint32_t workers;     /* EngineConfig.workers (engines.hpp:66; the CLI's --workers /
                             MINDIST_WORKERS, cli.cpp:78-79), default 1: echoed as the JSON
                             record's "workers"; the GPU engine's parallelism is the device
                             (and "devices" ranks), so it sets no thread count here */
} mdg_config;
#define MDG_GAMMA_HOST 0
#define MDG_GAMMA_GPU 1
void mdg_config_default(mdg_config* cfg);
int mdg_min_weight(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n, const mdg_config* cfg,
                   mdg_run** out);

/* Batch front door: mdg_min_weight for `count` codes (code i: k[i] rows of
 * n[i] bits at G[i], the mdg_parse_matrix packing, configuration cfg[i]; cfg
 * NULL = mdg_config_default for all) on ctx's device. Up to
 * `streams` codes are in flight at once, each on its own engine and CUDA
 * stream: one code's host Gamma search and upload overlap the others' device
 * level loops, and their small rounds fill the SMs around the large ones.
 * streams = 0 picks 4. out[i] receives code i's run (free each with
 * mdg_run_free); every result equals mdg_min_weight's on that code. On error
 * no run is returned. No reference counterpart (the reference takes one
 * matrix per call); see INTEGRATION.md. */
int mdg_min_weight_batch(mdg_ctx* ctx, uint32_t count, const uint64_t* const* G, const uint32_t* k,
                         const uint32_t* n, const mdg_config* cfg, uint32_t streams,
                         mdg_run** out);

/* The level loop over the Gamma set already loaded into ctx (mdg_load_gset):
 * the device-resident variant of the front door (no Gamma search, no upload). */
int mdg_bz_loop_device(mdg_ctx* ctx, const mdg_gset* gs, const mdg_config* cfg, mdg_run** out);
/* mdg_bz_loop_device for `count` codes at once: code i's Gamma set gs[i] is resident in ctxs[i]
 * (distinct contexts, one device or several), up to `streams` loops in flight from the
 * library's own worker threads (0 = 4). out[i] equals mdg_bz_loop_device(ctxs[i], gs[i], cfg).
 * No reference counterpart (one matrix per call there); cfg NULL = defaults for all. */
int mdg_bz_loop_device_batch(mdg_ctx* const* ctxs, const mdg_gset* const* gs, uint32_t count,
                             const mdg_config* cfg, uint32_t streams, mdg_run** out);
int mdg_bz_loop_device_dist(mdg_ctx* ctx, const mdg_gset* gs, const mdg_config* cfg,
                            uint32_t rank, uint32_t world, mdg_reduce_fn reduce_min, void* user,
                            mdg_run** out);

/* CUDA-event timer on the context's stream (includes host gaps between
 * launches), and the context's counters: kernel launches, H2D / D2H bytes. */
int mdg_timer_start(mdg_ctx* ctx);
int mdg_timer_stop(mdg_ctx* ctx, double* ms);
int mdg_ctx_counters(mdg_ctx* ctx, uint64_t* launches, uint64_t* h2d_bytes, uint64_t* d2h_bytes);
int mdg_device_info(mdg_ctx* ctx, int* sm_count, int* device);

/* Brute force over all 2^k - 1 nonzero codewords of row_basis(G) (the
 * reference's Algorithm::brute_gray, engines.cpp:480-558; min_weight's brute
 * branch, engines.cpp:623-628): rejects k > brute_cap (BruteCapError,
 * MDG_EINVAL; brute_cap in 1..63, EngineConfig::validate engines.cpp:90-91).
 * Result: d and a witness; m = k_last = 0 and no trace, as the reference. */
int mdg_brute_force(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n, uint32_t brute_cap,
                    mdg_run** out);

/* Multi-GPU (one process per GPU): every rank runs the same
 * host loop; each round's task range is split contiguously across ranks and
 * the per-round minimum key is combined with reduce_min (an NCCL
 * allreduce(min) in mdg_dist_*, or any callback). */
int mdg_min_weight_dist(mdg_ctx* ctx, const uint64_t* G, uint32_t k, uint32_t n,
                        const mdg_config* cfg, uint32_t rank, uint32_t world,
                        mdg_reduce_fn reduce_min, void* user, mdg_run** out);
/* NCCL reducer owned by the context (libnccl.so.2 loaded at runtime).
 * mdg_nccl_init also makes the ranks agree on the smallest SM count, so every
 * rank cuts a split round into the same tiles. */
int mdg_nccl_unique_id(uint8_t id[128]);
int mdg_nccl_init(mdg_ctx* ctx, const uint8_t id[128], uint32_t rank, uint32_t world);
int mdg_nccl_reduce_min(void* ctx, uint64_t* keys, uint32_t count); /* mdg_reduce_fn; user = ctx */

/* Cross-process shared bound ("a system-scope atomicMin into a peer-mapped
 * word ... also polled by every block for early exit"; the reference merges worker-local minima
 * only at join, parallel.cpp:20-31). Rank 0 creates a small ring of round-key words in its
 * device memory and passes the 64-byte CUDA IPC handle to the other ranks (any transport: the
 * NCCL / MPI / torch.distributed bootstrap), which map it (same GPU, or peers with native
 * atomics over NVLink). From then on every split round of mdg_min_weight_dist / mdg_bz_loop_
 * device_dist -- the chained NCCL loop and the callback loop alike -- also publishes each tile
 * result into the round's shared word and polls it at every tile fetch: one rank's find lowers
 * the others' pruning bound and fires their early exit. Results are unchanged (the round's key
 * is still the reduction of the ranks' own keys); MDG_NO_SHARED_BOUND disables it. Every rank
 * must create / open before the first split round and run the same sequence of split rounds. */
int mdg_shared_bound_create(mdg_ctx* ctx, uint8_t handle[64]);
int mdg_shared_bound_open(mdg_ctx* ctx, const uint8_t handle[64]);
int mdg_shared_bound_close(mdg_ctx* ctx);

/* In-process exchange group: `world` contexts in ONE process (on one device,
 * or on devices with peer access), each driven by its own thread, run the
 * same level loop; a split round's key is min-reduced by a stream-ordered
 * kernel after cudaStreamWaitEvent on every member's round event (no NCCL, no
 * kernel waiting on another). Same results as the NCCL path (the reference's
 * merge of local minima, engines.cpp:432-441 / parallel.cpp:20-31). Attach
 * each context with its rank, then call mdg_min_weight_dist / mdg_bz_loop_
 * device_dist from one thread per member with reduce_min =
 * mdg_group_reduce_min (a marker: calling it directly is an error). */
typedef struct mdg_group mdg_group;
int mdg_group_create(uint32_t world, mdg_group** out);   /* 1 <= world <= 16 */
void mdg_group_free(mdg_group* g);
int mdg_group_attach(mdg_ctx* ctx, mdg_group* g, uint32_t rank); /* g == NULL detaches */
int mdg_group_reduce_min(void* user, uint64_t* keys, uint32_t count);

/* Single-process multi-GPU front door: min_weight(G) with every round of at
 * least cfg->split_min codewords split across the `world` contexts (their
 * devices; the same device twice is allowed) through an exchange group, one
 * host thread per context. out[r] receives rank r's record (the same d, trace
 * and Gamma set on every rank; per-rank evaluated counts). */
int mdg_min_weight_multi(mdg_ctx* const* ctxs, uint32_t world, const uint64_t* G, uint32_t k,
                         uint32_t n, const mdg_config* cfg, mdg_run** out);

/* Result accessors. */
typedef struct {
    uint32_t d;              /* U at termination, or at the level cap */
    uint32_t capped;         /* 1 when level_cap stopped the loop (d = upper bound) */
    uint32_t n, k, m, k_last, g_final;
    uint32_t n_rounds, n_levels;
    uint32_t witness_ok;     /* 1: witness weight == d and it lies in the code */
    uint64_t combinations;   /* sum of C(k,c) over executed rounds (reference counter) */
    uint64_t evaluated;      /* codewords evaluated on the device(s) */
    uint64_t row_additions;  /* one row XOR per evaluated codeword */
    double wall_seconds;     /* whole call */
    double device_seconds;   /* sum of round kernel times */
    double gamma_seconds;    /* Gamma search on the host */
    double loop_seconds;     /* CUDA-event time of the whole level loop (host gaps included) */
    uint64_t launches;       /* kernels launched by the call */
    uint64_t h2d_bytes, d2h_bytes; /* host<->device traffic of the call */
} mdg_run_info;
int mdg_run_info_get(const mdg_run* r, mdg_run_info* info);
int mdg_run_rounds(const mdg_run* r, mdg_round_rec* out);     /* n_rounds entries */
int mdg_run_levels(const mdg_run* r, mdg_level_rec* out);     /* n_levels entries */
int mdg_run_witness(const mdg_run* r, uint64_t* row);         /* W words, original columns */
/* per executed round (n_rounds entries): codewords evaluated, kernel ms */
int mdg_run_round_perf(const mdg_run* r, uint64_t* evaluated, double* device_ms);
int mdg_run_perm(const mdg_run* r, uint32_t* perm);           /* column_perm (n) */
uint64_t mdg_run_gamma_hash(const mdg_run* r, uint32_t j);
/* The reference CLI's JSON record (cli.cpp:223-238) plus the new keys. */
long mdg_run_json(const mdg_run* r, char* buf, size_t cap);
void mdg_run_free(mdg_run* r);

/* ----------------------------------------------------------- misc / I/O */
/* parse_matrix (io.cpp:33-73): rows_out NULL to query k, n. Errors carry
 * "line L, column C: ..." like ParseError (io.cpp:8-12). */
int mdg_parse_matrix(const char* text, uint32_t* k, uint32_t* n, uint64_t* rows_out);
long mdg_serialize_matrix(const uint64_t* rows, uint32_t k, uint32_t n, char* buf, size_t cap);
/* Config input generator: std::mt19937_64(seed), one draw
 * per bit, bit = draw & 1, row-major; identity != 0 gives G = (I_k | A). */
int mdg_gen_matrix(uint32_t n, uint32_t k, uint64_t seed, int identity, uint64_t* rows);
uint32_t mdg_rank(const uint64_t* rows, uint32_t k, uint32_t n);
uint64_t mdg_hash_rows(const uint64_t* rows, uint32_t k, uint32_t n);
/* Exact binomial (enumeration.cpp:9-20); returns MDG_EOVERFLOW past 64 bits. */
int mdg_binomial(uint32_t p, uint32_t q, uint64_t* out);
/* Revolving-door order (Knuth 7.2.1.3 Alg. R): rank <-> combination. */
int mdg_rd_unrank(uint32_t c, uint64_t rank, uint32_t* idx);
uint64_t mdg_rd_rank(uint32_t c, const uint32_t* idx);

#ifdef __cplusplus
}
#endif
#endif /* MDG_H */
