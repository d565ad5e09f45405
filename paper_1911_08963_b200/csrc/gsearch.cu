// GPU permutation search: best_gamma_over_permutations
// (gamma.cpp:77-94) for many trials at once. One warp per trial:
//   1. the trial's column order: identity shuffled by Fisher-Yates (util.hpp:28-33,
//      j = next() % i) with SplitMix64 (util.hpp:12-24) positioned at draw t*(n-1) -- the
//      reference draws n-1 values per trial from one generator, and SplitMix64's state
//      after N draws is seed + N*gamma, so every trial is independent here;
//   2. (m, k_last) of compute_gamma_matrices (gamma.cpp:32-75) on that order without
//      building the Gammas: block j's pivot columns are the greedy independent set of the
//      columns at positions >= j*k in the current order (row operations keep column
//      dependencies), and a pick at position pc swaps it with position `target` exactly
//      as the reference's column swap. A warp tests 32 candidate positions at once,
//      reducing each column against the block's echelon basis (one broadcast smem row
//      per step); the scan pointer only moves forward (everything it skipped is
//      dependent and stays so while the basis grows).
//   3. key = (m, k_last, earliest trial) packed for atomicMax.
// The host recomputes the winning trial's Gammas (and the identity's) and keeps the
// reference's strict-improvement rule, so the result equals the host search bit for bit.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "engine.hpp"

namespace mdg {

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw CudaError(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x);      \
    } while (0)

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t splitmix_at(uint64_t state) {
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct SearchArgs {
    const uint64_t* cols; // n column vectors of KW u64 words (bit r = row r)
    uint32_t n, k, wpb;   // columns, rows, warps per block
    uint64_t seed, trials;
    unsigned long long* best;
};

template <int KW>
__global__ void __launch_bounds__(256) perm_search(SearchArgs a) {
    extern __shared__ __align__(16) uint64_t smem[];
    const uint32_t n = a.n, k = a.k;
    uint64_t* cols = smem;                                     // n * KW
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t per_warp = size_t(k) * KW + (size_t(n) + 3) / 4 + (size_t(k) + 3) / 4;
    uint64_t* basis = smem + size_t(n) * KW + warp * per_warp; // k * KW
    uint16_t* order = reinterpret_cast<uint16_t*>(basis + size_t(k) * KW);
    uint16_t* piv = order + ((n + 3) & ~3u);
    for (uint32_t i = threadIdx.x; i < n * KW; i += blockDim.x) cols[i] = a.cols[i];
    __syncthreads();

    for (uint64_t t = uint64_t(blockIdx.x) * a.wpb + warp; t < a.trials; t += uint64_t(gridDim.x) * a.wpb) {
        for (uint32_t i = lane; i < n; i += 32) order[i] = uint16_t(i);
        __syncwarp();
        if (lane == 0) {
            uint64_t st = a.seed + t * uint64_t(n - 1) * kGolden;
            for (uint32_t i = n; i > 1; --i) {
                st += kGolden;
                const uint32_t j = uint32_t(splitmix_at(st) % i);
                const uint16_t x = order[i - 1];
                order[i - 1] = order[j];
                order[j] = x;
            }
        }
        __syncwarp();
        uint32_t m = 0, k_last = 0;
        for (uint32_t o = 0; o < n; o += k) {
            uint32_t cnt = 0, target = o, s = o;
            while (cnt < k && target < n) {
                bool found = false;
                for (; s < n && !found; s += 32) {
                    const uint32_t pos = s + lane;
                    uint64_t v[KW];
#pragma unroll
                    for (int w = 0; w < KW; ++w) v[w] = pos < n ? cols[size_t(order[pos]) * KW + w] : 0;
                    for (uint32_t i = 0; i < cnt; ++i) {
                        const uint32_t p = piv[i];
                        if ((v[p >> 6] >> (p & 63)) & 1u) {
#pragma unroll
                            for (int w = 0; w < KW; ++w) v[w] ^= basis[size_t(i) * KW + w];
                        }
                    }
                    uint64_t any = 0;
#pragma unroll
                    for (int w = 0; w < KW; ++w) any |= v[w];
                    const uint32_t mask = __ballot_sync(0xFFFFFFFFu, pos < n && any != 0);
                    if (mask) {
                        const uint32_t li = __ffs(mask) - 1;
                        const uint32_t pc = s + li;
                        if (lane == li) {
                            uint32_t p = 0;
#pragma unroll
                            for (int w = KW - 1; w >= 0; --w)
                                if (v[w]) p = uint32_t(w) * 64 + __ffsll(static_cast<long long>(v[w])) - 1;
#pragma unroll
                            for (int w = 0; w < KW; ++w) basis[size_t(cnt) * KW + w] = v[w];
                            piv[cnt] = uint16_t(p);
                            const uint16_t x = order[target];
                            order[target] = order[pc];
                            order[pc] = x;
                        }
                        __syncwarp();
                        ++cnt;
                        ++target;
                        s = pc + 1 - 32; // the loop's s += 32 lands on pc + 1
                        found = true;
                    }
                }
                if (!found) break;
            }
            if (cnt == 0) break;
            ++m;
            k_last = cnt;
            if (cnt < k) break;
        }
        if (lane == 0) {
            const unsigned long long key = (static_cast<unsigned long long>(m) << kSearchMShift) |
                                           (static_cast<unsigned long long>(k_last) << kSearchKShift) |
                                           ((1ull << kSearchKShift) - 1 - t);
            atomicMax(a.best, key);
        }
        __syncwarp();
    }
}

template <int KW>
void launch_search(const SearchArgs& base, size_t col_bytes, size_t warp_bytes, int sms, cudaStream_t st) {
    SearchArgs a = base;
    auto fn = perm_search<KW>;
    const size_t budget = 200 * 1024;
    uint32_t wpb = 8;
    while (wpb > 1 && col_bytes + wpb * warp_bytes > budget) --wpb;
    if (col_bytes + wpb * warp_bytes > budget)
        throw std::invalid_argument("gpu permutation search: matrix too large for shared memory");
    a.wpb = wpb;
    const size_t smem = col_bytes + wpb * warp_bytes;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    uint64_t blocks = (a.trials + wpb - 1) / wpb;
    const uint64_t cap = uint64_t(sms) * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    fn<<<uint32_t(blocks), wpb * 32, smem, st>>>(a);
}

} // namespace

// Best (m, k_last, earliest trial) over `trials` shuffled orders of G's columns;
// returns (m << 51 | k_last << 41 | (2^41 - 1 - t)) for the best trial t (engine.hpp).
uint64_t Engine::permutation_search(const uint64_t* rows, uint32_t k, uint32_t n, uint32_t trials,
                                    uint64_t seed) {
    if (k < 1 || k > 512 || n < k || n > 4096)
        throw std::invalid_argument("gpu permutation search: needs 1 <= k <= 512, k <= n <= 4096");
    if (trials < 1 || uint64_t(trials) >= (uint64_t{1} << kSearchKShift))
        throw std::invalid_argument("best_gamma_over_permutations: trials must be >= 1");
    CK(cudaSetDevice(device_));
    const uint32_t W = (n + 63) / 64;
    const uint32_t KW = k <= 64 ? 1 : k <= 128 ? 2 : k <= 256 ? 4 : 8;
    std::vector<uint64_t> cols(size_t(n) * KW, 0);
    for (uint32_t r = 0; r < k; ++r)
        for (uint32_t c = 0; c < n; ++c)
            if ((rows[size_t(r) * W + (c >> 6)] >> (c & 63)) & 1u)
                cols[size_t(c) * KW + (r >> 6)] |= uint64_t{1} << (r & 63);
    uint64_t* d_cols = static_cast<uint64_t*>(scratch(cols.size() * 8 + 8));
    unsigned long long* d_best = reinterpret_cast<unsigned long long*>(d_cols + cols.size());
    cudaStream_t st = stream();
    CK(cudaMemcpyAsync(d_cols, cols.data(), cols.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_best, 0, 8, st));
    SearchArgs a{};
    a.cols = d_cols;
    a.n = n;
    a.k = k;
    a.seed = seed;
    a.trials = trials;
    a.best = d_best;
    const size_t col_bytes = size_t(n) * KW * 8;
    const size_t warp_bytes = (size_t(k) * KW + (size_t(n) + 3) / 4 + (size_t(k) + 3) / 4) * 8;
    switch (KW) {
        case 1: launch_search<1>(a, col_bytes, warp_bytes, sms_, st); break;
        case 2: launch_search<2>(a, col_bytes, warp_bytes, sms_, st); break;
        case 4: launch_search<4>(a, col_bytes, warp_bytes, sms_, st); break;
        default: launch_search<8>(a, col_bytes, warp_bytes, sms_, st); break;
    }
    CK(cudaGetLastError());
    count_launch();
    uint64_t key = 0;
    CK(cudaMemcpyAsync(&key, d_best, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return key;
}

} // namespace mdg
