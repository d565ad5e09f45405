// Integer pipe-rate microbenchmark for sm_100a: the denominators of the
// round kernel's roofline (SURVEY.md §8d asks to confirm POPC / LOP3 issue
// rates on the box instead of trusting the cc<=9.0 throughput table).
//
// Each kernel runs NCH independent dependency chains per thread of a single
// instruction class, long enough that issue throughput (not latency) binds.
// ops/clk/SM = (threads * iters * NCH) / (elapsed_s * f_sm * SMs), with f_sm
// measured in-kernel: clock64() is a per-SM counter, so the span from the first
// block start to the last block end ON ONE SM (blocks run in several waves) over the
// CUDA-event wall time. (Round 1 divided block 0's span alone by the wall time: block 0
// ran one of four waves, which gave f ~ 485 MHz and 4x inflated per-clock rates; its
// Gops column was right.)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes tools/pipes_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 16

__device__ unsigned long long g_sink;
__device__ long long g_clk[2 * 4096];
__device__ unsigned g_smid[4096];

template <int OP>
__global__ void pipe_kernel(uint32_t seed, int iters) {
    uint32_t a[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
    uint32_t b = seed ^ 0x5bd1e995u, c = seed * 3u + 1u;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            if (OP == 0) {        // LOP3: 3-input xor
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
            } else if (OP == 1) { // POPC chain
                asm volatile("popc.b32 %0, %0;" : "+r"(a[i]));
            } else if (OP == 2) { // IADD3
                asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            } else if (OP == 3) { // IMNMX
                asm volatile("min.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            } else if (OP == 4) { // IMAD (fma pipe)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
            } else if (OP == 6) { // PRMT (byte permute)
                asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a[i]) : "r"(b));
            } else if (OP == 7) { // SHF funnel shift (rotate)
                asm volatile("shf.l.wrap.b32 %0, %0, %1, 16;" : "+r"(a[i]) : "r"(b));
            } else if (OP == 8) { // LOP3 and IMNMX interleaved: separate pipes?
                if (i & 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
                else asm volatile("min.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            } else if (OP == 9) { // LOP3 and POPC interleaved 4:1
                if ((i & 3) == 3) asm volatile("popc.b32 %0, %0;" : "+r"(a[i]));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
            } else if (OP == 10) { // LOP3 and PRMT interleaved 1:1
                if (i & 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
                else asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a[i]) : "r"(b));
            } else if (OP == 5) { // POPC of a 64-bit value (2x POPC + add)
                uint64_t v = ((uint64_t)a[i] << 32) | b;
                uint32_t r;
                asm volatile("popc.b64 %0, %1;" : "=r"(r) : "l"(v));
                a[i] = r;
            }
        }
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc ^= a[i];
    if (acc == 0xFFFFFFFFu) g_sink = acc;
    if (threadIdx.x == 0 && blockIdx.x < 4096) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_clk[2 * blockIdx.x] = t0;
        g_clk[2 * blockIdx.x + 1] = t1;
        g_smid[blockIdx.x] = smid;
    }
}

template <int OP>
void run(const char* name, int sms) {
    int threads = 512, blocks = sms * 4, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    pipe_kernel<OP><<<blocks, threads>>>(1u, 64); // warm-up
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    pipe_kernel<OP><<<blocks, threads>>>(7u, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    static long long clk[2 * 4096];
    static unsigned smid[4096];
    cudaMemcpyFromSymbol(clk, g_clk, sizeof(long long) * 2 * blocks);
    cudaMemcpyFromSymbol(smid, g_smid, sizeof(unsigned) * blocks);
    long long lo = -1, hi = -1; // first start .. last end of the blocks on block 0's SM
    for (int b = 0; b < blocks; ++b)
        if (smid[b] == smid[0]) {
            if (lo < 0 || clk[2 * b] < lo) lo = clk[2 * b];
            if (hi < 0 || clk[2 * b + 1] > hi) hi = clk[2 * b + 1];
        }
    double f_mhz = double(hi - lo) / (ms * 1e3); // the timed loop spans ~the whole kernel
    double ops = (double)threads * blocks * iters * NCH;
    double per_clk_sm = ops / (ms * 1e-3) / (f_mhz * 1e6) / sms;
    printf("{\"op\": \"%s\", \"ms\": %.3f, \"f_mhz_est\": %.0f, \"ops_per_clk_per_sm\": %.2f, \"Gops\": %.1f}\n",
           name, ms, f_mhz, per_clk_sm, ops / (ms * 1e-3) / 1e9);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"clock_khz_attr\": %d}\n",
           p.name, p.multiProcessorCount, p.major, p.minor, clk_khz);
    int sms = p.multiProcessorCount;
    run<0>("lop3", sms);
    run<1>("popc32", sms);
    run<2>("iadd", sms);
    run<3>("imnmx", sms);
    run<4>("imad", sms);
    run<5>("popc64", sms);
    run<6>("prmt", sms);
    run<7>("shf_rot", sms);
    run<8>("lop3+imnmx_1:1", sms);
    run<9>("lop3+popc_3:1", sms);
    run<10>("lop3+prmt_1:1", sms);
    return 0;
}
