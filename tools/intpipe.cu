// intpipe.cu — integer-pipe microbenchmark for the roofline denominator (SURVEY §8(d), Appendix B:
// "which pipe (ALU / FMA) and what lanes/clk VIADDMNMX, VIMNMX3, PRMT, SHFL and IADD3 run at").
//
// Each test runs 8 independent dependency chains per thread of one instruction type at full
// occupancy; per-block cycle counts (clock64) give lane-ops / clk / SM.  Mixed tests interleave
// two instruction types to see whether they dual-issue on different pipes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/intpipe tools/intpipe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <int OP>
__device__ __forceinline__ void step(uint32_t (&x)[CH], uint32_t y, uint32_t z) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        uint32_t v = x[c];
        if (OP == 0) v = (uint32_t)__viaddmax_s32((int)v, (int)y, (int)z);
        if (OP == 1) v = __viaddmax_s16x2(v, y, z);
        if (OP == 2) v = __vimax3_s16x2_relu(v, y, z);
        if (OP == 3) v = (uint32_t)max((int)v, (int)y);
        if (OP == 4) v = prmt(v, y, z);
        if (OP == 5) v = v + y + z;
        if (OP == 6) v = v * y + z;
        if (OP == 7) v = __vadd2(v, y);
        if (OP == 8) v = v ^ y ^ (z & v);
        if (OP == 9) v = (c & 1) ? __viaddmax_s16x2(v, y, z) : v * y + z;  // alu/fma mix?
        if (OP == 10) v = (c & 1) ? __viaddmax_s16x2(v, y, z) : __vimax3_s16x2_relu(v, y, z);
        if (OP == 11) v = (c & 1) ? __viaddmax_s16x2(v, y, z) : prmt(v, y, z);
        if (OP == 12) v = (c & 1) ? __viaddmax_s16x2(v, y, z) : __vadd2(v, y);
        if (OP == 13) v = __shfl_xor_sync(0xffffffffu, v, 1) + y;
        if (OP == 14) v = (uint32_t)__vimax3_s32_relu((int)v, (int)y, (int)z);
        if (OP == 15) v = (c & 1) ? (uint32_t)__viaddmax_s32((int)v, (int)y, (int)z) : v + y + z;
        x[c] = v;
    }
}

template <int OP>
__global__ void bench(uint32_t* out, long long* cyc, uint32_t y, uint32_t z) {
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 7 + c;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) step<OP>(x, y + i, z);
    __syncthreads();
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) acc ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms, double ops_per_iter_per_chain) {
    const int threads = 256;
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bench<OP>, threads, 0);
    const int blocks = sms * nb;
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(uint32_t) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    bench<OP><<<blocks, threads>>>(out, cyc, 3, 5);  // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<OP><<<blocks, threads>>>(out, cyc, 3, 5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int b = 0; b < blocks; ++b) mean += double(h[b]);
    mean /= blocks;
    const double lane_ops_per_block = double(threads) * ITERS * CH * ops_per_iter_per_chain;
    const double per_clk_sm = lane_ops_per_block * nb / mean;
    const double clk_ghz = mean / (ms * 1e6);  // cycles per ns, approximately the SM clock
    printf("{\"op\": \"%s\", \"lane_ops_per_clk_per_sm\": %.1f, \"blocks_per_sm\": %d, \"ms\": %.3f, "
           "\"approx_clk_ghz\": %.3f, \"tera_lane_ops_per_s\": %.2f}\n",
           name, per_clk_sm, nb, ms, clk_ghz, lane_ops_per_block * blocks / (ms * 1e-3) / 1e12);
    delete[] h;
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("VIADDMNMX.s32", sms, 1);
    run<1>("VIADDMNMX.S16x2", sms, 1);
    run<2>("VIMNMX3.S16x2.RELU", sms, 1);
    run<3>("IMNMX.s32", sms, 1);
    run<4>("PRMT", sms, 1);
    run<5>("IADD3(2 adds)", sms, 1);
    run<6>("IMAD", sms, 1);
    run<7>("VIADD.16x2", sms, 1);
    run<8>("LOP3", sms, 1);
    run<9>("mix VIADDMNMX.S16x2+IMAD", sms, 1);
    run<10>("mix VIADDMNMX.S16x2+VIMNMX3", sms, 1);
    run<11>("mix VIADDMNMX.S16x2+PRMT", sms, 1);
    run<12>("mix VIADDMNMX.S16x2+VIADD.16x2", sms, 1);
    run<13>("SHFL+IADD", sms, 1);
    run<14>("VIMNMX3.s32.RELU", sms, 1);
    run<15>("mix VIADDMNMX.s32+IADD3", sms, 1);
    return 0;
}
