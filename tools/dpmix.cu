// dpmix.cu — ceiling of the int16x2 cell-update instruction mix on B200 (no memory traffic).
//
// Each thread runs the dp_i16 per-step block (8 columns x R rows, two pairs per register) on
// register-resident state for STEPS steps; the top row of a step is the thread's own bottom row of
// the previous step.  Reports cell updates per second for several instruction orders/occupancies,
// i.e. what the ALU-bound recurrence can reach with zero overhead around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dpmix tools/dpmix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t vaddmax(uint32_t a, uint32_t b, uint32_t c) { return __viaddmax_s16x2(a, b, c); }
__device__ __forceinline__ uint32_t vmax3relu(uint32_t a, uint32_t b, uint32_t c) { return __vimax3_s16x2_relu(a, b, c); }
__device__ __forceinline__ uint32_t vmax3(uint32_t a, uint32_t b, uint32_t c) { return __vimax3_s16x2(a, b, c); }
__device__ __forceinline__ uint32_t vadd(uint32_t a, uint32_t b) { return __vadd2(a, b); }
__device__ __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) { return __vmaxs2(a, b); }

constexpr int STEPS = 4096;

// ORDER 0: column-major (x outer, r inner) as in dp_i16.  ORDER 1: anti-diagonal order (cells with
// equal x + r issued together).  ORDER 2: column-major with a compiler barrier between columns
// (models one basic block per column).
template <int R, int ORDER, int MINB>
__global__ void __launch_bounds__(128, MINB) mix(uint32_t* out, uint32_t seed) {
    uint32_t tabA[R], tabB[R], Hl[R], En[R], sel[8], topH[8], topF[8];
    const uint32_t t = threadIdx.x * 2654435761u ^ seed;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        tabA[r] = 0xFCFCFC01u ^ (((t >> r) & 3u) * 0x01010101u & 0x03030303u);
        tabB[r] = 0xFCFC01FCu;
        Hl[r] = 0;
        En[r] = 0xFFF9FFF9u;
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
        sel[x] = 0xC4C4C4C4u ^ ((t >> x) & 0x01010101u);
        sel[x] = 0xBB33 | (((x + (t & 3)) & 3) * 0x11u) | 0x88880000u;
        topH[x] = 0;
        topF[x] = 0xFFF9FFF9u;
    }
    const uint32_t nbeta = 0xFFFFFFFFu, nalpha = 0xFFF9FFF9u;
    uint32_t M0 = 0, M1 = 0, M2 = 0, M3 = 0, corner = 0;
    for (int s = 0; s < STEPS; ++s) {
        if (ORDER == 1) {
            uint32_t f[8], ha[8], hd[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                f[x] = topF[x];
                ha[x] = vadd(topH[x], nalpha);
                hd[x] = x == 0 ? corner : topH[x - 1];
            }
            const uint32_t c7 = topH[7];
#pragma unroll
            for (int dg = 0; dg < R + 7; ++dg) {
                int cnt = 0;
                uint32_t dprev = 0;
#pragma unroll
                for (int x = 7; x >= 0; --x) {
                    const int r = dg - x;
                    if (r < 0 || r >= R) continue;
                    const uint32_t ff = vaddmax(f[x], nbeta, ha[x]);
                    const uint32_t e = En[r];
                    const uint32_t sc = prmt(tabA[r], tabB[r], sel[x]);
                    const uint32_t d = vadd(hd[x], sc);
                    const uint32_t h = vmax3relu(d, e, ff);
                    const uint32_t hh = vadd(h, nalpha);
                    hd[x] = Hl[r];
                    Hl[r] = h;
                    En[r] = vaddmax(e, nbeta, hh);
                    ha[x] = hh;
                    f[x] = ff;
                    if (cnt & 1) {
                        if ((dg & 3) == 0) M0 = vmax3(M0, dprev, d);
                        if ((dg & 3) == 1) M1 = vmax3(M1, dprev, d);
                        if ((dg & 3) == 2) M2 = vmax3(M2, dprev, d);
                        if ((dg & 3) == 3) M3 = vmax3(M3, dprev, d);
                    }
                    dprev = d;
                    ++cnt;
                    if (r == R - 1) {
                        topH[x] = h;
                        topF[x] = ff;
                    }
                }
            }
            corner = c7;
        } else {
            uint32_t botH[8], botF[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                uint32_t hup = topH[x], fup = topF[x];
                uint32_t haup = vadd(hup, nalpha);
                uint32_t hdiag = (x == 0) ? corner : topH[x - 1];
                uint32_t dprev = 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t f = vaddmax(fup, nbeta, haup);
                    const uint32_t e = En[r];
                    const uint32_t sc = prmt(tabA[r], tabB[r], sel[x]);
                    const uint32_t d = vadd(hdiag, sc);
                    const uint32_t h = vmax3relu(d, e, f);
                    const uint32_t ha = vadd(h, nalpha);
                    hdiag = Hl[r];
                    Hl[r] = h;
                    En[r] = vaddmax(e, nbeta, ha);
                    hup = h;
                    haup = ha;
                    fup = f;
                    if (r & 1) {
                        if ((r & 7) == 1) M0 = vmax3(M0, dprev, d);
                        if ((r & 7) == 3) M1 = vmax3(M1, dprev, d);
                        if ((r & 7) == 5) M2 = vmax3(M2, dprev, d);
                        if ((r & 7) == 7) M3 = vmax3(M3, dprev, d);
                    }
                    dprev = d;
                }
                botH[x] = hup;
                botF[x] = fup;
                if (ORDER == 2) asm volatile("" ::: "memory");
            }
            corner = topH[7];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                topH[x] = botH[x];
                topF[x] = botF[x];
            }
        }
#pragma unroll
        for (int x = 0; x < 8; ++x) sel[x] = prmt(sel[x], 0u, 0x1032);  // vary the selectors per step
    }
    uint32_t acc = vmax(vmax(M0, M1), vmax(M2, M3));
#pragma unroll
    for (int r = 0; r < R; ++r) acc ^= Hl[r] ^ En[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int R, int ORDER, int MINB>
void run(const char* name, int sms) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, mix<R, ORDER, MINB>, 128, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, mix<R, ORDER, MINB>);
    const int blocks = sms * nb * 4;
    uint32_t* out;
    cudaMalloc(&out, sizeof(uint32_t) * blocks * 128);
    mix<R, ORDER, MINB><<<blocks, 128>>>(out, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<R, ORDER, MINB><<<blocks, 128>>>(out, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cells = double(blocks) * 128 * STEPS * 8 * R * 2;
    printf("{\"variant\": \"%s\", \"regs\": %d, \"local_bytes\": %zu, \"blocks_per_sm\": %d, \"ms\": %.3f, \"tcups\": %.3f}\n",
           name, fa.numRegs, fa.localSizeBytes, nb, ms, cells / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<16, 0, 3>("R16 colmajor minb3", sms);
    run<16, 0, 4>("R16 colmajor minb4", sms);
    run<16, 2, 3>("R16 colmajor-barrier minb3", sms);
    run<16, 1, 3>("R16 antidiag minb3", sms);
    run<16, 1, 4>("R16 antidiag minb4", sms);
    run<8, 0, 4>("R8 colmajor minb4", sms);
    run<8, 0, 6>("R8 colmajor minb6", sms);
    run<8, 1, 6>("R8 antidiag minb6", sms);
    run<32, 0, 2>("R32 colmajor minb2", sms);
    run<16, 0, 1>("R16 colmajor minb1", sms);
    run<16, 0, 2>("R16 colmajor minb2", sms);
    return 0;
}
