// common.cuh — shared device-side definitions of the saloba library (product path only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "saloba.h"

#define SALOBA_API extern "C" __attribute__((visibility("default")))

namespace saloba {

// process-wide count of this library's own kernel launches (saloba_kernel_launches)
void count_launches(int n);
// SM count of the current device (cached per device, api.cu)
int sm_count_current();
// status word helpers (pack.cu): init to "no error" (all ones), final maps it to -1 / first index
void launch_status_init(int64_t* st, cudaStream_t s);
void launch_status_final(int64_t* st, cudaStream_t s);

// ---- bins ------------------------------------------------------------------------------------
// bin = path * 8 + gidx; gidx = log2(G) (G in {1,2,4,8,16,32}); path 0 = int32 exact kernel,
// path 1 = int16x2 pair-SIMD two-pass kernel.  Bin 15 collects invalid pairs (never launched).
constexpr int NBINS = 16;
constexpr int BIN_SKIP = 15;
// Bin 14: int16x2 G=1 pairs whose QUERY contains N (dp_i16_kernel<1, R, MODE, 4, QN=true>): an
// N column's substitution is forced to `mismatch` by one LOP3 per register (the 4-entry row
// tables have no "never matches" slot for a query code).  Target N needs no fix-up: its rows use
// an all-mismatch table.
constexpr int QN_BIN = 14;
constexpr int QN2_BIN = 6;  // the same variant at G = 2 (reads the cost model gives two lanes)
// Bin 7: int32 pairs whose values could reach 2^28 (the packed best-cell keys of the FAST int32
// kernel would overflow) or every int32 pair of a call whose scores do not fit int8; runs the plain
// int32 kernel at G = 32.
constexpr int I32_WIDE_BIN = 7;
constexpr int PATH_I32 = 0, PATH_I16 = 1;
constexpr int NGROUPS = 6;
// Largest query block count Q = ceil(qlen/8) a bin of group size G accepts: bounds the spill pool
// (one chunk-boundary row per subwarp slot).  G = 32 takes everything up to the batch maximum.
__host__ __device__ constexpr int qmax_for_gidx(int gidx) {
    return gidx == 0 ? 80 : gidx == 1 ? 160 : gidx == 2 ? 320 : gidx == 3 ? 640 : gidx == 4 ? 1280 : (1 << 17);
}
constexpr int MAX_LEN = 1 << 20;   // S:151 overflow envelope for int32 cells
constexpr int MAX_H0 = 1 << 29;
constexpr int BLOCK_THREADS = 256;
#ifndef I16_BLOCK
#define I16_BLOCK 128
#endif
constexpr int I16_THREADS = I16_BLOCK;
// target rows per lane (strip height) of the int16x2 kernel: 16 = two packed target words
constexpr int I16_ROWS_DEFAULT = 16;
constexpr int I32_ROWS = 8;

struct SortKV {
    uint32_t* keys_in;
    uint32_t* keys_out;
    uint32_t* vals_in;
    uint32_t* vals_out;
    void* cub_temp;
    size_t cub_temp_bytes;
};

struct ClassifyArgs {
    const uint32_t* q_words;  // to detect N in queries (int16x2 path needs N-free queries)
    const int64_t* q_word_off;
    int fmt;
    int match;
    const int32_t* q_len;
    const int32_t* t_len;
    const int32_t* h0;
    int64_t n;
    int mode;
    int force_gidx;   // -1 = auto
    int force_path;   // 0 auto, 1 int32, 2 int16x2 preferred
    int keep_order;
    int i16_rows;
    int64_t max_q_supported;  // query length the spill pool was sized for
    int32_t* score;
    int32_t* q_end;
    int32_t* t_end;
    uint32_t* keys;
    uint32_t* vals;
    int32_t* bin_count;  // [NBINS]
    unsigned long long* status;
    int32_t* long_qmax;  // max Q (8-base blocks) of the int16x2 long bin (atomicMax)
    const int32_t* band_w;  // NEXT-2: per-pair band half-width, or nullptr (banded pairs take the int32 path)
    int32_t i32_fast;       // 1: int32 pairs below the 2^28 value bound go to the FAST kernels (bins 0..5)
    int32_t min_gidx;       // latency floor on log2(G) for batches too small to fill the GPU at G = 1
};

// Queries of >= LONG_Q blocks take the int16x2 "long bin" (bin PATH_I16*8 + NGROUPS-1); its width
// (G=16 or G=32) is decided on the device once the bin is counted (long_bin_gidx).
constexpr int LONG_Q = 256;
constexpr int LONG_BIN = PATH_I16 * 8 + NGROUPS - 1;

// Everything a DP kernel needs; passed by value.
struct AlignArgs {
    const uint32_t* q_words;
    const int64_t* q_word_off;
    const int32_t* q_len;
    const uint32_t* t_words;
    const int64_t* t_word_off;
    const int32_t* t_len;
    const int32_t* h0;
    int64_t n_pairs;
    int32_t match, mismatch, alpha, beta;
    int32_t fmt;  // 4 or 2
    int32_t* score;
    int32_t* q_end;
    int32_t* t_end;
    const uint32_t* perm;     // sorted position -> input index
    const int32_t* bin_start; // [NBINS + 1]
    int32_t* bin_counter;     // [NBINS] dynamic work queues
    int32_t* spill;           // pool (int32 view), cut into block slots of block_slot_words
    int64_t spill_stride;     // elements per (subwarp slot, buffer, H|F) row
    int64_t block_slot_words; // pool words per resident block
    uint32_t* slot_bitmap;    // one bit per block slot: set while a resident block owns it
    int32_t slot_words;       // 32-bit words in slot_bitmap
    int32_t i16_rows;         // target rows per lane of the int16x2 kernel (8 or 16)
    const int32_t* long_gidx; // group index that runs LONG_BIN (set by bin_scan_kernel); others exit
    const int32_t* band_w;    // NEXT-2: per-pair band half-width (cells |i-j| <= w), or nullptr
    int32_t i32_fast;         // 1: the call's scores fit int8 (FAST int32 kernels in bins 0..5)
    unsigned long long* counters;  // NEXT-4 instrumentation (saloba_options.counters) or nullptr
};


// NEXT-4 counters: a warp-wide sum of each lane's contribution, one atomic per counter per warp
__device__ __forceinline__ void count_warp(unsigned long long* ctr, int idx, unsigned long long v) {
    unsigned long long t = v;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(ctr + idx, t);
}

// 8 consecutive bases [8w, 8w+8) of a packed sequence as 8 nibbles (base c in nibble c).
// PACK4: one word.  PACK2: half of a word expanded to nibbles (no N, no padding code: the caller
// masks by length).
__device__ __forceinline__ uint32_t load_block8(const uint32_t* __restrict__ words, int w, int fmt) {
    if (fmt == SALOBA_PACK4) return __ldg(words + w);
    uint32_t x = __ldg(words + (w >> 1)) >> ((w & 1) * 16);  // 8 x 2-bit codes in the low 16 bits
    // spread 2-bit fields into 4-bit nibbles
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r |= ((x >> (2 * c)) & 3u) << (4 * c);
    return r;
}

__device__ __forceinline__ int nib(uint32_t w, int c) { return (w >> (4 * c)) & 15; }

// Block-slot allocator for the spill pool.  Bins run as concurrent kernels, so slots are owned by
// RESIDENT blocks rather than indexed by blockIdx: the pool holds (SMs x max resident blocks per SM)
// block slots, a resident block claims a free bit at start and releases it at exit.  A free bit
// always exists because at most that many blocks can be resident at once.
__device__ __forceinline__ int acquire_block_slot(uint32_t* bitmap, int words) {
    __shared__ int s_slot;
    if (threadIdx.x == 0) {
        int got = -1;
        for (int it = 0; got < 0; ++it) {
            const int w = int((blockIdx.x + it) % unsigned(words));
            uint32_t cur = *((volatile uint32_t*)bitmap + w);
            while (cur != 0xFFFFFFFFu) {
                const int b = __ffs(~cur) - 1;
                const uint32_t old = atomicOr(bitmap + w, 1u << b);
                if (!(old & (1u << b))) {
                    got = w * 32 + b;
                    break;
                }
                cur = old | (1u << b);
            }
        }
        s_slot = got;
    }
    __syncthreads();
    return s_slot;
}
__device__ __forceinline__ void release_block_slot(uint32_t* bitmap, int slot) {
    __syncthreads();
    if (threadIdx.x == 0) atomicAnd(bitmap + (slot >> 5), ~(1u << (slot & 31)));
}

}  // namespace saloba
