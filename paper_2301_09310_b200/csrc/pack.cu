// pack.cu — A1: ASCII -> 4-bit / 2-bit packed words on the GPU (
// SPEC.md S:44-52).  HBM-bound: ~1 byte read + 0.5 (0.25) byte written per base.
//
// Layout (closed form, no scan): sequence s occupies words [byte_off[s]/B + s, ...) with
// B = 8 (PACK4) or 16 (PACK2); ceil(len/B) <= floor(end/B) - floor(start/B) + 1 words fit.
// One warp per sequence, one lane per output word: the warp reads 256 contiguous bytes per
// instruction (32 lanes x 8 bytes), so reads coalesce; 4-bit output words coalesce likewise.
#include "common.cuh"

namespace saloba {

// code table: A/a 0, C/c 1, G/g 2, T/t/U/u 3, N/n 4, anything else 0xFF (invalid)
__device__ __forceinline__ uint32_t base_code(uint32_t b) {
    uint32_t u = b & 0xDF;  // upper-case ASCII letters
    uint32_t c = 0xFF;
    c = (u == 'A') ? 0u : c;
    c = (u == 'C') ? 1u : c;
    c = (u == 'G') ? 2u : c;
    c = (u == 'T' || u == 'U') ? 3u : c;
    c = (u == 'N') ? 4u : c;
    // reject non-letters that alias after the case fold (e.g. 'A' ^ 0x20 = 'a' is fine, but 0x01 etc.)
    c = ((b | 0x20) >= 'a' && (b | 0x20) <= 'z') ? c : 0xFFu;
    return c;
}

__device__ __forceinline__ uint64_t load8_unaligned(const uint8_t* __restrict__ base, int64_t pos, int64_t total) {
    // 8 bytes starting at base[pos] (bytes beyond `total` are returned as 0)
    int64_t a = pos & ~int64_t(7);
    int sh = int(pos & 7) * 8;
    if (a + 16 <= total) {
        uint64_t lo = __ldg(reinterpret_cast<const unsigned long long*>(base + a));
        uint64_t hi = __ldg(reinterpret_cast<const unsigned long long*>(base + a + 8));
        return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
    }
    uint64_t r = 0;
    for (int k = 0; k < 8; ++k)
        if (pos + k < total) r |= uint64_t(base[pos + k]) << (8 * k);
    return r;
}

template <int BITS>
__global__ void __launch_bounds__(256) pack_kernel(const uint8_t* __restrict__ ascii, const int64_t* __restrict__ byte_off,
                                                   int64_t n_seqs, int64_t base, uint32_t* __restrict__ words,
                                                   int64_t* __restrict__ word_off, int32_t* __restrict__ lens,
                                                   unsigned long long* __restrict__ status) {
    constexpr int B = 32 / BITS;  // bases per word
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t total = byte_off[n_seqs];  // ascii is readable up to here
    for (int64_t s = warp; s < n_seqs; s += nwarps) {
        const int64_t b0 = byte_off[s], b1 = byte_off[s + 1];
        const int64_t len = b1 - b0;
        const int64_t w0 = b0 / B + s + base;
        if (lane == 0) {
            word_off[s] = w0;
            if (lens) lens[s] = int32_t(len);
            if (s == n_seqs - 1) word_off[n_seqs] = byte_off[n_seqs] / B + n_seqs + base;
        }
        const int64_t nw = (len + B - 1) / B;
        for (int64_t w = lane; w < nw; w += 32) {
            uint32_t out = 0;
            unsigned long long bad = ~0ull;
#pragma unroll
            for (int half = 0; half < B / 8; ++half) {
                const int64_t p0 = w * B + half * 8;  // first base of this 8-base group
                uint64_t bytes = load8_unaligned(ascii, b0 + p0, total);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int64_t p = p0 + c;
                    uint32_t code;
                    if (p < len) {
                        code = base_code(uint32_t(bytes >> (8 * c)) & 0xFF);
                        if (code == 0xFF || (BITS == 2 && code == 4)) {
                            if (bad == ~0ull) bad = (unsigned long long)(b0 + p);
                            code = BITS == 4 ? 15u : 0u;
                        }
                    } else {
                        code = BITS == 4 ? 15u : 0u;  // padding (never scored)
                    }
                    out |= code << (BITS * (half * 8 + c));
                }
            }
            words[w0 + w] = out;
            if (bad != ~0ull) atomicMin(status, bad);
        }
    }
}

__global__ void status_init(unsigned long long* st) { *st = ~0ull >> 1; }
__global__ void status_final(unsigned long long* st) {
    if (*st == (~0ull >> 1)) *st = (unsigned long long)(-1ll);
}

void launch_status_init(int64_t* st, cudaStream_t s) {
    status_init<<<1, 1, 0, s>>>((unsigned long long*)st);
    count_launches(1);
}
void launch_status_final(int64_t* st, cudaStream_t s) {
    status_final<<<1, 1, 0, s>>>((unsigned long long*)st);
    count_launches(1);
}

int sm_count_current();

// Pack sequences [0, n) of byte_off; `base` shifts the closed-form word layout so that slices of
// a larger batch land where a single whole-batch pack would put them.
void launch_pack_range(const uint8_t* ascii, const int64_t* byte_off, int64_t n, int64_t base, int fmt,
                       uint32_t* words, int64_t* word_off, int32_t* lens, int64_t* status, cudaStream_t s) {
    launch_status_init(status, s);
    if (n > 0) {
        const int64_t g8 = int64_t(sm_count_current()) * 8;
        const int grid = int((n + 7) / 8 < g8 ? (n + 7) / 8 : g8);
        if (fmt == SALOBA_PACK4)
            pack_kernel<4><<<grid, 256, 0, s>>>(ascii, byte_off, n, base, words, word_off, lens,
                                                (unsigned long long*)status);
        else
            pack_kernel<2><<<grid, 256, 0, s>>>(ascii, byte_off, n, base, words, word_off, lens,
                                                (unsigned long long*)status);
        count_launches(1);
    }
    launch_status_final(status, s);
}

}  // namespace saloba

using namespace saloba;

SALOBA_API int64_t saloba_packed_words(int64_t total_bases, int64_t n_seqs, saloba_packing fmt) {
    if (total_bases < 0 || n_seqs < 0 || (fmt != SALOBA_PACK4 && fmt != SALOBA_PACK2)) return -1;
    const int B = fmt == SALOBA_PACK4 ? 8 : 16;
    return total_bases / B + n_seqs + 1;
}

SALOBA_API int saloba_pack(const uint8_t* ascii, const int64_t* byte_off, int64_t n_seqs, saloba_packing fmt,
                           uint32_t* words, int64_t words_capacity, int64_t* word_off, int32_t* lens,
                           int64_t* status, void* stream) {
    if (n_seqs < 0 || !byte_off || !words || !word_off || !status || (n_seqs > 0 && !ascii)) return SALOBA_EINVAL;
    if (fmt != SALOBA_PACK4 && fmt != SALOBA_PACK2) return SALOBA_EINVAL;
    if (words_capacity < 0) return SALOBA_EINVAL;
    launch_pack_range(ascii, byte_off, n_seqs, 0, int(fmt), words, word_off, lens, status, (cudaStream_t)stream);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}
