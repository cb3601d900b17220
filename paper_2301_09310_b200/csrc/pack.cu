// pack.cu — A1: ASCII -> 4-bit / 2-bit packed words on the GPU (
// SPEC.md S:44-52).  HBM-bound: ~1 byte read + 0.5 (0.25) byte written per base.
//
// Layout (closed form, no scan): sequence s occupies words [byte_off[s]/B + s, ...) with
// B = 8 (PACK4) or 16 (PACK2); ceil(len/B) <= floor(end/B) - floor(start/B) + 1 words fit.
// A warp packs tiles of 8 consecutive sequences with lanes over the tile's flattened words, so
// reads (8 bytes per lane) and 4-bit word writes coalesce and short sequences leave no lane idle.

#include "common.cuh"

namespace saloba {

// Byte -> code table (A/a 0, C/c 1, G/g 2, T/t/U/u 3, N/n 4 [PACK4 only], else 0xFF = invalid),
// staged in shared memory per block; lookups of ASCII letters hit distinct banks.
__device__ __forceinline__ void build_lut(uint8_t* lut, int bits) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        const int u = i & 0xDF;
        const bool letter = ((i | 0x20) >= 'a' && (i | 0x20) <= 'z');
        uint8_t c = 0xFF;
        if (letter) {
            if (u == 'A') c = 0;
            else if (u == 'C') c = 1;
            else if (u == 'G') c = 2;
            else if (u == 'T' || u == 'U') c = 3;
            else if (u == 'N' && bits == 4) c = 4;
        }
        lut[i] = c;
    }
}

// 8 bytes starting at base[pos] (only bytes < total are read; others come back as 0).  The word
// loads are aligned on the ADDRESS (the buffer itself need not be 4-byte aligned: a slice of a
// larger buffer, tests/test_gpu_parity.py) and never touch bytes before base.
__device__ __forceinline__ uint2 load8(const uint8_t* __restrict__ base, int64_t pos, int64_t total) {
    const int mis = int(reinterpret_cast<uintptr_t>(base + pos) & 3u);
    const int64_t a = pos - mis;
    const int sh = mis * 8;
    if (a >= 0 && a + 12 <= total) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(base + a);
        const uint32_t w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2);
        return make_uint2(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh));
    }
    uint32_t lo = 0, hi = 0;
    for (int k = 0; k < 8; ++k) {
        const uint32_t b = (pos + k < total) ? base[pos + k] : 0u;
        if (k < 4) lo |= b << (8 * k);
        else hi |= b << (8 * (k - 4));
    }
    return make_uint2(lo, hi);
}

// 8 ASCII bases -> 8 nibble codes, fast path: if all 8 are A/C/G/T (either case) the codes come
// from bit arithmetic (A 0x41 -> 0, C 0x43 -> 1, G 0x47 -> 2, T 0x54 -> 3: ((u>>1)&3) ^ ((u>>2)&1))
// and a whole-word compare against the re-synthesised canonical letters proves every byte valid.
// Returns false (caller takes the table path) for U, N, invalid bytes.
__device__ __forceinline__ bool fast_acgt8(uint2 by, uint32_t& out) {
    uint32_t nib[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t u = (h ? by.y : by.x) & 0xDFDFDFDFu;                   // upper case
        const uint32_t code = ((u >> 1) ^ ((u >> 2) & 0x01010101u)) & 0x03030303u;
        const uint32_t t = code | (code >> 4);
        uint32_t sel, canon;
        asm("prmt.b32 %0, %1, 0, 0x4420;" : "=r"(sel) : "r"(t));              // 4 codes as nibbles
        asm("prmt.b32 %0, %1, 0, %2;" : "=r"(canon) : "r"(0x54474341u), "r"(sel));  // "ACGT"[code]
        if (canon != u) return false;
        nib[h] = sel & 0xFFFFu;
    }
    out = nib[0] | (nib[1] << 16);
    return true;
}

// A warp packs a tile of 32 consecutive sequences, one lane per sequence: lane i walks its own
// sequence word by word (8-byte loads, L1-served across the lane's consecutive iterations) — no
// per-word bookkeeping.  Common words take the bit-arithmetic path above; words with U, N, padding
// or invalid bytes take the shared-memory byte->code table.
// Tile sweep: per warp, the tile's per-sequence data (exclusive word counts,
// byte and word offsets relative to the tile, lengths) is staged in shared memory; each lane packs
// U consecutive words of the tile's flattened word list (one binary search per lane, then a
// forward walk across sequence ends), so a warp reads ~1 KB of contiguous ASCII per iteration and
// addresses are 32-bit offsets from the tile base.  Partial last words are masked branch-free.
template <int BITS>
__global__ void __launch_bounds__(256) pack_tile2_kernel(const uint8_t* __restrict__ ascii,
                                                         const int64_t* __restrict__ byte_off, int64_t n_seqs,
                                                         int64_t base, uint32_t* __restrict__ words, int64_t cap,
                                                         int64_t* __restrict__ word_off, int32_t* __restrict__ lens,
                                                         unsigned long long* __restrict__ status) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int B = 32 / BITS;  // bases per word
    constexpr int U = 4;          // consecutive words per lane per iteration
    __shared__ uint8_t lut[256];
    __shared__ int s_ex[8][33], s_b0[8][32], s_len[8][32], s_w0[8][32];
    build_lut(lut, BITS);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t total = byte_off[n_seqs];
    // capacity: the closed-form layout ends at word total/B + n_seqs + base; a buffer smaller than
    // that gets no writes at all and the status reports byte index `total` (one past the last byte)
    if (total / (32 / BITS) + n_seqs + base > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicMin(status, (unsigned long long)total);
        return;
    }
    const int64_t tiles = (n_seqs + 31) / 32;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
    for (int64_t tile = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; tile < tiles; tile += warps) {
        const int64_t s = tile * 32 + lane;
        const bool has = s < n_seqs;
        const int64_t b0 = has ? byte_off[s] : byte_off[n_seqs];
        const int len = has ? int(byte_off[s + 1] - b0) : 0;
        const int64_t w0 = b0 / B + s + base;
        if (has) {
            word_off[s] = w0;
            if (lens) lens[s] = len;
            if (s == n_seqs - 1) word_off[n_seqs] = byte_off[n_seqs] / B + n_seqs + base;
        }
        const int nw = (len + B - 1) / B;
        int incl = nw;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, off);
            if (lane >= off) incl += v;
        }
        const int tot = __shfl_sync(FULL, incl, 31);
        const int64_t tb0 = __shfl_sync(FULL, b0, 0), tw0 = __shfl_sync(FULL, w0, 0);
        s_ex[wid][lane] = incl - nw;
        if (lane == 31) s_ex[wid][32] = incl;
        s_b0[wid][lane] = int(b0 - tb0);
        s_len[wid][lane] = len;
        s_w0[wid][lane] = int(w0 - tw0);
        __syncwarp();
        const uint8_t* abase = ascii + tb0;
        uint32_t* wbase = words + tw0;
        for (int j0 = 0; j0 < tot; j0 += 32 * U) {
            const int j = j0 + lane * U;
            if (j < tot) {
                int own = 0;  // last sequence whose first flattened word is <= j
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1)
                    if (own + step <= 31 && s_ex[wid][own + step] <= j) own += step;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int jj = j + u;
                    if (jj >= tot) break;
                    while (s_ex[wid][own + 1] <= jj) ++own;  // crossed a sequence end
                    const int w = jj - s_ex[wid][own];
                    const int rb = s_b0[wid][own] + w * B;  // first byte of this word (tile-relative)
                    const int olen = s_len[wid][own];
                    const int nv = min(B, olen - w * B);     // valid bases in this word (>= 1)
                    uint32_t out = 0, bad = 0;
                    bool fast = false;
                    const uint2 by0 = load8(ascii, tb0 + rb, total);  // absolute: keeps the 4-byte alignment
                    if (BITS == 4) {
                        // bases past the sequence end read as 'A' for the check, become padding nibbles
                        const uint32_t klo = nv >= 4 ? 0xFFFFFFFFu : (1u << (8 * nv)) - 1u;
                        const uint32_t khi = nv >= 8 ? 0xFFFFFFFFu : nv <= 4 ? 0u : (1u << (8 * (nv - 4))) - 1u;
                        const uint2 by = make_uint2((by0.x & klo) | (0x41414141u & ~klo), (by0.y & khi) | (0x41414141u & ~khi));
                        uint32_t n0 = 0;
                        fast = fast_acgt8(by, n0);
                        out = nv >= 8 ? n0 : (n0 | (0xFFFFFFFFu << (4 * nv)));
                    } else if (nv == B) {
                        uint32_t n0 = 0, n1 = 0;
                        fast = fast_acgt8(by0, n0) && fast_acgt8(load8(ascii, tb0 + rb + 8, total), n1);
                        uint32_t a = n0, b = n1;  // 16 nibbles (each <= 3) -> 16 two-bit fields
                        a = (a | (a >> 2)) & 0x0F0F0F0Fu; a = (a | (a >> 4)) & 0x00FF00FFu; a = (a | (a >> 8)) & 0xFFFFu;
                        b = (b | (b >> 2)) & 0x0F0F0F0Fu; b = (b | (b >> 4)) & 0x00FF00FFu; b = (b | (b >> 8)) & 0xFFFFu;
                        out = a | (b << 16);
                    }
                    if (!fast) {  // U, N (PACK4), lower-case-free table path, invalid bytes
                        out = 0;
#pragma unroll
                        for (int half = 0; half < B / 8; ++half) {
                            const uint2 by = half == 0 ? by0 : load8(ascii, tb0 + rb + 8, total);
                            const int nvalid = min(8, nv - half * 8);
#pragma unroll
                            for (int c = 0; c < 8; ++c) {
                                const uint32_t byte = ((c < 4 ? by.x : by.y) >> (8 * (c & 3))) & 0xFFu;
                                uint32_t code = lut[byte];
                                if (c < nvalid) bad |= code;
                                if (c >= nvalid || code == 0xFFu) code = BITS == 4 ? 15u : 0u;
                                out |= code << (BITS * (half * 8 + c));
                            }
                        }
                    }
                    wbase[s_w0[wid][own] + w] = out;
                    if (bad & 0x80u) {
                        for (int c = 0; c < nv; ++c)
                            if (lut[abase[rb + c]] == 0xFF) {
                                atomicMin(status, (unsigned long long)(tb0 + rb + c));
                                break;
                            }
                    }
                }
            }
        }
        __syncwarp();  // the next tile overwrites this warp's staging
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
                       uint32_t* words, int64_t cap, int64_t* word_off, int32_t* lens, int64_t* status,
                       cudaStream_t s) {
    launch_status_init(status, s);
    if (n > 0) {
        const int64_t g8 = int64_t(sm_count_current()) * 8;
        const int64_t need = (n + 255) / 256;  // one warp per 32-sequence tile, 8 warps per block
        const int grid = int(need < g8 ? need : g8);
        if (fmt == SALOBA_PACK4)
            pack_tile2_kernel<4><<<grid, 256, 0, s>>>(ascii, byte_off, n, base, words, cap, word_off, lens,
                                                      (unsigned long long*)status);
        else
            pack_tile2_kernel<2><<<grid, 256, 0, s>>>(ascii, byte_off, n, base, words, cap, word_off, lens,
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
    if (words_capacity < n_seqs + 1) return SALOBA_EWORKSPACE;  // below the layout's minimum
    launch_pack_range(ascii, byte_off, n_seqs, 0, int(fmt), words, words_capacity, word_off, lens, status,
                      (cudaStream_t)stream);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}
