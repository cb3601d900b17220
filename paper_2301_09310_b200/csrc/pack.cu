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

// Stream pack (round 2).  Lanes cover the batch's ASCII in 16-byte chunks aligned to the buffer
// (one coalesced 16-byte load per lane, 512 bytes per warp "window"), convert all 16 bytes to codes
// at once, and every packed word is emitted by the lane whose chunk holds its first byte: the word
// is a funnel shift of that chunk's codes and the next lane's (one shuffle).  A warp walks a
// CONTIGUOUS range of windows, so the sequence holding each window's start carries over from the
// previous window (one binary search per warp, not per window: per-window searches made a first
// version 4x slower than the tile kernel); inside a window each lane finds its sequence from one
// boundary per lane (a shared-memory histogram + warp prefix sum).
// Algorithmic bytes per base: 1 read + 1/2 (PACK4) or 1/4 (PACK2) written.
__device__ __forceinline__ uint32_t lut_word(const uint8_t* lut, uint32_t w, uint32_t& bad, uint32_t inv) {
    uint32_t out = 0;  // 4 bytes -> 4 nibble codes; invalid bytes flag bit c of `bad` and become `inv`
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t code = lut[(w >> (8 * c)) & 0xFFu];
        const bool b = code == 0xFFu;
        bad |= (b ? 1u : 0u) << c;
        out |= (b ? inv : code) << (4 * c);
    }
    return out;
}

template <int BITS>
__global__ void __launch_bounds__(256) pack_stream_kernel(const uint8_t* __restrict__ ascii,
                                                          const int64_t* __restrict__ byte_off, int64_t n_seqs,
                                                          int64_t base, uint32_t* __restrict__ words, int64_t cap,
                                                          int64_t* __restrict__ word_off, int32_t* __restrict__ lens,
                                                          unsigned long long* __restrict__ status) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int B = 32 / BITS;  // bases per word
    __shared__ uint8_t lut[256];
    __shared__ int hist[8][33];
    build_lut(lut, BITS);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t first = byte_off[0], total = byte_off[n_seqs];
    if (total / B + n_seqs + base > cap) {  // capacity (closed-form layout): no writes at all
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicMin(status, (unsigned long long)total);
        return;
    }
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, nthr = int64_t(gridDim.x) * blockDim.x;
    for (int64_t sq = tid; sq < n_seqs; sq += nthr) {
        const int64_t b0 = byte_off[sq];
        word_off[sq] = b0 / B + sq + base;
        if (lens) lens[sq] = int(byte_off[sq + 1] - b0);
    }
    if (tid == 0) word_off[n_seqs] = total / B + n_seqs + base;
    if (total <= first) return;
    // chunk j covers stream bytes [16 j - mis, 16 j - mis + 16): 16-byte aligned addresses
    const int64_t mis = int64_t(reinterpret_cast<uintptr_t>(ascii) & 15u);
    const int64_t j0 = (first + mis) >> 4, j1 = (total + mis + 15) >> 4;  // chunks [j0, j1)
    const int64_t nwin = (j1 - j0 + 31) >> 5;
    const int64_t warps = nthr >> 5, gw = tid >> 5;
    const int64_t per = (nwin + warps - 1) / warps;
    const int64_t win_lo = gw * per, win_hi = min(nwin, win_lo + per);
    if (win_lo >= win_hi) return;
    int64_t s0 = 0;  // sequence holding the current window's first byte (or the first sequence)
    if (lane == 0) {
        const int64_t w0 = 16 * (j0 + win_lo * 32) - mis, x = w0 > first ? w0 : first;
        int64_t lo = 0, hi = n_seqs - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (byte_off[mid] <= x) lo = mid;
            else hi = mid - 1;
        }
        s0 = lo;
    }
    s0 = __shfl_sync(FULL, s0, 0);
    for (int64_t win = win_lo; win < win_hi; ++win) {
        const int64_t jw = j0 + win * 32;
        const int64_t c0 = 16 * (jw + lane) - mis;  // my chunk's first stream byte
        const int64_t w0 = 16 * jw - mis;           // the window's first stream byte
        const int64_t bi = byte_off[min(s0 + 1 + lane, n_seqs)];  // end of sequence s0 + lane
        uint32_t by[8];
        auto load16 = [&](int64_t c, uint32_t* o) {
            if (c >= first && c + 16 <= total) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(ascii + c));
                o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
            } else {  // batch edges: bytes outside [first, total) read as 'A'
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t x = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int64_t i = c + 4 * q + k;
                        x |= uint32_t(i >= first && i < total ? ascii[i] : uint8_t('A')) << (8 * k);
                    }
                    o[q] = x;
                }
            }
        };
        load16(c0, by);
        if (lane == 31) load16(c0 + 16, by + 4);
        // codes: bit arithmetic per 8 ACGT bytes, the table otherwise
        uint32_t code[4] = {0, 0, 0, 0};
        uint32_t badmask = 0;
        const int nhalf = lane == 31 ? 4 : 2;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (h >= nhalf) break;
            uint32_t nib = 0;
            if (!fast_acgt8(make_uint2(by[2 * h], by[2 * h + 1]), nib)) {
                uint32_t bad0 = 0, bad1 = 0;
                const uint32_t inv = BITS == 4 ? 15u : 0u;
                nib = lut_word(lut, by[2 * h], bad0, inv) | (lut_word(lut, by[2 * h + 1], bad1, inv) << 16);
                if (h < 2) badmask |= (bad0 | (bad1 << 4)) << (8 * h);
            }
            if (BITS == 4) {
                code[h] = nib;
            } else {  // 8 nibbles (each <= 3) -> 8 two-bit fields
                uint32_t t = nib;
                t = (t | (t >> 2)) & 0x0F0F0F0Fu;
                t = (t | (t >> 4)) & 0x00FF00FFu;
                t = (t | (t >> 8)) & 0xFFFFu;
                code[h >> 1] |= t << (16 * (h & 1));
            }
        }
        if (badmask) {  // first invalid byte of my chunk inside the batch (PACK2: N included)
            for (int k = 0; k < 16; ++k) {
                const int64_t i = c0 + k;
                if (((badmask >> k) & 1u) && i >= first && i < total) {
                    atomicMin(status, (unsigned long long)i);
                    break;
                }
            }
        }
        uint32_t nx0 = __shfl_down_sync(FULL, code[0], 1);  // the next chunk's first codes
        if (lane == 31) nx0 = BITS == 4 ? code[2] : code[1];
        // the sequence holding each lane's chunk start: boundaries at or before it, counted by lane
        hist[wid][lane] = 0;
        __syncwarp();
        {
            const int64_t k = (bi - w0 + 15) >> 4;  // first lane L with c0(L) >= bi
            if (s0 + 1 + lane <= n_seqs && k <= 31) atomicAdd(&hist[wid][k < 0 ? 0 : int(k)], 1);
        }
        __syncwarp();
        int cntL = hist[wid][lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(FULL, cntL, off);
            if (lane >= off) cntL += v;
        }
        const int64_t b31 = __shfl_sync(FULL, bi, 31);
        int64_t s = s0 + cntL;
        if (b31 <= c0 && s0 + 32 < n_seqs) {  // > 32 sequence ends before my chunk: search the rest
            int64_t lo = s0 + 32, hi = n_seqs - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (byte_off[mid] <= c0) lo = mid;
                else hi = mid - 1;
            }
            s = lo;
        }
        // the next window's first sequence: lane 31's, advanced past ends inside its chunk
        int64_t sn = s;
        // emit the words whose first byte is in my chunk [c0, c0 + 16)
        for (; s < n_seqs; ++s) {
            const int64_t st = byte_off[s], en = byte_off[s + 1];
            if (st >= c0 + 16) break;
            if (en <= c0 + 16) sn = s + 1;
            if (en <= c0) continue;
            int64_t w = st >= c0 ? 0 : (c0 - st + B - 1) / B;
            const int64_t wbase = st / B + s + base;
            for (int64_t b = st + B * w; b < en && b < c0 + 16; b += B, ++w) {
                const int o = int(b - c0);  // 0..15
                uint32_t val;
                if (BITS == 4) {  // bits [4o, 4o + 32) of code[0] | code[1] << 32 | nx0 << 64
                    const int k = 4 * o;
                    val = k < 32 ? __funnelshift_r(code[0], code[1], k) : __funnelshift_r(code[1], nx0, k - 32);
                    const int64_t nv = en - b;
                    if (nv < 8) val |= 0xFFFFFFFFu << (4 * nv);
                } else {
                    val = __funnelshift_r(code[0], nx0, 2 * o);
                    const int64_t nv = en - b;
                    if (nv < 16) val &= (1u << (2 * nv)) - 1u;
                }
                words[wbase + w] = val;
            }
        }
        s0 = __shfl_sync(FULL, sn < n_seqs ? sn : n_seqs - 1, 31);
        __syncwarp();  // hist is rewritten by the next window
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
#if SALOBA_PACK_TILE
        if (fmt == SALOBA_PACK4)
            pack_tile2_kernel<4><<<grid, 256, 0, s>>>(ascii, byte_off, n, base, words, cap, word_off, lens,
                                                      (unsigned long long*)status);
        else
            pack_tile2_kernel<2><<<grid, 256, 0, s>>>(ascii, byte_off, n, base, words, cap, word_off, lens,
                                                      (unsigned long long*)status);
#else
        (void)grid;
        if (fmt == SALOBA_PACK4)
            pack_stream_kernel<4><<<int(g8), 256, 0, s>>>(ascii, byte_off, n, base, words, cap, word_off, lens,
                                                          (unsigned long long*)status);
        else
            pack_stream_kernel<2><<<int(g8), 256, 0, s>>>(ascii, byte_off, n, base, words, cap, word_off, lens,
                                                          (unsigned long long*)status);
#endif
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
