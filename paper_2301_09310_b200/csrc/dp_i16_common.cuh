// dp_i16_common.cuh — device helpers shared by the int16x2 kernels (dp_i16.cu: any G;
// dp_g1.cu: the G = 1 kernel).  Product path only.
#pragma once
#include <climits>

#include "common.cuh"

namespace saloba {

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t vaddmax(uint32_t a, uint32_t b, uint32_t c) { return __viaddmax_s16x2(a, b, c); }
__device__ __forceinline__ uint32_t vaddmin(uint32_t a, uint32_t b, uint32_t c) { return __viaddmin_s16x2(a, b, c); }
__device__ __forceinline__ uint32_t vmaxrelu(uint32_t a, uint32_t b) { return __vimax_s16x2_relu(a, b); }
__device__ __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) { return __vmaxs2(a, b); }
__device__ __forceinline__ uint32_t vmax3(uint32_t a, uint32_t b, uint32_t c) { return __vimax3_s16x2(a, b, c); }
__device__ __forceinline__ uint32_t vmax3u(uint32_t a, uint32_t b, uint32_t c) { return __vimax3_u16x2(a, b, c); }
__device__ __forceinline__ uint32_t vmax3relu(uint32_t a, uint32_t b, uint32_t c) { return __vimax3_s16x2_relu(a, b, c); }
__device__ __forceinline__ uint32_t vadd(uint32_t a, uint32_t b) { return __vadd2(a, b); }
__device__ __forceinline__ uint32_t pack2(int lo, int hi) { return (uint32_t(lo) & 0xFFFFu) | (uint32_t(hi) << 16); }
__device__ __forceinline__ int lo16(uint32_t v) { return int(int16_t(v & 0xFFFF)); }
__device__ __forceinline__ int hi16(uint32_t v) { return int(int16_t(v >> 16)); }

// 8 bases of block w of a packed sequence as nibbles; positions >= len read as 15 (padding)
template <int FMT>
__device__ __forceinline__ uint32_t block_codes(const uint32_t* __restrict__ words, int w, int len) {
    const int valid = len - 8 * w;
    if (valid <= 0) return 0xFFFFFFFFu;
    uint32_t x = load_block8(words, w, FMT);
    if (valid < 8) x |= 0xFFFFFFFFu << (4 * valid);
    return x;
}

// substitution table of one target base t (nibble code) over query codes 0..3, as 4 int8 bytes
__device__ __forceinline__ uint32_t row_table(uint32_t t, int ma, int mm) {
    const uint32_t base = (uint32_t(mm) & 0xFFu) * 0x01010101u;
    if (t >= 4) return base;  // N or padding: never matches
    const uint32_t diff = (uint32_t(ma) ^ uint32_t(mm)) & 0xFFu;
    return base ^ (diff << (8 * t));
}

// the 8 PRMT selectors of one query block for halves A (codes qa) and B (codes qb):
// selector nibbles [a, a|8, b^4, (b^4)|8]; code 15 (padding) becomes a sign-replicating index.
__device__ __forceinline__ void make_selectors(uint32_t qa, uint32_t qb, uint32_t (&sel)[8]) {
    const uint32_t ae = qa & 0x0F0F0F0Fu, ao = (qa >> 4) & 0x0F0F0F0Fu;                     // cols 0,2,4,6 / 1,3,5,7
    const uint32_t be = (qb & 0x0F0F0F0Fu) ^ 0x04040404u, bo = ((qb >> 4) & 0x0F0F0F0Fu) ^ 0x04040404u;
    const uint32_t sae = ae | (ae << 4) | 0x80808080u, sao = ao | (ao << 4) | 0x80808080u;  // [x, x|8] per byte
    const uint32_t sbe = be | (be << 4) | 0x80808080u, sbo = bo | (bo << 4) | 0x80808080u;
    sel[0] = prmt(sae, sbe, 0x0040);
    sel[1] = prmt(sao, sbo, 0x0040);
    sel[2] = prmt(sae, sbe, 0x0051);
    sel[3] = prmt(sao, sbo, 0x0051);
    sel[4] = prmt(sae, sbe, 0x0062);
    sel[5] = prmt(sao, sbo, 0x0062);
    sel[6] = prmt(sae, sbe, 0x0073);
    sel[7] = prmt(sao, sbo, 0x0073);
}

struct HalfInfo {
    int n, m, h0, p;  // p < 0: dummy half
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
// the same copies to a 32-bit shared-space address (computed once per strip: no per-step
// generic-to-shared conversion, whose S2UR of the CTA id was a per-step stall in ncu)
__device__ __forceinline__ void cp_async16s(uint32_t s, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4s(uint32_t s, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void st_global16(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// base + i * stride (bytes) as one mad.wide: a 32-bit index into a 64-bit pointer without the
// 64-bit add chain (signed: banded strips address rows relative to a base step and may step below it)
template <typename T>
__device__ __forceinline__ T* wide_at(T* base, int32_t i, uint32_t stride_bytes) {
    uint64_t r;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(i), "r"(stride_bytes), "l"(reinterpret_cast<uint64_t>(base)));
    return reinterpret_cast<T*>(r);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// nibble codes of block w from a staged packed word (FMT 4: the word; FMT 2: half of word w/2),
// with positions >= len as padding 15 (same contract as block_codes)
template <int FMT>
__device__ __forceinline__ uint32_t staged_codes(uint32_t word, int w, int len) {
    const int valid = len - 8 * w;
    if (valid <= 0) return 0xFFFFFFFFu;
    uint32_t x = word;
    if (FMT == SALOBA_PACK2) {
        const uint32_t h = word >> ((w & 1) * 16);
        x = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) x |= ((h >> (2 * c)) & 3u) << (4 * c);
    }
    if (valid < 8) x |= 0xFFFFFFFFu << (4 * valid);
    return x;
}

// Pass-2 hit search in one column of R rows (R <= 16): bit r of the low half / bit 16+r of the
// high half of the result is set where row r equals the half's target (one VSETP-class compare and
// one LOP3 per row for both halves).
__device__ __forceinline__ uint32_t eq_bits(uint32_t h, uint32_t target, int r) {
    return __vcmpeq2(h, target) & (0x00010001u << r);
}
// fold one column's hit bits into the first-hit-in-row-major-order record (rows first, then columns)
__device__ __forceinline__ void take_hit(uint32_t bits, int col, int rA, int rB, int (&hit)[4]) {
    const uint32_t mA = bits & 0xFFFFu, mB = bits >> 16;
    if (mA) {
        const int r = rA + __ffs(mA) - 1;
        if (r < hit[0] || (r == hit[0] && col < hit[1])) {
            hit[0] = r;
            hit[1] = col;
        }
    }
    if (mB) {
        const int r = rB + __ffs(mB) - 1;
        if (r < hit[2] || (r == hit[2] && col < hit[3])) {
            hit[2] = r;
            hit[3] = col;
        }
    }
}

}  // namespace saloba
