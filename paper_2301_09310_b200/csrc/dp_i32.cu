// dp_i32.cu — A3 (int32 exact path): anti-diagonal wavefront DP over a subwarp of G lanes per pair.
//
// Decomposition (§IV-A): the DP table is cut into 8x8-cell
// blocks (one packed word of each sequence).  A strip is a row of blocks (8 target
// rows); a chunk is G strips, one per lane.  At step s lane k computes block (strip k, column
// w = s - k), so a chunk takes Q + G - 1 steps ("Q + 31" for G = 32).
// Dependencies (Fig. 4(c)): the left column (H, E of 8 rows) and the top-left
// corner stay in registers; the top row (H, F of 8 columns) comes from lane k-1's previous step
// through __shfl_up_sync (the paper used shared memory; §VII-A found them equivalent).
// Only chunk-bottom rows leave the SM: lane G-1 writes them to a per-subwarp spill row
// that lane 0 of the next chunk reads (double-buffered by chunk parity).
//
// Best-cell tracking is exact and in-pass: per row, a strict '>' keeps the first column reaching
// the row maximum; chunk end reduces rows -> lanes (lexicographic value desc, i asc, j asc) and a
// strict '>' across chunks keeps the earliest rows.
// This path handles everything (N anywhere, both modes, the full int32 envelope of S:151) and is
// the route for pairs the int16x2 path cannot take.
//
// BAND (reading 16): only cells |i - j| <= w are in the table, the
// rest read as 0.  Lane k of chunk c (rows r0..r0+7) computes only blocks [blo, bhi] of columns
// that meet the band; the chunk's step loop covers just the union of its lanes' ranges (so the
// work is ~ rows x (2w + 8) instead of rows x n), plus one non-computing visit to block blo - 1
// that delivers the top-left corner.  A lane that does not compute a block passes an all-zero
// bottom row to the lane below (out-of-band cells are 0), lane 0 reads the previous chunk's spilled
// row only where that chunk computed it, and blocks crossing the band edge mask their cells.
#include <climits>

#include "common.cuh"

namespace saloba {

__device__ __forceinline__ uint32_t prmt32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// FAST (every call whose scores fit int8; pairs whose values could reach 2^28 go to bin 7, which
// runs FAST = false): the substitution is one PRMT from a per-row int8 table over the query codes,
// sign-extended to 32 bits (query N / padding select the second source, a `mismatch` byte); the
// EXTEND dead-zero rule is min(hdiag + s, lambda*hdiag) (one VIADDMNMX, lambda = 2^k >= match+1,
// as in dp_i16.cu); E is kept one column ahead and H = max3relu(D, E, F) (DPX, as dp_i16.cu); and
// the per-row best is tracked per step on packed keys D*9 + (7 - x) (an IMAD, one 3-input max per
// two cells, then one compare per row per step) instead of compare + 2 selects per cell.  Same
// results: max value, first (smallest) column within the row.
template <int G, int MODE, bool BAND, bool FAST>
__global__ void __launch_bounds__(BLOCK_THREADS) dp_i32_kernel(AlignArgs a, int bin) {
    const int lane = threadIdx.x & 31;
    const int k = lane & (G - 1);
    const int sub_base = lane & ~(G - 1);
    const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << sub_base);
    {   // blocks the bin cannot use exit before claiming a spill slot (empty bins: every block)
        const int per_block = BLOCK_THREADS / G;  // pairs one grab-round of a block takes
        if (int64_t(blockIdx.x) * per_block >= int64_t(a.bin_start[bin + 1] - a.bin_start[bin])) return;
    }
    const int bslot = acquire_block_slot(a.slot_bitmap, a.slot_words);
    int32_t* const spill = a.spill + bslot * a.block_slot_words + (threadIdx.x / G) * 4 * a.spill_stride;

    const int start = a.bin_start[bin];
    const int cnt = a.bin_start[bin + 1] - start;
    const int al = a.alpha, be = a.beta, ma = a.match, mm = a.mismatch;

    for (;;) {
        int item = 0;
        if (k == 0) item = atomicAdd(a.bin_counter + bin, 1);
        item = __shfl_sync(mask, item, 0, G);
        if (item >= cnt) break;
        const int p = int(a.perm[start + item]);
        const int n = a.q_len[p], m = a.t_len[p];
        const int h0 = MODE ? a.h0[p] : 0;
        const uint32_t* __restrict__ qw = a.q_words + a.q_word_off[p];
        const uint32_t* __restrict__ tw = a.t_words + a.t_word_off[p];
        const int Q = (n + 7) >> 3, strips = (m + 7) >> 3, chunks = (strips + G - 1) / G;
        const int wb = BAND ? a.band_w[p] : 0;  // band half-width (>= 0, validated by classify)

        int bestv = MODE ? h0 : 0, besti = MODE ? -1 : 0, bestj = MODE ? -1 : 0;

        for (int c = 0; c < chunks; ++c) {
            const int strip = c * G + k, r0 = strip * 8;
            const int32_t* rdH = spill + ((c & 1) ^ 1) * 2 * a.spill_stride;
            const int32_t* rdF = rdH + a.spill_stride;
            int32_t* wrH = spill + (c & 1) * 2 * a.spill_stride;
            int32_t* wrF = wrH + a.spill_stride;

            // target codes of my 8 rows; rows past m and N never match (0xFF)
            const uint32_t tword = (strip < strips) ? load_block8(tw, strip, a.fmt) : 0u;
            int tc[8];
            uint32_t tab[FAST ? 8 : 1];  // FAST: int8 scores of row r against query codes 0..3
            const uint32_t mmb = (uint32_t(mm) & 0xFFu) * 0x01010101u;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int code = nib(tword, r);
                tc[r] = (r0 + r < m && code < 4) ? code : 0xFF;
                if constexpr (FAST)
                    tab[r] = tc[r] == 0xFF ? mmb : mmb ^ (((uint32_t(ma) ^ uint32_t(mm)) & 0xFFu) << (8 * tc[r]));
            }
            uint32_t lam = 2;
            while (int(lam) < ma + 1) lam <<= 1;
            int Hl[8], El[8], bv[8], bc[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                Hl[r] = MODE ? max(0, h0 - al - be * (r0 + r)) : 0;  // H(i,-1)
                El[r] = FAST ? max(Hl[r] - al, -be) : 0;              // FAST: E(i,0); else E(i,-1)
                bv[r] = MODE ? h0 : 0;                                // only cells beating this count
                bc[r] = -1;
            }
            int corner = MODE ? (r0 == 0 ? h0 : max(0, h0 - al - be * (r0 - 1))) : 0;  // H(r0-1, -1)
            int botH[8], botF[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) botH[x] = botF[x] = 0;

            // blocks of columns my rows meet inside the band (all of [0, Q) without a band), the
            // previous chunk's last lane's upper block (its spilled row ends there), and the step
            // range of the chunk: lane 0's first block - 1 (corner visit) .. lane G-1's last block
            // Spill rows are indexed relative to the reading chunk's first block (roff for the row
            // I read, woff for the row lane G-1 writes), so a banded row needs ~(2w + 8)/8 + 3
            // blocks of capacity whatever the query length.
            int blo = 0, bhi = Q - 1, bhi_prev = Q - 1, s_begin = 0, s_end = Q + G - 1, roff = 0, woff = 0;
            if (BAND) {
                blo = max(0, r0 - wb) >> 3;
                bhi = min(Q - 1, (r0 + 7 + wb) >> 3);
                bhi_prev = min(Q - 1, (c * G * 8 - 1 + wb) >> 3);
                const int c0 = c * G * 8, c1 = min(m - 1, c0 + G * 8 - 1);
                s_begin = max(0, (max(0, c0 - wb) >> 3) - 1);
                s_end = min(Q - 1, (c1 + wb) >> 3) + G;  // exclusive
                roff = s_begin;
                woff = max(0, (max(0, c0 + G * 8 - wb) >> 3) - 1);  // s_begin of chunk c + 1
            }
            for (int s = s_begin; s < s_end; ++s) {
                const int w = s - k;
                int topH[8], topF[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    topH[x] = __shfl_up_sync(mask, botH[x], 1, G);
                    topF[x] = __shfl_up_sync(mask, botF[x], 1, G);
                }
                if (k == 0 && w < Q) {
                    if (c == 0) {
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            topH[x] = MODE ? max(0, h0 - al - be * (8 * w + x)) : 0;  // H(-1, j)
                            topF[x] = 0;
                        }
                    } else if (BAND && w > bhi_prev) {  // never written by the previous chunk: out of band
#pragma unroll
                        for (int x = 0; x < 8; ++x) topH[x] = topF[x] = 0;
                    } else {
                        const int4* ph = reinterpret_cast<const int4*>(rdH + 8 * (w - roff));
                        const int4* pf = reinterpret_cast<const int4*>(rdF + 8 * (w - roff));
                        int4 h0v = ph[0], h1v = ph[1], f0v = pf[0], f1v = pf[1];
                        topH[0] = h0v.x; topH[1] = h0v.y; topH[2] = h0v.z; topH[3] = h0v.w;
                        topH[4] = h1v.x; topH[5] = h1v.y; topH[6] = h1v.z; topH[7] = h1v.w;
                        topF[0] = f0v.x; topF[1] = f0v.y; topF[2] = f0v.z; topF[3] = f0v.w;
                        topF[4] = f1v.x; topF[5] = f1v.y; topF[6] = f1v.z; topF[7] = f1v.w;
                    }
                }
                if (BAND && !(w >= blo && w <= bhi && r0 < m)) {
                    // not computed: the corner of my next block (w >= 0: column -1's corner is the
                    // boundary value set before the loop), and zeros for the lane below
                    if (w >= 0) corner = topH[7];
#pragma unroll
                    for (int x = 0; x < 8; ++x) botH[x] = botF[x] = 0;
                    if (w >= 0 && w < blo) {  // left of my band: the column left of block blo is out of
#pragma unroll                                 // band (H = E = 0), not the column -1 boundary
                        for (int r = 0; r < 8; ++r) {
                            Hl[r] = 0;
                            El[r] = FAST ? -be : 0;  // FAST: E(i, 8*blo) = max(0 - alpha, 0 - beta)
                        }
                    }
                    continue;
                }
                if (w >= 0 && w < Q && r0 < m) {
                    const uint32_t qword = load_block8(qw, w, a.fmt);
                    // BAND: does this block cross the band edge? (then cells are masked)
                    const bool edge = BAND && ((r0 + 7) - 8 * w > wb || (8 * w + 7) - r0 > wb);
                    int qc[8];
                    uint32_t sel[FAST ? 8 : 1];
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        qc[x] = (8 * w + x < n) ? nib(qword, x) : 15;
                        if constexpr (FAST) {
                            const uint32_t cx = qc[x] < 4 ? uint32_t(qc[x]) : 4u;  // N / padding -> mismatch byte
                            sel[x] = cx * 0x1111u | 0x8880u;                      // [c, sign, sign, sign]
                        }
                    }
                    int smax[FAST ? 8 : 1];  // FAST: per-row max of h*8 + (7 - x) over this step
#pragma unroll
                    for (int r = 0; r < (FAST ? 8 : 1); ++r) smax[r] = -1;
                    int kprev[FAST ? 8 : 1];
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        int hup = topH[x], fup = topF[x];
                        int hdiag = (x == 0) ? corner : topH[x - 1];
                        const int col = 8 * w + x;
                        int haup = hup - al;  // FAST: H - alpha shared by the next row's F and my E
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            // FAST keeps E one column ahead in El (as dp_i16.cu): e = E(i, j) here
                            const int e = FAST ? El[r] : max(Hl[r] - al, El[r] - be);
                            const int f = FAST ? __viaddmax_s32(fup, -be, haup) : max(hup - al, fup - be);
                            int d;
                            if constexpr (FAST) {
                                const int sc = int(prmt32(tab[r], mmb, sel[x]));
                                d = MODE ? min(hdiag + sc, hdiag * int(lam)) : hdiag + sc;
                            } else {
                                d = hdiag + ((tc[r] == qc[x]) ? ma : mm);
                                if (MODE) d = (hdiag > 0) ? d : 0;
                            }
                            int h = FAST ? __vimax3_s32_relu(d, e, f) : max(max(0, e), max(f, d));
                            int ee = e, ff = f;
                            if (BAND && edge && abs(r0 + r - col) > wb) h = ee = ff = d = 0;  // outside the band
                            const int ha = h - al;
                            if constexpr (FAST) ee = __viaddmax_s32(ee, -be, ha);  // E(i, j+1)
                            if constexpr (FAST) {
                                // keys over D, not H: the best cell is never a gap cell (a gap value is
                                // below the cell it opened from), so the result is unchanged, and D
                                // staying live keeps its add on the FMA pipe (as in dp_i16.cu); *9 is
                                // an IMAD (FMA pipe) where *8 would be an ALU LEA
                                const int key = d * 9 + (7 - x);
                                if (x & 1) smax[r] = max(smax[r], max(kprev[r], key));
                                else kprev[r] = key;
                            } else if (h > bv[r]) {
                                bv[r] = h;
                                bc[r] = col;
                            }
                            hdiag = Hl[r];
                            Hl[r] = h;
                            El[r] = ee;
                            hup = h;
                            haup = ha;
                            fup = ff;
                        }
                        botH[x] = hup;
                        botF[x] = fup;
                    }
                    if constexpr (FAST) {
#pragma unroll
                        for (int r = 0; r < 8; ++r)
                            if (smax[r] > bv[r] * 9 + 8) {  // key / 9 > bv
                                bv[r] = smax[r] / 9;
                                bc[r] = 8 * w + 7 - (smax[r] - 9 * bv[r]);
                            }
                    }
                    corner = topH[7];
                    if (k == G - 1 && c + 1 < chunks) {
                        int4* ph = reinterpret_cast<int4*>(wrH + 8 * (w - woff));
                        int4* pf = reinterpret_cast<int4*>(wrF + 8 * (w - woff));
                        ph[0] = make_int4(botH[0], botH[1], botH[2], botH[3]);
                        ph[1] = make_int4(botH[4], botH[5], botH[6], botH[7]);
                        pf[0] = make_int4(botF[0], botF[1], botF[2], botF[3]);
                        pf[1] = make_int4(botF[4], botF[5], botF[6], botF[7]);
                    }
                }
            }
            // lane best: max value, then smallest row (rows ascend), column already first-max
            int lv = MODE ? h0 : 0, li = INT_MAX, lj = INT_MAX;
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (bc[r] >= 0 && bv[r] > lv) {
                    lv = bv[r];
                    li = r0 + r;
                    lj = bc[r];
                }
            // subwarp reduction: (value desc, i asc, j asc)
#pragma unroll
            for (int off = 1; off < G; off <<= 1) {
                const int ov = __shfl_xor_sync(mask, lv, off, G);
                const int oi = __shfl_xor_sync(mask, li, off, G);
                const int oj = __shfl_xor_sync(mask, lj, off, G);
                const bool take = (ov > lv) || (ov == lv && (oi < li || (oi == li && oj < lj)));
                if (take) {
                    lv = ov;
                    li = oi;
                    lj = oj;
                }
            }
            if (li != INT_MAX && lv > bestv) {
                bestv = lv;
                besti = li;
                bestj = lj;
            }
            __syncwarp(mask);  // spill row written by lane G-1 is read by lane 0 next chunk
        }
        if (k == 0) {
            a.score[p] = bestv;
            a.q_end[p] = bestj;
            a.t_end[p] = besti;
        }
    }
    release_block_slot(a.slot_bitmap, bslot);
}

template <int MODE, bool BAND, bool FAST>
static const void* kptr_mode(int gidx) {
    switch (gidx) {
    case 0: return (const void*)dp_i32_kernel<1, MODE, BAND, FAST>;
    case 1: return (const void*)dp_i32_kernel<2, MODE, BAND, FAST>;
    case 2: return (const void*)dp_i32_kernel<4, MODE, BAND, FAST>;
    case 3: return (const void*)dp_i32_kernel<8, MODE, BAND, FAST>;
    case 4: return (const void*)dp_i32_kernel<16, MODE, BAND, FAST>;
    default: return (const void*)dp_i32_kernel<32, MODE, BAND, FAST>;
    }
}
template <bool FAST>
static const void* kptr_fast(int mode, int gidx, bool band) {
    if (band) return mode == SALOBA_EXTEND ? kptr_mode<1, true, FAST>(gidx) : kptr_mode<0, true, FAST>(gidx);
    return mode == SALOBA_EXTEND ? kptr_mode<1, false, FAST>(gidx) : kptr_mode<0, false, FAST>(gidx);
}
const void* dp_i32_kernel_ptr(int mode, int gidx, bool band, bool fast) {
    return fast ? kptr_fast<true>(mode, gidx, band) : kptr_fast<false>(mode, gidx, band);
}

void launch_dp_i32(int mode, int gidx, int grid, const AlignArgs& a, int bin, cudaStream_t s) {
    // bins 0..5: FAST when the call's scores fit int8; bin I32_WIDE_BIN (G = 32): the plain kernel
    const void* fn = dp_i32_kernel_ptr(mode, gidx, a.band_w != nullptr, bin != I32_WIDE_BIN && a.i32_fast);
    AlignArgs args = a;
    void* params[] = {&args, &bin};
    cudaLaunchKernel(fn, dim3(grid), dim3(BLOCK_THREADS), params, 0, s);
    count_launches(1);
}

}  // namespace saloba
