// dp_g1.cu — A3 for short reads: the int16x2 pair-SIMD DP kernel at subwarp size G = 1.
//
// The scheduler sends every int16x2 pair whose cost model prefers one lane per pair here (config 2:
// all 1M pairs; most of configs 3 and 5).  Same method as dp_i16.cu (§IV-A, P:579-642;
// Eqs. 1-3; two exact passes), specialised for G = 1, where every 16-row
// strip of the target is a chunk of its own and the only inter-strip boundary is the thread's OWN
// spilled bottom row:
//
//   * no shuffles and no Q+G-1 ramp: a chunk is Q steps of one 8-column block each;
//   * PRMT selectors are built once per pair-duo (during chunk 0, from the packed query words) and
//     stored to the thread's scratch as 8 x 16-bit selectors per block ([w][thread]: one warp
//     load is 512 contiguous bytes); later chunks and pass 2 fetch them instead of rebuilding them
//     (~30 fewer ALU instructions per step, ~5% of the step's ALU work);
//   * the shared-memory stage is [slot][quad][thread]: conflict-free LDS.128, one per column pair,
//     issued a pair ahead;
//   * pass 2 tests a candidate column's 16 rows in registers (no local-memory parking).
// Measured on B200, config 2, against the generic kernel at G = 1: DP +0-6% LOCAL,
// +1.5% EXTEND, -2% on config 3's longer reads.  Alternatives measured and not kept: 4 blocks per
// SM (L2 spill-row residency), interleaved spill rows, L2 evict-first/last hints, stage-in at the
// end of the previous step, F/E opened from H directly (shorter dependency chain but one more
// FMA-pipe op per cell: issue-bound), a one-pass keyed maximum (D*128 + position; 2 more FMA-pipe
// ops per cell: issue-bound, -3%).
//
// Cell update per 32-bit register (2 cells, one per pair of the duo): see dp_i16.cu.
// Exactness of the 16-bit lanes is guaranteed by routing (schedule.cu): scores fit int8 and all
// H, E, F stay inside int16 (SURVEY §8(c) reading 8).
#include <cstddef>
#include <type_traits>

#include "dp_i16_common.cuh"

namespace saloba {

constexpr int G1_T = 128;    // threads per block
constexpr int G1_R = 16;     // target rows per strip (two packed target words per half)
#ifndef G1_DEPTH_CFG
#define G1_DEPTH_CFG 4
#endif
constexpr int G1_DEPTH = G1_DEPTH_CFG;  // stage slots in pass 1 (inputs requested DEPTH-1 steps ahead)
constexpr int G1_NBUF = 4;   // spill buffers per thread: read, write, two checkpoints
// Resident blocks per SM: 3.  Not register-bound: the spill rows of all resident threads must stay
// L2-resident between a chunk writing them and the next chunk reading them (reuse distance =
// resident threads x Q x 64 B); measured on B200 (config 2) with 4 blocks per SM the L2 hit rate
// fell and the kernel ran ~6% slower.
constexpr int G1_MINB = 3;

// Scratch words per thread per query block: 8 selector words (4 compact ones when the query has
// no N) + G1_NBUF spill rows of 16 words.
__host__ __device__ constexpr int g1_words_per_block() { return 8 + G1_NBUF * 16; }

// pass-1 stage depth: the QN variant keeps 3 (its 8-word selectors double the selector rows)
template <bool QN>
__host__ __device__ constexpr int g1_depth() { return QN && G1_DEPTH > 3 ? 3 : G1_DEPTH; }
#ifndef G1_ROLL
#define G1_ROLL 1
#endif
// The per-item prologue writes the selectors of every query block to scratch so chunk 0 runs the
// hot strip.  EXTEND also writes its (h0-dependent) boundary top row to a spill buffer; LOCAL's
// boundary row is constant (H = 0, F = "no gap") and is put into the stage once per strip instead.
// Same-box A/B on config 2 (tools/sess_var.sh): EXTEND prologue +1.5% vs chunk 0 in the compact
// generic strip; LOCAL with the boundary row in memory -3.5%, with the constant row +0.5%.
// 3 = that (default); 2 = EXTEND only; 1 = both modes with the row in memory; 0 = neither.
#ifndef G1_PROLOGUE
#define G1_PROLOGUE 3
#endif
template <int MODE>
__host__ __device__ constexpr bool g1_prologue_on() { return G1_PROLOGUE == 1 || G1_PROLOGUE == 3 || (G1_PROLOGUE == 2 && MODE == 1); }
template <int MODE>
__host__ __device__ constexpr bool g1_const_top() { return G1_PROLOGUE == 3 && MODE == 0; }
#ifndef G1_CW2
#define G1_CW2 4  // columns per rolled iteration of the compact pass-2 body
#endif
#ifndef G1_DEPTH2_CFG
#define G1_DEPTH2_CFG 2
#endif
// Per-block stage in dynamic shared memory: ENTRY rows of one uint4 per thread ([entry][G1_T]), so
// thread t owns column t in every layout and pass 1 and pass 2 (a block's threads may be in either)
// can number the rows differently over the same bytes.  Per pass, with D stage slots:
//   sel(slot, h) = slot*NS + h        the step's selectors (QN: 8 words with N flags, NS = 2;
//                                     otherwise 8 compact 16-bit selectors, NS = 1)
//   q(slot)      = D*NS + slot        chunk 0 / banded: the step's packed query words (.x A, .y B)
//   top(slot, q) = D*(NS+1) + 4*slot + q   top-row quads (H[2q], F[2q], H[2q+1], F[2q+1]); pass 2
//                                     stages half B's checkpoint row in slots D..2D-1
template <bool QN>
struct G1Stage {
    static constexpr int D = g1_depth<QN>();  // pass 1
    static constexpr int D2 = G1_DEPTH2_CFG;   // pass 2
    static constexpr int NS = QN ? 2 : 1;
    static constexpr int E1 = D * (NS + 1) + 4 * D, E2 = D2 * (NS + 1) + 8 * D2;
    uint4 e[E1 > E2 ? E1 : E2][G1_T];
};

// Scratch of one thread slot inside the block's pool slot:
//   sel  [Qcap][2][G1_T] uint4          PRMT selectors per query block: 8 x 16 bits in [w][0]
//                                       (QN: 8 words with N flags in bytes 2-3, [w][0..1]); all
//                                       lanes use the same w at once: a warp's load is 512
//                                       contiguous bytes
//   row  [G1_T][G1_NBUF][Qcap][4] uint4 spilled chunk-bottom rows (H, F of 8 columns), contiguous
//                                       per thread.  The buffer rotation differs from lane to lane
//                                       (it follows each lane's checkpoints), so a [buf][w][q][thread]
//                                       interleave shares every 128-byte line between lanes on
//                                       different buffers: measured on B200 it partially wrote lines
//                                       of dead rows and cut the L2 hit rate from 63% to 18% (DRAM
//                                       reads 5x, kernel 30% slower).
struct G1Scratch {
    uint4* sel;
    uint4* row;
    int qcap;
    __device__ __forceinline__ uint4* sel_at(int w, int h) const { return sel + (size_t(w) * 2 + h) * G1_T + threadIdx.x; }
    __device__ __forceinline__ uint4* row_at(int buf, int w, int q) const {
        return row + ((size_t(threadIdx.x) * G1_NBUF + buf) * qcap + w) * 4 + q;
    }
};

// the 4 raw packed target words of a strip starting at rows rA / rB (2 per half)
template <int FMT>
__device__ __forceinline__ void g1_target_raw(const HalfInfo& A, const HalfInfo& B, const uint32_t* twA,
                                              const uint32_t* twB, int rA, int rB, uint32_t (&raw)[4]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int ba = (rA >> 3) + i, bb = (rB >> 3) + i;
        raw[i] = (8 * ba < A.m) ? __ldg(twA + (FMT == SALOBA_PACK2 ? (ba >> 1) : ba)) : 0u;
        raw[2 + i] = (8 * bb < B.m) ? __ldg(twB + (FMT == SALOBA_PACK2 ? (bb >> 1) : bb)) : 0u;
    }
}

// NEXT-2 banded DP (reading 16) on this kernel: the step range of a strip, the spill-row
// index bases and the band half-widths (both halves).  Without a band: [0, Q-1], bases 0.
struct G1Band {
    int s_begin, s_first, s_end;  // steps [s_begin, s_end]; s_begin = s_first - 1 is a corner visit
    int rbaseA, rbaseB;           // index base of the spill row read (per half: pass 2 may split)
    int hiA, hiB;                 // last block the strip above computed; its top row beyond is 0
    int wbase;                    // index base of the spill row written
    uint32_t wpk, nwpk;           // pack2(wA, wB), pack2(-wA, -wB)
};

// BAND: in-band flags of an 8 x 16 block whose top-left cell has i - j = d: bit (r - x + 7) is set
// when |d + r - x| <= w (r - x in [-7, 15]; the block's column x reads bits x .. x + 15 after >> (7 - x))
__device__ __forceinline__ uint32_t band_bits(int d, int w) {
    const int lo = max(-w - d, -7) + 7, hi = min(w - d, 15) + 7;
    return lo > hi ? 0u : ((2u << hi) - 1u) & ~((1u << lo) - 1u);
}

// The step's 8 PRMT selectors from the two packed query words (QN: N flags in bytes 2 / 3 of each
// selector word for half A / B; PRMT reads only the low 16 bits, the compute loop expands them).
template <int FMT, bool QN>
__device__ __forceinline__ void g1_selectors(uint32_t qwordA, uint32_t qwordB, int s, const HalfInfo& A,
                                             const HalfInfo& B, uint32_t (&sel)[8]) {
    const uint32_t qcA = staged_codes<FMT>(qwordA, s, A.n);
    const uint32_t qcB = staged_codes<FMT>(qwordB, s, B.n);
    make_selectors(qcA, qcB, sel);
    if constexpr (QN) {
        const uint32_t vA = qcA ^ 0x44444444u, vB = qcB ^ 0x44444444u;
        const uint32_t zA = ~(((vA & 0x77777777u) + 0x77777777u) | vA) & 0x88888888u;
        const uint32_t zB = ~(((vB & 0x77777777u) + 0x77777777u) | vB) & 0x88888888u;
#pragma unroll
        for (int x = 0; x < 8; ++x)
            sel[x] = (sel[x] & 0xFFFFu) | (((zA >> (4 * x + 3)) & 1u) * 0x00FF0000u) |
                     (((zB >> (4 * x + 3)) & 1u) * 0xFF000000u);
    }
}

// One 16-row strip of both halves.
//   PASS2 = false: returns the lane's maximum of the diagonal candidates D over the strip (max H =
//     max(0, max D): a positive H reached through a gap is strictly below an earlier cell).
//   PASS2 = true: records the first cell (row-major) equal to `target` per half into hit[].
//   selgen: build the selectors from the query words every step (banded strips; unbanded items get
//     theirs from the prologue's scratch).
//   topA / topB: spill buffer of the top row per half (-1: the table boundary); bot: buffer that
//     receives the bottom row (-1: none).
//   HOT: pass 1 without a band (the bulk of the work; chunk 0 reads the prologue's boundary row):
//     compile-time selgen = false and top row from memory, so the step loop carries no boundary or
//     selector-build code.
//   BAND: only cells |i - j| <= w (per half) are in the table; the strip runs steps
//     [bd.s_begin, bd.s_end] (a corner visit + the union of the warp's band blocks), blocks that
//     cross a band edge mask their out-of-band cells to H = E = F = 0, selectors are built every
//     step (no selector scratch), and spill rows are indexed relative to the writing strip's first
//     step so a row needs ~(2w + 16)/8 + 3 blocks whatever the query length.
template <int MODE, int FMT, bool PASS2, bool QN, bool BAND = false, bool HOT = false>
__device__ __forceinline__ uint32_t g1_strip(const AlignArgs& a, const int Q, const HalfInfo& A, const HalfInfo& B,
                                             const uint32_t* __restrict__ qwA, const uint32_t* __restrict__ qwB,
                                             const int rA, const int rB, const int topA, const int topB,
                                             const int bot, const bool selgen_rt, const uint32_t target,
                                             int (&hit)[4], G1Stage<QN>& st, const G1Scratch& sc,
                                             const uint32_t (&twraw)[4], const G1Band& bd) {
    const int tid = threadIdx.x;
    const int al = a.alpha, be = a.beta;
    const uint32_t nbeta = pack2(-be, -be), nalpha = pack2(-al, -al), noGap = pack2(-al - be, -al - be);
    const uint32_t mmw = pack2(a.mismatch, a.mismatch);  // QN: substitution of an N column
    uint32_t lam = 2;
    while (int(lam) < a.match + 1) lam <<= 1;
    uint32_t tabA[G1_R], tabB[G1_R];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t ta = staged_codes<FMT>(twraw[i], (rA >> 3) + i, A.m);
        const uint32_t tb = staged_codes<FMT>(twraw[2 + i], (rB >> 3) + i, B.m);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            tabA[8 * i + r] = row_table((ta >> (4 * r)) & 15u, a.match, a.mismatch);
            tabB[8 * i + r] = row_table((tb >> (4 * r)) & 15u, a.match, a.mismatch);
        }
    }
    // Left boundary H(i,-1) and E one column ahead (E(i,-1) as "no gap": only non-positive E values
    // change, which never reach H = max(0, ...)); corner H(r0-1, -1).
    uint32_t Hl[G1_R], En[G1_R];
#pragma unroll
    for (int r = 0; r < G1_R; ++r) {
        // BAND: H(i, -1) of rows i > w feeds only out-of-band cells; 0 keeps E <= 0 left of the band
        const int ha = MODE && !(BAND && rA + r > int(bd.wpk & 0xFFFFu)) ? max(0, A.h0 - al - be * (rA + r)) : 0;
        const int hb = MODE && !(BAND && rB + r > int(bd.wpk >> 16)) ? max(0, B.h0 - al - be * (rB + r)) : 0;
        Hl[r] = pack2(ha, hb);
        En[r] = vadd(Hl[r], nalpha);
    }
    uint32_t corner;
    {
        const int ca = MODE ? (rA == 0 ? A.h0 : max(0, A.h0 - al - be * (rA - 1))) : 0;
        const int cb = MODE ? (rB == 0 ? B.h0 : max(0, B.h0 - al - be * (rB - 1))) : 0;
        corner = pack2(ca, cb);
    }
    uint32_t M0 = 0, M1 = 0, M2 = 0, M3 = 0;
    constexpr int DEPTH = PASS2 ? G1Stage<QN>::D2 : G1Stage<QN>::D;
    constexpr int NS = G1Stage<QN>::NS;
    constexpr int BOFF = DEPTH;  // pass 2: stage slot of half B's top row = BOFF + slot
    constexpr int Q0 = DEPTH * NS, T0 = DEPTH * (NS + 1);  // first q / top entry rows
    auto ENT = [&](int e) -> uint4& { return st.e[e][tid]; };
    auto TOP = [&](int slot, int q) -> uint4& { return ENT(T0 + slot * 4 + q); };
    static_assert(!HOT || (!PASS2 && !BAND), "HOT is the unbanded pass-1 strip");
    const bool selgen = HOT ? false : selgen_rt;
    const bool topA_mem = (HOT && !g1_const_top<MODE>()) ? true : topA >= 0;
    const bool topB_mem = PASS2 && topB >= 0 && topB != topA;
    const bool split = PASS2 && (topB != topA || rB != rA);  // pass 2 halves at different chunks
    const int s_last = BAND ? bd.s_end : Q - 1;
    // shared-space addresses of this thread's stage entries and the global bases of its rows, once
    // per strip (the per-step generic-to-shared conversion re-read the CTA id: an S2UR stall per step)
    const uint32_t st_s = static_cast<uint32_t>(__cvta_generic_to_shared(&st));
    const uint32_t s_ent = st_s + tid * 16;  // + entry * G1_T*16
    const uint4* const g_sel = sc.sel_at(0, 0);                                 // + s * 2*G1_T*16 B
    const uint4* const g_topA = sc.row_at(topA_mem ? topA : 0, 0, 0);           // + idx * 64 B
    const uint4* const g_topB = sc.row_at(topB_mem ? topB : 0, 0, 0);
    uint4* const g_bot = sc.row_at(bot >= 0 ? bot : 0, 0, 0);
    constexpr uint32_t str64 = 64, str_sel = 2 * G1_T * 16;
    auto prefetch = [&](int s2, int slot) {
        if (s2 <= s_last) {
            if (selgen) {
                const int wi = FMT == SALOBA_PACK2 ? (s2 >> 1) : s2;
                if (8 * s2 < A.n) cp_async4s(s_ent + (Q0 + slot) * (G1_T * 16), qwA + wi);
                if (8 * s2 < B.n) cp_async4s(s_ent + (Q0 + slot) * (G1_T * 16) + 4, qwB + wi);
            } else {
                const uint4* g = wide_at(g_sel, s2, str_sel);
                cp_async16s(s_ent + (slot * NS) * (G1_T * 16), g);
                if (QN) cp_async16s(s_ent + (slot * NS + 1) * (G1_T * 16), g + G1_T);
            }
            if (topA_mem && (!BAND || (s2 <= bd.hiA && s2 >= bd.rbaseA))) {
                const uint4* g = wide_at(g_topA, BAND ? s2 - bd.rbaseA : s2, str64);
#pragma unroll
                for (int q = 0; q < 4; ++q) cp_async16s(s_ent + (T0 + slot * 4 + q) * (G1_T * 16), g + q);
            }
            if (topB_mem && (!BAND || (s2 <= bd.hiB && s2 >= bd.rbaseB))) {
                const uint4* g = wide_at(g_topB, BAND ? s2 - bd.rbaseB : s2, str64);
#pragma unroll
                for (int q = 0; q < 4; ++q) cp_async16s(s_ent + (T0 + (BOFF + slot) * 4 + q) * (G1_T * 16), g + q);
            }
        }
        cp_async_commit();
    };
    const int s0 = BAND ? bd.s_begin : 0;
#pragma unroll
    for (int p = 0; p < DEPTH - 1; ++p) prefetch(s0 + p, p);
    // Stage-in of step s2's inputs (slot `slot`): wait for its cp.async group, write table-boundary
    // top rows into the slot, and read the step's selectors and first top-row quad.  (Issuing this
    // at the end of the previous step instead measured 1-4% slower on B200.)
    uint32_t nq0 = 0, nq1 = 0;
    uint4 nsel0 = make_uint4(0, 0, 0, 0), nsel1 = nsel0, ntq = nsel0, ntb = nsel0;
    if (HOT && !topA_mem) {  // constant boundary top row (LOCAL chunk 0): every stage slot, once
        const uint4 cb = make_uint4(0u, noGap, 0u, noGap);
#pragma unroll
        for (int sl = 0; sl < DEPTH; ++sl)
#pragma unroll
            for (int q = 0; q < 4; ++q) TOP(sl, q) = cb;
    }
    auto stage_in = [&](int s2, int slot) {
        cp_async_wait<DEPTH - 2>();
        if (!HOT && !topA_mem) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 8 * s2 + 2 * q;
                // BAND: H(-1, j) of columns j > w feeds only out-of-band cells; 0 keeps F <= 0 above the band
                const int wA = BAND ? int(bd.wpk & 0xFFFFu) : INT_MAX, wB = BAND ? int(bd.wpk >> 16) : INT_MAX;
                const uint32_t h0v = pack2(MODE && j <= wA ? max(0, A.h0 - al - be * j) : 0,
                                           MODE && j <= wB ? max(0, B.h0 - al - be * j) : 0);
                const uint32_t h1v = pack2(MODE && j + 1 <= wA ? max(0, A.h0 - al - be * (j + 1)) : 0,
                                           MODE && j + 1 <= wB ? max(0, B.h0 - al - be * (j + 1)) : 0);
                TOP(slot, q) = make_uint4(h0v, noGap, h1v, noGap);
            }
        }
        if (PASS2 && split && !topB_mem) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 8 * s2 + 2 * q;
                const int wB = BAND ? int(bd.wpk >> 16) : INT_MAX;
                TOP(BOFF + slot, q) = make_uint4(pack2(0, MODE && j <= wB ? max(0, B.h0 - al - be * j) : 0), noGap,
                                                      pack2(0, MODE && j + 1 <= wB ? max(0, B.h0 - al - be * (j + 1)) : 0), noGap);
            }
        }
        if (BAND) {  // top-row blocks the strip above never computed are out of band: H = F = 0
            // (and blocks before the first one it wrote: a split pass 2 starts at the union of both
            // halves' ranges, which can precede one half's row; those are left of its band.  Read as
            // garbage they reached the OTHER half through EXTEND's 32-bit lambda * hdiag IMAD carry.)
            if (topA_mem && (s2 > bd.hiA || s2 < bd.rbaseA)) {
#pragma unroll
                for (int q = 0; q < 4; ++q) TOP(slot, q) = make_uint4(0, 0, 0, 0);
            }
            if (PASS2 && split && topB_mem && (s2 > bd.hiB || s2 < bd.rbaseB)) {
#pragma unroll
                for (int q = 0; q < 4; ++q) TOP(BOFF + slot, q) = make_uint4(0, 0, 0, 0);
            }
        }
        if (selgen) {
            const uint4 qq = ENT(Q0 + slot);
            nq0 = qq.x;
            nq1 = qq.y;
        } else {
            nsel0 = ENT(slot * NS);
            if constexpr (QN) nsel1 = ENT(slot * NS + 1);
        }
        ntq = TOP(slot, 0);
        if (PASS2 && split) ntb = TOP(BOFF + slot, 0);
    };

    int cur = 0;
    for (int s = s0; s <= s_last; ++s) {
        stage_in(s, cur);
        prefetch(s + DEPTH - 1, cur == 0 ? DEPTH - 1 : cur - 1);
        if (BAND && s < bd.s_first) {
            // corner visit of the block left of the band: nothing computed; the corner of the first
            // band block is this block's top-row H at its last column, and the column left of the
            // band is out of band for every row of the strip (H = E = 0)
            const uint4 t3 = TOP(cur, 3);
            corner = t3.z;
            if (PASS2 && split) corner = prmt(corner, TOP(BOFF + cur, 3).z, 0x7610);
#pragma unroll
            for (int r = 0; r < G1_R; ++r) {
                Hl[r] = 0;
                En[r] = nbeta;  // E(i, first band column) = max(0 - alpha, 0 - beta)
            }
            // the block is out of band for every row of the strip: its bottom row is H = F = 0
            // (written, so every block of the row from its base on holds a value)
            if (bot >= 0) {
                uint4* g = wide_at(g_bot, s - bd.wbase, str64);
#pragma unroll
                for (int q = 0; q < 4; ++q) st_global16(g + q, make_uint4(0u, 0u, 0u, 0u));
            }
            cur = (cur == DEPTH - 1) ? 0 : cur + 1;
            continue;
        }
        // BAND: does this block cross a band edge of either half (warp-uniform: then every lane masks)
        bool edge = false;
        uint32_t dpk = 0;
        if (BAND) {
            const int wA = int(bd.wpk & 0xFFFFu), wB = int(bd.wpk >> 16);
            const bool inA = rA + 15 - 8 * s <= wA && 8 * s + 7 - rA <= wA;
            const bool inB = rB + 15 - 8 * s <= wB && 8 * s + 7 - rB <= wB;
            edge = __any_sync(0xffffffffu, !(inA && inB));
            // i - j at (r, x) = (r0 - 8s) + (r - x), clamped far outside any band (int16 halves)
            dpk = pack2(min(max(rA - 8 * s, -16000), 16000), min(max(rB - 8 * s, -16000), 16000));
        }
        uint32_t sel[8];
        if (selgen) {  // banded strips build their selectors every step (no selector scratch)
            g1_selectors<FMT, QN>(nq0, nq1, s, A, B, sel);
            if (!BAND && !g1_prologue_on<MODE>()) {  // chunk 0 without the prologue stores them for later chunks
                if (QN) {
                    *sc.sel_at(s, 0) = make_uint4(sel[0], sel[1], sel[2], sel[3]);
                    *sc.sel_at(s, 1) = make_uint4(sel[4], sel[5], sel[6], sel[7]);
                } else {
                    *sc.sel_at(s, 0) = make_uint4(prmt(sel[0], sel[1], 0x5410), prmt(sel[2], sel[3], 0x5410),
                                                  prmt(sel[4], sel[5], 0x5410), prmt(sel[6], sel[7], 0x5410));
                }
            }
        } else if (QN) {
            sel[0] = nsel0.x; sel[1] = nsel0.y; sel[2] = nsel0.z; sel[3] = nsel0.w;
            sel[4] = nsel1.x; sel[5] = nsel1.y; sel[6] = nsel1.z; sel[7] = nsel1.w;
        } else {
            // odd columns: the high 16 bits, moved down by IMAD.HI (FMA pipe) to spare the ALU pipe
            sel[0] = nsel0.x; sel[1] = __umulhi(nsel0.x, 0x10000u);
            sel[2] = nsel0.y; sel[3] = __umulhi(nsel0.y, 0x10000u);
            sel[4] = nsel0.z; sel[5] = __umulhi(nsel0.z, 0x10000u);
            sel[6] = nsel0.w; sel[7] = __umulhi(nsel0.w, 0x10000u);
        }
        const int slot = cur;
        cur = (cur == DEPTH - 1) ? 0 : cur + 1;
        // the step body: 8 columns x 16 rows fully unrolled, one straight-line block
        uint32_t botH[8], botF[8];
        auto step_body = [&](auto) {
            uint32_t hdiag_top = corner;
            // top-row quads: one conflict-free LDS.128 per column pair, issued a pair ahead
            uint4 tq = ntq, tqn = ntq, tb = ntb, tbn = ntb;
    #pragma unroll
            for (int x = 0; x < 8; ++x) {
                uint32_t hup, fup;
                {
                    if (!(x & 1)) {
                        tq = tqn;
                        if (PASS2 && split) tb = tbn;
                        if (x + 2 < 8) {
                            tqn = TOP(slot, (x >> 1) + 1);
                            if (PASS2 && split) tbn = TOP(BOFF + slot, (x >> 1) + 1);
                        }
                    }
                    hup = (x & 1) ? tq.z : tq.x;
                    fup = (x & 1) ? tq.w : tq.y;
                    if (PASS2 && split) {  // high halves from half B's own checkpoint row
                        hup = prmt(hup, (x & 1) ? tb.z : tb.x, 0x7610);
                        fup = prmt(fup, (x & 1) ? tb.w : tb.y, 0x7610);
                    }
                }
                uint32_t haup = vadd(hup, nalpha);
                uint32_t hdiag = hdiag_top;
                hdiag_top = hup;
                [[maybe_unused]] uint32_t nm = 0;
                if constexpr (QN) nm = prmt(sel[x], 0u, 0x3322);  // 0xFFFF per half whose column is N
                uint32_t dprev = 0;
    #pragma unroll
                for (int r = 0; r < G1_R; ++r) {
                    const uint32_t f = vaddmax(fup, nbeta, haup);
                    const uint32_t e = En[r];
                    uint32_t scv = prmt(tabA[r], tabB[r], sel[x]);
                    if constexpr (QN) scv = (scv & ~nm) | (mmw & nm);
                    uint32_t d;
                    if (MODE) {
                        // dead-zero (EXTEND): D = hdiag + s if hdiag > 0, else <= 0, as
                        // min(hdiag + s, lambda * hdiag) with lambda = 2^k >= match + 1 (one IMAD
                        // scales both halves: hdiag >= 0 and lambda * hdiag <= 32767 by routing)
                        d = vaddmin(hdiag, scv, hdiag * lam);
                    } else {
                        d = vadd(hdiag, scv);
                    }
                    const uint32_t h = vmax3relu(d, e, f);
                    hdiag = Hl[r];
                    Hl[r] = h;
                    En[r] = vaddmax(e, nbeta, vadd(h, nalpha));
                    hup = h;
                    haup = vadd(h, nalpha);
                    fup = f;
                    if (!PASS2) {
                        if (r & 1) {
                            if ((r & 7) == 1) M0 = vmax3(M0, dprev, d);
                            if ((r & 7) == 3) M1 = vmax3(M1, dprev, d);
                            if ((r & 7) == 5) M2 = vmax3(M2, dprev, d);
                            if ((r & 7) == 7) M3 = vmax3(M3, dprev, d);
                        }
                        dprev = d;
                    }
                }
                // chunk-bottom row -> spill, one 16-byte store per column pair (predicated, not branched,
                // so the step stays one basic block)
                botH[x] = hup;
                botF[x] = fup;
                if (PASS2) {
                    // a cell can only equal `target` (the pair maximum) where the column maximum reaches it;
                    // such columns are rare (about one per pair): test their rows in registers
                    uint32_t cm = vmax3(vmax3(Hl[0], Hl[1], Hl[2]), vmax3(Hl[3], Hl[4], Hl[5]), vmax3(Hl[6], Hl[7], Hl[8]));
                    cm = vmax3(cm, vmax3(Hl[9], Hl[10], Hl[11]), vmax3(Hl[12], Hl[13], Hl[14]));
                    cm = vmax(cm, Hl[15]);
                    if (lo16(cm) >= lo16(target) || hi16(cm) >= hi16(target)) {
                        uint32_t bits = 0;
    #pragma unroll
                        for (int r = 0; r < G1_R; ++r) bits |= eq_bits(Hl[r], target, r);
                        take_hit(bits, 8 * s + x, rA, rB, hit);
                    }
                }
            }
            corner = hdiag_top;
        };
        // Band-edge steps take a compact variant (column pairs in a rolled loop: a second fully
        // unrolled body made the step code too large for the instruction cache, ncu: 44% no-instruction
        // stalls).  Only H is masked to 0 out of band: E and F there may hold garbage, which never
        // reaches the band (E moves right, F down: out of band right of / below the band they only
        // leave it; left of / above it H = 0 and the boundary inputs are <= 0, so E, F <= 0 there,
        // and a non-positive E or F never changes any H = max(0, ...) — S:142-143).  The lane maximum
        // tracks the masked H instead of D (same value: max H = max(0, max D)).
        // MASK = false: the same compact body without band masking, for the strips outside the hot
        // pass-1 loop (chunk 0, pass 2; G1_ROLL): their steps are 1/8 of the work, and a second and
        // third fully unrolled body made the kernel's hot code outgrow the instruction cache (ncu:
        // no-instruction stalls at every branch of pass 2's unrolled body)
        // CW columns per rolled iteration (2 or 4): more columns, more independent chains in flight
        auto edge_body = [&](auto mask_tag, auto cw_tag) {
            constexpr bool MASK = decltype(mask_tag)::value;
            constexpr int CW = decltype(cw_tag)::value, NPI = CW / 2;
            const uint32_t wbA = MASK ? band_bits(rA - 8 * s, int(bd.wpk & 0xFFFFu)) : 0u;
            const uint32_t wbB = MASK ? band_bits(rB - 8 * s, int(bd.wpk >> 16)) : 0u;
            uint32_t hdiag_top = corner;
#pragma unroll 1
            for (int p = 0; p < 8 / CW; ++p) {
                uint4 tq[NPI], tb[NPI];
#pragma unroll
                for (int i = 0; i < NPI; ++i) {
                    tq[i] = TOP(slot, NPI * p + i);
                    tb[i] = tq[i];
                    if (PASS2 && split) tb[i] = TOP(BOFF + slot, NPI * p + i);
                }
                uint32_t sx[CW];
#pragma unroll
                for (int xx = 0; xx < CW; ++xx) {
                    sx[xx] = sel[xx];
#pragma unroll
                    for (int k = 1; k < 8 / CW; ++k) sx[xx] = p == k ? sel[CW * k + xx] : sx[xx];
                }
                uint32_t bh[CW], bf[CW];
#pragma unroll
                for (int xx = 0; xx < CW; ++xx) {
                    const int x = CW * p + xx;
                    const uint4 tqp = tq[xx >> 1], tbp = tb[xx >> 1];
                    uint32_t hup = (xx & 1) ? tqp.z : tqp.x, fup = (xx & 1) ? tqp.w : tqp.y;
                    if (PASS2 && split) {
                        hup = prmt(hup, (xx & 1) ? tbp.z : tbp.x, 0x7610);
                        fup = prmt(fup, (xx & 1) ? tbp.w : tbp.y, 0x7610);
                    }
                    const uint32_t selx = sx[xx];
                    // in-band rows of column x: bit r (half A) / bit 16 + r (half B)
                    const uint32_t m = MASK ? prmt(wbA >> (7 - x), wbB >> (7 - x), 0x5410) : 0u;
                    [[maybe_unused]] uint32_t nm = 0;
                    if constexpr (QN) nm = prmt(selx, 0u, 0x3322);  // 0xFFFF per half whose column is N
                    uint32_t haup = vadd(hup, nalpha);
                    uint32_t hdiag = hdiag_top;
                    hdiag_top = hup;
                    uint32_t hprev = 0;
#pragma unroll
                    for (int r = 0; r < G1_R; ++r) {
                        const uint32_t f = vaddmax(fup, nbeta, haup);
                        const uint32_t e = En[r];
                        uint32_t scv = prmt(tabA[r], tabB[r], selx);
                        if constexpr (QN) scv = (scv & ~nm) | (mmw & nm);
                        const uint32_t d = MODE ? vaddmin(hdiag, scv, hdiag * lam) : vadd(hdiag, scv);
                        // bits r and 16 + r moved to the sign bits of the halves, replicated by PRMT
                        uint32_t h = vmax3relu(d, e, f);
                        if constexpr (MASK) h &= prmt(m << (15 - r), 0u, 0xbb99);
                        hdiag = Hl[r];
                        Hl[r] = h;
                        En[r] = vaddmax(e, nbeta, vadd(h, nalpha));
                        hup = h;
                        haup = vadd(h, nalpha);
                        fup = f;
                        if (!PASS2) {
                            if (r & 1) {
                                if ((r & 7) == 1) M0 = vmax3(M0, hprev, h);
                                if ((r & 7) == 3) M1 = vmax3(M1, hprev, h);
                                if ((r & 7) == 5) M2 = vmax3(M2, hprev, h);
                                if ((r & 7) == 7) M3 = vmax3(M3, hprev, h);
                            }
                            hprev = h;
                        }
                    }
                    bh[xx] = hup;
                    bf[xx] = fup;
                    if (PASS2) {
                        uint32_t cm = vmax3(vmax3(Hl[0], Hl[1], Hl[2]), vmax3(Hl[3], Hl[4], Hl[5]), vmax3(Hl[6], Hl[7], Hl[8]));
                        cm = vmax3(cm, vmax3(Hl[9], Hl[10], Hl[11]), vmax3(Hl[12], Hl[13], Hl[14]));
                        cm = vmax(cm, Hl[15]);
                        if (lo16(cm) >= lo16(target) || hi16(cm) >= hi16(target)) {
                            uint32_t bits = 0;
#pragma unroll
                            for (int r = 0; r < G1_R; ++r) bits |= eq_bits(Hl[r], target, r);
                            take_hit(bits, 8 * s + x, rA, rB, hit);
                        }
                    }
                }
                if (bot >= 0) {
#pragma unroll
                    for (int i = 0; i < NPI; ++i)
                        st_global16(wide_at(g_bot, s - bd.wbase, str64) + NPI * p + i,
                                    make_uint4(bh[2 * i], bf[2 * i], bh[2 * i + 1], bf[2 * i + 1]));
                }
            }
            corner = hdiag_top;
        };
        if (BAND && edge) {
            edge_body(std::true_type{}, std::integral_constant<int, 2>{});
        } else if (!HOT && !BAND && G1_ROLL) {
            edge_body(std::false_type{}, std::integral_constant<int, G1_CW2>{});
        } else {
            step_body(std::false_type{});
            if (bot >= 0) {
                uint4* g = wide_at(g_bot, BAND ? s - bd.wbase : s, str64);
#pragma unroll
                for (int q = 0; q < 4; ++q) st_global16(g + q, make_uint4(botH[2 * q], botF[2 * q], botH[2 * q + 1], botF[2 * q + 1]));
            }
        }
    }
    return vmax(vmax(M0, M1), vmax(M2, M3));
}

// Unbanded items (g1_prologue_on), before pass 1: every query block's selectors into the thread's
// scratch and (ROW: EXTEND) the table-boundary top row H(-1, j), F(-1, j) into spill buffer `buf`,
// so that chunk 0 runs the same hot strip as every other chunk instead of building both per step in
// the compact generic strip.
template <int MODE, int FMT, bool QN, bool ROW = true>
__device__ __forceinline__ void g1_prologue(const AlignArgs& a, int Q, const HalfInfo& A, const HalfInfo& B,
                                            const uint32_t* __restrict__ qwA, const uint32_t* __restrict__ qwB,
                                            const G1Scratch& sc, int buf) {
    const int al = a.alpha, be = a.beta;
    const uint32_t noGap = pack2(-al - be, -al - be);
#pragma unroll 4
    for (int s = 0; s < Q; ++s) {
        const int wi = FMT == SALOBA_PACK2 ? (s >> 1) : s;
        const uint32_t qa = 8 * s < A.n ? __ldg(qwA + wi) : 0u, qb = 8 * s < B.n ? __ldg(qwB + wi) : 0u;
        uint32_t sel[8];
        g1_selectors<FMT, QN>(qa, qb, s, A, B, sel);
        if (QN) {
            st_global16(sc.sel_at(s, 0), make_uint4(sel[0], sel[1], sel[2], sel[3]));
            st_global16(sc.sel_at(s, 1), make_uint4(sel[4], sel[5], sel[6], sel[7]));
        } else {  // compact: two 16-bit selectors per word (PRMT reads only the low 16 bits)
            st_global16(sc.sel_at(s, 0), make_uint4(prmt(sel[0], sel[1], 0x5410), prmt(sel[2], sel[3], 0x5410),
                                                    prmt(sel[4], sel[5], 0x5410), prmt(sel[6], sel[7], 0x5410)));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!ROW) break;
            const int j = 8 * s + 2 * q;
            const uint32_t h0v = pack2(MODE ? max(0, A.h0 - al - be * j) : 0, MODE ? max(0, B.h0 - al - be * j) : 0);
            const uint32_t h1v =
                pack2(MODE ? max(0, A.h0 - al - be * (j + 1)) : 0, MODE ? max(0, B.h0 - al - be * (j + 1)) : 0);
            st_global16(sc.row_at(buf, s, q), make_uint4(h0v, noGap, h1v, noGap));
        }
    }
}

// warp-uniform band step range of a strip starting at row r0 (both halves, union over the warp);
// a half without rows in the strip, or a dummy half, contributes nothing
__device__ __forceinline__ void g1_band_range(int rA, int rB, const HalfInfo& A, const HalfInfo& B, int wA, int wB,
                                              int& lo, int& hi) {
    int l = INT_MAX, h = -1;
    if (A.p >= 0 && rA < A.m) {
        l = max(0, rA - wA) >> 3;
        h = min(((A.n + 7) >> 3) - 1, (rA + 15 + wA) >> 3);
    }
    if (B.p >= 0 && rB < B.m) {
        l = min(l, max(0, rB - wB) >> 3);
        h = max(h, min(((B.n + 7) >> 3) - 1, (rB + 15 + wB) >> 3));
    }
    lo = int(__reduce_min_sync(0xffffffffu, unsigned(l)));
    hi = int(__reduce_max_sync(0xffffffffu, unsigned(h + 1))) - 1;
}

template <int MODE, int FMT, bool QN, bool BAND>
__global__ void __launch_bounds__(G1_T, G1_MINB) dp_g1_kernel(AlignArgs a, int bin) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int start = a.bin_start[bin];
    const int cnt = a.bin_start[bin + 1] - start;
    const int items = (cnt + 1) >> 1;  // pair-duos
    // blocks the bin cannot use exit before claiming a scratch slot (empty bins: every block)
    if (int64_t(blockIdx.x) * G1_T >= int64_t(items)) return;
    const int bslot = acquire_block_slot(a.slot_bitmap, a.slot_words);
    G1Scratch sc;
    sc.qcap = int(a.spill_stride);
    {
        uint4* pool = reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(a.spill) + bslot * a.block_slot_words);
        sc.sel = pool;
        sc.row = pool + size_t(sc.qcap) * 2 * G1_T;
    }
    extern __shared__ __align__(16) unsigned char g1_smem[];
    G1Stage<QN>& st = *reinterpret_cast<G1Stage<QN>*>(g1_smem);

    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(a.bin_counter + bin, 32);
        base = __shfl_sync(FULL, base, 0);
        if (base >= items) break;
        const int item = base + lane;
        const bool has = item < items;
        HalfInfo A, B;
        A.p = has ? int(a.perm[start + 2 * item]) : -1;
        B.p = (has && 2 * item + 1 < cnt) ? int(a.perm[start + 2 * item + 1]) : -1;
        A.n = A.p >= 0 ? a.q_len[A.p] : 0;
        A.m = A.p >= 0 ? a.t_len[A.p] : 0;
        A.h0 = (MODE && A.p >= 0) ? a.h0[A.p] : 0;
        B.n = B.p >= 0 ? a.q_len[B.p] : 0;
        B.m = B.p >= 0 ? a.t_len[B.p] : 0;
        B.h0 = (MODE && B.p >= 0) ? a.h0[B.p] : 0;
        const uint32_t* qwA = A.p >= 0 ? a.q_words + a.q_word_off[A.p] : a.q_words;
        const uint32_t* twA = A.p >= 0 ? a.t_words + a.t_word_off[A.p] : a.t_words;
        const uint32_t* qwB = B.p >= 0 ? a.q_words + a.q_word_off[B.p] : qwA;
        const uint32_t* twB = B.p >= 0 ? a.t_words + a.t_word_off[B.p] : twA;
        const int Qi = (max(A.n, B.n) + 7) >> 3;
        const int chunks = max((A.m + G1_R - 1) / G1_R, (B.m + G1_R - 1) / G1_R);
        const int Q = int(__reduce_max_sync(FULL, unsigned(Qi)));  // warp-uniform loop bounds
        const int chunks_w = int(__reduce_max_sync(FULL, unsigned(chunks)));

        const int floorA = MODE ? A.h0 : 0, floorB = MODE ? B.h0 : 0;
        // NEXT-2 band half-widths (clamped: a band past the table is the whole table)
        const int wA = BAND && A.p >= 0 ? min(a.band_w[A.p], 32000) : 32000;
        const int wB = BAND && B.p >= 0 ? min(a.band_w[B.p], 32000) : 32000;
        G1Band bd{0, 0, Q - 1, 0, 0, Q, Q, 0, pack2(wA, wB), pack2(-wA, -wB)};
        int prev_base = 0, prev_hi = -1;     // BAND: the strip above's spill base and last block
        int ckbA = 0, ckbB = 0, ckhA = -1, ckhB = -1;  // BAND: base / last block of each checkpoint
        // pass 1 -------------------------------------------------------------------------------
        int bestA = floorA, bestB = floorB;  // running maxima (strict improvement records the chunk)
        int ckA = -1, ckB = -1;              // chunk holding the first maximum (-1: none above floor)
        int bufA = -1, bufB = -1;            // buffer holding that chunk's top row (-1: boundary)
        int rd = -1, wr = 0;
        if constexpr (!BAND && g1_prologue_on<MODE>()) {
            g1_prologue<MODE, FMT, QN, !g1_const_top<MODE>()>(a, Q, A, B, qwA, qwB, sc, G1_NBUF - 1);
            if (!g1_const_top<MODE>()) rd = G1_NBUF - 1;  // chunk 0's top row: the boundary row just written
        }
        uint32_t twn[4];
        g1_target_raw<FMT>(A, B, twA, twB, 0, 0, twn);
        for (int c = 0; c < chunks_w; ++c) {
            uint32_t twc[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) twc[i] = twn[i];
            if (c + 1 < chunks_w) g1_target_raw<FMT>(A, B, twA, twB, (c + 1) * G1_R, (c + 1) * G1_R, twn);
            const bool last = (c + 1 >= chunks);
            int dummy[4];
            uint32_t m = 0;
            int hi_now = -1;
            bool run = true;
            if (BAND) {
                int lo, hi;
                g1_band_range(c * G1_R, c * G1_R, A, B, wA, wB, lo, hi);
                run = lo <= hi;
                bd.s_first = lo;
                bd.s_begin = max(0, lo - 1);
                bd.s_end = hi;
                bd.wbase = bd.s_begin;
                bd.rbaseA = bd.rbaseB = prev_base;
                bd.hiA = bd.hiB = prev_hi;
                hi_now = run ? hi : -1;
            }
            if (!BAND && (g1_prologue_on<MODE>() || c > 0)) {
                if constexpr (!BAND)
                    m = g1_strip<MODE, FMT, false, QN, false, true>(a, Q, A, B, qwA, qwB, c * G1_R, c * G1_R, rd, rd,
                                                                    last ? -1 : wr, false, 0u, dummy, st, sc, twc, bd);
            } else if (run) {
                m = g1_strip<MODE, FMT, false, QN, BAND>(a, Q, A, B, qwA, qwB, c * G1_R, c * G1_R, rd, rd,
                                                         last ? -1 : wr, true, 0u, dummy, st, sc, twc, bd);
            }
            if (c < chunks) {
                if (lo16(m) > bestA) {
                    bestA = lo16(m);
                    ckA = c;
                    bufA = rd;
                    ckbA = prev_base;
                    ckhA = prev_hi;
                }
                if (hi16(m) > bestB) {
                    bestB = hi16(m);
                    ckB = c;
                    bufB = rd;
                    ckbB = prev_base;
                    ckhB = prev_hi;
                }
            }
            if (BAND) {
                prev_base = bd.wbase;
                prev_hi = hi_now;
            }
            if (!last) {
                rd = wr;
                int nw = 0;  // next write buffer: not the new read buffer nor a live checkpoint
                while (nw == rd || nw == bufA || nw == bufB) ++nw;
                wr = nw;
            }
        }
        // pass 2 -------------------------------------------------------------------------------
        int hit[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
        const bool need2 = ckA >= 0 || ckB >= 0;
        if (__any_sync(FULL, need2)) {
            const int cA = ckA >= 0 ? ckA : (ckB >= 0 ? ckB : 0), cB = ckB >= 0 ? ckB : cA;
            const int bA = ckA >= 0 ? bufA : (ckB >= 0 ? bufB : -1), bB = ckB >= 0 ? bufB : bA;
            const uint32_t target = pack2(ckA >= 0 ? bestA : 0x7FFF, ckB >= 0 ? bestB : 0x7FFF);
            uint32_t tw2[4];
            g1_target_raw<FMT>(A, B, twA, twB, cA * G1_R, cB * G1_R, tw2);
            if (BAND) {
                int lo, hi;
                g1_band_range(cA * G1_R, cB * G1_R, A, B, wA, wB, lo, hi);
                bd.s_first = lo;
                bd.s_begin = max(0, lo - 1);
                bd.s_end = hi;
                bd.rbaseA = ckA >= 0 ? ckbA : ckbB;
                bd.hiA = ckA >= 0 ? ckhA : ckhB;
                bd.rbaseB = ckB >= 0 ? ckbB : bd.rbaseA;
                bd.hiB = ckB >= 0 ? ckhB : bd.hiA;
            }
            if (!BAND || bd.s_first <= bd.s_end)
                g1_strip<MODE, FMT, true, QN, BAND>(a, Q, A, B, qwA, qwB, cA * G1_R, cB * G1_R, bA, bB, -1, BAND, target,
                                                    hit, st, sc, tw2, bd);
        }
        __syncwarp(FULL);
        if (a.counters) {  // NEXT-4 instrumentation (saloba_options.counters)
            const bool it = A.p >= 0;
            const bool p2 = __any_sync(FULL, need2);
            count_warp(a.counters, 0, it ? chunks_w : 0);
            count_warp(a.counters, 1, it ? uint64_t(chunks_w) * Q : 0);
            count_warp(a.counters, 2, it ? uint64_t(chunks - 1) * Q : 0);
            count_warp(a.counters, 3, it ? uint64_t(chunks_w - 1) * Q : 0);
            count_warp(a.counters, 4, it && p2 ? 1 : 0);
            count_warp(a.counters, 5, it && p2 ? Q : 0);
            count_warp(a.counters, 6, it ? chunks_w : 0);
            count_warp(a.counters, 7, it ? 1 : 0);
        }
        if (A.p >= 0) {
            const int z = MODE ? -1 : 0;
            a.score[A.p] = bestA;
            a.t_end[A.p] = ckA >= 0 ? (hit[0] == INT_MAX ? -3 : hit[0]) : z;
            a.q_end[A.p] = ckA >= 0 ? (hit[1] == INT_MAX ? -3 : hit[1]) : z;
            if (B.p >= 0) {
                a.score[B.p] = bestB;
                a.t_end[B.p] = ckB >= 0 ? (hit[2] == INT_MAX ? -3 : hit[2]) : z;
                a.q_end[B.p] = ckB >= 0 ? (hit[3] == INT_MAX ? -3 : hit[3]) : z;
            }
        }
    }
    release_block_slot(a.slot_bitmap, bslot);
}

template <int MODE, bool BAND>
static const void* g1_ptr(int fmt, bool qn) {
    if (qn && !BAND) return (const void*)dp_g1_kernel<MODE, SALOBA_PACK4, true, false>;
    return fmt == SALOBA_PACK2 ? (const void*)dp_g1_kernel<MODE, SALOBA_PACK2, false, BAND>
                               : (const void*)dp_g1_kernel<MODE, SALOBA_PACK4, false, BAND>;
}
// banded calls (NEXT-2) run the BAND variant; query-N pairs of banded calls take the int32 path
const void* dp_g1_kernel_ptr(int mode, int fmt, bool qn, bool band) {
    if (band) return mode == SALOBA_EXTEND ? g1_ptr<1, true>(fmt, false) : g1_ptr<0, true>(fmt, false);
    return mode == SALOBA_EXTEND ? g1_ptr<1, false>(fmt, qn) : g1_ptr<0, false>(fmt, qn);
}
int g1_threads() { return G1_T; }
size_t g1_smem_bytes(bool qn) { return qn ? sizeof(G1Stage<true>) : sizeof(G1Stage<false>); }
// the stage is dynamic shared memory above the 48 KB default: opt every instance in (per device)
void g1_set_smem_attrs() {
    for (int mode = 0; mode < 2; ++mode)
        for (int band = 0; band < 2; ++band)
            for (int fmt : {int(SALOBA_PACK2), int(SALOBA_PACK4)})
                for (int qn = 0; qn < 2; ++qn) {
                    const bool q = qn && !band;
                    cudaFuncSetAttribute(dp_g1_kernel_ptr(mode, fmt, q, band != 0),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(g1_smem_bytes(q)));
                }
}
int64_t g1_scratch_words(int64_t qcap) { return int64_t(G1_T) * g1_words_per_block() * qcap; }

void launch_dp_g1(int mode, int grid, const AlignArgs& a, int bin, bool qn, cudaStream_t s) {
    const void* fn = dp_g1_kernel_ptr(mode, a.fmt, qn, a.band_w != nullptr);
    AlignArgs args = a;
    void* params[] = {&args, &bin};
    cudaLaunchKernel(fn, dim3(grid), dim3(G1_T), params, g1_smem_bytes(qn && a.band_w == nullptr), s);
    count_launches(1);
}

}  // namespace saloba
