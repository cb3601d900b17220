// dp_i16.cu — A3 fast path: int16x2 "pair-SIMD" wavefront DP, two passes, exact results.
//
// Same wavefront as dp_i32.cu (§IV-A: 8x8 blocks, a strip of 8 target rows
// per lane, G lanes per chunk, Q + G - 1 steps per chunk, top rows passed lane-to-lane by
// __shfl_up_sync, only chunk-bottom rows spilled), but every 32-bit register holds the same cell
// of TWO pairs (low / high 16 bits), so each sm_100a DPX instruction (VIADDMNMX.S16x2,
// VIMNMX3.S16x2(.RELU), VIADD.16x2) advances two DP tables.  Measured on B200 (tools/intpipe.cu,
// profiles/intpipe_b200.json): VIADDMNMX / VIMNMX3 / PRMT issue on the ALU pipe, VIADD.16x2 and
// IMAD on the FMA-heavy pipe, each 64 lanes/clk/SM; the update below puts 4.5 of its 6.5
// instructions per register on the ALU pipe and 2 on the FMA pipe.  The scheduler sorts
// pairs by shape, so the two halves of a work item have (near-)identical dimensions.
//
// Cell update (Eqs. 1-3), per register = 2 cells:
//     f  = max(f_up - beta, ha_up)          VIADDMNMX   (ha = H - alpha, shared by E and F)
//     e  = max(e_left - beta, ha_left)      VIADDMNMX   (computed one column ahead)
//     s  = PRMT(table_A[row], table_B[row], selector[col])      substitution score (int8 -> int16)
//     d  = h_diag + s                       VIADD.16x2  (FMA pipe; EXTEND: min(d, lambda*h_diag))
//     h  = max(0, d, e, f)                  VIMNMX3.RELU
//     ha = h - alpha                        VIADD.16x2  (FMA pipe)
//     M  = max(M, h, h')                    VIMNMX3     (running maximum, 1 per 2 cells)
//
// Exact end coordinates without per-cell bookkeeping:
//   pass 1 tracks only the running maximum, reduced per chunk; the first chunk that reaches the
//   pair's maximum contains the tie-rule winner (rows grow with the chunk index).
//   The top boundary of that chunk is the previous chunk's spilled bottom row, kept alive by a
//   4-buffer rotation.  Pass 2 recomputes only that chunk from its checkpoint and finds the first
//   cell (row-major) equal to the maximum.  Cost: ~1/chunks of pass 1.
//
// Exactness of the 16-bit lanes is guaranteed by routing (schedule.cu): all H, E, F stay in
// [-alpha-beta, bound] with bound = match*min(m,n) (+h0, x2 in EXTEND) <= 32767 - match.
// Padding: query columns past a half's length use selectors that sign-replicate a table byte,
// giving S in {0, -1}; target rows past its length (and target N) use an all-mismatch table.
// Padding cells are therefore never larger than a valid cell with a strictly smaller row (same
// row: strictly smaller column), so they can neither raise the maximum nor win its tie-break.
// Queries containing N are routed to the int32 path (a 4-entry table has no "never matches" slot).
#include "dp_i16_common.cuh"

namespace saloba {


// raw packed target words of a lane's R-row strip starting at rows rA / rB (no use of the loaded
// values here, so the loads stay in flight until run_chunk consumes them)
template <int R, int FMT>
__device__ __forceinline__ void load_target_raw(const HalfInfo& A, const HalfInfo& B, const uint32_t* twA,
                                                const uint32_t* twB, int rA, int rB, uint32_t (&raw)[R / 4]) {
#pragma unroll
    for (int i = 0; i < R / 8; ++i) {
        const int ba = (rA >> 3) + i, bb = (rB >> 3) + i;
        raw[i] = (8 * ba < A.m) ? __ldg(twA + (FMT == SALOBA_PACK2 ? (ba >> 1) : ba)) : 0u;
        raw[R / 8 + i] = (8 * bb < B.m) ? __ldg(twB + (FMT == SALOBA_PACK2 ? (bb >> 1) : bb)) : 0u;
    }
}

// Top/bottom rows of one chunk.  topX == nullptr: the table boundary (row -1) for half X.
// Spill rows are interleaved: 16 words per 8-column block, (H0, F0, H1, F1, ..., H7, F7).
struct ChunkIO {
    const uint32_t* topA;  // top row for the low halves (and, outside pass 2, the high halves)
    const uint32_t* topB;  // pass 2: top row for the high halves
    uint32_t* bot;         // nullptr: no spill (last chunk, or pass 2)
};

__device__ __forceinline__ void load8(const uint32_t* p, uint32_t (&v)[8]) {
    const uint4 a = reinterpret_cast<const uint4*>(p)[0], b = reinterpret_cast<const uint4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// One chunk of the wavefront for both halves.  PASS 1 returns the lane's running maximum of the
// diagonal candidates D (max H = max(0, max D): any positive H not reached through D is a gap value
// strictly below an earlier cell).  PASS 2 searches the first cell equal to `target` per half.
// rowA0 / rowB0: first target row of lane 0 of this chunk in each half (they differ in pass 2).
// Per-block shared-memory stage for cp.async prefetching, STAGE_DEPTH slots (inputs of step s are
// requested during step s - STAGE_DEPTH + 1): the two packed query words of each lane's block, and
// per subwarp the spilled top row(s) of lane 0 (A and, in pass 2, B checkpoint).
constexpr int STAGE_DEPTH = 3;
#ifndef I16_MINB16
#define I16_MINB16 3
#endif
template <int G, int T = I16_THREADS>
struct Stage {
    uint32_t q[STAGE_DEPTH][2][T];
#ifdef SALOBA_NO_BSTAGE
    uint4 top[STAGE_DEPTH][T / G][4];
#else
    uint4 top[4][T / G][4];  // pass 1: slots 0..STAGE_DEPTH-1; pass 2: A rows 0..1, B rows 2..3
#endif  // pass 1: slots 0..STAGE_DEPTH-1; pass 2: A rows 0..1, B rows 2..3
};

// Cooperative long-pair kernel (dp_coop_kernel below): a chunk's top row is produced by ANOTHER warp
// of the block while this chunk runs.  `in` is the producer's progress word, `in_tag | blocks` once
// `blocks` bottom-row blocks of the producing task are in global memory; `out` is this chunk's own.
#ifndef COOP_PUB_CFG
#define COOP_PUB_CFG 8
#endif
#ifndef COOP_LAG_CFG
#define COOP_LAG_CFG 16
#endif
constexpr int COOP_PUB = COOP_PUB_CFG;  // bottom-row blocks per progress publication
constexpr int COOP_LAG = COOP_LAG_CFG;  // extra blocks a chunk waits for before its first step
struct CoopIO {
    const volatile unsigned long long* in;
    unsigned long long in_tag;
    volatile unsigned long long* out;
    unsigned long long out_tag;
};

template <int G, int R, int MODE, int FMT, bool PASS2, bool QN = false, bool COOP = false, int T = I16_THREADS>
__device__ __forceinline__ uint32_t run_chunk(const AlignArgs& a, const unsigned mask, const int k, const int Q,
                                              const HalfInfo& A, const HalfInfo& B,
                                              const uint32_t* __restrict__ twA, const uint32_t* __restrict__ twB,
                                              const uint32_t* __restrict__ qwA, const uint32_t* __restrict__ qwB,
                                              const int rowA0, const int rowB0,
                                              const ChunkIO io, const uint32_t target, int (&hit)[4], Stage<G, T>& st,
                                              const int sub, const uint32_t (&twraw)[R / 4],
                                              const CoopIO cio = CoopIO{}) {
    const int al = a.alpha, be = a.beta;
    const uint32_t nbeta = pack2(-be, -be), nalpha = pack2(-al, -al), noGap = pack2(-al - be, -al - be);
    const uint32_t mmw = pack2(a.mismatch, a.mismatch);  // QN: substitution of an N column
    uint32_t lam = 2;
    while (int(lam) < a.match + 1) lam <<= 1;
    const int rA = rowA0 + R * k, rB = rowB0 + R * k;  // my first row in each half (R rows per lane)
    uint32_t tabA[R], tabB[R];
#pragma unroll
    for (int i = 0; i < R / 8; ++i) {
        // twraw: raw target words of my strip, loaded by the caller one chunk ahead
        const uint32_t ta = staged_codes<FMT>(twraw[i], (rA >> 3) + i, A.m);
        const uint32_t tb = staged_codes<FMT>(twraw[R / 8 + i], (rB >> 3) + i, B.m);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            tabA[8 * i + r] = row_table((ta >> (4 * r)) & 15u, a.match, a.mismatch);
            tabB[8 * i + r] = row_table((tb >> (4 * r)) & 15u, a.match, a.mismatch);
        }
    }
    // Left boundary of my strip: H(i,-1), and E(i,0) = max(H(i,-1) - alpha, E(i,-1) - beta) with
    // E(i,-1) taken as "no gap" (only non-positive E values change; they never reach
    // H = max(0, ...): clamp neutrality; same for F(-1, j)); corner H(r0-1, -1).
    uint32_t Hl[R], En[R], corner;
    uint32_t M0 = 0, M1 = 0, M2 = 0, M3 = 0;
    auto reset_left = [&]() {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int ha = MODE ? max(0, A.h0 - al - be * (rA + r)) : 0;
            const int hb = MODE ? max(0, B.h0 - al - be * (rB + r)) : 0;
            Hl[r] = pack2(ha, hb);
            En[r] = vadd(Hl[r], nalpha);
        }
        const int ca = MODE ? (rA == 0 ? A.h0 : max(0, A.h0 - al - be * (rA - 1))) : 0;
        const int cb = MODE ? (rB == 0 ? B.h0 : max(0, B.h0 - al - be * (rB - 1))) : 0;
        corner = pack2(ca, cb);
        M0 = M1 = M2 = M3 = 0;
    };
    reset_left();
    // my bottom row of the previous step (shuffled to the lane below at the start of each step)
    uint32_t botH[8], botF[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) botH[x] = botF[x] = 0;
    // pass 2: candidate columns of one step, parked in local memory (scalar words or quads, below)
    uint32_t colbuf[PASS2 ? 8 : 1][R];
    uint4 colbuf4[PASS2 ? 8 : 1][R / 4];
    const int steps = Q + G - 1;
    // pass 2 stages the B-half checkpoint rows as well, at depth 2 (4 top-row slots per subwarp)
#ifdef SALOBA_NO_BSTAGE
    constexpr int DEPTH = STAGE_DEPTH;
#else
    constexpr int DEPTH = PASS2 ? 2 : STAGE_DEPTH;
#endif
    // Inputs of step s+1 are fetched during step s with cp.async into a 2-slot shared-memory stage
    // (no registers held): every lane's 8 selectors, and on lane 0 the spilled top row(s) of its
    // next block.  Measured (ncu source view) before staging: the lane-0 top-row load was the top
    // stall of the kernel (~23% of samples), because the whole warp waits for it.
#ifdef SALOBA_PROBE_NOSPILL  // perf probe only (wrong results): no spill traffic
    const bool topA_mem = false;
#else
    const bool topA_mem = io.topA != nullptr;
#endif
    const bool topB_mem = PASS2 && io.topB != io.topA && io.topB != nullptr;
    [[maybe_unused]] int avail = 0;  // COOP: top-row blocks known to be published
    auto prefetch = [&](int s2, int slot) {
        const int w2 = s2 - k;
        if (unsigned(w2) < unsigned(Q)) {
            const int wi = FMT == SALOBA_PACK2 ? (w2 >> 1) : w2;
            if (8 * w2 < A.n) cp_async4(&st.q[slot][0][threadIdx.x], qwA + wi);
            if (8 * w2 < B.n) cp_async4(&st.q[slot][1][threadIdx.x], qwB + wi);
            if (k == 0) {
                if (topA_mem) {
                    if constexpr (COOP) {  // block w2 of the producer's bottom row must be in memory
                        if (w2 >= avail) {  // re-read (and fence) only past what is known published
                            // the first wait of a chunk also asks for COOP_LAG blocks of slack, so
                            // the consumer does not trail its producer by less than one batch
                            const int need = min(Q, w2 + 1 + (avail == 0 ? COOP_LAG : 0));
                            unsigned long long v;
                            unsigned ns = 32;
                            while ((v = *cio.in) < (cio.in_tag | unsigned(need))) {
                                __nanosleep(ns);  // a sleeping warp leaves its issue slots to the others
                                ns = min(ns * 2, 1024u);
                            }
                            avail = v >= cio.in_tag + (1ull << 32) ? Q : int(v - cio.in_tag);
                            __threadfence_block();
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) cp_async16(&st.top[slot][sub][q], io.topA + 16 * w2 + 4 * q);
                }
#ifndef SALOBA_NO_BSTAGE
                if (topB_mem) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) cp_async16(&st.top[2 + slot][sub][q], io.topB + 16 * w2 + 4 * q);
                }
#endif
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int p = 0; p < DEPTH - 1; ++p) prefetch(p, p);
    int cur = 0;  // stage slot of step s (s % DEPTH)
    // Every lane takes part in every step's shuffles (warp-uniform loop bounds, full mask); lanes
    // compute only while 0 <= w < Q.
    for (int s = 0; s < steps; ++s) {
        const int w = s - k;
        const bool active = unsigned(w) < unsigned(Q);
        cp_async_wait<DEPTH - 2>();  // this step's stage (issued DEPTH-1 steps ago) has landed
        prefetch(s + DEPTH - 1, cur == 0 ? DEPTH - 1 : cur - 1);
        uint32_t topH[8], topF[8], sel[8];
        if constexpr (G > 1) {  // G == 1: the top row always comes from the spill row / boundary
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                topH[x] = __shfl_up_sync(mask, botH[x], 1, G);
                topF[x] = __shfl_up_sync(mask, botF[x], 1, G);
            }
        }
        const uint32_t qcA = staged_codes<FMT>(st.q[cur][0][threadIdx.x], w, A.n);
        const uint32_t qcB = staged_codes<FMT>(st.q[cur][1][threadIdx.x], w, B.n);
        make_selectors(qcA, qcB, sel);
        // QN: per column, 0xFFFF in each half whose query base is N (nibble 4); those columns take
        // `mismatch` instead of the table byte (N never matches)
        uint32_t nm[QN ? 8 : 1];
        if constexpr (QN) {
            const uint32_t vA = qcA ^ 0x44444444u, vB = qcB ^ 0x44444444u;  // N nibble -> 0
            const uint32_t zA = ~(((vA & 0x77777777u) + 0x77777777u) | vA) & 0x88888888u;
            const uint32_t zB = ~(((vB & 0x77777777u) + 0x77777777u) | vB) & 0x88888888u;
#pragma unroll
            for (int x = 0; x < 8; ++x)
                nm[x] = (((zA >> (4 * x + 3)) & 1u) * 0xFFFFu) | (((zB >> (4 * x + 3)) & 1u) * 0xFFFF0000u);
        }
        if (k == 0 && active) {
            // top row of the chunk: spilled row of the previous chunk, or the table boundary
            if (topA_mem) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 v = st.top[cur][sub][q];
                    topH[2 * q] = v.x; topF[2 * q] = v.y; topH[2 * q + 1] = v.z; topF[2 * q + 1] = v.w;
                }
            } else {
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const int j = 8 * w + x;
                    topH[x] = pack2(MODE ? max(0, A.h0 - al - be * j) : 0, MODE ? max(0, B.h0 - al - be * j) : 0);
                    topF[x] = noGap;
                }
            }
            if (PASS2 && io.topB != io.topA) {  // high halves from half B's own checkpoint
                uint32_t bh[8], bf[8];
                if (topB_mem) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
#ifdef SALOBA_NO_BSTAGE
                        const uint4 v = reinterpret_cast<const uint4*>(io.topB + 16 * w)[q];
#else
                        const uint4 v = st.top[2 + cur][sub][q];
#endif
                        bh[2 * q] = v.x; bf[2 * q] = v.y; bh[2 * q + 1] = v.z; bf[2 * q + 1] = v.w;
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        const int j = 8 * w + x;
                        bh[x] = pack2(0, MODE ? max(0, B.h0 - al - be * j) : 0);
                        bf[x] = noGap;
                    }
                }
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    topH[x] = prmt(topH[x], bh[x], 0x7610);
                    topF[x] = prmt(topF[x], bf[x], 0x7610);
                }
            }
        }
        const int cur_now = cur;
        cur = (cur == DEPTH - 1) ? 0 : cur + 1;
        (void)cur_now;
        if (!active) continue;
        unsigned cand = 0;  // pass 2: columns of this step that may hold `target`
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
                uint32_t sc = prmt(tabA[r], tabB[r], sel[x]);
                if constexpr (QN) sc = (sc & ~nm[x]) | (mmw & nm[x]);
                uint32_t d;
                if (MODE) {
                    // dead-zero (EXTEND): D = hdiag + s if hdiag > 0, else <= 0:
                    // D = min(hdiag + s, lambda * hdiag), lambda = 2^k >= match + 1.  hdiag >= 0 and
                    // lambda * hdiag <= 32767 (routing bound), so one 32-bit IMAD scales both halves.
                    d = vaddmin(hdiag, sc, hdiag * lam);
                } else {
                    d = vadd(hdiag, sc);  // FMA pipe
                }
                const uint32_t h = vmax3relu(d, e, f);
                const uint32_t ha = vadd(h, nalpha);  // FMA pipe
                hdiag = Hl[r];
                Hl[r] = h;
                En[r] = vaddmax(e, nbeta, ha);
                hup = h;
                haup = ha;
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
            botH[x] = hup;
            botF[x] = fup;
            if (PASS2 && active) {
                // column maximum; a cell can only equal `target` (the pair maximum) if it is >= it
                uint32_t cm = vmax3(vmax3(Hl[0], Hl[1], Hl[2]), vmax3(Hl[3], Hl[4], Hl[5]), vmax(Hl[6], Hl[7]));
#pragma unroll
                for (int r = 8; r < R; r += 2) cm = vmax3(cm, Hl[r], Hl[r + 1]);
                // Where the pair maximum may sit in this column (rare per lane): park the column in
                // local memory and scan it after the step, outside the unrolled hot code (ncu: 20%
                // no-instruction stalls in pass 2 with a full scan inlined per column).  Measured
                // on config 2 (B200): LOCAL is fastest with scalar words and a rolled scan (5.16 vs
                // 4.98 TCUPS with quads), EXTEND with quads and an unrolled bit-mask scan (4.55 vs
                // 4.41 scalar); neither order is explained by the SASS, so each mode keeps its best.
                constexpr bool QUADS = MODE == SALOBA_EXTEND;
                if (lo16(cm) >= lo16(target) || hi16(cm) >= hi16(target)) {
                    if (QUADS) {
#pragma unroll
                        for (int q = 0; q < R / 4; ++q)
                            colbuf4[x][q] = make_uint4(Hl[4 * q], Hl[4 * q + 1], Hl[4 * q + 2], Hl[4 * q + 3]);
                    } else {
#pragma unroll
                        for (int r = 0; r < R; ++r) colbuf[x][r] = Hl[r];
                    }
                    cand |= 1u << x;
                }
            }
        }
        if (PASS2 && cand) {
#pragma unroll 1
            for (; cand; cand &= cand - 1) {
                const int x = __ffs(cand) - 1, col = 8 * w + x;
                if (MODE == SALOBA_EXTEND) {
                    uint32_t bits = 0;
#pragma unroll
                    for (int q = 0; q < R / 4; ++q) {
                        const uint4 v = colbuf4[x][q];
                        bits |= eq_bits(v.x, target, 4 * q) | eq_bits(v.y, target, 4 * q + 1) |
                                eq_bits(v.z, target, 4 * q + 2) | eq_bits(v.w, target, 4 * q + 3);
                    }
                    take_hit(bits, col, rA, rB, hit);
                } else {
#pragma unroll 1
                    for (int r = 0; r < R; ++r) {
                        const uint32_t h = colbuf[x][r];
                        if (lo16(h) == lo16(target) && (rA + r < hit[0] || (rA + r == hit[0] && col < hit[1]))) {
                            hit[0] = rA + r;
                            hit[1] = col;
                        }
                        if (hi16(h) == hi16(target) && (rB + r < hit[2] || (rB + r == hit[2] && col < hit[3]))) {
                            hit[2] = rB + r;
                            hit[3] = col;
                        }
                    }
                }
            }
        }
        corner = topH[7];
#ifdef SALOBA_PROBE_NOSPILL
        if (false) {
#else
        if (io.bot && k == G - 1) {  // chunk-bottom row -> spill (interleaved H, F)
#endif
            uint4* p = reinterpret_cast<uint4*>(io.bot + 16 * w);
#pragma unroll
            for (int q = 0; q < 4; ++q) p[q] = make_uint4(botH[2 * q], botF[2 * q], botH[2 * q + 1], botF[2 * q + 1]);
            if constexpr (COOP) {  // publish blocks [0, w] every COOP_PUB blocks (one fence per batch)
                if ((w + 1) % COOP_PUB == 0 || w + 1 == Q) {
                    __threadfence_block();
                    *cio.out = cio.out_tag | unsigned(w + 1);
                }
            }
        }
    }
    return vmax(vmax(M0, M1), vmax(M2, M3));
}

template <int G, int R, int MODE, int FMT, bool QN = false>
__global__ void __launch_bounds__(I16_THREADS, R == 8 ? 4 * 128 / I16_THREADS : I16_MINB16) dp_i16_kernel(AlignArgs a, int bin) {
    // Warp-uniform control flow: a warp takes 32/G consecutive work items at once (one atomic),
    // and runs the warp-maximum of their query blocks and chunk counts; subwarps with a smaller
    // item compute padding (harmless by the dominance argument above).  Shuffles can then use the
    // full mask and compile to plain SHFL (no MATCH/convergence bookkeeping).
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int k = lane & (G - 1);
    const int64_t S = a.spill_stride;
    // per subwarp: 4 spill buffers (interleaved H,F rows of 2S words) inside this block's pool slot
    constexpr int GIDX = G == 1 ? 0 : G == 2 ? 1 : G == 4 ? 2 : G == 8 ? 3 : G == 16 ? 4 : 5;
    if (bin == LONG_BIN && *a.long_gidx != GIDX) return;  // the long bin runs at the other width
    {   // blocks the bin cannot use exit before claiming a spill slot (empty bins: every block)
        const int c0 = a.bin_start[bin], c1 = a.bin_start[bin + 1];
        const int per_block = (I16_THREADS / 32) * (32 / G);  // work items one grab-round of a block takes
        if (int64_t(blockIdx.x) * per_block >= int64_t((c1 - c0 + 1) >> 1)) return;
    }
    const int bslot = acquire_block_slot(a.slot_bitmap, a.slot_words);
    uint32_t* const spill = reinterpret_cast<uint32_t*>(a.spill) + bslot * a.block_slot_words + (threadIdx.x / G) * 8 * S;
    __shared__ Stage<G> st;
    const int sub = threadIdx.x / G;  // subwarp index within the block

    const int start = a.bin_start[bin];
    const int cnt = a.bin_start[bin + 1] - start;
    const int items = (cnt + 1) >> 1;

    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(a.bin_counter + bin, 32 / G);
        base = __shfl_sync(FULL, base, 0);
        if (base >= items) break;
        const int item = base + lane / G;
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
        const int chunksA = ((A.m + R - 1) / R + G - 1) / G, chunksB = ((B.m + R - 1) / R + G - 1) / G;
        const int chunks = max(chunksA, chunksB);
        const int Q = int(__reduce_max_sync(FULL, unsigned(Qi)));        // warp-uniform
        const int chunks_w = int(__reduce_max_sync(FULL, unsigned(chunks)));


        // pass 1 -------------------------------------------------------------------------------
        const int floorA = MODE ? A.h0 : 0, floorB = MODE ? B.h0 : 0;
        int bestA = floorA, bestB = floorB;   // running maxima (strict improvement records chunk)
        int ckA = -1, ckB = -1;               // chunk holding the first maximum (-1: none above floor)
        int bufA = -1, bufB = -1;             // buffer holding that chunk's top row (-1: boundary)
        int rd = -1, wr = 0;
        uint32_t twn[R / 4];
        load_target_raw<R, FMT>(A, B, twA, twB, R * k, R * k, twn);
        for (int c = 0; c < chunks_w; ++c) {
            uint32_t twc[R / 4];
#pragma unroll
            for (int i = 0; i < R / 4; ++i) twc[i] = twn[i];
            if (c + 1 < chunks_w)
                load_target_raw<R, FMT>(A, B, twA, twB, (c + 1) * R * G + R * k, (c + 1) * R * G + R * k, twn);
            const bool last = (c + 1 >= chunks);
            ChunkIO io;
            io.topA = io.topB = rd >= 0 ? spill + (2 * rd) * S : nullptr;
            io.bot = last ? nullptr : spill + (2 * wr) * S;
            int dummy[4];
            uint32_t m = run_chunk<G, R, MODE, FMT, false, QN>(a, FULL, k, Q, A, B, twA, twB, qwA, qwB, c * R * G, c * R * G,
                                                        io, 0u, dummy, st, sub, twc);
#pragma unroll
            for (int off = 1; off < G; off <<= 1) m = vmax(m, __shfl_xor_sync(FULL, m, off, G));
            if (c < chunks) {
                if (lo16(m) > bestA) {
                    bestA = lo16(m);
                    ckA = c;
                    bufA = rd;
                }
                if (hi16(m) > bestB) {
                    bestB = hi16(m);
                    ckB = c;
                    bufB = rd;
                }
            }
            __syncwarp(FULL);
            if (!last) {
                rd = wr;
                // next write buffer: not the new read buffer nor a live checkpoint
                int nw = 0;
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
            ChunkIO io;
            io.topA = bA >= 0 ? spill + (2 * bA) * S : nullptr;
            io.topB = bB >= 0 ? spill + (2 * bB) * S : nullptr;
            io.bot = nullptr;
            const uint32_t target = pack2(ckA >= 0 ? bestA : 0x7FFF, ckB >= 0 ? bestB : 0x7FFF);
            uint32_t tw2[R / 4];
            load_target_raw<R, FMT>(A, B, twA, twB, cA * R * G + R * k, cB * R * G + R * k, tw2);
            run_chunk<G, R, MODE, FMT, true, QN>(a, FULL, k, Q, A, B, twA, twB, qwA, qwB, cA * R * G, cB * R * G, io, target,
                                             hit, st, sub, tw2);
            // first hit in row-major order across the subwarp (rows grow with the lane index)
#pragma unroll
            for (int off = 1; off < G; off <<= 1) {
                const int r0 = __shfl_xor_sync(FULL, hit[0], off, G), c0 = __shfl_xor_sync(FULL, hit[1], off, G);
                const int r1 = __shfl_xor_sync(FULL, hit[2], off, G), c1 = __shfl_xor_sync(FULL, hit[3], off, G);
                if (r0 < hit[0] || (r0 == hit[0] && c0 < hit[1])) {
                    hit[0] = r0;
                    hit[1] = c0;
                }
                if (r1 < hit[2] || (r1 == hit[2] && c1 < hit[3])) {
                    hit[2] = r1;
                    hit[3] = c1;
                }
            }
        }
        __syncwarp(FULL);
        if (a.counters) {  // NEXT-4 instrumentation: one contribution per work item (its lane k = 0)
            const bool it = k == 0 && A.p >= 0;
            const bool p2 = __any_sync(FULL, need2);
            count_warp(a.counters, 0, it ? chunks_w : 0);
            count_warp(a.counters, 1, it ? uint64_t(chunks_w) * (Q + G - 1) : 0);
            count_warp(a.counters, 2, it ? uint64_t(chunks - 1) * Q : 0);
            count_warp(a.counters, 3, it ? uint64_t(chunks_w - 1) * Q : 0);
            count_warp(a.counters, 4, it && p2 ? 1 : 0);
            count_warp(a.counters, 5, it && p2 ? Q + G - 1 : 0);
            count_warp(a.counters, 6, it ? uint64_t(chunks_w) * G : 0);
            count_warp(a.counters, 7, it ? 1 : 0);
        }
        if (k == 0 && A.p >= 0) {
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

// ---- cooperative long-pair kernel (§III-A load imbalance; §IV) ----
// With few long pairs, one warp per pair-duo leaves the GPU waiting on its longest duos: a duo of
// 10 kbp reads is ~20 chunks of 512 rows that one warp runs one after another.  Here a block of
// COOP_W warps shares each duo: chunk c runs on warp c % COOP_W as soon as chunk c-1 (on the
// previous warp) has published the first blocks of its bottom row, so COOP_W chunks of the same duo
// are in flight, staggered, each a G = 32 wavefront (run_chunk).  Per block the work is a stream
// of TASKS: for each duo taken from the long bin, its chunks 0..C-1, then the pass-2 task of the
// PREVIOUS duo; task t runs on warp t % COOP_W.  A pass-2 task placed right after its own duo's
// chunks waited up to a whole chunk for the last of them (ncu: a third of the warps asleep on
// config 4); one duo later, its chunks are done and it overlaps the next duo's chunks.
//   * chunk-boundary rows live in the block's spill slot: task t writes row t % COOP_NROW (COOP_NROW =
//     COOP_W + 1: the next writer of that row is task t + COOP_NROW, which runs on the same warp as the
//     row's only reader, task t + 1, and after it);
//   * progress words (one per warp, (task << 32) | blocks written) order a chunk's reads of its top row
//     after the producer's writes (fence.cta on both sides);
//   * the tie rule needs the running maximum in CHUNK order: a chunk's bookkeeping waits for its
//     predecessor's, and a chunk that raises a half's maximum copies its top row (still intact: its
//     next writer runs on this warp, later) to that half's checkpoint row for pass 2.
// Every wait is on a task with a smaller index, and a warp runs its tasks in index order, so the
// smallest unfinished task can always proceed (no deadlock); all warps of a block are co-resident.
// A warp that needs a new duo descriptor never blocks on the publishing lock while the descriptor
// may still appear: the lock holder can itself be waiting for an older duo's pass 2, whose warp may
// need a descriptor published meanwhile (that cycle hung small batches until it was fixed).
// 8 warps (measured +8.5% over 4 on config 5's 1.25M-pair slice, -2% on config 4 at 4k pairs);
// __maxnreg__(168) leaves room for one block of another bin on the SM.
#ifndef COOP_WARPS
#define COOP_WARPS 8
#endif
constexpr int COOP_W = COOP_WARPS;  // warps per block = chunks of one duo in flight
constexpr int COOP_T = 32 * COOP_W;
constexpr int COOP_NDUO = 3;           // duo descriptors in flight per block (spill slot: (COOP_W + 1 + 2 NDUO) rows)
constexpr int COOP_NROW = COOP_W + 1;  // chunk-boundary rows; checkpoint rows follow (2 per descriptor)
constexpr int COOP_GIDX = NGROUPS;     // long_gidx value that selects this kernel for the long bin

struct CoopDuo {
    int index;       // duo number n this descriptor holds (slot n % COOP_NDUO); -1 while rewritten
    int item;        // work item (pair-duo) index in the bin, -1: the bin is exhausted
    int t0;          // first task of the duo
    int chunks;      // chunk tasks; task t0 + chunks is the pass 2 of the previous duo
    int bestA, bestB, ckA, ckB, bufA, bufB;  // running maxima / first chunk reaching them / its top row
    int done_chunk;  // last chunk whose bookkeeping is complete
    int finished;    // pass 2 done and results written: the descriptor may be reused
};
struct CoopShared {
    unsigned long long prog[COOP_W];
    CoopDuo duo[COOP_NDUO];
    int n_duos;  // descriptors published
    int next_t;  // first task of the next duo
    int lock;
};

__device__ __forceinline__ void coop_halves(const AlignArgs& a, int start, int cnt, int item, HalfInfo& A, HalfInfo& B) {
    A.p = int(a.perm[start + 2 * item]);
    B.p = 2 * item + 1 < cnt ? int(a.perm[start + 2 * item + 1]) : -1;
    A.n = a.q_len[A.p];
    A.m = a.t_len[A.p];
    A.h0 = a.h0 ? a.h0[A.p] : 0;
    B.n = B.p >= 0 ? a.q_len[B.p] : 0;
    B.m = B.p >= 0 ? a.t_len[B.p] : 0;
    B.h0 = (a.h0 && B.p >= 0) ? a.h0[B.p] : 0;
}

template <int MODE, int FMT>
__global__ void __maxnreg__(168) dp_coop_kernel(AlignArgs a, int bin) {
    constexpr int G = 32, R = 16, CH = G * R;  // rows per chunk
    constexpr unsigned FULL = 0xffffffffu;
    if (*a.long_gidx != COOP_GIDX) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int start = a.bin_start[bin];
    const int cnt = a.bin_start[bin + 1] - start;
    const int items = (cnt + 1) >> 1;
    if (int64_t(blockIdx.x) >= int64_t(items)) return;
    const int bslot = acquire_block_slot(a.slot_bitmap, a.slot_words);
    const int64_t S = a.spill_stride;
    uint32_t* const pool = reinterpret_cast<uint32_t*>(a.spill) + bslot * a.block_slot_words;
    auto row = [&](int r) { return pool + int64_t(r) * 2 * S; };
    __shared__ Stage<G, COOP_T> st;
    __shared__ CoopShared cs;
    if (threadIdx.x == 0) {
        cs.n_duos = 0;
        cs.next_t = 0;
        cs.lock = 0;
        for (int i = 0; i < COOP_NDUO; ++i) {
            cs.duo[i].finished = 1;
            cs.duo[i].index = -1;
        }
    }
    if (threadIdx.x < COOP_W) cs.prog[threadIdx.x] = 0;
    __syncthreads();
    volatile CoopShared& vs = cs;

    int n = 0;  // duo of this warp's current task (descriptors are published in task order)
    for (int t = warp;; t += COOP_W) {
        // ---- the descriptor holding task t (lane 0 finds it, publishing new ones under the block
        // lock; the result is broadcast so the warp stays uniform) ----
        int item = -1, t0 = 0, chunks = 0;
        if (lane == 0) {
            for (;;) {
                // Publish up to descriptor n under the lock, unless another warp does it first: a
                // lock holder may wait (below) for an older duo's pass 2, whose warp can need a
                // descriptor published meanwhile, so waiters must not block on the lock itself.
                bool got = false;
                while (n >= vs.n_duos) {
                    if (atomicCAS(&cs.lock, 0, 1) == 0) {
                        got = true;
                        break;
                    }
                    __nanosleep(64);
                }
                if (got) {
                    __threadfence_block();
                    while (vs.n_duos <= n) {
                        const int slot = vs.n_duos % COOP_NDUO;
                        while (!vs.duo[slot].finished) __nanosleep(256);  // duo n_duos - COOP_NDUO still in use
                        const int it = atomicAdd(a.bin_counter + bin, 1);
                        int ch = 0;
                        HalfInfo A{}, B{};
                        if (it < items) {
                            coop_halves(a, start, cnt, it, A, B);
                            ch = max((A.m + CH - 1) / CH, (B.m + CH - 1) / CH);
                        }
                        volatile CoopDuo& d = vs.duo[slot];
                        d.index = -1;
                        __threadfence_block();
                        d.item = it < items ? it : -1;
                        d.t0 = vs.next_t;
                        d.chunks = ch;
                        d.bestA = MODE ? A.h0 : 0;  // the floors (strict improvement records a chunk)
                        d.bestB = MODE ? B.h0 : 0;
                        d.ckA = d.ckB = d.bufA = d.bufB = -1;
                        d.done_chunk = -1;
                        d.finished = it < items ? 0 : 1;
                        vs.next_t = it < items ? vs.next_t + ch + 1 : INT_MAX;
                        __threadfence_block();
                        d.index = vs.n_duos;
                        __threadfence_block();
                        vs.n_duos = vs.n_duos + 1;
                    }
                    __threadfence_block();
                    atomicExch(&cs.lock, 0);
                }
                // A descriptor no longer holding duo n means duo n finished and its slot was reused:
                // this warp's (unfinished) task is in a later duo.  Fields are read between two reads
                // of `index` (the publisher invalidates it first and sets it last).
                const volatile CoopDuo& d = vs.duo[n % COOP_NDUO];
                const int i1 = d.index;
                __threadfence_block();
                item = d.item;
                t0 = d.t0;
                chunks = d.chunks;
                __threadfence_block();
                const int i2 = d.index;
                if (i1 == n && i2 == n && (item < 0 || t <= t0 + chunks)) break;
                ++n;
            }
        }
        n = __shfl_sync(FULL, n, 0);
        item = __shfl_sync(FULL, item, 0);
        t0 = __shfl_sync(FULL, t0, 0);
        chunks = __shfl_sync(FULL, chunks, 0);
        __syncwarp(FULL);
        const int c = t - t0;
        // block of descriptor n: its duo's chunk tasks, then the pass-2 task of duo n - 1 (placed after
        // duo n's chunks, so it rarely waits for duo n - 1's last chunk); the exhausted descriptor's
        // block is that last pass-2 task alone
        if (item < 0 && c > chunks) break;  // the bin is exhausted
        const bool chunk_task = c < chunks;
        if (!chunk_task && n == 0) continue;  // (no duo before the first)
        const int dn = chunk_task ? n : n - 1;  // the duo this task works on
        volatile CoopDuo& d = vs.duo[dn % COOP_NDUO];
        const int ditem = chunk_task ? item : __shfl_sync(FULL, lane == 0 ? d.item : 0, 0);
        HalfInfo A, B;
        coop_halves(a, start, cnt, ditem, A, B);
        if (!MODE) A.h0 = B.h0 = 0;
        const uint32_t* qwA = a.q_words + a.q_word_off[A.p];
        const uint32_t* twA = a.t_words + a.t_word_off[A.p];
        const uint32_t* qwB = B.p >= 0 ? a.q_words + a.q_word_off[B.p] : qwA;
        const uint32_t* twB = B.p >= 0 ? a.t_words + a.t_word_off[B.p] : twA;
        const int Q = (max(A.n, B.n) + 7) >> 3;
        if (chunk_task) {
            // ---- chunk task ----
            ChunkIO io;
            io.topA = io.topB = c > 0 ? row((t - 1) % COOP_NROW) : nullptr;
            io.bot = c + 1 < chunks ? row(t % COOP_NROW) : nullptr;
            const CoopIO cio{&cs.prog[(t - 1 + COOP_W) % COOP_W], (unsigned long long)(t - 1) << 32, &cs.prog[warp],
                             (unsigned long long)t << 32};
            uint32_t tw[R / 4];
            load_target_raw<R, FMT>(A, B, twA, twB, c * CH + R * lane, c * CH + R * lane, tw);
            int dummy[4];
            uint32_t m = run_chunk<G, R, MODE, FMT, false, false, true, COOP_T>(a, FULL, lane, Q, A, B, twA, twB, qwA, qwB,
                                                                        c * CH, c * CH, io, 0u, dummy, st, warp, tw, cio);
#pragma unroll
            for (int off = 1; off < G; off <<= 1) m = vmax(m, __shfl_xor_sync(FULL, m, off));
            // bookkeeping in chunk order (strict improvement keeps the first chunk reaching a maximum)
            int upd = 0;
            if (lane == 0) {
                while (d.done_chunk != c - 1) __nanosleep(128);
                __threadfence_block();
                const int bA = d.bestA, bB = d.bestB;
                upd = (lo16(m) > bA ? 1 : 0) | (B.p >= 0 && hi16(m) > bB ? 2 : 0);
                d.bestA = max(bA, lo16(m));
                d.bestB = max(bB, hi16(m));
            }
            upd = __shfl_sync(FULL, upd, 0);
            const int slot = dn % COOP_NDUO;
            for (int h = 0; h < 2; ++h) {
                if (!(upd & (1 << h))) continue;
                const int ck = COOP_NROW + 2 * slot + h;
                if (c > 0) {  // this chunk's top row becomes the half's checkpoint
                    const uint4* src = reinterpret_cast<const uint4*>(row((t - 1) % COOP_NROW));
                    uint4* dst = reinterpret_cast<uint4*>(row(ck));
                    for (int i = lane; i < 4 * Q; i += 32) dst[i] = __ldcg(src + i);
                }
                if (lane == 0) {
                    if (h == 0) {
                        d.ckA = c;
                        d.bufA = c > 0 ? ck : -1;
                    } else {
                        d.ckB = c;
                        d.bufB = c > 0 ? ck : -1;
                    }
                }
            }
            __syncwarp(FULL);
            if (lane == 0) {
                __threadfence_block();
                d.done_chunk = c;
            }
            __syncwarp(FULL);
        } else {
            // ---- pass-2 task: the first cell (row-major) equal to each half's maximum ----
            int ckA = 0, ckB = 0, bestA = 0, bestB = 0, bufA = 0, bufB = 0;
            if (lane == 0) {
                const int dchunks = d.chunks;
                while (d.done_chunk != dchunks - 1) __nanosleep(256);
                __threadfence_block();
                ckA = d.ckA, ckB = d.ckB, bestA = d.bestA, bestB = d.bestB, bufA = d.bufA, bufB = d.bufB;
            }
            ckA = __shfl_sync(FULL, ckA, 0);
            ckB = __shfl_sync(FULL, ckB, 0);
            bestA = __shfl_sync(FULL, bestA, 0);
            bestB = __shfl_sync(FULL, bestB, 0);
            bufA = __shfl_sync(FULL, bufA, 0);
            bufB = __shfl_sync(FULL, bufB, 0);
            int hit[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
            if (ckA >= 0 || ckB >= 0) {
                const int cA = ckA >= 0 ? ckA : ckB, cB = ckB >= 0 ? ckB : cA;
                const int bA = ckA >= 0 ? bufA : bufB, bB = ckB >= 0 ? bufB : bA;
                ChunkIO io;
                io.topA = bA >= 0 ? row(bA) : nullptr;
                io.topB = bB >= 0 ? row(bB) : nullptr;
                io.bot = nullptr;
                const uint32_t target = pack2(ckA >= 0 ? bestA : 0x7FFF, ckB >= 0 ? bestB : 0x7FFF);
                uint32_t tw2[R / 4];
                load_target_raw<R, FMT>(A, B, twA, twB, cA * CH + R * lane, cB * CH + R * lane, tw2);
                run_chunk<G, R, MODE, FMT, true, false, false, COOP_T>(a, FULL, lane, Q, A, B, twA, twB, qwA, qwB, cA * CH, cB * CH, io, target,
                                                 hit, st, warp, tw2);
#pragma unroll
                for (int off = 1; off < G; off <<= 1) {
                    const int r0 = __shfl_xor_sync(FULL, hit[0], off), c0 = __shfl_xor_sync(FULL, hit[1], off);
                    const int r1 = __shfl_xor_sync(FULL, hit[2], off), c1 = __shfl_xor_sync(FULL, hit[3], off);
                    if (r0 < hit[0] || (r0 == hit[0] && c0 < hit[1])) {
                        hit[0] = r0;
                        hit[1] = c0;
                    }
                    if (r1 < hit[2] || (r1 == hit[2] && c1 < hit[3])) {
                        hit[2] = r1;
                        hit[3] = c1;
                    }
                }
            }
            if (lane == 0) {
                const int z = MODE ? -1 : 0;
                a.score[A.p] = bestA;
                a.t_end[A.p] = ckA >= 0 ? (hit[0] == INT_MAX ? -3 : hit[0]) : z;
                a.q_end[A.p] = ckA >= 0 ? (hit[1] == INT_MAX ? -3 : hit[1]) : z;
                if (B.p >= 0) {
                    a.score[B.p] = bestB;
                    a.t_end[B.p] = ckB >= 0 ? (hit[2] == INT_MAX ? -3 : hit[2]) : z;
                    a.q_end[B.p] = ckB >= 0 ? (hit[3] == INT_MAX ? -3 : hit[3]) : z;
                }
                __threadfence_block();
                d.finished = 1;
            }
            __syncwarp(FULL);
        }
    }
    release_block_slot(a.slot_bitmap, bslot);
}

const void* dp_coop_kernel_ptr(int mode, int fmt) {
    if (mode == SALOBA_EXTEND) return fmt == SALOBA_PACK2 ? (const void*)dp_coop_kernel<1, 2> : (const void*)dp_coop_kernel<1, 4>;
    return fmt == SALOBA_PACK2 ? (const void*)dp_coop_kernel<0, 2> : (const void*)dp_coop_kernel<0, 4>;
}
void launch_dp_coop(int mode, int grid, const AlignArgs& a, cudaStream_t s) {
    const void* fn = dp_coop_kernel_ptr(mode, a.fmt);
    AlignArgs args = a;
    int bin = LONG_BIN;
    void* params[] = {&args, &bin};
    cudaLaunchKernel(fn, dim3(grid), dim3(COOP_T), params, 0, s);
    count_launches(1);
}
int coop_threads() { return COOP_T; }
int coop_rows() { return COOP_NROW + 2 * COOP_NDUO; }  // spill rows (2 x spill_stride words each) per block slot

template <int MODE, int FMT, int R>
static const void* kptr16(int gidx) {
    switch (gidx) {
    case 0: return (const void*)dp_i16_kernel<1, R, MODE, FMT>;
    case 1: return (const void*)dp_i16_kernel<2, R, MODE, FMT>;
    case 2: return (const void*)dp_i16_kernel<4, R, MODE, FMT>;
    case 3: return (const void*)dp_i16_kernel<8, R, MODE, FMT>;
    case 4: return (const void*)dp_i16_kernel<16, R, MODE, FMT>;
    default: return (const void*)dp_i16_kernel<32, R, MODE, FMT>;
    }
}
template <int R>
static const void* kptr16_r(int mode, int gidx, int fmt) {
    if (mode == SALOBA_EXTEND) return fmt == SALOBA_PACK2 ? kptr16<1, 2, R>(gidx) : kptr16<1, 4, R>(gidx);
    return fmt == SALOBA_PACK2 ? kptr16<0, 2, R>(gidx) : kptr16<0, 4, R>(gidx);
}
const void* dp_i16_kernel_ptr(int mode, int gidx, int fmt, int rows) {
    return rows == 8 ? kptr16_r<8>(mode, gidx, fmt) : kptr16_r<16>(mode, gidx, fmt);
}
// QN variant (query contains N): G = 1 (bin QN_BIN) or G = 2 (bin QN2_BIN), PACK4 only (2-bit
// sequences cannot hold N)
template <int G>
static const void* kptr_qn(int mode, int rows) {
    if (rows == 8)
        return mode == SALOBA_EXTEND ? (const void*)dp_i16_kernel<G, 8, 1, 4, true> : (const void*)dp_i16_kernel<G, 8, 0, 4, true>;
    return mode == SALOBA_EXTEND ? (const void*)dp_i16_kernel<G, 16, 1, 4, true> : (const void*)dp_i16_kernel<G, 16, 0, 4, true>;
}
const void* dp_i16_qn_kernel_ptr(int mode, int rows, int gidx) {
    return gidx == 0 ? kptr_qn<1>(mode, rows) : kptr_qn<2>(mode, rows);
}
void launch_dp_i16_qn(int mode, int gidx, int grid, const AlignArgs& a, cudaStream_t s) {
    const void* fn = dp_i16_qn_kernel_ptr(mode, a.i16_rows, gidx);
    AlignArgs args = a;
    int bin = gidx == 0 ? QN_BIN : QN2_BIN;
    void* params[] = {&args, &bin};
    cudaLaunchKernel(fn, dim3(grid), dim3(I16_THREADS), params, 0, s);
    count_launches(1);
}

void launch_dp_i16(int mode, int gidx, int grid, const AlignArgs& a, int bin, cudaStream_t s) {
    const void* fn = dp_i16_kernel_ptr(mode, gidx, a.fmt, a.i16_rows);
    AlignArgs args = a;
    void* params[] = {&args, &bin};
    cudaLaunchKernel(fn, dim3(grid), dim3(I16_THREADS), params, 0, s);
    count_launches(1);
}

}  // namespace saloba
