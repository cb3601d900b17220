// schedule.cu — A2: length-aware scheduler (§III-A P:517-529 load imbalance; §IV-C
// P:688-702 subwarp trade-off; §VII-C P:1743 "dynamic assignment or preprocessing with
// approximate sorting").
//
// Per pair: validate, pick the precision path and the subwarp size G from a lane-step cost model
// (the Q+G-1 ramp of SPEC S:262-279 plus a per-chunk-boundary spill term), then build a 32-bit
// sort key  [bin:4][~min(Q,16383):14][~min(tlen,16383):14]  so that one stable CUB radix sort
// (4 passes; 64-bit keys took 8) groups each bin contiguously,
// longest queries first (LPT order for the persistent kernels' dynamic work queues), and places
// pairs of near-identical shape next to each other (the int16x2 path packs neighbours).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace saloba {

// modelled lane-steps (one step = one 8x8 block on one lane) + spill cost, for group index g
// m: target rows; R: rows per lane.  Lane-steps of 8 x R blocks (the Q+G-1 ramp per chunk), a
// spill term per chunk boundary, and (int16x2) the pass-2 re-run of one chunk.
__host__ __device__ inline float group_cost(int Q, int m, int g, int R, bool repass) {
    const int G = 1 << g;
    const int strips = (m + R - 1) / R;
    const int chunks = (strips + G - 1) / G;
    const float per_chunk = float(Q + G - 1) * float(G) * float(R / 8);
    const float spill = 0.1f * float(chunks - 1) * float(Q);  // write+read of 16 words per block column
    return float(chunks) * per_chunk + spill + (repass ? per_chunk : 0.f);
}

__host__ __device__ inline int choose_gidx(int Q, int m, int force_gidx, int min_gidx, int R, bool repass) {
    if (force_gidx >= 0 && Q <= qmax_for_gidx(force_gidx)) return force_gidx;
    // long queries: every chunk-boundary row is Q*64 B, and with many resident subwarps the rows no
    // longer fit in L2.  Measured on config 4 (B200, round 1): G=16 6.1 TCUPS at 100k pairs, G=8
    // 3.8, G=4 3.4 -> long queries take G >= 16 (the cost model picks 16 or 32).
    if (Q >= LONG_Q) min_gidx = 4;
    int best = NGROUPS - 1;
    float bc = group_cost(Q, m, best, R, repass);
    for (int g = NGROUPS - 2; g >= min_gidx; --g) {
        if (Q > qmax_for_gidx(g)) continue;
        const float c = group_cost(Q, m, g, R, repass);
        if (c < bc) {
            bc = c;
            best = g;
        }
    }
    return best;
}


// int16x2 routing: bit-exact iff every H, E, F fits in int16 — all values lie in
// [-alpha-2beta, B] with B = match*min(m,n) (LOCAL) or h0 + match*min(m,n) (EXTEND); EXTEND also
// forms 2^k*H (2^k >= match+1) for its dead-zero rule.  Queries must be N-free (4-entry tables).
// NEXT-2 banded pairs (int32 path): a chunk of G strips meets only the columns of its rows' band,
// ~ (8G + 2w)/8 blocks, so the Q+G-1 ramp is paid on that width, not on Q.  Banded spill rows are
// indexed relative to the chunk's first block (dp_i32.cu), so G only needs room for
// min(Q, (2w + 8)/8 + 3) blocks.  G >= 2: the int32 kernel at G = 1 measured 3x slower than G = 2
// on B200 (profiles/r01_ablation.json: 0.50 vs 1.49 TCUPS, config 2).
__host__ __device__ inline int choose_gidx_banded(int Q, int m, int w, int force_gidx) {
    const int need = min(Q, (2 * w + 8) / 8 + 3);
    if (force_gidx >= 0 && need <= qmax_for_gidx(force_gidx)) return force_gidx;
    int best = NGROUPS - 1;
    float bc = 3.4e38f;
    for (int g = NGROUPS - 1; g >= 1; --g) {
        if (need > qmax_for_gidx(g)) continue;
        const int G = 1 << g;
        const int chunks = ((m + 7) / 8 + G - 1) / G;
        const int width = min(Q, (8 * G + 2 * w + 7) / 8 + 1);
        const float c = float(chunks) * float(width + G - 1) * float(G) + 0.1f * float(chunks - 1) * float(width);
        if (c < bc) {
            bc = c;
            best = g;
        }
    }
    return best;
}

__device__ inline int i16_eligible(const ClassifyArgs& a, int64_t k, int n, int m) {  // 0: int32, 1: int16x2, 2: int16x2 with N in the query (QN)
    // the int16x2 kernels build their substitution rows as int8 bytes (dp_i16.cu row_table, PRMT
    // sign replication): a call whose match or mismatch does not fit int8 is int32-only
    if (!a.i32_fast) return 0;
    const long long mn = n < m ? n : m;
    long long B = (long long)a.match * mn;
    long long lam = 1;
    if (a.mode == SALOBA_EXTEND) {
        B += a.h0[k];
        lam = 2;
        while (lam < a.match + 1) lam <<= 1;
    }
    if (lam * B + a.match > 32767) return 0;
    if (a.fmt == SALOBA_PACK2) return 1;  // 2-bit sequences cannot hold N
    const uint32_t* w = a.q_words + a.q_word_off[k];
    const int nw = (n + 7) >> 3;
    for (int i = 0; i < nw; ++i) {
        const uint32_t v = __ldg(w + i) ^ 0x44444444u;  // nibble == 4 (N) -> zero nibble
        if ((v - 0x11111111u) & ~v & 0x88888888u) return 2;
    }
    return 1;
}

__global__ void __launch_bounds__(256) classify_kernel(ClassifyArgs a) {
    __shared__ int cnt[NBINS];
    if (threadIdx.x < NBINS) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < a.n; k += int64_t(gridDim.x) * blockDim.x) {
        const int n = a.q_len[k], m = a.t_len[k];
        bool ok = n >= 1 && m >= 1 && n <= MAX_LEN && m <= MAX_LEN && n <= a.max_q_supported;
        if (a.band_w) ok = ok && a.band_w[k] >= 0;
        if (a.mode == SALOBA_EXTEND) {
            const int h = a.h0[k];
            ok = ok && h >= 1 && h <= MAX_H0;
        }
        int bin;
        uint32_t key;
        if (!ok) {
            bin = BIN_SKIP;
            a.score[k] = -1;
            a.q_end[k] = -2;
            a.t_end[k] = -2;
            atomicMin(a.status, (unsigned long long)k);
            key = uint32_t(bin) << 28;
        } else {
            const int Q = (n + 7) >> 3;
            int elig = a.force_path != 1 ? i16_eligible(a, k, n, m) : 0;
            // query N: the QN variant exists for G = 1 and G = 2 (short and mid-length reads)
            bool qn = false;
            int qn_g = 0;
            if (elig == 2) {
                qn_g = choose_gidx(Q, m, a.force_gidx, a.min_gidx, a.i16_rows, true);
                qn = !a.band_w && qn_g <= 1;
                if (!qn) elig = 0;
            }
            // NEXT-2 banded pairs: the int16x2 G = 1 kernel (BAND variant) when the band's spill rows
            // fit its 80-block rows ((2w + 16)/8 + 4 blocks, indexed per strip) and the batch fills the
            // GPU at one lane per pair (min_gidx == 0: G = 1 on a small batch of long reads left 80% of
            // the warps idle, measured 0.5 TCUPS in-band on 20k config-4 pairs; Options.force_path = 2
            // overrides that), else int32 banded
            if (elig == 1 && a.band_w &&
                (a.i16_rows == 8 || (a.min_gidx > 0 && a.force_path != 2) ||
                 min(Q + 1, (2 * min(a.band_w[k], 1 << 20) + 16) / 8 + 4) > qmax_for_gidx(0)))
                elig = 0;
            const int path = elig ? PATH_I16 : PATH_I32;
            int g = (path == PATH_I16 && a.band_w) ? 0
                    : path == PATH_I16 ? choose_gidx(Q, m, a.force_gidx, a.min_gidx, a.i16_rows, true)
                    : a.band_w        ? choose_gidx_banded(Q, m, a.band_w[k], a.force_gidx)
                                      : choose_gidx(Q, m, a.force_gidx, max(1, a.min_gidx), I32_ROWS, false);  // int32 G=1 measured 3x slower than G=2
            if (path == PATH_I16 && !a.band_w && a.force_gidx < 0 && g >= NGROUPS - 2) {
                g = NGROUPS - 1;  // the long bin: G=16 or G=32 decided once it is counted
                atomicMax(a.long_qmax, Q);
            }
            bin = qn ? (qn_g == 0 ? QN_BIN : QN2_BIN) : path * 8 + g;
            if (path == PATH_I32) {
                // FAST int32 kernels pack h*8 + column keys and form lambda*H: values must stay < 2^27
                const long long mn = n < m ? n : m;
                long long B = (long long)a.match * mn, lam = 1;
                if (a.mode == SALOBA_EXTEND) {
                    B += a.h0[k];
                    lam = 2;
                    while (lam < a.match + 1) lam <<= 1;
                }
                if (!a.i32_fast || lam * B + a.match >= (1ll << 27)) bin = I32_WIDE_BIN;
            }
            if (a.keep_order)
                key = uint32_t(bin) << 28;  // stable sort: input order inside the bin
            else
                key = (uint32_t(bin) << 28) | ((16383u - uint32_t(min(Q, 16383))) << 14) |
                      (16383u - uint32_t(min(m, 16383)));  // longest query, then target, first
        }
        a.keys[k] = key;
        a.vals[k] = uint32_t(k);
        atomicAdd(&cnt[bin], 1);
    }
    __syncthreads();
    if (threadIdx.x < NBINS && cnt[threadIdx.x]) atomicAdd(a.bin_count + threadIdx.x, cnt[threadIdx.x]);
}

// Long-bin width.  G=16 has the better throughput (config 4 alone, 88k long pairs: 5.49 vs 5.21
// TCUPS) but twice the per-pair latency of G=32; when the bin holds only a few waves of pairs
// (config 5: 8,950 long pairs among 10M short ones) those long items finish last and G=32 wins
// (4.85 vs 4.16 TCUPS).  Rule: G=16 iff the bin fills >= 4 waves of G=16 subwarps and every query
// fits G=16's spill stride.  cap16 = pairs one G=16 wave holds (2 per subwarp).
// A long bin of fewer than `coop_pairs` pairs (too few duos to keep every SM busy until the longest
// one ends) runs on the cooperative kernel instead (long_gidx = NGROUPS, dp_coop_kernel in dp_i16.cu).
__global__ void bin_scan_kernel(const int32_t* count, int32_t* start, const int32_t* long_qmax, int32_t* long_gidx,
                                int64_t cap16, int force_gidx, int64_t coop_pairs) {
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int b = 0; b < NBINS; ++b) {
            start[b] = acc;
            acc += count[b];
        }
        start[NBINS] = acc;
        const bool g16 = force_gidx < 0 && int64_t(count[LONG_BIN]) >= 4 * cap16 && *long_qmax <= qmax_for_gidx(NGROUPS - 2);
        // (and only for genuinely long queries: a small batch of mid-length reads lifted into the
        // long bin by the latency floor ran 1.6x slower cooperatively, config 3 at 3k pairs)
        const bool coop = force_gidx < 0 && int64_t(count[LONG_BIN]) < coop_pairs && *long_qmax >= LONG_Q;
        *long_gidx = coop ? NGROUPS : g16 ? NGROUPS - 2 : NGROUPS - 1;
    }
}

size_t cub_sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, int(n > 0 ? n : 1), 0, 32);
    return bytes;
}

cudaError_t run_classify_sort(const ClassifyArgs& ca, const SortKV& kv, int32_t* bin_start, int sms,
                              int32_t* long_gidx, int64_t cap16, int64_t coop_pairs, cudaStream_t s) {
    if (ca.n > 0) {
        const int64_t g8 = int64_t(sms) * 8;
        const int grid = int((ca.n + 255) / 256 < g8 ? (ca.n + 255) / 256 : g8);
        classify_kernel<<<grid, 256, 0, s>>>(ca);
        count_launches(1);
        size_t tb = kv.cub_temp_bytes;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(kv.cub_temp, tb, kv.keys_in, kv.keys_out, kv.vals_in,
                                                        kv.vals_out, int(ca.n), 0, 32, s);
        if (e != cudaSuccess) return e;
    }
    bin_scan_kernel<<<1, 32, 0, s>>>(ca.bin_count, bin_start, ca.long_qmax, long_gidx, cap16, ca.force_gidx, coop_pairs);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace saloba
