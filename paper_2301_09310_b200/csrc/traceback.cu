// traceback.cu — SURVEY §8(f) NEXT-3: CIGAR of LOCAL results (reading 18).
//
// The alignment of a LOCAL result is the global affine (Gotoh) alignment of t[t_start..t_end] x
// q[q_start..q_end] (ends from saloba_align_batch, starts from saloba_locate_start), whose optimum
// equals the local score; among several optimal alignments the one whose op string, read from the
// end, is smallest with M < D < I.  One warp per pair:
//
//   1. anti-diagonal sweep of the region (cell (i, j) of diagonal d = i + j on lane i % 32), the
//      last diagonals of H, E, F in shared memory; every cell leaves a 4-bit direction code:
//        bits 0-1  H source: 0 match/mismatch, 1 F (deletion), 2 E (insertion)  (that preference)
//        bit  2    F state here opens the gap (else it extends): open holds and (extend does not
//                  hold, or state H at (i-1, j) would not continue with an insertion)
//        bit  3    E state here opens the gap (open holds; opening first is never larger)
//      stored in 16x16-cell tiles (128 bytes) so the walk stays inside a tile for ~16 steps;
//   2. lane 0 walks back from (M-1, N-1), emitting ops; the runs are written reversed, then the warp
//      reverses them in place (BAM encoding: (length << 4) | op, M = 0, I = 1, D = 2).
// Regions up to TB_SMEM_ROWS rows and TB_SMEM_CELLS tiled cells live in shared memory; larger ones use the
// warp's slot of the workspace.  Memory-latency / issue bound; not on the bench's hot path.
#include <climits>

#include "common.cuh"

namespace saloba {

constexpr int TB_WARPS = 4;
constexpr int TB_SMEM_ROWS = 256;           // diagonal buffers in shared memory up to this many rows
constexpr int TB_SMEM_CELLS = 32 * 1024;    // direction codes in shared memory (16x16 tiles) up to this many
constexpr int TB_NEG = -(1 << 29);

struct TbWarpSmem {
    int32_t H[3][TB_SMEM_ROWS + 1];
    int32_t E[2][TB_SMEM_ROWS + 1];
    int32_t F[2][TB_SMEM_ROWS + 1];
    uint8_t src[2][TB_SMEM_ROWS + 1];
    uint32_t dir[TB_SMEM_CELLS / 8];
};

struct TbArgs {
    const uint32_t* q_words;
    const int64_t* q_word_off;
    const uint32_t* t_words;
    const int64_t* t_word_off;
    int64_t n_pairs;
    int32_t fmt, match, mismatch, alpha, beta;
    const int32_t *score, *q_start, *q_end, *t_start, *t_end;
    uint32_t* cigar;
    int32_t cap;
    int32_t* n_ops;
    int32_t* counter;
    char* gslot;             // per resident warp: rows words x 7 + src + dir for the largest region
    int64_t gslot_bytes, g_rows, g_cells;
    uint32_t* slot_bitmap;
    int32_t slot_words;
    unsigned long long* status;
};

__device__ __forceinline__ int tb_code_at(const uint32_t* w, int j, int fmt) {
    if (fmt == SALOBA_PACK4) return int((__ldg(w + (j >> 3)) >> (4 * (j & 7))) & 15u);
    return int((__ldg(w + (j >> 4)) >> (2 * (j & 15))) & 3u);
}
// nibble index of cell (i, j) in 16x16 tiles, tiles row-major over ceil(N/16) tile columns
__device__ __forceinline__ int64_t tb_nib(int i, int j, int tcols) {
    return ((int64_t(i >> 4) * tcols + (j >> 4)) << 8) | ((i & 15) << 4) | (j & 15);
}

__global__ void __launch_bounds__(32 * TB_WARPS) traceback_kernel(TbArgs a) {
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char tb_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    TbWarpSmem* sm = reinterpret_cast<TbWarpSmem*>(tb_smem) + warp;
    const int bslot = a.gslot ? acquire_block_slot(a.slot_bitmap, a.slot_words) : -1;
    char* gs = a.gslot ? a.gslot + (int64_t(bslot) * TB_WARPS + warp) * a.gslot_bytes : nullptr;
    const int al = a.alpha, be = a.beta;
    for (int x = lane; x < TB_SMEM_CELLS / 8; x += 32) sm->dir[x] = 0;  // codes are OR-ed in
    __syncwarp(FULL);
    for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(a.counter, 1);
        k = __shfl_sync(FULL, k, 0);
        if (int64_t(k) >= a.n_pairs) break;
        const int sc = a.score[k];
        if (sc <= 0) {  // score 0: no alignment (0 ops); negative: a pair the forward call rejected
            if (lane == 0) a.n_ops[k] = sc == 0 ? 0 : -1;
            continue;
        }
        const int ts = a.t_start[k], te = a.t_end[k], qs = a.q_start[k], qe = a.q_end[k];
        const int M = te - ts + 1, N = qe - qs + 1;
        const int64_t tiled = int64_t((M + 15) >> 4) * ((N + 15) >> 4) * 256;  // nibbles in 16x16 tiles
        const bool in_smem = M <= TB_SMEM_ROWS && tiled <= TB_SMEM_CELLS;
        const bool in_glob = gs && M <= a.g_rows && tiled <= a.g_cells;
        if (ts < 0 || qs < 0 || M < 1 || N < 1 || (!in_smem && !in_glob)) {
            if (lane == 0) {
                a.n_ops[k] = -1;
                atomicMin(a.status, (unsigned long long)k);
            }
            continue;
        }
        int32_t *Hb, *Eb, *Fb;
        uint8_t* Sb;
        uint32_t* dir;
        int rs;  // row stride of the diagonal buffers
        if (in_smem) {
            Hb = &sm->H[0][0]; Eb = &sm->E[0][0]; Fb = &sm->F[0][0]; Sb = &sm->src[0][0]; dir = sm->dir;
            rs = TB_SMEM_ROWS + 1;
        } else {
            rs = int(a.g_rows) + 1;
            Hb = reinterpret_cast<int32_t*>(gs);
            Eb = Hb + 3 * rs;
            Fb = Eb + 2 * rs;
            Sb = reinterpret_cast<uint8_t*>(Fb + 2 * rs);
            dir = reinterpret_cast<uint32_t*>(gs + ((7 * int64_t(rs) * 4 + 2 * rs + 15) & ~int64_t(15)));
        }
        const uint32_t* qw = a.q_words + a.q_word_off[k];
        const uint32_t* tw = a.t_words + a.t_word_off[k];
        const int tcols = (N + 15) >> 4;
        // ---- 1. anti-diagonal sweep --------------------------------------------------------------
        for (int d = 0; d <= M + N - 2; ++d) {
            const int ilo = d - (N - 1) > 0 ? d - (N - 1) : 0, ihi = d < M - 1 ? d : M - 1;
            const int c2 = (d + 1) % 3, c1 = (d + 2) % 3, c0 = d % 3;  // H rows of d-2, d-1, d
            for (int i = ilo + lane; i <= ihi; i += 32) {
                const int j = d - i;
                const int hd = (i > 0 && j > 0) ? Hb[c2 * rs + i - 1]
                               : (i == 0 && j == 0) ? 0
                               : (i == 0) ? -(al + be * (j - 1)) : -(al + be * (i - 1));
                const int hl = j > 0 ? Hb[c1 * rs + i] : -(al + be * i);
                const int el = j > 0 ? Eb[((d - 1) & 1) * rs + i] : TB_NEG;
                const int hu = i > 0 ? Hb[c1 * rs + i - 1] : -(al + be * j);
                const int fu = i > 0 ? Fb[((d - 1) & 1) * rs + i - 1] : TB_NEG;
                const int su = i > 0 ? Sb[((d - 1) & 1) * rs + i - 1] : 0;
                const int tc = tb_code_at(tw, ts + i, a.fmt), qc = tb_code_at(qw, qs + j, a.fmt);
                const int s = (tc == qc && tc < 4) ? a.match : a.mismatch;
                const int eo = hl - al, ex = el - be, fo = hu - al, fx = fu - be;
                const int e = eo > ex ? eo : ex, f = fo > fx ? fo : fx, mm = hd + s;
                int h = mm > e ? mm : e;
                h = h > f ? h : f;
                const int src = h == mm ? 0 : h == f ? 1 : 2;
                const bool fopen = f == fo && (f != fx || su != 2);
                const bool eopen = e == eo;
                Hb[c0 * rs + i] = h;
                Eb[(d & 1) * rs + i] = e;
                Fb[(d & 1) * rs + i] = f;
                Sb[(d & 1) * rs + i] = uint8_t(src);
                const uint32_t code = uint32_t(src) | (fopen ? 4u : 0u) | (eopen ? 8u : 0u);
                const int64_t nb = tb_nib(i, j, tcols);
                atomicOr(&dir[nb >> 3], code << (4 * (nb & 7)));
            }
            __syncwarp(FULL);
        }
        const int gscore = __shfl_sync(FULL, Hb[((M + N - 2) % 3) * rs + M - 1], 0);
        // ---- 2. walk back (lane 0), runs written reversed, then reversed in place ----------------
        uint32_t* out = a.cigar + int64_t(k) * a.cap;
        int nruns = 0;
        bool over = false;
        if (lane == 0) {
            int i = M - 1, j = N - 1, state = 0, cur = -1, len = 0;
            auto emit = [&](int op) {
                if (op == cur) {
                    ++len;
                    return;
                }
                if (cur >= 0) {
                    if (nruns < a.cap) out[nruns] = (uint32_t(len) << 4) | uint32_t(cur);
                    else over = true;
                    ++nruns;
                }
                cur = op;
                len = 1;
            };
            while (i >= 0 || j >= 0) {
                if (i < 0) { emit(1); --j; continue; }
                if (j < 0) { emit(2); --i; continue; }
                const int64_t nb = tb_nib(i, j, tcols);
                const uint32_t code = (dir[nb >> 3] >> (4 * (nb & 7))) & 15u;
                if (state == 0) {
                    const uint32_t src = code & 3u;
                    if (src == 0) { emit(0); --i; --j; }
                    else state = src == 1 ? 1 : 2;
                } else if (state == 1) {
                    emit(2);
                    state = (code & 4u) ? 0 : 1;
                    --i;
                } else {
                    emit(1);
                    state = (code & 8u) ? 0 : 2;
                    --j;
                }
            }
            emit(-1);  // flush the last run
        }
        nruns = __shfl_sync(FULL, nruns, 0);
        over = __shfl_sync(FULL, over ? 1 : 0, 0) != 0;
        __syncwarp(FULL);
        if (!over) {
            for (int x = lane; x < nruns / 2; x += 32) {
                const uint32_t u = out[x], v = out[nruns - 1 - x];
                out[x] = v;
                out[nruns - 1 - x] = u;
            }
        }
        if (lane == 0) {
            a.n_ops[k] = over ? -1 : nruns;
            if (over || gscore != sc) atomicMin(a.status, (unsigned long long)k);
        }
        // clear the direction codes for the next pair (they are OR-ed in)
        const int64_t words = ((int64_t(M + 15) >> 4) * tcols * 256 + 7) >> 3;
        for (int64_t x = lane; x < words; x += 32) dir[x] = 0;
        __syncwarp(FULL);
    }
    if (a.gslot) release_block_slot(a.slot_bitmap, bslot);
}

}  // namespace saloba

using namespace saloba;

namespace {
size_t tb_al256(size_t x) { return (x + 255) / 256 * 256; }
struct TbPlan {
    int sms = 0, blocks = 0;
    int64_t slots = 0, g_rows = 0, g_cells = 0, slot_bytes = 0;
};
TbPlan tb_plan(int32_t max_rows, int32_t max_cols) {
    TbPlan p;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = int(sizeof(TbWarpSmem)) * TB_WARPS;
    cudaFuncSetAttribute(traceback_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.blocks, traceback_kernel, 32 * TB_WARPS, smem);
    if (p.blocks < 1) p.blocks = 1;
    const int64_t R = max_rows > 0 ? max_rows : 1, C = max_cols > 0 ? max_cols : 1;
    const int64_t tiles = ((R + 15) >> 4) * ((C + 15) >> 4);
    if (R > TB_SMEM_ROWS || tiles * 256 > TB_SMEM_CELLS) {  // regions beyond shared memory: global slots
        p.g_rows = R;
        p.g_cells = tiles * 256;
        p.slot_bytes = int64_t(tb_al256(size_t(((7 * (R + 1) * 4 + 2 * (R + 1) + 15) & ~int64_t(15)) + tiles * 128)));
        p.slots = (int64_t(p.sms) * p.blocks + 32 + 31) / 32 * 32;
    }
    return p;
}
}  // namespace

SALOBA_API size_t saloba_traceback_workspace_bytes(int64_t n_pairs, int32_t max_qlen, int32_t max_tlen, int device) {
    if (n_pairs < 0 || max_qlen < 0 || max_tlen < 0) return 0;
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) return 0;
    const TbPlan p = tb_plan(max_tlen, max_qlen);
    cudaSetDevice(prev);
    return 512 + size_t(p.slots) * TB_WARPS * size_t(p.slot_bytes);
}

SALOBA_API int saloba_traceback(const uint32_t* q_words, const int64_t* q_word_off, const uint32_t* t_words,
                                const int64_t* t_word_off, int64_t n_pairs, saloba_scoring sc, saloba_packing fmt,
                                const int32_t* score, const int32_t* q_start, const int32_t* q_end,
                                const int32_t* t_start, const int32_t* t_end, int32_t max_qlen, int32_t max_tlen,
                                uint32_t* cigar, int32_t cigar_cap, int32_t* n_ops, void* workspace,
                                size_t workspace_bytes, int64_t* status, void* stream) {
    if (n_pairs < 0 || n_pairs > int64_t(INT32_MAX) - 1024 || !status || !workspace || cigar_cap < 1 ||
        max_qlen < 0 || max_tlen < 0)
        return SALOBA_EINVAL;
    if (n_pairs > 0 && (!q_words || !q_word_off || !t_words || !t_word_off || !score || !q_start || !q_end ||
                        !t_start || !t_end || !cigar || !n_ops))
        return SALOBA_EINVAL;
    if (fmt != SALOBA_PACK4 && fmt != SALOBA_PACK2) return SALOBA_EINVAL;
    if (sc.match < 1 || sc.match > 1024 || sc.mismatch > -1 || sc.mismatch < -1024 || sc.gap_extend < 1 ||
        sc.gap_open < sc.gap_extend || sc.gap_open > 1024)
        return SALOBA_EINVAL;
    if (reinterpret_cast<uintptr_t>(workspace) % 256) return SALOBA_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SALOBA_ECUDA;
    if (workspace_bytes < saloba_traceback_workspace_bytes(n_pairs, max_qlen, max_tlen, dev)) return SALOBA_EWORKSPACE;
    const TbPlan p = tb_plan(max_tlen, max_qlen);
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = static_cast<char*>(workspace);
    if (cudaMemsetAsync(ws, 0, 512, s) != cudaSuccess) return SALOBA_ECUDA;
    launch_status_init(status, s);
    if (n_pairs > 0) {
        TbArgs A{};
        A.q_words = q_words; A.q_word_off = q_word_off; A.t_words = t_words; A.t_word_off = t_word_off;
        A.n_pairs = n_pairs; A.fmt = int(fmt);
        A.match = sc.match; A.mismatch = sc.mismatch; A.alpha = sc.gap_open; A.beta = sc.gap_extend;
        A.score = score; A.q_start = q_start; A.q_end = q_end; A.t_start = t_start; A.t_end = t_end;
        A.cigar = cigar; A.cap = cigar_cap; A.n_ops = n_ops;
        A.counter = reinterpret_cast<int32_t*>(ws);
        A.slot_bitmap = reinterpret_cast<uint32_t*>(ws + 256);
        A.status = (unsigned long long*)status;
        if (p.slots > 0) {
            A.gslot = ws + 512;
            A.gslot_bytes = p.slot_bytes;
            A.g_rows = p.g_rows;
            A.g_cells = p.g_cells;
            A.slot_words = int(p.slots / 32);
            if (cudaMemsetAsync(ws + 512, 0, size_t(p.slots) * TB_WARPS * size_t(p.slot_bytes), s) != cudaSuccess)
                return SALOBA_ECUDA;
        }
        const int smem = int(sizeof(TbWarpSmem)) * TB_WARPS;
        traceback_kernel<<<p.sms * p.blocks, 32 * TB_WARPS, smem, s>>>(A);
        count_launches(1);
    }
    launch_status_final(status, s);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}
