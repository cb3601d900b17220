// ksw.cu — SURVEY §8(f) NEXT-1: BWA-MEM-compatible seed extension (ksw_extend2 semantics, DESIGN.md
// reading 17) on the GPU.
//
// Why not the wavefront kernels: ksw_extend2 trims each row to [first, last nonzero of the previous
// row + 2) and stops on z-drop, so row i+1's extent depends on ALL of row i — non-causal for an
// anti-diagonal wavefront, where row i+1 runs one step behind row i.  But its gaps open from M (the
// diagonal value), never from H, so inside a row no cell depends on its left neighbour's H:
//
//     M(i,j) = H(i-1,j-1) ? H(i-1,j-1) + S : 0          (row i-1 only)
//     E(i,j) from row i-1 (vertical), stored in eh[j].e  (row i-1 only)
//     F(i,j) = max(F(i,j-1) - e_ins, max(M(i,j-1) - oe_ins, 0))
//
// and F is a max-plus prefix scan of the row's M values: with Phi(j) = F(i,j) + j*e_ins,
// Phi(j+1) = max(Phi(j), max(M(i,j) - oe_ins, 0) + (j+1)*e_ins), a plain prefix maximum.  So one warp
// sweeps a row 32 columns at a time (column j on lane j % 32, a 5-step shuffle max-scan per 32
// columns), and the row bookkeeping (row maximum and its last column, end-to-end score, z-drop, the
// next row's [beg, end)) is warp-uniform — exactly the order of ksw_extend2, including the eh[]
// entries beyond `end` that a later row may read (they live in the per-warp eh array as in BWA).
//
// Roofline: integer ALU/issue bound like the wavefront kernels, but with ~25-30 instructions per 32
// cells (scan, bookkeeping) instead of 4.5 per 2 cells: the price of BWA's row-dependent trimming.
#include <climits>

#include "common.cuh"

namespace saloba {

constexpr int KSW_WARPS = 4;          // warps per block (one pair per warp)
constexpr int KSW_SMEM_COLS = 1024;   // eh[] in shared memory when q_len + 1 <= this

struct KswArgs {
    const uint32_t* q_words;
    const int64_t* q_word_off;
    const int32_t* q_len;
    const uint32_t* t_words;
    const int64_t* t_word_off;
    const int32_t* t_len;
    const int32_t* h0;
    int64_t n_pairs;
    int32_t fmt;
    saloba_ksw_params p;
    int32_t* out;          // [7][n_pairs]: score, qle, tle, gtle, gscore, max_off, clip
    int32_t* counter;      // dynamic work queue over pairs
    int2* geh;             // eh[] of long queries: per resident warp slot, gcols entries
    int64_t gcols;
    uint32_t* slot_bitmap; // block slots of geh
    int32_t slot_words;
    unsigned long long* status;
};

__device__ __forceinline__ int code_at(const uint32_t* words, int j, int fmt) {
    if (fmt == SALOBA_PACK4) return int((words[j >> 3] >> (4 * (j & 7))) & 15u);
    return int((words[j >> 4] >> (2 * (j & 15))) & 3u);
}

template <bool SMEM>
__global__ void __launch_bounds__(32 * KSW_WARPS) ksw_kernel(KswArgs A) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int2 s_eh[SMEM ? KSW_WARPS : 1][SMEM ? KSW_SMEM_COLS : 1];
    __shared__ uint32_t s_q[SMEM ? KSW_WARPS : 1][SMEM ? KSW_SMEM_COLS / 8 : 1];
    int bslot = -1;
    if (!SMEM) bslot = acquire_block_slot(A.slot_bitmap, A.slot_words);
    int2* eh = SMEM ? s_eh[warp] : A.geh + (int64_t(bslot) * KSW_WARPS + warp) * A.gcols;
    const saloba_ksw_params P = A.p;
    const int oe_del = P.o_del + P.e_del, oe_ins = P.o_ins + P.e_ins;

    for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(A.counter, 1);
        k = __shfl_sync(FULL, k, 0);
        if (int64_t(k) >= A.n_pairs) break;
        const int n = A.q_len[k], m = A.t_len[k], h0 = A.h0[k];
        // int32 arithmetic as ksw_extend2: every H, E, F and the scan keys (j+1)*e_ins stay below 2^31
        const bool ok = n >= 1 && m >= 1 && n <= MAX_LEN && m <= MAX_LEN && h0 >= 1 && h0 <= MAX_H0 &&
                        int64_t(h0) + int64_t(n) * P.a + (int64_t(n) + 1) * P.e_ins < int64_t(INT_MAX) &&
                        (SMEM ? n + 1 <= KSW_SMEM_COLS : int64_t(n) + 1 <= A.gcols);
        if (!ok) {
            if (lane < 7) A.out[int64_t(lane) * A.n_pairs + k] = lane == 0 ? -1 : -2;
            if (lane == 0) atomicMin(A.status, (unsigned long long)k);
            continue;
        }
        const uint32_t* qg = A.q_words + A.q_word_off[k];
        const uint32_t* tw = A.t_words + A.t_word_off[k];
        const uint32_t* qw = qg;
        if (SMEM) {  // the query's packed words, staged once per pair
            const int nw = A.fmt == SALOBA_PACK4 ? (n + 7) >> 3 : (n + 15) >> 4;
            for (int x = lane; x < nw; x += 32) s_q[warp][x] = __ldg(qg + x);
            qw = s_q[warp];
        }
        // row -1: eh[0].h = h0, eh[j].h = max(0, h0 - oe_ins - (j-1)*e_ins), eh[].e = 0
        for (int j = lane; j <= n; j += 32) {
            const int v = j == 0 ? h0 : h0 - oe_ins - (j - 1) * P.e_ins;
            eh[j] = make_int2(v > 0 ? v : 0, 0);
        }
        __syncwarp(FULL);
        // band adjustment (max_S = a)
        int w = P.w;
        {
            int mi = int(double(n * P.a + P.end_bonus - P.o_ins) / P.e_ins + 1.);
            mi = mi > 1 ? mi : 1;
            w = w < mi ? w : mi;
            int md = int(double(n * P.a + P.end_bonus - P.o_del) / P.e_del + 1.);
            md = md > 1 ? md : 1;
            w = w < md ? w : md;
        }
        int best = h0, max_i = -1, max_j = -1, max_ie = -1, gscore = -1, max_off = 0;
        int beg = 0, end = n;
        uint32_t tword = 0;
        for (int i = 0; i < m; ++i) {
            // target code of row i (one broadcast load per 8 / 16 rows)
            if (A.fmt == SALOBA_PACK4) {
                if ((i & 7) == 0) tword = __ldg(tw + (i >> 3));
            } else if ((i & 15) == 0) {
                tword = __ldg(tw + (i >> 4));
            }
            const int tc = A.fmt == SALOBA_PACK4 ? int((tword >> (4 * (i & 7))) & 15u) : int((tword >> (2 * (i & 15))) & 3u);
            if (beg < i - w) beg = i - w;
            if (end > i + w + 1) end = i + w + 1;
            if (end > n) end = n;
            int h1 = 0;
            if (beg == 0) {
                h1 = h0 - (P.o_del + P.e_del * (i + 1));
                h1 = h1 > 0 ? h1 : 0;
            }
            const int h1_init = h1;
            int phi = beg * P.e_ins;       // Phi(beg) = F(i, beg) + beg*e_ins with F(i, beg) = 0
            int hcarry = h1;               // H(i, j0 - 1) entering a 32-column round
            int rmax = 0, rj = -1;         // this lane's row maximum and its last column
            int first_nz = INT_MAX, last_nz = -1;
            for (int j0 = beg & ~31; j0 < end; j0 += 32) {
                const int j = j0 + lane;
                const bool act = j >= beg && j < end;
                int M = 0, e = 0;
                if (act) {
                    const int2 v = eh[j];
                    M = v.x;
                    e = v.y;
                    const int qc = code_at(qw, j, A.fmt);
                    const int s = (tc == 4 || qc == 4) ? -1 : (tc == qc ? P.a : -P.b);
                    M = M ? M + s : 0;
                }
                // F by a prefix maximum of max(M - oe_ins, 0) + (j+1)*e_ins over the row
                const int ti = M - oe_ins;
                int v = act ? (ti > 0 ? ti : 0) + (j + 1) * P.e_ins : INT_MIN;
                int incl = v;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int u = __shfl_up_sync(FULL, incl, off);
                    if (lane >= off) incl = incl > u ? incl : u;
                }
                int excl = __shfl_up_sync(FULL, incl, 1);
                if (lane == 0) excl = INT_MIN;
                const int ph = phi > excl ? phi : excl;
                const int f = ph - j * P.e_ins;
                int h = M > e ? M : e;
                h = h > f ? h : f;
                // eh[j].h = H(i, j-1): the left neighbour's h (carry across rounds, h1 at beg)
                int hp = __shfl_up_sync(FULL, h, 1);
                if (lane == 0) hp = hcarry;
                if (j == beg) hp = h1_init;
                const int td = M - oe_del;
                int en = e - P.e_del;
                en = en > (td > 0 ? td : 0) ? en : (td > 0 ? td : 0);
                if (act) {
                    eh[j] = make_int2(hp, en);
                    if (h >= rmax) {  // the LAST column of the row maximum (ties -> larger j)
                        rmax = h;
                        rj = j;
                    }
                    if (hp != 0 || en != 0) {
                        first_nz = first_nz < j ? first_nz : j;
                        last_nz = j;
                    }
                }
                phi = phi > __shfl_sync(FULL, incl, 31) ? phi : __shfl_sync(FULL, incl, 31);
                const int last_lane = (end - 1 - j0) < 31 ? (end - 1 - j0) : 31;
                hcarry = __shfl_sync(FULL, h, last_lane);
            }
            // h1 = H(i, end-1) (h1_init when the row is empty); eh[end] = {h1, 0}
            h1 = end > beg ? hcarry : h1_init;
            if (lane == (end & 31)) eh[end] = make_int2(h1, 0);
            // warp reductions: row maximum (last column on ties) and the nonzero extent
            int mrow = rmax, mj = rj;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const int om = __shfl_xor_sync(FULL, mrow, off), oj = __shfl_xor_sync(FULL, mj, off);
                if (om > mrow || (om == mrow && oj > mj)) {
                    mrow = om;
                    mj = oj;
                }
            }
            if (mrow == 0) mj = -1;  // ksw_extend2 never records a column for an all-zero row
            first_nz = int(__reduce_min_sync(FULL, unsigned(first_nz)));
            last_nz = int(__reduce_max_sync(FULL, unsigned(last_nz + 1))) - 1;
            if (h1 != 0) last_nz = end;  // eh[end] = (h1, 0)
            __syncwarp(FULL);
            if ((beg < end ? end : beg) == n) {  // ksw_extend2 tests its column index after the row loop
                max_ie = gscore > h1 ? max_ie : i;
                gscore = gscore > h1 ? gscore : h1;
            }
            if (mrow == 0) break;
            if (mrow > best) {
                best = mrow;
                max_i = i;
                max_j = mj;
                const int off = mj > i ? mj - i : i - mj;
                max_off = max_off > off ? max_off : off;
            } else if (P.zdrop > 0) {
                if (i - max_i > mj - max_j) {
                    if (best - mrow - ((i - max_i) - (mj - max_j)) * P.e_del > P.zdrop) break;
                } else {
                    if (best - mrow - ((mj - max_j) - (i - max_i)) * P.e_ins > P.zdrop) break;
                }
            }
            // next row's [beg, end): first / last column whose (eh.h, eh.e) is not (0, 0)
            const int nb = first_nz < end ? first_nz : end;
            const int lastj = last_nz >= nb ? last_nz : nb - 1;
            beg = nb;
            end = lastj + 2 < n ? lastj + 2 : n;
        }
        if (lane == 0) {
            const int64_t N = A.n_pairs;
            A.out[k] = best;
            A.out[N + k] = max_j + 1;
            A.out[2 * N + k] = max_i + 1;
            A.out[3 * N + k] = max_ie + 1;
            A.out[4 * N + k] = gscore;
            A.out[5 * N + k] = max_off;
            A.out[6 * N + k] = (gscore <= 0 || gscore <= best - P.end_bonus) ? 1 : 0;
        }
        __syncwarp(FULL);
    }
    if (!SMEM) release_block_slot(A.slot_bitmap, bslot);
}

}  // namespace saloba

using namespace saloba;

namespace {
struct KswDev {
    int sms = 0, blocks_smem = 0, blocks_glob = 0;
};
KswDev ksw_dev() {
    KswDev d;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.blocks_smem, ksw_kernel<true>, 32 * KSW_WARPS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.blocks_glob, ksw_kernel<false>, 32 * KSW_WARPS, 0);
    d.blocks_smem = d.blocks_smem > 0 ? d.blocks_smem : 1;
    d.blocks_glob = d.blocks_glob > 0 ? d.blocks_glob : 1;
    return d;
}
size_t al256(size_t x) { return (x + 255) / 256 * 256; }
bool ksw_params_ok(const saloba_ksw_params* p) {
    const int lim = 1 << 10;
    return p && p->a >= 1 && p->a <= lim && p->b >= 1 && p->b <= lim && p->o_del >= 0 && p->o_del <= lim &&
           p->e_del >= 1 && p->e_del <= lim && p->o_ins >= 0 && p->o_ins <= lim && p->e_ins >= 1 &&
           p->e_ins <= lim && p->w >= 0 && p->end_bonus >= 0 && p->end_bonus <= lim && p->zdrop >= 0;
}
}  // namespace

SALOBA_API size_t saloba_ksw_workspace_bytes(int64_t n_pairs, int32_t max_qlen, int device) {
    if (n_pairs < 0 || max_qlen < 0) return 0;
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) return 0;
    const KswDev d = ksw_dev();
    cudaSetDevice(prev);
    size_t bytes = 256 + 256;  // counter + slot bitmap
    if (int64_t(max_qlen) + 1 > KSW_SMEM_COLS) {
        const int64_t slots = (int64_t(d.sms) * d.blocks_glob + 32 + 31) / 32 * 32;
        bytes += al256(size_t(slots) * KSW_WARPS * size_t(max_qlen + 1) * sizeof(int2));
    }
    return bytes;
}

SALOBA_API int saloba_ksw_extend(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                                 const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len,
                                 const int32_t* h0, int64_t n_pairs, const saloba_ksw_params* params,
                                 saloba_packing fmt, int32_t max_qlen, int32_t* out, void* workspace,
                                 size_t workspace_bytes, int64_t* status, void* stream) {
    if (n_pairs < 0 || n_pairs > int64_t(INT32_MAX) - 1024 || !status || !workspace || max_qlen < 0)
        return SALOBA_EINVAL;
    if (n_pairs > 0 && (!q_words || !q_word_off || !q_len || !t_words || !t_word_off || !t_len || !h0 || !out))
        return SALOBA_EINVAL;
    if (fmt != SALOBA_PACK4 && fmt != SALOBA_PACK2) return SALOBA_EINVAL;
    if (!ksw_params_ok(params)) return SALOBA_EINVAL;
    if (reinterpret_cast<uintptr_t>(workspace) % 256) return SALOBA_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SALOBA_ECUDA;
    if (workspace_bytes < saloba_ksw_workspace_bytes(n_pairs, max_qlen, dev)) return SALOBA_EWORKSPACE;
    const KswDev d = ksw_dev();
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = static_cast<char*>(workspace);
    if (cudaMemsetAsync(ws, 0, 512, s) != cudaSuccess) return SALOBA_ECUDA;
    launch_status_init(status, s);
    if (n_pairs > 0) {
        KswArgs A{};
        A.q_words = q_words; A.q_word_off = q_word_off; A.q_len = q_len;
        A.t_words = t_words; A.t_word_off = t_word_off; A.t_len = t_len;
        A.h0 = h0; A.n_pairs = n_pairs; A.fmt = int(fmt); A.p = *params; A.out = out;
        A.counter = reinterpret_cast<int32_t*>(ws);
        A.slot_bitmap = reinterpret_cast<uint32_t*>(ws + 256);
        A.status = (unsigned long long*)status;
        const bool smem = int64_t(max_qlen) + 1 <= KSW_SMEM_COLS;
        if (smem) {
            const int grid = d.sms * d.blocks_smem;
            ksw_kernel<true><<<grid, 32 * KSW_WARPS, 0, s>>>(A);
        } else {
            const int64_t slots = (int64_t(d.sms) * d.blocks_glob + 32 + 31) / 32 * 32;
            A.geh = reinterpret_cast<int2*>(ws + 512);
            A.gcols = int64_t(max_qlen) + 1;
            A.slot_words = int(slots / 32);
            const int grid = d.sms * d.blocks_glob;
            ksw_kernel<false><<<grid, 32 * KSW_WARPS, 0, s>>>(A);
        }
        count_launches(1);
    }
    launch_status_final(status, s);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}
