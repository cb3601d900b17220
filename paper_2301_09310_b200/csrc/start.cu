// start.cu — start coordinates of LOCAL alignments (reading 15).
//
// The paper reports only the score and end of an alignment; SPEC marks traceback out
// of scope.  The start is the first aligned column of an optimal alignment ending at
// the reported end cell (t_end, q_end), found the standard way without traceback: align the
// REVERSED prefixes t' = t[t_end] .. t[0] and q' = q[q_end] .. q[0] in LOCAL mode.  Any optimal
// alignment of the reversed prefixes is an optimal forward alignment inside [0..t_end] x [0..q_end]
// whose forward end cell has H = score and is componentwise <= (t_end, q_end); by the tie rule
// (t_end, q_end) is the lexicographically smallest cell with H = score, so that end IS (t_end,
// q_end).  The reversed end (i', j') chosen by the same tie rule (smallest i', then j') gives
// t_start = t_end - i', q_start = q_end - j': among all optimal alignments ending at the end cell,
// the largest t_start, then the largest q_start.  Score 0: start = (0, 0), like the end.
//
// Device work: reverse_prefix_kernel writes the reversed prefixes into the workspace at the SAME
// word offsets as the forward sequences (a prefix never needs more words), the existing
// schedule + DP kernels align them (LOCAL), and start_finalize_kernel maps the reversed ends back.
// The reversed pass costs (q_end+1)(t_end+1) cells per pair, at most the forward pass.
#include <climits>

#include "common.cuh"

namespace saloba {

// bases of one packed word in reverse order (PACK4: byte swap + nibble swap; PACK2: bit reverse +
// swap of the two bits of every field)
template <int FMT>
__device__ __forceinline__ uint32_t rev_bases(uint32_t x) {
    if (FMT == SALOBA_PACK4) {
        x = __byte_perm(x, 0, 0x0123);
        return ((x >> 4) & 0x0F0F0F0Fu) | ((x & 0x0F0F0F0Fu) << 4);
    }
    x = __brev(x);
    return ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
}

// One warp per pair (grid-stride).  Pairs whose forward score is <= 0 (no alignment, or an invalid
// pair) get a 1-base prefix so the batch stays valid; their results are ignored by finalize.
template <int FMT>
__global__ void reverse_prefix_kernel(const uint32_t* __restrict__ words, const int64_t* __restrict__ word_off,
                                      const int32_t* __restrict__ end, const int32_t* __restrict__ score, int64_t n,
                                      uint32_t* __restrict__ out, int32_t* __restrict__ out_len) {
    constexpr int B = FMT == SALOBA_PACK4 ? 8 : 16;      // bases per word
    constexpr int BITS = FMT == SALOBA_PACK4 ? 4 : 2;
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
    for (int64_t p = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; p < n; p += warps) {
        const int e = score[p] > 0 ? end[p] : 0;  // last forward position of the prefix
        const int len = e + 1;
        const uint32_t* src = words + word_off[p];
        uint32_t* dst = out + word_off[p];
        const int nw = (len + B - 1) / B;
        for (int w = lane; w < nw; w += 32) {
            // reversed bases 8w.. (16w.. for PACK2) are forward positions hi, hi-1, ...: the
            // concatenation [rev(word q-1) : rev(word q)] shifted so that position hi comes first
            // (rev = base order reversed inside a word; word -1 = padding)
            const int hi = e - B * w;
            const int q = hi / B, o = hi % B;
            const uint32_t wq = __ldg(src + q);
            const uint32_t wp = q > 0 ? __ldg(src + q - 1) : (FMT == SALOBA_PACK4 ? 0xFFFFFFFFu : 0u);
            dst[w] = __funnelshift_r(rev_bases<FMT>(wq), rev_bases<FMT>(wp), BITS * (B - 1 - o));
        }
        if (lane == 0) out_len[p] = len;
    }
}

// start = end - reversed end; checks that the reversed pass reached the forward score.
__global__ void start_finalize_kernel(const int32_t* __restrict__ score, const int32_t* __restrict__ q_end,
                                      const int32_t* __restrict__ t_end, const int32_t* __restrict__ rscore,
                                      const int32_t* __restrict__ rq_end, const int32_t* __restrict__ rt_end,
                                      int64_t n, int32_t* __restrict__ q_start, int32_t* __restrict__ t_start,
                                      unsigned long long* status) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
        const int s = score[p];
        int qs = 0, ts = 0;
        if (s < 0) {
            qs = ts = -2;  // invalid pair in the forward call
        } else if (s > 0) {
            if (rscore[p] != s) {  // cannot happen for a consistent forward result
                qs = ts = -3;
                atomicMin(status, (unsigned long long)p);
            } else {
                qs = q_end[p] - rq_end[p];
                ts = t_end[p] - rt_end[p];
            }
        }
        q_start[p] = qs;
        t_start[p] = ts;
    }
}

void launch_reverse_prefix(int fmt, const uint32_t* words, const int64_t* word_off, const int32_t* end,
                           const int32_t* score, int64_t n, uint32_t* out, int32_t* out_len, int sms, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t need = (n + 7) / 8;  // 8 warps per block
    const int grid = int(need < int64_t(sms) * 16 ? need : int64_t(sms) * 16);
    if (fmt == SALOBA_PACK4)
        reverse_prefix_kernel<4><<<grid, 256, 0, s>>>(words, word_off, end, score, n, out, out_len);
    else
        reverse_prefix_kernel<2><<<grid, 256, 0, s>>>(words, word_off, end, score, n, out, out_len);
    count_launches(1);
}

void launch_start_finalize(const int32_t* score, const int32_t* q_end, const int32_t* t_end, const int32_t* rscore,
                           const int32_t* rq_end, const int32_t* rt_end, int64_t n, int32_t* q_start,
                           int32_t* t_start, int64_t* status, int sms, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t need = (n + 255) / 256;
    const int grid = int(need < int64_t(sms) * 8 ? need : int64_t(sms) * 8);
    start_finalize_kernel<<<grid, 256, 0, s>>>(score, q_end, t_end, rscore, rq_end, rt_end, n, q_start, t_start,
                                               (unsigned long long*)status);
    count_launches(1);
}

}  // namespace saloba
