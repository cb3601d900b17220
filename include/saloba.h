/*
 * saloba.h — C ABI of the B200-native batched affine-gap seed-extension library.
 *
 * The operation (§II-A, Eqs. 1-3):
 * for every pair k, fill the DP table of query q (columns j = 0..n-1) against target t
 * (rows i = 0..m-1, "reference at i and query at j") with
 *
 *     E(i,j) = max(H(i,j-1) - alpha, E(i,j-1) - beta)                     (Eq. 2)
 *     F(i,j) = max(H(i-1,j) - alpha, F(i-1,j) - beta)                     (Eq. 3)
 *     H(i,j) = max(0, E(i,j), F(i,j), H(i-1,j-1) + S(t_i, q_j))           (Eq. 1)
 *
 * with S = match if the bases are equal and not N, else mismatch (N never matches),
 * and return the best score and its end coordinates: maximal score, then smallest target index
 * i, then smallest query index j.
 *
 *   SALOBA_LOCAL  — Smith-Waterman local mode: boundary 0; score >= 0; ends (0,0) when score = 0
 *                   (S:249).
 *   SALOBA_EXTEND — seed-anchored extension ("extending to both directions from the
 *                   found seeds"; exact reading in DESIGN.md §2 / SURVEY §8(c)): an anchor
 *                   H(-1,-1) = h0 (the seed's score), leading-gap boundaries
 *                   H(-1,j) = max(0, h0-alpha-beta*j), H(i,-1) = max(0, h0-alpha-beta*i), no fresh
 *                   local starts (H(i-1,j-1) == 0 kills the diagonal), score = max(h0, max H),
 *                   ends (-1,-1) when no cell exceeds h0.
 *
 * alpha ("gap_open") is the cost of a gap's FIRST base and beta ("gap_extend") of each further
 * base, literal to Eqs. 2-3 (BWA-MEM o=6,e=1 is alpha=7, beta=1).
 *
 * Entry points: saloba_pack (A1); saloba_workspace_bytes + saloba_align_batch (A2-A4, device
 * buffers); saloba_align_host[_ctx] (A1-A4 from host buffers); saloba_partition (A5, shards for
 * the GPUs of one box); saloba_align_banded (banded DP);
 * saloba_locate_start (LOCAL start coordinates, NEXT-3); saloba_traceback (CIGAR, NEXT-3);
 * saloba_scatter_results (A5, rank 0
 * puts gathered shards back in input order); saloba_ksw_extend (BWA-MEM-compatible extension,
 * NEXT-1); diagnostics at the end.
 *
 * Conventions for every entry point:
 *   - Pointers marked [dev] are device pointers owned by the caller (e.g. torch tensors); the
 *     library never frees them and allocates nothing on the hot path.  [host] are host pointers.
 *   - `stream` is a cudaStream_t passed as void*; NULL means the legacy default stream.  Device
 *     calls are asynchronous on `stream`; outputs are valid after the stream is synchronised.
 *   - Host-checkable errors return a negative SALOBA_E* code synchronously and launch nothing.
 *   - Data-dependent errors are reported through the [dev] int64 `status` word: the call sets
 *     it to -1 (no error) or to the smallest offending index (atomicMin), readable after the
 *     stream is synchronised.
 *   - Thread-safe across host threads and streams.  Process-wide state: a per-device cache of
 *     occupancy numbers (computed once) and, per (device, caller stream), the auxiliary streams and
 *     fork/join events a call's concurrent bin kernels run on (created on first use, kept for the
 *     process), so calls on different streams overlap and a CUDA-graph capture of one stream
 *     never involves another stream's work.
 */
#ifndef SALOBA_H
#define SALOBA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SALOBA_VERSION 2

typedef struct {
    int32_t match;      /* >= 1        */
    int32_t mismatch;   /* <= -1        */
    int32_t gap_open;   /* alpha: cost of a gap's first base; alpha >= beta   */
    int32_t gap_extend; /* beta: cost of each further gap base; beta >= 1    */
} saloba_scoring;

typedef enum { SALOBA_LOCAL = 0, SALOBA_EXTEND = 1 } saloba_mode;

/* Packed base formats:
 *   SALOBA_PACK4: 8 bases per uint32, base p in nibble p%8 (least-significant nibble first),
 *                 codes A=0 C=1 G=2 T/U=3 N=4, padding nibble 15.
 *   SALOBA_PACK2: 16 bases per uint32, base p in bits 2(p%16)..+1, codes A=0 C=1 G=2 T/U=3;
 *                 N is not representable (pack reports it as an invalid base); padding bits 0
 *                 and never scored (lengths mask it). */
typedef enum { SALOBA_PACK2 = 2, SALOBA_PACK4 = 4 } saloba_packing;

enum {
    SALOBA_OK = 0,
    SALOBA_EINVAL = -1,       /* bad argument (null pointer, n < 0, bad scheme, bad enum)      */
    SALOBA_ECUDA = -2,        /* a CUDA runtime call failed                                    */
    SALOBA_EWORKSPACE = -3,   /* workspace too small for n_pairs                               */
    SALOBA_EUNSUPPORTED = -4, /* no B200 (sm_100) device or a feature this build lacks         */
};

/* Per-call tuning / test / profiling knobs.  Pass NULL for the defaults (all zero). */
typedef struct {
    int32_t force_group;  /* 0: the scheduler picks the subwarp size G per pair; else G in {1,2,4,8,16,32}
                             (pairs whose query exceeds that G's spill-row bound keep the scheduler's G) */
    int32_t force_path;   /* 0: auto; 1: int32 exact path for every pair; 2: prefer the int16x2 path */
    int32_t keep_order;   /* 1: do not sort pairs by length (A/B test of the scheduler)            */
    int32_t i16_rows;     /* 0: default (16); 8: target rows per lane of the int16x2 kernel (A/B knob) */
    void* ev_dp_begin;    /* optional cudaEvent_t recorded on `stream` right before the first DP
                             kernel launch of the call (after packing/scheduling), for profiling */
    void* ev_dp_end;      /* optional cudaEvent_t recorded on `stream` after the last DP kernel   */
    int32_t* bin_counts;  /* optional [dev] int32[16]: pairs per scheduler bin of this call, bin =
                             path*8 + log2(G), path 0 = int32 exact, 1 = int16x2; bin 15 = invalid.
                             Bin 13 is the int16x2 "long bin" (queries >= 2048 bp and every pair the
                             cost model gives G >= 16): it runs at G=16 or G=32, see long_group.
                             Bins 14 / 6: int16x2 G=1 / G=2 pairs whose query contains N (an N
                             column's substitution is forced to mismatch; other query-N pairs run
                             int32).  Bin 7: int32 pairs whose values could reach 2^27 */
    int32_t* long_group;  /* optional [dev] int32[1]: how the long bin ran this call: 4 or 5 = log2(G)
                             of the one-warp-per-duo kernel (G=16 iff the bin holds >= 4 waves of
                             G=16 subwarps, else G=32: half the per-pair latency), 6 = the cooperative
                             kernel (fewer long pairs than two waves of G=32 warps hold: the warps of a
                             block share each duo, one 512-row chunk each) */
    unsigned long long* counters; /* optional [dev] uint64[8], ADDED to (SURVEY §8(f) NEXT-4 instrumentation
                             of the int16x2 kernels, §IV-A / SPEC acceptance 3-5): [0] pass-1
                             chunk passes of all work items (a work item = two pairs, one per 16-bit
                             half); [1] their wavefront steps (Q + G - 1 per chunk pass, Q at G = 1);
                             [2] spilled 64-byte blocks (the chunk-bottom H and F of 8 columns, both
                             halves) written; [3] spilled blocks read back; [4] pass-2 chunk passes;
                             [5] pass-2 steps; [6] pass-1 lane-strips (chunk passes x G); [7] work items.
                             The counting costs one warp reduction + atomic per chunk; NULL: none */
    int32_t reserved[2];
} saloba_options;

/* ---- A1: packing --------------------------------------------------------------------------- */

/* Capacity (uint32 words) that saloba_pack needs for n_seqs sequences of total_bases bases.
 * The packed layout is closed-form: sequence s starts at word byte_off[s]/B + s
 * (B = 8 for PACK4, 16 for PACK2), so no scan is needed and every sequence is word-aligned. */
int64_t saloba_packed_words(int64_t total_bases, int64_t n_seqs, saloba_packing fmt);

/* ASCII {A,C,G,T,U,N; any case} -> packed words (SPEC S:44-52 pack_sequence).
 *   ascii     [dev] uint8[byte_off[n_seqs]]      the concatenated sequences
 *   byte_off  [dev] int64[n_seqs+1]              sequence s = ascii[byte_off[s] .. byte_off[s+1])
 *   words     [dev] uint32[words_capacity]       output (see saloba_packed_words)
 *   word_off  [dev] int64[n_seqs+1]              output: first word of each sequence (+ end)
 *   lens      [dev] int32[n_seqs]                output: bases per sequence (may be NULL)
 *   status    [dev] int64[1]                     -1, or the smallest byte index that is not a
 *                                                valid base (InvalidBase; N under PACK2).
 *                                                Empty sequences are legal here (0 words, lens 0);
 *                                                saloba_align_batch reports them (EmptySequence).
 *                                                byte_off[n_seqs] (one past the last byte) when
 *                                                words_capacity < saloba_packed_words(
 *                                                byte_off[n_seqs], n_seqs, fmt): nothing is written.
 * Returns SALOBA_OK or a negative code (nothing launched): SALOBA_EWORKSPACE when words_capacity is
 * below n_seqs + 1 (the layout's minimum, checkable without reading the device offsets). */
int saloba_pack(const uint8_t* ascii, const int64_t* byte_off, int64_t n_seqs, saloba_packing fmt,
                uint32_t* words, int64_t words_capacity, int64_t* word_off, int32_t* lens, int64_t* status,
                void* stream);

/* ---- A2-A4: schedule, DP, write-back ------------------------------------------------------- */

/* Device workspace (bytes) saloba_align_batch needs for n_pairs pairs whose query lengths are
 * <= max_qlen (target lengths are unbounded up to 2^20; max_tlen is accepted for forward
 * compatibility).  device = CUDA ordinal whose SM count sizes the persistent grids. */
size_t saloba_workspace_bytes(int64_t n_pairs, int32_t max_qlen, int32_t max_tlen, int device);

/* Align n_pairs packed pairs.
 *   q_words, t_words        [dev] packed sequences (format fmt)
 *   q_word_off, t_word_off  [dev] int64[n_pairs]  first word of pair k's query / target
 *   q_len, t_len            [dev] int32[n_pairs]  lengths in bases (1 .. 2^20)
 *   h0                      [dev] int32[n_pairs]  EXTEND: initial (seed) score, 1 .. 2^29;
 *                                                  must be NULL-free in EXTEND, ignored in LOCAL
 *   score, q_end, t_end     [dev] int32[n_pairs]  results, in INPUT order (SoA)
 *   workspace               [dev] >= saloba_workspace_bytes(...) bytes, 256-byte aligned
 *   status                  [dev] int64[1]        -1, or the smallest pair index with invalid
 *                                                  data (length 0 or > 2^20, query longer than the
 *                                                  workspace was sized for, h0 out of range);
 *                                                  such pairs get score = -1, q_end = t_end = -2
 *   opt                     [host] may be NULL
 * Host-checked: pointers, n_pairs >= 0, scheme (match >= 1, mismatch <= -1, alpha >= beta >= 1,
 * all |values| <= 2^10), mode/fmt enums, workspace size.
 * Results are bit-identical regardless of G, precision path, batch order and sharding. */
int saloba_align_batch(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                       const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len,
                       const int32_t* h0, int64_t n_pairs, saloba_scoring sc, saloba_mode mode,
                       saloba_packing fmt, int32_t* score, int32_t* q_end, int32_t* t_end, void* workspace,
                       size_t workspace_bytes, int64_t* status, const saloba_options* opt, void* stream);

/* ---- banded DP ------------------------------------------------------------ */

/* As saloba_align_batch, but pair k's table holds only the cells |i - j| <= band_w[k] (the band
 * around the diagonal through the table origin / the EXTEND anchor, as BWA-MEM's extension band;
 * PAPER.md P:1728-1735 names banded DP as the long-read direction).  Cells outside the band read
 * as H = E = F = 0, like out-of-table cells, and are never computed: the work per pair is about
 * t_len x (2 band_w + 8) cells instead of q_len x t_len (reading 16).
 *   band_w  [dev] int32[n_pairs]  band half-width >= 0; a negative value is invalid data
 *                                 (status / score -1, ends -2), band_w >= max(q_len, t_len) gives
 *                                 the unbanded result.
 * Banded pairs run on the exact int32 kernel; same workspace (saloba_workspace_bytes), same
 * ownership, stream and error conventions as saloba_align_batch. */
int saloba_align_banded(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                        const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len,
                        const int32_t* h0, const int32_t* band_w, int64_t n_pairs, saloba_scoring sc,
                        saloba_mode mode, saloba_packing fmt, int32_t* score, int32_t* q_end, int32_t* t_end,
                        void* workspace, size_t workspace_bytes, int64_t* status, const saloba_options* opt,
                        void* stream);

/* ---- start coordinates (LOCAL mode) ----------------------------------- */

/* The paper reports score and end only (SPEC S:16/S:215 put traceback out of scope).
 * Start = the first aligned column (t_start, q_start) of an optimal alignment that ends at the
 * reported end cell; among several, the largest t_start, then the largest q_start (DESIGN.md
 * reading 15).  Computed without traceback by aligning the reversed prefixes t[t_end..0] and
 * q[q_end..0] in LOCAL mode with the same kernels: start = end - (reversed end).
 * (EXTEND alignments start at the seed anchor by definition, so they need no start pass.)
 *
 * Workspace for saloba_locate_start: n_pairs pairs whose packed query / target buffers hold
 * q_words_total / t_words_total words (the reversed prefixes are written at the same word
 * offsets) and whose queries are <= max_qlen bases.  0 on a bad argument or device. */
size_t saloba_start_workspace_bytes(int64_t n_pairs, int64_t q_words_total, int64_t t_words_total,
                                    int32_t max_qlen, int device);

/* Start coordinates of LOCAL results produced by saloba_align_batch on the same packed pairs.
 *   q_words, q_word_off, t_words, t_word_off, fmt   [dev] as passed to saloba_align_batch
 *   q_words_total, t_words_total   capacity (words) of q_words / t_words
 *   sc                              the scoring scheme of the forward call
 *   score, q_end, t_end   [dev] int32[n_pairs]  the forward LOCAL results (input)
 *   q_start, t_start      [dev] int32[n_pairs]  output: start coordinates (0-based, inclusive);
 *                                               (0, 0) when score == 0; (-2, -2) when score < 0
 *                                               (a pair the forward call rejected)
 *   workspace             [dev] >= saloba_start_workspace_bytes(...), 256-byte aligned
 *   status                [dev] int64[1]  -1, or the smallest pair index whose reversed pass did
 *                                         not reproduce `score` (inconsistent input; start -3)
 * Asynchronous on `stream`; host-checked errors as saloba_align_batch. */
int saloba_locate_start(const uint32_t* q_words, const int64_t* q_word_off, int64_t q_words_total,
                        const uint32_t* t_words, const int64_t* t_word_off, int64_t t_words_total, int64_t n_pairs,
                        saloba_scoring sc, saloba_packing fmt, const int32_t* score, const int32_t* q_end,
                        const int32_t* t_end, int32_t* q_start, int32_t* t_start, void* workspace,
                        size_t workspace_bytes, int64_t* status, const saloba_options* opt, void* stream);

/* ---- CIGAR traceback (LOCAL mode) ------------------------------------------ */

/* Workspace for saloba_traceback: n_pairs pairs whose aligned regions span at most max_tlen target
 * and max_qlen query bases (regions up to 256 rows and 32,768 cells in 16x16 tiles need no workspace
 * beyond 512 B). */
size_t saloba_traceback_workspace_bytes(int64_t n_pairs, int32_t max_qlen, int32_t max_tlen, int device);

/* The CIGAR of each LOCAL result (reading 18; the paper reports score and end only,
 * P:132-149): the global affine alignment of t[t_start..t_end] x q[q_start..q_end]
 * under the same scheme (its optimum equals the local score), the optimal one whose op string read
 * from the end is smallest with M < D < I (indels left-aligned).
 *   q_words..t_word_off, fmt, sc  [dev] as for saloba_align_batch / saloba_locate_start
 *   score, q_end, t_end           [dev] int32[n_pairs] forward LOCAL results
 *   q_start, t_start              [dev] int32[n_pairs] from saloba_locate_start
 *   max_qlen, max_tlen            bounds of the aligned region (q_end - q_start + 1 etc.)
 *   cigar   [dev] uint32[n_pairs][cigar_cap]  output: BAM-encoded elements (length << 4 | op),
 *                                             op M = 0, I = 1, D = 2, in forward order
 *   n_ops   [dev] int32[n_pairs]   output: elements written; 0 when score == 0; -1 when score < 0
 *                                  (a rejected pair) or the CIGAR does not fit cigar_cap
 *   status  [dev] int64[1]  -1, or the smallest pair whose region's global score differs from
 *                           `score` (inconsistent input), whose CIGAR overflowed, or whose region
 *                           exceeds the workspace bounds
 * Asynchronous on `stream`. */
int saloba_traceback(const uint32_t* q_words, const int64_t* q_word_off, const uint32_t* t_words,
                     const int64_t* t_word_off, int64_t n_pairs, saloba_scoring sc, saloba_packing fmt,
                     const int32_t* score, const int32_t* q_start, const int32_t* q_end, const int32_t* t_start,
                     const int32_t* t_end, int32_t max_qlen, int32_t max_tlen, uint32_t* cigar, int32_t cigar_cap,
                     int32_t* n_ops, void* workspace, size_t workspace_bytes, int64_t* status, void* stream);

/* ---- A5: length-balanced sharding over the GPUs of one box ------------------------ */

/* Workspace (bytes) saloba_partition needs for n_pairs pairs (0 on a bad n_pairs). */
size_t saloba_partition_workspace_bytes(int64_t n_pairs);

/* Assign each pair to one of `world` ranks so that the modelled work is balanced (PAPER.md
 * the paper's equal split leaves GPUs idle on skewed batches; it names "dynamic
 * assignment or preprocessing with approximate sorting" as the fix).  cost = q_len*t_len + 2048,
 * one stable radix sort by descending cost, then snake order over the ranks
 * (0..W-1, W-1..0, ...).  Deterministic: every rank computing it from the same lengths gets the
 * same assignment, so no collective is needed to agree on it.
 *   q_len, t_len  [dev] int32[n_pairs]   lengths (negative values count as 0)
 *   owner         [dev] int32[n_pairs]   output: rank of each pair, in 0..world-1
 *   workspace     [dev] >= saloba_partition_workspace_bytes(n_pairs), 256-byte aligned
 * Asynchronous on `stream`.  Host-checked errors only (EINVAL / EWORKSPACE). */
int saloba_partition(const int32_t* q_len, const int32_t* t_len, int64_t n_pairs, int32_t world, int32_t* owner,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Rank 0's reassembly step (SURVEY §8(e) "rank 0 unpermutes with the partition it computed"):
 * the shards gathered from `world` ranks are written back to input order.
 *   parts    [dev] int32[world][3][stride]   rank r's results (rows score, q_end, t_end), as
 *                                            gathered (each shard padded to `stride` columns)
 *   index    [dev] int32[world][stride]      global input index of each gathered column; -1 marks
 *                                            a padding column (ignored)
 *   score, q_end, t_end  [dev] int32[n_total]  output, input order
 *   status   [dev] int64[1]   -1, or the smallest flat slot r*stride+i whose index is >= n_total
 *                             (inconsistent index; that column is not written)
 * Every index in 0..n_total-1 should appear exactly once; positions no rank owns are left as they
 * were.  Asynchronous on `stream`.  Host-checked: pointers, stride >= 0, world >= 1,
 * 0 <= n_total <= INT32_MAX. */
int saloba_scatter_results(const int32_t* parts, const int32_t* index, int64_t stride, int32_t world,
                           int64_t n_total, int32_t* score, int32_t* q_end, int32_t* t_end, int64_t* status,
                           void* stream);

/* ---- BWA-MEM-compatible seed extension ------------------------------------ */

/* BWA-MEM's extension parameters (mem_opt_t): scores a (match), b (mismatch penalty, > 0), N
 * scores -1; a deletion of k target bases costs o_del + k*e_del, an insertion of k query bases
 * o_ins + k*e_ins; band w; end_bonus; zdrop (0 disables).  BWA-MEM defaults: a 1, b 4, o 6, e 1,
 * w 100, end_bonus 5, zdrop 100. */
typedef struct {
    int32_t a, b, o_del, e_del, o_ins, e_ins, w, end_bonus, zdrop;
} saloba_ksw_params;

/* Workspace (bytes) for saloba_ksw_extend on n_pairs pairs whose queries are <= max_qlen bases
 * (0 on a bad argument or device). */
size_t saloba_ksw_workspace_bytes(int64_t n_pairs, int32_t max_qlen, int device);

/* Seed extension with BWA-MEM's ksw_extend2 semantics (PAPER.md P:1300-1306 — the paper's real
 * inputs are BWA-MEM seeds; the definition is DESIGN.md reading 17): gaps open from
 * the match state only, separate insertion / deletion costs, N scores -1, the band w (lowered by
 * BWA's max_ins / max_del bounds), per-row trimming to the previous row's nonzero extent + 2,
 * z-drop, the end-to-end score of the last query column, BWA's tie rules (first row, LAST column).
 *   q_words..t_len, fmt  [dev] packed pairs as for saloba_align_batch
 *   h0                   [dev] int32[n_pairs] seed scores, 1 .. 2^29
 *   params               [host] see saloba_ksw_params (|values| <= 2^10, w >= 0, zdrop >= 0)
 *   max_qlen             the longest query (sizes the per-warp row buffers; longer queries are
 *                        reported as invalid)
 *   out                  [dev] int32[7][n_pairs], rows: score (max), qle, tle (ends, exclusive;
 *                        0 when nothing beats h0), gtle, gscore (end-to-end score at the last query
 *                        column, -1 if no row reached it), max_off, clip (1: BWA-MEM keeps the
 *                        local extension, 0: it takes the end-to-end one: gscore > 0 and
 *                        gscore > score - end_bonus)
 *   status               [dev] int64[1]: -1 or the smallest invalid pair (length 0 or > 2^20, h0
 *                        out of range, query longer than max_qlen, values that could overflow
 *                        int32); such pairs get score -1 and -2 elsewhere
 * Asynchronous on `stream`; host-checked errors as
 * saloba_align_batch. */
int saloba_ksw_extend(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                      const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len, const int32_t* h0,
                      int64_t n_pairs, const saloba_ksw_params* params, saloba_packing fmt, int32_t max_qlen,
                      int32_t* out, void* workspace, size_t workspace_bytes, int64_t* status, void* stream);

/* ---- end-to-end from host buffers ----------------------------------------------------------- */

/* Host-resident ASCII pairs in, host results out (the call a read mapper makes).  The batch is cut
 * into slices; slice i+1 is uploaded on an internal copy stream while slice i is packed and aligned
 * on `stream`, and results are downloaded as slices finish.  Host buffers should be pinned
 * (cudaHostAlloc / torch pin_memory) for the copies to overlap.
 *   q_ascii, t_ascii  [host] uint8   concatenated sequences;  q_off, t_off [host] int64[n_pairs+1]
 *   h0                [host] int32[n_pairs] (EXTEND) or NULL (LOCAL)
 *   score, q_end, t_end [host] int32[n_pairs]      results in input order
 *   host_status       [host] int64: -1 or the smallest bad pair index (invalid base, empty or
 *                     over-long sequence, bad h0); outputs of such pairs are unspecified
 * The call synchronises `stream` before returning. */
typedef struct saloba_host_ctx saloba_host_ctx;

/* Device buffers, streams and events for batches of up to max_pairs pairs, max_q_bytes /
 * max_t_bytes ASCII bytes and queries of up to max_qlen bases, on `device`.  NULL on failure. */
saloba_host_ctx* saloba_host_ctx_create(int64_t max_pairs, int64_t max_q_bytes, int64_t max_t_bytes,
                                        int32_t max_qlen, int device);
void saloba_host_ctx_destroy(saloba_host_ctx* ctx);

/* Align one host batch with a context (allocation-free; SALOBA_EWORKSPACE if it exceeds the
 * context's capacity). */
int saloba_align_host_ctx(saloba_host_ctx* ctx, const uint8_t* q_ascii, const int64_t* q_off,
                          const uint8_t* t_ascii, const int64_t* t_off, const int32_t* h0, int64_t n_pairs,
                          saloba_scoring sc, saloba_mode mode, int32_t* score, int32_t* q_end, int32_t* t_end,
                          int64_t* host_status, const saloba_options* opt, void* stream);

/* Streaming host batches: two host contexts used alternately, so batch k+1's upload (and
 * packing) overlaps batch k's alignment and download — steady-state throughput is bounded by the
 * slower of the host-device link and the GPU, not by their sum.  Results of a batch are valid in
 * its host buffers after a later submit on the same context (two calls later) or after
 * saloba_stream_wait; *host_status is written then too.  Host buffers should be pinned and must
 * stay untouched until then.  Not thread-safe: one host thread per stream context. */
typedef struct saloba_stream_ctx saloba_stream_ctx;
saloba_stream_ctx* saloba_stream_create(int64_t max_pairs, int64_t max_q_bytes, int64_t max_t_bytes,
                                        int32_t max_qlen, int device);
void saloba_stream_destroy(saloba_stream_ctx* sctx);
/* Enqueue one batch (arguments as saloba_align_host_ctx, without a stream); blocks only to finish
 * the batch submitted two calls earlier.  Returns that finish's code, or a host-checked error. */
int saloba_stream_submit(saloba_stream_ctx* sctx, const uint8_t* q_ascii, const int64_t* q_off,
                         const uint8_t* t_ascii, const int64_t* t_off, const int32_t* h0, int64_t n_pairs,
                         saloba_scoring sc, saloba_mode mode, int32_t* score, int32_t* q_end, int32_t* t_end,
                         int64_t* host_status, const saloba_options* opt);
/* Wait for every submitted batch (their results and statuses are then valid). */
int saloba_stream_wait(saloba_stream_ctx* sctx);

/* Convenience: create a context sized for this batch, align, destroy. */
int saloba_align_host(const uint8_t* q_ascii, const int64_t* q_off, const uint8_t* t_ascii, const int64_t* t_off,
                      const int32_t* h0, int64_t n_pairs, saloba_scoring sc, saloba_mode mode, int32_t* score,
                      int32_t* q_end, int32_t* t_end, int64_t* host_status, const saloba_options* opt,
                      void* stream);

/* Static description of an error code. */
const char* saloba_strerror(int code);

/* SALOBA_VERSION of the built library. */
int saloba_version(void);

/* Diagnostics: number of this library's own kernels launched so far in this process (all devices;
 * CUB radix-sort launches are not counted).  Process-wide atomic counter. */
int64_t saloba_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* SALOBA_H */
