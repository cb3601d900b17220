// api.cu — host side of the C ABI: argument validation, workspace layout, launch plan, and the
// host-buffer end-to-end entry point.  No compute happens here; every step runs in kernels.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace saloba {

static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

cudaError_t run_classify_sort(const ClassifyArgs& ca, const SortKV& kv, int32_t* bin_start, int sms,
                              int32_t* long_gidx, int64_t cap16, int64_t coop_pairs, cudaStream_t s);
size_t cub_sort_temp_bytes(int64_t n);
void launch_status_init(int64_t* st, cudaStream_t s);
void launch_status_final(int64_t* st, cudaStream_t s);
void launch_dp_i32(int mode, int gidx, int grid, const AlignArgs& a, int bin, cudaStream_t s);
const void* dp_i32_kernel_ptr(int mode, int gidx, bool band, bool fast);
void launch_dp_i16(int mode, int gidx, int grid, const AlignArgs& a, int bin, cudaStream_t s);
const void* dp_i16_kernel_ptr(int mode, int gidx, int fmt, int rows);
const void* dp_i16_qn_kernel_ptr(int mode, int rows, int gidx);
void launch_dp_i16_qn(int mode, int gidx, int grid, const AlignArgs& a, cudaStream_t s);
const void* dp_g1_kernel_ptr(int mode, int fmt, bool qn, bool band);
int g1_threads();
const void* dp_coop_kernel_ptr(int mode, int fmt);
void launch_dp_coop(int mode, int grid, const AlignArgs& a, cudaStream_t s);
int coop_threads();
int coop_rows();
size_t g1_smem_bytes(bool qn);
void g1_set_smem_attrs();
int64_t g1_scratch_words(int64_t qcap);
void launch_dp_g1(int mode, int grid, const AlignArgs& a, int bin, bool qn, cudaStream_t s);
// the G = 1 int16x2 bins run the dedicated kernel of dp_g1.cu (16-row strips, banded variant);
// 8-row strips (Options.i16_rows = 8, an A/B knob) keep the generic dp_i16 kernel
static bool use_g1(int rows) { return rows != 8; }
void launch_reverse_prefix(int fmt, const uint32_t* words, const int64_t* word_off, const int32_t* end,
                           const int32_t* score, int64_t n, uint32_t* out, int32_t* out_len, int sms, cudaStream_t s);
void launch_start_finalize(const int32_t* score, const int32_t* q_end, const int32_t* t_end, const int32_t* rscore,
                           const int32_t* rq_end, const int32_t* rt_end, int64_t n, int32_t* q_start,
                           int32_t* t_start, int64_t* status, int sms, cudaStream_t s);
void launch_pack_range(const uint8_t* ascii, const int64_t* byte_off, int64_t n, int64_t base, int fmt,
                       uint32_t* words, int64_t cap, int64_t* word_off, int32_t* lens, int64_t* status,
                       cudaStream_t s);

// ---- per-device cache (computed once) ---------------------------------------------------------
struct DevInfo {
    bool init = false;
    int sms = 0;
    int major = 0;
    int blocks_i32[2][NGROUPS] = {};
    int blocks_i16[2][2][NGROUPS] = {};  // [rows 8|16][mode][gidx]
    int blocks_i16qn[2][2][2] = {};      // QN variant: [rows 8|16][mode][G = 1|2]
    int blocks_g1[2][2] = {};            // dp_g1 kernel: [mode][QN]
    int blocks_coop[2] = {};             // dp_coop_kernel (cooperative long pairs): [mode]
    int max_blocks_per_sm = 1;           // max resident blocks of any DP kernel (block-slot pool)
};
constexpr int NAUX = 4;
static std::mutex g_mu;
static DevInfo g_dev[64];

static const DevInfo* dev_info(int device) {
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    DevInfo& d = g_dev[device];
    if (!d.init) {
        if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return nullptr;
        cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, device);
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (int mode = 0; mode < 2; ++mode)
            for (int g = 0; g < NGROUPS; ++g) {
                int nb = 1;  // max over the plain / banded (NEXT-2) / FAST int32 variants
                for (int v = 0; v < 4; ++v) {
                    int x = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, dp_i32_kernel_ptr(mode, g, v & 1, v >> 1),
                                                                  BLOCK_THREADS, 0);
                    nb = std::max(nb, x);
                }
                d.blocks_i32[mode][g] = nb;
                for (int ri = 0; ri < 2; ++ri) {
                    nb = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp_i16_kernel_ptr(mode, g, SALOBA_PACK4, ri ? 16 : 8),
                                                                  I16_THREADS, 0);
                    d.blocks_i16[ri][mode][g] = std::max(1, nb);
                    if (g <= 1) {
                        nb = 0;
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp_i16_qn_kernel_ptr(mode, ri ? 16 : 8, g),
                                                                      I16_THREADS, 0);
                        d.blocks_i16qn[ri][mode][g] = std::max(1, nb);
                    }
                }
            }
        g1_set_smem_attrs();
        for (int mode = 0; mode < 2; ++mode) {
            int nb = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp_coop_kernel_ptr(mode, SALOBA_PACK4), coop_threads(), 0);
            d.blocks_coop[mode] = std::max(1, nb);
            d.max_blocks_per_sm = std::max(d.max_blocks_per_sm, d.blocks_coop[mode]);
        }
        for (int mode = 0; mode < 2; ++mode)
            for (int qn = 0; qn < 2; ++qn) {
                int nb = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp_g1_kernel_ptr(mode, SALOBA_PACK4, qn != 0, false),
                                                              g1_threads(), g1_smem_bytes(qn != 0));
                int nbb = 0;  // the banded variant (NEXT-2): the grid takes the smaller occupancy
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbb, dp_g1_kernel_ptr(mode, SALOBA_PACK4, false, true),
                                                              g1_threads(), g1_smem_bytes(false));
                if (nbb > 0) nb = std::min(nb, nbb);
                d.blocks_g1[mode][qn] = std::max(1, nb);
                d.max_blocks_per_sm = std::max(d.max_blocks_per_sm, d.blocks_g1[mode][qn]);
            }
        for (int mode = 0; mode < 2; ++mode)
            for (int g = 0; g < NGROUPS; ++g) {
                d.max_blocks_per_sm = std::max(d.max_blocks_per_sm, d.blocks_i32[mode][g]);
                for (int ri = 0; ri < 2; ++ri) {
                    d.max_blocks_per_sm = std::max(d.max_blocks_per_sm, d.blocks_i16[ri][mode][g]);
                    d.max_blocks_per_sm = std::max(d.max_blocks_per_sm, d.blocks_i16qn[ri][mode][0]);
                    d.max_blocks_per_sm = std::max(d.max_blocks_per_sm, d.blocks_i16qn[ri][mode][1]);
                }
            }
        cudaSetDevice(prev);
        d.init = true;
    }
    return &d;
}

// Auxiliary streams of one caller stream: the bins of a call run as concurrent kernels forked onto
// them and joined back (fork / join events created once with the set).  One set per (device,
// caller stream), created on first use, so calls on different streams or threads never share aux
// streams (they overlap instead of serialising, and a CUDA-graph capture on one stream does not
// pull in another stream's work).  Calls on the SAME stream share its set; the events then order
// a superset of each call's work, which is still correct.
struct AuxSet {
    cudaStream_t aux[NAUX] = {};
    cudaEvent_t fork = nullptr;
    cudaEvent_t join[NAUX] = {};
    bool init(int device) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        bool ok = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; i < NAUX && ok; ++i)
            ok = cudaStreamCreateWithFlags(&aux[i], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming) == cudaSuccess;
        cudaSetDevice(prev);
        return ok;
    }
    void destroy() {
        for (int i = 0; i < NAUX; ++i) {
            if (aux[i]) cudaStreamDestroy(aux[i]);
            if (join[i]) cudaEventDestroy(join[i]);
        }
        if (fork) cudaEventDestroy(fork);
    }
};
static std::mutex g_aux_mu;
static std::unordered_map<uint64_t, AuxSet*> g_aux;  // key: caller stream handle x device
static const AuxSet* aux_for(int device, cudaStream_t s) {
    const uint64_t key = reinterpret_cast<uint64_t>(s) * 64 + uint64_t(device);
    std::lock_guard<std::mutex> lk(g_aux_mu);
    auto it = g_aux.find(key);
    if (it != g_aux.end()) return it->second;
    AuxSet* a = new AuxSet();
    if (!a->init(device)) {
        a->destroy();
        delete a;
        return nullptr;
    }
    g_aux.emplace(key, a);
    return a;
}

int sm_count_current() {
    int dev = 0;
    cudaGetDevice(&dev);
    const DevInfo* d = dev_info(dev);
    return d ? d->sms : 148;
}

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- workspace layout -------------------------------------------------------------------------
struct Layout {
    size_t keys_in, keys_out, vals_in, vals_out, cub, cub_bytes, small, spill, total;
};

static int grid_for(const DevInfo* d, int mode, int path, int g, int rows = 16) {
    if (path == PATH_I16 && g == 0 && use_g1(rows)) return d->sms * d->blocks_g1[mode][0];
    return d->sms * (path == PATH_I16 ? d->blocks_i16[rows == 8 ? 0 : 1][mode][g] : d->blocks_i32[mode][g]);
}
static int threads_for(int path) { return path == PATH_I16 ? I16_THREADS : BLOCK_THREADS; }
// spill rows per subwarp slot: int32 path 2 buffers x (H, F); int16x2 path 4 interleaved (H, F) buffers
static int rows_for(int path) { return path == PATH_I16 ? 8 : 4; }

// spill words one resident block of bin (path, g) needs when the longest query has Qmax blocks
static int64_t block_need_words(int path, int g, int64_t Qmax) {
    const int64_t G = int64_t(1) << g;
    const int64_t q = std::min<int64_t>(qmax_for_gidx(g), Qmax);
    const int64_t generic = int64_t(threads_for(path)) / G * rows_for(path) * (8 * q + 8);
    // G = 1 int16x2 bins: the dp_g1 kernel's selector + spill scratch (dp_g1.cu), or the generic one;
    // the long bin: also the cooperative kernel's rows (dp_coop_kernel)
    if (path == PATH_I16 && g == 0) return std::max(generic, g1_scratch_words(q));
    if (path == PATH_I16 && g == NGROUPS - 1) return std::max(generic, int64_t(coop_rows()) * 2 * (8 * q + 8));
    return generic;
}
static int64_t block_slot_words(int64_t Qmax) {
    int64_t w = 0;
    for (int g = 0; g < NGROUPS; ++g)
        for (int path = 0; path < 2; ++path) w = std::max(w, block_need_words(path, g, Qmax));
    return (w + 63) / 64 * 64;
}
static int block_slots(const DevInfo* d) { return (d->sms * d->max_blocks_per_sm + 32 + 31) / 32 * 32; }  // whole bitmap words
static size_t spill_pool_bytes(const DevInfo* d, int64_t Qmax) {
    return size_t(block_slots(d)) * size_t(block_slot_words(Qmax)) * sizeof(int32_t);
}

static Layout layout(int64_t n, size_t spill_bytes) {
    Layout L{};
    size_t off = 0;
    const size_t nn = size_t(std::max<int64_t>(n, 1));
    L.keys_in = off; off = align_up(off + nn * 4, 256);
    L.keys_out = off; off = align_up(off + nn * 4, 256);
    L.vals_in = off; off = align_up(off + nn * 4, 256);
    L.vals_out = off; off = align_up(off + nn * 4, 256);
    L.cub_bytes = cub_sort_temp_bytes(n);
    L.cub = off; off = align_up(off + L.cub_bytes, 256);
    L.small = off; off = align_up(off + 1024, 256);
    L.spill = off; off = align_up(off + spill_bytes, 256);
    L.total = off;
    return L;
}

// largest query block count Qmax such that the layout fits in ws_bytes (0 if even Q=1 does not fit)
static int64_t max_q_blocks_for(const DevInfo* d, int64_t n, size_t ws_bytes) {
    const size_t fixed = layout(n, 0).total;
    if (ws_bytes < fixed) return 0;
    const size_t avail = ws_bytes - fixed;
    int64_t lo = 0, hi = MAX_LEN / 8;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (spill_pool_bytes(d, mid) <= avail) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

static bool scheme_ok(const saloba_scoring& sc) {
    const int lim = 1 << 10;
    return sc.match >= 1 && sc.match <= lim && sc.mismatch <= -1 && sc.mismatch >= -lim && sc.gap_extend >= 1 &&
           sc.gap_open >= sc.gap_extend && sc.gap_open <= lim;
}

}  // namespace saloba

using namespace saloba;


SALOBA_API size_t saloba_workspace_bytes(int64_t n_pairs, int32_t max_qlen, int32_t max_tlen, int device) {
    (void)max_tlen;
    const DevInfo* d = dev_info(device);
    if (!d || n_pairs < 0) return 0;
    const int64_t Qmax = (std::max(1, max_qlen) + 7) / 8;
    return layout(n_pairs, spill_pool_bytes(d, Qmax)).total;
}

static int gidx_of(int G) {
    switch (G) {
    case 1: return 0;
    case 2: return 1;
    case 4: return 2;
    case 8: return 3;
    case 16: return 4;
    case 32: return 5;
    default: return -2;
    }
}

// aux_in: the aux set the bins fork onto (nullptr: the caller stream's own set)
static int align_batch_impl(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                            const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len,
                            const int32_t* h0, int64_t n_pairs, saloba_scoring sc, saloba_mode mode,
                            saloba_packing fmt, int32_t* score, int32_t* q_end, int32_t* t_end, void* workspace,
                            size_t workspace_bytes, int64_t* status, const saloba_options* opt, void* stream,
                            const AuxSet* aux_in, const int32_t* band_w = nullptr) {
    if (n_pairs < 0 || n_pairs > int64_t(INT32_MAX) - 1024) return SALOBA_EINVAL;
    if (!status || !workspace) return SALOBA_EINVAL;
    if (n_pairs > 0 && (!q_words || !q_word_off || !q_len || !t_words || !t_word_off || !t_len || !score ||
                        !q_end || !t_end))
        return SALOBA_EINVAL;
    if (mode != SALOBA_LOCAL && mode != SALOBA_EXTEND) return SALOBA_EINVAL;
    if (mode == SALOBA_EXTEND && n_pairs > 0 && !h0) return SALOBA_EINVAL;
    if (fmt != SALOBA_PACK4 && fmt != SALOBA_PACK2) return SALOBA_EINVAL;
    if (!scheme_ok(sc)) return SALOBA_EINVAL;
    if (reinterpret_cast<uintptr_t>(workspace) % 256) return SALOBA_EINVAL;
    saloba_options o{};
    if (opt) o = *opt;
    int force_g = -1;
    if (o.force_group) {
        force_g = gidx_of(o.force_group);
        if (force_g < 0) return SALOBA_EINVAL;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SALOBA_ECUDA;
    const DevInfo* d = dev_info(dev);
    if (!d) return SALOBA_ECUDA;
    if (d->major < 10) return SALOBA_EUNSUPPORTED;

    const int64_t Qsup = max_q_blocks_for(d, n_pairs, workspace_bytes);
    if (Qsup < 1) return SALOBA_EWORKSPACE;
    const Layout L = layout(n_pairs, 0);
    char* ws = static_cast<char*>(workspace);
    cudaStream_t s = (cudaStream_t)stream;

    int32_t* small = reinterpret_cast<int32_t*>(ws + L.small);
    int32_t* bin_count = small;               // [NBINS]
    int32_t* bin_start = small + 32;          // [NBINS+1]
    int32_t* bin_counter = small + 64;        // [NBINS]
    int32_t* long_qmax = small + 240;         // max Q of the long bin
    int32_t* long_gidx = small + 241;         // group index chosen for the long bin
    if (cudaMemsetAsync(small, 0, 1024, s) != cudaSuccess) return SALOBA_ECUDA;
    launch_status_init(status, s);

    SortKV kv{reinterpret_cast<uint32_t*>(ws + L.keys_in), reinterpret_cast<uint32_t*>(ws + L.keys_out),
              reinterpret_cast<uint32_t*>(ws + L.vals_in), reinterpret_cast<uint32_t*>(ws + L.vals_out),
              ws + L.cub, L.cub_bytes};
    const int i16_rows = o.i16_rows == 8 ? 8 : I16_ROWS_DEFAULT;
    const int i32_fast = (sc.match <= 127 && sc.mismatch >= -128) ? 1 : 0;  // int8 substitution tables
    // Latency floor for small batches: at G = 1 every int16x2 lane holds two pairs, so a batch of
    // fewer pairs than resident lanes leaves most of the GPU idle and each pair takes its full
    // single-lane latency; the smallest G with (n/2)*G >= resident lanes spreads the pairs instead
    // (config 1, 1k pairs: the whole call becomes a few short chunks per pair).
    int min_gidx = 0;
    {
        const int64_t lanes = int64_t(grid_for(d, int(mode), PATH_I16, 0, i16_rows)) * I16_THREADS;
        const int64_t duos = (n_pairs + 1) / 2;
        if (duos > 0 && duos * 2 < lanes)
            while (min_gidx < NGROUPS - 1 && duos * (int64_t(1) << min_gidx) < lanes) ++min_gidx;
    }
    ClassifyArgs ca{q_words, q_word_off, int(fmt), sc.match, q_len, t_len, h0, n_pairs, int(mode), force_g,
                    o.force_path, o.keep_order, i16_rows, Qsup * 8, score, q_end, t_end, kv.keys_in,
                    kv.vals_in, bin_count, (unsigned long long*)status, long_qmax, band_w, i32_fast, min_gidx};
    const int64_t cap16 = int64_t(grid_for(d, int(mode), PATH_I16, NGROUPS - 2, i16_rows)) * (I16_THREADS / 16) * 2;
    // cooperative long-pair kernel below two waves of one-warp duos (SALOBA_COOP_PAIRS overrides: 0 = off)
    int64_t coop_pairs = int64_t(d->sms) * d->blocks_i16[1][int(mode)][NGROUPS - 1] * (I16_THREADS / 32) * 2 * 2;
    if (const char* e = getenv("SALOBA_COOP_PAIRS")) coop_pairs = atoll(e);
    if (i16_rows != 16) coop_pairs = 0;  // the cooperative kernel is built for 16-row strips
    if (run_classify_sort(ca, kv, bin_start, d->sms, long_gidx, cap16, coop_pairs, s) != cudaSuccess) return SALOBA_ECUDA;

    if (n_pairs > 0) {
        AlignArgs a{};
        a.q_words = q_words; a.q_word_off = q_word_off; a.q_len = q_len;
        a.t_words = t_words; a.t_word_off = t_word_off; a.t_len = t_len;
        a.h0 = h0; a.n_pairs = n_pairs;
        a.match = sc.match; a.mismatch = sc.mismatch; a.alpha = sc.gap_open; a.beta = sc.gap_extend;
        a.fmt = int(fmt);
        a.score = score; a.q_end = q_end; a.t_end = t_end;
        a.perm = kv.vals_out; a.bin_start = bin_start; a.bin_counter = bin_counter;
        a.spill = reinterpret_cast<int32_t*>(ws + L.spill);
        a.block_slot_words = block_slot_words(Qsup);
        a.slot_bitmap = reinterpret_cast<uint32_t*>(small + 96);
        a.slot_words = (block_slots(d) + 31) / 32;
        a.i16_rows = i16_rows;
        a.long_gidx = long_gidx;
        a.band_w = band_w;
        a.i32_fast = i32_fast;
        a.counters = o.counters;
        if (o.bin_counts) cudaMemcpyAsync(o.bin_counts, bin_count, NBINS * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        if (o.long_group) cudaMemcpyAsync(o.long_group, long_gidx, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        if (o.ev_dp_begin) cudaEventRecord((cudaEvent_t)o.ev_dp_begin, s);
        // All bins run as concurrent kernels (fork/join over the device's auxiliary streams), longest
        // bins first: a few long pairs then overlap the bulk of short ones instead of leaving most SMs
        // idle in a tail (§III-A load imbalance).  Blocks without work exit at once.
        const AuxSet* xs = aux_in ? aux_in : aux_for(dev, s);
        if (!xs) return SALOBA_ECUDA;
        const cudaStream_t* aux = xs->aux;
        cudaEventRecord(xs->fork, s);
        for (int i = 0; i < NAUX; ++i) cudaStreamWaitEvent(aux[i], xs->fork, 0);
        int j = 0;
        for (int path = PATH_I16; path >= PATH_I32; --path)
            for (int g = NGROUPS - 1; g >= 0; --g, ++j) {
                cudaStream_t as = aux[j % NAUX];
                a.spill_stride = 8 * std::min<int64_t>(qmax_for_gidx(g), Qsup) + 8;
                if (path == PATH_I16 && path * 8 + g == LONG_BIN) {
                    // the long bin: the cooperative kernel first (its blocks must be resident before
                    // the short bins' persistent kernels take the slots: it holds the critical path),
                    // then the one-warp kernel at both widths; the ones not chosen exit at once
                    if (i16_rows == 16) launch_dp_coop(int(mode), d->sms * d->blocks_coop[int(mode)], a, as);
                    launch_dp_i16(int(mode), g, grid_for(d, int(mode), path, g, i16_rows), a, LONG_BIN, as);
                    AlignArgs a16 = a;
                    a16.spill_stride = 8 * std::min<int64_t>(qmax_for_gidx(g - 1), Qsup) + 8;
                    launch_dp_i16(int(mode), g - 1, grid_for(d, int(mode), path, g - 1, i16_rows), a16, LONG_BIN, as);
                } else if (path == PATH_I16 && g == 0 && use_g1(i16_rows)) {
                    AlignArgs a1 = a;
                    a1.spill_stride = std::min<int64_t>(qmax_for_gidx(0), Qsup);  // dp_g1: query-block capacity
                    launch_dp_g1(int(mode), grid_for(d, int(mode), path, g, i16_rows), a1, path * 8 + g, false, as);
                } else if (path == PATH_I16)
                    launch_dp_i16(int(mode), g, grid_for(d, int(mode), path, g, i16_rows), a, path * 8 + g, as);
                else
                    launch_dp_i32(int(mode), g, grid_for(d, int(mode), path, g), a, path * 8 + g, as);
            }
        {   // int32 wide bin (values may reach 2^28, or scores beyond int8): the plain kernel, G = 32
            a.spill_stride = 8 * std::min<int64_t>(qmax_for_gidx(NGROUPS - 1), Qsup) + 8;
            launch_dp_i32(int(mode), NGROUPS - 1, grid_for(d, int(mode), PATH_I32, NGROUPS - 1), a, I32_WIDE_BIN,
                          aux[(j + 1) % NAUX]);
        }
        if (fmt == SALOBA_PACK4 && !band_w) {  // QN bins: int16x2 G=1 / G=2 pairs whose query contains N
                                               // (query-N pairs of banded calls run int32)
            for (int g = 0; g <= 1; ++g) {
                if (g == 0 && use_g1(i16_rows)) {
                    AlignArgs a1 = a;
                    a1.spill_stride = std::min<int64_t>(qmax_for_gidx(0), Qsup);
                    launch_dp_g1(int(mode), d->sms * d->blocks_g1[int(mode)][1], a1, QN_BIN, true, aux[(j + g) % NAUX]);
                    continue;
                }
                a.spill_stride = 8 * std::min<int64_t>(qmax_for_gidx(g), Qsup) + 8;
                launch_dp_i16_qn(int(mode), g, d->sms * d->blocks_i16qn[i16_rows == 8 ? 0 : 1][int(mode)][g], a,
                                 aux[(j + g) % NAUX]);
            }
        }
        for (int i = 0; i < NAUX; ++i) {
            cudaEventRecord(xs->join[i], aux[i]);
            cudaStreamWaitEvent(s, xs->join[i], 0);
        }
        if (o.ev_dp_end) cudaEventRecord((cudaEvent_t)o.ev_dp_end, s);
    }
    launch_status_final(status, s);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}

SALOBA_API int saloba_align_batch(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                                  const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len,
                                  const int32_t* h0, int64_t n_pairs, saloba_scoring sc, saloba_mode mode,
                                  saloba_packing fmt, int32_t* score, int32_t* q_end, int32_t* t_end,
                                  void* workspace, size_t workspace_bytes, int64_t* status,
                                  const saloba_options* opt, void* stream) {
    return align_batch_impl(q_words, q_word_off, q_len, t_words, t_word_off, t_len, h0, n_pairs, sc, mode, fmt, score,
                            q_end, t_end, workspace, workspace_bytes, status, opt, stream, nullptr);
}

// ---- banded DP ----------------------------------------------------------
SALOBA_API int saloba_align_banded(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                                   const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len,
                                   const int32_t* h0, const int32_t* band_w, int64_t n_pairs, saloba_scoring sc,
                                   saloba_mode mode, saloba_packing fmt, int32_t* score, int32_t* q_end,
                                   int32_t* t_end, void* workspace, size_t workspace_bytes, int64_t* status,
                                   const saloba_options* opt, void* stream) {
    if (n_pairs > 0 && !band_w) return SALOBA_EINVAL;
    return align_batch_impl(q_words, q_word_off, q_len, t_words, t_word_off, t_len, h0, n_pairs, sc, mode, fmt, score,
                            q_end, t_end, workspace, workspace_bytes, status, opt, stream, nullptr,
                            n_pairs > 0 ? band_w : nullptr);
}

// ---- start coordinates (LOCAL) -----------------------------------------
namespace {
struct StartLayout {
    size_t rq, rt, rql, rtl, rres, inner, total;
};
StartLayout start_layout(int64_t n, int64_t qw, int64_t tw) {
    StartLayout L{};
    const size_t nn = size_t(std::max<int64_t>(n, 1));
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t at = off;
        off = align_up(off + std::max<size_t>(bytes, 1), 256);
        return at;
    };
    L.rq = take(size_t(std::max<int64_t>(qw, 1)) * 4);
    L.rt = take(size_t(std::max<int64_t>(tw, 1)) * 4);
    L.rql = take(nn * 4);
    L.rtl = take(nn * 4);
    L.rres = take(3 * nn * 4);
    L.inner = off;
    L.total = off;
    return L;
}
}  // namespace

SALOBA_API size_t saloba_start_workspace_bytes(int64_t n_pairs, int64_t q_words_total, int64_t t_words_total,
                                               int32_t max_qlen, int device) {
    if (n_pairs < 0 || q_words_total < 0 || t_words_total < 0) return 0;
    const size_t inner = saloba_workspace_bytes(n_pairs, max_qlen, 0, device);
    if (!inner) return 0;
    return start_layout(n_pairs, q_words_total, t_words_total).total + inner;
}

SALOBA_API int saloba_locate_start(const uint32_t* q_words, const int64_t* q_word_off, int64_t q_words_total,
                                   const uint32_t* t_words, const int64_t* t_word_off, int64_t t_words_total,
                                   int64_t n_pairs, saloba_scoring sc, saloba_packing fmt, const int32_t* score,
                                   const int32_t* q_end, const int32_t* t_end, int32_t* q_start, int32_t* t_start,
                                   void* workspace, size_t workspace_bytes, int64_t* status,
                                   const saloba_options* opt, void* stream) {
    if (n_pairs < 0 || n_pairs > int64_t(INT32_MAX) - 1024 || !status || !workspace) return SALOBA_EINVAL;
    if (n_pairs > 0 && (!q_words || !q_word_off || !t_words || !t_word_off || !score || !q_end || !t_end ||
                        !q_start || !t_start || q_words_total < 1 || t_words_total < 1))
        return SALOBA_EINVAL;
    if (fmt != SALOBA_PACK4 && fmt != SALOBA_PACK2) return SALOBA_EINVAL;
    if (!scheme_ok(sc)) return SALOBA_EINVAL;
    if (reinterpret_cast<uintptr_t>(workspace) % 256) return SALOBA_EINVAL;
    const StartLayout L = start_layout(n_pairs, q_words_total, t_words_total);
    if (workspace_bytes <= L.total) return SALOBA_EWORKSPACE;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SALOBA_ECUDA;
    const DevInfo* d = dev_info(dev);
    if (!d) return SALOBA_ECUDA;
    char* ws = static_cast<char*>(workspace);
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t* rq = reinterpret_cast<uint32_t*>(ws + L.rq);
    uint32_t* rt = reinterpret_cast<uint32_t*>(ws + L.rt);
    int32_t* rql = reinterpret_cast<int32_t*>(ws + L.rql);
    int32_t* rtl = reinterpret_cast<int32_t*>(ws + L.rtl);
    int32_t* rres = reinterpret_cast<int32_t*>(ws + L.rres);
    const int64_t nn = std::max<int64_t>(n_pairs, 1);
    launch_reverse_prefix(int(fmt), q_words, q_word_off, q_end, score, n_pairs, rq, rql, d->sms, s);
    launch_reverse_prefix(int(fmt), t_words, t_word_off, t_end, score, n_pairs, rt, rtl, d->sms, s);
    // the reversed prefixes are aligned by the same schedule + DP kernels (LOCAL); `status`
    // receives that call's status, then finalize adds any pair whose reversed score differs
    const int rc = align_batch_impl(rq, q_word_off, rql, rt, t_word_off, rtl, nullptr, n_pairs, sc, SALOBA_LOCAL, fmt,
                                    rres, rres + nn, rres + 2 * nn, ws + L.inner, workspace_bytes - L.inner, status,
                                    opt, stream, nullptr);
    if (rc != SALOBA_OK) return rc;
    launch_start_finalize(score, q_end, t_end, rres, rres + nn, rres + 2 * nn, n_pairs, q_start, t_start, status,
                          d->sms, s);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}

// ---- end-to-end from host buffers -----------------------------------------------------------
namespace saloba {
__global__ void rebase_offsets(int64_t* off, int64_t n, int64_t base) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        off[k] -= base;
}
}  // namespace saloba

constexpr int HOST_SLICES = 16;  // capacity; the slice count and shape are per context
// Slice plan of the host path: SALOBA_HOST_SLICES slices (default 4, <= 16) whose sizes grow
// linearly (1, 2, 3, 4: the first upload is short) unless SALOBA_HOST_RAMP=0.  Measured on B200
// (config 2, tools/diag_e2e.py): 4 ramped slices 12.4-11.8 ms, 8 equal 13.0-13.3 ms, 16 equal 15.8 ms.
static void host_slice_fracs(int& nsl, double* frac) {
    const char* e = getenv("SALOBA_HOST_SLICES");
    nsl = (e && *e) ? std::max(1, std::min(HOST_SLICES, atoi(e))) : 4;
    const char* r = getenv("SALOBA_HOST_RAMP");
    const bool ramp = !(r && *r == '0');
    double tot = 0;
    for (int i = 0; i < nsl; ++i) tot += ramp ? double(i + 1) : 1.0;
    double acc = 0;
    frac[0] = 0;
    for (int i = 0; i < nsl; ++i) {
        acc += ramp ? double(i + 1) : 1.0;
        frac[i + 1] = acc / tot;
    }
}

struct saloba_host_ctx {
    int device = 0;
    int64_t max_pairs = 0, max_q_bytes = 0, max_t_bytes = 0;
    int32_t max_qlen = 0;
    int64_t slice_pairs = 0;
    size_t ws_bytes = 0;
    void *q = nullptr, *t = nullptr, *qo = nullptr, *to = nullptr, *qw = nullptr, *tw = nullptr, *qwo = nullptr,
         *two = nullptr, *ql = nullptr, *tl = nullptr, *h0 = nullptr, *res = nullptr, *st = nullptr;
    // two compute pipelines (workspace + stream + auxiliary streams) so that slice i+1 packs and
    // aligns while slice i drains
    void* ws[2] = {nullptr, nullptr};
    cudaStream_t cs[2] = {nullptr, nullptr};
    AuxSet aux[2];
    cudaEvent_t fork = nullptr, pjoin[2] = {nullptr, nullptr};
    int64_t qwcap = 0, twcap = 0;
    cudaStream_t copy = nullptr, down = nullptr;
    cudaEvent_t up[HOST_SLICES], done[HOST_SLICES];
    int64_t* hst = nullptr;  // pinned status readback
    // the batch enqueued last and not yet finished (saloba_stream_*: several contexts in flight)
    struct Pending {
        bool active = false;
        int nsl = 0, rc = SALOBA_OK;
        int64_t cut[HOST_SLICES + 1] = {};
        const int64_t *q_off = nullptr, *t_off = nullptr;
        int64_t qb0 = 0, tb0 = 0, n_pairs = 0;
        cudaStream_t s = nullptr;
        int64_t* host_status = nullptr;
    } pend;
};

SALOBA_API void saloba_host_ctx_destroy(saloba_host_ctx* c) {
    if (!c) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    void* bufs[] = {c->q, c->t, c->qo, c->to, c->qw, c->tw, c->qwo, c->two, c->ql, c->tl, c->h0, c->res, c->ws[0], c->ws[1], c->st};
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (int p = 0; p < 2; ++p) {
        if (c->cs[p]) cudaStreamDestroy(c->cs[p]);
        c->aux[p].destroy();
        if (c->pjoin[p]) cudaEventDestroy(c->pjoin[p]);
    }
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->copy) {
        for (int i = 0; i < HOST_SLICES; ++i) {
            cudaEventDestroy(c->up[i]);
            cudaEventDestroy(c->done[i]);
        }
        cudaStreamDestroy(c->copy);
    }
    if (c->down) cudaStreamDestroy(c->down);
    if (c->hst) cudaFreeHost(c->hst);
    cudaSetDevice(prev);
    delete c;
}

SALOBA_API saloba_host_ctx* saloba_host_ctx_create(int64_t max_pairs, int64_t max_q_bytes, int64_t max_t_bytes,
                                                   int32_t max_qlen, int device) {
    if (max_pairs < 0 || max_q_bytes < 0 || max_t_bytes < 0 || max_qlen < 1) return nullptr;
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) return nullptr;
    saloba_host_ctx* c = new saloba_host_ctx();
    c->device = device;
    c->max_pairs = max_pairs;
    c->max_q_bytes = max_q_bytes;
    c->max_t_bytes = max_t_bytes;
    c->max_qlen = max_qlen;
    {
        int nsl = 8;
        double fr[HOST_SLICES + 1];
        host_slice_fracs(nsl, fr);
        double mx = 0;
        for (int i = 0; i < nsl; ++i) mx = std::max(mx, fr[i + 1] - fr[i]);
        c->slice_pairs = int64_t(double(max_pairs) * mx) + 2;
    }
    c->qwcap = saloba_packed_words(max_q_bytes, max_pairs, SALOBA_PACK4);
    c->twcap = saloba_packed_words(max_t_bytes, max_pairs, SALOBA_PACK4);
    c->ws_bytes = saloba_workspace_bytes(std::max<int64_t>(c->slice_pairs, 1), max_qlen, 0, device);
    auto al = [](void** p, size_t n) { return cudaMalloc(p, std::max<size_t>(n, 256)) == cudaSuccess; };
    const int64_t np1 = max_pairs + 1;
    bool ok = c->ws_bytes > 0 && al(&c->q, max_q_bytes) && al(&c->t, max_t_bytes) && al(&c->qo, np1 * 8) &&
              al(&c->to, np1 * 8) && al(&c->qw, c->qwcap * 4) && al(&c->tw, c->twcap * 4) && al(&c->qwo, np1 * 8) &&
              al(&c->two, np1 * 8) && al(&c->ql, max_pairs * 4) && al(&c->tl, max_pairs * 4) &&
              al(&c->h0, max_pairs * 4) && al(&c->res, max_pairs * 12) && al(&c->ws[0], c->ws_bytes) &&
              al(&c->ws[1], c->ws_bytes) &&
              al(&c->st, 4 * HOST_SLICES * 8) &&
              cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->down, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMallocHost((void**)&c->hst, 4 * HOST_SLICES * 8) == cudaSuccess;
    if (ok && c->copy) {
        for (int i = 0; i < HOST_SLICES; ++i) {
            cudaEventCreateWithFlags(&c->up[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&c->done[i], cudaEventDisableTiming);
        }
        for (int p = 0; p < 2; ++p) {
            cudaStreamCreateWithFlags(&c->cs[p], cudaStreamNonBlocking);
            ok = ok && c->aux[p].init(device);
            cudaEventCreateWithFlags(&c->pjoin[p], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
    }
    cudaSetDevice(prev);
    if (!ok) {
        saloba_host_ctx_destroy(c);
        return nullptr;
    }
    return c;
}

namespace {
int64_t pair_of_byte(const int64_t* off, int64_t n, int64_t byte) {  // k with off[k] <= byte < off[k+1]
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (off[mid] <= byte) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
}  // namespace

// Enqueue one host batch on a context (no host synchronisation); host_finish() waits for it and
// fills *host_status.  saloba_align_host_ctx = enqueue + finish; saloba_stream_* keeps two contexts
// in flight so one batch's upload overlaps the previous batch's compute.
static int host_enqueue(saloba_host_ctx* c, const uint8_t* q_ascii, const int64_t* q_off, const uint8_t* t_ascii,
                        const int64_t* t_off, const int32_t* h0, int64_t n_pairs, saloba_scoring sc,
                        saloba_mode mode, int32_t* score, int32_t* q_end, int32_t* t_end, int64_t* host_status,
                        const saloba_options* opt, void* stream, bool allow_trace) {
    if (!c || n_pairs < 0 || !q_off || !t_off || !host_status) return SALOBA_EINVAL;
    if (n_pairs > 0 && (!q_ascii || !t_ascii || !score || !q_end || !t_end)) return SALOBA_EINVAL;
    if (mode == SALOBA_EXTEND && n_pairs > 0 && !h0) return SALOBA_EINVAL;
    if (!scheme_ok(sc)) return SALOBA_EINVAL;
    *host_status = -1;
    if (n_pairs == 0) return SALOBA_OK;
    const int64_t qb0 = q_off[0], tb0 = t_off[0];
    const int64_t qbytes = q_off[n_pairs] - qb0, tbytes = t_off[n_pairs] - tb0;
    if (n_pairs > c->max_pairs || qbytes > c->max_q_bytes || tbytes > c->max_t_bytes) return SALOBA_EWORKSPACE;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;

    int nsl = 8;
    double fr[HOST_SLICES + 1];
    host_slice_fracs(nsl, fr);
    nsl = int(std::min<int64_t>(nsl, n_pairs));
    int64_t cut[HOST_SLICES + 1];
    for (int i = 0; i <= nsl; ++i) cut[i] = i == nsl ? n_pairs : std::min<int64_t>(n_pairs, int64_t(double(n_pairs) * fr[i]));
    for (int i = 1; i <= nsl; ++i) cut[i] = std::max(cut[i], cut[i - 1] + 1);  // no empty slice
    cut[nsl] = n_pairs;
    uint8_t* qd = static_cast<uint8_t*>(c->q);
    uint8_t* td = static_cast<uint8_t*>(c->t);
    int64_t* qo = static_cast<int64_t*>(c->qo);
    int64_t* to = static_cast<int64_t*>(c->to);
    int64_t* st = static_cast<int64_t*>(c->st);
    int32_t* res = static_cast<int32_t*>(c->res);
    int32_t* h0d = h0 ? static_cast<int32_t*>(c->h0) : nullptr;

    // the two compute pipelines start after everything already queued on the caller's stream
    cudaEventRecord(c->fork, s);
    cudaStreamWaitEvent(c->cs[0], c->fork, 0);
    cudaStreamWaitEvent(c->cs[1], c->fork, 0);
    // offsets (8 B per pair) and h0 first; rebased on the device so the host never touches them
    cudaMemcpyAsync(qo, q_off, (n_pairs + 1) * 8, cudaMemcpyHostToDevice, c->copy);
    cudaMemcpyAsync(to, t_off, (n_pairs + 1) * 8, cudaMemcpyHostToDevice, c->copy);
    if (h0) cudaMemcpyAsync(h0d, h0, n_pairs * 4, cudaMemcpyHostToDevice, c->copy);
    if (qb0 || tb0) {
        rebase_offsets<<<64, 256, 0, c->copy>>>(qo, n_pairs + 1, qb0);
        rebase_offsets<<<64, 256, 0, c->copy>>>(to, n_pairs + 1, tb0);
        count_launches(2);
    }
    int rc = SALOBA_OK;
    // optional timeline (SALOBA_TRACE=1): upload-done / compute-start / compute-end per slice
    static const bool trace = getenv("SALOBA_TRACE") != nullptr;
    cudaEvent_t tr0 = nullptr, tup[HOST_SLICES] = {}, tcs[HOST_SLICES] = {}, tce[HOST_SLICES] = {};
    if (trace) {
        cudaEventCreate(&tr0);
        cudaEventRecord(tr0, c->copy);
        for (int i = 0; i < nsl; ++i) {
            cudaEventCreate(&tup[i]);
            cudaEventCreate(&tcs[i]);
            cudaEventCreate(&tce[i]);
        }
    }
    for (int i = 0; i < nsl && rc == SALOBA_OK; ++i) {
        const int64_t a0 = cut[i], a1 = cut[i + 1], na = a1 - a0;
        const int64_t qs = q_off[a0] - qb0, qe = q_off[a1] - qb0, ts = t_off[a0] - tb0, te = t_off[a1] - tb0;
        cudaMemcpyAsync(qd + qs, q_ascii + q_off[a0], qe - qs, cudaMemcpyHostToDevice, c->copy);
        cudaMemcpyAsync(td + ts, t_ascii + t_off[a0], te - ts, cudaMemcpyHostToDevice, c->copy);
        cudaEventRecord(c->up[i], c->copy);
        if (trace) cudaEventRecord(tup[i], c->copy);
        const int pp = i & 1;
        cudaStream_t ps = c->cs[pp];
        cudaStreamWaitEvent(ps, c->up[i], 0);
        if (trace) cudaEventRecord(tcs[i], ps);
        launch_pack_range(qd, qo + a0, na, a0, SALOBA_PACK4, static_cast<uint32_t*>(c->qw), c->qwcap,
                          static_cast<int64_t*>(c->qwo) + a0, static_cast<int32_t*>(c->ql) + a0, st + 4 * i + 0, ps);
        launch_pack_range(td, to + a0, na, a0, SALOBA_PACK4, static_cast<uint32_t*>(c->tw), c->twcap,
                          static_cast<int64_t*>(c->two) + a0, static_cast<int32_t*>(c->tl) + a0, st + 4 * i + 1, ps);
        rc = align_batch_impl(static_cast<uint32_t*>(c->qw), static_cast<int64_t*>(c->qwo) + a0,
                              static_cast<int32_t*>(c->ql) + a0, static_cast<uint32_t*>(c->tw),
                              static_cast<int64_t*>(c->two) + a0, static_cast<int32_t*>(c->tl) + a0,
                              h0d ? h0d + a0 : nullptr, na, sc, mode, SALOBA_PACK4, res + a0, res + n_pairs + a0,
                              res + 2 * n_pairs + a0, c->ws[pp], c->ws_bytes, st + 4 * i + 2, opt, ps, &c->aux[pp]);
        cudaEventRecord(c->done[i], ps);
        if (trace) cudaEventRecord(tce[i], ps);
        cudaStreamWaitEvent(c->down, c->done[i], 0);
        cudaMemcpyAsync(score + a0, res + a0, na * 4, cudaMemcpyDeviceToHost, c->down);
        cudaMemcpyAsync(q_end + a0, res + n_pairs + a0, na * 4, cudaMemcpyDeviceToHost, c->down);
        cudaMemcpyAsync(t_end + a0, res + 2 * n_pairs + a0, na * 4, cudaMemcpyDeviceToHost, c->down);
    }
    cudaMemcpyAsync(c->hst, st, sizeof(int64_t) * 4 * nsl, cudaMemcpyDeviceToHost, c->down);
    for (int p = 0; p < 2; ++p) {  // the caller's stream resumes after both pipelines
        cudaEventRecord(c->pjoin[p], c->cs[p]);
        cudaStreamWaitEvent(s, c->pjoin[p], 0);
    }
    if (trace && allow_trace) {
        cudaStreamSynchronize(s);
        for (int i = 0; i < nsl; ++i) {
            float u = 0, cs = 0, ce = 0;
            cudaEventElapsedTime(&u, tr0, tup[i]);
            cudaEventElapsedTime(&cs, tr0, tcs[i]);
            cudaEventElapsedTime(&ce, tr0, tce[i]);
            fprintf(stderr, "[saloba trace] slice %d: upload done %.3f ms, compute %.3f -> %.3f ms\n", i, u, cs, ce);
        }
    }
    if (trace) {
        for (int i = 0; i < nsl; ++i) {
            cudaEventDestroy(tup[i]);
            cudaEventDestroy(tcs[i]);
            cudaEventDestroy(tce[i]);
        }
        cudaEventDestroy(tr0);
    }
    cudaSetDevice(prev);
    auto& P = c->pend;
    P.active = true;
    P.nsl = nsl;
    P.rc = rc;
    for (int i = 0; i <= nsl; ++i) P.cut[i] = cut[i];
    P.q_off = q_off;
    P.t_off = t_off;
    P.qb0 = qb0;
    P.tb0 = tb0;
    P.n_pairs = n_pairs;
    P.s = s;
    P.host_status = host_status;
    return rc;
}

static int host_finish(saloba_host_ctx* c) {
    auto& P = c->pend;
    if (!P.active) return SALOBA_OK;
    P.active = false;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->copy);
    const cudaError_t e = cudaStreamSynchronize(c->down);
    cudaStreamSynchronize(P.s);
    cudaSetDevice(prev);
    if (P.rc != SALOBA_OK) return P.rc;
    if (e != cudaSuccess) return SALOBA_ECUDA;
    int64_t bad = INT64_MAX;
    for (int i = 0; i < P.nsl; ++i) {
        if (c->hst[4 * i + 0] >= 0) bad = std::min(bad, pair_of_byte(P.q_off, P.n_pairs, c->hst[4 * i + 0] + P.qb0));
        if (c->hst[4 * i + 1] >= 0) bad = std::min(bad, pair_of_byte(P.t_off, P.n_pairs, c->hst[4 * i + 1] + P.tb0));
        if (c->hst[4 * i + 2] >= 0) bad = std::min(bad, P.cut[i] + c->hst[4 * i + 2]);
    }
    *P.host_status = bad == INT64_MAX ? -1 : bad;
    return SALOBA_OK;
}

SALOBA_API int saloba_align_host_ctx(saloba_host_ctx* c, const uint8_t* q_ascii, const int64_t* q_off,
                                     const uint8_t* t_ascii, const int64_t* t_off, const int32_t* h0, int64_t n_pairs,
                                     saloba_scoring sc, saloba_mode mode, int32_t* score, int32_t* q_end,
                                     int32_t* t_end, int64_t* host_status, const saloba_options* opt, void* stream) {
    if (!c) return SALOBA_EINVAL;
    const int rf = host_finish(c);  // a batch left in flight by the streaming API
    if (rf != SALOBA_OK) return rf;
    const int rc = host_enqueue(c, q_ascii, q_off, t_ascii, t_off, h0, n_pairs, sc, mode, score, q_end, t_end,
                                host_status, opt, stream, true);
    if (rc != SALOBA_OK) {
        c->pend.active = false;
        return rc;
    }
    return host_finish(c);
}

// ---- streaming host batches (two host contexts in flight) -------------------------------------
struct saloba_stream_ctx {
    saloba_host_ctx* h[2] = {nullptr, nullptr};
    cudaStream_t s[2] = {nullptr, nullptr};  // private caller streams (the legacy stream would serialise)
    int64_t submitted = 0;
    int device = 0;
};

SALOBA_API void saloba_stream_destroy(saloba_stream_ctx* x) {
    if (!x) return;
    for (int i = 0; i < 2; ++i) {
        if (x->h[i]) {
            host_finish(x->h[i]);
            saloba_host_ctx_destroy(x->h[i]);
        }
        if (x->s[i]) cudaStreamDestroy(x->s[i]);
    }
    delete x;
}

SALOBA_API saloba_stream_ctx* saloba_stream_create(int64_t max_pairs, int64_t max_q_bytes, int64_t max_t_bytes,
                                                   int32_t max_qlen, int device) {
    saloba_stream_ctx* x = new saloba_stream_ctx();
    x->device = device;
    int prev = 0;
    cudaGetDevice(&prev);
    bool ok = cudaSetDevice(device) == cudaSuccess;
    for (int i = 0; i < 2 && ok; ++i) {
        x->h[i] = saloba_host_ctx_create(max_pairs, max_q_bytes, max_t_bytes, max_qlen, device);
        ok = x->h[i] != nullptr && cudaStreamCreateWithFlags(&x->s[i], cudaStreamNonBlocking) == cudaSuccess;
    }
    cudaSetDevice(prev);
    if (!ok) {
        saloba_stream_destroy(x);
        return nullptr;
    }
    return x;
}

SALOBA_API int saloba_stream_submit(saloba_stream_ctx* x, const uint8_t* q_ascii, const int64_t* q_off,
                                    const uint8_t* t_ascii, const int64_t* t_off, const int32_t* h0, int64_t n_pairs,
                                    saloba_scoring sc, saloba_mode mode, int32_t* score, int32_t* q_end,
                                    int32_t* t_end, int64_t* host_status, const saloba_options* opt) {
    if (!x || !host_status) return SALOBA_EINVAL;
    const int slot = int(x->submitted & 1);
    saloba_host_ctx* c = x->h[slot];
    const int rf = host_finish(c);  // the batch submitted two calls ago on this context
    if (rf != SALOBA_OK) return rf;
    const int rc = host_enqueue(c, q_ascii, q_off, t_ascii, t_off, h0, n_pairs, sc, mode, score, q_end, t_end,
                                host_status, opt, x->s[slot], false);
    if (rc != SALOBA_OK) {
        c->pend.active = false;
        return rc;
    }
    ++x->submitted;
    return SALOBA_OK;
}

SALOBA_API int saloba_stream_wait(saloba_stream_ctx* x) {
    if (!x) return SALOBA_EINVAL;
    int rc = SALOBA_OK;
    for (int k = 0; k < 2; ++k) {  // the older batch first
        const int r = host_finish(x->h[int((x->submitted + k) & 1)]);
        if (r != SALOBA_OK && rc == SALOBA_OK) rc = r;
    }
    return rc;
}

SALOBA_API int saloba_align_host(const uint8_t* q_ascii, const int64_t* q_off, const uint8_t* t_ascii,
                                 const int64_t* t_off, const int32_t* h0, int64_t n_pairs, saloba_scoring sc,
                                 saloba_mode mode, int32_t* score, int32_t* q_end, int32_t* t_end,
                                 int64_t* host_status, const saloba_options* opt, void* stream) {
    if (n_pairs < 0 || !q_off || !t_off || !host_status) return SALOBA_EINVAL;
    if (n_pairs == 0) {
        *host_status = -1;
        return SALOBA_OK;
    }
    int32_t max_q = 1;
    for (int64_t k = 0; k < n_pairs; ++k) max_q = std::max<int32_t>(max_q, int32_t(q_off[k + 1] - q_off[k]));
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SALOBA_ECUDA;
    saloba_host_ctx* c = saloba_host_ctx_create(n_pairs, q_off[n_pairs] - q_off[0], t_off[n_pairs] - t_off[0], max_q, dev);
    if (!c) return SALOBA_ECUDA;
    const int rc = saloba_align_host_ctx(c, q_ascii, q_off, t_ascii, t_off, h0, n_pairs, sc, mode, score, q_end, t_end,
                                         host_status, opt, stream);
    saloba_host_ctx_destroy(c);
    return rc;
}

SALOBA_API const char* saloba_strerror(int code) {
    switch (code) {
    case SALOBA_OK: return "ok";
    case SALOBA_EINVAL: return "invalid argument";
    case SALOBA_ECUDA: return "CUDA runtime error";
    case SALOBA_EWORKSPACE: return "workspace too small";
    case SALOBA_EUNSUPPORTED: return "unsupported device or feature";
    default: return "unknown error";
    }
}

SALOBA_API int saloba_version(void) { return SALOBA_VERSION; }

SALOBA_API int64_t saloba_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }
