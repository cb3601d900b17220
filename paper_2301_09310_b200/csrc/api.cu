// api.cu — host side of the C ABI: argument validation, workspace layout, launch plan, and the
// host-buffer end-to-end entry point.  No compute happens here; every step runs in kernels.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace saloba {

static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

cudaError_t run_classify_sort(const ClassifyArgs& ca, const SortKV& kv, int32_t* bin_start, int sms, cudaStream_t s);
size_t cub_sort_temp_bytes(int64_t n);
void launch_status_init(int64_t* st, cudaStream_t s);
void launch_status_final(int64_t* st, cudaStream_t s);
void launch_dp_i32(int mode, int gidx, int grid, const AlignArgs& a, int bin, cudaStream_t s);
const void* dp_i32_kernel_ptr(int mode, int gidx);
void launch_dp_i16(int mode, int gidx, int grid, const AlignArgs& a, int bin, cudaStream_t s);
const void* dp_i16_kernel_ptr(int mode, int gidx, int fmt);
void launch_pack_range(const uint8_t* ascii, const int64_t* byte_off, int64_t n, int64_t base, int fmt,
                       uint32_t* words, int64_t* word_off, int32_t* lens, int64_t* status, cudaStream_t s);

// ---- per-device cache (computed once) ---------------------------------------------------------
struct DevInfo {
    bool init = false;
    int sms = 0;
    int major = 0;
    int blocks_i32[2][NGROUPS] = {};
    int blocks_i16[2][NGROUPS] = {};
};
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
                int nb = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp_i32_kernel_ptr(mode, g), BLOCK_THREADS, 0);
                d.blocks_i32[mode][g] = std::max(1, nb);
                nb = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp_i16_kernel_ptr(mode, g, SALOBA_PACK4), I16_THREADS, 0);
                d.blocks_i16[mode][g] = std::max(1, nb);
            }
        cudaSetDevice(prev);
        d.init = true;
    }
    return &d;
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

static int grid_for(const DevInfo* d, int mode, int path, int g) {
    return d->sms * (path == PATH_I16 ? d->blocks_i16[mode][g] : d->blocks_i32[mode][g]);
}
static int threads_for(int path) { return path == PATH_I16 ? I16_THREADS : BLOCK_THREADS; }
// spill rows per subwarp slot: int32 path 2 buffers x (H, F); int16x2 path 4 buffers x (H, F) + selectors
static int rows_for(int path) { return path == PATH_I16 ? 9 : 4; }

// bytes of spill pool the bin (mode, path, g) needs when the longest query has Qmax blocks
static size_t spill_need(const DevInfo* d, int mode, int path, int g, int64_t Qmax) {
    const int64_t G = int64_t(1) << g;
    const int64_t slots = int64_t(grid_for(d, mode, path, g)) * threads_for(path) / G;
    const int64_t q = std::min<int64_t>(qmax_for_gidx(g), Qmax);
    const int64_t stride = 8 * q + 8;
    return size_t(slots) * rows_for(path) * size_t(stride) * sizeof(int32_t);
}

static size_t spill_pool_bytes(const DevInfo* d, int64_t Qmax) {
    size_t need = 0;
    for (int mode = 0; mode < 2; ++mode)
        for (int g = 0; g < NGROUPS; ++g)
            for (int path = 0; path < 2; ++path) need = std::max(need, spill_need(d, mode, path, g, Qmax));
    return need;
}

static Layout layout(int64_t n, size_t spill_bytes) {
    Layout L{};
    size_t off = 0;
    const size_t nn = size_t(std::max<int64_t>(n, 1));
    L.keys_in = off; off = align_up(off + nn * 8, 256);
    L.keys_out = off; off = align_up(off + nn * 8, 256);
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

SALOBA_API int saloba_align_batch(const uint32_t* q_words, const int64_t* q_word_off, const int32_t* q_len,
                                  const uint32_t* t_words, const int64_t* t_word_off, const int32_t* t_len,
                                  const int32_t* h0, int64_t n_pairs, saloba_scoring sc, saloba_mode mode,
                                  saloba_packing fmt, int32_t* score, int32_t* q_end, int32_t* t_end,
                                  void* workspace, size_t workspace_bytes, int64_t* status,
                                  const saloba_options* opt, void* stream) {
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
    if (cudaMemsetAsync(small, 0, 1024, s) != cudaSuccess) return SALOBA_ECUDA;
    launch_status_init(status, s);

    SortKV kv{reinterpret_cast<uint64_t*>(ws + L.keys_in), reinterpret_cast<uint64_t*>(ws + L.keys_out),
              reinterpret_cast<uint32_t*>(ws + L.vals_in), reinterpret_cast<uint32_t*>(ws + L.vals_out),
              ws + L.cub, L.cub_bytes};
    ClassifyArgs ca{q_words, q_word_off, int(fmt), sc.match, q_len, t_len, h0, n_pairs, int(mode), force_g, o.force_path, o.keep_order, Qsup * 8,
                    score, q_end, t_end, kv.keys_in, kv.vals_in, bin_count, (unsigned long long*)status};
    if (run_classify_sort(ca, kv, bin_start, d->sms, s) != cudaSuccess) return SALOBA_ECUDA;

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
        if (o.bin_counts) cudaMemcpyAsync(o.bin_counts, bin_count, NBINS * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        if (o.ev_dp_begin) cudaEventRecord((cudaEvent_t)o.ev_dp_begin, s);
        for (int path = PATH_I16; path >= PATH_I32; --path)
            for (int g = NGROUPS - 1; g >= 0; --g) {
                a.spill_stride = 8 * std::min<int64_t>(qmax_for_gidx(g), Qsup) + 8;
                if (path == PATH_I16)
                    launch_dp_i16(int(mode), g, grid_for(d, int(mode), path, g), a, path * 8 + g, s);
                else
                    launch_dp_i32(int(mode), g, grid_for(d, int(mode), path, g), a, path * 8 + g, s);
            }
        if (o.ev_dp_end) cudaEventRecord((cudaEvent_t)o.ev_dp_end, s);
    }
    launch_status_final(status, s);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}

// ---- end-to-end from host buffers -----------------------------------------------------------
namespace {
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(n, 256)); }
};

int64_t first_pair_of_byte(const int64_t* off, int64_t n, int64_t byte) {
    // pair k with off[k] <= byte < off[k+1]
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (off[mid] <= byte) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
}  // namespace

SALOBA_API int saloba_align_host(const uint8_t* q_ascii, const int64_t* q_off, const uint8_t* t_ascii,
                                 const int64_t* t_off, const int32_t* h0, int64_t n_pairs, saloba_scoring sc,
                                 saloba_mode mode, int32_t* score, int32_t* q_end, int32_t* t_end,
                                 int64_t* host_status, const saloba_options* opt, void* stream) {
    if (n_pairs < 0 || !q_off || !t_off || !host_status) return SALOBA_EINVAL;
    if (n_pairs > 0 && (!q_ascii || !t_ascii || !score || !q_end || !t_end)) return SALOBA_EINVAL;
    if (mode == SALOBA_EXTEND && n_pairs > 0 && !h0) return SALOBA_EINVAL;
    if (!scheme_ok(sc)) return SALOBA_EINVAL;
    *host_status = -1;
    if (n_pairs == 0) return SALOBA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SALOBA_ECUDA;

    const int64_t qbytes = q_off[n_pairs] - q_off[0], tbytes = t_off[n_pairs] - t_off[0];
    int32_t max_q = 1;
    for (int64_t k = 0; k < n_pairs; ++k) max_q = std::max<int32_t>(max_q, int32_t(q_off[k + 1] - q_off[k]));

    // slices of ~equal bytes, at least 4 MB each, up to 8
    const int64_t total = qbytes + tbytes;
    int nslices = int(std::min<int64_t>(8, std::max<int64_t>(1, total / (4 << 20))));
    nslices = int(std::min<int64_t>(nslices, n_pairs));
    std::vector<int64_t> cut(nslices + 1);
    for (int i = 0; i <= nslices; ++i) cut[i] = n_pairs * i / nslices;
    int64_t max_slice = 0;
    for (int i = 0; i < nslices; ++i) max_slice = std::max(max_slice, cut[i + 1] - cut[i]);

    DevBuf dq, dt, dqo, dto, dqw, dtw, dqwo, dtwo, dql, dtl, dh0, dres, dws, dst;
    const int64_t qwcap = saloba_packed_words(qbytes, n_pairs, SALOBA_PACK4);
    const int64_t twcap = saloba_packed_words(tbytes, n_pairs, SALOBA_PACK4);
    const size_t wsb = saloba_workspace_bytes(max_slice, max_q, 0, dev);
    if (dq.alloc(qbytes) || dt.alloc(tbytes) || dqo.alloc((n_pairs + 1) * 8) || dto.alloc((n_pairs + 1) * 8) ||
        dqw.alloc(qwcap * 4) || dtw.alloc(twcap * 4) || dqwo.alloc((n_pairs + 1) * 8) ||
        dtwo.alloc((n_pairs + 1) * 8) || dql.alloc(n_pairs * 4) || dtl.alloc(n_pairs * 4) ||
        dh0.alloc(n_pairs * 4) || dres.alloc(n_pairs * 12) || dws.alloc(wsb) || dst.alloc(64 * 8))
        return SALOBA_ECUDA;

    // device offsets relative to the start of each host buffer
    std::vector<int64_t> qo(n_pairs + 1), to(n_pairs + 1);
    for (int64_t k = 0; k <= n_pairs; ++k) {
        qo[k] = q_off[k] - q_off[0];
        to[k] = t_off[k] - t_off[0];
    }
    uint8_t* q_base = static_cast<uint8_t*>(dq.p);
    uint8_t* t_base = static_cast<uint8_t*>(dt.p);
    int64_t* st = static_cast<int64_t*>(dst.p);
    int32_t* res = static_cast<int32_t*>(dres.p);

    cudaStream_t cs = nullptr;
    cudaEvent_t ev_up[8], ev_done[8];
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return SALOBA_ECUDA;
    for (int i = 0; i < nslices; ++i) {
        cudaEventCreateWithFlags(&ev_up[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming);
    }
    // offsets (small) first, synchronously ordered on the copy stream
    cudaMemcpyAsync(dqo.p, qo.data(), (n_pairs + 1) * 8, cudaMemcpyHostToDevice, cs);
    cudaMemcpyAsync(dto.p, to.data(), (n_pairs + 1) * 8, cudaMemcpyHostToDevice, cs);
    if (h0) cudaMemcpyAsync(dh0.p, h0, n_pairs * 4, cudaMemcpyHostToDevice, cs);
    const int32_t* dh0p = h0 ? static_cast<int32_t*>(dh0.p) : nullptr;
    int rc = SALOBA_OK;
    for (int i = 0; i < nslices && rc == SALOBA_OK; ++i) {
        const int64_t a0 = cut[i], a1 = cut[i + 1], na = a1 - a0;
        cudaMemcpyAsync(q_base + qo[a0], q_ascii + q_off[a0], qo[a1] - qo[a0], cudaMemcpyHostToDevice, cs);
        cudaMemcpyAsync(t_base + to[a0], t_ascii + t_off[a0], to[a1] - to[a0], cudaMemcpyHostToDevice, cs);
        cudaEventRecord(ev_up[i], cs);
        cudaStreamWaitEvent(s, ev_up[i], 0);
        launch_pack_range(q_base, static_cast<int64_t*>(dqo.p) + a0, na, a0, SALOBA_PACK4,
                          static_cast<uint32_t*>(dqw.p), static_cast<int64_t*>(dqwo.p) + a0,
                          static_cast<int32_t*>(dql.p) + a0, st + 4 * i + 0, s);
        launch_pack_range(t_base, static_cast<int64_t*>(dto.p) + a0, na, a0, SALOBA_PACK4,
                          static_cast<uint32_t*>(dtw.p), static_cast<int64_t*>(dtwo.p) + a0,
                          static_cast<int32_t*>(dtl.p) + a0, st + 4 * i + 1, s);
        rc = saloba_align_batch(static_cast<uint32_t*>(dqw.p), static_cast<int64_t*>(dqwo.p) + a0,
                                static_cast<int32_t*>(dql.p) + a0, static_cast<uint32_t*>(dtw.p),
                                static_cast<int64_t*>(dtwo.p) + a0, static_cast<int32_t*>(dtl.p) + a0,
                                dh0p ? dh0p + a0 : nullptr, na, sc, mode, SALOBA_PACK4, res + a0,
                                res + n_pairs + a0, res + 2 * n_pairs + a0, dws.p, wsb, st + 4 * i + 2, opt, s);
        cudaEventRecord(ev_done[i], s);
        cudaStreamWaitEvent(cs, ev_done[i], 0);
        cudaMemcpyAsync(score + a0, res + a0, na * 4, cudaMemcpyDeviceToHost, cs);
        cudaMemcpyAsync(q_end + a0, res + n_pairs + a0, na * 4, cudaMemcpyDeviceToHost, cs);
        cudaMemcpyAsync(t_end + a0, res + 2 * n_pairs + a0, na * 4, cudaMemcpyDeviceToHost, cs);
    }
    int64_t hst[64];
    cudaMemcpyAsync(hst, st, sizeof(int64_t) * 4 * nslices, cudaMemcpyDeviceToHost, cs);
    cudaError_t e = cudaStreamSynchronize(cs);
    cudaStreamSynchronize(s);
    for (int i = 0; i < nslices; ++i) {
        cudaEventDestroy(ev_up[i]);
        cudaEventDestroy(ev_done[i]);
    }
    cudaStreamDestroy(cs);
    if (rc != SALOBA_OK) return rc;
    if (e != cudaSuccess) return SALOBA_ECUDA;
    // status: smallest bad pair over all slices (invalid byte -> its pair; align status is slice-local)
    int64_t bad = INT64_MAX;
    for (int i = 0; i < nslices; ++i) {
        if (hst[4 * i + 0] >= 0) bad = std::min(bad, first_pair_of_byte(qo.data(), n_pairs, hst[4 * i + 0]));
        if (hst[4 * i + 1] >= 0) bad = std::min(bad, first_pair_of_byte(to.data(), n_pairs, hst[4 * i + 1]));
        if (hst[4 * i + 2] >= 0) bad = std::min(bad, cut[i] + hst[4 * i + 2]);
    }
    *host_status = bad == INT64_MAX ? -1 : bad;
    return SALOBA_OK;
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
