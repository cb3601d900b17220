// partition.cu — A5: length-balanced assignment of pairs to the GPUs of one box (
// PAPER.md §VII-C: the paper splits the queries equally and names "dynamic assignment
// or preprocessing with approximate sorting" as the fix for the imbalance this causes).
//
// cost(k) = q_len·t_len + kappa (cells plus a per-pair overhead, §8(a) A2), sorted descending by
// one CUB radix sort (stable: equal costs keep input order, so every rank computing the partition
// from the same lengths gets the same answer), then dealt in snake order over the ranks
// (0, 1, .., W-1, W-1, .., 0, ...): rank totals differ by at most one pair of each cost class.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace saloba {

constexpr uint64_t PARTITION_KAPPA = 2048;  // per-pair overhead in cell units

__global__ void partition_cost_kernel(const int32_t* __restrict__ q_len, const int32_t* __restrict__ t_len,
                                      int64_t n, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t q = uint64_t(max(q_len[k], 0)), t = uint64_t(max(t_len[k], 0));
        keys[k] = ~(q * t + PARTITION_KAPPA);  // ascending sort of ~cost = descending cost
        vals[k] = uint32_t(k);
    }
}

__global__ void partition_snake_kernel(const uint32_t* __restrict__ order, int64_t n, int world,
                                       int32_t* __restrict__ owner) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t round = k / world;
        const int pos = int(k % world);
        owner[order[k]] = (round & 1) ? world - 1 - pos : pos;
    }
}

static size_t sort_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, int(n > 0 ? n : 1), 0, 64);
    return bytes;
}
static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace saloba

using namespace saloba;

SALOBA_API size_t saloba_partition_workspace_bytes(int64_t n_pairs) {
    if (n_pairs < 0 || n_pairs > int64_t(INT32_MAX) - 1024) return 0;
    const size_t nn = size_t(n_pairs > 0 ? n_pairs : 1);
    return 2 * al256(nn * 8) + 2 * al256(nn * 4) + al256(sort_bytes(n_pairs));
}

SALOBA_API int saloba_partition(const int32_t* q_len, const int32_t* t_len, int64_t n_pairs, int32_t world,
                                int32_t* owner, void* workspace, size_t workspace_bytes, void* stream) {
    if (n_pairs < 0 || n_pairs > int64_t(INT32_MAX) - 1024 || world < 1 || !workspace) return SALOBA_EINVAL;
    if (n_pairs > 0 && (!q_len || !t_len || !owner)) return SALOBA_EINVAL;
    if (reinterpret_cast<uintptr_t>(workspace) % 256) return SALOBA_EINVAL;
    if (workspace_bytes < saloba_partition_workspace_bytes(n_pairs)) return SALOBA_EWORKSPACE;
    if (n_pairs == 0) return SALOBA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t nn = size_t(n_pairs);
    char* ws = static_cast<char*>(workspace);
    uint64_t* kin = reinterpret_cast<uint64_t*>(ws);
    uint64_t* kout = reinterpret_cast<uint64_t*>(ws + al256(nn * 8));
    uint32_t* vin = reinterpret_cast<uint32_t*>(ws + 2 * al256(nn * 8));
    uint32_t* vout = reinterpret_cast<uint32_t*>(ws + 2 * al256(nn * 8) + al256(nn * 4));
    void* tmp = ws + 2 * al256(nn * 8) + 2 * al256(nn * 4);
    size_t tb = sort_bytes(n_pairs);
    const int64_t need = (n_pairs + 255) / 256;
    const int64_t cap = int64_t(sm_count_current()) * 8;
    const int grid = int(need < cap ? need : cap);
    partition_cost_kernel<<<grid, 256, 0, s>>>(q_len, t_len, n_pairs, kin, vin);
    if (cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, int(n_pairs), 0, 64, s) != cudaSuccess)
        return SALOBA_ECUDA;
    partition_snake_kernel<<<grid, 256, 0, s>>>(vout, n_pairs, world, owner);
    count_launches(2);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}

// ---- A5 reassembly: gathered per-rank results back to input order ("Rank 0
// unpermutes with the partition it computed") ------------------------------------------------------
namespace saloba {
__global__ void scatter_results_kernel(const int32_t* __restrict__ parts, const int32_t* __restrict__ index,
                                       int64_t stride, int64_t world_stride, int64_t n_total,
                                       int32_t* __restrict__ score, int32_t* __restrict__ q_end,
                                       int32_t* __restrict__ t_end, unsigned long long* __restrict__ status) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < world_stride;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int32_t dst = index[k];
        if (dst < 0) continue;  // padding slot of a shorter shard
        if (int64_t(dst) >= n_total) {
            atomicMin(status, (unsigned long long)k);
            continue;
        }
        const int64_t r = k / stride, i = k - r * stride;
        const int32_t* p = parts + r * 3 * stride;  // rank r's (3, stride) block: score, q_end, t_end rows
        score[dst] = p[i];
        q_end[dst] = p[stride + i];
        t_end[dst] = p[2 * stride + i];
    }
}
}  // namespace saloba

SALOBA_API int saloba_scatter_results(const int32_t* parts, const int32_t* index, int64_t stride, int32_t world,
                                      int64_t n_total, int32_t* score, int32_t* q_end, int32_t* t_end,
                                      int64_t* status, void* stream) {
    if (stride < 0 || world < 1 || n_total < 0 || n_total > int64_t(INT32_MAX) || !status) return SALOBA_EINVAL;
    if (stride > 0 && (!parts || !index)) return SALOBA_EINVAL;
    if (n_total > 0 && (!score || !q_end || !t_end)) return SALOBA_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    launch_status_init(status, s);
    const int64_t total = stride * int64_t(world);
    if (total > 0) {
        const int64_t need = (total + 255) / 256;
        const int cap = sm_count_current() * 8;
        scatter_results_kernel<<<int(need < cap ? need : cap), 256, 0, s>>>(
            parts, index, stride, total, n_total, score, q_end, t_end, (unsigned long long*)status);
        count_launches(1);
    }
    launch_status_final(status, s);
    return cudaGetLastError() == cudaSuccess ? SALOBA_OK : SALOBA_ECUDA;
}
