// sat_cand.cu -- launch_cand<T, SRC> for one (time type, candidate source) pair; compiled once
// per pair (SAT_CAND_T / SAT_CAND_SRC) so the node-size specialisations build in parallel.
#include "sat_cand.cuh"

#ifndef SAT_CAND_T
#define SAT_CAND_T int32_t
#define SAT_CAND_SRC SAT_SRC_SUBSTREAM
#endif

namespace sat {

template <typename T, int SRC, int G, int L>
static int launch_cand_g(const sat_problem_t *p, CandArgs a, uint64_t n_cand, const std::vector<uint8_t> &blob,
                         void *d_ws, size_t ws_bytes, cudaStream_t stream) {
    if constexpr ((L == kLayoutOne16 || L == kLayoutMulti16) && sizeof(T) != 4) {
        return SAT_ERR_UNSUPPORTED;      // packed slots are grid-time only
    } else {
    const size_t blob_bytes = blob.size();
    const int N = (L == kLayoutMulti || L == kLayoutMulti16) ? p->N : 1;
    const int smem = (int)blob_bytes +
                     kCandWarps * cand_warp_bytes(p->J, N, G, cand_slot_bytes<T, L>(), SRC == SAT_SRC_INDEX);
    if (smem > 220 * 1024) return SAT_ERR_TOO_LARGE;
    auto kern = k_cand<T, SRC, G, L>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SAT_ERR_CUDA;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCandThreads, smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    uint64_t blocks = (uint64_t)device_sms() * (uint64_t)per_sm;
    const uint64_t chunks = (n_cand + 32ull * a.per_lane - 1) / (32ull * a.per_lane);   // warp chunks
    const uint64_t need = (chunks + kCandWarps - 1) / kCandWarps;
    if (blocks > need) blocks = std::max<uint64_t>(1, need);
    const size_t part_off = (blob_bytes + 255) & ~(size_t)255;
    const size_t cur_off = part_off + (size_t)blocks * sizeof(sat_best_t);
    const size_t need_ws = cur_off + sizeof(unsigned long long);
    if (!d_ws || ws_bytes < need_ws) return SAT_ERR_INVALID;
    uint8_t *ws = static_cast<uint8_t *>(d_ws);
    if (cudaMemcpyAsync(ws, blob.data(), blob_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return SAT_ERR_CUDA;
    if (cudaMemsetAsync(ws + cur_off, 0, sizeof(unsigned long long), stream) != cudaSuccess) return SAT_ERR_CUDA;
    a.blob = ws;
    a.partials = reinterpret_cast<sat_best_t *>(ws + part_off);
    a.cursor = reinterpret_cast<unsigned long long *>(ws + cur_off);
    kern<<<(unsigned)blocks, kCandThreads, smem, stream>>>(a);
    if (cudaGetLastError() != cudaSuccess) return SAT_ERR_CUDA;
    if (sizeof(T) == 8) {
        k_fold_partials<<<1, 32, 0, stream>>>(a.partials, (int)blocks, a.best);
        if (cudaGetLastError() != cudaSuccess) return SAT_ERR_CUDA;
    }
    return SAT_OK;
    }
}

template <typename T, int SRC>
int launch_cand(const sat_problem_t *p, CandArgs a, uint64_t n_cand, void *d_ws, size_t ws_bytes,
                cudaStream_t stream) {
    // durations ride in the step records when they do not depend on the node and every
    // option may run on every node (grid time, fits the 20-bit payload)
    a.rec_d = records_carry_duration(p) ? 1 : 0;
    std::vector<uint8_t> blob;
    int st = pack_blob(p, blob, a.rec_d != 0);
    if (st) return st;
    const bool multi = p->N > 1;
    // 16-bit packed slots when no free time can reach 2^16 - 1 (one node, grid time, records
    // carry the durations): bound = latest initial free time + latest release + sum of the
    // longest option of every job
    bool p16 = false;
    if (sizeof(T) == 4 && a.rec_d && p->G >= 2) {
        int64_t bound = 0, rel = 0, init = 0;
        for (int j = 0; j < p->J; ++j) {
            int32_t dm = 0;
            for (int o = 0; o < p->radix[j]; ++o) dm = std::max(dm, p->dur_i32[(j * p->Cmax + o) * p->N]);
            bound += dm;
            if (p->release_i32) rel = std::max<int64_t>(rel, p->release_i32[j]);
        }
        for (int n = 0; n < p->N; ++n)
            for (int i = 0; i < p->node_gpus[n]; ++i)
                if (p->init_free_i32) init = std::max<int64_t>(init, p->init_free_i32[n * p->G + i]);
        p16 = bound + rel + init < 0xffff;
    }
    switch (p->G) {
#define SAT_CASE(K)                                                                                      \
    case K:                                                                                              \
        if (multi && K >= 2 && p16)                                                                      \
            return launch_cand_g<T, SRC, (K <= 16 ? (K >= 2 ? K : 2) : 16), kLayoutMulti16>(p, a, n_cand, blob, d_ws, ws_bytes, stream); \
        if (multi)                                                                                       \
            return launch_cand_g<T, SRC, (K <= 16 ? K : 16), kLayoutMulti>(p, a, n_cand, blob, d_ws, ws_bytes, stream); \
        if (K >= 2 && p16)                                                                               \
            return launch_cand_g<T, SRC, (K >= 2 ? K : 2), kLayoutOne16>(p, a, n_cand, blob, d_ws, ws_bytes, stream); \
        return launch_cand_g<T, SRC, K, kLayoutOne>(p, a, n_cand, blob, d_ws, ws_bytes, stream);
        SAT_CASE(1) SAT_CASE(2) SAT_CASE(4) SAT_CASE(8) SAT_CASE(16) SAT_CASE(32)
#undef SAT_CASE
        default: return SAT_ERR_UNSUPPORTED;
    }
}

template int launch_cand<SAT_CAND_T, SAT_CAND_SRC>(const sat_problem_t *, CandArgs, uint64_t, void *, size_t,
                                                   cudaStream_t);

// ---------------------------------------------------------------- local search
template <int SRC, int G, int L, int K>
static int launch_ls_k(const sat_problem_t *p, LsArgs a, const std::vector<uint8_t> &blob, void *d_ws,
                       size_t ws_bytes, cudaStream_t stream) {
    const size_t blob_bytes = blob.size();
    const int N = (L == kLayoutMulti || L == kLayoutMulti16) ? p->N : 1;
    const int smem = (int)blob_bytes +
                     ls_block_bytes(p->J, N, G, cand_slot_bytes<int32_t, L>(), cache_state_words<G, L>(N), K);
    if (smem > 220 * 1024) return SAT_ERR_TOO_LARGE;
    auto kern = k_ls<SRC, G, L, K>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SAT_ERR_CUDA;
    int per_sm = 0;
    constexpr int BW = ls_block_warps(K);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BW * 32, smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    uint64_t blocks = (uint64_t)device_sms() * (uint64_t)per_sm;
    a.group_warps = K;
    const uint64_t need = ((a.hi - a.lo) * (uint64_t)K + BW - 1) / BW;
    if (blocks > need) blocks = std::max<uint64_t>(1, need);
    const size_t cur_off = (blob_bytes + 255) & ~(size_t)255;
    if (!d_ws || ws_bytes < cur_off + 2 * sizeof(unsigned long long)) return SAT_ERR_INVALID;
    uint8_t *ws = static_cast<uint8_t *>(d_ws);
    if (cudaMemcpyAsync(ws, blob.data(), blob_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return SAT_ERR_CUDA;
#ifdef SAT_LS_PROFILE
    constexpr int kCounters = 8;       // cursor, rounds, 5 profile counters
#else
    constexpr int kCounters = 2;       // cursor, rounds
#endif
    if (cudaMemsetAsync(ws + cur_off, 0, kCounters * sizeof(unsigned long long), stream) != cudaSuccess)
        return SAT_ERR_CUDA;
    a.blob = ws;
    a.cursor = reinterpret_cast<unsigned long long *>(ws + cur_off);
    a.rounds = a.cursor + 1;
    kern<<<(unsigned)blocks, BW * 32, smem, stream>>>(a);
    return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
}

// warps per walker: long orders scan long (J = 32: ~72 rounds of 32 moves per scan), so a
// 256-thread block evaluating 8 rounds at once shortens the walk's critical path (sequential
// steps / 6.9 on cfg5, instrumented oracle; measured cfg4 / cfg5 time to the bound: K = 1
// 17.5 / 35 ms, K = 4 7.5 / 14.5 ms, K = 8 5.7 / 13.2 ms); short orders keep a walker per
// warp (more walkers in flight, no block barriers).  SATURN_LS_GROUP = 1 / 4 / 8 overrides.
template <int SRC, int G, int L>
static int launch_ls_g(const sat_problem_t *p, LsArgs a, const std::vector<uint8_t> &blob, void *d_ws,
                       size_t ws_bytes, cudaStream_t stream) {
    int K = p->J >= 24 ? 16 : 1;
    if (const char *env = std::getenv("SATURN_LS_GROUP")) {
        const int k = std::atoi(env);
        if (k == 1 || k == kCandWarps || k == 8 || k == 16 || k == 32) K = k;
    }
    if (K == 1) return launch_ls_k<SRC, G, L, 1>(p, a, blob, d_ws, ws_bytes, stream);
    if (K == 8) return launch_ls_k<SRC, G, L, 8>(p, a, blob, d_ws, ws_bytes, stream);
    if (K == 16) return launch_ls_k<SRC, G, L, 16>(p, a, blob, d_ws, ws_bytes, stream);
    if (K == 32) return launch_ls_k<SRC, G, L, 32>(p, a, blob, d_ws, ws_bytes, stream);
    return launch_ls_k<SRC, G, L, kCandWarps>(p, a, blob, d_ws, ws_bytes, stream);
}

template <int SRC>
int launch_ls(const sat_problem_t *p, LsArgs a, void *d_ws, size_t ws_bytes, cudaStream_t stream) {
    if (p->time_mode != SAT_TIME_GRID_I32) return SAT_ERR_UNSUPPORTED;
    a.rec_d = records_carry_duration(p) ? 1 : 0;
    std::vector<uint8_t> blob;
    int st = pack_blob(p, blob, a.rec_d != 0);
    if (st) return st;
    const bool multi = p->N > 1;
    bool p16 = false;
    if (a.rec_d && p->G >= 2) {
        int64_t bound = 0, rel = 0, init = 0;
        for (int j = 0; j < p->J; ++j) {
            int32_t dm = 0;
            for (int o = 0; o < p->radix[j]; ++o) dm = std::max(dm, p->dur_i32[(j * p->Cmax + o) * p->N]);
            bound += dm;
            if (p->release_i32) rel = std::max<int64_t>(rel, p->release_i32[j]);
        }
        for (int n = 0; n < p->N; ++n)
            for (int i = 0; i < p->node_gpus[n]; ++i)
                if (p->init_free_i32) init = std::max<int64_t>(init, p->init_free_i32[n * p->G + i]);
        p16 = bound + rel + init < 0xffff;
    }
    switch (p->G) {
#define SAT_LCASE(K)                                                                                   \
    case K:                                                                                            \
        if (multi && K >= 2 && p16)                                                                    \
            return launch_ls_g<SRC, (K <= 16 ? (K >= 2 ? K : 2) : 16), kLayoutMulti16>(p, a, blob, d_ws, ws_bytes, stream); \
        if (multi)                                                                                     \
            return launch_ls_g<SRC, (K <= 16 ? K : 16), kLayoutMulti>(p, a, blob, d_ws, ws_bytes, stream); \
        if (K >= 2 && p16)                                                                             \
            return launch_ls_g<SRC, (K >= 2 ? K : 2), kLayoutOne16>(p, a, blob, d_ws, ws_bytes, stream); \
        return launch_ls_g<SRC, K, kLayoutOne>(p, a, blob, d_ws, ws_bytes, stream);
        SAT_LCASE(1) SAT_LCASE(2) SAT_LCASE(4) SAT_LCASE(8) SAT_LCASE(16) SAT_LCASE(32)
#undef SAT_LCASE
        default: return SAT_ERR_UNSUPPORTED;
    }
}



}  // namespace sat

// the local search runs in grid time only: instantiate it in the int32 translation units
#if defined(SAT_LS_INSTANTIATE)
namespace sat {
template int launch_ls<SAT_CAND_SRC>(const sat_problem_t *, LsArgs, void *, size_t, cudaStream_t);
}
#endif
