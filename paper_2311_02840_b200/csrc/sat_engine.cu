// sat_engine.cu -- B200 (sm_100a) plan-search engine behind include/saturn_engine.h.
//
// What one candidate is: an option digit
// per job plus a submission order.  Its makespan comes from per-GPU free-time list
// scheduling: in order, each job can start on a node at that node's g-th smallest
// GPU free time (max'd with the job's release); it goes to the node where it
// FINISHES earliest (lowest node on ties; with node-independent durations this is
// the earliest-starting node); its g earliest-free GPUs then become free at
// start + duration; the makespan is the largest free time at the end.
//
// Representation used on the device: per node, the free times are kept SORTED.
// Placing a (g, d) job that starts at s (= max(release, a[g-1])) with end e = s+d
// turns the sorted vector a into
//        b[i] = max(a[i], min(a[i+g], e))         (a[i+g] = +inf past the end)
// which is the sorted merge of a[g..] with g copies of e (proof in DESIGN.md).
// Every slot update is one min and one max, with no data-dependent branches.
//
// Kernel families:
//   k_tree<G, BNB>  (sat_tree.cuh) prefix-shared exhaustive walk for one node in grid time:
//       each lane owns a distinct prefix (first P jobs of the order + their options)
//       and the warp walks the remaining J-P jobs' orders x options in lock step, so
//       the job sequence and gang sizes are warp-uniform and only free times differ
//       per lane.  Every candidate still gets its full makespan computed.  BNB = the
//       bound-and-prune variant (same result key, subtrees above the best skipped).
//   k_cand<T, SRC, G, L>  (sat_cand.cuh) one candidate per thread: decoded on the
//       device from an index (mixed radix + Lehmer, odometer-advanced) or a SplitMix64
//       stream, list-scheduled with its sorted free times in registers / its own
//       shared-memory column.  Multi-node, releases, int32 grid or fp64 time.  The
//       search kernel for everything k_tree does not cover (sampled configs).
//   k_ls<SRC, G, L>  (sat_cand.cuh) local search: a walker per warp, a move per lane,
//       each move scheduled by the same list scheduler as k_cand.
//   k_generic<T, SRC, RECORD=true>  one candidate per W-lane warp segment (lane = GPU
//       slot); records each placement (option, node, start) of a few given candidates
//       -- sat_schedule, i.e. decode_plan of the winner and fixed-plan evaluation.
//
// Best-plan selection: key = (makespan, index) lexicographic, lowest index wins on
// equal makespans.  Grid mode packs it into one u64 and uses
// atomicMin; float mode reduces per block and merges in a second tiny kernel.
#include "sat_cand.cuh"

#include <list>
#include <memory>
#include <mutex>
#include <nvtx3/nvToolsExt.h>

namespace sat {
template <typename T, int SRC, bool RECORD>
__global__ void __launch_bounds__(kGenThreads)
k_generic(GenArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const BlobHeader &h = *reinterpret_cast<const BlobHeader *>(smem);
    {
        const int nwords = (*reinterpret_cast<const BlobHeader *>(a.blob)).bytes / 16;
        const int4 *src = reinterpret_cast<const int4 *>(a.blob);
        int4 *dst = reinterpret_cast<int4 *>(smem);
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int J = h.J, N = h.N, G = h.G, W = h.W;
    GenTables tb;
    load_tables(tb, smem, h);
    const T *dur = reinterpret_cast<const T *>(smem + h.off_dur);
    const T *release = reinterpret_cast<const T *>(smem + h.off_release);
    const T *lane_init = reinterpret_cast<const T *>(smem + h.off_lane_init);
    const bool rec_d = a.rec_d != 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warp_bytes = J * 32 * (4 + (SRC == SAT_SRC_INDEX ? 2 : 0));
    uint8_t *wscr = smem + h.bytes + warp * warp_bytes;
    uint32_t *steps = reinterpret_cast<uint32_t *>(wscr);            // [J][32]
    uint32_t *my_steps = steps + lane;
    uint8_t *my_opt = wscr + J * 128 + lane;                         // [J][32] (index source)
    uint8_t *my_ord = my_opt + J * 32;

    const int sl = lane & (W - 1), seg = lane / W, node = sl / G, slot = sl - node * G;
    const int seg_base = seg * W;
    const int segs = 32 / W;
    const T INF = TimeTraits<T>::inf();
    const T init_max = sizeof(T) == 4 ? (T)h.init_max_i32 : (T)h.init_max_f64;
    const T my_init = lane_init[sl];
    const bool multi = N > 1;

    T best_ms = INF;
    uint64_t best_ix = ~0ull;

    const uint64_t total = a.hi - a.lo;
    const int per_lane = (SRC == SAT_SRC_INDEX && !RECORD) ? a.per_lane : 1;
    const uint64_t per_batch = 32ull * (uint64_t)per_lane;
    const uint64_t nbatches = (total + per_batch - 1) / per_batch;
    const uint64_t gwarp = (uint64_t)blockIdx.x * kGenWarps + warp;
    const uint64_t nwarps = (uint64_t)gridDim.x * kGenWarps;

    for (uint64_t b = gwarp; b < nbatches; b += nwarps) {
        const uint64_t first = b * per_batch + (uint64_t)lane * per_lane;   // offset from lo
        for (int k = 0; k < per_lane; ++k) {
            const uint64_t off = first + k;
            const bool valid = off < total;
            uint64_t id = a.lo + off;
            if (RECORD && a.ids) id = a.ids[valid ? off : 0];
            // ---- decode (thread per candidate) ----
            if (valid) {
                if (SRC == SAT_SRC_INDEX) {
                    if (k == 0 || RECORD) decode_index(id, J, tb.radix, my_opt, my_ord);
                    else advance_index(J, tb.radix, my_opt, my_ord);
                    for (int kk = 0; kk < J; ++kk) {
                        const int job = my_ord[kk * 32];
                        my_steps[kk * 32] = rec_for(tb, job, my_opt[job * 32]);
                    }
                } else if (SRC == SAT_SRC_SUBSTREAM) {
                    decode_stream(mix64((a.seed ^ id) + kGolden), tb, my_steps);
                } else if (SRC == SAT_SRC_SEED) {
                    decode_stream(a.seed + id, tb, my_steps);
                } else {
                    // memory safety only: the host validates explicit candidates before upload
                    const uint8_t *e = a.expl + (size_t)(RECORD ? off : id) * (2 * J);
                    for (int kk = 0; kk < J; ++kk) {
                        const int job = e[J + kk] % J;
                        my_steps[kk * 32] = rec_for(tb, job, min((int)e[job], tb.radix[job] - 1));
                    }
                }
            } else {
                // no candidate for this lane: park a harmless one (its key is discarded)
                for (int kk = 0; kk < J; ++kk) my_steps[kk * 32] = rec_for(tb, kk, 0);
            }
            __syncwarp();
            // ---- schedule: segment `seg` handles candidate slot pass * segs + seg ----
            for (int pass = 0; pass < W; ++pass) {
                const int c = pass * segs + seg;
                const uint64_t c_off = __shfl_sync(0xffffffffu, off, c);
                const bool c_valid = __shfl_sync(0xffffffffu, (int)valid, c) != 0;
                // every segment on a parked slot (no candidate): nothing to schedule in this pass
                if (!__any_sync(0xffffffffu, c_valid)) continue;
                const uint64_t c_id = shfl_u64(id, c);
                const uint32_t *c_steps = steps + c;
                T av = my_init;
                T mx = init_max;
                for (int kk = 0; kk < J; ++kk) {
                    const uint32_t r = c_steps[kk * 32];
                    const int g = (int)(r & 63u) + 1;
                    const uint32_t pay = r >> 12;
                    T t = __shfl_sync(0xffffffffu, av, seg_base + node * G + g - 1);
                    T d;
                    if (rec_d) {
                        d = (T)(int32_t)pay;
                    } else {
                        if (multi && !((tb.optmask[pay] >> node) & 1u)) t = INF;
                        d = node < N ? dur[pay * N + node] : (T)0;
                    }
                    if (h.has_release) t = tmax(t, release[(r >> 6) & 63u]);
                    // node finishing the job earliest, lowest node on ties
                    T bt = t, be = t + d;
                    int bn = node;
                    for (int x = G; x < W; x <<= 1) {
                        const T oe = __shfl_xor_sync(0xffffffffu, be, x);
                        const T ot = __shfl_xor_sync(0xffffffffu, bt, x);
                        const int on = __shfl_xor_sync(0xffffffffu, bn, x);
                        if (oe < be || (oe == be && on < bn)) { be = oe; bt = ot; bn = on; }
                    }
                    int src = lane + g;
                    src = src > 31 ? 31 : src;
                    T up = __shfl_sync(0xffffffffu, av, src);
                    if (slot + g >= G) up = INF;
                    if (node == bn) av = tmax(av, tmin(up, be));
                    mx = tmax(mx, be);
                    if (RECORD && sl == 0 && c_valid) {
                        const int job = (int)((r >> 6) & 63u);
                        const size_t o = (size_t)c_off * J + job;
                        if (a.rec_opt) a.rec_opt[o] = (int32_t)pay - tb.optbase[job];
                        if (a.rec_node) a.rec_node[o] = bn;
                        if (sizeof(T) == 4) { if (a.rec_start_i32) a.rec_start_i32[o] = (int32_t)bt; }
                        else { if (a.rec_start_f64) a.rec_start_f64[o] = (double)bt; }
                    }
                }
                if (sl == 0 && c_valid) {
                    if (RECORD) {
                        if (sizeof(T) == 4) { if (a.rec_ms_i64) a.rec_ms_i64[c_off] = (int64_t)mx; }
                        else { if (a.rec_ms_f64) a.rec_ms_f64[c_off] = (double)mx; }
                    } else if (key_less(mx, c_id, best_ms, best_ix)) {
                        best_ms = mx;
                        best_ix = c_id;
                    }
                }
            }
            __syncwarp();
        }
    }
    if constexpr (!RECORD) {
        // ---- warp -> block -> grid argmin ----
        for (int x = 16; x >= 1; x >>= 1) {
            T oms = __shfl_xor_sync(0xffffffffu, best_ms, x);
            uint64_t oix = shfl_u64(best_ix, lane ^ x);
            if (key_less(oms, oix, best_ms, best_ix)) { best_ms = oms; best_ix = oix; }
        }
        __shared__ T s_ms[kGenWarps];
        __shared__ uint64_t s_ix[kGenWarps];
        if (lane == 0) { s_ms[warp] = best_ms; s_ix[warp] = best_ix; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < kGenWarps; ++w)
                if (key_less(s_ms[w], s_ix[w], best_ms, best_ix)) { best_ms = s_ms[w]; best_ix = s_ix[w]; }
            if (sizeof(T) == 4) {
                if (best_ms < INF) {
                    const uint64_t key = ((uint64_t)(uint32_t)best_ms << h.idx_bits) | best_ix;
                    atomicMin(reinterpret_cast<unsigned long long *>(&a.best->hi), (unsigned long long)key);
                }
            } else {
                a.partials[blockIdx.x].hi = (uint64_t)__double_as_longlong((double)best_ms);
                a.partials[blockIdx.x].lo = best_ix;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// ALU probe: independent IMNMX chains (8 per thread) for the INT32 roofline
// ---------------------------------------------------------------------------
__global__ void k_alu_probe(int iters, unsigned long long *ops, int32_t *sink) {
    // 16 independent min/max chains; asm volatile keeps every IMNMX
    int32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (int32_t)threadIdx.x + i;
    const int32_t lo = (int32_t)(blockIdx.x & 7), hi = (int32_t)(blockIdx.x | 1024);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            asm volatile("min.s32 %0, %0, %1;" : "+r"(v[i]) : "r"(hi));
            asm volatile("max.s32 %0, %0, %1;" : "+r"(v[i]) : "r"(lo));
        }
    }
    int32_t r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) r ^= v[i];
    if (r == 0x7fffffff) sink[0] = r;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        *ops = (unsigned long long)gridDim.x * blockDim.x * (unsigned long long)iters * 32ull;
}

// the same chains on two 16-bit lanes per register (min/max .u16x2 -> VIMNMX.U16x2): the
// peak of k_tree's packed pair pass, counted as 2 ops per lane per instruction
__global__ void k_alu_probe16(int iters, unsigned long long *ops, int32_t *sink) {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (uint32_t)threadIdx.x * 0x10001u + (uint32_t)i;
    const uint32_t lo = (blockIdx.x & 7u) * 0x10001u, hi = (blockIdx.x | 1024u) * 0x10001u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            asm volatile("min.u16x2 %0, %0, %1;" : "+r"(v[i]) : "r"(hi));
            asm volatile("max.u16x2 %0, %0, %1;" : "+r"(v[i]) : "r"(lo));
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) r ^= v[i];
    if (r == 0x7fffffffu) sink[0] = (int32_t)r;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        *ops = (unsigned long long)gridDim.x * blockDim.x * (unsigned long long)iters * 64ull;
}

// ---------------------------------------------------------------------------
// host side: validation, packing, launch sizing
// ---------------------------------------------------------------------------
inline int check_cuda(cudaError_t e) { return e == cudaSuccess ? SAT_OK : SAT_ERR_CUDA; }

int validate(const sat_problem_t *p) {
    if (!p) return SAT_ERR_INVALID;
    if (p->J < 1 || p->J > SAT_MAX_JOBS || p->N < 1 || p->G < 1 || p->Cmax < 1) return SAT_ERR_INVALID;
    if ((p->G & (p->G - 1)) != 0) return SAT_ERR_INVALID;
    if ((int64_t)p->N * p->G > SAT_MAX_LANES) return SAT_ERR_UNSUPPORTED;
    if (p->time_mode != SAT_TIME_GRID_I32 && p->time_mode != SAT_TIME_F64) return SAT_ERR_INVALID;
    if (!p->radix || !p->gpus || !p->node_gpus) return SAT_ERR_INVALID;
    if (p->time_mode == SAT_TIME_GRID_I32 && !p->dur_i32) return SAT_ERR_INVALID;
    if (p->time_mode == SAT_TIME_F64 && !p->dur_f64) return SAT_ERR_INVALID;
    for (int n = 0; n < p->N; ++n)
        if (p->node_gpus[n] < 1 || p->node_gpus[n] > p->G) return SAT_ERR_INVALID;
    for (int j = 0; j < p->J; ++j) {
        if (p->radix[j] < 1) return SAT_ERR_NO_OPTIONS;
        if (p->radix[j] > p->Cmax || p->radix[j] > 255) return SAT_ERR_INVALID;
        for (int o = 0; o < p->radix[j]; ++o) {
            const int g = p->gpus[j * p->Cmax + o];
            if (g < 1 || g > p->G) return SAT_ERR_INVALID;
            const uint32_t m = p->node_mask ? p->node_mask[j * p->Cmax + o] : ~0u;
            bool any = false;
            for (int n = 0; n < p->N; ++n)
                if (((m >> n) & 1u) && p->node_gpus[n] >= g) any = true;
            if (!any) return SAT_ERR_INVALID;
        }
    }
    if (p->time_mode == SAT_TIME_GRID_I32 && (p->idx_bits < 1 || p->idx_bits > 62)) return SAT_ERR_INVALID;
    return SAT_OK;
}

inline int align16(int x) { return (x + 15) & ~15; }

int device_sms() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return sms > 0 ? sms : 148;
}

bool records_carry_duration(const sat_problem_t *p) {
    if (p->time_mode != SAT_TIME_GRID_I32) return false;
    const uint32_t all = p->N >= 32 ? ~0u : ((1u << p->N) - 1u);
    for (int j = 0; j < p->J; ++j)
        for (int o = 0; o < p->radix[j]; ++o) {
            const int q = j * p->Cmax + o;
            const int32_t d0 = p->dur_i32[q * p->N];
            if (d0 < 0 || d0 >= (1 << 20)) return false;
            if (p->node_mask && (p->node_mask[q] & all) != all) return false;
            for (int n = 1; n < p->N; ++n)
                if (p->dur_i32[q * p->N + n] != d0) return false;
        }
    return true;
}

// Build the generic blob.  Lane init: for W lanes, node = lane / G, slot = lane % G.
int pack_blob(const sat_problem_t *p, std::vector<uint8_t> &blob, bool rec_d) {
    const int J = p->J, N = p->N, G = p->G;
    int W = 8;
    while (W < N * G) W <<= 1;
    const bool f64 = p->time_mode == SAT_TIME_F64;
    const int tsz = f64 ? 8 : 4;
    int n_opt = 0, max_n = J;
    for (int j = 0; j < J; ++j) { n_opt += p->radix[j]; max_n = std::max(max_n, (int)p->radix[j]); }
    BlobHeader h{};
    h.J = J; h.N = N; h.G = G; h.W = W;
    h.time_mode = p->time_mode; h.idx_bits = p->idx_bits; h.n_opt = n_opt;
    h.max_n = max_n;
    int off = sizeof(BlobHeader);
    h.off_radix = off; off = align16(off + 4 * J);
    h.off_optbase = off; off = align16(off + 4 * J);
    // tables only the paths that read them get: node masks with several nodes, the
    // duration table unless every record carries its duration
    const bool need_mask = N > 1, need_dur = !rec_d;
    h.off_g = off;                                     // (gang sizes ride in the records)
    h.off_mask = off; off = align16(off + (need_mask ? 4 * n_opt : 0));
    h.off_dur = off; off = align16(off + (need_dur ? tsz * n_opt * N : 0));
    h.off_release = off; off = align16(off + tsz * J);
    h.off_lane_init = off; off = align16(off + tsz * W);
    h.off_modn = off; off = align16(off + (int)sizeof(ModN) * (max_n + 1));
    h.off_prerec = off; off = align16(off + 4 * n_opt);
    h.off_jobinfo = off; off = align16(off + (int)sizeof(JobInfo) * J);
    h.bytes = off;
    blob.assign(off, 0);
    int32_t *radix = reinterpret_cast<int32_t *>(&blob[h.off_radix]);
    int32_t *optbase = reinterpret_cast<int32_t *>(&blob[h.off_optbase]);
    uint32_t *om = reinterpret_cast<uint32_t *>(&blob[h.off_mask]);
    int q = 0;
    bool has_release = false;
    for (int j = 0; j < J; ++j) {
        radix[j] = p->radix[j];
        optbase[j] = q;
        for (int o = 0; o < p->radix[j]; ++o, ++q) {
            const int src = j * p->Cmax + o;
            uint32_t m = p->node_mask ? p->node_mask[src] : ((N >= 32) ? ~0u : ((1u << N) - 1u));
            if (N < 32) m &= (1u << N) - 1u;
            if (need_mask) om[q] = m;
            for (int n = 0; n < N && need_dur; ++n) {
                if (f64) reinterpret_cast<double *>(&blob[h.off_dur])[q * N + n] = p->dur_f64[src * N + n];
                else reinterpret_cast<int32_t *>(&blob[h.off_dur])[q * N + n] = p->dur_i32[src * N + n];
            }
        }
        if (f64) {
            const double r = p->release_f64 ? p->release_f64[j] : 0.0;
            reinterpret_cast<double *>(&blob[h.off_release])[j] = r;
            has_release |= r != 0.0;
        } else {
            const int32_t r = p->release_i32 ? p->release_i32[j] : 0;
            reinterpret_cast<int32_t *>(&blob[h.off_release])[j] = r;
            has_release |= r != 0;
        }
    }
    h.has_release = has_release ? 1 : 0;
    int64_t imax_i = 0;
    double imax_f = 0.0;
    for (int l = 0; l < W; ++l) {
        const int n = l / G, s = l % G;
        const bool real = n < N && s < p->node_gpus[n];
        if (f64) {
            double v = real ? (p->init_free_f64 ? p->init_free_f64[n * G + s] : 0.0)
                            : __builtin_inf();
            reinterpret_cast<double *>(&blob[h.off_lane_init])[l] = v;
            if (real) imax_f = std::max(imax_f, v);
        } else {
            int32_t v = real ? (p->init_free_i32 ? p->init_free_i32[n * G + s] : 0) : SAT_INF_I32;
            reinterpret_cast<int32_t *>(&blob[h.off_lane_init])[l] = v;
            if (real) imax_i = std::max<int64_t>(imax_i, v);
        }
    }
    h.init_max_i32 = imax_i;
    h.init_max_f64 = imax_f;
    ModN *mods = reinterpret_cast<ModN *>(&blob[h.off_modn]);
    for (int n = 1; n <= max_n; ++n) {
        const unsigned __int128 two64 = (unsigned __int128)1 << 64;
        mods[n].reject_rem = (uint64_t)(two64 % (unsigned)n);
        mods[n].magic = ~0ull / (uint64_t)n;
    }
    uint32_t *prerec = reinterpret_cast<uint32_t *>(&blob[h.off_prerec]);
    JobInfo *ji = reinterpret_cast<JobInfo *>(&blob[h.off_jobinfo]);
    for (int j = 0, qq = 0; j < J; ++j) {
        ji[j].radix = p->radix[j];
        ji[j].optbase = qq;
        ji[j].magic = ~0ull / (uint64_t)p->radix[j];
        for (int o = 0; o < p->radix[j]; ++o, ++qq) {
            const int src = j * p->Cmax + o;
            const uint32_t pay = rec_d ? (uint32_t)p->dur_i32[src * N] : (uint32_t)qq;
            prerec[qq] = (uint32_t)(p->gpus[src] - 1) | ((uint32_t)j << 6) | (pay << 12);
        }
    }
    std::memcpy(blob.data(), &h, sizeof(h));
    return SAT_OK;
}


int gen_blocks(const void *kernel, int smem_bytes) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kGenThreads, smem_bytes) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    return device_sms() * per_sm;
}

template <typename T, int SRC, bool RECORD>
int launch_generic(const sat_problem_t *p, GenArgs a, uint64_t n_cand, void *d_ws, size_t ws_bytes,
                   cudaStream_t stream) {
    std::vector<uint8_t> blob;
    a.rec_d = 0;                 // recorded plans need the option id in every record
    int st = pack_blob(p, blob, false);
    if (st) return st;
    const size_t blob_bytes = blob.size();
    const int smem = (int)blob_bytes + kGenWarps * p->J * 32 * (4 + (SRC == SAT_SRC_INDEX ? 2 : 0));
    if (smem > 200 * 1024) return SAT_ERR_TOO_LARGE;
    auto kern = k_generic<T, SRC, RECORD>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SAT_ERR_CUDA;
    int blocks = gen_blocks((const void *)kern, smem);
    const uint64_t per_batch = 32ull * (uint64_t)std::max(1, a.per_lane);
    const uint64_t batches = (n_cand + per_batch - 1) / per_batch;
    const uint64_t need = (batches + kGenWarps - 1) / kGenWarps;
    if ((uint64_t)blocks > need) blocks = (int)std::max<uint64_t>(1, need);
    const size_t part_off = (blob_bytes + 255) & ~(size_t)255;
    const size_t need_ws = part_off + (size_t)blocks * sizeof(sat_best_t);
    if (!d_ws || ws_bytes < need_ws) return SAT_ERR_INVALID;
    uint8_t *ws = static_cast<uint8_t *>(d_ws);
    if (cudaMemcpyAsync(ws, blob.data(), blob_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return SAT_ERR_CUDA;
    a.blob = ws;
    a.partials = reinterpret_cast<sat_best_t *>(ws + part_off);
    kern<<<blocks, kGenThreads, smem, stream>>>(a);
    if (cudaGetLastError() != cudaSuccess) return SAT_ERR_CUDA;
    if (!RECORD && sizeof(T) == 8) {
        k_fold_partials<<<1, 32, 0, stream>>>(a.partials, blocks, a.best);
        if (cudaGetLastError() != cudaSuccess) return SAT_ERR_CUDA;
    }
    return SAT_OK;
}

uint64_t factorial_u64(int n) {
    uint64_t f = 1;
    for (int k = 2; k <= n; ++k) f *= (uint64_t)k;
    return f;
}

// n! * prod(radix) without overflow?  Returns false if > 2^63.
bool space_size(const sat_problem_t *p, uint64_t *out) {
    unsigned __int128 s = 1;
    for (int k = 2; k <= p->J; ++k) { s *= (unsigned)k; if (s > ((unsigned __int128)1 << 63)) return false; }
    for (int j = 0; j < p->J; ++j) { s *= (unsigned)p->radix[j]; if (s > ((unsigned __int128)1 << 63)) return false; }
    *out = (uint64_t)s;
    return true;
}

// ---- tree layout ----
struct TreeLayout {
    int P = 0;
    std::vector<uint32_t> sets;
    std::vector<uint64_t> cum, prod;
    uint64_t n_tasks = 0, n_cand = 0, n_steps = 0;
};

// number of placements in the full walk below a remaining-set (memoised by mask)
uint64_t walk_nodes(const int32_t *radix, uint32_t rem, std::vector<int64_t> &memo, uint32_t full) {
    if (!rem) return 0;
    // memo indexed by rem (sub-mask of `full`): compress via the mask itself when small
    if (memo[rem] >= 0) return (uint64_t)memo[rem];
    uint64_t tot = 0;
    for (uint32_t m = rem; m; m &= m - 1) {
        const int j = __builtin_ctz(m);
        tot += (uint64_t)radix[j] * (1 + walk_nodes(radix, rem & ~(1u << j), memo, full));
    }
    memo[rem] = (int64_t)tot;
    return tot;
}

// Relative device cost of one warp walking the suffix set `rem` (shard balancing): a pair node
// costs a fixed part plus one group per gang of each of its two jobs (the pair pass folds the
// last job's options into per-gang minima, so its cost is r_a + r_b groups, not r_a * r_b
// leaves); every upper-level node one merge.  Constants: warp instructions per unit in the
// ncu source view of k_tree<8> (r01e: pair fixed ~110, group ~14, merge ~25, task ~250).
constexpr double kCostPair = 110.0, kCostGroup = 14.0, kCostMerge = 25.0, kCostTask = 250.0;

double walk_cost(const int32_t *radix, uint32_t rem, std::vector<double> &memo) {
    const int n = __builtin_popcount(rem);
    if (n < 2) return 0.0;
    if (memo[rem] >= 0) return memo[rem];
    double tot = 0;
    if (n == 2) {
        const int a = __builtin_ctz(rem), b = 31 - __builtin_clz(rem);
        tot = kCostPair + kCostGroup * (double)(radix[a] + radix[b]);
    } else {
        for (uint32_t m = rem; m; m &= m - 1) {
            const int j = __builtin_ctz(m);
            tot += (double)radix[j] * (kCostMerge + walk_cost(radix, rem & ~(1u << j), memo));
        }
    }
    memo[rem] = tot;
    return tot;
}

int tree_layout_build(const sat_problem_t *p, int prefix_len, TreeLayout &lay) {
    const int J = p->J;
    if (p->N != 1 || p->time_mode != SAT_TIME_GRID_I32) return SAT_ERR_UNSUPPORTED;
    if (J < 3 || J > kTreeMaxJ) return SAT_ERR_UNSUPPORTED;
    if (p->release_i32)
        for (int j = 0; j < J; ++j) if (p->release_i32[j] != 0) return SAT_ERR_UNSUPPORTED;
    int n_opt = 0;
    for (int j = 0; j < J; ++j) n_opt += p->radix[j];
    if (n_opt > kTreeMaxOpt) return SAT_ERR_UNSUPPORTED;
    uint64_t space;
    if (!space_size(p, &space)) return SAT_ERR_TOO_LARGE;
    auto build = [&](int P, TreeLayout &L) -> bool {
        L = TreeLayout();
        L.P = P;
        const uint64_t fP = factorial_u64(P);
        for (uint32_t S = 0; S < (1u << J); ++S) {
            if (__builtin_popcount(S) != P) continue;
            unsigned __int128 pr = 1;
            for (int j = 0; j < J; ++j) if (S >> j & 1u) pr *= (unsigned)p->radix[j];
            L.sets.push_back(S);
            L.prod.push_back((uint64_t)pr);
            L.cum.push_back(L.n_tasks);
            L.n_tasks += ((uint64_t)pr * fP + 31) / 32;
            if (L.sets.size() > (size_t)kTreeMaxSets) return false;
        }
        L.cum.push_back(L.n_tasks);
        L.n_cand = space;
        return true;
    };
    int P = prefix_len;
    if (P <= 0) {
        // smallest prefix giving enough warp tasks for one GPU's dynamic cursor (2^15, ~5 per
        // resident warp) whose suffix the fixed-depth walkers cover (<= 4 jobs; deeper suffixes
        // take the generic local-memory walk).  cfg1: P = 4, 8.2 ms against 8.6 ms at P = 5
        // (profiles/r01e_shard_emulation.txt).  Sharded callers pass a longer prefix.
        P = 0;
        for (int cand = std::max(1, J - 4); cand <= J - 2; ++cand) {
            TreeLayout t;
            if (!build(cand, t) || t.n_tasks >= (1ull << 31)) break;
            if (t.n_tasks >= (1ull << 15)) { P = cand; break; }
        }
        if (P == 0) {   // large problems: the shortest prefix with 2^17 tasks (generic walk below)
            P = J - 2;
            for (int cand = 1; cand <= J - 2; ++cand) {
                TreeLayout t;
                if (!build(cand, t)) break;
                if (t.n_tasks >= (1ull << 17)) { P = cand; break; }
            }
        }
    }
    if (P < 1 || P > J - 2) return SAT_ERR_INVALID;
    if (!build(P, lay)) return SAT_ERR_UNSUPPORTED;
    // placements: P per lane prefix + the suffix walk
    std::vector<int64_t> memo((size_t)1 << J, -1);
    const uint32_t full = (1u << J) - 1u;
    const uint64_t fP = factorial_u64(P);
    lay.n_steps = 0;
    for (size_t s = 0; s < lay.sets.size(); ++s) {
        const uint64_t npref = fP * lay.prod[s];
        lay.n_steps += npref * ((uint64_t)P + walk_nodes(p->radix, full & ~lay.sets[s], memo, full));
    }
    return SAT_OK;
}

// tree_layout is a pure function of (J, radix[], requested prefix): memoised per process so that
// repeated solves, re-solves and the host's prefix probing (Engine.bnb_prefix calls sat_tree_plan
// once per P) do not redo the 2^J set enumeration and walk memo each call.  A small LRU under a
// mutex keeps the C ABI reentrant; results are identical with or without it.
struct LayoutKey {
    int J = 0, P = 0;
    int32_t radix[kTreeMaxJ] = {};
    bool operator==(const LayoutKey &o) const {
        return J == o.J && P == o.P && std::memcmp(radix, o.radix, sizeof(int32_t) * J) == 0;
    }
};
struct LayoutEntry {
    LayoutKey key;
    int status = SAT_OK;
    TreeLayout lay;
    std::vector<long double> per_task;     // sat_tree_shard's per-task cost, filled on first use
};
static std::mutex g_layout_mu;
static std::list<std::shared_ptr<LayoutEntry>> g_layouts;     // most recent first
constexpr size_t kLayoutCacheEntries = 32;

std::shared_ptr<LayoutEntry> tree_layout_cached(const sat_problem_t *p, int prefix_len) {
    LayoutKey k;
    k.J = p->J;
    k.P = prefix_len <= 0 ? 0 : prefix_len;
    if (p->J >= 1 && p->J <= kTreeMaxJ) std::memcpy(k.radix, p->radix, sizeof(int32_t) * p->J);
    {
        std::lock_guard<std::mutex> g(g_layout_mu);
        for (auto it = g_layouts.begin(); it != g_layouts.end(); ++it)
            if ((*it)->key == k) {
                auto e = *it;
                g_layouts.erase(it);
                g_layouts.push_front(e);
                return e;
            }
    }
    auto e = std::make_shared<LayoutEntry>();
    e->key = k;
    e->status = tree_layout_build(p, prefix_len, e->lay);
    std::lock_guard<std::mutex> g(g_layout_mu);
    g_layouts.push_front(e);
    if (g_layouts.size() > kLayoutCacheEntries) g_layouts.pop_back();
    return e;
}

// the shape checks tree_layout_build makes that do not depend on the radices (the cache key)
int tree_layout(const sat_problem_t *p, int prefix_len, TreeLayout &lay) {
    if (p->N != 1 || p->time_mode != SAT_TIME_GRID_I32) return SAT_ERR_UNSUPPORTED;
    if (p->J < 3 || p->J > kTreeMaxJ) return SAT_ERR_UNSUPPORTED;
    if (p->release_i32)
        for (int j = 0; j < p->J; ++j) if (p->release_i32[j] != 0) return SAT_ERR_UNSUPPORTED;
    auto e = tree_layout_cached(p, prefix_len);
    if (e->status == SAT_OK) lay = e->lay;
    return e->status;
}

struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

}  // namespace sat

using namespace sat;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int sat_abi_version(void) { return SAT_ABI_VERSION; }

const char *sat_error_string(int status) {
    switch (status) {
        case SAT_OK: return "ok";
        case SAT_ERR_INVALID: return "invalid problem or arguments";
        case SAT_ERR_NO_OPTIONS: return "a job has no feasible option";
        case SAT_ERR_TOO_LARGE: return "search space, key or tables exceed the engine encoding";
        case SAT_ERR_UNSUPPORTED: return "problem shape not supported by this kernel";
        case SAT_ERR_CUDA: return "CUDA launch or runtime failure";
        default: return "unknown status";
    }
}

int sat_device_info(int device, int32_t *sm_count, int32_t *cc_major, int32_t *cc_minor) {
    int v = 0;
    if (sm_count) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return SAT_ERR_CUDA;
        *sm_count = v;
    }
    if (cc_major) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) return SAT_ERR_CUDA;
        *cc_major = v;
    }
    if (cc_minor) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess) return SAT_ERR_CUDA;
        *cc_minor = v;
    }
    return SAT_OK;
}

int sat_best_reset(sat_best_t *d_best, void *stream) {
    if (!d_best) return SAT_ERR_INVALID;
    return check_cuda(cudaMemsetAsync(d_best, 0xFF, sizeof(sat_best_t), (cudaStream_t)stream));
}

// ---- cross-rank shared incumbent (NVLink peer memory) ----
int sat_best_set(sat_best_t *d_best, uint64_t hi, uint64_t lo, void *stream) {
    if (!d_best) return SAT_ERR_INVALID;
    // a kernel-free 16-byte write: cudaMemcpyAsync from pageable host memory completes the
    // host-side copy before returning, so a stack value is safe
    const sat_best_t v{hi, lo};
    return check_cuda(cudaMemcpyAsync(d_best, &v, sizeof(v), cudaMemcpyHostToDevice, (cudaStream_t)stream));
}

int sat_best_copy(sat_best_t *d_dst, const sat_best_t *d_src, void *stream) {
    if (!d_dst || !d_src) return SAT_ERR_INVALID;
    return check_cuda(cudaMemcpyAsync(d_dst, d_src, sizeof(sat_best_t), cudaMemcpyDefault, (cudaStream_t)stream));
}

// ---- search key hand-off (ABI v7): one launch instead of the host library's elementwise ops ----
// out[0..n_words) = the best cell's words, "empty" (all ones) -> INT64_MAX; out[n_words + e] =
// extra[e]; ids[0] = the replay id of out[0] (grid key: low idx_bits; an empty or out-of-range
// key -> 0, an id the decode can take).  best == NULL: ids only (after a cross-rank MIN of out).
static __global__ void k_key_finish(const uint64_t *best, int n_words, const uint64_t *extra, int n_extra,
                                    int64_t *out, uint64_t *ids, int idx_bits, uint64_t n_idx, int check) {
    const int i = threadIdx.x;
    if (best && i < n_words) {
        const uint64_t v = best[i];
        out[i] = v == ~0ull ? INT64_MAX : (int64_t)v;
    }
    if (i < n_extra) out[n_words + i] = (int64_t)extra[i];
    if (ids && i == 0) {
        const uint64_t v = best ? best[0] : (uint64_t)out[0];
        const int64_t k = (best && v == ~0ull) ? INT64_MAX : (int64_t)v;
        const uint64_t idx = (uint64_t)k & ((idx_bits >= 64) ? ~0ull : ((1ull << idx_bits) - 1ull));
        ids[0] = (k == INT64_MAX || (check && idx >= n_idx)) ? 0ull : idx;
    }
}

int sat_key_finish(const sat_best_t *d_best, int32_t n_words, const uint64_t *d_extra, int32_t n_extra,
                   int64_t *d_out, uint64_t *d_ids, int32_t idx_bits, uint64_t n_idx, int32_t check_range,
                   void *stream) {
    if (!d_out || n_words < 1 || n_words > 2 || n_extra < 0 || n_extra > 30 || (n_extra && !d_extra) ||
        idx_bits < 1 || idx_bits > 64)
        return SAT_ERR_INVALID;
    k_key_finish<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<const uint64_t *>(d_best), n_words,
                                                    d_extra, n_extra, d_out, d_ids, idx_bits, n_idx, check_range);
    return check_cuda(cudaGetLastError());
}

int sat_shared_best_alloc(sat_best_t **d_cell, uint8_t *handle_out) {
    if (!d_cell || !handle_out) return SAT_ERR_INVALID;
    static_assert(sizeof(cudaIpcMemHandle_t) == SAT_IPC_HANDLE_BYTES, "IPC handle size");
    void *p = nullptr;
    if (cudaMalloc(&p, 2 * sizeof(sat_best_t)) != cudaSuccess) return SAT_ERR_CUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) { cudaFree(p); return SAT_ERR_CUDA; }
    std::memcpy(handle_out, &h, sizeof(h));
    if (cudaMemset(p, 0xFF, 2 * sizeof(sat_best_t)) != cudaSuccess) { cudaFree(p); return SAT_ERR_CUDA; }
    *d_cell = static_cast<sat_best_t *>(p);
    return SAT_OK;
}

int sat_shared_best_open(const uint8_t *handle, sat_best_t **d_cell) {
    if (!d_cell || !handle) return SAT_ERR_INVALID;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return SAT_ERR_CUDA;
    *d_cell = static_cast<sat_best_t *>(p);
    return SAT_OK;
}

int sat_shared_best_close(sat_best_t *d_cell, int32_t owner) {
    if (!d_cell) return SAT_ERR_INVALID;
    return check_cuda(owner ? cudaFree(d_cell) : cudaIpcCloseMemHandle(d_cell));
}

int sat_peer_atomics(int32_t dev_a, int32_t dev_b, int32_t *supported) {
    if (!supported) return SAT_ERR_INVALID;
    if (dev_a == dev_b) { *supported = 1; return SAT_OK; }
    int v = 0;
    if (cudaDeviceGetP2PAttribute(&v, cudaDevP2PAttrNativeAtomicSupported, dev_a, dev_b) != cudaSuccess)
        return SAT_ERR_CUDA;
    *supported = v;
    return SAT_OK;
}

int sat_workspace_bytes(const sat_problem_t *p, size_t *bytes) {
    int st = validate(p);
    if (st) return st;
    std::vector<uint8_t> blob;
    st = pack_blob(p, blob, records_carry_duration(p));
    if (st) return st;
    const size_t part_off = (blob.size() + 255) & ~(size_t)255;
    *bytes = part_off + (size_t)device_sms() * 32 * sizeof(sat_best_t) + 256;   // + k_cand chunk cursor
    return SAT_OK;
}

int sat_search_index(const sat_problem_t *p, uint64_t lo, uint64_t hi, sat_best_t *d_best, void *d_ws,
                     size_t ws_bytes, void *stream) {
    NvtxRange nvtx("sat_search_index");
    int st = validate(p);
    if (st) return st;
    if (!d_best || hi < lo) return SAT_ERR_INVALID;
    uint64_t space;
    if (!space_size(p, &space)) return SAT_ERR_TOO_LARGE;
    if (hi > space) return SAT_ERR_INVALID;
    if (p->time_mode == SAT_TIME_GRID_I32 && p->idx_bits < 64 && (space - 1) >> p->idx_bits) return SAT_ERR_TOO_LARGE;
    if (hi == lo) return SAT_OK;
    CandArgs a{};
    a.lo = lo; a.hi = hi; a.best = d_best;
    a.per_lane = 16;
    cudaStream_t s = (cudaStream_t)stream;
    if (p->time_mode == SAT_TIME_F64)
        return launch_cand<double, SAT_SRC_INDEX>(p, a, hi - lo, d_ws, ws_bytes, s);
    return launch_cand<int32_t, SAT_SRC_INDEX>(p, a, hi - lo, d_ws, ws_bytes, s);
}

int sat_search_sampled(const sat_problem_t *p, int32_t source, uint64_t seed, uint64_t lo, uint64_t hi,
                       sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx("sat_search_sampled");
    int st = validate(p);
    if (st) return st;
    if (!d_best || hi < lo) return SAT_ERR_INVALID;
    if (source != SAT_SRC_SUBSTREAM && source != SAT_SRC_SEED) return SAT_ERR_INVALID;
    if (p->time_mode == SAT_TIME_GRID_I32 && hi > 0 && ((hi - 1) >> p->idx_bits)) return SAT_ERR_TOO_LARGE;
    if (hi == lo) return SAT_OK;
    CandArgs a{};
    a.lo = lo; a.hi = hi; a.best = d_best; a.seed = seed; a.per_lane = 8;
    cudaStream_t s = (cudaStream_t)stream;
    if (p->time_mode == SAT_TIME_F64) {
        if (source == SAT_SRC_SUBSTREAM)
            return launch_cand<double, SAT_SRC_SUBSTREAM>(p, a, hi - lo, d_ws, ws_bytes, s);
        return launch_cand<double, SAT_SRC_SEED>(p, a, hi - lo, d_ws, ws_bytes, s);
    }
    if (source == SAT_SRC_SUBSTREAM)
        return launch_cand<int32_t, SAT_SRC_SUBSTREAM>(p, a, hi - lo, d_ws, ws_bytes, s);
    return launch_cand<int32_t, SAT_SRC_SEED>(p, a, hi - lo, d_ws, ws_bytes, s);
}

int sat_schedule(const sat_problem_t *p, int32_t source, uint64_t seed, const uint64_t *d_ids,
                 const uint8_t *d_explicit, int32_t n, int32_t *d_option, int32_t *d_node,
                 int32_t *d_start_i32, double *d_start_f64, int64_t *d_makespan_i64,
                 double *d_makespan_f64, void *d_ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx("sat_schedule");
    int st = validate(p);
    if (st) return st;
    if (n < 0) return SAT_ERR_INVALID;
    if (n == 0) return SAT_OK;
    if (source == SAT_SRC_EXPLICIT ? !d_explicit : !d_ids) return SAT_ERR_INVALID;
    GenArgs a{};
    a.lo = 0; a.hi = (uint64_t)n; a.seed = seed; a.per_lane = 1;
    a.ids = d_ids; a.expl = d_explicit;
    a.rec_opt = d_option; a.rec_node = d_node;
    a.rec_start_i32 = d_start_i32; a.rec_start_f64 = d_start_f64;
    a.rec_ms_i64 = d_makespan_i64; a.rec_ms_f64 = d_makespan_f64;
    cudaStream_t s = (cudaStream_t)stream;
    const uint64_t nn = (uint64_t)n;
    if (p->time_mode == SAT_TIME_F64) {
        switch (source) {
            case SAT_SRC_INDEX: return launch_generic<double, SAT_SRC_INDEX, true>(p, a, nn, d_ws, ws_bytes, s);
            case SAT_SRC_SUBSTREAM: return launch_generic<double, SAT_SRC_SUBSTREAM, true>(p, a, nn, d_ws, ws_bytes, s);
            case SAT_SRC_SEED: return launch_generic<double, SAT_SRC_SEED, true>(p, a, nn, d_ws, ws_bytes, s);
            case SAT_SRC_EXPLICIT: return launch_generic<double, SAT_SRC_EXPLICIT, true>(p, a, nn, d_ws, ws_bytes, s);
            default: return SAT_ERR_INVALID;
        }
    }
    switch (source) {
        case SAT_SRC_INDEX: return launch_generic<int32_t, SAT_SRC_INDEX, true>(p, a, nn, d_ws, ws_bytes, s);
        case SAT_SRC_SUBSTREAM: return launch_generic<int32_t, SAT_SRC_SUBSTREAM, true>(p, a, nn, d_ws, ws_bytes, s);
        case SAT_SRC_SEED: return launch_generic<int32_t, SAT_SRC_SEED, true>(p, a, nn, d_ws, ws_bytes, s);
        case SAT_SRC_EXPLICIT: return launch_generic<int32_t, SAT_SRC_EXPLICIT, true>(p, a, nn, d_ws, ws_bytes, s);
        default: return SAT_ERR_INVALID;
    }
}

// k_tree's pair pass runs on 16-bit pairs when every free time a schedule can reach (the
// latest initial free time + the sum of every job's longest option) stays below
// kTreePackLimit, on nodes of <= kTreePackMaxG GPUs (SATURN_TREE_PACKED=0 forces the
// 32-bit pass, for A/B checks)
static bool tree_pair_packed(const sat_problem_t *p) {
    const int G = p->node_gpus[0];
    if (G < 2 || G > kTreePackMaxG) return false;
    const char *env = std::getenv("SATURN_TREE_PACKED");
    if (env && env[0] == '0') return false;
    int64_t horizon = 0;
    for (int i = 0; i < G; ++i) horizon = std::max<int64_t>(horizon, p->init_free_i32 ? p->init_free_i32[i] : 0);
    for (int j = 0; j < p->J; ++j) {
        int32_t dmax = 0;
        for (int o = 0; o < p->radix[j]; ++o) dmax = std::max(dmax, p->dur_i32[j * p->Cmax + o]);
        horizon += dmax;
    }
    return horizon < kTreePackLimit;
}

int sat_tree_plan(const sat_problem_t *p, int32_t prefix_len, sat_tree_info_t *info) {
    int st = validate(p);
    if (st) return st;
    if (!info) return SAT_ERR_INVALID;
    TreeLayout lay;
    st = tree_layout(p, prefix_len, lay);
    if (st) return st;
    info->prefix_len = lay.P;
    info->n_sets = (int32_t)lay.sets.size();
    info->n_tasks = lay.n_tasks;
    info->n_candidates = lay.n_cand;
    info->n_job_steps = lay.n_steps;
    info->pair_packed = tree_pair_packed(p) ? 1 : 0;
    info->reserved = 0;
    return SAT_OK;
}

static int search_tree_impl(const sat_problem_t *p, int32_t prefix_len, uint64_t task_lo, uint64_t task_hi,
                            sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream, bool bnb) {
    NvtxRange nvtx(bnb ? "sat_search_bnb" : "sat_search_tree");
    int st = validate(p);
    if (st) return st;
    if (!d_best || task_hi < task_lo) return SAT_ERR_INVALID;
    if (!d_ws || ws_bytes < SAT_TREE_WS_BYTES) return SAT_ERR_INVALID;
    TreeLayout lay;
    st = tree_layout(p, prefix_len, lay);
    if (st) return st;
    if (task_hi > lay.n_tasks) return SAT_ERR_INVALID;
    if (task_hi - task_lo >= (1ull << 32)) return SAT_ERR_TOO_LARGE;   // task ids travel as 32-bit
    if ((lay.n_cand - 1) >> p->idx_bits) return SAT_ERR_TOO_LARGE;
    if (task_hi == task_lo) return SAT_OK;
    TreeParams tp;
    std::memset(&tp, 0, sizeof(tp));
    const int J = p->J;
    tp.J = J; tp.P = lay.P; tp.Q = J - lay.P; tp.Gr = p->node_gpus[0];
    tp.n_sets = (int32_t)lay.sets.size(); tp.idx_bits = p->idx_bits;
    tp.fact[0] = 1;
    for (int k = 1; k <= J; ++k) tp.fact[k] = tp.fact[k - 1] * (uint64_t)k;
    uint64_t w = 1;
    for (int j = J - 1; j >= 0; --j) { tp.wJ[j] = w * tp.fact[J]; w *= (uint64_t)p->radix[j]; }
    int q = 0;
    for (int j = 0; j < J; ++j) {
        tp.radix[j] = p->radix[j];
        tp.optbase[j] = q;
        for (int o = 0; o < p->radix[j]; ++o, ++q) {
            const int g = p->gpus[j * p->Cmax + o];
            tp.optg[q] = g;
            tp.optoff[q] = (g - 1) * 32;
            tp.optd[q] = p->dur_i32[j * p->Cmax + o];
        }
    }
    for (int j = 0; j < J; ++j) {
        for (int k = 0; k < 32; ++k) tp.dg[j][k] = SAT_INF_I32;
        for (int o = 0; o < p->radix[j]; ++o) {
            const int g = p->gpus[j * p->Cmax + o];
            tp.dg[j][g - 1] = std::min(tp.dg[j][g - 1], p->dur_i32[j * p->Cmax + o]);
        }
    }
    int32_t imax = 0;
    for (int i = 0; i < 32; ++i) {
        const bool real = i < tp.Gr;
        const int32_t v = real ? (p->init_free_i32 ? p->init_free_i32[i] : 0) : SAT_INF_I32;
        tp.init_free[i] = v;
        if (real) imax = std::max(imax, v);
    }
    tp.init_max = imax;
    tp.packed = tree_pair_packed(p) ? 1 : 0;
    for (int j = 0; j < J; ++j)
        for (int w = 0; w < kTreePackMaxG / 2; ++w) {
            uint32_t lo = kTreeInf16, hi = kTreeInf16;
            if (2 * w < tp.Gr && tp.dg[j][2 * w] < SAT_INF_I32) lo = (uint32_t)tp.dg[j][2 * w];
            if (2 * w + 1 < tp.Gr && tp.dg[j][2 * w + 1] < SAT_INF_I32) hi = (uint32_t)tp.dg[j][2 * w + 1];
            tp.dgp[j][w] = tp.packed ? (lo | (hi << 16)) : 0u;
        }
    for (size_t s = 0; s < lay.sets.size(); ++s) {
        tp.set_mask[s] = lay.sets[s];
        tp.set_cum[s] = lay.cum[s];
        tp.set_prod[s] = lay.prod[s];
    }
    tp.set_cum[lay.sets.size()] = lay.cum.back();
    tp.task_lo = task_lo; tp.task_hi = task_hi;
    tp.best = d_best;
    tp.cursor = static_cast<unsigned long long *>(d_ws);
    tp.stats = tp.cursor + 1;
    for (int j = 0; j < J; ++j) {
        int32_t a = SAT_INF_I32;
        for (int o = 0; o < p->radix[j]; ++o)
            a = std::min<int64_t>(a, (int64_t)p->gpus[j * p->Cmax + o] * p->dur_i32[j * p->Cmax + o]);
        tp.minarea[j] = a;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(d_ws, 0, 3 * sizeof(unsigned long long), s) != cudaSuccess) return SAT_ERR_CUDA;
    // the walk is specialised on the node's exact GPU count (no ghost slots)
    switch (tp.Gr) {
#define SAT_G(K) case K: return launch_tree_g<K>(tp, tp.Q, bnb, s);
        SAT_G(1) SAT_G(2) SAT_G(3) SAT_G(4) SAT_G(5) SAT_G(6) SAT_G(7) SAT_G(8)
        SAT_G(9) SAT_G(10) SAT_G(11) SAT_G(12) SAT_G(13) SAT_G(14) SAT_G(15) SAT_G(16)
        SAT_G(17) SAT_G(18) SAT_G(19) SAT_G(20) SAT_G(21) SAT_G(22) SAT_G(23) SAT_G(24)
        SAT_G(25) SAT_G(26) SAT_G(27) SAT_G(28) SAT_G(29) SAT_G(30) SAT_G(31) SAT_G(32)
#undef SAT_G
        default: return SAT_ERR_UNSUPPORTED;
    }
}

size_t sat_tree_param_bytes(void) { return sizeof(TreeParams); }

int sat_tree_shard(const sat_problem_t *p, int32_t prefix_len, int32_t world, int32_t rank, uint64_t *task_lo,
                   uint64_t *task_hi) {
    int st = validate(p);
    if (st) return st;
    if (world < 1 || rank < 0 || rank >= world || !task_lo || !task_hi) return SAT_ERR_INVALID;
    TreeLayout lay;
    st = tree_layout(p, prefix_len, lay);
    if (st) return st;
    // per-task device cost of set s: the prefix decode + the warp's suffix walk (walk_cost),
    // computed once per cached layout
    auto entry = tree_layout_cached(p, prefix_len);
    std::vector<long double> per_task;
    {
        std::lock_guard<std::mutex> g(g_layout_mu);
        per_task = entry->per_task;
    }
    if (per_task.empty()) {
        const uint32_t full = (1u << p->J) - 1u;
        std::vector<double> memo((size_t)1 << p->J, -1.0);
        per_task.resize(lay.sets.size());
        for (size_t s = 0; s < lay.sets.size(); ++s)
            per_task[s] = (long double)(kCostTask + walk_cost(p->radix, full & ~lay.sets[s], memo));
        std::lock_guard<std::mutex> g(g_layout_mu);
        entry->per_task = per_task;
    }
    long double total = 0;
    for (size_t s = 0; s < lay.sets.size(); ++s) total += per_task[s] * (long double)(lay.cum[s + 1] - lay.cum[s]);
    auto boundary = [&](int32_t r) -> uint64_t {      // first task whose prefix work >= total * r / world
        if (r <= 0) return 0;
        if (r >= world) return lay.n_tasks;
        const long double target = total * (long double)r / (long double)world;
        long double acc = 0;
        for (size_t s = 0; s < lay.sets.size(); ++s) {
            const uint64_t nt = lay.cum[s + 1] - lay.cum[s];
            const long double c = per_task[s] * (long double)nt;
            if (acc + c >= target) {
                const uint64_t k = (uint64_t)((target - acc) / per_task[s]);
                return lay.cum[s] + std::min<uint64_t>(k, nt);
            }
            acc += c;
        }
        return lay.n_tasks;
    };
    *task_lo = boundary(rank);
    *task_hi = boundary(rank + 1);
    return SAT_OK;
}

int sat_ls_counter_offset(const sat_problem_t *p, size_t *offset) {
    int st = validate(p);
    if (st) return st;
    if (!offset) return SAT_ERR_INVALID;
    std::vector<uint8_t> blob;
    st = pack_blob(p, blob, records_carry_duration(p));
    if (st) return st;
    *offset = ((blob.size() + 255) & ~(size_t)255) + sizeof(unsigned long long);
    return SAT_OK;
}

// greedy starts: per job the least-area usable option (area = g x its least duration over
// the nodes that can run it; ties: lowest option) and that duration, the order key's base
static bool ls_greedy_tables(const sat_problem_t *p, uint8_t *gopt, uint32_t *gdur) {
    if (p->J > 64) return false;
    const uint32_t all = p->N >= 32 ? ~0u : ((1u << p->N) - 1u);
    for (int j = 0; j < p->J; ++j) {
        int64_t best_area = INT64_MAX;
        int best_o = -1;
        int32_t best_d = 0;
        for (int o = 0; o < p->radix[j]; ++o) {
            const int q = j * p->Cmax + o;
            const uint32_t m = p->node_mask ? p->node_mask[q] & all : all;
            int32_t d = INT32_MAX;
            for (int n = 0; n < p->N; ++n)
                if (((m >> n) & 1u) && p->gpus[q] <= p->node_gpus[n]) d = std::min(d, p->dur_i32[q * p->N + n]);
            if (d == INT32_MAX) continue;
            const int64_t area = (int64_t)p->gpus[q] * d;
            if (area < best_area) { best_area = area; best_o = o; best_d = d; }
        }
        if (best_o < 0) return false;
        gopt[j] = (uint8_t)best_o;
        gdur[j] = (uint32_t)std::max<int32_t>(best_d, 0);
    }
    return true;
}

int sat_local_search(const sat_problem_t *p, int32_t source, uint64_t seed, uint64_t lo, uint64_t hi,
                     int32_t max_rounds, int32_t stop_ms, sat_best_t *d_best, uint8_t *d_state_out, void *d_ws,
                     size_t ws_bytes,
                     void *stream) {
    NvtxRange nvtx("sat_local_search");
    int st = validate(p);
    if (st) return st;
    if (!d_best || hi < lo || max_rounds < 0 || max_rounds >= (1 << SAT_LS_ROUND_BITS)) return SAT_ERR_INVALID;
    if (source != SAT_SRC_SUBSTREAM && source != SAT_SRC_SEED && source != SAT_SRC_GREEDY) return SAT_ERR_INVALID;
    if (p->time_mode != SAT_TIME_GRID_I32) return SAT_ERR_UNSUPPORTED;
    if (p->J < 2) return SAT_ERR_UNSUPPORTED;
    if (hi > 0 && ((hi - 1) >> p->idx_bits)) return SAT_ERR_TOO_LARGE;
    if (p->idx_bits + SAT_LS_ROUND_BITS > 56) return SAT_ERR_TOO_LARGE;     // the makespan keeps >= 7 bits
    if (hi == lo) return SAT_OK;
    LsArgs a{};
    a.lo = lo; a.hi = hi; a.seed = seed; a.max_rounds = max_rounds; a.best = d_best; a.state_out = d_state_out;
    a.stop_ms = stop_ms < 0 ? -1 : stop_ms; a.idx_bits = p->idx_bits;
    cudaStream_t s = (cudaStream_t)stream;
    if (source == SAT_SRC_GREEDY) {
        if (!ls_greedy_tables(p, a.gopt, a.gdur)) return SAT_ERR_NO_OPTIONS;
        a.greedy = 1;                                  // noise from the walker's substream
        return launch_ls<SAT_SRC_SUBSTREAM>(p, a, d_ws, ws_bytes, s);
    }
    if (source == SAT_SRC_SUBSTREAM) return launch_ls<SAT_SRC_SUBSTREAM>(p, a, d_ws, ws_bytes, s);
    return launch_ls<SAT_SRC_SEED>(p, a, d_ws, ws_bytes, s);
}

int sat_search_tree(const sat_problem_t *p, int32_t prefix_len, uint64_t task_lo, uint64_t task_hi,
                    sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream) {
    return search_tree_impl(p, prefix_len, task_lo, task_hi, d_best, d_ws, ws_bytes, stream, false);
}

int sat_search_bnb(const sat_problem_t *p, int32_t prefix_len, uint64_t task_lo, uint64_t task_hi,
                   sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream) {
    return search_tree_impl(p, prefix_len, task_lo, task_hi, d_best, d_ws, ws_bytes, stream, true);
}

int sat_alu_probe(int32_t blocks, int32_t threads, int32_t iters, uint64_t *d_ops_out, int32_t *d_sink,
                  void *stream) {
    if (blocks < 1 || threads < 32 || iters < 1 || !d_ops_out || !d_sink) return SAT_ERR_INVALID;
    k_alu_probe<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, (unsigned long long *)d_ops_out, d_sink);
    return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
}

int sat_alu_probe16(int32_t blocks, int32_t threads, int32_t iters, uint64_t *d_ops_out, int32_t *d_sink,
                    void *stream) {
    if (blocks < 1 || threads < 32 || iters < 1 || !d_ops_out || !d_sink) return SAT_ERR_INVALID;
    k_alu_probe16<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, (unsigned long long *)d_ops_out, d_sink);
    return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
}

}  // extern "C"
