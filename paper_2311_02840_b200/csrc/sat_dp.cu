// sat_dp.cu -- state-space search of the list-scheduling candidate space (one node, grid time).
//
// Every candidate (options + submission order) is a path of J placements.  After k placements
// the list scheduler's whole future depends only on the STATE (set of jobs still to place,
// sorted GPU free times): the makespan of any completion is a function of that state and of
// the remaining choices.  Many prefixes reach the same state (different orders of jobs that
// end up at the same free-time profile), so enumerating distinct states level by level covers
// the prod(radix) x J! candidates with far fewer nodes than the prefix tree of k_tree.
//
// sat_search_dp answers "is there a candidate with makespan <= T?" exactly:
//   level k -> k+1: every state x (job j still to place) x (option o of j) is placed with the
//   same sorted-vector update as the other kernels (b[i] = max(a[i], min(a[i+g], e)), start =
//   max(a[g-1], release)); children whose makespan lower bound exceeds T are cut -- the bound
//   is the bound-and-prune one: committed end e <= T, area (sum of free times + least area of
//   every job still to place <= T x G), and every remaining job's earliest end
//   (min_k max(b[k], rel) + least duration at gang k+1 <= T).  Distinct children go to a
//   global hash set keyed EXACTLY (R bits x C(T+G, G) + combinatorial rank of the sorted free
//   times: the state itself, no fingerprints, so the dedup is sound).  An empty level proves
//   that no candidate reaches T (the proof configs 3-5's lower bound cannot give); a
//   non-empty last level yields one such candidate, rebuilt backwards level by level
//   (deterministically: the smallest-key final state, then the smallest-key parent and the
//   lowest option at each step).
//
// One thread per (state, job); the level loop is driven from the host (one small read-back
// per level).  HBM holds every level's states (kept for the reconstruction).
#include "sat_common.cuh"

#include <nvtx3/nvToolsExt.h>

#include <cmath>

namespace sat {

constexpr int kDpMaxJ = 64;
constexpr int kDpMaxOpt = 1024;
constexpr int kDpThreads = 256;
constexpr uint64_t kDpEmpty = ~0ull;

struct DpParams {
    int32_t J, Gr, T, rank_unused;
    uint64_t cnum;                    // C(T + Gr, Gr): sorted free-time vectors with values <= T
    int32_t ubase[kDpMaxJ], ucnt[kDpMaxJ];   // usable options of job j: [ubase, ubase + ucnt)
    int32_t release[kDpMaxJ];
    int32_t minarea[kDpMaxJ];         // least g x d over the job's usable options
    uint8_t ug[kDpMaxOpt];            // gang size of usable option q
    int16_t ud[kDpMaxOpt];            // duration of usable option q
    int16_t dg[kDpMaxJ][32];          // least usable duration of job j at gang k+1 (T+1: none)
    uint32_t dgp[kDpMaxJ][16];        // dg as 16-bit pairs (gangs 2w+1, 2w+2), for VIADDMNMX.U16x2
    int32_t nrem;                     // jobs still to place in the level being expanded
    int32_t has_release;
    int32_t umax;                     // most usable options of any job
    const uint64_t *binom;            // [(T + Gr + 1)][Gr + 1]: C(n, k)
    uint64_t *table;                  // hash set of state keys, kDpEmpty = free
    uint64_t cap_mask;
    int32_t cap_log2;
    int32_t max_probe;
    uint64_t *all_R;                  // every level's states, appended level after level:
    uint16_t *all_A;                  //   remaining-job sets, sorted free times [][Gr]
    uint64_t max_states;
    unsigned long long *lvl_cnt;      // [J + 1] states of each level
    unsigned long long *lvl_base;     // [J + 2] first state of each level
    unsigned int *overflow;           // level + 1 whose expansion exceeded the budget or probe limit
    // reconstruction: one level's states
    const uint64_t *in_R;
    const uint16_t *in_A;
    uint64_t n_in;
    // reconstruction (k_dp_parent): the child state searched for
    uint64_t child_R;
    uint16_t child_A[32];
    unsigned long long *min_key;
};

__device__ __forceinline__ uint64_t dp_rank(const DpParams &p, const int32_t *b) {
    const int K = p.Gr + 1;
    uint64_t r = 0;
    for (int i = 0; i < p.Gr; ++i) r += __ldg(&p.binom[(b[i] + i) * K + (i + 1)]);
    return r;
}

// place option q (gang g, duration d) of a job with release rel on the sorted vector a
// (a[Gr..] = +inf); returns the end time, b = the new sorted vector
template <int GM>
__device__ __forceinline__ int32_t dp_place(const int32_t *a, int Gr, int g, int d, int rel, int32_t *b) {
    const int32_t t = max(a[g - 1], rel);
    const int32_t e = t + d;
#pragma unroll
    for (int i = 0; i < GM; ++i) {
        if (i < Gr) {
            const int32_t up = (i + g < Gr) ? a[i + g] : 0x7fffffff;
            b[i] = max(a[i], min(up, e));
        }
    }
    return e;
}

// per-block copies of the tables the expansion indexes by job / option: the threads of a warp
// work on different jobs, and divergent indices into the kernel parameters (constant bank)
// serialise, while shared-memory reads of distinct words do not
template <int GM>
struct DpShared {
    uint32_t dgp[kDpMaxJ][GM / 2];
    int32_t minarea[kDpMaxJ], release[kDpMaxJ], ubase[kDpMaxJ], ucnt[kDpMaxJ];
    int16_t ud[kDpMaxOpt];
    uint8_t ug[kDpMaxOpt];
};

template <int GM>
__device__ __forceinline__ void dp_stage(const DpParams &p, DpShared<GM> &sh) {
    constexpr int W = GM / 2;
    const int nopt = p.J ? p.ubase[p.J - 1] + p.ucnt[p.J - 1] : 0;
    for (int x = threadIdx.x; x < p.J * W; x += blockDim.x) sh.dgp[x / W][x % W] = p.dgp[x / W][x % W];
    for (int x = threadIdx.x; x < p.J; x += blockDim.x) {
        sh.minarea[x] = p.minarea[x];
        sh.release[x] = p.release[x];
        sh.ubase[x] = p.ubase[x];
        sh.ucnt[x] = p.ucnt[x];
    }
    for (int x = threadIdx.x; x < nopt; x += blockDim.x) { sh.ud[x] = p.ud[x]; sh.ug[x] = p.ug[x]; }
}

// bound-and-prune test of a packed child state (R2, bp): can some completion end by T?  Each
// remaining job's earliest end is GM/2 fused add-mins (VIADDMNMX.U16x2) of the packed state and
// its packed least durations; free times and durations are <= T + 1 <= 30001 and padding 0x7FFF,
// so no pair sum carries.  Slots >= Gr hold 0x7FFF and are taken back out of the area.
template <int GM>
__device__ __forceinline__ bool dp_viable16p(const DpParams &p, const DpShared<GM> &sh, uint64_t R2,
                                             const uint32_t (&bp)[GM / 2]) {
    constexpr int W = GM / 2;
    int64_t area = -(int64_t)(GM - p.Gr) * 0x7FFF;
#pragma unroll
    for (int w = 0; w < W; ++w) area += (bp[w] & 0xFFFFu) + (bp[w] >> 16);
    for (uint64_t m = R2; m; m &= m - 1) {
        const int i = __ffsll((long long)m) - 1;
        area += sh.minarea[i];
        uint32_t m2 = 0xFFFFFFFFu;
        if (p.has_release) {
            const uint32_t r2 = (uint32_t)sh.release[i] * 0x10001u;
#pragma unroll
            for (int w = 0; w < W; ++w) m2 = __viaddmin_u16x2(__vmaxu2(bp[w], r2), sh.dgp[i][w], m2);
        } else {
#pragma unroll
            for (int w = 0; w < W; ++w) m2 = __viaddmin_u16x2(bp[w], sh.dgp[i][w], m2);
        }
        if ((int32_t)min(m2 & 0xFFFFu, m2 >> 16) > p.T) return false;
    }
    return area <= (int64_t)p.T * p.Gr;
}

// dp_rank of a packed state
template <int GM>
__device__ __forceinline__ uint64_t dp_rank16(const DpParams &p, const uint32_t (&bp)[GM / 2]) {
    const int K = p.Gr + 1;
    uint64_t r = 0;
#pragma unroll
    for (int i = 0; i < GM; ++i)
        if (i < p.Gr) {
            const int32_t v = (int32_t)((bp[i / 2] >> (16 * (i & 1))) & 0xFFFFu);
            r += __ldg(&p.binom[(v + i) * K + (i + 1)]);
        }
    return r;
}

template <int GM>
__global__ void __launch_bounds__(kDpThreads) k_dp_expand(const __grid_constant__ DpParams p, int L) {
    // Level L -> L + 1, sized on the device: the level's state count and offset are read from
    // lvl_cnt / lvl_base (written by the previous level's launch), so the host queues every
    // level without a read-back in between.  A fixed grid strides over the level's
    // (state, job still to place) pairs -- every state has J - L such jobs.  Options are taken
    // in block-wide rounds (round r = every thread's r-th usable option) so that the states a
    // round appends are claimed with ONE atomicAdd per block on the level's counter.
    __shared__ uint32_t warp_new[2][kDpThreads / 32];  // double-buffered by round parity
    __shared__ unsigned long long block_base[2];
    __shared__ unsigned int stop;
    __shared__ DpShared<GM> sh;
    // per thread: the parent's packed slots (GM/2 words), then GM/2 + 1 words of 0x7FFF pairs --
    // the shift by the option's gang is one PRMT of two column words (k_cand's scheme)
    __shared__ uint32_t scol[(GM + 1) * kDpThreads];
    constexpr int H = GM / 2;
    uint32_t *col = scol + threadIdx.x;
    int par = 0;
    if (threadIdx.x == 0) stop = *reinterpret_cast<volatile unsigned int *>(p.overflow);
    __syncthreads();
    if (stop) return;                                  // an earlier level ran out of budget
    dp_stage<GM>(p, sh);
    __syncthreads();
    const uint64_t n_in = p.lvl_cnt[L], in_base = p.lvl_base[L];
    const uint64_t out_base = in_base + n_in;
    if (blockIdx.x == 0 && threadIdx.x == 0) p.lvl_base[L + 1] = out_base;
    const uint64_t out_cap = p.max_states - out_base;
    const uint64_t *in_R = p.all_R + in_base;
    const uint16_t *in_A = p.all_A + in_base * p.Gr;
    uint64_t *out_R = p.all_R + out_base;
    uint16_t *out_A = p.all_A + out_base * p.Gr;
    unsigned long long *count = p.lvl_cnt + L + 1;
    const int nrem = p.J - L;
    const uint64_t total = n_in * (uint64_t)nrem;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t t0 = (uint64_t)blockIdx.x * kDpThreads; t0 < total; t0 += (uint64_t)gridDim.x * kDpThreads) {
        // out of budget (this level or a probe limit): stop striding at once -- the hash set
        // keeps filling with states that can no longer be appended, and probes lengthen
        if (t0 != (uint64_t)blockIdx.x * kDpThreads) {
            if (threadIdx.x == 0) stop = *reinterpret_cast<volatile unsigned int *>(p.overflow);
            __syncthreads();
            if (stop) return;
        }
        const uint64_t tid = t0 + threadIdx.x;
        int j = 0, nq = 0;
        uint64_t R2 = 0;
        uint32_t ap[H], bp[H];
        if (tid < total) {
            const uint64_t s = tid / (uint64_t)nrem;
            const int kk = (int)(tid - s * (uint64_t)nrem);
            const uint64_t R = in_R[s];
            const uint32_t Rlo = (uint32_t)R, Rhi = (uint32_t)(R >> 32);
            const int nlo = __popc(Rlo);
            j = kk < nlo ? (int)__fns(Rlo, 0, kk + 1) : 32 + (int)__fns(Rhi, 0, kk - nlo + 1);
            R2 = R & ~(1ull << j);
            nq = sh.ucnt[j];
#pragma unroll
            for (int w = 0; w < H; ++w) {
                const uint32_t lo = 2 * w < p.Gr ? (uint32_t)in_A[s * p.Gr + 2 * w] : 0x7FFFu;
                const uint32_t hi = 2 * w + 1 < p.Gr ? (uint32_t)in_A[s * p.Gr + 2 * w + 1] : 0x7FFFu;
                ap[w] = lo | (hi << 16);
                col[w * kDpThreads] = ap[w];
                col[(H + w) * kDpThreads] = 0x7FFF7FFFu;
            }
            col[GM * kDpThreads] = 0x7FFF7FFFu;
        }
        for (int r = 0; r < p.umax; ++r) {
            bool fresh = false;
            if (r < nq) {
                const int q = sh.ubase[j] + r;
                const int g = sh.ug[q], gm = g - 1;
                const uint32_t selt = 0x4410u + (uint32_t)(gm & 1) * 0x22u;
                const int32_t t = max((int32_t)__byte_perm(col[(gm >> 1) * kDpThreads], 0u, selt), sh.release[j]);
                const int32_t e = t + (int32_t)sh.ud[q];
                bool ok = e <= p.T;
                if (ok) {
                    // b[i] = max(a[i], min(a[i + g], e)); slots past Gr stay 0x7FFF (> any e <= T)
                    const uint32_t e2 = (uint32_t)e * 0x10001u;
                    const uint32_t sel = (g & 1) ? 0x5432u : 0x3210u;
                    const uint32_t *src = col + (g >> 1) * kDpThreads;
#pragma unroll
                    for (int k = 0; k < H; ++k)
                        bp[k] = __vmaxu2(ap[k], __vminu2(__byte_perm(src[k * kDpThreads], src[(k + 1) * kDpThreads], sel), e2));
                    ok = dp_viable16p<GM>(p, sh, R2, bp);
                }
                if (ok) {
                    const uint64_t key = R2 * p.cnum + dp_rank16<GM>(p, bp);
                    uint64_t h = (key * kGolden) >> (64 - p.cap_log2);
                    for (int probe = 0;; ++probe) {
                        if (probe > p.max_probe) { atomicExch(p.overflow, (unsigned)L + 1u); break; }
                        const unsigned long long old = atomicCAS(
                            reinterpret_cast<unsigned long long *>(&p.table[h]), (unsigned long long)kDpEmpty,
                            (unsigned long long)key);
                        if (old == kDpEmpty) { fresh = true; break; }   // first time this state is reached
                        if (old == key) break;                          // already in the level
                        h = (h + 1) & p.cap_mask;
                    }
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, fresh);
            uint32_t *wn = warp_new[par];
            if (lane == 0) wn[warp] = __popc(bal);
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t tot = 0;
#pragma unroll
                for (int w = 0; w < kDpThreads / 32; ++w) { const uint32_t c = wn[w]; wn[w] = tot; tot += c; }
                block_base[par] = tot ? atomicAdd(count, (unsigned long long)tot) : 0ull;
            }
            __syncthreads();
            // (the next round writes the other buffer; the one after that only once every
            // thread has passed the next round's first barrier, i.e. finished reading this one)
            if (fresh) {
                const unsigned long long idx = block_base[par] + wn[warp] + __popc(bal & ((1u << lane) - 1u));
                if (idx >= out_cap) {
                    atomicExch(p.overflow, (unsigned)L + 1u);
                } else {
                    out_R[idx] = R2;
#pragma unroll
                    for (int i = 0; i < GM; ++i)
                        if (i < p.Gr) out_A[idx * p.Gr + i] = (uint16_t)(bp[i / 2] >> (16 * (i & 1)));
                }
            }
            par ^= 1;
        }
    }
}

// smallest key among a level's states (the final state of the reconstruction)
__global__ void k_dp_min_key(const __grid_constant__ DpParams p) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= p.n_in) return;
    int32_t a[32];
    for (int i = 0; i < p.Gr; ++i) a[i] = p.in_A[s * p.Gr + i];
    atomicMin(p.min_key, (unsigned long long)(p.in_R[s] * p.cnum + dp_rank(p, a)));
}

// smallest key among the level's states that reach (child_R, child_A) with one placement
template <int GM>
__global__ void __launch_bounds__(kDpThreads) k_dp_parent(const __grid_constant__ DpParams p) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= p.n_in) return;
    const uint64_t R = p.in_R[s];
    const uint64_t diff = R ^ p.child_R;
    if ((R & p.child_R) != p.child_R || __popcll(diff) != 1) return;
    const int j = __ffsll((long long)diff) - 1;
    int32_t a[GM], b[GM];
#pragma unroll
    for (int i = 0; i < GM; ++i) a[i] = i < p.Gr ? (int32_t)p.in_A[s * p.Gr + i] : 0x7fffffff;
    for (int q = p.ubase[j]; q < p.ubase[j] + p.ucnt[j]; ++q) {
        dp_place<GM>(a, p.Gr, p.ug[q], p.ud[q], p.release[j], b);
        bool same = true;
#pragma unroll
        for (int i = 0; i < GM; ++i)
            if (i < p.Gr && b[i] != (int32_t)p.child_A[i]) same = false;
        if (same) {
            atomicMin(p.min_key, (unsigned long long)(R * p.cnum + dp_rank(p, a)));
            return;
        }
    }
}

// ---------------------------------------------------------------------------------- host side
struct DpPlan {
    DpParams p{};
    std::vector<int32_t> uorig;       // usable option q -> option digit of its job
    std::vector<int32_t> a0;          // initial sorted free times (Gr)
    std::vector<uint64_t> binom;      // host copy of the table
    int status = -1;                  // SAT_DP_* when decided without a search
    size_t binom_bytes = 0, table_bytes = 0, R_bytes = 0, A_bytes = 0;
    uint64_t cap = 0;
};

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// usable options, bound tables, key encoding and workspace layout for (p, T, max_states)
static int dp_prepare(const sat_problem_t *pr, int32_t T, uint64_t max_states, DpPlan &d) {
    if (pr->N != 1 || pr->time_mode != SAT_TIME_GRID_I32) return SAT_ERR_UNSUPPORTED;
    if (pr->J > kDpMaxJ || max_states < 1) return SAT_ERR_INVALID;
    const int J = pr->J, Gr = pr->node_gpus[0];
    if (Gr > 32 || T < 0 || T > 30000) return SAT_ERR_UNSUPPORTED;
    DpParams &p = d.p;
    p.J = J; p.Gr = Gr; p.T = T;
    d.a0.assign(Gr, 0);
    int64_t sum0 = 0;
    for (int i = 0; i < Gr; ++i) {
        d.a0[i] = pr->init_free_i32 ? pr->init_free_i32[i] : 0;
        sum0 += d.a0[i];
    }
    if (!std::is_sorted(d.a0.begin(), d.a0.end())) return SAT_ERR_INVALID;
    if (d.a0[Gr - 1] > T) { d.status = SAT_DP_INFEASIBLE; return SAT_OK; }
    // least area per job over the options that can end by T at all, then the area slack
    int64_t need = sum0;
    std::vector<int64_t> least(J);
    for (int j = 0; j < J; ++j) {
        const int32_t rel = pr->release_i32 ? pr->release_i32[j] : 0;
        int64_t m = INT64_MAX;
        for (int o = 0; o < pr->radix[j]; ++o) {
            const int q = j * pr->Cmax + o;
            const int g = pr->gpus[q];
            const int32_t dd = pr->dur_i32[q];
            if (g > Gr || std::max(d.a0[g - 1], rel) + (int64_t)dd > T) continue;
            m = std::min<int64_t>(m, (int64_t)g * dd);
        }
        if (m == INT64_MAX) { d.status = SAT_DP_INFEASIBLE; return SAT_OK; }
        least[j] = m;
        need += m;
    }
    const int64_t slack = (int64_t)T * Gr - need;
    if (slack < 0) { d.status = SAT_DP_INFEASIBLE; return SAT_OK; }
    int q = 0;
    for (int j = 0; j < J; ++j) {
        const int32_t rel = pr->release_i32 ? pr->release_i32[j] : 0;
        p.release[j] = rel;
        p.ubase[j] = q;
        p.minarea[j] = (int32_t)least[j];
        for (int k = 0; k < 32; ++k) p.dg[j][k] = (int16_t)(T + 1);
        for (int o = 0; o < pr->radix[j]; ++o) {
            const int src = j * pr->Cmax + o;
            const int g = pr->gpus[src];
            const int32_t dd = pr->dur_i32[src];
            if (g > Gr || std::max(d.a0[g - 1], rel) + (int64_t)dd > T) continue;
            if ((int64_t)g * dd > least[j] + slack) continue;      // would overrun the area on its own
            if (q >= kDpMaxOpt) return SAT_ERR_TOO_LARGE;
            p.ug[q] = (uint8_t)g;
            p.ud[q] = (int16_t)dd;
            d.uorig.push_back(o);
            p.dg[j][g - 1] = (int16_t)std::min<int32_t>(p.dg[j][g - 1], dd);
            ++q;
        }
        p.ucnt[j] = q - p.ubase[j];
        for (int w = 0; w < 16; ++w) {
            const uint32_t lo = 2 * w < Gr ? (uint32_t)std::min<int32_t>(p.dg[j][2 * w], 0x7FFF) : 0x7FFFu;
            const uint32_t hi = 2 * w + 1 < Gr ? (uint32_t)std::min<int32_t>(p.dg[j][2 * w + 1], 0x7FFF) : 0x7FFFu;
            p.dgp[j][w] = lo | (hi << 16);
        }
        p.has_release |= rel != 0;
        p.umax = std::max(p.umax, p.ucnt[j]);
    }
    // exact key: R x C(T + Gr, Gr) + rank must stay below 2^63
    const int n_max = T + Gr;
    d.binom.assign((size_t)(n_max + 1) * (Gr + 1), 0);
    for (int n = 0; n <= n_max; ++n) {
        d.binom[(size_t)n * (Gr + 1)] = 1;
        for (int k = 1; k <= Gr && k <= n; ++k) {
            const unsigned __int128 v = (unsigned __int128)d.binom[(size_t)(n - 1) * (Gr + 1) + k - 1] +
                                        (k <= n - 1 ? d.binom[(size_t)(n - 1) * (Gr + 1) + k] : 0);
            if (v >> 62) return SAT_ERR_UNSUPPORTED;
            d.binom[(size_t)n * (Gr + 1) + k] = (uint64_t)v;
        }
    }
    p.cnum = d.binom[(size_t)n_max * (Gr + 1) + Gr];
    if ((unsigned __int128)p.cnum << J >= ((unsigned __int128)1 << 63)) return SAT_ERR_UNSUPPORTED;
    // workspace: binomials | hash set (>= 2x the states + slack, power of two) | R | A | counters
    uint64_t cap = 1;
    int lg = 0;
    while (cap < 2 * max_states + (1u << 16)) { cap <<= 1; ++lg; }
    d.cap = cap;
    p.cap_mask = cap - 1;
    p.cap_log2 = lg;
    p.max_probe = 1 << 14;
    d.binom_bytes = align256(d.binom.size() * sizeof(uint64_t));
    d.table_bytes = align256(cap * sizeof(uint64_t));
    d.R_bytes = align256(max_states * sizeof(uint64_t));
    d.A_bytes = align256(max_states * Gr * sizeof(uint16_t));
    return SAT_OK;
}

// level counters: [0, 8) scalars (min key, overflow), [8, 8 + J + 1) counts, then J + 2 bases
constexpr size_t kDpCtrBytes = (8 + 2 * (kDpMaxJ + 2)) * sizeof(unsigned long long);
static size_t dp_ws_bytes(const DpPlan &d) { return d.binom_bytes + d.table_bytes + d.R_bytes + d.A_bytes + kDpCtrBytes; }

template <int GM>
static int dp_launch_expand(const DpParams &p, int L, cudaStream_t s) {
    static int blocks = 0;                             // a full resident generation, once
    if (!blocks) {
        int dev = 0, sms = 0, per = 0;
        if (cudaGetDevice(&dev) || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_dp_expand<GM>, kDpThreads, 0))
            return SAT_ERR_CUDA;
        blocks = std::max(1, sms * per);
    }
    k_dp_expand<GM><<<blocks, kDpThreads, 0, s>>>(p, L);
    return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
}

template <int GM>
static int dp_launch_parent(const DpParams &p, cudaStream_t s) {
    const uint64_t blocks = (p.n_in + kDpThreads - 1) / kDpThreads;
    if (blocks == 0) return SAT_OK;
    k_dp_parent<GM><<<(unsigned)blocks, kDpThreads, 0, s>>>(p);
    return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
}

static int dp_expand(const DpParams &p, int L, cudaStream_t s) {
    if (p.Gr <= 8) return dp_launch_expand<8>(p, L, s);
    if (p.Gr <= 16) return dp_launch_expand<16>(p, L, s);
    return dp_launch_expand<32>(p, L, s);
}

static int dp_parent(const DpParams &p, cudaStream_t s) {
    if (p.Gr <= 8) return dp_launch_parent<8>(p, s);
    if (p.Gr <= 16) return dp_launch_parent<16>(p, s);
    return dp_launch_parent<32>(p, s);
}

// host: key -> (R, sorted free times)
static void dp_unrank(const DpPlan &d, uint64_t key, uint64_t *R, int32_t *a) {
    const int Gr = d.p.Gr, K = Gr + 1;
    *R = key / d.p.cnum;
    uint64_t r = key % d.p.cnum;
    int c = d.p.T + Gr - 1;
    for (int i = Gr - 1; i >= 0; --i) {
        while (c >= 0 && d.binom[(size_t)c * K + (i + 1)] > r) --c;
        r -= d.binom[(size_t)c * K + (i + 1)];
        a[i] = c - i;
        --c;
    }
}

static int32_t dp_host_place(const DpPlan &d, const int32_t *a, int q, int rel, int32_t *b) {
    const int Gr = d.p.Gr, g = d.p.ug[q];
    const int32_t e = std::max(a[g - 1], rel) + d.p.ud[q];
    for (int i = 0; i < Gr; ++i) b[i] = std::max(a[i], std::min(i + g < Gr ? a[i + g] : INT32_MAX, e));
    return e;
}

// ------------------------------------------------------------------------------------------
// Wide states (several nodes, or keys beyond 63 bits): a PROVER.  The state is R plus every
// node's sorted free-time vector; the key R x prod_n C(T + G_n, G_n) + ranks is exact in 128
// bits, kept in a hash set of 16-byte slots claimed with a 128-bit atomicCAS
// (ATOMG.E.CAS.128).  Interchangeable nodes (same GPU count and memory, same option
// eligibility and durations) are canonicalised -- their vectors sorted by rank -- and a job
// whose earliest finish ties on several nodes is placed on EACH of them: the list scheduler
// picks the lowest label among tied nodes, and labels are what canonicalisation forgets, so
// the level sets cover (a superset of) every candidate's states.  An empty level therefore
// still proves that no candidate reaches T; a non-empty last level proves nothing (no
// candidate is rebuilt: status FEASIBLE, makespan -1).
// ------------------------------------------------------------------------------------------
constexpr int kDpWideMaxN = 8;
constexpr int kDpWideSlots = 32;

struct DpWideParams {
    int32_t J, N, T, Gtot;
    int32_t node_off[kDpWideMaxN], node_g[kDpWideMaxN], node_grp[kDpWideMaxN];
    uint64_t cnum[kDpWideMaxN];             // C(T + G_n, G_n)
    int32_t ubase[kDpMaxJ], ucnt[kDpMaxJ], release[kDpMaxJ], minarea[kDpMaxJ];
    int32_t Kb;                             // binomial table row width (max G_n + 1)
    int32_t nrem;                           // jobs still to place in the level being expanded
    int32_t exact;                          // 1: labelled nodes, the list scheduler's own node choice
    const uint8_t *ue;                      // [n_usable] every node the option is eligible on (exact)
    const int16_t *uf;                      // [n_usable][N] its duration there (exact)
    const uint64_t *binom;                  // [(T + maxG + 1)][Kb]
    const uint8_t *ug;                      // [n_usable] gang size
    const uint8_t *um;                      // [n_usable] node eligibility bits
    const int16_t *ud;                      // [n_usable][N] duration per node
    const int16_t *dg;                      // [J][N][32] least usable duration at gang k+1 (T+1: none)
    const uint32_t *dgp;                    // [J][16] the same per global slot (node_off[n] + k), two
                                            // 16-bit slots per word, 0x7fff past Gtot
    unsigned __int128 *table;
    uint64_t cap_mask;
    int32_t cap_log2, max_probe;
    const uint64_t *in_R;
    const uint16_t *in_A;                   // [n_in][Gtot]
    uint64_t n_in;
    uint64_t *out_R;
    uint16_t *out_A;
    uint64_t out_cap;
    unsigned long long *count;
    unsigned int *overflow;
    // exact mode, candidate rebuild (k_dpw_pick_state)
    uint64_t child_R;
    uint16_t child_A[kDpWideSlots];
    unsigned long long *pick_hi, *pick_lo;
    uint64_t *pick_R;
    uint16_t *pick_A;
};

__device__ __forceinline__ unsigned __int128 cas128(unsigned __int128 *addr, unsigned __int128 cmp,
                                                    unsigned __int128 val) {
    uint64_t o0, o1;
    const uint64_t c0 = (uint64_t)cmp, c1 = (uint64_t)(cmp >> 64);
    const uint64_t v0 = (uint64_t)val, v1 = (uint64_t)(val >> 64);
    asm volatile("{\n\t.reg .b128 c, v, d;\n\t"
                 "mov.b128 c, {%2, %3};\n\t"
                 "mov.b128 v, {%4, %5};\n\t"
                 "atom.global.cas.b128 d, [%6], c, v;\n\t"
                 "mov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(o0), "=l"(o1)
                 : "l"(c0), "l"(c1), "l"(v0), "l"(v1), "l"(addr)
                 : "memory");
    return ((unsigned __int128)o1 << 64) | o0;
}

__device__ __forceinline__ uint64_t dpw_rank(const DpWideParams &p, const int32_t *v, int g, const uint64_t *bt) {
    uint64_t r = 0;
    for (int i = 0; i < g; ++i) r += bt[(v[i] + i) * p.Kb + (i + 1)];
    return r;
}

// canonical key of a full state (vectors are permuted in place into canonical node order)
__device__ __forceinline__ unsigned __int128 dpw_key(const DpWideParams &p, uint64_t R, int32_t *a,
                                                     const uint64_t *bt) {
    uint64_t rk[kDpWideMaxN];
    for (int n = 0; n < p.N; ++n) rk[n] = dpw_rank(p, a + p.node_off[n], p.node_g[n], bt);
    // sort interchangeable nodes by rank (insertion sort over the <= 8 nodes, within groups)
    for (int n = 1; n < p.N; ++n)
        for (int m = n; m > 0 && p.node_grp[m - 1] == p.node_grp[m] && rk[m - 1] > rk[m]; --m) {
            const uint64_t t = rk[m]; rk[m] = rk[m - 1]; rk[m - 1] = t;
            int32_t *x = a + p.node_off[m - 1], *y = a + p.node_off[m];
            for (int i = 0; i < p.node_g[m]; ++i) { const int32_t z = x[i]; x[i] = y[i]; y[i] = z; }
        }
    unsigned __int128 key = R;
    for (int n = 0; n < p.N; ++n) key = key * p.cnum[n] + rk[n];
    return key;
}

// Viability of a child state b (R2 = its jobs still to place): every such job must be able to end
// by T -- min over nodes and gangs k of max(b[slot k-1], release) + least duration at gang k --
// and the GPU time left must hold their least areas.  The per-job minimum runs on 16-bit pairs:
// b packed once per child, 16 VIADDMNMX.U16x2 per job against its packed row `sdgp` (staged in
// shared memory); every value is <= T + 1 <= 30 001, so sums stay below 2^16.  b holds
// kDpWideSlots entries, zero past Gtot (the packing needs no per-slot bound test).
__device__ __forceinline__ bool dpw_viable(const DpWideParams &p, uint64_t R2, const int32_t *b,
                                           const uint32_t *sdgp) {
    uint32_t area = 0;                         // <= 32 slots x 30 000
    uint32_t bp[16];
#pragma unroll
    for (int w = 0; w < 16; ++w) {
        const uint32_t lo = (uint32_t)b[2 * w], hi = (uint32_t)b[2 * w + 1];
        area += lo + hi;
        bp[w] = lo | (hi << 16);
    }
    for (uint64_t m = R2; m; m &= m - 1) {
        const int i = __ffsll((long long)m) - 1;
        area += p.minarea[i];
        const uint32_t *dj = sdgp + i * 16;
        uint32_t acc = 0xFFFFFFFFu;
        const int32_t rel = p.release[i];
        if (rel == 0) {
#pragma unroll
            for (int w = 0; w < 16; ++w) acc = __viaddmin_u16x2(bp[w], dj[w], acc);
        } else {
            const uint32_t r2 = (uint32_t)rel * 0x10001u;
#pragma unroll
            for (int w = 0; w < 16; ++w) acc = __viaddmin_u16x2(__vmaxu2(bp[w], r2), dj[w], acc);
        }
        if ((int32_t)min(acc & 0xFFFFu, acc >> 16) > p.T) return false;
    }
    return (int64_t)area <= (int64_t)p.T * p.Gtot;
}

// exact mode: node the list scheduler gives usable option q of job j from state a (earliest end
// over every eligible node, lowest label on ties; -1: none)
__device__ __forceinline__ int dpw_pick(const DpWideParams &p, const int32_t *a, int q, int j) {
    const int g = p.ug[q];
    const uint32_t em = p.ue[q];
    int32_t best = 0x7fffffff;
    int bn = -1;
    for (int n = 0; n < p.N; ++n) {
        if (!((em >> n) & 1u) || g > p.node_g[n]) continue;
        const int32_t e = max(a[p.node_off[n] + g - 1], p.release[j]) + (int32_t)p.uf[q * p.N + n];
        if (e < best) { best = e; bn = n; }
    }
    return bn;
}

// the state after placing usable option q of job j on node n (exact-mode durations); returns the end
__device__ __forceinline__ int32_t dpw_place(const DpWideParams &p, const int32_t *a, int q, int j, int n,
                                             int32_t *b) {
    const int g = p.ug[q];
    for (int i = 0; i < p.Gtot; ++i) b[i] = a[i];
    const int32_t *an = a + p.node_off[n];
    int32_t *bn = b + p.node_off[n];
    const int G = p.node_g[n];
    const int32_t e = max(an[g - 1], p.release[j]) + (int32_t)p.uf[q * p.N + n];
    for (int i = 0; i < G; ++i) bn[i] = max(an[i], min(i + g < G ? an[i + g] : 0x7fffffff, e));
    return e;
}

// claim the state's key in the hash set and append it to the level; false = out of budget
__device__ __forceinline__ bool dpw_insert(const DpWideParams &p, uint64_t R2, int32_t *b, const uint64_t *bt) {
    const unsigned __int128 key = dpw_key(p, R2, b, bt);
    const uint64_t hh = ((uint64_t)key ^ (uint64_t)(key >> 64) * 0xBF58476D1CE4E5B9ull) * kGolden;
    uint64_t h = hh >> (64 - p.cap_log2);
    const unsigned __int128 EMPTY = ~(unsigned __int128)0;
    for (int probe = 0;; ++probe) {
        if (probe > p.max_probe) { atomicOr(p.overflow, 1u); return false; }
        const unsigned __int128 old = cas128(&p.table[h], EMPTY, key);
        if (old == EMPTY) {
            const unsigned long long idx = atomicAdd(p.count, 1ull);
            if (idx >= p.out_cap) { atomicOr(p.overflow, 1u); return false; }
            p.out_R[idx] = R2;
            for (int i = 0; i < p.Gtot; ++i) p.out_A[idx * p.Gtot + i] = (uint16_t)b[i];
            return true;
        }
        if (old == key) return true;
        h = (h + 1) & p.cap_mask;
    }
}

__global__ void __launch_bounds__(kDpThreads, 6) k_dp_expand_wide(const __grid_constant__ DpWideParams p) {
    __shared__ uint32_t sdgp[kDpMaxJ * 16];
    for (int i = threadIdx.x; i < p.J * 16; i += blockDim.x) sdgp[i] = p.dgp[i];
    __syncthreads();
    const uint64_t *bt = p.binom;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= p.n_in * (uint64_t)p.nrem) return;
    if (*reinterpret_cast<volatile unsigned int *>(p.overflow)) return;
    const uint64_t s = tid / (uint64_t)p.nrem;                  // (state, k-th job still to place)
    const int kk = (int)(tid - s * (uint64_t)p.nrem);
    const uint64_t R = p.in_R[s];
    const uint32_t Rlo = (uint32_t)R, Rhi = (uint32_t)(R >> 32);
    const int nlo = __popc(Rlo);
    const int j = kk < nlo ? (int)__fns(Rlo, 0, kk + 1) : 32 + (int)__fns(Rhi, 0, kk - nlo + 1);
    const uint64_t R2 = R & ~(1ull << j);
    int32_t a[kDpWideSlots], b[kDpWideSlots];
#pragma unroll
    for (int i = 0; i < kDpWideSlots; ++i) {           // slots past Gtot stay 0 (dpw_viable packs all 32)
        a[i] = i < p.Gtot ? (int32_t)p.in_A[s * p.Gtot + i] : 0;
        b[i] = 0;
    }
    for (int q = p.ubase[j]; q < p.ubase[j] + p.ucnt[j]; ++q) {
        const int g = p.ug[q];
        const uint32_t mask = p.um[q];
        if (p.exact) {
            // the list scheduler's node: earliest end over EVERY eligible node, lowest label on
            // ties; a node outside the usable set there means the candidate cannot reach T
            const int bn = dpw_pick(p, a, q, j);
            if (bn < 0 || !((mask >> bn) & 1u)) continue;
            const int32_t e = dpw_place(p, a, q, j, bn, b);
            if (e > p.T || !dpw_viable(p, R2, b, sdgp)) continue;
            if (!dpw_insert(p, R2, b, bt)) return;
            continue;
        }
        int32_t best = 0x7fffffff;
        for (int n = 0; n < p.N; ++n)
            if ((mask >> n) & 1u && g <= p.node_g[n])
                best = min(best, max(a[p.node_off[n] + g - 1], p.release[j]) + (int32_t)p.ud[q * p.N + n]);
        if (best > p.T) continue;
        for (int n = 0; n < p.N; ++n) {                    // every node tying for the earliest finish
            if (!((mask >> n) & 1u) || g > p.node_g[n]) continue;
            const int32_t *an = a + p.node_off[n];
            if (max(an[g - 1], p.release[j]) + (int32_t)p.ud[q * p.N + n] != best) continue;
            for (int i = 0; i < p.Gtot; ++i) b[i] = a[i];
            int32_t *bn = b + p.node_off[n];
            const int G = p.node_g[n];
            for (int i = 0; i < G; ++i) bn[i] = max(an[i], min(i + g < G ? an[i + g] : 0x7fffffff, best));
            if (!dpw_viable(p, R2, b, sdgp)) continue;
            if (!dpw_insert(p, R2, b, bt)) return;
        }
    }
}

// Exact mode, backwards: the final state (mode 0: every state of the level) or the parents of
// (child_R, child_A) (mode 1: states of the previous level with a job j and a usable option whose
// exact placement gives the child) -- phase 0: min of the high key words, phase 1: min of the low
// words among those, phase 2: the state holding (min_hi, min_lo) writes itself out.  Keys are the
// labelled (uncanonicalised) exact keys, so the choice is deterministic.
__global__ void __launch_bounds__(kDpThreads) k_dpw_pick_state(const __grid_constant__ DpWideParams p, int mode,
                                                                 int phase) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int nrem = mode == 0 ? 1 : p.nrem;
    if (tid >= p.n_in * (uint64_t)nrem) return;
    const uint64_t s = tid / (uint64_t)nrem;
    const uint64_t R = p.in_R[s];
    int32_t a[kDpWideSlots], b[kDpWideSlots];
    for (int i = 0; i < p.Gtot; ++i) a[i] = p.in_A[s * p.Gtot + i];
    if (mode == 1) {
        const int kk = (int)(tid - s * (uint64_t)nrem);
        const uint32_t Rlo = (uint32_t)R, Rhi = (uint32_t)(R >> 32);
        const int nlo = __popc(Rlo);
        const int j = kk < nlo ? (int)__fns(Rlo, 0, kk + 1) : 32 + (int)__fns(Rhi, 0, kk - nlo + 1);
        if ((R & ~(1ull << j)) != p.child_R) return;
        bool hit = false;
        for (int q = p.ubase[j]; q < p.ubase[j] + p.ucnt[j] && !hit; ++q) {
            const int bn = dpw_pick(p, a, q, j);
            if (bn < 0 || !((p.um[q] >> bn) & 1u)) continue;
            dpw_place(p, a, q, j, bn, b);
            bool eq = true;
            for (int i = 0; i < p.Gtot; ++i) eq &= b[i] == (int32_t)p.child_A[i];
            hit = eq;
        }
        if (!hit) return;
    }
    const unsigned __int128 key = dpw_key(p, R, a, p.binom);   // exact mode: no canonical permutation
    const unsigned long long hi = (unsigned long long)(uint64_t)(key >> 64), lo = (unsigned long long)(uint64_t)key;
    if (phase == 0) {
        atomicMin(p.pick_hi, hi);
    } else if (phase == 1) {
        if (hi == *p.pick_hi) atomicMin(p.pick_lo, lo);
    } else if (hi == *p.pick_hi && lo == *p.pick_lo) {
        *p.pick_R = R;                                   // (equal states write equal values)
        for (int i = 0; i < p.Gtot; ++i) p.pick_A[i] = (uint16_t)a[i];
    }
}

// ------------------------------------------------------------------------------------------
// Wide expansion specialised on homogeneous nodes (N nodes of G GPUs, G even, N x G <= 32): the
// state lives in registers as N x G/2 words of 16-bit pairs; the shift by a thread's own gang is
// a read of its shared-memory column (node n at words n*G .. n*G+G/2-1, +inf words after it, one
// pad word at the end) with one PRMT per word -- the k_cand Multi16 scheme -- so no state array
// sits in local memory.  Same children, viability, canonical keys and appends as
// k_dp_expand_wide (the generic kernel keeps every other shape).
// ------------------------------------------------------------------------------------------
template <int N, int G>
__global__ void __launch_bounds__(kDpThreads) k_dpw_expand_h(const __grid_constant__ DpWideParams p) {
    constexpr int H = G / 2, W = N * H, CW = N * G + 1;     // words: per node, state, column
    constexpr bool LEAN = N * G >= 16;   // large states: the parent stays in the column only (registers)
    __shared__ uint32_t sdgp[kDpMaxJ * 16];
    extern __shared__ uint32_t scol[];                      // [CW][kDpThreads]
    for (int i = threadIdx.x; i < p.J * 16; i += blockDim.x) sdgp[i] = p.dgp[i];
    __syncthreads();
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= p.n_in * (uint64_t)p.nrem) return;
    if (*reinterpret_cast<volatile unsigned int *>(p.overflow)) return;
    const uint64_t s = tid / (uint64_t)p.nrem;
    const int kk = (int)(tid - s * (uint64_t)p.nrem);
    const uint64_t R = p.in_R[s];
    const uint32_t Rlo = (uint32_t)R, Rhi = (uint32_t)(R >> 32);
    const int nlo = __popc(Rlo);
    const int j = kk < nlo ? (int)__fns(Rlo, 0, kk + 1) : 32 + (int)__fns(Rhi, 0, kk - nlo + 1);
    const uint64_t R2 = R & ~(1ull << j);
    uint32_t ap[LEAN ? 1 : W];
    const uint32_t *inw = reinterpret_cast<const uint32_t *>(p.in_A + s * (uint64_t)(N * G));
    uint32_t *col = scol + threadIdx.x;
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
        for (int k = 0; k < H; ++k) {
            const uint32_t v = inw[n * H + k];
            if constexpr (!LEAN) ap[n * H + k] = v;
            col[(n * G + k) * kDpThreads] = v;
            col[(n * G + H + k) * kDpThreads] = 0xFFFFFFFFu;
        }
    col[(CW - 1) * kDpThreads] = 0xFFFFFFFFu;
    const int32_t rel = p.release[j];
    const int64_t cap = (int64_t)p.T * (N * G);
    const uint64_t *bt = p.binom;
    // child on node bn (gang g, end e) from the parent: packed, then viability, key, append
    auto child = [&](int g, int bn, int32_t e) -> bool {
        const uint32_t e2 = (uint32_t)e * 0x10001u;
        const uint32_t sel = (g & 1) ? 0x5432u : 0x3210u;
        const uint32_t *nb = col + bn * G * kDpThreads;
        const uint32_t *src = nb + (g >> 1) * kDpThreads;
        uint32_t nw[H];
#pragma unroll
        for (int k = 0; k < H; ++k)
            nw[k] = __vmaxu2(nb[k * kDpThreads],
                             __vminu2(__byte_perm(src[k * kDpThreads], src[(k + 1) * kDpThreads], sel), e2));
        uint32_t bp[W];
        uint32_t area = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if constexpr (LEAN)
                bp[w] = (w / H == bn) ? nw[w % H] : col[((w / H) * G + w % H) * kDpThreads];
            else
                bp[w] = (w / H == bn) ? nw[w % H] : ap[LEAN ? 0 : w];
            area += (bp[w] & 0xFFFFu) + (bp[w] >> 16);
        }
        // viability: every remaining job can end by T; their least areas fit
        for (uint64_t m = R2; m; m &= m - 1) {
            const int i = __ffsll((long long)m) - 1;
            area += p.minarea[i];
            const uint32_t *dj = sdgp + i * 16;
            uint32_t acc = 0xFFFFFFFFu;
            const int32_t ri = p.release[i];
            if (ri == 0) {
#pragma unroll
                for (int w = 0; w < W; ++w) acc = __viaddmin_u16x2(bp[w], dj[w], acc);
            } else {
                const uint32_t r2 = (uint32_t)ri * 0x10001u;
#pragma unroll
                for (int w = 0; w < W; ++w) acc = __viaddmin_u16x2(__vmaxu2(bp[w], r2), dj[w], acc);
            }
            if ((int32_t)min(acc & 0xFFFFu, acc >> 16) > p.T) return true;
        }
        if ((int64_t)area > cap) return true;
        // canonical key: ranks per node, interchangeable nodes sorted by rank (as dpw_key)
        uint64_t rk[N];
#pragma unroll
        for (int n = 0; n < N; ++n) {
            uint64_t r = 0;
#pragma unroll
            for (int k = 0; k < G; ++k) {
                const int32_t v = (int32_t)((bp[n * H + k / 2] >> (16 * (k & 1))) & 0xFFFFu);
                r += __ldg(&bt[(v + k) * p.Kb + (k + 1)]);
            }
            rk[n] = r;
        }
#pragma unroll
        for (int n = 1; n < N; ++n)
#pragma unroll
            for (int m = n; m > 0; --m) {
                const bool sw = p.node_grp[m - 1] == p.node_grp[m] && rk[m - 1] > rk[m];
                const uint64_t t0 = rk[m - 1], t1 = rk[m];
                rk[m - 1] = sw ? t1 : t0;
                rk[m] = sw ? t0 : t1;
#pragma unroll
                for (int k = 0; k < H; ++k) {
                    const uint32_t x = bp[(m - 1) * H + k], y = bp[m * H + k];
                    bp[(m - 1) * H + k] = sw ? y : x;
                    bp[m * H + k] = sw ? x : y;
                }
            }
        unsigned __int128 key = R2;
#pragma unroll
        for (int n = 0; n < N; ++n) key = key * p.cnum[n] + rk[n];
        const uint64_t hh = ((uint64_t)key ^ (uint64_t)(key >> 64) * 0xBF58476D1CE4E5B9ull) * kGolden;
        uint64_t h = hh >> (64 - p.cap_log2);
        const unsigned __int128 EMPTY = ~(unsigned __int128)0;
        for (int probe = 0;; ++probe) {
            if (probe > p.max_probe) { atomicOr(p.overflow, 1u); return false; }
            const unsigned __int128 old = cas128(&p.table[h], EMPTY, key);
            if (old == EMPTY) {
                const unsigned long long idx = atomicAdd(p.count, 1ull);
                if (idx >= p.out_cap) { atomicOr(p.overflow, 1u); return false; }
                p.out_R[idx] = R2;
                uint32_t *ow = reinterpret_cast<uint32_t *>(p.out_A + idx * (uint64_t)(N * G));
#pragma unroll
                for (int w = 0; w < W; ++w) ow[w] = bp[w];
                return true;
            }
            if (old == key) return true;
            h = (h + 1) & p.cap_mask;
        }
    };
    for (int q = p.ubase[j]; q < p.ubase[j] + p.ucnt[j]; ++q) {
        const int g = p.ug[q];
        const uint32_t mask = p.um[q];
        const int gm = g - 1;
        const uint32_t selt = 0x4410u + (uint32_t)(gm & 1) * 0x22u;
        int32_t t[N];
#pragma unroll
        for (int n = 0; n < N; ++n)
            t[n] = max((int32_t)__byte_perm(col[(n * G + (gm >> 1)) * kDpThreads], 0u, selt), rel);
        if (p.exact) {
            const uint32_t em = p.ue[q];
            int32_t best = 0x7fffffff;
            int bn = -1;
#pragma unroll
            for (int n = 0; n < N; ++n) {
                const int32_t e = t[n] + (int32_t)p.uf[q * N + n];
                if (((em >> n) & 1u) && e < best) { best = e; bn = n; }
            }
            if (bn < 0 || !((mask >> bn) & 1u) || best > p.T) continue;
            if (!child(g, bn, best)) return;
            continue;
        }
        int32_t best = 0x7fffffff;
#pragma unroll
        for (int n = 0; n < N; ++n)
            if ((mask >> n) & 1u) best = min(best, t[n] + (int32_t)p.ud[q * N + n]);
        if (best > p.T) continue;
#pragma unroll
        for (int n = 0; n < N; ++n) {                       // every node tying for the earliest finish
            if (!((mask >> n) & 1u) || t[n] + (int32_t)p.ud[q * N + n] != best) continue;
            if (!child(g, n, best)) return;
        }
    }
}

// launch of one wide level: the homogeneous specialisation when the shape has one
static int dpw_launch_level(const DpWideParams &p, unsigned blocks, cudaStream_t s) {
    bool homog = p.Gtot == p.N * p.node_g[0];
    for (int n = 1; n < p.N; ++n) homog &= p.node_g[n] == p.node_g[0];
    const int G = p.node_g[0];
    const size_t smem = (size_t)(p.N * G + 1) * kDpThreads * 4;
#define SAT_DPW(NN, GG)                                                                   \
    if (homog && p.N == NN && G == GG) {                                                  \
        k_dpw_expand_h<NN, GG><<<blocks, kDpThreads, smem, s>>>(p);                      \
        return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;                 \
    }
    SAT_DPW(2, 4) SAT_DPW(3, 4) SAT_DPW(4, 4) SAT_DPW(2, 8) SAT_DPW(3, 8) SAT_DPW(4, 8)
#undef SAT_DPW
    k_dp_expand_wide<<<blocks, kDpThreads, 0, s>>>(p);
    return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
}

struct DpWidePlan {
    DpWideParams p{};
    std::vector<uint8_t> ug, um, ue;
    std::vector<int16_t> ud, dg, uf;
    std::vector<int> uorig, ujob;           // original option digit / job of each usable option
    std::vector<uint32_t> dgp;              // [J][16] packed least durations per global slot
    std::vector<uint64_t> binom;
    std::vector<uint16_t> a0;
    int status = -1;
    size_t binom_bytes = 0, aux_bytes = 0, table_bytes = 0, R_bytes = 0, A_bytes = 0;
    uint64_t cap = 0;
};

static int dpw_prepare(const sat_problem_t *pr, int32_t T, uint64_t max_states, DpWidePlan &d, bool exact = false) {
    if (pr->time_mode != SAT_TIME_GRID_I32) return SAT_ERR_UNSUPPORTED;
    if (pr->J > kDpMaxJ || max_states < 1) return SAT_ERR_INVALID;
    const int J = pr->J, N = pr->N;
    if (N > kDpWideMaxN || T < 0 || T > 30000) return SAT_ERR_UNSUPPORTED;
    DpWideParams &p = d.p;
    p.J = J; p.N = N; p.T = T;
    p.exact = exact ? 1 : 0;
    int off = 0, gmax = 1;
    for (int n = 0; n < N; ++n) {
        p.node_off[n] = off;
        p.node_g[n] = pr->node_gpus[n];
        off += pr->node_gpus[n];
        gmax = std::max(gmax, (int)pr->node_gpus[n]);
    }
    if (off > kDpWideSlots) return SAT_ERR_UNSUPPORTED;
    p.Gtot = off;
    // initial state: each node's initial free times (ascending per node)
    d.a0.assign(off, 0);
    int64_t sum0 = 0;
    for (int n = 0; n < N; ++n)
        for (int i = 0; i < p.node_g[n]; ++i) {
            const int32_t v = pr->init_free_i32 ? pr->init_free_i32[n * pr->G + i] : 0;
            if (v > T) { d.status = SAT_DP_INFEASIBLE; return SAT_OK; }
            if (i > 0 && v < (int32_t)d.a0[p.node_off[n] + i - 1]) return SAT_ERR_INVALID;
            d.a0[p.node_off[n] + i] = (uint16_t)v;
            sum0 += v;
        }
    const uint32_t all = N >= 32 ? ~0u : ((1u << N) - 1u);
    auto dur = [&](int j, int o, int n) { return pr->dur_i32[(j * pr->Cmax + o) * N + n]; };
    auto elig = [&](int j, int o, int n) {
        const uint32_t m = pr->node_mask ? pr->node_mask[j * pr->Cmax + o] & all : all;
        return ((m >> n) & 1u) && pr->gpus[j * pr->Cmax + o] <= p.node_g[n];
    };
    auto can_end = [&](int j, int o, int n, int32_t rel) {
        const int g = pr->gpus[j * pr->Cmax + o];
        return elig(j, o, n) && std::max<int64_t>(d.a0[p.node_off[n] + g - 1], rel) + dur(j, o, n) <= T;
    };
    int64_t need = sum0;
    std::vector<int64_t> least(J);
    for (int j = 0; j < J; ++j) {
        const int32_t rel = pr->release_i32 ? pr->release_i32[j] : 0;
        int64_t m = INT64_MAX;
        for (int o = 0; o < pr->radix[j]; ++o)
            for (int n = 0; n < N; ++n)
                if (can_end(j, o, n, rel)) m = std::min<int64_t>(m, (int64_t)pr->gpus[j * pr->Cmax + o] * dur(j, o, n));
        if (m == INT64_MAX) { d.status = SAT_DP_INFEASIBLE; return SAT_OK; }
        least[j] = m;
        need += m;
    }
    const int64_t slack = (int64_t)T * off - need;
    if (slack < 0) { d.status = SAT_DP_INFEASIBLE; return SAT_OK; }
    d.dg.assign((size_t)J * N * 32, (int16_t)(T + 1));
    int q = 0;
    for (int j = 0; j < J; ++j) {
        const int32_t rel = pr->release_i32 ? pr->release_i32[j] : 0;
        p.release[j] = rel;
        p.minarea[j] = (int32_t)least[j];
        p.ubase[j] = q;
        for (int o = 0; o < pr->radix[j]; ++o) {
            const int g = pr->gpus[j * pr->Cmax + o];
            uint8_t m = 0;
            for (int n = 0; n < N; ++n)
                if (can_end(j, o, n, rel) && (int64_t)g * dur(j, o, n) <= least[j] + slack) m |= (uint8_t)(1u << n);
            if (!m) continue;
            d.ug.push_back((uint8_t)g);
            d.um.push_back(m);
            d.uorig.push_back(o);
            d.ujob.push_back(j);
            uint8_t em = 0;                       // exact mode: every eligible node and its duration
            for (int n = 0; n < N; ++n) {
                if (elig(j, o, n)) em |= (uint8_t)(1u << n);
                d.uf.push_back((int16_t)(elig(j, o, n) ? std::min<int32_t>(dur(j, o, n), 0x7fff) : 0x7fff));
            }
            d.ue.push_back(em);
            for (int n = 0; n < N; ++n) {
                const int32_t dd = ((m >> n) & 1u) ? dur(j, o, n) : T + 1;
                d.ud.push_back((int16_t)dd);
                if ((m >> n) & 1u) {
                    int16_t &slot = d.dg[((size_t)j * N + n) * 32 + g - 1];
                    slot = (int16_t)std::min<int32_t>(slot, dd);
                }
            }
            ++q;
        }
        p.ucnt[j] = q - p.ubase[j];
    }
    // interchangeable nodes: same size and, for every usable option, the same eligibility
    // and duration
    for (int n = 0; n < N; ++n) {
        p.node_grp[n] = n;
        if (exact) continue;                  // exact mode keeps node labels (no canonical order)
        for (int m = 0; m < n; ++m) {
            if (p.node_grp[m] != m || p.node_g[m] != p.node_g[n]) continue;
            bool same = true;
            for (int qq = 0; qq < q && same; ++qq)
                same = ((d.um[qq] >> m) & 1u) == ((d.um[qq] >> n) & 1u) && d.ud[qq * N + m] == d.ud[qq * N + n];
            if (same) { p.node_grp[n] = m; break; }
        }
    }
    // canonical node order: group members adjacent (stable by first member); rebuild the
    // per-node tables in that order
    std::vector<int> ord(N);
    for (int n = 0; n < N; ++n) ord[n] = n;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return p.node_grp[x] < p.node_grp[y]; });
    {
        DpWideParams p2 = p;
        std::vector<uint8_t> um2(d.um.size()), ue2(d.ue.size());
        std::vector<int16_t> ud2(d.ud.size()), dg2(d.dg.size()), uf2(d.uf.size());
        std::vector<uint16_t> a02(off);
        int o2 = 0;
        for (int k = 0; k < N; ++k) {
            const int n = ord[k];
            p2.node_g[k] = p.node_g[n];
            p2.node_grp[k] = p.node_grp[n];
            p2.node_off[k] = o2;
            for (int i = 0; i < p.node_g[n]; ++i) a02[o2 + i] = d.a0[p.node_off[n] + i];
            o2 += p.node_g[n];
        }
        for (size_t qq = 0; qq < d.um.size(); ++qq) {
            uint8_t m2 = 0, e2 = 0;
            for (int k = 0; k < N; ++k) {
                if ((d.um[qq] >> ord[k]) & 1u) m2 |= (uint8_t)(1u << k);
                if ((d.ue[qq] >> ord[k]) & 1u) e2 |= (uint8_t)(1u << k);
                ud2[qq * N + k] = d.ud[qq * N + ord[k]];
                uf2[qq * N + k] = d.uf[qq * N + ord[k]];
            }
            um2[qq] = m2;
            ue2[qq] = e2;
        }
        for (int j = 0; j < J; ++j)
            for (int k = 0; k < N; ++k)
                for (int g = 0; g < 32; ++g) dg2[((size_t)j * N + k) * 32 + g] = d.dg[((size_t)j * N + ord[k]) * 32 + g];
        p = p2; d.um = um2; d.ud = ud2; d.dg = dg2; d.a0 = a02; d.ue = ue2; d.uf = uf2;
    }
    // per job, the least usable durations per global slot, packed two per word (kernel viability)
    d.dgp.assign((size_t)J * 16, 0x7FFF7FFFu);
    for (int j = 0; j < J; ++j)
        for (int n = 0; n < N; ++n)
            for (int k = 0; k < p.node_g[n]; ++k) {
                const int slot = p.node_off[n] + k;
                const uint32_t v = (uint32_t)(uint16_t)d.dg[((size_t)j * N + n) * 32 + k];
                uint32_t &wd = d.dgp[(size_t)j * 16 + slot / 2];
                wd = (slot & 1) ? ((wd & 0xFFFFu) | (v << 16)) : ((wd & 0xFFFF0000u) | v);
            }
    // key width: 2^J x prod C(T + G_n, G_n) < 2^127
    const int n_max = T + gmax;
    p.Kb = gmax + 1;
    d.binom.assign((size_t)(n_max + 1) * p.Kb, 0);
    for (int n = 0; n <= n_max; ++n) {
        d.binom[(size_t)n * p.Kb] = 1;
        for (int k = 1; k <= gmax && k <= n; ++k) {
            const unsigned __int128 v = (unsigned __int128)d.binom[(size_t)(n - 1) * p.Kb + k - 1] +
                                        (k <= n - 1 ? d.binom[(size_t)(n - 1) * p.Kb + k] : 0);
            if (v >> 62) return SAT_ERR_UNSUPPORTED;
            d.binom[(size_t)n * p.Kb + k] = (uint64_t)v;
        }
    }
    double bits = J;
    for (int n = 0; n < N; ++n) {
        p.cnum[n] = d.binom[(size_t)(T + p.node_g[n]) * p.Kb + p.node_g[n]];
        bits += std::log2((double)p.cnum[n]);
    }
    if (bits > 126.0) return SAT_ERR_UNSUPPORTED;
    uint64_t cap = 1;
    int lg = 0;
    while (cap < 2 * max_states + (1u << 16)) { cap <<= 1; ++lg; }
    d.cap = cap;
    p.cap_mask = cap - 1;
    p.cap_log2 = lg;
    p.max_probe = 1 << 14;
    d.binom_bytes = align256(d.binom.size() * sizeof(uint64_t));
    d.aux_bytes = align256(d.ug.size() + 16) + align256(d.um.size() + 16) + align256(d.ud.size() * 2 + 16) +
                  align256(d.dg.size() * 2) + align256(d.ue.size() + 16) + align256(d.uf.size() * 2 + 16) +
                  align256(d.dgp.size() * 4);
    d.table_bytes = align256(cap * 16);
    d.R_bytes = align256(max_states * sizeof(uint64_t));
    d.A_bytes = align256(max_states * off * sizeof(uint16_t));
    return SAT_OK;
}

static size_t dpw_ws_bytes(const DpWidePlan &d) {
    return d.binom_bytes + d.aux_bytes + d.table_bytes + d.R_bytes + d.A_bytes + 256;
}

static int dpw_run(const sat_problem_t *pr, uint64_t max_states, sat_dp_info_t *info, void *d_ws, size_t ws_bytes,
                   cudaStream_t s, DpWidePlan &d, uint8_t *h_candidate = nullptr) {
    if (!d_ws || ws_bytes < dpw_ws_bytes(d)) return SAT_ERR_INVALID;
    DpWideParams &p = d.p;
    uint8_t *ws = static_cast<uint8_t *>(d_ws);
    size_t o = 0;
    auto take = [&](size_t bytes) { uint8_t *r = ws + o; o += bytes; return r; };
    uint64_t *binom = reinterpret_cast<uint64_t *>(take(d.binom_bytes));
    uint8_t *ug = take(align256(d.ug.size() + 16));
    uint8_t *um = take(align256(d.um.size() + 16));
    int16_t *ud = reinterpret_cast<int16_t *>(take(align256(d.ud.size() * 2 + 16)));
    int16_t *dg = reinterpret_cast<int16_t *>(take(align256(d.dg.size() * 2)));
    uint8_t *ue = take(align256(d.ue.size() + 16));
    int16_t *uf = reinterpret_cast<int16_t *>(take(align256(d.uf.size() * 2 + 16)));
    uint32_t *dgp = reinterpret_cast<uint32_t *>(take(align256(d.dgp.size() * 4)));
    auto *table = reinterpret_cast<unsigned __int128 *>(take(d.table_bytes));
    uint64_t *Rs = reinterpret_cast<uint64_t *>(take(d.R_bytes));
    uint16_t *As = reinterpret_cast<uint16_t *>(take(d.A_bytes));
    auto *ctr = reinterpret_cast<unsigned long long *>(take(256));
    const int J = pr->J, Gt = p.Gtot;
    if (cudaMemcpyAsync(binom, d.binom.data(), d.binom.size() * 8, cudaMemcpyHostToDevice, s) ||
        (d.ug.size() && cudaMemcpyAsync(ug, d.ug.data(), d.ug.size(), cudaMemcpyHostToDevice, s)) ||
        (d.um.size() && cudaMemcpyAsync(um, d.um.data(), d.um.size(), cudaMemcpyHostToDevice, s)) ||
        (d.ud.size() && cudaMemcpyAsync(ud, d.ud.data(), d.ud.size() * 2, cudaMemcpyHostToDevice, s)) ||
        cudaMemcpyAsync(dg, d.dg.data(), d.dg.size() * 2, cudaMemcpyHostToDevice, s) ||
        (d.ue.size() && cudaMemcpyAsync(ue, d.ue.data(), d.ue.size(), cudaMemcpyHostToDevice, s)) ||
        (d.uf.size() && cudaMemcpyAsync(uf, d.uf.data(), d.uf.size() * 2, cudaMemcpyHostToDevice, s)) ||
        cudaMemcpyAsync(dgp, d.dgp.data(), d.dgp.size() * 4, cudaMemcpyHostToDevice, s) ||
        cudaMemsetAsync(table, 0xFF, d.cap * 16, s) || cudaMemsetAsync(ctr, 0, 256, s))
        return SAT_ERR_CUDA;
    const uint64_t full = J == 64 ? ~0ull : ((1ull << J) - 1ull);
    if (cudaMemcpyAsync(Rs, &full, 8, cudaMemcpyHostToDevice, s) ||
        cudaMemcpyAsync(As, d.a0.data(), Gt * 2, cudaMemcpyHostToDevice, s))
        return SAT_ERR_CUDA;
    p.binom = binom; p.ug = ug; p.um = um; p.ud = ud; p.dg = dg; p.table = table;
    p.ue = ue; p.uf = uf; p.dgp = dgp;
    p.count = ctr;
    p.overflow = reinterpret_cast<unsigned int *>(ctr + 1);
    p.pick_hi = ctr + 2;
    p.pick_lo = ctr + 3;
    p.pick_R = reinterpret_cast<uint64_t *>(ctr + 4);
    p.pick_A = reinterpret_cast<uint16_t *>(ctr + 5);          // 32 x u16 = ctr[5..12]
    std::vector<uint64_t> lv_base(J + 1, 0), lv_size(J + 1, 0);
    lv_size[0] = 1;
    uint64_t base = 0, size = 1, total = 1, widest = 1;
    int level = 0;
    for (; level < J; ++level) {
        p.in_R = Rs + base; p.in_A = As + base * Gt; p.n_in = size;
        const uint64_t nb = base + size;
        p.out_R = Rs + nb; p.out_A = As + nb * Gt; p.out_cap = max_states - nb;
        if (cudaMemsetAsync(ctr, 0, 8, s)) return SAT_ERR_CUDA;
        p.nrem = J - level;
        const uint64_t blocks = (p.n_in * (uint64_t)p.nrem + kDpThreads - 1) / kDpThreads;
        if (blocks > 0x7fffffffull) return SAT_ERR_TOO_LARGE;
        if (dpw_launch_level(p, (unsigned)blocks, s) != SAT_OK) return SAT_ERR_CUDA;
        unsigned long long got[2];
        if (cudaMemcpyAsync(got, ctr, sizeof(got), cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
            return SAT_ERR_CUDA;
        if ((unsigned int)got[1]) {
            info->status = SAT_DP_BUDGET;
            info->levels = level; info->states = total; info->widest_level = widest;
            return SAT_OK;
        }
        base = nb; size = got[0];
        lv_base[level + 1] = base;
        lv_size[level + 1] = size;
        total += size;
        widest = std::max(widest, size);
        if (size == 0) { ++level; break; }
    }
    info->levels = level; info->states = total; info->widest_level = widest;
    info->status = (level < J || size == 0) ? SAT_DP_INFEASIBLE : SAT_DP_FEASIBLE;
    info->makespan = -1;                      // the prover rebuilds no candidate
    if (info->status != SAT_DP_FEASIBLE || !p.exact) return SAT_OK;
    // exact mode: a candidate reaching T -- the smallest-key final state, then backwards the
    // smallest-key parent and (on the host) its lowest usable option producing the child
    const unsigned long long ones[2] = {~0ull, ~0ull};
    auto pick = [&](int lv, int mode, uint64_t &R, std::vector<int32_t> &A) -> int {
        p.in_R = Rs + lv_base[lv]; p.in_A = As + lv_base[lv] * Gt; p.n_in = lv_size[lv];
        p.nrem = J - lv;
        if (cudaMemcpyAsync(p.pick_hi, ones, sizeof(ones), cudaMemcpyHostToDevice, s)) return SAT_ERR_CUDA;
        const uint64_t work = p.n_in * (uint64_t)(mode == 0 ? 1 : p.nrem);
        const unsigned blocks = (unsigned)((work + kDpThreads - 1) / kDpThreads);
        for (int ph = 0; ph < 3; ++ph) {
            k_dpw_pick_state<<<blocks, kDpThreads, 0, s>>>(p, mode, ph);
            if (cudaGetLastError() != cudaSuccess) return SAT_ERR_CUDA;
        }
        unsigned long long back[11];                    // hi, lo, R, A (64 bytes)
        if (cudaMemcpyAsync(back, ctr + 2, sizeof(back), cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
            return SAT_ERR_CUDA;
        if (back[0] == ~0ull && back[1] == ~0ull) return SAT_ERR_CUDA;   // nothing picked: cannot happen
        R = back[2];
        const uint16_t *a16 = reinterpret_cast<const uint16_t *>(back + 3);
        A.assign(Gt, 0);
        for (int i = 0; i < Gt; ++i) A[i] = a16[i];
        return SAT_OK;
    };
    std::vector<int32_t> cur, par, tmp(Gt);
    uint64_t curR = 0, parR = 0;
    int st = pick(J, 0, curR, cur);
    if (st) return st;
    info->makespan = *std::max_element(cur.begin(), cur.end());
    auto host_pick = [&](const std::vector<int32_t> &a, int q, int j) {
        int32_t best = 0x7fffffff;
        int bn = -1;
        for (int n = 0; n < p.N; ++n) {
            if (!((d.ue[q] >> n) & 1u) || d.ug[q] > p.node_g[n]) continue;
            const int32_t e = std::max<int32_t>(a[p.node_off[n] + d.ug[q] - 1], p.release[j]) + d.uf[q * p.N + n];
            if (e < best) { best = e; bn = n; }
        }
        return bn;
    };
    std::vector<int> order(J), opt(J);
    for (int lv = J; lv >= 1; --lv) {
        p.child_R = curR;
        for (int i = 0; i < Gt; ++i) p.child_A[i] = (uint16_t)cur[i];
        if ((st = pick(lv - 1, 1, parR, par))) return st;
        const int j = __builtin_ctzll(parR ^ curR);
        int found = -1;
        for (int q = p.ubase[j]; q < p.ubase[j] + p.ucnt[j] && found < 0; ++q) {
            const int bn = host_pick(par, q, j);
            if (bn < 0 || !((d.um[q] >> bn) & 1u)) continue;
            tmp = par;
            const int g = d.ug[q], G = p.node_g[bn], off = p.node_off[bn];
            const int32_t e = std::max<int32_t>(par[off + g - 1], p.release[j]) + d.uf[q * p.N + bn];
            for (int i = 0; i < G; ++i) tmp[off + i] = std::max(par[off + i], std::min(i + g < G ? par[off + i + g] : 0x7fffffff, e));
            if (tmp == cur) found = q;
        }
        if (found < 0) return SAT_ERR_CUDA;
        order[lv - 1] = j;
        opt[j] = d.uorig[found];
        curR = parR;
        cur = par;
    }
    if (h_candidate) {
        for (int j = 0; j < J; ++j) h_candidate[j] = (uint8_t)opt[j];
        for (int k = 0; k < J; ++k) h_candidate[J + k] = (uint8_t)order[k];
    }
    return SAT_OK;
}

}  // namespace sat

using namespace sat;

extern "C" {

int sat_dp_workspace_bytes_ex(const sat_problem_t *p, int32_t target, uint64_t max_states, int32_t flags,
                              size_t *bytes) {
    if (!bytes || (flags & ~SAT_DP_EXACT)) return SAT_ERR_INVALID;
    int st = validate(p);
    if (st) return st;
    DpPlan d;
    st = dp_prepare(p, target, max_states, d);
    if (st == SAT_OK) {
        *bytes = d.status >= 0 ? 256 : dp_ws_bytes(d);
        return SAT_OK;
    }
    if (st != SAT_ERR_UNSUPPORTED) return st;
    DpWidePlan w;                                    // several nodes / wide keys: the prover
    st = dpw_prepare(p, target, max_states, w, (flags & SAT_DP_EXACT) != 0);
    if (st) return st;
    *bytes = w.status >= 0 ? 256 : dpw_ws_bytes(w);
    return SAT_OK;
}

int sat_dp_workspace_bytes(const sat_problem_t *p, int32_t target, uint64_t max_states, size_t *bytes) {
    return sat_dp_workspace_bytes_ex(p, target, max_states, 0, bytes);
}

int sat_search_dp(const sat_problem_t *pr, int32_t target, uint64_t max_states, uint8_t *h_candidate,
                  sat_dp_info_t *info, void *d_ws, size_t ws_bytes, void *stream) {
    return sat_search_dp_ex(pr, target, max_states, 0, h_candidate, info, d_ws, ws_bytes, stream);
}

int sat_search_dp_ex(const sat_problem_t *pr, int32_t target, uint64_t max_states, int32_t flags,
                     uint8_t *h_candidate, sat_dp_info_t *info, void *d_ws, size_t ws_bytes, void *stream) {
    if (!info || (flags & ~SAT_DP_EXACT)) return SAT_ERR_INVALID;
    int st = validate(pr);
    if (st) return st;
    nvtxRangePushA("sat_search_dp");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_on_exit;
    std::memset(info, 0, sizeof(*info));
    DpPlan d;
    st = dp_prepare(pr, target, max_states, d);
    if (st == SAT_ERR_UNSUPPORTED) {                 // several nodes / wide keys: the prover
        DpWidePlan w;
        st = dpw_prepare(pr, target, max_states, w, (flags & SAT_DP_EXACT) != 0);
        if (st) return st;
        if (w.status >= 0) {
            // decided on the host (an initial free time or every option past the target):
            // INFEASIBLE, never FEASIBLE without a search
            info->status = w.status; info->makespan = -1; return SAT_OK;
        }
        return dpw_run(pr, max_states, info, d_ws, ws_bytes, (cudaStream_t)stream, w, h_candidate);
    }
    if (st) return st;
    if (d.status >= 0) { info->status = d.status; return SAT_OK; }
    if (!d_ws || ws_bytes < dp_ws_bytes(d)) return SAT_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t *ws = static_cast<uint8_t *>(d_ws);
    uint64_t *binom = reinterpret_cast<uint64_t *>(ws);
    uint64_t *table = reinterpret_cast<uint64_t *>(ws + d.binom_bytes);
    uint64_t *Rs = reinterpret_cast<uint64_t *>(ws + d.binom_bytes + d.table_bytes);
    uint16_t *As = reinterpret_cast<uint16_t *>(ws + d.binom_bytes + d.table_bytes + d.R_bytes);
    auto *ctr = reinterpret_cast<unsigned long long *>(ws + d.binom_bytes + d.table_bytes + d.R_bytes + d.A_bytes);
    DpParams &p = d.p;
    const int J = pr->J, Gr = p.Gr;
    // level 0: every job to place, the initial free times; lvl_cnt[0] = 1, every other count 0
    std::vector<unsigned long long> ctr_init(kDpCtrBytes / sizeof(unsigned long long), 0ull);
    ctr_init[8] = 1;
    if (cudaMemcpyAsync(binom, d.binom.data(), d.binom.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s) ||
        cudaMemsetAsync(table, 0xFF, d.cap * sizeof(uint64_t), s) ||
        cudaMemcpyAsync(ctr, ctr_init.data(), kDpCtrBytes, cudaMemcpyHostToDevice, s))
        return SAT_ERR_CUDA;
    const uint64_t full = J == 64 ? ~0ull : ((1ull << J) - 1ull);
    std::vector<uint16_t> a0(Gr);
    for (int i = 0; i < Gr; ++i) a0[i] = (uint16_t)d.a0[i];
    if (cudaMemcpyAsync(Rs, &full, sizeof(full), cudaMemcpyHostToDevice, s) ||
        cudaMemcpyAsync(As, a0.data(), Gr * sizeof(uint16_t), cudaMemcpyHostToDevice, s))
        return SAT_ERR_CUDA;
    p.binom = binom;
    p.table = table;
    p.min_key = ctr;
    p.overflow = reinterpret_cast<unsigned int *>(ctr + 1);
    p.lvl_cnt = ctr + 8;
    p.lvl_base = ctr + 8 + (kDpMaxJ + 1);
    p.all_R = Rs;
    p.all_A = As;
    p.max_states = max_states;
    // every level queued back to back; one read-back of the counts at the end
    for (int L = 0; L < J; ++L)
        if ((st = dp_expand(p, L, s))) return st;
    std::vector<unsigned long long> got(kDpCtrBytes / sizeof(unsigned long long));
    if (cudaMemcpyAsync(got.data(), ctr, kDpCtrBytes, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
        return SAT_ERR_CUDA;
    const unsigned int ovf = (unsigned int)got[1];
    std::vector<uint64_t> base(J + 2, 0), size(J + 2, 0);
    uint64_t total = 0, widest = 0;
    int level = 0;
    size[0] = 1;
    for (int L = 0; L <= J; ++L) {
        if (ovf && L == (int)ovf) {                     // level L's expansion from L - 1 overflowed
            info->status = SAT_DP_BUDGET;
            info->levels = L - 1;
            info->states = total;
            info->widest_level = widest;
            return SAT_OK;
        }
        size[L] = got[8 + L];
        if (L > 0) base[L] = base[L - 1] + size[L - 1];
        total += size[L];
        widest = std::max<uint64_t>(widest, size[L]);
        level = L;
        if (size[L] == 0) break;
    }
    info->levels = level;
    info->states = total;
    info->widest_level = widest;
    if (level < J || size[J] == 0) { info->status = SAT_DP_INFEASIBLE; return SAT_OK; }
    // a candidate reaching T: smallest-key final state, then backwards the smallest-key parent
    // and its lowest option producing the child
    info->status = SAT_DP_FEASIBLE;
    const unsigned long long ones = ~0ull;
    auto min_key_of = [&](int lv, auto launch) -> int {
        p.in_R = Rs + base[lv];
        p.in_A = As + base[lv] * Gr;
        p.n_in = size[lv];
        if (cudaMemcpyAsync(p.min_key, &ones, sizeof(ones), cudaMemcpyHostToDevice, s)) return SAT_ERR_CUDA;
        return launch();
    };
    st = min_key_of(J, [&]() {
        const uint64_t blocks = (p.n_in + kDpThreads - 1) / kDpThreads;
        k_dp_min_key<<<(unsigned)blocks, kDpThreads, 0, s>>>(p);
        return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
    });
    if (st) return st;
    unsigned long long key;
    if (cudaMemcpyAsync(&key, p.min_key, sizeof(key), cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
        return SAT_ERR_CUDA;
    std::vector<int32_t> cur(Gr), par(Gr), tmp(Gr);
    uint64_t curR;
    dp_unrank(d, key, &curR, cur.data());
    info->makespan = cur[Gr - 1];
    std::vector<int> order(J), opt(J);
    for (int lv = J; lv >= 1; --lv) {
        p.child_R = curR;
        for (int i = 0; i < Gr; ++i) p.child_A[i] = (uint16_t)cur[i];
        st = min_key_of(lv - 1, [&]() { return dp_parent(p, s); });
        if (st) return st;
        if (cudaMemcpyAsync(&key, p.min_key, sizeof(key), cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
            return SAT_ERR_CUDA;
        if (key == ones) return SAT_ERR_CUDA;          // no parent: cannot happen
        uint64_t parR;
        dp_unrank(d, key, &parR, par.data());
        const int j = __builtin_ctzll(parR ^ curR);
        int found = -1;
        for (int q = p.ubase[j]; q < p.ubase[j] + p.ucnt[j] && found < 0; ++q) {
            dp_host_place(d, par.data(), q, p.release[j], tmp.data());
            if (std::equal(tmp.begin(), tmp.end(), cur.begin())) found = q;
        }
        if (found < 0) return SAT_ERR_CUDA;
        order[lv - 1] = j;
        opt[j] = d.uorig[found];
        curR = parR;
        cur = par;
    }
    if (h_candidate) {
        for (int j = 0; j < J; ++j) h_candidate[j] = (uint8_t)opt[j];
        for (int k = 0; k < J; ++k) h_candidate[J + k] = (uint8_t)order[k];
    }
    return SAT_OK;
}

}  // extern "C"
