// sat_cand.cuh -- k_cand<T, SRC, G, L>: one candidate per THREAD.
//
// The search kernel for everything the prefix-shared walk (k_tree) does not cover:
// sampled candidate streams (plan_random draws, configs 3-5), multi-node clusters,
// float64 time, release times and initial free times (re-solve), and exhaustive
// index ranges of such problems.
//
// Each thread decodes its candidate into J step records (g-1 | job<<6 | payload<<12)
// in its own shared-memory column, then list-schedules it.  Per node the GPU free
// times are kept sorted ascending; placing a (g, d) job that can start at
// s = max(a[g-1], release) with end e = s + d turns the vector into
//        b[i] = max(a[i], min(a[i+g], e))          (a[k] = +inf for k >= G)
// (DESIGN.md section 4.1).  The shift by the thread's own g is a read of its own
// shared-memory column at rows i+g: every lane stays in its own bank (row stride 32
// words), so a warp's 32 different g values cost one wavefront per row, and the
// thread's vector itself stays in registers (one node) or in the column (several
// nodes: the node is chosen at run time).  Rows G..2G-1 of a node hold +inf.
//
// Per placement: 1 + G shared loads, G shared stores, G min + G max, 1 add, 1 max
// (one node); multi-node adds N loads + the earliest-finish node pick.  When no free
// time can reach 2^16 (grid time, one node) two slots share a word: G/2 + 2 loads,
// G/2 stores, G/2 PRMT + G/2 VIMNMX.U16x2 min + G/2 max per placement.
#pragma once

#include "sat_decode.cuh"

namespace sat {

constexpr int kCandThreads = 128;
constexpr int kCandWarps = kCandThreads / 32;

struct CandArgs {
    const uint8_t *blob;
    uint64_t lo, hi;            // candidate ids [lo, hi)
    uint64_t seed;
    int32_t per_lane;           // consecutive ids per thread per warp chunk
    unsigned long long *cursor; // warp chunks handed out so far (zeroed before the launch)
    int32_t rec_d;              // records carry the duration (node-independent, all nodes eligible)
    sat_best_t *best;           // grid mode result
    sat_best_t *partials;       // float mode per-block partials
};

// bytes of one warp's private region: records, index scratch, free-time columns
// (slot_bytes: 4 int32, 8 fp64, 2 packed 16-bit -- every node has 2G slots, G of them +inf)
// Packed layouts read one row past a node's slots (the unused partner word when g is even):
// a trailing pad row keeps the last node's read inside the warp's region.
__host__ __device__ inline int cand_warp_bytes(int J, int N, int G, int slot_bytes, bool index_src) {
    return J * 128 + (index_src ? J * 64 : 0) + N * 2 * G * 32 * slot_bytes + (slot_bytes == 2 ? 128 : 0);
}

// Layouts of the free-time state (template parameter L)
constexpr int kLayoutOne = 0;     // one node, 32-bit (or fp64) slots
constexpr int kLayoutMulti = 1;   // several nodes, node chosen per placement
constexpr int kLayoutOne16 = 2;   // one node, two 16-bit slots per word (grid time < 2^16)
constexpr int kLayoutMulti16 = 3; // several nodes, 16-bit slots, records carry durations

template <typename T, int L>
__host__ __device__ constexpr int cand_slot_bytes() {
    return (L == kLayoutOne16 || L == kLayoutMulti16) ? 2 : (int)sizeof(T);
}

// Everything the list scheduler reads, resolved once per kernel (pointers are per lane).
template <typename T>
struct SchedCtx {
    T *st;                   // the lane's free-time column: [N][2G][32] (T) or [N][G][32] words (packed)
    uint32_t *st16;
    const T *lane_init;      // [N][G] initial free times (+inf on ghost slots)
    const T *release;        // [J]
    const T *dur;            // [n_opt][N] (when records carry option ids)
    const uint32_t *optmask; // [n_opt] node eligibility (several nodes)
    int J, N, n_opt;
    bool rec_d, has_release;
    T init_max, INF;
};

// List-schedule the J step records in the lane's record column (stride 32) and return the
// makespan.  Layout L as in the file comment; G = padded GPUs per node.
// Prefix cache (local search): cin / cout point at a warp-shared array of J + 1 entries of
// cache_words<G, L>(N) words -- the free-time state before position k, then the makespan
// so far.  With cin the schedule resumes at position k0 from entry k0 (records before k0 are
// not read); with cout (written by `writer` only) every entry of this candidate is stored.
template <int G, int L>
__host__ __device__ constexpr int cache_state_words(int N) {
    return (L == kLayoutOne16 || L == kLayoutMulti16) ? N * (G / 2) : N * G;
}

// Record providers: schedule_records reads the record of position k through `rec(k)`.
//   RecCol   -- the lane's materialised record column (k_cand: decoded candidates);
//   RecMove  -- k_ls: the walker's current records (one shared copy per walker) seen through
//               a move, computed per position (no per-move record column to build or hold).
struct RecCol {
    const uint32_t *p;                           // lane's column, stride 32
    __device__ __forceinline__ uint32_t operator()(int k) const { return p[k * 32]; }
};

// Early exit (CUT, k_ls move evaluation): a move is only of interest if it IMPROVES the current
// candidate's (makespan, load).  List scheduling is monotone -- a placement's new vector is
// non-decreasing in the old one -- so the evaluation stops, returning makespan cut + 1 (an
// objective above the current one), as soon as (a) the running makespan exceeds `cut` (the
// current makespan), or (b) past the last position the move changes (klast) the free-time
// state dominates the current candidate's state at the same position (cin = the walker's
// prefix cache): every later state, the makespan and the load can then only be >= the current
// ones.  Improving moves are scheduled to the end, so the walk is unchanged.
#ifndef SAT_LS_CUT
#define SAT_LS_CUT 1     // 0: no early exit, 1: running makespan only, 2: + dominance (measured:
                         // cfg5 11.5 / 12.3 / 15.4 ms, cfg3 5.2 / 5.0 / 5.2 ms -- the dominance test
                         // costs more than it saves)
#endif
#ifndef SAT_LS_CUT_REG
#define SAT_LS_CUT_REG 0 // the same exits in the register-shift evaluation (schedule_eval16)
#endif
// Multi16 placement loop (schedule_records, several nodes, 16-bit slots): NN = the node count
// when every node slot of the layout is used (compile-time loops), 0 = runtime N; REL = the
// problem has release times.
template <typename T, int G, int NN, bool REL, typename RecF>
__device__ __forceinline__ T m16_walk(const SchedCtx<T> &c, const RecF rec, int k0, T mx, uint32_t *cout, bool wr) {
    constexpr int NMAX = 32 / G;
    uint32_t *st16 = c.st16;
    const int J = c.J, N = NN > 0 ? NN : c.N;
    const bool rec_d = c.rec_d;
    (void)rec_d;
    const int SW = N * (G / 2), CW = SW + 1;
    (void)CW;
        for (int kk = k0; kk < J; ++kk) {
            const uint32_t r = rec(kk);
            const int g = (int)(r & 63u) + 1;
            SAT_ASSERT(g >= 1 && g <= G && (int)((r >> 6) & 63u) < J);
            SAT_ASSERT(rec_d || (int)(r >> 12) < c.n_opt);
            const int gm = g - 1;
            const int32_t rel = REL ? (int32_t)c.release[(r >> 6) & 63u] : 0;
            const uint32_t selt = 0x4410u + (uint32_t)(gm & 1) * 0x22u;
            uint32_t kb = 0xffffffffu;
#pragma unroll
            for (int n = 0; n < NMAX; ++n) {
                if (NN > 0 || n < N) {
                    int32_t t = (int32_t)__byte_perm(st16[(n * G + (gm >> 1)) * 32], 0u, selt);
                    if (REL) t = max(t, rel);
                    kb = min(kb, (uint32_t)t * 32u + (uint32_t)n);
                }
            }
            const int bn = (int)(kb & 31u);
            SAT_ASSERT(bn < N);
            const int32_t e = (int32_t)(kb >> 5) + (int32_t)(r >> 12);
            const uint32_t e2 = (uint32_t)e * 0x10001u;
            const uint32_t sel = (g & 1) ? 0x5432u : 0x3210u;
            uint32_t *nb = st16 + bn * G * 32;
            const uint32_t *src = nb + (g >> 1) * 32;
            uint32_t w[G / 2 + 1], cur[G / 2];
#pragma unroll
            for (int k = 0; k <= G / 2; ++k) w[k] = src[k * 32];
#pragma unroll
            for (int k = 0; k < G / 2; ++k) cur[k] = nb[k * 32];
#pragma unroll
            for (int k = 0; k < G / 2; ++k)
                nb[k * 32] = __vmaxu2(cur[k], __vminu2(__byte_perm(w[k], w[k + 1], sel), e2));
            mx = tmax(mx, (T)e);
            if (wr) {
#pragma unroll
                for (int n = 0; n < NMAX; ++n)
                    if (NN > 0 || n < N)
#pragma unroll
                        for (int q = 0; q < G / 2; ++q) cout[(kk + 1) * CW + n * (G / 2) + q] = st16[(n * G + q) * 32];
                cout[(kk + 1) * CW + SW] = (uint32_t)(int32_t)mx;
            }
        }
    return mx;
}

template <typename T, int G, int L, bool LOAD = false, typename RecF = RecCol, bool CUT = false,
          bool NOREL = false>   // NOREL: the problem has no release times (no per-placement release read)
__device__ __forceinline__ T schedule_records(const SchedCtx<T> &c, const RecF rec,
                                             uint64_t *load = nullptr, int k0 = 0,
                                             const uint32_t *cin = nullptr, uint32_t *cout = nullptr,
                                             bool writer = false, int cut = 0, int klast = 0) {
    constexpr bool P16 = L == kLayoutOne16;
    constexpr bool M16 = L == kLayoutMulti16;
    constexpr int NMAX = (L == kLayoutMulti || M16) ? (32 / G) : 1;
    T *st = c.st;
    uint32_t *st16 = c.st16;
    const T *lane_init = c.lane_init;
    const T *release = c.release;
    const T *dur = c.dur;
    const int J = c.J, N = c.N;
    const bool rec_d = c.rec_d, has_release = c.has_release;
    const T INF = c.INF;
    (void)INF; (void)dur; (void)N;
    const int SW = cache_state_words<G, L>(N), CW = SW + 1;
    T mx = cin ? (T)(int32_t)cin[k0 * CW + SW] : c.init_max;
    const bool wr = cout != nullptr && writer;
    (void)SW; (void)CW; (void)wr;
    if constexpr (P16) {
        // slots 2w (low half) and 2w+1 (high half) of word w; rows G/2..G-1 = +inf.
        // Shift by the thread's g: word k of the shifted vector is word g/2 + k (g even)
        // or the high half of word g/2 + k joined to the low half of the next (g odd):
        // one PRMT with a per-thread selector either way.
        uint32_t av[G / 2];
#pragma unroll
        for (int w = 0; w < G / 2; ++w) {
            av[w] = cin ? cin[k0 * CW + w]
                        : (uint32_t)(uint16_t)lane_init[2 * w] | ((uint32_t)(uint16_t)lane_init[2 * w + 1] << 16);
            st16[w * 32] = av[w];
            if (wr) cout[k0 * CW + w] = av[w];
        }
        if (wr) cout[k0 * CW + SW] = (uint32_t)(int32_t)mx;
        for (int kk = k0; kk < J; ++kk) {
            const uint32_t r = rec(kk);
            const int g = (int)(r & 63u) + 1;
            SAT_ASSERT(g >= 1 && g <= G && (int)((r >> 6) & 63u) < J);
            SAT_ASSERT(rec_d || (int)(r >> 12) < c.n_opt);
            const int gm = g - 1;
            // slot g-1 = one half of word (g-1)/2 (read as the word: no type-punned loads)
            const uint32_t selt = 0x4410u + (uint32_t)(gm & 1) * 0x22u;
            int32_t t = (int32_t)__byte_perm(st16[(gm >> 1) * 32], 0u, selt);
            if (!NOREL && has_release) t = max(t, (int32_t)release[(r >> 6) & 63u]);
            const int32_t e = t + (int32_t)(r >> 12);
            const uint32_t e2 = (uint32_t)e * 0x10001u;
            const uint32_t sel = (g & 1) ? 0x5432u : 0x3210u;
            const uint32_t *src = st16 + (g >> 1) * 32;
            uint32_t w[G / 2 + 1];
#pragma unroll
            for (int k = 0; k <= G / 2; ++k) w[k] = src[k * 32];
#pragma unroll
            for (int k = 0; k < G / 2; ++k) {
                const uint32_t s = __byte_perm(w[k], w[k + 1], sel);
                av[k] = __vmaxu2(av[k], __vminu2(s, e2));
                st16[k * 32] = av[k];
            }
            mx = tmax(mx, (T)e);
            if constexpr (CUT && SAT_LS_CUT > 0) {
                bool worse = mx > (T)cut;
                if (SAT_LS_CUT > 1 && !worse && cin && kk >= klast) {
                    uint32_t diff = 0;
#pragma unroll
                    for (int k = 0; k < G / 2; ++k) {
                        const uint32_t cw = cin[(kk + 1) * CW + k];
                        diff |= __vmaxu2(av[k], cw) ^ av[k];
                    }
                    worse = diff == 0;
                }
                if (worse) {
                    if constexpr (LOAD) *load = 0;
                    return (T)(cut + 1);
                }
            }
            if (wr) {
#pragma unroll
                for (int w = 0; w < G / 2; ++w) cout[(kk + 1) * CW + w] = av[w];
                cout[(kk + 1) * CW + SW] = (uint32_t)(int32_t)mx;
            }
        }
        if constexpr (LOAD) {
            uint64_t sum = 0;
#pragma unroll
            for (int w = 0; w < G / 2; ++w) {
                const uint32_t lo = av[w] & 0xffffu, hi = av[w] >> 16;
                sum += (lo != 0xffffu ? lo : 0u) + (hi != 0xffffu ? hi : 0u);
            }
            *load = sum;
        }
    } else if constexpr (L == kLayoutOne) {
        T av[G];
#pragma unroll
        for (int i = 0; i < G; ++i) {
            av[i] = cin ? (T)(int32_t)cin[k0 * CW + i] : lane_init[i];
            st[i * 32] = av[i];
            if (wr) cout[k0 * CW + i] = (uint32_t)(int32_t)av[i];
        }
        if (wr) cout[k0 * CW + SW] = (uint32_t)(int32_t)mx;
        for (int kk = k0; kk < J; ++kk) {
            const uint32_t r = rec(kk);
            const int g = (int)(r & 63u) + 1;
            SAT_ASSERT(g >= 1 && g <= G && (int)((r >> 6) & 63u) < J);
            SAT_ASSERT(rec_d || (int)(r >> 12) < c.n_opt);
            const T d = rec_d ? (T)(int32_t)(r >> 12) : dur[r >> 12];
            T t = st[(g - 1) * 32];
            if (!NOREL && has_release) t = tmax(t, release[(r >> 6) & 63u]);
            const T e = t + d;
            T s[G];
#pragma unroll
            for (int i = 0; i < G; ++i) s[i] = st[(i + g) * 32];
#pragma unroll
            for (int i = 0; i < G; ++i) {
                av[i] = tmax(av[i], tmin(s[i], e));
                st[i * 32] = av[i];
            }
            mx = tmax(mx, e);
            if constexpr (CUT && SAT_LS_CUT > 0) {
                bool worse = mx > (T)cut;
                if (SAT_LS_CUT > 1 && !worse && cin && kk >= klast) {
                    bool dom = true;
#pragma unroll
                    for (int i = 0; i < G; ++i) dom &= av[i] >= (T)(int32_t)cin[(kk + 1) * CW + i];
                    worse = dom;
                }
                if (worse) {
                    if constexpr (LOAD) *load = 0;
                    return (T)(cut + 1);
                }
            }
            if (wr) {
#pragma unroll
                for (int i = 0; i < G; ++i) cout[(kk + 1) * CW + i] = (uint32_t)(int32_t)av[i];
                cout[(kk + 1) * CW + SW] = (uint32_t)(int32_t)mx;
            }
        }
        if constexpr (LOAD) {
            uint64_t sum = 0;
#pragma unroll
            for (int i = 0; i < G; ++i) sum += (av[i] != INF) ? (uint64_t)(int64_t)av[i] : 0ull;
            *load = sum;
        }
    } else if constexpr (M16) {
        // per node n: words n*G .. n*G+G/2-1 = slots, n*G+G/2 .. n*G+G-1 = +inf.  Node pick:
        // min over nodes of (start << 5 | n) = earliest start, lowest node on ties
        // (durations are node-independent in this layout, so earliest start = earliest end).
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
            if (n < N)
#pragma unroll
                for (int w = 0; w < G / 2; ++w) {
                    const uint32_t v = cin ? cin[k0 * CW + n * (G / 2) + w]
                                           : (uint32_t)(uint16_t)lane_init[n * G + 2 * w] |
                                                 ((uint32_t)(uint16_t)lane_init[n * G + 2 * w + 1] << 16);
                    st16[(n * G + w) * 32] = v;
                    if (wr) cout[k0 * CW + n * (G / 2) + w] = v;
                }
        if (wr) cout[k0 * CW + SW] = (uint32_t)(int32_t)mx;
        // the placement loop specialised on (every node slot used, release times present):
        // no per-node predicates and no release max on the common sampled / local-search path
        if (N == NMAX) {
            mx = has_release ? m16_walk<T, G, NMAX, true>(c, rec, k0, mx, cout, wr)
                             : m16_walk<T, G, NMAX, false>(c, rec, k0, mx, cout, wr);
        } else {
            mx = has_release ? m16_walk<T, G, 0, true>(c, rec, k0, mx, cout, wr)
                             : m16_walk<T, G, 0, false>(c, rec, k0, mx, cout, wr);
        }
        if constexpr (LOAD) {
            uint64_t sum = 0;
#pragma unroll
            for (int n = 0; n < NMAX; ++n)
                if (n < N)
#pragma unroll
                    for (int w = 0; w < G / 2; ++w) {
                        const uint32_t v = st16[(n * G + w) * 32];
                        const uint32_t lo = v & 0xffffu, hi = v >> 16;
                        sum += (lo != 0xffffu ? lo : 0u) + (hi != 0xffffu ? hi : 0u);
                    }
            *load = sum;
        }
    } else {
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
            if (n < N)
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    const T v = cin ? (T)(int32_t)cin[k0 * CW + n * G + i] : lane_init[n * G + i];
                    st[(n * 2 * G + i) * 32] = v;
                    if (wr) cout[k0 * CW + n * G + i] = (uint32_t)(int32_t)v;
                }
        if (wr) cout[k0 * CW + SW] = (uint32_t)(int32_t)mx;
        for (int kk = k0; kk < J; ++kk) {
            const uint32_t r = rec(kk);
            const int g = (int)(r & 63u) + 1;
            SAT_ASSERT(g >= 1 && g <= G && (int)((r >> 6) & 63u) < J);
            SAT_ASSERT(rec_d || (int)(r >> 12) < c.n_opt);
            const uint32_t pay = r >> 12;
            const T rel = (!NOREL && has_release) ? release[(r >> 6) & 63u] : (T)0;
            // node finishing the job earliest, lowest node on ties
            T be = INF;
            int bn = 0;
#pragma unroll
            for (int n = 0; n < NMAX; ++n) {
                if (n < N) {
                    T t = st[(n * 2 * G + g - 1) * 32];
                    T d;
                    if (rec_d) {
                        d = (T)(int32_t)pay;
                    } else {
                        if (!((c.optmask[pay] >> n) & 1u)) t = INF;
                        d = dur[pay * N + n];
                    }
                    t = tmax(t, rel);
                    const T e = t + d;
                    if (n == 0 || e < be) { be = e; bn = n; }
                }
            }
            SAT_ASSERT(bn >= 0 && bn < N);
            T *sb = st + bn * 2 * G * 32;
            T cur[G], s[G];
#pragma unroll
            for (int i = 0; i < G; ++i) {
                cur[i] = sb[i * 32];
                s[i] = sb[(i + g) * 32];
            }
#pragma unroll
            for (int i = 0; i < G; ++i) sb[i * 32] = tmax(cur[i], tmin(s[i], be));
            mx = tmax(mx, be);
            if (wr) {
#pragma unroll
                for (int n = 0; n < NMAX; ++n)
                    if (n < N)
#pragma unroll
                        for (int q = 0; q < G; ++q) cout[(kk + 1) * CW + n * G + q] = (uint32_t)(int32_t)st[(n * 2 * G + q) * 32];
                cout[(kk + 1) * CW + SW] = (uint32_t)(int32_t)mx;
            }
        }
        if constexpr (LOAD) {
            uint64_t sum = 0;
#pragma unroll
            for (int n = 0; n < NMAX; ++n)
                if (n < N)
#pragma unroll
                    for (int i = 0; i < G; ++i) {
                        const T v = st[(n * 2 * G + i) * 32];
                        sum += (v != INF) ? (uint64_t)(int64_t)v : 0ull;
                    }
            *load = sum;
        }
    }
    return mx;
}

// One placement of a (g, d) job on the register-resident packed state (One16 layout) with a
// compile-time gang size: the shift by g is a register choice, no shared-memory round trip.
// Words are updated in ascending order: word w reads old words >= w only.
template <int G, int g>
__device__ __forceinline__ void place16_reg(uint32_t (&av)[G / 2], int32_t rel, bool has_release, int32_t d,
                                            int32_t &mx) {
    constexpr int W = G / 2;
    int32_t t = (int32_t)((av[(g - 1) / 2] >> (16 * ((g - 1) & 1))) & 0xFFFFu);
    if (has_release) t = max(t, rel);
    const int32_t e = t + d;
    const uint32_t e2 = (uint32_t)e * 0x10001u;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const int s0 = w + g / 2;                               // word holding slot 2w + g (g even)
        uint32_t sh;
        if constexpr (g % 2 == 0) {
            sh = s0 < W ? av[s0 < W ? s0 : 0] : 0xFFFFFFFFu;
        } else {
            const uint32_t lo = s0 < W ? av[s0 < W ? s0 : 0] : 0xFFFFFFFFu;
            const uint32_t hi = s0 + 1 < W ? av[s0 + 1 < W ? s0 + 1 : 0] : 0xFFFFFFFFu;
            sh = __byte_perm(lo, hi, 0x5432u);                  // slots 2w+g, 2w+g+1
        }
        av[w] = __vmaxu2(av[w], __vminu2(sh, e2));
    }
    mx = max(mx, e);
}

// k_ls move evaluation on the One16 layout.  The participating lanes walk positions in step
// (from the smallest resume point k0 in the warp; a lane joins at its own k0 with the cached
// state), so where every active lane places a job of the same gang size -- the positions a
// move leaves in place, typically most of them -- the placement runs on registers with a
// compile-time shift (one uniform branch); otherwise the generic shared-memory shift of
// schedule_records.  Same arithmetic, same result.
template <int G, typename RecF>
__device__ __forceinline__ int32_t schedule_eval16(const SchedCtx<int32_t> &c, const RecF rec, uint64_t *load,
                                                   int k0, const uint32_t *cin, int cut, int klast) {
    constexpr int W = G / 2;
    const int J = c.J;
    const int SW = W, CW = SW + 1;
    uint32_t *st16 = c.st16;
    const unsigned act = __activemask();
    const int kmin = (int)__reduce_min_sync(act, (unsigned)k0);
    uint32_t av[W];
#pragma unroll
    for (int w = 0; w < W; ++w) av[w] = 0u;
    int32_t mx = 0;
    bool dirty = true;                 // column st16 does not hold av
    bool live = true;                  // false once the move is known not to improve (early exit)
    for (int kk = kmin; kk < J; ++kk) {
        if (SAT_LS_CUT_REG > 0 && !__any_sync(act, live)) break;
        const bool on = kk >= k0 && live;
        if (kk == k0) {                // join: the cached state before position k0
#pragma unroll
            for (int w = 0; w < W; ++w) av[w] = cin ? cin[k0 * CW + w]
                                                    : (uint32_t)(uint16_t)c.lane_init[2 * w] |
                                                          ((uint32_t)(uint16_t)c.lane_init[2 * w + 1] << 16);
            mx = cin ? (int32_t)cin[k0 * CW + SW] : (int32_t)c.init_max;
        }
        const uint32_t r = on ? rec(kk) : 0u;
        const int g = (int)(r & 63u) + 1;
        SAT_ASSERT(!on || (g >= 1 && g <= G && (int)((r >> 6) & 63u) < J));
        const unsigned onm = __ballot_sync(act, on);
        const int g0 = __shfl_sync(act, g, __ffs(onm) - 1);
        const bool uni = __all_sync(act, !on || g == g0);
        const int32_t rel = (on && c.has_release) ? (int32_t)c.release[(r >> 6) & 63u] : 0;
        const int32_t d = (int32_t)(r >> 12);
        if (uni) {
            if (on) {
                switch (g0) {
#define SAT_P16(K) case K: if constexpr (K <= G) place16_reg<G, (K <= G ? K : 1)>(av, rel, c.has_release, d, mx); break;
                    SAT_P16(1) SAT_P16(2) SAT_P16(3) SAT_P16(4) SAT_P16(5) SAT_P16(6) SAT_P16(7) SAT_P16(8)
                    SAT_P16(9) SAT_P16(10) SAT_P16(11) SAT_P16(12) SAT_P16(13) SAT_P16(14) SAT_P16(15) SAT_P16(16)
                    SAT_P16(17) SAT_P16(18) SAT_P16(19) SAT_P16(20) SAT_P16(21) SAT_P16(22) SAT_P16(23) SAT_P16(24)
                    SAT_P16(25) SAT_P16(26) SAT_P16(27) SAT_P16(28) SAT_P16(29) SAT_P16(30) SAT_P16(31) SAT_P16(32)
#undef SAT_P16
                    default: break;
                }
                dirty = true;
            }
        } else if (on) {
            if (dirty) {
#pragma unroll
                for (int w = 0; w < W; ++w) st16[w * 32] = av[w];
                dirty = false;
            }
            const int gm = g - 1;
            const uint32_t selt = 0x4410u + (uint32_t)(gm & 1) * 0x22u;
            int32_t t = (int32_t)__byte_perm(st16[(gm >> 1) * 32], 0u, selt);
            if (c.has_release) t = max(t, rel);
            const int32_t e = t + d;
            const uint32_t e2 = (uint32_t)e * 0x10001u;
            const uint32_t sel = (g & 1) ? 0x5432u : 0x3210u;
            const uint32_t *src = st16 + (g >> 1) * 32;
            uint32_t wv[W + 1];
#pragma unroll
            for (int k = 0; k <= W; ++k) wv[k] = src[k * 32];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const uint32_t sh = __byte_perm(wv[k], wv[k + 1], sel);
                av[k] = __vmaxu2(av[k], __vminu2(sh, e2));
                st16[k * 32] = av[k];
            }
            mx = max(mx, e);
        }
        if (SAT_LS_CUT_REG > 0 && on) {    // early exit (see schedule_records, CUT)
            bool worse = mx > cut;
            if (SAT_LS_CUT_REG > 1 && !worse && cin && kk >= klast) {
                uint32_t diff = 0;
#pragma unroll
                for (int k = 0; k < W; ++k) diff |= __vmaxu2(av[k], cin[(kk + 1) * CW + k]) ^ av[k];
                worse = diff == 0;
            }
            if (worse) live = false;
        }
    }
    if (!live) {
        *load = 0;
        return cut + 1;
    }
    uint64_t sum = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const uint32_t lo = av[w] & 0xffffu, hi = av[w] >> 16;
        sum += (lo != 0xffffu ? lo : 0u) + (hi != 0xffffu ? hi : 0u);
    }
    *load = sum;
    return mx;
}

template <typename T, int SRC, int G, int L>
__global__ void __launch_bounds__(kCandThreads, SRC == SAT_SRC_INDEX ? 8 : (G <= 8 ? 12 : (G <= 16 ? 10 : 8)))
k_cand(CandArgs a) {
    constexpr bool MULTI = L == kLayoutMulti;
    constexpr bool P16 = L == kLayoutOne16;
    constexpr bool M16 = L == kLayoutMulti16;
    extern __shared__ __align__(16) uint8_t smem[];
    {
        const int nwords = (*reinterpret_cast<const BlobHeader *>(a.blob)).bytes / 16;
        const int4 *src = reinterpret_cast<const int4 *>(a.blob);
        int4 *dst = reinterpret_cast<int4 *>(smem);
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const BlobHeader &h = *reinterpret_cast<const BlobHeader *>(smem);
    const int J = h.J;
    const int N = (MULTI || M16) ? h.N : 1;
    GenTables tb;
    load_tables(tb, smem, h);
    const T *dur = reinterpret_cast<const T *>(smem + h.off_dur);
    const T *release = reinterpret_cast<const T *>(smem + h.off_release);
    const T *lane_init = reinterpret_cast<const T *>(smem + h.off_lane_init);   // [N][G] (blob G == G)
    const bool rec_d = a.rec_d != 0;
    const bool has_release = h.has_release != 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr bool kIndex = SRC == SAT_SRC_INDEX;
    uint8_t *wbase = smem + h.bytes + warp * cand_warp_bytes(J, N, G, cand_slot_bytes<T, L>(), kIndex);
    SAT_ASSERT(N >= 1 && N * G <= 32 && J >= 1 && J <= SAT_MAX_JOBS);
    uint32_t *rec = reinterpret_cast<uint32_t *>(wbase) + lane;          // [J][32]
    uint8_t *opt = wbase + J * 128 + lane;                               // [J][32] (index source)
    uint8_t *ord = opt + J * 32;                                         // [J][32]
    T *st = reinterpret_cast<T *>(wbase + J * 128 + (kIndex ? J * 64 : 0)) + lane;   // [N][2G][32]
    uint32_t *st16 = reinterpret_cast<uint32_t *>(st);                               // [G][32] words

    const T INF = TimeTraits<T>::inf();
    if constexpr (P16 || M16) {
        for (int n = 0; n < N; ++n)
#pragma unroll
            for (int w = G / 2; w < G; ++w) st16[(n * G + w) * 32] = 0xffffffffu;
    } else {
        for (int n = 0; n < N; ++n)
#pragma unroll
            for (int i = G; i < 2 * G; ++i) st[(n * 2 * G + i) * 32] = INF;
    }
    const T init_max = sizeof(T) == 4 ? (T)h.init_max_i32 : (T)h.init_max_f64;
    SchedCtx<T> sc{st, st16, lane_init, release, dur, tb.optmask, J, N, h.n_opt, rec_d, has_release, init_max, INF};

    T best_ms = INF;
    uint64_t best_ix = ~0ull;

    const uint64_t total = a.hi - a.lo;
    // warps take chunks of 32 x per_lane candidates from a cursor (thread: per_lane
    // consecutive ids, so the index source can advance instead of re-decoding)
    const int per_lane = a.per_lane;
    const uint64_t chunk = 32ull * (uint64_t)per_lane;
    const uint64_t nchunks = (total + chunk - 1) / chunk;
    auto next_chunk = [&]() -> uint64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(a.cursor, 1ull);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    for (uint64_t c = next_chunk(); c < nchunks; c = next_chunk()) {
        for (int k = 0; k < per_lane; ++k) {
            const uint64_t off = c * chunk + (uint64_t)lane * per_lane + k;
            if (off >= total) break;
            const uint64_t id = a.lo + off;
            // ---- decode into this thread's record column ----
            if (kIndex) {
                if (k == 0) decode_index(id, J, tb.radix, opt, ord);
                else advance_index(J, tb.radix, opt, ord);
                for (int kk = 0; kk < J; ++kk) {
                    const int job = ord[kk * 32];
                    rec[kk * 32] = rec_for(tb, job, opt[job * 32]);
                }
            } else if (SRC == SAT_SRC_SUBSTREAM) {
                decode_stream(mix64((a.seed ^ id) + kGolden), tb, rec);
            } else {
                decode_stream(a.seed + id, tb, rec);
            }
            const T mx = has_release ? schedule_records<T, G, L>(sc, RecCol{rec})
                                     : schedule_records<T, G, L, false, RecCol, false, true>(sc, RecCol{rec});
            if (key_less(mx, id, best_ms, best_ix)) {
                best_ms = mx;
                best_ix = id;
            }
        }
    }

    // ---- warp -> block -> grid argmin ----
    for (int x = 16; x >= 1; x >>= 1) {
        const T oms = __shfl_xor_sync(0xffffffffu, best_ms, x);
        const uint64_t oix = shfl_u64(best_ix, lane ^ x);
        if (key_less(oms, oix, best_ms, best_ix)) { best_ms = oms; best_ix = oix; }
    }
    __shared__ T s_ms[kCandWarps];
    __shared__ uint64_t s_ix[kCandWarps];
    if (lane == 0) { s_ms[warp] = best_ms; s_ix[warp] = best_ix; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kCandWarps; ++w)
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

// ---------------------------------------------------------------------------
// k_ls: local search from sampled starting points (one walker per warp, one move per lane)
// ---------------------------------------------------------------------------
// Walker w starts at candidate w of the stream (the sampled search's candidate w) and
// descends: moves in a fixed order -- [0, M1) swap positions a < b; [M1, M1+M2) job j takes
// option o' != its own; [M1+M2, M) the job at position a moves to position b -- are scanned
// 32 at a time (a lane per move, each scheduled to its makespan and load = sum of the final
// GPU free times); the first round holding an improvement of (makespan, load) applies its
// best move (lowest objective, then lowest move id) and the scan restarts at move 0.  A
// full scan without improvement, or max_rounds rounds, ends the walk; the walker's result
// is (makespan, w).  oracle/oracle.c restates the same walk with its per-GPU scheduler.
struct LsArgs {
    const uint8_t *blob;
    uint64_t lo, hi;            // walkers [lo, hi)
    uint64_t seed;
    int32_t max_rounds;
    int32_t rec_d;
    int32_t stop_ms;            // a walker ends once its makespan is <= stop_ms (-1: never)
    int32_t idx_bits;
    int32_t group_warps;        // warps per walker (the kernel's K: 1, 4 or 8): rounds evaluated at once
    sat_best_t *best;
    unsigned long long *cursor;
    unsigned long long *rounds; // rounds of 32 moves executed, summed over walkers (zeroed before)
    uint8_t *state_out;         // [hi - lo][2J] final options then order of every walker (abandoned: untouched), or null
    // greedy starts (SAT_SRC_GREEDY): every job takes its least-area option gopt[j]; the order
    // is by the noisy key gdur[j] x (2^17 + u_j) descending (ties: lower job first), u_j the
    // top 16 bits of the j-th draw of the walker's stream -- longest jobs first, perturbed
    int32_t greedy;
    uint8_t gopt[64];
    uint32_t gdur[64];
};

// the greedy start's order key of job j (LsArgs::greedy); s0 = the walker's stream state
__host__ __device__ inline uint64_t ls_greedy_key(uint32_t gdur, uint64_t s0, int j) {
    const uint64_t u = mix64(s0 + (uint64_t)(j + 1) * kGolden) >> 48;
    return (uint64_t)gdur * (131072ull + u);
}

// bytes of one block's region: every warp's free-time columns (a move's records are computed
// per position from the walker's, no per-warp record column), then per walker its options /
// order / job positions (3 x 64 bytes), its current records (64 words) and its prefix cache
__host__ __device__ inline int ls_walker_bytes(int J, int cache_state_words) {
    return 192 + 256 + (J + 1) * (cache_state_words + 1) * 4;
}
__host__ __device__ inline int ls_warp_bytes(int J, int N, int G, int slot_bytes) {
    return cand_warp_bytes(J, N, G, slot_bytes, false) - J * 128;
}
// warps per k_ls block: 4, or 8 when one walker takes 8 warps
__host__ __device__ constexpr int ls_block_warps(int K) { return K > kCandWarps ? K : kCandWarps; }
__host__ __device__ inline int ls_block_bytes(int J, int N, int G, int slot_bytes, int cache_state_words, int K) {
    return ls_block_warps(K) * ls_warp_bytes(J, N, G, slot_bytes) +
           (ls_block_warps(K) / K) * ls_walker_bytes(J, cache_state_words);
}

// neighbour of (opt, ord) under move m: source position of position k, and the option override
struct LsMove {
    int kind;      // 0 swap, 1 option, 2 insertion
    int a, b;      // positions (swap / insertion) or (job, option) for kind 1
};

__device__ __forceinline__ LsMove ls_decode_move(int m, int J, int M1, int M2, const int32_t *radix,
                                                 const uint8_t *wopt) {
    LsMove mv;
    if (m < M1) {
        int a = 0, rest = m;
        while (rest >= J - 1 - a) { rest -= J - 1 - a; ++a; }
        mv.kind = 0; mv.a = a; mv.b = a + 1 + rest;
    } else if (m < M1 + M2) {
        int rest = m - M1, j = 0;
        while (rest >= radix[j] - 1) { rest -= radix[j] - 1; ++j; }
        mv.kind = 1; mv.a = j; mv.b = rest < (int)wopt[j] ? rest : rest + 1;
    } else {
        const int rest = m - M1 - M2;
        const int a = rest / (J - 1), bi = rest - a * (J - 1);
        mv.kind = 2; mv.a = a; mv.b = bi < a ? bi : bi + 1;
    }
    return mv;
}

__device__ __forceinline__ int ls_src(const LsMove &mv, int k) {
    if (mv.kind == 0) return k == mv.a ? mv.b : (k == mv.b ? mv.a : k);
    if (mv.kind == 1) return k;
    if (mv.a < mv.b) return (k < mv.a || k > mv.b) ? k : (k == mv.b ? mv.a : k + 1);
    return (k < mv.b || k > mv.a) ? k : (k == mv.b ? mv.a : k - 1);
}

// the neighbour's record at position k: the walker's record at the source position, or (option
// move) the moved job's record with its new option at the job's own position
struct RecMove {
    const uint32_t *crec;                        // walker's current records [J] (shared by its warps)
    LsMove mv;
    int spk;                                     // option move: the job's position (-1: none)
    uint32_t sprec;
    __device__ __forceinline__ uint32_t operator()(int k) const {
        return k == spk ? sprec : crec[ls_src(mv, k)];
    }
};

struct RecWalker {
    const uint32_t *crec;
    __device__ __forceinline__ uint32_t operator()(int k) const { return crec[k]; }
};

// One walker per group of K = group_warps warps (K = 1: a walker per warp; K = kCandWarps: a
// walker per block).  The group's warps evaluate consecutive rounds of the current scan at
// once (warp w of the group: round q + w); the first of them, in scan order, holding an
// improvement is the round the sequential walk would have applied, so the walk -- moves,
// tie-breaks, round count -- is exactly the one-round-at-a-time walk (oracle.c restates
// that), in ~1/K of the sequential steps when scans are long (the critical path of a wave is
// its longest walk); K = 1 keeps the most walkers in flight when throughput matters.
template <int SRC, int G, int L, int K>
__global__ void __launch_bounds__(ls_block_warps(K) * 32, K >= 8 ? 32 / K : 8)   // <= 64 registers
k_ls(LsArgs a) {
    using T = int32_t;
    static_assert(K == 1 || K == 2 || K == kCandWarps || K == 8 || K == 16 || K == 32, "warps per walker");
    constexpr int BW = ls_block_warps(K);                // warps per block
    extern __shared__ __align__(16) uint8_t smem[];
    {
        const int nwords = (*reinterpret_cast<const BlobHeader *>(a.blob)).bytes / 16;
        const int4 *src = reinterpret_cast<const int4 *>(a.blob);
        int4 *dst = reinterpret_cast<int4 *>(smem);
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const BlobHeader &h = *reinterpret_cast<const BlobHeader *>(smem);
    const int J = h.J;
    const int N = (L == kLayoutMulti || L == kLayoutMulti16) ? h.N : 1;
    GenTables tb;
    load_tables(tb, smem, h);
    const T *dur = reinterpret_cast<const T *>(smem + h.off_dur);
    const T *release = reinterpret_cast<const T *>(smem + h.off_release);
    const T *lane_init = reinterpret_cast<const T *>(smem + h.off_lane_init);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = warp / K, gw = warp - grp * K;                 // walker group, warp within it
    const bool leader = gw == 0 && lane == 0;
    const int SW = cache_state_words<G, L>(N);
    const int wbytes = ls_warp_bytes(J, N, G, cand_slot_bytes<T, L>());
    uint8_t *wbase = smem + h.bytes + warp * wbytes;
    T *st = reinterpret_cast<T *>(wbase) + lane;
    uint32_t *st16 = reinterpret_cast<uint32_t *>(st);
    uint8_t *wopt = smem + h.bytes + BW * wbytes + grp * ls_walker_bytes(J, SW);   // [64] walker state
    uint8_t *word = wopt + 64;                                                           // [64]
    uint8_t *wpos = word + 64;                                                           // [64] job -> position
    uint32_t *crec = reinterpret_cast<uint32_t *>(wpos + 64);                           // [64] records by position
    uint32_t *cache = crec + 64;                                                         // [J + 1][SW + 1]
    __shared__ uint64_t s_key[BW];                     // per warp: its round's best (objective, move)
    __shared__ int s_move[BW];
    __shared__ unsigned long long s_walker[BW];        // per group
    __shared__ uint64_t s_cur_key[BW];
    __shared__ int s_beaten[BW];
    uint64_t *g_key = s_key + grp * K;
    int *g_move = s_move + grp * K;
    // group barrier: the warp itself (K = 1) or a named barrier over the group's K warps
    auto gsync = [&]() {
        if constexpr (K == 1) __syncwarp();
        else if constexpr (K == BW) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(K * 32) : "memory");
    };
    const T INF = SAT_INF_I32;
    if constexpr (L == kLayoutOne16 || L == kLayoutMulti16) {
        for (int n = 0; n < N; ++n)
            for (int w = G / 2; w < G; ++w) st16[(n * G + w) * 32] = 0xffffffffu;
    } else {
        for (int n = 0; n < N; ++n)
            for (int i = G; i < 2 * G; ++i) st[(n * 2 * G + i) * 32] = INF;
    }
    SchedCtx<T> sc{st, st16, lane_init, release, dur, tb.optmask, J, N, h.n_opt, a.rec_d != 0,
                   h.has_release != 0, (T)h.init_max_i32, INF};
    int M2 = 0;
    for (int j = 0; j < J; ++j) M2 += tb.radix[j] - 1;
    const int M1 = J * (J - 1) / 2, M = M1 + M2 + J * (J - 1);
    // the prefix cache pays off only on long orders (measured: +10 % at 64 jobs, -15 % at 16)
    const bool use_cache = J >= 24;

    // keys: (makespan, rounds the walk scanned, walker) lexicographic -- among walkers ending at
    // the same makespan the one that got there in the fewest rounds wins (then the lowest id), so
    // a running walker that has already scanned as many rounds as a published key at the bound
    // can no longer win and is abandoned (the wave ends when its fastest walker reaches the bound
    // plus the rounds every other walker needs to fall behind it)
    constexpr int RB = SAT_LS_ROUND_BITS;
    const int ib = a.idx_bits;
    auto walker_key = [&](T ms, int r, uint64_t w) -> uint64_t {
        const uint64_t rr = (uint64_t)min(r, (1 << RB) - 1);
        return ((uint64_t)(uint32_t)ms << (ib + RB)) | (rr << ib) | w;
    };
    // published key at <= stop_ms with at most `r` rounds: a still-running walker (its final
    // round count will exceed r) cannot beat it
    auto beaten_at = [&](int r) -> bool {
        const unsigned long long k = *reinterpret_cast<volatile unsigned long long *>(&a.best->hi);
        return k != ~0ull && (int64_t)(k >> (ib + RB)) <= (int64_t)a.stop_ms &&
               (int64_t)((k >> ib) & ((1ull << RB) - 1ull)) <= (int64_t)r;
    };
    uint64_t best_key = ~0ull;             // group leader: the group's best walker key
    const uint64_t total = a.hi - a.lo;
#ifdef SAT_LS_PROFILE
    // steps, improving steps, cycles evaluating (+ barrier wait), cycles applying, sum of the
    // improving round's position in its step -- summed over walkers (a.rounds[1..5])
    long long prof[5] = {0, 0, 0, 0, 0};
#endif
    for (;;) {
        if (leader) s_walker[grp] = atomicAdd(a.cursor, 1ull);
        gsync();
        const uint64_t wk = s_walker[grp];
        if (wk >= total) break;
        const uint64_t id = a.lo + wk;
        const uint64_t s0 = SRC == SAT_SRC_SUBSTREAM ? mix64((a.seed ^ id) + kGolden) : a.seed + id;
        if (a.greedy) {            // greedy start: least-area options, perturbed longest-first order
            if (gw == 0) {
                for (int j = lane; j < J; j += 32) wopt[j] = a.gopt[j];
                const uint64_t k0 = lane < J ? ls_greedy_key(a.gdur[lane], s0, lane) : 0;
                const uint64_t k1 = lane + 32 < J ? ls_greedy_key(a.gdur[lane + 32], s0, lane + 32) : 0;
                int r0 = 0, r1 = 0;        // rank = jobs ahead: larger key, or equal key and lower id
                for (int i = 0; i < J; ++i) {
                    const uint64_t ki = __shfl_sync(0xffffffffu, i < 32 ? k0 : k1, i & 31);
                    r0 += ki > k0 || (ki == k0 && i < lane);
                    r1 += ki > k1 || (ki == k1 && i < lane + 32);
                }
                if (lane < J) { word[r0] = (uint8_t)lane; wpos[lane] = (uint8_t)r0; }
                if (lane + 32 < J) { word[r1] = (uint8_t)(lane + 32); wpos[lane + 32] = (uint8_t)r1; }
            }
        } else if (leader) {       // the walker's start: candidate id of the stream (plan_random's draw order)
            Stream s{s0};
            for (int j = 0; j < J; ++j) wopt[j] = (uint8_t)s.below((uint32_t)tb.radix[j], tb.mods);
            for (int k = 0; k < J; ++k) word[k] = (uint8_t)k;
            for (int i = J - 1; i >= 1; --i) {
                const int k = (int)s.below((uint32_t)(i + 1), tb.mods);
                const uint8_t t = word[i]; word[i] = word[k]; word[k] = t;
            }
            for (int k = 0; k < J; ++k) wpos[word[k]] = (uint8_t)k;
        }
        gsync();
        if (gw == 0) {
            for (int k = lane; k < J; k += 32) { const int job = word[k]; crec[k] = rec_for(tb, job, wopt[job]); }
            __syncwarp();
        }
        gsync();
        if (gw == 0) {             // objective of the start; lane 0 fills the prefix cache
            uint64_t load = 0;
            const T c0 = schedule_records<T, G, L, true>(sc, RecWalker{crec}, &load, 0, nullptr,
                                                        use_cache ? cache : nullptr, lane == 0);
            if (lane == 0) s_cur_key[grp] = ((uint64_t)(uint32_t)c0 << 34) | load;
        }
        gsync();
        uint64_t cur_key = s_cur_key[grp];
        T cur = (T)(cur_key >> 34);
        int rounds = 0;
        // Early stop (stop_ms = the problem's lower bound): the makespan never rises along a
        // walk, so a walker at stop_ms has its final key (stop_ms, rounds, id) and ends there; a
        // still-running walker that has scanned at least as many rounds as a published key at
        // <= stop_ms cannot win and is abandoned.  Neither changes the search result.
        bool abandoned = false;
        for (;;) {
            if (cur <= a.stop_ms) break;
            bool improved = false;
            for (int q = 0;; q += K) {      // rounds q .. q+K-1 of this scan, one per warp
#ifdef SAT_LS_PROFILE
                const long long prof_t0 = clock64();
#endif
                const int r0 = (q + gw) * 32;
                const bool valid = r0 < M && rounds + gw < a.max_rounds;
                uint64_t bk = ~0ull;
                int bm = 0x7fffffff;
                if (valid) {
                    const int m = r0 + lane;
                    if (m < M) {
                        const LsMove mv = ls_decode_move(m, J, M1, M2, tb.radix, wopt);
                        // positions before the first changed one schedule exactly as the current
                        // candidate: resume from the prefix cache there
                        const int kpos = mv.kind == 1 ? (int)wpos[mv.a] : -1;
                        const int k0 = !use_cache ? 0 : (mv.kind == 1 ? kpos : min(mv.a, mv.b));
                        const RecMove rec{crec, mv, kpos, mv.kind == 1 ? rec_for(tb, mv.a, mv.b) : 0u};
                        uint64_t ld = 0;
                        T ms;
                        // register shifts pay off on wide nodes (G = 32: ~110 instructions per
                        // shared-memory placement) in the 8-warp walker (cfg5 13.2 -> 11.7 ms); with
                        // 1 or 4 warps per walker, or at G = 8, the warp votes cost more than they save
                        // (profiles/r01g_ls_group_sweep.txt)
                        // last position the move changes: past it, the records are the current
                        // candidate's (the dominance exit applies)
                        const int klast = mv.kind == 1 ? kpos : max(mv.a, mv.b);
                        if constexpr (L == kLayoutOne16 && G >= 16 && K >= 8)
                            ms = schedule_eval16<G>(sc, rec, &ld, k0, use_cache ? cache : nullptr, cur, klast);
                        else if constexpr (L == kLayoutOne16 || L == kLayoutOne)
                            ms = schedule_records<T, G, L, true, RecMove, true>(
                                sc, rec, &ld, k0, use_cache ? cache : nullptr, nullptr, false, cur, klast);
                        else
                            ms = schedule_records<T, G, L, true>(sc, rec, &ld, k0, use_cache ? cache : nullptr);
                        bk = ((uint64_t)(uint32_t)ms << 34) | ld;
                        bm = m;
                    }
                    // warp argmin of (objective, move id)
                    for (int x = 16; x >= 1; x >>= 1) {
                        const uint64_t ok = shfl_u64(bk, lane ^ x);
                        const int om = __shfl_xor_sync(0xffffffffu, bm, x);
                        if (ok < bk || (ok == bk && om < bm)) { bk = ok; bm = om; }
                    }
                }
                // every thread takes the same decision: the first valid round (scan order) with
                // an improvement, else all valid rounds were scanned without one
                int first = -1, nvalid = 0;
                uint64_t nk = bk;
                int nm = bm;
                if constexpr (K == 1) {               // the warp's own round (all lanes hold it)
                    nvalid = valid ? 1 : 0;
                    if (valid && bk < cur_key) first = 0;
                } else {
                    if (lane == 0) { g_key[gw] = bk; g_move[gw] = bm; }
                    gsync();
                    for (int w = 0; w < K; ++w) {
                        if (!((q + w) * 32 < M && rounds + w < a.max_rounds)) break;
                        ++nvalid;
                        if (g_key[w] < cur_key) { first = w; break; }
                    }
                    if (first >= 0) { nk = g_key[first]; nm = g_move[first]; }
                }
#ifdef SAT_LS_PROFILE
                const long long prof_t1 = clock64();
                if (leader) { prof[0] += 1; prof[2] += prof_t1 - prof_t0; }
#endif
                if (first >= 0) {
                    // positions before the first one the move changes keep their records and
                    // their prefix-cache entries (decoded before the leader rewrites the walker)
                    const LsMove amv = ls_decode_move(nm, J, M1, M2, tb.radix, wopt);
                    const int kc = amv.kind == 1 ? (int)wpos[amv.a] : min(amv.a, amv.b);
                    gsync();                          // every thread has read the slots
                    if (leader) {
                        const LsMove &mv = amv;
                        // still running after this move (not yet at stop_ms) and already behind a
                        // published key at the bound: abandoned
                        s_beaten[grp] = a.stop_ms >= 0 && (T)(nk >> 34) > a.stop_ms && beaten_at(rounds + first + 1);
                        if (mv.kind == 0) {
                            const uint8_t t = word[mv.a]; word[mv.a] = word[mv.b]; word[mv.b] = t;
                        } else if (mv.kind == 1) {
                            wopt[mv.a] = (uint8_t)mv.b;
                        } else {
                            const uint8_t x = word[mv.a];
                            if (mv.a < mv.b) for (int k = mv.a; k < mv.b; ++k) word[k] = word[k + 1];
                            else for (int k = mv.a; k > mv.b; --k) word[k] = word[k - 1];
                            word[mv.b] = x;
                        }
                        for (int k = 0; k < J; ++k) wpos[word[k]] = (uint8_t)k;
                    }
                    gsync();
                    if (gw == 0) {                  // the new current candidate's records (and prefix cache)
                        for (int k = kc + lane; k < J; k += 32) { const int job = word[k]; crec[k] = rec_for(tb, job, wopt[job]); }
                        __syncwarp();
                        if (use_cache)
                            schedule_records<T, G, L, false>(sc, RecWalker{crec}, nullptr, kc, cache, cache, lane == 0);
                    }
                    gsync();
#ifdef SAT_LS_PROFILE
                    if (leader) { prof[1] += 1; prof[3] += clock64() - prof_t1; prof[4] += first; }
#endif
                    if (s_beaten[grp]) { abandoned = true; break; }
                    cur_key = nk;
                    cur = (T)(nk >> 34);
                    rounds += first + 1;
                    improved = true;
                    break;
                }
                rounds += nvalid;
                if (a.stop_ms >= 0) {                 // fallen behind a published key at the bound?
                    if (leader) s_beaten[grp] = beaten_at(rounds);
                    gsync();                          // (also: slots are rewritten by the next rounds)
                    const bool beaten = s_beaten[grp] != 0;
                    gsync();
                    if (beaten) { abandoned = true; break; }
                } else if constexpr (K > 1) {
                    gsync();                          // slots are rewritten by the next rounds
                }
                if (nvalid < K) break;                // scan exhausted or round budget spent
            }
            if (!improved || rounds >= a.max_rounds) break;
        }
        if (leader) {
            const uint64_t wkey = walker_key(cur, rounds, id);
            if (!abandoned && wkey < best_key) {
                best_key = wkey;
                if (cur <= a.stop_ms)      // publish now: walkers behind it are abandoned
                    atomicMin(reinterpret_cast<unsigned long long *>(&a.best->hi), (unsigned long long)wkey);
            }
            atomicAdd(a.rounds, (unsigned long long)rounds + 1ull);   // + the start's round
#ifdef SAT_LS_PROFILE
            for (int i = 0; i < 5; ++i) { atomicAdd(a.rounds + 1 + i, (unsigned long long)prof[i]); prof[i] = 0; }
#endif
            if (a.state_out && !abandoned) {      // walker wk's final candidate
                uint8_t *so = a.state_out + wk * (uint64_t)(2 * J);
                for (int j = 0; j < J; ++j) so[j] = wopt[j];
                for (int k = 0; k < J; ++k) so[J + k] = word[k];
            }
        }
        gsync();
    }
    if (leader && best_key != ~0ull)
        atomicMin(reinterpret_cast<unsigned long long *>(&a.best->hi), (unsigned long long)best_key);
}

template <int SRC>
int launch_ls(const sat_problem_t *p, LsArgs a, void *d_ws, size_t ws_bytes, cudaStream_t stream);

// host launcher for one (T, SRC) pair; dispatches on the padded node size and layout
template <typename T, int SRC>
int launch_cand(const sat_problem_t *p, CandArgs a, uint64_t n_cand, void *d_ws, size_t ws_bytes,
                cudaStream_t stream);

}  // namespace sat
