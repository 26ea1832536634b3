// sat_tree.cuh -- k_tree<G>: the prefix-shared exhaustive walk (single node, grid time),
// specialised on the node's exact GPU count G.  Instantiated by sat_tree_g.cu.
#pragma once

#include "sat_common.cuh"

namespace sat {

// Merge of a register-resident sorted vector A with a compile-time gang size g;
// result goes to the lane's column of smem (stride 32 words).
template <int G, int g>
__device__ __forceinline__ void merge_store(const int32_t (&A)[G], int32_t d, int32_t *out) {
    const int32_t e = A[g - 1] + d;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        int32_t v;
        if (i + g < G) v = min(A[(i + g < G) ? i + g : 0], e);
        else v = e;
        if (i >= g) v = max(A[i], v);
        out[i * 32] = v;
    }
}

template <int G>
__device__ __forceinline__ void merge_dispatch(int g, const int32_t (&A)[G], int32_t d, int32_t *out) {
    switch (g) {
#define SAT_CASE(K) case K: if constexpr (K <= G) merge_store<G, (K <= G ? K : 1)>(A, d, out); break;
        SAT_CASE(1) SAT_CASE(2) SAT_CASE(3) SAT_CASE(4) SAT_CASE(5) SAT_CASE(6) SAT_CASE(7) SAT_CASE(8)
        SAT_CASE(9) SAT_CASE(10) SAT_CASE(11) SAT_CASE(12) SAT_CASE(13) SAT_CASE(14) SAT_CASE(15) SAT_CASE(16)
        SAT_CASE(17) SAT_CASE(18) SAT_CASE(19) SAT_CASE(20) SAT_CASE(21) SAT_CASE(22) SAT_CASE(23) SAT_CASE(24)
        SAT_CASE(25) SAT_CASE(26) SAT_CASE(27) SAT_CASE(28) SAT_CASE(29) SAT_CASE(30) SAT_CASE(31) SAT_CASE(32)
#undef SAT_CASE
        default: break;
    }
}


// Value of the best candidate below one (first job j1 with option of gang g, then the
// second job): with B = the state after j1, the last job's best end over its options is
// min_k (B[k] + D2[k]) where D2[k] = least duration among its options of gang k+1, and
// the makespan is max(B[G-1], that).  B is never materialised: each slot costs at most a
// min, a max and one fused add-min (VIADDMNMX).
template <int G, int g>
__device__ __forceinline__ int32_t group_value(const int32_t (&A)[G], int32_t d, const int32_t (&D2)[G]) {
    const int32_t e = A[g - 1] + d;
    int32_t m = SAT_INF_I32, blast = e;
#pragma unroll
    for (int k = 0; k < G; ++k) {
        int32_t b = (k + g < G) ? min(A[(k + g < G) ? k + g : 0], e) : e;
        if (k >= g) b = max(A[k], b);
        m = min(m, b + D2[k]);
        if (k == G - 1) blast = b;
    }
    return max(blast, m);
}

// All gang sizes of the first job at compile time: D1[g-1] = least duration of its options
// with gang g (INF: none), so only existing gangs cost work (one uniform branch each).
template <int G, int g>
__device__ __forceinline__ void side_fold(const int32_t (&A)[G], const int32_t (&D1)[G], const int32_t (&D2)[G],
                                          int32_t &v) {
    if constexpr (g <= G) {
        if (D1[g - 1] < SAT_INF_I32) v = min(v, group_value<G, g>(A, D1[g - 1], D2));
        side_fold<G, g + 1>(A, D1, D2, v);
    }
}

// ---- packed pair pass: the same value on two 16-bit slots per word ----
// P0[w] = (A[2w], A[2w+1]), P1[w] = (A[2w+1], A[2w+2]) (slots >= G: kTreeInf16), so the
// shift by a compile-time g is a register choice (P0 for even g, P1 for odd g); per word
// VIMNMX.U16x2 min + max and one VIADDMNMX.U16x2 cover two slots.  The group's makespan
// max(B[G-1], min_k(B[k] + D2[k])) distributes over the two halves of the running min:
// max(bl, min(h0, h1)) = min(max(bl, h0), max(bl, h1)), so halves are folded once per node.
template <int G>
struct Pk { static constexpr int W = (G + 1) / 2; };

// slot k of a packed vector, replicated into both halves
template <int k>
__device__ __forceinline__ uint32_t rep16(const uint32_t *P0) {
    return __byte_perm(P0[k / 2], 0u, (k & 1) ? 0x3232u : 0x1010u);
}

// B = the state after a (g, e) placement, as 16-bit pairs: word w holds slots 2w, 2w+1 of
// max(A[k], min(A[k+g], e)) (slots k < g: min(A[k+g], e); A[k+g] = INF past the node)
template <int G, int g>
__device__ __forceinline__ void merge16(const uint32_t (&P0)[Pk<G>::W], const uint32_t (&P1)[Pk<G>::W],
                                        uint32_t e2, uint32_t (&B)[Pk<G>::W]) {
    constexpr int W = Pk<G>::W;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const int src = 2 * w + g;                                // shifted slot of the low half
        uint32_t b;
        if (src >= G) {
            b = e2;                                               // min(INF, e)
        } else {
            const uint32_t sh = (g & 1) ? P1[(src - 1) / 2 < W ? (src - 1) / 2 : 0] : P0[src / 2 < W ? src / 2 : 0];
            b = __vminu2(sh, e2);
        }
        if (2 * w + 1 >= g) b = __vmaxu2(P0[w], b);               // slots k >= g keep max(A[k], .)
        B[w] = b;
    }
}

// P1 (slots 2w+1, 2w+2) of a packed vector from its P0
template <int G>
__device__ __forceinline__ void odd_pairs(const uint32_t (&P0)[Pk<G>::W], uint32_t (&P1)[Pk<G>::W]) {
    constexpr int W = Pk<G>::W;
#pragma unroll
    for (int w = 0; w < W; ++w) P1[w] = __byte_perm(P0[w], w + 1 < W ? P0[w + 1 < W ? w + 1 : 0] : kTreeInf16, 0x5432u);
}

template <int G, int g>
__device__ __forceinline__ uint32_t group_value16(const uint32_t (&P0)[Pk<G>::W], const uint32_t (&P1)[Pk<G>::W],
                                                  uint32_t d2, const uint32_t (&D2)[Pk<G>::W]) {
    constexpr int W = Pk<G>::W;
    const uint32_t e2 = rep16<g - 1>(P0) + d2;                   // e in both halves (no carry: e < 2^15)
    uint32_t B[W];
    merge16<G, g>(P0, P1, e2, B);
    uint32_t m2 = 0xFFFFFFFFu;
#pragma unroll
    for (int w = 0; w < W; ++w) m2 = __viaddmin_u16x2(B[w], D2[w], m2);
    return __vmaxu2(m2, rep16<G - 1>(B));
}

template <int G, int g>
__device__ __forceinline__ void side_fold16(const uint32_t (&P0)[Pk<G>::W], const uint32_t (&P1)[Pk<G>::W],
                                            const int32_t *D1, const uint32_t (&D2)[Pk<G>::W], uint32_t &v2) {
    if constexpr (g <= G) {
        const int32_t d = D1[g - 1];                               // uniform (parameter block)
        if (d < SAT_INF_I32) v2 = __vminu2(v2, group_value16<G, g>(P0, P1, (uint32_t)d * 0x10001u, D2));
        side_fold16<G, g + 1>(P0, P1, D1, D2, v2);
    }
}

// value of a pair node from its packed state: min over both orders of the two jobs
template <int G>
__device__ __forceinline__ int32_t pair_value16(const uint32_t (&P0)[Pk<G>::W], const uint32_t (&P1)[Pk<G>::W],
                                                const int32_t *sdg, int ja, int jb,
                                                const uint32_t (&Pa)[Pk<G>::W], const uint32_t (&Pb)[Pk<G>::W]) {
    uint32_t v2 = 0xFFFFFFFFu;
    side_fold16<G, 1>(P0, P1, sdg + ja * 32, Pb, v2);
    side_fold16<G, 1>(P0, P1, sdg + jb * 32, Pa, v2);
    return (int32_t)min(v2 & 0xFFFFu, v2 >> 16);
}

// Exact pass over a pair node: per (first job, option) group, the makespan and the lowest
// option of the last job reaching it, with the full candidate index for the tie-break.
template <int G>
__device__ __noinline__ void tree_pair_exact(const TreeParams &p, const int32_t *U, int32_t *B, int ja,
                                             int jb, uint64_t base, LaneBest &lb) {
    int32_t A[G];                                    // reloaded from the column: no spill of A per node
#pragma unroll
    for (int i = 0; i < G; ++i) A[i] = U[i * 32];
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        const int j1 = side ? jb : ja;
        const int j2 = side ? ja : jb;
        const uint64_t base1 = base + (uint64_t)side;     // Lehmer digit of position J-2
        const int r1 = p.radix[j1], ob1 = p.optbase[j1];
        const int r2 = p.radix[j2], ob2 = p.optbase[j2];
        const uint64_t w1 = p.wJ[j1], w2 = p.wJ[j2];
#pragma unroll 1
        for (int o1 = 0; o1 < r1; ++o1) {
            merge_dispatch<G>(p.optg[ob1 + o1], A, p.optd[ob1 + o1], B);
            const int32_t blast = B[(G - 1) * 32];
            int32_t ms = SAT_INF_I32;
            int best_o2 = 0;
#pragma unroll 1
            for (int o2 = 0; o2 < r2; ++o2) {
                const int32_t v = max(B[p.optoff[ob2 + o2]] + p.optd[ob2 + o2], blast);
                if (v < ms) { ms = v; best_o2 = o2; }
            }
            if (ms <= lb.ms) {
                const uint64_t ix = base1 + (uint64_t)o1 * w1 + (uint64_t)best_o2 * w2;
                if (ms < lb.ms || ix < lb.ix) { lb.ms = ms; lb.ix = ix; }
            }
        }
    }
}

// A pair node's candidates have indices >= base and makespans >= v: it can only matter
// when (v, base) ties or beats the lane's best and, in the full scan, the best any warp has
// published so far (keys order by makespan, then index; an unset index is ~0, so ties with
// a seed bound pass).  The published key is read only for nodes that pass the lane test;
// bound-and-prune skips that read (its subtrees were already cut against the published
// bound, and most of its pair nodes pass the lane test).
template <bool PUB>
__device__ __forceinline__ bool pair_needs_exact(const TreeParams &p, int32_t v, uint64_t base,
                                                 const LaneBest &lb) {
    if (!(v < lb.ms || (v == lb.ms && base <= lb.ix))) return false;
    if constexpr (!PUB) return true;
    const unsigned long long hi = *reinterpret_cast<volatile unsigned long long *>(&p.best->hi);
    if (hi == ~0ull) return true;
    const int32_t pms = (int32_t)(hi >> p.idx_bits);
    return v < pms || (v == pms && base <= (hi & ((1ull << p.idx_bits) - 1ull)));
}

// Two jobs left (a < b): both orders x all options of the first x all options of the
// second.  Fast value pass in registers (per-gang minimum durations are exact for the
// value: a shorter first job never hurts, a shorter last job never hurts); the exact pass
// only runs when this pair node can tie or beat the lane's best.
template <int G, bool BNB>
__device__ __forceinline__ void tree_pair(const TreeParams &p, const int32_t *U, int32_t *B,
                                          const int32_t *sdg, uint32_t rem, uint64_t base, bool valid,
                                          LaneBest &lb) {
    int32_t A[G];
    const int ja = __ffs(rem) - 1;
    const int jb = 31 - __clz(rem);
#pragma unroll
    for (int i = 0; i < G; ++i) A[i] = U[i * 32];
    int32_t v = SAT_INF_I32;
    if constexpr (G <= kTreePackMaxG && G >= 2) {
        if (p.packed) {
            constexpr int W = Pk<G>::W;
            uint32_t P0[W], P1[W], Pa[W], Pb[W];
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const uint32_t a0 = (uint32_t)A[2 * w];
                const uint32_t a1 = 2 * w + 1 < G ? (uint32_t)A[2 * w + 1 < G ? 2 * w + 1 : 0] : kTreeInf16;
                P0[w] = __byte_perm(a0, a1, 0x5410u);
                Pa[w] = p.dgp[ja][w];
                Pb[w] = p.dgp[jb][w];
            }
            odd_pairs<G>(P0, P1);
            v = pair_value16<G>(P0, P1, sdg, ja, jb, Pa, Pb);
            if (valid && pair_needs_exact<!BNB>(p, v, base, lb)) tree_pair_exact<G>(p, U, B, ja, jb, base, lb);
            return;
        }
    }
    int32_t Da[G], Db[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        Da[i] = sdg[ja * 32 + i];
        Db[i] = sdg[jb * 32 + i];
    }
    side_fold<G, 1>(A, Da, Db, v);
    side_fold<G, 1>(A, Db, Da, v);
    if (valid && pair_needs_exact<!BNB>(p, v, base, lb)) tree_pair_exact<G>(p, U, B, ja, jb, base, lb);
}

// Packed merge with a warp-uniform runtime gang size (one uniform branch to the compile-time
// shift)
template <int G>
__device__ __forceinline__ void merge_dispatch16(int g, const uint32_t (&P0)[Pk<G>::W], const uint32_t (&P1)[Pk<G>::W],
                                                 uint32_t d2, uint32_t (&C)[Pk<G>::W]) {
    switch (g) {
#define SAT_CASE16(K) \
    case K: if constexpr (K <= G) merge16<G, (K <= G ? K : 1)>(P0, P1, rep16<(K <= G ? K : 1) - 1>(P0) + d2, C); break;
        SAT_CASE16(1) SAT_CASE16(2) SAT_CASE16(3) SAT_CASE16(4) SAT_CASE16(5) SAT_CASE16(6) SAT_CASE16(7)
        SAT_CASE16(8) SAT_CASE16(9) SAT_CASE16(10) SAT_CASE16(11) SAT_CASE16(12) SAT_CASE16(13)
        SAT_CASE16(14) SAT_CASE16(15) SAT_CASE16(16)
#undef SAT_CASE16
        default: break;
    }
}

// Three jobs left, full scan, packed pair pass: the level-1 state (after the first of the
// three) stays in registers as 16-bit pairs -- no shared-memory round trip per pair node; it
// is written to the level-1 column only when a pair node needs its exact pass.
template <int G>
__device__ __forceinline__ void walk_q3_16(const TreeParams &p, const int32_t *L0, int32_t *dst, int32_t *Bbuf,
                                           const int32_t *sdg, uint32_t rem, uint64_t acc_in, bool ok,
                                           LaneBest &lb) {
    constexpr int W = Pk<G>::W;
    uint32_t P0[W], P1[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const uint32_t a0 = (uint32_t)L0[2 * w * 32];
        const uint32_t a1 = 2 * w + 1 < G ? (uint32_t)L0[(2 * w + 1 < G ? 2 * w + 1 : 0) * 32] : kTreeInf16;
        P0[w] = __byte_perm(a0, a1, 0x5410u);
    }
    odd_pairs<G>(P0, P1);
    const uint64_t fq = p.fact[2];                    // Lehmer weight of the first of three positions
    for (uint32_t m = rem; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const uint32_t rem2 = rem & ~(1u << j);
        const int ja = __ffs(rem2) - 1;
        const int jb = 31 - __clz(rem2);
        uint32_t Pa[W], Pb[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            Pa[w] = p.dgp[ja][w];
            Pb[w] = p.dgp[jb][w];
        }
        const uint64_t acc_j = acc_in + (uint64_t)__popc(rem & ((1u << j) - 1u)) * fq;
        const int r = p.radix[j], ob = p.optbase[j];
        const uint64_t wj = p.wJ[j];
        for (int o = 0; o < r; ++o) {
            uint32_t C0[W], C1[W];
            merge_dispatch16<G>(p.optg[ob + o], P0, P1, (uint32_t)p.optd[ob + o] * 0x10001u, C0);
            odd_pairs<G>(C0, C1);
            const int32_t v = pair_value16<G>(C0, C1, sdg, ja, jb, Pa, Pb);
            const uint64_t acc = acc_j + (uint64_t)o * wj;
            if (ok && pair_needs_exact<true>(p, v, acc, lb)) {
#pragma unroll
                for (int i = 0; i < G; ++i) dst[i * 32] = (int32_t)((C0[i / 2] >> (16 * (i & 1))) & 0xFFFFu);
                tree_pair_exact<G>(p, dst, Bbuf, ja, jb, acc, lb);
            }
        }
    }
}

// Upper-level merge with a warp-uniform runtime gang size, smem column to smem column.
template <int G>
__device__ __forceinline__ void merge_cols(const int32_t *src, int32_t *dst, int g, int32_t d) {
    SAT_ASSERT(g >= 1 && g <= G);
    const int32_t e = src[(g - 1) * 32] + d;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int32_t v = max(src[i * 32], min(src[(i + g) * 32], e));   // src rows G..2G-1 = INF
        dst[i * 32] = v;
    }
}

// Lower bound on the makespan of every completion of a partial schedule (bound-and-prune):
// the lane's sorted free times `col` (stride 32) after the placed jobs, `rem` unplaced.
//   - the largest free time already committed;
//   - each unplaced job j ends no earlier than min over its gangs k of (col[k] + dg[j][k])
//     (free times only grow, and a g-gang cannot start before the g-th free time);
//   - area: the GPU time from the free times to the makespan must hold every unplaced
//     job's least g * d:  M * G >= sum(col) + sum_j minarea_j.
// Every completion of the prefix has makespan >= the bound, so pruning on bound > best
// keeps every candidate that could tie or beat the best (the result equals exhaustive).
template <int G>
__device__ __forceinline__ int32_t lane_bound(const TreeParams &p, const int32_t *col, const int32_t *sdg,
                                              uint32_t rem) {
    int32_t A[G];
    int32_t area = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        A[i] = col[i * 32];
        area += A[i];
    }
    int32_t lb = A[G - 1];
    for (uint32_t m = rem; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        area += p.minarea[j];
        int32_t e = SAT_INF_I32;
#pragma unroll
        for (int k = 0; k < G; ++k) e = min(e, A[k] + sdg[j * 32 + k]);
        lb = max(lb, e);
    }
    return max(lb, (area + G - 1) / G);
}

// best makespan published so far (makespan part of the packed key), +inf if none
__device__ __forceinline__ int32_t published_ms(const TreeParams &p) {
    const unsigned long long hi = *reinterpret_cast<volatile unsigned long long *>(&p.best->hi);
    return hi == ~0ull ? SAT_INF_I32 : (int32_t)(hi >> p.idx_bits);
}

// Word offset of level buffer L in a warp's region.  Level buffers hold 2G rows (rows G..2G-1
// = INF, read by the shifted merge).  In the compact layout (full scan, packed pair pass,
// suffixes of 3-4 jobs) only level 0 is merged from with a shift: deeper levels are the
// register walk's input / the exact pass's input and hold G rows.
template <int G>
__host__ __device__ __forceinline__ int tree_level_off(int L, bool compact) {
    return compact ? (L == 0 ? 0 : (2 * G + (L - 1) * G) * 32) : L * 2 * G * 32;
}
// Compact: the last level (the register walk's exact-pass input) shares the exact pass's
// scratch column Bbuf (the exact pass reads its input into registers before writing).
template <int G>
__host__ __device__ __forceinline__ int tree_warp_words(int Q, bool compact) {
    return tree_level_off<G>(compact ? Q - 2 : Q - 1, compact) + G * 32;   // level buffers, then Bbuf
}
__host__ __device__ __forceinline__ bool tree_compact(bool bnb, bool packed, int G, int Q) {
    return !bnb && packed && G >= 2 && G <= kTreePackMaxG && (Q == 3 || Q == 4);
}

// Suffix walk with a compile-time number D of upper levels (Q = D + 2 jobs left): the
// level state (remaining set, index accumulator, cursor) stays in registers instead of the
// local-memory stack of the generic walk.  Level L's free times are the lane's column in
// level buffer L; children go to buffer L + 1; the last two jobs are the pair pass.
template <int G, bool BNB, int D>
__device__ __forceinline__ void walk_fixed(const TreeParams &p, int32_t *wbase, int lane, int L, int Q,
                                           uint32_t rem, uint64_t acc_in, bool ok, int32_t *Bbuf,
                                           const int32_t *sdg, LaneBest &lb, int32_t &U,
                                           unsigned long long &n_pairs) {
    const bool compact = tree_compact(BNB, p.packed != 0, G, Q);
    const int32_t *src = wbase + tree_level_off<G>(L, compact) + lane;
    int32_t *dst = wbase + tree_level_off<G>(L + 1, compact) + lane;
    const uint64_t fq = p.fact[Q - 1 - L];
    for (uint32_t m = rem; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const uint32_t rem2 = rem & ~(1u << j);
        const uint64_t acc_j = acc_in + (uint64_t)__popc(rem & ((1u << j) - 1u)) * fq;
        const int r = p.radix[j], ob = p.optbase[j];
        const uint64_t wj = p.wJ[j];
        for (int o = 0; o < r; ++o) {
            merge_cols<G>(src, dst, p.optg[ob + o], p.optd[ob + o]);
            const uint64_t acc = acc_j + (uint64_t)o * wj;
            bool child_ok = ok;
            if constexpr (BNB) {
                if (__any_sync(0xffffffffu, child_ok)) {
                    U = min(U, lb.ms);
                    child_ok = child_ok && lane_bound<G>(p, dst, sdg, rem2) <= U;
                }
                if (!__any_sync(0xffffffffu, child_ok)) continue;
            }
            if constexpr (D == 1) {
                if (BNB && lane == 0) ++n_pairs;
                tree_pair<G, BNB>(p, dst, Bbuf, sdg, rem2, acc, child_ok, lb);
            } else {
                bool done = false;
                if constexpr (!BNB && D == 2 && G >= 2 && G <= kTreePackMaxG) {
                    if (p.packed) {     // three jobs left: the register-resident packed walk
                        walk_q3_16<G>(p, dst, Bbuf, Bbuf, sdg, rem2, acc, child_ok, lb);
                        done = true;
                    }
                }
                if (!done)
                    walk_fixed<G, BNB, D - 1>(p, wbase, lane, L + 1, Q, rem2, acc, child_ok, Bbuf, sdg, lb, U, n_pairs);
            }
        }
    }
}

// occupancy target per node size: 12 blocks (40 regs) up to 8 GPUs, fewer for larger nodes.
// BNB = bound-and-prune: subtrees whose bound exceeds the best makespan found so far (by
// any warp: published after every task) are skipped; the key found is the exhaustive one.
// DEEP = the generic walk (suffixes beyond the fixed-depth walkers) and prefixes of more than 8
// jobs: their per-lane stacks live in local memory, so they get their own instantiation and
// the common kernel (config 1: 4-job prefix, 4-job suffix) keeps no stack frame at all.
#ifndef SAT_TREE_MINB8
#define SAT_TREE_MINB8 10    // blocks per SM the register budget targets for nodes of <= 8 GPUs
#endif
template <int G, bool BNB, bool DEEP>
__global__ void __launch_bounds__(kTreeThreads, G <= 8 ? SAT_TREE_MINB8 : (G <= 16 ? 8 : 4))
k_tree(const __grid_constant__ TreeParams p) {
    extern __shared__ __align__(16) int32_t tsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Q = p.Q, P = p.P, J = p.J;
    const int upper = Q - 1;                         // level buffers 0..Q-2 (padded)
    const bool compact = tree_compact(BNB, p.packed != 0, G, Q);
    int32_t *wbase = tsm + warp * tree_warp_words<G>(Q, compact);
    int32_t *Bbuf = wbase + tree_level_off<G>(compact ? upper - 1 : upper, compact) + lane;
    // per (job, gang) least durations, shared by the block (broadcast loads in the pair pass)
    // per (job, gang) least durations, read straight from the parameter block: the job index
    // is warp-uniform, so these are uniform constant loads and the gang branches uniform
    const int32_t *sdg = &p.dg[0][0];
    // padding rows of every level buffer = INF (never rewritten)
    for (int L = 0; L < (compact ? 1 : upper); ++L)
        for (int i = G; i < 2 * G; ++i) wbase[tree_level_off<G>(L, compact) + i * 32 + lane] = SAT_INF_I32;

    // bound-and-prune records only candidates at or below the seed bound (the key's makespan
    // field is sized for it); the full scan records everything
    LaneBest lb{BNB ? min(published_ms(p), (int32_t)SAT_INF_I32) : (int32_t)SAT_INF_I32, ~0ull};
    const uint32_t all = (J >= 32) ? 0xffffffffu : ((1u << J) - 1u);
    unsigned long long published = ~0ull;          // BNB: last key this warp published
    unsigned long long n_pruned = 0, n_pairs = 0;   // BNB counters (lane 0)

    // dynamic task cursor: a warp takes the next task when it finishes one (task costs
    // differ by the remaining jobs' radices; a static split leaves a long tail)
    // (the host keeps a launch below 2^32 tasks, so the id travels as a 32-bit warp reduction,
    // which the compiler knows to be warp-uniform)
    auto next_task = [&]() -> uint64_t {
        unsigned v = 0xffffffffu;
        if (lane == 0) v = (unsigned)atomicAdd(p.cursor, 1ull);
        return p.task_lo + (uint64_t)__reduce_min_sync(0xffffffffu, v);
    };
    for (uint64_t t = next_task(); t < p.task_hi; t = next_task()) {
        // ---- which prefix set (warp-uniform binary search) ----
        int lo = 0, hi = p.n_sets - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.set_cum[mid] <= t) lo = mid; else hi = mid - 1;
        }
        const int s = lo;
        const uint32_t S = p.set_mask[s];
        uint64_t fP = p.fact[P];
        const uint64_t npref = fP * p.set_prod[s];
        const uint64_t q = (t - p.set_cum[s]) * 32ull + (uint64_t)lane;
        const bool valid = q < npref;
        const uint64_t qq = valid ? q : 0;

        // ---- decode this lane's prefix: order of S (Lehmer) and options of S ----
        uint64_t code = qq / fP;
        uint64_t prank = qq - code * fP;
        int32_t *L0 = wbase + lane;
        for (int i = 0; i < G; ++i) L0[i * 32] = p.init_free[i];
        // options of S's jobs: mixed radix, highest job id least significant; kept as 8-bit
        // fields indexed by the job's rank within S (P <= 8: one u64 register; else local)
        uint64_t popt_lo = 0;
        uint8_t popt_hi[DEEP ? kTreeMaxJ : 1];
        {
            uint32_t m = S;
            int rank = P;
            while (m) {
                const int j = 31 - __clz(m);
                m &= ~(1u << j);
                --rank;
                const uint64_t r = (uint64_t)p.radix[j];
                const uint64_t qd = code / r;
                const uint64_t dig = code - qd * r;
                if (rank < 8) popt_lo |= dig << (8 * rank);
                else if constexpr (DEEP) popt_hi[rank] = (uint8_t)dig;
                code = qd;
            }
        }
        uint64_t base = 0;
        const uint32_t unplaced = all & ~S;          // warp-uniform: the suffix jobs
        uint32_t unpl = all, avail = S;
        for (int k = 0; k < P; ++k) {
            fP /= (uint64_t)(P - k);
            const uint64_t digit = prank / fP;
            prank -= digit * fP;
            uint32_t m = avail;
            for (uint64_t x = 0; x < digit; ++x) m &= m - 1;
            const int j = __ffs(m) - 1;
            avail &= ~(1u << j);
            const int rk = __popc(S & ((1u << j) - 1u));
            int o = (int)((popt_lo >> (8 * (rk & 7))) & 0xffu);
            if constexpr (DEEP) if (rk >= 8) o = (int)popt_hi[rk];
            base += (uint64_t)__popc(unpl & ((1u << j) - 1u)) * p.fact[J - 1 - k] + (uint64_t)o * p.wJ[j];
            unpl &= ~(1u << j);
            // per-lane gang size: in-place merge on the lane's column
            const int q2 = p.optbase[j] + o;
            const int g = p.optg[q2];
            SAT_ASSERT(j >= 0 && j < J && o < p.radix[j] && g >= 1 && g <= G);
            const int32_t e = L0[(g - 1) * 32] + p.optd[q2];
            for (int i = 0; i < G; ++i) L0[i * 32] = max(L0[i * 32], min(L0[(i + g) * 32], e));
        }
        __syncwarp();
        bool lane_ok = valid;
        int32_t U = SAT_INF_I32;
        if constexpr (BNB) {
            U = min(published_ms(p), lb.ms);
            lane_ok = valid && lane_bound<G>(p, L0, sdg, unplaced) <= U;
            if (!__any_sync(0xffffffffu, lane_ok)) {
                if (lane == 0) ++n_pruned;
                continue;
            }
        }

        // ---- warp-uniform walk over the suffix (jobs in `unplaced`) ----
        if (Q == 2) {
            if (BNB && lane == 0) ++n_pairs;
            tree_pair<G, BNB>(p, L0, Bbuf, sdg, unplaced, base, lane_ok, lb);
        } else if (Q == 3) {
            bool done = false;
            if constexpr (!BNB && G >= 2 && G <= kTreePackMaxG) {
                if (p.packed) {
                    walk_q3_16<G>(p, L0, Bbuf, Bbuf, sdg, unplaced, base, lane_ok, lb);
                    done = true;
                }
            }
            if (!done) walk_fixed<G, BNB, 1>(p, wbase, lane, 0, Q, unplaced, base, lane_ok, Bbuf, sdg, lb, U, n_pairs);
        } else if (Q == 4) {
            walk_fixed<G, BNB, 2>(p, wbase, lane, 0, Q, unplaced, base, lane_ok, Bbuf, sdg, lb, U, n_pairs);
        } else if (BNB && Q == 5) {
            walk_fixed<G, BNB, 3>(p, wbase, lane, 0, Q, unplaced, base, lane_ok, Bbuf, sdg, lb, U, n_pairs);
        } else if (BNB && Q == 6) {
            walk_fixed<G, BNB, 4>(p, wbase, lane, 0, Q, unplaced, base, lane_ok, Bbuf, sdg, lb, U, n_pairs);
        } else if (BNB && Q == 7) {
            walk_fixed<G, BNB, 5>(p, wbase, lane, 0, Q, unplaced, base, lane_ok, Bbuf, sdg, lb, U, n_pairs);
        } else if constexpr (DEEP) {
            uint32_t rem_st[kTreeMaxJ];
            uint64_t acc_st[kTreeMaxJ];
            int cj[kTreeMaxJ], co[kTreeMaxJ];
            uint32_t okbits = lane_ok ? 1u : 0u;    // bit L: this lane's level-L node is live
            int L = 0;
            rem_st[0] = unplaced;
            acc_st[0] = base;
            cj[0] = -1;
            co[0] = 0;
            while (L >= 0) {
                // advance the cursor of level L to its next (job, option)
                int j = cj[L], o = co[L] + 1;
                if (j < 0 || o >= p.radix[j]) {
                    const uint32_t later = (j < 0) ? rem_st[L] : (rem_st[L] & ~((2u << j) - 1u));
                    if (!later) { --L; continue; }
                    j = __ffs(later) - 1;
                    o = 0;
                }
                cj[L] = j;
                co[L] = o;
                const int32_t *src = wbase + tree_level_off<G>(L, compact) + lane;
                int32_t *dst = wbase + tree_level_off<G>(L + 1, compact) + lane;
                const int q2 = p.optbase[j] + o;
                merge_cols<G>(src, dst, p.optg[q2], p.optd[q2]);
                const uint32_t rem = rem_st[L];
                const uint64_t acc = acc_st[L] +
                    (uint64_t)__popc(rem & ((1u << j) - 1u)) * p.fact[Q - 1 - L] + (uint64_t)o * p.wJ[j];
                const uint32_t rem2 = rem & ~(1u << j);
                bool child_ok = (okbits >> L) & 1u;
                if constexpr (BNB) {
                    if (__any_sync(0xffffffffu, child_ok)) {
                        U = min(U, lb.ms);
                        child_ok = child_ok && lane_bound<G>(p, dst, sdg, rem2) <= U;
                    }
                    if (!__any_sync(0xffffffffu, child_ok)) continue;
                }
                if (L + 1 == Q - 2) {
                    if (BNB && lane == 0) ++n_pairs;
                    tree_pair<G, BNB>(p, dst, Bbuf, sdg, rem2, acc, child_ok, lb);
                } else {
                    ++L;
                    rem_st[L] = rem2;
                    acc_st[L] = acc;
                    cj[L] = -1;
                    co[L] = 0;
                    okbits = (okbits & ((1u << L) - 1u)) | ((child_ok ? 1u : 0u) << L);
                }
            }
        }
        __syncwarp();
        {
            // publish an improvement right away: every warp prunes (bnb) and skips exact
            // pair passes (both modes) against it
            uint64_t key = (lb.ix != ~0ull) ? (((uint64_t)(uint32_t)lb.ms << p.idx_bits) | lb.ix) : ~0ull;
            for (int x = 16; x >= 1; x >>= 1) {
                const uint64_t o = shfl_u64(key, lane ^ x);
                key = o < key ? o : key;
            }
            if (key < published) {
                published = key;
                if (lane == 0) atomicMin(reinterpret_cast<unsigned long long *>(&p.best->hi), (unsigned long long)key);
            }
        }
    }

    // ---- warp argmin, one atomic per warp ----
    uint64_t key = (lb.ix != ~0ull) ? (((uint64_t)(uint32_t)lb.ms << p.idx_bits) | lb.ix) : ~0ull;
    for (int x = 16; x >= 1; x >>= 1) {
        const uint64_t o = shfl_u64(key, lane ^ x);
        key = o < key ? o : key;
    }
    if (lane == 0 && key != ~0ull)
        atomicMin(reinterpret_cast<unsigned long long *>(&p.best->hi), (unsigned long long)key);
    if (BNB && lane == 0 && p.stats) {
        atomicAdd(&p.stats[SAT_BNB_STAT_PRUNED_TASKS], n_pruned);
        atomicAdd(&p.stats[SAT_BNB_STAT_PAIR_NODES], n_pairs);
    }
}

template <int G, bool BNB>
int launch_tree_k(const TreeParams &tp, int Q, cudaStream_t stream) {
    const int smem = kTreeWarps * tree_warp_words<G>(Q, tree_compact(BNB, tp.packed != 0, G, Q)) * 4;
    if (smem > 200 * 1024) return SAT_ERR_UNSUPPORTED;
    // the fixed-depth walkers cover Q <= 4 (full scan) / Q <= 7 (bound-and-prune) with prefixes
    // of <= 8 jobs; anything else takes the DEEP instantiation
    const bool deep = tp.P > 8 || Q > (BNB ? 7 : 4);
    auto kern = deep ? k_tree<G, BNB, true> : k_tree<G, BNB, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SAT_ERR_CUDA;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTreeThreads, smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    uint64_t blocks = (uint64_t)device_sms() * per_sm;
    const uint64_t tasks = tp.task_hi - tp.task_lo;
    const uint64_t need = (tasks + kTreeWarps - 1) / kTreeWarps;
    if (blocks > need) blocks = std::max<uint64_t>(1, need);
    kern<<<(unsigned)blocks, kTreeThreads, smem, stream>>>(tp);
    return cudaGetLastError() == cudaSuccess ? SAT_OK : SAT_ERR_CUDA;
}

template <int G>
int launch_tree_g(const TreeParams &tp, int Q, bool bnb, cudaStream_t stream) {
    return bnb ? launch_tree_k<G, true>(tp, Q, stream) : launch_tree_k<G, false>(tp, Q, stream);
}

}  // namespace sat
