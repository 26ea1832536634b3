// sat_decode.cuh -- the problem blob and the candidate decoders shared by the
// per-candidate kernels (k_generic in sat_engine.cu, k_cand in sat_cand.cu).
#pragma once

#include "sat_common.cuh"

namespace sat {
// ---------------------------------------------------------------------------
// Generic problem blob (host-packed, copied to the workspace, staged to smem)
// ---------------------------------------------------------------------------
struct BlobHeader {
    int32_t J, N, G, W;
    int32_t time_mode, idx_bits, n_opt, has_release;
    int32_t max_n;            // largest n that below(n) is asked for (sampled decode)
    int32_t bytes;            // total blob bytes
    int32_t off_radix, off_optbase, off_g, off_mask, off_dur, off_release, off_lane_init, off_modn;
    int32_t off_prerec, off_jobinfo;   // per-option step records, per-job draw constants
    int64_t init_max_i32;
    double init_max_f64;
};
static_assert(sizeof(BlobHeader) % 16 == 0, "blob header alignment");

// per-n constants for SplitMix64 below(n): rejection threshold and a reciprocal
struct ModN {
    uint64_t reject_rem;  // (2^64 mod n): accept r iff r <= ~0 - reject_rem   (rng.py:37-41)
    uint64_t magic;       // floor((2^64 - 1) / n)
};

__device__ inline uint64_t mod_small(uint64_t r, uint32_t n, uint64_t magic) {
    uint64_t q = __umul64hi(r, magic);
    uint64_t rem = r - q * (uint64_t)n;
    while (rem >= n) rem -= n;
    return rem;
}

// r mod n for n <= 255 without a loop: q = umulhi(r, floor((2^64-1)/n)) is floor(r/n) or
// one less (r*magic/2^64 lies in (r/n - 1, r/n]), so r - q*n < 2n < 2^32 is exact in the
// low word and needs at most one conditional subtract.
__device__ __forceinline__ uint32_t mod_small_fast(uint64_t r, uint32_t n, uint64_t magic) {
    const uint64_t q = __umul64hi(r, magic);
    const uint32_t rem = (uint32_t)r - (uint32_t)q * n;
    return min(rem, rem - n);          // rem - n wraps above rem exactly when rem < n
}

// SplitMix64 stream with a draw counter: k-th output = mix64(state0 + k*GOLDEN)
struct Stream {
    uint64_t state;
    __device__ inline uint64_t next() {
        state += kGolden;
        return mix64(state);
    }
    // exact below(n) (rng.py:34-42), rejection loop included
    __device__ inline uint32_t below(uint32_t n, const ModN *mods) {
        const ModN m = mods[n];
        uint64_t r = next();
        while (r > ~0ull - m.reject_rem) r = next();   // rejection (practically never taken)
        return (uint32_t)mod_small(r, n, m.magic);
    }
    // below(n) assuming no rejection; `hi_max` accumulates the draws' high words.  A draw
    // can only be rejected when r >= 2^64 - (2^64 mod n) > 2^64 - 2^32, i.e. its high word
    // is all ones, so hi_max != 0xffffffff proves every fast draw equals the exact one.
    __device__ __forceinline__ uint32_t below_fast(uint32_t n, uint64_t magic, uint32_t &hi_max) {
        const uint64_t r = next();
        hi_max = max(hi_max, (uint32_t)(r >> 32));
        return mod_small_fast(r, n, magic);
    }
};

// ---------------------------------------------------------------------------
// k_generic: candidate decode (one lane per candidate) + W-lane list scheduling
// ---------------------------------------------------------------------------
struct GenArgs {
    const uint8_t *blob;
    uint64_t lo, hi;            // candidate ids [lo, hi)
    uint64_t seed;
    int32_t per_lane;           // consecutive candidates per lane per batch (index source)
    int32_t rec_d;              // step records carry the duration itself (one node, grid, search)
    const uint64_t *ids;        // RECORD: explicit candidate ids (index/stream sources)
    const uint8_t *expl;        // EXPLICIT source: [n][2J]
    sat_best_t *best;           // grid mode result
    sat_best_t *partials;       // float mode per-block partials
    int32_t *rec_opt, *rec_node;
    int32_t *rec_start_i32;
    double *rec_start_f64;
    int64_t *rec_ms_i64;
    double *rec_ms_f64;
};

template <typename T>
__device__ inline bool key_less(T ms_a, uint64_t ix_a, T ms_b, uint64_t ix_b) {
    return ms_a < ms_b || (ms_a == ms_b && ix_a < ix_b);
}

// A candidate is decoded into J step records, one per position of the submission order:
//   bits 0-5  gang size - 1      bits 6-11  job      bits 12-31  duration or global option q
// stored lane-interleaved (record k of lane l at word k*32 + l): decode writes are
// conflict-free and a W-lane segment reads its candidate's record as one broadcast.
__device__ inline uint32_t step_rec(int g, int job, uint32_t payload) {
    return (uint32_t)(g - 1) | ((uint32_t)job << 6) | (payload << 12);
}

// per-job constants of the option draw below(radix_j): one 16-byte broadcast load
struct JobInfo {
    int32_t radix;
    int32_t optbase;     // global id of option 0 of the job
    uint64_t magic;      // floor((2^64 - 1) / radix)
};

struct GenTables {
    const int32_t *radix, *optbase;
    const uint32_t *optmask;
    const uint32_t *prerec;    // [n_opt] step record of every option (host-built)
    const JobInfo *jobinfo;    // [J]
    const ModN *mods;
    int J, N;
};

// step record of job `job` running option `o` (payload = duration or global option id,
// fixed per problem on the host)
__device__ __forceinline__ uint32_t rec_for(const GenTables &t, int job, int o) {
    return t.prerec[t.optbase[job] + o];
}

__device__ inline void load_tables(GenTables &tb, const uint8_t *smem, const BlobHeader &h) {
    tb.radix = reinterpret_cast<const int32_t *>(smem + h.off_radix);
    tb.optbase = reinterpret_cast<const int32_t *>(smem + h.off_optbase);
    tb.optmask = reinterpret_cast<const uint32_t *>(smem + h.off_mask);
    tb.prerec = reinterpret_cast<const uint32_t *>(smem + h.off_prerec);
    tb.jobinfo = reinterpret_cast<const JobInfo *>(smem + h.off_jobinfo);
    tb.mods = reinterpret_cast<const ModN *>(smem + h.off_modn);
    tb.J = h.J;
    tb.N = h.N;
}

// index -> option digits (job 0 most significant) and Lehmer-ranked order, into the
// lane's interleaved u8 scratch
__device__ inline void decode_index(uint64_t id, int J, const int32_t *radix, uint8_t *opt, uint8_t *ord) {
    uint64_t f = 1;
    for (int k = 2; k <= J; ++k) f *= (uint64_t)k;
    uint64_t conf = id / f;
    uint64_t perm = id - conf * f;
    for (int j = J - 1; j >= 0; --j) {
        const uint64_t r = (uint64_t)radix[j];
        const uint64_t qd = conf / r;
        opt[j * 32] = (uint8_t)(conf - qd * r);
        conf = qd;
    }
    uint64_t unused = (J == 64) ? ~0ull : ((1ull << J) - 1ull);
    for (int k = 0; k < J; ++k) {
        f /= (uint64_t)(J - k);                       // (J-1-k)!
        const uint64_t digit = perm / f;
        perm -= digit * f;
        uint64_t m = unused;
        for (uint64_t x = 0; x < digit; ++x) m &= m - 1;
        const int job = __ffsll((long long)m) - 1;
        ord[k * 32] = (uint8_t)job;
        unused &= ~(1ull << job);
    }
}

// index + 1: next lexicographic permutation; on wrap, odometer the option digits
__device__ inline void advance_index(int J, const int32_t *radix, uint8_t *opt, uint8_t *ord) {
    int i = J - 2;
    while (i >= 0 && ord[i * 32] >= ord[(i + 1) * 32]) --i;
    if (i >= 0) {
        int k = J - 1;
        while (ord[k * 32] <= ord[i * 32]) --k;
        uint8_t t = ord[i * 32]; ord[i * 32] = ord[k * 32]; ord[k * 32] = t;
        for (int a = i + 1, b = J - 1; a < b; ++a, --b) { t = ord[a * 32]; ord[a * 32] = ord[b * 32]; ord[b * 32] = t; }
        return;
    }
    for (int k = 0; k < J; ++k) ord[k * 32] = (uint8_t)k;
    for (int j = J - 1; j >= 0; --j) {
        if ((int)opt[j * 32] + 1 < radix[j]) { opt[j * 32] += 1; return; }
        opt[j * 32] = 0;
    }
}

// plan_random draw order: below(radix_j) per job in id order, then a
// Fisher-Yates shuffle of the order -- applied directly to the step records.  The
// common path skips the rejection tests; in the (p ~ 1e-17 per draw) case a draw could
// have been rejected, the candidate is decoded again with the exact loops.
__device__ inline void decode_stream(uint64_t state0, const GenTables &t, uint32_t *steps) {
    Stream s{state0};
    uint32_t hi_max = 0;
    for (int j = 0; j < t.J; ++j) {
        const JobInfo ji = t.jobinfo[j];
        const int o = (int)s.below_fast((uint32_t)ji.radix, ji.magic, hi_max);
        SAT_ASSERT(o >= 0 && o < ji.radix);
        steps[j * 32] = t.prerec[ji.optbase + o];
    }
    for (int i = t.J - 1; i >= 1; --i) {                 // rng.py:44-48
        const int k = (int)s.below_fast((uint32_t)(i + 1), t.mods[i + 1].magic, hi_max);
        SAT_ASSERT(k >= 0 && k <= i);
        const uint32_t x = steps[i * 32];
        steps[i * 32] = steps[k * 32];
        steps[k * 32] = x;
    }
    if (hi_max == 0xffffffffu) {
        s.state = state0;
        for (int j = 0; j < t.J; ++j) {
            const int o = (int)s.below((uint32_t)t.radix[j], t.mods);
            steps[j * 32] = rec_for(t, j, o);
        }
        for (int i = t.J - 1; i >= 1; --i) {
            const int k = (int)s.below((uint32_t)(i + 1), t.mods);
            const uint32_t x = steps[i * 32];
            steps[i * 32] = steps[k * 32];
            steps[k * 32] = x;
        }
    }
}


// float mode: fold per-block partials into *best (lexicographic on (ms bits, index))
static __global__ void k_fold_partials(const sat_best_t *partials, int n, sat_best_t *best) {
    uint64_t hi = best->hi, lo = best->lo;
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
            const uint64_t ph = partials[i].hi, pl = partials[i].lo;
            if (ph < hi || (ph == hi && pl < lo)) { hi = ph; lo = pl; }
        }
        best->hi = hi;
        best->lo = lo;
    }
}


// host (sat_engine.cu): whether step records can carry the duration itself (grid time,
// node-independent durations < 2^20, every option runnable on every node), and the blob
// staged to shared memory (records carry durations iff rec_d)
bool records_carry_duration(const sat_problem_t *p);
int pack_blob(const sat_problem_t *p, std::vector<uint8_t> &blob, bool rec_d);

}  // namespace sat
