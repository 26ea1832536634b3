// sat_common.cuh -- definitions shared by the engine's translation units
// (sat_engine.cu: generic kernel, host packing, C ABI; sat_tree_*.cu: the walk kernels).
#pragma once


#include "../../include/saturn_engine.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define SAT_INF_I32 0x3FFFFFFF

// Device-side bounds checks for the debug build of the library (build.py --debug ->
// libsaturn_b200_debug.so, -DSAT_DEBUG_BOUNDS): every index that addresses a thread's or
// warp's shared-memory region is checked against the region; a violation traps.  The
// release build compiles them out.  (compute-sanitizer is not available on this pool.)
#ifdef SAT_DEBUG_BOUNDS
#define SAT_ASSERT(c)                                                                  \
    do {                                                                               \
        if (!(c)) {                                                                    \
            printf("SAT_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);           \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define SAT_ASSERT(c) do { } while (0)
#endif

namespace sat {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;
constexpr int kGenThreads = 256;
constexpr int kGenWarps = kGenThreads / 32;
constexpr int kTreeThreads = 128;
constexpr int kTreeWarps = kTreeThreads / 32;

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    return z ^ (z >> 31);
}

template <typename T> struct TimeTraits;
template <> struct TimeTraits<int32_t> {
    __device__ static int32_t inf() { return SAT_INF_I32; }
};
template <> struct TimeTraits<double> {
    __device__ static double inf() { return __longlong_as_double(0x7ff0000000000000ll); }
};

__device__ inline int32_t tmin(int32_t a, int32_t b) { return min(a, b); }
__device__ inline int32_t tmax(int32_t a, int32_t b) { return max(a, b); }
__device__ inline double tmin(double a, double b) { return fmin(a, b); }
__device__ inline double tmax(double a, double b) { return fmax(a, b); }

__device__ inline uint64_t shfl_u64(uint64_t v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}


int device_sms();                          // sat_engine.cu
int validate(const sat_problem_t *p);      // sat_engine.cu

// ---------------------------------------------------------------------------
// k_tree: prefix-shared exhaustive walk, one node, grid int32 time
// ---------------------------------------------------------------------------
constexpr int kTreeMaxJ = 20;
constexpr int kTreeMaxOpt = 384;
constexpr int kTreeMaxSets = 768;

// Packed pair pass (k_tree, G <= kTreePackMaxG): two 16-bit free times per word when every
// time the walk can produce stays below kTreePackLimit (host-checked); missing gangs and
// padding slots hold kTreeInf16, so a slot sum b + D2 <= 0x7FFF + 0x7FFF never carries.
constexpr uint32_t kTreeInf16 = 0x7FFFu;
constexpr int32_t kTreePackLimit = 0x7000;
constexpr int kTreePackMaxG = 16;

struct TreeParams {
    int32_t J, P, Q, Gr, n_sets, idx_bits, init_max;
    int32_t packed;                   // 1: pair pass on 16-bit pairs (dgp valid)
    int32_t radix[kTreeMaxJ];
    int32_t optbase[kTreeMaxJ];
    uint64_t wJ[kTreeMaxJ];           // option-digit weight in the index: W_j * J!
    uint64_t fact[kTreeMaxJ + 1];     // k!
    int32_t init_free[32];            // ascending (only the first G = node GPUs are used)
    int32_t optg[kTreeMaxOpt];
    int32_t optoff[kTreeMaxOpt];      // (g - 1) * 32: smem word offset of slot g-1
    int32_t optd[kTreeMaxOpt];
    int32_t dg[kTreeMaxJ][32];        // per job and gang size g: min duration over its options (INF: none)
    uint32_t dgp[kTreeMaxJ][kTreePackMaxG / 2];   // dg as 16-bit pairs (gangs 2w+1, 2w+2; kTreeInf16: none)
    uint32_t set_mask[kTreeMaxSets];
    uint64_t set_cum[kTreeMaxSets + 1];  // cumulative warp tasks
    uint64_t set_prod[kTreeMaxSets];     // prod of radix over the set
    int32_t minarea[kTreeMaxJ];       // per job: least g * d over its options (bound-and-prune)
    uint64_t task_lo, task_hi;
    sat_best_t *best;
    unsigned long long *cursor;       // tasks handed out so far (zeroed before the launch)
    unsigned long long *stats;        // bound-and-prune counters (SAT_BNB_STAT_*), or null
};

// Per-lane running best (makespan, index).
struct LaneBest {
    int32_t ms;
    uint64_t ix;
};

template <int G>
int launch_tree_g(const TreeParams &tp, int Q, bool bnb, cudaStream_t stream);   // sat_tree.cuh

}  // namespace sat
