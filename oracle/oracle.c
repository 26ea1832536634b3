/*
 * oracle.c -- CPU ORACLE for the plan-search hot path.  TEST INFRASTRUCTURE ONLY:
 * used by tests/ as the checker and by bench.py as the CPU baseline (cpu_baseline,
 * --impl reference).  Never linked into or called by the product engine.
 *
 * C restatement of the same semantics as oracle/saturn_oracle.py (which it is
 * checked against in tests/test_oracle.py, test_c_oracle_matches_python):
 *   - candidate space of SURVEY.md Appendix A1 (index = c * J! + p), SplitMix64
 *     draws of plan_random (rng.py:20-56),
 *   - list scheduling "earliest-fit" over explicit per-GPU free
 *     times with GPU ids: node = the one finishing the job earliest (start = g-th
 *     smallest free time max release, + duration on that node), lowest node on ties; the g earliest-free GPUs (lowest id on ties) run the job,
 *   - best = lowest (makespan, id),
 *   - the engine's local search (oracle_local_search: sampled or greedy starts, the same
 *     moves, tie-breaks, rounds and stop rule as k_ls).
 * Times are doubles in both modes (grid intervals are small integers, exact).
 * OpenMP splits the id range into contiguous chunks, one per thread.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OMAX_J 64
#define OMAX_N 32
#define OMAX_G 32

typedef struct {
    int J, N, Cmax;
    const int *radix;        /* [J]            */
    const int *gpus;         /* [J*Cmax]       */
    const unsigned *mask;    /* [J*Cmax]       */
    const double *dur;       /* [J*Cmax*N]     */
    const int *node_gpus;    /* [N]            */
    const double *release;   /* [J] or NULL    */
    const double *init_free; /* [N*OMAX_G] or NULL, per GPU id */
} oproblem;

static const uint64_t GOLD = 0x9E3779B97F4A7C15ull;

static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint32_t below(uint64_t *state, uint32_t n) {
    /* limit = 2^64 - (2^64 mod n); accept r < limit */
    uint64_t rem = (uint64_t)(((unsigned __int128)1 << 64) % n);
    for (;;) {
        *state += GOLD;
        uint64_t r = mix(*state);
        if (rem == 0 || r < (uint64_t)0 - rem) return (uint32_t)(r % n);
    }
}

static void decode_stream(const oproblem *p, uint64_t state, int *opt, int *ord) {
    for (int j = 0; j < p->J; ++j) opt[j] = (int)below(&state, (uint32_t)p->radix[j]);
    for (int k = 0; k < p->J; ++k) ord[k] = k;
    for (int i = p->J - 1; i >= 1; --i) {
        int k = (int)below(&state, (uint32_t)(i + 1));
        int t = ord[i]; ord[i] = ord[k]; ord[k] = t;
    }
}

static void decode_index(const oproblem *p, uint64_t id, int *opt, int *ord) {
    int J = p->J;
    uint64_t f = 1;
    for (int k = 2; k <= J; ++k) f *= (uint64_t)k;
    uint64_t conf = id / f, perm = id % f;
    for (int j = J - 1; j >= 0; --j) { opt[j] = (int)(conf % (uint64_t)p->radix[j]); conf /= (uint64_t)p->radix[j]; }
    int pool[OMAX_J];
    for (int k = 0; k < J; ++k) pool[k] = k;
    int left = J;
    for (int k = 0; k < J; ++k) {
        f /= (uint64_t)(J - k);
        int d = (int)(perm / f);
        perm %= f;
        ord[k] = pool[d];
        memmove(pool + d, pool + d + 1, sizeof(int) * (size_t)(left - d - 1));
        --left;
    }
}

/* next candidate in index order (next lexicographic permutation, then options) */
static void next_index(const oproblem *p, int *opt, int *ord) {
    int J = p->J, i = J - 2;
    while (i >= 0 && ord[i] > ord[i + 1]) --i;
    if (i >= 0) {
        int k = J - 1;
        while (ord[k] < ord[i]) --k;
        int t = ord[i]; ord[i] = ord[k]; ord[k] = t;
        for (int a = i + 1, b = J - 1; a < b; ++a, --b) { t = ord[a]; ord[a] = ord[b]; ord[b] = t; }
        return;
    }
    for (int k = 0; k < J; ++k) ord[k] = k;
    for (int j = J - 1; j >= 0; --j) {
        if (opt[j] + 1 < p->radix[j]) { opt[j]++; return; }
        opt[j] = 0;
    }
}

/* list schedule one candidate; optional per-job start / node outputs; *load_out (optional) =
 * sum of the final free times of every GPU (the local search's tie-breaking objective) */
static double eval_full(const oproblem *p, const int *opt, const int *ord, double *start, int *node_out,
                        double *load_out) {
    double free_t[OMAX_N][OMAX_G];
    for (int n = 0; n < p->N; ++n)
        for (int k = 0; k < p->node_gpus[n]; ++k)
            free_t[n][k] = p->init_free ? p->init_free[n * OMAX_G + k] : 0.0;
    for (int kk = 0; kk < p->J; ++kk) {
        int j = ord[kk], o = opt[j];
        int q = j * p->Cmax + o;
        int g = p->gpus[q];
        double best_t = INFINITY, best_e = INFINITY;
        int best_n = -1;
        for (int n = 0; n < p->N; ++n) {
            if (!((p->mask[q] >> n) & 1u) || p->node_gpus[n] < g) continue;
            /* g-th smallest free time on node n (selection by counting) */
            double t = INFINITY;
            for (int a = 0; a < p->node_gpus[n]; ++a) {
                int less = 0, lesseq = 0;
                for (int b = 0; b < p->node_gpus[n]; ++b) {
                    less += free_t[n][b] < free_t[n][a];
                    lesseq += free_t[n][b] <= free_t[n][a];
                }
                if (less < g && g <= lesseq) { t = free_t[n][a]; break; }
            }
            if (p->release && p->release[j] > t) t = p->release[j];
            double e = t + p->dur[q * p->N + n];          /* earliest finish, lowest node on ties */
            if (best_n < 0 || e < best_e) { best_e = e; best_t = t; best_n = n; }
        }
        double e = best_e;
        /* the g earliest-free GPUs, lowest id on ties */
        int taken[OMAX_G] = {0};
        for (int c = 0; c < g; ++c) {
            int pick = -1;
            for (int a = 0; a < p->node_gpus[best_n]; ++a)
                if (!taken[a] && (pick < 0 || free_t[best_n][a] < free_t[best_n][pick])) pick = a;
            taken[pick] = 1;
        }
        for (int a = 0; a < p->node_gpus[best_n]; ++a)
            if (taken[a]) free_t[best_n][a] = e;
        if (start) start[j] = best_t;
        if (node_out) node_out[j] = best_n;
    }
    double ms = 0.0, load = 0.0;
    for (int n = 0; n < p->N; ++n)
        for (int k = 0; k < p->node_gpus[n]; ++k) {
            if (free_t[n][k] > ms) ms = free_t[n][k];
            load += free_t[n][k];
        }
    if (load_out) *load_out = load;
    return ms;
}

double oracle_eval(const oproblem *p, const int *opt, const int *ord, double *start, int *node_out) {
    return eval_full(p, opt, ord, start, node_out, NULL);
}

/* source: 0 index, 1 substream(seed, id), 2 SplitMix64(seed + id) */
int oracle_search(const oproblem *p, int source, uint64_t seed, uint64_t lo, uint64_t hi, int threads,
                  double *best_ms, uint64_t *best_id) {
    if (p->J < 1 || p->J > OMAX_J || p->N < 1 || p->N > OMAX_N) return 1;
    double gms = INFINITY;
    uint64_t gid = UINT64_MAX;
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
    {
        int nt = omp_get_num_threads(), t = omp_get_thread_num();
        uint64_t n = hi - lo;
        uint64_t a = lo + (uint64_t)((unsigned __int128)n * (unsigned)t / (unsigned)nt);
        uint64_t b = lo + (uint64_t)((unsigned __int128)n * (unsigned)(t + 1) / (unsigned)nt);
        int opt[OMAX_J], ord[OMAX_J];
        double ms_l = INFINITY;
        uint64_t id_l = UINT64_MAX;
        for (uint64_t id = a; id < b; ++id) {
            if (source == 0) {
                if (id == a) decode_index(p, id, opt, ord);
                else next_index(p, opt, ord);
            } else if (source == 1) {
                decode_stream(p, mix((seed ^ id) + GOLD), opt, ord);
            } else {
                decode_stream(p, seed + id, opt, ord);
            }
            double ms = oracle_eval(p, opt, ord, NULL, NULL);
            if (ms < ms_l) { ms_l = ms; id_l = id; }   /* ids ascend: first wins ties */
        }
#pragma omp critical
        {
            if (ms_l < gms || (ms_l == gms && id_l < gid)) { gms = ms_l; gid = id_l; }
        }
    }
    *best_ms = gms;
    *best_id = gid;
    return 0;
}

/* evaluate makespans of ids [lo, hi) into out[hi-lo] (window checks) */
int oracle_makespans(const oproblem *p, int source, uint64_t seed, uint64_t lo, uint64_t hi, double *out) {
    int opt[OMAX_J], ord[OMAX_J];
    for (uint64_t id = lo; id < hi; ++id) {
        if (source == 0) {
            if (id == lo) decode_index(p, id, opt, ord);
            else next_index(p, opt, ord);
        } else if (source == 1) {
            decode_stream(p, mix((seed ^ id) + GOLD), opt, ord);
        } else {
            decode_stream(p, seed + id, opt, ord);
        }
        out[id - lo] = oracle_eval(p, opt, ord, NULL, NULL);
    }
    return 0;
}

int oracle_decode(const oproblem *p, int source, uint64_t seed, uint64_t id, int *opt, int *ord) {
    if (source == 0) decode_index(p, id, opt, ord);
    else if (source == 1) decode_stream(p, mix((seed ^ id) + GOLD), opt, ord);
    else decode_stream(p, seed + id, opt, ord);
    return 0;
}

/* ---------------------------------------------------------------- local search
 * Same semantics as the engine's sat_local_search, restated with the
 * literal per-GPU list scheduler above:
 *   start: candidate `walker` of the stream (source 1 substream / 2 seed)
 *   moves, in this order:  [0, M1)       swap positions (a, b), a < b, lexicographic
 *                          [M1, M1+M2)   job j takes option o' != opt[j] (j, then o' ascending)
 *                          [M1+M2, M)    the job at position a moves to position b != a
 *                                        (a ascending, then b ascending)
 *   objective: (makespan, load) lexicographic, load = sum of the final free times of every
 *   GPU (it breaks the plateaus where several jobs pin the makespan)
 *   a round = 32 consecutive move ids; rounds are scanned from move 0; the first round
 *   holding a move with objective < current applies its best move (lowest objective, then
 *   lowest id) and the scan restarts at 0; a scan without improvement, or max_rounds
 *   rounds in total, ends the walk; with stop_ms >= 0 (the problem's lower bound) the walk
 *   also ends as soon as the current makespan is <= stop_ms.
 *   search over walkers: the lowest (makespan, rounds scanned, walker). */
static int ls_counts(const oproblem *p, int *M1, int *M2) {
    int J = p->J, m2 = 0;
    for (int j = 0; j < J; ++j) m2 += p->radix[j] - 1;
    *M1 = J * (J - 1) / 2;
    *M2 = m2;
    return *M1 + m2 + J * (J - 1);
}

static void ls_neighbor(const oproblem *p, int m, int M1, int M2, const int *opt, const int *ord, int *nopt,
                        int *nord) {
    int J = p->J;
    memcpy(nopt, opt, sizeof(int) * (size_t)J);
    memcpy(nord, ord, sizeof(int) * (size_t)J);
    if (m < M1) {
        int a = 0, rest = m;
        while (rest >= J - 1 - a) { rest -= J - 1 - a; ++a; }
        int b = a + 1 + rest;
        int t = nord[a]; nord[a] = nord[b]; nord[b] = t;
    } else if (m < M1 + M2) {
        int rest = m - M1, j = 0;
        while (rest >= p->radix[j] - 1) { rest -= p->radix[j] - 1; ++j; }
        nopt[j] = rest < opt[j] ? rest : rest + 1;
    } else {
        int rest = m - M1 - M2;
        int a = rest / (J - 1), bi = rest % (J - 1);
        int b = bi < a ? bi : bi + 1;
        int x = nord[a];
        if (a < b) memmove(nord + a, nord + a + 1, sizeof(int) * (size_t)(b - a));
        else memmove(nord + b + 1, nord + b, sizeof(int) * (size_t)(a - b));
        nord[b] = x;
    }
}

static double ls_walk(const oproblem *p, int max_rounds, int stop_ms, int *opt, int *ord, int *rounds_out);

/* greedy start (source 4; engine SAT_SRC_GREEDY): every job at its least-area option (area = g
 * x the least duration over the nodes that can run it, lowest option on ties); jobs ordered by
 * key = that duration x (2^17 + u_j) descending, lower job first on ties, u_j = the top 16 bits
 * of the j-th SplitMix64 output of the walker's substream state s0 */
static void greedy_start(const oproblem *p, uint64_t s0, int *opt, int *ord) {
    uint64_t key[OMAX_J];
    for (int j = 0; j < p->J; ++j) {
        double best_area = INFINITY, best_d = 0.0;
        int best_o = 0;
        for (int o = 0; o < p->radix[j]; ++o) {
            int q = j * p->Cmax + o;
            double d = INFINITY;
            for (int n = 0; n < p->N; ++n)
                if (((p->mask[q] >> n) & 1u) && p->gpus[q] <= p->node_gpus[n] && p->dur[q * p->N + n] < d)
                    d = p->dur[q * p->N + n];
            if (isinf(d)) continue;
            double area = (double)p->gpus[q] * d;
            if (area < best_area) { best_area = area; best_o = o; best_d = d; }
        }
        opt[j] = best_o;
        uint64_t u = mix(s0 + (uint64_t)(j + 1) * GOLD) >> 48;
        key[j] = (uint64_t)best_d * (131072ull + u);
    }
    for (int k = 0; k < p->J; ++k) {                  /* insertion sort: stable, key descending */
        int x = k, i = k;
        while (i > 0 && key[ord[i - 1]] < key[x]) { ord[i] = ord[i - 1]; --i; }
        ord[i] = x;
    }
}

double oracle_local_search(const oproblem *p, int source, uint64_t seed, uint64_t walker, int max_rounds,
                           int stop_ms, int *opt, int *ord, int *rounds_out) {
    if (source == 4) greedy_start(p, mix((seed ^ walker) + GOLD), opt, ord);
    else if (source == 1) decode_stream(p, mix((seed ^ walker) + GOLD), opt, ord);
    else decode_stream(p, seed + walker, opt, ord);
    return ls_walk(p, max_rounds, stop_ms, opt, ord, rounds_out);
}

/* the same walk from a given start (opt, ord are read, then overwritten with the final
 * candidate): walkers seeded with explicit candidates */
double oracle_local_search_from(const oproblem *p, int max_rounds, int stop_ms, int *opt, int *ord,
                                int *rounds_out) {
    return ls_walk(p, max_rounds, stop_ms, opt, ord, rounds_out);
}

static double ls_walk(const oproblem *p, int max_rounds, int stop_ms, int *opt, int *ord, int *rounds_out) {
    int M1, M2;
    int M = ls_counts(p, &M1, &M2);
    double cur_load;
    double cur = eval_full(p, opt, ord, NULL, NULL, &cur_load);
    int rounds = 0, nopt[OMAX_J], nord[OMAX_J];
    for (;;) {
        if (stop_ms >= 0 && cur <= (double)stop_ms) break;   /* at the bound: the walk ends */
        int improved = 0;
        for (int r0 = 0; r0 < M && rounds < max_rounds; r0 += 32, ++rounds) {
            double bms = INFINITY, bload = INFINITY;
            int bm = -1;
            for (int m = r0; m < r0 + 32 && m < M; ++m) {
                ls_neighbor(p, m, M1, M2, opt, ord, nopt, nord);
                double load;
                double ms = eval_full(p, nopt, nord, NULL, NULL, &load);
                if (ms < bms || (ms == bms && load < bload)) { bms = ms; bload = load; bm = m; }
            }
            if (bms < cur || (bms == cur && bload < cur_load)) {
                ls_neighbor(p, bm, M1, M2, opt, ord, nopt, nord);
                memcpy(opt, nopt, sizeof(int) * (size_t)p->J);
                memcpy(ord, nord, sizeof(int) * (size_t)p->J);
                cur = bms;
                cur_load = bload;
                improved = 1;
                ++rounds;
                break;
            }
        }
        if (!improved || rounds >= max_rounds) break;
    }
    if (rounds_out) *rounds_out = rounds;
    return cur;
}

int oracle_ls_search(const oproblem *p, int source, uint64_t seed, uint64_t lo, uint64_t hi, int max_rounds,
                     int stop_ms, int threads, double *best_ms, uint64_t *best_id) {
    double gms = INFINITY;
    uint64_t gid = UINT64_MAX;
    if (threads < 1) threads = omp_get_max_threads();
    int grounds = INT32_MAX;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (long long w = (long long)lo; w < (long long)hi; ++w) {
        int opt[OMAX_J], ord[OMAX_J], rounds = 0;
        double ms = oracle_local_search(p, source, seed, (uint64_t)w, max_rounds, stop_ms, opt, ord, &rounds);
#pragma omp critical
        {
            /* (makespan, rounds scanned, walker) lexicographic: the engine's local-search key */
            if (ms < gms || (ms == gms && (rounds < grounds || (rounds == grounds && (uint64_t)w < gid)))) {
                gms = ms; grounds = rounds; gid = (uint64_t)w;
            }
        }
    }
    *best_ms = gms;
    *best_id = gid;
    return 0;
}
