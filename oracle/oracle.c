/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the ScaleGANN
 * hot path computes (arxiv 2605.10135; /root/reference/PAPER.md, "P:n" below is
 * a PAPER.md line).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_2605_10135_b200/csrc); neither includes or links the other.
 *
 * Build: gcc -O2 -std=c11 -fPIC -shared -ffp-contract=off -fopenmp oracle.c
 * (no -ffast-math; fmaf() is used exactly where the reading says so).  OpenMP
 * parallelises over independent rows only, so results do not depend on the
 * thread count.
 *
 * Functions and what pins them (see DESIGN.md "Oracle readings" and tests/):
 *   oracle_kmeans          P0  k-means++ + Lloyd.  Pinned by
 *                              k=1 -> mean, k=#distinct -> 0 distortion,
 *                              non-increasing distortion.  Not in the bit-exact
 *                              chain (centroids are an input to partition).
 *   oracle_kmeans_distortion  the sample distortion that judges the GPU
 *                              k-means (R0); pinned by hand values on a line.
 *   oracle_centroid_dist   P1  fixed fp32 fmaf chain (reading R1).  Pinned by
 *                              exact small-integer cases.
 *   oracle_partition       P2/P3  blockwise-adaptive primaries + Algorithm 1
 *                              selective replicas (Alg. P:325-355).
 *                              Pinned by the Fig. 2 worked example
 *                              (tests/golden/fig2_partition.json), eps<=1 and
 *                              omega=1 degenerate cases, brute-force audit.
 *   oracle_knn             P4  exact brute-force top-L (definition).  Pinned
 *                              by 1-D line cases and m = L+1.
 *   oracle_prune           P5  rank-based detour-count prune.  PARITY UNPINNED
 *                              BY THE PAPER (the rule is CAGRA prior art, not in
 *                              PAPER.md); pinned by the hand-worked example of
 *                              tests/golden/prune_reverse_example.json and
 *                              invariants only.
 *   oracle_reverse         P6  reverse-edge insertion.  PARITY UNPINNED BY THE
 *                              PAPER (same reason); hand example + invariants,
 *                              and a second hand example where the (k, x) cap
 *                              order of rev[] decides the output
 *                              (tests/golden/reverse_order_example.json;
 *                              oracle_reverse_lists exposes rev[]).
 *   oracle_merge           P7  edge union + re-prune.  Pinned
 *                              by single-shard identity and the {a,b}u{b,c}
 *                              example, truncation optimality.
 *   oracle_entry_points    P7  entry point reading.
 *   oracle_search          P8  greedy best-first beam search.  Pinned
 *                              by beam = n -> exact top-k on a connected graph.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SENT 0xFFFFFFFFu

/* ---------------------------------------------------------------- helpers */

static float xval(const void* x, int dtype, uint64_t row, uint32_t d, uint32_t j) {
    if (dtype == 0) return (float)((const uint8_t*)x)[row * d + j];   /* u8 promoted exactly */
    return ((const float*)x)[row * d + j];
}

/* Exact distance of P4: u8 in int64, f32 in fp64, then rounded (RN) to float.
 * metric 0 = squared L2, 1 = negative inner product. */
static float exact_dist(const void* xa, uint64_t ra, const void* xb, uint64_t rb, int dtype,
                        uint32_t d, int metric) {
    if (dtype == 0) {
        const uint8_t* a = (const uint8_t*)xa + ra * d;
        const uint8_t* b = (const uint8_t*)xb + rb * d;
        int64_t s = 0;
        for (uint32_t j = 0; j < d; j++) {
            int64_t u = a[j], v = b[j];
            if (metric == 0) s += (u - v) * (u - v);
            else s -= u * v;
        }
        return (float)s;
    } else {
        const float* a = (const float*)xa + ra * d;
        const float* b = (const float*)xb + rb * d;
        double s = 0.0;
        for (uint32_t j = 0; j < d; j++) {
            double u = (double)a[j], v = (double)b[j];
            if (metric == 0) s += (u - v) * (u - v);
            else s -= u * v;
        }
        return (float)s;
    }
}

typedef struct { float d; uint32_t id; } pair_t;

static int cmp_pair(const void* pa, const void* pb) {   /* (dist, id) ascending */
    const pair_t* a = (const pair_t*)pa; const pair_t* b = (const pair_t*)pb;
    if (a->d < b->d) return -1;
    if (a->d > b->d) return 1;
    return (a->id > b->id) - (a->id < b->id);
}

static int cmp_pair_id(const void* pa, const void* pb) { /* (id, dist) ascending */
    const pair_t* a = (const pair_t*)pa; const pair_t* b = (const pair_t*)pb;
    if (a->id != b->id) return (a->id > b->id) - (a->id < b->id);
    return (a->d > b->d) - (a->d < b->d);
}

/* splitmix64: the counter-based generator the k-means seeding draws from */
static uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------ P0 */
/* k-means on a strided sample ("partitions the large dataset ... using
 * k-means clustering"; sampling per SPEC S:172).  sample[i] = floor(i*n/S),
 * S = min(n, spc*k).  k-means++ seeding from splitmix64(seed); Lloyd with fp64
 * distances, fp64 sums in sample order rounded to f32; empty cluster re-seeded
 * with the farthest point of the largest cluster; stop after max_iter or when
 * the relative distortion improvement is <= 1e-4.  Returns distortion (sum of
 * squared distances over the sample) of the returned centroids. */
static double d2_point_center(const void* x, int dtype, uint64_t row, uint32_t d, const float* c) {
    double s = 0.0;
    for (uint32_t j = 0; j < d; j++) {
        double t = (double)xval(x, dtype, row, d, j) - (double)c[j];
        s += t * t;
    }
    return s;
}

int oracle_kmeans(const void* x, int dtype, uint64_t n, uint32_t d, uint32_t k, uint64_t seed,
                  uint32_t max_iter, uint32_t spc, float* C, double* distortion_out) {
    if (k == 0 || n == 0 || d == 0) return 1;
    uint64_t S = (uint64_t)spc * k; if (S > n) S = n;
    if (S < k) return 1;
    uint64_t* smp = (uint64_t*)malloc(S * sizeof(uint64_t));
    for (uint64_t i = 0; i < S; i++) smp[i] = (uint64_t)(((unsigned __int128)i * n) / S);
    double* D2 = (double*)malloc(S * sizeof(double));
    uint32_t* asg = (uint32_t*)malloc(S * sizeof(uint32_t));
    double* sums = (double*)malloc((size_t)k * d * sizeof(double));
    uint64_t* cnt = (uint64_t*)malloc(k * sizeof(uint64_t));
    uint64_t st = seed;

    /* k-means++ seeding */
    uint64_t first = splitmix64(&st) % S;
    for (uint32_t j = 0; j < d; j++) C[j] = xval(x, dtype, smp[first], d, j);
    for (uint64_t i = 0; i < S; i++) D2[i] = d2_point_center(x, dtype, smp[i], d, C);
    for (uint32_t c = 1; c < k; c++) {
        double total = 0.0;
        for (uint64_t i = 0; i < S; i++) total += D2[i];
        double u = (double)(splitmix64(&st) >> 11) * (1.0 / 9007199254740992.0) * total;
        uint64_t pick = 0; double acc = 0.0;
        for (uint64_t i = 0; i < S; i++) { acc += D2[i]; if (acc > u) { pick = i; break; } pick = i; }
        for (uint32_t j = 0; j < d; j++) C[(size_t)c * d + j] = xval(x, dtype, smp[pick], d, j);
        for (uint64_t i = 0; i < S; i++) {
            double t = d2_point_center(x, dtype, smp[i], d, C + (size_t)c * d);
            if (t < D2[i]) D2[i] = t;
        }
    }

    double prev = INFINITY, dist = 0.0;
    for (uint32_t it = 0; it <= max_iter; it++) {
        /* assignment by (d^2, c) */
        dist = 0.0;
        for (uint64_t i = 0; i < S; i++) {
            double best = INFINITY; uint32_t bc = 0;
            for (uint32_t c = 0; c < k; c++) {
                double t = d2_point_center(x, dtype, smp[i], d, C + (size_t)c * d);
                if (t < best) { best = t; bc = c; }
            }
            asg[i] = bc; D2[i] = best; dist += best;
        }
        if (it == max_iter) break;
        if (prev < INFINITY && (prev - dist) <= 1e-4 * prev) break;
        prev = dist;
        /* update: fp64 sums in sample order, rounded to f32 */
        memset(sums, 0, (size_t)k * d * sizeof(double));
        memset(cnt, 0, k * sizeof(uint64_t));
        for (uint64_t i = 0; i < S; i++) {
            cnt[asg[i]]++;
            for (uint32_t j = 0; j < d; j++) sums[(size_t)asg[i] * d + j] += (double)xval(x, dtype, smp[i], d, j);
        }
        for (uint32_t c = 0; c < k; c++) {
            if (cnt[c] == 0) {
                uint32_t big = 0;
                for (uint32_t c2 = 1; c2 < k; c2++) if (cnt[c2] > cnt[big]) big = c2;
                uint64_t far = 0; double fd = -1.0;
                for (uint64_t i = 0; i < S; i++) if (asg[i] == big && D2[i] > fd) { fd = D2[i]; far = i; }
                for (uint32_t j = 0; j < d; j++) C[(size_t)c * d + j] = xval(x, dtype, smp[far], d, j);
                D2[far] = 0.0;
            } else {
                for (uint32_t j = 0; j < d; j++) C[(size_t)c * d + j] = (float)(sums[(size_t)c * d + j] / (double)cnt[c]);
            }
        }
    }
    if (distortion_out) *distortion_out = dist;
    free(smp); free(D2); free(asg); free(sums); free(cnt);
    return 0;
}

/* Distortion of given centroids on the same strided sample (for the GPU
 * k-means acceptance rule: <= 1.01 x the oracle's). */
double oracle_kmeans_distortion(const void* x, int dtype, uint64_t n, uint32_t d, uint32_t k,
                                uint32_t spc, const float* C) {
    uint64_t S = (uint64_t)spc * k; if (S > n) S = n;
    double dist = 0.0;
    for (uint64_t i = 0; i < S; i++) {
        uint64_t row = (uint64_t)(((unsigned __int128)i * n) / S);
        double best = INFINITY;
        for (uint32_t c = 0; c < k; c++) {
            double t = d2_point_center(x, dtype, row, d, C + (size_t)c * d);
            if (t < best) best = t;
        }
        dist += best;
    }
    return dist;
}

/* ------------------------------------------------------------------ P1 */
/* d^2(v,c) = fold_j acc = fmaf(diff, diff, acc), diff = (float)x_j - c_j (RN),
 * acc starting at 0 (reading R1 — the paper fixes no formula; this one makes
 * every eps/radius/capacity decision reproducible). */
void oracle_centroid_dist(const void* x, int dtype, uint64_t n, uint32_t d, const float* C,
                          uint32_t k, float* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < (int64_t)n; v++) {
        for (uint32_t c = 0; c < k; c++) {
            float acc = 0.0f;
            for (uint32_t j = 0; j < d; j++) {
                float diff = xval(x, dtype, (uint64_t)v, d, j) - C[(size_t)c * d + j];
                acc = fmaf(diff, diff, acc);
            }
            out[(size_t)v * k + c] = acc;
        }
    }
}

/* ------------------------------------------------------------------ P2/P3 */
/* capacity = ceil(1.15 * ceil(n / (k (1 - theta0)))) in integers (reading R9).
 * Replicas may take up to theta0*cap of a cluster (budget, R4), so this sizing keeps
 * k*cap*(1-theta0) >= 1.15 n: room for every original vector is always left, as P:307
 * requires ("each cluster must reserve capacity for original vectors processed later") and
 * SPEC S:182 states as an invariant.  SPEC S:242's ceil(1.15*ceil(n(1+theta0)/k)) does not
 * guarantee it (replicas can exhaust it: SG_ERR_CAPACITY on clustered data). */
uint64_t oracle_capacity(uint64_t n, uint32_t k, uint32_t theta0_ppm) {
    unsigned __int128 num = (unsigned __int128)1000000u * n;
    unsigned __int128 den = (unsigned __int128)(1000000u - theta0_ppm) * k;
    unsigned __int128 base = (num + den - 1) / den;
    return (uint64_t)((base * 115 + 99) / 100);
}

/* Replica budget (reading R4, SPEC S:259 made exact):
 * floor(t * cap * min(k*prim_c, P) / (1e6 * k * prim_c)), t = theta0_ppm,
 * P = sum of primaries; prim_c = 0 -> floor(t * cap / 1e6). */
static uint64_t budget_of(uint64_t prim_c, uint64_t P, uint32_t k, uint32_t t, uint64_t cap) {
    if (prim_c == 0) return (uint64_t)(((unsigned __int128)t * cap) / 1000000u);
    unsigned __int128 kp = (unsigned __int128)k * prim_c;
    unsigned __int128 mn = kp < P ? kp : (unsigned __int128)P;
    unsigned __int128 num = (unsigned __int128)t * cap * mn;
    unsigned __int128 den = (unsigned __int128)1000000u * kp;
    return (uint64_t)(num / den);
}

/* Blockwise-adaptive partition with selective replication.
 * For each block b (B vectors in id order): (1) every vector to its
 * nearest cluster with size < capacity, radius over
 * primaries (reading R6); (2) update statistics: tau_b = 1 + alpha/(1+b)
 * (reading R5) and replica budgets (R4); (3) Algorithm 1 lines 1-11
 * for each vector in id order: iterate clusters by ascending (d^2, c), stop
 * at omega homes, skip the primary, skip clusters failing checkSizeLimit
 * (size < cap and repl < budget, reading R7), place a replica iff
 * d' < eps*d and d' < (eps*tau_b)*radius[c'] (fp32 RN products).
 * home[v*omega ..] = [primary, replicas in placement order, SENT...].
 * Returns 0, or 4 (= SG_ERR_CAPACITY) when a primary finds every cluster full. */
int oracle_partition(const void* x, int dtype, uint64_t n, uint32_t d, const float* C, uint32_t k,
                     uint32_t omega, float eps, uint32_t theta0_ppm, float alpha, uint64_t capacity,
                     uint32_t block_size, uint32_t* home, float* primary_d, uint64_t* sizes,
                     uint64_t* prim, uint64_t* repl, float* radius_out) {
    uint64_t cap = capacity ? capacity : oracle_capacity(n, k, theta0_ppm);
    float* dist = (float*)malloc((size_t)n * k * sizeof(float));
    oracle_centroid_dist(x, dtype, n, d, C, k, dist);
    float* radius = (float*)calloc(k, sizeof(float));
    uint64_t* budget = (uint64_t*)calloc(k, sizeof(uint64_t));
    uint32_t* order = (uint32_t*)malloc(k * sizeof(uint32_t));
    for (uint32_t c = 0; c < k; c++) { sizes[c] = 0; prim[c] = 0; repl[c] = 0; }
    int status = 0;
    uint64_t nblocks = (n + block_size - 1) / block_size;
    for (uint64_t b = 0; b < nblocks && status == 0; b++) {
        uint64_t v0 = b * block_size, v1 = v0 + block_size < n ? v0 + block_size : n;
        /* (1) primaries */
        for (uint64_t v = v0; v < v1; v++) {
            const float* dv = dist + v * k;
            for (uint32_t i = 0; i < k; i++) {            /* insertion sort by (d, c) */
                uint32_t c = i, j = i;
                while (j > 0 && (dv[order[j - 1]] > dv[c])) { order[j] = order[j - 1]; j--; }
                order[j] = c;
            }
            uint32_t p = SENT;
            for (uint32_t i = 0; i < k; i++) if (sizes[order[i]] < cap) { p = order[i]; break; }
            if (p == SENT) { status = 4; break; }
            sizes[p]++; prim[p]++;
            if (dv[p] > radius[p]) radius[p] = dv[p];
            home[v * omega] = p;
            for (uint32_t h = 1; h < omega; h++) home[v * omega + h] = SENT;
            primary_d[v] = dv[p];
        }
        if (status) break;
        /* (2) statistics and thresholds */
        float tau = 1.0f + alpha / (float)(1 + b);
        uint64_t P = 0;
        for (uint32_t c = 0; c < k; c++) P += prim[c];
        for (uint32_t c = 0; c < k; c++) budget[c] = budget_of(prim[c], P, k, theta0_ppm, cap);
        /* (3) Algorithm 1 */
        for (uint64_t v = v0; v < v1; v++) {
            const float* dv = dist + v * k;
            for (uint32_t i = 0; i < k; i++) {
                uint32_t c = i, j = i;
                while (j > 0 && (dv[order[j - 1]] > dv[c])) { order[j] = order[j - 1]; j--; }
                order[j] = c;
            }
            uint32_t p = home[v * omega];
            float dd = dv[p];
            uint32_t assigned = 1;
            for (uint32_t i = 0; i < k; i++) {
                uint32_t c2 = order[i];
                if (assigned >= omega) break;
                if (c2 == p) continue;
                if (!(sizes[c2] < cap && repl[c2] < budget[c2])) continue;
                float d2 = dv[c2];
                float e_d = eps * dd;
                float e_t = eps * tau;
                float e_t_r = e_t * radius[c2];
                if (d2 < e_d && d2 < e_t_r) {
                    sizes[c2]++; repl[c2]++;
                    home[v * omega + assigned] = c2;
                    assigned++;
                }
            }
        }
    }
    if (radius_out) memcpy(radius_out, radius, k * sizeof(float));
    free(dist); free(radius); free(budget); free(order);
    return status;
}

/* idmap_s = ascending global ids of {v : s in home[v]} (reading R8). */
uint64_t oracle_idmap(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t s, uint32_t* out) {
    uint64_t m = 0;
    for (uint64_t v = 0; v < n; v++)
        for (uint32_t h = 0; h < omega; h++)
            if (home[v * omega + h] == s) { if (out) out[m] = (uint32_t)v; m++; break; }
    return m;
}

/* ------------------------------------------------------------------ P4 */
/* Exact kNN: for each row i of A, the L smallest (dist, j) over rows j of B,
 * j != i when self_exclude (A and B the same set).  ida/idb map local -> global
 * rows of the data arrays (NULL = identity).  Padded with (SENT, +inf). */
/* (dist, id) order of cmp_pair as a predicate: a before b */
static int pair_before(float da, uint32_t ia, float db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

void oracle_knn(const void* xa, const uint32_t* ida, uint64_t ma, const void* xb, const uint32_t* idb,
                uint64_t mb, int dtype, uint32_t d, int self_exclude, uint32_t L, int metric,
                uint32_t* out_ids, float* out_d) {
    if (L == 0) return;
    /* The L smallest (dist, j) are kept in a sorted list (insertion), which equals the
     * first L entries of the fully sorted candidate list without sorting all mb of them. */
    #pragma omp parallel
    {
        pair_t* best = (pair_t*)malloc((L + 1) * sizeof(pair_t));
        #pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < (int64_t)ma; i++) {
            uint64_t ra = ida ? ida[i] : (uint64_t)i;
            uint32_t cnt = 0;
            for (uint64_t j = 0; j < mb; j++) {
                if (self_exclude && j == (uint64_t)i) continue;
                uint64_t rb = idb ? idb[j] : j;
                float dj = exact_dist(xa, ra, xb, rb, dtype, d, metric);
                if (cnt == L && !pair_before(dj, (uint32_t)j, best[L - 1].d, best[L - 1].id)) continue;
                uint32_t p = cnt < L ? cnt++ : L - 1;      /* drop the current L-th when full */
                while (p > 0 && pair_before(dj, (uint32_t)j, best[p - 1].d, best[p - 1].id)) {
                    best[p] = best[p - 1];
                    p--;
                }
                best[p].d = dj;
                best[p].id = (uint32_t)j;
            }
            for (uint32_t p = 0; p < L; p++) {
                if (p < cnt) { out_ids[i * L + p] = best[p].id; out_d[i * L + p] = best[p].d; }
                else { out_ids[i * L + p] = SENT; out_d[i * L + p] = INFINITY; }
            }
        }
        free(best);
    }
}

/* ------------------------------------------------------------------ P5 */
/* Rank-based detour-count prune (reading R10; CAGRA prior art, not in PAPER.md).
 * For node a with list N[a] (rank = position): for every r_ad, delta = N[a][r_ad],
 * for every r_db, b = N[delta][r_db]: if b is in N[a] at rank r_ab and
 * max(r_ad, r_db) < r_ab (rule 0) [rule 1: r_ad < r_ab], cnt[r_ab]++.
 * Keep the first R ranks of the stable order by (cnt, rank), sentinel ranks last. */
void oracle_prune(const uint32_t* knn, const float* knn_d, uint64_t m, uint32_t L, uint32_t R,
                  int rule, uint32_t* out, float* out_d) {
    #pragma omp parallel
    {
        uint64_t* key = (uint64_t*)malloc(L * sizeof(uint64_t));
        uint32_t* cnt = (uint32_t*)malloc(L * sizeof(uint32_t));
        /* rank_of[b] = r_ab for b in N[a] (first occurrence), SENT otherwise; set for the
         * current a and cleared after it */
        uint32_t* rank_of = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
        for (uint64_t b = 0; b < m; b++) rank_of[b] = SENT;
        #pragma omp for schedule(dynamic, 64)
        for (int64_t a = 0; a < (int64_t)m; a++) {
            const uint32_t* Na = knn + (uint64_t)a * L;
            memset(cnt, 0, L * sizeof(uint32_t));
            for (uint32_t r = L; r-- > 0;)
                if (Na[r] != SENT) rank_of[Na[r]] = r;
            for (uint32_t r_ad = 0; r_ad < L; r_ad++) {
                uint32_t delta = Na[r_ad];
                if (delta == SENT) continue;
                const uint32_t* Nd = knn + (uint64_t)delta * L;
                for (uint32_t r_db = 0; r_db < L; r_db++) {
                    uint32_t b = Nd[r_db];
                    if (b == SENT || b == (uint32_t)a) continue;
                    uint32_t r_ab = rank_of[b];
                    if (r_ab == SENT) continue;             /* b not in N[a] */
                    uint32_t mx = rule == 0 ? (r_ad > r_db ? r_ad : r_db) : r_ad;
                    if (mx < r_ab) cnt[r_ab]++;
                }
            }
            for (uint32_t r = 0; r < L; r++)
                if (Na[r] != SENT) rank_of[Na[r]] = SENT;
            for (uint32_t r = 0; r < L; r++)
                key[r] = Na[r] == SENT ? (0xFFFFFFFFull << 32) | r : ((uint64_t)cnt[r] << 32) | r;
            for (uint32_t i = 1; i < L; i++) {     /* stable insertion sort */
                uint64_t kk = key[i]; uint32_t j = i;
                while (j > 0 && key[j - 1] > kk) { key[j] = key[j - 1]; j--; }
                key[j] = kk;
            }
            for (uint32_t i = 0; i < R; i++) {
                uint32_t r = (uint32_t)(key[i] & 0xFFFFFFFFu);
                out[(uint64_t)a * R + i] = Na[r];
                out_d[(uint64_t)a * R + i] = knn_d[(uint64_t)a * L + r];
            }
        }
        free(key); free(cnt); free(rank_of);
    }
}

/* ------------------------------------------------------------------ P6 */
/* Reverse-edge insertion (reading R11).  rev[y] = sources x ordered by (k, x)
 * where y = pruned[x][k], appended while |rev[y]| < R.  With h protected
 * forward edges: rev_np = [x in rev[y] : x not in pruned[y][0..h)],
 * tail = rev_np ++ [f in pruned[y][h..R) : f not in rev_np],
 * out[y] = pruned[y][0..h) ++ tail[0..R-h).  A reverse edge y->x carries the
 * distance of x->y. */
/* rev[y] (m x R, SENT padded) and |rev[y]| (rc) of reading R11: sources x in (k, x)
 * order -- k outer, x inner -- appended while |rev[y]| < R; rev_d carries d(x -> y). */
void oracle_reverse_lists(const uint32_t* pruned, const float* pruned_d, uint64_t m, uint32_t R,
                          uint32_t* rev, float* rev_d, uint32_t* rc) {
    for (uint64_t y = 0; y < m * R; y++) { rev[y] = SENT; rev_d[y] = INFINITY; }
    memset(rc, 0, m * sizeof(uint32_t));
    for (uint32_t k = 0; k < R; k++)
        for (uint64_t x = 0; x < m; x++) {
            uint32_t y = pruned[x * R + k];
            if (y == SENT) continue;
            if (rc[y] < R) { rev[(uint64_t)y * R + rc[y]] = (uint32_t)x; rev_d[(uint64_t)y * R + rc[y]] = pruned_d[x * R + k]; rc[y]++; }
        }
}

void oracle_reverse(const uint32_t* pruned, const float* pruned_d, uint64_t m, uint32_t R,
                    uint32_t h, uint32_t* out, float* out_d) {
    uint32_t* rev = (uint32_t*)malloc((size_t)m * R * sizeof(uint32_t));
    float* rev_d = (float*)malloc((size_t)m * R * sizeof(float));
    uint32_t* rc = (uint32_t*)calloc(m, sizeof(uint32_t));
    oracle_reverse_lists(pruned, pruned_d, m, R, rev, rev_d, rc);
    #pragma omp parallel
    {
        uint32_t* tail = (uint32_t*)malloc(2 * R * sizeof(uint32_t));
        float* tail_d = (float*)malloc(2 * R * sizeof(float));
        #pragma omp for schedule(static)
        for (int64_t y = 0; y < (int64_t)m; y++) {
            const uint32_t* P = pruned + (uint64_t)y * R;
            const float* Pd = pruned_d + (uint64_t)y * R;
            uint32_t nt = 0, nrev = 0;
            for (uint32_t i = 0; i < rc[y]; i++) {
                uint32_t xx = rev[(uint64_t)y * R + i];
                int in_p = 0;
                for (uint32_t j = 0; j < h; j++) if (P[j] == xx) { in_p = 1; break; }
                if (!in_p) { tail[nt] = xx; tail_d[nt] = rev_d[(uint64_t)y * R + i]; nt++; }
            }
            nrev = nt;
            for (uint32_t j = h; j < R; j++) {
                int in_r = 0;
                for (uint32_t i = 0; i < nrev; i++) if (tail[i] == P[j]) { in_r = 1; break; }
                if (!in_r) { tail[nt] = P[j]; tail_d[nt] = Pd[j]; nt++; }
            }
            for (uint32_t j = 0; j < h; j++) { out[(uint64_t)y * R + j] = P[j]; out_d[(uint64_t)y * R + j] = Pd[j]; }
            for (uint32_t j = h; j < R; j++) { out[(uint64_t)y * R + j] = tail[j - h]; out_d[(uint64_t)y * R + j] = tail_d[j - h]; }
        }
        free(tail); free(tail_d);
    }
    free(rev); free(rev_d); free(rc);
}

/* ------------------------------------------------------------------ P7 */
static uint64_t local_of(const uint32_t* idmap, uint64_t m, uint32_t g) {   /* binary search */
    uint64_t lo = 0, hi = m;
    while (lo < hi) { uint64_t mid = (lo + hi) / 2; if (idmap[mid] < g) lo = mid + 1; else hi = mid; }
    return lo;
}

/* Merge by edge union (reading R12).  For each
 * global g with homes H: |H| = 1 -> the home row mapped local->global as is;
 * |H| > 1 -> union of the mapped rows, dedupe by gid keeping the minimum
 * carried distance, sort by (dist, gid), first R. */
void oracle_merge(const uint32_t* home, uint64_t n, uint32_t omega, const uint32_t* const* idmaps,
                  const uint64_t* sizes, const uint32_t* const* graphs, const float* const* graphs_d,
                  uint32_t R, uint32_t* merged, float* merged_d) {
    #pragma omp parallel
    {
        pair_t* U = (pair_t*)malloc((size_t)omega * R * sizeof(pair_t));
        #pragma omp for schedule(static)
        for (int64_t g = 0; g < (int64_t)n; g++) {
            uint32_t nh = 0;
            for (uint32_t h = 0; h < omega; h++) if (home[(uint64_t)g * omega + h] != SENT) nh++;
            if (nh == 1) {
                uint32_t s = home[(uint64_t)g * omega];
                uint64_t l = local_of(idmaps[s], sizes[s], (uint32_t)g);
                for (uint32_t j = 0; j < R; j++) {
                    uint32_t lid = graphs[s][l * R + j];
                    merged[(uint64_t)g * R + j] = lid == SENT ? SENT : idmaps[s][lid];
                    merged_d[(uint64_t)g * R + j] = graphs_d[s][l * R + j];
                }
                continue;
            }
            uint32_t nu = 0;
            for (uint32_t h = 0; h < omega; h++) {
                uint32_t s = home[(uint64_t)g * omega + h];
                if (s == SENT) continue;
                uint64_t l = local_of(idmaps[s], sizes[s], (uint32_t)g);
                for (uint32_t j = 0; j < R; j++) {
                    uint32_t lid = graphs[s][l * R + j];
                    if (lid == SENT) continue;
                    U[nu].id = idmaps[s][lid]; U[nu].d = graphs_d[s][l * R + j]; nu++;
                }
            }
            qsort(U, nu, sizeof(pair_t), cmp_pair_id);
            uint32_t w = 0;
            for (uint32_t i = 0; i < nu; i++) if (w == 0 || U[w - 1].id != U[i].id) U[w++] = U[i];
            qsort(U, w, sizeof(pair_t), cmp_pair);
            for (uint32_t j = 0; j < R; j++) {
                merged[(uint64_t)g * R + j] = j < w ? U[j].id : SENT;
                merged_d[(uint64_t)g * R + j] = j < w ? U[j].d : INFINITY;
            }
        }
        free(U);
    }
}

/* Entry points (reading R13): per shard, argmin over its primaries of
 * (primary_d, gid); global: the entry of the largest shard, ties -> lower id. */
uint32_t oracle_entry_points(const uint32_t* home, const float* primary_d, uint64_t n, uint32_t omega,
                             uint32_t k, const uint64_t* sizes, uint32_t* entry_per_shard) {
    for (uint32_t s = 0; s < k; s++) entry_per_shard[s] = SENT;
    float* best = (float*)malloc(k * sizeof(float));
    for (uint32_t s = 0; s < k; s++) best[s] = INFINITY;
    for (uint64_t g = 0; g < n; g++) {
        uint32_t s = home[g * omega];
        if (entry_per_shard[s] == SENT || primary_d[g] < best[s]) { best[s] = primary_d[g]; entry_per_shard[s] = (uint32_t)g; }
    }
    free(best);
    uint32_t big = 0;
    for (uint32_t s = 1; s < k; s++) if (sizes[s] > sizes[big]) big = s;
    return entry_per_shard[big];
}

/* ------------------------------------------------------------------ P8 */
/* Greedy best-first beam search ("following DiskANN's search strategy";
 * SPEC S:455-481; reading R14).  pool = [(d(q,entry), entry)], visited = {entry};
 * repeat: take the lowest (dist, id) unexpanded u, mark it expanded, add every
 * non-sentinel unvisited neighbour v of u as (d(q,v), v), sort by (dist, id),
 * truncate to beam; stop when every pool entry is expanded; return the first topk. */
typedef struct { float d; uint32_t id; uint32_t exp; } pool_t;
static int cmp_pool(const void* pa, const void* pb) {
    const pool_t* a = (const pool_t*)pa; const pool_t* b = (const pool_t*)pb;
    if (a->d < b->d) return -1;
    if (a->d > b->d) return 1;
    return (a->id > b->id) - (a->id < b->id);
}

void oracle_search(const void* x, int dtype, uint64_t n, uint32_t d, const uint32_t* graph, uint32_t R,
                   uint32_t entry, const void* q, uint32_t nq, uint32_t topk, uint32_t beam, int metric,
                   uint32_t* out_ids, float* out_d, uint64_t* n_dist) {
    #pragma omp parallel
    {
        uint8_t* visited = (uint8_t*)malloc(n);
        pool_t* pool = (pool_t*)malloc((beam + R + 1) * sizeof(pool_t));
        #pragma omp for schedule(dynamic, 4)
        for (int64_t qi = 0; qi < (int64_t)nq; qi++) {
            memset(visited, 0, n);
            uint64_t nd = 1;
            uint32_t np = 1;
            pool[0].d = exact_dist(q, (uint64_t)qi, x, entry, dtype, d, metric);
            pool[0].id = entry; pool[0].exp = 0;
            visited[entry] = 1;
            for (;;) {
                uint32_t u = SENT;
                for (uint32_t i = 0; i < np; i++) if (!pool[i].exp) { u = i; break; }
                if (u == SENT) break;
                pool[u].exp = 1;
                uint32_t node = pool[u].id;
                for (uint32_t j = 0; j < R; j++) {
                    uint32_t v = graph[(uint64_t)node * R + j];
                    if (v == SENT || visited[v]) continue;
                    visited[v] = 1;
                    pool[np].d = exact_dist(q, (uint64_t)qi, x, v, dtype, d, metric);
                    pool[np].id = v; pool[np].exp = 0; np++; nd++;
                }
                qsort(pool, np, sizeof(pool_t), cmp_pool);
                if (np > beam) np = beam;
            }
            for (uint32_t i = 0; i < topk; i++) {
                out_ids[(uint64_t)qi * topk + i] = i < np ? pool[i].id : SENT;
                if (out_d) out_d[(uint64_t)qi * topk + i] = i < np ? pool[i].d : INFINITY;
            }
            if (n_dist) n_dist[qi] = nd;
        }
        free(visited); free(pool);
    }
}

/* exported for the budget pin ("2x the mean primary share -> theta0 x cap x 0.5") */
uint64_t oracle_budget(uint64_t prim_c, uint64_t P, uint32_t k, uint32_t theta0_ppm, uint64_t cap) {
    return budget_of(prim_c, P, k, theta0_ppm, cap);
}
