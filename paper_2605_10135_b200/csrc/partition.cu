// a2-a3 — overlapping balanced partition (Algorithm 1).
//
// K1 centroid_dist_order: d^2(v,c) for every vector and centroid in the fixed fp32 order of
//    reading R1 (acc = fma(diff, diff, acc), diff = x_j - c_j, j = 0..d-1), plus the
//    preference order of v = clusters sorted by (d^2, c).  Rows are staged through shared
//    memory 32 x 32 at a time so the HBM reads are coalesced.
// K2 assign_kernel: the block-by-block sequential semantics of P:312 (primaries -> statistics
//    -> replicas, each vector in id order) computed by ONE cooperative CTA with
//    speculate-and-verify: every vector of the block proposes its choice(s) against the
//    current set of open clusters; per-cluster prefix counts locate the first vector whose
//    placement would overflow a cluster; everything before it is exactly what the sequential
//    pass does; the cluster closes (it never reopens) and speculation resumes at that vector.
//    So a block costs <= k+1 rounds per phase and the result is bit-identical to the oracle.
//    Default: assign_grid_kernel runs each round on the whole GPU (cooperative launch, grid
//    barriers between count / cut / commit); assign_kernel (one CTA) stays as the reference
//    variant (SG_PART_SINGLE_CTA=1).
#include <stdlib.h>

#include "common.cuh"

namespace sg {
namespace {

constexpr int K2_THREADS = 1024;
constexpr int KMAX = 64;

// KB >= k: compile-time bound for the per-vector arrays (registers, static indexing); the
// centroids are staged in shared memory when they fit (SMEM_C), else read through L1.
template <int KB, bool SMEM_C>
__global__ void __launch_bounds__(256) centroid_dist_order(const void* __restrict__ x, int dtype, uint64_t n,
                                                           uint32_t d, const float* __restrict__ C, uint32_t k,
                                                           float* __restrict__ dist, uint8_t* __restrict__ order) {
    __shared__ float tile[8][32][33];
    extern __shared__ float sC[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (SMEM_C) {
        for (uint32_t e = threadIdx.x; e < k * d; e += blockDim.x) sC[e] = C[e];
        __syncthreads();
    }
    const float* Cs = SMEM_C ? sC : C;
    const uint64_t v0 = ((uint64_t)blockIdx.x * 8 + warp) * 32;
    if (v0 >= n) return;
    const uint64_t v = v0 + lane;
    float acc[KB];
#pragma unroll
    for (int c = 0; c < KB; c++) acc[c] = 0.f;
    for (uint32_t j0 = 0; j0 < d; j0 += 32) {
        // coalesced load of rows v0..v0+31, columns j0..j0+31 (transposed through smem)
        for (int rr = 0; rr < 32; rr++) {
            uint64_t row = v0 + rr;
            uint32_t col = j0 + lane;
            float val = 0.f;
            if (row < n && col < d)
                val = dtype == SG_U8 ? (float)((const uint8_t*)x)[row * d + col] : ((const float*)x)[row * d + col];
            tile[warp][rr][lane] = val;
        }
        __syncwarp();
        const uint32_t jn = d - j0 < 32 ? d - j0 : 32;
        if (SMEM_C && (d & 3) == 0 && jn == 32) {
            // 4 dimensions of this lane's vector in registers, reused by every centroid (read
            // as one 16-byte broadcast); per (v, c) the fmaf chain stays in j order (reading R1)
            for (uint32_t jj = 0; jj < 32; jj += 4) {
                const float t0 = tile[warp][lane][jj], t1 = tile[warp][lane][jj + 1];
                const float t2 = tile[warp][lane][jj + 2], t3 = tile[warp][lane][jj + 3];
#pragma unroll
                for (int c = 0; c < KB; c++) {
                    if ((uint32_t)c < k) {
                        const float4 c4 = *(const float4*)(Cs + (size_t)c * d + j0 + jj);
                        float a = acc[c], df;
                        df = __fsub_rn(t0, c4.x); a = __fmaf_rn(df, df, a);
                        df = __fsub_rn(t1, c4.y); a = __fmaf_rn(df, df, a);
                        df = __fsub_rn(t2, c4.z); a = __fmaf_rn(df, df, a);
                        df = __fsub_rn(t3, c4.w); a = __fmaf_rn(df, df, a);
                        acc[c] = a;
                    }
                }
            }
        } else {
#pragma unroll
            for (int c = 0; c < KB; c++) {
                if ((uint32_t)c < k) {
                    float a = acc[c];
                    const float* cc = Cs + (size_t)c * d + j0;
                    for (uint32_t jj = 0; jj < jn; jj++) {
                        // the fixed fp32 order of reading R1: acc = fma(diff, diff, acc), j ascending
                        float diff = __fsub_rn(tile[warp][lane][jj], SMEM_C ? cc[jj] : __ldg(cc + jj));
                        a = __fmaf_rn(diff, diff, a);
                    }
                    acc[c] = a;
                }
            }
        }
        __syncwarp();
    }
    if (v >= n) return;
    // preference order by (d^2, c): the rank of c is the number of (d^2, c') before it
#pragma unroll
    for (int c = 0; c < KB; c++) {
        if ((uint32_t)c < k) {
            dist[v * k + c] = acc[c];
            uint32_t rank = 0;
#pragma unroll
            for (int c2 = 0; c2 < KB; c2++)
                if ((uint32_t)c2 < k && (acc[c2] < acc[c] || (acc[c2] == acc[c] && c2 < c))) rank++;
            order[v * k + rank] = (uint8_t)c;
        }
    }
}

struct PartState {
    uint64_t size[KMAX], prim[KMAX], repl[KMAX], budget[KMAX];
    float radius[KMAX];
    int status;
};

struct PartArgs {
    const float* dist;      // n x k
    const uint8_t* order;   // n x k
    uint32_t* home;         // n x omega
    float* primary_d;       // n
    PartState* state;       // global copy of the final state
    uint64_t n, cap;
    uint32_t k, omega, block, theta0;
    float eps, alpha;
};

__device__ __forceinline__ uint64_t budget_of(uint64_t prim_c, uint64_t P, uint32_t k, uint32_t t, uint64_t cap) {
    if (prim_c == 0) return (uint64_t)(((unsigned __int128)t * cap) / 1000000u);
    unsigned __int128 kp = (unsigned __int128)k * prim_c;
    unsigned __int128 mn = kp < (unsigned __int128)P ? kp : (unsigned __int128)P;
    return (uint64_t)(((unsigned __int128)t * cap * mn) / ((unsigned __int128)1000000u * kp));
}

// replica picks of one vector against the open mask; returns the count and fills picks[]
__device__ __forceinline__ uint32_t replica_picks(const PartArgs& a, uint64_t v, uint64_t open, float tau,
                                                  const float* radius, uint32_t* picks) {
    const float* dv = a.dist + v * a.k;
    const uint8_t* ov = a.order + v * a.k;
    const uint32_t p = a.home[v * a.omega];
    const float dd = dv[p];
    const float e_d = __fmul_rn(a.eps, dd);
    const float e_t = __fmul_rn(a.eps, tau);
    uint32_t assigned = 1, np = 0;
    for (uint32_t i = 0; i < a.k; i++) {
        if (assigned >= a.omega) break;
        const uint32_t c = ov[i];
        if (c == p) continue;
        const float d2 = dv[c];
        if (!(d2 < e_d)) break;   // order is ascending in d2: every later c fails the distance test too
        if (!((open >> c) & 1ull)) continue;
        if (d2 < __fmul_rn(e_t, radius[c])) { picks[np++] = c; assigned++; }
    }
    return np;
}

__global__ void __launch_bounds__(K2_THREADS, 1) assign_kernel(PartArgs a) {
    __shared__ PartState st;
    __shared__ uint32_t scan_tmp[33];
    __shared__ uint64_t s_cut;
    __shared__ uint32_t s_cut_c;
    extern __shared__ uint16_t cnts[];   // [k][K2_THREADS] per-thread counts for the current round
    const uint32_t tid = threadIdx.x;
    const uint32_t k = a.k;
    if (tid < k) { st.size[tid] = st.prim[tid] = st.repl[tid] = st.budget[tid] = 0; st.radius[tid] = 0.f; }
    if (tid == 0) st.status = 0;
    __syncthreads();
    const uint64_t nblocks = (a.n + a.block - 1) / a.block;
    for (uint64_t b = 0; b < nblocks; b++) {
        const uint64_t v0 = b * a.block, v1 = min(a.n, v0 + a.block);
        const uint64_t seg = (v1 - v0 + K2_THREADS - 1) / K2_THREADS;
        const uint64_t s0 = v0 + tid * seg, s1 = min(v1, s0 + seg);
        // ---------------- (1) primaries: nearest cluster with size < capacity
        uint64_t start = v0;
        while (true) {
            uint64_t open = 0;
            for (uint32_t c = 0; c < k; c++) if (st.size[c] < a.cap) open |= 1ull << c;
            __syncthreads();
            if (open == 0) { if (tid == 0) st.status = SG_ERR_CAPACITY; break; }
            for (uint32_t c = 0; c < k; c++) cnts[c * K2_THREADS + tid] = 0;
            const uint64_t lo = max(start, s0);
            for (uint64_t v = lo; v < s1; v++) {
                const uint8_t* ov = a.order + v * k;
                uint32_t c = 0;
                for (uint32_t i = 0; i < k; i++) if ((open >> ov[i]) & 1ull) { c = ov[i]; break; }
                cnts[c * K2_THREADS + tid]++;
            }
            if (tid == 0) { s_cut = ~0ull; s_cut_c = 0; }
            __syncthreads();
            for (uint32_t c = 0; c < k; c++) {
                uint32_t mine = cnts[c * K2_THREADS + tid];
                uint32_t pre = block_excl_scan(mine, scan_tmp, nullptr);
                const uint64_t room = a.cap - st.size[c];
                if ((uint64_t)pre <= room && (uint64_t)pre + mine > room) {
                    // the (room - pre + 1)-th choice of c in my segment overflows
                    uint64_t need = room - pre + 1, seen = 0;
                    for (uint64_t v = lo; v < s1; v++) {
                        const uint8_t* ov = a.order + v * k;
                        uint32_t cc = 0;
                        for (uint32_t i = 0; i < k; i++) if ((open >> ov[i]) & 1ull) { cc = ov[i]; break; }
                        if (cc == c && ++seen == need) { atomicMin((unsigned long long*)&s_cut, v); break; }
                    }
                }
            }
            __syncthreads();
            const uint64_t cut = s_cut;
            // commit [start, cut): these placements are exactly the sequential ones
            for (uint64_t v = lo; v < min(s1, cut); v++) {
                const uint8_t* ov = a.order + v * k;
                uint32_t c = 0;
                for (uint32_t i = 0; i < k; i++) if ((open >> ov[i]) & 1ull) { c = ov[i]; break; }
                const float dv = a.dist[v * k + c];
                a.home[v * a.omega] = c;
                for (uint32_t h = 1; h < a.omega; h++) a.home[v * a.omega + h] = SG_SENT;
                a.primary_d[v] = dv;
                atomicAdd((unsigned long long*)&st.size[c], 1ull);
                atomicAdd((unsigned long long*)&st.prim[c], 1ull);
                atomicMax((unsigned int*)&st.radius[c], __float_as_uint(dv));   // d >= 0: int order == float order
            }
            __syncthreads();
            if (cut == ~0ull) break;
            start = cut;
        }
        if (st.status) break;
        // ---------------- (2) statistics and thresholds (R4, R5)
        const float tau = __fadd_rn(1.0f, __fdiv_rn(a.alpha, (float)(1 + b)));
        if (tid == 0) {
            uint64_t P = 0;
            for (uint32_t c = 0; c < k; c++) P += st.prim[c];
            for (uint32_t c = 0; c < k; c++) st.budget[c] = budget_of(st.prim[c], P, k, a.theta0, a.cap);
        }
        __syncthreads();
        // ---------------- (3) Algorithm 1 replicas, speculate-and-verify
        if (a.omega > 1) {
            start = v0;
            while (true) {
                uint64_t open = 0;
                for (uint32_t c = 0; c < k; c++)
                    if (st.size[c] < a.cap && st.repl[c] < st.budget[c]) open |= 1ull << c;
                __syncthreads();
                if (open == 0) break;
                for (uint32_t c = 0; c < k; c++) cnts[c * K2_THREADS + tid] = 0;
                const uint64_t lo = max(start, s0);
                uint32_t picks[KMAX];
                for (uint64_t v = lo; v < s1; v++) {
                    uint32_t np = replica_picks(a, v, open, tau, st.radius, picks);
                    for (uint32_t i = 0; i < np; i++) cnts[picks[i] * K2_THREADS + tid]++;
                }
                if (tid == 0) s_cut = ~0ull;
                __syncthreads();
                for (uint32_t c = 0; c < k; c++) {
                    uint32_t mine = cnts[c * K2_THREADS + tid];
                    uint32_t pre = block_excl_scan(mine, scan_tmp, nullptr);
                    const uint64_t room = min(a.cap - st.size[c], st.budget[c] - st.repl[c]);
                    if ((uint64_t)pre <= room && (uint64_t)pre + mine > room) {
                        uint64_t need = room - pre + 1, seen = 0;
                        for (uint64_t v = lo; v < s1; v++) {
                            uint32_t np = replica_picks(a, v, open, tau, st.radius, picks);
                            bool hit = false;
                            for (uint32_t i = 0; i < np; i++) if (picks[i] == c) hit = true;
                            if (hit && ++seen == need) { atomicMin((unsigned long long*)&s_cut, v); break; }
                        }
                    }
                }
                __syncthreads();
                const uint64_t cut = s_cut;
                for (uint64_t v = lo; v < min(s1, cut); v++) {
                    uint32_t np = replica_picks(a, v, open, tau, st.radius, picks);
                    for (uint32_t i = 0; i < np; i++) {
                        a.home[v * a.omega + 1 + i] = picks[i];
                        atomicAdd((unsigned long long*)&st.size[picks[i]], 1ull);
                        atomicAdd((unsigned long long*)&st.repl[picks[i]], 1ull);
                    }
                }
                __syncthreads();
                if (cut == ~0ull) break;
                start = cut;
            }
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid < k) {
        a.state->size[tid] = st.size[tid];
        a.state->prim[tid] = st.prim[tid];
        a.state->repl[tid] = st.repl[tid];
        a.state->budget[tid] = st.budget[tid];
        a.state->radius[tid] = st.radius[tid];
    }
    if (tid == 0) a.state->status = st.status;
}

// ---------------------------------------------------------------------------------------------
// K2 on the whole GPU: the same speculate-and-verify rounds, one round spread over G CTAs x GT
// threads (a thread owns a contiguous segment of the block's vectors, CTAs in id order), with
// grid-wide barriers between the steps of a round (count -> find the first overflow -> commit).
// Cooperative launch guarantees the CTAs are co-resident.  Bit-identical to assign_kernel.
constexpr int GT = 512;
constexpr int MAXG = 1024;

struct GridScratch {
    unsigned bar_count, bar_gen;
    unsigned long long cut;
    unsigned cta_cnt[KMAX * MAXG];
};

__device__ __forceinline__ void grid_sync(GridScratch* g) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = &g->bar_gen;
        const unsigned my = *gen;
        __threadfence();
        if (atomicAdd(&g->bar_count, 1u) == gridDim.x - 1) {
            g->bar_count = 0;
            __threadfence();
            atomicAdd(&g->bar_gen, 1u);
        } else {
            while (*gen == my) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t primary_choice(const PartArgs& a, uint64_t v, uint64_t open) {
    const uint8_t* ov = a.order + v * a.k;
    for (uint32_t i = 0; i < a.k; i++) if ((open >> ov[i]) & 1ull) return ov[i];
    return 0;
}

// One speculate-and-verify round over [start, v1) of the current block.  PRIM: primaries, else
// replicas.  Returns the cut (first vector not committed; ~0 when the whole range is done).
template <bool PRIM>
__device__ uint64_t grid_round(const PartArgs& a, PartState* gs, GridScratch* g, uint64_t start, uint64_t s0, uint64_t s1,
                               uint64_t open, float tau, const float* radius, uint64_t* s_room,
                               uint32_t (*s_wtot)[GT / 32], uint32_t* s_pre, unsigned long long* s_inc,
                               unsigned long long* s_inc2, unsigned* s_rmax) {
    const uint32_t k = a.k, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = GT / 32;
    const uint64_t lo = max(start, s0);
    uint32_t picks[KMAX];
    // the choices of this thread's vectors are computed once per round (a segment is usually one
    // vector) instead of once per cluster; longer segments / wide omega recompute them
    constexpr uint32_t SEGC = 2, PMAX = 3;
    const uint32_t nv = s1 > lo ? (uint32_t)(s1 - lo) : 0;
    const bool cached = nv <= SEGC && (PRIM || a.omega - 1 <= PMAX);
    uint32_t cch[SEGC][PMAX], cnp[SEGC] = {0, 0};
    if (cached) {
#pragma unroll
        for (uint32_t t = 0; t < SEGC; t++) {
            if (t >= nv) break;
            if (PRIM) {
                cch[t][0] = primary_choice(a, lo + t, open);
                cnp[t] = 1;
            } else {
                cnp[t] = replica_picks(a, lo + t, open, tau, radius, picks);
                for (uint32_t i = 0; i < PMAX; i++) cch[t][i] = i < cnp[t] ? picks[i] : 0xFFFFFFFFu;
            }
        }
    }
    auto count_mine = [&](uint32_t c) -> uint32_t {
        uint32_t m = 0;
        if (cached) {
#pragma unroll
            for (uint32_t t = 0; t < SEGC; t++)
#pragma unroll
                for (uint32_t i = 0; i < PMAX; i++) m += (i < cnp[t] && cch[t][i] == c) ? 1u : 0u;
            return m;
        }
        for (uint64_t v = lo; v < s1; v++) {
            if (PRIM) {
                m += primary_choice(a, v, open) == c;
            } else {
                const uint32_t np = replica_picks(a, v, open, tau, radius, picks);
                for (uint32_t i = 0; i < np; i++) m += picks[i] == c;
            }
        }
        return m;
    };
    // (a) per-cluster counts: warp-exclusive prefixes and per-warp totals, CTA totals to global
    for (uint32_t c = 0; c < k; c++) {
        const uint32_t mine = count_mine(c);
        uint32_t inc = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += t;
        }
        if (lane == 31) s_wtot[c][warp] = inc;
    }
    __syncthreads();
    if (tid < k) {
        uint32_t run = 0;
        for (uint32_t w = 0; w < nw; w++) { const uint32_t t = s_wtot[tid][w]; s_wtot[tid][w] = run; run += t; }
        g->cta_cnt[tid * gridDim.x + blockIdx.x] = run;
    }
    grid_sync(g);
    // (b) global prefix of this CTA; the thread whose segment holds the first overflow of c
    //     proposes it as the cut
    if (tid < k) {
        uint32_t pre = 0;
        for (uint32_t j = 0; j < blockIdx.x; j++) pre += ((volatile unsigned*)g->cta_cnt)[tid * gridDim.x + j];
        s_pre[tid] = pre;
    }
    __syncthreads();
    for (uint32_t c = 0; c < k; c++) {
        const uint32_t mine = count_mine(c);
        uint32_t inc = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += t;
        }
        const uint64_t pre = (uint64_t)s_pre[c] + s_wtot[c][warp] + inc - mine;
        const uint64_t room = s_room[c];
        if (pre <= room && pre + mine > room) {
            const uint64_t need = room - pre + 1;
            uint64_t seen = 0;
            for (uint64_t v = lo; v < s1; v++) {
                bool hit;
                if (PRIM) {
                    hit = primary_choice(a, v, open) == c;
                } else {
                    const uint32_t np = replica_picks(a, v, open, tau, radius, picks);
                    hit = false;
                    for (uint32_t i = 0; i < np; i++) hit |= picks[i] == c;
                }
                if (hit && ++seen == need) { atomicMin(&g->cut, (unsigned long long)v); break; }
            }
        }
    }
    grid_sync(g);
    const uint64_t cut = *(volatile unsigned long long*)&g->cut;
    // (c) commit [lo, cut) of my segment; state increments aggregated per CTA
    if (tid < k) { s_inc[tid] = 0; s_inc2[tid] = 0; s_rmax[tid] = 0; }
    __syncthreads();
    for (uint64_t v = lo; v < min(s1, cut); v++) {
        if (PRIM) {
            const uint32_t c = primary_choice(a, v, open);
            const float dv = a.dist[v * k + c];
            a.home[v * a.omega] = c;
            for (uint32_t h = 1; h < a.omega; h++) a.home[v * a.omega + h] = SG_SENT;
            a.primary_d[v] = dv;
            atomicAdd(&s_inc[c], 1ull);
            atomicMax(&s_rmax[c], __float_as_uint(dv));   // d >= 0: int order == float order
        } else {
            const uint32_t np = replica_picks(a, v, open, tau, radius, picks);
            for (uint32_t i = 0; i < np; i++) {
                a.home[v * a.omega + 1 + i] = picks[i];
                atomicAdd(&s_inc[picks[i]], 1ull);
            }
        }
    }
    __syncthreads();
    if (tid < k && s_inc[tid]) {
        atomicAdd((unsigned long long*)&gs->size[tid], s_inc[tid]);
        if (PRIM) {
            atomicAdd((unsigned long long*)&gs->prim[tid], s_inc[tid]);
            atomicMax((unsigned*)&gs->radius[tid], s_rmax[tid]);
        } else {
            atomicAdd((unsigned long long*)&gs->repl[tid], s_inc[tid]);
        }
    }
    (void)s_inc2;
    grid_sync(g);
    if (blockIdx.x == 0 && tid == 0) g->cut = ~0ull;   // read by everyone before the barrier above
    return cut;
}

__global__ void __launch_bounds__(GT, 1) assign_grid_kernel(PartArgs a, PartState* gs, GridScratch* g) {
    __shared__ uint64_t s_room[KMAX];
    __shared__ uint32_t s_wtot[KMAX][GT / 32];
    __shared__ uint32_t s_pre[KMAX];
    __shared__ unsigned long long s_inc[KMAX], s_inc2[KMAX];
    __shared__ unsigned s_rmax[KMAX];
    __shared__ uint64_t s_open;
    __shared__ float s_radius[KMAX];
    const uint32_t k = a.k, tid = threadIdx.x;
    const uint64_t T = (uint64_t)gridDim.x * GT, gtid = (uint64_t)blockIdx.x * GT + tid;
    volatile PartState* vs = gs;
    const uint64_t nblocks = (a.n + a.block - 1) / a.block;
    for (uint64_t b = 0; b < nblocks; b++) {
        const uint64_t v0 = b * a.block, v1 = min(a.n, v0 + a.block);
        const uint64_t seg = (v1 - v0 + T - 1) / T;
        const uint64_t s0 = min(v1, v0 + gtid * seg), s1 = min(v1, s0 + seg);
        // ---------------- (1) primaries: nearest cluster with size < capacity
        uint64_t start = v0;
        while (true) {
            if (tid == 0) {
                uint64_t open = 0;
                for (uint32_t c = 0; c < k; c++) if (vs->size[c] < a.cap) open |= 1ull << c;
                s_open = open;
            }
            if (tid < k) s_room[tid] = a.cap - vs->size[tid];
            __syncthreads();
            const uint64_t open = s_open;
            if (open == 0) { if (blockIdx.x == 0 && tid == 0) gs->status = SG_ERR_CAPACITY; break; }
            const uint64_t cut = grid_round<true>(a, gs, g, start, s0, s1, open, 0.f, s_radius, s_room, s_wtot, s_pre,
                                                  s_inc, s_inc2, s_rmax);
            if (cut == ~0ull) break;
            start = cut;
        }
        if (s_open == 0) break;
        // ---------------- (2) statistics and thresholds (R4, R5)
        const float tau = __fadd_rn(1.0f, __fdiv_rn(a.alpha, (float)(1 + b)));
        if (blockIdx.x == 0 && tid == 0) {
            uint64_t P = 0;
            for (uint32_t c = 0; c < k; c++) P += vs->prim[c];
            for (uint32_t c = 0; c < k; c++) gs->budget[c] = budget_of(vs->prim[c], P, k, a.theta0, a.cap);
        }
        grid_sync(g);
        // ---------------- (3) Algorithm 1 replicas, speculate-and-verify
        if (a.omega > 1) {
            start = v0;
            while (true) {
                if (tid == 0) {
                    uint64_t open = 0;
                    for (uint32_t c = 0; c < k; c++)
                        if (vs->size[c] < a.cap && vs->repl[c] < vs->budget[c]) open |= 1ull << c;
                    s_open = open;
                }
                if (tid < k) {
                    const uint64_t r1 = a.cap - vs->size[tid], r2 = vs->budget[tid] - vs->repl[tid];
                    s_room[tid] = r1 < r2 ? r1 : r2;
                    s_radius[tid] = vs->radius[tid];   // updated by other CTAs' atomics: no L1 copy
                }
                __syncthreads();
                const uint64_t open = s_open;
                if (open == 0) break;
                const uint64_t cut = grid_round<false>(a, gs, g, start, s0, s1, open, tau, s_radius, s_room, s_wtot,
                                                       s_pre, s_inc, s_inc2, s_rmax);
                if (cut == ~0ull) break;
                start = cut;
            }
        }
        __syncthreads();
    }
}

}  // namespace

uint64_t derive_capacity(uint64_t n, uint32_t k, uint32_t t) {
    unsigned __int128 num = (unsigned __int128)1000000u * n;
    unsigned __int128 den = (unsigned __int128)(1000000u - t) * k;
    unsigned __int128 base = (num + den - 1) / den;
    return (uint64_t)((base * 115 + 99) / 100);
}

size_t partition_ws(uint64_t n, uint32_t k) {
    Carver cv(nullptr, 0);
    cv.take<float>(n * k);
    cv.take<uint8_t>(n * k);
    cv.take<PartState>(1);
    cv.take<GridScratch>(1);
    return cv.off + 1024;
}

sg_status partition_run(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const float* C,
                        const sg_partition_params* p, uint32_t* home, float* primary_d, uint64_t* counts_host,
                        void* ws, size_t ws_bytes, cudaStream_t st) {
    Carver cv(ws, ws_bytes);
    float* dist = cv.take<float>(n * p->k);
    uint8_t* order = cv.take<uint8_t>(n * p->k);
    PartState* state = cv.take<PartState>(1);
    GridScratch* gscr = cv.take<GridScratch>(1);
    if (!cv.ok()) { set_error("partition: workspace too small"); return SG_ERR_WORKSPACE; }
    const uint64_t cap = p->capacity ? p->capacity : derive_capacity(n, p->k, p->theta0_ppm);
    SG_CHECK_ARG(cap * p->k >= n, "partition: capacity * k < n");
    const uint64_t nwarps = (n + 31) / 32;
    {
        const unsigned g = (unsigned)((nwarps + 7) / 8);
        const size_t cb = (size_t)p->k * d * sizeof(float);
        const bool sm = cb <= 160 * 1024;   // + the 34 KB transpose tile, within the 227 KB budget
        cudaError_t ae = cudaSuccess;
        auto launch = [&](auto kern) {
            if (sm) ae = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cb);
            kern<<<g, 256, sm ? cb : 0, st>>>(x, dtype, n, d, C, p->k, dist, order);
        };
        const uint32_t k = p->k;
        if (sm) {
            if (k <= 4) launch(centroid_dist_order<4, true>);
            else if (k <= 8) launch(centroid_dist_order<8, true>);
            else if (k <= 16) launch(centroid_dist_order<16, true>);
            else if (k <= 32) launch(centroid_dist_order<32, true>);
            else launch(centroid_dist_order<64, true>);
        } else {
            if (k <= 4) launch(centroid_dist_order<4, false>);
            else if (k <= 8) launch(centroid_dist_order<8, false>);
            else if (k <= 16) launch(centroid_dist_order<16, false>);
            else if (k <= 32) launch(centroid_dist_order<32, false>);
            else launch(centroid_dist_order<64, false>);
        }
        SG_CUDA(ae);
        SG_LAUNCHED("centroid_dist_order");
    }
    PartArgs a{};
    a.dist = dist; a.order = order; a.home = home; a.primary_d = primary_d; a.state = state;
    a.n = n; a.cap = cap; a.k = p->k; a.omega = p->omega; a.block = p->block_size; a.theta0 = p->theta0_ppm;
    a.eps = p->epsilon; a.alpha = p->alpha;
    static int single = -1;
    if (single < 0) { const char* e = getenv("SG_PART_SINGLE_CTA"); single = e ? atoi(e) : 0; }
    if (single) {   // one-CTA reference variant of K2 (kept for comparison)
        const size_t smem = (size_t)p->k * K2_THREADS * sizeof(uint16_t);
        SG_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        assign_kernel<<<1, K2_THREADS, smem, st>>>(a);
        SG_LAUNCHED("assign_kernel");
    } else {
        SG_CUDA(cudaMemsetAsync(state, 0, sizeof(PartState), st));
        SG_CUDA(cudaMemsetAsync(gscr, 0, sizeof(GridScratch), st));
        SG_CUDA(cudaMemsetAsync(&gscr->cut, 0xFF, sizeof(unsigned long long), st));
        int per_sm = 0;
        SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, assign_grid_kernel, GT, 0));
        const uint64_t need = (p->block_size + GT - 1) / GT;   // at most one vector per thread per block
        uint64_t g = (uint64_t)num_sms() * (per_sm > 0 ? 1 : 0);
        if (g > need) g = need;
        if (g > MAXG) g = MAXG;
        if (g < 1) g = 1;
        PartState* gs = state;
        void* args[] = {(void*)&a, (void*)&gs, (void*)&gscr};
        SG_CUDA(cudaLaunchCooperativeKernel((const void*)assign_grid_kernel, dim3((unsigned)g), dim3(GT), args, 0, st));
        SG_LAUNCHED("assign_grid_kernel");
    }
    PartState hs;
    SG_CUDA(cudaMemcpyAsync(&hs, state, sizeof(PartState), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    if (hs.status) { set_error("partition: every cluster full for a primary (capacity)"); return SG_ERR_CAPACITY; }
    if (counts_host)
        for (uint32_t c = 0; c < p->k; c++) {
            counts_host[c] = hs.size[c];
            counts_host[p->k + c] = hs.prim[c];
            counts_host[2 * p->k + c] = hs.repl[c];
        }
    return SG_OK;
}

// ------------------------------------------------------------------ a4: shard membership
namespace {
__global__ void member_flags(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, uint32_t s,
                             uint32_t* __restrict__ flags) {
    uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uint32_t f = 0;
    for (uint32_t h = 0; h < omega; h++) f |= home[v * omega + h] == s;
    flags[v] = f;
}
__global__ void member_scatter(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, uint32_t s,
                               const uint32_t* __restrict__ flags, const uint64_t* __restrict__ pos,
                               uint32_t* __restrict__ idmap, uint32_t* __restrict__ inv) {
    uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || !flags[v]) return;
    const uint64_t l = pos[v];
    idmap[l] = (uint32_t)v;
    if (inv)
        for (uint32_t h = 0; h < omega; h++)
            if (home[v * omega + h] == s) inv[v * omega + h] = (uint32_t)l;
}
__global__ void entry_kernel(const uint32_t* __restrict__ home, const float* __restrict__ pd, uint64_t n,
                             uint32_t omega, unsigned long long* best) {
    uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const uint32_t s = home[g * omega];
    atomicMin(&best[s], ((unsigned long long)f2ord(pd[g]) << 32) | (uint32_t)g);
}
}  // namespace

size_t idmap_ws(uint64_t n) {
    Carver cv(nullptr, 0);
    cv.take<uint32_t>(n);
    cv.take<uint64_t>(n + 1);
    return cv.off + scan_workspace(n) + 1024;
}

sg_status idmap_run(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t s, uint32_t* idmap, uint32_t* inv,
                    uint64_t* m_host, void* ws, size_t ws_bytes, cudaStream_t st) {
    Carver cv(ws, ws_bytes);
    uint32_t* flags = cv.take<uint32_t>(n);
    uint64_t* pos = cv.take<uint64_t>(n + 1);
    if (!cv.ok()) { set_error("idmap: workspace too small"); return SG_ERR_WORKSPACE; }
    const unsigned nb = (unsigned)((n + 255) / 256);
    member_flags<<<nb, 256, 0, st>>>(home, n, omega, s, flags);
    SG_LAUNCHED("member_flags");
    SG_TRY(excl_scan_u32_to_u64(flags, pos, n, cv, st));
    if (idmap) {
        member_scatter<<<nb, 256, 0, st>>>(home, n, omega, s, flags, pos, idmap, inv);
        SG_LAUNCHED("member_scatter");
    }
    if (m_host) {
        SG_CUDA(cudaMemcpyAsync(m_host, pos + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        SG_CUDA(cudaStreamSynchronize(st));
    }
    return SG_OK;
}

sg_status entry_run(const uint32_t* home, const float* pd, uint64_t n, uint32_t omega, uint32_t k,
                    const uint64_t* sizes_host, uint32_t* entry_host, uint32_t* global_host, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
    Carver cv(ws, ws_bytes);
    unsigned long long* best = cv.take<unsigned long long>(k);
    if (!cv.ok()) { set_error("entry_points: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(best, 0xFF, k * sizeof(unsigned long long), st));
    entry_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(home, pd, n, omega, best);
    SG_LAUNCHED("entry_kernel");
    unsigned long long hb[KMAX];
    SG_CUDA(cudaMemcpyAsync(hb, best, k * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    uint32_t big = 0;
    for (uint32_t s = 0; s < k; s++) {
        entry_host[s] = hb[s] == ~0ull ? SG_SENT : (uint32_t)(hb[s] & 0xFFFFFFFFu);
        if (sizes_host[s] > sizes_host[big]) big = s;
    }
    if (global_host) *global_host = entry_host[big];
    return SG_OK;
}

}  // namespace sg
