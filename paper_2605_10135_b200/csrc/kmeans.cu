// a1 — centroids ("partitions the large dataset ... using k-means clustering",
// P:298; reading R0).  Strided sample floor(i*n/S), S = min(n, spc*k); k-means++ seeding with
// draws from splitmix64(seed) (one CTA, a warp per sample); Lloyd iterations as launches: the
// assignment over the whole GPU (a warp per sample, fp64 distances), then one CTA for the
// distortion / stop test and the fp64 per-cluster sums in sample order (samples bucketed by
// centre with order kept, a thread per (centre, dimension): deterministic); empty clusters are
// re-seeded with the farthest point of the largest cluster; stop after max_iter or when the
// relative distortion improvement is <= 1e-4 (a device flag, so no host synchronisation).
// Not bit-exact with the oracle (reduction order of the seeding totals differs); accepted
// when its sample distortion is within 1% of the oracle's.
#include "common.cuh"

namespace sg {
namespace {

constexpr int KT = 1024;

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ double block_sum(double v, double* tmp) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) tmp[w] = v;
    __syncthreads();
    double t = 0;
    if (threadIdx.x == 0) { for (int i = 0; i < KT / 32; i++) t += tmp[i]; tmp[32] = t; }
    __syncthreads();
    t = tmp[32];
    __syncthreads();
    return t;
}

struct KmArgs {
    const void* x;
    int dtype;
    uint64_t n;
    uint32_t d, k, S, max_iter;
    uint64_t seed;
    float* smp;       // S x d
    double* D2;       // S
    uint32_t* asg;    // S
    double* sums;     // k x d
    float* C;         // k x d out
    double* distortion;
};

__device__ double d2(const float* p, const float* c, uint32_t d) {
    double s = 0;
    for (uint32_t j = 0; j < d; j++) { double t = (double)p[j] - (double)c[j]; s += t * t; }
    return s;
}

// warp-cooperative fp64 squared distance (lanes over dimensions, fixed reduction order)
__device__ __forceinline__ double d2_warp(const float* p, const float* c, uint32_t d, uint32_t lane) {
    double s = 0;
    for (uint32_t j = lane; j < d; j += 32) { const double t = (double)p[j] - (double)c[j]; s += t * t; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// sample + k-means++ seeding (one CTA; k steps over S samples, a warp per sample)
__global__ void __launch_bounds__(KT, 1) kmeans_seed_kernel(KmArgs a, uint64_t* rng, int* stop) {
    __shared__ double tmp[33];
    __shared__ double part[KT];
    __shared__ uint64_t s_pick;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = KT / 32;
    const uint32_t S = a.S, d = a.d, k = a.k;
    for (uint64_t e = tid; e < (uint64_t)S * d; e += KT) {
        const uint64_t i = e / d, j = e % d;
        const uint64_t row = (uint64_t)(((unsigned __int128)i * a.n) / S);
        a.smp[e] = a.dtype == SG_U8 ? (float)((const uint8_t*)a.x)[row * d + j] : ((const float*)a.x)[row * d + j];
    }
    __syncthreads();
    uint64_t rs = a.seed;   // every thread advances the same stream identically
    const uint64_t first = splitmix64(rs) % S;
    for (uint32_t j = tid; j < d; j += KT) a.C[j] = a.smp[first * d + j];
    __syncthreads();
    for (uint32_t i = warp; i < S; i += nw) {
        const double t = d2_warp(a.smp + (uint64_t)i * d, a.C, d, lane);
        if (lane == 0) a.D2[i] = t;
    }
    __syncthreads();
    for (uint32_t c = 1; c < k; c++) {
        // contiguous chunk per thread -> prefix sums in sample order
        const uint32_t per = (S + KT - 1) / KT, i0 = tid * per, i1 = min(S, i0 + per);
        double loc = 0;
        for (uint32_t i = i0; i < i1; i++) loc += a.D2[i];
        const double total = block_sum(loc, tmp);
        const double u = (double)(splitmix64(rs) >> 11) * (1.0 / 9007199254740992.0) * total;
        part[tid] = loc;
        if (tid == 0) s_pick = S - 1;
        __syncthreads();
        if (tid == 0) {
            double acc = 0;
            for (uint32_t t = 0; t < KT; t++) {
                if (acc + part[t] > u) {
                    const uint32_t b0 = t * per, b1 = min(S, b0 + per);
                    for (uint32_t i = b0; i < b1; i++) { acc += a.D2[i]; if (acc > u) { s_pick = i; break; } }
                    break;
                }
                acc += part[t];
            }
        }
        __syncthreads();
        const uint64_t pick = s_pick;
        for (uint32_t j = tid; j < d; j += KT) a.C[(uint64_t)c * d + j] = a.smp[pick * d + j];
        __syncthreads();
        for (uint32_t i = warp; i < S; i += nw) {
            const double t = d2_warp(a.smp + (uint64_t)i * d, a.C + (uint64_t)c * d, d, lane);
            if (lane == 0 && t < a.D2[i]) a.D2[i] = t;
        }
        __syncthreads();
    }
    if (tid == 0) { *rng = rs; *stop = 0; a.distortion[1] = __longlong_as_double(0x7ff0000000000000ll); }
}

// Lloyd step 1: nearest centre of every sample by (d^2, c) (grid, a warp per sample)
__global__ void __launch_bounds__(256) kmeans_assign_kernel(KmArgs a, const int* stop) {
    if (*(volatile const int*)stop) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= a.S) return;
    const float* p = a.smp + i * a.d;
    double best = __longlong_as_double(0x7ff0000000000000ll);
    uint32_t bc = 0;
    for (uint32_t c = 0; c < a.k; c++) {
        const double t = d2_warp(p, a.C + (uint64_t)c * a.d, a.d, lane);
        if (t < best) { best = t; bc = c; }
    }
    if (lane == 0) { a.asg[i] = bc; a.D2[i] = best; }
}

// Lloyd step 2 (one CTA): distortion + stop test (relative improvement <= 1e-4 or max_iter), then
// means as fp64 sums in sample order: samples bucketed by centre (order kept), one thread per
// (centre, dimension); an empty cluster is re-seeded with the farthest point of the largest one.
__global__ void __launch_bounds__(KT, 1) kmeans_update_kernel(KmArgs a, int* stop, uint32_t it, uint32_t* order) {
    __shared__ double tmp[33];
    __shared__ uint32_t s_cnt[64], s_off[65];
    __shared__ uint32_t scan_tmp[33];
    __shared__ int s_stop;
    __shared__ uint64_t s_pick;
    if (*(volatile int*)stop) return;
    const uint32_t tid = threadIdx.x;
    const uint32_t S = a.S, d = a.d, k = a.k;
    const uint32_t per = (S + KT - 1) / KT, i0 = min(S, tid * per), i1 = min(S, i0 + per);
    double loc = 0;
    for (uint32_t i = i0; i < i1; i++) loc += a.D2[i];
    const double dist = block_sum(loc, tmp);
    if (tid == 0) {
        const double prev = a.distortion[1];
        s_stop = (it == a.max_iter) || (isfinite(prev) && (prev - dist) <= 1e-4 * prev);
        a.distortion[0] = dist;
        a.distortion[1] = dist;
        if (s_stop) *stop = 1;
    }
    __syncthreads();
    if (s_stop) return;
    // stable bucketing of the samples by centre: per centre, a block scan of each thread's chunk
    if (tid <= k) s_off[tid] = 0;
    __syncthreads();
    uint32_t base = 0;
    for (uint32_t c = 0; c < k; c++) {
        uint32_t mine = 0;
        for (uint32_t i = i0; i < i1; i++) mine += a.asg[i] == c;
        uint32_t tot;
        const uint32_t pre = block_excl_scan(mine, scan_tmp, &tot);
        uint32_t w = base + pre;
        for (uint32_t i = i0; i < i1; i++) if (a.asg[i] == c) order[w++] = i;
        if (tid == 0) { s_cnt[c] = tot; s_off[c] = base; }
        base += tot;
    }
    __syncthreads();
    for (uint32_t cj = tid; cj < k * d; cj += KT) {
        const uint32_t c = cj / d, j = cj % d;
        double sum = 0;
        for (uint32_t q = s_off[c]; q < s_off[c] + s_cnt[c]; q++) sum += (double)a.smp[(uint64_t)order[q] * d + j];
        a.sums[cj] = sum;
    }
    __syncthreads();
    for (uint32_t c = 0; c < k; c++) {
        if (s_cnt[c] == 0) {
            if (tid == 0) {
                uint32_t big = 0;
                for (uint32_t c2 = 1; c2 < k; c2++) if (s_cnt[c2] > s_cnt[big]) big = c2;
                uint64_t far = 0;
                double fd = -1;
                for (uint32_t i = 0; i < S; i++) if (a.asg[i] == big && a.D2[i] > fd) { fd = a.D2[i]; far = i; }
                s_pick = far;
                a.D2[far] = 0;
            }
            __syncthreads();
            for (uint32_t j = tid; j < d; j += KT) a.C[(uint64_t)c * d + j] = a.smp[s_pick * d + j];
        } else {
            for (uint32_t j = tid; j < d; j += KT)
                a.C[(uint64_t)c * d + j] = (float)(a.sums[(uint64_t)c * d + j] / (double)s_cnt[c]);
        }
        __syncthreads();
    }
}

}  // namespace

size_t kmeans_ws(uint64_t n, uint32_t d, uint32_t k, uint32_t spc) {
    uint64_t S = (uint64_t)spc * k;
    if (S > n) S = n;
    Carver cv(nullptr, 0);
    cv.take<float>(S * d);
    cv.take<double>(S);
    cv.take<uint32_t>(S);
    cv.take<double>((uint64_t)k * d);
    cv.take<double>(2);
    cv.take<uint32_t>(S);        // bucketed sample order
    cv.take<uint64_t>(2);        // rng state, stop flag
    return cv.off + 1024;
}

sg_status kmeans_run(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, uint32_t k, uint64_t seed,
                     uint32_t max_iter, uint32_t spc, float* C, void* ws, size_t ws_bytes, cudaStream_t st) {
    uint64_t S = (uint64_t)spc * k;
    if (S > n) S = n;
    SG_CHECK_ARG(S >= k, "kmeans: sample smaller than k");
    Carver cv(ws, ws_bytes);
    KmArgs a{};
    a.x = x; a.dtype = dtype; a.n = n; a.d = d; a.k = k; a.S = (uint32_t)S; a.max_iter = max_iter; a.seed = seed;
    a.smp = cv.take<float>(S * d);
    a.D2 = cv.take<double>(S);
    a.asg = cv.take<uint32_t>(S);
    a.sums = cv.take<double>((uint64_t)k * d);
    a.distortion = cv.take<double>(2);
    uint32_t* order = cv.take<uint32_t>(S);
    uint64_t* misc = cv.take<uint64_t>(2);
    a.C = C;
    if (!cv.ok()) { set_error("kmeans: workspace too small"); return SG_ERR_WORKSPACE; }
    int* stop = (int*)(misc + 1);
    kmeans_seed_kernel<<<1, KT, 0, st>>>(a, misc, stop);
    SG_LAUNCHED("kmeans_seed_kernel");
    const unsigned ag = (unsigned)((S * 32 + 255) / 256);
    for (uint32_t it = 0; it <= max_iter; it++) {   // kernels exit at once after convergence (stop flag)
        kmeans_assign_kernel<<<ag, 256, 0, st>>>(a, stop);
        SG_LAUNCHED("kmeans_assign_kernel");
        kmeans_update_kernel<<<1, KT, 0, st>>>(a, stop, it, order);
        SG_LAUNCHED("kmeans_update_kernel");
    }
    return SG_OK;
}

}  // namespace sg
