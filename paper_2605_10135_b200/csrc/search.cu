// a9 — recall evaluation: greedy best-first beam search over the merged graph (PAPER P:507
// "following DiskANN's search strategy"; reading R14) + recall@k against an exact
// ground truth computed by the tensor-core kNN (a5 with A = queries, B = dataset).
//
// One warp per query.  The pool (<= beam entries, keys (ord(dist) << 32 | id)) stays sorted in
// shared memory; each expansion takes the lowest unexpanded entry, marks its unvisited
// neighbours in the query's visited set, computes their distances (lane per neighbour), sorts
// the new keys and merges them into the pool by rank (binary search in both lists), truncating
// to beam — the same semantics as sorting the union by (dist, id) and truncating.
// Distances follow P4/P8 exactly: u8 rows in integer arithmetic, f32 rows as the sequential fp64
// sum of the squared differences (products), rounded once to f32 — the oracle's definition.
// The visited set is a bitmap over the n vectors (small n) or an open-addressing hash set of
// ids (large n; 8 x beam x R slots per query, overflow reported), whichever is smaller.
#include "common.cuh"

namespace sg {
namespace {

constexpr int SW = 4;   // queries (warps) per CTA

struct SearchArgs {
    const void* x;
    const void* q;
    const uint32_t* graph;
    uint32_t* visited;     // batch x words: bitmap (hash == 0) or hash slots (hash == 1)
    uint32_t* out_ids;     // may be NULL when out_keys is set
    uint64_t* out_keys;    // optional: the first topk pool keys (ord(dist) << 32 | id), ~0 past np
    uint64_t n, words;
    uint32_t d, R, entry, nq, q0, topk, beam, poolcap, newcap;
    int dtype, metric;
    int hash;              // visited set: 0 bitmap of n bits, 1 hash set of `words` slots
    unsigned long long* ndist;
    int* overflow;         // set when a hash set fills up
};

// P4 / P8 exact distance of query qv (kept as loaded: u8 codes or f32) to row v
__device__ __forceinline__ float qdist(const SearchArgs& a, const float* qv, uint32_t v) {
    if (a.dtype == SG_U8) {
        // integer arithmetic (exact: d * 255^2 < 2^31), rounded once to f32 like the oracle's int64
        int s = 0;
        if ((a.d & 15) == 0 && ((uintptr_t)a.x & 15) == 0) {
            const uint4* row = (const uint4*)((const uint8_t*)a.x + (uint64_t)v * a.d);
            for (uint32_t j16 = 0; j16 < (a.d >> 4); j16++) {
                const uint4 w = __ldg(row + j16);
                const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
                const float* qq = qv + 16 * j16;
#pragma unroll
                for (int b = 0; b < 16; b++) {
                    const int t = (int)((wd[b >> 2] >> (8 * (b & 3))) & 0xffu), u = (int)qq[b];
                    s += a.metric == SG_IP ? -t * u : (t - u) * (t - u);
                }
            }
        } else {
            const uint8_t* row = (const uint8_t*)a.x + (uint64_t)v * a.d;
            for (uint32_t j = 0; j < a.d; j++) {
                const int t = row[j], u = (int)qv[j];
                s += a.metric == SG_IP ? -t * u : (t - u) * (t - u);
            }
        }
        return (float)s;
    }
    // f32: fp64 products summed in index order, one rounding to f32 (no FMA contraction)
    double s = 0.0;
    if ((a.d & 3) == 0 && ((uintptr_t)a.x & 15) == 0) {
        const float4* row = (const float4*)((const float*)a.x + (uint64_t)v * a.d);
        for (uint32_t j4 = 0; j4 < (a.d >> 2); j4++) {
            const float4 t = __ldg(row + j4);
            const float tt[4] = {t.x, t.y, t.z, t.w};
            const float* qq = qv + 4 * j4;
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const double x = (double)tt[b], y = (double)qq[b];
                s = a.metric == SG_IP ? __dsub_rn(s, __dmul_rn(x, y)) : __dadd_rn(s, __dmul_rn(x - y, x - y));
            }
        }
    } else {
        const float* row = (const float*)a.x + (uint64_t)v * a.d;
        for (uint32_t j = 0; j < a.d; j++) {
            const double x = (double)__ldg(row + j), y = (double)qv[j];
            s = a.metric == SG_IP ? __dsub_rn(s, __dmul_rn(x, y)) : __dadd_rn(s, __dmul_rn(x - y, x - y));
        }
    }
    return (float)s;
}

// first visit of v? (marks it visited)
__device__ __forceinline__ bool visit(const SearchArgs& a, uint32_t* vis, uint32_t v) {
    if (!a.hash) {
        const uint32_t bit = 1u << (v & 31);
        return !(atomicOr(&vis[v >> 5], bit) & bit);
    }
    const uint32_t mask = (uint32_t)a.words - 1u;
    uint32_t h = (v * 0x9E3779B1u) & mask;
    for (uint32_t probe = 0; probe <= mask; probe++) {
        const uint32_t old = atomicCAS(&vis[h], SG_SENT, v);
        if (old == SG_SENT) return true;
        if (old == v) return false;
        h = (h + 1) & mask;
    }
    atomicExch(a.overflow, 1);
    return false;
}

__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* arr, uint32_t n, uint64_t key) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (arr[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(SW * 32) beam_kernel(SearchArgs a) {
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t per = ((2 * a.poolcap + a.newcap) * 8 + 2 * a.poolcap * 4 + a.d * 4 + 15) & ~15u;   // 16-byte aligned
    uint8_t* base = sm + w * per;
    uint64_t* pool = (uint64_t*)base;
    uint64_t* pool2 = pool + a.poolcap;
    uint64_t* nb = pool2 + a.poolcap;
    uint32_t* ex = (uint32_t*)(nb + a.newcap);
    uint32_t* ex2 = ex + a.poolcap;
    float* qv = (float*)(ex2 + a.poolcap);
    const uint32_t qi = a.q0 + blockIdx.x * SW + w;
    if (qi >= a.nq) return;
    uint32_t* vis = a.visited + (uint64_t)(blockIdx.x * SW + w) * a.words;
    for (uint32_t j = lane; j < a.d; j += 32)
        qv[j] = a.dtype == SG_U8 ? (float)((const uint8_t*)a.q)[(uint64_t)qi * a.d + j]
                                 : ((const float*)a.q)[(uint64_t)qi * a.d + j];
    const uint32_t clear = a.hash ? SG_SENT : 0u;
    for (uint64_t i = lane; i < a.words; i += 32) vis[i] = clear;
    __syncwarp();
    __threadfence_block();
    unsigned long long nd = 1;
    if (lane == 0) {
        pool[0] = ((uint64_t)f2ord(qdist(a, qv, a.entry)) << 32) | a.entry;
        ex[0] = 0;
        visit(a, vis, a.entry);
    }
    uint32_t np = 1;
    __syncwarp();
    while (true) {
        // lowest unexpanded entry
        uint32_t u = SG_SENT;
        for (uint32_t i0 = 0; i0 < np && u == SG_SENT; i0 += 32) {
            const uint32_t i = i0 + lane;
            const uint32_t bal = __ballot_sync(0xffffffffu, i < np && ex[i] == 0);
            if (bal) u = i0 + __ffs(bal) - 1;
        }
        if (u == SG_SENT) break;
        const uint32_t node = (uint32_t)pool[u];
        __syncwarp();
        if (lane == 0) ex[u] = 1;
        // new neighbours
        uint32_t nn = 0;
        for (uint32_t j0 = 0; j0 < a.R; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint64_t key = 0;
            bool fresh = false;
            if (j < a.R) {
                const uint32_t v = a.graph[(uint64_t)node * a.R + j];
                if (v != SG_SENT) {
                    fresh = visit(a, vis, v);
                    if (fresh) key = ((uint64_t)f2ord(qdist(a, qv, v)) << 32) | v;
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, fresh);
            if (fresh) nb[nn + __popc(bal & ((1u << lane) - 1u))] = key;
            nn += __popc(bal);
        }
        SG_DCHECK(nn <= a.newcap && np <= a.beam);
        nd += nn;
        if (nn == 0) { __syncwarp(); continue; }
        uint32_t p2 = 32;
        while (p2 < nn) p2 <<= 1;
        for (uint32_t i = nn + lane; i < p2; i += 32) nb[i] = ~0ull;
        __syncwarp();
        warp_sort_u64(nb, p2, lane);
        // merge pool[0..np) and nb[0..nn) by rank, keep the first `beam`
        for (uint32_t i = lane; i < np; i += 32) {
            const uint32_t pos = i + lower_bound_u64(nb, nn, pool[i]);
            if (pos < a.beam) { pool2[pos] = pool[i]; ex2[pos] = ex[i]; }
        }
        for (uint32_t j = lane; j < nn; j += 32) {
            const uint32_t pos = j + lower_bound_u64(pool, np, nb[j]);
            if (pos < a.beam) { pool2[pos] = nb[j]; ex2[pos] = 0; }
        }
        np = min(a.beam, np + nn);
        __syncwarp();
        for (uint32_t i = lane; i < np; i += 32) { pool[i] = pool2[i]; ex[i] = ex2[i]; }
        __syncwarp();
    }
    for (uint32_t i = lane; i < a.topk; i += 32) {
        if (a.out_ids) a.out_ids[(uint64_t)qi * a.topk + i] = i < np ? (uint32_t)pool[i] : SG_SENT;
        if (a.out_keys) a.out_keys[(uint64_t)qi * a.topk + i] = i < np ? pool[i] : ~0ull;
    }
    if (lane == 0 && a.ndist) atomicAdd(a.ndist, nd);
}

__global__ void recall_kernel(const uint32_t* __restrict__ ret, const uint32_t* __restrict__ gt, uint32_t nq,
                              uint32_t topk, unsigned long long* hits) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long h = 0;
    for (uint32_t i = 0; i < topk; i++) {
        const uint32_t r = ret[(uint64_t)q * topk + i];
        if (r == SG_SENT) continue;
        for (uint32_t j = 0; j < topk; j++) if (gt[(uint64_t)q * topk + j] == r) { h++; break; }
    }
    atomicAdd(hits, h);
}

// Per-shard search + result merge (split-only mode; reading R15): keys[s][q][0..topk)
// are the per-entry results; the merged list is the topk smallest distinct keys, i.e. the union
// ordered by (dist, id) with duplicate ids (the same vector reached from two entries) kept once.
__global__ void shard_merge_kernel(const uint64_t* __restrict__ keys, uint32_t ns, uint32_t nq, uint32_t topk,
                                   uint32_t* __restrict__ out) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    uint64_t last = 0;
    bool first = true;
    for (uint32_t i = 0; i < topk; i++) {
        uint64_t best = ~0ull;
        for (uint32_t s = 0; s < ns; s++) {
            const uint64_t* row = keys + ((uint64_t)s * nq + q) * topk;
            for (uint32_t j = 0; j < topk; j++) {
                const uint64_t k = row[j];
                if ((first || k > last) && k < best) best = k;
            }
        }
        out[(uint64_t)q * topk + i] = best == ~0ull ? SG_SENT : (uint32_t)best;
        last = best;
        first = false;
    }
}

}  // namespace

static uint32_t pow2_at_least(uint32_t v) { uint32_t p = 32; while (p < v) p <<= 1; return p; }

// visited-set words per query: the n-bit bitmap, or a hash set of 8 x beam x R slots when that
// is smaller (large n); the second value says which
static uint64_t vis_words(uint64_t n, uint32_t beam, uint32_t R, int* hash) {
    const uint64_t bitmap = (n + 31) / 32;
    uint64_t slots = 1024;
    while (slots < 8ull * beam * R) slots <<= 1;
    *hash = slots < bitmap;
    return *hash ? slots : bitmap;
}

static uint64_t vis_batch(uint64_t words, uint32_t nq) {
    uint64_t batch = (1ull << 30) / (words * 4 + 1);
    if (batch < SW) batch = SW;
    if (batch > nq) batch = (nq + SW - 1) / SW * SW;
    return batch / SW * SW;
}

size_t beam_ws(uint64_t n, uint32_t nq, uint32_t beam, uint32_t R) {
    int hash;
    const uint64_t words = vis_words(n, beam, R, &hash);
    return vis_batch(words, nq) * words * 4 + 4096 + 512;
}

sg_status beam_run(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const uint32_t* graph, uint32_t R,
                   uint32_t entry, const void* q, uint32_t nq, uint32_t topk, uint32_t beam, int metric,
                   uint32_t* out_ids, unsigned long long* ndist, Carver& cv, cudaStream_t st,
                   uint64_t* out_keys) {
    int hash = 0;
    const uint64_t words = vis_words(n, beam, R, &hash);
    const uint64_t batch = vis_batch(words, nq);
    uint32_t* vis = cv.take<uint32_t>(batch * words);
    int* overflow = cv.take<int>(1);
    if (!cv.ok()) { set_error("search: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int), st));
    SearchArgs a{};
    a.x = x; a.q = q; a.graph = graph; a.visited = vis; a.out_ids = out_ids; a.out_keys = out_keys; a.n = n; a.words = words;
    a.d = d; a.R = R; a.entry = entry; a.nq = nq; a.topk = topk; a.beam = beam;
    a.poolcap = pow2_at_least(beam + R);
    a.newcap = pow2_at_least(R);
    a.dtype = dtype; a.metric = metric; a.ndist = ndist; a.hash = hash; a.overflow = overflow;
    const size_t per = ((2 * a.poolcap + a.newcap) * 8 + 2 * a.poolcap * 4 + d * 4 + 15) & ~(size_t)15;
    const size_t smem = per * SW;
    SG_CHECK_ARG(smem <= 200 * 1024, "search: beam/R/d too large for shared memory");
    SG_CUDA(cudaFuncSetAttribute(beam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (uint64_t q0 = 0; q0 < nq; q0 += batch) {
        a.q0 = (uint32_t)q0;
        const uint64_t cnt = batch < nq - q0 ? batch : nq - q0;
        beam_kernel<<<(unsigned)((cnt + SW - 1) / SW), SW * 32, smem, st>>>(a);
        SG_LAUNCHED("beam_kernel");
    }
    if (hash) {
        int h = 0;
        SG_CUDA(cudaMemcpyAsync(&h, overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
        SG_CUDA(cudaStreamSynchronize(st));
        if (h) { set_error("search: a visited hash set overflowed (8 x beam x R slots)"); return SG_ERR_WORKSPACE; }
    }
    return SG_OK;
}

sg_status shard_merge_run(const uint64_t* keys, uint32_t ns, uint32_t nq, uint32_t topk, uint32_t* out_ids,
                          cudaStream_t st) {
    shard_merge_kernel<<<(nq + 127) / 128, 128, 0, st>>>(keys, ns, nq, topk, out_ids);
    SG_LAUNCHED("shard_merge_kernel");
    return SG_OK;
}

sg_status recall_run(const uint32_t* ret, const uint32_t* gt, uint32_t nq, uint32_t topk, double* recall_host,
                     Carver& cv, cudaStream_t st) {
    unsigned long long* hits = cv.take<unsigned long long>(1);
    if (!cv.ok()) { set_error("search: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(hits, 0, sizeof(unsigned long long), st));
    recall_kernel<<<(nq + 255) / 256, 256, 0, st>>>(ret, gt, nq, topk, hits);
    SG_LAUNCHED("recall_kernel");
    unsigned long long h = 0;
    SG_CUDA(cudaMemcpyAsync(&h, hits, sizeof(h), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    *recall_host = nq ? (double)h / ((double)nq * topk) : 0.0;
    return SG_OK;
}

}  // namespace sg
