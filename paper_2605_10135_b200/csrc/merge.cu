// a8 — cross-shard merge by edge union + re-prune ("edge union"; reading R12),
// streamed shard by shard and distributed by primary owner.
//
// The merged row of g lives on the rank that owns g's primary shard (owner rows only, ascending
// gid, `owned_index[g]` = its row).  A shard is merged right after it is built, so its graph can
// be freed before the next one:
//   * a row of a vector with ONE home is its shard row mapped to global ids, as is;
//   * a row of a vector with several homes is the top-R by (dist, gid) of the union of the
//     homes' rows, deduplicated by gid with the minimum carried distance.  The union is formed
//     incrementally in the merged row (each home's row is folded in as it arrives); because a
//     gid's minimum distance only decreases and the top-R of a superset keeps every element
//     that is top-R in it, the result is the same for any arrival order;
//   * a row whose primary is owned by another rank becomes a record [g, h, R gids, R dist bits]
//     in the send buffer, grouped by destination rank and ascending g; the owner folds received
//     records in after the exchange (one pass per home index h, so no two folds of the same
//     row run concurrently).
#include "common.cuh"

namespace sg {
namespace {

constexpr int KMAXM = 64;
constexpr int MW = 8;          // warps per CTA in the fold kernels
constexpr uint32_t RMAX = 128;

struct Owners {
    int32_t owner[KMAXM];
};

__device__ __forceinline__ uint32_t n_homes(const uint32_t* home, uint64_t g, uint32_t omega) {
    uint32_t nh = 1;
    while (nh < omega && home[g * omega + nh] != SG_SENT) nh++;
    return nh;
}

// ---------------------------------------------------------------- plan
__global__ void owned_flags(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, Owners o, int rank,
                            uint32_t* __restrict__ flags) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) flags[g] = o.owner[home[g * omega]] == rank;
}

__global__ void owned_index_kernel(const uint32_t* __restrict__ flags, const uint64_t* __restrict__ pos, uint64_t n,
                                   uint32_t* __restrict__ owned_index) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) owned_index[g] = flags[g] ? (uint32_t)pos[g] : SG_SENT;
}

// records this rank sends to / receives from every rank (rows built here whose primary is owned
// elsewhere / rows built elsewhere whose primary is owned here)
__global__ void count_kernel(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, Owners o, int rank,
                             int world, unsigned long long* send, unsigned long long* recv) {
    __shared__ unsigned long long s_send[KMAXM], s_recv[KMAXM];
    if (threadIdx.x < KMAXM) { s_send[threadIdx.x] = 0; s_recv[threadIdx.x] = 0; }
    __syncthreads();
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) {
        const int own = o.owner[home[g * omega]];
        for (uint32_t h = 1; h < omega; h++) {
            const uint32_t s = home[g * omega + h];
            if (s == SG_SENT) break;
            const int src = o.owner[s];
            if (src == own) continue;   // folded locally by the owner
            if (src == rank) atomicAdd(&s_send[own], 1ull);
            if (own == rank) atomicAdd(&s_recv[src], 1ull);
        }
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)world) {
        if (s_send[threadIdx.x]) atomicAdd(&send[threadIdx.x], s_send[threadIdx.x]);
        if (s_recv[threadIdx.x]) atomicAdd(&recv[threadIdx.x], s_recv[threadIdx.x]);
    }
}

__global__ void dest_flags(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, Owners o, int rank, int dest,
                           uint32_t* __restrict__ flags) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    uint32_t c = 0;
    if (o.owner[home[g * omega]] == dest)
        for (uint32_t h = 1; h < omega; h++) {
            const uint32_t s = home[g * omega + h];
            if (s == SG_SENT) break;
            c += o.owner[s] == rank;
        }
    flags[g] = c;
}

__global__ void slot_kernel(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, Owners o, int rank,
                            const uint32_t* __restrict__ flags, const uint64_t* __restrict__ pos, uint64_t base,
                            uint32_t* __restrict__ rec_slot) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || flags[g] == 0) return;
    uint64_t r = base + pos[g];
    for (uint32_t h = 1; h < omega; h++) {
        const uint32_t s = home[g * omega + h];
        if (s == SG_SENT) break;
        if (o.owner[s] == rank) rec_slot[g * omega + h] = (uint32_t)r++;
    }
}

// ---------------------------------------------------------------- fold
// Fold row B (nb <= R entries: global ids, dists; SENT ids skipped) into the merged row M
// (sorted by (dist, gid), distinct gids, SENT / +inf padded): dedupe by gid keeping the smaller
// distance (ties keep M's entry), then the first R of the (dist, gid) merge of the two sorted
// lists.  One warp; `sm` is the warp's shared scratch.
struct FoldSmem {
    uint64_t mk[RMAX];     // M keys (ord(dist) << 32 | gid), then compacted
    uint64_t bk[RMAX];     // B keys, then sorted
    uint32_t tab[2 * RMAX];   // hash table gid -> M index (open addressing)
};

__device__ __forceinline__ uint32_t fold_hash(uint32_t g) { return (g * 0x9E3779B1u) >> 24; }   // 256 slots

__device__ void fold_row(uint32_t* __restrict__ mrow, float* __restrict__ mrow_d, const uint32_t* bid, const float* bd,
                         uint32_t R, FoldSmem& sm, uint32_t lane) {
    for (uint32_t i = lane; i < 2 * RMAX; i += 32) sm.tab[i] = SG_SENT;
    __syncwarp();
    // M (sorted, SENT at the end)
    uint32_t a = 0;
    for (uint32_t i0 = 0; i0 < R; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t id = i < R ? mrow[i] : SG_SENT;
        const bool real = id != SG_SENT;
        if (real) {
            sm.mk[i] = ((uint64_t)f2ord(mrow_d[i]) << 32) | id;
            uint32_t hs = fold_hash(id);
            while (atomicCAS(&sm.tab[hs], SG_SENT, i) != SG_SENT) hs = (hs + 1) & (2 * RMAX - 1);
        }
        a += __popc(__ballot_sync(0xffffffffu, real));
    }
    __syncwarp();
    // B: dedupe against M
    uint32_t b = 0;
    for (uint32_t j0 = 0; j0 < R; j0 += 32) {
        const uint32_t j = j0 + lane;
        const uint32_t id = j < R ? bid[j] : SG_SENT;
        bool keep = id != SG_SENT;
        uint64_t key = 0;
        if (keep) {
            key = ((uint64_t)f2ord(bd[j]) << 32) | id;
            uint32_t hs = fold_hash(id);
            for (;;) {
                const uint32_t mi = sm.tab[hs];
                if (mi == SG_SENT) break;
                if ((uint32_t)sm.mk[mi] == id) {
                    if (key < sm.mk[mi]) sm.mk[mi] = ~0ull;   // B's entry is closer: M's copy goes
                    else keep = false;
                    break;
                }
                hs = (hs + 1) & (2 * RMAX - 1);
            }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) sm.bk[b + __popc(bal & ((1u << lane) - 1u))] = key;
        b += __popc(bal);
    }
    __syncwarp();
    // compact M (removed entries are ~0; the survivors stay sorted)
    uint32_t a2 = 0;
    for (uint32_t i0 = 0; i0 < a; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint64_t k = i < a ? sm.mk[i] : ~0ull;
        const bool keep = k != ~0ull;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) sm.mk[a2 + __popc(bal & ((1u << lane) - 1u))] = k;
        a2 += __popc(bal);
        __syncwarp();
    }
    SG_DCHECK(a <= R && b <= R && a2 <= a);
    // sort B (bitonic over the next power of two)
    uint32_t np = 32;
    while (np < b) np <<= 1;
    for (uint32_t j = b + lane; j < np; j += 32) sm.bk[j] = ~0ull;
    __syncwarp();
    warp_sort_u64(sm.bk, np, lane);
    // merge: output position = own index + number of smaller entries of the other list
    for (uint32_t i = lane; i < a2; i += 32) {
        const uint64_t k = sm.mk[i];
        uint32_t lo = 0, hi = b;
        while (lo < hi) { const uint32_t md = (lo + hi) >> 1; if (sm.bk[md] < k) lo = md + 1; else hi = md; }
        const uint32_t p = i + lo;
        if (p < R) { mrow[p] = (uint32_t)k; mrow_d[p] = ord2f((uint32_t)(k >> 32)); }
    }
    for (uint32_t j = lane; j < b; j += 32) {
        const uint64_t k = sm.bk[j];
        uint32_t lo = 0, hi = a2;
        while (lo < hi) { const uint32_t md = (lo + hi) >> 1; if (sm.mk[md] < k) lo = md + 1; else hi = md; }
        const uint32_t p = j + lo;
        if (p < R) { mrow[p] = (uint32_t)k; mrow_d[p] = ord2f((uint32_t)(k >> 32)); }
    }
    for (uint32_t p = a2 + b + lane; p < R; p += 32) { mrow[p] = SG_SENT; mrow_d[p] = __int_as_float(0x7f800000); }
    __syncwarp();
}

// one warp per local row of the shard just built
__global__ void __launch_bounds__(MW * 32) merge_shard_kernel(
    const uint32_t* __restrict__ home, uint32_t omega, Owners o, int rank, uint32_t shard,
    const uint32_t* __restrict__ idmap, uint64_t m, const uint32_t* __restrict__ graph, const float* __restrict__ graph_d,
    uint32_t R, const uint32_t* __restrict__ owned_index, const uint32_t* __restrict__ rec_slot,
    uint32_t* __restrict__ merged, float* __restrict__ merged_d, uint32_t* __restrict__ sendbuf) {
    __shared__ FoldSmem s_f[MW];
    __shared__ uint32_t s_id[MW][RMAX];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * MW;
    const uint32_t W = 2 + 2 * R;
    for (uint64_t l = (uint64_t)blockIdx.x * MW + w; l < m; l += nwarps) {
        const uint64_t g = idmap[l];
        uint32_t h = 0;
        while (home[g * omega + h] != shard) h++;
        const uint32_t nh = n_homes(home, g, omega);
        const uint32_t* grow = graph + l * R;
        const float* grow_d = graph_d + l * R;
        if (o.owner[home[g * omega]] == rank) {
            const uint64_t oi = owned_index[g];
            SG_DCHECK(oi != SG_SENT);
            uint32_t* mrow = merged + oi * R;
            float* mrow_d = merged_d + oi * R;
            if (nh == 1) {   // single home: the shard row as is
                for (uint32_t j = lane; j < R; j += 32) {
                    const uint32_t lid = grow[j];
                    mrow[j] = lid == SG_SENT ? SG_SENT : idmap[lid];
                    mrow_d[j] = grow_d[j];
                }
            } else {
                for (uint32_t j = lane; j < R; j += 32) {
                    const uint32_t lid = grow[j];
                    s_id[w][j] = lid == SG_SENT ? SG_SENT : idmap[lid];
                }
                __syncwarp();
                fold_row(mrow, mrow_d, s_id[w], grow_d, R, s_f[w], lane);
            }
        } else {   // primary owned elsewhere: a record for its owner
            SG_DCHECK(rec_slot[g * omega + h] != SG_SENT);
            uint32_t* r = sendbuf + (uint64_t)rec_slot[g * omega + h] * W;
            if (lane == 0) { r[0] = (uint32_t)g; r[1] = h; }
            for (uint32_t j = lane; j < R; j += 32) {
                const uint32_t lid = grow[j];
                r[2 + j] = lid == SG_SENT ? SG_SENT : idmap[lid];
                r[2 + R + j] = __float_as_uint(grow_d[j]);
            }
        }
        __syncwarp();
    }
}

// fold the received records of home index `pass` (at most one per g)
__global__ void __launch_bounds__(MW * 32) merge_recv_kernel(const uint32_t* __restrict__ recv, uint64_t n_recv,
                                                             uint32_t R, uint32_t pass,
                                                             const uint32_t* __restrict__ owned_index,
                                                             uint32_t* __restrict__ merged, float* __restrict__ merged_d,
                                                             int* __restrict__ err) {
    __shared__ FoldSmem s_f[MW];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * MW;
    const uint32_t W = 2 + 2 * R;
    for (uint64_t i = (uint64_t)blockIdx.x * MW + w; i < n_recv; i += nwarps) {
        const uint32_t* r = recv + i * W;
        if (r[1] != pass) continue;
        const uint64_t oi = owned_index[r[0]];
        if (oi == SG_SENT) { if (lane == 0) atomicExch(err, 1); continue; }
        fold_row(merged + oi * R, merged_d + oi * R, r + 2, (const float*)(r + 2 + R), R, s_f[w], lane);
    }
}

sg_status make_owners(Owners* o, uint32_t k, const int32_t* owner, int world) {
    SG_CHECK_ARG(k >= 1 && k <= KMAXM, "merge: k must be in [1, 64]");
    SG_CHECK_ARG(world >= 1 && world <= KMAXM, "merge: world must be in [1, 64]");
    for (uint32_t s = 0; s < KMAXM; s++) o->owner[s] = s < k ? (owner ? owner[s] : 0) : -1;
    for (uint32_t s = 0; s < k; s++) SG_CHECK_ARG(o->owner[s] >= 0 && o->owner[s] < world, "merge: owner out of range");
    return SG_OK;
}

inline unsigned blocks_for(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

size_t merge_plan_ws(uint64_t n) {
    Carver cv(nullptr, 0);
    cv.take<unsigned long long>(2 * KMAXM);
    cv.take<uint32_t>(n);        // flags
    cv.take<uint64_t>(n + 1);    // positions
    return cv.off + scan_workspace(n) + 2048;
}

sg_status merge_plan_run(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k, const int32_t* owner, int rank,
                         int world, uint32_t* owned_index, uint32_t* rec_slot, uint64_t* send_host, uint64_t* recv_host,
                         uint64_t* n_owned_host, void* ws, size_t ws_bytes, cudaStream_t st) {
    SG_CHECK_ARG(home && n > 0 && omega >= 1 && rank >= 0 && rank < world, "merge_plan: bad arguments");
    Owners o;
    SG_TRY(make_owners(&o, k, owner, world));
    Carver cv(ws, ws_bytes);
    unsigned long long* cnt = cv.take<unsigned long long>(2 * KMAXM);
    uint32_t* flags = cv.take<uint32_t>(n);
    uint64_t* pos = cv.take<uint64_t>(n + 1);
    if (!cv.ok()) { set_error("merge_plan: workspace too small"); return SG_ERR_WORKSPACE; }
    const unsigned nb = blocks_for(n, 256);
    SG_CUDA(cudaMemsetAsync(cnt, 0, 2 * KMAXM * sizeof(unsigned long long), st));
    count_kernel<<<nb, 256, 0, st>>>(home, n, omega, o, rank, world, cnt, cnt + KMAXM);
    SG_LAUNCHED("count_kernel");
    // owned rows, ascending gid
    owned_flags<<<nb, 256, 0, st>>>(home, n, omega, o, rank, flags);
    SG_LAUNCHED("owned_flags");
    {
        Carver c2 = cv;
        SG_TRY(excl_scan_u32_to_u64(flags, pos, n, c2, st));
    }
    if (owned_index) {
        owned_index_kernel<<<nb, 256, 0, st>>>(flags, pos, n, owned_index);
        SG_LAUNCHED("owned_index_kernel");
    }
    uint64_t n_owned = 0;
    unsigned long long h[2 * KMAXM];
    SG_CUDA(cudaMemcpyAsync(&n_owned, pos + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    if (n_owned_host) *n_owned_host = n_owned;
    for (int r = 0; r < world; r++) {
        if (send_host) send_host[r] = h[r];
        if (recv_host) recv_host[r] = h[KMAXM + r];
    }
    // send slots: grouped by destination rank, ascending g (then h) within a destination
    if (rec_slot) {
        SG_CUDA(cudaMemsetAsync(rec_slot, 0xFF, n * omega * sizeof(uint32_t), st));
        uint64_t base = 0;
        for (int dest = 0; dest < world; dest++) {
            if (h[dest] == 0) continue;
            dest_flags<<<nb, 256, 0, st>>>(home, n, omega, o, rank, dest, flags);
            SG_LAUNCHED("dest_flags");
            Carver c2 = cv;
            SG_TRY(excl_scan_u32_to_u64(flags, pos, n, c2, st));
            slot_kernel<<<nb, 256, 0, st>>>(home, n, omega, o, rank, flags, pos, base, rec_slot);
            SG_LAUNCHED("slot_kernel");
            base += h[dest];
        }
    }
    return SG_OK;
}

sg_status merge_init_run(uint64_t n_owned, uint32_t R, uint32_t* merged, float* merged_d, cudaStream_t st) {
    if (n_owned == 0) return SG_OK;
    SG_CUDA(cudaMemsetAsync(merged, 0xFF, n_owned * R * sizeof(uint32_t), st));
    SG_CUDA(cudaMemsetAsync(merged_d, 0x7F, n_owned * R * sizeof(float), st));   // 0x7F7F7F7F: finite, never read
    return SG_OK;
}

sg_status merge_shard_run(const uint32_t* home, uint32_t omega, uint32_t k, const int32_t* owner, int rank, int world,
                          uint32_t shard, const uint32_t* idmap, uint64_t m, const uint32_t* graph, const float* graph_d,
                          uint32_t R, const uint32_t* owned_index, const uint32_t* rec_slot, uint32_t* merged,
                          float* merged_d, uint32_t* sendbuf, cudaStream_t st) {
    SG_CHECK_ARG(R >= 1 && R <= RMAX, "merge: R must be in [1, 128]");
    SG_CHECK_ARG(shard < k, "merge: shard out of range");
    Owners o;
    SG_TRY(make_owners(&o, k, owner, world));
    if (m == 0) return SG_OK;
    const uint64_t blocks = (m + MW - 1) / MW, cap = (uint64_t)num_sms() * 8;
    merge_shard_kernel<<<(unsigned)(blocks < cap ? blocks : cap), MW * 32, 0, st>>>(
        home, omega, o, rank, shard, idmap, m, graph, graph_d, R, owned_index, rec_slot, merged, merged_d, sendbuf);
    SG_LAUNCHED("merge_shard_kernel");
    return SG_OK;
}

sg_status merge_finish_run(uint32_t omega, uint32_t R, const uint32_t* owned_index, const uint32_t* recvbuf,
                           uint64_t n_recv, uint32_t* merged, float* merged_d, int* err_dev, cudaStream_t st) {
    SG_CHECK_ARG(R >= 1 && R <= RMAX, "merge: R must be in [1, 128]");
    if (n_recv == 0) return SG_OK;
    SG_CUDA(cudaMemsetAsync(err_dev, 0, sizeof(int), st));
    const uint64_t blocks = (n_recv + MW - 1) / MW, cap = (uint64_t)num_sms() * 8;
    for (uint32_t pass = 1; pass < omega; pass++) {
        merge_recv_kernel<<<(unsigned)(blocks < cap ? blocks : cap), MW * 32, 0, st>>>(recvbuf, n_recv, R, pass,
                                                                                      owned_index, merged, merged_d,
                                                                                      err_dev);
        SG_LAUNCHED("merge_recv_kernel");
    }
    int herr = 0;
    SG_CUDA(cudaMemcpyAsync(&herr, err_dev, sizeof(int), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    if (herr) { set_error("merge: a received record is for a row not owned here"); return SG_ERR_INVALID_ARG; }
    return SG_OK;
}

}  // namespace sg
