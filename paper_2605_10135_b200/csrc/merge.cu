// a8 — cross-shard merge by edge union + re-prune ("edge union", P:242;
// reading R12).  Distributed by primary owner: every replica row (g, h >= 1) built on this
// rank travels to the rank that owns g's primary shard as a record
// [g, h, R global ids, R distance bits]; the owner unions its primary row with the received
// rows, dedupes by gid keeping the minimum carried distance, sorts by (dist, gid) and keeps R.
#include "common.cuh"

namespace sg {
namespace {

constexpr int KMAXM = 64;
constexpr int MW = 8;   // warps per CTA in the union kernel

struct ShardTabs {
    const uint32_t* idmap[KMAXM];
    const uint32_t* graph[KMAXM];
    const float* graph_d[KMAXM];
    int32_t owner[KMAXM];
};

__global__ void count_kernel(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, ShardTabs t, int rank,
                             int world, unsigned long long* send, unsigned long long* recv) {
    __shared__ unsigned long long s_send[KMAXM], s_recv[KMAXM];
    if (threadIdx.x < KMAXM) { s_send[threadIdx.x] = 0; s_recv[threadIdx.x] = 0; }
    __syncthreads();
    uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) {
        const int own = t.owner[home[g * omega]];
        for (uint32_t h = 1; h < omega; h++) {
            const uint32_t s = home[g * omega + h];
            if (s == SG_SENT) break;
            if (t.owner[s] == rank) atomicAdd(&s_send[own], 1ull);
            if (own == rank) atomicAdd(&s_recv[t.owner[s]], 1ull);
        }
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)world) {
        if (s_send[threadIdx.x]) atomicAdd(&send[threadIdx.x], s_send[threadIdx.x]);
        if (s_recv[threadIdx.x]) atomicAdd(&recv[threadIdx.x], s_recv[threadIdx.x]);
    }
}

// number of records g contributes to destination `dest`
__global__ void dest_flags(const uint32_t* __restrict__ home, uint64_t n, uint32_t omega, ShardTabs t, int rank,
                           int dest, uint32_t* __restrict__ flags) {
    uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    uint32_t c = 0;
    if (t.owner[home[g * omega]] == dest)
        for (uint32_t h = 1; h < omega; h++) {
            const uint32_t s = home[g * omega + h];
            if (s == SG_SENT) break;
            c += t.owner[s] == rank;
        }
    flags[g] = c;
}

__global__ void pack_kernel(const uint32_t* __restrict__ home, const uint32_t* __restrict__ inv, uint64_t n,
                            uint32_t omega, ShardTabs t, int rank, const uint32_t* __restrict__ flags,
                            const uint64_t* __restrict__ pos, uint64_t base, uint32_t R, uint32_t* __restrict__ sendbuf) {
    const uint64_t g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (g >= n || flags[g] == 0) return;
    const uint32_t W = 2 + 2 * R;
    uint64_t rec = base + pos[g];
    for (uint32_t h = 1; h < omega; h++) {
        const uint32_t s = home[g * omega + h];
        if (s == SG_SENT) break;
        if (t.owner[s] != rank) continue;
        const uint64_t l = inv[g * omega + h];
        uint32_t* r = sendbuf + rec * W;
        if (lane == 0) { r[0] = (uint32_t)g; r[1] = h; }
        for (uint32_t j = lane; j < R; j += 32) {
            const uint32_t lid = t.graph[s][l * R + j];
            r[2 + j] = lid == SG_SENT ? SG_SENT : t.idmap[s][lid];
            r[2 + R + j] = __float_as_uint(t.graph_d[s][l * R + j]);
        }
        rec++;
    }
}

__global__ void index_records(const uint32_t* __restrict__ recv, uint64_t nrec, uint32_t R, uint32_t omega,
                              uint32_t* __restrict__ rec_index) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrec) return;
    const uint32_t* r = recv + i * (2 + 2 * R);
    rec_index[(uint64_t)r[0] * omega + r[1]] = (uint32_t)i;
}

__global__ void __launch_bounds__(MW * 32) union_kernel(const uint32_t* __restrict__ home, const uint32_t* __restrict__ inv,
                                                         uint64_t n, uint32_t omega, ShardTabs t, int rank,
                                                         const uint32_t* __restrict__ recv,
                                                         const uint32_t* __restrict__ rec_index, uint32_t R,
                                                         uint32_t* __restrict__ merged, float* __restrict__ merged_d,
                                                         int* __restrict__ err) {
    __shared__ uint64_t s_buf[MW][512];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* buf = s_buf[w];
    const uint32_t W = 2 + 2 * R;
    const uint64_t nwarps = (uint64_t)gridDim.x * MW;
    for (uint64_t g = (uint64_t)blockIdx.x * MW + w; g < n; g += nwarps) {
        const uint32_t s0 = home[g * omega];
        if (t.owner[s0] != rank) continue;
        uint32_t nh = 1;
        while (nh < omega && home[g * omega + nh] != SG_SENT) nh++;
        const uint64_t l0 = inv[g * omega];
        if (nh == 1) {
            for (uint32_t j = lane; j < R; j += 32) {
                const uint32_t lid = t.graph[s0][l0 * R + j];
                merged[g * R + j] = lid == SG_SENT ? SG_SENT : t.idmap[s0][lid];
                merged_d[g * R + j] = t.graph_d[s0][l0 * R + j];
            }
            continue;
        }
        // union candidates keyed (gid, dist) for the dedupe
        uint32_t np = 32;
        while (np < nh * R) np <<= 1;
        for (uint32_t i = lane; i < np; i += 32) buf[i] = ~0ull;
        __syncwarp();
        for (uint32_t j = lane; j < R; j += 32) {
            const uint32_t lid = t.graph[s0][l0 * R + j];
            if (lid != SG_SENT)
                buf[j] = ((uint64_t)t.idmap[s0][lid] << 32) | f2ord(t.graph_d[s0][l0 * R + j]);
        }
        for (uint32_t h = 1; h < nh; h++) {
            const uint32_t ri = rec_index[g * omega + h];
            if (ri == SG_SENT) { if (lane == 0) atomicExch(err, 1); continue; }
            const uint32_t* r = recv + (uint64_t)ri * W;
            for (uint32_t j = lane; j < R; j += 32) {
                const uint32_t gid = r[2 + j];
                if (gid != SG_SENT) buf[h * R + j] = ((uint64_t)gid << 32) | f2ord(__uint_as_float(r[2 + R + j]));
            }
        }
        __syncwarp();
        warp_sort_u64(buf, np, lane);
        // dedupe: first of each gid run has the minimum distance; re-key as (dist, gid)
        uint64_t rk[16];
#pragma unroll
        for (int q = 0; q < 16; q++) {
            const uint32_t i = q * 32 + lane;
            rk[q] = ~0ull;
            if (i < np) {
                const uint64_t cur = buf[i];
                const bool first = cur != ~0ull && (i == 0 || (buf[i - 1] >> 32) != (cur >> 32));
                if (first) rk[q] = ((uint64_t)(uint32_t)cur << 32) | (cur >> 32);
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 16; q++) {
            const uint32_t i = q * 32 + lane;
            if (i < np) buf[i] = rk[q];
        }
        __syncwarp();
        warp_sort_u64(buf, np, lane);
        for (uint32_t j = lane; j < R; j += 32) {
            const uint64_t v = buf[j];
            merged[g * R + j] = v == ~0ull ? SG_SENT : (uint32_t)v;
            merged_d[g * R + j] = v == ~0ull ? __int_as_float(0x7f800000) : ord2f((uint32_t)(v >> 32));
        }
        __syncwarp();
    }
}

sg_status make_tabs(ShardTabs* t, uint32_t k, const int32_t* owner, const uint32_t* const* idmaps,
                    const uint32_t* const* graphs, const float* const* graphs_d) {
    SG_CHECK_ARG(k >= 1 && k <= KMAXM, "merge: k must be in [1, 64]");
    memset(t, 0, sizeof(*t));
    for (uint32_t s = 0; s < k; s++) {
        t->owner[s] = owner ? owner[s] : 0;
        t->idmap[s] = idmaps ? idmaps[s] : nullptr;
        t->graph[s] = graphs ? graphs[s] : nullptr;
        t->graph_d[s] = graphs_d ? graphs_d[s] : nullptr;
    }
    return SG_OK;
}

}  // namespace

sg_status merge_counts_run(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k, const int32_t* owner,
                           int rank, int world, uint64_t* send_host, uint64_t* recv_host, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
    SG_CHECK_ARG(world >= 1 && world <= KMAXM && rank >= 0 && rank < world, "merge: bad rank/world");
    ShardTabs t;
    SG_TRY(make_tabs(&t, k, owner, nullptr, nullptr, nullptr));
    Carver cv(ws, ws_bytes);
    unsigned long long* d = cv.take<unsigned long long>(2 * KMAXM);
    if (!cv.ok()) { set_error("merge: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(d, 0, 2 * KMAXM * sizeof(unsigned long long), st));
    count_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(home, n, omega, t, rank, world, d, d + KMAXM);
    SG_LAUNCHED("count_kernel");
    unsigned long long h[2 * KMAXM];
    SG_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < world; r++) {
        if (send_host) send_host[r] = h[r];
        if (recv_host) recv_host[r] = h[KMAXM + r];
    }
    return SG_OK;
}

size_t merge_ws(uint64_t n, uint32_t omega) {
    Carver cv(nullptr, 0);
    cv.take<unsigned long long>(2 * KMAXM);
    cv.take<uint32_t>(n);        // flags
    cv.take<uint64_t>(n + 1);    // positions
    cv.take<uint32_t>(n * omega);// record index
    cv.take<int>(1);
    return cv.off + scan_workspace(n) + 2048;
}

sg_status merge_pack_run(const uint32_t* home, const uint32_t* inv, uint64_t n, uint32_t omega, uint32_t k,
                         const int32_t* owner, int rank, int world, const uint32_t* const* idmaps,
                         const uint32_t* const* graphs, const float* const* graphs_d, uint32_t R, uint32_t* sendbuf,
                         void* ws, size_t ws_bytes, cudaStream_t st) {
    ShardTabs t;
    SG_TRY(make_tabs(&t, k, owner, idmaps, graphs, graphs_d));
    uint64_t send[KMAXM];
    SG_TRY(merge_counts_run(home, n, omega, k, owner, rank, world, send, nullptr, ws, ws_bytes, st));
    Carver cv(ws, ws_bytes);
    cv.take<unsigned long long>(2 * KMAXM);
    uint32_t* flags = cv.take<uint32_t>(n);
    uint64_t* pos = cv.take<uint64_t>(n + 1);
    if (!cv.ok()) { set_error("merge: workspace too small"); return SG_ERR_WORKSPACE; }
    uint64_t base = 0;
    const unsigned nb = (unsigned)((n + 255) / 256);
    for (int dest = 0; dest < world; dest++) {
        if (send[dest] == 0) continue;
        Carver cv2 = cv;
        dest_flags<<<nb, 256, 0, st>>>(home, n, omega, t, rank, dest, flags);
        SG_LAUNCHED("dest_flags");
        SG_TRY(excl_scan_u32_to_u64(flags, pos, n, cv2, st));
        pack_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(home, inv, n, omega, t, rank, flags, pos, base,
                                                                         R, sendbuf);
        SG_LAUNCHED("pack_kernel");
        base += send[dest];
    }
    return SG_OK;
}

sg_status merge_union_run(const uint32_t* home, const uint32_t* inv, uint64_t n, uint32_t omega, uint32_t k,
                          const int32_t* owner, int rank, const uint32_t* const* idmaps, const uint32_t* const* graphs,
                          const float* const* graphs_d, uint32_t R, const uint32_t* recvbuf, uint64_t n_recv,
                          uint32_t* merged, float* merged_d, void* ws, size_t ws_bytes, cudaStream_t st) {
    SG_CHECK_ARG(omega * R <= 512, "merge: omega * R must be <= 512");
    ShardTabs t;
    SG_TRY(make_tabs(&t, k, owner, idmaps, graphs, graphs_d));
    Carver cv(ws, ws_bytes);
    cv.take<unsigned long long>(2 * KMAXM);
    cv.take<uint32_t>(n);
    cv.take<uint64_t>(n + 1);
    uint32_t* rec_index = cv.take<uint32_t>(n * omega);
    int* err = cv.take<int>(1);
    if (!cv.ok()) { set_error("merge: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(rec_index, 0xFF, n * omega * sizeof(uint32_t), st));
    SG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
    if (n_recv) {
        index_records<<<(unsigned)((n_recv + 255) / 256), 256, 0, st>>>(recvbuf, n_recv, R, omega, rec_index);
        SG_LAUNCHED("index_records");
    }
    const uint64_t blocks = (n + MW - 1) / MW, cap = (uint64_t)num_sms() * 16;
    union_kernel<<<(unsigned)(blocks < cap ? blocks : cap), MW * 32, 0, st>>>(home, inv, n, omega, t, rank, recvbuf,
                                                                              rec_index, R, merged, merged_d, err);
    SG_LAUNCHED("union_kernel");
    int herr = 0;
    SG_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaStreamSynchronize(st));
    if (herr) { set_error("merge: a replica row was not received"); return SG_ERR_INVALID_ARG; }
    return SG_OK;
}

}  // namespace sg
