// One-call index build from HOST buffers (the "e2e" path of bench.py): the dataset is copied to
// the device, a1-a8 run through the library's own entry points (k-means on rank 0 + N1, the
// partition, each owned shard built and folded into the owner rows, N2, the final fold) and the
// merged rows this rank owns are copied back.  The exception to the library's "caller owns all
// memory" rule: this convenience call allocates its device temporaries stream-ordered
// (cudaMallocAsync, so repeated calls reuse the pool) and frees them before returning.
#include <stdlib.h>

#include "common.cuh"

namespace sg {

struct DevArena {   // stream-ordered device allocations freed together
    cudaStream_t st;
    void* ptrs[96];
    int n = 0;
    explicit DevArena(cudaStream_t s) : st(s) {
        // keep freed blocks in the device's default pool between calls (the default release
        // threshold of 0 would hand them back to the driver at every synchronisation, and the
        // next call would map gigabytes again)
        static bool once = false;
        if (!once) {
            int dev = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            cudaGetLastError();
            once = true;
        }
    }
    sg_status take(void** p, size_t bytes) {
        if (n == 96) { set_error("build_index: too many allocations"); return SG_ERR_INVALID_ARG; }
        SG_CUDA(cudaMallocAsync(p, bytes ? bytes : 256, st));
        ptrs[n++] = *p;
        return SG_OK;
    }
    void release() {
        for (int i = n - 1; i >= 0; i--) cudaFreeAsync(ptrs[i], st);
        n = 0;
    }
    ~DevArena() { release(); }
};

// longest-processing-time placement of shards by m^2, ties to the lower shard / rank (the
// placement pipeline.lpt_owner uses)
static void lpt_owner(const uint64_t* sizes, uint32_t k, int world, int32_t* owner) {
    double load[64] = {0};
    bool done[64] = {false};
    for (uint32_t it = 0; it < k; it++) {
        int s = -1;
        for (uint32_t t = 0; t < k; t++)
            if (!done[t] && (s < 0 || sizes[t] > sizes[s])) s = (int)t;
        int r = 0;
        for (int q = 1; q < world; q++)
            if (load[q] < load[r]) r = q;
        owner[s] = r;
        load[r] += (double)sizes[s] * (double)sizes[s];
        done[s] = true;
    }
}

sg_status comm_rank_world(void* comm, int* rank, int* world);

}  // namespace sg

using namespace sg;

extern "C" sg_status scalegann_build_index_host(void* comm, const void* x_host, sg_dtype dtype, uint64_t n, uint32_t d,
                                                const sg_partition_params* pp, const sg_build_params* bp,
                                                uint64_t kmeans_seed, uint32_t* merged_host, float* merged_d_host,
                                                uint64_t* n_owned_host, uint32_t* entry_host, void* stream) {
    SG_CHECK_ARG(x_host && pp && bp && merged_host && n_owned_host && n > 0 && d > 0, "build_index: bad arguments");
    SG_CHECK_ARG(dtype == SG_U8 || dtype == SG_F32, "build_index: bad dtype");
    SG_CHECK_ARG(pp->k >= 1 && pp->k <= 64 && pp->omega >= 1, "build_index: need 1 <= k <= 64, omega >= 1");
    cudaStream_t st = S(stream);
    int rank, world;
    SG_TRY(comm_rank_world(comm, &rank, &world));
    const uint32_t k = pp->k, omega = pp->omega, R = bp->R;
    const size_t esz = dtype == SG_U8 ? 1 : 4;
    DevArena ar(st);
    void *x, *C, *home, *pd, *owned_index, *rec_slot;
    SG_TRY(ar.take(&x, n * d * esz));
    SG_CUDA(cudaMemcpyAsync(x, x_host, n * d * esz, cudaMemcpyHostToDevice, st));
    SG_TRY(ar.take(&C, (size_t)k * d * 4));
    SG_TRY(ar.take(&home, n * omega * 4));
    SG_TRY(ar.take(&pd, n * 4));
    SG_TRY(ar.take(&owned_index, n * 4));
    SG_TRY(ar.take(&rec_slot, n * omega * 4));
    // one workspace for every step: the largest of their queries
    size_t ws_bytes = 4096, b = 0;
    SG_TRY(scalegann_kmeans_workspace(n, d, k, 256, &b));
    ws_bytes = b > ws_bytes ? b : ws_bytes;
    SG_TRY(scalegann_partition_workspace(n, d, pp, &b));
    ws_bytes = b > ws_bytes ? b : ws_bytes;
    SG_TRY(scalegann_shard_idmap_workspace(n, &b));
    ws_bytes = b > ws_bytes ? b : ws_bytes;
    SG_TRY(scalegann_merge_plan_workspace(n, &b));
    ws_bytes = b > ws_bytes ? b : ws_bytes;
    void* ws = nullptr;
    // a1: centroids on rank 0, N1 broadcast
    void* ws0;
    SG_TRY(ar.take(&ws0, ws_bytes));
    if (rank == 0)
        SG_TRY(scalegann_kmeans(x, dtype, n, d, k, kmeans_seed, 15, 256, (float*)C, ws0, ws_bytes, stream));
    SG_TRY(scalegann_broadcast_centroids(comm, (float*)C, k, d, stream));
    // a2-a3
    uint64_t counts[3 * 64];
    SG_TRY(scalegann_partition(x, dtype, n, d, (const float*)C, pp, (uint32_t*)home, (float*)pd, counts, ws0, ws_bytes,
                               stream));
    const uint64_t* sizes = counts;
    int32_t owner[64];
    lpt_owner(sizes, k, world, owner);
    // a8 plan + owner rows
    uint64_t send[64], recv[64], n_owned = 0, ns = 0, nr = 0;
    SG_TRY(scalegann_merge_plan((const uint32_t*)home, n, omega, k, owner, rank, world, (uint32_t*)owned_index,
                                (uint32_t*)rec_slot, send, recv, &n_owned, ws0, ws_bytes, stream));
    for (int r = 0; r < world; r++) { ns += send[r]; nr += recv[r]; }
    const uint32_t W = 2 + 2 * R;
    void *merged, *merged_d, *sendbuf, *recvbuf;
    SG_TRY(ar.take(&merged, n_owned * R * 4));
    SG_TRY(ar.take(&merged_d, n_owned * R * 4));
    SG_TRY(ar.take(&sendbuf, ns * W * 4));
    SG_TRY(ar.take(&recvbuf, nr * W * 4));
    SG_TRY(scalegann_merge_init(n_owned, R, (uint32_t*)merged, (float*)merged_d, stream));
    // a4-a7 per owned shard (the largest shard's workspace, allocated once), folded and freed
    uint64_t mmax = 0;
    for (uint32_t s = 0; s < k; s++)
        if (owner[s] == rank && sizes[s] > mmax) mmax = sizes[s];
    void *idmap = nullptr, *graph = nullptr, *graph_d = nullptr;
    if (mmax >= 2) {
        SG_TRY(scalegann_build_shard_workspace(mmax, d, dtype, bp, &b));
        SG_TRY(ar.take(&ws, b));
        SG_TRY(ar.take(&idmap, mmax * 4));
        SG_TRY(ar.take(&graph, mmax * R * 4));
        SG_TRY(ar.take(&graph_d, mmax * R * 4));
        for (uint32_t s = 0; s < k; s++) {
            if (owner[s] != rank || sizes[s] == 0) continue;
            const uint64_t m = sizes[s];
            SG_TRY(scalegann_shard_idmap((const uint32_t*)home, n, omega, s, (uint32_t*)idmap, nullptr, nullptr, ws0,
                                         ws_bytes, stream));
            SG_TRY(scalegann_build_shard(x, dtype, n, d, (const uint32_t*)idmap, m, bp, nullptr, nullptr,
                                         (uint32_t*)graph, (float*)graph_d, ws, b, stream));
            SG_TRY(scalegann_merge_shard((const uint32_t*)home, n, omega, k, owner, rank, world, s,
                                         (const uint32_t*)idmap, m, (const uint32_t*)graph, (const float*)graph_d, R,
                                         (const uint32_t*)owned_index, (const uint32_t*)rec_slot, (uint32_t*)merged,
                                         (float*)merged_d, (uint32_t*)sendbuf, stream));
        }
    }
    // N2 + fold of the received rows
    SG_TRY(scalegann_exchange_records(comm, (const uint32_t*)sendbuf, send, (uint32_t*)recvbuf, recv, W, stream));
    SG_TRY(scalegann_merge_finish(omega, R, (const uint32_t*)owned_index, (const uint32_t*)recvbuf, nr,
                                  (uint32_t*)merged, (float*)merged_d, ws0, ws_bytes, stream));
    SG_CUDA(cudaMemcpyAsync(merged_host, merged, n_owned * R * 4, cudaMemcpyDeviceToHost, st));
    if (merged_d_host) SG_CUDA(cudaMemcpyAsync(merged_d_host, merged_d, n_owned * R * 4, cudaMemcpyDeviceToHost, st));
    if (entry_host) {
        uint32_t per[64];
        SG_TRY(scalegann_entry_points((const uint32_t*)home, (const float*)pd, n, omega, k, sizes, per, entry_host, ws0,
                                      ws_bytes, stream));
    }
    SG_CUDA(cudaStreamSynchronize(st));
    *n_owned_host = n_owned;
    return SG_OK;
}
