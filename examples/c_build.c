/*
 * A C-only caller of libscalegann.so: the whole divide-and-merge build (a1-a8) on `world`
 * processes, one per GPU, through include/scalegann.h alone (no Python, no torch).
 *
 *   c_build DATA.bin n d k rank world UID_FILE OUT.bin
 *
 * DATA.bin holds n x d float32 rows.  Rank 0 writes the communicator's unique id to UID_FILE;
 * the other ranks wait for it (the out-of-band channel of scalegann_comm_init).  Each rank
 * writes its owned merged rows (n_owned x R uint32, ascending global id) to OUT.bin.<rank>.
 * Parameters: omega 2, eps 1.2, theta0 0.4, alpha 1, block 65536, L 64, R 32 (C0's degrees).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "../include/scalegann.h"

#define CHECK(call)                                                                       \
    do {                                                                                  \
        sg_status _s = (call);                                                            \
        if (_s != SG_OK) {                                                                \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)_s, scalegann_last_error()); \
            exit(1);                                                                      \
        }                                                                                 \
    } while (0)
#define CUDA(call)                                                                        \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) {                                                          \
            fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(_e));            \
            exit(1);                                                                      \
        }                                                                                 \
    } while (0)

static void* dalloc(size_t bytes) {
    void* p = NULL;
    CUDA(cudaMalloc(&p, bytes ? bytes : 256));
    return p;
}

/* longest-processing-time placement of shards by m^2 (ties to the lower shard / rank) */
static void lpt_owner(const uint64_t* sizes, uint32_t k, int world, int32_t* owner) {
    double load[64] = {0};
    int done[64] = {0};
    for (uint32_t it = 0; it < k; it++) {
        int s = -1;
        for (uint32_t t = 0; t < k; t++)
            if (!done[t] && (s < 0 || sizes[t] > sizes[s])) s = (int)t;
        int r = 0;
        for (int q = 1; q < world; q++)
            if (load[q] < load[r]) r = q;
        owner[s] = r;
        load[r] += (double)sizes[s] * (double)sizes[s];
        done[s] = 1;
    }
}

int main(int argc, char** argv) {
    if (argc != 9) {
        fprintf(stderr, "usage: c_build DATA.bin n d k rank world UID_FILE OUT.bin\n");
        return 2;
    }
    const uint64_t n = strtoull(argv[2], NULL, 10);
    const uint32_t d = (uint32_t)atoi(argv[3]), k = (uint32_t)atoi(argv[4]);
    const int rank = atoi(argv[5]), world = atoi(argv[6]);
    const uint32_t omega = 2, L = 64, R = 32;
    CUDA(cudaSetDevice(rank));
    cudaStream_t st;
    CUDA(cudaStreamCreate(&st));

    /* the dataset, on every rank (the partition runs identically everywhere) */
    float* xh = (float*)malloc(n * d * sizeof(float));
    FILE* f = fopen(argv[1], "rb");
    if (!f || fread(xh, sizeof(float), n * d, f) != n * d) { fprintf(stderr, "cannot read %s\n", argv[1]); return 1; }
    fclose(f);
    float* x = (float*)dalloc(n * d * sizeof(float));
    CUDA(cudaMemcpy(x, xh, n * d * sizeof(float), cudaMemcpyHostToDevice));

    /* the communicator: rank 0's unique id through a file */
    void* comm = NULL;
    if (world > 1) {
        uint8_t uid[128];
        char tmp[4096];
        if (rank == 0) {
            CHECK(scalegann_get_unique_id(uid));
            snprintf(tmp, sizeof(tmp), "%s.tmp", argv[7]);
            FILE* u = fopen(tmp, "wb");
            fwrite(uid, 1, 128, u);
            fclose(u);
            rename(tmp, argv[7]);
        } else {
            FILE* u = NULL;
            while (!(u = fopen(argv[7], "rb"))) usleep(10000);
            if (fread(uid, 1, 128, u) != 128) { fprintf(stderr, "short uid file\n"); return 1; }
            fclose(u);
        }
        CHECK(scalegann_comm_init(rank, world, uid, &comm));
    }

    /* one workspace, grown to the largest query */
    size_t ws_bytes = 0, b = 0;
    void* ws = NULL;
#define WS_NEED(q)                                              \
    do {                                                        \
        CHECK(q);                                               \
        if (b > ws_bytes) {                                     \
            if (ws) CUDA(cudaFree(ws));                         \
            ws_bytes = b;                                       \
            ws = dalloc(ws_bytes);                              \
        }                                                       \
    } while (0)

    /* a1: centroids on rank 0, N1 broadcast */
    float* C = (float*)dalloc((size_t)k * d * sizeof(float));
    WS_NEED(scalegann_kmeans_workspace(n, d, k, 256, &b));
    if (rank == 0) CHECK(scalegann_kmeans(x, SG_F32, n, d, k, 42, 15, 256, C, ws, ws_bytes, st));
    CHECK(scalegann_broadcast_centroids(comm, C, k, d, st));

    /* a2-a3: partition */
    sg_partition_params pp = {k, omega, 1.2f, 400000u, 1.0f, 65536u, 0};
    uint32_t* home = (uint32_t*)dalloc(n * omega * 4);
    float* pd = (float*)dalloc(n * 4);
    uint64_t counts[3 * 64];
    WS_NEED(scalegann_partition_workspace(n, d, &pp, &b));
    CHECK(scalegann_partition(x, SG_F32, n, d, C, &pp, home, pd, counts, ws, ws_bytes, st));
    const uint64_t* sizes = counts;
    int32_t owner[64];
    lpt_owner(sizes, k, world, owner);

    /* a8 plan: owned rows, send slots, record counts */
    uint32_t* owned_index = (uint32_t*)dalloc(n * 4);
    uint32_t* rec_slot = (uint32_t*)dalloc(n * omega * 4);
    uint64_t send[64], recv[64], n_owned = 0, ns = 0, nr = 0;
    WS_NEED(scalegann_merge_plan_workspace(n, &b));
    CHECK(scalegann_merge_plan(home, n, omega, k, owner, rank, world, owned_index, rec_slot, send, recv, &n_owned, ws,
                               ws_bytes, st));
    for (int r = 0; r < world; r++) { ns += send[r]; nr += recv[r]; }
    const uint32_t W = 2 + 2 * R;
    uint32_t* merged = (uint32_t*)dalloc(n_owned * R * 4);
    float* merged_d = (float*)dalloc(n_owned * R * 4);
    uint32_t* sendbuf = (uint32_t*)dalloc(ns * W * 4);
    uint32_t* recvbuf = (uint32_t*)dalloc(nr * W * 4);
    CHECK(scalegann_merge_init(n_owned, R, merged, merged_d, st));

    /* a4-a7 per owned shard, each folded into the merged rows and freed */
    sg_build_params bp = {L, R, SG_L2, SG_PREC_AUTO, 0, 0};
    for (uint32_t s = 0; s < k; s++) {
        if (owner[s] != rank || sizes[s] == 0) continue;
        const uint64_t m = sizes[s];
        uint32_t* idmap = (uint32_t*)dalloc(m * 4);
        uint32_t* graph = (uint32_t*)dalloc(m * R * 4);
        float* graph_d = (float*)dalloc(m * R * 4);
        WS_NEED(scalegann_shard_idmap_workspace(n, &b));
        CHECK(scalegann_shard_idmap(home, n, omega, s, idmap, NULL, NULL, ws, ws_bytes, st));
        WS_NEED(scalegann_build_shard_workspace(m, d, SG_F32, &bp, &b));
        CHECK(scalegann_build_shard(x, SG_F32, n, d, idmap, m, &bp, NULL, NULL, graph, graph_d, ws, ws_bytes, st));
        CHECK(scalegann_merge_shard(home, n, omega, k, owner, rank, world, s, idmap, m, graph, graph_d, R,
                                    owned_index, rec_slot, merged, merged_d, sendbuf, st));
        CUDA(cudaStreamSynchronize(st));
        CUDA(cudaFree(idmap));
        CUDA(cudaFree(graph));
        CUDA(cudaFree(graph_d));
    }

    /* N2 + fold of the received rows */
    CHECK(scalegann_exchange_records(comm, sendbuf, send, recvbuf, recv, W, st));
    CHECK(scalegann_merge_finish(omega, R, owned_index, recvbuf, nr, merged, merged_d, ws, ws_bytes, st));

    uint32_t* mh = (uint32_t*)malloc(n_owned * R * 4 + 4);
    CUDA(cudaMemcpy(mh, merged, n_owned * R * 4, cudaMemcpyDeviceToHost));
    char out[4096];
    snprintf(out, sizeof(out), "%s.%d", argv[8], rank);
    FILE* o = fopen(out, "wb");
    fwrite(mh, 4, n_owned * R, o);
    fclose(o);
    printf("rank %d: %llu owned rows, sent %llu, received %llu records\n", rank, (unsigned long long)n_owned,
           (unsigned long long)ns, (unsigned long long)nr);
    CHECK(scalegann_comm_destroy(comm));
    return 0;
}
