/*
 * scalegann.h — C ABI of libscalegann.so, the B200 (sm_100a) hot path of
 * ScaleGANN's divide-and-merge graph-index construction (arxiv 2605.10135).
 *
 * "P:n" cites /root/reference/PAPER.md line n; "S:n" cites SPEC.md; "R<n>" is
 * a numbered reading of the paper in DESIGN.md ("Readings").
 *
 * Conventions (all functions):
 *  - Plain C: no C++ types, no exceptions, no torch types.  `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Every pointer named x, home, idmap, graph, ... is DEVICE memory on the
 *    current CUDA device unless its name ends in `_host`.  Buffers are owned by
 *    the caller; the library never frees caller memory and allocates nothing:
 *    scratch comes from the caller's `ws` (device) of `ws_bytes`, sized by the
 *    matching *_workspace() query.  Too small a workspace -> SG_ERR_WORKSPACE.
 *  - Calls are stream-ordered and asynchronous except those with a `_host`
 *    output, which synchronise `stream` before returning.
 *  - Arguments are validated before any launch; on error nothing is launched
 *    (or, for errors found on the device, outputs are unspecified) and
 *    scalegann_last_error() returns a thread-local message.  CUDA errors map to
 *    SG_ERR_CUDA; asynchronous kernel faults surface at the next synchronising
 *    call.
 *  - Rows are row-major; ids are uint32 with SG_SENTINEL (0xFFFFFFFF)
 *    for "none"; vector data is n x d of SG_U8 or SG_F32 (paper Table
 *    tab:dataset).
 *  - Local ids of a shard index its idmap, which is ascending in global id
 *    (reading R8), so every (dist, id) tie-break agrees across shards.
 */
#ifndef SCALEGANN_H
#define SCALEGANN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCALEGANN_ABI_VERSION 2
#define SG_SENTINEL 0xFFFFFFFFu

typedef enum {
    SG_OK = 0,
    SG_ERR_INVALID_ARG = 1,
    SG_ERR_UNSUPPORTED = 2,
    SG_ERR_CUDA = 3,
    SG_ERR_CAPACITY = 4,    /* a primary found every cluster full */
    SG_ERR_WORKSPACE = 5,   /* ws_bytes smaller than the *_workspace() answer */
    SG_ERR_TOO_SMALL = 6,   /* shard with m < 2 */
    SG_ERR_NCCL = 7         /* a collective failed (NCCL) */
} sg_status;

typedef enum { SG_U8 = 0, SG_F32 = 1 } sg_dtype;
typedef enum { SG_L2 = 0, SG_IP = 1 } sg_metric;   /* squared L2 / negative inner product (R2) */

/* Operand precision of the distance GEMM; accumulation is always fp32 (R3). */
typedef enum {
    SG_PREC_AUTO = 0,       /* F16_EXACT when exact (u8, or integral f32 with the bound below), else TF32X3 */
    SG_PREC_F16_EXACT = 1,  /* kind::f16; exact when all values are integers |v| <= 2048 and 2*d*max^2 < 2^24 */
    SG_PREC_TF32 = 2,       /* kind::tf32, operands rounded to tf32 (RN) */
    SG_PREC_TF32X3 = 3      /* kind::tf32 on [hi|hi|lo].[hi|lo|hi]: ~fp32-accurate products */
} sg_precision;

/* Alg. 1 inputs + the paper-gap decisions of readings R4-R9. */
typedef struct {
    uint32_t k;            /* clusters = shards */
    uint32_t omega;        /* max homes per vector incl. the primary */
    float epsilon;         /* selectivity eps, default 1.2 */
    uint32_t theta0_ppm;   /* base replica fraction theta0 in ppm (R4), default 400000 */
    float alpha;           /* tau_b = 1 + alpha/(1+b) (R5), default 1.0 */
    uint32_t block_size;   /* vectors per block, default 65536 */
    uint64_t capacity;     /* max vectors per cluster; 0 = derive ceil(1.15 ceil(n/(k(1-theta0)))) (R9) */
} sg_partition_params;

typedef struct {
    uint32_t L;               /* intermediate kNN degree, <= 256 */
    uint32_t R;               /* final out-degree, R <= L, R <= 128 */
    int32_t metric;           /* sg_metric */
    int32_t precision;        /* sg_precision */
    uint32_t prune_rule;      /* 0 = rule P (R10), 1 = relaxed */
    uint32_t protected_edges; /* h forward edges kept by reverse insertion; 0 = R/2 (R11) */
} sg_build_params;

int scalegann_abi_version(void);
const char* scalegann_last_error(void);

/* ---- a1: centroids (reading R0) ----------------------------
 * k-means++ seeding + Lloyd on the strided sample floor(i*n/S), S =
 * min(n, spc*k), seeds drawn from splitmix64(seed).  Writes k x d float32
 * centroids (device).  Not bit-exact with the oracle: accepted when its sample
 * distortion is <= 1.01 x the oracle's.  Requires k <= 64, d <= 1024. */
sg_status scalegann_kmeans_workspace(uint64_t n, uint32_t d, uint32_t k, uint32_t spc, size_t* bytes);
sg_status scalegann_kmeans(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, uint32_t k,
                           uint64_t seed, uint32_t max_iter, uint32_t spc, float* centroids,
                           void* ws, size_t ws_bytes, void* stream);

/* ---- a2-a3: overlapping balanced partition (Alg. 1) --
 * For every vector v: d^2(v,c) to all centroids in the fixed fp32 fmaf order of
 * R1, then block by block (block_size vectors in id order): primaries to
 * the nearest cluster with size < capacity, statistics/thresholds
 * (R4, R5), replicas per Algorithm 1 with checkSizeLimit = R7.  Bit-exact with
 * the oracle.
 *   x          n x d vectors (device)
 *   centroids  k x d float32 (device)
 *   home       out, n x omega uint32: [primary, replicas in placement order, SENTINEL...]
 *   primary_d  out, n float32: d^2(v, primary)
 *   counts_host out (host), 3*k uint64: sizes[k], primaries[k], replicas[k]; synchronises
 * Errors: SG_ERR_INVALID_ARG (k == 0 or > 64, omega == 0 or > k, eps <= 0,
 * theta0_ppm not in (0, 1e6), capacity*k < n, block_size == 0), SG_ERR_CAPACITY. */
sg_status scalegann_partition_workspace(uint64_t n, uint32_t d, const sg_partition_params* p, size_t* bytes);
sg_status scalegann_partition(const void* x, sg_dtype dtype, uint64_t n, uint32_t d,
                              const float* centroids, const sg_partition_params* p, uint32_t* home,
                              float* primary_d, uint64_t* counts_host, void* ws, size_t ws_bytes,
                              void* stream);

/* ---- a4: shard membership (R8) --------------------------------------------
 * idmap = ascending global ids v with `shard` in home[v] (m entries, caller
 * sized from counts_host).  inv (optional, n x omega, device): for each (v, h)
 * with home[v*omega+h] == shard, inv[v*omega+h] = local id of v in the shard;
 * other entries untouched.  m_host (optional) receives m and synchronises. */
sg_status scalegann_shard_idmap_workspace(uint64_t n, size_t* bytes);
sg_status scalegann_shard_idmap(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t shard,
                                uint32_t* idmap, uint32_t* inv, uint64_t* m_host, void* ws,
                                size_t ws_bytes, void* stream);

/* ---- entry points (reading R13) ---------------------------------------------
 * entry_host[s] = argmin over primaries of shard s of (primary_d, gid), or
 * SENTINEL; returns the global entry (largest shard's entry, ties to lower s)
 * in *global_entry_host.  Synchronises. */
sg_status scalegann_entry_points(const uint32_t* home, const float* primary_d, uint64_t n,
                                 uint32_t omega, uint32_t k, const uint64_t* sizes_host,
                                 uint32_t* entry_host, uint32_t* global_entry_host, void* ws,
                                 size_t ws_bytes, void* stream);

/* ---- a5: exact kNN (north_star stage 2; R2, R3) ---------------------------
 * For each row i of A (rows ida[0..ma) of xa, or 0..ma-1 if ida == NULL): the L
 * smallest (dist, j) over rows j of B (idb / xb likewise), j != i when
 * self_exclude (A and B the same set).  dist = |a|^2 + |b|^2 - 2 a.b (L2) or
 * -a.b (IP), distance tiles on tcgen05 tensor cores with fp32 accumulation and
 * a fused per-row top-L.  ids/dists out: ma x L, rows sorted by (dist, id),
 * padded with (SENTINEL, +inf) when fewer than L candidates exist.
 * Limits: L <= 256; ma, mb < 2^31; up to 128 operand atoms of 128 bytes per row
 * (d <= 8176 F16_EXACT, 4088 TF32, 1362 TF32X3).  Rows up to 4 atoms (d <= 248
 * F16_EXACT with L2) keep the CTA's row block resident in shared memory; wider rows
 * stream both operands through the ring (slower per flop, same results). */
sg_status scalegann_knn_workspace(uint64_t ma, uint64_t mb, uint32_t d, sg_dtype dtype, uint32_t L,
                                  int32_t precision, size_t* bytes);
sg_status scalegann_knn(const void* xa, const uint32_t* ida, uint64_t ma, const void* xb,
                        const uint32_t* idb, uint64_t mb, sg_dtype dtype, uint32_t d, int self_exclude,
                        uint32_t L, int32_t metric, int32_t precision, uint32_t* ids, float* dists,
                        void* ws, size_t ws_bytes, void* stream);

/* ---- a6: rank-based detour-count prune (reading R10) ------------------------
 * knn m x L (local ids, rows sorted by (dist,id)) -> out m x R: the first R
 * ranks in the stable order by (detour count, rank), sentinel ranks last;
 * out_d carries the kNN distances.  Bit-exact with the oracle. L <= 256. */
sg_status scalegann_prune(const uint32_t* knn_ids, const float* knn_d, uint64_t m, uint32_t L,
                          uint32_t R, uint32_t rule, uint32_t* out, float* out_d, void* stream);

/* ---- a7: reverse-edge insertion (reading R11) -------------------------------
 * pruned m x R -> out m x R = pruned[y][0..h) ++ first R-h of
 * (rev_np ++ remaining forward), rev ordered by (rank, source) and capped at R.
 * Bit-exact with the oracle.  R <= 128. */
sg_status scalegann_reverse_workspace(uint64_t m, uint32_t R, size_t* bytes);
sg_status scalegann_reverse(const uint32_t* pruned, const float* pruned_d, uint64_t m, uint32_t R,
                            uint32_t h, uint32_t* out, float* out_d, void* ws, size_t ws_bytes,
                            void* stream);

/* ---- a4-a7: one shard build ("invokes a GPU-based indexing algorithm") --
 * gather rows idmap[0..m) of x, exact kNN (a5), prune (a6), reverse (a7).
 * knn_ids/knn_d (m x L) may be NULL (then kept in ws).  graph/graph_d m x R
 * local ids.  Errors: SG_ERR_TOO_SMALL when m < 2. */
sg_status scalegann_build_shard_workspace(uint64_t m, uint32_t d, sg_dtype dtype,
                                          const sg_build_params* p, size_t* bytes);
sg_status scalegann_build_shard(const void* x, sg_dtype dtype, uint64_t n, uint32_t d,
                                const uint32_t* idmap, uint64_t m, const sg_build_params* p,
                                uint32_t* knn_ids, float* knn_d, uint32_t* graph, float* graph_d,
                                void* ws, size_t ws_bytes, void* stream);
/* prune + reverse only: the parity entry point fed with an external kNN */
sg_status scalegann_optimize_from_knn(const uint32_t* knn_ids, const float* knn_d, uint64_t m,
                                      const sg_build_params* p, uint32_t* graph, float* graph_d,
                                      void* ws, size_t ws_bytes, void* stream);

/* ---- N1 / N2: the library's NCCL communicator ----------
 * One rank per GPU.  Rank 0 creates a 128-byte unique id, the caller shares it with every rank
 * out of band (file, MPI, torch.distributed, ...), and every rank calls scalegann_comm_init on
 * its own device.  comm == NULL everywhere below means world = 1.  The communicator is the only
 * resource the library owns; scalegann_comm_destroy releases it.  NCCL failures return
 * SG_ERR_NCCL. */
sg_status scalegann_get_unique_id(uint8_t out[128]);
sg_status scalegann_comm_init(int rank, int world, const uint8_t uid[128], void** comm);
sg_status scalegann_comm_destroy(void* comm);
sg_status scalegann_comm_rank(void* comm, int* rank, int* world);
/* N1: rank 0's k x d float32 centroids (device) to every rank, in place (ncclBroadcast). */
sg_status scalegann_broadcast_centroids(void* comm, float* centroids, uint32_t k, uint32_t d, void* stream);
/* N2: per-peer ncclSend/ncclRecv of merge records (`words` uint32 each) in one NCCL group.
 * sendbuf holds this rank's records grouped by destination rank in rank order (send_host[r]
 * records for rank r; those for this rank are skipped); recvbuf receives recv_host[r] records
 * from each rank r, grouped by source in rank order. */
sg_status scalegann_exchange_records(void* comm, const uint32_t* sendbuf, const uint64_t* send_host,
                                     uint32_t* recvbuf, const uint64_t* recv_host, uint32_t words, void* stream);

/* ---- a8: cross-shard merge by edge union + re-prune (R12) --------------------
 * The merged row of a global vector g is kept by the rank that owns g's primary shard
 * (home[g][0]): merged / merged_d hold n_owned x R rows of these g in ascending order
 * (owned_index[g] = its row, SENTINEL for rows owned elsewhere).  Rows of vectors with one home
 * are the shard row mapped to global ids as is; rows of vectors with several homes are the
 * first R of the union of the homes' rows by (dist, gid), deduplicated by gid keeping the
 * minimum carried distance, padded with (SENTINEL, +inf).  Bit-exact with the oracle.
 *
 * Streaming protocol (a shard's graph can be freed as soon as it has been merged):
 *   1. scalegann_merge_plan: owned_index (n), send slots rec_slot (n x omega), per-rank record
 *      counts send_host / recv_host (world each) and n_owned_host; synchronises;
 *   2. scalegann_merge_init: merged rows to (SENTINEL, +inf);
 *   3. scalegann_merge_shard for every shard built on this rank (graph: m x R local ids, idmap:
 *      the shard's ascending global ids): rows whose primary is owned here are folded into
 *      merged; the others become records [g, h, R global ids, R dist bits] in sendbuf
 *      (2 + 2R uint32 each), grouped by destination rank, ascending g within a destination;
 *   4. scalegann_exchange_records (N2);
 *   5. scalegann_merge_finish: the received records folded in (ws >= 256 bytes); synchronises.
 * owner_host: k ranks (shard s built on rank owner_host[s]); all ranks use the same home.
 * Limits: k <= 64, world <= 64, R <= 128, n < 2^32 - 1. */
sg_status scalegann_merge_plan_workspace(uint64_t n, size_t* bytes);
sg_status scalegann_merge_plan(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k,
                               const int32_t* owner_host, int rank, int world, uint32_t* owned_index,
                               uint32_t* rec_slot, uint64_t* send_host, uint64_t* recv_host,
                               uint64_t* n_owned_host, void* ws, size_t ws_bytes, void* stream);
sg_status scalegann_merge_init(uint64_t n_owned, uint32_t R, uint32_t* merged, float* merged_d, void* stream);
sg_status scalegann_merge_shard(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k,
                                const int32_t* owner_host, int rank, int world, uint32_t shard,
                                const uint32_t* idmap, uint64_t m, const uint32_t* graph,
                                const float* graph_d, uint32_t R, const uint32_t* owned_index,
                                const uint32_t* rec_slot, uint32_t* merged, float* merged_d,
                                uint32_t* sendbuf, void* stream);
sg_status scalegann_merge_finish(uint32_t omega, uint32_t R, const uint32_t* owned_index,
                                 const uint32_t* recvbuf, uint64_t n_recv, uint32_t* merged,
                                 float* merged_d, void* ws, size_t ws_bytes, void* stream);
/* Collective one-call merge of every shard built on this rank (all ranks call it; steps 1-5 in
 * the library, N2 over the communicator).  idmaps / graphs / graphs_d: HOST arrays of k DEVICE
 * pointers (NULL for shards built elsewhere); sizes_host: k shard sizes.  The workspace query
 * counts the records (synchronises) and returns n_owned (the rows of merged). */
sg_status scalegann_merge_workspace(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k,
                                    const int32_t* owner_host, void* comm, uint32_t R, size_t* bytes,
                                    uint64_t* n_owned_host, void* stream);
sg_status scalegann_merge(void* comm, const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k,
                          const int32_t* owner_host, const uint32_t* const* idmaps,
                          const uint64_t* sizes_host, const uint32_t* const* graphs,
                          const float* const* graphs_d, uint32_t R, uint32_t* merged, float* merged_d,
                          uint64_t* n_owned_host, void* ws, size_t ws_bytes, void* stream);

/* ---- a1-a8 in one call, HOST buffers (the e2e path) --------------------------------
 * x_host: n x d vectors in host memory (pinned for full copy speed).  Copies x to the device, runs
 * k-means (rank 0, seed kmeans_seed, 15 Lloyd steps, 256 samples per cluster) + N1, the
 * partition (pp), every shard LPT-placed on this rank (bp; built, folded into the owner rows and
 * reused), N2 and the final fold, then copies this rank's merged rows (ascending gid) to
 * merged_host (capacity n x R; the first *n_owned_host rows are written) and their distances to
 * merged_d_host (optional).  entry_host (optional) receives the global entry point (R13).
 * comm: the communicator (NULL = world 1); collective over its ranks.  Synchronises.  Unlike the
 * rest of the ABI this call allocates its device temporaries itself (stream-ordered, released
 * before it returns). */
sg_status scalegann_build_index_host(void* comm, const void* x_host, sg_dtype dtype, uint64_t n, uint32_t d,
                                     const sg_partition_params* pp, const sg_build_params* bp,
                                     uint64_t kmeans_seed, uint32_t* merged_host, float* merged_d_host,
                                     uint64_t* n_owned_host, uint32_t* entry_host, void* stream);

/* ---- a9: recall evaluation (reading R14) ------------------
 * Greedy best-first beam search from `entry` over graph (n x R global ids) for
 * nq queries (nq x d, same dtype as x); out_ids nq x topk.  Distances are P8's
 * exact ones (u8: integer; f32: fp64 sum of the squared differences, one
 * rounding to f32), so result lists equal the oracle's.  gt (nq x topk, device)
 * may be NULL, then it is computed exactly with scalegann_knn and written to
 * gt_out (if not NULL).  recall_host = |ret & gt| / (nq*topk); n_dist_host
 * (may be NULL) = distance computations over all queries (P:515-516's proxy of
 * search work); both synchronise.  beam <= 512, topk <= beam, R <= 128.  The
 * visited set is a bitmap of n bits per query, or a hash set of 8 x beam x R
 * ids when that is smaller; a hash set that fills up returns SG_ERR_WORKSPACE. */
sg_status scalegann_search_workspace(uint64_t n, uint32_t d, sg_dtype dtype, uint32_t nq, uint32_t topk,
                                     uint32_t beam, size_t* bytes);
sg_status scalegann_search_eval(const void* x, sg_dtype dtype, uint64_t n, uint32_t d,
                                const uint32_t* graph, uint32_t R, uint32_t entry, const void* queries,
                                uint32_t nq, uint32_t topk, uint32_t beam, int32_t metric,
                                const uint32_t* gt, uint32_t* gt_out, uint32_t* out_ids,
                                double* recall_host, uint64_t* n_dist_host, void* ws, size_t ws_bytes,
                                void* stream);

/* ---- a9, split-only mode: per-shard search + result merge (§8(f) NEXT-2;
 * reading R15) ------------------------------------------------------------------
 * The same beam search as scalegann_search_eval, run once from each of the n_entries entry
 * points (entries_host, host, e.g. every shard's entry from scalegann_entry_points), each
 * keeping its own beam; the per-entry top-topk lists are merged into the topk smallest
 * distinct (dist, id).  For a split-only graph (omega = 1, disjoint shards) this is "search
 * every shard and merge the results".  SENTINEL entries (empty shards) are skipped.  Errors as
 * scalegann_search_eval, plus SG_ERR_INVALID_ARG for n_entries outside [1, 1024], an entry >= n
 * that is not SENTINEL, or no real entry.  Synchronises when recall_host or n_dist_host is set. */
sg_status scalegann_search_shards_workspace(uint64_t n, uint32_t d, sg_dtype dtype, uint32_t nq, uint32_t topk,
                                            uint32_t beam, uint32_t n_entries, size_t* bytes);
sg_status scalegann_search_eval_shards(const void* x, sg_dtype dtype, uint64_t n, uint32_t d,
                                       const uint32_t* graph, uint32_t R, const uint32_t* entries_host,
                                       uint32_t n_entries, const void* queries, uint32_t nq, uint32_t topk,
                                       uint32_t beam, int32_t metric, const uint32_t* gt, uint32_t* gt_out,
                                       uint32_t* out_ids, double* recall_host, uint64_t* n_dist_host,
                                       void* ws, size_t ws_bytes, void* stream);

/* ---- diagnostics ------------------------------------------------------------
 * Raw distance-tile probe of the tcgen05 GEMM core (validation of the MMA
 * pipeline against a reference matmul): out[i][j] = a_i . b_j in fp32 for
 * 0 <= i < ma, 0 <= j < mb (operands converted as for `precision`). */
sg_status scalegann_gemm_probe(const void* xa, uint64_t ma, const void* xb, uint64_t mb, sg_dtype dtype,
                               uint32_t d, int32_t precision, float* out, void* ws, size_t ws_bytes,
                               void* stream);

/* Kernel accounting for the benchmark: every kernel launch of this library increments a
 * counter; with stats enabled, CUDA events are recorded on the launching stream around each
 * distance-kernel launch (a5).  scalegann_stats_read synchronises those events and returns
 * the summed device time, the number of distance launches and of all launches since the last
 * reset. */
sg_status scalegann_stats_enable(int on);
/* Diagnostics: when dev_counters (device, 80 x uint64, zeroed by the caller) is not NULL, every
 * later distance-kernel launch adds per-warp clock64 cycle counts to it: [warp*8 + i] with
 * i = 0 barrier waits, 1 TMEM load / full-barrier wait, 2 compaction, 3 pass masks,
 * 4 insertions, 5 final merge.  NULL disables. */
sg_status scalegann_knn_profile(unsigned long long* dev_counters);
sg_status scalegann_stats_read(double* knn_ms, uint64_t* knn_launches, uint64_t* kernel_launches, int reset);

#ifdef __cplusplus
}
#endif
#endif /* SCALEGANN_H */
