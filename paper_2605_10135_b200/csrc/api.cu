// extern "C" entry points of libscalegann.so (include/scalegann.h): argument validation,
// workspace carving and dispatch to the stage kernels.  No torch, no host fallback: every
// step of the path runs in this library's kernels.
#include <stdarg.h>

#include <utility>
#include <vector>

#include "common.cuh"

namespace sg {
// stage entry points implemented in the per-stage translation units
size_t kmeans_ws(uint64_t n, uint32_t d, uint32_t k, uint32_t spc);
sg_status kmeans_run(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, uint32_t k, uint64_t seed,
                     uint32_t max_iter, uint32_t spc, float* C, void* ws, size_t ws_bytes, cudaStream_t st);
size_t partition_ws(uint64_t n, uint32_t k);
sg_status partition_run(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const float* C,
                        const sg_partition_params* p, uint32_t* home, float* primary_d, uint64_t* counts_host,
                        void* ws, size_t ws_bytes, cudaStream_t st);
size_t idmap_ws(uint64_t n);
sg_status idmap_run(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t s, uint32_t* idmap, uint32_t* inv,
                    uint64_t* m_host, void* ws, size_t ws_bytes, cudaStream_t st);
sg_status entry_run(const uint32_t* home, const float* pd, uint64_t n, uint32_t omega, uint32_t k,
                    const uint64_t* sizes_host, uint32_t* entry_host, uint32_t* global_host, void* ws,
                    size_t ws_bytes, cudaStream_t st);
size_t reverse_ws(uint64_t m, uint32_t R);
size_t merge_plan_ws(uint64_t n);
sg_status merge_plan_run(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k, const int32_t* owner, int rank,
                         int world, uint32_t* owned_index, uint32_t* rec_slot, uint64_t* send_host, uint64_t* recv_host,
                         uint64_t* n_owned_host, void* ws, size_t ws_bytes, cudaStream_t st);
sg_status merge_init_run(uint64_t n_owned, uint32_t R, uint32_t* merged, float* merged_d, cudaStream_t st);
sg_status merge_shard_run(const uint32_t* home, uint32_t omega, uint32_t k, const int32_t* owner, int rank, int world,
                          uint32_t shard, const uint32_t* idmap, uint64_t m, const uint32_t* graph, const float* graph_d,
                          uint32_t R, const uint32_t* owned_index, const uint32_t* rec_slot, uint32_t* merged,
                          float* merged_d, uint32_t* sendbuf, cudaStream_t st);
sg_status merge_finish_run(uint32_t omega, uint32_t R, const uint32_t* owned_index, const uint32_t* recvbuf,
                           uint64_t n_recv, uint32_t* merged, float* merged_d, int* err_dev, cudaStream_t st);
sg_status comm_rank_world(void* comm, int* rank, int* world);
sg_status exchange_records_run(void* comm, const uint32_t* sendbuf, const uint64_t* send_host, uint32_t* recvbuf,
                               const uint64_t* recv_host, uint32_t words, cudaStream_t st);
size_t beam_ws(uint64_t n, uint32_t nq, uint32_t beam, uint32_t R);
sg_status beam_run(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const uint32_t* graph, uint32_t R,
                   uint32_t entry, const void* q, uint32_t nq, uint32_t topk, uint32_t beam, int metric,
                   uint32_t* out_ids, unsigned long long* ndist, Carver& cv, cudaStream_t st,
                   uint64_t* out_keys = nullptr);
sg_status shard_merge_run(const uint64_t* keys, uint32_t ns, uint32_t nq, uint32_t topk, uint32_t* out_ids,
                          cudaStream_t st);
sg_status recall_run(const uint32_t* ret, const uint32_t* gt, uint32_t nq, uint32_t topk, double* recall_host,
                     Carver& cv, cudaStream_t st);

void set_knn_profile(unsigned long long* buf);
static thread_local char g_err[512] = "";

// ---- diagnostics: launch counter + event timing of the distance kernel
struct Stats {
    bool on = false;
    uint64_t launches = 0, knn_launches = 0;
    cudaEvent_t pending_begin = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> knn;
};
static Stats g_stats;

void note_launch() { g_stats.launches++; }

void knn_time_begin(cudaStream_t st) {
    g_stats.knn_launches++;
    if (!g_stats.on) return;
    cudaEventCreate(&g_stats.pending_begin);
    cudaEventRecord(g_stats.pending_begin, st);
}

void knn_time_end(cudaStream_t st) {
    if (!g_stats.on || !g_stats.pending_begin) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    g_stats.knn.emplace_back(g_stats.pending_begin, e);
    g_stats.pending_begin = nullptr;
}

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

sg_status cuda_status(cudaError_t e, const char* what) {
    set_error("CUDA error %s (%d) in %s", cudaGetErrorString(e), (int)e, what);
    return SG_ERR_CUDA;
}

static uint32_t knn_full_atoms(int prec, int metric, uint32_t d) {
    uint32_t kdim, nfull, mini;
    operand_layout(prec, metric, d, &kdim, &nfull, &mini);
    return nfull;
}

// workspace of a kNN between ma rows and mb rows (both gathered); `same` = self-join
static size_t knn_total_ws(uint64_t ma, uint64_t mb, uint32_t d, int prec, uint32_t L, bool same) {
    size_t b = same ? operand_bytes(prec, SG_L2, d, ma, SIDE_A | SIDE_B)
                    : operand_bytes(prec, SG_L2, d, ma, SIDE_A) + operand_bytes(prec, SG_L2, d, mb, SIDE_B);
    return b + knn_core_workspace(L, ma, d, prec, SG_L2) + 2 * (ma * 4 + 256) + (same ? order_workspace(ma, d, prec, SG_L2) : 0) + 4096;
}

static int worst_prec(sg_dtype dtype, int32_t precision, uint32_t d) {
    // AUTO resolves at run time; size the workspace for the widest candidate.  u8 data is
    // F16_EXACT whenever 2 d 255^2 < 2^24 (gather.cu resolves it without looking at the data)
    if (precision != SG_PREC_AUTO) return precision;
    if (dtype == SG_U8 && 2ull * d * 255 * 255 < (1ull << 24)) return SG_PREC_F16_EXACT;
    return dtype == SG_U8 ? SG_PREC_TF32 : SG_PREC_TF32X3;
}

static sg_status check_knn_shape(int prec, int metric, uint32_t d, uint32_t L) {
    SG_CHECK_ARG(L >= 1 && L <= 256, "kNN: L must be in [1, 256]");
    const uint32_t nf = knn_full_atoms(prec, metric, d);
    if (nf > 128) {   // > 4 atoms: streamed-A kernel (knn_tc.cu); the bound only caps d
        set_error("kNN: d=%u needs %u 128-byte operand atoms per row with this precision (max 128)", d, nf);
        return SG_ERR_UNSUPPORTED;
    }
    return SG_OK;
}

}  // namespace sg

using namespace sg;

extern "C" {

int scalegann_abi_version(void) { return SCALEGANN_ABI_VERSION; }
const char* scalegann_last_error(void) { return g_err; }

sg_status scalegann_knn_profile(unsigned long long* dev_counters) {
    set_knn_profile(dev_counters);
    return SG_OK;
}

sg_status scalegann_stats_enable(int on) {
    g_stats.on = on != 0;
    return SG_OK;
}

sg_status scalegann_stats_read(double* knn_ms, uint64_t* knn_launches, uint64_t* kernel_launches, int reset) {
    double ms = 0;
    for (auto& pr : g_stats.knn) {
        float t = 0;
        SG_CUDA(cudaEventSynchronize(pr.second));
        SG_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second));
        ms += t;
    }
    if (knn_ms) *knn_ms = ms;
    if (knn_launches) *knn_launches = g_stats.knn_launches;
    if (kernel_launches) *kernel_launches = g_stats.launches;
    if (reset) {
        for (auto& pr : g_stats.knn) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
        g_stats.knn.clear();
        g_stats.knn_launches = 0;
        g_stats.launches = 0;
    }
    return SG_OK;
}

// ------------------------------------------------------------------ a1
sg_status scalegann_kmeans_workspace(uint64_t n, uint32_t d, uint32_t k, uint32_t spc, size_t* bytes) {
    SG_CHECK_ARG(bytes, "null bytes");
    *bytes = kmeans_ws(n, d, k, spc);
    return SG_OK;
}
sg_status scalegann_kmeans(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, uint32_t k, uint64_t seed,
                           uint32_t max_iter, uint32_t spc, float* centroids, void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(x && centroids && n > 0 && d > 0 && d <= 1024 && k >= 1 && k <= 64 && spc >= 1,
                 "kmeans: bad arguments (n>0, 0<d<=1024, 1<=k<=64)");
    SG_CHECK_ARG(dtype == SG_U8 || dtype == SG_F32, "kmeans: bad dtype");
    return kmeans_run(x, dtype, n, d, k, seed, max_iter, spc, centroids, ws, ws_bytes, S(stream));
}

// ------------------------------------------------------------------ a2-a3
sg_status scalegann_partition_workspace(uint64_t n, uint32_t d, const sg_partition_params* p, size_t* bytes) {
    SG_CHECK_ARG(p && bytes, "null argument");
    (void)d;
    *bytes = partition_ws(n, p->k);
    return SG_OK;
}
sg_status scalegann_partition(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const float* centroids,
                              const sg_partition_params* p, uint32_t* home, float* primary_d, uint64_t* counts_host,
                              void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(x && centroids && p && home && primary_d, "partition: null pointer");
    SG_CHECK_ARG(n > 0 && n < 0xFFFFFFFFull && d > 0, "partition: need 0 < n < 2^32-1, d > 0");
    SG_CHECK_ARG(dtype == SG_U8 || dtype == SG_F32, "partition: bad dtype");
    SG_CHECK_ARG(p->k >= 1 && p->k <= 64, "partition: k must be in [1, 64]");
    SG_CHECK_ARG(p->omega >= 1 && p->omega <= p->k, "partition: omega must be in [1, k]");
    SG_CHECK_ARG(p->epsilon > 0.f, "partition: epsilon must be > 0");
    SG_CHECK_ARG(p->theta0_ppm > 0 && p->theta0_ppm < 1000000, "partition: theta0_ppm must be in (0, 1e6)");
    SG_CHECK_ARG(p->block_size >= 1 && p->block_size <= (1u << 24), "partition: block_size in [1, 2^24]");
    return partition_run(x, dtype, n, d, centroids, p, home, primary_d, counts_host, ws, ws_bytes, S(stream));
}

// ------------------------------------------------------------------ a4
sg_status scalegann_shard_idmap_workspace(uint64_t n, size_t* bytes) {
    SG_CHECK_ARG(bytes, "null bytes");
    *bytes = idmap_ws(n);
    return SG_OK;
}
sg_status scalegann_shard_idmap(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t shard, uint32_t* idmap,
                                uint32_t* inv, uint64_t* m_host, void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(home && n > 0 && omega >= 1, "idmap: bad arguments");
    return idmap_run(home, n, omega, shard, idmap, inv, m_host, ws, ws_bytes, S(stream));
}

sg_status scalegann_entry_points(const uint32_t* home, const float* primary_d, uint64_t n, uint32_t omega, uint32_t k,
                                 const uint64_t* sizes_host, uint32_t* entry_host, uint32_t* global_entry_host,
                                 void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(home && primary_d && sizes_host && entry_host && k >= 1 && k <= 64, "entry_points: bad arguments");
    return entry_run(home, primary_d, n, omega, k, sizes_host, entry_host, global_entry_host, ws, ws_bytes, S(stream));
}

// ------------------------------------------------------------------ a5
sg_status scalegann_knn_workspace(uint64_t ma, uint64_t mb, uint32_t d, sg_dtype dtype, uint32_t L, int32_t precision,
                                  size_t* bytes) {
    SG_CHECK_ARG(bytes, "null bytes");
    const int pr = worst_prec(dtype, precision, d);
    *bytes = knn_total_ws(ma, mb, d, pr, L, false) + (ma == mb ? order_workspace(ma, d, pr, SG_L2) : 0);
    return SG_OK;
}

static sg_status knn_impl(const void* xa, const uint32_t* ida, uint64_t ma, const void* xb, const uint32_t* idb,
                          uint64_t mb, sg_dtype dtype, uint32_t d, int self_exclude, uint32_t L, int32_t metric,
                          int32_t precision, uint32_t* ids, float* dists, float* probe, void* ws, size_t ws_bytes,
                          cudaStream_t st) {
    SG_CHECK_ARG(xa && xb && (ids || probe) && (dists || probe), "kNN: null pointer");
    SG_CHECK_ARG(ma > 0 && mb > 0 && ma < (1ull << 31) && mb < (1ull << 31) && d > 0, "kNN: bad sizes");
    SG_CHECK_ARG(dtype == SG_U8 || dtype == SG_F32, "kNN: bad dtype");
    SG_CHECK_ARG(metric == SG_L2 || metric == SG_IP, "kNN: bad metric");
    SG_CHECK_ARG(precision >= SG_PREC_AUTO && precision <= SG_PREC_TF32X3, "kNN: bad precision");
    Carver cv(ws, ws_bytes);
    unsigned* flags = cv.take<unsigned>(2);
    if (!cv.ok()) { set_error("kNN: workspace too small"); return SG_ERR_WORKSPACE; }
    sg_status e;
    const int prec = resolve_precision(precision, dtype, d, xa, ida, ma, xb, idb, mb, flags, st, &e);
    if (e != SG_OK) return e;
    SG_TRY(check_knn_shape(prec, metric, d, L));
    const bool same = xa == xb && ida == idb && ma == mb;
    Operand A, B;
    if (same && self_exclude && !probe && order_groups(ma) >= 2) {
        // self-join: spatially ordered operand (order.cu), results mapped back to input order
        uint32_t* perm = cv.take<uint32_t>(ma);
        uint32_t* ids_perm = cv.take<uint32_t>(ma);
        if (!cv.ok()) { set_error("kNN: workspace too small"); return SG_ERR_WORKSPACE; }
        SG_TRY(spatial_order(xa, dtype, d, ida, ma, prec, metric, perm, ids_perm, cv, st));
        SG_TRY(gather_operand(xa, dtype, d, ids_perm, ma, prec, metric, SIDE_A | SIDE_B, cv, &A, st));
        return knn_core(A, A, metric, true, L, ids, dists, nullptr, cv, st, perm, perm, true);
    }
    SG_TRY(gather_operand(xa, dtype, d, ida, ma, prec, metric, same ? (SIDE_A | SIDE_B) : SIDE_A, cv, &A, st));
    if (same) B = A;
    else SG_TRY(gather_operand(xb, dtype, d, idb, mb, prec, metric, SIDE_B, cv, &B, st));
    if (prec == SG_PREC_TF32X3 && !same) {
        // A side uses [hi|hi|lo]; B side uses [hi|lo|hi]: A.a and B.b are already those layouts
    }
    return knn_core(A, B, metric, self_exclude != 0, L, ids, dists, probe, cv, st);
}

sg_status scalegann_knn(const void* xa, const uint32_t* ida, uint64_t ma, const void* xb, const uint32_t* idb,
                        uint64_t mb, sg_dtype dtype, uint32_t d, int self_exclude, uint32_t L, int32_t metric,
                        int32_t precision, uint32_t* ids, float* dists, void* ws, size_t ws_bytes, void* stream) {
    return knn_impl(xa, ida, ma, xb, idb, mb, dtype, d, self_exclude, L, metric, precision, ids, dists, nullptr, ws,
                    ws_bytes, S(stream));
}

sg_status scalegann_gemm_probe(const void* xa, uint64_t ma, const void* xb, uint64_t mb, sg_dtype dtype, uint32_t d,
                               int32_t precision, float* out, void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(out, "probe: null out");
    return knn_impl(xa, nullptr, ma, xb, nullptr, mb, dtype, d, 0, 1, SG_L2, precision, nullptr, nullptr, out, ws,
                    ws_bytes, S(stream));
}

// ------------------------------------------------------------------ a6 / a7
sg_status scalegann_prune(const uint32_t* knn_ids, const float* knn_d, uint64_t m, uint32_t L, uint32_t R, uint32_t rule,
                          uint32_t* out, float* out_d, void* stream) {
    SG_CHECK_ARG(knn_ids && knn_d && out && out_d, "prune: null pointer");
    SG_CHECK_ARG(L >= 1 && L <= 256 && R >= 1 && R <= L && rule <= 1, "prune: need 1 <= R <= L <= 256, rule in {0,1}");
    return launch_prune(knn_ids, knn_d, m, L, R, rule, out, out_d, S(stream));
}

sg_status scalegann_reverse_workspace(uint64_t m, uint32_t R, size_t* bytes) {
    SG_CHECK_ARG(bytes, "null bytes");
    *bytes = reverse_ws(m, R);
    return SG_OK;
}
sg_status scalegann_reverse(const uint32_t* pruned, const float* pruned_d, uint64_t m, uint32_t R, uint32_t h,
                            uint32_t* out, float* out_d, void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(pruned && pruned_d && out && out_d, "reverse: null pointer");
    SG_CHECK_ARG(R >= 1 && R <= 128 && h <= R, "reverse: need 1 <= R <= 128, h <= R");
    Carver cv(ws, ws_bytes);
    return launch_reverse(pruned, pruned_d, m, R, h, out, out_d, cv, S(stream));
}

// ------------------------------------------------------------------ a4-a7
static size_t build_ws(uint64_t m, uint32_t d, sg_dtype dtype, const sg_build_params* p) {
    const int prec = worst_prec(dtype, p->precision, d);
    size_t b = 1024;
    b += 2 * (m * p->L * 4 + 256);     // kNN ids + dists (when not caller-provided)
    b += 2 * (m * p->R * 4 + 256);     // pruned ids + dists
    size_t knn = 2 * (m * 4 + 256) + operand_bytes(prec, p->metric, d, m, SIDE_A | SIDE_B) + knn_core_workspace(p->L, m, d, prec, p->metric) +
                 order_workspace(m, d, prec, p->metric) + 1024;
    size_t rev = reverse_ws(m, p->R);
    return b + (knn > rev ? knn : rev);
}

sg_status scalegann_build_shard_workspace(uint64_t m, uint32_t d, sg_dtype dtype, const sg_build_params* p,
                                          size_t* bytes) {
    SG_CHECK_ARG(p && bytes, "null argument");
    *bytes = build_ws(m, d, dtype, p);
    return SG_OK;
}

static sg_status check_build(const sg_build_params* p, uint64_t m) {
    SG_CHECK_ARG(p, "build: null params");
    SG_CHECK_ARG(p->L >= 1 && p->L <= 256 && p->R >= 1 && p->R <= p->L && p->R <= 128,
                 "build: need 1 <= R <= L <= 256, R <= 128");
    SG_CHECK_ARG(p->metric == SG_L2 || p->metric == SG_IP, "build: bad metric");
    SG_CHECK_ARG(p->prune_rule <= 1 && p->protected_edges <= p->R, "build: bad prune_rule/protected_edges");
    if (m < 2) { set_error("build: shard has m < 2 vectors (S:301)"); return SG_ERR_TOO_SMALL; }
    SG_CHECK_ARG(m < (1ull << 31), "build: m must be < 2^31");
    return SG_OK;
}

sg_status scalegann_optimize_from_knn(const uint32_t* knn_ids, const float* knn_d, uint64_t m, const sg_build_params* p,
                                      uint32_t* graph, float* graph_d, void* ws, size_t ws_bytes, void* stream) {
    SG_TRY(check_build(p, m));
    SG_CHECK_ARG(knn_ids && knn_d && graph && graph_d, "optimize: null pointer");
    Carver cv(ws, ws_bytes);
    uint32_t* pr = cv.take<uint32_t>(m * p->R);
    float* prd = cv.take<float>(m * p->R);
    if (!cv.ok()) { set_error("optimize: workspace too small"); return SG_ERR_WORKSPACE; }
    cudaStream_t st = S(stream);
    SG_TRY(launch_prune(knn_ids, knn_d, m, p->L, p->R, p->prune_rule, pr, prd, st));
    const uint32_t h = p->protected_edges ? p->protected_edges : p->R / 2;
    return launch_reverse(pr, prd, m, p->R, h, graph, graph_d, cv, st);
}

sg_status scalegann_build_shard(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const uint32_t* idmap,
                                uint64_t m, const sg_build_params* p, uint32_t* knn_ids, float* knn_d, uint32_t* graph,
                                float* graph_d, void* ws, size_t ws_bytes, void* stream) {
    SG_TRY(check_build(p, m));
    SG_CHECK_ARG(x && idmap && graph && graph_d && n > 0 && d > 0, "build: null pointer or empty input");
    SG_CHECK_ARG(dtype == SG_U8 || dtype == SG_F32, "build: bad dtype");
    cudaStream_t st = S(stream);
    Carver cv(ws, ws_bytes);
    unsigned* flags = cv.take<unsigned>(2);
    uint32_t* kid = knn_ids ? knn_ids : cv.take<uint32_t>(m * p->L);
    float* kd = knn_d ? knn_d : cv.take<float>(m * p->L);
    uint32_t* pr = cv.take<uint32_t>(m * p->R);
    float* prd = cv.take<float>(m * p->R);
    if (!cv.ok()) { set_error("build: workspace too small"); return SG_ERR_WORKSPACE; }
    sg_status e;
    const int prec = resolve_precision(p->precision, dtype, d, x, idmap, m, nullptr, nullptr, 0, flags, st, &e);
    if (e != SG_OK) return e;
    SG_TRY(check_knn_shape(prec, p->metric, d, p->L));
    {
        // a4 gather in spatial order (order.cu) + a5 exact kNN; the scratch is reused by a6/a7
        Carver kc = cv;
        uint32_t* perm = kc.take<uint32_t>(m);
        uint32_t* ids_perm = kc.take<uint32_t>(m);
        if (!kc.ok()) { set_error("build: workspace too small"); return SG_ERR_WORKSPACE; }
        const bool ordered = order_groups(m) >= 2;
        if (ordered) SG_TRY(spatial_order(x, dtype, d, idmap, m, prec, p->metric, perm, ids_perm, kc, st));
        Operand A;
        SG_TRY(gather_operand(x, dtype, d, ordered ? ids_perm : idmap, m, prec, p->metric, SIDE_A | SIDE_B, kc, &A,
                              st));
        SG_TRY(knn_core(A, A, p->metric, true, p->L, kid, kd, nullptr, kc, st, ordered ? perm : nullptr,
                        ordered ? perm : nullptr, ordered));
    }
    SG_TRY(launch_prune(kid, kd, m, p->L, p->R, p->prune_rule, pr, prd, st));
    const uint32_t h = p->protected_edges ? p->protected_edges : p->R / 2;
    return launch_reverse(pr, prd, m, p->R, h, graph, graph_d, cv, st);
}

// ------------------------------------------------------------------ a8
sg_status scalegann_merge_plan_workspace(uint64_t n, size_t* bytes) {
    SG_CHECK_ARG(bytes, "null bytes");
    *bytes = merge_plan_ws(n);
    return SG_OK;
}
sg_status scalegann_merge_plan(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k, const int32_t* owner_host,
                               int rank, int world, uint32_t* owned_index, uint32_t* rec_slot, uint64_t* send_host,
                               uint64_t* recv_host, uint64_t* n_owned_host, void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(home && owner_host && omega >= 1 && n > 0 && n < 0xFFFFFFFFull, "merge_plan: bad arguments");
    return merge_plan_run(home, n, omega, k, owner_host, rank, world, owned_index, rec_slot, send_host, recv_host,
                          n_owned_host, ws, ws_bytes, S(stream));
}
sg_status scalegann_merge_init(uint64_t n_owned, uint32_t R, uint32_t* merged, float* merged_d, void* stream) {
    SG_CHECK_ARG((merged && merged_d) || n_owned == 0, "merge_init: null output");
    SG_CHECK_ARG(R >= 1 && R <= 128, "merge_init: R must be in [1, 128]");
    return merge_init_run(n_owned, R, merged, merged_d, S(stream));
}
sg_status scalegann_merge_shard(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k, const int32_t* owner_host,
                                int rank, int world, uint32_t shard, const uint32_t* idmap, uint64_t m,
                                const uint32_t* graph, const float* graph_d, uint32_t R, const uint32_t* owned_index,
                                const uint32_t* rec_slot, uint32_t* merged, float* merged_d, uint32_t* sendbuf,
                                void* stream) {
    SG_CHECK_ARG(home && owner_host && n > 0 && omega >= 1, "merge_shard: bad arguments");
    SG_CHECK_ARG(m == 0 || (idmap && graph && graph_d && owned_index && rec_slot), "merge_shard: null pointer");
    (void)n;
    return merge_shard_run(home, omega, k, owner_host, rank, world, shard, idmap, m, graph, graph_d, R, owned_index,
                           rec_slot, merged, merged_d, sendbuf, S(stream));
}
sg_status scalegann_merge_finish(uint32_t omega, uint32_t R, const uint32_t* owned_index, const uint32_t* recvbuf,
                                 uint64_t n_recv, uint32_t* merged, float* merged_d, void* ws, size_t ws_bytes,
                                 void* stream) {
    SG_CHECK_ARG(n_recv == 0 || (recvbuf && owned_index && merged && merged_d), "merge_finish: null pointer");
    Carver cv(ws, ws_bytes);
    int* err = cv.take<int>(1);
    if (!cv.ok() || !ws) { set_error("merge_finish: workspace too small"); return SG_ERR_WORKSPACE; }
    return merge_finish_run(omega, R, owned_index, recvbuf, n_recv, merged, merged_d, err, S(stream));
}

// collective merge: workspace = owned index + send slots + plan scratch + both record buffers
static sg_status merge_sizes(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k, const int32_t* owner_host,
                             void* comm, uint32_t R, size_t* bytes, uint64_t* n_owned, uint64_t* send, uint64_t* recv,
                             int* rank, int* world, void* ws, size_t ws_bytes, cudaStream_t st) {
    SG_TRY(comm_rank_world(comm, rank, world));
    const size_t pw = merge_plan_ws(n);
    Carver cv(nullptr, 0);
    cv.take<uint32_t>(n);           // owned_index
    cv.take<uint32_t>(n * omega);   // send slots
    cv.take<uint8_t>(pw);           // plan scratch
    cv.take<int>(1);
    const size_t fixed = cv.off + 4096;
    if (!ws) {
        // counting needs scratch of its own: the plan scratch alone, from a temporary buffer
        void* tmp = nullptr;
        SG_CUDA(cudaMallocAsync(&tmp, pw, st));
        sg_status e = merge_plan_run(home, n, omega, k, owner_host, *rank, *world, nullptr, nullptr, send, recv, n_owned,
                                     tmp, pw, st);
        cudaFreeAsync(tmp, st);
        SG_TRY(e);
    } else {
        if (ws_bytes < fixed) { set_error("merge: workspace too small"); return SG_ERR_WORKSPACE; }
        SG_TRY(merge_plan_run(home, n, omega, k, owner_host, *rank, *world, nullptr, nullptr, send, recv, n_owned, ws,
                              ws_bytes, st));
    }
    uint64_t ns = 0, nr = 0;
    for (int r = 0; r < *world; r++) { ns += send[r]; nr += recv[r]; }
    *bytes = fixed + (ns + nr) * (2 + 2 * (size_t)R) * 4 + 512;
    return SG_OK;
}

sg_status scalegann_merge_workspace(const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k,
                                    const int32_t* owner_host, void* comm, uint32_t R, size_t* bytes,
                                    uint64_t* n_owned_host, void* stream) {
    SG_CHECK_ARG(home && owner_host && bytes && n > 0 && omega >= 1, "merge_workspace: bad arguments");
    uint64_t send[64], recv[64], no = 0;
    int rank, world;
    SG_TRY(merge_sizes(home, n, omega, k, owner_host, comm, R, bytes, &no, send, recv, &rank, &world, nullptr, 0,
                       S(stream)));
    if (n_owned_host) *n_owned_host = no;
    return SG_OK;
}

sg_status scalegann_merge(void* comm, const uint32_t* home, uint64_t n, uint32_t omega, uint32_t k,
                          const int32_t* owner_host, const uint32_t* const* idmaps, const uint64_t* sizes_host,
                          const uint32_t* const* graphs, const float* const* graphs_d, uint32_t R, uint32_t* merged,
                          float* merged_d, uint64_t* n_owned_host, void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(home && owner_host && idmaps && sizes_host && graphs && graphs_d && n > 0 && omega >= 1,
                 "merge: bad arguments");
    SG_CHECK_ARG(k >= 1 && k <= 64 && R >= 1 && R <= 128, "merge: need 1 <= k <= 64, 1 <= R <= 128");
    cudaStream_t st = S(stream);
    uint64_t send[64], recv[64], no = 0;
    int rank, world;
    size_t need = 0;
    SG_TRY(merge_sizes(home, n, omega, k, owner_host, comm, R, &need, &no, send, recv, &rank, &world, ws, ws_bytes, st));
    if (ws_bytes < need) { set_error("merge: workspace too small (need %zu)", need); return SG_ERR_WORKSPACE; }
    SG_CHECK_ARG(no == 0 || (merged && merged_d), "merge: null merged output");
    for (uint32_t s = 0; s < k; s++)
        SG_CHECK_ARG(owner_host[s] != rank || sizes_host[s] == 0 || (idmaps[s] && graphs[s] && graphs_d[s]),
                     "merge: an owned shard has no graph");
    Carver cv(ws, ws_bytes);
    uint32_t* owned_index = cv.take<uint32_t>(n);
    uint32_t* rec_slot = cv.take<uint32_t>(n * omega);
    uint8_t* pws = cv.take<uint8_t>(merge_plan_ws(n));
    int* err = cv.take<int>(1);
    uint64_t ns = 0, nr = 0;
    for (int r = 0; r < world; r++) { ns += send[r]; nr += recv[r]; }
    const uint32_t W = 2 + 2 * R;
    uint32_t* sendbuf = cv.take<uint32_t>(ns * W);
    uint32_t* recvbuf = cv.take<uint32_t>(nr * W);
    if (!cv.ok()) { set_error("merge: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_TRY(merge_plan_run(home, n, omega, k, owner_host, rank, world, owned_index, rec_slot, send, recv, &no, pws,
                          merge_plan_ws(n), st));
    SG_TRY(merge_init_run(no, R, merged, merged_d, st));
    for (uint32_t s = 0; s < k; s++) {
        if (owner_host[s] != rank || sizes_host[s] == 0) continue;
        SG_TRY(merge_shard_run(home, omega, k, owner_host, rank, world, s, idmaps[s], sizes_host[s], graphs[s],
                               graphs_d[s], R, owned_index, rec_slot, merged, merged_d, sendbuf, st));
    }
    SG_TRY(exchange_records_run(comm, sendbuf, send, recvbuf, recv, W, st));
    SG_TRY(merge_finish_run(omega, R, owned_index, recvbuf, nr, merged, merged_d, err, st));
    if (n_owned_host) *n_owned_host = no;
    return SG_OK;
}

// ------------------------------------------------------------------ a9
sg_status scalegann_search_workspace(uint64_t n, uint32_t d, sg_dtype dtype, uint32_t nq, uint32_t topk, uint32_t beam,
                                     size_t* bytes) {
    SG_CHECK_ARG(bytes, "null bytes");
    (void)beam;
    size_t gt = knn_total_ws(nq, n, d, worst_prec(dtype, SG_PREC_AUTO, d), topk, false) + (size_t)nq * topk * 8 + 512;
    size_t bs = beam_ws(n, nq, beam, 128) + (size_t)nq * topk * 4 + 1024;   // sized for R <= 128
    *bytes = gt + bs;
    return SG_OK;
}

sg_status scalegann_search_eval(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const uint32_t* graph, uint32_t R,
                                uint32_t entry, const void* queries, uint32_t nq, uint32_t topk, uint32_t beam,
                                int32_t metric, const uint32_t* gt, uint32_t* gt_out, uint32_t* out_ids,
                                double* recall_host, uint64_t* n_dist_host, void* ws, size_t ws_bytes, void* stream) {
    SG_CHECK_ARG(x && graph && queries && out_ids && nq > 0 && n > 0 && d > 0 && d <= 1024, "search: bad arguments");
    SG_CHECK_ARG(entry < n, "search: entry out of range");
    SG_CHECK_ARG(R >= 1 && R <= 128 && topk >= 1 && topk <= beam && beam <= 512, "search: need R<=128, topk<=beam<=512");
    SG_CHECK_ARG(metric == SG_L2 || metric == SG_IP, "search: bad metric");
    cudaStream_t st = S(stream);
    Carver cv(ws, ws_bytes);
    const uint32_t* g = gt;
    if (!g) {
        uint32_t* gbuf = gt_out ? gt_out : cv.take<uint32_t>((size_t)nq * topk);
        float* gd = cv.take<float>((size_t)nq * topk);
        if (!cv.ok()) { set_error("search: workspace too small"); return SG_ERR_WORKSPACE; }
        Carver kc = cv;
        SG_TRY(knn_impl(queries, nullptr, nq, x, nullptr, n, dtype, d, 0, topk, metric, SG_PREC_AUTO, gbuf, gd, nullptr,
                        kc.base ? kc.base + kc.off : nullptr, kc.cap > kc.off ? kc.cap - kc.off : 0, st));
        g = gbuf;
    }
    unsigned long long* nd = cv.take<unsigned long long>(1);
    if (!cv.ok()) { set_error("search: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(nd, 0, sizeof(unsigned long long), st));
    SG_TRY(beam_run(x, dtype, n, d, graph, R, entry, queries, nq, topk, beam, metric, out_ids, nd, cv, st));
    if (n_dist_host) {
        SG_CUDA(cudaMemcpyAsync(n_dist_host, nd, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        SG_CUDA(cudaStreamSynchronize(st));
    }
    if (recall_host) return recall_run(out_ids, g, nq, topk, recall_host, cv, st);
    return SG_OK;
}

sg_status scalegann_search_shards_workspace(uint64_t n, uint32_t d, sg_dtype dtype, uint32_t nq, uint32_t topk,
                                            uint32_t beam, uint32_t n_entries, size_t* bytes) {
    SG_TRY(scalegann_search_workspace(n, d, dtype, nq, topk, beam, bytes));
    *bytes += (size_t)n_entries * nq * topk * 8 + 512;
    return SG_OK;
}

sg_status scalegann_search_eval_shards(const void* x, sg_dtype dtype, uint64_t n, uint32_t d, const uint32_t* graph,
                                       uint32_t R, const uint32_t* entries_host, uint32_t n_entries,
                                       const void* queries, uint32_t nq, uint32_t topk, uint32_t beam,
                                       int32_t metric, const uint32_t* gt, uint32_t* gt_out, uint32_t* out_ids,
                                       double* recall_host, uint64_t* n_dist_host, void* ws, size_t ws_bytes,
                                       void* stream) {
    SG_CHECK_ARG(x && graph && queries && out_ids && entries_host && nq > 0 && n > 0 && d > 0 && d <= 1024,
                 "search_shards: bad arguments");
    SG_CHECK_ARG(n_entries >= 1 && n_entries <= 1024, "search_shards: need 1 <= n_entries <= 1024");
    // SENTINEL entries (empty shards, scalegann_entry_points) are skipped; at least one is needed
    uint32_t n_real = 0;
    for (uint32_t s = 0; s < n_entries; s++) {
        SG_CHECK_ARG(entries_host[s] < n || entries_host[s] == SG_SENT, "search_shards: entry out of range");
        n_real += entries_host[s] != SG_SENT;
    }
    SG_CHECK_ARG(n_real >= 1, "search_shards: every entry is SENTINEL");
    SG_CHECK_ARG(R >= 1 && R <= 128 && topk >= 1 && topk <= beam && beam <= 512, "search: need R<=128, topk<=beam<=512");
    SG_CHECK_ARG(metric == SG_L2 || metric == SG_IP, "search: bad metric");
    cudaStream_t st = S(stream);
    Carver cv(ws, ws_bytes);
    uint64_t* keys = cv.take<uint64_t>((size_t)n_entries * nq * topk);
    if (!cv.ok()) { set_error("search_shards: workspace too small"); return SG_ERR_WORKSPACE; }
    const uint32_t* g = gt;
    if (!g) {
        uint32_t* gbuf = gt_out ? gt_out : cv.take<uint32_t>((size_t)nq * topk);
        float* gd = cv.take<float>((size_t)nq * topk);
        if (!cv.ok()) { set_error("search_shards: workspace too small"); return SG_ERR_WORKSPACE; }
        Carver kc = cv;
        SG_TRY(knn_impl(queries, nullptr, nq, x, nullptr, n, dtype, d, 0, topk, metric, SG_PREC_AUTO, gbuf, gd, nullptr,
                        kc.base ? kc.base + kc.off : nullptr, kc.cap > kc.off ? kc.cap - kc.off : 0, st));
        g = gbuf;
    }
    unsigned long long* nd = cv.take<unsigned long long>(1);
    if (!cv.ok()) { set_error("search_shards: workspace too small"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(nd, 0, sizeof(unsigned long long), st));
    uint32_t ns = 0;
    for (uint32_t s = 0; s < n_entries; s++) {
        if (entries_host[s] == SG_SENT) continue;
        Carver bc = cv;   // every per-entry search reuses the same visited-set scratch
        SG_TRY(beam_run(x, dtype, n, d, graph, R, entries_host[s], queries, nq, topk, beam, metric, nullptr, nd, bc, st,
                        keys + (size_t)ns * nq * topk));
        ns++;
    }
    SG_TRY(shard_merge_run(keys, ns, nq, topk, out_ids, st));
    if (n_dist_host) {
        SG_CUDA(cudaMemcpyAsync(n_dist_host, nd, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        SG_CUDA(cudaStreamSynchronize(st));
    }
    if (recall_host) return recall_run(out_ids, g, nq, topk, recall_host, cv, st);
    return SG_OK;
}

}  // extern "C"
