// Spatial order of a shard for the distance kernel (a5 performance; results unchanged).
//
// Rows of a shard arrive in ascending global id, which is random in space, so a row's true
// neighbours are spread over the whole column sweep and the running top-L threshold tightens
// slowly (many candidate insertions).  Here the rows are grouped by their nearest of Kc ~ m/1024
// sub-centroids (shard rows at a fixed stride; assignment = the tensor-core kNN with L = 1) and
// the distance kernel visits column tiles starting just before each row block's own group.
// The kNN result is exact and tie-broken by original local id, so it does not depend on this
// order (nor on the nondeterministic order inside a group).
#include <stdlib.h>

#include "common.cuh"

namespace sg {
namespace {

__global__ void strided_ids(const uint32_t* __restrict__ idmap, uint64_t m, uint32_t kc, uint32_t* __restrict__ out) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < kc) {
        const uint64_t i = (uint64_t)c * m / kc;
        out[c] = idmap ? idmap[i] : (uint32_t)i;
    }
}

__global__ void group_count(const uint32_t* __restrict__ asg, uint64_t m, uint32_t* __restrict__ cnt) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) atomicAdd(&cnt[asg[i]], 1u);
}

__global__ void group_scatter(const uint32_t* __restrict__ asg, uint64_t m, const uint64_t* __restrict__ off,
                              uint32_t* __restrict__ fill, const uint32_t* __restrict__ idmap,
                              uint32_t* __restrict__ perm, uint32_t* __restrict__ ids_perm) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t g = asg[i];
    const uint64_t pos = off[g] + atomicAdd(&fill[g], 1u);
    perm[pos] = (uint32_t)i;
    ids_perm[pos] = idmap ? idmap[i] : (uint32_t)i;
}

}  // namespace

static uint64_t group_rows() {
    static uint64_t g = 0;
    if (!g) {
        const char* e = getenv("SG_ORDER_GROUP_ROWS");
        g = e ? strtoull(e, nullptr, 10) : 1024;
        if (g < 128) g = 128;
    }
    return g;
}

uint32_t order_groups(uint64_t m) {
    // Off by default: with the extrapolated thresholds of the distance kernel (knn_tc.cu) the
    // columns must arrive in an order unrelated to the row's position, which the plain id order
    // is; the spatial order + rotated sweep remains available for comparison.
    static int on = -1;
    if (on < 0) { const char* e = getenv("SG_KNN_ORDER"); on = e ? atoi(e) : 0; }
    if (!on) return 0;
    uint64_t kc = m / group_rows();
    if (kc > 8192) kc = 8192;
    return (uint32_t)kc;
}

size_t order_workspace(uint64_t m, uint32_t d, int prec, int metric) {
    if (order_groups(m) < 2) return 0;   // ordering off (the default): no scratch
    const uint32_t kc = order_groups(m);
    Carver cv(nullptr, 0);
    cv.take<uint32_t>(kc);          // centroid row ids
    cv.take<uint32_t>(m);           // assignment
    cv.take<float>(m);              // assignment distances
    cv.take<uint32_t>(kc);          // counts
    cv.take<uint32_t>(kc);          // fill
    cv.take<uint64_t>(kc + 1);      // offsets
    return cv.off + operand_bytes(prec, metric, d, m, SIDE_A) + operand_bytes(prec, metric, d, kc, SIDE_B) +
           knn_core_workspace(1, m, d, prec, metric) + scan_workspace(kc) + 4096;
}

sg_status spatial_order(const void* x, sg_dtype dtype, uint32_t d, const uint32_t* idmap, uint64_t m, int prec,
                        int metric, uint32_t* perm, uint32_t* ids_perm, Carver cv, cudaStream_t st) {
    const uint32_t kc = order_groups(m);
    if (kc < 2) { set_error("order: shard too small to group"); return SG_ERR_INVALID_ARG; }
    uint32_t* cids = cv.take<uint32_t>(kc);
    uint32_t* asg = cv.take<uint32_t>(m);
    float* asd = cv.take<float>(m);
    uint32_t* cnt = cv.take<uint32_t>(kc);
    uint32_t* fill = cv.take<uint32_t>(kc);
    uint64_t* off = cv.take<uint64_t>(kc + 1);
    if (!cv.ok()) { set_error("order: workspace too small"); return SG_ERR_WORKSPACE; }
    strided_ids<<<(kc + 255) / 256, 256, 0, st>>>(idmap, m, kc, cids);
    SG_LAUNCHED("strided_ids");
    Operand A, B;
    SG_TRY(gather_operand(x, dtype, d, idmap, m, prec, metric, SIDE_A, cv, &A, st));
    SG_TRY(gather_operand(x, dtype, d, cids, kc, prec, metric, SIDE_B, cv, &B, st));
    SG_TRY(knn_core(A, B, metric, false, 1, asg, asd, nullptr, cv, st));
    SG_CUDA(cudaMemsetAsync(cnt, 0, kc * sizeof(uint32_t), st));
    SG_CUDA(cudaMemsetAsync(fill, 0, kc * sizeof(uint32_t), st));
    const unsigned g = (unsigned)((m + 255) / 256);
    group_count<<<g, 256, 0, st>>>(asg, m, cnt);
    SG_LAUNCHED("group_count");
    SG_TRY(excl_scan_u32_to_u64(cnt, off, kc, cv, st));
    group_scatter<<<g, 256, 0, st>>>(asg, m, off, fill, idmap, perm, ids_perm);
    SG_LAUNCHED("group_scatter");
    return SG_OK;
}

}  // namespace sg
