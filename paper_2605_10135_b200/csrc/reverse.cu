// a7 — reverse-edge insertion (north_star stage 3; reading R11).
//
//   rev[y] = sources x ordered by (k, x) where y = pruned[x][k], capped at R;
//   out[y] = pruned[y][0..h) ++ first R-h of (rev_np ++ [f in pruned[y][h..R) : f not in rev_np]),
//   rev_np = [x in rev[y] : x not in pruned[y][0..h)].
// Deterministic despite atomics: in-degrees are counted, scanned into CSR offsets, keys
// (k << 32 | x) scattered with atomic slots, and each row's segment is then sorted by key
// (bitonic in shared memory, chunked for hub rows with in-degree > 256) before the first R
// are taken — so the result never depends on atomic order.  Bit-exact with the oracle.
#include "common.cuh"

namespace sg {
namespace {

constexpr int RW = 8;        // warps (rows) per CTA
constexpr int SEGBUF = 256;  // sort buffer per warp

__global__ void indeg_kernel(const uint32_t* __restrict__ pruned, uint64_t edges, uint32_t* __restrict__ deg) {
    uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= edges) return;
    const uint32_t y = pruned[e];
    if (y != SG_SENT) atomicAdd(&deg[y], 1u);
}

__global__ void scatter_kernel(const uint32_t* __restrict__ pruned, uint64_t edges, uint32_t R,
                               const uint64_t* __restrict__ off, uint32_t* __restrict__ fill,
                               uint64_t* __restrict__ keys) {
    uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= edges) return;
    const uint32_t y = pruned[e];
    if (y == SG_SENT) return;
    const uint64_t x = e / R, k = e % R;
    const uint64_t pos = off[y] + atomicAdd(&fill[y], 1u);
    keys[pos] = (k << 32) | x;
}

__global__ void __launch_bounds__(RW * 32) reverse_merge_kernel(const uint32_t* __restrict__ pruned,
                                                                 const float* __restrict__ pruned_d, uint64_t m,
                                                                 uint32_t R, uint32_t h, const uint64_t* __restrict__ off,
                                                                 const uint64_t* __restrict__ keys,
                                                                 uint32_t* __restrict__ out, float* __restrict__ out_d) {
    __shared__ uint64_t s_buf[RW][SEGBUF];
    __shared__ uint32_t s_fw[RW][128];
    __shared__ float s_fwd[RW][128];
    __shared__ uint32_t s_t[RW][256];
    __shared__ float s_td[RW][256];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* buf = s_buf[w];
    uint32_t* fw = s_fw[w];
    float* fwd = s_fwd[w];
    uint32_t* tl = s_t[w];
    float* tld = s_td[w];
    const uint64_t nwarps = (uint64_t)gridDim.x * RW;
    for (uint64_t y = (uint64_t)blockIdx.x * RW + w; y < m; y += nwarps) {
        const uint64_t b0 = off[y], deg = off[y + 1] - b0;
        // ---- the first min(R, deg) keys of the segment in ascending order -> buf[0..nrev)
        uint32_t nrev = 0;
        if (deg > 0) {
            uint64_t done = 0;
            while (done < deg) {
                const uint32_t keep = nrev;                       // sorted survivors at buf[0..keep)
                const uint64_t rem = deg - done, room = SEGBUF - keep;
                const uint64_t take = rem < room ? rem : room;
                uint32_t np = 32;   // sort only the next power of two >= the entries present
                while (np < keep + take) np <<= 1;
                for (uint32_t i = lane; i < np - keep; i += 32)
                    buf[keep + i] = i < take ? keys[b0 + done + i] : ~0ull;
                __syncwarp();
                warp_sort_u64(buf, np, lane);
                done += take;
                nrev = (uint32_t)((uint64_t)R < keep + take ? (uint64_t)R : keep + take);
            }
        }
        // ---- forward row
        for (uint32_t j = lane; j < R; j += 32) { fw[j] = pruned[y * R + j]; fwd[j] = pruned_d[y * R + j]; }
        __syncwarp();
        // ---- rev_np = rev entries not among the h protected forward edges (order kept)
        uint32_t nt = 0;
        for (uint32_t i0 = 0; i0 < nrev; i0 += 32) {
            const uint32_t i = i0 + lane;
            bool keepit = false;
            uint32_t x = 0;
            float dx = 0.f;
            if (i < nrev) {
                const uint64_t key = buf[i];
                x = (uint32_t)key;
                const uint32_t k = (uint32_t)(key >> 32);
                dx = pruned_d[(uint64_t)x * R + k];
                keepit = true;
                for (uint32_t j = 0; j < h; j++) if (fw[j] == x) { keepit = false; break; }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keepit);
            if (keepit) {
                const uint32_t pos = nt + __popc(bal & ((1u << lane) - 1u));
                tl[pos] = x;
                tld[pos] = dx;
            }
            nt += __popc(bal);
        }
        __syncwarp();
        const uint32_t nrnp = nt;
        // ---- then the remaining forward edges not already in rev_np
        for (uint32_t j0 = h; j0 < R; j0 += 32) {
            const uint32_t j = j0 + lane;
            bool keepit = false;
            if (j < R) {
                keepit = true;
                const uint32_t f = fw[j];
                for (uint32_t i = 0; i < nrnp; i++) if (tl[i] == f) { keepit = false; break; }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keepit);
            __syncwarp();
            if (keepit) {
                const uint32_t pos = nt + __popc(bal & ((1u << lane) - 1u));
                tl[pos] = fw[j];
                tld[pos] = fwd[j];
            }
            nt += __popc(bal);
            __syncwarp();
        }
        __syncwarp();
        for (uint32_t j = lane; j < R; j += 32) {
            const bool prot = j < h;
            out[y * R + j] = prot ? fw[j] : tl[j - h];
            out_d[y * R + j] = prot ? fwd[j] : tld[j - h];
        }
        __syncwarp();
    }
}

}  // namespace

size_t reverse_ws(uint64_t m, uint32_t R) {
    Carver cv(nullptr, 0);
    cv.take<uint32_t>(m);       // deg
    cv.take<uint32_t>(m);       // fill
    cv.take<uint64_t>(m + 1);   // off
    cv.take<uint64_t>(m * R);   // keys
    return cv.off + scan_workspace(m) + 1024;
}

sg_status launch_reverse(const uint32_t* pruned, const float* pruned_d, uint64_t m, uint32_t R, uint32_t h,
                         uint32_t* out, float* out_d, Carver& cv, cudaStream_t st) {
    uint32_t* deg = cv.take<uint32_t>(m);
    uint32_t* fill = cv.take<uint32_t>(m);
    uint64_t* off = cv.take<uint64_t>(m + 1);
    uint64_t* keys = cv.take<uint64_t>(m * R);
    if (!cv.ok()) { set_error("reverse: workspace too small"); return SG_ERR_WORKSPACE; }
    if (m == 0) return SG_OK;
    SG_CUDA(cudaMemsetAsync(deg, 0, m * sizeof(uint32_t), st));
    SG_CUDA(cudaMemsetAsync(fill, 0, m * sizeof(uint32_t), st));
    const uint64_t edges = m * R;
    const unsigned eg = (unsigned)((edges + 255) / 256);
    indeg_kernel<<<eg, 256, 0, st>>>(pruned, edges, deg);
    SG_LAUNCHED("indeg_kernel");
    SG_TRY(excl_scan_u32_to_u64(deg, off, m, cv, st));
    scatter_kernel<<<eg, 256, 0, st>>>(pruned, edges, R, off, fill, keys);
    SG_LAUNCHED("scatter_kernel");
    const uint64_t blocks = (m + RW - 1) / RW, cap = (uint64_t)num_sms() * 16;
    reverse_merge_kernel<<<(unsigned)(blocks < cap ? blocks : cap), RW * 32, 0, st>>>(pruned, pruned_d, m, R, h, off,
                                                                                      keys, out, out_d);
    SG_LAUNCHED("reverse_merge_kernel");
    return SG_OK;
}

}  // namespace sg
