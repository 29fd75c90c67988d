// a6 — rank-based detour-count prune (north_star stage 3; reading R10, CAGRA prior art).
//
// One warp per node a.  N[a] (L ids) goes into a shared-memory open-addressing table
// id -> rank.  For each rank r_ad the warp reads the 2-hop row N[delta] (delta = N[a][r_ad])
// with coalesced 16-byte loads (4 rows in flight per lane batch) and, for every b in it that
// is also in N[a] at rank r_ab with max(r_ad, r_db) < r_ab (rule P; rule 1: r_ad < r_ab),
// increments cnt[r_ab] in shared memory.  The ranks are then bitonic-sorted by
// (cnt, rank) (sentinel ranks last) and the first R written with their kNN distances.
// Bit-exact with the oracle (integer work only).
#include "common.cuh"

namespace sg {
namespace {


__device__ __forceinline__ uint32_t hslot(uint32_t id, uint32_t bits) { return (id * 0x9E3779B1u) >> (32 - bits); }

template <int LPL, int PW>   // ranks per lane = L_pad / 32; warps (nodes) per CTA
__global__ void __launch_bounds__(PW * 32) prune_kernel(const uint32_t* __restrict__ knn, const float* __restrict__ knn_d,
                                                        uint64_t m, uint32_t L, uint32_t R, uint32_t rule,
                                                        uint32_t* __restrict__ out, float* __restrict__ out_d) {
    constexpr uint32_t LP = LPL * 32;          // padded L (power of two)
    constexpr uint32_t HS = 2 * LP;            // hash slots
    constexpr uint32_t HB = LPL == 1 ? 6 : LPL == 2 ? 7 : LPL == 4 ? 8 : 9;
    __shared__ uint32_t s_key[PW][HS];
    __shared__ uint16_t s_rank[PW][HS];
    __shared__ uint32_t s_cnt[PW][LP];
    __shared__ uint32_t s_na[PW][LP];
    __shared__ uint64_t s_sort[PW][LP];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* hk = s_key[w];
    uint16_t* hr = s_rank[w];
    uint32_t* cnt = s_cnt[w];
    uint32_t* na = s_na[w];
    uint64_t* keys = s_sort[w];
    const uint64_t nwarps = (uint64_t)gridDim.x * PW;
    for (uint64_t a = (uint64_t)blockIdx.x * PW + w; a < m; a += nwarps) {
        const uint32_t* Na = knn + a * L;
        for (uint32_t i = lane; i < HS; i += 32) hk[i] = SG_SENT;
        for (uint32_t r = lane; r < LP; r += 32) { na[r] = r < L ? Na[r] : SG_SENT; cnt[r] = 0; }
        __syncwarp();
        for (uint32_t r = lane; r < L; r += 32) {
            const uint32_t id = na[r];
            if (id == SG_SENT) continue;
            uint32_t h = hslot(id, HB);
            while (atomicCAS(&hk[h], SG_SENT, id) != SG_SENT) h = (h + 1) & (HS - 1);
            hr[h] = (uint16_t)r;
        }
        __syncwarp();
        for (uint32_t r0 = 0; r0 < L; r0 += 4) {
            uint32_t bv[4][LPL];
            uint32_t dl[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                dl[u] = r0 + u < L ? na[r0 + u] : SG_SENT;
#pragma unroll
                for (int q = 0; q < LPL; q++) {
                    const uint32_t rdb = q * 32 + lane;
                    bv[u][q] = (dl[u] != SG_SENT && rdb < L) ? __ldg(knn + (uint64_t)dl[u] * L + rdb) : SG_SENT;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t r_ad = r0 + u;
#pragma unroll
                for (int q = 0; q < LPL; q++) {
                    const uint32_t b = bv[u][q];
                    if (b == SG_SENT || b == (uint32_t)a) continue;
                    const uint32_t r_db = q * 32 + lane;
                    uint32_t h = hslot(b, HB), key;
                    while ((key = hk[h]) != SG_SENT && key != b) h = (h + 1) & (HS - 1);
                    if (key != b) continue;
                    const uint32_t r_ab = hr[h];
                    const uint32_t mx = rule == 0 ? max(r_ad, r_db) : r_ad;
                    if (mx < r_ab) atomicAdd(&cnt[r_ab], 1u);
                }
            }
        }
        __syncwarp();
        for (uint32_t r = lane; r < LP; r += 32)
            keys[r] = r >= L ? ~0ull : na[r] == SG_SENT ? ((0xFFFFFFFFull << 32) | r) : (((uint64_t)cnt[r] << 32) | r);
        __syncwarp();
        warp_sort_u64(keys, LP, lane);
        for (uint32_t i = lane; i < R; i += 32) {
            const uint32_t r = (uint32_t)keys[i];
            out[a * R + i] = na[r];
            out_d[a * R + i] = knn_d[a * L + r];
        }
        __syncwarp();
    }
}

}  // namespace

sg_status launch_prune(const uint32_t* knn, const float* knn_d, uint64_t m, uint32_t L, uint32_t R, uint32_t rule,
                       uint32_t* out, float* out_d, cudaStream_t st) {
    if (m == 0) return SG_OK;
    const uint64_t cap = (uint64_t)num_sms() * 16;
    auto grid = [&](int pw) { uint64_t b = (m + pw - 1) / pw; return (unsigned)(b < cap ? b : cap); };
    if (L <= 32) prune_kernel<1, 8><<<grid(8), 8 * 32, 0, st>>>(knn, knn_d, m, L, R, rule, out, out_d);
    else if (L <= 64) prune_kernel<2, 8><<<grid(8), 8 * 32, 0, st>>>(knn, knn_d, m, L, R, rule, out, out_d);
    else if (L <= 128) prune_kernel<4, 8><<<grid(8), 8 * 32, 0, st>>>(knn, knn_d, m, L, R, rule, out, out_d);
    else prune_kernel<8, 4><<<grid(4), 4 * 32, 0, st>>>(knn, knn_d, m, L, R, rule, out, out_d);
    SG_LAUNCHED("prune_kernel");
    return SG_OK;
}

}  // namespace sg
