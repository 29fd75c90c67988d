// Device-wide exclusive scan (uint32 in -> uint64 out, out[n] = total), three passes:
// per-1024 block sums, a single-CTA scan of the block sums, per-block scan + offset.
#include "common.cuh"

namespace sg {
namespace {
constexpr int TB = 1024;

__global__ void scan_block_sums(const uint32_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ sums) {
    __shared__ uint32_t tmp[33];
    uint64_t i = (uint64_t)blockIdx.x * TB + threadIdx.x;
    uint32_t v = i < n ? in[i] : 0, tot;
    block_excl_scan(v, tmp, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void scan_sums(uint64_t* sums, uint64_t nb) {
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint64_t base = 0; base < nb; base += TB) {
        uint64_t i = base + threadIdx.x;
        uint64_t v = i < nb ? sums[i] : 0, inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += t;
        }
        if (lane == 31) warp_tot[w] = inc;
        __syncthreads();
        if (w == 0) {
            uint64_t s = warp_tot[lane], si = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint64_t t = __shfl_up_sync(0xffffffffu, si, o);
                if (lane >= (uint32_t)o) si += t;
            }
            warp_tot[lane] = si - s;
        }
        __syncthreads();
        uint64_t excl = carry + warp_tot[w] + inc - v;
        if (i < nb) sums[i] = excl;
        __syncthreads();
        if (threadIdx.x == TB - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[nb] = carry;
}

__global__ void scan_apply(const uint32_t* __restrict__ in, uint64_t n, const uint64_t* __restrict__ sums,
                           uint64_t* __restrict__ out, uint64_t nb) {
    __shared__ uint32_t tmp[33];
    uint64_t i = (uint64_t)blockIdx.x * TB + threadIdx.x;
    uint32_t v = i < n ? in[i] : 0;
    uint32_t e = block_excl_scan(v, tmp, nullptr);
    if (i < n) out[i] = sums[blockIdx.x] + e;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = sums[nb];
}
}  // namespace

size_t scan_workspace(uint64_t n) { return ((n + TB - 1) / TB + 2) * sizeof(uint64_t) + 512; }

sg_status excl_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, Carver& cv, cudaStream_t st) {
    const uint64_t nb = (n + TB - 1) / TB;
    uint64_t* sums = cv.take<uint64_t>(nb + 1);
    if (!cv.ok()) { set_error("scan: workspace too small"); return SG_ERR_WORKSPACE; }
    if (n == 0) {
        SG_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), st));
        return SG_OK;
    }
    scan_block_sums<<<(unsigned)nb, TB, 0, st>>>(in, n, sums);
    SG_LAUNCHED("scan_block_sums");
    scan_sums<<<1, TB, 0, st>>>(sums, nb);
    SG_LAUNCHED("scan_sums");
    scan_apply<<<(unsigned)nb, TB, 0, st>>>(in, n, sums, out, nb);
    SG_LAUNCHED("scan_apply");
    return SG_OK;
}

}  // namespace sg
