// a5 — exact kNN: tcgen05 distance tiles + fused per-row top-L (north_star stage 2).
//
// dist(i, j) = |a_i|^2 + |b_j|^2 - 2 a_i.b_j (L2) or -a_i.b_j (IP) (reading R2).  The -2 a.b
// term is a dense contraction and runs on the 5th-gen tensor cores: operands staged in
// shared memory by TMA (128-byte swizzle), tcgen05.mma (kind::f16 or kind::tf32, fp32
// accumulate, M=128 N=128) issued by one thread, accumulators double-buffered in TMEM and
// read back with tcgen05.ld by four epilogue warps that fuse the top-L selection.
//
// Work decomposition (persistent, one CTA per SM):
//   - a CTA owns 128 consecutive A rows ("row block"); its A tile stays resident in smem
//     (NKA 16 KB swizzle atoms) while every B column tile (128 rows of B) streams through an
//     S-stage TMA ring.  All CTAs walk the columns in the same order so the B stream is
//     served from L2.
//   - epilogue thread = one row (TMEM lane).  Per 32-column chunk: key = fma(scale, acc,
//     |b_j|^2), min over the chunk, and only if min < the row's threshold are the passing
//     (key, j) appended to the row's candidate buffer in global memory (L2 resident).
//     Columns arrive in increasing j, so "key < threshold" realises the (dist, id) order.
//   - when a row's buffer nears full, its warp cooperatively radix-selects the exact L
//     smallest (key, j) pairs (8-bit digits, smem histogram) and resets the threshold to the
//     L-th key; at the end of the row block the survivors are sorted by (dist, id).
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2..5 epilogue (warp w reads TMEM lanes 32*(w%4) .. +31).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace sg {
namespace {

constexpr uint32_t BM = 128, BN = 128, ATOM = 128 * 128;   // bytes per swizzle atom (128 rows x 128 B)
constexpr uint32_t NEPI = 8;                          // epilogue warps
constexpr uint32_t NTHREADS = 64 + NEPI * 32;
constexpr uint32_t MAX_STAGES = 12;

// ----------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    const uint32_t a = smem_u32(b);
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
// same, but lets the waiting thread sleep in hardware until the phase completes (bounded hint)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    const uint32_t a = smem_u32(b);
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(1000000u)
            : "memory");
    }
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
template <int KIND>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    if constexpr (KIND == 0) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    }
}
// tcgen05.ld 32 lanes x 32 columns of 32-bit: thread t of the warp gets row (lane base + t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return v;
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: D fp32, A/B f16 (KIND 0) or tf32 (KIND 1), both K-major, M=128, N=128.
template <int KIND>
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4) | ((KIND ? 2u : 0u) << 7) | ((KIND ? 2u : 0u) << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);
}

struct KnnParams {
    const float* norm_a;   // rows of A (|a|^2, or 0 for IP)
    const float* norm_b;   // rows of B (|b|^2, or 0 for IP; +inf padding)
    uint64_t* cand;        // gridDim.x * 128 * C candidate words
    uint32_t* out_ids;     // ma x L
    float* out_d;          // ma x L
    float* probe;          // optional raw-dot dump (ma x mb)
    uint32_t ma, mb, L, C, n_rb, n_ct, stages;
    float scale;           // -2 (L2) or -1 (IP)
    int self_exclude;
};

struct __align__(8) Bars {
    uint64_t full[MAX_STAGES], empty[MAX_STAGES];
    uint64_t a_full, a_empty;
    uint64_t tm_full[2], tm_empty[2];
    uint32_t tmem_base;
};

// ----------------------------------------------------------------- top-L selection
// Warp-cooperative: keep the exactly-L smallest of row buffer rb[0..cnt) (in place at
// rb[0..L)), return the L-th key (ordered u32).  All 32 lanes call with the same args.
template <int EPL>
__device__ uint32_t select_L(uint64_t* rb, uint32_t cnt, uint32_t L, uint32_t* hist, uint32_t lane) {
    uint64_t e[EPL];
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        uint32_t idx = i * 32 + lane;
        e[i] = idx < cnt ? rb[idx] : ~0ull;
    }
    uint64_t pfx = 0;
    uint32_t want = L, cut = 0;
#pragma unroll 1
    for (int sh = 56; sh >= 0; sh -= 8) {
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        const uint64_t hm = sh == 56 ? 0ull : (~0ull << (sh + 8));
#pragma unroll
        for (int i = 0; i < EPL; i++)
            if ((e[i] & hm) == (pfx & hm)) atomicAdd(&hist[(uint32_t)(e[i] >> sh) & 255u], 1u);
        __syncwarp();
        uint32_t h[8], loc = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) { h[j] = hist[lane * 8 + j]; loc += h[j]; }
        uint32_t inc = warp_incl_scan(loc, lane), exc = inc - loc;
        bool mine = exc < want && want <= inc;
        uint32_t bal = __ballot_sync(0xffffffffu, mine);
        uint32_t dg = 0, before = 0, bc = 0;
        if (mine) {
            uint32_t run = exc;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (bc == 0 && run + h[j] >= want) { dg = lane * 8 + j; before = run; bc = h[j]; }
                run += h[j];
            }
        }
        int src = __ffs(bal) - 1;
        dg = __shfl_sync(0xffffffffu, dg, src);
        before = __shfl_sync(0xffffffffu, before, src);
        bc = __shfl_sync(0xffffffffu, bc, src);
        want -= before;
        pfx |= (uint64_t)dg << sh;
        __syncwarp();
        if (bc == want) { cut = sh; break; }
    }
    const uint64_t lim = pfx >> cut;
    uint32_t base = 0, mk = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        uint32_t idx = i * 32 + lane;
        bool s = idx < cnt && (e[i] >> cut) <= lim;
        uint32_t bal = __ballot_sync(0xffffffffu, s);
        if (s) {
            rb[base + __popc(bal & ((1u << lane) - 1u))] = e[i];
            mk = max(mk, (uint32_t)(e[i] >> 32));
        }
        base += __popc(bal);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mk = max(mk, __shfl_xor_sync(0xffffffffu, mk, o));
    __syncwarp();
    return mk;
}

// Merge the two column halves' survivors of one row (each <= L, any order), sort by
// (dist, id) with dist = |a_i|^2 + key, write the first L (sentinel / +inf padding).
__device__ void finish_row(const uint64_t* b0, uint32_t c0, const uint64_t* b1, uint32_t c1, uint32_t L,
                           uint64_t* sortbuf, float na, uint32_t* out_ids, float* out_d, uint32_t lane) {
    const uint32_t cnt = c0 + c1;
    uint32_t np = 32;
    while (np < cnt) np <<= 1;
    for (uint32_t p = lane; p < np; p += 32) {
        uint64_t w = ~0ull;
        if (p < cnt) {
            const uint64_t e = p < c0 ? b0[p] : b1[p - c0];
            const float dist = na + ord2f((uint32_t)(e >> 32));
            w = ((uint64_t)f2ord(dist) << 32) | (uint32_t)e;
        }
        sortbuf[p] = w;
    }
    __syncwarp();
    warp_sort_u64(sortbuf, np, lane);
    for (uint32_t p = lane; p < L; p += 32) {
        const uint64_t w = sortbuf[p];
        out_ids[p] = p < cnt ? (uint32_t)w : SG_SENT;
        out_d[p] = p < cnt ? ord2f((uint32_t)(w >> 32)) : __int_as_float(0x7f800000);
    }
    __syncwarp();
}

// ----------------------------------------------------------------- the kernel
template <int KIND, int NKA, int EPL>
__global__ void __launch_bounds__(NTHREADS, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, KnnParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;                                   // NKA atoms
    uint8_t* sB = smem + NKA * ATOM;                      // stages atoms
    Bars* bars = (Bars*)(sB + p.stages * ATOM);
    uint32_t* hist_all = (uint32_t*)(bars + 1);           // NEPI x 256
    uint64_t* sort_all = (uint64_t*)(hist_all + NEPI * 256);   // NEPI x 512
    uint32_t* s_cnt = (uint32_t*)(sort_all + NEPI * 512);      // 2 halves x 128 rows

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t EL = KIND ? 4 : 2;                 // bytes per element
    constexpr uint32_t ATOM_K = 128 / EL;                 // elements per atom along K

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; s++) { mbar_init(&bars->full[s], 1); mbar_init(&bars->empty[s], 1); }
        mbar_init(&bars->a_full, 1);
        mbar_init(&bars->a_empty, 1);
        for (int b = 0; b < 2; b++) { mbar_init(&bars->tm_full[b], 1); mbar_init(&bars->tm_empty[b], NEPI); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars->tmem_base)),
                     "r"(256u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            uint32_t stage = 0, sph = 0, it = 0;
            for (uint32_t rb = blockIdx.x; rb < p.n_rb; rb += gridDim.x, it++) {
                if (it > 0) mbar_wait_sleep(&bars->a_empty, (it - 1) & 1);
                mbar_expect_tx(&bars->a_full, NKA * ATOM);
                for (int ka = 0; ka < NKA; ka++) tma_load_2d(&tmA, &bars->a_full, sA + ka * ATOM, ka * ATOM_K, rb * BM);
                for (uint32_t t = 0; t < p.n_ct; t++) {
                    for (int ka = 0; ka < NKA; ka++) {
                        mbar_wait_sleep(&bars->empty[stage], sph ^ 1);
                        mbar_expect_tx(&bars->full[stage], ATOM);
                        tma_load_2d(&tmB, &bars->full[stage], sB + stage * ATOM, ka * ATOM_K, t * BN);
                        if (++stage == p.stages) { stage = 0; sph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc = instr_desc<KIND>();
            const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
            uint32_t stage = 0, sph = 0, it = 0, git = 0;
            for (uint32_t rb = blockIdx.x; rb < p.n_rb; rb += gridDim.x, it++) {
                mbar_wait_sleep(&bars->a_full, it & 1);
                tc_fence_after();
                for (uint32_t t = 0; t < p.n_ct; t++, git++) {
                    const uint32_t buf = git & 1;
                    mbar_wait_sleep(&bars->tm_empty[buf], ((git >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t dcol = tmem + buf * BN;
                    for (int ka = 0; ka < NKA; ka++) {
                        mbar_wait_sleep(&bars->full[stage], sph);
                        tc_fence_after();
#pragma unroll
                        for (uint32_t kk = 0; kk < 4; kk++) {
                            uint64_t ad = smem_desc(a_base + ka * ATOM + kk * 32);
                            uint64_t bd = smem_desc(b_base + stage * ATOM + kk * 32);
                            tc_mma<KIND>(dcol, ad, bd, idesc, (ka | kk) != 0);
                        }
                        tc_commit(&bars->empty[stage]);
                        if (++stage == p.stages) { stage = 0; sph ^= 1; }
                    }
                    tc_commit(&bars->tm_full[buf]);
                }
                tc_commit(&bars->a_empty);
            }
        }
    } else {
        // ===================== epilogue: fused distance + top-L =====================
        // warp e = warp-2 in 0..7: TMEM lane quadrant q (rows q*32..), column half h (64 cols)
        const uint32_t e = warp - 2, q = warp & 3, h = e >> 2;
        const uint32_t r = q * 32 + lane;                   // row within the block
        uint32_t* hist = hist_all + e * 256;
        uint64_t* sortbuf = sort_all + e * 512;
        const uint32_t C = p.C;
        uint64_t* half_base = p.cand + ((uint64_t)blockIdx.x * 2 + h) * BM * C;
        uint64_t* myrow = half_base + (uint64_t)r * C;
        uint64_t* warprows = half_base + (uint64_t)q * 32 * C;
        const float INF = __int_as_float(0x7f800000);
        const uint32_t tl = tmem + ((q * 32) << 16) + h * 64;
        uint32_t git = 0;
        for (uint32_t rb = blockIdx.x; rb < p.n_rb; rb += gridDim.x) {
            const uint32_t row = rb * BM + r;
            const bool valid = row < p.ma;
            float thr = valid ? INF : -INF;
            uint32_t cnt = 0;
            for (uint32_t t = 0; t < p.n_ct; t++, git++) {
                const uint32_t buf = git & 1;
                mbar_wait_sleep(&bars->tm_full[buf], (git >> 1) & 1);
                tc_fence_after();
                const uint32_t tb = tl + buf * BN;
                uint32_t v[2][32];
                tmem_ld32_nowait(tb, v[0]);
                tmem_ld32_nowait(tb + 32, v[1]);
                tmem_wait_ld();
                const bool diag = p.self_exclude && t == rb;
#pragma unroll
                for (uint32_t ch = 0; ch < 2; ch++) {
                    const uint32_t col0 = t * BN + h * 64 + ch * 32;
                    if (p.probe) {
                        if (valid)
                            for (int j = 0; j < 32; j++)
                                if (col0 + j < p.mb) p.probe[(uint64_t)row * p.mb + col0 + j] = __uint_as_float(v[ch][j]);
                        continue;
                    }
                    // make room: rows whose buffer cannot take another 32 candidates are compacted
                    uint32_t need = __ballot_sync(0xffffffffu, cnt > C - 32);
                    while (need) {
                        const int o = __ffs(need) - 1;
                        need &= need - 1;
                        const uint32_t c_o = __shfl_sync(0xffffffffu, cnt, o);
                        uint32_t kth = select_L<EPL>(warprows + (uint64_t)o * C, c_o, p.L, hist, lane);
                        if (lane == (uint32_t)o) { cnt = p.L; thr = ord2f(kth); }
                    }
                    const float4* nb4 = (const float4*)(p.norm_b + col0);
                    uint32_t mask = 0;
#pragma unroll
                    for (int j4 = 0; j4 < 8; j4++) {
                        const float4 nb = __ldg(nb4 + j4);
                        const float k0 = fmaf(p.scale, __uint_as_float(v[ch][4 * j4 + 0]), nb.x);
                        const float k1 = fmaf(p.scale, __uint_as_float(v[ch][4 * j4 + 1]), nb.y);
                        const float k2 = fmaf(p.scale, __uint_as_float(v[ch][4 * j4 + 2]), nb.z);
                        const float k3 = fmaf(p.scale, __uint_as_float(v[ch][4 * j4 + 3]), nb.w);
                        mask |= (k0 < thr ? 1u : 0u) << (4 * j4 + 0);
                        mask |= (k1 < thr ? 1u : 0u) << (4 * j4 + 1);
                        mask |= (k2 < thr ? 1u : 0u) << (4 * j4 + 2);
                        mask |= (k3 < thr ? 1u : 0u) << (4 * j4 + 3);
                    }
                    if (diag && ch + 2 * h == q) mask &= ~(1u << lane);   // self column
                    // rare path: walk the union of passing columns (warp-uniform), re-read each
                    // column from TMEM (uniform address) and append where this row passes
                    uint32_t U = __reduce_or_sync(0xffffffffu, mask);
                    while (U) {
                        const uint32_t c = __ffs(U) - 1;
                        U &= U - 1;
                        const uint32_t raw = tmem_ld1(tb + ch * 32 + c);
                        if ((mask >> c) & 1u) {
                            const float kv = fmaf(p.scale, __uint_as_float(raw), __ldg(p.norm_b + col0 + c));
                            myrow[cnt] = ((uint64_t)f2ord(kv) << 32) | (col0 + c);
                            cnt++;
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->tm_empty[buf]);
            }
            if (p.probe) continue;
            // ---- final: each half keeps its exact top-L, then the two halves of a row are merged
            __syncwarp();
            for (uint32_t o = 0; o < 32; o++) {
                uint32_t c_o = __shfl_sync(0xffffffffu, cnt, o);
                if (c_o > p.L) { select_L<EPL>(warprows + (uint64_t)o * C, c_o, p.L, hist, lane); c_o = p.L; }
                if (lane == 0) s_cnt[h * BM + q * 32 + o] = c_o;
            }
            __syncwarp();
            named_bar_sync(1 + q, 64);
            for (uint32_t i = 0; i < 16; i++) {
                const uint32_t rr = q * 32 + h * 16 + i;
                const uint32_t row_o = rb * BM + rr;
                if (row_o >= p.ma) continue;
                const uint32_t c0 = s_cnt[rr], c1 = s_cnt[BM + rr];
                const uint64_t* b0 = p.cand + ((uint64_t)blockIdx.x * 2 + 0) * BM * C + (uint64_t)rr * C;
                const uint64_t* b1 = p.cand + ((uint64_t)blockIdx.x * 2 + 1) * BM * C + (uint64_t)rr * C;
                finish_row(b0, c0, b1, c1, p.L, sortbuf, p.norm_a[row_o], p.out_ids + (uint64_t)row_o * p.L,
                           p.out_d + (uint64_t)row_o * p.L, lane);
            }
            named_bar_sync(1 + q, 64);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
    }
}

// ----------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    return fn;
}

sg_status make_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t kdim, uint32_t esize) {
    auto enc = get_encode();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return SG_ERR_CUDA; }
    cuuint64_t dims[2] = {kdim, rows};
    cuuint64_t strides[1] = {(cuuint64_t)kdim * esize};
    cuuint32_t box[2] = {128u / esize, 128u};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return SG_ERR_CUDA; }
    return SG_OK;
}

uint32_t cand_cap(uint32_t L) {
    uint32_t c = 128;
    while (c < 4 * L && c < 1024) c <<= 1;
    return c;
}

template <int KIND, int NKA, int EPL>
sg_status launch_t(const CUtensorMap& a, const CUtensorMap& b, KnnParams& p, cudaStream_t st) {
    const size_t fixed = NKA * ATOM + sizeof(Bars) + NEPI * 256 * 4 + NEPI * 512 * 8 + 2 * BM * 4 + 1024;
    const size_t budget = 227 * 1024;
    uint32_t stages = (uint32_t)((budget - fixed) / ATOM);
    if (stages > MAX_STAGES) stages = MAX_STAGES;
    if (stages < 2) { set_error("kNN: operand too wide for shared memory"); return SG_ERR_UNSUPPORTED; }
    p.stages = stages;
    const size_t smem = fixed + stages * ATOM;
    auto kern = knn_tc_kernel<KIND, NKA, EPL>;
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint32_t grid = p.n_rb < (uint32_t)num_sms() ? p.n_rb : (uint32_t)num_sms();
    knn_time_begin(st);
    kern<<<grid, NTHREADS, smem, st>>>(a, b, p);
    SG_LAUNCHED("knn_tc_kernel");
    knn_time_end(st);
    return SG_OK;
}

template <int KIND, int EPL>
sg_status launch_nka(int nka, const CUtensorMap& a, const CUtensorMap& b, KnnParams& p, cudaStream_t st) {
    switch (nka) {
        case 1: return launch_t<KIND, 1, EPL>(a, b, p, st);
        case 2: return launch_t<KIND, 2, EPL>(a, b, p, st);
        case 3: return launch_t<KIND, 3, EPL>(a, b, p, st);
        case 4: return launch_t<KIND, 4, EPL>(a, b, p, st);
        case 5: return launch_t<KIND, 5, EPL>(a, b, p, st);
        case 6: return launch_t<KIND, 6, EPL>(a, b, p, st);
    }
    set_error("kNN: unsupported operand width (%d atoms)", nka);
    return SG_ERR_UNSUPPORTED;
}

}  // namespace

size_t knn_core_workspace(uint32_t L) {
    return (size_t)num_sms() * 2 * BM * cand_cap(L) * sizeof(uint64_t) + 4096;
}

sg_status knn_core(const Operand& A, const Operand& B, int metric, bool self_exclude, uint32_t L,
                   uint32_t* ids, float* dists, float* probe, Carver& cv, cudaStream_t st) {
    if (A.kdim != B.kdim || A.esize != B.esize) { set_error("kNN: operand mismatch"); return SG_ERR_INVALID_ARG; }
    const int nka = (int)(A.kdim * A.esize / 128);
    KnnParams p{};
    p.norm_a = A.norm_a;
    p.norm_b = B.norm_b;
    p.C = cand_cap(L);
    p.cand = cv.take<uint64_t>((size_t)num_sms() * 2 * BM * p.C);
    if (!cv.ok()) { set_error("kNN: workspace too small"); return SG_ERR_WORKSPACE; }
    p.out_ids = ids;
    p.out_d = dists;
    p.probe = probe;
    p.ma = (uint32_t)A.rows;
    p.mb = (uint32_t)B.rows;
    p.L = L;
    p.n_rb = (uint32_t)(A.rows_pad / BM);
    p.n_ct = (uint32_t)(B.rows_pad / BN);
    p.scale = metric == SG_IP ? -1.f : -2.f;
    p.self_exclude = self_exclude ? 1 : 0;
    CUtensorMap ma, mb;
    SG_TRY(make_map(&ma, A.a, A.rows_pad, A.kdim, A.esize));
    SG_TRY(make_map(&mb, B.b, B.rows_pad, B.kdim, B.esize));
    const bool tf32 = A.esize == 4;
    const int epl = (int)(p.C / 32);
    if (tf32) {
        if (epl <= 4) return launch_nka<1, 4>(nka, ma, mb, p, st);
        if (epl <= 16) return launch_nka<1, 16>(nka, ma, mb, p, st);
        return launch_nka<1, 32>(nka, ma, mb, p, st);
    }
    if (epl <= 4) return launch_nka<0, 4>(nka, ma, mb, p, st);
    if (epl <= 16) return launch_nka<0, 16>(nka, ma, mb, p, st);
    return launch_nka<0, 32>(nka, ma, mb, p, st);
}

}  // namespace sg
