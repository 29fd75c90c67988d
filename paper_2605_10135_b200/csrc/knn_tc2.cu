// a5 — exact kNN on a CTA pair: tcgen05.mma.cta_group::2 distance tiles + fused per-row top-L
// (north_star stage 2; the same selection and the same results as knn_tc.cu).
//
// The keys are the augmented-operand contraction of knn_tc.cu (key(i, j) = |b_j|^2 - 2 a_i.b_j,
// gather.cu); this file only changes how the two SMs of a TPC share the work:
//   * a cluster of 2 CTAs owns a 256-row block; CTA r keeps rows [128 r, 128 r + 128) of it
//     resident in its shared memory (the A half of an M = 256 MMA);
//   * every 128-column B tile is split by columns: CTA r loads columns [64 r, 64 r + 64) (the B
//     half of an N = 128 MMA), so each SM reads 6 KB of operands per 64-cycle MMA (96 B/cycle,
//     under the 128 B/cycle shared-memory port) instead of 8 KB;
//   * one thread of the leader CTA issues tcgen05.mma.cta_group::2 for the pair; each CTA's
//     TMEM receives its 128 rows x 128 columns, so the 512 TMEM columns hold FOUR accumulator
//     buffers (the MMA runs up to three tiles ahead of the slowest epilogue warp);
//   * 16 epilogue warps per CTA: TMEM lane quadrant q = warp % 4 and column stream s (32 columns
//     of every tile, one tcgen05.ld per tile); per row, four stream buffers share one threshold.
// Barriers: the leader's full[]/a_full count one remote expect_tx arrival per CTA and both CTAs'
// TMA loads complete on them; the leader's commits arrive on empty[]/a_empty/tm_full[] of both
// CTAs (multicast); every epilogue warp of both CTAs arrives on the leader's tm_empty[].
//
// Status: bit-exact (the kNN parity suites pass with SG_KNN_2CTA=1) but OPT-IN.  Measured on
// B200 with the epilogue stubbed (SG_KNN_NOEPI=1, even without TMA loads and full-barrier
// waits): one M = 256, N = 128 cta_group::2 MMA takes ~231 cycles where the single-CTA kernel's
// M = 128, N = 128 MMA takes ~114, i.e. the pair delivers half the single-CTA rate at N = 128
// (566 vs 1234 TFLOP/s algorithmic at m = 75,776).  Both are far above the 64-cycle tile floor,
// which points at a per-instruction dispatch cost that only a wider N amortises.
#include "knn_common.cuh"

namespace sg {
namespace {

constexpr uint32_t BN2 = 128;            // columns per tile (MMA N over the pair)
constexpr uint32_t BNH = 64;             // columns of a tile loaded by one CTA
constexpr uint32_t M2 = 128;             // rows per CTA (MMA M = 256 over the pair)
constexpr uint32_t RB2 = 256;            // rows per row block
constexpr uint32_t NBUF2 = 4;            // TMEM accumulator buffers of 128 columns
constexpr uint32_t NSTR = 4;             // column streams per row (32 columns of each tile)
constexpr uint32_t NEPI2 = 16;           // epilogue warps (4 quadrants x 4 streams)
constexpr uint32_t NTH2 = 64 + NEPI2 * 32;
constexpr uint32_t SLOT2 = BNH * 128;    // ring slot: one 64-row B atom (8 KB)
constexpr uint32_t MAXST2 = 32;
constexpr uint32_t ROOM2 = 32;           // slots a row's stream buffer may gain per tile

struct __align__(8) Bars2 {
    uint64_t full[MAXST2], empty[MAXST2];
    uint64_t a_full, a_empty;
    uint64_t tm_full[NBUF2], tm_empty[NBUF2];
    uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the variable at shared::cta address `a` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cl_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_remote(uint32_t cl_addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(cl_addr), "r"(bytes)
                 : "memory");
}
// wait without a suspend-time hint: a phase completed by the peer CTA (remote arrive, TMA
// complete_tx, multicast commit) does not wake a thread suspended on the hint promptly
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t parity) {
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
// TMA load into this CTA's shared memory, completing on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_load_2d_cg2(const CUtensorMap* map, uint32_t bar_cl, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar_cl)
        : "memory");
}
template <int KIND>
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    if constexpr (KIND == 0) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    }
}
// completion of this thread's prior MMAs -> arrive on the mbarrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit2(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
template <int KIND>
__host__ __device__ constexpr uint32_t instr_desc2() {   // D f32, K-major A/B, M = 256, N = 128
    return (1u << 4) | ((KIND ? 2u : 0u) << 7) | ((KIND ? 2u : 0u) << 10) | ((BN2 >> 3) << 17) | ((RB2 >> 4) << 24);
}

template <int KIND, int EPL, bool DIAG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTH2, 1)
knn_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmAm, const __grid_constant__ CUtensorMap tmBm, KnnParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    constexpr uint32_t EL = KIND ? 4 : 2;
    constexpr uint32_t ATOM_K = 128 / EL;
    // operand atoms per row are a run-time value (one kernel per precision): NKA full 128-byte
    // atoms + MINI 32-byte atom
    const uint32_t NKA = p.nka, MINI = p.mini;
    const uint32_t nslot = NKA + MINI;
    const uint32_t AHALF = NKA * ATOM + (MINI ? MINIB : 0u);
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + AHALF;
    Bars2* bars = (Bars2*)(sB + p.stages * SLOT2);
    uint8_t* bars_end = (uint8_t*)(bars + 1);
    unsigned long long* s_pair = (unsigned long long*)(bars_end + ((128u - (smem_u32(bars_end) & 127u)) & 127u));
    uint32_t (*s_cnt)[M2] = (uint32_t (*)[M2])(s_pair + M2);           // [NSTR][M2]
    uint8_t* scratch_all = (uint8_t*)(s_pair + M2) + NSTR * M2 * 4;   // NEPI2 x SCRATCH

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t cr = cluster_rank();
    const uint32_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const uint32_t ma = p.n_rows_dev ? *(const volatile uint32_t*)p.n_rows_dev : p.ma;
    const uint32_t n_rb = (ma + RB2 - 1) / RB2;
    constexpr bool PROF = SG_KNN_PROF != 0;
    long long pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto clk = []() -> long long { return PROF ? clock64() : 0ll; };

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; s++) { mbar_init(&bars->full[s], 2); mbar_init(&bars->empty[s], 1); }
        mbar_init(&bars->a_full, 2);
        mbar_init(&bars->a_empty, 1);
        for (uint32_t b = 0; b < NBUF2; b++) { mbar_init(&bars->tm_full[b], 1); mbar_init(&bars->tm_empty[b], 2 * NEPI2); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
        if (MINI) {
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmAm) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmBm) : "memory");
        }
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars->tmem_base)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();   // barriers of both CTAs initialised, TMEM allocated in both
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (lane == 0) {
            const uint32_t lead_a_full = mapa(smem_u32(&bars->a_full), 0);
            uint32_t stage = 0, sph = 0, it = 0;
            for (uint32_t rb = cid; rb < n_rb; rb += ncl, it++) {
                if (it > 0) mbar_wait_cl(&bars->a_empty, (it - 1) & 1);
                mbar_expect_tx_remote(lead_a_full, AHALF);
                for (uint32_t ka = 0; ka < NKA; ka++)
                    tma_load_2d_cg2(&tmA, lead_a_full, sA + ka * ATOM, ka * ATOM_K, rb * RB2 + cr * M2);
                if (MINI) tma_load_2d_cg2(&tmAm, lead_a_full, sA + NKA * ATOM, NKA * ATOM_K, rb * RB2 + cr * M2);
                for (uint32_t ti = 0, t = tile_at(p, rb, 0); ti < p.n_ct; ti++, t = t + 1 == p.n_ct ? 0 : t + 1) {
                    for (uint32_t ka = 0; ka < nslot; ka++) {
                        mbar_wait_cl(&bars->empty[stage], sph ^ 1);
                        uint8_t* slot = sB + stage * SLOT2;
                        const uint32_t lead_full = mapa(smem_u32(&bars->full[stage]), 0);
                        if (DIAG && p.noload) {
                            mbar_arrive_remote(lead_full);
                        } else if (ka < NKA) {
                            mbar_expect_tx_remote(lead_full, SLOT2);
                            tma_load_2d_cg2(&tmB, lead_full, slot, ka * ATOM_K, t * BN2 + cr * BNH);
                        } else {
                            mbar_expect_tx_remote(lead_full, BNH * 32);
                            tma_load_2d_cg2(&tmBm, lead_full, slot, NKA * ATOM_K, t * BN2 + cr * BNH);
                        }
                        if (++stage == p.stages) { stage = 0; sph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA only) =====================
        if (lane == 0 && cr == 0) {
            constexpr uint32_t idesc = instr_desc2<KIND>();
            const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
            uint32_t stage = 0, sph = 0, it = 0, git = 0;
            for (uint32_t rb = cid; rb < n_rb; rb += ncl, it++) {
                mbar_wait_cl(&bars->a_full, it & 1);
                tc_fence_after();
                for (uint32_t ti = 0; ti < p.n_ct; ti++, git++) {
                    const uint32_t buf = git % NBUF2;
                    mbar_wait_cl(&bars->tm_empty[buf], ((git / NBUF2) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t dcol = tmem + buf * BN2;
                    for (uint32_t ka = 0; ka < nslot; ka++) {
                        if (!(DIAG && (p.abl & 2))) mbar_wait_cl(&bars->full[stage], sph);   // abl 2: MMA rate probe
                        tc_fence_after();
                        const uint32_t bslot = b_base + stage * SLOT2;
                        if (ka < NKA) {
#pragma unroll
                            for (uint32_t kk = 0; kk < 4; kk++)
                                tc_mma2<KIND>(dcol, desc_sw128(a_base + ka * ATOM + kk * 32), desc_sw128(bslot + kk * 32),
                                              idesc, (ka | kk) != 0);
                        } else {
                            tc_mma2<KIND>(dcol, desc_sw32(a_base + NKA * ATOM), desc_sw32(bslot), idesc, NKA != 0);
                        }
                        tc_commit2(&bars->empty[stage]);
                        if (++stage == p.stages) { stage = 0; sph ^= 1; }
                    }
                    tc_commit2(&bars->tm_full[buf]);
                }
                tc_commit2(&bars->a_empty);
            }
        }
    } else {
        // ===================== epilogue (both CTAs): fused selection, four column streams =====
        // Same rules as knn_tc.cu: inclusive insertion test against the row's shared (key, id)
        // pair, prefilter per 32-column pass, per-row insertion by one ballot, compaction by bit
        // descent, extrapolated thresholds (I1) checked per row at the end, self column removed
        // in the final phase.
        const uint32_t e = warp - 2, s = e >> 2, q = warp & 3;
        const uint32_t r = q * 32 + lane;                    // row within the CTA's 128
        uint8_t* scratch = scratch_all + e * SCRATCH;
        float* skeys = (float*)scratch;
        uint32_t* hist = (uint32_t*)scratch;
        uint64_t* sortbuf = (uint64_t*)scratch;
        const uint32_t C = p.C;
        auto rowbuf = [&](uint32_t R, uint32_t st) -> uint64_t* {
            return p.cand + (((uint64_t)blockIdx.x * NSTR + st) * M2 + R) * C;
        };
        const uint32_t mybase = (uint32_t)((((uint64_t)blockIdx.x * NSTR + s) * M2 + r) * C);
        uint64_t* warprows = rowbuf(q * 32, s);
        const uint32_t tl = tmem + ((q * 32) << 16) + s * 32;
        const uint64_t PINIT = pair_ord(3.40282347e38f, SG_SENT);
        const uint32_t nbar = NEPI2 * 32;
        // extrapolated target rank per stream (L/4 of the row's top-L expected per stream)
        const float slope = p.alpha100 * 0.0025f * (float)p.L * (float)BN2 / (float)p.mb;
        const uint32_t want_full = p.L + (p.self_exclude ? 1u : 0u);
        const uint32_t kmax_full = p.keep_max > want_full ? p.keep_max : want_full;
        uint32_t lead_tm_empty[NBUF2];
#pragma unroll
        for (uint32_t b = 0; b < NBUF2; b++) lead_tm_empty[b] = mapa(smem_u32(&bars->tm_empty[b]), 0);
        uint32_t git = 0;
        for (uint32_t rb = cid; rb < n_rb; rb += ncl) {
            const uint32_t row = rb * RB2 + cr * M2 + r;
            const bool valid = row < ma;
            uint32_t cnt = 0;
            if (s == 0) s_pair[r] = valid ? PINIT : pair_ord(-__int_as_float(0x7f800000), 0);
            named_bar_sync(1, nbar);
            for (uint32_t ti = 0, t = tile_at(p, rb, 0); ti < p.n_ct; ti++, git++, t = t + 1 == p.n_ct ? 0 : t + 1) {
                const uint32_t buf = git % NBUF2;
                long long c0 = clk();
                mbar_wait_cl(&bars->tm_full[buf], (git / NBUF2) & 1);
                long long c1 = clk();
                pw[0] += c1 - c0;
                tc_fence_after();
                float te = ord2f((uint32_t)(*(volatile unsigned long long*)&s_pair[r] >> 32) + 1u);
                uint32_t want = want_full, kmax = kmax_full, trig = C - ROOM2;
                if (p.alpha100) {
                    const uint32_t rr = (uint32_t)(slope * (float)(ti + 1)) + p.beta;
                    if (rr < want) { want = rr; kmax = want + ((C - ROOM2 - want) >> p.kshift); }
                    if (want + p.eager < trig) trig = want + p.eager;
                }
                uint32_t vv[32];
                tmem_ld32_nowait(tl + buf * BN2, vv);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(lead_tm_empty[buf]);
                c0 = clk();
                pw[1] += c0 - c1;
                const uint32_t col0 = t * BN2 + s * 32;
                const bool hit = min32(vv) < te;
                uint32_t hb = __ballot_sync(0xffffffffu, hit);
                if (DIAG) {
                    if ((vv[0] ^ vv[31]) == 0x7fc00001u) p.out_ids[0] = vv[1];   // keep the loads live
                    if (p.noepi || (p.abl & 1)) hb = 0;
                }
                c1 = clk();
                pw[3] += c1 - c0;
                if (hb) {
                    if (hit) stage_keys(skeys, lane, vv, te, mybase + cnt);
                    __syncwarp();
                    cnt += insert_rows(p, skeys, lane, hb, col0, pw);
                    __syncwarp();
                }
                c0 = clk();
                pw[4] += c0 - c1;
                uint32_t need = __ballot_sync(0xffffffffu, cnt > trig);
                if (need) {
                    do {
                        const int o = __ffs(need) - 1;
                        need &= need - 1;
                        const uint32_t c_o = __shfl_sync(0xffffffffu, cnt, o);
                        const uint32_t R = q * 32 + o;
                        uint64_t* ob = warprows + (uint64_t)o * C;
                        const uint64_t cap = *(volatile unsigned long long*)&s_pair[R];
                        uint32_t kept;
                        uint64_t P = select_pairs<EPL>(ob, c_o, cap, want, kmax, lane, &kept);
                        if (kept > C - ROOM2) P = select_L<EPL>(ob, kept, want, kmax, hist, lane, &kept);
                        if (lane == (uint32_t)o) {
                            cnt = kept;
                            atomicMin(&s_pair[R], (unsigned long long)P);
                            te = ord2f((uint32_t)(P >> 32) + 1u);
                        }
                    } while (need);
                }
                c1 = clk();
                pw[2] += c1 - c0;
            }
            if (DIAG && p.noepi) continue;
            const long long f0 = clk();
            s_cnt[s][r] = cnt;
            named_bar_sync(1, nbar);
            // ---- final: union of the row's four stream buffers without the self column,
            //      exactness check, sorted top-L; the quadrant's 32 rows split over its 4 warps
            for (uint32_t o = 8 * s; o < 8 * s + 8; o++) {
                const uint32_t R = q * 32 + o;
                const uint32_t row_o = rb * RB2 + cr * M2 + R;
                if (row_o >= ma) continue;
                const uint64_t P = s_pair[R];
                uint32_t cc[NSTR];
#pragma unroll
                for (int st = 0; st < (int)NSTR; st++) cc[st] = s_cnt[st][R];
                const uint32_t sid = !p.self_exclude ? SG_SENT
                                     : p.col_map ? p.col_map[p.self_col ? p.self_col[row_o] : row_o]
                                                 : (p.self_col ? p.self_col[row_o] : row_o);
                uint32_t n_le = 0;
#pragma unroll 1
                for (uint32_t st = 0; st < NSTR; st++) {
                    uint64_t* b = rowbuf(R, st);
                    uint32_t c = s_cnt[st][R];
                    // drop the self column (at most one entry carries its id)
                    for (uint32_t i0 = 0; i0 < c && sid != SG_SENT; i0 += 32) {
                        const uint32_t i = i0 + lane;
                        const uint32_t f = __ballot_sync(0xffffffffu, i < c && (uint32_t)b[i] == sid);
                        if (f) {
                            const uint32_t at = i0 + __ffs(f) - 1;
                            const uint64_t last = b[c - 1];
                            __syncwarp();
                            if (lane == 0) b[at] = last;
                            __syncwarp();
                            c--;
                            break;
                        }
                    }
                    if (c > p.L) {   // a stream's own top-L holds all its entries of the row's top-L
                        uint32_t kept;
                        select_pairs<EPL>(b, c, P, p.L, p.L, lane, &kept);
                        if (kept > SORT_MAX / NSTR) {
                            select_L<EPL>(b, kept, p.L, p.L, hist, lane, &kept);
                            kept = p.L;
                        }
                        c = kept;
                    }
                    for (uint32_t i0 = 0; i0 < c; i0 += 32) {
                        const uint32_t i = i0 + lane;
                        n_le += __popc(__ballot_sync(0xffffffffu, i < c && raw2ord(b[i]) <= P));
                    }
                    // stream counts after the final selection, kept in the (row-private) slot
                    if (lane == 0) s_cnt[st][R] = c;
                }
                __syncwarp();
#pragma unroll
                for (int st = 0; st < (int)NSTR; st++) cc[st] = s_cnt[st][R];
                if (p.alpha100 && P != PINIT && n_le < p.L) {
                    if (lane == 0) p.fail_rows[atomicAdd(p.fail_count, 1u)] = row_o;
                    continue;
                }
                const uint64_t orow = p.row_map ? p.row_map[row_o] : row_o;
                const uint64_t* const bl[NSTR] = {rowbuf(R, 0), rowbuf(R, 1), rowbuf(R, 2), rowbuf(R, 3)};
                finish_union_n<SORT_MAX / 32, NSTR>(bl, cc, p.L, sortbuf, p.norm_a[row_o], p.out_ids + orow * p.L,
                                                    p.out_d + orow * p.L, lane);
            }
            named_bar_sync(1, nbar);   // buffers and thresholds are reused by the next row block
            pw[5] += clk() - f0;
        }
    }
    if (PROF && p.prof && lane == 0)
        for (int i = 0; i < 8; i++) atomicAdd(p.prof + warp * 8 + i, (unsigned long long)pw[i]);
    tc_fence_before();
    cluster_sync();   // the peer's MMAs and remote arrivals are done before either CTA leaves
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

template <int KIND, int EPL>
sg_status launch2_t(const CUtensorMap* maps, KnnParams& p, cudaStream_t st) {
    const uint32_t AHALF = p.nka * ATOM + (p.mini ? MINIB : 0u);
    const size_t fixed = AHALF + sizeof(Bars2) + 128 + M2 * 8 + NSTR * M2 * 4 + NEPI2 * SCRATCH + 1024 + 64;
    const size_t budget = 227 * 1024;
    if (fixed + (p.nka + p.mini) * SLOT2 > budget) { set_error("kNN: operand too wide for shared memory"); return SG_ERR_UNSUPPORTED; }
    uint32_t stages = (uint32_t)((budget - fixed) / SLOT2);
    if (stages > MAXST2) stages = MAXST2;
    p.stages = stages;
    const size_t smem = fixed + stages * SLOT2;
    auto kern = knn_tc2_kernel<KIND, EPL, false>;
    if constexpr (KIND == 0) {
        if (p.noepi || p.noload || p.abl) kern = knn_tc2_kernel<KIND, EPL, true>;
    }
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // persistent: as many pairs as can be co-resident (not every SM finds a TPC partner, so
    // this is below num_sms / 2); a pair launched in a second wave would double the time
    static int max_cl = 0;
    if (!max_cl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * (num_sms() / 2), 1, 1);
        cfg.blockDim = dim3(NTH2, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = num_sms() / 2;
        }
        max_cl = n;
        if (getenv("SG_KNN_REPORT")) fprintf(stderr, "[knn2] co-resident CTA pairs: %d\n", max_cl);
    }
    uint32_t ncl = (uint32_t)max_cl;
    if (p.n_rb < ncl) ncl = p.n_rb;
    if (ncl == 0) ncl = 1;
    knn_time_begin(st);
    kern<<<2 * ncl, NTH2, smem, st>>>(maps[0], maps[1], maps[2], maps[3], p);
    SG_LAUNCHED("knn_tc2_kernel");
    knn_time_end(st);
    return SG_OK;
}

}  // namespace

uint32_t cand_cap(uint32_t L);

// The pair kernel: resident row halves (<= 4 operand atoms per row), L <= 128, no probe.
bool knn2_supported(uint32_t nka, uint32_t L, bool probe) {
    static int on = -1;
    // opt-in: measured at half the single-CTA MMA rate (see the file header)
    if (on < 0) { const char* e = getenv("SG_KNN_2CTA"); on = e ? atoi(e) : 0; }
    return on && nka >= 1 && nka <= 4 && L <= 128 && cand_cap(L) <= 256 && !probe;
}

// A: maps[0] A (128 B x 128 rows), maps[2] A mini (32 B x 128 rows); B: maps[1] (128 B x 64
// rows), maps[3] B mini (32 B x 64 rows).
sg_status launch_knn2(const CUtensorMap* maps, KnnParams& p, int esize, int nka, int mini, cudaStream_t st) {
    p.nka = (uint32_t)nka;
    p.mini = (uint32_t)mini;
    p.rb_rows = RB2;
    if (p.C / 32 > 8) { set_error("kNN pair kernel: candidate capacity above 256"); return SG_ERR_UNSUPPORTED; }
    return esize == 4 ? launch2_t<1, 8>(maps, p, st) : launch2_t<0, 8>(maps, p, st);
}

}  // namespace sg
