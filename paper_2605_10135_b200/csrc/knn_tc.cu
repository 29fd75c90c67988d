// a5 — exact kNN: tcgen05 distance tiles + fused per-row top-L (north_star stage 2).
//
// dist(i, j) = |a_i|^2 + |b_j|^2 - 2 a_i.b_j (L2) or -a_i.b_j (IP) (reading R2).  The whole
// per-column part of the key  key(i, j) = |b_j|^2 - 2 a_i.b_j  is one dense contraction: the
// operands are augmented (gather.cu) so that  A_i = [a_i, 1, 2048, 2048]  and
// B_j = [-2 b_j, c0, c1, 2048 c2]  with |b_j|^2 = c0 + 2^11 c1 + 2^22 c2 (f16-exact pieces), so
// the tensor-core accumulator IS the key (exact in fp32 for integer data: every partial sum is
// an integer below 2^24).  dist = |a_i|^2 + key is formed once per output.
//
// Pipeline (persistent, one CTA per SM, 18 warps).  A CTA owns a 256-row block (f16; 128 for
// tf32) held resident in shared memory as 128-row halves (NKA 128B-swizzle atoms + an optional
// 32B-swizzle "mini" atom for the K tail); every 128-column B tile streamed in is used by both
// halves (two M=128, N=128 MMAs), which halves the operand bytes per flop that L2 must deliver.
// Rows wider than 4 atoms use the streamed-A instantiation (NKA = 0): A and B atoms share the
// ring slots and one 128-row accumulator.
//   warp 0: TMA producer (A block, then the B tiles through a ring of 16 KB slots).
//   warp 1: TMEM allocator + single-thread tcgen05.mma issuer; accumulators [half][buffer] of
//           128 columns, 2 x 2 = all 512 columns, so a tile's MMAs overlap the previous drain.
//   warps 2..17: epilogue in two column streams (columns [64 s, 64 s + 64) of every tile);
//           warp (q, a, s) owns rows a*128 + q*32 + lane (TMEM lane quadrant q of half a).  Per
//           32-column pass a thread (= one row) takes the minimum of its 32 keys (16 FMNMX3) and
//           compares it with its row threshold; only the rows that pass (a few % after the first
//           tiles) stage their keys in shared memory, and the warp then takes those rows one at
//           a time, lane j testing column j: one ballot per row, the passing
//           (key bits << 32 | id) words appended to consecutive slots of the row's (row, stream)
//           buffer (global, L2 resident).  Both passes of a tile are loaded (and the TMEM
//           buffer handed back to the MMA) before any insertion or compaction.  A buffer above
//           its trigger is compacted by ballot-count bit descent (select_pairs); the row
//           threshold is one (key, id) pair in shared memory shared by both streams (atomicMin).
//           The self column is inserted like any other and removed in the final phase.
//           Thresholds are extrapolated from the fraction of columns seen (I1); the final phase
//           checks each row (>= L union entries at or below the pair), selects and sorts its
//           top-L, and lists the rows that fail for the fallback launch (rank-L thresholds).
#include "knn_common.cuh"

namespace sg {
namespace {

// ----------------------------------------------------------------- the kernel
constexpr uint32_t NEPI_R = 16;                         // epilogue warps (2 column streams x 8)
constexpr uint32_t NTHREADS_R = 64 + NEPI_R * 32;
static_assert(BN == 128, "the epilogue gives each column stream two 32-column passes per tile");

constexpr uint32_t ROOM = 64;   // candidate-buffer slots a row may gain between compactions (one tile)

// diagnostics instantiation: raw accumulator dump (probe) / keep the loads live (noepi)
__device__ __forceinline__ void diag_pass(const KnnParams& p, const uint32_t (&v)[32], uint32_t col0, uint32_t row,
                                          bool valid) {
    if (p.noepi) {
        if ((v[0] ^ v[31]) == 0x7fc00001u) p.out_ids[0] = v[1];
    } else if (p.probe && valid) {
#pragma unroll
        for (int j = 0; j < 32; j++)
            if (col0 + j < p.mb) p.probe[(uint64_t)row * p.mb + col0 + j] = __uint_as_float(v[j]);
    }
}

// DIAG: the instantiation that honours the probe / diagnostics switches (raw accumulator dump,
// stubbed epilogue, ablations); production launches use DIAG = false and skip those tests.
template <int KIND, int NKA, int MINI, int EPL, bool DIAG>
__global__ void __launch_bounds__(NTHREADS_R, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmAm, const __grid_constant__ CUtensorMap tmBm, KnnParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    constexpr uint32_t EL = KIND ? 4 : 2;                  // bytes per element
    constexpr uint32_t ATOM_K = 128 / EL;                  // elements per 128B atom
    // NKA == 0: streamed-A mode for wide operands (A does not fit in shared memory): every ring
    // slot carries one K atom of B (column tile) and of A (128-row block), the atom count is read
    // at run time (p.nka), one 128-row accumulator
    constexpr bool SA = NKA == 0;
    const uint32_t nka = SA ? p.nka : (uint32_t)NKA;
    const uint32_t nslot = nka + MINI;                     // ring slots per column tile
    constexpr uint32_t SLOTB = SA ? 2 * SLOT : SLOT;       // ring slot bytes (B atom | A atom)
    // f16 operands keep both 128-row halves of A resident; tf32 (wider A) keeps one
    constexpr uint32_t NACC = (KIND == 0 && !SA) ? NACC_MAX : 1;
    constexpr uint32_t RB = MSUB * NACC;                  // rows per row block of this instantiation
    constexpr uint32_t NBUF = 512 / (NACC * BN);
    constexpr uint32_t AHALF = SA ? 0u : NKA * ATOM + (MINI ? MINIB : 0u);   // smem bytes of one resident half
    // offsets from smem_raw (not integer casts) so the compiler keeps shared-space accesses (LDS/STS)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                                    // [NACC][NKA atoms + mini] (SS mode)
    uint8_t* sB = smem + NACC * AHALF;
    Bars* bars = (Bars*)(sB + p.stages * SLOTB);
    uint8_t* bars_end = (uint8_t*)(bars + 1);
    unsigned long long* s_pair = (unsigned long long*)(bars_end + ((128u - (smem_u32(bars_end) & 127u)) & 127u));
    uint32_t (*s_cnt)[BM] = (uint32_t (*)[BM])(s_pair + BM);          // [2][BM] stream counts
    uint8_t* scratch_all = (uint8_t*)(s_pair + BM) + 2 * BM * 4;       // NEPI_R x SCRATCH

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // fallback launch: the number of A rows is known only on the device
    const uint32_t ma = p.n_rows_dev ? *(const volatile uint32_t*)p.n_rows_dev : p.ma;
    const uint32_t n_rb = (ma + RB - 1) / RB;
    constexpr bool PROF = SG_KNN_PROF != 0;
    long long pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // cycle counters + event counts (PROF builds only)
    auto clk = []() -> long long { return PROF ? clock64() : 0ll; };

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; s++) { mbar_init(&bars->full[s], 1); mbar_init(&bars->empty[s], 1); }
        mbar_init(&bars->a_full, 1);
        mbar_init(&bars->a_empty, 1);
        for (uint32_t b = 0; b < NBUF_MAX; b++) { mbar_init(&bars->tm_full[b], 1); mbar_init(&bars->tm_empty[b], 8 * NACC); }
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
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bars->tmem_base)),
                     "r"(512u));
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
            for (uint32_t rb = blockIdx.x; rb < n_rb; rb += gridDim.x, it++) {
                if (!SA) {
                    if (it > 0) mbar_wait(&bars->a_empty, (it - 1) & 1);
                    mbar_expect_tx(&bars->a_full, NACC * AHALF);
                }
                for (uint32_t a = 0; a < NACC && !SA; a++) {
                    uint8_t* base = sA + a * AHALF;
                    for (int ka = 0; ka < NKA; ka++)
                        tma_load_2d(&tmA, &bars->a_full, base + ka * ATOM, ka * ATOM_K, rb * RB + a * MSUB);
                    if (MINI) tma_load_2d(&tmAm, &bars->a_full, base + NKA * ATOM, NKA * ATOM_K, rb * RB + a * MSUB);
                }
                for (uint32_t ti = 0, t = tile_at(p, rb, 0); ti < p.n_ct; ti++, t = t + 1 == p.n_ct ? 0 : t + 1) {
                    long long w0 = clk();
#pragma unroll
                    for (uint32_t ka = 0; ka < nslot; ka++) {
                        mbar_wait(&bars->empty[stage], sph ^ 1);
                        uint8_t* slot = sB + stage * SLOTB;
                        if (DIAG && p.noload) {
                            mbar_arrive(&bars->full[stage]);
                        } else if (ka < nka) {
                            mbar_expect_tx(&bars->full[stage], SA ? BATOM + ATOM : BATOM);
                            tma_load_2d(&tmB, &bars->full[stage], slot, ka * ATOM_K, t * BN);
                            if (SA) tma_load_2d(&tmA, &bars->full[stage], slot + SLOT, ka * ATOM_K, rb * RB);
                        } else {
                            mbar_expect_tx(&bars->full[stage], SA ? BMINI + MINIB : BMINI);
                            tma_load_2d(&tmBm, &bars->full[stage], slot, nka * ATOM_K, t * BN);
                            if (SA) tma_load_2d(&tmAm, &bars->full[stage], slot + SLOT, nka * ATOM_K, rb * RB);
                        }
                        if (++stage == p.stages) { stage = 0; sph ^= 1; }
                    }
                    pw[0] += clk() - w0;
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idesc = instr_desc<KIND>();
            const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
            uint32_t stage = 0, sph = 0, it = 0, git = 0;
            for (uint32_t rb = blockIdx.x; rb < n_rb; rb += gridDim.x, it++) {
                if (!SA) mbar_wait(&bars->a_full, it & 1);
                tc_fence_after();
                for (uint32_t ti = 0; ti < p.n_ct; ti++, git++) {
                    const uint32_t buf = git % NBUF;
                    const long long w0 = clk();
                    mbar_wait(&bars->tm_empty[buf], ((git / NBUF) & 1) ^ 1);
                    pw[0] += clk() - w0;
                    tc_fence_after();
#pragma unroll
                    for (uint32_t ka = 0; ka < nslot; ka++) {
                        const long long w1 = clk();
                        mbar_wait(&bars->full[stage], sph);
                        pw[1] += clk() - w1;
                        tc_fence_after();
                        const uint32_t bslot = b_base + stage * SLOTB;
#pragma unroll
                        for (uint32_t a = 0; a < NACC; a++) {
                            const uint32_t dcol = tmem + (a * NBUF + buf) * BN;
                            const uint32_t abase = a_base + a * AHALF;
                            if constexpr (SA) {
                                const uint32_t aslot = bslot + SLOT;   // this K atom of A
                                if (ka < nka) {
#pragma unroll
                                    for (uint32_t kk = 0; kk < 4; kk++)
                                        tc_mma<KIND>(dcol, desc_sw128(aslot + kk * 32), desc_sw128(bslot + kk * 32), idesc,
                                                     (ka | kk) != 0);
                                } else {
                                    tc_mma<KIND>(dcol, desc_sw32(aslot), desc_sw32(bslot), idesc, nka != 0);
                                }
                            } else {
                                if (ka < NKA) {
#pragma unroll
                                    for (uint32_t kk = 0; kk < 4; kk++)
                                        tc_mma<KIND>(dcol, desc_sw128(abase + ka * ATOM + kk * 32),
                                                     desc_sw128(bslot + kk * 32), idesc, (ka | kk) != 0);
                                } else {
                                    tc_mma<KIND>(dcol, desc_sw32(abase + NKA * ATOM), desc_sw32(bslot), idesc, NKA != 0);
                                }
                            }
                        }
                        tc_commit(&bars->empty[stage]);
                        if (++stage == p.stages) { stage = 0; sph ^= 1; }
                    }
                    tc_commit(&bars->tm_full[buf]);
                }
                if (!SA) tc_commit(&bars->a_empty);
            }
        }
    } else {
        // ===================== epilogue: fused selection, two column streams =====================
        // Warps 2..17.  Stream s takes columns [64 s, 64 s + 64) of every tile (both streams drain
        // the same TMEM buffer while the MMA fills the other), q = warp % 4 is the TMEM lane
        // quadrant, a the row half; thread = one row.  Each (row, stream) has its
        // own candidate buffer; the row threshold is ONE (key, id) pair in shared memory shared by
        // the two streams and lowered with atomicMin when either compacts.  The insertion test is
        // inclusive (key <= thr: equal keys with a larger id may enter, above the pair), so each
        // buffer holds every column of its stream at or below the final pair T, for any order; a
        // row is exact iff >= L union entries lie at or below T (always so with rank-L thresholds;
        // with extrapolated ones a row that misses it goes to the fallback launch).
        const uint32_t e = warp - 2, s = e >> 3, q = warp & 3, a = (e & 7) >> 2;
        const uint32_t r = a * MSUB + q * 32 + lane;         // row within the block
        uint8_t* scratch = scratch_all + (s * 4 * NACC + (e & 7)) * SCRATCH;   // active warps only
        float* skeys = (float*)scratch;                      // [32][KSTRIDE] staged keys (+ te, slot)
        uint32_t* hist = (uint32_t*)scratch;                 // 256 (aliases skeys)
        uint64_t* sortbuf = (uint64_t*)scratch;              // 512 (aliases skeys)
        const uint32_t C = p.C;
        const uint32_t keep_max = p.keep_max;                // in-loop compaction target (>= L)
        auto rowbuf = [&](uint32_t R, uint32_t st) -> uint64_t* {
            return p.cand + (((uint64_t)blockIdx.x * 2 + st) * BM + R) * C;
        };
        // word offset of this row's stream buffer from p.cand (the buffers span < 2^32 words)
        const uint32_t mybase = (uint32_t)((((uint64_t)blockIdx.x * 2 + s) * BM + r) * C);
        uint64_t* warprows = rowbuf(a * MSUB + q * 32, s);
        const uint32_t tl = tmem + ((q * 32) << 16) + a * NBUF * BN;
        const uint64_t PINIT = pair_ord(3.40282347e38f, SG_SENT);   // every finite key passes, +inf not
        const uint32_t nbar = NACC * 8 * 32;                 // active epilogue threads
        // extrapolated target rank per stream after tile ti: slope * (ti + 1) + beta
        const float slope = p.alpha100 * 0.005f * (float)p.L * (float)BN / (float)p.mb;
        // binomial target (p.z100 > 0): after a fraction f of the columns a stream holds on average
        // L f / 2 of the row's top-L, with variance L f / 2 (1 - f / 2)
        const float fstep = (float)BN / (float)p.mb, mu_step = 0.5f * (float)p.L * fstep, zf = 0.01f * (float)p.z100;
        // the self column is inserted like any other (its key is the row's smallest) and removed
        // in the final phase; with plain rank-L thresholds it takes one of the kept ranks
        const uint32_t want_full = p.L + (p.self_exclude ? 1u : 0u);
        const uint32_t kmax_full = keep_max > want_full ? keep_max : want_full;
        uint32_t git = 0;
        for (uint32_t rb = blockIdx.x; rb < n_rb && a < NACC; rb += gridDim.x) {
            const uint32_t row = rb * RB + r;
            const bool valid = row < ma;
            uint32_t cnt = 0;
            if (s == 0) s_pair[r] = valid ? PINIT : pair_ord(-__int_as_float(0x7f800000), 0);
            named_bar_sync(1, nbar);
            for (uint32_t ti = 0, t = tile_at(p, rb, 0); ti < p.n_ct; ti++, git++, t = t + 1 == p.n_ct ? 0 : t + 1) {
                const uint32_t buf = git % NBUF;
                long long c0 = clk();
                mbar_wait(&bars->tm_full[buf], (git / NBUF) & 1);
                long long c1 = clk();
                pw[0] += c1 - c0;
                tc_fence_after();
                const uint32_t tb = tl + buf * BN;
                // the row threshold (possibly lowered by the other stream) for this tile:
                // te = next_up(thr) is ord + 1 in the ordered key space, so key < te is key <= thr
                float te = ord2f((uint32_t)(*(volatile unsigned long long*)&s_pair[r] >> 32) + 1u);
                // compaction target rank per stream for this tile: L, or (extrapolated) the rank for
                // the fraction of columns seen; trigger: buffer full, or `eager` above the target
                uint32_t want = want_full, kmax = kmax_full, trig = C - ROOM;
                if (p.alpha100) {
                    uint32_t rr;
                    if (p.z100) {   // binomial target: mean + z sd of this stream's share of the top-L
                        const float mu = mu_step * (float)(ti + 1), fr = fstep * (float)(ti + 1);
                        rr = (uint32_t)(mu + zf * sqrtf(mu * fmaxf(1.f - 0.5f * fr, 0.f))) + p.beta;
                    } else {
                        rr = (uint32_t)(slope * (float)(ti + 1)) + p.beta;
                    }
                    if (rr < want) { want = rr; kmax = want + ((C - ROOM - want) >> p.kshift); }
                    if (want + p.eager < trig) trig = want + p.eager;
                }
                // this stream's two 32-column passes.  One TMEM load each (18 warps leave 96
                // registers per thread, too few to hold both); the rows whose prefilter hits stage
                // pass 0's keys in shared memory so that pass 1 is loaded and the buffer handed
                // back to the MMA before any insertion or compaction work
                const uint32_t cb = t * BN + s * 64;   // first column of pass 0
                uint32_t vv[32];
                tmem_ld32_nowait(tb + s * 64, vv);
                tmem_wait_ld();
                c0 = clk();
                pw[1] += c0 - c1;
                bool hit = min32(vv) < te;   // prefilter: smallest key of the pass vs the threshold
                uint32_t hb0 = __ballot_sync(0xffffffffu, hit);
                if (hit) stage_keys(skeys, lane, vv, te, mybase + cnt);
                if (DIAG) diag_pass(p, vv, cb, row, valid);
                c1 = clk();
                pw[3] += c1 - c0;
                tmem_ld32_nowait(tb + s * 64 + 32, vv);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->tm_empty[buf]);
                c0 = clk();
                pw[1] += c0 - c1;
                hit = min32(vv) < te;
                uint32_t hb1 = __ballot_sync(0xffffffffu, hit);
                if (DIAG) {
                    diag_pass(p, vv, cb + 32, row, valid);
                    if (p.noepi || p.probe || (p.abl & 1)) hb0 = hb1 = 0;
                }
                c1 = clk();
                pw[3] += c1 - c0;
                if (hb0) {
                    __syncwarp();
                    cnt += insert_rows(p, skeys, lane, hb0, cb, pw);
                }
                if (hb1) {
                    __syncwarp();   // pass 0's staged keys are consumed
                    if (hit) stage_keys(skeys, lane, vv, te, mybase + cnt);
                    __syncwarp();
                    cnt += insert_rows(p, skeys, lane, hb1, cb + 32, pw);
                }
                SG_DCHECK(cnt <= C);   // a tile's two passes fit the ROOM above the trigger
                c0 = clk();
                pw[4] += c0 - c1;
                // make room for the next tile (<= ROOM more entries): compact rows whose buffer
                // passed the trigger to the target rank per stream (L, or the extrapolated rank
                // for the fraction seen) under the row threshold, and lower the shared pair
                // (extrapolated mode: also eagerly, once a stream holds `eager` entries above its
                // target rank, so the shared threshold follows the fraction of columns seen)
                uint32_t need = __ballot_sync(0xffffffffu, cnt > trig);
                if (need) {
                    do {
                        const int o = __ffs(need) - 1;
                        need &= need - 1;
                        const uint32_t c_o = __shfl_sync(0xffffffffu, cnt, o);
                        const uint32_t R = a * MSUB + q * 32 + o;
                        uint64_t* ob = warprows + (uint64_t)o * C;
                        const uint64_t cap = *(volatile unsigned long long*)&s_pair[R];
                        uint32_t kept;
                        uint64_t P = select_pairs<EPL>(ob, c_o, cap, want, kmax, lane, &kept);
                        if (kept > C - ROOM)   // massive ties on the threshold key: split them by id
                            P = select_L<EPL>(ob, kept, want, kmax, hist, lane, &kept);
                        SG_DCHECK(kept <= C - ROOM);
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
            if (DIAG && (p.probe || p.noepi)) continue;
            const long long f0 = clk();
            s_cnt[s][r] = cnt;
            named_bar_sync(1, nbar);
            // ---- final: union of the row's two stream buffers without the self column, exactness
            //      check, sorted top-L; the 32 rows of this (q, a) group are split between its two
            //      stream warps
            for (uint32_t o = 16 * s; o < 16 * s + 16; o++) {
                const uint32_t R = a * MSUB + q * 32 + o;
                const uint32_t row_o = rb * RB + R;
                if (row_o >= ma) continue;
                const uint64_t P = s_pair[R];
                uint64_t* bb[2] = {rowbuf(R, 0), rowbuf(R, 1)};
                uint32_t cc[2] = {s_cnt[0][R], s_cnt[1][R]};
                if (p.self_exclude) {
                    // reported id of the self column; at most one entry carries it
                    const uint32_t sc = p.self_col ? p.self_col[row_o] : row_o;
                    const uint32_t sid = p.col_map ? p.col_map[sc] : sc;
#pragma unroll
                    for (int st = 0; st < 2; st++) {
                        for (uint32_t i0 = 0; i0 < cc[st]; i0 += 32) {
                            const uint32_t i = i0 + lane;
                            const uint32_t f = __ballot_sync(0xffffffffu, i < cc[st] && (uint32_t)bb[st][i] == sid);
                            if (f) {
                                const uint32_t at = i0 + __ffs(f) - 1;
                                const uint64_t last = bb[st][cc[st] - 1];
                                __syncwarp();
                                if (lane == 0) bb[st][at] = last;
                                __syncwarp();
                                cc[st]--;
                                break;
                            }
                        }
                    }
                }
                uint32_t n_le = 0;
#pragma unroll
                for (int st = 0; st < 2; st++) {
                    uint32_t kept;
                    if (cc[st] > p.L) {   // a stream's own top-L holds all its entries of the row's top-L
                        select_pairs<EPL>(bb[st], cc[st], P, p.L, p.L, lane, &kept);
                        if (kept > SORT_MAX / 2) {
                            select_L<EPL>(bb[st], kept, p.L, p.L, hist, lane, &kept);
                            kept = p.L;
                        }
                        cc[st] = kept;
                    }
                    for (uint32_t i0 = 0; i0 < cc[st]; i0 += 32) {
                        const uint32_t i = i0 + lane;
                        n_le += __popc(__ballot_sync(0xffffffffu, i < cc[st] && raw2ord(bb[st][i]) <= P));
                    }
                }
                if (p.alpha100 && P != PINIT && n_le < p.L) {
                    // extrapolated threshold was too tight for this row: recompute it (fallback)
                    if (lane == 0) p.fail_rows[atomicAdd(p.fail_count, 1u)] = row_o;
                    continue;
                }
                const uint64_t orow = p.row_map ? p.row_map[row_o] : row_o;
                finish_union<SORT_MAX / 32>(bb[0], cc[0], bb[1], cc[1], p.L, sortbuf, p.norm_a[row_o],
                                            p.out_ids + orow * p.L, p.out_d + orow * p.L, lane);
            }
            named_bar_sync(1, nbar);   // buffers and thresholds are reused by the next row block
            pw[5] += clk() - f0;
        }
    }
    if (PROF && p.prof && lane == 0)
        for (int i = 0; i < 8; i++) atomicAdd(p.prof + warp * 8 + i, (unsigned long long)pw[i]);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

}  // namespace

// Candidate buffer words per row: room for one tile above the kept set (>= L + 2 ROOM).
// SG_KNN_C overrides (tuning); SG_KNN_KEEP=1 makes in-loop compaction exact (keep L).
uint32_t cand_cap(uint32_t L) {
    static int env = -1;
    if (env < 0) { const char* e = getenv("SG_KNN_C"); env = e ? atoi(e) : 0; }
    uint32_t c = 256;
    while (c < 2 * L && c < 1024) c <<= 1;
    if (env > 0) c = (uint32_t)env < 1024u ? (uint32_t)env : 1024u;
    while (c < L + 2 * ROOM) c <<= 1;   // the trigger C - ROOM stays above the kept set (>= L + 1)
    return c;
}

namespace {
uint32_t keep_target(uint32_t L, uint32_t C) {
    static int env = -1;
    if (env < 0) { const char* e = getenv("SG_KNN_KEEP"); env = e ? atoi(e) : 0; }
    return env == 1 ? L : L + (C - ROOM - L) / 8;
}

template <int KIND, int NKA, int MINI, int EPL>
sg_status launch_t(const CUtensorMap* maps, KnnParams& p, cudaStream_t st) {
    constexpr bool SA = NKA == 0;
    constexpr uint32_t AHALF = SA ? 0u : NKA * ATOM + (MINI ? MINIB : 0u);
    constexpr uint32_t NACC = (KIND == 0 && !SA) ? NACC_MAX : 1;
    constexpr uint32_t SLOTB = SA ? 2 * SLOT : SLOT;
    const size_t fixed = NACC * AHALF + sizeof(Bars) + 128 + BM * 8 + 2 * BM * 4 + 8 * NACC * SCRATCH + 1024 + 64;
    const size_t budget = 227 * 1024;
    const size_t min_slots = SA ? 2 : NKA + MINI;
    if (fixed + min_slots * SLOTB > budget) { set_error("kNN: operand too wide for shared memory"); return SG_ERR_UNSUPPORTED; }
    uint32_t stages = (uint32_t)((budget - fixed) / SLOTB);
    if (stages > MAX_STAGES) stages = MAX_STAGES;
    p.stages = stages;
    const size_t smem = fixed + stages * SLOTB;
    // the diagnostics / probe instantiation exists for EPL = 8 only (the probe runs with L = 1 and
    // the diagnostics with L <= 128), which keeps the number of kernels and the build time down
    auto kern = knn_tc_kernel<KIND, NKA, MINI, EPL, false>;
    if constexpr (EPL == 8) {
        if (p.probe || p.noepi || p.noload || p.abl) kern = knn_tc_kernel<KIND, NKA, MINI, EPL, true>;
    } else if (p.probe) {
        set_error("kNN probe: unsupported candidate capacity");
        return SG_ERR_UNSUPPORTED;
    }
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint32_t grid = p.n_rb < (uint32_t)num_sms() ? p.n_rb : (uint32_t)num_sms();
    knn_time_begin(st);
    kern<<<grid, NTHREADS_R, smem, st>>>(maps[0], maps[1], maps[2], maps[3], p);
    SG_LAUNCHED("knn_tc_kernel");
    knn_time_end(st);
    return SG_OK;
}

template <int KIND, int MINI, int EPL>
sg_status launch_nka(int nka, const CUtensorMap* maps, KnnParams& p, cudaStream_t st) {
    // resident-A kernel when the row block fits in shared memory, else streamed A (any width)
    sg_status r = SG_ERR_UNSUPPORTED;
    switch (nka) {
        case 1: r = launch_t<KIND, 1, MINI, EPL>(maps, p, st); break;
        case 2: r = launch_t<KIND, 2, MINI, EPL>(maps, p, st); break;
        case 3: r = launch_t<KIND, 3, MINI, EPL>(maps, p, st); break;
        case 4: r = launch_t<KIND, 4, MINI, EPL>(maps, p, st); break;
    }
    if (r != SG_ERR_UNSUPPORTED) return r;
    p.nka = (uint32_t)nka;
    return launch_t<KIND, 0, MINI, EPL>(maps, p, st);
}

template <int KIND, int EPL>
sg_status launch_mini(int nka, int mini, const CUtensorMap* maps, KnnParams& p, cudaStream_t st) {
    return mini ? launch_nka<KIND, 1, EPL>(nka, maps, p, st) : launch_nka<KIND, 0, EPL>(nka, maps, p, st);
}

}  // namespace

unsigned long long* g_knn_prof = nullptr;
void set_knn_profile(unsigned long long* buf) { g_knn_prof = buf; }

uint32_t knn_row_align() { return BM; }

// transposed kernel (knn_tct.cu): L <= 128, selected unless SG_KNN_T=0
uint32_t knn_t_cap(uint32_t L, bool extrap);
sg_status launch_knn_t(const CUtensorMap* maps, KnnParams& p, int esize, int nka, int mini, cudaStream_t st);
bool knn2_supported(uint32_t nka, uint32_t L, bool probe);
sg_status launch_knn2(const CUtensorMap* maps, KnnParams& p, int esize, int nka, int mini, cudaStream_t st);
static bool use_transposed(uint32_t L) {
    static int on = -1;
    if (on < 0) { const char* e = getenv("SG_KNN_T"); on = e ? atoi(e) : 0; }
    return on && L <= 128;
}
static size_t cand_words_per_cta(uint32_t L) {
    const size_t row_major = 2 * (size_t)BM * cand_cap(L);   // two column streams
    const size_t transposed = use_transposed(L) ? (size_t)BM * 4 * knn_t_cap(L, false) : 0;
    return row_major > transposed ? row_major : transposed;
}

size_t knn_core_workspace(uint32_t L, uint64_t ma, uint32_t d, int prec, int metric) {
    // candidate buffers + fallback state (failed-row list, copy of their A rows)
    return (size_t)num_sms() * cand_words_per_cta(L) * sizeof(uint64_t) + 2 * ((ma + BM) * 4 + 256) +
           operand_bytes(prec, metric, d, ma, SIDE_A) + 8192;
}

namespace {
// A2 row i = A row fail_rows[i] (the rows the extrapolated launch could not finish); the count is
// read on the device, so the fallback needs no host synchronisation.
__global__ void copy_fail_rows(const uint32_t* __restrict__ a, const float* __restrict__ norm, uint32_t words,
                               const uint32_t* __restrict__ fail_rows, const uint32_t* __restrict__ fail_count,
                               uint32_t* __restrict__ a2, float* __restrict__ norm2) {
    const uint32_t cnt = *fail_count;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = warp; i < cnt; i += nw) {
        const uint32_t r = fail_rows[i];
        for (uint32_t w = lane; w < words; w += 32) a2[(uint64_t)i * words + w] = a[(uint64_t)r * words + w];
        if (lane == 0) norm2[i] = norm[r];
    }
}

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

sg_status launch_knn(const Operand& A, const Operand& B, KnnParams& p, cudaStream_t st) {
    CUtensorMap maps[4];
    if (!use_transposed(p.L) && knn2_supported(A.nfull, p.L, p.probe != nullptr)) {
        // CTA-pair kernel (knn_tc2.cu): each CTA loads 64 of every 128 B-tile rows
        SG_TRY(make_map(&maps[0], A.a, A.rows_pad, A.kdim, A.esize, 128, MSUB));
        SG_TRY(make_map(&maps[1], B.b, B.rows_pad, B.kdim, B.esize, 128, BN / 2));
        if (A.mini) {
            SG_TRY(make_map(&maps[2], A.a, A.rows_pad, A.kdim, A.esize, 32, MSUB));
            SG_TRY(make_map(&maps[3], B.b, B.rows_pad, B.kdim, B.esize, 32, BN / 2));
        } else {
            maps[2] = maps[0];
            maps[3] = maps[1];
        }
        return launch_knn2(maps, p, (int)A.esize, (int)A.nfull, (int)A.mini, st);
    }
    SG_TRY(make_map(&maps[0], A.a, A.rows_pad, A.kdim, A.esize, 128, MSUB));
    SG_TRY(make_map(&maps[1], B.b, B.rows_pad, B.kdim, B.esize, 128, BN));
    if (A.mini) {
        SG_TRY(make_map(&maps[2], A.a, A.rows_pad, A.kdim, A.esize, 32, MSUB));
        SG_TRY(make_map(&maps[3], B.b, B.rows_pad, B.kdim, B.esize, 32, BN));
    } else {
        maps[2] = maps[0];
        maps[3] = maps[1];
    }
    const int epl = (int)(p.C / 32);
    const int nka = (int)A.nfull, mini = (int)A.mini;
    if (use_transposed(p.L) && nka <= 4) return launch_knn_t(maps, p, (int)A.esize, nka, mini, st);
    if (A.esize == 4) {
        if (epl <= 8) return launch_mini<1, 8>(nka, mini, maps, p, st);
        if (epl <= 16) return launch_mini<1, 16>(nka, mini, maps, p, st);
        return launch_mini<1, 32>(nka, mini, maps, p, st);
    }
    if (epl <= 8) return launch_mini<0, 8>(nka, mini, maps, p, st);
    if (epl <= 16) return launch_mini<0, 16>(nka, mini, maps, p, st);
    return launch_mini<0, 32>(nka, mini, maps, p, st);
}
}  // namespace

sg_status knn_core(const Operand& A, const Operand& B, int /*metric*/, bool self_exclude, uint32_t L, uint32_t* ids,
                   float* dists, float* probe, Carver& cv, cudaStream_t st, const uint32_t* row_map,
                   const uint32_t* col_map, bool rotate) {
    if (A.kdim != B.kdim || A.esize != B.esize || A.nfull != B.nfull || A.mini != B.mini) {
        set_error("kNN: operand layout mismatch");
        return SG_ERR_INVALID_ARG;
    }
    if (A.rows_pad % BM || B.rows_pad % BN) { set_error("kNN: operand rows not padded"); return SG_ERR_INVALID_ARG; }
    KnnParams p{};
    p.norm_a = A.norm;
    p.a_words = A.kdim * A.esize / 4;
    p.C = cand_cap(L);
    p.keep_max = keep_target(L, p.C);
    p.cand = cv.take<uint64_t>((size_t)num_sms() * cand_words_per_cta(L));
    if (!cv.ok()) { set_error("kNN: workspace too small"); return SG_ERR_WORKSPACE; }
    p.out_ids = ids;
    p.out_d = dists;
    p.probe = probe;
    p.prof = g_knn_prof;
    p.ma = (uint32_t)A.rows;
    p.mb = (uint32_t)B.rows;
    p.L = L;
    p.rb_rows = MSUB * (A.esize == 2 ? NACC_MAX : 1);
    p.n_rb = (uint32_t)(A.rows_pad / p.rb_rows);
    p.n_ct = (uint32_t)(B.rows_pad / BN);
    p.self_exclude = self_exclude ? 1 : 0;
    p.row_map = row_map;
    p.col_map = col_map;
    p.rotate = rotate ? 1 : 0;
    static const int tb = env_int("SG_TBACK", 8), ne = env_int("SG_KNN_NOEPI", 0), nl = env_int("SG_KNN_NOLOAD", 0),
                     ab = env_int("SG_KNN_ABL", 0), alpha = env_int("SG_KNN_ALPHA", 150),
                     beta = env_int("SG_KNN_BETA", -1), report = env_int("SG_KNN_REPORT", 0),
                     eager = env_int("SG_KNN_EAGER", -1);
    p.t_back = (uint32_t)tb;
    const bool main_sweep = L > 1 && !probe;          // not the spatial-order assignment pass
    p.noepi = ne && main_sweep;
    p.noload = nl && p.noepi;
    p.abl = main_sweep ? ab : 0;
    // extrapolated thresholds need columns in an order unrelated to the rows' positions
    const bool extrap = main_sweep && !rotate && !row_map && alpha > 0 && B.rows >= 4ull * L && !p.noepi;
    const bool tr = use_transposed(L);
    if (tr) p.C = knn_t_cap(L, extrap);
    if (!extrap) return launch_knn(A, B, p, st);

    uint32_t* fail_count = cv.take<uint32_t>(1);
    uint32_t* fail_rows = cv.take<uint32_t>(A.rows_pad);
    Operand A2 = A;
    A2.a = cv.take<uint8_t>((size_t)A.rows_pad * A.kdim * A.esize);
    A2.norm = cv.take<float>(A.rows_pad);
    if (!cv.ok()) { set_error("kNN: workspace too small (fallback)"); return SG_ERR_WORKSPACE; }
    SG_CUDA(cudaMemsetAsync(fail_count, 0, sizeof(uint32_t), st));
    p.alpha100 = (uint32_t)alpha;
    p.beta = (uint32_t)(beta >= 0 ? beta : tr ? 6 : knn2_supported(A.nfull, L, false) ? 8 : 12);   // per column stream
    p.eager = (uint32_t)(eager >= 0 ? eager : tr ? 16 : 64);
    static const int z100 = env_int("SG_KNN_Z", 0);   // binomial thresholds: z score x 100 (0 = linear)
    p.z100 = (uint32_t)(z100 > 0 ? z100 : 0);
    static const int kshift = env_int("SG_KNN_KSHIFT", 3);   // in-loop compaction keeps want + room >> kshift
    p.kshift = (uint32_t)(kshift >= 0 && kshift < 16 ? kshift : 3);
    p.fail_count = fail_count;
    p.fail_rows = fail_rows;
    SG_TRY(launch_knn(A, B, p, st));
    if (report) {
        uint32_t h = 0;
        cudaMemcpyAsync(&h, fail_count, sizeof(h), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "[knn] extrapolated thresholds: %u of %llu rows recomputed\n", h, (unsigned long long)A.rows);
    }
    // fallback: the failed rows, plain rank-L thresholds, results to their own output rows
    copy_fail_rows<<<num_sms() * 4, 256, 0, st>>>((const uint32_t*)A.a, A.norm, p.a_words, fail_rows, fail_count,
                                                  (uint32_t*)A2.a, A2.norm);
    SG_LAUNCHED("copy_fail_rows");
    KnnParams p2 = p;
    p2.alpha100 = 0;
    if (tr) p2.C = knn_t_cap(L, false);
    p2.norm_a = A2.norm;
    p2.n_rows_dev = fail_count;
    p2.row_map = fail_rows;
    p2.self_col = self_exclude ? fail_rows : nullptr;
    return launch_knn(A2, B, p2, st);
}

}  // namespace sg
