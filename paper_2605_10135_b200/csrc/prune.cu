// a6 — rank-based detour-count prune (north_star stage 3; reading R10, CAGRA prior art).
//
// One warp per node a.  N[a] (L ids) goes into a shared-memory cuckoo table id -> rank (two
// 8-byte loads and two compares per lookup) and a 2048-bit register filter.  For each rank r_ad
// the warp reads the 2-hop row N[delta] (delta = N[a][r_ad]) with one vector load per row
// (4 rows in flight per lane batch) and, for every b in it that
// is also in N[a] at rank r_ab with max(r_ad, r_db) < r_ab (rule P; rule 1: r_ad < r_ab),
// increments cnt[r_ab] in shared memory.  The ranks are then ordered stably by (cnt, rank)
// (sentinel ranks last) with a counting sort and the first R written with their kNN distances.
// Bit-exact with the oracle (integer work only).
#include <stdlib.h>

#include "common.cuh"

namespace sg {
namespace {



// Membership table of N[a]: NB = LP/2 buckets of 8 slots (keys u32, ranks u8), one hash; a
// lookup reads the whole bucket with two 16-byte loads and compares 8 keys, with no probe loop (a
// probing table makes every lane wait for the warp's longest chain).  Keys that find their
// bucket full go to a small stash, scanned only when it is not empty (warp-uniform).
constexpr uint32_t STASH = 32;   // *nst > STASH flags a node whose table insertion did not settle

// Cuckoo table of N[a]: 8 NB = 4 L_pad slots of (id << 32 | rank), two hashes; a lookup reads
// both candidate slots (two 8-byte loads, two compares, no probe loop).  Parallel insertion
// (atomicExch, evicted entries move to their other slot) at load 1/4; a node whose insertion
// does not settle takes the exact slow path.
__device__ __forceinline__ uint32_t ch1(uint32_t id, uint32_t bits) { return (id * 0x9E3779B1u) >> (32 - bits); }
__device__ __forceinline__ uint32_t ch2(uint32_t id, uint32_t bits) {
    const uint32_t h = ((id ^ (id >> 16)) * 0x85EBCA6Bu) >> (32 - bits);
    return h == ch1(id, bits) ? h ^ 1u : h;
}
__device__ __forceinline__ uint32_t lookup(const uint64_t* tab, uint32_t bits, uint32_t b) {
    const uint64_t e1 = tab[ch1(b, bits)], e2 = tab[ch2(b, bits)];
    // an empty slot holds ~0: its low word is "no rank", so a SENT id (never inserted) misses
    return (uint32_t)(e1 >> 32) == b ? (uint32_t)e1 : (uint32_t)(e2 >> 32) == b ? (uint32_t)e2 : 0xFFFFFFFFu;
}

constexpr uint32_t QCAP = 256;   // lookup queue entries per warp (flushed every 256 / (32 LPL) rows)

// 2-hop rows r0..r0+3 of N[a]: lane holds ids [LPL lane, LPL lane + LPL) of each row (r_db =
// LPL lane + q), one vector load per row when the rows are full (L = 32 LPL)
template <int LPL>
__device__ __forceinline__ void load_rows(const uint32_t* __restrict__ knn, const uint32_t* na, uint32_t r0, uint32_t L,
                                          uint32_t lane, uint32_t (&bv)[4][LPL]) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
        const uint32_t dl = r0 + u < L ? na[r0 + u] : SG_SENT;
        const uint32_t* row = knn + (uint64_t)dl * L + LPL * lane;
        bool done = false;
        if (dl == SG_SENT) {
#pragma unroll
            for (int q = 0; q < LPL; q++) bv[u][q] = SG_SENT;
            done = true;
        } else if (L == 32 * LPL) {
            if constexpr (LPL == 4) {
                const uint4 v = __ldg((const uint4*)row);
                bv[u][0] = v.x; bv[u][1] = v.y; bv[u][2] = v.z; bv[u][3] = v.w;
                done = true;
            } else if constexpr (LPL == 2) {
                const uint2 v = __ldg((const uint2*)row);
                bv[u][0] = v.x; bv[u][1] = v.y;
                done = true;
            }
        }
        if (!done) {
#pragma unroll
            for (int q = 0; q < LPL; q++) bv[u][q] = LPL * lane + q < L ? __ldg(row + q) : SG_SENT;
        }
    }
}

// per-warp shared-memory layout (byte offsets, 16-byte aligned pieces)
template <int LPL>
struct PruneLayout {
    static constexpr uint32_t LP = LPL * 32, NB = LP / 2;
    static constexpr int FLUSH = QCAP / (32 * LPL) < 4 ? QCAP / (32 * LPL) : 4;
    static constexpr uint32_t al(size_t v) { return (uint32_t)((v + 15) / 16 * 16); }
    static constexpr uint32_t BKEYS = 0;                  // cuckoo table: 8 NB slots of 8 bytes
    static constexpr uint32_t NST = al(BKEYS + NB * 64);
    static constexpr uint32_t BLOOM = al(NST + 16);
    static constexpr uint32_t CNT = al(BLOOM + 256);
    static constexpr uint32_t NA = al(CNT + LP * 4);
    static constexpr uint32_t OFF = al(NA + LP * 4);
    static constexpr uint32_t STG = al(OFF + (LP + 1) * 4);
    static constexpr uint32_t QE = al(STG + 32 * FLUSH * LPL * 4);
    static constexpr uint32_t PER = al(QE + QCAP * 8);
};

template <int LPL, int PW, int RULE>   // ranks per lane = L_pad / 32; warps (nodes) per CTA; prune rule
__global__ void __launch_bounds__(PW * 32) prune_kernel(const uint32_t* __restrict__ knn, const float* __restrict__ knn_d,
                                                        uint64_t m, uint32_t L, uint32_t R, uint32_t rule,
                                                        uint32_t* __restrict__ out, float* __restrict__ out_d) {
    constexpr uint32_t LP = LPL * 32;          // padded L (power of two)
    constexpr uint32_t NB = LP / 2;            // buckets of 8 slots: load factor 1/4
    constexpr uint32_t NBB = LPL == 1 ? 4 : LPL == 2 ? 5 : LPL == 4 ? 6 : 7;
    constexpr int FLUSH = PruneLayout<LPL>::FLUSH;   // rows per queue flush
    static_assert((1u << NBB) == NB, "bucket bits");
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    using Lay = PruneLayout<LPL>;
    uint8_t* base = sm + (size_t)w * Lay::PER;
    uint64_t* tab = (uint64_t*)(base + Lay::BKEYS);    // [8 NB] cuckoo slots (id << 32 | rank)
    constexpr uint32_t TBITS = NBB + 3;
    uint32_t* nst = (uint32_t*)(base + Lay::NST);      // stash count
    uint32_t* bloom = (uint32_t*)(base + Lay::BLOOM);  // 64 words
    uint32_t* cnt = (uint32_t*)(base + Lay::CNT);      // detour count per rank
    uint32_t* na = (uint32_t*)(base + Lay::NA);        // N[a]
    uint32_t* off = (uint32_t*)(base + Lay::OFF);      // counting-sort offsets per count value (L + 1)
    uint32_t* stg = (uint32_t*)(base + Lay::STG);      // per lane: the 2-hop ids of one flush group
    uint64_t* qe = (uint64_t*)(base + Lay::QE);        // queue: max(r_ad, r_db) << 32 | id
    const uint64_t nwarps = (uint64_t)gridDim.x * PW;
    for (uint64_t a = (uint64_t)blockIdx.x * PW + w; a < m; a += nwarps) {
        const uint32_t* Na = knn + a * L;
        for (uint32_t i = lane; i < NB * 8; i += 32) tab[i] = ~0ull;
        if (lane == 0) *nst = 0;
        for (uint32_t r = lane; r < LP; r += 32) { na[r] = r < L ? Na[r] : SG_SENT; cnt[r] = 0; }
        for (uint32_t r = lane; r <= LP; r += 32) off[r] = 0;
        bloom[lane] = 0;
        bloom[32 + lane] = 0;
        __syncwarp();
        for (uint32_t r = lane; r < L; r += 32) {
            const uint32_t id = na[r];
            if (id == SG_SENT) continue;
            atomicOr(&bloom[(id >> 5) & 63u], 1u << (id & 31u));   // filter bit = id mod 2048
            uint64_t e = ((uint64_t)id << 32) | r;
            uint32_t slot = ch1(id, TBITS);
            uint32_t it = 0;
            for (; it < 64; it++) {
                const uint64_t old = atomicExch((unsigned long long*)&tab[slot], (unsigned long long)e);
                if (old == ~0ull) break;
                e = old;   // evicted: move it to its other slot
                const uint32_t oid = (uint32_t)(old >> 32), a1 = ch1(oid, TBITS);
                slot = slot == a1 ? ch2(oid, TBITS) : a1;
            }
            if (it == 64) atomicExch(nst, STASH + 1);   // did not settle: the node takes the slow path
        }
        __syncwarp();
        const uint32_t nstash = *nst;
        const uint32_t fword = bloom[lane], fword1 = bloom[32 + lane];   // 2048-bit filter, two words per lane
        if (nstash > STASH) {   // cuckoo insertion did not settle: exact but slow path
            for (uint32_t r0 = 0; r0 < L; r0++) {
                const uint32_t dl = na[r0];
                if (dl == SG_SENT) continue;
                for (uint32_t rdb = lane; rdb < L; rdb += 32) {
                    const uint32_t b = __ldg(knn + (uint64_t)dl * L + rdb);
                    if (b == SG_SENT || b == (uint32_t)a) continue;
                    const uint32_t mx = RULE == 0 ? max(r0, rdb) : r0;
                    for (uint32_t r = mx + 1; r < L; r++)
                        if (na[r] == b) { atomicAdd(&cnt[r], 1u); break; }
                }
            }
        } else {
            // ~92% of 2-hop ids are not in N[a]: a register filter settles most of them; the rest
            // are queued (ballot + prefix popc) and resolved densely against the table.  The next
            // batch of 2-hop rows is loaded while the current one is filtered.
            uint32_t bv[4][LPL], bn[4][LPL];
            load_rows<LPL>(knn, na, 0, L, lane, bv);
            for (uint32_t r0 = 0; r0 < L; r0 += 4) {
                if (r0 + 4 < L) load_rows<LPL>(knn, na, r0 + 4, L, lane, bn);
#pragma unroll
                for (int u0 = 0; u0 < 4; u0 += FLUSH) {
                    // (1) filter FLUSH rows x LPL ids per lane into a local bit mask (slot u * LPL + q);
                    //     SENT and a itself are never in the table, so they need no special case
                    uint32_t lm = 0;
#pragma unroll
                    for (int u = u0; u < u0 + FLUSH; u++)
#pragma unroll
                        for (int q = 0; q < LPL; q++) {
                            const uint32_t b = bv[u][q];
                            const uint32_t f0 = __shfl_sync(0xffffffffu, fword, (b >> 5) & 31u);
                            const uint32_t f1 = __shfl_sync(0xffffffffu, fword1, (b >> 5) & 31u);
                            const uint32_t fw = (b & 1024u) ? f1 : f0;
                            lm |= (__funnelshift_r(fw, fw, b) & 1u) << ((u - u0) * LPL + q);
                            stg[((u - u0) * LPL + q) * 32 + lane] = b;   // slot-major: conflict free
                        }
                    // (2) queue offsets: exclusive warp scan of the positives per lane
                    if (rule & 0x200u) lm = 0;   // diagnostics ablation: no queue
                    const uint32_t np = __popc(lm);
                    uint32_t inc = np;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                        if (lane >= (uint32_t)o) inc += t;
                    }
                    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
                    SG_DCHECK(total <= QCAP);
                    uint32_t pos = inc - np;
                    // (3) append (max(r_ad, r_db) << 32 | id) of the positives only (loop over the
                    //     set bits; the ids come back from the lane's staging slots)
                    while (lm) {
                        const uint32_t j = __ffs(lm) - 1;
                        lm &= lm - 1;
                        const uint32_t r_ad = r0 + u0 + j / LPL, r_db = LPL * lane + j % LPL;
                        // only ranks r_ab > max(r_ad, r_db) (rule P) / > r_ad (rule 1) count
                        const uint32_t mx = RULE == 0 ? max(r_ad, r_db) : r_ad;
                        qe[pos++] = ((uint64_t)mx << 32) | stg[j * 32 + lane];
                    }
                    __syncwarp();
                    // (4) resolve the queue densely against the table
                    for (uint32_t i = lane; i < ((rule & 0x100u) ? 0u : total); i += 32) {   // 0x100: no lookups
                        const uint64_t e = qe[i];
                        const uint32_t b = (uint32_t)e;
                        const uint32_t r_ab = lookup(tab, TBITS, b);
                        if (r_ab != 0xFFFFFFFFu && (uint32_t)(e >> 32) < r_ab) atomicAdd(&cnt[r_ab], 1u);
                    }
                    __syncwarp();
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int q = 0; q < LPL; q++) bv[u][q] = bn[u][q];
            }
        }
        __syncwarp();
        // stable counting sort of the ranks by detour count (sentinel ranks last): position of rank
        // r = #{count < cnt[r]} + #{r' < r with the same count}; the first R are written
        uint32_t cv[LPL];
#pragma unroll
        for (int i = 0; i < LPL; i++) {
            const uint32_t r = i * 32 + lane;
            cv[i] = r >= L ? 0xFFFFFFFFu : na[r] == SG_SENT ? L : cnt[r];   // counts are <= r < L
            if (r < L) atomicAdd(&off[cv[i]], 1u);
        }
        __syncwarp();
        {   // exclusive scan of off[0..L]
            uint32_t run = 0;
            for (uint32_t c0 = 0; c0 <= L; c0 += 32) {
                const uint32_t c = c0 + lane;
                const uint32_t v = c <= L ? off[c] : 0;
                uint32_t inc = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= (uint32_t)o) inc += t;
                }
                if (c <= L) off[c] = run + inc - v;
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < LPL; i++) {   // rank groups in increasing rank order
            const uint32_t r = i * 32 + lane;
            const uint32_t c = cv[i];
            const uint32_t grp = __match_any_sync(0xffffffffu, c);
            const uint32_t leader = __ffs(grp) - 1;
            uint32_t pos0 = 0;
            if (lane == leader && c != 0xFFFFFFFFu) pos0 = atomicAdd(&off[c], __popc(grp));
            const uint32_t pos = __shfl_sync(0xffffffffu, pos0, leader) + __popc(grp & lt);
            if (c != 0xFFFFFFFFu && pos < R) {
                out[a * R + pos] = na[r];
                out_d[a * R + pos] = knn_d[a * L + r];
            }
        }
        __syncwarp();
    }
}

template <int LPL, int PW>
size_t prune_smem() {
    return (size_t)PW * PruneLayout<LPL>::PER + 64;
}

template <int LPL, int PW, int RULE>
sg_status prune_launch(const uint32_t* knn, const float* knn_d, uint64_t m, uint32_t L, uint32_t R, uint32_t rule,
                       uint32_t* out, float* out_d, cudaStream_t st) {
    const size_t smem = prune_smem<LPL, PW>();
    auto kern = prune_kernel<LPL, PW, RULE>;
    SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PW * 32, smem));
    if (per_sm < 1) per_sm = 1;
    const uint64_t cap = (uint64_t)num_sms() * per_sm;
    const uint64_t blocks = (m + PW - 1) / PW;
    kern<<<(unsigned)(blocks < cap ? blocks : cap), PW * 32, smem, st>>>(knn, knn_d, m, L, R, rule, out, out_d);
    SG_LAUNCHED("prune_kernel");
    return SG_OK;
}

}  // namespace

sg_status launch_prune(const uint32_t* knn, const float* knn_d, uint64_t m, uint32_t L, uint32_t R, uint32_t rule,
                       uint32_t* out, float* out_d, cudaStream_t st) {
    static int abl = -1;   // diagnostics: SG_PRUNE_ABL bit 0 skips the table lookups, bit 1 the queue
    if (abl < 0) { const char* e = getenv("SG_PRUNE_ABL"); abl = e ? atoi(e) : 0; }
    const uint32_t rl = rule | ((uint32_t)abl << 8);
    if (m == 0) return SG_OK;
    if (rule == 0) {
        if (L <= 32) return prune_launch<1, 8, 0>(knn, knn_d, m, L, R, rl, out, out_d, st);
        if (L <= 64) return prune_launch<2, 8, 0>(knn, knn_d, m, L, R, rl, out, out_d, st);
        if (L <= 128) return prune_launch<4, 8, 0>(knn, knn_d, m, L, R, rl, out, out_d, st);
        return prune_launch<8, 4, 0>(knn, knn_d, m, L, R, rl, out, out_d, st);
    }
    if (L <= 32) return prune_launch<1, 8, 1>(knn, knn_d, m, L, R, rl, out, out_d, st);
    if (L <= 64) return prune_launch<2, 8, 1>(knn, knn_d, m, L, R, rl, out, out_d, st);
    if (L <= 128) return prune_launch<4, 8, 1>(knn, knn_d, m, L, R, rl, out, out_d, st);
    return prune_launch<8, 4, 1>(knn, knn_d, m, L, R, rl, out, out_d, st);
}

}  // namespace sg
