// Shared device code of the distance kernels (knn_tc.cu: row-per-lane epilogue; knn_tct.cu:
// transposed, column-per-lane epilogue): PTX wrappers, descriptors, parameters, selection.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "common.cuh"

namespace sg {
namespace {

constexpr uint32_t MSUB = 128;           // rows per accumulator (MMA M)
constexpr uint32_t NACC_MAX = 2;         // accumulators (row halves) per CTA: 2 (f16), 1 (tf32: wider A)
constexpr uint32_t BM = MSUB * NACC_MAX; // rows per CTA row block (operand padding unit)
#ifndef SG_BN
#define SG_BN 128
#endif
#ifndef SG_KNN_PROF
#define SG_KNN_PROF 0   // 1: per-warp cycle counters (diagnostics build only; costs registers + local memory)
#endif
constexpr uint32_t BN = SG_BN;           // columns per tile (MMA N); N=64 MMAs lose ~45% to issue overhead
constexpr uint32_t ATOM = 128 * 128;     // A atom: 128 rows x 128 B (128B swizzle)
constexpr uint32_t MINIB = 128 * 32;     // A mini atom: 128 rows x 32 B (32B swizzle)
constexpr uint32_t BATOM = BN * 128;     // B atom: 64 rows x 128 B
constexpr uint32_t BMINI = BN * 32;      // B mini atom: 64 rows x 32 B
constexpr uint32_t SLOT = BATOM;         // B ring slot
constexpr uint32_t NEPI = 8;             // epilogue warps
constexpr uint32_t NTHREADS = 64 + NEPI * 32;
constexpr uint32_t MAX_STAGES = 32;
constexpr uint32_t NBUF_MAX = 4;         // TMEM buffers per accumulator: 4 (A in smem) or 2 (A in TMEM)
constexpr uint32_t KSTRIDE = 36;         // floats per staged row (16B aligned, conflict-free)
constexpr uint32_t SCRATCH = 32 * KSTRIDE * 4 + 64 * 4;   // per warp: staged keys | hist | sort buffer (+ spare)
constexpr uint32_t SORT_MAX = 512;      // final sort buffer (u64 entries, aliases the staged keys)
static_assert(SORT_MAX * 8 <= 32 * KSTRIDE * 4, "sort buffer exceeds the warp scratch");

// ----------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
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
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(0x989680u)   // suspend-time hint: sleep until the phase flips
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

// Shared-memory matrix descriptors, K-major: 128B swizzle (8-row groups 1024 B apart) and
// 32B swizzle (8-row groups 256 B apart).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(256u >> 4) << 32) | (1ull << 46) | (6ull << 61);
}

// Instruction descriptor: D fp32, A/B f16 (KIND 0) or tf32 (KIND 1), both K-major, M=128, N=BN.
template <int KIND>
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4) | ((KIND ? 2u : 0u) << 7) | ((KIND ? 2u : 0u) << 10) | ((BN >> 3) << 17) | ((MSUB >> 4) << 24);
}

__device__ __forceinline__ float min3f(float a, float b, float c) {   // one FMNMX3 (sm_100)
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// smallest of 32 keys (raw float bits): a depth-4 tree of 16 FMNMX3
__device__ __forceinline__ float min32(const uint32_t (&v)[32]) {
    float m[12];
#pragma unroll
    for (int i = 0; i < 10; i++)
        m[i] = min3f(__uint_as_float(v[3 * i]), __uint_as_float(v[3 * i + 1]), __uint_as_float(v[3 * i + 2]));
    m[10] = __uint_as_float(v[30]);
    m[11] = __uint_as_float(v[31]);
    const float a = min3f(m[0], m[1], m[2]), b = min3f(m[3], m[4], m[5]), c = min3f(m[6], m[7], m[8]),
                d = min3f(m[9], m[10], m[11]);
    return fminf(min3f(a, b, c), d);
}

__device__ __forceinline__ float next_up(float x) {   // smallest float > x (x < +inf)
    return x == __int_as_float(0x7f800000) ? x : ord2f(f2ord(x) + 1u);
}

}  // namespace

// shared by both kernel translation units (external linkage: launch_knn_t takes it)
struct KnnParams {
    const float* norm_a;       // |a_i|^2 (0 for IP) for the final distance, operand row order
    uint64_t* cand;            // gridDim.x * BM rows * C candidate words
    uint32_t* out_ids;         // ma x L
    float* out_d;              // ma x L
    float* probe;              // optional raw accumulator dump (ma x mb)
    unsigned long long* prof;  // optional per-warp cycle counters (diagnostics)
    const uint32_t* row_map;   // A row (operand order) -> output row (nullptr = identity)
    const uint32_t* col_map;   // B row (operand order) -> reported id (nullptr = identity)
    uint32_t ma, mb, L, C, n_rb, n_ct, stages;
    uint32_t keep_max;         // in-loop compaction keeps between L and keep_max candidates
    uint32_t nka;              // streamed-A / pair kernels: full 128-byte K atoms per row (run time)
    uint32_t mini;             // pair kernel: 1 if a 32-byte K-tail atom follows
    // Extrapolated thresholds (columns in id order, no rotation): after `seen` of mb columns the
    // in-loop compaction keeps rank r = min(L, alpha100 * L * seen / (100 mb) + beta) instead of L.
    // The buffer always holds every seen column with (key, id) <= the threshold entry, so a row
    // that ends with >= L candidates is exact; one that ends with fewer is appended to fail_rows
    // and recomputed by the fallback launch (alpha100 = 0: plain rank-L thresholds).
    uint32_t alpha100, beta;
    uint32_t eager;            // transposed kernel: compact a stream once it holds want + eager
    uint32_t kshift;           // extrapolated compaction keeps <= want + ((C - ROOM - want) >> kshift)
    uint32_t z100;             // > 0: binomial extrapolated targets (z score x 100), else linear (alpha)
    uint32_t* fail_count;      // device counter of rows to recompute (extrapolated launch)
    uint32_t* fail_rows;       // their operand rows
    const uint32_t* n_rows_dev;   // fallback launch: A row count read on the device (nullptr: ma)
    const uint32_t* self_col;  // B column excluded for A row i (nullptr: column i)
    uint32_t rb_rows;          // rows per row block (128 * accumulators)
    uint32_t t_back;           // with rotate: a row block starts t_back tiles before its diagonal
    int rotate;                // column tiles visited from the diagonal - t_back cyclically
    int self_exclude;
    int noepi;                 // diagnostics: epilogue only drains TMEM (pipeline speed test)
    int noload;                // diagnostics: producer skips the B loads (tensor-core speed test)
    int abl;                   // diagnostics ablation bits: 1 no insertion, 2 no id fetch, 4 no clock64
    uint32_t a_words;          // 32-bit words per A row
};

namespace {


__device__ __forceinline__ uint32_t tile_at(const KnnParams& p, uint32_t rb, uint32_t i) {
    if (!p.rotate) return i;
    const uint32_t diag = rb * (p.rb_rows / BN) % p.n_ct;
    const uint32_t back = p.t_back % p.n_ct;
    return (diag + p.n_ct - back + i) % p.n_ct;
}

struct __align__(8) Bars {
    uint64_t full[MAX_STAGES], empty[MAX_STAGES];
    uint64_t a_full, a_empty;
    uint64_t tm_full[NBUF_MAX], tm_empty[NBUF_MAX];
    uint32_t tmem_base;
};

// Candidate words are stored raw as (float bits << 32 | col); selection works on the ordered
// form (ord(key) << 32 | col) whose unsigned order is the (key, col) order.
__device__ __forceinline__ uint64_t raw2ord(uint64_t w) {
    return ((uint64_t)f2ord(__uint_as_float((uint32_t)(w >> 32))) << 32) | (uint32_t)w;
}
__device__ __forceinline__ uint64_t ord2raw(uint64_t w) {
    return ((uint64_t)__float_as_uint(ord2f((uint32_t)(w >> 32))) << 32) | (uint32_t)w;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
    }
    return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// Warp-cooperative threshold selection over rb[0..cnt) by key only (ties on the key are never
// split).  Finds, by bit descent on the ordered 32-bit key (one ballot-count per bit, no shared
// memory), a threshold T with count(key <= T) >= want, stopping early once that count is at most
// keep_max, else at the smallest such T.  Keeps every entry with key <= T, in place at
// rb[0..kept), and returns T.  All 32 lanes call with the same arguments; cnt >= want.
template <int EPL>
__device__ __forceinline__ uint32_t select_keys(uint64_t* rb, uint32_t cnt, uint32_t want, uint32_t keep_max,
                                                uint32_t lane, uint32_t* kept) {
    uint64_t e[EPL];
    uint32_t k[EPL];
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        const uint32_t idx = i * 32 + lane;
        e[i] = idx < cnt ? rb[idx] : 0ull;
        k[i] = idx < cnt ? f2ord(__uint_as_float((uint32_t)(e[i] >> 32))) : 0xFFFFFFFFu;
        if (idx < cnt) { lo = min(lo, k[i]); hi = max(hi, k[i]); }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    uint32_t T = hi;
    if (lo != hi && cnt > keep_max) {
        int b = 31 - __clz(lo ^ hi);
        uint32_t pfx = b >= 31 ? 0u : lo & ~((2u << b) - 1u);   // bits above b are common to all keys
        bool done = false;
#pragma unroll 1
        for (; b >= 0; b--) {
            const uint32_t t = pfx | ((1u << b) - 1u);           // largest key with bit b = 0
            uint32_t c = 0;
#pragma unroll
            for (int i = 0; i < EPL; i++) c += __popc(__ballot_sync(0xffffffffu, k[i] <= t));
            if (c >= want) {
                T = t;
                if (c <= keep_max) { done = true; break; }
            } else {
                pfx |= 1u << b;
            }
        }
        if (!done) T = pfx;   // smallest key with count(key <= T) >= want
    }
    uint32_t base = 0;
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        const bool sel = k[i] <= T;
        const uint32_t bal = __ballot_sync(0xffffffffu, sel);
        if (sel) rb[base + __popc(bal & ((1u << lane) - 1u))] = e[i];
        base += __popc(bal);
    }
    __syncwarp();
    *kept = base;
    return T;
}

// Warp-cooperative radix selection over rb[0..cnt) (cnt > L).  Keeps, in place at rb[0..kept), a
// prefix of the (key, id) order with L <= kept <= keep_max (keep_max = L: exactly the L smallest)
// and returns the largest kept entry in ordered form (ord(key) << 32 | id).  8-bit digits start at the highest bit where the
// smallest and largest candidate differ (the shared prefix would put every candidate in one
// histogram bin), counted with shared-memory atomics.  All 32 lanes call with the same arguments.
template <int EPL>
__device__ __forceinline__ uint64_t select_L(uint64_t* rb, uint32_t cnt, uint32_t L, uint32_t keep_max,
                                             uint32_t* hist, uint32_t lane, uint32_t* kept) {
    uint64_t e[EPL];
    uint64_t lo = ~0ull, hi = 0;
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        const uint32_t idx = i * 32 + lane;
        e[i] = idx < cnt ? raw2ord(rb[idx]) : ~0ull;
        if (idx < cnt) { lo = e[i] < lo ? e[i] : lo; hi = e[i] > hi ? e[i] : hi; }
    }
    lo = warp_min_u64(lo);
    hi = warp_max_u64(hi);
    // bits [top, 64) are common to every candidate
    int top = 64 - __clzll(lo ^ hi);              // 0 only if all equal (cannot happen: ids differ)
    uint64_t pfx = top >= 64 ? 0ull : (lo >> top) << top;
    uint32_t want = L;
    int cut = top;
    uint32_t kp = 0;
#pragma unroll 1
    while (top > 0) {
        const int w = top >= 8 ? 8 : top;          // digit = bits [top - w, top)
        const int sh = top - w;
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        const uint64_t hm = top >= 64 ? 0ull : (~0ull << top);
        const uint32_t dmask = (1u << w) - 1u;
#pragma unroll
        for (int i = 0; i < EPL; i++)
            if (e[i] != ~0ull && (e[i] & hm) == (pfx & hm)) atomicAdd(&hist[(uint32_t)(e[i] >> sh) & dmask], 1u);
        __syncwarp();
        uint32_t hv[8], loc = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) { hv[j] = hist[lane * 8 + j]; loc += hv[j]; }
        const uint32_t inc = warp_incl_scan(loc, lane), exc = inc - loc;
        const bool mine = exc < want && want <= inc;
        const uint32_t bal = __ballot_sync(0xffffffffu, mine);
        uint32_t dg = 0, before = 0, bc = 0;
        if (mine) {
            uint32_t run = exc;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (bc == 0 && run + hv[j] >= want) { dg = lane * 8 + j; before = run; bc = hv[j]; }
                run += hv[j];
            }
        }
        const int src = __ffs(bal) - 1;
        dg = __shfl_sync(0xffffffffu, dg, src);
        before = __shfl_sync(0xffffffffu, before, src);
        bc = __shfl_sync(0xffffffffu, bc, src);
        want -= before;
        pfx |= (uint64_t)dg << sh;
        __syncwarp();
        top = sh;
        // entries strictly below the chosen bucket: L - want; cutting here keeps the bucket too
        if (L - want + bc <= keep_max || top == 0) { cut = sh; kp = L - want + bc; break; }
    }
    const uint64_t lim = cut >= 64 ? ~0ull : pfx >> cut;
    uint32_t base = 0;
    uint64_t mk = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        const uint32_t idx = i * 32 + lane;
        const bool s = idx < cnt && (cut >= 64 || (e[i] >> cut) <= lim);
        const uint32_t bal = __ballot_sync(0xffffffffu, s);
        if (s) {
            rb[base + __popc(bal & ((1u << lane) - 1u))] = ord2raw(e[i]);
            mk = e[i] > mk ? e[i] : mk;
        }
        base += __popc(bal);
    }
    mk = warp_max_u64(mk);
    __syncwarp();
    *kept = base;
    (void)kp;
    return mk;
}

__device__ __forceinline__ uint64_t pair_ord(float key, uint32_t id) { return ((uint64_t)f2ord(key) << 32) | id; }

// Compaction of one stream buffer rb[0..cnt) (raw words) under the row threshold pair `cap`:
// entries above `cap` are dropped; of the rest, if more than keep_max remain, only those with key
// <= T are kept, T found by bit descent on the ordered key (count(key <= T) >= want, stopping as
// soon as it is <= keep_max, else the smallest such T; ties on T are never split).  Returns the
// new threshold pair (T, SENT), or `cap` when nothing had to be selected.  All lanes call.
template <int EPL>
__device__ __forceinline__ uint64_t select_pairs(uint64_t* rb, uint32_t cnt, uint64_t cap, uint32_t want,
                                                 uint32_t keep_max, uint32_t lane, uint32_t* kept) {
    uint64_t e[EPL];
    uint32_t k[EPL];
    uint32_t n = 0;
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        const uint32_t idx = i * 32 + lane;
        e[i] = idx < cnt ? rb[idx] : 0ull;
        const uint64_t po = raw2ord(e[i]);
        const bool in = idx < cnt && po <= cap;
        k[i] = in ? (uint32_t)(po >> 32) : 0xFFFFFFFFu;
        n += __popc(__ballot_sync(0xffffffffu, in));
    }
    uint64_t P = cap;
    uint32_t T = 0xFFFFFFFEu;                   // keep every entry at or below cap
    if (n > keep_max && n > want) {
        uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll
        for (int i = 0; i < EPL; i++)
            if (k[i] != 0xFFFFFFFFu) { lo = min(lo, k[i]); hi = max(hi, k[i]); }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        T = hi;
        if (lo != hi) {
            int b = 31 - __clz(lo ^ hi);
            uint32_t pfx = b >= 31 ? 0u : lo & ~((2u << b) - 1u);
            bool done = false;
#pragma unroll 1
            for (; b >= 0; b--) {
                const uint32_t t = pfx | ((1u << b) - 1u);
                uint32_t c = 0;
#pragma unroll
                for (int i = 0; i < EPL; i++) c += __popc(__ballot_sync(0xffffffffu, k[i] <= t));
                if (c >= want) {
                    T = t;
                    if (c <= keep_max) { done = true; break; }
                } else {
                    pfx |= 1u << b;
                }
            }
            if (!done) T = pfx;
        }
        const uint64_t PT = ((uint64_t)T << 32) | SG_SENT;
        P = PT < cap ? PT : cap;
    }
    uint32_t base = 0;
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        const bool sel = k[i] <= T;
        const uint32_t bal = __ballot_sync(0xffffffffu, sel);
        if (sel) rb[base + __popc(bal & ((1u << lane) - 1u))] = e[i];
        base += __popc(bal);
    }
    __syncwarp();
    *kept = base;
    return P;
}

// a row whose prefilter hit stages its 32 keys, its threshold and its next buffer slot
__device__ __forceinline__ void stage_keys(float* skeys, uint32_t lane, const uint32_t (&v)[32], float te,
                                           uint32_t slot) {
    float4* st4 = (float4*)(skeys + lane * KSTRIDE);
#pragma unroll
    for (int j4 = 0; j4 < 8; j4++)
        st4[j4] = make_float4(__uint_as_float(v[4 * j4]), __uint_as_float(v[4 * j4 + 1]), __uint_as_float(v[4 * j4 + 2]),
                              __uint_as_float(v[4 * j4 + 3]));
    *(float2*)(skeys + lane * KSTRIDE + 32) = make_float2(te, __uint_as_float(slot));
}

// The warp takes the staged rows of `hb` one at a time, lane j testing column col0 + j: one
// ballot per row, the passing (key bits << 32 | id) words appended to consecutive slots of the
// row's buffer.  Returns how many entries this lane's own row gained.
__device__ __forceinline__ uint32_t insert_rows(const KnnParams& p, const float* skeys, uint32_t lane, uint32_t hb,
                                                uint32_t col0, long long (&pw)[8]) {
    const uint32_t myid = p.col_map ? __ldg(p.col_map + col0 + lane) : col0 + lane;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t add = 0;
    if constexpr (SG_KNN_PROF != 0) pw[7] += __popc(hb);
    do {   // two rows per iteration: independent load -> compare -> ballot -> store chains
        const int o1 = __ffs(hb) - 1;
        hb &= hb - 1;
        const bool two = hb != 0;
        const int o2 = two ? __ffs(hb) - 1 : o1;
        hb &= hb - 1;
        const float* k1 = skeys + o1 * KSTRIDE;
        const float* k2 = skeys + o2 * KSTRIDE;
        const float kv1 = k1[lane], kv2 = k2[lane];
        const float2 tw1 = *(const float2*)(k1 + 32), tw2 = *(const float2*)(k2 + 32);
        const bool ps1 = kv1 < tw1.x;           // key <= thr
        const bool ps2 = two && kv2 < tw2.x;
        const uint32_t b1 = __ballot_sync(0xffffffffu, ps1);
        const uint32_t b2 = __ballot_sync(0xffffffffu, ps2);
        if (ps1) p.cand[__float_as_uint(tw1.y) + __popc(b1 & lt)] = ((uint64_t)__float_as_uint(kv1) << 32) | myid;
        if (ps2) p.cand[__float_as_uint(tw2.y) + __popc(b2 & lt)] = ((uint64_t)__float_as_uint(kv2) << 32) | myid;
        add = lane == (uint32_t)o1 ? __popc(b1) : add;
        add = lane == (uint32_t)o2 && two ? __popc(b2) : add;
        if constexpr (SG_KNN_PROF != 0) pw[6] += __popc(b1) + __popc(b2);
    } while (hb);
    return add;
}

// Union of NL candidate lists: selected down to the keys <= the L-th smallest key in shared
// memory first (ties kept), then sorted by (dist, id) with dist = |a_i|^2 + key; first L written
// (sentinel / +inf padding).  sortbuf holds SORT_MAX words; the counts sum to <= SORT_MAX.
template <int EPL_S, int NL>
__device__ void finish_union_n(const uint64_t* const (&b)[NL], const uint32_t (&c)[NL], uint32_t L, uint64_t* sortbuf,
                               float na, uint32_t* out_ids, float* out_d, uint32_t lane) {
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < NL; k++) {
        for (uint32_t p = lane; p < c[k]; p += 32) sortbuf[cnt + p] = b[k][p];
        cnt += c[k];
    }
    __syncwarp();
    if (cnt > L) select_keys<EPL_S>(sortbuf, cnt, L, L, lane, &cnt);
    uint32_t np = 32;
    while (np < cnt) np <<= 1;
    for (uint32_t p = lane; p < np; p += 32) {
        uint64_t w = ~0ull;
        if (p < cnt) {
            const uint64_t e = sortbuf[p];
            const float dist = na + __uint_as_float((uint32_t)(e >> 32));
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
template <int EPL_S>
__device__ void finish_union(const uint64_t* b0, uint32_t c0, const uint64_t* b1, uint32_t c1, uint32_t L,
                             uint64_t* sortbuf, float na, uint32_t* out_ids, float* out_d, uint32_t lane) {
    const uint64_t* const b[2] = {b0, b1};
    const uint32_t c[2] = {c0, c1};
    finish_union_n<EPL_S, 2>(b, c, L, sortbuf, na, out_ids, out_d, lane);
}

// Merge the two column halves' survivors of one row (each <= L), sort by (dist, id) with
// dist = |a_i|^2 + key, write the first L (sentinel / +inf padding).
__device__ void finish_row(const uint64_t* b0, uint32_t c0, const uint64_t* b1, uint32_t c1, uint32_t L,
                           uint64_t* sortbuf, float na, uint32_t* out_ids, float* out_d, uint32_t lane) {
    const uint32_t cnt = c0 + c1;
    uint32_t np = 32;
    while (np < cnt) np <<= 1;
    for (uint32_t p = lane; p < np; p += 32) {
        uint64_t w = ~0ull;
        if (p < cnt) {
            const uint64_t e = p < c0 ? b0[p] : b1[p - c0];
            const float dist = na + __uint_as_float((uint32_t)(e >> 32));
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

// ----------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult qr;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    return fn;
}

// 2-D map over a rows x kdim operand; box = (box_bytes / esize) elements x box_rows rows.
sg_status make_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t kdim, uint32_t esize, uint32_t box_bytes,
                   uint32_t box_rows) {
    auto enc = get_encode();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return SG_ERR_CUDA; }
    cuuint64_t dims[2] = {kdim, rows};
    cuuint64_t strides[1] = {(cuuint64_t)kdim * esize};
    cuuint32_t box[2] = {box_bytes / esize, box_rows};
    cuuint32_t es[2] = {1, 1};
    const CUtensorMapSwizzle sw = box_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = enc(m, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return SG_ERR_CUDA; }
    return SG_OK;
}

}  // namespace
}  // namespace sg
