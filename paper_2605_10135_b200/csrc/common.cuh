// Internal helpers of libscalegann.so (CUDA path).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/scalegann.h"

#define SG_SENT 0xFFFFFFFFu

// ------------------------------------------------------------------ errors
namespace sg {
void set_error(const char* fmt, ...);
sg_status cuda_status(cudaError_t e, const char* what);
}  // namespace sg

#define SG_CHECK_ARG(cond, ...)              \
    do {                                     \
        if (!(cond)) {                       \
            sg::set_error(__VA_ARGS__);      \
            return SG_ERR_INVALID_ARG;       \
        }                                    \
    } while (0)

#define SG_CUDA(call)                                                  \
    do {                                                               \
        cudaError_t _e = (call);                                       \
        if (_e != cudaSuccess) return sg::cuda_status(_e, #call);      \
    } while (0)

#define SG_LAUNCHED(name)                                               \
    do {                                                                \
        cudaError_t _e = cudaGetLastError();                            \
        if (_e != cudaSuccess) return sg::cuda_status(_e, name);        \
        sg::note_launch();                                              \
    } while (0)

namespace sg {
// diagnostics (api.cu): kernel launch counter and CUDA-event timing of the distance kernel
void note_launch();
void knn_time_begin(cudaStream_t st);
void knn_time_end(cudaStream_t st);
}  // namespace sg

// Device-side invariant checks of the debug build (SG_NVCC_FLAGS=-DSG_DEBUG_CHECKS=1): a violated
// bound traps the kernel (the launch then fails loudly); compiled out of the production build.
#if defined(SG_DEBUG_CHECKS) && SG_DEBUG_CHECKS
#define SG_DCHECK(cond)          \
    do {                         \
        if (!(cond)) __trap();   \
    } while (0)
#else
#define SG_DCHECK(cond) \
    do {                \
    } while (0)
#endif

#define SG_TRY(call)                              \
    do {                                          \
        sg_status _s = (call);                    \
        if (_s != SG_OK) return _s;               \
    } while (0)

namespace sg {

// ------------------------------------------------------------------ workspace
// Bump allocator over the caller's workspace; used twice: once with base=null
// to size, once to carve.  256-byte alignment (TMA needs 16, vector loads 16).
struct Carver {
    uint8_t* base;
    size_t cap;
    size_t off = 0;
    Carver(void* b, size_t c) : base((uint8_t*)b), cap(c) {}
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~(size_t)255;
        T* p = base ? (T*)(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
    bool ok() const { return off <= cap; }
};

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

inline int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// ------------------------------------------------------------------ device helpers
// float -> uint32 with the same total order (ascending); -0 is canonicalised to +0.
__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t u = __float_as_uint(f + 0.0f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
    return __uint_as_float(u);
}

// Warp-cooperative bitonic sort (ascending) of n = power of two uint64 keys in
// shared memory, optionally carrying a uint32 payload.  All 32 lanes call it.
__device__ __forceinline__ void warp_sort_u64(uint64_t* a, uint32_t n, uint32_t lane) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < n; i += 32) {
                uint32_t p = i ^ j;
                if (p > i) {
                    uint64_t x = a[i], y = a[p];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) { a[i] = y; a[p] = x; }
                }
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ void warp_sort_u64_payload(uint64_t* a, uint32_t* pl, uint32_t n, uint32_t lane) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < n; i += 32) {
                uint32_t p = i ^ j;
                if (p > i) {
                    uint64_t x = a[i], y = a[p];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y; a[p] = x;
                        uint32_t t = pl[i]; pl[i] = pl[p]; pl[p] = t;
                    }
                }
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (uint32_t)o) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024,
// multiple of 32); `tmp` holds >= 33 words of shared memory.  Returns the
// exclusive prefix; *total receives the block sum.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* tmp, uint32_t* total) {
    uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = warp_incl_scan(v, lane);
    if (lane == 31) tmp[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < nw ? tmp[lane] : 0;
        uint32_t si = warp_incl_scan(s, lane);
        if (lane < nw) tmp[lane] = si - s;
        if (lane == 31) tmp[32] = si;
    }
    __syncthreads();
    uint32_t r = tmp[w] + inc - v;
    if (total) *total = tmp[32];
    __syncthreads();
    return r;
}

}  // namespace sg

// ------------------------------------------------------------------ internal launchers
// (host functions implemented in the per-stage .cu files, called by api.cu)
namespace sg {
// gather.cu
// Augmented tensor-core operand of a set of rows (gather.cu).  Row layout, K-major:
//   A side (query rows i):   [a_i (or hi|hi|lo), norm multipliers, 0...]
//   B side (column rows j):  [-2 b_j (or -b_j for IP), norm pieces of |b_j|^2, 0...]
// so that A_i . B_j = |b_j|^2 - 2 a_i.b_j (L2) or -a_i.b_j (IP) = the selection key.
// K = nfull 128-byte atoms + optional 32-byte mini atom.  Padding rows of the B side carry
// +inf in the first norm column so their keys are +inf.
struct Operand {
    void* a = nullptr;         // A side, rows_pad x kdim (nullptr if not built)
    void* b = nullptr;         // B side, rows_pad x kdim (nullptr if not built)
    float* norm = nullptr;     // rows_pad: |x|^2 (L2) or 0 (IP), for the final distance
    uint32_t kdim = 0;         // K in elements
    uint32_t nfull = 0;        // full 128-byte atoms
    uint32_t mini = 0;         // 1 if a 32-byte mini atom follows
    uint32_t esize = 2;        // 2 (f16) or 4 (tf32)
    uint64_t rows = 0, rows_pad = 0;
};
enum { SIDE_A = 1, SIDE_B = 2 };
// AUTO -> F16_EXACT when every referenced value is an integer with |v| <= 2048 and
// 2*d*max^2 < 2^24 (then dots, norms and distances are exact in fp32), else TF32.
int resolve_precision(int32_t precision, sg_dtype dtype, uint32_t d, const void* xa, const uint32_t* ida,
                      uint64_t ma, const void* xb, const uint32_t* idb, uint64_t mb, unsigned int* flags,
                      cudaStream_t st, sg_status* err);
void operand_layout(int prec, int metric, uint32_t d, uint32_t* kdim, uint32_t* nfull, uint32_t* mini);
size_t operand_bytes(int prec, int metric, uint32_t d, uint64_t rows, int sides);
sg_status gather_operand(const void* x, sg_dtype dtype, uint32_t d, const uint32_t* ids, uint64_t m,
                         int prec, int metric, int sides, Carver& cv, Operand* op, cudaStream_t st);
// knn_tc.cu
size_t knn_core_workspace(uint32_t L, uint64_t ma, uint32_t d, int prec, int metric);
// row_map / col_map translate operand order to output rows / reported ids (spatially
// reordered shards); rotate visits column tiles starting just before the diagonal.
sg_status knn_core(const Operand& A, const Operand& B, int metric, bool self_exclude, uint32_t L,
                   uint32_t* ids, float* dists, float* probe, Carver& cv, cudaStream_t st,
                   const uint32_t* row_map = nullptr, const uint32_t* col_map = nullptr, bool rotate = false);
// order.cu: spatial order of a shard (rows grouped by nearest sub-centroid)
uint32_t order_groups(uint64_t m);   // >= 2 when the spatial order is enabled (SG_KNN_ORDER=1) and worth computing
size_t order_workspace(uint64_t m, uint32_t d, int prec, int metric);
sg_status spatial_order(const void* x, sg_dtype dtype, uint32_t d, const uint32_t* idmap, uint64_t m, int prec,
                        int metric, uint32_t* perm, uint32_t* ids_perm, Carver cv, cudaStream_t st);
// prune.cu / reverse.cu
sg_status launch_prune(const uint32_t* knn, const float* knn_d, uint64_t m, uint32_t L, uint32_t R,
                       uint32_t rule, uint32_t* out, float* out_d, cudaStream_t st);
sg_status launch_reverse(const uint32_t* pruned, const float* pruned_d, uint64_t m, uint32_t R, uint32_t h,
                         uint32_t* out, float* out_d, Carver& cv, cudaStream_t st);
// scan.cu
size_t scan_workspace(uint64_t n);
sg_status excl_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, Carver& cv, cudaStream_t st);
}  // namespace sg
