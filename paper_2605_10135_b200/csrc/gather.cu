// a4 — shard materialisation: gather rows idmap[0..m) of x into the tensor-core operand
// layout (row-major, K padded to whole 128-byte swizzle atoms, rows padded to 128) and
// compute the fp32 row norms used by the distance epilogue (reading R3).
//   F16_EXACT: x -> f16 (exact for integers |v| <= 2048), K padded to 64.
//   TF32:      x -> tf32 (cvt.rna), K padded to 32.
//   TF32X3:    A = [hi | hi | lo], B = [hi | lo | hi] so A.B = hi.hi + hi.lo + lo.hi.
// One warp per row; |x|^2 accumulated in fp64 and rounded once (exact for integer data).
#include <cuda_fp16.h>

#include "common.cuh"

namespace sg {
namespace {

__device__ __forceinline__ float to_tf32(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

template <int PREC>
__global__ void gather_rows(const void* __restrict__ x, int dtype, uint32_t d, const uint32_t* __restrict__ ids,
                            uint64_t m, uint64_t rows_pad, uint32_t kdim, uint32_t dpad, int metric,
                            void* __restrict__ outa, void* __restrict__ outb, float* __restrict__ norm) {
    const uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (r >= rows_pad) return;
    double s = 0.0;
    const bool real = r < m;
    const uint64_t src = real ? (ids ? ids[r] : r) : 0;
    for (uint32_t j = lane; j < dpad; j += 32) {
        float v = 0.f;
        if (real && j < d)
            v = dtype == SG_U8 ? (float)((const uint8_t*)x)[src * d + j] : ((const float*)x)[src * d + j];
        s += (double)v * (double)v;
        if constexpr (PREC == SG_PREC_F16_EXACT) {
            ((__half*)outa)[r * kdim + j] = __float2half_rn(v);
        } else if constexpr (PREC == SG_PREC_TF32) {
            ((float*)outa)[r * kdim + j] = to_tf32(v);
        } else {
            const float hi = to_tf32(v), lo = to_tf32(v - hi);
            float* A = (float*)outa + r * kdim;
            float* B = (float*)outb + r * kdim;
            A[j] = hi; A[dpad + j] = hi; A[2 * dpad + j] = lo;
            B[j] = hi; B[dpad + j] = lo; B[2 * dpad + j] = hi;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) norm[r] = real ? (metric == SG_IP ? 0.f : (float)s) : __int_as_float(0x7f800000);
}

__global__ void exactness_probe(const float* __restrict__ x, const uint32_t* __restrict__ ids, uint64_t m,
                                uint32_t d, unsigned int* flags) {
    // flags[0] |= non-integral or non-finite seen; flags[1] = max |x| as float bits, over rows ids[0..m)
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x, cnt = m * d;
    unsigned nonint = 0, mx = 0;
    for (; i < cnt; i += stride) {
        const uint64_t r = i / d, j = i % d;
        const float v = x[(ids ? (uint64_t)ids[r] : r) * d + j];
        nonint |= (v != rintf(v)) || !isfinite(v);
        mx = max(mx, __float_as_uint(fabsf(v)));
    }
    if (nonint) atomicOr(&flags[0], 1u);
    atomicMax(&flags[1], mx);
}

}  // namespace

uint32_t operand_kdim(int prec, uint32_t d) {
    if (prec == SG_PREC_F16_EXACT) return (d + 63) / 64 * 64;
    if (prec == SG_PREC_TF32) return (d + 31) / 32 * 32;
    return 3 * ((d + 31) / 32 * 32);
}

size_t operand_bytes(int prec, uint32_t d, uint64_t rows) {
    const uint64_t rp = (rows + 127) / 128 * 128;
    const size_t e = prec == SG_PREC_F16_EXACT ? 2 : 4;
    size_t b = rp * operand_kdim(prec, d) * e + 256;
    if (prec == SG_PREC_TF32X3) b *= 2;
    return b + rp * sizeof(float) + 512;
}

int resolve_precision(int32_t precision, sg_dtype dtype, uint32_t d, const void* xa, const uint32_t* ida,
                      uint64_t ma, const void* xb, const uint32_t* idb, uint64_t mb, unsigned int* flags,
                      cudaStream_t st, sg_status* err) {
    *err = SG_OK;
    if (precision != SG_PREC_AUTO) return precision;
    if (dtype == SG_U8) return 2ull * d * 255 * 255 < (1ull << 24) ? SG_PREC_F16_EXACT : SG_PREC_TF32;
    cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned), st);
    exactness_probe<<<num_sms() * 4, 256, 0, st>>>((const float*)xa, ida, ma, d, flags);
    if (xb) exactness_probe<<<num_sms() * 4, 256, 0, st>>>((const float*)xb, idb, mb, d, flags);
    unsigned h[2];
    cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { *err = cuda_status(e, "exactness_probe"); return 0; }
    float mx;
    memcpy(&mx, &h[1], sizeof(float));
    const bool exact = !h[0] && mx <= 2048.f && 2.0 * d * (double)mx * mx < 16777216.0;
    return exact ? SG_PREC_F16_EXACT : SG_PREC_TF32;
}

sg_status gather_operand(const void* x, sg_dtype dtype, uint32_t d, const uint32_t* ids, uint64_t m, int prec,
                         int metric, bool /*as_columns*/, Carver& cv, Operand* op, cudaStream_t st) {
    op->kdim = operand_kdim(prec, d);
    op->esize = prec == SG_PREC_F16_EXACT ? 2 : 4;
    op->rows = m;
    op->rows_pad = (m + 127) / 128 * 128;
    const size_t elems = op->rows_pad * op->kdim;
    op->a = cv.take<uint8_t>(elems * op->esize);
    op->b = prec == SG_PREC_TF32X3 ? cv.take<uint8_t>(elems * op->esize) : op->a;
    op->norm_a = op->norm_b = cv.take<float>(op->rows_pad);
    if (!cv.ok()) { set_error("gather: workspace too small"); return SG_ERR_WORKSPACE; }
    const uint32_t dpad = prec == SG_PREC_TF32X3 ? op->kdim / 3 : op->kdim;
    const uint64_t threads = op->rows_pad * 32;
    const unsigned grid = (unsigned)((threads + 255) / 256);
    if (prec == SG_PREC_F16_EXACT)
        gather_rows<SG_PREC_F16_EXACT><<<grid, 256, 0, st>>>(x, dtype, d, ids, m, op->rows_pad, op->kdim, dpad, metric,
                                                             op->a, op->b, op->norm_a);
    else if (prec == SG_PREC_TF32)
        gather_rows<SG_PREC_TF32><<<grid, 256, 0, st>>>(x, dtype, d, ids, m, op->rows_pad, op->kdim, dpad, metric,
                                                        op->a, op->b, op->norm_a);
    else
        gather_rows<SG_PREC_TF32X3><<<grid, 256, 0, st>>>(x, dtype, d, ids, m, op->rows_pad, op->kdim, dpad, metric,
                                                          op->a, op->b, op->norm_a);
    SG_LAUNCHED("gather_rows");
    return SG_OK;
}

}  // namespace sg
