// Shared pieces of the K3 decode-attention kernels (SIMT and tensor-core
// variants): launch arguments, cp.async / ldmatrix / mma wrappers.
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

#include "cuda/common.cuh"

namespace prism {

struct DecodeDesc;

struct AttnArgs {
    KvGeom g;
    int layer;
    const __nv_bfloat16* q;   // [n_dec][n_q][D]
    __nv_bfloat16* out;       // [n_dec][n_q][D]
    const std::int32_t* table;
    const DecodeDesc* desc;   // [n_dec] {row, ctx, request}
    float scale_log2;         // softmax scale * log2(e)
    int chunk;                // tokens per split (multiple of the kernel tile)
    int max_splits;           // grid.x
    float* part_o;            // [n_dec * n_kv][max_splits][G][D]
    float* part_ml;           // [n_dec * n_kv][max_splits][G][2]
    int* tickets;             // [n_dec * n_kv], zero between launches
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float bf_lo(std::uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(std::uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ std::uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const std::uint32_t*>(&p);
}

__device__ __forceinline__ void ldmatrix_x4(std::uint32_t (&r)[4], const void* smem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(s));
}

__device__ __forceinline__ void ldmatrix_x4_trans(std::uint32_t (&r)[4], const void* smem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(s));
}

__device__ __forceinline__ std::uint32_t movmatrix_trans(std::uint32_t x) {
    std::uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
    return y;
}

// D (fp32 16x8) += A (bf16 16x16, row) * B (bf16 16x8, col)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const std::uint32_t (&a)[4], std::uint32_t b0,
                                               std::uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

}  // namespace prism
