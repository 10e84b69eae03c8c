// The 16-bit storage type of the half-precision copy of the model ("two
// copies of the model: a half-precision one for forward/backward and a full-precision one for
// the optimizer").  One library build per type: libaxonn.so (bf16, reading D-31) and
// libaxonn_fp16.so (-DAXONN_HALF_FP16, the paper's own fp16 with loss scaling, §8(f) N2).  Every
// kernel reads and writes 16-bit values through these names only; all arithmetic is fp32.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace axonn {

#ifdef AXONN_HALF_FP16
typedef __half hx;
typedef __half2 hx2;
__host__ __device__ __forceinline__ hx f2hx(float f) { return __float2half_rn(f); }
__host__ __device__ __forceinline__ float hx2f(hx x) { return __half2float(x); }
__device__ __forceinline__ hx2 f2hx2(float lo, float hi) { return __floats2half2_rn(lo, hi); }
__device__ __forceinline__ float2 hx22f2(hx2 x) { return __half22float2(x); }
__device__ __forceinline__ hx2 hx2_pack(hx lo, hx hi) { return __halves2half2(lo, hi); }
constexpr uint32_t kUmmaFmt = 0u;                       // kind::f16 A/B format: F16
#define AXONN_TMA_HALF CU_TENSOR_MAP_DATA_TYPE_FLOAT16
constexpr int kHalfDtype = 1;                           // AXONN_FP16
constexpr uint32_t kHalfExpMask = 0x7C00u;              // all-ones exponent: inf / NaN
#else
typedef __nv_bfloat16 hx;
typedef __nv_bfloat162 hx2;
__host__ __device__ __forceinline__ hx f2hx(float f) { return __float2bfloat16_rn(f); }
__host__ __device__ __forceinline__ float hx2f(hx x) { return __bfloat162float(x); }
__device__ __forceinline__ hx2 f2hx2(float lo, float hi) { return __floats2bfloat162_rn(lo, hi); }
__device__ __forceinline__ float2 hx22f2(hx2 x) { return __bfloat1622float2(x); }
__device__ __forceinline__ hx2 hx2_pack(hx lo, hx hi) { return __halves2bfloat162(lo, hi); }
constexpr uint32_t kUmmaFmt = 1u;                       // kind::f16 A/B format: BF16
#define AXONN_TMA_HALF CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
constexpr int kHalfDtype = 0;                           // AXONN_BF16
constexpr uint32_t kHalfExpMask = 0x7F80u;              // all-ones exponent: inf / NaN
#endif

}  // namespace axonn
