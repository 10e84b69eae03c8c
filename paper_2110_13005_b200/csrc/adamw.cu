// K9: fused AdamW (decoupled weight decay) with the bf16 theta16 cast fused in.
//
// "run the optimizer" (Alg. 1 l.7): Adam with
// lr 1e-3, beta 0.9/0.999, decoupled wd 0.01; the optimizer
// converts the half-precision gradients to full precision and descales them
// and updates the fp32 master copy; theta16 = RNE(theta).
// Op order = reading D-14, every operation IEEE
// round-to-nearest with no FMA contraction (__f*_rn), so the result is
// bit-identical to the fp32 oracle.  HBM-bound: 28 B/param (read theta, m, v,
// g16; write theta, m, v, theta16).  16-byte vector accesses, grid-stride
// loop sized to a multiple of the SM count.
#include <cuda_runtime.h>
#include "half.cuh"
#include <cstdint>

#include "kernels.h"

namespace axonn {

struct AdamScalars {
  float decay, b1, omb1, b2, omb2, step, bc2_sqrt, eps, inv_scale;
};

__device__ __forceinline__ void adam_one(float& th, float& m, float& v, float g16,
                                         const AdamScalars& s, hx& t16) {
  float g = __fmul_rn(g16, s.inv_scale);
  th = __fmul_rn(th, s.decay);
  m = __fadd_rn(__fmul_rn(s.b1, m), __fmul_rn(s.omb1, g));
  v = __fadd_rn(__fmul_rn(s.b2, v), __fmul_rn(s.omb2, __fmul_rn(g, g)));
  float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), s.bc2_sqrt), s.eps);
  th = __fsub_rn(th, __fmul_rn(s.step, __fdiv_rn(m, denom)));
  t16 = f2hx(th);
}

__global__ void __launch_bounds__(256) adamw_kernel(long long n, const hx* __restrict__ g16,
                                                    float* __restrict__ theta, float* __restrict__ m,
                                                    float* __restrict__ v,
                                                    hx* __restrict__ theta16,
                                                    AdamScalars s) {
  const long long nvec = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  auto step4 = [&](long long i, float4 th, float4 mm, float4 vv, uint2 graw) {
    hx2 g01 = *reinterpret_cast<hx2*>(&graw.x);
    hx2 g23 = *reinterpret_cast<hx2*>(&graw.y);
    hx o[4];
    adam_one(th.x, mm.x, vv.x, __low2float(g01), s, o[0]);
    adam_one(th.y, mm.y, vv.y, __high2float(g01), s, o[1]);
    adam_one(th.z, mm.z, vv.z, __low2float(g23), s, o[2]);
    adam_one(th.w, mm.w, vv.w, __high2float(g23), s, o[3]);
    reinterpret_cast<float4*>(theta)[i] = th;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    uint2 out;
    hx2 p01 = hx2_pack(o[0], o[1]);
    hx2 p23 = hx2_pack(o[2], o[3]);
    out.x = *reinterpret_cast<uint32_t*>(&p01);
    out.y = *reinterpret_cast<uint32_t*>(&p23);
    reinterpret_cast<uint2*>(theta16)[i] = out;
  };
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // two independent vectors per iteration: all eight loads in flight before the math
  for (; i + stride < nvec; i += 2 * stride) {
    const long long j = i + stride;
    const float4 th0 = __ldcs(reinterpret_cast<const float4*>(theta) + i);
    const float4 th1 = __ldcs(reinterpret_cast<const float4*>(theta) + j);
    const float4 m0 = __ldcs(reinterpret_cast<const float4*>(m) + i);
    const float4 m1 = __ldcs(reinterpret_cast<const float4*>(m) + j);
    const float4 v0 = __ldcs(reinterpret_cast<const float4*>(v) + i);
    const float4 v1 = __ldcs(reinterpret_cast<const float4*>(v) + j);
    const uint2 g0 = __ldcs(reinterpret_cast<const uint2*>(g16) + i);
    const uint2 g1 = __ldcs(reinterpret_cast<const uint2*>(g16) + j);
    step4(i, th0, m0, v0, g0);
    step4(j, th1, m1, v1, g1);
  }
  for (; i < nvec; i += stride)
    step4(i, reinterpret_cast<const float4*>(theta)[i], reinterpret_cast<const float4*>(m)[i],
          reinterpret_cast<const float4*>(v)[i], reinterpret_cast<const uint2*>(g16)[i]);
  // ragged tail (n % 4)
  for (long long i = nvec * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float th = theta[i], mm = m[i], vv = v[i];
    hx o;
    adam_one(th, mm, vv, hx2f(g16[i]), s, o);
    theta[i] = th;
    m[i] = mm;
    v[i] = vv;
    theta16[i] = o;
  }
}


int adamw_launch(long long n, const void* g16, float* theta, float* m, float* v, void* theta16,
                 const float* sc, cudaStream_t st) {
  if (n <= 0) return 0;
  if ((reinterpret_cast<uintptr_t>(g16) & 7) || (reinterpret_cast<uintptr_t>(theta) & 15) ||
      (reinterpret_cast<uintptr_t>(m) & 15) || (reinterpret_cast<uintptr_t>(v) & 15) ||
      (reinterpret_cast<uintptr_t>(theta16) & 7))
    return -2;
  const int g_sms_adam = device_sms();
  AdamScalars s{sc[0], sc[1], sc[2], sc[3], sc[4], sc[5], sc[6], sc[7], sc[8]};
  long long nvec = (n + 3) / 4;
  long long blocks = (nvec + 255) / 256;
  long long cap = (long long)g_sms_adam * 8;   // 8 resident 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  adamw_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, reinterpret_cast<const hx*>(g16),
                                                 theta, m, v,
                                                 reinterpret_cast<hx*>(theta16), s);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

}  // namespace axonn

namespace axonn {
int preload_adamw() {   // see preload_ops (ops.cu)
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)adamw_kernel) == cudaSuccess ? 0 : -1;
}
}  // namespace axonn
