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


// K9 with the column all-reduce fused in (reading D-35): the reduced gradient
// of element i is the fp32 sum, in ascending replica order j = 0..G-1, of the G replicas'
// half-precision gradients g16_j[i] -- read straight from the peers' buffers over NVLink
// (CUDA IPC mappings) or, for the loopback, from the other contexts' buffers on this device.
// Every replica computes the identical sum, so every replica applies the identical update and
// no all-reduce result is ever materialised.  Traffic per parameter: K9's 28 B of local HBM
// plus 2 (G - 1) B read from the peers over NVLink.
struct GradPtrs {
  const hx* g[kMaxReplicas];
  int ng;
};

__global__ void __launch_bounds__(256) adamw_sum_kernel(long long n, GradPtrs gp,
                                                        float* __restrict__ theta, float* __restrict__ m,
                                                        float* __restrict__ v, hx* __restrict__ theta16,
                                                        AdamScalars s) {
  const long long nvec = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    uint2 graw[kMaxReplicas];
#pragma unroll
    for (int j = 0; j < kMaxReplicas; ++j)
      if (j < gp.ng) graw[j] = __ldcs(reinterpret_cast<const uint2*>(gp.g[j]) + i);
    float4 th = __ldcs(reinterpret_cast<const float4*>(theta) + i);
    float4 mm = __ldcs(reinterpret_cast<const float4*>(m) + i);
    float4 vv = __ldcs(reinterpret_cast<const float4*>(v) + i);
    float g[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < kMaxReplicas; ++j) {
      if (j >= gp.ng) break;
      const hx2 g01 = *reinterpret_cast<const hx2*>(&graw[j].x);
      const hx2 g23 = *reinterpret_cast<const hx2*>(&graw[j].y);
      g[0] = __fadd_rn(g[0], __low2float(g01));
      g[1] = __fadd_rn(g[1], __high2float(g01));
      g[2] = __fadd_rn(g[2], __low2float(g23));
      g[3] = __fadd_rn(g[3], __high2float(g23));
    }
    hx o[4];
    adam_one(th.x, mm.x, vv.x, g[0], s, o[0]);
    adam_one(th.y, mm.y, vv.y, g[1], s, o[1]);
    adam_one(th.z, mm.z, vv.z, g[2], s, o[2]);
    adam_one(th.w, mm.w, vv.w, g[3], s, o[3]);
    reinterpret_cast<float4*>(theta)[i] = th;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    uint2 out;
    hx2 p01 = hx2_pack(o[0], o[1]);
    hx2 p23 = hx2_pack(o[2], o[3]);
    out.x = *reinterpret_cast<uint32_t*>(&p01);
    out.y = *reinterpret_cast<uint32_t*>(&p23);
    reinterpret_cast<uint2*>(theta16)[i] = out;
  }
  for (long long i = nvec * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float g = 0.f;
    for (int j = 0; j < gp.ng; ++j) g = __fadd_rn(g, hx2f(gp.g[j][i]));
    float th = theta[i], mm = m[i], vv = v[i];
    hx o;
    adam_one(th, mm, vv, g, s, o);
    theta[i] = th;
    m[i] = mm;
    v[i] = vv;
    theta16[i] = o;
  }
}

int adamw_sum_launch(long long n, const void* const* g16s, int ng, float* theta, float* m, float* v,
                     void* theta16, const float* sc, cudaStream_t st) {
  if (n <= 0) return 0;
  if (ng < 1 || ng > kMaxReplicas) return -1;
  GradPtrs gp{};
  gp.ng = ng;
  for (int j = 0; j < ng; ++j) {
    if (reinterpret_cast<uintptr_t>(g16s[j]) & 7) return -2;
    gp.g[j] = reinterpret_cast<const hx*>(g16s[j]);
  }
  if ((reinterpret_cast<uintptr_t>(theta) & 15) || (reinterpret_cast<uintptr_t>(m) & 15) ||
      (reinterpret_cast<uintptr_t>(v) & 15) || (reinterpret_cast<uintptr_t>(theta16) & 7))
    return -2;
  AdamScalars s{sc[0], sc[1], sc[2], sc[3], sc[4], sc[5], sc[6], sc[7], sc[8]};
  long long blocks = ((n + 3) / 4 + 255) / 256;
  const long long cap = (long long)device_sms() * 8;
  if (blocks > cap) blocks = cap;
  adamw_sum_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, gp, theta, m, v, reinterpret_cast<hx*>(theta16), s);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
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
  if (cudaFuncGetAttributes(&a, (const void*)adamw_kernel) != cudaSuccess) return -1;
  return cudaFuncGetAttributes(&a, (const void*)adamw_sum_kernel) == cudaSuccess ? 0 : -1;
}
}  // namespace axonn
