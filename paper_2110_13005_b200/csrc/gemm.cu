// K1: persistent, warp-specialised bf16 GEMM on tcgen05 tensor cores (sm_100a).
//
//   C[z] (epilogue)= A[z] (M x K) * B[z] (N x K)^T       fp32 accumulation in TMEM
//
// Every contraction of the transformer layer ("transformer
// kernel") runs through this kernel:
// forward X W^T (A, B K-major), dgrad dY W (B MN-major), wgrad dY^T X (A and
// B MN-major) and the batched attention products (4-D TMA maps over
// (sample, head)).  Layout of one CTA (192 threads, 1 CTA / SM):
//   warp 0      TMA producer  (cp.async.bulk.tensor, SWIZZLE_128B, OOB zero fill)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld -> registers -> fused epilogue -> global
// smem ring of 4 stages (A 128x64 + B BNx64 bf16), TMEM double-buffered
// accumulators (2 x BN fp32 columns) so the epilogue of tile i overlaps the
// MMAs of tile i+1.  Tiles are walked persistently (tile = blockIdx.x +
// k*gridDim.x, M fastest so B tiles are shared through L2).
#include <cuda.h>
#include <cuda_runtime.h>
#include "half.cuh"
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ptx.cuh"
#include "kernels.h"

namespace axonn {

constexpr int BM = 128, BK = 64, STAGES = 4;
// 8 epilogue warps: two per TMEM lane quarter, each draining half of the tile's columns, so
// the fp32 read-modify-write (wgrad) and GeLU epilogues keep enough loads in flight.
constexpr int EPI_WARPS = 8;
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;

struct GemmParams {
  int M, N, K, Z, Z1;
  int a_mn, b_mn, causal, epi, accumulate;
  int col_group_in, col_group_out, n_valid;
  void* C;
  long long ldc, c_s1, c_s2;
  const hx* bias;
  const hx* resid;
  long long ld_resid;
  hx* aux;
  long long ld_aux;
  float alpha;
  int num_m, num_n, total;
  int raster_n;       // tile order: 1 = N fastest (see fill_params)
  // L2 policies of the pair kernel (fill_params): the operand every wave of tiles sweeps again is
  // loaded evict_last when it fits in L2, the other evict_normal; a bf16 output larger than
  // 100 MB (cannot stay in L2 anyway: the 1.68 GB of LM-head logits, FC1 activations, QKV) is
  // stored evict_first so it does not evict the operands; smaller outputs stay evict_normal,
  // the next kernel reads them at once (measured: evict_first on every output slowed the
  // dgrads 1-2 % in the step)
  int keep_a, keep_b, stream_c;
};



template <int TBM = BM>
__device__ __forceinline__ bool tile_coords(const GemmParams& p, int BN, int t, int& z, int& m0,
                                            int& n0, int& kb0, int& kb1) {
  int per = p.num_m * p.num_n;
  z = t / per;
  int r = t - z * per;
  int nb, mb;
  if (p.raster_n) {   // N fastest: concurrent tiles share the A panel (A >> L2, B small)
    mb = r / p.num_n;
    nb = r - mb * p.num_n;
  } else {            // M fastest: concurrent tiles share the B panel
    nb = r / p.num_m;
    mb = r - nb * p.num_m;
  }
  m0 = mb * TBM;
  n0 = nb * BN;
  int lo = 0, hi = p.K;
  if (p.causal == 1 && n0 > m0 + TBM - 1) return false;  // scores tile above the diagonal
  if (p.causal == 2) hi = min(p.K, m0 + TBM);            // keys <= last query of the tile
  if (p.causal == 3) lo = m0;                            // queries >= first key of the tile
  kb0 = lo / BK;
  kb1 = (hi + BK - 1) / BK;
  return kb1 > kb0;
}

// Tiles of one CTA pair: pair, pair + npairs, ... (static round robin over the raster order).
struct PairUnits {
  int pair, npairs, i;
  __device__ __forceinline__ PairUnits(int pr, int np) : pair(pr), npairs(np), i(0) {}
  template <int TBM>
  __device__ __forceinline__ bool next(const GemmParams& p, int BN, int& t, int& z, int& m0, int& n0,
                                       int& kb0, int& kb1) {
    for (;;) {
      t = pair + i * npairs;
      ++i;
      if (t >= p.total) return false;
      if (tile_coords<TBM>(p, BN, t, z, m0, n0, kb0, kb1)) return true;
    }
  }
};

// tanh on the SFU (MUFU.TANH, rel. error ~2^-11: below the bf16 rounding of the output)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_f(float x) {   // D-5 tanh GeLU
  const float c = 0.7978845608028654f, a = 0.044715f;
  return 0.5f * x * (1.0f + tanh_fast(c * (x + a * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  float t = tanh_fast(c * (x + a * x * x * x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * c * (1.0f + 3.0f * a * x * x);
}
__device__ __forceinline__ void ld8_bf16(const hx* p, float* f) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const hx2* h = reinterpret_cast<const hx2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = hx22f2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void st8_bf16(hx* p, const float* f) {
  uint4 u;
  hx2* h = reinterpret_cast<hx2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = f2hx2(f[2 * i], f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ bool al16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int z, int row, int col0,
                                               const uint32_t (&r)[32]) {
  if (row >= p.M) return;
  const int z1 = z % p.Z1, z2 = z / p.Z1;
  const int lim = min(p.n_valid, p.N);
  const int ncols = min(32, lim - col0);
  if (ncols <= 0) return;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;

  if (p.epi == EPI_F32) {
    float* C = reinterpret_cast<float*>(p.C) + z2 * p.c_s2 + z1 * p.c_s1 + row * p.ldc + col0;
    if (ncols == 32 && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
      float4* C4 = reinterpret_cast<float4*>(C);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 o = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        if (p.accumulate) {
          float4 c = C4[i];
          o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
        }
        C4[i] = o;
      }
    } else {
      for (int i = 0; i < ncols; ++i) C[i] = p.accumulate ? C[i] + v[i] : v[i];
    }
    return;
  }
  {  // fast path: full 32-column chunk, every operand 16-byte aligned -> 16-byte accesses only
    hx* dst = reinterpret_cast<hx*>(p.C) + z2 * p.c_s2 + z1 * p.c_s1 +
                         row * p.ldc + col0;
    hx* auxp = p.aux ? p.aux + row * p.ld_aux + col0 : nullptr;
    const hx* rsp = p.resid ? p.resid + row * p.ld_resid + col0 : nullptr;
    const hx* bp = p.bias ? p.bias + col0 : nullptr;
    if (ncols == 32 && p.col_group_in == 0 && al16(dst) && (!auxp || al16(auxp)) &&
        (!rsp || al16(rsp)) && (!bp || al16(bp)) && !p.accumulate) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float* w = v + 8 * j;
        float t[8];
        if (bp) {
          ld8_bf16(bp + 8 * j, t);
#pragma unroll
          for (int i = 0; i < 8; ++i) w[i] += t[i];
        }
        if (p.epi == EPI_BIAS_GELU) {
          st8_bf16(auxp + 8 * j, w);              // pre-activation (bf16) for the backward
#pragma unroll
          for (int i = 0; i < 8; ++i)             // GeLU of the same rounded value
            w[i] = gelu_f(hx2f(f2hx(w[i])));
        } else if (p.epi == EPI_DGELU) {
          ld8_bf16(auxp + 8 * j, t);
#pragma unroll
          for (int i = 0; i < 8; ++i) w[i] *= gelu_grad_f(t[i]);
        }
        if (rsp) {
          ld8_bf16(rsp + 8 * j, t);
#pragma unroll
          for (int i = 0; i < 8; ++i) w[i] += t[i];
        }
        st8_bf16(dst + 8 * j, w);
      }
      return;
    }
  }
  if (p.bias) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) v[i] += hx2f(p.bias[col0 + i]);
  }
  if (p.epi == EPI_BIAS_GELU) {
    hx* aux = p.aux + row * p.ld_aux + col0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i < ncols) {
        hx pre = f2hx(v[i]);
        aux[i] = pre;
        v[i] = gelu_f(hx2f(pre));
      }
    }
  } else if (p.epi == EPI_DGELU) {
    const hx* aux = p.aux + row * p.ld_aux + col0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) v[i] *= gelu_grad_f(hx2f(aux[i]));
  }
  if (p.resid) {
    const hx* rs = p.resid + row * p.ld_resid + col0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) v[i] += hx2f(rs[i]);
  }
  hx* C = reinterpret_cast<hx*>(p.C) + z2 * p.c_s2 + z1 * p.c_s1 + row * p.ldc;
  if (p.accumulate) {   // half weight gradient (D-38): C = RN(C + RN(v)), as the TMA reduce-add
    hx* dst = C + col0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) dst[i] = f2hx(hx2f(dst[i]) + hx2f(f2hx(v[i])));
    return;
  }
  if (p.col_group_in == 0) {
    hx* dst = C + col0;
    if (ncols == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        hx2 h0 = f2hx2(v[8 * i + 0], v[8 * i + 1]);
        hx2 h1 = f2hx2(v[8 * i + 2], v[8 * i + 3]);
        hx2 h2 = f2hx2(v[8 * i + 4], v[8 * i + 5]);
        hx2 h3 = f2hx2(v[8 * i + 6], v[8 * i + 7]);
        uint4 o;
        o.x = *reinterpret_cast<uint32_t*>(&h0);
        o.y = *reinterpret_cast<uint32_t*>(&h1);
        o.z = *reinterpret_cast<uint32_t*>(&h2);
        o.w = *reinterpret_cast<uint32_t*>(&h3);
        d4[i] = o;
      }
    } else {
      for (int i = 0; i < ncols; ++i) dst[i] = f2hx(v[i]);
    }
  } else {
    for (int i = 0; i < ncols; ++i) {
      int c = col0 + i;
      int dc = (c / p.col_group_in) * p.col_group_out + (c % p.col_group_in);
      C[dc] = f2hx(v[i]);
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB, const GemmParams p) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    {   // whole warp runs the loop; one elected lane issues the TMA copies
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
        int z, m0, n0, kb0, kb1;
        if (!tile_coords(p, BN, t, z, m0, n0, kb0, kb1)) continue;
        const int z1 = z % p.Z1, z2 = z / p.Z1;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            uint8_t* sA = smem + stage * STAGE_BYTES;
            uint8_t* sB = sA + A_BYTES;
            const int k0 = kb * BK;
            if (!p.a_mn) {
              tma_load_4d(sA, &mapA, &full[stage], k0, m0, z1, z2);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_4d(sA + j * 8192, &mapA, &full[stage], m0 + 64 * j, k0, z1, z2);
            }
            if (!p.b_mn) {
              tma_load_4d(sB, &mapB, &full[stage], k0, n0, z1, z2);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_4d(sB + j * 8192, &mapB, &full[stage], n0 + 64 * j, k0, z1, z2);
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {   // whole warp runs the loop; one elected lane issues the MMAs
      const uint32_t idesc = umma_idesc_f16(BM, BN, p.a_mn, p.b_mn);
      const uint32_t s0 = smem_u32(smem);
      const uint64_t a_d0 = p.a_mn ? umma_desc_sw128(s0, 8192, 1024) : umma_desc_sw128(s0, 16, 1024);
      const uint64_t b_d0 = p.b_mn ? umma_desc_sw128(s0 + A_BYTES, 8192, 1024)
                                   : umma_desc_sw128(s0 + A_BYTES, 16, 1024);
      const uint64_t a_k = p.a_mn ? (2048 >> 4) : (32 >> 4);
      const uint64_t b_k = p.b_mn ? (2048 >> 4) : (32 >> 4);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
        int z, m0, n0, kb0, kb1;
        if (!tile_coords(p, BN, t, z, m0, n0, kb0, kb1)) continue;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t so = (uint64_t)((stage * STAGE_BYTES) >> 4);
          const uint64_t ad = a_d0 + so, bd = b_d0 + so;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_f16_ss(tmem_d, ad + k * a_k, bd + k * b_k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[acc]);
        __syncwarp();
        ++it;
      }
    }
  } else {
    const int q = warp & 3;                     // TMEM lane quarter this warp may access
    const int cpart = (warp - 2) / 4;           // which column slice of the tile
    constexpr int CW = BN / (EPI_WARPS / 4);    // columns per epilogue warp
    int it = 0;
    for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
      int z, m0, n0, kb0, kb1;
      if (!tile_coords(p, BN, t, z, m0, n0, kb0, kb1)) continue;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      for (int c = cpart * CW; c < (cpart + 1) * CW; c += 32) {
        if (n0 + c >= p.N) break;
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c, r);
        epilogue_chunk(p, z, row, n0 + c, r);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ CTA-pair version
// cta_group::2: a cluster of 2 CTAs (one TPC) computes a 256 x 256 tile.  Each CTA
// stages its 128 rows of A and its 128 rows (N/2) of B; the leader's single thread
// issues M=256 N=256 K=16 MMAs reading both CTAs' shared memory, accumulating
// 128 lanes x 256 fp32 columns in each CTA's TMEM (double-buffered: 512 columns).
// Per-SM smem traffic per MMA is half the 1-CTA 128x256 tile's.
//
// TE (TMA epilogue): each epilogue warp drains its 32 rows x 128 columns through two
// 4 KB SWIZZLE_128B staging boxes in shared memory and writes them with TMA stores
// (bf16) or TMA reduce-adds performed in L2 (fp32 weight-gradient accumulation, D-20),
// so no thread issues a strided global access; residual / GeLU pre-activation inputs
// arrive the same way (TMA loads into the staging boxes, prefetched before the tile's
// accumulator is ready).
constexpr int STAGES2 = 6;
constexpr int STAGES2_TE = 5;
constexpr int TE_BOX = 4096;                       // 32 rows x 128 B
constexpr int TE_SMEM = EPI_WARPS * 2 * TE_BOX;    // two boxes per epilogue warp

__device__ __forceinline__ void ld8_bias(const hx* bias, int col, int N, float* f) {
  if (col + 8 <= N) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(bias + col));
    const hx2* hh = reinterpret_cast<const hx2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = hx22f2(hh[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = col + i < N ? hx2f(bias[col + i]) : 0.f;
  }
}
__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const hx2* hh = reinterpret_cast<const hx2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = hx22f2(hh[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  hx2* hh = reinterpret_cast<hx2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) hh[i] = f2hx2(f[2 * i], f[2 * i + 1]);
  return u;
}

template <int BN, bool TE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tcgen05_pair(const __grid_constant__ CUtensorMap mapA,
                           const __grid_constant__ CUtensorMap mapB, const GemmParams p,
                           const __grid_constant__ CUtensorMap mapC,
                           const __grid_constant__ CUtensorMap mapX) {
  static_assert(BN == 128 || BN == 256, "pair tiles: 256 x 128 or 256 x 256");
  constexpr int NST = TE ? STAGES2_TE : STAGES2;
  constexpr int TBM = 2 * BM;                 // 256 rows per pair
  constexpr int A_BYTES = BM * BK * 2;        // this CTA's 128 rows
  constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's BN/2 rows
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;      // double-buffered accumulator
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg_all = smem + NST * STAGE_BYTES;          // TE staging boxes (1024-aligned)
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + (TE ? TE_SMEM : 0));
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;                          // TE: one input barrier per epilogue warp
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ebar + EPI_WARPS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    if (TE) {
      tma_prefetch_desc(&mapC);
      tma_prefetch_desc(&mapX);
    }
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI_WARPS);   // epilogue warps of both CTAs
    }
    for (int w = 0; w < EPI_WARPS; ++w) mbar_init(&ebar[w], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    {   // whole warp runs the loop; one elected lane issues the TMA copies
      int stage = 0;
      uint32_t phase = 0;
      PairUnits pu(pair, npairs);
      int t, z, m0, n0, kb0, kb1;
      const uint64_t pol_a = p.keep_a ? l2_policy_evict_last() : l2_policy_evict_normal();
      const uint64_t pol_b = p.keep_b ? l2_policy_evict_last() : l2_policy_evict_normal();
      while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1)) {
        const int z1 = z % p.Z1, z2 = z / p.Z1;
        const int am = m0 + (int)rank * BM;
        const int bn = n0 + (int)rank * (BN / 2);   // this CTA's BN/2 rows of B
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
            uint8_t* sA = smem + stage * STAGE_BYTES;
            uint8_t* sB = sA + A_BYTES;
            const int k0 = kb * BK;
            if (!p.a_mn) {
              tma_load_4d_pair_hint(sA, &mapA, &full[stage], k0, am, z1, z2, pol_a);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_4d_pair_hint(sA + j * 8192, &mapA, &full[stage], am + 64 * j, k0, z1, z2, pol_a);
            }
            if (!p.b_mn) {
              tma_load_4d_pair_hint(sB, &mapB, &full[stage], k0, bn, z1, z2, pol_b);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 128; ++j)
                tma_load_4d_pair_hint(sB + j * 8192, &mapB, &full[stage], bn + 64 * j, k0, z1, z2, pol_b);
            }
          }
          __syncwarp();
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {   // whole warp runs the loop; one elected lane issues (uniform registers)
      const uint32_t idesc = umma_idesc_f16(TBM, BN, p.a_mn, p.b_mn);
      // descriptors of stage 0 and the per-stage / per-k16 increments (address field = addr >> 4)
      const uint32_t s0 = smem_u32(smem);
      const uint64_t a_d0 = p.a_mn ? umma_desc_sw128(s0, 8192, 1024) : umma_desc_sw128(s0, 16, 1024);
      const uint64_t b_d0 = p.b_mn ? umma_desc_sw128(s0 + A_BYTES, 8192, 1024)
                                   : umma_desc_sw128(s0 + A_BYTES, 16, 1024);
      const uint64_t a_k = p.a_mn ? (2048 >> 4) : (32 >> 4);
      const uint64_t b_k = p.b_mn ? (2048 >> 4) : (32 >> 4);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      PairUnits pu(pair, npairs);
      int t, z, m0, n0, kb0, kb1;
      while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1)) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t so = (uint64_t)((stage * STAGE_BYTES) >> 4);
          const uint64_t ad = a_d0 + so, bd = b_d0 + so;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_f16_ss_pair(tmem_d, ad + k * a_k, bd + k * b_k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            mma_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit_pair(&tfull[acc]);
        __syncwarp();
        ++it;
      }
    }
  } else if (!TE) {
    const int q = warp & 3;
    const int cpart = (warp - 2) / 4;
    constexpr int CW = BN / (EPI_WARPS / 4);
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
    int it = 0;
    PairUnits pu(pair, npairs);
    int t, z, m0, n0, kb0, kb1;
    while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1)) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + (int)rank * BM + q * 32 + lane;
      for (int c = cpart * CW; c < (cpart + 1) * CW; c += 32) {
        if (n0 + c >= p.N) break;
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c, r);
        epilogue_chunk(p, z, row, n0 + c, r);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      ++it;
    }
  } else {
    // ---------------- TMA epilogue: warp (q, cpart) owns rows [32 q, +32) x columns
    // [cpart * BN/2, +BN/2) of this CTA's 128 x BN accumulator.
    const int q = warp & 3, cpart = (warp - 2) / 4, wi = warp - 2;
    constexpr int CW = BN / 2;
    static_assert(CW == 256 || CW == 128 || CW == 64, "TE epilogue: 64..256 columns per warp");
    uint8_t* box0 = stg_all + wi * 2 * TE_BOX;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
    const bool f32 = p.epi == EPI_F32;
    const bool gelu = p.epi == EPI_BIAS_GELU;
    const bool has_in = p.epi == EPI_DGELU || (p.epi == EPI_HALF && p.resid != nullptr);
    const int sw = lane & 7;
    uint8_t* my_row0 = box0 + lane * 128;
    const uint64_t pol_c = p.stream_c ? l2_policy_evict_first() : l2_policy_evict_normal();
    uint32_t ephase = 0;
    int it = 0;
    PairUnits pu(pair, npairs);
    int t, z, m0, n0, kb0, kb1;
    while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1)) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int row0 = m0 + (int)rank * BM + q * 32;
      const int cb = n0 + cpart * CW;
      if (has_in && lane == 0) {   // residual / pre-activation boxes, before the accumulator
        bulk_wait_read<0>();
        mbar_arrive_expect_tx(&ebar[wi], (CW / 64) * TE_BOX);
#pragma unroll
        for (int g = 0; g < CW / 64; ++g) tma_load_2d(box0 + g * TE_BOX, &mapX, &ebar[wi], cb + 64 * g, row0);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + cpart * CW;
      if (f32) {
#pragma unroll 1
        for (int g = 0; g < CW / 32; ++g) {   // 32 fp32 columns = one 128-byte box row
          uint32_t r[32];
          tmem_ld32(tb + 32 * g, r);
          if (g == CW / 32 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
          }
          uint8_t* row = my_row0 + (g & 1) * TE_BOX;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 o = make_float4(__uint_as_float(r[4 * j]) * p.alpha, __uint_as_float(r[4 * j + 1]) * p.alpha,
                                   __uint_as_float(r[4 * j + 2]) * p.alpha, __uint_as_float(r[4 * j + 3]) * p.alpha);
            *reinterpret_cast<float4*>(row + ((j ^ sw) << 4)) = o;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (p.accumulate) tma_reduce_add_2d(&mapC, box0 + (g & 1) * TE_BOX, cb + 32 * g, row0);
            else tma_store_2d_hint(&mapC, box0 + (g & 1) * TE_BOX, cb + 32 * g, row0, pol_c);
            bulk_commit();
          }
        }
      } else {
        if (has_in) {
          mbar_wait(&ebar[wi], ephase);
          ephase ^= 1;
        }
#pragma unroll 1
        for (int g = 0; g < CW / 64; ++g) {   // 64 bf16 columns = one 128-byte box row
          uint32_t r0[32], r1[32];
          tmem_ld32_nowait(tb + 64 * g, r0);
          tmem_ld32_nowait(tb + 64 * g + 32, r1);
          tmem_ld_wait();
          if (g == CW / 64 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
          }
          // gelu: pre -> box 0, act -> box 1 (ring of two commits); else box g (in place)
          uint8_t* rowA = my_row0 + (gelu ? 0 : (g & 1)) * TE_BOX;
          uint8_t* rowB = my_row0 + TE_BOX;
          if (!has_in) {   // gelu rewrites both boxes; otherwise the other box may be in flight
            if (lane == 0) {
              if (gelu) bulk_wait_read<0>();
              else bulk_wait_read<1>();
            }
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              v[i] = __uint_as_float(j < 4 ? r0[8 * j + i] : r1[8 * (j - 4) + i]) * p.alpha;
            const int col = cb + 64 * g + 8 * j;
            if (p.bias) {
              float b8[8];
              ld8_bias(p.bias, col, p.N, b8);
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] += b8[i];
            }
            uint4* slot = reinterpret_cast<uint4*>(rowA + ((j ^ sw) << 4));
            if (gelu) {
              const uint4 pre = pack8(v);
              *slot = pre;
              unpack8(pre, v);   // GeLU of the same rounded value
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = gelu_f(v[i]);
              *reinterpret_cast<uint4*>(rowB + ((j ^ sw) << 4)) = pack8(v);
            } else {
              float in8[8];
              if (has_in) {
                unpack8(*slot, in8);
                if (p.epi == EPI_DGELU) {
#pragma unroll
                  for (int i = 0; i < 8; ++i) v[i] *= gelu_grad_f(in8[i]);
                } else {
#pragma unroll
                  for (int i = 0; i < 8; ++i) v[i] += in8[i];
                }
              }
              *slot = pack8(v);
            }
          }
          if (p.col_group_in) {
            // column remap (heads padded d -> dp, D-7): the warp copies the box out of the
            // staging tile itself, 8 bytes per lane, 16 lanes per row (a TMA store cannot split
            // the box at a group edge: it takes no negative coordinates and clips to 16 bytes)
            __syncwarp();
            const int c0 = cb + 64 * g, h0 = c0 / p.col_group_in, j0 = c0 - h0 * p.col_group_in;
            const int u = lane & 15, cu = c0 + 4 * u;
            const int hu = j0 + 4 * u >= p.col_group_in ? 1 : 0;
            const long long coff = (long long)(h0 + hu) * p.col_group_out + j0 + 4 * u - hu * p.col_group_in;
            hx* const Cb = reinterpret_cast<hx*>(p.C) + coff;
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
              const int r = 2 * i + (lane >> 4), grow = row0 + r;
              const uint2 val = *reinterpret_cast<const uint2*>(
                  box0 + (g & 1) * TE_BOX + r * 128 + ((((u >> 1) ^ (r & 7)) << 4) | ((u & 1) << 3)));
              if (cu < p.N && grow < p.M) *reinterpret_cast<uint2*>(Cb + (long long)grow * p.ldc) = val;
            }
            __syncwarp();
            continue;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (gelu) {
              tma_store_2d_hint(&mapX, box0, cb + 64 * g, row0, pol_c);            // pre-activation
              bulk_commit();
              tma_store_2d_hint(&mapC, box0 + TE_BOX, cb + 64 * g, row0, pol_c);   // GeLU
              bulk_commit();
            } else if (p.accumulate) {   // half weight gradient (D-38): C = RN(C + RN(acc)) in L2
              tma_reduce_add_2d(&mapC, box0 + (g & 1) * TE_BOX, cb + 64 * g, row0);
              bulk_commit();
            } else {
              tma_store_2d_hint(&mapC, box0 + (g & 1) * TE_BOX, cb + 64 * g, row0, pol_c);
              bulk_commit();
            }
          }
        }
      }
      ++it;
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encoder() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(ptr);
  }
  return fn;
}

// 4-D bf16 map (inner, outer, z1, z2); strides in elements; box (64, box_outer, 1, 1).
static int make_map(CUtensorMap* map, const void* base, long long inner, long long outer,
                    long long ld, int Z1, long long s1, int Z2, long long s2, int box_outer) {
  PFN_encodeTiled_t enc = get_encoder();
  if (!enc) return -1;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 2) % 16) return -2;
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)Z1, (cuuint64_t)Z2};
  long long st1 = Z1 > 1 ? s1 : ld * outer;
  long long st2 = Z2 > 1 ? s2 : st1 * Z1;
  if ((st1 * 2) % 16 || (st2 * 2) % 16) return -2;
  cuuint64_t strides[3] = {(cuuint64_t)(ld * 2), (cuuint64_t)(st1 * 2), (cuuint64_t)(st2 * 2)};
  cuuint32_t box[4] = {64, (cuuint32_t)box_outer, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, AXONN_TMA_HALF, 4, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -3;
}

// exported for the fused attention kernels (attn.cu)
int make_tmap_4d(CUtensorMap* map, const void* base, long long inner, long long outer,
                 long long ld, int Z1, long long s1, int Z2, long long s2, int box_outer) {
  return make_map(map, base, inner, outer, ld, Z1, s1, Z2, s2, box_outer);
}


static void fill_params(GemmParams& p, const GemmArgs& g, int tbm, int bn) {
  memset(&p, 0, sizeof(p));
  p.M = g.M; p.N = g.N; p.K = g.K; p.Z = g.Z; p.Z1 = g.Z1;
  p.a_mn = g.a_mn; p.b_mn = g.b_mn; p.causal = g.causal; p.epi = g.epi;
  p.accumulate = g.accumulate;
  p.col_group_in = g.col_group_in; p.col_group_out = g.col_group_out;
  p.n_valid = g.n_valid > 0 ? g.n_valid : g.N;
  p.C = g.C; p.ldc = g.ldc; p.c_s1 = g.c_s1; p.c_s2 = g.c_s2;
  p.bias = reinterpret_cast<const hx*>(g.bias);
  p.resid = reinterpret_cast<const hx*>(g.resid);
  p.ld_resid = g.ld_resid;
  p.aux = reinterpret_cast<hx*>(g.aux);
  p.ld_aux = g.ld_aux;
  p.alpha = g.alpha;
  p.num_m = (g.M + tbm - 1) / tbm;
  p.num_n = (g.N + bn - 1) / bn;
  p.total = p.num_m * p.num_n * g.Z;
  const int g_num_sms = device_sms();
  // M-fastest order re-reads A once per N column of tiles; when A is far larger than L2 and
  // B is small (LM-head weight gradient: A = dlogits^T 419 MB, B = 16.8 MB: 4.5x the
  // algorithmic DRAM bytes; FC1 weight gradient 2x, profiles/r1/k1_traffic.json), walk N
  // fastest so each A panel is read from DRAM once and B stays L2-resident
  // General rule: an operand larger than ~L2/4 is re-read from DRAM once per wave of tiles
  // that sweeps it; pick the order whose estimated DRAM bytes are smaller.
  {
    const double a_bytes = 2.0 * g.M * g.K, b_bytes = 2.0 * g.N * g.K;
    const int units = tbm == 2 * BM ? g_num_sms / 2 : g_num_sms;   // pairs or CTAs
    const double waves = (double)((p.total + units - 1) / units);
    const double big = 32e6;
    const double cost_m = (a_bytes > big ? a_bytes * waves : a_bytes) + b_bytes;
    const double cost_n = (b_bytes > big ? b_bytes * waves : b_bytes) + a_bytes;
    p.raster_n = (g.Z == 1 && p.num_n > 1 && cost_n < 0.9 * cost_m) ? 1 : 0;
    // the operand each later wave re-reads: A when M runs fastest, B when N does; keep it in
    // L2 if it fits beside everything else (<= 80 MB of the 126 MB L2)
    const double keep_max = 80e6;
    p.keep_a = (waves > 1 && !p.raster_n && a_bytes <= keep_max) ? 1 : 0;
    p.keep_b = (waves > 1 && p.raster_n && b_bytes <= keep_max) ? 1 : 0;
    p.stream_c = 2.0 * g.M * g.N * g.Z > 100e6 ? 1 : 0;

  }
}

// A box rows a_rows (K-major) / B box rows b_rows (K-major); MN-major boxes are 64 x 64.
static int make_maps(CUtensorMap& ma, CUtensorMap& mb, const GemmArgs& g, int a_rows, int b_rows) {
  int Z2 = g.Z / g.Z1;
  int rc;
  if (!g.a_mn)
    rc = make_map(&ma, g.A, g.K, g.M, g.lda, g.Z1, g.a_s1, Z2, g.a_s2, a_rows);
  else
    rc = make_map(&ma, g.A, g.M, g.K, g.lda, g.Z1, g.a_s1, Z2, g.a_s2, 64);
  if (rc) return rc;
  if (!g.b_mn)
    rc = make_map(&mb, g.B, g.K, g.N, g.ldb, g.Z1, g.b_s1, Z2, g.b_s2, b_rows);
  else
    rc = make_map(&mb, g.B, g.N, g.K, g.ldb, g.Z1, g.b_s1, Z2, g.b_s2, 64);
  return rc;
}

template <int BN>
static int launch_bn(const GemmArgs& g, cudaStream_t st) {
  constexpr int SMEM = STAGES * (BM * BK * 2 + BN * BK * 2) + 1024 + 256;
  static bool attr_set[kMaxDevices] = {};
  const int dev = cur_device();
  const int g_num_sms = device_sms();
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(gemm_bf16_tcgen05<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM) != cudaSuccess)
      return -10;
    attr_set[dev] = true;
  }
  CUtensorMap ma, mb;
  int rc = make_maps(ma, mb, g, BM, BN);
  if (rc) return rc;
  GemmParams p;
  fill_params(p, g, BM, BN);
  int grid = p.total < g_num_sms ? p.total : g_num_sms;
  if (g.max_ctas > 0 && grid > g.max_ctas) grid = g.max_ctas;
  gemm_bf16_tcgen05<BN><<<grid, GEMM_THREADS, SMEM, st>>>(ma, mb, p);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

// 2-D map over a row-major [rows][ld] matrix for the TMA epilogue: box = 32 rows x 128 B
// (64 bf16 or 32 fp32 columns), SWIZZLE_128B to match the staging layout.
static int make_map_epi(CUtensorMap* map, const void* base, long long cols, long long rows,
                        long long ld, bool f32) {
  PFN_encodeTiled_t enc = get_encoder();
  if (!enc) return -1;
  const int es = f32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * es) % 16) return -2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / es), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : AXONN_TMA_HALF, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -3;
}

static bool al16h(const void* p, long long ld, int es) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld * es) % 16 == 0;
}

// The TMA epilogue covers the linear layers: one batch, every output column valid, 16-byte
// aligned bases and row pitches; a column remap (QKV forward, attention-output dgrad at
// d != dp) only for the plain bf16 epilogue, with groups of a multiple of 4 columns.
static bool te_eligible(const GemmArgs& g) {
  if (g.Z != 1 || (g.n_valid > 0 && g.n_valid < g.N)) return false;
  if (g.col_group_in != 0 &&
      (g.epi != EPI_HALF || g.resid || g.accumulate || g.col_group_in > g.col_group_out ||
       g.col_group_in < 64 || g.col_group_in % 4 || g.col_group_out % 4 || g.ldc % 4 ||
       (long long)((g.N + g.col_group_in - 1) / g.col_group_in) * g.col_group_out > g.ldc))
    return false;
  if (g.epi == EPI_F32) return al16h(g.C, g.ldc, 4);
  if (g.epi != EPI_HALF && g.epi != EPI_BIAS_GELU && g.epi != EPI_DGELU) return false;
  if (g.accumulate && (g.epi != EPI_HALF || g.bias || g.resid || g.col_group_in)) return false;
  if (!al16h(g.C, g.ldc, 2)) return false;
  if (g.bias && (reinterpret_cast<uintptr_t>(g.bias) & 15)) return false;
  if ((g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU) && !al16h(g.aux, g.ld_aux, 2)) return false;
  if (g.epi == EPI_HALF && g.resid && !al16h(g.resid, g.ld_resid, 2)) return false;
  if ((g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU) && g.resid) return false;
  return true;
}

template <int BN, bool TE>
static int launch_pair(const GemmArgs& g, cudaStream_t st) {
  constexpr int NST = TE ? STAGES2_TE : STAGES2;
  constexpr int SMEM = NST * (BM * BK * 2 + (BN / 2) * BK * 2) + (TE ? TE_SMEM : 0) + 1024 + 256;
  static bool attr_set[kMaxDevices] = {};
  const int dev = cur_device();
  const int g_num_sms = device_sms();
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(gemm_bf16_tcgen05_pair<BN, TE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
      return -10;
    attr_set[dev] = true;
  }
  CUtensorMap ma, mb, mc, mx;
  int rc = make_maps(ma, mb, g, BM, BN / 2);   // each CTA stages BN/2 rows of B
  if (rc) return rc;
  memset(&mc, 0, sizeof(mc));
  memset(&mx, 0, sizeof(mx));
  if (TE) {
    // (a remapped output is stored by the epilogue warps; the map is only prefetched)
    rc = make_map_epi(&mc, g.C, g.col_group_in ? g.ldc : g.N, g.M, g.ldc, g.epi == EPI_F32);
    if (!rc && (g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU))
      rc = make_map_epi(&mx, g.aux, g.N, g.M, g.ld_aux, false);
    else if (!rc && g.resid)
      rc = make_map_epi(&mx, g.resid, g.N, g.M, g.ld_resid, false);
    if (rc) return rc;
  }
  GemmParams p;
  fill_params(p, g, 2 * BM, BN);
  int pairs_avail = g_num_sms / 2;
  if (g.max_ctas > 0 && pairs_avail > g.max_ctas / 2) pairs_avail = g.max_ctas / 2;
  const int pairs = p.total < pairs_avail ? p.total : pairs_avail;
  gemm_bf16_tcgen05_pair<BN, TE><<<2 * pairs, GEMM_THREADS, SMEM, st>>>(ma, mb, p, mc, mx);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

int gemm_launch(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.Z <= 0 || g.Z1 <= 0 || g.Z % g.Z1) return -1;
  // narrow outputs (N <= 128) and small M: single-CTA 128 x {128, 256} tiles (the narrow
  // attention-path GEMMs measured 30 us single-CTA vs 36 us as 256 x 128 pairs at the 1.3B
  // shape); variant 2 forces the 256 x 128 pair for them
  if (g.N <= 128 && g.M >= 256 && g.variant == 2) return launch_pair<128, false>(g, st);
  if (g.variant == 1 || (g.variant == 0 && (g.N <= 128 || g.M <= 128)))
    return g.N <= 128 ? launch_bn<128>(g, st) : launch_bn<256>(g, st);
  // linear layers: 256 x 256 CTA-pair tiles with the TMA epilogue where eligible (variant 3
  // forces the thread-store epilogue)
  if (g.variant != 3 && te_eligible(g)) return launch_pair<256, true>(g, st);
  return launch_pair<256, false>(g, st);
}

}  // namespace axonn

namespace axonn {
int preload_gemm() {   // see preload_ops (ops.cu)
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)gemm_bf16_tcgen05<128>, (const void*)gemm_bf16_tcgen05<256>,
                       (const void*)gemm_bf16_tcgen05_pair<256, false>,
                       (const void*)gemm_bf16_tcgen05_pair<256, true>,
                       (const void*)gemm_bf16_tcgen05_pair<128, false>};
  for (const void* f : fns)
    if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return -1;
  return 0;
}
}  // namespace axonn
