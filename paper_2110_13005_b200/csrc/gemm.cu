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
  int dbg;   // AXONN_RS_DEBUG experiments (row-softmax epilogue): 0 normal
  // hybrid stream-K schedule of the pair kernel (sk = 1): the first sk_dp tiles are dealt
  // data-parallel, the remaining tiles' k-blocks are split into equal contiguous ranges of
  // sk_L iterations per pair; a tile cut between pairs is finished (in fixed order) by the
  // pair holding its k-block 0 from the fp32 partials the others leave in sk_ws
  int sk, sk_dp, sk_L, kbt;
  int raster_n;       // tile order: 1 = N fastest (see fill_params)
  float* sk_ws;
  unsigned* sk_flag;
  unsigned sk_epoch;
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

// Work units of one CTA pair: (tile, k-block range, role).  role 0 whole tile, 1 partial
// (k-blocks after the first of its tile: written to the pair's workspace slot), 2 finisher
// (holds k-block 0 of a cut tile: adds the partials of pairs first_prod..last_prod).
struct PairUnits {
  int pair, npairs, i, nfull, it, it1;
  __device__ __forceinline__ PairUnits(const GemmParams& p, int pr, int np) : pair(pr), npairs(np) {
    i = 0;
    if (p.sk) {
      nfull = p.sk_dp / np;
      const int I = (p.total - p.sk_dp) * p.kbt;
      it = min(pr * p.sk_L, I);
      it1 = min(it + p.sk_L, I);
    } else {
      nfull = 0;
      it = it1 = 0;
    }
  }
  template <int TBM>
  __device__ __forceinline__ bool next(const GemmParams& p, int BN, int& t, int& z, int& m0, int& n0,
                                       int& kb0, int& kb1, int& role, int& last_prod) {
    role = 0;
    last_prod = -1;
    if (!p.sk) {
      for (;;) {
        t = pair + i * npairs;
        ++i;
        if (t >= p.total) return false;
        if (tile_coords<TBM>(p, BN, t, z, m0, n0, kb0, kb1)) return true;
      }
    }
    if (i < nfull) {
      t = pair + i * npairs;
      ++i;
      tile_coords<TBM>(p, BN, t, z, m0, n0, kb0, kb1);
      return true;
    }
    if (it >= it1) return false;
    const int ts = it / p.kbt;
    t = p.sk_dp + ts;
    tile_coords<TBM>(p, BN, t, z, m0, n0, kb0, kb1);
    kb0 = it % p.kbt;
    kb1 = min(p.kbt, kb0 + (it1 - it));
    it += kb1 - kb0;
    if (kb0 > 0) {
      role = 1;
    } else if (kb1 < p.kbt) {
      role = 2;
      last_prod = ((ts + 1) * p.kbt - 1) / p.sk_L;
    }
    return true;
  }
};

__device__ __forceinline__ void st_release_u32(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// Stream-K fixup by one epilogue warp on its 32 rows x ncol columns of the accumulator at
// TMEM address tb (lane base already applied).  role 1: store the partial to this pair's
// slot and publish it; role 2: wait for the partials of pairs pair+1..last_prod and add them
// (ascending pair order: deterministic) into TMEM before the regular epilogue runs.
template <int BN>
__device__ __forceinline__ void sk_fixup(const GemmParams& p, int role, int pair, int last_prod,
                                         uint32_t rank, int wi, int rloc, int col0, int ncol,
                                         uint32_t tb, int lane) {
  auto slot_row = [&](int pr) {
    return p.sk_ws + ((size_t)(pr * 2 + (int)rank) * 128 + rloc) * BN + col0;
  };
  if (role == 1) {
    float* w = slot_row(pair);
    for (int c = 0; c < ncol; c += 32) {
      uint32_t r[32];
      tmem_ld32(tb + c, r);
      float4* w4 = reinterpret_cast<float4*>(w + c);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        __stcg(w4 + j, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_u32(p.sk_flag + (pair * 2 + (int)rank) * 8 + wi, p.sk_epoch);
    return;
  }
  for (int pr = pair + 1; pr <= last_prod; ++pr) {
    if (lane == 0)
      while (ld_acquire_u32(p.sk_flag + (pr * 2 + (int)rank) * 8 + wi) != p.sk_epoch) {
      }
    __syncwarp();
  }
  for (int c = 0; c < ncol; c += 32) {
    uint32_t r[32];
    tmem_ld32(tb + c, r);
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    for (int pr = pair + 1; pr <= last_prod; ++pr) {
      const float4* w4 = reinterpret_cast<const float4*>(slot_row(pr) + c);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 a = __ldcg(w4 + j);
        v[4 * j] += a.x;
        v[4 * j + 1] += a.y;
        v[4 * j + 2] += a.z;
        v[4 * j + 3] += a.w;
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(v[i]);
    tmem_st32(tb + c, r);
  }
  tmem_st_wait();
}

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
        (!rsp || al16(rsp)) && (!bp || al16(bp))) {
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
          if (p.dbg == 7) {
            if (elect_one()) mbar_arrive(&full[stage]);
          } else if (elect_one()) {
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
      for (int c = cpart * CW; c < (cpart + 1) * CW && p.dbg != 8; c += 32) {
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
  // BN = 512: two N = 256 MMAs per k-step into one 512-column accumulator (no TMEM double
  // buffer); per SM 48 KB of operands per 1024 MMA cycles instead of 32 KB per 512
  constexpr int NST = TE ? (BN == 512 ? 3 : STAGES2_TE) : (BN == 512 ? 4 : STAGES2);
  constexpr int NH = BN > 256 ? BN / 256 : 1;  // N = 256 MMAs per k-step
  constexpr int TBM = 2 * BM;                 // 256 rows per pair
  constexpr int A_BYTES = BM * BK * 2;        // this CTA's 128 rows
  constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's BN/2 rows (NH chunks of 128)
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = (2 * BN <= 512) ? 2 * BN : BN;
  constexpr int NACC = TMEM_COLS / BN;        // accumulator buffers
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
      PairUnits pu(p, pair, npairs);
      int t, z, m0, n0, kb0, kb1, role, last_prod;
      while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1, role, last_prod)) {
        const int z1 = z % p.Z1, z2 = z / p.Z1;
        const int am = m0 + (int)rank * BM;
        const int bn = n0 + (int)rank * 128;   // this CTA's 128 B rows of each 256-wide N chunk
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            if (p.dbg == 7) {   // experiment: no operand traffic (MMA on stale smem)
              if (leader) mbar_arrive(&full[stage]);
            } else {
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
              uint8_t* sA = smem + stage * STAGE_BYTES;
              uint8_t* sB = sA + A_BYTES;
              const int k0 = kb * BK;
              if (!p.a_mn) {
                tma_load_4d_pair(sA, &mapA, &full[stage], k0, am, z1, z2);
              } else {
#pragma unroll
                for (int j = 0; j < BM / 64; ++j)
                  tma_load_4d_pair(sA + j * 8192, &mapA, &full[stage], am + 64 * j, k0, z1, z2);
              }
#pragma unroll
              for (int h = 0; h < NH; ++h) {
                const int bnh = bn + 256 * h;
                if (!p.b_mn) {
                  tma_load_4d_pair(sB + h * 16384, &mapB, &full[stage], k0, bnh, z1, z2);
                } else {
#pragma unroll
                  for (int j = 0; j < 2; ++j)
                    tma_load_4d_pair(sB + h * 16384 + j * 8192, &mapB, &full[stage], bnh + 64 * j, k0, z1, z2);
                }
              }
            }
          }
          __syncwarp();
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {   // whole warp runs the loop; one elected lane issues (uniform registers)
      const uint32_t idesc = umma_idesc_f16(TBM, BN > 256 ? 256 : BN, p.a_mn, p.b_mn);
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
      PairUnits pu(p, pair, npairs);
      int t, z, m0, n0, kb0, kb1, role, last_prod;
      while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1, role, last_prod)) {
        const int acc = NACC == 2 ? (it & 1) : 0;
        const uint32_t acc_phase = NACC == 2 ? ((it >> 1) & 1) : (it & 1);
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
#pragma unroll
              for (int h = 0; h < NH; ++h)
                mma_f16_ss_pair(tmem_d + 256 * h, ad + k * a_k, bd + (uint64_t)(h * (16384 >> 4)) + k * b_k,
                                 idesc, (kb > kb0 || k > 0) ? 1u : 0u);
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
    PairUnits pu(p, pair, npairs);
    int t, z, m0, n0, kb0, kb1, role, last_prod;
    while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1, role, last_prod)) {
      const int acc = NACC == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = NACC == 2 ? ((it >> 1) & 1) : (it & 1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (role) {
        sk_fixup<BN>(p, role, pair, last_prod, rank, warp - 2, q * 32 + lane, cpart * CW, CW,
                     tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + cpart * CW, lane);
        if (role == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
          ++it;
          continue;
        }
      }
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
    uint32_t ephase = 0;
    int it = 0;
    PairUnits pu(p, pair, npairs);
    int t, z, m0, n0, kb0, kb1, role, last_prod;
    while (pu.next<TBM>(p, BN, t, z, m0, n0, kb0, kb1, role, last_prod)) {
      const int acc = NACC == 2 ? (it & 1) : 0;
      const uint32_t acc_phase = NACC == 2 ? ((it >> 1) & 1) : (it & 1);
      const int row0 = m0 + (int)rank * BM + q * 32;
      const int cb = n0 + cpart * CW;
      if (role == 1) {   // stream-K partial: no epilogue, publish the fp32 partial
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        sk_fixup<BN>(p, 1, pair, last_prod, rank, wi, q * 32 + lane, cpart * CW, CW,
                     tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + cpart * CW, lane);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
        ++it;
        continue;
      }
      if (has_in && lane == 0) {   // residual / pre-activation boxes, before the accumulator
        bulk_wait_read<0>();
        mbar_arrive_expect_tx(&ebar[wi], (CW / 64) * TE_BOX);
#pragma unroll
        for (int g = 0; g < CW / 64; ++g) tma_load_2d(box0 + g * TE_BOX, &mapX, &ebar[wi], cb + 64 * g, row0);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + cpart * CW;
      if (role == 2) sk_fixup<BN>(p, 2, pair, last_prod, rank, wi, q * 32 + lane, cpart * CW, CW, tb, lane);
      if (p.dbg == 8) {   // experiment: no epilogue work
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      } else if (f32) {
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
            else tma_store_2d(&mapC, box0 + (g & 1) * TE_BOX, cb + 32 * g, row0);
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
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (gelu) {
              tma_store_2d(&mapX, box0, cb + 64 * g, row0);            // pre-activation
              bulk_commit();
              tma_store_2d(&mapC, box0 + TE_BOX, cb + 64 * g, row0);   // GeLU
              bulk_commit();
            } else {
              tma_store_2d(&mapC, box0 + (g & 1) * TE_BOX, cb + 64 * g, row0);
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

// ------------------------------------------------------------------ row-softmax variant
// Attention scores with the causal softmax (or its backward) fused into the epilogue:
// one tile = 128 query rows x ALL keys (N <= 512: two N=256 MMAs filling the 512 TMEM
// columns), so every epilogue thread owns a complete score row in TMEM.
//   EPI_SOFTMAX     : C = P = softmax_k<=q(alpha * Q K^T)        (bf16, zeros for k > q)
//   EPI_SOFTMAX_BWD : C = dS = alpha * P * (dP - sum_k P dP)     (acc = dP = dO V^T, P = aux)
// Removes the fp32 score round trip and the separate softmax kernels (D-7, D-8).
constexpr int RS_STAGES = 2;
constexpr int RS_THREADS = 64 + 32 * 8;                 // 8 epilogue warps
constexpr int RS_EPI_SMEM = 3 * 2 * 128 * 4 + 8 * 4096;  // partial max/sum/dot + staging

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// v2 epilogue of gemm_rowsoftmax.  Warp pair (q, half) owns TMEM lane quarter q (score rows
// r0 .. r0+31, r0 = m0 + 32 q) and key columns [256 half, 256 half + 256).  A 32-column
// chunk c0 of those rows is FULL (c0 + 32 <= r0: every key <= every query), the DIAGONAL
// chunk (c0 == r0: key i valid for lane >= i) or MASKED (c0 > r0) — warp-uniform, so
// only the diagonal chunk is predicated.  Forward: exp2 with the 1/sqrt(d) * log2(e) scale
// folded into one FFMA, computed once and written back to TMEM (tcgen05.st), then
// rescaled by 1/sum in the store pass.  Backward: P is exactly 0 above the diagonal, so
// dS = alpha * P * (dP - dot) needs no mask at all.  P / dS leave (and P arrives) through a
// per-warp swizzled 32 x 64 bf16 staging tile as coalesced 128-byte row segments.
__device__ __forceinline__ void rowsoftmax_epilogue2(const GemmParams& p, uint32_t tmem_base,
                                                     uint64_t* tfull, uint64_t* tempty, int warp,
                                                     int lane) {
  const int q = warp & 3, half = (warp - 2) >> 2;
  const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
  __shared__ float red2[3 * 2 * 128];
  __shared__ uint4 stg2[8 * 256];
  float* red_max = red2;
  float* red_sum = red2 + 256;
  float* red_dot = red2 + 512;
  uint4* stg = stg2 + (warp - 2) * 256;
  const int rl = q * 32 + lane;
  const bool fwd = p.epi == EPI_SOFTMAX;
  const float c1 = p.alpha * 1.4426950408889634f;   // alpha * log2(e)
  int it = 0;
  for (int t = blockIdx.x; t < p.total; t += gridDim.x, ++it) {
    const int z = t / p.num_m, m0 = (t % p.num_m) * BM;
    const int z1 = z % p.Z1, z2 = z / p.Z1;
    const int kv = min(p.N, m0 + BM);
    const int r0 = m0 + q * 32;                 // first row of this warp = its diagonal chunk
    const int c_lo = half * 256;
    const int c_end = min(p.N, c_lo + 256);     // my columns to write
    const int c_val = min(min(kv, c_lo + 256), r0 + 32);   // columns [c_lo, c_val) hold scores
    const int c_full = min(c_val, r0);          // [c_lo, c_full) are full chunks
    const bool has_diag = r0 >= c_lo && r0 < c_val;   // diagonal chunk [r0, r0+32) is mine
    const long long base = z2 * p.c_s2 + z1 * p.c_s1;
    hx* out = reinterpret_cast<hx*>(p.C) + base;
    const hx* Pin = p.aux + base;
    mbar_wait(tfull, it & 1);
    tc_fence_after();
    uint32_t r[32];
    auto stage_P = [&](int g0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = i * 4 + lane / 8, ch = lane % 8;
        const int gr = r0 + rr;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (gr < p.M && g0 + ch * 8 < p.N)
          v = *reinterpret_cast<const uint4*>(Pin + (long long)gr * p.ldc + g0 + ch * 8);
        stg[rr * 8 + (ch ^ (rr & 7))] = v;
      }
      __syncwarp();
    };
    auto flush = [&](int g0) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = i * 4 + lane / 8, ch = lane % 8;
        const int gr = r0 + rr;
        if (gr < p.M && g0 + ch * 8 < p.N)
          *reinterpret_cast<uint4*>(out + (long long)gr * p.ldc + g0 + ch * 8) =
              stg[rr * 8 + (ch ^ (rr & 7))];
      }
      __syncwarp();
    };
    auto put8 = [&](int j, const float* v8) {
      uint4 u;
      hx2* h2 = reinterpret_cast<hx2*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) h2[i] = f2hx2(v8[2 * i], v8[2 * i + 1]);
      stg[lane * 8 + (j ^ (lane & 7))] = u;
    };
    auto get8 = [&](int j, float* v8) {
      uint4 u = stg[lane * 8 + (j ^ (lane & 7))];
      const hx2* h2 = reinterpret_cast<const hx2*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = hx22f2(h2[i]);
        v8[2 * i] = f.x;
        v8[2 * i + 1] = f.y;
      }
    };
    if (fwd) {
      float mx = -3.0e38f;   // max of the raw scores (alpha > 0)
      for (int c0 = c_lo; c0 < c_full; c0 += 32) {
        tmem_ld32(trow + c0, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(r[i]));
      }
      if (has_diag) {   // diagonal chunk
        tmem_ld32(trow + r0, r);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i <= lane) mx = fmaxf(mx, __uint_as_float(r[i]));
      }
      red_max[half * 128 + rl] = mx;
      named_bar(1 + q, 64);
      const float moff = fmaxf(red_max[rl], red_max[128 + rl]) * c1;
      float s0 = 0.f, s1 = 0.f;
      for (int c0 = c_lo; c0 < c_full; c0 += 32) {
        tmem_ld32(trow + c0, r);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float e0 = ex2_approx(fmaf(__uint_as_float(r[i]), c1, -moff));
          const float e1 = ex2_approx(fmaf(__uint_as_float(r[i + 1]), c1, -moff));
          s0 += e0;
          s1 += e1;
          r[i] = __float_as_uint(e0);
          r[i + 1] = __float_as_uint(e1);
        }
        tmem_st32(trow + c0, r);
      }
      if (has_diag) {
        tmem_ld32(trow + r0, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float e = i <= lane ? ex2_approx(fmaf(__uint_as_float(r[i]), c1, -moff)) : 0.f;
          s0 += e;
          r[i] = __float_as_uint(e);
        }
        tmem_st32(trow + r0, r);
      }
      tmem_st_wait();
      red_sum[half * 128 + rl] = s0 + s1;
      named_bar(1 + q, 64);
      const float inv = 1.f / (red_sum[rl] + red_sum[128 + rl]);
      for (int g0 = c_lo; g0 < c_end; g0 += 64) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c0 = g0 + 32 * hh;
          float v[32];
          if (c0 < c_val) {
            tmem_ld32(trow + c0, r);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * inv;
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) put8(4 * hh + j, v + 8 * j);
        }
        flush(g0);
      }
    } else {   // EPI_SOFTMAX_BWD
      float d0 = 0.f, d1 = 0.f;
      for (int g0 = c_lo; g0 < c_val; g0 += 64) {
        stage_P(g0);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c0 = g0 + 32 * hh;
          if (c0 < c_val) {
            tmem_ld32(trow + c0, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float pv[8];
              get8(4 * hh + j, pv);
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                d0 = fmaf(pv[i], __uint_as_float(r[8 * j + i]), d0);
                d1 = fmaf(pv[i + 1], __uint_as_float(r[8 * j + i + 1]), d1);
              }
            }
          }
        }
        __syncwarp();
      }
      red_dot[half * 128 + rl] = d0 + d1;
      named_bar(1 + q, 64);
      const float dot = red_dot[rl] + red_dot[128 + rl];
      for (int g0 = c_lo; g0 < c_end; g0 += 64) {
        if (g0 < c_val) stage_P(g0);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c0 = g0 + 32 * hh;
          float v[32];
          if (c0 < c_val) {
            tmem_ld32(trow + c0, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float pv[8];
              get8(4 * hh + j, pv);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                v[8 * j + i] = p.alpha * pv[i] * (__uint_as_float(r[8 * j + i]) - dot);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j) put8(4 * hh + j, v + 8 * j);
        }
        flush(g0);
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty);
  }
}

// Epilogue of gemm_rowsoftmax: warp pair (q, half) owns TMEM lane quarter q (32 score rows)
// and key columns [256 half, 256 half + 256).  Row statistics are combined across the pair
// through shared memory; P / dS rows leave (and P rows arrive) through a per-warp swizzled
// 32 x 64 bf16 staging tile so every global access is a coalesced 128-byte row segment.
__device__ __forceinline__ void rowsoftmax_epilogue(const GemmParams& p, uint32_t tmem_base,
                                                    uint64_t* tfull, uint64_t* tempty,
                                                    uint8_t* scratch, int warp, int lane) {
  const int q = warp & 3, half = (warp - 2) >> 2;
  const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
  // static __shared__ so the compiler emits STS/LDS (a pointer laundered through integer
  // arithmetic on the dynamic smem base turns into slow generic ST.E/LD.E)
  __shared__ float red_s[3 * 2 * 128];
  __shared__ uint4 stg_s[8 * 256];
  (void)scratch;
  float* red_max = red_s;                                  // [2][128]
  float* red_sum = red_s + 256;
  float* red_dot = red_s + 512;
  uint4* stg = stg_s + (warp - 2) * 256;                   // 32 rows x 8 x 16 B per warp
  const int rl = q * 32 + lane;                            // row within the 128-row tile
  const bool fwd = p.epi == EPI_SOFTMAX;
  int it = 0;
  for (int t = blockIdx.x; t < p.total; t += gridDim.x, ++it) {
    const int z = t / p.num_m, m0 = (t % p.num_m) * BM;
    const int z1 = z % p.Z1, z2 = z / p.Z1;
    const int kv = min(p.N, m0 + BM);
    const int row = m0 + rl;
    const long long base = z2 * p.c_s2 + z1 * p.c_s1;
    hx* out = reinterpret_cast<hx*>(p.C) + base;
    const hx* Pin = p.aux + base;
    const int c_lo = half * 256;
    const int c_hi = min(kv, c_lo + 256);                    // my columns holding scores
    const int c_end = min(p.N, c_lo + 256);                  // my columns to write
    mbar_wait(tfull, it & 1);
    tc_fence_after();
    uint32_t r[32];
    // coalesced load of P rows [m0 + 32 q, +32) x [g0, g0 + 64) into the staging tile
    auto stage_P = [&](int g0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = i * 4 + lane / 8, ch = lane % 8;
        const int gr = m0 + q * 32 + rr;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (gr < p.M && g0 + ch * 8 < p.N)
          v = *reinterpret_cast<const uint4*>(Pin + (long long)gr * p.ldc + g0 + ch * 8);
        stg[rr * 8 + (ch ^ (rr & 7))] = v;
      }
      __syncwarp();
    };
    // coalesced store of the staging tile to out rows [m0 + 32 q, +32) x [g0, g0 + 64)
    auto flush = [&](int g0) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = i * 4 + lane / 8, ch = lane % 8;
        const int gr = m0 + q * 32 + rr;
        if (gr < p.M && g0 + ch * 8 < p.N && p.dbg != 2)   // rows shorter than a 64-col group
          *reinterpret_cast<uint4*>(out + (long long)gr * p.ldc + g0 + ch * 8) = stg[rr * 8 + (ch ^ (rr & 7))];
      }
      __syncwarp();
    };
    auto put_row = [&](int j, const float* v8) {   // this thread's row, 16-byte chunk j
      uint4 u;
      hx2* h2 = reinterpret_cast<hx2*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) h2[i] = f2hx2(v8[2 * i], v8[2 * i + 1]);
      stg[lane * 8 + (j ^ (lane & 7))] = u;
    };
    auto get_row = [&](int j, float* v8) {
      uint4 u = stg[lane * 8 + (j ^ (lane & 7))];
      const hx2* h2 = reinterpret_cast<const hx2*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = hx22f2(h2[i]);
        v8[2 * i] = f.x;
        v8[2 * i + 1] = f.y;
      }
    };
    if (p.dbg == 4) {            // experiment: no epilogue work at all
    } else if (p.dbg == 3) {     // experiment: TMEM reads only
      float acc = 0.f;
      for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
        tmem_ld32(trow + c0, r);
        acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
      }
      if (acc == 1234.5f) red_max[rl] = acc;
    } else if (fwd) {
      float mx = -3.0e38f;
      for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
        tmem_ld32(trow + c0, r);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i <= row) mx = fmaxf(mx, __uint_as_float(r[i]) * p.alpha);
      }
      red_max[half * 128 + rl] = mx;
      named_bar(1 + q, 64);
      mx = fmaxf(red_max[rl], red_max[128 + rl]);
      float sum = 0.f;
      for (int c0 = c_lo; c0 < c_hi && p.dbg != 5; c0 += 32) {
        tmem_ld32(trow + c0, r);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i <= row) sum += __expf(__uint_as_float(r[i]) * p.alpha - mx);
      }
      red_sum[half * 128 + rl] = sum;
      named_bar(1 + q, 64);
      const float inv = 1.f / (red_sum[rl] + red_sum[128 + rl]);
      for (int g0 = c_lo; g0 < c_end && p.dbg < 5; g0 += 64) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c0 = g0 + 32 * hh;
          float v[32];
          if (c0 < c_hi) {
            tmem_ld32(trow + c0, r);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              v[i] = (c0 + i <= row) ? __expf(__uint_as_float(r[i]) * p.alpha - mx) * inv : 0.f;
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) put_row(4 * hh + j, v + 8 * j);
        }
        flush(g0);
      }
    } else {   // EPI_SOFTMAX_BWD: dS = alpha * P * (dP - rowsum(P dP))
      float dot = 0.f;
      for (int g0 = c_lo; g0 < c_hi; g0 += 64) {
        stage_P(g0);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c0 = g0 + 32 * hh;
          if (c0 < c_hi) {
            tmem_ld32(trow + c0, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float pv[8];
              get_row(4 * hh + j, pv);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (c0 + 8 * j + i <= row) dot += pv[i] * __uint_as_float(r[8 * j + i]);
            }
          }
        }
        __syncwarp();
      }
      red_dot[half * 128 + rl] = dot;
      named_bar(1 + q, 64);
      dot = red_dot[rl] + red_dot[128 + rl];
      for (int g0 = c_lo; g0 < c_end; g0 += 64) {
        if (g0 < c_hi) stage_P(g0);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c0 = g0 + 32 * hh;
          float v[32];
          if (c0 < c_hi) {
            tmem_ld32(trow + c0, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float pv[8];
              get_row(4 * hh + j, pv);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                v[8 * j + i] = (c0 + 8 * j + i <= row)
                                   ? p.alpha * pv[i] * (__uint_as_float(r[8 * j + i]) - dot) : 0.f;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          __syncwarp();   // everyone has read its P chunk before it is overwritten
#pragma unroll
          for (int j = 0; j < 4; ++j) put_row(4 * hh + j, v + 8 * j);
        }
        flush(g0);
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty);
  }
}
__global__ void __launch_bounds__(RS_THREADS, 1)
    gemm_rowsoftmax(const __grid_constant__ CUtensorMap mapA,
                    const __grid_constant__ CUtensorMap mapB, const GemmParams p) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int HALF_BYTES = 256 * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + 2 * HALF_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RS_STAGES * STAGE_BYTES);
  uint64_t* empty = full + RS_STAGES;
  uint64_t* tfull = empty + RS_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < RS_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 8);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int nkb = (p.K + BK - 1) / BK;

  if (warp == 0) {
    {   // whole warp; elected lane issues
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
        const int z = t / p.num_m, m0 = (t % p.num_m) * BM;
        const int z1 = z % p.Z1, z2 = z / p.Z1;
        const int kv = min(p.N, m0 + BM);
        const int nh = kv > 256 ? 2 : 1;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&full[stage], A_BYTES + nh * HALF_BYTES);
            uint8_t* sA = smem + stage * STAGE_BYTES;
            tma_load_4d(sA, &mapA, &full[stage], kb * BK, m0, z1, z2);
            for (int hh = 0; hh < nh; ++hh)
              tma_load_4d(sA + A_BYTES + hh * HALF_BYTES, &mapB, &full[stage], kb * BK, 256 * hh, z1, z2);
          }
          __syncwarp();
          if (++stage == RS_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {   // whole warp; elected lane issues
      const uint32_t idesc = umma_idesc_f16(BM, 256, 0, 0);
      const uint64_t d0 = umma_desc_sw128(smem_u32(smem), 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < p.total; t += gridDim.x, ++it) {
        const int m0 = (t % p.num_m) * BM;
        const int kv = min(p.N, m0 + BM);
        const int nh = kv > 256 ? 2 : 1;
        mbar_wait(tempty, (it & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = d0 + (uint64_t)((stage * STAGE_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              for (int hh = 0; hh < nh; ++hh) {
                const uint64_t bd = ad + (uint64_t)((A_BYTES + hh * HALF_BYTES) >> 4);
                mma_f16_ss(tmem_base + 256 * hh, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              }
            }
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == RS_STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(tfull);
        __syncwarp();
      }
    }
  } else {
    rowsoftmax_epilogue2(p, tmem_base, tfull, tempty, warp, lane);
  }
#if 0   // previous 4-warp row-per-thread epilogue (kept for reference, not compiled)
  } else {
    const int q = warp & 3;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    int it = 0;
    for (int t = blockIdx.x; t < p.total; t += gridDim.x, ++it) {
      const int z = t / p.num_m, m0 = (t % p.num_m) * BM;
      const int z1 = z % p.Z1, z2 = z / p.Z1;
      const int kv = min(p.N, m0 + BM);
      const int row = m0 + q * 32 + lane;
      const bool live = row < p.M;
      const long long off = z2 * p.c_s2 + z1 * p.c_s1 + (long long)row * p.ldc;
      hx* out = reinterpret_cast<hx*>(p.C) + off;
      const hx* Pin = p.aux + off;
      mbar_wait(tfull, it & 1);
      tc_fence_after();
      uint32_t r[32];
      if (p.epi == EPI_SOFTMAX) {
        float mx = -3.0e38f;
        for (int c0 = 0; c0 < kv; c0 += 32) {
          tmem_ld32(trow + c0, r);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c0 + i <= row) mx = fmaxf(mx, __uint_as_float(r[i]) * p.alpha);
        }
        float sum = 0.f;
        for (int c0 = 0; c0 < kv; c0 += 32) {
          tmem_ld32(trow + c0, r);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c0 + i <= row) sum += __expf(__uint_as_float(r[i]) * p.alpha - mx);
        }
        const float inv = 1.f / sum;
        for (int c0 = 0; c0 < p.N; c0 += 32) {
          float v[32];
          if (c0 < kv) {
            tmem_ld32(trow + c0, r);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              v[i] = (c0 + i <= row) ? __expf(__uint_as_float(r[i]) * p.alpha - mx) * inv : 0.f;
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          if (live) {
            uint4* d4 = reinterpret_cast<uint4*>(out + c0);
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
          }
        }
      } else {   // EPI_SOFTMAX_BWD
        float dot = 0.f;
        for (int c0 = 0; c0 < kv; c0 += 32) {
          tmem_ld32(trow + c0, r);
          if (live) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 pv = *reinterpret_cast<const uint4*>(Pin + c0 + i);
              const hx2* ph = reinterpret_cast<const hx2*>(&pv);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float2 pf = hx22f2(ph[j]);
                if (c0 + i + 2 * j <= row) dot += pf.x * __uint_as_float(r[i + 2 * j]);
                if (c0 + i + 2 * j + 1 <= row) dot += pf.y * __uint_as_float(r[i + 2 * j + 1]);
              }
            }
          }
        }
        for (int c0 = 0; c0 < p.N; c0 += 32) {
          float v[32];
          if (c0 < kv) {
            tmem_ld32(trow + c0, r);
            if (live) {
#pragma unroll
              for (int i = 0; i < 32; i += 8) {
                uint4 pv = *reinterpret_cast<const uint4*>(Pin + c0 + i);
                const hx2* ph = reinterpret_cast<const hx2*>(&pv);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  float2 pf = hx22f2(ph[j]);
                  v[i + 2 * j] = (c0 + i + 2 * j <= row)
                                     ? p.alpha * pf.x * (__uint_as_float(r[i + 2 * j]) - dot) : 0.f;
                  v[i + 2 * j + 1] = (c0 + i + 2 * j + 1 <= row)
                                         ? p.alpha * pf.y * (__uint_as_float(r[i + 2 * j + 1]) - dot) : 0.f;
                }
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          if (live) {
            uint4* d4 = reinterpret_cast<uint4*>(out + c0);
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
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
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

static int g_num_sms = 0;

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
  if (g_num_sms == 0) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
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
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_bf16_tcgen05<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM) != cudaSuccess)
      return -10;
    attr_set = true;
  }
  CUtensorMap ma, mb;
  int rc = make_maps(ma, mb, g, BM, BN);
  if (rc) return rc;
  GemmParams p;
  fill_params(p, g, BM, BN);
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("AXONN_GEMM_DBG");
      dbg = e ? atoi(e) : 0;
    }
    p.dbg = dbg;
  }
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

// The TMA epilogue covers the linear layers: one batch, no column remap, every output
// column valid, 16-byte aligned bases and row pitches.
static bool te_eligible(const GemmArgs& g) {
  if (g.Z != 1 || g.col_group_in != 0 || (g.n_valid > 0 && g.n_valid < g.N)) return false;
  if (g.epi == EPI_F32) return al16h(g.C, g.ldc, 4);
  if (g.epi != EPI_HALF && g.epi != EPI_BIAS_GELU && g.epi != EPI_DGELU) return false;
  if (!al16h(g.C, g.ldc, 2)) return false;
  if (g.bias && (reinterpret_cast<uintptr_t>(g.bias) & 15)) return false;
  if ((g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU) && !al16h(g.aux, g.ld_aux, 2)) return false;
  if (g.epi == EPI_HALF && g.resid && !al16h(g.resid, g.ld_resid, 2)) return false;
  if ((g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU) && g.resid) return false;
  return true;
}

static int g_te_mode = -1;   // AXONN_GEMM_TE=0 disables the TMA epilogue
static int g_bn512 = -1;     // AXONN_GEMM_BN512=1: 256 x 512 pair tiles where eligible
// AXONN_GEMM_SK=1 enables the hybrid stream-K schedule.  Off by default: measured slower on
// every layer shape (proj fwd 37.8 -> 53.2 us, FC1 dgrad 119.8 -> 148.5 us,
// profiles/r1/diag_stream_k.jsonl) — the data-parallel order keeps the pairs that share an
// operand panel on the same k-block at the same time (L2 serves them together), and the
// GEMMs are L2 -> SM bound; pieces starting mid-tile lose that alignment.
static int g_sk_mode = -1;

// Stream-K workspaces, one per concurrently launching stream (s_comp and s_wg run GEMMs at
// the same time): fp32 [74 pairs][2 CTAs][128 x 256] partials + per-warp flags.
constexpr int SK_SLOTS = 4;
static float* g_sk_ws[SK_SLOTS] = {};
static unsigned* g_sk_flag[SK_SLOTS] = {};
static unsigned g_sk_epoch[SK_SLOTS] = {};
static cudaStream_t g_sk_stream[SK_SLOTS] = {};
static int sk_slot(cudaStream_t st) {
  for (int i = 0; i < SK_SLOTS; ++i)
    if (g_sk_ws[i] && g_sk_stream[i] == st) return i;
  for (int i = 0; i < SK_SLOTS; ++i)
    if (!g_sk_ws[i]) {
      const size_t ws = (size_t)80 * 2 * 128 * 256 * 4;
      if (cudaMalloc(&g_sk_ws[i], ws) != cudaSuccess) return -1;
      if (cudaMalloc(&g_sk_flag[i], 80 * 2 * 8 * 4) != cudaSuccess) return -1;
      if (cudaMemset(g_sk_flag[i], 0, 80 * 2 * 8 * 4) != cudaSuccess) return -1;
      g_sk_stream[i] = st;
      return i;
    }
  return -1;
}

template <int BN, bool TE>
static int launch_pair(const GemmArgs& g, cudaStream_t st) {
  constexpr int NST = TE ? (BN == 512 ? 3 : STAGES2_TE) : (BN == 512 ? 4 : STAGES2);
  constexpr int SMEM = NST * (BM * BK * 2 + (BN / 2) * BK * 2) + (TE ? TE_SMEM : 0) + 1024 + 256;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_bf16_tcgen05_pair<BN, TE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
      return -10;
    attr_set = true;
  }
  CUtensorMap ma, mb, mc, mx;
  int rc = make_maps(ma, mb, g, BM, 128);
  if (rc) return rc;
  memset(&mc, 0, sizeof(mc));
  memset(&mx, 0, sizeof(mx));
  if (TE) {
    rc = make_map_epi(&mc, g.C, g.N, g.M, g.ldc, g.epi == EPI_F32);
    if (!rc && (g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU))
      rc = make_map_epi(&mx, g.aux, g.N, g.M, g.ld_aux, false);
    else if (!rc && g.resid)
      rc = make_map_epi(&mx, g.resid, g.N, g.M, g.ld_resid, false);
    if (rc) return rc;
  }
  GemmParams p;
  fill_params(p, g, 2 * BM, BN);
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("AXONN_GEMM_DBG");
      dbg = e ? atoi(e) : 0;
    }
    p.dbg = dbg;
  }
  int pairs_avail = g_num_sms / 2;
  if (g.max_ctas > 0 && pairs_avail > g.max_ctas / 2) pairs_avail = g.max_ctas / 2;
  int pairs = p.total < pairs_avail ? p.total : pairs_avail;
  // hybrid stream-K when the last wave of whole tiles would leave pairs idle (T % P != 0,
  // few waves); all but one full wave stay data-parallel
  p.kbt = (g.K + BK - 1) / BK;
  if (g_sk_mode < 0) {
    const char* e = getenv("AXONN_GEMM_SK");
    g_sk_mode = (e && e[0] == '1') ? 1 : 0;
  }
  const int T = p.total, P = pairs_avail;
  if (g_sk_mode && !g.no_sk && g.causal == 0 && g.Z == 1 && T % P != 0 && T < 6 * P && p.kbt >= 8 &&
      P <= 80 && p.dbg == 0) {
    const int slot = sk_slot(st);
    if (slot >= 0) {
      p.sk = 1;
      p.sk_dp = T >= P ? (T / P - 1) * P : 0;
      const int I = (T - p.sk_dp) * p.kbt;
      p.sk_L = (I + P - 1) / P;
      p.sk_ws = g_sk_ws[slot];
      p.sk_flag = g_sk_flag[slot];
      p.sk_epoch = ++g_sk_epoch[slot];
      pairs = P;
    }
  }
  gemm_bf16_tcgen05_pair<BN, TE><<<2 * pairs, GEMM_THREADS, SMEM, st>>>(ma, mb, p, mc, mx);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

static int launch_rowsoftmax(const GemmArgs& g, cudaStream_t st) {
  // dynamic part only; the epilogue's RS_EPI_SMEM bytes are static __shared__
  constexpr int SMEM = RS_STAGES * (BM * BK * 2 + 2 * 256 * BK * 2) + 1024 + 256;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_rowsoftmax, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) !=
        cudaSuccess)
      return -10;
    attr_set = true;
  }
  if (g.N > 512 || g.N % 32 || g.a_mn || g.b_mn || (g.ldc % 8) || (g.c_s1 % 8) || (g.c_s2 % 8))
    return -1;
  CUtensorMap ma, mb;
  int rc = make_maps(ma, mb, g, BM, 256);
  if (rc) return rc;
  GemmParams p;
  fill_params(p, g, BM, 512);
  p.num_n = 1;
  p.total = p.num_m * g.Z;
  {
    const char* e = getenv("AXONN_RS_DEBUG");
    p.dbg = e ? atoi(e) : 0;
  }
  int grid = p.total < g_num_sms ? p.total : g_num_sms;
  if (g.max_ctas > 0 && grid > g.max_ctas) grid = g.max_ctas;
  gemm_rowsoftmax<<<grid, RS_THREADS, SMEM, st>>>(ma, mb, p);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

static int g_pair_mode = -1;   // AXONN_GEMM_PAIR=0 disables the CTA-pair kernel

int gemm_launch(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.Z <= 0 || g.Z1 <= 0 || g.Z % g.Z1) return -1;
  if (g_pair_mode < 0) {
    const char* e = getenv("AXONN_GEMM_PAIR");
    g_pair_mode = (e && e[0] == '0') ? 0 : 1;
  }
  if (g.epi == EPI_SOFTMAX || g.epi == EPI_SOFTMAX_BWD) return launch_rowsoftmax(g, st);
  // narrow outputs (attention P V, dQ, dK, dV: N = head dim): 256 x 128 pair tiles halve the
  // per-SM A traffic of 128 x 128 single-CTA tiles
  // (measured: 36 us vs 30 us for the single-CTA 128 x 128 tiles at the 1.3B attention shape,
  // so narrow GEMMs use the pair only when forced with variant 2)
  if (g_te_mode < 0) {
    const char* e = getenv("AXONN_GEMM_TE");
    g_te_mode = (e && e[0] == '0') ? 0 : 1;
  }
  if (g.N <= 128 && g.M >= 256 && g.variant == 2) return launch_pair<128, false>(g, st);
  if (g.variant == 1 || (g.variant == 0 && (g.N <= 128 || !g_pair_mode || g.M <= 128)))
    return g.N <= 128 ? launch_bn<128>(g, st) : launch_bn<256>(g, st);
  if (g_bn512 < 0) {
    const char* e = getenv("AXONN_GEMM_BN512");
    g_bn512 = (e && e[0] == '1') ? 1 : 0;
  }
  // 256 x 512 pair tiles: epilogues without a tile-sized input (two staging boxes per warp)
  if (g_te_mode && te_eligible(g) && (g.variant == 4 || (g.variant == 0 && g_bn512)) &&
      g.N >= 2048 && !(g.epi == EPI_DGELU || (g.epi == EPI_HALF && g.resid)))
    return launch_pair<512, true>(g, st);
  if (g_te_mode && g.variant != 3 && te_eligible(g)) return launch_pair<256, true>(g, st);
  return launch_pair<256, false>(g, st);
}

}  // namespace axonn

namespace axonn {
int preload_gemm() {   // see preload_ops (ops.cu)
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)gemm_bf16_tcgen05<128>, (const void*)gemm_bf16_tcgen05<256>,
                       (const void*)gemm_bf16_tcgen05_pair<256, false>,
                       (const void*)gemm_bf16_tcgen05_pair<256, true>,
                       (const void*)gemm_bf16_tcgen05_pair<512, true>,
                       (const void*)gemm_bf16_tcgen05_pair<128, false>, (const void*)gemm_rowsoftmax};
  for (const void* f : fns)
    if (cudaFuncGetAttributes(&a, f) != cudaSuccess) return -1;
  return 0;
}
}  // namespace axonn
