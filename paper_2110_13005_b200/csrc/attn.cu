// Fused causal self-attention on tcgen05 (sm_100a) for the stage forward and backward (SURVEY.md
// §8(a) A2 / A4: "causal MHA"; readings D-7 scale 1/sqrt(d), D-8 causal mask).
// Forward: attn_fwd2_kernel (streamed key blocks, online softmax, two query tiles ping-ponged on
// the tensor core; S and P never leave TMEM).  Backward: attn_bwd_kernel<KA> (dK, dV) and
// <!KA> (dQ) with P recomputed from S and the forward's log2-domain row normaliser.
#include <cuda.h>
#include <cuda_runtime.h>
#include "half.cuh"
#include <cstring>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "kernels.h"
#include "ptx.cuh"

namespace axonn {

namespace {

__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// 32 lanes x 16 columns (32-bit) register -> TMEM
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void nbar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// Store up to 8 16-bit values (v) at dst, nvalid of them valid (even).  Head widths that are
// not a multiple of 8 (d = 188, 176) leave head bases only 8-byte aligned: 8-byte stores.
__device__ __forceinline__ void store8h(hx* dst, const uint4 v, int nvalid) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
  if (nvalid >= 8 && (a & 15) == 0) {
    *reinterpret_cast<uint4*>(dst) = v;
    return;
  }
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if ((a & 7) == 0) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      if (4 * hh + 4 <= nvalid)
        *reinterpret_cast<uint2*>(dst + 4 * hh) = make_uint2(w[2 * hh], w[2 * hh + 1]);
      else if (4 * hh + 2 <= nvalid)
        *reinterpret_cast<uint32_t*>(dst + 4 * hh) = w[2 * hh];
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (2 * e + 2 <= nvalid) *reinterpret_cast<uint32_t*>(dst + 2 * e) = w[e];
}

__device__ __forceinline__ uint32_t pack_hx2(float lo, float hi) {
  hx2 v = f2hx2(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// Static "snake" schedule over work-sorted units: unit list ordered heaviest tile first
// (all (sample, head) of the heaviest causal tile, then the next), dealt to the CTAs
// boustrophedon (round r forward when r is even, backward when odd) so per-CTA work stays
// within one unit of the mean even though causal tiles differ 4x in cost.
__device__ __forceinline__ int snake_unit(int r) {
  return r * (int)gridDim.x + ((r & 1) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x);
}

// ------------------------------------------------------------------ forward, streamed keys
// K2 forward for any s (v2).  One work unit = 256 queries of one (sample, head) as two
// 128-query tiles A (queries [256u, +128)) and B ([256u + 128, +128)) that share every key /
// value block they both need.  Keys stream in blocks of KB (128 when the padded head width
// NV <= 128, 64 when NV = 192, so that S_A, S_B (KB columns each) and O_A, O_B (NV each) fit
// the 512 TMEM columns).  Online softmax in the log2 domain with a lazy rescale: a row keeps
// its running max m until a block's max exceeds m + 8 (P <= 2^8 stays exact in bf16 / fp32),
// and only then rescales l and its O row.  Ping-pong: the MMA warp issues PV_A(j), S_A(j+1),
// then PV_B(j), S_B(j+1), so softmax A works on S_A(j+1) while the tensor core runs tile B's
// MMAs and vice versa.  P overwrites its S block in TMEM (bf16 pairs, KB/2 columns) and feeds
// PV as the TMEM A operand; tcgen05 MMAs execute in issue order, so S_X(j+1) (issued after
// PV_X(j)) cannot overwrite P_X(j) before PV_X(j) has read it.
// Warps: 0 TMA producer, 1 MMA issuer, 2-3 idle, 4-7 softmax + epilogue of tile A (TMEM lane
// quarter = warp % 4), 8-11 of tile B.  Each softmax thread owns one query row and keeps the
// row's KB scores of the block in registers (one TMEM read per score).
constexpr int F2_THREADS = 12 * 32;
// Diagnostic builds only (scripts/attn_exp.sh; never the shipped library): AXONN_ATTN_EXP bit 0
// skips the softmax math (P = 0), bit 1 skips the MMA instructions (commits only), bit 2 the
// epilogue's global stores of the forward; backward: bit 3 / 4 / 5 skip the KA / !KA / D
// launch, bit 6 the P / dS math, bit 7 the MMA instructions.
#ifndef AXONN_ATTN_EXP
#define AXONN_ATTN_EXP 0
#endif
constexpr float F2_RESCALE_TH = 8.0f;   // log2 units

struct AttnFwd2Params {
  int s, heads, d, nu, total;   // nu = units per (sample, head) = ceil(s / 256)
  float c1;                     // alpha * log2(e)
  hx* o;
  long long ldo;
  float* lse;
};

template <int NV, int KB>
__global__ void __launch_bounds__(F2_THREADS, 1)
    attn_fwd2_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                     const __grid_constant__ CUtensorMap mapV, const AttnFwd2Params p) {
  constexpr int NC = NV / 64;                 // 64-wide head-dim chunks
  constexpr int Q_BYTES = 128 * NV * 2;       // one 128-query tile
  constexpr int KV_BYTES = KB * NV * 2;       // one key (or value) block
  constexpr int KST = 2, VST = 2;
  // TMEM columns: S / P of tile x at x * KB, O of tile x at 2 KB + x * NV
#define S_COL(x) ((uint32_t)(x) * KB)
#define O_COL(x) (2u * KB + (uint32_t)(x) * NV)
  static_assert(2 * KB + 2 * NV <= 512, "TMEM budget");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                               // [2] tiles
  uint8_t* sK = smem + 2 * Q_BYTES;                 // [KST]
  uint8_t* sV = sK + KST * KV_BYTES;                // [VST]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VST * KV_BYTES);
  uint64_t* q_full = bars;            // [2]
  uint64_t* q_empty = bars + 2;       // [2]
  uint64_t* k_full = bars + 4;        // [KST]
  uint64_t* k_empty = k_full + KST;   // [KST]
  uint64_t* v_full = k_empty + KST;   // [VST]
  uint64_t* v_empty = v_full + VST;   // [VST]
  uint64_t* s_full = v_empty + VST;   // [2]
  uint64_t* p_ready = s_full + 2;     // [2], 4 warps
  uint64_t* o_full = p_ready + 2;     // [2]
  uint64_t* o_free = o_full + 2;      // [2], 4 warps
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_free + 2);
  __shared__ uint4 stg_all[8][32 * 4];   // per softmax warp: 32 rows x 32 half values

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapQ);
    tma_prefetch_desc(&mapK);
    tma_prefetch_desc(&mapV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_ready[i], 4);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 4);
    }
    for (int i = 0; i < KST; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < VST; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // unit t = (z, u): the units of one (sample, head) are consecutive, heaviest (last) first, so
  // the snake deal runs them on neighbouring CTAs at the same time and the key / value blocks
  // they share are read from DRAM once (L2 hits for the second); consecutive rounds alternate
  // each CTA between heavy and light units.
  // key blocks needed by the tile whose queries end (exclusive) at qend
  auto nblk = [&](int qend) { return (min(p.s, qend) + KB - 1) / KB; };

  if (warp == 0) {
    int ks = 0, vs = 0;
    uint32_t kph = 0, vph = 0;
    int uc = 0;   // units processed (q_empty parity)
    for (int rnd = 0;; ++rnd, ++uc) {
      const int t = snake_unit(rnd);
      if (t >= p.total) break;
      const int z = t / p.nu, u = p.nu - 1 - t % p.nu;
      const int z1 = z % p.heads, z2 = z / p.heads;
      const int nB = nblk(256 * u + 256);
      for (int x = 0; x < 2; ++x) {
        mbar_wait(&q_empty[x], (uint32_t)((uc & 1) ^ 1));
        if (elect_one()) {
          mbar_arrive_expect_tx(&q_full[x], Q_BYTES);
          for (int c = 0; c < NC; ++c)
            tma_load_4d(sQ + x * Q_BYTES + c * 16384, &mapQ, &q_full[x], 64 * c, 256 * u + 128 * x, z1, z2);
        }
        __syncwarp();
      }
      for (int j = 0; j < nB; ++j) {
        mbar_wait(&k_empty[ks], kph ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&k_full[ks], KV_BYTES);
          for (int c = 0; c < NC; ++c)
            tma_load_4d(sK + ks * KV_BYTES + c * KB * 128, &mapK, &k_full[ks], 64 * c, j * KB, z1, z2);
        }
        __syncwarp();
        if (++ks == KST) { ks = 0; kph ^= 1; }
        mbar_wait(&v_empty[vs], vph ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&v_full[vs], KV_BYTES);
          for (int c = 0; c < NC; ++c)
            tma_load_4d(sV + vs * KV_BYTES + c * KB * 128, &mapV, &v_full[vs], 64 * c, j * KB, z1, z2);
        }
        __syncwarp();
        if (++vs == VST) { vs = 0; vph ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t idS = umma_idesc_f16(128, KB, 0, 0);
    const uint32_t idO = umma_idesc_f16(128, NV, 0, 1);
    const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV);
    int ks = 0, vs = 0;
    uint32_t kph = 0, vph = 0;
    uint32_t pph[2] = {0, 0};   // p_ready parity per tile
    int uc = 0;
    auto issue_S = [&](int x, int kst) {   // S_x = Q_x K^T into TMEM columns S_COL(x)
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < ((AXONN_ATTN_EXP & 2) ? 0 : NV / 16); ++kk) {
          const int c = kk / 4, k = kk % 4;
          mma_f16_ss(tmem + S_COL(x), umma_desc_sw128(q0 + x * Q_BYTES + c * 16384 + 32 * k, 16, 1024),
                      umma_desc_sw128(k0 + kst * KV_BYTES + c * KB * 128 + 32 * k, 16, 1024), idS,
                      kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[x]);
      }
      __syncwarp();
    };
    auto issue_PV = [&](int x, int vst, bool acc) {   // O_x (+)= P_x V (P from TMEM)
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < ((AXONN_ATTN_EXP & 2) ? 0 : KB / 16); ++k)
          mma_f16_ts(tmem + O_COL(x), tmem + S_COL(x) + 8 * k,
                     umma_desc_sw128(v0 + vst * KV_BYTES + 2048 * k, KB * 128, 1024), idO,
                     (acc || k > 0) ? 1u : 0u);
      }
      __syncwarp();
    };
    for (int rnd = 0;; ++rnd, ++uc) {
      const int t = snake_unit(rnd);
      if (t >= p.total) break;
      const int u = p.nu - 1 - t % p.nu;
      const int nA = nblk(256 * u + 128), nB = nblk(256 * u + 256);
      // S_A(0), S_B(0)
      mbar_wait(&k_full[ks], kph);
      tc_fence_after();
      for (int x = 0; x < 2; ++x) {
        mbar_wait(&q_full[x], (uint32_t)(uc & 1));
        tc_fence_after();
        issue_S(x, ks);
        if ((x ? nB : nA) == 1 && elect_one()) mma_commit(&q_empty[x]);   // Q_x's last use
        __syncwarp();
      }
      if (elect_one()) mma_commit(&k_empty[ks]);
      __syncwarp();
      if (++ks == KST) { ks = 0; kph ^= 1; }
      for (int j = 0; j < nB; ++j) {
        mbar_wait(&v_full[vs], vph);
        tc_fence_after();
        const bool knext = j + 1 < nB;
        bool kwaited = false;
        for (int x = 0; x < 2; ++x) {
          const int nX = x ? nB : nA;
          if (j >= nX) continue;
          mbar_wait(&p_ready[x], pph[x]);
          pph[x] ^= 1;
          if (j == 0) mbar_wait(&o_free[x], (uint32_t)((uc & 1) ^ 1));   // previous unit drained
          tc_fence_after();
          issue_PV(x, vs, j > 0);
          if (j + 1 < nX) {
            if (!kwaited) {   // block j+1's keys: waited only here, after PV_x(j) is queued
              mbar_wait(&k_full[ks], kph);
              tc_fence_after();
              kwaited = true;
            }
            issue_S(x, ks);
            if (j + 2 == nX && elect_one()) mma_commit(&q_empty[x]);   // Q_x's last use
          } else if (elect_one()) {
            mma_commit(&o_full[x]);
          }
          __syncwarp();
        }
        if (elect_one()) {
          mma_commit(&v_empty[vs]);
          if (knext) mma_commit(&k_empty[ks]);
        }
        __syncwarp();
        if (++vs == VST) { vs = 0; vph ^= 1; }
        if (knext && ++ks == KST) { ks = 0; kph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int x = (warp - 4) / 4;              // tile
    const int q = warp & 3, wi = warp - 4;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    uint4* stg = stg_all[wi];
    uint32_t sph = 0;
    int uc = 0;
    for (int rnd = 0;; ++rnd, ++uc) {
      const int t = snake_unit(rnd);
      if (t >= p.total) break;
      const int z = t / p.nu, u = p.nu - 1 - t % p.nu;
      const int z1 = z % p.heads, z2 = z / p.heads;
      const int qt0 = 256 * u + 128 * x;      // first query of the tile
      const int row = qt0 + q * 32 + lane;    // this thread's query
      const int nX = nblk(qt0 + 128);
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nX; ++j) {
        mbar_wait(&s_full[x], sph);
        sph ^= 1;
        tc_fence_after();
        uint32_t sr[KB];
#pragma unroll
        for (int c = 0; c < KB / 32; ++c)
          tmem_ld32_nowait(trow + S_COL(x) + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        tmem_ld_wait();
        const int kb0 = j * KB;
        if (kb0 + KB - 1 > qt0 || kb0 + KB > p.s) {   // diagonal or ragged block: mask
#pragma unroll
          for (int i = 0; i < KB; ++i)
            if (kb0 + i > row || kb0 + i >= p.s) sr[i] = __float_as_uint(-INFINITY);
        }
        float bmax = -INFINITY;
#pragma unroll
        for (int i = 0; i < KB; ++i) bmax = fmaxf(bmax, __uint_as_float(sr[i]));
        const float bm = bmax * p.c1;
        float mnew = m;
        bool resc = false;
        if (j == 0) {
          mnew = bm;
        } else if (bm > m + F2_RESCALE_TH) {
          mnew = bm;
          resc = true;
        }
        const float factor = resc ? ex2_approx(m - mnew) : 1.f;
        float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
        for (int c = 0; c < KB / 64; ++c) {   // 64 scores -> 32 packed P columns (already read)
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            const float e0 = (AXONN_ATTN_EXP & 1) ? 0.f : ex2_approx(fmaf(__uint_as_float(sr[64 * c + i]), p.c1, -mnew));
            const float e1 = (AXONN_ATTN_EXP & 1) ? 0.f : ex2_approx(fmaf(__uint_as_float(sr[64 * c + i + 1]), p.c1, -mnew));
            sum0 += e0;
            sum1 += e1;
            pk[i / 2] = pack_hx2(e0, e1);
          }
          tmem_st32(trow + S_COL(x) + 32 * c, pk);
        }
        l = l * factor + (sum0 + sum1);
        m = mnew;
        if (__any_sync(0xffffffffu, resc)) {   // rare: rescale this warp's O rows (PV_X(j-1) done)
#pragma unroll 1
          for (int c = 0; c < NV / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(trow + O_COL(x) + 32 * c, r);
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * factor);
            tmem_st32(trow + O_COL(x) + 32 * c, r);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_ready[x]);
      }
      if (row < p.s) p.lse[(long long)z * p.s + row] = m + __log2f(l);
      // epilogue: O / l -> half -> o[token][head * d + j]
      mbar_wait(&o_full[x], (uint32_t)(uc & 1));
      tc_fence_after();
      const float inv = 1.f / l;
      hx* obase = p.o + ((long long)z2 * p.s) * p.ldo + (long long)z1 * p.d;
      const int r0 = qt0 + q * 32;
#pragma unroll 1
      for (int oc = 0; oc < NV && oc < p.d; oc += 32) {
        uint32_t r[32];
        tmem_ld32(trow + O_COL(x) + oc, r);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint4 w;
          w.x = pack_hx2(__uint_as_float(r[8 * jj + 0]) * inv, __uint_as_float(r[8 * jj + 1]) * inv);
          w.y = pack_hx2(__uint_as_float(r[8 * jj + 2]) * inv, __uint_as_float(r[8 * jj + 3]) * inv);
          w.z = pack_hx2(__uint_as_float(r[8 * jj + 4]) * inv, __uint_as_float(r[8 * jj + 5]) * inv);
          w.w = pack_hx2(__uint_as_float(r[8 * jj + 6]) * inv, __uint_as_float(r[8 * jj + 7]) * inv);
          stg[lane * 4 + (jj ^ (lane & 3))] = w;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = i * 8 + lane / 4, ch = lane & 3;
          const int gr = r0 + rr;
          const int col = oc + ch * 8;
          if (gr < p.s && col < p.d && !(AXONN_ATTN_EXP & 4)) {
            const uint4 v = stg[rr * 4 + (ch ^ (rr & 3))];
            store8h(obase + (long long)gr * p.ldo + col, v, p.d - col);
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[x]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

#undef S_COL
#undef O_COL

template <int NV, int KB>
constexpr int fwd2_smem() {
  return 2 * 128 * NV * 2 + 4 * KB * NV * 2 + 16 * 8 + 64 + 1024;
}

template <int NV, int KB>
int launch_fwd2(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                const AttnFwd2Params& p, cudaStream_t st) {
  constexpr int SMEM = fwd2_smem<NV, KB>();
  static bool attr[kMaxDevices] = {};
  const int dev = cur_device();
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(attn_fwd2_kernel<NV, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) !=
        cudaSuccess)
      return -10;
    attr[dev] = true;
  }
  const int nsm = device_sms();
  const int grid = p.total < nsm ? p.total : nsm;
  attn_fwd2_kernel<NV, KB><<<grid, F2_THREADS, SMEM, st>>>(mq, mk, mv, p);
  return cudaGetLastError() == cudaSuccess ? 0 : -11;
}

// ------------------------------------------------------------------ backward
// dS = alpha * P * (dP - D),  D_i = sum_j P_ij dP_ij = dO_i . O_i (computed by attn_bwd_d),
// P recomputed from S and the forward's lse2 (never stored).  Two kernels of one template:
//   KA (rows = 128 keys n): for every 64-query block m with queries >= keys:
//       X = K_n Q_m^T, Y = V_n dO_m^T -> P^T, dS^T packed bf16 in TMEM
//       -> dV_n += P^T dO_m,  dK_n += dS^T Q_m                                   (TS-MMAs)
//   !KA (rows = 128 queries m): for every 64-key block n <= m:
//       X = Q_m K_n^T, Y = dO_m V_n^T -> dS packed in TMEM -> dQ_m += dS K_n
// so every gradient element has exactly one writer (deterministic, no atomics).  The row
// operands (F1, F2) stay in smem for the unit; the 64-row column operands (G1, G2) stream
// through a ring, and one smem copy of each serves both the K-major (X, Y) and the MN-major
// (accumulation) descriptor.  X / Y are double-buffered in TMEM when the accumulators leave
// room, so the epilogue of block i overlaps the MMAs of block i+1.  8 epilogue warps:
// warp (q, half) owns TMEM lanes [32 q, +32) and block columns [32 half, +32).
#ifndef AXONN_ATTN_NBUF1_WAIT
#define AXONN_ATTN_NBUF1_WAIT 0   // diagnostic builds: the round-2 c19 behaviour (always wait)
#endif
struct AttnBwdParams {
  int s, heads, d, nv, nq, nk, total, stages, nbuf;
  int st_sh;           // log2(stages): stages is 2 or 4, so ring indices are masks and shifts
  int nfb, nab;        // row-operand smem buffers, accumulator TMEM buffers (1 or 2 each)
  int ld_bulk;         // KA: the producer bulk-copies each query block's lse / D slice into the
                       // ring stage (s % 64 == 0); else the epilogue loads them per block
  float c1, alpha;
  const float* lse;
  const float* D;
  hx* dq;   // dqkv base; dQ at column z1*d, dK at h + z1*d, dV at 2h + z1*d
  long long ldq;
  int h;
  unsigned long long* trace;   // diagnostic builds (AXONN_ATTN_EXP bit 8): CTA 0 event clocks
};
// diagnostic timeline (AXONN_ATTN_EXP & 256 only): event e of block / unit i of CTA 0
#define BWD_TRACE(e, i)                                                                       \
  do {                                                                                        \
    if ((AXONN_ATTN_EXP & 256) && blockIdx.x == 0 && (i) < 512)                                \
      p.trace[(e) * 512 + (i)] = clock64();                                                   \
  } while (0)

constexpr int BWD_THREADS = 64 + 8 * 32;
constexpr int GRB = 64;   // rows of one streamed block (queries for KA, keys for !KA)

__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                          int nv, int rows, int row0, int z1, int z2) {
  // [rows x nv] operand: d-chunk c (64 columns) at c * rows * 128, 64-row boxes
  for (int c = 0; c < nv / 64; ++c)
    for (int rb = 0; rb < rows / 64; ++rb)
      tma_load_4d(dst + c * rows * 128 + rb * 8192, map, bar, 64 * c, row0 + 64 * rb, z1, z2);
}

// 32 rows x 32 bf16 (this warp's chunk, row = lane) -> global rows r0.., columns col0..
// (only col < dvalid), through a swizzled 2 KB staging tile: 8 rows x 64 B per instruction
__device__ __forceinline__ void store_chunk32(uint4* stg, int lane, const uint32_t (&r)[32],
                                              float scale, hx* gbase, long long ld,
                                              int r0, int rows_valid, int col0, int dvalid) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 u;
    u.x = pack_hx2(__uint_as_float(r[8 * j + 0]) * scale, __uint_as_float(r[8 * j + 1]) * scale);
    u.y = pack_hx2(__uint_as_float(r[8 * j + 2]) * scale, __uint_as_float(r[8 * j + 3]) * scale);
    u.z = pack_hx2(__uint_as_float(r[8 * j + 4]) * scale, __uint_as_float(r[8 * j + 5]) * scale);
    u.w = pack_hx2(__uint_as_float(r[8 * j + 6]) * scale, __uint_as_float(r[8 * j + 7]) * scale);
    stg[lane * 4 + (j ^ (lane & 3))] = u;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = i * 8 + lane / 4, ch = lane & 3;
    const int gr = r0 + rr;
    const int col = col0 + ch * 8;
    if (gr < rows_valid && col < dvalid) {
      const uint4 v = stg[rr * 4 + (ch ^ (rr & 3))];
      store8h(gbase + (long long)gr * ld + col, v, dvalid - col);
    }
  }
  __syncwarp();
}

// x mod n and x / n for n in {1, 2} (row-operand / TMEM buffer counts) without an integer
// division in the per-block loops
__device__ __forceinline__ int m12(int x, int n) { return n == 2 ? (x & 1) : 0; }
__device__ __forceinline__ int d12(int x, int n) { return n == 2 ? (x >> 1) : x; }

template <bool KA>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                    const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapO,
                    const AttnBwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int FR = 128, GR = GRB;
  const int f_bytes = p.nv * FR * 2;         // one row operand
  const int g_bytes = p.nv * GR * 2;         // one streamed operand
  uint8_t* sF = smem;                        // [nfb] x (F1, F2)
  uint8_t* sG = smem + p.nfb * 2 * f_bytes;  // ring: stage i holds G1, G2
  float* sLD = reinterpret_cast<float*>(sG + p.stages * 2 * g_bytes);   // [stages][lse 64 | D 64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sG + p.stages * 2 * g_bytes + (KA ? p.stages * 512 : 0));
  uint64_t* f_full = bars;                   // [2]
  uint64_t* f_empty = bars + 2;              // [2]
  uint64_t* acc_full = bars + 4;             // [2]
  uint64_t* acc_free = bars + 6;             // [2], 8 arrivals
  uint64_t* xy_full = bars + 8;              // [2]
  uint64_t* pd_ready = bars + 10;            // [2], 8 arrivals
  uint64_t* acc_done = bars + 12;            // [2]
  uint64_t* g_full = bars + 14;              // [4]
  uint64_t* g_empty = bars + 18;             // [4]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 22);
  __shared__ __align__(16) float sL[2][GR], sD[2][GR];
  __shared__ uint4 stg_all[8][32 * 4];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // TMEM: buffer b: X [128 b, +64), Y [128 b + 64, +64); accumulators after the buffers
  // accumulator buffer ab: colA(ab) = 128 nbuf + ab * (KA ? 2 nv : nv), colB = colA + (KA ? nv : 0)
  const uint32_t acc_w = KA ? 2 * p.nv : p.nv;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapQ);
    tma_prefetch_desc(&mapK);
    tma_prefetch_desc(&mapV);
    tma_prefetch_desc(&mapO);
    for (int i = 0; i < 22; ++i) mbar_init(&bars[i], (i == 6 || i == 7 || i == 10 || i == 11) ? 8 : 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // unit t -> (z, tile): KA: key tile n ascending (most query blocks first); else query tile
  // m descending (most key blocks first)
  auto unit = [&](int t, int& z, int& r0, int& i0, int& ni) {
    // the tiles of one (sample, head) are consecutive, heaviest first: the snake deal runs them
    // on neighbouring CTAs at the same time, so the streamed blocks they share are read from
    // DRAM once (L2 hits), and consecutive rounds alternate each CTA between heavy and light
    // tiles (with per = 4 and 148 CTAs, CTA c gets tile c % 4, then 3 - c % 4, ...)
    const int per = KA ? p.nk : p.nq;
    z = t / per;
    const int k = t % per;
    if (KA) {
      r0 = k * 128;                     // keys [r0, r0 + 128)
      i0 = r0 / GR;                     // first query block touching the diagonal
      ni = (p.s + GR - 1) / GR - i0;
    } else {
      const int m = per - 1 - k;
      r0 = m * 128;                     // queries [r0, r0 + 128)
      i0 = 0;
      ni = min((p.s + GR - 1) / GR, (r0 + 128) / GR);   // key blocks with keys <= last query
    }
  };

  if (warp == 0) {
    int gp_count = 0;
    int stage = 0;
    uint32_t phase = 0;
    int u = 0;
    for (int rnd = 0;; ++rnd, ++u) {
      const int t = snake_unit(rnd);
      if (t >= p.total) break;
      int z, r0, i0, ni;
      unit(t, z, r0, i0, ni);
      const int z1 = z % p.heads, z2 = z / p.heads;
      const int fb = m12(u, p.nfb);
      mbar_wait(&f_empty[fb], (uint32_t)(((d12(u, p.nfb)) & 1) ^ 1));
      if (elect_one()) {
        uint8_t* f = sF + fb * 2 * f_bytes;
        mbar_arrive_expect_tx(&f_full[fb], 2 * f_bytes);
        load_rows(f, KA ? &mapK : &mapQ, &f_full[fb], p.nv, FR, r0, z1, z2);
        load_rows(f + f_bytes, KA ? &mapV : &mapO, &f_full[fb], p.nv, FR, r0, z1, z2);
      }
      __syncwarp();
      for (int it = 0; it < ni; ++it) {
        const int g0 = (i0 + it) * GR;
        mbar_wait(&g_empty[stage], phase ^ 1);
        if (lane == 0) BWD_TRACE(0, gp_count);
        ++gp_count;
        if (elect_one()) {
          uint8_t* g = sG + stage * 2 * g_bytes;
          const bool bulk = KA && p.ld_bulk;
          mbar_arrive_expect_tx(&g_full[stage], 2 * g_bytes + (bulk ? 512 : 0));
          load_rows(g, KA ? &mapQ : &mapK, &g_full[stage], p.nv, GR, g0, z1, z2);
          load_rows(g + g_bytes, KA ? &mapO : &mapV, &g_full[stage], p.nv, GR, g0, z1, z2);
          if (bulk) {   // this block's 64 queries: lse2 and D (consumed by the epilogue)
            bulk_g2s(sLD + stage * 128, p.lse + (long long)z * p.s + g0, 256, &g_full[stage]);
            bulk_g2s(sLD + stage * 128 + 64, p.D + (long long)z * p.s + g0, 256, &g_full[stage]);
          }
        }
        __syncwarp();
        if (++stage == p.stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t idXY = umma_idesc_f16(128, GR, 0, 0);
    const uint32_t idAcc = umma_idesc_f16(128, p.nv, 0, 1);
    const uint32_t sG0 = smem_u32(sG);
    int g = 0;                        // global block counter (stage / buffer / parity source)
    uint32_t accd_ph[2] = {0, 0};     // acc_done uses per buffer
    int accd_n[2] = {0, 0};
    int u = 0;
    uint32_t sF0 = 0;                 // current unit's row operands
    auto issue_xy = [&](int gi) {     // X, Y of global block gi into buffer gi % nbuf
      const int b = m12(gi, p.nbuf), stg = (gi & (p.stages - 1));
      mbar_wait(&g_full[stg], (uint32_t)(((gi >> p.st_sh)) & 1));
      if (lane == 0) BWD_TRACE(1, gi);
      // wait until the accumulation of block gi - nbuf (which reads P / dS from buffer b) is
      // complete.  In-order MMA issue alone would order the TMEM reuse, but measured: letting
      // X / Y of the next block run under the epilogue's TMEM traffic slows the epilogue
      // (the bottleneck) 2x -- 1.3B KA per block 2.5k -> 2.7k cycles, 12B worse
      // (profiles/r2/attn_bwd_trace_c10_c11.md).  With one X / Y buffer (KA at nv 192) X / Y of
      // block gi is issued after the accumulation of gi - 1, which waited for that block's
      // epilogue: nothing can overlap the epilogue, and the tensor pipe's in-order execution
      // already orders the reuse, so the wait would only add its round trip to the chain.  The dQ
      // kernel (!KA: its epilogue writes only dS) measured 2196 -> 1941 cycles per block without
      // the wait and an epilogue 6 % slower (c11 trace), so it skips the wait too
      if (((KA && p.nbuf == 2) || AXONN_ATTN_NBUF1_WAIT) && accd_n[b] > 0) mbar_wait(&acc_done[b], accd_ph[b] ^ 1);
      tc_fence_after();
      if (lane == 0) BWD_TRACE(2, gi);
      const uint32_t g1 = sG0 + stg * 2 * g_bytes, g2 = g1 + g_bytes;
      if (elect_one()) {
        for (int c = 0; c < ((AXONN_ATTN_EXP & 128) ? 0 : p.nv / 64); ++c) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acc = (c > 0 || k > 0) ? 1u : 0u;
            mma_f16_ss(tmem + 128 * b, umma_desc_sw128(sF0 + c * FR * 128 + 32 * k, 16, 1024),
                        umma_desc_sw128(g1 + c * GR * 128 + 32 * k, 16, 1024), idXY, acc);
            mma_f16_ss(tmem + 128 * b + 64,
                        umma_desc_sw128(sF0 + f_bytes + c * FR * 128 + 32 * k, 16, 1024),
                        umma_desc_sw128(g2 + c * GR * 128 + 32 * k, 16, 1024), idXY, acc);
          }
        }
        mma_commit(&xy_full[b]);
      }
      __syncwarp();
    };
    for (int rnd = 0;; ++rnd, ++u) {
      const int t = snake_unit(rnd);
      if (t >= p.total) break;
      int z, r0, i0, ni;
      unit(t, z, r0, i0, ni);
      const int fb = m12(u, p.nfb), ab = m12(u, p.nab);
      const uint32_t colA = 128 * p.nbuf + ab * acc_w, colB = colA + (KA ? p.nv : 0);
      mbar_wait(&f_full[fb], (uint32_t)((d12(u, p.nfb)) & 1));
      tc_fence_after();
      sF0 = smem_u32(sF + fb * 2 * f_bytes);
      const int g_first = g;
      issue_xy(g);
      if (ni == 1 && elect_one()) mma_commit(&f_empty[fb]);
      __syncwarp();
      for (int it = 0; it < ni; ++it, ++g) {
        const int b = m12(g, p.nbuf), stg = (g & (p.stages - 1));
        if (p.nbuf == 2 && it + 1 < ni) {
          issue_xy(g + 1);
          if (it + 2 == ni && elect_one()) mma_commit(&f_empty[fb]);
          __syncwarp();
        }
        mbar_wait(&pd_ready[b], (uint32_t)(d12(g, p.nbuf) & 1));
        if (lane == 0) BWD_TRACE(3, g);
        if (it == 0) mbar_wait(&acc_free[ab], (uint32_t)(((d12(u, p.nab)) & 1) ^ 1));
        if (it == 0 && lane == 0) BWD_TRACE(9, u);
        tc_fence_after();
        const uint32_t g1 = sG0 + stg * 2 * g_bytes, g2 = g1 + g_bytes;
        if (elect_one()) {
          // accumulate over the 64 rows of this block: A = packed P^T / dS (TMEM; columns of
          // the two 32-wide halves at +0 and +32), B = G operand MN-major
#pragma unroll
          for (int k = 0; k < ((AXONN_ATTN_EXP & 128) ? 0 : GR / 16); ++k) {
            const uint32_t acc = (it > 0 || k > 0) ? 1u : 0u;
            const uint32_t pc = 128 * b + (k >> 1) * 32 + (k & 1) * 8;
            if (KA)
              mma_f16_ts(tmem + colA, tmem + pc, umma_desc_sw128(g2 + 2048 * k, GR * 128, 1024),
                          idAcc, acc);
            mma_f16_ts(tmem + colB, tmem + pc + 64, umma_desc_sw128(g1 + 2048 * k, GR * 128, 1024),
                        idAcc, acc);
          }
          mma_commit(&g_empty[stg]);
          mma_commit(&acc_done[b]);
          BWD_TRACE(4, g);
          if (it == ni - 1) mma_commit(&acc_full[ab]);
        }
        __syncwarp();
        accd_ph[b] ^= 1;
        ++accd_n[b];
        if (p.nbuf == 1 && it + 1 < ni) {
          issue_xy(g + 1);
          if (it + 2 == ni && elect_one()) mma_commit(&f_empty[fb]);
          __syncwarp();
        }
      }
      (void)g_first;
    }
  } else {
    const int q = warp & 3, half = (warp - 2) >> 2, wi = warp - 2;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    uint4* stg = stg_all[wi];
    int u = 0, g = 0;
    for (int rnd = 0;; ++rnd, ++u) {
      const int t = snake_unit(rnd);
      if (t >= p.total) break;
      int z, r0, i0, ni;
      unit(t, z, r0, i0, ni);
      const int z1 = z % p.heads, z2 = z / p.heads;
      const int row = r0 + q * 32 + lane;     // key (KA) or query (!KA) index
      const float* lse = p.lse + (long long)z * p.s;
      const float* Dz = p.D + (long long)z * p.s;
      float Lr = 0.f, Dr = 0.f;
      if (!KA && row < p.s) {
        Lr = lse[row];
        Dr = Dz[row];
      }
      for (int it = 0; it < ni; ++it, ++g) {
        const int b = m12(g, p.nbuf);
        const int g0 = (i0 + it) * GR;        // first query (KA) or key (!KA) of the block
        const int sb = g & 1;
        const float* Lblk = sL[sb];
        const float* Dblk = sD[sb];
        if (KA && p.ld_bulk) {   // the ring stage holds this block's slices (TMA-visible after g_full)
          const int stg = (g & (p.stages - 1));
          mbar_wait(&g_full[stg], (uint32_t)(((g >> p.st_sh)) & 1));
          Lblk = sLD + stg * 128;
          Dblk = Lblk + 64;
        } else if (KA) {
          const int tid = threadIdx.x - 64;
          if (tid < GR) {
            const int i = g0 + tid;
            sL[sb][tid] = i < p.s ? lse[i] : 0.f;
            sD[sb][tid] = i < p.s ? Dz[i] : 0.f;
          }
          nbar(1, 256);
        }
        mbar_wait(&xy_full[b], (uint32_t)(d12(g, p.nbuf) & 1));
        if (warp == 2 && lane == 0) BWD_TRACE(5, g);
        tc_fence_after();
        const int c0 = 32 * half;             // this warp's 32 block columns
        uint32_t x[32], y[32];
        tmem_ld32_nowait(trow + 128 * b + c0, x);
        tmem_ld32_nowait(trow + 128 * b + 64 + c0, y);
        tmem_ld_wait();
        uint32_t pp[16], pd[16];
        // this warp's 32 columns: per-column (KA: query) or per-row (!KA) lse2 and D, masks only
        // in blocks that cross the diagonal or s (warp-uniform test)
        float nL[32], Da[32];
        if (KA) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 l4 = *reinterpret_cast<const float4*>(Lblk + c0 + i);
            const float4 d4 = *reinterpret_cast<const float4*>(Dblk + c0 + i);
            nL[i] = -l4.x; nL[i + 1] = -l4.y; nL[i + 2] = -l4.z; nL[i + 3] = -l4.w;
            Da[i] = d4.x; Da[i + 1] = d4.y; Da[i + 2] = d4.z; Da[i + 3] = d4.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) { nL[i] = -Lr; Da[i] = Dr; }
        }
        const int cb = g0 + c0;               // first column (query for KA, key for !KA)
        const int rlo = r0 + q * 32;          // this warp's first row
        const bool full = KA ? (cb >= rlo + 31 && cb + 31 < p.s) : (cb + 31 <= rlo);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float P2[2], S2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = cb + i + e;
            const bool ok = full || (KA ? (col >= row && col < p.s) : (col <= row));
            const float P = (ok && !(AXONN_ATTN_EXP & 64)) ? ex2_approx(fmaf(__uint_as_float(x[i + e]), p.c1, nL[i + e])) : 0.f;
            P2[e] = P;
            S2[e] = P * ((__uint_as_float(y[i + e]) - Da[i + e]) * p.alpha);
          }
          pp[i / 2] = pack_hx2(P2[0], P2[1]);
          pd[i / 2] = pack_hx2(S2[0], S2[1]);
        }
        if (KA) tmem_st16(trow + 128 * b + c0, pp);
        tmem_st16(trow + 128 * b + 64 + c0, pd);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (warp == 2 && lane == 0) BWD_TRACE(6, g);
        if (lane == 0) mbar_arrive(&pd_ready[b]);
      }
      // drain the accumulators of the unit: KA -> dV (acc_a), dK (acc_b); else dQ (acc_b)
      const int ab = m12(u, p.nab);
      const uint32_t colA = 128 * p.nbuf + ab * acc_w, colB = colA + (KA ? p.nv : 0);
      mbar_wait(&acc_full[ab], (uint32_t)((d12(u, p.nab)) & 1));
      if (warp == 2 && lane == 0) BWD_TRACE(7, u);
      tc_fence_after();
      hx* base = p.dq + (long long)z2 * p.s * p.ldq + (long long)z1 * p.d;
      const int r0w = r0 + q * 32;
      for (int which = KA ? 0 : 1; which < 2; ++which) {
        const uint32_t ca = which == 0 ? colA : colB;
        hx* gb = base + (KA ? (which == 0 ? 2 * p.h : p.h) : 0);
        for (int cc = 0; cc < p.nv / 2; cc += 32) {
          const int oc = half * (p.nv / 2) + cc;
          uint32_t r[32];
          tmem_ld32(trow + ca + oc, r);
          store_chunk32(stg, lane, r, 1.f, gb, p.ldq, r0w, p.s, oc, p.d);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (warp == 2 && lane == 0) BWD_TRACE(8, u);
      if (lane == 0) mbar_arrive(&acc_free[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// D[z * s + i] = sum_j dO[i, head, j] * O[i, head * d + j]   (fp32); 16 lanes per (token, head),
// DITEMS (token, head) items per 16-lane group with every load issued before the math
constexpr int DITEMS = 4;
// Group g of 16 lanes handles DITEMS = 4 items; lane l holds 8 (or 4) head-dim columns of each
// item's row and a 16-lane reduction finishes each dot product.
//   TOK (heads % 4 == 0): the items are 4 consecutive heads of one token, g = token * heads / 4
//     + head / 4 -- a group reads 4 * d contiguous elements of dO and of O, a warp two groups
//     of the same or the next token: DRAM sees whole rows (the head-major order read 2 d-wide
//     slices of rows 4 KB apart and ran at 2.3 TB/s);
//   else: 4 consecutive query rows of one head (z = sample * heads + head), one 16-byte store.
template <bool TOK>
__global__ void attn_bwd_d_kernel(const hx* __restrict__ dO, long long ld_do, int dp,
                                  const hx* __restrict__ O, long long ld_o, int d,
                                  int s, int heads, long long ntok, float* __restrict__ D) {
  const long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 16;
  const int l = threadIdx.x & 15;
  const long long ngrp = ntok * heads / DITEMS;
  const bool live = grp < ngrp;
  long long tok_u[DITEMS], out_u[DITEMS];
  int hd_u[DITEMS];
  if (TOK) {
    const long long tok = live ? grp / (heads / DITEMS) : 0;
    const int h0 = live ? (int)(grp % (heads / DITEMS)) * DITEMS : 0;
    const long long sample = tok / s;
    const int i = (int)(tok % s);
#pragma unroll
    for (int u = 0; u < DITEMS; ++u) {
      tok_u[u] = tok;
      hd_u[u] = h0 + u;
      out_u[u] = (sample * heads + h0 + u) * s + i;
    }
  } else {
    const long long z = live ? grp / (s / DITEMS) : 0;
    const int i0 = live ? (int)(grp % (s / DITEMS)) * DITEMS : 0;
    const long long sample = z / heads;
#pragma unroll
    for (int u = 0; u < DITEMS; ++u) {
      tok_u[u] = sample * s + i0 + u;
      hd_u[u] = (int)(z % heads);
      out_u[u] = z * s + i0 + u;
    }
  }
  float acc[DITEMS];
  if ((d & 7) == 0 && (dp & 7) == 0 && d <= 128) {
    uint4 x[DITEMS], y[DITEMS];
#pragma unroll
    for (int u = 0; u < DITEMS; ++u) {
      const int j = 8 * l;
      x[u] = y[u] = make_uint4(0, 0, 0, 0);
      if (live && j < d) {
        x[u] = __ldg(reinterpret_cast<const uint4*>(dO + tok_u[u] * ld_do + (long long)hd_u[u] * dp + j));
        y[u] = __ldg(reinterpret_cast<const uint4*>(O + tok_u[u] * ld_o + (long long)hd_u[u] * d + j));
      }
    }
#pragma unroll
    for (int u = 0; u < DITEMS; ++u) {
      const hx2* xh = reinterpret_cast<const hx2*>(&x[u]);
      const hx2* yh = reinterpret_cast<const hx2*>(&y[u]);
      float a = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xf = hx22f2(xh[e]), yf = hx22f2(yh[e]);
        a = fmaf(xf.x, yf.x, fmaf(xf.y, yf.y, a));
      }
      acc[u] = a;
    }
  } else if ((d & 3) == 0 && (dp & 3) == 0 && (ld_o & 3) == 0 && (ld_do & 3) == 0 && d <= 256) {
    // head width a multiple of 4 but not 8 (d = 188, 176): 8-byte loads, every load of the
    // DITEMS rows issued before the math (16 lanes x 4 elements = 64 per pass, <= 4 passes)
    uint2 x[DITEMS][4], y[DITEMS][4];
#pragma unroll
    for (int u = 0; u < DITEMS; ++u) {
#pragma unroll
      for (int ps = 0; ps < 4; ++ps) {
        const int j = 4 * l + 64 * ps;
        x[u][ps] = y[u][ps] = make_uint2(0, 0);
        if (live && j < d) {
          x[u][ps] = __ldg(reinterpret_cast<const uint2*>(dO + tok_u[u] * ld_do + (long long)hd_u[u] * dp + j));
          y[u][ps] = __ldg(reinterpret_cast<const uint2*>(O + tok_u[u] * ld_o + (long long)hd_u[u] * d + j));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < DITEMS; ++u) {
      float a = 0.f;
#pragma unroll
      for (int ps = 0; ps < 4; ++ps) {
        const hx2* xh = reinterpret_cast<const hx2*>(&x[u][ps]);
        const hx2* yh = reinterpret_cast<const hx2*>(&y[u][ps]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float2 xf = hx22f2(xh[e]), yf = hx22f2(yh[e]);
          a = fmaf(xf.x, yf.x, fmaf(xf.y, yf.y, a));
        }
      }
      acc[u] = a;
    }
  } else {
#pragma unroll
    for (int u = 0; u < DITEMS; ++u) {
      float a = 0.f;
      if (live) {
        const hx* xa = dO + tok_u[u] * ld_do + (long long)hd_u[u] * dp;
        const hx* ya = O + tok_u[u] * ld_o + (long long)hd_u[u] * d;
        for (int j = 2 * l; j < d; j += 32) {
          const float2 xf = hx22f2(*reinterpret_cast<const hx2*>(xa + j));
          const float2 yf = hx22f2(*reinterpret_cast<const hx2*>(ya + j));
          a = fmaf(xf.x, yf.x, fmaf(xf.y, yf.y, a));
        }
      }
      acc[u] = a;
    }
  }
#pragma unroll
  for (int u = 0; u < DITEMS; ++u) {
    float a = acc[u];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    acc[u] = a;
  }
  if (l == 0 && live) {
    if (TOK) {
#pragma unroll
      for (int u = 0; u < DITEMS; ++u) D[out_u[u]] = acc[u];
    } else {
      *reinterpret_cast<float4*>(D + out_u[0]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
  }
}

}  // namespace

int attn_fwd(const void* qkv, long long lq, int b, int heads, int s, int d, int dp, float alpha,
             void* o, long long ldo, float* lse, cudaStream_t st) {
  if (s <= 0 || d <= 0 || dp < d || dp % 2 || (d & 1)) return -1;
  const int nv = (dp + 63) / 64 * 64;
  if (nv > 192) return -1;
  const char* base = static_cast<const char*>(qkv);
  const int kb = nv <= 128 ? 128 : 64;
  CUtensorMap mq, mk, mv;
  const long long s2 = (long long)s * lq;
  int rc = make_tmap_4d(&mq, base, dp, s, lq, heads, dp, b, s2, 128);
  if (!rc) rc = make_tmap_4d(&mk, base + (size_t)heads * dp * 2, dp, s, lq, heads, dp, b, s2, kb);
  if (!rc) rc = make_tmap_4d(&mv, base + (size_t)2 * heads * dp * 2, dp, s, lq, heads, dp, b, s2, kb);
  if (rc) return rc;
  AttnFwd2Params p;
  p.s = s;
  p.heads = heads;
  p.d = d;
  p.nu = (s + 255) / 256;
  p.total = p.nu * b * heads;
  p.c1 = alpha * 1.4426950408889634f;
  p.o = static_cast<hx*>(o);
  p.ldo = ldo;
  p.lse = lse;
  if (nv == 64) return launch_fwd2<64, 128>(mq, mk, mv, p, st);
  if (nv == 128) return launch_fwd2<128, 128>(mq, mk, mv, p, st);
  return launch_fwd2<192, 64>(mq, mk, mv, p, st);
}

int attn_bwd(const void* qkv, long long lq, const void* dO, const void* o, long long ldo,
             const float* lse, float* Dbuf, int b, int heads, int s, int d, int dp, float alpha,
             void* dqkv, long long ldq, cudaStream_t st) {
  if (s <= 0 || s > 512 || s % 4 || d <= 0 || dp < d || dp % 2 || (d & 1) || (ldq & 1)) return -1;
  const int nv = (dp + 63) / 64 * 64;
  if (nv > 256) return -1;
  const long long ntok = (long long)b * s;
  if (!(AXONN_ATTN_EXP & 32)) {
    const long long nthreads = (ntok * heads + DITEMS - 1) / DITEMS * 16;
    auto kd = heads % DITEMS == 0 ? attn_bwd_d_kernel<true> : attn_bwd_d_kernel<false>;
    kd<<<(unsigned)((nthreads + 255) / 256), 256, 0, st>>>(
        static_cast<const hx*>(dO), (long long)heads * dp, dp,
        static_cast<const hx*>(o), ldo, d, s, heads, ntok, Dbuf);
  }
  const char* base = static_cast<const char*>(qkv);
  CUtensorMap mq, mk, mv, mo;
  const long long s2 = (long long)s * lq;
  int rc = make_tmap_4d(&mq, base, dp, s, lq, heads, dp, b, s2, 64);
  if (!rc) rc = make_tmap_4d(&mk, base + (size_t)heads * dp * 2, dp, s, lq, heads, dp, b, s2, 64);
  if (!rc) rc = make_tmap_4d(&mv, base + (size_t)2 * heads * dp * 2, dp, s, lq, heads, dp, b, s2, 64);
  if (!rc) rc = make_tmap_4d(&mo, dO, dp, s, (long long)heads * dp, heads, dp, b,
                             (long long)s * heads * dp, 64);
  if (rc) return rc;
  int nsm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  AttnBwdParams p;
  p.s = s; p.heads = heads; p.d = d; p.nv = nv;
  p.nq = (s + 127) / 128;
  p.nk = (s + 127) / 128;
  p.c1 = alpha * 1.4426950408889634f;
  p.alpha = alpha;
  p.lse = lse;
  p.D = Dbuf;
  p.dq = static_cast<hx*>(dqkv);
  p.ldq = ldq;
  p.h = heads * d;
  p.trace = nullptr;
#if AXONN_ATTN_EXP & 256
  static unsigned long long* trace_buf = nullptr;
  if (!trace_buf && cudaMalloc(&trace_buf, 2 * 10 * 512 * sizeof(unsigned long long)) != cudaSuccess) return -10;
#endif
  const int max_smem = 227 * 1024 - 1024 - 256 - 18 * 1024;   // dynamic budget beside static
  p.ld_bulk = s % GRB == 0;
  for (int ka = 1; ka >= 0; --ka) {
    if ((ka && (AXONN_ATTN_EXP & 8)) || (!ka && (AXONN_ATTN_EXP & 16))) continue;
    const int f_bytes = nv * 128 * 2, g_bytes = nv * GRB * 2 + (ka ? 256 : 0);   // + lse/D slices
    // one row-operand buffer (a second one measured no faster and costs ring depth)
    p.nfb = 1;
    int stages = 4;
    if (p.nfb * 2 * f_bytes + stages * 2 * g_bytes > max_smem) stages = 2;   // ring depth 4 or 2
    if (p.nfb * 2 * f_bytes + stages * 2 * g_bytes > max_smem) return -1;
    p.stages = stages;
    p.st_sh = stages == 4 ? 2 : 1;
    // X / Y double buffer (256 TMEM columns) when the accumulators fit beside it; then
    // double-buffered accumulators (the drain of unit u overlaps unit u+1)
    const int accw = ka ? 2 * nv : nv;
    p.nbuf = (256 + accw <= 512) ? 2 : 1;
    if (128 * p.nbuf + accw > 512) return -1;
    p.nab = (128 * p.nbuf + 2 * accw <= 512) ? 2 : 1;
    p.total = b * heads * (ka ? p.nk : p.nq);
    const int smem = p.nfb * 2 * f_bytes + stages * 2 * g_bytes + 1024 + 256;   // g_bytes counts the slices
    void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, AttnBwdParams) =
        ka ? attn_bwd_kernel<true> : attn_bwd_kernel<false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return -10;
    const int grid = p.total < nsm ? p.total : nsm;
#if AXONN_ATTN_EXP & 256
    p.trace = trace_buf + (ka ? 0 : 10 * 512);
    cudaMemsetAsync(p.trace, 0, 10 * 512 * sizeof(unsigned long long), st);
#endif
    kern<<<grid, BWD_THREADS, smem, st>>>(mq, mk, mv, mo, p);
    if (cudaGetLastError() != cudaSuccess) return -11;
#if AXONN_ATTN_EXP & 256
    if (const char* tf = getenv("AXONN_TRACE_FILE")) {   // diagnostic builds only
      std::vector<unsigned long long> h(10 * 512);
      cudaStreamSynchronize(st);
      cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost);
      if (FILE* f = fopen((std::string(tf) + (ka ? ".ka.csv" : ".q.csv")).c_str(), "w")) {
        fprintf(f, "i,prod_gempty,mma_gfull,mma_xy_issue,mma_pd,mma_acc_issue,epi_xyfull,epi_pd,drain_start,drain_end,mma_accfree\n");
        for (int i = 0; i < 512; ++i) {
          fprintf(f, "%d", i);
          for (int e = 0; e < 10; ++e) fprintf(f, ",%llu", h[e * 512 + i]);
          fprintf(f, "\n");
        }
        fclose(f);
      }
    }
#endif
  }
  return 0;
}

int preload_attn() {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, attn_fwd2_kernel<64, 128>) != cudaSuccess) return -1;
  if (cudaFuncGetAttributes(&a, attn_fwd2_kernel<128, 128>) != cudaSuccess) return -1;
  if (cudaFuncGetAttributes(&a, attn_fwd2_kernel<192, 64>) != cudaSuccess) return -1;
  if (cudaFuncGetAttributes(&a, attn_bwd_kernel<true>) != cudaSuccess) return -1;
  if (cudaFuncGetAttributes(&a, attn_bwd_kernel<false>) != cudaSuccess) return -1;
  if (cudaFuncGetAttributes(&a, attn_bwd_d_kernel<true>) != cudaSuccess) return -1;
  return cudaFuncGetAttributes(&a, attn_bwd_d_kernel<false>) == cudaSuccess ? 0 : -1;
}

}  // namespace axonn
