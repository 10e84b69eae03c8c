// Internal launcher declarations for the sm_100a kernels (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "half.cuh"

namespace axonn {

// Per-device one-time state (kernel attributes and SM counts are per device; one process may
// drive several devices, e.g. axonn_calibrate_speed or the loopback transport).
constexpr int kMaxDevices = 64;
constexpr int kMaxReplicas = 8;   // G_data limit of the fused column reduction (adamw_sum_launch)
inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}
inline int device_sms() {
  static int cache[kMaxDevices] = {};
  const int d = cur_device();
  if (!cache[d]) cudaDeviceGetAttribute(&cache[d], cudaDevAttrMultiProcessorCount, d);
  return cache[d];
}

enum Epi {
  EPI_HALF = 0, EPI_BIAS_GELU = 1, EPI_DGELU = 2, EPI_F32 = 3
};

struct GemmArgs {
  int M, N, K;          // per-batch GEMM: C[M,N] = A[M,K] * B[N,K]^T
  int Z, Z1;            // batch count; z1 = z % Z1, z2 = z / Z1 index the 4-D TMA maps
  const void* A;        // bf16; K-major: [M][lda] ; MN-major (a_mn=1): [K][lda]
  long long lda, a_s1, a_s2;
  int a_mn;
  const void* B;        // bf16; K-major: [N][ldb] ; MN-major (b_mn=1): [K][ldb]
  long long ldb, b_s1, b_s2;
  int b_mn;
  void* C;              // bf16 or fp32 (EPI_F32)
  long long ldc, c_s1, c_s2;
  int epi, causal, accumulate;
  int col_group_in, col_group_out, n_valid;
  const void* bias;     // bf16 [N]
  const void* resid;    // bf16 [M][ld_resid]
  long long ld_resid;
  void* aux;            // bf16 [M][ld_aux]: GeLU pre-activation (stored by BIAS_GELU, read by DGELU)
  long long ld_aux;
  float alpha;
  int max_ctas;
  int variant;          // 0 auto, 1 single CTA, 2 CTA pair (TMA epilogue when eligible), 3 CTA pair, thread-store epilogue
};

int gemm_launch(const GemmArgs& g, cudaStream_t st);
// 4-D bf16 TMA map (inner, outer, z1, z2), strides in elements, box (64, box_outer), SWIZZLE_128B
int make_tmap_4d(CUtensorMap* map, const void* base, long long inner, long long outer,
                 long long ld, int Z1, long long s1, int Z2, long long s2, int box_outer);

// attn.cu: fused causal attention over the packed [tokens, 3, heads, dp] QKV buffer (s <= 512).
// Forward: o = softmax_causal(alpha Q K^T) V written to o[token][head * d + j] (j < d), and the
// per-row log2-domain normaliser lse2 = max(alpha log2e S) + log2(sum) to lse[z * s + row].
int attn_fwd(const void* qkv, long long lq, int b, int heads, int s, int d, int dp, float alpha,
             void* o, long long ldo, float* lse, cudaStream_t st);
// Backward: dqkv[:, 0:h) = dQ, [h, 2h) = dK, [2h, 3h) = dV (head n at n*d; ld = ldq), from dO
// (bf16 [tokens][heads*dp], padded like q) and the forward's o / lse.  Dbuf: fp32 [b*heads*s]
// workspace (D_i = dO_i . O_i).  P is recomputed from S and lse (never stored).
int attn_bwd(const void* qkv, long long lq, const void* dO, const void* o, long long ldo,
             const float* lse, float* Dbuf, int b, int heads, int s, int d, int dp, float alpha,
             void* dqkv, long long ldq, cudaStream_t st);
int preload_attn();
int preload_gemm();    // force-load kernels (no lazy module load behind a spinning NCCL kernel)
int preload_ops();
int preload_adamw();
int adamw_launch(long long n, const void* g16, float* theta, float* m, float* v, void* theta16,
                 const float* scalars9, cudaStream_t st);
// AdamW on g = fp32 sum over j < ng (ascending) of g16s[j][0..n) (the column all-reduce fused in)
int adamw_sum_launch(long long n, const void* const* g16s, int ng, float* theta, float* m, float* v,
                     void* theta16, const float* scalars9, cudaStream_t st);

// ops.cu
int embed_fwd(const int32_t* tok, long long tok_ld, int b, int s, int h, const void* etok,
              const void* epos, void* out, cudaStream_t st);
int embed_bwd(const int32_t* tok, long long tok_ld, int b, int s, int h, int vocab, const void* dx,
              float* detok, float* dpos, cudaStream_t st);
int ln_fwd(const void* x, int rows, int h, const void* g, const void* b, void* y, float* mean,
           float* rstd, cudaStream_t st);
int ln_bwd(const void* dy, const void* x, const float* mean, const float* rstd, int rows, int h,
           const void* g, const void* dres, void* dx, cudaStream_t st);
int colsum_chunks(int rows);
// LayerNorm backward (as ln_bwd) with d gamma (+)= sum_r du xhat, d beta (+)= sum_r du and, if
// out_s, out_s (+)= sum_r bf16(dx) fused; workspace >= 3 * ln_bwd_cs_parts(rows) * h floats
int ln_bwd_cs(const void* du, const void* x, const float* mean, const float* rstd, int rows, int h,
              const void* g, const void* dres, void* dx, float* out_g, float* out_b, float* out_s,
              int accumulate, float* workspace, cudaStream_t st);
int ln_bwd_cs_parts(int rows);
// out (+)= column sums of a bf16 [rows][h] tensor in ln_bwd_cs's summation order
int colsum_lnc(const void* dy, int rows, int h, float* out, int accumulate, float* workspace,
               cudaStream_t st);
int colsum(const void* dy, const void* x, const float* mean, const float* rstd, int rows, int n,
           float* workspace, float* out_b, float* out_g, int accumulate, cudaStream_t st);
int softmax_fwd(const float* S, long long nrows, int s, void* P, cudaStream_t st);
int softmax_bwd(const void* P, const float* dP, long long nrows, int s, float scale, void* dS,
                cudaStream_t st);
int xent(void* z, const int32_t* labels, long long lab_ld, int rows, int s, int V, float coef,
         float* row_loss, cudaStream_t st);
int reduce_sum(const float* x, int n, float scale, double* out, cudaStream_t st);
// flag = 1 if any of the n int32 token ids is outside [0, vocab) (flag is not cleared)
int token_check(const int32_t* tok, long long n, int vocab, int* flag, cudaStream_t st);
int cast_f32_hx(const float* in, void* out, long long n, cudaStream_t st);
// flag = 1 if any of the n 16-bit values is inf / NaN (flag is not cleared)
int nonfinite_scan(const void* x, long long n, int* flag, cudaStream_t st);
int cast_hx_f32(const void* in, float* out, long long n, cudaStream_t st);
int init_normal(void* out, float* master, long long n, uint64_t seed, float mean, float stdv,
                cudaStream_t st);

}  // namespace axonn
