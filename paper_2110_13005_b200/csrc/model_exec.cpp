// nn_shard.Forward / nn_shard.Backward of one pipeline stage (Alg. 2 l.6, 14,
// 16, 22, 25) as a chain of sm_100a kernels on s_comp.
//
// Layer = GPT-2 pre-LN block (readings D-1..D-8):
//   u = LN1(x); qkv = u Wqkv^T + b; S = Q K^T / sqrt(d) (causal); P = softmax(S);
//   o = P V; x1 = x + o Wo^T + bo; w = LN2(x1); pre = w W1^T + b1; a = GeLU(pre);
//   out = x1 + a W2^T + b2.
// Every contraction is K1 (tcgen05 GEMM) with its elementwise tail fused in the
// epilogue (bias, GeLU + pre-activation store, residual add, GeLU' in dgrad,
// fp32 weight-gradient accumulation).  The last stage adds LN_f, the untied LM
// head and the fused cross entropy with the loss pre-divided by the number of
// microbatches in the batch (D-9).
#include <cmath>
#include <cstdio>
#include <cstring>

#include "engine.h"

namespace axonn {

void Ctx::wg_fork() {
  cudaEvent_t e = ev();
  cudaEventRecord(e, s_comp);
  cudaStreamWaitEvent(s_wg, e, 0);
}
void Ctx::wg_note(const void* buf) {
  cudaEvent_t e = ev();
  cudaEventRecord(e, s_wg);
  for (auto& pr : wg_reads)
    if (pr.first == buf) { pr.second = e; return; }
  wg_reads.emplace_back(buf, e);
}
void Ctx::wg_guard(const void* buf) {
  for (auto& pr : wg_reads)
    if (pr.first == buf) cudaStreamWaitEvent(s_comp, pr.second, 0);
}
void Ctx::wg_join() {
  cudaEvent_t e = ev();
  cudaEventRecord(e, s_wg);
  cudaStreamWaitEvent(s_comp, e, 0);
  wg_reads.clear();
}

int Ctx::gemm(GemmArgs g, double flops) {
  cudaStream_t st = gst ? gst : s_comp;
  if (g.Z == 0) g.Z = 1;
  if (g.Z1 == 0) g.Z1 = 1;
  if (g.alpha == 0.f) g.alpha = 1.f;
  // NCCL links: leave two TPCs to the posted one-CTA NCCL P2P kernels (receive act/grad,
  // short sends).  Peer-copy links run on the copy engines and need no SM.
  if (g.max_ctas == 0 && g_inter > 1 && !p2p_ipc) g.max_ctas = num_sms - 4;
  // overlapped column all-reduce running (G_data > 1): leave its CTAs their SMs
  if (g.max_ctas == 0 && ar_active && g_data > 1 && dp_ctas > 0) g.max_ctas = num_sms - ((dp_ctas + 1) & ~1);
  ProfRec pr{};
  if (prof_mb) {
    pr.a = ev();
    pr.b = ev();
    pr.work = flops >= 0 ? flops : 2.0 * g.M * g.N * g.K * g.Z;
    pr.kind = flops >= 0 ? 0 : 2;
    const char* kind = flops < 0 ? "attn" : (g.a_mn && g.b_mn) ? "wgrad" : g.b_mn ? "dgrad" : "fwd";
    char key[96];
    snprintf(key, sizeof(key), "%s %dx%dx%d z%d epi%d", kind, g.M, g.N, g.K, g.Z, g.epi);
    pr.key = key;
    cudaEventRecord(pr.a, st);
  }
  int rc = gemm_launch(g, st);
  ++launches;
  if (rc) return fail(AXONN_ERR_CUDA, "gemm_launch failed rc=" + std::to_string(rc) +
                                          " M=" + std::to_string(g.M) + " N=" + std::to_string(g.N) +
                                          " K=" + std::to_string(g.K));
  if (prof_mb) {
    cudaEventRecord(pr.b, st);
    prof.push_back(pr);
  }
  return 0;
}

int Ctx::attn_call(bool fwd, LayerStash& st) {
  const int b = microbatch;
  const float alpha = 1.0f / sqrtf((float)d);
  ProfRec pr{};
  if (prof_mb) {
    pr.a = ev();
    pr.b = ev();
    // executed (causal) FLOPs: fwd Q K^T + P V, bwd recomputed S + dP + 3 accumulations
    const double half = 2.0 * b * heads * (double)s * s * dp / 2;
    pr.work = fwd ? 2 * half : 5 * half;
    pr.kind = 2;
    pr.key = fwd ? "attn_fwd (fused)" : "attn_bwd (fused)";
    cudaEventRecord(pr.a, s_comp);
  }
  int rc = fwd ? attn_fwd(st.qkv, lq, b, heads, s, d, dp, alpha, st.o, h, st.lse, s_comp)
               : attn_bwd(st.qkv, lq, dO, st.o, h, st.lse, attn_D, b, heads, s, d, dp, alpha, dqkv,
                          3LL * h, s_comp);
  launches += fwd ? 1 : 3;
  if (rc) return fail(AXONN_ERR_CUDA, std::string("attention kernel failed rc=") + std::to_string(rc));
  if (prof_mb) {
    cudaEventRecord(pr.b, s_comp);
    prof.push_back(pr);
  }
  return 0;
}

static GemmArgs lin_fwd(const void* X, const void* W, int M, int N, int K, void* out) {
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.M = M; g.N = N; g.K = K;
  g.A = X; g.lda = K;
  g.B = W; g.ldb = K;
  g.C = out; g.ldc = N;
  g.epi = EPI_HALF;
  return g;
}
// dX[M, Kin] = dY[M, Nout] W[Nout, Kin]
static GemmArgs lin_dgrad(const void* dY, const void* W, int M, int Nout, int Kin, void* dX) {
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.M = M; g.N = Kin; g.K = Nout;
  g.A = dY; g.lda = Nout;
  g.B = W; g.ldb = Kin; g.b_mn = 1;
  g.C = dX; g.ldc = Kin;
  g.epi = EPI_HALF;
  return g;
}
// dW[Nout, Kin] (+)= dY^T X
static GemmArgs lin_wgrad(const void* dY, const void* X, int M, int Nout, int Kin, float* dW,
                          int accumulate) {
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.M = Nout; g.N = Kin; g.K = M;
  g.A = dY; g.lda = Nout; g.a_mn = 1;
  g.B = X; g.ldb = Kin; g.b_mn = 1;
  g.C = dW; g.ldc = Kin;
  g.epi = EPI_F32;
  g.accumulate = accumulate;
  return g;
}

// dW[Nout, Kin] (+)= dY^T X into the tensor at flat offset off: fp32 (D-20), or with
// grad_accum_fp32 = 0 straight into the half gradient, RN(dW + RN(dY^T X)) (reading D-38)
GemmArgs Ctx::wgrad_args(const void* dY, const void* X, int M_, int Nout, int Kin, int64_t off, int acc) const {
  GemmArgs g = lin_wgrad(dY, X, M_, Nout, Kin, half_accum ? nullptr : g32(off), acc);
  if (half_accum) {
    g.C = static_cast<char*>(grad16) + off * 2;
    g.epi = EPI_HALF;
  }
  return g;
}

#define TRY(x)              \
  do {                      \
    int _rc = (x);          \
    if (_rc) return _rc;    \
  } while (0)
#define KCHK(x)                                                                       \
  do {                                                                                \
    ++launches;                                                                       \
    if ((x) != 0) return fail(AXONN_ERR_CUDA, std::string("kernel launch failed: ") + #x); \
  } while (0)

int Ctx::layer_fwd(int li, const void* x, LayerStash& st) {
  const LayerOff& o = loff[li];
  const int b = microbatch;
  const double dM = M, dh = h;
  const int hm = lhalf[li];   // attention block (bit 0) and / or MLP block (bit 1) on this stage
  if (hm & 1) {
  KCHK(ln_fwd(x, M, h, p16(o.ln1_g), p16(o.ln1_b), st.u, st.mean1, st.rstd1, s_comp));
  {
    GemmArgs g = lin_fwd(st.u, p16(o.w_qkv), M, 3 * h, h, st.qkv);
    g.bias = p16(o.b_qkv);
    g.ldc = lq;   // packed [M, 3, heads, dp]: heads padded to dp (TMA strides, D-7)
    if (dp != d) { g.col_group_in = d; g.col_group_out = dp; }
    TRY(gemm(g, 2 * dM * 3 * dh * dh));
  }
  if (flash_attn()) {   // K2: o = softmax_causal(Q K^T / sqrt(d)) V, S and P stay in TMEM
    TRY(attn_call(true, st));
  } else {
    {  // S = Q K^T / sqrt(d) per (sample, head), causal tile skipping (D-7, D-8)
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.M = s; g.N = s; g.K = dp; g.Z = b * heads; g.Z1 = heads;
      g.A = st.qkv; g.lda = lq; g.a_s1 = dp; g.a_s2 = (long long)s * lq;
      g.B = static_cast<char*>(st.qkv) + (size_t)heads * dp * 2; g.ldb = lq; g.b_s1 = dp;
      g.b_s2 = (long long)s * lq;
      g.C = S; g.ldc = s; g.c_s1 = (long long)s * s; g.c_s2 = (long long)heads * s * s;
      g.epi = EPI_F32; g.causal = 1; g.alpha = 1.0f / sqrtf((float)d);
      TRY(gemm(g, -1));
      KCHK(softmax_fwd(S, (long long)b * heads * s, s, st.P, s_comp));
    }
    {  // o = P V, heads merged into [M, h]
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.M = s; g.N = dp; g.K = s; g.Z = b * heads; g.Z1 = heads; g.n_valid = d;
      g.A = st.P; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)heads * s * s;
      g.B = static_cast<char*>(st.qkv) + (size_t)2 * heads * dp * 2; g.ldb = lq; g.b_s1 = dp;
      g.b_s2 = (long long)s * lq; g.b_mn = 1;
      g.C = st.o; g.ldc = h; g.c_s1 = d; g.c_s2 = (long long)s * h;
      g.epi = EPI_HALF; g.causal = 2;
      TRY(gemm(g, -1));
    }
  }
  {
    // a stage cut after this attention block sends x1: written straight into the peer's slot
    void* x1_dst = (!(hm & 2) && out_redirect) ? out_redirect : st.x1;
    GemmArgs g = lin_fwd(st.o, p16(o.w_o), M, h, h, x1_dst);
    g.bias = p16(o.b_o);
    g.resid = x; g.ld_resid = h;
    TRY(gemm(g, 2 * dM * dh * dh));
  }
  }   // attention block
  if (!(hm & 2)) return 0;
  const void* x1 = (hm & 1) ? st.x1 : x;   // a stage starting at the MLP block receives x1
  KCHK(ln_fwd(x1, M, h, p16(o.ln2_g), p16(o.ln2_b), st.w, st.mean2, st.rstd2, s_comp));
  {
    GemmArgs g = lin_fwd(st.w, p16(o.w_fc1), M, 4 * h, h, st.act);
    g.bias = p16(o.b_fc1);
    g.epi = EPI_BIAS_GELU; g.aux = st.pre; g.ld_aux = 4 * h;
    TRY(gemm(g, 2 * dM * 4 * dh * dh));
  }
  {
    // the stage output: straight into the next stage's receive slot (direct send, §5 / N3)
    GemmArgs g = lin_fwd(st.act, p16(o.w_fc2), M, h, 4 * h, out_redirect ? out_redirect : st.out);
    g.bias = p16(o.b_fc2);
    g.resid = x1; g.ld_resid = h;
    TRY(gemm(g, 2 * dM * 4 * dh * dh));
  }
  return 0;
}

int Ctx::layer_bwd(int li, const void* x, LayerStash& st, const void* dout, void* din) {
  const LayerOff& o = loff[li];
  const int b = microbatch;
  const int acc = bwd_count > 0 ? 1 : 0;
  const double dM = M, dh = h;
  // Weight gradients (dW GEMM + bias column sum) go to s_wg, concurrent with the
  // data-gradient chain on s_comp; wg_guard() orders any later overwrite of a buffer
  // s_wg still reads.
  const int hm = lhalf[li];
  // the column sum of dout (this layer's first bias gradient) was fused into the LayerNorm
  // backward that produced dout (LN1 of the layer above, or LN_f) -- see ln_bwd_cs
  const bool dout_summed = dout_bias_fused;
  dout_bias_fused = false;
  float* const ws_ln = cs_ws_ln + 1024;   // ln_bwd_cs partials (past colsum2's tickets)
  // gradient w.r.t. x1: from the MLP block, or (stage cut after the attention block) dout
  const void* gx1 = dout;
  bool gx1_summed = dout_summed;
  if (hm & 2) {
  const void* x1 = (hm & 1) ? st.x1 : x;
  void* dx1o = (hm & 1) ? dx1 : din;   // MLP-only layer: dx1 is the stage's input gradient
  // FC2: dpre = (dout W2) * GeLU'(pre);  dW2 += dout^T act;  db2 += colsum(dout)
  wg_fork();
  gst = wgs();
  TRY(gemm(wgrad_args(dout, st.act, M, h, 4 * h, o.w_fc2, acc), 2 * dM * 4 * dh * dh));
  gst = s_comp;
  if (!dout_summed)   // received output gradient: the fused sum's order (bitwise = G_inter 1)
    KCHK(colsum_lnc(dout, M, h, g32(o.b_fc2), acc, cs_ws + 1024, wgs()));
  wg_note(dout);
  wg_guard(dpre);
  {
    GemmArgs g = lin_dgrad(dout, p16(o.w_fc2), M, h, 4 * h, dpre);
    g.epi = EPI_DGELU; g.aux = st.pre; g.ld_aux = 4 * h;
    TRY(gemm(g, 2 * dM * 4 * dh * dh));
  }
  // FC1: du = dpre W1;  dW1 += dpre^T w;  db1 += colsum(dpre)
  wg_fork();
  gst = wgs();
  TRY(gemm(wgrad_args(dpre, st.w, M, 4 * h, h, o.w_fc1, acc), 2 * dM * 4 * dh * dh));
  gst = s_comp;
  KCHK(colsum(dpre, nullptr, nullptr, nullptr, M, 4 * h, cs_ws, g32(o.b_fc1), nullptr, acc, wgs()));
  wg_note(dpre);
  TRY(gemm(lin_dgrad(dpre, p16(o.w_fc1), M, 4 * h, h, du), 2 * dM * 4 * dh * dh));
  // LN2: dx1 = dout + LN2'(du);  dg2, db2; and dbo = colsum(dx1) when the attention block follows
  wg_guard(dx1o);
  KCHK(ln_bwd_cs(du, x1, st.mean2, st.rstd2, M, h, p16(o.ln2_g), dout, dx1o, g32(o.ln2_g), g32(o.ln2_b),
                 (hm & 1) ? g32(o.b_o) : nullptr, acc, ws_ln, s_comp));
  gx1 = dx1o;
  gx1_summed = (hm & 1) != 0;
  }   // MLP block
  if (!(hm & 1)) return 0;
  // proj: dO = dx1 Wo;  dWo += dx1^T o;  dbo += colsum(dx1)
  wg_fork();
  gst = wgs();
  TRY(gemm(wgrad_args(gx1, st.o, M, h, h, o.w_o, acc), 2 * dM * dh * dh));
  gst = s_comp;
  if (!gx1_summed)   // received gradient of x1 (stage cut after this attention block)
    KCHK(colsum_lnc(gx1, M, h, g32(o.b_o), acc, cs_ws + 1024, wgs()));
  wg_note(gx1);
  {
    GemmArgs g = lin_dgrad(gx1, p16(o.w_o), M, h, h, dO);
    g.ldc = (long long)heads * dp;   // dO per head, padded like q/k/v
    if (dp != d) { g.col_group_in = d; g.col_group_out = dp; }
    TRY(gemm(g, 2 * dM * dh * dh));
  }
  wg_guard(dqkv);
  // attention backward
  if (flash_attn()) {   // K2 backward: dQ, dK, dV straight into dqkv (P recomputed)
    TRY(attn_call(false, st));
  } else {
    {  // dP = dO V^T (fp32 into S)
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.M = s; g.N = s; g.K = dp; g.Z = b * heads; g.Z1 = heads;
      g.A = dO; g.lda = (long long)heads * dp; g.a_s1 = dp; g.a_s2 = (long long)s * heads * dp;
      g.B = static_cast<char*>(st.qkv) + (size_t)2 * heads * dp * 2; g.ldb = lq; g.b_s1 = dp;
      g.b_s2 = (long long)s * lq;
      g.C = S; g.ldc = s; g.c_s1 = (long long)s * s; g.c_s2 = (long long)heads * s * s;
      g.epi = EPI_F32; g.causal = 1;
      TRY(gemm(g, -1));
      KCHK(softmax_bwd(st.P, S, (long long)b * heads * s, s, 1.0f / sqrtf((float)d), dS, s_comp));
    }
    {  // dQ = dS K  -> dqkv[:, 0:h]
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.M = s; g.N = dp; g.K = s; g.Z = b * heads; g.Z1 = heads; g.n_valid = d;
      g.A = dS; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)heads * s * s;
      g.B = static_cast<char*>(st.qkv) + (size_t)heads * dp * 2; g.ldb = lq; g.b_s1 = dp;
      g.b_s2 = (long long)s * lq; g.b_mn = 1;
      g.C = dqkv; g.ldc = 3 * h; g.c_s1 = d; g.c_s2 = (long long)s * 3 * h;
      g.epi = EPI_HALF; g.causal = 2;
      TRY(gemm(g, -1));
    }
    {  // dK = dS^T Q -> dqkv[:, h:2h]
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.M = s; g.N = dp; g.K = s; g.Z = b * heads; g.Z1 = heads; g.n_valid = d;
      g.A = dS; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)heads * s * s; g.a_mn = 1;
      g.B = st.qkv; g.ldb = lq; g.b_s1 = dp; g.b_s2 = (long long)s * lq; g.b_mn = 1;
      g.C = static_cast<char*>(dqkv) + (size_t)h * 2; g.ldc = 3 * h; g.c_s1 = d;
      g.c_s2 = (long long)s * 3 * h;
      g.epi = EPI_HALF; g.causal = 3;
      TRY(gemm(g, -1));
    }
    {  // dV = P^T dO -> dqkv[:, 2h:3h]
      GemmArgs g;
      memset(&g, 0, sizeof(g));
      g.M = s; g.N = dp; g.K = s; g.Z = b * heads; g.Z1 = heads; g.n_valid = d;
      g.A = st.P; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)heads * s * s; g.a_mn = 1;
      g.B = dO; g.ldb = (long long)heads * dp; g.b_s1 = dp; g.b_s2 = (long long)s * heads * dp;
      g.b_mn = 1;
      g.C = static_cast<char*>(dqkv) + (size_t)2 * h * 2; g.ldc = 3 * h; g.c_s1 = d;
      g.c_s2 = (long long)s * 3 * h;
      g.epi = EPI_HALF; g.causal = 3;
      TRY(gemm(g, -1));
    }
  }
  // QKV: du = dqkv Wqkv;  dWqkv += dqkv^T u;  dbqkv += colsum(dqkv)
  wg_fork();
  gst = wgs();
  TRY(gemm(wgrad_args(dqkv, st.u, M, 3 * h, h, o.w_qkv, acc), 2 * dM * 3 * dh * dh));
  gst = s_comp;
  KCHK(colsum(dqkv, nullptr, nullptr, nullptr, M, 3 * h, cs_ws, g32(o.b_qkv), nullptr, acc, wgs()));
  wg_note(dqkv);
  TRY(gemm(lin_dgrad(dqkv, p16(o.w_qkv), M, 3 * h, h, du), 2 * dM * 3 * dh * dh));
  // LN1: din = dx1 + LN1'(du)   (din is the buffer the layer above read as dout)
  wg_guard(din);
  // LN1, with the column sum of din fused when it is the output gradient of the layer below
  // on this stage (whose first bias gradient is its FC2 bias: only a stage's top layer can
  // lack its MLP block)
  float* below = li > 0 ? g32(loff[li - 1].b_fc2) : nullptr;
  KCHK(ln_bwd_cs(du, x, st.mean1, st.rstd1, M, h, p16(o.ln1_g), gx1, din, g32(o.ln1_g), g32(o.ln1_b), below,
                 acc, ws_ln, s_comp));
  dout_bias_fused = below != nullptr;
  return 0;
}

// nn_shard.Forward for microbatch mb into slot sl.  Stage 0 embeds its tokens;
// the last stage also runs LN_f, the LM head and the fused, pre-divided loss.
int Ctx::forward(Slot& sl, int mb) {
  cudaEvent_t b0 = ev(), b1 = ev();   // busy span (after any message wait the caller enqueued)
  cudaEventRecord(b0, s_comp);
  const int rc = forward_impl(sl, mb);
  cudaEventRecord(b1, s_comp);
  busy_ev.emplace_back(b0, b1);
  busy_tag.push_back(2 * mb);
  return rc;
}

int Ctx::forward_impl(Slot& sl, int mb) {
  // K1 launches are bracketed by CUDA events only for one microbatch of the batch (every
  // microbatch runs the same GEMM shapes; bracketing all of them would perturb the timed step
  // by several percent): a middle one, (m - 1) / 2, whose kernels do not share the GPU with
  // the optimizer chunks that start during the last backward (A8)
  prof_mb = profiling && mb == (cur_m - 1) / 2;
  const int b = microbatch;
  const int32_t* tok = dtok + (size_t)mb * b * (s + 1);
  if (first) {
    wait_params(pos_emb + ((int64_t)s * h + 63) / 64 * 64);   // overlapped optimizer step (D-32)
    KCHK(embed_fwd(tok, s + 1, b, s, h, p16(tok_emb), p16(pos_emb), sl.in, s_comp));
  }
  const void* x = sl.in;
  for (int li = 0; li < nl; ++li) {
    wait_params(layer_end(li));
    if (ac > 1) {   // the segment's last layer writes the kept segment boundary
      LayerStash st = stash(sl, li);
      if (li % ac == ac - 1) st.out = sl.seg[li / ac + 1];
      TRY(layer_fwd(li, x, st));
      x = st.out;
    } else {
      // direct send: the top layer's output GEMM stores into the next stage's slot
      out_redirect = (li == nl - 1 && !last && direct_send) ? peer_act[mb % limit] : nullptr;
      const int rf = layer_fwd(li, x, sl.L[li]);
      out_redirect = nullptr;
      TRY(rf);
      x = layer_out(sl.L[li], li);
    }
  }
  if (!last) return 0;
  wait_params(nflat);
  KCHK(ln_fwd(x, M, h, p16(lnf_g), p16(lnf_b), sl.hf, sl.meanf, sl.rstdf, s_comp));
  TRY(gemm(lin_fwd(sl.hf, p16(head_w), M, V, h, logits), 2.0 * M * V * h));
  const float coef = (float)(oc.loss_scale / ((double)cur_mtotal * (double)M));
  KCHK(xent(logits, tok + 1, s + 1, M, s, V, coef, row_loss, s_comp));
  KCHK(reduce_sum(row_loss, M, 1.0f / ((float)cur_mtotal * (float)M), d_loss, s_comp));
  // the batch loss is final after the last microbatch's forward (forwards run in ascending mb)
  if (mb == cur_m - 1 && cudaEventRecord(ev_loss, s_comp) != cudaSuccess)
    return fail(AXONN_ERR_CUDA, "loss event");
  return 0;
}

// nn_shard.Backward: dout = received output-gradient (nullptr on the last
// stage, where Backward(1) starts from the cross-entropy gradient already
// written in place of the logits).  The input gradient goes to sl.gsend.
int Ctx::backward(Slot& sl, int mb, const void* dout) {
  cudaEvent_t b0 = ev(), b1 = ev();
  cudaEventRecord(b0, s_comp);
  const int rc = backward_impl(sl, mb, dout);
  cudaEventRecord(b1, s_comp);
  busy_ev.emplace_back(b0, b1);
  busy_tag.push_back(2 * mb + 1);
  return rc;
}

int Ctx::backward_impl(Slot& sl, int mb, const void* dout) {
  prof_mb = profiling && mb == (cur_m - 1) / 2;
  if (half_accum && bwd_count == 0) {   // the batch's first write of grad16 (D-38)
    // the previous optimizer step (this rank's K9, and with the fused column reduction the
    // peers' K9) must be done reading grad16
    if (opt_pending)
      if (int rc = check_cuda(cudaStreamWaitEvent(s_comp, ev_opt_done, 0), "half accum wait opt")) return rc;
    if (dp_fused && dp_epoch > 1)
      if (int rc = dp_wait(s_comp, g_data, dp_epoch - 1)) return rc;
  }
  const int b = microbatch;
  const int acc = bwd_count > 0 ? 1 : 0;
  const int32_t* tok = dtok + (size_t)mb * b * (s + 1);
  const bool ar_last = ar_overlap && bwd_count == cur_m - 1;   // backwards run in ascending mb
  dout_bias_fused = false;   // a received output gradient has no fused column sum
  void* cur = dh0;
  void* nxt = dh1;
  if (last) {
    const void* xL = stage_out(sl);
    wg_fork();
    gst = wgs();
    TRY(gemm(wgrad_args(logits, sl.hf, M, V, h, head_w, acc), 2.0 * M * V * h));
    gst = s_comp;
    TRY(gemm(lin_dgrad(logits, p16(head_w), M, V, h, du), 2.0 * M * V * h));
    // LN_f, with the column sum of its output gradient (the top layer's first bias gradient)
    float* top = nullptr;
    if (nl > 0) top = (lhalf[nl - 1] & 2) ? g32(loff[nl - 1].b_fc2) : g32(loff[nl - 1].b_o);
    KCHK(ln_bwd_cs(du, xL, sl.meanf, sl.rstdf, M, h, p16(lnf_g), nullptr, cur, g32(lnf_g), g32(lnf_b), top,
                   acc, cs_ws_ln + 1024, s_comp));
    dout_bias_fused = top != nullptr;
    if (ar_last) TRY(ar_ready(lnf_g));
  } else {
    cur = const_cast<void*>(dout);
  }
  for (int li = nl - 1; li >= 0; --li) {
    const void* x;
    if (ac > 1) {
      const int sg = li / ac;
      if (li % ac == ac - 1) {   // recompute the segment's forward from its kept input
        wg_join();                 // s_wg may still read the scratch stash of the segment above
        const void* xr = sl.seg[sg];
        for (int j = sg * ac; j <= li; ++j) {
          TRY(layer_fwd(j, xr, stash(sl, j)));
          xr = stash(sl, j).out;
        }
      }
      x = li % ac == 0 ? sl.seg[sg] : stash(sl, li - 1).out;
    } else {
      x = li > 0 ? layer_out(sl.L[li - 1], li - 1) : sl.in;
    }
    // direct send: the stage-input gradient goes straight into the previous stage's slot
    void* din = (li == 0 && !first) ? (direct_send ? peer_grad[mb % limit] : sl.gsend) : nxt;
    TRY(layer_bwd(li, x, stash(sl, li), cur, din));
    if (ar_last && !(first && li == 0)) TRY(ar_ready(layer_begin(li)));
    if (li == 0 && !first) {
      cur = din;
    } else {
      cur = din;
      nxt = (din == dh0) ? dh1 : dh0;
    }
  }
  if (first) {
    // embedding gradients (fp32, zeroed at batch start): deterministic scatter-add
    KCHK(embed_bwd(tok, s + 1, b, s, h, V, cur, g32(tok_emb), g32(pos_emb), s_comp));
  }
  if (ar_last) TRY(ar_ready(0));
  wg_join();   // stash, logits and gradient buffers are reused by the next microbatch
  ++bwd_count;
  return 0;
}

}  // namespace axonn
