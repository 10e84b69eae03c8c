// Host engine of the AxoNN hybrid step (H1 context, H2 scheduler, H3 optimizer
// driver, H5 batch plumbing).  Internal — the boundary is
// include/axonn.h.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/axonn.h"
#include "kernels.h"

namespace axonn {

#ifdef AXONN_HALF_FP16
constexpr ncclDataType_t kNcclHalf = ncclFloat16;
#else
constexpr ncclDataType_t kNcclHalf = ncclBfloat16;
#endif

struct TensorRec {
  std::string name;
  int64_t rows, cols, numel, off;   // off: element offset in every flat buffer
  int64_t off32;                    // offset in grad32; -1: accumulates in grad16 (grad_accum_fp32 = 0)
};

// Element offsets of one layer's tensors in the flat buffers (D-2 layout).
struct LayerOff {
  int64_t ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_fc1, b_fc1, w_fc2, b_fc2;
};

// Activations saved by a layer's forward for its backward (one microbatch).
struct LayerStash {
  void *u, *qkv, *P, *o, *x1, *w, *pre, *act, *out;
  float *mean1, *rstd1, *mean2, *rstd2;
  float* lse = nullptr;               // fused attention: log2-domain row normaliser [b*heads*s]
};

// One in-flight microbatch on this stage (pipeline_limit of them, Alg. 2).
struct Slot {
  void* in = nullptr;                 // stage input [M, h]: embedding output or received activation
  std::vector<LayerStash> L;          // full stash per layer (no checkpointing)
  std::vector<void*> seg;             // checkpointing: input of segment j (seg[0] = in), seg[nl/ac] = stage output
  void* hf = nullptr;                 // last stage: LN_f output
  float *meanf = nullptr, *rstdf = nullptr;
  void* gsend = nullptr;              // gradient w.r.t. the stage input, sent to stage i-1
  void* grecv = nullptr;              // output gradient received from stage i+1
  int mb = -1;
};

struct ProfRec {
  cudaEvent_t a, b;
  double work;
  int kind;   // 0 linear-layer GEMM, 1 adam, 2 attention GEMM
  std::string key;   // "fwd|dgrad|wgrad|attn MxNxK epi"
};

struct Ctx {
  // ---- configuration
  int g_inter = 1, g_data = 1, microbatch = 1;
  axonn_model_cfg mc{};
  axonn_opt_cfg oc{};
  int rank = 0, world = 1, device = 0;
  int stage = 0, replica = 0;
  bool first = true, last = true;
  int nl = 0, layer0 = 0;             // local layers, first global layer id
  int h = 0, heads = 0, d = 0, s = 0, V = 0, M = 0;   // M = microbatch * seq tokens
  int dp = 0;                         // head dim padded to a multiple of 8 (16-B TMA strides)
  long long lq = 0;                   // row stride of the packed qkv buffer = 3 * heads * dp
  int limit = 1;
  std::string err;
  bool sticky = false;
  int num_sms = 148;

  // ---- parameters
  std::vector<TensorRec> tensors;
  int64_t nflat = 0;
  int64_t tok_emb = -1, pos_emb = -1, lnf_g = -1, lnf_b = -1, head_w = -1;
  std::vector<LayerOff> loff;
  // per local layer: bit 0 its attention block, bit 1 its MLP block lives on this stage (3 =
  // whole layer; a balanced split, stage_balance, may cut a layer after its attention block)
  std::vector<int> lhalf;
  void* theta16 = nullptr;            // bf16 [nflat]
  float* grad32 = nullptr;            // fp32 accumulation (D-20); with half_accum only the
                                      // vectors and embedding tables (TensorRec::off32)
  int64_t n32 = 0;                    // elements of grad32
  bool half_accum = false;            // grad_accum_fp32 = 0: matrices accumulate in grad16 (D-38)
  void* grad16 = nullptr;             // bf16 all-reduce / optimizer input
  float *master = nullptr, *adam_m = nullptr, *adam_v = nullptr;   // device or pinned host
  float* ring[3][3] = {};             // offload ring: [slot][theta, m, v]
  int64_t t_step = 0;

  // ---- activations / workspace
  std::vector<void*> allocs;
  std::vector<Slot> slots;
  float* S = nullptr;                 // scores / dP fp32 [b a s s]
  void* dS = nullptr;                 // bf16 [b a s s]
  void *dh0 = nullptr, *dh1 = nullptr, *dqkv = nullptr, *dpre = nullptr, *dO = nullptr,
       *du = nullptr, *dx1 = nullptr;
  float* cs_ws = nullptr;             // column-sum workspace (bias sums, s_wg)
  float* cs_ws_ln = nullptr;          // column-sum workspace (LayerNorm sums, s_comp)
  void* logits = nullptr;             // [M, V] bf16 (last stage)
  float* row_loss = nullptr;
  double* d_loss = nullptr;           // device loss accumulator
  double* h_loss = nullptr;           // pinned
  int* d_flag = nullptr;              // fp16 overflow flag (reading D-12), in d_loss's 64 B
  int* h_flag = nullptr;              // pinned copy, in h_loss's 64 B
  int32_t* dtok = nullptr;            // this replica's token shard [B/G_data, s+1]
  int64_t dtok_cap = 0;

  // ---- streams / events / comms
  cudaStream_t s_comp = nullptr, s_send_act = nullptr, s_send_grad = nullptr,
               s_recv_act = nullptr, s_recv_grad = nullptr, s_dp = nullptr, s_h2d = nullptr,
               s_d2h = nullptr, s_opt = nullptr;
  // batch loss (C5): its world all-reduce and D2H run here, off s_dp, so run_batch can return
  // once the loss is known while the gradient chunks are still being reduced on s_dp
  cudaStream_t s_loss = nullptr;
  // weight-gradient side stream: dW GEMMs and bias column sums of the backward run here,
  // concurrently with the data-gradient chain on s_comp (fills GEMM tail waves)
  cudaStream_t s_wg = nullptr;
  cudaStream_t gst = nullptr;         // stream the next gemm() launches on (s_comp default)
  std::vector<std::pair<const void*, cudaEvent_t>> wg_reads;   // buffers s_wg still reads
  ncclComm_t world_comm = nullptr, dp_comm = nullptr, act_out = nullptr, act_in = nullptr,
             grad_out = nullptr, grad_in = nullptr;
  std::vector<ncclComm_t> owned_comms;
  // Pipeline link transport (Alg. 2 messages).  p2p_ipc = 1 (default): the
  // sender's copy engine writes the message over NVLink straight into the neighbour's receive
  // slot (CUDA IPC mapping), then a stream memop stores the message's sequence number into
  // the receiver's flag; the receiver's stream waits on that flag (no SM is held by a
  // pending receive).  p2p_ipc = 0 (AXONN_P2P=nccl): NCCL send/recv on 2-rank link comms.
  int p2p_ipc = 0;
  uint32_t* flags = nullptr;          // device [2 * limit]: act slot k, then grad slot k
  std::vector<void*> peer_act;        // stage + 1's slot.in buffers, mapped here
  std::vector<void*> peer_grad;       // stage - 1's slot.grecv buffers, mapped here
  uint32_t* peer_flags_next = nullptr;   // stage + 1's flags
  uint32_t* peer_flags_prev = nullptr;   // stage - 1's flags
  std::vector<void*> ipc_opened;
  // test-only loopback transport (axonn_local_group, include/axonn.h): flags are host-mapped
  // and observed by this context's host thread; loss / overflow flag reduced through the group
  axonn_local_group* lg = nullptr;
  volatile uint32_t* flags_host = nullptr;
  // Fused column reduction (reading D-35; G_data > 1, bf16 build): there is
  // no all-reduce call.  During the last backward each replica casts its gradient chunks to
  // the half format (Ctx::ar_ready) and stores a progress value into every peer's flag word;
  // each replica's K9 then waits for its chunk's flags and sums the G_data replicas' half
  // gradients itself, reading the peers' grad16 over NVLink (CUDA IPC mappings; loopback:
  // buffers of the other contexts on this device).  After its last K9 a replica stores a
  // read-done value into every peer, and a replica's next cast waits for all of them.
  // AXONN_DP=nccl selects ncclAllReduce instead (the fp16 build always does: its overflow
  // scan needs the reduced gradient).
  bool dp_fused = false;
  std::vector<const void*> dp_g16;    // [G_data] grad16 of replica j (own one at [replica])
  uint32_t* dp_flags = nullptr;       // device-visible [2 G_data]: progress of j, read-done of j
  volatile uint32_t* dp_flags_host = nullptr;   // loopback: host view of dp_flags
  std::vector<uint32_t*> dp_peer_flags;         // [G_data] replica k's dp_flags (mapped)
  uint32_t dp_epoch = 0;              // batches reduced so far (1-based during a batch)
  int64_t n_chunks = 0;
  int dp_wait(cudaStream_t st, int base, uint32_t value);     // every peer's flag base + j >= value
  int dp_signal(cudaStream_t st, int slot, uint32_t value);   // store value into every peer's slot
  uint32_t dp_progress(int64_t chunk) const {                 // chunk ready in this epoch
    return dp_epoch * (uint32_t)(n_chunks + 1) + (uint32_t)(n_chunks - chunk);
  }
  // Direct send: with peer-copy links and no activation checkpointing the
  // kernel that produces a message writes it straight into the neighbour's mapped receive slot
  // (the top layer's output GEMM through its TMA epilogue; the stage-input gradient's
  // LayerNorm backward by P2P stores) and a stream memop then stores the sequence number into
  // the neighbour's flag -- no copy-engine pass.  AXONN_P2P=copy keeps the copy.
  bool direct_send = false;
  void* out_redirect = nullptr;       // output of the top layer's last GEMM (during its forward)
  uint32_t msg_base = 0;              // sequence number base: messages of earlier batches
  cudaEvent_t ev_grads_ready = nullptr, ev_opt_done = nullptr, ev_loss = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  cudaEvent_t ev_h2d[3] = {}, ev_adam[3] = {}, ev_d2h[3] = {};
  cudaEvent_t timer[8] = {};
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;

  // ---- state / stats
  bool grads_ready = false;           // run_batch (or GRAD writes) done, optimizer pending
  int bwd_count = 0;                  // backwards done in this batch (first one stores)
  int cur_mtotal = 1;
  int cur_m = 1;                      // microbatches of this replica in the current batch
  bool prof_mb = false;               // profile the launches of the current microbatch
  int write_grad_mask = 0;
  std::vector<char> grad_written;
  bool profiling = false;
  std::vector<ProfRec> prof;
  // optimizer / next-batch overlap (overlap_next_batch, reading D-32)
  bool opt_pending = false;           // an optimizer step is still running on s_opt
  // phase events per step parity: [0] phase start, [1] phase end (s_comp), [2] all-reduce
  // done, [3] optimizer done; busy spans = (start, end) event pairs around Forward/Backward
  cudaEvent_t ph[2][4] = {};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> busy_ev;
  std::vector<int> busy_tag;          // 2 mb (+1 for a Backward) per busy span
  std::vector<std::pair<int, cudaEvent_t>> msg_ev;   // message landed: (2 mb (+1 grad), event)
  void phase_stats_ar_opt(int par);
  int pipe_stats_par = -1;            // batch whose pipeline phase statistics are pending
  void pipe_stats(int par);
  // Chunked gradient hand-off during the batch's last backward (reading D-32): as each layer's
  // gradients become final (reverse layer order = descending flat index) its range is cast to
  // the half format on s_dp and every chunk (k * bsize elements) lying wholly
  // above the frontier is all-reduced over the column (G_data > 1) or just marked ready
  // (G_data = 1), top chunk first, one event per chunk.  The optimizer step then runs its
  // buckets in chunk-completion order, each waiting only for its chunk (A8),
  // so K9 starts while the rest of the backward and of the all-reduce are still running.
  bool ar_overlap = false;            // this batch hands gradients off chunk by chunk
  bool ar_active = false;             // an overlapped all-reduce has been issued (SM reservation)
  int dp_ctas = 0;                    // AXONN_DP_CTAS: cap of the column comm's CTAs, reserved
  int64_t ar_hi = 0;                  // gradients [ar_hi, nflat) are cast and handed to s_dp
  int64_t ar_next_chunk = -1;         // highest chunk not yet issued
  int ar_ready(int64_t lo);           // gradients [lo, ar_hi) are final on s_comp / s_wg
  std::vector<cudaEvent_t> ev_bucket; // K9 of bucket b done (theta16 of the bucket written)
  std::vector<ProfRec> prof_opt;      // AdamW records of the pending step
  void wait_params(int64_t off_end);  // s_comp waits until theta16[0, off_end) is updated
  void collect_stats();               // kernel-time statistics from completed records
  double stats[AXONN_STAT_COUNT] = {};
  std::string prof_json = "{}";       // per-shape K1 / K9 timing of the last profiled step
  long long launches = 0;

  // helpers
  cudaEvent_t ev();                   // next event from the pool (reset per batch)
  std::vector<cudaEvent_t> ev_pool_opt;   // optimizer-step events (reset per step: they must
  size_t ev_next_opt = 0;                 // outlive the overlapped next batch)
  cudaEvent_t ev_opt();
  void* dalloc(size_t bytes);
  int check_cuda(cudaError_t e, const char* what);
  int check_nccl(ncclResult_t r, const char* what);
  int fail(int code, const std::string& msg);

  void* p16(int64_t off) const { return static_cast<char*>(theta16) + off * 2; }
  float* g32(int64_t off) const {   // fp32 accumulator of the tensor starting at off
    if (!half_accum) return grad32 + off;
    const TensorRec* t = tensor_at(off);
    return t && t->off32 >= 0 ? grad32 + t->off32 : nullptr;
  }
  const TensorRec* tensor_at(int64_t off) const {   // tensors are in ascending off
    size_t lo = 0, hi = tensors.size();
    while (lo < hi) {
      const size_t mid = (lo + hi) / 2;
      if (tensors[mid].off < off) lo = mid + 1;
      else hi = mid;
    }
    return lo < tensors.size() && tensors[lo].off == off ? &tensors[lo] : nullptr;
  }
  int cast_grads(int64_t lo, int64_t hi, cudaStream_t st);   // grad32 -> grad16 over [lo, hi)
  GemmArgs wgrad_args(const void* dY, const void* X, int M_, int Nout, int Kin, int64_t off, int acc) const;

  // model execution (model_exec.cpp)
  int gemm(GemmArgs g, double flops);
  // K2 fused attention when the shape fits it; else the general path (S = Q K^T by K1 into an
  // fp32 score buffer, softmax kernels, P V by K1)
  bool flash_attn() const { return s <= 512 && d % 2 == 0 && ((dp + 63) / 64) * 64 <= 256; }
  float* attn_D = nullptr;            // fused attention backward workspace (D = dO . O)
  int attn_call(bool fwd, LayerStash& st);   // K2 launch (+ profiling events)
  int forward(Slot& sl, int mb);          // nn_shard.Forward (and the loss on the last stage)
  int backward(Slot& sl, int mb, const void* dout);   // nn_shard.Backward
  int forward_impl(Slot& sl, int mb);
  int backward_impl(Slot& sl, int mb, const void* dout);
  int layer_fwd(int li, const void* x, LayerStash& st);
  // activation checkpointing: with ac > 1 the layers share ac scratch
  // stashes; a slot keeps only the segment inputs and the backward recomputes each segment
  int ac = 1;
  std::vector<LayerStash> ck;
  LayerStash& stash(Slot& sl, int li) { return ac > 1 ? ck[li % ac] : sl.L[li]; }
  // output of local layer li: x1 when the stage ends after the layer's attention block
  const void* layer_out(const LayerStash& st, int li) const { return (lhalf[li] & 2) ? st.out : st.x1; }
  const void* stage_out(const Slot& sl) const {
    if (ac > 1) return sl.seg[nl / ac];
    return nl > 0 ? layer_out(sl.L[nl - 1], nl - 1) : sl.in;
  }
  int64_t layer_end(int li) const {   // one past the last flat element of layer li on this stage
    return ((lhalf[li] & 2) ? loff[li].b_fc2 : loff[li].b_o) + ((int64_t)h + 63) / 64 * 64;
  }
  int64_t layer_begin(int li) const { return (lhalf[li] & 1) ? loff[li].ln1_g : loff[li].ln2_g; }
  int layer_bwd(int li, const void* x, LayerStash& st, const void* dout, void* din);
  bool dout_bias_fused = false;       // the next layer_bwd's dout column sum is already done
  void wg_fork();                       // s_wg waits for everything enqueued on s_comp so far
  void wg_note(const void* buf);        // s_wg reads buf (recorded after its last enqueued read)
  void wg_guard(const void* buf);       // s_comp waits before overwriting buf
  void wg_join();                       // s_comp waits for all of s_wg
  // the profiled microbatch runs its weight gradients in order on s_comp so the CUDA-event
  // duration of every K1 launch is its own (overlapped launches would share the GPU)
  cudaStream_t wgs() const { return prof_mb ? s_comp : s_wg; }
};

}  // namespace axonn
