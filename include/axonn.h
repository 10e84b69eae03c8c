/* axonn.h — C-ABI of the B200-native AxoNN hybrid training step.
 *
 * The library implements ONE thing: the data-parallel hot path of AxoNN
 * (arXiv 2110.13005, /root/reference/PAPER.md), i.e. Alg. 1 `train` /
 * `data_parallel_step` with the Alg. 2 message-driven
 * inter-layer step, the data-parallel gradient all-reduce
 * and the bucketed, host-offloaded optimizer with
 * all-reduce/optimizer overlap — for a GPT-style
 * transformer (readings D-1..D-9 in DESIGN.md §2).
 *
 * Conventions (all calls):
 *  - every call returns an axonn_status; no exception crosses the ABI;
 *  - one context per process / GPU; calls are not thread-safe; every call
 *    makes the context's device current;
 *  - the library owns the device memory, pinned host memory, CUDA streams,
 *    events and NCCL communicators it creates; caller pointers are borrowed
 *    for the duration of the call only;
 *  - CUDA and NCCL errors are sticky: after one, only axonn_last_error and
 *    axonn_free are valid on that context;
 *  - there is no CPU fallback: without a usable sm_100a device axonn_init
 *    fails with AXONN_ERR_CUDA.
 */
#ifndef AXONN_H
#define AXONN_H

#include <stdint.h>

#if defined(__GNUC__)
#define AXONN_API __attribute__((visibility("default")))
#else
#define AXONN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct axonn_ctx axonn_ctx;

typedef enum {
  AXONN_OK = 0,
  AXONN_ERR_INVALID_ARG = -1,          /* bad pointer / size / hyperparameter */
  AXONN_ERR_GRID_MISMATCH = -2,        /* world_size != g_inter * g_data */
  AXONN_ERR_NONDIVISIBLE_LAYERS = -3,  /* g_inter does not divide n_layers */
  AXONN_ERR_NONDIVISIBLE_BATCH = -4,   /* g_data * microbatch does not divide batch */
  AXONN_ERR_OOM = -5,
  AXONN_ERR_CUDA = -6,
  AXONN_ERR_NCCL = -7,
  AXONN_ERR_STATE = -8,                /* call out of order (e.g. optimizer_step without run_batch) */
  AXONN_ERR_NONFINITE = -9,            /* non-finite gradient: step skipped, t not incremented */
  AXONN_ERR_TIMEOUT = -10              /* scheduler watchdog: no message progress */
} axonn_status;

/* Half-precision format of theta16, activations, messages and the all-reduce
 * (PAPER.md:193-206 mixed precision).  bf16 is the B200 default (reading D-31);
 * fp16 is the paper's own format and needs a loss scale (D-11) with the
 * overflow skip of D-12.  The format is a build-time specialisation of every
 * kernel: libaxonn.so computes in bf16, libaxonn_fp16.so in fp16, both export
 * this same ABI (axonn_half_dtype says which). */
typedef enum { AXONN_BF16 = 0, AXONN_FP16 = 1 } axonn_dtype;

/* GPT shape (layers, hidden size, heads; seq and vocab PAPER.md:839-840). */
typedef struct {
  int n_layers, hidden, heads, seq_len, vocab;
  uint64_t init_seed;   /* weights N(0,0.02) (D-22) generated on device; overwrite with axonn_write_tensor */
  int dtype;            /* axonn_dtype; must equal axonn_half_dtype() of the loaded library,
                           else axonn_init returns AXONN_ERR_INVALID_ARG */
} axonn_model_cfg;

/* Optimizer and memory-optimisation knobs. */
typedef struct {
  double lr, beta1, beta2, eps, weight_decay; /* paper: 1e-3, 0.9, 0.999, (1e-8, D-13), 0.01;
                                                 step scalars are formed in double, rounded once (D-14) */
  double loss_scale;                          /* S (D-11): static; the loss (hence every gradient)
                                                 is multiplied by S in the backward and K9 divides
                                                 it out.  1 for bf16; fp16: a
                                                 power of two such as 1024 */
  int offload;                                /* 1: fp32 theta + Adam state in pinned host memory */
  int64_t bucket_elems;                       /* bsize in elements (D-16); paper 4M */
  int coarsen_k;                              /* all-reduce chunk = k * bsize elements; paper 4 */
  int pipeline_limit;                         /* 0 -> G_inter */
  int checkpoint_interval;                    /* activation checkpointing ac: 0 or 1
                                                 off; -1 the paper's rule (factor of n_layers / G_inter
                                                 closest to sqrt(n_layers)); k > 1 explicit, must divide
                                                 the stage's layer count (else AXONN_ERR_INVALID_ARG,
                                                 "BadCheckpointInterval").  Values are unchanged. */
  int overlap_next_batch;                     /* 1: axonn_optimizer_step returns once every bucket is
                                                 enqueued; the next axonn_run_batch starts at once and
                                                 each layer's forward waits only for the buckets that
                                                 hold its parameters (results are identical; reading
                                                 D-32).  0: the step completes before returning. */
  int stage_balance;                          /* 0: l / G_inter whole layers per stage (PAPER.md:615-617,
                                                 D-21).  1: stage boundaries at half-layer granularity
                                                 (after a layer's attention block or after its MLP
                                                 block) chosen to minimise the largest stage cost in
                                                 forward FLOPs including the last stage's LM head
                                                 (reading D-21b); G_inter need not divide n_layers.
                                                 Values are unchanged; requires checkpoint_interval <= 1. */
  const double* stage_speed;                  /* NULL: every GPU equally fast.  Else G_inter relative
                                                 speeds (finite, > 0; borrowed, read only inside
                                                 axonn_init) of the GPUs holding stage i, the slowest
                                                 replica of that stage (e.g. axonn_calibrate_speed on
                                                 every rank, min over each column): with stage_balance
                                                 each stage's cost is divided by its speed, so a GPU
                                                 held back by the power cap gets fewer blocks (reading
                                                 D-21c).  Must be identical on every rank (the column
                                                 replicas hold the same layers).  Ignored when
                                                 stage_balance = 0; non-positive or non-finite ->
                                                 AXONN_ERR_INVALID_ARG. */
  int grad_accum_fp32;                        /* 1: weight gradients accumulate over the microbatches in
                                                 fp32 and are rounded to half once per batch (reading
                                                 D-20; 8 phi device bytes with offload).  0: the paper's
                                                 footprint: the weight
                                                 matrices (w_qkv, w_o, w_fc1, w_fc2, head_w) accumulate
                                                 straight into the half gradient, grad <- RN(grad +
                                                 RN(microbatch gradient)) (reading D-38); the bias /
                                                 LayerNorm vectors and the embedding tables keep fp32
                                                 accumulators (4 phi + 4 (V + s) h on the first stage +
                                                 16 bsize with offload).  AXONN_T_GRAD32 of a matrix is
                                                 then AXONN_ERR_INVALID_ARG. */
} axonn_opt_cfg;

/* The stage split stage_balance = 1 picks (reading D-21b/c), host-only (no device work):
 * bounds[0..g_inter] receives the block boundaries 0 = b_0 < ... < b_G = 2 n_layers, stage i
 * holding residual blocks [b_i, b_{i+1}) (block 2L = attention block of layer L, 2L + 1 its
 * MLP block).  stage_speed as in axonn_opt_cfg (NULL = uniform).  Errors:
 * AXONN_ERR_INVALID_ARG for NULL model/bounds, g_inter < 1, 2 n_layers < g_inter or a bad speed. */
AXONN_API axonn_status axonn_stage_partition(const axonn_model_cfg* model, int g_inter,
                                             const double* stage_speed, int* bounds);

/* Sustained throughput of this library's K1 GEMM (C[M,N] = A[M,K] B[N,K]^T, half operands
 * N(0,1), half output) on CUDA device `device`: iters/4 + 1 untimed launches, then `iters`
 * back-to-back launches timed with CUDA events; *tflops = 2 M N K iters / time.  Allocates and
 * frees its own buffers (2 (MK + NK + MN) bytes) and stream; the calling thread's current
 * device becomes `device`.  Used to calibrate stage_speed (reading D-21c).  Errors:
 * AXONN_ERR_INVALID_ARG (M, N < 128, K < 64, any not a multiple of 8,
 * iters outside [1, 100000], NULL out),
 * AXONN_ERR_CUDA (no sm_100a device, allocation or launch failure). */
AXONN_API int axonn_calibrate_speed(int device, int M, int N, int K, int iters, double* tflops);

/* Process placement in the G_inter x G_data grid: world_rank = j * G_inter + i
 * (i = stage, j = replica, reading D-29).  nccl_id: 128-byte ncclUniqueId made
 * by rank 0 with axonn_get_unique_id and broadcast by the caller (the Python
 * binding uses torch.distributed for that; PyTorch is plumbing only).
 * Ignored when world_size == 1. */
typedef struct axonn_local_group axonn_local_group;
typedef struct {
  int world_rank, world_size;
  const void* nccl_id;
  int device;   /* CUDA ordinal */
  /* NULL (production): one process per GPU, NCCL communicators from nccl_id.
   * Non-NULL: the test-only loopback transport below; nccl_id is ignored. */
  axonn_local_group* local_group;
} axonn_dist;

/* Test-only loopback transport (SURVEY.md §4 "optional test-only loopback transport"):
 * the G_inter stages of ONE pipeline (G_data = 1) as G_inter contexts in ONE process, each
 * created and driven by its own host thread, on the same device or on different devices.
 * The Alg. 2 scheduler runs unchanged: pre-posted receives into the
 * `pipeline_limit` slots, backward-first dispatch among landed messages (D-19), stage-0
 * injection after each backward (Alg. 2 l.24-26), and the production peer-copy link: a
 * message for microbatch mb is a copy-engine copy into the neighbour's slot mb mod limit
 * followed, on the same stream, by a stream-memop store of the message's sequence number
 * into the neighbour's flag.  The only difference: the flag words live in host-mapped
 * pinned memory and the receiving stage's host thread observes them (a stream wait per
 * receive on G_inter contexts x 10 streams of one device could share a hardware queue with
 * the sender's stream and deadlock).  Slot and flag pointers are exchanged through the
 * group at axonn_init (a host rendezvous of all `size` contexts); the loss sum (C5) and the
 * fp16 overflow flag (D-12) are reduced on the host through the group.  No NCCL call is
 * made.  axonn_init with a group: world_size must equal `size`, g_data must be 1 (else
 * AXONN_ERR_INVALID_ARG); every collective call (axonn_init, axonn_run_batch,
 * axonn_optimizer_step) must be made by all `size` contexts concurrently, from different
 * threads.  If one context fails inside a collective call the group is marked failed and
 * the others return AXONN_ERR_STATE instead of waiting.  The caller frees the group after
 * every context using it (axonn_free).  Errors: AXONN_ERR_INVALID_ARG (size < 1, NULL out),
 * AXONN_ERR_OOM. */
AXONN_API axonn_status axonn_local_group_create(int size, axonn_local_group** out);
AXONN_API void axonn_local_group_free(axonn_local_group* group);

/* Tensor kinds for inspection (canonical oracle layout, fp32 on the host). */
typedef enum {
  AXONN_T_PARAM16 = 0,   /* theta16 (bf16 / fp16 on device)                            */
  AXONN_T_GRAD = 1,      /* reduced half-precision gradient (x S), input of the optimizer */
  AXONN_T_MASTER = 2,    /* fp32 master theta (device or pinned host)                  */
  AXONN_T_ADAM_M = 3,
  AXONN_T_ADAM_V = 4,
  AXONN_T_GRAD32 = 5     /* fp32 accumulation buffer (D-20)                            */
} axonn_which;

/* The half-precision format this library build computes in (axonn_dtype). */
AXONN_API int axonn_half_dtype(void);

/* Writes rank 0's 128-byte ncclUniqueId into out. */
AXONN_API axonn_status axonn_get_unique_id(void* out128);

/* Alg. 1 l.2: validate, instantiate the nn_shard of g^{i,j},
 * allocate theta16 and the gradient buffers on the device and theta32/m/v on
 * the device or in pinned host memory (offload), build NCCL communicators
 * (column all-reduce group, neighbour links).  Collective over all ranks.
 * *out = NULL on error.  Errors: GRID_MISMATCH, NONDIVISIBLE_LAYERS,
 * INVALID_ARG, OOM, CUDA, NCCL. */
AXONN_API axonn_status axonn_init(int g_inter, int g_data, int microbatch, const axonn_model_cfg* model,
                        const axonn_opt_cfg* opt, const axonn_dist* dist, axonn_ctx** out);

/* Alg. 1 l.4-6: one data_parallel_step.  Collective (SPMD).
 * tokens: host int32 [batch][seq_len + 1], the FULL batch (inputs = [:, :s],
 * labels = [:, 1:]); replica j uses rows [j*batch/G_data, (j+1)*batch/G_data).
 * Every token id must lie in [0, vocab): the whole batch is checked on the host
 * before any device work, and a bad id returns AXONN_ERR_INVALID_ARG on every
 * rank (not sticky).
 * Runs Alg. 2 on this rank; during the last microbatch's backward each layer's
 * gradients are cast to the half format and handed off in chunks of k * bsize
 * elements -- all-reduced over the column when G_data > 1 --
 * as soon as they are final.  Returns once the batch loss is known (the last
 * backward and the all-reduce may still be running on the device; the next
 * call orders after them).  *loss_out (may be NULL) = batch-mean token cross
 * entropy, unscaled, identical on all ranks.
 * Errors: NONDIVISIBLE_BATCH, INVALID_ARG (NULL tokens, token id out of range),
 * STATE (two run_batch without optimizer_step), TIMEOUT, CUDA, NCCL. */
AXONN_API axonn_status axonn_run_batch(axonn_ctx* ctx, const int32_t* tokens, int batch, float* loss_out);

/* Same as axonn_run_batch with this replica's shard already resident on the
 * device: d_tokens = device int32 [batch/G_data][seq_len + 1].  The shard's ids
 * are range-checked by a device kernel whose flag is MAX-reduced over the world
 * (one small synchronisation per batch); a bad id returns AXONN_ERR_INVALID_ARG
 * on every rank. */
AXONN_API axonn_status axonn_run_batch_device(axonn_ctx* ctx, const int32_t* d_tokens, int batch,
                                    float* loss_out);

/* Alg. 1 l.7 "run the optimizer": AdamW on every parameter of
 * this stage, bucket by bucket, each bucket's update
 * enqueued as soon as its all-reduce chunk completes;
 * refreshes theta16 = RNE(theta32).  Collective.  Errors: STATE, NONFINITE,
 * CUDA, NCCL.
 * fp16 build (reading D-12): before any bucket is updated the reduced
 * gradients of the stage are scanned for inf/NaN and the flag is MAX-reduced
 * over all ranks; if set, no parameter or Adam state changes, t is not
 * incremented and every rank returns AXONN_ERR_NONFINITE (not sticky: the
 * context stays usable and the next call is axonn_run_batch).  This scan
 * needs the whole all-reduce first, so the fp16 build gives up the
 * chunk-by-chunk all-reduce/optimizer interleave. */
AXONN_API axonn_status axonn_optimizer_step(axonn_ctx* ctx);

/* Synchronise and release everything the context owns. */
AXONN_API void axonn_free(axonn_ctx* ctx);

AXONN_API const char* axonn_last_error(const axonn_ctx* ctx);

/* Inspection (parity harness): tensors of THIS stage in canonical order
 * (oracle layout: linear weights [out, in] row-major, QKV rows q|k|v). */
AXONN_API int axonn_num_tensors(const axonn_ctx* ctx);
AXONN_API axonn_status axonn_tensor_info(const axonn_ctx* ctx, int idx, char name[64], int64_t shape[2],
                               int64_t* numel);
/* Synchronising fp32 copies; host buffers hold numel floats.  Writing
 * AXONN_T_GRAD for every tensor marks the gradients reduced, so
 * axonn_optimizer_step can run without run_batch (values are rounded to the half format).
 * Writing AXONN_T_MASTER also refreshes theta16 = RNE(theta32). */
AXONN_API axonn_status axonn_read_tensor(axonn_ctx* ctx, int which, int idx, float* host_dst);
AXONN_API axonn_status axonn_write_tensor(axonn_ctx* ctx, int which, int idx, const float* host_src);

/* The activation checkpointing interval ac this context uses (checkpoint_interval resolved;
 * 1 = off), or -1 for a NULL context.  For checkpoint_interval = -1 it is the paper's rule
 * (PAPER.md:570-573): the factor of this stage's layer count closest to sqrt(n_layers), ties
 * to the smaller factor. */
AXONN_API int axonn_checkpoint_interval(const axonn_ctx* ctx);

/* Statistics of the last batch; see AXONN_STAT_* for the index meaning. */
enum {
  AXONN_STAT_T_BATCH_MS = 0,      /* run_batch wall time (host)                 */
  AXONN_STAT_T_OPT_MS = 1,        /* optimizer_step wall time                   */
  AXONN_STAT_GEMM_MS = 2,         /* sum of K1 launch durations (profiling on)  */
  AXONN_STAT_GEMM_FLOP = 3,       /* algorithmic FLOPs of those launches        */
  AXONN_STAT_GEMM_LAUNCHES = 4,
  AXONN_STAT_KERNEL_LAUNCHES = 5, /* all own kernels launched in the last batch+step */
  AXONN_STAT_ADAM_MS = 6,         /* sum of K9 launch durations (profiling on)  */
  AXONN_STAT_ADAM_BYTES = 7,
  AXONN_STAT_P2P_BYTES = 8,
  AXONN_STAT_ALLREDUCE_BYTES = 9,
  AXONN_STAT_H2D_BYTES = 10,
  AXONN_STAT_D2H_BYTES = 11,
  /* device-timed phases (CUDA events; PAPER.md:704-708, 720-723 phase bars) */
  AXONN_STAT_T_PIPE_MS = 12,      /* Alg. 2 phase: first forward issued .. last backward done   */
  AXONN_STAT_T_BUSY_MS = 13,      /* sum of this stage's Forward/Backward spans in that phase   */
  AXONN_STAT_T_ALLREDUCE_MS = 14, /* gradient cast + column all-reduce after the phase          */
  AXONN_STAT_T_OPT_EXPOSED_MS = 15, /* optimizer time after the all-reduce (overlap: prev. step)*/
  AXONN_STAT_COUNT = 16
};
AXONN_API axonn_status axonn_stats(const axonn_ctx* ctx, double* out, int n);
/* Per-shape timing of the last profiled batch + step as a JSON object
 * {"fwd|dgrad|wgrad|attn MxNxK zZ epiE": [ms, flop, launches], "adamw": [ms, bytes, n]}.
 * Copies at most n-1 characters into buf (NUL-terminated); returns the full length. */
AXONN_API int axonn_profile_json(const axonn_ctx* ctx, char* buf, int n);
/* 1: bracket the K1 launches of the last microbatch of each batch and every K9
 * launch with CUDA events on their streams (roofline numbers in bench.py);
 * 0: off (default). */
AXONN_API axonn_status axonn_set_profiling(axonn_ctx* ctx, int on);

/* Device-side timing for benchmarks: axonn_timer_mark(ctx, id) records CUDA
 * event id (0..7) on the context's compute stream after all work enqueued so
 * far (including the optimizer); axonn_timer_elapsed synchronises on the
 * later event and returns the device time between two marks in ms. */
AXONN_API axonn_status axonn_timer_mark(axonn_ctx* ctx, int id);
AXONN_API axonn_status axonn_timer_elapsed(axonn_ctx* ctx, int id0, int id1, double* ms);

/* ---------------------------------------------------------------------------
 * Kernel-level entry points (device pointers; enqueue on `stream`, a
 * cudaStream_t or NULL for the legacy stream).  "16-bit" below = the library's
 * half format (bf16 in libaxonn.so, fp16 in libaxonn_fp16.so; the bf16 named in
 * the comments reads as that format).  Used by the kernel parity
 * tests and microbenchmarks.  Return 0 on success, < 0 on a bad argument or
 * launch failure.
 * ------------------------------------------------------------------------- */

/* K1: C[z] = epilogue(alpha * A[z] * B[z]^T), bf16 in, fp32 TMEM accumulation.
 * A: a_mn = 0 -> [M][lda] (K contiguous), a_mn = 1 -> [K][lda] (M contiguous).
 * B: b_mn = 0 -> [N][ldb], b_mn = 1 -> [K][ldb].  Batch z in [0, Z):
 * z1 = z % Z1, z2 = z / Z1, element offsets z1*s1 + z2*s2.  Leading
 * dimensions and batch strides must be multiples of 8 elements and bases
 * 16-byte aligned (TMA).  epi: 0 bf16 (+bias[N], +resid), 1 bias + GeLU
 * (stores pre-activation to aux), 2 multiply by GeLU'(aux), 3 fp32
 * (accumulate = 1 adds into C).  causal: 0 none, 1 skip tiles above the
 * diagonal, 2 k < m0 + 128, 3 k >= m0.  col_group_in/out: column remap
 * c -> (c / in) * out + c % in (0 = identity); n_valid: columns >= n_valid are
 * not stored (0 = N). */
typedef struct {
  int M, N, K, Z, Z1;
  const void* A; int64_t lda, a_s1, a_s2; int a_mn;
  const void* B; int64_t ldb, b_s1, b_s2; int b_mn;
  void* C; int64_t ldc, c_s1, c_s2;
  int epi, causal, accumulate, col_group_in, col_group_out, n_valid;
  const void* bias; const void* resid; int64_t ld_resid; void* aux; int64_t ld_aux;
  float alpha;
  int max_ctas;   /* cap on resident CTAs (0 = all SMs) */
  int variant;    /* 0 auto (CTA pairs for the linear layers, single CTAs for N <= 128 or M <= 128),
                     1 single-CTA 128 x {128, 256} tiles, 2 CTA-pair 256 x 256 tiles (cta_group::2; the
                     TMA-store epilogue when eligible; 256 x 128 pairs for N <= 128), 3 CTA pairs with the
                     thread-store epilogue; other values: as 2 but 256 x 256 pairs for N <= 128 too */
} axonn_gemm_args;
AXONN_API int axonn_k_gemm(const axonn_gemm_args* args, void* stream);

/* K9: fused AdamW over n elements (reading D-14 op order, IEEE round-to-nearest,
 * no FMA contraction).  g16: bf16 gradients; theta/m/v fp32 (in place);
 * theta16: bf16 out = RNE(theta).  Scalars as produced by the host in double
 * and rounded once to fp32: decay = 1 - lr*wd, b1, omb1 = 1 - b1, b2,
 * omb2 = 1 - b2, step = lr / (1 - b1^t), bc2_sqrt = sqrt(1 - b2^t), eps,
 * inv_scale = 1 / S. */
AXONN_API int axonn_k_adamw(int64_t n, const void* g16, float* theta, float* m, float* v, void* theta16,
                  const float scalars[9], void* stream);

/* K2: fused causal self-attention forward over one microbatch ("transformer
 * kernel", SURVEY.md §8(a) A2 "causal MHA"; readings D-7 scale alpha = 1/sqrt(d), D-8 causal).
 * qkv: bf16 [b*s][lq], lq = 3*heads*dp; Q of head n at columns [n*dp, n*dp+d), K at
 * heads*dp + n*dp, V at 2*heads*dp + n*dp (pad columns d..dp-1 must be zero).
 * o: bf16 [b*s][ldo], head n written to columns [n*d, (n+1)*d).
 * lse: fp32 [b*heads*s] (index (sample*heads + head)*s + query): log2-domain row normaliser
 * max_k(alpha*log2(e)*S) + log2(sum_k exp2(...)), consumed by the backward.
 * Limits: s <= 512, dp even and dp <= 256, d even.  Device pointers; no allocation;
 * returns 0 or a negative code (invalid shape / launch failure). */
AXONN_API int axonn_k_attn_fwd(const void* qkv, int64_t lq, int b, int heads, int s, int d, int dp,
                               float alpha, void* o, int64_t ldo, float* lse, void* stream);

/* K2 backward (same passage and readings).  From dO (bf16 [b*s][heads*dp], head n at n*dp,
 * pad columns zero), the forward's o and lse and the same qkv, writes into dqkv (bf16
 * [b*s][ldq]): dQ at columns [n*d, ...), dK at h + n*d, dV at 2h + n*d (h = heads*d), with
 * dS = alpha * P * (dP - D), D_i = dO_i . o_i.  P is recomputed from S and lse (never stored);
 * every output element has one writer (no atomics: bitwise reproducible).  dbuf: fp32
 * workspace of b*heads*s elements (receives D).  Same limits as axonn_k_attn_fwd, and
 * s % 4 == 0 (D is written 4 rows per 16-byte store); else returns -1. */
AXONN_API int axonn_k_attn_bwd(const void* qkv, int64_t lq, const void* dO, const void* o, int64_t ldo,
                               const float* lse, float* dbuf, int b, int heads, int s, int d, int dp,
                               float alpha, void* dqkv, int64_t ldq, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AXONN_H */
