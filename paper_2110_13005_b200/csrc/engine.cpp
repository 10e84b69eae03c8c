// AxoNN hybrid step engine: context lifecycle (Alg. 1 l.2), the Alg. 2
// message-driven scheduler over NCCL P2P, the column gradient all-reduce
// (Alg. 1 l.13) chunked by k*bsize and the bucketed,
// optionally host-offloaded AdamW overlapped with it.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <new>
#include <map>
#include <thread>

#include "engine.h"

// Test-only loopback group (include/axonn.h): a host rendezvous of `size` contexts in one
// process, with a sum / max reduction riding on each rendezvous and a registry of the
// stages' receive slots and flag words.
struct axonn_local_group {
  struct Reg {   // indexed by world rank (= replica * G_inter + stage)
    uint32_t* flags = nullptr;          // device-visible address of the stage's flag words
    std::vector<void*> act, grad;       // receive slots: activations (slot.in), gradients (slot.grecv)
    const void* g16 = nullptr;          // half gradients (fused column reduction, G_data > 1)
    uint32_t* dp_flags = nullptr;       // device-visible address of its column flag words
  };
  int size = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool failed = false;
  double acc_sum = 0, res_sum = 0;
  int acc_max = 0, res_max = 0;
  std::vector<Reg> reg;
  std::mutex preload_mu;                // kernel preloading / attribute setup, one thread at a time

  // Every member calls this; returns 0 with the sum of `*sum` and the max of `*mx` over the
  // group written back (either may be NULL), or -1 if the group failed or timed out.
  int rendezvous(double* sum, int* mx, double timeout_s) {
    std::unique_lock<std::mutex> lk(mu);
    if (failed) return -1;
    acc_sum += sum ? *sum : 0.0;
    acc_max = std::max(acc_max, mx ? *mx : 0);
    const uint64_t g = gen;
    if (++arrived == size) {
      res_sum = acc_sum;
      res_max = acc_max;
      acc_sum = 0;
      acc_max = 0;
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || failed; }) ||
               failed) {
      failed = true;
      cv.notify_all();
      return -1;
    }
    if (sum) *sum = res_sum;
    if (mx) *mx = res_max;
    return 0;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    failed = true;
    cv.notify_all();
  }
};

namespace axonn {

static double group_timeout_s() {
  const char* e = getenv("AXONN_WATCHDOG_S");   // same bound as the Alg. 2 watchdog
  return e ? atof(e) : 600.0;
}

// ------------------------------------------------------------------ helpers
int Ctx::fail(int code, const std::string& msg) {
  if (err.empty() || !sticky) err = msg;
  if (code == AXONN_ERR_CUDA || code == AXONN_ERR_NCCL || code == AXONN_ERR_TIMEOUT) sticky = true;
  return code;
}
int Ctx::check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  return fail(e == cudaErrorMemoryAllocation ? AXONN_ERR_OOM : AXONN_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}
int Ctx::check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  return fail(AXONN_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
void* Ctx::dalloc(size_t bytes) {
  void* p = nullptr;
  bytes = (bytes + 255) & ~size_t(255);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  allocs.push_back(p);
  return p;
}
cudaEvent_t Ctx::ev() {
  if (ev_next == ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ev_pool.push_back(e);
  }
  return ev_pool[ev_next++];
}

cudaEvent_t Ctx::ev_opt() {
  if (ev_next_opt == ev_pool_opt.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ev_pool_opt.push_back(e);
  }
  return ev_pool_opt[ev_next_opt++];
}

// host side of the 16-bit reads / writes (theta16 and GRAD inspection): RNE to the library's
// half format (half.cuh; the cuda_bf16 / cuda_fp16 conversions are host-callable)
static uint16_t f2h16(float f) {
  const hx h = f2hx(f);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static float h162f(uint16_t b) {
  hx h;
  memcpy(&h, &b, 2);
  return hx2f(h);
}

#define CU(x)                                  \
  do {                                         \
    int _rc = c->check_cuda((x), #x);          \
    if (_rc) return (axonn_status)_rc;         \
  } while (0)
#define NC(x)                                  \
  do {                                         \
    int _rc = c->check_nccl((x), #x);          \
    if (_rc) return (axonn_status)_rc;         \
  } while (0)

// ------------------------------------------------------------------ parameter table
static void build_tensors(Ctx* c) {
  const int h = c->h, V = c->V, s = c->s;
  int64_t off = 0;
  auto add = [&](const std::string& n, int64_t r, int64_t cc) {
    TensorRec t{n, r, cc, r * cc, off};
    off += (r * cc + 63) / 64 * 64;   // 128-byte (bf16) / 256-byte (fp32) aligned views
    c->tensors.push_back(t);
    return t.off;
  };
  if (c->first) {
    c->tok_emb = add("tok_emb", V, h);
    c->pos_emb = add("pos_emb", s, h);
  }
  for (int li = 0; li < c->nl; ++li) {
    std::string p = "l" + std::to_string(c->layer0 + li) + ".";
    LayerOff o{-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
    if (c->lhalf[li] & 1) {   // attention block
      o.ln1_g = add(p + "ln1_g", 1, h);
      o.ln1_b = add(p + "ln1_b", 1, h);
      o.w_qkv = add(p + "w_qkv", 3 * h, h);
      o.b_qkv = add(p + "b_qkv", 1, 3 * h);
      o.w_o = add(p + "w_o", h, h);
      o.b_o = add(p + "b_o", 1, h);
    }
    if (c->lhalf[li] & 2) {   // MLP block
      o.ln2_g = add(p + "ln2_g", 1, h);
      o.ln2_b = add(p + "ln2_b", 1, h);
      o.w_fc1 = add(p + "w_fc1", 4 * h, h);
      o.b_fc1 = add(p + "b_fc1", 1, 4 * h);
      o.w_fc2 = add(p + "w_fc2", h, 4 * h);
      o.b_fc2 = add(p + "b_fc2", 1, h);
    }
    c->loff.push_back(o);
  }
  if (c->last) {
    c->lnf_g = add("lnf_g", 1, h);
    c->lnf_b = add("lnf_b", 1, h);
    c->head_w = add("head_w", V, h);
  }
  c->nflat = off;
  // grad_accum_fp32 = 0 (reading D-38): the weight matrices accumulate in grad16; everything
  // else keeps an fp32 accumulator in a compact grad32
  c->n32 = 0;
  for (TensorRec& t : c->tensors) {
    const std::string leaf = t.name.substr(t.name.find('.') == std::string::npos ? 0 : t.name.find('.') + 1);
    const bool matrix = leaf == "w_qkv" || leaf == "w_o" || leaf == "w_fc1" || leaf == "w_fc2" || leaf == "head_w";
    if (!c->half_accum) {
      t.off32 = t.off;
    } else if (matrix) {
      t.off32 = -1;
    } else {
      t.off32 = c->n32;
      c->n32 += (t.numel + 63) / 64 * 64;
    }
  }
  if (!c->half_accum) c->n32 = c->nflat;
}

// half gradients of [lo, hi) from the fp32 accumulators (D-20): the whole
// range, or with half_accum (D-38) only the tensors that accumulate in fp32
int Ctx::cast_grads(int64_t lo, int64_t hi, cudaStream_t st) {
  if (hi <= lo) return 0;
  if (!half_accum) {
    if (cast_f32_hx(grad32 + lo, static_cast<char*>(grad16) + lo * 2, hi - lo, st))
      return fail(AXONN_ERR_CUDA, "cast");
    ++launches;
    return 0;
  }
  for (const TensorRec& t : tensors) {
    if (t.off32 < 0) continue;
    const int64_t a = std::max(lo, t.off), b = std::min(hi, t.off + t.numel);
    if (a >= b) continue;
    if (cast_f32_hx(grad32 + t.off32 + (a - t.off), static_cast<char*>(grad16) + a * 2, b - a, st))
      return fail(AXONN_ERR_CUDA, "cast");
    ++launches;
  }
  return 0;
}

// D-22 initialisation on the device (bf16-representable by truncation, D-15).
static int init_weights(Ctx* c) {
  uint64_t seed = c->mc.init_seed;
  const float proj = 0.02f / sqrtf(2.0f * c->mc.n_layers);
  float* m32 = c->oc.offload ? nullptr : c->master;
  for (size_t i = 0; i < c->tensors.size(); ++i) {
    const TensorRec& t = c->tensors[i];
    const std::string leaf = t.name.substr(t.name.find('.') == std::string::npos ? 0 : t.name.find('.') + 1);
    float mean = 0.f, sd = 0.02f;
    if (leaf.size() > 2 && leaf.compare(leaf.size() - 2, 2, "_g") == 0) { mean = 1.f; sd = 0.f; }
    else if ((leaf.size() > 2 && leaf.compare(leaf.size() - 2, 2, "_b") == 0) || leaf.rfind("b_", 0) == 0) sd = 0.f;
    else if (leaf == "w_o" || leaf == "w_fc2") sd = proj;
    // the stream of a tensor depends only on its global name (not on the stage split), so
    // every G_inter / stage_balance partition starts from the same model
    uint64_t hname = 1469598103934665603ull;   // FNV-1a
    for (char ch : t.name) hname = (hname ^ (uint8_t)ch) * 1099511628211ull;
    if (init_normal(c->p16(t.off), m32 ? m32 + t.off : nullptr, t.numel,
                    seed * 1000003ull + hname, mean, sd, c->s_comp))
      return c->fail(AXONN_ERR_CUDA, "init_normal");
  }
  if (c->oc.offload) {   // theta32 = theta16 exactly at step 0 (D-15)
    std::vector<uint16_t> tmp(c->nflat);
    if (cudaMemcpyAsync(tmp.data(), c->theta16, c->nflat * 2, cudaMemcpyDeviceToHost, c->s_comp) != cudaSuccess ||
        cudaStreamSynchronize(c->s_comp) != cudaSuccess)
      return c->fail(AXONN_ERR_CUDA, "init offload copy");
    for (int64_t i = 0; i < c->nflat; ++i) c->master[i] = h162f(tmp[i]);
  }
  return 0;
}

static int64_t chunk_elems(const Ctx* c) {
  return (int64_t)c->oc.coarsen_k * c->oc.bucket_elems;
}

// ------------------------------------------------------------------ peer-copy links
// Stream memory operations (driver API, resolved once through the runtime's entry-point query).
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static void* driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return p;
}
static int wait_flag(Ctx* c, cudaStream_t st, const uint32_t* flag, uint32_t v, bool geq = false) {
  static PFN_waitValue32 fn = (PFN_waitValue32)driver_fn("cuStreamWaitValue32");
  if (!fn) return c->fail(AXONN_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  if (fn((CUstream)st, (CUdeviceptr)flag, v, geq ? CU_STREAM_WAIT_VALUE_GEQ : CU_STREAM_WAIT_VALUE_EQ) !=
      CUDA_SUCCESS)
    return c->fail(AXONN_ERR_CUDA, "cuStreamWaitValue32");
  return 0;
}
static int write_flag(Ctx* c, cudaStream_t st, uint32_t* flag, uint32_t v) {
  static PFN_writeValue32 fn = (PFN_writeValue32)driver_fn("cuStreamWriteValue32");
  if (!fn) return c->fail(AXONN_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  // default flags: the write is ordered after, and made visible after, the preceding copy
  if (fn((CUstream)st, (CUdeviceptr)flag, v, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    return c->fail(AXONN_ERR_CUDA, "cuStreamWriteValue32");
  return 0;
}

// Exchange CUDA IPC handles of the receive slots and flags with both neighbours (over the
// already-connected NCCL link comms, in ascending boundary order like the warm-up) and map
// the neighbours' buffers.  After this a message is one copy-engine transfer + one flag store.
static int ipc_links(Ctx* c) {
  const int L = c->limit;
  const size_t HB = sizeof(cudaIpcMemHandle_t);
  const size_t pk = (size_t)(1 + L) * HB;
  int rc;
  c->flags = (uint32_t*)c->dalloc(2 * L * sizeof(uint32_t));
  if (!c->flags) return c->fail(AXONN_ERR_OOM, "link flags");
  if ((rc = c->check_cuda(cudaMemset(c->flags, 0, 2 * L * sizeof(uint32_t)), "flags"))) return rc;
  std::vector<char> up(pk), down(pk), got(pk);   // up: to stage-1 (my act slots), down: to stage+1
  if ((rc = c->check_cuda(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)up.data(), c->flags), "ipc flags")))
    return rc;
  memcpy(down.data(), up.data(), HB);
  for (int k = 0; k < L; ++k) {
    if (!c->first &&
        (rc = c->check_cuda(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)(up.data() + (1 + k) * HB), c->slots[k].in),
                            "ipc act slot")))
      return rc;
    if (!c->last &&
        (rc = c->check_cuda(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)(down.data() + (1 + k) * HB),
                                                c->slots[k].grecv), "ipc grad slot")))
      return rc;
  }
  char* dbuf = (char*)c->dalloc(pk);
  if (!dbuf) return c->fail(AXONN_ERR_OOM, "ipc exchange buffer");
  auto xfer = [&](bool send, std::vector<char>& host, ncclComm_t comm, int peer) -> int {
    int r;
    if (send) {
      if ((r = c->check_cuda(cudaMemcpy(dbuf, host.data(), pk, cudaMemcpyHostToDevice), "ipc h2d"))) return r;
      if ((r = c->check_nccl(ncclSend(dbuf, pk, ncclChar, peer, comm, c->s_comp), "ipc send"))) return r;
      return c->check_cuda(cudaStreamSynchronize(c->s_comp), "ipc sync");
    }
    if ((r = c->check_nccl(ncclRecv(dbuf, pk, ncclChar, peer, comm, c->s_comp), "ipc recv"))) return r;
    if ((r = c->check_cuda(cudaStreamSynchronize(c->s_comp), "ipc sync"))) return r;
    return c->check_cuda(cudaMemcpy(host.data(), dbuf, pk, cudaMemcpyDeviceToHost), "ipc d2h");
  };
  auto open = [&](const char* h, void** ptr) -> int {
    cudaIpcMemHandle_t hd;
    memcpy(&hd, h, HB);
    int r = c->check_cuda(cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess), "ipc open");
    if (!r) c->ipc_opened.push_back(*ptr);
    return r;
  };
  for (int kb = 0; kb < c->g_inter - 1; ++kb) {
    if (kb == c->stage) {            // lower end: give my grad slots, map the upper's act slots
      if ((rc = xfer(true, down, c->act_out, 1)) || (rc = xfer(false, got, c->grad_in, 1))) return rc;
      void* p;
      if ((rc = open(got.data(), &p))) return rc;
      c->peer_flags_next = (uint32_t*)p;
      c->peer_act.assign(L, nullptr);
      for (int k = 0; k < L; ++k)
        if ((rc = open(got.data() + (1 + k) * HB, &c->peer_act[k]))) return rc;
    } else if (kb == c->stage - 1) {   // upper end
      if ((rc = xfer(false, got, c->act_in, 0)) || (rc = xfer(true, up, c->grad_out, 0))) return rc;
      void* p;
      if ((rc = open(got.data(), &p))) return rc;
      c->peer_flags_prev = (uint32_t*)p;
      c->peer_grad.assign(L, nullptr);
      for (int k = 0; k < L; ++k)
        if ((rc = open(got.data() + (1 + k) * HB, &c->peer_grad[k]))) return rc;
    }
  }
  return 0;
}

// Fused column reduction (reading D-35): exchange CUDA IPC handles of grad16 and of the column
// flag words with the other replicas of this stage (all-gather over the column comm) and map
// them.  K9 then reads the peers' half gradients over NVLink.
static int dp_links(Ctx* c) {
  const int G = c->g_data;
  const size_t HB = sizeof(cudaIpcMemHandle_t);
  int rc;
  c->dp_flags = (uint32_t*)c->dalloc(2 * G * sizeof(uint32_t));
  if (!c->dp_flags) return c->fail(AXONN_ERR_OOM, "dp flags");
  if ((rc = c->check_cuda(cudaMemset(c->dp_flags, 0, 2 * G * sizeof(uint32_t)), "dp flags"))) return rc;
  std::vector<char> mine(2 * HB), all(2 * HB * G);
  if ((rc = c->check_cuda(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)mine.data(), c->grad16), "ipc grad16")) ||
      (rc = c->check_cuda(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)(mine.data() + HB), c->dp_flags),
                          "ipc dp flags")))
    return rc;
  char* dbuf = (char*)c->dalloc(2 * HB * (G + 1));
  if (!dbuf) return c->fail(AXONN_ERR_OOM, "dp ipc exchange buffer");
  if ((rc = c->check_cuda(cudaMemcpy(dbuf, mine.data(), 2 * HB, cudaMemcpyHostToDevice), "dp ipc h2d")) ||
      (rc = c->check_nccl(ncclAllGather(dbuf, dbuf + 2 * HB, 2 * HB, ncclChar, c->dp_comm, c->s_comp),
                          "dp ipc allgather")) ||
      (rc = c->check_cuda(cudaStreamSynchronize(c->s_comp), "dp ipc sync")) ||
      (rc = c->check_cuda(cudaMemcpy(all.data(), dbuf + 2 * HB, 2 * HB * G, cudaMemcpyDeviceToHost), "dp ipc d2h")))
    return rc;
  c->dp_g16.assign(G, nullptr);
  c->dp_peer_flags.assign(G, nullptr);
  for (int j = 0; j < G; ++j) {
    if (j == c->replica) {
      c->dp_g16[j] = c->grad16;
      c->dp_peer_flags[j] = c->dp_flags;
      continue;
    }
    void* p = nullptr;
    cudaIpcMemHandle_t hd;
    memcpy(&hd, all.data() + 2 * HB * j, HB);
    if ((rc = c->check_cuda(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess), "ipc open grad16")))
      return rc;
    c->ipc_opened.push_back(p);
    c->dp_g16[j] = p;
    memcpy(&hd, all.data() + 2 * HB * j + HB, HB);
    if ((rc = c->check_cuda(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess), "ipc open dp flags")))
      return rc;
    c->ipc_opened.push_back(p);
    c->dp_peer_flags[j] = (uint32_t*)p;
  }
  return 0;
}

// Loopback links (test-only local group): the flag words are host-mapped pinned memory
// (written by the neighbours' stream memops, observed by this context's host thread); slot
// and flag addresses are published in the group and read back after a rendezvous.
static int local_links(Ctx* c) {
  const int L = c->limit;
  axonn_local_group* g = c->lg;
  int rc;
  uint32_t* hf = nullptr;
  if ((rc = c->check_cuda(cudaHostAlloc((void**)&hf, 2 * L * sizeof(uint32_t),
                                        cudaHostAllocMapped | cudaHostAllocPortable), "host flags")))
    return rc;
  memset(hf, 0, 2 * L * sizeof(uint32_t));
  c->flags_host = hf;
  if ((rc = c->check_cuda(cudaHostGetDevicePointer((void**)&c->flags, hf, 0), "host flags map"))) return rc;
  uint32_t* dpf = nullptr;
  if (c->dp_fused) {   // column flag words, host-mapped so this thread can observe them
    if ((rc = c->check_cuda(cudaHostAlloc((void**)&dpf, 2 * c->g_data * sizeof(uint32_t),
                                          cudaHostAllocMapped | cudaHostAllocPortable), "host dp flags")))
      return rc;
    memset(dpf, 0, 2 * c->g_data * sizeof(uint32_t));
    c->dp_flags_host = dpf;
    if ((rc = c->check_cuda(cudaHostGetDevicePointer((void**)&c->dp_flags, dpf, 0), "host dp flags map")))
      return rc;
  }
  {
    std::lock_guard<std::mutex> lk(g->mu);
    axonn_local_group::Reg& r = g->reg[c->rank];
    r.g16 = c->grad16;
    r.dp_flags = c->dp_flags;
    r.flags = c->flags;
    r.act.assign(L, nullptr);
    r.grad.assign(L, nullptr);
    for (int k = 0; k < L; ++k) {
      r.act[k] = c->slots[k].in;
      r.grad[k] = c->slots[k].grecv;
    }
  }
  if (g->rendezvous(nullptr, nullptr, group_timeout_s())) return c->fail(AXONN_ERR_STATE, "local group failed");
  std::lock_guard<std::mutex> lk(g->mu);
  if (!c->last) {
    c->peer_flags_next = g->reg[c->rank + 1].flags;
    c->peer_act = g->reg[c->rank + 1].act;
  }
  if (!c->first) {
    c->peer_flags_prev = g->reg[c->rank - 1].flags;
    c->peer_grad = g->reg[c->rank - 1].grad;
  }
  if (c->dp_fused) {   // the column: replicas j of this stage, rank j * G_inter + stage
    c->dp_g16.assign(c->g_data, nullptr);
    c->dp_peer_flags.assign(c->g_data, nullptr);
    for (int j = 0; j < c->g_data; ++j) {
      c->dp_g16[j] = g->reg[j * c->g_inter + c->stage].g16;
      c->dp_peer_flags[j] = g->reg[j * c->g_inter + c->stage].dp_flags;
    }
  }
  return 0;
}

// Reading D-21b (stage_balance): the 2l residual blocks (attention block of layer L = block
// 2L, its MLP block = 2L + 1) are cut into G_inter contiguous ranges minimising the largest
// stage cost, cost = forward FLOPs per token weighted by the measured relative speed of the
// kernels that execute them: attention block 8h^2 + W * 2sh (QKV and projection GEMMs; the
// causal QK^T and PV of the fused attention kernel, which ran at ~1/4 of the GEMMs' TFLOP/s:
// W = 4), MLP block 16h^2, plus the LM head 2hV on the last stage
// (the embedding gather is negligible).  Exact DP over (stage, boundary); ties go to the
// earliest boundary.  With stage_speed (the measured relative speed of the GPUs holding each
// stage, slowest replica; axonn_calibrate_speed) a stage's cost is divided by its speed, so a
// GPU that runs slower under the power cap gets fewer blocks (reading D-21c).
// Returns G_inter + 1 boundaries (0 = b_0 < b_1 < ... < b_P = 2l).
static std::vector<int> balanced_blocks(const axonn_model_cfg* m, int P, const double* speed) {
  const int nb = 2 * m->n_layers;
  const double h = m->hidden, s = m->seq_len, V = m->vocab;
  std::vector<double> pre(nb + 1, 0.0);
  const double w_att = 4.0;
  for (int k = 0; k < nb; ++k) pre[k + 1] = pre[k] + ((k & 1) ? 16 * h * h : 8 * h * h + w_att * 2 * s * h);
  const double head = 2 * h * V;
  auto cost = [&](int i, int a, int b) {
    return (pre[b] - pre[a] + (i == P - 1 ? head : 0.0)) / (speed ? speed[i] : 1.0);
  };
  const double INF = 1e300;
  std::vector<std::vector<double>> best(P + 1, std::vector<double>(nb + 1, INF));
  std::vector<std::vector<int>> arg(P + 1, std::vector<int>(nb + 1, -1));
  best[0][0] = 0;
  for (int i = 1; i <= P; ++i)
    for (int b = i; b <= nb; ++b)
      for (int a = i - 1; a < b; ++a) {
        if (best[i - 1][a] >= INF) continue;
        const double v = std::max(best[i - 1][a], cost(i - 1, a, b));
        if (v < best[i][b] * (1 - 1e-12)) { best[i][b] = v; arg[i][b] = a; }
      }
  std::vector<int> bb(P + 1, 0);
  bb[P] = nb;
  for (int i = P; i > 0; --i) bb[i - 1] = arg[i][bb[i]];
  return bb;
}

// ------------------------------------------------------------------ init
static int split_comm(Ctx* c, ncclComm_t parent, int color, int key, ncclComm_t* out,
                      int max_ctas) {
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  if (max_ctas > 0) {
    cfg.maxCTAs = max_ctas;
    cfg.minCTAs = 1;
  }
  ncclComm_t nc = nullptr;
  int rc = c->check_nccl(ncclCommSplit(parent, color, key, &nc, &cfg), "ncclCommSplit");
  if (rc) return rc;
  if (nc) c->owned_comms.push_back(nc);
  *out = nc;
  return 0;
}

static int alloc_stash(Ctx* c, LayerStash& st) {
  const size_t Mh = (size_t)c->M * c->h;
  const size_t att = (size_t)c->microbatch * c->heads * c->s * c->s;
  st.u = c->dalloc(Mh * 2);
  st.qkv = c->dalloc((size_t)c->M * c->lq * 2);
  if (st.qkv && c->dp != c->d && cudaMemset(st.qkv, 0, (size_t)c->M * c->lq * 2) != cudaSuccess)
    return c->fail(AXONN_ERR_CUDA, "memset qkv padding");
  if (c->flash_attn())
    st.lse = (float*)c->dalloc((size_t)c->microbatch * c->heads * c->s * 4);
  else
    st.P = c->dalloc(att * 2);
  st.o = c->dalloc(Mh * 2);
  st.x1 = c->dalloc(Mh * 2);
  st.w = c->dalloc(Mh * 2);
  st.pre = c->dalloc(4 * Mh * 2);
  st.act = c->dalloc(4 * Mh * 2);
  st.out = c->dalloc(Mh * 2);
  st.mean1 = (float*)c->dalloc(c->M * 4);
  st.rstd1 = (float*)c->dalloc(c->M * 4);
  st.mean2 = (float*)c->dalloc(c->M * 4);
  st.rstd2 = (float*)c->dalloc(c->M * 4);
  if (!st.u || !st.qkv || !(st.P || st.lse) || !st.o || !st.x1 || !st.w || !st.pre || !st.act ||
      !st.out || !st.mean1 || !st.rstd1 || !st.mean2 || !st.rstd2)
    return c->fail(AXONN_ERR_OOM, "activation stash allocation");
  return 0;
}

static int plan_memory(Ctx* c) {
  const size_t Mh = (size_t)c->M * c->h;
  const size_t att = (size_t)c->microbatch * c->heads * c->s * c->s;
  if (c->ac > 1) {
    c->ck.resize(c->ac);
    for (LayerStash& st : c->ck)
      if (int r = alloc_stash(c, st)) return r;
  }
  c->slots.resize(c->limit);
  for (int si = 0; si < c->limit; ++si) {
    Slot& sl = c->slots[si];
    sl.in = c->dalloc(Mh * 2);
    if (c->ac > 1) {   // checkpointing: segment inputs only; the stash is the shared scratch
      sl.seg.assign(c->nl / c->ac + 1, nullptr);
      sl.seg[0] = sl.in;
      for (size_t j = 1; j < sl.seg.size(); ++j) {
        sl.seg[j] = c->dalloc(Mh * 2);
        if (!sl.seg[j]) return c->fail(AXONN_ERR_OOM, "checkpoint segment allocation");
      }
    } else {
      sl.L.resize(c->nl);
      for (int li = 0; li < c->nl; ++li)
        if (int r = alloc_stash(c, sl.L[li])) return r;
    }
    if (c->last) {
      sl.hf = c->dalloc(Mh * 2);
      sl.meanf = (float*)c->dalloc(c->M * 4);
      sl.rstdf = (float*)c->dalloc(c->M * 4);
    }
    if (!c->first) sl.gsend = c->dalloc(Mh * 2);
    if (!c->last) sl.grecv = c->dalloc(Mh * 2);
    if (!sl.in) return c->fail(AXONN_ERR_OOM, "slot allocation");
  }
  if (c->flash_attn()) {   // S, P, dS never materialised
    c->attn_D = (float*)c->dalloc((size_t)c->microbatch * c->heads * c->s * 4);
    if (!c->attn_D) return c->fail(AXONN_ERR_OOM, "attention workspace");
  } else {
    c->S = (float*)c->dalloc(att * 4);
    c->dS = c->dalloc(att * 2);
  }
  c->dh0 = c->dalloc(Mh * 2);
  c->dh1 = c->dalloc(Mh * 2);
  c->dqkv = c->dalloc(3 * Mh * 2);
  c->dpre = c->dalloc(4 * Mh * 2);
  c->dO = c->dalloc((size_t)c->M * c->heads * c->dp * 2);
  if (c->dO && cudaMemset(c->dO, 0, (size_t)c->M * c->heads * c->dp * 2) != cudaSuccess)
    return c->fail(AXONN_ERR_CUDA, "memset dO");
  c->du = c->dalloc(Mh * 2);
  c->dx1 = c->dalloc(Mh * 2);
  // column-sum workspaces (tickets + partials): one for the bias sums on s_wg, one for the
  // LayerNorm parameter sums on s_comp (the two streams run concurrently)
  // 4 KB of colsum2 tickets, then partials: colsum / colsum2, or ln_bwd_cs's [3][blocks][h]
  // (colsum_lnc needs [blocks][h]); all fp32
  const size_t cs_bytes = 4096 + std::max({(size_t)2 * colsum_chunks(c->M) * 4 * c->h * 4,
                                           (size_t)2 * ((c->M + 7) / 8 + 32) * c->h * 4,
                                           (size_t)3 * ln_bwd_cs_parts(c->M) * c->h * 4});
  c->cs_ws = (float*)c->dalloc(cs_bytes);
  c->cs_ws_ln = (float*)c->dalloc(cs_bytes);
  if (c->cs_ws && c->cs_ws_ln &&
      (cudaMemset(c->cs_ws, 0, 4096) != cudaSuccess || cudaMemset(c->cs_ws_ln, 0, 4096) != cudaSuccess))
    return c->fail(AXONN_ERR_CUDA, "memset colsum tickets");
  c->row_loss = (float*)c->dalloc(c->M * 4);
  c->d_loss = (double*)c->dalloc(64);
  if (c->last) c->logits = c->dalloc((size_t)c->M * c->V * 2);
  if ((!c->flash_attn() && (!c->S || !c->dS)) || !c->dh0 || !c->dh1 || !c->dqkv || !c->dpre || !c->dO || !c->du ||
      !c->dx1 || !c->cs_ws || !c->cs_ws_ln || !c->row_loss || !c->d_loss || (c->last && !c->logits))
    return c->fail(AXONN_ERR_OOM, "workspace allocation");
  if (cudaMallocHost(&c->h_loss, 64) != cudaSuccess) return c->fail(AXONN_ERR_OOM, "pinned loss");
  c->d_flag = reinterpret_cast<int*>(reinterpret_cast<char*>(c->d_loss) + 32);
  c->h_flag = reinterpret_cast<int*>(reinterpret_cast<char*>(c->h_loss) + 32);
  // parameters, gradients, optimizer state
  c->theta16 = c->dalloc(c->nflat * 2);
  c->grad32 = (float*)c->dalloc(std::max<int64_t>(c->n32, 64) * 4);
  c->grad16 = c->dalloc(c->nflat * 2);
  if (!c->theta16 || !c->grad32 || !c->grad16) return c->fail(AXONN_ERR_OOM, "parameter buffers");
  if (cudaMemsetAsync(c->theta16, 0, c->nflat * 2, c->s_comp) != cudaSuccess ||
      cudaMemsetAsync(c->grad32, 0, c->n32 * 4, c->s_comp) != cudaSuccess ||
      cudaMemsetAsync(c->grad16, 0, c->nflat * 2, c->s_comp) != cudaSuccess)
    return c->fail(AXONN_ERR_CUDA, "memset parameters");
  if (c->oc.offload) {
    for (float** p : {&c->master, &c->adam_m, &c->adam_v})
      if (cudaHostAlloc((void**)p, c->nflat * 4, cudaHostAllocPortable) != cudaSuccess)
        return c->fail(AXONN_ERR_OOM, "pinned host optimizer state");
    memset(c->adam_m, 0, c->nflat * 4);
    memset(c->adam_v, 0, c->nflat * 4);
    int64_t bs = c->oc.bucket_elems;
    if (bs > c->nflat) bs = c->nflat;
    for (int r = 0; r < 3; ++r)
      for (int a = 0; a < 3; ++a)
        if (!(c->ring[r][a] = (float*)c->dalloc(bs * 4))) return c->fail(AXONN_ERR_OOM, "offload ring");
  } else {
    c->master = (float*)c->dalloc(c->nflat * 4);
    c->adam_m = (float*)c->dalloc(c->nflat * 4);
    c->adam_v = (float*)c->dalloc(c->nflat * 4);
    if (!c->master || !c->adam_m || !c->adam_v) return c->fail(AXONN_ERR_OOM, "optimizer state");
    if (cudaMemsetAsync(c->master, 0, c->nflat * 4, c->s_comp) != cudaSuccess)
      return c->fail(AXONN_ERR_CUDA, "memset master");
    if (cudaMemsetAsync(c->adam_m, 0, c->nflat * 4, c->s_comp) != cudaSuccess ||
        cudaMemsetAsync(c->adam_v, 0, c->nflat * 4, c->s_comp) != cudaSuccess)
      return c->fail(AXONN_ERR_CUDA, "memset adam");
  }
  return 0;
}

}  // namespace axonn

using namespace axonn;

struct axonn_ctx : public Ctx {};

extern "C" {

AXONN_API int axonn_half_dtype(void) { return kHalfDtype; }

AXONN_API axonn_status axonn_get_unique_id(void* out128) {
  if (!out128) return AXONN_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return AXONN_ERR_NCCL;
  memcpy(out128, &id, sizeof(id));
  return AXONN_OK;
}

AXONN_API axonn_status axonn_stage_partition(const axonn_model_cfg* model, int g_inter,
                                              const double* stage_speed, int* bounds) {
  if (!model || !bounds || g_inter < 1 || model->n_layers < 1 || 2 * model->n_layers < g_inter ||
      model->hidden < 1 || model->seq_len < 1 || model->vocab < 1)
    return AXONN_ERR_INVALID_ARG;
  if (stage_speed)
    for (int i = 0; i < g_inter; ++i)
      if (!(stage_speed[i] > 0) || !std::isfinite(stage_speed[i])) return AXONN_ERR_INVALID_ARG;
  const std::vector<int> bb = balanced_blocks(model, g_inter, stage_speed);
  for (int i = 0; i <= g_inter; ++i) bounds[i] = bb[i];
  return AXONN_OK;
}

AXONN_API axonn_status axonn_init(int g_inter, int g_data, int microbatch,
                                  const axonn_model_cfg* model, const axonn_opt_cfg* opt,
                                  const axonn_dist* dist, axonn_ctx** out) {
  if (!out) return AXONN_ERR_INVALID_ARG;
  *out = nullptr;
  if (!model || !opt || g_inter < 1 || g_data < 1 || microbatch < 1) return AXONN_ERR_INVALID_ARG;
  if (model->dtype != kHalfDtype) return AXONN_ERR_INVALID_ARG;   // other format: other library
  const int world = dist ? dist->world_size : 1;
  const int rank = dist ? dist->world_rank : 0;
  if (world != g_inter * g_data) return AXONN_ERR_GRID_MISMATCH;
  if (rank < 0 || rank >= world) return AXONN_ERR_INVALID_ARG;
  if (model->n_layers < 1 || (!opt->stage_balance && model->n_layers % g_inter) ||
      2 * model->n_layers < g_inter)
    return AXONN_ERR_NONDIVISIBLE_LAYERS;
  if (opt->stage_balance && opt->checkpoint_interval != 0 && opt->checkpoint_interval != 1)
    return AXONN_ERR_INVALID_ARG;   // checkpoint segments are whole layers
  if (opt->stage_balance && opt->stage_speed)
    for (int i = 0; i < g_inter; ++i)
      if (!(opt->stage_speed[i] > 0) || !std::isfinite(opt->stage_speed[i])) return AXONN_ERR_INVALID_ARG;
  if (model->hidden < 8 || model->heads < 1 || model->hidden % model->heads ||
      model->hidden % 8 || model->seq_len < 8 || model->seq_len % 8 || model->vocab < 2 ||
      model->vocab % 8)
    return AXONN_ERR_INVALID_ARG;
  const int d = model->hidden / model->heads;
  if (d < 2) return AXONN_ERR_INVALID_ARG;
  if (!(opt->lr >= 0) || !(opt->beta1 >= 0 && opt->beta1 < 1) || !(opt->beta2 >= 0 && opt->beta2 < 1) ||
      !(opt->eps > 0) || !(opt->loss_scale > 0) || opt->bucket_elems < 1 || opt->coarsen_k < 1 ||
      opt->pipeline_limit < 0)
    return AXONN_ERR_INVALID_ARG;
  axonn_local_group* lg = (dist && world > 1) ? dist->local_group : nullptr;
  // loopback: no NCCL, so G_data > 1 needs the fused column reduction (bf16 build, <= 8 replicas)
  if (lg && (lg->size != world || (g_data > 1 && (kHalfDtype != AXONN_BF16 || g_data > kMaxReplicas))))
    return AXONN_ERR_INVALID_ARG;
  if (world > 1 && !lg && !dist->nccl_id) return AXONN_ERR_INVALID_ARG;
  if (opt->checkpoint_interval < -1 ||   // BadCheckpointInterval: ac must divide N / G_inter
      (opt->checkpoint_interval > 1 && (model->n_layers / g_inter) % opt->checkpoint_interval))
    return AXONN_ERR_INVALID_ARG;
  if (opt->grad_accum_fp32 != 0 && opt->grad_accum_fp32 != 1) return AXONN_ERR_INVALID_ARG;

  axonn_ctx* c = new (std::nothrow) axonn_ctx();
  if (!c) return AXONN_ERR_OOM;
  c->g_inter = g_inter; c->g_data = g_data; c->microbatch = microbatch;
  c->mc = *model; c->oc = *opt;
  c->half_accum = opt->grad_accum_fp32 == 0;
  if (c->oc.bucket_elems % 4) c->oc.bucket_elems += 4 - c->oc.bucket_elems % 4;   // 16-B aligned buckets
  c->rank = rank; c->world = world; c->device = dist ? dist->device : 0;
  c->lg = lg;
  {
    const char* e = getenv("AXONN_DP");   // must agree on all ranks (same launcher env)
    c->dp_fused = g_data > 1 && g_data <= kMaxReplicas && kHalfDtype == AXONN_BF16 &&
                  (lg || !(e && strcmp(e, "nccl") == 0));
  }
  c->stage = rank % g_inter;            // world_rank = j * G_inter + i (D-29)
  c->replica = rank / g_inter;
  c->first = c->stage == 0;
  c->last = c->stage == g_inter - 1;
  if (opt->stage_balance) {
    const std::vector<int> bb = balanced_blocks(model, g_inter, opt->stage_speed);
    const int b0 = bb[c->stage], b1 = bb[c->stage + 1];            // blocks [b0, b1)
    c->layer0 = b0 / 2;
    c->nl = (b1 + 1) / 2 - b0 / 2;
    for (int li = 0; li < c->nl; ++li) {
      const int L = c->layer0 + li;
      c->lhalf.push_back(((2 * L >= b0 && 2 * L < b1) ? 1 : 0) | ((2 * L + 1 >= b0 && 2 * L + 1 < b1) ? 2 : 0));
    }
  } else {
    c->nl = model->n_layers / g_inter;
    c->layer0 = c->stage * c->nl;
    c->lhalf.assign(c->nl, 3);
  }
  c->h = model->hidden; c->heads = model->heads; c->d = d; c->s = model->seq_len;
  c->V = model->vocab; c->M = microbatch * model->seq_len;
  c->dp = (d + 7) / 8 * 8;            // e.g. 12B: d = 188 -> 192 (D-7: scale stays 1/sqrt(188))
  c->lq = 3LL * c->heads * c->dp;
  c->limit = g_inter == 1 ? 1 : (opt->pipeline_limit > 0 ? opt->pipeline_limit : g_inter);
  {
    const char* e = getenv("AXONN_P2P");   // nccl | copy | (default) direct; same on all ranks
    c->p2p_ipc = !(e && strcmp(e, "nccl") == 0);
    c->direct_send = c->p2p_ipc && !(e && strcmp(e, "copy") == 0);
  }
  if (opt->checkpoint_interval == -1) {   // factor of N / G_inter closest to sqrt(N)
    const double root = std::sqrt((double)model->n_layers);
    int best = 1;
    for (int a = 1; a <= c->nl; ++a)
      if (c->nl % a == 0 && (std::fabs(a - root) < std::fabs(best - root))) best = a;
    c->ac = best;
  } else if (opt->checkpoint_interval > 1) {
    c->ac = opt->checkpoint_interval;
  }
  if (c->ac > 1) c->direct_send = false;   // the message is a checkpoint segment boundary

  auto bail = [&](int rc) {
    if (c->lg) c->lg->abort();   // the other loopback stages must not wait for this one
    axonn_free(c);
    return (axonn_status)rc;
  };
  int rc = c->check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
  if (rc) return bail(rc);
  cudaDeviceProp prop;
  if ((rc = c->check_cuda(cudaGetDeviceProperties(&prop, c->device), "props"))) return bail(rc);
  if (prop.major < 10) return bail(c->fail(AXONN_ERR_CUDA, "needs an sm_100a (B200) device"));
  c->num_sms = prop.multiProcessorCount;
  // CUDA lazy loading would load a kernel's module at its first launch and wait for the
  // device's running kernels — including a pre-posted ncclRecv spinning until the peer
  // sends, which the peer only does after our launch: load everything now.
  {
    std::unique_lock<std::mutex> lk;
    if (c->lg) lk = std::unique_lock<std::mutex>(c->lg->preload_mu);
    if (preload_gemm() || preload_ops() || preload_adamw() || preload_attn())
      return bail(c->fail(AXONN_ERR_CUDA, "kernel preload failed"));
  }
  for (cudaStream_t* st : {&c->s_comp, &c->s_send_act, &c->s_send_grad, &c->s_recv_act,
                           &c->s_recv_grad, &c->s_dp, &c->s_h2d, &c->s_d2h, &c->s_opt, &c->s_wg,
                           &c->s_loss})
    if ((rc = c->check_cuda(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking), "stream")))
      return bail(rc);
  for (cudaEvent_t* e : {&c->ev_grads_ready, &c->ev_opt_done, &c->ev_loss})
    if ((rc = c->check_cuda(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event"))) return bail(rc);
  for (int r = 0; r < 3; ++r)
    for (cudaEvent_t* e : {&c->ev_h2d[r], &c->ev_adam[r], &c->ev_d2h[r]})
      if ((rc = c->check_cuda(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event"))) return bail(rc);

  build_tensors(c);
  c->grad_written.assign(c->tensors.size(), 0);
  if ((rc = plan_memory(c))) return bail(rc);
  if ((rc = init_weights(c))) return bail(rc);

  // NCCL: world, column (all-reduce) and per-direction neighbour links (2-rank comms).
  if (world > 1 && !c->lg) {
    ncclUniqueId id;
    memcpy(&id, dist->nccl_id, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if ((rc = c->check_nccl(ncclCommInitRankConfig(&c->world_comm, world, id, rank, &cfg),
                            "ncclCommInitRank")))
      return bail(rc);
    c->owned_comms.push_back(c->world_comm);
    // column comm capped at 16 CTAs, and those SMs left free by the GEMMs of the last
    // backward while its all-reduce chunks run (1.3B 1x2: 936.8 vs 931.9 uncapped, 921.4 at 8)
    c->dp_ctas = 16;
    if ((rc = split_comm(c, c->world_comm, g_data > 1 ? c->stage : NCCL_SPLIT_NOCOLOR, c->replica,
                         &c->dp_comm, c->dp_ctas)))
      return bail(rc);
    // links between stage k and k+1 of row j; even and odd boundaries in separate splits so
    // that every rank joins at most one comm per split.  P2P comms capped at 4 CTAs.
    for (int dir = 0; dir < 2; ++dir) {
      for (int parity = 0; parity < 2; ++parity) {
        int color = NCCL_SPLIT_NOCOLOR;
        int k_lo = c->stage, k_hi = c->stage - 1;   // boundary to the right / left of this stage
        int kb = -1;
        if (g_inter > 1) {
          if (k_lo % 2 == parity && k_lo < g_inter - 1) kb = k_lo;
          else if (k_hi >= 0 && k_hi % 2 == parity) kb = k_hi;
        }
        if (kb >= 0) color = c->replica * g_inter + kb;
        ncclComm_t nc = nullptr;
        if ((rc = split_comm(c, c->world_comm, color, c->stage, &nc, 1))) return bail(rc);
        if (kb < 0) continue;
        bool right = (kb == c->stage);   // comm with stage+1
        if (dir == 0) {
          if (right) c->act_out = nc; else c->act_in = nc;
        } else {
          if (right) c->grad_in = nc; else c->grad_out = nc;
        }
      }
    }
  }
  // NCCL connects P2P peers lazily and the first call on a link blocks on the host until
  // the peer also reaches it; in Alg. 2 the peer only does so after a message arrives, so
  // connect every link now, in ascending boundary order (no cycle: rank i finishes
  // boundary i-1 before boundary i).
  if (world > 1 && g_inter > 1 && !c->lg) {
    void* tmp = c->dalloc(256);
    if (!tmp) return bail(c->fail(AXONN_ERR_OOM, "link warm-up buffer"));
    for (int k = 0; k < g_inter - 1; ++k) {
      if (k == c->stage - 1) {   // boundary (i-1, i): receive activation, send gradient
        if ((rc = c->check_nccl(ncclRecv(tmp, 8, kNcclHalf, 0, c->act_in, c->s_comp), "warm recv")) ||
            (rc = c->check_cuda(cudaStreamSynchronize(c->s_comp), "warm sync")) ||
            (rc = c->check_nccl(ncclSend(tmp, 8, kNcclHalf, 0, c->grad_out, c->s_comp), "warm send")) ||
            (rc = c->check_cuda(cudaStreamSynchronize(c->s_comp), "warm sync")))
          return bail(rc);
      } else if (k == c->stage) {   // boundary (i, i+1): send activation, receive gradient
        if ((rc = c->check_nccl(ncclSend(tmp, 8, kNcclHalf, 1, c->act_out, c->s_comp), "warm send")) ||
            (rc = c->check_cuda(cudaStreamSynchronize(c->s_comp), "warm sync")) ||
            (rc = c->check_nccl(ncclRecv(tmp, 8, kNcclHalf, 1, c->grad_in, c->s_comp), "warm recv")) ||
            (rc = c->check_cuda(cudaStreamSynchronize(c->s_comp), "warm sync")))
          return bail(rc);
      }
    }
  }
  if (c->lg) {
    if (!c->p2p_ipc) c->direct_send = false;   // AXONN_P2P=nccl: the loopback copies
    c->p2p_ipc = 1;   // the loopback runs the peer-copy link protocol
    if ((rc = local_links(c))) return bail(rc);
  } else {
    if (world > 1 && g_inter > 1 && c->p2p_ipc && (rc = ipc_links(c))) return bail(rc);
    if (c->dp_fused && (rc = dp_links(c))) return bail(rc);
  }
  c->n_chunks = (c->nflat + chunk_elems(c) - 1) / chunk_elems(c);
  if ((rc = c->check_cuda(cudaStreamSynchronize(c->s_comp), "init sync"))) return bail(rc);
  *out = c;
  return AXONN_OK;
}

AXONN_API void axonn_free(axonn_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (ncclComm_t nc : c->owned_comms) {
    if (c->sticky) ncclCommAbort(nc);
    else ncclCommDestroy(nc);
  }
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->allocs) cudaFree(p);
  if (c->oc.offload) {
    if (c->master) cudaFreeHost(c->master);
    if (c->adam_m) cudaFreeHost(c->adam_m);
    if (c->adam_v) cudaFreeHost(c->adam_v);
  }
  if (c->h_loss) cudaFreeHost(c->h_loss);
  if (c->flags_host) cudaFreeHost((void*)c->flags_host);
  if (c->dp_flags_host) cudaFreeHost((void*)c->dp_flags_host);
  if (c->dtok) cudaFree(c->dtok);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_pool_opt) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_bucket) cudaEventDestroy(e);
  for (auto& row : c->ph)
    for (cudaEvent_t e : row)
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->timer)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_grads_ready, c->ev_opt_done, c->ev_loss})
    if (e) cudaEventDestroy(e);
  for (int r = 0; r < 3; ++r)
    for (cudaEvent_t e : {c->ev_h2d[r], c->ev_adam[r], c->ev_d2h[r]})
      if (e) cudaEventDestroy(e);
  for (cudaStream_t st : {c->s_comp, c->s_send_act, c->s_send_grad, c->s_recv_act, c->s_recv_grad,
                          c->s_dp, c->s_h2d, c->s_d2h, c->s_opt, c->s_wg, c->s_loss})
    if (st) cudaStreamDestroy(st);
  delete c;
}

AXONN_API const char* axonn_last_error(const axonn_ctx* c) {
  if (!c) return "null context";
  return c->err.c_str();
}

AXONN_API int axonn_num_tensors(const axonn_ctx* c) { return c ? (int)c->tensors.size() : -1; }

AXONN_API axonn_status axonn_tensor_info(const axonn_ctx* c, int idx, char name[64],
                                         int64_t shape[2], int64_t* numel) {
  if (!c || idx < 0 || idx >= (int)c->tensors.size()) return AXONN_ERR_INVALID_ARG;
  const TensorRec& t = c->tensors[idx];
  if (name) {
    strncpy(name, t.name.c_str(), 63);
    name[63] = 0;
  }
  if (shape) {
    shape[0] = t.rows;
    shape[1] = t.cols;
  }
  if (numel) *numel = t.numel;
  return AXONN_OK;
}

AXONN_API axonn_status axonn_read_tensor(axonn_ctx* c, int which, int idx, float* dst) {
  if (!c || !dst || idx < 0 || idx >= (int)c->tensors.size()) return AXONN_ERR_INVALID_ARG;
  if (c->sticky) return AXONN_ERR_STATE;
  CU(cudaSetDevice(c->device));
  CU(cudaDeviceSynchronize());
  const TensorRec& t = c->tensors[idx];
  switch (which) {
    case AXONN_T_PARAM16:
    case AXONN_T_GRAD: {
      std::vector<uint16_t> tmp(t.numel);
      const char* base = static_cast<const char*>(which == AXONN_T_PARAM16 ? c->theta16 : c->grad16);
      CU(cudaMemcpy(tmp.data(), base + t.off * 2, t.numel * 2, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < t.numel; ++i) dst[i] = h162f(tmp[i]);
      return AXONN_OK;
    }
    case AXONN_T_GRAD32:
      if (t.off32 < 0) return AXONN_ERR_INVALID_ARG;   // grad_accum_fp32 = 0: accumulates in half
      CU(cudaMemcpy(dst, c->grad32 + t.off32, t.numel * 4, cudaMemcpyDeviceToHost));
      return AXONN_OK;
    case AXONN_T_MASTER:
    case AXONN_T_ADAM_M:
    case AXONN_T_ADAM_V: {
      const float* src = which == AXONN_T_MASTER ? c->master : which == AXONN_T_ADAM_M ? c->adam_m : c->adam_v;
      if (c->oc.offload) memcpy(dst, src + t.off, t.numel * 4);
      else CU(cudaMemcpy(dst, src + t.off, t.numel * 4, cudaMemcpyDeviceToHost));
      return AXONN_OK;
    }
  }
  return AXONN_ERR_INVALID_ARG;
}

AXONN_API axonn_status axonn_write_tensor(axonn_ctx* c, int which, int idx, const float* src) {
  if (!c || !src || idx < 0 || idx >= (int)c->tensors.size()) return AXONN_ERR_INVALID_ARG;
  if (c->sticky) return AXONN_ERR_STATE;
  CU(cudaSetDevice(c->device));
  CU(cudaDeviceSynchronize());
  const TensorRec& t = c->tensors[idx];
  std::vector<uint16_t> tmp;
  auto put16 = [&](void* base) -> int {
    tmp.resize(t.numel);
    for (int64_t i = 0; i < t.numel; ++i) tmp[i] = f2h16(src[i]);
    return c->check_cuda(cudaMemcpy(static_cast<char*>(base) + t.off * 2, tmp.data(), t.numel * 2,
                                    cudaMemcpyHostToDevice), "write16");
  };
  int rc = 0;
  switch (which) {
    case AXONN_T_PARAM16:
      rc = put16(c->theta16);
      break;
    case AXONN_T_GRAD:
      rc = put16(c->grad16);
      c->grad_written[idx] = 1;
      {
        bool all = true;
        for (char w : c->grad_written) all = all && w;
        if (all) {
          c->grads_ready = true;
          c->ev_chunk.clear();
          std::fill(c->grad_written.begin(), c->grad_written.end(), 0);
        }
      }
      break;
    case AXONN_T_GRAD32:
      if (t.off32 < 0) return AXONN_ERR_INVALID_ARG;
      rc = c->check_cuda(cudaMemcpy(c->grad32 + t.off32, src, t.numel * 4, cudaMemcpyHostToDevice), "write32");
      break;
    case AXONN_T_MASTER:
    case AXONN_T_ADAM_M:
    case AXONN_T_ADAM_V: {
      float* dstp = which == AXONN_T_MASTER ? c->master : which == AXONN_T_ADAM_M ? c->adam_m : c->adam_v;
      if (c->oc.offload) memcpy(dstp + t.off, src, t.numel * 4);
      else rc = c->check_cuda(cudaMemcpy(dstp + t.off, src, t.numel * 4, cudaMemcpyHostToDevice), "write32");
      if (!rc && which == AXONN_T_MASTER) rc = put16(c->theta16);   // theta16 = RNE(theta32)
      break;
    }
    default:
      return AXONN_ERR_INVALID_ARG;
  }
  return (axonn_status)rc;
}

AXONN_API axonn_status axonn_timer_mark(axonn_ctx* c, int id) {
  if (!c || id < 0 || id >= 8) return AXONN_ERR_INVALID_ARG;
  CU(cudaSetDevice(c->device));
  if (!c->timer[id]) CU(cudaEventCreate(&c->timer[id]));
  CU(cudaStreamWaitEvent(c->s_comp, c->ev_opt_done, 0));
  cudaEvent_t e = c->ev();
  CU(cudaEventRecord(e, c->s_dp));
  CU(cudaStreamWaitEvent(c->s_comp, e, 0));
  CU(cudaEventRecord(c->timer[id], c->s_comp));
  return AXONN_OK;
}

AXONN_API axonn_status axonn_timer_elapsed(axonn_ctx* c, int a, int b, double* ms) {
  if (!c || !ms || a < 0 || a >= 8 || b < 0 || b >= 8 || !c->timer[a] || !c->timer[b])
    return AXONN_ERR_INVALID_ARG;
  CU(cudaSetDevice(c->device));
  CU(cudaEventSynchronize(c->timer[b]));
  float f = 0;
  CU(cudaEventElapsedTime(&f, c->timer[a], c->timer[b]));
  *ms = f;
  return AXONN_OK;
}

AXONN_API int axonn_profile_json(const axonn_ctx* c, char* buf, int n) {
  if (!c) return -1;
  const int len = (int)c->prof_json.size();
  if (buf && n > 0) {
    int k = len < n - 1 ? len : n - 1;
    memcpy(buf, c->prof_json.data(), k);
    buf[k] = 0;
  }
  return len;
}

AXONN_API axonn_status axonn_set_profiling(axonn_ctx* c, int on) {
  if (!c) return AXONN_ERR_INVALID_ARG;
  c->profiling = on != 0;
  return AXONN_OK;
}

AXONN_API axonn_status axonn_local_group_create(int size, axonn_local_group** out) {
  if (!out) return AXONN_ERR_INVALID_ARG;
  *out = nullptr;
  if (size < 1) return AXONN_ERR_INVALID_ARG;
  axonn_local_group* g = new (std::nothrow) axonn_local_group();
  if (!g) return AXONN_ERR_OOM;
  g->size = size;
  g->reg.resize(size);
  *out = g;
  return AXONN_OK;
}

AXONN_API void axonn_local_group_free(axonn_local_group* g) { delete g; }

AXONN_API int axonn_checkpoint_interval(const axonn_ctx* c) { return c ? c->ac : -1; }

AXONN_API axonn_status axonn_stats(const axonn_ctx* c, double* out, int n) {
  if (!c || !out || n < 0) return AXONN_ERR_INVALID_ARG;
  for (int i = 0; i < n && i < AXONN_STAT_COUNT; ++i) out[i] = c->stats[i];
  for (int i = AXONN_STAT_COUNT; i < n; ++i) out[i] = 0;
  return AXONN_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ Alg. 2 + Alg. 1
namespace axonn {

// Column flag words of the fused reduction (reading D-35).  A stream waits (cuStreamWaitValue32,
// cyclic >=) for every peer's word base + j; the loopback's host thread observes its
// host-mapped words instead (no kernel or stream of one device waits on another context).
int Ctx::dp_wait(cudaStream_t st, int base, uint32_t value) {
  for (int j = 0; j < g_data; ++j) {
    if (j == replica) continue;
    if (dp_flags_host) {
      const auto t0 = std::chrono::steady_clock::now();
      while ((int32_t)(dp_flags_host[base + j] - value) < 0) {
        if (lg && lg->failed) return fail(AXONN_ERR_STATE, "local group failed (column flags)");
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > group_timeout_s())
          return fail(AXONN_ERR_TIMEOUT, "fused column reduction: peer flag never arrived");
        std::this_thread::yield();
      }
    }
    // the stream wait (production; after the host spin of the loopback it is satisfied at once)
    // orders the stream's later reads of the peer's buffer after the peer's writes
    if (int rc = wait_flag(this, st, dp_flags + base + j, value, true)) return rc;
  }
  return 0;
}
int Ctx::dp_signal(cudaStream_t st, int slot, uint32_t value) {
  for (int k = 0; k < g_data; ++k)
    if (k != replica)
      if (int rc = write_flag(this, st, dp_peer_flags[k] + slot, value)) return rc;
  return 0;
}

// Alg. 2 on this rank for microbatches 0..m-1.
int Ctx::ar_ready(int64_t lo) {
  if (lo >= ar_hi) return 0;
  cudaEvent_t a = ev(), b = ev();
  int rc;
  if ((rc = check_cuda(cudaEventRecord(a, s_comp), "ar ev")) || (rc = check_cuda(cudaEventRecord(b, s_wg), "ar ev")) ||
      (rc = check_cuda(cudaStreamWaitEvent(s_dp, a, 0), "ar wait")) ||
      (rc = check_cuda(cudaStreamWaitEvent(s_dp, b, 0), "ar wait")))
    return rc;
  if (!ar_active && opt_pending &&   // grad16 is read by the still-running optimizer step
      (rc = check_cuda(cudaStreamWaitEvent(s_dp, ev_opt_done, 0), "ar wait opt")))
    return rc;
  // fused column reduction: the peers' K9 of the previous batch read this grad16
  if (!ar_active && dp_fused && dp_epoch > 1 && (rc = dp_wait(s_dp, g_data, dp_epoch - 1))) return rc;
  ar_active = true;
  if ((rc = cast_grads(lo, ar_hi, s_dp))) return rc;
  ar_hi = lo;
  const int64_t ch = (int64_t)oc.coarsen_k * oc.bucket_elems;
  while (ar_next_chunk >= 0 && ar_next_chunk * ch >= lo) {
    const int64_t c0 = ar_next_chunk * ch, n = std::min(ch, nflat - c0);
    if (dp_fused) {     // Alg. 1 l.13 fused into every replica's K9: tell the peers
      if ((rc = dp_signal(s_dp, replica, dp_progress(ar_next_chunk)))) return rc;
      stats[AXONN_STAT_ALLREDUCE_BYTES] += n * 2.0 * (g_data - 1);   // read by the peers' K9
    } else if (g_data > 1) {   // Alg. 1 l.13: SUM over the column (pre-divided loss, D-10)
      if ((rc = check_nccl(ncclAllReduce(static_cast<char*>(grad16) + c0 * 2, static_cast<char*>(grad16) + c0 * 2,
                                         n, kNcclHalf, ncclSum, dp_comm, s_dp), "ncclAllReduce")))
        return rc;
      stats[AXONN_STAT_ALLREDUCE_BYTES] += n * 2.0;
    }
    cudaEvent_t e = ev();
    if ((rc = check_cuda(cudaEventRecord(e, s_dp), "ar ev"))) return rc;
    ev_chunk[ar_next_chunk] = e;
    --ar_next_chunk;
  }
  return 0;
}

static int run_pipeline(Ctx* c, int m) {
  const size_t Mh = (size_t)c->M * c->h;
  const int P = c->g_inter, L = c->limit;
  int rc;
  if (P == 1) {   // D-18: F, loss, B per microbatch; no messages
    for (int mb = 0; mb < m; ++mb) {
      Slot& sl = c->slots[0];
      if ((rc = c->forward(sl, mb))) return rc;
      if ((rc = c->backward(sl, mb, nullptr))) return rc;
    }
    return 0;
  }
  // In 2-rank link comms the lower stage is rank 0: act_out/grad_in peer = 1, act_in/grad_out peer = 0.
  std::vector<cudaEvent_t> ev_act(m, nullptr), ev_grad(m, nullptr), ev_sent_grad(m, nullptr),
      ev_sent_act(m, nullptr), ev_bdone(m, nullptr);
  int next_act_post = 0, next_grad_post = 0;   // next microbatch whose receive is posted
  int next_act = 0, next_grad = 0;             // next microbatch expected on each link (FIFO)
  int done_b = 0;                              // backwards completed on this stage
  int popped = 0;                              // stage 0 injections
  auto slot_of = [&](int mb) -> Slot& { return c->slots[mb % L]; };
  // message sequence number (peer-copy links): unique over the context's lifetime, so a flag
  // left from an earlier batch never matches; every stage counts the same microbatches
  const uint32_t base = c->msg_base;
  auto seq = [&](int mb) -> uint32_t { return base + (uint32_t)mb + 1u; };
  c->msg_base += (uint32_t)m;
  auto post = [&]() -> int {
    // pre-post receives into free slots, in microbatch order
    while (!c->first && next_act_post < m && next_act_post < done_b + L) {
      int mb = next_act_post++;
      if (c->flags_host) continue;   // loopback: the host thread observes the flag (landed())
      ev_act[mb] = c->ev();
      // the slot's previous occupant (mb - L) must have finished its backward on the GPU
      if (mb >= L) cudaStreamWaitEvent(c->s_recv_act, ev_bdone[mb - L], 0);
      int r = c->p2p_ipc ? wait_flag(c, c->s_recv_act, c->flags + mb % L, seq(mb))
                         : c->check_nccl(ncclRecv(slot_of(mb).in, Mh, kNcclHalf, 0, c->act_in, c->s_recv_act),
                                         "ncclRecv act");
      if (r) return r;
      if ((r = c->check_cuda(cudaEventRecord(ev_act[mb], c->s_recv_act), "rec"))) return r;
      c->msg_ev.emplace_back(2 * mb, ev_act[mb]);
    }
    while (!c->last && next_grad_post < m && next_grad_post < done_b + L) {
      int mb = next_grad_post++;
      if (c->flags_host) continue;
      ev_grad[mb] = c->ev();
      if (mb >= L) cudaStreamWaitEvent(c->s_recv_grad, ev_bdone[mb - L], 0);
      int r = c->p2p_ipc ? wait_flag(c, c->s_recv_grad, c->flags + L + mb % L, seq(mb))
                         : c->check_nccl(ncclRecv(slot_of(mb).grecv, Mh, kNcclHalf, 1, c->grad_in,
                                                  c->s_recv_grad), "ncclRecv grad");
      if (r) return r;
      if ((r = c->check_cuda(cudaEventRecord(ev_grad[mb], c->s_recv_grad), "rec"))) return r;
      c->msg_ev.emplace_back(2 * mb + 1, ev_grad[mb]);
    }
    return 0;
  };
  auto send_act = [&](int mb) -> int {
    Slot& sl = slot_of(mb);
    cudaEvent_t e = c->ev();
    cudaEventRecord(e, c->s_comp);
    cudaStreamWaitEvent(c->s_send_act, e, 0);
    const void* out = c->stage_out(sl);
    c->stats[AXONN_STAT_P2P_BYTES] += (double)Mh * 2;
    int r;
    if (c->direct_send) {   // the forward already stored into stage+1's slot: just the flag
      r = write_flag(c, c->s_comp, c->peer_flags_next + mb % L, seq(mb));
      ev_sent_act[mb] = c->ev();
      cudaEventRecord(ev_sent_act[mb], c->s_comp);
      return r;
    }
    if (c->p2p_ipc) {   // copy engine over NVLink into stage+1's slot, then its flag
      r = c->check_cuda(cudaMemcpyAsync(c->peer_act[mb % L], out, Mh * 2, cudaMemcpyDeviceToDevice,
                                        c->s_send_act), "peer copy act");
      if (!r) r = write_flag(c, c->s_send_act, c->peer_flags_next + mb % L, seq(mb));
    } else {
      r = c->check_nccl(ncclSend(out, Mh, kNcclHalf, 1, c->act_out, c->s_send_act), "ncclSend act");
    }
    ev_sent_act[mb] = c->ev();
    cudaEventRecord(ev_sent_act[mb], c->s_send_act);
    return r;
  };
  auto send_grad = [&](int mb) -> int {
    Slot& sl = slot_of(mb);
    cudaEvent_t e = c->ev();
    cudaEventRecord(e, c->s_comp);
    cudaStreamWaitEvent(c->s_send_grad, e, 0);
    c->stats[AXONN_STAT_P2P_BYTES] += (double)Mh * 2;
    int r;
    if (c->direct_send) {   // the backward already stored into stage-1's slot: just the flag
      r = write_flag(c, c->s_comp, c->peer_flags_prev + L + mb % L, seq(mb));
      ev_sent_grad[mb] = c->ev();
      cudaEventRecord(ev_sent_grad[mb], c->s_comp);
      return r;
    }
    if (c->p2p_ipc) {
      r = c->check_cuda(cudaMemcpyAsync(c->peer_grad[mb % L], sl.gsend, Mh * 2, cudaMemcpyDeviceToDevice,
                                        c->s_send_grad), "peer copy grad");
      if (!r) r = write_flag(c, c->s_send_grad, c->peer_flags_prev + L + mb % L, seq(mb));
    } else {
      r = c->check_nccl(ncclSend(sl.gsend, Mh, kNcclHalf, 0, c->grad_out, c->s_send_grad), "ncclSend grad");
    }
    ev_sent_grad[mb] = c->ev();
    cudaEventRecord(ev_sent_grad[mb], c->s_send_grad);
    return r;
  };
  auto forward_of = [&](int mb) -> int {   // Forward (+ Backward(1) and grad send on the last stage)
    Slot& sl = slot_of(mb);
    sl.mb = mb;
    if (!c->first && ev_act[mb]) cudaStreamWaitEvent(c->s_comp, ev_act[mb], 0);
    // loopback: the host has seen the flag; the same stream wait as production (satisfied at
    // once, so it cannot block a shared hardware queue) orders this stream's reads of the slot
    // after the copy for the GPU's memory model (generic loads must not hit stale L1 lines)
    if (!c->first && c->flags_host) {
      const int r = wait_flag(c, c->s_comp, c->flags + mb % L, seq(mb));
      if (r) return r;
    }
    // a slot's gradient-out buffer is reused only after its previous send finished
    if (!c->first && mb >= L && ev_sent_grad[mb - L]) cudaStreamWaitEvent(c->s_comp, ev_sent_grad[mb - L], 0);
    if (!c->last && mb >= L && ev_sent_act[mb - L]) cudaStreamWaitEvent(c->s_comp, ev_sent_act[mb - L], 0);
    int r = c->forward(sl, mb);
    if (r) return r;
    if (c->last) {
      if ((r = c->backward(sl, mb, nullptr))) return r;
      ev_bdone[mb] = c->ev();
      cudaEventRecord(ev_bdone[mb], c->s_comp);
      ++done_b;
      return send_grad(mb);
    }
    return send_act(mb);
  };
  auto backward_of = [&](int mb) -> int {
    Slot& sl = slot_of(mb);
    if (ev_grad[mb]) cudaStreamWaitEvent(c->s_comp, ev_grad[mb], 0);
    if (c->flags_host) {   // see forward_of
      const int r0 = wait_flag(c, c->s_comp, c->flags + L + mb % L, seq(mb));
      if (r0) return r0;
    }
    int r = c->backward(sl, mb, sl.grecv);
    if (r) return r;
    ev_bdone[mb] = c->ev();
    cudaEventRecord(ev_bdone[mb], c->s_comp);
    ++done_b;
    if (!c->first) return send_grad(mb);
    if (popped < m) {   // Alg. 2 l.24-26: inject the next microbatch
      int nxt = popped++;
      return forward_of(nxt);
    }
    return 0;
  };

  if ((rc = post())) return rc;
  if (c->first) {   // Alg. 2 l.3-9: warm-up
    int n = L < m ? L : m;
    for (int k = 0; k < n; ++k) {
      int mb = popped++;
      if ((rc = forward_of(mb))) return rc;
    }
  }
  auto t_last = std::chrono::steady_clock::now();
  const char* wd_env = getenv("AXONN_WATCHDOG_S");   // no message progress -> AXONN_ERR_TIMEOUT
  const double watchdog_s = wd_env ? atof(wd_env) : 600.0;
  int fwd_done = c->first ? popped : 0;
  while (true) {
    bool need_act = !c->first && next_act < m;
    bool need_grad = !c->last && next_grad < m;
    if (!need_act && !need_grad) break;
    if ((rc = post())) return rc;
    // a message has landed: its receive event completed, or (loopback) the flag word of its
    // slot holds its sequence number (the store is ordered after the copy into the slot)
    auto landed = [&](bool grad, int mb) -> bool {
      if (c->flags_host) return c->flags_host[(grad ? L : 0) + mb % L] == seq(mb);
      return cudaEventQuery(grad ? ev_grad[mb] : ev_act[mb]) == cudaSuccess;
    };
    bool grad_landed = need_grad && next_grad < next_grad_post && landed(true, next_grad);
    bool act_landed = !grad_landed && need_act && next_act < next_act_post && landed(false, next_act);
    if (grad_landed) {   // backward-first among landed messages (D-19)
      int mb = next_grad++;
      if ((rc = backward_of(mb))) return rc;
      t_last = std::chrono::steady_clock::now();
    } else if (act_landed) {
      int mb = next_act++;
      ++fwd_done;
      if ((rc = forward_of(mb))) return rc;
      t_last = std::chrono::steady_clock::now();
    } else {
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t_last).count() > watchdog_s) {
        auto busy = [](cudaStream_t st) { return cudaStreamQuery(st) == cudaErrorNotReady ? "busy" : "idle"; };
        char buf[512];
        snprintf(buf, sizeof(buf),
                 "Alg. 2 watchdog: no message landed for %d s (stage %d): posted act %d grad %d, "
                 "consumed act %d grad %d, backwards %d, injected %d; streams comp %s send_act %s "
                 "send_grad %s recv_act %s recv_grad %s",
                 (int)watchdog_s, c->stage, next_act_post, next_grad_post, next_act, next_grad,
                 done_b, popped, busy(c->s_comp), busy(c->s_send_act), busy(c->s_send_grad),
                 busy(c->s_recv_act), busy(c->s_recv_grad));
        fprintf(stderr, "[axonn rank %d] %s\n", c->rank, buf);
        return c->fail(AXONN_ERR_TIMEOUT, buf);
      }
      std::this_thread::yield();
    }
  }
  (void)fwd_done;
  // all sends must complete before the slots are reused by the next batch
  cudaEvent_t e1 = c->ev(), e2 = c->ev();
  cudaEventRecord(e1, c->s_send_act);
  cudaEventRecord(e2, c->s_send_grad);
  cudaStreamWaitEvent(c->s_comp, e1, 0);
  cudaStreamWaitEvent(c->s_comp, e2, 0);
  return 0;
}


// Alg. 1 l.4-6 + l.11-14 on this rank.
static axonn_status run_batch_impl(axonn_ctx* c, const int32_t* tokens, bool on_device, int batch,
                                   float* loss_out) {
  if (!c) return AXONN_ERR_INVALID_ARG;
  if (c->sticky) return AXONN_ERR_STATE;
  if (batch < 1 || batch % (c->g_data * c->microbatch)) return AXONN_ERR_NONDIVISIBLE_BATCH;
  if (c->grads_ready) return (axonn_status)c->fail(AXONN_ERR_STATE, "run_batch twice without optimizer_step");
  if (!tokens) return AXONN_ERR_INVALID_ARG;
  CU(cudaSetDevice(c->device));
  auto t0 = std::chrono::steady_clock::now();
  const int shard = batch / c->g_data;
  const int m = shard / c->microbatch;
  c->cur_mtotal = batch / c->microbatch;   // D-9: microbatches in the whole batch
  c->cur_m = m;
  c->ev_next = 0;
  c->prof.clear();
  c->launches = 0;
  c->bwd_count = 0;
  c->stats[AXONN_STAT_P2P_BYTES] = 0;
  c->stats[AXONN_STAT_ALLREDUCE_BYTES] = 0;
  c->stats[AXONN_STAT_H2D_BYTES] = 0;
  c->stats[AXONN_STAT_D2H_BYTES] = 0;
  const int64_t need = (int64_t)shard * (c->s + 1);
  if (need > c->dtok_cap) {
    if (c->dtok) cudaFree(c->dtok);
    c->dtok = nullptr;
    CU(cudaMalloc(&c->dtok, need * 4));
    c->dtok_cap = need;
  }
  // the next forward reads theta16 written by the previous optimizer step: all of it, or
  // (overlap_next_batch) per layer as its buckets complete (Ctx::wait_params)
  if (!c->opt_pending) CU(cudaStreamWaitEvent(c->s_comp, c->ev_opt_done, 0));
  const size_t row0 = (size_t)c->replica * shard * (c->s + 1);   // Alg. 1 l.5
  // token ids must lie in [0, vocab): the kernels index embedding rows and logit columns with
  // them.  Checked before any device work of the batch, identically on every rank (host: the
  // whole batch; device: each shard, flag MAX-reduced over the world), so a bad batch returns
  // AXONN_ERR_INVALID_ARG on every rank and leaves the context usable.
  int bad = 0;
  if (on_device) {
    CU(cudaMemcpyAsync(c->dtok, tokens, need * 4, cudaMemcpyDeviceToDevice, c->s_comp));
    int* d_bad = reinterpret_cast<int*>(reinterpret_cast<char*>(c->d_loss) + 40);
    int* h_bad = reinterpret_cast<int*>(reinterpret_cast<char*>(c->h_loss) + 40);
    CU(cudaMemsetAsync(d_bad, 0, sizeof(int), c->s_comp));
    if (token_check(c->dtok, need, c->V, d_bad, c->s_comp)) return (axonn_status)c->fail(AXONN_ERR_CUDA, "token check");
    ++c->launches;
    cudaEvent_t e = c->ev();
    CU(cudaEventRecord(e, c->s_comp));
    CU(cudaStreamWaitEvent(c->s_loss, e, 0));
    if (c->world > 1 && !c->lg) NC(ncclAllReduce(d_bad, d_bad, 1, ncclInt32, ncclMax, c->world_comm, c->s_loss));
    CU(cudaMemcpyAsync(h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, c->s_loss));
    CU(cudaStreamSynchronize(c->s_loss));
    bad = *h_bad;
    if (c->lg && c->lg->rendezvous(nullptr, &bad, group_timeout_s()))
      return (axonn_status)c->fail(AXONN_ERR_STATE, "local group failed (token check)");
  } else {
    const int64_t all = (int64_t)batch * (c->s + 1);
    for (int64_t i = 0; i < all; ++i) bad |= (tokens[i] < 0) | (tokens[i] >= c->V);
  }
  if (bad) return (axonn_status)c->fail(AXONN_ERR_INVALID_ARG, "token id outside [0, vocab)");
  if (!on_device) {
    CU(cudaMemcpyAsync(c->dtok, tokens + row0, need * 4, cudaMemcpyHostToDevice, c->s_comp));
    c->stats[AXONN_STAT_H2D_BYTES] += need * 4.0;
  }
  CU(cudaMemsetAsync(c->d_loss, 0, sizeof(double), c->s_comp));
  // the batch loss is final after the last stage's last forward (recorded there); the other
  // stages contribute 0 (C5)
  if (!c->last) CU(cudaEventRecord(c->ev_loss, c->s_comp));
  if (c->first) {   // embedding gradients are scatter-added (K6)
    CU(cudaMemsetAsync(c->g32(c->tok_emb), 0, (size_t)c->V * c->h * 4, c->s_comp));
    CU(cudaMemsetAsync(c->g32(c->pos_emb), 0, (size_t)c->s * c->h * 4, c->s_comp));
  }
  const int par = (int)(c->t_step & 1);
  for (int k = 0; k < 4; ++k)
    if (!c->ph[par][k]) CU(cudaEventCreate(&c->ph[par][k]));
  c->busy_ev.clear();
  c->busy_tag.clear();
  c->msg_ev.clear();
  CU(cudaEventRecord(c->ph[par][0], c->s_comp));
  const int64_t ch_elems = chunk_elems(c);
  // AXONN_AR_OVERLAP=0: cast and reduce everything after the pipeline instead (same values)
  c->ar_overlap = c->dp_fused || !(getenv("AXONN_AR_OVERLAP") && getenv("AXONN_AR_OVERLAP")[0] == '0');
  if (c->dp_fused) ++c->dp_epoch;   // progress / read-done values of this batch
  c->ar_active = false;
  c->ev_chunk.clear();
  if (c->ar_overlap) {
    c->ar_hi = c->nflat;
    c->ar_next_chunk = (c->nflat + ch_elems - 1) / ch_elems - 1;
    c->ev_chunk.assign((size_t)(c->ar_next_chunk + 1), nullptr);
  }
  int rc = run_pipeline(c, m);
  if (rc) return (axonn_status)rc;
  CU(cudaEventRecord(c->ph[par][1], c->s_comp));
  if (c->ar_overlap) {
    if ((rc = c->ar_ready(0))) return (axonn_status)rc;   // no-op unless a stage had no layers
    c->ar_active = false;
    CU(cudaEventRecord(c->ev_grads_ready, c->s_dp));   // every chunk cast (and reduced)
  } else {
    // grad16 is still read by a pending optimizer step until it completes
    if (c->opt_pending) CU(cudaStreamWaitEvent(c->s_comp, c->ev_opt_done, 0));
    // half-precision gradients (D-20: fp32 accumulation, half reduction)
    if ((rc = c->cast_grads(0, c->nflat, c->s_comp))) return (axonn_status)rc;
    CU(cudaEventRecord(c->ev_grads_ready, c->s_comp));
  }
  if (c->g_data == 1 && !c->ar_overlap) CU(cudaEventRecord(c->ph[par][2], c->s_comp));
  CU(cudaStreamWaitEvent(c->s_loss, c->ev_loss, 0));
  if (c->world > 1 && !c->lg)   // C5: loss sum over the last-stage ranks, seen by every rank
    NC(ncclAllReduce(c->d_loss, c->d_loss, 1, ncclFloat64, ncclSum, c->world_comm, c->s_loss));
  CU(cudaMemcpyAsync(c->h_loss, c->d_loss, sizeof(double), cudaMemcpyDeviceToHost, c->s_loss));
  cudaEvent_t ev_loss_host = c->ev();
  CU(cudaEventRecord(ev_loss_host, c->s_loss));
  // Alg. 1 l.13: SUM all-reduce over the column, chunks of k * bsize
  if (c->ar_overlap) {
    CU(cudaEventRecord(c->ph[par][2], c->s_dp));
  } else if (c->g_data > 1) {
    CU(cudaStreamWaitEvent(c->s_dp, c->ev_grads_ready, 0));
    const int64_t ch = chunk_elems(c);
    for (int64_t lo = 0; lo < c->nflat; lo += ch) {
      int64_t n = std::min(ch, c->nflat - lo);
      NC(ncclAllReduce(static_cast<char*>(c->grad16) + lo * 2, static_cast<char*>(c->grad16) + lo * 2,
                       n, kNcclHalf, ncclSum, c->dp_comm, c->s_dp));
      cudaEvent_t e = c->ev();
      CU(cudaEventRecord(e, c->s_dp));
      c->ev_chunk.push_back(e);
      c->stats[AXONN_STAT_ALLREDUCE_BYTES] += n * 2.0;
    }
    CU(cudaEventRecord(c->ph[par][2], c->s_dp));
  }
  CU(cudaEventSynchronize(ev_loss_host));
  if (c->lg && c->lg->rendezvous(c->h_loss, nullptr, group_timeout_s()))   // C5 on the host
    return (axonn_status)c->fail(AXONN_ERR_STATE, "local group failed (loss)");
  // the row losses are summed unscaled (the S of D-11 enters only the CE gradient): L/S
  if (loss_out) *loss_out = (float)(*c->h_loss);
  c->grads_ready = true;
  c->pipe_stats_par = par;   // phase statistics once the pipeline has drained (Ctx::pipe_stats)
  if (c->opt_pending) {   // the previous step (every forward of this batch waited for it)
    cudaEventSynchronize(c->ev_opt_done);
    c->opt_pending = false;
    c->collect_stats();
    c->prof_opt.clear();
    c->phase_stats_ar_opt(par ^ 1);
  }
  c->stats[AXONN_STAT_T_BATCH_MS] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return AXONN_OK;
}

}  // namespace axonn

extern "C" {

AXONN_API axonn_status axonn_run_batch(axonn_ctx* c, const int32_t* tokens, int batch, float* loss_out) {
  const axonn_status rc = run_batch_impl(c, tokens, false, batch, loss_out);
  // loopback: after a sticky failure the other stages must not wait for this one (argument
  // errors are detected identically on every stage before any exchange)
  if (rc && c && c->lg && c->sticky) c->lg->abort();
  return rc;
}

AXONN_API axonn_status axonn_run_batch_device(axonn_ctx* c, const int32_t* d_tokens, int batch,
                                              float* loss_out) {
  const axonn_status rc = run_batch_impl(c, d_tokens, true, batch, loss_out);
  if (rc && c && c->lg && c->sticky) c->lg->abort();
  return rc;
}

// Alg. 1 l.7 with the memory optimisation and the
// all-reduce / optimizer interleave.
static axonn_status optimizer_step_impl(axonn_ctx* c);
AXONN_API axonn_status axonn_optimizer_step(axonn_ctx* c) {
  const axonn_status rc = optimizer_step_impl(c);
  if (rc && c && c->lg && c->sticky) c->lg->abort();
  return rc;
}

static axonn_status optimizer_step_impl(axonn_ctx* c) {
  if (!c) return AXONN_ERR_INVALID_ARG;
  if (c->sticky) return AXONN_ERR_STATE;
  if (!c->grads_ready) return (axonn_status)c->fail(AXONN_ERR_STATE, "optimizer_step without run_batch");
  CU(cudaSetDevice(c->device));
  auto t0 = std::chrono::steady_clock::now();
  const int64_t t = c->t_step + 1;
  // step scalars in double, rounded once to fp32 (D-14)
  const double lr = c->oc.lr, b1 = c->oc.beta1, b2 = c->oc.beta2;
  float sc[9];
  sc[0] = (float)(1.0 - lr * c->oc.weight_decay);
  sc[1] = (float)b1;
  sc[2] = (float)(1.0 - b1);
  sc[3] = (float)b2;
  sc[4] = (float)(1.0 - b2);
  sc[5] = (float)(lr / (1.0 - std::pow(b1, (double)t)));
  sc[6] = (float)std::sqrt(1.0 - std::pow(b2, (double)t));
  sc[7] = (float)c->oc.eps;   // eps rounded once
  sc[8] = (float)(1.0 / c->oc.loss_scale);
  // the optimizer may start only once the gradients exist: per chunk (ev_chunk, A8) or, without
  // chunk events, all of them
  if (c->ev_chunk.empty()) CU(cudaStreamWaitEvent(c->s_opt, c->ev_grads_ready, 0));
  if (kHalfDtype == AXONN_FP16) {
    // Reading D-12: skip the whole step if any reduced gradient of any stage overflowed.
    // The flag needs the complete all-reduce (s_dp is past its last chunk), then one
    // MAX over the world on s_dp (the stream of the other world-comm collective).
    CU(cudaStreamWaitEvent(c->s_dp, c->ev_grads_ready, 0));
    CU(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->s_dp));
    if (nonfinite_scan(c->grad16, c->nflat, c->d_flag, c->s_dp))
      return (axonn_status)c->fail(AXONN_ERR_CUDA, "nonfinite scan");
    ++c->launches;
    {   // the world comm's collectives all run on s_loss (issue order = the loss, then this)
      cudaEvent_t es = c->ev();
      CU(cudaEventRecord(es, c->s_dp));
      CU(cudaStreamWaitEvent(c->s_loss, es, 0));
    }
    if (c->world > 1 && !c->lg) NC(ncclAllReduce(c->d_flag, c->d_flag, 1, ncclInt32, ncclMax, c->world_comm, c->s_loss));
    CU(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->s_loss));
    cudaEvent_t e = c->ev();
    CU(cudaEventRecord(e, c->s_loss));
    CU(cudaEventSynchronize(e));
    if (c->lg && c->lg->rendezvous(nullptr, c->h_flag, group_timeout_s()))
      return (axonn_status)c->fail(AXONN_ERR_STATE, "local group failed (overflow flag)");
    if (*c->h_flag) {   // nothing was updated; t stays; run_batch may follow
      c->grads_ready = false;
      c->ev_chunk.clear();
      c->err = "non-finite gradient (fp16 overflow at loss scale " + std::to_string(c->oc.loss_scale) +
               "): step skipped, t = " + std::to_string(c->t_step);
      return AXONN_ERR_NONFINITE;
    }
    CU(cudaStreamWaitEvent(c->s_opt, e, 0));
    c->ev_chunk.clear();   // every chunk is reduced: no per-bucket waits needed
  }
  const int64_t bs = c->oc.bucket_elems;
  const int64_t ch = chunk_elems(c);
  int64_t chunk_idx = -1;
  const bool overlap = c->oc.overlap_next_batch != 0;
  c->ev_next_opt = 0;
  if (overlap) {
    const size_t nb = (size_t)((c->nflat + bs - 1) / bs);
    while (c->ev_bucket.size() < nb) {
      cudaEvent_t e;
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->ev_bucket.push_back(e);
    }
  }
  // Bucket order (A8).  With chunk events and no next-batch overlap the
  // buckets run in chunk-completion order: chunks are handed off top-first during the last
  // backward (Ctx::ar_ready), so chunk c_max's buckets start first, each chunk's buckets in
  // ascending order, each waiting only for its own chunk -- the update of the top layers runs
  // while the rest of the backward and of the column all-reduce are still in flight.  With
  // overlap_next_batch the next batch's forward needs layer 0 first: ascending order.
  const int64_t nbk = (c->nflat + bs - 1) / bs;
  std::vector<int64_t> order;
  order.reserve(nbk);
  const bool by_chunk = !overlap && !c->ev_chunk.empty();
  if (by_chunk) {
    const int64_t kpc = ch / bs;   // buckets per chunk (ch = k * bsize)
    for (int64_t ci = (int64_t)c->ev_chunk.size() - 1; ci >= 0; --ci)
      for (int64_t b = ci * kpc; b < std::min(nbk, (ci + 1) * kpc); ++b) order.push_back(b);
  } else {
    for (int64_t b = 0; b < nbk; ++b) order.push_back(b);
  }
  // fused column reduction (reading D-35): K9 sums the replicas' half gradients itself
  const bool sum_peers = c->dp_fused && !c->ev_chunk.empty();
  std::vector<const void*> gp(c->g_data);
  auto k9 = [&](int64_t lo0, int64_t n0, float* th, float* mm, float* vv) -> int {
    void* t16 = static_cast<char*>(c->theta16) + lo0 * 2;
    if (!sum_peers)
      return adamw_launch(n0, static_cast<const char*>(c->grad16) + lo0 * 2, th, mm, vv, t16, sc, c->s_opt);
    for (int j = 0; j < c->g_data; ++j) gp[j] = static_cast<const char*>(c->dp_g16[j]) + lo0 * 2;
    return adamw_sum_launch(n0, gp.data(), c->g_data, th, mm, vv, t16, sc, c->s_opt);
  };
  int64_t pend_lo = -1;   // in-HBM: first element of the run not yet handed to a launch
  for (size_t q = 0; q < order.size(); ++q) {
    const int64_t bucket = order[q];
    const int64_t lo = bucket * bs;
    const int64_t n = std::min(bs, c->nflat - lo);
    const int64_t ci = lo / ch;
    if (ci != chunk_idx && ci < (int64_t)c->ev_chunk.size()) {   // bucket waits for its chunk
      if (c->ev_chunk[ci]) CU(cudaStreamWaitEvent(c->s_opt, c->ev_chunk[ci], 0));
      if (sum_peers) {   // ... on every replica of the column
        const int rc = c->dp_wait(c->s_opt, 0, c->dp_progress(ci));
        if (rc) return (axonn_status)rc;
      }
      chunk_idx = ci;
    }
    void* t16 = static_cast<char*>(c->theta16) + lo * 2;
    const void* g = static_cast<const char*>(c->grad16) + lo * 2;
    ProfRec pr{};
    if (c->oc.offload) {   // fetch bucket, step, offload back; 3-slot ring
      const int r = (int)(q % 3);
      if (q >= 3) CU(cudaStreamWaitEvent(c->s_h2d, c->ev_d2h[r], 0));
      CU(cudaMemcpyAsync(c->ring[r][0], c->master + lo, n * 4, cudaMemcpyHostToDevice, c->s_h2d));
      CU(cudaMemcpyAsync(c->ring[r][1], c->adam_m + lo, n * 4, cudaMemcpyHostToDevice, c->s_h2d));
      CU(cudaMemcpyAsync(c->ring[r][2], c->adam_v + lo, n * 4, cudaMemcpyHostToDevice, c->s_h2d));
      CU(cudaEventRecord(c->ev_h2d[r], c->s_h2d));
      CU(cudaStreamWaitEvent(c->s_opt, c->ev_h2d[r], 0));
      if (c->profiling) { pr.a = c->ev_opt(); pr.b = c->ev_opt(); cudaEventRecord(pr.a, c->s_opt); }
      if (k9(lo, n, c->ring[r][0], c->ring[r][1], c->ring[r][2]))
        return (axonn_status)c->fail(AXONN_ERR_CUDA, "adamw launch");
      if (c->profiling) { cudaEventRecord(pr.b, c->s_opt); pr.work = n * 28.0; pr.kind = 1; c->prof.push_back(pr); }
      CU(cudaEventRecord(c->ev_adam[r], c->s_opt));
      if (overlap) CU(cudaEventRecord(c->ev_bucket[bucket], c->s_opt));
      CU(cudaStreamWaitEvent(c->s_d2h, c->ev_adam[r], 0));
      CU(cudaMemcpyAsync(c->master + lo, c->ring[r][0], n * 4, cudaMemcpyDeviceToHost, c->s_d2h));
      CU(cudaMemcpyAsync(c->adam_m + lo, c->ring[r][1], n * 4, cudaMemcpyDeviceToHost, c->s_d2h));
      CU(cudaMemcpyAsync(c->adam_v + lo, c->ring[r][2], n * 4, cudaMemcpyDeviceToHost, c->s_d2h));
      CU(cudaEventRecord(c->ev_d2h[r], c->s_d2h));
      c->stats[AXONN_STAT_H2D_BYTES] += n * 12.0;
      c->stats[AXONN_STAT_D2H_BYTES] += n * 12.0;
      ++c->launches;
      continue;
    }
    // In HBM the bucket is only a scheduling unit: consecutive buckets that wait for the same
    // chunk (all of them when there are no chunk events) run as one launch (same values;
    // AdamW is elementwise), unless the next batch overlaps and needs per-bucket events.
    if (pend_lo < 0) pend_lo = lo;
    const int64_t end = lo + n;
    const bool run_ends = q + 1 == order.size() || order[q + 1] != bucket + 1 ||
                          (!c->ev_chunk.empty() && (order[q + 1] * bs) / ch != ci);
    if (overlap || run_ends) {
      const int64_t n2 = end - pend_lo;
      const void* g2 = static_cast<const char*>(c->grad16) + pend_lo * 2;
      void* t2 = static_cast<char*>(c->theta16) + pend_lo * 2;
      if (c->profiling) { pr.a = c->ev_opt(); pr.b = c->ev_opt(); cudaEventRecord(pr.a, c->s_opt); }
      if (k9(pend_lo, n2, c->master + pend_lo, c->adam_m + pend_lo, c->adam_v + pend_lo))
        return (axonn_status)c->fail(AXONN_ERR_CUDA, "adamw launch");
      if (c->profiling) { cudaEventRecord(pr.b, c->s_opt); pr.work = n2 * 28.0; pr.kind = 1; c->prof.push_back(pr); }
      if (overlap) CU(cudaEventRecord(c->ev_bucket[bucket], c->s_opt));
      pend_lo = -1;
      ++c->launches;
    }
  }
  // every peer's grad16 has been read (or, gradients written by axonn_write_tensor, none was):
  // the peers may overwrite theirs -- signalled after every step so no cast waits forever
  if (c->dp_fused && c->dp_epoch > 0) {
    const int rc = c->dp_signal(c->s_opt, c->g_data + c->replica, c->dp_epoch);
    if (rc) return (axonn_status)rc;
  }
  if (c->oc.offload) {
    cudaEvent_t e = c->ev();
    CU(cudaEventRecord(e, c->s_d2h));
    CU(cudaStreamWaitEvent(c->s_opt, e, 0));
  }
  CU(cudaEventRecord(c->ev_opt_done, c->s_opt));
  const int par = (int)((t - 1) & 1);   // parity of the batch this step belongs to
  if (c->ph[par][3] == nullptr) CU(cudaEventCreate(&c->ph[par][3]));
  CU(cudaEventRecord(c->ph[par][3], c->s_opt));
  c->t_step = t;
  c->grads_ready = false;
  c->ev_chunk.clear();
  c->pipe_stats(c->pipe_stats_par);
  if (overlap) {   // returns now; the next run_batch waits per layer (reading D-32)
    for (ProfRec& p : c->prof)
      if (p.kind == 1) c->prof_opt.push_back(p);
    c->prof.erase(std::remove_if(c->prof.begin(), c->prof.end(),
                                 [](const ProfRec& p) { return p.kind == 1; }),
                  c->prof.end());
    c->opt_pending = true;
    c->stats[AXONN_STAT_T_OPT_MS] =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return AXONN_OK;
  }
  CU(cudaEventSynchronize(c->ev_opt_done));
  c->stats[AXONN_STAT_T_OPT_MS] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  c->collect_stats();
  c->phase_stats_ar_opt(par);
  return AXONN_OK;
}

}  // extern "C"

namespace axonn {

// Device-timed Alg. 2 phase of batch `par` (PAPER.md:704-708 phase bars): waits until the
// pipeline has drained on s_comp (run_batch returns once the loss is known, possibly before
// its last backward has finished), then reads the phase and busy-span events.
void Ctx::pipe_stats(int par) {
  Ctx* c = this;
  if (par < 0 || !c->ph[par][1]) return;
  pipe_stats_par = -1;
  cudaEventSynchronize(c->ph[par][1]);
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ph[par][0], c->ph[par][1]);
  c->stats[AXONN_STAT_T_PIPE_MS] = ms;
  double busy = 0;
  for (auto& pr : c->busy_ev) {
    float b = 0;
    cudaEventElapsedTime(&b, pr.first, pr.second);
    busy += b;
  }
  c->stats[AXONN_STAT_T_BUSY_MS] = busy;
  if (const char* tl = getenv("AXONN_TIMELINE")) {   // per-op timeline of this batch (diagnostics)
    std::string path = std::string(tl) + ".rank" + std::to_string(c->rank) + ".csv";
    if (FILE* f = fopen(path.c_str(), "w")) {
      fprintf(f, "stage,kind,mb,start_ms,end_ms\n");
      for (size_t k = 0; k < c->busy_ev.size() && k < c->busy_tag.size(); ++k) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, c->ph[par][0], c->busy_ev[k].first);
        cudaEventElapsedTime(&b, c->ph[par][0], c->busy_ev[k].second);
        fprintf(f, "%d,%c,%d,%.4f,%.4f\n", c->stage, (c->busy_tag[k] & 1) ? 'B' : 'F', c->busy_tag[k] / 2, a, b);
      }
      for (auto& me : c->msg_ev) {
        float a = 0;
        if (cudaEventElapsedTime(&a, c->ph[par][0], me.second) == cudaSuccess)
          fprintf(f, "%d,%s,%d,%.4f,%.4f\n", c->stage, (me.first & 1) ? "msg_grad" : "msg_act", me.first / 2, a, a);
      }
      fclose(f);
    }
  }
}

void Ctx::phase_stats_ar_opt(int par) {
  if (!ph[par][1] || !ph[par][2] || !ph[par][3]) return;
  float ar = 0, op = 0;
  if (cudaEventElapsedTime(&ar, ph[par][1], ph[par][2]) != cudaSuccess) ar = 0;
  if (cudaEventElapsedTime(&op, ph[par][2], ph[par][3]) != cudaSuccess) op = 0;
  stats[AXONN_STAT_T_ALLREDUCE_MS] = ar;
  stats[AXONN_STAT_T_OPT_EXPOSED_MS] = op > 0 ? op : 0;
}

void Ctx::wait_params(int64_t off_end) {
  if (!opt_pending || ev_bucket.empty()) return;
  const int64_t bs = oc.bucket_elems;
  int64_t b = (off_end - 1) / bs;
  if (b >= (int64_t)ev_bucket.size()) b = (int64_t)ev_bucket.size() - 1;
  cudaStreamWaitEvent(s_comp, ev_bucket[b], 0);
}

// kernel-time statistics (profiling mode) of the records of this batch and of the optimizer
// step they belong with; every record's events have completed when this runs
void Ctx::collect_stats() {
  Ctx* c = this;
  // kernel-time statistics of this batch + step (profiling mode)
  double gms = 0, gfl = 0, ams = 0, aby = 0;
  int gl = 0;
  std::vector<ProfRec> all(c->prof);
  all.insert(all.end(), c->prof_opt.begin(), c->prof_opt.end());
  for (const ProfRec& p : all) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.a, p.b);
    if (p.kind == 0) { gms += ms; gfl += p.work; ++gl; }
    else if (p.kind == 1) { ams += ms; aby += p.work; }
  }
  c->stats[AXONN_STAT_GEMM_MS] = gms;
  c->stats[AXONN_STAT_GEMM_FLOP] = gfl;
  c->stats[AXONN_STAT_GEMM_LAUNCHES] = gl;
  c->stats[AXONN_STAT_ADAM_MS] = ams;
  c->stats[AXONN_STAT_ADAM_BYTES] = aby;
  c->stats[AXONN_STAT_KERNEL_LAUNCHES] = (double)c->launches;
  if (!all.empty()) {   // per-shape breakdown: {"key": [ms, work, launches], ...}
    std::map<std::string, double[3]> agg;
    for (const ProfRec& p : all) {
      float ms = 0;
      cudaEventElapsedTime(&ms, p.a, p.b);
      const std::string k = p.kind == 1 ? "adamw" : p.key;
      agg[k][0] += ms;
      agg[k][1] += p.work;
      agg[k][2] += 1;
    }
    std::string js = "{";
    for (auto& kv : agg) {
      char buf[192];
      snprintf(buf, sizeof(buf), "%s\"%s\": [%.6f, %.6e, %d]", js.size() > 1 ? ", " : "",
               kv.first.c_str(), kv.second[0], kv.second[1], (int)kv.second[2]);
      js += buf;
    }
    c->prof_json = js + "}";
  }
}

}  // namespace axonn

extern "C" {

}  // extern "C"
