"""Python wrapper of one libaxonn context (one process per GPU).

Argument marshalling only: construction calls ``axonn_init``, ``run_batch``
calls ``axonn_run_batch`` (Alg. 1 l.4-6 + Alg. 2 + the column all-reduce),
``optimizer_step`` calls ``axonn_optimizer_step`` (Alg. 1 l.7 with the
bucketed offload and all-reduce/optimizer overlap).  See include/axonn.h."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

T_PARAM16, T_GRAD, T_MASTER, T_ADAM_M, T_ADAM_V, T_GRAD32 = range(6)

STAT_NAMES = ["t_batch_ms", "t_opt_ms", "gemm_ms", "gemm_flop", "gemm_launches",
              "kernel_launches", "adam_ms", "adam_bytes", "p2p_bytes", "allreduce_bytes",
              "h2d_bytes", "d2h_bytes", "t_pipe_ms", "t_busy_ms", "t_allreduce_ms",
              "t_opt_exposed_ms"]

STATUS = {0: "OK", -1: "INVALID_ARG", -2: "GRID_MISMATCH", -3: "NONDIVISIBLE_LAYERS",
          -4: "NONDIVISIBLE_BATCH", -5: "OOM", -6: "CUDA", -7: "NCCL", -8: "STATE",
          -9: "NONFINITE", -10: "TIMEOUT"}


class AxoNNError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class LocalGroup:
    """Test-only loopback transport (include/axonn.h axonn_local_group_create): the G_inter
    stages of one pipeline as contexts of this process, each created and driven by its own
    thread (ctypes releases the GIL during library calls).  See ``run_stages``."""

    def __init__(self, size: int, dtype: str = "bf16"):
        self.lib = _lib.load(dtype)
        self.size = size
        self.handle = C.c_void_p()
        rc = self.lib.axonn_local_group_create(size, C.byref(self.handle))
        if rc != 0:
            raise AxoNNError(rc, "axonn_local_group_create failed")

    def free(self):
        if self.handle:
            self.lib.axonn_local_group_free(self.handle)
            self.handle = C.c_void_p()


def run_stages(fn, n: int):
    """Call fn(i) for i in range(n) on n threads at once (the loopback stages' collective
    calls); returns the results in order and re-raises the first exception."""
    import threading
    out, err = [None] * n, [None] * n

    def body(i):
        try:
            out[i] = fn(i)
        except BaseException as e:   # noqa: BLE001 -- re-raised in the caller
            err[i] = e
    th = [threading.Thread(target=body, args=(i,)) for i in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


class AxoNN:
    """One g^{i,j} of the G_inter x G_data grid."""

    def __init__(self, g_inter: int, g_data: int, microbatch: int, *, n_layers: int, hidden: int,
                 heads: int, seq_len: int, vocab: int, init_seed: int = 42, lr: float = 1e-3,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.01, loss_scale: float = 1.0, offload: bool = False,
                 bucket_elems: int = 4_000_000, coarsen_k: int = 4, pipeline_limit: int = 0,
                 overlap_next_batch: bool | None = None, checkpoint_interval: int = 0,
                 stage_balance: bool | str = False, stage_speed=None,
                 grad_accum_fp32: bool = True,
                 rank: int = 0, world_size: int = 1, device: int = 0, nccl_id: bytes | None = None,
                 dtype: str = "bf16", local_group: "LocalGroup | None" = None):
        # the half format picks the library build (include/axonn.h axonn_dtype)
        self.lib = _lib.load(dtype)
        self.dtype = dtype
        self.mc = _lib.ModelCfg(n_layers, hidden, heads, seq_len, vocab, init_seed, _lib.DTYPES[dtype])
        self.oc = _lib.OptCfg(lr, beta1, beta2, eps, weight_decay, loss_scale, int(offload),
                              bucket_elems, coarsen_k, pipeline_limit, checkpoint_interval,
                              # default: overlap when the optimizer is host-link bound (offload);
                              # in HBM the AdamW kernels only compete with the GEMMs for SMs
                              int(offload if overlap_next_batch is None else overlap_next_batch),
                              int(bool(stage_balance)), None,
                              # False: the paper's footprint, weight matrices accumulate in
                              # the half gradient (reading D-38)
                              int(bool(grad_accum_fp32)))
        # reading D-21c: stage_balance="calibrate" measures every rank's sustained K1 speed
        # on the stage's FC1 shape and splits by the slowest replica of each stage
        if stage_balance == "calibrate" and stage_speed is None and g_inter > 1:
            stage_speed = self.calibrate_stage_speed(
                self.lib, g_inter, g_data, microbatch * seq_len, hidden, rank, world_size, device)
        self.stage_speed = None if stage_speed is None else [float(x) for x in stage_speed]
        if self.stage_speed is not None:
            self._speed = (C.c_double * g_inter)(*self.stage_speed)
            self.oc.stage_speed = self._speed
        self._id = C.create_string_buffer(nccl_id if nccl_id else b"\0" * 128, 128)
        self._group = local_group    # keeps the loopback group alive as long as this context
        self.dist = _lib.Dist(rank, world_size, C.cast(self._id, C.c_void_p), device,
                              local_group.handle if local_group is not None else None)
        self.ctx = C.c_void_p()
        rc = self.lib.axonn_init(g_inter, g_data, microbatch, C.byref(self.mc), C.byref(self.oc),
                                 C.byref(self.dist), C.byref(self.ctx))
        if rc != 0:
            raise AxoNNError(rc, "axonn_init failed")
        self.g_inter, self.g_data, self.microbatch = g_inter, g_data, microbatch
        self.seq_len = seq_len
        self.rank, self.world_size = rank, world_size
        self.stage, self.replica = rank % g_inter, rank // g_inter
        self._tensors = None

    @staticmethod
    def calibrate_stage_speed(lib, g_inter, g_data, M, hidden, rank, world_size, device,
                              seconds: float = 0.4):
        """Per-stage speeds for axonn_opt_cfg.stage_speed: every rank times the library's K1
        on the FC1 shape (M x 4h x h) for about ``seconds`` (axonn_calibrate_speed), the
        TFLOP/s are all-gathered over the host process group, and stage i takes the minimum
        over its column (replicas share the layer split).  Host-side marshalling only."""
        N, K = 4 * hidden, hidden
        M, N, K = (max(128, (x + 7) // 8 * 8) for x in (M, N, K))
        # about `seconds` at ~1 PFLOP/s, clamped: tiny shapes are launch-bound (~5 us a launch)
        iters = min(4000, max(8, int(seconds * 1.0e15 / (2.0 * M * N * K))))
        tf = C.c_double()
        rc = lib.axonn_calibrate_speed(device, M, N, K, iters, C.byref(tf))
        if rc != 0:
            raise AxoNNError(rc, "axonn_calibrate_speed failed")
        speeds = [tf.value]
        if world_size > 1:
            import torch.distributed as dist
            speeds = [None] * world_size
            dist.all_gather_object(speeds, tf.value)
        return [min(speeds[j * g_inter + i] for j in range(g_data)) for i in range(g_inter)]

    def partition(self):
        """The block boundaries of the stage split (axonn_stage_partition)."""
        out = (C.c_int * (self.g_inter + 1))()
        rc = self.lib.axonn_stage_partition(C.byref(self.mc), self.g_inter, self.oc.stage_speed, out)
        if rc != 0:
            raise AxoNNError(rc, "axonn_stage_partition failed")
        return list(out)

    # ------------------------------------------------------------- lifecycle
    def close(self):
        if self.ctx:
            self.lib.axonn_free(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc != 0:
            msg = self.lib.axonn_last_error(self.ctx)
            raise AxoNNError(rc, f"{what}: {msg.decode() if msg else ''}")

    # ------------------------------------------------------------- hot path
    def run_batch(self, tokens: np.ndarray) -> float:
        """tokens: int32 [batch, seq_len + 1], the full batch (Alg. 1 l.4)."""
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        assert tok.ndim == 2 and tok.shape[1] == self.seq_len + 1
        loss = C.c_float()
        self._check(self.lib.axonn_run_batch(self.ctx, tok.ctypes.data_as(C.c_void_p),
                                             tok.shape[0], C.byref(loss)), "run_batch")
        return loss.value

    def run_batch_device(self, d_tokens_ptr: int, batch: int) -> float:
        """This replica's shard [batch/G_data, seq_len + 1] already on the device."""
        loss = C.c_float()
        self._check(self.lib.axonn_run_batch_device(self.ctx, C.c_void_p(d_tokens_ptr), batch,
                                                    C.byref(loss)), "run_batch_device")
        return loss.value

    def optimizer_step(self):
        self._check(self.lib.axonn_optimizer_step(self.ctx), "optimizer_step")

    # ------------------------------------------------------------- inspection
    def tensors(self):
        if self._tensors is None:
            out = []
            name = C.create_string_buffer(64)
            shape = (C.c_int64 * 2)()
            numel = C.c_int64()
            for i in range(self.lib.axonn_num_tensors(self.ctx)):
                self._check(self.lib.axonn_tensor_info(self.ctx, i, name, shape, C.byref(numel)),
                            "tensor_info")
                rows, cols = shape[0], shape[1]
                shp = (cols,) if rows == 1 else (rows, cols)
                out.append((name.value.decode(), shp, numel.value))
            self._tensors = out
        return self._tensors

    def read(self, which: int, idx: int) -> np.ndarray:
        name, shp, n = self.tensors()[idx]
        buf = np.empty(n, dtype=np.float32)
        self._check(self.lib.axonn_read_tensor(self.ctx, which, idx, buf.ctypes.data_as(C.c_void_p)),
                    f"read {name}")
        return buf.reshape(shp)

    def write(self, which: int, idx: int, values) -> None:
        name, shp, n = self.tensors()[idx]
        buf = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        assert buf.size == n, (name, buf.size, n)
        self._check(self.lib.axonn_write_tensor(self.ctx, which, idx, buf.ctypes.data_as(C.c_void_p)),
                    f"write {name}")

    def read_all(self, which: int) -> dict:
        return {name: self.read(which, i) for i, (name, _, _) in enumerate(self.tensors())}

    def write_all(self, which: int, values: dict) -> None:
        for i, (name, _, _) in enumerate(self.tensors()):
            self.write(which, i, values[name])

    def checkpoint_interval(self) -> int:
        """The activation checkpointing interval in use (axonn_checkpoint_interval)."""
        return self.lib.axonn_checkpoint_interval(self.ctx)

    def timer_mark(self, i: int):
        self._check(self.lib.axonn_timer_mark(self.ctx, i), "timer_mark")

    def timer_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        self._check(self.lib.axonn_timer_elapsed(self.ctx, a, b, C.byref(ms)), "timer_elapsed")
        return ms.value

    def profile(self) -> dict:
        """Per-shape K1/K9 timing of the last profiled batch: key -> (ms, work, launches)."""
        import json
        n = self.lib.axonn_profile_json(self.ctx, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib.axonn_profile_json(self.ctx, buf, n + 1)
        return json.loads(buf.value.decode() or "{}")

    def set_profiling(self, on: bool):
        self._check(self.lib.axonn_set_profiling(self.ctx, int(on)), "set_profiling")

    def stats(self) -> dict:
        buf = (C.c_double * len(STAT_NAMES))()
        self._check(self.lib.axonn_stats(self.ctx, buf, len(STAT_NAMES)), "stats")
        return dict(zip(STAT_NAMES, list(buf)))
