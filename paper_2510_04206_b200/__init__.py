"""paper_2510_04206_b200 -- B200-native (sm_100a) AgentRL hot path.

Thin ctypes binding over ``libagentrl.so`` (C ABI: ``include/agentrl.h``).  This
module only marshals arguments: every step of the path runs in the library's CUDA
kernels.  PyTorch is used for device memory, streams and process groups.  There is
no CPU fallback: importing this package without the built library raises.

Entry points (same names as the C ABI):
    agentrl_task_adv_norm        PAPER.md P:543-579 (sec 3.2 Eq.1) after P:1263 (GRPO)
    agentrl_policy_loss_fwd_bwd
    agentrl_grpo_step            both, back to back
plus ``Step`` (owns workspace/outputs for repeated calls) and ``Comm`` (NCCL).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# AGENTRL_LIB: an alternative in-tree build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("AGENTRL_LIB") or os.path.join(_HERE, "libagentrl.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not built: run `python paper_2510_04206_b200/build.py` "
        "(there is no CPU fallback for this package)")

_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

# ---- status codes / bits (include/agentrl.h)
OK = 0
ERR_INVALID_ARG, ERR_SHAPE, ERR_WORKSPACE, ERR_CUDA, ERR_NCCL, ERR_UNSUPPORTED = -1, -2, -3, -4, -5, -6
ST_BAD_TARGET, ST_NONFINITE, ST_BAD_OFFSETS = 1, 2, 4
ST_GROUP_SPANS_TASKS, ST_GROUP_TOO_SMALL, ST_NO_TOKENS = 8, 16, 32
ST_COMM_TIMEOUT = 64
ST_ROWS_OVERFLOW = 128

EXPORTED = (
    "agentrl_task_adv_norm_workspace_size", "agentrl_task_adv_norm",
    "agentrl_policy_loss_workspace_size", "agentrl_policy_loss_workspace_size_vp",
    "agentrl_policy_loss_fwd_bwd",
    "agentrl_grpo_step_workspace_size", "agentrl_grpo_step",
    "agentrl_comm_unique_id", "agentrl_comm_init", "agentrl_comm_destroy",
    "agentrl_status_string", "agentrl_version", "agentrl_last_launch_count",
    "agentrl_profile_start", "agentrl_profile_stop", "agentrl_kernel_name",
    "agentrl_debug_adv_phase_ns", "agentrl_comm_init_callback",
    "agentrl_logprob_workspace_size", "agentrl_logprob_fwd", "agentrl_comm_set_reduce_scatter",
    "agentrl_comm_enable_peer_window", "agentrl_debug_bookkeeping",
    "agentrl_debug_throttle_waits",
)
NUM_KERNEL_IDS = 12


class LogprobArgs(C.Structure):
    _fields_ = [("T", C.c_int64), ("d", C.c_int32), ("V", C.c_int32), ("hidden", C.c_void_p),
                ("W_head", C.c_void_p), ("target", C.c_void_p), ("loss_mask", C.c_void_p),
                ("logit_scale", C.c_float), ("max_rows", C.c_int32)]


class Batch(C.Structure):
    _fields_ = [("T", C.c_int64), ("n_traj", C.c_int32), ("n_groups", C.c_int32),
                ("n_tasks", C.c_int32), ("traj_offsets", C.c_void_p), ("task_id", C.c_void_p),
                ("group_id", C.c_void_p), ("rewards", C.c_void_p), ("loss_mask", C.c_void_p)]


class LossArgs(C.Structure):
    _fields_ = [("T", C.c_int64), ("d", C.c_int32), ("V", C.c_int32), ("hidden", C.c_void_p),
                ("W_head", C.c_void_p), ("target", C.c_void_p), ("adv_tok", C.c_void_p),
                ("old_logp", C.c_void_p), ("loss_mask", C.c_void_p),
                ("clip_eps_low", C.c_float), ("clip_eps_high", C.c_float),
                ("logit_scale", C.c_float), ("n_mask_global", C.c_void_p),
                ("grad_W_mode", C.c_int32), ("max_rows", C.c_int32),
                ("kl_beta", C.c_float), ("loss_agg", C.c_int32), ("ref_logp", C.c_void_p),
                ("tok_weight", C.c_void_p)]


class LossOut(C.Structure):
    _fields_ = [("loss", C.c_void_p), ("logp", C.c_void_p), ("grad_hidden", C.c_void_p),
                ("grad_W", C.c_void_p), ("loss_stats", C.c_void_p)]


_P, _i64, _i32, _f64, _sz = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_size_t
_lib.agentrl_task_adv_norm_workspace_size.argtypes = [_i64, _i32, _i32, _i32]
_lib.agentrl_task_adv_norm_workspace_size.restype = _sz
_lib.agentrl_task_adv_norm.argtypes = [C.POINTER(Batch), _f64, _P, _P, _P, _P, _sz, _P, _P, _P]
_lib.agentrl_policy_loss_workspace_size.argtypes = [_i64, _i64, _i32, _i32]
_lib.agentrl_policy_loss_workspace_size.restype = _sz
_lib.agentrl_policy_loss_workspace_size_vp.argtypes = [_i64, _i64, _i32, _i32, _i32]
_lib.agentrl_policy_loss_workspace_size_vp.restype = _sz
_lib.agentrl_policy_loss_fwd_bwd.argtypes = [C.POINTER(LossArgs), C.POINTER(LossOut), _P, _sz,
                                             _P, _P, _P]
_lib.agentrl_grpo_step_workspace_size.argtypes = [_i64, _i32, _i32, _i32, _i64, _i32, _i32]
_lib.agentrl_grpo_step_workspace_size.restype = _sz
_lib.agentrl_grpo_step.argtypes = [C.POINTER(Batch), _f64, C.POINTER(LossArgs),
                                   C.POINTER(LossOut), _P, _P, _P, _sz, _P, _P, _P]
_lib.agentrl_comm_unique_id.argtypes = [C.c_char_p]
_lib.agentrl_comm_init.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_char_p]
_lib.agentrl_comm_destroy.argtypes = [_P]
_lib.agentrl_comm_set_reduce_scatter.argtypes = [_P, C.c_void_p]
_lib.agentrl_comm_enable_peer_window.argtypes = [_P, _sz]
_lib.agentrl_comm_init_callback.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_void_p,
                                            C.c_void_p]
_lib.agentrl_logprob_workspace_size.argtypes = [_i64, _i64, _i32, _i32]
_lib.agentrl_logprob_workspace_size.restype = _sz
_lib.agentrl_logprob_fwd.argtypes = [C.POINTER(LogprobArgs), _P, _P, _P, _sz, _P, _P]
_lib.agentrl_debug_bookkeeping.argtypes = [_P, _i64, _i32, _i32, _i32, _P, _P, _P, _P, _P]
_lib.agentrl_status_string.argtypes = [C.c_int]
_lib.agentrl_status_string.restype = C.c_char_p
_lib.agentrl_version.restype = C.c_int
_lib.agentrl_last_launch_count.restype = C.c_int
_lib.agentrl_profile_start.argtypes = [C.c_int]
_lib.agentrl_profile_stop.argtypes = [_P, _P, C.c_int]
_lib.agentrl_kernel_name.argtypes = [C.c_int]
_lib.agentrl_kernel_name.restype = C.c_char_p


def lib():
    return _lib


def status_string(code: int) -> str:
    return _lib.agentrl_status_string(int(code)).decode()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _check(rc: int, what: str) -> None:
    if rc != OK:
        raise RuntimeError(f"{what} failed: {rc} ({status_string(rc)})")


# --------------------------------------------------------------------------- C ABI mirrors
def make_batch(b) -> Batch:
    """``b``: dict of device tensors traj_offsets (int64), task_id, group_id (int32),
    rewards (float32), loss_mask (uint8), plus ints T, n_groups, n_tasks."""
    return Batch(int(b["T"]), int(b["task_id"].numel()), int(b["n_groups"]), int(b["n_tasks"]),
                 _ptr(b["traj_offsets"]), _ptr(b["task_id"]), _ptr(b["group_id"]),
                 _ptr(b["rewards"]), _ptr(b["loss_mask"]))


def make_loss_args(T, hidden, W_head, target, old_logp, loss_mask, adv_tok=None,
                   n_mask_global=None, eps_low=0.2, eps_high=0.2, logit_scale=1.0,
                   grad_W_mode=0, kl_beta=0.0, loss_agg=0, ref_logp=None,
                   tok_weight=None, max_rows=0) -> LossArgs:
    d = int(hidden.shape[1])
    V = int(W_head.shape[0])
    return LossArgs(int(T), d, V, _ptr(hidden), _ptr(W_head), _ptr(target), _ptr(adv_tok),
                    _ptr(old_logp), _ptr(loss_mask), float(eps_low), float(eps_high),
                    float(logit_scale), _ptr(n_mask_global), int(grad_W_mode), int(max_rows),
                    float(kl_beta), int(loss_agg), _ptr(ref_logp), _ptr(tok_weight))


def make_loss_out(loss, grad_hidden, grad_W, logp=None, loss_stats=None) -> LossOut:
    return LossOut(_ptr(loss), _ptr(logp), _ptr(grad_hidden), _ptr(grad_W), _ptr(loss_stats))


def agentrl_task_adv_norm_workspace_size(T, n_traj, n_groups, n_tasks) -> int:
    return int(_lib.agentrl_task_adv_norm_workspace_size(T, n_traj, n_groups, n_tasks))


def agentrl_policy_loss_workspace_size(T, d, V, max_rows=0) -> int:
    """max_rows: bound on the masked tokens (<= 0: T); pass the same value in the args"""
    return int(_lib.agentrl_policy_loss_workspace_size(T, max_rows, d, V))


def agentrl_policy_loss_workspace_size_vp(T, d, V, world, max_rows=0) -> int:
    """grad_W_mode = 3 (vocabulary-parallel head): V = this rank's shard rows"""
    return int(_lib.agentrl_policy_loss_workspace_size_vp(T, max_rows, d, V, world))


def agentrl_grpo_step_workspace_size(T, n_traj, n_groups, n_tasks, d, V, max_rows=0) -> int:
    return int(_lib.agentrl_grpo_step_workspace_size(T, n_traj, n_groups, n_tasks, max_rows, d,
                                                     V))


def agentrl_task_adv_norm(batch: Batch, eps_std, adv_tok, task_stats, n_mask_global, ws,
                          comm=None, d_status=None, stream=None) -> int:
    return _lib.agentrl_task_adv_norm(C.byref(batch), float(eps_std), _ptr(adv_tok),
                                      _ptr(task_stats), _ptr(n_mask_global), _ptr(ws),
                                      ws.numel() * ws.element_size(), comm, _ptr(d_status),
                                      _stream(stream))


def agentrl_policy_loss_fwd_bwd(args: LossArgs, out: LossOut, ws, comm=None, d_status=None,
                                stream=None) -> int:
    return _lib.agentrl_policy_loss_fwd_bwd(C.byref(args), C.byref(out), _ptr(ws),
                                            ws.numel() * ws.element_size(), comm,
                                            _ptr(d_status), _stream(stream))


def agentrl_grpo_step(batch: Batch, eps_std, args: LossArgs, out: LossOut, adv_tok_out,
                      task_stats, ws, comm=None, d_status=None, stream=None) -> int:
    return _lib.agentrl_grpo_step(C.byref(batch), float(eps_std), C.byref(args), C.byref(out),
                                  _ptr(adv_tok_out), _ptr(task_stats), _ptr(ws),
                                  ws.numel() * ws.element_size(), comm, _ptr(d_status),
                                  _stream(stream))


def agentrl_logprob_workspace_size(T, d, V, max_rows=0) -> int:
    return int(_lib.agentrl_logprob_workspace_size(T, max_rows, d, V))


def agentrl_logprob_fwd(T, hidden, W_head, target, loss_mask, logp, entropy, ws, d_status,
                        logit_scale=1.0, stream=None, max_rows=0) -> int:
    """Forward-only log-probs (and entropies if ``entropy`` is a tensor) of the masked tokens."""
    a = LogprobArgs(int(T), int(hidden.shape[1]), int(W_head.shape[0]), _ptr(hidden),
                    _ptr(W_head), _ptr(target), _ptr(loss_mask), float(logit_scale),
                    int(max_rows))
    return _lib.agentrl_logprob_fwd(C.byref(a), _ptr(logp), _ptr(entropy), _ptr(ws),
                                    ws.numel() * ws.element_size(), _ptr(d_status),
                                    _stream(stream))


def agentrl_debug_bookkeeping(ws, T, n_traj, n_groups, n_tasks, n_g=None, K=None, idx=None,
                              rows=None, stream=None) -> int:
    """Copy part 1's n_g [n_traj], K_j [n_groups], compaction idx [T] and local row count out
    of workspace ``ws`` (int32 / int64 device tensors, any may be None)."""
    return _lib.agentrl_debug_bookkeeping(_ptr(ws), int(T), int(n_traj), int(n_groups),
                                          int(n_tasks), _ptr(n_g), _ptr(K), _ptr(idx),
                                          _ptr(rows), _stream(stream))


def bookkeeping(ws, T, n_traj, n_groups, n_tasks, stream=None):
    """(n_g, K, idx[:rows], rows) as host numpy arrays (synchronises the stream)."""
    import torch
    dev = ws.device
    n_g = torch.empty(max(n_traj, 1), dtype=torch.int32, device=dev)
    K = torch.empty(max(n_groups, 1), dtype=torch.int32, device=dev)
    idx = torch.empty(max(T, 1), dtype=torch.int32, device=dev)
    rows = torch.empty(1, dtype=torch.int64, device=dev)
    _check(agentrl_debug_bookkeeping(ws, T, n_traj, n_groups, n_tasks, n_g, K, idx, rows, stream),
           "agentrl_debug_bookkeeping")
    (stream or torch.cuda.current_stream()).synchronize()
    r = int(rows.item())
    return (n_g[:n_traj].cpu().numpy(), K[:n_groups].cpu().numpy(), idx[:r].cpu().numpy(), r)


def last_launch_count() -> int:
    return int(_lib.agentrl_last_launch_count())


def profile_start(max_pairs: int = 4096) -> None:
    """Record a CUDA-event pair around every kernel the library launches (on the stream
    it launches on) until profile_stop()."""
    _check(_lib.agentrl_profile_start(int(max_pairs)), "agentrl_profile_start")


def profile_stop() -> dict:
    """{kernel name: (summed ms, launches)} since profile_start()."""
    ms = (C.c_double * NUM_KERNEL_IDS)()
    cnt = (C.c_int * NUM_KERNEL_IDS)()
    _check(_lib.agentrl_profile_stop(C.cast(ms, C.c_void_p), C.cast(cnt, C.c_void_p),
                                     NUM_KERNEL_IDS), "agentrl_profile_stop")
    return {_lib.agentrl_kernel_name(i).decode(): (float(ms[i]), int(cnt[i]))
            for i in range(NUM_KERNEL_IDS)}


def debug_adv_phase_ns():
    """Phase boundary timestamps (ns) of the last single-GPU agentrl_task_adv_norm launch."""
    buf = (C.c_ulonglong * 8)()
    _check(_lib.agentrl_debug_adv_phase_ns(buf), "agentrl_debug_adv_phase_ns")
    return [int(x) for x in buf]


def debug_throttle_waits():
    """[forward, grad_W, grad_hidden] progress-throttle wait episodes since the library loaded."""
    buf = (C.c_ulonglong * 3)()
    _check(_lib.agentrl_debug_throttle_waits(buf), "agentrl_debug_throttle_waits")
    return [int(x) for x in buf]


def alloc_workspace(nbytes: int, device="cuda"):
    """uint8 device buffer with a 1024-byte aligned base (torch allocations are >= 512 B
    aligned; over-allocate and slice to be safe)."""
    import torch
    raw = torch.empty(int(nbytes) + 1024, dtype=torch.uint8, device=device)
    off = (-raw.data_ptr()) % 1024
    return raw[off:off + int(nbytes)]


class Comm:
    """NCCL communicator owned by the library (bootstrap id broadcast by the caller)."""

    def __init__(self, world: int, rank: int, uid: bytes):
        h = C.c_void_p()
        _check(_lib.agentrl_comm_init(C.byref(h), int(world), int(rank), uid), "agentrl_comm_init")
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib.agentrl_comm_unique_id(buf), "agentrl_comm_unique_id")
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None):
        """Bootstrap over an initialised torch.distributed group (plumbing only)."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = cls.unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8,
                         device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.broadcast(t, src=0, group=group)
        return cls(world, rank, bytes(t.cpu().tolist()))

    def enable_peer_window(self, nbytes: int):
        """Fused grad_W reduce-scatter over peer memory (collective; include/agentrl.h);
        nbytes = 0 frees the window (back to the collective reduce-scatter)."""
        _check(_lib.agentrl_comm_enable_peer_window(self.handle, int(nbytes)),
               "agentrl_comm_enable_peer_window")

    def destroy(self):
        if self.handle:
            _lib.agentrl_comm_destroy(self.handle)
            self.handle = None


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)


class CallbackComm(Comm):
    """Communicator whose all-reduces call back into Python (plumbing for hosts without NCCL
    between the ranks, e.g. several test ranks sharing one GPU).  ``fn(dev_ptr, count, dtype,
    stream_handle) -> None`` must all-reduce (sum) the device buffer in place, ordered on the
    stream; dtype is 0 = f64, 1 = f32, 2 = i64.  Optional ``rs_fn(dev_ptr, recv_count, dtype,
    stream_handle)``: in-place reduce-scatter (grad_W_mode=2); else the all-reduce is used."""

    def __init__(self, world: int, rank: int, fn, rs_fn=None):
        def _tramp(user, buf, n, dtype, stream):
            try:
                fn(buf, int(n), int(dtype), stream)
                return 0
            except Exception:  # noqa: BLE001 -- report failure through the C return code
                import traceback
                traceback.print_exc()
                return 1
        self._cb = ALLREDUCE_FN(_tramp)  # keep alive
        h = C.c_void_p()
        _check(_lib.agentrl_comm_init_callback(C.byref(h), int(world), int(rank), self._cb, None),
               "agentrl_comm_init_callback")
        self.handle = h
        self._rs = None
        if rs_fn is not None:
            def _rs_tramp(user, buf, n, dtype, stream):
                try:
                    rs_fn(buf, int(n), int(dtype), stream)
                    return 0
                except Exception:  # noqa: BLE001
                    import traceback
                    traceback.print_exc()
                    return 1
            self._rs = ALLREDUCE_FN(_rs_tramp)  # same C signature
            _check(_lib.agentrl_comm_set_reduce_scatter(h, self._rs),
                   "agentrl_comm_set_reduce_scatter")


def gloo_reduce_scatter_fn(world, rank, group=None):
    """Reduce-scatter callback (in place, block `rank` of world blocks gets the sum) over
    torch.distributed reduce_scatter_tensor through host memory (test plumbing)."""
    import torch
    import torch.distributed as dist
    cudart = _cudart()
    tmap = {0: torch.float64, 1: torch.float32, 2: torch.int64}

    def fn(buf, m, dtype, stream):
        if stream:
            torch.cuda.ExternalStream(stream).synchronize()
        else:
            torch.cuda.synchronize()
        host = torch.empty(world * m, dtype=tmap[dtype])
        es = host.element_size()
        if cudart.cudaMemcpy(C.c_void_p(host.data_ptr()), C.c_void_p(buf), C.c_size_t(host.numel() * es), 2):
            raise RuntimeError("cudaMemcpy D2H failed")
        out = torch.empty(m, dtype=tmap[dtype])
        dist.reduce_scatter_tensor(out, host, group=group)
        if cudart.cudaMemcpy(C.c_void_p(buf + rank * m * es), C.c_void_p(out.data_ptr()), C.c_size_t(m * es), 1):
            raise RuntimeError("cudaMemcpy H2D failed")
    return fn


def gloo_allreduce_fn(group=None):
    """Callback for CallbackComm: stream sync, device->host copy, torch.distributed
    all_reduce (any backend, e.g. gloo), host->device copy (test plumbing)."""
    import torch
    import torch.distributed as dist
    cudart = _cudart()
    tmap = {0: torch.float64, 1: torch.float32, 2: torch.int64}

    def fn(buf, n, dtype, stream):
        if stream:  # a null handle is the legacy default stream
            torch.cuda.ExternalStream(stream).synchronize()
        else:
            torch.cuda.synchronize()
        host = torch.empty(n, dtype=tmap[dtype])
        nbytes = n * host.element_size()
        if cudart.cudaMemcpy(C.c_void_p(host.data_ptr()), C.c_void_p(buf), C.c_size_t(nbytes), 2):
            raise RuntimeError("cudaMemcpy D2H failed")
        dist.all_reduce(host, group=group)
        if cudart.cudaMemcpy(C.c_void_p(buf), C.c_void_p(host.data_ptr()), C.c_size_t(nbytes), 1):
            raise RuntimeError("cudaMemcpy H2D failed")
    return fn


def _cudart():
    import glob
    import torch
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime",
                                   "lib", "libcudart.so*")) + ["libcudart.so.12"]
    for c in cands:
        try:
            lib = C.CDLL(c)
            lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
            return lib
        except OSError:
            continue
    raise OSError("libcudart not found")


class Step:
    """Owns the workspace and outputs of repeated ``agentrl_grpo_step`` calls on fixed shapes.

    ``batch``: device tensors (see make_batch); ``W_head`` bf16 [V,d]; per call pass hidden
    (bf16 [T,d]), target (int32), old_logp (float32).  Outputs are attributes.
    """

    def __init__(self, T, n_traj, n_groups, n_tasks, d, V, device="cuda", eps_std=1e-6,
                 eps_low=0.2, eps_high=0.2, logit_scale=1.0, comm: Comm | None = None,
                 grad_W_mode=None, kl_beta=0.0, loss_agg=0, max_rows=0):
        import torch
        self.T, self.d, self.V = int(T), int(d), int(V)
        self.eps_std, self.eps_low, self.eps_high, self.scale = eps_std, eps_low, eps_high, logit_scale
        self.kl_beta, self.loss_agg = float(kl_beta), int(loss_agg)
        self.comm = comm
        self.grad_W_mode = (1 if comm is not None else 0) if grad_W_mode is None else grad_W_mode
        # max_rows: bound on the local masked tokens (<= 0: T); the P~ intermediate is sized by it
        self.max_rows = int(max_rows)
        self.ws = alloc_workspace(agentrl_grpo_step_workspace_size(T, n_traj, n_groups, n_tasks,
                                                                   d, V, self.max_rows), device)
        self.n_tasks = n_tasks
        self.adv_tok = torch.empty(T, dtype=torch.float32, device=device)
        self.task_stats = torch.empty(n_tasks, 3, dtype=torch.float64, device=device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)
        self.logp = torch.empty(T, dtype=torch.float32, device=device)
        self.grad_hidden = torch.empty(T, d, dtype=torch.bfloat16, device=device)
        self.grad_W = torch.empty(V, d, dtype=torch.float32, device=device)
        self.loss_stats = torch.zeros(5, dtype=torch.float64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)

    def __call__(self, batch, hidden, W_head, target, old_logp, stream=None, zero_status=True,
                 ref_logp=None, tok_weight=None):
        if zero_status:
            self.status.zero_()
        b = make_batch(batch)
        a = make_loss_args(self.T, hidden, W_head, target, old_logp, batch["loss_mask"],
                           eps_low=self.eps_low, eps_high=self.eps_high,
                           logit_scale=self.scale, grad_W_mode=self.grad_W_mode,
                           kl_beta=self.kl_beta, loss_agg=self.loss_agg, ref_logp=ref_logp,
                           tok_weight=tok_weight, max_rows=self.max_rows)
        o = make_loss_out(self.loss, self.grad_hidden, self.grad_W, self.logp, self.loss_stats)
        rc = agentrl_grpo_step(b, self.eps_std, a, o, self.adv_tok, self.task_stats, self.ws,
                               self.comm.handle if self.comm else None, self.status, stream)
        _check(rc, "agentrl_grpo_step")
        return self
