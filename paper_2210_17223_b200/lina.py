"""Thin ctypes binding of include/lina.h — argument marshalling only.

Every step of the MoE layer runs in liblina.so's CUDA kernels; this module only
turns torch tensors into device pointers and streams into cudaStream_t handles.
There is no CPU fallback: importing it without the built library, or calling a
compute entry point without an sm_100 GPU, raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblina.so")

LINA_OK = 0
STATUS_NAMES = {0: "LINA_OK", 1: "LINA_ERR_INVALID_ARGUMENT", 2: "LINA_ERR_UNSUPPORTED",
                3: "LINA_ERR_INFEASIBLE_PLAN", 4: "LINA_ERR_CUDA", 5: "LINA_ERR_NCCL",
                6: "LINA_ERR_WORKSPACE"}
LINA_F32, LINA_BF16 = 0, 1
LINA_SCHED_BASELINE, LINA_SCHED_LINA, LINA_SCHED_NAIVE, LINA_SCHED_DEFER = 0, 1, 2, 3

# Every symbol declared in include/lina.h (tests check the library exports all of them).
ABI_SYMBOLS = [
    "lina_last_error", "lina_version", "lina_get_unique_id", "lina_comm_init", "lina_comm_destroy",
    "lina_comm_check", "lina_comm_info", "lina_placement_compute", "lina_replica_split",
    "lina_moe_workspace_size", "lina_moe_forward", "lina_moe_backward", "lina_moe_infer_forward",
    "lina_moe_infer_workspace_size", "lina_sched_config", "lina_allreduce_submit",
    "lina_allreduce_wait", "lina_sched_stats", "lina_profile_enable", "lina_profile_read",
    "lina_popprof_create", "lina_popprof_destroy", "lina_popprof_add", "lina_popprof_estimate",
    "lina_phase_two_check", "lina_moe_infer_forward_two_phase", "lina_popprof_save", "lina_popprof_load",
    "lina_popprof_info", "lina_infer_last_rows", "lina_pack_decide", "lina_pack_ctl_create", "lina_pack_ctl_step",
    "lina_pack_ctl_destroy", "lina_pack_weights", "lina_comm_init_host",
]


class LinaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class MoEDesc(ctypes.Structure):
    _fields_ = [("num_tokens", ctypes.c_int32), ("d_model", ctypes.c_int32), ("d_ffn", ctypes.c_int32),
                ("num_experts", ctypes.c_int32), ("k", ctypes.c_int32), ("capacity", ctypes.c_int32),
                ("n_chunks", ctypes.c_int32), ("dtype", ctypes.c_int32), ("pack", ctypes.c_int32)]


class Route(ctypes.Structure):
    _fields_ = [("idx", ctypes.c_void_p), ("gate", ctypes.c_void_p), ("slot", ctypes.c_void_p),
                ("counts", ctypes.c_void_p), ("probs", ctypes.c_void_p),
                ("override_routing", ctypes.c_int32)]


class Profile(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("gemm_launches", ctypes.c_int64),
                ("gemm_ms", ctypes.c_double), ("gemm_phases", ctypes.c_int64),
                ("a2a_window_ms", ctypes.c_double), ("gemm_in_a2a_ms", ctypes.c_double),
                ("a2a_windows", ctypes.c_int64), ("a2a_op_ms", ctypes.c_double), ("a2a_ops", ctypes.c_int64)]


class Placement(ctypes.Structure):
    _fields_ = [("num_experts", ctypes.c_int32), ("num_devices", ctypes.c_int32),
                ("max_per_device", ctypes.c_int32), ("max_replicas", ctypes.c_int32),
                ("replicas", ctypes.POINTER(ctypes.c_int32)),
                ("replica_device", ctypes.POINTER(ctypes.c_int32)),
                ("hosted", ctypes.POINTER(ctypes.c_int32))]


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2210_17223_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
    P = ctypes.POINTER
    sig = {
        "lina_last_error": ([], ctypes.c_char_p),
        "lina_version": ([], ctypes.c_char_p),
        "lina_get_unique_id": ([ctypes.c_char_p], i32),
        "lina_comm_init": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, P(vp)], i32),
        "lina_comm_init_host": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, HostAllgather, vp, P(vp)], i32),
        "lina_comm_destroy": ([vp], i32),
        "lina_comm_check": ([vp], i32),
        "lina_comm_info": ([vp, P(ctypes.c_int), P(ctypes.c_int)], i32),
        "lina_placement_compute": ([P(ctypes.c_double), i32, i32, i32, P(Placement)], i32),
        "lina_replica_split": ([i32, i32, i32, P(i32)], i32),
        "lina_popprof_create": ([i32, i32, i32, i32, P(vp)], i32),
        "lina_popprof_destroy": ([vp], i32),
        "lina_popprof_add": ([vp, P(i32), ctypes.c_int64], i32),
        "lina_popprof_estimate": ([vp, i32, P(i32), ctypes.c_int64, P(ctypes.c_double), P(i32)], i32),
        "lina_phase_two_check": ([P(ctypes.c_double), P(i32), i32, i32, P(i32)], i32),
        "lina_popprof_save": ([vp, ctypes.c_char_p], i32),
        "lina_popprof_load": ([ctypes.c_char_p, P(vp)], i32),
        "lina_popprof_info": ([vp, P(i32), P(i32), P(i32), P(i32)], i32),
        "lina_moe_workspace_size": ([vp, P(MoEDesc), P(sz), P(sz)], i32),
        "lina_moe_forward": ([vp, P(MoEDesc), vp, vp, vp, vp, vp, vp, vp, sz, P(Route), vp], i32),
        "lina_moe_backward": ([vp, P(MoEDesc), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
        "lina_moe_infer_forward": ([vp, P(MoEDesc), vp, vp, vp, vp, vp, P(Placement), i32, P(Placement),
                                    vp, sz, vp], i32),
        "lina_moe_infer_workspace_size": ([vp, P(MoEDesc), i32, P(sz)], i32),
        "lina_moe_infer_forward_two_phase": ([vp, P(MoEDesc), vp, vp, vp, vp, vp, P(Placement),
                                              P(ctypes.c_double), P(Placement), P(i32), vp, sz, vp], i32),
        "lina_sched_config": ([vp, i32, sz], i32),
        "lina_allreduce_submit": ([vp, vp, sz, i32, vp], i32),
        "lina_allreduce_wait": ([vp, vp], i32),
        "lina_sched_stats": ([vp, P(ctypes.c_int64), P(ctypes.c_int64)], i32),
        "lina_infer_last_rows": ([vp, P(i32), P(i32)], i32),
        "lina_pack_decide": ([i32, i32, ctypes.c_double, ctypes.c_double, P(i32)], i32),
        "lina_pack_ctl_create": ([i32, i32, i32, P(vp)], i32),
        "lina_pack_ctl_step": ([vp, ctypes.c_double, ctypes.c_double, P(i32), P(i32)], i32),
        "lina_pack_ctl_destroy": ([vp], i32),
        "lina_pack_weights": ([vp, i32, i32, i32, sz, i32, vp, vp, vp], i32),
        "lina_profile_enable": ([vp, ctypes.c_int], i32),
        "lina_profile_read": ([vp, P(Profile)], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(status: int):
    if status != LINA_OK:
        raise LinaError(status, load().lina_last_error().decode())


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dtype_code(dtype) -> int:
    if dtype in (torch.float32, "f32", LINA_F32):
        return LINA_F32
    if dtype in (torch.bfloat16, "bf16", LINA_BF16):
        return LINA_BF16
    raise ValueError(f"unsupported dtype {dtype}")


def torch_dtype(code: int):
    return torch.float32 if code == LINA_F32 else torch.bfloat16


# ----------------------------------------------------------------------------- entry points


def lina_version() -> str:
    return load().lina_version().decode()


def lina_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().lina_get_unique_id(buf))
    return buf.raw


# lina_host_allgather_fn: int (*)(const void* send, void* recv, size_t bytes, void* ctx)
HostAllgather = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


class Comm:
    """One lina_comm per rank (lina_comm_init / lina_comm_init_host / lina_comm_destroy)."""

    @classmethod
    def host(cls, world: int, rank: int, device: int, allgather):
        """lina_comm_init_host: no NCCL; `allgather(data: bytes) -> list[bytes]` (one entry per
        rank, rank order) carries the bootstrap exchanges, e.g. over a torch gloo group."""
        obj = cls.__new__(cls)
        obj.handle = ctypes.c_void_p()

        def cb(send, recv, nbytes, _ctx):
            try:
                parts = allgather(ctypes.string_at(send, nbytes))
                buf = b"".join(parts)
                if len(buf) != nbytes * world:
                    return 1
                ctypes.memmove(recv, buf, len(buf))
                return 0
            except Exception:  # noqa: BLE001 - reported as a failed exchange by the library
                return 1

        obj._cb = HostAllgather(cb)  # kept alive with the communicator
        _check(load().lina_comm_init_host(world, rank, device, obj._cb, None, ctypes.byref(obj.handle)))
        obj.world, obj.rank, obj.device = world, rank, device
        return obj

    def __init__(self, world: int = 1, rank: int = 0, device: int = 0, unique_id: bytes | None = None,
                 nccl_max_ctas: int = 0):
        self.handle = ctypes.c_void_p()
        uid = None if unique_id is None else ctypes.create_string_buffer(unique_id, 128)
        _check(load().lina_comm_init(world, rank, device, uid, nccl_max_ctas, ctypes.byref(self.handle)))
        self.world, self.rank, self.device = world, rank, device

    def close(self):
        if self.handle:
            _check(load().lina_comm_destroy(self.handle))
            self.handle = ctypes.c_void_p()

    def check(self):
        _check(load().lina_comm_check(self.handle))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lina_comm_init(world=1, rank=0, device=0, unique_id=None, nccl_max_ctas=0) -> Comm:
    return Comm(world, rank, device, unique_id, nccl_max_ctas)


def make_desc(num_tokens, d_model, d_ffn, num_experts, k, capacity, n_chunks, dtype, pack=1) -> MoEDesc:
    return MoEDesc(num_tokens, d_model, d_ffn, num_experts, k, capacity, n_chunks, _dtype_code(dtype), pack)


def lina_moe_workspace_size(comm: Comm, desc: MoEDesc):
    ws, sv = ctypes.c_size_t(), ctypes.c_size_t()
    _check(load().lina_moe_workspace_size(comm.handle, ctypes.byref(desc), ctypes.byref(ws), ctypes.byref(sv)))
    return ws.value, sv.value


def lina_moe_forward(comm: Comm, desc: MoEDesc, tokens, gate_w, w1, w2, out, saved, workspace,
                     route: Route | None = None, stream=None):
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(load().lina_moe_forward(comm.handle, ctypes.byref(desc), _ptr(tokens), _ptr(gate_w), _ptr(w1),
                                   _ptr(w2), _ptr(out), _ptr(saved), _ptr(workspace), ws_bytes,
                                   ctypes.byref(route) if route is not None else None, _stream(stream)))


def lina_moe_backward(comm: Comm, desc: MoEDesc, saved, dout, tokens, gate_w, w1, w2, dtokens, dgate_w,
                      dw1, dw2, workspace, stream=None):
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(load().lina_moe_backward(comm.handle, ctypes.byref(desc), _ptr(saved), _ptr(dout), _ptr(tokens),
                                    _ptr(gate_w), _ptr(w1), _ptr(w2), _ptr(dtokens), _ptr(dgate_w),
                                    _ptr(dw1), _ptr(dw2), _ptr(workspace), ws_bytes, _stream(stream)))


def lina_moe_infer_workspace_size(comm: Comm, desc: MoEDesc, max_per_device: int) -> int:
    ws = ctypes.c_size_t()
    _check(load().lina_moe_infer_workspace_size(comm.handle, ctypes.byref(desc), max_per_device,
                                                ctypes.byref(ws)))
    return ws.value


@dataclass
class PlacementTables:
    replicas: list
    replica_device: list
    hosted: list


def _alloc_placement(E, N, mpd):
    rep = (ctypes.c_int32 * E)()
    rdev = (ctypes.c_int32 * (E * N))()
    hosted = (ctypes.c_int32 * (N * mpd))()
    pl = Placement(E, N, mpd, N, ctypes.cast(rep, ctypes.POINTER(ctypes.c_int32)),
                   ctypes.cast(rdev, ctypes.POINTER(ctypes.c_int32)),
                   ctypes.cast(hosted, ctypes.POINTER(ctypes.c_int32)))
    pl._keep = (rep, rdev, hosted)
    return pl


def placement_to_tables(pl: Placement) -> PlacementTables:
    E, N, mpd, mr = pl.num_experts, pl.num_devices, pl.max_per_device, pl.max_replicas
    rep = [pl.replicas[e] for e in range(E)]
    rdev = [[pl.replica_device[e * mr + q] for q in range(rep[e])] for e in range(E)]
    hosted = [[x for x in (pl.hosted[dv * mpd + i] for i in range(mpd)) if x >= 0] for dv in range(N)]
    return PlacementTables(rep, rdev, hosted)


def tables_to_placement(t: PlacementTables, N: int, mpd: int) -> Placement:
    E = len(t.replicas)
    pl = _alloc_placement(E, N, mpd)
    for e in range(E):
        pl.replicas[e] = t.replicas[e]
        for q in range(N):
            pl.replica_device[e * N + q] = t.replica_device[e][q] if q < len(t.replica_device[e]) else -1
    for dv in range(N):
        for i in range(mpd):
            pl.hosted[dv * mpd + i] = t.hosted[dv][i] if i < len(t.hosted[dv]) else -1
    return pl


def lina_placement_compute(popularity, num_devices: int, max_per_device: int) -> PlacementTables:
    E = len(popularity)
    pop = (ctypes.c_double * E)(*[float(x) for x in popularity])
    pl = _alloc_placement(E, num_devices, max_per_device)
    _check(load().lina_placement_compute(pop, E, num_devices, max_per_device, ctypes.byref(pl)))
    return placement_to_tables(pl)


def lina_replica_split(count: int, replicas: int, source_rank: int) -> list:
    out = (ctypes.c_int32 * replicas)()
    _check(load().lina_replica_split(count, replicas, source_rank, out))
    return list(out)


class PopProfile:
    """Sample-path popularity profile (lina_popprof_*; §5.2).

    Host-only: arrays are numpy int32 ([T, L, k] traces, [T, l, k] histories)."""

    def __init__(self, num_layers: int, num_experts: int, k: int, path_len: int):
        import numpy as np  # noqa: F401  (callers pass numpy arrays)
        h = ctypes.c_void_p()
        _check(load().lina_popprof_create(num_layers, num_experts, k, path_len, ctypes.byref(h)))
        self._h, self.L, self.E, self.k, self.l = h, num_layers, num_experts, k, path_len

    def close(self):
        if self._h:
            load().lina_popprof_destroy(self._h)
            self._h = None

    def save(self, path: str):
        _check(load().lina_popprof_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str) -> "PopProfile":
        """A profile saved by save() (lina_popprof_load); its shape comes from the file."""
        h = ctypes.c_void_p()
        _check(load().lina_popprof_load(os.fsencode(path), ctypes.byref(h)))
        dims = [ctypes.c_int32() for _ in range(4)]
        _check(load().lina_popprof_info(h, *[ctypes.byref(x) for x in dims]))
        obj = cls.__new__(cls)
        obj._h = h
        obj.L, obj.E, obj.k, obj.l = (x.value for x in dims)
        return obj

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _i32(a, shape_tail):
        import numpy as np
        a = np.ascontiguousarray(a, dtype=np.int32)
        if a.ndim != 3 or tuple(a.shape[1:]) != shape_tail:
            raise ValueError(f"expected [T, {shape_tail[0]}, {shape_tail[1]}] int32, got {a.shape}")
        return a

    def add(self, sel):
        a = self._i32(sel, (self.L, self.k))
        _check(load().lina_popprof_add(self._h, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), a.shape[0]))

    def estimate(self, layer: int, history):
        """Phase-one popularity of `layer` (list of E floats) and each token's top-k ([T, k], -1 = none)."""
        import numpy as np
        a = self._i32(history, (self.l, self.k))
        pop = (ctypes.c_double * self.E)()
        topk = np.empty((a.shape[0], self.k), dtype=np.int32)
        _check(load().lina_popprof_estimate(self._h, layer, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                            a.shape[0], pop, topk.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        return list(pop), topk


def lina_phase_two_check(estimated, actual_counts, k: int) -> bool:
    """True when the estimated and actual top-2k expert sets are identical."""
    E = len(estimated)
    est = (ctypes.c_double * E)(*[float(x) for x in estimated])
    act = (ctypes.c_int32 * E)(*[int(x) for x in actual_counts])
    out = ctypes.c_int32()
    _check(load().lina_phase_two_check(est, act, E, k, ctypes.byref(out)))
    return bool(out.value)


def lina_moe_infer_forward(comm: Comm, desc: MoEDesc, tokens, gate_w, w1_all, w2_all, out, workspace,
                           placement: PlacementTables | None = None, max_per_device: int = 0,
                           want_plan: bool = True, stream=None):
    """max_per_device is the hosted-table pitch: the planner's limit when placement is None,
    else the pitch of the given tables (>= the longest hosted list)."""
    N = comm.world
    mpd = max(max_per_device, max(len(h) for h in placement.hosted) if placement else 1)
    pl_in = None if placement is None else tables_to_placement(placement, N, mpd)
    pl_out = _alloc_placement(desc.num_experts, N, mpd) if want_plan else None
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(load().lina_moe_infer_forward(comm.handle, ctypes.byref(desc), _ptr(tokens), _ptr(gate_w),
                                         _ptr(w1_all), _ptr(w2_all), _ptr(out),
                                         ctypes.byref(pl_in) if pl_in is not None else None,
                                         mpd,
                                         ctypes.byref(pl_out) if pl_out is not None else None,
                                         _ptr(workspace), ws_bytes, _stream(stream)))
    return placement_to_tables(pl_out) if pl_out is not None else None


def lina_moe_infer_forward_two_phase(comm: Comm, desc: MoEDesc, tokens, gate_w, w1_all, w2_all, out,
                                     workspace, placement: PlacementTables, estimated, stream=None):
    """Phase-one `placement` (from `estimated`, [E] popularity) checked after gating.

    Returns (plan used, replanned: bool).  The workspace must fit the placement's pitch."""
    N = comm.world
    mpd = max(len(h) for h in placement.hosted)
    pl_in = tables_to_placement(placement, N, mpd)
    pl_out = _alloc_placement(desc.num_experts, N, mpd)
    est = (ctypes.c_double * desc.num_experts)(*[float(x) for x in estimated])
    rep = ctypes.c_int32(-1)
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(load().lina_moe_infer_forward_two_phase(comm.handle, ctypes.byref(desc), _ptr(tokens), _ptr(gate_w),
                                                   _ptr(w1_all), _ptr(w2_all), _ptr(out), ctypes.byref(pl_in),
                                                   est, ctypes.byref(pl_out), ctypes.byref(rep),
                                                   _ptr(workspace), ws_bytes, _stream(stream)))
    return placement_to_tables(pl_out), bool(rep.value)


def lina_infer_last_rows(comm: Comm):
    """(rows received from each source, rows sent to each device) of the last inference call."""
    recv = (ctypes.c_int32 * comm.world)()
    sent = (ctypes.c_int32 * comm.world)()
    _check(load().lina_infer_last_rows(comm.handle, recv, sent))
    return list(recv), list(sent)


def lina_pack_decide(world: int, pack: int, ffn_ms: float, a2a_ms: float) -> int:
    out = ctypes.c_int32()
    _check(load().lina_pack_decide(world, pack, ffn_ms, a2a_ms, ctypes.byref(out)))
    return out.value


class PackController:
    """lina_pack_ctl_create / _step / _destroy (host state of the packing controller)."""

    def __init__(self, world: int, start_step: int = 10, every: int = 4):
        self.handle = ctypes.c_void_p()
        _check(load().lina_pack_ctl_create(world, start_step, every, ctypes.byref(self.handle)))

    def step(self, ffn_ms: float, a2a_ms: float):
        pack, changed = ctypes.c_int32(), ctypes.c_int32()
        _check(load().lina_pack_ctl_step(self.handle, ffn_ms, a2a_ms, ctypes.byref(pack), ctypes.byref(changed)))
        return pack.value, bool(changed.value)

    def close(self):
        if self.handle:
            load().lina_pack_ctl_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lina_pack_weights(comm: Comm, num_experts: int, pack_from: int, pack_to: int, w_from, w_to, stream=None):
    """w_from [m0*E_l, ...] -> w_to [m1*E_l, ...] (same per-expert shape and dtype)."""
    per = w_from[0].numel() if w_from.dim() > 0 else 0
    _check(load().lina_pack_weights(comm.handle, num_experts, pack_from, pack_to, per, _dtype_code(w_from.dtype),
                                    _ptr(w_from), _ptr(w_to), _stream(stream)))


def lina_sched_config(comm: Comm, policy: int, partition_bytes: int):
    _check(load().lina_sched_config(comm.handle, policy, partition_bytes))


def lina_allreduce_submit(comm: Comm, grad, ready_stream=None):
    _check(load().lina_allreduce_submit(comm.handle, _ptr(grad), grad.numel(), _dtype_code(grad.dtype),
                                        _stream(ready_stream)))


def lina_allreduce_wait(comm: Comm, stream=None):
    _check(load().lina_allreduce_wait(comm.handle, _stream(stream)))


def lina_sched_stats(comm: Comm):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(load().lina_sched_stats(comm.handle, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def lina_profile_enable(comm: Comm, on=True):
    """on: bool or bit flags (1 timing, 2 skip collectives, 4 collectives only)."""
    _check(load().lina_profile_enable(comm.handle, int(on)))


def lina_profile_read(comm: Comm) -> dict:
    p = Profile()
    _check(load().lina_profile_read(comm.handle, ctypes.byref(p)))
    return {"kernel_launches": p.kernel_launches, "gemm_launches": p.gemm_launches,
            "gemm_ms": p.gemm_ms, "gemm_phases": p.gemm_phases, "a2a_window_ms": p.a2a_window_ms,
            "gemm_in_a2a_ms": p.gemm_in_a2a_ms, "a2a_windows": p.a2a_windows, "a2a_op_ms": p.a2a_op_ms,
            "a2a_ops": p.a2a_ops}


# ----------------------------------------------------------------------------- convenience layer


class MoELayer:
    """Owns the workspace/saved buffers for one descriptor and calls the C ABI.

    Pure marshalling: buffers are torch allocations, the compute is liblina.so."""

    def __init__(self, comm: Comm, num_tokens, d_model, d_ffn, num_experts, k, capacity, n_chunks=1,
                 dtype=torch.bfloat16, device=None, pack=1):
        self.comm = comm
        self.desc = make_desc(num_tokens, d_model, d_ffn, num_experts, k, capacity, n_chunks, dtype, pack)
        self.dtype = torch_dtype(self.desc.dtype)
        self.device = device or torch.device("cuda", comm.device)
        ws, sv = lina_moe_workspace_size(comm, self.desc)
        self.workspace = torch.empty(max(ws, 1), dtype=torch.uint8, device=self.device)
        self.saved = torch.empty(max(sv, 1), dtype=torch.uint8, device=self.device)
        T, E, kk = num_tokens, num_experts, k
        self.route_t = {
            "idx": torch.empty((T, kk), dtype=torch.int32, device=self.device),
            "gate": torch.empty((T, kk), dtype=torch.float32, device=self.device),
            "slot": torch.empty((T, kk), dtype=torch.int32, device=self.device),
            "counts": torch.empty((E,), dtype=torch.int32, device=self.device),
            "probs": torch.empty((T, E), dtype=torch.float32, device=self.device),
        }

    def route(self, override: bool = False) -> Route:
        r = self.route_t
        return Route(r["idx"].data_ptr(), r["gate"].data_ptr(), r["slot"].data_ptr(), r["counts"].data_ptr(),
                     r["probs"].data_ptr(), 1 if override else 0)

    def forward(self, tokens, gate_w, w1, w2, out=None, want_route=False, override_routing=False, stream=None):
        if out is None:
            out = torch.empty((self.desc.num_tokens, self.desc.d_model), dtype=self.dtype, device=self.device)
        route = self.route(override_routing) if (want_route or override_routing) else None
        lina_moe_forward(self.comm, self.desc, tokens, gate_w, w1, w2, out, self.saved, self.workspace,
                         route, stream)
        return out

    def backward(self, dout, tokens, gate_w, w1, w2, dtokens=None, dgate_w=None, dw1=None, dw2=None, stream=None):
        T, d = self.desc.num_tokens, self.desc.d_model
        if dtokens is None:
            dtokens = torch.empty((T, d), dtype=self.dtype, device=self.device)
        if dgate_w is None:
            dgate_w = torch.empty_like(gate_w)
        if dw1 is None:
            dw1 = torch.empty_like(w1)
        if dw2 is None:
            dw2 = torch.empty_like(w2)
        lina_moe_backward(self.comm, self.desc, self.saved, dout, tokens, gate_w, w1, w2, dtokens, dgate_w,
                          dw1, dw2, self.workspace, stream)
        return dtokens, dgate_w, dw1, dw2
