"""ctypes marshalling for libpst.so.  No arithmetic of the method lives here."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PST_LIB=bf16 / f16 selects another precision build (libpst_bf16.so / libpst_f16.so)
_LIB_PATH = os.path.join(_HERE, {"bf16": "libpst_bf16.so", "f16": "libpst_f16.so", "exp": "libpst_exp.so"}.get(
    os.environ.get("PST_LIB", ""), "libpst.so"))
if os.environ.get("PST_LIB_PATH"):   # experiment builds (tools/); still the same C ABI
    _LIB_PATH = os.environ["PST_LIB_PATH"]

PST_OK = 0
_STATUS = {0: "PST_OK", -1: "PST_E_INVALID", -2: "PST_E_OOM", -3: "PST_E_CUDA", -4: "PST_E_NCCL",
           -5: "PST_E_STATE", -6: "PST_E_UNSUPPORTED"}
W_PARAMS, W_MOMENTUM, W_BNSTATS = 1, 2, 4
NCCL_ID_BYTES = 128


class PstError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


class _Layer(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "cin", "cout", "k", "stride", "pad", "bias", "bn",
                                         "block_begin", "residual", "relu", "pool")] + [("dropout", C.c_float)]


class _Net(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("layers", C.POINTER(_Layer)), ("in_c", C.c_int32),
                ("in_h", C.c_int32), ("in_w", C.c_int32), ("n_classes", C.c_int32),
                ("init_params", C.POINTER(C.c_float)), ("n_params", C.c_int64)]


class _Partition(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("ppv", C.POINTER(C.c_int32)), ("devices", C.POINTER(C.c_int32)),
                ("mapping", C.c_int32)]

MAP_PER_GPU, MAP_FS_BKS = 0, 1


class _HParams(C.Structure):
    _fields_ = [("batch", C.c_int32), ("momentum", C.c_float), ("weight_decay", C.c_float),
                ("lr_pipelined", C.POINTER(C.c_float)), ("lr_nonpipelined", C.c_float),
                ("n_milestones", C.c_int32), ("milestone_epochs", C.POINTER(C.c_int64)),
                ("gamma", C.c_float), ("steps_per_epoch", C.c_int64),
                ("solver", C.c_int32), ("nesterov", C.c_int32), ("lr_policy", C.c_int32),
                ("inv_gamma", C.c_float), ("inv_power", C.c_float), ("dropout_seed", C.c_uint32)]


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p)]


class _Batch(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("on_device", C.c_int32), ("stream", C.c_void_p)]


_lib = None


def lib():
    """Load libpst.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} not found; build it with `python -m paper_1912_12675_b200.build` "
                          "(or __graft_entry__.build()).  There is no CPU fallback.")
    L = C.CDLL(_LIB_PATH)
    P = C.POINTER
    sig = {
        "pst_create": (C.c_int, [P(_Net), P(_Partition), P(_HParams), P(_Dist), P(C.c_void_p)]),
        "pst_step": (C.c_int, [C.c_void_p, P(_Batch)]),
        "pst_set_hybrid": (C.c_int, [C.c_void_p, C.c_int64]),
        "pst_flush": (C.c_int, [C.c_void_p]),
        "pst_weights": (C.c_int, [C.c_void_p, C.c_uint32, P(C.c_float), C.c_int64, P(C.c_int64)]),
        "pst_losses": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(C.c_float)]),
        "pst_versions": (C.c_int, [C.c_void_p, P(C.c_int64), C.c_int32]),
        "pst_progress": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64)]),
        "pst_stream": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_void_p)]),
        "pst_sync": (C.c_int, [C.c_void_p]),
        "pst_destroy": (None, [C.c_void_p]),
        "pst_memory": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_int64), C.c_int32]),
        "pst_last_error": (C.c_char_p, [C.c_void_p]),
        "pst_nccl_unique_id": (C.c_int, [C.c_void_p]),
        "pst_partition_ranges": (C.c_int, [P(_Net), P(_Partition), P(C.c_int32)]),
        "pst_param_count": (C.c_int64, [P(_Net)]),
        "pst_schedule": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_int64, P(C.c_int64),
                                   P(C.c_int64), P(C.c_int64)]),
        "pst_build_info": (C.c_char_p, []),
        "pst_ring_slots": (C.c_int, [C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_int32)]),
        "pst_launches": (C.c_int, [C.c_void_p, P(C.c_int64)]),
        "pst_profile": (C.c_int, [C.c_void_p, C.c_int32]),
        "pst_stage_timing": (C.c_int, [C.c_void_p, C.c_int32]),
        "pst_stage_times": (C.c_int, [C.c_void_p, P(C.c_double), C.c_int32, P(C.c_int64)]),
        "pst_profile_read": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_double), P(C.c_int64), P(C.c_double),
                                       P(C.c_double)]),
        "pst_op_conv2d_fwd": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 8),
        "pst_op_conv2d_dgrad": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 8),
        "pst_op_conv2d_wgrad": (C.c_int, [C.c_void_p] * 3 + [C.c_int] * 8),
        "pst_op_time_conv": (C.c_int, [C.c_int] * 10 + [P(C.c_float)]),
        "pst_op_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(rc, ctx=None):
    if rc != PST_OK:
        msg = lib().pst_last_error(ctx)
        raise PstError(rc, msg.decode() if msg else "")


def build_info() -> str:
    return lib().pst_build_info().decode()


# --------------------------------------------------------------------------- structs
def net_struct(net, params: Optional[np.ndarray] = None):
    """pst_workloads.NetSpec (+ canonical float32 params) -> (pst_net, keepalive)."""
    kinds = {"conv": 0, "fc": 1}
    pools = {"none": 0, "max2": 1, "gap": 2}
    arr = (_Layer * len(net.layers))()
    for i, L in enumerate(net.layers):
        arr[i] = _Layer(kinds[L.kind], L.cin, L.cout, L.k, L.stride, L.pad, int(L.bias), int(L.bn),
                        int(L.block_begin), int(L.residual), int(L.relu), pools[L.pool],
                        float(getattr(L, "dropout", 0.0)))
    keep = [arr]
    n = _Net()
    n.n_layers = len(net.layers)
    n.layers = C.cast(arr, C.POINTER(_Layer))
    n.in_c, n.in_h, n.in_w = net.in_shape
    n.n_classes = net.n_classes
    if params is not None:
        p = np.ascontiguousarray(params, dtype=np.float32)
        keep.append(p)
        n.init_params = p.ctypes.data_as(C.POINTER(C.c_float))
        n.n_params = p.size
    return n, keep


def _partition(ppv, devices=None, mapping=0):
    K = len(ppv) + 1
    pp = (C.c_int32 * max(1, K - 1))(*ppv)
    part = _Partition(K, C.cast(pp, C.POINTER(C.c_int32)), None, mapping)
    keep = [pp]
    if devices is not None:
        dv = (C.c_int32 * len(devices))(*devices)
        part.devices = C.cast(dv, C.POINTER(C.c_int32))
        keep.append(dv)
    return part, keep


def schedule(K: int, s: int, t: int, n_total: int = -1):
    b, f, v = C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib().pst_schedule(K, s, t, n_total, C.byref(b), C.byref(f), C.byref(v)))
    return b.value, f.value, v.value


def ring_slots(K: int, s: int):
    """(saved-state slots, input-ring slots, graph-key period) of stage s (pst_ring_slots)."""
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib().pst_ring_slots(K, s, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def partition_ranges(net, ppv):
    n, keep = net_struct(net)
    part, keep2 = _partition(ppv)
    out = (C.c_int32 * (2 * (len(ppv) + 1)))()
    _check(lib().pst_partition_ranges(C.byref(n), C.byref(part), out))
    return [(out[2 * i], out[2 * i + 1]) for i in range(len(ppv) + 1)]


def param_count(net) -> int:
    n, keep = net_struct(net)
    v = lib().pst_param_count(C.byref(n))
    if v < 0:
        _check(int(v))
    return int(v)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(lib().pst_nccl_unique_id(buf))
    return buf.raw


# --------------------------------------------------------------------------- pipeline
class Pipeline:
    """One pst_ctx.  Local mode (all stages in this process) unless `rank`/`nccl_id` given."""

    def __init__(self, net, params, ppv: Sequence[int], batch: int, lr_pipelined: Sequence[float],
                 lr_nonpipelined: float, momentum: float = 0.9, weight_decay: float = 0.0,
                 milestones: Sequence[int] = (), gamma: float = 0.1, steps_per_epoch: int = 1 << 62,
                 devices: Optional[Sequence[int]] = None, rank: Optional[int] = None,
                 nccl_id: Optional[bytes] = None, solver: str = "torch", nesterov: bool = False,
                 lr_policy: str = "multistep", inv_gamma: float = 0.0, inv_power: float = 0.0,
                 dropout_seed: int = 0, mapping: int = 0):
        L = lib()
        self.net = net
        self.K = len(ppv) + 1
        self.batch = batch
        n, self._keep_net = net_struct(net, params)
        part, self._keep_part = _partition(list(ppv), devices, mapping)
        lrs = (C.c_float * self.K)(*lr_pipelined)
        ms = (C.c_int64 * max(1, len(milestones)))(*milestones)
        hp = _HParams(batch, momentum, weight_decay, C.cast(lrs, C.POINTER(C.c_float)), lr_nonpipelined,
                      len(milestones), C.cast(ms, C.POINTER(C.c_int64)), gamma, steps_per_epoch,
                      {"torch": 0, "caffe": 1}[solver], int(bool(nesterov)),
                      {"multistep": 0, "inv": 1}[lr_policy], inv_gamma, inv_power, dropout_seed & 0xFFFFFFFF)
        self._keep_hp = (lrs, ms)
        dist = None
        if rank is not None:
            self._nid = C.create_string_buffer(nccl_id, NCCL_ID_BYTES)
            dist = _Dist(rank, self.K, C.cast(self._nid, C.c_void_p))
        self.rank = rank
        ctx = C.c_void_p()
        rc = L.pst_create(C.byref(n), C.byref(part), C.byref(hp), C.byref(dist) if dist else None,
                          C.byref(ctx))
        _check(rc)
        self._ctx = ctx

    # -- helpers
    def _c(self, rc):
        _check(rc, self._ctx)

    def step(self, x, y):
        """x: float32 NCHW, y: int32 labels; numpy (host) arrays or torch CUDA tensors."""
        b = _Batch()
        t = x if hasattr(x, "data_ptr") else y
        if hasattr(t, "data_ptr"):
            import torch
            b.x = x.data_ptr() if x is not None else None
            b.y = y.data_ptr() if y is not None else None
            b.on_device = 1
            b.stream = torch.cuda.current_stream(t.device).cuda_stream   # the producer stream
        else:
            xs = np.ascontiguousarray(x, dtype=np.float32) if x is not None else None
            ys = np.ascontiguousarray(y, dtype=np.int32) if y is not None else None
            b.x = xs.ctypes.data if xs is not None else None
            b.y = ys.ctypes.data if ys is not None else None
            b.on_device = 0
        self._c(lib().pst_step(self._ctx, C.byref(b)))

    def set_hybrid(self, switch_epoch: int):
        self._c(lib().pst_set_hybrid(self._ctx, switch_epoch))

    def flush(self):
        self._c(lib().pst_flush(self._ctx))

    def weights(self, what: int = W_PARAMS) -> np.ndarray:
        n = C.c_int64()
        self._c(lib().pst_weights(self._ctx, what, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        self._c(lib().pst_weights(self._ctx, what, out.ctypes.data_as(C.POINTER(C.c_float)), out.size,
                                  C.byref(n)))
        return out

    def losses(self, first_mb: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self._c(lib().pst_losses(self._ctx, first_mb, n, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def versions(self) -> np.ndarray:
        v = (C.c_int64 * self.K)()
        self._c(lib().pst_versions(self._ctx, v, self.K))
        n = self.K if self.rank is None else 1
        return np.array(v[:n], dtype=np.int64)

    def progress(self):
        s, f = C.c_int64(), C.c_int64()
        self._c(lib().pst_progress(self._ctx, C.byref(s), C.byref(f)))
        return s.value, f.value

    def stream(self, stage: int) -> int:
        p = C.c_void_p()
        self._c(lib().pst_stream(self._ctx, stage, C.byref(p)))
        return p.value or 0

    def sync(self):
        self._c(lib().pst_sync(self._ctx))

    def memory(self, stage: int) -> dict:
        """Device memory of an owned stage (pst_memory)."""
        out = (C.c_int64 * 6)()
        self._c(lib().pst_memory(self._ctx, stage, out, 6))
        return {"bytes_total": out[0], "ring_slots": out[1], "paper_slots": out[2], "bytes_per_slot": out[3],
                "param_bytes": out[4], "input_ring_slots": out[5]}

    def launches(self) -> int:
        n = C.c_int64()
        self._c(lib().pst_launches(self._ctx, C.byref(n)))
        return n.value

    def profile(self, enable: bool):
        self._c(lib().pst_profile(self._ctx, 1 if enable else 0))

    def stage_timing(self, enable: bool):
        """Serialise the stages within each step and time each one (pst_stage_timing)."""
        self._c(lib().pst_stage_timing(self._ctx, 1 if enable else 0))

    def stage_times(self):
        """(ms per owned stage accumulated since stage_timing(True), timed steps)."""
        n = self.K if self.rank is None else 1
        ms = (C.c_double * n)()
        steps = C.c_int64()
        self._c(lib().pst_stage_times(self._ctx, ms, n, C.byref(steps)))
        return np.array(ms[:n]), steps.value

    KERNEL_CLASSES = ("conv_fwd", "conv_dgrad", "conv_wgrad", "bn_apply", "bwd_pre", "bn_bwd", "pool", "sgd",
                      "loss", "misc")

    def profile_read(self):
        """{class: (ms, launches, alg_bytes, alg_flops)} since profile(True)."""
        out = {}
        for i, name in enumerate(self.KERNEL_CLASSES):
            ms, n, b, f = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
            self._c(lib().pst_profile_read(self._ctx, i, C.byref(ms), C.byref(n), C.byref(b), C.byref(f)))
            out[name] = (ms.value, n.value, b.value, f.value)
        return out

    def close(self):
        if getattr(self, "_ctx", None):
            lib().pst_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------- single ops
class _Ops:
    """pst_ops.h on torch CUDA tensors (float32 NCHW / OIHW)."""

    @staticmethod
    def _run(fn, *ptrs_and_ints):
        rc = fn(*ptrs_and_ints)
        if rc != PST_OK:
            raise PstError(rc, lib().pst_op_last_error().decode())

    def conv2d_fwd(self, x, w, stride, pad):
        import torch
        N, Cin, H, W = x.shape
        Cout, _, k, _ = w.shape
        Ho, Wo = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
        y = torch.empty((N, Cout, Ho, Wo), dtype=torch.float32, device=x.device)
        self._run(lib().pst_op_conv2d_fwd, x.data_ptr(), w.data_ptr(), y.data_ptr(), N, Cin, H, W, Cout, k,
                  stride, pad)
        return y

    def conv2d_dgrad(self, gy, w, in_hw, stride, pad):
        import torch
        N, Cout = gy.shape[:2]
        _, Cin, k, _ = w.shape
        H, W = in_hw
        gx = torch.empty((N, Cin, H, W), dtype=torch.float32, device=gy.device)
        self._run(lib().pst_op_conv2d_dgrad, gy.data_ptr(), w.data_ptr(), gx.data_ptr(), N, Cin, H, W, Cout, k,
                  stride, pad)
        return gx

    def conv2d_wgrad(self, x, gy, k, stride, pad):
        import torch
        N, Cin, H, W = x.shape
        Cout = gy.shape[1]
        gw = torch.empty((Cout, Cin, k, k), dtype=torch.float32, device=x.device)
        self._run(lib().pst_op_conv2d_wgrad, x.data_ptr(), gy.data_ptr(), gw.data_ptr(), N, Cin, H, W, Cout, k,
                  stride, pad)
        return gw

    def time_conv(self, which, N, Cin, H, W, Cout, k, stride, pad, iters=50):
        """Mean device microseconds of one fwd (0) / dgrad (1) / wgrad (2) launch (tuning aid)."""
        us = C.c_float(0.0)
        self._run(lib().pst_op_time_conv, which, N, Cin, H, W, Cout, k, stride, pad, iters, C.byref(us))
        return us.value


ops = _Ops()
