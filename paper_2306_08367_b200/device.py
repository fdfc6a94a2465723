"""Device plumbing: a C-ABI context bound to torch's current CUDA stream, and
helpers that move numpy <-> torch device tensors.  torch is used for device
memory and streams only; every operator runs in liblaq_b200.so."""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _abi, errors

_tls = threading.local()


class Context:
    """laq_ctx (include/laq_b200.h): one device, one stream."""

    transport = "single process"  # set by dist.attach

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise errors.CudaError("no CUDA device: the LAQ engine has no CPU fallback")
        self.device = device
        self.lib = _abi.lib()
        h = C.c_void_p()
        rc = self.lib.laq_ctx_create(device, C.byref(h))
        if rc != 0:
            raise errors.BY_CODE.get(rc, errors.Error)(f"laq_ctx_create failed ({rc})")
        self.h = h
        self.bind_stream()

    def bind_stream(self, stream: torch.cuda.Stream | None = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.stream = s
        self.lib.laq_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream))

    def check(self, rc: int):
        if rc != 0:
            errors.raise_for(rc, self.lib.laq_ctx_last_error(self.h).decode(errors="replace"))

    def sync(self):
        self.check(self.lib.laq_ctx_synchronize(self.h))

    # ---- row-sharded multi-GPU (laq_ctx_attach_nccl / laq_ctx_set_allreduce_host)
    def attach_nccl(self, nranks: int, rank: int, uid: bytes):
        """Attach an NCCL communicator (uid: 128 bytes from nccl_unique_id() on rank 0)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
        self.check(self.lib.laq_ctx_attach_nccl(self.h, nranks, rank, buf))

    def set_allreduce_host(self, nranks: int, rank: int, fn):
        """fn(np.ndarray int64) sums the array in place across ranks (any host transport)."""
        if fn is None:
            self._hook = None
            self.check(self.lib.laq_ctx_set_allreduce_host(self.h, 1, 0, None, None))
            return

        def tramp(buf, count, _user):
            try:
                fn(np.ctypeslib.as_array(buf, shape=(count,)))
                return 0
            except Exception:  # noqa: BLE001 - reported as a C status
                return 1
        self._hook = _abi.ALLREDUCE_HOST_FN(tramp)  # keep the thunk alive
        self.check(self.lib.laq_ctx_set_allreduce_host(self.h, nranks, rank, self._hook, None))

    @property
    def comm(self) -> tuple[int, int]:
        n, r = C.c_int32(), C.c_int32()
        self.check(self.lib.laq_ctx_comm_info(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def allreduce_acc(self, acc: torch.Tensor):
        """Sum an int64 device accumulator across the attached ranks (in place)."""
        assert acc.dtype == torch.int64 and acc.is_cuda and acc.is_contiguous()
        self.check(self.lib.laq_allreduce_acc(self.h, C.c_void_p(acc.data_ptr()), acc.numel()))
        return acc

    @property
    def launches(self) -> int:
        return int(self.lib.laq_ctx_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.laq_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = _abi.lib().laq_nccl_unique_id(buf)
    if rc != 0:
        errors.raise_for(rc, "laq_nccl_unique_id failed")
    return bytes(buf)


def context(device: int = 0) -> Context:
    """Per-thread default context on `device`, bound to the current stream."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = ctxs[device] = Context(device)
    else:
        ctx.bind_stream()
    return ctx


def dev(x, dtype=None, device: int = 0) -> torch.Tensor:
    """numpy / list / tensor -> contiguous CUDA tensor (no copy if already there)."""
    if isinstance(x, torch.Tensor):
        t = x
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.device.type != "cuda":
            t = t.to(f"cuda:{device}", non_blocking=False)
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(x))
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(f"cuda:{device}")


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else (
        C.c_void_p(t.data_ptr()) if t is not None else None)


def ptrs(ts):
    return _abi.ptr_array([t.data_ptr() if t is not None else None for t in ts])
