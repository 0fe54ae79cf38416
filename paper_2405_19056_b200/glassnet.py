"""Thin Python binding of libglassnet.so (include/glassnet.h): argument marshalling only.

Every step of the forward pass runs in the library's sm_100a kernels; torch provides
device memory, streams and process groups.  There is no fallback: if the shared
library is missing or the device is not a B200 this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GN_LIB", os.path.join(_HERE, "libglassnet.so"))   # GN_LIB: diagnostic builds

GLASSNET_ABI_VERSION = 1
BF16, FP32 = 0, 1
POOL_SUM, POOL_MEAN = 0, 1
FLAG_R_TAKES_LD, FLAG_INPUT_NORM, FLAG_SIGMA_COND, FLAG_SUPERSAMPLE, FLAG_OBJECTS = 1, 2, 4, 8, 16
ERRORS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "UNSUPPORTED", 3: "CUDA", 4: "NCCL", 5: "OUT_OF_MEMORY"}

EXPORTS = ["glassnet_weight_count", "glassnet_create", "glassnet_forward", "glassnet_forward_host",
           "glassnet_workspace_bytes", "glassnet_weight_bytes", "glassnet_launches_per_forward",
           "glassnet_set_kernel_family", "glassnet_get_unique_id", "glassnet_comm_create",
           "glassnet_comm_destroy", "glassnet_tile_rows", "glassnet_forward_sharded",
           "glassnet_destroy", "glassnet_last_error", "glassnet_profile_begin", "glassnet_profile_end",
           "glassnet_forward_sharded_local", "glassnet_debug_psi", "glassnet_supersample",
           "glassnet_objects_begin", "glassnet_objects_add", "glassnet_objects_finish"]


class GlassNetError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"glassnet error {code} ({ERRORS.get(code, '?')}): {msg}")
        self.code = code


class Dims(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("max_batch", ctypes.c_int32), ("k_slots", ctypes.c_int32), ("levels", ctypes.c_int32),
                ("widths", ctypes.c_int32 * 4), ("t_hidden", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("pool", ctypes.c_int32), ("flags", ctypes.c_uint32)]


_lib = None


def lib():
    """Load libglassnet.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        L.glassnet_weight_count.restype = sz
        L.glassnet_weight_count.argtypes = [ctypes.POINTER(Dims)]
        L.glassnet_create.restype = ctypes.c_int
        L.glassnet_create.argtypes = [vp, sz, ctypes.POINTER(Dims), ctypes.c_int, ctypes.POINTER(vp)]
        for f in ("glassnet_forward", "glassnet_forward_host"):
            getattr(L, f).restype = ctypes.c_int
            getattr(L, f).argtypes = [vp, vp, vp, vp, vp, vp, i32, vp]
        L.glassnet_workspace_bytes.restype = sz
        L.glassnet_workspace_bytes.argtypes = [vp]
        L.glassnet_weight_bytes.restype = sz
        L.glassnet_weight_bytes.argtypes = [vp]
        L.glassnet_launches_per_forward.restype = ctypes.c_int
        L.glassnet_launches_per_forward.argtypes = [vp, i32]
        L.glassnet_set_kernel_family.restype = ctypes.c_int
        L.glassnet_set_kernel_family.argtypes = [vp, ctypes.c_int]
        L.glassnet_get_unique_id.restype = ctypes.c_int
        L.glassnet_get_unique_id.argtypes = [vp]
        L.glassnet_comm_create.restype = ctypes.c_int
        L.glassnet_comm_create.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
        L.glassnet_comm_destroy.restype = None
        L.glassnet_comm_destroy.argtypes = [vp]
        L.glassnet_tile_rows.restype = ctypes.c_int
        L.glassnet_tile_rows.argtypes = [ctypes.POINTER(Dims), i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.glassnet_forward_sharded.restype = ctypes.c_int
        L.glassnet_forward_sharded.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.glassnet_profile_begin.restype = ctypes.c_int
        L.glassnet_profile_begin.argtypes = [vp, i32]
        L.glassnet_profile_end.restype = ctypes.c_int
        L.glassnet_profile_end.argtypes = [vp, i32, vp, vp, vp, vp]
        L.glassnet_forward_sharded_local.restype = ctypes.c_int
        L.glassnet_forward_sharded_local.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
        L.glassnet_objects_begin.restype = ctypes.c_int
        L.glassnet_objects_begin.argtypes = [vp, i32, vp]
        L.glassnet_objects_add.restype = ctypes.c_int
        L.glassnet_objects_add.argtypes = [vp, vp, vp, i32, vp]
        L.glassnet_objects_finish.restype = ctypes.c_int
        L.glassnet_objects_finish.argtypes = [vp, vp, vp, vp, i32, vp]
        L.glassnet_supersample.restype = ctypes.c_int
        L.glassnet_supersample.argtypes = [vp, vp, vp, vp, i32, vp]
        L.glassnet_debug_psi.restype = ctypes.c_int
        L.glassnet_debug_psi.argtypes = [vp, vp, i32, vp]
        L.glassnet_destroy.restype = None
        L.glassnet_destroy.argtypes = [vp]
        L.glassnet_last_error.restype = ctypes.c_char_p
        L.glassnet_last_error.argtypes = []
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise GlassNetError(rc, lib().glassnet_last_error().decode())


def make_dims(height, width, k_slots, widths, t_hidden, levels=None, precision="bf16", max_batch=1,
              pool="sum", r_takes_ld=True, input_norm=True, sigma_cond=False, supersample=False, pe_L=0,
              objects=False) -> Dims:
    levels = len(widths) if levels is None else levels
    w = (ctypes.c_int32 * 4)(*(list(widths)[:levels] + [0] * (4 - levels)))
    flags = ((FLAG_R_TAKES_LD if r_takes_ld else 0) | (FLAG_INPUT_NORM if input_norm else 0)
             | (FLAG_SIGMA_COND if sigma_cond else 0) | (FLAG_SUPERSAMPLE if supersample else 0)
             | (FLAG_OBJECTS if objects else 0) | (int(pe_L) << 8))   # N2: GLASSNET_FLAG_POSENC(L)
    return Dims(GLASSNET_ABI_VERSION, height, width, max_batch, k_slots, levels, w, t_hidden,
                BF16 if precision == "bf16" else FP32, POOL_MEAN if pool == "mean" else POOL_SUM, flags)


def weight_count(dims: Dims) -> int:
    return int(lib().glassnet_weight_count(ctypes.byref(dims)))


def tile_rows(dims: Dims, nranks: int, rank: int):
    r0, n = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().glassnet_tile_rows(ctypes.byref(dims), nranks, rank, ctypes.byref(r0), ctypes.byref(n)))
    return r0.value, n.value


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data)


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class GlassNet:
    """Handle over glassnet_create/forward/destroy."""

    def __init__(self, weights, dims: Dims, device: int = 0):
        w = np.ascontiguousarray(weights, dtype="<f4")
        self.dims = dims
        self.device = device
        h = ctypes.c_void_p()
        _check(lib().glassnet_create(w.ctypes.data_as(ctypes.c_void_p), w.size, ctypes.byref(dims), device,
                                     ctypes.byref(h)))
        self._h = h

    # -- marshalling helpers --------------------------------------------------------------
    def _check_inputs(self, gbuf, direct, tbuf, tcount, out, device=True):
        import torch
        d = self.dims
        B = gbuf.shape[0]
        dt = torch.bfloat16 if d.precision == BF16 else torch.float32
        want = {"gbuf": (gbuf, (B, d.height, d.width, 12), dt), "direct": (direct, (B, d.height, d.width, 3), dt),
                "tbuf": (tbuf, (B, d.height, d.width, d.k_slots, 11), dt),
                "tcount": (tcount, (B, d.height, d.width), torch.uint8),
                "out": (out, (B, d.height, d.width, 3), torch.float32)}
        for name, (t, shape, dtype) in want.items():
            if tuple(t.shape) != shape or t.dtype != dtype or not t.is_contiguous():
                raise ValueError(f"{name}: want {shape} {dtype} contiguous, got {tuple(t.shape)} {t.dtype}")
            if device and not t.is_cuda:
                raise ValueError(f"{name} must be a CUDA tensor")
            if not device and t.is_cuda:
                raise ValueError(f"{name} must be a host tensor")
        return B

    def forward(self, gbuf, direct, tbuf, tcount, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(gbuf.shape[:3] + (3,), dtype=torch.float32, device=gbuf.device)
        B = self._check_inputs(gbuf, direct, tbuf, tcount, out)
        _check(lib().glassnet_forward(self._h, _ptr(gbuf), _ptr(direct), _ptr(tbuf), _ptr(tcount), _ptr(out), B,
                                      _stream(stream)))
        return out

    def forward_host(self, gbuf, direct, tbuf, tcount, out, stream=None):
        B = self._check_inputs(gbuf, direct, tbuf, tcount, out, device=False)
        _check(lib().glassnet_forward_host(self._h, _ptr(gbuf), _ptr(direct), _ptr(tbuf), _ptr(tcount), _ptr(out),
                                           B, _stream(stream)))
        return out

    def forward_sharded(self, comm, gbuf, direct, tbuf, tcount, out, stream=None):
        _check(lib().glassnet_forward_sharded(self._h, comm._h, _ptr(gbuf), _ptr(direct), _ptr(tbuf),
                                              _ptr(tcount), _ptr(out), _stream(stream)))
        return out

    # -- N4 object-major T (include/glassnet.h glassnet_objects_*) -------------------------
    def objects_begin(self, batch, stream=None):
        _check(lib().glassnet_objects_begin(self._h, batch, _stream(stream)))

    def objects_add(self, obj, cover, stream=None):
        """obj [B][H][W][11] (dims precision), cover [B][H][W] uint8, both on the device."""
        import torch
        d = self.dims
        B = obj.shape[0]
        dt = torch.bfloat16 if d.precision == BF16 else torch.float32
        if tuple(obj.shape) != (B, d.height, d.width, 11) or obj.dtype != dt or not obj.is_contiguous():
            raise ValueError(f"obj: want {(B, d.height, d.width, 11)} {dt}, got {tuple(obj.shape)} {obj.dtype}")
        if tuple(cover.shape) != (B, d.height, d.width) or cover.dtype != torch.uint8 or not cover.is_contiguous():
            raise ValueError(f"cover: want {(B, d.height, d.width)} uint8, got {tuple(cover.shape)} {cover.dtype}")
        _check(lib().glassnet_objects_add(self._h, _ptr(obj), _ptr(cover), B, _stream(stream)))

    def objects_finish(self, gbuf, direct, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(gbuf.shape[:3] + (3,), dtype=torch.float32, device=gbuf.device)
        _check(lib().glassnet_objects_finish(self._h, _ptr(gbuf), _ptr(direct), _ptr(out), gbuf.shape[0],
                                             _stream(stream)))
        return out

    def supersample(self, img, gbuf_hi, out=None, stream=None):
        """N3: the x2 super-sampler S (include/glassnet.h glassnet_supersample): img [B][H][W][3]
        fp32, gbuf_hi [B][2H][2W][12] (dims precision) -> out [B][2H][2W][3] fp32, all on the device."""
        import torch
        d = self.dims
        B = img.shape[0]
        dt = torch.bfloat16 if d.precision == BF16 else torch.float32
        if out is None:
            out = torch.empty((B, 2 * d.height, 2 * d.width, 3), dtype=torch.float32, device=img.device)
        for name, t, shape, dtype in (("img", img, (B, d.height, d.width, 3), torch.float32),
                                      ("gbuf_hi", gbuf_hi, (B, 2 * d.height, 2 * d.width, 12), dt),
                                      ("out", out, (B, 2 * d.height, 2 * d.width, 3), torch.float32)):
            if tuple(t.shape) != shape or t.dtype != dtype or not t.is_contiguous() or not t.is_cuda:
                raise ValueError(f"{name}: want {shape} {dtype} contiguous CUDA, got {tuple(t.shape)} {t.dtype}")
        _check(lib().glassnet_supersample(self._h, _ptr(img), _ptr(gbuf_hi), _ptr(out), B, _stream(stream)))
        return out

    def debug_psi(self, batch, stream=None):
        """psi of the last forward ([batch][H][W][3] fp32 device tensor; test/diagnostic)."""
        import torch
        d = self.dims
        out = torch.empty((batch, d.height, d.width, 3), dtype=torch.float32, device=f"cuda:{self.device}")
        _check(lib().glassnet_debug_psi(self._h, _ptr(out), batch, _stream(stream)))
        return out

    def workspace_bytes(self):
        return int(lib().glassnet_workspace_bytes(self._h))

    def weight_bytes(self):
        return int(lib().glassnet_weight_bytes(self._h))

    def launches_per_forward(self, batch):
        return int(lib().glassnet_launches_per_forward(self._h, batch))

    def set_kernel_family(self, tensor_cores: bool):
        _check(lib().glassnet_set_kernel_family(self._h, 1 if tensor_cores else 0))

    def profile_begin(self, max_launches):
        _check(lib().glassnet_profile_begin(self._h, max_launches))

    def profile_end(self, max_stages=64):
        """-> {stage: (total_ms, launches)} (synchronises)."""
        names = ctypes.create_string_buffer(32 * max_stages)
        tot = (ctypes.c_double * max_stages)()
        cnt = (ctypes.c_int32 * max_stages)()
        n = ctypes.c_int32()
        _check(lib().glassnet_profile_end(self._h, max_stages, names, tot, cnt, ctypes.byref(n)))
        raw = names.raw
        return {raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): (tot[i], cnt[i]) for i in range(min(n.value, max_stages))}

    def close(self):
        if getattr(self, "_h", None):
            lib().glassnet_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def forward_sharded_local(nets, tiles, stream=None):
    """Row-tile decomposition of one frame emulated on one device: nets[r] = rank r's
    handle, tiles[r] = (gbuf, direct, tbuf, tcount, out) device tensors of rank r's rows."""
    n = len(nets)
    arr = lambda i: (ctypes.c_void_p * n)(*[tiles[r][i].data_ptr() for r in range(n)])
    hs = (ctypes.c_void_p * n)(*[net._h.value for net in nets])
    _check(lib().glassnet_forward_sharded_local(hs, n, arr(0), arr(1), arr(2), arr(3), arr(4), _stream(stream)))


def get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().glassnet_get_unique_id(buf))
    return bytes(buf)


class Comm:
    def __init__(self, uid: bytes, nranks: int, rank: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(lib().glassnet_comm_create(buf, nranks, rank, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().glassnet_comm_destroy(self._h)
            self._h = None
