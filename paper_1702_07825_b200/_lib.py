"""Thin ctypes binding of libdvw.so (include/dvw.h).  Argument marshalling only:
every step of generation runs in the library's CUDA kernels.  There is no CPU
fallback -- if libdvw.so is missing this module raises on import.

torch is used for device memory and streams: tensors are passed by data_ptr()
and the current torch CUDA stream is passed as the cudaStream_t.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdvw.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_1702_07825_b200.build` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

DVW_OK = 0
STATUS = {0: "DVW_OK", 1: "DVW_E_INVALID_ARG", 2: "DVW_E_SHAPE", 3: "DVW_E_UNSUPPORTED",
          4: "DVW_E_STATE", 5: "DVW_E_OOM", 6: "DVW_E_CUDA", 7: "DVW_E_DEVICE_TIMEOUT"}
KERNEL_AUTO, KERNEL_STREAM, KERNEL_CLUSTER, KERNEL_TC, KERNEL_PARALLEL = 0, 1, 2, 3, 4
KERNEL_NAMES = {0: "auto", 1: "stream", 2: "cluster", 3: "tc", 4: "parallel"}

EXPORTS = ("dvw_create", "dvw_weights_numel", "dvw_load_weights", "dvw_generate", "dvw_logits",
           "dvw_generate_host", "dvw_set_kernel", "dvw_set_precision", "dvw_set_weight_bits",
           "dvw_set_weight_quant", "dvw_set_sampler", "dvw_set_trace",
           "dvw_get_info", "dvw_measure_floor", "dvw_sync", "dvw_destroy", "dvw_last_error",
           "dvw_session_create", "dvw_session_generate", "dvw_session_position", "dvw_session_destroy",
           "dvwc_create", "dvwc_weights_numel", "dvwc_load_weights", "dvwc_run", "dvwc_destroy")
SAMPLERS = {"direct": 0, "temperature": 1, "mean": 2, "mode": 3, "top_k": 4}
PRECISION_FP32, PRECISION_TF32, PRECISION_APPROX, PRECISION_APPC = 0, 1, 2, 3
PRECISION_NAMES = {0: "fp32", 1: "tf32", 2: "approx", 3: "appc"}


class _Config(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("residual", ctypes.c_int32), ("skip", ctypes.c_int32),
                ("levels", ctypes.c_int32), ("dilations", ctypes.POINTER(ctypes.c_int32)),
                ("device", ctypes.c_int32)]


class _Info(ctypes.Structure):
    _fields_ = [("last_kernel", ctypes.c_int32), ("last_grid", ctypes.c_int32),
                ("last_cluster", ctypes.c_int32), ("last_threads", ctypes.c_int32),
                ("last_launches", ctypes.c_int64), ("weight_bytes", ctypes.c_int64),
                ("workspace_bytes", ctypes.c_int64), ("chain_ctas", ctypes.c_int32),
                ("max_clusters", ctypes.c_int32), ("streams_per_cluster", ctypes.c_int32),
                ("max_clusters_pipe", ctypes.c_int32)]


_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_lib.dvw_create.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(_vp)]
_lib.dvw_create.restype = _i32
_lib.dvw_weights_numel.argtypes = [ctypes.POINTER(_Config)]
_lib.dvw_weights_numel.restype = _i64
_lib.dvw_load_weights.argtypes = [_vp, _vp, _i64, _i32]
_lib.dvw_load_weights.restype = _i32
_lib.dvw_generate.argtypes = [_vp, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _vp]
_lib.dvw_generate.restype = _i32
_lib.dvw_logits.argtypes = [_vp, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _vp]
_lib.dvw_logits.restype = _i32
_lib.dvw_generate_host.argtypes = [_vp, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _vp]
_lib.dvw_generate_host.restype = _i32
_lib.dvw_set_kernel.argtypes = [_vp, _i32]
_lib.dvw_set_kernel.restype = _i32
_lib.dvw_set_precision.argtypes = [_vp, _i32]
_lib.dvw_set_precision.restype = _i32
_lib.dvw_set_weight_bits.argtypes = [_vp, _i32]
_lib.dvw_set_weight_bits.restype = _i32
_lib.dvw_set_weight_quant.argtypes = [_vp, _i32, _i32]
_lib.dvw_set_weight_quant.restype = _i32
QUANT_SCHEMES = {"per_row": 0, "per_tensor": 1}
class _CConfig(ctypes.Structure):
    _fields_ = [("in_channels", ctypes.c_int32), ("hidden", ctypes.c_int32), ("n_layers", ctypes.c_int32),
                ("residual", ctypes.c_int32), ("device", ctypes.c_int32)]


_lib.dvwc_create.argtypes = [ctypes.POINTER(_CConfig), ctypes.POINTER(ctypes.c_void_p)]
_lib.dvwc_create.restype = ctypes.c_int32
_lib.dvwc_weights_numel.argtypes = [ctypes.POINTER(_CConfig)]
_lib.dvwc_weights_numel.restype = ctypes.c_int64
_lib.dvwc_load_weights.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32]
_lib.dvwc_load_weights.restype = ctypes.c_int32
_lib.dvwc_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                          ctypes.c_void_p]
_lib.dvwc_run.restype = ctypes.c_int32
_lib.dvwc_destroy.argtypes = [ctypes.c_void_p]
_lib.dvwc_destroy.restype = None
_lib.dvw_session_create.argtypes = [_vp, _i32, ctypes.POINTER(_vp)]
_lib.dvw_session_create.restype = _i32
_lib.dvw_session_generate.argtypes = [_vp, _vp, _vp, _i64, _i32, _vp, _i64, _vp, _vp]
_lib.dvw_session_generate.restype = _i32
_lib.dvw_session_position.argtypes = [_vp]
_lib.dvw_session_position.restype = _i64
_lib.dvw_session_destroy.argtypes = [_vp]
_lib.dvw_session_destroy.restype = None
_lib.dvw_set_sampler.argtypes = [_vp, _i32, ctypes.c_float, _i32]
_lib.dvw_set_sampler.restype = _i32
_lib.dvw_set_trace.argtypes = [_vp, _vp, _i64, _i32]
_lib.dvw_set_trace.restype = _i32
_lib.dvw_get_info.argtypes = [_vp, ctypes.POINTER(_Info)]
_lib.dvw_get_info.restype = _i32
class _Floor(ctypes.Structure):
    _fields_ = [("layer_cycles", ctypes.c_double), ("hop_cycles", ctypes.c_double),
                ("head_stage_cycles", ctypes.c_double), ("sampler_cycles", ctypes.c_double),
                ("sm_ghz", ctypes.c_double)]


_lib.dvw_measure_floor.argtypes = [_i32, ctypes.POINTER(_Floor)]
_lib.dvw_measure_floor.restype = _i32
_lib.dvw_sync.argtypes = [_vp]
_lib.dvw_sync.restype = _i32
_lib.dvw_destroy.argtypes = [_vp]
_lib.dvw_destroy.restype = None
_lib.dvw_last_error.argtypes = []
_lib.dvw_last_error.restype = ctypes.c_char_p


class DvwError(RuntimeError):
    def __init__(self, status: int, text: str):
        super().__init__(f"{STATUS.get(status, status)}: {text}")
        self.status = status
        self.name = STATUS.get(status, str(status))


def _check(st: int):
    if st != DVW_OK:
        raise DvwError(st, (_lib.dvw_last_error() or b"").decode())


def _make_config(n_layers, residual, skip, levels=256, dilations=None, device=0):
    cfg = _Config(n_layers, residual, skip, levels, None, device)
    keep = None
    if dilations is not None:
        keep = (ctypes.c_int32 * len(dilations))(*dilations)
        cfg.dilations = ctypes.cast(keep, ctypes.POINTER(ctypes.c_int32))
    return cfg, keep


def weights_numel(n_layers, residual, skip, levels=256) -> int:
    cfg, _ = _make_config(n_layers, residual, skip, levels)
    return int(_lib.dvw_weights_numel(ctypes.byref(cfg)))


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dptr(t, dtype, what):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA torch tensor")
    if t.dtype != dtype:
        raise TypeError(f"{what} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return t.data_ptr()


class Model:
    """Handle on one device (dvw_create ... dvw_destroy)."""

    def __init__(self, n_layers: int, residual: int, skip: int, levels: int = 256,
                 dilations: Optional[Sequence[int]] = None, device: int = 0):
        cfg, keep = _make_config(n_layers, residual, skip, levels, dilations, device)
        h = _vp()
        _check(_lib.dvw_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.n_layers, self.residual, self.skip, self.levels = n_layers, residual, skip, levels
        self.device = device
        self.numel = int(_lib.dvw_weights_numel(ctypes.byref(cfg)))
        del keep

    @classmethod
    def from_config(cls, cfg, device: int = 0):
        return cls(cfg.n_layers, cfg.residual, cfg.skip, cfg.levels, cfg.dilations, device)

    def close(self):
        if getattr(self, "_h", None):
            _lib.dvw_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, blob):
        """Load weights from a numpy fp32 array (host) or a CUDA fp32 tensor."""
        if isinstance(blob, np.ndarray):
            b = np.ascontiguousarray(blob, dtype=np.float32)
            _check(_lib.dvw_load_weights(self._h, b.ctypes.data, b.size, 0))
        else:
            _check(_lib.dvw_load_weights(self._h, _dptr(blob, blob.dtype, "blob"), blob.numel(), 1))
        return self

    def set_kernel(self, kernel):
        if isinstance(kernel, str):
            kernel = {v: k for k, v in KERNEL_NAMES.items()}[kernel]
        _check(_lib.dvw_set_kernel(self._h, int(kernel)))
        return self

    def set_precision(self, precision):
        """Arithmetic tier (include/dvw.h dvw_precision): "fp32" (default; batched kernel as a
        3-pass tf32 split, fp32-faithful), "tf32" (batched one pass; within the 1e-3 logit
        gate, not bit-exact), "approx" (hardware tanh gate, batch-1 kernels) or "appc" (the
        paper's App. C tanh / sigma / exp approximations; cluster, stream, parallel)."""
        if isinstance(precision, str):
            precision = {v: k for k, v in PRECISION_NAMES.items()}[precision]
        _check(_lib.dvw_set_precision(self._h, int(precision)))
        return self

    def set_weight_bits(self, bits: int):
        """Quantise every weight matrix per row to `bits` (16 or 8; 0 = off) at the next
        load() (include/dvw.h dvw_set_weight_bits)."""
        _check(_lib.dvw_set_weight_bits(self._h, int(bits)))
        return self

    def set_weight_quant(self, bits: int, scheme: str = "per_row"):
        """Quantisation with a chosen scale granularity: "per_row" (R32) or "per_tensor"
        (R33, SPEC's QuantizedWeightSet), applied at the next load() (dvw_set_weight_quant)."""
        _check(_lib.dvw_set_weight_quant(self._h, int(bits), QUANT_SCHEMES[scheme]))
        return self

    def set_sampler(self, kind="direct", temperature: float = 1.0, top_k: int = 256):
        """App. A.4 strategy for generate(): "direct", "temperature", "mean", "mode", "top_k"."""
        if isinstance(kind, str):
            kind = SAMPLERS[kind]
        _check(_lib.dvw_set_sampler(self._h, int(kind), float(temperature), int(top_k)))
        return self

    def session(self, n_streams: int = 1) -> "Session":
        """A streaming session: generate one utterance chunk by chunk (dvw_session_*)."""
        return Session(self, n_streams)

    def set_trace(self, buf=None, first_sample: int = 0):
        """Record per-event %globaltimer stamps into a CUDA uint64/int64 tensor
        [n][16][32] (see include/dvw.h dvw_set_trace); None disables."""
        if buf is None:
            _check(_lib.dvw_set_trace(self._h, None, 0, 0))
        else:
            _check(_lib.dvw_set_trace(self._h, buf.data_ptr(), first_sample, int(buf.shape[0])))
        self._trace = buf
        return self

    def info(self) -> dict:
        i = _Info()
        _check(_lib.dvw_get_info(self._h, ctypes.byref(i)))
        d = {f: getattr(i, f) for f, _ in _Info._fields_}
        d["last_kernel_name"] = KERNEL_NAMES.get(d["last_kernel"], "?")
        return d

    def sync(self):
        _check(_lib.dvw_sync(self._h))

    def generate(self, cond, uniforms, hop: int, out=None, stream=None):
        """cond float32 [S][F][l][2r], uniforms float32 [S][N] (CUDA) -> uint8 [S][N]."""
        import torch
        S, F = int(cond.shape[0]), int(cond.shape[1])
        N = int(uniforms.shape[-1])
        if out is None:
            out = torch.empty((S, N), dtype=torch.uint8, device=cond.device)
        _check(_lib.dvw_generate(self._h, _dptr(cond, torch.float32, "cond"), F, hop,
                                 _dptr(uniforms, torch.float32, "uniforms"), N, S,
                                 _dptr(out, torch.uint8, "out"), _stream_handle(stream)))
        return out

    def logits(self, cond, codes, hop: int, out=None, stream=None):
        """Teacher-forced: codes uint8 [S][N] (CUDA) -> float32 [S][N][256] pre-softmax."""
        import torch
        S, F = int(cond.shape[0]), int(cond.shape[1])
        N = int(codes.shape[-1])
        if out is None:
            out = torch.empty((S, N, self.levels), dtype=torch.float32, device=cond.device)
        _check(_lib.dvw_logits(self._h, _dptr(cond, torch.float32, "cond"), F, hop,
                               _dptr(codes, torch.uint8, "codes"), N, S,
                               _dptr(out, torch.float32, "out"), _stream_handle(stream)))
        return out

    def generate_host(self, cond: np.ndarray, uniforms: np.ndarray, hop: int, out=None, stream=None):
        """Host (numpy, optionally pinned torch CPU) buffers in and out; synchronous."""
        def hptr(a):
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        S, F = int(cond.shape[0]), int(cond.shape[1])
        N = int(uniforms.shape[-1])
        if out is None:
            out = np.empty((S, N), dtype=np.uint8)
        _check(_lib.dvw_generate_host(self._h, hptr(cond), F, hop, hptr(uniforms), N, S, hptr(out),
                                      _stream_handle(stream)))
        return out


def measure_floor(device: int = 0) -> dict:
    """dvw_measure_floor: cycles of the batch-1 critical path's pieces on `device`."""
    f = _Floor()
    _check(_lib.dvw_measure_floor(int(device), ctypes.byref(f)))
    return {k: getattr(f, k) for k, _ in _Floor._fields_}


def raw_call(name: str, *args) -> int:
    """Direct access for the ABI negative tests."""
    return int(getattr(_lib, name)(*args))


def last_error() -> str:
    return (_lib.dvw_last_error() or b"").decode()


def conditioner_numel(in_channels: int, hidden: int, n_layers: int, residual: int) -> int:
    cfg = _CConfig(in_channels, hidden, n_layers, residual, 0)
    return int(_lib.dvwc_weights_numel(ctypes.byref(cfg)))


class Conditioner:
    """Handle on the GPU conditioning network (dvwc_*, include/dvw.h; App. A.2):
    features [S][T][in_channels] (CUDA fp32) -> cond [S][T][n_layers][2 residual] for
    Model.generate."""

    def __init__(self, in_channels: int, hidden: int, n_layers: int, residual: int, device: int = 0):
        cfg = _CConfig(in_channels, hidden, n_layers, residual, device)
        h = _vp()
        _check(_lib.dvwc_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.in_channels, self.hidden, self.n_layers, self.residual = in_channels, hidden, n_layers, residual
        self.numel = int(_lib.dvwc_weights_numel(ctypes.byref(cfg)))

    def close(self):
        if getattr(self, "_h", None):
            _lib.dvwc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, blob):
        if isinstance(blob, np.ndarray):
            b = np.ascontiguousarray(blob, dtype=np.float32)
            _check(_lib.dvwc_load_weights(self._h, b.ctypes.data, b.size, 0))
        else:
            _check(_lib.dvwc_load_weights(self._h, _dptr(blob, blob.dtype, "blob"), blob.numel(), 1))
        return self

    def run(self, features, out=None, stream=None):
        import torch
        S, T = int(features.shape[0]), int(features.shape[1])
        if out is None:
            out = torch.empty((S, T, self.n_layers, 2 * self.residual), dtype=torch.float32, device=features.device)
        _check(_lib.dvwc_run(self._h, _dptr(features, torch.float32, "features"), T, S,
                             _dptr(out, torch.float32, "out"), _stream_handle(stream)))
        return out


class Session:
    """dvw_session_*: consecutive chunks of the same utterances, bitwise equal to one call."""

    def __init__(self, model: "Model", n_streams: int = 1):
        h = _vp()
        _check(_lib.dvw_session_create(model._h, int(n_streams), ctypes.byref(h)))
        self._h, self.model, self.n_streams = h, model, n_streams

    @property
    def position(self) -> int:
        return int(_lib.dvw_session_position(self._h))

    def generate(self, cond, uniforms, hop: int, out=None, stream=None):
        """cond: the WHOLE utterance's conditioning [S][F][l][2r]; uniforms: this chunk's [S][n]."""
        import torch
        S, F = int(cond.shape[0]), int(cond.shape[1])
        n = int(uniforms.shape[-1])
        if out is None:
            out = torch.empty((S, n), dtype=torch.uint8, device=cond.device)
        _check(_lib.dvw_session_generate(self.model._h, self._h, _dptr(cond, torch.float32, "cond"), F, hop,
                                         _dptr(uniforms, torch.float32, "uniforms"), n,
                                         _dptr(out, torch.uint8, "out"), _stream_handle(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.dvw_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
