"""Thin ctypes binding of include/deepinverse.h (argument marshalling only).

Every step of the recovery runs inside libdeepinverse.so (hand-written sm_100a kernels).  There is no
Python or CPU compute path: if the library is missing this module raises ImportError-like errors
instead of falling back.  PyTorch is used only for device memory and streams (tensors' data_ptr()
and torch.cuda streams are passed through as raw pointers).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DI_LIB selects another build (the experiment library libdeepinverse_exp.so, build.py); default: the product library
LIB_PATH = os.environ.get("DI_LIB") or os.path.join(_HERE, "libdeepinverse.so")

DI_OK, DI_ERR_ARG, DI_ERR_DIM, DI_ERR_DOMAIN, DI_ERR_DEVICE, DI_ERR_OOM, DI_ERR_CUDA = range(7)
DI_PREC_FP32, DI_PREC_TF32, DI_PREC_BF16 = 0, 1, 2
DI_DTYPE_F32, DI_DTYPE_BF16 = 0, 1
DI_FLAG_XCORR, DI_FLAG_FULLMAP_BIAS, DI_FLAG_FINAL_RELU = 1, 2, 4
PRECISIONS = {"f32": DI_PREC_FP32, "tf32": DI_PREC_TF32, "bf16": DI_PREC_BF16}

# every symbol include/deepinverse.h declares (checked by tests/test_abi.py)
EXPORTS = ["di_create", "di_recover", "di_recover_host", "di_destroy", "di_status_string", "di_last_error",
           "di_get_info", "di_set_profiling", "di_stage_times", "di_debug_stage", "di_debug_get_phi",
           "di_measure", "di_add_noise", "di_metrics", "di_recover_metrics", "di_num_params", "di_ctx_num_params", "di_train_grad", "di_sgd_step",
           "di_get_params", "di_proxy_partial", "di_recover_from_proxy", "di_proxy_scatter", "di_recover_from_slots"]


class DiError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({_status_name(status)}): {detail}")
        self.status = status


def _status_name(s: int) -> str:
    names = ["DI_OK", "DI_ERR_ARG", "DI_ERR_DIM", "DI_ERR_DOMAIN", "DI_ERR_DEVICE", "DI_ERR_OOM", "DI_ERR_CUDA"]
    return names[s] if 0 <= s < len(names) else "?"


class di_layer(ctypes.Structure):
    _fields_ = [("cin", ctypes.c_int), ("cout", ctypes.c_int), ("w", ctypes.c_void_p), ("b", ctypes.c_void_p)]


class di_create_args(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("n1", ctypes.c_int), ("n2", ctypes.c_int),
                ("phi", ctypes.c_void_p), ("phi_dtype", ctypes.c_int),
                ("w1", ctypes.c_void_p), ("b1", ctypes.c_void_p),
                ("w2", ctypes.c_void_p), ("b2", ctypes.c_void_p),
                ("w3", ctypes.c_void_p), ("b3", ctypes.c_void_p),
                ("precision", ctypes.c_int), ("flags", ctypes.c_uint),
                ("device", ctypes.c_int), ("max_batch", ctypes.c_int), ("lift", ctypes.c_void_p),
                ("n_layers", ctypes.c_int), ("layers", ctypes.c_void_p)]


class di_info(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("n1", ctypes.c_int), ("n2", ctypes.c_int), ("max_batch", ctypes.c_int),
                ("precision", ctypes.c_int), ("flags", ctypes.c_uint), ("launches_per_recover", ctypes.c_int),
                ("workspace_bytes", ctypes.c_longlong), ("stage_kernels", ctypes.c_char_p * 4)]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libdeepinverse.so (build it first with paper_1701_03891_b200.build.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built: run `python -m paper_1701_03891_b200.build` "
                                "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    V, I, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
    lib.di_create.argtypes = [ctypes.POINTER(di_create_args), ctypes.POINTER(V)]
    lib.di_recover.argtypes = [V, V, LL, I, V, V]
    lib.di_recover_host.argtypes = [V, V, LL, I, V, V]
    lib.di_destroy.argtypes = [V]
    lib.di_status_string.argtypes = [I]
    lib.di_status_string.restype = ctypes.c_char_p
    lib.di_last_error.argtypes = []
    lib.di_last_error.restype = ctypes.c_char_p
    lib.di_get_info.argtypes = [V, ctypes.POINTER(di_info)]
    lib.di_set_profiling.argtypes = [V, I]
    lib.di_stage_times.argtypes = [V, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(I), I]
    lib.di_debug_stage.argtypes = [V, I, V, V, I, V]
    lib.di_debug_get_phi.argtypes = [V, V, LL]
    lib.di_measure.argtypes = [V, V, I, V, LL, V]
    lib.di_add_noise.argtypes = [V, V, LL, I, ctypes.c_double, ctypes.c_ulonglong, V]
    lib.di_metrics.argtypes = [V, V, V, I, V, V]
    lib.di_recover_metrics.argtypes = [V, V, LL, I, V, V, V, V]
    lib.di_num_params.argtypes = []
    lib.di_num_params.restype = LL
    lib.di_ctx_num_params.argtypes = [V]
    lib.di_ctx_num_params.restype = LL
    lib.di_train_grad.argtypes = [V, V, LL, V, I, ctypes.c_double, V, V, V]
    lib.di_sgd_step.argtypes = [V, V, ctypes.c_double, ctypes.c_double, V]
    lib.di_get_params.argtypes = [V, V, V]
    lib.di_proxy_partial.argtypes = [V, V, LL, I, V, V]
    lib.di_recover_from_proxy.argtypes = [V, V, I, V, V]
    lib.di_proxy_scatter.argtypes = [V, V, LL, I, V, I, I, V]
    lib.di_recover_from_slots.argtypes = [V, V, I, I, V, V]
    for f in ("di_create", "di_recover", "di_recover_host", "di_destroy", "di_get_info", "di_set_profiling",
              "di_stage_times", "di_debug_stage", "di_debug_get_phi", "di_measure", "di_add_noise", "di_metrics", "di_recover_metrics",
              "di_train_grad", "di_sgd_step", "di_get_params", "di_proxy_partial", "di_recover_from_proxy", "di_proxy_scatter",
              "di_recover_from_slots"):
        getattr(lib, f).restype = I
    _lib = lib
    return lib


def _check(status: int, where: str):
    if status != DI_OK:
        raise DiError(status, where, load().di_last_error().decode(errors="replace"))


def _ptr(a) -> int | None:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor
        return a.data_ptr()
    if isinstance(a, int):      # raw device pointer (e.g. a cudaMalloc'd staging buffer)
        return a
    return a.ctypes.data


def _stream_handle(stream, device: int | None = None) -> int | None:
    """The raw cudaStream_t: `stream` (torch.cuda.Stream or int), else torch's current stream of `device` (the
    context's device; torch's current device when None)."""
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream(device).cuda_stream
        except Exception:  # pragma: no cover
            return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


# ------------------------------------------------------------------ same names as the C ABI
def di_create(args: di_create_args) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(load().di_create(ctypes.byref(args), ctypes.byref(h)), "di_create")
    return h


def di_recover(ctx, y, ldy: int, batch: int, xhat, stream=None):
    _check(load().di_recover(ctx, _ptr(y), ldy, batch, _ptr(xhat), _stream_handle(stream)), "di_recover")


def di_recover_host(ctx, y_host, ldy: int, batch: int, xhat_host, stream=None):
    _check(load().di_recover_host(ctx, _ptr(y_host), ldy, batch, _ptr(xhat_host), _stream_handle(stream)),
           "di_recover_host")


def di_proxy_partial(ctx, y, ldy: int, batch: int, xt_part, stream=None):
    _check(load().di_proxy_partial(ctx, _ptr(y), ldy, batch, _ptr(xt_part), _stream_handle(stream)),
           "di_proxy_partial")


def di_recover_from_proxy(ctx, xt, batch: int, xhat, stream=None):
    _check(load().di_recover_from_proxy(ctx, _ptr(xt), batch, _ptr(xhat), _stream_handle(stream)),
           "di_recover_from_proxy")


def di_proxy_scatter(ctx, y, ldy: int, batch: int, slots, world: int, rank: int, stream=None):
    """slots: sequence of `world` device pointers (ints)."""
    arr = (ctypes.c_void_p * world)(*[int(p) for p in slots])
    _check(load().di_proxy_scatter(ctx, _ptr(y), ldy, batch, arr, world, rank, _stream_handle(stream)),
           "di_proxy_scatter")


def di_recover_from_slots(ctx, staging, world: int, nb: int, xhat, stream=None):
    _check(load().di_recover_from_slots(ctx, _ptr(staging), world, nb, _ptr(xhat), _stream_handle(stream)),
           "di_recover_from_slots")


def di_destroy(ctx):
    _check(load().di_destroy(ctx), "di_destroy")


def di_debug_stage(ctx, stage: int, x_in, x_out, batch: int, stream=None):
    _check(load().di_debug_stage(ctx, stage, _ptr(x_in), _ptr(x_out), batch, _stream_handle(stream)),
           "di_debug_stage")


def di_measure(ctx, x, batch: int, y, ldy: int, stream=None):
    _check(load().di_measure(ctx, _ptr(x), batch, _ptr(y), ldy, _stream_handle(stream)), "di_measure")


def di_add_noise(ctx, y, ldy: int, batch: int, snr_db: float, seed: int, stream=None):
    _check(load().di_add_noise(ctx, _ptr(y), ldy, batch, float(snr_db), int(seed), _stream_handle(stream)),
           "di_add_noise")


def di_metrics(ctx, xhat, x, batch: int, out, stream=None):
    _check(load().di_metrics(ctx, _ptr(xhat), _ptr(x), batch, _ptr(out), _stream_handle(stream)), "di_metrics")


def di_recover_metrics(ctx, y, ldy: int, batch: int, x_true, xhat, metrics, stream=None):
    _check(load().di_recover_metrics(ctx, _ptr(y), ldy, batch, _ptr(x_true), _ptr(xhat), _ptr(metrics),
                                     _stream_handle(stream)), "di_recover_metrics")


def di_num_params() -> int:
    return int(load().di_num_params())


def di_train_grad(ctx, y, ldy: int, x_true, batch: int, scale: float, grads, loss, stream=None):
    _check(load().di_train_grad(ctx, _ptr(y), ldy, _ptr(x_true), batch, float(scale), _ptr(grads), _ptr(loss),
                                _stream_handle(stream)), "di_train_grad")


def di_sgd_step(ctx, grads, lr: float, momentum: float = 0.0, stream=None):
    _check(load().di_sgd_step(ctx, _ptr(grads), float(lr), float(momentum), _stream_handle(stream)), "di_sgd_step")


def di_get_params(ctx, params, stream=None):
    _check(load().di_get_params(ctx, _ptr(params), _stream_handle(stream)), "di_get_params")


def di_status_string(s: int) -> str:
    return load().di_status_string(s).decode()


def di_last_error() -> str:
    return load().di_last_error().decode(errors="replace")


# ------------------------------------------------------------------ convenience owner object
class DeepInverse:
    """Owns one di_ctx.  phi: [m][n1*n2] (fp32 numpy; bf16 configs pass bf16-representable values),
    params: synth.Params-like (w: arrays [C_out][C_in][11][11], b: per-channel or full-map biases).  The paper's
    three layers (64, 32, 1) use w1..b3; any other stack (widths per include/deepinverse.h)
    is passed as di_create_args.layers."""

    def __init__(self, phi: np.ndarray, params, n1: int, n2: int, precision: str = "bf16", flags: int = 0,
                 device: int = 0, max_batch: int = 1, lift: np.ndarray | None = None):
        load()
        phi = np.ascontiguousarray(phi, dtype=np.float32)
        self.m = phi.shape[0]
        self.N = phi.shape[1]
        self.n1, self.n2, self.precision, self.max_batch = n1, n2, precision, max_batch
        self.device = device
        ws = [np.ascontiguousarray(w, np.float32) for w in params.w]
        has_bias = params.b is not None and any(np.any(np.asarray(b) != 0) for b in params.b)
        bs = [np.ascontiguousarray(b, np.float32) for b in params.b] if has_bias else [None, None, None]
        if getattr(params, "fullmap_bias", False) and has_bias:
            flags |= DI_FLAG_FULLMAP_BIAS
        self.flags = flags
        lift = None if lift is None else np.ascontiguousarray(lift, dtype=np.float32)
        if lift is not None and lift.shape != (phi.shape[1], phi.shape[0]):
            raise ValueError(f"lift must be [N][m] = {(phi.shape[1], phi.shape[0])}")
        widths = tuple(w.shape[0] for w in ws)
        self.shapes = [tuple(w.shape) for w in ws]
        self.custom = len(ws) != 3 or widths != (64, 32, 1)
        if self.custom:
            if len(bs) < len(ws):
                bs = [None] * len(ws)
            arr = (di_layer * len(ws))(*[di_layer(w.shape[1], w.shape[0], w.ctypes.data, _ptr(b))
                                         for w, b in zip(ws, bs)])
            self._keep = (phi, ws, bs, lift, arr)
            a = di_create_args(self.m, n1, n2, phi.ctypes.data, DI_DTYPE_F32, None, None, None, None, None, None,
                               PRECISIONS[precision], flags, device, max_batch, _ptr(lift), len(ws),
                               ctypes.cast(arr, ctypes.c_void_p))
        else:
            self._keep = (phi, ws, bs, lift)
            a = di_create_args(self.m, n1, n2, phi.ctypes.data, DI_DTYPE_F32,
                               ws[0].ctypes.data, _ptr(bs[0]), ws[1].ctypes.data, _ptr(bs[1]),
                               ws[2].ctypes.data, _ptr(bs[2]), PRECISIONS[precision], flags, device, max_batch,
                               _ptr(lift), 0, None)
        self.ctx = di_create(a)
        self._keep = None

    @property
    def storage_dtype(self):
        import torch
        return torch.bfloat16 if self.precision == "bf16" else torch.float32

    def _check_y(self, y):
        if not hasattr(y, "is_cuda") or y.dtype != self.storage_dtype or not y.is_cuda:
            raise TypeError(f"y must be a CUDA {self.storage_dtype} tensor")
        if y.device.index != self.device:
            raise TypeError(f"y is on {y.device}, the context on cuda:{self.device}")
        if y.dim() != 2 or y.shape[1] != self.m or y.stride(1) != 1:
            raise TypeError(f"y must be [B][{self.m}] with unit column stride (rows may be padded), got "
                            f"{tuple(y.shape)} strides {y.stride()}")

    def _check_out(self, t, shape, what):
        import torch
        if (t.dtype != torch.float32 or not t.is_cuda or t.device.index != self.device or not t.is_contiguous()
                or tuple(t.shape) != tuple(shape)):
            raise TypeError(f"{what} must be a contiguous float32 tensor {tuple(shape)} on cuda:{self.device}")

    def _stream(self, stream):
        return _stream_handle(stream, self.device)

    def recover(self, y, xhat=None, stream=None):
        """y: device tensor [B][ldy] of the storage dtype; returns x_hat [B][n1][n2] fp32 (device)."""
        import torch
        self._check_y(y)
        b = y.shape[0]
        if xhat is None:
            xhat = torch.empty((b, self.n1, self.n2), dtype=torch.float32, device=y.device)
        self._check_out(xhat, (b, self.n1, self.n2), "xhat")
        di_recover(self.ctx, y, y.stride(0), b, xhat, self._stream(stream))
        return xhat

    def proxy_partial(self, y, out=None, stream=None):
        """Row-sharded lifting (NEXT-4): y device [B][ldy] over this context's rows of Phi -> fp32 partial
        x_tilde [B][n1*n2] (device), to be summed across ranks."""
        import torch
        if y.dtype != self.storage_dtype or not y.is_cuda:
            raise TypeError(f"y must be a CUDA {self.storage_dtype} tensor")
        b = y.shape[0]
        if out is None:
            out = torch.empty((b, self.n1 * self.n2), dtype=torch.float32, device=y.device)
        di_proxy_partial(self.ctx, y, y.stride(0), b, out, self._stream(stream))
        return out

    def recover_from_proxy(self, xt, xhat=None, stream=None):
        """Convolutions on a (summed) fp32 proxy x_tilde [B][n1*n2] (device) -> x_hat [B][n1][n2] fp32."""
        import torch
        if xt.dtype != torch.float32 or not xt.is_cuda or not xt.is_contiguous():
            raise TypeError("xt must be a contiguous CUDA float32 tensor [B][n1*n2]")
        b = xt.shape[0]
        if xhat is None:
            xhat = torch.empty((b, self.n1, self.n2), dtype=torch.float32, device=xt.device)
        di_recover_from_proxy(self.ctx, xt, b, xhat, self._stream(stream))
        return xhat

    def proxy_scatter(self, y, slots, world: int, rank: int, stream=None):
        """Row-sharded lifting with the reduce-scatter in the GEMM epilogue (NEXT-4): the partial rows of image b go
        to slots[b // nb] (device pointers: the owners' [world][nb][N] fp32 staging buffers, peer-mapped)."""
        if y.dtype != self.storage_dtype or not y.is_cuda:
            raise TypeError(f"y must be a CUDA {self.storage_dtype} tensor")
        di_proxy_scatter(self.ctx, y, y.stride(0), y.shape[0], slots, world, rank, self._stream(stream))

    def recover_from_slots(self, staging, world: int, xhat=None, stream=None):
        """Owner side: x_tilde = sum of the world slots of `staging` [world][nb][N] fp32 (rank order), then the convs."""
        import torch
        nb = staging.shape[1]
        if xhat is None:
            xhat = torch.empty((nb, self.n1, self.n2), dtype=torch.float32, device=staging.device)
        di_recover_from_slots(self.ctx, staging, world, nb, xhat, self._stream(stream))
        return xhat

    def recover_host(self, y_host, xhat_host=None, stream=None):
        """End-to-end: host y (numpy or CPU torch tensor, [B][m] of the storage dtype, unit column stride; pinned
        memory gives the fast copies) -> host x_hat fp32 [B][n1][n2] (numpy or CPU torch, contiguous)."""
        if hasattr(y_host, "is_cuda"):            # torch
            import torch
            if y_host.is_cuda or y_host.dtype != self.storage_dtype:
                raise TypeError(f"y_host must be a CPU {self.storage_dtype} tensor")
            if y_host.dim() != 2 or y_host.shape[1] != self.m or y_host.stride(1) != 1:
                raise TypeError(f"y_host must be [B][{self.m}] with unit column stride")
            ldy = y_host.stride(0)
        else:
            if self.precision == "bf16":
                raise TypeError("a bf16 context takes y_host as a CPU torch.bfloat16 tensor (numpy has no bf16)")
            y_host = np.asarray(y_host)
            if y_host.dtype != np.float32 or y_host.ndim != 2 or y_host.shape[1] != self.m or \
                    y_host.strides[1] != 4:
                raise TypeError(f"y_host must be float32 [B][{self.m}] with unit column stride")
            ldy = y_host.strides[0] // 4
        b = y_host.shape[0]
        if xhat_host is None:
            xhat_host = np.empty((b, self.n1, self.n2), np.float32)
        if hasattr(xhat_host, "is_cuda"):
            import torch
            ok = (not xhat_host.is_cuda and xhat_host.dtype == torch.float32 and xhat_host.is_contiguous() and
                  tuple(xhat_host.shape) == (b, self.n1, self.n2))
        else:
            ok = (isinstance(xhat_host, np.ndarray) and xhat_host.dtype == np.float32 and
                  xhat_host.flags.c_contiguous and xhat_host.shape == (b, self.n1, self.n2))
        if not ok:
            raise TypeError(f"xhat_host must be a contiguous host float32 array {(b, self.n1, self.n2)}")
        di_recover_host(self.ctx, y_host, ldy, b, xhat_host, self._stream(stream))
        return xhat_host

    def measure(self, x, y=None, stream=None):
        """y = Phi x: x device fp32 [B][n1][n2] -> y device [B][m] in the storage dtype."""
        import torch
        if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
            raise TypeError("x must be a contiguous CUDA float32 tensor [B][n1][n2]")
        b = x.shape[0]
        if y is None:
            y = torch.empty((b, self.m), dtype=self.storage_dtype, device=x.device)
        di_measure(self.ctx, x, b, y, y.stride(0), self._stream(stream))
        return y

    def add_noise(self, y, snr_db: float, seed: int, stream=None):
        """In place: y_b += N(0, ||y_b||^2 / (m 10^(snr/10))) noise (Table 3 reading, Q14)."""
        di_add_noise(self.ctx, y, y.stride(0), y.shape[0], snr_db, seed, self._stream(stream))
        return y

    def metrics(self, xhat, x, stream=None):
        """Per-image PSNR, NMSE and success on the device, fp64: [3][B] numpy."""
        import torch
        b = x.shape[0]
        out = torch.empty((3, b), dtype=torch.float64, device=x.device)
        di_metrics(self.ctx, xhat, x, b, out, self._stream(stream))
        return out.cpu().numpy()

    def recover_metrics(self, y, x, xhat=None, stream=None):
        """x_hat = M(y) and, per image, PSNR / NMSE / success against the ground truth x (device fp32 [B][n1][n2]);
        fused into conv layer 3's epilogue on the BF16 path.  Returns (x_hat device tensor, metrics numpy [3][B])."""
        import torch
        self._check_y(y)
        b = y.shape[0]
        self._check_out(x, (b, self.n1, self.n2), "x")
        if xhat is None:
            xhat = torch.empty((b, self.n1, self.n2), dtype=torch.float32, device=y.device)
        self._check_out(xhat, (b, self.n1, self.n2), "xhat")
        out = torch.empty((3, b), dtype=torch.float64, device=y.device)
        di_recover_metrics(self.ctx, y, y.stride(0), b, x, xhat, out, self._stream(stream))
        return xhat, out.cpu().numpy()

    # ------------------------------------------------------------ training (NEXT-2; paper stack, per-channel biases)
    def train_grad(self, y, x, scale=None, grads=None, stream=None):
        """Loss scale * sum ||M(y) - x||^2 (scale defaults to 1/batch) and its gradient (device fp32
        [di_num_params()]).  y: device [B][ldy] of the storage dtype; x: device fp32 [B][n1][n2].
        Returns (loss tensor (device, float64 [1]), grads)."""
        import torch
        if y.dtype != self.storage_dtype or not y.is_cuda:
            raise TypeError(f"y must be a CUDA {self.storage_dtype} tensor")
        b = y.shape[0]
        if grads is None:
            grads = torch.empty(self.num_params(), dtype=torch.float32, device=y.device)
        loss = torch.empty(1, dtype=torch.float64, device=y.device)
        di_train_grad(self.ctx, y, y.stride(0), x, b, 1.0 / b if scale is None else scale, grads, loss, self._stream(stream))
        return loss, grads

    def sgd_step(self, grads, lr: float, momentum: float = 0.0, stream=None):
        di_sgd_step(self.ctx, grads, lr, momentum, self._stream(stream))

    def num_params(self) -> int:
        """Length of this context's parameter vector (include/deepinverse.h: di_ctx_num_params)."""
        return int(load().di_ctx_num_params(self.ctx))

    def params(self, stream=None):
        """Current parameters as numpy arrays ([W_0, ...], [b_0, ...]) in the orientation given at creation."""
        import torch
        p = torch.empty(self.num_params(), dtype=torch.float32, device=f"cuda:{self.device}")
        di_get_params(self.ctx, p, self._stream(stream))
        return split_params(p.cpu().numpy(), self.shapes)

    def split(self, flat):
        """[W_0 | ... | W_L-1 | b_0 | ... | b_L-1] -> ([W_0, ...], [b_0, ...]) (views)."""
        return split_params(np.asarray(flat), self.shapes)

    def debug_stage(self, stage: int, x_in, x_out, batch: int, stream=None):
        di_debug_stage(self.ctx, stage, x_in, x_out, batch, self._stream(stream))

    def info(self) -> dict:
        inf = di_info()
        _check(load().di_get_info(self.ctx, ctypes.byref(inf)), "di_get_info")
        return {"m": inf.m, "n1": inf.n1, "n2": inf.n2, "max_batch": inf.max_batch, "precision": inf.precision,
                "flags": inf.flags, "launches_per_recover": inf.launches_per_recover,
                "workspace_bytes": inf.workspace_bytes,
                "stage_kernels": [s.decode() if s else "" for s in inf.stage_kernels]}

    def set_profiling(self, on: bool):
        _check(load().di_set_profiling(self.ctx, int(on)), "di_set_profiling")

    def stage_times(self, reset: bool = False):
        ms = (ctypes.c_float * 4)()
        calls = ctypes.c_int()
        _check(load().di_stage_times(self.ctx, ms, ctypes.byref(calls), int(reset)), "di_stage_times")
        return list(ms), calls.value

    def phi_device_copy(self) -> np.ndarray:
        elt = 2 if self.precision == "bf16" else 4
        out = np.empty(self.m * self.n1 * self.n2 * elt, np.uint8)
        _check(load().di_debug_get_phi(self.ctx, out.ctypes.data, out.nbytes), "di_debug_get_phi")
        return out.view(np.uint16 if elt == 2 else np.float32).reshape(self.m, self.n1 * self.n2)

    def close(self):
        if getattr(self, "ctx", None):
            di_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PARAM_SHAPES = [(64, 1, 11, 11), (32, 64, 11, 11), (1, 32, 11, 11)]


def split_params(flat, shapes=None):
    """[W_0 | ... | W_L-1 | b_0 | ... | b_L-1] -> ([W_0, ...], [b_0, ...]) (views of `flat`); the paper's stack by
    default."""
    shapes = PARAM_SHAPES if shapes is None else shapes
    ws, o = [], 0
    for sh in shapes:
        n = int(np.prod(sh))
        ws.append(flat[o:o + n].reshape(sh))
        o += n
    bs = []
    for sh in shapes:
        bs.append(flat[o:o + sh[0]])
        o += sh[0]
    return ws, bs
