"""paper_1809_07851_b200 -- B200-native tiled fast-convolution forward pass.

Thin ctypes binding over the C-ABI in ``include/fastconv.h`` (argument
marshalling only: every stage runs in the hand-written sm_100a kernels of
``libfastconv.so``).  PyTorch supplies device memory and the current stream.
There is no CPU fallback: if the library is missing or a call fails, this
module raises.

Methods: ``"winograd"`` F(m^2, r^2) (Eq. 1/4),
``"regular_fft"`` (Eq. 2), ``"gauss_fft"`` and the
``"direct"`` check path.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

from . import _build

_PKG = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(_PKG), "include", "fastconv.h")

METHODS = {"direct": 0, "winograd": 1, "regular_fft": 2, "gauss_fft": 3}
GEMMS = {"auto": 0, "tcgen05": 1, "ffma": 2, "f16x3": 3}
GEMM_NAMES = {0: "auto", 1: "tcgen05_3xtf32", 2: "ffma", 3: "tcgen05_f16x3"}
STATUS = {0: "CONV_OK", 1: "CONV_ERR_INVALID_ARG", 2: "CONV_ERR_UNSUPPORTED",
          3: "CONV_ERR_OUT_OF_MEMORY", 4: "CONV_ERR_CUDA", 5: "CONV_ERR_DEVICE_MISMATCH"}


class ConvError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__("%s: %s" % (STATUS.get(status, status), detail))


class PlanOptions(ctypes.Structure):
    """conv_plan_options (include/fastconv.h): every plan choice besides the layer shape."""
    _fields_ = [("struct_size", ctypes.c_int), ("gemm", ctypes.c_int), ("gauss_combine", ctypes.c_int),
                ("complex_mode", ctypes.c_int), ("chunk_images", ctypes.c_int),
                ("generic_transforms", ctypes.c_int), ("single_cta_mma", ctypes.c_int),
                ("e2e_chunks", ctypes.c_int), ("overlap_kernel_transform", ctypes.c_int),
                ("fused", ctypes.c_int)]


def options(gemm: str = "auto", **kw) -> PlanOptions:
    """conv_plan_options_init() defaults, then ``gemm`` and any field given by name."""
    o = PlanOptions()
    load().conv_plan_options_init(ctypes.byref(o))
    o.gemm = GEMMS[gemm]
    for k, v in kw.items():
        if k not in dict(PlanOptions._fields_):
            raise TypeError("unknown plan option %r" % k)
        setattr(o, k, int(v))
    return o


class PlanInfo(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_int) for n in
                 ("B", "C", "Cout", "H", "W", "r", "m", "method", "Ho", "Wo", "t", "n_h", "n_w",
                  "N", "h", "E", "planes")] +
                [("BN", ctypes.c_longlong), ("BN_pad", ctypes.c_longlong)] +
                [(n, ctypes.c_int) for n in ("gemm_Z", "gemm_M", "gemm_K")] +
                [(n, ctypes.c_size_t) for n in ("bytes_U", "bytes_V", "bytes_X", "workspace_bytes")] +
                [("alg_bytes", ctypes.c_double * 4), ("alg_flops", ctypes.c_double * 4),
                 ("direct_flops", ctypes.c_double), ("chunk", ctypes.c_int), ("nchunks", ctypes.c_int),
                 ("gemm", ctypes.c_int), ("nd", ctypes.c_int)] +
                [(n, ctypes.c_int * 3) for n in ("in_shape", "kernel_shape", "m_shape", "t_shape", "tiles",
                                                 "out_shape")] +
                [("x_planes", ctypes.c_int), ("fused", ctypes.c_int)])

    def as_dict(self) -> dict:
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if isinstance(v, ctypes.Array) else v
        return d


_lib = None


def library_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = False):
    """Load libfastconv.so (raise if absent: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB):
        if not build_if_missing:
            raise RuntimeError("libfastconv.so is not built; run __graft_entry__.build() "
                               "(or python paper_1809_07851_b200/_build.py)")
        _build.build()
    lib = ctypes.CDLL(_build.LIB)
    vp, i, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    dp = ctypes.POINTER(ctypes.c_double)
    fp = ctypes.POINTER(ctypes.c_float)
    sigs = {
        "conv_plan_query": ([i] * 8 + [ctypes.POINTER(PlanInfo)], i),
        "conv_plan_query_opts": ([i] * 8 + [ctypes.POINTER(PlanOptions), ctypes.POINTER(PlanInfo)], i),
        "conv_plan_options_init": ([ctypes.POINTER(PlanOptions)], None),
        "conv_plan_best_m": ([i] * 7 + [ctypes.POINTER(PlanOptions), ctypes.POINTER(i), dp, i,
                                        ctypes.POINTER(i), ctypes.POINTER(i), dp], i),
        "conv_plan_best_method": ([i] * 6 + [ctypes.POINTER(PlanOptions), ctypes.POINTER(i), ctypes.POINTER(i),
                                          dp], i),
        "conv_plan": ([ctypes.POINTER(vp)] + [i] * 8, i),
        "conv_plan_ex": ([ctypes.POINTER(vp)] + [i] * 9, i),
        "conv_plan_opts": ([ctypes.POINTER(vp)] + [i] * 8 + [ctypes.POINTER(PlanOptions)], i),
        "conv_plan_nd": ([ctypes.POINTER(vp)] + [i] * 4 + [ctypes.POINTER(i), ctypes.POINTER(i), i,
                                                           ctypes.POINTER(i), ctypes.POINTER(PlanOptions)], i),
        "conv_plan_query_nd": ([i] * 4 + [ctypes.POINTER(i), ctypes.POINTER(i), i, ctypes.POINTER(i),
                                          ctypes.POINTER(PlanOptions), ctypes.POINTER(PlanInfo)], i),
        "conv_plan_get_info": ([vp, ctypes.POINTER(PlanInfo)], i),
        "conv_workspace_bytes": ([vp], sz),
        "conv_forward": ([vp, vp, vp, vp, vp, sz, vp], i),
        "conv_forward_profiled": ([vp, vp, vp, vp, vp, sz, vp, fp], i),
        "conv_forward_host": ([vp, vp, vp, vp, vp, vp, vp, vp, sz, vp], i),
        "conv_run_stage": ([vp, i, vp, vp, vp, vp, sz, vp], i),
        "conv_workspace_layout": ([vp, ctypes.POINTER(sz)], i),
        "conv_workspace_aux": ([vp, ctypes.POINTER(sz)], i),
        "conv_plan_winograd_matrices": ([vp, dp, dp, dp], i),
        "conv_winograd_matrices": ([i, i, dp, dp, dp], i),
        "conv_destroy": ([vp], None),
        "conv_status_string": ([i], ctypes.c_char_p),
        "conv_last_error": ([], ctypes.c_char_p),
        "conv_forward_launch_count": ([vp], i),
        "conv_transform_weights": ([vp, vp, vp, sz, vp], i),
        "conv_forward_cached": ([vp, vp, vp, vp, sz, vp], i),
        "conv_timer_create": ([ctypes.POINTER(vp), i], i),
        "conv_forward_timed": ([vp, vp, vp, vp, vp, sz, vp, vp], i),
        "conv_timer_read": ([vp, fp, ctypes.POINTER(i)], i),
        "conv_timer_reset": ([vp], None),
        "conv_timer_destroy": ([vp], None),
        "conv_graph_create": ([vp, vp, vp, vp, vp, sz, i, i, ctypes.POINTER(vp)], i),
        "conv_graph_launch": ([vp, vp], i),
        "conv_graph_destroy": ([vp], None),
        "conv_eshard_create": ([ctypes.POINTER(vp), i, i, ctypes.POINTER(i)] + [i] * 7 +
                               [ctypes.POINTER(PlanOptions)], i),
        "conv_eshard_sizes": ([vp] + [ctypes.POINTER(sz)] * 5, i),
        "conv_eshard_get_info": ([vp, ctypes.POINTER(PlanInfo), ctypes.POINTER(i), ctypes.POINTER(i)], i),
        "conv_eshard_forward_a": ([vp, vp, vp, vp, vp, vp, sz, vp], i),
        "conv_eshard_forward_b": ([vp, vp, vp, vp, vp, sz, vp], i),
        "conv_eshard_forward_c": ([vp, vp, vp, vp, sz, vp], i),
        "conv_eshard_destroy": ([vp], None),
        "conv_eshard_forward_a_peer": ([vp, vp, vp, ctypes.POINTER(vp), vp, vp, sz, vp], i),
        "conv_eshard_forward_b_peer": ([vp, vp, vp, ctypes.POINTER(vp), vp, sz, vp], i),
        "conv_ipc_alloc": ([sz, ctypes.POINTER(vp), vp], i),
        "conv_ipc_free": ([vp], i),
        "conv_ipc_open": ([vp, ctypes.POINTER(vp)], i),
        "conv_ipc_close": ([vp], i),
        "conv_plan_backward": ([ctypes.POINTER(vp)] + [i] * 9 + [ctypes.POINTER(PlanOptions)], i),
        "conv_backward_data": ([vp, vp, vp, vp, vp, sz, vp], i),
        "conv_backward_filter": ([vp, vp, vp, vp, vp, sz, vp], i),
    }
    for name, (args, res) in sigs.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def header_functions() -> list[str]:
    """Names of every function include/fastconv.h declares."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(conv_[a-z_]+)\s*\(", src)))


def _check(st: int):
    if st != 0:
        raise ConvError(st, load().conv_last_error().decode())


def plan_query(B, C, Cout, H, W, r, method: str, m: int = 0, gemm: str = "auto", **opts) -> dict:
    """conv_plan_query_opts: the geometry and algorithmic costs of the plan these options build
    (m = 0: the planner's tile)."""
    info = PlanInfo()
    o = options(gemm, **opts)
    _check(load().conv_plan_query_opts(B, C, Cout, H, W, r, METHODS[method], m, ctypes.byref(o), ctypes.byref(info)))
    return info.as_dict()


def best_method(B, C, Cout, H, W, r, gemm: str = "auto", **opts):
    """conv_plan_best_method: (method name, m, predicted ms) -- the paper's rule on
    the calibrated stage-sum model."""
    o = options(gemm, **opts)
    meth, m, ms = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    _check(load().conv_plan_best_method(B, C, Cout, H, W, r, ctypes.byref(o), ctypes.byref(meth), ctypes.byref(m),
                                        ctypes.byref(ms)))
    return {v: k for k, v in METHODS.items()}[meth.value], m.value, ms.value


def plan_query_nd(B, C, Cout, in_shape, kernel_shape, method: str, m=None, gemm: str = "auto", **opts) -> dict:
    """conv_plan_query_nd: geometry and algorithmic costs of an N-D / non-isotropic plan."""
    nd = len(in_shape)
    info = PlanInfo()
    o = options(gemm, **opts)
    ia = (ctypes.c_int * 3)(*in_shape)
    ka = (ctypes.c_int * 3)(*kernel_shape)
    ma = (ctypes.c_int * 3)(*(m or [1] * nd))
    _check(load().conv_plan_query_nd(nd, B, C, Cout, ia, ka, METHODS[method], ma, ctypes.byref(o), ctypes.byref(info)))
    return info.as_dict()


def best_m(B, C, Cout, H, W, r, method: str, gemm: str = "auto", **opts):
    """conv_plan_best_m: (m, predicted ms, {m: predicted ms}) from the paper's stage-sum model
    with B200 constants, over every compiled tile size."""
    o = options(gemm, **opts)
    m = ctypes.c_int()
    ms = ctypes.c_double()
    cap = 64
    n = ctypes.c_int()
    cm = (ctypes.c_int * cap)()
    cms = (ctypes.c_double * cap)()
    _check(load().conv_plan_best_m(B, C, Cout, H, W, r, METHODS[method], ctypes.byref(o), ctypes.byref(m),
                                   ctypes.byref(ms), cap, ctypes.byref(n), cm, cms))
    return m.value, ms.value, {cm[k]: cms[k] for k in range(n.value)}


def winograd_matrices(m: int, r: int):
    """(AT [m][t], BT [t][t], G [t][r]) as nested lists of floats (exact rationals in fp64)."""
    t = m + r - 1
    AT = (ctypes.c_double * (m * t))()
    BT = (ctypes.c_double * (t * t))()
    G = (ctypes.c_double * (t * r))()
    _check(load().conv_winograd_matrices(m, r, AT, BT, G))
    return ([list(AT[i * t:(i + 1) * t]) for i in range(m)],
            [list(BT[i * t:(i + 1) * t]) for i in range(t)],
            [list(G[i * r:(i + 1) * r]) for i in range(t)])


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _nbytes(t: torch.Tensor) -> int:
    return t.numel() * t.element_size()


def _check_tensor(x: torch.Tensor, name: str, shape=None):
    if not isinstance(x, torch.Tensor):
        raise TypeError("%s must be a torch.Tensor" % name)
    if x.dtype != torch.float32:
        raise TypeError("%s must be float32" % name)
    if not x.is_cuda:
        raise ValueError("%s must be a CUDA tensor" % name)
    if not x.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    if shape is not None and tuple(x.shape) != tuple(shape):
        raise ValueError("%s has shape %s, expected %s" % (name, tuple(x.shape), tuple(shape)))


class Plan:
    """conv_plan(B, C, C', H, W, r, method, m) -- immutable; owns only host metadata + constants."""

    def __init__(self, B, C, Cout, H, W, r, method: str, m: int = 0, gemm: str = "auto", _nd=None, **opts):
        lib = load()
        h = ctypes.c_void_p()
        o = options(gemm, **opts)
        if _nd is None:
            _check(lib.conv_plan_opts(ctypes.byref(h), B, C, Cout, H, W, r, METHODS[method], m, ctypes.byref(o)))
        else:
            in_shape, k_shape, m_shape = _nd
            nd = len(in_shape)
            ia = (ctypes.c_int * 3)(*in_shape)
            ka = (ctypes.c_int * 3)(*k_shape)
            ma = (ctypes.c_int * 3)(*(m_shape or [1] * nd))
            _check(lib.conv_plan_nd(ctypes.byref(h), nd, B, C, Cout, ia, ka, METHODS[method], ma, ctypes.byref(o)))
        self._h = h
        self.method = method
        info = PlanInfo()
        _check(lib.conv_plan_get_info(h, ctypes.byref(info)))
        self.info = info.as_dict()
        self.workspace_bytes = int(lib.conv_workspace_bytes(h))
        offs = (ctypes.c_size_t * 4)()
        _check(lib.conv_workspace_layout(h, offs))
        self.layout = {"V": offs[0], "Vlo": offs[1], "U": offs[2], "X": offs[3]}
        aux = (ctypes.c_size_t * 2)()
        _check(lib.conv_workspace_aux(h, aux))
        self.layout.update({"vscale": aux[0], "umax": aux[1]})
        self.gemm = gemm
        self.launches = int(lib.conv_forward_launch_count(h))
        if _nd is None:
            self.in_shape = (B, C, H, W)
            self.w_shape = (Cout, C, r, r)
            self.out_shape = (B, Cout, H - r + 1, W - r + 1)
        else:
            self.in_shape = (B, C) + tuple(in_shape)
            self.w_shape = (Cout, C) + tuple(k_shape)
            self.out_shape = (B, Cout) + tuple(a - k + 1 for a, k in zip(in_shape, k_shape))

    @classmethod
    def nd(cls, B, C, Cout, in_shape, kernel_shape, method: str, m=None, gemm: str = "auto", **opts) -> "Plan":
        """conv_plan_nd: 1-3 spatial axes, per-axis kernel sizes and output tiles m."""
        in_shape, kernel_shape = tuple(in_shape), tuple(kernel_shape)
        if len(in_shape) != len(kernel_shape) or not 1 <= len(in_shape) <= 3:
            raise ValueError("in_shape and kernel_shape need the same length 1..3")
        m = None if m is None else tuple(m)
        return cls(B, C, Cout, 0, 0, 0, method, 0, gemm, _nd=(in_shape, kernel_shape, m), **opts)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.conv_destroy(h)
            self._h = None

    def alloc_workspace(self, device=None) -> torch.Tensor:
        n = max(self.workspace_bytes, 16)
        return torch.empty(n, dtype=torch.uint8, device=device or "cuda")

    def forward(self, x, w, out=None, workspace=None, stream=None) -> torch.Tensor:
        _check_tensor(x, "input", self.in_shape)
        _check_tensor(w, "weights", self.w_shape)
        if out is None:
            out = torch.empty(self.out_shape, dtype=torch.float32, device=x.device)
        _check_tensor(out, "out", self.out_shape)
        if workspace is None:
            workspace = self.alloc_workspace(x.device)
        _check(load().conv_forward(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                   workspace.data_ptr(), _nbytes(workspace),
                                   _stream_ptr(stream)))
        return out

    def transform_weights(self, w, workspace, stream=None):
        """NK1 once into the workspace's V region (conv_transform_weights)."""
        _check_tensor(w, "weights", self.w_shape)
        _check(load().conv_transform_weights(self._h, w.data_ptr(), workspace.data_ptr(), _nbytes(workspace),
                                             _stream_ptr(stream)))

    def forward_cached(self, x, workspace, out=None, stream=None) -> torch.Tensor:
        """NK2 -> NK3 -> NK4 against the V left in `workspace` by transform_weights."""
        _check_tensor(x, "input", self.in_shape)
        if out is None:
            out = torch.empty(self.out_shape, dtype=torch.float32, device=x.device)
        _check_tensor(out, "out", self.out_shape)
        _check(load().conv_forward_cached(self._h, x.data_ptr(), out.data_ptr(), workspace.data_ptr(),
                                          _nbytes(workspace), _stream_ptr(stream)))
        return out

    def forward_profiled(self, x, w, out, workspace, stream=None):
        ms = (ctypes.c_float * 4)()
        _check(load().conv_forward_profiled(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                            workspace.data_ptr(), _nbytes(workspace), _stream_ptr(stream), ms))
        return list(ms)

    def forward_host(self, h_in, h_w, h_out, d_in, d_w, d_out, workspace, stream=None):
        """End-to-end call with host (pinned) buffers; async on ``stream``."""
        for t_, n in ((h_in, "h_in"), (h_w, "h_w"), (h_out, "h_out")):
            if t_.is_cuda or not t_.is_contiguous() or t_.dtype != torch.float32:
                raise ValueError("%s must be a contiguous float32 host tensor" % n)
        _check(load().conv_forward_host(self._h, h_in.data_ptr(), h_w.data_ptr(), h_out.data_ptr(),
                                        d_in.data_ptr(), d_w.data_ptr(), d_out.data_ptr(),
                                        workspace.data_ptr(), _nbytes(workspace), _stream_ptr(stream)))

    def run_stage(self, stage: int, x=None, w=None, out=None, workspace=None, stream=None):
        p = lambda t_: 0 if t_ is None else t_.data_ptr()
        _check(load().conv_run_stage(self._h, stage, p(x), p(w), p(out), workspace.data_ptr(),
                                     _nbytes(workspace), _stream_ptr(stream)))

    def capture(self, x, w, out, workspace, steps: int = 1, cached: bool = False) -> "Graph":
        """conv_graph_create: `steps` forwards on these fixed buffers as one CUDA graph."""
        _check_tensor(x, "input", self.in_shape)
        _check_tensor(out, "out", self.out_shape)
        if not cached:
            _check_tensor(w, "weights", self.w_shape)
        h = ctypes.c_void_p()
        _check(load().conv_graph_create(self._h, x.data_ptr(), 0 if cached else w.data_ptr(), out.data_ptr(),
                                        workspace.data_ptr(), _nbytes(workspace), int(steps), int(bool(cached)),
                                        ctypes.byref(h)))
        return Graph(h, (self, x, w, out, workspace))

    def winograd_matrices(self):
        m, t, r = self.info["m"], self.info["t"], self.info["r"]
        AT = (ctypes.c_double * (m * t))()
        BT = (ctypes.c_double * (t * t))()
        G = (ctypes.c_double * (t * r))()
        _check(load().conv_plan_winograd_matrices(self._h, AT, BT, G))
        return list(AT), list(BT), list(G)


class BackwardPlan:
    """conv_plan_backward: gradients of the layer through the fast forward pipeline
    (which = "data": dX from dY and W; "filter": dW from X and dY)."""

    def __init__(self, which: str, B, C, Cout, H, W, r, method: str, m: int = 0, gemm: str = "auto", **opts):
        lib = load()
        h = ctypes.c_void_p()
        o = options(gemm, **opts)
        k = {"data": 1, "filter": 2}[which]
        _check(lib.conv_plan_backward(ctypes.byref(h), k, B, C, Cout, H, W, r, METHODS[method], m, ctypes.byref(o)))
        self._h = h
        self.which = which
        self.workspace_bytes = int(lib.conv_workspace_bytes(h))
        info = PlanInfo()
        _check(lib.conv_plan_get_info(h, ctypes.byref(info)))
        self.info = info.as_dict()
        self.x_shape = (B, C, H, W)
        self.w_shape = (Cout, C, r, r)
        self.y_shape = (B, Cout, H - r + 1, W - r + 1)

    def alloc_workspace(self, device=None) -> torch.Tensor:
        return torch.empty(max(self.workspace_bytes, 16), dtype=torch.uint8, device=device or "cuda")

    def data(self, dy, w, dx=None, workspace=None, stream=None) -> torch.Tensor:
        _check_tensor(dy, "dy", self.y_shape)
        _check_tensor(w, "weights", self.w_shape)
        dx = torch.empty(self.x_shape, device=dy.device) if dx is None else dx
        _check_tensor(dx, "dx", self.x_shape)
        ws = self.alloc_workspace(dy.device) if workspace is None else workspace
        _check(load().conv_backward_data(self._h, dy.data_ptr(), w.data_ptr(), dx.data_ptr(), ws.data_ptr(),
                                         _nbytes(ws), _stream_ptr(stream)))
        return dx

    def filter(self, x, dy, dw=None, workspace=None, stream=None) -> torch.Tensor:
        _check_tensor(x, "x", self.x_shape)
        _check_tensor(dy, "dy", self.y_shape)
        dw = torch.empty(self.w_shape, device=x.device) if dw is None else dw
        _check_tensor(dw, "dw", self.w_shape)
        ws = self.alloc_workspace(x.device) if workspace is None else workspace
        _check(load().conv_backward_filter(self._h, x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(),
                                           _nbytes(ws), _stream_ptr(stream)))
        return dw

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.conv_destroy(h)
            self._h = None


class EShard:
    """conv_eshard_*: element-sharded forward of one rank.  Argument
    marshalling only; parallel.eshard_forward runs the exchanges between the three calls."""

    def __init__(self, world: int, rank: int, batch, C, Cout, H, W, r, method: str, m: int, gemm: str = "auto",
                 **opts):
        lib = load()
        h = ctypes.c_void_p()
        o = options(gemm, **opts)
        ba = (ctypes.c_int * world)(*batch)
        _check(lib.conv_eshard_create(ctypes.byref(h), world, rank, ba, C, Cout, H, W, r, METHODS[method], m,
                                      ctypes.byref(o)))
        self._h = h
        self.world, self.rank, self.batch = world, rank, list(batch)
        wsb = ctypes.c_size_t()
        arrs = [(ctypes.c_size_t * world)() for _ in range(4)]
        _check(lib.conv_eshard_sizes(h, ctypes.byref(wsb), *arrs))
        self.workspace_bytes = int(wsb.value)
        self.u_send, self.u_recv, self.x_send, self.x_recv = ([int(v) for v in a] for a in arrs)
        info = PlanInfo()
        elo, ecnt = ctypes.c_int(), ctypes.c_int()
        _check(lib.conv_eshard_get_info(h, ctypes.byref(info), ctypes.byref(elo), ctypes.byref(ecnt)))
        self.info = info.as_dict()
        self.e_lo, self.e_count = elo.value, ecnt.value
        B = batch[rank]
        self.in_shape = (B, C, H, W)
        self.w_shape = (Cout, C, r, r)
        self.out_shape = (B, Cout, H - r + 1, W - r + 1)

    def alloc_workspace(self, device=None) -> torch.Tensor:
        return torch.empty(max(self.workspace_bytes, 16), dtype=torch.uint8, device=device or "cuda")

    def forward_a(self, x, w, u_send, umax_out, workspace, stream=None):
        _check_tensor(x, "input", self.in_shape)
        _check_tensor(w, "weights", self.w_shape)
        _check(load().conv_eshard_forward_a(self._h, x.data_ptr(), w.data_ptr(), u_send.data_ptr(),
                                            umax_out.data_ptr(), workspace.data_ptr(), _nbytes(workspace),
                                            _stream_ptr(stream)))

    def forward_b(self, u_recv, umax_all, x_send, workspace, stream=None):
        _check(load().conv_eshard_forward_b(self._h, u_recv.data_ptr(), umax_all.data_ptr(), x_send.data_ptr(),
                                            workspace.data_ptr(), _nbytes(workspace), _stream_ptr(stream)))

    def forward_a_peer(self, x, w, u_recv_peers, umax_out, workspace, stream=None):
        """u_recv_peers: per rank k, the device address (int) of rank k's u_recv buffer mapped
        into this process (IPCBuffer.peer_ptrs)."""
        _check_tensor(x, "input", self.in_shape)
        _check_tensor(w, "weights", self.w_shape)
        arr = (ctypes.c_void_p * self.world)(*u_recv_peers)
        _check(load().conv_eshard_forward_a_peer(self._h, x.data_ptr(), w.data_ptr(), arr, umax_out.data_ptr(),
                                                 workspace.data_ptr(), _nbytes(workspace), _stream_ptr(stream)))

    def forward_b_peer(self, u_recv_ptr, umax_all, x_recv_peers, workspace, stream=None):
        arr = (ctypes.c_void_p * self.world)(*x_recv_peers)
        _check(load().conv_eshard_forward_b_peer(self._h, u_recv_ptr, umax_all.data_ptr(), arr,
                                                 workspace.data_ptr(), _nbytes(workspace), _stream_ptr(stream)))

    def forward_c(self, x_recv, out, workspace, stream=None):
        _check_tensor(out, "out", self.out_shape)
        xr = x_recv if isinstance(x_recv, int) else x_recv.data_ptr()  # tensor or IPCBuffer.ptr
        _check(load().conv_eshard_forward_c(self._h, xr, out.data_ptr(), workspace.data_ptr(),
                                            _nbytes(workspace), _stream_ptr(stream)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.conv_eshard_destroy(h)
            self._h = None


class IPCBuffer:
    """Device memory shareable between processes (conv_ipc_alloc): `handle` (64 bytes) goes to
    the peers, which map it with IPCBuffer.open(handle); `ptr` is this process's address."""

    def __init__(self, nbytes: int):
        lib = load()
        p = ctypes.c_void_p()
        h = (ctypes.c_char * 64)()
        _check(lib.conv_ipc_alloc(max(int(nbytes), 16), ctypes.byref(p), h))
        self.ptr, self.handle, self.nbytes, self._owned = int(p.value), bytes(h), int(nbytes), True

    @staticmethod
    def open(handle: bytes) -> int:
        """Map a peer's buffer; returns its device address in this process."""
        p = ctypes.c_void_p()
        h = (ctypes.c_char * 64).from_buffer_copy(handle)
        _check(load().conv_ipc_open(h, ctypes.byref(p)))
        return int(p.value)

    @staticmethod
    def close(ptr: int):
        _check(load().conv_ipc_close(ctypes.c_void_p(ptr)))

    def __del__(self):
        if getattr(self, "_owned", False) and _lib is not None:
            _lib.conv_ipc_free(ctypes.c_void_p(self.ptr))
            self._owned = False


class Graph:
    """An instantiated CUDA graph of forward passes (conv_graph_*); keeps its buffers alive."""

    def __init__(self, h, keep):
        self._h = h
        self._keep = keep

    def launch(self, stream=None):
        _check(load().conv_graph_launch(self._h, _stream_ptr(stream)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.conv_graph_destroy(h)
            self._h = None


class StageTimer:
    """conv_timer_*: per-stage CUDA-event timing of conv_forward_timed calls, read once
    (synchronising) after a timed loop."""

    def __init__(self, max_launches: int):
        h = ctypes.c_void_p()
        _check(load().conv_timer_create(ctypes.byref(h), int(max_launches)))
        self._h = h

    def forward(self, plan: "Plan", x, w, out, workspace, stream=None):
        _check(load().conv_forward_timed(plan._h, x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                         workspace.data_ptr(), _nbytes(workspace), _stream_ptr(stream),
                                         self._h))

    def read(self):
        ms = (ctypes.c_float * 4)()
        n = ctypes.c_int()
        _check(load().conv_timer_read(self._h, ms, ctypes.byref(n)))
        return list(ms), n.value

    def reset(self):
        load().conv_timer_reset(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.conv_timer_destroy(h)
            self._h = None


_PLAN_CACHE: dict = {}
_PLAN_CACHE_MAX = 32


def forward(x: torch.Tensor, w: torch.Tensor, method: str = "winograd", m: int = 4,
            gemm: str = "auto") -> torch.Tensor:
    """One-shot forward: plans (cached by shape, method, m, gemm and device), allocates the
    workspace and output with torch, runs on the current stream.  m = 0: the planner's tile;
    method = "auto": the planner's method and tile (conv_plan_best_method)."""
    B, C, H, W = x.shape
    Cout, C2, r, _ = w.shape
    if C2 != C:
        raise ValueError("channel mismatch")
    if method == "auto":
        method, m, _ = best_method(B, C, Cout, H, W, r, gemm)
    key = (B, C, Cout, H, W, r, method, m, gemm, x.device.index if x.is_cuda else -1)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        if len(_PLAN_CACHE) >= _PLAN_CACHE_MAX:
            _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
        plan = _PLAN_CACHE[key] = Plan(B, C, Cout, H, W, r, method, m, gemm)
    return plan.forward(x, w)
